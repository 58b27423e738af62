// hw_small2d.cu — persistent small-grid 2D acoustic kernel (binary16), sm_100a.
//
// For grids whose rows fit in the CTAs' shared memory (the reference presets' 150^2 /
// 600^2, BASELINE config 1) the per-step cost of the streaming kernel is latency, not
// bandwidth.  Here ONE cooperative launch runs every step: each CTA keeps its band of
// rows of all six fields resident in shared memory, and per step
//   1. ingests its neighbours' boundary rows (3 rows of p, vy, rvy above / below) from a
//      global exchange area (double-buffered by step parity),
//   2. updates vx (own rows), vy (own rows + the 2 / 1 halo rows, recomputed redundantly
//      like the fused slab kernel), p (own rows) -- the reference's step
//      (acoustic.py:162-181) with the same helpers, identical bits,
//   3. publishes its new boundary rows, records failures / energy partials / traces,
//   4. meets the other CTAs at a grid barrier; after it every CTA sees the same failure
//      record, so the state stops exactly after the failing step (acoustic.py:208-229).
// The barrier spin is bounded: a broken barrier traps instead of hanging the GPU.
#include <cuda_runtime.h>

#include "hw_fused2d.h"
#include "hw_params.h"
#include "hw_stream.cuh"
#include "../../include/halfwave_b200.h"
#include <string.h>

namespace hw {

constexpr int SX_ROWS = 12;  // published rows per CTA: p top 3 / bottom 3, vy top 1 / bottom 2, rvy likewise

struct SmallParams {
    AcFusedParams F;          // A buffers (in == out), medium, receivers, control, energy
    __half* xch;              // exchange area [2][nb][SX_ROWS][nx]
    unsigned int* gbar;       // grid barrier {count, generation}
    const double* src;        // source samples [nt] (device)
    double* partials2;        // second energy-partial buffer (alternating sample steps)
    int32_t every, energy;
};

__device__ __forceinline__ void grid_barrier(unsigned int* gbar, int nb) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned int* genp = gbar + 1;
        const unsigned int gen = *genp;
        __threadfence();
        if (atomicAdd(gbar, 1u) == (unsigned int)(nb - 1)) {
            gbar[0] = 0u;
            __threadfence();
            atomicAdd(gbar + 1, 1u);
        } else {
            unsigned long long spins = 0;
            while (*genp == gen) {
                __nanosleep(64);
                if (++spins > (1ull << 26)) __trap();  // never hang the GPU on a broken barrier
            }
        }
        __threadfence();
    }
    __syncthreads();
}

// x taps of the pair at x (row in shared memory, periodic x): to_int shifts (-2..1), else (-1..2)
template <int ORDER>
__device__ __forceinline__ EH2 s_xfold(const __half c[4], const __half* row, int x, int xl, int xr, bool to_int) {
    EH2 a, b, d;
    a.h2 = *reinterpret_cast<const __half2*>(row + xl);
    b.h2 = *reinterpret_cast<const __half2*>(row + x);
    d.h2 = *reinterpret_cast<const __half2*>(row + xr);
    return to_int ? e_fold<ORDER>(c, a, vshift<16, 2>(a, b), b, vshift<16, 2>(b, d))
                  : e_fold<ORDER>(c, vshift<16, 2>(a, b), b, vshift<16, 2>(b, d), d);
}

__device__ __forceinline__ EH2 s_ld(const __half* p) {
    EH2 r;
    r.h2 = *reinterpret_cast<const __half2*>(p);
    return r;
}
__device__ __forceinline__ void s_st(__half* p, EH2 v) { *reinterpret_cast<__half2*>(p) = v.h2; }

// exchange-area reads bypass L1 (not coherent across SMs; a parity buffer is re-read two steps later)
__device__ __forceinline__ EH2 s_ldx(const __half* p) {
    const unsigned int u = __ldcg(reinterpret_cast<const unsigned int*>(p));
    EH2 r;
    *reinterpret_cast<unsigned int*>(&r.h2) = u;
    return r;
}

template <int V, bool RM>
__device__ __forceinline__ void s_update(EH2 rhs, const PlaneView& pv, int row, int x, __half2 dt2, int src_lane,
                                         __half srch, double src, EH2& u, EH2& t) {
    if constexpr (RM) {
        e_finish_rc<V>(rhs, __ldg(pv.rcp + (int64_t)row * pv.ss), dt2, src_lane, srch, u, t);
    } else {
        finish<16, 16, 2>(rhs, &pv, row, 0, x, dt2.x, V, src_lane, src, u, t);
    }
}

template <int V, int ORDER, bool RM>
__global__ void __launch_bounds__(1024, 1) k_ac2d_small(SmallParams S, int64_t nt) {
    const AcFusedParams& P = S.F;
    extern __shared__ __align__(16) unsigned char smem[];
    const int nx = (int)P.nx, ns = (int)P.ns, nb = gridDim.x, b = blockIdx.x;
    const int64_t pitch = P.pitch;
    const int g0 = (int)((int64_t)b * ns / nb), R = (int)((int64_t)(b + 1) * ns / nb) - g0;
    const int above = (b + nb - 1) % nb, below = (b + 1) % nb;
    const int tid = threadIdx.x, x = 2 * tid;
    constexpr bool comp = V != 0;
    // shared rows: p [-3, R+3), vx [0, R), vy [-2, R+1), rp [0, R), rvx [0, R), rvy [-2, R+1)
    __half* sp = reinterpret_cast<__half*>(smem) + 3 * nx;
    __half* svx = sp + (R + 3) * nx;
    __half* svy = svx + R * nx + 2 * nx;
    __half* srp = svy + (R + 1) * nx;
    __half* srvx = srp + R * nx;
    __half* srvy = srvx + R * nx + 2 * nx;
    auto grow = [&](int r) { r += g0; return r < 0 ? r + ns : (r >= ns ? r - ns : r); };  // global row (periodic)
    // load the band from the A buffers
    for (int r = 0; r < R; r++) {
        const int64_t o = (int64_t)(g0 + r) * pitch + x;
        s_st(sp + r * nx + x, s_ld(P.in[0] + o));
        s_st(svx + r * nx + x, s_ld(P.in[1] + o));
        s_st(svy + r * nx + x, s_ld(P.in[2] + o));
        if (comp) {
            s_st(srp + r * nx + x, s_ld(P.in[3] + o));
            s_st(srvx + r * nx + x, s_ld(P.in[4] + o));
            s_st(srvy + r * nx + x, s_ld(P.in[5] + o));
        }
    }
    auto xrow = [&](int par, int blk, int k) { return S.xch + ((int64_t)(par * nb + blk) * SX_ROWS + k) * nx; };
    auto publish = [&](int par) {  // rows the neighbours need, from shared memory
        for (int k = 0; k < 3; k++) {
            s_st(xrow(par, b, k) + x, s_ld(sp + k * nx + x));
            s_st(xrow(par, b, 3 + k) + x, s_ld(sp + (R - 3 + k) * nx + x));
        }
        s_st(xrow(par, b, 6) + x, s_ld(svy + x));
        s_st(xrow(par, b, 7) + x, s_ld(svy + (R - 2) * nx + x));
        s_st(xrow(par, b, 8) + x, s_ld(svy + (R - 1) * nx + x));
        if (comp) {
            s_st(xrow(par, b, 9) + x, s_ld(srvy + x));
            s_st(xrow(par, b, 10) + x, s_ld(srvy + (R - 2) * nx + x));
            s_st(xrow(par, b, 11) + x, s_ld(srvy + (R - 1) * nx + x));
        }
    };
    __syncthreads();
    publish(0);
    grid_barrier(S.gbar, nb);

    __half c[4];
#pragma unroll
    for (int j = 0; j < 4; j++) c[j] = lconst<16>(P.k, j);
    const __half2 dt2 = __half2half2(lconst<16>(P.k, 4));
    const int xl = x == 0 ? nx - 2 : x - 2, xr = x + 2 >= nx ? 0 : x + 2;
    const bool src_col = P.has_src && P.src_x >= x && P.src_x < x + 2;
    const int src_lane = (int)(P.src_x - x) & 1;
    const int src_row = (int)P.src_s - g0;  // local row of the point source (if in this band)
    const bool erow = (P.e_beta.sx | P.e_rho_x.sx | P.e_rho_s.sx) == 0;
    __half2 acc[6];
#pragma unroll
    for (int q = 0; q < 6; q++) acc[q] = __float2half2_rn(0.f);

    for (int64_t n = 0; n < nt; n++) {
        const int par = (int)(n & 1);
        // 1. ingest the neighbours' boundary rows of step n
        for (int k = 0; k < 3; k++) {
            s_st(sp + (k - 3) * nx + x, s_ldx(xrow(par, above, 3 + k) + x));
            s_st(sp + (R + k) * nx + x, s_ldx(xrow(par, below, k) + x));
        }
        s_st(svy - 2 * nx + x, s_ldx(xrow(par, above, 7) + x));
        s_st(svy - nx + x, s_ldx(xrow(par, above, 8) + x));
        s_st(svy + R * nx + x, s_ldx(xrow(par, below, 6) + x));
        if (comp) {
            s_st(srvy - 2 * nx + x, s_ldx(xrow(par, above, 10) + x));
            s_st(srvy - nx + x, s_ldx(xrow(par, above, 11) + x));
            s_st(srvy + R * nx + x, s_ldx(xrow(par, below, 9) + x));
        }
        __syncthreads();
        const double srcv = S.src ? S.src[n] : 0.0;
        const __half srch = __double2half(srcv);
        const int sample = S.energy && ((n + 1) % S.every == 0);
        double e[NCOMP] = {0.0, 0.0, 0.0, 0.0, 0.0};
        // 2a. vx own rows, vy rows [-2, R+1) (acoustic.py:167-170)
        for (int r = 0; r < R; r++) {
            const EH2 d = s_xfold<ORDER>(c, sp + r * nx, x, xl, xr, false);
            EH2 v = s_ld(svx + r * nx + x);
            EH2 t = comp ? s_ld(srvx + r * nx + x) : EH2{};
            s_update<V, RM>(d, P.rho_x, grow(r), x, dt2, -1, srch, 0.0, v, t);
            s_st(svx + r * nx + x, v);
            acc[1] = __hmax2_nan(acc[1], __habs2(v.h2));
            if (comp) {
                s_st(srvx + r * nx + x, t);
                acc[4] = __hmax2_nan(acc[4], __habs2(t.h2));
            }
            if (sample) {
                const float2 f = __half22float2(v.h2);
                const double a = (double)__fmul_rn(f.x, f.x), bb = (double)__fmul_rn(f.y, f.y);
                if (erow) e[1] += p64(P.e_rho_x, grow(r), 0, 0) * (a + bb);
                else e[1] += p64(P.e_rho_x, grow(r), 0, x) * a + p64(P.e_rho_x, grow(r), 0, x + 1) * bb;
            }
        }
        for (int r = -2; r < R + 1; r++) {
            const EH2 d = e_fold<ORDER>(c, s_ld(sp + (r - 1) * nx + x), s_ld(sp + r * nx + x), s_ld(sp + (r + 1) * nx + x),
                                        s_ld(sp + (r + 2) * nx + x));
            EH2 v = s_ld(svy + r * nx + x);
            EH2 t = comp ? s_ld(srvy + r * nx + x) : EH2{};
            s_update<V, RM>(d, P.rho_s, grow(r), x, dt2, -1, srch, 0.0, v, t);
            s_st(svy + r * nx + x, v);
            if (comp) s_st(srvy + r * nx + x, t);
            if (r >= 0 && r < R) {
                acc[2] = __hmax2_nan(acc[2], __habs2(v.h2));
                if (comp) acc[5] = __hmax2_nan(acc[5], __habs2(t.h2));
                if (sample) {
                    const float2 f = __half22float2(v.h2);
                    const double a = (double)__fmul_rn(f.x, f.x), bb = (double)__fmul_rn(f.y, f.y);
                    if (erow) e[2] += p64(P.e_rho_s, grow(r), 0, 0) * (a + bb);
                    else e[2] += p64(P.e_rho_s, grow(r), 0, x) * a + p64(P.e_rho_s, grow(r), 0, x + 1) * bb;
                }
            }
        }
        __syncthreads();
        // 2b. p own rows: fl(ddx vx + dds vy) (+ src at (n+1/2) dt) (acoustic.py:172-181)
        for (int k = 0; k < R; k++) {
            const EH2 gx = s_xfold<ORDER>(c, svx + k * nx, x, xl, xr, true);
            const EH2 gs = e_fold<ORDER>(c, s_ld(svy + (k - 2) * nx + x), s_ld(svy + (k - 1) * nx + x),
                                         s_ld(svy + k * nx + x), s_ld(svy + (k + 1) * nx + x));
            const EH2 pold = s_ld(sp + k * nx + x);
            EH2 pn = pold;
            EH2 t = comp ? s_ld(srp + k * nx + x) : EH2{};
            const int sl = (src_col && k == src_row && srcv != 0.0) ? src_lane : -1;
            s_update<V, RM>(EO2::add(gx, gs), P.beta, grow(k), x, dt2, sl, srch, srcv, pn, t);
            acc[0] = __hmax2_nan(acc[0], __habs2(pn.h2));
            if (comp) {
                s_st(srp + k * nx + x, t);
                acc[3] = __hmax2_nan(acc[3], __habs2(t.h2));
            }
            if (sample) {
                const float2 a = __half22float2(pold.h2), bb = __half22float2(pn.h2);
                const double u0 = (double)__fmul_rn(a.x, bb.x), u1 = (double)__fmul_rn(a.y, bb.y);
                if (erow) e[0] += p64(P.e_beta, grow(k), 0, 0) * (u0 + u1);
                else e[0] += p64(P.e_beta, grow(k), 0, x) * u0 + p64(P.e_beta, grow(k), 0, x + 1) * u1;
            }
            // receiver traces of p after the step (acoustic.py:217-218)
            int rc = rec_lower(P.rec, 0, P.n_rec, g0 + k, x);
            for (; rc < P.n_rec && __ldg(P.rec + 3 * rc) == g0 + k && __ldg(P.rec + 3 * rc + 1) < x + 2; rc++) {
                const int o = __ldg(P.rec + 3 * rc + 1) - x;
                P.traces[(int64_t)__ldg(P.rec + 3 * rc + 2) * P.nt + n] = (double)__half2float(pn.e[o]);
            }
            s_st(sp + k * nx + x, pn);  // p rows k-1 .. are no longer read (vy of this step is done)
        }
        __syncthreads();
        // 3. publish, failures, energy partials
        publish((int)((n + 1) & 1));
        unsigned int mask = 0;
#pragma unroll
        for (int q = 0; q < 6; q++) {
            const unsigned int bits = *reinterpret_cast<const unsigned int*>(&acc[q]);
            if (((bits & 0x7c00u) == 0x7c00u) || ((bits & 0x7c000000u) == 0x7c000000u)) mask |= 1u << q;
        }
        record_failure(P.ctrl, n, mask);
        double* part = (n / S.every) & 1 ? S.partials2 : P.partials;
        if (sample) block_partials(e, part);
        // 4. one grid barrier per step; then everyone sees the same failure record
        grid_barrier(S.gbar, nb);
        if (sample && b == 0) {
            const double tsum = finalize_partials(part, nb);
            if (tid == 0) P.e_vals[(n + 1) / S.every] = P.scale * tsum;
        }
        if (*reinterpret_cast<const volatile int64_t*>(&P.ctrl->fail_step) <= n) break;
    }
    // write the band back to the A buffers (out == in)
    for (int r = 0; r < R; r++) {
        const int64_t o = (int64_t)(g0 + r) * pitch + x;
        s_st(P.out[0] + o, s_ld(sp + r * nx + x));
        s_st(P.out[1] + o, s_ld(svx + r * nx + x));
        s_st(P.out[2] + o, s_ld(svy + r * nx + x));
        if (comp) {
            s_st(P.out[3] + o, s_ld(srp + r * nx + x));
            s_st(P.out[4] + o, s_ld(srvx + r * nx + x));
            s_st(P.out[5] + o, s_ld(srvy + r * nx + x));
        }
    }
}

// ---------------------------------------------------------------- elastic (2D, velocity-stress)
// Same design for ElasticSolver._step_work (elastic.py:176-238): per step two neighbour
// exchanges and two grid barriers (stress halos before the velocity phase, velocity halos
// before the stress phase; each CTA updates only its own rows, so single-buffered exchange
// rows suffice).  Free surfaces: the edge CTAs fill their outer halos with the reference's
// images (stencil.py:121-144: odd sxy / syy, even vx / vy), the surface rows use the
// plane-stress modulus for sxx and a zero increment for syy (elastic.py:215-230).
constexpr int SE_ROWS = 12;  // published rows: sxy 1 + 2, syy 2 + 1, vx 2 + 1, vy 1 + 2

struct SmallElParams {
    ElParams P;
    double* traces;           // [n_rec][nt]
    const int* rec;           // receivers sorted by (row, x)
    int32_t n_rec, every, energy, pad;
    int64_t nt;
    double* e_vals;
    double scale;
    __half* xch;              // [nb][SE_ROWS][nx]
    unsigned int* gbar;
    const double* src;        // [nt]
    double* partials2;
};

template <int V, int ORDER>
__global__ void __launch_bounds__(1024, 1) k_el2d_small(SmallElParams S, int64_t nt) {
    const ElParams& P = S.P;
    extern __shared__ __align__(16) unsigned char smem[];
    const int nx = (int)P.g.nx, nh = (int)P.vs.rows, nb = gridDim.x, b = blockIdx.x;  // nh: half rows (= ns)
    const int64_t pitch = P.g.pitch;
    const bool fs = P.fs != 0, top = b == 0, bot = b == nb - 1;
    const int g0 = (int)((int64_t)b * nh / nb), Rh = (int)((int64_t)(b + 1) * nh / nb) - g0;
    const int Ri = Rh + ((fs && bot) ? 1 : 0);  // the last band also owns the bottom surface row
    const int above = (b + nb - 1) % nb, below = (b + 1) % nb;
    const int tid = threadIdx.x, x = 2 * tid;
    constexpr bool comp = V != 0;
    // shared rows: syy [-1, Rh+2), sxy [-2, Ri+1), vx [-1, Rh+2), vy [-2, Ri+1), sxx / residuals own rows
    __half* base = reinterpret_cast<__half*>(smem);
    int off = 0;
    auto alloc = [&](int lo, int hi) { __half* p = base + (off - lo) * nx; off += hi - lo; return p; };
    __half* syy = alloc(-1, Rh + 2);
    __half* sxy = alloc(-2, Ri + 1);
    __half* vx = alloc(-1, Rh + 2);
    __half* vy = alloc(-2, Ri + 1);
    __half* sxx = alloc(0, Ri);
    __half* rvx = alloc(0, Ri);
    __half* rvy = alloc(0, Rh);
    __half* rsxx = alloc(0, Ri);
    __half* rsyy = alloc(0, Ri);
    __half* rsxy = alloc(0, Rh);
    auto gl = [&](const FieldView& f, int r) { return reinterpret_cast<__half*>(f.base) + (int64_t)(g0 + r) * pitch + x; };
    for (int r = 0; r < Ri; r++) {  // load the band from the A buffers
        s_st(vx + r * nx + x, s_ld(gl(P.vx, r)));
        s_st(sxx + r * nx + x, s_ld(gl(P.sxx, r)));
        s_st(syy + r * nx + x, s_ld(gl(P.sss, r)));
        if (comp) {
            s_st(rvx + r * nx + x, s_ld(gl(P.rvx, r)));
            s_st(rsxx + r * nx + x, s_ld(gl(P.rsxx, r)));
            s_st(rsyy + r * nx + x, s_ld(gl(P.rsss, r)));
        }
    }
    for (int r = 0; r < Rh; r++) {
        s_st(vy + r * nx + x, s_ld(gl(P.vs, r)));
        s_st(sxy + r * nx + x, s_ld(gl(P.sxs, r)));
        if (comp) {
            s_st(rvy + r * nx + x, s_ld(gl(P.rvs, r)));
            s_st(rsxy + r * nx + x, s_ld(gl(P.rsxs, r)));
        }
    }
    auto xr = [&](int blk, int k) { return S.xch + ((int64_t)blk * SE_ROWS + k) * nx + x; };
    auto neg = [](EH2 v) { return vneg<16, 2>(v); };
    // stress rows for the neighbours: sxy row 0 | sxy rows Rh-2, Rh-1 | syy rows 0, 1 | syy row Ri-1
    auto publish_s = [&]() {
        s_st(xr(b, 0), s_ld(sxy + x));
        s_st(xr(b, 1), s_ld(sxy + (Rh - 2) * nx + x));
        s_st(xr(b, 2), s_ld(sxy + (Rh - 1) * nx + x));
        s_st(xr(b, 3), s_ld(syy + x));
        s_st(xr(b, 4), s_ld(syy + nx + x));
        s_st(xr(b, 5), s_ld(syy + (Ri - 1) * nx + x));
    };
    // velocity rows: vx rows 0, 1 | vx row Ri-1 | vy row 0 | vy rows Rh-2, Rh-1
    auto publish_v = [&]() {
        s_st(xr(b, 6), s_ld(vx + x));
        s_st(xr(b, 7), s_ld(vx + nx + x));
        s_st(xr(b, 8), s_ld(vx + (Ri - 1) * nx + x));
        s_st(xr(b, 9), s_ld(vy + x));
        s_st(xr(b, 10), s_ld(vy + (Rh - 2) * nx + x));
        s_st(xr(b, 11), s_ld(vy + (Rh - 1) * nx + x));
    };
    auto ingest_s = [&]() {  // sxy rows -2, -1 and [Rh, Ri+1); syy row -1 and [Ri, Rh+2)
        if (fs && top) {
            s_st(sxy - nx + x, neg(s_ld(sxy + x)));
            s_st(sxy - 2 * nx + x, neg(s_ld(sxy + nx + x)));
            s_st(syy - nx + x, neg(s_ld(syy + nx + x)));
        } else {
            s_st(sxy - 2 * nx + x, s_ldx(xr(above, 1)));
            s_st(sxy - nx + x, s_ldx(xr(above, 2)));
            s_st(syy - nx + x, s_ldx(xr(above, 5)));
        }
        if (fs && bot) {  // sxy rows ns, ns+1; syy row ns+1 (images about the bottom surface)
            s_st(sxy + Rh * nx + x, neg(s_ld(sxy + (Rh - 1) * nx + x)));
            s_st(sxy + (Rh + 1) * nx + x, neg(s_ld(sxy + (Rh - 2) * nx + x)));
            s_st(syy + (Rh + 1) * nx + x, neg(s_ld(syy + (Ri - 2) * nx + x)));
        } else {
            s_st(sxy + Rh * nx + x, s_ldx(xr(below, 0)));
            s_st(syy + Ri * nx + x, s_ldx(xr(below, 3)));
            s_st(syy + (Ri + 1) * nx + x, s_ldx(xr(below, 4)));
        }
    };
    auto ingest_v = [&]() {  // vx row -1 and [Ri, Rh+2); vy rows -2, -1 and [Rh, Ri+1)
        if (fs && top) {
            s_st(vx - nx + x, s_ld(vx + nx + x));
            s_st(vy - nx + x, s_ld(vy + x));
            s_st(vy - 2 * nx + x, s_ld(vy + nx + x));
        } else {
            s_st(vx - nx + x, s_ldx(xr(above, 8)));
            s_st(vy - 2 * nx + x, s_ldx(xr(above, 10)));
            s_st(vy - nx + x, s_ldx(xr(above, 11)));
        }
        if (fs && bot) {
            s_st(vx + (Rh + 1) * nx + x, s_ld(vx + (Ri - 2) * nx + x));
            s_st(vy + Rh * nx + x, s_ld(vy + (Rh - 1) * nx + x));
            s_st(vy + (Rh + 1) * nx + x, s_ld(vy + (Rh - 2) * nx + x));
        } else {
            s_st(vx + Ri * nx + x, s_ldx(xr(below, 6)));
            s_st(vx + (Ri + 1) * nx + x, s_ldx(xr(below, 7)));
            s_st(vy + Rh * nx + x, s_ldx(xr(below, 9)));
        }
    };
    __syncthreads();
    publish_s();
    grid_barrier(S.gbar, nb);

    __half c[4];
#pragma unroll
    for (int j = 0; j < 4; j++) c[j] = lconst<16>(P.k, j);
    const __half2 dt2 = __half2half2(lconst<16>(P.k, 4));
    const int xl = x == 0 ? nx - 2 : x - 2, xrr = x + 2 >= nx ? 0 : x + 2;
    const bool src_col = P.src_x >= x && P.src_x < x + 2;
    const int src_lane = (int)(P.src_x - x) & 1, src_row = (int)P.src_s - g0;
    const int ni = (int)P.sxx.nglob;  // integer rows globally (ns + 1 with free surfaces)
    __half2 acc[10];
#pragma unroll
    for (int q = 0; q < 10; q++) acc[q] = __float2half2_rn(0.f);
    auto track = [&](int q, EH2 v) { acc[q] = __hmax2_nan(acc[q], __habs2(v.h2)); };

    for (int64_t n = 0; n < nt; n++) {
        const double srcv = S.src ? S.src[n] : 0.0;
        const __half srch = __double2half(srcv);
        const int sample = S.energy && ((n + 1) % S.every == 0);
        double e[NCOMP] = {0.0, 0.0, 0.0, 0.0, 0.0};
        // ---- velocity phase (stress halos of step n)
        ingest_s();
        __syncthreads();
        for (int r = 0; r < Ri; r++) {  // vx = fl(fl(ddx sxx + dds sxy) / rho_x dt)
            const EH2 a = EO2::add(s_xfold<ORDER>(c, sxx + r * nx, x, xl, xrr, false),
                                   e_fold<ORDER>(c, s_ld(sxy + (r - 2) * nx + x), s_ld(sxy + (r - 1) * nx + x),
                                                 s_ld(sxy + r * nx + x), s_ld(sxy + (r + 1) * nx + x)));
            EH2 v = s_ld(vx + r * nx + x), t = comp ? s_ld(rvx + r * nx + x) : EH2{};
            finish<16, 16, 2>(a, &P.rho_x, g0 + r, 0, x, dt2.x, V, -1, 0.0, v, t);
            s_st(vx + r * nx + x, v);
            track(0, v);
            if (comp) {
                s_st(rvx + r * nx + x, t);
                track(5, t);
            }
        }
        for (int r = 0; r < Rh; r++) {  // vy = fl(fl(ddx sxy + dds syy) (+ src) / rho_y dt)
            const EH2 a = EO2::add(s_xfold<ORDER>(c, sxy + r * nx, x, xl, xrr, true),
                                   e_fold<ORDER>(c, s_ld(syy + (r - 1) * nx + x), s_ld(syy + r * nx + x),
                                                 s_ld(syy + (r + 1) * nx + x), s_ld(syy + (r + 2) * nx + x)));
            EH2 v = s_ld(vy + r * nx + x), t = comp ? s_ld(rvy + r * nx + x) : EH2{};
            const int sl = (P.src_kind == HW_SRC_VSLOW && src_col && r == src_row && srcv != 0.0) ? src_lane : -1;
            finish<16, 16, 2>(a, &P.rho_s, g0 + r, 0, x, dt2.x, V, sl, srcv, v, t);
            s_st(vy + r * nx + x, v);
            track(1, v);
            if (comp) {
                s_st(rvy + r * nx + x, t);
                track(6, t);
            }
            // receiver traces of vy after the step (elastic.py:283-284)
            for (int q = rec_lower(S.rec, 0, S.n_rec, g0 + r, x);
                 q < S.n_rec && __ldg(S.rec + 3 * q) == g0 + r && __ldg(S.rec + 3 * q + 1) < x + 2; q++)
                S.traces[(int64_t)__ldg(S.rec + 3 * q + 2) * S.nt + n] = (double)__half2float(v.e[__ldg(S.rec + 3 * q + 1) - x]);
        }
        __syncthreads();
        publish_v();
        grid_barrier(S.gbar, nb);
        // ---- stress phase (velocity halos of step n+1/2)
        ingest_v();
        __syncthreads();
        for (int r = 0; r < Ri; r++) {  // sxx, syy at integer rows
            const int sg = g0 + r;
            const bool surf = fs && (sg == 0 || sg == ni - 1);
            const EH2 dvx = s_xfold<ORDER>(c, vx + r * nx, x, xl, xrr, true);
            const EH2 dvs = e_fold<ORDER>(c, s_ld(vy + (r - 2) * nx + x), s_ld(vy + (r - 1) * nx + x),
                                          s_ld(vy + r * nx + x), s_ld(vy + (r + 1) * nx + x));
            const EH2 stiff = pload<16, 2>(P.stiff, sg, 0, x), lam = pload<16, 2>(P.lam, sg, 0, x);
            EH2 a1, a2;
            if (surf) {
                a1 = EO2::mul(pload<16, 2>(P.ep, sg == 0 ? 0 : 1, 0, x), dvx);
                a2 = vsplat<16, 2>(lane<16>::zero());
            } else {
                a1 = EO2::add(EO2::mul(stiff, dvx), EO2::mul(lam, dvs));
                a2 = EO2::add(EO2::mul(lam, dvx), EO2::mul(stiff, dvs));
            }
            const int sl = (P.src_kind == HW_SRC_EXPLOSIVE && src_col && r == src_row && srcv != 0.0) ? src_lane : -1;
            const EH2 xo = s_ld(sxx + r * nx + x), so = s_ld(syy + r * nx + x);
            EH2 xn = xo, sn = so;
            EH2 t1 = comp ? s_ld(rsxx + r * nx + x) : EH2{}, t2 = comp ? s_ld(rsyy + r * nx + x) : EH2{};
            finish<16, 16, 2>(a1, nullptr, sg, 0, x, dt2.x, V, sl, srcv, xn, t1);
            finish<16, 16, 2>(a2, nullptr, sg, 0, x, dt2.x, V, sl, srcv, sn, t2);
            s_st(sxx + r * nx + x, xn);
            s_st(syy + r * nx + x, sn);
            track(2, xn);
            track(3, sn);
            if (comp) {
                s_st(rsxx + r * nx + x, t1);
                s_st(rsyy + r * nx + x, t2);
                track(7, t1);
                track(8, t2);
            }
            if (sample) {  // kinetic x + strain energy at this integer row (diagnostics.py:100-162)
                const EH2 vxo = s_ld(vx + r * nx + x);
#pragma unroll
                for (int k = 0; k < 2; k++) {
                    const int xi = x + k;
                    const double w = surf ? 0.5 : 1.0;
                    const double v = (double)__half2float(vxo.e[k]);
                    e[0] += (w * p64(P.e_rho_x, sg, 0, xi)) * (v * v);
                    const double lamd = p64(P.e_lam, sg, 0, xi), mu = p64(P.e_mu, sg, 0, xi);
                    const double xa = (double)__half2float(xo.e[k]), x1 = (double)__half2float(xn.e[k]);
                    const double sa = (double)__half2float(so.e[k]), s1 = (double)__half2float(sn.e[k]);
                    const double stiffd = lamd + 2.0 * mu, dd = 4.0 * mu * (lamd + mu);
                    double val;
                    if (mu == 0.0) val = surf ? 0.0 : (xa * x1) / (lamd + mu);
                    else if (surf) val = xa * x1 * stiffd / dd;
                    else val = (stiffd * (xa * x1 + sa * s1) - lamd * (xa * s1 + sa * x1)) / dd;
                    if (surf) val = 0.5 * val;
                    e[3] += val;
                }
            }
        }
        for (int r = 0; r < Rh; r++) {  // sxy = fl(mu fl(dds vx + ddx vy)) at half rows
            const int sg = g0 + r;
            const EH2 a = EO2::mul(pload<16, 2>(P.mu_n, sg, 0, x),
                                   EO2::add(e_fold<ORDER>(c, s_ld(vx + (r - 1) * nx + x), s_ld(vx + r * nx + x),
                                                          s_ld(vx + (r + 1) * nx + x), s_ld(vx + (r + 2) * nx + x)),
                                            s_xfold<ORDER>(c, vy + r * nx, x, xl, xrr, false)));
            const EH2 old = s_ld(sxy + r * nx + x);
            EH2 sv = old, t = comp ? s_ld(rsxy + r * nx + x) : EH2{};
            finish<16, 16, 2>(a, nullptr, sg, 0, x, dt2.x, V, -1, 0.0, sv, t);
            s_st(sxy + r * nx + x, sv);
            track(4, sv);
            if (comp) {
                s_st(rsxy + r * nx + x, t);
                track(9, t);
            }
            if (sample) {  // kinetic y + shear energy at this half row
                const EH2 vyo = s_ld(vy + r * nx + x);
#pragma unroll
                for (int k = 0; k < 2; k++) {
                    const double v = (double)__half2float(vyo.e[k]);
                    e[1] += p64(P.e_rho_s, sg, 0, x + k) * (v * v);
                    const double mun = p64(P.e_mu_n, sg, 0, x + k);
                    const double a0 = (double)__half2float(old.e[k]), a1 = (double)__half2float(sv.e[k]);
                    e[4] += mun > 0.0 ? (a0 * a1) / mun : 0.0;
                }
            }
        }
        __syncthreads();
        publish_s();
        unsigned int mask = 0;  // external order vx vy sxx syy sxy, then residuals
#pragma unroll
        for (int q = 0; q < 10; q++) {
            const unsigned int bits = *reinterpret_cast<const unsigned int*>(&acc[q]);
            if (((bits & 0x7c00u) == 0x7c00u) || ((bits & 0x7c000000u) == 0x7c000000u)) mask |= 1u << q;
        }
        record_failure(P.ctrl, n, mask);
        double* part = (n / S.every) & 1 ? S.partials2 : P.partials;
        if (sample) block_partials(e, part);
        grid_barrier(S.gbar, nb);
        if (sample && b == 0) {
            const double tsum = finalize_partials(part, nb);
            if (tid == 0) S.e_vals[(n + 1) / S.every] = S.scale * tsum;
        }
        if (*reinterpret_cast<const volatile int64_t*>(&P.ctrl->fail_step) <= n) break;
    }
    for (int r = 0; r < Ri; r++) {  // write the band back (A buffers)
        s_st(gl(P.vx, r), s_ld(vx + r * nx + x));
        s_st(gl(P.sxx, r), s_ld(sxx + r * nx + x));
        s_st(gl(P.sss, r), s_ld(syy + r * nx + x));
        if (comp) {
            s_st(gl(P.rvx, r), s_ld(rvx + r * nx + x));
            s_st(gl(P.rsxx, r), s_ld(rsxx + r * nx + x));
            s_st(gl(P.rsss, r), s_ld(rsyy + r * nx + x));
        }
    }
    for (int r = 0; r < Rh; r++) {
        s_st(gl(P.vs, r), s_ld(vy + r * nx + x));
        s_st(gl(P.sxs, r), s_ld(sxy + r * nx + x));
        if (comp) {
            s_st(gl(P.rvs, r), s_ld(rvy + r * nx + x));
            s_st(gl(P.rsxs, r), s_ld(rsxy + r * nx + x));
        }
    }
}

// ---------------------------------------------------------------- host side

static int small_blocks(int64_t ns, int nsm) {
    int64_t nb = ns / 3;  // at least 3 rows per band (the published boundary rows)
    return (int)(nb < nsm ? nb : nsm);
}

static size_t small_smem(int64_t nx, int64_t ns, int nb) {
    const int64_t R = (ns + nb - 1) / nb;
    return (size_t)(6 * R + 12) * nx * sizeof(__half);
}

bool small2d_eligible(int64_t nx, int64_t ns, int nsm, int max_smem) {
    if (nx % 2 != 0 || nx < 16 || nx / 2 > 1024 || ns < 6) return false;
    const int nb = small_blocks(ns, nsm);
    if (nb < 2) return false;
    return small_smem(nx, ns, nb) <= (size_t)max_smem && small_smem(nx, ns, nb) <= 160 * 1024;
}

template <bool RM>
static void* small_fn(int variant, int order) {
    if (order == 2) {
        if (variant == 0) return (void*)k_ac2d_small<0, 2, RM>;
        if (variant == 3) return (void*)k_ac2d_small<3, 2, RM>;
        return (void*)k_ac2d_small<6, 2, RM>;
    }
    if (variant == 0) return (void*)k_ac2d_small<0, 4, RM>;
    if (variant == 3) return (void*)k_ac2d_small<3, 4, RM>;
    return (void*)k_ac2d_small<6, 4, RM>;
}

int small2d_blocks(int64_t ns, int nsm) { return small_blocks(ns, nsm); }

size_t small2d_xch_bytes(int64_t nx, int nb) { return (size_t)2 * nb * SX_ROWS * nx * sizeof(__half); }

cudaError_t small2d_prepare(int64_t nx, int64_t ns, int nb) {
    const int bytes = (int)small_smem(nx, ns, nb);
    for (int v : {0, 3, 6})
        for (int o : {2, 4})
            for (void* fn : {small_fn<false>(v, o), small_fn<true>(v, o)}) {
                cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
                if (e != cudaSuccess) return e;
            }
    return cudaSuccess;
}

bool fused2d_rowmed(const AcFusedParams& P);

cudaError_t launch_ac2d_small(int variant, int order, const AcFusedParams& F, __half* xch, unsigned int* gbar,
                              const double* src_dev, double* partials2, int every, int energy, int nb, int64_t nt,
                              cudaStream_t st) {
    SmallParams S;
    S.F = F;
    S.xch = xch;
    S.gbar = gbar;
    S.src = src_dev;
    S.partials2 = partials2;
    S.every = every;
    S.energy = energy;
    void* fn = fused2d_rowmed(F) ? small_fn<true>(variant, order) : small_fn<false>(variant, order);
    void* args[] = {(void*)&S, (void*)&nt};
    return cudaLaunchCooperativeKernel(fn, dim3(nb), dim3((unsigned)(F.nx / 2)), args, small_smem(F.nx, F.ns, nb), st);
}

// elastic: bands of >= 3 half rows; shared rows 10 R + 17 (R = max half rows + 1)
static size_t small_el_smem(int64_t nx, int64_t nh, int nb) {
    const int64_t R = (nh + nb - 1) / nb + 1;
    return (size_t)(10 * R + 17) * nx * sizeof(__half);
}

bool small_el2d_eligible(int64_t nx, int64_t nh, int nsm, int max_smem) {
    if (nx % 2 != 0 || nx < 16 || nx / 2 > 1024 || nh < 6) return false;
    const int nb = small_blocks(nh, nsm);
    if (nb < 2) return false;
    return small_el_smem(nx, nh, nb) <= (size_t)max_smem && small_el_smem(nx, nh, nb) <= 160 * 1024;
}

size_t small_el2d_xch_bytes(int64_t nx, int nb) { return (size_t)nb * SE_ROWS * nx * sizeof(__half); }

static void* small_el_fn(int variant, int order) {
    if (order == 2) {
        if (variant == 0) return (void*)k_el2d_small<0, 2>;
        if (variant == 3) return (void*)k_el2d_small<3, 2>;
        return (void*)k_el2d_small<6, 2>;
    }
    if (variant == 0) return (void*)k_el2d_small<0, 4>;
    if (variant == 3) return (void*)k_el2d_small<3, 4>;
    return (void*)k_el2d_small<6, 4>;
}

cudaError_t small_el2d_prepare(int64_t nx, int64_t nh, int nb) {
    const int bytes = (int)small_el_smem(nx, nh, nb);
    for (int v : {0, 3, 6})
        for (int o : {2, 4}) {
            cudaError_t e = cudaFuncSetAttribute(small_el_fn(v, o), cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
            if (e != cudaSuccess) return e;
        }
    return cudaSuccess;
}

cudaError_t launch_el2d_small(int variant, int order, const ElParams& P, const StreamIO& IO, __half* xch,
                              unsigned int* gbar, const double* src_dev, double* partials2, int every, int energy,
                              int nb, int64_t nt, cudaStream_t st) {
    SmallElParams S;
    memset(&S, 0, sizeof(S));
    S.P = P;
    S.traces = IO.traces;
    S.rec = IO.rec;
    S.n_rec = IO.n_rec;
    S.every = every;
    S.energy = energy;
    S.nt = IO.nt;
    S.e_vals = IO.e_vals;
    S.scale = IO.scale;
    S.xch = xch;
    S.gbar = gbar;
    S.src = src_dev;
    S.partials2 = partials2;
    void* args[] = {(void*)&S, (void*)&nt};
    return cudaLaunchCooperativeKernel(small_el_fn(variant, order), dim3(nb), dim3((unsigned)(P.g.nx / 2)), args,
                                       small_el_smem(P.g.nx, P.vs.rows, nb), st);
}

}  // namespace hw
