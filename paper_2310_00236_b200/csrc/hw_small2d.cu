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

}  // namespace hw
