// hw_fused2d.cu — single-pass fused leapfrog step for the 2D acoustic solver,
// binary16 state (the BASELINE config-2 hot path), sm_100a.
//
// One kernel per time step does both phases of AcousticSolver._step_work
// (acoustic.py:162-181): velocities from p^n, then p from div v^{n+1/2}, with
// the reference's exact operation order (same device helpers as the phase
// kernels, so the bits are identical).
//
// Work decomposition:
//   * CTA b owns output rows [y0, y1) and the FULL row width: periodic x wraps
//     inside the CTA, so no x halo is recomputed.  One CTA per SM.
//   * The CTA streams rows f = y0-3 .. y1+2 top to bottom.  Input rows arrive
//     in shared memory through 1D TMA bulk copies (cp.async.bulk + mbarrier
//     complete_tx), FR ring slots, prefetched FR-1 rows ahead by one thread.
//   * At front row f a thread (8 x cells, 4 half2) computes vx[f] (x taps from
//     the smem row), vy[f-2] (slow taps from its register queue of p rows
//     f-3..f), d/dx vx[f] (from a shared row, queued 3 rows) and finally p[f-3]
//     (div = queued d/dx vx + slow taps of its vy queue), so every input byte
//     is read from HBM once (plus a 6-row p / 3-row vy halo per CTA) and every
//     output byte written once: 24 B per cell-step.
//   * New state goes to the ping-pong buffer (no intra-step hazards between
//     CTAs); energy partials (diagnostics.py:76-87), receiver traces and the
//     non-finite flag are fused; the last CTA reduces the energy partials in a
//     fixed order (deterministic).
#include <cuda_runtime.h>

#include "hw_fused2d.h"
#include "hw_params.h"
#include "hw_tma.cuh"

namespace hw {

constexpr int FCPT = 8;  // cells per thread
constexpr int FR = 4;    // TMA ring slots (prefetch distance FR-1)
constexpr int NSTREAM = FUSED_NSTREAM;
enum { S_P = 0, S_VX = 1, S_VS = 2, S_RP = 3, S_RVX = 4, S_RVS = 5 };

using H2 = vec<16, 2>;
using O2 = vops<16, 2>;

struct V8 {
    H2 q[4];
};

__device__ __forceinline__ V8 lds8(const __half* p) {
    V8 r;
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    *reinterpret_cast<unsigned int*>(&r.q[0].h2) = u.x;
    *reinterpret_cast<unsigned int*>(&r.q[1].h2) = u.y;
    *reinterpret_cast<unsigned int*>(&r.q[2].h2) = u.z;
    *reinterpret_cast<unsigned int*>(&r.q[3].h2) = u.w;
    return r;
}

__device__ __forceinline__ void st8(__half* p, const V8& v) {
    uint4 u;
    u.x = *reinterpret_cast<const unsigned int*>(&v.q[0].h2);
    u.y = *reinterpret_cast<const unsigned int*>(&v.q[1].h2);
    u.z = *reinterpret_cast<const unsigned int*>(&v.q[2].h2);
    u.w = *reinterpret_cast<const unsigned int*>(&v.q[3].h2);
    *reinterpret_cast<uint4*>(p) = u;
}

__device__ __forceinline__ H2 ld2(const __half* p) {
    H2 r;
    r.h2 = *reinterpret_cast<const __half2*>(p);
    return r;
}

template <int ORDER>
__device__ __forceinline__ H2 fold2(const __half c[4], H2 t0, H2 t1, H2 t2, H2 t3) {
    H2 inner = O2::add(O2::mul(vsplat<16, 2>(c[1]), t1), O2::mul(vsplat<16, 2>(c[2]), t2));
    if (ORDER == 2) return inner;
    H2 outer = O2::add(O2::mul(vsplat<16, 2>(c[0]), t0), O2::mul(vsplat<16, 2>(c[3]), t3));
    return O2::add(inner, outer);
}

// x derivative of 8 cells from the pair sequence Q[-1..4] (Q[0..3] = own cells).
// to_int: shifts (-2,-1,0,1); else (-1,0,1,2)  (stencil.py:39-40).
template <int ORDER>
__device__ __forceinline__ V8 xfold8(const __half c[4], H2 left, const V8& own, H2 right, bool to_int) {
    H2 Q[6];
    Q[0] = left;
#pragma unroll
    for (int j = 0; j < 4; j++) Q[j + 1] = own.q[j];
    Q[5] = right;
    H2 S[5];  // S[j] = cells (x+2j-1, x+2j)
#pragma unroll
    for (int j = 0; j < 5; j++) S[j] = vshift<16, 2>(Q[j], Q[j + 1]);
    V8 r;
#pragma unroll
    for (int j = 0; j < 4; j++)
        r.q[j] = to_int ? fold2<ORDER>(c, Q[j], S[j], Q[j + 1], S[j + 1]) : fold2<ORDER>(c, S[j], Q[j + 1], S[j + 1], Q[j + 2]);
    return r;
}

__device__ __forceinline__ H2 plane2(const PlaneView& pv, int64_t s, int64_t x) {
    return pload<16, 2>(pv, s, 0, x);
}

// running max(|x|) with NaN propagation: the field went non-finite iff the
// accumulator ends at inf/NaN (one VHMNMX.NAN per two half2 values)
__device__ __forceinline__ void track(__half2& acc, const V8& v) {
#pragma unroll
    for (int j = 0; j < 4; j++) acc = __hmax2_nan(acc, __habs2(v.q[j].h2));
}

__device__ __forceinline__ unsigned int nonfinite_acc(__half2 acc) {
    const unsigned int b = *reinterpret_cast<const unsigned int*>(&acc);
    return (((b & 0x7c00u) == 0x7c00u) || ((b & 0x7c000000u) == 0x7c000000u)) ? 1u : 0u;
}

// increment (stepping.py:58-80) + advance (efsum.py:100-121) for one half2 pair,
// division by a row-uniform divisor through its verified reciprocal (DIV_CHEAP)
template <int V>
__device__ __forceinline__ void finish_row(H2 rhs, float rcp, __half2 dt2, int src_lane, __half srch, H2& u, H2& t) {
    if (src_lane == 0) rhs.e[0] = __hadd_rn(rhs.e[0], srch);
    else if (src_lane == 1) rhs.e[1] = __hadd_rn(rhs.e[1], srch);
    const float2 fx = __half22float2(rhs.h2);
    H2 x;
    x.h2 = __hmul2_rn(__floats2half2_rn(__fmul_rn(fx.x, rcp), __fmul_rn(fx.y, rcp)), dt2);
    if (V == 0) {
        u.h2 = __hadd2_rn(u.h2, x.h2);
        return;
    }
    const __half2 r = __hadd2_rn(t.h2, x.h2);
    const __half2 s = __hadd2_rn(u.h2, r);
    if (V == 3) {
        t.h2 = __hsub2_rn(r, __hsub2_rn(s, u.h2));
    } else {
        const __half2 pa = __hsub2_rn(s, r);
        const __half2 pb = __hsub2_rn(s, pa);
        t.h2 = __hadd2_rn(__hsub2_rn(u.h2, pa), __hsub2_rn(r, pb));
    }
    u.h2 = s;
}

template <int V, int ORDER, bool ROWMED>
__global__ void __launch_bounds__(512, 1)
    k_ac2d_fused(AcFusedParams P, int64_t n, double src, int sample, int64_t eidx) {
    // Programmatic dependent launch: the next step's grid may launch as soon as this
    // one is running (its CTAs take SMs as ours retire); it waits here until every
    // write of the previous step is visible.
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (halted(P.ctrl, n)) return;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
    __half* ring = reinterpret_cast<__half*>(smem + 256);
    const int64_t nx = P.nx, ns = P.ns, pitch = P.pitch;
    __half* xrows = ring + (int64_t)FR * NSTREAM * nx;  // two rows, alternating by iteration parity
    const int b = blockIdx.x;
    int y0, y1, pidx, nb;  // this CTA's rows, its energy-partial slot, CTAs of the whole step
    if (P.band_mode == 1) {  // edge bands: launched ahead of the interior so the halo exchange overlaps it
        y0 = b == 0 ? 0 : (int)ns - P.edge;
        y1 = b == 0 ? P.edge : (int)ns;
        pidx = b;
        nb = P.nb_total;
    } else if (P.band_mode == 2) {
        const int64_t ni = ns - 2 * P.edge;
        y0 = P.edge + (int)((int64_t)b * ni / gridDim.x);
        y1 = P.edge + (int)((int64_t)(b + 1) * ni / gridDim.x);
        pidx = 2 + b;
        nb = P.nb_total;
    } else {
        nb = gridDim.x;
        y0 = (int)((int64_t)b * ns / nb);
        y1 = (int)((int64_t)(b + 1) * ns / nb);
        pidx = b;
    }
    const int F0 = y0 - 3;
    const int NI = (y1 + 3) - F0;
    const int tid = threadIdx.x;
    const int x = tid * FCPT;
    constexpr bool comp = V != 0;
    const uint32_t rb = (uint32_t)(nx * sizeof(__half));

    auto slot_row = [&](int slot, int st) { return ring + (slot * NSTREAM + st) * nx; };
    // rows outside [0, ns): periodic wrap in a single domain, ghost rows (filled by the
    // halo exchange, G >= 3 deep) in a slab
    auto wrap_row = [&](int64_t r) {
        if (P.slab) return r;
        r %= ns;
        return r < 0 ? r + ns : r;
    };
    auto issue = [&](int64_t i, int slot) {  // TMA loads of iteration i (front row F0 + i)
        const int64_t f = F0 + i;
        const bool lvx = f >= y0 && f < y1;
        const bool lvs = f >= y0 && f < y1 + 3;
        const bool lrp = comp && f >= y0 + 3 && f < y1 + 3;
        const uint32_t rows = 1 + (lvx ? (comp ? 2 : 1) : 0) + (lvs ? (comp ? 2 : 1) : 0) + (lrp ? 1 : 0);
        mbar_arrive_expect_tx(&bar[slot], rows * rb);
        tma_load_1d(slot_row(slot, S_P), P.in[S_P] + wrap_row(f) * pitch, rb, &bar[slot]);
        if (lvx) {
            tma_load_1d(slot_row(slot, S_VX), P.in[S_VX] + f * pitch, rb, &bar[slot]);
            if (comp) tma_load_1d(slot_row(slot, S_RVX), P.in[S_RVX] + f * pitch, rb, &bar[slot]);
        }
        if (lvs) {
            const int64_t r = wrap_row(f - 2);
            tma_load_1d(slot_row(slot, S_VS), P.in[S_VS] + r * pitch, rb, &bar[slot]);
            if (comp) tma_load_1d(slot_row(slot, S_RVS), P.in[S_RVS] + r * pitch, rb, &bar[slot]);
        }
        if (lrp) tma_load_1d(slot_row(slot, S_RP), P.in[S_RP] + (f - 3) * pitch, rb, &bar[slot]);
    };

    if (tid == 0) {
        for (int s = 0; s < FR; s++) mbar_init(&bar[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0)
        for (int64_t i = 0; i < FR - 1 && i < NI; i++) issue(i, (int)i);
    int rcur = rec_lower(P.rec, 0, P.n_rec, y0, INT_MIN);  // this CTA's receivers [rcur, rhi)
    const int rhi = rec_lower(P.rec, rcur, P.n_rec, y1, INT_MIN);

    __half c[4];
#pragma unroll
    for (int j = 0; j < 4; j++) c[j] = lconst<16>(P.k, j);
    const __half2 dt2 = __half2half2(lconst<16>(P.k, 4));
    const __half srch = __double2half(src);
    const int xl = x == 0 ? (int)nx - 2 : x - 2;                // left neighbour pair
    const int xr = x + FCPT >= (int)nx ? 0 : x + FCPT;          // right neighbour pair
    const bool src_here = P.has_src && src != 0.0 && P.src_x >= x && P.src_x < x + FCPT;
    const int src_j = (int)((P.src_x - x) >> 1), src_lane = (int)((P.src_x - x) & 1);

    V8 pq[4], vq[4], gq[4];  // p rows, vy_new rows, d/dx vx_new rows ([3] = newest)
    __half2 acc[NSTREAM];
#pragma unroll
    for (int q = 0; q < NSTREAM; q++) acc[q] = __float2half2_rn(0.f);
    double e[NCOMP] = {0.0, 0.0, 0.0, 0.0, 0.0};
    // energy planes constant along x (layered media): sum the products per row, apply the
    // fp64 coefficient once per row (same terms regrouped; agrees to ~1e-16 relative)
    const bool erow = (P.e_beta.sx | P.e_rho_x.sx | P.e_rho_s.sx) == 0;

    // Rolled row loop (one copy of the body: the unrolled form was instruction-cache
    // bound); the register queues rotate, [3] = this iteration's row.  fw is the
    // wrapped front row, advanced without integer division; the row-uniform divisor
    // reciprocals of the next iteration are prefetched into registers.
    const int ns32 = (int)ns;
    const bool slab = P.slab != 0;
    auto back = [&](int r, int k) { r -= k; return (!slab && r < 0) ? r + ns32 : r; };  // wrapped r - k (k < ns)
    int fw = (int)wrap_row(F0);
    float rcx = 0.f, rcs = 0.f, rcb = 0.f;
    if constexpr (ROWMED) {
        rcx = __ldg(P.rho_x.rcp + fw * P.rho_x.ss);
        rcs = __ldg(P.rho_s.rcp + back(fw, 2) * P.rho_s.ss);
        rcb = __ldg(P.beta.rcp + back(fw, 3) * P.beta.ss);
    }
    // energy coefficients of the rows of the next iteration (sample steps, row-uniform planes)
    const bool epre = sample && erow;
    double ex = 0.0, es = 0.0, eb = 0.0;
    if (epre) {
        ex = p64(P.e_rho_x, fw, 0, 0);
        es = p64(P.e_rho_s, back(fw, 2), 0, 0);
        eb = p64(P.e_beta, back(fw, 3), 0, 0);
    }
#pragma unroll 1
    for (int i = 0; i < NI; i++) {
        const int u = i % FR;
        const uint32_t par = (uint32_t)((i / FR) & 1);
        const int fwn = (!slab && fw + 1 == ns32) ? 0 : fw + 1;
        float rcx_n = 0.f, rcs_n = 0.f, rcb_n = 0.f;
        if constexpr (ROWMED) {
            rcx_n = __ldg(P.rho_x.rcp + fwn * P.rho_x.ss);
            rcs_n = __ldg(P.rho_s.rcp + back(fwn, 2) * P.rho_s.ss);
            rcb_n = __ldg(P.beta.rcp + back(fwn, 3) * P.beta.ss);
        }
        double ex_n = 0.0, es_n = 0.0, eb_n = 0.0;
        if (epre) {
            ex_n = p64(P.e_rho_x, fwn, 0, 0);
            es_n = p64(P.e_rho_s, back(fwn, 2), 0, 0);
            eb_n = p64(P.e_beta, back(fwn, 3), 0, 0);
        }
        {
            {
                const int f = F0 + i;
                __half* xrow = xrows + (i & 1) * nx;
#pragma unroll
                for (int q = 0; q < 3; q++) {
                    pq[q] = pq[q + 1];
                    vq[q] = vq[q + 1];
                    gq[q] = gq[q + 1];
                }
                if (tid == 0 && i + FR - 1 < NI) {
                    fence_proxy_async_smem();
                    issue(i + FR - 1, (i + FR - 1) % FR);
                }
                mbar_wait(&bar[u], par);
                const __half* prow = slot_row(u, S_P);
                pq[3] = lds8(prow + x);
                const bool do_vx = f >= y0 && f < y1;
                if (do_vx) {  // vx[f] (acoustic.py:167-168)
                    V8 d = xfold8<ORDER>(c, ld2(prow + xl), pq[3], ld2(prow + xr), false);
                    V8 vxn = lds8(slot_row(u, S_VX) + x);
                    V8 r = comp ? lds8(slot_row(u, S_RVX) + x) : V8{};
                    if constexpr (ROWMED) {
                        const float rc = rcx;
#pragma unroll
                        for (int j = 0; j < 4; j++) finish_row<V>(d.q[j], rc, dt2, -1, srch, vxn.q[j], r.q[j]);
                    } else {
#pragma unroll
                        for (int j = 0; j < 4; j++)
                            finish<16, 16, 2>(d.q[j], &P.rho_x, f, 0, x + 2 * j, dt2.x, V, -1, 0.0, vxn.q[j], r.q[j]);
                    }
                    st8(P.out[S_VX] + f * pitch + x, vxn);
                    track(acc[S_VX], vxn);
                    if (comp) {
                        st8(P.out[S_RVX] + f * pitch + x, r);
                        track(acc[S_RVX], r);
                    }
                    st8(xrow + x, vxn);
                    if (sample) {  // per-row sum when the plane is row-uniform (one multiply per row);
                        // a product of two binary16 values is exact in binary32 (<= 22 bits)
                        double sv = 0.0;
#pragma unroll
                        for (int j = 0; j < 4; j++) {
                            const float2 v = __half22float2(vxn.q[j].h2);
                            const double a = (double)__fmul_rn(v.x, v.x), b = (double)__fmul_rn(v.y, v.y);
                            if (erow) {
                                sv += a;
                                sv += b;
                            } else {
                                e[1] += p64(P.e_rho_x, f, 0, x + 2 * j) * a;
                                e[1] += p64(P.e_rho_x, f, 0, x + 2 * j + 1) * b;
                            }
                        }
                        if (erow) e[1] += ex * sv;
                    }
                }
                const int k = f - 3;
                const bool do_p = k >= y0 && k < y1;
                V8 rp = (comp && do_p) ? lds8(slot_row(u, S_RP) + x) : V8{};  // all ring reads before the barrier
                if (f >= y0 && f < y1 + 3) {  // vy[f-2] from p rows f-3..f (acoustic.py:169-170)
                    const int r = f - 2;
                    const int rw = back(fw, 2);
                    V8 vsn = lds8(slot_row(u, S_VS) + x);
                    V8 rr = comp ? lds8(slot_row(u, S_RVS) + x) : V8{};
                    const V8& t0 = pq[0];
                    const V8& t1 = pq[1];
                    const V8& t2 = pq[2];
                    if constexpr (ROWMED) {
                        const float rc = rcs;
#pragma unroll
                        for (int j = 0; j < 4; j++)
                            finish_row<V>(fold2<ORDER>(c, t0.q[j], t1.q[j], t2.q[j], pq[3].q[j]), rc, dt2, -1, srch,
                                          vsn.q[j], rr.q[j]);
                    } else {
#pragma unroll
                        for (int j = 0; j < 4; j++)
                            finish<16, 16, 2>(fold2<ORDER>(c, t0.q[j], t1.q[j], t2.q[j], pq[3].q[j]), &P.rho_s, rw, 0,
                                              x + 2 * j, dt2.x, V, -1, 0.0, vsn.q[j], rr.q[j]);
                    }
                    if (r >= y0 && r < y1) {
                        st8(P.out[S_VS] + r * pitch + x, vsn);
                        track(acc[S_VS], vsn);
                        if (comp) {
                            st8(P.out[S_RVS] + r * pitch + x, rr);
                            track(acc[S_RVS], rr);
                        }
                        if (sample) {
                            double sv = 0.0;
#pragma unroll
                            for (int j = 0; j < 4; j++) {
                                const float2 v = __half22float2(vsn.q[j].h2);
                                const double a = (double)__fmul_rn(v.x, v.x), b = (double)__fmul_rn(v.y, v.y);
                                if (erow) {
                                    sv += a;
                                    sv += b;
                                } else {
                                    e[2] += p64(P.e_rho_s, r, 0, x + 2 * j) * a;
                                    e[2] += p64(P.e_rho_s, r, 0, x + 2 * j + 1) * b;
                                }
                            }
                            if (erow) e[2] += es * sv;
                        }
                    }
                    vq[3] = vsn;
                }
                // One barrier per row: xrow[f&1] now holds vx_new[f] and every thread is past
                // its ring-slot reads, so the producer may refill this slot next iteration;
                // xrow[f&1] is rewritten two iterations later, after another barrier.
                __syncthreads();
                if (do_vx) gq[3] = xfold8<ORDER>(c, ld2(xrow + xl), lds8(xrow + x), ld2(xrow + xr), true);
                if (do_p) {  // p[k] (acoustic.py:172-181)
                    const V8& pold = pq[0];
                    V8 pn = pold;
                    const V8& g = gq[0];
                    const V8& a0 = vq[0];
                    const V8& a1 = vq[1];
                    const V8& a2 = vq[2];
                    const bool sk = src_here && k == P.src_s;
                    if constexpr (ROWMED) {
                        const float rc = rcb;
#pragma unroll
                        for (int j = 0; j < 4; j++) {
                            H2 dv = O2::add(g.q[j], fold2<ORDER>(c, a0.q[j], a1.q[j], a2.q[j], vq[3].q[j]));
                            finish_row<V>(dv, rc, dt2, (sk && j == src_j) ? src_lane : -1, srch, pn.q[j], rp.q[j]);
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < 4; j++) {
                            H2 dv = O2::add(g.q[j], fold2<ORDER>(c, a0.q[j], a1.q[j], a2.q[j], vq[3].q[j]));
                            finish<16, 16, 2>(dv, &P.beta, k, 0, x + 2 * j, dt2.x, V, (sk && j == src_j) ? src_lane : -1,
                                              src, pn.q[j], rp.q[j]);
                        }
                    }
                    st8(P.out[S_P] + k * pitch + x, pn);
                    track(acc[S_P], pn);
                    if (comp) {
                        st8(P.out[S_RP] + k * pitch + x, rp);
                        track(acc[S_RP], rp);
                    }
                    if (sample) {
                        double sp = 0.0;
#pragma unroll
                        for (int j = 0; j < 4; j++) {
                            const float2 a = __half22float2(pold.q[j].h2), bb = __half22float2(pn.q[j].h2);
                            const double u0 = (double)__fmul_rn(a.x, bb.x), u1 = (double)__fmul_rn(a.y, bb.y);
                            if (erow) {
                                sp += u0;
                                sp += u1;
                            } else {
                                e[0] += p64(P.e_beta, k, 0, x + 2 * j) * u0;
                                e[0] += p64(P.e_beta, k, 0, x + 2 * j + 1) * u1;
                            }
                        }
                        if (erow) e[0] += eb * sp;
                    }
                    // receiver traces (acoustic.py:217-218)
                    rec_row(P.rec, rcur, rhi, k, x, P.traces, P.nt, n, [&](int o) {
                        double v = 0.0;
#pragma unroll
                        for (int j = 0; j < FCPT; j++)
                            if (j == o) v = (double)__half2float(pn.q[j >> 1].e[j & 1]);
                        return v;
                    });
                }
            }
        }
        fw = fwn;
        ex = ex_n;
        es = es_n;
        eb = eb_n;
        rcx = rcx_n;
        rcs = rcs_n;
        rcb = rcb_n;
    }
    unsigned int mask = 0;
    // bit order = external field order p vx vy rp rvx rvy == stream order
#pragma unroll
    for (int q = 0; q < NSTREAM; q++) mask |= nonfinite_acc(acc[q]) << q;
    record_failure(P.ctrl, n, mask);
    if (!sample) return;
    block_partials(e, P.partials, pidx);
    __threadfence();
    __syncthreads();
    __shared__ unsigned int is_last;
    if (tid == 0) is_last = atomicAdd(P.counter, 1u) == (unsigned int)(nb - 1);
    __syncthreads();
    if (!is_last) return;
    const double t = finalize_partials(P.partials, nb);
    if (tid == 0) {
        P.e_vals[eidx] = P.scale * t;
        *P.counter = 0u;
    }
}

size_t fused2d_smem_bytes(int64_t nx) { return 256 + ((size_t)FR * NSTREAM + 2) * nx * sizeof(__half); }

int fused2d_threads(int64_t nx) { return (int)(nx / FCPT); }

bool fused2d_eligible(int64_t nx, int max_smem) {
    // 8 cells per thread, 16-byte TMA rows: nx % 8 == 0 (nx / 8 threads; the last warp may
    // be partial -- the collectives use the existing lanes only)
    if (nx % 8 != 0 || nx < 64 || nx / FCPT > 512) return false;
    return fused2d_smem_bytes(nx) <= (size_t)max_smem;
}

template <bool RM>
static void* fused_fn(int variant, int order) {
    if (order == 2) {
        if (variant == 0) return (void*)k_ac2d_fused<0, 2, RM>;
        if (variant == 3) return (void*)k_ac2d_fused<3, 2, RM>;
        return (void*)k_ac2d_fused<6, 2, RM>;
    }
    if (variant == 0) return (void*)k_ac2d_fused<0, 4, RM>;
    if (variant == 3) return (void*)k_ac2d_fused<3, 4, RM>;
    return (void*)k_ac2d_fused<6, 4, RM>;
}

cudaError_t fused2d_prepare(int64_t nx) {
    const int bytes = (int)fused2d_smem_bytes(nx);
    for (int v : {0, 3, 6})
        for (int o : {2, 4})
            for (void* fn : {fused_fn<false>(v, o), fused_fn<true>(v, o)}) {
                cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
                if (e != cudaSuccess) return e;
            }
    return cudaSuccess;
}

bool fused2d_rowmed(const AcFusedParams& P) {
    auto ok = [](const PlaneView& v) { return v.div_mode == DIV_CHEAP && v.sx == 0 && v.sm == 0; };
    return ok(P.rho_x) && ok(P.rho_s) && ok(P.beta);
}

void launch_ac2d_fused(int variant, int order, const AcFusedParams& P, int nblocks, int64_t n, double src, int sample,
                       int64_t eidx, cudaStream_t st) {
    const int threads = fused2d_threads(P.nx);
    const size_t bytes = fused2d_smem_bytes(P.nx);
    void* fn = fused2d_rowmed(P) ? fused_fn<true>(variant, order) : fused_fn<false>(variant, order);
    void* args[] = {(void*)&P, (void*)&n, (void*)&src, (void*)&sample, (void*)&eidx};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nblocks);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = bytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelExC(&cfg, fn, args);
}

}  // namespace hw
