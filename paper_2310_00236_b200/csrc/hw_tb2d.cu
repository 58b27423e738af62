// hw_tb2d.cu — two leapfrog steps per launch (temporal blocking) for the 2D acoustic
// solver, binary16 state (BASELINE config 2), sm_100a.
//
// Step n ("stage A") runs the single-pass row pipeline of hw_fused2d.cu on the input
// buffer; step n+1 ("stage B") consumes stage A's rows straight from registers and
// shared memory, a few rows behind, so the intermediate state never touches HBM:
// 24 B per cell per TWO steps plus the halos.  Arithmetic is the reference's, op for
// op (same helpers as the single-step kernel), so the bits are identical.
//
// Decomposition: x tiles of XT = min(nx, 1024) output cells with an 8-cell halo on
// each side (two steps reach 6 cells in x), 4 cells per thread; row bands per CTA.
// For output rows [y0, y1) stage A produces vx rows [y0-3, y1+3), vy rows
// [y0-5, y1+4), p rows [y0-3, y1+3) (its halo rows are recomputed by the neighbour
// bands).  Front row f = y0-6 .. y1+6, per iteration:
//   phase 1: stage A vx[f] (x taps of the p row), vy[f-2] (queued p rows f-3..f)
//   barrier
//   phase 2: stage A d/dx vx[f] and p[f-3];
//            stage B d/dx vx[f-5], vx[f-4] (x taps of stage-A p row f-4, in smem since
//            the previous iteration), vy[f-6] (queued stage-A p rows), p[f-7].
// Stage B writes its rows [y0, y1) x [x0, x0+XT) to the output buffer.  A failure in
// stage A is reported for step n; the host then replays step n alone (hw_api.cu).
#include <cuda_runtime.h>

#include "hw_fused2d.h"
#include "hw_params.h"
#include "hw_tma.cuh"

namespace hw {

constexpr int TCPT = 4;      // cells per thread
constexpr int TR = 4;        // TMA ring slots
constexpr int THALO = 8;     // x halo cells per side
constexpr int TXT_MAX = 1024;
enum { T_P = 0, T_VX = 1, T_VS = 2, T_RP = 3, T_RVX = 4, T_RVS = 5, T_NS = 6 };

using H2 = vec<16, 2>;
using O2 = vops<16, 2>;

struct V4 {
    H2 q[2];
};

__device__ __forceinline__ V4 ld4(const __half* p) {
    V4 r;
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    *reinterpret_cast<unsigned int*>(&r.q[0].h2) = u.x;
    *reinterpret_cast<unsigned int*>(&r.q[1].h2) = u.y;
    return r;
}

__device__ __forceinline__ void st4(__half* p, const V4& v) {
    uint2 u;
    u.x = *reinterpret_cast<const unsigned int*>(&v.q[0].h2);
    u.y = *reinterpret_cast<const unsigned int*>(&v.q[1].h2);
    *reinterpret_cast<uint2*>(p) = u;
}

__device__ __forceinline__ H2 tld2(const __half* p) {
    H2 r;
    r.h2 = *reinterpret_cast<const __half2*>(p);
    return r;
}

template <int ORDER>
__device__ __forceinline__ H2 tfold(const __half c[4], H2 t0, H2 t1, H2 t2, H2 t3) {
    H2 inner = O2::add(O2::mul(vsplat<16, 2>(c[1]), t1), O2::mul(vsplat<16, 2>(c[2]), t2));
    if (ORDER == 2) return inner;
    H2 outer = O2::add(O2::mul(vsplat<16, 2>(c[0]), t0), O2::mul(vsplat<16, 2>(c[3]), t3));
    return O2::add(inner, outer);
}

// x derivative of 4 cells from a shared row (window coordinates; edge threads read
// clamped neighbours: their results lie in the halo and are never used)
template <int ORDER>
__device__ __forceinline__ V4 txfold(const __half c[4], const __half* row, int w, int wl, int wr, bool to_int) {
    H2 Q[4];
    Q[0] = tld2(row + wl);
    const V4 own = ld4(row + w);
    Q[1] = own.q[0];
    Q[2] = own.q[1];
    Q[3] = tld2(row + wr);
    H2 S[3];
#pragma unroll
    for (int j = 0; j < 3; j++) S[j] = vshift<16, 2>(Q[j], Q[j + 1]);
    V4 r;
#pragma unroll
    for (int j = 0; j < 2; j++)
        r.q[j] = to_int ? tfold<ORDER>(c, Q[j], S[j], Q[j + 1], S[j + 1]) : tfold<ORDER>(c, S[j], Q[j + 1], S[j + 1], Q[j + 2]);
    return r;
}

template <int ORDER>
__device__ __forceinline__ V4 tsfold(const __half c[4], const V4& a, const V4& b, const V4& d, const V4& e) {
    V4 r;
#pragma unroll
    for (int j = 0; j < 2; j++) r.q[j] = tfold<ORDER>(c, a.q[j], b.q[j], d.q[j], e.q[j]);
    return r;
}

__device__ __forceinline__ void ttrack(__half2& acc, const V4& v) {
    acc = __hmax2_nan(acc, __habs2(v.q[0].h2));
    acc = __hmax2_nan(acc, __habs2(v.q[1].h2));
}

__device__ __forceinline__ unsigned int tnonfinite(__half2 acc) {
    const unsigned int b = *reinterpret_cast<const unsigned int*>(&acc);
    return (((b & 0x7c00u) == 0x7c00u) || ((b & 0x7c000000u) == 0x7c000000u)) ? 1u : 0u;
}

// increment + advance for one pair with a row-uniform verified reciprocal (DIV_CHEAP)
template <int V>
__device__ __forceinline__ void tfinish_row(H2 rhs, float rcp, __half2 dt2, int src_lane, __half srch, H2& u, H2& t) {
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

// one field update of 4 cells: row-uniform (ROWMED) or per-cell medium (plane x = gx)
template <int V, bool ROWMED>
__device__ __forceinline__ void tupdate(const V4& rhs, const PlaneView& pv, int row, int gx, __half2 dt2,
                                        int src_j, int src_lane, __half srch, double src, V4& u, V4& t) {
    if constexpr (ROWMED) {
        const float rc = __ldg(pv.rcp + (int64_t)row * pv.ss);
#pragma unroll
        for (int j = 0; j < 2; j++) tfinish_row<V>(rhs.q[j], rc, dt2, j == src_j ? src_lane : -1, srch, u.q[j], t.q[j]);
    } else {
#pragma unroll
        for (int j = 0; j < 2; j++)
            finish<16, 16, 2>(rhs.q[j], &pv, row, 0, gx + 2 * j, dt2.x, V, j == src_j ? src_lane : -1, src, u.q[j], t.q[j]);
    }
}

template <int D>
struct TQ {  // register queue of V4 rows, q[D-1] newest
    V4 q[D];
    __device__ __forceinline__ void push(const V4& v) {
#pragma unroll
        for (int k = 0; k < D - 1; k++) q[k] = q[k + 1];
        q[D - 1] = v;
    }
};

__device__ __forceinline__ double tpick(const V4& v, int o) {
    double r = 0.0;
#pragma unroll
    for (int j = 0; j < TCPT; j++)
        if (j == o) r = (double)__half2float(v.q[j >> 1].e[j & 1]);
    return r;
}

struct AcTb2Params {
    AcFusedParams F;  // fields, medium, receivers, control (in / out buffers)
    int64_t xt;       // output cells per x tile
    int32_t ntiles, nbands;
    double* partials_b;  // stage-B energy partials
};

template <int V, int ORDER, bool ROWMED>
__global__ void __launch_bounds__(288, 1)
    k_ac2d_tb2(AcTb2Params T, int64_t n, double srcA, double srcB, int sampleA, int sampleB, int64_t eidxA,
               int64_t eidxB) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const AcFusedParams& P = T.F;
    if (halted(P.ctrl, n)) return;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
    const int nx = (int)P.nx, ns = (int)P.ns;
    const int64_t pitch = P.pitch;
    const int XT = (int)T.xt, WW = XT + 2 * THALO;  // window width (cells)
    __half* ring = reinterpret_cast<__half*>(smem + 128);
    __half* xrA = ring + (int64_t)TR * T_NS * WW;  // stage A vx rows (2, by parity)
    __half* xrP = xrA + 2 * WW;                    // stage A p rows (2)
    __half* xrB = xrP + 2 * WW;                    // stage B vx rows (2)
    const int tile = blockIdx.x % T.ntiles, band = blockIdx.x / T.ntiles;
    const int x0 = tile * XT;
    const int y0 = (int)((int64_t)band * ns / T.nbands), y1 = (int)((int64_t)(band + 1) * ns / T.nbands);
    const int F0 = y0 - 6, NI = (y1 + 7) - F0;  // fronts y0-6 .. y1+6
    const int tid = threadIdx.x;
    const int w = tid * TCPT;  // window position of the thread's first cell
    const bool active = w < WW;
    int gx = x0 - THALO + w;  // global x of the first cell (periodic)
    gx = gx < 0 ? gx + nx : (gx >= nx ? gx - nx : gx);
    const bool own_x = w >= THALO && w < THALO + XT;
    constexpr bool comp = V != 0;
    const uint32_t rowb = (uint32_t)(WW * sizeof(__half));

    auto wrap_row = [&](int r) { r %= ns; return r < 0 ? r + ns : r; };
    auto slot_row = [&](int slot, int st) { return ring + (slot * T_NS + st) * (int64_t)WW; };
    // one window row [x0-8, x0+XT+8) of field `base` at row r, periodic in x and rows
    auto load_row = [&](__half* dst, const __half* base, int r, uint64_t* b) {
        const __half* src = base + (int64_t)wrap_row(r) * pitch;
        int a = x0 - THALO, done = 0;
        while (done < WW) {
            const int ga = a < 0 ? a + nx : (a >= nx ? a - nx : a);
            const int seg = min(WW - done, nx - ga);
            tma_load_1d(dst + done, src + ga, (uint32_t)(seg * sizeof(__half)), b);
            done += seg;
            a += seg;
        }
    };
    // rows each stage-A quantity is needed on (CTA-uniform predicates of the front row f)
    auto need_vx = [&](int f) { return f >= y0 - 3 && f < y1 + 3; };  // vx_A rows [y0-3, y1+3)
    auto need_vy = [&](int f) { return f >= y0 - 3 && f < y1 + 6; };  // vy_A rows f-2 in [y0-5, y1+4)
    auto need_rp = [&](int f) { return comp && f >= y0 && f < y1 + 6; };  // p_A rows f-3 in [y0-3, y1+3)
    auto issue = [&](int i) {
        const int f = F0 + i, slot = i % TR;
        const uint32_t rows = 1 + (need_vx(f) ? (comp ? 2 : 1) : 0) + (need_vy(f) ? (comp ? 2 : 1) : 0) +
                              (need_rp(f) ? 1 : 0);
        mbar_arrive_expect_tx(&bar[slot], rows * rowb);
        load_row(slot_row(slot, T_P), P.in[T_P], f, &bar[slot]);
        if (need_vx(f)) {
            load_row(slot_row(slot, T_VX), P.in[T_VX], f, &bar[slot]);
            if (comp) load_row(slot_row(slot, T_RVX), P.in[T_RVX], f, &bar[slot]);
        }
        if (need_vy(f)) {
            load_row(slot_row(slot, T_VS), P.in[T_VS], f - 2, &bar[slot]);
            if (comp) load_row(slot_row(slot, T_RVS), P.in[T_RVS], f - 2, &bar[slot]);
        }
        if (need_rp(f)) load_row(slot_row(slot, T_RP), P.in[T_RP], f - 3, &bar[slot]);
    };

    if (tid == 0) {
        for (int s = 0; s < TR; s++) mbar_init(&bar[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0)
        for (int i = 0; i < TR - 1 && i < NI; i++) issue(i);

    __half c[4];
#pragma unroll
    for (int j = 0; j < 4; j++) c[j] = lconst<16>(P.k, j);
    const __half2 dt2 = __half2half2(lconst<16>(P.k, 4));
    const __half srchA = __double2half(srcA), srchB = __double2half(srcB);
    const int wl = w >= 2 ? w - 2 : 0;                      // left neighbour pair (clamped at the window edge)
    const int wr = w + TCPT <= WW - 2 ? w + TCPT : WW - 2;  // right neighbour pair
    const bool src_col = P.has_src && P.src_x >= gx && P.src_x < gx + TCPT;
    const int src_lane = (int)((P.src_x - gx) & 1);
    const int sjA = (src_col && srcA != 0.0) ? (int)((P.src_x - gx) >> 1) : -1;
    const int sjB = (src_col && srcB != 0.0) ? (int)((P.src_x - gx) >> 1) : -1;

    // Register queues, pushed EVERY iteration so that q[k] always maps to a fixed row
    // offset from the front (rows outside a stage's range carry unused values).
    TQ<4> p0q;          // input p rows f-3 .. f
    TQ<5> vxAq, rvxAq;  // stage A vx rows f-4 .. f
    TQ<5> vyAq, rvyAq;  // stage A vy rows f-6 .. f-2
    TQ<4> gAq;          // stage A d/dx vx rows f-3 .. f
    TQ<5> pAq, rpAq;    // stage A p rows f-7 .. f-3
    TQ<3> gBq;          // stage B d/dx vx rows f-7 .. f-5
    TQ<4> vyBq;         // stage B vy rows f-9 .. f-6
    __half2 accA[T_NS], accB[T_NS];
#pragma unroll
    for (int k = 0; k < T_NS; k++) accA[k] = accB[k] = __float2half2_rn(0.f);
    double eA[NCOMP] = {0.0, 0.0, 0.0, 0.0, 0.0}, eB[NCOMP] = {0.0, 0.0, 0.0, 0.0, 0.0};
    int rcA = rec_lower(P.rec, 0, P.n_rec, y0, INT_MIN);  // receiver cursors of this band
    int rcB = rcA;

    auto back = [&](int r, int k) { r -= k; return r < 0 ? r + ns : r; };  // wrapped row r - k (k < ns)
    int fw = wrap_row(F0);  // wrapped front row, advanced incrementally (no integer division in the loop)
#pragma unroll 1
    for (int i = 0; i < NI; i++, fw = fw + 1 == ns ? 0 : fw + 1) {
        const int f = F0 + i, slot = i % TR;
        if (tid == 0 && i + TR - 1 < NI) {
            fence_proxy_async_smem();
            issue(i + TR - 1);
        }
        mbar_wait(&bar[slot], (uint32_t)((i / TR) & 1));
        // ------------------------------------------------ phase 1 (stage A, step n)
        V4 rp0{};
        if (active) {
            p0q.push(ld4(slot_row(slot, T_P) + w));
            {  // vx_A[f] (acoustic.py:167-168)
                const V4 d = txfold<ORDER>(c, slot_row(slot, T_P), w, wl, wr, false);
                V4 v = ld4(slot_row(slot, T_VX) + w);
                V4 r = comp ? ld4(slot_row(slot, T_RVX) + w) : V4{};
                tupdate<V, ROWMED>(d, P.rho_x, fw, gx, dt2, -1, 0, srchA, 0.0, v, r);
                st4(xrA + (f & 1) * WW + w, v);
                vxAq.push(v);
                rvxAq.push(r);
                if (own_x && f >= y0 && f < y1) {
                    ttrack(accA[T_VX], v);
                    if (comp) ttrack(accA[T_RVX], r);
                    if (sampleA)
#pragma unroll
                        for (int k = 0; k < TCPT; k++) {
                            const double a = (double)__half2float(v.q[k >> 1].e[k & 1]);
                            eA[1] += p64(P.e_rho_x, f, 0, gx + k) * (a * a);
                        }
                }
            }
            {  // vy_A[f-2] from p rows f-3 .. f (acoustic.py:169-170)
                const int r = f - 2;
                const V4 d = tsfold<ORDER>(c, p0q.q[0], p0q.q[1], p0q.q[2], p0q.q[3]);
                V4 v = ld4(slot_row(slot, T_VS) + w);
                V4 rr = comp ? ld4(slot_row(slot, T_RVS) + w) : V4{};
                tupdate<V, ROWMED>(d, P.rho_s, back(fw, 2), gx, dt2, -1, 0, srchA, 0.0, v, rr);
                vyAq.push(v);
                rvyAq.push(rr);
                if (own_x && r >= y0 && r < y1) {
                    ttrack(accA[T_VS], v);
                    if (comp) ttrack(accA[T_RVS], rr);
                    if (sampleA)
#pragma unroll
                        for (int k = 0; k < TCPT; k++) {
                            const double a = (double)__half2float(v.q[k >> 1].e[k & 1]);
                            eA[2] += p64(P.e_rho_s, r, 0, gx + k) * (a * a);
                        }
                }
            }
            if (comp) rp0 = ld4(slot_row(slot, T_RP) + w);
        }
        // one barrier per row: xrA[f&1] holds vx_A[f]; xrP[(f-4)&1] holds p_A[f-4] and
        // xrB[(f-5)&1] holds vx_B[f-5] (both written in the previous iteration); every
        // thread is past its ring-slot reads.
        __syncthreads();
        // ------------------------------------------------ phase 2
        if (active) {
            gAq.push(txfold<ORDER>(c, xrA + (f & 1) * WW, w, wl, wr, true));
            {  // p_A[f-3] (acoustic.py:172-181)
                const int k = f - 3, kw = back(fw, 3);
                V4 pn = p0q.q[0];
                V4 rp = rp0;
                V4 dv;
#pragma unroll
                for (int j = 0; j < 2; j++)
                    dv.q[j] = O2::add(gAq.q[0].q[j],
                                      tfold<ORDER>(c, vyAq.q[1].q[j], vyAq.q[2].q[j], vyAq.q[3].q[j], vyAq.q[4].q[j]));
                tupdate<V, ROWMED>(dv, P.beta, kw, gx, dt2, kw == P.src_s ? sjA : -1, src_lane, srchA, srcA, pn, rp);
                st4(xrP + (k & 1) * WW + w, pn);
                if (own_x && k >= y0 && k < y1) {
                    ttrack(accA[T_P], pn);
                    if (comp) ttrack(accA[T_RP], rp);
                    if (sampleA)
#pragma unroll
                        for (int q = 0; q < TCPT; q++) {
                            const double a = (double)__half2float(p0q.q[0].q[q >> 1].e[q & 1]);
                            const double b = (double)__half2float(pn.q[q >> 1].e[q & 1]);
                            eA[0] += p64(P.e_beta, k, 0, gx + q) * (a * b);
                        }
                    rec_row(P.rec, rcA, P.n_rec, k, gx, P.traces, P.nt, n, [&](int o) { return tpick(pn, o); }, TCPT);
                }
                pAq.push(pn);
                rpAq.push(rp);
            }
            // ---------------------------------------- stage B (step n+1)
            gBq.push(txfold<ORDER>(c, xrB + ((f - 5) & 1) * WW, w, wl, wr, true));  // d/dx vx_B[f-5]
            {  // vx_B[f-4]: x taps of p_A[f-4]
                const int k = f - 4;
                V4 v = vxAq.q[0];
                V4 r = rvxAq.q[0];
                const V4 d = txfold<ORDER>(c, xrP + (k & 1) * WW, w, wl, wr, false);
                tupdate<V, ROWMED>(d, P.rho_x, back(fw, 4), gx, dt2, -1, 0, srchB, 0.0, v, r);
                st4(xrB + (k & 1) * WW + w, v);
                if (own_x && k >= y0 && k < y1) {
                    st4(P.out[T_VX] + (int64_t)k * pitch + gx, v);
                    ttrack(accB[T_VX], v);
                    if (comp) {
                        st4(P.out[T_RVX] + (int64_t)k * pitch + gx, r);
                        ttrack(accB[T_RVX], r);
                    }
                    if (sampleB)
#pragma unroll
                        for (int q = 0; q < TCPT; q++) {
                            const double a = (double)__half2float(v.q[q >> 1].e[q & 1]);
                            eB[1] += p64(P.e_rho_x, k, 0, gx + q) * (a * a);
                        }
                }
            }
            {  // vy_B[f-6] from stage-A p rows f-7 .. f-4
                const int k = f - 6;
                V4 v = vyAq.q[0];
                V4 rr = rvyAq.q[0];
                const V4 d = tsfold<ORDER>(c, pAq.q[0], pAq.q[1], pAq.q[2], pAq.q[3]);
                tupdate<V, ROWMED>(d, P.rho_s, back(fw, 6), gx, dt2, -1, 0, srchB, 0.0, v, rr);
                vyBq.push(v);
                if (own_x && k >= y0 && k < y1) {
                    st4(P.out[T_VS] + (int64_t)k * pitch + gx, v);
                    ttrack(accB[T_VS], v);
                    if (comp) {
                        st4(P.out[T_RVS] + (int64_t)k * pitch + gx, rr);
                        ttrack(accB[T_RVS], rr);
                    }
                    if (sampleB)
#pragma unroll
                        for (int q = 0; q < TCPT; q++) {
                            const double a = (double)__half2float(v.q[q >> 1].e[q & 1]);
                            eB[2] += p64(P.e_rho_s, k, 0, gx + q) * (a * a);
                        }
                }
            }
            {  // p_B[f-7]
                const int k = f - 7;
                if (k >= y0 && k < y1) {
                    V4 pn = pAq.q[0];
                    V4 rp = rpAq.q[0];
                    V4 dv;
#pragma unroll
                    for (int j = 0; j < 2; j++)
                        dv.q[j] = O2::add(gBq.q[0].q[j], tfold<ORDER>(c, vyBq.q[0].q[j], vyBq.q[1].q[j],
                                                                       vyBq.q[2].q[j], vyBq.q[3].q[j]));
                    tupdate<V, ROWMED>(dv, P.beta, k, gx, dt2, k == P.src_s ? sjB : -1, src_lane, srchB, srcB, pn, rp);
                    if (own_x) {
                        st4(P.out[T_P] + (int64_t)k * pitch + gx, pn);
                        ttrack(accB[T_P], pn);
                        if (comp) {
                            st4(P.out[T_RP] + (int64_t)k * pitch + gx, rp);
                            ttrack(accB[T_RP], rp);
                        }
                        if (sampleB)
#pragma unroll
                            for (int q = 0; q < TCPT; q++) {
                                const double a = (double)__half2float(pAq.q[0].q[q >> 1].e[q & 1]);
                                const double b = (double)__half2float(pn.q[q >> 1].e[q & 1]);
                                eB[0] += p64(P.e_beta, k, 0, gx + q) * (a * b);
                            }
                        rec_row(P.rec, rcB, P.n_rec, k, gx, P.traces, P.nt, n + 1, [&](int o) { return tpick(pn, o); },
                                TCPT);
                    }
                }
            }
        }
    }
    unsigned int maskA = 0, maskB = 0;
#pragma unroll
    for (int k = 0; k < T_NS; k++) {  // bit order p vx vy rp rvx rvy == stream order
        maskA |= tnonfinite(accA[k]) << k;
        maskB |= tnonfinite(accB[k]) << k;
    }
    record_failure(P.ctrl, n, maskA);
    record_failure(P.ctrl, n + 1, maskB);
    if (!sampleA && !sampleB) return;
    if (sampleA) block_partials(eA, P.partials);
    __syncthreads();  // block_partials' scratch is reused
    if (sampleB) block_partials(eB, T.partials_b);
    __threadfence();
    __syncthreads();
    __shared__ unsigned int is_last;
    if (tid == 0) is_last = atomicAdd(P.counter, 1u) == (unsigned int)(gridDim.x - 1);
    __syncthreads();
    if (!is_last) return;
    for (int st = 0; st < 2; st++) {  // fixed-order fp64 reduction of each stage's block partials
        if (!(st == 0 ? sampleA : sampleB)) continue;
        const double t = finalize_partials(st == 0 ? P.partials : T.partials_b, (int)gridDim.x);
        if (tid == 0) P.e_vals[st == 0 ? eidxA : eidxB] = P.scale * t;
        __syncthreads();
    }
    if (tid == 0) *P.counter = 0u;
}

// ---------------------------------------------------------------- host side

static int64_t tb2_xt(int64_t nx) { return nx < TXT_MAX ? nx : TXT_MAX; }

size_t tb2_smem_bytes(int64_t nx) {
    const int64_t WW = tb2_xt(nx) + 2 * THALO;
    return 128 + ((size_t)TR * T_NS + 6) * WW * sizeof(__half);
}

static int tb2_threads(int64_t nx) {
    const int64_t WW = tb2_xt(nx) + 2 * THALO;
    return (int)((WW / TCPT + 31) / 32 * 32);
}

bool tb2_eligible(int64_t nx, int64_t ns, int max_smem) {
    const int64_t xt = tb2_xt(nx);
    if (nx % 256 != 0 || nx % xt != 0 || ns < 16) return false;
    if (tb2_threads(nx) > 288) return false;
    return tb2_smem_bytes(nx) <= (size_t)max_smem;
}

// CTAs: x tiles x row bands, about one per SM
void tb2_grid(int64_t nx, int64_t ns, int nsm, int* ntiles, int* nbands) {
    const int t = (int)(nx / tb2_xt(nx));
    int b = nsm / t;
    if (b < 1) b = 1;
    if (b > ns / 8) b = (int)(ns / 8);
    if (b < 1) b = 1;
    *ntiles = t;
    *nbands = b;
}

template <bool RM>
static void* tb2_fn(int variant, int order) {
    if (order == 2) {
        if (variant == 0) return (void*)k_ac2d_tb2<0, 2, RM>;
        if (variant == 3) return (void*)k_ac2d_tb2<3, 2, RM>;
        return (void*)k_ac2d_tb2<6, 2, RM>;
    }
    if (variant == 0) return (void*)k_ac2d_tb2<0, 4, RM>;
    if (variant == 3) return (void*)k_ac2d_tb2<3, 4, RM>;
    return (void*)k_ac2d_tb2<6, 4, RM>;
}

cudaError_t tb2_prepare(int64_t nx) {
    const int bytes = (int)tb2_smem_bytes(nx);
    for (int v : {0, 3, 6})
        for (int o : {2, 4})
            for (void* fn : {tb2_fn<false>(v, o), tb2_fn<true>(v, o)}) {
                cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
                if (e != cudaSuccess) return e;
            }
    return cudaSuccess;
}

bool fused2d_rowmed(const AcFusedParams& P);

void launch_ac2d_tb2(int variant, int order, const AcFusedParams& F, int ntiles, int nbands, double* partials_b,
                     int64_t n, double srcA, double srcB, int sampleA, int sampleB, int64_t eidxA, int64_t eidxB,
                     cudaStream_t st) {
    AcTb2Params T;
    T.F = F;
    T.xt = tb2_xt(F.nx);
    T.ntiles = ntiles;
    T.nbands = nbands;
    T.partials_b = partials_b;
    void* fn = fused2d_rowmed(F) ? tb2_fn<true>(variant, order) : tb2_fn<false>(variant, order);
    void* args[] = {(void*)&T, (void*)&n, (void*)&srcA, (void*)&srcB, (void*)&sampleA, (void*)&sampleB,
                    (void*)&eidxA, (void*)&eidxB};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ntiles * nbands);
    cfg.blockDim = dim3(tb2_threads(F.nx));
    cfg.dynamicSmemBytes = tb2_smem_bytes(F.nx);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelExC(&cfg, fn, args);
}

}  // namespace hw
