// hw_elastic3d_fused.cu — one-pass 3D elastic leapfrog step, binary16 state, 2nd order,
// periodic (BASELINE config 5: 512^3, layered), sm_100a.
//
// Both phases of the 3D velocity-stress step (ElasticSolver._step_work, elastic.py:176-238,
// 3D extension of SURVEY §8 a'; the same ops and fold orders as k_el_vel / k_el_stress and the
// streaming kernels, so the bits are identical) in ONE kernel per step, state n read from
// buffer A and state n+1 written to buffer B.  The two streaming phase kernels move ~93 B per
// cell-step; this one moves the algorithmic 72 B plus one halo row per mid tile and field.
//
// A CTA (512 threads, 4 cells = 2 half2 each) owns a tile of TM = 2048/nx mid rows x the full
// x width and streams it along the slow axis ((tile, slab) units split evenly over the CTAs).
// Iteration i has front F = sb - 2 + i; the tap ring (4 slots) holds the six stress tiles of
// slabs F-2 .. F+1 (slab F+1 is requested at the top of iteration i, one iteration ahead):
//   sxx, sxs, sss : mid rows m0 .. m0+TM        (x / slow taps of vx, vs incl. their halo row m0+TM)
//   sxm, sms, smm : mid rows m0-1 .. m0+TM      (mid taps of vx, vs; x / slow / mid taps of vm incl.
//                                                its halo row m0-1)
// phase A: velocities of slab k = F-1 for the tile rows plus the halo rows vx, vs (m0+TM) and
//   vm (m0-1) (recomputed redundantly, never stored; rows j = 0, 1, 2 of threads take one each),
//   written to a velocity tile generation in shared memory;
// phase B: stresses of slab s = F-2 from the previous generation (x / mid taps, own rows of slab
//   s) and this generation's own rows (slow taps of vx, vm at s+1), v_slow(s-1) from registers.
// Old velocities / residuals of slab F-1 come through one staged slot (read in phase A, refilled
// during phase B), the stress residuals of slab F-2 through another (read in phase B, refilled
// during phase A).  All slab indices wrap (single periodic domain).
#include <cuda_runtime.h>

#include "hw_params.h"
#include "hw_stream.cuh"
#include "hw_tma.cuh"
#include "../../include/halfwave_b200.h"

namespace hw {

#ifndef HW_X3C
#define HW_X3C 4
#endif
constexpr int X3C = HW_X3C;        // cells per thread (X3C / 2 half2): 4 or 8
constexpr int X3T = 2048 / X3C;    // threads per CTA (TM = 2048 / nx either way)
constexpr int X3P = X3C / 2;       // half2 pairs per thread
constexpr int XR = 4;     // tap ring slots

struct E4 {
    EH2 q[X3P];
};

__device__ __forceinline__ E4 ld4(const __half* p) {
    E4 r;
    if constexpr (X3P == 2) {
        const uint2 u = *reinterpret_cast<const uint2*>(p);
        *reinterpret_cast<unsigned int*>(&r.q[0].h2) = u.x;
        *reinterpret_cast<unsigned int*>(&r.q[1].h2) = u.y;
    } else {
        const uint4 u = *reinterpret_cast<const uint4*>(p);
        *reinterpret_cast<unsigned int*>(&r.q[0].h2) = u.x;
        *reinterpret_cast<unsigned int*>(&r.q[1].h2) = u.y;
        *reinterpret_cast<unsigned int*>(&r.q[2].h2) = u.z;
        *reinterpret_cast<unsigned int*>(&r.q[3].h2) = u.w;
    }
    return r;
}

__device__ __forceinline__ void st4(__half* p, const E4& v) {
    if constexpr (X3P == 2) {
        uint2 u;
        u.x = *reinterpret_cast<const unsigned int*>(&v.q[0].h2);
        u.y = *reinterpret_cast<const unsigned int*>(&v.q[1].h2);
        *reinterpret_cast<uint2*>(p) = u;
    } else {
        uint4 u;
        u.x = *reinterpret_cast<const unsigned int*>(&v.q[0].h2);
        u.y = *reinterpret_cast<const unsigned int*>(&v.q[1].h2);
        u.z = *reinterpret_cast<const unsigned int*>(&v.q[2].h2);
        u.w = *reinterpret_cast<const unsigned int*>(&v.q[3].h2);
        *reinterpret_cast<uint4*>(p) = u;
    }
}

// x derivative of 4 cells (periodic) from a shared row; to_int: shifts (-1, 0) else (0, 1) (2nd order)
__device__ __forceinline__ E4 xf4(const __half c[4], const __half* row, int x, int xl, int xr, bool to_int) {
    EH2 Q[X3P + 2];
    Q[0] = e_ld2(row + xl);
    const E4 own = ld4(row + x);
#pragma unroll
    for (int j = 0; j < X3P; j++) Q[1 + j] = own.q[j];
    Q[X3P + 1] = e_ld2(row + xr);
    EH2 S[X3P + 1];
#pragma unroll
    for (int j = 0; j < X3P + 1; j++) S[j] = vshift<16, 2>(Q[j], Q[j + 1]);
    E4 r;
#pragma unroll
    for (int j = 0; j < X3P; j++)
        r.q[j] = to_int ? e_fold<2>(c, Q[j], S[j], Q[j + 1], S[j + 1]) : e_fold<2>(c, S[j], Q[j + 1], S[j + 1], Q[j + 2]);
    return r;
}

// 2nd-order fold of two rows a (first tap), b (second tap)
__device__ __forceinline__ E4 f4(const __half c[4], const E4& a, const E4& b) {
    E4 r;
#pragma unroll
    for (int j = 0; j < X3P; j++) r.q[j] = e_fold<2>(c, a.q[j], a.q[j], b.q[j], b.q[j]);
    return r;
}

__device__ __forceinline__ E4 add4(const E4& a, const E4& b) {
    E4 r;
#pragma unroll
    for (int j = 0; j < X3P; j++) r.q[j] = EO2::add(a.q[j], b.q[j]);
    return r;
}

__device__ __forceinline__ void track4(__half2& acc, const E4& v) {
#pragma unroll
    for (int j = 0; j < X3P; j++) acc = __hmax2_nan(acc, __habs2(v.q[j].h2));
}

// store of a row of 4 cells at element offset goff = s * slab + off; periodic ghost slabs written through
__device__ __forceinline__ void store4(const FieldView& f, int64_t slab, int s, int64_t off, const E4& v,
                                       bool inner) {
    __half* base = reinterpret_cast<__half*>(f.base);
    st4(base + (int64_t)s * slab + off, v);
    if (!inner && f.gtop == GHOST_PERIODIC) {  // inner: G <= s < rows - G, no ghost copy
        const int n = (int)f.rows;
        if (s >= n - G) st4(base + (int64_t)(s - n) * slab + off, v);
        if (s < G) st4(base + (int64_t)(n + s) * slab + off, v);
    }
}

// divisor finish for a velocity pair: row reciprocal (DIV_CHEAP, row-uniform) or the generic path
template <int V>
__device__ __forceinline__ void x3_finish_v(EH2 a, bool rm, float rc, const PlaneView& rho, int64_t s, int64_t m,
                                            int xc, __half dt, __half2 dt2, int src_lane, __half srch, double src,
                                            EH2& u, EH2& t) {
    if (rm) e_finish_rc<V>(a, rc, dt2, src_lane, srch, u, t);
    else finish<16, 16, 2>(a, &rho, s, m, xc, dt, V, src_lane, src, u, t);
}

// point source into the right-hand side of the source cell (the first op of finish()); a
// register select per pair (no dynamic indexing)
__device__ __forceinline__ void add_src2(EH2 r[X3P], int sj, int sln, __half srch) {
#pragma unroll
    for (int h = 0; h < X3P; h++)
        if (h == sj) {
            if (sln == 0) r[h].e[0] = __hadd_rn(r[h].e[0], srch);
            else r[h].e[1] = __hadd_rn(r[h].e[1], srch);
        }
}

enum { T_SXX = 0, T_SXS, T_SSS, T_SXM, T_SMS, T_SMM };

template <int V, bool SAMPLE>
__global__ void __launch_bounds__(X3T, 1)
    k_el3d_fused(ElParams P, El3In in, StreamIO IO, int64_t n, double src, int64_t eidx) {
    constexpr bool sample = SAMPLE;
    constexpr bool comp = V != 0;
    e_pdl_enter();
    if (halted(P.ctrl, n)) return;
    extern __shared__ __align__(128) unsigned char smem[];
    const int nx = (int)P.g.nx, nm = (int)P.g.nm, ns = (int)P.sxx.rows;
    const int64_t pitch = P.g.pitch, slab = P.g.slab;
    const int TM = X3T * X3C / nx, TPR = nx / X3C;
    const int tid = threadIdx.x, j = tid / TPR, x = (tid % TPR) * X3C;
    // shared layout (rows of pitch elements)
    const int tr1 = TM + 1, tr2 = TM + 2;                        // tile heights
    const int o_t[6] = {0, tr1, 2 * tr1, 3 * tr1, 3 * tr1 + tr2, 3 * tr1 + 2 * tr2};
    const int slot_rows = 3 * tr1 + 3 * tr2;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);            // XR tap barriers, A, B
    __half* ring = reinterpret_cast<__half*>(smem + 128);
    __half* arow = ring + (int64_t)XR * slot_rows * pitch;        // vx, vs, vm [rvx, rvs, rvm] (TM+1 rows each)
    __half* brow = arow + (int64_t)6 * tr1 * pitch;               // rsxx rsss rsmm rsxs rsxm rsms (TM rows each)
    __half* vtile = brow + (int64_t)6 * TM * pitch;               // 2 generations x [vx, vs, vm] (TM+1 rows each)
    auto tap = [&](int sl, int t) { return ring + ((int64_t)sl * slot_rows + o_t[t]) * pitch; };
    auto vt = [&](int gen, int q) { return vtile + ((int64_t)gen * 3 + q) * tr1 * pitch; };
    const uint32_t rb = (uint32_t)(pitch * sizeof(__half));
    if (tid == 0) {
        for (int q = 0; q < XR + 2; q++) mbar_init(&bar[q], 1);
        fence_mbar_init();
    }
    __syncthreads();
    uint64_t* abar = bar + XR;
    uint64_t* bbar = bar + XR + 1;

    __half c[4];
#pragma unroll
    for (int q = 0; q < 4; q++) c[q] = lconst<16>(P.k, q);
    const __half dt = lconst<16>(P.k, 4);
    const __half2 dt2 = __half2half2(dt);
    const __half srch = __double2half(src);
    const int xl = x == 0 ? nx - 2 : x - 2, xr = x + X3C >= nx ? 0 : x + X3C;
    const bool vsrc = P.src_kind == HW_SRC_VSLOW && src != 0.0;      // warp-uniform
    const bool ssrc = P.src_kind == HW_SRC_EXPLOSIVE && src != 0.0;  // warp-uniform
    const bool src_col = (vsrc || ssrc) && P.src_x >= x && P.src_x < x + X3C;
    const int sj = (int)((P.src_x - x) >> 1), sln = (int)((P.src_x - x) & 1);
    const bool rm = e_rowdiv(P.rho_x) && e_rowdiv(P.rho_s) && e_rowdiv(P.rho_m);
    const bool mrow = P.stiff.sx == 0 && P.lam.sx == 0 && P.mu_n.sx == 0;
    const bool erow = ((P.e_rho_x.sx | P.e_rho_s.sx | P.e_rho_m.sx | P.e_lam.sx | P.e_mu.sx | P.e_mu_n.sx) |
                       (P.e_rho_x.sm | P.e_rho_s.sm | P.e_rho_m.sm | P.e_lam.sm | P.e_mu.sm | P.e_mu_n.sm)) == 0;
    const FieldView* OS[6] = {&P.sxx, &P.sss, &P.smm, &P.sxs, &P.sxm, &P.sms};
    const FieldView* ORS[6] = {&P.rsxx, &P.rsss, &P.rsmm, &P.rsxs, &P.rsxm, &P.rsms};
    __half2 acc[9];
#pragma unroll
    for (int q = 0; q < 9; q++) acc[q] = __float2half2_rn(0.f);
    double e[NCOMP] = {0.0, 0.0, 0.0, 0.0, 0.0};

    auto wrap = [&](int s) { return s < 0 ? s + ns : (s >= ns ? s - ns : s); };
    const int tiles = nm / TM;
    const int64_t U = (int64_t)tiles * ns;
    int64_t u = (int64_t)blockIdx.x * U / gridDim.x;
    const int64_t u1 = (int64_t)(blockIdx.x + 1) * U / gridDim.x;
    int gi = 0, ga = 0, gb = 0;  // running use counters of the tap slots, the A and the B slot
    while (u < u1) {
        const int tile = (int)(u / ns), sb = (int)(u % ns);
        const int se = (int)min((int64_t)ns, sb + (u1 - u));
        u += se - sb;
        const int m0 = tile * TM, m = m0 + j;
        const int mlo = m0 == 0 ? nm - 1 : m0 - 1, mhi = m0 + TM == nm ? 0 : m0 + TM;  // halo rows (periodic)
        const int F0 = sb - 2, NI = se - sb + 4;
        const int gi0 = gi, ga0 = ga, gb0 = gb;
        auto issue_tap = [&](int i) {  // the six stress tiles of slab F0 + i
            const int sl = (gi0 + i) % XR, s = wrap(F0 + i);
            uint64_t* b = &bar[sl];
            mbar_arrive_expect_tx(b, (uint32_t)slot_rows * rb);
            a3_rows(tap(sl, T_SXX), in.sxx, slab, s, m0, m0 + TM + 1, nm, pitch, b);
            a3_rows(tap(sl, T_SXS), in.sxs, slab, s, m0, m0 + TM + 1, nm, pitch, b);
            a3_rows(tap(sl, T_SSS), in.sss, slab, s, m0, m0 + TM + 1, nm, pitch, b);
            a3_rows(tap(sl, T_SXM), in.sxm, slab, s, m0 - 1, m0 + TM + 1, nm, pitch, b);
            a3_rows(tap(sl, T_SMS), in.sms, slab, s, m0 - 1, m0 + TM + 1, nm, pitch, b);
            a3_rows(tap(sl, T_SMM), in.smm, slab, s, m0 - 1, m0 + TM + 1, nm, pitch, b);
        };
        auto issue_a = [&](int i) {  // old velocities (+ residuals) of slab F0 + i - 1
            const int s = wrap(F0 + i - 1);
            mbar_arrive_expect_tx(abar, (uint32_t)((comp ? 6 : 3) * tr1) * rb);
            a3_rows(arow, in.vx, slab, s, m0, m0 + TM + 1, nm, pitch, abar);
            a3_rows(arow + (int64_t)tr1 * pitch, in.vs, slab, s, m0, m0 + TM + 1, nm, pitch, abar);
            a3_rows(arow + (int64_t)2 * tr1 * pitch, in.vm, slab, s, m0 - 1, m0 + TM, nm, pitch, abar);
            if (comp) {
                a3_rows(arow + (int64_t)3 * tr1 * pitch, in.rvx, slab, s, m0, m0 + TM + 1, nm, pitch, abar);
                a3_rows(arow + (int64_t)4 * tr1 * pitch, in.rvs, slab, s, m0, m0 + TM + 1, nm, pitch, abar);
                a3_rows(arow + (int64_t)5 * tr1 * pitch, in.rvm, slab, s, m0 - 1, m0 + TM, nm, pitch, abar);
            }
        };
        auto issue_b = [&](int i) {  // stress residuals of slab F0 + i - 2 (own rows)
            const int s = wrap(F0 + i - 2);
            const int64_t off = (int64_t)s * slab + (int64_t)m0 * pitch;
            const uint32_t tb = (uint32_t)TM * rb;
            mbar_arrive_expect_tx(bbar, 6 * tb);
            const __half* R[6] = {in.rsxx, in.rsss, in.rsmm, in.rsxs, in.rsxm, in.rsms};
#pragma unroll
            for (int q = 0; q < 6; q++) tma_load_1d(brow + (int64_t)q * TM * pitch, R[q] + off, tb, bbar);
        };
        if (tid == 0) {
            issue_tap(0);
            issue_a(0);
        }
        E4 vs_m1, vs_m2;  // v_slow own rows of slabs F-2, F-3 (new)
#pragma unroll 1
        for (int i = 0; i < NI; i++) {
            const int F = F0 + i;
            const int s0 = (gi0 + i) % XR, s1 = (gi0 + i + XR - 1) % XR, s2 = (gi0 + i + XR - 2) % XR;  // F, F-1, F-2
            const int gen = i & 1;
            if (tid == 0 && i + 1 < NI) {  // slot (i+1) % XR held slab F-3: last read in iteration i-1
                fence_proxy_async_smem();
                issue_tap(i + 1);
            }
            mbar_wait(&bar[s0], (uint32_t)(((gi0 + i) / XR) & 1));
            mbar_wait(abar, (uint32_t)((ga0 + i) & 1));
            const bool vel = i >= 2;
            E4 vs_new;
            if (vel) {  // ---- velocities of slab k = F-1 (elastic.py:191-205, 3D)
                const int k = wrap(F - 1);
                const int64_t jr = (int64_t)j * pitch;
                // own rows: vx, vs at tile index j (row m), vm at index j + 1 of its tile
                E4 vx = ld4(arow + jr + x), vsv = ld4(arow + (int64_t)tr1 * pitch + jr + x);
                E4 vm = ld4(arow + (int64_t)(2 * tr1 + 1) * pitch + jr + x);
                E4 rvx = comp ? ld4(arow + (int64_t)3 * tr1 * pitch + jr + x) : E4{};
                E4 rvs = comp ? ld4(arow + (int64_t)4 * tr1 * pitch + jr + x) : E4{};
                E4 rvm = comp ? ld4(arow + (int64_t)(5 * tr1 + 1) * pitch + jr + x) : E4{};
                const float rcx = rm ? e_rcp_at(P.rho_x, k, m) : 0.f;
                const float rcs = rm ? e_rcp_at(P.rho_s, k, m) : 0.f;
                const float rcm = rm ? e_rcp_at(P.rho_m, k, m) : 0.f;
                // vx: fl(fl(ddx sxx + dds sxs) + ddm sxm)
                E4 ax = add4(add4(xf4(c, tap(s1, T_SXX) + jr, x, xl, xr, false),
                                  f4(c, ld4(tap(s2, T_SXS) + jr + x), ld4(tap(s1, T_SXS) + jr + x))),
                             f4(c, ld4(tap(s1, T_SXM) + jr + x), ld4(tap(s1, T_SXM) + jr + pitch + x)));
                // v_slow: fl(fl(ddx sxs + dds sss) + ddm sms) (+ src)
                E4 as = add4(add4(xf4(c, tap(s1, T_SXS) + jr, x, xl, xr, true),
                                  f4(c, ld4(tap(s1, T_SSS) + jr + x), ld4(tap(s0, T_SSS) + jr + x))),
                             f4(c, ld4(tap(s1, T_SMS) + jr + x), ld4(tap(s1, T_SMS) + jr + pitch + x)));
                // v_mid: fl(fl(ddx sxm + dds sms) + ddm smm)
                E4 am = add4(add4(xf4(c, tap(s1, T_SXM) + jr + pitch, x, xl, xr, true),
                                  f4(c, ld4(tap(s2, T_SMS) + jr + pitch + x), ld4(tap(s1, T_SMS) + jr + pitch + x))),
                             f4(c, ld4(tap(s1, T_SMM) + jr + pitch + x), ld4(tap(s1, T_SMM) + jr + 2 * pitch + x)));
                if (vsrc && k == P.src_s && m == P.src_m && src_col) {
                    add_src2(as.q, sj, sln, srch);
                }
#pragma unroll
                for (int h = 0; h < X3P; h++) {
                    x3_finish_v<V>(ax.q[h], rm, rcx, P.rho_x, k, m, x + 2 * h, dt, dt2, -1, srch, 0.0, vx.q[h], rvx.q[h]);
                    x3_finish_v<V>(as.q[h], rm, rcs, P.rho_s, k, m, x + 2 * h, dt, dt2, -1, srch, 0.0, vsv.q[h], rvs.q[h]);
                    x3_finish_v<V>(am.q[h], rm, rcm, P.rho_m, k, m, x + 2 * h, dt, dt2, -1, srch, 0.0, vm.q[h], rvm.q[h]);
                }
                st4(vt(gen, 0) + jr + x, vx);
                st4(vt(gen, 1) + jr + x, vsv);
                st4(vt(gen, 2) + jr + pitch + x, vm);
                vs_new = vsv;
                const int sk = F - 1;  // unwrapped: stored only inside the segment
                if (sk >= sb && sk < se) {
                    const int64_t off = (int64_t)m * pitch + x;
                    const bool kin = k >= G && k < ns - G;
                    store4(P.vx, slab, k, off, vx, kin);
                    store4(P.vs, slab, k, off, vsv, kin);
                    store4(P.vm, slab, k, off, vm, kin);
                    track4(acc[0], vx);
                    track4(acc[1], vsv);
                    track4(acc[2], vm);
                    if (comp) {
                        store4(P.rvx, slab, k, off, rvx, kin);
                        store4(P.rvs, slab, k, off, rvs, kin);
                        store4(P.rvm, slab, k, off, rvm, kin);
                    }
                }
                // halo rows (recomputed, not stored): j = 0 -> vm(m0-1), j = 1 -> vx(m0+TM), j = 2 -> vs(m0+TM)
                if (j == 0) {
                    E4 h = ld4(arow + (int64_t)2 * tr1 * pitch + x);
                    E4 rh = comp ? ld4(arow + (int64_t)5 * tr1 * pitch + x) : E4{};
                    const E4 a = add4(add4(xf4(c, tap(s1, T_SXM), x, xl, xr, true),
                                           f4(c, ld4(tap(s2, T_SMS) + x), ld4(tap(s1, T_SMS) + x))),
                                      f4(c, ld4(tap(s1, T_SMM) + x), ld4(tap(s1, T_SMM) + pitch + x)));
                    const float rc = rm ? e_rcp_at(P.rho_m, k, mlo) : 0.f;
#pragma unroll
                    for (int q = 0; q < X3P; q++)
                        x3_finish_v<V>(a.q[q], rm, rc, P.rho_m, k, mlo, x + 2 * q, dt, dt2, -1, srch, 0.0, h.q[q], rh.q[q]);
                    st4(vt(gen, 2) + x, h);
                } else if (j == 1) {
                    const int64_t hr = (int64_t)TM * pitch;
                    E4 h = ld4(arow + hr + x);
                    E4 rh = comp ? ld4(arow + (int64_t)3 * tr1 * pitch + hr + x) : E4{};
                    const E4 a = add4(add4(xf4(c, tap(s1, T_SXX) + hr, x, xl, xr, false),
                                           f4(c, ld4(tap(s2, T_SXS) + hr + x), ld4(tap(s1, T_SXS) + hr + x))),
                                      f4(c, ld4(tap(s1, T_SXM) + hr + x), ld4(tap(s1, T_SXM) + hr + pitch + x)));
                    const float rc = rm ? e_rcp_at(P.rho_x, k, mhi) : 0.f;
#pragma unroll
                    for (int q = 0; q < X3P; q++)
                        x3_finish_v<V>(a.q[q], rm, rc, P.rho_x, k, mhi, x + 2 * q, dt, dt2, -1, srch, 0.0, h.q[q], rh.q[q]);
                    st4(vt(gen, 0) + hr + x, h);
                } else if (j == 2) {
                    const int64_t hr = (int64_t)TM * pitch;
                    E4 h = ld4(arow + (int64_t)tr1 * pitch + hr + x);
                    E4 rh = comp ? ld4(arow + (int64_t)4 * tr1 * pitch + hr + x) : E4{};
                    E4 a = add4(add4(xf4(c, tap(s1, T_SXS) + hr, x, xl, xr, true),
                                     f4(c, ld4(tap(s1, T_SSS) + hr + x), ld4(tap(s0, T_SSS) + hr + x))),
                                f4(c, ld4(tap(s1, T_SMS) + hr + x), ld4(tap(s1, T_SMS) + hr + pitch + x)));
                    if (vsrc && k == P.src_s && mhi == P.src_m && src_col) {
                        add_src2(a.q, sj, sln, srch);
                    }
                    const float rc = rm ? e_rcp_at(P.rho_s, k, mhi) : 0.f;
#pragma unroll
                    for (int q = 0; q < X3P; q++)
                        x3_finish_v<V>(a.q[q], rm, rc, P.rho_s, k, mhi, x + 2 * q, dt, dt2, -1, srch, 0.0, h.q[q], rh.q[q]);
                    st4(vt(gen, 1) + hr + x, h);
                }
            }
            __syncthreads();  // velocity tiles of slab F-1 visible; the A slot and tap slot (i+1) % XR are free
            if (tid == 0 && i + 1 < NI) {
                fence_proxy_async_smem();
                issue_a(i + 1);
            }
            const int s = F - 2;  // stress slab (unwrapped)
            if (s >= sb && s < se) {  // ---- stresses of slab s (elastic.py:210-238, 3D)
                mbar_wait(bbar, (uint32_t)((gb0 + (i - 4)) & 1));
                const int64_t jr = (int64_t)j * pitch;
                const int pg = gen ^ 1;  // generation of slab s
                const __half* vxt = vt(pg, 0);  // rows m0 .. m0+TM
                const __half* vst = vt(pg, 1);  // rows m0 .. m0+TM
                const __half* vmt = vt(pg, 2);  // rows m0-1 .. m0+TM-1
                const E4 dvx = xf4(c, vxt + jr, x, xl, xr, true);
                const E4 dvs = f4(c, vs_m2, vs_m1);  // v_slow(s-1), v_slow(s) (own rows)
                const E4 dvm = f4(c, ld4(vmt + jr + x), ld4(vmt + jr + pitch + x));
                E4 old[6], nw[6], rr[6];
                old[0] = ld4(tap(s2, T_SXX) + jr + x);
                old[1] = ld4(tap(s2, T_SSS) + jr + x);
                old[2] = ld4(tap(s2, T_SMM) + jr + pitch + x);
                old[3] = ld4(tap(s2, T_SXS) + jr + x);
                old[4] = ld4(tap(s2, T_SXM) + jr + pitch + x);
                old[5] = ld4(tap(s2, T_SMS) + jr + pitch + x);
#pragma unroll
                for (int q = 0; q < 6; q++) {
                    nw[q] = old[q];
                    rr[q] = comp ? ld4(brow + (int64_t)q * TM * pitch + jr + x) : E4{};
                }
                const int sw = s;  // (s in [0, ns): no wrap)
                EH2 stiff_r, lam_r, mu_r;
                if (mrow) {
                    stiff_r = e_val_at(P.stiff, sw, m);
                    lam_r = e_val_at(P.lam, sw, m);
                    mu_r = e_val_at(P.mu_n, sw, m);
                }
                EH2 a0[X3P], a1[X3P], a2[X3P];
#pragma unroll
                for (int h = 0; h < X3P; h++) {
                    const EH2 stiff = mrow ? stiff_r : pload<16, 2>(P.stiff, sw, m, x + 2 * h);
                    const EH2 lam = mrow ? lam_r : pload<16, 2>(P.lam, sw, m, x + 2 * h);
                    a0[h] = EO2::add(EO2::add(EO2::mul(stiff, dvx.q[h]), EO2::mul(lam, dvs.q[h])), EO2::mul(lam, dvm.q[h]));
                    a1[h] = EO2::add(EO2::add(EO2::mul(lam, dvx.q[h]), EO2::mul(stiff, dvs.q[h])), EO2::mul(lam, dvm.q[h]));
                    a2[h] = EO2::add(EO2::add(EO2::mul(lam, dvx.q[h]), EO2::mul(lam, dvs.q[h])), EO2::mul(stiff, dvm.q[h]));
                }
                if (ssrc && sw == P.src_s && m == P.src_m && src_col) {  // explosive source into the normal stresses
                    add_src2(a0, sj, sln, srch);
                    add_src2(a1, sj, sln, srch);
                    add_src2(a2, sj, sln, srch);
                }
                // shear: fl(mu fl(dd_a v_b + dd_b v_a)), to-half taps
                const E4 sxs_a = f4(c, ld4(vxt + jr + x), ld4(vt(gen, 0) + jr + x));      // vx(s), vx(s+1)
                const E4 sxs_b = xf4(c, vst + jr, x, xl, xr, false);
                const E4 sxm_a = f4(c, ld4(vxt + jr + x), ld4(vxt + jr + pitch + x));     // vx rows m, m+1
                const E4 sxm_b = xf4(c, vmt + jr + pitch, x, xl, xr, false);
                const E4 sms_a = f4(c, ld4(vmt + jr + pitch + x), ld4(vt(gen, 2) + jr + pitch + x));  // vm(s), vm(s+1)
                const E4 sms_b = f4(c, ld4(vst + jr + x), ld4(vst + jr + pitch + x));     // vs rows m, m+1
#pragma unroll
                for (int h = 0; h < X3P; h++) {
                    e2_finish_nd<V>(a0[h], dt2, -1, srch, nw[0].q[h], rr[0].q[h]);
                    e2_finish_nd<V>(a1[h], dt2, -1, srch, nw[1].q[h], rr[1].q[h]);
                    e2_finish_nd<V>(a2[h], dt2, -1, srch, nw[2].q[h], rr[2].q[h]);
                    const EH2 mu = mrow ? mu_r : pload<16, 2>(P.mu_n, sw, m, x + 2 * h);
                    e2_finish_nd<V>(EO2::mul(mu, EO2::add(sxs_a.q[h], sxs_b.q[h])), dt2, -1, srch, nw[3].q[h], rr[3].q[h]);
                    e2_finish_nd<V>(EO2::mul(mu, EO2::add(sxm_a.q[h], sxm_b.q[h])), dt2, -1, srch, nw[4].q[h], rr[4].q[h]);
                    e2_finish_nd<V>(EO2::mul(mu, EO2::add(sms_a.q[h], sms_b.q[h])), dt2, -1, srch, nw[5].q[h], rr[5].q[h]);
                }
                const int64_t off = (int64_t)m * pitch + x;
                const bool sin = sw >= G && sw < ns - G;
#pragma unroll
                for (int q = 0; q < 6; q++) {
                    store4(*OS[q], slab, sw, off, nw[q], sin);
                    track4(acc[3 + q], nw[q]);
                    if (comp) store4(*ORS[q], slab, sw, off, rr[q], sin);
                }
                if (sample) {  // diagnostics.py:100-162, 3D compliance form (k_el_stress)
                    const E4 vxo = ld4(vxt + jr + x), vmo = ld4(vmt + jr + pitch + x), vso = ld4(vst + jr + x);
                    auto f = [&](const E4& a, int q) { return (double)__half2float(a.q[q >> 1].e[q & 1]); };
                    if (erow) {
                        double skx = 0.0, skm = 0.0, sks = 0.0, sx1 = 0.0, sdot = 0.0, str = 0.0, ssh = 0.0;
#pragma unroll
                        for (int q = 0; q < X3C; q++) {
                            const double a = f(vxo, q), b = f(vmo, q), g = f(vso, q);
                            skx += a * a;
                            skm += b * b;
                            sks += g * g;
                            const double xn = f(old[0], q), x1 = f(nw[0], q), sn = f(old[1], q), s1 = f(nw[1], q);
                            const double mn = f(old[2], q), m1 = f(nw[2], q);
                            sx1 += xn * x1;
                            sdot += xn * x1 + sn * s1 + mn * m1;
                            str += (xn + sn + mn) * (x1 + s1 + m1);
                            ssh += f(old[3], q) * f(nw[3], q) + f(old[4], q) * f(nw[4], q) + f(old[5], q) * f(nw[5], q);
                        }
                        e[0] += p64(P.e_rho_x, sw, 0, 0) * skx;
                        e[2] += p64(P.e_rho_m, sw, 0, 0) * skm;
                        e[1] += p64(P.e_rho_s, sw, 0, 0) * sks;
                        const double lamd = p64(P.e_lam, sw, 0, 0), mu = p64(P.e_mu, sw, 0, 0);
                        if (mu == 0.0) e[3] += sx1 / (lamd + mu);
                        else e[3] += sdot / (2.0 * mu) - lamd * str / (2.0 * mu * (3.0 * lamd + 2.0 * mu));
                        const double mun = p64(P.e_mu_n, sw, 0, 0);
                        e[4] += mun > 0.0 ? ssh / mun : 0.0;
                    } else {
#pragma unroll
                        for (int q = 0; q < X3C; q++) {
                            const int xi = x + q;
                            const double a = f(vxo, q), b = f(vmo, q), g = f(vso, q);
                            e[0] += p64(P.e_rho_x, sw, m, xi) * (a * a);
                            e[2] += p64(P.e_rho_m, sw, m, xi) * (b * b);
                            e[1] += p64(P.e_rho_s, sw, m, xi) * (g * g);
                            const double lamd = p64(P.e_lam, sw, m, xi), mu = p64(P.e_mu, sw, m, xi);
                            const double xn = f(old[0], q), x1 = f(nw[0], q), sn = f(old[1], q), s1 = f(nw[1], q);
                            const double mn = f(old[2], q), m1 = f(nw[2], q);
                            if (mu == 0.0) {
                                e[3] += (xn * x1) / (lamd + mu);
                            } else {
                                const double dot = xn * x1 + sn * s1 + mn * m1;
                                e[3] += dot / (2.0 * mu) -
                                        lamd * (xn + sn + mn) * (x1 + s1 + m1) / (2.0 * mu * (3.0 * lamd + 2.0 * mu));
                            }
                            const double mun = p64(P.e_mu_n, sw, m, xi);
                            for (int w = 3; w < 6; w++) e[4] += mun > 0.0 ? (f(old[w], q) * f(nw[w], q)) / mun : 0.0;
                        }
                    }
                }
            }
            if (vel) {
                vs_m2 = vs_m1;
                vs_m1 = vs_new;
            }
            __syncthreads();  // the previous velocity generation and the B slot are free
            if (tid == 0 && i + 1 < NI && F + 1 - 2 >= sb && F + 1 - 2 < se) {
                fence_proxy_async_smem();
                issue_b(i + 1);
            }
        }
        gi += NI;
        ga += NI;
        gb += se - sb;
    }
    unsigned int mask = 0;
    mask |= e_nonfinite(acc[0]) << P.vx.bit;  // (residuals: see k_el2d_fused)
    mask |= e_nonfinite(acc[1]) << P.vs.bit;
    mask |= e_nonfinite(acc[2]) << P.vm.bit;
#pragma unroll
    for (int q = 0; q < 6; q++) mask |= e_nonfinite(acc[3 + q]) << OS[q]->bit;
    record_failure(P.ctrl, n, mask);
    if constexpr (!SAMPLE) return;
    block_partials(e, P.partials);
    __threadfence();
    __syncthreads();
    __shared__ unsigned int is_last;
    if (tid == 0) is_last = atomicAdd(IO.counter, 1u) == (unsigned int)(gridDim.x - 1);
    __syncthreads();
    if (!is_last) return;
    const double t = finalize_partials(P.partials, (int)gridDim.x);  // fixed-order fp64 reduction
    if (tid == 0) {
        IO.e_vals[eidx] = IO.scale * t;
        *IO.counter = 0u;
    }
}

// ---------------------------------------------------------------- host side

static size_t x3_bytes(int64_t nx) {
    const int64_t TM = X3T * X3C / nx;
    const int64_t rows = XR * (6 * TM + 9) + 6 * (TM + 1) + 6 * TM + 6 * (TM + 1);
    return 128 + (size_t)rows * nx * sizeof(__half);
}

bool el3d_fused_eligible(int64_t nx, int64_t nm, int64_t ns, int64_t pitch, int order, int max_smem) {
    if (order != 2 || nx % 256 != 0 || nx > X3T * X3C || pitch != nx || ns < 4) return false;
    const int64_t TM = X3T * X3C / nx;
    if (TM < 3 || nm % TM != 0 || nm < 2 * TM) return false;  // the three halo rows take thread rows j = 0, 1, 2
    return x3_bytes(nx) <= (size_t)max_smem;
}

cudaError_t el3d_fused_prepare(int64_t nx) {
    const int b = (int)x3_bytes(nx);
    void* fns[] = {(void*)k_el3d_fused<0, false>, (void*)k_el3d_fused<3, false>, (void*)k_el3d_fused<6, false>,
                   (void*)k_el3d_fused<0, true>, (void*)k_el3d_fused<3, true>, (void*)k_el3d_fused<6, true>};
    for (void* fn : fns) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
    return cudaGetLastError();
}

void launch_el3d_fused(int variant, const ElParams& P, const El3In& in, const StreamIO& IO, int nblocks, int64_t n,
                       double src, int sample, int64_t eidx, cudaStream_t st) {
    void* fn;
    if (sample) fn = variant == 0 ? (void*)k_el3d_fused<0, true> : (variant == 3 ? (void*)k_el3d_fused<3, true> : (void*)k_el3d_fused<6, true>);
    else fn = variant == 0 ? (void*)k_el3d_fused<0, false> : (variant == 3 ? (void*)k_el3d_fused<3, false> : (void*)k_el3d_fused<6, false>);
    void* args[] = {(void*)&P, (void*)&in, (void*)&IO, (void*)&n, (void*)&src, (void*)&eidx};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nblocks);
    cfg.blockDim = dim3(X3T);
    cfg.dynamicSmemBytes = x3_bytes(P.g.nx);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelExC(&cfg, fn, args);
}

}  // namespace hw
