// hw_acoustic3d_fused.cu — one-pass 3D acoustic leapfrog step, binary16 state, 2nd order
// (BASELINE config 3: 512^3, per-cell beta, periodic), sm_100a.
//
// Both phases of AcousticSolver._step_work (acoustic.py:162-181, 3D extension of SURVEY
// §8 a') in ONE kernel per step, reading state n from buffer A and writing state n+1 to
// buffer B (ping-pong: no CTA ever reads a value another CTA has already advanced).
// The two-phase streaming kernels (hw_acoustic3d_stream.cu) move 42 B per cell-step; this
// one moves the algorithmic 34 B plus the mid-axis halo rows (p: 2 rows, vm/rvm: 1 row
// per TM-row tile).
//
// A CTA owns a tile of TM = 4096/nx mid rows x the full x width and streams it along the
// slow axis (the (tile, slab) units are split evenly over the CTAs, as in the streaming
// kernels).  Iteration i has front F = sb - 1 + i and output slab s = F - 1:
//   * the tap ring (5 slots, filled 3 slabs ahead) brings the p tile of slab F, rows
//     m0-1 .. m0+TM (TM+2 rows, periodic wrap);
//   * the own ring (2 slots, one slab ahead) brings vx, vs, rp, beta, rvx, rvs (TM rows)
//     and vm, rvm (TM+1 rows from m0-1) of slab s;
//   * v_slow(s) = fold(p(s), p(s+1)) from a 2-deep register queue of p rows;
//     vx(s) from the p tile of slab s (previous slot), x taps;
//     vm(s) for rows m0-1 .. m0+TM-1 (row m0-1 recomputed redundantly by the j = 0
//     threads: it is the to-int mid tap of row m0);
//   * the new vx and vm rows go to shared memory (their x / mid neighbours belong to
//     other threads), one barrier, then p(s) = fold(fl(fl(ddx vx + dds vs) + ddm vm))
//     with v_slow(s-1) from the register queue.
// The first iteration of a segment only fills the queue, the second computes
// v_slow(sb-1) (not stored: the neighbouring segment owns it).  Every op and fold order is
// the one k_ac_vel / k_ac_pres (and the streaming kernels) use, so the bits are identical.
#include <cuda_runtime.h>

#include "hw_params.h"
#include "hw_stream.cuh"
#include "hw_tma.cuh"
#include "../../include/halfwave_b200.h"

namespace hw {

constexpr int FR = 5;      // tap ring slots (slot i-1 is read during iteration i)
constexpr int FD = 3;      // prefetch distance
constexpr int F3T = 512;   // threads per CTA; TM = F3T * ECPT / nx

// own-ring row blocks (units of TM rows, + 1 row for the two mid-halo fields)
enum { O_VX = 0, O_VS, O_RP, O_BETA, O_RVX, O_RVS, O_NTM };

struct F3Layout {
    uint64_t* bar;
    uint64_t* obar;
    __half* ring;   // FR slots x (TM + 2) rows
    __half* own;    // 2 slots x (O_NTM * TM + 2 * (TM + 1)) rows
    __half* xv;     // TM rows: new vx of slab s
    __half* vmn;    // TM + 1 rows: new vm of slab s, rows m0-1 .. m0+TM-1
    int64_t slot, oslot, tm, pitch;
    __device__ __forceinline__ F3Layout(unsigned char* smem, int TM, int64_t pitch_)
        : bar(reinterpret_cast<uint64_t*>(smem)), obar(reinterpret_cast<uint64_t*>(smem + 64)),
          ring(reinterpret_cast<__half*>(smem + 128)),
          own(ring + (int64_t)FR * (TM + 2) * pitch_),
          xv(own + 2 * ((int64_t)O_NTM * TM + 2 * (TM + 1)) * pitch_),
          vmn(xv + (int64_t)TM * pitch_),
          slot((int64_t)(TM + 2) * pitch_), oslot(((int64_t)O_NTM * TM + 2 * (TM + 1)) * pitch_),
          tm((int64_t)TM * pitch_), pitch(pitch_) {}
    __device__ __forceinline__ __half* sl(int k) const { return ring + k * slot; }
    __device__ __forceinline__ __half* ob(int os, int q) const { return own + os * oslot + q * tm; }
    __device__ __forceinline__ __half* ovm(int os) const { return own + os * oslot + O_NTM * tm; }
    __device__ __forceinline__ __half* orvm(int os) const { return ovm(os) + tm + pitch; }
};

static size_t f3_bytes(int64_t nx) {
    const int64_t TM = F3T * ECPT / nx;
    const int64_t rows = FR * (TM + 2) + 2 * (O_NTM * TM + 2 * (TM + 1)) + TM + (TM + 1);
    return 128 + (size_t)rows * nx * sizeof(__half);
}

// one finished velocity row: row-uniform reciprocal rc (prefetched) or the generic plane path
template <int V>
__device__ __forceinline__ void f3_finish_v(const E8& a, bool rm, float rc, const PlaneView& rho, int64_t s, int64_t m,
                                            int x, __half dt, __half2 dt2, __half zero_h, E8& v, E8& rr) {
    if (rm) {
#pragma unroll
        for (int h = 0; h < 4; h++) e_finish_rc<V>(a.q[h], rc, dt2, -1, zero_h, v.q[h], rr.q[h]);
    } else {
#pragma unroll
        for (int h = 0; h < 4; h++) finish<16, 16, 2>(a.q[h], &rho, s, m, x + 2 * h, dt, V, -1, 0.0, v.q[h], rr.q[h]);
    }
}

// NXC: the row width as a compile-time constant (512, BASELINE config 3: shared-memory and row
// offsets fold into immediates) or 0 (runtime width); SAMPLE: energy sample step.
template <int V, int NXC, bool SAMPLE>
__global__ void __launch_bounds__(F3T, 1)
    k_ac3d_fused(AcParams P, Ac3In in, StreamIO IO, int64_t n, double src, int64_t eidx) {
    constexpr bool sample = SAMPLE;
    e_pdl_enter();
    if (halted(P.ctrl, n)) return;
    extern __shared__ __align__(128) unsigned char smem[];
    const int nx = NXC ? NXC : (int)P.g.nx, nm = (int)P.g.nm, ns = (int)P.p.rows;
    const int64_t pitch = NXC ? NXC : P.g.pitch, slab = (int64_t)nm * pitch;
    const int TM = F3T * ECPT / nx, TPR = nx / ECPT;
    const F3Layout L(smem, TM, pitch);
    const int tid = threadIdx.x, j = tid / TPR, x = (tid % TPR) * ECPT;
    constexpr bool comp = V != 0;
    const bool bfull = P.beta.sx != 0;
    const bool brow = !bfull && e_rowdiv(P.beta);
    const bool rm = e_rowdiv(P.rho_x) && e_rowdiv(P.rho_s) && e_rowdiv(P.rho_m);
    const uint32_t tmb = (uint32_t)(L.tm * sizeof(__half));
    // own bytes per slab: vx, vs [, beta] [, rp, rvx, rvs] (TM rows) + vm [, rvm] (TM + 1 rows)
    const uint32_t own_tx = (uint32_t)((2 + (bfull ? 1 : 0) + (comp ? 3 : 0)) * L.tm * sizeof(__half) +
                                       (comp ? 2 : 1) * (L.tm + pitch) * sizeof(__half));
    if (tid == 0) {
        for (int q = 0; q < FR; q++) mbar_init(&L.bar[q], 1);
        for (int q = 0; q < 2; q++) mbar_init(&L.obar[q], 1);
        fence_mbar_init();
    }
    __syncthreads();
    __half c[4];
#pragma unroll
    for (int q = 0; q < 4; q++) c[q] = lconst<16>(P.k, q);
    const __half dt = lconst<16>(P.k, 4);
    const __half2 dt2 = __half2half2(dt);
    const __half zero_h = __float2half(0.f);
    const __half srch = __double2half(src);
    const int xl = x == 0 ? nx - 2 : x - 2, xr = x + ECPT >= nx ? 0 : x + ECPT;
    const bool src_col = P.has_src && src != 0.0 && P.src_x >= x && P.src_x < x + ECPT;
    const int sj = (int)((P.src_x - x) >> 1), sln = (int)((P.src_x - x) & 1);
    __half2 acc[8];
#pragma unroll
    for (int q = 0; q < 8; q++) acc[q] = __float2half2_rn(0.f);
    __shared__ double ered[32];  // per-warp energy partials of one (tile, slab) unit (sample steps)

    // groups of `grp` CTAs own `grp` adjacent mid tiles and stream the same slab range side by side:
    // the halo rows one CTA reads are rows its neighbour in the group reads at about the same time
    // (L2 hits instead of DRAM re-reads); the (tile group, slab) units are split evenly over the groups
    const int grp = in.group, ngrp = (int)gridDim.x / grp, gid = (int)blockIdx.x / grp, gr = (int)blockIdx.x % grp;
    const int tiles = nm / TM / grp;  // tile groups
    // Band mode (NCCL slab, exchange overlapped): 1 = the edge slabs 0 and ns-1 (every row the halo
    // exchange sends; the only slabs that read ghost rows), 2 = the interior [1, ns-1), 0 = every slab.
    // t indexes the band's slabs; a segment never straddles the two edge slabs.
    const int E = in.edge, bm = in.band;
    const int nsl = bm == 0 ? ns : (bm == 1 ? 2 * E : ns - 2 * E);
    auto slab_of = [&](int t) { return bm == 0 ? t : (bm == 1 ? (t < E ? t : ns - 2 * E + t) : E + t); };
    const int64_t U = (int64_t)tiles * nsl;
    int64_t u = (int64_t)gid * U / ngrp;
    const int64_t u1 = (int64_t)(gid + 1) * U / ngrp;
    int gi = 0, gk = 0;  // running tap / own use counters (slot and parity continue across segments)
    while (u < u1) {
        const int t0 = (int)(u % nsl);
        int te = (int)min((int64_t)nsl, t0 + (u1 - u));
        if (bm == 1 && t0 < E) te = min(te, E);
        const int tile = (int)(u / nsl) * grp + gr, sb = slab_of(t0), se = sb + (te - t0);
        u += te - t0;
        const int m0 = tile * TM, m = m0 + j;
        const int mh = m0 == 0 ? nm - 1 : m0 - 1;  // mid halo row (periodic)
        const int F0 = sb - 1, NI = se - sb + 2;
        const int gi0 = gi, gk0 = gk;
        auto issue = [&](int i) {
            const int F = F0 + i, k = (gi0 + i) % FR;
            mbar_arrive_expect_tx(&L.bar[k], (uint32_t)(L.slot * sizeof(__half)));
            a3_rows(L.sl(k), in.p, slab, e_row(F), m0 - 1, m0 + TM + 1, nm, pitch, &L.bar[k]);
        };
        auto issue_own = [&](int kk) {  // slab sb - 1 + kk (periodic: slab -1 is ns - 1, residuals have no ghosts;
                                        // a decomposed domain's slab: ghost row -1 from the exchange)
            const int os = (gk0 + kk) & 1, s = sb - 1 + kk < 0 ? (in.slab ? -1 : ns - 1) : sb - 1 + kk;
            const int64_t off = (int64_t)s * slab + (int64_t)m0 * pitch;
            uint64_t* b = &L.obar[os];
            mbar_arrive_expect_tx(b, own_tx);
            tma_load_1d(L.ob(os, O_VX), in.vx + off, tmb, b);
            tma_load_1d(L.ob(os, O_VS), in.vs + off, tmb, b);
            if (bfull) tma_load_1d(L.ob(os, O_BETA), reinterpret_cast<const __half*>(P.beta.p) + s * P.beta.ss +
                                                          (int64_t)m0 * P.beta.sm, tmb, b);
            a3_rows(L.ovm(os), in.vm, slab, s, m0 - 1, m0 + TM, nm, pitch, b);
            if (comp) {
                tma_load_1d(L.ob(os, O_RP), in.rp + off, tmb, b);
                tma_load_1d(L.ob(os, O_RVX), in.rvx + off, tmb, b);
                tma_load_1d(L.ob(os, O_RVS), in.rvs + off, tmb, b);
                a3_rows(L.orvm(os), in.rvm, slab, s, m0 - 1, m0 + TM, nm, pitch, b);
            }
        };
        // the TMA requests come from lane 0 of warps 1 and 2 (the tap ring, the own ring): two SM
        // sub-partitions, so no warp carries all of them into the barriers
        if (tid == 32)
            for (int i = 0; i < FD && i < NI; i++) issue(i);
        if (tid == 64) issue_own(0);
        int rcur = rec_lower(IO.rec, 0, IO.n_rec, sb * nm + m, INT_MIN);  // receivers: key (s nm + m, x)
        E8 qp0, qp1, vsq;  // p rows F-1, F at the thread's cells; v_slow(s-1)
#pragma unroll 1
        for (int i = 0; i < NI; i++) {
            const int k = (gi0 + i) % FR, kp = (gi0 + i + FR - 1) % FR;
            if (tid == 32 && i + FD < NI) {
                fence_proxy_async_smem();
                issue(i + FD);
            }
            // row-uniform reciprocals of slab s = F - 1, loaded before the waits (latency off the chain)
            const int sw = F0 + i - 1 < 0 ? (in.slab ? -1 : ns - 1) : F0 + i - 1;  // v_slow(-1): row ns-1's medium (periodic) or the slab's halo row
            float rcx = 0.f, rcs = 0.f, rcm = 0.f, rch = 0.f;
            if (rm && i > 0) {
                rcs = e_rcp_at(P.rho_s, sw, m);
                rcx = e_rcp_at(P.rho_x, sw, m);
                rcm = e_rcp_at(P.rho_m, sw, m);
                rch = e_rcp_at(P.rho_m, sw, mh);
            }
            mbar_wait(&L.bar[k], (uint32_t)(((gi0 + i) / FR) & 1));
            qp0 = qp1;
            qp1 = e_ld8(L.sl(k) + (int64_t)(j + 1) * pitch + x);
            if (i > 0) {
                const int s = F0 + i - 1, kr = i - 1, os = (gk0 + kr) & 1;
                if (tid == 64 && s + 1 < se) {  // that own slot was last read before the previous barrier
                    fence_proxy_async_smem();
                    issue_own(kr + 1);
                }
                mbar_wait(&L.obar[os], (uint32_t)(((gk0 + kr) >> 1) & 1));
                const int64_t ro = (int64_t)j * pitch + x, off = (int64_t)m * pitch + x;
                // v_slow(s) from p rows s, s+1 (acoustic.py:169-170, to-half shifts (0, 1))
                E8 vsn = e_ld8(L.ob(os, O_VS) + ro);
                E8 rvs = comp ? e_ld8(L.ob(os, O_RVS) + ro) : E8{};
                f3_finish_v<V>(e_sfold<2>(c, qp0, qp0, qp1, qp1), rm, rcs, P.rho_s, sw, m, x, dt, dt2, zero_h, vsn, rvs);
                if (i > 1) {
                    const __half* pt = L.sl(kp);  // p tile of slab s: row m at index j + 1
                    // vx(s) = fl(fl(ddx p / rho_x) dt) (acoustic.py:167-168)
                    E8 vxn = e_ld8(L.ob(os, O_VX) + ro);
                    E8 rvx = comp ? e_ld8(L.ob(os, O_RVX) + ro) : E8{};
                    f3_finish_v<V>(e_xfold<2>(c, pt + (int64_t)(j + 1) * pitch, x, xl, xr, false), rm, rcx, P.rho_x, s, m,
                                   x, dt, dt2, zero_h, vxn, rvx);
                    e_st8(L.xv + ro, vxn);
                    // vm(s) rows m (and m0-1 for j == 0) from p mid rows r, r+1
                    {
                        const __half* t = pt + (int64_t)(j + 1) * pitch + x;
                        const E8 a = e_ld8(t), b = e_ld8(t + pitch);
                        E8 vmn = e_ld8(L.ovm(os) + ro + pitch);
                        E8 rvm = comp ? e_ld8(L.orvm(os) + ro + pitch) : E8{};
                        f3_finish_v<V>(e_sfold<2>(c, a, a, b, b), rm, rcm, P.rho_m, s, m, x, dt, dt2, zero_h, vmn, rvm);
                        e_st8(L.vmn + ro + pitch, vmn);
                        e_store_row(P.vm, slab, s, (int)off, vmn);
                        e_track(acc[3], vmn);
                        if (comp) {
                            e_store_row(P.rvm, slab, s, (int)off, rvm);
                            e_track(acc[7], rvm);
                        }
                    }
                    if (j == 0) {  // halo row m0-1: recomputed, not stored
                        const __half* t = pt + x;
                        const E8 a = e_ld8(t), b = e_ld8(t + pitch);
                        E8 vmh = e_ld8(L.ovm(os) + x);
                        E8 rvh = comp ? e_ld8(L.orvm(os) + x) : E8{};
                        f3_finish_v<V>(e_sfold<2>(c, a, a, b, b), rm, rch, P.rho_m, s, mh, x, dt, dt2, zero_h, vmh, rvh);
                        e_st8(L.vmn + x, vmh);
                    }
                    e_store_row(P.vx, slab, s, (int)off, vxn);
                    e_track(acc[1], vxn);
                    e_store_row(P.vs, slab, s, (int)off, vsn);
                    e_track(acc[2], vsn);
                    if (comp) {
                        e_store_row(P.rvx, slab, s, (int)off, rvx);
                        e_track(acc[5], rvx);
                        e_store_row(P.rvs, slab, s, (int)off, rvs);
                        e_track(acc[6], rvs);
                    }
                    __syncthreads();
                    // p(s): fl(fl(ddx vx + dds v_slow) + ddm vm) (acoustic.py:172-175), to-int taps
                    const E8 tx = e_xfold<2>(c, L.xv + (int64_t)j * pitch, x, xl, xr, true);
                    const E8 ts = e_sfold<2>(c, vsq, vsq, vsn, vsn);
                    const E8 m1 = e_ld8(L.vmn + ro), m2 = e_ld8(L.vmn + ro + pitch);
                    const E8 tmv = e_sfold<2>(c, m1, m1, m2, m2);
                    const bool sk = src_col && s == P.src_s && m == P.src_m;
                    const E8 pold = e_ld8(pt + (int64_t)(j + 1) * pitch + x);
                    E8 pn = pold;
                    E8 rr = comp ? e_ld8(L.ob(os, O_RP) + ro) : E8{};
                    if (bfull) {
                        const E8 bv = e_ld8(L.ob(os, O_BETA) + ro);
#pragma unroll
                        for (int h = 0; h < 4; h++)
                            a3_finish<V>(EO2::add(EO2::add(tx.q[h], ts.q[h]), tmv.q[h]), bv.q[h], P.beta.div_mode, dt,
                                         (sk && h == sj) ? sln : -1, src, pn.q[h], rr.q[h]);
                    } else if (brow) {
                        const float rc = e_rcp_at(P.beta, s, m);
#pragma unroll
                        for (int h = 0; h < 4; h++)
                            e_finish_rc<V>(EO2::add(EO2::add(tx.q[h], ts.q[h]), tmv.q[h]), rc, dt2,
                                           (sk && h == sj) ? sln : -1, srch, pn.q[h], rr.q[h]);
                    } else {
#pragma unroll
                        for (int h = 0; h < 4; h++)
                            finish<16, 16, 2>(EO2::add(EO2::add(tx.q[h], ts.q[h]), tmv.q[h]), &P.beta, s, m, x + 2 * h,
                                              dt, V, (sk && h == sj) ? sln : -1, src, pn.q[h], rr.q[h]);
                    }
                    e_store_row(P.p, slab, s, (int)off, pn);
                    e_track(acc[0], pn);
                    if (comp) {
                        e_store_row(P.rp, slab, s, (int)off, rr);
                        e_track(acc[4], rr);
                    }
                    // receiver traces of p after the step (acoustic.py:217-218)
                    rec_row(IO.rec, rcur, IO.n_rec, s * nm + m, x, IO.traces, IO.nt, n,
                            [&](int o) { return e_pick(pn, o); });
                    if (sample) {  // E = dx^3/2 [sum beta p^n p^{n+1} + sum rho v^2] (diagnostics.py:76-87)
                        double e[NCOMP] = {0.0, 0.0, 0.0, 0.0, 0.0};  // this (tile, slab) unit's share
                        const E8 vxo = e_ld8(L.xv + ro);
#pragma unroll
                        for (int q = 0; q < ECPT; q++) {
                            const int xi = x + q;
                            auto f = [&](const E8& a) { return (double)__half2float(a.q[q >> 1].e[q & 1]); };
                            const double a = f(vxo), b = f(vsn), g = f(m2);
                            e[0] += p64(P.e_beta, s, m, xi) * (f(pold) * f(pn));
                            e[1] += p64(P.e_rho_x, s, m, xi) * (a * a);
                            e[2] += p64(P.e_rho_s, s, m, xi) * (b * b);
                            e[3] += p64(P.e_rho_m, s, m, xi) * (g * g);
                        }
                        // per-plane partials (decomposition-invariant energy, as hw_elastic3d_fused.cu)
                        const double a = warp_sum(((e[0] + e[1]) + e[2]) + e[3]);
                        if ((tid & 31) == 0) ered[tid >> 5] = a;
                    }
                }
                vsq = vsn;
            }
            __syncthreads();
            if (sample && tid == 0 && i > 1) {  // the unit's partial (slab F0 + i - 1), warps in order
                double a = ered[0];
                for (int w = 1; w < (int)(blockDim.x >> 5); w++) a += ered[w];
                in.eplane[(int64_t)(F0 + i - 1) * (nm / TM) + tile] = a;
            }
        }
        gi += NI;
        gk += se - sb + 1;
    }
    unsigned int mask = 0;
    mask |= e_nonfinite(acc[0]) << P.p.bit;
    mask |= e_nonfinite(acc[1]) << P.vx.bit;
    mask |= e_nonfinite(acc[2]) << P.vs.bit;
    mask |= e_nonfinite(acc[3]) << P.vm.bit;
    if (comp) {
        mask |= e_nonfinite(acc[4]) << P.rp.bit;
        mask |= e_nonfinite(acc[5]) << P.rvx.bit;
        mask |= e_nonfinite(acc[6]) << P.rvs.bit;
        mask |= e_nonfinite(acc[7]) << P.rvm.bit;
    }
    record_failure(P.ctrl, n, mask);
    if constexpr (!SAMPLE) return;
    __threadfence();
    __syncthreads();
    __shared__ unsigned int is_last;
    // (edge + interior launches of one step share the counter: nb_total CTAs in all)
    const unsigned int nbt = in.nb_total > 0 ? (unsigned int)in.nb_total : gridDim.x;
    if (tid == 0) is_last = atomicAdd(IO.counter, 1u) == nbt - 1;
    __syncthreads();
    if (!is_last) return;
    // plane totals T[s] = sum_tile partial[s][tile], tiles in order (el3_energy_from_planes, hw_api.cu)
    const int tiles_all = nm / TM;
    for (int sp = tid; sp < ns; sp += (int)blockDim.x) {
        double t = __ldcg(&in.eplane[(int64_t)sp * tiles_all]);
        for (int t2 = 1; t2 < tiles_all; t2++) t += __ldcg(&in.eplane[(int64_t)sp * tiles_all + t2]);
        in.etot[eidx * (int64_t)ns + sp] = t;
    }
    if (tid == 0) *IO.counter = 0u;
}

// ---------------------------------------------------------------- host side

bool ac3d_fused_eligible(int64_t nx, int64_t nm, int64_t ns, int64_t pitch, int order, int max_smem) {
    if (order != 2 || nx % 256 != 0 || nx > F3T * ECPT || pitch != nx || ns < 2) return false;
    const int64_t TM = F3T * ECPT / nx;
    if (nm % TM != 0 || nm < 2) return false;
    return f3_bytes(nx) <= (size_t)max_smem;
}

template <int NXC, bool SAMPLE>
static void f3_attrs(int b) {
    cudaFuncSetAttribute((void*)k_ac3d_fused<0, NXC, SAMPLE>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
    cudaFuncSetAttribute((void*)k_ac3d_fused<3, NXC, SAMPLE>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
    cudaFuncSetAttribute((void*)k_ac3d_fused<6, NXC, SAMPLE>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
}

cudaError_t ac3d_fused_prepare(int64_t nx) {
    const int b = (int)f3_bytes(nx);
    f3_attrs<0, false>(b);
    f3_attrs<0, true>(b);
    f3_attrs<512, false>(b);
    f3_attrs<512, true>(b);
    return cudaGetLastError();
}

template <int NXC, bool SAMPLE>
static void* f3_fn(int variant) {
    return variant == 0 ? (void*)k_ac3d_fused<0, NXC, SAMPLE>
                        : (variant == 3 ? (void*)k_ac3d_fused<3, NXC, SAMPLE> : (void*)k_ac3d_fused<6, NXC, SAMPLE>);
}

void launch_ac3d_fused(int variant, const AcParams& P, const Ac3In& in, const StreamIO& IO, int nblocks, int64_t n,
                       double src, int sample, int64_t eidx, cudaStream_t st) {
    const bool c512 = P.g.nx == 512 && P.g.pitch == 512;
    void* fn = c512 ? (sample ? f3_fn<512, true>(variant) : f3_fn<512, false>(variant))
                    : (sample ? f3_fn<0, true>(variant) : f3_fn<0, false>(variant));
    void* args[] = {(void*)&P, (void*)&in, (void*)&IO, (void*)&n, (void*)&src, (void*)&eidx};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nblocks);
    cfg.blockDim = dim3(F3T);
    cfg.dynamicSmemBytes = f3_bytes(P.g.nx);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelExC(&cfg, fn, args);
}

}  // namespace hw
