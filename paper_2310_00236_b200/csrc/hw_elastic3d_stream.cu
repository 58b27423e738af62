// hw_elastic3d_stream.cu — streaming phase kernels for the 3D elastic solver, binary16
// state (BASELINE config 5: 512^3, 2nd order, layered), sm_100a.
//
// The two phases of the 3D velocity-stress step (ElasticSolver._step_work, elastic.py:
// 176-238, extended to 3D as SURVEY §8 a'; identical bits to k_el_vel / k_el_stress).
// A CTA owns a tile of TM = 2048/nx mid rows x the full x width and streams it along
// the slow axis; (tile, slab) work units are split evenly over the CTAs.  Output slab s
// = front F - 2.  Shared memory is the limit with nine fields, so each slot holds:
//   * queue rows at F (to-half slow taps s-1..s+2) -- own TM rows only;
//   * "delayed" rows / tiles at F-1: to-int slow-tap queues (s-2..s+1), and one
//     iteration later, in the PREVIOUS slot, the slab-s rows whose x / mid taps are
//     needed (prefetch distance 2 with 4 slots keeps slot i-1 valid during i);
//   * rows / mid tiles (TM+4 rows, periodic wrap) at F-2 = s.
// A 2-slot own ring (one slab ahead) holds the old values and residuals of slab s.
#include <cuda_runtime.h>

#include "hw_params.h"
#include "hw_stream.cuh"
#include "hw_tma.cuh"
#include "../../include/halfwave_b200.h"

namespace hw {

constexpr int QR = 4;     // tap ring slots
constexpr int QD = 2;     // prefetch distance (slot i-1 stays valid during i)
constexpr int E3T = 256;  // threads per CTA; TM = E3T * ECPT / nx

struct E3Layout {
    uint64_t* bar;
    uint64_t* obar;
    __half* ring;
    __half* own;
    int64_t slot, tm;
    int nown;
    __device__ __forceinline__ E3Layout(unsigned char* smem, int64_t slot_rows, int TM, int64_t pitch, int own_rows)
        : bar(reinterpret_cast<uint64_t*>(smem)), obar(reinterpret_cast<uint64_t*>(smem + 64)),
          ring(reinterpret_cast<__half*>(smem + 128)), own(ring + QR * slot_rows * pitch),
          slot(slot_rows * pitch), tm((int64_t)TM * pitch), nown(own_rows) {}
    __device__ __forceinline__ __half* sl(int k) const { return ring + (int64_t)k * slot; }
    __device__ __forceinline__ __half* orow(int os, int q) const { return own + (os * nown + q) * tm; }
};

__device__ __forceinline__ void e3_init(const E3Layout& L) {
    if (threadIdx.x == 0) {
        for (int s = 0; s < QR; s++) mbar_init(&L.bar[s], 1);
        for (int s = 0; s < 2; s++) mbar_init(&L.obar[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
}

// fold of 4 consecutive rows t0 .. t0+3 of a tile (mid taps) at the thread's cells; 2nd
// order reads only the inner pair (t0 may then lie one row before the tile)
template <int ORDER>
__device__ __forceinline__ E8 e3_mfold(const __half c[4], const __half* t0, int64_t pitch) {
    const E8 b = e_ld8(t0 + pitch), d = e_ld8(t0 + 2 * pitch);
    if (ORDER == 2) return e_sfold<2>(c, b, b, d, d);
    return e_sfold<ORDER>(c, e_ld8(t0), b, d, e_ld8(t0 + 3 * pitch));
}

__device__ __forceinline__ E8 e3_add(const E8& a, const E8& b) {
    E8 r;
#pragma unroll
    for (int h = 0; h < 4; h++) r.q[h] = EO2::add(a.q[h], b.q[h]);
    return r;
}

__device__ __forceinline__ void e3_shift(E8 q[4], const E8& v) {
    q[0] = q[1];
    q[1] = q[2];
    q[2] = q[3];
    q[3] = v;
}

// ---------------------------------------------------------------- velocity phase
// slot rows: [sss(F) TM | sxs(F-1) TM | sms tile(F-1) | sxx(s) TM | sxm tile(s) | smm tile(s)], tiles of
// TM + 2H - 1 rows (H = ORDER/2): a tile read by to-int mid taps holds rows m0-H .. m0+TM+H-2 (row m
// at index j + H), one read by to-half mid taps rows m0-H+1 .. m0+TM+H-1 (row m at index j + H - 1)
template <int V, int ORDER>
__global__ void __launch_bounds__(E3T, 1) k_el3d_vel_stream(ElParams P, int64_t n, double src) {
    e_pdl_enter();
    if (halted(P.ctrl, n)) return;
    extern __shared__ __align__(128) unsigned char smem[];
    const int nx = (int)P.g.nx, nm = (int)P.g.nm, ns = (int)P.vx.rows;
    const int64_t pitch = P.g.pitch, slab = P.g.slab;
    const int TM = E3T * ECPT / nx, TPR = nx / ECPT;
    constexpr int H = ORDER / 2;
    constexpr int TH = 2 * H - 1;  // halo rows of a one-sided tile
    const E3Layout L(smem, 6 * TM + 3 * TH, TM, pitch, 6);
    const int o_sxs = TM, o_sms = 2 * TM, o_sxx = 3 * TM + TH, o_sxm = 4 * TM + TH, o_smm = 5 * TM + 2 * TH;
    const int tid = threadIdx.x, j = tid / TPR, x = (tid % TPR) * ECPT;
    constexpr bool comp = V != 0;
    constexpr int NOWN = comp ? 6 : 3;  // vx vs vm [rvx rvs rvm]
    const __half* SSS = reinterpret_cast<const __half*>(P.sss.base);
    const __half* SXS = reinterpret_cast<const __half*>(P.sxs.base);
    const __half* SMS = reinterpret_cast<const __half*>(P.sms.base);
    const __half* SXX = reinterpret_cast<const __half*>(P.sxx.base);
    const __half* SXM = reinterpret_cast<const __half*>(P.sxm.base);
    const __half* SMM = reinterpret_cast<const __half*>(P.smm.base);
    const __half* OWN[6] = {reinterpret_cast<const __half*>(P.vx.base), reinterpret_cast<const __half*>(P.vs.base),
                            reinterpret_cast<const __half*>(P.vm.base), reinterpret_cast<const __half*>(P.rvx.base),
                            reinterpret_cast<const __half*>(P.rvs.base), reinterpret_cast<const __half*>(P.rvm.base)};
    const FieldView* OF[6] = {&P.vx, &P.vs, &P.vm, &P.rvx, &P.rvs, &P.rvm};
    const uint32_t tmb = (uint32_t)(L.tm * sizeof(__half));
    e3_init(L);
    __half c[4];
#pragma unroll
    for (int q = 0; q < 4; q++) c[q] = lconst<16>(P.k, q);
    const __half dt = lconst<16>(P.k, 4);
    const int xl = x == 0 ? nx - 2 : x - 2, xr = x + ECPT >= nx ? 0 : x + ECPT;
    const bool vsrc = P.src_kind == HW_SRC_VSLOW && src != 0.0;  // warp-uniform
    const bool src_col = vsrc && P.src_x >= x && P.src_x < x + ECPT;
    const bool rm = e_rowdiv(P.rho_x) && e_rowdiv(P.rho_s) && e_rowdiv(P.rho_m);  // one reciprocal per row
    const __half2 dt2 = __half2half2(dt);
    const __half srch = __double2half(src);
    const int sj = (int)((P.src_x - x) >> 1), sln = (int)((P.src_x - x) & 1);
    __half2 acc[6];
#pragma unroll
    for (int q = 0; q < 6; q++) acc[q] = __float2half2_rn(0.f);

    const int tiles = nm / TM;
    const int64_t U = (int64_t)tiles * ns;
    int64_t u = (int64_t)blockIdx.x * U / gridDim.x;
    const int64_t u1 = (int64_t)(blockIdx.x + 1) * U / gridDim.x;
    int gi = 0, gk = 0;
    while (u < u1) {
        const int tile = (int)(u / ns), sb = (int)(u % ns);
        const int se = (int)min((int64_t)ns, sb + (u1 - u));
        u += se - sb;
        const int m0 = tile * TM, m = m0 + j;
        const int F0 = sb - 2, NI = se - sb + 4;
        const int gi0 = gi, gk0 = gk;
        auto issue = [&](int i) {
            const int F = F0 + i, k = (gi0 + i) % QR;
            __half* d = L.sl(k);
            const int64_t mo = (int64_t)m0 * pitch;
            mbar_arrive_expect_tx(&L.bar[k], (uint32_t)((6 * TM + 3 * TH) * pitch * sizeof(__half)));
            tma_load_1d(d, SSS + e_row(F) * slab + mo, tmb, &L.bar[k]);
            tma_load_1d(d + o_sxs * pitch, SXS + e_row(F - 1) * slab + mo, tmb, &L.bar[k]);
            a3_rows(d + o_sms * pitch, SMS, slab, e_row(F - 1), m0 - H, m0 + TM + H - 1, nm, pitch, &L.bar[k]);
            tma_load_1d(d + o_sxx * pitch, SXX + e_row(F - 2) * slab + mo, tmb, &L.bar[k]);
            a3_rows(d + o_sxm * pitch, SXM, slab, e_row(F - 2), m0 - H, m0 + TM + H - 1, nm, pitch, &L.bar[k]);
            a3_rows(d + o_smm * pitch, SMM, slab, e_row(F - 2), m0 - H + 1, m0 + TM + H, nm, pitch, &L.bar[k]);
        };
        auto issue_own = [&](int kk) {
            const int os = (gk0 + kk) & 1;
            const int64_t off = (int64_t)(sb + kk) * slab + (int64_t)m0 * pitch;
            mbar_arrive_expect_tx(&L.obar[os], NOWN * tmb);
#pragma unroll
            for (int q = 0; q < NOWN; q++) tma_load_1d(L.orow(os, q), OWN[q] + off, tmb, &L.obar[os]);
        };
        if (tid == 0) {
            for (int i = 0; i < QD && i < NI; i++) issue(i);
            issue_own(0);
        }
        E8 qss[4], qxs[4], qms[4];  // sss rows s-1..s+2; sxs, sms rows s-2..s+1 ([3] newest)
#pragma unroll 1
        for (int i = 0; i < NI; i++) {
            const int k = (gi0 + i) % QR, kp = (gi0 + i + QR - 1) % QR;
            if (tid == 0 && i + QD < NI) {
                fence_proxy_async_smem();
                issue(i + QD);
            }
            const int s = F0 + i - 2;
            float rcx = 0.f, rcs = 0.f, rcm = 0.f;  // row reciprocals, loaded before the waits
            if (rm && s >= sb) {
                rcx = e_rcp_at(P.rho_x, s, m);
                rcs = e_rcp_at(P.rho_s, s, m);
                rcm = e_rcp_at(P.rho_m, s, m);
            }
            mbar_wait(&L.bar[k], (uint32_t)(((gi0 + i) / QR) & 1));
            const __half* d = L.sl(k);
            const __half* pd = L.sl(kp);  // slab F-2 = s rows / tiles of the delayed streams
            const int64_t jr = (int64_t)j * pitch;
            e3_shift(qss, e_ld8(d + jr + x));
            e3_shift(qxs, e_ld8(d + o_sxs * pitch + jr + x));
            e3_shift(qms, e_ld8(d + o_sms * pitch + jr + H * pitch + x));
            if (s >= sb) {
                const int kr = s - sb, os = (gk0 + kr) & 1;
                if (tid == 0 && s + 1 < se) {
                    fence_proxy_async_smem();
                    issue_own(kr + 1);
                }
                mbar_wait(&L.obar[os], (uint32_t)(((gk0 + kr) >> 1) & 1));
                const int64_t ro = jr + x, off = (int64_t)m * pitch + x;
                const int64_t goff = (int64_t)s * slab + off;
                const bool inner = s >= G && s < ns - G;  // stores that never touch a ghost slab
                E8 v[3], rr[3];
#pragma unroll
                for (int q = 0; q < 3; q++) {
                    v[q] = e_ld8(L.orow(os, q) + ro);
                    rr[q] = comp ? e_ld8(L.orow(os, 3 + q) + ro) : E8{};
                }
                // vx: fl(fl(ddx sxx + dds sxs) + ddm sxm) (elastic.py:191-194 + mid term)
                E8 a = e_xfold<ORDER>(c, d + o_sxx * pitch + jr, x, xl, xr, false);
                a = e3_add(a, e_sfold<ORDER>(c, qxs[0], qxs[1], qxs[2], qxs[3]));
                a = e3_add(a, e3_mfold<ORDER>(c, d + o_sxm * pitch + jr + (H - 2) * pitch + x, pitch));
                if (rm) {
#pragma unroll
                    for (int h = 0; h < 4; h++) e_finish_rc<V>(a.q[h], rcx, dt2, -1, srch, v[0].q[h], rr[0].q[h]);
                } else {
#pragma unroll
                    for (int h = 0; h < 4; h++)
                        finish<16, 16, 2>(a.q[h], &P.rho_x, s, m, x + 2 * h, dt, V, -1, 0.0, v[0].q[h], rr[0].q[h]);
                }
                // v_slow: fl(fl(ddx sxs + dds sss) + ddm sms) (+ src) (elastic.py:196-205)
                a = e_xfold<ORDER>(c, pd + o_sxs * pitch + jr, x, xl, xr, true);
                a = e3_add(a, e_sfold<ORDER>(c, qss[0], qss[1], qss[2], qss[3]));
                a = e3_add(a, e3_mfold<ORDER>(c, pd + o_sms * pitch + jr + (H - 2) * pitch + x, pitch));
                const bool sk = src_col && s == P.src_s && m == P.src_m;
                if (rm) {
                    if (vsrc && s == P.src_s && m == P.src_m) e2_add_src(a.q, sk, sj, sln, srch);  // (m: warp-uniform)
#pragma unroll
                    for (int h = 0; h < 4; h++) e_finish_rc<V>(a.q[h], rcs, dt2, -1, srch, v[1].q[h], rr[1].q[h]);
                } else {
#pragma unroll
                    for (int h = 0; h < 4; h++)
                        finish<16, 16, 2>(a.q[h], &P.rho_s, s, m, x + 2 * h, dt, V, (sk && h == sj) ? sln : -1, src,
                                          v[1].q[h], rr[1].q[h]);
                }
                // v_mid: fl(fl(ddx sxm + dds sms) + ddm smm)
                a = e_xfold<ORDER>(c, d + o_sxm * pitch + jr + H * pitch, x, xl, xr, true);
                a = e3_add(a, e_sfold<ORDER>(c, qms[0], qms[1], qms[2], qms[3]));
                a = e3_add(a, e3_mfold<ORDER>(c, d + o_smm * pitch + jr + (H - 2) * pitch + x, pitch));  // to-half tile
                if (rm) {
#pragma unroll
                    for (int h = 0; h < 4; h++) e_finish_rc<V>(a.q[h], rcm, dt2, -1, srch, v[2].q[h], rr[2].q[h]);
                } else {
#pragma unroll
                    for (int h = 0; h < 4; h++)
                        finish<16, 16, 2>(a.q[h], &P.rho_m, s, m, x + 2 * h, dt, V, -1, 0.0, v[2].q[h], rr[2].q[h]);
                }
#pragma unroll
                for (int q = 0; q < 3; q++) {
                    e2_store(inner, *OF[q], goff, slab, s, (int)off, v[q]);
                    e_track(acc[q], v[q]);
                    if (comp) e2_store(inner, *OF[3 + q], goff, slab, s, (int)off, rr[q]);
                }
            }
            __syncthreads();
        }
        gi += NI;
        gk += se - sb;
    }
    unsigned int mask = 0;
#pragma unroll
    for (int q = 0; q < 3; q++) {
        mask |= e_nonfinite(acc[q]) << OF[q]->bit;  // (residuals: see k_el2d_fused)
    }
    record_failure(P.ctrl, n, mask);
}

// ---------------------------------------------------------------- stress phase
// slot rows: [vx(F) TM | vm(F) TM | vs tile(F-1) | vx tile(s) | vm tile(s)] (vs, vx: to-half tiles; vm: to-int)
// SAMPLE: energy sample step (separate instantiation: the energy code stays out of the loop
// body -- instruction cache -- and the register budget of the other steps)
template <int V, int ORDER, bool SAMPLE>
__global__ void __launch_bounds__(E3T, 1)
    k_el3d_stress_stream(ElParams P, StreamIO IO, int64_t n, double src, int64_t eidx) {
    constexpr bool sample = SAMPLE;
    e_pdl_enter();
    if (halted(P.ctrl, n)) return;
    extern __shared__ __align__(128) unsigned char smem[];
    const int nx = (int)P.g.nx, nm = (int)P.g.nm, ns = (int)P.sxx.rows;
    const int64_t pitch = P.g.pitch, slab = P.g.slab;
    const int TM = E3T * ECPT / nx, TPR = nx / ECPT;
    constexpr int H = ORDER / 2;
    constexpr int TH = 2 * H - 1;  // halo rows of a one-sided tile
    const E3Layout L(smem, 5 * TM + 3 * TH, TM, pitch, 12);
    const int o_vm = TM, o_vs = 2 * TM, o_vxt = 3 * TM + TH, o_vmt = 4 * TM + 2 * TH;
    const int tid = threadIdx.x, j = tid / TPR, x = (tid % TPR) * ECPT;
    constexpr bool comp = V != 0;
    constexpr int NOWN = comp ? 12 : 6;  // sxx sss smm sxs sxm sms [residuals]
    const __half* VX = reinterpret_cast<const __half*>(P.vx.base);
    const __half* VS = reinterpret_cast<const __half*>(P.vs.base);
    const __half* VM = reinterpret_cast<const __half*>(P.vm.base);
    const FieldView* OF[12] = {&P.sxx, &P.sss, &P.smm, &P.sxs, &P.sxm, &P.sms,
                               &P.rsxx, &P.rsss, &P.rsmm, &P.rsxs, &P.rsxm, &P.rsms};
    const uint32_t tmb = (uint32_t)(L.tm * sizeof(__half));
    e3_init(L);
    __half c[4];
#pragma unroll
    for (int q = 0; q < 4; q++) c[q] = lconst<16>(P.k, q);
    const __half dt = lconst<16>(P.k, 4);
    const int xl = x == 0 ? nx - 2 : x - 2, xr = x + ECPT >= nx ? 0 : x + ECPT;
    const bool ssrc = P.src_kind == HW_SRC_EXPLOSIVE && src != 0.0;  // warp-uniform
    const bool src_col = ssrc && P.src_x >= x && P.src_x < x + ECPT;
    const __half2 dt2 = __half2half2(dt);
    const __half srch = __double2half(src);
    const bool mrow = P.stiff.sx == 0 && P.lam.sx == 0 && P.mu_n.sx == 0;
    const int sj = (int)((P.src_x - x) >> 1), sln = (int)((P.src_x - x) & 1);
    // energy planes constant within a slab (layered along the slow axis): per-slab sums
    const bool erow = ((P.e_rho_x.sx | P.e_rho_s.sx | P.e_rho_m.sx | P.e_lam.sx | P.e_mu.sx | P.e_mu_n.sx) |
                       (P.e_rho_x.sm | P.e_rho_s.sm | P.e_rho_m.sm | P.e_lam.sm | P.e_mu.sm | P.e_mu_n.sm)) == 0;
    __half2 acc[12];
#pragma unroll
    for (int q = 0; q < 12; q++) acc[q] = __float2half2_rn(0.f);
    double e[NCOMP] = {0.0, 0.0, 0.0, 0.0, 0.0};

    const int tiles = nm / TM;
    const int64_t U = (int64_t)tiles * ns;
    int64_t u = (int64_t)blockIdx.x * U / gridDim.x;
    const int64_t u1 = (int64_t)(blockIdx.x + 1) * U / gridDim.x;
    int gi = 0, gk = 0;
    while (u < u1) {
        const int tile = (int)(u / ns), sb = (int)(u % ns);
        const int se = (int)min((int64_t)ns, sb + (u1 - u));
        u += se - sb;
        const int m0 = tile * TM, m = m0 + j;
        const int F0 = sb - 2, NI = se - sb + 4;
        const int gi0 = gi, gk0 = gk;
        auto issue = [&](int i) {
            const int F = F0 + i, k = (gi0 + i) % QR;
            __half* d = L.sl(k);
            const int64_t mo = (int64_t)m0 * pitch;
            mbar_arrive_expect_tx(&L.bar[k], (uint32_t)((5 * TM + 3 * TH) * pitch * sizeof(__half)));
            tma_load_1d(d, VX + e_row(F) * slab + mo, tmb, &L.bar[k]);
            tma_load_1d(d + o_vm * pitch, VM + e_row(F) * slab + mo, tmb, &L.bar[k]);
            a3_rows(d + o_vs * pitch, VS, slab, e_row(F - 1), m0 - H + 1, m0 + TM + H, nm, pitch, &L.bar[k]);
            a3_rows(d + o_vxt * pitch, VX, slab, e_row(F - 2), m0 - H + 1, m0 + TM + H, nm, pitch, &L.bar[k]);
            a3_rows(d + o_vmt * pitch, VM, slab, e_row(F - 2), m0 - H, m0 + TM + H - 1, nm, pitch, &L.bar[k]);
        };
        auto issue_own = [&](int kk) {
            const int os = (gk0 + kk) & 1;
            const int64_t off = (int64_t)(sb + kk) * slab + (int64_t)m0 * pitch;
            mbar_arrive_expect_tx(&L.obar[os], NOWN * tmb);
            for (int q = 0; q < NOWN; q++)
                tma_load_1d(L.orow(os, q), reinterpret_cast<const __half*>(OF[q]->base) + off, tmb, &L.obar[os]);
        };
        if (tid == 0) {
            for (int i = 0; i < QD && i < NI; i++) issue(i);
            issue_own(0);
        }
        E8 qvx[4], qvm[4], qvs[4];  // vx, vm rows s-1..s+2; vs rows s-2..s+1 ([3] newest)
#pragma unroll 1
        for (int i = 0; i < NI; i++) {
            const int k = (gi0 + i) % QR, kp = (gi0 + i + QR - 1) % QR;
            if (tid == 0 && i + QD < NI) {
                fence_proxy_async_smem();
                issue(i + QD);
            }
            mbar_wait(&L.bar[k], (uint32_t)(((gi0 + i) / QR) & 1));
            const __half* d = L.sl(k);
            const __half* pd = L.sl(kp);  // vs tile at slab s
            const int64_t jr = (int64_t)j * pitch;
            e3_shift(qvx, e_ld8(d + jr + x));
            e3_shift(qvm, e_ld8(d + o_vm * pitch + jr + x));
            e3_shift(qvs, e_ld8(d + o_vs * pitch + jr + (H - 1) * pitch + x));  // to-half tile: row m at j + H - 1
            const int s = F0 + i - 2;
            if (s >= sb) {
                const int kr = s - sb, os = (gk0 + kr) & 1;
                if (tid == 0 && s + 1 < se) {
                    fence_proxy_async_smem();
                    issue_own(kr + 1);
                }
                mbar_wait(&L.obar[os], (uint32_t)(((gk0 + kr) >> 1) & 1));
                const int64_t ro = jr + x, off = (int64_t)m * pitch + x;
                const int64_t goff = (int64_t)s * slab + off;
                const bool inner = s >= G && s < ns - G;  // stores that never touch a ghost slab
                // tile row pointers at row m - 2 (row m at index j + H; 2nd order never reads m - 2)
                const __half* vxt = d + o_vxt * pitch + jr + (H - 3) * pitch;  // (to-half tile)
                const __half* vmt = d + o_vmt * pitch + jr + (H - 2) * pitch;  // (to-int tile)
                const __half* vst = pd + o_vs * pitch + jr + (H - 3) * pitch;  // (to-half tile)
                // normal stresses from dvx, dvs, dvm (to-int taps)
                const E8 dvx = e_xfold<ORDER>(c, vxt + 2 * pitch, x, xl, xr, true);
                const E8 dvs = e_sfold<ORDER>(c, qvs[0], qvs[1], qvs[2], qvs[3]);
                const E8 dvm = e3_mfold<ORDER>(c, vmt + x, pitch);
                E8 old[6], nw[6], rr[6];
#pragma unroll
                for (int q = 0; q < 6; q++) {
                    old[q] = e_ld8(L.orow(os, q) + ro);
                    nw[q] = old[q];
                    rr[q] = comp ? e_ld8(L.orow(os, 6 + q) + ro) : E8{};
                }
                const bool sk = src_col && s == P.src_s && m == P.src_m;
                EH2 stiff_r, lam_r, mu_r;  // moduli constant along x: one load per row
                if (mrow) {
                    stiff_r = e_val_at(P.stiff, s, m);
                    lam_r = e_val_at(P.lam, s, m);
                    mu_r = e_val_at(P.mu_n, s, m);
                }
                EH2 a0[4], a1[4], a2[4];
#pragma unroll
                for (int h = 0; h < 4; h++) {
                    const EH2 stiff = mrow ? stiff_r : pload<16, 2>(P.stiff, s, m, x + 2 * h);
                    const EH2 lam = mrow ? lam_r : pload<16, 2>(P.lam, s, m, x + 2 * h);
                    // sxx: fl(fl(fl(stiff dvx) + fl(lam dvs)) + fl(lam dvm)); s_slow / s_mid likewise
                    a0[h] = EO2::add(EO2::add(EO2::mul(stiff, dvx.q[h]), EO2::mul(lam, dvs.q[h])), EO2::mul(lam, dvm.q[h]));
                    a1[h] = EO2::add(EO2::add(EO2::mul(lam, dvx.q[h]), EO2::mul(stiff, dvs.q[h])), EO2::mul(lam, dvm.q[h]));
                    a2[h] = EO2::add(EO2::add(EO2::mul(lam, dvx.q[h]), EO2::mul(lam, dvs.q[h])), EO2::mul(stiff, dvm.q[h]));
                }
                if (ssrc && s == P.src_s && m == P.src_m) {  // explosive source into the normal stresses
                    e2_add_src(a0, sk, sj, sln, srch);
                    e2_add_src(a1, sk, sj, sln, srch);
                    e2_add_src(a2, sk, sj, sln, srch);
                }
#pragma unroll
                for (int h = 0; h < 4; h++) {
                    e2_finish_nd<V>(a0[h], dt2, -1, srch, nw[0].q[h], rr[0].q[h]);
                    e2_finish_nd<V>(a1[h], dt2, -1, srch, nw[1].q[h], rr[1].q[h]);
                    e2_finish_nd<V>(a2[h], dt2, -1, srch, nw[2].q[h], rr[2].q[h]);
                }
                // shear: fl(mu fl(dd_a v_b + dd_b v_a)) (elastic.py:232-238 per plane), to-half taps
                const E8 sxs_a = e_sfold<ORDER>(c, qvx[0], qvx[1], qvx[2], qvx[3]);
                const E8 sxs_b = e_xfold<ORDER>(c, vst + 2 * pitch, x, xl, xr, false);
                const E8 sxm_a = e3_mfold<ORDER>(c, vxt + pitch + x, pitch);
                const E8 sxm_b = e_xfold<ORDER>(c, vmt + 2 * pitch, x, xl, xr, false);
                const E8 sms_a = e_sfold<ORDER>(c, qvm[0], qvm[1], qvm[2], qvm[3]);
                const E8 sms_b = e3_mfold<ORDER>(c, vst + pitch + x, pitch);
#pragma unroll
                for (int h = 0; h < 4; h++) {
                    const EH2 mu = mrow ? mu_r : pload<16, 2>(P.mu_n, s, m, x + 2 * h);
                    e2_finish_nd<V>(EO2::mul(mu, EO2::add(sxs_a.q[h], sxs_b.q[h])), dt2, -1, srch, nw[3].q[h], rr[3].q[h]);
                    e2_finish_nd<V>(EO2::mul(mu, EO2::add(sxm_a.q[h], sxm_b.q[h])), dt2, -1, srch, nw[4].q[h], rr[4].q[h]);
                    e2_finish_nd<V>(EO2::mul(mu, EO2::add(sms_a.q[h], sms_b.q[h])), dt2, -1, srch, nw[5].q[h], rr[5].q[h]);
                }
#pragma unroll
                for (int q = 0; q < 6; q++) {
                    e2_store(inner, *OF[q], goff, slab, s, (int)off, nw[q]);
                    e_track(acc[q], nw[q]);
                    if (comp) e2_store(inner, *OF[6 + q], goff, slab, s, (int)off, rr[q]);
                }
                if (sample) {  // diagnostics.py:100-162, 3D compliance form (k_el_stress)
                    const E8 vxo = e_ld8(vxt + 2 * pitch + x), vmo = e_ld8(vmt + 2 * pitch + x);
                    const E8 vso = e_ld8(vst + 2 * pitch + x);
                    if (erow) {
                        double skx = 0.0, skm = 0.0, sks = 0.0, sx1 = 0.0, sdot = 0.0, str = 0.0, ssh = 0.0;
#pragma unroll
                        for (int q = 0; q < ECPT; q++) {
                            auto f = [&](const E8& a) { return (double)__half2float(a.q[q >> 1].e[q & 1]); };
                            const double a = f(vxo), b = f(vmo), g = f(vso);
                            skx += a * a;
                            skm += b * b;
                            sks += g * g;
                            const double xn = f(old[0]), x1 = f(nw[0]), sn = f(old[1]), s1 = f(nw[1]);
                            const double mn = f(old[2]), m1 = f(nw[2]);
                            sx1 += xn * x1;
                            sdot += xn * x1 + sn * s1 + mn * m1;
                            str += (xn + sn + mn) * (x1 + s1 + m1);
                            ssh += f(old[3]) * f(nw[3]) + f(old[4]) * f(nw[4]) + f(old[5]) * f(nw[5]);
                        }
                        e[0] += p64(P.e_rho_x, s, 0, 0) * skx;
                        e[2] += p64(P.e_rho_m, s, 0, 0) * skm;
                        e[1] += p64(P.e_rho_s, s, 0, 0) * sks;
                        const double lamd = p64(P.e_lam, s, 0, 0), mu = p64(P.e_mu, s, 0, 0);
                        if (mu == 0.0) e[3] += sx1 / (lamd + mu);
                        else e[3] += sdot / (2.0 * mu) - lamd * str / (2.0 * mu * (3.0 * lamd + 2.0 * mu));
                        const double mun = p64(P.e_mu_n, s, 0, 0);
                        e[4] += mun > 0.0 ? ssh / mun : 0.0;
                    } else {
#pragma unroll
                        for (int q = 0; q < ECPT; q++) {
                            auto f = [&](const E8& a) { return (double)__half2float(a.q[q >> 1].e[q & 1]); };
                            const int xi = x + q;
                            const double a = f(vxo), b = f(vmo), g = f(vso);
                            e[0] += p64(P.e_rho_x, s, m, xi) * (a * a);
                            e[2] += p64(P.e_rho_m, s, m, xi) * (b * b);
                            e[1] += p64(P.e_rho_s, s, m, xi) * (g * g);
                            const double lamd = p64(P.e_lam, s, m, xi), mu = p64(P.e_mu, s, m, xi);
                            const double xn = f(old[0]), x1 = f(nw[0]), sn = f(old[1]), s1 = f(nw[1]);
                            const double mn = f(old[2]), m1 = f(nw[2]);
                            if (mu == 0.0) {
                                e[3] += (xn * x1) / (lamd + mu);
                            } else {
                                const double dot = xn * x1 + sn * s1 + mn * m1;
                                e[3] += dot / (2.0 * mu) -
                                        lamd * (xn + sn + mn) * (x1 + s1 + m1) / (2.0 * mu * (3.0 * lamd + 2.0 * mu));
                            }
                            const double mun = p64(P.e_mu_n, s, m, xi);
                            for (int w = 3; w < 6; w++) e[4] += mun > 0.0 ? (f(old[w]) * f(nw[w])) / mun : 0.0;
                        }
                    }
                }
            }
            __syncthreads();
        }
        gi += NI;
        gk += se - sb;
    }
    unsigned int mask = 0;
#pragma unroll
    for (int q = 0; q < 6; q++) {
        mask |= e_nonfinite(acc[q]) << OF[q]->bit;  // (residuals: see k_el2d_fused)
    }
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

static size_t e3_vel_bytes(int64_t nx, int order) {
    const int64_t TM = E3T * ECPT / nx, H = order / 2;
    return 128 + ((size_t)QR * (6 * TM + 3 * (2 * H - 1)) + 2 * 6 * TM) * nx * sizeof(__half);
}
static size_t e3_stress_bytes(int64_t nx, int order) {
    const int64_t TM = E3T * ECPT / nx, H = order / 2;
    return 128 + ((size_t)QR * (5 * TM + 3 * (2 * H - 1)) + 2 * 12 * TM) * nx * sizeof(__half);
}

// (the tile halos are sized by the order: nx = 1024 fits at 2nd order -- the per-GPU slab of BASELINE
// config 5's 1024^3 / 8-GPU grid -- but not at 4th)
bool el3d_stream_eligible(int64_t nx, int64_t nm, int64_t pitch, int order, int max_smem) {
    if (nx % 256 != 0 || nx > E3T * ECPT || pitch != nx || (order != 2 && order != 4)) return false;
    const int64_t TM = E3T * ECPT / nx;
    if (nm % TM != 0) return false;
    return e3_vel_bytes(nx, order) <= (size_t)max_smem && e3_stress_bytes(nx, order) <= (size_t)max_smem;
}

template <int V, int O>
static void e3_attrs(int64_t nx) {
    cudaFuncSetAttribute((void*)k_el3d_vel_stream<V, O>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)e3_vel_bytes(nx, O));
    cudaFuncSetAttribute((void*)k_el3d_stress_stream<V, O, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)e3_stress_bytes(nx, O));
    cudaFuncSetAttribute((void*)k_el3d_stress_stream<V, O, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)e3_stress_bytes(nx, O));
}

cudaError_t el3d_stream_prepare(int64_t nx, int order) {
    if (order == 2) {
        e3_attrs<0, 2>(nx); e3_attrs<3, 2>(nx); e3_attrs<6, 2>(nx);
    } else {
        e3_attrs<0, 4>(nx); e3_attrs<3, 4>(nx); e3_attrs<6, 4>(nx);
    }
    return cudaGetLastError();
}

#define E3_DISPATCH(variant, order, CALL)                                            \
    if (order == 2) {                                                                \
        if (variant == 0) { constexpr int V_ = 0, O_ = 2; CALL; }                    \
        else if (variant == 3) { constexpr int V_ = 3, O_ = 2; CALL; }               \
        else { constexpr int V_ = 6, O_ = 2; CALL; }                                 \
    } else {                                                                         \
        if (variant == 0) { constexpr int V_ = 0, O_ = 4; CALL; }                    \
        else if (variant == 3) { constexpr int V_ = 3, O_ = 4; CALL; }               \
        else { constexpr int V_ = 6, O_ = 4; CALL; }                                 \
    }

static void e3_launch(void* fn, int nblocks, size_t bytes, cudaStream_t st, void** args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nblocks);
    cfg.blockDim = dim3(E3T);
    cfg.dynamicSmemBytes = bytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelExC(&cfg, fn, args);
}

void launch_el3d_vel_stream(int variant, int order, const ElParams& P, int nblocks, int64_t n, double src,
                            cudaStream_t st) {
    void* fn = nullptr;
    E3_DISPATCH(variant, order, (fn = (void*)k_el3d_vel_stream<V_, O_>))
    void* args[] = {(void*)&P, (void*)&n, (void*)&src};
    e3_launch(fn, nblocks, e3_vel_bytes(P.g.nx, order), st, args);
}

void launch_el3d_stress_stream(int variant, int order, const ElParams& P, const StreamIO& IO, int nblocks, int64_t n,
                               double src, int sample, int64_t eidx, cudaStream_t st) {
    void* fn = nullptr;
    if (sample) {
        E3_DISPATCH(variant, order, (fn = (void*)k_el3d_stress_stream<V_, O_, true>))
    } else {
        E3_DISPATCH(variant, order, (fn = (void*)k_el3d_stress_stream<V_, O_, false>))
    }
    void* args[] = {(void*)&P, (void*)&IO, (void*)&n, (void*)&src, (void*)&eidx};
    e3_launch(fn, nblocks, e3_stress_bytes(P.g.nx, order), st, args);
}

}  // namespace hw
