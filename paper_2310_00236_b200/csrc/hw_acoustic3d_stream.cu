// hw_acoustic3d_stream.cu — streaming phase kernels for the 3D acoustic solver,
// binary16 state (BASELINE config 3: 512^3, 2nd order, per-cell beta), sm_100a.
//
// Same two phases as AcousticSolver._step_work (acoustic.py:162-181) extended to 3D
// (the generic k_ac_vel / k_ac_pres compute identical bits with the same helpers).
// A CTA owns a tile of TM = 4096/nx mid rows x the full x width (x periodic inside the
// CTA) and streams it along the slow axis; the (tile, slab) work units are split
// evenly over the CTAs.  Per slab a 4-slot TMA ring (filled 3 slabs ahead) brings the
// slow-tap queue rows (own cells, into register queues), the x-tap rows and a mid-axis
// tile with 2 halo rows each side (periodic wrap = two bulk copies); a 2-slot own ring
// (filled one slab ahead) brings the old values, residuals and per-cell divisors.
#include <cuda_runtime.h>

#include "hw_params.h"
#include "hw_stream.cuh"
#include "hw_tma.cuh"
#include "../../include/halfwave_b200.h"

namespace hw {

constexpr int AR = 4;      // tap ring slots
constexpr int AD = 3;      // prefetch distance (every datum of iteration i sits in slot i)
constexpr int A3T = 512;   // threads per CTA; TM = A3T * ECPT / nx rows of the mid axis
constexpr int AOWN = 6;    // own-ring rows (in units of TM rows) per slot

struct A3Layout {
    uint64_t* bar;   // AR tap barriers
    uint64_t* obar;  // 2 own barriers
    __half* ring;
    __half* own;
    int64_t slot;    // elements per tap slot
    int64_t tm;      // elements per TM-row block
    __device__ __forceinline__ A3Layout(unsigned char* smem, int64_t slot_rows, int TM, int64_t pitch)
        : bar(reinterpret_cast<uint64_t*>(smem)), obar(reinterpret_cast<uint64_t*>(smem + 64)),
          ring(reinterpret_cast<__half*>(smem + 128)), own(ring + AR * slot_rows * pitch),
          slot(slot_rows * pitch), tm((int64_t)TM * pitch) {}
    __device__ __forceinline__ __half* orow(int os, int q) const { return own + (os * AOWN + q) * tm; }
};

__device__ __forceinline__ void a3_init(const A3Layout& L) {
    if (threadIdx.x == 0) {
        for (int s = 0; s < AR; s++) mbar_init(&L.bar[s], 1);
        for (int s = 0; s < 2; s++) mbar_init(&L.obar[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
}

__device__ __forceinline__ bool a3_full(const PlaneView& v) { return v.sx != 0; }

// ---------------------------------------------------------------- velocity phase
// Segment (tile m0, slabs [sb, se)): iteration i has front F = sb - 1 + i and output
// slab s = F - 2.  Slot: [p[F] own rows (TM) | p[s] tile rows m0-2 .. m0+TM+2 (TM+4)].
template <int V, int ORDER>
__global__ void __launch_bounds__(A3T, 1) k_ac3d_vel_stream(AcParams P, int64_t n) {
    e_pdl_enter();
    if (halted(P.ctrl, n)) return;
    extern __shared__ __align__(128) unsigned char smem[];
    const int nx = (int)P.g.nx, nm = (int)P.g.nm, ns = (int)P.p.rows;
    const int64_t pitch = P.g.pitch, slab = P.g.slab;
    const int TM = A3T * ECPT / nx, TPR = nx / ECPT;
    const A3Layout L(smem, 2 * TM + 4, TM, pitch);
    const int tid = threadIdx.x, j = tid / TPR, x = (tid % TPR) * ECPT;
    constexpr bool comp = V != 0;
    constexpr int NOWN = comp ? 6 : 3;  // vx vs vm [rvx rvs rvm]
    const __half* PB = reinterpret_cast<const __half*>(P.p.base);
    const __half* OWN[6] = {reinterpret_cast<const __half*>(P.vx.base), reinterpret_cast<const __half*>(P.vs.base),
                            reinterpret_cast<const __half*>(P.vm.base), reinterpret_cast<const __half*>(P.rvx.base),
                            reinterpret_cast<const __half*>(P.rvs.base), reinterpret_cast<const __half*>(P.rvm.base)};
    const uint32_t tmb = (uint32_t)(L.tm * sizeof(__half));
    a3_init(L);
    __half c[4];
#pragma unroll
    for (int q = 0; q < 4; q++) c[q] = lconst<16>(P.k, q);
    const __half dt = lconst<16>(P.k, 4);
    const int xl = x == 0 ? nx - 2 : x - 2, xr = x + ECPT >= nx ? 0 : x + ECPT;
    // divisors constant along x: one reciprocal per (slab, row) instead of a plane load per pair
    const bool rm = e_rowdiv(P.rho_x) && e_rowdiv(P.rho_s) && e_rowdiv(P.rho_m);
    const __half2 dt2 = __half2half2(dt);
    const __half zero_h = __float2half(0.f);
    __half2 acc[6];
#pragma unroll
    for (int q = 0; q < 6; q++) acc[q] = __float2half2_rn(0.f);

    const int tiles = nm / TM;
    const int64_t U = (int64_t)tiles * ns;
    int64_t u = (int64_t)blockIdx.x * U / gridDim.x;
    const int64_t u1 = (int64_t)(blockIdx.x + 1) * U / gridDim.x;
    int gi = 0, gk = 0;  // running tap / own use counters (slot and parity continue across segments)
    while (u < u1) {
        const int tile = (int)(u / ns), sb = (int)(u % ns);
        const int se = (int)min((int64_t)ns, sb + (u1 - u));
        u += se - sb;
        const int m0 = tile * TM, m = m0 + j;
        const int F0 = sb - 1, NI = se - sb + 3;
        const int gi0 = gi, gk0 = gk;
        auto issue = [&](int i) {
            const int F = F0 + i, sl = (gi0 + i) % AR;
            __half* d = L.ring + sl * L.slot;
            mbar_arrive_expect_tx(&L.bar[sl], (uint32_t)((2 * TM + 4) * pitch * sizeof(__half)));
            tma_load_1d(d, PB + e_row(F) * slab + (int64_t)m0 * pitch, tmb, &L.bar[sl]);
            a3_rows(d + L.tm, PB, slab, e_row(F - 2), m0 - 2, m0 + TM + 2, nm, pitch, &L.bar[sl]);
        };
        auto issue_own = [&](int k) {
            const int os = (gk0 + k) & 1;
            const int64_t off = (int64_t)(sb + k) * slab + (int64_t)m0 * pitch;
            mbar_arrive_expect_tx(&L.obar[os], NOWN * tmb);
#pragma unroll
            for (int q = 0; q < NOWN; q++) tma_load_1d(L.orow(os, q), OWN[q] + off, tmb, &L.obar[os]);
        };
        if (tid == 0) {
            for (int i = 0; i < AD && i < NI; i++) issue(i);
            issue_own(0);
        }
        E8 q[4];  // p rows F-3 .. F at the thread's cells ([3] newest)
#pragma unroll 1
        for (int i = 0; i < NI; i++) {
            const int sl = (gi0 + i) % AR;
            if (tid == 0 && i + AD < NI) {
                fence_proxy_async_smem();
                issue(i + AD);
            }
            mbar_wait(&L.bar[sl], (uint32_t)(((gi0 + i) / AR) & 1));
            const __half* d = L.ring + sl * L.slot;
            q[0] = q[1]; q[1] = q[2]; q[2] = q[3];
            q[3] = e_ld8(d + (int64_t)j * pitch + x);
            const int s = F0 + i - 2;
            if (s >= sb) {
                const int kr = s - sb, os = (gk0 + kr) & 1;
                if (tid == 0 && s + 1 < se) {  // own slot was last read before the previous barrier
                    fence_proxy_async_smem();
                    issue_own(kr + 1);
                }
                mbar_wait(&L.obar[os], (uint32_t)(((gk0 + kr) >> 1) & 1));
                const __half* tile_row = d + L.tm + (int64_t)(j + 2) * pitch;  // p[s][m]
                const int64_t ro = (int64_t)j * pitch + x, off = (int64_t)m * pitch + x;
                // vx = fl(fl(ddx p / rho_x) dt) (acoustic.py:167-168)
                {
                    const E8 a = e_xfold<ORDER>(c, tile_row, x, xl, xr, false);
                    E8 v = e_ld8(L.orow(os, 0) + ro);
                    E8 rr = comp ? e_ld8(L.orow(os, 3) + ro) : E8{};
                    if (rm) {
                        const float rc = e_rcp_at(P.rho_x, s, m);
#pragma unroll
                        for (int h = 0; h < 4; h++) e_finish_rc<V>(a.q[h], rc, dt2, -1, zero_h, v.q[h], rr.q[h]);
                    } else {
#pragma unroll
                        for (int h = 0; h < 4; h++)
                            finish<16, 16, 2>(a.q[h], &P.rho_x, s, m, x + 2 * h, dt, V, -1, 0.0, v.q[h], rr.q[h]);
                    }
                    e_store_row(P.vx, slab, s, (int)off, v);
                    e_track(acc[0], v);
                    if (comp) {
                        e_store_row(P.rvx, slab, s, (int)off, rr);
                        e_track(acc[3], rr);
                    }
                }
                // v_slow from p rows s-1 .. s+2 (acoustic.py:169-170)
                {
                    const E8 a = e_sfold<ORDER>(c, q[0], q[1], q[2], q[3]);
                    E8 v = e_ld8(L.orow(os, 1) + ro);
                    E8 rr = comp ? e_ld8(L.orow(os, 4) + ro) : E8{};
                    if (rm) {
                        const float rc = e_rcp_at(P.rho_s, s, m);
#pragma unroll
                        for (int h = 0; h < 4; h++) e_finish_rc<V>(a.q[h], rc, dt2, -1, zero_h, v.q[h], rr.q[h]);
                    } else {
#pragma unroll
                        for (int h = 0; h < 4; h++)
                            finish<16, 16, 2>(a.q[h], &P.rho_s, s, m, x + 2 * h, dt, V, -1, 0.0, v.q[h], rr.q[h]);
                    }
                    e_store_row(P.vs, slab, s, (int)off, v);
                    e_track(acc[1], v);
                    if (comp) {
                        e_store_row(P.rvs, slab, s, (int)off, rr);
                        e_track(acc[4], rr);
                    }
                }
                // v_mid from p mid rows m-1 .. m+2 (3D extension)
                {
                    const __half* t0 = d + L.tm + (int64_t)(j + 1) * pitch + x;
                    const E8 a = e_sfold<ORDER>(c, e_ld8(t0), e_ld8(t0 + pitch), e_ld8(t0 + 2 * pitch),
                                                e_ld8(t0 + 3 * pitch));
                    E8 v = e_ld8(L.orow(os, 2) + ro);
                    E8 rr = comp ? e_ld8(L.orow(os, 5) + ro) : E8{};
                    if (rm) {
                        const float rc = e_rcp_at(P.rho_m, s, m);
#pragma unroll
                        for (int h = 0; h < 4; h++) e_finish_rc<V>(a.q[h], rc, dt2, -1, zero_h, v.q[h], rr.q[h]);
                    } else {
#pragma unroll
                        for (int h = 0; h < 4; h++)
                            finish<16, 16, 2>(a.q[h], &P.rho_m, s, m, x + 2 * h, dt, V, -1, 0.0, v.q[h], rr.q[h]);
                    }
                    e_store_row(P.vm, slab, s, (int)off, v);
                    e_track(acc[2], v);
                    if (comp) {
                        e_store_row(P.rvm, slab, s, (int)off, rr);
                        e_track(acc[5], rr);
                    }
                }
            }
            __syncthreads();
        }
        gi += NI;
        gk += se - sb;
    }
    unsigned int mask = 0;
    mask |= e_nonfinite(acc[0]) << P.vx.bit;
    mask |= e_nonfinite(acc[1]) << P.vs.bit;
    mask |= e_nonfinite(acc[2]) << P.vm.bit;
    if (comp) {
        mask |= e_nonfinite(acc[3]) << P.rvx.bit;
        mask |= e_nonfinite(acc[4]) << P.rvs.bit;
        mask |= e_nonfinite(acc[5]) << P.rvm.bit;
    }
    record_failure(P.ctrl, n, mask);
}

// ---------------------------------------------------------------- pressure phase
// Iteration i: front F = sb - 2 + i, output slab s = F - 1.
// Slot: [v_slow[F] own rows (TM) | vx[s] rows (TM) | v_mid[s] tile rows m0-2 .. m0+TM+2].
// Own ring: p, rp and (per-cell beta) rows of slab s.
template <int V, int ORDER>
__global__ void __launch_bounds__(A3T, 1)
    k_ac3d_pres_stream(AcParams P, StreamIO IO, int64_t n, double src, int sample, int64_t eidx) {
    e_pdl_enter();
    if (halted(P.ctrl, n)) return;
    extern __shared__ __align__(128) unsigned char smem[];
    const int nx = (int)P.g.nx, nm = (int)P.g.nm, ns = (int)P.p.rows;
    const int64_t pitch = P.g.pitch, slab = P.g.slab;
    const int TM = A3T * ECPT / nx, TPR = nx / ECPT;
    const A3Layout L(smem, 3 * TM + 4, TM, pitch);
    const int tid = threadIdx.x, j = tid / TPR, x = (tid % TPR) * ECPT;
    constexpr bool comp = V != 0;
    const bool bfull = a3_full(P.beta);
    const bool brow = !bfull && e_rowdiv(P.beta);
    const __half2 dt2 = __half2half2(lconst<16>(P.k, 4));
    const __half srch = __double2half(src);
    const int NOWN = 1 + (comp ? 1 : 0) + (bfull ? 1 : 0);  // p [rp] [beta]
    const __half* VS = reinterpret_cast<const __half*>(P.vs.base);
    const __half* VX = reinterpret_cast<const __half*>(P.vx.base);
    const __half* VM = reinterpret_cast<const __half*>(P.vm.base);
    const __half* PP = reinterpret_cast<const __half*>(P.p.base);
    const __half* RP = reinterpret_cast<const __half*>(P.rp.base);
    const __half* BB = reinterpret_cast<const __half*>(P.beta.p);
    const uint32_t tmb = (uint32_t)(L.tm * sizeof(__half));
    a3_init(L);
    __half c[4];
#pragma unroll
    for (int q = 0; q < 4; q++) c[q] = lconst<16>(P.k, q);
    const __half dt = lconst<16>(P.k, 4);
    const int xl = x == 0 ? nx - 2 : x - 2, xr = x + ECPT >= nx ? 0 : x + ECPT;
    const bool src_col = P.has_src && src != 0.0 && P.src_x >= x && P.src_x < x + ECPT;
    const int sj = (int)((P.src_x - x) >> 1), sln = (int)((P.src_x - x) & 1);
    __half2 acc[2];
    acc[0] = acc[1] = __float2half2_rn(0.f);
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
        const int F0 = sb - 2, NI = se - sb + 3;
        const int gi0 = gi, gk0 = gk;
        auto issue = [&](int i) {
            const int F = F0 + i, sl = (gi0 + i) % AR;
            __half* d = L.ring + sl * L.slot;
            mbar_arrive_expect_tx(&L.bar[sl], (uint32_t)((3 * TM + 4) * pitch * sizeof(__half)));
            tma_load_1d(d, VS + e_row(F) * slab + (int64_t)m0 * pitch, tmb, &L.bar[sl]);
            tma_load_1d(d + L.tm, VX + e_row(F - 1) * slab + (int64_t)m0 * pitch, tmb, &L.bar[sl]);
            a3_rows(d + 2 * L.tm, VM, slab, e_row(F - 1), m0 - 2, m0 + TM + 2, nm, pitch, &L.bar[sl]);
        };
        auto issue_own = [&](int k) {
            const int os = (gk0 + k) & 1, s = sb + k;
            const int64_t off = (int64_t)s * slab + (int64_t)m0 * pitch;
            mbar_arrive_expect_tx(&L.obar[os], NOWN * tmb);
            tma_load_1d(L.orow(os, 0), PP + off, tmb, &L.obar[os]);
            if (comp) tma_load_1d(L.orow(os, 1), RP + off, tmb, &L.obar[os]);
            if (bfull) tma_load_1d(L.orow(os, 2), BB + s * P.beta.ss + (int64_t)m0 * P.beta.sm, tmb, &L.obar[os]);
        };
        if (tid == 0) {
            for (int i = 0; i < AD && i < NI; i++) issue(i);
            issue_own(0);
        }
        int rcur = rec_lower(IO.rec, 0, IO.n_rec, sb * nm + m, INT_MIN);  // receivers: key (s nm + m, x)
        E8 q[4];  // v_slow rows F-3 .. F ([3] newest)
#pragma unroll 1
        for (int i = 0; i < NI; i++) {
            const int sl = (gi0 + i) % AR;
            if (tid == 0 && i + AD < NI) {
                fence_proxy_async_smem();
                issue(i + AD);
            }
            mbar_wait(&L.bar[sl], (uint32_t)(((gi0 + i) / AR) & 1));
            const __half* d = L.ring + sl * L.slot;
            q[0] = q[1]; q[1] = q[2]; q[2] = q[3];
            q[3] = e_ld8(d + (int64_t)j * pitch + x);
            const int s = F0 + i - 1;
            if (s >= sb) {
                const int kr = s - sb, os = (gk0 + kr) & 1;
                if (tid == 0 && s + 1 < se) {
                    fence_proxy_async_smem();
                    issue_own(kr + 1);
                }
                mbar_wait(&L.obar[os], (uint32_t)(((gk0 + kr) >> 1) & 1));
                const int64_t ro = (int64_t)j * pitch + x, off = (int64_t)m * pitch + x;
                // divergence fl(fl(ddx vx + dds v_slow) + ddm v_mid) (acoustic.py:172-175)
                const __half* vxrow = d + L.tm + (int64_t)j * pitch;
                const E8 tx = e_xfold<ORDER>(c, vxrow, x, xl, xr, true);
                const E8 ts = e_sfold<ORDER>(c, q[0], q[1], q[2], q[3]);
                const __half* t0 = d + 2 * L.tm + (int64_t)j * pitch + x;  // v_mid rows m-2 .. m+1
                const E8 tm = e_sfold<ORDER>(c, e_ld8(t0), e_ld8(t0 + pitch), e_ld8(t0 + 2 * pitch),
                                             e_ld8(t0 + 3 * pitch));
                const bool sk = src_col && s == P.src_s && m == P.src_m;
                const E8 pold = e_ld8(L.orow(os, 0) + ro);
                E8 pn = pold;
                E8 rr = comp ? e_ld8(L.orow(os, 1) + ro) : E8{};
                if (bfull) {
                    const E8 bv = e_ld8(L.orow(os, 2) + ro);
#pragma unroll
                    for (int h = 0; h < 4; h++)
                        a3_finish<V>(EO2::add(EO2::add(tx.q[h], ts.q[h]), tm.q[h]), bv.q[h], P.beta.div_mode, dt,
                                     (sk && h == sj) ? sln : -1, src, pn.q[h], rr.q[h]);
                } else if (brow) {
                    const float rc = e_rcp_at(P.beta, s, m);
#pragma unroll
                    for (int h = 0; h < 4; h++)
                        e_finish_rc<V>(EO2::add(EO2::add(tx.q[h], ts.q[h]), tm.q[h]), rc, dt2, (sk && h == sj) ? sln : -1,
                                       srch, pn.q[h], rr.q[h]);
                } else {
#pragma unroll
                    for (int h = 0; h < 4; h++)
                        finish<16, 16, 2>(EO2::add(EO2::add(tx.q[h], ts.q[h]), tm.q[h]), &P.beta, s, m, x + 2 * h, dt,
                                          V, (sk && h == sj) ? sln : -1, src, pn.q[h], rr.q[h]);
                }
                e_store_row(P.p, slab, s, (int)off, pn);
                e_track(acc[0], pn);
                if (comp) {
                    e_store_row(P.rp, slab, s, (int)off, rr);
                    e_track(acc[1], rr);
                }
                // receiver traces of p after the step (acoustic.py:217-218)
                rec_row(IO.rec, rcur, IO.n_rec, s * nm + m, x, IO.traces, IO.nt, n, [&](int o) { return e_pick(pn, o); });
                if (sample) {  // E = dx^3/2 [sum beta p^n p^{n+1} + sum rho v^2] (diagnostics.py:76-87)
                    const E8 vxo = e_ld8(vxrow + x), vso = q[2];
                    const E8 vmo = e_ld8(t0 + 2 * pitch);
#pragma unroll
                    for (int k = 0; k < ECPT; k++) {
                        const int xi = x + k;
                        const double po = (double)__half2float(pold.q[k >> 1].e[k & 1]);
                        const double p1 = (double)__half2float(pn.q[k >> 1].e[k & 1]);
                        const double a = (double)__half2float(vxo.q[k >> 1].e[k & 1]);
                        const double b = (double)__half2float(vso.q[k >> 1].e[k & 1]);
                        const double g = (double)__half2float(vmo.q[k >> 1].e[k & 1]);
                        e[0] += p64(P.e_beta, s, m, xi) * (po * p1);
                        e[1] += p64(P.e_rho_x, s, m, xi) * (a * a);
                        e[2] += p64(P.e_rho_s, s, m, xi) * (b * b);
                        e[3] += p64(P.e_rho_m, s, m, xi) * (g * g);
                    }
                }
            }
            __syncthreads();
        }
        gi += NI;
        gk += se - sb;
    }
    unsigned int mask = 0;
    mask |= e_nonfinite(acc[0]) << P.p.bit;
    if (comp) mask |= e_nonfinite(acc[1]) << P.rp.bit;
    record_failure(P.ctrl, n, mask);
    if (!sample) return;
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

static size_t a3_vel_bytes(int64_t nx) {
    const int64_t TM = A3T * ECPT / nx;
    return 128 + ((size_t)AR * (2 * TM + 4) + 2 * AOWN * TM) * nx * sizeof(__half);
}
static size_t a3_pres_bytes(int64_t nx) {
    const int64_t TM = A3T * ECPT / nx;
    return 128 + ((size_t)AR * (3 * TM + 4) + 2 * AOWN * TM) * nx * sizeof(__half);
}

bool ac3d_stream_eligible(int64_t nx, int64_t nm, int64_t pitch, int max_smem) {
    if (nx % 256 != 0 || nx > A3T * ECPT || pitch != nx) return false;
    const int64_t TM = A3T * ECPT / nx;
    if (nm % TM != 0) return false;
    return a3_vel_bytes(nx) <= (size_t)max_smem && a3_pres_bytes(nx) <= (size_t)max_smem;
}

template <int V, int O>
static void a3_attrs(int64_t nx) {
    cudaFuncSetAttribute((void*)k_ac3d_vel_stream<V, O>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)a3_vel_bytes(nx));
    cudaFuncSetAttribute((void*)k_ac3d_pres_stream<V, O>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)a3_pres_bytes(nx));
}

cudaError_t ac3d_stream_prepare(int64_t nx) {
    a3_attrs<0, 2>(nx); a3_attrs<3, 2>(nx); a3_attrs<6, 2>(nx);
    a3_attrs<0, 4>(nx); a3_attrs<3, 4>(nx); a3_attrs<6, 4>(nx);
    return cudaGetLastError();
}

#define A3_DISPATCH(variant, order, CALL)                                            \
    if (order == 2) {                                                                \
        if (variant == 0) { constexpr int V_ = 0, O_ = 2; CALL; }                    \
        else if (variant == 3) { constexpr int V_ = 3, O_ = 2; CALL; }               \
        else { constexpr int V_ = 6, O_ = 2; CALL; }                                 \
    } else {                                                                         \
        if (variant == 0) { constexpr int V_ = 0, O_ = 4; CALL; }                    \
        else if (variant == 3) { constexpr int V_ = 3, O_ = 4; CALL; }               \
        else { constexpr int V_ = 6, O_ = 4; CALL; }                                 \
    }

static void a3_launch(void* fn, int nblocks, size_t bytes, cudaStream_t st, void** args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nblocks);
    cfg.blockDim = dim3(A3T);
    cfg.dynamicSmemBytes = bytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelExC(&cfg, fn, args);
}

void launch_ac3d_vel_stream(int variant, int order, const AcParams& P, int nblocks, int64_t n, cudaStream_t st) {
    void* fn = nullptr;
    A3_DISPATCH(variant, order, (fn = (void*)k_ac3d_vel_stream<V_, O_>))
    void* args[] = {(void*)&P, (void*)&n};
    a3_launch(fn, nblocks, a3_vel_bytes(P.g.nx), st, args);
}

void launch_ac3d_pres_stream(int variant, int order, const AcParams& P, const StreamIO& IO, int nblocks, int64_t n,
                             double src, int sample, int64_t eidx, cudaStream_t st) {
    void* fn = nullptr;
    A3_DISPATCH(variant, order, (fn = (void*)k_ac3d_pres_stream<V_, O_>))
    void* args[] = {(void*)&P, (void*)&IO, (void*)&n, (void*)&src, (void*)&sample, (void*)&eidx};
    a3_launch(fn, nblocks, a3_pres_bytes(P.g.nx), st, args);
}

}  // namespace hw
