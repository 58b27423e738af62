// hw_elastic2d_fused.cu — one-pass 2D elastic leapfrog step, binary16 state
// (BASELINE config 4: 4096^2, free surface, op6), sm_100a.
//
// Both phases of ElasticSolver._step_work (elastic.py:176-238) in ONE kernel per step,
// reading state n from buffer A and writing state n+1 to buffer B (ping-pong: no CTA
// reads a value another CTA has already advanced).  The two streaming phase kernels
// (hw_elastic2d_stream.cu) move 50 B per cell-step; this one moves the algorithmic
// 40 B plus a 6-row halo per CTA.  Every op and fold order is the one k_el_vel /
// k_el_stress (and the streaming kernels) use, so the bits are identical.
//
// CTA b owns rows [y0, y1) of every field and the full row width (x periodic inside
// the CTA).  Iteration i has front F = y0 - 3 + i:
//   phase A  vx_new[F-1] from the sxx[F-1] row (x taps) and sxy rows F-3..F;
//            vy_new[F-2] from the sxy[F-2] row (x taps) and syy rows F-3..F;
//            both also pushed into register queues (vx F-4..F-1, vy F-5..F-2) and
//            written to shared rows for their x taps;
//   barrier, then the TMA loads of the tap ring and the velocity own rows of
//            iteration i+1 are issued;
//   phase B  d/dx vy_new[F-2] (used next iteration), then the stresses of row
//            k = F-3: sxx, syy from d/dx vx_new[k] and the vy queue, sxy from the vx
//            queue and d/dx vy_new[k];
//   barrier, then the stress residual rows of iteration i+1 are issued (two barriers per row).
// Velocity rows outside [y0, y1) are recomputed redundantly (never stored).  Rows
// outside the domain: periodic -> the wrapped rows (all loads wrap); free surface ->
// the reference's image rows (stencil.py:121-144, even parity for vx / vy) built from
// queue entries: bottom images from rows already computed, top images patched in when
// their source row (1 for vx; 0, 1 for vy) is computed, before any stress uses them.
//
// Shared memory (nx = 4096: 27 rows of 8 KB): the tap ring (5 slots: sxy[F], syy[F],
// sxx[F-1]; a slot is read during iterations i .. i+3: slow taps, x taps, old values),
// one slot of velocity own rows (vx/rvx[F-1], vy/rvy[F-2]: read in phase A, refilled
// during phase B) and one of stress residual rows (rsxx/rsyy/rsxy[F-3]: read in phase B,
// refilled during phase A), three rows of vx_new (F-3..F-1) and two parity rows of
// vy_new.  Register queues hold only the new velocities (the tap rows stay in shared
// memory), which keeps the kernel inside 128 registers at 512 threads.
#include <cuda_runtime.h>

#include "hw_params.h"
#include "hw_stream.cuh"
#include "hw_tma.cuh"
#include "../../include/halfwave_b200.h"

namespace hw {

constexpr int LR = 5;  // tap ring slots
enum { L_SXS = 0, L_SSS, L_SXX, L_N };
enum { A_VX = 0, A_RVX, A_VS, A_RVS, A_N };  // velocity own rows
enum { B_RSXX = 0, B_RSSS, B_RSXS, B_N };    // stress residual rows

struct E2F {
    uint64_t* lbar;  // LR tap barriers, then the A and B barriers
    __half* lring;
    __half* arow;
    __half* brow;
    __half* vrow;  // vx_new rows (F-3..F-1, slot r % 3), then vy_new parity rows
    int64_t nx;
    __device__ __forceinline__ E2F(unsigned char* smem, int64_t n)
        : lbar(reinterpret_cast<uint64_t*>(smem)), lring(reinterpret_cast<__half*>(smem + 128)),
          arow(lring + (int64_t)LR * L_N * n), brow(arow + (int64_t)A_N * n), vrow(brow + (int64_t)B_N * n), nx(n) {}
    __device__ __forceinline__ uint64_t* abar() const { return lbar + LR; }
    __device__ __forceinline__ uint64_t* bbar() const { return lbar + LR + 1; }
    __device__ __forceinline__ __half* l(int slot, int st) const { return lring + (slot * L_N + st) * nx; }
    __device__ __forceinline__ __half* a(int st) const { return arow + st * nx; }
    __device__ __forceinline__ __half* b(int st) const { return brow + st * nx; }
    __device__ __forceinline__ __half* vx(int slot) const { return vrow + slot * nx; }
    __device__ __forceinline__ __half* vy(int par) const { return vrow + (3 + par) * nx; }
};

size_t el2d_fused_smem_bytes(int64_t nx) { return 128 + (size_t)(LR * L_N + A_N + B_N + 5) * nx * sizeof(__half); }

// 4-row register queue (named members, not an array: no local-memory indexing)
struct Q4 {
    E8 q0, q1, q2, q3;  // q3 = newest
    __device__ __forceinline__ void push(const E8& v) {
        q0 = q1;
        q1 = q2;
        q2 = q3;
        q3 = v;
    }
};

// SAMPLE: energy sample step (a separate instantiation: the fp64 accumulators and energy code
// stay out of the register budget of the other steps)
template <int V, int ORDER, bool RM, bool SAMPLE, bool FS>
__global__ void __launch_bounds__(512, 1)
    k_el2d_fused(ElParams P, El2In in, StreamIO IO, int64_t n, double src, int64_t eidx) {
    constexpr bool sample = SAMPLE;
    e_pdl_enter();
    if (halted(P.ctrl, n)) return;
    extern __shared__ __align__(128) unsigned char smem[];
    const E2F S(smem, P.g.nx);
    const int64_t pitch = P.g.slab;  // row stride (2D: nm = 1)
    const int nx = (int)P.g.nx;
    const int ri = (int)P.sxx.rows, rh = (int)P.sxs.rows;  // integer / half sub-grid rows
    const int b = blockIdx.x;
    int y0, y1, pidx = b, nb = gridDim.x;  // this CTA's rows, its energy-partial slot, CTAs of the whole step
    if (in.band == 1) {  // edge bands: launched ahead of the interior so the halo exchange overlaps it
        y0 = b == 0 ? 0 : ri - in.edge;
        y1 = b == 0 ? in.edge : ri;
        nb = in.nb_total;
    } else if (in.band == 2) {
        const int64_t nin = ri - 2 * in.edge;
        y0 = in.edge + (int)((int64_t)b * nin / gridDim.x);
        y1 = in.edge + (int)((int64_t)(b + 1) * nin / gridDim.x);
        pidx = 2 + b;
        nb = in.nb_total;
    } else {
        y0 = (int)((int64_t)b * ri / nb);
        y1 = (int)((int64_t)(b + 1) * ri / nb);
    }
    const int F0 = y0 - 3, NI = y1 - y0 + 6;
    const int tid = threadIdx.x, x = tid * ECPT;
    constexpr bool comp = V != 0;
    constexpr bool fs = FS;  // free surfaces (else periodic): a template parameter, the row logic folds away
    const uint32_t rb = (uint32_t)(nx * sizeof(__half));
    // rows outside the domain: periodic -> wrapped; free surface -> clamped (those values
    // are never used: image rows replace them); tap rows with images use the ghost slabs
    // (a slab of a decomposed domain: no wrap; clamping only at the global ends it owns)
    const bool slabm = in.slab != 0, gtop = !slabm || in.top, gbot = !slabm || in.bot;
    auto orow = [&](int r, int rows) {
        if (slabm) return fs ? ((r < 0 && gtop) ? 0 : ((r >= rows && gbot) ? rows - 1 : r)) : r;
        return fs ? (r < 0 ? 0 : (r >= rows ? rows - 1 : r)) : (r < 0 ? r + rows : (r >= rows ? r - rows : r));
    };
    auto trow = [&](int r, int rows) {  // (free surface: stay inside the G ghost slabs)
        return fs ? (int64_t)(r < -G ? -G : (r > rows + G - 1 ? rows + G - 1 : r)) : (int64_t)orow(r, rows);
    };
    // row of a TMA load: on a slab the first iterations of the top band ask for rows -4 and -5 (values never
    // used: no velocity is computed before iteration 3) -- keep the copy inside the G ghost rows
    auto lrow = [&](int r, int rows) {
        const int o = orow(r, rows);
        return (int64_t)(slabm ? (o < -G ? -G : (o > rows + G - 1 ? rows + G - 1 : o)) : o);
    };
    auto issue_l = [&](int i) {  // tap rows of iteration i (front F0 + i)
        const int F = F0 + i, ls = i % LR;
        mbar_arrive_expect_tx(&S.lbar[ls], L_N * rb);
        tma_load_1d(S.l(ls, L_SXS), in.sxs + trow(F, rh) * pitch, rb, &S.lbar[ls]);
        tma_load_1d(S.l(ls, L_SSS), in.sss + trow(F, ri) * pitch, rb, &S.lbar[ls]);
        tma_load_1d(S.l(ls, L_SXX), in.sxx + lrow(F - 1, ri) * pitch, rb, &S.lbar[ls]);
    };
    auto issue_a = [&](int i) {  // velocity own rows of iteration i
        const int F = F0 + i;
        mbar_arrive_expect_tx(S.abar(), (comp ? 4 : 2) * rb);
        tma_load_1d(S.a(A_VX), in.vx + lrow(F - 1, ri) * pitch, rb, S.abar());
        tma_load_1d(S.a(A_VS), in.vs + lrow(F - 2, rh) * pitch, rb, S.abar());
        if (comp) {
            tma_load_1d(S.a(A_RVX), in.rvx + lrow(F - 1, ri) * pitch, rb, S.abar());
            tma_load_1d(S.a(A_RVS), in.rvs + lrow(F - 2, rh) * pitch, rb, S.abar());
        }
    };
    // stress residual rows of iteration i (compensated runs; only iterations with an own
    // stress row, i >= 6, so every arming of the barrier is waited before the next one)
    auto issue_b = [&](int i) {
        const int F = F0 + i;
        mbar_arrive_expect_tx(S.bbar(), 3 * rb);
        tma_load_1d(S.b(B_RSXX), in.rsxx + lrow(F - 3, ri) * pitch, rb, S.bbar());
        tma_load_1d(S.b(B_RSSS), in.rsss + lrow(F - 3, ri) * pitch, rb, S.bbar());
        tma_load_1d(S.b(B_RSXS), in.rsxs + lrow(F - 3, rh) * pitch, rb, S.bbar());
    };
    if (tid == 0) {
        for (int q = 0; q < LR + 2; q++) mbar_init(&S.lbar[q], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0) {
        issue_l(0);
        issue_a(0);
    }

    __half c[4];
#pragma unroll
    for (int j = 0; j < 4; j++) c[j] = lconst<16>(P.k, j);
    const __half dt = lconst<16>(P.k, 4);
    const __half2 dt2 = __half2half2(dt);
    const __half srch = __double2half(src);
    const int xl = x == 0 ? nx - 2 : x - 2, xr = x + ECPT >= nx ? 0 : x + ECPT;
    const bool vsrc = in.vsrc && src != 0.0;  // warp-uniform; on a slab its row may be a halo row
    const bool ssrc = P.src_kind == HW_SRC_EXPLOSIVE && src != 0.0;  // warp-uniform
    const bool src_v = vsrc && P.src_x >= x && P.src_x < x + ECPT;
    const bool src_s = ssrc && P.src_x >= x && P.src_x < x + ECPT;
    const int sj = (int)((P.src_x - x) >> 1), sln = (int)((P.src_x - x) & 1);
    int rcur = rec_lower(IO.rec, 0, IO.n_rec, y0, INT_MIN);  // this CTA's receivers [rcur, rhi)
    const int rhi = rec_lower(IO.rec, rcur, IO.n_rec, y1, INT_MIN);
    const bool erow = (P.e_rho_x.sx | P.e_rho_s.sx | P.e_lam.sx | P.e_mu.sx | P.e_mu_n.sx) == 0;

    Q4 vxq, vyq;         // vx_new rows F-4..F-1, vy_new rows F-5..F-2
    E8 gyp;              // d/dx vy_new row F-3 (computed last iteration)
    // running max |value| per field; residuals are not tracked: a non-finite residual implies a
    // non-finite value of the same field in the same step (r = t + x non-finite makes s = u + r
    // non-finite; with r, s finite every EFT term is finite), and values precede residuals in
    // the check_finite order (stepping.py:101-105), so the reported first field is the same
    __half2 acc[5];
#pragma unroll
    for (int q = 0; q < 5; q++) acc[q] = __float2half2_rn(0.f);
    double e[NCOMP] = {0.0, 0.0, 0.0, 0.0, 0.0};

    int l0 = 0;         // tap slot of iteration i (= i % LR)
    uint32_t lpar = 0;  // its barrier parity (= (i / LR) & 1)
#pragma unroll 1
    for (int i = 0; i < NI; i++) {
        const int F = F0 + i, par = i & 1;
        const int l1 = l0 == 0 ? LR - 1 : l0 - 1, l2 = l1 == 0 ? LR - 1 : l1 - 1;  // tap slots of fronts F-1, F-2
        const int l3 = l2 == 0 ? LR - 1 : l2 - 1, ls = l0;                         // F-3, F
        const int rx = F - 1, ry = F - 2, k = F - 3;  // vx_new row, vy_new row, stress row
        const int rxw = orow(rx, ri), ryw = orow(ry, rh), kwi = orow(k, ri), kwh = orow(k, rh);  // medium rows
        // rows whose stores never touch a ghost slab (periodic wrap copies / surface images)
        const bool inner_v = rx >= G && rx < rh - G && ry >= G && ry < rh - G;
        const bool inner_k = k >= G && k < rh - G;
        const int64_t ox = (int64_t)rx * pitch + x, oy = (int64_t)ry * pitch + x, ok = (int64_t)k * pitch + x;
        // row-uniform coefficients of this iteration's rows, loaded before the waits
        float rcx = 0.f, rcs = 0.f;
        EH2 stiff_r, lam_r, mu_r;
        if (RM) {
            rcx = __ldg(P.rho_x.rcp + rxw * P.rho_x.ss);
            rcs = __ldg(P.rho_s.rcp + ryw * P.rho_s.ss);
            stiff_r = e_rowval(P.stiff, kwi);
            lam_r = e_rowval(P.lam, kwi);
            mu_r = e_rowval(P.mu_n, kwh);
        }
        mbar_wait(&S.lbar[ls], lpar);
        mbar_wait(S.abar(), (uint32_t)(i & 1));
        const bool vel = i >= 3;
        if (vel) {
            // vx_new[rx] = fl(fl(ddx sxx + dds sxy) / rho_x * dt) (elastic.py:191-194) and
            // vy_new[ry] = fl(fl(ddx sxy + dds syy) (+src) / rho_y * dt) (elastic.py:196-205),
            // computed side by side (one basic block: the two dependency chains interleave)
            E8 v = e_ld8(S.a(A_VX) + x), w = e_ld8(S.a(A_VS) + x);
            E8 rr = comp ? e_ld8(S.a(A_RVX) + x) : E8{};
            E8 rw = comp ? e_ld8(S.a(A_RVS) + x) : E8{};
            {
                const E8 ax = e_xfold<ORDER>(c, S.l(ls, L_SXX), x, xl, xr, false);
                const E8 dx = e_sfold<ORDER>(c, e_ld8(S.l(l3, L_SXS) + x), e_ld8(S.l(l2, L_SXS) + x),
                                             e_ld8(S.l(l1, L_SXS) + x), e_ld8(S.l(ls, L_SXS) + x));  // sxy F-3..F
                const E8 ay = e_xfold<ORDER>(c, S.l(l2, L_SXS), x, xl, xr, true);
                const E8 dy = e_sfold<ORDER>(c, e_ld8(S.l(l3, L_SSS) + x), e_ld8(S.l(l2, L_SSS) + x),
                                             e_ld8(S.l(l1, L_SSS) + x), e_ld8(S.l(ls, L_SSS) + x));  // syy F-3..F
                const int vrow = slabm ? ry : ryw;  // (single periodic domain: halo rows are the wrapped rows)
                const bool sk = src_v && vrow == in.vsrc_s;
                if constexpr (RM) {
                    EH2 hx[4], hy[4];
#pragma unroll
                    for (int j = 0; j < 4; j++) {
                        hx[j] = EO2::add(ax.q[j], dx.q[j]);
                        hy[j] = EO2::add(ay.q[j], dy.q[j]);
                    }
                    if (vsrc && vrow == in.vsrc_s) e2_add_src(hy, sk, sj, sln, srch);
#pragma unroll
                    for (int j = 0; j < 4; j++) {
                        e_finish_rc<V>(hx[j], rcx, dt2, -1, srch, v.q[j], rr.q[j]);
                        e_finish_rc<V>(hy[j], rcs, dt2, -1, srch, w.q[j], rw.q[j]);
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 4; j++) {
                        finish<16, 16, 2>(EO2::add(ax.q[j], dx.q[j]), &P.rho_x, rxw, 0, x + 2 * j, dt, V, -1, 0.0,
                                          v.q[j], rr.q[j]);
                        finish<16, 16, 2>(EO2::add(ay.q[j], dy.q[j]), &P.rho_s, ryw, 0, x + 2 * j, dt, V,
                                          (sk && j == sj) ? sln : -1, src, w.q[j], rw.q[j]);
                    }
                }
            }
            if (fs && gbot && rx >= ri) {  // bottom images: rows ri-2, ri-3 (pre-push)
                if (rx == ri) v = vxq.q2;
                else v = vxq.q0;
            }
            if (fs && gbot && ry >= rh) {  // bottom images: rows rh-1, rh-2 (pre-push)
                if (ry == rh) w = vyq.q3;
                else w = vyq.q1;
            }
            e_st8(S.vx((rx + 3) % 3) + x, v);  // rx >= -1
            e_st8(S.vy(par) + x, w);
            if (rx >= y0 && rx < y1 && rx < ri) {
                e2_store(inner_v, P.vx, ox, pitch, rx, x, v);
                e_track(acc[0], v);
                if (comp) e2_store(inner_v, P.rvx, ox, pitch, rx, x, rr);
            }
            if (ry >= y0 && ry < y1 && ry < rh) {
                e2_store(inner_v, P.vs, oy, pitch, ry, x, w);
                e_track(acc[1], w);
                if (comp) e2_store(inner_v, P.rvs, oy, pitch, ry, x, rw);
                // receiver traces of vy after the step (elastic.py:283-284)
                rec_row(IO.rec, rcur, rhi, ry, x, IO.traces, IO.nt, n, [&](int o) { return e_pick(w, o); });
            }
            vxq.push(v);
            vyq.push(w);
            if (fs && gtop && rx == 1) vxq.q1 = vxq.q3;  // top images: vx row -1 = row 1
            if (fs && gtop && ry == 0) vyq.q2 = vyq.q3;  //             vy row -1 = row 0
            if (fs && gtop && ry == 1) vyq.q0 = vyq.q3;  //             vy row -2 = row 1
        }
        __syncthreads();  // vx / vy rows visible; every read of tap slot (i+1) % LR and of the A rows is done
        if (tid == 0 && i + 1 < NI) {
            fence_proxy_async_smem();
            issue_l(i + 1);
            issue_a(i + 1);
        }
        const E8 gy = vel ? e_xfold<ORDER>(c, S.vy(par), x, xl, xr, false) : E8{};  // d/dx vy_new[ry] (to-half)
        const bool own_k = k >= y0 && k < y1;
        if (comp && own_k) mbar_wait(S.bbar(), (uint32_t)(i & 1));
        if (own_k) {  // stresses of row k (k < ri always; sxy only for k < rh)
            const int sg = (int)P.sxx.row0 + k;
            const bool surf = fs && (sg == 0 || sg == (int)P.sxx.nglob - 1);
            const bool sk = src_s && k == P.src_s;
            const E8 dvs = e_sfold<ORDER>(c, vyq.q0, vyq.q1, vyq.q2, vyq.q3);      // vy rows k-2..k+1 (to-int)
            const E8 dvx = e_xfold<ORDER>(c, S.vx((k + 3) % 3), x, xl, xr, true);  // d/dx vx_new[k] (to-int)
            const E8 dvxy = e_sfold<ORDER>(c, vxq.q0, vxq.q1, vxq.q2, vxq.q3);     // vx rows k-1..k+2 (to-half)
            const E8 sxx_old = e_ld8(S.l(l2, L_SXX) + x);  // sxx[F-3], loaded at i-2
            const E8 sss_old = e_ld8(S.l(l3, L_SSS) + x);  // syy[F-3]
            const E8 old = e_ld8(S.l(l3, L_SXS) + x);      // sxy[F-3]
            E8 sxx = sxx_old, sss = sss_old, s = old;
            E8 rsxx = comp ? e_ld8(S.b(B_RSXX) + x) : E8{};
            E8 rsss = comp ? e_ld8(S.b(B_RSSS) + x) : E8{};
            E8 rs = comp ? e_ld8(S.b(B_RSXS) + x) : E8{};
            EH2 a1[4], a2[4];
            if (!surf) {  // sxx, syy (elastic.py:210-214)
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const EH2 stiff = RM ? stiff_r : pload<16, 2>(P.stiff, k, 0, x + 2 * j);
                    const EH2 lam = RM ? lam_r : pload<16, 2>(P.lam, k, 0, x + 2 * j);
                    a1[j] = EO2::add(EO2::mul(stiff, dvx.q[j]), EO2::mul(lam, dvs.q[j]));
                    a2[j] = EO2::add(EO2::mul(lam, dvx.q[j]), EO2::mul(stiff, dvs.q[j]));
                }
            } else {  // plane-stress surface row; syy takes a zero increment (elastic.py:215-230)
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    a1[j] = EO2::mul(pload<16, 2>(P.ep, sg == 0 ? 0 : 1, 0, x + 2 * j), dvx.q[j]);
                    a2[j] = vsplat<16, 2>(lane<16>::zero());
                }
            }
            if (ssrc && k == P.src_s) {  // explosive source into both normal stresses
                e2_add_src(a1, sk, sj, sln, srch);
                e2_add_src(a2, sk, sj, sln, srch);
            }
#pragma unroll
            for (int j = 0; j < 4; j++) {
                e2_finish_nd<V>(a1[j], dt2, -1, srch, sxx.q[j], rsxx.q[j]);
                e2_finish_nd<V>(a2[j], dt2, -1, srch, sss.q[j], rsss.q[j]);
                // sxy = fl(mu fl(dds vx + ddx vy)) (elastic.py:232-238)
                const EH2 mu = RM ? mu_r : pload<16, 2>(P.mu_n, kwh, 0, x + 2 * j);
                e2_finish_nd<V>(EO2::mul(mu, EO2::add(dvxy.q[j], gyp.q[j])), dt2, -1, srch, s.q[j], rs.q[j]);
            }
            e2_store(inner_k, P.sxx, ok, pitch, k, x, sxx);
            e2_store(inner_k, P.sss, ok, pitch, k, x, sss);
            e_track(acc[2], sxx);
            e_track(acc[3], sss);
            if (comp) {
                e2_store(inner_k, P.rsxx, ok, pitch, k, x, rsxx);
                e2_store(inner_k, P.rsss, ok, pitch, k, x, rsss);
            }
            if (k < rh) {
                e2_store(inner_k, P.sxs, ok, pitch, k, x, s);
                e_track(acc[4], s);
                if (comp) e2_store(inner_k, P.rsxs, ok, pitch, k, x, rs);
            }
            {
                if (sample) {  // kinetic x + strain energy at this integer row (diagnostics.py:100-162)
                    const E8& vxr = vxq.q1;  // vx_new[k]
                    const double w = surf ? 0.5 : 1.0;
                    if (erow) {  // row-uniform medium: per-row sums, coefficients once
                        double sv = 0.0, sxx2 = 0.0, sss2 = 0.0, sq = 0.0;
#pragma unroll
                        for (int q = 0; q < ECPT; q++) {
                            const double v = (double)__half2float(vxr.q[q >> 1].e[q & 1]);
                            const double xn = (double)__half2float(sxx_old.q[q >> 1].e[q & 1]);
                            const double x1 = (double)__half2float(sxx.q[q >> 1].e[q & 1]);
                            const double sn = (double)__half2float(sss_old.q[q >> 1].e[q & 1]);
                            const double s1 = (double)__half2float(sss.q[q >> 1].e[q & 1]);
                            sv += v * v;
                            sxx2 += xn * x1;
                            sss2 += sn * s1;
                            sq += xn * s1 + sn * x1;
                        }
                        e[0] += (w * p64(P.e_rho_x, k, 0, 0)) * sv;
                        const double lamd = p64(P.e_lam, k, 0, 0), mu = p64(P.e_mu, k, 0, 0);
                        const double stiffd = lamd + 2.0 * mu;
                        const double dd = 4.0 * mu * (lamd + mu);
                        double val;
                        if (mu == 0.0) val = surf ? 0.0 : sxx2 / (lamd + mu);
                        else if (surf) val = sxx2 * stiffd / dd;
                        else val = (stiffd * (sxx2 + sss2) - lamd * sq) / dd;
                        if (surf) val = 0.5 * val;
                        e[3] += val;
                    } else {
#pragma unroll
                        for (int q = 0; q < ECPT; q++) {
                            const int xi = x + q;
                            const double v = (double)__half2float(vxr.q[q >> 1].e[q & 1]);
                            e[0] += (w * p64(P.e_rho_x, k, 0, xi)) * (v * v);
                            const double lamd = p64(P.e_lam, k, 0, xi), mu = p64(P.e_mu, k, 0, xi);
                            const double xn = (double)__half2float(sxx_old.q[q >> 1].e[q & 1]);
                            const double x1 = (double)__half2float(sxx.q[q >> 1].e[q & 1]);
                            const double sn = (double)__half2float(sss_old.q[q >> 1].e[q & 1]);
                            const double s1 = (double)__half2float(sss.q[q >> 1].e[q & 1]);
                            const double stiffd = lamd + 2.0 * mu;
                            const double dd = 4.0 * mu * (lamd + mu);
                            double val;
                            if (mu == 0.0) val = surf ? 0.0 : (xn * x1) / (lamd + mu);
                            else if (surf) val = xn * x1 * stiffd / dd;
                            else val = (stiffd * (xn * x1 + sn * s1) - lamd * (xn * s1 + sn * x1)) / dd;
                            if (surf) val = 0.5 * val;
                            e[3] += val;
                        }
                    }
                }
            }
            if (k < rh) {
                if (sample) {  // kinetic y + shear energy at this half row
                    const E8& vyr = vyq.q2;  // vy_new[k]
                    if (erow) {
                        double sv = 0.0, sa = 0.0;
#pragma unroll
                        for (int q = 0; q < ECPT; q++) {
                            const double v = (double)__half2float(vyr.q[q >> 1].e[q & 1]);
                            sv += v * v;
                            sa += (double)__half2float(old.q[q >> 1].e[q & 1]) * (double)__half2float(s.q[q >> 1].e[q & 1]);
                        }
                        e[1] += p64(P.e_rho_s, k, 0, 0) * sv;
                        const double mun = p64(P.e_mu_n, k, 0, 0);
                        e[4] += mun > 0.0 ? sa / mun : 0.0;
                    } else {
#pragma unroll
                        for (int q = 0; q < ECPT; q++) {
                            const int xi = x + q;
                            const double v = (double)__half2float(vyr.q[q >> 1].e[q & 1]);
                            e[1] += p64(P.e_rho_s, k, 0, xi) * (v * v);
                            const double mun = p64(P.e_mu_n, k, 0, xi);
                            const double o0 = (double)__half2float(old.q[q >> 1].e[q & 1]);
                            const double o1 = (double)__half2float(s.q[q >> 1].e[q & 1]);
                            e[4] += mun > 0.0 ? (o0 * o1) / mun : 0.0;
                        }
                    }
                }
            }
        }
        gyp = gy;
        if (++l0 == LR) {
            l0 = 0;
            lpar ^= 1u;
        }
        // every read of the B rows and of vx_new row k is done: refill B for iteration i + 1
        // (vx_new row k's slot is rewritten in phase A of the next iteration)
        __syncthreads();
        if (comp && tid == 0 && i + 1 < NI && i + 1 >= 6) {
            fence_proxy_async_smem();
            issue_b(i + 1);
        }
    }
    unsigned int mask = 0;
    mask |= e_nonfinite(acc[0]) << P.vx.bit;
    mask |= e_nonfinite(acc[1]) << P.vs.bit;
    mask |= e_nonfinite(acc[2]) << P.sxx.bit;
    mask |= e_nonfinite(acc[3]) << P.sss.bit;
    mask |= e_nonfinite(acc[4]) << P.sxs.bit;
    record_failure(P.ctrl, n, mask);
    if constexpr (!SAMPLE) return;
    block_partials(e, P.partials, pidx);
    __threadfence();
    __syncthreads();
    __shared__ unsigned int is_last;
    if (tid == 0) is_last = atomicAdd(IO.counter, 1u) == (unsigned int)(nb - 1);
    __syncthreads();
    if (!is_last) return;
    const double t = finalize_partials(P.partials, nb);  // fixed-order fp64 reduction
    if (tid == 0) {
        IO.e_vals[eidx] = IO.scale * t;
        *IO.counter = 0u;
    }
}

// ---------------------------------------------------------------- host side

bool el2d_fused_eligible(int64_t nx, int64_t ns, int max_smem) {
    // nx / 8 threads (a partial last warp is fine: the collectives use the existing lanes);
    // widths that are not a multiple of 256 only on large grids, as the streaming kernels
    if (nx % 8 != 0 || nx < 64 || nx / ECPT > 512 || ns < 8) return false;
    if (nx % 256 != 0 && nx * ns < ((int64_t)1 << 21)) return false;
    return el2d_fused_smem_bytes(nx) <= (size_t)max_smem;
}

template <int V, int O, bool F>
static void el2f_attrs1(int bytes) {
    cudaFuncSetAttribute((void*)k_el2d_fused<V, O, false, false, F>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    cudaFuncSetAttribute((void*)k_el2d_fused<V, O, true, false, F>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    cudaFuncSetAttribute((void*)k_el2d_fused<V, O, false, true, F>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    cudaFuncSetAttribute((void*)k_el2d_fused<V, O, true, true, F>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}
template <int V, int O>
static void el2f_attrs(int bytes) {
    el2f_attrs1<V, O, false>(bytes);
    el2f_attrs1<V, O, true>(bytes);
}

cudaError_t el2d_fused_prepare(int64_t nx) {
    const int bytes = (int)el2d_fused_smem_bytes(nx);
    el2f_attrs<0, 2>(bytes); el2f_attrs<3, 2>(bytes); el2f_attrs<6, 2>(bytes);
    el2f_attrs<0, 4>(bytes); el2f_attrs<3, 4>(bytes); el2f_attrs<6, 4>(bytes);
    return cudaGetLastError();
}

static bool el2f_rowmed(const ElParams& P) {
    auto div = [](const PlaneView& v) { return v.div_mode == DIV_CHEAP && v.sx == 0 && v.sm == 0; };
    auto row = [](const PlaneView& v) { return v.sx == 0 && v.sm == 0; };
    return div(P.rho_x) && div(P.rho_s) && row(P.stiff) && row(P.lam) && row(P.mu_n);
}

#define EL2F_DISPATCH(variant, order, CALL)                                          \
    if (order == 2) {                                                                \
        if (variant == 0) { constexpr int V_ = 0, O_ = 2; CALL; }                    \
        else if (variant == 3) { constexpr int V_ = 3, O_ = 2; CALL; }               \
        else { constexpr int V_ = 6, O_ = 2; CALL; }                                 \
    } else {                                                                         \
        if (variant == 0) { constexpr int V_ = 0, O_ = 4; CALL; }                    \
        else if (variant == 3) { constexpr int V_ = 3, O_ = 4; CALL; }               \
        else { constexpr int V_ = 6, O_ = 4; CALL; }                                 \
    }

void launch_el2d_fused(int variant, int order, const ElParams& P, const El2In& in, const StreamIO& IO, int nblocks,
                       int64_t n, double src, int sample, int64_t eidx, cudaStream_t st) {
    void* fn = nullptr;
    const bool rm = el2f_rowmed(P);
#define EL2F_PICK(FS_)                                                                    \
    if (rm && sample) {                                                                   \
        EL2F_DISPATCH(variant, order, (fn = (void*)k_el2d_fused<V_, O_, true, true, FS_>))   \
    } else if (rm) {                                                                      \
        EL2F_DISPATCH(variant, order, (fn = (void*)k_el2d_fused<V_, O_, true, false, FS_>))  \
    } else if (sample) {                                                                  \
        EL2F_DISPATCH(variant, order, (fn = (void*)k_el2d_fused<V_, O_, false, true, FS_>))  \
    } else {                                                                              \
        EL2F_DISPATCH(variant, order, (fn = (void*)k_el2d_fused<V_, O_, false, false, FS_>)) \
    }
    if (P.fs) {
        EL2F_PICK(true)
    } else {
        EL2F_PICK(false)
    }
#undef EL2F_PICK
    void* args[] = {(void*)&P, (void*)&in, (void*)&IO, (void*)&n, (void*)&src, (void*)&eidx};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nblocks);
    cfg.blockDim = dim3((unsigned)(P.g.nx / ECPT));
    cfg.dynamicSmemBytes = el2d_fused_smem_bytes(P.g.nx);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelExC(&cfg, fn, args);
}

}  // namespace hw
