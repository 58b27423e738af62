// hw_elastic3d_fused.cu — one-pass 3D elastic leapfrog step, binary16 state, 2nd order,
// periodic (BASELINE config 5: 512^3, layered), sm_100a.
//
// Both phases of the 3D velocity-stress step (ElasticSolver._step_work, elastic.py:176-238,
// 3D extension of SURVEY §8 a'; the same ops and fold orders as k_el_vel / k_el_stress and the
// streaming kernels, so the bits are identical) in ONE kernel per step, state n read from
// buffer A and state n+1 written to buffer B.  The two streaming phase kernels move ~93 B per
// cell-step; this one moves the algorithmic 72 B plus one halo row per mid tile and field.
//
// A CTA (2048 / CPT threads, CPT cells = CPT/2 half2 each) owns a tile of TM = 2048/NX mid
// rows x the full x width and streams it along the slow axis ((tile, slab) units split evenly
// over the CTAs).  Iteration i has front F = sb - 2 + i; the tap ring (4 slots) holds the six
// stress tiles of slabs F-2 .. F+1 (slab F+1 is requested at the top of iteration i):
//   sxx, sxs, sss : mid rows m0 .. m0+TM        (x / slow taps of vx, vs incl. their halo row m0+TM)
//   sxm, sms, smm : mid rows m0-1 .. m0+TM      (mid taps of vx, vs; x / slow / mid taps of vm incl.
//                                                its halo row m0-1)
// phase A: velocities of slab k = F-1 for the tile rows plus the halo rows vx, vs (m0+TM) and
//   vm (m0-1) (recomputed redundantly, never stored; thread rows j = 0, 1, 2 take one each),
//   written to a velocity tile generation in shared memory;
// phase B: stresses of slab s = F-2 from the previous generation (x / mid taps, own rows of slab
//   s) and this generation's own rows (slow taps of vx, vm at s+1), v_slow(s-1) from registers.
// Old velocities / residuals of slab F-1 come through one staged slot (read in phase A, refilled
// during phase B), the stress residuals of slab F-2 through another (read in phase B, refilled
// during phase A).  All slab indices wrap (single periodic domain).
//
// Instruction budget (the kernel is issue-bound, not DRAM-bound, at 512^3): the grid geometry
// (NX, TM, cells per thread) is compile-time, so every shared-memory tap is a 32-bit
// per-thread offset plus a uniform slot offset plus an immediate; the medium coefficients of a
// (slab, mid row) come from one host-built table row (row reciprocals of the three densities,
// the three stencil-lane moduli: two 16-byte loads per iteration); global stores add one
// per-thread 64-bit offset to the field base; the periodic ghost write-through is a
// CTA-uniform branch taken on the first / last G slabs only.
#include <cuda_runtime.h>

#include "hw_params.h"
#include "hw_stream.cuh"
#include "hw_tma.cuh"
#include "../../include/halfwave_b200.h"

namespace hw {

template <int NX_, int CPT_>
struct X3G {
    static constexpr int NX = NX_, CPT = CPT_, P = CPT / 2;
    static constexpr int NT = 2048 / CPT;  // threads per CTA
    static constexpr int TM = 2048 / NX;   // mid rows per tile
    static constexpr int TPR = NX / CPT;   // threads per tile row
    static constexpr int R1 = TM + 1, R2 = TM + 2;
    // tap-ring slot: six stress tiles (rows)
    static constexpr int O_SXX = 0, O_SXS = R1, O_SSS = 2 * R1, O_SXM = 3 * R1, O_SMS = 3 * R1 + R2,
                         O_SMM = 3 * R1 + 2 * R2;
    static constexpr int SLOT = 3 * R1 + 3 * R2;
    // 3 tap slots (slabs F-1, F, F+1; slab F+1 requested a full iteration ahead).  The slab-(F-2) values a
    // step needs (slow-axis taps of sxs / sms, the old stresses of the stress phase) are carried in
    // registers from the iteration before, when that slab sat in slot F-1 (CARRY) -- a fourth slot
    // holding slab F-2 measured 1.3 % slower at nx = 512 (216 vs 183 KB of shared memory: less L1 left)
    // and does not fit at nx = 1024 (264 KB); a fourth slot used to prefetch two iterations ahead: 0.6 % slower
    static constexpr int RING = 3;
    static constexpr bool CARRY = true;
    static constexpr int PD = RING - 2;  // tap prefetch distance in iterations
    // element offsets of the staged slots and the velocity tile generations
    static constexpr int A0 = RING * SLOT * NX;      // vx, vs, vm [rvx, rvs, rvm]: R1 rows each
    static constexpr int B0 = A0 + 6 * R1 * NX;      // rsxx rsss rsmm rsxs rsxm rsms: TM rows each
    static constexpr int V0 = B0 + 6 * TM * NX;      // 2 generations x [vx, vs, vm]: R1 rows each
    static constexpr int END = V0 + 6 * R1 * NX;
    static constexpr size_t BYTES = 128 + (size_t)END * 2;
};

template <int P>
struct EV {
    EH2 q[P];
};

template <int P>
__device__ __forceinline__ EV<P> ldv(const __half* p) {
    EV<P> r;
    if constexpr (P == 2) {
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

template <int P>
__device__ __forceinline__ void stv(__half* p, const EV<P>& v) {
    if constexpr (P == 2) {
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

// x derivative of the thread's cells (periodic) from a shared row block: `row` + to (own
// cells), + tl / + tr (the neighbouring pairs); to_int: shifts (-1, 0) else (0, 1) (2nd order)
template <int P>
__device__ __forceinline__ EV<P> xfv(const __half c[4], const __half* row, int to, int tl, int tr, bool to_int) {
    EH2 Q[P + 2];
    Q[0] = e_ld2(row + tl);
    const EV<P> own = ldv<P>(row + to);
#pragma unroll
    for (int q = 0; q < P; q++) Q[1 + q] = own.q[q];
    Q[P + 1] = e_ld2(row + tr);
    EH2 S[P + 1];
#pragma unroll
    for (int q = 0; q < P + 1; q++) S[q] = vshift<16, 2>(Q[q], Q[q + 1]);
    EV<P> r;
#pragma unroll
    for (int q = 0; q < P; q++)
        r.q[q] = to_int ? e_fold<2>(c, Q[q], S[q], Q[q + 1], S[q + 1]) : e_fold<2>(c, S[q], Q[q + 1], S[q + 1], Q[q + 2]);
    return r;
}

// 2nd-order fold of two rows a (first tap), b (second tap)
template <int P>
__device__ __forceinline__ EV<P> fv(const __half c[4], const EV<P>& a, const EV<P>& b) {
    EV<P> r;
#pragma unroll
    for (int q = 0; q < P; q++) r.q[q] = e_fold<2>(c, a.q[q], a.q[q], b.q[q], b.q[q]);
    return r;
}

template <int P>
__device__ __forceinline__ EV<P> addv(const EV<P>& a, const EV<P>& b) {
    EV<P> r;
#pragma unroll
    for (int q = 0; q < P; q++) r.q[q] = EO2::add(a.q[q], b.q[q]);
    return r;
}

template <int P>
__device__ __forceinline__ void trackv(__half2& acc, const EV<P>& v) {
#pragma unroll
    for (int q = 0; q < P; q++) acc = __hmax2_nan(acc, __habs2(v.q[q].h2));
}

// point source into the right-hand side of the source cell (the first op of finish()); a
// register select per pair (no dynamic indexing)
template <int P>
__device__ __forceinline__ void add_srcv(EH2 r[P], int sj, int sln, __half srch) {
#pragma unroll
    for (int h = 0; h < P; h++)
        if (h == sj) {
            if (sln == 0) r[h].e[0] = __hadd_rn(r[h].e[0], srch);
            else r[h].e[1] = __hadd_rn(r[h].e[1], srch);
        }
}

// store of the thread's cells of slab s at element offset so = s * slab + goff.  No ghost rows: the
// kernel never reads them on a single domain (its slab indices wrap) and a slab's come from the halo
// exchange, so the write-through copies of the phase kernels are not needed here.
template <int P>
__device__ __forceinline__ void gst(const FieldView& f, int64_t so, const EV<P>& v) {
    stv<P>(reinterpret_cast<__half*>(f.base) + so, v);
}

// binary16 -> binary64, one conversion (exact)
__device__ __forceinline__ double h2d(__half h) {
    double r;
    asm("cvt.f64.f16 %0, %1;" : "=d"(r) : "h"(__half_as_ushort(h)));
    return r;
}

// velocity increment + advance for one pair, divided by the row-uniform density b:
//   DIV_CHEAP: fl16(fl32(a * rcp_rn(b))) with the table-verified reciprocal cf (inline);
//   DIV_FAST : the branch-free exact division of lane<16>::div (hw_lanes.cuh) with b = cf and its
//              rcp.approx rf computed once per row -- the same ops, so the same bits (inline);
//   DIV_IEEE : zero / non-finite divisors.
__device__ __forceinline__ __half x3_div1(__half a, float fb, float r) {
    const float fa = __half2float(a);
    const float q0 = __fmul_rn(fa, r);
    const float e = __fmaf_rn(-fb, q0, fa);
    const float q1 = __fmaf_rn(e, r, q0);
    const bool keep = (e == 0.0f) || !(fabsf(q0) < INFINITY);
    return __float2half_rn(keep ? q0 : q1);
}
__device__ __forceinline__ EH2 x3_div_ieee(EH2 a, float fb) {
    return EO2::div_ieee(a, vsplat<16, 2>(__float2half_rn(fb)));
}
template <int V>
__device__ __forceinline__ void x3_finish(EH2 a, float cf, float rf, int mode, __half2 dt2, __half srch, EH2& u,
                                          EH2& t) {
    if (mode == DIV_CHEAP) {
        e_finish_rc<V>(a, cf, dt2, -1, srch, u, t);
    } else {
        EH2 q;
        if (mode == DIV_FAST) {
            q.e[0] = x3_div1(a.e[0], cf, rf);
            q.e[1] = x3_div1(a.e[1], cf, rf);
        } else {
            q = x3_div_ieee(a, cf);
        }
        e2_finish_nd<V>(q, dt2, -1, srch, u, t);  // x dt, then the advance (same ops as finish())
    }
}
__device__ __forceinline__ float x3_rcp(float b) {  // lane<16>::div's reciprocal
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(b));
    return r;
}

// TMA requests of one slot (thread 0)
template <int NX, int TM>
__device__ __forceinline__ void x3_issue_tap(__half* d, uint64_t* b, const __half* sxx, const __half* sxs,
                                          const __half* sss, const __half* sxm, const __half* sms, const __half* smm,
                                          int64_t slab, int s, int m0, int nm) {
    constexpr int R1 = TM + 1, R2 = TM + 2;
    constexpr uint32_t rb = NX * sizeof(__half);
    mbar_arrive_expect_tx(b, (uint32_t)(3 * R1 + 3 * R2) * rb);
    a3_rows(d, sxx, slab, s, m0, m0 + TM + 1, nm, NX, b);
    a3_rows(d + R1 * NX, sxs, slab, s, m0, m0 + TM + 1, nm, NX, b);
    a3_rows(d + 2 * R1 * NX, sss, slab, s, m0, m0 + TM + 1, nm, NX, b);
    a3_rows(d + 3 * R1 * NX, sxm, slab, s, m0 - 1, m0 + TM + 1, nm, NX, b);
    a3_rows(d + (3 * R1 + R2) * NX, sms, slab, s, m0 - 1, m0 + TM + 1, nm, NX, b);
    a3_rows(d + (3 * R1 + 2 * R2) * NX, smm, slab, s, m0 - 1, m0 + TM + 1, nm, NX, b);
}
template <int NX, int TM>
__device__ __forceinline__ void x3_issue_a(__half* d, uint64_t* b, const __half* vx, const __half* vs, const __half* vm,
                                        const __half* rvx, const __half* rvs, const __half* rvm, int comp,
                                        int64_t slab, int s, int m0, int nm) {
    constexpr int R1 = TM + 1;
    constexpr uint32_t rb = NX * sizeof(__half);
    mbar_arrive_expect_tx(b, (uint32_t)((comp ? 6 : 3) * R1) * rb);
    a3_rows(d, vx, slab, s, m0, m0 + TM + 1, nm, NX, b);
    a3_rows(d + R1 * NX, vs, slab, s, m0, m0 + TM + 1, nm, NX, b);
    a3_rows(d + 2 * R1 * NX, vm, slab, s, m0 - 1, m0 + TM, nm, NX, b);
    if (comp) {
        a3_rows(d + 3 * R1 * NX, rvx, slab, s, m0, m0 + TM + 1, nm, NX, b);
        a3_rows(d + 4 * R1 * NX, rvs, slab, s, m0, m0 + TM + 1, nm, NX, b);
        a3_rows(d + 5 * R1 * NX, rvm, slab, s, m0 - 1, m0 + TM, nm, NX, b);
    }
}
template <int NX, int TM>
__device__ __forceinline__ void x3_issue_b(__half* d, uint64_t* b, const __half* r0, const __half* r1, const __half* r2,
                                        const __half* r3, const __half* r4, const __half* r5, int64_t off) {
    constexpr uint32_t tb = (uint32_t)(TM * NX * sizeof(__half));
    mbar_arrive_expect_tx(b, 6 * tb);
    tma_load_1d(d, r0 + off, tb, b);
    tma_load_1d(d + TM * NX, r1 + off, tb, b);
    tma_load_1d(d + 2 * TM * NX, r2 + off, tb, b);
    tma_load_1d(d + 3 * TM * NX, r3 + off, tb, b);
    tma_load_1d(d + 4 * TM * NX, r4 + off, tb, b);
    tma_load_1d(d + 5 * TM * NX, r5 + off, tb, b);
}

template <int V, int NX, int CPT, bool SAMPLE>
__global__ void __launch_bounds__(2048 / CPT, 1)
    k_el3d_fused(ElParams P, El3In in, StreamIO IO, int64_t n, double src, int64_t eidx) {
    using X = X3G<NX, CPT>;
    constexpr int PP = X::P, TM = X::TM, R1 = X::R1, SLOT = X::SLOT;
    constexpr bool sample = SAMPLE;
    constexpr bool comp = V != 0;
    e_pdl_enter();
    if (halted(P.ctrl, n)) return;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);  // RING tap barriers, A, B
    uint64_t* abar = bar + X::RING;
    uint64_t* bbar = bar + X::RING + 1;
    __half* S = reinterpret_cast<__half*>(smem + 128);
    const int nm = (int)P.g.nm, ns = (int)P.sxx.rows;
    const int64_t slab = (int64_t)nm * NX;  // pitch == NX (eligibility)
    const int tid = threadIdx.x, j = tid / X::TPR, x = (tid % X::TPR) * CPT;
    // per-thread element offsets inside a block of rows: own cells, left / right neighbour pairs
    const int to = j * NX + x, tl = j * NX + (x == 0 ? NX - 2 : x - 2), tr = j * NX + (x + CPT >= NX ? 0 : x + CPT);
    constexpr uint32_t rb = NX * sizeof(__half);
    if (tid == 0) {
        for (int q = 0; q < X::RING + 2; q++) mbar_init(&bar[q], 1);
        fence_mbar_init();
    }
    __syncthreads();

    __half c[4];
#pragma unroll
    for (int q = 0; q < 4; q++) c[q] = lconst<16>(P.k, q);
    const __half dt = lconst<16>(P.k, 4);
    const __half2 dt2 = __half2half2(dt);
    const __half srch = __double2half(src);
    const bool vsrc = in.vsrc && src != 0.0;  // CTA-uniform; its row may be a slab's halo row (-1 or L)
    const bool ssrc = P.src_kind == HW_SRC_EXPLOSIVE && src != 0.0;  // CTA-uniform
    const bool src_col = (vsrc || ssrc) && P.src_x >= x && P.src_x < x + CPT;
    const int sj = (int)((P.src_x - x) >> 1), sln = (int)((P.src_x - x) & 1);
    const bool erow = in.ecoef != nullptr;  // energy planes constant within a slab (per-slab table)
    const FieldView* OS[6] = {&P.sxx, &P.sss, &P.smm, &P.sxs, &P.sxm, &P.sms};
    const FieldView* ORS[6] = {&P.rsxx, &P.rsss, &P.rsmm, &P.rsxs, &P.rsxm, &P.rsms};
    __half2 acc[9];
#pragma unroll
    for (int q = 0; q < 9; q++) acc[q] = __float2half2_rn(0.f);
    __shared__ double ered[32];  // per-warp energy partials of one (tile, slab) unit
    const int cm = (int)in.coef_m;  // coefficient rows per slab: 1 (slow-layered) or nm

    // single periodic domain: slab indices wrap; slab of a decomposed domain: rows -2 .. ns+1 are
    // ghost rows filled by the halo exchange (HW_PLAN_FUSED_EL3) before every step
    const bool slabm = in.slab != 0;
    auto wrap = [&](int s) { return slabm ? s : (s < 0 ? s + ns : (s >= ns ? s - ns : s)); };
    // Work split: groups of `grp` CTAs own `grp` adjacent mid tiles and stream the same slab
    // range side by side, so the halo rows one CTA reads are the rows its neighbour in the
    // group reads (or wrote) at about the same time: L2 hits instead of DRAM re-reads.  The
    // group's (tile group, slab) units are split evenly over the groups.
    // Band mode (slab of a decomposed domain, exchange overlapped): 1 = the edge slabs [0, E) and
    // [ns-E, ns) -- every row the halo exchange sends --, 2 = the interior [E, ns-E) (reads no ghost
    // row), 0 = every slab.  t indexes the band's slabs; segments never straddle the two edge runs.
    const int E = in.edge, bm = in.band;
    const int nsl = bm == 0 ? ns : (bm == 1 ? 2 * E : ns - 2 * E);
    auto slab_of = [&](int t) { return bm == 0 ? t : (bm == 1 ? (t < E ? t : ns - 2 * E + t) : E + t); };
    const int grp = in.group, ngrp = (int)gridDim.x / grp, gid = (int)blockIdx.x / grp, gr = (int)blockIdx.x % grp;
    const int tiles = nm / TM / grp;  // tile groups
    const int64_t U = (int64_t)tiles * nsl;
    int64_t u = (int64_t)gid * U / ngrp;
    const int64_t u1 = (int64_t)(gid + 1) * U / ngrp;
    int gi = 0, ga = 0, gb = 0;  // running use counters of the tap slots, the A and the B slot
    while (u < u1) {
        const int t0 = (int)(u % nsl);
        int te = (int)min((int64_t)nsl, t0 + (u1 - u));
        if (bm == 1 && t0 < E) te = min(te, E);
        const int tile = (int)(u / nsl) * grp + gr, sb = slab_of(t0);
        const int se = sb + (te - t0);
        u += te - t0;
        const int m0 = tile * TM, m = m0 + j;
        const int mlo = m0 == 0 ? nm - 1 : m0 - 1, mhi = m0 + TM == nm ? 0 : m0 + TM;  // halo rows (periodic)
        const int mh = j == 0 ? mlo : mhi;            // this thread row's halo row (j < 3)
        const int hq = j == 0 ? 2 : (j == 1 ? 0 : 1);  // ... and its density (rho_m, rho_x, rho_s)
        const int64_t goff = (int64_t)m * NX + x;
        const int F0 = sb - 2, NI = se - sb + 4;
        const int gi0 = gi, ga0 = ga, gb0 = gb;
        auto issue_tap = [&](int i) {  // the six stress tiles of slab F0 + i
            const int sl = (gi0 + i) % X::RING;
            x3_issue_tap<NX, TM>(S + sl * SLOT * NX, &bar[sl], in.sxx, in.sxs, in.sss, in.sxm, in.sms, in.smm, slab,
                                 wrap(F0 + i), m0, nm);
        };
        auto issue_a = [&](int i) {  // old velocities (+ residuals) of slab F0 + i - 1
            x3_issue_a<NX, TM>(S + X::A0, abar, in.vx, in.vs, in.vm, in.rvx, in.rvs, in.rvm, comp ? 1 : 0, slab,
                               wrap(F0 + i - 1), m0, nm);
        };
        auto issue_b = [&](int i) {  // stress residuals of slab F0 + i - 2 (own rows)
            x3_issue_b<NX, TM>(S + X::B0, bbar, in.rsxx, in.rsss, in.rsmm, in.rsxs, in.rsxm, in.rsms,
                               (int64_t)wrap(F0 + i - 2) * slab + (int64_t)m0 * NX);
        };
        // the TMA requests are issued by lane 0 of warps 1, 2 and 3 (the tap ring, the A slot, the B
        // slot): one on each of three SM sub-partitions, so no warp carries all of them into the barriers
        if (tid == 32) {
            issue_tap(0);
            if (X::PD > 1 && NI > 1) issue_tap(1);
        }
        if (tid == 64) issue_a(0);
        EV<PP> vs_m1, vs_m2;  // v_slow own rows of slabs F-2, F-3 (new)
        // CARRY: the thread's slab-(F-2) stress values (own cells of the six fields; its halo-row cells of
        // sms / sxs), read from slot F-1 at the end of the previous iteration
        EV<PP> cold[6], chalo;
        float4 cs = make_float4(0.f, 0.f, 0.f, 0.f);  // (stiff, lam, mu) of the stress slab (previous k)
#pragma unroll 1
        for (int i = 0; i < NI; i++) {
            const int F = F0 + i;
            const int s0 = (gi0 + i) % X::RING, s1 = (gi0 + i + X::RING - 1) % X::RING;  // F, F-1
            const int s2 = X::CARRY ? s1 : (gi0 + i + 2) % X::RING;  // F-2 (CARRY: never read; its values are in registers)
            const int gen = i & 1;
            const __half* T0 = S + s0 * SLOT * NX;
            const __half* T1 = S + s1 * SLOT * NX;
            const __half* T2 = S + s2 * SLOT * NX;
            if (tid == 32 && i + X::PD < NI) {  // slot (i + PD) % RING held slab F-2: last read in iteration i-1
                fence_proxy_async_smem();
                issue_tap(i + X::PD);
            }
            const bool vel = i >= 2;
            const int k = wrap(F - 1);
            // medium coefficients of slab k (loaded before the ring waits)
            float4 cv = make_float4(0.f, 0.f, 0.f, 0.f), cn = cv;
            float rch = 0.f, rch2 = 0.f;
            if (vel) {
                const float4* cr = reinterpret_cast<const float4*>(in.coef) + 2 * ((int64_t)k * cm + (cm > 1 ? m : 0));
                cv = __ldg(cr);
                cn = __ldg(cr + 1);
                if (j < 3) rch = __ldg(in.coef + 8 * ((int64_t)k * cm + (cm > 1 ? mh : 0)) + hq);
                if (TM < 3 && j == 1) rch2 = __ldg(in.coef + 8 * ((int64_t)k * cm + (cm > 1 ? mhi : 0)) + 1);  // rho_s of vs(m0+TM)
            }
            mbar_wait(&bar[s0], (uint32_t)(((gi0 + i) / X::RING) & 1));
            if (!vel) mbar_wait(abar, (uint32_t)((ga0 + i) & 1));
            EV<PP> vs_new;
            if (vel) {  // ---- velocities of slab k = F-1 (elastic.py:191-205, 3D)
                const __half* A = S + X::A0;
                __half* VT = S + X::V0 + gen * 3 * R1 * NX;
                // vx: fl(fl(ddx sxx + dds sxs) + ddm sxm)
                const EV<PP> ax =
                    addv<PP>(addv<PP>(xfv<PP>(c, T1 + X::O_SXX * NX, to, tl, tr, false),
                                      fv<PP>(c, X::CARRY ? cold[3] : ldv<PP>(T2 + X::O_SXS * NX + to), ldv<PP>(T1 + X::O_SXS * NX + to))),
                             fv<PP>(c, ldv<PP>(T1 + X::O_SXM * NX + to), ldv<PP>(T1 + (X::O_SXM + 1) * NX + to)));
                // v_slow: fl(fl(ddx sxs + dds sss) + ddm sms) (+ src)
                EV<PP> as =
                    addv<PP>(addv<PP>(xfv<PP>(c, T1 + X::O_SXS * NX, to, tl, tr, true),
                                      fv<PP>(c, ldv<PP>(T1 + X::O_SSS * NX + to), ldv<PP>(T0 + X::O_SSS * NX + to))),
                             fv<PP>(c, ldv<PP>(T1 + X::O_SMS * NX + to), ldv<PP>(T1 + (X::O_SMS + 1) * NX + to)));
                // v_mid: fl(fl(ddx sxm + dds sms) + ddm smm)
                const EV<PP> am = addv<PP>(
                    addv<PP>(xfv<PP>(c, T1 + (X::O_SXM + 1) * NX, to, tl, tr, true),
                             fv<PP>(c, X::CARRY ? cold[5] : ldv<PP>(T2 + (X::O_SMS + 1) * NX + to), ldv<PP>(T1 + (X::O_SMS + 1) * NX + to))),
                    fv<PP>(c, ldv<PP>(T1 + (X::O_SMM + 1) * NX + to), ldv<PP>(T1 + (X::O_SMM + 2) * NX + to)));
                if (vsrc && k == in.vsrc_s && m == P.src_m && src_col) add_srcv<PP>(as.q, sj, sln, srch);
                // the old values are waited for only now: the A slot was refilled during the previous
                // iteration's stress phase, the stencil sums above overlap the rest of its latency
                mbar_wait(abar, (uint32_t)((ga0 + i) & 1));
                const float rx = x3_rcp(cv.x), ry = x3_rcp(cv.y), rz = x3_rcp(cv.z);  // (DIV_FAST rows)
                // own rows: vx, vs at tile index j (row m), vm at index j + 1 of its tile
                EV<PP> vx = ldv<PP>(A + to), vsv = ldv<PP>(A + R1 * NX + to), vm = ldv<PP>(A + (2 * R1 + 1) * NX + to);
                EV<PP> rvx, rvs, rvm;
                if (comp) {
                    rvx = ldv<PP>(A + 3 * R1 * NX + to);
                    rvs = ldv<PP>(A + 4 * R1 * NX + to);
                    rvm = ldv<PP>(A + (5 * R1 + 1) * NX + to);
                }
#pragma unroll
                for (int h = 0; h < PP; h++) {
                    x3_finish<V>(ax.q[h], cv.x, rx, in.div_mode[0], dt2, srch, vx.q[h], rvx.q[h]);
                    x3_finish<V>(as.q[h], cv.y, ry, in.div_mode[1], dt2, srch, vsv.q[h], rvs.q[h]);
                    x3_finish<V>(am.q[h], cv.z, rz, in.div_mode[2], dt2, srch, vm.q[h], rvm.q[h]);
                }
                stv<PP>(VT + to, vx);
                stv<PP>(VT + R1 * NX + to, vsv);
                stv<PP>(VT + (2 * R1 + 1) * NX + to, vm);
                vs_new = vsv;
                const int sk = F - 1;  // unwrapped: stored only inside the segment
                if (sk >= sb && sk < se) {
                    const int64_t so = (int64_t)k * slab + goff;
                    gst<PP>(P.vx, so, vx);
                    gst<PP>(P.vs, so, vsv);
                    gst<PP>(P.vm, so, vm);
                    trackv<PP>(acc[0], vx);
                    trackv<PP>(acc[1], vsv);
                    trackv<PP>(acc[2], vm);
                    if (comp) {
                        gst<PP>(P.rvx, so, rvx);
                        gst<PP>(P.rvs, so, rvs);
                        gst<PP>(P.rvm, so, rvm);
                    }
                }
                // halo rows (recomputed, not stored): j = 0 -> vm(m0-1), j = 1 -> vx(m0+TM), j = 2 -> vs(m0+TM)
                if (j == 0) {
                    const int a0 = x;  // row 0 of the tiles
                    EV<PP> h = ldv<PP>(A + 2 * R1 * NX + a0);
                    EV<PP> rh;
                    if (comp) rh = ldv<PP>(A + 5 * R1 * NX + a0);
                    const EV<PP> a =
                        addv<PP>(addv<PP>(xfv<PP>(c, T1 + X::O_SXM * NX, to, tl, tr, true),
                                          fv<PP>(c, X::CARRY ? chalo : ldv<PP>(T2 + X::O_SMS * NX + a0), ldv<PP>(T1 + X::O_SMS * NX + a0))),
                                 fv<PP>(c, ldv<PP>(T1 + X::O_SMM * NX + a0), ldv<PP>(T1 + (X::O_SMM + 1) * NX + a0)));
#pragma unroll
                    for (int q = 0; q < PP; q++) x3_finish<V>(a.q[q], rch, x3_rcp(rch), in.div_mode[2], dt2, srch, h.q[q], rh.q[q]);
                    stv<PP>(VT + 2 * R1 * NX + a0, h);
                } else if (j == 1 || (TM >= 3 && j == 2)) {
                    // thread row jj's halo row: jj = 1 -> vx(m0+TM), jj = 2 -> vs(m0+TM); a tile of TM = 2 rows has
                    // no thread row 2, so its row 1 takes both
                    auto halo_hi = [&](int jj, float rc) {
                        const int a0 = TM * NX + x;  // row TM of the tiles
                        const int fo = jj == 1 ? 0 : R1 * NX;  // vx or vs in the A slot / the velocity tile
                        const int dj = (jj - j) * NX, to_ = to + dj, tl_ = tl + dj, tr_ = tr + dj;
                        EV<PP> h = ldv<PP>(A + fo + a0);
                        EV<PP> rh;
                        if (comp) rh = ldv<PP>(A + 3 * R1 * NX + fo + a0);
                        EV<PP> a;
                        if (jj == 1) {
                            a = addv<PP>(addv<PP>(xfv<PP>(c, T1 + X::O_SXX * NX + (TM - 1) * NX, to_, tl_, tr_, false),
                                                  fv<PP>(c, X::CARRY ? chalo : ldv<PP>(T2 + X::O_SXS * NX + a0), ldv<PP>(T1 + X::O_SXS * NX + a0))),
                                         fv<PP>(c, ldv<PP>(T1 + X::O_SXM * NX + a0), ldv<PP>(T1 + (X::O_SXM + 1) * NX + a0)));
                        } else {
                            a = addv<PP>(addv<PP>(xfv<PP>(c, T1 + X::O_SXS * NX + (TM - 2) * NX, to_, tl_, tr_, true),
                                                  fv<PP>(c, ldv<PP>(T1 + X::O_SSS * NX + a0), ldv<PP>(T0 + X::O_SSS * NX + a0))),
                                         fv<PP>(c, ldv<PP>(T1 + X::O_SMS * NX + a0), ldv<PP>(T1 + (X::O_SMS + 1) * NX + a0)));
                            if (vsrc && k == in.vsrc_s && mhi == P.src_m && src_col) add_srcv<PP>(a.q, sj, sln, srch);
                        }
                        const int hm = in.div_mode[jj == 1 ? 0 : 1];
#pragma unroll
                        for (int q = 0; q < PP; q++) x3_finish<V>(a.q[q], rc, x3_rcp(rc), hm, dt2, srch, h.q[q], rh.q[q]);
                        stv<PP>(VT + fo + a0, h);
                    };
                    if constexpr (TM >= 3) {
                        halo_hi(j, rch);
                    } else {
                        halo_hi(1, rch);
                        halo_hi(2, rch2);
                    }
                }
            }
            __syncthreads();  // velocity tiles of slab F-1 visible; the A slot and tap slot (i+1) % RING are free
            if (tid == 64 && i + 1 < NI) {
                fence_proxy_async_smem();
                issue_a(i + 1);
            }
            const int s = F - 2;  // stress slab (unwrapped; in [0, ns) when computed)
            if (s >= sb && s < se) {  // ---- stresses of slab s (elastic.py:210-238, 3D)
                const int pg = gen ^ 1;  // generation of slab s
                const __half* vxt = S + X::V0 + pg * 3 * R1 * NX;  // rows m0 .. m0+TM
                const __half* vst = vxt + R1 * NX;                 // rows m0 .. m0+TM
                const __half* vmt = vxt + 2 * R1 * NX;             // rows m0-1 .. m0+TM-1
                const __half* vxn = S + X::V0 + gen * 3 * R1 * NX;  // slab s+1
                const __half* vmn = vxn + 2 * R1 * NX;
                const EV<PP> dvx = xfv<PP>(c, vxt, to, tl, tr, true);
                const EV<PP> dvs = fv<PP>(c, vs_m2, vs_m1);  // v_slow(s-1), v_slow(s) (own rows)
                const EV<PP> dvm = fv<PP>(c, ldv<PP>(vmt + to), ldv<PP>(vmt + NX + to));
                EV<PP> old[6], nw[6], rr[6];
                if constexpr (X::CARRY) {
#pragma unroll
                    for (int q = 0; q < 6; q++) old[q] = cold[q];
                } else {
                    old[0] = ldv<PP>(T2 + X::O_SXX * NX + to);
                    old[1] = ldv<PP>(T2 + X::O_SSS * NX + to);
                    old[2] = ldv<PP>(T2 + (X::O_SMM + 1) * NX + to);
                    old[3] = ldv<PP>(T2 + X::O_SXS * NX + to);
                    old[4] = ldv<PP>(T2 + (X::O_SXM + 1) * NX + to);
                    old[5] = ldv<PP>(T2 + (X::O_SMS + 1) * NX + to);
                }
#pragma unroll
                for (int q = 0; q < 6; q++) nw[q] = old[q];
                const EH2 stiff = vsplat<16, 2>(__float2half_rn(cs.x)), lam = vsplat<16, 2>(__float2half_rn(cs.y));
                const EH2 mu = vsplat<16, 2>(__float2half_rn(cs.z));  // (binary16 values: exact round trips)
                EH2 a0[PP], a1[PP], a2[PP];
#pragma unroll
                for (int h = 0; h < PP; h++) {
                    a0[h] = EO2::add(EO2::add(EO2::mul(stiff, dvx.q[h]), EO2::mul(lam, dvs.q[h])), EO2::mul(lam, dvm.q[h]));
                    a1[h] = EO2::add(EO2::add(EO2::mul(lam, dvx.q[h]), EO2::mul(stiff, dvs.q[h])), EO2::mul(lam, dvm.q[h]));
                    a2[h] = EO2::add(EO2::add(EO2::mul(lam, dvx.q[h]), EO2::mul(lam, dvs.q[h])), EO2::mul(stiff, dvm.q[h]));
                }
                if (ssrc && s == P.src_s && m == P.src_m && src_col) {  // explosive source into the normal stresses
                    add_srcv<PP>(a0, sj, sln, srch);
                    add_srcv<PP>(a1, sj, sln, srch);
                    add_srcv<PP>(a2, sj, sln, srch);
                }
                // shear: fl(mu fl(dd_a v_b + dd_b v_a)), to-half taps
                const EV<PP> sxs_a = fv<PP>(c, ldv<PP>(vxt + to), ldv<PP>(vxn + to));                  // vx(s), vx(s+1)
                const EV<PP> sxs_b = xfv<PP>(c, vst, to, tl, tr, false);
                const EV<PP> sxm_a = fv<PP>(c, ldv<PP>(vxt + to), ldv<PP>(vxt + NX + to));             // vx rows m, m+1
                const EV<PP> sxm_b = xfv<PP>(c, vmt + NX, to, tl, tr, false);
                const EV<PP> sms_a = fv<PP>(c, ldv<PP>(vmt + NX + to), ldv<PP>(vmn + NX + to));        // vm(s), vm(s+1)
                const EV<PP> sms_b = fv<PP>(c, ldv<PP>(vst + to), ldv<PP>(vst + NX + to));             // vs rows m, m+1
                // stress residuals (B slot, refilled during this iteration's velocity phase): waited for last
                mbar_wait(bbar, (uint32_t)((gb0 + (i - 4)) & 1));
                if (comp) {
#pragma unroll
                    for (int q = 0; q < 6; q++) rr[q] = ldv<PP>(S + X::B0 + q * TM * NX + to);
                }
#pragma unroll
                for (int h = 0; h < PP; h++) {
                    e2_finish_nd<V>(a0[h], dt2, -1, srch, nw[0].q[h], rr[0].q[h]);
                    e2_finish_nd<V>(a1[h], dt2, -1, srch, nw[1].q[h], rr[1].q[h]);
                    e2_finish_nd<V>(a2[h], dt2, -1, srch, nw[2].q[h], rr[2].q[h]);
                    e2_finish_nd<V>(EO2::mul(mu, EO2::add(sxs_a.q[h], sxs_b.q[h])), dt2, -1, srch, nw[3].q[h], rr[3].q[h]);
                    e2_finish_nd<V>(EO2::mul(mu, EO2::add(sxm_a.q[h], sxm_b.q[h])), dt2, -1, srch, nw[4].q[h], rr[4].q[h]);
                    e2_finish_nd<V>(EO2::mul(mu, EO2::add(sms_a.q[h], sms_b.q[h])), dt2, -1, srch, nw[5].q[h], rr[5].q[h]);
                }
                const int64_t so = (int64_t)s * slab + goff;
#pragma unroll
                for (int q = 0; q < 6; q++) {
                    gst<PP>(*OS[q], so, nw[q]);
                    trackv<PP>(acc[3 + q], nw[q]);
                    if (comp) gst<PP>(*ORS[q], so, rr[q]);
                }
                if (sample) {  // diagnostics.py:100-162, 3D compliance form (k_el_stress)
                    double e[NCOMP] = {0.0, 0.0, 0.0, 0.0, 0.0};  // this (tile, slab) unit's share
                    const EV<PP> vxo = ldv<PP>(vxt + to), vmo = ldv<PP>(vmt + NX + to), vso = ldv<PP>(vst + to);
                    auto f = [&](const EV<PP>& a, int q) { return (double)__half2float(a.q[q >> 1].e[q & 1]); };
                    if (erow) {  // per-slab medium: raw sums per iteration, one coefficient row per slab
                        double skx = 0.0, skm = 0.0, sks = 0.0, sx1 = 0.0, sdot = 0.0, str = 0.0, ssh = 0.0;
#pragma unroll
                        for (int q = 0; q < CPT; q++) {
                            auto g = [&](const EV<PP>& a) { return h2d(a.q[q >> 1].e[q & 1]); };
                            const double a = g(vxo), b = g(vmo), w = g(vso);
                            skx += a * a;
                            skm += b * b;
                            sks += w * w;
                            const double xn = g(old[0]), x1 = g(nw[0]), sn = g(old[1]), s1 = g(nw[1]);
                            const double mn = g(old[2]), m1 = g(nw[2]);
                            sx1 += xn * x1;
                            sdot += xn * x1 + sn * s1 + mn * m1;
                            str += (xn + sn + mn) * (x1 + s1 + m1);
                            // shear: products of binary16 pairs are exact in binary32 (22-bit significands,
                            // no underflow), so each product takes one conversion instead of two
                            auto hp = [&](int w) {
                                const __half a1 = old[w].q[q >> 1].e[q & 1], b1 = nw[w].q[q >> 1].e[q & 1];
                                return (double)__fmul_rn(__half2float(a1), __half2float(b1));
                            };
                            ssh += (hp(3) + hp(4)) + hp(5);
                        }
                        // rho_x, rho_s, rho_m, 1/(lam+mu) [mu = 0], 1/(2 mu), lam/(2 mu (3 lam + 2 mu)), 1/mu_n
                        const double* ec = in.ecoef + 8 * (int64_t)s;
                        e[0] += __ldg(ec + 0) * skx;
                        e[1] += __ldg(ec + 1) * sks;
                        e[2] += __ldg(ec + 2) * skm;
                        e[3] += (__ldg(ec + 3) * sx1 + __ldg(ec + 4) * sdot) - __ldg(ec + 5) * str;
                        e[4] += __ldg(ec + 6) * ssh;
                    } else {
#pragma unroll
                        for (int q = 0; q < CPT; q++) {
                            const int xi = x + q;
                            const double a = f(vxo, q), b = f(vmo, q), g = f(vso, q);
                            e[0] += p64(P.e_rho_x, s, m, xi) * (a * a);
                            e[2] += p64(P.e_rho_m, s, m, xi) * (b * b);
                            e[1] += p64(P.e_rho_s, s, m, xi) * (g * g);
                            const double lamd = p64(P.e_lam, s, m, xi), mud = p64(P.e_mu, s, m, xi);
                            const double xn = f(old[0], q), x1 = f(nw[0], q), sn = f(old[1], q), s1 = f(nw[1], q);
                            const double mn = f(old[2], q), m1 = f(nw[2], q);
                            if (mud == 0.0) {
                                e[3] += (xn * x1) / (lamd + mud);
                            } else {
                                const double dot = xn * x1 + sn * s1 + mn * m1;
                                e[3] += dot / (2.0 * mud) -
                                        lamd * (xn + sn + mn) * (x1 + s1 + m1) / (2.0 * mud * (3.0 * lamd + 2.0 * mud));
                            }
                            const double mun = p64(P.e_mu_n, s, m, xi);
                            for (int w = 3; w < 6; w++) e[4] += mun > 0.0 ? (f(old[w], q) * f(nw[w], q)) / mun : 0.0;
                        }
                    }
                    // per-plane partials (decomposition-invariant energy): the thread's share of the
                    // unit, a warp tree now, the warps' sums combined by lane 0 of warp 0 after the
                    // end-of-iteration barrier
                    const double a = warp_sum((((e[0] + e[1]) + e[2]) + e[3]) + e[4]);
                    if ((tid & 31) == 0) ered[tid >> 5] = a;
                }
            }
            if (vel) {
                vs_m2 = vs_m1;
                vs_m1 = vs_new;
                cs = cn;  // moduli of slab k: the next iteration's stress slab
            }
            if constexpr (X::CARRY) {  // slab F-1 is the next iteration's slab F-2: its slot is refilled then
                if (i >= 1) {
                    cold[0] = ldv<PP>(T1 + X::O_SXX * NX + to);
                    cold[1] = ldv<PP>(T1 + X::O_SSS * NX + to);
                    cold[2] = ldv<PP>(T1 + (X::O_SMM + 1) * NX + to);
                    cold[3] = ldv<PP>(T1 + X::O_SXS * NX + to);
                    cold[4] = ldv<PP>(T1 + (X::O_SXM + 1) * NX + to);
                    cold[5] = ldv<PP>(T1 + (X::O_SMS + 1) * NX + to);
                    chalo = ldv<PP>(T1 + (j == 0 ? X::O_SMS * NX : (X::O_SXS + TM) * NX) + x);
                }
            }
            __syncthreads();  // the previous velocity generation and the B slot are free
            if (tid == 96 && i + 1 < NI && F + 1 - 2 >= sb && F + 1 - 2 < se) {
                fence_proxy_async_smem();
                issue_b(i + 1);
            }
            if (sample && tid == 0 && s >= sb && s < se) {  // the unit's partial, warps in order
                double a = ered[0];
                for (int w = 1; w < X::NT / 32; w++) a += ered[w];
                in.eplane[(int64_t)s * (nm / TM) + tile] = a;
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
    __threadfence();
    __syncthreads();
    __shared__ unsigned int is_last;
    // (edge + interior launches of one step share the counter: in.nb_total CTAs in all)
    const unsigned int nbt = in.nb_total > 0 ? (unsigned int)in.nb_total : gridDim.x;
    if (tid == 0) is_last = atomicAdd(IO.counter, 1u) == nbt - 1;
    __syncthreads();
    if (!is_last) return;
    // plane totals T[s] = sum_tile partial[s][tile], tiles in order: the host sums the planes of all
    // slabs in global order (el3_energy_from_planes, hw_api.cu)
    const int tiles_all = nm / TM;
    for (int sp = tid; sp < ns; sp += X::NT) {
        double t = __ldcg(&in.eplane[(int64_t)sp * tiles_all]);
        for (int t2 = 1; t2 < tiles_all; t2++) t += __ldcg(&in.eplane[(int64_t)sp * tiles_all + t2]);
        in.etot[eidx * (int64_t)ns + sp] = t;
    }
    if (tid == 0) *IO.counter = 0u;
}

// Plane totals of a generic energy launch (k_el_energy: one block partial per (x chunk, mid
// row, slab), slab-major): T[s] = sum_c (sum_b partial[s][b][c]) with every order fixed -- per
// component a thread-strided sum, a warp tree and the warps in order -- so the same for any
// decomposition (E(0) of the one-pass kernel's runs).  One CTA of 256 threads per slab.
__global__ void __launch_bounds__(256) k_plane_totals(const double* partials, int64_t blocks_per_plane, double* out) {
    __shared__ double red[8];
    const int64_t sp = blockIdx.x;
    const int tid = threadIdx.x;
    double t = 0.0;
    for (int c = 0; c < NCOMP; c++) {
        double a = 0.0;
        for (int64_t b = tid; b < blocks_per_plane; b += 256) a += partials[(sp * blocks_per_plane + b) * NCOMP + c];
        a = warp_sum(a);
        if ((tid & 31) == 0) red[tid >> 5] = a;
        __syncthreads();
        if (tid == 0) {
            double w = red[0];
            for (int k = 1; k < 8; k++) w += red[k];
            t += w;
        }
        __syncthreads();
    }
    if (tid == 0) out[sp] = t;
}

// Medium coefficient table of the one-pass kernel: per (slab, mid row) -- one row per slab
// when every plane is constant along mid -- rho_x, rho_s, rho_m as their verified reciprocals
// (DIV_CHEAP planes) or their values, and the stencil-lane stiff, lam, mu_n, all as binary32
// (exact: binary16 values / binary32 reciprocals).
__global__ void k_el3_coef(PlaneView rx, PlaneView rs, PlaneView rm, PlaneView st, PlaneView la, PlaneView mu,
                           float* out, int64_t s0, int64_t ns, int64_t cm) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ns * cm) return;
    const int64_t s = s0 + i / cm, m = i % cm;
    float* o = out + 8 * i;
    const PlaneView* rho[3] = {&rx, &rs, &rm};
    for (int q = 0; q < 3; q++) {
        const PlaneView& v = *rho[q];
        const int64_t k = s * v.ss + m * v.sm;
        o[q] = v.div_mode == DIV_CHEAP ? v.rcp[k] : __half2float(reinterpret_cast<const __half*>(v.p)[k]);
    }
    o[3] = 0.f;
    o[4] = __half2float(reinterpret_cast<const __half*>(st.p)[s * st.ss + m * st.sm]);
    o[5] = __half2float(reinterpret_cast<const __half*>(la.p)[s * la.ss + m * la.sm]);
    o[6] = __half2float(reinterpret_cast<const __half*>(mu.p)[s * mu.ss + m * mu.sm]);
    o[7] = 0.f;
}

// Energy coefficients of slow-layered media (every fp64 energy plane constant within a slab), per
// slab: rho_x, rho_s, rho_m, then the compliance factors of diagnostics.py:100-162 (3D form)
// 1/(lam+mu) when mu = 0 (else 0), 1/(2 mu) and lam/(2 mu (3 lam + 2 mu)) when mu > 0 (else 0),
// 1/mu_n when mu_n > 0 (else 0): the sample steps multiply instead of dividing per iteration.
__global__ void k_el3_ecoef(Plane64 rx, Plane64 rs, Plane64 rm, Plane64 la, Plane64 mu, Plane64 mn, double* out,
                            int64_t ns) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= ns) return;
    double* o = out + 8 * s;
    o[0] = p64(rx, s, 0, 0);
    o[1] = p64(rs, s, 0, 0);
    o[2] = p64(rm, s, 0, 0);
    const double l = p64(la, s, 0, 0), m = p64(mu, s, 0, 0), n = p64(mn, s, 0, 0);
    o[3] = m == 0.0 ? 1.0 / (l + m) : 0.0;
    o[4] = m == 0.0 ? 0.0 : 1.0 / (2.0 * m);
    o[5] = m == 0.0 ? 0.0 : l / (2.0 * m * (3.0 * l + 2.0 * m));
    o[6] = n > 0.0 ? 1.0 / n : 0.0;
    o[7] = 0.0;
}

// ---------------------------------------------------------------- host side

#ifndef HW_X3C
#define HW_X3C 4
#endif
constexpr int X3C = HW_X3C;  // cells per thread (4 or 8)

static size_t x3_bytes(int64_t nx) {
    return nx == 1024 ? X3G<1024, X3C>::BYTES : (nx == 512 ? X3G<512, X3C>::BYTES : X3G<256, X3C>::BYTES);
}

bool el3d_fused_eligible(const ElParams& P, int64_t nx, int64_t nm, int64_t ns, int64_t pitch, int order,
                         int max_smem) {
    if (order != 2 || P.fs || (nx != 256 && nx != 512 && nx != 1024) || pitch != nx || ns < 4) return false;
    const int64_t TM = 2048 / nx;
    if (nm % TM != 0 || nm < 2 * TM || x3_bytes(nx) > (size_t)max_smem) return false;
    // densities and moduli constant along x (slow-layered or per (slab, mid) row)
    return P.rho_x.sx == 0 && P.rho_s.sx == 0 && P.rho_m.sx == 0 && P.stiff.sx == 0 && P.lam.sx == 0 &&
           P.mu_n.sx == 0;
}

int64_t el3d_fused_coef_rows(const ElParams& P) {
    return (P.rho_x.sm | P.rho_s.sm | P.rho_m.sm | P.stiff.sm | P.lam.sm | P.mu_n.sm) == 0 ? 1 : P.g.nm;
}

bool el3d_fused_erow(const ElParams& P) {
    return ((P.e_rho_x.sx | P.e_rho_s.sx | P.e_rho_m.sx | P.e_lam.sx | P.e_mu.sx | P.e_mu_n.sx) |
            (P.e_rho_x.sm | P.e_rho_s.sm | P.e_rho_m.sm | P.e_lam.sm | P.e_mu.sm | P.e_mu_n.sm)) == 0;
}

cudaError_t el3d_fused_ecoef(const ElParams& P, double* out, int64_t ns, cudaStream_t st) {
    k_el3_ecoef<<<(unsigned)((ns + 127) / 128), 128, 0, st>>>(P.e_rho_x, P.e_rho_s, P.e_rho_m, P.e_lam, P.e_mu,
                                                             P.e_mu_n, out, ns);
    return cudaGetLastError();
}

cudaError_t el3d_fused_coef(const ElParams& P, float* out, int64_t s0, int64_t ns, int64_t cm, cudaStream_t st) {
    const int64_t cnt = ns * cm;
    k_el3_coef<<<(unsigned)((cnt + 255) / 256), 256, 0, st>>>(P.rho_x, P.rho_s, P.rho_m, P.stiff, P.lam, P.mu_n, out,
                                                              s0, ns, cm);
    return cudaGetLastError();
}

void launch_plane_totals(const double* partials, int64_t blocks_per_plane, int64_t nplanes, double* out,
                         cudaStream_t st) {
    k_plane_totals<<<(unsigned)nplanes, 256, 0, st>>>(partials, blocks_per_plane, out);
}

template <int NX>
static void x3_attrs() {
    const int b = (int)X3G<NX, X3C>::BYTES;
    void* fns[] = {(void*)k_el3d_fused<0, NX, X3C, false>, (void*)k_el3d_fused<3, NX, X3C, false>,
                   (void*)k_el3d_fused<6, NX, X3C, false>,  (void*)k_el3d_fused<0, NX, X3C, true>,
                   (void*)k_el3d_fused<3, NX, X3C, true>,   (void*)k_el3d_fused<6, NX, X3C, true>};
    for (void* fn : fns) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
}

cudaError_t el3d_fused_prepare(int64_t nx) {
    if (nx == 1024) x3_attrs<1024>();
    else if (nx == 512) x3_attrs<512>();
    else x3_attrs<256>();
    return cudaGetLastError();
}

template <int NX>
static void* x3_fn(int variant, int sample) {
    if (sample)
        return variant == 0 ? (void*)k_el3d_fused<0, NX, X3C, true>
                            : (variant == 3 ? (void*)k_el3d_fused<3, NX, X3C, true> : (void*)k_el3d_fused<6, NX, X3C, true>);
    return variant == 0 ? (void*)k_el3d_fused<0, NX, X3C, false>
                        : (variant == 3 ? (void*)k_el3d_fused<3, NX, X3C, false> : (void*)k_el3d_fused<6, NX, X3C, false>);
}

void launch_el3d_fused(int variant, const ElParams& P, const El3In& in, const StreamIO& IO, int nblocks, int64_t n,
                       double src, int sample, int64_t eidx, cudaStream_t st) {
    void* fn = P.g.nx == 1024 ? x3_fn<1024>(variant, sample)
                              : (P.g.nx == 512 ? x3_fn<512>(variant, sample) : x3_fn<256>(variant, sample));
    void* args[] = {(void*)&P, (void*)&in, (void*)&IO, (void*)&n, (void*)&src, (void*)&eidx};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nblocks);
    cfg.blockDim = dim3(2048 / X3C);
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
