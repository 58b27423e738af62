// hw_acoustic3d_fused32.cu — one-pass 3D acoustic leapfrog step, binary32 lanes (S = U =
// fp32), 2nd order, sm_100a: the fp32 comparison arm of BASELINE config 3 ("fp16 compensated
// vs fp32 naive"), on the same one-pass streaming structure as the binary16 kernel
// (hw_acoustic3d_fused.cu), so that the two precision modes are compared on equally tuned
// kernels.
//
// AcousticSolver._step_work (acoustic.py:162-181, 3D extension of SURVEY §8 a') with
// fp32 stencil and update lanes: every op is one IEEE binary32 op (__fadd_rn / __fmul_rn /
// __fdiv_rn, no FMA contraction), in the fold orders of k_ac_vel / k_ac_pres, so the bits
// equal the generic kernels' and the oracle's.  Any variant (naive / op3 / op6) is
// supported; BASELINE uses naive.
//
// State n is read from buffer A and state n+1 written to buffer B (ping-pong).  A CTA
// (512 threads, 4 cells = one float4 each) owns a tile of TM = 2048/nx mid rows x the full x
// width and streams it along the slow axis ((tile, slab) units split evenly over the CTAs).
// Iteration i has front F = sb - 1 + i and output slab s = F - 1:
//   * the tap ring (3 slots, 1 slab ahead) brings the p tile of slab F, mid rows m0-1 .. m0+TM;
//   * the own ring (2 slots, one slab ahead) brings vx, vs, beta [, rp, rvx, rvs] (TM rows) and
//     vm [, rvm] (TM+1 rows from m0-1) of slab s;
//   * v_slow(s) from a 2-deep register queue of p rows; vx(s) from the p tile of slab s (x taps);
//     vm(s) for rows m0-1 .. m0+TM-1 (row m0-1 recomputed by the j = 0 threads);
//   * new vx / vm rows to shared memory, one barrier, then p(s) = fl(fl(ddx vx + dds vs) + ddm vm).
// Divisors: a plane constant along x whose row value is a power of two divides by multiplying
// with its exact reciprocal (x / 2^k and x * 2^-k are the same real, rounded once: identical
// bits, subnormals included); every other divisor takes __fdiv_rn (zero dividends inline).
#include <cuda_runtime.h>

#include "hw_params.h"
#include "hw_stream.cuh"
#include "hw_tma.cuh"
#include "../../include/halfwave_b200.h"

namespace hw {

#ifndef HW_Q3C
#define HW_Q3C 4
#endif
constexpr int Q3C = HW_Q3C;      // cells per thread (one or two float4)
constexpr int Q3T = 2048 / Q3C;  // threads per CTA (TM = 2048 / nx either way)
constexpr int QR = 3;     // tap ring slots (5 slots, 3 ahead measured 1.8 % slower: 24 KB more shared memory, less L1)
constexpr int QD = 1;     // prefetch distance

enum { Q_VX = 0, Q_VS, Q_RP, Q_BETA, Q_RVX, Q_RVS, Q_NTM };

struct F4 {
    float e[Q3C];
};

__device__ __forceinline__ F4 q_ld(const float* p) {
    F4 r;
#pragma unroll
    for (int h = 0; h < Q3C / 4; h++) {
        const float4 v = *reinterpret_cast<const float4*>(p + 4 * h);
        r.e[4 * h] = v.x;
        r.e[4 * h + 1] = v.y;
        r.e[4 * h + 2] = v.z;
        r.e[4 * h + 3] = v.w;
    }
    return r;
}
__device__ __forceinline__ void q_st(float* p, const F4& v) {
#pragma unroll
    for (int h = 0; h < Q3C / 4; h++)
        *reinterpret_cast<float4*>(p + 4 * h) = make_float4(v.e[4 * h], v.e[4 * h + 1], v.e[4 * h + 2], v.e[4 * h + 3]);
}
// 2nd-order fold of the inner tap pair: fl(fl(c1 a) + fl(c2 b)) (stencil.py:72-79, outer pair dropped)
__device__ __forceinline__ float q_fold(float c1, float c2, float a, float b) {
    return __fadd_rn(__fmul_rn(c1, a), __fmul_rn(c2, b));
}
__device__ __forceinline__ F4 q_sfold(float c1, float c2, const F4& a, const F4& b) {
    F4 r;
#pragma unroll
    for (int i = 0; i < Q3C; i++) r.e[i] = q_fold(c1, c2, a.e[i], b.e[i]);
    return r;
}
// x derivative of 4 cells (periodic) from a shared row: to-int shifts (-1, 0), to-half (0, 1)
__device__ __forceinline__ F4 q_xfold(float c1, float c2, const float* row, int x, int xl, int xr, bool to_int) {
    const F4 o = q_ld(row + x);
    F4 r;
    if (to_int) {
        const float l = row[xl];
        r.e[0] = q_fold(c1, c2, l, o.e[0]);
#pragma unroll
        for (int i = 1; i < Q3C; i++) r.e[i] = q_fold(c1, c2, o.e[i - 1], o.e[i]);
    } else {
        const float rr = row[xr];
#pragma unroll
        for (int i = 0; i < Q3C - 1; i++) r.e[i] = q_fold(c1, c2, o.e[i], o.e[i + 1]);
        r.e[Q3C - 1] = q_fold(c1, c2, o.e[Q3C - 1], rr);
    }
    return r;
}
__device__ __forceinline__ F4 q_add(const F4& a, const F4& b) {
    F4 r;
#pragma unroll
    for (int i = 0; i < Q3C; i++) r.e[i] = __fadd_rn(a.e[i], b.e[i]);
    return r;
}

// running max of |x| that propagates NaN: non-finite iff the result is inf or NaN
__device__ __forceinline__ void q_track(float& acc, const F4& v) {
#pragma unroll
    for (int i = 0; i < Q3C; i++) asm("max.NaN.f32 %0, %0, %1;" : "+f"(acc) : "f"(fabsf(v.e[i])));
}
__device__ __forceinline__ unsigned int q_nonfinite(float acc) {
    return (__float_as_uint(acc) & 0x7f800000u) == 0x7f800000u ? 1u : 0u;
}

// divisor of one (slow, mid) row: a plane constant along x (sx == 0) gives one value per row
struct QDiv {
    float d, r;
    bool row, pow2, ok;  // ok: d finite and nonzero (the inline zero-dividend answer applies)
};
__device__ __forceinline__ QDiv q_rowdiv(const PlaneView& v, int64_t s, int64_t m) {
    QDiv q{0.f, 0.f, v.sx == 0, false, false};
    if (q.row) {
        q.d = __ldg(reinterpret_cast<const float*>(v.p) + (int)(s * v.ss + m * v.sm));  // (planes < 2^31 elements)
        const unsigned int b = __float_as_uint(q.d), e = (b >> 23) & 0xffu;
        q.pow2 = (b & 0x7fffffu) == 0u && e >= 1u && e <= 253u;  // 2^k with a normal reciprocal
        q.r = __uint_as_float((b & 0x80000000u) | ((254u - e) << 23));  // 2^-k exactly (used when pow2)
        q.ok = fabsf(q.d) < INFINITY && q.d != 0.0f;
    }
    return q;
}
// QDiv through shared memory: (d, r, flags) -- one uniform 16-byte load per use
__device__ __forceinline__ float4 q_pack(const QDiv& q) {
    return make_float4(q.d, q.r, __int_as_float((q.row ? 1 : 0) | (q.pow2 ? 2 : 0) | (q.ok ? 4 : 0)), 0.f);
}
__device__ __forceinline__ QDiv q_unpack(const float4& t) {
    const int f = __float_as_int(t.z);
    return QDiv{t.x, t.y, (f & 1) != 0, (f & 2) != 0, (f & 4) != 0};
}
// IEEE quotient a / b (__fdiv_rn) with zero dividends answered inline: __fdiv_rn sends a
// zero dividend down its slow path (a subroutine call per element), and the state is zero
// wherever the wave has not arrived yet.  ±0 / b for finite nonzero b is the signed zero.
__device__ __forceinline__ float q_divz(float a, float b, bool bok) {
    if (a == 0.0f && bok) return __uint_as_float((__float_as_uint(a) ^ __float_as_uint(b)) & 0x80000000u);
    return __fdiv_rn(a, b);
}

// UpdatePipeline.increment + advance (stepping.py:58-98, efsum.py:100-121) for 4 cells:
// rhs [+ round_U(src) on lane src_lane] -> / divisor -> x dt -> naive / op3 / op6 advance.
// The source and the division mode are warp-uniform branches around all four cells.
template <int V, bool ROWONLY>
__device__ __forceinline__ void q_finish(const F4& rhs, const QDiv& q, const float* dcell, float dt, int src_lane,
                                         float srcf, F4& u, F4& t) {
    F4 xq = rhs;
    if (src_lane >= 0) {
#pragma unroll
        for (int i = 0; i < Q3C; i++)
            if (i == src_lane) xq.e[i] = __fadd_rn(xq.e[i], srcf);
    }
    if (q.row && q.pow2) {
#pragma unroll
        for (int i = 0; i < Q3C; i++) xq.e[i] = __fmul_rn(xq.e[i], q.r);
    } else if (q.row) {
#pragma unroll
        for (int i = 0; i < Q3C; i++) xq.e[i] = q_divz(xq.e[i], q.d, q.ok);
    } else if constexpr (!ROWONLY) {  // per-cell divisors (staged in shared memory, or the plane row in global memory)
        const F4 dv = q_ld(dcell);
#pragma unroll
        for (int i = 0; i < Q3C; i++) xq.e[i] = q_divz(xq.e[i], dv.e[i], fabsf(dv.e[i]) < INFINITY && dv.e[i] != 0.0f);
    }
#pragma unroll
    for (int i = 0; i < Q3C; i++) {
        const float x = __fmul_rn(xq.e[i], dt);
        if (V == 0) {
            u.e[i] = __fadd_rn(u.e[i], x);
            continue;
        }
        const float r = __fadd_rn(t.e[i], x);
        const float sm = __fadd_rn(u.e[i], r);
        if (V == 3) {
            t.e[i] = __fsub_rn(r, __fsub_rn(sm, u.e[i]));
        } else {
            const float pa = __fsub_rn(sm, r);
            const float pb = __fsub_rn(sm, pa);
            t.e[i] = __fadd_rn(__fsub_rn(u.e[i], pa), __fsub_rn(r, pb));
        }
        u.e[i] = sm;
    }
}

// per-cell divisors of a plane that varies along x (sx == 1): its cells at (s, m, x); read
// only by q_finish's per-cell branch
__device__ __forceinline__ const float* q_dcell(const PlaneView& v, int64_t s, int64_t m, int x) {
    return reinterpret_cast<const float*>(v.p) + s * v.ss + m * v.sm + x;
}

// store one row segment (4 cells) and its periodic / image ghost copies (as e_store_row)
// (inner: G <= s < rows - G, a warp-uniform flag: no ghost copy)
__device__ __forceinline__ void q_store(const FieldView& f, int64_t slab, int s, int64_t off, const F4& v,
                                        bool inner) {
    float* base = reinterpret_cast<float*>(f.base);
    q_st(base + (int64_t)s * slab + off, v);
    if (inner || (f.gtop | f.gbot) == GHOST_NONE) return;
    const int n = (int)f.rows;
    if (f.gtop == GHOST_PERIODIC && s >= n - G) q_st(base + (int64_t)(s - n) * slab + off, v);
    if (f.gbot == GHOST_PERIODIC && s < G) q_st(base + (int64_t)(n + s) * slab + off, v);
    if ((f.gtop | f.gbot) & GHOST_IMAGE) {
        F4 w = v;
        if (f.odd) {
#pragma unroll
            for (int i = 0; i < Q3C; i++) w.e[i] = lane<32>::neg(v.e[i]);
        }
        const int sg = (int)f.row0 + s, ng = (int)f.nglob;
        if (f.gtop == GHOST_IMAGE) {
            const int k1 = f.half_s ? -sg - 1 : -sg;
            if (k1 < 0 && k1 >= -G) q_st(base + (int64_t)(k1 - (int)f.row0) * slab + off, w);
        }
        if (f.gbot == GHOST_IMAGE) {
            const int k2 = f.half_s ? 2 * ng - 1 - sg : 2 * ng - 2 - sg;
            if (k2 >= ng && k2 < ng + G) q_st(base + (int64_t)(k2 - (int)f.row0) * slab + off, w);
        }
    }
}

// TMA copy of mid rows [a, b) (periodic) of slab s
__device__ __forceinline__ void q_rows(float* dst, const float* fbase, int64_t slab, int64_t s, int a, int b, int nm,
                                       int64_t pitch, uint64_t* bar) {
    const float* sb = fbase + s * slab;
    for (int r = a; r < b;) {
        const int rr = a3_wrap(r, nm);
        const int seg = min(b - r, nm - rr);
        tma_load_1d(dst, sb + (int64_t)rr * pitch, (uint32_t)(seg * pitch * sizeof(float)), bar);
        dst += (int64_t)seg * pitch;
        r += seg;
    }
}

static size_t q3_bytes(int64_t nx) {
    const int64_t TM = Q3T * Q3C / nx;
    const int64_t rows = QR * (TM + 2) + 2 * (Q_NTM * TM + 2 * (TM + 1)) + TM + (TM + 1);
    return 256 + (size_t)rows * nx * sizeof(float);
}

// RR: the three density planes are constant along x (constant / layered media): no per-cell
// density code is compiled in.  NXC: the row width as a compile-time constant (512, BASELINE
// config 3: every shared-memory and row offset folds into immediates) or 0 (runtime width).
// SAMPLE: energy sample step (the fp64 energy code and its registers stay out of the other steps).
template <int V, bool RR, int NXC, bool SAMPLE>
__global__ void __launch_bounds__(Q3T, 1)
    k_ac3d_fused32(AcParams P, Ac3In in_, StreamIO IO, int64_t n, double src, int64_t eidx) {
    constexpr bool sample = SAMPLE;
    e_pdl_enter();
    if (halted(P.ctrl, n)) return;
    extern __shared__ __align__(128) unsigned char smem[];
    const float* in_p = reinterpret_cast<const float*>(in_.p);
    const float* in_vx = reinterpret_cast<const float*>(in_.vx);
    const float* in_vs = reinterpret_cast<const float*>(in_.vs);
    const float* in_vm = reinterpret_cast<const float*>(in_.vm);
    const float* in_rp = reinterpret_cast<const float*>(in_.rp);
    const float* in_rvx = reinterpret_cast<const float*>(in_.rvx);
    const float* in_rvs = reinterpret_cast<const float*>(in_.rvs);
    const float* in_rvm = reinterpret_cast<const float*>(in_.rvm);
    const int nx = NXC ? NXC : (int)P.g.nx, nm = (int)P.g.nm, ns = (int)P.p.rows;
    const int64_t pitch = NXC ? NXC : P.g.pitch, slab = (int64_t)nm * pitch;
    const int TM = Q3T * Q3C / nx, TPR = nx / Q3C;
    const int tid = threadIdx.x, j = tid / TPR, x = (tid % TPR) * Q3C;
    constexpr bool comp = V != 0;
    const bool bfull = P.beta.sx != 0;
    // shared layout (rows of pitch floats)
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
    uint64_t* obar = reinterpret_cast<uint64_t*>(smem + 64);
    float4* qdiv = reinterpret_cast<float4*>(smem + 128);  // [2][4]: row divisors of the next / this slab
    float* ring = reinterpret_cast<float*>(smem + 256);
    const int64_t tm = (int64_t)TM * pitch, slot = (int64_t)(TM + 2) * pitch;
    const int64_t oslot = ((int64_t)Q_NTM * TM + 2 * (TM + 1)) * pitch;
    float* own = ring + QR * slot;
    float* xv = own + 2 * oslot;  // TM rows: new vx of slab s
    float* vmn = xv + tm;         // TM + 1 rows: new vm of slab s, rows m0-1 .. m0+TM-1
    auto sl = [&](int k) { return ring + k * slot; };
    auto ob = [&](int os, int q) { return own + os * oslot + q * tm; };
    auto ovm = [&](int os) { return own + os * oslot + Q_NTM * tm; };
    auto orvm = [&](int os) { return ovm(os) + tm + pitch; };
    const uint32_t tmb = (uint32_t)(tm * sizeof(float));
    const uint32_t own_tx = (uint32_t)((2 + (bfull ? 1 : 0) + (comp ? 3 : 0)) * tm * sizeof(float) +
                                       (comp ? 2 : 1) * (tm + pitch) * sizeof(float));
    if (tid == 0) {
        for (int q = 0; q < QR; q++) mbar_init(&bar[q], 1);
        for (int q = 0; q < 2; q++) mbar_init(&obar[q], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const float c1 = lconst<32>(P.k, 1), c2 = lconst<32>(P.k, 2);
    const float dt = lconst<32>(P.k, 4);
    const float srcf = __double2float_rn(src);
    const int xl = x == 0 ? nx - 1 : x - 1, xr = x + Q3C >= nx ? 0 : x + Q3C;
    const bool src_col = P.has_src && src != 0.0 && P.src_x >= x && P.src_x < x + Q3C;
    const int sln = (int)(P.src_x - x);
    float acc[8];
#pragma unroll
    for (int q = 0; q < 8; q++) acc[q] = 0.f;
    __shared__ double ered[32];  // per-warp energy partials of one (tile, slab) unit (sample steps)

    // groups of `grp` CTAs own `grp` adjacent mid tiles and stream the same slab range side by side:
    // the halo rows one CTA reads are rows its neighbour in the group reads at about the same time
    // (L2 hits instead of DRAM re-reads); the (tile group, slab) units are split evenly over the groups
    const int grp = in_.group, ngrp = (int)gridDim.x / grp, gid = (int)blockIdx.x / grp, gr = (int)blockIdx.x % grp;
    const int tiles = nm / TM / grp;  // tile groups
    // Band mode (NCCL slab, exchange overlapped): 1 = the edge slabs 0 and ns-1 (every row the halo
    // exchange sends; the only slabs that read ghost rows), 2 = the interior [1, ns-1), 0 = every slab.
    // t indexes the band's slabs; a segment never straddles the two edge slabs.
    const int E = in_.edge, bm = in_.band;
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
            const int F = F0 + i, k = (gi0 + i) % QR;
            mbar_arrive_expect_tx(&bar[k], (uint32_t)(slot * sizeof(float)));
            q_rows(sl(k), in_p, slab, e_row(F), m0 - 1, m0 + TM + 1, nm, pitch, &bar[k]);
        };
        auto issue_own = [&](int kk) {  // slab sb - 1 + kk (periodic: slab -1 is ns - 1)
            const int os = (gk0 + kk) & 1, s = sb - 1 + kk < 0 ? (in_.slab ? -1 : ns - 1) : sb - 1 + kk;
            const int64_t off = (int64_t)s * slab + (int64_t)m0 * pitch;
            uint64_t* b = &obar[os];
            mbar_arrive_expect_tx(b, own_tx);
            tma_load_1d(ob(os, Q_VX), in_vx + off, tmb, b);
            tma_load_1d(ob(os, Q_VS), in_vs + off, tmb, b);
            if (bfull)
                tma_load_1d(ob(os, Q_BETA), reinterpret_cast<const float*>(P.beta.p) + s * P.beta.ss +
                                                (int64_t)m0 * P.beta.sm, tmb, b);
            q_rows(ovm(os), in_vm, slab, s, m0 - 1, m0 + TM, nm, pitch, b);
            if (comp) {
                tma_load_1d(ob(os, Q_RP), in_rp + off, tmb, b);
                tma_load_1d(ob(os, Q_RVX), in_rvx + off, tmb, b);
                tma_load_1d(ob(os, Q_RVS), in_rvs + off, tmb, b);
                q_rows(orvm(os), in_rvm, slab, s, m0 - 1, m0 + TM, nm, pitch, b);
            }
        };
        // the TMA requests come from lane 0 of warps 1 and 2 (the tap ring, the own ring): two SM
        // sub-partitions, so no warp carries all of them into the barriers
        if (tid == 32)
            for (int i = 0; i < QD && i < NI; i++) issue(i);
        if (tid == 64) issue_own(0);
        int rcur = rec_lower(IO.rec, 0, IO.n_rec, sb * nm + m, INT_MIN);  // receivers: key (s nm + m, x)
        F4 qp0{}, qp1{}, vsq{};  // p rows F-1, F at the thread's cells; v_slow(s-1)
        int k = gi0 % QR;                      // tap slot of iteration i (running, no division per iteration)
        uint32_t kph = (uint32_t)((gi0 / QR) & 1);  // its mbarrier phase
#pragma unroll 1
        for (int i = 0; i < NI; i++, k = k + 1 == QR ? 0 : k + 1, kph ^= (k == 0)) {
            const int kp = k == 0 ? QR - 1 : k - 1;
            if (tid == 32 && i + QD < NI) {
                fence_proxy_async_smem();
                issue(i + QD);
            }
            const int sw = F0 + i - 1 < 0 ? (in_.slab ? -1 : ns - 1) : F0 + i - 1;  // v_slow(-1): row ns-1's medium (periodic) or the slab's halo row
            // row divisors: threads 0-3 stage those of the next iteration's slab (F0 + i) in shared memory
            // (constant / slow-layered planes depend on the slab only; the barriers below order the use)
            if (tid < 4 && i + 1 < NI) {
                const int sn = F0 + i < 0 ? (in_.slab ? -1 : ns - 1) : F0 + i;
                const PlaneView& pv = tid == 0 ? P.rho_s : (tid == 1 ? P.rho_x : (tid == 2 ? P.rho_m : P.beta));
                qdiv[((i + 1) & 1) * 4 + tid] = q_pack(q_rowdiv(pv, sn, 0));
            }
            QDiv d_s{}, d_x{}, d_m{}, d_b{};
            if (i > 0) {
                const float4* qd = qdiv + (i & 1) * 4;
                d_s = q_unpack(qd[0]);
                d_x = q_unpack(qd[1]);
                d_m = q_unpack(qd[2]);
                d_b = q_unpack(qd[3]);
            }
            mbar_wait(&bar[k], kph);
            qp0 = qp1;
            qp1 = q_ld(sl(k) + (int64_t)(j + 1) * pitch + x);
            if (i > 0) {
                const int s = F0 + i - 1, kr = i - 1, os = (gk0 + kr) & 1;
                if (tid == 64 && s + 1 < se) {  // that own slot was last read before the previous barrier
                    fence_proxy_async_smem();
                    issue_own(kr + 1);
                }
                mbar_wait(&obar[os], (uint32_t)(((gk0 + kr) >> 1) & 1));
                const int64_t ro = (int64_t)j * pitch + x, off = (int64_t)m * pitch + x;
                const bool sin = s >= G && s < ns - G;
                // v_slow(s) from p rows s, s+1 (acoustic.py:169-170, to-half shifts (0, 1))
                F4 vsn = q_ld(ob(os, Q_VS) + ro);
                F4 rvs = comp ? q_ld(ob(os, Q_RVS) + ro) : F4{};
                q_finish<V, RR>(q_sfold(c1, c2, qp0, qp1), d_s, RR ? nullptr : q_dcell(P.rho_s, sw, m, x), dt, -1,
                            srcf, vsn, rvs);
                if (i > 1) {
                    const float* pt = sl(kp);  // p tile of slab s: row m at index j + 1
                    // vx(s) = fl(fl(ddx p / rho_x) dt) (acoustic.py:167-168)
                    F4 vxn = q_ld(ob(os, Q_VX) + ro);
                    F4 rvx = comp ? q_ld(ob(os, Q_RVX) + ro) : F4{};
                    q_finish<V, RR>(q_xfold(c1, c2, pt + (int64_t)(j + 1) * pitch, x, xl, xr, false),
                                d_x, RR ? nullptr : q_dcell(P.rho_x, s, m, x), dt, -1, srcf, vxn, rvx);
                    q_st(xv + ro, vxn);
                    {  // vm(s) row m from p mid rows m, m+1
                        const float* t = pt + (int64_t)(j + 1) * pitch + x;
                        F4 vmv = q_ld(ovm(os) + ro + pitch);
                        F4 rvm = comp ? q_ld(orvm(os) + ro + pitch) : F4{};
                        q_finish<V, RR>(q_sfold(c1, c2, q_ld(t), q_ld(t + pitch)), d_m,
                                    RR ? nullptr : q_dcell(P.rho_m, s, m, x), dt, -1, srcf, vmv, rvm);
                        q_st(vmn + ro + pitch, vmv);
                        q_store(P.vm, slab, s, off, vmv, sin);
                        q_track(acc[3], vmv);
                        if (comp) {
                            q_store(P.rvm, slab, s, off, rvm, sin);
                            q_track(acc[7], rvm);
                        }
                    }
                    if (j == 0) {  // halo row m0-1: recomputed, not stored
                        const float* t = pt + x;
                        F4 vmh = q_ld(ovm(os) + x);
                        F4 rvh = comp ? q_ld(orvm(os) + x) : F4{};
                        q_finish<V, RR>(q_sfold(c1, c2, q_ld(t), q_ld(t + pitch)), d_m,
                                    RR ? nullptr : q_dcell(P.rho_m, s, mh, x), dt, -1, srcf, vmh, rvh);
                        q_st(vmn + x, vmh);
                    }
                    q_store(P.vx, slab, s, off, vxn, sin);
                    q_track(acc[1], vxn);
                    q_store(P.vs, slab, s, off, vsn, sin);
                    q_track(acc[2], vsn);
                    if (comp) {
                        q_store(P.rvx, slab, s, off, rvx, sin);
                        q_track(acc[5], rvx);
                        q_store(P.rvs, slab, s, off, rvs, sin);
                        q_track(acc[6], rvs);
                    }
                    __syncthreads();
                    // p(s): fl(fl(ddx vx + dds v_slow) + ddm vm) (acoustic.py:172-175), to-int taps
                    const F4 tx = q_xfold(c1, c2, xv + (int64_t)j * pitch, x, xl, xr, true);
                    const F4 ts = q_sfold(c1, c2, vsq, vsn);
                    const F4 m1 = q_ld(vmn + ro), m2 = q_ld(vmn + ro + pitch);
                    const F4 tmv = q_sfold(c1, c2, m1, m2);
                    const bool sk = src_col && s == P.src_s && m == P.src_m;
                    const F4 pold = q_ld(pt + (int64_t)(j + 1) * pitch + x);
                    F4 pn = pold;
                    F4 rr = comp ? q_ld(ob(os, Q_RP) + ro) : F4{};
                    q_finish<V, false>(q_add(q_add(tx, ts), tmv), d_b, ob(os, Q_BETA) + ro, dt, sk ? sln : -1, srcf,
                                pn, rr);
                    q_store(P.p, slab, s, off, pn, sin);
                    q_track(acc[0], pn);
                    if (comp) {
                        q_store(P.rp, slab, s, off, rr, sin);
                        q_track(acc[4], rr);
                    }
                    // receiver traces of p after the step (acoustic.py:217-218)
                    rec_row(IO.rec, rcur, IO.n_rec, s * nm + m, x, IO.traces, IO.nt, n,
                            [&](int o) {
                                double r = 0.0;
#pragma unroll
                                for (int q = 0; q < Q3C; q++)
                                    if (q == o) r = (double)pn.e[q];
                                return r;
                            },
                            Q3C);
                    if (sample) {  // E = dx^3/2 [sum beta p^n p^{n+1} + sum rho v^2] (diagnostics.py:76-87)
                        double e[NCOMP] = {0.0, 0.0, 0.0, 0.0, 0.0};  // this (tile, slab) unit's share
                        const F4 vxo = q_ld(xv + ro);
#pragma unroll
                        for (int q = 0; q < Q3C; q++) {
                            const int xi = x + q;
                            const double a = vxo.e[q], b = vsn.e[q], g = m2.e[q];
                            e[0] += p64(P.e_beta, s, m, xi) * ((double)pold.e[q] * (double)pn.e[q]);
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
                in_.eplane[(int64_t)(F0 + i - 1) * (nm / TM) + tile] = a;
            }
        }
        gi += NI;
        gk += se - sb + 1;
    }
    unsigned int mask = 0;
    mask |= q_nonfinite(acc[0]) << P.p.bit;
    mask |= q_nonfinite(acc[1]) << P.vx.bit;
    mask |= q_nonfinite(acc[2]) << P.vs.bit;
    mask |= q_nonfinite(acc[3]) << P.vm.bit;
    if (comp) {
        mask |= q_nonfinite(acc[4]) << P.rp.bit;
        mask |= q_nonfinite(acc[5]) << P.rvx.bit;
        mask |= q_nonfinite(acc[6]) << P.rvs.bit;
        mask |= q_nonfinite(acc[7]) << P.rvm.bit;
    }
    record_failure(P.ctrl, n, mask);
    if constexpr (!SAMPLE) return;
    __threadfence();
    __syncthreads();
    __shared__ unsigned int is_last;
    // (edge + interior launches of one step share the counter: nb_total CTAs in all)
    const unsigned int nbt = in_.nb_total > 0 ? (unsigned int)in_.nb_total : gridDim.x;
    if (tid == 0) is_last = atomicAdd(IO.counter, 1u) == nbt - 1;
    __syncthreads();
    if (!is_last) return;
    // plane totals T[s] = sum_tile partial[s][tile], tiles in order (el3_energy_from_planes, hw_api.cu)
    const int tiles_all = nm / TM;
    for (int sp = tid; sp < ns; sp += (int)blockDim.x) {
        double t = __ldcg(&in_.eplane[(int64_t)sp * tiles_all]);
        for (int t2 = 1; t2 < tiles_all; t2++) t += __ldcg(&in_.eplane[(int64_t)sp * tiles_all + t2]);
        in_.etot[eidx * (int64_t)ns + sp] = t;
    }
    if (tid == 0) *IO.counter = 0u;
}

// ---------------------------------------------------------------- host side

bool ac3d_fused32_eligible(int64_t nx, int64_t nm, int64_t ns, int64_t pitch, int order, int max_smem) {
    if (order != 2 || nx % 128 != 0 || nx > Q3T * Q3C || pitch != nx || ns < 2) return false;
    const int64_t TM = Q3T * Q3C / nx;
    if (nm % TM != 0 || nm < 2) return false;
    return q3_bytes(nx) <= (size_t)max_smem;
}

template <int NXC, bool SAMPLE>
static void q3_attrs(int b) {
    void* fns[] = {(void*)k_ac3d_fused32<0, false, NXC, SAMPLE>, (void*)k_ac3d_fused32<3, false, NXC, SAMPLE>,
                   (void*)k_ac3d_fused32<6, false, NXC, SAMPLE>, (void*)k_ac3d_fused32<0, true, NXC, SAMPLE>,
                   (void*)k_ac3d_fused32<3, true, NXC, SAMPLE>,  (void*)k_ac3d_fused32<6, true, NXC, SAMPLE>};
    for (void* fn : fns) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
}

cudaError_t ac3d_fused32_prepare(int64_t nx) {
    const int b = (int)q3_bytes(nx);
    q3_attrs<0, false>(b);
    q3_attrs<0, true>(b);
    q3_attrs<512, false>(b);
    q3_attrs<512, true>(b);
    return cudaGetLastError();
}

template <int NXC, bool SAMPLE>
static void* q3_fn(int variant, bool rr) {
    return rr ? (variant == 0 ? (void*)k_ac3d_fused32<0, true, NXC, SAMPLE>
                              : (variant == 3 ? (void*)k_ac3d_fused32<3, true, NXC, SAMPLE>
                                              : (void*)k_ac3d_fused32<6, true, NXC, SAMPLE>))
              : (variant == 0 ? (void*)k_ac3d_fused32<0, false, NXC, SAMPLE>
                              : (variant == 3 ? (void*)k_ac3d_fused32<3, false, NXC, SAMPLE>
                                              : (void*)k_ac3d_fused32<6, false, NXC, SAMPLE>));
}

void launch_ac3d_fused32(int variant, const AcParams& P, const Ac3In& in, const StreamIO& IO, int nblocks, int64_t n,
                         double src, int sample, int64_t eidx, cudaStream_t st) {
    const bool rr = P.rho_x.sx == 0 && P.rho_s.sx == 0 && P.rho_m.sx == 0;
    const bool c512 = P.g.nx == 512 && P.g.pitch == 512;
    void* fn = c512 ? (sample ? q3_fn<512, true>(variant, rr) : q3_fn<512, false>(variant, rr))
                    : (sample ? q3_fn<0, true>(variant, rr) : q3_fn<0, false>(variant, rr));
    void* args[] = {(void*)&P, (void*)&in, (void*)&IO, (void*)&n, (void*)&src, (void*)&eidx};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nblocks);
    cfg.blockDim = dim3(Q3T);
    cfg.dynamicSmemBytes = q3_bytes(P.g.nx);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelExC(&cfg, fn, args);
}

}  // namespace hw
