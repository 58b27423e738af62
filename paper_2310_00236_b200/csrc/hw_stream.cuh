// hw_stream.cuh — helpers shared by the full-row streaming kernels (binary16 state):
// 8 cells per thread as four half2, shared-memory row taps, register slow-axis queues,
// write-through ghost stores, failure tracking and PDL entry.
#pragma once
#include <cuda_runtime.h>

#include "hw_common.cuh"
#include "hw_tma.cuh"

namespace hw {

constexpr int ECPT = 8;   // cells per thread

using EH2 = vec<16, 2>;
using EO2 = vops<16, 2>;

struct E8 {
    EH2 q[4];
};

__device__ __forceinline__ E8 e_ld8(const __half* p) {
    E8 r;
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    *reinterpret_cast<unsigned int*>(&r.q[0].h2) = u.x;
    *reinterpret_cast<unsigned int*>(&r.q[1].h2) = u.y;
    *reinterpret_cast<unsigned int*>(&r.q[2].h2) = u.z;
    *reinterpret_cast<unsigned int*>(&r.q[3].h2) = u.w;
    return r;
}

__device__ __forceinline__ void e_st8(__half* p, const E8& v) {
    uint4 u;
    u.x = *reinterpret_cast<const unsigned int*>(&v.q[0].h2);
    u.y = *reinterpret_cast<const unsigned int*>(&v.q[1].h2);
    u.z = *reinterpret_cast<const unsigned int*>(&v.q[2].h2);
    u.w = *reinterpret_cast<const unsigned int*>(&v.q[3].h2);
    *reinterpret_cast<uint4*>(p) = u;
}

__device__ __forceinline__ EH2 e_ld2(const __half* p) {
    EH2 r;
    r.h2 = *reinterpret_cast<const __half2*>(p);
    return r;
}

__device__ __forceinline__ E8 e_neg8(const E8& v) {
    E8 r;
#pragma unroll
    for (int j = 0; j < 4; j++) r.q[j] = vneg<16, 2>(v.q[j]);
    return r;
}

template <int ORDER>
__device__ __forceinline__ EH2 e_fold(const __half c[4], EH2 t0, EH2 t1, EH2 t2, EH2 t3) {
    EH2 inner = EO2::add(EO2::mul(vsplat<16, 2>(c[1]), t1), EO2::mul(vsplat<16, 2>(c[2]), t2));
    if (ORDER == 2) return inner;
    EH2 outer = EO2::add(EO2::mul(vsplat<16, 2>(c[0]), t0), EO2::mul(vsplat<16, 2>(c[3]), t3));
    return EO2::add(inner, outer);
}

// x derivative of 8 cells (periodic) from a shared row; to_int: shifts (-2..1) else (-1..2)
template <int ORDER>
__device__ __forceinline__ E8 e_xfold(const __half c[4], const __half* row, int x, int xl, int xr, bool to_int) {
    EH2 Q[6];
    Q[0] = e_ld2(row + xl);
    const E8 own = e_ld8(row + x);
#pragma unroll
    for (int j = 0; j < 4; j++) Q[j + 1] = own.q[j];
    Q[5] = e_ld2(row + xr);
    EH2 S[5];
#pragma unroll
    for (int j = 0; j < 5; j++) S[j] = vshift<16, 2>(Q[j], Q[j + 1]);
    E8 r;
#pragma unroll
    for (int j = 0; j < 4; j++)
        r.q[j] = to_int ? e_fold<ORDER>(c, Q[j], S[j], Q[j + 1], S[j + 1]) : e_fold<ORDER>(c, S[j], Q[j + 1], S[j + 1], Q[j + 2]);
    return r;
}

// slow taps from a 4-deep register queue (q[k] = row base + k) for each of the 4 pairs
template <int ORDER>
__device__ __forceinline__ E8 e_sfold(const __half c[4], const E8& a, const E8& b, const E8& d, const E8& e) {
    E8 r;
#pragma unroll
    for (int j = 0; j < 4; j++) r.q[j] = e_fold<ORDER>(c, a.q[j], b.q[j], d.q[j], e.q[j]);
    return r;
}

__device__ __forceinline__ unsigned int e_nonfinite(__half2 acc) {  // |max| is inf or NaN
    const unsigned int b = *reinterpret_cast<const unsigned int*>(&acc);
    return (((b & 0x7c00u) == 0x7c00u) || ((b & 0x7c000000u) == 0x7c000000u)) ? 1u : 0u;
}

// ring rows below the first ghost slab are never consumed (r < y0); keep the copy in bounds
__device__ __forceinline__ int64_t e_row(int r) { return (int64_t)(r < -G ? -G : r); }

__device__ __forceinline__ void e_track(__half2& acc, const E8& v) {
#pragma unroll
    for (int j = 0; j < 4; j++) acc = __hmax2_nan(acc, __habs2(v.q[j].h2));
}

// store one row (8 cells per thread) of field f and its write-through ghost rows
__device__ __forceinline__ void e_store_row(const FieldView& f, int64_t pitch, int s, int x, const E8& v) {
    __half* base = reinterpret_cast<__half*>(f.base);
    e_st8(base + (int64_t)s * pitch + x, v);
    if ((f.gtop | f.gbot) == GHOST_NONE) return;
    const int n = (int)f.rows;
    if (f.gtop == GHOST_PERIODIC && s >= n - G) e_st8(base + (int64_t)(s - n) * pitch + x, v);
    if (f.gbot == GHOST_PERIODIC && s < G) e_st8(base + (int64_t)(n + s) * pitch + x, v);
    if ((f.gtop | f.gbot) & GHOST_IMAGE) {
        const E8 w = f.odd ? e_neg8(v) : v;
        const int sg = (int)f.row0 + s, ng = (int)f.nglob;
        if (f.gtop == GHOST_IMAGE) {
            const int k1 = f.half_s ? -sg - 1 : -sg;
            if (k1 < 0 && k1 >= -G) e_st8(base + (int64_t)(k1 - (int)f.row0) * pitch + x, w);
        }
        if (f.gbot == GHOST_IMAGE) {
            const int k2 = f.half_s ? 2 * ng - 1 - sg : 2 * ng - 2 - sg;
            if (k2 >= ng && k2 < ng + G) e_st8(base + (int64_t)(k2 - (int)f.row0) * pitch + x, w);
        }
    }
}

// Programmatic dependent launch: the next phase's grid may launch while this one runs
// (its CTAs take SMs as ours retire); it waits here until every prior write is visible.
__device__ __forceinline__ void e_pdl_enter() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

__device__ __forceinline__ double e_pick(const E8& v, int o) {  // register select, no local memory
    double r = 0.0;
#pragma unroll
    for (int j = 0; j < ECPT; j++)
        if (j == o) r = (double)__half2float(v.q[j >> 1].e[j & 1]);
    return r;
}

// increment + advance for one pair, division by a row-uniform divisor through its
// verified reciprocal (DIV_CHEAP): the same ops as finish() (stepping.py:58-98,
// efsum.py:100-121), without the per-pair plane load and mode dispatch
template <int V>
__device__ __forceinline__ void e_finish_rc(EH2 rhs, float rc, __half2 dt2, int src_lane, __half srch, EH2& u,
                                            EH2& t) {
    if (src_lane == 0) rhs.e[0] = __hadd_rn(rhs.e[0], srch);
    else if (src_lane == 1) rhs.e[1] = __hadd_rn(rhs.e[1], srch);
    const float2 fx = __half22float2(rhs.h2);
    EH2 x;
    x.h2 = __hmul2_rn(__floats2half2_rn(__fmul_rn(fx.x, rc), __fmul_rn(fx.y, rc)), dt2);
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

// planes constant along x (constant, slow-layered, or per (slow, mid) row in 3D)
__host__ __device__ __forceinline__ bool e_rowdiv(const PlaneView& v) { return v.div_mode == DIV_CHEAP && v.sx == 0; }
__device__ __forceinline__ float e_rcp_at(const PlaneView& v, int64_t s, int64_t m) {
    return __ldg(v.rcp + s * v.ss + m * v.sm);
}
__device__ __forceinline__ EH2 e_val_at(const PlaneView& v, int64_t s, int64_t m) {
    return vsplat<16, 2>(__ldg(reinterpret_cast<const __half*>(v.p) + s * v.ss + m * v.sm));
}

// row-uniform binary16 plane value at slow row r (plane strides (ss, 0, 0))
__device__ __forceinline__ EH2 e_rowval(const PlaneView& pv, int64_t r) {
    return vsplat<16, 2>(__ldg(reinterpret_cast<const __half*>(pv.p) + r * pv.ss));
}

// ---- mid-axis tiles (3D streaming kernels)
__device__ __forceinline__ int a3_wrap(int r, int n) { return r < 0 ? r + n : (r >= n ? r - n : r); }

// TMA copy of mid rows [a, b) (periodic) of slab s into dst (row stride = pitch)
__device__ __forceinline__ void a3_rows(__half* dst, const __half* fbase, int64_t slab, int64_t s, int a, int b,
                                        int nm, int64_t pitch, uint64_t* bar) {
    const __half* sb = fbase + s * slab;
    for (int r = a; r < b;) {
        const int rr = a3_wrap(r, nm);
        const int seg = min(b - r, nm - rr);
        tma_load_1d(dst, sb + (int64_t)rr * pitch, (uint32_t)(seg * pitch * sizeof(__half)), bar);
        dst += (int64_t)seg * pitch;
        r += seg;
    }
}

// division by a binary16 divisor pair staged in shared memory (same three modes as finish())
__device__ __forceinline__ EH2 a3_div(EH2 x, EH2 b, int mode) {
    if (mode == DIV_CHEAP) {
        const float r[2] = {__frcp_rn(__half2float(b.e[0])), __frcp_rn(__half2float(b.e[1]))};
        return vdiv_cheap<2>(x, r);
    }
    if (mode == DIV_FAST) return EO2::div(x, b);
    return EO2::div_ieee(x, b);
}

// finish() with the divisor values given (staged per-cell plane)
template <int V>
__device__ __forceinline__ void a3_finish(EH2 rhs, EH2 b, int mode, __half dt, int src_lane, double src, EH2& u,
                                          EH2& t) {
    EH2 xv = rhs;
    if (src_lane >= 0 && src != 0.0) xv.e[src_lane] = lane<16>::add(xv.e[src_lane], lane<16>::from_f64(src));
    xv = EO2::mul(a3_div(xv, b, mode), vsplat<16, 2>(dt));
    if (V == 0) {
        u = EO2::add(u, xv);
        return;
    }
    const EH2 r = EO2::add(t, xv);
    const EH2 sm = EO2::add(u, r);
    if (V == 3) {
        t = EO2::sub(r, EO2::sub(sm, u));
    } else {
        const EH2 pa = EO2::sub(sm, r);
        const EH2 pb = EO2::sub(sm, pa);
        t = EO2::add(EO2::sub(u, pa), EO2::sub(r, pb));
    }
    u = sm;
}

// row store at element offset off = s * pitch + x; rows away from the slow-axis ends skip
// the write-through ghost logic
__device__ __forceinline__ void e2_store(bool inner, const FieldView& f, int64_t off, int64_t pitch, int s, int x,
                                         const E8& v) {
    if (inner) e_st8(reinterpret_cast<__half*>(f.base) + off, v);
    else e_store_row(f, pitch, s, x, v);
}

// finish() without a divisor (stresses, elastic.py:210-238): source (round_U(s), lane
// src_lane) before x dt, then the advance -- the same ops as finish<16, 16, 2>
template <int V>
__device__ __forceinline__ void e2_finish_nd(EH2 rhs, __half2 dt2, int src_lane, __half srch, EH2& u, EH2& t) {
    if (src_lane == 0) rhs.e[0] = __hadd_rn(rhs.e[0], srch);
    else if (src_lane == 1) rhs.e[1] = __hadd_rn(rhs.e[1], srch);
    EH2 x;
    x.h2 = __hmul2_rn(rhs.h2, dt2);
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

// point source: add round_U(s) to the right-hand side of the source cell (the first op of
// finish(), stepping.py:71-80); called only on the source row (warp-uniform branch)
__device__ __forceinline__ void e2_add_src(EH2 r[4], bool here, int sj, int sln, __half srch) {
#pragma unroll
    for (int j = 0; j < 4; j++)
        if (here && j == sj) {
            if (sln == 0) r[j].e[0] = __hadd_rn(r[j].e[0], srch);
            else r[j].e[1] = __hadd_rn(r[j].e[1], srch);
        }
}

}  // namespace hw
