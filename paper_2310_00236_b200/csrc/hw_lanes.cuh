// hw_lanes.cuh — correctly rounded lane arithmetic for sm_100a.
//
// Device restatement of the reference precision model (precision.py:287-339,
// Lane.add/sub/mul/div): every operation is computed once and rounded once (RNE)
// into the lane.  binary16 uses the native IEEE fp16 ALU (__hadd_rn & co., which
// also forbid mul+add contraction); binary32/binary64 use the explicit _rn
// intrinsics.  Division is never __hdiv (approximate): binary16 quotients are the
// binary32 correctly rounded quotient rounded once more to binary16, exact by the
// 2p+2 double-rounding bound the reference relies on (precision.py:8-14).
// Conversions: widening is exact; narrowing is a single direct cvt.rn
// (demote, precision.py:272-284).  Build with -fmad=false as a second guard.
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

namespace hw {

template <int L> struct lane;

template <> struct lane<16> {
    using T = __half;
    static __device__ __forceinline__ T add(T a, T b) { return __hadd_rn(a, b); }
    static __device__ __forceinline__ T sub(T a, T b) { return __hsub_rn(a, b); }
    static __device__ __forceinline__ T mul(T a, T b) { return __hmul_rn(a, b); }
    // Correctly rounded binary16 quotient without the IEEE-division slow path:
    // q0 = a * rcp(b), one exact FMA residual, one FMA correction, then a single
    // RNE to binary16.  Exhaustively verified bit-identical to
    // __float2half_rn(__fdiv_rn(a, b)) for every binary16 a and every finite
    // nonzero binary16 b (hw_selftest_div16, tests/test_gpu_parity.py); zero or
    // non-finite divisors take div_ieee (the host picks per medium plane).
    static __device__ __forceinline__ T div(T a, T b) {
        const float fa = __half2float(a), fb = __half2float(b);
        float r;
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(fb));
        const float q0 = __fmul_rn(fa, r);
        const float e = __fmaf_rn(-fb, q0, fa);
        const float q1 = __fmaf_rn(e, r, q0);
        const bool keep = (e == 0.0f) || !(fabsf(q0) < INFINITY);
        return __float2half_rn(keep ? q0 : q1);
    }
    static __device__ __forceinline__ T div_ieee(T a, T b) {
        return __float2half_rn(__fdiv_rn(__half2float(a), __half2float(b)));
    }
    static __device__ __forceinline__ bool finite(T a) {
        return (__half_as_ushort(a) & 0x7c00u) != 0x7c00u;
    }
    static __device__ __forceinline__ T neg(T a) { return __ushort_as_half(__half_as_ushort(a) ^ 0x8000u); }
    static __device__ __forceinline__ double to_f64(T a) { return (double)__half2float(a); }
    static __device__ __forceinline__ T from_f64(double x) { return __double2half(x); }  // cvt.rn.f16.f64
    static __device__ __forceinline__ T zero() { return __ushort_as_half(0); }
};

// IEEE quotients with zero dividends answered inline: __fdiv_rn / __ddiv_rn send a zero dividend
// down their slow path (a subroutine call), and wavefields are zero wherever the wave has not
// arrived.  +-0 / b for finite nonzero b is the signed zero (identical bits).
template <> struct lane<32> {
    using T = float;
    static __device__ __forceinline__ T add(T a, T b) { return __fadd_rn(a, b); }
    static __device__ __forceinline__ T sub(T a, T b) { return __fsub_rn(a, b); }
    static __device__ __forceinline__ T mul(T a, T b) { return __fmul_rn(a, b); }
    static __device__ __forceinline__ T div(T a, T b) { return div_ieee(a, b); }
    static __device__ __forceinline__ T div_ieee(T a, T b) {
        if (a == 0.0f && fabsf(b) < INFINITY && b != 0.0f)
            return __uint_as_float((__float_as_uint(a) ^ __float_as_uint(b)) & 0x80000000u);
        return __fdiv_rn(a, b);
    }
    static __device__ __forceinline__ bool finite(T a) {
        return (__float_as_uint(a) & 0x7f800000u) != 0x7f800000u;
    }
    static __device__ __forceinline__ T neg(T a) { return __uint_as_float(__float_as_uint(a) ^ 0x80000000u); }
    static __device__ __forceinline__ double to_f64(T a) { return (double)a; }
    static __device__ __forceinline__ T from_f64(double x) { return __double2float_rn(x); }
    static __device__ __forceinline__ T zero() { return 0.0f; }
};

template <> struct lane<64> {
    using T = double;
    static __device__ __forceinline__ T add(T a, T b) { return __dadd_rn(a, b); }
    static __device__ __forceinline__ T sub(T a, T b) { return __dsub_rn(a, b); }
    static __device__ __forceinline__ T mul(T a, T b) { return __dmul_rn(a, b); }
    static __device__ __forceinline__ T div(T a, T b) { return div_ieee(a, b); }
    static __device__ __forceinline__ T div_ieee(T a, T b) {
        if (a == 0.0 && fabs(b) < INFINITY && b != 0.0)
            return __longlong_as_double((__double_as_longlong(a) ^ __double_as_longlong(b)) &
                                        (long long)0x8000000000000000ull);
        return __ddiv_rn(a, b);
    }
    static __device__ __forceinline__ bool finite(T a) {
        return (__double_as_longlong(a) & 0x7ff0000000000000ll) != 0x7ff0000000000000ll;
    }
    static __device__ __forceinline__ T neg(T a) {
        return __longlong_as_double(__double_as_longlong(a) ^ (long long)0x8000000000000000ull);
    }
    static __device__ __forceinline__ double to_f64(T a) { return a; }
    static __device__ __forceinline__ T from_f64(double x) { return x; }
    static __device__ __forceinline__ T zero() { return 0.0; }
};

// Single-rounding conversion between lanes (UpdatePipeline._convert, stepping.py:32-45).
template <int LT, int LF> struct cvt_t {
    static __device__ __forceinline__ typename lane<LT>::T go(typename lane<LF>::T a) {
        return lane<LT>::from_f64(lane<LF>::to_f64(a));  // widen exactly, then one cvt.rn
    }
};
template <int L> struct cvt_t<L, L> {
    static __device__ __forceinline__ typename lane<L>::T go(typename lane<L>::T a) { return a; }
};
template <> struct cvt_t<32, 16> {
    static __device__ __forceinline__ float go(__half a) { return __half2float(a); }
};
template <> struct cvt_t<16, 32> {
    static __device__ __forceinline__ __half go(float a) { return __float2half_rn(a); }
};
template <int LT, int LF>
__device__ __forceinline__ typename lane<LT>::T cvt(typename lane<LF>::T a) { return cvt_t<LT, LF>::go(a); }

// ---------------------------------------------------------------- W-wide vectors
// W consecutive x cells handled by one thread.  W = 2 maps binary16 onto the
// packed half2 ALU (two correctly rounded results per instruction, identical
// bits to two scalar ops) and gives 4/8/16-byte coalesced accesses.

template <int L, int W> struct vec {
    typename lane<L>::T e[W];
};
// binary16 pairs live in one 32-bit register as __half2 so the packed ALU ops
// need no repacking; e[] aliases the two halves for per-element access.
template <> struct vec<16, 2> {
    union {
        __half2 h2;
        __half e[2];
    };
    __device__ __forceinline__ vec() { *reinterpret_cast<unsigned int*>(&h2) = 0u; }
    __device__ __forceinline__ vec(const vec& o) { *reinterpret_cast<unsigned int*>(&h2) = *reinterpret_cast<const unsigned int*>(&o.h2); }
    __device__ __forceinline__ vec& operator=(const vec& o) {
        *reinterpret_cast<unsigned int*>(&h2) = *reinterpret_cast<const unsigned int*>(&o.h2);
        return *this;
    }
};

template <int L, int W> struct vops {
    using V = vec<L, W>;
    using ln = lane<L>;
    static __device__ __forceinline__ V add(V a, V b) { V r; _Pragma("unroll") for (int i = 0; i < W; i++) r.e[i] = ln::add(a.e[i], b.e[i]); return r; }
    static __device__ __forceinline__ V sub(V a, V b) { V r; _Pragma("unroll") for (int i = 0; i < W; i++) r.e[i] = ln::sub(a.e[i], b.e[i]); return r; }
    static __device__ __forceinline__ V mul(V a, V b) { V r; _Pragma("unroll") for (int i = 0; i < W; i++) r.e[i] = ln::mul(a.e[i], b.e[i]); return r; }
    static __device__ __forceinline__ V div(V a, V b) { V r; _Pragma("unroll") for (int i = 0; i < W; i++) r.e[i] = ln::div(a.e[i], b.e[i]); return r; }
    static __device__ __forceinline__ V div_ieee(V a, V b) { V r; _Pragma("unroll") for (int i = 0; i < W; i++) r.e[i] = ln::div_ieee(a.e[i], b.e[i]); return r; }
};

template <> struct vops<16, 2> {
    using V = vec<16, 2>;
    static __device__ __forceinline__ V mk(__half2 x) { V r; r.h2 = x; return r; }
    static __device__ __forceinline__ V add(V a, V b) { return mk(__hadd2_rn(a.h2, b.h2)); }
    static __device__ __forceinline__ V sub(V a, V b) { return mk(__hsub2_rn(a.h2, b.h2)); }
    static __device__ __forceinline__ V mul(V a, V b) { return mk(__hmul2_rn(a.h2, b.h2)); }
    static __device__ __forceinline__ V div(V a, V b) {
        V r;
        r.e[0] = lane<16>::div(a.e[0], b.e[0]);
        r.e[1] = lane<16>::div(a.e[1], b.e[1]);
        return r;
    }
    static __device__ __forceinline__ V div_ieee(V a, V b) {
        V r;
        r.e[0] = lane<16>::div_ieee(a.e[0], b.e[0]);
        r.e[1] = lane<16>::div_ieee(a.e[1], b.e[1]);
        return r;
    }
};

// Binary16 division by a divisor whose reciprocal rcp = __frcp_rn(b) makes
// fl16(fl32(a * rcp)) == fl16(a / b) for EVERY binary16 a; which divisors qualify
// is decided exhaustively on the device (k_cheap_div_table in hw_api.cu).
template <int W>
__device__ __forceinline__ vec<16, W> vdiv_cheap(vec<16, W> a, const float* rcp) {
    vec<16, W> r;
    if constexpr (W == 2) {
        const float2 f = __half22float2(a.h2);
        r.h2 = __floats2half2_rn(__fmul_rn(f.x, rcp[0]), __fmul_rn(f.y, rcp[1]));
    } else {
#pragma unroll
        for (int i = 0; i < W; i++) r.e[i] = __float2half_rn(__fmul_rn(__half2float(a.e[i]), rcp[i]));
    }
    return r;
}

template <int L, int W>
__device__ __forceinline__ vec<L, W> vsplat(typename lane<L>::T x) {
    if constexpr (L == 16 && W == 2) {
        vec<16, 2> r;
        r.h2 = __half2half2(x);
        return r;
    }
    vec<L, W> r;
#pragma unroll
    for (int i = 0; i < W; i++) r.e[i] = x;
    return r;
}

template <int LT, int LF, int W>
__device__ __forceinline__ vec<LT, W> vcvt(vec<LF, W> a) {
    vec<LT, W> r;
#pragma unroll
    for (int i = 0; i < W; i++) r.e[i] = cvt<LT, LF>(a.e[i]);
    return r;
}

template <int L, int W>
__device__ __forceinline__ vec<L, W> vneg(vec<L, W> a) {
    if constexpr (L == 16 && W == 2) {
        vec<16, 2> r;
        r.h2 = __halves2half2(lane<16>::neg(__low2half(a.h2)), lane<16>::neg(__high2half(a.h2)));
        return r;
    }
    vec<L, W> r;
#pragma unroll
    for (int i = 0; i < W; i++) r.e[i] = lane<L>::neg(a.e[i]);
    return r;
}

// (a.e[W-1], b.e[0], ...): the vector shifted by one cell between neighbours a|b
template <int L, int W>
__device__ __forceinline__ vec<L, W> vshift(vec<L, W> a, vec<L, W> b) {
    if constexpr (L == 16 && W == 2) {
        vec<16, 2> r;
        r.h2 = __halves2half2(__high2half(a.h2), __low2half(b.h2));  // one PRMT
        return r;
    }
    vec<L, W> r;
    r.e[0] = a.e[W - 1];
#pragma unroll
    for (int i = 1; i < W; i++) r.e[i] = b.e[i - 1];
    return r;
}

// per-element non-finite mask bit
template <int L, int W>
__device__ __forceinline__ bool vfinite(vec<L, W> a) {
    if constexpr (L == 16 && W == 2) {
        const unsigned int b = *reinterpret_cast<const unsigned int*>(&a.h2);
        return ((b & 0x7c00u) != 0x7c00u) && ((b & 0x7c000000u) != 0x7c000000u);
    }
    bool ok = true;
#pragma unroll
    for (int i = 0; i < W; i++) ok = ok && lane<L>::finite(a.e[i]);
    return ok;
}

template <int L, int W>
__device__ __forceinline__ vec<L, W> vload(const typename lane<L>::T* p) {
    vec<L, W> r;
    if constexpr (W == 1) {
        r.e[0] = p[0];
    } else if constexpr (L == 16) {
        r.h2 = *reinterpret_cast<const __half2*>(p);
    } else if constexpr (L == 32) {
        float2 x = *reinterpret_cast<const float2*>(p);
        r.e[0] = x.x;
        r.e[1] = x.y;
    } else {
        double2 x = *reinterpret_cast<const double2*>(p);
        r.e[0] = x.x;
        r.e[1] = x.y;
    }
    return r;
}

// Read-only (non-coherent) load: for fields no thread writes during the kernel,
// so the compiler may batch them ahead of the stores to other fields.
template <int L, int W>
__device__ __forceinline__ vec<L, W> vload_nc(const typename lane<L>::T* p) {
    vec<L, W> r;
    if constexpr (W == 1) {
        r.e[0] = __ldg(p);
    } else if constexpr (L == 16) {
        r.h2 = __ldg(reinterpret_cast<const __half2*>(p));
    } else if constexpr (L == 32) {
        float2 x = __ldg(reinterpret_cast<const float2*>(p));
        r.e[0] = x.x;
        r.e[1] = x.y;
    } else {
        double2 x = __ldg(reinterpret_cast<const double2*>(p));
        r.e[0] = x.x;
        r.e[1] = x.y;
    }
    return r;
}

template <int L, int W>
__device__ __forceinline__ void vstore(typename lane<L>::T* p, vec<L, W> v) {
    if constexpr (W == 1) {
        p[0] = v.e[0];
    } else if constexpr (L == 16) {
        *reinterpret_cast<__half2*>(p) = v.h2;
    } else if constexpr (L == 32) {
        *reinterpret_cast<float2*>(p) = make_float2(v.e[0], v.e[1]);
    } else {
        *reinterpret_cast<double2*>(p) = make_double2(v.e[0], v.e[1]);
    }
}

}  // namespace hw
