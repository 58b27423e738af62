// hw_common.cuh — device data layout and shared step machinery.
//
// HBM layout:
//   * every field is [rows + 2G][nm][pitch] in its update-lane storage type, with
//     G = 3 ghost slabs on each end of the slow axis and pitch a multiple of 32
//     elements (64 B rows for fp16); `base` points at (s=0, m=0, x=0).
//   * x and mid are periodic through index arithmetic; the slow axis reads its
//     ghost slabs, which encode the boundary condition and are kept current by the
//     kernel that writes the field ("write-through ghosts": periodic wrap copies or
//     free-surface image rows with a parity sign flip, stencil.py:121-144), or by
//     the NCCL halo exchange at slab boundaries of a multi-GPU job.
//   * medium planes are strided views: constant (0,0,0), slow-layered (1,0,0) or
//     full (nm*nx, nx, 1), so layered media cost no HBM traffic per cell.
#pragma once
#include <limits.h>
#include <stdint.h>
#include "hw_lanes.cuh"

namespace hw {

constexpr int G = 3;          // ghost slabs per side: 4th-order staggered reach (2) + the fused
                              // kernel's redundant vy halo rows, which read p rows -3 .. L+2 (slab mode)
constexpr int NCOMP = 5;      // energy partial components per block
constexpr int BLOCK = 256;    // threads per block for the phase kernels

enum GhostMode { GHOST_NONE = 0, GHOST_PERIODIC = 1, GHOST_IMAGE = 2 };

struct FieldView {
    void* base;       // element (s=0, m=0, x=0) of this rank's slab
    int64_t rows;     // local slow-axis extent
    int64_t row0;     // global slow index of local row 0 (slab decomposition)
    int64_t nglob;    // global slow-axis extent of the field (ns or ns+1)
    int32_t gtop;     // GhostMode of the top ghost slabs (NONE = filled by the halo exchange)
    int32_t gbot;     // GhostMode of the bottom ghost slabs
    int32_t half_s;   // field sits on the half-offset slow sub-grid
    int32_t odd;      // free-surface parity: image rows are negated
    int32_t bit;      // external field index (check_finite order) for failure masks
    int32_t pad;
};

struct Geom {
    int64_t nx, nm, pitch;
    int64_t slab;     // elements per slow index = nm * pitch
};

// Division mode of a divisor plane (chosen on the host per plane, see hw_api.cu):
enum DivMode {
    DIV_NONE = 0,
    DIV_FAST = 1,   // branch-free exact binary16 division (finite nonzero divisors)
    DIV_IEEE = 2,   // __fdiv_rn / __ddiv_rn path
    DIV_CHEAP = 3,  // binary16: fl16(a * rcp), every plane value verified exhaustively
};

struct PlaneView {    // lane-rounded medium plane (storage type of its lane)
    const void* p;
    const float* rcp; // __frcp_rn of each binary16 value (same strides), DIV_CHEAP planes
    int64_t ss, sm, sx;
    int32_t div_mode;
    int32_t pad;
};

// Lane constants converted once on the host (exact: the values are already
// rounded into their lane): taps c1..c4 in the stencil lane, dt in the update lane.
struct LaneConsts {
    uint16_t h[5];
    float f[5];
    double d[5];
};

template <int L>
__device__ __forceinline__ typename lane<L>::T lconst(const LaneConsts& c, int i) {
    if constexpr (L == 16) return __ushort_as_half(c.h[i]);
    else if constexpr (L == 32) return c.f[i];
    else return c.d[i];
}

struct Plane64 {      // fp64 medium plane for the energy functionals
    const double* p;
    int64_t ss, sm, sx;
};

struct Ctrl {         // device-side run control
    int64_t fail_step;      // first local step index with a non-finite write (INT64_MAX if none)
    unsigned int fail_mask; // external field bits recorded at that step
    unsigned int pad;
    int64_t gfail_step;     // first failing step of ANY rank known so far (NCCL transport: min-allreduced
                            // after every step; INT64_MAX otherwise)
};

template <typename T>
__device__ __forceinline__ T* frow(const FieldView& f, const Geom& g, int64_t s, int64_t m) {
    return reinterpret_cast<T*>(f.base) + s * g.slab + m * g.pitch;
}

template <int W>
__device__ __forceinline__ void prcp(const PlaneView& pv, int64_t s, int64_t m, int64_t x, float r[W]) {
    const float* p = pv.rcp + s * pv.ss + m * pv.sm;
    if (pv.sx == 0) {
#pragma unroll
        for (int i = 0; i < W; i++) r[i] = p[0];
    } else {
#pragma unroll
        for (int i = 0; i < W; i++) r[i] = p[x + i];
    }
}

template <int L, int W>
__device__ __forceinline__ vec<L, W> pload(const PlaneView& pv, int64_t s, int64_t m, int64_t x) {
    using T = typename lane<L>::T;
    const T* p = reinterpret_cast<const T*>(pv.p) + s * pv.ss + m * pv.sm;
    if (pv.sx == 0) return vsplat<L, W>(p[0]);
    return vload<L, W>(p + x);
}

__device__ __forceinline__ double p64(const Plane64& pv, int64_t s, int64_t m, int64_t x) {
    return pv.p[s * pv.ss + m * pv.sm + x * pv.sx];
}

__device__ __forceinline__ int64_t wrap(int64_t i, int64_t n) {
    return i < 0 ? i + n : (i >= n ? i - n : i);
}

// Four x taps around the W cells starting at x (periodic x, ddx_work stencil.py:98-107).
// to_int: input on the half grid, shifts (-2,-1,0,1); else (-1,0,1,2).
template <int LU, int W>
__device__ __forceinline__ void xtaps(const typename lane<LU>::T* row, int64_t x, int64_t nx, bool to_int,
                                      vec<LU, W> t[4]) {
    if constexpr (W == 2) {
        vec<LU, W> a = vload<LU, W>(row + wrap(x - 2, nx));
        vec<LU, W> b = vload<LU, W>(row + x);
        vec<LU, W> c = vload<LU, W>(row + wrap(x + 2, nx));
        if (to_int) {
            t[0] = a; t[1] = vshift(a, b); t[2] = b; t[3] = vshift(b, c);
        } else {
            t[0] = vshift(a, b); t[1] = b; t[2] = vshift(b, c); t[3] = c;
        }
    } else {
        int64_t b0 = to_int ? x - 2 : x - 1;
#pragma unroll
        for (int j = 0; j < 4; j++) t[j].e[0] = row[wrap(b0 + j, nx)];
    }
}

// Fixed fold (stencil.py:72-79) in the stencil lane; order 2 keeps the inner pair.
// Taps arrive in the update lane and enter the stencil lane through one rounding
// (UpdatePipeline.to_stencil, stepping.py:39-41; identity when the lanes agree).
template <int LS, int LU, int W>
__device__ __forceinline__ vec<LS, W> fold(const typename lane<LS>::T c[4], const vec<LU, W> tu[4], int order) {
    using O = vops<LS, W>;
    vec<LS, W> t1 = vcvt<LS, LU, W>(tu[1]), t2 = vcvt<LS, LU, W>(tu[2]);
    vec<LS, W> inner = O::add(O::mul(vsplat<LS, W>(c[1]), t1), O::mul(vsplat<LS, W>(c[2]), t2));
    if (order == 2) return inner;
    vec<LS, W> t0 = vcvt<LS, LU, W>(tu[0]), t3 = vcvt<LS, LU, W>(tu[3]);
    vec<LS, W> outer = O::add(O::mul(vsplat<LS, W>(c[0]), t0), O::mul(vsplat<LS, W>(c[3]), t3));
    return O::add(inner, outer);
}

// Slow-axis taps of field f landing on row s (ghost slabs hold wrap / images).
template <int LU, int W>
__device__ __forceinline__ void staps(const FieldView& f, const Geom& g, int64_t s, int64_t m, int64_t x,
                                      bool to_int, int order, vec<LU, W> t[4]) {
    using T = typename lane<LU>::T;
    int64_t b0 = to_int ? s - 2 : s - 1;
#pragma unroll
    for (int j = 0; j < 4; j++) {
        if (order == 2 && (j == 0 || j == 3)) continue;
        t[j] = vload<LU, W>(frow<T>(f, g, b0 + j, m) + x);
    }
    if (order == 2) { t[0] = t[1]; t[3] = t[2]; }
}

// Mid-axis taps (3D, periodic).
template <int LU, int W>
__device__ __forceinline__ void mtaps(const FieldView& f, const Geom& g, int64_t s, int64_t m, int64_t x,
                                      bool to_int, int order, vec<LU, W> t[4]) {
    using T = typename lane<LU>::T;
    int64_t b0 = to_int ? m - 2 : m - 1;
#pragma unroll
    for (int j = 0; j < 4; j++) {
        if (order == 2 && (j == 0 || j == 3)) continue;
        t[j] = vload<LU, W>(frow<T>(f, g, s, wrap(b0 + j, g.nm)) + x);
    }
    if (order == 2) { t[0] = t[1]; t[3] = t[2]; }
}

// ---------------------------------------------------------------- per-thread addressing
// Offsets computed once per thread; every tap is then base + off + constant.
struct Cell {
    int64_t off;     // (s, m, x) element offset from a field's base
    int64_t xo[5];   // x offsets of x-2 .. x+2 relative to x (periodic wrap folded in)
    int64_t mo[5];   // mid-axis offsets of m-2 .. m+2 relative to m (periodic wrap folded in)
    int64_t slab;    // slow-axis stride
};

__device__ __forceinline__ Cell make_cell(const Geom& g, int64_t s, int64_t m, int64_t x) {
    Cell c;
    c.off = s * g.slab + m * g.pitch + x;
    c.slab = g.slab;
#pragma unroll
    for (int j = 0; j < 5; j++) c.xo[j] = wrap(x - 2 + j, g.nx) - x;
#pragma unroll
    for (int j = 0; j < 5; j++) c.mo[j] = (wrap(m - 2 + j, g.nm) - m) * g.pitch;
    return c;
}

template <typename T>
__device__ __forceinline__ const T* fptr(const FieldView& f, const Cell& c) {
    return reinterpret_cast<const T*>(f.base) + c.off;
}

// Tap loaders.  Every field they read is read-only within the kernel that calls
// them (velocity kernels read p / stresses, pressure-stress kernels read v), so
// they use the non-coherent path.
// x taps relative to p = &field[s][m][x]
template <int LU, int W>
__device__ __forceinline__ void xtaps_c(const typename lane<LU>::T* p, const Cell& c, bool to_int, vec<LU, W> t[4]) {
    if constexpr (W == 2) {
        vec<LU, W> a = vload_nc<LU, W>(p + c.xo[0]);
        vec<LU, W> b = vload_nc<LU, W>(p);
        vec<LU, W> d = vload_nc<LU, W>(p + c.xo[4]);
        if (to_int) {
            t[0] = a; t[1] = vshift(a, b); t[2] = b; t[3] = vshift(b, d);
        } else {
            t[0] = vshift(a, b); t[1] = b; t[2] = vshift(b, d); t[3] = d;
        }
    } else {
        const int b0 = to_int ? 0 : 1;
#pragma unroll
        for (int j = 0; j < 4; j++) t[j].e[0] = __ldg(p + c.xo[b0 + j]);
    }
}

template <int LU, int W>
__device__ __forceinline__ void staps_c(const typename lane<LU>::T* p, const Cell& c, bool to_int, int order,
                                        vec<LU, W> t[4]) {
    const int64_t b0 = to_int ? -2 : -1;
#pragma unroll
    for (int j = 0; j < 4; j++) {
        if (order == 2 && (j == 0 || j == 3)) continue;
        t[j] = vload_nc<LU, W>(p + (b0 + j) * c.slab);
    }
    if (order == 2) { t[0] = t[1]; t[3] = t[2]; }
}

template <int LU, int W>
__device__ __forceinline__ void mtaps_c(const typename lane<LU>::T* p, const Cell& c, bool to_int, int order,
                                        vec<LU, W> t[4]) {
    const int b0 = to_int ? 0 : 1;
#pragma unroll
    for (int j = 0; j < 4; j++) {
        if (order == 2 && (j == 0 || j == 3)) continue;
        t[j] = vload_nc<LU, W>(p + c.mo[b0 + j]);
    }
    if (order == 2) { t[0] = t[1]; t[3] = t[2]; }
}

// UpdatePipeline.increment (stepping.py:58-80) + .advance (stepping.py:82-98,
// efsum.py:100-121) for W cells.  src_lane >= 0 marks the element holding the
// point source, injected as round_U(src) before the division when src != 0.
template <int LS, int LU, int W>
__device__ __forceinline__ void finish(vec<LS, W> rhs, const PlaneView* div, int64_t s, int64_t m, int64_t x,
                                       typename lane<LU>::T dt, int variant, int src_lane, double src,
                                       vec<LU, W>& u, vec<LU, W>& t) {
    using O = vops<LU, W>;
    using ln = lane<LU>;
    vec<LU, W> xv = vcvt<LU, LS, W>(rhs);
    if (src_lane >= 0 && src != 0.0) {
#pragma unroll
        for (int i = 0; i < W; i++)
            if (i == src_lane) xv.e[i] = ln::add(xv.e[i], ln::from_f64(src));
    }
    if (div) {
        if constexpr (LU == 16) {
            if (div->div_mode == DIV_CHEAP) {
                float r[W];
                prcp<W>(*div, s, m, x, r);
                xv = vdiv_cheap<W>(xv, r);
            } else if (div->div_mode == DIV_FAST) {
                xv = O::div(xv, pload<LU, W>(*div, s, m, x));
            } else {
                xv = O::div_ieee(xv, pload<LU, W>(*div, s, m, x));
            }
        } else {
            xv = O::div_ieee(xv, pload<LU, W>(*div, s, m, x));
        }
    }
    xv = O::mul(xv, vsplat<LU, W>(dt));
    if (variant == 0) {
        u = O::add(u, xv);
        return;
    }
    vec<LU, W> r = O::add(t, xv);
    vec<LU, W> sm_ = O::add(u, r);
    if (variant == 3) {
        vec<LU, W> z = O::sub(sm_, u);
        t = O::sub(r, z);
    } else {
        vec<LU, W> pa = O::sub(sm_, r);
        vec<LU, W> pb = O::sub(sm_, pa);
        vec<LU, W> da = O::sub(u, pa);
        vec<LU, W> db = O::sub(r, pb);
        t = O::add(da, db);
    }
    u = sm_;
}

// Store W cells of field f at local row s and keep its ghost slabs current
// ("write-through ghosts"): periodic wrap copies within a single-rank domain, or
// free-surface image rows (stencil.py:121-144) on the ranks owning a global boundary.
// Ghosts facing another rank are filled by the halo exchange instead.
template <int LU, int W>
__device__ __forceinline__ void store_field(const FieldView& f, const Geom& g, int64_t s, int64_t m, int64_t x,
                                            vec<LU, W> v) {
    using T = typename lane<LU>::T;
    vstore<LU, W>(frow<T>(f, g, s, m) + x, v);
    if ((f.gtop | f.gbot) == GHOST_NONE) return;
    const int64_t n = f.rows;
    if (f.gtop == GHOST_PERIODIC && s >= n - G) vstore<LU, W>(frow<T>(f, g, s - n, m) + x, v);
    if (f.gbot == GHOST_PERIODIC && s < G) vstore<LU, W>(frow<T>(f, g, n + s, m) + x, v);
    if ((f.gtop | f.gbot) & GHOST_IMAGE) {
        const vec<LU, W> w = f.odd ? vneg<LU, W>(v) : v;
        const int64_t sg = f.row0 + s, ng = f.nglob;
        if (f.gtop == GHOST_IMAGE) {
            const int64_t k1 = f.half_s ? -sg - 1 : -sg;
            if (k1 < 0 && k1 >= -G) vstore<LU, W>(frow<T>(f, g, k1 - f.row0, m) + x, w);
        }
        if (f.gbot == GHOST_IMAGE) {
            const int64_t k2 = f.half_s ? 2 * ng - 1 - sg : 2 * ng - 2 - sg;
            if (k2 >= ng && k2 < ng + G) vstore<LU, W>(frow<T>(f, g, k2 - f.row0, m) + x, w);
        }
    }
}

// store_field with precomputed addressing (s = local slow row of the cell)
template <int LU, int W>
__device__ __forceinline__ void store_c(const FieldView& f, const Cell& c, int64_t s, vec<LU, W> v) {
    using T = typename lane<LU>::T;
    T* p = reinterpret_cast<T*>(f.base) + c.off;
    vstore<LU, W>(p, v);
    if ((f.gtop | f.gbot) == GHOST_NONE) return;
    const int64_t n = f.rows;
    if (f.gtop == GHOST_PERIODIC && s >= n - G) vstore<LU, W>(p - n * c.slab, v);
    if (f.gbot == GHOST_PERIODIC && s < G) vstore<LU, W>(p + n * c.slab, v);
    if ((f.gtop | f.gbot) & GHOST_IMAGE) {
        const vec<LU, W> w = f.odd ? vneg<LU, W>(v) : v;
        const int64_t sg = f.row0 + s, ng = f.nglob;
        if (f.gtop == GHOST_IMAGE) {
            const int64_t k1 = f.half_s ? -sg - 1 : -sg;
            if (k1 < 0 && k1 >= -G) vstore<LU, W>(p + (k1 - sg) * c.slab, w);
        }
        if (f.gbot == GHOST_IMAGE) {
            const int64_t k2 = f.half_s ? 2 * ng - 1 - sg : 2 * ng - 2 - sg;
            if (k2 >= ng && k2 < ng + G) vstore<LU, W>(p + (k2 - sg) * c.slab, w);
        }
    }
}

// Receivers sorted by (local row, x): int triples (row, x, trace index).  The streaming
// kernels walk rows in order: a CTA-uniform cursor finds each row's receivers, and a
// thread binary-searches its own x range only on rows that have any.
__device__ __forceinline__ int rec_lower(const int* rec, int lo, int hi, int r, int x) {
    while (lo < hi) {  // first index with (row, x) >= (r, x)
        const int mid = (lo + hi) >> 1;
        const int mr = __ldg(rec + 3 * mid), mx = __ldg(rec + 3 * mid + 1);
        if (mr < r || (mr == r && mx < x)) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Record the trace samples of row r for cells [x, x + width) (values from get(offset));
// cur is the uniform cursor (first receiver with row >= previous row).
template <typename GET>
__device__ __forceinline__ void rec_row(const int* rec, int& cur, int hi, int r, int x, double* traces, int64_t nt,
                                        int64_t n, GET get, int width = 8) {
    if (cur >= hi) return;
    if (__ldg(rec + 3 * cur) < r) cur = rec_lower(rec, cur, hi, r, INT_MIN);
    if (cur >= hi || __ldg(rec + 3 * cur) != r) return;
    for (int q = rec_lower(rec, cur, hi, r, x); q < hi; q++) {
        const int rr = __ldg(rec + 3 * q), rx = __ldg(rec + 3 * q + 1);
        if (rr != r || rx >= x + width) break;
        traces[(int64_t)__ldg(rec + 3 * q + 2) * nt + n] = get(rx - x);
    }
}

// Blocks need not be a multiple of 32 threads (the fused 2D kernel runs nx/8 threads):
// the collectives below use only the lanes that exist.
__device__ __forceinline__ int warp_lanes() {
    const int rem = (int)blockDim.x - (int)(threadIdx.x & ~31u);
    return rem < 32 ? rem : 32;
}

// fixed-tree warp sum (lane 0 holds the result); identical bits to the full-warp tree
__device__ __forceinline__ double warp_sum(double a) {
    const int lane = threadIdx.x & 31, nl = warp_lanes();
    const unsigned m = nl == 32 ? 0xffffffffu : ((1u << nl) - 1u);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double b = __shfl_down_sync(m, a, o);
        if (lane + o < nl) a += b;
    }
    return a;
}

// Warp-aggregated failure record: first failing step + external field bits (the bits of that
// step only: a record from a later step -- possible only while another rank's failure is in
// flight -- leaves the mask alone).
__device__ __forceinline__ void record_failure(Ctrl* ctrl, int64_t n, unsigned int mask) {
    const int nl = warp_lanes();
    unsigned int any = __reduce_or_sync(nl == 32 ? 0xffffffffu : ((1u << nl) - 1u), mask);
    if (any && (threadIdx.x & 31) == 0) {
        const unsigned long long old =
            atomicMin(reinterpret_cast<unsigned long long*>(&ctrl->fail_step), (unsigned long long)n);
        if (old >= (unsigned long long)n) atomicOr(&ctrl->fail_mask, any);
    }
}

// A step kernel exits at entry once any step before it failed on this rank or on any rank.
__device__ __forceinline__ bool halted(const Ctrl* ctrl, int64_t n) {
    const int64_t a = *reinterpret_cast<const volatile int64_t*>(&ctrl->fail_step);
    const int64_t b = *reinterpret_cast<const volatile int64_t*>(&ctrl->gfail_step);
    return (a < b ? a : b) < n;
}

// Block-wide fp64 sum of NCOMP components; thread 0 writes the block partial (row idx,
// default: the linear block index).
__device__ __forceinline__ void block_partials(double v[NCOMP], double* out, int64_t idx = -1) {
    __shared__ double red[32][NCOMP];  // any block size up to 1024 threads
    const int tid = threadIdx.x;
    int lane_id = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int c = 0; c < NCOMP; c++) {
        const double a = warp_sum(v[c]);
        if (lane_id == 0) red[warp][c] = a;
    }
    __syncthreads();
    if (tid < NCOMP) {
        double a = 0.0;
        for (int w = 0; w < (int)((blockDim.x + 31) >> 5); w++) a += red[w][tid];
        const int64_t bid = idx >= 0 ? idx : ((int64_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
        out[bid * NCOMP + tid] = a;
    }
}

// Last-CTA energy finalisation: warp w sums components w, w + nwarps, ... of the nb
// block partials (fixed lane-strided order + fixed shuffle tree: deterministic), thread 0
// combines the components left to right.  Any block size >= 32; total on thread 0.
__device__ __forceinline__ double finalize_partials(const double* part, int nb) {
    __shared__ double tot[NCOMP];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = (int)((blockDim.x + 31) >> 5);
    const int nl = warp_lanes();
    for (int c = w; c < NCOMP; c += nw) {
        double a = 0.0;
        // UN loads in flight per lane ahead of the sum (the L2 latencies overlap instead of chaining);
        // the adds stay in the fixed order bi = lane, lane + nl, ... (identical bits)
        constexpr int UN = 8;
        for (int b0 = lane; b0 < nb; b0 += UN * nl) {
            double v[UN];
#pragma unroll
            for (int q = 0; q < UN; q++) {
                const int bi = b0 + q * nl;
                v[q] = bi < nb ? __ldcg(&part[(int64_t)bi * NCOMP + c]) : 0.0;
            }
#pragma unroll
            for (int q = 0; q < UN; q++)
                if (b0 + q * nl < nb) a += v[q];
        }
        a = warp_sum(a);
        if (lane == 0) tot[c] = a;
    }
    __syncthreads();
    double t = tot[0];
    for (int c = 1; c < NCOMP; c++) t += tot[c];
    return t;
}

// Launch shape of the phase kernels: x vectors across blockIdx.x (one row segment
// per block), mid index on blockIdx.y, slow index on blockIdx.z, so (s, m) stay
// warp-uniform (uniform datapath for row addressing); no integer division.
inline int block_threads(int64_t nxv) {
    int64_t b = (nxv + 31) / 32 * 32;
    return (int)(b > BLOCK ? BLOCK : (b < 32 ? 32 : b));
}
inline dim3 block3(const Geom& g, int W) { return dim3(block_threads(g.nx / W)); }
inline dim3 grid3(const Geom& g, int W, int64_t rows) {
    int64_t nxv = g.nx / W;
    int bt = block_threads(nxv);
    return dim3((unsigned)((nxv + bt - 1) / bt), (unsigned)g.nm, (unsigned)rows);
}
inline int64_t grid_blocks(const Geom& g, int W, int64_t rows) {
    dim3 gr = grid3(g, W, rows);
    return (int64_t)gr.x * gr.y * gr.z;
}

}  // namespace hw
