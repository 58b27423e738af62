// hw_api.cu — the C ABI (include/halfwave_b200.h): device state, medium
// materialisation, the step loop and the per-step epilogue kernel.
//
// One hw_solver per rank/GPU.  The whole time loop of AcousticSolver.run /
// ElasticSolver.run (acoustic.py:185-236, elastic.py:242-296) is issued from here
// onto one CUDA stream; the host synchronises once per hw_run.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cmath>
#include <cstdint>
#include <string>
#include <vector>
#include <algorithm>
#include <array>
#include <map>
#include <mutex>

#include "../../include/halfwave_b200.h"
#include "hw_params.h"

using namespace hw;

#include "hw_fused2d.h"

namespace {

thread_local std::string g_err;

// ---------------------------------------------------------------- kernel-path options
// Process-wide switches set through hw_set_option (tests and A/B measurements); read
// when a handle is created.  Defaults are the production choices.
struct Option {
    const char* name;
    int64_t value, lo, hi;
    const char* doc;
};
Option g_opts[] = {
    {"path", 0, 0, 1, "0 = fastest eligible kernels, 1 = generic phase kernels only"},
    {"div", 0, 0, 2, "binary16 division: 0 = table-verified cheap / fast / IEEE per plane, 1 = no cheap path, 2 = IEEE only"},
    {"small", 1, 0, 1, "persistent small-grid 2D kernels for grids of <= 2^20 cells"},
    {"tb", 0, 0, 1, "two steps per launch for the fused 2D acoustic kernel (measured slower; opt-in)"},
    {"fused_el", 1, 0, 1, "one-pass 2D elastic kernel"},
    {"fused3", 1, 0, 1, "one-pass 3D acoustic kernels (binary16 and binary32 lanes)"},
    {"fused_el3", 1, 0, 1, "one-pass 3D elastic kernel (2nd order, media constant along x) | 0 two-phase kernels"},
    {"el3_group", 4, 1, 4, "one-pass 3D elastic kernel: at most this many CTAs stream adjacent tiles side by side"},
    {"ac3_group", 4, 1, 4, "one-pass 3D acoustic kernels: at most this many CTAs stream adjacent tiles side by side"},
    {"guard", 0, 0, 2, "device allocations between unmapped pages (tests): 1 = start at a mapping start, 2 = end at a mapping end"},
    {"el3_overlap_min_rows", 0, 0, 1 << 20, "one-pass 3D elastic kernel on an NCCL slab: thinner slabs exchange in stream order after one launch (no edge / interior split)"},
    {"el3_edge_ctas", 0, 0, 64, "one-pass 3D elastic kernel on an NCCL slab: CTAs of the edge launch (0 = automatic)"},
    {"nccl_self", 0, 0, 1, "a one-rank job with an NCCL id takes the NCCL transport (self exchange: tests)"},
};
int64_t opt(const char* name) {
    for (const Option& o : g_opts)
        if (strcmp(o.name, name) == 0) return o.value;
    return 0;
}

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

// ---------------------------------------------------------------- guarded device allocations
// Option "guard" (tests; compute-sanitizer's memcheck is not available on every box): every device
// buffer of the library becomes its own virtual-memory mapping with unmapped pages on both sides,
// starting at the mapping's first byte (guard = 1: a read or write before the buffer faults) or ending
// at its last (guard = 2: one past the end faults, to 256-byte rounding).  An out-of-bounds access of
// any kernel, TMA requests included, then stops the run with an illegal-address error instead of
// reading a neighbouring allocation unnoticed.  guard = 0 (the default) is plain cudaMalloc.
struct VmmRec {
    CUdeviceptr va, mapped;
    size_t span, msize;
    CUmemGenericAllocationHandle hnd;
};
std::map<void*, VmmRec> g_vmm;
std::mutex g_vmm_mu;

template <typename F>
bool drv(const char* name, F* fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || !p) return false;
    *fn = reinterpret_cast<F>(p);
    return true;
}

cudaError_t hw_dev_alloc(void** out, size_t bytes) {
    const int64_t g = opt("guard");
    if (g == 0) return ::cudaMalloc(out, bytes);
    CUresult (*memCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long);
    CUresult (*memGran)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags);
    CUresult (*memReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
    CUresult (*memMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
    CUresult (*memAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
    if (!drv("cuMemCreate", &memCreate) || !drv("cuMemGetAllocationGranularity", &memGran) ||
        !drv("cuMemAddressReserve", &memReserve) || !drv("cuMemMap", &memMap) || !drv("cuMemSetAccess", &memAccess))
        return cudaErrorNotSupported;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    cudaFree(nullptr);  // (a context on this device)
    CUmemAllocationProp prop = {};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = dev;
    size_t gran = 0;
    if (memGran(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM) != CUDA_SUCCESS || !gran) return cudaErrorUnknown;
    const size_t need = ((bytes ? bytes : 1) + 255) / 256 * 256;
    VmmRec r;
    r.msize = (need + gran - 1) / gran * gran;
    r.span = r.msize + 2 * gran;
    if (memReserve(&r.va, r.span, gran, 0, 0) != CUDA_SUCCESS) return cudaErrorMemoryAllocation;
    if (memCreate(&r.hnd, r.msize, &prop, 0) != CUDA_SUCCESS) return cudaErrorMemoryAllocation;
    r.mapped = r.va + gran;
    if (memMap(r.mapped, r.msize, 0, r.hnd, 0) != CUDA_SUCCESS) return cudaErrorMemoryAllocation;
    CUmemAccessDesc acc = {};
    acc.location = prop.location;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    if (memAccess(r.mapped, r.msize, &acc, 1) != CUDA_SUCCESS) return cudaErrorMemoryAllocation;
    void* p = reinterpret_cast<void*>(g == 1 ? r.mapped : r.mapped + (r.msize - need));
    std::lock_guard<std::mutex> lk(g_vmm_mu);
    g_vmm[p] = r;
    *out = p;
    return cudaSuccess;
}

cudaError_t hw_dev_free(void* p) {
    if (!p) return cudaSuccess;
    VmmRec r;
    {
        std::lock_guard<std::mutex> lk(g_vmm_mu);
        auto it = g_vmm.find(p);
        if (it == g_vmm.end()) return ::cudaFree(p);
        r = it->second;
        g_vmm.erase(it);
    }
    CUresult (*memUnmap)(CUdeviceptr, size_t);
    CUresult (*memRelease)(CUmemGenericAllocationHandle);
    CUresult (*memFree)(CUdeviceptr, size_t);
    if (!drv("cuMemUnmap", &memUnmap) || !drv("cuMemRelease", &memRelease) || !drv("cuMemAddressFree", &memFree))
        return cudaErrorNotSupported;
    cudaDeviceSynchronize();
    memUnmap(r.mapped, r.msize);
    memRelease(r.hnd);
    memFree(r.va, r.span);
    return cudaSuccess;
}
// every allocation below goes through the two functions above
#define cudaMalloc(p, n) hw_dev_alloc((void**)(p), (size_t)(n))
#define cudaFree(p) hw_dev_free((void*)(p))

#define CU(call)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return fail(HW_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));        \
    } while (0)

// ---------------------------------------------------------------- host rounding
// Single RNE rounding of a binary64 value into a lane (round_to, precision.py:108-118),
// used for dt_U.  binary16: the magic-constant add rounds at the binary16 quantum.
double round_lane(int lane_bits, double x) {
    if (lane_bits == 64) return x;
    if (lane_bits == 32) return (double)(float)x;
    uint64_t b;
    memcpy(&b, &x, 8);
    int64_t e = (int64_t)((b >> 52) & 0x7ff) - 1023;
    e = e < -14 ? -14 : (e > 16 ? 16 : e);
    uint64_t mb = (uint64_t)(e + 42 + 1023) << 52;
    double m;
    memcpy(&m, &mb, 8);
    volatile double a = fabs(x);
    volatile double y = a + m;
    double z = y - m;
    if (z > 65504.0) z = INFINITY;
    return copysign(z, x);
}

int lane_bytes(int L) { return L == 16 ? 2 : (L == 32 ? 4 : 8); }

// binary16 bit pattern of a value already exactly representable in binary16.
uint16_t half_bits(double v) {
    uint16_t sign = std::signbit(v) ? 0x8000 : 0;
    double a = std::fabs(v);
    if (a == 0.0) return sign;
    if (std::isinf(a)) return sign | 0x7c00;
    if (std::isnan(a)) return 0x7e00;
    int e;
    double m = std::frexp(a, &e);  // a = m 2^e, m in [0.5, 1)
    int E = e - 1;
    if (E >= -14) return sign | (uint16_t)((E + 15) << 10) | (uint16_t)std::lround((m * 2.0 - 1.0) * 1024.0);
    return sign | (uint16_t)std::lround(std::ldexp(a, 24));
}

LaneConsts make_consts(const double taps[4], double dt_u) {
    LaneConsts c;
    for (int j = 0; j < 5; j++) {
        double v = j < 4 ? taps[j] : dt_u;
        c.h[j] = half_bits(v);
        c.f[j] = (float)v;
        c.d[j] = v;
    }
    return c;
}

// internal field ids (generic axes) and their staggers (half_x, half_m, half_s)
enum { F_P, F_VX, F_VS, F_VM, F_SXX, F_SSS, F_SMM, F_SXS, F_SXM, F_SMS, F_N };
const int HALF_S[F_N] = {0, 0, 1, 0, 0, 0, 0, 1, 0, 1};
constexpr int EL3_EDGE = 2;  // edge slabs per side of an overlapped one-pass 3D elastic slab step
constexpr double EL3_EDGE_SHARE = 1.0;  // CTAs of the edge launch relative to its share of the work

const int EXT_AC2[] = {F_P, F_VX, F_VS};
const int EXT_AC3[] = {F_P, F_VX, F_VM, F_VS};
const int EXT_EL2[] = {F_VX, F_VS, F_SXX, F_SSS, F_SXS};
const int EXT_EL3[] = {F_VX, F_VM, F_VS, F_SXX, F_SMM, F_SSS, F_SXM, F_SXS, F_SMS};

const int* ext_order(int eq, int ndim, int* nsol) {
    if (eq == HW_EQ_ACOUSTIC) {
        *nsol = ndim == 3 ? 4 : 3;
        return ndim == 3 ? EXT_AC3 : EXT_AC2;
    }
    *nsol = ndim == 3 ? 9 : 5;
    return ndim == 3 ? EXT_EL3 : EXT_EL2;
}

// ---------------------------------------------------------------- small kernels

template <typename T>
__global__ void k_round_plane(const double* in, T* out, int64_t n, int lane_bits) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if constexpr (sizeof(T) == 2) out[i] = __double2half(in[i]);
    else if constexpr (sizeof(T) == 4) out[i] = __double2float_rn(in[i]);
    else out[i] = in[i];
}

// Initial ghost fill of the write-through slabs (periodic wrap or global free-surface
// images); slabs facing another rank are filled by the halo exchange.
template <typename T>
__global__ void k_fill_ghosts(FieldView f, Geom g) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t per = g.nm * g.nx;
    if (i >= 2 * G * per) return;
    int64_t q = i / per, rem = i % per;
    int64_t m = rem / g.nx, x = rem % g.nx;
    const int64_t n = f.rows;
    const int64_t k = q < G ? q - G : n + (q - G);  // -G .. -1, n .. n+G-1
    const int mode = k < 0 ? f.gtop : f.gbot;
    if (mode == GHOST_NONE) return;
    int64_t src;
    bool neg = false;
    if (mode == GHOST_PERIODIC) {
        src = k < 0 ? k + n : k - n;
    } else {
        const int64_t kg = f.row0 + k, ng = f.nglob;
        const int64_t sg = f.half_s ? (kg < 0 ? -kg - 1 : 2 * ng - 1 - kg) : (kg < 0 ? -kg : 2 * ng - 2 - kg);
        src = sg - f.row0;
        neg = f.odd;
    }
    T* base = reinterpret_cast<T*>(f.base);
    T v = base[src * g.slab + m * g.pitch + x];
    if (neg) {
        if constexpr (sizeof(T) == 2) v = lane<16>::neg(v);
        else if constexpr (sizeof(T) == 4) v = lane<32>::neg(v);
        else v = lane<64>::neg(v);
    }
    base[k * g.slab + m * g.pitch + x] = v;
}

// Naive runs never rewrite the residual fields, so a non-finite value uploaded in
// one of them fails step 0 (check_finite after the first step, stepping.py:101-105):
// flag it on the device as part of the run's control block.
template <typename T>
__global__ void k_flag_nonfinite(const T* base, Geom g, int64_t rows, unsigned int bit, Ctrl* ctrl) {
    const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t m = blockIdx.y, s = blockIdx.z;
    if (x >= g.nx || s >= rows) return;
    const T v = base[s * g.slab + m * g.pitch + x];
    bool bad;
    if constexpr (sizeof(T) == 2) bad = !lane<16>::finite(v);
    else if constexpr (sizeof(T) == 4) bad = !lane<32>::finite(v);
    else bad = !lane<64>::finite(v);
    if (bad) {
        atomicMin(reinterpret_cast<unsigned long long*>(&ctrl->fail_step), 0ull);
        atomicOr(&ctrl->fail_mask, 1u << bit);
    }
}

// Per-step epilogue: receiver traces (acoustic.py:217-218) and the fixed-order
// reduction of the block energy partials into one fp64 sample.
template <int LU>
__global__ void k_epilogue(EpParams E, int64_t n, int sample, int64_t eidx) {
    if (n >= 0 && halted(E.ctrl, n)) return;
    using TU = typename lane<LU>::T;
    if (n >= 0) {
        const TU* b = reinterpret_cast<const TU*>(E.trace_base);
        for (int j = threadIdx.x; j < E.n_rec; j += blockDim.x)  // receivers of this slab only
            if (E.rec_off[j] >= 0) E.traces[(int64_t)j * E.nt + n] = lane<LU>::to_f64(b[E.rec_off[j]]);
    }
    if (!sample) return;
    __shared__ double red[NCOMP][256];
    for (int c = 0; c < NCOMP; c++) {
        double a = 0.0;
        for (int bi = threadIdx.x; bi < E.nblocks; bi += blockDim.x) a += E.partials[(int64_t)bi * NCOMP + c];
        red[c][threadIdx.x] = a;
    }
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w)
            for (int c = 0; c < NCOMP; c++) red[c][threadIdx.x] += red[c][threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        double tot = red[0][0];
        for (int c = 1; c < NCOMP; c++) tot += red[c][0];
        E.e_vals[eidx] = E.scale * tot;
    }
}

// For every positive finite binary16 divisor b: does fl16(fl32(a * __frcp_rn(b)))
// equal the correctly rounded fl16(a / b) for ALL 65536 binary16 a?  One CTA per b.
__global__ void k_cheap_div_table(unsigned int* ok) {
    const unsigned int b = blockIdx.x + 1;
    if (b > 0x7bffu) return;
    const __half hb = __ushort_as_half((unsigned short)b);
    const float r = __frcp_rn(__half2float(hb));
    bool good = true;
    for (unsigned int a = threadIdx.x; a < 65536u; a += blockDim.x) {
        const __half ha = __ushort_as_half((unsigned short)a);
        const unsigned short x = __half_as_ushort(__float2half_rn(__fmul_rn(__half2float(ha), r)));
        const unsigned short y = __half_as_ushort(lane<16>::div_ieee(ha, hb));
        const bool xn = (x & 0x7c00u) == 0x7c00u && (x & 0x3ffu);
        const bool yn = (y & 0x7c00u) == 0x7c00u && (y & 0x3ffu);
        if (x != y && !(xn && yn)) good = false;
    }
    good = __syncthreads_and(good);
    if (threadIdx.x == 0 && good) atomicOr(&ok[b >> 5], 1u << (b & 31));
}

__global__ void k_rcp_plane(const __half* in, float* out, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = __frcp_rn(__half2float(in[i]));
}

// Exhaustive check of the branch-free binary16 division against the IEEE one:
// every binary16 a (incl. inf/NaN/zero/subnormal) x every finite nonzero b.
__global__ void k_selftest_div16(unsigned long long* bad, unsigned int* first) {
    const unsigned int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= 65536u) return;
    const __half ha = __ushort_as_half((unsigned short)a);
    unsigned long long nbad = 0;
    for (unsigned int b = 0; b < 65536u; b++) {
        if ((b & 0x7fffu) == 0 || (b & 0x7c00u) == 0x7c00u) continue;
        const __half hb = __ushort_as_half((unsigned short)b);
        const unsigned short x = __half_as_ushort(lane<16>::div(ha, hb));
        const unsigned short y = __half_as_ushort(lane<16>::div_ieee(ha, hb));
        const bool xn = (x & 0x7c00u) == 0x7c00u && (x & 0x3ffu);
        const bool yn = (y & 0x7c00u) == 0x7c00u && (y & 0x3ffu);
        if (x != y && !(xn && yn)) {
            nbad++;
            atomicCAS(first, 0xffffffffu, (a << 16) | b);
        }
    }
    if (nbad) atomicAdd(bad, nbad);
}

}  // namespace

namespace {
std::vector<uint32_t> g_cheap_table[64];

int cheap_div_table(int device, const std::vector<uint32_t>** out) {
    if (device < 0 || device >= 64) return fail(HW_EINVAL, "device ordinal out of range");
    if (g_cheap_table[device].empty()) {
        unsigned int* ok = nullptr;
        CU(cudaMalloc(&ok, 1024 * 4));
        CU(cudaMemset(ok, 0, 1024 * 4));
        k_cheap_div_table<<<0x7bff, 256>>>(ok);
        CU(cudaGetLastError());
        std::vector<uint32_t> t(1024);
        CU(cudaMemcpy(t.data(), ok, 1024 * 4, cudaMemcpyDeviceToHost));
        cudaFree(ok);
        g_cheap_table[device] = t;
    }
    *out = &g_cheap_table[device];
    return HW_OK;
}
}  // namespace

namespace hw {
void launch_epilogue(int LU, const EpParams& E, int64_t n, int sample, int64_t eidx, cudaStream_t st) {
    HW_DISPATCH_LU(LU, k_epilogue<LU_><<<1, 256, 0, st>>>(E, n, sample, eidx))
}
}  // namespace hw

// ---------------------------------------------------------------- NCCL (loaded on demand)
// Multi-process runs exchange halo slabs with NCCL send/recv over NVLink.  The
// library resolves NCCL with dlopen only when world_size > 1, so single-GPU and
// in-process slab groups carry no NCCL dependency.
#include <dlfcn.h>
#include <nccl.h>

namespace {
struct NcclApi {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*);
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*GroupStart)();
    ncclResult_t (*GroupEnd)();
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    const char* (*GetErrorString)(ncclResult_t);
};
NcclApi g_nccl;

int nccl_load() {
    if (g_nccl.ok) return HW_OK;
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) return fail(HW_ENCCL, std::string("cannot load libnccl.so.2: ") + dlerror());
#define SYM(name) *(void**)(&g_nccl.name) = dlsym(lib, "nccl" #name); if (!g_nccl.name) return fail(HW_ENCCL, "missing nccl" #name)
    SYM(GetUniqueId); SYM(CommInitRank); SYM(CommDestroy); SYM(Send); SYM(Recv); SYM(GroupStart);
    SYM(GroupEnd); SYM(AllReduce); SYM(AllGather); SYM(Broadcast); SYM(GetErrorString);
#undef SYM
    g_nccl.ok = true;
    return HW_OK;
}

#define NC(call)                                                                              \
    do {                                                                                      \
        ncclResult_t r_ = (call);                                                             \
        if (r_ != ncclSuccess) return fail(HW_ENCCL, std::string(#call) + ": " + g_nccl.GetErrorString(r_)); \
    } while (0)
}  // namespace

// ---------------------------------------------------------------- the handle

struct hw_group;

struct hw_solver {
    hw_desc d;
    int LS, LU, W, nsol, d3, fs, ac;
    const int* ext;
    Geom g;
    FieldView fv[F_N], rv[F_N];
    void* mem[2 * F_N] = {};
    std::vector<void*> plane_mem;
    PlaneView lp[HW_NPLANES];
    Plane64 ep64[HW_NPLANES];
    Ctrl* ctrl = nullptr;
    bool owns_ctrl = true;
    double* partials = nullptr;
    int64_t nblocks = 0;
    int64_t max_rows = 0;
    double* traces = nullptr;
    int64_t traces_cap = 0;
    double* evals = nullptr;
    int64_t evals_cap = 0;
    int64_t* rec_off = nullptr;
    int* rec_sorted = nullptr;  // owned receivers as (local row, x, j), sorted by (row, x)
    int n_rec_sorted = 0;
    cudaStream_t st = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaEvent_t ev_phase = nullptr, ev_copied = nullptr;
    int64_t launches = 0;
    double kernel_ms = 0.0;
    double dt_u = 0.0;
    // fused single-pass path (2D acoustic, binary16): ping-pong partner buffers
    bool fused = false;
    int fused_blocks = 0;
    // NCCL slab of the fused kernel: edge bands + exchange on st, interior bands on st2
    cudaStream_t st2 = nullptr;
    cudaEvent_t ev_edge[2] = {}, ev_int[2] = {};
    int nb_int = 0;
    // persistent small-grid kernel: one cooperative launch per run, state in shared memory
    bool small = false, small_el = false;
    int small_nb = 0;
    __half* xch = nullptr;
    unsigned int* gbar = nullptr;
    double* src_dev = nullptr;
    int64_t src_cap = 0;
    double* partials2 = nullptr;
    bool tb2 = false;  // two steps per launch (temporal blocking, hw_tb2d.cu)
    int tb2_tiles = 0, tb2_bands = 0;
    double* partials_b = nullptr;  // stage-B energy partials of the two-step kernel
    void* mem_b[2 * F_N] = {};
    // streaming phase kernels (2D elastic, binary16): in place on the standard layout
    bool el_stream = false;   // streaming 2D elastic phases
    bool ac3_stream = false;  // streaming 3D acoustic phases
    bool fused3 = false;      // one-pass 3D acoustic step (2nd order), ping-pong A <-> B
    bool fused3_32 = false;   // the same in binary32 lanes (config 3's fp32 arm), ping-pong A <-> B
    bool fused_el = false;    // one-pass 2D elastic step, ping-pong A <-> B
    bool fused_el3 = false;   // one-pass 3D elastic step (2nd order), ping-pong A <-> B
    float* el3_coef = nullptr;  // its medium coefficient table ([ns][el3_cm][8], in plane_mem)
    int64_t el3_cm = 0;
    int el3_group = 1;          // CTA groups of adjacent tiles of the one-pass 3D kernels (elastic and acoustic)
    double* el3_ecoef = nullptr;  // its per-slab energy coefficients (slow-layered media; in plane_mem)
    bool el3_slab = false;        // ... on a slab of a decomposed domain (ghosts from HW_PLAN_FUSED_EL3)
    int ac3_nb_edge = 0, ac3_nb_int = 0;  // one-pass 3D acoustic kernels on an NCCL slab: CTAs of the edge / interior launches
    int el3_nb_edge = 0, el3_nb_int = 0;  // ... NCCL slab: CTAs of the edge / interior launches (overlap)
    // Plane-ordered energy of the one-pass 3D kernels (fused_el3, fused3, fused3_32): per-(slab, tile)
    // partials, per-slab totals per sample, summed on the host in global slab order -- the same bits
    // for any decomposition into slabs
    double* el3_eplane = nullptr; // energy partials per (slab, tile) unit (in plane_mem)
    double* el3_etot = nullptr;   // energy plane totals per sample
    int64_t el3_etot_cap = 0;
    bool plane_energy() const { return fused_el3 || fused3 || fused3_32; }
    bool el3_stream = false;  // streaming 3D elastic phases
    int stream_blocks = 0;
    unsigned int* counter = nullptr;  // CTA arrival counter of the streaming stress kernel
    // slab decomposition over the slow axis
    int world = 1, rank = 0;
    int64_t r0 = 0, ns_loc = 0;
    int transport = 0;  // 0 single domain, 1 in-process slab group, 2 NCCL
    hw_group* group = nullptr;
    ncclComm_t nccl = nullptr;
    int src_active = 0;
    int64_t src_s_loc = 0;
    std::vector<int> rec_owned;  // receiver j lives on this slab
};

struct hw_group {
    std::vector<hw_solver*> ranks;
};

namespace {

int64_t nglob_rows(const hw_solver* h, int f) { return h->d.ns + ((h->fs && !HALF_S[f]) ? 1 : 0); }

int64_t field_rows(const hw_solver* h, int f) {
    return h->ns_loc + ((h->fs && !HALF_S[f] && h->rank == h->world - 1) ? 1 : 0);
}

// fields read by a slow-axis derivative: they need ghost slabs (stencil.py ddy_*)
bool needs_ghosts(const hw_solver* h, int f) {
    if (h->ac) return f == F_P || f == F_VS;
    return f == F_VX || f == F_VS || f == F_VM || f == F_SXS || f == F_SSS || f == F_SMS;
}
bool is_velocity(int f) { return f == F_VX || f == F_VS || f == F_VM; }


int plane_lane(const hw_solver* h, int pl) {
    switch (pl) {
        case HW_PL_RHO_X: case HW_PL_RHO_S: case HW_PL_RHO_M: case HW_PL_BETA: return h->LU;
        case HW_PL_LAM: case HW_PL_STIFF: case HW_PL_MU_N: case HW_PL_EP: return h->LS;
        default: return 0;  // energy only
    }
}

// local rows of the field each plane is shaped like (0 = plane unused)
int64_t plane_rows(const hw_solver* h, int pl) {
    bool el = !h->ac;
    switch (pl) {
        case HW_PL_RHO_X: return field_rows(h, F_VX);
        case HW_PL_RHO_S: return field_rows(h, F_VS);
        case HW_PL_RHO_M: return h->d3 ? field_rows(h, F_VM) : 0;
        case HW_PL_BETA: return h->ac ? field_rows(h, F_P) : 0;
        case HW_PL_LAM: case HW_PL_MU: case HW_PL_STIFF: return el ? field_rows(h, F_SXX) : 0;
        case HW_PL_MU_N: return el ? field_rows(h, F_SXS) : 0;
        case HW_PL_EP: return (el && h->fs) ? 2 : 0;
    }
    return 0;
}

// Upload this slab's rows of one fp64 plane, compressed to constant / slow-layered /
// full, plus its lane copy and (binary16 divisors) its division mode.
int upload_plane(hw_solver* h, int pl) {
    int64_t rows = plane_rows(h, pl);
    h->lp[pl] = PlaneView{nullptr, nullptr, 0, 0, 0, 0, 0};
    h->ep64[pl] = Plane64{nullptr, 0, 0, 0};
    if (!rows) return HW_OK;
    int64_t nm = pl == HW_PL_EP ? 1 : h->d.nm, nx = h->d.nx;
    int64_t per = nm * nx;
    if (!h->d.plane[pl]) return fail(HW_EINVAL, "medium plane " + std::to_string(pl) + " missing");
    const double* src = h->d.plane[pl] + (pl == HW_PL_EP ? 0 : h->r0 * per);
    // Slab mode: 2G halo rows each side (global rows wrapped, or clamped at a free
    // surface), views pointing at local row 0, so kernels that recompute halo rows (the
    // fused 2D kernel's vy, rows -2 .. L) find their coefficients, and its row-uniform
    // coefficient prefetch (front rows -6 .. L+3 of the first / last band) stays inside
    // the allocation.
    const int64_t pad = ((h->world > 1 || h->transport == 2) && pl != HW_PL_EP) ? 2 * G : 0;
    std::vector<double> ext;
    if (pad) {
        static const int PLANE_FIELD[HW_NPLANES] = {F_VX, F_VS, F_VM, F_P, F_SXX, F_SXX, F_SXX, F_SXS, F_SXX};
        const int64_t ng = nglob_rows(h, PLANE_FIELD[pl]);
        ext.resize((rows + 2 * pad) * per);
        for (int64_t r = -pad; r < rows + pad; r++) {
            int64_t gr = h->r0 + r;
            if (h->fs) gr = gr < 0 ? 0 : (gr >= ng ? ng - 1 : gr);
            else gr = ((gr % ng) + ng) % ng;
            memcpy(&ext[(r + pad) * per], h->d.plane[pl] + gr * per, per * sizeof(double));
        }
        src = ext.data();
        rows += 2 * pad;
    }
    const int64_t n = rows * per;
    bool cst = true, layered = true;
    for (int64_t i = 1; i < n && cst; i++) cst = memcmp(&src[i], &src[0], 8) == 0;
    if (!cst)
        for (int64_t s = 0; s < rows && layered; s++)
            for (int64_t i = 1; i < per && layered; i++) layered = memcmp(&src[s * per + i], &src[s * per], 8) == 0;
    std::vector<double> packed;
    int64_t ss, sm, sx;
    if (cst) {
        packed.assign(1, src[0]);
        ss = sm = sx = 0;
    } else if (layered) {
        packed.resize(rows);
        for (int64_t s = 0; s < rows; s++) packed[s] = src[s * per];
        ss = 1; sm = 0; sx = 0;
    } else {
        packed.assign(src, src + n);
        ss = per; sm = nx; sx = 1;
    }
    int64_t cnt = (int64_t)packed.size();
    const int64_t off = pad * ss;  // elements before local row 0
    double* d64 = nullptr;
    CU(cudaMalloc(&d64, cnt * 8));
    h->plane_mem.push_back(d64);
    CU(cudaMemcpy(d64, packed.data(), cnt * 8, cudaMemcpyHostToDevice));
    h->ep64[pl] = Plane64{d64 + off, ss, sm, sx};
    int L = plane_lane(h, pl);
    if (L) {
        void* dl = nullptr;
        CU(cudaMalloc(&dl, cnt * lane_bytes(L) + 16));
        h->plane_mem.push_back(dl);
        int64_t nb = (cnt + 255) / 256;
        if (L == 16) k_round_plane<__half><<<nb, 256>>>(d64, (__half*)dl, cnt, L);
        else if (L == 32) k_round_plane<float><<<nb, 256>>>(d64, (float*)dl, cnt, L);
        else k_round_plane<double><<<nb, 256>>>(d64, (double*)dl, cnt, L);
        CU(cudaGetLastError());
        int mode = DIV_NONE;
        const float* rcp = nullptr;
        const bool divisor = pl == HW_PL_RHO_X || pl == HW_PL_RHO_S || pl == HW_PL_RHO_M || pl == HW_PL_BETA;
        if (divisor) {
            mode = DIV_IEEE;
            if (L == 16) {
                const std::vector<uint32_t>* tab = nullptr;
                int trc = cheap_div_table(h->d.device, &tab);
                if (trc) return trc;
                bool fast = true, cheap = true;  // every lane value finite and nonzero / table-verified
                for (double v : packed) {
                    double r = round_lane(16, v);
                    if (!(r != 0.0 && std::isfinite(r))) fast = false;
                    uint16_t hb = half_bits(r);
                    if (hb == 0 || hb > 0x7bff || !(((*tab)[hb >> 5] >> (hb & 31)) & 1u)) cheap = false;
                }
                if (opt("div") == 2) fast = cheap = false;
                if (opt("div") == 1) cheap = false;
                mode = cheap ? DIV_CHEAP : (fast ? DIV_FAST : DIV_IEEE);
                if (cheap) {
                    float* dr = nullptr;
                    CU(cudaMalloc(&dr, cnt * sizeof(float) + 16));
                    h->plane_mem.push_back(dr);
                    k_rcp_plane<<<(cnt + 255) / 256, 256>>>((const __half*)dl, dr, cnt);
                    CU(cudaGetLastError());
                    rcp = dr;
                }
            }
        }
        h->lp[pl] = PlaneView{(const char*)dl + off * lane_bytes(L), rcp ? rcp + off : nullptr, ss, sm, sx, mode, 0};
    }
    return HW_OK;
}

void fill_params(const hw_solver* h, AcParams& P) {
    memset(&P, 0, sizeof(P));
    P.g = h->g;
    P.p = h->fv[F_P]; P.vx = h->fv[F_VX]; P.vs = h->fv[F_VS]; P.vm = h->fv[F_VM];
    P.rp = h->rv[F_P]; P.rvx = h->rv[F_VX]; P.rvs = h->rv[F_VS]; P.rvm = h->rv[F_VM];
    P.rho_x = h->lp[HW_PL_RHO_X]; P.rho_s = h->lp[HW_PL_RHO_S]; P.rho_m = h->lp[HW_PL_RHO_M];
    P.beta = h->lp[HW_PL_BETA];
    P.e_beta = h->ep64[HW_PL_BETA]; P.e_rho_x = h->ep64[HW_PL_RHO_X];
    P.e_rho_s = h->ep64[HW_PL_RHO_S]; P.e_rho_m = h->ep64[HW_PL_RHO_M];
    P.k = make_consts(h->d.taps, h->dt_u);
    P.order = h->d.order;
    P.d3 = h->d3;
    P.has_src = h->d.src_kind == HW_SRC_PRESSURE && h->src_active;
    P.src_x = h->d.src_x; P.src_m = h->d.src_m; P.src_s = h->src_s_loc;
    P.ctrl = h->ctrl;
    P.partials = h->partials;
}

void fill_params(const hw_solver* h, ElParams& P) {
    memset(&P, 0, sizeof(P));
    P.g = h->g;
    P.vx = h->fv[F_VX]; P.vs = h->fv[F_VS]; P.vm = h->fv[F_VM];
    P.sxx = h->fv[F_SXX]; P.sss = h->fv[F_SSS]; P.smm = h->fv[F_SMM];
    P.sxs = h->fv[F_SXS]; P.sxm = h->fv[F_SXM]; P.sms = h->fv[F_SMS];
    P.rvx = h->rv[F_VX]; P.rvs = h->rv[F_VS]; P.rvm = h->rv[F_VM];
    P.rsxx = h->rv[F_SXX]; P.rsss = h->rv[F_SSS]; P.rsmm = h->rv[F_SMM];
    P.rsxs = h->rv[F_SXS]; P.rsxm = h->rv[F_SXM]; P.rsms = h->rv[F_SMS];
    P.rho_x = h->lp[HW_PL_RHO_X]; P.rho_s = h->lp[HW_PL_RHO_S]; P.rho_m = h->lp[HW_PL_RHO_M];
    P.stiff = h->lp[HW_PL_STIFF]; P.lam = h->lp[HW_PL_LAM]; P.mu_n = h->lp[HW_PL_MU_N]; P.ep = h->lp[HW_PL_EP];
    P.e_rho_x = h->ep64[HW_PL_RHO_X]; P.e_rho_s = h->ep64[HW_PL_RHO_S]; P.e_rho_m = h->ep64[HW_PL_RHO_M];
    P.e_lam = h->ep64[HW_PL_LAM]; P.e_mu = h->ep64[HW_PL_MU]; P.e_mu_n = h->ep64[HW_PL_MU_N];
    P.k = make_consts(h->d.taps, h->dt_u);
    P.order = h->d.order;
    P.d3 = h->d3;
    P.fs = h->fs;
    P.src_kind = h->src_active ? h->d.src_kind : HW_SRC_NONE;
    P.src_x = h->d.src_x; P.src_m = h->d.src_m; P.src_s = h->src_s_loc;
    P.ctrl = h->ctrl;
    P.partials = h->partials;
}

int check_desc(const hw_desc* d) {
    if (!d) return fail(HW_EINVAL, "null descriptor");
    if (d->abi_version != HW_ABI_VERSION) return fail(HW_EINVAL, "ABI version mismatch");
    if (d->equation != HW_EQ_ACOUSTIC && d->equation != HW_EQ_ELASTIC) return fail(HW_EINVAL, "bad equation");
    if (d->ndim != 2 && d->ndim != 3) return fail(HW_EINVAL, "ndim must be 2 or 3");
    if (d->order != 2 && d->order != 4) return fail(HW_EINVAL, "order must be 2 or 4");
    auto okl = [](int L) { return L == 16 || L == 32 || L == 64; };
    if (!okl(d->lane_s) || !okl(d->lane_u)) return fail(HW_EINVAL, "lanes must be 16, 32 or 64");
    if (d->nx < 8 || d->ns < 8 || d->nm < 1 || (d->ndim == 2 && d->nm != 1) || (d->ndim == 3 && d->nm < 8))
        return fail(HW_EINVAL, "grid must be at least 8 cells per axis");
    if (d->bc_slow == HW_BC_FREE_SURFACE && (d->equation != HW_EQ_ELASTIC || d->ndim != 2))
        return fail(HW_EINVAL, "free surfaces are supported for the 2D elastic solver only");
    if (d->bc_slow != HW_BC_PERIODIC && d->bc_slow != HW_BC_FREE_SURFACE) return fail(HW_EINVAL, "bad bc");
    if (d->energy_every < 1) return fail(HW_EINVAL, "energy_every must be at least 1");
    if (!(d->dx > 0.0) || !(d->dt > 0.0)) return fail(HW_EINVAL, "dx and dt must be positive");
    if (d->world_size < 1 || d->rank < 0 || d->rank >= d->world_size) return fail(HW_EINVAL, "bad world_size/rank");
    if (d->world_size > 1 && d->ns / d->world_size < 4) return fail(HW_EINVAL, "slabs need at least 4 rows per rank");
    if (d->n_receivers < 0 || (d->n_receivers > 0 && !d->receivers)) return fail(HW_EINVAL, "bad receivers");
    return HW_OK;
}

// The slab's field buffers, ghost policies, medium, source and receivers.
// Ping-pong partner buffers (B) of the one-pass kernels: same shape as the fields' own buffers (A).
int alloc_partner_buffers(hw_solver* h) {
    const int esz = lane_bytes(h->LU);
    for (int j = 0; j < 2 * h->nsol; j++) {
        const int f = h->ext[j % h->nsol];
        const size_t bytes = (size_t)(field_rows(h, f) + 2 * G) * h->g.slab * esz;
        if (cudaMalloc(&h->mem_b[j], bytes) != cudaSuccess) return fail(HW_ECUDA, "out of memory (B)");
        CU(cudaMemset(h->mem_b[j], 0, bytes));
    }
    return HW_OK;
}

// Second stream + events of an NCCL slab's overlapped step (edge bands and exchange | interior bands).
int make_overlap_streams(hw_solver* h) {
    CU(cudaStreamCreateWithFlags(&h->st2, cudaStreamNonBlocking));
    for (int k = 0; k < 2; k++) {
        CU(cudaEventCreateWithFlags(&h->ev_edge[k], cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&h->ev_int[k], cudaEventDisableTiming));
    }
    return HW_OK;
}

int setup_handle(hw_solver* h) {
    const hw_desc* desc = &h->d;
    int rc;
    CU(cudaSetDevice(desc->device));
    h->LS = desc->lane_s;
    h->LU = desc->lane_u;
    h->W = (desc->nx % 2 == 0) ? 2 : 1;
    h->d3 = desc->ndim == 3;
    h->fs = desc->bc_slow == HW_BC_FREE_SURFACE;
    h->ac = desc->equation == HW_EQ_ACOUSTIC;
    h->ext = ext_order(desc->equation, desc->ndim, &h->nsol);
    h->dt_u = round_lane(h->LU, desc->dt);
    h->r0 = (int64_t)h->rank * desc->ns / h->world;
    h->ns_loc = (int64_t)(h->rank + 1) * desc->ns / h->world - h->r0;
    int64_t pitch = (desc->nx + 31) / 32 * 32;
    h->g = Geom{desc->nx, desc->nm, pitch, desc->nm * pitch};
    CU(cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking));
    CU(cudaEventCreate(&h->ev0));
    CU(cudaEventCreate(&h->ev1));
    CU(cudaEventCreateWithFlags(&h->ev_phase, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&h->ev_copied, cudaEventDisableTiming));
    const int esz = lane_bytes(h->LU);
    int64_t max_rows = 0;
    const bool top_image = h->fs && h->rank == 0, bot_image = h->fs && h->rank == h->world - 1;
    for (int j = 0; j < 2 * h->nsol; j++) {
        int f = h->ext[j % h->nsol];
        bool resid = j >= h->nsol;
        int64_t rows = field_rows(h, f);
        max_rows = rows > max_rows ? rows : max_rows;
        size_t bytes = (size_t)(rows + 2 * G) * h->g.slab * esz;
        void* p = nullptr;
        if (cudaMalloc(&p, bytes) != cudaSuccess) return fail(HW_ECUDA, "out of device memory for fields");
        CU(cudaMemset(p, 0, bytes));
        h->mem[j] = p;
        FieldView fv;
        memset(&fv, 0, sizeof(fv));
        fv.base = (char*)p + (size_t)G * h->g.slab * esz;
        fv.rows = rows;
        fv.row0 = h->r0;
        fv.nglob = nglob_rows(h, f);
        fv.half_s = HALF_S[f];
        fv.bit = j;
        fv.gtop = fv.gbot = GHOST_NONE;
        if (!resid && needs_ghosts(h, f)) {
            // parity of the image: odd for sxy/syy (elastic.py:186-189), even for vx/vy (:210-236)
            fv.odd = (f == F_SXS || f == F_SSS) ? 1 : 0;
            if (h->world == 1 && !h->fs && h->transport != 2) fv.gtop = fv.gbot = GHOST_PERIODIC;
            if (top_image) fv.gtop = GHOST_IMAGE;
            if (bot_image) fv.gbot = GHOST_IMAGE;
        }
        (resid ? h->rv : h->fv)[f] = fv;
    }
    for (int pl = 0; pl < HW_NPLANES; pl++)
        if ((rc = upload_plane(h, pl))) return rc;
    {
        const bool want = opt("path") == 0;
        int dev_smem = 0, nsm = 0;
        cudaDeviceGetAttribute(&dev_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, desc->device);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, desc->device);
        // fused 2D kernel: single domain, or one slab of a decomposed domain (ghost rows
        // exchanged once per step; periodic slow axis only, as the acoustic solver)
        if (want && h->ac && !h->d3 && h->LS == 16 && h->LU == 16 && !h->fs && field_rows(h, F_P) >= 8 &&
            fused2d_eligible(desc->nx, dev_smem)) {
            if ((rc = alloc_partner_buffers(h))) return rc;
            if (fused2d_prepare(desc->nx) != cudaSuccess) return fail(HW_ECUDA, "fused kernel setup failed");
            int64_t nbf = field_rows(h, F_P) / 4;
            if (nbf < 1) nbf = 1;
            h->fused_blocks = (int)(nbf < nsm ? nbf : nsm);
            h->fused = true;
            if (h->transport == 2 && field_rows(h, F_P) >= 5 * FUSED_EDGE) {  // overlapped halo exchange
                if ((rc = make_overlap_streams(h))) return rc;
                int64_t ni = (field_rows(h, F_P) - 2 * FUSED_EDGE) / 4;
                h->nb_int = (int)(ni < nsm - 2 ? ni : nsm - 2);
            }
            // two steps per launch: opt-in (HALFWAVE_TB=1); measured slower than the
            // single-step kernel on B200 (compute/latency-bound)
            if (opt("tb") == 1 && h->world == 1 && h->transport != 2 &&
                tb2_eligible(desc->nx, desc->ns, dev_smem)) {
                if (tb2_prepare(desc->nx) != cudaSuccess) return fail(HW_ECUDA, "two-step kernel setup failed");
                tb2_grid(desc->nx, desc->ns, nsm, &h->tb2_tiles, &h->tb2_bands);
                h->tb2 = true;
            }
        }
        // small grids: the persistent kernel (latency, not bandwidth, bounds them)
        const bool small_ok = opt("small") == 1;
        if (want && small_ok && h->ac && !h->d3 && h->LS == 16 && h->LU == 16 &&
            h->world == 1 && h->transport == 0 && desc->nx * desc->ns <= (int64_t)1 << 20 &&
            small2d_eligible(desc->nx, desc->ns, nsm, dev_smem)) {
            h->small_nb = small2d_blocks(desc->ns, nsm);
            if (small2d_prepare(desc->nx, desc->ns, h->small_nb) != cudaSuccess)
                return fail(HW_ECUDA, "small-grid kernel setup failed");
            CU(cudaMalloc(&h->xch, small2d_xch_bytes(desc->nx, h->small_nb)));
            CU(cudaMemset(h->xch, 0, small2d_xch_bytes(desc->nx, h->small_nb)));
            CU(cudaMalloc(&h->gbar, 2 * sizeof(unsigned int)));
            CU(cudaMalloc(&h->partials2, (size_t)h->small_nb * NCOMP * sizeof(double)));
            h->small = true;
        }
        if (want && small_ok && !h->ac && !h->d3 && h->LS == 16 && h->LU == 16 &&
            h->world == 1 && h->transport == 0 && desc->nx * desc->ns <= (int64_t)1 << 20 &&
            small_el2d_eligible(desc->nx, desc->ns, nsm, dev_smem)) {
            h->small_nb = small2d_blocks(desc->ns, nsm);
            if (small_el2d_prepare(desc->nx, desc->ns, h->small_nb) != cudaSuccess)
                return fail(HW_ECUDA, "small-grid kernel setup failed");
            CU(cudaMalloc(&h->xch, small_el2d_xch_bytes(desc->nx, h->small_nb)));
            CU(cudaMemset(h->xch, 0, small_el2d_xch_bytes(desc->nx, h->small_nb)));
            CU(cudaMalloc(&h->gbar, 2 * sizeof(unsigned int)));
            CU(cudaMalloc(&h->partials2, (size_t)h->small_nb * NCOMP * sizeof(double)));
            h->small_el = true;
        }
        // one-pass 2D elastic step (a single domain, or a slab of a decomposed one: ghost rows from
        // HW_PLAN_FUSED_EL2 once per step): ping-pong partner buffers
        if (want && !h->small_el && opt("fused_el") == 1 && !h->ac && !h->d3 && h->LS == 16 &&
            h->LU == 16 && el2d_fused_eligible(desc->nx, field_rows(h, F_SXS), dev_smem)) {
            if ((rc = alloc_partner_buffers(h))) return rc;
            if (el2d_fused_prepare(desc->nx) != cudaSuccess) return fail(HW_ECUDA, "fused elastic kernel setup failed");
            int64_t nbs = max_rows / 4;
            if (nbs < 1) nbs = 1;
            h->stream_blocks = (int)(nbs < nsm ? nbs : nsm);
            h->fused_el = true;
            // NCCL slab: the two edge bands + the exchange on st, the interior bands on st2 (as the
            // fused 2D acoustic kernel)
            if (h->transport == 2 && field_rows(h, F_SXS) >= 5 * FUSED_EDGE) {
                if ((rc = make_overlap_streams(h))) return rc;
                int64_t ni = (field_rows(h, F_SXS) - 2 * FUSED_EDGE) / 4;
                h->nb_int = (int)(ni < nsm - 2 ? ni : nsm - 2);
            }
        }
        if (want && !h->small_el && !h->fused_el && !h->ac && !h->d3 && h->LS == 16 && h->LU == 16 &&
            el2d_stream_eligible(desc->nx, desc->ns, dev_smem)) {
            if (el2d_stream_prepare(desc->nx) != cudaSuccess) return fail(HW_ECUDA, "streaming kernel setup failed");
            int64_t nbs = max_rows / 4;
            if (nbs < 1) nbs = 1;
            h->stream_blocks = (int)(nbs < nsm ? nbs : nsm);
            h->el_stream = true;
        }
        // one-pass 3D acoustic step (2nd order; a single domain or a slab of a decomposed one, whose
        // ghost rows p(-1), p(L), v_slow(-1) come from HW_PLAN_FUSED_AC3 once per step): ping-pong buffers
        const bool f3_ok = opt("fused3") == 1;
        if (want && f3_ok && h->ac && h->d3 && h->LS == 16 && h->LU == 16 && !h->fs &&
            ac3d_fused_eligible(desc->nx, desc->nm, field_rows(h, F_P), h->g.pitch, desc->order, dev_smem)) {
            if ((rc = alloc_partner_buffers(h))) return rc;
            if (ac3d_fused_prepare(desc->nx) != cudaSuccess) return fail(HW_ECUDA, "fused 3D kernel setup failed");
            const int64_t tiles = desc->nm / (4096 / desc->nx), units = tiles * max_rows;
            int64_t nbs = units / 4;
            if (nbs < 1) nbs = 1;
            h->stream_blocks = (int)(nbs < nsm ? nbs : nsm);
            for (int g : {4, 2, 1})  // CTA groups of adjacent tiles (halo rows shared through L2)
                if (g <= opt("ac3_group") && h->stream_blocks % g == 0 && tiles % g == 0 &&
                    (tiles / g) * max_rows >= h->stream_blocks / g) {
                    h->el3_group = g;
                    break;
                }
            h->fused3 = true;
            if (h->transport == 2 && max_rows >= 16 && nsm > 8) {  // overlapped halo exchange (edge slabs 0, L-1)
                if ((rc = make_overlap_streams(h))) return rc;
                // the edge launch (CTA groups of 1): 2 one-slab units per tile, ~3 ring iterations each -- 4 CTAs
                // finish them well before the interior launch ends, so the exchange hides behind it
                const int g = h->el3_group;
                h->ac3_nb_edge = (int)(2 * tiles < 4 ? 2 * tiles : 4);
                int64_t ni = (tiles / g) * (max_rows - 2);  // interior (tile group, slab) units
                if (ni > (nsm - h->ac3_nb_edge) / g) ni = (nsm - h->ac3_nb_edge) / g;
                h->ac3_nb_int = (int)(ni < 1 ? 1 : ni) * g;
            }
            CU(cudaMalloc(&h->el3_eplane, (size_t)max_rows * (desc->nm / (4096 / desc->nx)) * sizeof(double)));
            h->plane_mem.push_back(h->el3_eplane);
        }
        // the one-pass 3D acoustic step in binary32 lanes (BASELINE config 3's fp32 arm)
        if (want && f3_ok && h->ac && h->d3 && h->LS == 32 && h->LU == 32 && !h->fs &&
            ac3d_fused32_eligible(desc->nx, desc->nm, field_rows(h, F_P), h->g.pitch, desc->order, dev_smem)) {
            if ((rc = alloc_partner_buffers(h))) return rc;
            if (ac3d_fused32_prepare(desc->nx) != cudaSuccess) return fail(HW_ECUDA, "fused 3D fp32 kernel setup failed");
            const int64_t tiles = desc->nm / (2048 / desc->nx), units = tiles * max_rows;
            int64_t nbs = units / 4;
            if (nbs < 1) nbs = 1;
            h->stream_blocks = (int)(nbs < nsm ? nbs : nsm);
            for (int g : {4, 2, 1})  // CTA groups of adjacent tiles (halo rows shared through L2)
                if (g <= opt("ac3_group") && h->stream_blocks % g == 0 && tiles % g == 0 &&
                    (tiles / g) * max_rows >= h->stream_blocks / g) {
                    h->el3_group = g;
                    break;
                }
            h->fused3_32 = true;
            if (h->transport == 2 && max_rows >= 16 && nsm > 8) {  // overlapped halo exchange (edge slabs 0, L-1)
                if ((rc = make_overlap_streams(h))) return rc;
                // the edge launch (CTA groups of 1): 2 one-slab units per tile, ~3 ring iterations each -- 4 CTAs
                // finish them well before the interior launch ends, so the exchange hides behind it
                const int g = h->el3_group;
                h->ac3_nb_edge = (int)(2 * tiles < 4 ? 2 * tiles : 4);
                int64_t ni = (tiles / g) * (max_rows - 2);  // interior (tile group, slab) units
                if (ni > (nsm - h->ac3_nb_edge) / g) ni = (nsm - h->ac3_nb_edge) / g;
                h->ac3_nb_int = (int)(ni < 1 ? 1 : ni) * g;
            }
            CU(cudaMalloc(&h->el3_eplane, (size_t)max_rows * (desc->nm / (2048 / desc->nx)) * sizeof(double)));
            h->plane_mem.push_back(h->el3_eplane);
        }
        if (want && !h->fused3 && h->ac && h->d3 && h->LS == 16 && h->LU == 16 &&
            ac3d_stream_eligible(desc->nx, desc->nm, h->g.pitch, dev_smem)) {
            if (ac3d_stream_prepare(desc->nx) != cudaSuccess) return fail(HW_ECUDA, "streaming kernel setup failed");
            const int64_t units = (desc->nm / (4096 / desc->nx)) * max_rows;
            int64_t nbs = units / 4;
            if (nbs < 1) nbs = 1;
            h->stream_blocks = (int)(nbs < nsm ? nbs : nsm);
            h->ac3_stream = true;
        }
        // one-pass 3D elastic step (2nd order, periodic, media constant along x): a single domain, or
        // one slab of a decomposed domain (ghost rows exchanged once per step, halo velocities
        // recomputed from them)
        ElParams EP;
        if (!h->ac && h->d3) fill_params(h, EP);
        if (want && opt("fused_el3") == 1 && !h->ac && h->d3 && h->LS == 16 && h->LU == 16 &&
            el3d_fused_eligible(EP, desc->nx, desc->nm, field_rows(h, F_SXX), h->g.pitch, desc->order, dev_smem)) {
            if ((rc = alloc_partner_buffers(h))) return rc;
            if (el3d_fused_prepare(desc->nx) != cudaSuccess) return fail(HW_ECUDA, "fused 3D elastic setup failed");
            h->el3_slab = h->world > 1 || h->transport != 0;
            h->el3_cm = el3d_fused_coef_rows(EP);
            const int64_t lo = h->el3_slab ? G : 0;  // slab: coefficient rows -G .. rows+G (halo velocities)
            CU(cudaMalloc(&h->el3_coef, (size_t)(max_rows + 2 * lo) * h->el3_cm * 8 * sizeof(float)));
            h->plane_mem.push_back(h->el3_coef);
            CU(el3d_fused_coef(EP, h->el3_coef, -lo, max_rows + 2 * lo, h->el3_cm, 0));
            h->el3_coef += lo * h->el3_cm * 8;  // (plane_mem keeps the allocation base)
            if (el3d_fused_erow(EP)) {
                CU(cudaMalloc(&h->el3_ecoef, (size_t)max_rows * 8 * sizeof(double)));
                h->plane_mem.push_back(h->el3_ecoef);
                CU(el3d_fused_ecoef(EP, h->el3_ecoef, max_rows, 0));
            }
            CU(cudaMalloc(&h->el3_eplane, (size_t)max_rows * (desc->nm / (2048 / desc->nx)) * sizeof(double)));
            h->plane_mem.push_back(h->el3_eplane);
            const int64_t units = (desc->nm / (2048 / desc->nx)) * max_rows;
            int64_t nbs = units / 4;
            if (nbs < 1) nbs = 1;
            h->stream_blocks = (int)(nbs < nsm ? nbs : nsm);
            const int64_t tiles = desc->nm / (2048 / desc->nx);
            for (int g : {4, 2, 1})
                if (g <= opt("el3_group") && h->stream_blocks % g == 0 && tiles % g == 0 &&
                    (tiles / g) * max_rows >= h->stream_blocks / g) {
                    h->el3_group = g;
                    break;
                }
            h->fused_el3 = true;
            // NCCL slab: edge slabs (every row the exchange sends) + the exchange on st, the interior
            // slabs on st2; CTAs split so both launches take about as long (an edge segment of
            // 2 slabs costs ~3 slabs: the ring fill)
            if (h->transport == 2 && max_rows >= 5 * EL3_EDGE && max_rows >= opt("el3_overlap_min_rows")) {
                if ((rc = make_overlap_streams(h))) return rc;
                const double we = 3.0 * 2 * EL3_EDGE, wi = (double)(max_rows - 2 * EL3_EDGE);
                int ne = opt("el3_edge_ctas") > 0 ? (int)opt("el3_edge_ctas") : (int)(nsm * EL3_EDGE_SHARE * we / (we + wi) + 0.5);
                ne = ne < 1 ? 1 : (ne > nsm / 2 ? nsm / 2 : ne);
                int ni = nsm - ne;
                if (ni % h->el3_group) ni -= ni % h->el3_group;
                h->el3_nb_edge = nsm - ni;  // (the CTAs the interior's group rounding leaves go to the edges)
                h->el3_nb_int = ni;
            }
        }
        if (want && !h->fused_el3 && !h->ac && h->d3 && h->LS == 16 && h->LU == 16 &&
            el3d_stream_eligible(desc->nx, desc->nm, h->g.pitch, desc->order, dev_smem)) {
            if (el3d_stream_prepare(desc->nx, desc->order) != cudaSuccess) return fail(HW_ECUDA, "streaming kernel setup failed");
            const int64_t units = (desc->nm / (2048 / desc->nx)) * max_rows;
            int64_t nbs = units / 4;
            if (nbs < 1) nbs = 1;
            h->stream_blocks = (int)(nbs < nsm ? nbs : nsm);
            h->el3_stream = true;
        }
        if (h->el_stream || h->ac3_stream || h->el3_stream || h->fused || h->fused3 || h->fused3_32 || h->fused_el ||
            h->fused_el3) {
            CU(cudaMalloc(&h->counter, sizeof(unsigned int)));
            CU(cudaMemset(h->counter, 0, sizeof(unsigned int)));
        }
    }
    if (!h->ctrl) CU(cudaMalloc(&h->ctrl, sizeof(Ctrl)));
    h->max_rows = max_rows;
    h->nblocks = grid_blocks(h->g, h->W, max_rows);
    {
        int64_t np = h->nblocks > h->stream_blocks ? h->nblocks : h->stream_blocks;
        const int64_t ntb = (int64_t)h->tb2_tiles * h->tb2_bands;
        np = np > ntb ? np : ntb;
        CU(cudaMalloc(&h->partials, 2 * np * NCOMP * sizeof(double)));
        h->partials_b = h->partials + np * NCOMP;
    }
    // the point source belongs to the slab holding its row
    int srcf = desc->src_kind == HW_SRC_PRESSURE ? F_P : (desc->src_kind == HW_SRC_VSLOW ? F_VS : F_SXX);
    if (desc->src_kind != HW_SRC_NONE && desc->src_s >= h->r0 && desc->src_s < h->r0 + field_rows(h, srcf)) {
        h->src_active = 1;
        h->src_s_loc = desc->src_s - h->r0;
    }
    if (desc->n_receivers > 0) {
        int f = h->ac ? F_P : F_VS;
        std::vector<int64_t> off(desc->n_receivers);
        h->rec_owned.assign(desc->n_receivers, 0);
        for (int j = 0; j < desc->n_receivers; j++) {
            const int64_t* r = desc->receivers + 3 * j;
            if (r[0] < 0 || r[0] >= desc->nx || r[1] < 0 || r[1] >= desc->nm || r[2] < 0 || r[2] >= nglob_rows(h, f))
                return fail(HW_EINVAL, "receiver outside the grid");
            const int64_t sl = r[2] - h->r0;
            const bool own = sl >= 0 && sl < field_rows(h, f);
            h->rec_owned[j] = own;
            off[j] = own ? sl * h->g.slab + r[1] * h->g.pitch + r[0] : -1;
        }
        CU(cudaMalloc(&h->rec_off, off.size() * 8));
        CU(cudaMemcpy(h->rec_off, off.data(), off.size() * 8, cudaMemcpyHostToDevice));
        std::vector<std::array<int, 3>> srt;
        for (int j = 0; j < desc->n_receivers; j++)
            if (h->rec_owned[j])  // key (local slow row * nm + mid row, x)
                srt.push_back({(int)((desc->receivers[3 * j + 2] - h->r0) * desc->nm + desc->receivers[3 * j + 1]),
                               (int)desc->receivers[3 * j], j});
        std::sort(srt.begin(), srt.end());
        h->n_rec_sorted = (int)srt.size();
        if (!srt.empty()) {
            CU(cudaMalloc(&h->rec_sorted, srt.size() * sizeof(srt[0])));
            CU(cudaMemcpy(h->rec_sorted, srt.data(), srt.size() * sizeof(srt[0]), cudaMemcpyHostToDevice));
        }
    }
    CU(cudaDeviceSynchronize());
    return HW_OK;
}

void release_handle(hw_solver* h) {
    cudaSetDevice(h->d.device);
    for (void* p : h->mem) if (p) cudaFree(p);
    for (void* p : h->mem_b) if (p) cudaFree(p);
    for (void* p : h->plane_mem) cudaFree(p);
    if (h->ctrl && h->owns_ctrl) cudaFree(h->ctrl);
    if (h->partials) cudaFree(h->partials);
    if (h->traces) cudaFree(h->traces);
    if (h->evals) cudaFree(h->evals);
    if (h->rec_off) cudaFree(h->rec_off);
    if (h->rec_sorted) cudaFree(h->rec_sorted);
    if (h->xch) cudaFree(h->xch);
    if (h->gbar) cudaFree(h->gbar);
    if (h->src_dev) cudaFree(h->src_dev);
    if (h->partials2) cudaFree(h->partials2);
    if (h->el3_etot) cudaFree(h->el3_etot);
    for (int k = 0; k < 2; k++) {
        if (h->ev_edge[k]) cudaEventDestroy(h->ev_edge[k]);
        if (h->ev_int[k]) cudaEventDestroy(h->ev_int[k]);
    }
    if (h->st2) cudaStreamDestroy(h->st2);
    if (h->counter) cudaFree(h->counter);
    if (h->ev0) cudaEventDestroy(h->ev0);
    if (h->ev1) cudaEventDestroy(h->ev1);
    if (h->ev_phase) cudaEventDestroy(h->ev_phase);
    if (h->ev_copied) cudaEventDestroy(h->ev_copied);
    if (h->st) cudaStreamDestroy(h->st);
    if (h->nccl && g_nccl.ok) g_nccl.CommDestroy(h->nccl);
    delete h;
}

// ---------------------------------------------------------------- halo exchange
// The halo plan is computed on the host from the slab geometry alone (no CUDA; exported as
// hw_exchange_plan) and executed by both transports.  Kinds:
//   HW_PLAN_VEL    after the velocity kernels: the velocities with slow-axis derivatives;
//   HW_PLAN_STRESS after the pressure / stress kernels: the rest of the ghosted fields;
//   HW_PLAN_FUSED  once per step of the fused 2D acoustic kernel on slabs: p (its redundant vy
//                  halo rows read p rows -3 .. L+2), vy and rvy (old values of those rows), G rows.
// Per field the phase kinds move the slow-axis stencil reach (1 row at 2nd order, 2 at 4th):
// bottom rows -> next rank's top ghosts and top rows -> previous rank's bottom ghosts, in a
// canonical order (every field's bottom-going pair, then every field's top-going pair) so that
// paired send/recv match even when previous == next (N = 2, periodic) or both are the rank
// itself (one-rank NCCL self exchange).  Free surfaces: the global ends keep their images.
struct PlanGeom {
    int ac, d3, fs, order, world, rank, nsol;
    int64_t ns_loc;
    const int* ext;
};

PlanGeom plan_geom(const hw_solver* h) {
    return PlanGeom{h->ac ? 1 : 0, h->d3 ? 1 : 0, h->fs ? 1 : 0, h->d.order, h->world, h->rank, h->nsol, h->ns_loc,
                    h->ext};
}

int64_t pg_rows(const PlanGeom& g, int f) {
    return g.ns_loc + ((g.fs && !HALF_S[f] && g.rank == g.world - 1) ? 1 : 0);
}
bool pg_ghosts(const PlanGeom& g, int f) {
    if (g.ac) return f == F_P || f == F_VS;
    return f == F_VX || f == F_VS || f == F_VM || f == F_SXS || f == F_SSS || f == F_SMS;
}
int pg_prev(const PlanGeom& g) { return g.rank > 0 ? g.rank - 1 : (g.fs ? -1 : g.world - 1); }
int pg_next(const PlanGeom& g) { return g.rank < g.world - 1 ? g.rank + 1 : (g.fs ? -1 : 0); }

std::vector<hw_xfer> halo_plan(const PlanGeom& g, int kind) {
    std::vector<int> js;   // external field indices, in external order
    int64_t depth = 0;
    std::vector<int64_t> dep;  // per-field depth (HW_PLAN_FUSED_EL3)
    if (kind == HW_PLAN_FUSED) {
        js = {0, 2, 5};  // p, vy, rvy of p vx vy rp rvx rvy
        depth = G;
    } else if (kind == HW_PLAN_FUSED_EL2) {
        // one-pass 2D elastic slab (hw_elastic2d_fused.cu): its CTAs stream rows -3 .. L+2 and recompute
        // the velocity rows of the halo: the five fields and the velocity residuals, G rows each way
        js = {0, 1, 2, 3, 4, 5, 6};  // vx vy sxx syy sxy rvx rvy
        depth = G;
    } else if (kind == HW_PLAN_FUSED_AC3) {
        // one-pass 3D acoustic slab: p rows -1 and L, v_slow and its residual row -1 (1 row each way)
        for (int j = 0; j < g.nsol; j++)
            if (g.ext[j] == F_P || g.ext[j] == F_VS) js.push_back(j);
        for (int j = 0; j < g.nsol; j++)
            if (g.ext[j] == F_VS) js.push_back(g.nsol + j);
        depth = 1;
    } else if (kind == HW_PLAN_FUSED_EL3) {
        // one-pass 3D elastic slab (hw_elastic3d_fused.cu): its halo velocities v(-1), v(L) are
        // recomputed from stress rows -2 .. L and the old velocities / residuals of rows -1, L
        js = {3, 4, 5, 6, 7, 8, 0, 1, 2, 9, 10, 11};  // sxx syy szz sxy sxz syz, vx vy vz, rvx rvy rvz
        dep = {2, 2, 2, 2, 2, 2, 1, 1, 1, 1, 1, 1};
    } else {
        for (int j = 0; j < g.nsol; j++) {
            const int f = g.ext[j];
            if (pg_ghosts(g, f) && is_velocity(f) == (kind == HW_PLAN_VEL)) js.push_back(j);
        }
        depth = g.order == 2 ? 1 : 2;
    }
    const int pv = pg_prev(g), nx_ = pg_next(g);
    std::vector<hw_xfer> out;
    for (size_t q = 0; q < js.size(); q++) {
        const int j = js[q];
        const int64_t n = pg_rows(g, g.ext[j % g.nsol]), d = dep.empty() ? depth : dep[q];
        if (nx_ >= 0) out.push_back(hw_xfer{j, nx_, 1, 0, n - d, d});
        if (pv >= 0) out.push_back(hw_xfer{j, pv, 0, 0, -d, d});
    }
    for (size_t q = 0; q < js.size(); q++) {
        const int j = js[q];
        const int64_t n = pg_rows(g, g.ext[j % g.nsol]), d = dep.empty() ? depth : dep[q];
        if (pv >= 0) out.push_back(hw_xfer{j, pv, 1, 0, 0, d});
        if (nx_ >= 0) out.push_back(hw_xfer{j, nx_, 0, 0, n, d});
    }
    return out;
}

// Device address of local row `row` of external field j for a plan kind (buf: fused 2D
// ping-pong buffer, 0 = A, 1 = B).
char* plan_row(const hw_solver* h, int kind, int buf, int j, int64_t row) {
    const size_t rb = (size_t)h->g.slab * lane_bytes(h->LU);
    char* base;
    if (kind >= HW_PLAN_FUSED) base = (char*)(buf ? h->mem_b[j] : h->mem[j]) + G * rb;  // ping-pong buffers
    else base = (char*)(j < h->nsol ? h->fv : h->rv)[h->ext[j % h->nsol]].base;
    return base + row * (int64_t)rb;
}

int exchange_nccl_plan(hw_solver* h, int kind, int buf) {
    const size_t rb = (size_t)h->g.slab * lane_bytes(h->LU);
    NC(g_nccl.GroupStart());
    for (const hw_xfer& x : halo_plan(plan_geom(h), kind)) {
        void* p = plan_row(h, kind, buf, x.field, x.row0);
        if (x.send) NC(g_nccl.Send(p, x.nrows * rb, ncclInt8, x.peer, h->nccl, h->st));
        else NC(g_nccl.Recv(p, x.nrows * rb, ncclInt8, x.peer, h->nccl, h->st));
    }
    NC(g_nccl.GroupEnd());
    if (kind != HW_PLAN_VEL) {
        // every rank learns the first failing step of every rank before its next step's kernels
        // (they exit at entry past it): the state of every rank stops exactly after the global
        // first failing step (acoustic.py:208-229); the overlapped fused 2D path may run one
        // interior band further into the other ping-pong buffer, which the copy-back discards
        NC(g_nccl.AllReduce(&h->ctrl->fail_step, &h->ctrl->gfail_step, 1, ncclInt64, ncclMin, h->nccl, h->st));
    }
    return HW_OK;
}

int exchange_nccl(hw_solver* h, int phase) { return exchange_nccl_plan(h, phase == 0 ? HW_PLAN_VEL : HW_PLAN_STRESS, 0); }

// In-process slab group: every rank pulls its ghosts from its neighbours' slabs with peer
// copies ordered by events (one GPU or NVLink peers).  The k-th receive of rank b from rank a
// takes the k-th send of a to b, as NCCL pairs point-to-point operations.
int exchange_group_plan(hw_group* grp, int kind, int buf) {
    for (hw_solver* h : grp->ranks) {
        CU(cudaSetDevice(h->d.device));
        CU(cudaEventRecord(h->ev_phase, h->st));
    }
    const size_t rb = (size_t)grp->ranks[0]->g.slab * lane_bytes(grp->ranks[0]->LU);
    for (hw_solver* b : grp->ranks) {
        CU(cudaSetDevice(b->d.device));
        const std::vector<hw_xfer> mine = halo_plan(plan_geom(b), kind);
        std::vector<int> waited;
        for (size_t k = 0; k < mine.size(); k++) {
            const hw_xfer& r = mine[k];
            if (r.send) continue;
            hw_solver* a = grp->ranks[r.peer];
            if (std::find(waited.begin(), waited.end(), r.peer) == waited.end()) {
                CU(cudaStreamWaitEvent(b->st, a->ev_phase, 0));
                waited.push_back(r.peer);
            }
            int nth = 0;  // r is the nth receive of b from a
            for (size_t q = 0; q < k; q++) nth += (!mine[q].send && mine[q].peer == r.peer) ? 1 : 0;
            const std::vector<hw_xfer> theirs = halo_plan(plan_geom(a), kind);
            const hw_xfer* s = nullptr;
            for (const hw_xfer& t : theirs)
                if (t.send && t.peer == b->rank && nth-- == 0) {
                    s = &t;
                    break;
                }
            if (!s || s->nrows != r.nrows || s->field != r.field) return fail(HW_EINVAL, "inconsistent halo plan");
            CU(cudaMemcpyPeerAsync(plan_row(b, kind, buf, r.field, r.row0), b->d.device,
                                   plan_row(a, kind, buf, s->field, s->row0), a->d.device, r.nrows * rb, b->st));
        }
        CU(cudaEventRecord(b->ev_copied, b->st));
    }
    // a rank may overwrite its boundary rows only after its neighbours copied them
    for (hw_solver* a : grp->ranks) {
        CU(cudaSetDevice(a->d.device));
        const PlanGeom g = plan_geom(a);
        const int pv = pg_prev(g), nx_ = pg_next(g);
        if (pv >= 0) CU(cudaStreamWaitEvent(a->st, grp->ranks[pv]->ev_copied, 0));
        if (nx_ >= 0) CU(cudaStreamWaitEvent(a->st, grp->ranks[nx_]->ev_copied, 0));
    }
    return HW_OK;
}

int exchange_group(hw_group* grp, int phase) {
    return exchange_group_plan(grp, phase == 0 ? HW_PLAN_VEL : HW_PLAN_STRESS, 0);
}

int exchange(hw_solver* h, int phase) {
    if (h->transport == 2) return exchange_nccl(h, phase);
    if (h->world == 1) return HW_OK;
    return HW_OK;  // group ranks are exchanged by the group driver
}

// Decomposition-invariant energy of the one-pass 3D elastic kernel: E_k = scale * (sum over the
// global slow planes, in order, of the plane totals T_k[s]) -- bit-identical for any slab count.
// planes[r] holds rank r's [ne][rows_r] totals.
void el3_energy_from_planes(const std::vector<std::vector<double>>& planes, const std::vector<int64_t>& rows,
                            int64_t ne, double scale, double* e_vals) {
    for (int64_t k = 0; k < ne; k++) {
        double t = 0.0;
        bool first = true;
        for (size_t r = 0; r < planes.size(); r++)
            for (int64_t sp = 0; sp < rows[r]; sp++) {
                const double v = planes[r][k * rows[r] + sp];
                t = first ? v : t + v;
                first = false;
            }
        e_vals[k] = scale * t;
    }
}

double C_scale(const hw_solver* h) { return 0.5 * h->d.dx * h->d.dx * (h->d3 ? h->d.dx : 1.0); }

int el3_planes_host(hw_solver* h, int64_t ne, std::vector<double>& out) {
    out.resize(ne * h->max_rows);
    CU(cudaSetDevice(h->d.device));
    CU(cudaStreamSynchronize(h->st));
    if (ne > 0) CU(cudaMemcpy(out.data(), h->el3_etot, out.size() * sizeof(double), cudaMemcpyDeviceToHost));
    return HW_OK;
}

}  // namespace

extern "C" {

int hw_num_fields(int32_t equation, int32_t ndim) {
    int nsol;
    ext_order(equation, ndim, &nsol);
    return 2 * nsol;
}

int hw_field_shape(const hw_desc* d, int32_t field, int64_t shape[3]) {
    int nsol;
    const int* ext = ext_order(d->equation, d->ndim, &nsol);
    if (field < 0 || field >= 2 * nsol) return fail(HW_EINVAL, "field index out of range");
    int f = ext[field % nsol];
    shape[0] = d->ns + ((d->bc_slow == HW_BC_FREE_SURFACE && !HALF_S[f]) ? 1 : 0);
    shape[1] = d->nm;
    shape[2] = d->nx;
    return HW_OK;
}

int hw_nccl_unique_id(void* out128) {
    int rc = nccl_load();
    if (rc) return rc;
    ncclUniqueId id;
    NC(g_nccl.GetUniqueId(&id));
    memcpy(out128, &id, sizeof(id));
    return HW_OK;
}

int hw_create(const hw_desc* desc, hw_solver** out) {
    int rc = check_desc(desc);
    if (rc) return rc;
    hw_solver* h = new hw_solver();
    h->d = *desc;
    h->world = desc->world_size;
    h->rank = desc->rank;
    // option nccl_self (test hook): a one-rank job still takes the NCCL transport, its
    // periodic ghosts filled by send/recv to itself, so the whole NCCL path runs on one GPU
    const bool nccl_self = h->world == 1 && opt("nccl_self") == 1 && desc->nccl_unique_id;
    if (h->world > 1 || nccl_self) {  // one process per GPU: NCCL transport
        if (!desc->nccl_unique_id) { release_handle(h); return fail(HW_EINVAL, "world_size > 1 needs nccl_unique_id"); }
        if ((rc = nccl_load())) { release_handle(h); return rc; }
        h->transport = 2;
        CU(cudaSetDevice(desc->device));
        ncclUniqueId id;
        memcpy(&id, desc->nccl_unique_id, sizeof(id));
        ncclResult_t r = g_nccl.CommInitRank(&h->nccl, h->world, id, h->rank);
        if (r != ncclSuccess) { release_handle(h); return fail(HW_ENCCL, std::string("ncclCommInitRank: ") + g_nccl.GetErrorString(r)); }
    }
    if ((rc = setup_handle(h))) { release_handle(h); return rc; }
    *out = h;
    return HW_OK;
}

int hw_create_group(const hw_desc* desc, int32_t nslabs, const int32_t* devices, hw_solver** out) {
    hw_desc d = *desc;
    d.world_size = nslabs;
    d.rank = 0;
    int rc = check_desc(&d);
    if (rc) return rc;
    hw_group* grp = new hw_group();
    Ctrl* shared = nullptr;
    for (int r = 0; r < nslabs; r++) {
        hw_solver* h = new hw_solver();
        h->d = d;
        h->d.rank = r;
        h->d.device = devices ? devices[r] : desc->device;
        h->world = nslabs;
        h->rank = r;
        h->transport = 1;
        h->group = grp;
        if (r == 0) {
            CU(cudaSetDevice(h->d.device));
            CU(cudaMalloc(&shared, sizeof(Ctrl)));  // one run-control block: exact failure semantics
        } else {
            h->owns_ctrl = false;
            if (h->d.device != grp->ranks[0]->d.device) {
                cudaSetDevice(h->d.device);
                cudaDeviceEnablePeerAccess(grp->ranks[0]->d.device, 0);
                cudaGetLastError();
            }
        }
        h->ctrl = shared;
        grp->ranks.push_back(h);
        if ((rc = setup_handle(h))) {
            for (hw_solver* x : grp->ranks) release_handle(x);
            delete grp;
            return rc;
        }
        out[r] = h;
    }
    return HW_OK;
}

int hw_destroy(hw_solver* h) {
    if (!h) return HW_OK;
    hw_group* grp = h->group;
    if (grp) {  // destroying any rank of a group releases the whole group
        for (hw_solver* x : grp->ranks) release_handle(x);
        delete grp;
        return HW_OK;
    }
    release_handle(h);
    return HW_OK;
}

int hw_set_state(hw_solver* h, const void* const* fields) {
    CU(cudaSetDevice(h->d.device));
    int esz = lane_bytes(h->LU);
    const size_t off = (size_t)h->r0 * h->d.nm * h->d.nx * esz;  // this slab's rows of the global arrays
    for (int j = 0; j < 2 * h->nsol; j++) {
        int f = h->ext[j % h->nsol];
        const FieldView& fv = j < h->nsol ? h->fv[f] : h->rv[f];
        const char* src = (const char*)fields[j] + off;
        CU(cudaMemcpy2DAsync(fv.base, h->g.pitch * esz, src, h->d.nx * esz, h->d.nx * esz, fv.rows * h->d.nm,
                             cudaMemcpyHostToDevice, h->st));
        if ((fv.gtop | fv.gbot) != GHOST_NONE) {
            int64_t nthr = 2 * G * h->d.nm * h->d.nx;
            int64_t nb = (nthr + 255) / 256;
            if (esz == 2) k_fill_ghosts<__half><<<nb, 256, 0, h->st>>>(fv, h->g);
            else if (esz == 4) k_fill_ghosts<float><<<nb, 256, 0, h->st>>>(fv, h->g);
            else k_fill_ghosts<double><<<nb, 256, 0, h->st>>>(fv, h->g);
        }
    }
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(h->st));
    return HW_OK;  // ghosts facing other ranks are exchanged at the start of each run
}

int hw_get_state(hw_solver* h, void* const* fields) {
    CU(cudaSetDevice(h->d.device));
    int esz = lane_bytes(h->LU);
    const size_t off = (size_t)h->r0 * h->d.nm * h->d.nx * esz;
    for (int j = 0; j < 2 * h->nsol; j++) {
        int f = h->ext[j % h->nsol];
        const FieldView& fv = j < h->nsol ? h->fv[f] : h->rv[f];
        CU(cudaMemcpy2DAsync((char*)fields[j] + off, h->d.nx * esz, fv.base, h->g.pitch * esz, h->d.nx * esz,
                             fv.rows * h->d.nm, cudaMemcpyDeviceToHost, h->st));
    }
    CU(cudaStreamSynchronize(h->st));
    return HW_OK;
}

static int ensure(double** p, int64_t* cap, int64_t need) {
    if (need <= *cap) return HW_OK;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *cap = 0;
    CU(cudaMalloc(p, need * sizeof(double)));
    *cap = need;
    return HW_OK;
}

// Per-run setup shared by every driver: buffers, control block, kernel params, E(0).
struct RunCtx {
    EpParams E;
    AcParams A;
    ElParams L;
    int64_t nt = 0, every = 1;
    bool energy = false;
    int variant = 0;
};

static int run_begin(hw_solver* h, int32_t variant, int64_t nt, bool energy, bool reset_ctrl, RunCtx& C) {
    if (variant != HW_NAIVE && variant != HW_OP3 && variant != HW_OP6) return fail(HW_EINVAL, "bad variant");
    if (nt < 0) return fail(HW_EINVAL, "nt must be nonnegative");
    CU(cudaSetDevice(h->d.device));
    int rc;
    const int64_t nrec = h->d.n_receivers;
    if ((rc = ensure(&h->traces, &h->traces_cap, nrec * nt > 0 ? nrec * nt : 1))) return rc;
    if ((rc = ensure(&h->evals, &h->evals_cap, 1 + nt / h->d.energy_every))) return rc;
    if (nrec * nt > 0) CU(cudaMemsetAsync(h->traces, 0, nrec * nt * sizeof(double), h->st));
    if (reset_ctrl) {
        Ctrl c0;
        c0.fail_step = INT64_MAX;
        c0.fail_mask = 0;
        c0.pad = 0;
        c0.gfail_step = INT64_MAX;
        CU(cudaMemcpyAsync(h->ctrl, &c0, sizeof(Ctrl), cudaMemcpyHostToDevice, h->st));
    }
    if (variant == HW_NAIVE && nt > 0) {  // untouched non-finite residuals fail step 0
        const int esz = lane_bytes(h->LU);
        for (int j = h->nsol; j < 2 * h->nsol; j++) {
            const FieldView& fv = h->rv[h->ext[j - h->nsol]];
            dim3 gr((unsigned)((h->d.nx + 255) / 256), (unsigned)h->d.nm, (unsigned)fv.rows);
            if (esz == 2) k_flag_nonfinite<__half><<<gr, 256, 0, h->st>>>((const __half*)fv.base, h->g, fv.rows, j, h->ctrl);
            else if (esz == 4) k_flag_nonfinite<float><<<gr, 256, 0, h->st>>>((const float*)fv.base, h->g, fv.rows, j, h->ctrl);
            else k_flag_nonfinite<double><<<gr, 256, 0, h->st>>>((const double*)fv.base, h->g, fv.rows, j, h->ctrl);
        }
    }
    memset(&C.E, 0, sizeof(C.E));
    C.E.trace_base = (h->ac ? h->fv[F_P] : h->fv[F_VS]).base;
    C.E.rec_off = h->rec_off;
    C.E.n_rec = (int32_t)nrec;
    C.E.nblocks = (int32_t)h->nblocks;
    C.E.traces = h->traces;
    C.E.nt = nt;
    C.E.e_vals = h->evals;
    C.E.scale = 0.5 * h->d.dx * h->d.dx * (h->d3 ? h->d.dx : 1.0);
    C.E.partials = h->partials;
    C.E.ctrl = h->ctrl;
    if (h->ac) fill_params(h, C.A);
    else fill_params(h, C.L);
    C.A.variant = C.L.variant = variant;
    C.variant = variant;
    C.nt = nt;
    C.every = h->d.energy_every;
    C.energy = energy;
    h->launches = 0;
    if (h->plane_energy() && energy) {  // energy plane totals per sample (el3_energy_from_planes)
        int64_t cap = h->el3_etot_cap;
        if ((rc = ensure(&h->el3_etot, &cap, (1 + nt / h->d.energy_every) * h->max_rows))) return rc;
        h->el3_etot_cap = cap;
    }
    if (energy) {  // E(t=0) pairs the state with itself
        if (h->ac) launch_ac_energy(h->LU, h->W, C.A, h->max_rows, h->st);
        else launch_el_energy(h->LU, h->W, C.L, h->max_rows, h->st);
        h->launches++;
        if (!h->plane_energy()) {
            launch_epilogue(h->LU, C.E, -1, 1, 0, h->st);
            h->launches++;
        } else {  // ... and its per-slab totals (one block partial per (x chunk, mid row, slab))
            const dim3 gr = grid3(h->g, h->W, h->max_rows);
            launch_plane_totals(h->partials, (int64_t)gr.x * gr.y, h->max_rows, h->el3_etot, h->st);
            h->launches++;
        }
    }
    CU(cudaGetLastError());
    return HW_OK;
}

static StreamIO stream_io(const hw_solver* h, const RunCtx& C) {
    StreamIO IO;
    memset(&IO, 0, sizeof(IO));
    IO.rec = h->rec_sorted;
    IO.n_rec = h->n_rec_sorted;
    IO.traces = h->traces;
    IO.nt = C.nt;
    IO.e_vals = h->evals;
    IO.scale = C.E.scale;
    IO.counter = h->counter;
    return IO;
}

// one leapfrog phase (0 = velocities, 1 = pressure / stresses) of step n
static void run_phase(hw_solver* h, const RunCtx& C, int phase, int64_t n, const double* src) {
    const int sk = h->d.src_kind;
    const double s = src ? src[n] : 0.0;
    const int sample = C.energy && ((n + 1) % C.every == 0);
    if (phase == 0) {
        if (h->ac3_stream) launch_ac3d_vel_stream(C.variant, h->d.order, C.A, h->stream_blocks, n, h->st);
        else if (h->ac) launch_ac_vel(h->LS, h->LU, h->W, C.A, n, h->max_rows, h->st);
        else if (h->el3_stream)
            launch_el3d_vel_stream(C.variant, h->d.order, C.L, h->stream_blocks, n, sk == HW_SRC_VSLOW ? s : 0.0, h->st);
        else if (h->el_stream) launch_el2d_vel_stream(C.variant, h->d.order, C.L, stream_io(h, C), h->stream_blocks, n,
                                                      sk == HW_SRC_VSLOW ? s : 0.0, h->st);
        else launch_el_vel(h->LS, h->LU, h->W, C.L, n, sk == HW_SRC_VSLOW ? s : 0.0, h->max_rows, h->st);
    } else {
        if (h->ac3_stream)
            launch_ac3d_pres_stream(C.variant, h->d.order, C.A, stream_io(h, C), h->stream_blocks, n,
                                    sk == HW_SRC_PRESSURE ? s : 0.0, sample, (n + 1) / C.every, h->st);
        else if (h->ac) launch_ac_pres(h->LS, h->LU, h->W, C.A, n, sk == HW_SRC_PRESSURE ? s : 0.0, sample, h->max_rows, h->st);
        else if (h->el3_stream)
            launch_el3d_stress_stream(C.variant, h->d.order, C.L, stream_io(h, C), h->stream_blocks, n,
                                      sk == HW_SRC_EXPLOSIVE ? s : 0.0, sample, (n + 1) / C.every, h->st);
        else if (h->el_stream)
            launch_el2d_stress_stream(C.variant, h->d.order, C.L, stream_io(h, C), h->stream_blocks, n,
                                      sk == HW_SRC_EXPLOSIVE ? s : 0.0, sample, (n + 1) / C.every, h->st);
        else launch_el_stress(h->LS, h->LU, h->W, C.L, n, sk == HW_SRC_EXPLOSIVE ? s : 0.0, sample, h->max_rows, h->st);
    }
    h->launches++;
}

static void run_epilogue(hw_solver* h, const RunCtx& C, int64_t n) {
    const int sample = C.energy && ((n + 1) % C.every == 0);
    if (h->el_stream || h->ac3_stream) return;  // traces and energy are recorded inside the streaming kernels
    if (h->el3_stream) {  // energy is finalised inside; receiver traces from the epilogue
        if (C.E.n_rec > 0) {
            launch_epilogue(h->LU, C.E, n, 0, 0, h->st);
            h->launches++;
        }
        return;
    }
    if (sample || C.E.n_rec > 0) {
        launch_epilogue(h->LU, C.E, n, sample, (n + 1) / C.every, h->st);
        h->launches++;
    }
}

// Parameters of the fused 2D kernels (in / out buffers are set per launch).
static AcFusedParams fused_params(const hw_solver* h, int64_t nt) {
    AcFusedParams F;
    memset(&F, 0, sizeof(F));
    F.nx = h->d.nx;
    F.ns = field_rows(h, F_P);  // local rows (= ns in a single domain)
    F.pitch = h->g.pitch;
    F.slab = (h->world > 1 || h->transport == 2) ? 1 : 0;
    F.counter = h->counter;
    F.rho_x = h->lp[HW_PL_RHO_X]; F.rho_s = h->lp[HW_PL_RHO_S]; F.beta = h->lp[HW_PL_BETA];
    F.e_beta = h->ep64[HW_PL_BETA]; F.e_rho_x = h->ep64[HW_PL_RHO_X]; F.e_rho_s = h->ep64[HW_PL_RHO_S];
    F.k = make_consts(h->d.taps, h->dt_u);
    F.has_src = h->d.src_kind == HW_SRC_PRESSURE && h->src_active;
    F.src_x = h->d.src_x;
    F.src_s = h->src_s_loc;
    F.n_rec = h->n_rec_sorted;
    F.rec = h->rec_sorted;
    F.traces = h->traces;
    F.nt = nt;
    F.ctrl = h->ctrl;
    F.partials = h->partials;
    F.e_vals = h->evals;
    F.scale = 0.5 * h->d.dx * h->d.dx;
    return F;
}

// Field views / input pointers of the one-pass 3D kernel reading buffer `cur` (0 = A,
// 1 = B) and writing the other one (same ghost policies: write-through periodic slabs).
static void fused3_bufs(const hw_solver* h, int cur, AcParams& P, Ac3In& in) {
    const int64_t ghost = (int64_t)G * h->g.slab * lane_bytes(h->LU);  // bytes before row 0
    const __half* src[2 * F_N] = {};
    for (int j = 0; j < 2 * h->nsol; j++) {
        const int f = h->ext[j % h->nsol];
        void* const* rd = cur ? h->mem_b : h->mem;
        void* const* wr = cur ? h->mem : h->mem_b;
        FieldView& v = j < h->nsol ? (f == F_P ? P.p : f == F_VX ? P.vx : f == F_VS ? P.vs : P.vm)
                                   : (f == F_P ? P.rp : f == F_VX ? P.rvx : f == F_VS ? P.rvs : P.rvm);
        v.base = (char*)wr[j] + ghost;
        src[(j < h->nsol ? 0 : F_N) + f] = (const __half*)((const char*)rd[j] + ghost);
    }
    in.p = src[F_P]; in.vx = src[F_VX]; in.vs = src[F_VS]; in.vm = src[F_VM];
    in.rp = src[F_N + F_P]; in.rvx = src[F_N + F_VX]; in.rvs = src[F_N + F_VS]; in.rvm = src[F_N + F_VM];
    in.slab = (h->world > 1 || h->transport != 0) ? 1 : 0;
    in.group = h->el3_group;
    in.band = in.edge = in.nb_total = in.pad = 0;
    in.eplane = h->el3_eplane;
    in.etot = h->el3_etot;
}

// The same for the one-pass 2D elastic kernel (external order vx vy sxx syy sxy + residuals).
static void fused_el_bufs(const hw_solver* h, int cur, ElParams& P, El2In& in) {
    const int64_t ghost = (int64_t)G * h->g.slab * 2;  // bytes before row 0
    void* const* rd = cur ? h->mem_b : h->mem;
    void* const* wr = cur ? h->mem : h->mem_b;
    FieldView* out[10] = {&P.vx, &P.vs, &P.sxx, &P.sss, &P.sxs, &P.rvx, &P.rvs, &P.rsxx, &P.rsss, &P.rsxs};
    const __half** src[10] = {&in.vx, &in.vs, &in.sxx, &in.sss, &in.sxs, &in.rvx, &in.rvs, &in.rsxx, &in.rsss, &in.rsxs};
    for (int j = 0; j < 10; j++) {  // EXT_EL2 = vx vs sxx sss sxs: slot j holds field j (j % 5)
        out[j]->base = (char*)wr[j] + ghost;
        *src[j] = (const __half*)((const char*)rd[j] + ghost);
    }
    in.slab = (h->world > 1 || h->transport != 0) ? 1 : 0;
    in.top = h->rank == 0;
    in.bot = h->rank == h->world - 1;
    in.vsrc = 0;
    in.vsrc_s = 0;
    in.band = in.edge = in.nb_total = in.pad = 0;
    if (h->d.src_kind == HW_SRC_VSLOW) {  // this slab also computes the halo velocity rows -3 .. rows + 2
        const int64_t r = h->d.src_s - h->r0;
        if (r >= -G && r < field_rows(h, F_VS) + G) {
            in.vsrc = 1;
            in.vsrc_s = r;
        }
    }
}

// The same for the one-pass 3D elastic kernel.
static void fused_el3_bufs(const hw_solver* h, int cur, ElParams& P, El3In& in) {
    const int64_t ghost = (int64_t)G * h->g.slab * 2;  // bytes before row 0
    void* const* rd = cur ? h->mem_b : h->mem;
    void* const* wr = cur ? h->mem : h->mem_b;
    for (int j = 0; j < 2 * h->nsol; j++) {
        const int f = h->ext[j % h->nsol];
        const bool r = j >= h->nsol;
        FieldView* o = nullptr;
        const __half** q = nullptr;
        switch (f) {
            case F_VX: o = r ? &P.rvx : &P.vx; q = r ? &in.rvx : &in.vx; break;
            case F_VS: o = r ? &P.rvs : &P.vs; q = r ? &in.rvs : &in.vs; break;
            case F_VM: o = r ? &P.rvm : &P.vm; q = r ? &in.rvm : &in.vm; break;
            case F_SXX: o = r ? &P.rsxx : &P.sxx; q = r ? &in.rsxx : &in.sxx; break;
            case F_SSS: o = r ? &P.rsss : &P.sss; q = r ? &in.rsss : &in.sss; break;
            case F_SMM: o = r ? &P.rsmm : &P.smm; q = r ? &in.rsmm : &in.smm; break;
            case F_SXS: o = r ? &P.rsxs : &P.sxs; q = r ? &in.rsxs : &in.sxs; break;
            case F_SXM: o = r ? &P.rsxm : &P.sxm; q = r ? &in.rsxm : &in.sxm; break;
            default: o = r ? &P.rsms : &P.sms; q = r ? &in.rsms : &in.sms; break;
        }
        o->base = (char*)wr[j] + ghost;
        *q = (const __half*)((const char*)rd[j] + ghost);
    }
    in.coef = h->el3_coef;
    in.coef_m = h->el3_cm;
    in.div_mode[0] = h->lp[HW_PL_RHO_X].div_mode;
    in.div_mode[1] = h->lp[HW_PL_RHO_S].div_mode;
    in.div_mode[2] = h->lp[HW_PL_RHO_M].div_mode;
    in.group = h->el3_group;
    in.ecoef = h->el3_ecoef;
    in.eplane = h->el3_eplane;
    in.etot = h->el3_etot;
    in.slab = h->el3_slab ? 1 : 0;
    in.vsrc = 0;
    in.vsrc_s = 0;
    in.band = 0;
    in.edge = 0;
    in.nb_total = 0;
    in.pad2 = 0;
    if (h->d.src_kind == HW_SRC_VSLOW) {  // this slab also computes the halo velocity rows -1 and L
        const int64_t r = h->d.src_s - h->r0;
        if (r >= -1 && r <= h->ns_loc) {
            in.vsrc = 1;
            in.vsrc_s = r;
        }
    }
}

static void fused_bufs(const hw_solver* h, __half* bufs[2][FUSED_NSTREAM]) {
    const int64_t ghost = (int64_t)G * h->g.slab * 2;  // bytes before row 0
    for (int j = 0; j < FUSED_NSTREAM; j++) {  // external order p vx vy rp rvx rvy == stream order
        bufs[0][j] = (__half*)((char*)h->mem[j] + ghost);
        bufs[1][j] = (__half*)((char*)h->mem_b[j] + ghost);
    }
}

// The time loop (acoustic.py:210-226 / elastic.py:271-286) of one handle on the device.
static int run_impl(hw_solver* h, int32_t variant, int64_t nt, const double* src, bool energy, bool timed) {
    if (h->transport == 1) return fail(HW_EINVAL, "slab-group handles run through hw_run_group");
    RunCtx C;
    int rc = run_begin(h, variant, nt, energy, true, C);
    if (rc) return rc;
    const bool fused_slab = h->fused && h->transport == 2;
    if (fused_slab || (h->transport == 2 && (h->fused_el3 || h->fused3 || h->fused3_32 || h->fused_el))) {  // halos
        const int kind = fused_slab ? HW_PLAN_FUSED
                                    : (h->fused_el3 ? HW_PLAN_FUSED_EL3 : (h->fused_el ? HW_PLAN_FUSED_EL2 : HW_PLAN_FUSED_AC3));
        if ((rc = exchange_nccl_plan(h, kind, 0))) return rc;
    } else if ((rc = exchange(h, 0)) || (rc = exchange(h, 1))) {
        return rc;
    }
    if (timed) CU(cudaEventRecord(h->ev0, h->st));
    if (h->small || h->small_el) {  // every step in one cooperative launch (hw_small2d.cu)
        if (src && nt > h->src_cap) {
            if (h->src_dev) cudaFree(h->src_dev);
            h->src_dev = nullptr;
            h->src_cap = 0;
            CU(cudaMalloc(&h->src_dev, nt * sizeof(double)));
            h->src_cap = nt;
        }
        if (src && nt > 0) CU(cudaMemcpyAsync(h->src_dev, src, nt * sizeof(double), cudaMemcpyHostToDevice, h->st));
        CU(cudaMemsetAsync(h->gbar, 0, 2 * sizeof(unsigned int), h->st));
        if (h->small_el) {
            if (nt > 0) {
                CU(launch_el2d_small(variant, h->d.order, C.L, stream_io(h, C), h->xch, h->gbar,
                                     src ? h->src_dev : nullptr, h->partials2, (int)C.every, energy ? 1 : 0,
                                     h->small_nb, nt, h->st));
                h->launches++;
            }
        } else {
            AcFusedParams F = fused_params(h, nt);
            for (int j = 0; j < FUSED_NSTREAM; j++)
                F.in[j] = F.out[j] = (__half*)((char*)h->mem[j] + (int64_t)G * h->g.slab * 2);
            if (nt > 0) {
                CU(launch_ac2d_small(variant, h->d.order, F, h->xch, h->gbar, src ? h->src_dev : nullptr, h->partials2,
                                     (int)C.every, energy ? 1 : 0, h->small_nb, nt, h->st));
                h->launches++;
            }
        }
    } else if (h->fused && fused_slab && h->st2) {
        // NCCL slab, overlapped: per step the two thin edge bands run first on st and the
        // ghost exchange follows them on st, while the interior bands run on st2.
        //   st : wait interior(n-1) | edge(n) | record E(n) | exchange(n)
        //   st2: wait edge(n-1)     | interior(n) | record I(n)
        // (edge(n) overwrites rows interior(n-1) reads and vice versa: ping-pong buffers)
        AcFusedParams F = fused_params(h, nt);
        __half* bufs[2][FUSED_NSTREAM];
        fused_bufs(h, bufs);
        const int64_t every = C.every;
        AcFusedParams Fe = F, Fi = F;
        Fe.band_mode = 1;
        Fi.band_mode = 2;
        Fe.edge = Fi.edge = FUSED_EDGE;
        Fe.nb_total = Fi.nb_total = 2 + h->nb_int;
        CU(cudaEventRecord(h->ev_edge[1], h->st));  // st2 starts after everything queued on st
        int cur = 0;
        for (int64_t n = 0; n < nt; n++) {
            for (int j = 0; j < FUSED_NSTREAM; j++) {
                Fe.in[j] = Fi.in[j] = bufs[cur][j];
                Fe.out[j] = Fi.out[j] = bufs[cur ^ 1][j];
            }
            const double sv = src ? src[n] : 0.0;
            const int sample = energy && ((n + 1) % every == 0);
            if (n > 0) CU(cudaStreamWaitEvent(h->st, h->ev_int[(n - 1) & 1], 0));
            launch_ac2d_fused(variant, h->d.order, Fe, 2, n, sv, sample, (n + 1) / every, h->st);
            CU(cudaEventRecord(h->ev_edge[n & 1], h->st));
            CU(cudaStreamWaitEvent(h->st2, h->ev_edge[(n + 1) & 1], 0));  // edge(n-1), or the start
            launch_ac2d_fused(variant, h->d.order, Fi, h->nb_int, n, sv, sample, (n + 1) / every, h->st2);
            CU(cudaEventRecord(h->ev_int[n & 1], h->st2));
            h->launches += 2;
            cur ^= 1;
            if ((rc = exchange_nccl_plan(h, HW_PLAN_FUSED, cur))) return rc;
        }
        if (nt > 0) CU(cudaStreamWaitEvent(h->st, h->ev_int[(nt - 1) & 1], 0));
    } else if ((h->fused3 || h->fused3_32) && h->transport == 2 && h->st2) {
        // NCCL slab, overlapped (as the fused 2D kernel): edge slabs 0 and L-1 + the exchange on st,
        // the interior slabs on st2
        const StreamIO IO = stream_io(h, C);
        const int sk = h->d.src_kind;
        CU(cudaEventRecord(h->ev_edge[1], h->st));  // st2 starts after everything queued on st
        int cur = 0;
        for (int64_t n = 0; n < nt; n++) {
            AcParams P = C.A;
            Ac3In in;
            fused3_bufs(h, cur, P, in);
            in.edge = 1;
            in.nb_total = h->ac3_nb_edge + h->ac3_nb_int;
            Ac3In ie = in, ii = in;
            ie.band = 1;
            ie.group = 1;
            ii.band = 2;
            const int sample = energy && ((n + 1) % C.every == 0);
            const double sv = (src && sk == HW_SRC_PRESSURE) ? src[n] : 0.0;
            auto launch = [&](const Ac3In& a, int nb, cudaStream_t st) {
                if (h->fused3_32) launch_ac3d_fused32(variant, P, a, IO, nb, n, sv, sample, (n + 1) / C.every, st);
                else launch_ac3d_fused(variant, P, a, IO, nb, n, sv, sample, (n + 1) / C.every, st);
            };
            if (n > 0) CU(cudaStreamWaitEvent(h->st, h->ev_int[(n - 1) & 1], 0));
            launch(ie, h->ac3_nb_edge, h->st);
            CU(cudaEventRecord(h->ev_edge[n & 1], h->st));
            CU(cudaStreamWaitEvent(h->st2, h->ev_edge[(n + 1) & 1], 0));  // edge(n-1), or the start
            launch(ii, h->ac3_nb_int, h->st2);
            CU(cudaEventRecord(h->ev_int[n & 1], h->st2));
            h->launches += 2;
            cur ^= 1;
            if ((rc = exchange_nccl_plan(h, HW_PLAN_FUSED_AC3, cur))) return rc;
        }
        if (nt > 0) CU(cudaStreamWaitEvent(h->st, h->ev_int[(nt - 1) & 1], 0));
    } else if (h->fused3 || h->fused3_32) {  // one-pass 3D kernel, ping-pong A <-> B: step n reads buffer n % 2
        const StreamIO IO = stream_io(h, C);
        const int sk = h->d.src_kind;
        int cur = 0;
        for (int64_t n = 0; n < nt; n++) {
            AcParams P = C.A;
            Ac3In in;
            fused3_bufs(h, cur, P, in);
            const int sample = energy && ((n + 1) % C.every == 0);
            const double sv = (src && sk == HW_SRC_PRESSURE) ? src[n] : 0.0;
            if (h->fused3_32) launch_ac3d_fused32(variant, P, in, IO, h->stream_blocks, n, sv, sample, (n + 1) / C.every, h->st);
            else launch_ac3d_fused(variant, P, in, IO, h->stream_blocks, n, sv, sample, (n + 1) / C.every, h->st);
            h->launches++;
            cur ^= 1;
            if (h->transport == 2 && (rc = exchange_nccl_plan(h, HW_PLAN_FUSED_AC3, cur))) return rc;
        }
    } else if (h->fused_el3 && h->transport == 2 && h->st2) {
        // NCCL slab, overlapped (as the fused 2D kernel):
        //   st : wait interior(n-1) | edge slabs(n) | record E(n) | exchange(n)
        //   st2: wait edge(n-1)     | interior slabs(n) | [wait E(n) | traces] | record I(n)
        const StreamIO IO = stream_io(h, C);
        CU(cudaEventRecord(h->ev_edge[1], h->st));  // st2 starts after everything queued on st
        int cur = 0;
        for (int64_t n = 0; n < nt; n++) {
            ElParams P = C.L;
            El3In in;
            fused_el3_bufs(h, cur, P, in);
            in.edge = EL3_EDGE;
            in.nb_total = h->el3_nb_edge + h->el3_nb_int;
            El3In ie = in, ii = in;
            ie.band = 1;
            ie.group = 1;
            ii.band = 2;
            const int sample = energy && ((n + 1) % C.every == 0);
            const double sv = src ? src[n] : 0.0;
            if (n > 0) CU(cudaStreamWaitEvent(h->st, h->ev_int[(n - 1) & 1], 0));
            launch_el3d_fused(variant, P, ie, IO, h->el3_nb_edge, n, sv, sample, (n + 1) / C.every, h->st);
            CU(cudaEventRecord(h->ev_edge[n & 1], h->st));
            CU(cudaStreamWaitEvent(h->st2, h->ev_edge[(n + 1) & 1], 0));  // edge(n-1), or the start
            launch_el3d_fused(variant, P, ii, IO, h->el3_nb_int, n, sv, sample, (n + 1) / C.every, h->st2);
            h->launches += 2;
            if (C.E.n_rec > 0) {  // traces after the step (both bands done), on st2: the exchange goes on
                CU(cudaStreamWaitEvent(h->st2, h->ev_edge[n & 1], 0));
                EpParams E = C.E;
                E.trace_base = P.vs.base;
                launch_epilogue(h->LU, E, n, 0, 0, h->st2);
                h->launches++;
            }
            CU(cudaEventRecord(h->ev_int[n & 1], h->st2));
            cur ^= 1;
            if ((rc = exchange_nccl_plan(h, HW_PLAN_FUSED_EL3, cur))) return rc;
        }
        if (nt > 0) CU(cudaStreamWaitEvent(h->st, h->ev_int[(nt - 1) & 1], 0));
    } else if (h->fused_el3) {  // one-pass 3D elastic kernel, ping-pong A <-> B; traces from the epilogue
        const StreamIO IO = stream_io(h, C);
        int cur = 0;
        for (int64_t n = 0; n < nt; n++) {
            ElParams P = C.L;
            El3In in;
            fused_el3_bufs(h, cur, P, in);
            const int sample = energy && ((n + 1) % C.every == 0);
            launch_el3d_fused(variant, P, in, IO, h->stream_blocks, n, src ? src[n] : 0.0, sample, (n + 1) / C.every,
                              h->st);
            h->launches++;
            if (C.E.n_rec > 0) {  // receiver traces of v_slow after the step, from the buffer just written
                EpParams E = C.E;
                E.trace_base = P.vs.base;
                launch_epilogue(h->LU, E, n, 0, 0, h->st);
                h->launches++;
            }
            cur ^= 1;
            if (h->transport == 2 && (rc = exchange_nccl_plan(h, HW_PLAN_FUSED_EL3, cur))) return rc;
        }
    } else if (h->fused_el && h->transport == 2 && h->st2) {
        // NCCL slab, overlapped (as the fused 2D acoustic kernel):
        //   st : wait interior(n-1) | edge bands(n) | record E(n) | exchange(n)
        //   st2: wait edge(n-1)     | interior bands(n) | record I(n)
        const StreamIO IO = stream_io(h, C);
        CU(cudaEventRecord(h->ev_edge[1], h->st));  // st2 starts after everything queued on st
        int cur = 0;
        for (int64_t n = 0; n < nt; n++) {
            ElParams P = C.L;
            El2In in;
            fused_el_bufs(h, cur, P, in);
            in.edge = FUSED_EDGE;
            in.nb_total = 2 + h->nb_int;
            El2In ie = in, ii = in;
            ie.band = 1;
            ii.band = 2;
            const int sample = energy && ((n + 1) % C.every == 0);
            const double sv = src ? src[n] : 0.0;
            if (n > 0) CU(cudaStreamWaitEvent(h->st, h->ev_int[(n - 1) & 1], 0));
            launch_el2d_fused(variant, h->d.order, P, ie, IO, 2, n, sv, sample, (n + 1) / C.every, h->st);
            CU(cudaEventRecord(h->ev_edge[n & 1], h->st));
            CU(cudaStreamWaitEvent(h->st2, h->ev_edge[(n + 1) & 1], 0));  // edge(n-1), or the start
            launch_el2d_fused(variant, h->d.order, P, ii, IO, h->nb_int, n, sv, sample, (n + 1) / C.every, h->st2);
            CU(cudaEventRecord(h->ev_int[n & 1], h->st2));
            h->launches += 2;
            cur ^= 1;
            if ((rc = exchange_nccl_plan(h, HW_PLAN_FUSED_EL2, cur))) return rc;
        }
        if (nt > 0) CU(cudaStreamWaitEvent(h->st, h->ev_int[(nt - 1) & 1], 0));
    } else if (h->fused_el) {  // one-pass 2D elastic kernel, ping-pong A <-> B: step n reads buffer n % 2
        const StreamIO IO = stream_io(h, C);
        int cur = 0;
        for (int64_t n = 0; n < nt; n++) {
            ElParams P = C.L;
            El2In in;
            fused_el_bufs(h, cur, P, in);
            const int sample = energy && ((n + 1) % C.every == 0);
            launch_el2d_fused(variant, h->d.order, P, in, IO, h->stream_blocks, n, src ? src[n] : 0.0, sample,
                              (n + 1) / C.every, h->st);
            h->launches++;
            cur ^= 1;
            if (h->transport == 2 && (rc = exchange_nccl_plan(h, HW_PLAN_FUSED_EL2, cur))) return rc;
        }
    } else if (h->fused) {  // fused kernels, ping-pong A <-> B: launch L reads buffer L % 2
        AcFusedParams F = fused_params(h, nt);
        __half* bufs[2][FUSED_NSTREAM];
        fused_bufs(h, bufs);
        const int64_t every = C.every;
        int cur = 0;
        for (int64_t n = 0; n < nt;) {
            for (int j = 0; j < FUSED_NSTREAM; j++) {
                F.in[j] = bufs[cur][j];
                F.out[j] = bufs[cur ^ 1][j];
            }
            if (h->tb2 && n + 1 < nt) {  // steps n and n+1 in one launch
                launch_ac2d_tb2(variant, h->d.order, F, h->tb2_tiles, h->tb2_bands, h->partials_b, n,
                                src ? src[n] : 0.0, src ? src[n + 1] : 0.0, energy && ((n + 1) % every == 0),
                                energy && ((n + 2) % every == 0), (n + 1) / every, (n + 2) / every, h->st);
                n += 2;
            } else {
                launch_ac2d_fused(variant, h->d.order, F, h->fused_blocks, n, src ? src[n] : 0.0,
                                  energy && ((n + 1) % every == 0), (n + 1) / every, h->st);
                n += 1;
            }
            cur ^= 1;
            h->launches++;
            if (fused_slab && (rc = exchange_nccl_plan(h, HW_PLAN_FUSED, cur))) return rc;
        }
    } else {
        for (int64_t n = 0; n < nt; n++) {
            run_phase(h, C, 0, n, src);
            if ((rc = exchange(h, 0))) return rc;
            run_phase(h, C, 1, n, src);
            if ((rc = exchange(h, 1))) return rc;
            run_epilogue(h, C, n);
        }
    }
    if (timed) CU(cudaEventRecord(h->ev1, h->st));
    CU(cudaGetLastError());
    return HW_OK;
}

// After `executed` fused steps (L launches: one per step, or one per pair of steps
// with the two-step kernel) the newest state sits in buffer B when L is odd: copy it
// home so buffer A is always current between calls.
static int fused_copy_back(hw_solver* h, int64_t executed, int32_t variant) {
    const int64_t launches = h->tb2 ? (executed + 1) / 2 : executed;
    if (!(h->fused || h->fused3 || h->fused3_32 || h->fused_el || h->fused_el3) || h->small || (launches & 1) == 0) return HW_OK;  // the small-grid kernel writes A itself
    const int nf = variant == HW_NAIVE ? h->nsol : 2 * h->nsol;  // naive runs never touch residuals
    for (int j = 0; j < nf; j++) {
        int f = h->ext[j % h->nsol];
        size_t bytes = (size_t)(field_rows(h, f) + 2 * G) * h->g.slab * lane_bytes(h->LU);
        CU(cudaMemcpyAsync(h->mem[j], h->mem_b[j], bytes, cudaMemcpyDeviceToDevice, h->st));
    }
    CU(cudaStreamSynchronize(h->st));
    return HW_OK;
}

static void fill_times(const hw_solver* h, double* e_times, int64_t ne) {
    if (!e_times || ne <= 0) return;
    e_times[0] = 0.0;
    for (int64_t k = 1; k < ne; k++) {
        int64_t n = k * h->d.energy_every - 1;
        e_times[k] = ((double)n + 0.5) * h->d.dt;  // local step index, as acoustic.py:226
    }
}

// A two-step launch whose FIRST step went non-finite has also written step n+1: replay
// step n alone with the single-step kernel from the launch's untouched input buffer,
// so the state, failure record and traces are exactly "after the failing step".
static int tb2_replay(hw_solver* h, int32_t variant, int64_t nt, const double* src, bool energy, Ctrl& c) {
    if (!h->tb2 || c.fail_step == INT64_MAX || (c.fail_step & 1) || c.fail_step + 1 >= nt) return HW_OK;
    const int64_t n = c.fail_step, every = h->d.energy_every;
    const int cur = (int)((n / 2) & 1);
    AcFusedParams F = fused_params(h, nt);
    __half* bufs[2][FUSED_NSTREAM];
    fused_bufs(h, bufs);
    for (int j = 0; j < FUSED_NSTREAM; j++) {
        F.in[j] = bufs[cur][j];
        F.out[j] = bufs[cur ^ 1][j];
    }
    Ctrl c0;
    c0.fail_step = INT64_MAX;
    c0.fail_mask = 0;
    c0.pad = 0;
    c0.gfail_step = INT64_MAX;
    CU(cudaMemcpyAsync(h->ctrl, &c0, sizeof(Ctrl), cudaMemcpyHostToDevice, h->st));
    for (int64_t j = 0; j < h->n_rec_sorted; j++)  // the pair's second step recorded samples at n+1
        CU(cudaMemsetAsync(h->traces + j * nt + n + 1, 0, (nt - n - 1) * sizeof(double), h->st));
    launch_ac2d_fused(variant, h->d.order, F, h->fused_blocks, n, src ? src[n] : 0.0,
                      energy && ((n + 1) % every == 0), (n + 1) / every, h->st);
    h->launches++;
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(&c, h->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, h->st));
    CU(cudaStreamSynchronize(h->st));
    return HW_OK;
}

int hw_run(hw_solver* h, int32_t variant, int64_t step0, int64_t nt, const double* src_samples, double* traces,
           double* e_times, double* e_vals, int64_t* n_energy, int64_t* fail_step, int32_t* fail_field) {
    if (!h) return fail(HW_EINVAL, "null solver");
    bool energy = e_vals != nullptr || e_times != nullptr || n_energy != nullptr;
    int rc = run_impl(h, variant, nt, src_samples, energy, false);
    if (rc) return rc;
    Ctrl c;
    CU(cudaMemcpyAsync(&c, h->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, h->st));
    CU(cudaStreamSynchronize(h->st));
    if ((rc = tb2_replay(h, variant, nt, src_samples, energy, c))) return rc;
    if (h->transport == 2) {  // agree on the first failure across ranks; combine energy and traces
        Ctrl* all = nullptr;
        CU(cudaMalloc(&all, sizeof(Ctrl) * h->world));
        NC(g_nccl.AllGather(h->ctrl, all, sizeof(Ctrl), ncclInt8, h->nccl, h->st));
        std::vector<Ctrl> hc(h->world);
        CU(cudaMemcpyAsync(hc.data(), all, sizeof(Ctrl) * h->world, cudaMemcpyDeviceToHost, h->st));
        CU(cudaStreamSynchronize(h->st));
        cudaFree(all);
        c.fail_step = INT64_MAX;
        c.fail_mask = 0;
        for (const Ctrl& x : hc) c.fail_step = x.fail_step < c.fail_step ? x.fail_step : c.fail_step;
        for (const Ctrl& x : hc) if (x.fail_step == c.fail_step) c.fail_mask |= x.fail_mask;
    }
    int64_t done = nt;
    int status = HW_OK;
    if (c.fail_step != INT64_MAX) {
        done = c.fail_step + 1;
        status = HW_RANGE_FAILURE;
        int bit = 0;
        while (bit < 32 && !((c.fail_mask >> bit) & 1u)) bit++;
        if (fail_step) *fail_step = step0 + c.fail_step;
        if (fail_field) *fail_field = bit;
        g_err = "non-finite value after step " + std::to_string(step0 + c.fail_step);
    }
    if ((rc = fused_copy_back(h, done, variant))) return rc;
    const int64_t nrec = h->d.n_receivers;
    const int64_t ne = energy ? 1 + (status == HW_OK ? nt / h->d.energy_every : (done - 1) / h->d.energy_every) : 0;
    if (h->transport == 2) {
        if (ne > 0 && h->plane_energy()) {  // plane totals of every rank, summed in global plane order
            std::vector<double> mine;
            if ((rc = el3_planes_host(h, ne, mine))) return rc;
            const int64_t lmax = (h->d.ns + h->world - 1) / h->world;
            std::vector<double> pad((size_t)ne * lmax, 0.0), allh((size_t)ne * lmax * h->world);
            for (int64_t q = 0; q < ne * h->max_rows; q++) pad[q] = mine[q];
            double* dev = nullptr;
            CU(cudaMalloc(&dev, sizeof(double) * ne * lmax * (h->world + 1)));
            CU(cudaMemcpy(dev, pad.data(), sizeof(double) * ne * lmax, cudaMemcpyHostToDevice));
            NC(g_nccl.AllGather(dev, dev + ne * lmax, ne * lmax, ncclFloat64, h->nccl, h->st));
            CU(cudaMemcpyAsync(allh.data(), dev + ne * lmax, sizeof(double) * ne * lmax * h->world,
                               cudaMemcpyDeviceToHost, h->st));
            CU(cudaStreamSynchronize(h->st));
            cudaFree(dev);
            std::vector<std::vector<double>> planes(h->world);
            std::vector<int64_t> rows(h->world);
            for (int r = 0; r < h->world; r++) {
                rows[r] = (int64_t)(r + 1) * h->d.ns / h->world - (int64_t)r * h->d.ns / h->world;
                planes[r].resize(ne * rows[r]);
                for (int64_t k = 0; k < ne * rows[r]; k++) planes[r][k] = allh[(size_t)r * ne * lmax + k];
            }
            std::vector<double> tot(ne);
            el3_energy_from_planes(planes, rows, ne, C_scale(h), tot.data());
            CU(cudaMemcpy(h->evals, tot.data(), sizeof(double) * ne, cudaMemcpyHostToDevice));
        } else if (ne > 0) {  // per-rank energy totals gathered, then summed in rank order on every rank
            double* all = nullptr;
            CU(cudaMalloc(&all, sizeof(double) * ne * h->world));
            NC(g_nccl.AllGather(h->evals, all, ne, ncclFloat64, h->nccl, h->st));
            std::vector<double> hv((size_t)ne * h->world), tot(ne, 0.0);
            CU(cudaMemcpyAsync(hv.data(), all, sizeof(double) * ne * h->world, cudaMemcpyDeviceToHost, h->st));
            CU(cudaStreamSynchronize(h->st));
            cudaFree(all);
            for (int64_t k = 0; k < ne; k++) {
                double t = hv[k];
                for (int r = 1; r < h->world; r++) t += hv[(size_t)r * ne + k];
                tot[k] = t;
            }
            CU(cudaMemcpy(h->evals, tot.data(), sizeof(double) * ne, cudaMemcpyHostToDevice));
        }
        for (int64_t j = 0; j < nrec && nt > 0; j++) {  // receiver traces from their owning slab
            int owner = 0;
            for (int r = 0; r < h->world; r++) {
                int64_t r0 = (int64_t)r * h->d.ns / h->world, r1 = (int64_t)(r + 1) * h->d.ns / h->world;
                if (h->d.receivers[3 * j + 2] >= r0 && h->d.receivers[3 * j + 2] < r1) owner = r;
            }
            NC(g_nccl.Broadcast(h->traces + j * nt, h->traces + j * nt, nt, ncclFloat64, owner, h->nccl, h->st));
        }
        CU(cudaStreamSynchronize(h->st));
    }
    if (h->plane_energy() && h->transport == 0 && ne > 0) {  // the same plane-ordered sum on one domain
        std::vector<std::vector<double>> planes(1);
        if ((rc = el3_planes_host(h, ne, planes[0]))) return rc;
        std::vector<double> tot(ne);
        el3_energy_from_planes(planes, {h->max_rows}, ne, C_scale(h), tot.data());
        CU(cudaMemcpy(h->evals, tot.data(), sizeof(double) * ne, cudaMemcpyHostToDevice));
    }
    if (traces && nrec > 0 && nt > 0) CU(cudaMemcpy(traces, h->traces, nrec * nt * sizeof(double), cudaMemcpyDeviceToHost));
    if (e_vals && ne > 0) CU(cudaMemcpy(e_vals, h->evals, ne * sizeof(double), cudaMemcpyDeviceToHost));
    fill_times(h, e_times, ne);
    if (n_energy) *n_energy = ne;
    return status;
}

int hw_run_group(hw_solver* const* hs, int32_t nslabs, int32_t variant, int64_t step0, int64_t nt,
                 const double* src_samples, double* traces, double* e_times, double* e_vals, int64_t* n_energy,
                 int64_t* fail_step, int32_t* fail_field) {
    if (!hs || nslabs < 1 || !hs[0]->group || (int)hs[0]->group->ranks.size() != nslabs)
        return fail(HW_EINVAL, "hw_run_group needs the handles of one slab group");
    hw_group* grp = hs[0]->group;
    bool energy = e_vals != nullptr || e_times != nullptr || n_energy != nullptr;
    std::vector<RunCtx> C(nslabs);
    int rc;
    // slab 0 resets the shared control block; every other slab orders its work
    // (naive-residual flags, E(0), first step) after that reset
    if ((rc = run_begin(grp->ranks[0], variant, nt, energy, true, C[0]))) return rc;
    CU(cudaEventRecord(grp->ranks[0]->ev_phase, grp->ranks[0]->st));
    for (int r = 1; r < nslabs; r++) {
        CU(cudaSetDevice(grp->ranks[r]->d.device));
        CU(cudaStreamWaitEvent(grp->ranks[r]->st, grp->ranks[0]->ev_phase, 0));
        if ((rc = run_begin(grp->ranks[r], variant, nt, energy, false, C[r]))) return rc;
    }
    if (grp->ranks[0]->fused) {  // fused 2D slabs: one kernel per step per slab, one exchange per step
        std::vector<AcFusedParams> F(nslabs);
        std::vector<std::array<std::array<__half*, FUSED_NSTREAM>, 2>> bufs(nslabs);
        for (hw_solver* h : grp->ranks) {
            F[h->rank] = fused_params(h, nt);
            __half* b[2][FUSED_NSTREAM];
            fused_bufs(h, b);
            for (int k = 0; k < 2; k++)
                for (int j = 0; j < FUSED_NSTREAM; j++) bufs[h->rank][k][j] = b[k][j];
        }
        if ((rc = exchange_group_plan(grp, HW_PLAN_FUSED, 0))) return rc;  // halos of the uploaded state
        int cur = 0;
        for (int64_t n = 0; n < nt; n++) {
            for (hw_solver* h : grp->ranks) {
                cudaSetDevice(h->d.device);
                AcFusedParams& P = F[h->rank];
                for (int j = 0; j < FUSED_NSTREAM; j++) {
                    P.in[j] = bufs[h->rank][cur][j];
                    P.out[j] = bufs[h->rank][cur ^ 1][j];
                }
                const int64_t every = h->d.energy_every;
                launch_ac2d_fused(variant, h->d.order, P, h->fused_blocks, n, src_samples ? src_samples[n] : 0.0,
                                  energy && ((n + 1) % every == 0), (n + 1) / every, h->st);
                h->launches++;
            }
            cur ^= 1;
            if ((rc = exchange_group_plan(grp, HW_PLAN_FUSED, cur))) return rc;
        }
    } else if (grp->ranks[0]->fused_el) {  // one-pass 2D elastic slabs: one exchange per step
        if ((rc = exchange_group_plan(grp, HW_PLAN_FUSED_EL2, 0))) return rc;  // halos of the uploaded state
        int cur = 0;
        for (int64_t n = 0; n < nt; n++) {
            for (hw_solver* h : grp->ranks) {
                cudaSetDevice(h->d.device);
                RunCtx& Cr = C[h->rank];
                ElParams P = Cr.L;
                El2In in;
                fused_el_bufs(h, cur, P, in);
                const int sample = energy && ((n + 1) % Cr.every == 0);
                launch_el2d_fused(variant, h->d.order, P, in, stream_io(h, Cr), h->stream_blocks, n,
                                  src_samples ? src_samples[n] : 0.0, sample, (n + 1) / Cr.every, h->st);
                h->launches++;
            }
            cur ^= 1;
            if ((rc = exchange_group_plan(grp, HW_PLAN_FUSED_EL2, cur))) return rc;
        }
    } else if (grp->ranks[0]->fused3 || grp->ranks[0]->fused3_32) {  // one-pass 3D acoustic slabs
        if ((rc = exchange_group_plan(grp, HW_PLAN_FUSED_AC3, 0))) return rc;  // halos of the uploaded state
        int cur = 0;
        for (int64_t n = 0; n < nt; n++) {
            for (hw_solver* h : grp->ranks) {
                cudaSetDevice(h->d.device);
                RunCtx& Cr = C[h->rank];
                AcParams P = Cr.A;
                Ac3In in;
                fused3_bufs(h, cur, P, in);
                const int sample = energy && ((n + 1) % Cr.every == 0);
                const double sv = (src_samples && h->d.src_kind == HW_SRC_PRESSURE) ? src_samples[n] : 0.0;
                if (h->fused3_32)
                    launch_ac3d_fused32(variant, P, in, stream_io(h, Cr), h->stream_blocks, n, sv, sample, (n + 1) / Cr.every, h->st);
                else
                    launch_ac3d_fused(variant, P, in, stream_io(h, Cr), h->stream_blocks, n, sv, sample, (n + 1) / Cr.every, h->st);
                h->launches++;
            }
            cur ^= 1;
            if ((rc = exchange_group_plan(grp, HW_PLAN_FUSED_AC3, cur))) return rc;
        }
    } else if (grp->ranks[0]->fused_el3) {  // one-pass 3D elastic slabs: one exchange per step
        if ((rc = exchange_group_plan(grp, HW_PLAN_FUSED_EL3, 0))) return rc;  // halos of the uploaded state
        int cur = 0;
        for (int64_t n = 0; n < nt; n++) {
            for (hw_solver* h : grp->ranks) {
                cudaSetDevice(h->d.device);
                RunCtx& Cr = C[h->rank];
                ElParams P = Cr.L;
                El3In in;
                fused_el3_bufs(h, cur, P, in);
                const int sample = energy && ((n + 1) % Cr.every == 0);
                launch_el3d_fused(variant, P, in, stream_io(h, Cr), h->stream_blocks, n,
                                  src_samples ? src_samples[n] : 0.0, sample, (n + 1) / Cr.every, h->st);
                h->launches++;
                if (Cr.E.n_rec > 0) {
                    EpParams E = Cr.E;
                    E.trace_base = P.vs.base;
                    launch_epilogue(h->LU, E, n, 0, 0, h->st);
                    h->launches++;
                }
            }
            cur ^= 1;
            if ((rc = exchange_group_plan(grp, HW_PLAN_FUSED_EL3, cur))) return rc;
        }
    } else {
    if (nslabs > 1) {
        if ((rc = exchange_group(grp, 0)) || (rc = exchange_group(grp, 1))) return rc;  // halos of the uploaded state
    }
    for (int64_t n = 0; n < nt; n++) {
        for (int phase = 0; phase < 2; phase++) {
            for (hw_solver* h : grp->ranks) {
                cudaSetDevice(h->d.device);
                run_phase(h, C[h->rank], phase, n, src_samples);
            }
            if (nslabs > 1 && (rc = exchange_group(grp, phase))) return rc;
        }
        for (hw_solver* h : grp->ranks) {
            cudaSetDevice(h->d.device);
            run_epilogue(h, C[h->rank], n);
        }
    }
    }
    for (hw_solver* h : grp->ranks) {
        CU(cudaSetDevice(h->d.device));
        CU(cudaGetLastError());
        CU(cudaStreamSynchronize(h->st));
    }
    hw_solver* h0 = grp->ranks[0];
    Ctrl c;
    CU(cudaSetDevice(h0->d.device));
    CU(cudaMemcpy(&c, h0->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost));
    int64_t done = nt;
    int status = HW_OK;
    if (c.fail_step != INT64_MAX) {
        done = c.fail_step + 1;
        status = HW_RANGE_FAILURE;
        int bit = 0;
        while (bit < 32 && !((c.fail_mask >> bit) & 1u)) bit++;
        if (fail_step) *fail_step = step0 + c.fail_step;
        if (fail_field) *fail_field = bit;
        g_err = "non-finite value after step " + std::to_string(step0 + c.fail_step);
    }
    for (hw_solver* h : grp->ranks) {  // fused slabs: newest state home to buffer A
        CU(cudaSetDevice(h->d.device));
        if ((rc = fused_copy_back(h, done, variant))) return rc;
    }
    const int64_t nrec = h0->d.n_receivers;
    const int64_t ne = energy ? 1 + (status == HW_OK ? nt / h0->d.energy_every : (done - 1) / h0->d.energy_every) : 0;
    std::vector<double> tmp;
    if (e_vals && ne > 0 && h0->plane_energy()) {  // plane totals of every slab, in global plane order
        std::vector<std::vector<double>> planes(nslabs);
        std::vector<int64_t> rows(nslabs);
        for (hw_solver* h : grp->ranks) {
            if ((rc = el3_planes_host(h, ne, planes[h->rank]))) return rc;
            rows[h->rank] = h->max_rows;
        }
        el3_energy_from_planes(planes, rows, ne, C_scale(h0), e_vals);
    } else if (e_vals && ne > 0) {  // per-slab energies summed in slab order (fixed)
        std::fill(e_vals, e_vals + ne, 0.0);
        tmp.resize(ne);
        for (hw_solver* h : grp->ranks) {
            CU(cudaSetDevice(h->d.device));
            CU(cudaMemcpy(tmp.data(), h->evals, ne * sizeof(double), cudaMemcpyDeviceToHost));
            for (int64_t k = 0; k < ne; k++) e_vals[k] += tmp[k];
        }
    }
    if (traces && nrec > 0 && nt > 0) {
        for (hw_solver* h : grp->ranks) {
            CU(cudaSetDevice(h->d.device));
            for (int64_t j = 0; j < nrec; j++)
                if (h->rec_owned[j])
                    CU(cudaMemcpy(traces + j * nt, h->traces + j * nt, nt * sizeof(double), cudaMemcpyDeviceToHost));
        }
    }
    fill_times(h0, e_times, ne);
    if (n_energy) *n_energy = ne;
    return status;
}

int hw_run_device(hw_solver* h, int32_t variant, int64_t step0, int64_t nt, const double* src_samples, float* ms) {
    (void)step0;
    if (!h) return fail(HW_EINVAL, "null solver");
    int rc = run_impl(h, variant, nt, src_samples, true, true);
    if (rc) return rc;
    CU(cudaEventSynchronize(h->ev1));
    float t = 0.f;
    CU(cudaEventElapsedTime(&t, h->ev0, h->ev1));
    Ctrl c;
    CU(cudaMemcpy(&c, h->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost));
    if ((rc = tb2_replay(h, variant, nt, src_samples, true, c))) return rc;
    if ((rc = fused_copy_back(h, c.fail_step != INT64_MAX ? c.fail_step + 1 : nt, variant))) return rc;
    if (ms) *ms = t;
    h->kernel_ms = nt > 0 ? t / nt : 0.0;
    return HW_OK;
}

int64_t hw_last_launch_count(const hw_solver* h) { return h ? h->launches : 0; }

const char* hw_kernel_path(const hw_solver* h) {
    if (!h) return "";
    return (h->small || h->small_el) ? "small2d" : h->tb2 ? "fused2d-tb2" : h->fused ? "fused2d" : h->fused3 ? "fused3d" : h->fused3_32 ? "fused3d-f32" : h->fused_el ? "fused2d-el" : h->fused_el3 ? "fused3d-el" : (h->el_stream ? "stream2d" : ((h->ac3_stream || h->el3_stream) ? "stream3d" : "generic"));
}

int32_t hw_transport(const hw_solver* h) { return h ? h->transport : -1; }

double hw_last_kernel_ms(const hw_solver* h) { return h ? h->kernel_ms : 0.0; }

const char* hw_last_error(void) { return g_err.c_str(); }

__global__ void k_selftest_guard(const unsigned char* p, int64_t off, unsigned int* sink) {
    *sink = p[off];
}

int hw_selftest_guard(int32_t device, int64_t offset) {
    CU(cudaSetDevice(device));
    unsigned char* buf = nullptr;
    unsigned int* sink = nullptr;
    CU(cudaMalloc(&buf, 4096));
    CU(cudaMalloc(&sink, 4));
    k_selftest_guard<<<1, 1>>>(buf, offset, sink);
    CU(cudaGetLastError());
    CU(cudaDeviceSynchronize());  // an unmapped address ends here (the context is lost after that)
    cudaFree(buf);
    cudaFree(sink);
    return HW_OK;
}

int hw_selftest_div16(int32_t device, uint64_t* mismatches, uint32_t* first_pair) {
    CU(cudaSetDevice(device));
    unsigned long long* bad = nullptr;
    unsigned int* first = nullptr;
    CU(cudaMalloc(&bad, 8));
    CU(cudaMalloc(&first, 4));
    cudaMemset(bad, 0, 8);
    cudaMemset(first, 0xff, 4);
    k_selftest_div16<<<256, 256>>>(bad, first);
    CU(cudaGetLastError());
    unsigned long long nb = 0;
    unsigned int fp = 0;
    CU(cudaMemcpy(&nb, bad, 8, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(&fp, first, 4, cudaMemcpyDeviceToHost));
    cudaFree(bad);
    cudaFree(first);
    if (mismatches) *mismatches = nb;
    if (first_pair) *first_pair = fp;
    return HW_OK;
}

int hw_cheap_div_table(int32_t device, uint32_t* bits1024) {
    CU(cudaSetDevice(device));
    const std::vector<uint32_t>* tab = nullptr;
    int rc = cheap_div_table(device, &tab);
    if (rc) return rc;
    memcpy(bits1024, tab->data(), 1024 * 4);
    return HW_OK;
}

int hw_plane_div_mode(const hw_solver* h, int32_t plane) {
    if (!h || plane < 0 || plane >= HW_NPLANES) return -1;
    return h->lp[plane].div_mode;
}

int hw_exchange_plan(const hw_desc* desc, int32_t world, int32_t rank, int32_t kind, hw_xfer* out, int32_t cap,
                     int32_t* n) {
    if (!desc || !n || world < 1 || rank < 0 || rank >= world || kind < 0 || kind > 5)
        return fail(HW_EINVAL, "hw_exchange_plan: bad arguments");
    PlanGeom g;
    g.ac = desc->equation == HW_EQ_ACOUSTIC;
    g.d3 = desc->ndim == 3;
    g.fs = desc->bc_slow == HW_BC_FREE_SURFACE;
    g.order = desc->order;
    g.world = world;
    g.rank = rank;
    g.ext = ext_order(desc->equation, desc->ndim, &g.nsol);
    g.ns_loc = (int64_t)(rank + 1) * desc->ns / world - (int64_t)rank * desc->ns / world;
    if (kind == HW_PLAN_FUSED && !(g.ac && !g.d3)) return fail(HW_EINVAL, "hw_exchange_plan: fused plan is 2D acoustic");
    if (kind == HW_PLAN_FUSED_EL3 && !(!g.ac && g.d3)) return fail(HW_EINVAL, "hw_exchange_plan: HW_PLAN_FUSED_EL3 is 3D elastic");
    if (kind == HW_PLAN_FUSED_AC3 && !(g.ac && g.d3)) return fail(HW_EINVAL, "hw_exchange_plan: HW_PLAN_FUSED_AC3 is 3D acoustic");
    if (kind == HW_PLAN_FUSED_EL2 && !(!g.ac && !g.d3)) return fail(HW_EINVAL, "hw_exchange_plan: HW_PLAN_FUSED_EL2 is 2D elastic");
    const std::vector<hw_xfer> p = halo_plan(g, kind);
    *n = (int32_t)p.size();
    if (out)
        for (int32_t k = 0; k < *n && k < cap; k++) out[k] = p[k];
    return HW_OK;
}

int hw_set_option(const char* name, int64_t value) {
    if (!name) return fail(HW_EINVAL, "hw_set_option: null name");
    for (Option& o : g_opts)
        if (strcmp(o.name, name) == 0) {
            if (value < o.lo || value > o.hi) return fail(HW_EINVAL, std::string("hw_set_option: value out of range for ") + name);
            o.value = value;
            return HW_OK;
        }
    return fail(HW_EINVAL, std::string("hw_set_option: unknown option ") + name);
}

int hw_get_option(const char* name, int64_t* value) {
    if (!name || !value) return fail(HW_EINVAL, "hw_get_option: null argument");
    for (const Option& o : g_opts)
        if (strcmp(o.name, name) == 0) {
            *value = o.value;
            return HW_OK;
        }
    return fail(HW_EINVAL, std::string("hw_get_option: unknown option ") + name);
}

const char* hw_version(void) { return "halfwave_b200 abi=1 arch=sm_100a"; }

}  // extern "C"
