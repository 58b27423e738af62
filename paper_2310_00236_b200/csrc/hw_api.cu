// hw_api.cu — the C ABI (include/halfwave_b200.h): device state, medium
// materialisation, the step loop and the per-step epilogue kernel.
//
// One hw_solver per rank/GPU.  The whole time loop of AcousticSolver.run /
// ElasticSolver.run (acoustic.py:185-236, elastic.py:242-296) is issued from here
// onto one CUDA stream; the host synchronises once per hw_run.
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/halfwave_b200.h"
#include "hw_params.h"

using namespace hw;

#include "hw_fused2d.h"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

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

// Initial ghost fill (write-through keeps them current afterwards).
template <typename T>
__global__ void k_fill_ghosts(FieldView f, Geom g, int esize) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t per = g.nm * g.nx;
    if (i >= 2 * G * per) return;
    int64_t q = i / per, rem = i % per;
    int64_t m = rem / g.nx, x = rem % g.nx;
    int64_t n = f.rows;
    int64_t k = q < G ? q - G : n + (q - G);  // -2,-1, n, n+1
    int64_t src;
    bool neg = false;
    if (f.gmode == GHOST_PERIODIC) {
        src = k < 0 ? k + n : k - n;
    } else {
        if (f.half_s) src = k < 0 ? -k - 1 : 2 * n - 1 - k;
        else src = k < 0 ? -k : 2 * n - 2 - k;
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
    (void)esize;
}

// Per-step epilogue: receiver traces (acoustic.py:217-218) and the fixed-order
// reduction of the block energy partials into one fp64 sample.
template <int LU>
__global__ void k_epilogue(EpParams E, int64_t n, int sample, int64_t eidx) {
    if (n >= 0 && halted(E.ctrl, n)) return;
    using TU = typename lane<LU>::T;
    if (n >= 0) {
        const TU* b = reinterpret_cast<const TU*>(E.trace_base);
        for (int j = threadIdx.x; j < E.n_rec; j += blockDim.x)
            E.traces[(int64_t)j * E.nt + n] = lane<LU>::to_f64(b[E.rec_off[j]]);
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

// ---------------------------------------------------------------- the handle

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
    double* partials = nullptr;
    int64_t nblocks = 0;
    int64_t max_rows = 0;
    double* traces = nullptr;
    int64_t traces_cap = 0;
    double* evals = nullptr;
    int64_t evals_cap = 0;
    int64_t* rec_off = nullptr;
    int64_t* rec_xyz = nullptr;
    unsigned int res_bad = 0;   // residual fields holding non-finite values at upload
    cudaStream_t st = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    int64_t launches = 0;
    double kernel_ms = 0.0;
    double dt_u = 0.0;
    // fused single-pass path (2D acoustic, binary16): ping-pong partner buffers
    bool fused = false;
    int fused_blocks = 0;
    void* mem_b[2 * F_N] = {};
};

namespace {

int64_t field_rows(const hw_solver* h, int f) { return h->d.ns + ((h->fs && !HALF_S[f]) ? 1 : 0); }

int plane_lane(const hw_solver* h, int pl) {
    switch (pl) {
        case HW_PL_RHO_X: case HW_PL_RHO_S: case HW_PL_RHO_M: case HW_PL_BETA: return h->LU;
        case HW_PL_LAM: case HW_PL_STIFF: case HW_PL_MU_N: case HW_PL_EP: return h->LS;
        default: return 0;  // energy only
    }
}

// rows of the field each plane is shaped like (0 = plane unused)
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

// Upload one fp64 plane, compressed to constant / slow-layered / full, plus its lane copy.
int upload_plane(hw_solver* h, int pl) {
    int64_t rows = plane_rows(h, pl);
    h->lp[pl] = PlaneView{nullptr, nullptr, 0, 0, 0, 0, 0};
    h->ep64[pl] = Plane64{nullptr, 0, 0, 0};
    if (!rows) return HW_OK;
    const double* src = h->d.plane[pl];
    if (!src) return fail(HW_EINVAL, "medium plane " + std::to_string(pl) + " missing");
    int64_t nm = pl == HW_PL_EP ? 1 : h->d.nm, nx = h->d.nx;
    int64_t per = nm * nx, n = rows * per;
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
    double* d64 = nullptr;
    CU(cudaMalloc(&d64, cnt * 8));
    h->plane_mem.push_back(d64);
    CU(cudaMemcpy(d64, packed.data(), cnt * 8, cudaMemcpyHostToDevice));
    h->ep64[pl] = Plane64{d64, ss, sm, sx};
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
                const char* env = getenv("HALFWAVE_DIV");
                if (env && strcmp(env, "ieee") == 0) fast = cheap = false;
                if (env && strcmp(env, "fast") == 0) cheap = false;
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
        h->lp[pl] = PlaneView{dl, rcp, ss, sm, sx, mode, 0};
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
    P.has_src = h->d.src_kind == HW_SRC_PRESSURE;
    P.src_x = h->d.src_x; P.src_m = h->d.src_m; P.src_s = h->d.src_s;
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
    P.src_kind = h->d.src_kind;
    P.src_x = h->d.src_x; P.src_m = h->d.src_m; P.src_s = h->d.src_s;
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
    if (d->world_size != 1) return fail(HW_EINVAL, "world_size > 1 requires the NCCL build");
    if (d->n_receivers < 0 || (d->n_receivers > 0 && !d->receivers)) return fail(HW_EINVAL, "bad receivers");
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

int hw_create(const hw_desc* desc, hw_solver** out) {
    int rc = check_desc(desc);
    if (rc) return rc;
    CU(cudaSetDevice(desc->device));
    hw_solver* h = new hw_solver();
    h->d = *desc;
    h->LS = desc->lane_s;
    h->LU = desc->lane_u;
    h->W = (desc->nx % 2 == 0) ? 2 : 1;
    h->d3 = desc->ndim == 3;
    h->fs = desc->bc_slow == HW_BC_FREE_SURFACE;
    h->ac = desc->equation == HW_EQ_ACOUSTIC;
    h->ext = ext_order(desc->equation, desc->ndim, &h->nsol);
    h->dt_u = round_lane(h->LU, desc->dt);
    int64_t pitch = (desc->nx + 31) / 32 * 32;
    h->g = Geom{desc->nx, desc->nm, pitch, desc->nm * pitch};
    auto cleanup = [&](int code) { hw_destroy(h); return code; };
    if (cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreate(&h->ev0) != cudaSuccess || cudaEventCreate(&h->ev1) != cudaSuccess)
        return cleanup(fail(HW_ECUDA, "stream/event creation failed"));
    int esz = lane_bytes(h->LU);
    int64_t max_rows = 0;
    for (int j = 0; j < 2 * h->nsol; j++) {
        int f = h->ext[j % h->nsol];
        bool resid = j >= h->nsol;
        int64_t rows = field_rows(h, f);
        max_rows = rows > max_rows ? rows : max_rows;
        size_t bytes = (size_t)(rows + 2 * G) * h->g.slab * esz;
        void* p = nullptr;
        if (cudaMalloc(&p, bytes) != cudaSuccess) return cleanup(fail(HW_ECUDA, "out of device memory for fields"));
        cudaMemset(p, 0, bytes);
        h->mem[j] = p;
        FieldView fv;
        fv.base = (char*)p + (size_t)G * h->g.slab * esz;
        fv.rows = rows;
        fv.half_s = HALF_S[f];
        fv.bit = j;
        fv.odd = 0;
        fv.gmode = GHOST_NONE;
        if (!resid) {
            if (!h->fs) {
                fv.gmode = GHOST_PERIODIC;
            } else if (f == F_VX || f == F_VS) {
                fv.gmode = GHOST_IMAGE;  // even parity (dvx_y, dvy: elastic.py:210-213, 233-236)
            } else if (f == F_SXS || f == F_SSS) {
                fv.gmode = GHOST_IMAGE;  // odd parity (dsxy_y, dsyy_y: elastic.py:186-189)
                fv.odd = 1;
            }
        }
        (resid ? h->rv : h->fv)[f] = fv;
    }
    for (int pl = 0; pl < HW_NPLANES; pl++)
        if ((rc = upload_plane(h, pl))) return cleanup(rc);
    {
        const char* path = getenv("HALFWAVE_PATH");
        bool want = !(path && strcmp(path, "generic") == 0);
        int dev_smem = 0, nsm = 0;
        cudaDeviceGetAttribute(&dev_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, desc->device);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, desc->device);
        if (want && h->ac && !h->d3 && h->LS == 16 && h->LU == 16 && desc->world_size == 1 &&
            fused2d_eligible(desc->nx, dev_smem)) {
            for (int j = 0; j < 2 * h->nsol; j++) {
                int f = h->ext[j % h->nsol];
                size_t bytes = (size_t)(field_rows(h, f) + 2 * G) * h->g.slab * esz;
                if (cudaMalloc(&h->mem_b[j], bytes) != cudaSuccess) return cleanup(fail(HW_ECUDA, "out of memory (B)"));
                cudaMemset(h->mem_b[j], 0, bytes);
            }
            if (fused2d_prepare(desc->nx) != cudaSuccess) return cleanup(fail(HW_ECUDA, "fused kernel setup failed"));
            int64_t nbf = desc->ns / 4;
            if (nbf < 1) nbf = 1;
            h->fused_blocks = (int)(nbf < nsm ? nbf : nsm);
            h->fused = true;
        }
    }
    if (cudaMalloc(&h->ctrl, sizeof(Ctrl)) != cudaSuccess) return cleanup(fail(HW_ECUDA, "ctrl alloc"));
    h->max_rows = max_rows;
    h->nblocks = grid_blocks(h->g, h->W, max_rows);
    if (cudaMalloc(&h->partials, h->nblocks * NCOMP * sizeof(double)) != cudaSuccess)
        return cleanup(fail(HW_ECUDA, "partials alloc"));
    if (desc->n_receivers > 0) {
        int f = h->ac ? F_P : F_VS;
        std::vector<int64_t> off(desc->n_receivers);
        for (int j = 0; j < desc->n_receivers; j++) {
            const int64_t* r = desc->receivers + 3 * j;
            if (r[0] < 0 || r[0] >= desc->nx || r[1] < 0 || r[1] >= desc->nm || r[2] < 0 || r[2] >= field_rows(h, f))
                return cleanup(fail(HW_EINVAL, "receiver outside the grid"));
            off[j] = r[2] * h->g.slab + r[1] * h->g.pitch + r[0];
        }
        if (cudaMalloc(&h->rec_off, off.size() * 8) != cudaSuccess) return cleanup(fail(HW_ECUDA, "rec alloc"));
        cudaMemcpy(h->rec_off, off.data(), off.size() * 8, cudaMemcpyHostToDevice);
        if (cudaMalloc(&h->rec_xyz, off.size() * 24) != cudaSuccess) return cleanup(fail(HW_ECUDA, "rec alloc"));
        cudaMemcpy(h->rec_xyz, desc->receivers, off.size() * 24, cudaMemcpyHostToDevice);
    }
    if (cudaDeviceSynchronize() != cudaSuccess) return cleanup(fail(HW_ECUDA, "setup failed"));
    *out = h;
    return HW_OK;
}

int hw_destroy(hw_solver* h) {
    if (!h) return HW_OK;
    cudaSetDevice(h->d.device);
    for (void* p : h->mem) if (p) cudaFree(p);
    for (void* p : h->mem_b) if (p) cudaFree(p);
    for (void* p : h->plane_mem) cudaFree(p);
    if (h->ctrl) cudaFree(h->ctrl);
    if (h->partials) cudaFree(h->partials);
    if (h->traces) cudaFree(h->traces);
    if (h->evals) cudaFree(h->evals);
    if (h->rec_off) cudaFree(h->rec_off);
    if (h->rec_xyz) cudaFree(h->rec_xyz);
    if (h->ev0) cudaEventDestroy(h->ev0);
    if (h->ev1) cudaEventDestroy(h->ev1);
    if (h->st) cudaStreamDestroy(h->st);
    delete h;
    return HW_OK;
}

int hw_set_state(hw_solver* h, const void* const* fields) {
    CU(cudaSetDevice(h->d.device));
    int esz = lane_bytes(h->LU);
    h->res_bad = 0;
    for (int j = 0; j < 2 * h->nsol; j++) {
        int f = h->ext[j % h->nsol];
        const FieldView& fv = j < h->nsol ? h->fv[f] : h->rv[f];
        CU(cudaMemcpy2DAsync(fv.base, h->g.pitch * esz, fields[j], h->d.nx * esz, h->d.nx * esz,
                             fv.rows * h->d.nm, cudaMemcpyHostToDevice, h->st));
        if (j >= h->nsol) {  // naive runs never rewrite residuals: remember non-finite ones
            int64_t n = fv.rows * h->d.nm * h->d.nx;
            bool bad = false;
            for (int64_t i = 0; i < n && !bad; i++) {
                double v;
                if (esz == 2) {
                    uint16_t b = ((const uint16_t*)fields[j])[i];
                    bad = (b & 0x7c00) == 0x7c00;
                    continue;
                } else if (esz == 4) v = ((const float*)fields[j])[i];
                else v = ((const double*)fields[j])[i];
                bad = !std::isfinite(v);
            }
            if (bad) h->res_bad |= 1u << j;
        }
        if (fv.gmode != GHOST_NONE) {
            int64_t nthr = 2 * G * h->d.nm * h->d.nx;
            int64_t nb = (nthr + 255) / 256;
            if (esz == 2) k_fill_ghosts<__half><<<nb, 256, 0, h->st>>>(fv, h->g, esz);
            else if (esz == 4) k_fill_ghosts<float><<<nb, 256, 0, h->st>>>(fv, h->g, esz);
            else k_fill_ghosts<double><<<nb, 256, 0, h->st>>>(fv, h->g, esz);
        }
    }
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(h->st));
    return HW_OK;
}

int hw_get_state(hw_solver* h, void* const* fields) {
    CU(cudaSetDevice(h->d.device));
    int esz = lane_bytes(h->LU);
    for (int j = 0; j < 2 * h->nsol; j++) {
        int f = h->ext[j % h->nsol];
        const FieldView& fv = j < h->nsol ? h->fv[f] : h->rv[f];
        CU(cudaMemcpy2DAsync(fields[j], h->d.nx * esz, fv.base, h->g.pitch * esz, h->d.nx * esz,
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

// The time loop (acoustic.py:210-226 / elastic.py:271-286) on the device.
static int run_impl(hw_solver* h, int32_t variant, int64_t nt, const double* src, bool energy, bool timed) {
    if (variant != HW_NAIVE && variant != HW_OP3 && variant != HW_OP6) return fail(HW_EINVAL, "bad variant");
    if (nt < 0) return fail(HW_EINVAL, "nt must be nonnegative");
    CU(cudaSetDevice(h->d.device));
    int rc;
    int64_t nrec = h->d.n_receivers;
    if ((rc = ensure(&h->traces, &h->traces_cap, nrec * nt > 0 ? nrec * nt : 1))) return rc;
    int64_t ecap = 1 + nt / h->d.energy_every;
    if ((rc = ensure(&h->evals, &h->evals_cap, ecap))) return rc;
    Ctrl c0;
    c0.fail_step = INT64_MAX;
    c0.fail_mask = 0;
    c0.pad = 0;
    if (variant == HW_NAIVE && h->res_bad && nt > 0) {  // untouched non-finite residuals fail step 0
        c0.fail_step = 0;
        c0.fail_mask = h->res_bad;
    }
    CU(cudaMemcpyAsync(h->ctrl, &c0, sizeof(Ctrl), cudaMemcpyHostToDevice, h->st));
    EpParams E;
    memset(&E, 0, sizeof(E));
    E.trace_base = (h->ac ? h->fv[F_P] : h->fv[F_VS]).base;
    E.rec_off = h->rec_off;
    E.n_rec = (int32_t)nrec;
    E.nblocks = (int32_t)h->nblocks;
    E.traces = h->traces;
    E.nt = nt;
    E.e_vals = h->evals;
    E.scale = 0.5 * h->d.dx * h->d.dx * (h->d3 ? h->d.dx : 1.0);
    E.partials = h->partials;
    E.ctrl = h->ctrl;
    AcParams A;
    ElParams L;
    if (h->ac) fill_params(h, A);
    else fill_params(h, L);
    A.variant = L.variant = variant;
    const int LS = h->LS, LU = h->LU, W = h->W;
    const int64_t nb = h->max_rows;  // launchers take the slow extent of the grid
    const int64_t every = h->d.energy_every;
    const int sk = h->d.src_kind;
    int64_t launches = 0;
    if (energy) {  // E(t=0) pairs the state with itself
        if (h->ac) launch_ac_energy(LU, W, A, nb, h->st);
        else launch_el_energy(LU, W, L, nb, h->st);
        launch_epilogue(LU, E, -1, 1, 0, h->st);
        launches += 2;
    }
    if (timed) CU(cudaEventRecord(h->ev0, h->st));
    if (h->fused) {  // one fused kernel per step, ping-pong A <-> B
        AcFusedParams F;
        memset(&F, 0, sizeof(F));
        F.nx = h->d.nx;
        F.ns = h->d.ns;
        F.pitch = h->g.pitch;
        const int64_t ghost = (int64_t)G * h->g.slab * 2;  // bytes before row 0
        __half* bufs[2][FUSED_NSTREAM];
        // external order p vx vy rp rvx rvy == fused stream order
        for (int j = 0; j < FUSED_NSTREAM; j++) {
            bufs[0][j] = (__half*)((char*)h->mem[j] + ghost);
            bufs[1][j] = (__half*)((char*)h->mem_b[j] + ghost);
        }
        F.rho_x = h->lp[HW_PL_RHO_X]; F.rho_s = h->lp[HW_PL_RHO_S]; F.beta = h->lp[HW_PL_BETA];
        F.e_beta = h->ep64[HW_PL_BETA]; F.e_rho_x = h->ep64[HW_PL_RHO_X]; F.e_rho_s = h->ep64[HW_PL_RHO_S];
        F.k = make_consts(h->d.taps, h->dt_u);
        F.has_src = sk == HW_SRC_PRESSURE;
        F.src_x = h->d.src_x;
        F.src_s = h->d.src_s;
        F.n_rec = (int32_t)nrec;
        F.rec = h->rec_xyz;
        F.traces = h->traces;
        F.nt = nt;
        F.ctrl = h->ctrl;
        F.partials = h->partials;
        F.e_vals = h->evals;
        F.scale = E.scale;
        for (int64_t n = 0; n < nt; n++) {
            const int sample = energy && ((n + 1) % every == 0);
            for (int j = 0; j < FUSED_NSTREAM; j++) {
                F.in[j] = bufs[n & 1][j];
                F.out[j] = bufs[(n + 1) & 1][j];
            }
            launch_ac2d_fused(variant, h->d.order, F, h->fused_blocks, n, src ? src[n] : 0.0, sample,
                              (n + 1) / every, h->st);
            launches++;
        }
        if (timed) CU(cudaEventRecord(h->ev1, h->st));
        CU(cudaGetLastError());
        h->launches = launches;
        return HW_OK;
    }
    for (int64_t n = 0; n < nt; n++) {
        const int sample = energy && ((n + 1) % every == 0);
        const double s = src ? src[n] : 0.0;
        if (h->ac) {
            launch_ac_vel(LS, LU, W, A, n, nb, h->st);
            launch_ac_pres(LS, LU, W, A, n, sk == HW_SRC_PRESSURE ? s : 0.0, sample, nb, h->st);
        } else {
            launch_el_vel(LS, LU, W, L, n, sk == HW_SRC_VSLOW ? s : 0.0, nb, h->st);
            launch_el_stress(LS, LU, W, L, n, sk == HW_SRC_EXPLOSIVE ? s : 0.0, sample, nb, h->st);
        }
        launches += 2;
        if (sample || nrec > 0) {
            launch_epilogue(LU, E, n, sample, (n + 1) / every, h->st);
            launches++;
        }
    }
    if (timed) CU(cudaEventRecord(h->ev1, h->st));
    CU(cudaGetLastError());
    h->launches = launches;
    return HW_OK;
}

// After `executed` fused steps the newest state sits in buffer B when the count is
// odd: copy it home so buffer A is always current between calls.
static int fused_copy_back(hw_solver* h, int64_t executed, int32_t variant) {
    if (!h->fused || (executed & 1) == 0) return HW_OK;
    const int nf = variant == HW_NAIVE ? h->nsol : 2 * h->nsol;  // naive runs never touch residuals
    for (int j = 0; j < nf; j++) {
        int f = h->ext[j % h->nsol];
        size_t bytes = (size_t)(field_rows(h, f) + 2 * G) * h->g.slab * lane_bytes(h->LU);
        CU(cudaMemcpyAsync(h->mem[j], h->mem_b[j], bytes, cudaMemcpyDeviceToDevice, h->st));
    }
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
    int64_t nrec = h->d.n_receivers;
    if (traces && nrec > 0 && nt > 0) CU(cudaMemcpy(traces, h->traces, nrec * nt * sizeof(double), cudaMemcpyDeviceToHost));
    // energy samples of completed steps only: E0 + one per sample step before the failure
    int64_t ne = energy ? 1 + (status == HW_OK ? nt / h->d.energy_every : (done - 1) / h->d.energy_every) : 0;
    if (e_vals && ne > 0) CU(cudaMemcpy(e_vals, h->evals, ne * sizeof(double), cudaMemcpyDeviceToHost));
    if (e_times && ne > 0) {
        e_times[0] = 0.0;
        for (int64_t k = 1; k < ne; k++) {
            int64_t n = k * h->d.energy_every - 1;
            e_times[k] = ((double)n + 0.5) * h->d.dt;  // local step index, as acoustic.py:226
        }
    }
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
    if ((rc = fused_copy_back(h, c.fail_step != INT64_MAX ? c.fail_step + 1 : nt, variant))) return rc;
    if (ms) *ms = t;
    h->kernel_ms = nt > 0 ? t / nt : 0.0;
    return HW_OK;
}

int64_t hw_last_launch_count(const hw_solver* h) { return h ? h->launches : 0; }

double hw_last_kernel_ms(const hw_solver* h) { return h ? h->kernel_ms : 0.0; }

const char* hw_last_error(void) { return g_err.c_str(); }

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

const char* hw_version(void) { return "halfwave_b200 abi=1 arch=sm_100a"; }

}  // extern "C"
