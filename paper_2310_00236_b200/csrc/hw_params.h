// hw_params.h — kernel parameter blocks shared by the launch layer and kernels.
#pragma once
#include <cuda_runtime.h>
#include "hw_common.cuh"

// compile-time dispatch over lanes / vector width
#define HW_DISPATCH_LU(LU, ...)                              \
    switch (LU) {                                            \
        case 16: { constexpr int LU_ = 16; __VA_ARGS__; } break; \
        case 32: { constexpr int LU_ = 32; __VA_ARGS__; } break; \
        default: { constexpr int LU_ = 64; __VA_ARGS__; } break; \
    }
#define HW_DISPATCH_LS(LS, ...)                              \
    switch (LS) {                                            \
        case 16: { constexpr int LS_ = 16; __VA_ARGS__; } break; \
        case 32: { constexpr int LS_ = 32; __VA_ARGS__; } break; \
        default: { constexpr int LS_ = 64; __VA_ARGS__; } break; \
    }
#define HW_DISPATCH_W(W, ...)                                \
    if ((W) == 2) { constexpr int W_ = 2; __VA_ARGS__; }     \
    else { constexpr int W_ = 1; __VA_ARGS__; }

namespace hw {

// Acoustic p-v leapfrog (acoustic.py:162-181), generic 2D / 3D.
struct AcParams {
    Geom g;
    FieldView p, vx, vs, vm, rp, rvx, rvs, rvm;
    PlaneView rho_x, rho_s, rho_m, beta;      // update lane (stepping.py:47-52)
    Plane64 e_beta, e_rho_x, e_rho_s, e_rho_m; // fp64 (diagnostics.py:76-87)
    LaneConsts k;                              // taps (stencil lane) + dt (update lane)
    int32_t order, variant, d3, has_src;
    int64_t src_x, src_m, src_s;
    Ctrl* ctrl;
    double* partials;                          // [nblocks][NCOMP]
};

// Elastic velocity-stress leapfrog (elastic.py:176-238), generic 2D / 3D.
struct ElParams {
    Geom g;
    FieldView vx, vs, vm, sxx, sss, smm, sxs, sxm, sms;
    FieldView rvx, rvs, rvm, rsxx, rsss, rsmm, rsxs, rsxm, rsms;
    PlaneView rho_x, rho_s, rho_m;             // update lane
    PlaneView stiff, lam, mu_n, ep;            // stencil lane; ep rows: 0 top, 1 bottom
    Plane64 e_rho_x, e_rho_s, e_rho_m, e_lam, e_mu, e_mu_n;
    LaneConsts k;
    int32_t order, variant, d3, fs;
    int32_t src_kind;                          // HW_SRC_VSLOW / HW_SRC_EXPLOSIVE / none
    int32_t pad;
    int64_t src_x, src_m, src_s;
    Ctrl* ctrl;
    double* partials;
};

struct EpParams {      // per-step epilogue: receiver traces + energy finalisation
    const void* trace_base; // field base for traces
    const int64_t* rec_off; // element offsets from trace_base
    int32_t n_rec;
    int32_t nblocks;        // partial rows to reduce
    double* traces;         // [n_rec][nt]
    int64_t nt;
    double* e_vals;
    double scale;           // 0.5 dx^2 (2D) or 0.5 dx^3 (3D)
    const double* partials;
    const Ctrl* ctrl;
};

// launchers (one instantiation per lane pair and vector width)
void launch_ac_vel(int LS, int LU, int W, const AcParams& P, int64_t n, int64_t nblocks, cudaStream_t st);
void launch_ac_pres(int LS, int LU, int W, const AcParams& P, int64_t n, double src, int sample, int64_t nblocks,
                    cudaStream_t st);
void launch_ac_energy(int LU, int W, const AcParams& P, int64_t nblocks, cudaStream_t st);
void launch_el_vel(int LS, int LU, int W, const ElParams& P, int64_t n, double src, int64_t nblocks, cudaStream_t st);
void launch_el_stress(int LS, int LU, int W, const ElParams& P, int64_t n, double src, int sample, int64_t nblocks,
                      cudaStream_t st);
void launch_el_energy(int LU, int W, const ElParams& P, int64_t nblocks, cudaStream_t st);
// In-kernel receiver traces and energy finalisation of the streaming kernels.
struct StreamIO {
    const int* rec;         // receivers sorted by (row, x): (local row, x, trace index)
    int32_t n_rec;
    int32_t pad;
    double* traces;         // [n_rec][nt]
    int64_t nt;
    double* e_vals;
    double scale;           // 0.5 dx^2
    unsigned int* counter;  // per-handle CTA arrival counter: the last CTA reduces the partials
};

// streaming 2D elastic phase kernels (hw_elastic2d_stream.cu)
bool el2d_stream_eligible(int64_t nx, int64_t ns, int max_smem);
cudaError_t el2d_stream_prepare(int64_t nx);
void launch_el2d_vel_stream(int variant, int order, const ElParams& P, const StreamIO& IO, int nblocks, int64_t n,
                            double src, cudaStream_t st);
void launch_el2d_stress_stream(int variant, int order, const ElParams& P, const StreamIO& IO, int nblocks, int64_t n,
                               double src, int sample, int64_t eidx, cudaStream_t st);
// streaming 3D acoustic phase kernels (hw_acoustic3d_stream.cu)
bool ac3d_stream_eligible(int64_t nx, int64_t nm, int64_t pitch, int max_smem);
cudaError_t ac3d_stream_prepare(int64_t nx);
void launch_ac3d_vel_stream(int variant, int order, const AcParams& P, int nblocks, int64_t n, cudaStream_t st);
void launch_ac3d_pres_stream(int variant, int order, const AcParams& P, const StreamIO& IO, int nblocks, int64_t n,
                             double src, int sample, int64_t eidx, cudaStream_t st);
// one-pass 3D acoustic step, 2nd order (hw_acoustic3d_fused.cu): state n read from these
// buffers (A), state n+1 written through the AcParams field views (B)
struct Ac3In {
    const __half *p, *vx, *vs, *vm, *rp, *rvx, *rvs, *rvm;
    int32_t slab;  // slab of a decomposed domain: slab -1 is a ghost row (HW_PLAN_FUSED_AC3), not slab ns-1
    int32_t group;  // CTAs per group of adjacent tiles (divides the grid and the tile count)
    // overlapped halo exchange (NCCL slab): band 1 = the edge slabs 0 and ns-1, 2 = the interior, 0 = all;
    // edge = slabs per edge (1); nb_total = CTAs of the step over both launches (last-CTA count)
    int32_t band, edge, nb_total, pad;
    double* eplane;  // [ns][tiles] energy partials of the (tile, slab) units (sample steps)
    double* etot;    // [samples][ns] energy plane totals (sample eidx at etot + eidx * ns)
};
bool ac3d_fused_eligible(int64_t nx, int64_t nm, int64_t ns, int64_t pitch, int order, int max_smem);
cudaError_t ac3d_fused_prepare(int64_t nx);
void launch_ac3d_fused(int variant, const AcParams& P, const Ac3In& in, const StreamIO& IO, int nblocks, int64_t n,
                       double src, int sample, int64_t eidx, cudaStream_t st);
// the same step in binary32 lanes (hw_acoustic3d_fused32.cu; Ac3In pointers hold float data)
bool ac3d_fused32_eligible(int64_t nx, int64_t nm, int64_t ns, int64_t pitch, int order, int max_smem);
cudaError_t ac3d_fused32_prepare(int64_t nx);
void launch_ac3d_fused32(int variant, const AcParams& P, const Ac3In& in, const StreamIO& IO, int nblocks, int64_t n,
                         double src, int sample, int64_t eidx, cudaStream_t st);
// one-pass 2D elastic step (hw_elastic2d_fused.cu): state n read from these buffers (A),
// state n+1 written through the ElParams field views (B)
struct El2In {
    const __half *vx, *vs, *sxx, *sss, *sxs, *rvx, *rvs, *rsxx, *rsss, *rsxs;
    // slab of a decomposed domain (ghost rows from HW_PLAN_FUSED_EL2): rows outside the slab are read
    // from the ghosts, not wrapped; free-surface images only at the global ends this slab owns
    int32_t slab, top, bot;
    int32_t vsrc;   // a v_slow point source on local row vsrc_s (-3 .. rows + 2: halo rows included)
    int64_t vsrc_s;
    // overlapped halo exchange (NCCL slab): band 1 = the two edge bands [0, edge) and [rows - edge, rows)
    // (every row the exchange sends), 2 = the interior (reads no ghost row), 0 = every row;
    // nb_total = CTAs of the step over both launches (energy partial slots, last-CTA count)
    int32_t band, edge, nb_total, pad;
};
bool el2d_fused_eligible(int64_t nx, int64_t ns, int max_smem);
cudaError_t el2d_fused_prepare(int64_t nx);
void launch_el2d_fused(int variant, int order, const ElParams& P, const El2In& in, const StreamIO& IO, int nblocks,
                       int64_t n, double src, int sample, int64_t eidx, cudaStream_t st);
// one-pass 3D elastic step, 2nd order (hw_elastic3d_fused.cu)
struct El3In {
    const __half *vx, *vs, *vm, *sxx, *sss, *smm, *sxs, *sxm, *sms;
    const __half *rvx, *rvs, *rvm, *rsxx, *rsss, *rsmm, *rsxs, *rsxm, *rsms;
    const float* coef;   // [ns][coef_m][8]: rcp(rho_x, rho_s, rho_m), 0, stiff, lam, mu_n, 0
    int64_t coef_m;      // coefficient rows per slab: 1 (planes constant along mid) or nm
    int32_t div_mode[3]; // DivMode of rho_x, rho_s, rho_m
    int32_t group;       // CTAs per group of adjacent mid tiles streamed side by side (divides the grid)
    const double* ecoef; // [ns][8] energy coefficients of slow-layered media (k_el3_ecoef), or null
    double* eplane;      // [ns][tiles] energy partials of the (tile, slab) units (sample steps)
    double* etot;        // [samples][ns] energy plane totals (sample eidx at etot + eidx * ns)
    int32_t slab;        // slab of a decomposed domain (ghost rows from the halo exchange), else 0
    int32_t vsrc;        // a v_slow point source whose row vsrc_s (local, -1 .. ns) this slab computes
    int64_t vsrc_s;
    int32_t band, edge;  // band mode (0 all slabs, 1 edge slabs [0,edge) + [ns-edge,ns), 2 interior)
    int32_t nb_total;    // CTAs of all launches of one step (edge + interior; 0 = this grid)
    int32_t pad2;
};
bool el3d_fused_eligible(const ElParams& P, int64_t nx, int64_t nm, int64_t ns, int64_t pitch, int order,
                         int max_smem);
int64_t el3d_fused_coef_rows(const ElParams& P);
bool el3d_fused_erow(const ElParams& P);
cudaError_t el3d_fused_ecoef(const ElParams& P, double* out, int64_t ns, cudaStream_t st);
cudaError_t el3d_fused_coef(const ElParams& P, float* out, int64_t s0, int64_t ns, int64_t cm, cudaStream_t st);
void launch_plane_totals(const double* partials, int64_t blocks_per_plane, int64_t nplanes, double* out,
                         cudaStream_t st);
cudaError_t el3d_fused_prepare(int64_t nx);
void launch_el3d_fused(int variant, const ElParams& P, const El3In& in, const StreamIO& IO, int nblocks, int64_t n,
                       double src, int sample, int64_t eidx, cudaStream_t st);
// streaming 3D elastic phase kernels (hw_elastic3d_stream.cu)
bool el3d_stream_eligible(int64_t nx, int64_t nm, int64_t pitch, int order, int max_smem);
cudaError_t el3d_stream_prepare(int64_t nx, int order);
void launch_el3d_vel_stream(int variant, int order, const ElParams& P, int nblocks, int64_t n, double src,
                            cudaStream_t st);
void launch_el3d_stress_stream(int variant, int order, const ElParams& P, const StreamIO& IO, int nblocks, int64_t n,
                               double src, int sample, int64_t eidx, cudaStream_t st);
// persistent small-grid 2D elastic kernel (hw_small2d.cu)
bool small_el2d_eligible(int64_t nx, int64_t nh, int nsm, int max_smem);
size_t small_el2d_xch_bytes(int64_t nx, int nb);
cudaError_t small_el2d_prepare(int64_t nx, int64_t nh, int nb);
cudaError_t launch_el2d_small(int variant, int order, const ElParams& P, const StreamIO& IO, __half* xch,
                              unsigned int* gbar, const double* src_dev, double* partials2, int every, int energy,
                              int nb, int64_t nt, cudaStream_t st);
int small2d_blocks(int64_t ns, int nsm);
void launch_epilogue(int LU, const EpParams& E, int64_t n, int sample, int64_t eidx, cudaStream_t st);

}  // namespace hw
