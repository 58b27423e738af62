// hw_fused2d.h — host-side interface of the fused 2D acoustic step (hw_fused2d.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "hw_common.cuh"

namespace hw {
constexpr int FUSED_NSTREAM = 6;
constexpr int FUSED_EDGE = 8;  // rows of each edge band when the halo exchange is overlapped
struct AcFusedParams {
    int64_t nx, ns, pitch;
    const __half* in[FUSED_NSTREAM];  // p vx vy rp rvx rvy
    __half* out[FUSED_NSTREAM];
    PlaneView rho_x, rho_s, beta;
    Plane64 e_beta, e_rho_x, e_rho_s;
    LaneConsts k;
    int32_t has_src, n_rec;
    int64_t src_x, src_s;
    const int* rec;               // receivers sorted by (row, x): (row, x, trace index)
    double* traces;
    int64_t nt;
    Ctrl* ctrl;
    double* partials;
    double* e_vals;
    double scale;
    unsigned int* counter;        // per-handle CTA arrival counter (last CTA reduces the energy)
    int32_t slab;                 // slab of a decomposed domain: rows outside [0, ns) are ghost rows
    int32_t band_mode;            // 0: CTAs split [0, ns); 1: the two edge bands [0, edge), [ns-edge, ns);
                                  // 2: the interior [edge, ns-edge) (overlapped halo exchange)
    int32_t edge;                 // rows per edge band (band_mode 1/2)
    int32_t nb_total;             // CTAs of the step over both launches (band_mode 1/2)
};
size_t fused2d_smem_bytes(int64_t nx);
bool fused2d_eligible(int64_t nx, int max_smem);
cudaError_t fused2d_prepare(int64_t nx);
// two steps per launch (hw_tb2d.cu)
size_t tb2_smem_bytes(int64_t nx);
bool tb2_eligible(int64_t nx, int64_t ns, int max_smem);
void tb2_grid(int64_t nx, int64_t ns, int nsm, int* ntiles, int* nbands);
cudaError_t tb2_prepare(int64_t nx);
void launch_ac2d_tb2(int variant, int order, const AcFusedParams& F, int ntiles, int nbands, double* partials_b,
                     int64_t n, double srcA, double srcB, int sampleA, int sampleB, int64_t eidxA, int64_t eidxB,
                     cudaStream_t st);
// persistent small-grid kernel (hw_small2d.cu)
bool small2d_eligible(int64_t nx, int64_t ns, int nsm, int max_smem);
int small2d_blocks(int64_t ns, int nsm);
size_t small2d_xch_bytes(int64_t nx, int nb);
cudaError_t small2d_prepare(int64_t nx, int64_t ns, int nb);
cudaError_t launch_ac2d_small(int variant, int order, const AcFusedParams& F, __half* xch, unsigned int* gbar,
                              const double* src_dev, double* partials2, int every, int energy, int nb, int64_t nt,
                              cudaStream_t st);
void launch_ac2d_fused(int variant, int order, const AcFusedParams& P, int nblocks, int64_t n, double src, int sample,
                       int64_t eidx, cudaStream_t st);
}  // namespace hw
