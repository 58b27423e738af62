// bw_probe.cu — calibrate achievable HBM bandwidth for the fused kernel's access
// pattern with no arithmetic: each CTA streams `rows` rows of 6 arrays in through a
// TMA ring (or plain LDG) and writes 6 arrays out, 148 CTAs, 4096 fp16 per row.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bw_probe tools/bw_probe.cu
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "../paper_2310_00236_b200/csrc/hw_tma.cuh"

using namespace hw;
constexpr int NX = 4096, NS = 6, FR = 4;

__device__ __forceinline__ size_t rowoff(int q, int y, int per, int il) {
    return il ? ((size_t)y * NS + q) * NX : (size_t)q * per + (size_t)y * NX;
}

__global__ void __launch_bounds__(512, 1) k_tma(const __half* in, __half* out, int ny, int per, int il) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = (uint64_t*)smem;
    unsigned* rel = (unsigned*)(full + FR);
    __half* ring = (__half*)(smem + 256);
    int b = blockIdx.x, nb = gridDim.x;
    int y0 = (int)((long)b * ny / nb), y1 = (int)((long)(b + 1) * ny / nb), NI = y1 - y0;
    int tid = threadIdx.x, lane = tid & 31, nw = blockDim.x / 32;
    auto issue = [&](int i) {
        int s = i % FR;
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&full[s], NS * NX * 2);
        for (int q = 0; q < NS; q++)
            tma_load_1d(ring + (s * NS + q) * NX, in + rowoff(q, y0 + i, per, il), NX * 2, &full[s]);
    };
    if (tid == 0) {
        for (int s = 0; s < FR; s++) { mbar_init(&full[s], 1); rel[s] = 0; }
        fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0) for (int j = 0; j < FR && j < NI; j++) issue(j);
    uint4 acc = make_uint4(0, 0, 0, 0);
    for (int i = 0; i < NI; i++) {
        int s = i % FR;
        mbar_wait(&full[s], (i / FR) & 1);
        for (int q = 0; q < NS; q++) {
            uint4 v = *(const uint4*)(ring + (s * NS + q) * NX + tid * 8);
            acc.x ^= v.x;
            *(uint4*)(out + rowoff(q, y0 + i, per, il) + tid * 8) = v;
        }
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();
            if (atomicAdd(&rel[s], 1u) == (unsigned)(nw - 1)) {
                rel[s] = 0;
                __threadfence_block();
                if (i + FR < NI) issue(i + FR);
            }
        }
    }
    if (acc.x == 0x12345678) out[0] = __float2half(1.f);
}

__global__ void __launch_bounds__(512, 1) k_ldg(const __half* in, __half* out, int ny, int per) {
    int b = blockIdx.x, nb = gridDim.x;
    int y0 = (int)((long)b * ny / nb), y1 = (int)((long)(b + 1) * ny / nb);
    int tid = threadIdx.x;
    for (int y = y0; y < y1; y++)
        for (int q = 0; q < NS; q++) {
            uint4 v = *(const uint4*)(in + (size_t)q * per + (size_t)y * NX + tid * 8);
            *(uint4*)(out + (size_t)q * per + (size_t)y * NX + tid * 8) = v;
        }
}

__global__ void k_copy(const uint4* in, uint4* out, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) out[i] = in[i];
}

int main() {
    const int ny = 4096;
    const size_t per = (size_t)NX * ny;
    __half *in, *out;
    cudaMalloc(&in, NS * per * 2);
    cudaMalloc(&out, NS * per * 2);
    cudaMemset(in, 0, NS * per * 2);
    int smem = 256 + FR * NS * NX * 2;
    cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    double bytes = 2.0 * NS * per * 2;
    for (int mode = 0; mode < 4; mode++) {
        for (int w = 0; w < 3; w++) {
            if (mode == 0 || mode == 3) k_tma<<<148, 512, smem>>>(in, out, ny, (int)per, mode == 3);
            else if (mode == 1) k_ldg<<<148, 512>>>(in, out, ny, (int)per);
            else k_copy<<<148 * 8, 256>>>((const uint4*)in, (uint4*)out, NS * per * 2 / 16);
        }
        cudaEventRecord(a);
        const int reps = 20;
        for (int r = 0; r < reps; r++) {
            if (mode == 0 || mode == 3) k_tma<<<148, 512, smem>>>(in, out, ny, (int)per, mode == 3);
            else if (mode == 1) k_ldg<<<148, 512>>>(in, out, ny, (int)per);
            else k_copy<<<148 * 8, 256>>>((const uint4*)in, (uint4*)out, NS * per * 2 / 16);
        }
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const char* nm[] = {"tma-ring rows", "ldg rows", "grid-stride copy", "tma-ring interleaved"};
        printf("%-18s %8.1f us/iter  %7.0f GB/s  (%s)\n", nm[mode], ms * 1e3 / reps, bytes * reps / (ms * 1e-3) / 1e9,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
