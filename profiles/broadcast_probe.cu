// Probe: cost of warp-uniform record reads on sm_100a.
//  k_lds128: LDS.128 broadcast;  k_shfl: SHFL.IDX broadcast from lane-held floats;
//  k_ldg128: LDG.128 broadcast (same global address for all lanes, L1 hit)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_lds128(int iters, float* out) {
    __shared__ float4 s[64];
    if (threadIdx.x < 64) s[threadIdx.x] = make_float4(threadIdx.x, 1, 2, 3);
    __syncthreads();
    float a = 0.f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            float4 v = s[(i * 16 + r) & 63];
            a += v.x * v.y + v.z * v.w;
        }
    }
    if (a == 1.2345f) out[0] = a;
}
__global__ void k_shfl(int iters, float* out) {
    float x0 = threadIdx.x, x1 = x0 + 1.f;
    float a = 0.f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            float v0 = __shfl_sync(0xffffffffu, x0, (r * 4) & 31);
            float v1 = __shfl_sync(0xffffffffu, x0, (r * 4 + 1) & 31);
            float v2 = __shfl_sync(0xffffffffu, x1, (r * 4 + 2) & 31);
            float v3 = __shfl_sync(0xffffffffu, x1, (r * 4 + 3) & 31);
            a += v0 * v1 + v2 * v3;
        }
        x0 += a * 1e-30f;
    }
    if (a == 1.2345f) out[0] = a;
}
__global__ void k_ldg128(const float4* __restrict__ g, int iters, float* out) {
    float a = 0.f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            float4 v = __ldg(g + ((i * 16 + r) & 63) + (blockIdx.x & 7) * 64);
            a += v.x * v.y + v.z * v.w;
        }
    }
    if (a == 1.2345f) out[0] = a;
}
int main() {
    float* out; float4* g;
    cudaMalloc(&out, 4); cudaMalloc(&g, 16 * 4096); cudaMemset(g, 0, 16 * 4096);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int blocks = 148 * 8, iters = 2000;
    for (int k = 0; k < 3; ++k) {
        for (int which = 0; which < 3; ++which) {
            cudaEventRecord(e0);
            if (which == 0) k_lds128<<<blocks, 256>>>(iters, out);
            if (which == 1) k_shfl<<<blocks, 256>>>(iters, out);
            if (which == 2) k_ldg128<<<blocks, 256>>>(g, iters, out);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            double warp_reads = (double)blocks * 8 * iters * 16;  // one 16-B broadcast per warp per (i, r)
            printf("%s: %.3f ms, %.2f broadcast-16B per clk per SM (1.965 GHz)\n",
                   which == 0 ? "lds128" : which == 1 ? "shfl x4" : "ldg128", ms,
                   warp_reads / (ms * 1e-3) / 148 / 1.965e9);
        }
    }
    return 0;
}
