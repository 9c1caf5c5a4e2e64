// Roofline denominators the driver does not measure (MEASURED_PEAKS.json has
// HBM copy and bf16 GEMM only): FP32 FFMA throughput and L1-hit load
// bandwidth, each a saturating microbenchmark timed by the caller with CUDA
// events.
#include "mvb_common.cuh"

namespace mvb {

// 8 independent FFMA chains per thread, 4 chains share operands through
// registers only: pure FMA-pipe throughput.
__global__ void __launch_bounds__(256) k_peak_ffma(int iters, float seed, float* out) {
    float a0 = seed + threadIdx.x, a1 = a0 + 1.f, a2 = a0 + 2.f, a3 = a0 + 3.f;
    float a4 = a0 + 4.f, a5 = a0 + 5.f, a6 = a0 + 6.f, a7 = a0 + 7.f;
    const float m = 0.9999999f, c = 1e-7f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            a0 = fmaf(a0, m, c); a1 = fmaf(a1, m, c); a2 = fmaf(a2, m, c); a3 = fmaf(a3, m, c);
            a4 = fmaf(a4, m, c); a5 = fmaf(a5, m, c); a6 = fmaf(a6, m, c); a7 = fmaf(a7, m, c);
        }
    }
    float s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (s == 12345.678f) out[blockIdx.x] = s;  // keep the chains alive
}

// The same shape in fp64 (DFMA): the exact engine's roofline denominator.
__global__ void __launch_bounds__(256) k_peak_dfma(int iters, double seed, double* out) {
    double a0 = seed + threadIdx.x, a1 = a0 + 1.0, a2 = a0 + 2.0, a3 = a0 + 3.0;
    double a4 = a0 + 4.0, a5 = a0 + 5.0, a6 = a0 + 6.0, a7 = a0 + 7.0;
    const double m = 0.9999999999, c = 1e-12;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
            a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
        }
    }
    double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (s == 12345.678) out[blockIdx.x] = s;
}

// Every warp streams a 16 KB per-CTA window with coalesced 16-byte loads:
// L1 hits after the first pass (same access shape as the synthesis gather).
__global__ void __launch_bounds__(256) k_peak_l1(const float4* __restrict__ buf, int iters,
                                                 float* out) {
    const float4* b = buf + (blockIdx.x & 63) * 1024;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            float4 v = __ldg(b + ((threadIdx.x + 256 * r + 32 * i) & 1023));
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
    }
    if (acc.x + acc.y + acc.z + acc.w == 12345.678f) out[blockIdx.x] = acc.x;
}

}  // namespace mvb

using namespace mvb;

extern "C" {

/* FP32 FMA peak probe: grid blocks x 256 threads x iters x 128 FFMA. */
int mvb_peak_ffma(int blocks, int iters, float* d_sink, void* stream) {
    if (blocks < 1 || iters < 1 || !d_sink) return fail(MVB_EINVAL, "peak_ffma: args");
    k_peak_ffma<<<blocks, 256, 0, as_stream(stream)>>>(iters, 1.0f, d_sink);
    return check_launch("peak_ffma");
}

/* FP64 FMA peak probe: grid blocks x 256 threads x iters x 128 DFMA. */
int mvb_peak_dfma(int blocks, int iters, double* d_sink, void* stream) {
    if (blocks < 1 || iters < 1 || !d_sink) return fail(MVB_EINVAL, "peak_dfma: args");
    k_peak_dfma<<<blocks, 256, 0, as_stream(stream)>>>(iters, 1.0, d_sink);
    return check_launch("peak_dfma");
}

/* L1 load probe: blocks x 256 threads x iters x 4 x 16 B from a 64x16 KB buffer. */
int mvb_peak_l1(int blocks, int iters, const float* d_buf, float* d_sink, void* stream) {
    if (blocks < 1 || iters < 1 || !d_buf || !d_sink) return fail(MVB_EINVAL, "peak_l1: args");
    k_peak_l1<<<blocks, 256, 0, as_stream(stream)>>>(reinterpret_cast<const float4*>(d_buf), iters,
                                                     d_sink);
    return check_launch("peak_l1");
}

}  // extern "C"
