// Shared helpers for libmvb.so (sm_100a).  Error plumbing for the C ABI,
// launch checks, and the exact-arithmetic primitives the reference-faithful
// kernels use (explicit _rn intrinsics are never contracted into FMAs, which
// keeps them bit-identical to numba with fastmath off, _kernels.py:12-13).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <set>
#include <string>

#include "mvb.h"

namespace mvb {

void set_error(const std::string& msg);
const char* get_error();

inline int fail(int code, const std::string& msg) {
    set_error(msg);
    return code;
}

inline int check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(MVB_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
    return MVB_OK;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// MVB_CARVEOUT=<percent> (diagnostic): every libmvb kernel prefers the same
// shared-memory carveout, so kernels of different streams can share an SM
// without the SM draining to reconfigure its L1 / shared split.
// MVB_GEO_CARVEOUT=<percent>: the same for every kernel but the fast
// synthesis (which keeps the driver's choice).  Unset: per-kernel defaults.
inline void prefer_carveout(const void* kernel, bool synthesis = false) {
    static const int pct_all = [] {
        const char* e = getenv("MVB_CARVEOUT");
        return e ? atoi(e) : -1;
    }();
    static const int pct_geo = [] {
        const char* e = getenv("MVB_GEO_CARVEOUT");
        return e ? atoi(e) : -1;
    }();
    const int pct = pct_all >= 0 ? pct_all : (synthesis ? -1 : pct_geo);
    if (pct < 0) return;
    static std::mutex mu;
    static std::set<const void*> seen;
    std::lock_guard<std::mutex> g(mu);
    if (seen.insert(kernel).second)
        cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
}

// Time-shard windows (mvb_job w0/w1/e0/e1; all zero = the whole job).
// Path samples [p0, p1) whose delays the window's output samples read:
// sample n < T reads the track at n, samples n >= T the held value at T - 1.
__host__ __device__ __forceinline__ int64_t win_p0(const mvb_job& J) {
    return J.w0 < J.T - 1 ? (int64_t)J.w0 : (int64_t)J.T - 1;
}
__host__ __device__ __forceinline__ int64_t win_p1(const mvb_job& J) {
    return (J.w1 > 0 && J.w1 < J.T) ? (int64_t)J.w1 : (int64_t)J.T;
}
// Coarse samples [k0, k1) (of K) a factor-N image of the job needs: the
// window's path range and sort-segment centres [e0, e1), widened by the
// 65-tap upsampler's +-32 coarse samples and one more for the records' dw.
constexpr int64_t WIN_HALO = 34;
__host__ __device__ __forceinline__ void win_coarse(const mvb_job& J, int64_t N, int64_t K,
                                                    int64_t& k0, int64_t& k1) {
    if (J.e1 <= 0) { k0 = 0; k1 = K; return; }
    k0 = J.e0 / N - WIN_HALO;
    k1 = (J.e1 - 1) / N + 1 + WIN_HALO;
    k0 = k0 < 0 ? 0 : k0;
    k1 = k1 > K ? K : k1;
}

inline unsigned grid_for(int64_t n, int block) {
    int64_t g = (n + block - 1) / block;
    return (unsigned)(g > 0 ? g : 1);
}

// exact reference arithmetic --------------------------------------------------
__device__ __forceinline__ double xmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double xadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double xsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double xdiv(double a, double b) { return __ddiv_rn(a, b); }

// |off + sign*p - mic| in the order of _kernels.py:58-61:
// dx = (off + sign*p) - mic ; sqrt((dx*dx + dy*dy) + dz*dz)
__device__ __forceinline__ double exact_distance(double ox, double oy, double oz, double sx,
                                                 double sy, double sz, const double* p,
                                                 const double* m) {
    double dx = xsub(xadd(ox, xmul(sx, p[0])), m[0]);
    double dy = xsub(xadd(oy, xmul(sy, p[1])), m[1]);
    double dz = xsub(xadd(oz, xmul(sz, p[2])), m[2]);
    return __dsqrt_rn(xadd(xadd(xmul(dx, dx), xmul(dy, dy)), xmul(dz, dz)));
}

// 65-tap upsampled track value at sample m (_kernels.py:169-180), with the
// phase table stored transposed (col-major: tabT[col * factor + phase]) so
// that consecutive samples read consecutive addresses.
__device__ __forceinline__ double exact_upsample(const double* __restrict__ coarse, int64_t nc,
                                                 const double* __restrict__ tabT,
                                                 int64_t factor, int64_t m) {
    const int64_t half = 32;
    int64_t base = m / factor;
    int64_t phase = m - base * factor;
    double acc = 0.0;
#pragma unroll 5
    for (int col = 0; col < 65; ++col) {
        int64_t j = base + (col - half);
        j = j < 0 ? 0 : (j >= nc ? nc - 1 : j);
        acc = xadd(acc, xmul(__ldg(tabT + (int64_t)col * factor + phase), __ldg(coarse + j)));
    }
    return acc;
}

// Bounds checks of the checked build (-DMVB_CHECKED -> libmvb_checked.so;
// compute-sanitizer is not available on the GPU pool).  Each translation unit
// keeps its own device counters; mvb_check_violations sums them.
enum MvbCheck {
    CHK_GATHER_ROW = 0,   // fast synthesis: record row outside [0, rec_rows)
    CHK_RECORD_INDEX,     // interval record k outside [0, n_coarse)
    CHK_STAGE_SIZE,       // staged records exceed the warp's slot
    CHK_ALIGN,            // cp.async source / destination not 16-byte aligned
    CHK_WORK,             // work item outside its sorted image table / segment
    CHK_BRANCH_ROW,       // branch records: row outside [0, rec_rows)
    CHK_EXACT_INDEX,      // exact engine: coarse / stream index out of range
    CHK_COUNT
};
#ifdef MVB_CHECKED
static __device__ unsigned long long mvb_check_counts[CHK_COUNT];
#define MVB_CHECK(cond, id)                                              \
    do {                                                                 \
        if (!(cond)) atomicAdd(&::mvb::mvb_check_counts[(id)], 1ull);      \
    } while (0)
// host: add this TU's counters into h (CHK_COUNT entries) and reset them
static inline void mvb_check_collect(int64_t* h) {
    unsigned long long c[CHK_COUNT] = {};
    cudaMemcpyFromSymbol(c, mvb_check_counts, sizeof(c));
    for (int i = 0; i < CHK_COUNT; ++i) h[i] += (int64_t)c[i];
    const unsigned long long z[CHK_COUNT] = {};
    cudaMemcpyToSymbol(mvb_check_counts, z, sizeof(z));
}
#else
#define MVB_CHECK(cond, id) \
    do {                    \
    } while (0)
#endif

}  // namespace mvb
