// Hierarchical delay tracks (synth.py:122-158, trajectory.py:260-298,
// _kernels.py:149-190) for batched fused renders.  Every kernel covers all
// jobs of a batch in one launch; an image finds its job, paths and tier
// constants through the fields of mvb_image.
//
//   k_coarse           coarse distances per (image, coarse sample): the
//                      reference's distance arithmetic on pos[::N]
//   k_bounds_coarse    per-image lower/upper bound of the upsampled max
//   k_bounds_full      exact per-sample max of full-rate images
//   k_select/k_exact_max  exact max over the images that can hold it
//   k_coeffs           fast-path interval records: the 65-tap Kaiser
//                      upsampler refit per coarse interval as a degree-8
//                      polynomial in u, anchored in fp64, pre-split (B, f)
//   k_sort_keys        per-(job, time segment) delay-sort keys (L1 locality)
#include <cfloat>

#include "mvb_common.cuh"

namespace mvb {

__device__ __forceinline__ double image_distance(const mvb_image& im, const double* p,
                                                 const double* m) {
    return exact_distance(im.off[0], im.off[1], im.off[2], (double)im.sign[0],
                          (double)im.sign[1], (double)im.sign[2], p, m);
}

// receiver position row for full-rate sample t of job J
__device__ __forceinline__ const double* mic_row(const mvb_job& J, const double* paths, int64_t t) {
    return paths + 3 * (J.mic_off + (J.mic_moving ? t : 0));
}

// atomic max for non-negative doubles (their bit patterns order like int64)
__device__ __forceinline__ void atomic_max_pos(double* addr, double v) {
    atomicMax(reinterpret_cast<unsigned long long*>(addr),
              (unsigned long long)__double_as_longlong(v));
}

__device__ __forceinline__ double block_max(double v, double* red) {
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    const int nw = (blockDim.x + 31) >> 5;
    v = l < nw ? red[l] : -DBL_MAX;
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// one block per selected image
__global__ void k_coarse(const mvb_image* __restrict__ images, const int32_t* __restrict__ sel,
                         const mvb_job* __restrict__ jobs, const double* __restrict__ paths,
                         double* __restrict__ coarse) {
    const mvb_image im = images[sel[blockIdx.x]];
    const mvb_job& J = jobs[im.job];
    const int64_t K = im.n_coarse;
    const double* src = paths + 3 * im.cpath;
    const double* mic = J.mic_moving ? src + 3 * K : paths + 3 * J.mic_off;
    for (int64_t k = threadIdx.x; k < K; k += blockDim.x)
        coarse[im.coarse + k] = image_distance(im, src + 3 * k, mic + (J.mic_moving ? 3 * k : 0));
}

// Decimated images: lb = largest coarse sample (attained to ~1e-12 m: the
// phase-0 row of the table is a unit impulse up to sinc(integer) rounding);
// ub = max over 64-sample segments s of M + negsum (M - m), M/m the max/min
// over segments s-1..s+1 (a superset of every 65-tap window centred in s).
// With weights summing to 1 whose negative mass is <= negsum, any window
// value is <= wmax + negsum (wmax - wmin).
__global__ void k_bounds_coarse(const mvb_image* __restrict__ images,
                                const double* __restrict__ coarse, double negsum,
                                double* __restrict__ lb, double* __restrict__ ub) {
    __shared__ double red[32];
    const int64_t i = blockIdx.x;
    const mvb_image im = images[i];
    if (im.factor == 1) return;
    const double* c = coarse + im.coarse;
    const int64_t K = im.n_coarse;
    const int64_t nseg = (K + 63) / 64;
    double best_lb = 0.0, best_ub = 0.0;
    for (int64_t s = threadIdx.x; s < nseg; s += blockDim.x) {
        double M = -DBL_MAX, mn = DBL_MAX, own = -DBL_MAX;
        for (int64_t q = s - 1; q <= s + 1; ++q) {
            int64_t a = q * 64, b = a + 64;
            if (a < 0) a = 0;
            if (b > K) b = K;
            for (int64_t t = a; t < b; ++t) {
                const double v = c[t];
                M = fmax(M, v);
                mn = fmin(mn, v);
                if (q == s) own = fmax(own, v);
            }
        }
        best_lb = fmax(best_lb, own);
        best_ub = fmax(best_ub, M + negsum * (M - mn) + 1e-9);
    }
    best_lb = block_max(best_lb, red);
    best_ub = block_max(best_ub, red);
    if (threadIdx.x == 0) {
        lb[i] = best_lb;
        ub[i] = best_ub;
    }
}

// Full-rate images: exact per-sample max, merged atomically (lb/ub zeroed).
__global__ void k_bounds_full(const mvb_image* __restrict__ images, const int32_t* __restrict__ sel,
                              const mvb_job* __restrict__ jobs, const double* __restrict__ paths,
                              double* __restrict__ lb, double* __restrict__ ub) {
    __shared__ double red[32];
    const int32_t i = sel[blockIdx.y];
    const mvb_image im = images[i];
    const mvb_job& J = jobs[im.job];
    double best = 0.0;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < J.T;
         t += (int64_t)gridDim.x * blockDim.x)
        best = fmax(best, image_distance(im, paths + 3 * (J.pos_off + t), mic_row(J, paths, t)));
    best = block_max(best, red);
    if (threadIdx.x == 0) {
        atomic_max_pos(lb + i, best);
        atomic_max_pos(ub + i, best);
    }
}

// One block per job.  scratch region of job j starts at img_off + j:
// [count, candidate image indices...].  dmax[j] <- exact max of the job's
// full-rate images; k_exact_max raises it with the candidates.
__global__ void k_select(const mvb_image* __restrict__ images, const mvb_job* __restrict__ jobs,
                         const double* __restrict__ lb, const double* __restrict__ ub,
                         int32_t* __restrict__ scratch, double* __restrict__ dmax) {
    __shared__ double red[32];
    const int64_t j = blockIdx.x;
    const mvb_job J = jobs[j];
    double m = 0.0, mf = 0.0;
    for (int64_t q = threadIdx.x; q < J.n_img; q += blockDim.x) {
        const int64_t i = J.img_off + q;
        m = fmax(m, lb[i]);
        if (images[i].factor == 1) mf = fmax(mf, lb[i]);
    }
    m = block_max(m, red);
    mf = block_max(mf, red);
    int32_t* sc = scratch + J.img_off + j;
    if (threadIdx.x == 0) {
        sc[0] = 0;
        dmax[j] = mf;
    }
    __syncthreads();
    const double LB = m - 1e-9;
    for (int64_t q = threadIdx.x; q < J.n_img; q += blockDim.x) {
        const int64_t i = J.img_off + q;
        if (images[i].factor != 1 && ub[i] >= LB) {
            const int slot = atomicAdd(sc, 1);
            sc[1 + slot] = (int32_t)i;
        }
    }
}

__global__ void k_exact_max(const mvb_image* __restrict__ images, const mvb_job* __restrict__ jobs,
                            const double* __restrict__ coarse, const double* __restrict__ tables,
                            const int32_t* __restrict__ scratch, double* __restrict__ dmax) {
    __shared__ double red[32];
    const int64_t j = blockIdx.z;
    const mvb_job& J = jobs[j];
    const int32_t* sc = scratch + J.img_off + j;
    const int count = sc[0];
    for (int slot = blockIdx.y; slot < count; slot += gridDim.y) {
        const mvb_image im = images[sc[1 + slot]];
        double best = 0.0;
        for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < J.T;
             t += (int64_t)gridDim.x * blockDim.x)
            best = fmax(best, exact_upsample(coarse + im.coarse, im.n_coarse, tables + im.table,
                                             im.factor, t));
        best = block_max(best, red);
        if (threadIdx.x == 0) atomic_max_pos(dmax + j, best);
    }
}

// Fast-path interval records.  One block per image; chunks of 512
// consecutive intervals stage their coarse window (512 + 64 samples) in
// shared memory (skewed by one word per 16 so the 4-interval stride is
// conflict-free); each thread forms 4 consecutive intervals' 9 coefficients.
// The factor's (9, 65) refit matrix is a by-value kernel parameter, i.e. it
// sits in the constant bank and every DFMA reads it as a free operand: per
// tap, one shared load feeds 36 fp64 FMAs (585 FMAs per interval).
constexpr int COEF_BLOCK = 128;
constexpr int COEF_KI = 4;
constexpr int COEF_SPAN = COEF_BLOCK * COEF_KI;

struct FitParam {
    double v[9 * 65];
};

__device__ __forceinline__ int skew16(int e) { return e + (e >> 4); }

__global__ void __launch_bounds__(COEF_BLOCK) k_coeffs(
    const __grid_constant__ FitParam fit, const mvb_image* __restrict__ images,
    const int32_t* __restrict__ sel, const mvb_job* __restrict__ jobs,
    const double* __restrict__ coarse, mvb_coef32* __restrict__ out) {
    __shared__ double win[COEF_SPAN + 64 + (COEF_SPAN + 64) / 16 + 1];
    const mvb_image im = images[sel[blockIdx.x]];
    const mvb_job& J = jobs[im.job];
    const double kappa = J.kappa;
    const double shift = (double)(J.L - J.d0);
    const int64_t K = im.n_coarse;
    const double* c = coarse + im.coarse;
    const int e0 = COEF_KI * threadIdx.x;
    // blockIdx.y-th span of 512 intervals (grid.y = max spans over images)
    for (int64_t k0 = (int64_t)blockIdx.y * COEF_SPAN; k0 < K; k0 += (int64_t)gridDim.y * COEF_SPAN) {
        __syncthreads();
        for (int t = threadIdx.x; t < COEF_SPAN + 64; t += blockDim.x) {
            int64_t q = k0 - 32 + t;
            q = q < 0 ? 0 : (q >= K ? K - 1 : q);
            win[skew16(t)] = c[q];
        }
        __syncthreads();
        if (k0 + e0 >= K) continue;
        double g[COEF_KI][9];
#pragma unroll
        for (int q = 0; q < COEF_KI; ++q)
#pragma unroll
            for (int p = 0; p < 9; ++p) g[q][p] = 0.0;
        double w[COEF_KI];
#pragma unroll
        for (int q = 0; q < COEF_KI - 1; ++q) w[q + 1] = win[skew16(e0 + q)];
#pragma unroll
        for (int col = 0; col < 65; ++col) {
#pragma unroll
            for (int q = 0; q < COEF_KI - 1; ++q) w[q] = w[q + 1];
            w[COEF_KI - 1] = win[skew16(e0 + col + COEF_KI - 1)];
#pragma unroll
            for (int p = 0; p < 9; ++p)
#pragma unroll
                for (int q = 0; q < COEF_KI; ++q) g[q][p] = fma(fit.v[p * 65 + col], w[q], g[q][p]);
        }
#pragma unroll
        for (int q = 0; q < COEF_KI; ++q) {
            const int64_t k = k0 + e0 + q;
            if (k >= K) break;
            mvb_coef32 r;
            const double base = fma(kappa, g[q][0], shift);
            const double B = floor(base);
            r.B = (int32_t)B;
            r.f = (float)(base - B - 0.5);
            r.d_mid = (float)g[q][0];
            r.pad = 0.f;
#pragma unroll
            for (int p = 0; p < 8; ++p) r.g[p] = (float)(kappa * g[q][p + 1]);
            out[im.coef + k] = r;
        }
    }
}

__global__ void k_sort_keys(const mvb_image* __restrict__ images, const mvb_job* __restrict__ jobs,
                            int64_t max_n_img, int64_t max_n_seg, int64_t seg_len,
                            const double* __restrict__ paths, const double* __restrict__ coarse,
                            double* __restrict__ key) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t s = blockIdx.y, j = blockIdx.z;
    const mvb_job& J = jobs[j];
    if (i >= J.n_img || s * seg_len >= J.T) return;
    const mvb_image im = images[J.img_off + i];
    int64_t t = s * seg_len + seg_len / 2;
    if (t > J.T - 1) t = J.T - 1;
    double k;
    if (im.factor == 1) {
        k = image_distance(im, paths + 3 * (J.pos_off + t), mic_row(J, paths, t));
    } else {
        int64_t c = t / im.factor;
        if (c >= im.n_coarse) c = im.n_coarse - 1;
        k = coarse[im.coarse + c];
    }
    key[(j * max_n_seg + s) * max_n_img + i] = k;
}

}  // namespace mvb

using namespace mvb;

extern "C" {

int mvb_coarse_distances(const mvb_image* images, const int32_t* sel, int64_t n_sel,
                         const mvb_job* jobs, const double* paths, double* coarse, void* stream) {
    if (n_sel < 0 || n_sel > 0x7fffffff) return fail(MVB_EINVAL, "coarse_distances: n_sel");
    if (n_sel == 0) return MVB_OK;
    if (!images || !sel || !jobs || !paths || !coarse) return fail(MVB_EINVAL, "coarse_distances: null");
    k_coarse<<<(unsigned)n_sel, 256, 0, as_stream(stream)>>>(images, sel, jobs, paths, coarse);
    return check_launch("coarse_distances");
}

int mvb_track_bounds(const mvb_image* images, int64_t n_img, const int32_t* full_sel,
                     int64_t n_full, const mvb_job* jobs, const double* paths,
                     const double* coarse, double negsum, double* lb, double* ub, void* stream) {
    if (n_img < 0 || n_img > 0x7fffffff || n_full < 0 || n_full > 65535)
        return fail(MVB_EINVAL, "track_bounds: sizes");
    if (n_img == 0) return MVB_OK;
    if (!images || !jobs || !lb || !ub) return fail(MVB_EINVAL, "track_bounds: null");
    cudaStream_t s = as_stream(stream);
    if (cudaMemsetAsync(lb, 0, sizeof(double) * n_img, s) != cudaSuccess ||
        cudaMemsetAsync(ub, 0, sizeof(double) * n_img, s) != cudaSuccess)
        return fail(MVB_ECUDA, "track_bounds: memset");
    if (coarse) k_bounds_coarse<<<(unsigned)n_img, 128, 0, s>>>(images, coarse, negsum, lb, ub);
    if (n_full > 0) {
        if (!full_sel || !paths) return fail(MVB_EINVAL, "track_bounds: null full-rate inputs");
        k_bounds_full<<<dim3(16, (unsigned)n_full), 256, 0, s>>>(images, full_sel, jobs, paths, lb, ub);
    }
    return check_launch("track_bounds");
}

int mvb_track_max(const mvb_image* images, const mvb_job* jobs, int64_t n_jobs,
                  const double* coarse, const double* tables, const double* lb, const double* ub,
                  int32_t* scratch, double* dmax, void* stream) {
    if (n_jobs < 1 || n_jobs > 65535) return fail(MVB_EINVAL, "track_max: n_jobs");
    if (!images || !jobs || !lb || !ub || !scratch || !dmax) return fail(MVB_EINVAL, "track_max: null");
    cudaStream_t s = as_stream(stream);
    k_select<<<(unsigned)n_jobs, 256, 0, s>>>(images, jobs, lb, ub, scratch, dmax);
    if (coarse && tables)
        k_exact_max<<<dim3(64, 8, (unsigned)n_jobs), 256, 0, s>>>(images, jobs, coarse, tables,
                                                                   scratch, dmax);
    return check_launch("track_max");
}

int mvb_track_coeffs(const mvb_image* images, const int32_t* sel, int64_t n_sel,
                     int64_t max_K, const mvb_job* jobs, const double* coarse,
                     const double* h_fit, mvb_coef32* coef, void* stream) {
    if (n_sel < 0 || n_sel > 0x7fffffff) return fail(MVB_EINVAL, "track_coeffs: n_sel");
    if (n_sel == 0) return MVB_OK;
    if (!images || !sel || !jobs || !coarse || !h_fit || !coef)
        return fail(MVB_EINVAL, "track_coeffs: null");
    if (max_K < 1) return fail(MVB_EINVAL, "track_coeffs: max_K");
    FitParam fp;
    for (int i = 0; i < 9 * 65; ++i) fp.v[i] = h_fit[i];
    int64_t spans = (max_K + COEF_SPAN - 1) / COEF_SPAN;
    if (spans > 65535) spans = 65535;
    k_coeffs<<<dim3((unsigned)n_sel, (unsigned)spans), COEF_BLOCK, 0, as_stream(stream)>>>(
        fp, images, sel, jobs, coarse, coef);
    return check_launch("track_coeffs");
}

int mvb_sort_keys(const mvb_image* images, const mvb_job* jobs, int64_t n_jobs, int64_t max_n_img,
                  int64_t max_n_seg, int64_t seg_len, const double* paths, const double* coarse,
                  double* key, void* stream) {
    if (n_jobs < 0 || n_jobs > 65535 || max_n_img < 0 || max_n_seg < 0 || max_n_seg > 65535 ||
        seg_len < 1)
        return fail(MVB_EINVAL, "sort_keys: sizes");
    if (n_jobs == 0 || max_n_img == 0 || max_n_seg == 0) return MVB_OK;
    if (!images || !jobs || !paths || !key) return fail(MVB_EINVAL, "sort_keys: null");
    dim3 g(grid_for(max_n_img, 256), (unsigned)max_n_seg, (unsigned)n_jobs);
    k_sort_keys<<<g, 256, 0, as_stream(stream)>>>(images, jobs, max_n_img, max_n_seg, seg_len, paths,
                                                  coarse, key);
    return check_launch("sort_keys");
}

}  // extern "C"
