// Static impulse responses, their convolution and the splice baseline
// (reference reference.py:49-187).
//
//   k_static_kernel   one thread per (block, image, tap): image distance,
//                     tau, amplitude and the 65 Kaiser-windowed-sinc tap
//                     values of reference.py:49-66 / :86-93.
//   k_static_gather   the reference's scatter-add of those kernels into the
//                     tap train (reference.py:94-100) restated as a gather:
//                     one thread per output tap walks the images whose
//                     65-tap support covers it (images pre-sorted by base),
//                     so the sum is deterministic without atomics.
//   k_block_conv      direct fp64 convolution of a (windowed) signal block
//                     with a tap train: static_render (reference.py:103-117,
//                     one block) and the per-block pieces of splice_baseline
//                     (reference.py:137-179).  Register-blocked: a thread owns
//                     R consecutive outputs and slides its signal window in
//                     registers; taps are smem broadcasts.
//   k_splice_sum      the overlap-add of the pieces in block order
//                     (reference.py:180-186).
//
// All fp64.  The reference's own static_render switches to FFT convolution
// above 5e6 products (reference.py:116); direct summation is the exact form
// that FFT approximates, and both agree to roundoff.
#include "mvb_common.cuh"

namespace mvb {
namespace {

constexpr int HW = 32;        // UPSAMPLE_HALFWIDTH (trajectory.py)
constexpr int NK = 2 * HW + 1;
constexpr double KAISER_BETA = 7.857;
constexpr double PI = 3.141592653589793;

// Modified Bessel I0 by its power series sum_k ((z/2)^2)^k / (k!)^2; for the
// window's arguments (z <= 7.857) the terms fall below 1e-17 of the sum
// within ~35 terms.  numpy.i0 (Cephes Chebyshev form) agrees to ~1e-16.
__device__ double bessel_i0(double z) {
    const double q = 0.25 * z * z;
    double term = 1.0, sum = 1.0;
    for (int k = 1; k < 64; ++k) {
        term *= q / ((double)k * (double)k);
        sum += term;
        if (term < 1e-17 * sum) break;
    }
    return sum;
}

// reference.py:49-66: entry i = sinc(arg) * window(arg), arg = (i - hw) - frac
__device__ double sinc_kernel_tap(int i, double frac, double inv_i0b) {
    const double arg = (double)(i - HW) - frac;
    double win = 0.0;
    if (fabs(arg) <= (double)HW) {
        double u = fmin(fmax(arg / (double)HW, -1.0), 1.0);
        win = bessel_i0(KAISER_BETA * sqrt(1.0 - u * u)) * inv_i0b;
    }
    const double y = PI * (arg == 0.0 ? 1.0e-20 : arg);  // numpy.sinc
    return (sin(y) / y) * win;
}

__global__ void k_static_kernel(const double* __restrict__ off, const double* __restrict__ sgn,
                                const double* __restrict__ beta, int64_t S,
                                const double* __restrict__ src, int64_t B,
                                const double* __restrict__ mic, double rate, double c,
                                double d_min, double inv_i0b, int64_t* __restrict__ base,
                                double* __restrict__ tau_out, double* __restrict__ ker) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= B * S * NK) return;
    const int k = (int)(t % NK);
    const int64_t bi = t / NK;  // b * S + i
    const int64_t i = bi % S, b = bi / S;
    const double* p = src + 3 * b;
    // image_position - mic (room.py:146-165), norm
    double dx = (off[3 * i + 0] + sgn[3 * i + 0] * p[0]) - mic[0];
    double dy = (off[3 * i + 1] + sgn[3 * i + 1] * p[1]) - mic[1];
    double dz = (off[3 * i + 2] + sgn[3 * i + 2] * p[2]) - mic[2];
    const double d = sqrt(dx * dx + dy * dy + dz * dz);
    const double tau = rate * d / c;
    const double amp = beta[i] / (4.0 * PI * fmax(d, d_min));
    const double fb = floor(tau);
    if (k == 0) {
        base[bi] = (int64_t)fb;
        tau_out[bi] = tau;
    }
    ker[bi * NK + k] = amp * sinc_kernel_tap(k, tau - fb, inv_i0b);
}

// taps[b, n] = sum over images with base - hw <= n <= base + hw of
// ker[b, img, n - base + hw]; images visited in ascending base (stable in
// canonical order for equal bases).
__global__ void k_static_gather(const int64_t* __restrict__ base_sorted,
                                const int64_t* __restrict__ perm, const double* __restrict__ ker,
                                int64_t S, const int64_t* __restrict__ n_taps, int64_t stride,
                                double* __restrict__ taps) {
    const int64_t b = blockIdx.y;
    const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (n >= stride) return;
    double acc = 0.0;
    if (n < n_taps[b]) {
        const int64_t* row = base_sorted + b * S;
        // first image with base >= n - hw
        int64_t lo = 0, hi = S;
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if (row[mid] < n - HW) lo = mid + 1; else hi = mid;
        }
        for (int64_t j = lo; j < S && row[j] <= n + HW; ++j) {
            const int64_t img = perm[b * S + j];
            acc += ker[(b * S + img) * NK + (n - row[j] + HW)];
        }
    }
    taps[b * stride + n] = acc;
}

// Splice window of block b at sample k (reference.py:150-165); 1 inside the
// block, linear ramps (i + 0.5) / crossfade on the fades.
__device__ __forceinline__ double splice_window(int64_t k, int64_t b, int64_t n, int64_t hop,
                                                int64_t cf, int64_t n_blocks) {
    const int64_t start = b * hop;
    const int64_t stop = min(n, start + hop);
    if (k >= start && k < stop) {
        if (cf > 0 && b > 0 && k < start + cf) return ((double)(k - start) + 0.5) / (double)cf;
        return 1.0;
    }
    if (cf > 0 && b < n_blocks - 1 && k >= stop && k < stop + cf && k < n) {
        const double ramp = ((double)(k - stop) + 0.5) / (double)cf;
        return stop + cf <= n ? 1.0 - ramp : fmax(0.0, 1.0 - ramp);
    }
    return 0.0;
}

__host__ __device__ __forceinline__ void block_support(int64_t b, int64_t n, int64_t hop,
                                                       int64_t cf, int64_t n_blocks,
                                                       int64_t* lo, int64_t* hi) {
    const int64_t start = b * hop;
    const int64_t stop = start + hop < n ? start + hop : n;
    int64_t end = stop;
    if (cf > 0 && b < n_blocks - 1) end = stop + cf < n ? stop + cf : n;
    *lo = start;
    *hi = end;
}

constexpr int CONV_THREADS = 128;
constexpr int CONV_R = 8;                              // outputs per thread
constexpr int CONV_TILE = CONV_THREADS * CONV_R;       // outputs per CTA
constexpr int CONV_KC = 256;                           // taps per smem stage
constexpr int CONV_XS = CONV_TILE + CONV_KC;           // signal window per stage
__host__ __device__ constexpr int xpad(int i) { return i + (i >> 3); }  // stride-8 reads

// piece_b[j] = sum_k xw_b[k] h_b[j - k], xw_b = x * window_b on the block's
// support [lo, hi), j in [0, (hi - lo) + nt_b - 1).  One CTA per
// (1024-output tile, block).
__global__ void __launch_bounds__(CONV_THREADS)
k_block_conv(const double* __restrict__ x, int64_t n, int64_t hop, int64_t cf, int64_t n_blocks,
             int windowed, const double* __restrict__ taps, const int64_t* __restrict__ n_taps,
             int64_t tap_stride, double* __restrict__ pieces, int64_t piece_stride) {
    __shared__ double sh[CONV_KC];
    __shared__ double sx[xpad(CONV_XS) + 8];
    const int64_t b = blockIdx.y;
    int64_t lo, hi;
    block_support(b, n, hop, cf, n_blocks, &lo, &hi);
    const int64_t seg = hi - lo;
    const int64_t nt = n_taps[b];
    const int64_t plen = seg + nt - 1;
    const int64_t j0 = (int64_t)blockIdx.x * CONV_TILE;
    if (seg <= 0 || j0 >= plen) return;
    const double* h = taps + b * tap_stride;
    const int tid = threadIdx.x;
    double acc[CONV_R];
#pragma unroll
    for (int r = 0; r < CONV_R; ++r) acc[r] = 0.0;
    // taps k that can reach this tile: j - k in [0, seg)  ->  k in (j0 - seg, j0 + TILE)
    int64_t k_begin = j0 - seg + 1;
    if (k_begin < 0) k_begin = 0;
    int64_t k_end = j0 + CONV_TILE;
    if (k_end > nt) k_end = nt;
    for (int64_t k0 = k_begin; k0 < k_end; k0 += CONV_KC) {
        __syncthreads();
        for (int i = tid; i < CONV_KC; i += CONV_THREADS) {
            int64_t k = k0 + i;
            sh[i] = k < k_end ? h[k] : 0.0;
        }
        // signal indices m = j - k for j in [j0, j0+TILE), k in [k0, k0+KC):
        // m in (j0 - k0 - KC, j0 - k0 + TILE); sx[i] = xw[m0 + i]
        const int64_t m0 = j0 - k0 - CONV_KC + 1;
        for (int i = tid; i < CONV_XS; i += CONV_THREADS) {
            int64_t m = m0 + i;
            double v = 0.0;
            if (m >= 0 && m < seg) {
                v = x[lo + m];
                if (windowed) v *= splice_window(lo + m, b, n, hop, cf, n_blocks);
            }
            sx[xpad(i)] = v;
        }
        __syncthreads();
        // thread outputs j = j0 + R*tid + r; for local tap kk the signal
        // index is R*tid + r - kk + KC - 1 in sx
        const int jb = CONV_R * tid + CONV_KC - 1;
        double w[CONV_R];
#pragma unroll
        for (int r = 0; r < CONV_R; ++r) w[r] = sx[xpad(jb + r)];
        for (int kk = 0; kk < CONV_KC; kk += CONV_R) {
#pragma unroll
            for (int q = 0; q < CONV_R; ++q) {
                const double hv = sh[kk + q];
                // w holds xw at indices jb + r - (kk + q) for r = 0..R-1, as a
                // ring: slot (r + q) % R  (rotation resolved at compile time)
#pragma unroll
                for (int r = 0; r < CONV_R; ++r) acc[r] = fma(hv, w[(r + CONV_R - q) % CONV_R], acc[r]);
                // next tap needs index jb - (kk + q + 1) at ring slot (R - 1 - q) % R
                const int nxt = jb - (kk + q + 1);
                w[(CONV_R - 1 - q + CONV_R) % CONV_R] = nxt >= 0 ? sx[xpad(nxt)] : 0.0;
            }
        }
    }
    double* out = pieces + b * piece_stride;
#pragma unroll
    for (int r = 0; r < CONV_R; ++r) {
        int64_t j = j0 + CONV_R * tid + r;
        if (j < plen) out[j] = acc[r];
    }
}

// out[i] = sum over blocks b (in order) of piece_b[i - lo_b]
__global__ void k_splice_sum(const double* __restrict__ pieces, int64_t piece_stride, int64_t n,
                             int64_t hop, int64_t cf, int64_t n_blocks,
                             const int64_t* __restrict__ n_taps, int64_t max_span,
                             double* __restrict__ out, int64_t out_len) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= out_len) return;
    int64_t b_lo = (i - max_span) / hop;
    if (b_lo < 0) b_lo = 0;
    int64_t b_hi = i / hop;
    if (b_hi > n_blocks - 1) b_hi = n_blocks - 1;
    double acc = 0.0;
    for (int64_t b = b_lo; b <= b_hi; ++b) {
        int64_t lo, hi;
        block_support(b, n, hop, cf, n_blocks, &lo, &hi);
        const int64_t plen = (hi - lo) + n_taps[b] - 1;
        const int64_t j = i - lo;
        if (hi > lo && j >= 0 && j < plen) acc += pieces[b * piece_stride + j];
    }
    out[i] = acc;
}

}  // namespace
}  // namespace mvb

using namespace mvb;

extern "C" {

int mvb_static_taps(const double* off, const double* sgn, const double* beta, int64_t S,
                    const double* src, int64_t B, const double* mic, double rate, double c,
                    double d_min, int64_t* base, double* tau, double* ker, void* stream) {
    if (S < 0 || B < 0) return fail(MVB_EINVAL, "static_taps: bad sizes");
    if (S == 0 || B == 0) return MVB_OK;
    if (!off || !sgn || !beta || !src || !mic || !base || !tau || !ker)
        return fail(MVB_EINVAL, "static_taps: null");
    if (!(rate > 0) || !(c > 0) || !(d_min > 0)) return fail(MVB_EINVAL, "static_taps: rate/c/d_min");
    // i0(beta) on the host with the same series
    double q = 0.25 * KAISER_BETA * KAISER_BETA, term = 1.0, i0b = 1.0;
    for (int k = 1; k < 64; ++k) {
        term *= q / ((double)k * (double)k);
        i0b += term;
        if (term < 1e-17 * i0b) break;
    }
    const int64_t total = B * S * NK;
    prefer_carveout((const void*)k_static_kernel);
    k_static_kernel<<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(
        off, sgn, beta, S, src, B, mic, rate, c, d_min, 1.0 / i0b, base, tau, ker);
    return check_launch("static_taps");
}

int mvb_static_gather(const int64_t* base_sorted, const int64_t* perm, const double* ker,
                      int64_t S, int64_t B, const int64_t* n_taps, int64_t stride, double* taps,
                      void* stream) {
    if (S < 1 || B < 0 || stride < 1 || B > 65535) return fail(MVB_EINVAL, "static_gather: bad sizes");
    if (B == 0) return MVB_OK;
    if (!base_sorted || !perm || !ker || !n_taps || !taps) return fail(MVB_EINVAL, "static_gather: null");
    dim3 g(grid_for(stride, 256), (unsigned)B);
    prefer_carveout((const void*)k_static_gather);
    k_static_gather<<<g, 256, 0, as_stream(stream)>>>(base_sorted, perm, ker, S, n_taps, stride, taps);
    return check_launch("static_gather");
}

int mvb_block_convolve(const double* x, int64_t n, int64_t hop, int64_t crossfade,
                       int64_t n_blocks, int windowed, const double* taps,
                       const int64_t* n_taps, int64_t tap_stride, int64_t max_piece,
                       double* pieces, int64_t piece_stride, void* stream) {
    if (n < 1 || hop < 1 || crossfade < 0 || crossfade > hop || n_blocks < 1 || n_blocks > 65535 ||
        tap_stride < 1 || max_piece < 1 || piece_stride < max_piece)
        return fail(MVB_EINVAL, "block_convolve: bad sizes");
    if (!x || !taps || !n_taps || !pieces) return fail(MVB_EINVAL, "block_convolve: null");
    dim3 g(grid_for(max_piece, CONV_TILE), (unsigned)n_blocks);
    prefer_carveout((const void*)k_block_conv);
    k_block_conv<<<g, CONV_THREADS, 0, as_stream(stream)>>>(x, n, hop, crossfade, n_blocks,
                                                          windowed, taps, n_taps, tap_stride,
                                                          pieces, piece_stride);
    return check_launch("block_convolve");
}

int mvb_splice_sum(const double* pieces, int64_t piece_stride, int64_t n, int64_t hop,
                   int64_t crossfade, int64_t n_blocks, const int64_t* n_taps, int64_t max_span,
                   double* out, int64_t out_len, void* stream) {
    if (n < 1 || hop < 1 || crossfade < 0 || n_blocks < 1 || out_len < 0 || max_span < 0)
        return fail(MVB_EINVAL, "splice_sum: bad sizes");
    if (out_len == 0) return MVB_OK;
    if (!pieces || !n_taps || !out) return fail(MVB_EINVAL, "splice_sum: null");
    prefer_carveout((const void*)k_splice_sum);
    k_splice_sum<<<grid_for(out_len, 256), 256, 0, as_stream(stream)>>>(
        pieces, piece_stride, n, hop, crossfade, n_blocks, n_taps, max_span, out, out_len);
    return check_launch("splice_sum");
}

}  // extern "C"
