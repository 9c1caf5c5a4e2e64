// Hand-written fp64 FFTs for the decimation decision and the anti-alias
// low-pass of decimate() (trajectory.py:214-232 _lowpass_columns,
// :316-339 bandwidth_estimate): the paths' rFFT / irFFT ran through cuFFT
// (a library) until round 2.
//
//   fft_c2c        batched complex FFT of any length n, rows contiguous:
//                  mixed-radix Stockham autosort (radices 4, 2, 3, 5, 7; one
//                  kernel per pass, ping-pong between two buffers, exact-
//                  argument sincospi twiddles) for 7-smooth n, Bluestein's
//                  chirp convolution through a smooth length M >= 2n - 1
//                  otherwise.  The sign is -1 (forward) or +1 (unnormalised
//                  inverse).
//   real rows      the low-pass packs two real rows into one complex row
//                  (x + i y): a real, even gain filters both parts at once;
//                  the bandwidth decision transforms each real row alone
//                  (see k_pack_centred).
//
// mvb_path_spectrum_index: centred paths -> power spectrum per (path, axis)
// -> first bin holding `fraction` of the energy (the bandwidth decision).
// mvb_lowpass_paths: odd-reflection padding, raised-cosine brickwall gain,
// inverse, crop -- the reference's _lowpass_columns for (G, T, 3) paths.
#include <cfloat>
#include <cstdlib>
#include <vector>

#include "mvb_common.cuh"

namespace mvb {
namespace {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
// e^{sign * 2 pi i num / den}, exact rational argument (num reduced mod den)
__device__ __forceinline__ double2 twiddle(int sign, int64_t num, int64_t den) {
    double s, c;
    sincospi(2.0 * (double)(num % den) / (double)den, &s, &c);
    return make_double2(c, sign * s);
}

// in-register DFT of size R: V[s] = sum_q v[q] e^{sign 2 pi i q s / R}
template <int R>
__device__ __forceinline__ void dft(double2 (&v)[R], int sign) {
    if constexpr (R == 2) {
        const double2 a = v[0], b = v[1];
        v[0] = cadd(a, b);
        v[1] = csub(a, b);
    } else if constexpr (R == 4) {
        const double2 s02 = cadd(v[0], v[2]), d02 = csub(v[0], v[2]);
        const double2 s13 = cadd(v[1], v[3]), d13 = csub(v[1], v[3]);
        const double2 id13 = make_double2(-sign * d13.y, sign * d13.x);  // sign * i * d13
        v[0] = cadd(s02, s13);
        v[2] = csub(s02, s13);
        v[1] = cadd(d02, id13);
        v[3] = csub(d02, id13);
    } else {
        // cos / sin (2 pi m / R), m < R (R = 3, 5, 7), correctly rounded
        constexpr double C3[3] = {1.0, -0.5, -0.5};
        constexpr double S3[3] = {0.0, 0.8660254037844386467637232, -0.8660254037844386467637232};
        constexpr double C5[5] = {1.0, 0.3090169943749474241022934, -0.8090169943749474241022934,
                                  -0.8090169943749474241022934, 0.3090169943749474241022934};
        constexpr double S5[5] = {0.0, 0.9510565162951535721164393, 0.587785252292473129168706,
                                  -0.587785252292473129168706, -0.9510565162951535721164393};
        constexpr double C7[7] = {1.0, 0.6234898018587335305250049, -0.2225209339563144042889026,
                                  -0.9009688679024191262361023, -0.9009688679024191262361023,
                                  -0.2225209339563144042889026, 0.6234898018587335305250049};
        constexpr double S7[7] = {0.0, 0.7818314824680298087084445, 0.9749279121818236070181317,
                                  0.4338837391175581204757683, -0.4338837391175581204757683,
                                  -0.9749279121818236070181317, -0.7818314824680298087084445};
        double2 out[R];
#pragma unroll
        for (int s = 0; s < R; ++s) {
            double2 acc = v[0];
#pragma unroll
            for (int q = 1; q < R; ++q) {
                const int m = (q * s) % R;
                const double c = R == 3 ? C3[m] : (R == 5 ? C5[m] : C7[m]);
                const double sn = R == 3 ? S3[m] : (R == 5 ? S5[m] : S7[m]);
                acc = cadd(acc, cmul(v[q], make_double2(c, sign * sn)));
            }
            out[s] = acc;
        }
#pragma unroll
        for (int s = 0; s < R; ++s) v[s] = out[s];
    }
}

// One Stockham pass of radix R over `rows` rows of length N: item j < N/R
// takes in[j + r N/R], twiddles by e^{sign 2 pi i (j mod Ns) r / (Ns R)},
// transforms, and writes out[(j / Ns) Ns R + (j mod Ns) + r Ns].
template <int R>
__global__ void k_fft_pass(const double2* __restrict__ in, double2* __restrict__ out, int64_t N,
                           int64_t Ns, int64_t rows, int sign) {
    const int64_t NR = N / R;
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= rows * NR) return;
    const int64_t row = t / NR, j = t - row * NR;
    const double2* a = in + row * N;
    double2* b = out + row * N;
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = a[j + r * NR];
    const int64_t k = j % Ns;
    if (k != 0) {
        // w^r by repeated products of w = e^{sign 2 pi i k / (Ns R)} (one
        // sincospi per item; <= 6 roundings of drift for R <= 7)
        const double2 w = twiddle(sign, k, Ns * R);
        double2 wr = w;
#pragma unroll
        for (int r = 1; r < R; ++r) {
            v[r] = cmul(v[r], wr);
            if (r + 1 < R) wr = cmul(wr, w);
        }
    }
    dft<R>(v, sign);
    const int64_t d = (j / Ns) * Ns * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) b[d + r * Ns] = v[r];
}

bool smooth_radices(int64_t n, std::vector<int>& rad) {
    rad.clear();
    for (int r : {4, 2, 3, 5, 7})
        while (n % r == 0) {
            rad.push_back(r);
            n /= r;
        }
    return n == 1;
}

int64_t next_smooth(int64_t m) {
    for (;; ++m) {
        int64_t q = m;
        for (int r : {2, 3, 5, 7})
            while (q % r == 0) q /= r;
        if (q == 1) return m;
    }
}

// run the passes of a smooth length n: input in `a`, result in `a`
// (scratch `b` holds the odd passes; a final copy when their count is odd)
// The decision's kernels run on the high-priority staging stream while a
// synthesis occupies the SMs; a kernel whose shared-memory carveout differs
// from the synthesis' makes an SM drain before it can host it.  Their
// preferred carveout is set once to MVB_FFT_CARVEOUT percent (default: the
// synthesis' 100 KB of 228).
template <class K>
void set_carveout(K* kernel) {
    static int pct = -2;
    if (pct == -2) {
        const char* e = getenv("MVB_FFT_CARVEOUT");
        pct = e ? atoi(e) : 44;
    }
    if (pct >= 0) cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
}

void set_fft_carveouts();

int stockham(double2* a, double2* b, int64_t rows, int64_t n, int sign, cudaStream_t s) {
    set_fft_carveouts();
    std::vector<int> rad;
    smooth_radices(n, rad);
    int64_t Ns = 1;
    double2 *src = a, *dst = b;
    for (int R : rad) {
        const int64_t items = rows * (n / R);
        const unsigned g = grid_for(items, 256);
        prefer_carveout(R == 2 ? (const void*)k_fft_pass<2> : R == 3 ? (const void*)k_fft_pass<3>
                        : R == 4 ? (const void*)k_fft_pass<4> : R == 5 ? (const void*)k_fft_pass<5>
                                                                  : (const void*)k_fft_pass<7>);
        switch (R) {
            case 2: k_fft_pass<2><<<g, 256, 0, s>>>(src, dst, n, Ns, rows, sign); break;
            case 3: k_fft_pass<3><<<g, 256, 0, s>>>(src, dst, n, Ns, rows, sign); break;
            case 4: k_fft_pass<4><<<g, 256, 0, s>>>(src, dst, n, Ns, rows, sign); break;
            case 5: k_fft_pass<5><<<g, 256, 0, s>>>(src, dst, n, Ns, rows, sign); break;
            default: k_fft_pass<7><<<g, 256, 0, s>>>(src, dst, n, Ns, rows, sign); break;
        }
        Ns *= R;
        double2* t = src;
        src = dst;
        dst = t;
    }
    if (src != a && cudaMemcpyAsync(a, src, sizeof(double2) * rows * n, cudaMemcpyDeviceToDevice, s) !=
                        cudaSuccess)
        return fail(MVB_ECUDA, "fft: copy");
    return check_launch("fft pass");
}

// Bluestein helpers: chirp c_j = e^{sign i pi j^2 / n} (exact j^2 mod 2n)
__device__ __forceinline__ double2 chirp(int sign, int64_t j, int64_t n) {
    const int64_t q = (j * j) % (2 * n);
    double s, c;
    sincospi((double)q / (double)n, &s, &c);
    return make_double2(c, sign * s);
}

// a[row][j] = x[row][j] c_j (j < n), 0 for n <= j < M
__global__ void k_blue_pre(const double2* __restrict__ x, double2* __restrict__ a, int64_t rows,
                           int64_t n, int64_t M, int sign) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= rows * M) return;
    const int64_t row = t / M, j = t - row * M;
    a[t] = j < n ? cmul(x[row * n + j], chirp(sign, j, n)) : make_double2(0.0, 0.0);
}

// b_j = conj c_j for j < n and b_{M-j} = conj c_j for 0 < j < n, else 0
__global__ void k_blue_kernel(double2* __restrict__ b, int64_t n, int64_t M, int sign) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= M) return;
    const int64_t q = j < n ? j : (M - j < n ? M - j : -1);
    b[j] = q >= 0 ? chirp(-sign, q, n) : make_double2(0.0, 0.0);
}

__global__ void k_blue_mul(double2* __restrict__ a, const double2* __restrict__ B, int64_t rows,
                           int64_t M) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= rows * M) return;
    a[t] = cmul(a[t], B[t % M]);
}

// X[row][k] = c_k a[row][k] / M, k < n
__global__ void k_blue_post(const double2* __restrict__ a, double2* __restrict__ X, int64_t rows,
                            int64_t n, int64_t M, int sign) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= rows * n) return;
    const int64_t row = t / n, k = t - row * n;
    const double2 v = cmul(a[row * M + k], chirp(sign, k, n));
    X[t] = make_double2(v.x / (double)M, v.y / (double)M);
}

}  // namespace

// complex elements of scratch fft_c2c needs for (rows, n)
int64_t fft_scratch_elems(int64_t rows, int64_t n) {
    std::vector<int> rad;
    if (smooth_radices(n, rad)) return rows * n;
    const int64_t M = next_smooth(2 * n - 1);
    return 2 * rows * M + 2 * M;  // a, its ping-pong partner, the kernel b and its partner
}

// in place on d (rows x n), scratch as fft_scratch_elems
int fft_c2c(double2* d, int64_t rows, int64_t n, int sign, double2* scratch, cudaStream_t s) {
    if (n <= 1 || rows <= 0) return MVB_OK;
    std::vector<int> rad;
    if (smooth_radices(n, rad)) return stockham(d, scratch, rows, n, sign, s);
    const int64_t M = next_smooth(2 * n - 1);
    double2* a = scratch;                 // rows x M
    double2* a2 = scratch + rows * M;     // rows x M
    double2* b = scratch + 2 * rows * M;  // M
    double2* b2 = b + M;                  // M
    prefer_carveout((const void*)k_blue_pre);
    k_blue_pre<<<grid_for(rows * M, 256), 256, 0, s>>>(d, a, rows, n, M, sign);
    prefer_carveout((const void*)k_blue_kernel);
    k_blue_kernel<<<grid_for(M, 256), 256, 0, s>>>(b, n, M, sign);
    int rc = stockham(a, a2, rows, M, -1, s);
    if (rc) return rc;
    rc = stockham(b, b2, 1, M, -1, s);
    if (rc) return rc;
    prefer_carveout((const void*)k_blue_mul);
    k_blue_mul<<<grid_for(rows * M, 256), 256, 0, s>>>(a, b, rows, M);
    rc = stockham(a, a2, rows, M, +1, s);
    if (rc) return rc;
    prefer_carveout((const void*)k_blue_post);
    k_blue_post<<<grid_for(rows * n, 256), 256, 0, s>>>(a, d, rows, n, M, sign);
    return check_launch("fft bluestein");
}

namespace {

// ---- bandwidth decision ---------------------------------------------------
// real rows p = 3 g + axis of the centred paths, one per complex row: for
// even T the row's own sample pairs z_j = x_{2j} + i x_{2j+1} (a half-length
// transform, packed_power unpacks it), else the samples with imag 0.  Two
// different rows are never packed together: the split would leak the
// partner row's spectrum at the eps * |Y_k| level, which decides the energy
// index of a (near-)constant axis next to a moving one.
__global__ void k_pack_centred(const double* __restrict__ x, int64_t G, int64_t T,
                               const double* __restrict__ mean, double2* __restrict__ z) {
    const int64_t P = 3 * G, half = T % 2 == 0, n = half ? T / 2 : T;
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= P * n) return;
    const int64_t p = t / n, j = t - p * n;
    const double* col = x + 3 * (p / 3) * T + p % 3;
    z[t] = half ? make_double2(col[3 * (2 * j)] - mean[p], col[3 * (2 * j + 1)] - mean[p])
                : make_double2(col[3 * j] - mean[p], 0.0);
}

// per-(path, axis) means in two wide passes (fixed order): PARTS partial
// sums per real row, then one warp per row folds them
constexpr int PARTS = 256;
__device__ __forceinline__ int64_t part_lo(int64_t n, int q) { return (n * q) / PARTS; }

__global__ void k_row_partials(const double* __restrict__ x, int64_t T, double* __restrict__ part) {
    __shared__ double red[8];
    const int64_t p = blockIdx.y, g = p / 3, ax = p % 3;
    const int q = blockIdx.x;
    double s = 0.0;
    for (int64_t t = part_lo(T, q) + threadIdx.x; t < part_lo(T, q + 1); t += blockDim.x)
        s += x[3 * (g * T + t) + ax];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        part[p * PARTS + q] = t;
    }
}

__global__ void k_row_means(const double* __restrict__ part, int64_t T, double* __restrict__ mean) {
    const int64_t p = blockIdx.x;
    double t = 0.0;
    for (int q = threadIdx.x; q < PARTS; q += 32) t += part[p * PARTS + q];
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) mean[p] = t / (double)T;
}

// |X_k|^2 of real row p (hypot, numpy.abs).  half = 0: row p holds the
// complex transform of the real row (length n).  half = 1 (even length
// 2n): row p holds the length-n transform Z of z_j = x_{2j} + i x_{2j+1}, and
// X_k = E_k + e^{-2 pi i k / 2n} O_k with E_k = (Z_k + conj Z_{n-k}) / 2,
// O_k = (Z_k - conj Z_{n-k}) / 2i (indices mod n) -- one signal's own
// even / odd halves, so no cross-row leakage.
__device__ __forceinline__ double packed_power(const double2* __restrict__ z, int64_t n, int64_t p,
                                               int64_t k, int half) {
    const double2* row = z + p * n;
    double re, im;
    if (!half) {
        re = row[k].x;
        im = row[k].y;
    } else {
        const double2 a = row[k % n], b = row[(n - k % n) % n];
        const double er = 0.5 * (a.x + b.x), ei = 0.5 * (a.y - b.y);  // E_k
        const double orr = 0.5 * (a.y + b.y), oi = -0.5 * (a.x - b.x);  // O_k
        double sw, cw;
        sincospi((double)k / (double)n, &sw, &cw);  // e^{-2 pi i k / 2n} = cw - i sw
        re = er + (cw * orr + sw * oi);
        im = ei + (cw * oi - sw * orr);
    }
    const double m = hypot(re, im);
    return m * m;
}

constexpr int IDX_THREADS = 256;

// power partial sums over bin ranges: part[p][q] = sum of |X_k|^2, k in part q
__global__ void k_power_partials(const double2* __restrict__ z, int64_t n, int64_t F, int half,
                                 double* __restrict__ part) {
    __shared__ double red[8];
    const int64_t p = blockIdx.y;
    const int q = blockIdx.x;
    double s = 0.0;
    for (int64_t k = part_lo(F, q) + threadIdx.x; k < part_lo(F, q + 1); k += blockDim.x)
        s += packed_power(z, n, p, k, half);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        part[p * PARTS + q] = t;
    }
}

// first bin k < F whose cumulative power reaches fraction x total (-1 when
// the row is all zero): warp 0 scans the PARTS partials (8 per lane) to find
// the part, then the block scans that part's bins in 256-wide tiles
__global__ void __launch_bounds__(IDX_THREADS) k_power_find(const double2* __restrict__ z, int64_t n,
                                                            int64_t F, double fraction, int half,
                                                            const double* __restrict__ part,
                                                            int64_t* __restrict__ out) {
    static_assert(PARTS == 256, "8 parts per lane");
    __shared__ double wsum[IDX_THREADS / 32];
    __shared__ double carry, thr_s;
    __shared__ int part_s, found;
    const int64_t p = blockIdx.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (w == 0) {
        const double* pp = part + p * PARTS + 8 * lane;
        double loc[8], sum = 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            loc[k] = pp[k];
            sum += loc[k];
        }
        double inc = sum;
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        const double tot = __shfl_sync(0xffffffffu, inc, 31);
        if (lane == 0) {
            part_s = -1;
            found = 0x7fffffff;
        }
        if (tot > 0.0) {
            const double thr = fraction * tot;
            double acc = inc - sum;
            int hit = -1;
            double hit_acc = 0.0;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                if (hit < 0 && acc + loc[k] >= thr) {
                    hit = 8 * lane + k;
                    hit_acc = acc;
                }
                acc += loc[k];
            }
            const unsigned m = __ballot_sync(0xffffffffu, hit >= 0);
            const int src = m ? __ffs(m) - 1 : 31;
            const int q = __shfl_sync(0xffffffffu, hit, src);
            const double a = __shfl_sync(0xffffffffu, hit_acc, src);
            if (lane == 0) {
                part_s = q >= 0 ? q : PARTS - 1;  // rounding: the last part
                thr_s = thr;
                if (q >= 0) carry = a;
            }
            if (q < 0 && lane == 31) carry = inc - loc[7];
        }
    }
    __syncthreads();
    if (part_s < 0) {
        if (threadIdx.x == 0) out[p] = -1;
        return;
    }
    const double thr = thr_s;
    const int64_t f0 = part_lo(F, part_s), f1 = part_lo(F, part_s + 1);
    for (int64_t base = f0; base < f1; base += IDX_THREADS) {
        const int64_t k = base + threadIdx.x;
        double v = k < f1 ? packed_power(z, n, p, k, half) : 0.0;
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += y;
        }
        if (lane == 31) wsum[w] = v;
        __syncthreads();
        double pre = carry;
        for (int q = 0; q < w; ++q) pre += wsum[q];
        if (k < f1 && pre + v >= thr) atomicMin(&found, (int)threadIdx.x);
        __syncthreads();
        if (found != 0x7fffffff) {
            if (threadIdx.x == 0) out[p] = base + found;
            return;
        }
        if (threadIdx.x == IDX_THREADS - 1) carry = pre + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) out[p] = f1 - 1;  // rounding: the part's end reaches thr
}

// ---- low-pass --------------------------------------------------------------
// odd-reflection padded rows (trajectory.py:219-222): ext = [2 x0 - x[pad:0:-1],
// x, 2 x[-1] - x[-2:-pad-2:-1]], two real rows per complex row
__device__ __forceinline__ double ext_at(const double* __restrict__ x, int64_t T, int64_t pad,
                                         int64_t p, int64_t e) {
    const int64_t g = p / 3, ax = p % 3;
    const double* col = x + 3 * g * T + ax;
    if (e < pad) return 2.0 * col[0] - col[3 * (pad - e)];
    if (e < pad + T) return col[3 * (e - pad)];
    const int64_t u = e - pad - T;  // 0 .. pad-1: x[-2 - u]
    return 2.0 * col[3 * (T - 1)] - col[3 * (T - 2 - u)];
}

__global__ void k_pack_ext(const double* __restrict__ x, int64_t G, int64_t T, int64_t pad,
                           int64_t m, double2* __restrict__ z) {
    const int64_t P = 3 * G, Q = (P + 1) / 2;
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= Q * m) return;
    const int64_t q = t / m, e = t - q * m;
    const double re = ext_at(x, T, pad, 2 * q, e);
    const double im = 2 * q + 1 < P ? ext_at(x, T, pad, 2 * q + 1, e) : 0.0;
    z[t] = make_double2(re, im);
}

// spectrum x gain: rfftfreq f_k = k * (1 / (m * (1 / rate))) for the bin's
// |frequency| (bins k and m - k share it); raised-cosine edge on (lo, hi]
__global__ void k_lowpass_gain(double2* __restrict__ z, int64_t rows, int64_t m, double rate,
                               double cutoff) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= rows * m) return;
    const int64_t k = t % m;
    const int64_t kk = k <= m - k ? k : m - k;
    const double f = (double)kk * (1.0 / ((double)m * (1.0 / rate)));
    const double lo = 0.8 * cutoff, hi = cutoff;
    double g = 1.0;
    if (f > hi) g = 0.0;
    else if (f > lo) g = 0.5 * (1.0 + cos(M_PI * (f - lo) / (hi - lo)));
    z[t] = make_double2(z[t].x * g, z[t].y * g);
}

// out (G, T, 3) = ext[pad : pad + T] / m of the inverse transform
__global__ void k_unpack_crop(const double2* __restrict__ z, int64_t G, int64_t T, int64_t pad,
                              int64_t m, double* __restrict__ out) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= 3 * G * T) return;
    const int64_t g = t / (3 * T), r = t - g * 3 * T, s = r / 3, ax = r % 3;
    const int64_t p = 3 * g + ax;
    const double2 v = z[(p / 2) * m + pad + s];
    out[t] = ((p & 1) ? v.y : v.x) / (double)m;
}

void set_fft_carveouts() {
    static bool done = false;
    if (done) return;
    done = true;
    set_carveout(k_fft_pass<2>);
    set_carveout(k_fft_pass<3>);
    set_carveout(k_fft_pass<4>);
    set_carveout(k_fft_pass<5>);
    set_carveout(k_fft_pass<7>);
    set_carveout(k_blue_pre);
    set_carveout(k_blue_kernel);
    set_carveout(k_blue_mul);
    set_carveout(k_blue_post);
    set_carveout(k_row_partials);
    set_carveout(k_row_means);
    set_carveout(k_pack_centred);
    set_carveout(k_power_partials);
    set_carveout(k_power_find);
    set_carveout(k_pack_ext);
    set_carveout(k_lowpass_gain);
    set_carveout(k_unpack_crop);
}

}  // namespace
}  // namespace mvb

using namespace mvb;

extern "C" {

int64_t mvb_fft_scratch_elems(int64_t rows, int64_t n) { return fft_scratch_elems(rows, n); }

int mvb_fft_c2c(double* d_data, int64_t rows, int64_t n, int sign, double* d_scratch, void* stream) {
    if (rows < 0 || n < 0 || (sign != 1 && sign != -1)) return fail(MVB_EINVAL, "fft_c2c: args");
    if (rows == 0 || n <= 1) return MVB_OK;
    if (!d_data || !d_scratch) return fail(MVB_EINVAL, "fft_c2c: null");
    return fft_c2c(reinterpret_cast<double2*>(d_data), rows, n, sign,
                   reinterpret_cast<double2*>(d_scratch), as_stream(stream));
}

int64_t mvb_path_spectrum_scratch(int64_t G, int64_t T) {
    const int64_t P = 3 * G;
    return 2 * P * T + 2 * fft_scratch_elems(P, T) + P * (PARTS + 1) + 8;  // doubles
}

int mvb_path_spectrum_index(const double* d_x, int64_t G, int64_t T, double fraction,
                            double* d_scratch, int64_t* d_index, void* stream) {
    if (G < 0 || G > 65535 || T < 0 || !(fraction > 0.0 && fraction < 1.0))
        return fail(MVB_EINVAL, "path_spectrum_index: args");
    if (G == 0 || T < 2) return MVB_OK;
    if (!d_x || !d_scratch || !d_index) return fail(MVB_EINVAL, "path_spectrum_index: null");
    set_fft_carveouts();
    cudaStream_t s = as_stream(stream);
    const int64_t P = 3 * G, F = T / 2 + 1;
    const int half = T % 2 == 0;
    const int64_t n = half ? T / 2 : T;  // transform length per row
    double2* z = reinterpret_cast<double2*>(d_scratch);
    double2* fs = z + P * T;
    double* part = reinterpret_cast<double*>(fs + fft_scratch_elems(P, T));  // P x PARTS
    double* mean = part + P * PARTS;                                          // P
    prefer_carveout((const void*)k_row_partials);
    k_row_partials<<<dim3(PARTS, (unsigned)P), 256, 0, s>>>(d_x, T, part);
    prefer_carveout((const void*)k_row_means);
    k_row_means<<<(unsigned)P, 32, 0, s>>>(part, T, mean);
    prefer_carveout((const void*)k_pack_centred);
    k_pack_centred<<<grid_for(P * n, 256), 256, 0, s>>>(d_x, G, T, mean, z);
    const int rc = fft_c2c(z, P, n, -1, fs, s);
    if (rc) return rc;
    prefer_carveout((const void*)k_power_partials);
    k_power_partials<<<dim3(PARTS, (unsigned)P), 256, 0, s>>>(z, n, F, half, part);
    prefer_carveout((const void*)k_power_find);
    k_power_find<<<(unsigned)P, IDX_THREADS, 0, s>>>(z, n, F, fraction, half, part, d_index);
    return check_launch("path_spectrum_index");
}

int64_t mvb_lowpass_scratch(int64_t G, int64_t T) {
    const int64_t pad = T - 1 < (T / 4 > 16 ? T / 4 : 16) ? T - 1 : (T / 4 > 16 ? T / 4 : 16);
    const int64_t m = T + 2 * pad, Q = (3 * G + 1) / 2;
    return 2 * Q * m + 2 * fft_scratch_elems(Q, m);  // doubles
}

int mvb_lowpass_paths(const double* d_x, int64_t G, int64_t T, double rate, double cutoff,
                      double* d_scratch, double* d_out, void* stream) {
    if (G < 0 || G > 65535 || T < 0 || !(rate > 0.0)) return fail(MVB_EINVAL, "lowpass_paths: args");
    if (G == 0 || T == 0) return MVB_OK;
    if (!d_x || !d_scratch || !d_out) return fail(MVB_EINVAL, "lowpass_paths: null");
    if (T < 2) return cudaMemcpyAsync(d_out, d_x, 24 * G * T, cudaMemcpyDeviceToDevice,
                                      as_stream(stream)) == cudaSuccess
                          ? MVB_OK : fail(MVB_ECUDA, "lowpass_paths: copy");
    cudaStream_t s = as_stream(stream);
    // pad = min(n - 1, max(16, n // 4)) (trajectory.py:217)
    const int64_t pad = T - 1 < (T / 4 > 16 ? T / 4 : 16) ? T - 1 : (T / 4 > 16 ? T / 4 : 16);
    const int64_t m = T + 2 * pad, Q = (3 * G + 1) / 2;
    double2* z = reinterpret_cast<double2*>(d_scratch);
    double2* fs = z + Q * m;
    prefer_carveout((const void*)k_pack_ext);
    k_pack_ext<<<grid_for(Q * m, 256), 256, 0, s>>>(d_x, G, T, pad, m, z);
    int rc = fft_c2c(z, Q, m, -1, fs, s);
    if (rc) return rc;
    prefer_carveout((const void*)k_lowpass_gain);
    k_lowpass_gain<<<grid_for(Q * m, 256), 256, 0, s>>>(z, Q, m, rate, cutoff);
    rc = fft_c2c(z, Q, m, +1, fs, s);
    if (rc) return rc;
    prefer_carveout((const void*)k_unpack_crop);
    k_unpack_crop<<<grid_for(3 * G * T, 256), 256, 0, s>>>(z, G, T, pad, m, d_out);
    return check_launch("lowpass_paths");
}

}  // extern "C"
