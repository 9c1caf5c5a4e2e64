// Operator boundary of libmvb.so: the reference's kernel trio
// (/root/reference/pkg/src/moverb/_kernels.py), its branch filter
// (farrow.py:214-229) and the image lattice (room.py:98-143, 175-187).
//
// These are fp64 and follow the reference's per-element arithmetic order
// exactly (explicit _rn intrinsics, no FMA contraction), so their results are
// bit-identical to the numba kernels on identical inputs.  One thread per
// output element; each thread's reduction runs in the reference's order.
#include <mutex>
#include <string>

#include "mvb_common.cuh"

namespace mvb {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
const char* get_error() { return g_err.c_str(); }

// _kernels.py:54-62
__global__ void k_distance(const double* __restrict__ off, const double* __restrict__ sgn,
                           const double* __restrict__ mic, const double* __restrict__ pos,
                           int64_t S, int64_t T, double* __restrict__ out) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t i = blockIdx.y;
    if (t >= T || i >= S) return;
    double m[3] = {mic[0], mic[1], mic[2]};
    out[i * T + t] = exact_distance(off[3 * i], off[3 * i + 1], off[3 * i + 2], sgn[3 * i],
                                    sgn[3 * i + 1], sgn[3 * i + 2], pos + 3 * t, m);
}

// _kernels.py:109-123: thread n walks the images in order, like the numba
// loop nest does for each n.
__global__ void k_accumulate(double* __restrict__ out, int64_t out_len,
                             const double* __restrict__ streams, int64_t nb, int64_t ls,
                             const double* __restrict__ tau, const double* __restrict__ amp,
                             int64_t S, int64_t offset, int64_t d0) {
    int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (n >= out_len) return;
    double o = out[n];
    const double off = (double)offset, dd0 = (double)d0;
    for (int64_t i = 0; i < S; ++i) {
        double shifted = xadd(tau[i * out_len + n], off);
        double d_int = floor(xsub(shifted, dd0));
        double mu = xsub(xsub(shifted, dd0), d_int);
        int64_t idx = n + offset - (int64_t)d_int;
        if (idx >= 0 && idx < ls) {
            double acc = streams[(nb - 1) * ls + idx];
            for (int64_t k = nb - 2; k >= 0; --k) acc = xadd(xmul(acc, mu), streams[k * ls + idx]);
            o = xadd(o, xmul(amp[i * out_len + n], acc));
        }
    }
    out[n] = o;
}

// _kernels.py:164-181, batched over rows
__global__ void k_upsample(const double* __restrict__ coarse, int64_t rows, int64_t nc,
                           const double* __restrict__ table, int64_t factor, int64_t ntaps,
                           int64_t out_len, double* __restrict__ out) {
    int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t r = blockIdx.y;
    if (m >= out_len || r >= rows) return;
    const double* c = coarse + r * nc;
    int64_t half = (ntaps - 1) / 2;
    int64_t base = m / factor, phase = m - (m / factor) * factor;
    double acc = 0.0;
    for (int64_t col = 0; col < ntaps; ++col) {
        int64_t j = base + (col - half);
        j = j < 0 ? 0 : (j >= nc ? nc - 1 : j);
        acc = xadd(acc, xmul(table[phase * ntaps + col], c[j]));
    }
    out[r * out_len + m] = acc;
}

// farrow.py:214-229 (full convolution per branch, sequential sum over taps)
__global__ void k_branch_filter(const double* __restrict__ x, int64_t T,
                                const double* __restrict__ br, int64_t nb, int64_t L,
                                double* __restrict__ out) {
    int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t k = blockIdx.y;
    int64_t ls = T + L - 1;
    if (m >= ls || k >= nb) return;
    int64_t jlo = m - (T - 1) > 0 ? m - (T - 1) : 0;
    int64_t jhi = m < L - 1 ? m : L - 1;
    const double* c = br + k * L;
    double acc = 0.0;
    for (int64_t j = jlo; j <= jhi; ++j) acc = xadd(acc, xmul(c[j], x[m - j]));
    out[k * ls + m] = acc;
}

// ---------------------------------------------------------------------------
// image lattice: one CTA per (room, order o); each thread decodes image
// triples of order o, keys them by (lattice, parity) and ranks them inside
// the order block (the canonical order of room.py:82-95 sorts by order
// first, so blocks are contiguous at base(o) = count(order < o)).

__device__ __forceinline__ void decode_triple(int o, int idx, int& jx, int& jy, int& jz) {
    if (o == 0) { jx = jy = jz = 0; return; }
    for (int x = -o; x <= o; ++x) {
        int m = o - (x < 0 ? -x : x);
        int cnt = m == 0 ? 1 : 4 * m;
        if (idx >= cnt) { idx -= cnt; continue; }
        jx = x;
        for (int y = -m; y <= m; ++y) {
            int r = m - (y < 0 ? -y : y);
            int c2 = r == 0 ? 1 : 2;
            if (idx >= c2) { idx -= c2; continue; }
            jy = y;
            jz = r == 0 ? 0 : (idx == 0 ? -r : r);
            return;
        }
    }
}

__device__ __forceinline__ int pydiv2(int a) { return a >= 0 ? a / 2 : -((-a + 1) / 2); }

// x^n for integer n >= 0, carried in double-double (error-free products via
// FMA) and rounded once: the correctly rounded power, which is what the
// reference's `float ** int` (glibc pow) returns.
__device__ double ipow_rn(double x, int n) {
    double rh = 1.0, rl = 0.0;  // result
    double bh = x, bl = 0.0;    // base^(2^k)
    while (n > 0) {
        if (n & 1) {
            double p = rh * bh;
            double e = fma(rh, bh, -p) + (rh * bl + rl * bh);
            rh = p + e;
            rl = e - (rh - p);
        }
        n >>= 1;
        if (n) {
            double p = bh * bh;
            double e = fma(bh, bh, -p) + 2.0 * bh * bl;
            bh = p + e;
            bl = e - (bh - p);
        }
    }
    return rh + rl;
}

__global__ void k_enumerate(const double* __restrict__ dims, const double* __restrict__ walls,
                            int max_order, int64_t S, int32_t* __restrict__ lattice,
                            int32_t* __restrict__ parity, int32_t* __restrict__ order,
                            double* __restrict__ beta, double* __restrict__ offset,
                            double* __restrict__ sign) {
    extern __shared__ int64_t keys[];
    const int o = blockIdx.x;
    const int64_t room = blockIdx.y;
    const int n = o == 0 ? 1 : 4 * o * o + 2;
    // blockIdx.z: which 256-image chunk of the order this block ranks
    const int c0 = blockIdx.z * blockDim.x;
    if (c0 >= n) return;
    int64_t base = 0;
    if (o > 0) {
        base = 1;
        for (int q = 1; q < o; ++q) base += 4LL * q * q + 2;
    }
    for (int idx = threadIdx.x; idx < n; idx += blockDim.x) {
        int js[3];
        decode_triple(o, idx, js[0], js[1], js[2]);
        int64_t key = 0;
        for (int k = 0; k < 3; ++k) {
            int q = js[k] & 1;
            int l = pydiv2(js[k] + q);
            key = (key << 7) | (int64_t)(l + 64);
        }
        for (int k = 0; k < 3; ++k) key = (key << 1) | (int64_t)(js[k] & 1);
        keys[idx] = key;
    }
    __syncthreads();
    const double* dm = dims + 3 * room;
    const double* wl = walls + 6 * room;
    for (int idx = c0 + threadIdx.x; idx < n && idx < c0 + (int)blockDim.x; idx += blockDim.x) {
        int64_t mine = keys[idx];
        int rank = 0;
        for (int j = 0; j < n; ++j) rank += keys[j] < mine;
        int js[3];
        decode_triple(o, idx, js[0], js[1], js[2]);
        int64_t row = room * S + base + rank;
        double b = 1.0;
        for (int k = 0; k < 3; ++k) {
            int j = js[k];
            int q = j & 1;
            int l = pydiv2(j + q);
            int hm, hp;  // room.py:98-105
            if (j >= 0) { hm = j / 2; hp = (j + 1) / 2; }
            else { hm = (-j + 1) / 2; hp = (-j) / 2; }
            b = xmul(b, xmul(ipow_rn(wl[2 * k], hm), ipow_rn(wl[2 * k + 1], hp)));
            if (lattice) lattice[3 * row + k] = l;
            if (parity) parity[3 * row + k] = q;
            if (offset) offset[3 * row + k] = xmul(xmul(2.0, (double)l), dm[k]);
            if (sign) sign[3 * row + k] = q ? -1.0 : 1.0;
        }
        if (order) order[row] = o;
        if (beta) beta[row] = b;
    }
}

}  // namespace mvb

using namespace mvb;

extern "C" {

int mvb_abi_version(void) { return MVB_ABI_VERSION; }

#ifdef MVB_CHECKED
void mvb_check_collect_synth(int64_t* h);
#endif

int mvb_check_violations(int64_t* h_counts, int n) {
#ifdef MVB_CHECKED
    if (!h_counts || n < 1) return fail(MVB_EINVAL, "check_violations: args");
    int64_t c[CHK_COUNT] = {};
    mvb_check_collect(c);       // this unit's counters
    mvb_check_collect_synth(c); // the synthesis kernels'
    for (int i = 0; i < n && i < CHK_COUNT; ++i) h_counts[i] = c[i];
    return CHK_COUNT;
#else
    (void)h_counts;
    (void)n;
    return fail(MVB_EINVAL, "check_violations: not a checked build (libmvb_checked.so)");
#endif
}
const char* mvb_last_error(void) { return get_error(); }

int mvb_device_info(int* sm_count, int* cc_major, int* cc_minor) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return fail(MVB_ECUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
    cudaDeviceProp p;
    e = cudaGetDeviceProperties(&p, dev);
    if (e != cudaSuccess) return fail(MVB_ECUDA, cudaGetErrorString(e));
    if (sm_count) *sm_count = p.multiProcessorCount;
    if (cc_major) *cc_major = p.major;
    if (cc_minor) *cc_minor = p.minor;
    return MVB_OK;
}

int mvb_copy_batch(void* const* dst, const void* const* src, const int64_t* bytes, int64_t n,
                   int32_t* issued, int require_pinned, void* stream) {
    if (n < 0) return fail(MVB_EINVAL, "copy_batch: n");
    if (n == 0) return MVB_OK;
    if (!dst || !src || !bytes || !issued) return fail(MVB_EINVAL, "copy_batch: null");
    cudaStream_t s = as_stream(stream);
    for (int64_t i = 0; i < n; ++i) {
        issued[i] = 0;
        if (bytes[i] < 0) return fail(MVB_EINVAL, "copy_batch: negative size");
        if (bytes[i] == 0) {
            issued[i] = 1;
            continue;
        }
        if (require_pinned) {
            cudaPointerAttributes a;
            if (cudaPointerGetAttributes(&a, src[i]) != cudaSuccess) {
                cudaGetLastError();  // pageable memory on old runtimes: not an error here
                continue;
            }
            if (a.type != cudaMemoryTypeHost) continue;
        }
        cudaError_t e = cudaMemcpyAsync(dst[i], src[i], (size_t)bytes[i], cudaMemcpyDefault, s);
        if (e != cudaSuccess) return fail(MVB_ECUDA, std::string("copy_batch: ") + cudaGetErrorString(e));
        issued[i] = 1;
    }
    return MVB_OK;
}

int mvb_struct_sizes(int* image, int* job, int* work, int* coef) {
    if (image) *image = (int)sizeof(mvb_image);
    if (job) *job = (int)sizeof(mvb_job);
    if (work) *work = (int)sizeof(mvb_work);
    if (coef) *coef = (int)sizeof(mvb_coef32);
    return MVB_OK;
}

int mvb_distance_streams(const double* off, const double* sgn, const double* mic,
                         const double* pos, int64_t S, int64_t T, double* out, void* stream) {
    if (S < 0 || T < 0 || S > 65535) return fail(MVB_EINVAL, "distance_streams: bad S/T");
    if (S == 0 || T == 0) return MVB_OK;
    if (!off || !sgn || !mic || !pos || !out) return fail(MVB_EINVAL, "distance_streams: null");
    dim3 g(grid_for(T, 256), (unsigned)S);
    prefer_carveout((const void*)k_distance);
    k_distance<<<g, 256, 0, as_stream(stream)>>>(off, sgn, mic, pos, S, T, out);
    return check_launch("distance_streams");
}

int mvb_accumulate_images(double* out, int64_t out_len, const double* streams, int64_t nb,
                          int64_t ls, const double* tau, const double* amp, int64_t S,
                          int64_t offset, int64_t d0, void* stream) {
    if (out_len < 0 || S < 0 || nb < 1 || ls < 0) return fail(MVB_EINVAL, "accumulate: bad sizes");
    if (out_len == 0 || S == 0) return MVB_OK;
    if (!out || !streams || !tau || !amp) return fail(MVB_EINVAL, "accumulate: null");
    prefer_carveout((const void*)k_accumulate);
    k_accumulate<<<grid_for(out_len, 128), 128, 0, as_stream(stream)>>>(out, out_len, streams, nb,
                                                                        ls, tau, amp, S, offset, d0);
    return check_launch("accumulate_images");
}

int mvb_upsample_streams(const double* coarse, int64_t rows, int64_t nc, const double* table,
                         int64_t factor, int64_t ntaps, int64_t out_len, double* out,
                         void* stream) {
    if (rows < 0 || nc < 1 || factor < 1 || ntaps < 1 || out_len < 0 || rows > 65535)
        return fail(MVB_EINVAL, "upsample: bad sizes");
    if (rows == 0 || out_len == 0) return MVB_OK;
    if (!coarse || !table || !out) return fail(MVB_EINVAL, "upsample: null");
    dim3 g(grid_for(out_len, 256), (unsigned)rows);
    prefer_carveout((const void*)k_upsample);
    k_upsample<<<g, 256, 0, as_stream(stream)>>>(coarse, rows, nc, table, factor, ntaps, out_len, out);
    return check_launch("upsample_streams");
}

int mvb_branch_filter(const double* x, int64_t T, const double* br, int64_t nb, int64_t L,
                      double* out, void* stream) {
    if (T < 1 || nb < 1 || L < 1 || nb > 65535) return fail(MVB_EINVAL, "branch_filter: bad sizes");
    if (!x || !br || !out) return fail(MVB_EINVAL, "branch_filter: null");
    dim3 g(grid_for(T + L - 1, 256), (unsigned)nb);
    prefer_carveout((const void*)k_branch_filter);
    k_branch_filter<<<g, 256, 0, as_stream(stream)>>>(x, T, br, nb, L, out);
    return check_launch("branch_filter");
}

int64_t mvb_image_count(int max_order) {
    if (max_order < 0) return 0;
    int64_t n = 1;
    for (int o = 1; o <= max_order; ++o) n += 4LL * o * o + 2;
    return n;
}

int mvb_enumerate(const double* dims, const double* walls, int64_t n_rooms, int max_order,
                  int32_t* lattice, int32_t* parity, int32_t* order, double* beta,
                  double* offset, double* sign, void* stream) {
    // one order block's keys live in shared memory: 8 * (4 o^2 + 2) bytes
    if (max_order < 0 || max_order > 80) return fail(MVB_EINVAL, "enumerate: max_order in [0,80]");
    if (n_rooms < 0 || n_rooms > 65535) return fail(MVB_EINVAL, "enumerate: n_rooms");
    if (n_rooms == 0) return MVB_OK;
    if (!dims || !walls) return fail(MVB_EINVAL, "enumerate: null dims/walls");
    int64_t S = mvb_image_count(max_order);
    int nmax = max_order == 0 ? 1 : 4 * max_order * max_order + 2;
    size_t smem = sizeof(int64_t) * (size_t)nmax;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k_enumerate, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return fail(MVB_ECUDA, cudaGetErrorString(e));
    }
    dim3 g((unsigned)(max_order + 1), (unsigned)n_rooms, (unsigned)((nmax + 255) / 256));
    prefer_carveout((const void*)k_enumerate);
    k_enumerate<<<g, 256, smem, as_stream(stream)>>>(dims, walls, max_order, S, lattice, parity,
                                                    order, beta, offset, sign);
    return check_launch("enumerate");
}

}  // extern "C"
