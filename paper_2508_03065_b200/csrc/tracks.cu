// Hierarchical delay tracks (synth.py:122-158, trajectory.py:260-298,
// _kernels.py:149-190) for batched fused renders.  Every kernel covers all
// jobs of a batch in one launch; an image finds its job, paths and tier
// constants through the fields of mvb_image.
//
//   k_coarse_bounds    coarse distances per (image, coarse sample) -- the
//                      reference's distance arithmetic on pos[::N] -- fused
//                      with the per-image bounds of the upsampled max
//   k_path_bbox / k_bounds_full  bounds of the full-rate images' max
//   k_select/k_exact_max  exact max over the images that can hold it
//   k_coeffs           fast-path interval records: the 65-tap Kaiser
//                      upsampler refit per coarse interval as a degree-8
//                      polynomial in u, anchored in fp64, pre-split (B, f)
//   k_sort_keys        per-(job, time segment) delay-sort keys (L1 locality)
#include <algorithm>
#include <cfloat>

#include <cub/block/block_radix_sort.cuh>

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

// Decimated images: lb = largest coarse sample (attained to ~1e-12 m: the
// phase-0 row of the table is a unit impulse up to sinc(integer) rounding);
// ub = max over 64-sample segments s of M + negsum (M - m), M/m the max/min
// over segments s-1..s+1 (a superset of every 65-tap window centred in s).
// With weights summing to 1 whose negative mass is <= negsum, any window
// value is <= wmax + negsum (wmax - wmin).
__device__ __forceinline__ void warp_maxmin(double& M, double& m) {
    for (int o = 16; o > 0; o >>= 1) {
        M = fmax(M, __shfl_xor_sync(0xffffffffu, M, o));
        m = fmin(m, __shfl_xor_sync(0xffffffffu, m, o));
    }
}

// max / min of coarse samples [64 s, 64 s + 64) (clipped to K), warp-uniform
__device__ __forceinline__ void seg_maxmin(const double* c, int64_t K, int64_t s, int lane,
                                           double& M, double& m) {
    M = -DBL_MAX;
    m = DBL_MAX;
    const int64_t a = 64 * s + lane, b = a + 32;
    if (a < K) { const double v = c[a]; M = v; m = v; }
    if (b < K) { const double v = c[b]; M = fmax(M, v); m = fmin(m, v); }
    warp_maxmin(M, m);
}

// Coarse distances of the decimated images (the reference's distance
// arithmetic on pos[::N]) fused with their track bounds: a warp handles
// CB_SEGS 64-sample segments of one image (blockIdx.y = chunk), computes and
// writes them in order and keeps a sliding window of three segments (the
// neighbours just outside the chunk are recomputed, not written), so the
// coarse array is written once and never re-read for the bounds.  The
// window bound only has to be an upper bound, so segment max / min are
// reduced in fp32 rounded outward (one SHFL + FMNMX per step; an fp64
// shuffle-max costs ~20 instructions); lb, which seeds the exact maximum,
// stays the exact fp64 coarse max (lane-local, one reduction per chunk).
// Chunk results merge atomically into the zero-initialised lb / ub.
constexpr int CB_SEGS = 16;  // chunk length of large launches (8 for small ones, below)

__device__ __forceinline__ void warp_maxmin_f(float& M, float& m) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
        m = fminf(m, __shfl_xor_sync(0xffffffffu, m, o));
    }
}

template <int CB_SEGS>
__global__ void k_coarse_bounds(const mvb_image* __restrict__ images, const int32_t* __restrict__ sel,
                                int64_t n_sel, const mvb_job* __restrict__ jobs,
                                const double* __restrict__ paths, double negsum,
                                double* __restrict__ coarse, double* __restrict__ lb,
                                double* __restrict__ ub) {
    // The CTA's eight warps (images of one factor class, consecutive in
    // `sel`, normally of one job) read the same coarse source path window:
    // it is staged once per CTA in shared memory (the kernel is bound by the
    // latency of these loads); a warp whose image has another path reads
    // global memory.
    __shared__ double sp[3 * 64 * (CB_SEGS + 2)];
    // segments [seg_lo, seg_hi) of an image: its job's time-shard window
    // (win_coarse; the whole track without one), chunk blockIdx.y of them
    auto seg_range = [&](const mvb_image& q, int64_t& lo, int64_t& hi) {
        int64_t k0, k1;
        win_coarse(jobs[q.job], q.factor, q.n_coarse, k0, k1);
        lo = k0 / 64;
        hi = (k1 + 63) / 64;
    };
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (int64_t)blockIdx.x * (blockDim.x >> 5);
    int64_t r0 = 0, r1 = 0, ref_cpath = -1;
    {
        const mvb_image& ref = images[sel[w0]];  // w0 < n_sel by the grid
        const int64_t Kr = ref.n_coarse;
        int64_t lo, nsr;
        seg_range(ref, lo, nsr);
        const int64_t s0 = lo + (int64_t)blockIdx.y * CB_SEGS;
        if (s0 < nsr) {
            const int64_t s1r = s0 + CB_SEGS < nsr ? s0 + CB_SEGS : nsr;
            r0 = s0 > 0 ? 64 * (s0 - 1) : 0;
            r1 = 64 * (s1r + 1) < Kr ? 64 * (s1r + 1) : Kr;
            ref_cpath = ref.cpath;
            const double* g = paths + 3 * ref.cpath + 3 * r0;
            for (int64_t t = threadIdx.x; t < 3 * (r1 - r0); t += blockDim.x) sp[t] = g[t];
        }
    }
    __syncthreads();
    const int64_t w = w0 + (threadIdx.x >> 5);
    if (w >= n_sel) return;
    const int32_t i = sel[w];
    const mvb_image im = images[i];
    const int64_t K = im.n_coarse;
    const int64_t nseg = (K + 63) / 64;
    int64_t seg_lo, seg_hi;
    seg_range(im, seg_lo, seg_hi);
    const int64_t s0 = seg_lo + (int64_t)blockIdx.y * CB_SEGS;
    if (s0 >= seg_hi) return;
    const int64_t s1 = s0 + CB_SEGS < seg_hi ? s0 + CB_SEGS : seg_hi;
    const mvb_job& J = jobs[im.job];
    const bool staged = im.cpath == ref_cpath;  // same path rows, same K
    const double* src = staged ? sp : paths + 3 * im.cpath;
    const int64_t soff = staged ? r0 : 0;       // src row of coarse sample k: k - soff
    const double* mic = J.mic_moving ? paths + 3 * (im.cpath + K) : paths + 3 * J.mic_off;
    const int64_t mstep = J.mic_moving ? 3 : 0;
    double* c = coarse + im.coarse;
    double vmax = 0.0;  // lane-local exact max of the written samples (lb)
    // segment s: distances of its 64 samples (written when `write`), and
    // its max / min rounded outward to fp32, warp-uniform
    auto segment = [&](int64_t s, bool write, float& M, float& m) {
        M = -FLT_MAX;
        m = FLT_MAX;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t k = 64 * s + 32 * h + lane;
            if (k < K) {
                const double v = image_distance(im, src + 3 * (k - soff), mic + mstep * k);
                if (write) {
                    c[k] = v;
                    vmax = v > vmax ? v : vmax;
                }
                M = fmaxf(M, __double2float_ru(v));
                m = fminf(m, __double2float_rd(v));
            }
        }
        warp_maxmin_f(M, m);
    };
    float Mp = -FLT_MAX, mp = FLT_MAX, Mc, mc, Mn, mn;
    if (s0 > 0) segment(s0 - 1, false, Mp, mp);
    segment(s0, true, Mc, mc);
    float best_ub = 0.f;
    const float ns = __double2float_ru(negsum);
    for (int64_t s = s0; s < s1; ++s) {
        if (s + 1 < nseg) segment(s + 1, s + 1 < s1, Mn, mn);
        else { Mn = -FLT_MAX; mn = FLT_MAX; }
        const float M = fmaxf(Mp, fmaxf(Mc, Mn)), m = fminf(mp, fminf(mc, mn));
        // M + negsum (M - m) + 1e-9 evaluated upward (fp32 ulp at 400 m: 3e-5 m)
        best_ub = fmaxf(best_ub, __fadd_ru(M, __fmul_ru(ns, __fsub_ru(M, m))));
        Mp = Mc; mp = mc; Mc = Mn; mc = mn;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double t = __shfl_xor_sync(0xffffffffu, vmax, o);
        vmax = t > vmax ? t : vmax;
    }
    if (lb && lane == 0) {
        atomic_max_pos(lb + i, vmax);
        atomic_max_pos(ub + i, (double)best_ub + 1e-9);
    }
}

// Axis-aligned bounding boxes of every job's source path and receiver
// (moving or fixed) and their largest per-sample step:
// bbox[j] = (src lo xyz, src hi xyz, mic lo xyz, mic hi xyz, src max step,
// mic max step, 0, 0) -- the steps bound the delay excursion of a coarse
// interval (the fp32 fast path's accuracy envelope, engine.Geometry).
// BBOX_PARTS blocks per job reduce row ranges in one pass over all three
// axes (partials after the n_jobs final boxes), k_bbox_reduce folds them.
constexpr int BBOX_PARTS = 64;
constexpr int BBOX_WORDS = 16;

__device__ __forceinline__ double block_min(double v, double* red) { return -block_max(-v, red); }

// rows[j] = (source path first row, T, receiver first row, receiver moving).
// Each thread folds its rows (unrolled, independent loads in flight), then
// the 14 running values reduce in one pass: warp shuffles, one shared-memory
// exchange, one barrier.
constexpr int BBOX_THREADS = 256;

__device__ __forceinline__ double red_op(double a, double b, bool lo) { return lo ? fmin(a, b) : fmax(a, b); }

__global__ void __launch_bounds__(BBOX_THREADS) k_path_bbox(const int64_t* __restrict__ rows,
                                                            const double* __restrict__ paths,
                                                            int64_t n_jobs, double* __restrict__ bbox) {
    __shared__ double red[14][BBOX_THREADS / 32];
    const int64_t* R = rows + 4 * blockIdx.y;
    double* part = bbox + BBOX_WORDS * (n_jobs + (int64_t)blockIdx.y * BBOX_PARTS + blockIdx.x);
    double v[14];
#pragma unroll
    for (int which = 0; which < 2; ++which) {
        const double* P = paths + 3 * (which == 0 ? R[0] : R[2]);
        const int64_t n = which == 0 || R[3] ? R[1] : 1;
        double lo0 = DBL_MAX, lo1 = DBL_MAX, lo2 = DBL_MAX, hi0 = -DBL_MAX, hi1 = -DBL_MAX,
               hi2 = -DBL_MAX, step = 0.0;
        const int64_t stride = (int64_t)gridDim.x * blockDim.x;
#pragma unroll 4
        for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += stride) {
            const double x = P[3 * t], y = P[3 * t + 1], z = P[3 * t + 2];
            lo0 = fmin(lo0, x); lo1 = fmin(lo1, y); lo2 = fmin(lo2, z);
            hi0 = fmax(hi0, x); hi1 = fmax(hi1, y); hi2 = fmax(hi2, z);
            if (t + 1 < n) {
                const double dx = P[3 * t + 3] - x, dy = P[3 * t + 4] - y, dz = P[3 * t + 5] - z;
                step = fmax(step, dx * dx + dy * dy + dz * dz);
            }
        }
        v[7 * which + 0] = lo0; v[7 * which + 1] = lo1; v[7 * which + 2] = lo2;
        v[7 * which + 3] = hi0; v[7 * which + 4] = hi1; v[7 * which + 5] = hi2;
        v[7 * which + 6] = step;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < 14; ++q) {
        const bool lo = (q % 7) < 3;
        for (int o = 16; o > 0; o >>= 1) v[q] = red_op(v[q], __shfl_xor_sync(0xffffffffu, v[q], o), lo);
        if (lane == 0) red[q][warp] = v[q];
    }
    __syncthreads();
    if (threadIdx.x < 14) {
        const int q = threadIdx.x;
        const bool lo = (q % 7) < 3;
        double r = red[q][0];
        for (int w = 1; w < BBOX_THREADS / 32; ++w) r = red_op(r, red[q][w], lo);
        // word layout: src lo xyz, src hi xyz, mic lo xyz, mic hi xyz, src step, mic step
        const int which = q / 7, k = q % 7;
        if (k < 6) part[6 * which + k] = r;
        else part[12 + which] = sqrt(r) * (1.0 + 1e-12);
    }
    if (threadIdx.x == 14) part[14] = part[15] = 0.0;
}

// One warp per (job, word): lanes fold the BBOX_PARTS partials, shuffles
// finish the reduction.
__global__ void k_bbox_reduce(int64_t n_jobs, double* __restrict__ bbox) {
    const int64_t j = blockIdx.x;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (j >= n_jobs || w >= BBOX_WORDS) return;
    const double* part = bbox + BBOX_WORDS * (n_jobs + j * BBOX_PARTS);
    const bool lo = w < 12 && (w % 6) < 3;
    double v = part[BBOX_WORDS * lane + w];
    for (int q = lane + 32; q < BBOX_PARTS; q += 32) v = red_op(v, part[BBOX_WORDS * q + w], lo);
    for (int o = 16; o > 0; o >>= 1) v = red_op(v, __shfl_xor_sync(0xffffffffu, v, o), lo);
    if (lane == 0) bbox[BBOX_WORDS * j + w] = v;
}

// Full-rate images: lb = exact distance at the first, middle and last
// sample; ub = largest distance between the image path's bounding box and
// the receiver's (exact box algebra, + 1e-9 m for rounding).  Images whose
// ub can reach the job's largest lb are scanned exactly by k_exact_max.
__global__ void k_bounds_full(const mvb_image* __restrict__ images, const int32_t* __restrict__ sel,
                              int64_t n_full, const mvb_job* __restrict__ jobs,
                              const double* __restrict__ paths, const double* __restrict__ bbox,
                              double* __restrict__ lb, double* __restrict__ ub) {
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= n_full) return;
    const int32_t i = sel[q];
    const mvb_image im = images[i];
    const mvb_job& J = jobs[im.job];
    double best = 0.0;
    const int64_t ts[3] = {0, (J.T - 1) / 2, J.T - 1};
    for (int k = 0; k < 3; ++k)
        best = fmax(best, image_distance(im, paths + 3 * (J.pos_off + ts[k]), mic_row(J, paths, ts[k])));
    const double* b = bbox + BBOX_WORDS * im.job;
    double sq = 0.0;
    for (int a = 0; a < 3; ++a) {
        // image coordinate off + sign * p over p in [lo, hi]
        const double e1 = im.off[a] + (double)im.sign[a] * b[a];
        const double e2 = im.off[a] + (double)im.sign[a] * b[3 + a];
        const double xlo = fmin(e1, e2), xhi = fmax(e1, e2);
        const double g = fmax(fabs(xhi - b[6 + a]), fabs(b[9 + a] - xlo));
        sq += g * g;
    }
    lb[i] = best;
    ub[i] = sqrt(sq) * (1.0 + 1e-12) + 1e-9;
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
    double m = 0.0;
    for (int64_t q = threadIdx.x; q < J.n_img; q += blockDim.x) m = fmax(m, lb[J.img_off + q]);
    m = block_max(m, red);
    int32_t* sc = scratch + MVB_EXACT_LIST_WORDS + J.img_off + j;
    const double LB = m - 1e-9;
    if (j == 0 && threadIdx.x == 0) scratch[0] = 0;  // survivor list of k_exact_scan
    if (threadIdx.x == 0) {
        sc[0] = 0;
        // every lb is attained by its track to ~1e-12 m, so the exact max is
        // >= LB: seeding dmax with LB is exact and lets k_exact_max skip
        // sample chunks whose bound stays below the running maximum
        dmax[j] = LB > 0.0 ? LB : 0.0;
    }
    __syncthreads();
    for (int64_t q = threadIdx.x; q < J.n_img; q += blockDim.x) {
        const int64_t i = J.img_off + q;
        if (ub[i] >= LB) {
            const int slot = atomicAdd(sc, 1);
            sc[1 + slot] = (int32_t)i;
        }
    }
}

// Exact maxima of the candidates over t < T, in chunks of EXACT_CHUNK
// samples, in two kernels.  k_exact_scan: one warp per (candidate, chunk)
// pair, pairs grid-strided over the job's warps (blockIdx.y = job).  A
// decimated candidate's chunk is dropped when the bound of its coarse window
// (max + negsum (max - min), the window covering every 65-tap sum in the
// chunk) cannot exceed the running maximum (dmax only grows, so dropping is
// exact); a surviving chunk is appended to the survivor list in scratch
// (full-rate candidates, and chunks past the list's capacity, are evaluated
// in place).  k_exact_eval then spreads the survivors over the whole GPU,
// one output sample per thread: the 65-tap fp64 upsample of a chunk is the
// expensive part, and there are typically a handful of surviving chunks of
// a single candidate.  List entry: job (16 bits) | slot (24) | chunk (24).
constexpr int EXACT_CHUNK = 2048;
constexpr int EXACT_SUB = 256;  // samples per k_exact_eval block
constexpr int EXACT_LIST_CAP = (MVB_EXACT_LIST_WORDS - 2) / 2;

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// bound of the upsampled track over samples [t0, t1): coarse window max +
// negsum (max - min) + 1e-9 (lane-parallel, warp-uniform result)
__device__ __forceinline__ double window_bound(const double* __restrict__ c, int64_t K,
                                               int64_t N, int64_t t0, int64_t t1, double negsum,
                                               int lane) {
    int64_t k0 = t0 / N - 32, k1 = (t1 - 1) / N + 32;
    k0 = k0 < 0 ? 0 : k0;
    k1 = k1 > K - 1 ? K - 1 : k1;
    double M = -DBL_MAX, m = -DBL_MAX;  // m holds -min
    for (int64_t k = k0 + lane; k <= k1; k += 32) {
        const double v = c[k];
        M = fmax(M, v);
        m = fmax(m, -v);
    }
    M = warp_max(M);
    m = -warp_max(m);
    return M + negsum * (M - m) + 1e-9;
}

__global__ void k_exact_scan(const mvb_image* __restrict__ images, const mvb_job* __restrict__ jobs,
                             const double* __restrict__ coarse, const double* __restrict__ tables,
                             const double* __restrict__ paths, double negsum,
                             int32_t* __restrict__ scratch, double* __restrict__ dmax) {
    const int64_t j = blockIdx.y;
    const mvb_job& J = jobs[j];
    const int32_t* sc = scratch + MVB_EXACT_LIST_WORDS + J.img_off + j;
    const int count = sc[0];
    const int lane = threadIdx.x & 31;
    // sample chunks of the job's path range (its time-shard window's, win_p0/1)
    const int64_t p0 = win_p0(J), p1 = win_p1(J);
    const int64_t c_lo = p0 / EXACT_CHUNK;
    const int64_t n_chunks = (p1 - 1) / EXACT_CHUNK + 1 - c_lo;
    const int64_t pairs = (int64_t)count * n_chunks;
    const int64_t wpb = blockDim.x >> 5;
    volatile double* dm = dmax + j;
    unsigned long long* list = reinterpret_cast<unsigned long long*>(scratch + 2);
    for (int64_t p = blockIdx.x * wpb + (threadIdx.x >> 5); p < pairs; p += gridDim.x * wpb) {
        const int slot = (int)(p / n_chunks);
        const int64_t ch = c_lo + p - (int64_t)slot * n_chunks;
        const mvb_image im = images[sc[1 + slot]];
        const int64_t t0 = ch * EXACT_CHUNK > p0 ? ch * EXACT_CHUNK : p0;
        const int64_t t1 = (ch + 1) * EXACT_CHUNK < p1 ? (ch + 1) * EXACT_CHUNK : p1;
        double best = 0.0;
        if (im.factor == 1) {
            for (int64_t t = t0 + lane; t < t1; t += 32)
                best = fmax(best, image_distance(im, paths + 3 * (J.pos_off + t), mic_row(J, paths, t)));
        } else {
            const double* c = coarse + im.coarse;
            if (window_bound(c, im.n_coarse, im.factor, t0, t1, negsum, lane) < *dm) continue;
            int at = 0;
            if (lane == 0) at = atomicAdd(scratch, 1);
            at = __shfl_sync(0xffffffffu, at, 0);
            if (at < EXACT_LIST_CAP) {
                if (lane == 0)
                    list[at] = ((unsigned long long)j << 48) | ((unsigned long long)slot << 24) |
                               (unsigned long long)ch;
                continue;
            }
            for (int64_t t = t0 + lane; t < t1; t += 32)  // list full: evaluate in place
                best = fmax(best, exact_upsample(c, im.n_coarse, tables + im.table, im.factor, t));
        }
        best = warp_max(best);
        if (lane == 0 && best > 0.0) atomic_max_pos(dmax + j, best);
    }
}

__global__ void __launch_bounds__(EXACT_SUB) k_exact_eval(
    const mvb_image* __restrict__ images, const mvb_job* __restrict__ jobs,
    const double* __restrict__ coarse, const double* __restrict__ tables,
    const int32_t* __restrict__ scratch, double* __restrict__ dmax) {
    __shared__ double red[32];
    const int n = min(scratch[0], EXACT_LIST_CAP);
    const unsigned long long* list = reinterpret_cast<const unsigned long long*>(scratch + 2);
    constexpr int SUBS = EXACT_CHUNK / EXACT_SUB;
    for (int u = blockIdx.x; u < n * SUBS; u += gridDim.x) {
        const unsigned long long e = list[u / SUBS];
        const int64_t j = (int64_t)(e >> 48), slot = (int64_t)((e >> 24) & 0xffffff),
                      ch = (int64_t)(e & 0xffffff);
        const mvb_job& J = jobs[j];
        const int32_t* sc = scratch + MVB_EXACT_LIST_WORDS + J.img_off + j;
        const mvb_image& im = images[sc[1 + slot]];
        const int64_t t = ch * EXACT_CHUNK + (int64_t)(u % SUBS) * EXACT_SUB + threadIdx.x;
        double v = 0.0;
        if (t >= win_p0(J) && t < win_p1(J) && t < (ch + 1) * EXACT_CHUNK)
            v = exact_upsample(coarse + im.coarse, im.n_coarse, tables + im.table, im.factor, t);
        v = block_max(v, red);
        if (threadIdx.x == 0 && v > 0.0) atomic_max_pos(dmax + j, v);
        __syncthreads();  // red is reused by the next unit
    }
}

// Fast-path interval records, by summation by parts.  With the factor's
// (9, 65) refit F (track on interval k: d(u) = sum_p g_p u^p,
// g_p = sum_c F[p][c] w[k + c - 32], w the coarse distances) and
// sum_c F[p][c] = [p == 0]:
//     g_p - [p == 0] w[k] = sum_{j<64} G[p][j] * dw[k - 32 + j],
//     dw[i] = w[i+1] - w[i],   G = partial sums of F's rows.
// dw is formed once per coarse sample in fp64 and rounded to fp32 (|dw| is
// one coarse step of motion, so its rounding error is ~1e-9 m); the 576
// products per interval then run as fp32 FMAs, paired into FFMA2 over
// (g_p, g_p+1).  Measured against the exact 65-tap track (tests) the
// residual error is < 4e-9 m, i.e. < 6e-7 samples of delay at 48 kHz.
// One block per (image, span of BLOCK x KI intervals); KI consecutive
// intervals per thread so each shared-memory load of dw feeds KI x 5 FMA
// instructions.

#ifndef MVB_WIN_COEF_MINB
#define MVB_WIN_COEF_MINB 16
#endif
struct SbpParam {
    float g[64][10];  // G[p][j] stored per tap j: (g0..g8, pad)
};

// skew one word per 32 so the 8-interval thread stride is conflict-free
__device__ __forceinline__ int skew32(int e) { return e + (e >> 5); }

template <int COEF_BLOCK, int COEF_KI>
struct CoefShape {
    static constexpr int SPAN = COEF_BLOCK * COEF_KI;
    // a thread's KI records (3 float4 each) plus one float4 of padding, so
    // the lanes' 16-byte record stores fall in distinct banks
    static constexpr int REC_F4 = 3 * COEF_KI + 1;
    static constexpr int DW = SPAN + 64 + (SPAN + 64) / 32 + 1;
    static constexpr size_t SMEM = sizeof(float4) * REC_F4 * COEF_BLOCK + sizeof(float) * DW;
};

// windowed one-warp CTAs: at most 128 registers so 16 CTAs fit an SM (the
// register file capped them at 12 -- 17% warp occupancy, FMA pipe ~55%)
template <int COEF_BLOCK, int COEF_KI, bool WIN>
__global__ void __launch_bounds__(COEF_BLOCK, (WIN && COEF_BLOCK == 32) ? MVB_WIN_COEF_MINB : 1) k_coeffs(
    const __grid_constant__ SbpParam sp, const mvb_image* __restrict__ images,
    const int32_t* __restrict__ sel, const mvb_job* __restrict__ jobs,
    const double* __restrict__ coarse, mvb_coef32* __restrict__ out) {
    // records of the span are staged here and written out coalesced
    extern __shared__ __align__(16) unsigned char coef_smem[];
    constexpr int COEF_SPAN = CoefShape<COEF_BLOCK, COEF_KI>::SPAN;
    constexpr int REC_F4 = CoefShape<COEF_BLOCK, COEF_KI>::REC_F4;
    float4* srec = reinterpret_cast<float4*>(coef_smem);
    float* dw = reinterpret_cast<float*>(coef_smem + sizeof(float4) * REC_F4 * COEF_BLOCK);
    const mvb_image im = images[sel[blockIdx.x]];
    const mvb_job& J = jobs[im.job];
    const double kappa = J.kappa;
    const double shift = (double)(J.L - J.d0);
    const int64_t K = im.n_coarse;
    const double* c = coarse + im.coarse;
    const int e0 = COEF_KI * threadIdx.x;
    // intervals [k_first, i1) and the coarse samples [lo, hi] that exist:
    // the whole track, or (WIN, time shards) what the job's output window
    // reads (win_p0 / win_p1, win_coarse).  A separate instantiation: the
    // window bounds live across the loop cost ~16 registers (124 -> 140)
    // and 13% of the unwindowed kernel's time (c4)
    int lo = 0, hi = (int)K - 1, i1 = (int)K, k_first = 0;
    if constexpr (WIN) {
        int64_t ck0, ck1;
        win_coarse(J, im.factor, K, ck0, ck1);
        lo = (int)ck0;
        hi = (int)ck1 - 1;
        k_first = (int)(win_p0(J) / im.factor);
        i1 = (int)((win_p1(J) - 1) / im.factor + 1);
    }
    for (int k0 = k_first + (int)blockIdx.y * COEF_SPAN; k0 < i1; k0 += (int)gridDim.y * COEF_SPAN) {
        __syncthreads();
        // coarse samples k0 - 32 .. k0 + COEF_SPAN + 32 (clamped: samples hold)
        // staged once in the record area (free until the epilogue), then
        // dw[i] = c[i + 1] - c[i] in fp64, stored fp32 (skewed)
        double* cw = reinterpret_cast<double*>(srec);
        const int base = k0 - 32;
        for (int t = threadIdx.x; t < COEF_SPAN + 65; t += blockDim.x) {
            int a = base + t;
            a = a < lo ? lo : (a > hi ? hi : a);
            cw[t] = c[a];
        }
        __syncthreads();
        // the anchors c[k] of this thread's intervals, read before the
        // epilogue reuses the staging area (and off the global-load path)
        double anchor[COEF_KI];
#pragma unroll
        for (int q = 0; q < COEF_KI; ++q) anchor[q] = cw[e0 + q + 32 < COEF_SPAN + 65 ? e0 + q + 32 : 0];
        for (int t = threadIdx.x; t < COEF_SPAN + 64; t += blockDim.x)
            dw[skew32(t)] = (float)(cw[t + 1] - cw[t]);
        __syncthreads();
        if (k0 + e0 < i1) {
        static_assert(COEF_KI % 2 == 0, "the g8 accumulators pair adjacent intervals");
        float2 acc[COEF_KI][4];
        float2 acc8[COEF_KI / 2];  // (interval 2h, interval 2h+1) of coefficient 8
#pragma unroll
        for (int q = 0; q < COEF_KI; ++q) {
#pragma unroll
            for (int p = 0; p < 4; ++p) acc[q][p] = make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int h = 0; h < COEF_KI / 2; ++h) acc8[h] = make_float2(0.f, 0.f);
        float x[COEF_KI];
#pragma unroll
        for (int q = 0; q < COEF_KI - 1; ++q) x[q + 1] = dw[skew32(e0 + q)];
#pragma unroll
        for (int j = 0; j < 64; ++j) {
#pragma unroll
            for (int q = 0; q < COEF_KI - 1; ++q) x[q] = x[q + 1];
            x[COEF_KI - 1] = dw[skew32(e0 + j + COEF_KI - 1)];
            const float* g = sp.g[j];
#pragma unroll
            for (int q = 0; q < COEF_KI; ++q) {
                const float2 xx = make_float2(x[q], x[q]);
#pragma unroll
                for (int p = 0; p < 4; ++p)
                    acc[q][p] = __ffma2_rn(make_float2(g[2 * p], g[2 * p + 1]), xx, acc[q][p]);
            }
#pragma unroll
            for (int h = 0; h < COEF_KI / 2; ++h)
                acc8[h] = __ffma2_rn(make_float2(g[8], g[8]), make_float2(x[2 * h], x[2 * h + 1]),
                                     acc8[h]);
        }
#pragma unroll
        for (int q = 0; q < COEF_KI; ++q) {
            const int64_t k = k0 + e0 + q;
            if (k >= i1) break;
            const double g0 = anchor[q] + (double)acc[q][0].x;
            mvb_coef32 r;
            const double base = fma(kappa, g0, shift);
            const double B = floor(base);
            r.B = (int32_t)B;
            r.f = (float)(base - B - 0.5);
            r.d_mid = (float)g0;
            r.pad = 0.f;
            const float kf = (float)kappa;
            r.g[0] = kf * acc[q][0].y;
            r.g[1] = kf * acc[q][1].x;
            r.g[2] = kf * acc[q][1].y;
            r.g[3] = kf * acc[q][2].x;
            r.g[4] = kf * acc[q][2].y;
            r.g[5] = kf * acc[q][3].x;
            r.g[6] = kf * acc[q][3].y;
            r.g[7] = kf * ((q & 1) ? acc8[q >> 1].y : acc8[q >> 1].x);
            const float4* rv = reinterpret_cast<const float4*>(&r);
            float4* dstq = srec + REC_F4 * threadIdx.x + 3 * q;
            dstq[0] = rv[0];
            dstq[1] = rv[1];
            dstq[2] = rv[2];
        }
        }
        __syncthreads();
        // coalesced copy of the span's records (16 B per thread per pass)
        const int64_t n_rec = i1 - k0 < COEF_SPAN ? i1 - k0 : COEF_SPAN;
        const float4* src = srec;
        float4* dst = reinterpret_cast<float4*>(out + im.coef + k0);
        for (int64_t t = threadIdx.x; t < n_rec * 3; t += blockDim.x) {
            const int rec = (int)(t / 3), part = (int)(t - 3 * (t / 3));  // record e = rec
            dst[t] = src[REC_F4 * (rec / COEF_KI) + 3 * (rec % COEF_KI) + part];
        }
    }
}

// images_sorted[q] = images[idx[q]]: 16-byte chunks, six per record
__global__ void k_gather_images(const mvb_image* __restrict__ images, const int64_t* __restrict__ idx,
                                int64_t n, mvb_image* __restrict__ out) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    constexpr int CH = sizeof(mvb_image) / 16;
    if (t >= n * CH) return;
    const int64_t q = t / CH, c = t - q * CH;
    reinterpret_cast<float4*>(out + q)[c] = __ldg(reinterpret_cast<const float4*>(images + idx[q]) + c);
}

// Sort segment s of a windowed job that none of the window's tiles reads
// (a tile reads segment min(n / seg_len, last), n its first sample).
__device__ __forceinline__ bool outside_window(const mvb_job& J, int64_t s, int64_t seg_len) {
    if (J.w0 == 0 && J.w1 <= 0) return false;
    const int64_t last = (J.T + seg_len - 1) / seg_len - 1;
    const int64_t a = J.w0 / seg_len < last ? J.w0 / seg_len : last;
    const int64_t b = J.w1 > 0 && (J.w1 - 1) / seg_len < last ? (J.w1 - 1) / seg_len : last;
    return s < a || s > b;
}

__global__ void k_sort_keys(const mvb_image* __restrict__ images, const mvb_job* __restrict__ jobs,
                            int64_t max_n_img, int64_t max_n_seg, int64_t seg_len,
                            const double* __restrict__ paths, const double* __restrict__ coarse,
                            double* __restrict__ key) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t s = blockIdx.y, j = blockIdx.z;
    const mvb_job& J = jobs[j];
    if (i >= J.n_img || s * seg_len >= J.T || outside_window(J, s, seg_len)) return;
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

// Fused delay sort: one CTA per (segment s, job j).  Key of image i = its
// delay in whole samples at the segment centre, kappa * d (k_sort_keys'
// distance), clamped to key_bits bits -- the host's delay bound fixes the
// bit count, so c3's 57k-sample delays sort in 16 bits (four 4-bit radix
// passes instead of eight for fp32 keys); a stable block radix sort
// (deterministic); the records are gathered in that order, striped so
// consecutive threads write consecutive 96-byte records.  Slots past the
// job's images (padding keys, all ones, sort last: stable, larger indices)
// and segments past its track (all keys padding: identity order) hold
// index min(q, n - 1).
template <int BT, int IPT>
__global__ void __launch_bounds__(BT) k_delay_sort(const mvb_image* __restrict__ images,
                                                   const mvb_job* __restrict__ jobs,
                                                   int64_t max_n_img, int64_t max_n_seg,
                                                   int64_t seg_len, const double* __restrict__ paths,
                                                   const double* __restrict__ coarse, int key_bits,
                                                   int64_t run_len, mvb_image* __restrict__ out,
                                                   unsigned* __restrict__ keys_out) {
    using Sort = cub::BlockRadixSort<unsigned, BT, IPT, int>;
    extern __shared__ __align__(16) unsigned char dsort_smem[];
    auto& temp = *reinterpret_cast<typename Sort::TempStorage*>(dsort_smem);
    const int64_t s = blockIdx.x, j = blockIdx.y;
    const mvb_job& J = jobs[j];
    if (outside_window(J, s, seg_len)) return;  // block-uniform: no tile reads it
    // run blockIdx.z: slots [base, base + run_len) of the job's table, its
    // images [base, base + n) sorted on their own (one run: the whole job)
    const int64_t base = (int64_t)blockIdx.z * run_len;
    if (base >= max_n_img) return;
    const int n = (int)(J.n_img - base < run_len ? (J.n_img > base ? J.n_img - base : 0) : run_len);
    const int slots = (int)(max_n_img - base < run_len ? max_n_img - base : run_len);
    const bool active = s * seg_len < J.T;
    int64_t t = s * seg_len + seg_len / 2;
    if (t > J.T - 1) t = J.T - 1;
    const mvb_image* __restrict__ im0 = images + J.img_off + base;
    const unsigned kmax = key_bits >= 32 ? 0xffffffffu : (1u << key_bits) - 1u;
    const double kappa = J.kappa;
    unsigned keys[IPT];
    int vals[IPT];
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
        const int i = threadIdx.x * IPT + k;  // blocked arrangement
        unsigned key = kmax;
        if (active && i < n) {
            const mvb_image& im = im0[i];
            double d;
            if (im.factor == 1) {
                d = image_distance(im, paths + 3 * (J.pos_off + t), mic_row(J, paths, t));
            } else {
                int64_t c = t / im.factor;
                if (c >= im.n_coarse) c = im.n_coarse - 1;
                d = coarse[im.coarse + c];
            }
            const double tau = d * kappa;
            key = tau < (double)kmax ? (unsigned)tau : kmax;
        }
        keys[k] = key;
        vals[k] = i;
    }
    Sort(temp).SortBlockedToStriped(keys, vals, 0, key_bits);
    mvb_image* __restrict__ dst = out + (j * max_n_seg + s) * max_n_img + base;
    unsigned* __restrict__ kdst = keys_out ? keys_out + (j * max_n_seg + s) * max_n_img + base : nullptr;
    constexpr int CH = sizeof(mvb_image) / 16;
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
        const int q = k * BT + threadIdx.x;  // striped arrangement
        if (q < slots) {
            // the sorted keys (ascending within the run; the synthesis
            // narrows a tile's image range on them, k_synth_f32)
            if (kdst) kdst[q] = keys[k];
            // padding slots (past the job's images) repeat an own image
            const int64_t src = n > 0 ? (vals[k] < n - 1 ? vals[k] : n - 1) : J.n_img - 1 - base;
            const float4* a = reinterpret_cast<const float4*>(im0 + src);
            float4* b = reinterpret_cast<float4*>(dst + q);
#pragma unroll
            for (int c = 0; c < CH; ++c) b[c] = __ldg(a + c);
        }
    }
}

template <int BT, int IPT>
static int launch_delay_sort(const mvb_image* images, const mvb_job* jobs, int64_t n_jobs,
                             int64_t max_n_img, int64_t max_n_seg, int64_t seg_len,
                             const double* paths, const double* coarse, int key_bits,
                             int64_t run_len, mvb_image* out, unsigned* keys, cudaStream_t s) {
    using Sort = cub::BlockRadixSort<unsigned, BT, IPT, int>;
    const size_t smem = sizeof(typename Sort::TempStorage);
    static bool attr = false;  // one opt-in per process and instantiation
    if (!attr) {
        cudaFuncSetAttribute(k_delay_sort<BT, IPT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        attr = true;
    }
    const int64_t runs = (max_n_img + run_len - 1) / run_len;
    prefer_carveout((const void*)k_delay_sort<BT, IPT>);
    k_delay_sort<BT, IPT><<<dim3((unsigned)max_n_seg, (unsigned)n_jobs, (unsigned)runs), BT, smem,
                            s>>>(images, jobs, max_n_img, max_n_seg, seg_len, paths, coarse,
                                 key_bits, run_len, out, keys);
    return MVB_OK;
}

// Coarse path rows: dst[dst_row[q] + k] = src[src_row[q] + k * N], k < K
// (decimate: pos[::N], trajectory.py:279-298), 3 doubles per row.
__global__ void k_decimate_rows(const double* __restrict__ src, const int64_t* __restrict__ rows,
                                int64_t n, int64_t K, int64_t N, double* __restrict__ dst) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n * K * 3) return;
    const int64_t a = t % 3, k = (t / 3) % K, q = t / (3 * K);
    dst[3 * (rows[2 * q + 1] + k) + a] = src[3 * (rows[2 * q] + k * N) + a];
}

// Bandwidth decision helpers (trajectory.py:316-339) ----------------------
// Mean removal of x (G, T, 3) along T (the reference's x - x.mean()), wide:
// chunk sums, then every block of the subtraction folds the chunk sums of
// its path in a fixed order (deterministic, identical in every block).
constexpr int SPEC_PARTS = MVB_SPEC_PARTS;  // blocks per path: enough loads in flight for one path

__device__ __forceinline__ int64_t part_begin(int64_t F, int q) { return (F * q) / SPEC_PARTS; }

__global__ void k_path_sums(const double* __restrict__ x, int64_t T, double* __restrict__ partial) {
    __shared__ double red[3][32];
    const int64_t g = blockIdx.y;
    const int q = blockIdx.x;
    const int64_t t0 = part_begin(T, q), t1 = part_begin(T, q + 1);
    double s[3] = {0.0, 0.0, 0.0};
    for (int64_t t = t0 + threadIdx.x; t < t1; t += blockDim.x)
#pragma unroll
        for (int a = 0; a < 3; ++a) s[a] += x[3 * (g * T + t) + a];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        for (int o = 16; o > 0; o >>= 1) s[a] += __shfl_xor_sync(0xffffffffu, s[a], o);
        if (l == 0) red[a][w] = s[a];
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        double t = 0.0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += red[threadIdx.x][k];
        partial[(g * 3 + threadIdx.x) * SPEC_PARTS + q] = t;
    }
}

// fold of a path's SPEC_PARTS partial sums of axis a (warp a, fixed order:
// lane-strided sums then a shuffle tree)
__device__ __forceinline__ double fold_parts(const double* __restrict__ p, int lane) {
    double t = 0.0;
    for (int q = lane; q < SPEC_PARTS; q += 32) t += p[q];
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    return t;
}

__global__ void k_path_center(const double* __restrict__ x, int64_t T,
                              const double* __restrict__ partial, double* __restrict__ out) {
    __shared__ double mean[3];
    const int64_t g = blockIdx.y;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (w < 3) {
        const double t = fold_parts(partial + (g * 3 + w) * SPEC_PARTS, lane);
        if (lane == 0) mean[w] = t / (double)T;
    }
    __syncthreads();
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < 3 * T;
         e += (int64_t)gridDim.x * blockDim.x)
        out[3 * g * T + e] = x[3 * g * T + e] - mean[e % 3];
}

// Spectra of the centred paths as cuFFT returns them for (G, T, 3)
// transformed along T: spec[(g F + f) 3 + a] (complex).  Row (g, a) power
// |X_f|^2 with |X| = hypot (numpy.abs).
__device__ __forceinline__ double spec_power(const double2* spec, int64_t F, int64_t row, int64_t f) {
    const int64_t g = row / 3, a = row % 3;
    const double2 v = spec[(g * F + f) * 3 + a];
    const double m = hypot(v.x, v.y);
    return m * m;
}

// partial[row][q] = power summed over bins [part_begin(q), part_begin(q+1))
__global__ void k_spec_partial(const double2* __restrict__ spec, int64_t F, double* __restrict__ partial) {
    __shared__ double red[32];
    const int64_t row = blockIdx.y;
    const int q = blockIdx.x;
    const int64_t f0 = part_begin(F, q), f1 = part_begin(F, q + 1);
    double s = 0.0;
    for (int64_t f = f0 + threadIdx.x; f < f1; f += blockDim.x) s += spec_power(spec, F, row, f);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) red[w] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += red[k];
        partial[row * SPEC_PARTS + q] = t;
    }
}

// First bin whose cumulative power reaches fraction x total (-1: all zero):
// prefix of the row's partials locates the part, a block scan of that part
// (tiles of 256 bins) locates the bin.
__global__ void __launch_bounds__(256) k_spec_find(const double2* __restrict__ spec, int64_t F,
                                                   const double* __restrict__ partial,
                                                   double fraction, int64_t* __restrict__ out) {
    __shared__ double wsum[8];
    __shared__ double carry;
    __shared__ int part, found;
    const int64_t row = blockIdx.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double thr = 0.0;
    if (w == 0) {
        // warp 0: lane l holds parts [8l, 8l + 8); an inclusive warp scan of
        // the lane sums gives every part's prefix; the first part whose
        // prefix reaches fraction x total is the one to scan bin by bin
        static_assert(SPEC_PARTS == 256, "8 parts per lane");
        const double* p = partial + row * SPEC_PARTS + 8 * lane;
        double loc[8], sum = 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            loc[k] = p[k];
            sum += loc[k];
        }
        double inc = sum;
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        const double tot = __shfl_sync(0xffffffffu, inc, 31);
        if (lane == 0) {
            part = -1;
            found = 0x7fffffff;
        }
        if (tot > 0.0) {
            thr = fraction * tot;
            // part q is the first with prefix_before(q) + p[q] >= thr (the
            // last part if rounding keeps every prefix below thr)
            double acc = inc - sum;  // exclusive prefix of this lane's parts
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
                part = q >= 0 ? q : SPEC_PARTS - 1;  // rounding: the last part
                wsum[0] = thr;
            }
            if (q >= 0 && lane == 0) carry = a;
            if (q < 0 && lane == 31) carry = inc - loc[7];  // prefix before the last part
        }
    }
    __syncthreads();
    if (part < 0) {
        if (threadIdx.x == 0) out[row] = -1;
        return;
    }
    thr = wsum[0];
    __syncthreads();
    const int64_t f0 = part_begin(F, part), f1 = part_begin(F, part + 1);
    for (int64_t base = f0; base < f1; base += 256) {
        const int64_t f = base + threadIdx.x;
        double v = f < f1 ? spec_power(spec, F, row, f) : 0.0;
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += y;
        }
        if (lane == 31) wsum[w] = v;
        __syncthreads();
        double pre = carry;
        for (int q = 0; q < w; ++q) pre += wsum[q];
        if (f < f1 && pre + v >= thr) atomicMin(&found, (int)(f - base));
        __syncthreads();
        if (found != 0x7fffffff) {
            if (threadIdx.x == 0) out[row] = base + found;
            return;
        }
        if (threadIdx.x == 255) carry = pre + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) out[row] = f1 - 1;  // rounding: the part's end reaches thr
}

}  // namespace mvb

using namespace mvb;

__global__ void k_build_images(const double* __restrict__ toff, const double* __restrict__ tsgn,
                               const double* __restrict__ tbeta, int64_t S0,
                               const int32_t* __restrict__ img, int64_t S,
                               const int64_t* __restrict__ job, int64_t G,
                               const mvb_class_table cls, int64_t img_base,
                               mvb_image* __restrict__ out, int32_t* __restrict__ full_sel,
                               int32_t* __restrict__ dec_sel, int32_t* __restrict__ class_sel) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= G * S) return;
    const int64_t g = t / S, s = t - g * S;
    const int nC = cls.n;
    const int32_t* im = img + s * (2 + nC);
    const int64_t* jb = job + g * (4 + nC);
    const int64_t src = im[0];
    const int c = im[1];
    const int64_t room = jb[0], T = jb[1];
    // coarse index: the job's first + the intervals of its earlier images
    int64_t coarse = jb[3];
    int full_rank = 0, dec_rank = 0;
    for (int q = 0; q < nC; ++q) {
        const int N = cls.factor[q];
        if (N > 1) {
            coarse += (int64_t)im[2 + q] * ((T + N - 1) / N);
            dec_rank += im[2 + q];
        } else {
            full_rank += im[2 + q];
        }
    }
    const int N = cls.factor[c];
    const int64_t r = room * S0 + src;
    mvb_image o;
    o.off[0] = toff[3 * r + 0];
    o.off[1] = toff[3 * r + 1];
    o.off[2] = toff[3 * r + 2];
    o.beta = tbeta[r];
    o.sign[0] = (float)tsgn[3 * r + 0];
    o.sign[1] = (float)tsgn[3 * r + 1];
    o.sign[2] = (float)tsgn[3 * r + 2];
    o.amp_num = (float)(o.beta / (4.0 * 3.141592653589793));
    o.factor = N;
    o.n_coarse = N > 1 ? (int32_t)((T + N - 1) / N) : 0;
    o.coarse = coarse;
    o.coef = coarse;  // one interval record per coarse sample
    o.table = cls.table[c];
    o.cpath = jb[4 + c];
    o.job = (int32_t)jb[2];
    o.fit = cls.fit[c];
    const int64_t gi = img_base + t;
    out[gi] = o;
    if (N > 1) {
        int dec_count = 0;
        for (int q = 0; q < nC; ++q)
            if (cls.factor[q] > 1) dec_count += cls.count[q];
        dec_sel[g * dec_count + dec_rank] = (int32_t)gi;
        class_sel[cls.sel_off[c] + g * cls.count[c] + im[2 + c]] = (int32_t)gi;
    } else {
        full_sel[g * cls.count[c] + full_rank] = (int32_t)gi;
    }
}

template <int BLOCK, int KI, bool WIN>
static int launch_coeffs(const SbpParam& sp, const mvb_image* images, const int32_t* sel,
                         int64_t n_sel, int64_t max_K, const mvb_job* jobs, const double* coarse,
                         mvb_coef32* coef, void* stream, int64_t n_int = 0) {
    using S = CoefShape<BLOCK, KI>;
    // spans per image: the whole track, or (windowed) the window's intervals
    // (the kernel's span loop covers any remainder)
    int64_t spans = ((n_int > 0 ? n_int : max_K) + S::SPAN - 1) / S::SPAN;
    if (spans > 65535) spans = 65535;
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(k_coeffs<BLOCK, KI, WIN>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMEM);
        if (e != cudaSuccess) return fail(MVB_ECUDA, cudaGetErrorString(e));
        attr_set = true;
    }
    prefer_carveout((const void*)k_coeffs<BLOCK, KI, WIN>);
    k_coeffs<BLOCK, KI, WIN><<<dim3((unsigned)n_sel, (unsigned)spans), BLOCK, S::SMEM,
                               as_stream(stream)>>>(sp, images, sel, jobs, coarse, coef);
    return check_launch("track_coeffs");
}

extern "C" {

int mvb_build_images(const double* toff, const double* tsgn, const double* tbeta, int64_t S0,
                     const int32_t* img, int64_t S, const int64_t* job, int64_t G,
                     const mvb_class_table* classes, int64_t img_base, mvb_image* images,
                     int32_t* full_sel, int64_t full_off, int32_t* dec_sel, int64_t dec_off,
                     int32_t* class_sel, void* stream) {
    if (S < 0 || G < 0 || S0 < 1 || !classes || classes->n < 1 || classes->n > MVB_MAX_CLASSES)
        return fail(MVB_EINVAL, "build_images: bad sizes / classes");
    if (S == 0 || G == 0) return MVB_OK;
    if (!toff || !tsgn || !tbeta || !img || !job || !images)
        return fail(MVB_EINVAL, "build_images: null");
    if (img_base + G * S > 0x7fffffff) return fail(MVB_EINVAL, "build_images: > 2^31 images");
    prefer_carveout((const void*)k_build_images);
    k_build_images<<<grid_for(G * S, 256), 256, 0, as_stream(stream)>>>(
        toff, tsgn, tbeta, S0, img, S, job, G, *classes, img_base, images,
        full_sel ? full_sel + full_off : nullptr, dec_sel ? dec_sel + dec_off : nullptr, class_sel);
    return check_launch("build_images");
}

int mvb_coarse_distances(const mvb_image* images, const int32_t* sel, int64_t n_sel,
                         int64_t max_K, const mvb_job* jobs, const double* paths, double negsum,
                         double* coarse, double* lb, double* ub, void* stream) {
    if (n_sel < 0 || n_sel > 0x7fffffff) return fail(MVB_EINVAL, "coarse_distances: n_sel");
    if (n_sel == 0) return MVB_OK;
    if (!images || !sel || !jobs || !paths || !coarse) return fail(MVB_EINVAL, "coarse_distances: null");
    if ((lb == nullptr) != (ub == nullptr)) return fail(MVB_EINVAL, "coarse_distances: lb/ub");
    if (max_K < 1) return fail(MVB_EINVAL, "coarse_distances: max_K");
    // warps walk CB_SEGS-segment chunks serially: launches with few images
    // (image shards) use shorter chunks for more parallel warps (c3 W=8:
    // 50 -> 37 us), large ones the longer chunks (fewer recomputed edges)
    const int64_t chunks16 = ((max_K + 63) / 64 + CB_SEGS - 1) / CB_SEGS;
    if (n_sel * chunks16 < 148 * 64) {
        const int64_t chunks = ((max_K + 63) / 64 + 7) / 8;
        if (chunks > 65535) return fail(MVB_EINVAL, "coarse_distances: coarse track too long");
        prefer_carveout((const void*)k_coarse_bounds<8>);
        k_coarse_bounds<8><<<dim3(grid_for(n_sel, 8), (unsigned)chunks), 256, 0,
                             as_stream(stream)>>>(images, sel, n_sel, jobs, paths, negsum, coarse,
                                                  lb, ub);
        return check_launch("coarse_distances");
    }
    const int64_t chunks = chunks16;
    if (chunks > 65535) return fail(MVB_EINVAL, "coarse_distances: coarse track too long");
    prefer_carveout((const void*)k_coarse_bounds<CB_SEGS>);
    k_coarse_bounds<CB_SEGS><<<dim3(grid_for(n_sel, 8), (unsigned)chunks), 256, 0, as_stream(stream)>>>(
        images, sel, n_sel, jobs, paths, negsum, coarse, lb, ub);
    return check_launch("coarse_distances");
}

int mvb_path_bbox(const int64_t* rows, int64_t n_jobs, const double* paths, double* bbox,
                  void* stream) {
    if (n_jobs < 0 || n_jobs > 65535) return fail(MVB_EINVAL, "path_bbox: n_jobs");
    if (n_jobs == 0) return MVB_OK;
    if (!rows || !paths || !bbox) return fail(MVB_EINVAL, "path_bbox: null");
    cudaStream_t s = as_stream(stream);
    prefer_carveout((const void*)k_path_bbox);
    k_path_bbox<<<dim3(BBOX_PARTS, (unsigned)n_jobs), BBOX_THREADS, 0, s>>>(rows, paths, n_jobs, bbox);
    prefer_carveout((const void*)k_bbox_reduce);
    k_bbox_reduce<<<(unsigned)n_jobs, 32 * BBOX_WORDS, 0, s>>>(n_jobs, bbox);
    return check_launch("path_bbox");
}

int mvb_track_bounds(const mvb_image* images, const int32_t* full_sel, int64_t n_full,
                     const mvb_job* jobs, const double* paths, const double* bbox, double* lb,
                     double* ub, void* stream) {
    if (n_full < 0 || n_full > 0x7fffffff) return fail(MVB_EINVAL, "track_bounds: sizes");
    if (n_full == 0) return MVB_OK;
    if (!images || !full_sel || !jobs || !paths || !bbox || !lb || !ub)
        return fail(MVB_EINVAL, "track_bounds: null");
    prefer_carveout((const void*)k_bounds_full);
    k_bounds_full<<<grid_for(n_full, 128), 128, 0, as_stream(stream)>>>(images, full_sel, n_full, jobs,
                                                                       paths, bbox, lb, ub);
    return check_launch("track_bounds");
}

// out_len of every job from its exact track maximum, as synth.py:211-212:
// len(s) + ceil(rate * dmax / c) + L, written into the job table (the
// kernels mask by it); lengths[j] for the host; err = 1 if a length exceeds
// the capacity the host planned (jobs[j].out_len on entry).
__global__ void k_finalize_lengths(mvb_job* __restrict__ jobs, int64_t n_jobs,
                                   const double* __restrict__ dmax, int64_t* __restrict__ lengths,
                                   int32_t* __restrict__ err) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= n_jobs) return;
    mvb_job& J = jobs[j];
    const int64_t sig_len = J.ls - J.L + 1;
    const int64_t len = sig_len + (int64_t)ceil(J.rate * dmax[j] / J.c) + J.L;
    if (len > J.out_len) atomicExch(err, 1);
    J.out_len = len < J.out_len ? len : J.out_len;
    lengths[j] = len;
}

int mvb_finalize_lengths(mvb_job* jobs, int64_t n_jobs, const double* dmax, int64_t* lengths,
                         int32_t* err, void* stream) {
    if (n_jobs < 0) return fail(MVB_EINVAL, "finalize_lengths: n_jobs");
    if (n_jobs == 0) return MVB_OK;
    if (!jobs || !dmax || !lengths || !err) return fail(MVB_EINVAL, "finalize_lengths: null");
    prefer_carveout((const void*)k_finalize_lengths);
    k_finalize_lengths<<<grid_for(n_jobs, 128), 128, 0, as_stream(stream)>>>(jobs, n_jobs, dmax,
                                                                            lengths, err);
    return check_launch("finalize_lengths");
}

int mvb_gather_images(const mvb_image* images, const int64_t* idx, int64_t n, mvb_image* out,
                      void* stream) {
    if (n < 0) return fail(MVB_EINVAL, "gather_images: n");
    if (n == 0) return MVB_OK;
    if (!images || !idx || !out) return fail(MVB_EINVAL, "gather_images: null");
    const int64_t chunks = n * (int64_t)(sizeof(mvb_image) / 16);
    prefer_carveout((const void*)k_gather_images);
    k_gather_images<<<grid_for(chunks, 256), 256, 0, as_stream(stream)>>>(images, idx, n, out);
    return check_launch("gather_images");
}

int mvb_track_max(const mvb_image* images, const mvb_job* jobs, int64_t n_jobs,
                  const double* coarse, const double* tables, const double* paths, double negsum,
                  const double* lb, const double* ub, int32_t* scratch, double* dmax,
                  void* stream) {
    if (n_jobs < 1 || n_jobs > 65535) return fail(MVB_EINVAL, "track_max: n_jobs");
    if (!images || !jobs || !paths || !lb || !ub || !scratch || !dmax)
        return fail(MVB_EINVAL, "track_max: null");
    cudaStream_t s = as_stream(stream);
    prefer_carveout((const void*)k_select);
    k_select<<<(unsigned)n_jobs, 256, 0, s>>>(images, jobs, lb, ub, scratch, dmax);
    // scan: ~2 blocks of 8 warps per SM for one job, fewer per job for batches
    const unsigned bx = (unsigned)std::max<int64_t>(4, std::min<int64_t>(296, 1184 / n_jobs));
    prefer_carveout((const void*)k_exact_scan);
    k_exact_scan<<<dim3(bx, (unsigned)n_jobs), 256, 0, s>>>(images, jobs, coarse, tables, paths,
                                                           negsum, scratch, dmax);
    prefer_carveout((const void*)k_exact_eval);
    k_exact_eval<<<592, EXACT_SUB, 0, s>>>(images, jobs, coarse, tables, scratch, dmax);
    return check_launch("track_max");
}

static int track_coeffs(const mvb_image* images, const int32_t* sel, int64_t n_sel,
                        int64_t max_K, const mvb_job* jobs, const double* coarse,
                        const double* h_fit, mvb_coef32* coef, bool windowed, void* stream) {
    if (n_sel < 0 || n_sel > 0x7fffffff) return fail(MVB_EINVAL, "track_coeffs: n_sel");
    if (n_sel == 0) return MVB_OK;
    if (!images || !sel || !jobs || !coarse || !h_fit || !coef)
        return fail(MVB_EINVAL, "track_coeffs: null");
    if (max_K < 1 || max_K > 0x7fffffff) return fail(MVB_EINVAL, "track_coeffs: max_K");
    // summation-by-parts weights G[p][j] = sum_{c>j} F[p][c] (j >= 32) or
    // -sum_{c<=j} F[p][c] (j < 32), formed in fp64, stored fp32 per tap
    SbpParam sp;
    for (int j = 0; j < 64; ++j) {
        for (int p = 0; p < 9; ++p) {
            double acc = 0.0;
            if (j >= 32)
                for (int cc = j + 1; cc < 65; ++cc) acc += h_fit[p * 65 + cc];
            else
                for (int cc = 0; cc <= j; ++cc) acc -= h_fit[p * 65 + cc];
            sp.g[j][p] = (float)acc;
        }
        sp.g[j][9] = 0.f;
    }
    // 64 threads x 8 intervals: measured best of {64,128,256} x {4,8} on c3/c4
    // (more resident blocks hide the staging prologue; 70% of the FFMA peak on c4).
    // Time-shard windows (~250 intervals of a N = 256 image at W = 8) would
    // leave half of a 512-interval span idle: one warp x 8 there.
    if (windowed) {
        // a window's intervals (max_K less the 2 x 34 halo and the 64 of
        // alignment, coarse_span) in the span that wastes the fewest thread
        // slots: 128 (1 warp x 4), 256 (1 warp x 8) or 512 (2 warps x 8)
        // intervals per CTA pass (ties: the larger span).  c3 at W = 8: the
        // N = 256 tier's ~310 intervals run as 3 x 128, not 2 x 256
        const int64_t n_int = max_K - 64 - 66 > 1 ? max_K - 64 - 66 : 1;
        const int64_t w128 = (n_int + 127) / 128 * 128, w256 = (n_int + 255) / 256 * 256,
                      w512 = (n_int + 511) / 512 * 512;
        if (w512 <= w256 && w512 <= w128)
            return launch_coeffs<64, 8, true>(sp, images, sel, n_sel, max_K, jobs, coarse, coef,
                                              stream, n_int);
        if (w256 <= w128)
            return launch_coeffs<32, 8, true>(sp, images, sel, n_sel, max_K, jobs, coarse, coef,
                                              stream, n_int);
        return launch_coeffs<32, 4, true>(sp, images, sel, n_sel, max_K, jobs, coarse, coef,
                                          stream, n_int);
    }
    return launch_coeffs<64, 8, false>(sp, images, sel, n_sel, max_K, jobs, coarse, coef, stream);
}

int mvb_track_coeffs(const mvb_image* images, const int32_t* sel, int64_t n_sel,
                     int64_t max_K, const mvb_job* jobs, const double* coarse,
                     const double* h_fit, mvb_coef32* coef, void* stream) {
    return track_coeffs(images, sel, n_sel, max_K, jobs, coarse, h_fit, coef, false, stream);
}

int mvb_track_coeffs_windowed(const mvb_image* images, const int32_t* sel, int64_t n_sel,
                              int64_t max_K, const mvb_job* jobs, const double* coarse,
                              const double* h_fit, mvb_coef32* coef, void* stream) {
    return track_coeffs(images, sel, n_sel, max_K, jobs, coarse, h_fit, coef, true, stream);
}

static int delay_sort_runs(const mvb_image* images, const mvb_job* jobs, int64_t n_jobs,
                           int64_t max_n_img, int64_t max_n_seg, int64_t seg_len,
                           const double* paths, const double* coarse, int64_t key_bits,
                           int64_t run_len, mvb_image* out, unsigned* keys, void* stream) {
    if (n_jobs < 0 || n_jobs > 65535 || max_n_img < 0 || max_n_seg < 0 ||
        max_n_seg > 0x7fffffff || seg_len < 1)
        return fail(MVB_EINVAL, "delay_sort: sizes");
    if (run_len < 1 || run_len > MVB_DELAY_SORT_MAX)
        return fail(MVB_EINVAL, "delay_sort: too many images per run");
    if ((max_n_img + run_len - 1) / run_len > 65535) return fail(MVB_EINVAL, "delay_sort: runs");
    if (key_bits < 1 || key_bits > 32) return fail(MVB_EINVAL, "delay_sort: key_bits");
    if (n_jobs == 0 || max_n_img == 0 || max_n_seg == 0) return MVB_OK;
    if (!images || !jobs || !paths || !out) return fail(MVB_EINVAL, "delay_sort: null");
    cudaStream_t s = as_stream(stream);
    const int kb = (int)key_bits;
    int rc;
    if (run_len <= 1024)
        rc = launch_delay_sort<256, 4>(images, jobs, n_jobs, max_n_img, max_n_seg, seg_len, paths,
                                       coarse, kb, run_len, out, keys, s);
    else if (run_len <= 2048)
        rc = launch_delay_sort<256, 8>(images, jobs, n_jobs, max_n_img, max_n_seg, seg_len, paths,
                                       coarse, kb, run_len, out, keys, s);
    else if (run_len <= 4096)
        rc = launch_delay_sort<512, 8>(images, jobs, n_jobs, max_n_img, max_n_seg, seg_len, paths,
                                       coarse, kb, run_len, out, keys, s);
    else if (run_len <= 8192)
        rc = launch_delay_sort<1024, 8>(images, jobs, n_jobs, max_n_img, max_n_seg, seg_len,
                                        paths, coarse, kb, run_len, out, keys, s);
    else
        rc = launch_delay_sort<1024, 16>(images, jobs, n_jobs, max_n_img, max_n_seg, seg_len,
                                         paths, coarse, kb, run_len, out, keys, s);
    if (rc != MVB_OK) return rc;
    return check_launch("delay_sort");
}

int mvb_delay_sort(const mvb_image* images, const mvb_job* jobs, int64_t n_jobs,
                   int64_t max_n_img, int64_t max_n_seg, int64_t seg_len, const double* paths,
                   const double* coarse, int64_t key_bits, mvb_image* out, void* stream) {
    if (max_n_img > MVB_DELAY_SORT_MAX) return fail(MVB_EINVAL, "delay_sort: too many images");
    return delay_sort_runs(images, jobs, n_jobs, max_n_img, max_n_seg, seg_len, paths, coarse,
                           key_bits, max_n_img > 0 ? max_n_img : 1, out, nullptr, stream);
}

int mvb_delay_sort_runs(const mvb_image* images, const mvb_job* jobs, int64_t n_jobs,
                        int64_t max_n_img, int64_t max_n_seg, int64_t seg_len,
                        const double* paths, const double* coarse, int64_t key_bits,
                        int64_t run_len, mvb_image* out, void* stream) {
    return delay_sort_runs(images, jobs, n_jobs, max_n_img, max_n_seg, seg_len, paths, coarse,
                           key_bits, run_len, out, nullptr, stream);
}

int mvb_delay_sort_keyed(const mvb_image* images, const mvb_job* jobs, int64_t n_jobs,
                         int64_t max_n_img, int64_t max_n_seg, int64_t seg_len,
                         const double* paths, const double* coarse, int64_t key_bits,
                         int64_t run_len, mvb_image* out, uint32_t* keys, void* stream) {
    if (!keys) return fail(MVB_EINVAL, "delay_sort_keyed: null keys");
    if (run_len <= 0) {
        if (max_n_img > MVB_DELAY_SORT_MAX) return fail(MVB_EINVAL, "delay_sort: too many images");
        run_len = max_n_img > 0 ? max_n_img : 1;
    }
    return delay_sort_runs(images, jobs, n_jobs, max_n_img, max_n_seg, seg_len, paths, coarse,
                           key_bits, run_len, out, keys, stream);
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
    prefer_carveout((const void*)k_sort_keys);
    k_sort_keys<<<g, 256, 0, as_stream(stream)>>>(images, jobs, max_n_img, max_n_seg, seg_len, paths,
                                                  coarse, key);
    return check_launch("sort_keys");
}

}  // extern "C"

// ---------------------------------------------------------------------------
// decimation decision (trajectory.py:316-339 bandwidth_estimate): per power
// spectrum row, the first index whose cumulative energy reaches `fraction`
// of the row total (searchsorted-left on cumsum/total), -1 for an empty row.
// One block per row: block reduction for the total, then a chunked block scan
// that stops at the first crossing.

namespace mvb {

__global__ void __launch_bounds__(256) k_energy_index(const double* __restrict__ pw, int64_t F,
                                                      double fraction, int64_t* __restrict__ out) {
    __shared__ double wsum[8];
    __shared__ double carry_s;
    __shared__ int found_s;
    const double* p = pw + (int64_t)blockIdx.x * F;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double s = 0.0;
    for (int64_t f = threadIdx.x; f < F; f += 256) s += p[f];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) wsum[w] = s;
    __syncthreads();
    double tot = 0.0;
    for (int q = 0; q < 8; ++q) tot += wsum[q];
    if (!(tot > 0.0)) {
        if (threadIdx.x == 0) out[blockIdx.x] = -1;
        return;
    }
    const double thr = fraction * tot;
    if (threadIdx.x == 0) { carry_s = 0.0; found_s = 0x7fffffff; }
    __syncthreads();
    for (int64_t base = 0; base < F; base += 256) {
        const int64_t f = base + threadIdx.x;
        double v = f < F ? p[f] : 0.0;
        // inclusive warp scan, then across warps
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += y;
        }
        __syncthreads();
        if (lane == 31) wsum[w] = v;
        __syncthreads();
        double pre = carry_s;
        for (int q = 0; q < w; ++q) pre += wsum[q];
        const double cum = pre + v;
        if (f < F && cum >= thr) atomicMin(&found_s, (int)(f - base));
        __syncthreads();
        if (found_s != 0x7fffffff) {
            if (threadIdx.x == 0) out[blockIdx.x] = base + found_s;
            return;
        }
        if (threadIdx.x == 255) carry_s = cum;
        __syncthreads();
    }
    if (threadIdx.x == 0) out[blockIdx.x] = F - 1;
}

}  // namespace mvb

extern "C" int mvb_decimate_rows(const double* src, const int64_t* rows, int64_t n, int64_t K,
                                 int64_t N, double* dst, void* stream) {
    using namespace mvb;
    if (n < 0 || K < 0 || N < 1) return fail(MVB_EINVAL, "decimate_rows: sizes");
    if (n == 0 || K == 0) return MVB_OK;
    if (!src || !rows || !dst) return fail(MVB_EINVAL, "decimate_rows: null");
    prefer_carveout((const void*)k_decimate_rows);
    k_decimate_rows<<<grid_for(n * K * 3, 256), 256, 0, as_stream(stream)>>>(src, rows, n, K, N, dst);
    return check_launch("decimate_rows");
}

extern "C" int mvb_center_paths(const double* x, int64_t G, int64_t T, double* scratch,
                                double* out, void* stream) {
    using namespace mvb;
    if (G < 0 || G > 65535 || T < 1) return fail(MVB_EINVAL, "center_paths: sizes");
    if (G == 0) return MVB_OK;
    if (!x || !scratch || !out) return fail(MVB_EINVAL, "center_paths: null");
    cudaStream_t s = as_stream(stream);
    prefer_carveout((const void*)k_path_sums);
    k_path_sums<<<dim3(SPEC_PARTS, (unsigned)G), 256, 0, s>>>(x, T, scratch);
    unsigned bx = grid_for(3 * T, 256);
    if (bx > 256) bx = 256;
    prefer_carveout((const void*)k_path_center);
    k_path_center<<<dim3(bx, (unsigned)G), 256, 0, s>>>(x, T, scratch, out);
    return check_launch("center_paths");
}

extern "C" int mvb_spectrum_index(const double* spec, int64_t G, int64_t F, double fraction,
                                  double* scratch, int64_t* out, void* stream) {
    using namespace mvb;
    if (G < 0 || G > 0x7fffffff / 3 || F < 1 || !(fraction > 0.0 && fraction < 1.0))
        return fail(MVB_EINVAL, "spectrum_index: args");
    if (G == 0) return MVB_OK;
    if (!spec || !scratch || !out) return fail(MVB_EINVAL, "spectrum_index: null");
    if (3 * G > 65535) return fail(MVB_EINVAL, "spectrum_index: too many paths per call");
    cudaStream_t s = as_stream(stream);
    const double2* sp = reinterpret_cast<const double2*>(spec);
    prefer_carveout((const void*)k_spec_partial);
    k_spec_partial<<<dim3(SPEC_PARTS, (unsigned)(3 * G)), 256, 0, s>>>(sp, F, scratch);
    prefer_carveout((const void*)k_spec_find);
    k_spec_find<<<(unsigned)(3 * G), 256, 0, s>>>(sp, F, scratch, fraction, out);
    return check_launch("spectrum_index");
}

extern "C" int mvb_energy_index(const double* pw, int64_t rows, int64_t F, double fraction,
                                int64_t* out, void* stream) {
    using namespace mvb;
    if (rows < 0 || rows > 0x7fffffff || F < 1 || !(fraction > 0.0 && fraction < 1.0))
        return fail(MVB_EINVAL, "energy_index: args");
    if (rows == 0) return MVB_OK;
    if (!pw || !out) return fail(MVB_EINVAL, "energy_index: null");
    prefer_carveout((const void*)k_energy_index);
    k_energy_index<<<(unsigned)rows, 256, 0, as_stream(stream)>>>(pw, F, fraction, out);
    return check_launch("energy_index");
}
