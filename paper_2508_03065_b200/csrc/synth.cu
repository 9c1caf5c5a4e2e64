// Fractional-delay synthesis (synth.py:194-258 + _kernels.py:90-136).
//
// Fast path (fp32 I/O, the B200 roofline path)
//   k_branch_records_f32  v'_k = x (*) c'_k for the centred Farrow bank,
//                         stored interleaved: one 32-byte record (8 floats)
//                         per input sample, zero-padded on both sides so the
//                         gather needs no bounds test (the reference's
//                         `valid` window reads zeros outside [0, ls)).
//   k_synth_f32           one CTA per (job, 32*U-sample tile, image chunk);
//                         8 warps walk the chunk's delay-sorted images, lane
//                         l of a warp owns samples n0 + 32u + l, u < U.  Per
//                         update: the interval polynomial of the track (fp32
//                         around an fp64 anchor), the (D, mu) split, one
//                         2x16-byte coalesced record gather (L1), Horner in
//                         mu - 1/2, gain 1/(4 pi d) and one FMA into a register
//                         accumulator.  Warps are reduced in fixed order in
//                         shared memory, then written coalesced.
//   k_reduce_f32          fixed-order sum of chunk partials.
//
// Exact path (fp64): k_synth_f64 repeats the reference arithmetic for every
// (image, sample) -- 65-tap upsampled or per-sample distances, tau =
// (rate*d)/c, gain, floor split, Horner in mu -- and its summation order:
// 32-image blocks in canonical order, then the pairwise block tree
// (synth.py:182-191) evaluated with an equivalent merge stack.
#include "mvb_common.cuh"

namespace mvb {

// ---------------------------------------------------------------------------
// branch records

template <int NB>
__global__ void k_branch_records_f32(const float* __restrict__ x, int64_t T,
                                     const double* __restrict__ cb, int M1, int L, int64_t pad,
                                     float* __restrict__ rec) {
    extern __shared__ float sx[];  // [blockDim.x + L - 1]
    __shared__ float sc[NB * 128];
    const int64_t m0 = (int64_t)blockIdx.x * blockDim.x;
    for (int t = threadIdx.x; t < NB * L && t < NB * 128; t += blockDim.x) {
        int k = t / L, j = t - (t / L) * L;
        sc[k * L + j] = k < M1 ? (float)cb[k * L + j] : 0.f;
    }
    for (int t = threadIdx.x; t < (int)blockDim.x + L - 1; t += blockDim.x) {
        int64_t q = m0 - (L - 1) + t;
        sx[t] = (q >= 0 && q < T) ? x[q] : 0.f;
    }
    __syncthreads();
    const int64_t m = m0 + threadIdx.x;
    if (m >= T + L - 1) return;
    float acc[NB];
#pragma unroll
    for (int k = 0; k < NB; ++k) acc[k] = 0.f;
    // v_k[m] = sum_j c_k[j] x[m - j]; sx[threadIdx.x + L-1 - j] = x[m - j]
    for (int j = 0; j < L; ++j) {
        float xv = sx[threadIdx.x + L - 1 - j];
#pragma unroll
        for (int k = 0; k < NB; ++k) acc[k] = fmaf(sc[k * L + j], xv, acc[k]);
    }
    float4* o = reinterpret_cast<float4*>(rec + (pad + m) * NB);
#pragma unroll
    for (int q = 0; q < NB / 4; ++q) o[q] = make_float4(acc[4 * q], acc[4 * q + 1], acc[4 * q + 2], acc[4 * q + 3]);
}

// ---------------------------------------------------------------------------
// fast synthesis

template <int NB>
__device__ __forceinline__ float gather_horner(const float4* __restrict__ R, int64_t idx, float mc) {
    const float4* p = R + idx * (NB / 4);
    float h;
    if constexpr (NB == 4) {
        float4 a = __ldg(p);
        h = fmaf(fmaf(fmaf(a.w, mc, a.z), mc, a.y), mc, a.x);
    } else if constexpr (NB == 8) {
        float4 a = __ldg(p), b = __ldg(p + 1);
        h = b.w;
        h = fmaf(h, mc, b.z);
        h = fmaf(h, mc, b.y);
        h = fmaf(h, mc, b.x);
        h = fmaf(h, mc, a.w);
        h = fmaf(h, mc, a.z);
        h = fmaf(h, mc, a.y);
        h = fmaf(h, mc, a.x);
    } else {
        float v[NB];
#pragma unroll
        for (int q = 0; q < NB / 4; ++q) {
            float4 a = __ldg(p + q);
            v[4 * q] = a.x; v[4 * q + 1] = a.y; v[4 * q + 2] = a.z; v[4 * q + 3] = a.w;
        }
        h = v[NB - 1];
#pragma unroll
        for (int k = NB - 2; k >= 0; --k) h = fmaf(h, mc, v[k]);
    }
    return h;
}

constexpr int SYNTH_WARPS = 8;
#ifndef SYNTH_U
#define SYNTH_U 32
#endif
#ifndef SYNTH_MINB
#define SYNTH_MINB 2
#endif

template <int U, int NB, int MINB>
__global__ void __launch_bounds__(SYNTH_WARPS * 32, MINB) k_synth_f32(
    const mvb_job* __restrict__ jobs, const mvb_work* __restrict__ work,
    const mvb_image* __restrict__ images, const mvb_coef32* __restrict__ coef,
    const float* __restrict__ rec, const double* __restrict__ paths, float* __restrict__ out,
    float* __restrict__ part) {
    constexpr int TN = 32 * U;
    __shared__ float red[SYNTH_WARPS][TN];
    const mvb_work* wp = work + blockIdx.x;
    const int img_begin = wp->img_begin, img_end = wp->img_end;
    const mvb_job* Jp = jobs + wp->job;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t n0 = (int64_t)wp->tile * TN;
    const int T = Jp->T;
    const int Lsh = Jp->L;
    const float4* __restrict__ R = reinterpret_cast<const float4*>(rec) + Jp->rec_base * (NB / 4);
    const mvb_image* __restrict__ imgs = images + Jp->img_off;
    float* __restrict__ row = red[warp];
#pragma unroll
    for (int u = 0; u < U; ++u) row[32 * u + lane] = 0.f;
    float acc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) acc[u] = 0.f;

    for (int i = img_begin + warp; i < img_end; i += SYNTH_WARPS) {
        const mvb_image* ip = imgs + i;
        const int N = ip->factor;
        const float an = ip->amp_num;
        if (N == 1) {
            // near images (full-rate tier): exact fp64 distance per sample,
            // accumulated in the warp's own shared-memory row
            const double kappa = Jp->kappa;
            const double sL = (double)(Lsh - Jp->d0);
            const float dmin = (float)Jp->d_min;
            const double ox = ip->off[0], oy = ip->off[1], oz = ip->off[2];
            const double sx = ip->sign[0], sy = ip->sign[1], sz = ip->sign[2];
            const double* P = paths + 3 * Jp->pos_off;
            const int moving = Jp->mic_moving;
            const double* Q = paths + 3 * Jp->mic_off;
#pragma unroll 1
            for (int u = 0; u < U; ++u) {
                const int64_t n = n0 + 32 * u + lane;
                const int64_t m = n < T ? n : T - 1;
                const double* p = P + 3 * m;
                const double* q = moving ? Q + 3 * m : Q;
                double dx = ox + sx * p[0] - q[0];
                double dy = oy + sy * p[1] - q[1];
                double dz = oz + sz * p[2] - q[2];
                double d = sqrt(dx * dx + dy * dy + dz * dz);
                double s = fma(d, kappa, sL);
                double D = floor(s);
                float mc = (float)(s - D) - 0.5f;
                int64_t idx = n + Lsh - (int64_t)D;
                float A = __fdividef(an, fmaxf((float)d, dmin));
                row[32 * u + lane] = fmaf(A, gather_horner<NB>(R, idx, mc), row[32 * u + lane]);
            }
        } else {
            const mvb_coef32* __restrict__ cf = coef + ip->coef;
            const float twoInvN = 2.0f / (float)N;
            const float invk = (float)(1.0 / Jp->kappa);
            const float dmin = (float)Jp->d_min;
            // (k, r) of each lane's first sample, then advanced by 32 per step
            const int mfirst = (int)(n0 + lane < T ? n0 + lane : T - 1);
            int k = mfirst / N;
            int r = mfirst - k * N;
            const int kT = (T - 1) / N, rT = (T - 1) - kT * N;
            int kc = -1;
            int B = 0;
            float f = 0.f, dm = 0.f, g0 = 0.f, g1 = 0.f, g2 = 0.f, g3 = 0.f, g4 = 0.f, g5 = 0.f,
                  g6 = 0.f, g7 = 0.f;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t n = n0 + 32 * u + lane;
                if (u > 0) {
                    if (n < T) {
                        r += 32;
                        while (r >= N) { r -= N; ++k; }
                    } else {
                        k = kT;
                        r = rT;
                    }
                }
                if (k != kc) {
                    const float4* c4 = reinterpret_cast<const float4*>(cf + k);
                    float4 h0 = __ldg(c4), h1 = __ldg(c4 + 1), h2 = __ldg(c4 + 2);
                    B = __float_as_int(h0.x);
                    f = h0.y; dm = h0.z;
                    g0 = h1.x; g1 = h1.y; g2 = h1.z; g3 = h1.w;
                    g4 = h2.x; g5 = h2.y; g6 = h2.z; g7 = h2.w;
                    kc = k;
                }
                const float uu = fmaf((float)r, twoInvN, -1.f);
                float t = g7;
                t = fmaf(t, uu, g6);
                t = fmaf(t, uu, g5);
                t = fmaf(t, uu, g4);
                t = fmaf(t, uu, g3);
                t = fmaf(t, uu, g2);
                t = fmaf(t, uu, g1);
                t = fmaf(t, uu, g0);
                const float res = t * uu;  // kappa * (d - g0)
                t = f + res;
                const float rt = rintf(t);
                const float mc = t - rt;
                const int idx = (int)n + Lsh - B - (int)rt;
                const float d = fmaf(res, invk, dm);
                const float A = __fdividef(an, fmaxf(d, dmin));
                acc[u] = fmaf(A, gather_horner<NB>(R, idx, mc), acc[u]);
            }
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) row[32 * u + lane] += acc[u];
    __syncthreads();
    const int64_t out_len = Jp->out_len;
    const int n_chunks = Jp->n_chunks;
    float* dst = n_chunks == 1 ? out + Jp->out_off : part + Jp->part_off + (int64_t)wp->chunk * out_len;
    for (int t = threadIdx.x; t < TN; t += blockDim.x) {
        float s = red[0][t];
#pragma unroll
        for (int q = 1; q < SYNTH_WARPS; ++q) s += red[q][t];
        const int64_t n = n0 + t;
        if (n < out_len) dst[n] = s;
    }
}

__global__ void k_reduce_f32(const mvb_job* __restrict__ jobs, const float* __restrict__ part,
                             float* __restrict__ out) {
    const mvb_job J = jobs[blockIdx.y];
    if (J.n_chunks <= 1) return;
    for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < J.out_len;
         n += (int64_t)gridDim.x * blockDim.x) {
        const float* p = part + J.part_off + n;
        float s = p[0];
        for (int c = 1; c < J.n_chunks; ++c) s += p[(int64_t)c * J.out_len];
        out[J.out_off + n] = s;
    }
}

// ---------------------------------------------------------------------------
// exact synthesis

__global__ void __launch_bounds__(128) k_synth_f64(
    const mvb_job* __restrict__ jobs, const mvb_image* __restrict__ images,
    const double* __restrict__ coarse, const double* __restrict__ tables,
    const double* __restrict__ streams, const double* __restrict__ paths,
    double* __restrict__ out) {
    const mvb_job J = jobs[blockIdx.y];
    const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (n >= J.out_len) return;
    const int64_t m = n < J.T ? n : J.T - 1;
    const double* p = paths + 3 * (J.pos_off + m);
    const double* q = paths + 3 * (J.mic_off + (J.mic_moving ? m : 0));
    const double P[3] = {p[0], p[1], p[2]};
    const double Q[3] = {q[0], q[1], q[2]};
    const double* V = streams + J.rec_base;
    const double L = (double)J.L, d0 = (double)J.d0;
    const double four_pi = 4.0 * 3.141592653589793;  // 4.0 * np.pi
    // pairwise merge stack (equivalent to synth.py:182-191, see tests)
    double st_v[40];
    int st_l[40];
    int sp = 0;
    for (int64_t b0 = 0; b0 < J.n_img; b0 += 32) {
        const int64_t b1 = b0 + 32 < J.n_img ? b0 + 32 : J.n_img;
        double s = 0.0;
        for (int64_t i = b0; i < b1; ++i) {
            const mvb_image im = images[J.img_off + i];
            double d;
            if (im.factor == 1)
                d = exact_distance(im.off[0], im.off[1], im.off[2], (double)im.sign[0],
                                   (double)im.sign[1], (double)im.sign[2], P, Q);
            else
                d = exact_upsample(coarse + im.coarse, im.n_coarse, tables + im.table, im.factor, m);
            const double tau = xdiv(xmul(J.rate, d), J.c);
            const double amp = xdiv(im.beta, xmul(four_pi, d > J.d_min ? d : J.d_min));
            const double shifted = xadd(tau, L);
            const double d_int = floor(xsub(shifted, d0));
            const double mu = xsub(xsub(shifted, d0), d_int);
            const int64_t idx = n + J.L - (int64_t)d_int;
            if (idx >= 0 && idx < J.ls) {
                double acc = V[(int64_t)(J.nb - 1) * J.ls + idx];
                for (int k = J.nb - 2; k >= 0; --k) acc = xadd(xmul(acc, mu), V[(int64_t)k * J.ls + idx]);
                s = xadd(s, xmul(amp, acc));
            }
        }
        double v = s;
        int l = 0;
        while (sp > 0 && st_l[sp - 1] == l) {
            v = xadd(st_v[--sp], v);
            ++l;
        }
        st_v[sp] = v;
        st_l[sp++] = l;
    }
    double v = sp > 0 ? st_v[--sp] : 0.0;
    while (sp > 0) v = xadd(st_v[--sp], v);
    out[J.out_off + n] = v;
}

}  // namespace mvb

using namespace mvb;

extern "C" {

int mvb_branch_records_f32(const float* x, int64_t T, const double* cb, int M1, int L, int nb,
                           int64_t pad, float* rec, void* stream) {
    if (T < 1 || L < 1 || M1 < 1 || M1 > nb || pad < 0) return fail(MVB_EINVAL, "branch_records: sizes");
    if (!x || !cb || !rec) return fail(MVB_EINVAL, "branch_records: null");
    if (nb * L > nb * 128) return fail(MVB_EINVAL, "branch_records: L > 128");
    const int block = 256;
    size_t smem = sizeof(float) * (block + L - 1);
    unsigned g = grid_for(T + L - 1, block);
    cudaStream_t s = as_stream(stream);
    switch (nb) {
        case 4: k_branch_records_f32<4><<<g, block, smem, s>>>(x, T, cb, M1, L, pad, rec); break;
        case 8: k_branch_records_f32<8><<<g, block, smem, s>>>(x, T, cb, M1, L, pad, rec); break;
        case 12: k_branch_records_f32<12><<<g, block, smem, s>>>(x, T, cb, M1, L, pad, rec); break;
        case 16: k_branch_records_f32<16><<<g, block, smem, s>>>(x, T, cb, M1, L, pad, rec); break;
        default: return fail(MVB_EINVAL, "branch_records: nb must be 4, 8, 12 or 16");
    }
    return check_launch("branch_records_f32");
}

int mvb_synthesize_f32(const mvb_job* jobs, const mvb_work* work, int64_t n_work,
                       const mvb_image* images, const mvb_coef32* coef, const float* rec,
                       const double* paths, float* out, float* part, int nb, void* stream) {
    if (n_work < 0 || n_work > 0x7fffffff) return fail(MVB_EINVAL, "synthesize_f32: n_work");
    if (n_work == 0) return MVB_OK;
    if (!jobs || !work || !images || !rec || !paths || !out)
        return fail(MVB_EINVAL, "synthesize_f32: null");
    cudaStream_t s = as_stream(stream);
    const unsigned g = (unsigned)n_work;
    const int block = SYNTH_WARPS * 32;
    switch (nb) {
        case 4: k_synth_f32<SYNTH_U, 4, SYNTH_MINB><<<g, block, 0, s>>>(jobs, work, images, coef, rec, paths, out, part); break;
        case 8: k_synth_f32<SYNTH_U, 8, SYNTH_MINB><<<g, block, 0, s>>>(jobs, work, images, coef, rec, paths, out, part); break;
        case 12: k_synth_f32<SYNTH_U, 12, SYNTH_MINB><<<g, block, 0, s>>>(jobs, work, images, coef, rec, paths, out, part); break;
        case 16: k_synth_f32<SYNTH_U, 16, SYNTH_MINB><<<g, block, 0, s>>>(jobs, work, images, coef, rec, paths, out, part); break;
        default: return fail(MVB_EINVAL, "synthesize_f32: nb must be 4, 8, 12 or 16");
    }
    return check_launch("synthesize_f32");
}

int mvb_reduce_partials_f32(const mvb_job* jobs, int64_t n_jobs, int64_t max_out_len,
                            const float* part, float* out, void* stream) {
    if (n_jobs < 0 || n_jobs > 65535 || max_out_len < 0) return fail(MVB_EINVAL, "reduce: sizes");
    if (n_jobs == 0 || max_out_len == 0) return MVB_OK;
    unsigned gx = grid_for(max_out_len, 256);
    if (gx > 1024) gx = 1024;
    k_reduce_f32<<<dim3(gx, (unsigned)n_jobs), 256, 0, as_stream(stream)>>>(jobs, part, out);
    return check_launch("reduce_partials_f32");
}

int mvb_synthesize_f64(const mvb_job* jobs, int64_t n_jobs, int64_t max_out_len,
                       const mvb_image* images, const double* coarse, const double* tables,
                       const double* streams, const double* paths, double* out, void* stream) {
    if (n_jobs < 0 || n_jobs > 65535 || max_out_len < 0) return fail(MVB_EINVAL, "synthesize_f64: sizes");
    if (n_jobs == 0 || max_out_len == 0) return MVB_OK;
    if (!jobs || !images || !streams || !paths || !out)
        return fail(MVB_EINVAL, "synthesize_f64: null");
    dim3 g(grid_for(max_out_len, 128), (unsigned)n_jobs);
    k_synth_f64<<<g, 128, 0, as_stream(stream)>>>(jobs, images, coarse, tables, streams, paths, out);
    return check_launch("synthesize_f64");
}

}  // extern "C"
