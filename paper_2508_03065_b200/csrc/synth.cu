// Fractional-delay synthesis (synth.py:194-258 + _kernels.py:90-136).
//
// Fast path (fp32 I/O, the B200 roofline path)
//   k_branch_records_f32  v'_k = x (*) c'_k for the centred Farrow bank.
//                         Record layout: one row per input sample (zero-padded
//                         on both sides so the gather needs no bounds test --
//                         the reference's `valid` window reads zeros), the
//                         row's 4 NP branch values contiguous (32 B for the
//                         8-branch bank): one IMAD.WIDE and one 256-bit load
//                         (LDG.256) per update; a warp's 32 consecutive rows
//                         are one coalesced 1 KiB access.
//   k_synth_f32           one CTA per (job, 32*U-sample tile, image chunk);
//                         8 warps walk the chunk's delay-sorted images, lane
//                         l of a warp owns samples n0 + 32u + l, u < U.  Per
//                         update: the interval polynomial of the track (fp32
//                         around an fp64 anchor), the (D, mu) split, one
//                         coalesced 16-byte load per plane (L1), an even/odd
//                         Horner in mu - 1/2 on paired FMAs (FFMA2), gain
//                         1/(4 pi d) and one FMA into a register accumulator.
//                         Decimated tiers with N | 1024 run an N-templated
//                         body whose interval reloads sit at compile-time
//                         steps, so the 32 unrolled steps are straight-line
//                         code and overlap.  Warps reduce in fixed order in
//                         shared memory, then write coalesced.
//   k_reduce_f32          fixed-order sum of chunk partials.
//
// Exact path (fp64): k_synth_f64 repeats the reference arithmetic for every
// (image, sample) -- 65-tap upsampled or per-sample distances, tau =
// (rate*d)/c, gain, floor split, Horner in mu -- and its summation order:
// 32-image blocks in canonical order, then the pairwise block tree
// (synth.py:182-191) evaluated with an equivalent merge stack.
#include <cfloat>
#include <cstdlib>
#include <mutex>
#include <type_traits>
#include <utility>
#include <vector>

#include "mvb_common.cuh"

namespace mvb {

// ---------------------------------------------------------------------------
// record layout

// a record row holds the nb = 4 NP branch values of one input sample,
// contiguous and padded to a whole number of 32-byte units when NP > 1, so a
// row is one (NP = 1) 16-byte or NP/2 (rounded up) 32-byte loads
template <int NP>
__host__ __device__ constexpr int row_f4() { return NP == 1 ? 1 : 2 * ((NP + 1) / 2); }

// &base[row r] as one IMAD.WIDE.U32
template <int NP>
__device__ __forceinline__ const float4* rec_row(const float4* base, unsigned r) {
    const float4* p;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(p) : "r"(r), "n"(16 * row_f4<NP>()), "l"(base));
    return p;
}

// 32-byte read-only load (sm_100 LDG.256)
__device__ __forceinline__ void ldg8(float4& a, float4& b, const float4* p) {
    asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
        : "l"(p));
}

// One launch for every distinct dry signal of a batch: blockIdx.y selects
// the signal (x_all + off[y], length len[y], record rows from row0[y]).
// Thread t of a block computes the rows m0 + t + q * blockDim.x, q < BR_Q
// (consecutive threads: consecutive rows, coalesced 32-byte row stores);
// per tap j one broadcast float4 read per 4 branches serves BR_Q x NB FMAs.
constexpr int BR_Q = 4;

template <int NP>
__global__ void k_branch_records_f32(const float* __restrict__ x_all,
                                     const int64_t* __restrict__ sig_off,
                                     const int64_t* __restrict__ sig_len,
                                     const int64_t* __restrict__ sig_row0,
                                     const int64_t* __restrict__ sig_zlo,
                                     const int64_t* __restrict__ sig_zhi,
                                     const double* __restrict__ cb, int M1, int L,
                                     float* __restrict__ rec) {
    constexpr int NB = 4 * NP;
    extern __shared__ float sx[];      // [BR_Q * blockDim.x + L - 1]
    __shared__ float4 sc[128 * NP];    // tap j, branches 4p..4p+3 at sc[j * NP + p]
    const int B = blockDim.x;
    const int64_t T = sig_len[blockIdx.y];
    const int64_t row0 = sig_row0[blockIdx.y];
    // rows [mlo, mhi) relative to sample 0: the signal rows [0, T + L - 1)
    // and, with sig_zlo / sig_zhi, the zero pads around them (written here
    // so the caller need not zero-fill the buffer)
    const int64_t mlo = sig_zlo ? sig_zlo[blockIdx.y] - row0 : 0;
    const int64_t mhi = sig_zhi ? sig_zhi[blockIdx.y] - row0 : T + L - 1;
    const int64_t m0 = mlo + (int64_t)blockIdx.x * B * BR_Q;
    if (m0 >= mhi) return;
    float4* const rows4 = reinterpret_cast<float4*>(rec);
    if (m0 + BR_Q * B <= 0 || m0 >= T + L - 1) {  // the block lies in a pad: zeros
        for (int q = 0; q < BR_Q; ++q) {
            const int64_t m = m0 + threadIdx.x + (int64_t)q * B;
            if (m >= mhi) break;
#pragma unroll
            for (int p = 0; p < NP; ++p)
                rows4[(size_t)(row0 + m) * row_f4<NP>() + p] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        return;
    }
    const float* __restrict__ x = x_all + sig_off[blockIdx.y];
    float* scf = reinterpret_cast<float*>(sc);
    for (int t = threadIdx.x; t < NB * L; t += B) {
        const int j = t / NB, k = t - (t / NB) * NB;
        scf[t] = k < M1 ? (float)cb[k * L + j] : 0.f;
    }
    for (int t = threadIdx.x; t < BR_Q * B + L - 1; t += B) {
        const int64_t q = m0 - (L - 1) + t;
        sx[t] = (q >= 0 && q < T) ? x[q] : 0.f;
    }
    __syncthreads();
    float acc[BR_Q][NB];
#pragma unroll
    for (int q = 0; q < BR_Q; ++q)
#pragma unroll
        for (int k = 0; k < NB; ++k) acc[q][k] = 0.f;
    // v_k[m] = sum_j c_k[j] x[m - j] (j ascending, one rounding per FMA);
    // sx[threadIdx.x + q * B + L-1 - j] = x[m - j]
    for (int j = 0; j < L; ++j) {
        float4 c[NP];
#pragma unroll
        for (int p = 0; p < NP; ++p) c[p] = sc[j * NP + p];
#pragma unroll
        for (int q = 0; q < BR_Q; ++q) {
            const float xv = sx[threadIdx.x + q * B + L - 1 - j];
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                acc[q][4 * p] = fmaf(c[p].x, xv, acc[q][4 * p]);
                acc[q][4 * p + 1] = fmaf(c[p].y, xv, acc[q][4 * p + 1]);
                acc[q][4 * p + 2] = fmaf(c[p].z, xv, acc[q][4 * p + 2]);
                acc[q][4 * p + 3] = fmaf(c[p].w, xv, acc[q][4 * p + 3]);
            }
        }
    }
#pragma unroll
    for (int q = 0; q < BR_Q; ++q) {
        const int64_t m = m0 + threadIdx.x + (int64_t)q * B;
        if (m >= mhi) break;
        float4* o = rows4 + (size_t)(row0 + m) * row_f4<NP>();
#pragma unroll
        for (int p = 0; p < NP; ++p)
            o[p] = make_float4(acc[q][4 * p], acc[q][4 * p + 1], acc[q][4 * p + 2], acc[q][4 * p + 3]);
    }
}

// ---------------------------------------------------------------------------
// fast synthesis helpers

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

// Even/odd Horner with paired FMAs (SASS FFMA2):  sum_k v_k x^k =
// E(x^2) + x O(x^2); the (even, odd) coefficient pairs are adjacent floats
// of the records, i.e. ready-made float2 operands.
template <int NP>
__device__ __forceinline__ float gather_horner(const float4* __restrict__ R, unsigned row,
                                               float mc) {
    const float y = mc * mc;
    const float2 yy = f2(y, y);
    const float4* a = rec_row<NP>(R, row);
    float4 v[NP];
    if (NP == 1) {
        v[0] = __ldg(a);
    } else {
#pragma unroll
        for (int p = 0; p + 1 < NP; p += 2) ldg8(v[p], v[p + 1], a + p);
        if (NP % 2) v[NP - 1] = __ldg(a + NP - 1);
    }
    float2 q = f2(v[NP - 1].z, v[NP - 1].w);
    q = __ffma2_rn(q, yy, f2(v[NP - 1].x, v[NP - 1].y));
#pragma unroll
    for (int p = NP - 2; p >= 0; --p) {
        q = __ffma2_rn(q, yy, f2(v[p].z, v[p].w));
        q = __ffma2_rn(q, yy, f2(v[p].x, v[p].y));
    }
    return fmaf(mc, q.y, q.x);
}

// The update's fractional-delay gather behind one interface, so the same
// synthesis kernel runs the Farrow records (the product) or the literal
// per-fraction table (the SURVEY H2 A/B, mvb_synthesize_f32_table).
template <int NP>
struct FarrowGather {
    const float4* __restrict__ R;
    unsigned rows;  // record rows (bounds check of the checked build)
    __device__ __forceinline__ float operator()(unsigned row, float mc) const {
        MVB_CHECK(row < rows, CHK_GATHER_ROW);
        return gather_horner<NP>(R, row, mc);
    }
    __device__ __forceinline__ float at(unsigned row, float mc, int) const { return (*this)(row, mc); }
};

// The same Horner with the row fetched through the texture pipe (two
// float4 texels per 32-byte row; a separate L1TEX data path from the LSU
// one the LDG.256 gathers saturate).  TEXM 1: every step, 2: odd steps only
// (the even ones stay LDG.256).  Measurement variants (MVB_TEX_GATHER).
template <int TEXM>
struct TexFarrowGather {
    const float4* __restrict__ R;
    unsigned rows;
    cudaTextureObject_t tex;
    __device__ __forceinline__ float horner(const float4 v0, const float4 v1, float mc) const {
        const float y = mc * mc;
        const float2 yy = f2(y, y);
        float2 q = f2(v1.z, v1.w);
        q = __ffma2_rn(q, yy, f2(v1.x, v1.y));
        q = __ffma2_rn(q, yy, f2(v0.z, v0.w));
        q = __ffma2_rn(q, yy, f2(v0.x, v0.y));
        return fmaf(mc, q.y, q.x);
    }
    __device__ __forceinline__ float operator()(unsigned row, float mc) const {
        MVB_CHECK(row < rows, CHK_GATHER_ROW);
        const float4 v0 = tex1Dfetch<float4>(tex, (int)(2 * row));
        const float4 v1 = tex1Dfetch<float4>(tex, (int)(2 * row + 1));
        return horner(v0, v1, mc);
    }
    __device__ __forceinline__ float at(unsigned row, float mc, int u) const {
        if (TEXM == 2 && (u & 1) == 0) return gather_horner<2>(R, row, mc);
        return (*this)(row, mc);
    }
};

// Literal per-fraction table: taps h_j(mu) at mu = p / TAB_P, p = 0..TAB_P,
// in shared memory (row stride L + 1: lanes at different fractions hit
// different banks), linearly interpolated in mu, then a direct L-tap gather
// of the zero-padded signal plane xp (row r <-> branch row r, so the
// reference's valid window and the zero pads are the Farrow path's):
// sum_j h_j(mu) xp[r - j].  Per tap: two shared loads, one global load, two
// FMAs plus the interpolation -- the structure the H2 estimate bounds.
constexpr int TAB_P = 512;
struct TableGather {
    const float* __restrict__ xp;
    const float* tab;  // shared memory
    int L;
    unsigned rows;
    __device__ __forceinline__ float at(unsigned row, float mc, int) const { return (*this)(row, mc); }
    __device__ __forceinline__ float operator()(unsigned row, float mc) const {
        MVB_CHECK(row < rows && row >= (unsigned)(L - 1), CHK_GATHER_ROW);
        const float sc = (mc + 0.5f) * (float)TAB_P;
        int p = (int)sc;
        p = p < 0 ? 0 : (p > TAB_P - 1 ? TAB_P - 1 : p);
        const float a = sc - (float)p;
        const float* t0 = tab + p * (L + 1);
        const float* t1 = t0 + (L + 1);
        const float* x = xp + row;
        float acc = 0.f;
#pragma unroll 8
        for (int j = 0; j < L; ++j) {
            const float h0 = t0[j];
            acc = fmaf(fmaf(a, t1[j] - h0, h0), __ldg(x - j), acc);
        }
        return acc;
    }
};

// Track residual kappa*(d(u) - g0) = u * sum_{p=1..8} g_p u^(p-1), same
// even/odd pairing over the record's (g1,g2), (g3,g4), (g5,g6), (g7,g8).
__device__ __forceinline__ float track_residual(const float4& c1, const float4& c2, float uu) {
    const float y = uu * uu;
    const float2 yy = f2(y, y);
    float2 q = f2(c2.z, c2.w);
    q = __ffma2_rn(q, yy, f2(c2.x, c2.y));
    q = __ffma2_rn(q, yy, f2(c1.z, c1.w));
    q = __ffma2_rn(q, yy, f2(c1.x, c1.y));
    return fmaf(uu, q.y, q.x) * uu;
}

__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// predicated 16-byte read-only load: v keeps its value when !pred
__device__ __forceinline__ void ldg4_if(float4& v, const float4* p, bool pred) {
    asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t"
        "@q ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];\n\t}"
        : "+f"(v.x), "+f"(v.y), "+f"(v.z), "+f"(v.w)
        : "l"(p), "r"((int)pred));
}

// rint via the 1.5*2^23 trick: v = t + MAGIC holds rint(t) in its low
// mantissa bits (|t| < 2^22): bits(v) = 0x4B400000 + rint(t).
constexpr float MAGIC_F = 12582912.0f;
constexpr int MAGIC_I = 0x4B400000;

// One decimated-image step given the interval record (c0, c1, c2):
// nlB = rec_base + n0 + lane + L + MAGIC_I - B.  Returns the contribution.
template <class G>
__device__ __forceinline__ float dec_step(const float4& c0, const float4& c1, const float4& c2,
                                          float uu, int rowbase, const G& g,
                                          float an, float invk, float dmin, int u = 0) {
    const float res = track_residual(c1, c2, uu);  // kappa * (d - g0)
    const float t = c0.y + res;
    const float v = t + MAGIC_F;
    const float mc = t - (v - MAGIC_F);
    const unsigned row = (unsigned)(rowbase - __float_as_int(v));
    const float d = fmaf(res, invk, c0.z);
    const float A = an * rcp_approx(fmaxf(d, dmin));
    return A * g.at(row, mc, u);
}

// Decimated image on a tile wholly inside [0, T) with TILE % NT == 0 (its
// records staged in shared memory by the warp's cp.async pipeline): the
// tile starts on an interval boundary, interval q covers steps
// [q*SPI, (q+1)*SPI) and u = 2r/N - 1 is a per-step constant plus a lane
// term -- no per-step bookkeeping, straight-line steps.
template <int U, int NT, class G>
__device__ __forceinline__ void dec_static(float (&acc)[U], const float4* __restrict__ cs,
                                           const G& g, int lane, int nl,
                                           float an, float invk, float dmin) {
    constexpr int SPI = NT / 32;  // steps per coarse interval
    const float lt = (float)lane * (2.0f / NT);
    float4 c0, c1, c2;
    int nlB = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
        if (u % SPI == 0) {  // interval records staged in shared memory
            const float4* c = cs + 3 * (u / SPI);
            c0 = c[0];
            c1 = c[1];
            c2 = c[2];
            nlB = nl - __float_as_int(c0.x);
        }
        const float uu = lt + ((float)((u % SPI) * 32) * (2.0f / NT) - 1.0f);
        acc[u] += dec_step(c0, c1, c2, uu, nlB + 32 * u, g, an, invk, dmin, u);
    }
}

constexpr int SYNTH_WARPS = 8;

#ifdef MVB_CTA_TIMING
// diagnostic build: per-CTA (start, end, smid, work index) of the fast synthesis
__device__ unsigned long long g_cta_time[4 * 65536];
#endif

// 16-byte asynchronous global -> shared copy (LDGSTS), L2-only caching
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Staging transport: lane-parallel 16-byte LDGSTS (cp.async), or with
// -DMVB_STAGE_BULK one 1-D bulk copy per staged object (cp.async.bulk
// through the TMA unit, completion on a per-warp mbarrier with a
// transaction count; VERDICT r1 lever).  Measured (same box, 10 steps): c3
// synthesis 8.20 ms LDGSTS vs 8.40 bulk (8.33 without the per-image proxy
// fence), c4 65.7 vs 66.2 (65.6) -- the one-lane issue and mbarrier wait
// put more latency on the warp's one-image-ahead pipeline than the LDGSTS
// wavefronts cost, so LDGSTS stays the default.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bar_init(unsigned long long* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
    // visible to the async proxy (CTA scope; the cluster-scope
    // fence.mbarrier_init compiles to an L1 invalidate)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void bar_arrive_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "MVB_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra MVB_WAIT_%=;\n\t}"
        ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
// generic-proxy reads of a slot happen before the async-proxy write that
// overwrites it
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Per-warp staging area: image structs for the current, next and next-next
// image of the warp, and the interval records of the current and next image
// over this tile (only for factors N >= 32, at most TN/32 + 1 records).
template <int U>
struct alignas(16) WarpStage {
    static constexpr int RMAX = U + 1;
    static_assert(3 * RMAX <= 64, "stage_records copies at most two 16-byte chunks per lane");
    mvb_image img[3];
    mvb_coef32 rec[2][RMAX];
    unsigned long long bar;  // bulk-copy completion (per warp)
};

// issue the copies of image q's interval records over [n0, n0+TN) into slot
// `dst` (lane-parallel 16-byte chunks); the records exist only for factor >= 32
template <int U>
__device__ __forceinline__ unsigned stage_records(WarpStage<U>& st, int slot, const mvb_image& q,
                                              const mvb_coef32* __restrict__ coef, int n0, int T,
                                              int lane) {
    constexpr int TN = 32 * U;
    const int N = q.factor;
    // tiles past the track end (n0 >= T) read the held record directly: cnt <= 0
    if (N >= 32 && n0 < T) {
        const int nlast = n0 + TN - 1 < T - 1 ? n0 + TN - 1 : T - 1;
        int k0, last;
        if ((N & (N - 1)) == 0) {  // power of two: shifts, not divisions
            const int sh = 31 - __clz(N);
            k0 = n0 >> sh;
            last = nlast >> sh;
        } else {
            k0 = n0 / N;
            last = nlast / N;
        }
        const int chunks = 3 * (last - k0 + 1);  // <= 3 (U + 1) for N >= 32
        const char* src = reinterpret_cast<const char*>(coef + q.coef) + 48 * k0;
        char* dst = reinterpret_cast<char*>(st.rec[slot]);
        MVB_CHECK(k0 >= 0 && last < q.n_coarse, CHK_RECORD_INDEX);
        MVB_CHECK(chunks <= 3 * WarpStage<U>::RMAX, CHK_STAGE_SIZE);
        MVB_CHECK(((uintptr_t)src & 15) == 0 && ((uintptr_t)dst & 15) == 0, CHK_ALIGN);
#ifndef MVB_STAGE_BULK
        // at most two 16-byte chunks per lane, no loop
        if (lane < chunks) cp_async16(dst + 16 * lane, src + 16 * lane);
        if (lane + 32 < chunks) cp_async16(dst + 16 * (lane + 32), src + 16 * (lane + 32));
#else
        if (lane == 0) bulk_g2s(dst, src, 16u * chunks, &st.bar);
        return 16u * chunks;
#endif
    }
    return 0u;
}

template <int U>
__device__ __forceinline__ unsigned stage_image(WarpStage<U>& st, int slot, const mvb_image* src,
                                                int lane) {
#ifndef MVB_STAGE_BULK
    if (lane < (int)(sizeof(mvb_image) / 16))
        cp_async16(reinterpret_cast<char*>(&st.img[slot]) + 16 * lane,
                   reinterpret_cast<const char*>(src) + 16 * lane);
#else
    if (lane == 0) bulk_g2s(&st.img[slot], src, (unsigned)sizeof(mvb_image), &st.bar);
#endif
    return (unsigned)sizeof(mvb_image);
}

// One staging phase of a warp: the copies issued since the last wait land
// before the next stage_wait.  LDGSTS: commit / wait_all; bulk: lane 0 arms
// the warp's mbarrier with the phase's byte count (after issuing -- the
// phase cannot complete before its one arrival), all lanes wait on parity.
template <int U>
__device__ __forceinline__ void stage_commit(WarpStage<U>& st, unsigned bytes, int lane) {
#ifndef MVB_STAGE_BULK
    cp_async_commit();
#else
    if (lane == 0) bar_arrive_tx(&st.bar, bytes);
#endif
}
template <int U>
__device__ __forceinline__ void stage_wait(WarpStage<U>& st, unsigned& parity) {
#ifndef MVB_STAGE_BULK
    cp_async_wait_all();
#else
    bar_wait(&st.bar, parity);
    parity ^= 1u;
#endif
    __syncwarp();
}

// Active image range of a tile.  The delay sort's keys (k_delay_sort:
// floor(kappa * d) at the sort segment's centre, ascending within each run
// of the job's table) bound every image's delay over the tile: |tau(n) -
// tau(t_key)| <= E = 2 * kappa * (largest source step + largest receiver
// step) * (|n - t_key| + max factor) + 8 samples (the factor covers the
// decimated key's coarse sample, the 2 any overshoot of the band-limited
// track or a low-passed path over the full-rate steps).  An image whose key
// lies outside (klo, khi] reads only the zero pads of the branch records
// over the whole tile -- it has not arrived yet or its signal has ended --
// so the warps never visit it (the in-loop tests below would skip it too,
// after paying for its staging).  The sorted table's images with keys in
// (klo, khi] are a contiguous range of each run, found by a warp-parallel
// 32-ary search (2-3 dependent loads).
struct RangeArgs {
    const unsigned* keys;  // parallel to the sorted image table; null: no narrowing
    const double* bbox;    // mvb_path_bbox records (16 words per job)
    int run_len;           // sorted run length of the table (a job's whole table: >= n_img)
    int seg_len;           // sort segment length (samples)
    int max_factor;        // largest decimation factor of the batch
    cudaTextureObject_t tex;  // branch records as float4 texels (TexFarrowGather) or 0
};

// first positions in [b, e) whose key exceeds x0 / x1 (sorted keys), both
// searches in the same rounds; has0 / has1 false: the search is skipped
// (the position is b, resp. e).  Per round the lanes probe 32 increasing
// positions, the last lane the range's end, so a range wholly above or
// below x settles in one round (a tile in the middle of the signal).
__device__ __forceinline__ void bound_round(const unsigned* __restrict__ k, int& lo, int& len,
                                            unsigned x, int lane) {
    if (len <= 0) return;
    const int s = (len + 30) / 31;
    int q = lane == 31 ? lo + len - 1 : lo + lane * s;
    const bool valid = q < lo + len;
    const bool t = valid && __ldg(k + q) <= x;
    const int last_true = __reduce_max_sync(0xffffffffu, t ? q : lo - 1);
    const int first_false = __reduce_min_sync(0xffffffffu, valid && !t ? q : lo + len);
    lo = last_true + 1;
    len = first_false - lo;
}

__device__ __forceinline__ void upper_bounds(const unsigned* __restrict__ k, int b, int e,
                                             bool has0, unsigned x0, bool has1, unsigned x1,
                                             int lane, int& p0, int& p1) {
    int lo0 = b, len0 = has0 ? e - b : 0, lo1 = has1 ? b : e, len1 = has1 ? e - b : 0;
    while (len0 > 0 || len1 > 0) {  // warp-uniform
        bound_round(k, lo0, len0, x0, lane);
        bound_round(k, lo1, len1, x1, lane);
    }
    p0 = lo0;
    p1 = lo1;
}

// Warp w's image sequence over a tile: the positions p == b + w (mod 8) of
// the chunk [b, e) that lie in the active parts [a0, a1) and [c0, c1) --
// the same warp and order every image has without narrowing, so the warps'
// sums (and the output) are bit-identical: the skipped images add exact
// zeros.  k-th position: k < nA ? fA + 8k : fC + 8(k - nA); n in all.
struct ActiveRange {
    int fA, nA, fC, n;
    __device__ __forceinline__ int operator[](int k) const {
        return k < nA ? fA + SYNTH_WARPS * k : fC + SYNTH_WARPS * (k - nA);
    }
};

// first position >= a congruent to r (mod 8), and the count of such in [a, z)
__device__ __forceinline__ void congruent(int a, int z, int r, int& f, int& cnt) {
    f = a + ((r - a) & (SYNTH_WARPS - 1));
    cnt = z > f ? (z - f + SYNTH_WARPS - 1) / SYNTH_WARPS : 0;
}

template <int TN>
__device__ __forceinline__ ActiveRange active_range(const RangeArgs& ra, const mvb_job& J,
                                                    const mvb_work& w, int n0, int warp,
                                                    int lane) {
    const int b = w.img_begin, e = w.img_end;
    ActiveRange r;
    congruent(b, e, b + warp, r.fA, r.nA);
    r.fC = e;
    r.n = r.nA;
    if (ra.keys == nullptr || e <= b) return r;
    const double* box = ra.bbox + 16 * (int64_t)w.job;
    const double rate = 2.0 * J.kappa * (box[12] + box[13]);
    int64_t tk = (int64_t)w.seg * ra.seg_len + ra.seg_len / 2;
    if (tk > J.T - 1) tk = J.T - 1;
    const int64_t na = n0 < J.T - 1 ? n0 : J.T - 1;
    const int64_t nb = n0 + TN - 1 < J.T - 1 ? n0 + TN - 1 : J.T - 1;
    const int64_t dist = max(llabs(na - tk), llabs(nb - tk)) + ra.max_factor;
    const double E = rate * (double)dist + 8.0;
    const double lo = (double)n0 + J.d0 - (double)J.ls - E - 3.0;
    const double hi = (double)n0 + TN + J.d0 + E + 2.0;
    const bool has0 = lo >= 0.0, has1 = hi < 4294967295.0;
    if (!has0 && !has1) return r;
    const unsigned x0 = has0 ? (unsigned)lo : 0u, x1 = has1 ? (unsigned)hi : 0u;
    const unsigned* k = ra.keys + J.img_off + (int64_t)w.seg * J.img_stride;
    // the chunk's runs: at most two (chunks are no longer than a run)
    const int rb = (b / ra.run_len + 1) * ra.run_len;
    if (rb >= e) {
        int p0, p1;
        upper_bounds(k, b, e, has0, x0, has1, x1, lane, p0, p1);
        congruent(p0, p1, b + warp, r.fA, r.nA);
        r.n = r.nA;
        return r;
    }
    if (rb + ra.run_len < e) return r;  // spans three runs: no narrowing
    int p0, p1, q0, q1, nC;
    upper_bounds(k, b, rb, has0, x0, has1, x1, lane, p0, p1);
    upper_bounds(k, rb, e, has0, x0, has1, x1, lane, q0, q1);
    congruent(p0, p1, b + warp, r.fA, r.nA);
    congruent(q0, q1, b + warp, r.fC, nC);
    r.n = r.nA + nC;
    return r;
}

template <int U, int NP, int MINB, bool TAB = false, int TEXM = 0>
__global__ void __launch_bounds__(SYNTH_WARPS * 32, MINB) k_synth_f32(
    const mvb_job* __restrict__ jobs, const mvb_work* __restrict__ work,
    const mvb_image* __restrict__ images, const mvb_coef32* __restrict__ coef,
    const float* __restrict__ rec, const double* __restrict__ paths, float* __restrict__ out,
    float* __restrict__ part, const __grid_constant__ RangeArgs ra,
    const float* __restrict__ table = nullptr) {
    constexpr int TN = 32 * U;
    __shared__ float red[SYNTH_WARPS][TN];
    __shared__ WarpStage<U> stage[SYNTH_WARPS];
#ifdef MVB_CTA_TIMING
    unsigned long long t_start;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
#endif
    const mvb_work* wp = work + blockIdx.x;
    const mvb_job* Jp = jobs + wp->job;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int n0 = wp->tile * TN;
    if (n0 >= Jp->out_len) return;  // tile planned for the length bound only
    const int T = Jp->T;
    const int Lsh = Jp->L;
    // rows are indexed globally: row = rec_base + (n + L - D) >= 0 thanks to
    // the zero front pad of every signal's region
    const int rb = (int)Jp->rec_base;
    using Gather = std::conditional_t<TAB, TableGather,
                                      std::conditional_t<(TEXM > 0), TexFarrowGather<TEXM>,
                                                         FarrowGather<NP>>>;
    Gather g;
    if constexpr (TAB) {
        // the fraction table: (TAB_P + 1) rows of L taps, padded to L + 1
        extern __shared__ float tab_smem[];
        const int Lt = Jp->L;
        for (int t = threadIdx.x; t < (TAB_P + 1) * Lt; t += blockDim.x)
            tab_smem[(t / Lt) * (Lt + 1) + t % Lt] = table[t];
        __syncthreads();
        g = TableGather{rec, tab_smem, Lt, (unsigned)Jp->rec_rows};
    } else {
        if constexpr (TEXM > 0)
            g = TexFarrowGather<TEXM>{reinterpret_cast<const float4*>(rec), (unsigned)Jp->rec_rows,
                                      ra.tex};
        else
            g = FarrowGather<NP>{reinterpret_cast<const float4*>(rec), (unsigned)Jp->rec_rows};
    }
    MVB_CHECK(wp->seg >= 0 && (Jp->img_stride == 0 || wp->img_end <= Jp->img_stride) &&
                  wp->img_begin >= 0 && wp->img_begin <= wp->img_end, CHK_WORK);
    // the images this tile can read anything but zero pads from
    // (kept in shared memory: the mapping is read once per image, and three
    // more live registers across the image loop cost spills)
    __shared__ ActiveRange ranges[SYNTH_WARPS];
    {
        const ActiveRange a = active_range<TN>(ra, *Jp, *wp, n0, warp, lane);
        if (lane == 0) ranges[warp] = a;
        __syncwarp();
    }
    const ActiveRange& ar = ranges[warp];
    const int nv = ar.n;
    // this tile's delay-sorted image table (sort segment wp->seg)
    const mvb_image* __restrict__ imgs = images + Jp->img_off + (int64_t)wp->seg * Jp->img_stride;
    const float invk = (float)(1.0 / Jp->kappa);
    const float dmin = (float)Jp->d_min;
    float* __restrict__ row = red[warp];
    WarpStage<U>& st = stage[warp];
#pragma unroll
    for (int u = 0; u < U; ++u) row[32 * u + lane] = 0.f;
    float acc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) acc[u] = 0.f;
    const bool inside = n0 + TN <= T;  // no hold-extension inside this tile
    const bool tail = n0 >= T;         // wholly hold-extended: one delay per image
    // Exact zeros: an image contributes nothing to this tile when every
    // gather row lies in the zero pads of the branch records, i.e. outside
    // the signal rows [rb, rb + ls) -- before its first sample arrives (delay
    // beyond the tile) or after the signal ended.  Skipping it is
    // bit-identical (the Horner of zero rows adds 0).  Tail tiles test the
    // held delay exactly; `front` tiles (n0 below the largest possible
    // delay, ~10% of c3's tiles) bound a decimated image's delay from its
    // staged interval records.  c3: ~10% of all updates are such zeros.
    const int ls = (int)Jp->ls;
    const bool front = n0 + TN <= (int)(Jp->out_len - Jp->ls) + 2;

    // prologue of the staging pipeline: structs of the first two images, then
    // the first image's records
    // the warp's image sequence ar[k]: the loop carries only the count left
    // and the position two images ahead (as many live registers as a plain
    // strided walk -- more spill into the image loop at the 80-register cap)
#ifdef MVB_STAGE_BULK
    if (lane == 0) bar_init(&st.bar);
    __syncwarp();
#endif
    unsigned parity = 0, bytes = 0;
    if (0 < nv) bytes += stage_image(st, 0, imgs + ar[0], lane);
    if (1 < nv) bytes += stage_image(st, 1, imgs + ar[1], lane);
    stage_commit(st, bytes, lane);
    stage_wait(st, parity);
    bytes = 0;
    if (0 < nv) bytes += stage_records(st, 0, st.img[0], coef, n0, T, lane);
    stage_commit(st, bytes, lane);
    int pos2 = ar[2];  // position of the image two ahead (valid while rem > 2)
    // a chunk over two sorted runs (time shards) has a second part; only
    // then does the walk read the range again (an LDS per image is ~1% of
    // the data-pipe wavefronts the image costs)
    const bool two_parts = nv > ar.nA;

    // staging slots rotate: struct slots (cur, nx1, nx2), record slot rcur,
    // packed in one register (bits 0-1, 2-3, 4-5, 6)
    int slots = 0 | (1 << 2) | (2 << 4);
    for (int rem = nv; rem > 0; --rem,
             slots = ((slots >> 2) & 15) | ((slots & 3) << 4) | ((slots & 64) ^ 64)) {
        const int cur = slots & 3, nx1 = (slots >> 2) & 3, nx2 = (slots >> 4) & 3,
                  rcur = (slots >> 6) & 1;
        // everything issued one image ago has landed: records(i), struct(i+1)
        stage_wait(st, parity);
        // stream the next image's records and the struct after it while
        // this image is processed (their slots were last read two images ago)
#if defined(MVB_STAGE_BULK) && !defined(MVB_NO_PROXY_FENCE)
        if (lane == 0) fence_proxy_async();
#endif
        unsigned bytes = 0;
        if (rem > 1) bytes += stage_records(st, rcur ^ 1, st.img[nx1], coef, n0, T, lane);
        if (rem > 2) {
            bytes += stage_image(st, nx2, imgs + pos2, lane);
            // next position: +8, or the second part's first at the first one's end
            pos2 += SYNTH_WARPS;
            if (two_parts && pos2 == ar.fA + SYNTH_WARPS * ar.nA) pos2 = ar.fC;
        }
        stage_commit(st, bytes, lane);

        const mvb_image& im = st.img[cur];
        const int N = im.factor;
        const float an = im.amp_num;
        if (tail) {
            // hold-extended tile (synth.py:213-216): every sample sees the
            // track value at T-1, so the delay split and the gain are one
            // warp-uniform computation; per step only the gather remains
            float mc, A;
            int row0;
            if (N == 1) {
                const double* p = paths + 3 * (Jp->pos_off + (int64_t)(T - 1));
                const double* q = paths + 3 * (Jp->mic_off + (Jp->mic_moving ? (int64_t)(T - 1) : 0));
                const double dx = im.off[0] + im.sign[0] * p[0] - q[0];
                const double dy = im.off[1] + im.sign[1] * p[1] - q[1];
                const double dz = im.off[2] + im.sign[2] * p[2] - q[2];
                const double d = sqrt(dx * dx + dy * dy + dz * dz);
                const double sv = fma(d, Jp->kappa, (double)(Lsh - Jp->d0));
                const double D = floor(sv);
                mc = (float)(sv - D) - 0.5f;
                row0 = rb + n0 + lane + Lsh - (int)D;
                A = an * rcp_approx(fmaxf((float)d, dmin));
            } else {
                const int kT = (T - 1) / N, rT = (T - 1) - kT * N;
                MVB_CHECK(kT < im.n_coarse, CHK_RECORD_INDEX);
                const float4* c = reinterpret_cast<const float4*>(coef + im.coef) + 3u * (unsigned)kT;
                const float4 c0 = __ldg(c), c1 = __ldg(c + 1), c2 = __ldg(c + 2);
                const float res = track_residual(c1, c2, fmaf((float)rT, 2.0f / (float)N, -1.f));
                const float tq = c0.y + res;
                const float v = tq + MAGIC_F;
                mc = tq - (v - MAGIC_F);
                row0 = rb + n0 + lane + Lsh + MAGIC_I - __float_as_int(c0.x) - __float_as_int(v);
                A = an * rcp_approx(fmaxf(fmaf(res, invk, c0.z), dmin));
            }
            const int rfirst = row0 - lane;  // row of the tile's first sample (warp-uniform)
            if (rfirst + TN <= rb || rfirst >= rb + ls) continue;  // all in the zero pads
#pragma unroll
            for (int u = 0; u < U; ++u) acc[u] += A * g.at((unsigned)(row0 + 32 * u), mc, u);
            continue;
        }
        if (N == 1) {
            // near images (full-rate tier): exact fp64 distance per sample,
            // accumulated in the warp's own shared-memory row
            const double kappa = Jp->kappa;
            const double sL = (double)(Lsh - Jp->d0);
            const double ox = im.off[0], oy = im.off[1], oz = im.off[2];
            const double sx = im.sign[0], sy = im.sign[1], sz = im.sign[2];
            const double* P = paths + 3 * Jp->pos_off;
            const int moving = Jp->mic_moving;
            const double* Q = paths + 3 * Jp->mic_off;
#pragma unroll 1
            for (int u = 0; u < U; ++u) {
                const int n = n0 + 32 * u + lane;
                const int m = n < T ? n : T - 1;
                const double* p = P + 3 * (int64_t)m;
                const double* q = moving ? Q + 3 * (int64_t)m : Q;
                const double dx = ox + sx * p[0] - q[0];
                const double dy = oy + sy * p[1] - q[1];
                const double dz = oz + sz * p[2] - q[2];
                const double d = sqrt(dx * dx + dy * dy + dz * dz);
                const double s = fma(d, kappa, sL);
                const double D = floor(s);
                const float mc = (float)(s - D) - 0.5f;
                const unsigned r = (unsigned)(rb + n + Lsh - (int)D);
                const float A = an * rcp_approx(fmaxf((float)d, dmin));
                row[32 * u + lane] = fmaf(A, g.at(r, mc, u), row[32 * u + lane]);
            }
            continue;
        }
        const int nl = rb + n0 + lane + Lsh + MAGIC_I;
        const float4* __restrict__ cs = reinterpret_cast<const float4*>(st.rec[rcur]);
        if (inside && (N == 32 || N == 64 || N == 128 || N == 256)) {
            if (front) {
                // delay lower bound over the tile from its TN/N staged records:
                // D = B + rint(f + res), |res| <= sum |kappa g_p| (|u| <= 1)
                float lo = FLT_MAX;
                if (lane < TN / N) {
                    const float4* c = cs + 3 * lane;
                    const float4 a = c[0], b = c[1], d = c[2];
                    const float S = fabsf(b.x) + fabsf(b.y) + fabsf(b.z) + fabsf(b.w) + fabsf(d.x) +
                                    fabsf(d.y) + fabsf(d.z) + fabsf(d.w);
                    lo = (float)__float_as_int(a.x) + a.y - S - 1.0f;
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
                if (lo > (float)(n0 + TN + Lsh)) continue;  // every row before the signal
            }
            // staged records: slot j = interval n0/N + j
            switch (N) {
                case 32: dec_static<U, 32>(acc, cs, g, lane, nl, an, invk, dmin); break;
                case 64: dec_static<U, 64>(acc, cs, g, lane, nl, an, invk, dmin); break;
                case 128: dec_static<U, 128>(acc, cs, g, lane, nl, an, invk, dmin); break;
                default: dec_static<U, 256>(acc, cs, g, lane, nl, an, invk, dmin); break;
            }
        } else {
            // ---- generic: per-lane intervals (other factors, or the tile
            // reaches the hold-extended tail n >= T); records from global ----
            const float4* __restrict__ cf4 = reinterpret_cast<const float4*>(coef + im.coef);
            const float twoInvN = 2.0f / (float)N;
            const int mfirst = n0 + lane < T ? n0 + lane : T - 1;
            int k = mfirst / N;
            int r = mfirst - k * N;
            const int kT = (T - 1) / N, rT = (T - 1) - kT * N;
            int kc = -1;
            float4 c0 = make_float4(0.f, 0.f, 0.f, 0.f), c1 = c0, c2 = c0;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int n = n0 + 32 * u + lane;
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
                    MVB_CHECK(k >= 0 && k < im.n_coarse, CHK_RECORD_INDEX);
                    const float4* c = cf4 + 3u * (unsigned)k;
                    c0 = __ldg(c); c1 = __ldg(c + 1); c2 = __ldg(c + 2);
                    kc = k;
                }
                const float uu = fmaf((float)r, twoInvN, -1.f);
                acc[u] += dec_step(c0, c1, c2, uu, nl - __float_as_int(c0.x) + 32 * u, g, an,
                                       invk, dmin, u);
            }
        }
    }
    cp_async_wait_all();
#pragma unroll
    for (int u = 0; u < U; ++u) row[32 * u + lane] += acc[u];
    __syncthreads();
    const int64_t out_len = Jp->out_len;
    const int n_chunks = Jp->n_chunks;
    float* dst = n_chunks == 1 ? out + Jp->out_off : part + Jp->part_off + (int64_t)wp->chunk * out_len;
#pragma unroll
    for (int q = 0; q < TN / (SYNTH_WARPS * 32); ++q) {
        const int t2 = q * SYNTH_WARPS * 32 + threadIdx.x;
        float s = red[0][t2];
#pragma unroll
        for (int w = 1; w < SYNTH_WARPS; ++w) s += red[w][t2];
        const int64_t n = (int64_t)n0 + t2;
        if (n < out_len) dst[n] = s;
    }
#ifdef MVB_CTA_TIMING
    if (threadIdx.x == 0 && blockIdx.x < 65536) {
        unsigned long long t_end;
        unsigned smid;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_cta_time[4 * blockIdx.x] = t_start;
        g_cta_time[4 * blockIdx.x + 1] = t_end;
        g_cta_time[4 * blockIdx.x + 2] = smid;
        g_cta_time[4 * blockIdx.x + 3] = ((unsigned long long)wp->tile << 32) | (unsigned)wp->chunk;
    }
#endif
}

// Zero-padded signal plane of the table A/B: xp[row0 + i] = x[i] (the
// caller zero-fills xp), rows numbered like the branch records.
__global__ void k_signal_plane(const float* __restrict__ x_all, const int64_t* __restrict__ sig_off,
                               const int64_t* __restrict__ sig_len,
                               const int64_t* __restrict__ sig_row0, float* __restrict__ xp) {
    const int64_t T = sig_len[blockIdx.y];
    const float* x = x_all + sig_off[blockIdx.y];
    float* dst = xp + sig_row0[blockIdx.y];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < T;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = x[i];
}

__global__ void k_reduce_f32(const mvb_job* __restrict__ jobs, const float* __restrict__ part,
                             float* __restrict__ out) {
    const mvb_job J = jobs[blockIdx.y];
    if (J.n_chunks <= 1) return;
    // a time shard's partials exist only on its window [w0, w1)
    const int64_t n1 = J.w1 > 0 && J.w1 < J.out_len ? J.w1 : J.out_len;
    for (int64_t n = J.w0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < n1;
         n += (int64_t)gridDim.x * blockDim.x) {
        const float* p = part + J.part_off + n;
        float s = p[0];
        for (int c = 1; c < J.n_chunks; ++c) s += p[(int64_t)c * J.out_len];
        out[J.out_off + n] = s;
    }
}

// ---------------------------------------------------------------------------
// exact synthesis
//
// One CTA per (job, 32-sample tile); lane l of every warp owns sample
// n0 + l.  Images are processed in chunks of F64_CHUNK_BLOCKS 32-image
// blocks of the canonical order:
//   1. every warp computes the contributions A * Horner(mu) of images
//      w, w + 8, ... of the chunk (the 65-tap upsample is the cost) into
//      shared memory -- contributions are independent, only their sum is
//      ordered;
//   2. warp b sums block b of the chunk sequentially over its 32 images,
//      (((0 + c_0) + c_1) + ...) -- the order of _accumulate_numba's image
//      loop into a zeroed block buffer (_kernels.py:112-122, synth.py:246-251);
//      an image whose read index is outside the branch streams adds +0.0,
//      which leaves the sum unchanged (a sum that starts at +0.0 never
//      becomes -0.0 in round-to-nearest);
//   3. warp 0 folds the chunk's block sums into the pairwise tree of
//      synth.py:182-191, kept as a merge stack of (value, level): a full
//      chunk is a perfect subtree of level log2(F64_CHUNK_BLOCKS), a
//      partial last chunk splits into aligned power-of-two subtrees --
//      equivalent to pushing its blocks one by one (binary counter).
// Bit-identical to the reference arithmetic (explicit _rn operations, no
// FMA contraction), deterministic, and parallel over images as well as
// samples, so small image sets (c1: 63 images) still fill the GPU.

constexpr int F64_WARPS = 8;
constexpr int F64_CHUNK_BLOCKS = 4;  // power of two
constexpr int F64_CHUNK = 32 * F64_CHUNK_BLOCKS;
constexpr int F64_LOG_CHUNK = 2;
static_assert((1 << F64_LOG_CHUNK) == F64_CHUNK_BLOCKS, "chunk is a power of two");
// a tile's slice of a factor's transposed phase table, tab[col * N + ph0 +
// lane] for the 65 columns (the tile's 32 samples share one interval), kept
// in shared memory for up to F64_TAB_SLOTS factors: one LDS per tap instead
// of an LDG plus its 64-bit address arithmetic
constexpr int F64_TAB_SLOTS = 2;
// images per warp evaluated together: their 65-tap upsample chains are
// independent, so G chains hide the fp64 add latency of one (each chain
// keeps the reference's tap order)
// (a template parameter G of k_synth_f64: 4 at 2 CTAs/SM, or 2 at 3 CTAs/SM
// for large image sets -- mvb_synthesize_f64_ex)
// each warp's F64_G coarse windows (65 samples, padded) staged in shared
// memory before the tap loop: all their loads in flight at once instead of
// one L1/L2 round trip per unrolled batch of taps
constexpr int F64_WIN = 66;
constexpr size_t f64_smem_bytes(int G) {
    return sizeof(double) * (F64_CHUNK * 32 + F64_CHUNK_BLOCKS * 32 + F64_TAB_SLOTS * 65 * 32 +
                             F64_WARPS * G * F64_WIN);
}

__device__ __forceinline__ void merge_push(double* st_v, int* st_l, int& sp, double v, int l) {
    while (sp > 0 && st_l[sp - 1] == l) {
        v = xadd(st_v[--sp], v);
        ++l;
    }
    st_v[sp] = v;
    st_l[sp++] = l;
}

template <int MINB, int F64_G>
__global__ void __launch_bounds__(F64_WARPS * 32, MINB) k_synth_f64(
    const mvb_job* __restrict__ jobs, const mvb_image* __restrict__ images,
    const double* __restrict__ coarse, const double* __restrict__ tables,
    const double* __restrict__ streams, const double* __restrict__ paths,
    double* __restrict__ out) {
    extern __shared__ double f64_smem[];
    double* contrib = f64_smem;                 // [F64_CHUNK images][32 lanes]
    double* bsum = f64_smem + F64_CHUNK * 32;   // [F64_CHUNK_BLOCKS][32 lanes]
    double* tslice = bsum + F64_CHUNK_BLOCKS * 32;  // [F64_TAB_SLOTS][65 cols][32 lanes]
    double* wwin = tslice + F64_TAB_SLOTS * 65 * 32;  // [F64_WARPS][F64_G][F64_WIN]
    __shared__ int64_t slot_tab[F64_TAB_SLOTS];     // table offset cached in each slot (-1: none)
    const mvb_job& J = jobs[blockIdx.y];
    const int64_t out_len = J.out_len;
    const int64_t n0 = (int64_t)blockIdx.x * 32;
    if (n0 >= out_len) return;  // CTA-uniform
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t n = n0 + lane;
    const bool valid = n < out_len;
    const int64_t m = (valid ? n : out_len - 1) < J.T ? (valid ? n : out_len - 1) : J.T - 1;
    const double* p = paths + 3 * (J.pos_off + m);
    const double* q = paths + 3 * (J.mic_off + (J.mic_moving ? m : 0));
    const double P[3] = {p[0], p[1], p[2]};
    const double Q[3] = {q[0], q[1], q[2]};
    const double* V = streams + J.rec_base;
    const double L = (double)J.L, d0 = (double)J.d0;
    const double four_pi = 4.0 * 3.141592653589793;  // 4.0 * np.pi
    const int64_t n_img = J.n_img;
    const mvb_image* __restrict__ imgs = images + J.img_off;
    // merge stack (warp 0's lanes): at most one entry per level
    double st_v[40];
    int st_l[40];
    int sp = 0;
    if (threadIdx.x < F64_TAB_SLOTS) slot_tab[threadIdx.x] = -1;
    const bool tile_in_track = n0 + 31 < J.T;  // every lane a distinct sample before the end
    for (int64_t c0 = 0; c0 < n_img; c0 += F64_CHUNK) {
        const int cn = n_img - c0 < F64_CHUNK ? (int)(n_img - c0) : F64_CHUNK;
        // 0. table slices for the factors of the chunk's first and last images
        //    (tiers are contiguous in the canonical order, so a chunk rarely
        //    spans more than two factors; others read the global table)
        if (tile_in_track) {
            __syncthreads();  // the previous chunk's readers are done with the slots
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const mvb_image& ie = imgs[c0 + (e == 0 ? 0 : cn - 1)];
                const int64_t tb = ie.table;
                const int Nf = ie.factor;
                if (Nf == 1 || Nf % 32 != 0 || slot_tab[0] == tb || slot_tab[1] == tb) continue;
                // replace the slot not holding the other end's table
                const int64_t other = imgs[c0 + (e == 0 ? cn - 1 : 0)].table;
                const int sl = slot_tab[0] == other ? 1 : 0;
                __syncthreads();
                const int ph0 = (int)(n0 % Nf);
                for (int t = threadIdx.x; t < 65 * 32; t += blockDim.x)
                    tslice[sl * 65 * 32 + t] = __ldg(tables + tb + (int64_t)(t >> 5) * Nf + ph0 + (t & 31));
                __syncthreads();
                if (threadIdx.x == 0) slot_tab[sl] = tb;
                __syncthreads();
            }
        }
        // 1. contributions of the chunk's images: warp w takes images
        //    w, w + 8, ... in groups of F64_G evaluated together
        for (int kb = warp; kb < cn; kb += F64_WARPS * F64_G) {
            double d[F64_G], acc[F64_G];
            const double* cp[F64_G];
            const double* tp[F64_G];
            int64_t base[F64_G], nc[F64_G], fac[F64_G], phase[F64_G];
            bool dec[F64_G], fast[F64_G];
            const double* ts[F64_G];  // the member's table slice in shared memory
#pragma unroll
            for (int g = 0; g < F64_G; ++g) {
                const int k = kb + g * F64_WARPS;
                dec[g] = fast[g] = false;
                ts[g] = tslice + lane;
                d[g] = 0.0;
                acc[g] = 0.0;
                cp[g] = tp[g] = nullptr;
                base[g] = nc[g] = phase[g] = 0;
                fac[g] = 1;
                if (k < cn) {
                    const mvb_image& im = imgs[c0 + k];
                    if (im.factor == 1) {
                        d[g] = exact_distance(im.off[0], im.off[1], im.off[2], (double)im.sign[0],
                                              (double)im.sign[1], (double)im.sign[2], P, Q);
                    } else {
                        dec[g] = true;
                        cp[g] = coarse + im.coarse;
                        tp[g] = tables + im.table;
                        nc[g] = im.n_coarse;
                        fac[g] = im.factor;
                        base[g] = m / fac[g];
                        phase[g] = m - base[g] * fac[g];
                        // warp-uniform: the tile's 32 samples share one coarse
                        // interval (N % 32 == 0, 32-aligned tiles, all before
                        // the track end) and the 65-sample window needs no clamp
                        // ... and the factor's table slice is cached
                        const int sl = slot_tab[0] == im.table ? 0 : (slot_tab[1] == im.table ? 1 : -1);
                        fast[g] = sl >= 0 && (im.factor % 32 == 0) && tile_in_track &&
                                  (n0 / im.factor) >= 32 && (n0 / im.factor) + 32 < im.n_coarse;
                        if (fast[g]) ts[g] = tslice + sl * 65 * 32 + lane;
                    }
                }
            }
            // the 65-tap upsample of _kernels.py:169-180 (exact_upsample):
            // the clamp-free members as F64_G independent chains (each in the
            // reference's tap order; other members run a dummy chain on a
            // valid address, discarded), then the rare clamped members alone
            {
                double* ws = wwin + warp * (F64_G * F64_WIN);
                __syncwarp();  // the previous group's tap loop is done with ws
#pragma unroll
                for (int g = 0; g < F64_G; ++g) {
                    if (!fast[g]) continue;  // warp-uniform
                    const double* src = cp[g] + (base[g] - 32);
                    for (int c = lane; c < 65; c += 32) ws[g * F64_WIN + c] = __ldg(src + c);
                }
                __syncwarp();
                const double* w[F64_G];
#pragma unroll
                for (int g = 0; g < F64_G; ++g) w[g] = ws + g * F64_WIN;
                // members of one factor (the common case: a tier is contiguous
                // in the canonical order) read the same table slice: one
                // shared-memory load per tap serves all F64_G chains (the
                // slice loads were half of the kernel's data-pipe wavefronts)
                bool one_slice = true;
#pragma unroll
                for (int g = 1; g < F64_G; ++g) one_slice = one_slice && (!fast[g] || ts[g] == ts[0]);
                if (one_slice) {
                    const double* t0 = ts[0];
#pragma unroll 5
                    for (int col = 0; col < 65; ++col) {
                        const double tv = t0[col * 32];
#pragma unroll
                        for (int g = 0; g < F64_G; ++g) {
                            MVB_CHECK(!fast[g] || (base[g] - 32 + col >= 0 && base[g] - 32 + col < nc[g]),
                                      CHK_EXACT_INDEX);
                            acc[g] = xadd(acc[g], xmul(tv, w[g][col]));
                        }
                    }
                } else {
#pragma unroll 5
                    for (int col = 0; col < 65; ++col) {
#pragma unroll
                        for (int g = 0; g < F64_G; ++g) {
                            MVB_CHECK(!fast[g] || (base[g] - 32 + col >= 0 && base[g] - 32 + col < nc[g]),
                                      CHK_EXACT_INDEX);
                            acc[g] = xadd(acc[g], xmul(ts[g][col * 32], w[g][col]));
                        }
                    }
                }
            }
#pragma unroll
            for (int g = 0; g < F64_G; ++g)
                if (dec[g] && !fast[g]) acc[g] = exact_upsample(cp[g], nc[g], tp[g], fac[g], m);
#pragma unroll
            for (int g = 0; g < F64_G; ++g) {
                const int k = kb + g * F64_WARPS;
                if (k >= cn) continue;
                if (dec[g]) d[g] = acc[g];
                const mvb_image& im = imgs[c0 + k];
                const double tau = xdiv(xmul(J.rate, d[g]), J.c);
                const double amp = xdiv(im.beta, xmul(four_pi, d[g] > J.d_min ? d[g] : J.d_min));
                const double shifted = xadd(tau, L);
                const double d_int = floor(xsub(shifted, d0));
                const double mu = xsub(xsub(shifted, d0), d_int);
                const int64_t idx = n + J.L - (int64_t)d_int;
                double c = 0.0;
                if (idx >= 0 && idx < J.ls) {
                    double h = V[(int64_t)(J.nb - 1) * J.ls + idx];
                    for (int b = J.nb - 2; b >= 0; --b) h = xadd(xmul(h, mu), V[(int64_t)b * J.ls + idx]);
                    c = xmul(amp, h);
                }
                contrib[k * 32 + lane] = c;
            }
        }
        __syncthreads();
        // 2. block sums, sequential over each block's images
        const int nblk = (cn + 31) / 32;
        if (warp < nblk) {
            const int k1 = (warp + 1) * 32 < cn ? (warp + 1) * 32 : cn;
            double sum = 0.0;
            for (int k = warp * 32; k < k1; ++k) sum = xadd(sum, contrib[k * 32 + lane]);
            bsum[warp * 32 + lane] = sum;
        }
        __syncthreads();
        // 3. pairwise tree: aligned power-of-two subtrees of the chunk's blocks
        if (warp == 0) {
            int off = 0;
            for (int k = F64_LOG_CHUNK; k >= 0; --k) {
                const int size = 1 << k;
                if (!(nblk & size)) continue;
                for (int step = 1; step < size; step <<= 1)
                    for (int b = off; b < off + size; b += 2 * step)
                        bsum[b * 32 + lane] = xadd(bsum[b * 32 + lane], bsum[(b + step) * 32 + lane]);
                merge_push(st_v, st_l, sp, bsum[off * 32 + lane], k);
                off += size;
            }
        }
        __syncthreads();  // contrib / bsum are rewritten by the next chunk
    }
    if (warp == 0 && valid) {
        double v = sp > 0 ? st_v[--sp] : 0.0;
        while (sp > 0) v = xadd(st_v[--sp], v);
        out[J.out_off + n] = v;
    }
}

}  // namespace mvb

using namespace mvb;

template <int MINB, int G>
static int launch_f64(const mvb_job* jobs, int64_t n_jobs, int64_t max_out_len,
                      const mvb_image* images, const double* coarse, const double* tables,
                      const double* streams, const double* paths, double* out, void* stream) {
    static bool attr = false;  // one opt-in per process and instantiation
    if (!attr) {
        if (cudaFuncSetAttribute(k_synth_f64<MINB, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)f64_smem_bytes(G)) != cudaSuccess)
            return check_launch("synthesize_f64 (smem attribute)");
        attr = true;
    }
    dim3 g(grid_for(max_out_len, 32), (unsigned)n_jobs);
    prefer_carveout((const void*)k_synth_f64<MINB, G>);
    k_synth_f64<MINB, G><<<g, F64_WARPS * 32, f64_smem_bytes(G), as_stream(stream)>>>(
        jobs, images, coarse, tables, streams, paths, out);
    return check_launch("synthesize_f64");
}

extern "C" {

#ifdef MVB_CHECKED
void mvb_check_collect_synth(int64_t* h) { mvb_check_collect(h); }
#endif

int mvb_branch_records_f32(const float* x_all, const int64_t* sig_off, const int64_t* sig_len,
                           const int64_t* sig_row0, const int64_t* sig_zlo,
                           const int64_t* sig_zhi, int64_t n_sig, int64_t max_rows,
                           const double* cb, int M1, int L, int nb, float* rec, void* stream) {
    if (n_sig < 0 || n_sig > 65535 || max_rows < 1 || L < 1 || L > 128 || M1 < 1 || M1 > nb)
        return fail(MVB_EINVAL, "branch_records: sizes");
    if (n_sig == 0) return MVB_OK;
    if (!x_all || !sig_off || !sig_len || !sig_row0 || !cb || !rec ||
        ((sig_zlo == nullptr) != (sig_zhi == nullptr)))
        return fail(MVB_EINVAL, "branch_records: null");
    const int block = 256;
    const size_t smem = sizeof(float) * (BR_Q * block + L - 1);
    const dim3 g(grid_for(max_rows, BR_Q * block), (unsigned)n_sig);
    cudaStream_t s = as_stream(stream);
#define MVB_BR(NP) prefer_carveout((const void*)k_branch_records_f32<NP>); \
    k_branch_records_f32<NP><<<g, block, smem, s>>>(x_all, sig_off, sig_len, \
                                                                   sig_row0, sig_zlo, sig_zhi, \
                                                                   cb, M1, L, rec)
    switch (nb) {
        case 4: MVB_BR(1); break;
        case 8: MVB_BR(2); break;
        case 12: MVB_BR(3); break;
        case 16: MVB_BR(4); break;
        default: return fail(MVB_EINVAL, "branch_records: nb must be 4, 8, 12 or 16");
    }
#undef MVB_BR
    return check_launch("branch_records_f32");
}

static int synthesize_f32(const mvb_job* jobs, const mvb_work* work, int64_t n_work,
                          const mvb_image* images, const mvb_coef32* coef, const float* rec,
                          const double* paths, float* out, float* part, int nb, int u_steps,
                          const RangeArgs& ra, void* stream) {
    if (n_work < 0 || n_work > 0x7fffffff) return fail(MVB_EINVAL, "synthesize_f32: n_work");
    if (n_work == 0) return MVB_OK;
    if (!jobs || !work || !images || !rec || !paths || !out)
        return fail(MVB_EINVAL, "synthesize_f32: null");
    if (u_steps != 16) return fail(MVB_EINVAL, "synthesize_f32: u_steps must be 16");
    cudaStream_t s = as_stream(stream);
    const unsigned g = (unsigned)n_work;
    const int block = SYNTH_WARPS * 32;
    // U = 16: 512-sample tiles, 3 CTAs/SM
#define MVB_SYNTH(U, NP, MB) prefer_carveout((const void*)k_synth_f32<U, NP, MB>, true); \
    k_synth_f32<U, NP, MB><<<g, block, 0, s>>>( \
        jobs, work, images, coef, rec, paths, out, part, ra)
#define MVB_SYNTH_NB(U, MB)                         \
    switch (nb) {                                   \
        case 4: MVB_SYNTH(U, 1, MB); break;         \
        case 8: MVB_SYNTH(U, 2, MB); break;         \
        case 12: MVB_SYNTH(U, 3, MB); break;        \
        case 16: MVB_SYNTH(U, 4, MB); break;        \
        default: return fail(MVB_EINVAL, "synthesize_f32: nb must be 4, 8, 12 or 16"); \
    }
    MVB_SYNTH_NB(16, 3)
#undef MVB_SYNTH_NB
#undef MVB_SYNTH
    return check_launch("synthesize_f32");
}

int mvb_synthesize_f32(const mvb_job* jobs, const mvb_work* work, int64_t n_work,
                       const mvb_image* images, const mvb_coef32* coef, const float* rec,
                       const double* paths, float* out, float* part, int nb, int u_steps,
                       void* stream) {
    return synthesize_f32(jobs, work, n_work, images, coef, rec, paths, out, part, nb, u_steps,
                          RangeArgs{nullptr, nullptr, 1, 1, 1, 0}, stream);
}

int mvb_synthesize_f32_ranged(const mvb_job* jobs, const mvb_work* work, int64_t n_work,
                              const mvb_image* images, const uint32_t* keys, int64_t run_len,
                              int64_t seg_len, int max_factor, const double* bbox,
                              const mvb_coef32* coef, const float* rec, const double* paths,
                              float* out, float* part, int nb, int u_steps, void* stream) {
    if (!keys || !bbox) return fail(MVB_EINVAL, "synthesize_f32_ranged: null keys / bbox");
    if (run_len < 1 || run_len > 0x7fffffff || seg_len < 1 || seg_len > 0x7fffffff ||
        max_factor < 1)
        return fail(MVB_EINVAL, "synthesize_f32_ranged: run_len / seg_len / max_factor");
    return synthesize_f32(jobs, work, n_work, images, coef, rec, paths, out, part, nb, u_steps,
                          RangeArgs{keys, bbox, (int)run_len, (int)seg_len, max_factor, 0}, stream);
}

// Measurement variant: the ranged synthesis with the branch-record gathers
// (or every other step's) through the texture pipe.  The texture object of
// (rec, rec_floats) is created once and cached (never destroyed: a
// diagnostic entry point).
int mvb_synthesize_f32_tex(const mvb_job* jobs, const mvb_work* work, int64_t n_work,
                           const mvb_image* images, const uint32_t* keys, int64_t run_len,
                           int64_t seg_len, int max_factor, const double* bbox,
                           const mvb_coef32* coef, const float* rec, int64_t rec_floats,
                           const double* paths, float* out, float* part, int nb, int mode,
                           void* stream) {
    if (nb != 8 || (mode != 1 && mode != 2) || !keys || !bbox || rec_floats < 8 ||
        rec_floats / 4 > 0x7fffffff)
        return fail(MVB_EINVAL, "synthesize_f32_tex: nb 8, mode 1/2, keys, bbox, size");
    if (n_work <= 0) return MVB_OK;
    static std::mutex mu;
    static std::vector<std::pair<std::pair<const float*, int64_t>, cudaTextureObject_t>> cache;
    cudaTextureObject_t tex = 0;
    {
        std::lock_guard<std::mutex> lk(mu);
        for (auto& e : cache)
            if (e.first.first == rec && e.first.second == rec_floats) tex = e.second;
        if (!tex) {
            cudaResourceDesc rd{};
            rd.resType = cudaResourceTypeLinear;
            rd.res.linear.devPtr = const_cast<float*>(rec);
            rd.res.linear.desc = cudaCreateChannelDesc<float4>();
            rd.res.linear.sizeInBytes = (size_t)rec_floats * sizeof(float);
            cudaTextureDesc td{};
            td.readMode = cudaReadModeElementType;
            // allowed inside a (render plan's) stream capture
            cudaStreamCaptureMode m = cudaStreamCaptureModeRelaxed;
            cudaThreadExchangeStreamCaptureMode(&m);
            const cudaError_t e = cudaCreateTextureObject(&tex, &rd, &td, nullptr);
            cudaThreadExchangeStreamCaptureMode(&m);
            if (e != cudaSuccess) return fail(MVB_ECUDA, cudaGetErrorString(e));
            cache.push_back({{rec, rec_floats}, tex});
        }
    }
    const RangeArgs ra{keys, bbox, (int)run_len, (int)seg_len, max_factor, tex};
    cudaStream_t s = as_stream(stream);
    if (mode == 1) {
        prefer_carveout((const void*)k_synth_f32<16, 2, 3, false, 1>, true);
        k_synth_f32<16, 2, 3, false, 1><<<(unsigned)n_work, SYNTH_WARPS * 32, 0, s>>>(
            jobs, work, images, coef, rec, paths, out, part, ra);
    } else {
        prefer_carveout((const void*)k_synth_f32<16, 2, 3, false, 2>, true);
        k_synth_f32<16, 2, 3, false, 2><<<(unsigned)n_work, SYNTH_WARPS * 32, 0, s>>>(
            jobs, work, images, coef, rec, paths, out, part, ra);
    }
    return check_launch("synthesize_f32_tex");
}

#ifdef MVB_CTA_TIMING
int mvb_cta_timing(unsigned long long* host, int n) {
    if (n > 4 * 65536) n = 4 * 65536;
    return cudaMemcpyFromSymbol(host, g_cta_time, sizeof(unsigned long long) * n) == cudaSuccess
               ? MVB_OK : fail(MVB_ECUDA, "cta_timing");
}
#endif

int mvb_signal_plane_f32(const float* x_all, const int64_t* sig_off, const int64_t* sig_len,
                         const int64_t* sig_row0, int64_t n_sig, int64_t max_len, float* xp,
                         void* stream) {
    if (n_sig < 0 || n_sig > 65535 || max_len < 0) return fail(MVB_EINVAL, "signal_plane: sizes");
    if (n_sig == 0 || max_len == 0) return MVB_OK;
    if (!x_all || !sig_off || !sig_len || !sig_row0 || !xp) return fail(MVB_EINVAL, "signal_plane: null");
    unsigned gx = grid_for(max_len, 256);
    if (gx > 4096) gx = 4096;
    prefer_carveout((const void*)k_signal_plane);
    k_signal_plane<<<dim3(gx, (unsigned)n_sig), 256, 0, as_stream(stream)>>>(x_all, sig_off, sig_len,
                                                                              sig_row0, xp);
    return check_launch("signal_plane_f32");
}

int mvb_synthesize_f32_table(const mvb_job* jobs, const mvb_work* work, int64_t n_work,
                             const mvb_image* images, const mvb_coef32* coef, const float* xp,
                             const double* paths, float* out, float* part, const float* table,
                             int L, void* stream) {
    if (n_work < 0 || n_work > 0x7fffffff) return fail(MVB_EINVAL, "synthesize_f32_table: n_work");
    if (n_work == 0) return MVB_OK;
    if (!jobs || !work || !images || !xp || !paths || !out || !table)
        return fail(MVB_EINVAL, "synthesize_f32_table: null");
    if (L < 1 || L > 128) return fail(MVB_EINVAL, "synthesize_f32_table: L");
    const size_t smem = sizeof(float) * (size_t)(TAB_P + 1) * (L + 1);
    if (cudaFuncSetAttribute(k_synth_f32<16, 1, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
        return check_launch("synthesize_f32_table (smem attribute)");
    prefer_carveout((const void*)k_synth_f32<16, 1, 1, true>);
    k_synth_f32<16, 1, 1, true><<<(unsigned)n_work, SYNTH_WARPS * 32, smem, as_stream(stream)>>>(
        jobs, work, images, coef, xp, paths, out, part, RangeArgs{nullptr, nullptr, 1, 1, 1, 0}, table);
    return check_launch("synthesize_f32_table");
}

int mvb_reduce_partials_f32(const mvb_job* jobs, int64_t n_jobs, int64_t max_out_len,
                            const float* part, float* out, void* stream) {
    if (n_jobs < 0 || n_jobs > 65535 || max_out_len < 0) return fail(MVB_EINVAL, "reduce: sizes");
    if (n_jobs == 0 || max_out_len == 0) return MVB_OK;
    unsigned gx = grid_for(max_out_len, 256);
    if (gx > 1024) gx = 1024;
    prefer_carveout((const void*)k_reduce_f32);
    k_reduce_f32<<<dim3(gx, (unsigned)n_jobs), 256, 0, as_stream(stream)>>>(jobs, part, out);
    return check_launch("reduce_partials_f32");
}

int mvb_synthesize_f64_ex(const mvb_job* jobs, int64_t n_jobs, int64_t max_out_len,
                          const mvb_image* images, const double* coarse, const double* tables,
                          const double* streams, const double* paths, double* out,
                          int64_t max_images, void* stream) {
    if (n_jobs < 0 || n_jobs > 65535 || max_out_len < 0) return fail(MVB_EINVAL, "synthesize_f64: sizes");
    if (n_jobs == 0 || max_out_len == 0) return MVB_OK;
    if (!jobs || !images || !streams || !paths || !out)
        return fail(MVB_EINVAL, "synthesize_f64: null");
    // chains per warp / CTAs per SM: four chains at 2 CTAs/SM (126
    // registers) for small image sets (c1: 0.142 ms vs 0.147), two chains at
    // 3 CTAs/SM (80 registers, no spills) from 1024 images on (c3 fp64 -6%);
    // MVB_F64_VARIANT = 4 / 2 forces one
    static const int forced = [] {
        const char* e = getenv("MVB_F64_VARIANT");
        return e ? atoi(e) : 0;
    }();
    const int g = forced == 2 || forced == 4 ? forced : (max_images >= 1024 ? 2 : 4);
    if (g == 2)
        return launch_f64<3, 2>(jobs, n_jobs, max_out_len, images, coarse, tables, streams, paths,
                                out, stream);
    return launch_f64<2, 4>(jobs, n_jobs, max_out_len, images, coarse, tables, streams, paths, out,
                            stream);
}

int mvb_synthesize_f64(const mvb_job* jobs, int64_t n_jobs, int64_t max_out_len,
                       const mvb_image* images, const double* coarse, const double* tables,
                       const double* streams, const double* paths, double* out, void* stream) {
    return mvb_synthesize_f64_ex(jobs, n_jobs, max_out_len, images, coarse, tables, streams, paths,
                                 out, 0, stream);
}

}  // extern "C"
