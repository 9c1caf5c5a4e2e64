// Single-call render of one (scene, channel) job -- the C counterpart of
// the reference's render()/synthesize() pair (synth.py:291-294, 194-258)
// for hosts that bind the C ABI directly.
//
// mvb_render_tracks_and_synthesize runs the fast (fp32, fp64-anchored)
// engine end to end on the caller's stream from device inputs: image
// enumeration, image records, coarse tracks and their bounds, the exact
// track maximum (-> the reference's out_len), interval records, the
// per-segment delay sort, branch records, the synthesis and the partial
// reduction -- the same kernels and the same plan (tiling, chunking,
// record pads) as the Python engine (engine.py Geometry + prepare_render).
// The host-side constants it needs are computed here: the refit of each
// factor's phase table (trajectory.py phase_fit, least squares by
// Householder QR), the centred Farrow bank and its degree-7 reduction
// (engine.py _fast_bank), the image classes of the tier table.
//
// What stays with the caller, as in the reference: the decimation itself
// (trajectory.py:279-298 decimate(), including its conditional anti-alias
// low-pass) -- the caller passes each decimated tier's coarse source (and
// receiver) path -- and the reference's phase table of each factor
// (trajectory.py:235-257 _phase_table), so out_len is bit-exact.
//
// The call synchronizes the stream once: after the track maximum, whose
// value fixes out_len and with it the tiling.  Scratch memory is
// stream-ordered (cudaMallocAsync / cudaFreeAsync).
#include <algorithm>
#include <cmath>
#include <vector>

#include "mvb_common.cuh"

namespace mvb {
namespace {

constexpr int TILE = 512;           // mvb_synthesize_f32 u_steps = 16
constexpr int SEG_LEN = 32 * TILE;  // delay-sort segment (engine.SEG_LEN)
constexpr int PAD_MARGIN = 64;
constexpr int CHUNK_MIN_IMAGES = 320;        // engine.py CHUNK_MIN_IMAGES
constexpr int SMALL_GRID_TILES = 512, SMALL_GRID_CHUNK_MIN = 160;  // engine.py _chunking
constexpr int FIT_DEGREE = 8;

// least squares min ||A x - b|| for every column of B (m x k), A (m x n)
// row-major, m >= n: Householder QR, then back substitution.  Returns X
// (n x k) row-major.
std::vector<double> lstsq(std::vector<double> A, int m, int n, std::vector<double> B, int k) {
    for (int j = 0; j < n; ++j) {
        double norm = 0.0;
        for (int i = j; i < m; ++i) norm += A[i * n + j] * A[i * n + j];
        norm = std::sqrt(norm);
        if (norm == 0.0) continue;
        const double alpha = A[j * n + j] > 0 ? -norm : norm;
        std::vector<double> v(m, 0.0);
        for (int i = j; i < m; ++i) v[i] = A[i * n + j];
        v[j] -= alpha;
        double vv = 0.0;
        for (int i = j; i < m; ++i) vv += v[i] * v[i];
        if (vv == 0.0) continue;
        for (int c = j; c < n; ++c) {
            double s = 0.0;
            for (int i = j; i < m; ++i) s += v[i] * A[i * n + c];
            s = 2.0 * s / vv;
            for (int i = j; i < m; ++i) A[i * n + c] -= s * v[i];
        }
        for (int c = 0; c < k; ++c) {
            double s = 0.0;
            for (int i = j; i < m; ++i) s += v[i] * B[i * k + c];
            s = 2.0 * s / vv;
            for (int i = j; i < m; ++i) B[i * k + c] -= s * v[i];
        }
    }
    std::vector<double> X((size_t)n * k, 0.0);
    for (int c = 0; c < k; ++c)
        for (int j = n - 1; j >= 0; --j) {
            double s = B[j * k + c];
            for (int q = j + 1; q < n; ++q) s -= A[j * n + q] * X[q * k + c];
            X[j * k + c] = A[j * n + j] != 0.0 ? s / A[j * n + j] : 0.0;
        }
    return X;
}

// (FIT_DEGREE + 1, 65) refit of a factor's (N, 65) phase table in
// u = 2r/N - 1 (trajectory.py phase_fit)
std::vector<double> phase_fit(const double* tab, int N) {
    const int P = FIT_DEGREE + 1;
    std::vector<double> V((size_t)N * P), B(tab, tab + (size_t)N * 65);
    for (int r = 0; r < N; ++r) {
        const double u = 2.0 * r / N - 1.0;
        double p = 1.0;
        for (int q = 0; q < P; ++q, p *= u) V[r * P + q] = p;
    }
    if (N >= P) return lstsq(V, N, P, B, 65);
    // N < 9 phases: the minimum-norm solution (numpy lstsq's), X = V^T Y with
    // (V V^T) Y = B
    std::vector<double> G((size_t)N * N, 0.0);
    for (int i = 0; i < N; ++i)
        for (int j = 0; j < N; ++j)
            for (int q = 0; q < P; ++q) G[i * N + j] += V[i * P + q] * V[j * P + q];
    std::vector<double> Y = lstsq(G, N, N, B, 65);
    std::vector<double> X((size_t)P * 65, 0.0);
    for (int q = 0; q < P; ++q)
        for (int c = 0; c < 65; ++c)
            for (int i = 0; i < N; ++i) X[q * 65 + c] += V[i * P + q] * Y[i * 65 + c];
    return X;
}

double negative_mass(const double* tab, int N) {
    double worst = 0.0;
    for (int r = 0; r < N; ++r) {
        double s = 0.0;
        for (int c = 0; c < 65; ++c) s += tab[r * 65 + c] < 0 ? -tab[r * 65 + c] : 0.0;
        worst = std::max(worst, s);
    }
    return worst;
}

// centred Farrow bank c'_k with sum_k c'_k (mu - 1/2)^k == sum_k c_k mu^k
// (farrow.py centered_branches), reduced to degree 7 when that changes no
// tap by more than 5e-7 of the largest (engine.py _fast_bank)
std::vector<double> fast_bank(const double* br, int M1, int L, int& M1_out, int& nb) {
    std::vector<double> cb((size_t)M1 * L, 0.0);
    std::vector<double> binom(M1 * M1, 0.0);
    for (int j = 0; j < M1; ++j) {
        binom[j * M1 + 0] = 1.0;
        for (int k = 1; k <= j; ++k)
            binom[j * M1 + k] = binom[(j - 1) * M1 + k - 1] + (k < j ? binom[(j - 1) * M1 + k] : 0.0);
    }
    for (int j = 0; j < M1; ++j)
        for (int k = 0; k <= j; ++k) {
            const double w = binom[j * M1 + k] * std::pow(0.5, j - k);
            for (int t = 0; t < L; ++t) cb[k * L + t] += br[j * L + t] * w;
        }
    M1_out = M1;
    if (M1 > 8) {
        const int G = 256, D = 8;
        std::vector<double> h((size_t)G * L, 0.0), V((size_t)G * D);
        for (int i = 0; i < G; ++i) {
            const double mu = 0.5 - 0.5 * std::cos(M_PI * (i + 0.5) / G), u = mu - 0.5;
            double p = 1.0;
            for (int k = 0; k < M1; ++k, p *= u)
                for (int t = 0; t < L; ++t) h[i * L + t] += p * cb[k * L + t];
            // Chebyshev basis T_q(2u)
            const double x = 2.0 * u;
            double t0 = 1.0, t1 = x;
            for (int q = 0; q < D; ++q) {
                V[i * D + q] = q == 0 ? 1.0 : (q == 1 ? x : 0.0);
                if (q >= 2) {
                    const double t2 = 2.0 * x * t1 - t0;
                    V[i * D + q] = t2;
                    t0 = t1;
                    t1 = t2;
                }
            }
        }
        std::vector<double> ch = lstsq(V, G, D, h, L);  // (D, L) Chebyshev coefficients
        // Chebyshev -> monomials in x = 2u -> monomials in u (x^p = 2^p u^p)
        std::vector<double> Tm((size_t)D * D, 0.0);  // Tm[q][p]: coefficient of x^p in T_q
        Tm[0] = 1.0;
        if (D > 1) Tm[1 * D + 1] = 1.0;
        for (int q = 2; q < D; ++q)
            for (int p = 0; p < D; ++p)
                Tm[q * D + p] = (p > 0 ? 2.0 * Tm[(q - 1) * D + p - 1] : 0.0) - Tm[(q - 2) * D + p];
        std::vector<double> red((size_t)D * L, 0.0);
        for (int p = 0; p < D; ++p)
            for (int t = 0; t < L; ++t) {
                double s = 0.0;
                for (int q = 0; q < D; ++q) s += Tm[q * D + p] * ch[q * L + t];
                red[p * L + t] = s * std::pow(2.0, p);
            }
        double err = 0.0, big = 0.0;
        for (int i = 0; i <= 2000; ++i) {
            const double u = -0.5 + i / 2000.0;
            for (int t = 0; t < L; ++t) {
                double ex = 0.0, ap = 0.0, p = 1.0;
                for (int k = 0; k < M1; ++k, p *= u) ex += p * cb[k * L + t];
                p = 1.0;
                for (int k = 0; k < D; ++k, p *= u) ap += p * red[k * L + t];
                err = std::max(err, std::fabs(ex - ap));
                big = std::max(big, std::fabs(ex));
            }
        }
        if (err <= 5e-7 * big) {
            cb = red;
            M1_out = D;
        }
    }
    nb = M1_out <= 4 ? 4 : M1_out <= 8 ? 8 : M1_out <= 12 ? 12 : 16;
    return cb;
}

int64_t count_order(int o) { return o == 0 ? 1 : 4LL * o * o + 2; }

struct Scratch {
    cudaStream_t s;
    std::vector<void*> blocks;
    explicit Scratch(cudaStream_t st) : s(st) {}
    ~Scratch() {
        for (void* p : blocks) cudaFreeAsync(p, s);
    }
    template <class T>
    T* get(size_t n) {
        void* p = nullptr;
        if (cudaMallocAsync(&p, std::max<size_t>(n, 1) * sizeof(T), s) != cudaSuccess) return nullptr;
        blocks.push_back(p);
        return static_cast<T*>(p);
    }
};

#define MVB_TRY(call)                 \
    do {                              \
        const int rc__ = (call);      \
        if (rc__ != MVB_OK) return rc__; \
    } while (0)
#define MVB_CUDA(call)                                                               \
    do {                                                                             \
        const cudaError_t e__ = (call);                                              \
        if (e__ != cudaSuccess) return fail(MVB_ECUDA, std::string("render: ") +      \
                                                           cudaGetErrorString(e__)); \
    } while (0)

}  // namespace
}  // namespace mvb

using namespace mvb;

extern "C" int mvb_render_tracks_and_synthesize(const mvb_render_args* a, float* d_out,
                                                int64_t out_capacity, int64_t* h_out_len,
                                                void* stream) {
    // ---- validation (the reference's ValueErrors are the Python layer's;
    // here: shapes and ranges) ----
    if (!a || !h_out_len) return fail(MVB_EINVAL, "render: null args");
    if (!a->d_signal || a->n_signal < 1) return fail(MVB_EINVAL, "render: empty signal");
    if (!a->d_pos || a->T < 1 || !a->d_mic) return fail(MVB_EINVAL, "render: path / receiver");
    if (a->max_order < 0 || a->max_order > 40) return fail(MVB_EINVAL, "render: max_order");
    if (a->n_tiers < 1 || a->n_tiers > MVB_MAX_CLASSES) return fail(MVB_EINVAL, "render: n_tiers");
    if (!a->h_branches || a->branch_len < 1 || a->branch_len > 128 || a->poly_order < 0 ||
        a->poly_order > 15 || a->nominal_delay < 0 || a->nominal_delay >= a->branch_len)
        return fail(MVB_EINVAL, "render: filter bank");
    if (!(a->rate > 0) || !(a->c > 0) || !(a->d_min > 0)) return fail(MVB_EINVAL, "render: rate/c/d_min");
    for (int t = 0; t < a->n_tiers; ++t) {
        if (a->tier_factor[t] < 1 || (t && a->tier_order[t] <= a->tier_order[t - 1]))
            return fail(MVB_EINVAL, "render: tier table (ascending orders, factors >= 1)");
        if (a->tier_factor[t] > 1 && (!a->d_coarse_pos[t] || !a->h_phase_table[t] ||
                                      (a->mic_moving && !a->d_coarse_mic[t])))
            return fail(MVB_EINVAL, "render: decimated tier needs coarse paths and its phase table");
    }
    if (a->tier_order[a->n_tiers - 1] < a->max_order) return fail(MVB_EINVAL, "render: tiers do not cover max_order");
    const int64_t S = mvb_image_count(a->max_order);
    if (S > MVB_DELAY_SORT_MAX) return fail(MVB_EINVAL, "render: more images than MVB_DELAY_SORT_MAX");
    cudaStream_t st = as_stream(stream);
    Scratch mem(st);
    const int64_t T = a->T, n = a->n_signal, L = a->branch_len, d0 = a->nominal_delay;
    const int mv = a->mic_moving ? 1 : 0;

    // ---- classes: distinct factors, images per class, prefix counts ----
    std::vector<int> factors;
    for (int t = 0; t < a->n_tiers; ++t)
        if (std::find(factors.begin(), factors.end(), a->tier_factor[t]) == factors.end())
            factors.push_back(a->tier_factor[t]);
    std::sort(factors.begin(), factors.end());
    const int nC = (int)factors.size();
    std::vector<int32_t> img_tab((size_t)S * (2 + nC));
    std::vector<int32_t> counts(nC, 0);
    {
        int64_t i = 0;
        for (int o = 0; o <= a->max_order; ++o) {
            int N = 1;
            for (int t = 0; t < a->n_tiers; ++t)
                if (o <= a->tier_order[t]) { N = a->tier_factor[t]; break; }
            const int c = (int)(std::find(factors.begin(), factors.end(), N) - factors.begin());
            for (int64_t q = 0; q < count_order(o); ++q, ++i) {
                int32_t* r = &img_tab[i * (2 + nC)];
                r[0] = (int32_t)i;
                r[1] = c;
                for (int k = 0; k < nC; ++k) r[2 + k] = counts[k];
                ++counts[c];
            }
        }
    }
    // ---- paths buffer: source rows, receiver rows, coarse rows per factor ----
    std::vector<int64_t> cpath(nC, 0);
    int64_t rows = T + (mv ? T : 1);
    for (int c = 0; c < nC; ++c)
        if (factors[c] > 1) {
            cpath[c] = rows;
            rows += ((T + factors[c] - 1) / factors[c]) * (1 + mv);
        }
    double* paths = mem.get<double>(3 * rows);
    if (!paths) return fail(MVB_ECUDA, "render: scratch allocation");
    MVB_CUDA(cudaMemcpyAsync(paths, a->d_pos, 24 * T, cudaMemcpyDeviceToDevice, st));
    MVB_CUDA(cudaMemcpyAsync(paths + 3 * T, a->d_mic, 24 * (mv ? T : 1), cudaMemcpyDeviceToDevice, st));
    for (int c = 0; c < nC; ++c) {
        if (factors[c] == 1) continue;
        int t = 0;
        while (a->tier_factor[t] != factors[c]) ++t;
        const int64_t K = (T + factors[c] - 1) / factors[c];
        MVB_CUDA(cudaMemcpyAsync(paths + 3 * cpath[c], a->d_coarse_pos[t], 24 * K,
                                 cudaMemcpyDeviceToDevice, st));
        if (mv)
            MVB_CUDA(cudaMemcpyAsync(paths + 3 * (cpath[c] + K), a->d_coarse_mic[t], 24 * K,
                                     cudaMemcpyDeviceToDevice, st));
    }
    // ---- factor constants: transposed tables (65, N), refits, negative mass ----
    std::vector<int64_t> table_off(nC, 0);
    std::vector<std::vector<double>> fits(nC);
    int64_t tab_len = 0;
    double negsum = 0.0;
    std::vector<double> tabT;
    for (int c = 0; c < nC; ++c) {
        const int N = factors[c];
        if (N == 1) continue;
        int t = 0;
        while (a->tier_factor[t] != N) ++t;
        const double* tab = a->h_phase_table[t];
        table_off[c] = tab_len;
        tabT.resize(tab_len + 65 * (int64_t)N);
        for (int col = 0; col < 65; ++col)
            for (int r = 0; r < N; ++r) tabT[tab_len + col * N + r] = tab[r * 65 + col];
        tab_len += 65 * (int64_t)N;
        fits[c] = phase_fit(tab, N);
        negsum = std::max(negsum, negative_mass(tab, N));
    }
    double* tables = mem.get<double>(std::max<int64_t>(tab_len, 1));
    if (tab_len) MVB_CUDA(cudaMemcpyAsync(tables, tabT.data(), 8 * tab_len, cudaMemcpyHostToDevice, st));
    // ---- image records (enumeration + classes) ----
    mvb_class_table ct{};
    ct.n = nC;
    int64_t sel_acc = 0, n_full = 0, coarse_total = 0;
    for (int c = 0; c < nC; ++c) {
        ct.factor[c] = factors[c];
        ct.fit[c] = c;
        ct.count[c] = counts[c];
        ct.table[c] = table_off[c];
        if (factors[c] > 1) {
            ct.sel_off[c] = sel_acc;
            sel_acc += counts[c];
            coarse_total += (int64_t)counts[c] * ((T + factors[c] - 1) / factors[c]);
        } else {
            n_full += counts[c];
        }
    }
    std::vector<int64_t> job_tab(4 + nC);
    job_tab[0] = 0;
    job_tab[1] = T;
    job_tab[2] = 0;
    job_tab[3] = 0;
    for (int c = 0; c < nC; ++c) job_tab[4 + c] = cpath[c];
    const double room[9] = {a->dims[0], a->dims[1], a->dims[2], a->walls[0], a->walls[1],
                            a->walls[2], a->walls[3], a->walls[4], a->walls[5]};
    double* d_room = mem.get<double>(9);
    double* toff = mem.get<double>(3 * S);
    double* tsgn = mem.get<double>(3 * S);
    double* tbeta = mem.get<double>(S);
    int32_t* d_img = mem.get<int32_t>(img_tab.size());
    int64_t* d_jobtab = mem.get<int64_t>(job_tab.size());
    mvb_image* images = mem.get<mvb_image>(S);
    int32_t* full_sel = mem.get<int32_t>(std::max<int64_t>(n_full, 1));
    int32_t* dec_sel = mem.get<int32_t>(std::max<int64_t>(S - n_full, 1));
    int32_t* class_sel = mem.get<int32_t>(std::max<int64_t>(sel_acc, 1));
    if (!d_room || !toff || !tsgn || !tbeta || !d_img || !d_jobtab || !images || !full_sel ||
        !dec_sel || !class_sel)
        return fail(MVB_ECUDA, "render: scratch allocation");
    MVB_CUDA(cudaMemcpyAsync(d_room, room, sizeof(room), cudaMemcpyHostToDevice, st));
    MVB_CUDA(cudaMemcpyAsync(d_img, img_tab.data(), 4 * img_tab.size(), cudaMemcpyHostToDevice, st));
    MVB_CUDA(cudaMemcpyAsync(d_jobtab, job_tab.data(), 8 * job_tab.size(), cudaMemcpyHostToDevice, st));
    MVB_TRY(mvb_enumerate(d_room, d_room + 3, 1, a->max_order, nullptr, nullptr, nullptr, tbeta,
                          toff, tsgn, stream));
    MVB_TRY(mvb_build_images(toff, tsgn, tbeta, S, d_img, S, d_jobtab, 1, &ct, 0, images, full_sel,
                             0, dec_sel, 0, class_sel, stream));
    // ---- job rows: geometry (canonical images) and synthesis (sorted) ----
    mvb_job J{};
    J.img_off = 0;
    J.n_img = S;
    J.pos_off = 0;
    J.mic_off = T;
    J.T = (int32_t)T;
    J.mic_moving = mv;
    J.L = (int32_t)L;
    J.d0 = (int32_t)d0;
    J.n_chunks = 1;
    J.rate = a->rate;
    J.c = a->c;
    J.d_min = a->d_min;
    J.kappa = a->rate / a->c;
    J.ls = n + L - 1;
    J.out_len = INT64_MAX / 4;  // capacity for finalize_lengths: the exact length is read back
    mvb_job* d_pre = mem.get<mvb_job>(1);
    if (!d_pre) return fail(MVB_ECUDA, "render: scratch allocation");
    MVB_CUDA(cudaMemcpyAsync(d_pre, &J, sizeof(J), cudaMemcpyHostToDevice, st));
    // ---- tracks: coarse distances + bounds, full-rate bounds, exact maximum ----
    double* coarse = mem.get<double>(std::max<int64_t>(coarse_total, 1));
    double* lb = mem.get<double>(S);
    double* ub = mem.get<double>(S);
    double* bbox = mem.get<double>(65 * 16);
    int64_t* box_rows = mem.get<int64_t>(4);
    int32_t* scratch = mem.get<int32_t>(MVB_EXACT_LIST_WORDS + S + 2);
    double* dmax = mem.get<double>(1);
    int64_t* d_len = mem.get<int64_t>(1);
    int32_t* d_err = mem.get<int32_t>(1);
    if (!coarse || !lb || !ub || !bbox || !box_rows || !scratch || !dmax || !d_len || !d_err)
        return fail(MVB_ECUDA, "render: scratch allocation");
    const int64_t rows4[4] = {0, T, T, mv};
    MVB_CUDA(cudaMemcpyAsync(box_rows, rows4, sizeof(rows4), cudaMemcpyHostToDevice, st));
    MVB_CUDA(cudaMemsetAsync(lb, 0, 8 * S, st));
    MVB_CUDA(cudaMemsetAsync(ub, 0, 8 * S, st));
    MVB_CUDA(cudaMemsetAsync(d_err, 0, 4, st));
    MVB_TRY(mvb_path_bbox(box_rows, 1, paths, bbox, stream));
    for (int c = 0; c < nC; ++c)
        if (factors[c] > 1)
            MVB_TRY(mvb_coarse_distances(images, class_sel + ct.sel_off[c], counts[c],
                                         (T + factors[c] - 1) / factors[c], d_pre, paths, negsum,
                                         coarse, lb, ub, stream));
    if (n_full)
        MVB_TRY(mvb_track_bounds(images, full_sel, n_full, d_pre, paths, bbox, lb, ub, stream));
    MVB_TRY(mvb_track_max(images, d_pre, 1, coarse_total ? coarse : nullptr, tables, paths, negsum,
                          lb, ub, scratch, dmax, stream));
    MVB_TRY(mvb_finalize_lengths(d_pre, 1, dmax, d_len, d_err, stream));
    int64_t out_len = 0;
    MVB_CUDA(cudaMemcpyAsync(&out_len, d_len, 8, cudaMemcpyDeviceToHost, st));
    MVB_CUDA(cudaStreamSynchronize(st));  // the one host wait: out_len fixes the tiling
    *h_out_len = out_len;
    if (!d_out || out_len > out_capacity)
        return fail(MVB_EINVAL, "render: output capacity " + std::to_string(out_capacity) +
                                    " < out_len " + std::to_string(out_len) + " (*h_out_len)");
    const int64_t tau_ceil = out_len - n - L;
    // ---- interval records, one launch per decimation factor ----
    mvb_coef32* coef = mem.get<mvb_coef32>(std::max<int64_t>(coarse_total, 1));
    if (!coef) return fail(MVB_ECUDA, "render: scratch allocation");
    for (int c = 0; c < nC; ++c)
        if (factors[c] > 1)
            MVB_TRY(mvb_track_coeffs(images, class_sel + ct.sel_off[c], counts[c],
                                     (T + factors[c] - 1) / factors[c], d_pre, coarse,
                                     fits[c].data(), coef, stream));
    // ---- delay sort per time segment ----
    const int64_t n_seg = (T + SEG_LEN - 1) / SEG_LEN;
    mvb_image* sorted = mem.get<mvb_image>(n_seg * S);
    uint32_t* keys = mem.get<uint32_t>(n_seg * S);
    if (!sorted || !keys) return fail(MVB_ECUDA, "render: scratch allocation");
    int key_bits = 1;
    while (key_bits < 32 && (tau_ceil + 2) >= (1LL << key_bits)) ++key_bits;
    // keyed: the synthesis narrows every tile to its active images
    MVB_TRY(mvb_delay_sort_keyed(images, d_pre, 1, S, n_seg, SEG_LEN, paths, coarse, key_bits, 0,
                                 sorted, keys, stream));
    // ---- branch records: [front pad | n + L - 1 rows | back pad] ----
    int M1 = 0, nb = 0;
    std::vector<double> cb = fast_bank(a->h_branches, a->poly_order + 1, (int)L, M1, nb);
    const int64_t front = tau_ceil + 1 + L + PAD_MARGIN;
    const int64_t back = front + TILE + PAD_MARGIN;
    const int64_t rec_rows = front + n + L - 1 + back;
    if (rec_rows + n + tau_ceil + 2 * L >= (1LL << 31) - 0x4B400000LL)
        return fail(MVB_EINVAL, "render: signal too long for 32-bit record rows");
    const int64_t row_floats = nb == 4 ? 4 : 8 * ((nb + 7) / 8);
    float* rec = mem.get<float>(rec_rows * row_floats);
    double* d_cb = mem.get<double>(cb.size());
    int64_t* sig_tab = mem.get<int64_t>(5);
    if (!rec || !d_cb || !sig_tab) return fail(MVB_ECUDA, "render: scratch allocation");
    const int64_t sig5[5] = {0, n, front, 0, rec_rows};  // off, len, row0, zero pads [0, rec_rows)
    MVB_CUDA(cudaMemcpyAsync(d_cb, cb.data(), 8 * cb.size(), cudaMemcpyHostToDevice, st));
    MVB_CUDA(cudaMemcpyAsync(sig_tab, sig5, sizeof(sig5), cudaMemcpyHostToDevice, st));
    MVB_TRY(mvb_branch_records_f32(a->d_signal, sig_tab, sig_tab + 1, sig_tab + 2, sig_tab + 3,
                                   sig_tab + 4, 1, rec_rows, d_cb, M1, (int)L, nb, rec, stream));
    // ---- work list: (tile, image chunk) CTAs (engine.py _work_list / _chunking) ----
    int sm = 148, ccmaj = 0, ccmin = 0;
    MVB_TRY(mvb_device_info(&sm, &ccmaj, &ccmin));
    const int64_t tiles = (out_len + TILE - 1) / TILE;
    const int64_t want = 54LL * sm;  // 18 waves of 3 CTAs per SM (engine.py CHUNK_WAVES)
    int64_t nc = 1;
    if (tiles < want) {
        nc = std::max<int64_t>(1, (want + tiles - 1) / tiles);
        const int64_t cmin = tiles < SMALL_GRID_TILES ? SMALL_GRID_CHUNK_MIN : CHUNK_MIN_IMAGES;
        nc = std::min<int64_t>(nc, std::max<int64_t>(1, S / cmin));
    }
    std::vector<mvb_work> work((size_t)(nc * tiles));
    for (int64_t ch = 0; ch < nc; ++ch)
        for (int64_t t = 0; t < tiles; ++t) {
            mvb_work& w = work[ch * tiles + t];
            w.job = 0;
            w.tile = (int32_t)t;
            w.img_begin = (int32_t)((S * ch) / nc);
            w.img_end = (int32_t)((S * (ch + 1)) / nc);
            w.chunk = (int32_t)ch;
            w.seg = (int32_t)std::min<int64_t>(t * TILE / SEG_LEN, n_seg - 1);
            w.pad1 = w.pad2 = 0;
        }
    if (tiles >= SMALL_GRID_TILES && work.size() > 1) {
        // tiles by estimated cost, most first, a tile's chunks adjacent
        // (engine.py _work_list, order 3): per image kappa |j * dims| (the
        // image of the room centre) weighted by its tier's cost, the images of
        // each chunk (sorted-delay positions) that admit a row inside the
        // signal over the tile
        const double kap = a->rate / a->c;
        const int K = a->max_order;
        std::vector<std::pair<double, double>> tw;  // (tau, weight)
        tw.reserve((size_t)S);
        for (int x = -K; x <= K; ++x)
            for (int y = -K; y <= K; ++y)
                for (int z = -K; z <= K; ++z) {
                    const int o = std::abs(x) + std::abs(y) + std::abs(z);
                    if (o > K) continue;
                    int N = 1;
                    for (int t = 0; t < a->n_tiers; ++t)
                        if (o <= a->tier_order[t]) { N = a->tier_factor[t]; break; }
                    const double dx = x * a->dims[0], dy = y * a->dims[1], dz = z * a->dims[2];
                    const double w = N == 1 ? 3.0 : 1.0 + (6.0 * 32.0 / N) / 8.75;
                    tw.push_back({kap * std::sqrt(dx * dx + dy * dy + dz * dz), w});
                }
        std::sort(tw.begin(), tw.end());
        std::vector<double> tau(tw.size()), W(tw.size() + 1, 0.0);
        for (size_t i = 0; i < tw.size(); ++i) {
            tau[i] = tw[i].first;
            W[i + 1] = W[i] + tw[i].second;
        }
        const double ls = (double)(n + L - 1);
        std::vector<double> tcost((size_t)tiles, 0.0);
        for (const mvb_work& w : work) {
            const double n0 = (double)w.tile * TILE;
            auto pos = [&](double v) {  // searchsorted(tau, v, side="right") clipped to the chunk
                int64_t p = std::upper_bound(tau.begin(), tau.end(), v) - tau.begin();
                return std::min<int64_t>(std::max<int64_t>(p, w.img_begin), w.img_end);
            };
            tcost[w.tile] += W[pos(n0 + TILE)] - W[pos(n0 - ls)] + 0.05 * (w.img_end - w.img_begin);
        }
        std::stable_sort(work.begin(), work.end(), [&](const mvb_work& p, const mvb_work& q) {
            if (tcost[p.tile] != tcost[q.tile]) return tcost[p.tile] > tcost[q.tile];
            if (p.tile != q.tile) return p.tile < q.tile;
            return p.chunk < q.chunk;
        });
    }
    mvb_job Js = J;
    Js.out_off = 0;
    Js.out_len = out_len;
    Js.rec_base = front;
    Js.n_chunks = (int32_t)nc;
    Js.part_off = 0;
    Js.nb = nb;
    Js.img_off = 0;
    Js.img_stride = (int32_t)S;
    Js.rec_rows = (int32_t)rec_rows;
    mvb_job* d_job = mem.get<mvb_job>(1);
    mvb_work* d_work = mem.get<mvb_work>(work.size());
    float* part = nc > 1 ? mem.get<float>(nc * out_len) : nullptr;
    if (!d_job || !d_work || (nc > 1 && !part)) return fail(MVB_ECUDA, "render: scratch allocation");
    MVB_CUDA(cudaMemcpyAsync(d_job, &Js, sizeof(Js), cudaMemcpyHostToDevice, st));
    MVB_CUDA(cudaMemcpyAsync(d_work, work.data(), sizeof(mvb_work) * work.size(),
                             cudaMemcpyHostToDevice, st));
    MVB_CUDA(cudaMemsetAsync(d_out, 0, 4 * out_len, st));
    int max_factor = 1;
    for (int c = 0; c < nC; ++c) max_factor = std::max(max_factor, factors[c]);
    MVB_TRY(mvb_synthesize_f32_ranged(d_job, d_work, (int64_t)work.size(), sorted, keys, S, SEG_LEN,
                                      max_factor, bbox, coef, rec, paths, d_out, part, nb, 16,
                                      stream));
    if (nc > 1) MVB_TRY(mvb_reduce_partials_f32(d_job, 1, out_len, part, d_out, stream));
    // host sources above are pageable: cudaMemcpyAsync has staged them before
    // returning; the scratch blocks are freed stream-ordered (Scratch)
    return MVB_OK;
}
