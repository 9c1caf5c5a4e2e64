/*
 * mvb_oracle.c -- CPU restatement of the reference moving-source path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2508_03065_b200/)
 * may link, load or call this file.  It is used by tests/, by
 * __graft_entry__.smoke() as the checker, and by bench.py's cpu_baseline /
 * --impl reference arm as the timed CPU implementation ("port").
 *
 * Every routine restates one piece of the reference package `moverb`
 * (paths relative to /root/reference/pkg/src/moverb/) with the same
 * arithmetic order, so that on identical inputs the results agree bit for
 * bit with the reference's numba kernels where the reference itself is
 * deterministic (compile with -ffp-contract=off, no -ffast-math):
 *
 *   orc_enumerate        room.py:98-143 (+ ImageSourceSpec order room.py:82-95,
 *                        as_arrays room.py:175-187)
 *   orc_distance         _kernels.py:54-62   (_distance_numba)
 *   orc_upsample         _kernels.py:164-181 (_upsample_numba)
 *   orc_accumulate       _kernels.py:109-123 (_accumulate_numba)
 *   orc_branch_filter    farrow.py:214-229   (np.convolve per branch; plain
 *                        sequential sum, equal to numpy within rounding)
 *   orc_render_window    synth.py:194-258 (synthesize, receiver modulation)
 *                        composed with synth.py:122-158 (low/high order
 *                        distances, any number of tiers) evaluated only for
 *                        output samples [n0, n1): memory stays bounded, the
 *                        per-sample arithmetic, the 32-image block sums and
 *                        the pairwise block merge (synth.py:182-191,
 *                        SUMMATION_BLOCK synth.py:36) are the reference's.
 *   orc_hann_sinc_gather direct exact-tap Hann-windowed-sinc gather (the
 *                        configs' fractional-delay filter)
 *                        used to pin the Farrow fit of that filter.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

#define ORC_BLOCK 32 /* synth.py:36 SUMMATION_BLOCK */

/* ------------------------------------------------------------------ */
/* tiny pthread parallel-for: chunks of [lo,hi) handed out by an atomic
 * counter; each index is computed by exactly one thread, so results do not
 * depend on the thread count.                                            */

typedef void (*orc_body)(void* ctx, int64_t i0, int64_t i1, void* scratch);
typedef struct {
    orc_body body; void* ctx; int64_t lo, hi, chunk; int64_t next;
    size_t scratch_bytes; pthread_mutex_t mu;
} orc_pfor;

static void* orc_worker(void* arg) {
    orc_pfor* p = (orc_pfor*)arg;
    void* scratch = p->scratch_bytes ? malloc(p->scratch_bytes) : NULL;
    for (;;) {
        pthread_mutex_lock(&p->mu);
        int64_t i0 = p->next;
        p->next += p->chunk;
        pthread_mutex_unlock(&p->mu);
        if (i0 >= p->hi) break;
        int64_t i1 = i0 + p->chunk < p->hi ? i0 + p->chunk : p->hi;
        p->body(p->ctx, i0, i1, scratch);
    }
    free(scratch);
    return NULL;
}

int orc_default_threads(void) {
    long n = sysconf(_SC_NPROCESSORS_ONLN);
    return n > 0 ? (int)n : 1;
}

static void orc_parallel_for(int nthreads, int64_t lo, int64_t hi, int64_t chunk,
                             size_t scratch_bytes, orc_body body, void* ctx) {
    if (nthreads <= 0) nthreads = orc_default_threads();
    orc_pfor p;
    p.body = body; p.ctx = ctx; p.lo = lo; p.hi = hi; p.chunk = chunk > 0 ? chunk : 1;
    p.next = lo; p.scratch_bytes = scratch_bytes;
    pthread_mutex_init(&p.mu, NULL);
    if (nthreads == 1) { orc_worker(&p); pthread_mutex_destroy(&p.mu); return; }
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
    for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, orc_worker, &p);
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(th);
    pthread_mutex_destroy(&p.mu);
}

/* ------------------------------------------------------------------ */
/* image lattice                                                        */

int64_t orc_image_count(int max_order) {
    /* synth.py:297-299: order o contributes 4 o^2 + 2 images */
    if (max_order < 0) return 0;
    int64_t n = 1;
    for (int o = 1; o <= max_order; ++o) n += 4LL * o * o + 2;
    return n;
}

typedef struct {
    int32_t order;
    int32_t lat[3];
    int32_t par[3];
    double beta;
    int32_t j[3];
} orc_spec;

static int spec_cmp(const void* a_, const void* b_) {
    const orc_spec* a = (const orc_spec*)a_;
    const orc_spec* b = (const orc_spec*)b_;
    /* dataclass(order=True) field order: order, lattice, parity (room.py:82-95);
     * beta never decides because (lattice, parity) is unique per image */
    if (a->order != b->order) return a->order < b->order ? -1 : 1;
    for (int k = 0; k < 3; ++k)
        if (a->lat[k] != b->lat[k]) return a->lat[k] < b->lat[k] ? -1 : 1;
    for (int k = 0; k < 3; ++k)
        if (a->par[k] != b->par[k]) return a->par[k] < b->par[k] ? -1 : 1;
    return 0;
}

static int floordiv(int a, int b) { /* python // for b > 0 */
    int q = a / b;
    if ((a % b != 0) && (a < 0)) --q;
    return q;
}

/* Fills S = orc_image_count(max_order) rows in canonical order.
 * offset = 2*lattice*dims, sign = -1 where the axis is flipped (room.py:175-187). */
int64_t orc_enumerate(const double dims[3], const double walls[6], int max_order,
                      int32_t* jxyz, int32_t* lattice, int32_t* parity,
                      int32_t* order, double* beta, double* offset, double* sign) {
    int64_t S = orc_image_count(max_order);
    if (S <= 0) return 0;
    orc_spec* specs = (orc_spec*)malloc(sizeof(orc_spec) * (size_t)S);
    int64_t n = 0;
    for (int jx = -max_order; jx <= max_order; ++jx) {
        int rx = max_order - abs(jx);
        for (int jy = -rx; jy <= rx; ++jy) {
            int ry = rx - abs(jy);
            for (int jz = -ry; jz <= ry; ++jz) {
                int js[3] = {jx, jy, jz};
                orc_spec* sp = &specs[n++];
                double b = 1.0;
                for (int k = 0; k < 3; ++k) {
                    int j = js[k];
                    int q = ((j % 2) + 2) % 2; /* python j % 2 */
                    sp->lat[k] = floordiv(j + q, 2);
                    sp->par[k] = q;
                    sp->j[k] = j;
                    int hm, hp; /* room.py:98-105 */
                    if (j >= 0) { hm = j / 2; hp = (j + 1) / 2; }
                    else { int a = -j; hm = (a + 1) / 2; hp = a / 2; }
                    b *= pow(walls[2 * k], (double)hm) * pow(walls[2 * k + 1], (double)hp);
                }
                sp->beta = b;
                sp->order = abs(jx) + abs(jy) + abs(jz);
            }
        }
    }
    qsort(specs, (size_t)S, sizeof(orc_spec), spec_cmp);
    for (int64_t i = 0; i < S; ++i) {
        const orc_spec* sp = &specs[i];
        for (int k = 0; k < 3; ++k) {
            if (jxyz) jxyz[3 * i + k] = sp->j[k];
            if (lattice) lattice[3 * i + k] = sp->lat[k];
            if (parity) parity[3 * i + k] = sp->par[k];
            if (offset) offset[3 * i + k] = 2.0 * (double)sp->lat[k] * dims[k];
            if (sign) sign[3 * i + k] = sp->par[k] ? -1.0 : 1.0;
        }
        if (order) order[i] = sp->order;
        if (beta) beta[i] = sp->beta;
    }
    free(specs);
    return S;
}

/* ------------------------------------------------------------------ */
/* the reference kernel trio                                             */

static inline double dist1(const double* off, const double* sg, const double* mic,
                           const double* p) {
    double dx = off[0] + sg[0] * p[0] - mic[0];
    double dy = off[1] + sg[1] * p[1] - mic[1];
    double dz = off[2] + sg[2] * p[2] - mic[2];
    return sqrt(dx * dx + dy * dy + dz * dz);
}

void orc_distance(const double* offset, const double* sign, const double* mic,
                  const double* pos, int64_t S, int64_t T, double* out) {
    for (int64_t i = 0; i < S; ++i)
        for (int64_t t = 0; t < T; ++t)
            out[i * T + t] = dist1(offset + 3 * i, sign + 3 * i, mic, pos + 3 * t);
}

static inline double upsample_at(const double* coarse, int64_t nc, const double* table,
                                 int64_t factor, int64_t ntaps, int64_t m) {
    int64_t half = (ntaps - 1) / 2;
    int64_t base = m / factor, phase = m % factor;
    const double* row = table + phase * ntaps;
    double acc = 0.0;
    for (int64_t col = 0; col < ntaps; ++col) {
        int64_t j = base + (col - half);
        if (j < 0) j = 0;
        else if (j >= nc) j = nc - 1;
        acc += row[col] * coarse[j];
    }
    return acc;
}

void orc_upsample(const double* coarse, int64_t nc, const double* table, int64_t factor,
                  int64_t ntaps, int64_t out_len, double* out) {
    for (int64_t m = 0; m < out_len; ++m)
        out[m] = upsample_at(coarse, nc, table, factor, ntaps, m);
}

static inline double horner(const double* streams, int64_t nb, int64_t ls, int64_t idx,
                            double mu) {
    double acc = streams[(nb - 1) * ls + idx];
    for (int64_t k = nb - 2; k >= 0; --k) acc = acc * mu + streams[k * ls + idx];
    return acc;
}

void orc_accumulate(double* out, int64_t out_len, const double* streams, int64_t nb,
                    int64_t ls, const double* tau, const double* amp, int64_t S,
                    int64_t offset, int64_t d0) {
    for (int64_t i = 0; i < S; ++i) {
        for (int64_t n = 0; n < out_len; ++n) {
            double shifted = tau[i * out_len + n] + (double)offset;
            double d_int = floor(shifted - (double)d0);
            double mu = shifted - (double)d0 - d_int;
            int64_t idx = n + offset - (int64_t)d_int;
            if (idx >= 0 && idx < ls)
                out[n] += amp[i * out_len + n] * horner(streams, nb, ls, idx, mu);
        }
    }
}

void orc_branch_filter(const double* x, int64_t T, const double* branches, int64_t nb,
                       int64_t L, double* out) {
    int64_t ls = T + L - 1;
    for (int64_t k = 0; k < nb; ++k) {
        const double* c = branches + k * L;
        for (int64_t m = 0; m < ls; ++m) {
            int64_t jlo = m - (T - 1) > 0 ? m - (T - 1) : 0;
            int64_t jhi = m < L - 1 ? m : L - 1;
            double acc = 0.0;
            for (int64_t j = jlo; j <= jhi; ++j) acc += c[j] * x[m - j];
            out[k * ls + m] = acc;
        }
    }
}

/* ------------------------------------------------------------------ */
/* windowed render                                                       */

typedef struct {
    int64_t S;             /* images, canonical order                      */
    const double* offset;  /* (S,3)                                        */
    const double* sign;    /* (S,3)                                        */
    const double* beta;    /* (S,)                                         */
    const int64_t* factor; /* (S,) decimation N of the image's tier (1=full)*/
    const int64_t* coarse_off; /* (S,) row start in `coarse` (N>1 only)    */
    const int64_t* coarse_len; /* (S,) coarse length ceil(T/N)             */
    const double* coarse;  /* concatenated coarse distance rows            */
    const int64_t* table_off;  /* (S,) start of the N x ntaps phase table  */
    const double* tables;  /* concatenated phase tables                    */
    int64_t ntaps;         /* 65 (trajectory.py:24, 2*32+1)                */
    const double* pos;     /* (T,3) source path at the audio rate          */
    const double* mic;     /* (T,3) when mic_moving, else (3,)             */
    int32_t mic_moving;
    int64_t T;
    const double* streams; /* (nb, ls) branch streams                      */
    int64_t nb, ls;
    int64_t shift;         /* = L, synth.py:222                            */
    int64_t d0;            /* nominal delay (L-1)//2                       */
    double rate, c, d_min;
} orc_scene;

static inline double track_at(const orc_scene* sc, int64_t i, int64_t n) {
    int64_t m = n < sc->T ? n : sc->T - 1; /* hold-extension, synth.py:213-217 */
    if (sc->factor[i] == 1) {
        const double* mic = sc->mic_moving ? sc->mic + 3 * m : sc->mic;
        return dist1(sc->offset + 3 * i, sc->sign + 3 * i, mic, sc->pos + 3 * m);
    }
    return upsample_at(sc->coarse + sc->coarse_off[i], sc->coarse_len[i],
                       sc->tables + sc->table_off[i], sc->factor[i], sc->ntaps, m);
}

/* Contribution of image i at output n following _kernels.py:114-122 and the
 * tau/amp formulas of synth.py:218-220.  Returns 0 with *valid=0 when the
 * read index falls outside the branch streams. */
static inline double contrib(const orc_scene* sc, int64_t i, int64_t n, int* valid) {
    double d = track_at(sc, i, n);
    double tau = sc->rate * d / sc->c;
    double amp = sc->beta[i] / (4.0 * M_PI * (d > sc->d_min ? d : sc->d_min));
    double shifted = tau + (double)sc->shift;
    double d_int = floor(shifted - (double)sc->d0);
    double mu = shifted - (double)sc->d0 - d_int;
    int64_t idx = n + sc->shift - (int64_t)d_int;
    if (idx < 0 || idx >= sc->ls) { *valid = 0; return 0.0; }
    *valid = 1;
    return amp * horner(sc->streams, sc->nb, sc->ls, idx, mu);
}

/* out[n-n0] for n in [n0,n1).  Block sums over 32 canonical-order images,
 * then the fixed pairwise tree over blocks -> the reference's bits given the
 * same tracks and branch streams.  Work is split over 256-sample tiles; inside
 * a tile the loop is image-outer / sample-inner like _accumulate_numba, and
 * every sample's sum order is the reference's regardless of thread count. */
#define ORC_TILE 256

typedef struct { const orc_scene* sc; int64_t n0, n1; double* out; int64_t nblk; } rw_ctx;

static void rw_body(void* ctx_, int64_t t0, int64_t t1, void* scratch) {
    rw_ctx* c = (rw_ctx*)ctx_;
    const orc_scene* sc = c->sc;
    double* buf = (double*)scratch; /* nblk x ORC_TILE */
    for (int64_t t = t0; t < t1; ++t) {
        int64_t a = c->n0 + t * ORC_TILE;
        int64_t b = a + ORC_TILE < c->n1 ? a + ORC_TILE : c->n1;
        int64_t w = b - a;
        for (int64_t blk = 0; blk < c->nblk; ++blk) {
            double* acc = buf + blk * ORC_TILE;
            for (int64_t k = 0; k < w; ++k) acc[k] = 0.0;
            int64_t i1 = (blk + 1) * ORC_BLOCK < sc->S ? (blk + 1) * ORC_BLOCK : sc->S;
            for (int64_t i = blk * ORC_BLOCK; i < i1; ++i)
                for (int64_t k = 0; k < w; ++k) {
                    int valid;
                    double v = contrib(sc, i, a + k, &valid);
                    if (valid) acc[k] += v;
                }
        }
        for (int64_t k = 0; k < w; ++k) {
            int64_t cnt = c->nblk;
            while (cnt > 1) { /* synth.py:182-191 */
                int64_t m = 0;
                for (int64_t q = 0; q + 1 < cnt; q += 2)
                    buf[(m++) * ORC_TILE + k] = buf[q * ORC_TILE + k] + buf[(q + 1) * ORC_TILE + k];
                if (cnt % 2) buf[(m++) * ORC_TILE + k] = buf[(cnt - 1) * ORC_TILE + k];
                cnt = m;
            }
            c->out[a + k - c->n0] = c->nblk > 0 ? buf[k] : 0.0;
        }
    }
}

void orc_render_window(const orc_scene* sc, int64_t n0, int64_t n1, double* out,
                       int nthreads) {
    if (n1 <= n0) return;
    rw_ctx c = {sc, n0, n1, out, (sc->S + ORC_BLOCK - 1) / ORC_BLOCK};
    int64_t ntiles = (n1 - n0 + ORC_TILE - 1) / ORC_TILE;
    size_t scratch = sizeof(double) * (size_t)((c.nblk > 0 ? c.nblk : 1) * ORC_TILE);
    orc_parallel_for(nthreads, 0, ntiles, 1, scratch, rw_body, &c);
}

/* tracks of every image over output samples [n0, n1) (hold-extended past
 * T, synth.py:213-217): out (S, n1 - n0) row-major, images split over
 * threads.  Feeds the L0 kernel-only baseline (oracle/l0.py). */
typedef struct { const orc_scene* sc; int64_t n0, n1; double* out; } tw_ctx;

static void tw_body(void* ctx_, int64_t i0, int64_t i1, void* scratch) {
    (void)scratch;
    tw_ctx* c = (tw_ctx*)ctx_;
    const int64_t w = c->n1 - c->n0;
    for (int64_t i = i0; i < i1; ++i)
        for (int64_t k = 0; k < w; ++k) c->out[i * w + k] = track_at(c->sc, i, c->n0 + k);
}

void orc_tracks_window(const orc_scene* sc, int64_t n0, int64_t n1, double* out, int nthreads) {
    if (n1 <= n0) return;
    tw_ctx c = {sc, n0, n1, out};
    orc_parallel_for(nthreads, 0, sc->S, 16, 0, tw_body, &c);
}

/* max over images and samples t < T of the track, as synth.py:201 uses it */
typedef struct { const orc_scene* sc; double* best; } tm_ctx;

static void tm_body(void* ctx_, int64_t i0, int64_t i1, void* scratch) {
    (void)scratch;
    tm_ctx* c = (tm_ctx*)ctx_;
    for (int64_t i = i0; i < i1; ++i) {
        double b = -1.0;
        for (int64_t t = 0; t < c->sc->T; ++t) {
            double d = track_at(c->sc, i, t);
            if (d > b) b = d;
        }
        c->best[i] = b;
    }
}

double orc_track_max(const orc_scene* sc, int nthreads) {
    double* per = (double*)malloc(sizeof(double) * (size_t)(sc->S > 0 ? sc->S : 1));
    tm_ctx c = {sc, per};
    orc_parallel_for(nthreads, 0, sc->S, 1, 0, tm_body, &c);
    double best = -1.0;
    for (int64_t i = 0; i < sc->S; ++i)
        if (per[i] > best) best = per[i];
    free(per);
    return best;
}

/* Direct L-tap gather with exact Hann-windowed-sinc taps (no Farrow fit):
 * y(n) = sum_i A_i(n) sum_j h(j, mu) x(n + shift - D - j), h(j,mu) =
 * sinc(t) * 0.5(1+cos(2 pi t/L)), t = j - D0 - mu.  Same tracks, same D/mu
 * split as contrib(); plain sequential sum over images (pins the fit only). */
typedef struct { const orc_scene* sc; const double* x; int64_t Tx, L, n0; double* out; } hs_ctx;

static void hs_body(void* ctx_, int64_t a, int64_t b, void* scratch) {
    (void)scratch;
    hs_ctx* c = (hs_ctx*)ctx_;
    const orc_scene* sc = c->sc;
    for (int64_t n = a; n < b; ++n) {
        double y = 0.0;
        for (int64_t i = 0; i < sc->S; ++i) {
            double d = track_at(sc, i, n);
            double tau = sc->rate * d / sc->c;
            double amp = sc->beta[i] / (4.0 * M_PI * (d > sc->d_min ? d : sc->d_min));
            double shifted = tau + (double)sc->shift;
            double d_int = floor(shifted - (double)sc->d0);
            double mu = shifted - (double)sc->d0 - d_int;
            int64_t base = n + sc->shift - (int64_t)d_int;
            double acc = 0.0;
            for (int64_t j = 0; j < c->L; ++j) {
                int64_t xi = base - j;
                if (xi < 0 || xi >= c->Tx) continue;
                double t = (double)j - (double)sc->d0 - mu;
                double w = fabs(t) <= 0.5 * (double)c->L
                               ? 0.5 * (1.0 + cos(2.0 * M_PI * t / (double)c->L)) : 0.0;
                double s = t == 0.0 ? 1.0 : sin(M_PI * t) / (M_PI * t);
                acc += s * w * c->x[xi];
            }
            y += amp * acc;
        }
        c->out[n - c->n0] = y;
    }
}

void orc_hann_sinc_gather(const orc_scene* sc, const double* x, int64_t Tx, int64_t L,
                          int64_t n0, int64_t n1, double* out, int nthreads) {
    hs_ctx c = {sc, x, Tx, L, n0, out};
    orc_parallel_for(nthreads, n0, n1, 64, 0, hs_body, &c);
}
