/*
 * mvb.h -- C ABI of libmvb.so, the B200 (sm_100a) moving-source synthesis
 * library (arXiv 2508.03065 hot path).  Drop-in boundary for the reference
 * package `moverb` (paths below are relative to /root/reference/pkg/src/moverb/).
 *
 * Conventions
 *   - every entry point returns int: MVB_OK (0) or a negative MVB_E* code;
 *     mvb_last_error() returns the message of the calling thread's last
 *     failure.  No C++ exception crosses the ABI.
 *   - pointers named d_* are DEVICE pointers owned by the caller (e.g. torch
 *     tensors); h_* are host pointers read synchronously during the call.
 *   - every launch is ordered on the caller's `stream` (a cudaStream_t, NULL =
 *     legacy default stream); calls never synchronize the device unless they
 *     say so.  No global mutable state.
 *   - there is no CPU implementation behind any of these symbols.
 */
#ifndef MVB_H
#define MVB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MVB_ABI_VERSION 1

#define MVB_OK 0
#define MVB_EINVAL (-1) /* bad argument (size, null pointer, range)           */
#define MVB_ECUDA (-2)  /* CUDA launch/runtime error, or no sm_100 device     */

int mvb_abi_version(void);
/* Bounds-check counters of the checked build (libmvb_checked.so, compiled
 * with -DMVB_CHECKED: the fast synthesis verifies every gather row, interval
 * record index, staging size and cp.async alignment; the branch-record and
 * exact kernels their rows).  Copies up to n counters (one per check, see
 * csrc/mvb_common.cuh) into h_counts and resets them; returns the number of
 * counters, or MVB_EINVAL from a normal build (no checks compiled in). */
int mvb_check_violations(int64_t* h_counts, int n);
const char* mvb_last_error(void);
/* Fills SM count and compute capability of the current device. */
int mvb_device_info(int* h_sm_count, int* h_cc_major, int* h_cc_minor);
/* sizeof of the structs below as compiled into the library (for bindings
 * that pack them by hand): image, job, work, coef32. */
int mvb_struct_sizes(int* h_image, int* h_job, int* h_work, int* h_coef32);
/* Batched asynchronous copies on `stream` (the input staging of batch
 * renders: one call instead of one runtime call per job input).  Entry i
 * copies h_bytes[i] bytes from h_src[i] to h_dst[i] (cudaMemcpyDefault:
 * host or device pointers).  With require_pinned != 0 an entry whose source
 * is not page-locked host memory is skipped (h_issued[i] = 0; the caller
 * stages it itself), otherwise h_issued[i] = 1.  Launches no kernel. */
int mvb_copy_batch(void* const* h_dst, const void* const* h_src, const int64_t* h_bytes,
                   int64_t n, int32_t* h_issued, int require_pinned, void* stream);

/* ------------------------------------------------------------------------
 * 1. Operator boundary: the reference's kernel swap point (_kernels.py:21-31).
 *    Same semantics and fp64 arithmetic order as the numba kernels -- results
 *    are bit-identical to the reference on identical inputs.
 * --------------------------------------------------------------------- */

/* _kernels.py:65-78 distance_streams: d_out (S,T) = |offset + sign*pos - mic| */
int mvb_distance_streams(const double* d_offset, const double* d_sign, const double* d_mic,
                         const double* d_pos, int64_t S, int64_t T, double* d_out,
                         void* stream);

/* _kernels.py:126-136 accumulate_images: mutates d_out (out_len,) in place.
 * d_streams (n_branches, stream_len); d_tau, d_amp (S, out_len). */
int mvb_accumulate_images(double* d_out, int64_t out_len, const double* d_streams,
                          int64_t n_branches, int64_t stream_len, const double* d_tau,
                          const double* d_amp, int64_t S, int64_t offset, int64_t d0,
                          void* stream);

/* _kernels.py:184-190 upsample_stream, batched over `rows` coarse sequences:
 * d_coarse (rows, n_coarse), d_table (factor, n_taps) row-major as the
 * reference's _phase_table, d_out (rows, out_len). */
int mvb_upsample_streams(const double* d_coarse, int64_t rows, int64_t n_coarse,
                         const double* d_table, int64_t factor, int64_t n_taps,
                         int64_t out_len, double* d_out, void* stream);

/* farrow.py:214-229 branch_filter: d_out (n_branches, T+L-1) = x (*) c_k,
 * sequential fp64 sums (equal to np.convolve within rounding). */
int mvb_branch_filter(const double* d_x, int64_t T, const double* d_branches,
                      int64_t n_branches, int64_t L, double* d_out, void* stream);

/* ------------------------------------------------------------------------
 * 2. Image lattice (room.py:98-143 enumerate_images, room.py:175-187
 *    as_arrays), one thread per image, canonical (order, lattice, parity)
 *    order.  Batched over n_rooms rooms of the same max_order; every output
 *    is (n_rooms, S, ...) and may be NULL.
 * --------------------------------------------------------------------- */

int64_t mvb_image_count(int max_order);
int mvb_enumerate(const double* d_dims, const double* d_walls, int64_t n_rooms,
                  int max_order, int32_t* d_lattice, int32_t* d_parity,
                  int32_t* d_order, double* d_beta, double* d_offset, double* d_sign,
                  void* stream);

/* ------------------------------------------------------------------------
 * 3. Fused moving-source render (synth.py:194-294 generalised to any tier
 *    list, fixed or moving receiver, batches of scenes/channels).  A batch
 *    is a job table (one job = one (scene, channel) output), one image
 *    table holding every job's images, and one fp64 `paths` buffer of
 *    (x, y, z) rows holding every source path, receiver path/position and
 *    decimated path.  Every kernel below covers the whole batch per launch.
 *
 *    Call order (no host wait after the decimation decision):
 *      paths:  path_bbox; path_spectrum_index (own FFT) -> lowpass_paths
 *              (host: low-pass decision, output capacity bound from the
 *              boxes) -> decimate_rows
 *      images: enumerate (cacheable per rooms + order) -> build_images
 *      tracks: coarse_distances (+ bounds; one call per factor) ->
 *              track_bounds -> track_max
 *      fast:   branch_records_f32, track_coeffs (per factor),
 *              delay_sort_keyed (or sort_keys -> sort -> gather_images beyond
 *              MVB_DELAY_SORT_MAX images), finalize_lengths (exact out_len =
 *              len(s) + ceil(rate*dmax/c) + L, synth.py:211-212, on the
 *              device) -> synthesize_f32_ranged (after the keyed sort; else
 *              synthesize_f32) [-> reduce_partials_f32]
 *              (track_max, track_coeffs, delay_sort and branch_records_f32
 *              depend only on the coarse tracks / the signal: independent
 *              streams may run them concurrently)
 *      exact:  branch_filter (per signal), finalize_lengths, synthesize_f64_ex
 *              (or synthesize_f64: the small-batch variant)
 * --------------------------------------------------------------------- */

/* One image of one job (96 B). */
typedef struct mvb_image {
    double off[3];    /* 2*lattice*dims                                     */
    double beta;      /* product of wall reflection coefficients            */
    float sign[3];    /* +-1 per axis                                        */
    float amp_num;    /* beta / (4 pi), fast path                            */
    int32_t factor;   /* decimation N of the image's tier (1 = per sample)   */
    int32_t n_coarse; /* K = ceil(T / N) for factor > 1                       */
    int64_t coarse;   /* first of its K coarse distances (factor > 1)        */
    int64_t coef;     /* first of its K fast-path interval records            */
    int64_t table;    /* first element of the factor's (65, N) transposed table */
    int64_t cpath;    /* first row of its coarse source path in `paths`; with a
                         moving receiver the K coarse receiver rows follow     */
    int32_t job;      /* owning job                                           */
    int32_t fit;      /* index of the factor's (9, 65) refit block            */
} mvb_image;

/* One (scene, channel) render. */
typedef struct mvb_job {
    int64_t out_off, out_len; /* slice of the flat output                       */
    int64_t part_off;         /* slice of the partial buffer (n_chunks > 1)     */
    int64_t rec_base;         /* record / stream index of branch sample 0       */
    int64_t ls;               /* branch stream length len(s) + L - 1            */
    int64_t img_off, n_img;   /* slice of the image table                       */
    int64_t pos_off, mic_off; /* first row of the source path / receiver in paths */
    int32_t T, mic_moving;    /* track length len(traj); receiver path has T rows */
    int32_t L, d0;            /* branch length (= delay shift) and D0           */
    int32_t n_chunks, nb;     /* image chunks; branches per record / stream     */
    double rate, c, d_min, kappa; /* kappa = rate / c                           */
    int32_t img_stride;       /* fast path: images per sort segment in the
                                 delay-sorted table (segment s of this job
                                 starts at img_off + s * img_stride)            */
    int32_t rec_rows;         /* rows of the record buffer (bounds checks of
                                 the checked build, libmvb_checked.so)         */
    int32_t w0, w1;           /* time shard: output samples [w0, w1) only
                                 (w1 <= 0: to the end; all zero: no window);
                                 tracks, records, maxima and sort segments are
                                 computed for the samples the window needs    */
    int32_t e0, e1;           /* path samples [e0, e1) whose coarse tracks the
                                 window needs (its samples and the centres of
                                 its sort segments; e1 <= 0: the whole path)  */
} mvb_job;

/* One CTA of the fast synthesis grid: samples [32U*tile, 32U*(tile+1)) of
 * `job`, images [img_begin, img_end) of the job's image table sorted by
 * delay at the centre of sort segment `seg`. */
typedef struct mvb_work {
    int32_t job, tile, img_begin, img_end, chunk, seg, pad1, pad2;
} mvb_work;

/* Fast-path interval record: the reference's upsampled track on coarse
 * interval k (samples kN .. kN+N-1) refit as a degree-8 polynomial in
 * u = 2 r / N - 1, anchored and pre-split in fp64 (48 B). */
typedef struct mvb_coef32 {
    int32_t B;   /* floor(kappa*g0 + L - D0)                                  */
    float f;     /* kappa*g0 + L - D0 - B - 1/2                               */
    float d_mid; /* g0 (metres, the track at u = 0)                           */
    float pad;
    float g[8];  /* kappa * g_p, p = 1..8                                     */
} mvb_coef32;

/* Image classes of one job group (one class per decimation factor). */
#define MVB_MAX_CLASSES 8
typedef struct mvb_class_table {
    int32_t n;                        /* classes, <= MVB_MAX_CLASSES            */
    int32_t factor[MVB_MAX_CLASSES];  /* decimation factor N of the class       */
    int32_t fit[MVB_MAX_CLASSES];     /* refit block index of N                 */
    int32_t count[MVB_MAX_CLASSES];   /* images of the class per job            */
    int64_t table[MVB_MAX_CLASSES];   /* offset of N's transposed table         */
    int64_t sel_off[MVB_MAX_CLASSES]; /* this group's block in d_class_sel (N > 1) */
} mvb_class_table;

/* Image records of a group of G jobs sharing (max_order, tiers, image
 * subset): image (g, s) -> d_images[img_base + g*S + s] from the enumerated
 * room tables (d_tab_offset (R,S0,3), d_tab_sign (R,S0,3), d_tab_beta
 * (R,S0), room_table.py canonical order).  d_img (S, 2+nC) int32 per image:
 * canonical source index, class, and the number of earlier images in each
 * class; d_job (G, 4+nC) int64 per job: room, T, job id, first coarse
 * index, coarse path row per class.  Also writes the image selections:
 * d_full_sel / d_dec_sel (factor 1 / > 1 images, row g of each block
 * holding job g's images in order, at full_off / dec_off) and d_class_sel
 * (per class blocks at classes->sel_off[c]). */
int mvb_build_images(const double* d_tab_offset, const double* d_tab_sign, const double* d_tab_beta,
                     int64_t S0, const int32_t* d_img, int64_t S, const int64_t* d_job, int64_t G,
                     const mvb_class_table* h_classes, int64_t img_base, mvb_image* d_images,
                     int32_t* d_full_sel, int64_t full_off, int32_t* d_dec_sel, int64_t dec_off,
                     int32_t* d_class_sel, void* stream);

/* Coarse distances of the n_sel images d_sel (factor > 1) on their coarse
 * paths -> d_coarse[image.coarse + k], k < K.  _kernels.py:54-62 arithmetic:
 * bitwise equal to distance_streams on decimate(traj, N).positions.  Unless
 * d_lb / d_ub are NULL, also the bounds of each image's track maximum over
 * t < T (synth.py:201): lb = largest coarse sample (attained), ub = rigorous
 * bound of the band-limited reconstruction, window max + negsum * window
 * range (negsum: the upsampler's negative tap mass); d_lb / d_ub must be
 * zero-initialised (maxima of track chunks merge atomically).  max_K: the
 * largest K of the selection. */
int mvb_coarse_distances(const mvb_image* d_images, const int32_t* d_sel, int64_t n_sel,
                         int64_t max_K, const mvb_job* d_jobs, const double* d_paths,
                         double negsum, double* d_coarse, double* d_lb, double* d_ub,
                         void* stream);

/* Axis-aligned bounding boxes of every job's source path and receiver:
 * d_rows (n_jobs, 4) int64 = (source first row, T, receiver first row,
 * receiver moving); d_bbox: n_jobs x 65 x 16 doubles, the first n_jobs x 16
 * being (src lo xyz, src hi xyz, mic lo xyz, mic hi xyz, src max step, mic
 * max step, 0, 0) -- a step is |p[t+1] - p[t]| in metres -- the rest scratch. */
int mvb_path_bbox(const int64_t* d_rows, int64_t n_jobs, const double* d_paths, double* d_bbox,
                  void* stream);

/* Bounds of the track maximum of the factor-1 images d_full_sel: lb =
 * exact distance at the first / middle / last sample, ub = the largest
 * distance between the bounding boxes (d_bbox, mvb_path_bbox) of the image
 * path and the receiver. */
int mvb_track_bounds(const mvb_image* d_images, const int32_t* d_full_sel, int64_t n_full,
                     const mvb_job* d_jobs, const double* d_paths, const double* d_bbox,
                     double* d_lb, double* d_ub, void* stream);

/* Exact track max of every job (d_dmax[n_jobs]): only the images whose ub
 * reaches the job's largest lb are evaluated (exact distance for factor 1,
 * the reference's 65-tap upsample otherwise), in 2048-sample chunks; a
 * decimated candidate's chunk whose coarse-window bound (negsum as in
 * mvb_coarse_distances) stays below the running maximum is skipped; the
 * surviving chunks are evaluated one sample per thread across the GPU.
 * d_scratch: MVB_EXACT_LIST_WORDS + n_img + n_jobs int32 (8-byte aligned). */
#define MVB_EXACT_LIST_WORDS 16386
int mvb_track_max(const mvb_image* d_images, const mvb_job* d_jobs, int64_t n_jobs,
                  const double* d_coarse, const double* d_tables, const double* d_paths,
                  double negsum, const double* d_lb, const double* d_ub, int32_t* d_scratch,
                  double* d_dmax, void* stream);

/* Exact output lengths on the device (synth.py:211-212): for every job,
 * len(s) + ceil(rate * d_dmax[j] / c) + L with len(s) = ls - L + 1, written
 * into d_jobs[j].out_len (which holds the host's capacity on entry; the
 * render kernels mask by it) and d_lengths[j]; *d_err = 1 if a length
 * exceeds its capacity.  Lets the host plan from an upper bound without
 * waiting for the track maxima. */
int mvb_finalize_lengths(mvb_job* d_jobs, int64_t n_jobs, const double* d_dmax,
                         int64_t* d_lengths, int32_t* d_err, void* stream);

/* d_out[q] = d_images[d_idx[q]], q < n (delay-sorted image tables). */
int mvb_gather_images(const mvb_image* d_images, const int64_t* d_idx, int64_t n,
                      mvb_image* d_out, void* stream);

/* Coarse path rows (decimate's pos[::N], trajectory.py:279-298) for n
 * paths: d_dst[d_rows[2q+1] + k] = d_src[d_rows[2q] + k*N], k < K (rows of
 * 3 doubles; d_rows holds (source row, destination row) pairs). */
int mvb_decimate_rows(const double* d_src, const int64_t* d_rows, int64_t n, int64_t K,
                      int64_t N, double* d_dst, void* stream);

/* Decimation decision (trajectory.py:316-339) around a cuFFT rFFT:
 * mvb_center_paths: d_out = x - mean over T of each axis of the paths
 * d_x (G, T, 3) (d_scratch: 3 G x MVB_SPEC_PARTS doubles; G <= 65535);
 * mvb_spectrum_index: for the rFFT of the centred paths along T (d_spec =
 * complex (G, F, 3), re/im interleaved), for each (path, axis) the first
 * bin whose cumulative power |X|^2 (|X| = hypot) reaches fraction x total
 * -> d_index[3g + a], -1 when all zero (d_scratch: 3 G x MVB_SPEC_PARTS doubles). */
#define MVB_SPEC_PARTS 256
int mvb_center_paths(const double* d_x, int64_t G, int64_t T, double* d_scratch, double* d_out,
                     void* stream);
int mvb_spectrum_index(const double* d_spec, int64_t G, int64_t F, double fraction,
                       double* d_scratch, int64_t* d_index, void* stream);

/* Hand-written fp64 FFT path of decimate() (round 2; replaces the cuFFT
 * calls around the two helpers above).  mvb_fft_c2c: in-place batched
 * complex FFT (interleaved re/im doubles, rows x n contiguous) of any
 * length -- mixed-radix Stockham for 7-smooth n, Bluestein otherwise; sign
 * -1 forward, +1 unnormalised inverse; d_scratch holds
 * mvb_fft_scratch_elems(rows, n) complex values.
 * mvb_path_spectrum_index: the whole bandwidth decision of d_x (G, T, 3)
 * (mean removal, spectrum, energy index -> d_index[3g + a], -1 when all
 * zero), d_scratch mvb_path_spectrum_scratch(G, T) doubles.
 * mvb_lowpass_paths: trajectory.py:214-232 _lowpass_columns for every
 * path of d_x (G, T, 3) -> d_out (G, T, 3), d_scratch
 * mvb_lowpass_scratch(G, T) doubles. */
int64_t mvb_fft_scratch_elems(int64_t rows, int64_t n);
int mvb_fft_c2c(double* d_data, int64_t rows, int64_t n, int sign, double* d_scratch, void* stream);
int64_t mvb_path_spectrum_scratch(int64_t G, int64_t T);
int mvb_path_spectrum_index(const double* d_x, int64_t G, int64_t T, double fraction,
                            double* d_scratch, int64_t* d_index, void* stream);
int64_t mvb_lowpass_scratch(int64_t G, int64_t T);
int mvb_lowpass_paths(const double* d_x, int64_t G, int64_t T, double rate, double cutoff,
                      double* d_scratch, double* d_out, void* stream);

/* Decimation decision helper (trajectory.py:316-339): for each of `rows`
 * power-spectrum rows of length F (fp64, contiguous), the first index whose
 * cumulative energy reaches fraction * row total; -1 for an all-zero row. */
int mvb_energy_index(const double* d_power, int64_t rows, int64_t F, double fraction,
                     int64_t* d_index, void* stream);

/* Fast-path interval records of the images d_sel, all of one decimation
 * factor N: d_coef[image.coef + k] for k < K (K <= max_K), from the coarse
 * distances and h_fit, the factor's (9, 65) refit of its phase-table
 * columns in u = 2r/N - 1 (HOST pointer; passed to the kernel by value). */
int mvb_track_coeffs(const mvb_image* d_images, const int32_t* d_sel, int64_t n_sel,
                     int64_t max_K, const mvb_job* d_jobs, const double* d_coarse,
                     const double* h_fit, mvb_coef32* d_coef, void* stream);
/* The same for time-shard jobs (mvb_job w0/w1/e0/e1): only the intervals
 * the job's output window reads, from the coarse samples its window has
 * (max_K = the largest such coarse range).  A separate entry so the
 * unwindowed kernel keeps its register budget. */
int mvb_track_coeffs_windowed(const mvb_image* d_images, const int32_t* d_sel, int64_t n_sel,
                              int64_t max_K, const mvb_job* d_jobs, const double* d_coarse,
                              const double* h_fit, mvb_coef32* d_coef, void* stream);

/* Delay-sort keys: d_key[(j * max_n_seg + s) * max_n_img + i] = distance of
 * image i of job j at the centre of segment s (samples [s*seg_len,
 * (s+1)*seg_len), clamped to the track), coarse sample for factor > 1.
 * Entries beyond a job's images / segments are not written. */
int mvb_sort_keys(const mvb_image* d_images, const mvb_job* d_jobs, int64_t n_jobs,
                  int64_t max_n_img, int64_t max_n_seg, int64_t seg_len,
                  const double* d_paths, const double* d_coarse, double* d_key, void* stream);

/* Fused delay sort (replaces mvb_sort_keys + an argsort + mvb_gather_images
 * when max_n_img <= MVB_DELAY_SORT_MAX): for every job j and time segment s
 * (samples [s*seg_len, (s+1)*seg_len)), d_out[(j * max_n_seg + s) *
 * max_n_img + q] = the job's image records ordered by their delay in whole
 * samples (kappa * distance) at the segment centre, clamped to key_bits
 * bits (1..32; the host passes the bit length of its delay bound), stable
 * sort; slots q >= n_img and segments past the track hold image
 * min(q, n_img - 1) of the canonical order.  One block radix sort per
 * (job, segment); locality only -- any order renders the same result up to
 * fp32 summation order. */
#define MVB_DELAY_SORT_MAX 16384
int mvb_delay_sort(const mvb_image* d_images, const mvb_job* d_jobs, int64_t n_jobs,
                   int64_t max_n_img, int64_t max_n_seg, int64_t seg_len,
                   const double* d_paths, const double* d_coarse, int64_t key_bits,
                   mvb_image* d_out, void* stream);

/* mvb_delay_sort in independent runs: slots [r * run_len, (r + 1) * run_len)
 * of every (job, segment) hold the job's images of that table range sorted
 * on their own (any image count; run_len <= MVB_DELAY_SORT_MAX).  Used for
 * time-shard jobs, whose image table is in delay-band order (parallel.py
 * band_order): band-local sorts then approximate the full sort, in one
 * block per (segment, band) instead of one 16k-key block per segment. */
int mvb_delay_sort_runs(const mvb_image* d_images, const mvb_job* d_jobs, int64_t n_jobs,
                        int64_t max_n_img, int64_t max_n_seg, int64_t seg_len,
                        const double* d_paths, const double* d_coarse, int64_t key_bits,
                        int64_t run_len, mvb_image* d_out, void* stream);

/* Fast path: fp32 branch records v'_k = x (*) c'_k (d_cbranch (M1, L) fp64
 * in the centred basis (mu - 1/2)^k, zero branches k >= M1) of n_sig dry
 * signals in one launch: signal q is d_x_all[sig_off[q] ..] of length
 * sig_len[q], its sample m < len + L - 1 goes to global row sig_row0[q] + m
 * (device arrays).  With d_sig_zlo / d_sig_zhi (global rows, or both NULL)
 * the rows [zlo, row0) and [row0 + len + L - 1, zhi) -- the zero pads the
 * synthesis gathers rely on -- are written as zeros in the same launch, so
 * the buffer need not be zero-filled first.  max_rows: the largest row
 * count written for one signal (len + L - 1, or zhi - zlo).  Layout: row r =
 * the nb branch values contiguous, row stride 16 B for nb = 4, else 32 B *
 * ceil(nb / 8) (nb = 12 is padded to 16 floats, the padding is not
 * written).  L <= 128; rows < 2^31. */
int mvb_branch_records_f32(const float* d_x_all, const int64_t* d_sig_off,
                           const int64_t* d_sig_len, const int64_t* d_sig_row0,
                           const int64_t* d_sig_zlo, const int64_t* d_sig_zhi, int64_t n_sig,
                           int64_t max_rows, const double* d_cbranch, int M1, int L, int nb,
                           float* d_rec, void* stream);

/* Fast synthesis (fp32 I/O, fp64 anchors), one CTA per work item covering
 * 32*u_steps output samples (u_steps = 16); jobs with n_chunks > 1 write
 * d_part[part_off + chunk*out_len + n].  Gather rows are rec_base + n + L - D
 * (global, never negative: front zero pad). */
int mvb_synthesize_f32(const mvb_job* d_jobs, const mvb_work* d_work, int64_t n_work,
                       const mvb_image* d_images, const mvb_coef32* d_coef,
                       const float* d_rec, const double* d_paths, float* d_out,
                       float* d_part, int nb, int u_steps, void* stream);

/* mvb_delay_sort / mvb_delay_sort_runs (run_len <= 0: one run per job,
 * max_n_img <= MVB_DELAY_SORT_MAX) that also writes the sorted keys:
 * d_keys[(j * max_n_seg + s) * max_n_img + q] = the key (whole samples of
 * delay at the segment centre) of the image in slot q, ascending within each
 * run (padding slots: all ones).  The input of mvb_synthesize_f32_ranged. */
int mvb_delay_sort_keyed(const mvb_image* d_images, const mvb_job* d_jobs, int64_t n_jobs,
                         int64_t max_n_img, int64_t max_n_seg, int64_t seg_len,
                         const double* d_paths, const double* d_coarse, int64_t key_bits,
                         int64_t run_len, mvb_image* d_out, uint32_t* d_keys, void* stream);

/* mvb_synthesize_f32 over a keyed sorted table (mvb_delay_sort_keyed with
 * the same run_len -- a job's whole table: run_len >= its image count -- and
 * seg_len): each work item's warps visit only the images whose key admits a
 * gather row inside the signal over the tile, bounded with the path steps
 * of d_bbox (mvb_path_bbox) and max_factor (largest decimation factor of the
 * batch); the others would read only zero pads.  Same output as
 * mvb_synthesize_f32 (the skipped images add exact zeros). */
int mvb_synthesize_f32_ranged(const mvb_job* d_jobs, const mvb_work* d_work, int64_t n_work,
                              const mvb_image* d_images, const uint32_t* d_keys, int64_t run_len,
                              int64_t seg_len, int max_factor, const double* d_bbox,
                              const mvb_coef32* d_coef, const float* d_rec,
                              const double* d_paths, float* d_out, float* d_part, int nb,
                              int u_steps, void* stream);

/* Measurement variant of mvb_synthesize_f32_ranged (nb = 8 only): the
 * branch-record gathers through the texture pipe (mode 1: every step;
 * mode 2: odd steps, the others LDG.256); rec_floats = the record buffer's
 * size in floats.  Same output. */
int mvb_synthesize_f32_tex(const mvb_job* d_jobs, const mvb_work* d_work, int64_t n_work,
                           const mvb_image* d_images, const uint32_t* d_keys, int64_t run_len,
                           int64_t seg_len, int max_factor, const double* d_bbox,
                           const mvb_coef32* d_coef, const float* d_rec, int64_t rec_floats,
                           const double* d_paths, float* d_out, float* d_part, int nb, int mode,
                           void* stream);

/* Fixed-order sum of the n_chunks partial rows of every job. */
int mvb_reduce_partials_f32(const mvb_job* d_jobs, int64_t n_jobs, int64_t max_out_len,
                            const float* d_part, float* d_out, void* stream);

/* Single-call render of one (scene, channel) job on the fast engine (fp32
 * signal and output, fp64 delay anchors): the C counterpart of the
 * reference's render() / synthesize() (synth.py:291-294, 194-258) for hosts
 * that bind this ABI directly.  Runs, on `stream`, every step of the fused
 * path above (enumeration, image records, coarse tracks + bounds, exact
 * track maximum, interval records, delay sort, branch records, synthesis)
 * with the Python engine's plan.  The caller keeps the reference's
 * decimation (trajectory.py:279-298 decimate(): pos[::N] or its low-passed
 * version) and passes, per tier, the coarse source path (and receiver path
 * for a moving receiver, K = ceil(T / N) rows each) and the factor's phase
 * table (trajectory.py:235-257 _phase_table(N), N x 65, row-major).
 * Writes *h_out_len = len(s) + ceil(rate * max d / c) + L (synth.py:211-212)
 * and the output into d_out[0 .. out_len); returns MVB_EINVAL (with
 * *h_out_len set) when out_capacity is too small.  Synchronizes `stream`
 * once (after the track maximum, which fixes out_len); scratch memory is
 * stream-ordered.  Up to MVB_DELAY_SORT_MAX images (max_order <= 23). */
typedef struct mvb_render_args {
    const float* d_signal;   /* dry signal (n_signal,) fp32                    */
    int64_t n_signal;
    const double* d_pos;     /* source path (T, 3) at the audio rate            */
    int64_t T;
    const double* d_mic;     /* receiver (3,) or, with mic_moving, (T, 3)        */
    int32_t mic_moving;
    int32_t max_order;
    double dims[3];          /* room (Lx, Ly, Lz)                                */
    double walls[6];         /* reflection coefficients (-x, +x, -y, +y, -z, +z) */
    int32_t n_tiers;         /* tier t: orders <= tier_order[t] at 1/tier_factor[t] */
    int32_t tier_order[MVB_MAX_CLASSES];
    int32_t tier_factor[MVB_MAX_CLASSES];
    const double* d_coarse_pos[MVB_MAX_CLASSES]; /* decimated tiers: (K, 3)       */
    const double* d_coarse_mic[MVB_MAX_CLASSES]; /* moving receiver: (K, 3)      */
    const double* h_phase_table[MVB_MAX_CLASSES];/* decimated tiers: (N, 65) host */
    const double* h_branches; /* Farrow bank (poly_order + 1, branch_len), host,
                                 reference basis sum_k c_k mu^k (farrow.py:42-63) */
    int32_t poly_order, branch_len, nominal_delay;
    double rate, c, d_min;
} mvb_render_args;
int mvb_render_tracks_and_synthesize(const mvb_render_args* h_args, float* d_out,
                                     int64_t out_capacity, int64_t* h_out_len, void* stream);

/* SURVEY H2 A/B (measurement only, not the product path): the literal
 * per-fraction-table fractional delay.  mvb_signal_plane_f32 writes the
 * dry signals into a zero-filled fp32 plane d_xp with the branch-record row
 * numbering (row0 = sample 0); mvb_synthesize_f32_table runs the fast
 * synthesis with a direct L-tap gather of that plane, the taps linearly
 * interpolated in mu from d_table ((MVB_TAB_P + 1) x L floats, h_j(p/P) of
 * the filter), staged in shared memory. */
#define MVB_TAB_P 512
int mvb_signal_plane_f32(const float* d_x_all, const int64_t* d_sig_off, const int64_t* d_sig_len,
                         const int64_t* d_sig_row0, int64_t n_sig, int64_t max_len, float* d_xp,
                         void* stream);
int mvb_synthesize_f32_table(const mvb_job* d_jobs, const mvb_work* d_work, int64_t n_work,
                             const mvb_image* d_images, const mvb_coef32* d_coef,
                             const float* d_xp, const double* d_paths, float* d_out,
                             float* d_part, const float* d_table, int L, void* stream);

/* Exact synthesis (fp64): per-sample reference arithmetic (exact or 65-tap
 * upsampled distance, tau = (rate*d)/c, gain, floor split, Horner in mu)
 * in the reference's summation order (32-image blocks of the canonical
 * order, then the pairwise block tree).  d_streams holds each job's
 * (nb, ls) branch streams at rec_base. */
int mvb_synthesize_f64(const mvb_job* d_jobs, int64_t n_jobs, int64_t max_out_len,
                       const mvb_image* d_images, const double* d_coarse,
                       const double* d_tables, const double* d_streams,
                       const double* d_paths, double* d_out, void* stream);

/* mvb_synthesize_f64 for batches of up to max_images images per job: from
 * 1024 images on, two 65-tap chains per warp at 3 CTAs/SM instead of four
 * at 2 (same arithmetic and order: bit-identical output). */
int mvb_synthesize_f64_ex(const mvb_job* d_jobs, int64_t n_jobs, int64_t max_out_len,
                          const mvb_image* d_images, const double* d_coarse,
                          const double* d_tables, const double* d_streams,
                          const double* d_paths, double* d_out, int64_t max_images,
                          void* stream);

/* ------------------------------------------------------------------------
 * 4. Static responses and the splice baseline (reference.py:49-187), fp64.
 *    Sequence: mvb_static_taps -> sort each row of d_base (stable) ->
 *    mvb_static_gather -> mvb_block_convolve [-> mvb_splice_sum].
 * --------------------------------------------------------------------- */
/* reference.py:67-93 for B source positions d_src (B,3) and the S images
 * (d_offset (S,3), d_sign (S,3), d_beta (S,)): d_base (B,S) = floor(tau),
 * d_tau (B,S) = rate*d/c, d_kernel (B,S,65) = beta/(4 pi max(d,d_min)) *
 * Kaiser(7.857)-windowed sinc at (i - 32) - frac (reference.py:49-64). */
int mvb_static_taps(const double* d_offset, const double* d_sign, const double* d_beta,
                    int64_t S, const double* d_src, int64_t B, const double* d_mic,
                    double rate, double c, double d_min, int64_t* d_base, double* d_tau,
                    double* d_kernel, void* stream);
/* reference.py:94-100 (scatter-add into the tap train, clipped to
 * [0, n_taps)) as a gather: d_taps (B, tap_stride), row b zero beyond
 * d_n_taps[b].  d_base_sorted / d_perm: each row of d_base sorted ascending
 * and the image index of every sorted entry. */
int mvb_static_gather(const int64_t* d_base_sorted, const int64_t* d_perm, const double* d_kernel,
                      int64_t S, int64_t B, const int64_t* d_n_taps, int64_t tap_stride,
                      double* d_taps, void* stream);
/* Direct convolution of block b's windowed support of x (n,) with tap row
 * b: d_pieces (n_blocks, piece_stride), row b = (x * w_b)[lo_b:hi_b] (*)
 * taps_b, length (hi_b - lo_b) + n_taps_b - 1 <= max_piece.  Blocks and
 * windows as splice_baseline (reference.py:145-165; lo_b = b*hop, windowed
 * = 1); static_render (reference.py:103-117) is n_blocks = 1, hop = n,
 * crossfade = 0, windowed = 0. */
int mvb_block_convolve(const double* d_x, int64_t n, int64_t hop, int64_t crossfade,
                       int64_t n_blocks, int windowed, const double* d_taps,
                       const int64_t* d_n_taps, int64_t tap_stride, int64_t max_piece,
                       double* d_pieces, int64_t piece_stride, void* stream);
/* reference.py:180-186: d_out[i] = sum over blocks in order of the pieces
 * covering output sample i (max_span = longest piece). */
int mvb_splice_sum(const double* d_pieces, int64_t piece_stride, int64_t n, int64_t hop,
                   int64_t crossfade, int64_t n_blocks, const int64_t* d_n_taps,
                   int64_t max_span, double* d_out, int64_t out_len, void* stream);

/* ------------------------------------------------------------------------
 * 5. Roofline probes (measurement only): FP32 FFMA throughput
 *    (blocks x 256 threads x iters x 128 FFMA) and L1-hit 16-byte load
 *    bandwidth (blocks x 256 threads x iters x 4 x 16 B).  Time them with
 *    CUDA events on `stream`.
 * --------------------------------------------------------------------- */
int mvb_peak_ffma(int blocks, int iters, float* d_sink, void* stream);
/* FP64 FMA peak probe: blocks x 256 threads x iters x 128 DFMA. */
int mvb_peak_dfma(int blocks, int iters, double* d_sink, void* stream);
int mvb_peak_l1(int blocks, int iters, const float* d_buf /* 1 MiB */, float* d_sink,
                void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MVB_H */
