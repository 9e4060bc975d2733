/*
 * smoe.h -- C ABI of the B200-native Rasterized SMoE hot path.
 *
 * Method: Rasterized Steered Mixture-of-Experts regression, arxiv 2510.05814
 * (citations: P:n = PAPER.md line n; S:n = SPEC.md line n; Q-numbers are the
 * readings listed in DESIGN.md).  A pixel x of an H x W x C image is
 *
 *     y(x) = sum_{j in K_n} m_j(x) w_j(x),                  Eq. (5)
 *     w_j(x) = pi_j K_j(x) / sum_{i in K_n} pi_i K_i(x),     Eq. (4)
 *     K_j(x) = exp(-1/2 (x-mu_j)^T Sigma_j^-1 (x-mu_j)),     Eq. (3)
 *
 * with Sigma_j = L_j L_j^T (Cholesky), pi_j = exp(log_pi_j), experts
 * m_j(x) = m_j (constant) or m_j + W_j (x - mu_j) (linear), each kernel
 * truncated at its 99% confidence ellipse d^2 <= R2 = 2 ln 100 (
 * Q1-Q3) and binned into 16x16 blocks through the square box whose side is
 * the major axis of that ellipse.  Pixel (row i, col j) is
 * centred at (j, i); a pixel with no contributing kernel renders 0 (Q7).
 *
 * Every entry point returns a smoe_status; no C++ exception crosses the ABI.
 * Host-side argument checks are synchronous.  Device work is enqueued on the
 * handle's stream and is asynchronous unless stated otherwise.  Device-side
 * faults (non-finite values, pair-capacity overflow) are latched on the
 * device and reported by the next synchronising call (smoe_sync, smoe_step
 * with stats, smoe_render to a host buffer).
 *
 * Memory: the caller owns params, targets, outputs and gradient buffers.
 * Parameters must be DEVICE pointers (CUDA device memory of the handle's
 * device).  `target` and `out` may be device or host pointers (host buffers
 * are copied through a library staging buffer on the handle's stream; pinned
 * host memory makes those copies asynchronous).  The library owns its
 * workspace (kernel records, block lists, accumulators) and the Adam state and
 * never frees caller memory.  A handle is bound to one device and one stream
 * and is not thread-safe.
 */
#ifndef SMOE_H
#define SMOE_H

#ifdef __cplusplus
extern "C" {
#endif

#define SMOE_ABI_VERSION 2

typedef struct smoe_ctx *smoe_handle;

typedef enum {
    SMOE_OK = 0,
    SMOE_ERR_INVALID_ARG = 1,   /* bad shape, NULL pointer, unsupported C/order   */
    SMOE_ERR_CUDA = 2,          /* a CUDA runtime call failed (see smoe_last_error) */
    SMOE_ERR_OUT_OF_MEMORY = 3, /* workspace allocation failed                      */
    SMOE_ERR_NONFINITE = 4,     /* NaN/Inf in parameters, loss or gradients */
    SMOE_ERR_CAPACITY = 5,      /* (block, kernel) pair list overflowed; buffers were
                                   grown, the affected asynchronous calls were
                                   skipped and must be repeated                    */
    SMOE_ERR_BAD_HANDLE = 6
} smoe_status;

/* Kernel parameters, caller-owned DEVICE float32 arrays (struct of arrays):
 *   mu[K][2]       centre (x, y) in source pixels             (Eq. 3, mu_j)
 *   chol[K][3]     (l11, l21, l22), Sigma = L L^T, l11,l22>0
 *   log_pi[K]      log gate weight, pi = exp(log_pi)          (Eq. 4, pi_j)
 *   expert[K][C][E] E = 1: (m_c); E = 3: (m_c, Wx_c, Wy_c)    (Eq. 2, m_j(x)) */
typedef struct {
    float *mu;
    float *chol;
    float *log_pi;
    float *expert;
} smoe_params;

/* Per-group Adam learning rates for one step, already scheduled by
 * the caller (smoe_paper_lr gives the paper's schedule).  A rate of 0 freezes
 * the group (its Adam moments still advance). */
typedef struct {
    float mu;      /* centres                    (0.01 -> 1e-5)      */
    float chol;    /* Cholesky factors           (1e-3)              */
    float log_pi;  /* gate log-weights           (Q11: 0, frozen)           */
    float expert;  /* expert constants m_c       (1e-3)              */
    float slope;   /* linear-expert slopes W     (Q13: 2e-4)                */
} smoe_lr;

/* Step statistics, measured by the step's own forward pass (before the
 * parameter update).  loss = SSE/(H W C) (Q8); psnr_db = 10 log10(1/MSE) on
 * [0,1]-clamped images; pairs = number of (block, kernel) list
 * entries (sum_n |K_n|, "Avg. kernel" = pairs / n_tiles). */
typedef struct {
    double loss;
    double psnr_db;
    double sse;
    double sse_clamped;
    long long pairs;
    long long uncovered_px;
    long long n_tiles;
} smoe_stats;

typedef struct {
    int K, H, W, C, expert_order;  /* C in {1,3}; expert_order in {0,1}           */
    double R2;                     /* truncation radius^2; default 2 ln 100 (Q1) */
    int device;                    /* CUDA device ordinal, -1 = current device   */
    long long pair_capacity;       /* initial pair capacity, 0 = automatic        */
    int backward_mode;             /* -1 = auto (default: kernel-parallel), 0 =
                                      pixel-parallel with warp reductions, 1 =
                                      kernel-parallel over per-warp pixel-pair
                                      lists                     */
    int use_graphs;                /* 1 (default): smoe_step / smoe_grad replay
                                      their launch sequence as a CUDA graph     */
    int head;                      /* regression head: 0 = SMoE soft gates
                                      (Eq. 2/4, default); 1 = RBF weighted sum
                                      of kernels y = sum_j m_j(x) pi_j K_j(x)
                                      (Eq. 1; GaussianImage-style,
                                      SURVEY §8(f) f2).  R2 = INFINITY gives the
                                      dense global (untruncated) model (GSMoE,
                                      P:173-180).                               */
    int box_mode;                  /* block listing (reading Q4):
                                      0 = square box of side 2 R sqrt(lambda_max)
                                      (the paper's); 1 = the ellipse's axis-
                                      aligned box (half sides R sqrt(Sigma_xx),
                                      R sqrt(Sigma_yy); the default: equal to
                                      the square for isotropic kernels, fewer
                                      blocks as kernels turn anisotropic, 1.4-4%
                                      faster fit steps measured on fitted pools,
                                      DESIGN.md §5); 2 = exact: the blocks of
                                      mode 1 whose rectangle of pixel-centre
                                      sample points meets the ellipse.  Pixels,
                                      losses and gradients do not depend on the
                                      mode; the lists (smoe_bin) and the work do */
} smoe_options;

/* Fill `o` with the defaults (R2 = 2 ln 100, device = -1, automatic capacity,
 * automatic backward form, CUDA graphs on, box_mode = 1). */
smoe_status smoe_default_options(smoe_options *o);

/* Create a handle for K kernels fitting an H x W x C image (B.json:
 * smoe_create(K, H, W, C, expert_order)).  Allocates the workspace and the
 * Adam state (zeroed, step t = 0) on the current device.  K, H, W >= 1. */
smoe_status smoe_create(int K, int H, int W, int C, int expert_order, smoe_handle *out);
smoe_status smoe_create_ex(const smoe_options *opt, smoe_handle *out);
smoe_status smoe_destroy(smoe_handle h);

/* Bind the handle to a CUDA stream (cudaStream_t passed as void*; NULL = the
 * legacy default stream).  All later device work is ordered on it. */
smoe_status smoe_set_stream(smoe_handle h, void *stream);

/* Native super-resolution render (B.json smoe_render(params,
 * out_H, out_W)): out[C][out_H][out_W] (planar float32) = y sampled at the
 * source point ((j+1/2) W/out_W - 1/2, (i+1/2) H/out_H - 1/2) of every output
 * pixel (Q16); out_H = H, out_W = W is the plain reconstruction.  Pure: does
 * not touch Adam state.  `out` may be host (call returns after the copy and
 * capacity check) or device (asynchronous). */
smoe_status smoe_render(smoe_handle h, const smoe_params *p, int out_H, int out_W, float *out);

/* Render options.  sharpen = s in (0, 1]: native
 * sharpening by kernel editing, "reducing the bandwidths of the kernels by a
 * sharpening factor": the render uses Sigma_j -> s Sigma_j
 * (every Cholesky factor times sqrt(s)); s = 1 is the plain
 * render.  accumulate = w != 0: out += w y instead of
 * out = y, so H hypotheses fuse into their average y_m = (1/H) sum_h y_h
 * (Eq. 11) with w = 1/H; needs a device `out`.  The caller's
 * parameters are not modified.  Pixels are identical for both store modes. */
typedef struct {
    float sharpen;
    float accumulate;
    int vector_stores;   /* 1: stage the block's outputs in shared memory and
                            write 16-byte float4 rows (st.global.v4); 0
                            (default): each thread stores its pixels (measured
                            faster: the render is not store-bound) */
} smoe_render_options;
smoe_status smoe_render_ex(smoe_handle h, const smoe_params *p, int out_H, int out_W, float *out,
                           const smoe_render_options *opt);

/* One training iteration (B.json smoe_step(params, target, lr)): forward,
 * MSE loss, analytic gradients of all kernel parameters, fused Adam update
 * (beta = 0.9/0.999, eps = 1e-8, Q9) and clamp l11,l22 >= 1e-3, in
 * place on `p`.  target[C][H][W] float32, host or device.  If `stats` is
 * non-NULL the call synchronises and fills it (pre-update loss/PSNR);
 * otherwise it is asynchronous. */
smoe_status smoe_step(smoe_handle h, smoe_params *p, const float *target,
                      const smoe_lr *lr, smoe_stats *stats);

/* Fused records: when the training grid uses the two-stage
 * binning, the Adam update of smoe_step also writes the next step's kernel
 * records and tile boxes (the geometry of P:215-221) for the parameters it
 * just updated, and the next smoe_step / smoe_grad on the SAME parameter
 * buffers, band and box mode skips that preprocessing pass.  The library
 * notices its own calls that change parameters, records or band
 * (smoe_apply(_ex), smoe_render(_ex), smoe_bin, smoe_set_band, a failed
 * call); a caller that writes the parameter buffers itself between steps
 * must call smoe_invalidate first (the Python binding does this from the
 * tensors' version counters).  No arguments besides the handle; never fails
 * on a valid handle. */
smoe_status smoe_invalidate(smoe_handle h);

/* Multi-GPU band split (tile-row bands): restrict
 * smoe_grad to block rows [tile_row0, tile_row1) of the ceil(H/16) rows.
 * The loss normalisation stays 1/(H W C) of the full image, so per-band
 * gradients add up to the full-image gradient.  (0, 0) = whole image. */
smoe_status smoe_set_band(smoe_handle h, int tile_row0, int tile_row1);

/* Gradient of the loss restricted to the current band: grad[K][Pk] float32
 * with Pk = 6 + C E, per kernel (mu_x, mu_y, l11, l21, l22, log_pi, expert
 * block in the expert layout); sums[4] float64 = (SSE, clamped SSE, uncovered
 * pixels, skipped) of the band.  grad and sums may be host or device pointers.
 * target[C][H][W] is the full image; a host target has only the band's
 * pixel rows copied to the device (the other rows are never read).
 * Capacity: with grad and sums both on the device the call is asynchronous;
 * if the band's block lists overflowed their capacity the raster is skipped,
 * grad is written as zeros and sums = (0, 0, 0, 1): the caller must not apply
 * that gradient (smoe_apply_ex with `sums` does the check on the device) and
 * the next synchronising call (smoe_sync) grows the lists and returns
 * SMOE_ERR_CAPACITY.  With a host grad or sums the call synchronises, grows
 * and redoes the pass itself (sums[3] = 0). */
smoe_status smoe_grad(smoe_handle h, const smoe_params *p, const float *target,
                      float *grad, double *sums);

/* Adam update with a caller-supplied gradient (e.g. all-reduced over ranks):
 * same update and clamp as smoe_step.  grad[K][Pk] host or device. */
smoe_status smoe_apply(smoe_handle h, smoe_params *p, const float *grad, const smoe_lr *lr);

/* Sharded Adam update (multi-GPU reduce-scatter -> per-rank update ->
 * all-gather): updates kernels [k0, k1) only, with
 * grad[(k1-k0)][Pk] (rows relative to k0; host or device) and the Adam
 * moments of those kernels; parameters of other kernels are untouched.
 * `sums` (NULL, or the all-reduced sums[4] of smoe_grad, host or device):
 * if sums[3] != 0 some rank's binning overflowed and no parameter is updated
 * (checked on the device for a device pointer, so the call stays
 * asynchronous).  0 <= k0 <= k1 <= K.  The Adam step counter advances when
 * k1 > k0 and the update is not skipped. */
smoe_status smoe_apply_ex(smoe_handle h, smoe_params *p, const float *grad, const smoe_lr *lr, int k0, int k1,
                          const double *sums);

/* Zero the Adam moments and the step counter. */
smoe_status smoe_reset_adam(smoe_handle h);

/* Checkpoint / resume of the optimiser state: the first and
 * second Adam moments as m1[K][Pk], m2[K][Pk] float32 (gradient layout, host
 * or device) and the step counter t.  Together with the caller-owned
 * parameters this resumes a fit (identical up to the run-to-run rounding
 * order of the backward's float atomics).  Synchronous. */
smoe_status smoe_get_adam(smoe_handle h, float *m1, float *m2, long long *t);
smoe_status smoe_set_adam(smoe_handle h, const float *m1, const float *m2, long long t);

/* Stream-ordered statistics for pipelined loops: smoe_stats_async enqueues
 * a device->host copy of the most recent step's raw statistics into `dst`
 * (caller-owned, ideally pinned host memory) without synchronising; once the
 * caller knows the copy completed (a later smoe_sync, an event, or reading
 * it k steps later after a sync), smoe_stats_from_raw converts it. */
typedef struct {
    double sse, sse_clamped, uncovered;
    long long pairs;
} smoe_raw_stats;
smoe_status smoe_stats_async(smoe_handle h, smoe_raw_stats *dst);
smoe_status smoe_stats_from_raw(smoe_handle h, const smoe_raw_stats *raw, smoe_stats *out);

/* Wait for the handle's stream and report latched device faults.  If `last`
 * is non-NULL it receives the statistics of the most recent step/grad. */
smoe_status smoe_sync(smoe_handle h, smoe_stats *last);

/* Diagnostic view of the block binning on an out_H x out_W
 * raster: tile_range[n_tiles+1] (int32, [start, end) of block n), ids[P]
 * (int32 kernel ids, ascending within a block) and tilebox[K][4] int32
 * (tx0, tx1, ty0, ty1; -1 when the box misses the raster).  Synchronous.
 * Any output pointer may be NULL; ids must hold ids_cap entries.
 * *n_pairs receives P. */
smoe_status smoe_bin(smoe_handle h, const smoe_params *p, int out_H, int out_W,
                     int *tile_range, int *ids, long long ids_cap, long long *n_pairs,
                     int *tilebox);

/* The paper's mu learning rate at 0-based step t of a T-step fit:
 * 0.01 * (1e-3)^(t/T), and the fixed group rates. */
smoe_lr smoe_paper_lr(int t, int T);

/* Device-time profiling of the library's own launches (bench.py uses it to
 * time the dominant kernel inside the timed region, on the handle's stream).
 * smoe_profile_begin: record a CUDA event pair around each of the next
 * max_launches launches of the kernels in kernel_mask (bit i = kernel id i,
 * 0 = all; inside graph replays the pairs are graph event nodes); with bit
 * SMOE_PROFILE_COUNT_WORK set the rasteriser also counts the (pixel, kernel) pairs the rasteriser
 * tests and the pairs inside the truncation ellipse (the work units of the
 * roofline).  smoe_profile_end: synchronise, return per-kernel
 * totals in times[SMOE_KERNEL_COUNT] and the work counters, stop profiling. */
enum {
    SMOE_KERNEL_PREPROCESS = 0,    /* a1 + a2 (the last CTA scans); with the
                                      two-stage binning (K >= 16 384): a1 only
                                      (k_records)                             */
    SMOE_KERNEL_SCATTER = 1,       /* a3                                     */
    SMOE_KERNEL_RASTER_TRAIN = 2,  /* a4 (bucket sort) + a5-a7               */
    SMOE_KERNEL_RASTER_RENDER = 3, /* a4 + a5/a9                             */
    SMOE_KERNEL_ADAM = 4,          /* a8                                     */
    SMOE_KERNEL_BIN = 5,           /* a1-a3 fused cooperative binner (CSR)   */
    SMOE_KERNEL_SCAN = 6,          /* a2 decoupled look-back scan (CSR)      */
    SMOE_KERNEL_EMIT = 7,          /* a3 two-stage binning: CTA-aggregated
                                      bucket emission over a spatial order     */
    SMOE_KERNEL_COUNT = 8
};
#define SMOE_PROFILE_COUNT_WORK 0x80000000u
typedef struct {
    double total_ms;
    long long launches;
} smoe_kernel_time;
typedef struct {
    long long tested_pairs;   /* valid pixel x listed kernel, forward sweep */
    long long hit_pairs;      /* of those, d^2 <= R2                        */
    long long sort_cycles;    /* SM cycles the raster CTAs spent in the a4
                                 bucket sort (summed over CTAs)             */
    long long cta_cycles;     /* SM cycles of the raster CTAs in total      */
} smoe_work;
smoe_status smoe_profile_begin(smoe_handle h, int max_launches, unsigned kernel_mask);
smoe_status smoe_profile_end(smoe_handle h, smoe_kernel_time *times, smoe_work *work);
const char *smoe_kernel_name(int id);

/* Segmentation-guided initialisation (Eq. 9,
 * P:424 thresholds 10/20), host code run once before a fit.  The paper only
 * cites its "modified DBSCAN"; this implements the reading of S:417-438:
 * smoe_segment: 4-connected region growing on the host image[C][H][W] in
 * [0,1]: a pixel joins the region when the max-channel |pixel - running
 * mean| <= threshold (0-255 scale); regions smaller than min_size merge into
 * the closest adjacent region.  labels[H][W] (host) receive ids 0..N-1,
 * *n_segments = N.
 * smoe_segment_init: K kernels over the N segments, max(1, floor(K|R|/HW))
 * each plus largest-remainder top-up to exactly K (Eq. 9: |B_j| ~ |R_j|/n_k);
 * centres uniform over the segment's pixels, L = (scale_px, 0, scale_px),
 * log_pi = 0, expert = segment mean colour, slopes 0.  Outputs are HOST
 * arrays in the smoe_params layout.  K < N, H < 1, W < 1, a label outside
 * [0, N) or a segment id in [0, N) that owns no pixel give
 * SMOE_ERR_INVALID_ARG. */
smoe_status smoe_segment(const float *image, int H, int W, int C, float threshold, int min_size, int *labels,
                         int *n_segments);
smoe_status smoe_segment_init(const float *image, int H, int W, int C, const int *labels, int n_segments, int K,
                              int expert_order, unsigned long long seed, float scale_px, float *mu, float *chol,
                              float *log_pi, float *expert);

/* Number of device kernel launches issued by the library since creation. */
long long smoe_launch_count(smoe_handle h);

const char *smoe_status_string(smoe_status s);
const char *smoe_last_error(smoe_handle h);
int smoe_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SMOE_H */
