/*
 * fdl_b200.h — C ABI of the B200-native Fourier Disparity Layer hot paths.
 *
 * The reference (`fdl`, /root/reference/pkg/src/fdl) is pure Python/numpy and
 * has no FFI of its own; these entry points are what its Python layer would
 * bind (ctypes stub in INTEGRATION.md) to replace, stage by stage:
 *
 *   fdl_views_to_spectra   np.pad + np.fft.rfft2 + sum |b|^2   construct.py:250-266
 *   fdl_solve_bins         _phase_tables/_system_chunk/_solve_chunk
 *                          (per-frequency regularised LS)      construct.py:68-80,168-211,277-284
 *   fdl_symmetrize         self-conjugate column post-pass      construct.py:286-297
 *   fdl_render_spectra     evaluate_scaled_grid + _weighted_layer_sum
 *                                                               lfmodel.py:101-122, render.py:190-207,238-245
 *   fdl_spectra_to_images  irfft_fast + crop + srgb_encode      spectra.py:202-208, render.py:210-225
 *   fdl_audit_bins /       the 1e-8 normal-equation residual test and the minimum-norm
 *   fdl_resolve_bins       fallback `_stacked_lstsq`                construct.py:157-165,196-210
 *   fdl_calib_solve/_terms _solve_batch, _objective_terms, _grad_p  calibrate.py:139-229
 *   fdl_view_sqerr         psnr / mse_per_channel numerators        pipeline.py:30-51
 *   fdl_images_to_u8       the service's 8-bit quantisation         serve.py:127
 *   fdl_dequantise_views   the loader's 8- / 16-bit decode           io.py:54-59
 *
 * Conventions (all calls):
 *   - return 0 (FDL_OK) on success, a negative FDL_ERR_* code otherwise; the
 *     message is available from fdl_last_error() (thread-local);
 *   - every buffer named *_dev is caller-allocated DEVICE memory, every other
 *     pointer is HOST memory read during the call (not retained);
 *   - work is enqueued on `stream` (a cudaStream_t, NULL = legacy default
 *     stream) and is stream-ordered; no call synchronises the device unless
 *     stated; no global mutable state is shared between calls (re-entrant,
 *     one call per stream at a time);
 *   - complex numbers are interleaved (re, im) pairs: fdl_c64 = 2 x float.
 *
 * Data layouts in HBM:
 *   views    (m, H, W, C)            float32   (ViewSet.images order, lfmodel.py:125-191)
 *   spectra  (m, C, rows, Whp)       fdl_c64   Whp = Wp/2 + 1 (half-plane, spectra.py:41-101)
 *   layers   (n, C, rows, Whp)       fdl_c64   (FDL1 file order, io.py:175)
 *   images   (V, H, W, C)            float32
 * where `rows` is the number of frequency rows of the slab held by this call
 * (all Hp rows on one GPU; a mirrored-pair slab on a multi-GPU shard).
 */
#ifndef FDL_B200_H
#define FDL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FDL_OK 0
#define FDL_ERR_INVALID -1      /* invalid argument (reference: ValueError) */
#define FDL_ERR_CUDA -2         /* CUDA / cuFFT failure */
#define FDL_ERR_UNSUPPORTED -3  /* shape outside this build's kernels */
#define FDL_ERR_RANK -4         /* singular unregularised system (reference: RankDeficiencyError) */

/* per-bin status written by fdl_solve_bins */
#define FDL_BIN_OK 0
#define FDL_BIN_BREAKDOWN 1     /* Cholesky pivot <= 0 or non-finite result */
#define FDL_BIN_SUSPECT 2       /* solved, but max diag(G) ||x|| / ||rhs|| is large enough that the reference's
                                   1e-8 residual test (construct.py:198-204) could fire: run fdl_audit_bins */

typedef struct fdl_c64 { float re, im; } fdl_c64;

/* Sampled aperture spectrum psi_hat (ApertureSpec, lfmodel.py:39-122).
 * table is (rows, cols) row-major, float64; table_im NULL for a real table.
 * Axis k has node i at xi0_k + i * step_k (lfmodel.py:72-79 uses
 * step = xi[1] - xi[0] and pos = (q - xi[0]) / step). */
typedef struct fdl_aperture {
  int32_t rows, cols;
  const double* table_re;
  const double* table_im;
  double xi0_x, step_x;
  double xi0_y, step_y;
} fdl_aperture;

/* ------------------------------------------------------------------------ */
/* Library                                                                   */
/* ------------------------------------------------------------------------ */

int fdl_version(void);
const char* fdl_last_error(void);

/* Device self-test of the FP64 tensor-core (DMMA) fragment layouts the K1
 * kernels rely on; *max_err receives the largest deviation (synchronises). */
int fdl_selftest(double* max_err);

/* Kernel-launch timer (measurement instrumentation for bench.py, not part of
 * the reference interface).  While enabled, the library records a pair of CUDA
 * events on the launch stream around every launch of its main kernels:
 *   FDL_TIMER_K1  the per-bin solve kernel of fdl_solve_bins (K1),
 *   FDL_TIMER_K3  the main render-spectra tile of fdl_render_spectra (K3).
 * fdl_kernel_timer(1) clears and enables (this host thread); fdl_kernel_timer(0)
 * disables.  fdl_kernel_timer_read synchronises on the recorded events and
 * returns the summed launch durations and the launch count of one kernel. */
#define FDL_TIMER_K1 0
#define FDL_TIMER_K3 1
int fdl_kernel_timer(int32_t enable);
int fdl_kernel_timer_read(int32_t which, double* total_ms, int32_t* launches);

/* CUDA-graph capture support.  The entry points stage their host parameter
 * blocks through a reused pinned ring (a reuse waits on an event), which a
 * captured graph must not depend on.  Between fdl_staging_arena_begin() and
 * fdl_staging_arena_end() on this host thread every block is staged in a fresh
 * pinned allocation owned by the arena and nothing synchronises, so the calls
 * can be stream-captured (pass n_breakdown = NULL to fdl_solve_bins) and the
 * graph replayed for as long as the arena lives; fdl_staging_arena_free()
 * releases it after the graph is destroyed.  Warm every call up once before
 * capturing (cuFFT plans, constant tables and kernel attributes are set up on
 * first use). */
void* fdl_staging_arena_begin(void);
int fdl_staging_arena_end(void* arena);
int fdl_staging_arena_free(void* arena);

/* Test hook (not part of the reference interface): force_cufft = 1 makes K0 /
 * K4 on this host thread use cuFFT even where the library's own FFT engine
 * applies (grid sides 67 * 2^a, 131 * 2^a), so tests can compare the two. */
int fdl_fft_force_cufft(int32_t force_cufft);

/* ------------------------------------------------------------------------ */
/* K0: pad + R2C + per-view sum |b|^2   (construct.py:250-266)               */
/* ------------------------------------------------------------------------ */

/* Bytes of device workspace fdl_views_to_spectra needs. */
size_t fdl_views_to_spectra_workspace(int32_t m, int32_t H, int32_t W, int32_t C, int32_t pad);

/* views_dev (m,H,W,C) f32 -> spectra_dev (m,C,Hp,Whp) c64 with Hp = H + 2 pad,
 * Wp = W + 2 pad; view_sumsq_dev (m) float64 receives sum_{c,q} |b|^2 per view
 * (the joint-over-channels numerator of default_lambda, construct.py:214-216). */
int fdl_views_to_spectra(const float* views_dev, int32_t m, int32_t H, int32_t W, int32_t C,
                         int32_t pad, fdl_c64* spectra_dev, double* view_sumsq_dev,
                         void* workspace_dev, size_t workspace_bytes, void* stream);

/* fdl_views_to_spectra for sRGB-encoded views: every value is decoded to
 * linear light (render.py:39-42 srgb_decode) as K0 loads it, so a caller
 * gets the spectra of srgb_decode(views) -- what the reference builds from
 * after load_lightfield(..., to_linear=True) (io.py:147-149) -- without a
 * decoded copy of the views in HBM.  Same workspace as fdl_views_to_spectra. */
int fdl_views_to_spectra_srgb(const float* views_dev, int32_t m, int32_t H, int32_t W, int32_t C,
                              int32_t pad, fdl_c64* spectra_dev, double* view_sumsq_dev,
                              void* workspace_dev, size_t workspace_bytes, void* stream);

/* Gather whole frequency rows of view spectra into a contiguous slab:
 * dst (m, C, nrows, Whp) <- src (m, C, Hp, Whp)[..., rows[i], :].  Used to pack
 * the all-to-all send buffers of the multi-GPU path. */
int fdl_gather_rows(const fdl_c64* src_dev, int32_t m, int32_t C, int32_t Hp, int32_t Whp,
                    const int32_t* rows_dev, int32_t nrows, fdl_c64* dst_dev, void* stream);

/* default_lambda on the device (construct.py:214-216): lam = 1e-4 * (sum_j
 * view_sumsq[j] / Q) / m, the per-view sums added in view order by one thread
 * -- bit-identical to the host formula for any sharding of the views. */
int fdl_default_lambda(const double* view_sumsq_dev, int32_t m, int64_t Q, double* lam_dev, void* stream);

/* ------------------------------------------------------------------------ */
/* K1: per-bin regularised least squares   (construct.py:168-211)           */
/* ------------------------------------------------------------------------ */

typedef struct fdl_solve_desc {
  int32_t m, n, C;         /* views, layers, channels */
  int32_t Hp, Wp;          /* padded grid; Whp = Wp/2 + 1 */
  int32_t nrows;           /* frequency rows in this slab */
  const int32_t* rows;     /* host, nrows ky indices (NULL: rows 0..nrows-1) */
  /* shift model (ShiftParams, lfmodel.py:204-267): factored (u, v) or relaxed (pu, pv) */
  const double* u;         /* host, m (NULL when relaxed) */
  const double* v;         /* host, m */
  const double* pu;        /* host, m*n row-major (NULL when factored) */
  const double* pv;        /* host, m*n */
  const double* d;         /* host, n layer disparities */
  /* wide-aperture views (construct.py:170-179); view_aperture NULL = all pinhole */
  const int32_t* view_aperture; /* host, m: index into apertures or -1 for a pinhole */
  const double* s;         /* host, m refocus parameters */
  const double* scale;     /* host, m aperture scales */
  int32_t n_apertures;
  const fdl_aperture* apertures;
  double lam, eps;         /* lambda (>= 0) and the absolute eps of reg (construct.py:283) */
  const fdl_c64* spectra_dev;  /* (m, C, nrows, Whp) */
  fdl_c64* layers_dev;         /* (n, C, nrows, Whp) */
  int8_t* status_dev;          /* (nrows, Whp) FDL_BIN_* or NULL */
  int32_t force_path;          /* 0 = auto; 1 = symmetric-real, 2 = real-A, 3 = complex embedding;
                                  4 = auto formulation on the generic (non-DMMA) kernel (testing) */
  int32_t plane_rows;          /* 0: spectra/layers hold just the slab rows (buffer row i <-> rows[i]);
                                  Hp: full-grid buffers (m or n, C, Hp, Whp) and the listed rows
                                  are solved in place (buffer row rows[i]); status stays
                                  (nrows, Whp).  Lets a caller solve a full spectrum in row slabs. */
  const double* lam_dev;       /* optional device scalar that replaces lam (the default lambda
                                  computed on the device by fdl_default_lambda: no host round trip
                                  between K0 and K1); NULL: use lam */
} fdl_solve_desc;

/* Bytes of device workspace fdl_solve_bins needs (0 for the current kernels
 * beyond the parameter block; always query). */
size_t fdl_solve_bins_workspace(const fdl_solve_desc* desc);

/* Solve every bin of the slab.  Returns FDL_OK even when some bins break
 * down or are suspect; they are flagged in status_dev (FDL_BIN_BREAKDOWN /
 * FDL_BIN_SUSPECT) and counted together in *n_breakdown when non-NULL (which
 * synchronises the stream). */
int fdl_solve_bins(const fdl_solve_desc* desc, void* workspace_dev, size_t workspace_bytes,
                   int32_t* n_breakdown, void* stream);

/* Which path fdl_solve_bins picks for this descriptor (1, 2, 3 as force_path). */
int fdl_solve_path(const fdl_solve_desc* desc);

/* Re-solve the bins fdl_solve_bins flagged (FDL_BIN_BREAKDOWN) with the
 * reference's minimum-norm fallback `_stacked_lstsq` (construct.py:157-165,
 * 205-210): A, b and reg of each listed bin are rebuilt on the device and
 * [A; sqrt(lam reg)] x = [b; 0] is solved by an fp64 Jacobi SVD.  bins is a
 * HOST array of flat slab bin indices (row * Whp + kx).  lam must be > 0. */
size_t fdl_resolve_bins_workspace(const fdl_solve_desc* desc, int32_t nbins);
int fdl_resolve_bins(const fdl_solve_desc* desc, const int32_t* bins, int32_t nbins, void* workspace_dev,
                     size_t workspace_bytes, void* stream);

/* The reference's per-bin acceptance test (construct.py:198-210) on the bins
 * fdl_solve_bins marked FDL_BIN_SUSPECT: A, b and reg of each listed bin are
 * rebuilt on the device, the normal equations are solved in fp64 (LDL^H), and a
 * bin whose residual ||G x - rhs||_F exceeds 1e-8 ||rhs||_F is re-solved by the
 * minimum-norm `_stacked_lstsq` (lam > 0).  The layers of every listed bin are
 * rewritten and status_dev becomes FDL_BIN_OK / FDL_BIN_BREAKDOWN.
 * audit_status (HOST, nbins; the call synchronises): 0 normal equations
 * accepted, 2 minimum-norm fallback used, 1 fallback failed, 3 test failed at
 * lam = 0 (the reference raises RankDeficiencyError).  Workspace: as
 * fdl_resolve_bins_workspace.  desc->lam_dev must be NULL (pass lam). */
int fdl_audit_bins(const fdl_solve_desc* desc, const int32_t* bins, int32_t nbins, int8_t* audit_status,
                   void* workspace_dev, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------ */
/* Explicit per-bin systems   (solve_frequency, construct.py:123-165)        */
/* ------------------------------------------------------------------------ */

typedef struct fdl_dense_desc {
  int32_t batch, m, n, C;      /* problems, rows, unknowns (<= 64), right-hand sides */
  const void* A_dev;           /* (batch, m, n) complex128 */
  const void* b_dev;           /* (batch, m, C) complex128 */
  const double* reg_dev;       /* (batch, n) diagonal regulariser, or NULL */
  const void* R_dev;           /* (batch, n, n) complex128 Hermitian regulariser, or NULL */
  double lam;                  /* >= 0 */
  void* x_dev;                 /* (batch, n, C) complex128 */
  int8_t* status_dev;          /* (batch): 0 normal equations accepted, 2 minimum-norm fallback used,
                                  1 fallback failed, 3 singular / inaccurate at lam = 0 */
} fdl_dense_desc;

size_t fdl_solve_dense_workspace(const fdl_dense_desc* desc);
int fdl_solve_dense(const fdl_dense_desc* desc, void* workspace_dev, size_t workspace_bytes, void* stream);

/* Minimum-norm least squares x = lstsq(A, b) per problem (numpy's rcond=None
 * cutoff), fp64 one-sided Jacobi SVD: the reference's degenerate-case
 * fallback in the calibration solve (calibrate.py:164-169, lstsq(G, rhs)).
 * A (batch, rows, n), b (batch, rows, C), x (batch, n, C) complex128;
 * status (batch): 2 solved (the dense API's "minimum-norm solution" code), 1 failed. */
size_t fdl_lstsq_minnorm_workspace(int32_t batch, int32_t rows, int32_t n, int32_t C);
int fdl_lstsq_minnorm(int32_t batch, int32_t rows, int32_t n, int32_t C, const void* A_dev, const void* b_dev,
                      void* x_dev, int8_t* status_dev, void* workspace_dev, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------ */
/* Calibration batches   (calibrate.py:139-229)                             */
/* ------------------------------------------------------------------------ */

/* One stochastic-descent evaluation over B frequency bins of the (unpadded)
 * luminance spectra: A_jk = exp(2 pi i (Pu_jk wx + Pv_jk wy)) with the
 * reference's phase rounding (`_system_batch`, calibrate.py:139-141),
 * x = (A^H A + lam Gamma^T Gamma)^-1 A^H b (`_solve_batch`, :157-170),
 * objective sum |A x - b|^2 + lam |Gamma x|^2 (`_objective_terms`, :172-178)
 * and the shift-matrix gradients 4 pi sum_q w_q Im(conj(x_qk) conj(A_qjk) r_qj)
 * (`_grad_p`, :219-229), summed over the batch in a fixed order. */
typedef struct fdl_calib_desc {
  int32_t m, n, B;            /* views, layers (<= 64), bins in this batch */
  int32_t H, W;               /* spectrum grid: H rows x (W/2 + 1) stored columns */
  const int32_t* bins;        /* host, B: flat stored-bin indices ky * (W/2+1) + kx */
  const double* pu;           /* host, (m, n) */
  const double* pv;           /* host, (m, n) */
  const double* gamma;        /* host, (n, n) the layer regulariser Gamma (calibrate.py:113-123) */
  double lam;                 /* >= 0 */
  const void* spec_dev;       /* (H * (W/2+1), m) complex128 luminance spectra */
  void* x_dev;                /* (B, n) complex128: written by _solve, read by _terms */
  int8_t* status_dev;         /* (B): 0 solved, 2 Cholesky breakdown (G, rhs left for the fallback) */
  void* gfall_dev;            /* (B, n, n) complex128: G of flagged bins */
  void* rfall_dev;            /* (B, n) complex128: rhs of flagged bins */
  double* obj_dev;            /* (1): sum of the batch's objective terms (_terms) */
  double* grad_dev;           /* (2, m, n): gradients w.r.t. Pu and Pv summed over the batch, or NULL */
} fdl_calib_desc;

size_t fdl_calib_workspace(const fdl_calib_desc* desc);
int fdl_calib_solve(const fdl_calib_desc* desc, void* workspace_dev, size_t workspace_bytes, void* stream);
int fdl_calib_terms(const fdl_calib_desc* desc, void* workspace_dev, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------ */
/* K2: conjugate-pair symmetrisation of self-conjugate columns (construct.py:286-297) */
/* ------------------------------------------------------------------------ */

/* layers (n, C, nrows, Whp); rows/mirror are host arrays: mirror[i] is the
 * slab index of row (Hp - rows[i]) % Hp (must be in the slab). */
int fdl_symmetrize(fdl_c64* layers_dev, int32_t n, int32_t C, int32_t Hp, int32_t Wp,
                   int32_t nrows, const int32_t* rows, const int32_t* mirror, void* stream);

/* K2 on a subset of the rows of full-grid layers (n, C, Hp, Whp): every
 * (ky, Hp-ky) pair listed in rows (host, nrows; the set must be closed under
 * ky -> (Hp-ky) % Hp) is symmetrised as fdl_symmetrize does. */
int fdl_symmetrize_rows(fdl_c64* layers_dev, int32_t n, int32_t C, int32_t Hp, int32_t Wp,
                        int32_t nrows, const int32_t* rows, void* stream);

/* Stream-ordered copy of the frequency rows [r0, r1) of every (layer,
 * channel) plane of full-grid layers (planes, Hp, Whp) into the same rows of
 * a host array of the same shape (pinned memory for asynchrony): one 2D copy.
 * Used to overlap the read-back of finished row slabs with the solves. */
int fdl_rows_to_host(const fdl_c64* layers_dev, fdl_c64* layers_host, int32_t planes, int32_t Hp,
                     int32_t Whp, int32_t r0, int32_t r1, void* stream);

/* ------------------------------------------------------------------------ */
/* K3: batched render spectra   (render.py:190-207, lfmodel.py:101-122)      */
/* ------------------------------------------------------------------------ */

typedef struct fdl_render_desc {
  int32_t n, C, Hp, Wp;    /* layers (n, C, Hp, Whp) */
  int32_t V;               /* output views in this batch */
  const double* d;         /* host, n */
  const double* pu;        /* host, V*n per-(view, layer) x shifts (u_v * d_k for render) */
  const double* pv;        /* host, V*n */
  const double* t;         /* host, V*n aperture scale t = f (s - d_k); ignored where view_aperture < 0 */
  const int32_t* view_aperture; /* host, V (NULL = all pinhole) */
  int32_t n_apertures;
  const fdl_aperture* apertures;
  const fdl_c64* layers_dev;
  fdl_c64* out_dev;        /* (V, C, Hp, Whp) */
  int64_t* oob_dev;        /* (V) out-of-range aperture lookups (lfmodel.py:118-121), or NULL */
} fdl_render_desc;

size_t fdl_render_workspace(const fdl_render_desc* desc);
/* O(1) upper bound of fdl_render_workspace (no scan of the descriptor's arrays):
 * aperture_entries = sum of rows*cols over the batch's aperture tables. */
size_t fdl_render_workspace_bound(int32_t n, int32_t C, int32_t Hp, int32_t Wp, int32_t V, int32_t n_apertures,
                                  int64_t aperture_entries);
int fdl_render_spectra(const fdl_render_desc* desc, void* workspace_dev, size_t workspace_bytes,
                       void* stream);

/* ------------------------------------------------------------------------ */
/* K4: C2R + crop + optional sRGB   (spectra.py:202-208, render.py:210-225) */
/* ------------------------------------------------------------------------ */

size_t fdl_spectra_to_images_workspace(int32_t V, int32_t C, int32_t Hp, int32_t Wp);

/* spectra (V, C, Hp, Whp) c64 (DESTROYED: used as the C2R input; its
 * self-conjugate columns are first projected onto their Hermitian part, which
 * is what numpy's irfft2 inverts) -> images (V, Ho, Wo, C) f32, cropped to [pad, pad+Ho) x
 * [pad, pad+Wo) (pass pad = 0, Ho = Hp, Wo = Wp for no crop), sRGB-encoded
 * when srgb != 0. */
int fdl_spectra_to_images(fdl_c64* spectra_dev, int32_t V, int32_t C, int32_t Hp,
                          int32_t Wp, int32_t pad, int32_t Ho, int32_t Wo, int32_t srgb,
                          float* images_dev, void* workspace_dev, size_t workspace_bytes,
                          void* stream);

/* ------------------------------------------------------------------------ */
/* K6: GPU-resident pipeline report and service quantisation                 */
/*     (pipeline.py:30-51,205-218; serve.py:127)                             */
/* ------------------------------------------------------------------------ */

/* sqerr_dev (V, C) float64 <- sum over pixels of (images - ref)^2 per view and
 * channel, the numerators of `psnr` / `mse_per_channel` (pipeline.py:30-51):
 * images_dev (V, H, W, C) f32 renders, ref_dev (V, H, W, C) the input views
 * (f32, or f64 when ref_is_f64 != 0).  Differences and sums in float64, fixed
 * summation order (the report does not depend on scheduling). */
size_t fdl_view_sqerr_workspace(int32_t V, int32_t C);
int fdl_view_sqerr(const float* images_dev, const void* ref_dev, int32_t ref_is_f64, int32_t V, int32_t H,
                   int32_t W, int32_t C, double* sqerr_dev, void* workspace_dev, size_t workspace_bytes,
                   void* stream);

/* out_dev[i] = uint8(round_half_even(clip(images_dev[i], 0, 1) * 255)), evaluated
 * in float64 like the service's encoder input (serve.py:127). */
int fdl_images_to_u8(const float* images_dev, int64_t count, uint8_t* out_dev, void* stream);

/* out_dev[i] = float32(float64(q_dev[i]) / (2^bits - 1)), bits = 8 (uint8 samples) or 16
 * (uint16): the reference loader's decode (io.py:54-59, arr.astype(float64) / 255.0 or
 * / 65535.0) followed by the float32 cast of the upload, evaluated on the device so that
 * quantised views cross PCIe as 1 or 2 bytes per sample.  Correctly rounded fp64 division,
 * then round-to-nearest-even to float32: bit-identical to the host decode. */
int fdl_dequantise_views(const void* q_dev, int32_t bits, int64_t count, float* out_dev, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FDL_B200_H */
