/*
 * vdamp_b200.h -- C ABI of the B200-native VDAMP hot path.
 *
 * The reference (csmri, pure Python/numpy) has no FFI of its own; its public
 * boundary for this path is the Python function
 *     csmri.vdamp.run(y, mask, pmap, noise_var, scales, n_iters,
 *                     ground_truth=None, keep_r_iters=())
 * (/root/reference/pkg/src/csmri/vdamp.py:153-197) plus the operators it
 * calls.  These entry points are what a ctypes binding of that boundary
 * binds (INTEGRATION.md shows the stub); the Python package
 * paper_1911_01234_b200 is that binding and mirrors the reference names.
 *
 * Conventions
 *   - Every function returns an int status (VDAMP_OK == 0); on failure
 *     vdamp_last_error() returns a message for the calling thread.
 *   - All data pointers are DEVICE pointers on the plan's device unless
 *     the comment says "host".  No ownership is transferred.
 *   - Complex arrays are interleaved (re, im) in the plan precision:
 *     float2 for VDAMP_FP32, double2 for VDAMP_FP64.
 *   - Images are row-major H x W, batch-major (image b at b*H*W).
 *   - Wavelet coefficient vectors use the reference flat layout
 *     (src/wavelet.py:52-61): approx_s, then (H, V, D) for scale s..1,
 *     every block row-major; image b at b*H*W.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).
 */
#ifndef VDAMP_B200_H
#define VDAMP_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define VDAMP_API __attribute__((visibility("default")))
#else
#define VDAMP_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum {
    VDAMP_OK = 0,
    VDAMP_ERR_ARG = 1,        /* bad argument (maps to ValueError)                */
    VDAMP_ERR_SHAPE = 2,      /* shape not divisible by 2^scales (DimensionError) */
    VDAMP_ERR_UNSUPPORTED = 3,/* outside the build's scope (non-power-of-two, ...) */
    VDAMP_ERR_CUDA = 4,       /* CUDA runtime error                               */
    VDAMP_ERR_OOM = 5,        /* device allocation failed                         */
    VDAMP_ERR_STATE = 6       /* call order violated (e.g. run before set_*)      */
};

enum { VDAMP_FP32 = 0, VDAMP_FP64 = 1 };

/* per (iteration, image, subband) trace record, VDAMP_TRACE_FIELDS doubles:
 *   0 tau (unfloored, src/vdamp.py:115)
 *   1 threshold t
 *   2 lambda = t / max(tau, 1e-300)            (src/denoise.py:170)
 *   3 alpha after the clamp                    (src/vdamp.py:121-124)
 *   4 alpha before the clamp                   (src/denoise.py:169)
 *   5 clamp flag (0/1)
 *   6 subband error |r - w0|^2, 7 subband energy |w0|^2
 *     (src/diagnostics.py:37-51; zero unless ground truth is set) */
#define VDAMP_TRACE_FIELDS 8
/* per (iteration, image) NMSE record: |x_hat - x0|^2, |x0|^2 (src/diagnostics.py:21-34) */
#define VDAMP_NMSE_FIELDS 2

typedef struct vdamp_plan_s* vdamp_plan_t;

VDAMP_API const char* vdamp_last_error(void);
VDAMP_API int vdamp_abi_version(void);

/* Plan for a batch of `batch` images of height x width, `scales` Haar levels.
 * Validates like SubbandLayout.create (src/wavelet.py:43-63): scales >= 1
 * (VDAMP_ERR_ARG), divisibility by 2^scales (VDAMP_ERR_SHAPE); this build
 * additionally requires power-of-two sizes in [2, 2048] (VDAMP_ERR_UNSUPPORTED).
 * Allocates all device workspace and builds the separable subband spectra
 * (replaces compute_spectra/_masked_profiles, src/vdamp.py:41-56). */
VDAMP_API int vdamp_plan_create(int height, int width, int scales, int batch, int precision,
                      int device, vdamp_plan_t* out);
VDAMP_API int vdamp_plan_destroy(vdamp_plan_t plan);
/* number of subbands S = 1 + 3*scales and their offsets/lengths (host arrays of S) */
VDAMP_API int vdamp_plan_layout(vdamp_plan_t plan, int64_t* offsets, int64_t* lengths);
VDAMP_API int vdamp_plan_workspace_bytes(vdamp_plan_t plan, size_t* bytes);

/* Measurements for every image of the batch (the per-run constants of
 * vdamp.run, src/vdamp.py:153-175; y aligned with mask.indices as in
 * KSpaceData, src/fourier.py:39-49).
 *   y         device, concatenation over images of n_b complex values
 *   indices   device int64, concatenation of each image's row-major sampled
 *             positions (mask.indices, src/fourier.py:26)
 *   counts    host int64[batch], n_b per image (>= 1)
 *   probs     device float64 H*W sampling probabilities in (0,1] per image;
 *             probs_batch_stride = 0 shares one map over the batch
 *   noise_var host float64[batch], >= 0 */
VDAMP_API int vdamp_set_measurements(vdamp_plan_t plan, const void* y, const int64_t* indices,
                           const int64_t* counts, const double* probs,
                           int64_t probs_batch_stride, const double* noise_var, void* stream);
/* Validation of the measurements (the reference raises ValueError for a bad
 * mask or density: src/fourier.py:65-74, src/sampling.py:45-46).  The
 * scatter kernel skips an index outside [0, H*W) and flags it, a repeated
 * index and a probability outside (0, 1] at a sampled point; the flags are
 * reported as VDAMP_ERR_ARG.  synchronous = 1 (default): vdamp_set_measurements
 * waits for the check and returns the error itself.  synchronous = 0 (the
 * pipelined serving path): the flags are read back asynchronously and
 * reported by the first later call on the plan that finds them landed, or by
 * vdamp_measurement_status. */
VDAMP_API int vdamp_set_validation(vdamp_plan_t plan, int synchronous);
/* VDAMP_ERR_ARG if any measurements set so far were flagged; wait = 1 blocks
 * until the last check has landed, wait = 0 reports only what has. */
VDAMP_API int vdamp_measurement_status(vdamp_plan_t plan, int wait);
/* Host-side check of HOST arrays before any upload (no device needed): the same
 * rules as the kernel plus counts in [1, H*W] and noise_var >= 0. */
VDAMP_API int vdamp_check_measurements(int height, int width, int batch, const int64_t* indices,
                                       const int64_t* counts, const double* probs,
                                       int64_t probs_batch_stride, const double* noise_var);
/* Ground truth images (complex, batch x H x W): enables the per-iteration
 * NMSE / subband NMSE records (src/vdamp.py:189-193). NULL disables. */
VDAMP_API int vdamp_set_ground_truth(vdamp_plan_t plan, const void* x0, void* stream);

/* Full loop (src/vdamp.py:153-197): reset to r_tilde_0 = 0 (initial_state,
 * src/vdamp.py:95-96), n_iters iterations, exact data-consistency finalize.
 *   x_hat       out: complex batch x H x W
 *   trace       out or NULL: float64 [n_iters][batch][S][VDAMP_TRACE_FIELDS]
 *   nmse        out or NULL: float64 [n_iters][batch][VDAMP_NMSE_FIELDS]
 *               (requires ground truth)
 *   snapshots   host array of n_iters device pointers or NULL; a non-NULL
 *               entry k receives r_k (batch x N complex), src/vdamp.py:194-195 */
VDAMP_API int vdamp_run(vdamp_plan_t plan, int n_iters, void* x_hat, double* trace, double* nmse,
              void* const* snapshots, void* stream);

/* Step-wise interface (src/vdamp.py:99-144) for teacher forcing:
 * one iteration from a caller-given r_tilde (batch x N complex).
 * Outputs (any may be NULL): r, r_tilde_next, w_hat (batch x N complex),
 * trace [batch][S][VDAMP_TRACE_FIELDS]. */
VDAMP_API int vdamp_iterate(vdamp_plan_t plan, const void* r_tilde, void* r, void* r_tilde_next,
                  void* w_hat, double* trace, void* stream);

/* Operators on the plan's geometry (batch images each). */
VDAMP_API int vdamp_dwt(vdamp_plan_t plan, const void* image, void* coeffs, void* stream);    /* src/wavelet.py:132-148 */
VDAMP_API int vdamp_idwt(vdamp_plan_t plan, const void* coeffs, void* image, void* stream);   /* src/wavelet.py:169-181 */
VDAMP_API int vdamp_fft2c(vdamp_plan_t plan, const void* in, void* out, int inverse, void* stream); /* src/fourier.py:52-59 */
/* finalize (src/vdamp.py:147-150) of caller-given w_hat; needs measurements */
VDAMP_API int vdamp_finalize(vdamp_plan_t plan, const void* w_hat, void* x_hat, void* stream);
/* denoise_colored (src/denoise.py:147-178): tau device float64 [batch][S] (> 0);
 * w_hat complex out (NULL ok); trace [batch][S][VDAMP_TRACE_FIELDS] out (NULL ok)
 * carries t, lambda and alpha (field 4 = unclamped, as denoise_colored returns). */
VDAMP_API int vdamp_denoise_colored(vdamp_plan_t plan, const void* r, const double* tau, void* w_hat,
                          double* trace, void* stream);

/* Baselines on the same kernels (src/baselines.py): algorithm 0 = FISTA with the
 * global threshold lam[b] (device float64 [batch]); 1 = SURE-IT with the oracle
 * tau_k = |r_k - w0|^2 / N (needs vdamp_set_ground_truth).  Set measurements with
 * p = 1 (no density compensation).  x_hat = idwt(w_hat); trace (SURE-IT: tau, t,
 * lambda, alpha per subband; FISTA: fields 6/7 = |w_hat - w0|^2, |w0|^2 per
 * subband) and nmse ([n_iters][batch][2] of w_hat vs w0, = image NMSE since Psi
 * is orthonormal) are optional. */
VDAMP_API int vdamp_baseline_run(vdamp_plan_t plan, int algorithm, int n_iters, const double* lam, void* x_hat,
                                 double* trace, double* nmse, void* stream);

/* Monte Carlo accumulation over the batch (reference tests/conftest.py:41-81):
 *   r       batch x N complex iterates r_k of one iteration k, one per draw
 *   w0      N complex reference coefficients dwt(x0)
 *   sum_r   N complex128 (float64 pairs), += sum over draws of r_b
 *   sum_sq  S float64, += per-subband mean over entries of sum over draws |r_b - w0|^2
 *   scratch N float64 workspace */
VDAMP_API int vdamp_mc_accumulate(vdamp_plan_t plan, const void* r, const void* w0, double* sum_r,
                                  double* sum_sq, double* scratch, void* stream);

/* Instrumentation.  Kernel classes: 0 synthesis+row FFT, 1 column FFT/residual,
 * 2 row IFFT+analysis, 3 SURE select, 4 finalize, 5 other. */
#define VDAMP_KERNEL_CLASSES 6
VDAMP_API int vdamp_set_timing(vdamp_plan_t plan, int enable);
/* Synchronises the recorded events; ms[c] = summed device time, launches[c] = count. */
VDAMP_API int vdamp_kernel_times(vdamp_plan_t plan, double* ms, int64_t* launches);
/* vdamp_run captures its whole launch sequence as a CUDA graph (default: on for
 * plans of at most 64 x 256^2 pixels, where the host's launch rate limits the run;
 * env VDAMP_GRAPHS=0/1 overrides) and replays it while the outputs, iteration count,
 * stream and flags are unchanged; the graphs of the last few other combinations are
 * kept (a pipelined caller alternating output buffers never re-captures).  With
 * timing enabled each graph run synchronises once to accumulate the kernel times. */
VDAMP_API int vdamp_set_graphs(vdamp_plan_t plan, int enable);
/* Image lanes of vdamp_run (with trace, NMSE or snapshots only when interleaved,
 * each lane writing its image range of every record): the batch runs as `lanes` contiguous image ranges on their own streams, forked from
 * and joined back into the caller's stream, launched iteration-major (every lane
 * gets iteration k before any lane gets k+1; env VDAMP_INTERLEAVE=0: lane-major).
 * When graphs are on, the fork/join is captured into the graph.  Results are
 * identical for any lane count (images are independent).  Default min(4, batch / 16) (2 from 128 images, 1 from 256), env VDAMP_LANES overrides;
 * lanes = 0 restores the default. */
VDAMP_API int vdamp_set_lanes(vdamp_plan_t plan, int lanes);
/* Per-iteration device time of vdamp_run (the reference records each iteration's own
 * wall time, src/vdamp.py:176-179): when enabled, CUDA events bracket K1..K4 of every
 * iteration on the stream of the first image lane.  vdamp_iteration_times (after the
 * run; synchronises) returns ms[k] for k < n_iters and *images = the images sharing
 * that stream (the per-image share of an iteration is ms[k] / *images). */
VDAMP_API int vdamp_set_iteration_timing(vdamp_plan_t plan, int enable);
VDAMP_API int vdamp_iteration_times(vdamp_plan_t plan, int n_iters, double* ms, int* images);
/* total kernel launches issued by this plan since creation or the last reset */
VDAMP_API int vdamp_launch_count(vdamp_plan_t plan, int64_t* count, int reset);

#ifdef __cplusplus
}
#endif
#endif /* VDAMP_B200_H */
