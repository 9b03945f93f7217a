/*
 * seqreg_b200.h — C-ABI of the B200 (sm_100a) engine for the groupwise
 * correlation dissimilarity D(y) and its gradient (arXiv 2001.06613).
 *
 * The reference (`seqreg`, pure Python) has no FFI.  Its hot-path boundary is
 * the Python trio
 *     correlation_state(seq, stack, subset, weights, cell_volume, threads)
 *                                          /root/reference/pkg/src/seqreg/similarity.py:128-164
 *     dissimilarity(state)                 similarity.py:167-177
 *     dissimilarity_gradient(state, seq, stack, subset, threads)
 *                                          similarity.py:180-220
 * The entry points below are what a binding of that trio needs (see
 * INTEGRATION.md for the ctypes binding and the `seqreg.temporal` rebinding).
 * Each one is a split of the trio along the device boundary:
 *
 *   sr_corr_partial   warp + feature + raw Gram over a pixel slab   (similarity.py:143-155, grid.py:199-243)
 *   [caller: NCCL all-reduce of the raw sums when the pixels are sharded]
 *   sr_corr_finalize  centre / normalise / C / degenerate / D / gradient
 *                     coefficients                                  (similarity.py:73-87,154-155,167-177,203-211)
 *   sr_grad           re-warp + chain rule back to y or to the affine
 *                     parameters                                    (similarity.py:203-220, grid.py:246-253)
 *   sr_curvature      curvature regulariser S(y) and its gradient   (absent in the reference)
 *   sr_evaluate_reg   sr_evaluate + S(y) (fused into pass 2 on the split NGF path)
 *   sr_sample         warped values T_j(y_j(x)) (CorrelationState.features; off the evaluation path)
 *   sr_ls_predict     temporal prolongation: smoothing least squares
 *                     with a shared tridiagonal matrix               (temporal.py:194-239, thomas_solve 166-191)
 *   sr_interp_linear  temporal prolongation at the coarsest level    (temporal.py:109-127)
 *
 * Conventions (all follow grid.py:1-16):
 *  - images are flat, first axis fastest; dims[a] >= 2; cell centres at
 *    origin + (i + 0.5) * spacing;
 *  - a frame stack is [nframes][N] of `dtype`, N = prod(dims);
 *  - displacement fields y are [k][ndim][y_stride]: y_j,c(p) is at
 *    y[(j*ndim + c)*y_stride + (p - y_off)] (absolute positions, not offsets);
 *  - subset positions j = 0..k-1 follow the caller's subset order, frame_index[j]
 *    is the 0-based frame (the reference's 1-based k minus one, similarity.py:144);
 *  - affine parameters are rows of ndim*ndim + ndim doubles, row-major vec(A) ++ b
 *    (transform.py:58-68);
 *  - every pointer named *_dev is device memory on the context's device;
 *    everything else is host memory.  Calls are asynchronous on the context's
 *    stream unless stated otherwise.
 *
 * Every function returns SR_OK (0) or an error code; it never throws across
 * the ABI.  sr_last_error() gives the message of the last failing call.
 */
#ifndef SEQREG_B200_H
#define SEQREG_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define SR_API __attribute__((visibility("default")))
#else
#define SR_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define SR_ABI_VERSION 1

/* status codes */
#define SR_OK 0
#define SR_ERR_ARG 1         /* invalid argument (the Python shim raises ValueError) */
#define SR_ERR_CUDA 2        /* CUDA runtime error (RuntimeError) */
#define SR_ERR_SINGULAR 3    /* vanishing Thomas pivot (temporal.py:141-142 SingularSystemError) */
#define SR_ERR_UNSUPPORTED 4 /* e.g. more than SR_MAX_FRAMES subset frames */
#define SR_ERR_CALLBACK 5    /* a caller-supplied callback returned non-zero (its error is the caller's) */

#define SR_MAX_FRAMES 160    /* subset size limit: the kernels see <= 128 frames, larger subsets run as
                                blocks of 64 frames (two per launch); the K x K finalize of a subset must
                                fit in shared memory */

/* dtype */
#define SR_F32 0
#define SR_F64 1
/* feature function f ("e.g., NCC, NGF") */
#define SR_NCC 0             /* similarity.py:73-87 */
#define SR_NGF 1             /* normalised gradient field, defined in DESIGN.md §3 */
/* parametrisation of the transformations y_k */
#define SR_AFFINE 0          /* transform.py:35-96 */
#define SR_DISPLACEMENT 1    /* per-cell positions y_k(x) (north_star) */

typedef struct sr_ctx sr_ctx;

/* Cell-centred rectilinear grid (grid.py:61-99). Unused axes: dims 1. */
typedef struct sr_grid {
    int32_t ndim;        /* 2 or 3 */
    int32_t dims[3];
    double spacing[3];
    double origin[3];
} sr_grid;

/* One objective evaluation's inputs. */
typedef struct sr_problem {
    sr_grid grid;
    int32_t dtype;            /* SR_F32 / SR_F64: frames, y, gradient and kernel arithmetic */
    int32_t feature;          /* SR_NCC / SR_NGF */
    int32_t param;            /* SR_AFFINE / SR_DISPLACEMENT */
    double ngf_eps;           /* NGF edge parameter epsilon (> 0 when feature == SR_NGF) */
    int32_t k;                /* subset size, 1..SR_MAX_FRAMES */
    const int32_t* frame_index; /* host [k] 0-based frame of each subset position */
    const void* frames_dev;   /* [nframes][N] */
    int32_t nframes;
    const void* shifts_dev;   /* [nframes] per-frame intensity shift (sr_frame_shifts), or NULL */
    int64_t pix_lo, pix_hi;   /* flat pixel range owned by this call (a slab); whole grid: 0, N */
    const void* y_dev;        /* displacement: [k][ndim][y_stride] */
    int64_t y_off, y_stride;  /* flat pixel of element 0, and plane stride, of y_dev */
    const double* affine;     /* affine: host [k][ndim*ndim + ndim] */
} sr_problem;

/* Size in doubles of the raw-sums buffer: [G (k*k) | s (k) | vmax (k) | -vmin (k) | count].
 * When pixels are sharded, all-reduce the two extremum blocks with MAX and the rest with SUM. */
SR_API int64_t sr_raw_size(int32_t k);
/* Size in doubles of the stats buffer written by sr_corr_finalize (layout in DESIGN.md §4):
 *   [0] D, [1] k, [2] N, [3] cell_volume,
 *   [8 ..)           C        k*k   (exactly symmetric, zero rows for degenerate frames)
 *   next             sigma    k     (center_norms: NCC ||v - mean||, NGF ||n||)
 *   next             mean     k     (NCC mean of the warped values)
 *   next             vmax     k
 *   next             degen    k     (0/1)
 *   next             weights  k
 *   next             M        k*k   (gradient coefficients, row i col j)
 *   next             beta     k
 *   next             shift    k
 *   next             M as float  (k*k floats packed in doubles' storage) */
SR_API int64_t sr_stats_size(int32_t k);
SR_API int64_t sr_stats_offset(int32_t k, int32_t field); /* field: 0 C,1 sigma,2 mean,3 vmax,4 degen,5 weights,6 M,7 beta,8 shift,9 Mf */

SR_API int sr_abi_version(void);
SR_API const char* sr_last_error(void);
SR_API const char* sr_status_string(int status);

SR_API int sr_create(int32_t device, sr_ctx** out);
SR_API int sr_destroy(sr_ctx* ctx);
/* Use this cudaStream_t (NULL = legacy default stream) for every later call.  A context's calls are
 * ordered: on a change of stream the new stream first waits (device-side event) for the work already
 * queued on the previous one, because a context's scratch buffers are shared by all its calls.  Use one
 * context per concurrent stream for overlapping evaluations. */
SR_API int sr_set_stream(sr_ctx* ctx, void* stream);
/* Number of CTAs the persistent kernels launch (defaults to a multiple of the SM count). */
SR_API int sr_set_grid_ctas(sr_ctx* ctx, int32_t ctas);
/* Allow sr_grad to reuse the per-sample values and interpolant gradients that the preceding
 * sr_corr_partial on this context cached for the same problem (same y pointer, slab, frames and
 * subset), instead of re-gathering them.  Enable only when y is not modified between the two calls
 * (the reference's D + grad D pattern); sr_evaluate always reuses within its own call.
 * Default: off. */
SR_API int sr_set_sample_reuse(sr_ctx* ctx, int32_t enable);

/* Per-frame intensity shift (the frame mean, in fp64 then cast to dtype) used to
 * centre the raw Gram sums before they are formed. */
SR_API int sr_frame_shifts(sr_ctx* ctx, int32_t dtype, const void* frames_dev, int32_t nframes,
                    int64_t n, void* shifts_dev);

/* Pass 1 over [pix_lo, pix_hi): raw sums of the shifted features, reduced over
 * CTAs in a fixed order, written to raw_dev (sr_raw_size(k) doubles). */
SR_API int sr_corr_partial(sr_ctx* ctx, const sr_problem* prob, double* raw_dev);

/* Turn (possibly all-reduced) raw sums into C, sigma, degenerate flags, D and the
 * gradient coefficients.  n_total = pixel count of the whole grid. */
SR_API int sr_corr_finalize(sr_ctx* ctx, const sr_problem* prob, const double* raw_dev,
                     const double* weights /* host [k] */, double cell_volume,
                     int64_t n_total, double* stats_dev);

/* Pass 2 over [pix_lo, pix_hi).
 * Displacement: writes dD/dy to grad_dev laid out like y: [k][ndim][g_stride], element
 *   (j,c,p) at grad_dev[(j*ndim + c)*g_stride + (p - g_off)].
 * Affine: writes the slab's partial dD/d(params) rows, [k][ndim*ndim + ndim] doubles,
 *   to grad_dev (sum them over slabs; similarity.py:214-217). */
SR_API int sr_grad(sr_ctx* ctx, const sr_problem* prob, const double* stats_dev, void* grad_dev,
            int64_t g_off, int64_t g_stride);

/* One whole evaluation on one device (pass 1, finalize, pass 2): D lands in
 * stats_dev[0]; grad_dev may be NULL for a D-only evaluation (temporal.py:297-301). */
SR_API int sr_evaluate(sr_ctx* ctx, const sr_problem* prob, const double* weights, double cell_volume,
                double* raw_dev, double* stats_dev, void* grad_dev);

/* sr_evaluate plus the curvature regulariser S(y) (alpha > 0, displacement fields): the gradient gets
 * alpha h L L (y - x) added and S goes to s_out_dev[0].  The split fp32 NGF path adds the term inside its
 * pass-2 kernel (one launch, no read-modify-write of grad); every other path runs sr_curvature's kernel
 * after pass 2.  alpha = 0 is sr_evaluate.  (J = D + S, temporal.py:334-336 with S in place of the
 * affine drift penalty; north_star kernel 4.) */
SR_API int sr_evaluate_reg(sr_ctx* ctx, const sr_problem* prob, const double* weights, double cell_volume,
                    double alpha, double* raw_dev, double* stats_dev, void* grad_dev, double* s_out_dev);

/* Curvature regulariser on displacement fields:
 *   S = alpha/2 * h * sum_{j,c} || L (y_jc - x_c) ||^2,  grad += alpha * h * L L (y - x),
 * L the Neumann 2d+1-point Laplacian.  Adds into grad_dev (layout as sr_grad) over
 * [pix_lo, pix_hi) and writes this slab's S to s_out_dev[0] (one double). */
SR_API int sr_curvature(sr_ctx* ctx, const sr_problem* prob, double alpha, double cell_volume,
                 void* grad_dev, int64_t g_off, int64_t g_stride, double* s_out_dev);

/* The warped values T_j(y_j(x)) (affine rows or displacement fields, the sampling of grid.py:199-243)
 * of every subset frame over [pix_lo, pix_hi): out_dev[j * (pix_hi - pix_lo) + (p - pix_lo)], in the
 * problem's dtype.  Backs the lazily materialised CorrelationState.features (similarity.py:109-125);
 * not on the evaluation path. */
SR_API int sr_sample(sr_ctx* ctx, const sr_problem* prob, void* out_dev);

/* Temporal prolongation for fields of m components per frame (temporal.py:194-239):
 * solves (Mask + beta*Lap) zeta = Mask*eta + beta*Lap*ref for every component.
 * eta_dev, ref_dev, zeta_dev are [n][m] (frame-major); eta rows of inactive frames
 * are ignored.  mask: host [n] of 0/1.  Returns SR_ERR_SINGULAR like thomas_solve. */
SR_API int sr_ls_predict(sr_ctx* ctx, int32_t dtype, int32_t n, int64_t m, const uint8_t* mask,
                  double beta, const void* eta_dev, const void* ref_dev, void* zeta_dev);

/* Piecewise-linear interpolation in time (temporal.py:109-127): for each target frame
 * t, zeta[t] = (1-theta) * src[left] + theta * src[right], or a copy of src[t] when t
 * is a source.  src_dev/zeta_dev are [n][m]; left/right/theta are host [n]. */
SR_API int sr_interp_linear(sr_ctx* ctx, int32_t dtype, int32_t n, int64_t m, const int32_t* left,
                     const int32_t* right, const double* theta, const void* src_dev,
                     void* zeta_dev);

/* ------------------------------------------------------------------ spatial hierarchy
 * One pyramid step for every frame of a stack (pyramid.py:22-54; build_pyramid 68-91 applies it
 * level by level): dst = restrict(smooth(src)).  smooth = separable [1,2,1]/4 with reflective
 * boundaries (scipy.ndimage.convolve1d mode="reflect"), restrict = block means of 2^ndim cells with
 * a smaller trailing block on odd axes.  src_dev [nframes][prod(dims)], dst_dev
 * [nframes][prod(ceil(dims/2))]; the coarse grid has doubled spacing and the same origin.
 * fp64 results are bit-identical to the reference. */
SR_API int sr_pyramid_step(sr_ctx* ctx, int32_t dtype, int32_t ndim, const int32_t* dims, int32_t nframes,
                           const void* src_dev, void* dst_dev);

/* Spatial prolongation of displacement fields (absent in the reference): yc_dev
 * [k][ndim][N_coarse] absolute positions on `coarse` -> yf_dev [k][ndim][N_fine] on `fine`, by
 * multilinear interpolation of u = y - x at the fine cell centres, coordinates clamped to the hull
 * of the coarse centres (edge replication), y_fine = x_fine + u. */
SR_API int sr_prolong_field(sr_ctx* ctx, int32_t dtype, const sr_grid* coarse, const sr_grid* fine, int32_t k,
                            const void* yc_dev, void* yf_dev);

/* ------------------------------------------------------------------ device L-BFGS
 * lbfgs_minimize (optimizer.py:76-168) with every vector (x, g, the search direction,
 * the m curvature pairs) resident in device memory as fp64.  Same algorithm: two-loop
 * recursion (optimizer.py:59-73), Armijo backtracking only, curvature pairs with
 * s.y <= 1e-10 |s| |y| clear the history, the five stop reasons.  Element-wise updates
 * round like numpy (no FMA contraction); dot products use a fixed-order reduction
 * (deterministic; their summation order differs from BLAS, so results agree with the
 * reference to rounding, iteration counts and stop reasons match except on knife edges).
 *
 * The objective is a caller callback on device buffers:
 *   objective(user, x_dev, &f, g_dev) -> 0 on success; x_dev, g_dev are [n] fp64 on the
 *   context's device, valid for the duration of the call; the callback must have finished
 *   writing g_dev when it returns (the driver synchronises its stream before the call).
 * trace (optional) is called after every accepted step like optimizer.py:155-156. */
typedef int (*sr_objective_fn)(void* user, const double* x_dev, double* f_out, double* g_dev);
typedef void (*sr_trace_fn)(void* user, int32_t iteration, double f, double grad_inf, double step,
                            int32_t evaluations);

typedef struct sr_lbfgs_options { /* OptimOptions, optimizer.py:27-46 (same defaults) */
  int32_t memory;           /* 5 */
  int32_t max_iters;        /* 50 */
  double grad_tol;          /* 1e-4, on |g|_inf relative to the first iterate */
  double step_tol;          /* 1e-7 */
  double f_tol;             /* 1e-5, on the accepted decrease relative to 1 + |f| */
  double armijo_c1;         /* 1e-4 */
  double backtrack_factor;  /* 0.5 */
  int32_t max_backtracks;   /* 20 */
} sr_lbfgs_options;

#define SR_LBFGS_GRAD_TOL 0
#define SR_LBFGS_STEP_TOL 1
#define SR_LBFGS_F_TOL 2
#define SR_LBFGS_MAX_ITERS 3
#define SR_LBFGS_LINE_SEARCH_FAILURE 4

typedef struct sr_lbfgs_result { /* OptimResult, optimizer.py:49-56 (x_final is x_dev itself) */
  double f_final;
  double f_initial;
  int32_t iterations;
  int32_t objective_evaluations;
  int32_t converged_reason; /* SR_LBFGS_* */
} sr_lbfgs_result;

/* Fills `opts` with the reference defaults. */
SR_API void sr_lbfgs_defaults(sr_lbfgs_options* opts);

/* Minimise from x_dev (in: x0, out: the final iterate), n >= 1 parameters.  Returns
 * SR_ERR_ARG for invalid options (optimizer.py:38-46 messages) or a non-finite objective at
 * the start ("objective is not finite at the starting point"), SR_ERR_CALLBACK when the
 * objective returns non-zero.  Synchronous (returns after the last evaluation). */
SR_API int sr_lbfgs_minimize(sr_ctx* ctx, int64_t n, double* x_dev, const sr_lbfgs_options* opts,
                             sr_objective_fn objective, void* objective_user, sr_trace_fn trace,
                             void* trace_user, sr_lbfgs_result* result);

#ifdef __cplusplus
}
#endif
#endif /* SEQREG_B200_H */
