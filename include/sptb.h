/*
 * sptb.h -- C ABI of the B200-native sparse-matrix tomography operators.
 *
 * Drop-in boundary for the hot path of the reference package `sptomo`
 * (/root/reference/pkg/src/sptomo).  Every entry point names the reference
 * interface it replaces (file:line).  Plain C types only: opaque plan handle,
 * raw pointers (device OR host -- detected per call), sizes, status codes.
 *
 * Numerics: complex64 production (SPTB_PREC_F32) or complex128 validation
 * (SPTB_PREC_F64) for every stage (gridding SpMM, cuFFT, elementwise).
 * Index conventions follow the reference after an internal remap: the
 * reference's Fortran-order grid index gx*n_y+gy (gridding.py:10-11) becomes
 * row-major y*n_x+x on device; sinograms keep the (theta, p) row-major order.
 */
#ifndef SPTB_H
#define SPTB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (mapped to sptomo.errors by the host shim) ------------ */
#define SPTB_OK              0
#define SPTB_ERR_SHAPE       1  /* ShapeMismatchError       errors.py:8   */
#define SPTB_ERR_ARG         2  /* ValueError                              */
#define SPTB_ERR_NEAR_ZERO   3  /* NearZeroDenominatorError errors.py:12  */
#define SPTB_ERR_CUDA        4  /* RuntimeError (CUDA runtime)             */
#define SPTB_ERR_CUFFT       5  /* RuntimeError (cuFFT)                    */
#define SPTB_ERR_OOM         6  /* MemoryError                             */
#define SPTB_ERR_NONFINITE   7  /* NonFiniteError           errors.py:36  */
#define SPTB_ERR_DIVERGENCE  8  /* DivergenceError          errors.py:32  */
#define SPTB_ERR_STATE       9  /* RuntimeError (misuse of the plan)      */

#define SPTB_PREC_F32 0
#define SPTB_PREC_F64 1

/* data formats of caller arrays: element type | layout kind */
#define SPTB_FMT_F32      0x0   /* float32 elements                       */
#define SPTB_FMT_F64      0x1   /* float64 elements                       */
#define SPTB_FMT_REAL     0x0   /* n real slices; slices (2k,2k+1) share one
                                   complex vector (pipeline.py:122-134)    */
#define SPTB_FMT_COMPLEX  0x2   /* n interleaved complex arrays (re, im)   */

/* matrices held by a plan */
#define SPTB_MAT_S   0  /* S   (n_grid x n_samples), spread  (gridding.py:63-70) */
#define SPTB_MAT_SH  1  /* S^H (n_samples x n_grid), interp  (gridding.py:72-81) */
#define SPTB_MAT_SW  2  /* S diag(w), filter folded  (operators.py:352-353)      */

#define SPTB_KERNEL_KB    0
#define SPTB_KERNEL_GAUSS 1

/* ScanGeometry (geometry.py:32-111).  cos/sin of the angles are passed in by
 * the caller so polar sample positions are bit-identical to the reference's
 * numpy evaluation (geometry.py:202-215). */
typedef struct sptb_geometry {
    int32_t n_p;
    int32_t n_theta;
    int32_t n_x;
    int32_t n_y;
    double center;
    const double* cos_theta;   /* host, n_theta */
    const double* sin_theta;   /* host, n_theta */
} sptb_geometry;

/* KernelSpec (geometry.py:115-139) */
typedef struct sptb_kernel {
    int32_t family;            /* SPTB_KERNEL_KB | SPTB_KERNEL_GAUSS */
    int32_t width;             /* odd */
    double beta;
    double sigma;
} sptb_kernel;

typedef struct sptb_plan sptb_plan;

/* Thread-local message for the last non-OK status. */
const char* sptb_last_error(void);
int32_t sptb_version(void);

/* Build the gridding matrices on the device and the deapodization grid.
 * Replaces build_matrix + deapodization_compute inside build_operators
 * (operators.py:317-339, gridding.py:84-195, geometry.py:254-272).
 * max_batch = largest number of complex vectors processed per launch.   */
int sptb_plan_create(sptb_plan** out, const sptb_geometry* geom,
                     const sptb_kernel* kernel, int32_t precision,
                     int32_t max_batch, int32_t device, double threshold);
int sptb_plan_destroy(sptb_plan* plan);

/* Re-read the SPTB_* path-selection environment switches (tests and A/B
 * measurements only; no reference counterpart).  The library reads them once
 * at first use; production never sets them. */
int sptb_reload_switches(void);

/* CUDA stream (cudaStream_t as void*) for all subsequent work; NULL = legacy. */
int sptb_plan_set_stream(sptb_plan* plan, void* stream);

/* Radial (n_p) or per-sample (n_theta*n_p) filter weights, folded into a
 * copy of S's values (operators.py:345-353, sample_weights :74-82).  kind is
 * informational (0 none).  Also records the weights for apply_weights.    */
int sptb_plan_set_filter(sptb_plan* plan, const double* weights, int64_t n_weights);

/* calib = 1 / mean_disk(iradon_w(radon(disk)))  (operators.py:302-314). */
int sptb_plan_calibrate(sptb_plan* plan, double* calib_out);
int sptb_plan_set_calibration(sptb_plan* plan, double calib);

/* density_filter_solve (operators.py:189-236): CGLS on || |S| d - 1 ||_2 over
 * per-sample weights d (max_iter iterations, relative tolerance tol), clamped
 * >= 0 and symmetrised in p.  weights_out: n_theta * n_p doubles (sample
 * order); residual_history: max_iter + 1 doubles, *n_history filled. */
int sptb_density_filter(sptb_plan* plan, int32_t max_iter, double tol, double* weights_out,
                        double* residual_history, int32_t* n_history, int32_t* converged,
                        double* final_residual);

/* Matrix introspection: nnz and (optionally) a host copy of the CSR in the
 * device index convention.  Any pointer may be NULL.                      */
int sptb_plan_matrix_info(sptb_plan* plan, int32_t which, int64_t* rows,
                          int64_t* cols, int64_t* nnz);
int sptb_plan_matrix_copy(sptb_plan* plan, int32_t which, int32_t* row_ptr,
                          int32_t* col_idx, double* vals_ri);
/* Deapodization grid (n_y x n_x, float64 host) -- Deapodization.values. */
int sptb_plan_deapo_copy(sptb_plan* plan, double* out);

/* ---- operators (operators.py:124-187, 252-299) ------------------------- */
/* in/out may be device or host pointers; n = slices (REAL) or complex arrays
 * (COMPLEX).  Output format's kind must equal the input's (.real semantics,
 * operators.py:166-167,185-186); element types may differ.               */

/* radon(tomo)  (operators.py:153-168):  (n, n_y, n_x) -> (n, n_theta, n_p) */
int sptb_radon(sptb_plan* plan, const void* in, int32_t in_fmt,
               void* out, int32_t out_fmt, int64_t n);
/* radon_adjoint(sino) = iradon(sino, S) unfiltered, scale 1 (:255-257)    */
int sptb_radon_adjoint(sptb_plan* plan, const void* in, int32_t in_fmt,
                       void* out, int32_t out_fmt, int64_t n);
/* iradon(sino) through the folded filter and calibration (:259-267)       */
int sptb_iradon(sptb_plan* plan, const void* in, int32_t in_fmt,
                void* out, int32_t out_fmt, int64_t n);
/* apply_weights(sino) = ifft(fft(sino) * w)  (:293-299, :99-105)           */
int sptb_apply_weights(sptb_plan* plan, const void* in, int32_t in_fmt,
                       void* out, int32_t out_fmt, int64_t n);

/* iradon(sino, csr|csr_filtered, deapo, geom, scale=scale) -- the free
 * function form (operators.py:171-187): filtered != 0 selects the folded
 * matrix S diag(w).                                                        */
int sptb_backproject(sptb_plan* plan, int32_t filtered, double scale,
                     const void* in, int32_t in_fmt, void* out, int32_t out_fmt,
                     int64_t n);
/* _spectral_apply(sino, weights) (operators.py:99-105) with caller weights
 * (n_p or n_theta*n_p, host float64); precondition_apply passes sqrt(w).   */
int sptb_spectral_apply(sptb_plan* plan, const double* weights, int64_t n_weights,
                        const void* in, int32_t in_fmt, void* out, int32_t out_fmt,
                        int64_t n);

/* spmm(csr, x, adjoint) (operators.py:124-136) in the REFERENCE index
 * convention: x is (cols, nrhs) and y is (rows, nrhs), complex, row-major
 * (nrhs innermost), F-order grid index.  which = SPTB_MAT_S | SPTB_MAT_SH. */
int sptb_spmm(sptb_plan* plan, int32_t which, const void* x, void* y,
              int64_t nrhs, int32_t fmt);

/* ---- solvers (solvers.py:31-64, 122-473) -------------------------------- */
#define SPTB_ALGO_FBP  0
#define SPTB_ALGO_SIRT 1
#define SPTB_ALGO_CGLS 2
#define SPTB_ALGO_TV   3

typedef struct sptb_solver_config {   /* SolverConfig (solvers.py:31-56) */
    int32_t algorithm;
    int32_t max_iter;
    double tol;
    double mu;                /* <= 0: default 0.1 max|A^H b| per channel */
    int32_t tv_inner_iter;
    int32_t bb_enabled;
    int32_t nonneg;
    int32_t cgs_mode;
} sptb_solver_config;

/* Solve every unit (complex pair, or one real slice for an odd tail) of
 * `sino` (n slices / complex arrays, fmt as for operators) into `rec`.
 * Per unit u: hist[u*max_iter + k] = residual after iteration k,
 * iters[u], converged[u], status[u] (SPTB_OK / _DIVERGENCE / _NONFINITE).
 * Returns the first failing unit's status (or OK).  report pointers are host. */
int sptb_solve(sptb_plan* plan, const sptb_solver_config* cfg,
               const void* sino, int32_t in_fmt, void* rec, int32_t out_fmt,
               int64_t n, double* hist, int32_t* iters, int32_t* converged,
               int32_t* status);

/* Timing hook for benchmarks: number of kernels this library launched
 * (hand-written kernels only; cuFFT executions are counted separately). */
int64_t sptb_launch_count(void);
int64_t sptb_fft_count(void);

/* Benchmark hook: time `reps` back-to-back launches of the gridding SpMM
 * (`which` = SPTB_MAT_S / _SH / _SW) over B complex columns in the layouts the
 * operators use, with CUDA events on the plan's stream.  Returns the mean
 * milliseconds per launch and the matrix's distinct referenced input rows
 * (U_in of the algorithmic-bytes model).          */
int sptb_time_spmm(sptb_plan* plan, int32_t which, int32_t B, int32_t reps,
                   double* ms_per_launch, int64_t* distinct_inputs);

#ifdef __cplusplus
}
#endif
#endif /* SPTB_H */
