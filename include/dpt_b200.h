/*
 * dpt_b200.h -- C ABI of the B200-native DPT iteration path.
 *
 * This is the drop-in boundary for the hot path of the reference C++ library
 * `dynspec` (arXiv:2002.12872).  The reference exposes the path as C++ free
 * functions in proj/include/dynspec/dpt.hpp (namespace dynspec); each entry
 * point below replaces one of them, with plain pointers and sizes instead of
 * DenseMatrix / SparseMatrix / PartitionedProblem.  The C++ shim
 * (paper_2002_12872_b200/shim/dynspec_b200.cpp) maps the
 * reference's exact signatures onto these calls, so the reference's callers
 * (tools/main.cpp, src/rspt.cpp, src/analysis.cpp, the tests) link unchanged.
 *
 * Data model (real FP64, row-major -- the reference's DenseMatrix layout,
 * proj/include/dynspec/matrix.hpp:34-59):
 *   d        unperturbed levels theta_i (DiagonalMatrix::d, real parts)
 *   delta    the perturbation Delta (PartitionedProblem::delta, NOT delta_t):
 *            dense row-major n*n, or CSR (int64 row offsets, int32 sorted
 *            columns, FP64 values; SparseMatrix, matrix.hpp:73-106)
 *   A        the iterate, row i = chart row i (ConvergenceReport::state.a)
 * Arithmetic: the reference computes in std::complex<double>.  Real inputs run
 * the real FP64 kernels (4x fewer flops, identical results: the reference's
 * imaginary parts stay exactly 0); is_complex selects the complex FP64 path
 * (same kernels over interleaved re/im data).
 *
 * Errors follow the reference's exception taxonomy (dpt.hpp, partition.hpp:13-26):
 * non-convergence is a STATUS in the report, never an error code.
 * Every function is reentrant: state lives in the caller's dpt_ctx.
 */
#ifndef DPT_B200_H
#define DPT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DPT_B200_ABI_VERSION 2

/* ConvergenceStatus, dpt.hpp:13-18 (same order). */
typedef enum dpt_status {
  DPT_CONVERGED = 0,
  DPT_BOUNDED_NON_CONVERGED = 1,
  DPT_DIVERGED = 2,
  DPT_MAX_ITERATIONS = 3
} dpt_status;

/* Error codes; the shim maps them back to the reference's exceptions. */
typedef enum dpt_error {
  DPT_OK = 0,
  DPT_ERR_SHAPE = 1,        /* ShapeError (matrix.hpp:16-19) */
  DPT_ERR_DEGENERATE = 2,   /* DegenerateSpectrum(i, j, e_i, e_j) (partition.hpp:13-26) */
  DPT_ERR_INVALID_ARG = 3,  /* std::invalid_argument (dpt.cpp:376-382, :393-394) */
  DPT_ERR_CUDA = 4,
  DPT_ERR_NCCL = 5,
  DPT_ERR_NON_REAL = 6,     /* documented deviation: complex input */
  DPT_ERR_NO_DEVICE = 7,
  DPT_ERR_TRACE = 8,        /* the trace callback asked to abort */
  DPT_ERR_UNSUPPORTED = 9,
  DPT_ERR_IO = 10           /* IoError (matrix_market.hpp:10-13) */
} dpt_error;

/* Where the pointers of a call live. */
typedef enum dpt_mem { DPT_MEM_HOST = 0, DPT_MEM_DEVICE = 1 } dpt_mem;

/* DPT_DELTA_DENSE_T: dense, but `delta` holds Delta^T (the reference's cached
 * PartitionedProblem::delta_t, partition.hpp:43-50); accepted by the
 * single-step entry points (step_full), transposed on the device. */
typedef enum dpt_delta_kind { DPT_DELTA_DENSE = 0, DPT_DELTA_CSR = 1, DPT_DELTA_DENSE_T = 2 } dpt_delta_kind;

/* IterationOptions, dpt.hpp:22-31 -- field for field, same defaults
 * (dpt_options_default). */
typedef struct dpt_options {
  double tol;                  /* 1e-12 */
  double residual_tol;         /* 1e-10 */
  int max_iter;                /* 10000 */
  double divergence_threshold; /* 1e8 */
  int cycle_window;            /* 16 */
  double degeneracy_tol;       /* 1e-12 */
} dpt_options;

/* A PartitionedProblem (partition.hpp:43-50) in plain arrays. */
typedef struct dpt_problem {
  int64_t n;
  const double* d;       /* [n] */
  int delta_kind;        /* dpt_delta_kind */
  const double* delta;   /* dense: [n*n] row-major */
  const int64_t* rowptr; /* CSR: [n+1] */
  const int32_t* cols;   /* CSR: [nnz], sorted within rows */
  const double* vals;    /* CSR: [nnz] */
  int64_t nnz;
  double lambda;         /* Re PartitionedProblem::lambda */
  int mem;               /* dpt_mem of d / delta / rowptr / cols / vals */
  int is_complex;        /* 1: d, delta, vals are std::complex<double> arrays
                            (interleaved re, im), lambda_im used, and every
                            complex output (a, eigenvalues, z) is interleaved */
  double lambda_im;      /* Im PartitionedProblem::lambda */
} dpt_problem;

/* ConvergenceReport / SingleRowReport scalars (dpt.hpp:39-46, :98-105). */
typedef struct dpt_report {
  int status;        /* dpt_status */
  int iterations;
  double step_norm;
  double eigenvalue; /* single-row modes */
  double residual;   /* single-row modes */
  int64_t row;       /* dominant_eigenpair: chart index (DominantEigenpair::row) */
  /* timings of the call on the device (not part of the reference report) */
  double device_ms;
  int launches;
  double eigenvalue_im; /* single-row modes, complex problems */
} dpt_report;

/* DegenerateSpectrum payload + message for any error (partition.hpp:13-26). */
typedef struct dpt_error_info {
  int code;
  int64_t i, j;
  double ei, ej;       /* real parts of the offending levels */
  char message[256];
  double ei_im, ej_im; /* imaginary parts (complex problems) */
} dpt_error_info;

/* TraceSink, dpt.hpp:48-49: (k, step_norm, max_residual).  Called on the
 * calling thread, in k order, before the call returns.  Return nonzero to
 * abort the solve with DPT_ERR_TRACE (the reference propagates an exception
 * thrown by the sink). */
typedef int (*dpt_trace_fn)(int k, double step_norm, double max_residual, void* user);

typedef struct dpt_ctx dpt_ctx;

/* ---- context ------------------------------------------------------------- */
int dpt_ctx_create(int device, dpt_ctx** out, dpt_error_info* err);
void dpt_ctx_destroy(dpt_ctx* ctx);
/* Multi-GPU (column-of-the-paper / row-of-the-reference sharding across one
 * process per GPU): every rank calls with the same NCCL unique id bytes
 * (ncclGetUniqueId on rank 0, broadcast by the caller). world == 1 disables. */
int dpt_ctx_set_comm(dpt_ctx* ctx, int rank, int world, const void* nccl_id, size_t id_bytes,
                     dpt_error_info* err);
int dpt_nccl_unique_id(void* out, size_t bytes, dpt_error_info* err);
/* TEST-ONLY loopback communicator: makes ctxs[0..world-1] (distinct contexts
 * of ONE device, no NCCL communicator) ranks 0..world-1 of one sharded group.
 * Each rank must then be driven by its own host thread making the same
 * sequence of calls; the collectives (max-allreduce of the statistics, the
 * final all-gathers) are host rendezvous plus stream-event dependencies and
 * device copies -- no kernel waits on another rank's kernel.  Lets the
 * world > 1 path (shard_rows -> per-rank step -> allreduce -> decide ->
 * gather) run on a single GPU.  world <= 8. */
int dpt_ctx_set_loopback(dpt_ctx** ctxs, int world, dpt_error_info* err);
/* CUDA stream used by the context (cudaStream_t as void*). */
void* dpt_ctx_stream(dpt_ctx* ctx);
/* Kernel launches issued by this context so far (for gpu_launches accounting). */
int64_t dpt_ctx_launch_count(const dpt_ctx* ctx);
/* Device-loop graph cache of this context: replays of a cached graph (hits)
 * and captures (misses) so far (tests of the cache key). */
void dpt_ctx_graph_stats(const dpt_ctx* ctx, int64_t* hits, int64_t* misses);

void dpt_options_default(dpt_options* o);
const char* dpt_status_string(int status); /* to_string, dpt.cpp:297-309 */
int dpt_abi_version(void);

/* ---- full map (the row form of dpt.hpp:51-57) ----------------------------- */

/* iterate_full (dpt.hpp:74-83).  Outputs (all may be host or device pointers
 * per out_mem; any may be NULL to skip):
 *   a_out   [n*n] final iterate (ConvergenceReport::state.a)
 *   eig_out [n]   eigenvalues (NaN when Diverged)
 *   res_out [n]   per-row residuals (NaN when Diverged)          */
int dpt_iterate_full(dpt_ctx* ctx, const dpt_problem* p, const dpt_options* opts,
                     dpt_trace_fn trace, void* user, double* a_out, double* eig_out,
                     double* res_out, int out_mem, dpt_report* rep, dpt_error_info* err);

/* iterate_ramped (dpt.hpp:85-92): lambda_k = lambda (1 - alpha^(k-1)). */
int dpt_iterate_ramped(dpt_ctx* ctx, const dpt_problem* p, double alpha, const dpt_options* opts,
                       dpt_trace_fn trace, void* user, double* a_out, double* eig_out,
                       double* res_out, int out_mem, dpt_report* rep, dpt_error_info* err);

/* iterate_fixed (dpt.hpp:94-96): exactly k applications from I at `lambda`. */
int dpt_iterate_fixed(dpt_ctx* ctx, const dpt_problem* p, int k, double lambda, double* a_out,
                      int out_mem, dpt_report* rep, dpt_error_info* err);

/* step_full (dpt.hpp:51-57): one application of the map to `a` [n*n].
 * The reference passes GapMatrix + delta_t; here theta comes from p->d and
 * Delta from p (the shim recovers them), `lambda` is the step's coupling. */
int dpt_step_full(dpt_ctx* ctx, const dpt_problem* p, const double* a, double lambda,
                  double* out, int io_mem, dpt_error_info* err);

/* step_full with the caller's GapMatrix theta (n*n row-major, zero diagonal):
 * the reference's exact signature (dpt.hpp:56-57) passes theta, not levels;
 * p->d is then ignored by the map. */
int dpt_step_full_gap(dpt_ctx* ctx, const dpt_problem* p, const double* a, const double* gap,
                      double lambda, double* out, int io_mem, dpt_error_info* err);

/* Read-offs of a caller iterate: eig_i = d_i + lambda P(i,i), residual rows
 * (residuals_of, dpt.cpp:23-44) with P = a Delta^T.  [n] outputs. */
int dpt_readoffs(dpt_ctx* ctx, const dpt_problem* p, const double* a, double* eig_out, double* res_out,
                 int io_mem, dpt_error_info* err);

/* ---- row map -------------------------------------------------------------- */

/* iterate_single (dpt.hpp:107-111). z_out [n]. */
int dpt_iterate_single(dpt_ctx* ctx, const dpt_problem* p, int64_t row, const dpt_options* opts,
                       double ramp_alpha, dpt_trace_fn trace, void* user, double* z_out,
                       int out_mem, dpt_report* rep, dpt_error_info* err);

/* dominant_eigenpair (dpt.hpp:113-129). z_chart / z_unit [n]; rep->row. */
int dpt_dominant_eigenpair(dpt_ctx* ctx, const dpt_problem* p, const dpt_options* opts,
                           double* z_chart, double* z_unit, int out_mem, dpt_report* rep,
                           dpt_error_info* err);

/* step_single (dpt.hpp:59-66): one row-map application to z [n] for chart `row`. */
int dpt_step_single(dpt_ctx* ctx, const dpt_problem* p, const double* z, int64_t row,
                    double lambda, double* out, int io_mem, dpt_error_info* err);

/* step_single with the caller's GapRow (dpt.hpp:62-63): gap_row [n], zero at `row`. */
int dpt_step_single_gap(dpt_ctx* ctx, const dpt_problem* p, const double* z, int64_t row,
                        const double* gap_row, double lambda, double* out, int io_mem,
                        dpt_error_info* err);

/* eigenvalue_of (dpt.hpp:68-72): d_row + lambda (Delta z)_row. */
int dpt_eigenvalue_of(dpt_ctx* ctx, const dpt_problem* p, const double* z, int64_t row,
                      double lambda, double* out, int z_mem, dpt_error_info* err);

/* ---- complex coupling variants (the reference's cdouble lambda arguments) ---
 * Same as the real entry points with lambda = lambda + i lambda_im; for a
 * complex problem every array is interleaved std::complex<double>
 * (a, gap, z: n*n or n complex values; out2 of eigenvalue_of_c: 2 doubles). */
int dpt_iterate_fixed_c(dpt_ctx* ctx, const dpt_problem* p, int k, double lambda, double lambda_im,
                        double* a_out, int out_mem, dpt_report* rep, dpt_error_info* err);
int dpt_step_full_gap_c(dpt_ctx* ctx, const dpt_problem* p, const double* a, const double* gap,
                        double lambda, double lambda_im, double* out, int io_mem, dpt_error_info* err);
int dpt_step_single_gap_c(dpt_ctx* ctx, const dpt_problem* p, const double* z, int64_t row,
                          const double* gap_row, double lambda, double lambda_im, double* out, int io_mem,
                          dpt_error_info* err);
int dpt_eigenvalue_of_c(dpt_ctx* ctx, const dpt_problem* p, const double* z, int64_t row, double lambda,
                        double lambda_im, double* out2, int z_mem, dpt_error_info* err);

/* ---- plans: a problem kept resident in HBM ------------------------------------ */
/* For repeated calls on one perturbation (the reference's scan_domain / bench
 * loops call the solver many times on the same Delta) and for device-resident
 * throughput measurement.  single != 0 selects the row map for chart `row`. */
typedef struct dpt_plan dpt_plan;
int dpt_plan_create(dpt_ctx* ctx, const dpt_problem* p, int single, int64_t row, double lambda,
                    dpt_plan** out, dpt_error_info* err);
void dpt_plan_destroy(dpt_plan* plan);
/* restart from A_0 = I (z_0 = e_row) and apply the first step */
int dpt_plan_begin(dpt_plan* plan, dpt_error_info* err);
/* k more applications of the map (iterate_fixed semantics); kernel_ms (may be
 * NULL) receives the summed device time of the step kernels alone */
int dpt_plan_steps(dpt_plan* plan, int k, double* kernel_ms, dpt_error_info* err);
int dpt_plan_read(dpt_plan* plan, double* out, int out_mem, dpt_error_info* err);
/* stats of the latest step: {max|A_j - A_j-1|, max|A_j|, #nonfinite, max residual of A_j-1} */
int dpt_plan_stats(dpt_plan* plan, double* out4, dpt_error_info* err);

/* Measured FP64 tensor-core (DMMA) throughput of `device` in TFLOP/s: the
 * roofline denominator for the dense step (MEASURED_PEAKS.json has no FP64). */
int dpt_probe_fp64_peak(int device, double* tflops, dpt_error_info* err);

/* ---- host-only helpers (no GPU needed; used by CPU tests) ------------------ */

/* build_theta's degeneracy policy (partition.cpp:42-81) in O(n log n):
 * returns 1 and the reference's first (i, j) in row-major order if two levels
 * are within degeneracy_tol * max(1, spread), else 0. */
int dpt_check_degenerate(int64_t n, const double* d, double degeneracy_tol, int64_t* i,
                         int64_t* j);
double dpt_spectral_spread(int64_t n, const double* d);
int dpt_effective_window(int requested, int64_t n); /* dpt.cpp:83-90 */

/* ---- staged continuation ---------------------------
 * homotopy_solve, dpt.hpp:145-152 / dpt.cpp:505-556: `stages` solves along
 * lambda_s = lambda s / stages, each on the problem rebased by the product W of
 * the converged bases (R = W^-1 (lambda_s Delta + diag d) W, re-split with
 * lambda 1), all on the device (the basis algebra on the library-free DMMA
 * GEMM and cluster LU of linalg.cu, the stage solves on the solver's kernels).  Outputs as
 * dpt_iterate_full: a = the normalised eigenvector matrix, read-offs against
 * the original problem, rep.iterations = the sum over stages, rep.status = the
 * last stage's.  Errors: stages < 1 -> DPT_ERR_INVALID_ARG; a singular basis
 * -> DPT_ERR_UNSUPPORTED (the reference's std::runtime_error). */
/* matmul(DenseMatrix, DenseMatrix), matrix.cpp:130-143: c (m x n) = a (m x k)
 * b (k x n), row-major, complex interleaved when is_complex (the DMMA GEMM). */
int dpt_matmul_dense(dpt_ctx* ctx, int64_t m, int64_t k, int64_t n, int is_complex, const double* a, const double* b,
                     double* c, int mem, dpt_error_info* err);
/* solve_linear_multi(a, b), matrix.cpp:519-533: x (n x nrhs) = a^-1 b by LU
 * with partial pivoting (first row of maximal |a(i,k)|), on the device.  An
 * exactly-zero pivot -> DPT_ERR_UNSUPPORTED ("solve_linear: singular matrix",
 * the reference's std::runtime_error). */
int dpt_solve_linear_multi(dpt_ctx* ctx, int64_t n, int64_t nrhs, int is_complex, const double* a, const double* b,
                           double* x, int mem, dpt_error_info* err);
int dpt_homotopy_solve(dpt_ctx* ctx, const dpt_problem* p, int stages, const dpt_options* opts, double* a_out,
                       double* eig_out, double* res_out, int out_mem, dpt_report* rep, dpt_error_info* err);

/* ---- Matrix Market I/O ------------------------------
 * read_matrix_market / write_matrix_market, proj/include/dynspec/matrix_market.hpp
 * (proj/src/matrix_market.cpp:70-191): coordinate and array formats, real and
 * complex fields, general and symmetric symmetry (expanded).  Coordinate data
 * becomes CSR through from_triplets' steps (sorted by (row, col), duplicates
 * summed); array data a row-major dense matrix.  Values interleave (re, im) when
 * is_complex.  Results are bit-identical to the reference's; parsing and
 * formatting use `threads` host threads (0 = all).  Errors: DPT_ERR_IO with the
 * reference's IoError message. */
typedef struct dpt_mm_matrix {
  int64_t rows, cols;
  int is_sparse;    /* 1: CSR (coordinate file), 0: dense row-major (array file) */
  int is_complex;   /* field complex */
  int64_t nnz;      /* stored entries (dense: rows * cols) */
  int64_t* rowptr;  /* [rows + 1] (sparse) */
  int64_t* colidx;  /* [nnz] (sparse) */
  double* vals;     /* sparse: [nnz] scalars; dense: [rows * cols] scalars */
  void* store;      /* owner of the arrays (dpt_mm_free) */
} dpt_mm_matrix;
int dpt_mm_read(const char* path, int threads, dpt_mm_matrix* out, dpt_error_info* err);
void dpt_mm_free(dpt_mm_matrix* m);
int dpt_mm_write_dense(const char* path, int64_t rows, int64_t cols, const double* vals, int is_complex, int threads,
                       dpt_error_info* err);
int dpt_mm_write_csr(const char* path, int64_t rows, int64_t cols, const int64_t* rowptr, const int64_t* colidx,
                     const double* vals, int is_complex, int threads, dpt_error_info* err);

/* ---- batched lambda-plane scan -------------------
 * scan_domain, proj/src/analysis.cpp:68-138 (declared in
 * proj/include/dynspec/analysis.hpp:63-69): classify every cell of the grid by
 * solving the base problem at lambda = (re_at(j), im_at(i)).  The base
 * problem's lambda is ignored.  classes[i * res_re + j] receives CellClass
 * (0 Converged, 1 BoundedNonConverged -- including MaxIterations -- 2 Diverged),
 * iterations[] the report's iteration count.  n <= 32 (full) / 2048 (row)
 * run batched on the device, one warp per cell, in the reference's operation
 * order; larger problems are solved cell by cell. */
typedef struct dpt_scan_grid {
  double re_min, re_max, im_min, im_max;
  int64_t res_re, res_im;
} dpt_scan_grid;
enum { DPT_SCAN_FULL = 0, DPT_SCAN_SINGLE_ROW = 1 };
int dpt_scan_domain(dpt_ctx* ctx, const dpt_problem* base, const dpt_scan_grid* grid, int mode, int64_t row,
                    double ramp_alpha, const dpt_options* opts, uint8_t* classes, int32_t* iterations,
                    dpt_error_info* err);

/* The per-iteration decision function the device runs (dpt_state.h), exposed
 * for host-side tests: feeds one launch's statistics into the state machine.
 * state / opts are opaque byte blobs of dpt_sm_state_bytes() / dpt_sm_options_bytes(). */
size_t dpt_sm_state_bytes(void);
void dpt_sm_init(void* state, void* opts, const dpt_options* o, int win, int have_trace);
void dpt_sm_decide_host(void* state, const void* opts, const double* stats, int j,
                        int settled_prev, int settled_cur, double* trace_out);
void dpt_sm_query(const void* state, int* done, int* status, int* iterations, int* final_iter,
                  int* readoffs, int* cycle_pending, double* step_norm);

#ifdef __cplusplus
}
#endif
#endif /* DPT_B200_H */
