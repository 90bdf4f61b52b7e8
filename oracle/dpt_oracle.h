/* dpt_oracle.h -- TEST INFRASTRUCTURE ONLY (see dpt_oracle.c header). */
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_DENSE = 0, ORC_CSR = 1 };
/* ConvergenceStatus order, proj/include/dynspec/dpt.hpp:13-18 */
enum { ORC_CONVERGED = 0, ORC_BOUNDED = 1, ORC_DIVERGED = 2, ORC_MAXITER = 3 };
enum { ORC_OK = 0, ORC_ERR_SHAPE = 1, ORC_ERR_DEGENERATE = 2, ORC_ERR_INVALID = 3 };

typedef struct {
  int64_t n;
  const double* d; /* unperturbed levels theta_i (real parts of DiagonalMatrix::d) */
  int kind;        /* ORC_DENSE | ORC_CSR */
  const double* delta; /* dense: row-major n*n (PartitionedProblem::delta) */
  const int64_t* rowptr; /* CSR of delta, sorted columns */
  const int32_t* cols;
  const double* vals;
  double lambda;
} orc_problem;

/* IterationOptions, proj/include/dynspec/dpt.hpp:22-31 */
typedef struct {
  double tol;
  double residual_tol;
  int max_iter;
  double divergence_threshold;
  int cycle_window;
  double degeneracy_tol;
} orc_options;

typedef struct {
  int status, iterations;
  double step_norm;
  int64_t degenerate_i, degenerate_j;
} orc_report;

typedef struct {
  int status, iterations;
  double step_norm, eigenvalue, residual;
  int64_t degenerate_i, degenerate_j;
} orc_single_report;

double orc_spectral_spread(int64_t n, const double* d);
int orc_check_degenerate(int64_t n, const double* d, double tol, int64_t* bi, int64_t* bj);
int orc_effective_window(int requested, int64_t n);
int orc_iterate_full(const orc_problem* p, const orc_options* o, int ramped, double alpha,
                     double* a_out, double* eig_out, double* res_out, orc_report* rep,
                     double* trace_step, double* trace_res);
int orc_step_full(const orc_problem* p, const double* a, double lam, double* out);
int orc_iterate_fixed(const orc_problem* p, int k, double lam, double* a_out);
int orc_step_rows(const orc_problem* p, int64_t row0, int64_t rows, const double* a, double lam,
                  double* out);
int orc_iterate_single(const orc_problem* p, int64_t row, const orc_options* o, double ramp_alpha,
                       double* z_out, orc_single_report* rep, double* trace_step,
                       double* trace_res);
int orc_dominant_eigenpair(const orc_problem* p, const orc_options* o, double* z_chart,
                           double* z_unit, orc_single_report* rep, int64_t* row_out);
int orc_step_single(const orc_problem* p, const double* z, int64_t row, double lam, double* out);
int orc_eigenvalue_of(const orc_problem* p, const double* z, int64_t row, double lam, double* out);

#ifdef __cplusplus
}
#endif
