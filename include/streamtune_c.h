/*
 * streamtune_c.h -- C ABI over the streamtune C++ API (include/streamtune/).
 *
 * The reference's own interface for the stream-count side is the header-only
 * C++ namespace `streamtune` (/root/reference/proj/include/streamtune/
 * timing_model.hpp:35-146, errors.hpp:7-118) plus the predictor / regression
 * / dataset modules its spec defines.
 * C++ callers include the headers under include/streamtune/ directly; these
 * extern "C" entry points expose the same functions to C, ctypes (the test
 * suite) and other FFIs.  Every function returns ST_OK, ST_VALIDATION (a
 * streamtune::ValidationError was thrown) or ST_COMPUTATION (a
 * streamtune::ComputationError); `err` (may be NULL) receives
 * "<ExceptionClass>: <message>".
 */
#ifndef STREAMTUNE_C_H
#define STREAMTUNE_C_H

#include <stdint.h>

#include "pm_tridiag.h"

#ifdef __cplusplus
extern "C" {
#endif

#define ST_OK 0
#define ST_VALIDATION 1
#define ST_COMPUTATION 2

/* timing_model.hpp */
int st_stream_count_is_valid(int n);
int st_validate_stage_timings(const pm_stage_timings* t, char* err, int errlen);
double st_total_unstreamed(const pm_stage_timings* t);
double st_overlap_sum(const pm_stage_timings* t);
int st_streamed_lower_bound(const pm_stage_timings* t, int n, double overhead_ms, double* out,
                            char* err, int errlen);
int st_overhead_from_measurement(double t_str, double t_non_str, int n, double sum, double* out,
                                 char* err, int errlen);
int st_overlap_benefit(int n, double sum, double overhead_ms, double* out, char* err, int errlen);

/* predictor */
int st_predict_sum(const pm_model_bundle* b, uint64_t n, double* out, char* err, int errlen);
int st_predict_overhead(const pm_model_bundle* b, uint64_t n, int streams, double* out, char* err,
                        int errlen);
/* benefits[i], overheads[i] for the bundle's candidates; model_used 0 small / 1 big */
int st_recommend(const pm_model_bundle* b, uint64_t n, int* chosen, double* benefits,
                 double* overheads, double* predicted_sum, int* model_used, char* err, int errlen);
int st_recommend_fp32(const pm_model_bundle* b, uint64_t n, int* chosen, char* err, int errlen);
int st_gomez_luna_optimum(double sum, double tau, double* out, char* err, int errlen);

/* regression */
int st_train_test_split(int n, double train_fraction, int shuffle, uint64_t seed, int* order,
                        int* n_train, char* err, int errlen);
int st_fit_least_squares(const double* X, const double* y, int rows, int cols, double* beta,
                         char* err, int errlen);
int st_metrics(const double* predicted, const double* actual, int n, double* r2_mse_rmse,
               char* err, int errlen);
/* kind: 0 sum model (features [N, 1]), 1 overhead small, 2 overhead big.
 * coef[3] (2 used for kind 0), metrics[6] = train {r2, mse, rmse}, test {...} */
int st_fit_model(int kind, const uint64_t* sizes, const int* streams, const double* target,
                 int rows, double train_fraction, int shuffle, uint64_t seed, double* coef,
                 double* metrics, int* n_train, char* err, int errlen);

/* dataset + cmd_fit */
int st_load_stage_timings(const char* csv, pm_stage_timings* rows, int max_rows, int* n_rows,
                          char* err, int errlen);
int st_load_streamed_runs(const char* csv, uint64_t* sizes, int* streams, double* t_str,
                          int max_rows, int* n_rows, char* err, int errlen);
int st_derive_overhead_rows(const char* stage_csv, const char* runs_csv, uint64_t* sizes,
                            int* streams, double* overhead, int max_rows, int* n_rows, char* err,
                            int errlen);
/* Fits Eq. 4 and both Eq. 7 forms from the two CSV documents.
 * metrics[18] = sum/small/big x train/test x {r2, mse, rmse}. */
int st_fit_bundle(const char* stage_csv, const char* runs_csv, uint64_t size_threshold,
                  uint64_t seed, pm_model_bundle* out, double* metrics, char* err, int errlen);
/* The same with the anchored overhead fits (T_overhead(N, 1) = 0, coefficients
 * >= 0; streamtune::fit_overhead_*_anchored) -- the B200 re-fit. */
int st_fit_bundle_anchored(const char* stage_csv, const char* runs_csv, uint64_t size_threshold,
                           uint64_t seed, pm_model_bundle* out, double* metrics, char* err, int errlen);

/* simulator.  stages[7] = {stage1 h2d, comp, d2h, cpu (Stage 2),
 * stage3 h2d, comp, d2h} in ms; n a valid stream count; out[3] = {total, stage-1
 * makespan, stage-3 makespan}; trace (may be NULL) receives up to max_events rows of
 * 5 doubles {engine (0 h2d, 1 comp, 2 d2h), stream, stage (1|3), start_ms, end_ms}. */
int st_simulate(const double* stages, int n, double tau_ms, int hw_queues, double* out,
                double* trace, int max_events, int* n_events, char* err, int errlen);
/* holds = simulate.total >= Eq. 2 bound - 1e-9; dominance = Eq. 2 is exact */
int st_verify_lower_bound(const double* stages, int n, double tau_ms, int* holds, int* dominance,
                          char* err, int errlen);

/* ModelBundle document: JSON, 17 significant digits.  *needed = bytes
 * including the terminating NUL; a too-small buffer is a validation error. */
int st_bundle_to_json(const pm_model_bundle* b, char* out, int outlen, int* needed, char* err,
                      int errlen);
int st_bundle_from_json(const char* doc, pm_model_bundle* out, char* err, int errlen);

/* cmd_report: table in {table1, table2, table4, table5};
 * cells: up to max_cells rows of {expected, got, tolerance, status (0 pass, 1 fail,
 * 2 known deviation)} */
int st_report_table(const pm_model_bundle* b, const char* table, int* passed, int* failed,
                    int* known, double* cells, int max_cells, int* n_cells, char* err, int errlen);
/* cmd dump-reference: CSV of an embedded paper table (table1|table2|table4|table5|tau) */
int st_dump_reference(const char* table, char* out, int outlen, int* needed, char* err,
                      int errlen);

#ifdef __cplusplus
}
#endif

#endif /* STREAMTUNE_C_H */
