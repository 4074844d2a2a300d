/*
 * uot_oracle.h — CPU restatement of the MAP-UOT fused Sinkhorn-UOT path.
 *
 * TEST INFRASTRUCTURE ONLY. This is the parity checker for the sm_100a path
 * (paper_2412_11079_b200/csrc). Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it. The product
 * never links or calls it.
 *
 * Every function restates the reference algorithm (paths relative to
 * /root/reference/proj/core) in plain C; file:line citations are on each
 * declaration. Parity of this restatement is pinned two ways:
 *   - against the reference itself compiled here (oracle/_ref, see Makefile),
 *     tests/test_oracle.py::test_oracle_matches_reference_*;
 *   - against golden vectors produced by that build (tests/golden/).
 *
 * Status codes mirror the reference exception hierarchy (include/uot/error.hpp:9-37).
 */
#ifndef UOT_ORACLE_H
#define UOT_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  ORC_OK = 0,
  ORC_INVALID_PARAMETER = 1, /* uot::InvalidParameter */
  ORC_DEGENERATE_SUM = 2,    /* uot::DegenerateSum */
  ORC_PARTITION_ERROR = 3    /* uot::PartitionError */
};

/* SplitMix64 (include/uot/rng.hpp:9-25). */
uint64_t orc_splitmix64_next(uint64_t* state);
double orc_next_unit(uint64_t* state);

/* gen_problem_t (include/uot/problem_io.hpp:17-31): A row-major, then rpd, then
 * cpd, all from one SplitMix64 stream. Draw k (0-based) only depends on
 * seed + (k+1)*golden, so `threads` > 1 fills A in parallel, bit-identically. */
int orc_gen_problem_f32(uint64_t seed, size_t m, size_t n, float* a, double* rpd, double* cpd,
                        int threads);
int orc_gen_problem_f64(uint64_t seed, size_t m, size_t n, double* a, double* rpd, double* cpd,
                        int threads);

/* compute_fi / rescale_factor / convergence_error (src/scaling.cpp:9-29). */
int orc_compute_fi(double er, double ep, double* fi);
int orc_rescale_factor(double target, double sum, double fi, double* out);
double orc_convergence_error(const double* alpha, size_t m, const double* beta, size_t n);

/* balanced_blocks (src/plan.cpp:11-21): bounds[0..k], block w = [bounds[w], bounds[w+1]). */
void orc_balanced_blocks(size_t k, size_t rows, size_t* bounds);
/* RankPartition::make (src/plan.cpp:35-44): PartitionError when ranks < 1 or ranks > rows. */
int orc_rank_partition(size_t ranks, size_t rows, size_t* bounds);

/* init_col_sums, block-grouped (include/uot/fused.hpp:96-110); nblocks == 1 is the
 * plain row-major seed (fused.hpp:71-84). */
void orc_init_col_sums_f32(const float* a, size_t m, size_t n, size_t nblocks, double* cs);
void orc_init_col_sums_f64(const double* a, size_t m, size_t n, size_t nblocks, double* cs);

/* beta_from_state (include/uot/fused.hpp:146-157). */
int orc_beta_from_state(const double* col_sums, const double* cpd, size_t n, double fi,
                        double* beta);

/* fused_row_pass (include/uot/fused.hpp:119-144) on one row of n entries. */
int orc_fused_row_pass_f32(float* row, size_t n, const double* beta, double target, double fi,
                           double* next_cols, double* alpha);
int orc_fused_row_pass_f64(double* row, size_t n, const double* beta, double target, double fi,
                           double* next_cols, double* alpha);

/* fused_iterate_parallel (include/uot/fused.hpp:197-250): W worker threads over
 * balanced row blocks, per-worker partial column sums, ascending-worker
 * reduction. col_sums is the carried FusedState (in/out). W == 1 is
 * fused_iterate (fused.hpp:164-185) bit for bit. */
int orc_fused_iterate_f32(float* a, size_t m, size_t n, double* col_sums, const double* rpd,
                          const double* cpd, double fi, size_t workers, double* alpha,
                          double* beta);
int orc_fused_iterate_f64(double* a, size_t m, size_t n, double* col_sums, const double* rpd,
                          const double* cpd, double fi, size_t workers, double* alpha,
                          double* beta);

/* fused_solve (include/uot/fused.hpp:259-285). `a` is the plan, updated in place
 * (the reference copies p.a first, fused.hpp:268). Outputs iterations,
 * final_error, converged; col_sums (may be NULL) receives the carried state. */
int orc_fused_solve_f32(float* a, size_t m, size_t n, const double* rpd, const double* cpd,
                        double er, double ep, double tol, size_t max_iter, size_t workers,
                        double* alpha, double* beta, double* col_sums, size_t* iterations,
                        double* final_error, int* converged);
int orc_fused_solve_f64(double* a, size_t m, size_t n, const double* rpd, const double* cpd,
                        double er, double ep, double tol, size_t max_iter, size_t workers,
                        double* alpha, double* beta, double* col_sums, size_t* iterations,
                        double* final_error, int* converged);

/* allreduce_vectors (src/allreduce.cpp:6-15): ascending-rank elementwise sum. */
void orc_allreduce_vectors(const double* const* parts, size_t ranks, size_t n, double* out);

/* distributed_solve (include/uot/distributed.hpp:52-130): ranks own balanced row
 * blocks; one allreduce of the n-vector of column partials per iteration.
 * allreduce_calls / doubles_reduced mirror CommStats (distributed.hpp:24-27). */
int orc_distributed_solve_f32(float* a, size_t m, size_t n, const double* rpd, const double* cpd,
                              double er, double ep, double tol, size_t max_iter, size_t ranks,
                              double* alpha, double* beta, size_t* iterations,
                              double* final_error, int* converged, uint64_t* allreduce_calls,
                              uint64_t* doubles_reduced);

/* validate_problem's positivity/shape rules (include/uot/problem.hpp:64-98). */
int orc_validate_f32(const float* a, size_t m, size_t n, const double* rpd, const double* cpd,
                     double er, double ep);

#ifdef __cplusplus
}
#endif

#endif /* UOT_ORACLE_H */
