/*
 * uot_cuda.h — C ABI of the B200-native fused Sinkhorn-UOT solver.
 *
 * This is the drop-in boundary for the reference's solver API
 * (/root/reference/proj/core/include/uot, "namespace uot"). The reference has no
 * FFI of its own: its boundary is header-only C++ templates. Each entry point
 * below states the reference interface it replaces. A C++ facade with the
 * reference's exact types and exception classes sits on top
 * (include/uot/cuda.hpp); Python binds it with ctypes
 * (paper_2412_11079_b200/uot.py). See INTEGRATION.md.
 *
 * Conventions: plain pointers and sizes only; host buffers unless a name says
 * _device; every call returns a status code and never throws across the ABI.
 * The problem stays resident in HBM between calls ("session"): the reference's
 * per-iteration API mutates a host Matrix<T>& in place (fused.hpp:164-191),
 * which at 4 GiB per iteration would be PCIe-bound, so the host matrix is only
 * touched by uot_set_problem / uot_get_plan.
 */
#ifndef UOT_CUDA_H
#define UOT_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: the reference exception hierarchy (include/uot/error.hpp:9-37). */
#define UOT_OK 0
#define UOT_INVALID_PARAMETER 1 /* uot::InvalidParameter */
#define UOT_DEGENERATE_SUM 2    /* uot::DegenerateSum */
#define UOT_PARTITION_ERROR 3   /* uot::PartitionError */
#define UOT_CONFIG_ERROR 4      /* uot::ConfigError (launch configuration cannot cover the matrix) */
#define UOT_CUDA_ERROR 5        /* CUDA runtime failure (no reference analogue) */
#define UOT_NCCL_ERROR 6        /* NCCL failure (no reference analogue) */
#define UOT_IO_ERROR 7          /* uot::IoError (problem file container) */

/* Dtype codes: uot::Dtype (include/uot/matrix.hpp:13). Both have a kernel: f32
 * storage with f64 arithmetic (the products rounded once to fp32, as T(double)
 * in fused.hpp:128-140), or f64 storage (plain f64 products). The resident
 * (whole solve in one launch) path is f32-only. */
#define UOT_F32 1
#define UOT_F64 2

#if defined(__GNUC__)
#define UOT_API __attribute__((visibility("default")))
#else
#define UOT_API
#endif

typedef struct uot_ctx uot_ctx;

/* Layout and launch facts of a session (for tests, benches and DESIGN.md). */
typedef struct uot_layout {
  uint64_t rows;         /* local rows (row block of this rank) */
  uint64_t cols;         /* logical columns */
  uint64_t row_offset;   /* first global row of this rank */
  uint64_t global_rows;
  uint32_t pitch;        /* floats per device row (>= cols, multiple of 4*G) */
  uint32_t slice;        /* floats per CTA column slice */
  uint32_t G;            /* CTAs sharing a row */
  uint32_t groups;       /* row groups (grid = groups*G) */
  uint32_t rows_per_step;
  uint32_t threads;      /* CTA size of the sweep kernel */
  uint32_t chunks;       /* float4 chunks per thread per row */
  uint32_t smem_bytes;   /* dynamic shared memory of the sweep kernel */
  uint32_t nbuf;         /* shared-memory ring slots */
  uint32_t sms;
  int32_t rank, nranks, device, evict_first;
  int32_t smid_map;      /* sweep CTAs addressed by SM id (row groups on neighbouring SMs) */
  int32_t exchange;      /* 0 single GPU, 1 NCCL allreduce, 2 fused peer-memory exchange */
  int32_t resident;      /* uot_iterate runs as ONE persistent launch, matrix in shared memory (resident.cuh) */
  int32_t dtype;         /* UOT_F32 (Problem<float>) or UOT_F64 (Problem<double>) */
  int32_t dynamic;       /* 1: row batches handed out by a device counter (uot_set_schedule) */
  int32_t schedule;      /* UOT_SCHEDULE_* of the streaming sweep */
  int32_t pinned;        /* one sweep CTA on every SM, slot = SM id (the weighted schedule is available) */
  int32_t variant;       /* iteration schedule (UOT_VARIANT_*); rows wider than #SMs slices (G > #SMs,
                            > 1.2M fp32 columns on a B200) run UOT_VARIANT_TWO_PASS, the only one they allow */
  uint32_t keep_batches; /* static schedules of a streaming problem: each CTA stores its last keep_batches
                            batches L2-resident and the next sweep walks its row block the other way */
} uot_layout;

/* ---- sessions ---------------------------------------------------------- */

/* New session for a rows x cols problem on `device`. Replaces the problem/plan
 * copy at the top of fused_solve (fused.hpp:262-272). */
UOT_API int uot_create(uot_ctx** out, uint64_t rows, uint64_t cols, int dtype, int device);

/* Multi-GPU session: rank `rank` of `nranks` owns the row block
 * RankPartition::make(nranks, global_rows).blocks[rank] (src/plan.cpp:35-44;
 * PartitionError when nranks > global_rows) and joins the NCCL communicator
 * identified by `nccl_id` (128 bytes from uot_nccl_unique_id on rank 0).
 * Replaces distributed_solve's rank state (distributed.hpp:65-79). nranks == 1
 * with a non-NULL id builds a one-rank communicator and runs the same NCCL
 * exchange path (NULL: a plain single-GPU session). */
UOT_API int uot_create_dist(uot_ctx** out, uint64_t global_rows, uint64_t cols, int dtype, int device,
                    int rank, int nranks, const uint8_t* nccl_id);
UOT_API int uot_nccl_unique_id(uint8_t* out128);

/* Multi-GPU session whose per-iteration allreduce of the column sums
 * (distributed.hpp:88-94, allreduce_vectors src/allreduce.cpp:6-15) is fused
 * into the finalize kernels over peer memory (CUDA IPC over NVLink/NVSwitch; two
 * processes on one GPU also work): every rank pushes its column sums into all
 * peers' receive tables and sums the nranks rows in ascending rank order —
 * bit-identical on every rank, no NCCL. Collective protocol: create on every
 * rank, all-gather the 64-byte uot_peer_handle of each rank (any transport),
 * then uot_peer_connect(ctx, handles[nranks*64]) on every rank. */
UOT_API int uot_create_peer(uot_ctx** out, uint64_t global_rows, uint64_t cols, int dtype, int device,
                            int rank, int nranks);
UOT_API int uot_peer_handle(const uot_ctx* ctx, uint8_t* out64);
UOT_API int uot_peer_connect(uot_ctx* ctx, const uint8_t* handles);
/* 0 single GPU, 1 NCCL allreduce, 2 fused peer-memory exchange. */
UOT_API int uot_exchange_mode(const uot_ctx* ctx);

/* ---- single-process rank groups ------------------------------------------
 * The reference's in-process distributed_solve(p, tol, max_iter, ranks |
 * RankPartition) (distributed.hpp:52-136, 139-142): ONE process drives all
 * ranks. uot_create_group makes `nranks` peer sessions (rank r on devices[r];
 * devices NULL = round robin over the visible GPUs; ranks may share a GPU) over
 * the row blocks `bounds[0..nranks]` (NULL = RankPartition::make, plan.cpp:35-44;
 * a given partition must cover the rows with non-empty blocks, else
 * UOT_PARTITION_ERROR) and maps their exchange regions into each other directly
 * (peer access, no IPC). out[0..nranks) receives the sessions; on failure the
 * caller destroys every non-null entry. Per rank: uot_set_problem with its block
 * (uot_get_layout: row_offset, rows), then the collective calls below replace
 * uot_init_col_sums / uot_iterate (which refuse group ranks). The exchange is the
 * fused peer-memory one (ascending-rank sum, allreduce.cpp:6-15); stage 2 of
 * every rank is stream-ordered after stage 1 of all ranks. */
UOT_API int uot_create_group(uot_ctx** out, uint64_t global_rows, uint64_t cols, int dtype, const int* devices,
                             int nranks, const uint64_t* bounds);
UOT_API int uot_group_init_col_sums(uot_ctx* const* ctxs, int nranks);
UOT_API int uot_group_iterate(uot_ctx* const* ctxs, int nranks, uint64_t k, double tol, uint64_t* iterations,
                              double* final_error, int* converged);

/* ---- problem files (.uotp, problem_io.cpp:13-141) --------------------- */

/* read_problem's header checks (problem_io.cpp:106-135) without the payload:
 * extents, dtype (1 f32, 2 f64) and coefficients. UOT_IO_ERROR on a malformed
 * container; the message is uot_last_io_error(). Host only. */
UOT_API int uot_problem_file_info(const char* path, uint64_t* m, uint64_t* n, int* dtype, double* er, double* ep);
UOT_API const char* uot_last_io_error(void);
/* read_problem + uot_set_problem for this session's row block: the rows of this
 * rank are streamed from the file to HBM through page-locked staging (the
 * global matrix is never materialised on the host). f32 files only. */
UOT_API int uot_load_problem_file(uot_ctx* ctx, const char* path);
/* write_problem of the session's CURRENT plan with its marginals and er/ep, the
 * reference's container byte for byte. Multi-rank: every rank writes its rows
 * and rpd slice, rank 0 the header and cpd (collective on the path). */
UOT_API int uot_save_problem_file(uot_ctx* ctx, const char* path);

/* Iteration schedule of uot_iterate (single GPU). FUSED is the product path
 * (fused_iterate_parallel, fused.hpp:197-250: one read + one write of P per
 * iteration). TWO_PASS is the paper's GPU data flow emulated by tiled_iterate
 * (tiled.hpp:210-229: part4 -> row factors -> part2, 2 reads + 2 writes) and
 * BASELINE the reference's four-sweep baseline_iterate (baseline.hpp:100-110:
 * 4 reads + 2 writes) — ablations that measure the traffic model of
 * metrics.cpp:60-77 on HBM. All three compute the same iteration. */
#define UOT_VARIANT_FUSED 0
#define UOT_VARIANT_TWO_PASS 1
#define UOT_VARIANT_BASELINE 2
UOT_API int uot_set_variant(uot_ctx* ctx, int variant);

/* Row-batch schedule of the fused sweep. Every row group sums its column
 * partials in row order and the groups are reduced in ascending order, as the
 * reference's ordered reduction (fused.hpp:193-196, 242-248); the schedules
 * differ in which rows a group owns.
 *   UNIFORM (default): balanced_blocks (plan.cpp:11-21) over the groups —
 *     bit-reproducible run to run on any GPU; paced by the slowest SMs (B200
 *     SMs stream HBM at per-TPC rates that differ by up to 1.6x).
 *   WEIGHTED: static contiguous row blocks proportional to per-group weights
 *     (uot_set_group_weights, or measured by uot_calibrate_schedule); CTA slots
 *     are pinned to SMs, so the weights stay attached to the SMs they describe —
 *     bit-reproducible for given weights, and balanced.
 *   DYNAMIC: batches go to whichever CTA asks next (a device counter); the
 *     f64 column sums then add rows in a run-dependent order (results agree to
 *     ~1e-12 relative between runs).
 * WEIGHTED needs one sweep CTA on every SM (uot_layout.pinned). */
#define UOT_SCHEDULE_UNIFORM 0
#define UOT_SCHEDULE_WEIGHTED 1
#define UOT_SCHEDULE_DYNAMIC 2
UOT_API int uot_set_schedule(uot_ctx* ctx, int schedule);
/* on: WEIGHTED when weights are set, else UNIFORM; off: DYNAMIC. */
UOT_API int uot_set_deterministic(uot_ctx* ctx, int on);
/* Weights (1 .. 2^20) of the `n` = uot_layout.groups row groups, group g = CTA
 * slots g*G .. g*G+G-1 = SMs g*G .. ; selects WEIGHTED. */
UOT_API int uot_set_group_weights(uot_ctx* ctx, const uint32_t* weights, uint32_t n);
UOT_API int uot_get_group_weights(const uot_ctx* ctx, uint32_t* weights, uint32_t n);
/* Measure the weights on a scratch copy of the plan: k dynamic iterations
 * (k in [2, 64], the first discarded) give each group's first weight (the row
 * batches it took), then three rounds of two weighted iterations rescale each
 * weight by (mean completion time / the group's completion time)^0.75, so the
 * static row blocks finish together. The session's plan, factors, column sums
 * and stop state are unchanged. Needs a problem and init_col_sums; selects
 * WEIGHTED. Store the weights (uot_get_group_weights) to reuse them across
 * sessions and processes on the same GPU. */
UOT_API int uot_calibrate_schedule(uot_ctx* ctx, uint32_t k);
/* Schedule statistics of the last sweep: per CTA slot its SM id and the row
 * batches it streamed; per row group its weight (1 when none are set). Each
 * output may be NULL; sizes: grid = groups * G, groups (uot_get_layout). */
UOT_API int uot_get_schedule_stats(const uot_ctx* ctx, uint32_t* cta_smid, uint32_t* cta_batches,
                                   uint32_t* group_weight);
/* Small single-GPU f32 problems whose row blocks fit shared memory run a whole
 * uot_iterate call as ONE cooperative launch (resident.cuh). Default 1; 0 keeps
 * the streaming sweep + finalize per iteration (tests, ablations). */
UOT_API int uot_set_resident(uot_ctx* ctx, int on);

UOT_API void uot_destroy(uot_ctx* ctx);
UOT_API const char* uot_last_error(const uot_ctx* ctx);
UOT_API int uot_get_layout(const uot_ctx* ctx, uot_layout* out);
/* The CUDA stream every kernel of the session is launched on (cudaStream_t). */
UOT_API void* uot_get_stream(const uot_ctx* ctx);

/* ---- problem ----------------------------------------------------------- */

/* Upload Problem<float> {a (rows x cols row-major, this rank's rows), rpd
 * (this rank's rows), cpd (all cols), er, ep} (problem.hpp:19-28) and validate
 * it like require_valid (problem.hpp:64-103) -> UOT_INVALID_PARAMETER. fi =
 * compute_fi(er, ep) (scaling.cpp:9-13). Resets the iteration state. */
UOT_API int uot_set_problem(uot_ctx* ctx, const float* a, const double* rpd, const double* cpd, double er,
                    double ep);
/* Problem<double> (Dtype::f64 sessions): same contract, fp64 matrix. */
UOT_API int uot_set_problem_f64(uot_ctx* ctx, const double* a, const double* rpd, const double* cpd, double er,
                                double ep);
/* gen_problem_t<T>(seed, global_rows, cols) (problem_io.hpp:17-31) generated
 * directly in HBM, bit-identical to the host generator, then er/ep applied. */
UOT_API int uot_generate_problem(uot_ctx* ctx, uint64_t seed, double er, double ep);
/* Override the damping exponent (fused_iterate takes fi directly, fused.hpp:165).
 * fi must lie in (0, 1]. */
UOT_API int uot_set_fi(uot_ctx* ctx, double fi);
/* fused_iterate's inputs as the caller holds them (fused.hpp:164-191): the
 * current plan `a` (dtype UOT_F32 or UOT_F64, must match the session), rpd,
 * cpd and fi, uploaded WITHOUT require_valid's checks — the reference's
 * fused_iterate validates only shapes, and throws DegenerateSum from
 * rescale_factor, which the device reports the same way. Resets the iteration
 * state; follow with uot_set_col_sums (the FusedState) and uot_iterate(1). */
UOT_API int uot_set_iterate_input(uot_ctx* ctx, const void* a, int dtype, const double* rpd, const double* cpd,
                                  double fi);
/* Replace only the plan (the current matrix) of this rank; marginals stay. */
UOT_API int uot_set_plan(uot_ctx* ctx, const float* a);
UOT_API int uot_set_plan_f64(uot_ctx* ctx, const double* a);

/* ---- the path ---------------------------------------------------------- */

/* FusedState{init_col_sums(plan, blocks)} (fused.hpp:96-110, 271): one read
 * sweep over P, then column factors beta(1). Multi-GPU: the ranks' seeds are
 * allreduced (distributed.hpp:78 + 88-92). */
UOT_API int uot_init_col_sums(uot_ctx* ctx);
/* FusedState given by the caller (fused_iterate's state argument). */
UOT_API int uot_set_col_sums(uot_ctx* ctx, const double* col_sums);
UOT_API int uot_get_col_sums(const uot_ctx* ctx, double* out);

/* Run up to k fused iterations on the device (fused_iterate_parallel,
 * fused.hpp:197-250, one sm_100a sweep kernel + one finalize kernel each),
 * stopping after the first iteration whose convergence_error <= tol
 * (fused.hpp:273-281). Outputs: iterations completed by this call, the error of
 * the last completed iteration, and whether it converged. Use tol = 1e-300 for
 * fixed-length runs. A degenerate row or column sum returns UOT_DEGENERATE_SUM
 * (detected on device; the plan is then in an unspecified partially-updated
 * state, as after the reference's throw). */
UOT_API int uot_iterate(uot_ctx* ctx, uint64_t k, double tol, uint64_t* iterations, double* final_error,
                int* converged);

/* uot_iterate with the device time of the k iterations (CUDA events on the
 * session stream around all of its launches) in *device_ms. */
UOT_API int uot_iterate_timed(uot_ctx* ctx, uint64_t k, double tol, uint64_t* iterations,
                              double* final_error, int* converged, double* device_ms);
/* Wait for all work queued on the session stream. */
UOT_API int uot_synchronize(uot_ctx* ctx);

/* ScalingFactors of the last completed iteration (problem.hpp:30-33); alpha is
 * this rank's rows, beta all columns. */
UOT_API int uot_get_factors(const uot_ctx* ctx, double* alpha, double* beta);
/* The plan (rows x cols row-major) of this rank. */
UOT_API int uot_get_plan(const uot_ctx* ctx, float* out);
UOT_API int uot_get_plan_f64(const uot_ctx* ctx, double* out);
/* Completed iterations and the error of the last one. */
UOT_API int uot_get_report(const uot_ctx* ctx, uint64_t* iterations, double* final_error, int* converged);
/* CommStats (distributed.hpp:24-27). */
UOT_API int uot_get_comm_stats(const uot_ctx* ctx, uint64_t* allreduce_calls, uint64_t* doubles_reduced);

/* Device time of the sweep / finalize kernels of the last uot_iterate call when
 * timing is enabled (CUDA events on the session stream around each launch). */
UOT_API int uot_set_timing(uot_ctx* ctx, int enabled);
UOT_API int uot_get_timing(const uot_ctx* ctx, double* sweep_ms, double* finalize_ms, uint64_t* sweeps);
/* Number of kernels this session launched so far (all kinds). */
UOT_API uint64_t uot_kernel_launches(const uot_ctx* ctx);

/* Page-locked host memory (cudaMallocHost) for fast uploads / downloads. */
UOT_API void* uot_host_alloc(uint64_t bytes);
UOT_API void uot_host_free(void* p);

/* ---- scalars and plans (host; scaling.cpp:9-29, plan.cpp:11-44) -------- */
UOT_API int uot_compute_fi(double er, double ep, double* fi);
UOT_API int uot_rescale_factor(double target, double sum, double fi, double* out);
UOT_API double uot_convergence_error(const double* alpha, uint64_t m, const double* beta, uint64_t n);
/* bounds[0..ranks]: rank r owns [bounds[r], bounds[r+1]). */
UOT_API int uot_rank_partition(uint64_t ranks, uint64_t rows, uint64_t* bounds);
/* Rows [row0, row0+rows) of gen_problem_t<float>(seed, global_rows, n): the
 * block's A, its rpd slice and the full cpd (either may be NULL). */
UOT_API int uot_gen_block_f32(uint64_t seed, uint64_t global_rows, uint64_t n, uint64_t row0,
                              uint64_t rows, float* a, double* rpd, double* cpd, int threads);
UOT_API int uot_gen_block_f64(uint64_t seed, uint64_t global_rows, uint64_t n, uint64_t row0,
                              uint64_t rows, double* a, double* rpd, double* cpd, int threads);
/* gen_problem_t<float> on the host (threads > 1 fills A in parallel). */
UOT_API int uot_gen_problem_f32(uint64_t seed, uint64_t m, uint64_t n, float* a, double* rpd, double* cpd,
                        int threads);

#ifdef __cplusplus
}
#endif

#endif /* UOT_CUDA_H */
