/*
 * csrecon_b200 — C ABI of the B200-native ADMM + NUDFT reconstruction path.
 *
 * Drop-in boundary for the reference package csrecon (/root/reference/pkg,
 * Python).  The reference's plug-in point is its kernel table
 * (kernels.py:212-231) behind DftOperator.forward/adjoint
 * (operators.py:185-203), transform.theta/theta_adjoint/soft_threshold
 * (transform.py:14-42), tensor.hermitian_dot/axpy (tensor.py:44-64) and the
 * solver entry admm_reconstruct (solver.py:274-360).  Each entry point below
 * names the reference interface it replaces.  The Python host package
 * (paper_2006_14080_b200) binds these with ctypes; INTEGRATION.md shows the
 * binding a csrecon maintainer would add.
 *
 * Conventions
 *  - complex data are interleaved complex64 (float2), C-contiguous, in the
 *    reference's index order: image (T, nx, ny) with pixel n = x*ny + y
 *    (acquisition.py:15-43); k-space (T*M, C) sample-major, readout-major
 *    rows (acquisition.py:46-53, 99-122).  T = 1 for the static problem.
 *  - every buffer argument is caller-owned DEVICE memory unless documented
 *    as host; the plan owns its factors and workspace.  Hot calls never
 *    allocate.  Calls are ordered on the given stream (cudaStream_t passed
 *    as void*; NULL = legacy default stream).
 *  - a plan is bound to one device and is not re-entrant; different plans
 *    may be driven from different threads.
 *  - return value: CSR_OK or an error code; csr_last_error() gives the
 *    thread-local message.  The host wrapper maps CSR_ERR_SHAPE to
 *    ShapeMismatchError (tensor.py:17-18), CSR_ERR_NONFINITE to
 *    CgDivergenceError (solver.py:30-31), CSR_ERR_OOM to MemoryBudgetError
 *    (operators.py:26-27) and the rest to RuntimeError.
 *  - there is no CPU fallback: without a usable sm_100 device every call
 *    fails with CSR_ERR_CUDA.
 */
#ifndef CSRECON_B200_H
#define CSRECON_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CSR_OK 0
#define CSR_ERR_SHAPE 1
#define CSR_ERR_OOM 2
#define CSR_ERR_CUDA 3
#define CSR_ERR_NCCL 4
#define CSR_ERR_NONFINITE 5
#define CSR_ERR_ARG 6

typedef struct csr_plan csr_plan;
typedef struct csr_comm csr_comm;

/* Geometry of one encoding operator (one worker's shard).  Replaces
 * DftOperator.build(trajectory, grid, sens, mode, precision)
 * (operators.py:141-164): coords are the (T*M, 2) cycles/pixel sample
 * locations (host f64, Trajectory.coords, acquisition.py:46-73), sens the
 * (C, nx, ny) coil maps (device complex64).  Frames t use rows
 * [t*M, (t+1)*M).  Factors are generated on the device in f64 and rounded
 * once to complex64, exactly as _unit_phase (operators.py:50-59). */
typedef struct csr_plan_desc {
    int32_t nx, ny;
    int32_t n_frames;     /* T >= 1 */
    int32_t n_coils;      /* C >= 1 (coils owned by this plan) */
    int64_t n_samples;    /* M >= 1 samples per frame */
    const double *coords; /* HOST, (T*M, 2) */
    const void *sens;     /* DEVICE complex64 (C, nx, ny); copied */
    int32_t device;       /* CUDA ordinal */
    int32_t flags;        /* CSR_PLAN_FRAME_SHARD: this plan holds a contiguous
                             block of the frames of a 2-D+t problem split across
                             ranks; temporal differences at the block edges use
                             halo frames exchanged with the neighbour ranks.
                             CSR_PLAN_ORDERED_SAMPLES: this plan holds a run of
                             whole sample chunks of a static problem (see
                             csr_sample_chunking) */
    int64_t chunk_samples; /* CSR_PLAN_ORDERED_SAMPLES: the global chunk size */
    int64_t total_samples; /* CSR_PLAN_ORDERED_SAMPLES: samples of the whole
                              problem (all ranks) */
} csr_plan_desc;

#define CSR_PLAN_FRAME_SHARD 1
#define CSR_PLAN_ORDERED_SAMPLES 2

/* Order-stable sample sharding (the reference's default plan:
 * make_shard_plan(n_samples, n_workers, chunk_size), sharding.py:76-113, with
 * ChunkedDftOperator, operators.py:206-272, and ordered_chunk_sum,
 * sharding.py:174-208).  The global chunk grid of a static problem: chunk
 * k covers samples [k*chunk, min((k+1)*chunk, n_samples)).  A plan built with
 * CSR_PLAN_ORDERED_SAMPLES over any contiguous run of whole chunks computes
 * each of its samples' k-space values and each chunk's adjoint partial image
 * bit-identically to a plan of the whole problem; with a comm attached the
 * chunk partials of all ranks are gathered (NCCL all-gather) and folded in
 * global chunk order, so every reduced image is bitwise independent of the
 * number of ranks.  chunk is a multiple of 128 samples. */
int csr_sample_chunking(int32_t nx, int32_t ny, int32_t n_coils, int64_t n_samples,
                        int64_t *chunk_samples, int32_t *n_chunks);

typedef struct csr_plan_info {
    int64_t factor_bytes;    /* resident encoding factors */
    int64_t workspace_bytes; /* scratch owned by the plan */
    int32_t gemm_path;       /* 1 = tcgen05 tensor-core GEMMs, 0 = SIMT */
    int32_t split_k;         /* adjoint split-K factor */
} csr_plan_info;

int csr_plan_create(const csr_plan_desc *desc, csr_plan **out);
/* Release a plan.  Waits for the plan's pending work on every stream it was
 * used on (operator calls run on the caller's stream) before its memory is
 * returned to the device pool. */
int csr_plan_destroy(csr_plan *plan);

/* A plan from the reference's own factor arrays instead of coordinates
 * (one frame): DftOperator(factors, sens_maps, "separable")
 * (operators.py:109-139) with the DftFactors of build_factors
 * (operators.py:30-47, 72-82).  phase0 is P0 (M, nx); phase1 is P1 in one of
 * the layouts the reference's kernel table passes around (kernels.py
 * :257-262): the (M, ny) factor itself, the operator's phase1_t (ny, M)
 * (operators.py:136) or its phase1_conj (M, ny) (operators.py:137).  All
 * DEVICE complex64; copied into the plan. */
#define CSR_P1_ROWS 0
#define CSR_P1_T 1
#define CSR_P1_CONJ 2
typedef struct csr_factor_desc {
    int32_t nx, ny;
    int32_t n_coils;
    int64_t n_samples;
    const void *phase0;     /* (M, nx) */
    const void *phase1;     /* layout given by phase1_layout */
    int32_t phase1_layout;  /* CSR_P1_ROWS | CSR_P1_T | CSR_P1_CONJ */
    const void *sens;       /* (C, nx, ny) */
    int32_t device;
} csr_factor_desc;
int csr_plan_create_from_factors(const csr_factor_desc *desc, csr_plan **out);
int csr_plan_get_info(const csr_plan *plan, csr_plan_info *info);

/* Copy frame t's factors P0 (M, nx) and P1 (M, ny) (complex64) out —
 * build_factors / DftFactors (operators.py:30-82). */
int csr_plan_get_factors(const csr_plan *plan, int32_t frame, void *p0,
                         void *p1, void *stream);

/* DftOperator.forward (operators.py:185-193 -> kernels.nudft_forward_sep,
 * kernels.py:71-78): image (T, nx, ny) -> kdata (T*M, C). */
int csr_forward(csr_plan *plan, const void *image, void *kdata, void *stream);

/* DftOperator.adjoint (operators.py:195-203 -> kernels.nudft_adjoint_sep,
 * kernels.py:81-88): kdata (T*M, C) -> image (T, nx, ny); no 1/N. */
int csr_adjoint(csr_plan *plan, const void *kdata, void *image, void *stream);

/* The reference's kernel-table entries themselves (kernels.py:257-262,
 * _forward_sep_np / _adjoint_sep_np kernels.py:71-88), all DEVICE complex64
 * pointers: nudft_forward_sep(phase0 (M,nx), phase1_t (ny,M), sens (C,nx,ny),
 * image (nx,ny)) -> out (M,C); nudft_adjoint_sep(phase0, phase1_conj (M,ny),
 * sens, data (M,C)) -> out (nx,ny).  Each call builds a transient plan from
 * the factors (csr_plan_create_from_factors) and releases it: an exact
 * drop-in for one call; hot loops keep a plan. */
int csr_nudft_forward_sep(const void *phase0, const void *phase1_t, const void *sens,
                          const void *image, void *out, int32_t nx, int32_t ny,
                          int32_t n_coils, int64_t n_samples, void *stream);
int csr_nudft_adjoint_sep(const void *phase0, const void *phase1_conj, const void *sens,
                          const void *data, void *out, int32_t nx, int32_t ny,
                          int32_t n_coils, int64_t n_samples, void *stream);

/* ChunkedDftOperator.adjoint (operators.py:254-265): the per-chunk partial
 * images (n_chunks, nx, ny), unsummed, of an order-stable plan
 * (CSR_PLAN_ORDERED_SAMPLES; n_chunks = csr_plan_info.split_k).  Other
 * plans return their split-K partials. */
int csr_adjoint_chunks(csr_plan *plan, const void *kdata, void *chunks, void *stream);
/* The same with the k-space operand scale taken from a caller-supplied bound
 * on the data (component-wise max |Re|, |Im| over ALL workers' chunks): the
 * fp16 split's scale is an exact power of two of that bound, so chunk
 * partials computed by different workers are bit-identical however the
 * chunk maxima differ (csr_adjoint_chunks scales by this plan's own data;
 * the native multi-rank loop max-allreduces the bound itself).  A bound
 * below the plan's own max is raised to it. */
int csr_adjoint_chunks_bound(csr_plan *plan, const void *kdata, void *chunks, float bound,
                             void *stream);

/* normal_operator (solver.py:128-139) without the allreduce:
 * out = F^H F x + (beta/2) Theta^H Theta x. */
int csr_normal(csr_plan *plan, const void *x, void *out, double beta,
               void *stream);

/* transform.theta (transform.py:14-18 -> kernels.py:91-95): img (T,nx,ny)
 * -> diffs (D, T, nx, ny), D = 2 for T == 1 (the reference) and 3 for T > 1
 * (temporal component, extension). */
int csr_theta(int32_t n_frames, int32_t nx, int32_t ny, const void *img,
              void *diffs, void *stream);
/* transform.theta_adjoint (transform.py:21-26 -> kernels.py:98-101). */
int csr_theta_adjoint(int32_t n_frames, int32_t nx, int32_t ny,
                      const void *diffs, void *img, void *stream);
/* transform.soft_threshold (transform.py:29-42 -> kernels.py:104-108):
 * z*(1 - t/|z|) where |z| > t else 0; t < 0 -> CSR_ERR_ARG. */
int csr_soft_threshold(const void *z, int64_t n, float threshold, void *out,
                       void *stream);
/* tensor.hermitian_dot (tensor.py:44-50): out = sum conj(a)*b accumulated
 * in f64; out is DEVICE double[2] (re, im).  Deterministic. */
int csr_hermitian_dot(const void *a, const void *b, int64_t n, double *out,
                      void *stream);
/* sum |z| over complex64 z in f64 (objective's l1 term, solver.py:204);
 * out is DEVICE double[1]. */
int csr_abs_sum(const void *z, int64_t n, double *out, void *stream);
/* tensor.axpy (tensor.py:58-64): out = y + alpha*x, alpha cast to
 * complex64 first.  out may alias y. */
int csr_axpy(double alpha_re, double alpha_im, const void *x, const void *y,
             int64_t n, void *out, void *stream);

/* ReconParams (solver.py:34-61) + lam_t for the temporal term. */
typedef struct csr_admm_params {
    double lam, lam_t, beta, admm_rtol, cg_atol;
    int32_t admm_max_iters, cg_max_iters;
} csr_admm_params;

/* One RunReport.iterations record (solver.py:316-324). */
typedef struct csr_iter_log {
    int32_t iteration, cg_iterations;
    double alpha, cg_final_residual_sq;
} csr_iter_log;

typedef struct csr_run_stats {
    int32_t n_iterations;     /* ADMM iterations executed */
    int32_t allreduce_calls;  /* image collectives issued (CommStats) */
    double setup_ms, solve_ms; /* device time: F^H d setup, ADMM loop */
    int32_t graph_used;       /* 1 if the iteration ran as a CUDA graph */
    int32_t kernels_per_iter; /* kernel launches per ADMM iteration */
} csr_run_stats;

/* admm_reconstruct (solver.py:274-360) on this plan's device: rho0 = fhd =
 * allreduce(F^H d) (two setup collectives, solver.py:307-309), then the ADMM
 * loop (admm_step, solver.py:163-194) with zero-start CG (cg_solve,
 * solver.py:87-125) and one image allreduce per CG iteration when a comm
 * is attached.  kdata (T*M, C) device; rho_out (T, nx, ny) device;
 * log = HOST array of admm_max_iters records.  Non-finite CG residual ->
 * CSR_ERR_NONFINITE (CgDivergenceError).  snapshots (device, optional):
 * (admm_max_iters+1, T, nx, ny) receives rho0 and the image after every
 * iteration (the reference's rank-0 snapshots, solver.py:315-324). */
int csr_admm_run(csr_plan *plan, const csr_admm_params *params,
                 const void *kdata, void *rho_out, csr_iter_log *log,
                 csr_run_stats *stats, void *stream, void *snapshots);

/* Benchmark timing for csr_admm_run on this plan: when iter_ms (HOST,
 * >= admm_max_iters floats) is set, every ADMM iteration is bracketed by
 * CUDA events on the plan stream and its device time written there; when
 * flush_buf (DEVICE, flush_bytes > L2) is also set, a buffer-overwrite
 * kernel evicts L2 between iterations, outside the timed intervals.
 * solve_ms then is the sum of the per-iteration times.  NULLs disable. */
int csr_plan_set_timing(csr_plan *plan, void *flush_buf, int64_t flush_bytes,
                        float *iter_ms);

/* Benchmark: average device time per launch of the tensor-core NUDFT
 * forward and adjoint GEMM kernels inside the ADMM loop of the last timed
 * csr_admm_run (first-CTA start to last-CTA end, %globaltimer stamps taken
 * by the kernels themselves, so the timed graph is unchanged), and how many
 * launches were averaged.  Zero counts on the SIMT path. */
int csr_plan_kernel_times(csr_plan *plan, double *fwd_ms, double *adj_ms,
                          int64_t *n_fwd, int64_t *n_adj);

/* Benchmark: the same live timing for one kernel slot of the iteration:
 * 0 forward GEMM, 1 adjoint GEMM, 2 mu, 3 rhs, 4 operand prep, 5 fused CG
 * tail, 6 ADMM post-update. */
int csr_plan_probe(csr_plan *plan, int32_t slot, double *ms, int64_t *n);

/* simulate_kspace (acquisition.py:233-257), double precision on the GPU:
 * kspace[t*M + k, c] = sum_{x,y} sens[c,x,y] image[t,x,y]
 *                      exp(-2 pi i (kx_k (x - nx/2) + ky_k (y - ny/2))).
 * coords (T*M, 2) f64, sens (C, nx, ny) c128, image (T, nx, ny) c128,
 * kspace (T*M, C) c128: all DEVICE pointers; stream-ordered. */
int csr_simulate_kspace(int32_t nx, int32_t ny, int32_t n_frames, int32_t n_coils,
                        int64_t n_samples, const double *coords, const void *sens,
                        const void *image, void *kspace, void *stream);

/* adjoint_reconstruct (solver.py:363-406): image = allreduce(F^H d). */
int csr_adjoint_reconstruct(csr_plan *plan, const void *kdata, void *image,
                            void *stream);

/* NCCL communicator for sharded runs (replaces the thread-barrier
 * allreduce of sharding._Collective, sharding.py:211-250).  Rank 0 makes
 * the 128-byte unique id, the host broadcasts it (torch.distributed), every
 * rank creates its comm on its own device and attaches it to its plan.
 * A plan with a communicator runs the collective code path of its shard
 * mode for any rank count, one rank included (NCCL reduces / exchanges with
 * itself), so every collective also runs on a single GPU. */
int csr_comm_unique_id(void *id128);
int csr_comm_create(const void *id128, int32_t nranks, int32_t rank,
                    int32_t device, csr_comm **out);
int csr_comm_destroy(csr_comm *comm);
int csr_plan_set_comm(csr_plan *plan, csr_comm *comm);
/* In-place sum allreduce of n floats (device) over the comm. */
int csr_comm_allreduce(csr_comm *comm, void *buf, int64_t n_floats,
                       void *stream);

const char *csr_last_error(void);
/* Number of this library's kernels launched since load (diagnostics). */
int64_t csr_kernel_launches(void);

#ifdef __cplusplus
}
#endif

#endif /* CSRECON_B200_H */
