/*
 * lsk.h -- C ABI of the B200-native log-domain Sinkhorn library (liblsk.so).
 *
 * Plain C types only: every array argument is a DEVICE pointer (e.g. a torch
 * tensor's data_ptr()), sizes are int32/int64, `stream` is a cudaStream_t
 * passed as void* (NULL = legacy default stream). No C++ exceptions cross
 * this boundary: every entry point returns LSK_OK (0) or a negative LSK_E*
 * code and records a message retrievable with lsk_last_error() (thread
 * local). Nothing here synchronises the host unless documented.
 *
 * Each entry point replaces one function of the reference package's Python
 * solver API (/root/reference/pkg/src/logsinkhorn); the cited file:line is the
 * interface it stands in for. The Python drop-in (paper_2605_00837_b200) and
 * INTEGRATION.md show the binding a maintainer of the reference would add.
 *
 * Arithmetic contract (all fp32 entry points): eps32 = (float)eps,
 * inv_eps = 1.0f / eps32 (IEEE), neg_eps = -eps32 (solver.py:259-260);
 * arguments are built with separately rounded fp32 ops in the reference's
 * order (solver.py:77-79, 84-86, 98-101, 108-112). Potentials match the
 * reference fp32 path within 1e-5 relative (max-norm); the summation tree and
 * exp/log last bits differ.
 */
#ifndef LSK_H
#define LSK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LSK_OK 0
#define LSK_EINVAL (-1)       /* bad argument (maps to ValueError / DimensionMismatch) */
#define LSK_ECUDA (-2)        /* CUDA runtime error */
#define LSK_EUNSUPPORTED (-3) /* shape not supported by this entry point */
#define LSK_ENCCL (-4)        /* NCCL error (sharded solver) */

/* lsk_solve_dense_f32 flags */
#define LSK_FLAG_STALE_SHIFT 1 /* one-pass stale-shift iteration (default fast path) */
#define LSK_FLAG_COST 2        /* compute the transport cost after the loop */
#define LSK_FLAG_EXPANSION 8   /* points, eps >= 5e-3: cost as |x|^2+|y|^2-2x.y in the stale sweeps; the
                                  caller requests it only when (max|x-x0|^2 + max|y-x0|^2) 2^-24 /
                                  (eps * normaliser) is small (x0 = the problem's first source point) */
#define LSK_FLAG_MULT 32       /* OPT-IN approximation, dense m <= 8192, uniform nu, n*m >= 2^20, 1e-3 <= eps
                                  <= 2e-3, iterations 1..1000 of a solve: the multiplicative column update
                                  (g-side terms from the f-side ones, 1 instead of 2 ex2 per element). Its
                                  potentials drift from the reference's by up to 3e-5 (per-potential max
                                  norm, K = 1000; the direct default stays within 1e-5 where the reference's
                                  own rounding allows): profiles/r2_mult_drift.md */
#define LSK_FLAG_STD_MULTIKERNEL 64 /* standard domain: force the two-pass multi-kernel loop (fp32 m <= 8192
                                       otherwise runs the one-pass persistent kernel) */
#define LSK_FLAG_NO_CLUSTER 512 /* dense m <= 1024, n <= 30720, uniform nu: run the 148-CTA grid solver instead
                                   of the cluster solvers (single cluster n <= 128, multi-cluster above; A/B) */
#define LSK_FLAG_UNIFORM_NU 16 /* dense m <= 8192: caller asserts log_nu[j] == log_nu[0] for all j (uniform
                                  target weights); the kernel verifies it and a violation ends the solve as
                                  status 2 after 0 iterations */

/* result[] slots written by lsk_solve_dense_f32 (device int32[8]) */
#define LSK_RES_STATUS 0     /* 0 not_converged, 1 converged, 2 numerical_failure (types.py:35-37) */
#define LSK_RES_ITERS 1      /* SolveReport.iterations */
#define LSK_RES_NTRACE 2     /* entries written to trace_iter / trace_err */
#define LSK_RES_ROWGUARD 4   /* stale-shift row LSEs recomputed exactly */
#define LSK_RES_COLGUARD 5   /* iterations whose columns were recomputed exactly */

const char* lsk_last_error(void);
int32_t lsk_version(void);

/* Largest m the single-launch persistent dense solver handles (8192 in this
 * build); lsk_solve_dense_f32 serves larger m with a multi-kernel loop of the
 * half-step kernels below (same semantics, no host synchronisation). */
int32_t lsk_solve_dense_max_cols(void);
/* Trace capacity for a solve: ceil(max_iter / check_interval) + 1. */
int32_t lsk_trace_capacity(int32_t max_iter, int32_t check_interval);
size_t lsk_solve_dense_workspace_bytes(int32_t n, int32_t m);

/*
 * Whole log-domain solve on a dense fp32 cost matrix, ONE cooperative launch
 * for m <= lsk_solve_dense_max_cols() (else an enqueued multi-kernel loop).
 * Replaces logsinkhorn.solver.solve (solver.py:230-337): alpha-first
 * alternation from zero potentials, a marginal-error check every
 * check_interval iterations (finiteness, then err, trace, stop), the extra
 * check at a cap that is not a checkpoint, and the transport cost unless the
 * solve failed. C is row-major with row stride ldc (floats, multiple of 4,
 * 16-byte aligned; columns m..ldc-1 must be zero when m % 4 != 0).
 * log_mu/mu (n) and log_nu (m) are the fp32 casts of the fp64 weights
 * (solver.py:256-258). Outputs: f_out (n), g_out (m), trace_iter/trace_err
 * (lsk_trace_capacity entries), result (int32[8], LSK_RES_*),
 * result_f (float[2]: final marginal error, transport cost).
 */
int32_t lsk_solve_dense_f32(const float* C, int64_t ldc, int32_t n, int32_t m, const float* log_mu,
                            const float* log_nu, const float* mu, double eps, double tol, int32_t max_iter,
                            int32_t check_interval, int32_t flags, float* f_out, float* g_out,
                            int32_t* trace_iter, float* trace_err, int32_t* result, float* result_f,
                            void* workspace, size_t workspace_bytes, void* stream);

/* Test hook: out_k = fl(fl(fl(a_k - c_k) * inv_eps) + l_k) computed by the
 * solver's packed argument builder (count even), to prove bitwise that no
 * FMA contraction reaches the reference arithmetic (solver.py:77-79). */
int32_t lsk_debug_arg3_f32(const float* a, const float* c, double eps, const float* l, float* out, int32_t count,
                           void* stream);

/* alpha = neg_eps * LSE_j((beta_j - C_ij) * inv_eps + log_nu_j)
 * -- update_alpha, solver.py:118-140 (_alpha_step 76-80). Any n, m. */
int32_t lsk_update_alpha_f32(const float* C, int64_t ldc, int32_t n, int32_t m, const float* beta,
                             const float* log_nu, double eps, float* alpha_out, void* stream);

/* beta = neg_eps * LSE_i((alpha_i - C_ij) * inv_eps + log_mu_i), reading C
 * row-major (coalesced column partials + fixed-order combine) -- update_beta,
 * solver.py:143-176 (_beta_step_strided 83-87; the transposed path 90-94 is
 * served by the same kernel, so both are bit-identical as the reference
 * requires). */
size_t lsk_update_beta_workspace_bytes(int32_t n, int32_t m);
int32_t lsk_update_beta_f32(const float* C, int64_t ldc, int32_t n, int32_t m, const float* alpha,
                            const float* log_mu, double eps, float* beta_out, void* workspace,
                            size_t workspace_bytes, void* stream);

/* err = sum_i |exp(log_mu_i + LSE_j(((a_i + b_j) - C_ij) * inv + log_nu_j)) - mu_i|
 * -- marginal_error, solver.py:179-206 (_marginal_error 97-104). err_out is a
 * device float. Workspace: n floats. */
int32_t lsk_marginal_error_f32(const float* C, int64_t ldc, int32_t n, int32_t m, const float* mu,
                               const float* log_mu, const float* log_nu, const float* alpha,
                               const float* beta, double eps, float* err_out, void* workspace,
                               size_t workspace_bytes, void* stream);

/* cost = sum_ij C_ij * exp(((((a_i + b_j) - C_ij) * inv) + log_mu_i) + log_nu_j)
 * -- transport_cost, solver.py:209-227 (_transport_cost 107-115). Device
 * float out; workspace n floats. */
int32_t lsk_transport_cost_f32(const float* C, int64_t ldc, int32_t n, int32_t m, const float* log_mu,
                               const float* log_nu, const float* alpha, const float* beta, double eps,
                               float* cost_out, void* workspace, size_t workspace_bytes, void* stream);

/* P_ij = exp(same argument as the cost) into P (row stride ldp); counts
 * non-finite rows into *nonfinite_out (device int32, caller zeroes it)
 * -- materialize_plan, solver.py:434-458. */
int32_t lsk_materialize_plan_f32(const float* C, int64_t ldc, int32_t n, int32_t m, const float* log_mu,
                                 const float* log_nu, const float* alpha, const float* beta, double eps,
                                 float* P, int64_t ldp, int32_t* nonfinite_out, void* stream);

/* C_ij = fl32(sum_k (x_ik - y_jk)^2) from fp64 points (n,d)/(m,d), the sum in
 * coordinate order in fp64 -- squared_euclidean_cost, costs.py:36-50 -- then,
 * if normalize_max, divided in fp64 by the exact max (applications.py:186-188)
 * before the single fp32 rounding (solver.py:253). cmax_out: device double,
 * the max before normalisation. Workspace: lsk_build_cost_workspace_bytes(). */
size_t lsk_build_cost_workspace_bytes(void);
int32_t lsk_build_cost_f32(const double* X, const double* Y, int32_t n, int32_t m, int32_t d,
                           int32_t normalize_max, float* C, int64_t ldc, double* cmax_out, void* workspace,
                           size_t workspace_bytes, void* stream);

/* A host (pageable) cost matrix -> the padded device layout dst (row stride
 * ldd floats, zero tail), fp64 sources rounded once to fp32 (solver.py:253) on
 * the host: `threads` workers (0 = all cores) each round a row chunk into their
 * own pinned buffer and copy it asynchronously while rounding the next; the
 * copies are ordered before later work on `stream`. Replaces the pageable
 * cudaMemcpy + device cast of CostMatrix.values (types.py:60-86). Chunks are
 * ~1 MB of fp32 written with non-temporal stores when ldd % 4 == 0; the
 * rounding is bit-identical either way (LSK_H2D_NT=0 / LSK_H2D_CHUNK_KB=<kb>
 * in the environment override both, for experiments). */
int32_t lsk_h2d_cost_f32(const void* src, int32_t src_is_f64, int64_t lds, int32_t n, int32_t m, float* dst,
                         int64_t ldd, int32_t threads, void* stream);

/* The reference composition without materialising C64 on the host:
 * lsk_cost_range_f64 -> range_out[0] = max, range_out[1] = min of the fp64
 * cost (host doubles; CostMatrix.value_range = max - min, types.py:60-86;
 * synchronises `stream`); lsk_build_cost_div_f32 -> C_ij =
 * fl32(fl64(sum_k (x_ik - y_jk)^2) / divisor), divisor 0 = none: the fp32 cast
 * (solver.py:253) of CostMatrix(values=C64 / s) (applications.py:186-188,
 * estimator.py:87-89) bit for bit. */
int32_t lsk_cost_range_f64(const double* X, const double* Y, int32_t n, int32_t m, int32_t d, double* range_out,
                           void* workspace, size_t workspace_bytes, void* stream);
int32_t lsk_build_cost_div_f32(const double* X, const double* Y, int32_t n, int32_t m, int32_t d, double divisor,
                               float* C, int64_t ldc, void* stream);

/* dst = fl32(src) in a zero-padded row-major layout (row stride ldd floats,
 * a multiple of 4 for the solver): the one fp64 -> fp32 cast of the cost
 * matrix (solver.py:253), or a plain fp32 re-pad when src_is_f64 == 0. */
int32_t lsk_cast_cost_f32(const void* src, int32_t src_is_f64, int64_t lds, int32_t n, int32_t m, float* dst,
                          int64_t ldd, void* stream);


/* ---------------------------------------------------------------------------
 * fp64 (precision="double"; half-steps with float64 potentials, solver.py:60-65):
 * the same entry points in double with the reference's double arithmetic
 * (inv_eps = 1.0/eps, separately rounded ops, full-precision exp/log). C is a
 * row-major fp64 matrix (row stride ldc >= m, no alignment needs); all other
 * arrays double except trace_iter/result (int32). The solve is the exact
 * two-pass multi-kernel loop; result_f holds (final error, cost) as doubles. */
size_t lsk_solve_dense_f64_workspace_bytes(int32_t n, int32_t m);
int32_t lsk_solve_dense_f64(const double* C, int64_t ldc, int32_t n, int32_t m, const double* log_mu,
                            const double* log_nu, const double* mu, double eps, double tol, int32_t max_iter,
                            int32_t check_interval, int32_t flags, double* f_out, double* g_out, int32_t* trace_iter,
                            double* trace_err, int32_t* result, double* result_f, void* workspace,
                            size_t workspace_bytes, void* stream);
int32_t lsk_update_alpha_f64(const double* C, int64_t ldc, int32_t n, int32_t m, const double* beta,
                             const double* log_nu, double eps, double* alpha_out, void* stream);
size_t lsk_update_beta_f64_workspace_bytes(int32_t n, int32_t m);
int32_t lsk_update_beta_f64(const double* C, int64_t ldc, int32_t n, int32_t m, const double* alpha,
                            const double* log_mu, double eps, double* beta_out, void* workspace,
                            size_t workspace_bytes, void* stream);
int32_t lsk_marginal_error_f64(const double* C, int64_t ldc, int32_t n, int32_t m, const double* mu,
                               const double* log_mu, const double* log_nu, const double* alpha, const double* beta,
                               double eps, double* err_out, void* workspace, size_t workspace_bytes, void* stream);
int32_t lsk_transport_cost_f64(const double* C, int64_t ldc, int32_t n, int32_t m, const double* log_mu,
                               const double* log_nu, const double* alpha, const double* beta, double eps,
                               double* cost_out, void* workspace, size_t workspace_bytes, void* stream);
int32_t lsk_materialize_plan_f64(const double* C, int64_t ldc, int32_t n, int32_t m, const double* log_mu,
                                 const double* log_nu, const double* alpha, const double* beta, double eps, double* P,
                                 int64_t ldp, int32_t* nonfinite_out, void* stream);

/* ---------------------------------------------------------------------------
 * On-the-fly point-cloud solver (configs C4/C5): the squared-Euclidean cost is
 * recomputed in registers from fp32 points and never stored.
 *
 * Replaces the composition squared_euclidean_cost(X, Y) [/ C.max()] -> solve
 * (costs.py:36-50, applications.py:177-191 / estimator.py:78-99,
 * solver.py:230-337) for B independent problems of the same shape:
 * X (B, n, d) and Y (B, m, d) fp64 (rounded once to fp32 on the device),
 * d in 1..3; cost c_ij = scale[b] * sum_k (x_ik - y_jk)^2 with scale (B floats,
 * device) = 1 or 1/Cmax (lsk_points_cost_max). log_mu/mu (B, n), log_nu (B, m)
 * fp32 device. Same iteration, check, trace and status semantics as
 * lsk_solve_dense_f32, per problem; a problem that stops no longer runs, and
 * the host stops enqueueing once every problem has stopped.
 * Outputs: f_out (B, n), g_out (B, m), trace_iter/trace_err (B, capacity),
 * result (B, 8) int32 (LSK_RES_*), result_f (B, 2) float (final error, cost).
 *
 * comm: NULL, or an lsk_comm_create() communicator of P ranks (B must be 1;
 * SURVEY 8(e)). The design is chosen by the flags:
 *   LSK_FLAG_SHARD_PARTIALS  -- rank r owns a row slab of the source cloud
 *     (whole 2048-point chunks: rows [r R, (r+1) R), R = 2048 L/P with L the
 *     next power of two of ceil(n/2048)); f is local; for g each rank reduces
 *     its rows into per-column partials (stale sums or (max, sumexp) pairs),
 *     the complete subtree of the fixed chunk tree it owns; the P roots are
 *     allgathered and merged by the top of that tree. P must be a power of two
 *     <= L. Bit-identical to one GPU for every such P.
 *   LSK_FLAG_SHARD_ALLREDUCE -- as partials, but the stale sums are combined
 *     by ncclAllReduce(SUM) (NCCL's order: within rounding of one GPU, not
 *     bitwise).
 *   neither -- owner computes: rank r computes f for rows [r ceil(n/P), ...)
 *     and g for columns [r ceil(m/P), ...) against everything; the potential
 *     slabs are allgathered after each half-step. Any P; bit-identical.
 * Every design allgathers f after the f half-step. The sharded workspace is
 * lsk_solve_points_sharded_workspace_bytes(n, m, P, mode).
 * Numerics: fp32 direct-form cost (~2-3e-6 on potentials at
 * eps = 1e-3); use the dense path with lsk_build_cost_f32 below eps = 1e-3.
 */
#define LSK_FLAG_SHARD_PARTIALS 128
#define LSK_FLAG_SHARD_ALLREDUCE 256
/* CUDA graphs: after the first checkpoint the iteration loop is captured as
 * blocks of check_interval iterations and replayed (single-GPU, batched and
 * emulated solves, when there are >= 3 blocks and the caller is not already
 * capturing the stream). LSK_FLAG_NO_GRAPH enqueues every iteration;
 * LSK_FLAG_GRAPH_NCCL also captures the NCCL collectives of a sharded solve
 * (opt-in: not validated on a multi-GPU box by this build). */
#define LSK_FLAG_NO_GRAPH 1024
#define LSK_FLAG_GRAPH_NCCL 2048
#define LSK_SHARD_NONE 0
#define LSK_SHARD_OWNER 1
#define LSK_SHARD_PARTIALS 2
#define LSK_SHARD_ALLREDUCE 3
#define LSK_EMU_MAX_RANKS 16
size_t lsk_solve_points_workspace_bytes(int32_t B, int32_t n, int32_t m);
size_t lsk_solve_points_sharded_workspace_bytes(int32_t n, int32_t m, int32_t P, int32_t shard_mode);
int32_t lsk_solve_points_f32(const double* X, const double* Y, int32_t B, int32_t n, int32_t m, int32_t d,
                             const float* scale, const float* log_mu, const float* log_nu, const float* mu,
                             double eps, double tol, int32_t max_iter, int32_t check_interval, int32_t flags,
                             float* f_out, float* g_out, int32_t* trace_iter, float* trace_err, int32_t* result,
                             float* result_f, void* workspace, size_t workspace_bytes, void* comm, void* stream);

/* Single-GPU emulation of the P-rank decomposition (test hook; B = 1): the P
 * ranks' kernels run rank after rank on `stream`, each rank in its own slice
 * of the workspace (P x lsk_solve_points_sharded_workspace_bytes), and the
 * collectives become device copies (the allreduce a rank-order sum). Outputs
 * are rank 0's; *rank_mismatch (device int) counts ranks whose returned
 * potentials, status, iterations, error or cost differ in any bit from rank
 * 0's. shard_mode: LSK_SHARD_OWNER / _PARTIALS / _ALLREDUCE (P in 1..16), or
 * LSK_SHARD_NONE with P = 1. */
int32_t lsk_solve_points_emulated_f32(const double* X, const double* Y, int32_t n, int32_t m, int32_t d,
                                      const float* scale, const float* log_mu, const float* log_nu, const float* mu,
                                      double eps, double tol, int32_t max_iter, int32_t check_interval, int32_t flags,
                                      int32_t P, int32_t shard_mode, float* f_out, float* g_out, int32_t* trace_iter,
                                      float* trace_err, int32_t* result, float* result_f, int32_t* rank_mismatch,
                                      void* workspace, size_t workspace_bytes, void* stream);

/* Plan consumers without the plan (f, g from a solve; pi_ij as in
 * materialize_plan): mapped_out (B, n, d) = sum_j pi_ij y_j / sum_j pi_ij --
 * barycentric_map, applications.py:75-97 (*zero_rows counts rows with no
 * mass: ZeroRowMass); match_idx (B, n) = argmax_j pi_ij with the lowest j on
 * ties and match_w = that pi_ij -- the correspondences of
 * match_point_clouds, applications.py:195-204. Same cost/scale convention as
 * lsk_solve_points_f32. */
size_t lsk_points_consume_workspace_bytes(int32_t B, int32_t n, int32_t m);
int32_t lsk_points_consume_f32(const double* X, const double* Y, int32_t B, int32_t n, int32_t m, int32_t d,
                               const float* scale, const float* f, const float* g, const float* log_mu,
                               const float* log_nu, double eps, float* mapped_out, int32_t* match_idx,
                               float* match_w, int32_t* zero_rows, void* workspace, size_t workspace_bytes,
                               void* stream);

/* cmax_out[b] = max_ij sum_k (x_ik - y_jk)^2 in fp64 (device doubles), the
 * C.max() normaliser of applications.py:186-188, without materialising C
 * (fp32 screen of all pairs, exact fp64 re-evaluation of the near-maximal
 * ones; d in 1..3). */
size_t lsk_points_cost_max_workspace_bytes(int32_t B, int32_t n, int32_t m);
int32_t lsk_points_cost_max(const double* X, const double* Y, int32_t B, int32_t n, int32_t m, int32_t d,
                            double* cmax_out, void* workspace, size_t workspace_bytes, void* stream);

/* range_out (B, 2) device doubles: exact fp64 max and min of the cost per
 * problem (value_range = max - min, types.py:60-86: the pipelines divide by
 * C.max() only when it is > 0, applications.py:186-188). */
size_t lsk_points_cost_range_workspace_bytes(int32_t B, int32_t n, int32_t m);
int32_t lsk_points_cost_range(const double* X, const double* Y, int32_t B, int32_t n, int32_t m, int32_t d,
                              double* range_out, void* workspace, size_t workspace_bytes, void* stream);

/* NCCL communicator for the sharded points solve (one rank per GPU): rank 0
 * gets an id (lsk_nccl_unique_id_bytes() bytes), every rank passes it to
 * lsk_comm_create with its own device current. */
int32_t lsk_nccl_unique_id_bytes(void);
int32_t lsk_nccl_unique_id(void* id_out);
int32_t lsk_comm_create(const void* id, int32_t nranks, int32_t rank, void** comm_out);
int32_t lsk_comm_destroy(void* comm);

/* ---- colour-transfer pipeline, fp64 (applications.py:100-161)
 * Replaces: squared_euclidean_cost (costs.py:36-50) in double for the pipeline's
 * samples; materialize_plan + barycentric_map (solver.py:434-458,
 * applications.py:75-97) without the plan; the nearest-sample recolour loop
 * (applications.py:149-155). lsk_build_cost_f64 takes the arguments of
 * lsk_build_cost_f32 (normalize_max: C / C.max() when the range is non-zero,
 * estimator.py:87-89; workspace lsk_build_cost_workspace_bytes()). In the
 * barycentric map div != 0 divides every recomputed cost by div. flags[0] += rows with a non-finite plan entry
 * (NonFiniteResult), flags[1] += rows with zero mass (ZeroRowMass); flags is
 * caller-zeroed int32[2]. Recolour: RGB (3 doubles per pixel/sample), ties to
 * the lowest sample index, output clamped to [0, 1]; nearest may be NULL. */
int32_t lsk_build_cost_f64(const double* X, const double* Y, int32_t n, int32_t m, int32_t d, int32_t normalize_max,
                           double* C, int64_t ldc, double* cmax_out, void* workspace, size_t workspace_bytes,
                           void* stream);
int32_t lsk_barycentric_points_f64(const double* X, const double* Y, const double* T, int32_t n, int32_t m,
                                   int32_t d, int32_t dt, double div, const double* log_mu, const double* log_nu,
                                   const double* alpha, const double* beta, double eps, double* mapped,
                                   int32_t* flags, void* stream);
int32_t lsk_recolor_nearest_f64(const double* pixels, int64_t n_pixels, const double* samples, int32_t n_samples,
                                const double* mapped, double* out, int32_t* nearest, void* stream);
/* barycentric_map of a materialised (n, m) fp64 plan (applications.py:75-97);
 * flags[1] += zero-mass rows (ZeroRowMass); dt in 1..4. */
int32_t lsk_barycentric_plan_f64(const double* P, int64_t ldp, int32_t n, int32_t m, const double* T, int32_t dt,
                                 double* mapped, int32_t* flags, void* stream);
/* General nearest-sample map (SinkhornTransport.transform, estimator.py:118-132):
 * out[q] = mapped[argmin_s |x_q - s|^2] for d = dm in 1..4, optional clamp. */
int32_t lsk_nearest_map_f64(const double* queries, int64_t n_queries, int32_t d, const double* samples,
                            int32_t n_samples, const double* mapped, int32_t dm, int32_t clamp01, double* out,
                            int32_t* nearest, void* stream);

/* ---- the reference's deterministic reductions (reduction.py)
 * op: 0 max, 1 sum, 2 log-sum-exp; dtype: 0 float32, 1 float64. Rows: A is (R, L)
 * with row stride lda, one result per row. Cols: A is (L, R) with row stride lda,
 * one result per column. The ReductionPlan tree (lane fold over group_size lanes,
 * ceil-halving within chunk_width chunks, then across chunks) is replicated
 * exactly: max and sum are bit-identical to the reference; LSE (workspace
 * lsk_reduce_workspace_bytes(R, dtype)) matches to the exponential's ulps.
 * group_size <= 4096 (rows), <= 200 KB / (32 * sizeof) (cols). */
size_t lsk_reduce_workspace_bytes(int32_t R, int32_t dtype);
int32_t lsk_reduce_rows(const void* A, int64_t lda, int32_t R, int32_t L, int32_t dtype, int32_t op,
                        int32_t chunk_width, int32_t group_size, void* out, void* workspace, size_t workspace_bytes,
                        void* stream);
int32_t lsk_reduce_cols(const void* A, int64_t lda, int32_t L, int32_t R, int32_t dtype, int32_t op,
                        int32_t chunk_width, int32_t group_size, void* out, void* workspace, size_t workspace_bytes,
                        void* stream);

/* ---- plan diagnostics (solver.py:461-519)
 * lsk_kkt_residual: out_max = max |C + eps log(P/(mu nu)) - alpha - beta| over
 * P >= tiny(dtype) (0 if none), out_count[0] = masked entries, out_count[1] = 1
 * if a masked residual was NaN; C, P, mu, nu, alpha, beta in dtype (0 f32,
 * 1 f64), C and P with the same row stride ld; workspace 16 bytes.
 * lsk_regularized_objective_f64: <C,P> + eps (sum P (log(P/(mu nu)) - 1) + 1),
 * zero entries contributing 0; workspace 16 n bytes. */
int32_t lsk_kkt_residual(const void* C, const void* P, int64_t ld, int32_t n, int32_t m, const void* mu,
                         const void* nu, const void* alpha, const void* beta, double eps, int32_t dtype,
                         double* out_max, int32_t* out_count, void* workspace, size_t workspace_bytes, void* stream);
int32_t lsk_regularized_objective_f64(const double* C, const double* P, int64_t ld, int32_t n, int32_t m,
                                      const double* mu, const double* nu, double eps, double* out, void* workspace,
                                      size_t workspace_bytes, void* stream);

/* ---- standard-domain solve (solver.py:340-431)
 * K = exp(-C/eps) in the workspace, u = mu/(K v), v = nu/(K^T u) from ones,
 * checks / trace / cost as lsk_solve_dense_f32 (result[0..2], result_f[0..1]);
 * mu, nu are the WEIGHTS (not logs). Unguarded by design: non-finite values
 * surface as status 2 at the next checkpoint. */
size_t lsk_solve_standard_workspace_bytes(int32_t n, int32_t m, int32_t double_precision);
int32_t lsk_solve_standard_f32(const float* C, int64_t ldc, int32_t n, int32_t m, const float* mu, const float* nu,
                               double eps, double tol, int32_t max_iter, int32_t check, int32_t flags, float* u_out,
                               float* v_out, int32_t* trace_iter, float* trace_err, int32_t* result, float* result_f,
                               void* workspace, size_t workspace_bytes, void* stream);
int32_t lsk_solve_standard_f64(const double* C, int64_t ldc, int32_t n, int32_t m, const double* mu,
                               const double* nu, double eps, double tol, int32_t max_iter, int32_t check,
                               int32_t flags, double* u_out, double* v_out, int32_t* trace_iter, double* trace_err,
                               int32_t* result, double* result_f, void* workspace, size_t workspace_bytes,
                               void* stream);

#ifdef __cplusplus
}
#endif
#endif /* LSK_H */
