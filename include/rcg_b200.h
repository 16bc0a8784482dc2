/*
 * rcg_b200.h -- C-ABI of the B200-native deflated-ICCG hot path (librcg_b200.so).
 *
 * Plain pointers and sizes only; no torch or CUDA types in the signatures.  Every vector
 * argument may be a HOST pointer (pageable or pinned; the call stages it through HBM) or a
 * DEVICE pointer on the context's GPU (used in place) -- the library inspects the pointer.
 *
 * Each entry point names the reference declaration it replaces (paths relative to
 * /root/reference/proj/include/recycg).  Status codes map 1:1 onto the reference's exception
 * types so a C++ or ctypes binding can rethrow them:
 *   RCG_E_INVALID   -> std::invalid_argument   (config / size errors)
 *   RCG_E_BREAKDOWN -> recycg::BreakdownError  (non-SPD, pivot failure, W^T A W not SPD)
 *   RCG_E_PARSE     -> recycg::ParseError      (CSR validation failure)
 *   RCG_E_CUDA      -> runtime error           (no GPU, CUDA fault, out of device memory)
 * There is no CPU fallback: without a usable sm_100 device every compute call returns RCG_E_CUDA.
 */
#ifndef RCG_B200_H
#define RCG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RCG_OK 0
#define RCG_E_INVALID 1
#define RCG_E_BREAKDOWN 2
#define RCG_E_PARSE 3
#define RCG_E_CUDA 4

typedef struct rcg_ctx rcg_ctx;         /* one GPU, one stream, workspaces */
typedef struct rcg_matrix rcg_matrix;   /* device CSR (CsrMatrix) */
typedef struct rcg_ic rcg_ic;           /* device IC(0) factor + sweep schedules (IcFactor) */
typedef struct rcg_tall rcg_tall;       /* device n x k column block (TallDense) */
typedef struct rcg_basis rcg_basis;     /* W, AW, chol(W^T A W) (DeflationOperator / SC state) */
typedef struct rcg_sampler rcg_sampler; /* device snapshot slots (SamplerState) */
typedef struct rcg_dslab rcg_dslab;     /* one GPU's row slab of a multi-GPU solve */
typedef struct rcg_comm rcg_comm;       /* slab transport: NCCL (one slab per process) or loopback */
typedef struct rcg_dbasis rcg_dbasis;   /* row-partitioned W, AW + replicated chol(W^T A W) */
typedef struct rcg_seq rcg_seq;         /* prepared sequence: scaled A, D^-1/2, IC(0) (run_sequence) */

/* message of the last failing call on this thread; "" after success */
const char* rcg_last_error(void);
const char* rcg_build_info(void);

/* ------------------------------------------------------------------ context */
int rcg_ctx_create(int device, rcg_ctx** out);
void rcg_ctx_destroy(rcg_ctx* ctx);
int rcg_ctx_synchronize(rcg_ctx* ctx);
/* number of kernels this context has launched (for gpu_launches accounting) */
int64_t rcg_ctx_launch_count(const rcg_ctx* ctx);
/* device time (ms) accumulated by the named kernel class since the last reset, measured with
 * CUDA events on the context stream when profiling is enabled (class: 0 spmv, 1 fwd sweep,
 * 2 bwd sweep, 3 vector ops, 4 projection; 5-9 the same for batched multi-RHS solves, whose
 * launches each carry RT right-hand sides -- rcg_ctx_kernel_units returns the sum of RT over a
 * class's launches).  Used by bench.py for the roofline. */
int rcg_ctx_set_profiling(rcg_ctx* ctx, int enable);
/* which kernel classes are timed while profiling (bit c = class c; default all): timing a subset
 * keeps the event overhead out of a timed region */
int rcg_ctx_set_profiling_mask(rcg_ctx* ctx, unsigned mask);
/* CUDA events on the context stream (slots 0..15) for device-side timing by callers */
int rcg_ctx_event_record(rcg_ctx* ctx, int slot);
int rcg_ctx_event_elapsed(rcg_ctx* ctx, int slot_a, int slot_b, double* ms);
int rcg_ctx_kernel_stats(rcg_ctx* ctx, int cls, double* total_ms, int64_t* launches);
int rcg_ctx_kernel_units(rcg_ctx* ctx, int cls, int64_t* units);
void rcg_ctx_reset_stats(rcg_ctx* ctx);
/* IC sweep kernel selection (no effect on results: every variant is bitwise identical):
 * 0 = grid-wide sync-free sweep (k_sweep), 2 = default (one launch per level -- icsweep_lv.cu --
 * when the average level holds >= 600K rows, else k_sweep), 4 = one launch per level always;
 * RCG_SWEEP_CLUSTER overrides at context creation */
int rcg_ctx_set_sweep_kernel(rcg_ctx* ctx, int mode);

/* ------------------------------------------------------------------ CSR (csr_matrix.hpp) */
/* CsrMatrix(n, row_start, col_idx, values) -- csr_matrix.hpp:28-30.  validate != 0 runs the
 * reference invariants of CsrMatrix::validate (csr_matrix.cpp:36-87) on the host arrays and
 * returns RCG_E_PARSE with the reference message on failure. */
int rcg_matrix_create(rcg_ctx* ctx, int32_t n, const int32_t* row_start, const int32_t* col_idx,
                      const double* values, int validate, rcg_matrix** out);
void rcg_matrix_destroy(rcg_matrix* a);
int32_t rcg_matrix_n(const rcg_matrix* a);
int64_t rcg_matrix_nnz(const rcg_matrix* a);
int rcg_matrix_values(rcg_ctx* ctx, const rcg_matrix* a, double* values_out);
/* spmv(a, x, y) -- csr_matrix.hpp:54; bitwise equal to the reference (sequential row sums) */
int rcg_spmv(rcg_ctx* ctx, const rcg_matrix* a, const double* x, double* y);
/* spmv_dual(a, x1, x2, y1, y2) -- csr_matrix.hpp:56-59; each output bitwise equal to rcg_spmv */
int rcg_spmv_dual(rcg_ctx* ctx, const rcg_matrix* a, const double* x1, const double* x2,
                  double* y1, double* y2);
/* diagonal_scale(a) -- scaling.hpp:24-26: returns the scaled matrix and d_inv_sqrt (length n) */
int rcg_diagonal_scale(rcg_ctx* ctx, const rcg_matrix* a, rcg_matrix** scaled, double* d_inv_sqrt);

/* ------------------------------------------------------------------ IC(0) (ic_preconditioner.hpp) */
/* ic0_factorize(a, shift, num_blocks) -- ic_preconditioner.hpp:44: zero-fill L D L^T with the
 * reference shift ladder from CSR arrays (host or device): rcg_ic0_factorize_device over a
 * temporary device copy of the matrix. */
int rcg_ic0_factorize(rcg_ctx* ctx, int32_t n, const int32_t* row_start, const int32_t* col_idx,
                      const double* values, double shift, int num_blocks, rcg_ic** out);
/* ic0_factorize on the device (ic_preconditioner.cpp:12-121): pattern work (L / U
 * patterns, Kahn levels, level schedules) by device kernels, the numeric row merge + shift ladder
 * by a level-ordered sync-free kernel; the factor is bitwise the reference's. */
int rcg_ic0_factorize_device(rcg_ctx* ctx, const rcg_matrix* a, double shift, int num_blocks, rcg_ic** out);
/* upload an existing IcFactor (ic_preconditioner.hpp:18-37) so the operator is identical */
int rcg_ic_create(rcg_ctx* ctx, int32_t n, int num_blocks, const int32_t* block_bounds,
                  const int32_t* l_row_start, const int32_t* l_col, const double* l_val,
                  const double* d, const int32_t* u_row_start, const int32_t* u_col,
                  const double* u_val, double shift_used, rcg_ic** out);
void rcg_ic_destroy(rcg_ic* f);
/* factor metadata: nnz of L, shift used, forward/backward level counts */
int rcg_ic_info(const rcg_ic* f, int64_t* nnz_l, double* shift_used, int32_t* fwd_levels,
                int32_t* bwd_levels);
/* copy the host image of the factor out (arrays sized n+1 / nnz_l / n) */
int rcg_ic_export(const rcg_ic* f, int32_t* block_bounds, int32_t* l_row_start, int32_t* l_col,
                  double* l_val, double* d, int32_t* u_row_start, int32_t* u_col, double* u_val);
/* ic_apply(f, r, z) -- ic_preconditioner.hpp:47; bitwise equal to the reference */
int rcg_ic_apply(rcg_ctx* ctx, const rcg_ic* f, const double* r, double* z);

/* ------------------------------------------------------------------ TallDense (dense.hpp) */
int rcg_tall_create(rcg_ctx* ctx, int32_t n, int k, const double* cols, rcg_tall** out);
void rcg_tall_destroy(rcg_tall* t);
int rcg_tall_k(const rcg_tall* t);
int32_t rcg_tall_n(const rcg_tall* t);
/* column-major n x k, leading dimension n */
int rcg_tall_download(rcg_ctx* ctx, const rcg_tall* t, double* cols_out);
/* a TallDense held as k separate columns (host or device pointers, each of length n) -- the
 * reference's std::vector<Vector> layout (dense.hpp:11-22), no host-side packing needed */
int rcg_tall_create_cols(rcg_ctx* ctx, int32_t n, int k, const double* const* cols, rcg_tall** out);
/* mgs_orthonormalize(v, drop_tol) -- dense.hpp:50 */
int rcg_mgs_orthonormalize(rcg_ctx* ctx, const rcg_tall* v, double drop_tol, rcg_tall** out);

/* ------------------------------------------------------------------ samplers (sampling.hpp) */
#define RCG_SAMPLER_A 0
#define RCG_SAMPLER_B 1
/* SamplerState::method_a(m, cap) / method_b(m, eps) -- sampling.hpp:30-34 (slots of length n) */
int rcg_sampler_create(rcg_ctx* ctx, int method, int m, int iteration_cap, double eps, int32_t n,
                       rcg_sampler** out);
void rcg_sampler_destroy(rcg_sampler* s);
/* SamplerState::offer -- sampling.hpp:37 (host-driven offer of an arbitrary payload) */
int rcg_sampler_offer(rcg_ctx* ctx, rcg_sampler* s, int iteration, double relres,
                      const double* payload);
/* occupied()/stored_iteration() for all m slots; stored_count() returned */
int rcg_sampler_state(const rcg_sampler* s, int* occupied, int* stored_iter);
int rcg_sampler_slot(rcg_ctx* ctx, const rcg_sampler* s, int slot, double* out);

/* ------------------------------------------------------------------ recycling (recycling.hpp) */
/* harvest_errors(x_final, s) -- recycling.hpp:19 */
int rcg_harvest_errors(rcg_ctx* ctx, const double* x_final, const rcg_sampler* s, rcg_tall** out);
/* harvest_errors(x_final, s) -- recycling.hpp:19 -- for snapshots the caller holds: slots = the
 * k occupied slots of a host SamplerState in slot order (sampling.hpp:39-44); exactly-zero
 * differences are skipped (recycling.cpp:26) */
int rcg_harvest_columns(rcg_ctx* ctx, const double* x_final, int32_t n, int k, const double* const* slots,
                        rcg_tall** out);
/* harvest_stored(s) -- recycling.hpp:23 */
int rcg_harvest_stored(rcg_ctx* ctx, const rcg_sampler* s, rcg_tall** out);
/* rayleigh_ritz(a, e) -- recycling.hpp:38: values (k, host) and optional Ritz vectors */
int rcg_rayleigh_ritz(rcg_ctx* ctx, const rcg_matrix* a, const rcg_tall* e, double* values,
                      rcg_tall** vectors);
/* build_aux_matrix(a, errors, theta) -- recycling.hpp:47.  keep_count > 0 replaces theta by the
 * midpoint between the keep_count-th and (keep_count+1)-th Ritz values (all kept if fewer);
 * the chosen threshold is written to *theta_used.  values must hold errors->k doubles. */
int rcg_build_aux_matrix(rcg_ctx* ctx, const rcg_matrix* a, const rcg_tall* errors, double theta,
                         int keep_count, int* m_bar, double* values, double* theta_used,
                         rcg_tall** w);

/* ------------------------------------------------------------------ W basis */
#define RCG_BASIS_DEFLATION 0 /* build_deflation_operator -- deflation.hpp:37 */
#define RCG_BASIS_SC 1        /* ScPreconditioner ctor   -- subspace_correction.hpp:24-25 */
int rcg_basis_create(rcg_ctx* ctx, const rcg_matrix* a, const rcg_tall* w, int who, rcg_basis** out);
void rcg_basis_destroy(rcg_basis* b);
int rcg_basis_k(const rcg_basis* b);
/* a basis from the fields of an existing DeflationOperator / ScPreconditioner exactly as they are
 * (W and AW as k host or device columns of length n, chol(W^T A W) row-major k x k): the operator
 * that object applies, nothing recomputed */
int rcg_basis_create_from(rcg_ctx* ctx, int32_t n, int k, const double* const* w_cols, const double* const* aw_cols,
                          const double* chol_l, int who, rcg_basis** out);
/* the host fields of DeflationOperator / ScPreconditioner (deflation.hpp:18-20,
 * subspace_correction.hpp:31-36): AW column-major with leading dimension n (n * k doubles) and
 * chol(W^T A W) row-major k x k (SmallChol::l); either may be NULL */
int rcg_basis_export(rcg_ctx* ctx, const rcg_basis* b, double* aw_cols, double* chol_l);
/* DeflationOperator::project_pt / project_p / direct_component -- deflation.hpp:24-32 */
int rcg_project_pt(rcg_ctx* ctx, const rcg_basis* b, const double* y, double* out);
int rcg_project_p(rcg_ctx* ctx, const rcg_basis* b, const double* x, double* out);
int rcg_direct_component(rcg_ctx* ctx, const rcg_basis* b, const double* rhs, double* out);

/* ------------------------------------------------------------------ Krylov solvers (pcg.hpp) */
typedef struct {
    double eps;         /* SolverConfig::eps, in (0,1) */
    int max_iter;       /* SolverConfig::max_iter, >= 1 */
    int record_history; /* SolverConfig::record_history */
} rcg_solver_config;

typedef struct {
    int iterations;
    int converged;
    double wall_time;   /* seconds around the iteration loop (device events); a batched solve
                         * reports the batch's time divided by its right-hand sides */
    int cap;            /* capacity of the optional host arrays below */
    double* history;    /* relres per iteration (SolveReport::history) */
    double* alphas;     /* CG alpha_i per iteration (Lanczos input), optional */
    double* betas;      /* CG beta_i per iteration, 0 at i = 1, optional */
} rcg_solve_report;

#define RCG_PREC_IDENTITY 0 /* IdentityPreconditioner -- preconditioner.hpp:23 */
#define RCG_PREC_IC 1       /* IcPreconditioner       -- ic_preconditioner.hpp:51 */
#define RCG_PREC_SC 2       /* ScPreconditioner       -- subspace_correction.hpp:22 (inner = ic or identity) */
typedef struct {
    int kind;
    const rcg_ic* ic;
    const rcg_basis* sc;
} rcg_prec;

/* Preconditioner::apply(r, z) -- preconditioner.hpp:13 -- on the device: IcPreconditioner
 * (ic_apply, bitwise) or ScPreconditioner::apply (subspace_correction.cpp:47-57: inner, then
 * z += W chol(W^T r)); an identity preconditioner needs no call (z = r) */
int rcg_prec_apply(rcg_ctx* ctx, const rcg_prec* m, const double* r, double* z);

#define RCG_PAYLOAD_X 0 /* error_sampling_observer    -- sampling.hpp:67 */
#define RCG_PAYLOAD_R 1 /* residual_sampling_observer -- sampling.hpp:70 */

/* pcg_solve(a, b, m, x, cfg, observer) -- pcg.hpp:39-41.  observer: NULL or a sampler fed the
 * iterate (payload RCG_PAYLOAD_X) or residual (RCG_PAYLOAD_R) of each continuing iteration. */
int rcg_pcg_solve(rcg_ctx* ctx, const rcg_matrix* a, const double* b, const rcg_prec* m, double* x,
                  const rcg_solver_config* cfg, rcg_sampler* observer, int payload,
                  rcg_solve_report* rep);
/* deflated_pcg_solve(a, b, m, defl, x, cfg) -- pcg.hpp:50-52; defl NULL = empty W */
int rcg_deflated_pcg_solve(rcg_ctx* ctx, const rcg_matrix* a, const double* b, const rcg_prec* m,
                           const rcg_basis* defl, double* x, const rcg_solver_config* cfg,
                           rcg_solve_report* rep);

/* Batched independent solves (the sequence's solves 2..k, driver.cpp:181-195): nrhs <= 24
 * right-hand sides of one matrix run through ONE kernel sequence.  B and X hold nrhs vectors
 * of length n back to back (B + k*n is right-hand side k).  Each rhs keeps its own scalars,
 * convergence flag and report; results equal separate solves up to reduction order. */
int rcg_pcg_solve_batch(rcg_ctx* ctx, const rcg_matrix* a, const double* B, const rcg_prec* m, double* X,
                        const rcg_solver_config* cfg, int nrhs, rcg_solve_report* reps);
int rcg_deflated_pcg_solve_batch(rcg_ctx* ctx, const rcg_matrix* a, const double* B, const rcg_prec* m,
                                 const rcg_basis* defl, double* X, const rcg_solver_config* cfg, int nrhs,
                                 rcg_solve_report* reps);

/* ------------------------------------------------------------------ condest (condest.hpp) */
typedef struct {
    double lambda_max;
    double lambda_min;
    double kappa;
    int power_iterations;
    int power_unsettled;
    int lambda_min_available;
    int nritz;
    double* ritz_values;   /* caller buffer of >= m_samples doubles, optional */
    /* Lanczos tridiagonal estimate from the CG alpha/beta (no reference counterpart):
     * extreme eigenvalues of T estimate the spectrum of M^-1 A */
    double lanczos_lambda_min;
    double lanczos_lambda_max;
    double lanczos_kappa;
} rcg_cond_estimate;
/* pcg_with_condest(a, b, m, x, cfg, m_samples, v0_seed) -- condest.hpp:46-48 */
int rcg_pcg_with_condest(rcg_ctx* ctx, const rcg_matrix* a, const double* b, const rcg_prec* m,
                         double* x, const rcg_solver_config* cfg, int m_samples, uint64_t v0_seed,
                         rcg_solve_report* rep, rcg_cond_estimate* est);
/* Lanczos extremes from k alpha/beta pairs (host arithmetic, shared by every solver) */
int rcg_lanczos_extremes(int k, const double* alphas, const double* betas, double* lambda_min,
                         double* lambda_max);

/* ------------------------------------------------------------------ host generators
 * Seeded synthetic inputs shared by the GPU path, the oracle harness and bench.py (the
 * reference ships none).  Arrays are malloc'ed by the library; free with rcg_host_free. */
#define RCG_GEN_POISSON7 0   /* C1: 7-pt, diag 6, off -1, Dirichlet eliminated */
#define RCG_GEN_FV7_CONTRAST 1 /* C2/C4: 7-pt FV, harmonic faces, cube inclusions */
#define RCG_GEN_Q1_27PT 2    /* C3: trilinear hex stiffness, log-normal element coefficient */
#define RCG_GEN_KNN 3        /* C5: symmetric kNN graph Laplacian + shift */
typedef struct {
    int kind;
    int32_t grid;        /* N (stencils) or number of points (kNN) */
    int inclusions;      /* FV: number of cubes */
    int inclusion_size;  /* FV: cube edge in cells */
    double contrast;     /* FV: inclusion coefficient */
    double sigma;        /* Q1: std-dev of log coefficient */
    int knn_k;           /* kNN: neighbours per point */
    uint64_t seed;
} rcg_gen_params;
int rcg_generate(const rcg_gen_params* p, int32_t* n, int64_t* nnz, int32_t** row_start,
                 int32_t** col_idx, double** values);
/* every kind assembled directly in HBM, bitwise the host generator's CSR (
 * replaces the host assembly that feeds parse_matrix_market-style ingest, matrix_market.cpp:30-117):
 * POISSON7 / FV7_CONTRAST with no host arrays; Q1_27PT from the host's seeded element
 * coefficients ((N+1)^3 doubles); KNN from the host's seeded points (exact kNN search, symmetric
 * union and weights on the device; k <= 32) */
int rcg_matrix_generate(rcg_ctx* ctx, const rcg_gen_params* p, rcg_matrix** out);
/* the device matrix back to host arrays (row_start n + 1, col_idx / values nnz; any null skipped) */
int rcg_matrix_export(rcg_ctx* ctx, const rcg_matrix* a, int32_t* row_start, int32_t* col_idx, double* values);
/* UniformPm1 stream (rng.hpp:18-41): draws [skip, skip+n) of seed into out */
void rcg_uniform_pm1(uint64_t seed, uint64_t skip, int64_t n, double* out);
/* N(0,1) by Box-Muller over the same mt19937_64 stream (2 draws per pair) */
void rcg_normal(uint64_t seed, uint64_t skip, int64_t n, double* out);
void rcg_host_free(void* p);
/* IC(0) level depth of the natural ordering (diagnostics) */
int rcg_level_depth(int32_t n, const int32_t* row_start, const int32_t* col_idx, int32_t* depth);
/* Multicolour variant (a different operator, reported separately): greedy
 * colouring in natural order (red-black for 7-point, 8 colours for 27-point) and the symmetric
 * permutation P A P^T with ascending columns.  IC(0) of the permuted matrix has ncolors levels. */
int rcg_multicolor_order(int32_t n, const int32_t* row_start, const int32_t* col_idx, int32_t* new_of_old,
                         int32_t* ncolors);
int rcg_permute_symmetric(int32_t n, const int32_t* row_start, const int32_t* col_idx, const double* values,
                          const int32_t* new_of_old, int32_t** row_start_out, int32_t** col_idx_out,
                          double** values_out);

/* ------------------------------------------------------------------ multi-GPU row slabs
 * The reference has no distributed solver; its block-Jacobi IC(0) (ic0_factorize(a, s, G),
 * ic_preconditioner.cpp:97-121, bounds floor(b n / G)) is the operator the slabs apply: rank b
 * owns rows [floor(b n/G), floor((b+1) n/G)), factorises its diagonal block (no communication in
 * the preconditioner), and exchanges halo values of p (and of x once) before each SpMV; the three
 * dot products of an iteration are summed over ranks (NCCL allreduce), so every rank holds the
 * same scalars and stops at the same iteration.  A symmetric sparsity pattern is assumed (the
 * reference matrices are SPD): what rank q needs from rank b is b's rows with a column in q's
 * range. */
typedef struct {
    int32_t row_begin, row_end;  /* global rows of this slab */
    int32_t nloc, nhalo;         /* local rows, halo columns */
    int64_t nnz;                 /* local entries */
    int32_t* row_start;          /* nloc + 1 */
    int32_t* col_idx;            /* local columns: [0, nloc) own rows, nloc + h = halo_global[h] */
    double* values;
    int32_t* halo_global;        /* nhalo, ascending (so grouped by owning slab) */
    int32_t* recv_count;         /* nparts: halo values received from each slab */
    int32_t* send_count;         /* nparts: values sent to each slab */
    int32_t* send_idx;           /* sum(send_count) local rows, grouped by destination, ascending */
    int nparts, part;
} rcg_slab_plan;
/* host: the slab `part` of `nparts` of a global CSR (arrays malloc'ed; rcg_slab_plan_free) */
int rcg_slab_plan_create(int32_t n, const int32_t* row_start, const int32_t* col_idx, const double* values,
                         int nparts, int part, rcg_slab_plan* out);
void rcg_slab_plan_free(rcg_slab_plan* plan);
/* device slab on ctx's GPU/stream; ic (the slab's diagonal-block factor) may be null = identity */
int rcg_dslab_create(rcg_ctx* ctx, const rcg_slab_plan* plan, const rcg_ic* ic, rcg_dslab** out);
void rcg_dslab_destroy(rcg_dslab* s);
/* NCCL transport, one slab per process: id = 128-byte ncclUniqueId made by rank 0
 * (rcg_comm_nccl_unique_id) and broadcast by the caller.  libnccl is resolved at run time (the
 * copy the process already loaded, else libnccl.so.2). */
int rcg_comm_nccl_unique_id(void* id128);
int rcg_comm_create_nccl(const void* id128, int nranks, int rank, rcg_comm** out);
/* loopback transport: all nparts slabs in this process on one GPU (stream-ordered device copies
 * and a fixed-order sum; slabs never wait on each other inside a kernel) -- tests the distributed
 * iteration on one GPU */
int rcg_comm_create_loopback(int nparts, rcg_comm** out);
/* A host-staged transport over caller-supplied collectives (e.g. torch.distributed / gloo), one
 * slab per process: allreduce sums buf[0..count) over the ranks in place (identical result on every
 * rank); exchange sends send[send_off[q] .. + send_cnt[q]) to rank q and receives
 * recv[recv_off[q] .. + recv_cnt[q]) from rank q, for every q with a nonzero count.  Both return 0
 * on success.  Each collective synchronises the slab's stream (no kernel ever waits on another
 * rank), so ranks may share a GPU -- the multi-process test transport of the NCCL path's
 * iteration. */
typedef int (*rcg_host_allreduce_fn)(void* user, double* buf, int count);
typedef int (*rcg_host_exchange_fn)(void* user, const double* send, const int64_t* send_off,
                                    const int64_t* send_cnt, double* recv, const int64_t* recv_off,
                                    const int64_t* recv_cnt, int nranks);
int rcg_comm_create_host(int nranks, int rank, rcg_host_allreduce_fn allreduce,
                         rcg_host_exchange_fn exchange, void* user, rcg_comm** out);
void rcg_comm_destroy(rcg_comm* c);
/* distributed PCG (pcg.cpp:37-92 per rank with block-Jacobi IC or identity): nslabs = 1 with
 * NCCL, = nparts with loopback; b[s], x[s] are slab s's local rows (host or device) */
int rcg_dist_pcg_solve(rcg_comm* comm, int nslabs, rcg_dslab* const* slabs, const double* const* b,
                       double* const* x, const rcg_solver_config* cfg, rcg_solve_report* report);
/* build_deflation_operator / ScPreconditioner state over slabs (deflation.cpp:45-76): w[s] = slab
 * s's rows of W (column-major nloc x m); AW by halo exchange + local SpMV, the Gram allreduced
 * and factored identically on every rank.  kind: RCG_BASIS_DEFLATION or RCG_BASIS_SC. */
int rcg_dbasis_create(rcg_comm* comm, int nslabs, rcg_dslab* const* slabs, const double* const* w, int m, int kind,
                      rcg_dbasis** out);
void rcg_dbasis_destroy(rcg_dbasis* b);
/* distributed deflated PCG (basis kind DEFLATION, pcg.cpp:94-160) or SC-PCG around the block
 * IC(0) (kind SC, subspace_correction.cpp:27-57); basis null = rcg_dist_pcg_solve.  Per
 * iteration the m-vector W^T q (or W^T r) is allreduced before the replicated Cholesky solve. */
/* The accelerated solves of the sequence over THIS process's slab, batched (driver.cpp:181-195
 * over row slabs): nrhs <= 24 right-hand sides (B, X: nrhs x nloc, back to back, host or device)
 * through one kernel sequence -- the single-GPU batched solver with its reductions allreduced over
 * the ranks and p's halo rows exchanged (RT-interleaved) before each SpMV.  basis: deflation or
 * subspace correction (null: block-Jacobi ICCG).  One slab per process (NCCL / host transports;
 * loopback only at G = 1).  Reductions are fused (pcg.cpp:63-89 has one per dot): (p, q) travels
 * with W^T q, the (r, r) of the convergence check with the next iteration's (r, z) (subspace
 * correction: with W^T r) -- two allreduces per deflated iteration; environment RCG_DIST_FUSE=0
 * keeps one allreduce per dot. */
int rcg_dist_solve_batch(rcg_comm* comm, rcg_dslab* slab, const rcg_dbasis* basis, const double* B, double* X,
                         const rcg_solver_config* cfg, int nrhs, rcg_solve_report* reps);
int rcg_dist_solve(rcg_comm* comm, int nslabs, rcg_dslab* const* slabs, const rcg_dbasis* basis, const double* const* b,
                   double* const* x, const rcg_solver_config* cfg, rcg_solve_report* report);
/* solve 1 of the sequence over slabs: rcg_dist_pcg_solve with the error-sampling observer
 * (pcg.cpp:88 + sampling.cpp:66-78): observers[s] = slab s's sampler (rcg_sampler_create with
 * n = the slab's local rows, identical method / m / cap on every slab).  Every slab schedules the
 * same iterations (the scalars are allreduced) and snapshots its own rows of x. */
int rcg_dist_pcg_solve_sampled(rcg_comm* comm, int nslabs, rcg_dslab* const* slabs, rcg_sampler* const* observers,
                               const double* const* b, double* const* x, const rcg_solver_config* cfg,
                               rcg_solve_report* report);
/* the recycling step over slabs -- harvest_errors + build_aux_matrix + ScPreconditioner /
 * build_deflation_operator (recycling.cpp:17-96, deflation.cpp:45-76): errors x_final - slot per
 * slab (exactly-zero columns skipped globally), MGS with allreduced dots (same drop rule), A Q by
 * halo exchange, the allreduced Gram Q^T A Q eigensolved on every rank, Ritz values below theta
 * (or the keep_count smallest, keep_count > 0), W = Q T_sel per slab -> *out (kind
 * RCG_BASIS_DEFLATION or RCG_BASIS_SC; null when nothing is selected).  values receives the m_bar
 * Ritz values (ascending; caller sizes it to the sampler's m). */
int rcg_dist_recycle(rcg_comm* comm, int nslabs, rcg_dslab* const* slabs, rcg_sampler* const* samplers,
                     const double* const* x_final, double theta, int keep_count, int kind, int* m_bar, double* values,
                     double* theta_used, int* m_tilde, rcg_dbasis** out);

/* ------------------------------------------------------------------ the sequence (driver.cpp)
 * run_sequence (driver.cpp:108-222) on the device: rcg_seq_prepare scales A and factors IC(0)
 * once; rcg_seq_run runs one sequence of k_t right-hand sides (rhs: k_t vectors of length n back
 * to back, host or device; x receives the k_t solutions of A x = b): scaled solve 1 with the
 * error sampler, harvest + build_aux_matrix, SC preconditioner or deflation operator, solves
 * 2..k_t from x0 = 0 (batched when cfg->batch), solutions and true relative residuals in the
 * original scaling.  Errors use RCG_E_PARSE for invalid configs, as validate_config. */
#define RCG_METHOD_CG 0         /* "cg" */
#define RCG_METHOD_ICCG 1       /* "iccg" */
#define RCG_METHOD_ES_SC_ICCG 2 /* "es-sc-iccg" */
#define RCG_METHOD_ES_D_ICCG 3  /* "es-d-iccg" */
typedef struct {
    double eps;       /* RunConfig::eps */
    int max_iter;     /* RunConfig::max_iter */
    int sampling;     /* 'A' or 'B' (RunConfig::sampling) */
    int m;            /* RunConfig::m (method A uses max(m, 2) slots) */
    double theta;     /* RunConfig::theta (Ritz selection threshold) */
    int keep_count;   /* > 0: keep that many Ritz vectors instead of theta (extension) */
    int batch;        /* solves 2..k_t as batched multi-RHS kernel sequences */
    int memory;       /* 0: auto -- memory-lean recycling (errors / MGS in the sampler slots, streamed
                       * Gram) and unbatched solves when HBM is short (C4 on one GPU); 1: lean always */
} rcg_seq_config;
typedef struct {
    int* iterations;      /* k_t (caller arrays; each may be NULL) */
    int* converged;
    double* wall_time;
    double* true_relres;  /* ||b - A x|| / ||b|| with the unscaled A (driver.cpp:72-82) */
    double* ritz_values;  /* ritz_cap doubles */
    int ritz_cap;
    int m_bar, m_tilde;
    double theta_used;
    double w_build_time, avg_iterations, avg_wall_time, setup_time;
    int acceleration_inactive;
    /* k_t each (NULL to skip): the Lanczos estimate of every solve from its CG alpha / beta
     * (the extremes of the tridiagonal T_k): lambda_min, lambda_max and kappa of
     * the solve's preconditioned (solve 1: M^-1 A) or accelerated operator; NaN when a solve took
     * no iteration */
    double* lambda_min;
    double* lambda_max;
    double* kappa;
} rcg_seq_report;
int rcg_seq_prepare(rcg_ctx* ctx, const rcg_matrix* a_orig, int method, int blocks, rcg_seq** out);
void rcg_seq_destroy(rcg_seq* s);
int rcg_seq_run(rcg_seq* s, int k_t, const double* rhs, double* x, const rcg_seq_config* cfg, rcg_seq_report* rep);

#ifdef __cplusplus
}
#endif
#endif
