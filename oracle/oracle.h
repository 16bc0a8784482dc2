/*
 * oracle.h -- CPU restatement of the recycg reference algorithms (TEST INFRASTRUCTURE ONLY).
 *
 * This header declares the plain-C oracle used by tests/, bench.py's cpu_baseline leg and
 * __graft_entry__.smoke() as the *checker* of the CUDA product path.  Nothing in the product
 * (paper_2203_08498_b200/) may include, link or call it.
 *
 * Every function restates one reference routine with the same floating-point operation order
 * (sequential sums from 0.0, separate multiply and add roundings -- build with
 * -ffp-contract=off), so its results are bitwise equal to the reference built the same way.
 * That equality is pinned by tests/test_oracle.py against oracle/_ref (the reference itself,
 * compiled from /root/reference sources by oracle/Makefile) and against the reference's own
 * known-answer tests.  Citations are relative to /root/reference/proj.
 */
#ifndef RCG_ORACLE_H
#define RCG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_INVALID = 1, ORC_BREAKDOWN = 2 };

/* message of the last non-OK status on this thread */
const char* orc_last_error(void);

/* borrowed full-symmetric CSR (include/recycg/csr_matrix.hpp:20-51) */
typedef struct {
    int32_t n;
    const int32_t* rs;
    const int32_t* ci;
    const double* va;
} orc_csr;

/* ---- portable RNG (include/recycg/rng.hpp:18-41): mt19937_64, top 53 bits -> [-1,1) ---- */
typedef struct {
    uint64_t mt[312];
    int idx;
} orc_mt64;
void orc_mt64_seed(orc_mt64* g, uint64_t seed);
uint64_t orc_mt64_next(orc_mt64* g);
double orc_uniform_pm1(orc_mt64* g);
void orc_uniform_pm1_fill(uint64_t seed, uint64_t skip, int64_t n, double* out);

/* ---- sparse core ---- */
void orc_spmv(const orc_csr* a, const double* x, double* y);
void orc_spmv_dual(const orc_csr* a, const double* x1, const double* x2, double* y1, double* y2);
double orc_dot(int64_t n, const double* a, const double* b);
/* test-only: 0 = reference forward summation (default), 1 = reversed, 2 = pairwise tree
 * (rounding-floor probes of the problem's sensitivity to reduction order) */
void orc_set_dot_order(int order);
int orc_diagonal_scale(const orc_csr* a, double* va_out, double* d_inv_sqrt);

/* ---- IC(0) (src/ic_preconditioner.cpp) ---- */
typedef struct {
    int32_t n;
    int32_t nblocks;
    int32_t* bounds;     /* nblocks+1 */
    int32_t* lrs;        /* n+1 */
    int32_t* lcol;
    double* lval;
    double* d;           /* n */
    int32_t* urs;        /* n+1 */
    int32_t* ucol;
    double* uval;
    int64_t nnz_l;
    double shift;
} orc_ic;
int orc_ic0_factorize(const orc_csr* a, double shift, int nblocks, orc_ic** out);
void orc_ic_free(orc_ic* f);
void orc_ic_apply(const orc_ic* f, const double* r, double* z);

/* ---- small dense (src/dense.cpp) ---- */
int orc_chol_factor(int k, const double* s, double* l);
void orc_chol_solve(int k, const double* l, const double* f, double* u);
int orc_sym_eig(int k, const double* s, double* values, double* vectors);
int orc_mgs(int32_t n, int k, const double* v, double drop_tol, double* e);

/* ---- W basis shared by deflation and subspace correction ---- */
typedef struct {
    int32_t n;
    int k;
    double* w;   /* column-major n x k */
    double* aw;  /* column-major n x k */
    double* l;   /* k x k row-major Cholesky factor of W^T A W */
} orc_basis;
/* who: 0 = build_deflation_operator message, 1 = ScPreconditioner message */
int orc_basis_build(const orc_csr* a, int k, const double* w, int who, orc_basis** out);
void orc_basis_free(orc_basis* b);
void orc_project_pt(const orc_basis* b, const double* y, double* out);
void orc_project_p(const orc_basis* b, const double* x, double* out);
void orc_direct_component(const orc_basis* b, const double* rhs, double* out);

/* ---- preconditioner descriptor (include/recycg/preconditioner.hpp:10-26) ---- */
enum { ORC_PREC_IDENTITY = 0, ORC_PREC_IC = 1, ORC_PREC_SC = 2 };
typedef struct {
    int kind;
    const orc_ic* ic;      /* IC factor, or inner of SC when non-NULL */
    const orc_basis* sc;   /* SC basis when kind == ORC_PREC_SC */
} orc_prec;
void orc_prec_apply(const orc_prec* m, const double* r, double* z);

/* ---- samplers (src/sampling.cpp) ---- */
typedef struct {
    int method; /* 0 = A, 1 = B */
    int m;
    int32_t n;
    double* slots;       /* m x n */
    int* occupied;
    int* stored_iter;
    int l_max;
    int64_t h;
    double alpha;
    int next_slot;
} orc_sampler;
int orc_sampler_create_a(int m, int iteration_cap, int32_t n, orc_sampler** out);
int orc_sampler_create_b(int m, double eps, int32_t n, orc_sampler** out);
void orc_sampler_offer(orc_sampler* s, int iteration, double relres, const double* payload);
void orc_sampler_free(orc_sampler* s);

/* ---- Krylov solvers (src/pcg.cpp, src/condest.cpp) ---- */
typedef struct {
    int iterations;
    int converged;
    double wall_time;
    int cap;            /* capacity of the optional arrays below */
    double* history;    /* relres per iteration, optional */
    double* alphas;     /* alpha_i per iteration, optional (Lanczos) */
    double* betas;      /* beta_i per iteration (0 at i=1), optional (Lanczos) */
} orc_report;
/* observer: NULL, or a sampler fed x (payload_kind 0) or r (payload_kind 1) */
int orc_pcg_solve(const orc_csr* a, const double* b, const orc_prec* m, double* x, double eps,
                  int max_iter, orc_sampler* obs, int payload_kind, orc_report* rep);
int orc_deflated_pcg_solve(const orc_csr* a, const double* b, const orc_prec* m,
                           const orc_basis* defl, double* x, double eps, int max_iter,
                           orc_report* rep);

typedef struct {
    double lambda_max;
    double lambda_min;
    double kappa;
    int power_iterations;
    int power_unsettled;
    int lambda_min_available;
    int nritz;
    double* ritz_values; /* caller buffer of >= m_samples doubles */
} orc_condest;
int orc_pcg_with_condest(const orc_csr* a, const double* b, const orc_prec* m, double* x,
                         double eps, int max_iter, int m_samples, uint64_t v0_seed,
                         orc_report* rep, orc_condest* est);

/* ---- recycling (src/recycling.cpp) ---- */
int orc_harvest_errors(const double* x_final, const orc_sampler* s, double* e);
int orc_harvest_stored(const orc_sampler* s, double* e);
int orc_rayleigh_ritz(const orc_csr* a, int k, const double* e, double* values, double* vectors);
/* errors: column-major n x k.  Outputs: m_bar, spectrum values (k), W (n x m_tilde). */
int orc_build_aux(const orc_csr* a, int k, const double* errors, double theta, int* m_bar,
                  double* values, double* w, int* m_tilde);

/* ---- Lanczos tridiagonal estimate from CG alpha/beta (no reference) ---- */
int orc_lanczos_extremes(int k, const double* alphas, const double* betas, double* lmin,
                         double* lmax);

#ifdef __cplusplus
}
#endif
#endif
