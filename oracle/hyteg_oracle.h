/*
 * TEST INFRASTRUCTURE ONLY -- never linked into or called by the product.
 *
 * Plain-C restatement of the reference's P1 macro-face multigrid hot path
 * (arXiv 1805.10167 "hytegrid", /root/reference/proj), single logical rank,
 * on the reference's own per-primitive storage layout. It is the checker for
 * the CUDA path in tests/ and __graft_entry__.smoke(), and the "port" CPU
 * baseline. Pinned bitwise against the reference library (oracle/_ref) and
 * the committed golden vectors in tests/golden/ (tests/test_oracle_pins.py).
 *
 * Values cross the interface as owned-DoF vectors in GlobalDoFMap order.
 */
#ifndef HYTEG_ORACLE_H
#define HYTEG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct og_session og_session;

const char* og_last_error(void);
og_session* og_create(const char* mesh_text, int min_level, int max_level, const int* bc_markers,
                      const unsigned char* bc_flags, int nbc, int nfuncs);
void og_destroy(og_session* s);
int64_t og_owned(og_session* s, int level);
int og_set(og_session* s, int f, int level, const double* v);
int og_get(og_session* s, int f, int level, double* v);
int og_flags(og_session* s, int level, unsigned char* out);
int og_stencil(og_session* s, int64_t id, int level, double* out, int* len);
int og_keyed_uniform(og_session* s, int level, uint64_t seed, uint64_t stream, double lo, double hi, double* out);
int og_sync(og_session* s, int f, int level);
int og_apply(og_session* s, int src, int dst, int level, int mask);
int og_residual(og_session* s, int rhs, int x, int r, int level);
int og_jacobi(og_session* s, int rhs, int x, double omega, int level);
int og_gs(og_session* s, int rhs, int x, int level);
/* coloured hybrid GS: faces by (c + 2r) mod 3, edges odd then even k (no reference counterpart) */
int og_cgs(og_session* s, int rhs, int x, int level);
int og_restrict(og_session* s, int fine, int coarse, int lc, int mask);
int og_prolongate(og_session* s, int coarse, int fine, int lc, int mask);
int og_assign(og_session* s, double alpha, int x1, double beta, int x2, int dst, int level, int mask);
int og_add_scaled(og_session* s, int dst, double gamma, int y, int level, int mask);
int og_dot(og_session* s, int a, int b, int level, double* out);
/* coarse solve of og_vcycle / og_fmg / og_pcg: mode 0 (default) matrix-free
 * CG with sequential dots; mode 1 the product's: assembled constrained CSR and
 * the device kernels' fixed reduction shapes (nsm = SM count, 148 on B200) */
void og_coarse_solver(og_session* s, int mode, int nsm);
/* that CSR (min level) as COO in row / column order; f = a scratch function */
int og_coarse_matrix(og_session* s, int f, int64_t* rows, int64_t* cols, double* vals, int64_t cap, int64_t* nnz);
/* smoother 0 weighted Jacobi (omega), 1 hybrid GS, 2 coloured GS */
int og_vcycle(og_session* s, int rhs, int x, int level, int smoother, int nu1, int nu2, double omega,
              double coarse_tol, int ncycles, double* residuals);
int og_vcycle_jacobi(og_session* s, int rhs, int x, int level, int nu1, int nu2, double omega, double coarse_tol,
                     int ncycles, double* residuals);
/* full multigrid then V-cycles to tol * ||r(x=0)|| (configuration 4) */
int og_fmg(og_session* s, int rhs, int x, int level, int smoother, int nu1, int nu2, double omega, double coarse_tol,
           int per_level, double tol, int max_cycles, double* residuals, int* n_out);
/* CG preconditioned by one V(nu1, nu2) Jacobi cycle (configuration 5) */
int og_pcg(og_session* s, int rhs, int x, int level, int nu1, int nu2, double omega, double coarse_tol, int iters,
           double* residuals);

#ifdef __cplusplus
}
#endif
#endif
