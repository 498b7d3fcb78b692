/* oracle/gnp_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C (C11, f64) restatement of the reference's GNP hot path, used as the
 * parity checker for the CUDA product path.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it.  It is pinned against the
 * unmodified reference (oracle/_ref/libgnpref.so, built by oracle/Makefile) and
 * against the committed golden vectors in tests/golden/.
 *
 * Conventions: CSR = (n, row_ptr[n+1], col_idx[nnz], values[nnz]) with int64
 * indices and f64 values (include/gnp/csr.hpp:13-20).  Dense blocks are
 * column-major (include/gnp/dense.hpp:20-21).  Parameters are one flat f64
 * array in the reference's checkpoint order (src/gnn.cpp:40-55).
 * Functions returning int: 0 ok, -1 bad argument (oc_last_error()).
 */
#ifndef GNP_ORACLE_H
#define GNP_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* oc_last_error(void);

/* ---- RNG: mt19937_64 + (x>>11)*2^-53 + Box-Muller with spare (include/gnp/rng.hpp:13-52) */
typedef struct {
  uint64_t mt[312];
  int idx;
  int have_spare;
  double spare;
} oc_rng;
void oc_rng_init(oc_rng* r, uint64_t seed);
uint64_t oc_rng_next(oc_rng* r);
double oc_rng_uniform(oc_rng* r);
double oc_rng_uniform_symmetric(oc_rng* r, double bound);
double oc_rng_gaussian(oc_rng* r);
void oc_gaussian_vector(uint64_t seed, size_t n, double* out);

/* ---- sparse core (src/csr.cpp) */
/* out arrays sized m (worst case); *nnz_out receives the merged count. */
int oc_csr_from_triplets(size_t n, size_t m, const int64_t* rows, const int64_t* cols,
                         const double* vals, int64_t* rp, int64_t* ci, double* v,
                         size_t* nnz_out);
void oc_spmv(size_t n, const int64_t* rp, const int64_t* ci, const double* v,
             const double* x, double* y);
void oc_spmm(size_t n, const int64_t* rp, const int64_t* ci, const double* v,
             size_t k, const double* x, double* y);
void oc_spmv_transpose(size_t n, const int64_t* rp, const int64_t* ci, const double* v,
                       const double* x, double* y);
void oc_transpose(size_t n, const int64_t* rp, const int64_t* ci, const double* v,
                  int64_t* trp, int64_t* tci, double* tv);
double oc_gershgorin_gamma(size_t n, const int64_t* rp, const int64_t* ci, const double* v);
uint64_t oc_csr_hash(size_t n, const int64_t* rp, const int64_t* ci, const double* v);
/* gen_convection_diffusion (src/gen.cpp:11-38); arrays sized 5*grid*grid. */
int oc_gen_convection_diffusion(size_t grid, double conv, int64_t* rp, int64_t* ci,
                                double* v, size_t* nnz_out);

/* ---- GNP (src/gnn.cpp) */
size_t oc_param_count(size_t d, size_t hidden, size_t layers);
int oc_init_params(size_t d, size_t hidden, size_t layers, uint64_t seed, double* out);
int oc_gnn_apply(size_t n, const int64_t* rp, const int64_t* ci, const double* v,
                 size_t d, size_t hidden, size_t layers, const double* params,
                 const double* b, double* out);
int oc_gnn_forward_backward(size_t n, const int64_t* rp, const int64_t* ci,
                            const double* v, size_t d, size_t hidden, size_t layers,
                            const double* params, const double* b, const double* gout,
                            double* out, double* grads);
int oc_l1_residual_loss(size_t n, const int64_t* rp, const int64_t* ci, const double* v,
                        size_t batch, const double* out, const double* x, double* loss,
                        double* grad);
void oc_adam_step(size_t count, double* params, const double* grads, double* m1,
                  double* m2, size_t* t, double lr);
int oc_batch_loss_grads(size_t n, const int64_t* rp, const int64_t* ci, const double* v,
                        size_t d, size_t hidden, size_t layers, const double* params,
                        size_t batch, const double* x, const double* b, double* loss,
                        double* grads, double* out_batch);
/* Gaussian training batch (src/sampler.cpp:61-83, spectral_count = 0). */
int oc_gaussian_batch(size_t n, const int64_t* rp, const int64_t* ci, const double* v,
                      uint64_t seed, size_t skip_batches, size_t batch, double* x,
                      double* b);

/* ---- Krylov (src/krylov.cpp) */
int oc_hessenberg_lstsq(size_t k, const double* hbar, double beta, double* y,
                        double* tracked, int* singular);
/* kind: 0 none, 1 gnp(d,hidden,layers,params), 2 dense n x n col-major in params,
 * 3 identity, 4 callback (params points to an oc_op_cb: any FlexibleOperator,
 * e.g. the device GNP, driven by the oracle's f64 FGMRES).  Returns SolveStatus (0 converged, 1 maxiters, 2 timeout,
 * 3 solution_failure, 4 breakdown_exact) or -1. */
typedef struct {
  void (*fn)(void* ctx, const double* in, double* out, size_t n);
  void* ctx;
} oc_op_cb;
int oc_fgmres(size_t n, const int64_t* rp, const int64_t* ci, const double* v,
              const double* b, int kind, size_t d, size_t hidden, size_t layers,
              const double* params, const double* x0, double rtol, size_t maxiters,
              size_t restart, double timeout_secs, double* x_out, size_t* hist_iter,
              double* hist_rel, double* hist_t, size_t hist_cap, size_t* hist_len);

/* ---- spectral sampler (src/sampler.cpp:10-83, src/svd.cpp:10-80) */
int oc_arnoldi_cycle(size_t n, const int64_t* rp, const int64_t* ci, const double* v,
                     const double* r0, size_t m, double* vout, double* hbar, size_t* steps,
                     int* breakdown);
int oc_jacobi_svd(size_t rows, size_t cols, const double* a, double* u, double* s, double* v);
int oc_spectral_sampler(size_t n, const int64_t* rp, const int64_t* ci, const double* v,
                        size_t m, uint64_t seed, double* vout, double* zsv, double* s,
                        size_t* k_out, size_t* m_eff_out);
int oc_assemble_batch(size_t n, const int64_t* rp, const int64_t* ci, const double* v,
                      size_t k, size_t m_eff, const double* vb, const double* zsv,
                      const double* s, uint64_t seed, size_t skip_batches, size_t batch,
                      size_t spectral_count, double* x, double* b);

/* ---- full-size parity support (bit-identical threaded restatements) */
typedef struct {
  size_t n, nnz, cap;
  int64_t *rp, *ci;
  double* v;
} oc_csr_buf;
/* BASELINE config generators (the repo's recipes, gnp_host.cpp): kind
 * "c2_convdiff3d" | "c3_varcoeff2d" | "c4_powerlaw" | "c5_aniso9pt". */
int oc_gen_named(const char* kind, size_t size, double p0, double p1, uint64_t seed,
                 oc_csr_buf* out);
void oc_csr_buf_free(oc_csr_buf* a);
/* threads used by oc_fgmres's GNP operator (default 1) */
void oc_set_threads(size_t t);
int oc_gnn_apply_mt(size_t n, const int64_t* rp, const int64_t* ci, const double* v,
                    size_t d, size_t hidden, size_t layers, const double* params,
                    const double* b, double* out, size_t threads);
int oc_batch_loss_grads_mt(size_t n, const int64_t* rp, const int64_t* ci, const double* v,
                           size_t d, size_t hidden, size_t layers, const double* params,
                           size_t batch, const double* x, const double* b, double* loss,
                           double* grads, double* out_batch, size_t threads);

#ifdef __cplusplus
}
#endif
#endif
