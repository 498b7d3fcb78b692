/* include/gnpc.h — C ABI of the B200-native GNP hot path (libgnpc.so).
 *
 * Plain pointers and sizes only; no C++ or torch types cross this boundary and
 * no exception escapes it.  Every entry point returns a gnpc_status; on error
 * gnpc_last_error() holds a thread-local message.  Host arrays follow the
 * reference's conventions: CSR with int64 indices / f64 values
 * (include/gnp/csr.hpp:13-20), column-major dense blocks
 * (include/gnp/dense.hpp:20-21), and GNP parameters as ONE flat f64 array in
 * the reference's checkpoint order enc1, enc1_bias, enc2, enc2_bias,
 * (U_l, W_l)_l, dec1, dec1_bias, dec2, dec2_bias (src/gnn.cpp:40-55).
 * Device numerics: Â values fp32, indices int32, GNP arithmetic fp32 with fp32
 * accumulation; Krylov vectors V, Z, x, r and all Krylov scalars fp64.
 *
 * Each function names the reference interface it replaces
 * (paths relative to /root/reference/proj).  INTEGRATION.md shows the
 * reference-side bindings.
 */
#ifndef GNPC_H
#define GNPC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GNPC_ABI_VERSION 1

typedef enum {
  GNPC_OK = 0,
  GNPC_EINVAL = 1,        /* std::invalid_argument in the reference  */
  GNPC_ERANGE = 2,        /* std::out_of_range (triplet indices)     */
  GNPC_ERUNTIME = 3,      /* std::runtime_error (checkpoints, mmio)  */
  GNPC_ECUDA = 4,         /* CUDA runtime error                      */
  GNPC_ENOMEM = 5,        /* device allocation failed                */
  GNPC_EUNSUPPORTED = 6,  /* e.g. nnz >= 2^31, d > 64, hidden > 256  */
  GNPC_ENODEV = 7         /* no CUDA device: the device path never falls back to the CPU */
} gnpc_status;

/* SolveStatus (include/gnp/krylov.hpp:44-50), same numbering. */
typedef enum {
  GNPC_CONVERGED = 0,
  GNPC_MAXITERS = 1,
  GNPC_TIMEOUT = 2,
  GNPC_SOLUTION_FAILURE = 3,
  GNPC_BREAKDOWN_EXACT = 4
} gnpc_solve_status;

typedef struct gnpc_csr_s* gnpc_csr;         /* CsrMatrix + its device copy  */
typedef struct gnpc_model_s* gnpc_model;     /* GnnParams bound to Â         */
typedef struct gnpc_trainer_s* gnpc_trainer; /* batched training state       */

/* ------------------------------------------------------------------ runtime */
int gnpc_abi_version(void);
const char* gnpc_last_error(void);
int gnpc_device_count(int* count);
int gnpc_set_device(int device);
int gnpc_synchronize(void);
/* Kernel launches issued by this library since load (for bench "gpu_launches"). */
int gnpc_launch_count(int64_t* count);

/* ------------------------------------------------------------------ CSR
 * replaces csr_from_triplets / CsrMatrix (include/gnp/csr.hpp:13-28,
 * src/csr.cpp:10-50): sort by (row, col), sum duplicates, keep explicit zeros. */
int gnpc_csr_from_triplets(int64_t n, int64_t m, const int64_t* rows, const int64_t* cols,
                           const double* vals, gnpc_csr* out);
/* Wraps an existing CSR (validated: monotone row_ptr, sorted in-range cols). */
int gnpc_csr_create(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                    const double* values, gnpc_csr* out);
/* Generators: "convection_diffusion" (src/gen.cpp:11-38; size=grid, p0=convection),
 * "random_nonsymmetric" (src/gen.cpp:40-69; size=n, p0=offdiag, p1=dominance),
 * "c2_convdiff3d" (size=grid, p0=Peclet), "c3_varcoeff2d" (size=grid, p0=sigma),
 * "c4_powerlaw" (size=n, p0=alpha), "c5_aniso9pt" (size=grid, p0=eps, p1=theta deg). */
int gnpc_csr_generate(const char* kind, int64_t size, double p0, double p1, uint64_t seed,
                      gnpc_csr* out);
int gnpc_csr_read_matrix_market(const char* path, gnpc_csr* out); /* src/mmio.cpp:89-93 */
int gnpc_csr_info(gnpc_csr a, int64_t* n, int64_t* nnz);
/* Device layout of Â (introspection; the device copy is built on first use):
 * *uploaded = 1 once it exists; *sliced_ell = 0 when no TMA-pipeline layout
 * was built, else a bit mask: 1 the 128-row sliced-ELL copy, 2 its pair-union
 * form (d = 32), 4 the strip-window pair-union form (d = 32), 16 the
 * training strip windows (built when a trainer uses the matrix), 32 the
 * apply path's length-sorted node order (ragged matrices); *long_rows = rows routed to the chunked long-row path (> 32
 * nonzeros).  No reference counterpart. */
int gnpc_csr_device_layout(gnpc_csr a, int* uploaded, int* sliced_ell, int* long_rows);
int gnpc_csr_export(gnpc_csr a, int64_t* row_ptr, int64_t* col_idx, double* values);
int gnpc_csr_gershgorin_gamma(gnpc_csr a, double* gamma);          /* src/csr.cpp:127-143 */
int gnpc_csr_prescale(gnpc_csr a, double gamma, gnpc_csr* out);     /* src/csr.cpp:145-150 */
int gnpc_csr_transpose(gnpc_csr a, gnpc_csr* out);                  /* src/csr.cpp:108-125 */
int gnpc_csr_hash(gnpc_csr a, uint64_t* hash);                      /* src/csr.cpp:152-173 */
int gnpc_csr_destroy(gnpc_csr a);
/* y = A x on the device (fp32 Â values widened to fp64, fp64 x/y, fp64 sums);
 * replaces spmv (src/csr.cpp:52-62).  Host pointers. */
int gnpc_spmv(gnpc_csr a, const double* x, double* y);

/* x_i ~ N(0,1): the reference Rng(seed).gaussian_vector(n) stream
 * (include/gnp/rng.hpp:27-46; mt19937_64 + Box-Muller with spare), host. */
int gnpc_gaussian_vector(uint64_t seed, int64_t n, double* out);

/* ------------------------------------------------------------------ GNP model
 * replaces GnnParams/init_params/gnn_apply/apply_preconditioner
 * (include/gnp/gnn.hpp:16-46,48-79,125-126; src/gnn.cpp:92-206,455-474). */
int gnpc_param_count(int64_t d, int64_t hidden, int64_t layers, int64_t* count);
int gnpc_init_params(int64_t d, int64_t hidden, int64_t layers, uint64_t seed, double* params);
/* Binds params to Â (borrowed: the csr must outlive the model, as GnnOperator
 * borrows `ahat` at src/gnn.cpp:466).  d <= 64, hidden <= 256. */
int gnpc_model_create(gnpc_csr ahat, int64_t d, int64_t hidden, int64_t layers,
                      const double* params, gnpc_model* out);
int gnpc_model_set_params(gnpc_model m, const double* params);
int gnpc_model_get_params(gnpc_model m, double* params);
int gnpc_model_dims(gnpc_model m, int64_t* d, int64_t* hidden, int64_t* layers);
int gnpc_model_destroy(gnpc_model m);
/* out = M(b): host f64 in/out (the FlexibleOperator::apply drop-in). */
int gnpc_apply(gnpc_model m, const double* b, double* out);
/* Device-resident variants on a caller stream (cudaStream_t passed as void*).
 * Threading: a model owns one apply workspace (activations, τ partials, the
 * persistent apply's grid-barrier counter), so applies of ONE model must be
 * serialised (one stream / one thread at a time), like the reference's
 * "called from the solve's thread only".  Distinct models may
 * run concurrently.  After a trainer's Adam step updates a model's device
 * parameters, applies and gnpc_model_get_params return GNPC_EINVAL until
 * gnpc_trainer_sync_model (or gnpc_model_set_params) makes it consistent. */
int gnpc_apply_device_f32(gnpc_model m, const float* b, float* out, void* stream);
int gnpc_apply_device_f64(gnpc_model m, const double* b, double* out, void* stream);
/* Same as gnpc_apply_device_f32 with CUDA events between the pipeline's
 * kernels on `stream`; adds per-kind durations (ms) and launch counts into
 * ms_by_kind[5] / count_by_kind[5]: 0 norm, 1 lift (d = 32 strip windows:
 * the lift fused into the first layer, one kernel), 2 long-row ÂX, 3 fused
 * layer, 4 last layer + projection.  Used by bench.py's roofline. */
int gnpc_apply_profile(gnpc_model m, const float* b, float* out, void* stream, double* ms_by_kind,
                       int64_t* count_by_kind);

/* ------------------------------------------------------------------ checkpoints
 * GNPCKPT 1 format (src/gnn.cpp:480-570), byte-identical files. */
int gnpc_checkpoint_save(const char* path, int64_t d, int64_t hidden, int64_t layers,
                         const double* params, gnpc_csr a);
/* dims3 = {d, hidden, layers}; meta3 = {n, nnz, hash}; params may be NULL
 * (size query). */
int gnpc_checkpoint_load(const char* path, int64_t* dims3, uint64_t* meta3, double* params);

/* ------------------------------------------------------------------ FGMRES
 * replaces fgmres_solve / gmres_solve (include/gnp/krylov.hpp:29-58,81-86;
 * src/krylov.cpp:175-282) with the same history and status semantics. */
typedef struct {
  double rtol;          /* default 1e-8 */
  int64_t maxiters;     /* default 100  */
  int64_t restart;      /* default 10   */
  double timeout_secs;  /* < 0: none    */
} gnpc_solve_config;

typedef struct {
  int64_t* iteration; /* capacity entries (may be NULL when capacity == 0) */
  double* relres;
  double* elapsed;
  int64_t capacity;
  int64_t length;     /* out: full history length (may exceed capacity) */
  int64_t reorth;     /* out: Arnoldi steps that took the re-orthogonalisation pass */
} gnpc_history;

/* M: NULL = unpreconditioned (gmres_solve), else the device GNP.  Host
 * b/x0/x; x0 may be NULL (zero). *status receives a gnpc_solve_status. */
int gnpc_fgmres(gnpc_csr a, gnpc_model m, const double* b, const double* x0,
                const gnpc_solve_config* cfg, double* x, gnpc_history* hist, int* status);
/* Same with an arbitrary host FlexibleOperator (callback on host vectors,
 * once per Arnoldi step; a nonzero return aborts the solve with GNPC_ERUNTIME). */
typedef int (*gnpc_host_operator)(void* ctx, const double* in, double* out, int64_t n);
int gnpc_fgmres_host_operator(gnpc_csr a, gnpc_host_operator op, void* ctx, const double* b,
                              const double* x0, const gnpc_solve_config* cfg, double* x,
                              gnpc_history* hist, int* status);
/* Device-resident b / x (fp64) on a caller stream; history as above. */
int gnpc_fgmres_device(gnpc_csr a, gnpc_model m, const double* b_dev, double* x_dev,
                       const gnpc_solve_config* cfg, gnpc_history* hist, int* status,
                       void* stream);

/* ------------------------------------------------------------------ training
 * replaces the per-step body of train_preconditioner (src/gnn.cpp:422-449),
 * l1_residual_loss (src/gnn.cpp:309-335), gnn_backward (src/gnn.cpp:208-307)
 * and adam_step (src/gnn.cpp:345-363).  The batch of B samples is resident as
 * [n][B][d] so one Â row gather serves all samples. */
int gnpc_trainer_create(gnpc_model m, int64_t batch, double lr, gnpc_trainer* out);
int gnpc_trainer_destroy(gnpc_trainer t);
/* x, b: n x B column-major host f64 (the TrainingBatch of src/sampler.cpp:68-83).
 * Writes loss (and grads, flat f64, summed over the batch like
 * src/gnn.cpp:439-440; out n x B optional). No parameter update. */
int gnpc_forward_backward(gnpc_trainer t, const double* x, const double* b, double* loss,
                          double* grads, double* out);
/* One full step: forward, loss, backward, Adam (state kept in the trainer). */
int gnpc_train_step(gnpc_trainer t, const double* x, const double* b, double* loss);
/* Throughput mode: pairs x ~ N(0,I) drawn on the device (Philox4x32-10,
 * counter = (seed, step)), b = A x; one full step; loss read back. */
int gnpc_train_step_synthetic(gnpc_trainer t, uint64_t seed, double* loss);
/* Loss of the current params on a batch (monitoring_loss, src/gnn.cpp:390-397). */
int gnpc_monitor_loss(gnpc_trainer t, const double* x, const double* b, int64_t batch,
                      double* loss);
/* Data-parallel split of a step: the flat f64 device gradient
 * buffer (gradient of this trainer's batch loss (1/B)Σ_k, reference flat
 * order) that a collective averages in place over ranks between
 * gnpc_train_backward_only / gnpc_train_backward_synthetic and
 * gnpc_train_apply_grads (replaces accumulate, src/gnn.cpp:439-440). */
int gnpc_trainer_grad_buffer(gnpc_trainer t, double** dev_ptr, int64_t* count);
/* The CUDA stream (cudaStream_t) every kernel of this trainer runs on, for
 * callers that time or order work against it. */
int gnpc_trainer_stream(gnpc_trainer t, void** stream);
int gnpc_train_backward_only(gnpc_trainer t, const double* x, const double* b, double* loss);
int gnpc_train_backward_synthetic(gnpc_trainer t, uint64_t seed, double* loss);
int gnpc_train_apply_grads(gnpc_trainer t);
int gnpc_trainer_adam_state(gnpc_trainer t, double* m1, double* m2, int64_t* step);
/* Current f64 master parameters (flat reference order). */
int gnpc_trainer_params(gnpc_trainer t, double* params);
/* Copy the trainer's parameters into its model (inference view rebuilt). */
int gnpc_trainer_sync_model(gnpc_trainer t);

/* ------------------------------------------------------------------ sampler
 * build_spectral_sampler (src/sampler.cpp:10-39): an unpreconditioned
 * Arnoldi cycle of m steps from Rng(seed).gaussian_vector(n) on the device
 * (fp32 Â, fp64 basis; the device FGMRES kernels), then the host Jacobi SVD
 * of the (k+1) x k Hessenberg (src/svd.cpp:10-80); k < m on breakdown.
 * GNPC_ERUNTIME when the Hessenberg is numerically zero. */
typedef struct gnpc_sampler_s* gnpc_sampler;
int gnpc_sampler_create(gnpc_csr a, int64_t m, uint64_t seed, gnpc_sampler* out);
/* The host half alone, from a given cycle: v n x k basis, hbar (k+1) x k
 * (col-major), k >= 1 (src/sampler.cpp:19-38). */
int gnpc_sampler_from_arnoldi(int64_t n, int64_t k, const double* v, const double* hbar,
                              gnpc_sampler* out);
int gnpc_sampler_destroy(gnpc_sampler s);
/* k = basis columns kept (SpectralSampler::m), m_eff = retained rank. */
int gnpc_sampler_info(gnpc_sampler s, int64_t* k, int64_t* m_eff);
/* v: n x k, zsv: k x k (col-major), sv: k singular values; any may be NULL. */
int gnpc_sampler_export(gnpc_sampler s, double* v, double* zsv, double* sv);
/* assemble_batch (src/sampler.cpp:68-83) from Rng(seed) after dropping
 * skip_batches batches: n x batch col-major x and b = A x (f64, host).
 * s may be NULL when spectral_count == 0. */
int gnpc_assemble_batch(gnpc_sampler s, gnpc_csr a, uint64_t seed, int64_t skip_batches,
                        int64_t batch, int64_t spectral_count, double* x, double* b);
/* The same batch from the device generator gnpc_train_preconditioner uses
 * (reference Rng stream: host MT19937-64 words, device tempering and
 * Box-Muller; spectral x = V (Zsv S^-1 eps) and b = A x on the device,
 * src/sampler.cpp:41-83).  For parity tests against gnpc_assemble_batch. */
int gnpc_device_pairs(gnpc_sampler s, gnpc_csr a, uint64_t seed, int64_t skip_batches, int64_t batch,
                      int64_t spectral_count, double* x, double* b);

/* train_preconditioner (src/gnn.cpp:401-451): Gaussian and spectral pairs
 * (spectral_count of each batch), monitor batch, best snapshot.
 * losses: steps+1 entries. */
typedef struct {
  double lr;
  int64_t steps, batch, spectral_count, arnoldi_m;
  uint64_t seed;
  int64_t monitor_batch, d, hidden, layers;
} gnpc_train_config;
int gnpc_train_preconditioner(gnpc_csr a, const gnpc_train_config* cfg, double* best,
                              double* losses, double* best_loss);
/* The same run with device timings: timing_ms4 = {whole loop, pair generation
 * (Box-Muller / spectral x + b = A x), monitoring forward + best snapshot,
 * host wait for the pair stream}, milliseconds summed over the steps. */
int gnpc_train_preconditioner_timed(gnpc_csr a, const gnpc_train_config* cfg, double* best,
                                    double* losses, double* best_loss, double* timing_ms4);

#ifdef __cplusplus
}
#endif
#endif /* GNPC_H */
