// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// A flat extern "C" face over the UNMODIFIED reference library (gnprecond,
// /root/reference/proj/src/*.cpp), compiled by oracle/Makefile into
// oracle/_ref/libgnpref.so.  Tests, __graft_entry__.smoke() (indirectly via the
// restatement) and bench.py's cpu_baseline / --impl reference leg call it
// through ctypes to (1) pin the plain-C restatement (oracle/gnp_oracle.c) and
// (2) time the reference CPU path.  Every function here only marshals arrays
// into the reference's own types and calls the reference's own API:
//   CsrMatrix / csr_from_triplets ...... include/gnp/csr.hpp:13-28
//   gnn_forward / gnn_backward ......... include/gnp/gnn.hpp:70-79
//   l1_residual_loss / adam_step ....... include/gnp/gnn.hpp:81-96
//   train_preconditioner ................ include/gnp/gnn.hpp:120-123
//   fgmres_solve / arnoldi / lstsq ...... include/gnp/krylov.hpp:66-86
// Errors never cross the C boundary: -1 is returned and ref_last_error()
// holds the exception text.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "gnp/baselines.hpp"
#include "gnp/csr.hpp"
#include "gnp/gen.hpp"
#include "gnp/gnn.hpp"
#include "gnp/krylov.hpp"
#include "gnp/mmio.hpp"
#include "gnp/rng.hpp"
#include "gnp/sampler.hpp"
#include "gnp/svd.hpp"

using namespace gnp;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  } catch (...) {
    g_err = "unknown exception";
    return -1;
  }
}

CsrMatrix* H(void* h) { return static_cast<CsrMatrix*>(h); }

GnnDims dims_of(std::size_t d, std::size_t hidden, std::size_t layers) {
  GnnDims g;
  g.d = d;
  g.hidden = hidden;
  g.layers = layers;
  return g;
}

// Flat order = the reference's param_views order (src/gnn.cpp:40-55).
template <class Fn>
void walk(GnnParams& p, Fn&& fn) {
  fn(p.enc1.data(), p.enc1.size());
  fn(p.enc1_bias.data(), p.enc1_bias.size());
  fn(p.enc2.data().data(), p.enc2.data().size());
  fn(p.enc2_bias.data(), p.enc2_bias.size());
  for (auto& l : p.layers) {
    fn(l.u.data().data(), l.u.data().size());
    fn(l.w.data().data(), l.w.data().size());
  }
  fn(p.dec1.data().data(), p.dec1.data().size());
  fn(p.dec1_bias.data(), p.dec1_bias.size());
  fn(p.dec2.data(), p.dec2.size());
  fn(&p.dec2_bias, 1);
}

GnnParams unflat(std::size_t d, std::size_t hidden, std::size_t layers,
                 const double* flat) {
  Rng dummy(0);
  GnnParams p = init_params(dims_of(d, hidden, layers), dummy);
  std::size_t k = 0;
  walk(p, [&](double* x, std::size_t n) {
    std::memcpy(x, flat + k, n * sizeof(double));
    k += n;
  });
  return p;
}

void flat(const GnnParams& pc, double* out) {
  GnnParams& p = const_cast<GnnParams&>(pc);
  std::size_t k = 0;
  walk(p, [&](double* x, std::size_t n) {
    std::memcpy(out + k, x, n * sizeof(double));
    k += n;
  });
}

// Test-only operators (same roles as tests/test_krylov.cpp:16-32 fakes).
class DenseColMajorOperator final : public FlexibleOperator {
 public:
  DenseColMajorOperator(std::size_t n, const double* m) : n_(n), m_(m, m + n * n) {}
  DenseVector apply(const DenseVector& v) const override {
    DenseVector y(n_, 0.0);
    for (std::size_t j = 0; j < n_; ++j)
      for (std::size_t i = 0; i < n_; ++i) y[i] += m_[j * n_ + i] * v[j];
    return y;
  }
  std::string name() const override { return "dense"; }

 private:
  std::size_t n_;
  std::vector<double> m_;
};

class IdentityOp final : public FlexibleOperator {
 public:
  DenseVector apply(const DenseVector& v) const override { return v; }
  std::string name() const override { return "identity"; }
};

int status_code(SolveStatus s) { return static_cast<int>(s); }

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------- CSR
void* ref_csr_new(std::size_t n, const std::int64_t* rp, const std::int64_t* ci,
                  const double* v) {
  auto* a = new CsrMatrix;
  a->n = n;
  a->row_ptr.assign(rp, rp + n + 1);
  const std::size_t nnz = static_cast<std::size_t>(rp[n]);
  a->col_idx.assign(ci, ci + nnz);
  a->values.assign(v, v + nnz);
  return a;
}

void* ref_csr_from_triplets(std::size_t n, std::size_t m, const std::int64_t* r,
                            const std::int64_t* c, const double* v) {
  CsrMatrix* out = nullptr;
  int rc = guarded([&] {
    std::vector<std::size_t> rows(r, r + m), cols(c, c + m);
    std::vector<double> vals(v, v + m);
    out = new CsrMatrix(csr_from_triplets(n, std::move(rows), std::move(cols),
                                          std::move(vals)));
  });
  return rc == 0 ? out : nullptr;
}

void* ref_gen_convection_diffusion(std::size_t grid, double conv) {
  CsrMatrix* out = nullptr;
  guarded([&] { out = new CsrMatrix(gen_convection_diffusion(grid, conv)); });
  return out;
}

void* ref_gen_random_nonsymmetric(std::size_t n, std::size_t k, double dom,
                                  std::uint64_t seed) {
  CsrMatrix* out = nullptr;
  guarded([&] { out = new CsrMatrix(gen_random_nonsymmetric(n, k, dom, seed)); });
  return out;
}

void* ref_read_matrix_market(const char* path) {
  CsrMatrix* out = nullptr;
  guarded([&] { out = new CsrMatrix(read_matrix_market_file(path)); });
  return out;
}

void ref_csr_free(void* h) { delete H(h); }
std::size_t ref_csr_n(void* h) { return H(h)->n; }
std::size_t ref_csr_nnz(void* h) { return H(h)->nnz(); }

void ref_csr_export(void* h, std::int64_t* rp, std::int64_t* ci, double* v) {
  const CsrMatrix& a = *H(h);
  for (std::size_t i = 0; i <= a.n; ++i) rp[i] = static_cast<std::int64_t>(a.row_ptr[i]);
  for (std::size_t k = 0; k < a.nnz(); ++k) {
    ci[k] = static_cast<std::int64_t>(a.col_idx[k]);
    v[k] = a.values[k];
  }
}

double ref_gershgorin_gamma(void* h) { return gershgorin_gamma(*H(h)); }

void* ref_prescale(void* h, double gamma) {
  CsrMatrix* out = nullptr;
  guarded([&] { out = new CsrMatrix(prescale(*H(h), gamma)); });
  return out;
}

void* ref_transpose(void* h) { return new CsrMatrix(transpose(*H(h))); }
std::uint64_t ref_csr_hash(void* h) { return csr_content_hash(*H(h)); }

int ref_spmv(void* h, const double* x, double* y) {
  return guarded([&] {
    DenseVector xv(x, x + H(h)->n);
    DenseVector yv = spmv(*H(h), xv);
    std::memcpy(y, yv.data(), yv.size() * sizeof(double));
  });
}

int ref_spmv_transpose(void* h, const double* x, double* y) {
  return guarded([&] {
    DenseVector xv(x, x + H(h)->n);
    DenseVector yv = spmv_transpose(*H(h), xv);
    std::memcpy(y, yv.data(), yv.size() * sizeof(double));
  });
}

// x, y: n x k column-major
int ref_spmm(void* h, std::size_t k, const double* x, double* y) {
  return guarded([&] {
    DenseMatrix xm(H(h)->n, k);
    std::memcpy(xm.data().data(), x, xm.data().size() * sizeof(double));
    DenseMatrix ym = spmm(*H(h), xm);
    std::memcpy(y, ym.data().data(), ym.data().size() * sizeof(double));
  });
}

// ---------------------------------------------------------------- RNG
void ref_gaussian_vector(std::uint64_t seed, std::size_t n, double* out) {
  Rng rng(seed);
  DenseVector v = rng.gaussian_vector(n);
  std::memcpy(out, v.data(), n * sizeof(double));
}

// One Rng stream drawing `count` uniforms then `count` uniform_symmetric(1).
void ref_uniform_stream(std::uint64_t seed, std::size_t count, double* u, double* us) {
  Rng rng(seed);
  for (std::size_t i = 0; i < count; ++i) u[i] = rng.uniform();
  for (std::size_t i = 0; i < count; ++i) us[i] = rng.uniform_symmetric(1.0);
}

// ---------------------------------------------------------------- GNN
std::size_t ref_param_count(std::size_t d, std::size_t hidden, std::size_t layers) {
  Rng dummy(0);
  return init_params(dims_of(d, hidden, layers), dummy).total_parameters();
}

int ref_init_params(std::size_t d, std::size_t hidden, std::size_t layers,
                    std::uint64_t seed, double* out) {
  return guarded([&] {
    Rng rng(seed);
    flat(init_params(dims_of(d, hidden, layers), rng), out);
  });
}

int ref_gnn_apply(void* h, std::size_t d, std::size_t hidden, std::size_t layers,
                  const double* params, const double* b, double* out) {
  return guarded([&] {
    const GnnParams p = unflat(d, hidden, layers, params);
    DenseVector bv(b, b + H(h)->n);
    DenseVector o = gnn_apply(p, *H(h), bv);
    std::memcpy(out, o.data(), o.size() * sizeof(double));
  });
}

// Forward then backward for one column: out = M(b), grads = d<out,g>/dtheta.
int ref_gnn_forward_backward(void* h, std::size_t d, std::size_t hidden,
                             std::size_t layers, const double* params,
                             const double* b, const double* gout, double* out,
                             double* grads) {
  return guarded([&] {
    const GnnParams p = unflat(d, hidden, layers, params);
    DenseVector bv(b, b + H(h)->n);
    ForwardResult fr = gnn_forward(p, *H(h), bv);
    std::memcpy(out, fr.out.data(), fr.out.size() * sizeof(double));
    DenseVector gv(gout, gout + H(h)->n);
    flat(gnn_backward(p, *H(h), fr.cache, gv), grads);
  });
}

// out, x, grad: n x B column-major
int ref_l1_residual_loss(void* h, std::size_t batch, const double* out,
                         const double* x, double* loss, double* grad) {
  return guarded([&] {
    const std::size_t n = H(h)->n;
    DenseMatrix om(n, batch), xm(n, batch);
    std::memcpy(om.data().data(), out, n * batch * sizeof(double));
    std::memcpy(xm.data().data(), x, n * batch * sizeof(double));
    L1LossResult r = l1_residual_loss(*H(h), om, xm);
    *loss = r.loss;
    std::memcpy(grad, r.grad.data().data(), n * batch * sizeof(double));
  });
}

// One training step's summed gradient, composed exactly as
// train_preconditioner does it (src/gnn.cpp:426-440): forward per column,
// l1 loss over the batch, backward per column, accumulate in column order.
int ref_batch_loss_grads(void* h, std::size_t d, std::size_t hidden,
                         std::size_t layers, const double* params,
                         std::size_t batch, const double* x, const double* b,
                         double* loss, double* grads, double* out_batch) {
  return guarded([&] {
    const CsrMatrix& a = *H(h);
    const std::size_t n = a.n;
    const GnnParams p = unflat(d, hidden, layers, params);
    DenseMatrix out(n, batch), xm(n, batch);
    std::memcpy(xm.data().data(), x, n * batch * sizeof(double));
    std::vector<ForwardCache> caches(batch);
    for (std::size_t k = 0; k < batch; ++k) {
      DenseVector bk(b + k * n, b + (k + 1) * n);
      ForwardResult fr = gnn_forward(p, a, bk);
      out.set_col(k, fr.out);
      caches[k] = std::move(fr.cache);
    }
    const L1LossResult lr = l1_residual_loss(a, out, xm);
    *loss = lr.loss;
    const std::size_t total = p.total_parameters();
    std::vector<double> acc(total, 0.0), gk(total);
    for (std::size_t k = 0; k < batch; ++k) {
      flat(gnn_backward(p, a, caches[k], lr.grad.col_copy(k)), gk.data());
      for (std::size_t t = 0; t < total; ++t) acc[t] += gk[t];
    }
    std::memcpy(grads, acc.data(), total * sizeof(double));
    if (out_batch) std::memcpy(out_batch, out.data().data(), n * batch * sizeof(double));
  });
}

int ref_adam_step(std::size_t d, std::size_t hidden, std::size_t layers,
                  double* params, const double* grads, double* m1, double* m2,
                  std::size_t* t, double lr) {
  return guarded([&] {
    GnnParams p = unflat(d, hidden, layers, params);
    const GnnParams g = unflat(d, hidden, layers, grads);
    AdamState st = make_adam_state(p);
    const std::size_t total = p.total_parameters();
    st.m1.assign(m1, m1 + total);
    st.m2.assign(m2, m2 + total);
    st.t = *t;
    adam_step(p, g, st, lr);
    flat(p, params);
    std::memcpy(m1, st.m1.data(), total * sizeof(double));
    std::memcpy(m2, st.m2.data(), total * sizeof(double));
    *t = st.t;
  });
}

int ref_train(void* h, std::size_t d, std::size_t hidden, std::size_t layers,
              double lr, std::size_t steps, std::size_t batch,
              std::size_t spectral, std::size_t arnoldi_m, std::uint64_t seed,
              std::size_t monitor_batch, double* best, double* losses,
              double* best_loss) {
  return guarded([&] {
    TrainConfig cfg;
    cfg.lr = lr;
    cfg.steps = steps;
    cfg.batch = batch;
    cfg.spectral_count = spectral;
    cfg.arnoldi_m = arnoldi_m;
    cfg.seed = seed;
    cfg.monitor_batch = monitor_batch;
    cfg.dims = dims_of(d, hidden, layers);
    TrainResult r = train_preconditioner(*H(h), cfg);
    flat(r.best, best);
    std::memcpy(losses, r.loss_history.data(), r.loss_history.size() * sizeof(double));
    *best_loss = r.best_loss;
  });
}

// Gaussian training batch exactly as assemble_batch draws it with
// spectral_count = 0 (src/sampler.cpp:61-83): x_k then b_k = A x_k per column.
int ref_gaussian_batch(void* h, std::uint64_t seed, std::size_t skip_batches,
                       std::size_t batch, double* x, double* b) {
  return guarded([&] {
    const CsrMatrix& a = *H(h);
    Rng rng(seed);
    SpectralSampler unused;
    for (std::size_t s = 0; s < skip_batches; ++s)
      (void)assemble_batch(unused, a, batch, 0, rng);
    TrainingBatch tb = assemble_batch(unused, a, batch, 0, rng);
    std::memcpy(x, tb.x.data().data(), a.n * batch * sizeof(double));
    std::memcpy(b, tb.b.data().data(), a.n * batch * sizeof(double));
  });
}

// ---------------------------------------------------------------- spectral sampler
int ref_jacobi_svd(std::size_t rows, std::size_t cols, const double* a, double* u, double* s,
                   double* v) {
  return guarded([&] {
    DenseMatrix m(rows, cols);
    std::memcpy(m.data().data(), a, rows * cols * sizeof(double));
    SvdResult r = jacobi_svd(m);
    std::memcpy(u, r.u.data().data(), rows * cols * sizeof(double));
    std::memcpy(s, r.s.data(), cols * sizeof(double));
    std::memcpy(v, r.v.data().data(), cols * cols * sizeof(double));
  });
}

// build_spectral_sampler (src/sampler.cpp:10-39); outputs sized for m.
int ref_spectral_sampler(void* h, std::size_t m, std::uint64_t seed, double* v, double* zsv,
                         double* s, std::size_t* k, std::size_t* m_eff) {
  return guarded([&] {
    SpectralSampler sp = build_spectral_sampler(*H(h), m, seed);
    *k = sp.m;
    *m_eff = sp.m_eff;
    std::memcpy(v, sp.v.data().data(), sp.v.data().size() * sizeof(double));
    std::memcpy(zsv, sp.zm_sv.data().data(), sp.zm_sv.data().size() * sizeof(double));
    std::memcpy(s, sp.s.data(), sp.s.size() * sizeof(double));
  });
}

// assemble_batch (src/sampler.cpp:68-83) from a freshly built sampler:
// `skip` batches from Rng(seed) are drawn and dropped, then one is returned.
int ref_assemble_batch(void* h, std::size_t m, std::uint64_t sampler_seed, std::uint64_t seed,
                       std::size_t skip_batches, std::size_t batch, std::size_t spectral,
                       double* x, double* b) {
  return guarded([&] {
    const CsrMatrix& a = *H(h);
    SpectralSampler sp = build_spectral_sampler(a, m, sampler_seed);
    Rng rng(seed);
    for (std::size_t q = 0; q < skip_batches; ++q) (void)assemble_batch(sp, a, batch, spectral, rng);
    TrainingBatch tb = assemble_batch(sp, a, batch, spectral, rng);
    std::memcpy(x, tb.x.data().data(), a.n * batch * sizeof(double));
    std::memcpy(b, tb.b.data().data(), a.n * batch * sizeof(double));
  });
}

// ---------------------------------------------------------------- Krylov
int ref_hessenberg_lstsq(std::size_t k, const double* hbar, double beta,
                         double* y, double* tracked, int* singular) {
  return guarded([&] {
    DenseMatrix hm(k + 1, k);
    std::memcpy(hm.data().data(), hbar, (k + 1) * k * sizeof(double));
    LstsqResult r = hessenberg_lstsq(hm, beta);
    for (std::size_t i = 0; i < r.y.size(); ++i) y[i] = r.y[i];
    *tracked = r.tracked_res;
    *singular = r.singular ? 1 : 0;
  });
}

// precond: 0 none, 1 gnp (dims + params), 2 dense n x n col-major operator,
// 3 identity operator, 4 jacobi.
static std::unique_ptr<FlexibleOperator> make_op(void* h, int kind, std::size_t d,
                                                 std::size_t hidden, std::size_t layers,
                                                 const double* params,
                                                 GnnParams* keep) {
  switch (kind) {
    case 0: return nullptr;
    case 1:
      *keep = unflat(d, hidden, layers, params);
      return apply_preconditioner(*keep, *H(h));
    case 2: return std::make_unique<DenseColMajorOperator>(H(h)->n, params);
    case 3: return std::make_unique<IdentityOp>();
    case 4: return jacobi_build(*H(h));
    default: throw std::invalid_argument("unknown operator kind");
  }
}

int ref_arnoldi_cycle(void* h, const double* r0, std::size_t m, int kind,
                      std::size_t d, std::size_t hidden, std::size_t layers,
                      const double* params, double* v, double* hbar, double* z,
                      std::size_t* steps, int* breakdown) {
  return guarded([&] {
    GnnParams keep;
    auto op = make_op(h, kind, d, hidden, layers, params, &keep);
    DenseVector r(r0, r0 + H(h)->n);
    ArnoldiResult ar = arnoldi_cycle(*H(h), r, m, op.get());
    *steps = ar.fact.steps;
    *breakdown = ar.fact.breakdown ? 1 : 0;
    std::memcpy(v, ar.fact.v.data().data(), ar.fact.v.data().size() * sizeof(double));
    std::memcpy(hbar, ar.fact.hbar.data().data(), ar.fact.hbar.data().size() * sizeof(double));
    std::memcpy(z, ar.z.data().data(), ar.z.data().size() * sizeof(double));
  });
}

// Returns the SolveStatus as int (converged=0 ... breakdown_exact=4), or -1.
int ref_fgmres(void* h, const double* b, int kind, std::size_t d, std::size_t hidden,
               std::size_t layers, const double* params, const double* x0,
               double rtol, std::size_t maxiters, std::size_t restart,
               double timeout_secs, double* x_out, std::size_t* hist_iter,
               double* hist_rel, double* hist_t, std::size_t hist_cap,
               std::size_t* hist_len) {
  int status = -1;
  int rc = guarded([&] {
    GnnParams keep;
    auto op = make_op(h, kind, d, hidden, layers, params, &keep);
    const std::size_t n = H(h)->n;
    SolveConfig cfg;
    cfg.rtol = rtol;
    cfg.maxiters = maxiters;
    cfg.restart = restart;
    if (timeout_secs >= 0.0) cfg.timeout_secs = timeout_secs;
    DenseVector bv(b, b + n), xv(x0, x0 + n);
    SolveOutcome o = fgmres_solve(*H(h), bv, op.get(), xv, cfg);
    std::memcpy(x_out, o.x.data(), n * sizeof(double));
    const std::size_t len = std::min(hist_cap, o.history.size());
    for (std::size_t i = 0; i < len; ++i) {
      hist_iter[i] = o.history[i].iteration;
      hist_rel[i] = o.history[i].relres;
      hist_t[i] = o.history[i].elapsed_secs;
    }
    *hist_len = o.history.size();
    status = status_code(o.status);
  });
  return rc == 0 ? status : -1;
}

// ---------------------------------------------------------------- checkpoints
int ref_save_checkpoint(const char* path, std::size_t d, std::size_t hidden,
                        std::size_t layers, const double* params, void* h) {
  return guarded([&] {
    const GnnParams p = unflat(d, hidden, layers, params);
    save_checkpoint_file(path, p, matrix_meta_of(*H(h)));
  });
}

// dims_out[3], meta_out = {n, nnz, hash}; params sized by the caller after a
// first call with params == nullptr.
int ref_load_checkpoint(const char* path, std::size_t* dims_out,
                        std::uint64_t* meta_out, double* params) {
  return guarded([&] {
    Checkpoint c = load_checkpoint_file(path);
    dims_out[0] = c.params.dims.d;
    dims_out[1] = c.params.dims.hidden;
    dims_out[2] = c.params.dims.layers;
    meta_out[0] = c.meta.n;
    meta_out[1] = c.meta.nnz;
    meta_out[2] = c.meta.hash;
    if (params) flat(c.params, params);
  });
}

// ---------------------------------------------------------------- timing
// Wall seconds of `reps` gnn_apply calls (the CPU baseline leg of bench.py).
double ref_time_gnn_apply(void* h, std::size_t d, std::size_t hidden,
                          std::size_t layers, const double* params,
                          const double* b, std::size_t reps, double* out) {
  const GnnParams p = unflat(d, hidden, layers, params);
  DenseVector bv(b, b + H(h)->n), o;
  const auto t0 = std::chrono::steady_clock::now();
  for (std::size_t r = 0; r < reps; ++r) o = gnn_apply(p, *H(h), bv);
  const auto t1 = std::chrono::steady_clock::now();
  if (out) std::memcpy(out, o.data(), o.size() * sizeof(double));
  return std::chrono::duration<double>(t1 - t0).count();
}

}  // extern "C"
