// gnp_gpu: the reference's C++ API (namespace gnp, /root/reference/proj/include/gnp)
// restated over the C ABI (include/gnpc.h) so that a caller of the CPU
// library can switch to the B200 path by changing the namespace.  Header-only.
//   CsrMatrix & sparse helpers ...... include/gnp/csr.hpp:13-44
//   FlexibleOperator, SolveConfig,
//   SolveOutcome, fgmres_solve ...... include/gnp/krylov.hpp:15-86
//   GnnDims, GnnParams, gnn_apply,
//   apply_preconditioner, training,
//   checkpoints ...................... include/gnp/gnn.hpp:16-146
// Errors are rethrown as the reference's exception types
// (std::invalid_argument / std::out_of_range / std::runtime_error).
#pragma once

#include <algorithm>
#include <cstdint>
#include <exception>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../include/gnpc.h"

namespace gnp_gpu {

using DenseVector = std::vector<double>;

inline void check(int rc) {
  if (rc == GNPC_OK) return;
  const std::string msg = gnpc_last_error();
  switch (rc) {
    case GNPC_EINVAL: throw std::invalid_argument(msg);
    case GNPC_ERANGE: throw std::out_of_range(msg);
    default: throw std::runtime_error(msg);
  }
}

// ---------------------------------------------------------------- CSR
class CsrMatrix {
 public:
  CsrMatrix() = default;
  explicit CsrMatrix(gnpc_csr h) : h_(h, [](gnpc_csr p) { gnpc_csr_destroy(p); }) {}
  gnpc_csr handle() const { return h_.get(); }
  std::size_t n() const {
    int64_t n = 0;
    check(gnpc_csr_info(h_.get(), &n, nullptr));
    return static_cast<std::size_t>(n);
  }
  std::size_t nnz() const {
    int64_t z = 0;
    check(gnpc_csr_info(h_.get(), nullptr, &z));
    return static_cast<std::size_t>(z);
  }
  std::vector<int64_t> row_ptr() const {
    std::vector<int64_t> v(n() + 1);
    check(gnpc_csr_export(h_.get(), v.data(), nullptr, nullptr));
    return v;
  }
  std::vector<int64_t> col_idx() const {
    std::vector<int64_t> v(nnz());
    check(gnpc_csr_export(h_.get(), nullptr, v.data(), nullptr));
    return v;
  }
  std::vector<double> values() const {
    std::vector<double> v(nnz());
    check(gnpc_csr_export(h_.get(), nullptr, nullptr, v.data()));
    return v;
  }

 private:
  std::shared_ptr<gnpc_csr_s> h_;
};

inline CsrMatrix csr_from_triplets(std::size_t n, const std::vector<std::size_t>& rows,
                                   const std::vector<std::size_t>& cols,
                                   const std::vector<double>& vals) {
  std::vector<int64_t> r(rows.begin(), rows.end()), c(cols.begin(), cols.end());
  if (r.size() != vals.size() || c.size() != vals.size())
    throw std::invalid_argument("triplet arrays must have equal length");
  gnpc_csr h = nullptr;
  check(gnpc_csr_from_triplets(static_cast<int64_t>(n), static_cast<int64_t>(vals.size()),
                               r.data(), c.data(), vals.data(), &h));
  return CsrMatrix(h);
}
inline CsrMatrix csr_from_arrays(std::size_t n, const std::vector<int64_t>& rp,
                                 const std::vector<int64_t>& ci, const std::vector<double>& v) {
  if (rp.size() != n + 1) throw std::invalid_argument("csr: row_ptr must have n+1 entries");
  if (ci.size() != v.size()) throw std::invalid_argument("csr: col_idx/values length mismatch");
  if (static_cast<std::size_t>(rp.back()) != v.size())
    throw std::invalid_argument("csr: row_ptr[n] must equal nnz");
  gnpc_csr h = nullptr;
  check(gnpc_csr_create(static_cast<int64_t>(n), rp.data(), ci.data(), v.data(), &h));
  return CsrMatrix(h);
}
inline CsrMatrix generate(const std::string& kind, int64_t size, double p0, double p1,
                          uint64_t seed) {
  gnpc_csr h = nullptr;
  check(gnpc_csr_generate(kind.c_str(), size, p0, p1, seed, &h));
  return CsrMatrix(h);
}
inline CsrMatrix gen_convection_diffusion(std::size_t grid, double convection) {
  return generate("convection_diffusion", static_cast<int64_t>(grid), convection, 0.0, 0);
}
inline CsrMatrix gen_random_nonsymmetric(std::size_t n, std::size_t offdiag, double dominance,
                                         uint64_t seed) {
  return generate("random_nonsymmetric", static_cast<int64_t>(n), static_cast<double>(offdiag),
                  dominance, seed);
}
inline CsrMatrix read_matrix_market_file(const std::string& path) {
  gnpc_csr h = nullptr;
  check(gnpc_csr_read_matrix_market(path.c_str(), &h));
  return CsrMatrix(h);
}
inline double gershgorin_gamma(const CsrMatrix& a) {
  double g = 0.0;
  check(gnpc_csr_gershgorin_gamma(a.handle(), &g));
  return g;
}
inline CsrMatrix prescale(const CsrMatrix& a, double gamma) {
  gnpc_csr h = nullptr;
  check(gnpc_csr_prescale(a.handle(), gamma, &h));
  return CsrMatrix(h);
}
inline CsrMatrix transpose(const CsrMatrix& a) {
  gnpc_csr h = nullptr;
  check(gnpc_csr_transpose(a.handle(), &h));
  return CsrMatrix(h);
}
inline uint64_t csr_content_hash(const CsrMatrix& a) {
  uint64_t h = 0;
  check(gnpc_csr_hash(a.handle(), &h));
  return h;
}
inline DenseVector spmv(const CsrMatrix& a, const DenseVector& x) {
  if (x.size() != a.n()) throw std::invalid_argument("spmv: dimension mismatch");
  DenseVector y(x.size());
  check(gnpc_spmv(a.handle(), x.data(), y.data()));
  return y;
}

// ---------------------------------------------------------------- GNP
struct GnnDims {
  std::size_t d = 16;
  std::size_t hidden = 32;
  std::size_t layers = 8;
};

// Flat parameters in the reference's checkpoint order (src/gnn.cpp:40-55).
struct GnnParams {
  GnnDims dims;
  std::vector<double> flat;
  std::size_t total_parameters() const { return flat.size(); }
};

inline std::size_t param_count(const GnnDims& d) {
  int64_t c = 0;
  check(gnpc_param_count(static_cast<int64_t>(d.d), static_cast<int64_t>(d.hidden),
                         static_cast<int64_t>(d.layers), &c));
  return static_cast<std::size_t>(c);
}

// init_params(dims, Rng(seed)) (src/gnn.cpp:92-118).
inline GnnParams init_params(const GnnDims& dims, uint64_t seed) {
  GnnParams p;
  p.dims = dims;
  p.flat.resize(param_count(dims));
  check(gnpc_init_params(static_cast<int64_t>(dims.d), static_cast<int64_t>(dims.hidden),
                         static_cast<int64_t>(dims.layers), seed, p.flat.data()));
  return p;
}

class FlexibleOperator {
 public:
  virtual ~FlexibleOperator() = default;
  virtual DenseVector apply(const DenseVector& v) const = 0;
  virtual std::string name() const = 0;
};

// The device GNP bound to Â (GnnOperator, src/gnn.cpp:455-467).  Borrows the
// matrix like the reference; keeps a shared handle so it cannot dangle.
class GnpOperator final : public FlexibleOperator {
 public:
  GnpOperator(const GnnParams& p, const CsrMatrix& ahat) : ahat_(ahat), n_(ahat.n()) {
    if (p.flat.size() != param_count(p.dims))
      throw std::invalid_argument("gnp: parameter count does not match dims");
    gnpc_model m = nullptr;
    check(gnpc_model_create(ahat.handle(), static_cast<int64_t>(p.dims.d),
                            static_cast<int64_t>(p.dims.hidden),
                            static_cast<int64_t>(p.dims.layers), p.flat.data(), &m));
    m_.reset(m, [](gnpc_model q) { gnpc_model_destroy(q); });
  }
  DenseVector apply(const DenseVector& v) const override {
    if (v.size() != n_) throw std::invalid_argument("gnn_forward: dimension mismatch");
    DenseVector out(n_);
    check(gnpc_apply(m_.get(), v.data(), out.data()));
    return out;
  }
  std::string name() const override { return "gnp"; }
  gnpc_model model() const { return m_.get(); }
  const CsrMatrix& matrix() const { return ahat_; }

 private:
  CsrMatrix ahat_;
  std::size_t n_;
  std::shared_ptr<gnpc_model_s> m_;
};

inline std::unique_ptr<FlexibleOperator> apply_preconditioner(const GnnParams& p,
                                                              const CsrMatrix& ahat) {
  return std::make_unique<GnpOperator>(p, ahat);
}

inline DenseVector gnn_apply(const GnnParams& p, const CsrMatrix& ahat, const DenseVector& b) {
  return GnpOperator(p, ahat).apply(b);
}

// ---------------------------------------------------------------- Krylov
struct SolveConfig {
  double rtol = 1e-8;
  std::size_t maxiters = 100;
  std::size_t restart = 10;
  std::optional<double> timeout_secs;
};
struct HistoryEntry {
  std::size_t iteration;
  double relres;
  double elapsed_secs;
};
using ConvergenceHistory = std::vector<HistoryEntry>;
enum class SolveStatus { converged, maxiters, timeout, solution_failure, breakdown_exact };
inline std::string to_string(SolveStatus s) {
  switch (s) {
    case SolveStatus::converged: return "converged";
    case SolveStatus::maxiters: return "maxiters";
    case SolveStatus::timeout: return "timeout";
    case SolveStatus::solution_failure: return "solution_failure";
    case SolveStatus::breakdown_exact: return "breakdown_exact";
  }
  return "unknown";
}
struct SolveOutcome {
  DenseVector x;
  ConvergenceHistory history;
  SolveStatus status = SolveStatus::maxiters;
  std::size_t reorth_steps = 0;  // steps that took the second MGS pass
};

namespace detail {
struct HostOpCtx {
  const FlexibleOperator* op;
  std::exception_ptr err;
};
// Exceptions never cross the C ABI: they are parked here and rethrown.
inline int host_op_trampoline(void* ctx, const double* in, double* out, int64_t n) {
  auto* c = static_cast<HostOpCtx*>(ctx);
  try {
    const DenseVector z = c->op->apply(DenseVector(in, in + n));
    if (static_cast<int64_t>(z.size()) != n)
      throw std::invalid_argument("preconditioner output length mismatch");
    std::copy(z.begin(), z.end(), out);
    return 0;
  } catch (...) {
    c->err = std::current_exception();
    return 1;
  }
}
}  // namespace detail

// fgmres_solve (src/krylov.cpp:175-277): device GNP operators and the
// unpreconditioned case run fully on the device; any other FlexibleOperator
// is called on the host once per Arnoldi step.
inline SolveOutcome fgmres_solve(const CsrMatrix& a, const DenseVector& b,
                                 const FlexibleOperator* precond, const DenseVector& x0,
                                 const SolveConfig& cfg) {
  const std::size_t n = a.n();
  if (b.size() != n || x0.size() != n) throw std::invalid_argument("fgmres: dimension mismatch");
  gnpc_solve_config c{cfg.rtol, static_cast<int64_t>(cfg.maxiters),
                      static_cast<int64_t>(cfg.restart),
                      cfg.timeout_secs ? *cfg.timeout_secs : -1.0};
  const std::size_t cap = cfg.maxiters + 2;
  std::vector<int64_t> it(cap);
  std::vector<double> rel(cap), el(cap);
  gnpc_history h{it.data(), rel.data(), el.data(), static_cast<int64_t>(cap), 0, 0};
  SolveOutcome out;
  out.x.resize(n);
  int status = 0;
  const auto* gop = dynamic_cast<const GnpOperator*>(precond);
  if (precond == nullptr || gop != nullptr) {
    check(gnpc_fgmres(a.handle(), gop ? gop->model() : nullptr, b.data(), x0.data(), &c,
                      out.x.data(), &h, &status));
  } else {
    detail::HostOpCtx ctx{precond, nullptr};
    const int rc = gnpc_fgmres_host_operator(a.handle(), detail::host_op_trampoline, &ctx,
                                             b.data(), x0.data(), &c, out.x.data(), &h, &status);
    if (ctx.err) std::rethrow_exception(ctx.err);
    check(rc);
  }
  const std::size_t len = std::min<std::size_t>(static_cast<std::size_t>(h.length), cap);
  for (std::size_t i = 0; i < len; ++i)
    out.history.push_back({static_cast<std::size_t>(it[i]), rel[i], el[i]});
  out.status = static_cast<SolveStatus>(status);
  out.reorth_steps = static_cast<std::size_t>(h.reorth);
  return out;
}

inline SolveOutcome gmres_solve(const CsrMatrix& a, const DenseVector& b, const SolveConfig& cfg) {
  return fgmres_solve(a, b, nullptr, DenseVector(a.n(), 0.0), cfg);
}

// ---------------------------------------------------------------- training
struct TrainConfig {
  double lr = 1e-3;
  std::size_t steps = 2000;
  std::size_t batch = 16;
  std::size_t spectral_count = 8;
  std::size_t arnoldi_m = 40;
  std::uint64_t seed = 0;
  std::size_t monitor_batch = 16;
  GnnDims dims;
};
struct TrainResult {
  GnnParams best;
  std::vector<double> loss_history;
  double best_loss = 0.0;
};
inline TrainResult train_preconditioner(const CsrMatrix& a, const TrainConfig& cfg) {
  gnpc_train_config c{cfg.lr,
                      static_cast<int64_t>(cfg.steps),
                      static_cast<int64_t>(cfg.batch),
                      static_cast<int64_t>(cfg.spectral_count),
                      static_cast<int64_t>(cfg.arnoldi_m),
                      cfg.seed,
                      static_cast<int64_t>(cfg.monitor_batch),
                      static_cast<int64_t>(cfg.dims.d),
                      static_cast<int64_t>(cfg.dims.hidden),
                      static_cast<int64_t>(cfg.dims.layers)};
  TrainResult r;
  r.best.dims = cfg.dims;
  r.best.flat.resize(param_count(cfg.dims));
  r.loss_history.resize(cfg.steps + 1);
  check(gnpc_train_preconditioner(a.handle(), &c, r.best.flat.data(), r.loss_history.data(),
                                  &r.best_loss));
  return r;
}

// ---------------------------------------------------------------- checkpoints
struct MatrixMeta {
  std::size_t n = 0, nnz = 0;
  std::uint64_t hash = 0;
};
struct Checkpoint {
  GnnParams params;
  MatrixMeta meta;
};
inline void save_checkpoint_file(const std::string& path, const GnnParams& p, const CsrMatrix& a) {
  check(gnpc_checkpoint_save(path.c_str(), static_cast<int64_t>(p.dims.d),
                             static_cast<int64_t>(p.dims.hidden),
                             static_cast<int64_t>(p.dims.layers), p.flat.data(), a.handle()));
}
inline Checkpoint load_checkpoint_file(const std::string& path) {
  int64_t dims[3];
  uint64_t meta[3];
  check(gnpc_checkpoint_load(path.c_str(), dims, meta, nullptr));
  Checkpoint c;
  c.params.dims = {static_cast<std::size_t>(dims[0]), static_cast<std::size_t>(dims[1]),
                   static_cast<std::size_t>(dims[2])};
  c.params.flat.resize(param_count(c.params.dims));
  check(gnpc_checkpoint_load(path.c_str(), dims, meta, c.params.flat.data()));
  c.meta = {static_cast<std::size_t>(meta[0]), static_cast<std::size_t>(meta[1]), meta[2]};
  return c;
}

}  // namespace gnp_gpu
