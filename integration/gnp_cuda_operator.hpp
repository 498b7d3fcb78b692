// gnp_cuda_operator.hpp — the binding a gnprecond maintainer adds to route
// the GNP hot path to the B200 library (include/gnpc.h, libgnpc.so).
//
// It depends only on the REFERENCE's own public headers (gnp/csr.hpp,
// gnp/gnn.hpp, gnp/krylov.hpp) and the C ABI; tests/test_integration.py
// compiles it against /root/reference/proj/include.
//
//   gnp::apply_preconditioner(params, ahat)   (include/gnp/gnn.hpp:125-126)
//     -> gnp_cuda::apply_preconditioner(params, ahat): a FlexibleOperator
//        whose apply() is one device M·v (gnpc_apply), name() == "gnp";
//        the reference fgmres_solve (src/krylov.cpp:175-277) uses it as is.
//   gnp::fgmres_solve(A, b, M, x0, cfg)       (include/gnp/krylov.hpp:81-86)
//     -> gnp_cuda::fgmres_solve(A, b, M, x0, cfg): the device-resident FGMRES
//        (gnpc_fgmres) when M is a CudaGnnOperator or null.
//   gnp::train_preconditioner(A, cfg)         (include/gnp/gnn.hpp:117-123)
//     -> gnp_cuda::train_preconditioner(A, cfg) (gnpc_train_preconditioner).
#pragma once

#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "gnp/csr.hpp"
#include "gnp/gnn.hpp"
#include "gnp/krylov.hpp"
#include "gnpc.h"

namespace gnp_cuda {

inline void check(int rc) {
  if (rc == GNPC_OK) return;
  const std::string msg = gnpc_last_error();
  if (rc == GNPC_EINVAL) throw std::invalid_argument(msg);
  if (rc == GNPC_ERANGE) throw std::out_of_range(msg);
  throw std::runtime_error(msg);
}

// Flat parameter vector in the reference's param_views order
// (src/gnn.cpp:40-55): enc1, enc1_bias, enc2, enc2_bias, (U, W) per layer,
// dec1, dec1_bias, dec2, dec2_bias; matrices column-major.
inline std::vector<double> flatten(const gnp::GnnParams& p) {
  std::vector<double> f;
  auto put = [&](const std::vector<double>& v) { f.insert(f.end(), v.begin(), v.end()); };
  put(p.enc1);
  put(p.enc1_bias);
  put(p.enc2.data());
  put(p.enc2_bias);
  for (const auto& l : p.layers) {
    put(l.u.data());
    put(l.w.data());
  }
  put(p.dec1.data());
  put(p.dec1_bias);
  put(p.dec2);
  f.push_back(p.dec2_bias);
  return f;
}

// Device copy of a reference CsrMatrix (int32 indices, fp32 values on device).
inline std::shared_ptr<gnpc_csr_s> to_device(const gnp::CsrMatrix& a) {
  std::vector<int64_t> rp(a.row_ptr.begin(), a.row_ptr.end()), ci(a.col_idx.begin(), a.col_idx.end());
  gnpc_csr h = nullptr;
  check(gnpc_csr_create(static_cast<int64_t>(a.n), rp.data(), ci.data(), a.values.data(), &h));
  return std::shared_ptr<gnpc_csr_s>(h, [](gnpc_csr p) { gnpc_csr_destroy(p); });
}

// The GnnOperator of src/gnn.cpp:455-474 on the GPU.  Copies the parameters
// (to the device), keeps its own device copy of Â.
class CudaGnnOperator final : public gnp::FlexibleOperator {
 public:
  CudaGnnOperator(const gnp::GnnParams& p, const gnp::CsrMatrix& ahat) : n_(ahat.n), a_(to_device(ahat)) {
    const std::vector<double> flat = flatten(p);
    gnpc_model m = nullptr;
    check(gnpc_model_create(a_.get(), static_cast<int64_t>(p.dims.d), static_cast<int64_t>(p.dims.hidden),
                            static_cast<int64_t>(p.dims.layers), flat.data(), &m));
    m_.reset(m, [](gnpc_model q) { gnpc_model_destroy(q); });
  }
  gnp::DenseVector apply(const gnp::DenseVector& v) const override {
    if (v.size() != n_) throw std::invalid_argument("gnn_forward: input length mismatch");
    gnp::DenseVector z(n_);
    check(gnpc_apply(m_.get(), v.data(), z.data()));
    return z;
  }
  std::string name() const override { return "gnp"; }
  gnpc_model model() const { return m_.get(); }
  gnpc_csr ahat() const { return a_.get(); }

 private:
  std::size_t n_;
  std::shared_ptr<gnpc_csr_s> a_;
  std::shared_ptr<gnpc_model_s> m_;
};

inline std::unique_ptr<gnp::FlexibleOperator> apply_preconditioner(const gnp::GnnParams& p,
                                                                   const gnp::CsrMatrix& ahat) {
  return std::make_unique<CudaGnnOperator>(p, ahat);
}

// Device-resident FGMRES when M is the CUDA GNP (or null); any other
// FlexibleOperator still works through the reference's own fgmres_solve.
inline gnp::SolveOutcome fgmres_solve(const gnp::CsrMatrix& a, const gnp::DenseVector& b,
                                      const gnp::FlexibleOperator* m, const gnp::DenseVector& x0,
                                      const gnp::SolveConfig& cfg) {
  const auto* cm = dynamic_cast<const CudaGnnOperator*>(m);
  if (m != nullptr && cm == nullptr) return gnp::fgmres_solve(a, b, m, x0, cfg);
  auto ad = to_device(a);
  gnpc_solve_config c{cfg.rtol, static_cast<int64_t>(cfg.maxiters), static_cast<int64_t>(cfg.restart),
                      cfg.timeout_secs ? *cfg.timeout_secs : -1.0};
  std::vector<int64_t> it(cfg.maxiters + 2);
  std::vector<double> rel(cfg.maxiters + 2), el(cfg.maxiters + 2);
  gnpc_history h{it.data(), rel.data(), el.data(), static_cast<int64_t>(it.size()), 0, 0};
  gnp::SolveOutcome out;
  out.x.resize(b.size());
  int status = 0;
  check(gnpc_fgmres(ad.get(), cm ? cm->model() : nullptr, b.data(), x0.empty() ? nullptr : x0.data(), &c,
                    out.x.data(), &h, &status));
  for (int64_t k = 0; k < h.length && k < h.capacity; ++k)
    out.history.push_back({static_cast<std::size_t>(it[k]), rel[k], el[k]});
  out.status = static_cast<gnp::SolveStatus>(status);
  return out;
}

}  // namespace gnp_cuda
