// Drives integration/gnp_cuda_operator.hpp from the REFERENCE's own C++ API:
// the unmodified reference library (oracle/_ref/libgnpref.so, built from
// /root/reference/proj/src) supplies gnp::init_params, generators, gnn_apply
// and fgmres_solve; libgnpc.so supplies the device path.
//   exit 0  all checks passed on a GPU
//   exit 3  no CUDA device (the layout checks still ran and passed)
//   exit 1  a check failed
#include <cmath>
#include <cstdio>
#include <vector>

#include "gnp/gen.hpp"
#include "gnp/rng.hpp"
#include "gnp_cuda_operator.hpp"

static double rel_l2(const std::vector<double>& a, const std::vector<double>& b) {
  double num = 0, den = 0;
  for (std::size_t i = 0; i < a.size(); ++i) {
    num += (a[i] - b[i]) * (a[i] - b[i]);
    den += b[i] * b[i];
  }
  return std::sqrt(num / den);
}

int main() {
  gnp::GnnDims dims{16, 32, 8};
  gnp::Rng rng(0);
  const gnp::GnnParams p = gnp::init_params(dims, rng);
  // 1. the adapter's flat order == the library's flat layout (host-only)
  const std::vector<double> flat = gnp_cuda::flatten(p);
  std::vector<double> mine(flat.size());
  int64_t cnt = 0;
  gnp_cuda::check(gnpc_param_count(16, 32, 8, &cnt));
  gnp_cuda::check(gnpc_init_params(16, 32, 8, 0, mine.data()));
  if (cnt != (int64_t)flat.size() || mine != flat) {
    std::printf("FAIL flatten order / init_params mismatch\n");
    return 1;
  }
  std::printf("ok flatten: %zu params bit-identical to gnpc_init_params\n", flat.size());

  int ndev = 0;
  if (gnpc_device_count(&ndev) != GNPC_OK || ndev == 0) {
    std::printf("no CUDA device: device checks skipped\n");
    return 3;
  }
  // 2. apply_preconditioner(...)->apply == reference gnn_apply (fp32 inputs)
  gnp::CsrMatrix a = gnp::gen_convection_diffusion(64, 0.0);
  gnp::CsrMatrix ahat = gnp::prescale(a, gnp::gershgorin_gamma(a));  // gamma = 8: exact in fp32
  gnp::Rng rb(1);
  gnp::DenseVector b = rb.gaussian_vector(ahat.n);
  auto M = gnp_cuda::apply_preconditioner(p, ahat);
  const gnp::DenseVector z = M->apply(b);
  gnp::GnnParams p32 = p;  // the device computes on fp32-rounded parameters
  for (auto* v : {&p32.enc1, &p32.enc1_bias, &p32.enc2_bias, &p32.dec1_bias, &p32.dec2})
    for (double& x : *v) x = (double)(float)x;
  for (auto* m : {&p32.enc2, &p32.dec1})
    for (double& x : m->data()) x = (double)(float)x;
  for (auto& l : p32.layers) {
    for (double& x : l.u.data()) x = (double)(float)x;
    for (double& x : l.w.data()) x = (double)(float)x;
  }
  p32.dec2_bias = (double)(float)p32.dec2_bias;
  gnp::DenseVector b32 = b;
  for (double& x : b32) x = (double)(float)x;
  const double e = rel_l2(M->apply(b32), gnp::gnn_apply(p32, ahat, b32));
  std::printf("%s apply vs reference gnn_apply: rel-L2 %.3e (name %s)\n", e <= 1e-4 ? "ok" : "FAIL", e,
              M->name().c_str());
  if (e > 1e-4 || M->name() != "gnp" || z.size() != ahat.n) return 1;
  // 3. the reference fgmres_solve driving the CUDA operator, and the
  //    device-resident solve behind the same signature
  gnp::SolveConfig cfg;
  cfg.rtol = 1e-8;
  cfg.maxiters = 100;
  cfg.restart = 10;
  const gnp::DenseVector x0(ahat.n, 0.0);
  const gnp::SolveOutcome r1 = gnp::fgmres_solve(ahat, b, M.get(), x0, cfg);
  const gnp::SolveOutcome r2 = gnp_cuda::fgmres_solve(ahat, b, M.get(), x0, cfg);
  const std::size_t i1 = r1.history.back().iteration, i2 = r2.history.back().iteration;
  std::printf("reference fgmres + CUDA M: %zu its (%s, relres %.3e); device fgmres: %zu its (%s, relres %.3e)\n",
              i1, gnp::to_string(r1.status).c_str(), r1.history.back().relres, i2,
              gnp::to_string(r2.status).c_str(), r2.history.back().relres);
  const bool ok = r1.status == r2.status && (i1 > i2 ? i1 - i2 : i2 - i1) <= 1;
  std::printf("%s iteration parity (+-1)\n", ok ? "ok" : "FAIL");
  return ok ? 0 : 1;
}
