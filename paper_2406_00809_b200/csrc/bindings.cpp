// Python module `_gnp` for the B200 path.  Same names, kwargs and defaults as
// the reference bindings (/root/reference/proj/bindings/module.cpp:43-129) so
// `import paper_2406_00809_b200 as gnp` drops in for `import gnp`; new
// functionality is only added as new kwargs / new functions.  All compute goes
// through the C ABI (include/gnpc.h) via the gnp_gpu C++ API.
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <cmath>
#include <fstream>
#include <iomanip>
#include <sstream>

#include "api/gnp_gpu.hpp"

namespace py = pybind11;
using namespace gnp_gpu;

namespace {

// Jacobi z_i = v_i / a_ii (src/baselines.cpp:10-25, 89-100), host operator.
class JacobiOperator final : public FlexibleOperator {
 public:
  explicit JacobiOperator(const CsrMatrix& a) {
    const auto rp = a.row_ptr();
    const auto ci = a.col_idx();
    const auto v = a.values();
    inv_.assign(a.n(), 0.0);
    for (std::size_t i = 0; i < a.n(); ++i) {
      double d = 0.0;
      for (int64_t k = rp[i]; k < rp[i + 1]; ++k)
        if (static_cast<std::size_t>(ci[k]) == i) d = v[k];
      if (d == 0.0) throw std::invalid_argument("jacobi: zero diagonal entry");
      inv_[i] = 1.0 / d;
    }
  }
  DenseVector apply(const DenseVector& x) const override {
    DenseVector z(x.size());
    for (std::size_t i = 0; i < x.size(); ++i) z[i] = x[i] * inv_[i];
    return z;
  }
  std::string name() const override { return "jacobi"; }

 private:
  std::vector<double> inv_;
};

std::unique_ptr<FlexibleOperator> build_named(const CsrMatrix& a, const std::string& name,
                                              const GnnParams* params) {
  if (name == "none") return nullptr;
  if (name == "jacobi") return std::make_unique<JacobiOperator>(a);
  if (name == "gnp") {
    if (!params) throw std::invalid_argument("gnp requires trained params");
    return apply_preconditioner(*params, a);
  }
  if (name == "gmres" || name == "ilu0")
    throw std::invalid_argument("preconditioner '" + name +
                                "' is outside this build's scope (GNP hot path only)");
  throw std::invalid_argument("unknown preconditioner: " + name);
}

py::dict outcome_to_dict(const SolveOutcome& o) {
  py::dict d;
  d["status"] = to_string(o.status);
  d["x"] = o.x;
  py::list hist;
  for (const auto& e : o.history) hist.append(py::make_tuple(e.iteration, e.relres, e.elapsed_secs));
  d["history"] = hist;
  d["reorth_steps"] = o.reorth_steps;
  return d;
}

double log10_clamped(double r) { return std::log10(std::max(r, 1e-300)); }

}  // namespace

PYBIND11_MODULE(_gnp, m) {
  m.doc() = "B200 FGMRES with the graph neural preconditioner (device path over libgnpc)";

  py::class_<CsrMatrix>(m, "CsrMatrix")
      .def_property_readonly("n", &CsrMatrix::n)
      .def_property_readonly("nnz", &CsrMatrix::nnz)
      .def_property_readonly("row_ptr", &CsrMatrix::row_ptr)
      .def_property_readonly("col_idx", &CsrMatrix::col_idx)
      .def_property_readonly("values", &CsrMatrix::values)
      .def("__repr__", [](const CsrMatrix& a) {
        return "<CsrMatrix n=" + std::to_string(a.n()) + " nnz=" + std::to_string(a.nnz()) + ">";
      });

  py::class_<GnnParams>(m, "GnnParams")
      .def_property_readonly("dims",
                             [](const GnnParams& p) {
                               return py::make_tuple(p.dims.d, p.dims.hidden, p.dims.layers);
                             })
      .def_property_readonly("flat", [](const GnnParams& p) { return p.flat; })
      .def("total_parameters", &GnnParams::total_parameters);

  m.def("read_matrix_market", &read_matrix_market_file, py::arg("path"));
  m.def(
      "write_matrix_market",
      [](const std::string& path, const CsrMatrix& a) {
        std::ofstream f(path);
        if (!f) throw std::runtime_error("cannot open " + path + " for writing");
        const auto rp = a.row_ptr();
        const auto ci = a.col_idx();
        const auto v = a.values();
        f << "%%MatrixMarket matrix coordinate real general\n";
        f << a.n() << ' ' << a.n() << ' ' << a.nnz() << '\n';
        f.precision(17);
        for (std::size_t i = 0; i < a.n(); ++i)
          for (int64_t k = rp[i]; k < rp[i + 1]; ++k)
            f << i + 1 << ' ' << ci[k] + 1 << ' ' << v[k] << '\n';
      },
      py::arg("path"), py::arg("matrix"));
  m.def("gen_convection_diffusion", &gen_convection_diffusion, py::arg("grid"),
        py::arg("convection") = 0.5);
  m.def("gen_random_nonsymmetric", &gen_random_nonsymmetric, py::arg("n"),
        py::arg("offdiag_per_row") = 8, py::arg("dominance") = 1.5, py::arg("seed") = 0);
  m.def("gershgorin_gamma", &gershgorin_gamma);
  m.def("prescale", &prescale, py::arg("matrix"), py::arg("gamma"));
  m.def("spmv", &spmv, py::arg("matrix"), py::arg("x"));

  m.def(
      "solve",
      [](const CsrMatrix& a, const DenseVector& b, const std::string& precond,
          const GnnParams* params, double rtol, std::size_t maxiters, std::size_t restart,
          std::optional<double> timeout_secs) {
        SolveConfig cfg;
        cfg.rtol = rtol;
        cfg.maxiters = maxiters;
        cfg.restart = restart;
        cfg.timeout_secs = timeout_secs;
        const auto op = build_named(a, precond, params);
        SolveOutcome o;
        {
          py::gil_scoped_release nogil;
          o = fgmres_solve(a, b, op.get(), DenseVector(a.n(), 0.0), cfg);
        }
        return outcome_to_dict(o);
      },
      py::arg("matrix"), py::arg("b"), py::arg("precond") = "none", py::arg("params") = nullptr,
      py::arg("rtol") = 1e-8, py::arg("maxiters") = 100, py::arg("restart") = 10,
      py::arg("timeout_secs") = py::none());

  m.def(
      "train",
      [](const CsrMatrix& a, std::size_t steps, std::size_t batch, std::size_t spectral, double lr,
         std::size_t arnoldi_m, std::uint64_t seed, std::size_t d, std::size_t hidden,
         std::size_t layers, std::size_t monitor_batch) {
        TrainConfig cfg;
        cfg.steps = steps;
        cfg.batch = batch;
        cfg.spectral_count = spectral;
        cfg.lr = lr;
        cfg.arnoldi_m = arnoldi_m;
        cfg.seed = seed;
        cfg.dims = {d, hidden, layers};
        cfg.monitor_batch = monitor_batch;
        TrainResult res;
        {
          py::gil_scoped_release nogil;
          res = train_preconditioner(a, cfg);
        }
        return py::make_tuple(res.best, res.loss_history);
      },
      py::arg("matrix"), py::arg("steps") = 2000, py::arg("batch") = 16, py::arg("spectral") = 8,
      py::arg("lr") = 1e-3, py::arg("arnoldi_m") = 40, py::arg("seed") = 0, py::arg("d") = 16,
      py::arg("hidden") = 32, py::arg("layers") = 8, py::arg("monitor_batch") = 16);

  m.def("save_checkpoint", [](const std::string& path, const GnnParams& p, const CsrMatrix& a) {
    save_checkpoint_file(path, p, a);
  });
  m.def("load_checkpoint",
        [](const std::string& path) { return load_checkpoint_file(path).params; });

  using Hist = std::vector<std::tuple<std::size_t, double, double>>;
  // iter_auc / time_auc (src/bench.cpp:34-51)
  m.def(
      "iter_auc",
      [](const Hist& h, double rtol) {
        if (h.empty()) throw std::invalid_argument("iter_auc: empty history");
        const double lr = std::log10(rtol);
        double s = 0.0;
        for (const auto& e : h) s += log10_clamped(std::get<1>(e)) - lr;
        return s;
      },
      py::arg("history"), py::arg("rtol") = 1e-8);
  m.def(
      "time_auc",
      [](const Hist& h, double rtol) {
        if (h.size() < 2) return 0.0;
        const double lr = std::log10(rtol);
        double s = 0.0;
        for (std::size_t i = 1; i < h.size(); ++i)
          s += (log10_clamped(std::get<1>(h[i])) - lr) * (std::get<2>(h[i]) - std::get<2>(h[i - 1]));
        return s;
      },
      py::arg("history"), py::arg("rtol") = 1e-8);

  // ---- additions (not in the reference module)
  m.def(
      "csr_from_triplets",
      [](std::size_t n, const std::vector<std::size_t>& r, const std::vector<std::size_t>& c,
         const std::vector<double>& v) { return csr_from_triplets(n, r, c, v); },
      py::arg("n"), py::arg("rows"), py::arg("cols"), py::arg("vals"));
  m.def("csr_from_arrays", &csr_from_arrays, py::arg("n"), py::arg("row_ptr"), py::arg("col_idx"),
        py::arg("values"));
  m.def("generate", &generate, py::arg("kind"), py::arg("size"), py::arg("p0") = 0.0,
        py::arg("p1") = 0.0, py::arg("seed") = 0);
  m.def("transpose", &transpose);
  m.def("csr_content_hash", &csr_content_hash);
  m.def(
      "init_params",
      [](std::size_t d, std::size_t hidden, std::size_t layers, std::uint64_t seed) {
        return init_params({d, hidden, layers}, seed);
      },
      py::arg("d") = 16, py::arg("hidden") = 32, py::arg("layers") = 8, py::arg("seed") = 0);
  m.def(
      "params_from_flat",
      [](const std::vector<double>& flat, std::size_t d, std::size_t hidden, std::size_t layers) {
        GnnParams p;
        p.dims = {d, hidden, layers};
        if (flat.size() != param_count(p.dims))
          throw std::invalid_argument("params_from_flat: length does not match dims");
        p.flat = flat;
        return p;
      },
      py::arg("flat"), py::arg("d") = 16, py::arg("hidden") = 32, py::arg("layers") = 8);
  m.def(
      "gnn_apply",
      [](const CsrMatrix& a, const GnnParams& p, const DenseVector& b) {
        py::gil_scoped_release nogil;
        return gnn_apply(p, a, b);
      },
      py::arg("matrix"), py::arg("params"), py::arg("b"));
  m.def("abi_version", [] { return gnpc_abi_version(); });
  m.def("launch_count", [] {
    int64_t c = 0;
    check(gnpc_launch_count(&c));
    return c;
  });
}
