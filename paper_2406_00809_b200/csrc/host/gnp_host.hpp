// Host-side (CPU, C++20) half of the B200 GNP path: everything that the
// reference does once per matrix / per model on the host and that the device
// path needs bit-exact: CSR construction, Âᵀ, Gershgorin prescale, content
// hash, seeded RNG, parameter init/layout, GNPCKPT checkpoints, and the
// synthetic generators for BASELINE configs C1–C5.
//
// Reference interfaces mirrored (paths under /root/reference/proj):
//   CsrMatrix, csr_from_triplets, transpose, gershgorin_gamma, prescale,
//   csr_content_hash ................ include/gnp/csr.hpp:13-44, src/csr.cpp
//   Rng ................................ include/gnp/rng.hpp:13-52
//   GnnDims / param order / init ........ include/gnp/gnn.hpp:16-46, src/gnn.cpp:40-118
//   checkpoints ......................... src/gnn.cpp:480-570
//   gen_convection_diffusion,
//   gen_random_nonsymmetric ............. src/gen.cpp:11-69
//   parse_matrix_market ................. src/mmio.cpp:21-87
#pragma once

#include <cmath>
#include <cstdint>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace gnp_b200 {

// ---------------------------------------------------------------- RNG
// mt19937_64 + (x>>11)*2^-53 + Box-Muller with a cached spare: the exact
// stream of the reference Rng (include/gnp/rng.hpp:13-52).
class Rng {
 public:
  explicit Rng(std::uint64_t seed) : gen_(seed) {}
  double uniform() { return static_cast<double>(gen_() >> 11) * 0x1.0p-53; }
  double uniform_symmetric(double bound) { return (2.0 * uniform() - 1.0) * bound; }
  double gaussian() {
    if (have_spare_) {
      have_spare_ = false;
      return spare_;
    }
    double u1 = uniform();
    while (u1 <= 0.0) u1 = uniform();
    const double u2 = uniform();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double theta = 6.283185307179586476925286766559 * u2;
    spare_ = r * std::sin(theta);
    have_spare_ = true;
    return r * std::cos(theta);
  }
  std::vector<double> gaussian_vector(std::size_t n) {
    std::vector<double> v(n);
    for (double& x : v) x = gaussian();
    return v;
  }

 private:
  std::mt19937_64 gen_;
  bool have_spare_ = false;
  double spare_ = 0.0;
};

// ---------------------------------------------------------------- CSR
struct CsrHost {
  std::int64_t n = 0;
  std::vector<std::int64_t> row_ptr;  // n+1
  std::vector<std::int64_t> col_idx;  // strictly increasing within a row
  std::vector<double> values;
  std::int64_t nnz() const { return static_cast<std::int64_t>(values.size()); }
};

// src/csr.cpp:10-50 semantics: sort by (row, col), sum duplicates, keep
// explicit zeros. Stable sort (the reference's std::sort leaves the order of
// equal keys unspecified; sums of >=3 exact duplicates are order-sensitive).
// Throws std::invalid_argument / std::out_of_range like the reference.
CsrHost csr_from_triplets(std::int64_t n, const std::vector<std::int64_t>& rows,
                          const std::vector<std::int64_t>& cols,
                          const std::vector<double>& vals);
// Validates an existing CSR (monotone row_ptr, in-range sorted columns).
void csr_validate(const CsrHost& a);
CsrHost transpose(const CsrHost& a);                 // src/csr.cpp:108-125
double gershgorin_gamma(const CsrHost& a);            // src/csr.cpp:127-143
CsrHost prescale(const CsrHost& a, double gamma);     // src/csr.cpp:145-150
std::uint64_t csr_content_hash(const CsrHost& a);     // src/csr.cpp:152-173
std::vector<double> spmv(const CsrHost& a, const std::vector<double>& x);  // :52-62
// Rounds values once to fp32 (the device copy) and back to f64.
CsrHost round_values_f32(const CsrHost& a);

// ---------------------------------------------------------------- generators
CsrHost gen_convection_diffusion(std::int64_t grid, double convection);   // src/gen.cpp:11-38
CsrHost gen_random_nonsymmetric(std::int64_t n, std::int64_t offdiag, double dominance,
                                std::uint64_t seed);                      // src/gen.cpp:40-69
// BASELINE.json configs 2-5 (new generators; recipes in DESIGN.md §3).
CsrHost gen_convection_diffusion_3d(std::int64_t grid, double peclet);
CsrHost gen_varcoeff_diffusion_2d(std::int64_t grid, double sigma, std::uint64_t seed);
CsrHost gen_powerlaw_random(std::int64_t n, double alpha, std::int64_t kmin,
                            std::int64_t kmax, std::uint64_t seed);
CsrHost gen_anisotropic_9pt(std::int64_t grid, double eps, double theta_deg);
CsrHost parse_matrix_market(const std::string& text);  // src/mmio.cpp:21-87
CsrHost read_matrix_market_file(const std::string& path);

// ---------------------------------------------------------------- spectral sampler
// One-sided Jacobi SVD of a tall col-major rows x cols matrix (src/svd.cpp:10-80):
// u rows x cols, s descending, v cols x cols, all col-major.
struct SvdResult {
  std::int64_t rows = 0, cols = 0;
  std::vector<double> u, s, v;
};
SvdResult jacobi_svd(std::int64_t rows, std::int64_t cols, const std::vector<double>& a);

// SpectralSampler (include/gnp/sampler.hpp:13-22) minus the factors sampling
// never reads (vfull, wm).  The Arnoldi cycle that feeds it runs on the device
// (gnpc_sampler_create); this is the host half.
struct SpectralSampler {
  std::int64_t n = 0, m = 0, m_eff = 0;
  std::vector<double> v;      // n x m col-major, the first m Arnoldi basis vectors
  std::vector<double> zm_sv;  // m x m col-major, right singular vectors of Hbar
  std::vector<double> s;      // m singular values, descending
};
// src/sampler.cpp:19-38 given the cycle's k steps: v n x k, hbar (k+1) x k (col-major).
SpectralSampler spectral_from_arnoldi(std::int64_t n, std::int64_t k, std::vector<double> v,
                                      const std::vector<double>& hbar);
// src/sampler.cpp:41-59: coef = Zsv[:, :m_eff] diag(1/s) eps, x = V coef, b = A x.
void sample_spectral_pair(const SpectralSampler& sp, const CsrHost& a, Rng& rng, double* x,
                          double* b);
// src/sampler.cpp:68-83: columns k < spectral_count spectral, the rest Gaussian;
// x, b n x batch col-major.  sp may be null when spectral_count == 0.
void assemble_batch(const SpectralSampler* sp, const CsrHost& a, std::int64_t batch,
                    std::int64_t spectral_count, Rng& rng, double* x, double* b);

// ---------------------------------------------------------------- params
struct Dims {
  std::int64_t d = 16, hidden = 32, layers = 8;
};
struct ParamLayout {
  std::int64_t enc1, enc1_b, enc2, enc2_b, dec1, dec1_b, dec2, dec2_b, total;
  std::vector<std::int64_t> u, w;
};
ParamLayout param_layout(const Dims& dims);  // src/gnn.cpp:40-55 order
std::vector<double> init_params(const Dims& dims, std::uint64_t seed);  // src/gnn.cpp:92-118

struct MatrixMeta {
  std::int64_t n = 0, nnz = 0;
  std::uint64_t hash = 0;
};
std::string checkpoint_bytes(const Dims& dims, const std::vector<double>& params,
                             const MatrixMeta& meta);  // src/gnn.cpp:513-522
void checkpoint_parse(const std::string& bytes, Dims* dims, std::vector<double>* params,
                      MatrixMeta* meta);               // src/gnn.cpp:524-557

}  // namespace gnp_b200
