// Host-side CSR / RNG / params / checkpoint / generators. See gnp_host.hpp.
#include "gnp_host.hpp"

#include <algorithm>
#include <cstring>
#include <fstream>
#include <numeric>
#include <sstream>
#include <unordered_set>

namespace gnp_b200 {

// ======================================================================= CSR
CsrHost csr_from_triplets(std::int64_t n, const std::vector<std::int64_t>& rows,
                          const std::vector<std::int64_t>& cols,
                          const std::vector<double>& vals) {
  const std::size_t m = vals.size();
  if (rows.size() != m || cols.size() != m)
    throw std::invalid_argument("triplet arrays must have equal length");
  if (n < 0) throw std::invalid_argument("csr: negative dimension");
  for (std::size_t k = 0; k < m; ++k)
    if (rows[k] < 0 || cols[k] < 0 || rows[k] >= n || cols[k] >= n)
      throw std::out_of_range("triplet index out of range");

  // Already (row, col)-sorted input (every generator here) skips the sort.
  bool sorted = true;
  for (std::size_t k = 1; k < m && sorted; ++k)
    sorted = rows[k - 1] < rows[k] || (rows[k - 1] == rows[k] && cols[k - 1] <= cols[k]);
  std::vector<std::size_t> order;
  if (!sorted) {
    order.resize(m);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](std::size_t a, std::size_t b) {
      if (rows[a] != rows[b]) return rows[a] < rows[b];
      return cols[a] < cols[b];
    });
  }
  CsrHost out;
  out.n = n;
  out.row_ptr.assign(n + 1, 0);
  out.col_idx.reserve(m);
  out.values.reserve(m);
  std::int64_t last_row = -1;
  for (std::size_t k = 0; k < m; ++k) {
    const std::size_t t = sorted ? k : order[k];
    if (!out.values.empty() && rows[t] == last_row && cols[t] == out.col_idx.back()) {
      out.values.back() += vals[t];
    } else {
      last_row = rows[t];
      out.col_idx.push_back(cols[t]);
      out.values.push_back(vals[t]);
      out.row_ptr[rows[t] + 1]++;
    }
  }
  for (std::int64_t i = 0; i < n; ++i) out.row_ptr[i + 1] += out.row_ptr[i];
  return out;
}

void csr_validate(const CsrHost& a) {
  if (a.n < 0 || static_cast<std::int64_t>(a.row_ptr.size()) != a.n + 1)
    throw std::invalid_argument("csr: row_ptr must have n+1 entries");
  if (a.row_ptr[0] != 0 || a.row_ptr[a.n] != a.nnz() ||
      static_cast<std::int64_t>(a.col_idx.size()) != a.nnz())
    throw std::invalid_argument("csr: row_ptr/col_idx/values sizes disagree");
  for (std::int64_t i = 0; i < a.n; ++i) {
    if (a.row_ptr[i] > a.row_ptr[i + 1])
      throw std::invalid_argument("csr: row_ptr must be non-decreasing");
    for (std::int64_t k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) {
      if (a.col_idx[k] < 0 || a.col_idx[k] >= a.n)
        throw std::out_of_range("csr: column index out of range");
      if (k > a.row_ptr[i] && a.col_idx[k] <= a.col_idx[k - 1])
        throw std::invalid_argument("csr: columns must be strictly increasing within a row");
    }
  }
}

CsrHost transpose(const CsrHost& a) {
  CsrHost t;
  t.n = a.n;
  t.row_ptr.assign(a.n + 1, 0);
  t.col_idx.resize(a.nnz());
  t.values.resize(a.nnz());
  for (std::int64_t k = 0; k < a.nnz(); ++k) t.row_ptr[a.col_idx[k] + 1]++;
  for (std::int64_t i = 0; i < a.n; ++i) t.row_ptr[i + 1] += t.row_ptr[i];
  std::vector<std::int64_t> next(t.row_ptr.begin(), t.row_ptr.end() - 1);
  for (std::int64_t i = 0; i < a.n; ++i)
    for (std::int64_t k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) {
      const std::int64_t pos = next[a.col_idx[k]]++;
      t.col_idx[pos] = i;
      t.values[pos] = a.values[k];
    }
  return t;
}

double gershgorin_gamma(const CsrHost& a) {
  std::vector<double> col(a.n, 0.0);
  double max_row = 0.0;
  for (std::int64_t i = 0; i < a.n; ++i) {
    double row = 0.0;
    for (std::int64_t k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) {
      const double v = std::abs(a.values[k]);
      row += v;
      col[a.col_idx[k]] += v;
    }
    max_row = std::max(max_row, row);
  }
  double max_col = 0.0;
  for (double c : col) max_col = std::max(max_col, c);
  const double g = std::min(max_row, max_col);
  return g == 0.0 ? 1.0 : g;
}

CsrHost prescale(const CsrHost& a, double gamma) {
  if (gamma == 0.0) throw std::invalid_argument("prescale: gamma must be nonzero");
  CsrHost out = a;
  for (double& v : out.values) v /= gamma;
  return out;
}

std::uint64_t csr_content_hash(const CsrHost& a) {
  std::uint64_t h = 1469598103934665603ull;
  auto mix = [&h](const void* p, std::size_t bytes) {
    const auto* c = static_cast<const unsigned char*>(p);
    for (std::size_t i = 0; i < bytes; ++i) {
      h ^= c[i];
      h *= 1099511628211ull;
    }
  };
  const std::uint64_t n64 = static_cast<std::uint64_t>(a.n);
  mix(&n64, 8);
  for (std::int64_t v : a.row_ptr) {
    const std::uint64_t x = static_cast<std::uint64_t>(v);
    mix(&x, 8);
  }
  for (std::int64_t v : a.col_idx) {
    const std::uint64_t x = static_cast<std::uint64_t>(v);
    mix(&x, 8);
  }
  mix(a.values.data(), a.values.size() * sizeof(double));
  return h;
}

std::vector<double> spmv(const CsrHost& a, const std::vector<double>& x) {
  if (static_cast<std::int64_t>(x.size()) != a.n)
    throw std::invalid_argument("spmv: dimension mismatch");
  std::vector<double> y(a.n, 0.0);
  for (std::int64_t i = 0; i < a.n; ++i) {
    double s = 0.0;
    for (std::int64_t k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k)
      s += a.values[k] * x[a.col_idx[k]];
    y[i] = s;
  }
  return y;
}

CsrHost round_values_f32(const CsrHost& a) {
  CsrHost out = a;
  for (double& v : out.values) v = static_cast<double>(static_cast<float>(v));
  return out;
}

// ======================================================================= generators
namespace {
struct TripletSink {
  std::vector<std::int64_t> r, c;
  std::vector<double> v;
  void push(std::int64_t row, std::int64_t col, double val) {
    r.push_back(row);
    c.push_back(col);
    v.push_back(val);
  }
};
}  // namespace

CsrHost gen_convection_diffusion(std::int64_t grid, double convection) {
  if (grid < 2) throw std::invalid_argument("gen: grid must be >= 2");
  if (std::abs(convection) > 1.0)
    throw std::invalid_argument("gen: convection must lie in [-1, 1]");
  const std::int64_t n = grid * grid;
  TripletSink s;
  s.r.reserve(5 * n);
  s.c.reserve(5 * n);
  s.v.reserve(5 * n);
  auto idx = [grid](std::int64_t ix, std::int64_t iy) { return iy * grid + ix; };
  for (std::int64_t iy = 0; iy < grid; ++iy)
    for (std::int64_t ix = 0; ix < grid; ++ix) {
      const std::int64_t row = idx(ix, iy);
      s.push(row, row, 4.0);
      if (ix > 0) s.push(row, idx(ix - 1, iy), -1.0 - convection);
      if (ix + 1 < grid) s.push(row, idx(ix + 1, iy), -1.0 + convection);
      if (iy > 0) s.push(row, idx(ix, iy - 1), -1.0);
      if (iy + 1 < grid) s.push(row, idx(ix, iy + 1), -1.0);
    }
  return csr_from_triplets(n, s.r, s.c, s.v);
}

CsrHost gen_random_nonsymmetric(std::int64_t n, std::int64_t offdiag, double dominance,
                                std::uint64_t seed) {
  if (n < 1) throw std::invalid_argument("gen: n must be >= 1");
  if (offdiag >= n) throw std::invalid_argument("gen: too many off-diagonals per row");
  Rng rng(seed);
  TripletSink s;
  for (std::int64_t i = 0; i < n; ++i) {
    std::unordered_set<std::int64_t> used{i};
    double abs_sum = 0.0;
    for (std::int64_t k = 0; k < offdiag; ++k) {
      std::int64_t j;
      do {
        j = static_cast<std::int64_t>(rng.uniform() * static_cast<double>(n));
        if (j >= n) j = n - 1;
      } while (used.count(j));
      used.insert(j);
      const double v = rng.uniform_symmetric(1.0);
      abs_sum += std::abs(v);
      s.push(i, j, v);
    }
    s.push(i, i, dominance * abs_sum + 0.1 + 0.1 * rng.uniform());
  }
  return csr_from_triplets(n, s.r, s.c, s.v);
}

// C2: 3D convection-diffusion, 7-point stencil, first-order upwind for a
// constant velocity (1,1,1), global Peclet number Pe = |v|_inf L / nu with
// L = 1, so the equation is  -(1/Pe) Δu + (1,1,1)·∇u = f  on h = 1/(grid+1),
// Dirichlet; rows scaled by h^2 Pe:  diag 6 + 3 c, lower neighbours -1 - c,
// upper neighbours -1, c = Pe h.  nnz = 7 n - 6 grid^2.
CsrHost gen_convection_diffusion_3d(std::int64_t grid, double peclet) {
  if (grid < 2) throw std::invalid_argument("gen: grid must be >= 2");
  const std::int64_t n = grid * grid * grid;
  const double h = 1.0 / static_cast<double>(grid + 1);
  const double c = peclet * h;
  CsrHost a;
  a.n = n;
  a.row_ptr.assign(n + 1, 0);
  a.col_idx.reserve(7 * n);
  a.values.reserve(7 * n);
  const std::int64_t g2 = grid * grid;
  for (std::int64_t iz = 0; iz < grid; ++iz)
    for (std::int64_t iy = 0; iy < grid; ++iy)
      for (std::int64_t ix = 0; ix < grid; ++ix) {
        const std::int64_t row = iz * g2 + iy * grid + ix;
        auto push = [&](std::int64_t col, double v) {
          a.col_idx.push_back(col);
          a.values.push_back(v);
        };
        // ascending column order: -z, -y, -x, diag, +x, +y, +z
        if (iz > 0) push(row - g2, -1.0 - c);
        if (iy > 0) push(row - grid, -1.0 - c);
        if (ix > 0) push(row - 1, -1.0 - c);
        push(row, 6.0 + 3.0 * c);
        if (ix + 1 < grid) push(row + 1, -1.0);
        if (iy + 1 < grid) push(row + grid, -1.0);
        if (iz + 1 < grid) push(row + g2, -1.0);
        a.row_ptr[row + 1] = static_cast<std::int64_t>(a.values.size());
      }
  return a;
}

// C3: 2D variable-coefficient diffusion -∇·(κ∇u) on a grid x grid cell mesh,
// κ_cell = exp(sigma * N(0,1)) (lognormal(0, sigma^2)) drawn cell by cell in
// row-major order from Rng(seed); interior faces use the harmonic mean
// 2 κ_i κ_j / (κ_i + κ_j); Dirichlet boundary faces use κ_i.  5-point,
// nnz = 5 n - 4 grid.
CsrHost gen_varcoeff_diffusion_2d(std::int64_t grid, double sigma, std::uint64_t seed) {
  if (grid < 2) throw std::invalid_argument("gen: grid must be >= 2");
  const std::int64_t n = grid * grid;
  Rng rng(seed);
  std::vector<double> kap(n);
  for (auto& k : kap) k = std::exp(sigma * rng.gaussian());
  auto harm = [](double a, double b) { return 2.0 * a * b / (a + b); };
  CsrHost a;
  a.n = n;
  a.row_ptr.assign(n + 1, 0);
  a.col_idx.reserve(5 * n);
  a.values.reserve(5 * n);
  for (std::int64_t iy = 0; iy < grid; ++iy)
    for (std::int64_t ix = 0; ix < grid; ++ix) {
      const std::int64_t row = iy * grid + ix;
      const double kc = kap[row];
      const double fs = iy > 0 ? harm(kc, kap[row - grid]) : kc;
      const double fw = ix > 0 ? harm(kc, kap[row - 1]) : kc;
      const double fe = ix + 1 < grid ? harm(kc, kap[row + 1]) : kc;
      const double fn = iy + 1 < grid ? harm(kc, kap[row + grid]) : kc;
      auto push = [&](std::int64_t col, double v) {
        a.col_idx.push_back(col);
        a.values.push_back(v);
      };
      if (iy > 0) push(row - grid, -fs);
      if (ix > 0) push(row - 1, -fw);
      push(row, fs + fw + fe + fn);
      if (ix + 1 < grid) push(row + 1, -fe);
      if (iy + 1 < grid) push(row + grid, -fn);
      a.row_ptr[row + 1] = static_cast<std::int64_t>(a.values.size());
    }
  return a;
}

// C4: random nonsymmetric, off-diagonal row lengths k ~ P(k) ∝ k^-alpha on
// [kmin, kmax] (inverse CDF on one uniform), columns uniform without
// replacement excluding the diagonal (rejection on one uniform each),
// values N(0,1), diagonal = (Σ_j |a_ij|) * 10^U(-6,0).  One Rng(seed)
// stream consumed row by row in that order.
CsrHost gen_powerlaw_random(std::int64_t n, double alpha, std::int64_t kmin, std::int64_t kmax,
                            std::uint64_t seed) {
  if (n < 2 || kmin < 1 || kmax < kmin || kmax >= n)
    throw std::invalid_argument("gen_powerlaw_random: bad arguments");
  std::vector<double> cdf(kmax - kmin + 1);
  double acc = 0.0;
  for (std::int64_t k = kmin; k <= kmax; ++k) {
    acc += std::pow(static_cast<double>(k), -alpha);
    cdf[k - kmin] = acc;
  }
  for (double& c : cdf) c /= acc;
  Rng rng(seed);
  CsrHost a;
  a.n = n;
  a.row_ptr.assign(n + 1, 0);
  std::vector<std::int64_t> cols;
  std::vector<double> vals;
  std::vector<std::pair<std::int64_t, double>> row;
  std::unordered_set<std::int64_t> used;
  for (std::int64_t i = 0; i < n; ++i) {
    const double u = rng.uniform();
    const std::int64_t k =
        kmin + static_cast<std::int64_t>(std::lower_bound(cdf.begin(), cdf.end(), u) - cdf.begin());
    used.clear();
    used.insert(i);
    row.clear();
    double abs_sum = 0.0;
    for (std::int64_t t = 0; t < std::min(k, kmax); ++t) {
      std::int64_t j;
      do {
        j = static_cast<std::int64_t>(rng.uniform() * static_cast<double>(n));
        if (j >= n) j = n - 1;
      } while (used.count(j));
      used.insert(j);
      const double v = rng.gaussian();
      abs_sum += std::abs(v);
      row.emplace_back(j, v);
    }
    const double diag = abs_sum * std::pow(10.0, -6.0 * rng.uniform());
    row.emplace_back(i, diag);
    std::sort(row.begin(), row.end());
    for (const auto& [c, v] : row) {
      a.col_idx.push_back(c);
      a.values.push_back(v);
    }
    a.row_ptr[i + 1] = static_cast<std::int64_t>(a.values.size());
  }
  return a;
}

// C5: 2D anisotropic diffusion -∇·(K∇u), K = R(θ) diag(1, eps) R(θ)^T, on a
// grid x grid mesh, Dirichlet, standard 9-point stencil (mixed derivative by
// the 4-corner difference), rows scaled by h^2:
//   centre 2(k11 + k22), E/W -k11, N/S -k22, NE/SW -k12/2, NW/SE +k12/2.
// nnz = (3 grid - 2)^2.
CsrHost gen_anisotropic_9pt(std::int64_t grid, double eps, double theta_deg) {
  if (grid < 2) throw std::invalid_argument("gen: grid must be >= 2");
  const double th = theta_deg * 3.14159265358979323846 / 180.0;
  const double c = std::cos(th), s = std::sin(th);
  const double k11 = c * c + eps * s * s;
  const double k22 = s * s + eps * c * c;
  const double k12 = (1.0 - eps) * c * s;
  const std::int64_t n = grid * grid;
  CsrHost a;
  a.n = n;
  a.row_ptr.assign(n + 1, 0);
  a.col_idx.reserve(9 * n);
  a.values.reserve(9 * n);
  // Axis-aligned part st[dy+1][dx+1]; corners come from -2 k12 u_xy with
  // u_xy ≈ (u_NE - u_SE - u_NW + u_SW) / 4h^2, i.e. -k12/2 * dx * dy.
  // Visiting (dy, dx) row-major keeps the columns ascending.
  const double st[3][3] = {{0.0, -k22, 0.0}, {-k11, 2.0 * (k11 + k22), -k11}, {0.0, -k22, 0.0}};
  for (std::int64_t iy = 0; iy < grid; ++iy)
    for (std::int64_t ix = 0; ix < grid; ++ix) {
      const std::int64_t row = iy * grid + ix;
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          const std::int64_t jx = ix + dx, jy = iy + dy;
          if (jx < 0 || jy < 0 || jx >= grid || jy >= grid) continue;
          double v = st[dy + 1][dx + 1];
          if (dx != 0 && dy != 0) v = -0.5 * k12 * static_cast<double>(dx * dy);
          a.col_idx.push_back(jy * grid + jx);
          a.values.push_back(v);
        }
      a.row_ptr[row + 1] = static_cast<std::int64_t>(a.values.size());
    }
  return a;
}

CsrHost parse_matrix_market(const std::string& text) {
  std::istringstream in(text);
  std::string line;
  if (!std::getline(in, line)) throw std::runtime_error("empty stream");
  auto lower = [](std::string s) {
    for (auto& ch : s) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
    return s;
  };
  std::istringstream header(line);
  std::string banner, object, format, field, symmetry;
  header >> banner >> object >> format >> field >> symmetry;
  if (banner != "%%MatrixMarket" || lower(object) != "matrix")
    throw std::runtime_error("not a Matrix Market matrix file");
  format = lower(format);
  field = lower(field);
  symmetry = lower(symmetry);
  if (format != "coordinate") throw std::runtime_error("unsupported format: " + format);
  if (field != "real") throw std::runtime_error("unsupported field: " + field);
  const bool sym = symmetry == "symmetric", skew = symmetry == "skew-symmetric";
  if (!sym && !skew && symmetry != "general")
    throw std::runtime_error("unsupported symmetry: " + symmetry);
  while (std::getline(in, line))
    if (!line.empty() && line[0] != '%') break;
  std::istringstream sl(line);
  long long nr = -1, nc = -1, nnz = -1;
  sl >> nr >> nc >> nnz;
  if (nr < 0 || nc < 0 || nnz < 0) throw std::runtime_error("bad size line");
  if (nr != nc) throw std::runtime_error("matrix is not square");
  std::vector<std::int64_t> r, c;
  std::vector<double> v;
  long long seen = 0;
  while (seen < nnz) {
    if (!std::getline(in, line)) throw std::runtime_error("truncated entry list");
    if (line.empty() || line[0] == '%') continue;
    std::istringstream e(line);
    long long i = 0, j = 0;
    double x = 0.0;
    if (!(e >> i >> j >> x)) throw std::runtime_error("malformed entry: " + line);
    if (i < 1 || j < 1 || i > nr || j > nc) throw std::runtime_error("entry index out of range");
    r.push_back(i - 1);
    c.push_back(j - 1);
    v.push_back(x);
    if ((sym || skew) && i != j) {
      r.push_back(j - 1);
      c.push_back(i - 1);
      v.push_back(skew ? -x : x);
    }
    ++seen;
  }
  CsrHost a = csr_from_triplets(nr, r, c, v);
  for (double x : a.values)
    if (!std::isfinite(x)) throw std::runtime_error("non-finite value in matrix");
  return a;
}

CsrHost read_matrix_market_file(const std::string& path) {
  std::ifstream f(path);
  if (!f) throw std::runtime_error("cannot open " + path);
  std::stringstream ss;
  ss << f.rdbuf();
  return parse_matrix_market(ss.str());
}

// ======================================================================= params
ParamLayout param_layout(const Dims& dm) {
  ParamLayout l;
  std::int64_t o = 0;
  const std::int64_t d = dm.d, h = dm.hidden;
  l.enc1 = o; o += h;
  l.enc1_b = o; o += h;
  l.enc2 = o; o += h * d;
  l.enc2_b = o; o += d;
  for (std::int64_t i = 0; i < dm.layers; ++i) {
    l.u.push_back(o); o += d * d;
    l.w.push_back(o); o += d * d;
  }
  l.dec1 = o; o += d * h;
  l.dec1_b = o; o += h;
  l.dec2 = o; o += h;
  l.dec2_b = o; o += 1;
  l.total = o;
  return l;
}

std::vector<double> init_params(const Dims& dm, std::uint64_t seed) {
  if (dm.d < 1 || dm.hidden < 1 || dm.layers < 1)
    throw std::invalid_argument("init_params: dims must be >= 1");
  const ParamLayout l = param_layout(dm);
  std::vector<double> p(l.total, 0.0);
  Rng rng(seed);
  auto fill = [&](std::int64_t off, std::int64_t cnt, std::int64_t fi, std::int64_t fo) {
    const double bound = std::sqrt(6.0 / static_cast<double>(fi + fo));
    for (std::int64_t q = 0; q < cnt; ++q) p[off + q] = rng.uniform_symmetric(bound);
  };
  fill(l.enc1, dm.hidden, 1, dm.hidden);
  fill(l.enc2, dm.hidden * dm.d, dm.hidden, dm.d);
  for (std::int64_t i = 0; i < dm.layers; ++i) {
    fill(l.u[i], dm.d * dm.d, dm.d, dm.d);
    fill(l.w[i], dm.d * dm.d, dm.d, dm.d);
  }
  fill(l.dec1, dm.d * dm.hidden, dm.d, dm.hidden);
  fill(l.dec2, dm.hidden, dm.hidden, 1);
  return p;
}

namespace {
struct NamedArray {
  const char* name;
  std::int64_t off, size;
};
std::vector<NamedArray> named_arrays(const Dims& dm) {
  const ParamLayout l = param_layout(dm);
  std::vector<NamedArray> v{{"enc1", l.enc1, dm.hidden},
                            {"enc1_bias", l.enc1_b, dm.hidden},
                            {"enc2", l.enc2, dm.hidden * dm.d},
                            {"enc2_bias", l.enc2_b, dm.d}};
  for (std::int64_t i = 0; i < dm.layers; ++i) {
    v.push_back({"u", l.u[i], dm.d * dm.d});
    v.push_back({"w", l.w[i], dm.d * dm.d});
  }
  v.push_back({"dec1", l.dec1, dm.d * dm.hidden});
  v.push_back({"dec1_bias", l.dec1_b, dm.hidden});
  v.push_back({"dec2", l.dec2, dm.hidden});
  v.push_back({"dec2_bias", l.dec2_b, 1});
  return v;
}
}  // namespace

std::string checkpoint_bytes(const Dims& dm, const std::vector<double>& p,
                             const MatrixMeta& meta) {
  if (static_cast<std::int64_t>(p.size()) != param_layout(dm).total)
    throw std::invalid_argument("checkpoint: parameter count does not match dims");
  std::ostringstream out(std::ios::binary);
  out << "GNPCKPT 1\n";
  out << "dims " << dm.d << ' ' << dm.hidden << ' ' << dm.layers << '\n';
  out << "matrix " << meta.n << ' ' << meta.nnz << ' ' << std::hex << meta.hash << std::dec
      << '\n';
  for (const auto& a : named_arrays(dm)) {
    out << "array " << a.name << ' ' << a.size << '\n';
    out.write(reinterpret_cast<const char*>(p.data() + a.off),
              static_cast<std::streamsize>(a.size * sizeof(double)));
    out << '\n';
  }
  return out.str();
}

void checkpoint_parse(const std::string& bytes, Dims* dims, std::vector<double>* params,
                      MatrixMeta* meta) {
  std::istringstream in(bytes, std::ios::binary);
  std::string line;
  if (!std::getline(in, line)) throw std::runtime_error("empty checkpoint");
  {
    std::istringstream ls(line);
    std::string magic;
    int version = 0;
    ls >> magic >> version;
    if (magic != "GNPCKPT") throw std::runtime_error("not a checkpoint file");
    if (version != 1) throw std::runtime_error("unsupported checkpoint version");
  }
  Dims dm;
  {
    if (!std::getline(in, line)) throw std::runtime_error("checkpoint truncated");
    std::istringstream ls(line);
    std::string tag;
    ls >> tag >> dm.d >> dm.hidden >> dm.layers;
    if (tag != "dims" || !ls) throw std::runtime_error("bad dims line");
    if (dm.d < 1 || dm.hidden < 1 || dm.layers < 1) throw std::runtime_error("bad dims line");
  }
  MatrixMeta mm;
  {
    if (!std::getline(in, line)) throw std::runtime_error("checkpoint truncated");
    std::istringstream ls(line);
    std::string tag;
    ls >> tag >> mm.n >> mm.nnz >> std::hex >> mm.hash;
    if (tag != "matrix" || !ls) throw std::runtime_error("bad matrix line");
  }
  std::vector<double> p(param_layout(dm).total, 0.0);
  for (const auto& a : named_arrays(dm)) {
    if (!std::getline(in, line)) throw std::runtime_error("checkpoint truncated");
    std::istringstream ls(line);
    std::string tag, name;
    std::int64_t count = 0;
    ls >> tag >> name >> count;
    if (tag != "array" || name != a.name || count != a.size)
      throw std::runtime_error(std::string("checkpoint array mismatch: expected ") + a.name);
    in.read(reinterpret_cast<char*>(p.data() + a.off),
            static_cast<std::streamsize>(a.size * sizeof(double)));
    if (!in) throw std::runtime_error(std::string("checkpoint truncated in array ") + a.name);
    in.get();
  }
  *dims = dm;
  *params = std::move(p);
  *meta = mm;
}

// ---------------------------------------------------------------- spectral sampler
SvdResult jacobi_svd(std::int64_t rows, std::int64_t cols, const std::vector<double>& a) {
  if (rows < cols) throw std::invalid_argument("jacobi_svd: matrix must be tall");
  if (static_cast<std::int64_t>(a.size()) != rows * cols)
    throw std::invalid_argument("jacobi_svd: size mismatch");
  std::vector<double> b = a, v(cols * cols, 0.0);
  for (std::int64_t i = 0; i < cols; ++i) v[i * cols + i] = 1.0;
  auto B = [&](std::int64_t r, std::int64_t c) -> double& { return b[c * rows + r]; };
  auto Vm = [&](std::int64_t r, std::int64_t c) -> double& { return v[c * cols + r]; };
  // cyclic sweeps over column pairs, rotation zeroing the (p, q) inner product
  for (int sweep = 0; sweep < 60; ++sweep) {
    bool rotated = false;
    for (std::int64_t p = 0; p + 1 < cols; ++p) {
      for (std::int64_t q = p + 1; q < cols; ++q) {
        double app = 0.0, aqq = 0.0, apq = 0.0;
        for (std::int64_t r = 0; r < rows; ++r) {
          app += B(r, p) * B(r, p);
          aqq += B(r, q) * B(r, q);
          apq += B(r, p) * B(r, q);
        }
        if (std::abs(apq) <= 1e-15 * std::sqrt(app * aqq)) continue;
        rotated = true;
        const double zeta = (aqq - app) / (2.0 * apq);
        const double t =
            (zeta >= 0.0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / std::sqrt(1.0 + t * t), sn = cs * t;
        for (std::int64_t r = 0; r < rows; ++r) {
          const double t1 = B(r, p), t2 = B(r, q);
          B(r, p) = cs * t1 - sn * t2;
          B(r, q) = sn * t1 + cs * t2;
        }
        for (std::int64_t r = 0; r < cols; ++r) {
          const double t1 = Vm(r, p), t2 = Vm(r, q);
          Vm(r, p) = cs * t1 - sn * t2;
          Vm(r, q) = sn * t1 + cs * t2;
        }
      }
    }
    if (!rotated) break;
  }
  std::vector<double> sv(cols);
  for (std::int64_t j = 0; j < cols; ++j) {
    double nrm = 0.0;
    for (std::int64_t r = 0; r < rows; ++r) nrm += B(r, j) * B(r, j);
    sv[j] = std::sqrt(nrm);
  }
  std::vector<std::int64_t> order(cols);
  std::iota(order.begin(), order.end(), std::int64_t{0});
  std::sort(order.begin(), order.end(),
            [&sv](std::int64_t i, std::int64_t j) { return sv[i] > sv[j]; });
  SvdResult out;
  out.rows = rows;
  out.cols = cols;
  out.u.assign(rows * cols, 0.0);
  out.v.assign(cols * cols, 0.0);
  out.s.resize(cols);
  for (std::int64_t j = 0; j < cols; ++j) {
    const std::int64_t src = order[j];
    out.s[j] = sv[src];
    if (sv[src] > 0.0)
      for (std::int64_t r = 0; r < rows; ++r) out.u[j * rows + r] = B(r, src) / sv[src];
    for (std::int64_t r = 0; r < cols; ++r) out.v[j * cols + r] = Vm(r, src);
  }
  return out;
}

SpectralSampler spectral_from_arnoldi(std::int64_t n, std::int64_t k, std::vector<double> v,
                                      const std::vector<double>& hbar) {
  SvdResult svd = jacobi_svd(k + 1, k, hbar);
  SpectralSampler out;
  out.n = n;
  out.m = k;
  out.v = std::move(v);
  out.v.resize(n * k);
  out.zm_sv = std::move(svd.v);
  out.s = std::move(svd.s);
  const double floor = out.s.empty() ? 0.0 : out.s[0] * 1e-12;
  for (double sv : out.s)
    if (sv >= floor && sv > 0.0) ++out.m_eff;
  if (out.m_eff == 0) throw std::runtime_error("spectral sampler: Hessenberg is numerically zero");
  return out;
}

void sample_spectral_pair(const SpectralSampler& sp, const CsrHost& a, Rng& rng, double* x,
                          double* b) {
  std::vector<double> coef(sp.m, 0.0);
  for (std::int64_t j = 0; j < sp.m_eff; ++j) {
    const double scaled = rng.gaussian() / sp.s[j];
    for (std::int64_t i = 0; i < sp.m; ++i) coef[i] += sp.zm_sv[j * sp.m + i] * scaled;
  }
  std::fill(x, x + a.n, 0.0);
  for (std::int64_t j = 0; j < sp.m; ++j) {
    const double cj = coef[j];
    const double* vj = sp.v.data() + j * a.n;
    for (std::int64_t i = 0; i < a.n; ++i) x[i] += vj[i] * cj;
  }
  for (std::int64_t i = 0; i < a.n; ++i) {
    double s = 0.0;
    for (std::int64_t q = a.row_ptr[i]; q < a.row_ptr[i + 1]; ++q) s += a.values[q] * x[a.col_idx[q]];
    b[i] = s;
  }
}

void assemble_batch(const SpectralSampler* sp, const CsrHost& a, std::int64_t batch,
                    std::int64_t spectral_count, Rng& rng, double* x, double* b) {
  if (batch <= 0) throw std::invalid_argument("assemble_batch: empty batch");
  if (spectral_count > batch) throw std::invalid_argument("assemble_batch: spectral_count > batch");
  if (spectral_count > 0 && (!sp || sp->n != a.n))
    throw std::invalid_argument("assemble_batch: spectral columns need a sampler of this matrix");
  const std::int64_t n = a.n;
  for (std::int64_t k = 0; k < batch; ++k) {
    double* xk = x + k * n;
    double* bk = b + k * n;
    if (k < spectral_count) {
      sample_spectral_pair(*sp, a, rng, xk, bk);
      continue;
    }
    for (std::int64_t i = 0; i < n; ++i) xk[i] = rng.gaussian();
    for (std::int64_t i = 0; i < n; ++i) {
      double s = 0.0;
      for (std::int64_t q = a.row_ptr[i]; q < a.row_ptr[i + 1]; ++q)
        s += a.values[q] * xk[a.col_idx[q]];
      bk[i] = s;
    }
  }
}

}  // namespace gnp_b200
