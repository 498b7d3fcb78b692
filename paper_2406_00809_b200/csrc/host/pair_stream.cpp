// Reference-stream training pairs (see pair_stream.hpp).
#include "pair_stream.hpp"

#include <cmath>
#include <cstring>
#include <stdexcept>

namespace gnp_b200 {

namespace {
constexpr std::uint64_t kMatA = 0xB5026F5AA96619E9ull;
constexpr std::uint64_t kUM = 0xFFFFFFFF80000000ull;
constexpr std::uint64_t kLM = 0x7FFFFFFFull;

inline std::uint64_t step(std::uint64_t wk, std::uint64_t wk1, std::uint64_t wkm) {
  const std::uint64_t x = (wk & kUM) | (wk1 & kLM);
  return wkm ^ (x >> 1) ^ ((std::uint64_t)(-(std::int64_t)(x & 1)) & kMatA);
}
std::size_t align64(std::size_t b) { return (b + 63) & ~std::size_t(63); }
}  // namespace

// std::mt19937_64 seeding ([rand.eng.mers]): x0 = seed,
// x_i = 6364136223846793005 (x_{i-1} ^ (x_{i-1} >> 62)) + i.
RawMt64::RawMt64(std::uint64_t seed) {
  ring_[0] = seed;
  for (int i = 1; i < kN; ++i)
    ring_[i] = 6364136223846793005ull * (ring_[i - 1] ^ (ring_[i - 1] >> 62)) + (std::uint64_t)i;
  pos_ = 0;
}

std::uint64_t RawMt64::next_raw() {
  const std::uint64_t w = step(ring_[pos_], ring_[(pos_ + 1) % kN], ring_[(pos_ + kM) % kN]);
  ring_[pos_] = w;
  pos_ = (pos_ + 1) % kN;
  return w;
}

void RawMt64::bulk_raw(std::uint64_t* out, std::size_t count) {
  // relative index t: t < 312 is the ring (oldest first), t >= 312 is out[t - 312]
  auto get = [&](std::size_t t) -> std::uint64_t {
    return t < (std::size_t)kN ? ring_[(pos_ + t) % kN] : out[t - kN];
  };
  const std::size_t head = count < (std::size_t)kN ? count : (std::size_t)kN;
  for (std::size_t j = 0; j < head; ++j) out[j] = step(get(j), get(j + 1), get(j + kM));
  for (std::size_t j = kN; j < count; ++j) out[j] = step(out[j - kN], out[j - kN + 1], out[j - kM]);
  std::uint64_t nr[kN];
  for (std::size_t i = 0; i < (std::size_t)kN; ++i) nr[i] = get(count + i);
  std::memcpy(ring_, nr, sizeof nr);
  pos_ = 0;
}

// rng.hpp:27-40
double RawMt64::gaussian() {
  if (have_spare) {
    have_spare = false;
    return spare;
  }
  double u1 = uniform();
  while (u1 <= 0.0) u1 = uniform();
  const double u2 = uniform();
  const double r = std::sqrt(-2.0 * std::log(u1));
  const double theta = 6.283185307179586476925286766559 * u2;
  spare = r * std::sin(theta);
  have_spare = true;
  return r * std::cos(theta);
}

RawMt64::State RawMt64::save() const {
  State s;
  std::memcpy(s.ring, ring_, sizeof ring_);
  s.pos = pos_;
  s.have_spare = have_spare;
  s.spare = spare;
  return s;
}

void RawMt64::restore(const State& s) {
  std::memcpy(ring_, s.ring, sizeof ring_);
  pos_ = s.pos;
  have_spare = s.have_spare;
  spare = s.spare;
}

PairStream::PairStream(std::uint64_t seed, std::int64_t n, std::int64_t batch,
                       std::int64_t spectral_count, const SpectralSampler* sp)
    : rng_(seed), n_(n), B_(batch), S_(spectral_count), sp_(sp) {
  if (batch <= 0) throw std::invalid_argument("assemble_batch: empty batch");
  if (spectral_count > batch) throw std::invalid_argument("assemble_batch: spectral_count > batch");
  if (spectral_count > 0 && (!sp || sp->n != n))
    throw std::invalid_argument("assemble_batch: spectral columns need a sampler of this matrix");
  lay_.B = batch;
  lay_.S = spectral_count;
  lay_.n = n;
  lay_.m = spectral_count > 0 ? sp->m : 0;
  lay_.cols_off = 0;
  lay_.coef_off = align64(sizeof(PairCol) * (std::size_t)batch);
  lay_.words_off = align64(lay_.coef_off + sizeof(double) * (std::size_t)(spectral_count * lay_.m));
  lay_.bytes = lay_.words_off + sizeof(std::uint64_t) * (std::size_t)(batch - spectral_count) * (n + 2);
}

// One Gaussian column (src/sampler.cpp:77-78: x_k[i] = rng.gaussian() for
// i < n).  Returns true when the column fell back to host values.
bool PairStream::gaussian_column(PairCol& col, std::uint64_t* slots) {
  const RawMt64::State st = rng_.save();
  col.mode = 0;
  col.has_head = col.has_tail = 0;
  col.head = col.tail = 0.0;
  std::int64_t i = 0;
  if (rng_.have_spare) {  // x[0] is the spare cached by the previous draw
    col.has_head = 1;
    col.head = rng_.spare;
    rng_.have_spare = false;
    i = 1;
  }
  const std::int64_t rem = n_ - i, pairs = rem / 2;
  rng_.bulk_raw(slots, (std::size_t)(2 * pairs));
  // u1 <= 0 (a zero 53-bit mantissa) makes the reference draw one more word
  // for that pair; redo such a column on the host, draw for draw
  bool reject = false;
  for (std::int64_t p = 0; p < pairs; ++p) reject |= (RawMt64::temper(slots[2 * p]) >> 11) == 0;
  if (reject || col.off / (n_ + 2) + S_ == debug_force_reject) {
    rng_.restore(st);
    col.mode = 1;
    col.has_head = col.has_tail = 0;
    double* v = reinterpret_cast<double*>(slots);
    for (std::int64_t q = 0; q < n_; ++q) v[q] = rng_.gaussian();
    return true;
  }
  if (rem & 1) {  // the last value opens a new pair; its sine half stays cached
    col.has_tail = 1;
    col.tail = rng_.gaussian();
  }
  return false;
}

// src/sampler.cpp:68-83 (columns k < spectral_count spectral, the rest
// Gaussian); the spectral coefficients follow sample_spectral_pair
// (src/sampler.cpp:41-59): coef = Zsv[:, :m_eff] diag(1/s) eps.
int PairStream::fill(unsigned char* buf) {
  PairCol* cols = reinterpret_cast<PairCol*>(buf + lay_.cols_off);
  double* coef = reinterpret_cast<double*>(buf + lay_.coef_off);
  std::uint64_t* words = reinterpret_cast<std::uint64_t*>(buf + lay_.words_off);
  int fallbacks = 0;
  for (std::int64_t c = 0; c < B_; ++c) {
    PairCol& col = cols[c];
    if (c < S_) {
      const std::int64_t m = sp_->m;
      double* cf = coef + c * m;
      for (std::int64_t i = 0; i < m; ++i) cf[i] = 0.0;
      for (std::int64_t j = 0; j < sp_->m_eff; ++j) {
        const double scaled = rng_.gaussian() / sp_->s[j];
        for (std::int64_t i = 0; i < m; ++i) cf[i] += sp_->zm_sv[j * m + i] * scaled;
      }
      col.mode = 2;
      col.has_head = col.has_tail = 0;
      col.pad = 0;
      col.off = c;
      col.head = col.tail = 0.0;
      continue;
    }
    col.pad = 0;
    col.off = (c - S_) * (n_ + 2);
    fallbacks += gaussian_column(col, words + col.off) ? 1 : 0;
  }
  return fallbacks;
}

}  // namespace gnp_b200
