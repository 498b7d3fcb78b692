// Reference-stream training pairs with the Box-Muller on the device.
//
// The reference draws every training batch from one Rng(seed + 3)
// (src/gnn.cpp:405-414, src/sampler.cpp:61-83): std::mt19937_64 words,
// uniform = (w >> 11) 2^-53, Box-Muller with a cached spare
// (include/gnp/rng.hpp:13-52).  A C3 batch is 8.4M Gaussians; the host
// Box-Muller alone (log, sqrt, sin, cos per pair) costs more than the device
// step.  Here the host only advances the Mersenne Twister — as its raw linear
// recurrence w[k+312] = w[k+156] ^ A((w[k] & UM) | (w[k+1] & LM)), whose
// tempered terms are exactly std::mt19937_64's outputs — and ships raw words;
// the device tempers them and runs the Box-Muller.  Draws the device cannot
// take in bulk (a column that starts on a cached spare, an odd tail, the
// m_eff Gaussians behind a spectral column's coefficients, and any column in
// which the rare u1 <= 0 rejection would fire) are made on the host with the
// reference's own arithmetic, so the stream position and spare state follow
// the reference draw for draw.
#pragma once
#include <cstdint>
#include <vector>

#include "gnp_host.hpp"

namespace gnp_b200 {

class RawMt64 {
 public:
  static constexpr int kN = 312, kM = 156;
  explicit RawMt64(std::uint64_t seed);
  static std::uint64_t temper(std::uint64_t y) {
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    y ^= (y >> 43);
    return y;
  }
  std::uint64_t next_raw();
  std::uint64_t operator()() { return temper(next_raw()); }  // == std::mt19937_64()
  // the next `count` raw words (temper(out[j]) is the j-th next output)
  void bulk_raw(std::uint64_t* out, std::size_t count);
  // Rng semantics on this stream (include/gnp/rng.hpp:18-40)
  double uniform() { return static_cast<double>((*this)() >> 11) * 0x1.0p-53; }
  double gaussian();
  bool have_spare = false;
  double spare = 0.0;
  struct State {
    std::uint64_t ring[kN];
    int pos;
    bool have_spare;
    double spare;
  };
  State save() const;
  void restore(const State& s);

 private:
  std::uint64_t ring_[kN];
  int pos_ = 0;  // ring_[pos_] holds the oldest of the last 312 raw words
};

// One column of a device batch.
struct PairCol {
  std::int32_t mode;      // 0: raw words (device Box-Muller), 1: explicit values, 2: spectral
  std::int32_t has_head;  // mode 0: x[0] = head (a cached spare)
  std::int32_t has_tail;  // mode 0: x[n-1] = tail (cos half of a host-drawn pair)
  std::int32_t pad;
  std::int64_t off;       // modes 0/1: first slot (u64 index into the words area); 2: coef row
  double head, tail;
};

// Host side of one batch, laid out for a single H2D copy:
//   [PairCol x B][coef: S x m f64][per Gaussian column: n + 2 u64 slots]
// A Gaussian column's slots hold its raw words (mode 0) or, after a
// rejection fallback, its n values as f64 (mode 1).
struct PairBatchLayout {
  std::int64_t B = 0, S = 0, n = 0, m = 0;
  std::size_t cols_off = 0, coef_off = 0, words_off = 0, bytes = 0;
};

class PairStream {
 public:
  // spectral columns (k < spectral_count) use the sampler's factors; the
  // rest are Gaussian.  `sp` may be null when spectral_count == 0.
  PairStream(std::uint64_t seed, std::int64_t n, std::int64_t batch, std::int64_t spectral_count,
             const SpectralSampler* sp);
  const PairBatchLayout& layout() const { return lay_; }
  // fill one batch into `buf` (layout().bytes bytes); returns the number of
  // explicit-value columns (rejection fallbacks), normally 0
  int fill(unsigned char* buf);
  // test hook: treat this Gaussian column of every batch as rejected (host path)
  std::int64_t debug_force_reject = -1;

 private:
  bool gaussian_column(PairCol& col, std::uint64_t* slots);
  RawMt64 rng_;
  std::int64_t n_, B_, S_;
  const SpectralSampler* sp_;
  PairBatchLayout lay_;
};

}  // namespace gnp_b200
