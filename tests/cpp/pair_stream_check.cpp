// CPU check of the reference-stream pair generator (csrc/host/pair_stream.*):
// the batches it describes — raw MT words Box-Muller'd the way k_pairs_x does
// it (here with the host's libm, so bit-exact), host heads/tails/fallbacks,
// spectral x = V coef — must equal gnp_b200::assemble_batch driven by the
// reference Rng (pinned bitwise to src/sampler.cpp:61-83 by the CPU tests),
// batch after batch, including odd n (spares crossing columns and batches),
// spectral columns and a forced rejection fallback.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "host/gnp_host.hpp"
#include "host/pair_stream.hpp"

using namespace gnp_b200;

static int check_case(std::int64_t grid, std::int64_t B, std::int64_t S, std::int64_t force, int batches) {
  const CsrHost a = gen_convection_diffusion(grid, 0.3);
  const std::int64_t n = a.n;
  SpectralSampler sp;
  if (S > 0) {  // a synthetic sampler: any orthonormal-ish V and factors will do
    const std::int64_t m = 5;
    Rng r(77);
    std::vector<double> v(n * m), h((m + 1) * m);
    for (auto& x : v) x = r.gaussian();
    for (auto& x : h) x = r.gaussian();
    sp = spectral_from_arnoldi(n, m, v, h);
  }
  PairStream ps(11, n, B, S, S > 0 ? &sp : nullptr);
  ps.debug_force_reject = force;
  Rng ref(11);
  std::vector<unsigned char> buf(ps.layout().bytes);
  std::vector<double> xr(n * B), br(n * B), x(n * B);
  const auto& L = ps.layout();
  for (int t = 0; t < batches; ++t) {
    ps.fill(buf.data());
    assemble_batch(S > 0 ? &sp : nullptr, a, B, S, ref, xr.data(), br.data());
    const PairCol* cols = reinterpret_cast<const PairCol*>(buf.data() + L.cols_off);
    const double* coef = reinterpret_cast<const double*>(buf.data() + L.coef_off);
    const std::uint64_t* words = reinterpret_cast<const std::uint64_t*>(buf.data() + L.words_off);
    for (std::int64_t c = 0; c < B; ++c) {
      const PairCol& col = cols[c];
      for (std::int64_t i = 0; i < n; ++i) {
        double v;
        if (col.mode == 0) {
          if (col.has_head && i == 0) v = col.head;
          else if (col.has_tail && i == n - 1) v = col.tail;
          else {
            const std::int64_t j = i - col.has_head;
            const std::uint64_t* w = words + col.off + 2 * (j >> 1);
            const double u1 = (double)(RawMt64::temper(w[0]) >> 11) * 0x1.0p-53;
            const double u2 = (double)(RawMt64::temper(w[1]) >> 11) * 0x1.0p-53;
            const double r = std::sqrt(-2.0 * std::log(u1));
            const double th = 6.283185307179586476925286766559 * u2;
            v = r * ((j & 1) ? std::sin(th) : std::cos(th));
          }
        } else if (col.mode == 1) {
          v = reinterpret_cast<const double*>(words + col.off)[i];
        } else {
          double acc = 0.0;
          for (std::int64_t q = 0; q < L.m; ++q) acc += sp.v[q * n + i] * coef[col.off * L.m + q];
          v = acc;
        }
        x[c * n + i] = v;
      }
    }
    if (std::memcmp(x.data(), xr.data(), x.size() * 8) != 0) {
      std::printf("FAIL grid %ld B %ld S %ld force %ld batch %d\n", (long)grid, (long)B, (long)S,
                  (long)force, t);
      return 1;
    }
  }
  std::printf("ok grid %ld B %ld S %ld force %ld (%d batches)\n", (long)grid, (long)B, (long)S, (long)force,
              batches);
  return 0;
}

int main() {
  // raw recurrence == std::mt19937_64, scalar and bulk interleaved
  {
    std::mt19937_64 g(5);
    RawMt64 r(5);
    std::vector<std::uint64_t> w(1000);
    for (int rep = 0; rep < 5; ++rep) {
      for (int k = 0; k < 7; ++k)
        if (r() != g()) { std::printf("FAIL scalar\n"); return 1; }
      const std::size_t cnt = rep == 0 ? 3 : (rep == 1 ? 312 : (rep == 2 ? 313 : 999));
      r.bulk_raw(w.data(), cnt);
      for (std::size_t k = 0; k < cnt; ++k)
        if (RawMt64::temper(w[k]) != g()) { std::printf("FAIL bulk %d\n", rep); return 1; }
    }
    std::printf("ok raw recurrence\n");
  }
  int rc = 0;
  rc |= check_case(16, 8, 0, -1, 3);    // n even
  rc |= check_case(15, 5, 0, -1, 4);    // n odd: heads and tails, spares across batches
  rc |= check_case(15, 6, 2, -1, 3);    // spectral columns first
  rc |= check_case(15, 5, 1, 3, 3);     // forced host fallback in column 3
  rc |= check_case(9, 3, 0, 0, 5);      // forced fallback in column 0
  return rc;
}
