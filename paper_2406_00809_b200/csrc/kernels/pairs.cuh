// Device side of the reference-stream training pairs (host side:
// csrc/host/pair_stream.hpp) and the device-resident training-loop helpers.
//
//   k_pairs_x      x[i][c] for one batch in the trainer's [n][B] layout:
//                  mode 0: MT19937-64 tempering + Box-Muller of the host's raw
//                  words (include/gnp/rng.hpp:18-40), mode 1: host values,
//                  mode 2: spectral x = V coef (src/sampler.cpp:49-55)
//   k_spmm_nb_f64  b = A x over all B columns with the f64 matrix values in
//                  stored order, unfused multiply then add (src/csr.cpp:52-62:
//                  bit-identical to the host's b given x)
//   k_loss_fold    the loss as the host folds it (src/gnn.cpp:309-335 via
//                  k_loss_residual's per-block partials): sequential sum / B
//   k_best_keep    monitoring-loss best snapshot (src/gnn.cpp:443-448)
#pragma once
#include <cstdint>

#include "common.cuh"

namespace gnpk {

struct PairColDev {  // == gnp_b200::PairCol
  int mode, has_head, has_tail, pad;
  long long off;
  double head, tail;
};

__device__ __forceinline__ unsigned long long mt_temper(unsigned long long y) {
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= (y >> 43);
  return y;
}

// one thread per (node i, column c), c fastest: x[i * B + c]
__global__ void __launch_bounds__(kThreads)
k_pairs_x(const PairColDev* __restrict__ cols, const double* __restrict__ coef,
          const unsigned long long* __restrict__ words, const double* __restrict__ V, int m, int n,
          int B, double* __restrict__ x) {
  const size_t t = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<size_t>(n) * B) return;
  const int i = static_cast<int>(t / B), c = static_cast<int>(t % B);
  const PairColDev col = cols[c];
  double v;
  if (col.mode == 0) {
    if (col.has_head && i == 0) {
      v = col.head;
    } else if (col.has_tail && i == n - 1) {
      v = col.tail;
    } else {
      const int j = i - col.has_head;
      const unsigned long long* w = words + col.off + 2 * (j >> 1);
      const double u1 = static_cast<double>(mt_temper(w[0]) >> 11) * 0x1.0p-53;
      const double u2 = static_cast<double>(mt_temper(w[1]) >> 11) * 0x1.0p-53;
      const double r = __dsqrt_rn(__dmul_rn(-2.0, log(u1)));
      const double th = __dmul_rn(6.283185307179586476925286766559, u2);
      double s, co;
      sincos(th, &s, &co);
      v = __dmul_rn(r, (j & 1) ? s : co);
    }
  } else if (col.mode == 1) {
    v = reinterpret_cast<const double*>(words + col.off)[i];
  } else {
    const double* cf = coef + col.off * m;
    double acc = 0.0;
    for (int q = 0; q < m; ++q) acc = __dadd_rn(acc, __dmul_rn(V[static_cast<size_t>(q) * n + i], cf[q]));
    v = acc;
  }
  x[t] = v;
}

// b[i][c] = Σ_q a64[q] x[ci[q]][c] in stored order (warp per row, lanes over c)
__global__ void __launch_bounds__(kThreads)
k_spmm_nb_f64(DevCsr a, const double* __restrict__ a64, int B, const double* __restrict__ x,
              double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = wg; i < a.n; i += nw)
    for (int k = lane; k < B; k += 32) {
      double s = 0.0;
      for (int q = a.rp[i]; q < a.rp[i + 1]; ++q)
        s = __dadd_rn(s, __dmul_rn(a64[q], x[static_cast<size_t>(a.ci[q]) * B + k]));
      y[static_cast<size_t>(i) * B + k] = s;
    }
}

__global__ void k_loss_fold(const double* __restrict__ part, int count, int B, double* __restrict__ dst) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double acc = 0.0;
  for (int q = 0; q < count; ++q) acc += part[q];
  *dst = acc / static_cast<double>(B);
}

// if (loss < *best) { *best = loss; bestp = p }  — one block
__global__ void k_best_keep(const double* __restrict__ loss, double* __restrict__ best,
                            const double* __restrict__ p, double* __restrict__ bestp, int count) {
  const double l = *loss;
  const double b = *best;
  __syncthreads();
  if (!(l < b)) return;
  for (int k = threadIdx.x; k < count; k += blockDim.x) bestp[k] = p[k];
  if (threadIdx.x == 0) *best = l;
}

}  // namespace gnpk
