// Device-resident restarted FGMRES (src/krylov.cpp:17-277) on sm_100a.
//
// Per Arnoldi step j (one outer iteration):
//   [GNP apply vin -> zout]  (apply.cuh kernels, skipped once the cycle stops)
//   k_krylov_spmv   : w = A z_j, Z[:, j] = z_j                     (fp64)
//   k_krylov_ortho  : ONE cooperative kernel: ||w0||, modified Gram-Schmidt
//                     (dot of basis i+1 fused with the axpy of basis i, one
//                     grid barrier per basis vector), the same conditional
//                     re-orthogonalisation (||w|| < ||w0||/sqrt 2,
//                     src/krylov.cpp:47-56), breakdown test, v_{j+1} = w/||w||,
//                     then an incremental Givens update of the tracked
//                     residual by block 0 (bitwise the same rotations as the
//                     from-scratch hessenberg_lstsq, src/krylov.cpp:136-173),
//                     history entry + stop decision (converged / breakdown /
//                     timeout / maxiters) written to device state.
// Per cycle: back-substitution, x += Z y, true residual.  The host enqueues a
// whole cycle and synchronises once per cycle.
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"

namespace gnpk {

namespace cg = cooperative_groups;

// 4 lanes per row, fp64 sums of (double)a_ik * x_k; warp-uniform loop so the
// shuffles see all 32 lanes.
__device__ __forceinline__ double row_dot_q(const DevCsr& a, int i, bool valid,
                                            const double* __restrict__ x, int q) {
  double s = 0.0;
  if (valid) {
    const int e = __ldg(a.rp + i + 1);
    for (int k = __ldg(a.rp + i) + q; k < e; k += 4)
      s = fma(static_cast<double>(__ldg(a.v + k)), x[__ldg(a.ci + k)], s);
  }
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  return s;
}

// Eight rows per warp: rows of up to kSpmvLong entries by their quad
// (row_dot_q); longer rows (power-law matrices: up to thousands of entries,
// which left seven quads idle behind one) one after another by the whole
// warp, 32 lanes striding the row with two accumulators, then a shuffle tree.
// Every lane returns the sum of its quad's row.
constexpr int kSpmvLong = 64;
__device__ __forceinline__ double row_dot_warp8(const DevCsr& a, int base, const double* __restrict__ x,
                                                int lane) {
  const int q = lane & 3, g = lane >> 2;
  const int i = base + g;
  const bool valid = i < a.n;
  const int len = valid ? __ldg(a.rp + i + 1) - __ldg(a.rp + i) : 0;
  const bool is_long = len > kSpmvLong;
  double s = row_dot_q(a, i, valid && !is_long, x, q);
  unsigned m = __ballot_sync(0xffffffffu, is_long && q == 0);
  while (m) {
    const int gl = (__ffs(m) - 1) >> 2;
    m &= m - 1;
    const int ii = base + gl;
    const int e0 = __ldg(a.rp + ii), e1 = __ldg(a.rp + ii + 1);
    double t0 = 0.0, t1 = 0.0;
    int k = e0 + lane;
    for (; k + 32 < e1; k += 64) {
      t0 = fma(static_cast<double>(__ldg(a.v + k)), x[__ldg(a.ci + k)], t0);
      t1 = fma(static_cast<double>(__ldg(a.v + k + 32)), x[__ldg(a.ci + k + 32)], t1);
    }
    if (k < e1) t0 = fma(static_cast<double>(__ldg(a.v + k)), x[__ldg(a.ci + k)], t0);
    double t = t0 + t1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (g == gl) s = t;
  }
  return s;
}

// y = A x (fp64 vectors).
__global__ void __launch_bounds__(kThreads)
k_spmv_f64(DevCsr a, const double* __restrict__ x, double* __restrict__ y) {
  const int lane = threadIdx.x & 31, q = lane & 3;
  const int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int base = wg * 8; base < a.n; base += nw * 8) {
    const int i = base + (lane >> 2);
    const double s = row_dot_warp8(a, base, x, lane);
    if (q == 0 && i < a.n) y[i] = s;
  }
}

// w = A z_j; Z[:, j] = z_j when preconditioned.
__global__ void __launch_bounds__(kThreads) k_krylov_spmv(DevCsr a, KrylovDev k) {
  if (k.st->stop) return;
  const int j = k.st->j;
  const double* z = k.Z ? k.zout : k.V + static_cast<size_t>(j) * k.n;
  const int lane = threadIdx.x & 31, q = lane & 3;
  const int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int base = wg * 8; base < a.n; base += nw * 8) {
    const int i = base + (lane >> 2);
    const double s = row_dot_warp8(a, base, z, lane);
    if (q == 0 && i < a.n) {
      k.w[i] = s;
      if (k.Z) k.Z[static_cast<size_t>(j) * k.n + i] = z[i];
    }
  }
}

// Grid-wide deterministic sum (double-buffered partials, one grid barrier).
__device__ __forceinline__ double grid_sum(cg::grid_group& grid, double v, double* partials,
                                           int& phase, double* scratch) {
  v = block_sum(v, scratch);
  double* buf = partials + (phase & 1) * gridDim.x;
  if (threadIdx.x == 0) buf[blockIdx.x] = v;
  grid.sync();
  double t = 0.0;
  for (int q = threadIdx.x; q < (int)gridDim.x; q += blockDim.x)
    t += reinterpret_cast<volatile double*>(buf)[q];
  t = block_sum(t, scratch);
  ++phase;
  return t;
}

__device__ __forceinline__ double rot_a(double c, double s, double t1, double t2) {
  return __dadd_rn(__dmul_rn(c, t1), __dmul_rn(s, t2));  // c t1 + s t2, no contraction
}
__device__ __forceinline__ double rot_b(double c, double s, double t1, double t2) {
  return __dadd_rn(__dmul_rn(-s, t1), __dmul_rn(c, t2));  // -s t1 + c t2
}

// Block 0 / thread 0 tail of a step: Givens on column j, tracked residual,
// history, stop rule (src/krylov.cpp:221-238).
__device__ void givens_and_state(KrylovDev& k, int j, double wnorm, bool brk, bool reo) {
  KState* st = k.st;
  const int ld = k.m + 1;
  double* Hj = k.H + static_cast<size_t>(j) * ld;
  double* Rj = k.R + static_cast<size_t>(j) * ld;
  Hj[j + 1] = wnorm;
  for (int i = 0; i <= j + 1; ++i) Rj[i] = Hj[i];
  for (int i = 0; i < j; ++i) {
    const double t1 = Rj[i], t2 = Rj[i + 1];
    Rj[i] = rot_a(k.cs[i], k.sn[i], t1, t2);
    Rj[i + 1] = rot_b(k.cs[i], k.sn[i], t1, t2);
  }
  const double av = Rj[j], bv = Rj[j + 1];
  const double den = hypot(av, bv);
  const double c = den == 0.0 ? 1.0 : av / den;
  const double s = den == 0.0 ? 0.0 : bv / den;
  Rj[j] = rot_a(c, s, av, bv);
  Rj[j + 1] = rot_b(c, s, av, bv);
  k.cs[j] = c;
  k.sn[j] = s;
  const double t1 = k.g[j], t2 = k.g[j + 1];
  k.g[j] = rot_a(c, s, t1, t2);
  k.g[j + 1] = rot_b(c, s, t1, t2);
  const double tracked_rel = fabs(k.g[j + 1]) / st->bnorm;
  st->tracked_rel = tracked_rel;
  st->steps = j + 1;
  st->iter += 1;
  if (reo) st->reorth += 1;
  const long long now = static_cast<long long>(globaltimer_ns());
  k.hist_rel[j] = tracked_rel;
  k.hist_t[j] = now - st->t0;
  int stop = 0;
  if (brk) st->breakdown = 1;
  if (brk || tracked_rel <= st->rtol) {
    stop = 1;
  } else if (st->deadline >= 0 && now >= st->deadline) {
    st->budget_hit = 1;
    st->budget_status = 2;
    stop = 1;
  } else if (st->iter >= st->maxiters) {
    st->budget_hit = 1;
    st->budget_status = 1;
    stop = 1;
  }
  st->j = j + 1;
  __threadfence();
  st->stop = stop || (j + 1 >= st->cycle);
}

// EPT > 0: w lives in registers (EPT elements per thread, strided by the grid
// size); EPT == 0: w stays in global memory.
template <int EPT>
__global__ void __launch_bounds__(kThreads) k_krylov_ortho(KrylovDev k) {
  cg::grid_group grid = cg::this_grid();
  KState* st = k.st;
  if (st->stop) return;
  const int j = st->j;
  const int n = k.n;
  const int T = gridDim.x * blockDim.x;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  __shared__ double scratch[32];
  int phase = 0;
  constexpr int E = EPT > 0 ? EPT : 1;
  double w[E];
  double p = 0.0;
  if constexpr (EPT > 0) {
#pragma unroll
    for (int t = 0; t < EPT; ++t) {
      const int e = gt + t * T;
      w[t] = e < n ? k.w[e] : 0.0;
      p = fma(w[t], w[t], p);
    }
  } else {
    for (int e = gt; e < n; e += T) p = fma(k.w[e], k.w[e], p);
  }
  const double wnorm0 = sqrt(grid_sum(grid, p, k.partials, phase, scratch));
  const int ld = k.m + 1;
  double* Hj = k.H + static_cast<size_t>(j) * ld;

  // One MGS pass over v_0..v_j; returns ||w|| afterwards.  With w in
  // registers, v_s also stays in registers from its dot (step s) to its axpy
  // (step s + 1): every basis vector is read once per pass.
  // v_{s+1} is requested before step s's grid barrier (vnx), so its load
  // latency hides behind the barrier instead of following it.
  double vc[E], vnx[E];
  auto mgs_pass = [&](bool add) -> double {
    double hprev = 0.0;
    if constexpr (EPT > 0) {
#pragma unroll
      for (int t = 0; t < EPT; ++t) {
        const int e = gt + t * T;
        vnx[t] = e < n ? k.V[e] : 0.0;  // v_0
      }
    }
    for (int s = 0; s <= j + 1; ++s) {
      const double* vprev = k.V + static_cast<size_t>(s > 0 ? s - 1 : 0) * n;
      const double* vs = k.V + static_cast<size_t>(s) * n;
      double part = 0.0;
      if constexpr (EPT > 0) {
#pragma unroll
        for (int t = 0; t < EPT; ++t) {
          const int e = gt + t * T;
          if (e < n) {
            if (s > 0) w[t] = fma(-hprev, vc[t], w[t]);
            if (s <= j) {
              vc[t] = vnx[t];
              part = fma(w[t], vc[t], part);
            } else {
              part = fma(w[t], w[t], part);
            }
          }
        }
        if (s + 1 <= j) {
          const double* vn1 = vs + n;
#pragma unroll
          for (int t = 0; t < EPT; ++t) {
            const int e = gt + t * T;
            if (e < n) vnx[t] = vn1[e];
          }
        }
      } else {
        for (int e = gt; e < n; e += T) {
          double we = k.w[e];
          if (s > 0) {
            we = fma(-hprev, vprev[e], we);
            k.w[e] = we;
          }
          part = s <= j ? fma(we, vs[e], part) : fma(we, we, part);
        }
      }
      const double tot = grid_sum(grid, part, k.partials, phase, scratch);
      if (s <= j) {
        hprev = tot;
        if (gt == 0) Hj[s] = add ? Hj[s] + tot : tot;
      } else {
        return sqrt(tot);
      }
    }
    return 0.0;
  };

  double wnorm = mgs_pass(false);
  const bool reo = wnorm < 0.70710678118654752440 * wnorm0;
  if (reo) wnorm = mgs_pass(true);
  const bool brk = wnorm <= 1e-14 * wnorm0;
  if (!brk) {
    double* vn = k.V + static_cast<size_t>(j + 1) * n;
    if constexpr (EPT > 0) {
#pragma unroll
      for (int t = 0; t < EPT; ++t) {
        const int e = gt + t * T;
        if (e < n) {
          const double v = w[t] / wnorm;
          vn[e] = v;
          k.vin[e] = v;
        }
      }
    } else {
      for (int e = gt; e < n; e += T) {
        const double v = k.w[e] / wnorm;
        vn[e] = v;
        k.vin[e] = v;
      }
    }
  }
  if (gt == 0) givens_and_state(k, j, wnorm, brk, reo);
}

// The same step for vectors too long for w in registers at any grid size
// (C5: n = 4.19M): one 1024-thread CTA per SM owns a contiguous chunk of w,
// NR elements per thread in registers and the rest in shared memory, so w
// never goes back to HBM during the MGS sweeps; only the basis vectors stream
// (v_s once per step; v_{s-1} again for the shared-memory part, from L2).
// Arithmetic per element and the reductions are those of k_krylov_ortho.
constexpr int kOnchipThreads = 1024;
template <int NR>
__global__ void __launch_bounds__(kOnchipThreads, 1) k_krylov_ortho_onchip(KrylovDev k, int chunk) {
  cg::grid_group grid = cg::this_grid();
  KState* st = k.st;
  if (st->stop) return;
  extern __shared__ double wsm[];
  const int j = st->j;
  const int n = k.n;
  const int tid = threadIdx.x;
  const int base = blockIdx.x * chunk;
  const int len = max(0, min(chunk, n - base));
  constexpr int RB = NR * kOnchipThreads;  // chunk elements held in registers
  __shared__ double scratch[32];
  int phase = 0;
  double w[NR > 0 ? NR : 1], vc[NR > 0 ? NR : 1];
  double p = 0.0;
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const int c = r * kOnchipThreads + tid;
    w[r] = c < len ? k.w[base + c] : 0.0;
    p = fma(w[r], w[r], p);
  }
  for (int c = RB + tid; c < len; c += kOnchipThreads) {
    const double we = k.w[base + c];
    wsm[c - RB] = we;
    p = fma(we, we, p);
  }
  const double wnorm0 = sqrt(grid_sum(grid, p, k.partials, phase, scratch));
  const int ld = k.m + 1;
  double* Hj = k.H + static_cast<size_t>(j) * ld;

  auto mgs_pass = [&](bool add) -> double {
    double hprev = 0.0;
    for (int s = 0; s <= j + 1; ++s) {
      const double* vprev = k.V + static_cast<size_t>(s > 0 ? s - 1 : 0) * n + base;
      const double* vs = k.V + static_cast<size_t>(s) * n + base;
      double part = 0.0;
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const int c = r * kOnchipThreads + tid;
        if (c < len) {
          if (s > 0) w[r] = fma(-hprev, vc[r], w[r]);
          if (s <= j) {
            vc[r] = vs[c];
            part = fma(w[r], vc[r], part);
          } else {
            part = fma(w[r], w[r], part);
          }
        }
      }
      // (four elements per trip with their loads issued together: the loop
      // was latency-bound at one v_s / v_{s-1} pair in flight per thread)
      int c = RB + tid;
      for (; c + 3 * kOnchipThreads < len; c += 4 * kOnchipThreads) {
        double vp[4], vv[4], we[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          vp[u] = s > 0 ? vprev[c + u * kOnchipThreads] : 0.0;
          vv[u] = s <= j ? vs[c + u * kOnchipThreads] : 0.0;
          we[u] = wsm[c + u * kOnchipThreads - RB];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (s > 0) {
            we[u] = fma(-hprev, vp[u], we[u]);
            wsm[c + u * kOnchipThreads - RB] = we[u];
          }
          part = s <= j ? fma(we[u], vv[u], part) : fma(we[u], we[u], part);
        }
      }
      for (; c < len; c += kOnchipThreads) {
        double we = wsm[c - RB];
        if (s > 0) {
          we = fma(-hprev, vprev[c], we);
          wsm[c - RB] = we;
        }
        part = s <= j ? fma(we, vs[c], part) : fma(we, we, part);
      }
      const double tot = grid_sum(grid, part, k.partials, phase, scratch);
      if (s <= j) {
        hprev = tot;
        if (blockIdx.x == 0 && tid == 0) Hj[s] = add ? Hj[s] + tot : tot;
      } else {
        return sqrt(tot);
      }
    }
    return 0.0;
  };

  double wnorm = mgs_pass(false);
  const bool reo = wnorm < 0.70710678118654752440 * wnorm0;
  if (reo) wnorm = mgs_pass(true);
  const bool brk = wnorm <= 1e-14 * wnorm0;
  if (!brk) {
    double* vn = k.V + static_cast<size_t>(j + 1) * n + base;
    double* vi = k.vin + base;
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const int c = r * kOnchipThreads + tid;
      if (c < len) {
        const double v = w[r] / wnorm;
        vn[c] = v;
        vi[c] = v;
      }
    }
    for (int c = RB + tid; c < len; c += kOnchipThreads) {
      const double v = wsm[c - RB] / wnorm;
      vn[c] = v;
      vi[c] = v;
    }
  }
  if (blockIdx.x == 0 && tid == 0) givens_and_state(k, j, wnorm, brk, reo);
}

// r = b - A x (src/krylov.cpp:194-199), ||r|| with a last-block finish;
// writes st->current = ||r||/bnorm, st->beta = ||r||, st->t_end.
__global__ void __launch_bounds__(kThreads) k_residual(DevCsr a, KrylovDev k) {
  __shared__ double scratch[32];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, q = lane & 3;
  const int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  double p = 0.0;
  for (int base = wg * 8; base < a.n; base += nw * 8) {
    const int i = base + (lane >> 2);
    const double s = row_dot_warp8(a, base, k.x, lane);
    if (q == 0 && i < a.n) {
      const double ri = k.b[i] + -1.0 * s;
      k.r[i] = ri;
      p = fma(ri, ri, p);
    }
  }
  p = block_sum(p, scratch);
  if (threadIdx.x == 0) {
    k.partials[blockIdx.x] = p;
    __threadfence();
    last = atomicAdd(k.ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double t = 0.0;
  for (int z = threadIdx.x; z < (int)gridDim.x; z += blockDim.x)
    t += reinterpret_cast<volatile double*>(k.partials)[z];
  t = block_sum(t, scratch);
  if (threadIdx.x == 0) {
    const double rn = sqrt(t);
    k.st->beta = rn;
    k.st->current = rn / k.st->bnorm;
    k.st->t_end = static_cast<long long>(globaltimer_ns()) - k.st->t0;
    *k.ticket = 0u;
  }
}

// v_0 = r0 / beta (src/krylov.cpp:25), vin = v_0, reset the cycle state.
__global__ void __launch_bounds__(kThreads) k_cycle_begin(KrylovDev k, int cycle) {
  const double beta = k.st->beta;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < k.n; e += gridDim.x * blockDim.x) {
    const double v = k.r[e] / beta;
    k.V[e] = v;
    k.vin[e] = v;
  }
  if (blockIdx.x == 0) {
    for (int t = threadIdx.x; t < (k.m + 1) * k.m; t += blockDim.x) {
      k.H[t] = 0.0;
      k.R[t] = 0.0;
    }
    for (int t = threadIdx.x; t <= k.m; t += blockDim.x) k.g[t] = t == 0 ? beta : 0.0;
    if (threadIdx.x == 0) {
      KState* st = k.st;
      st->j = 0;
      st->steps = 0;
      st->cycle = cycle;
      st->breakdown = 0;
      st->budget_hit = 0;
      st->budget_status = 1;
      st->singular = 0;
      st->tracked_rel = beta / st->bnorm;
      st->stop = 0;
    }
  }
}

// Back-substitution on the rotated factor (src/krylov.cpp:160-172).
__global__ void k_cycle_solve(KrylovDev k) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  KState* st = k.st;
  const int kk = st->steps, ld = k.m + 1;
  for (int i = 0; i < kk; ++i) k.y[i] = 0.0;
  st->tracked_rel = fabs(k.g[kk]) / st->bnorm;
  st->singular = 0;
  for (int jj = kk - 1; jj >= 0; --jj) {
    const double d = k.R[static_cast<size_t>(jj) * ld + jj];
    if (d == 0.0) {
      st->singular = 1;
      return;
    }
    double s = k.g[jj];
    for (int col = jj + 1; col < kk; ++col)
      s = __dadd_rn(s, -__dmul_rn(k.R[static_cast<size_t>(col) * ld + jj], k.y[col]));
    k.y[jj] = s / d;
  }
}

// x += Z[:, :k] y in basis order (src/krylov.cpp:97-102).
__global__ void __launch_bounds__(kThreads) k_update_x(KrylovDev k) {
  const KState* st = k.st;
  if (st->singular) return;
  const int kk = st->steps;
  const double* Zb = k.Z ? k.Z : k.V;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < k.n; e += gridDim.x * blockDim.x) {
    double xe = k.x[e];
    for (int jj = 0; jj < kk; ++jj) xe = fma(Zb[static_cast<size_t>(jj) * k.n + e], k.y[jj], xe);
    k.x[e] = xe;
  }
}

}  // namespace gnpk
