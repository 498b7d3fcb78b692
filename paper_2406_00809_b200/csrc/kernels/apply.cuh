// GNP apply M(b) on sm_100a: norm → lift → L fused Res-GCONV layers (last one
// fused with the projection MLP).  Restates gnn_forward (src/gnn.cpp:120-201)
// in fp32 with fp32 accumulation; the data path per layer streams Â and X from
// HBM once (row-major n x DP feature blocks, DP = d padded to a power of two
// >= 4 with zero weights, so padding is exact).
#pragma once

#include "common.cuh"

namespace gnpk {

// Device fp32 parameters, padded to DP (see model upload in capi.cu).
struct NetView {
  const float* enc1;    // [hidden]
  const float* enc1_b;  // [hidden]
  const float* enc2;    // [hidden][DP]  row-major (h, j)
  const float* enc2_b;  // [DP]
  const float* uw;      // [layers][2*DP][DP]: rows 0..DP-1 = U(k, j), rows DP.. = W(k, j)
  const float* dec1;    // [DP][hidden]  row-major (j, h)
  const float* dec1_b;  // [hidden]
  const float* dec2;    // [hidden]
  float dec2_b;
  const float* dec2_bp;  // the same value in device memory (training reads it)
  int hidden;
  int layers;
  // Exact piecewise-linear form of the lift v -> enc2ᵀ relu(v enc1 + b1) + b2:
  // nbreak sorted kinks t_k = -b1_h/enc1_h; on interval k (#kinks <= v),
  // x1 = lift_a[k] * v + lift_b[k]   ([nbreak+1][DP] each, built in f64).
  const float* lift_t;
  const float* lift_a;
  const float* lift_b;
  int nbreak;
};

// ------------------------------------------------------------------ node renumbering
// Ragged matrices run the apply on length-sorted nodes (DevCsr::perm): the
// lift reads b[perm[i]] (the norm reads b in its own order, so τ does not
// depend on the layout), and dst[perm[i]] = src[i] after the last layer.
template <typename T>
__global__ void __launch_bounds__(kThreads)
k_perm_scatter(const T* __restrict__ src, const int* __restrict__ perm, int n, T* __restrict__ dst,
               const int* __restrict__ skip) {
  if (skip && *skip) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[perm[i]] = src[i];
}

// ------------------------------------------------------------------ lift (piecewise)
// Same map as k_lift: per row one binary search over <= hidden kinks, then
// DP FMAs (the H x DP MLP collapses because its input is a scalar).
template <int DP, typename T>
__global__ void __launch_bounds__(kThreads)
k_lift_pw(const T* __restrict__ in, int n, NetView net, const ApplyScalars* __restrict__ sc,
          float* __restrict__ X, const int* __restrict__ skip, const int* __restrict__ perm = nullptr) {
  if (skip && *skip) return;
  if (sc->zero) return;
  constexpr int G = DP / 4, NG = kThreads / G;
  extern __shared__ float4 sm4[];
  const int nb = net.nbreak;
  float* s_a = reinterpret_cast<float*>(sm4);  // [nb+1][DP]
  float* s_b = s_a + (nb + 1) * DP;            // [nb+1][DP]
  float* s_t = s_b + (nb + 1) * DP;            // [nb]
  for (int t = threadIdx.x; t < (nb + 1) * DP; t += kThreads) {
    s_a[t] = net.lift_a[t];
    s_b[t] = net.lift_b[t];
  }
  for (int t = threadIdx.x; t < nb; t += kThreads) s_t[t] = net.lift_t[t];
  __syncthreads();
  const int gl = threadIdx.x % G;
  const double in_scale = sc->in_scale;
  for (int row = blockIdx.x * NG + threadIdx.x / G; row < n; row += gridDim.x * NG) {
    const float v = static_cast<float>(in_scale * static_cast<double>(in[perm ? perm[row] : row]));
    int lo = 0, hi = nb;  // interval = #kinks <= v
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (s_t[mid] <= v) lo = mid + 1;
      else hi = mid;
    }
    const float4 al = *reinterpret_cast<const float4*>(s_a + lo * DP + 4 * gl);
    const float4 be = *reinterpret_cast<const float4*>(s_b + lo * DP + 4 * gl);
    st4(X + static_cast<size_t>(row) * DP + 4 * gl,
        make_float4(fmaf(al.x, v, be.x), fmaf(al.y, v, be.y), fmaf(al.z, v, be.z), fmaf(al.w, v, be.w)));
  }
}

// ------------------------------------------------------------------ τ = ||b||
// Block partials in f64 + last-block finalisation in a fixed order, so the
// result is deterministic for a fixed grid.  Restates src/gnn.cpp:128-136.
template <typename T>
__global__ void __launch_bounds__(kThreads)
k_apply_norm(const T* __restrict__ in, int n, double* __restrict__ partials,
             unsigned* __restrict__ ticket, ApplyScalars* __restrict__ sc,
             const int* __restrict__ skip) {
  if (skip && *skip) return;
  __shared__ double scratch[32];
  __shared__ bool last;
  // 8 independent loads in flight per thread (the loop was load-latency
  // bound: C5 35 us for 16.8 MB); the fixed order keeps it deterministic
  double s = 0.0;
  const int stride = gridDim.x * blockDim.x;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n; i += 8 * stride) {
    double x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = static_cast<double>(in[i + u * stride]);
#pragma unroll
    for (int u = 0; u < 8; ++u) s = fma(x[u], x[u], s);
  }
  for (; i < n; i += stride) {
    const double x = static_cast<double>(in[i]);
    s = fma(x, x, s);
  }
  s = block_sum(s, scratch);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = s;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double t = 0.0;
  for (int k = threadIdx.x; k < (int)gridDim.x; k += blockDim.x)
    t += reinterpret_cast<volatile double*>(partials)[k];
  t = block_sum(t, scratch);
  if (threadIdx.x == 0) {
    const double tau = sqrt(t);
    const double sn = sqrt(static_cast<double>(n));
    sc->tau = tau;
    sc->zero = tau == 0.0;
    sc->in_scale = tau == 0.0 ? 0.0 : sn / tau;
    sc->out_scale = tau / sn;
    *ticket = 0u;
  }
}

// ------------------------------------------------------------------ lift
// x1_i = enc2ᵀ relu(v_i enc1 + enc1_b) + enc2_b, v_i = (sqrt(n)/τ) b_i
// (src/gnn.cpp:138-157).  G = DP/4 lanes per row, each owning 4 features.
template <int DP, typename T>
__global__ void __launch_bounds__(kThreads)
k_lift(const T* __restrict__ in, int n, NetView net, const ApplyScalars* __restrict__ sc,
       float* __restrict__ X, const int* __restrict__ skip) {
  if (skip && *skip) return;
  if (sc->zero) return;
  constexpr int G = DP / 4, NG = kThreads / G;
  extern __shared__ float4 sm4[];
  float* sm = reinterpret_cast<float*>(sm4);
  const int H = net.hidden;
  float* s_enc2 = sm;                  // [H][DP]
  float* s_enc1 = s_enc2 + H * DP;     // [H]
  float* s_b1 = s_enc1 + H;            // [H]
  for (int t = threadIdx.x; t < H * DP; t += kThreads) s_enc2[t] = net.enc2[t];
  for (int t = threadIdx.x; t < H; t += kThreads) {
    s_enc1[t] = net.enc1[t];
    s_b1[t] = net.enc1_b[t];
  }
  __syncthreads();
  const int gl = threadIdx.x % G;
  const float4 b2 = ldg4(net.enc2_b + 4 * gl);
  const double in_scale = sc->in_scale;
  for (int row = blockIdx.x * NG + threadIdx.x / G; row < n; row += gridDim.x * NG) {
    const float v = static_cast<float>(in_scale * static_cast<double>(in[row]));
    float4 acc = f4zero();
    for (int h = 0; h < H; ++h) {
      const float t = relu(fmaf(v, s_enc1[h], s_b1[h]));
      fma4(acc, t, *reinterpret_cast<const float4*>(s_enc2 + h * DP + 4 * gl));
    }
    st4(X + static_cast<size_t>(row) * DP + 4 * gl, add4(acc, b2));
  }
}

// ------------------------------------------------------------------ long rows
// (ÂX)_i for rows with > kLongRow nonzeros: one CTA per row, the CTA's groups
// stride the row's nonzeros, then a fixed-order smem tree (deterministic).
template <int DP>
__global__ void __launch_bounds__(kThreads)
k_long_ax(DevCsr a, const float* __restrict__ X, float* __restrict__ AXL,
          const ApplyScalars* __restrict__ sc, const int* __restrict__ skip) {
  if (skip && *skip) return;
  if (sc && sc->zero) return;
  constexpr int G = DP / 4, NG = kThreads / G;
  __shared__ float4 red[kThreads];
  const int i = a.long_rows[blockIdx.x];
  const int gl = threadIdx.x % G, gid = threadIdx.x / G;
  float4 acc = f4zero();
  const int e = a.rp[i + 1];
  for (int k = a.rp[i] + gid; k < e; k += NG)
    fma4(acc, __ldg(a.v + k), ldg4(X + static_cast<size_t>(__ldg(a.ci + k)) * DP + 4 * gl));
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = NG / 2; s > 0; s >>= 1) {
    if (gid < s) red[threadIdx.x] = add4(red[threadIdx.x], red[threadIdx.x + s * G]);
    __syncthreads();
  }
  if (gid == 0) st4(AXL + static_cast<size_t>(i) * DP + 4 * gl, red[threadIdx.x]);
}

// Long rows, load-balanced: every long row is cut into chunks of <= kChunk
// nonzeros; one warp per chunk (32/G groups striding the chunk, shuffle tree
// across groups) writes a partial (ÂX) row, then k_long_combine sums each
// row's partials in chunk order (deterministic) into AXL.
constexpr int kChunk = 128;

struct LongPlan {
  int nchunks;
  const int* chunk_row;   // [nchunks]
  const int* chunk_k0;    // [nchunks]
  const int* chunk_k1;    // [nchunks]
  int nrows;
  const int* rows;        // [nrows] long rows
  const int* row_c0;      // [nrows + 1] chunk range of each long row
  float* partial;         // [nchunks][DP]
};

template <int DP>
__global__ void __launch_bounds__(kThreads)
k_long_chunks(DevCsr a, LongPlan lp, const float* __restrict__ X,
              const ApplyScalars* __restrict__ sc, const int* __restrict__ skip) {
  if (skip && *skip) return;
  if (sc && sc->zero) return;
  constexpr int G = DP / 4, NGW = 32 / G;  // groups per warp
  const int lane = threadIdx.x & 31, gl = lane % G, grp = lane / G;
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (c >= lp.nchunks) return;
  const int k0 = lp.chunk_k0[c], k1 = lp.chunk_k1[c];
  float4 acc = f4zero();
  int k = k0 + grp;
  // L2: the chunk's (col, val) stream evict_first, the X gathers evict_last
  const uint64_t ps = a.l2hint ? l2_policy_evict_first() : l2_policy_evict_normal();
  const uint64_t pk = a.l2hint ? l2_policy_evict_last() : l2_policy_evict_normal();
  for (; k + 3 * NGW < k1; k += 4 * NGW) {
    const int c0 = ldg_hint(a.ci + k, ps), c1 = ldg_hint(a.ci + k + NGW, ps);
    const int c2 = ldg_hint(a.ci + k + 2 * NGW, ps), c3 = ldg_hint(a.ci + k + 3 * NGW, ps);
    const float v0 = ldg_hint(a.v + k, ps), v1 = ldg_hint(a.v + k + NGW, ps);
    const float v2 = ldg_hint(a.v + k + 2 * NGW, ps), v3 = ldg_hint(a.v + k + 3 * NGW, ps);
    const float4 x0 = ldg4_hint(X + static_cast<size_t>(c0) * DP + 4 * gl, pk);
    const float4 x1 = ldg4_hint(X + static_cast<size_t>(c1) * DP + 4 * gl, pk);
    const float4 x2 = ldg4_hint(X + static_cast<size_t>(c2) * DP + 4 * gl, pk);
    const float4 x3 = ldg4_hint(X + static_cast<size_t>(c3) * DP + 4 * gl, pk);
    fma4(acc, v0, x0);
    fma4(acc, v1, x1);
    fma4(acc, v2, x2);
    fma4(acc, v3, x3);
  }
  for (; k < k1; k += NGW)
    fma4(acc, ldg_hint(a.v + k, ps), ldg4_hint(X + static_cast<size_t>(ldg_hint(a.ci + k, ps)) * DP + 4 * gl, pk));
#pragma unroll
  for (int o = G; o < 32; o <<= 1) {
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    acc.z += __shfl_xor_sync(0xffffffffu, acc.z, o);
    acc.w += __shfl_xor_sync(0xffffffffu, acc.w, o);
  }
  if (grp == 0) st4(lp.partial + static_cast<size_t>(c) * DP + 4 * gl, acc);
}

template <int DP>
__global__ void __launch_bounds__(kThreads)
k_long_combine(LongPlan lp, float* __restrict__ AXL, const ApplyScalars* __restrict__ sc,
               const int* __restrict__ skip) {
  if (skip && *skip) return;
  if (sc && sc->zero) return;
  constexpr int G = DP / 4;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int lr = t / G, gl = t % G;
  if (lr >= lp.nrows) return;
  float4 s = f4zero();
  for (int c = lp.row_c0[lr]; c < lp.row_c0[lr + 1]; ++c)
    s = add4(s, ldg4(lp.partial + static_cast<size_t>(c) * DP + 4 * gl));
  st4(AXL + static_cast<size_t>(lp.rows[lr]) * DP + 4 * gl, s);
}

// ------------------------------------------------------------------ fused layer
// Y = relu(X U + (Â X) W) for a tile of TM rows (src/gnn.cpp:164-176):
//   phase 1 (gather): G lanes per row stream the row's nonzeros with 128-bit
//            X-row loads, fp32 sums in stored (sorted-column) order;
//            [x_i | (ÂX)_i] staged in smem.
//   phase 2 (transform): register-blocked [TM x 2DP]·[2DP x DP] with [U; W]
//            in smem; each output is one fp32 sum over k = 0..2DP-1
//            (x·U then ÂX·W, the reference's XU + ÂXW grouping up to order).
//   LAST: relu'd tile goes back to smem and a thread per row runs the
//         projection MLP (src/gnn.cpp:178-199) and the τ/sqrt(n) unscale.
template <int DP>
struct LayerCfg {
  static constexpr int G = DP / 4;          // gather lanes per row
  static constexpr int CB = DP / 4;         // float4 column blocks
  static constexpr int RB = kThreads / CB;  // row slots in the transform
  static constexpr int TM = RB > 128 ? RB : 128;
  static constexpr int R = TM / RB;         // rows per thread in the transform
  static constexpr int SK = 2 * DP + 4;     // smem stride (floats) of the [x|ax] tile
  static size_t smem_bytes(bool last, int hidden) {
    size_t b = (size_t)TM * SK * 4 + (size_t)2 * DP * DP * 4;
    if (last) b += ((size_t)DP * hidden + 2 * (size_t)hidden) * 4;
    return b;
  }
};

template <int DP, bool LAST, typename OutT>
__global__ void __launch_bounds__(kThreads)
k_layer(DevCsr a, const float* __restrict__ X, float* __restrict__ Y,
        const float* __restrict__ uw, const float* __restrict__ axlong, NetView net,
        const ApplyScalars* __restrict__ sc, OutT* __restrict__ out,
        const int* __restrict__ skip) {
  using C = LayerCfg<DP>;
  constexpr int G = C::G, CB = C::CB, RB = C::RB, TM = C::TM, R = C::R, SK = C::SK;
  constexpr int NG = kThreads / G;
  if (skip && *skip) return;
  const int row0 = blockIdx.x * TM;
  if (sc->zero) {
    if constexpr (LAST) {
      for (int r = threadIdx.x; r < TM; r += kThreads)
        if (row0 + r < a.n) out[row0 + r] = OutT(0);
    }
    return;
  }
  extern __shared__ float4 sm4[];
  float* S = reinterpret_cast<float*>(sm4);  // [TM][SK]
  float* W = S + TM * SK;                    // [2DP][DP]
  for (int t = threadIdx.x; t < 2 * DP * DP / 4; t += kThreads)
    sm4[(TM * SK) / 4 + t] = reinterpret_cast<const float4*>(uw)[t];
  if constexpr (LAST) {
    float* D1 = W + 2 * DP * DP;
    const int H = net.hidden;
    for (int t = threadIdx.x; t < DP * H; t += kThreads) D1[t] = net.dec1[t];
    for (int t = threadIdx.x; t < H; t += kThreads) {
      D1[DP * H + t] = net.dec1_b[t];
      D1[DP * H + H + t] = net.dec2[t];
    }
  }

  // ---- phase 1: gather
  {
    const int gl = threadIdx.x % G, gid = threadIdx.x / G;
    for (int r = gid; r < TM; r += NG) {
      const int i = row0 + r;
      float4 ax = f4zero(), xi = f4zero();
      if (i < a.n) {
        const int s = __ldg(a.rp + i), e = __ldg(a.rp + i + 1);
        if (axlong != nullptr && e - s > kLongRow) {
          ax = ldg4(axlong + static_cast<size_t>(i) * DP + 4 * gl);
        } else {
          int k = s;
          for (; k + 4 <= e; k += 4) {
            const int c0 = __ldg(a.ci + k), c1 = __ldg(a.ci + k + 1);
            const int c2 = __ldg(a.ci + k + 2), c3 = __ldg(a.ci + k + 3);
            const float v0 = __ldg(a.v + k), v1 = __ldg(a.v + k + 1);
            const float v2 = __ldg(a.v + k + 2), v3 = __ldg(a.v + k + 3);
            const float4 x0 = ldg4(X + static_cast<size_t>(c0) * DP + 4 * gl);
            const float4 x1 = ldg4(X + static_cast<size_t>(c1) * DP + 4 * gl);
            const float4 x2 = ldg4(X + static_cast<size_t>(c2) * DP + 4 * gl);
            const float4 x3 = ldg4(X + static_cast<size_t>(c3) * DP + 4 * gl);
            fma4(ax, v0, x0);
            fma4(ax, v1, x1);
            fma4(ax, v2, x2);
            fma4(ax, v3, x3);
          }
          for (; k < e; ++k)
            fma4(ax, __ldg(a.v + k), ldg4(X + static_cast<size_t>(__ldg(a.ci + k)) * DP + 4 * gl));
        }
        xi = ldg4(X + static_cast<size_t>(i) * DP + 4 * gl);
      }
      st4(S + r * SK + 4 * gl, xi);
      st4(S + r * SK + DP + 4 * gl, ax);
    }
  }
  __syncthreads();

  // ---- phase 2: transform
  const int cb = threadIdx.x % CB, rb = threadIdx.x / CB;
  float4 acc[R];
#pragma unroll
  for (int r = 0; r < R; ++r) acc[r] = f4zero();
  const float4* W4 = reinterpret_cast<const float4*>(W);
#pragma unroll 4
  for (int k = 0; k < 2 * DP; k += 4) {
    const float4 w0 = W4[(k + 0) * CB + cb];
    const float4 w1 = W4[(k + 1) * CB + cb];
    const float4 w2 = W4[(k + 2) * CB + cb];
    const float4 w3 = W4[(k + 3) * CB + cb];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const float4 s = *reinterpret_cast<const float4*>(S + (rb + r * RB) * SK + k);
      fma4(acc[r], s.x, w0);
      fma4(acc[r], s.y, w1);
      fma4(acc[r], s.z, w2);
      fma4(acc[r], s.w, w3);
    }
  }

  if constexpr (!LAST) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = row0 + rb + r * RB;
      if (i < a.n) st4(Y + static_cast<size_t>(i) * DP + 4 * cb, relu4(acc[r]));
    }
  } else {
    __syncthreads();  // everyone is done reading the [x|ax] tile
#pragma unroll
    for (int r = 0; r < R; ++r) st4(S + (rb + r * RB) * SK + 4 * cb, relu4(acc[r]));
    __syncthreads();
    const int H = net.hidden;
    const float* D1 = W + 2 * DP * DP;
    const float* B1 = D1 + DP * H;
    const float* D2 = B1 + H;
    const double out_scale = sc->out_scale;
    for (int r = threadIdx.x; r < TM; r += kThreads) {
      const int i = row0 + r;
      if (i >= a.n) continue;
      float y[DP];
#pragma unroll
      for (int j = 0; j < DP; j += 4) {
        const float4 t = *reinterpret_cast<const float4*>(S + r * SK + j);
        y[j] = t.x; y[j + 1] = t.y; y[j + 2] = t.z; y[j + 3] = t.w;
      }
      float o = 0.f;
      for (int h = 0; h < H; ++h) {
        float t = 0.f;
#pragma unroll
        for (int j = 0; j < DP; ++j) t = fmaf(y[j], D1[j * H + h], t);
        o = fmaf(relu(t + B1[h]), D2[h], o);
      }
      out[i] = static_cast<OutT>(static_cast<double>(o + net.dec2_b) * out_scale);
    }
  }
}

}  // namespace gnpk
