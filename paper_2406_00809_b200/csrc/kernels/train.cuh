// Batched GNP training on sm_100a (src/gnn.cpp:208-451).
//
// A batch of B (b, x) pairs is resident as [n][B][·]: virtual row v = i*B + k
// is sample k at node i, so every Â / Âᵀ row gather serves all B samples
// (one 4 KiB contiguous block per neighbour at B = d = 32).  Forward layers
// and the backward data-gradient layers run on k_layer_tc (tcgen05) for
// d in {16, 32}, else on k_layer_batched below.  Weight gradients are
// deterministic two-stage outer-product reductions over the n*B rows.
#pragma once

#include "apply.cuh"
#include "tc.cuh"

namespace gnpk {

struct SampleScales {
  double in_scale;   // sqrt(n)/tau_k
  double out_scale;  // tau_k/sqrt(n)
  int zero;          // tau_k == 0: sample contributes M(b)=0 and no gradient
  int pad;
};

// ------------------------------------------------------------------ tau_k
// [n][B] f64 column norms: block partials [grid][B] then one block finishes
// in fixed order (deterministic).  blockDim = 256, B <= 1024.
__global__ void __launch_bounds__(kThreads)
k_col_norm_partials(const double* __restrict__ b, int n, int B, double* __restrict__ partials) {
  extern __shared__ double red[];  // [256]
  for (int k0 = 0; k0 < B; k0 += 32) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int k = k0 + lane;
    double s = 0.0;
    if (k < B)
      for (int i = blockIdx.x * 8 + w; i < n; i += gridDim.x * 8) {
        const double x = b[static_cast<size_t>(i) * B + k];
        s = fma(x, x, s);
      }
    red[threadIdx.x] = s;
    __syncthreads();
    if (w == 0 && k < B) {
      double t = 0.0;
      for (int q = 0; q < 8; ++q) t += red[q * 32 + lane];
      partials[static_cast<size_t>(blockIdx.x) * B + k] = t;
    }
    __syncthreads();
  }
}

// One warp per sample: lane l sums blocks l, l+32, ... (8 loads in flight),
// then a fixed shuffle tree (deterministic).
__global__ void k_col_norm_finish(const double* __restrict__ partials, int nblk, int n, int B,
                                  SampleScales* __restrict__ sc) {
  const int k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (k >= B) return;
  double t = 0.0;
  int q = lane;
  for (; q + 7 * 32 < nblk; q += 8 * 32) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = partials[static_cast<size_t>(q + 32 * u) * B + k];
#pragma unroll
    for (int u = 0; u < 8; ++u) t += v[u];
  }
  for (; q < nblk; q += 32) t += partials[static_cast<size_t>(q) * B + k];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (lane != 0) return;
  const double tau = sqrt(t), sn = sqrt(static_cast<double>(n));
  sc[k].zero = tau == 0.0;
  sc[k].in_scale = tau == 0.0 ? 0.0 : sn / tau;
  sc[k].out_scale = tau / sn;
}

// ------------------------------------------------------------------ lift (batched)
// X0[v] = enc2ᵀ relu(vv enc1 + enc1_b) + enc2_b, vv = (float)(in_scale_k b[v])
// (src/gnn.cpp:138-157); also writes vv (needed by the encoder backward).
template <int DP>
__global__ void __launch_bounds__(kThreads)
k_lift_batched(const double* __restrict__ b, int nv, int B, NetView net,
               const SampleScales* __restrict__ sc, float* __restrict__ X0,
               float* __restrict__ vv_out) {
  constexpr int G = DP / 4, NG = kThreads / G;
  extern __shared__ float4 sm4[];
  const int H = net.hidden;
  float* s_enc2 = reinterpret_cast<float*>(sm4);  // [H][DP]
  float* s_enc1 = s_enc2 + H * DP;
  float* s_b1 = s_enc1 + H;
  for (int t = threadIdx.x; t < H * DP; t += kThreads) s_enc2[t] = net.enc2[t];
  for (int t = threadIdx.x; t < H; t += kThreads) {
    s_enc1[t] = net.enc1[t];
    s_b1[t] = net.enc1_b[t];
  }
  __syncthreads();
  const int gl = threadIdx.x % G;
  const float4 b2 = ldg4(net.enc2_b + 4 * gl);
  for (int v = blockIdx.x * NG + threadIdx.x / G; v < nv; v += gridDim.x * NG) {
    const int k = v % B;
    const float x = static_cast<float>(sc[k].in_scale * b[v]);
    if (gl == 0) vv_out[v] = x;
    float4 acc = f4zero();
    for (int h = 0; h < H; ++h) {
      const float t = relu(fmaf(x, s_enc1[h], s_b1[h]));
      fma4(acc, t, *reinterpret_cast<const float4*>(s_enc2 + h * DP + 4 * gl));
    }
    st4(X0 + static_cast<size_t>(v) * DP + 4 * gl, add4(acc, b2));
  }
}

// ------------------------------------------------------------------ generic batched layer
// CUDA-core layer for widths without a tcgen05 path (small test dims):
// Y = epi([X | ÂX] · Bt) with Bt[j][k] (k < 2DP) in smem; one thread per
// output element, the row's [x | ax] staged in smem.  MODE as k_layer_tc.
template <int DP, int MODE>
__global__ void __launch_bounds__(kThreads)
k_layer_batched(DevCsr a, const float* __restrict__ X, float* __restrict__ Y,
                const float* __restrict__ bt /*[DP][2DP] = B operand, row j*/,
                float* __restrict__ axout, const float* __restrict__ mask, int bs) {
  constexpr int RPB = kThreads / DP;  // virtual rows per block iteration
  __shared__ float s_bt[DP * 2 * DP];
  __shared__ float s_row[RPB][2 * DP];
  for (int t = threadIdx.x; t < DP * 2 * DP; t += kThreads) s_bt[t] = bt[t];
  __syncthreads();
  const int nv = a.n * bs;
  const int rl = threadIdx.x / DP, j = threadIdx.x % DP;
  for (int v0 = blockIdx.x * RPB; v0 < nv; v0 += gridDim.x * RPB) {
    const int v = v0 + rl;
    if (v < nv) {
      const int node = v / bs, kk = v - node * bs;
      float ax = 0.f;
      for (int q = a.rp[node]; q < a.rp[node + 1]; ++q)
        ax = fmaf(a.v[q], X[(static_cast<size_t>(a.ci[q]) * bs + kk) * DP + j], ax);
      s_row[rl][j] = X[static_cast<size_t>(v) * DP + j];
      s_row[rl][DP + j] = ax;
      if (axout) axout[static_cast<size_t>(v) * DP + j] = ax;
    }
    __syncthreads();
    if (v < nv) {
      float y = 0.f;
      for (int k = 0; k < 2 * DP; ++k) y = fmaf(s_row[rl][k], s_bt[j * 2 * DP + k], y);
      if (MODE == 0) y = relu(y);
      else if (mask && !(mask[static_cast<size_t>(v) * DP + j] > 0.f)) y = 0.f;
      Y[static_cast<size_t>(v) * DP + j] = y;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ decoder
// out[v] = (dec2 · relu(dec1ᵀ x_L + dec1_b) + dec2_b) * out_scale_k (f64 store)
// (src/gnn.cpp:178-199).  One thread per virtual row, dec1 in smem.
template <int DP>
__global__ void __launch_bounds__(32 * 4)
k_decoder_fwd(const float* __restrict__ XL, int nv, int B, NetView net,
              const SampleScales* __restrict__ sc, double* __restrict__ out);

// Warp-staged row I/O for the per-row MLP kernels below: a warp owns 32
// consecutive virtual rows (lane = row).  Rows are loaded/stored as one
// contiguous block with 16-byte coalesced accesses and transposed through a
// padded shared tile [32][W + 1] (conflict-free for a lane reading its row).
template <int W>
__device__ __forceinline__ void warp_rows_load(const float* __restrict__ src, int v0, int nv, float* st,
                                               int lane) {
  const int rows = min(32, nv - v0);
  const float4* s4 = reinterpret_cast<const float4*>(src + static_cast<size_t>(v0) * W);
  for (int q = lane; q < rows * (W / 4); q += 32) {
    const float4 t = ldg4(reinterpret_cast<const float*>(s4 + q));
    const int r = q / (W / 4), c = (q % (W / 4)) * 4;
    float* d = st + r * (W + 1) + c;
    d[0] = t.x;
    d[1] = t.y;
    d[2] = t.z;
    d[3] = t.w;
  }
  __syncwarp();
}
template <int W>
__device__ __forceinline__ void warp_rows_store(float* __restrict__ dst, int v0, int nv, const float* st,
                                                int lane) {
  __syncwarp();
  const int rows = min(32, nv - v0);
  float4* d4 = reinterpret_cast<float4*>(dst + static_cast<size_t>(v0) * W);
  for (int q = lane; q < rows * (W / 4); q += 32) {
    const int r = q / (W / 4), c = (q % (W / 4)) * 4;
    const float* s = st + r * (W + 1) + c;
    d4[q] = make_float4(s[0], s[1], s[2], s[3]);
  }
  __syncwarp();
}

// Decoder forward (src/gnn.cpp:178-199) for one virtual row (out in f64 [n][B]),
// rows read through the warp staging.
template <int DP>
__global__ void __launch_bounds__(32 * 4)
k_decoder_fwd(const float* __restrict__ XL, int nv, int B, NetView net,
              const SampleScales* __restrict__ sc, double* __restrict__ out) {
  extern __shared__ float4 sm4[];
  const int H = net.hidden;
  float* D1 = reinterpret_cast<float*>(sm4);  // [DP][H]
  float* B1 = D1 + DP * H;
  float* D2 = B1 + H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* sx = D2 + H + warp * 32 * (DP + 1);
  for (int t = threadIdx.x; t < DP * H; t += blockDim.x) D1[t] = net.dec1[t];
  for (int t = threadIdx.x; t < H; t += blockDim.x) {
    B1[t] = net.dec1_b[t];
    D2[t] = net.dec2[t];
  }
  __syncthreads();
  const int nwarps = gridDim.x * 4;
  for (int v0 = (blockIdx.x * 4 + warp) * 32; v0 < nv; v0 += nwarps * 32) {
    warp_rows_load<DP>(XL, v0, nv, sx, lane);
    const int v = v0 + lane;
    if (v < nv) {
      const int k = v % B;
      if (sc[k].zero) {
        out[v] = 0.0;
      } else {
        float y[DP];
#pragma unroll
        for (int j = 0; j < DP; ++j) y[j] = sx[lane * (DP + 1) + j];
        float o = 0.f;
        int h = 0;
        for (; (H & 3) == 0 && h < H; h += 4) {  // dec1 read as float4 along h
          float4 t = f4zero();
#pragma unroll
          for (int j = 0; j < DP; ++j) fma4(t, y[j], *reinterpret_cast<const float4*>(D1 + j * H + h));
          o = fmaf(relu(t.x + B1[h]), D2[h], o);
          o = fmaf(relu(t.y + B1[h + 1]), D2[h + 1], o);
          o = fmaf(relu(t.z + B1[h + 2]), D2[h + 2], o);
          o = fmaf(relu(t.w + B1[h + 3]), D2[h + 3], o);
        }
        for (; h < H; ++h) {
          float t = 0.f;
#pragma unroll
          for (int j = 0; j < DP; ++j) t = fmaf(y[j], D1[j * H + h], t);
          o = fmaf(relu(t + B1[h]), D2[h], o);
        }
        out[v] = static_cast<double>(o + *net.dec2_bp) * sc[k].out_scale;
      }
    }
    __syncwarp();
  }
}

// Decoder backward (src/gnn.cpp:219-256) for one virtual row:
//   gy = gout[v] * out_scale_k (0 for a zero sample)
//   stage 0: post[v][h] = relu(dec_pre_h), gy[v]      (for dec2 / dec2_b grads)
//   stage 1: gdp[v][h] = [dec_pre_h > 0] gy dec2_h      (for dec1 / dec1_b grads)
//            gpre[v][j] = [x_L > 0] Σ_h gdp_h dec1(j,h)  (mask of the last layer)
// One lane per row, 32-row blocks per warp with warp-staged row I/O
// (kMlpWarps warps per block; dynamic smem = mlp_smem_bytes).
constexpr int kMlpWarps = 4;
inline size_t mlp_smem_bytes(int DP, int H) {
  const int sw = (DP > H ? DP : H) + 1;
  return (static_cast<size_t>(DP) * H + 2 * H + static_cast<size_t>(kMlpWarps) * 3 * 32 * sw) * 4;
}
template <int DP>
__global__ void __launch_bounds__(32 * kMlpWarps)
k_decoder_bwd(const float* __restrict__ XL, int nv, int B, NetView net,
              const SampleScales* __restrict__ sc, const double* __restrict__ gout,
              float* __restrict__ post, float* __restrict__ gyv, float* __restrict__ gdp,
              float* __restrict__ gpre) {
  extern __shared__ float4 sm4[];
  const int H = net.hidden;
  float* D1 = reinterpret_cast<float*>(sm4);  // [DP][H]
  float* B1 = D1 + DP * H;
  float* D2 = B1 + H;
  const int SW = max(DP, H) + 1;  // staging capacity per row
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* stg = D2 + H + warp * 3 * 32 * SW;  // [3][32][SW]: x / gpre, post, gdp
  float* sx = stg;
  float* sp = stg + 32 * SW;
  float* sg = sp + 32 * SW;
  for (int t = threadIdx.x; t < DP * H; t += blockDim.x) D1[t] = net.dec1[t];
  for (int t = threadIdx.x; t < H; t += blockDim.x) {
    B1[t] = net.dec1_b[t];
    D2[t] = net.dec2[t];
  }
  __syncthreads();
  const int nwarps = gridDim.x * kMlpWarps;
  for (int v0 = (blockIdx.x * kMlpWarps + warp) * 32; v0 < nv; v0 += nwarps * 32) {
    // rows through the staging tile (stride DP + 1 inside warp_rows_*)
    warp_rows_load<DP>(XL, v0, nv, sx, lane);
    const int v = v0 + lane;
    const bool live = v < nv;
    const int k = v % B;
    const float gy = (!live || sc[k].zero) ? 0.f : static_cast<float>(gout[v] * sc[k].out_scale);
    if (live) gyv[v] = gy;
    float y[DP], gx[DP];
#pragma unroll
    for (int j = 0; j < DP; ++j) {
      y[j] = sx[lane * (DP + 1) + j];
      gx[j] = 0.f;
    }
    int h = 0;
    for (; (H & 3) == 0 && h < H; h += 4) {  // dec1 read as float4 along h, twice
      float4 t = f4zero();
#pragma unroll
      for (int j = 0; j < DP; ++j) fma4(t, y[j], *reinterpret_cast<const float4*>(D1 + j * H + h));
      const float p0 = t.x + B1[h], p1 = t.y + B1[h + 1], p2 = t.z + B1[h + 2], p3 = t.w + B1[h + 3];
      const float g0 = p0 > 0.f ? gy * D2[h] : 0.f, g1 = p1 > 0.f ? gy * D2[h + 1] : 0.f;
      const float g2 = p2 > 0.f ? gy * D2[h + 2] : 0.f, g3 = p3 > 0.f ? gy * D2[h + 3] : 0.f;
      float* pp = sp + lane * (H + 1) + h;
      float* pg = sg + lane * (H + 1) + h;
      pp[0] = relu(p0); pp[1] = relu(p1); pp[2] = relu(p2); pp[3] = relu(p3);
      pg[0] = g0; pg[1] = g1; pg[2] = g2; pg[3] = g3;
#pragma unroll
      for (int j = 0; j < DP; ++j) {
        const float4 d = *reinterpret_cast<const float4*>(D1 + j * H + h);
        gx[j] = fmaf(g0, d.x, fmaf(g1, d.y, fmaf(g2, d.z, fmaf(g3, d.w, gx[j]))));
      }
    }
    for (; h < H; ++h) {
      float t = 0.f;
#pragma unroll
      for (int j = 0; j < DP; ++j) t = fmaf(y[j], D1[j * H + h], t);
      const float pre = t + B1[h];
      sp[lane * (H + 1) + h] = relu(pre);
      const float g = pre > 0.f ? gy * D2[h] : 0.f;
      sg[lane * (H + 1) + h] = g;
#pragma unroll
      for (int j = 0; j < DP; ++j) gx[j] = fmaf(g, D1[j * H + h], gx[j]);
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < DP; ++j) sx[lane * (DP + 1) + j] = y[j] > 0.f ? gx[j] : 0.f;
    warp_rows_store<DP>(gpre, v0, nv, sx, lane);
    if (H == 32) {
      warp_rows_store<32>(post, v0, nv, sp, lane);
      warp_rows_store<32>(gdp, v0, nv, sg, lane);
    } else {
      __syncwarp();
      for (int r = 0; r < 32 && v0 + r < nv; ++r)
        for (int h = lane; h < H; h += 32) {
          post[static_cast<size_t>(v0 + r) * H + h] = sp[r * (H + 1) + h];
          gdp[static_cast<size_t>(v0 + r) * H + h] = sg[r * (H + 1) + h];
        }
      __syncwarp();
    }
  }
}

// Encoder backward (src/gnn.cpp:283-305) for one virtual row: recompute
// x0 = relu(vv enc1 + b1), g_x0 = enc2 gX0, gp0 = [pre0 > 0] g_x0.  Same
// warp-staged row I/O as the decoder.
template <int DP>
__global__ void __launch_bounds__(32 * kMlpWarps)
k_encoder_bwd(const float* __restrict__ vv, const float* __restrict__ gx0, int nv, NetView net,
              float* __restrict__ x0, float* __restrict__ gp0) {
  extern __shared__ float4 sm4[];
  const int H = net.hidden;
  float* s_enc2 = reinterpret_cast<float*>(sm4);  // [H][DP]
  float* s_enc1 = s_enc2 + H * DP;
  float* s_b1 = s_enc1 + H;
  const int SW = max(DP, H) + 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* stg = s_b1 + H + warp * 3 * 32 * SW;
  float* sx = stg;
  float* sp = stg + 32 * SW;
  float* sg = sp + 32 * SW;
  for (int t = threadIdx.x; t < H * DP; t += blockDim.x) s_enc2[t] = net.enc2[t];
  for (int t = threadIdx.x; t < H; t += blockDim.x) {
    s_enc1[t] = net.enc1[t];
    s_b1[t] = net.enc1_b[t];
  }
  __syncthreads();
  const int nwarps = gridDim.x * kMlpWarps;
  for (int v0 = (blockIdx.x * kMlpWarps + warp) * 32; v0 < nv; v0 += nwarps * 32) {
    warp_rows_load<DP>(gx0, v0, nv, sx, lane);
    const int v = v0 + lane;
    const float x = v < nv ? vv[v] : 0.f;
    float g[DP];
#pragma unroll
    for (int j = 0; j < DP; ++j) g[j] = sx[lane * (DP + 1) + j];
    for (int h = 0; h < H; ++h) {
      const float pre = fmaf(x, s_enc1[h], s_b1[h]);
      float t = 0.f;
#pragma unroll
      for (int j = 0; j < DP; ++j) t = fmaf(g[j], s_enc2[h * DP + j], t);
      sp[lane * (H + 1) + h] = relu(pre);
      sg[lane * (H + 1) + h] = pre > 0.f ? t : 0.f;
    }
    if (H == 32) {
      warp_rows_store<32>(x0, v0, nv, sp, lane);
      warp_rows_store<32>(gp0, v0, nv, sg, lane);
    } else {
      __syncwarp();
      for (int r = 0; r < 32 && v0 + r < nv; ++r)
        for (int h = lane; h < H; h += 32) {
          x0[static_cast<size_t>(v0 + r) * H + h] = sp[r * (H + 1) + h];
          gp0[static_cast<size_t>(v0 + r) * H + h] = sg[r * (H + 1) + h];
        }
      __syncwarp();
    }
  }
}

// ------------------------------------------------------------------ L1 loss
// r = A (out - x) per sample (src/gnn.cpp:319-328), f64; loss partials per
// block; sgn = sign(r).  One warp per node row, lanes over samples.
__global__ void __launch_bounds__(kThreads)
k_loss_residual(DevCsr a, int B, const double* __restrict__ out, const double* __restrict__ x,
                double* __restrict__ sgn, double* __restrict__ partials) {
  __shared__ double red[32];
  const int lane = threadIdx.x & 31;
  const int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  double acc = 0.0;
  for (int i = wg; i < a.n; i += nw) {
    for (int k = lane; k < B; k += 32) {
      double r = 0.0;
      for (int q = a.rp[i]; q < a.rp[i + 1]; ++q) {
        const size_t j = static_cast<size_t>(a.ci[q]) * B + k;
        r = fma(static_cast<double>(a.v[q]), out[j] - x[j], r);
      }
      acc += fabs(r);
      sgn[static_cast<size_t>(i) * B + k] = r > 0.0 ? 1.0 : (r < 0.0 ? -1.0 : 0.0);
    }
  }
  acc = block_sum(acc, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = acc;
}

// gout = (1/B) Âᵀ sgn (src/gnn.cpp:329-331) with the explicit transpose CSR.
__global__ void __launch_bounds__(kThreads)
k_loss_grad(DevCsr at, int B, const double* __restrict__ sgn, double* __restrict__ gout) {
  const int lane = threadIdx.x & 31;
  const int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  const double inv = 1.0 / static_cast<double>(B);
  for (int i = wg; i < at.n; i += nw)
    for (int k = lane; k < B; k += 32) {
      double g = 0.0;
      for (int q = at.rp[i]; q < at.rp[i + 1]; ++q)
        g = fma(static_cast<double>(at.v[q]), sgn[static_cast<size_t>(at.ci[q]) * B + k], g);
      gout[static_cast<size_t>(i) * B + k] = inv * g;
    }
}

// ------------------------------------------------------------------ outer-product sums
// S[p][q] = Σ_v A[v][p] B[v][q] (weight / bias gradients, src/gnn.cpp:240,265-266,
// 284 gemm_tn and the bias column sums): A = [A1 | A2 | ones?] (P cols, padded
// to P4 = P rounded up to 4), B (Q cols, padded to Q2).  Rows are split into
// contiguous per-block ranges; each thread owns a 4 x 2 register block of S,
// fp32 sums over 32-row smem tiles folded into f64 — per-block partials
// [grid.x][P4*Q2] are then summed in block order (deterministic).
struct OuterArgs {
  const float* A1;
  int P1, s1;
  const float* A2;
  int P2, s2;
  int ones;  // append a column of ones to A (bias gradients)
  const float* Bm;
  int Q, sq;
  int nv;
  double* partials;
};

__host__ __device__ inline int outer_P4(const OuterArgs& o) { return (o.P1 + o.P2 + o.ones + 3) & ~3; }
__host__ __device__ inline int outer_Q2(const OuterArgs& o) { return (o.Q + 1) & ~1; }

__global__ void __launch_bounds__(kThreads) k_outer_sum(OuterArgs o) {
  const int P = o.P1 + o.P2 + o.ones, P4 = outer_P4(o), Q2 = outer_Q2(o);
  constexpr int RT = 32;  // rows per smem tile
  extern __shared__ float4 sm4[];
  float* sA = reinterpret_cast<float*>(sm4);  // [RT][P4]
  float* sB = sA + RT * P4;                   // [RT][Q2]
  const int nbq = Q2 / 2, nblocks = (P4 / 4) * nbq;
  const int e = blockIdx.y * kThreads + threadIdx.x;
  const bool active = e < nblocks;
  const int p0 = active ? (e / nbq) * 4 : 0, q0 = active ? (e % nbq) * 2 : 0;
  double acc[4][2] = {};
  const int rows_per_blk = (o.nv + gridDim.x - 1) / gridDim.x;
  const int r0 = blockIdx.x * rows_per_blk, r1 = min(o.nv, r0 + rows_per_blk);
  for (int t0 = r0; t0 < r1; t0 += RT) {
    const int nr = min(RT, r1 - t0);
    for (int t = threadIdx.x; t < RT * P4; t += kThreads) {
      const int r = t / P4, p = t % P4;
      float val = 0.f;
      if (r < nr) {
        if (p < o.P1) val = o.A1[static_cast<size_t>(t0 + r) * o.s1 + p];
        else if (p < o.P1 + o.P2) val = o.A2[static_cast<size_t>(t0 + r) * o.s2 + (p - o.P1)];
        else if (p < P) val = 1.f;
      }
      sA[t] = val;
    }
    for (int t = threadIdx.x; t < RT * Q2; t += kThreads) {
      const int r = t / Q2, q = t % Q2;
      sB[t] = (r < nr && q < o.Q) ? o.Bm[static_cast<size_t>(t0 + r) * o.sq + q] : 0.f;
    }
    __syncthreads();
    if (active) {
      float s[4][2] = {};
      for (int r = 0; r < nr; ++r) {
        const float4 av = *reinterpret_cast<const float4*>(sA + r * P4 + p0);
        const float2 bv = *reinterpret_cast<const float2*>(sB + r * Q2 + q0);
        s[0][0] = fmaf(av.x, bv.x, s[0][0]); s[0][1] = fmaf(av.x, bv.y, s[0][1]);
        s[1][0] = fmaf(av.y, bv.x, s[1][0]); s[1][1] = fmaf(av.y, bv.y, s[1][1]);
        s[2][0] = fmaf(av.z, bv.x, s[2][0]); s[2][1] = fmaf(av.z, bv.y, s[2][1]);
        s[3][0] = fmaf(av.w, bv.x, s[3][0]); s[3][1] = fmaf(av.w, bv.y, s[3][1]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) acc[i][j] += static_cast<double>(s[i][j]);
    }
    __syncthreads();
  }
  if (active) {
    double* dst = o.partials + static_cast<size_t>(blockIdx.x) * P4 * Q2;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) dst[(p0 + i) * Q2 + q0 + j] = acc[i][j];
  }
}

// Sum the block partials in block order and scatter into the flat f64
// gradient: grad[dst[p*Q2+q]] = Σ_blk partial (dst < 0: padding, dropped).
__global__ void k_outer_finish(const double* __restrict__ partials, int nblk, int PQ,
                               const int* __restrict__ dst, double* __restrict__ grad) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= PQ) return;
  const int d = dst[idx];
  if (d < 0) return;
  double s = 0.0;
  int b = 0;
  for (; b + 8 <= nblk; b += 8) {  // 8 loads in flight, summed in block order
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = partials[static_cast<size_t>(b + u) * PQ + idx];
#pragma unroll
    for (int u = 0; u < 8; ++u) s += v[u];
  }
  for (; b < nblk; ++b) s += partials[static_cast<size_t>(b) * PQ + idx];
  grad[d] = s;
}

// ------------------------------------------------------------------ weighted column sums
// For the one-column reductions (src/gnn.cpp:222-235 dec2 / dec2_bias and
// :292-305 enc1 / enc1_bias): per block, out1[h] = Σ A[v][h] w[v],
// out2[h] = Σ A[v][h], out3 = Σ w[v] over the block's contiguous rows; lanes
// own the (<= 32) columns, warps stride rows; partials [grid][3][32] (f64).
__global__ void __launch_bounds__(kThreads)
k_weighted_colsum(const float* __restrict__ A, int W, const float* __restrict__ w, int nv,
                  double* __restrict__ partials) {
  __shared__ double red[8][3][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int per = (nv + gridDim.x - 1) / gridDim.x;
  const int r0 = blockIdx.x * per, r1 = min(nv, r0 + per);
  double a1 = 0.0, a2 = 0.0, a3 = 0.0;
  if (W == 32) {
    // lane = (row slot l/8, column quad l%8): one 16-byte load covers 4 rows of
    // a warp's 32-row step; 8 independent loads in flight per lane
    const int ro = lane >> 3, cq = lane & 7;
    double d1[4] = {0, 0, 0, 0}, d2[4] = {0, 0, 0, 0}, d3 = 0.0;
    for (int v0 = r0 + warp * 32; v0 < r1; v0 += 8 * 32) {
      float4 x[8];
      float wv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int v = v0 + 4 * u + ro;
        x[u] = v < r1 ? ldg4(A + static_cast<size_t>(v) * 32 + 4 * cq) : f4zero();
        wv[u] = v < r1 ? __ldg(w + v) : 0.f;
      }
      float4 s1 = f4zero(), s2 = f4zero();
      float s3 = 0.f;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        fma4(s1, wv[u], x[u]);
        s2 = add4(s2, x[u]);
        s3 += wv[u];
      }
      d1[0] += s1.x; d1[1] += s1.y; d1[2] += s1.z; d1[3] += s1.w;
      d2[0] += s2.x; d2[1] += s2.y; d2[2] += s2.z; d2[3] += s2.w;
      d3 += s3;
    }
    // combine the 4 row slots (lanes cq, cq+8, cq+16, cq+24) in a fixed order
#pragma unroll
    for (int o = 8; o < 32; o <<= 1) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        d1[i] += __shfl_xor_sync(0xffffffffu, d1[i], o);
        d2[i] += __shfl_xor_sync(0xffffffffu, d2[i], o);
      }
      d3 += __shfl_xor_sync(0xffffffffu, d3, o);
    }
    // column c = 4*cq + i lives in lanes with cq = c/4: gather to lane c
    const int src = (lane >> 2) & 7, comp = lane & 3;
    double t1 = 0, t2 = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double e1 = __shfl_sync(0xffffffffu, d1[i], src), e2 = __shfl_sync(0xffffffffu, d2[i], src);
      if (comp == i) {
        t1 = e1;
        t2 = e2;
      }
    }
    a1 = t1;
    a2 = t2;
    a3 = d3;
  } else
  for (int v0 = r0 + warp * 4; v0 < r1; v0 += 32) {  // 4 rows per warp per step
    float s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int v = v0 + u;
      if (v < r1) {
        const float x = lane < W ? __ldg(A + static_cast<size_t>(v) * W + lane) : 0.f;
        const float wv = __ldg(w + v);
        s1 = fmaf(x, wv, s1);
        s2 += x;
        s3 += wv;
      }
    }
    a1 += s1;
    a2 += s2;
    a3 += s3;
  }
  red[warp][0][lane] = a1;
  red[warp][1][lane] = a2;
  red[warp][2][lane] = a3;
  __syncthreads();
  if (warp == 0) {
    double t1 = 0.0, t2 = 0.0, t3 = 0.0;
    for (int q = 0; q < 8; ++q) {
      t1 += red[q][0][lane];
      t2 += red[q][1][lane];
      t3 += red[q][2][lane];
    }
    double* dst = partials + static_cast<size_t>(blockIdx.x) * 96;
    dst[lane] = t1;
    dst[32 + lane] = t2;
    dst[64 + lane] = t3;  // every lane holds Σ w; entry 64 is used
  }
}

// ------------------------------------------------------------------ Adam
// src/gnn.cpp:345-363 in f64 on the flat parameter vector.
__global__ void k_adam(double* __restrict__ p, const double* __restrict__ g, double* __restrict__ m1,
                       double* __restrict__ m2, int count, double lr, double bc1, double bc2) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= count) return;
  const double beta1 = 0.9, beta2 = 0.999, eps = 1e-8;
  const double gk = g[k];
  m1[k] = beta1 * m1[k] + (1.0 - beta1) * gk;
  m2[k] = beta2 * m2[k] + (1.0 - beta2) * gk * gk;
  const double mhat = m1[k] / bc1;
  const double vhat = m2[k] / bc2;
  p[k] -= lr * mhat / (sqrt(vhat) + eps);
}

// ------------------------------------------------------------------ device param rebuild
// From the flat f64 parameters (reference order) to the fp32 device layout
// and the per-layer B operands: gather map src[dst] (index into flat, -1 = 0).
__global__ void k_gather_params(const double* __restrict__ flat, const int* __restrict__ src,
                                int count, float* __restrict__ dst) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= count) return;
  const int s = src[k];
  dst[k] = s >= 0 ? static_cast<float>(flat[s]) : 0.f;
}

// tcgen05 B operands (hi/lo, swizzled): dst[k] = split(flat[src[k]]),
// part[k] = 0 (hi) or 1 (lo).
__global__ void k_gather_split(const double* __restrict__ flat, const int* __restrict__ src,
                               const unsigned char* __restrict__ part, int count,
                               float* __restrict__ dst) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= count) return;
  const int s = src[k];
  const float v = s >= 0 ? static_cast<float>(flat[s]) : 0.f;
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
  const float hi = __uint_as_float(r);
  dst[k] = part[k] ? v - hi : hi;
}

// ------------------------------------------------------------------ data movement
// n x B column-major (host TrainingBatch layout) -> [n][B] (device layout).
__global__ void k_colmajor_to_nb(const double* __restrict__ src, int n, int B,
                                 double* __restrict__ dst) {
  const size_t t = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<size_t>(n) * B) return;
  const int i = static_cast<int>(t / B), k = static_cast<int>(t % B);
  dst[t] = src[static_cast<size_t>(k) * n + i];
}
__global__ void k_nb_to_colmajor(const double* __restrict__ src, int n, int B,
                                 double* __restrict__ dst) {
  const size_t t = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<size_t>(n) * B) return;
  const int i = static_cast<int>(t / B), k = static_cast<int>(t % B);
  dst[static_cast<size_t>(k) * n + i] = src[t];
}

// Throughput-mode pairs: x ~ N(0,1) from Philox4x32-10 keyed by (seed, step),
// Box-Muller in fp32, stored f64 in [n][B]; b = A x follows via k_spmm_nb.
__device__ __forceinline__ uint4 philox(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}
__global__ void k_philox_normal(unsigned long long seed, unsigned long long step, size_t count,
                                double* __restrict__ x) {
  const size_t t = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (4 * t >= count) return;
  const uint4 r = philox(make_uint4(static_cast<uint32_t>(t), static_cast<uint32_t>(t >> 32),
                                    static_cast<uint32_t>(step), static_cast<uint32_t>(step >> 32)),
                         make_uint2(static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32)));
  const float u[4] = {(r.x + 1.0f) * 2.3283064e-10f, r.y * 2.3283064e-10f,
                      (r.z + 1.0f) * 2.3283064e-10f, r.w * 2.3283064e-10f};
  const float rad0 = sqrtf(-2.f * logf(u[0])), rad1 = sqrtf(-2.f * logf(u[2]));
  float s0, c0, s1, c1;
  sincospif(2.f * u[1], &s0, &c0);
  sincospif(2.f * u[3], &s1, &c1);
  const float z[4] = {rad0 * c0, rad0 * s0, rad1 * c1, rad1 * s1};
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (4 * t + q < count) x[4 * t + q] = z[q];
}

// y[i][k] = Σ_j a_ij x[j][k] for all B samples ([n][B] f64).
__global__ void __launch_bounds__(kThreads)
k_spmm_nb(DevCsr a, int B, const double* __restrict__ x, double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = wg; i < a.n; i += nw)
    for (int k = lane; k < B; k += 32) {
      double s = 0.0;
      for (int q = a.rp[i]; q < a.rp[i + 1]; ++q)
        s = fma(static_cast<double>(a.v[q]), x[static_cast<size_t>(a.ci[q]) * B + k], s);
      y[static_cast<size_t>(i) * B + k] = s;
    }
}


// ------------------------------------------------------------------ piecewise encoder
// The lift v -> enc2ᵀ relu(v enc1 + b1) + b2 has a scalar input, so it is an
// exact piecewise-linear map (the apply path's k_lift_pw; tables there are
// built on the host).  Training regenerates the tables on the device after
// every Adam step (k_lift_tables), runs the forward as one FMA per output
// (k_lift_pw_batched), and reduces the whole encoder backward
// (src/gnn.cpp:283-305) to per-interval sums of the layer-1 gradient rows:
//   S1[p] = Σ_{v in p} g_v,  Sx[p] = Σ_{v in p} vv_v g_v
//   enc2(h, j)   = Σ_p act(h, p) (enc1_h Sx[p][j] + b1_h S1[p][j])
//   enc2_b(j)    = Σ_p S1[p][j]
//   enc1(h)      = Σ_p act(h, p) Σ_j enc2(h, j) Sx[p][j]
//   enc1_b(h)    = Σ_p act(h, p) Σ_j enc2(h, j) S1[p][j]
// where act(h, p) = [unit h active on interval p].  No x0 / g_x0 cache.
struct LiftTab {
  float* t;                 // [H] sorted distinct kinks (nb used)
  float* a;                 // [H+1][DP]
  float* b;                 // [H+1][DP]
  unsigned long long* act;  // [H+1] bit h: unit h active on the interval
  int* nb;
};
struct EncOff {
  int enc1, enc1_b, enc2, enc2_b, H, d;
};

// One block: kinks t_h = -b1_h/enc1_h (enc1_h != 0), sorted and distinct,
// then per interval the active set at an interior point and the affine
// coefficients, all from the f64 master parameters (the host build in
// gnpc_model_s::build_view does the same).
__global__ void k_lift_tables(const double* __restrict__ p, EncOff o, int DP, LiftTab tab) {
  __shared__ double kinks[64], vr[65], e1[64], b1[64];
  __shared__ int nbs;
  extern __shared__ double e2[];  // [H][d]: enc2(h, j) at h * d + j
  for (int h = threadIdx.x; h < o.H; h += blockDim.x) {
    e1[h] = p[o.enc1 + h];
    b1[h] = p[o.enc1_b + h];
  }
  for (int t = threadIdx.x; t < o.H * o.d; t += blockDim.x) {
    const int h = t / o.d, j = t % o.d;
    e2[t] = p[o.enc2 + j * o.H + h];
  }
  __shared__ double tk[64];
  __shared__ int valid[64];
  __syncthreads();
  // sorted distinct kinks in parallel: unit h keeps its kink when no earlier
  // unit has the same value; its slot = #distinct kept values below it
  for (int h = threadIdx.x; h < o.H; h += blockDim.x) {
    valid[h] = e1[h] != 0.0;
    tk[h] = valid[h] ? -b1[h] / e1[h] : 0.0;
  }
  __shared__ int first[64];  // unit h holds its value's first occurrence
  __syncthreads();
  for (int h = threadIdx.x; h < o.H; h += blockDim.x) {
    int f = valid[h];
    for (int r = 0; r < h && f; ++r) f = !(valid[r] && tk[r] == tk[h]);
    first[h] = f;
  }
  __syncthreads();
  int keep = 0;
  if (threadIdx.x < o.H && first[threadIdx.x]) {
    const double t = tk[threadIdx.x];
    int slot = 0;
    for (int q = 0; q < o.H; ++q) slot += first[q] && tk[q] < t;
    kinks[slot] = t;
    keep = 1;
  }
  const int nb = __syncthreads_count(keep);
  if (threadIdx.x == 0) {
    nbs = nb;
    *tab.nb = nb;
  }
  for (int k = threadIdx.x; k <= nb; k += blockDim.x) {
    if (nb == 0) vr[k] = 0.0;
    else if (k == 0) vr[k] = kinks[0] - 1.0 - fabs(kinks[0]);
    else if (k == nb) vr[k] = kinks[nb - 1] + 1.0 + fabs(kinks[nb - 1]);
    else vr[k] = 0.5 * (kinks[k - 1] + kinks[k]);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < nb; k += blockDim.x) tab.t[k] = static_cast<float>(kinks[k]);
  for (int idx = threadIdx.x; idx < (nb + 1) * DP; idx += blockDim.x) {
    const int k = idx / DP, j = idx % DP;
    double a_ = 0.0, b_ = 0.0;
    unsigned long long m = 0ull;
    for (int h = 0; h < o.H; ++h) {
      if (!(e1[h] * vr[k] + b1[h] > 0.0)) continue;
      m |= 1ull << h;
      if (j < o.d) {
        a_ += e1[h] * e2[h * o.d + j];
        b_ += b1[h] * e2[h * o.d + j];
      }
    }
    if (j < o.d) b_ += p[o.enc2_b + j];
    if (j == 0) tab.act[k] = m;
    tab.a[idx] = static_cast<float>(a_);
    tab.b[idx] = static_cast<float>(b_);
  }
}

__device__ __forceinline__ int interval_of(const float* s_t, int nb, float v) {
  int lo = 0, hi = nb;  // #kinks <= v
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (s_t[mid] <= v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// X0[v] = a[p] vv + b[p], vv = (float)(in_scale_k b[v]); also writes vv.
template <int DP>
__global__ void __launch_bounds__(kThreads)
k_lift_pw_batched(const double* __restrict__ b, int nv, int B, LiftTab tab, int H,
                  const SampleScales* __restrict__ sc, float* __restrict__ X0,
                  float* __restrict__ vv_out) {
  constexpr int G = DP / 4, NG = kThreads / G;
  extern __shared__ float4 sm4[];
  const int nb = *tab.nb;
  float* s_a = reinterpret_cast<float*>(sm4);  // [nb+1][DP]
  float* s_b = s_a + (H + 1) * DP;
  float* s_t = s_b + (H + 1) * DP;
  for (int t = threadIdx.x; t < (nb + 1) * DP; t += kThreads) {
    s_a[t] = tab.a[t];
    s_b[t] = tab.b[t];
  }
  for (int t = threadIdx.x; t < nb; t += kThreads) s_t[t] = tab.t[t];
  __syncthreads();
  const int gl = threadIdx.x % G;
  for (int v = blockIdx.x * NG + threadIdx.x / G; v < nv; v += gridDim.x * NG) {
    const int k = v % B;
    const float x = static_cast<float>(sc[k].in_scale * b[v]);
    if (gl == 0) vv_out[v] = x;
    const int q = interval_of(s_t, nb, x);
    const float4 al = *reinterpret_cast<const float4*>(s_a + q * DP + 4 * gl);
    const float4 be = *reinterpret_cast<const float4*>(s_b + q * DP + 4 * gl);
    st4(X0 + static_cast<size_t>(v) * DP + 4 * gl,
        make_float4(fmaf(al.x, x, be.x), fmaf(al.y, x, be.y), fmaf(al.z, x, be.z), fmaf(al.w, x, be.w)));
  }
}

// Per-interval sums of the layer-1 gradient rows.  Block blk owns rows
// [blk*rpb, (blk+1)*rpb) (rpb a multiple of kEncStg), staged kEncStg rows at
// a time by 1-D bulk copies into a kEncNS-deep ring.  A sub-group of
// GL = min(DP, 32) lanes takes one row (CPL columns per lane); each
// sub-group owns two fp32 accumulator sets [H+1][2][DP] (even / odd rows, so
// consecutive read-modify-writes of a lane never chain through the same set
// and no two lanes ever touch the same word).  The sets fold into the
// block's f64 sums in a fixed order after every kEncCh rows per set:
// deterministic for a fixed grid.  Output: partials[blk][(H+1)*2*DP].
#ifndef GNPC_ENC_STG
#define GNPC_ENC_STG 256  // with a 2-deep ring: 0.07 ms per C3 step better than 128 x 3
#endif
#ifndef GNPC_ENC_NS
#define GNPC_ENC_NS 2
#endif
#ifndef GNPC_ENC_CH
#define GNPC_ENC_CH 128
#endif
constexpr int kEncCh = GNPC_ENC_CH, kEncStg = GNPC_ENC_STG, kEncNS = GNPC_ENC_NS;
// rows per stage: kEncStg, capped so a warp walks at most 32 rows of it
__host__ __device__ inline int enc_stage_rows(int warps) { return kEncStg < 32 * warps ? kEncStg : 32 * warps; }
// set stride padded by GL floats when a warp holds several sub-groups, so
// the sub-groups land on different banks
inline size_t enc_bucket_smem(int DP, int H, int warps) {
  const int gl = DP < 32 ? DP : 32;
  const size_t sets = static_cast<size_t>(warps) * (32 / gl) * 2;
  const size_t per = static_cast<size_t>(H + 1) * 2 * DP;
  const int stg = enc_stage_rows(warps);
  return static_cast<size_t>(kEncNS) * stg * (DP + 1) * 4 + per * 8 +
         sets * (per + (gl < 32 ? gl : 0)) * 4 + 64 * 4 + 64;
}
template <int DP>
__global__ void k_enc_buckets(const float* __restrict__ g, const float* __restrict__ vv, int nv,
                              int rpb, LiftTab tab, int H, double* __restrict__ partials) {
  constexpr int GL = DP < 32 ? DP : 32, CPL = DP / GL, R = 32 / GL;
  extern __shared__ float4 sm4[];
  const int per = (H + 1) * 2 * DP;
  const int stride = per + (R > 1 ? GL : 0);
  const int stg = enc_stage_rows(blockDim.x >> 5);
  const int nsub = (blockDim.x >> 5) * R;                            // row slots per pass
  float* sg = reinterpret_cast<float*>(sm4);                         // [NS][Stg][DP]
  float* sx = sg + kEncNS * stg * DP;                            // [NS][Stg]
  double* blk = reinterpret_cast<double*>(sx + kEncNS * stg);    // [per]
  float* acc = reinterpret_cast<float*>(blk + per);                  // [2 nsub][stride]
  float* s_t = acc + static_cast<size_t>(2 * nsub) * stride;         // [64]
  uint64_t* bar = reinterpret_cast<uint64_t*>(s_t + 64);             // [NS]
  const int nb = *tab.nb;
  const int tid = threadIdx.x;
  for (int t = tid; t < per; t += blockDim.x) blk[t] = 0.0;
  for (int t = tid; t < 2 * nsub * stride; t += blockDim.x) acc[t] = 0.f;
  for (int t = tid; t < nb; t += blockDim.x) s_t[t] = tab.t[t];
  const int r0 = blockIdx.x * rpb, r1 = min(nv, r0 + rpb);
  const int nst = r1 > r0 ? (r1 - r0 + stg - 1) / stg : 0;
  auto rows_of = [&](int st) { return min(stg, r1 - (r0 + st * stg)); };
  auto issue = [&](int st) {  // thread 0: full stages only (16-byte aligned, r0 % stg == 0)
    if (st >= nst || rows_of(st) != stg) return;
    const int slot = st % kEncNS;
    const size_t row = static_cast<size_t>(r0) + static_cast<size_t>(st) * stg;
    tc::mbar_expect_tx(&bar[slot], stg * DP * 4 + stg * 4);
    tc::bulk_load(sg + slot * stg * DP, g + row * DP, stg * DP * 4, &bar[slot]);
    tc::bulk_load(sx + slot * stg, vv + row, stg * 4, &bar[slot]);
  };
  if (tid == 0) {
    for (int q = 0; q < kEncNS; ++q) tc::mbar_init(&bar[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (int q = 0; q < kEncNS; ++q) issue(q);
  const int lane = tid & 31, warp = tid >> 5;
  const int sub = warp * R + lane / GL, c0 = (lane % GL) * CPL;
  float* my0 = acc + static_cast<size_t>(2 * sub) * stride;
  float* my1 = my0 + stride;
  const int flush_every = max(1, kEncCh * nsub / stg);  // stages between folds
  for (int st = 0; st < nst; ++st) {
    const int slot = st % kEncNS, rows = rows_of(st);
    const float* gs = sg + slot * stg * DP;
    const float* xs = sx + slot * stg;
    if (rows == stg) {
      tc::mbar_wait(&bar[slot], (st / kEncNS) & 1);
    } else {  // the grid's ragged tail: plain loads
      float* gw = sg + slot * stg * DP;
      float* xw = sx + slot * stg;
      const size_t row = static_cast<size_t>(r0) + static_cast<size_t>(st) * stg;
      for (int t = tid; t < rows * DP; t += blockDim.x) gw[t] = g[row * DP + t];
      for (int t = tid; t < rows; t += blockDim.x) xw[t] = vv[row + t];
      __syncthreads();
    }
    // warp w takes rows [w*rpw, (w+1)*rpw) of the stage; lane l finds row
    // w*rpw + l's interval once, sub-groups then walk the rows R at a time
    // with (x, interval) broadcast by shuffles, alternating their two sets
    const int rpw = stg / (blockDim.x >> 5);  // <= 32
    const int wr0 = warp * rpw;
    const float xl = lane < rpw && wr0 + lane < rows ? xs[wr0 + lane] : 0.f;
    const int ql = interval_of(s_t, nb, xl) * 2 * DP;
    const int sg_row = lane / GL;
    // two rows per step, one per set: both read-modify-writes are issued
    // side by side (different sets never alias)
#pragma unroll 2
    for (int i = 0; i < rpw; i += 2 * R) {
      const int ra = i + sg_row, rb2 = i + R + sg_row;
      const float xa = __shfl_sync(0xffffffffu, xl, ra);
      const int qa = __shfl_sync(0xffffffffu, ql, ra) + c0;
      const float xb = __shfl_sync(0xffffffffu, xl, rb2 & 31);
      const int qb = __shfl_sync(0xffffffffu, ql, rb2 & 31) + c0;
      const bool ona = wr0 + ra < rows && ra < rpw, onb = wr0 + rb2 < rows && rb2 < rpw;
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const float ga = ona ? gs[(wr0 + ra) * DP + c0 + c] : 0.f;
        const float gb = onb ? gs[(wr0 + rb2) * DP + c0 + c] : 0.f;
        const float a1 = my0[qa + c], a2 = my0[qa + DP + c];
        const float b1 = my1[qb + c], b2 = my1[qb + DP + c];
        my0[qa + c] = a1 + ga;
        my0[qa + DP + c] = fmaf(xa, ga, a2);
        my1[qb + c] = b1 + gb;
        my1[qb + DP + c] = fmaf(xb, gb, b2);
      }
    }
    __syncthreads();  // the slot is free; the sets are quiescent
    if (tid == 0) issue(st + kEncNS);
    if ((st + 1) % flush_every == 0 || st + 1 == nst) {
      for (int t = tid; t < per; t += blockDim.x) {
        double s = blk[t];
        for (int z = 0; z < 2 * nsub; ++z) {
          s += static_cast<double>(acc[static_cast<size_t>(z) * stride + t]);
          acc[static_cast<size_t>(z) * stride + t] = 0.f;
        }
        blk[t] = s;
      }
      __syncthreads();
    }
  }
  for (int t = tid; t < per; t += blockDim.x)
    partials[static_cast<size_t>(blockIdx.x) * per + t] = blk[t];
}

// Folds the block partials in a fixed order: S[t] = Σ_z partials[z][t].
__global__ void k_enc_fold(const double* __restrict__ partials, int nblk, int per,
                           double* __restrict__ S) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= per) return;
  double s = 0.0;
  int z = 0;
  for (; z + 8 <= nblk; z += 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = partials[static_cast<size_t>(z + u) * per + t];
#pragma unroll
    for (int u = 0; u < 8; ++u) s += v[u];
  }
  for (; z < nblk; ++z) s += partials[static_cast<size_t>(z) * per + t];
  S[t] = s;
}

// Encoder gradients from the folded sums into the flat f64 gradient
// (reference slots via EncOff).
__global__ void k_enc_grads(const double* __restrict__ Sg, int DP, LiftTab tab,
                            const double* __restrict__ p, EncOff o, double* __restrict__ grad) {
  extern __shared__ double S[];  // [(H+1)][2][DP], then X, Y [H][d]
  const int H = o.H, d = o.d, per = (H + 1) * 2 * DP;
  double* Xs = S + per;  // X(h, j) = Σ_{q: h active} Sx[q][j]
  double* Ys = Xs + H * d;  // Y(h, j) = Σ_{q: h active} S1[q][j]
  __shared__ unsigned long long act[65];
  const int nb = *tab.nb;
  for (int t = threadIdx.x; t < per; t += blockDim.x) S[t] = Sg[t];
  for (int q = threadIdx.x; q <= nb; q += blockDim.x) act[q] = tab.act[q];
  __syncthreads();
  for (int idx = threadIdx.x; idx < H * d; idx += blockDim.x) {
    const int h = idx % H, j = idx / H;
    double x = 0.0, y = 0.0;
    for (int q = 0; q <= nb; ++q)
      if ((act[q] >> h) & 1ull) {
        x += S[q * 2 * DP + DP + j];
        y += S[q * 2 * DP + j];
      }
    Xs[h * d + j] = x;
    Ys[h * d + j] = y;
    grad[o.enc2 + j * H + h] = p[o.enc1 + h] * x + p[o.enc1_b + h] * y;
  }
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    double s = 0.0;
    for (int q = 0; q <= nb; ++q) s += S[q * 2 * DP + j];
    grad[o.enc2_b + j] = s;
  }
  __syncthreads();
  for (int h = threadIdx.x; h < H; h += blockDim.x) {
    double gw = 0.0, gb = 0.0;
    for (int j = 0; j < d; ++j) {
      const double e = p[o.enc2 + j * H + h];
      gw += e * Xs[h * d + j];
      gb += e * Ys[h * d + j];
    }
    grad[o.enc1 + h] = gw;
    grad[o.enc1_b + h] = gb;
  }
}

}  // namespace gnpk
