// Training decoder on the tensor cores (d = hidden = 32), src/gnn.cpp:178-256.
//
// Per 128-row tile of X_L (virtual rows v = node*B + k):
//   MMA1   P = X_L · dec1                    3xTF32: D[:, 0:32] = Y_hi·D1_lo,
//                                            D[:, 32:64] = Y_hi·D1_hi + Y_lo·D1_hi
//   FWD    out[v] = (Σ_h relu(P_h + b1_h) dec2_h + b2) · τ_k/√n        (f64)
//   BWD    gy = gout[v] τ_k/√n, g_z = [P + b1 > 0] gy dec2      (written: the
//          dec1 / dec1_b weight gradient reads it), per-thread sums of
//          relu(P + b1) gy (dec2) and gy (dec2_b);
//   MMA2   G = g_z · dec1ᵀ                   3xTF32 with g_z hi/lo in TMEM
//          G_L[v] = [X_L > 0] G                (the last layer's relu mask)
//
// One thread per tile row (4 warps, lane quarter = warp), thread 0 issues the
// TMA loads and the MMAs; tiles run synchronously inside a CTA and several
// CTAs per SM overlap.  X_L tiles arrive by TMA (SW128, the MMA's A_hi
// operand as is: kind::tf32 truncates); Y_lo and g_z hi/lo go to TMEM (TS-form
// MMAs), so no operand crosses shared memory twice.
//
//   MMA3   (backward) dec1 / dec1_b gradient [X_L | 1]ᵀ · g_z accumulated
//          in TMEM (bf16 hi/lo, MN-major: the wgb operand layout of
//          wgrad_tc.cuh), folded into per-CTA f64 partials every wgb::kFlushBf
//          tiles — g_z never goes to HBM
//
// TMEM columns: [0, 64) accumulator (MMA1, then MMA2), [64, 96) Y_lo then
// g_z lo, [96, 128) g_z hi, backward: [128, 160) the M = 64 weight-gradient
// accumulator.
#pragma once

#include "layer_sell.cuh"
#include "train.cuh"
#include "wgrad_tc.cuh"

namespace gnpk {

template <bool FWD>
struct DecTc {
  static constexpr bool WG = !FWD;                       // fused dec1 / dec1_b gradient
  static constexpr int TM = 128, NS = FWD ? 3 : 2, NT = 128;
  static constexpr uint32_t OPB = TM * 32 * 4;           // one [128][32] fp32 tile
  static constexpr uint32_t O_RING = 0;
  static constexpr uint32_t O_B1 = NS * OPB;              // [D1_lo; D1_hi]: rows h, K = j
  static constexpr uint32_t O_B2 = O_B1 + 64 * 128;       // [DT_lo; DT_hi]: rows j, K = h
  static constexpr uint32_t O_WG = O_B2 + 64 * 128;       // Ahi | Alo | Bhi | Blo (wgb layouts)
  static constexpr uint32_t O_SM = O_WG + (WG ? wgb::OPS : 0);  // b1[32], dec2[32]
  static constexpr uint32_t O_BAR = O_SM + 64 * 4;        // full[NS], mma
  static size_t smem_bytes() { return O_BAR + 8 * (NS + 1) + 16 + 1024; }
  static constexpr int TCOLS = WG ? 256 : 128;
};

// partials: [gridDim.x][33] per-CTA sums (dec2[h], then dec2_b) in f64;
// wpart: [gridDim.x][64][32] per-CTA dec1 (rows j < 32) / dec1_b (row 32)
// gradient partials in the wgrad partial layout (backward).
template <bool FWD>
__global__ void __launch_bounds__(DecTc<FWD>::NT, FWD ? 3 : 2)
k_decoder_tc(const __grid_constant__ CUtensorMap mapy, const float* __restrict__ Y, int nv, int B,
             NetView net, const SampleScales* __restrict__ sc, const double* __restrict__ gout,
             double* __restrict__ out, float* __restrict__ gpre, double* __restrict__ partials,
             double* __restrict__ wpart) {
  using C = DecTc<FWD>;
  extern __shared__ float4 smem_raw[];
  const uint32_t pad = (1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* base = reinterpret_cast<uint8_t*>(smem_raw) + pad;
  uint8_t* ring = base + C::O_RING;
  uint8_t* B1 = base + C::O_B1;
  uint8_t* B2 = base + C::O_B2;
  float* b1 = reinterpret_cast<float*>(base + C::O_SM);
  float* d2 = b1 + 32;
  uint64_t* full = reinterpret_cast<uint64_t*>(base + C::O_BAR);
  uint64_t* mbar = full + C::NS;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(mbar + 1);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // B operands, split hi = trunc(x), lo = x - hi (kind::tf32 truncates)
  for (int t = tid; t < 32 * 32; t += C::NT) {
    const int a = t / 32, c = t % 32;
    const float v1 = net.dec1[c * 32 + a];  // B1(h = a, j = c) = dec1(j, h)
    const float h1 = __int_as_float(__float_as_int(v1) & 0xffffe000);
    *reinterpret_cast<float*>(B1 + tc::swz_off<32>(a, c)) = v1 - h1;
    *reinterpret_cast<float*>(B1 + tc::swz_off<32>(32 + a, c)) = h1;
    const float v2 = net.dec1[a * 32 + c];  // B2(j = a, h = c) = dec1(j, h)
    const float h2 = __int_as_float(__float_as_int(v2) & 0xffffe000);
    *reinterpret_cast<float*>(B2 + tc::swz_off<32>(a, c)) = v2 - h2;
    *reinterpret_cast<float*>(B2 + tc::swz_off<32>(32 + a, c)) = h2;
  }
  if (tid < 32) {
    b1[tid] = net.dec1_b[tid];
    d2[tid] = net.dec2[tid];
  }
  uint8_t* WA = base + C::O_WG;  // Ahi | Alo | Bhi | Blo
  if constexpr (C::WG) {
    // A = [X_L | 1 | 0]: features 32..63 are constant (1.0 at 32: dec1_b)
    for (int j = tid; j < C::TM * 32; j += C::NT) {
      const int r = j / 32, m = 32 + j % 32;
      *reinterpret_cast<__nv_bfloat16*>(WA + wgb::offA(r, m)) = __float2bfloat16_rn(m == 32 ? 1.f : 0.f);
      *reinterpret_cast<__nv_bfloat16*>(WA + wgb::OPA + wgb::offA(r, m)) = __float2bfloat16_rn(0.f);
    }
    // this CTA's partials: thread (warp q, lane < 16) owns row 16 q + lane
    if ((tid & 31) < 16)
      for (int c = 0; c < 32; ++c)
        wpart[static_cast<size_t>(blockIdx.x) * 2048 + (16 * (tid >> 5) + (tid & 31)) * 32 + c] = 0.0;
  }
  if (tid == 0) {
    for (int s = 0; s < C::NS; ++s) tc::mbar_init(&full[s], 1);
    tc::mbar_init(mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tc::tmem_alloc(tslot, C::TCOLS);
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;
  const float b2 = *net.dec2_bp;

  const int ntiles = (nv + C::TM - 1) / C::TM;
  const int my = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  auto issue = [&](int it) {
    if (it >= my) return;
    const int s = it % C::NS;
    tc::mbar_expect_tx(&full[s], C::OPB);
    tc::tma_load_2d(ring + s * C::OPB, &mapy, 0, (blockIdx.x + it * gridDim.x) * C::TM, &full[s]);
  };
  if (tid == 0) {
    tc::tma_prefetch_desc(&mapy);
    for (int it = 0; it < C::NS; ++it) issue(it);
  }
  const uint32_t trow = static_cast<uint32_t>(32 * warp) << 16;  // this warp's lane quarter
  const uint32_t tD = tmem, tR1 = tmem + 64, tR2 = tmem + 96, tW = tmem + 128;
  int since_flush = 0;
  const uint32_t i64 = tc::idesc_tf32(128, 64), i32 = tc::idesc_tf32(128, 32);
  const uint32_t sB1 = tc::smem_u32(B1), sB2 = tc::smem_u32(B2);
  float acc[33];
#pragma unroll
  for (int h = 0; h < 33; ++h) acc[h] = 0.f;
  int mph = 0;
  int cur_it = 0;
  // the staged [128][32] tile of the current slot -> rows [t*128, t*128+128)
  // of dst, 16-byte chunk q = tid + 128 i (row q/8, chunk q%8): coalesced
  auto store_tile = [&](float* dst) {
    const uint8_t* st = ring + (cur_it % C::NS) * C::OPB;
    const size_t row0 = static_cast<size_t>(blockIdx.x + cur_it * gridDim.x) * C::TM;
    float4* d4 = reinterpret_cast<float4*>(dst + row0 * 32);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int q = tid + C::NT * i, r = q >> 3;
      if (row0 + r < static_cast<size_t>(nv))
        d4[q] = *reinterpret_cast<const float4*>(st + tc::swz_off<32>(r, 4 * (q & 7)));
    }
  };
  double gnext = 0.0;
  if (!FWD && my > 0) {
    const int v0 = blockIdx.x * C::TM + tid;
    gnext = v0 < nv ? gout[v0] : 0.0;
  }
  for (int it = 0; it < my; ++it) {
    const int s = it % C::NS;
    cur_it = it;
    const int v = (blockIdx.x + it * gridDim.x) * C::TM + tid;
    const bool live = v < nv;
    // per-row scalars first: their latency overlaps the TMA wait and MMA1
    const int k = v % B;
    const SampleScales scv = sc[k];
    // gout of this row: loaded one tile ahead (its latency hides behind a tile)
    const double gov = gnext;
    {
      const int vn = v + static_cast<int>(gridDim.x) * C::TM;
      gnext = (!FWD && it + 1 < my && vn < nv) ? gout[vn] : 0.0;
    }
    tc::mbar_wait(&full[s], (it / C::NS) & 1);
    // this row of X_L (swizzled), Y_lo into TMEM
    uint8_t* yt = ring + s * C::OPB;
    float y[32];
    uint32_t ymask = 0u;  // [X_L > 0] bits (the last layer's relu mask)
#pragma unroll
    for (int c = 0; c < 32; c += 4) {
      const float4 q = *reinterpret_cast<const float4*>(yt + tc::swz_off<32>(tid, c));
      y[c] = q.x;
      y[c + 1] = q.y;
      y[c + 2] = q.z;
      y[c + 3] = q.w;
    }
#pragma unroll
    for (int c = 0; c < 32; ++c) ymask |= (y[c] > 0.f ? 1u : 0u) << c;
    if constexpr (C::WG) {  // this row of [X_L | 1] as bf16 hi/lo (MMA3 of the previous tile completed)
#pragma unroll
      for (int c8 = 0; c8 < 4; ++c8) {
        uint4 hi, lo;
        wgb::split8(make_float4(y[8 * c8], y[8 * c8 + 1], y[8 * c8 + 2], y[8 * c8 + 3]),
                    make_float4(y[8 * c8 + 4], y[8 * c8 + 5], y[8 * c8 + 6], y[8 * c8 + 7]), hi, lo);
        *reinterpret_cast<uint4*>(WA + wgb::offA(tid, 8 * c8)) = hi;
        *reinterpret_cast<uint4*>(WA + wgb::OPA + wgb::offA(tid, 8 * c8)) = lo;
      }
    }
#pragma unroll
    for (int c = 0; c < 32; c += 8) {
      float lo[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) lo[e] = y[c + e] - __int_as_float(__float_as_int(y[c + e]) & 0xffffe000);
      tc::tmem_st8(tR1 + trow + c, lo);
    }
    tc::tmem_wait_st();
    tc::fence_before();
    __syncthreads();
    if (tid == 0) {
      tc::fence_after();
      const uint32_t sY = tc::smem_u32(yt);
#pragma unroll
      for (int k8 = 0; k8 < 4; ++k8) {
        tc::mma_tf32(tD, tc::make_desc_swz<32>(sY + k8 * 32), tc::make_desc_swz<32>(sB1 + k8 * 32), i64,
                     k8 > 0);
        tc::mma_tf32_ts(tD + 32, tR1 + 8 * k8, tc::make_desc_swz<32>(sB1 + 4096 + k8 * 32), i32, 1);
      }
      tc::mma_commit(mbar);
    }
    tc::mbar_wait(mbar, mph & 1);
    ++mph;
    tc::fence_after();
    float p[32];
    {
      float u[16], w[16];
#pragma unroll
      for (int h0 = 0; h0 < 32; h0 += 16) {
        tc::tmem_ld16(tD + trow + h0, u);
        tc::tmem_ld16(tD + trow + 32 + h0, w);
#pragma unroll
        for (int e = 0; e < 16; ++e) p[h0 + e] = u[e] + w[e] + b1[h0 + e];
      }
    }
    if constexpr (FWD) {
      tc::fence_before();
      if (live) {
        float o = 0.f;
#pragma unroll
        for (int h = 0; h < 32; ++h) o = fmaf(relu(p[h]), d2[h], o);
        out[v] = scv.zero ? 0.0 : static_cast<double>(o + b2) * scv.out_scale;
      }
    } else {
      const float gy = (!live || scv.zero) ? 0.f : static_cast<float>(gov * scv.out_scale);
      float gz[32];
#pragma unroll
      for (int h = 0; h < 32; ++h) {
        gz[h] = p[h] > 0.f ? gy * d2[h] : 0.f;
        acc[h] = fmaf(relu(p[h]), gy, acc[h]);
      }
      acc[32] += gy;
      // g_z as the weight gradient's B operand (bf16 hi/lo, MN-major)
#pragma unroll
      for (int c8 = 0; c8 < 4; ++c8) {
        uint4 hi, lo;
        wgb::split8(make_float4(gz[8 * c8], gz[8 * c8 + 1], gz[8 * c8 + 2], gz[8 * c8 + 3]),
                    make_float4(gz[8 * c8 + 4], gz[8 * c8 + 5], gz[8 * c8 + 6], gz[8 * c8 + 7]), hi, lo);
        *reinterpret_cast<uint4*>(WA + 2 * wgb::OPA + wgb::offB(tid, 8 * c8)) = hi;
        *reinterpret_cast<uint4*>(WA + 2 * wgb::OPA + wgb::OPB + wgb::offB(tid, 8 * c8)) = lo;
      }
#pragma unroll
      for (int c = 0; c < 32; c += 8) {
        float hi[8], lo[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          hi[e] = gz[c + e];
          lo[e] = gz[c + e] - __int_as_float(__float_as_int(gz[c + e]) & 0xffffe000);
        }
        tc::tmem_st8(tR2 + trow + c, hi);
        tc::tmem_st8(tR1 + trow + c, lo);
      }
      tc::tmem_wait_st();
      tc::fence_proxy_async();
      tc::fence_before();
      __syncthreads();
      if (tid == 0) {
        tc::fence_after();
#pragma unroll
        for (int k8 = 0; k8 < 4; ++k8) {
          tc::mma_tf32_ts(tD, tR2 + 8 * k8, tc::make_desc_swz<32>(sB2 + k8 * 32), i64, k8 > 0);
          tc::mma_tf32_ts(tD + 32, tR1 + 8 * k8, tc::make_desc_swz<32>(sB2 + 4096 + k8 * 32), i32, 1);
        }
        // MMA3: Dw (+)= [X_L | 1]ᵀ g_z, products hi·hi + hi·lo + lo·hi
        const uint32_t sAh = tc::smem_u32(WA), sAl = sAh + wgb::OPA;
        const uint32_t sBh = sAl + wgb::OPA, sBl = sBh + wgb::OPB;
        uint32_t accw = since_flush > 0 ? 1u : 0u;
#pragma unroll
        for (int ks = 0; ks < C::TM / 16; ++ks) {
          const uint64_t ah = wgb::desc_mn(sAh + ks * 2048, 1024, 2), al = wgb::desc_mn(sAl + ks * 2048, 1024, 2);
          const uint64_t bh = wgb::desc_mn(sBh + ks * 1024, 512, 4), bl = wgb::desc_mn(sBl + ks * 1024, 512, 4);
          wgb::mma_bf16(tW, ah, bh, accw);
          accw = 1;
          wgb::mma_bf16(tW, ah, bl, 1);
          wgb::mma_bf16(tW, al, bh, 1);
        }
        tc::mma_commit(mbar);
      }
      tc::mbar_wait(mbar, mph & 1);
      ++mph;
      tc::fence_after();
      float g[32];
      {
        float u[16], w[16];
#pragma unroll
        for (int j0 = 0; j0 < 32; j0 += 16) {
          tc::tmem_ld16(tD + trow + j0, u);
          tc::tmem_ld16(tD + trow + 32 + j0, w);
#pragma unroll
          for (int e = 0; e < 16; ++e) g[j0 + e] = (ymask >> (j0 + e)) & 1u ? u[e] + w[e] : 0.f;
        }
      }
      if (++since_flush == wgb::kFlushBf || it + 1 == my) {  // Dw -> this CTA's f64 partials
        float w1[16], w2[16];
        tc::tmem_ld16(tW + trow, w1);
        tc::tmem_ld16(tW + trow + 16, w2);
        if (lane < 16) {
          double* dst = wpart + static_cast<size_t>(blockIdx.x) * 2048 + (16 * warp + lane) * 32;
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            dst[c] += static_cast<double>(w1[c]);
            dst[16 + c] += static_cast<double>(w2[c]);
          }
        }
        since_flush = 0;
      }
      tc::fence_before();
      __syncthreads();  // every thread's G rows may enter the slot
#pragma unroll
      for (int c = 0; c < 32; c += 4)
        *reinterpret_cast<float4*>(yt + tc::swz_off<32>(tid, c)) = make_float4(g[c], g[c + 1], g[c + 2], g[c + 3]);
      __syncthreads();
      store_tile(gpre);
    }
    __syncthreads();  // every thread is done with this slot and the TMEM regions
    if (tid == 0) issue(it + C::NS);
  }
  if constexpr (!FWD) {
    // per-CTA sums in a fixed order: the per-thread values through the (now
    // idle) ring, then 33 threads add the 128 rows' values in f64
    __syncthreads();
    float* accs = reinterpret_cast<float*>(ring);  // [33][128]
#pragma unroll
    for (int h = 0; h < 33; ++h) accs[h * C::NT + tid] = acc[h];
    __syncthreads();
    if (tid < 33) {
      double t = 0.0;
      for (int r = 0; r < C::NT; ++r) t += static_cast<double>(accs[tid * C::NT + r]);
      partials[static_cast<size_t>(blockIdx.x) * 33 + tid] = t;
    }
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 0) tc::tmem_dealloc(tmem, C::TCOLS);
}

}  // namespace gnpk
