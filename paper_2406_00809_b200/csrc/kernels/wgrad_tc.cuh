// Weight / bias gradients on the tensor cores:
//
//   S[m][n] = Σ_v A[v][m] · Bm[v][n]      over all n*B virtual rows v
//
// with A = [A1 | A2] (two 32-feature atoms: layer input X and ÂX for ∂U/∂W,
// or x_L / x0 and a constant 1 for the decoder/encoder weights and biases)
// and Bm the 32-feature gradient rows (gpre, g_dec_pre, gX0).  Restates the
// gemm_tn reductions of src/gnn.cpp:240,265-266,284 (+ the bias column sums).
//
// The activation rows are loaded coalesced, split into tf32 hi/lo and
// transposed while staging into K-major 128B-swizzled operands (operand row =
// feature, K = tile row; MN-major tf32 descriptors produced no result on this
// part, see tests/cuda/tmem_probe.cu): per 128-row tile, 3 x 16
// tcgen05.mma.kind::tf32 (M=64, N=32, K=8; A_lo·B_hi + A_hi·B_lo + A_hi·B_hi),
// accumulator rows m at TMEM lanes 32(m/16) + m%16 (M=64 layout).  The fp32 TMEM
// accumulator is flushed into f64 registers every kFlush tiles, and each CTA
// writes one f64 partial; k_outer_finish sums partials in CTA order
// (deterministic).  Tiles are software-pipelined: the next tile's rows are
// loaded into registers while the tensor core works on the current one.
#pragma once

#include "common.cuh"
#include "tc.cuh"

namespace gnpk {

struct WgradArgs {
  const float* A1;  // [nv][sa1] (features 0..wa1-1 used)
  int wa1, sa1;
  const float* A2;  // [nv][sa2] or nullptr
  int wa2, sa2;
  int ones;         // A2 := [1, 0, 0, ...] (bias column sums)
  const float* Bm;  // [nv][sb] (features 0..wb-1 used, wb <= 32)
  int wb, sb;
  int nv;
  double* partials;  // [grid][64][32]
};

namespace wg {
constexpr int TM = 128;
constexpr int kFlush = 16;              // tiles per fp32 TMEM accumulation
}  // namespace wg
constexpr int kFlushTma = 16;
namespace wg {
constexpr uint32_t ATOM = TM * 128;     // one 32-feature x 128-row atom (bytes)
constexpr int CH = 24;                  // 16-byte chunks per row: 8 A1 + 8 A2 + 8 B
constexpr int CPT = TM * CH / kThreads; // chunks per thread per tile (12)
constexpr int SR = 100;                 // staging row stride (floats): 96 used
// A hi/lo (2 atoms each), B hi/lo, raw staging, mbarrier/TMEM slot, alignment
constexpr size_t smem_bytes() { return 6 * ATOM + TM * SR * 4 + 64 + 1024; }
}  // namespace wg

__global__ void __launch_bounds__(kThreads, 1) k_wgrad_tc(WgradArgs g) {
  using namespace wg;
  extern __shared__ float4 smem_raw[];
  const uint32_t pad = (1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* base = reinterpret_cast<uint8_t*>(smem_raw) + pad;
  uint8_t* Ahi = base;             // atoms 0,1
  uint8_t* Alo = base + 2 * ATOM;  // atoms 0,1
  uint8_t* Bhi = base + 4 * ATOM;
  uint8_t* Blo = base + 5 * ATOM;
  float* Stg = reinterpret_cast<float*>(base + 6 * ATOM);  // [TM][SR] raw staging
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + 6 * ATOM + TM * SR * 4);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) tc::mbar_init(bar, 1);
  if (warp == 0) tc::tmem_alloc(tslot, 32);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;
  constexpr uint32_t idesc = tc::idesc_tf32(64, 32);
  const uint32_t sAhi = tc::smem_u32(Ahi), sAlo = tc::smem_u32(Alo);
  const uint32_t sBhi = tc::smem_u32(Bhi), sBlo = tc::smem_u32(Blo);

  const int ntiles = (g.nv + TM - 1) / TM;
  // contiguous tile range per CTA (deterministic partition)
  const int per = (ntiles + gridDim.x - 1) / gridDim.x;
  const int t_begin = blockIdx.x * per, t_end = min(ntiles, t_begin + per);

  // features [f, f+4) of a row with w used features and stride st
  auto load4 = [](const float* row, int f, int w, int st) -> float4 {
    if (f >= w) return f4zero();
    if (f + 4 <= w && (st & 3) == 0) return ldg4(row + f);
    float t[4] = {0.f, 0.f, 0.f, 0.f};
    for (int i = 0; i < 4 && f + i < w; ++i) t[i] = __ldg(row + f + i);
    return make_float4(t[0], t[1], t[2], t[3]);
  };
  float4 reg[CPT];
  auto load_tile = [&](int tile) {
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
      const int c = tid + q * kThreads;
      const int r = c / CH, ch = c % CH;
      const int v = tile * TM + r;
      float4 x = f4zero();
      if (v < g.nv) {
        if (ch < 8) {
          x = load4(g.A1 + static_cast<size_t>(v) * g.sa1, 4 * ch, g.wa1, g.sa1);
        } else if (ch < 16) {
          const int f = 4 * (ch - 8);
          if (g.ones) x = make_float4(f == 0 ? 1.f : 0.f, 0.f, 0.f, 0.f);
          else if (g.A2) x = load4(g.A2 + static_cast<size_t>(v) * g.sa2, f, g.wa2, g.sa2);
        } else {
          x = load4(g.Bm + static_cast<size_t>(v) * g.sb, 4 * (ch - 16), g.wb, g.sb);
        }
      }
      reg[q] = x;
    }
  };
  // (1) raw rows -> staging [TM][SR] (16-byte stores, chunk-fastest: conflict-free)
  // (2) staging -> K-major operands: lane = row (row-fastest 16-byte reads are
  //     conflict-free since SR/4 = 25 is odd; the transposed scalar stores hit
  //     32 distinct banks under the 128B swizzle)
  auto store_tile = [&]() {
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
      const int c = tid + q * kThreads;
      st4(Stg + (c / CH) * SR + 4 * (c % CH), reg[q]);
    }
    __syncthreads();
#pragma unroll 4
    for (int q = 0; q < CPT; ++q) {
      const int j = tid + q * kThreads;
      const int r = j % TM, ch = j / TM;
      const float4 x = *reinterpret_cast<const float4*>(Stg + r * SR + 4 * ch);
      const float4 h = make_float4(tc::to_tf32(x.x), tc::to_tf32(x.y), tc::to_tf32(x.z), tc::to_tf32(x.w));
      const float4 l = make_float4(x.x - h.x, x.y - h.y, x.z - h.z, x.w - h.w);
      // transpose into the K-major operand: feature = operand row, tile row = K
      uint8_t *dh, *dl;
      int f, rows;
      if (ch < 16) {  // A: feature f in [0, 64)
        f = 4 * ch;
        rows = 64;
        dh = Ahi;
        dl = Alo;
      } else {
        f = 4 * (ch - 16);
        rows = 32;
        dh = Bhi;
        dl = Blo;
      }
      const float hv[4] = {h.x, h.y, h.z, h.w}, lv[4] = {l.x, l.y, l.z, l.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t off = tc::sw128_off(f + i, r, rows);
        *reinterpret_cast<float*>(dh + off) = hv[i];
        *reinterpret_cast<float*>(dl + off) = lv[i];
      }
    }
  };

  // f64 accumulators: warp w holds rows 16(w%4)..+15 (lanes 0..15) and the
  // 16 columns 16(w/4)..+15
  double acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = 0.0;
  uint32_t phase = 0;
  bool outstanding = false;
  auto wait_mma = [&]() {
    if (outstanding) {
      tc::mbar_wait(bar, phase);
      phase ^= 1;
      outstanding = false;
      tc::fence_after();
    }
  };
  auto flush = [&]() {
    wait_mma();
    float v[16];
    const int q = warp & 3, half = warp >> 2;
    tc::tmem_ld16(tmem + (static_cast<uint32_t>(32 * q) << 16) + 16 * half, v);
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] += static_cast<double>(v[i]);
    tc::fence_before();
  };

  int since_flush = 0;
  if (t_begin < t_end) load_tile(t_begin);
  for (int tile = t_begin; tile < t_end; ++tile) {
    wait_mma();  // the tensor core is done with the smem tile
    store_tile();
    tc::fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      tc::fence_after();
      uint32_t accf = since_flush > 0 ? 1u : 0u;
#pragma unroll
      for (int pass = 0; pass < 3; ++pass) {
        const uint32_t sa = pass == 0 ? sAlo : sAhi;
        const uint32_t sb = pass == 1 ? sBlo : sBhi;
#pragma unroll
        for (int s = 0; s < TM / 8; ++s) {
          // K-major: 32-row K atoms (A: 64 x 128 B, B: 32 x 128 B), +32 B per step
          const uint64_t ad = tc::make_desc_sw128(sa + (s >> 2) * 64 * 128 + (s & 3) * 32, 1024);
          const uint64_t bd = tc::make_desc_sw128(sb + (s >> 2) * 32 * 128 + (s & 3) * 32, 1024);
          tc::mma_tf32(tmem, ad, bd, idesc, accf);
          accf = 1;
        }
      }
      tc::mma_commit(bar);
    }
    outstanding = true;
    if (tile + 1 < t_end) load_tile(tile + 1);  // overlaps the MMAs
    if (++since_flush == kFlush) {
      flush();
      __syncthreads();  // all TMEM reads done before the accumulator restarts
      since_flush = 0;
    }
  }
  if (since_flush > 0) flush();
  // per-CTA partial [64][32]: rows 16q + lane (lanes < 16), columns 16 half + i
  {
    const int q = warp & 3, half = warp >> 2;
    if (lane < 16) {
      double* dst = g.partials + static_cast<size_t>(blockIdx.x) * 64 * 32 +
                    static_cast<size_t>(16 * q + lane) * 32 + 16 * half;
#pragma unroll
      for (int i = 0; i < 16; ++i) dst[i] = acc[i];
    }
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 0) tc::tmem_dealloc(tmem, 32);
}

}  // namespace gnpk

// ---------------------------------------------------------------------------
// TMA variant for 32-float rows (d = 32, hidden = 32: every C3 reduction).
// Each tile's A1 / A2 / B rows arrive by cp.async.bulk.tensor into a
// double-buffered 128B-swizzled staging area (mbarrier complete_tx), so the
// HBM latency of tile t+1 overlaps the transpose/split and MMAs of tile t;
// the swizzle makes the row-per-lane 16-byte reads conflict-free.
#include <cuda.h>

namespace gnpk {

struct WgradTmaArgs {
  CUtensorMap a1, a2, b;  // [nv][32] fp32 views, box {32 features, 128 rows}, SWIZZLE_128B
  int a2_mode;            // 0: zeros, 1: tensor a2, 2: ones column (bias sums)
  int nv;
  double* partials;       // [grid][64][32]
};

namespace wgt {
constexpr int TM = 128, TH = 512;
constexpr uint32_t ARR = TM * 128;      // one staged array tile (16 KiB)
constexpr uint32_t STAGE = 3 * ARR;
constexpr uint32_t OPA = 2 * ARR;       // A operand (64 x 128 K-major, 4 K-atoms)
constexpr uint32_t OPB = ARR;           // B operand (32 x 128)
constexpr size_t smem_bytes() { return 2 * STAGE + 2 * OPA + 2 * OPB + 64 + 1024; }
}  // namespace wgt

__global__ void __launch_bounds__(wgt::TH, 1) k_wgrad_tma(const __grid_constant__ WgradTmaArgs g) {
  using namespace wgt;
  extern __shared__ float4 smem_raw[];
  const uint32_t pad = (1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* base = reinterpret_cast<uint8_t*>(smem_raw) + pad;
  uint8_t* stage[2] = {base, base + STAGE};
  uint8_t* Ahi = base + 2 * STAGE;
  uint8_t* Alo = Ahi + OPA;
  uint8_t* Bhi = Alo + OPA;
  uint8_t* Blo = Bhi + OPB;
  uint64_t* full = reinterpret_cast<uint64_t*>(Blo + OPB);  // [2]
  uint64_t* mbar = full + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(mbar + 1);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ntiles = (g.nv + TM - 1) / TM;
  const int per = (ntiles + gridDim.x - 1) / gridDim.x;
  const int t_begin = blockIdx.x * per, t_end = min(ntiles, t_begin + per);
  const int narr = g.a2_mode == 1 ? 3 : 2;
  if (tid == 0) {
    tc::mbar_init(&full[0], 1);
    tc::mbar_init(&full[1], 1);
    tc::mbar_init(mbar, 1);
    tc::tma_prefetch_desc(&g.a1);
    tc::tma_prefetch_desc(&g.b);
    if (g.a2_mode == 1) tc::tma_prefetch_desc(&g.a2);
  }
  if (warp == 0) tc::tmem_alloc(tslot, 32);
  // A atom 1 is constant unless a2 is a tensor: 1.0 in feature 32 (bias) or 0
  if (g.a2_mode != 1) {
    for (int j = tid; j < 32 * TM; j += TH) {
      const int f = 32 + j / TM, r = j % TM;
      const float v = (g.a2_mode == 2 && f == 32) ? 1.f : 0.f;
      const uint32_t off = tc::sw128_off(f, r, 64);
      *reinterpret_cast<float*>(Ahi + off) = v;
      *reinterpret_cast<float*>(Alo + off) = 0.f;
    }
  }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;
  constexpr uint32_t idesc = tc::idesc_tf32(64, 32);
  const uint32_t sAhi = tc::smem_u32(Ahi), sAlo = tc::smem_u32(Alo);
  const uint32_t sBhi = tc::smem_u32(Bhi), sBlo = tc::smem_u32(Blo);

  auto issue = [&](int tile, int s) {
    tc::fence_proxy_async();
    tc::mbar_expect_tx(&full[s], narr * ARR);
    const int y = tile * TM;
    tc::tma_load_2d(stage[s], &g.a1, 0, y, &full[s]);
    tc::tma_load_2d(stage[s] + 2 * ARR, &g.b, 0, y, &full[s]);
    if (g.a2_mode == 1) tc::tma_load_2d(stage[s] + ARR, &g.a2, 0, y, &full[s]);
  };

  double acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.0;
  uint32_t mphase = 0;
  bool outstanding = false;
  auto wait_mma = [&]() {
    if (outstanding) {
      tc::mbar_wait(mbar, mphase);
      mphase ^= 1;
      outstanding = false;
      tc::fence_after();
    }
  };
  auto flush = [&]() {
    wait_mma();
    float v[8];
    const int q = warp & 3, cb = warp >> 2;  // 4 column blocks of 8
    tc::tmem_ld8(tmem + (static_cast<uint32_t>(32 * q) << 16) + 8 * cb, v);
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] += static_cast<double>(v[i]);
    tc::fence_before();
  };

  if (tid == 0 && t_begin < t_end) issue(t_begin, 0);
  int since_flush = 0;
  for (int tile = t_begin; tile < t_end; ++tile) {
    const int k = tile - t_begin, s = k & 1;
    if (tid == 0 && tile + 1 < t_end) issue(tile + 1, s ^ 1);
    tc::mbar_wait(&full[s], (k >> 1) & 1);
    wait_mma();
    // transpose + split: lane = row (conflict-free swizzled 16-byte reads)
    const uint8_t* st = stage[s];
    for (int j = tid; j < TM * 24; j += TH) {
      const int r = j % TM, ch = j / TM;  // ch: 0..7 A1, 8..15 A2, 16..23 B
      const int arr = ch >> 3, c = ch & 7;
      if (arr == 1 && g.a2_mode != 1) continue;
      const float4 x = *reinterpret_cast<const float4*>(st + arr * ARR + r * 128 + ((c ^ (r & 7)) << 4));
      const float xv[4] = {x.x, x.y, x.z, x.w};
      uint8_t* dh = arr == 2 ? Bhi : Ahi;
      uint8_t* dl = arr == 2 ? Blo : Alo;
      const int f0 = arr == 2 ? 4 * c : 4 * ch;
      const int rows = arr == 2 ? 32 : 64;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float h = tc::to_tf32(xv[i]);
        const uint32_t off = tc::sw128_off(f0 + i, r, rows);
        *reinterpret_cast<float*>(dh + off) = h;
        *reinterpret_cast<float*>(dl + off) = xv[i] - h;
      }
    }
    tc::fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      tc::fence_after();
      uint32_t accf = since_flush > 0 ? 1u : 0u;
#pragma unroll
      for (int pass = 0; pass < 3; ++pass) {
        const uint32_t sa = pass == 0 ? sAlo : sAhi;
        const uint32_t sb = pass == 1 ? sBlo : sBhi;
#pragma unroll
        for (int ks = 0; ks < TM / 8; ++ks) {
          const uint64_t ad = tc::make_desc_sw128(sa + (ks >> 2) * 64 * 128 + (ks & 3) * 32, 1024);
          const uint64_t bd = tc::make_desc_sw128(sb + (ks >> 2) * 32 * 128 + (ks & 3) * 32, 1024);
          tc::mma_tf32(tmem, ad, bd, idesc, accf);
          accf = 1;
        }
      }
      tc::mma_commit(mbar);
    }
    outstanding = true;
    if (++since_flush == kFlushTma) {
      flush();
      __syncthreads();
      since_flush = 0;
    }
  }
  if (since_flush > 0) flush();
  {
    const int q = warp & 3, cb = warp >> 2;
    if (lane < 16) {
      double* dst = g.partials + static_cast<size_t>(blockIdx.x) * 64 * 32 +
                    static_cast<size_t>(16 * q + lane) * 32 + 8 * cb;
#pragma unroll
      for (int i = 0; i < 8; ++i) dst[i] = acc[i];
    }
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 0) tc::tmem_dealloc(tmem, 32);
}

}  // namespace gnpk

// ---------------------------------------------------------------------------
// bf16x2-split variant (same arguments and partial layout as k_wgrad_tma).
// The tensor core takes bf16 operands MN-major (probed in tests/cuda/
// mn_bf16_probe.cu; tf32 does not), so the staged row-major tiles convert in
// place order — no transpose: each thread turns 8 features of a row into 8
// bf16 hi + 8 bf16 lo words (one 16-byte store each) in the 128B/64B
// swizzled MN-major operand layout.  x = hi + lo to ~2^-18 relative; the
// products hi·hi + hi·lo + lo·hi are accumulated (lo·lo is below the split
// error), fp32 in TMEM folded into f64 every kFlushBf tiles.  NSTG staged
// tiles stay in flight (the kernel is HBM-latency bound); NOPS operand sets.
#include <cuda_bf16.h>

namespace gnpk {
namespace wgb {
#ifndef GNPC_WGB_NSTG
#define GNPC_WGB_NSTG 2
#endif
#ifndef GNPC_WGB_NOPS
#define GNPC_WGB_NOPS 2  // double-buffered operands: conversion of tile k overlaps MMA(k-1) (C3 22.6 -> 22.3 ms vs 3 stages x 1 set)
#endif
constexpr int TM = 128, TH = 512, NSTG = GNPC_WGB_NSTG, NOPS = GNPC_WGB_NOPS;
constexpr uint32_t ARR = TM * 128;   // one staged fp32 array tile (16 KiB)
constexpr uint32_t STAGE = 3 * ARR;  // A1 | A2 | B
constexpr uint32_t OPA = TM * 128;   // bf16 [128 rows][64 features], SW128 (16 KiB)
constexpr uint32_t OPB = TM * 64;    // bf16 [128 rows][32 features], SW64 (8 KiB)
constexpr uint32_t OPS = 2 * OPA + 2 * OPB;  // one operand set: Ahi | Alo | Bhi | Blo
constexpr size_t smem_bytes() { return NSTG * STAGE + NOPS * OPS + 128 + 1024; }
#ifndef GNPC_FLUSH_BF
#define GNPC_FLUSH_BF 16  // 64 was 1 % faster at C3 but moved the U gradients by 1.9e-5 (fp32 folds over 8K rows)
#endif
constexpr int kFlushBf = GNPC_FLUSH_BF;

__device__ __forceinline__ uint32_t offA(int r, int m) {  // MN-major SW128, bf16
  return static_cast<uint32_t>((r >> 3) * 1024 + (r & 7) * 128 + ((((m >> 3) ^ (r & 7))) << 4) + (m & 7) * 2);
}
__device__ __forceinline__ uint32_t offB(int r, int n) {  // MN-major SW64, bf16
  return static_cast<uint32_t>((r >> 3) * 512 + (r & 7) * 64 + ((((n >> 3) ^ ((r & 7) >> 1)) & 3) << 4) +
                               (n & 7) * 2);
}
__device__ __forceinline__ uint64_t desc_mn(uint32_t saddr, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;  // SBO: stride between 8-row K groups
  d |= 1ull << 46;
  d |= static_cast<uint64_t>(layout) << 61;
  return d;
}
// kind::f16: F32 accumulate, BF16 A/B, both MN-major, N = 32, M = 64
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) | ((32u >> 3) << 17) |
                            ((64u >> 4) << 24);
__device__ __forceinline__ void mma_bf16(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(kIdesc), "r"(acc)
      : "memory");
}
// 2 fp32 -> packed bf16x2 hi and lo (x ≈ hi + lo): one cvt.rn.bf16x2 each,
// hi widened back to fp32 by shifts
__device__ __forceinline__ void split2(float a, float b, uint32_t& hi, uint32_t& lo) {
  uint32_t h;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(b), "f"(a));  // low half = a
  const float ha = __uint_as_float(h << 16), hb = __uint_as_float(h & 0xffff0000u);
  uint32_t l;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(l) : "f"(b - hb), "f"(a - ha));
  hi = h;
  lo = l;
}
__device__ __forceinline__ void split8(float4 x0, float4 x1, uint4& hi, uint4& lo) {
  split2(x0.x, x0.y, hi.x, lo.x);
  split2(x0.z, x0.w, hi.y, lo.y);
  split2(x1.x, x1.y, hi.z, lo.z);
  split2(x1.z, x1.w, hi.w, lo.w);
}
}  // namespace wgb

__global__ void __launch_bounds__(wgb::TH, 1) k_wgrad_bf16(const __grid_constant__ WgradTmaArgs g) {
  using namespace wgb;
  extern __shared__ float4 smem_raw[];
  const uint32_t pad = (1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* base = reinterpret_cast<uint8_t*>(smem_raw) + pad;
  uint8_t* stg = base;
  uint8_t* ops = base + NSTG * STAGE;  // [2] operand sets
  uint64_t* full = reinterpret_cast<uint64_t*>(ops + NOPS * OPS);  // [NSTG]
  uint64_t* mbar = full + NSTG;  // [2]: tile k's MMAs commit to mbar[k & 1]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(mbar + 2);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ntiles = (g.nv + TM - 1) / TM;
  const int per = (ntiles + gridDim.x - 1) / gridDim.x;
  const int t_begin = blockIdx.x * per, t_end = min(ntiles, t_begin + per);
  const int narr = g.a2_mode == 1 ? 3 : 2;
  if (tid == 0) {
    for (int s = 0; s < NSTG; ++s) tc::mbar_init(&full[s], 1);
    tc::mbar_init(&mbar[0], 1);
    tc::mbar_init(&mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    tc::tma_prefetch_desc(&g.a1);
    tc::tma_prefetch_desc(&g.b);
    if (g.a2_mode == 1) tc::tma_prefetch_desc(&g.a2);
  }
  if (warp == 0) tc::tmem_alloc(tslot, 32);
  // features 32..63 are constant unless a2 is a tensor: 1.0 at 32 (bias) or 0
  if (g.a2_mode != 1) {
    for (int j = tid; j < NOPS * TM * 32; j += TH) {
      const int b = j / (TM * 32), r = (j / 32) % TM, m = 32 + j % 32;
      const float v = (g.a2_mode == 2 && m == 32) ? 1.f : 0.f;
      *reinterpret_cast<__nv_bfloat16*>(ops + b * OPS + offA(r, m)) = __float2bfloat16_rn(v);
      *reinterpret_cast<__nv_bfloat16*>(ops + b * OPS + OPA + offA(r, m)) = __float2bfloat16_rn(0.f);
    }
  }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;

  auto issue = [&](int tile) {
    const int k = tile - t_begin, s = k % NSTG;
    uint8_t* st = stg + s * STAGE;
    tc::mbar_expect_tx(&full[s], narr * ARR);
    const int y = tile * TM;
    tc::tma_load_2d(st, &g.a1, 0, y, &full[s]);
    tc::tma_load_2d(st + 2 * ARR, &g.b, 0, y, &full[s]);
    if (g.a2_mode == 1) tc::tma_load_2d(st + ARR, &g.a2, 0, y, &full[s]);
  };

  double acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.0;
  // tile k's MMAs (local index) commit to mbar[k & 1] as that barrier's
  // (k >> 1)-th phase; a barrier never runs two phases ahead of its waiters
  // (tile k+2 commits only after every thread passed its wait for tile k)
  int committed = 0;
  auto wait_tile = [&](int k) {
    if (k < 0) return;
    tc::mbar_wait(&mbar[k & 1], (k >> 1) & 1);
    tc::fence_after();
  };
  auto wait_mma = [&]() { wait_tile(committed - 1); };  // in-order completion
  auto flush = [&]() {
    wait_mma();
    float v[8];
    const int q = warp & 3, cb = warp >> 2;  // 4 column blocks of 8
    tc::tmem_ld8(tmem + (static_cast<uint32_t>(32 * q) << 16) + 8 * cb, v);
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] += static_cast<double>(v[i]);
    tc::fence_before();
  };

  if (tid == 0)
    for (int t = t_begin; t < min(t_end, t_begin + NSTG); ++t) issue(t);
  int since_flush = 0;
  for (int tile = t_begin; tile < t_end; ++tile) {
    const int k = tile - t_begin, s = k % NSTG;
    tc::mbar_wait(&full[s], (k / NSTG) & 1);
    wait_tile(k - NOPS);  // MMA(k-NOPS) used this operand set
    uint8_t* Ahi = ops + (k % NOPS) * OPS;
    uint8_t* Alo = Ahi + OPA;
    uint8_t* Bhi = Alo + OPA;
    uint8_t* Blo = Bhi + OPB;
    // convert: thread = (row r, 8-feature chunk c8) of A1, A2 and B
    const uint8_t* st = stg + s * STAGE;
    {
      const int r = tid >> 2, c8 = tid & 3;
      const uint32_t i0 = (((2 * c8) ^ (r & 7)) << 4), i1 = (((2 * c8 + 1) ^ (r & 7)) << 4);
#pragma unroll
      for (int arr = 0; arr < 3; ++arr) {
        if (arr == 1 && g.a2_mode != 1) continue;
        const uint8_t* src = st + arr * ARR + r * 128;
        uint4 hi, lo;
        split8(*reinterpret_cast<const float4*>(src + i0), *reinterpret_cast<const float4*>(src + i1), hi, lo);
        if (arr < 2) {
          const uint32_t o = offA(r, 32 * arr + 8 * c8);
          *reinterpret_cast<uint4*>(Ahi + o) = hi;
          *reinterpret_cast<uint4*>(Alo + o) = lo;
        } else {
          const uint32_t o = offB(r, 8 * c8);
          *reinterpret_cast<uint4*>(Bhi + o) = hi;
          *reinterpret_cast<uint4*>(Blo + o) = lo;
        }
      }
    }
    tc::fence_proxy_async();
    tc::fence_before();
    __syncthreads();
    if (tid == 0) {
      tc::fence_after();
      const uint32_t sAhi = tc::smem_u32(Ahi), sAlo = tc::smem_u32(Alo);
      const uint32_t sBhi = tc::smem_u32(Bhi), sBlo = tc::smem_u32(Blo);
      uint32_t accf = since_flush > 0 ? 1u : 0u;
#pragma unroll
      for (int ks = 0; ks < TM / 16; ++ks) {
        const uint64_t ah = desc_mn(sAhi + ks * 2048, 1024, 2), al = desc_mn(sAlo + ks * 2048, 1024, 2);
        const uint64_t bh = desc_mn(sBhi + ks * 1024, 512, 4), bl = desc_mn(sBlo + ks * 1024, 512, 4);
        mma_bf16(tmem, ah, bh, accf);
        accf = 1;
        mma_bf16(tmem, ah, bl, 1);
        mma_bf16(tmem, al, bh, 1);
      }
      tc::mma_commit(&mbar[k & 1]);
      // stage s is consumed: it takes tile + NSTG
      if (tile + NSTG < t_end) issue(tile + NSTG);
    }
    ++committed;
    if (++since_flush == kFlushBf) {
      flush();
      __syncthreads();
      since_flush = 0;
    }
  }
  if (since_flush > 0) flush();
  {
    const int q = warp & 3, cb = warp >> 2;
    if (lane < 16) {
      double* dst = g.partials + static_cast<size_t>(blockIdx.x) * 64 * 32 +
                    static_cast<size_t>(16 * q + lane) * 32 + 8 * cb;
#pragma unroll
      for (int i = 0; i < 8; ++i) dst[i] = acc[i];
    }
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 0) tc::tmem_dealloc(tmem, 32);
}

}  // namespace gnpk
