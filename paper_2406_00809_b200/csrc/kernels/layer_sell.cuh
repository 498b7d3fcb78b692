// Fused Res-GCONV layer for the apply path on sliced-ELL matrices:
//
//   Y = relu(X·U + (ÂX)·W)                         (src/gnn.cpp:164-176)
//   last layer: out = τ/√n · (dec2ᵀ relu(dec1ᵀ y + b1) + b2)   (src/gnn.cpp:178-199)
//
// One persistent 512-thread CTA per SM walks 128-row tiles through an
// asynchronous pipeline so HBM streams stay in flight across tiles:
//
//   TMA ring (NS slots, thread 0): the X tile (2-D tensor load, swizzled, so
//     it IS the tensor core's A_hi operand for X·U — tcgen05 kind::tf32 reads
//     only the top 19 bits of an fp32 word, probed in tests/cuda/
//     tf32_round_probe.cu) and the tile's sliced-ELL (col, val) slice (1-D
//     bulk copy), issued NS-1 tiles ahead;
//   gather: G = DP/4 lanes per row, every row of the slice has K entries
//     (padding has weight 0), 128-bit X-row loads, fp32 sums in stored order;
//   epilogue of the previous tile (its MMA overlapped this gather): TMEM →
//     registers (warp w reads lanes 32(w%4).., column quarter w/4), relu,
//     swizzled smem staging, then ONE 2-D TMA store of the whole tile (or the
//     projection MLP for the last layer);
//   split: X_lo = X - trunc(X), (ÂX)_hi = ÂX, (ÂX)_lo into swizzled smem;
//   MMA (thread 0): 3xTF32 — A_lo·B_hi + A_hi·B_lo + A_hi·B_hi over the
//     (X, U) and (ÂX, W) operand pairs, M=128, N=DP, K=8 steps, into TMEM.
//
// Operands are K-major with the canonical swizzle of their row width:
// 128-byte rows (DP=32) use SWIZZLE_128B, 64-byte rows (DP=16) SWIZZLE_64B —
// the same pattern the TMA unit writes, so loaded tiles feed the MMA as is.
#pragma once

#include <cuda.h>

#include "layer_tc.cuh"

namespace gnpk {

namespace tc {

// Byte offset of fp32 element (row, k), 0 <= k < DP, in a K-major operand of
// DP-wide rows with the matching swizzle (16-byte chunk index XOR row bits).
template <int DP>
__host__ __device__ constexpr uint32_t swz_off(int row, int k) {
  if constexpr (DP == 32)
    return static_cast<uint32_t>((row >> 3) * 1024 + (row & 7) * 128 + (((k >> 2) ^ (row & 7)) << 4) +
                                 (k & 3) * 4);
  else
    return static_cast<uint32_t>((row >> 3) * 512 + (row & 7) * 64 +
                                 (((k >> 2) ^ ((row >> 1) & 3)) << 4) + (k & 3) * 4);
}

template <int DP>
__device__ __forceinline__ uint64_t make_desc_swz(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1u) << 16;                                 // LBO (unused, swizzled K-major)
  d |= static_cast<uint64_t>(((DP == 32 ? 1024u : 512u) >> 4) & 0x3FFFu) << 32;  // SBO: 8-row group
  d |= 1ull << 46;                                                      // version
  d |= static_cast<uint64_t>(DP == 32 ? 2 : 4) << 61;                   // SWIZZLE_128B / SWIZZLE_64B
  return d;
}

__device__ __forceinline__ void tmem_ld4(uint32_t taddr, float (&v)[4]) {
  uint32_t r[4];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i] = __uint_as_float(r[i]);
}

// 2-D tile store smem -> global (bulk-group completion).
__device__ __forceinline__ void tma_store_2d(const void* tmap, const void* src, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(tmap),
               "r"(smem_u32(src)), "r"(x), "r"(y)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

}  // namespace tc

template <int DP>
struct SellCfg {
  static constexpr int NW = 16;                  // math warps (gather / epilogue / split)
  static constexpr int NT = 32 * (NW + 1);       // + one control warp (MMA, TMA, stores)
  static constexpr int TM = 128;                 // rows per tile (MMA M)
  static constexpr int G = DP / 4;               // lanes per row
  static constexpr int NG = 32 * NW / G;         // row groups
  static constexpr int R = TM / NG;              // rows per group
  static constexpr int US = DP == 16 ? 8 : 3;    // slice entries per gather round
  static constexpr int NS = DP == 16 ? 4 : 3;    // TMA ring depth (tiles)
  static constexpr int KCAP = 24;                // slices with K <= KCAP are staged (mult. of US)
  static constexpr uint32_t OPB = TM * DP * 4;   // one A-type operand / X tile / Y tile (bytes)
  static constexpr uint32_t BB = DP * DP * 4;    // one B operand (bytes)
  static constexpr int TCOLS = 2 * DP;           // TMEM accumulator columns (two halves)
  static constexpr uint32_t CVB = KCAP * TM * 8; // staged slice (bytes)
  static constexpr uint32_t SLOT = ((OPB + CVB) + 1023) & ~1023u;  // ring slot: [X tile | slice]
  // layout (offsets from the 1024-aligned base)
  static constexpr uint32_t O_RING = 0;
  static constexpr uint32_t O_A = O_RING + NS * SLOT;     // A1_lo, A2_hi, A2_lo
  static constexpr uint32_t O_B = O_A + 3 * OPB;          // Bu_lo, Bu_hi, Bw_lo, Bw_hi
  static constexpr uint32_t O_Y = O_B + 4 * BB;           // Y staging [2]
  static constexpr uint32_t O_P = O_Y + 2 * OPB;          // LAST: dec1 [DP][H], b1 [H], dec2 [H]
  static size_t smem_bytes(bool last, int hidden) {
    size_t b = O_P + (last ? (size_t)(DP + 2) * hidden * 4 : 0);
    b = (b + 15) & ~size_t(15);
    return b + 128 + 1024;  // barriers + TMEM slot, 1024-B alignment slack
  }
};

struct SellMaps {
  CUtensorMap x;  // layer input  [n][DP], box {DP, 128}, swizzled
  CUtensorMap y;  // layer output [n][DP] (unused by the last layer)
};

// Sliced-ELL gather, R rows per group, rounds of US entries.  Slots past K
// read an in-bounds stale slice word (the ring is zeroed at start) and are
// given weight 0 and the round's first column, so no load is predicated.
template <int DP, int R, int US, int TM, bool SMEM>
__device__ __forceinline__ void gather_sell_rows(const float* __restrict__ X, int gl, const int2* cv,
                                                 int K, int gid, float4 (&acc)[R]) {
  const char* xb = reinterpret_cast<const char*>(X + 4 * gl);
  for (int k = 0; k < K; k += US) {
    int c[R][US];
    float w[R][US];
#pragma unroll
    for (int u = 0; u < US; ++u) {
      const bool on = k + u < K;
      // the group's R rows are adjacent: their entries are one vector load
      int2 e[R];
      const int2* src = cv + (k + u) * TM + R * gid;
      if constexpr (R == 2) {
        int4 v4;
        if constexpr (SMEM) {
          v4 = *reinterpret_cast<const int4*>(src);
        } else {
          v4 = on ? __ldg(reinterpret_cast<const int4*>(src)) : make_int4(0, 0, 0, 0);
        }
        e[0] = make_int2(v4.x, v4.y);
        e[1] = make_int2(v4.z, v4.w);
      } else {
#pragma unroll
        for (int j = 0; j < R; ++j) {
          if constexpr (SMEM) {
            e[j] = src[j];
          } else {
            e[j] = on ? __ldg(src + j) : make_int2(0, 0);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < R; ++j) {
        // past K: weight 0, and the round's first (valid, just requested)
        // column so the dead load hits the same line
        c[j][u] = (u == 0 || on) ? e[j].x : c[j][0];
        w[j][u] = on ? __int_as_float(e[j].y) : 0.f;
      }
    }
    float4 x[R][US];
#pragma unroll
    for (int u = 0; u < US; ++u)
#pragma unroll
      for (int j = 0; j < R; ++j)
        x[j][u] = ldg4(reinterpret_cast<const float*>(
            xb + static_cast<unsigned long long>(static_cast<unsigned>(c[j][u])) * (DP * 4ull)));
#pragma unroll
    for (int u = 0; u < US; ++u)
#pragma unroll
      for (int j = 0; j < R; ++j) fma4(acc[j], w[j][u], x[j][u]);
  }
}

__device__ __forceinline__ float4 f4_trunc_lo(float4 v) {
  return make_float4(v.x - __int_as_float(__float_as_int(v.x) & 0xffffe000),
                     v.y - __int_as_float(__float_as_int(v.y) & 0xffffe000),
                     v.z - __int_as_float(__float_as_int(v.z) & 0xffffe000),
                     v.w - __int_as_float(__float_as_int(v.w) & 0xffffe000));
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(bar)) : "memory");
}

// LAST = true: projection epilogue writing out[i] (no Y).  uwp: this layer's
// B operands [Bu_lo | Bu_hi | Bw_lo | Bw_hi] in the swz_off<DP> layout.
//
// Synchronisation (no CTA-wide barrier inside the loop):
//   full[s]  : ring slot s landed (TMA tx-count), control -> math warps
//   afull    : the tile's A operands + the previous tile's Y staging are
//              written (one arrival per math warp), math -> control warp
//   mma_bar  : MMA committed, control -> math warps; its completion also
//              implies the ring slot it read and the Y staging buffer the
//              next epilogue writes are free (the control warp waits for the
//              older store's smem reads before issuing the MMA).
template <int DP, bool LAST, typename OutT>
__global__ void __launch_bounds__(SellCfg<DP>::NT, 1)
k_layer_sell(DevCsr a, const __grid_constant__ SellMaps maps, const float* __restrict__ X,
             const float* __restrict__ axlong, const float* __restrict__ uwp, NetView net,
             const ApplyScalars* __restrict__ sc, OutT* __restrict__ out, const int* __restrict__ skip) {
  using C = SellCfg<DP>;
  constexpr int TM = C::TM, G = C::G, NG = C::NG, R = C::R, NS = C::NS, NW = C::NW;
  if (skip && *skip) return;
  const int n = a.n;
  const int ntiles = (n + TM - 1) / TM;
  if (sc->zero) {
    if constexpr (LAST) {
      for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        out[i] = OutT(0);
    }
    return;
  }
  extern __shared__ float4 smem_raw[];
  const uint32_t pad = (1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* base = reinterpret_cast<uint8_t*>(smem_raw) + pad;
  uint8_t* ring = base + C::O_RING;
  uint8_t* A1lo = base + C::O_A;
  uint8_t* A2hi = A1lo + C::OPB;
  uint8_t* A2lo = A2hi + C::OPB;
  uint8_t* Bs = base + C::O_B;
  uint8_t* Ystg = base + C::O_Y;
  float* D1 = reinterpret_cast<float*>(base + C::O_P);
  const int H = net.hidden;
  float* B1 = D1 + DP * H;
  float* D2 = B1 + H;
  uint64_t* full = reinterpret_cast<uint64_t*>(
      base + ((C::O_P + (LAST ? (DP + 2) * H * 4 : 0) + 15) & ~15u));
  uint64_t* mma_bar = full + NS;
  uint64_t* afull = mma_bar + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(afull + 1);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int t = tid; t < int(4 * C::BB / 16); t += C::NT)
    reinterpret_cast<float4*>(Bs)[t] = reinterpret_cast<const float4*>(uwp)[t];
  for (int t = tid; t < int(NS * C::SLOT / 16); t += C::NT)  // stale slice words must be valid columns
    reinterpret_cast<float4*>(ring)[t] = f4zero();
  if constexpr (LAST) {
    for (int t = tid; t < DP * H; t += C::NT) D1[t] = net.dec1[t];
    for (int t = tid; t < H; t += C::NT) {
      B1[t] = net.dec1_b[t];
      D2[t] = net.dec2[t];
    }
  }
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) tc::mbar_init(&full[s], 1);
    tc::mbar_init(mma_bar, 1);
    tc::mbar_init(afull, NW);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tc::tmem_alloc(tslot, C::TCOLS);
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;

  if (warp == NW) {
    // ============================================================ control warp
    if (lane == 0) {
      tc::tma_prefetch_desc(&maps.x);
      if (!LAST) tc::tma_prefetch_desc(&maps.y);
      auto issue = [&](int it) {
        const int t = blockIdx.x + it * gridDim.x;
        if (t >= ntiles) return;
        const int s = it % NS;
        uint8_t* slot = ring + s * C::SLOT;
        const int K = __ldg(a.sell_k + t) & 0xffff;
        const bool staged = K > 0 && K <= C::KCAP;
        tc::mbar_expect_tx(&full[s], C::OPB + (staged ? K * TM * 8 : 0));
        tc::tma_load_2d(slot, &maps.x, 0, t * TM, &full[s]);
        if (staged) tc::bulk_load(slot + C::OPB, a.sell + __ldg(a.sell_off + t), K * TM * 8, &full[s]);
      };
      for (int it = 0; it < NS - 1; ++it) issue(it);
      constexpr uint32_t idesc = tc::idesc_tf32(128, DP);
      const uint32_t sA1lo = tc::smem_u32(A1lo), sA2hi = tc::smem_u32(A2hi), sA2lo = tc::smem_u32(A2lo);
      const uint32_t sBstk = tc::smem_u32(Bs);
      constexpr uint32_t idesc2 = tc::idesc_tf32(128, 2 * DP);
      int it = 0, prev_row0 = -1;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        tc::mbar_wait(afull, it & 1);
        tc::fence_after();
        tc::bulk_wait_read0();  // Y staging the next epilogue writes is free
        const uint32_t sX = tc::smem_u32(ring + (it % NS) * C::SLOT);
        // 3xTF32 with the two A_hi products stacked along N (A_hi is read
        // once for both): D[:, 0:DP] = A_hi·B_lo, D[:, DP:2DP] = A_hi·B_hi +
        // A_lo·B_hi; the epilogue adds the halves.  Each part's B operands are
        // stored [B_lo | B_hi], i.e. as one 2DP-row operand.
        uint32_t accf = 0;
#pragma unroll
        for (int part = 0; part < 2; ++part) {
          const uint32_t sah = part == 0 ? sX : sA2hi, sal = part == 0 ? sA1lo : sA2lo;
          const uint32_t sbs = sBstk + part * 2 * C::BB;  // [B_lo; B_hi] of this part (2DP rows)
          const uint32_t sbh = sbs + C::BB;                // B_hi rows alone
#pragma unroll
          for (int k8 = 0; k8 < DP / 8; ++k8) {
            tc::mma_tf32(tmem, tc::make_desc_swz<DP>(sah + k8 * 32), tc::make_desc_swz<DP>(sbs + k8 * 32),
                         idesc2, accf);
            accf = 1;
            tc::mma_tf32(tmem + DP, tc::make_desc_swz<DP>(sal + k8 * 32), tc::make_desc_swz<DP>(sbh + k8 * 32),
                         idesc, 1);
          }
        }
        tc::mma_commit(mma_bar);
        if (!LAST && prev_row0 >= 0) {
          tc::tma_store_2d(&maps.y, Ystg + ((it - 1) & 1) * C::OPB, 0, prev_row0);
          tc::bulk_commit();
        }
        // MMA(it-1) completed before the math warps' epilogues released afull:
        // its ring slot takes tile it+NS-1
        issue(it + NS - 1);
        prev_row0 = tile * TM;
      }
      if (prev_row0 >= 0) {
        tc::mbar_wait(afull, it & 1);  // last tile's Y staging written
        if (!LAST) {
          tc::tma_store_2d(&maps.y, Ystg + ((it - 1) & 1) * C::OPB, 0, prev_row0);
          tc::bulk_commit();
        }
      }
      tc::bulk_wait0();
    }
    __syncwarp();
  } else {
    // ============================================================== math warps
    const int gl = tid % G, gid = tid / G;
    uint32_t mma_phase = 0;
    // epilogue of the tile whose accumulator sits in TMEM (local index itp).
    // Non-last layers: relu'd rows -> Ystg[itp & 1] (warp w: lanes 32(w%4)..,
    // column quarter w/4), stored by the control warp's TMA.  Last layer: the
    // projection group of this tile (warps 4*(itp%4)..+3, one per lane
    // quarter) pulls whole rows into registers `y` and projects them after
    // arriving — the groups rotate, so no CTA-wide barrier is needed.
    float y[LAST ? DP : 1];
    auto epilogue = [&](int itp) -> bool {
      tc::mbar_wait(mma_bar, mma_phase);
      mma_phase ^= 1;
      tc::fence_after();
      const int q = warp & 3, cq = warp >> 2;
      const uint32_t trow = tmem + (static_cast<uint32_t>(32 * q) << 16);
      if constexpr (LAST) {
        if (cq != (itp & 3)) return false;
#pragma unroll
        for (int c0 = 0; c0 < DP; c0 += 16) {
          float v[16], v2[16];
          tc::tmem_ld16(trow + c0, v);
          tc::tmem_ld16(trow + DP + c0, v2);
#pragma unroll
          for (int c = 0; c < 16; ++c) y[c0 + c] = relu(v[c] + v2[c]);
        }
        tc::fence_before();
        return true;
      } else {
        const int m = 32 * q + lane;
        constexpr int CW = DP / 4;  // columns per warp
        uint8_t* ys = Ystg + (itp & 1) * C::OPB;
        const uint32_t taddr = trow + cq * CW;
        if constexpr (CW == 8) {
          float v[8], v2[8];
          tc::tmem_ld8(taddr, v);
          tc::tmem_ld8(taddr + DP, v2);
#pragma unroll
          for (int c = 0; c < 8; ++c) v[c] += v2[c];
          *reinterpret_cast<float4*>(ys + tc::swz_off<DP>(m, cq * CW)) =
              make_float4(relu(v[0]), relu(v[1]), relu(v[2]), relu(v[3]));
          *reinterpret_cast<float4*>(ys + tc::swz_off<DP>(m, cq * CW + 4)) =
              make_float4(relu(v[4]), relu(v[5]), relu(v[6]), relu(v[7]));
        } else {
          float v[4], v2[4];
          tc::tmem_ld4(taddr, v);
          tc::tmem_ld4(taddr + DP, v2);
#pragma unroll
          for (int c = 0; c < 4; ++c) v[c] += v2[c];
          *reinterpret_cast<float4*>(ys + tc::swz_off<DP>(m, cq * CW)) =
              make_float4(relu(v[0]), relu(v[1]), relu(v[2]), relu(v[3]));
        }
        tc::fence_before();
        return false;
      }
    };
    auto arrive = [&]() {
      tc::fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(afull);
    };
    // LAST: projection MLP (src/gnn.cpp:178-199) of the row this lane holds
    // (row 32*(warp%4) + lane of the tile at row0): dec1 read as warp-uniform
    // float4 broadcasts.
    auto project = [&](int row0) {
      if constexpr (LAST) {
        float o = 0.f;
        if ((H & 3) == 0) {
          for (int h0 = 0; h0 < H; h0 += 4) {
            float4 t = f4zero();
#pragma unroll
            for (int j = 0; j < DP; ++j) fma4(t, y[j], *reinterpret_cast<const float4*>(D1 + j * H + h0));
            o = fmaf(relu(t.x + B1[h0]), D2[h0], o);
            o = fmaf(relu(t.y + B1[h0 + 1]), D2[h0 + 1], o);
            o = fmaf(relu(t.z + B1[h0 + 2]), D2[h0 + 2], o);
            o = fmaf(relu(t.w + B1[h0 + 3]), D2[h0 + 3], o);
          }
        } else {
          for (int h = 0; h < H; ++h) {
            float t = 0.f;
#pragma unroll
            for (int j = 0; j < DP; ++j) t = fmaf(y[j], D1[j * H + h], t);
            o = fmaf(relu(t + B1[h]), D2[h], o);
          }
        }
        const int i = row0 + 32 * (warp & 3) + lane;
        if (i < n) out[i] = static_cast<OutT>(static_cast<double>(o + net.dec2_b) * sc->out_scale);
      }
    };

    int it = 0, prev_row0 = -1;
    int kw = blockIdx.x < ntiles ? __ldg(a.sell_k + blockIdx.x) : 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int row0 = tile * TM;
      const int s = it % NS;
      uint8_t* slot = ring + s * C::SLOT;
      const int K = kw & 0xffff;
      const bool haslong = (kw >> 16) != 0;
      const bool staged = K > 0 && K <= C::KCAP;
      const int nxt = tile + gridDim.x;
      kw = nxt < ntiles ? __ldg(a.sell_k + nxt) : 0;  // prefetch

      // ----------------------------------------------------------- gather
      float4 acc[R];
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const int i = row0 + R * gid + j;
        acc[j] = f4zero();
        if (haslong && i < n && __ldg(a.rp + i + 1) - __ldg(a.rp + i) > kLongRow)
          acc[j] = ldg4(axlong + static_cast<size_t>(i) * DP + 4 * gl);
      }
      tc::mbar_wait(&full[s], (it / NS) & 1);
      if (staged)
        gather_sell_rows<DP, R, C::US, TM, true>(X, gl, reinterpret_cast<const int2*>(slot + C::OPB), K,
                                                     gid, acc);
      else
        gather_sell_rows<DP, R, C::US, TM, false>(X, gl, a.sell + __ldg(a.sell_off + tile), K, gid, acc);

      // ------------------------------------------ previous tile: epilogue
      const bool proj = prev_row0 >= 0 && epilogue(it - 1);

      // ------------------------------------------------------------ split
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const int r = R * gid + j;
        const uint32_t o = tc::swz_off<DP>(r, 4 * gl);
        const float4 xv = *reinterpret_cast<const float4*>(slot + o);
        *reinterpret_cast<float4*>(A1lo + o) = f4_trunc_lo(xv);
        *reinterpret_cast<float4*>(A2hi + o) = acc[j];
        *reinterpret_cast<float4*>(A2lo + o) = f4_trunc_lo(acc[j]);
      }
      arrive();
      if (proj) project(prev_row0);
      prev_row0 = row0;
    }
    if (prev_row0 >= 0) {
      const bool proj = epilogue(it - 1);
      arrive();
      if (proj) project(prev_row0);
    }
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 0) tc::tmem_dealloc(tmem, C::TCOLS);
}

}  // namespace gnpk
