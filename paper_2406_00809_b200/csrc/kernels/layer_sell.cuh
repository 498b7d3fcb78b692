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

// CSR = false: sliced-ELL slices (k_layer_sell on regular matrices);
// CSR = true : the short-row CSR ranges of the tile (ragged matrices).
template <int DP, bool CSR = false>
struct SellCfg {
  // one CTA per SM: 16 math warps on one tile at a time (two 8-warp CTAs per
  // SM measured slower at DP=16: C2 26.0 vs 24.4 us, C4 213 vs 160 us)
  static constexpr int NW = 16;                  // math warps (gather / epilogue / split)
  static constexpr int CPS = 1;                  // CTAs per SM
  static constexpr int NT = 32 * (NW + 1);       // + one control warp (MMA, TMA, stores)
  static constexpr int NQ = NW / 4;              // epilogue column groups (warps per TMEM lane quarter)
  static constexpr int TM = 128;                 // rows per tile (MMA M)
  static constexpr int G = DP / 4;               // lanes per row
  static constexpr int NG = 32 * NW / G;         // row groups
  static constexpr int R = TM / NG;              // rows per group
  static constexpr int US = DP == 16 ? 8 : 3;    // slice entries per gather round
  static constexpr int USC = DP == 16 ? 8 : 4;   // CSR entries per gather round
  // TMA ring depth (tiles) and epilogue lag (A/TMEM buffer sets), measured
  // per format: SELL DP16 (C2) best at NS 4 / LAG 1 (LAG 2 + NS 5: 25.7 vs
  // 24.4 us); CSR DP16 (C4) at NS 5 (166 vs 197 us at NS 4); DP32 fills smem
  static constexpr int NS = DP == 16 ? (CSR ? 5 : 4) : 3;
  static constexpr int KCAP = 24;                // slices with K <= KCAP are staged (mult. of US)
  static constexpr uint32_t OPB = TM * DP * 4;   // one A-type operand / X tile / Y tile (bytes)
  static constexpr uint32_t BB = DP * DP * 4;    // one B operand (bytes)
  static constexpr int TCOLS = 2 * DP;           // TMEM accumulator columns (two halves)
  static constexpr int LAG = 1;
  static constexpr int TALLOC = LAG * TCOLS < 32 ? 32 : LAG * TCOLS;  // power of two >= 32
  static constexpr uint32_t CVB = KCAP * TM * 8; // staged slice (bytes)
  // CSR: [X tile | row_ptr slice (TM+4 ints, 1 KiB) | col_idx (CAPC) | values (CAPC)]
  static constexpr int CAPC = 2048;              // staged short-row nonzeros per tile
  static constexpr uint32_t RPB = (TM + 4) * 4;  // row_ptr slice copy (bytes, 16-B multiple)
  static constexpr uint32_t O_RP = OPB, O_CI = OPB + 1024, O_V = O_CI + CAPC * 4;
  static constexpr uint32_t SLOT =
      CSR ? ((O_V + CAPC * 4 + 1023) & ~1023u) : (((OPB + CVB) + 1023) & ~1023u);
  // layout (offsets from the 1024-aligned base)
  static constexpr uint32_t O_RING = 0;
  static constexpr uint32_t O_A = O_RING + NS * SLOT;     // A1_lo, A2_hi, A2_lo
  static constexpr uint32_t O_B = O_A + LAG * 3 * OPB;    // Bu_lo, Bu_hi, Bw_lo, Bw_hi
  static constexpr uint32_t O_Y = O_B + 4 * BB;           // Y staging [2]
  static constexpr int NY = LAG + 1;                      // Y staging buffers
  static constexpr uint32_t O_P = O_Y + NY * OPB;         // LAST: dec1 [DP][H], b1 [H], dec2 [H]
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

// CSR gather: row r = R*gid + j of the tile spans [s_j, s_j + len_j) of the
// staged (or global) col/val arrays; rounds of US entries up to the longer
// of the group's rows.  Slots past a row's end get weight 0 and the row's own
// X row (in bounds, usually cached), so no load is predicated.
template <int DP, int R, int US>
__device__ __forceinline__ void gather_csr_rows(const float* __restrict__ X, int gl, const int* ci,
                                                const float* vv, const int (&s)[R], const int (&len)[R],
                                                const int (&self)[R], float4 (&acc)[R]) {
  const char* xb = reinterpret_cast<const char*>(X + 4 * gl);
  int kmax = len[0];
#pragma unroll
  for (int j = 1; j < R; ++j) kmax = max(kmax, len[j]);
  for (int k = 0; k < kmax; k += US) {
    int c[R][US];
    float w[R][US];
#pragma unroll
    for (int u = 0; u < US; ++u)
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const bool on = k + u < len[j];
        const int idx = s[j] + k + u;
        c[j][u] = on ? ci[idx] : self[j];
        w[j][u] = on ? vv[idx] : 0.f;
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
// Synchronisation (no CTA-wide barrier inside the loop).  Local iteration it
// gathers/splits tile it and runs the epilogue of tile it - LAG (LAG = 2
// double-buffers the A operands and the TMEM accumulator, so a warp waits for
// an MMA issued a whole iteration earlier; LAG = 1 where shared memory is
// short):
//   full[s]     : ring slot s landed (TMA tx-count), control -> math warps
//   afull[b]    : tile it's A operands and tile it-LAG's Y staging are
//                 written (one arrival per math warp; it % LAG == b), math ->
//                 control warp.  One barrier per lag slot: with a single one
//                 the math warps could complete two phases before the control
//                 warp observes the first (parity ABA)
//   mma_bar[b]  : MMA of a tile with it % LAG == b committed, control -> math
//                 warps.  Its completion also means the Y staging buffer the
//                 next epilogue writes is free (the control warp waits for the
//                 older store's smem reads before committing).
// afull(it) also tells the control warp that every warp passed its wait for
// MMA(it-LAG), so that tile's ring slot may be refilled.
template <int DP, bool LAST, typename OutT, bool CSR = false>
__global__ void __launch_bounds__(SellCfg<DP>::NT, SellCfg<DP>::CPS)
k_layer_sell(DevCsr a, const __grid_constant__ SellMaps maps, const float* __restrict__ X,
             const float* __restrict__ axlong, const float* __restrict__ uwp, NetView net,
             const ApplyScalars* __restrict__ sc, OutT* __restrict__ out, const int* __restrict__ skip) {
  using C = SellCfg<DP, CSR>;
  constexpr int TM = C::TM, G = C::G, R = C::R, NS = C::NS, NW = C::NW, NQ = C::NQ, LAG = C::LAG;
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
  uint8_t* Abuf = base + C::O_A;  // [LAG][A1_lo | A2_hi | A2_lo]
  uint8_t* Bs = base + C::O_B;
  uint8_t* Ystg = base + C::O_Y;
  float* D1 = reinterpret_cast<float*>(base + C::O_P);
  const int H = net.hidden;
  float* B1 = D1 + DP * H;
  float* D2 = B1 + H;
  uint64_t* full = reinterpret_cast<uint64_t*>(
      base + ((C::O_P + (LAST ? (DP + 2) * H * 4 : 0) + 15) & ~15u));
  uint64_t* mma_bar = full + NS;  // [LAG]
  uint64_t* afull = mma_bar + LAG;  // [LAG]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(afull + LAG);

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
    for (int b = 0; b < LAG; ++b) {
      tc::mbar_init(&mma_bar[b], 1);
      tc::mbar_init(&afull[b], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tc::tmem_alloc(tslot, C::TALLOC);
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;
  // local iterations: one per tile of this CTA, plus LAG drain iterations
  const int my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int iters = my_tiles > 0 ? my_tiles + LAG : 0;

  if (warp == NW) {
    // ============================================================ control warp
    if (lane == 0) {
      tc::tma_prefetch_desc(&maps.x);
      if (!LAST) tc::tma_prefetch_desc(&maps.y);
      auto issue = [&](int it) {
        if (it >= my_tiles) return;
        const int t = blockIdx.x + it * gridDim.x;
        const int s = it % NS;
        uint8_t* slot = ring + s * C::SLOT;
        if constexpr (CSR) {
          // the tile's short-row CSR range, 16-byte aligned superset [a0, a1)
          const int kb = __ldg(a.rps + t * TM), ke = __ldg(a.rps + min((t + 1) * TM, n));
          const int a0 = kb & ~3, cnt = ((ke + 3) & ~3) - a0;
          const bool staged = cnt <= C::CAPC;
          tc::mbar_expect_tx(&full[s], C::OPB + C::RPB + (staged ? 8 * cnt : 0));
          tc::tma_load_2d(slot, &maps.x, 0, t * TM, &full[s]);
          tc::bulk_load(slot + C::O_RP, a.rps + t * TM, C::RPB, &full[s]);
          if (staged && cnt > 0) {
            tc::bulk_load(slot + C::O_CI, a.cis + a0, 4 * cnt, &full[s]);
            tc::bulk_load(slot + C::O_V, a.vs + a0, 4 * cnt, &full[s]);
          }
        } else {
          const int K = __ldg(a.sell_k + t) & 0xffff;
          const bool staged = K > 0 && K <= C::KCAP;
          tc::mbar_expect_tx(&full[s], C::OPB + (staged ? K * TM * 8 : 0));
          tc::tma_load_2d(slot, &maps.x, 0, t * TM, &full[s]);
          if (staged) tc::bulk_load(slot + C::OPB, a.sell + __ldg(a.sell_off + t), K * TM * 8, &full[s]);
        }
      };
      for (int it = 0; it < NS - LAG; ++it) issue(it);
      constexpr uint32_t idesc = tc::idesc_tf32(128, DP);
      constexpr uint32_t idesc2 = tc::idesc_tf32(128, 2 * DP);
      const uint32_t sBstk = tc::smem_u32(Bs);
      for (int it = 0; it < iters; ++it) {
        tc::mbar_wait_dbg(&afull[it % LAG], (it / LAG) & 1, 1, it);
        tc::fence_after();
        // stores issued up to iteration it-1 have left the Y staging: the
        // buffer the epilogue after this MMA writes ((it) % NY) is free
        tc::bulk_wait_read0();
        if (it < my_tiles) {
          const int b = it % LAG;
          const uint32_t sA = tc::smem_u32(Abuf + b * 3 * C::OPB);
          const uint32_t sA1lo = sA, sA2hi = sA + C::OPB, sA2lo = sA + 2 * C::OPB;
          const uint32_t sX = tc::smem_u32(ring + (it % NS) * C::SLOT);
          const uint32_t acc = tmem + b * C::TCOLS;
          // 3xTF32 with the two A_hi products stacked along N (A_hi is read
          // once for both): D[:, 0:DP] = A_hi·B_lo, D[:, DP:2DP] = A_hi·B_hi +
          // A_lo·B_hi; the epilogue adds the halves.  Each part's B operands
          // are stored [B_lo | B_hi], i.e. as one 2DP-row operand.
          uint32_t accf = 0;
#pragma unroll
          for (int part = 0; part < 2; ++part) {
            const uint32_t sah = part == 0 ? sX : sA2hi, sal = part == 0 ? sA1lo : sA2lo;
            const uint32_t sbs = sBstk + part * 2 * C::BB;  // [B_lo; B_hi] of this part (2DP rows)
            const uint32_t sbh = sbs + C::BB;                // B_hi rows alone
#pragma unroll
            for (int k8 = 0; k8 < DP / 8; ++k8) {
              tc::mma_tf32(acc, tc::make_desc_swz<DP>(sah + k8 * 32), tc::make_desc_swz<DP>(sbs + k8 * 32),
                           idesc2, accf);
              accf = 1;
              tc::mma_tf32(acc + DP, tc::make_desc_swz<DP>(sal + k8 * 32),
                           tc::make_desc_swz<DP>(sbh + k8 * 32), idesc, 1);
            }
          }
          tc::mma_commit(&mma_bar[b]);
        }
        if (!LAST && it >= LAG) {  // tile it-LAG is fully staged
          tc::tma_store_2d(&maps.y, Ystg + ((it - LAG) % C::NY) * C::OPB, 0,
                           (blockIdx.x + (it - LAG) * gridDim.x) * TM);
          tc::bulk_commit();
        }
        // every warp passed its wait for MMA(it-LAG): that slot takes tile it+NS-LAG
        issue(it + NS - LAG);
      }
      tc::bulk_wait0();
    }
    __syncwarp();
  } else {
    // ============================================================== math warps
    const int gl = tid % G, gid = tid / G;
    // epilogue of tile itp (accumulator in TMEM buffer itp % LAG).
    // Non-last layers: relu'd rows -> Ystg[itp % NY] (warp w: lanes 32(w%4)..,
    // column group w/4), stored by the control warp's TMA.  Last layer: the
    // projection group of this tile (warps 4*(itp%NQ)..+3, one per lane
    // quarter) pulls whole rows into registers `y` and projects them after
    // arriving — the groups rotate, so no CTA-wide barrier is needed.
    float y[LAST ? DP : 1];
    auto epilogue = [&](int itp) -> bool {
      const int b = itp % LAG;
      tc::mbar_wait_dbg(&mma_bar[b], (itp / LAG) & 1, 2, itp);
      tc::fence_after();
      const int q = warp & 3, cq = warp >> 2;  // lane quarter, column group
      const uint32_t trow = tmem + b * C::TCOLS + (static_cast<uint32_t>(32 * q) << 16);
      if constexpr (LAST) {
        if (cq != itp % NQ) return false;
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
        constexpr int CW = DP / NQ;  // columns per warp: 4, 8 or 16
        uint8_t* ys = Ystg + (itp % C::NY) * C::OPB;
        const uint32_t taddr = trow + cq * CW;
        float v[CW];
        if constexpr (CW == 4) {
          float v2[4];
          tc::tmem_ld4(taddr, v);
          tc::tmem_ld4(taddr + DP, v2);
#pragma unroll
          for (int c = 0; c < 4; ++c) v[c] += v2[c];
        } else {
#pragma unroll
          for (int c0 = 0; c0 < CW; c0 += 8) {
            float u1[8], u2[8];
            tc::tmem_ld8(taddr + c0, u1);
            tc::tmem_ld8(taddr + DP + c0, u2);
#pragma unroll
            for (int c = 0; c < 8; ++c) v[c0 + c] = u1[c] + u2[c];
          }
        }
#pragma unroll
        for (int c = 0; c < CW; c += 4)
          *reinterpret_cast<float4*>(ys + tc::swz_off<DP>(m, cq * CW + c)) =
              make_float4(relu(v[c]), relu(v[c + 1]), relu(v[c + 2]), relu(v[c + 3]));
        tc::fence_before();
        return false;
      }
    };
    auto arrive = [&](int it) {
      tc::fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&afull[it % LAG]);
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

    const int* tinfo = CSR ? a.tflag : a.sell_k;  // per tile: K_t | has-long << 16 (SELL), has-long (CSR)
    int kw = my_tiles > 0 ? __ldg(tinfo + blockIdx.x) : 0;
    for (int it = 0; it < iters; ++it) {
      const bool have = it < my_tiles;
      const int tile = blockIdx.x + it * gridDim.x;
      const int row0 = tile * TM;
      const int s = it % NS;
      uint8_t* slot = ring + s * C::SLOT;
      float4 acc[R];
      if (have) {
        const int K = CSR ? 0 : (kw & 0xffff);
        const bool haslong = CSR ? kw != 0 : (kw >> 16) != 0;
        const bool staged = K > 0 && K <= C::KCAP;
        kw = it + 1 < my_tiles ? __ldg(tinfo + tile + gridDim.x) : 0;  // prefetch

        // --------------------------------------------------------- gather
#pragma unroll
        for (int j = 0; j < R; ++j) {
          const int i = row0 + R * gid + j;
          acc[j] = f4zero();
          if (haslong && i < n && __ldg(a.rp + i + 1) - __ldg(a.rp + i) > kLongRow)
            acc[j] = ldg4(axlong + static_cast<size_t>(i) * DP + 4 * gl);
        }
        tc::mbar_wait_dbg(&full[s], (it / NS) & 1, 3, it);
        if constexpr (CSR) {
          const int* rpt = reinterpret_cast<const int*>(slot + C::O_RP);
          const int kb = rpt[0], ke = rpt[min(TM, n - row0)];
          const int a0 = kb & ~3;
          const bool st = ((ke + 3) & ~3) - a0 <= C::CAPC;
          int sj[R], lj[R], self[R];
#pragma unroll
          for (int j = 0; j < R; ++j) {
            const int r = R * gid + j;
            const int e0 = rpt[r], e1 = rpt[r + 1];
            sj[j] = st ? e0 - a0 : e0;
            lj[j] = row0 + r < n ? e1 - e0 : 0;
            self[j] = min(row0 + r, n - 1);
          }
          if (st)
            gather_csr_rows<DP, R, C::USC>(X, gl, reinterpret_cast<const int*>(slot + C::O_CI),
                                           reinterpret_cast<const float*>(slot + C::O_V), sj, lj, self, acc);
          else
            gather_csr_rows<DP, R, C::USC>(X, gl, a.cis, a.vs, sj, lj, self, acc);
        } else {
          if (staged)
            gather_sell_rows<DP, R, C::US, TM, true>(X, gl, reinterpret_cast<const int2*>(slot + C::OPB), K,
                                                     gid, acc);
          else
            gather_sell_rows<DP, R, C::US, TM, false>(X, gl, a.sell + __ldg(a.sell_off + tile), K, gid, acc);
        }
      }

      // ------------------------------------- epilogue of tile it - LAG
      const bool proj = it >= LAG && epilogue(it - LAG);

      // -------------------------------------------------------------- split
      if (have) {
        uint8_t* A = Abuf + (it % LAG) * 3 * C::OPB;
#pragma unroll
        for (int j = 0; j < R; ++j) {
          const int r = R * gid + j;
          const uint32_t o = tc::swz_off<DP>(r, 4 * gl);
          const float4 xv = *reinterpret_cast<const float4*>(slot + o);
          *reinterpret_cast<float4*>(A + o) = f4_trunc_lo(xv);
          *reinterpret_cast<float4*>(A + C::OPB + o) = acc[j];
          *reinterpret_cast<float4*>(A + 2 * C::OPB + o) = f4_trunc_lo(acc[j]);
        }
      }
      arrive(it);
      if (proj) project((blockIdx.x + (it - LAG) * gridDim.x) * TM);
    }
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 0) tc::tmem_dealloc(tmem, C::TALLOC);
}

}  // namespace gnpk
