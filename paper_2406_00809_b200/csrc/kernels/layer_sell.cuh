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

__device__ __forceinline__ void tmem_ld4x2(uint32_t ta, uint32_t tb, float (&u)[4], float (&v)[4]) {
  uint32_t r[4], q[4];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(ta));
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3])
               : "r"(tb));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    u[i] = __uint_as_float(r[i]);
    v[i] = __uint_as_float(q[i]);
  }
}

// 2-D tile store smem -> global (bulk-group completion), under an L2 policy
__device__ __forceinline__ void tma_store_2d_hint(const void* tmap, const void* src, int x, int y, uint64_t pol) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3}], [%1], %4;" ::"l"(
                   tmap),
               "r"(smem_u32(src)), "r"(x), "r"(y), "l"(pol)
               : "memory");
}
// 2-D tile store smem -> global (bulk-group completion).
__device__ __forceinline__ void tma_store_2d(const void* tmap, const void* src, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(tmap),
               "r"(smem_u32(src)), "r"(x), "r"(y)
               : "memory");
}
// 1-D bulk copy shared -> global (bulk-group completion; 16-B aligned, size % 16 == 0).
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
// 128-bit shared-memory load by 32-bit shared address
__device__ __forceinline__ float4 lds4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

}  // namespace tc

// CSR = 0: sliced-ELL slices (k_layer_sell on regular matrices; CSR = 4:
//          the same with a deeper ring for d = 32 non-last layers);
// CSR = 1: the short-row CSR ranges of the tile (ragged matrices);
// CSR = 2: training — B virtual rows per node (v = node*B + k), the full CSR
//          ranges of the tile's 128/B nodes, plus a mask tile for the backward;
// CSR = 7 / 8 / 9: strip windows (DevCsr::pw, d = 32): 7 the non-last layers,
//          8 the last layer, 9 the FIRST layer with the lift fused in — its
//          windows are not loaded but computed from the scaled input by two
//          lift warps (x1 = lift_a[p] v + lift_b[p], src/gnn.cpp:138-157), so
//          the first activation never crosses HBM;
// CSR = 10: training over strip windows (DevCsr::tw, d = 32): CSR 2's virtual
//          rows with the X rows of the tile's neighbour nodes staged in shared
//          memory by TMA (node windows along strips, one new per tile).
template <int DP, int CSR = 0>
struct SellCfg {
  // one CTA per SM: 16 math warps on one tile at a time (two 8-warp CTAs per
  // SM measured slower at DP=16: C2 26.0 vs 24.4 us, C4 213 vs 160 us)
  static constexpr int NW = 16;                  // math warps (gather / epilogue / split)
  static constexpr int CPS = 1;                  // CTAs per SM
  // + one control warp (MMA, TMA, stores); the strip-window modes add a TMA
  // producer warp, so the MMA issue is not serialised behind the loads
#ifndef GNPC_TR_PROD
#define GNPC_TR_PROD 0  // measured neutral on C3 (19.34 ms either way)
#endif
  static constexpr int NPROD = (CSR == 7 || CSR == 8 || CSR == 9 || CSR == 10 || (CSR == 2 && GNPC_TR_PROD)) ? 1 : 0;
  // CSR = 9: + lift warps filling the strip windows from the layer-0 input
  static constexpr bool LIFT = CSR == 9;
  static constexpr int NLIFT = LIFT ? 5 : 0;
  // strip-window modes: the MMA work that does not need tile t's split —
  // X_hi·[U_lo; U_hi] and the projection of tile t-1 — is issued as soon as
  // the epilogues have read TMEM (efull), overlapping the split
#ifndef GNPC_PW_EARLY
#define GNPC_PW_EARLY 1
#endif
#ifndef GNPC_TR_EARLY
#define GNPC_TR_EARLY 0
#endif
#ifndef GNPC_TW_EARLY
#define GNPC_TW_EARLY 1  // C3 18.18 -> 18.02 ms
#endif
  // (measured neutral to slower on the d = 16 sliced-ELL / CSR layers: C2
  // 4820 vs 4980 applies/s, C4 unchanged, so those keep the plain order)
  static constexpr bool EARLY = ((CSR == 7 || CSR == 8 || CSR == 9) && GNPC_PW_EARLY) || (CSR == 2 && GNPC_TR_EARLY) ||
                                (CSR == 10 && GNPC_TW_EARLY);
  static constexpr int NT = 32 * (NW + 1 + NPROD + NLIFT);
  static constexpr int NQ = NW / 4;              // epilogue column groups (warps per TMEM lane quarter)
  static constexpr int TM = 128;                 // rows per tile (MMA M)
  static constexpr int G = DP / 4;               // lanes per row
  static constexpr int NG = 32 * NW / G;         // row groups
  static constexpr int R = TM / NG;              // rows per group
#ifndef GNPC_US32
#define GNPC_US32 3
#endif
#ifndef GNPC_KCAP32
#define GNPC_KCAP32 9  // staged slice words per row at d = 32 (a 9-point row; 12 left less L1: C5 283 vs 287 applies/s)
#endif
#ifndef GNPC_USP
#define GNPC_USP 6  // pair-union entries per gather round
#endif
#ifndef GNPC_KCAPP
#define GNPC_KCAPP 12  // staged pair-union entries per pair (a 9-point pair's union)
#endif
#ifndef GNPC_KCAPPW
#define GNPC_KCAPPW 12  // strip-window entries per pair (multiple of 4; every tile is staged; 16 overflows the last layer's smem)
#endif
  static constexpr int US = DP == 16 ? 8 : ((CSR == 5 || CSR == 6) ? GNPC_USP : GNPC_US32);  // entries per gather round
#ifndef GNPC_USC_TR
#define GNPC_USC_TR 5
#endif
  // CSR entries per gather round (training: B virtual rows share one list)
  static constexpr int USC = CSR == 2 ? GNPC_USC_TR : (DP == 16 ? 8 : 4);
  // TMA ring depth (tiles), measured per format: SELL DP16 (C2) best at 4
  // (an epilogue lag of 2 tiles with double-buffered A/TMEM and NS 5 measured
  // 25.7 vs 24.4 us); CSR DP16 (C4) at 5 (166 vs 197 us at 4); DP32 fills smem
  static constexpr bool CSRL = CSR == 1 || CSR == 2;    // CSR ranges staged per tile
#ifndef GNPC_MBITS
#define GNPC_MBITS 1  // per-row mask words instead of the X_l tile: frees 15.5 KB per ring slot
#endif
#ifndef GNPC_NS_TR32
#define GNPC_NS_TR32 (GNPC_MBITS ? 5 : 4)  // C3: 3 -> 4 (22.0 -> 20.3 ms), mask words + 5 (-> 19.3 ms)
#endif
  // CSR = 4: sliced-ELL at d = 32 with a 4-deep ring, for the non-last
  // layers (the last layer's projection operands need the smem of a slot)
  static constexpr bool DEEP = CSR == 4;
  static_assert(!DEEP || DP == 32, "the deep-ring sliced-ELL mode is a d = 32 layout");
#ifndef GNPC_NS_DEEP32
#define GNPC_NS_DEEP32 4
#endif
#ifndef GNPC_NS_CSR16
#define GNPC_NS_CSR16 5
#endif
#ifndef GNPC_NS_SELL16
#define GNPC_NS_SELL16 4
#endif
  // CSR = 5 / 6: pair-union sliced-ELL (d = 32): the 4-deep ring for the
  // non-last layers (5), 3 deep for the last (6)
  static constexpr bool PAIR = CSR == 5 || CSR == 6;
  static_assert(!PAIR || DP == 32, "pair-union slices are a d = 32 layout (two rows per 8-lane group)");
  // CSR = 7 / 8: strip-window pair-union (d = 32, DevCsr::pw): the ring holds
  // only the slices; X rows come from NWIN row windows (one new per tile in a
  // strip); 7 = non-last layers (4-deep ring), 8 = last layer (3 deep)
  static constexpr bool PW = CSR == 7 || CSR == 8 || CSR == 9;
  static_assert(!PW || DP == 32, "strip windows are a d = 32 layout");
  static constexpr bool TW = CSR == 10;       // training strip windows
  static_assert(!TW || DP == 32, "training strip windows are a d = 32 layout");
  static constexpr bool WINS = PW || TW;      // the window ring + producer machinery
#ifndef GNPC_NS_PW
#define GNPC_NS_PW 4  // 3 measured slower (C5 409 vs 368 us)
#endif
  static constexpr int NS = DP == 16 ? (CSRL ? GNPC_NS_CSR16 : GNPC_NS_SELL16)
                                     : (CSR == 2 ? GNPC_NS_TR32
                                                 : ((DEEP || CSR == 5) ? GNPC_NS_DEEP32
                                                                       : ((PW || CSR == 10) ? GNPC_NS_PW : 3)));
  // windows alive: the MMA's window of the current tile plus NS - 1 tiles
  // of lookahead (steady state: one new window per tile); a break tile
  // issued right after its predecessor's gathers needs the MMA window b,
  // the predecessor's c and three fresh seqs: c - b = 4 < NWIN
  static constexpr int NWIN = WINS ? (NS + 1 > 5 ? NS + 1 : 5) : 0;
  // window slot: PW 144 rows (8-row halos), TW up to 128 + 2 bs rows (bs <= 32)
  static constexpr uint32_t WINB = (TW ? kTwRowsMax : kPwRows) * DP * 4;
  // slices with K <= KCAP are staged; a multiple of US (the last round reads
  // up to round(K, US) words).  Kept small: every KB of shared memory is L1
  // the X-row gathers hit (C5 fused layer 531 -> 499 us going 24 -> 12)
#ifndef GNPC_KCAP16
#define GNPC_KCAP16 16
#endif
  // (pair-union: entries per pair; a union entry is 16 B for 2 rows, so the
  // staged bytes K * TM * 8 match the sliced-ELL formula)
  static constexpr int KCAP = DP == 16 ? GNPC_KCAP16
                                       : ((CSR == 5 || CSR == 6) ? GNPC_KCAPP
                                                                 : (PW ? GNPC_KCAPPW : GNPC_KCAP32));
  // the staged gather reads round(K, US) words of a slice: KCAP must be a
  // multiple of US or the last round would read past the staged slice
  static_assert(PW || KCAP % US == 0, "GNPC_KCAP16/GNPC_KCAP32 must be a multiple of the gather round");
  static_assert(!PW || KCAP % 4 == 0, "strip-window slices hold a multiple of 4 entries per pair");
  static constexpr uint32_t OPB = TM * DP * 4;   // one A-type operand / X tile / Y tile (bytes)
  static constexpr uint32_t BB = DP * DP * 4;    // one B operand (bytes)
  static constexpr int TCOLS = 2 * DP;           // TMEM accumulator columns (two halves)
  // + the X·U part's A_lo operand (DP columns, A in TMEM) at alo_col
  static constexpr int TALLOC = 4 * DP;          // power of two >= 3 DP
  static constexpr uint32_t CVB = PW ? KCAP * (TM / 2) * 10 : KCAP * TM * 8;  // staged slice (bytes)
  // CSR: [X tile | row_ptr slice (TM+4 ints, 1 KiB) | col_idx (CAPC) | values (CAPC)]
  static constexpr bool TR = CSR == 2 || CSR == 10;  // training (virtual rows, masks, ÂX out)
#ifndef GNPC_CAPC16
#define GNPC_CAPC16 2048
#endif
#ifndef GNPC_CAPC_TR
#define GNPC_CAPC_TR 256  // C3 tiles stage ~20 entries (4 nodes); 512 measured 0.4 % slower (less L1)
#endif
  static constexpr int CAPC = TR ? GNPC_CAPC_TR : (DP == 16 ? GNPC_CAPC16 : 1024);  // staged nonzeros per tile (DP=32
                                                                     // apply: fits the projection operands)
  static constexpr uint32_t RPB = (TM + 4) * 4;  // row_ptr slice copy (bytes, 16-B multiple)
  // training backward mask [X_l > 0]: at d = 32 one 32-bit word per row
  // (written by the forward layer's epilogue), else the X_l tile itself
  static constexpr bool MBITS = GNPC_MBITS && TR && DP == 32;
  static constexpr uint32_t MASKB = MBITS ? TM * 4 : OPB;
  // TW slot: [mask words | window slice]; the X rows live in the windows
  static constexpr uint32_t O_MASK = TW ? 0 : OPB;
  static constexpr uint32_t O_TWS = MASKB;
  static constexpr uint32_t O_RP = TR ? OPB + MASKB : OPB, O_CI = O_RP + 1024, O_V = O_CI + CAPC * 4;
  static constexpr uint32_t O_SL = PW ? 0 : OPB;  // staged slice (sliced-ELL modes)
  static constexpr uint32_t SLOT =
      TW ? 1024u : (CSRL ? ((O_V + CAPC * 4 + 1023) & ~1023u) : (((O_SL + CVB) + 1023) & ~1023u));
  static_assert(!TW || O_TWS + 2 * 40 + 6 * kTwKcap <= SLOT, "training window slice exceeds its ring slot");
  // layout (offsets from the 1024-aligned base)
  static constexpr uint32_t O_RING = 0;
  static constexpr uint32_t O_WIN = O_RING + NS * SLOT;   // strip windows [NWIN] (PW)
  static constexpr uint32_t O_A = O_WIN + NWIN * WINB;    // A2_hi (ÂX), A2_lo
  static constexpr uint32_t O_B = O_A + 2 * OPB;          // Bu_lo, Bu_hi, Bw_lo, Bw_hi
  static constexpr uint32_t O_Y = O_B + 4 * BB;           // Y staging [2]
  // last layer only: the dec1 B operand [D1_lo; D1_hi] (2H rows, swizzled
  // K-major, TCP), then dec1 (fp32, CUDA-core projection), b1, dec2
  // training forward at d = 32: the rows' [Y > 0] words staged [2][TM] next
  // to the Y staging, stored with it by one bulk copy
  static constexpr uint32_t O_MST = O_Y + 2 * OPB;
  static constexpr uint32_t o_p(int hidden, bool last) {
    // last layer with the tensor-core projection: no Y staging (the
    // projection operand lives in TMEM), the dec1 operand [D1_lo; D1_hi] sits
    // at O_Y, then dec1/b1/dec2.  Otherwise the Y staging stays (the fused
    // apply's earlier layers use it with the last layer's layout).
    return last && tc_proj(hidden) ? O_Y + 2 * hidden * DP * 4 : O_Y + 2 * OPB + (MBITS ? 2 * TM * 4 : 0);
  }
  static constexpr uint32_t o_bar(int hidden, bool last) {
    // last: dec1 (DP x H), b1, dec2, then the projection partials [2][NQ][TM]
    return (o_p(hidden, last) + (last ? (DP + 2) * hidden * 4 + 2 * NQ * TM * 4 : 0) + 15) & ~15u;
  }
  // PW: per-CTA schedule table (tile, K, slice offset) after the barriers
  static constexpr int KSCHED = PW ? 256 : (TW ? 512 : 0);
  // CSR = 9: the lift tables [kLiftIv][DP] a, b and the kinks (hidden <= 32)
  static constexpr int kLiftIv = 33;
  static constexpr uint32_t LIFTB = LIFT ? 2 * kLiftIv * DP * 4 + 32 * 4 : 0;
  static size_t smem_bytes(int hidden, bool last) {
    // barriers + TMEM slot, the schedule, the lift tables, 1024-B alignment slack
    return o_bar(hidden, last) + 128 + 3 * KSCHED * 4 + LIFTB + 1024;
  }
  static_assert(TR || DEEP || CSR == 5 || CSR == 7 || CSR == 9 || O_Y + 2 * 32 * DP * 4 + (DP + 2) * 32 * 4 + 128 + 1024 <= 227 * 1024,
                "last-layer layout must fit shared memory at hidden 32 (larger: host falls back)");
  static_assert(!TR || O_Y + 2 * OPB + 128 + 1024 <= 227 * 1024, "training layout must fit shared memory");
  // TMEM: layer accumulator [0, 2DP); last layer's projection accumulator at
  // [2DP, 2DP + 2H) (tensor-core projection when H % 16 == 0 and H <= 64)
  // last layer (tensor-core projection): Y_hi / Y_lo of two tiles in TMEM at
  // ycol(buf) = 256 + 2 DP buf, so the allocation is the whole 512 columns
  // (one CTA per SM)
  static constexpr int TALLOC_LAST = 512;
  static __host__ __device__ constexpr uint32_t ycol(int buf) { return 256 + 2 * DP * buf; }
  // TMEM column of X_lo, the A operand of X·U's A_lo·B_hi product: written
  // row-per-lane by the math warps (tcgen05.st), read by the TS-form MMA, so
  // it never crosses shared memory.  (ÂX_lo stays in shared memory: moving it
  // too needs the quarter's four warps to sync before the row-wise read, and
  // that coupling cost more than the wavefronts it saved — C4 162 -> 240 us.)
  static __host__ __device__ constexpr int alo_col(bool tcp) { return tcp ? 2 * DP + 128 : 2 * DP; }
  // DP=16: the CUDA-core projection is cheap (DP*H FMAs per row) and the
  // staging it saves is L1 for the gathers (fused C2: 27.3 vs 26.5 us LAST,
  // 18 vs 17 us per layer with the larger layout)
  // (re-measured in round 2 with the TMEM-resident projection operand, which
  // needs no staging: C2 4,809 vs 4,953 applies/s, C4 last layer 145 vs 140 us)
  static __host__ __device__ constexpr bool tc_proj(int hidden) {
    return DP == 32 && hidden % 16 == 0 && hidden <= 64;
  }
};

// the strip-window layouts fit one SM's shared memory (hidden 32)
static_assert(SellCfg<32, 7>::o_bar(32, false) + 128 + 3 * SellCfg<32, 7>::KSCHED * 4 + 1024 <= 227 * 1024,
              "strip-window layer layout exceeds shared memory");
static_assert(SellCfg<32, 9>::o_bar(32, false) + 128 + 3 * SellCfg<32, 9>::KSCHED * 4 + SellCfg<32, 9>::LIFTB + 1024 <=
                  227 * 1024,
              "fused-lift first-layer layout exceeds shared memory");
static_assert(SellCfg<32, 8>::o_bar(32, true) + 128 + 3 * SellCfg<32, 8>::KSCHED * 4 + 1024 <= 227 * 1024,
              "strip-window last-layer layout exceeds shared memory");

struct SellMaps {
  CUtensorMap x;   // layer input  [n][DP], box {DP, 128}, swizzled
  CUtensorMap y;   // layer output [n][DP] (unused by the last layer)
  CUtensorMap xw;  // layer input, box {DP, kPwRows} (strip windows, d = 32)
};

// Sliced-ELL gather, R rows per group, rounds of US entries.  Slots past K
// read an in-bounds stale slice word (the ring is zeroed at start) and are
// given weight 0 and the round's first column, so no load is predicated.
template <int DP, int R, int US, int TM, bool SMEM>
__device__ __forceinline__ void gather_sell_rows(const float* __restrict__ X, int gl, const int2* cv,
                                                 int K, int gid, float4 (&acc)[R], uint64_t pol) {
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
        x[j][u] = ldg4_hint(reinterpret_cast<const float*>(
            xb + static_cast<unsigned long long>(static_cast<unsigned>(c[j][u])) * (DP * 4ull)), pol);
#pragma unroll
    for (int u = 0; u < US; ++u)
#pragma unroll
      for (int j = 0; j < R; ++j) fma4(acc[j], w[j][u], x[j][u]);
  }
}

// Pair-union gather (CSR = 5/6): the group's two adjacent rows share one
// entry list; each entry's X row is loaded once and feeds both rows' sums
// (weight 0 where a row lacks the column, which adds exactly 0 and keeps each
// row's own terms in stored order).  Slots past K: weight 0, the round's
// first column.
template <int DP, int US, int NG, bool SMEM>
__device__ __forceinline__ void gather_pair_rows(const float* __restrict__ X, int gl, const int4* cv, int K,
                                                 int gid, float4 (&acc)[2], uint64_t pol) {
  const char* xb = reinterpret_cast<const char*>(X + 4 * gl);
  for (int k = 0; k < K; k += US) {
    int c[US];
    float w0[US], w1[US];
#pragma unroll
    for (int u = 0; u < US; ++u) {
      const bool on = k + u < K;
      const int4* src = cv + (k + u) * NG + gid;
      int4 e;
      if constexpr (SMEM) {
        e = *src;
      } else {
        e = on ? __ldg(src) : make_int4(0, 0, 0, 0);
      }
      c[u] = (u == 0 || on) ? e.x : c[0];
      w0[u] = on ? __int_as_float(e.y) : 0.f;
      w1[u] = on ? __int_as_float(e.z) : 0.f;
    }
    float4 x[US];
#pragma unroll
    for (int u = 0; u < US; ++u)
      x[u] = ldg4_hint(reinterpret_cast<const float*>(
                           xb + static_cast<unsigned long long>(static_cast<unsigned>(c[u])) * (DP * 4ull)),
                       pol);
#pragma unroll
    for (int u = 0; u < US; ++u) {
      fma4(acc[0], w0[u], x[u]);
      fma4(acc[1], w1[u], x[u]);
    }
  }
}

// Strip-window gather (CSR = 7/8): the tile's slice holds, per row pair,
// K entries {idx, w0, w1} as structure-of-arrays.  idx is the byte offset of
// the X row in the tile's three consecutive windows (a, b, c) laid end to end
// — R = 144 w + row, idx = 128 R + 16 (R & 7), i.e. with the SWIZZLE_128B
// chunk bits of lane group 0 — so lane gl reads (wbase + idx) ^ (gl << 4),
// wrapped once around the NWIN-window ring.  Padding entries carry weight 0.
// WRAP = false: the tile's three windows sit in consecutive ring slots
// without wrapping (3 tiles of NWIN = 5), so the per-entry wrap test is dropped.
template <int NG, bool WRAP>
__device__ __forceinline__ void gather_pw_rows(const uint8_t* sl, int K, int gid, int gl, uint32_t wbase,
                                               uint32_t wlim, uint32_t wring, float4 (&acc)[2]) {
  const uint16_t* idx = reinterpret_cast<const uint16_t*>(sl) + gid * K;
  const float* w0 = reinterpret_cast<const float*>(sl + NG * K * 2) + gid * K;
  const float* w1 = w0 + NG * K;
  const uint32_t gx = static_cast<uint32_t>(gl) << 4;
  for (int k = 0; k < K; k += 4) {
    const uint2 rr = *reinterpret_cast<const uint2*>(idx + k);
    const float4 a0 = *reinterpret_cast<const float4*>(w0 + k);
    const float4 a1 = *reinterpret_cast<const float4*>(w1 + k);
    const uint32_t e[4] = {rr.x & 0xffffu, rr.x >> 16, rr.y & 0xffffu, rr.y >> 16};
    float4 x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      uint32_t v = wbase + e[u];
      if constexpr (WRAP) v = v >= wlim ? v - wring : v;
      x[u] = tc::lds4(v ^ gx);
    }
    fma4(acc[0], a0.x, x[0]);
    fma4(acc[1], a1.x, x[0]);
    fma4(acc[0], a0.y, x[1]);
    fma4(acc[1], a1.y, x[1]);
    fma4(acc[0], a0.z, x[2]);
    fma4(acc[1], a1.z, x[2]);
    fma4(acc[0], a0.w, x[3]);
    fma4(acc[1], a1.w, x[3]);
  }
}

// CSR gather: row r = R*gid + j of the tile spans [s_j, s_j + len_j) of the
// staged (or global) col/val arrays; rounds of US entries up to the longer
// of the group's rows.  Slots past a row's end get weight 0 and the row's own
// X row (in bounds, usually cached), so no load is predicated.
template <int DP, int R, int US>
__device__ __forceinline__ void gather_csr_rows(const char* const (&xbj)[R], unsigned long long stride,
                                                const int* ci, const float* vv, const int (&s)[R],
                                                const int (&len)[R], const int (&self)[R], float4 (&acc)[R],
                                                uint64_t pol) {
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
      for (int j = 0; j < R; ++j) {
        const float* src = reinterpret_cast<const float*>(
            xbj[j] + static_cast<unsigned long long>(static_cast<unsigned>(c[j][u])) * stride);
        // (padding slots re-read the row's own X row: predicating them off
        // measured slower, C4 197 vs 158 us per layer)
        x[j][u] = ldg4_hint(src, pol);
      }
#pragma unroll
    for (int u = 0; u < US; ++u)
#pragma unroll
      for (int j = 0; j < R; ++j) fma4(acc[j], w[j][u], x[j][u]);
  }
}

// Training gather when a group's R rows are consecutive samples of ONE node
// (bs % R == 0): the node's (col, val) list is read once per entry for all R
// rows, and row j's X row is row 0's plus j rows (j * DP floats).
template <int DP, int R, int US>
__device__ __forceinline__ void gather_csr_node(const char* xb0, unsigned long long stride, const int* ci,
                                                const float* vv, int s, int len, int self,
                                                float4 (&acc)[R]) {
  for (int k = 0; k < len; k += US) {
    int c[US];
    float w[US];
#pragma unroll
    for (int u = 0; u < US; ++u) {
      const bool on = k + u < len;
      c[u] = on ? ci[s + k + u] : self;
      w[u] = on ? vv[s + k + u] : 0.f;
    }
    float4 x[R][US];
#pragma unroll
    for (int u = 0; u < US; ++u) {
      const char* base = xb0 + static_cast<unsigned long long>(static_cast<unsigned>(c[u])) * stride;
#pragma unroll
      for (int j = 0; j < R; ++j) x[j][u] = ldg4(reinterpret_cast<const float*>(base + j * DP * 4));
    }
#pragma unroll
    for (int u = 0; u < US; ++u)
#pragma unroll
      for (int j = 0; j < R; ++j) fma4(acc[j], w[u], x[j][u]);
  }
}

// Training extras for sell_layer (CSR = 2): B virtual rows per node; KIND 1
// (forward) also stores the tile's ÂX (= the A2_hi operand, raw fp32) through
// mapax, and at d = 32 the rows' [Y > 0] bits (mask_out, one 32-bit word per
// row); KIND 2 (backward) multiplies by [X_l > 0] when use_mask, from those
// bits (mask_in, d = 32) or from the X_l tile (mapmask).
// Fused-lift extras (CSR = 9): the apply's input vector (f32 or f64) and the
// scale sandwich's scalars.
struct LiftIO {
  const void* in;
  int f64;
  const ApplyScalars* sc;
};

struct TrainIO {
  const CUtensorMap* mapax;
  const CUtensorMap* mapmask;
  int bs;
  int use_mask;
  const uint32_t* mask_in;
  uint8_t* mask_out;
  int no_ax;  // KIND 1: skip the ÂX store (forward-only passes: the monitoring batch)
};

__device__ __forceinline__ float4 f4_trunc_lo(float4 v) {
  return make_float4(v.x - __int_as_float(__float_as_int(v.x) & 0xffffe000),
                     v.y - __int_as_float(__float_as_int(v.y) & 0xffffe000),
                     v.z - __int_as_float(__float_as_int(v.z) & 0xffffe000),
                     v.w - __int_as_float(__float_as_int(v.w) & 0xffffe000));
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(bar)) : "memory");
}

#ifdef GNPC_TILE_TRACE
// debug (tools/tile_trace.py): per-tile clock stamps of block 0 (math warp 0
// and the MMA warp) for the GNPC_TILE_TRACE-th sell_layer call of the process
__device__ unsigned long long g_trace[64 * 16];
__device__ int g_trace_layer, g_trace_on;
// (math warps: the LAST warp to reach the stamp, by atomicMax)
#define GNPC_TR_STAMP(k)                                                                    \
  do {                                                                                      \
    if (tr_on && lane == 0 && it < 64) atomicMax(&g_trace[it * 16 + (k)], (unsigned long long)clock64()); \
  } while (0)
#else
#define GNPC_TR_STAMP(k) \
  do {                   \
  } while (0)
#endif

// ---------------------------------------------------------------------------
// The layer pipeline as device functions shared by the per-layer kernel
// (k_layer_sell) and the whole-apply persistent kernel (k_apply_sell).
//
// Synchronisation inside a layer (no CTA-wide barrier in the tile loop):
//   full[s]  : ring slot s landed (TMA tx-count), control -> math warps
//   afull    : a tile's A operands and the previous tile's Y staging are
//              written (one arrival per math warp), math -> control warp
//   mma_bar  : MMA committed, control -> math warps.  Its completion also
//              means the Y staging buffer the next epilogue writes is free
//              (the control warp waits for older stores' smem reads first).
// afull(t) tells the control warp every warp passed its wait for MMA(t-1),
// so tile t-1's ring slot may be refilled.  The phase counters run on across
// the layers of the persistent kernel.
template <int DP, int CSR>
struct SellPipe {
  using C = SellCfg<DP, CSR>;
  uint8_t* ring;
  uint8_t* win;  // strip windows (PW)
  int* sched;    // PW: the CTA's tile schedule [3][KSCHED]
  float* lift;   // CSR = 9: lift tables a[33][DP], b[33][DP], t[32]
  uint8_t* A;  // [A2_hi | A2_lo]
  uint8_t* Bs;
  uint8_t* Ystg;
  uint8_t* D1op;
  float* D1;
  uint64_t* full;
  uint64_t* mma_bar;
  uint64_t* afull;
  uint64_t* efull;  // PW: a tile's epilogue (and the previous projection epilogue) read TMEM
  uint64_t* pbar;   // last layer: the projection MMA of a tile completed
  int* prog;
  uint32_t tmem;
  int talloc;
  int ring_it = 0, mma_it = 0, af_it = 0;  // phase counters (identical in every thread)
  int ef_it = 0;                           // efull phases (EARLY), across the layers of one launch
};

// Window sequence of the strip-window mode, replayed identically by the
// producer warp (which loads the windows), the MMA warp and the math warps
// (which read them): tile position j gets windows (a, b, c) = those of tiles
// u - S, u, u + S; window seq q lives in slot q % NWIN.  Along a strip
// (u = previous + S) only c is new; at a break (chunk start, strip end) three
// fresh seqs follow the last one.  Seqs strictly increase, so the issue rule
// "every seq below the current tile's MMA window b(it) is dead" makes a load
// into slot q % NWIN safe once q - NWIN < b(it).  (Reusing the previous
// tile's c seq for a break's a lets a break tile issued two tiles ahead
// overwrite a window its predecessor still gathers from.)
struct WinSeq {
  int last = -1, pb = -1, pc = -1, ctr = 0;
  // returns the number of new windows (3 at a break, else 1)
  __device__ __forceinline__ int next(int tile, int S, int& sa, int& sb, int& sc) {
    const bool brk = last < 0 || tile != last + S;
    int nnew;
    if (brk) {
      sa = ctr;
      sb = ctr + 1;
      sc = ctr + 2;
      nnew = 3;
    } else {
      sa = pb;
      sb = pc;
      sc = ctr;
      nnew = 1;
    }
    ctr = sc + 1;
    pb = sb;
    pc = sc;
    last = tile;
    return nnew;
  }
  // c of the next tile without advancing
  __device__ __forceinline__ int peek_c(int tile, int S) const {
    return (last < 0 || tile != last + S) ? ctr + 2 : ctr;
  }
};

// smem carve-up, barrier init, TMEM allocation (all threads of the CTA)
template <int DP, int CSR>
__device__ __forceinline__ SellPipe<DP, CSR> sell_setup(int hidden, bool last) {
  using C = SellCfg<DP, CSR>;
  extern __shared__ float4 smem_raw[];
  const uint32_t pad = (1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* base = reinterpret_cast<uint8_t*>(smem_raw) + pad;
  SellPipe<DP, CSR> p;
  p.ring = base + C::O_RING;
  p.win = base + C::O_WIN;
  p.A = base + C::O_A;
  p.Bs = base + C::O_B;
  p.Ystg = base + C::O_Y;
  p.D1op = base + C::O_Y;  // last layers only
  p.D1 = reinterpret_cast<float*>(base + C::o_p(hidden, last));
  p.full = reinterpret_cast<uint64_t*>(base + C::o_bar(hidden, last));
  p.talloc = last ? C::TALLOC_LAST : C::TALLOC;
  p.mma_bar = p.full + C::NS;
  p.afull = p.mma_bar + 1;
  p.efull = p.afull + 1;
  p.pbar = p.efull + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(p.pbar + 1);
  p.prog = reinterpret_cast<int*>(tslot + 1);  // PW: tiles whose MMA the control warp has issued
  p.sched = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(p.full) + 128);
  p.lift = reinterpret_cast<float*>(p.sched + 3 * C::KSCHED);
  const int tid = threadIdx.x;
  for (int t = tid; t < int(C::NS * C::SLOT / 16); t += C::NT)  // stale slice words must be valid columns
    reinterpret_cast<float4*>(p.ring)[t] = f4zero();
  if (tid == 0) {
    // (CSR = 9: + one arrival per lift warp, after it wrote the slot's new windows)
    for (int s = 0; s < C::NS; ++s) tc::mbar_init(&p.full[s], 1 + C::NLIFT);
    tc::mbar_init(p.mma_bar, 1);
    tc::mbar_init(p.afull, C::NW);
    tc::mbar_init(p.efull, C::NW);
    tc::mbar_init(p.pbar, 1);
    *p.prog = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if ((tid >> 5) == 0) tc::tmem_alloc(tslot, p.talloc);
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  p.tmem = *tslot;
  return p;
}

template <int DP, int CSR>
__device__ __forceinline__ void sell_teardown(const SellPipe<DP, CSR>& p) {
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if ((threadIdx.x >> 5) == 0) tc::tmem_dealloc(p.tmem, p.talloc);
}

// One fused Res-GCONV layer over this CTA's tiles (all threads call it).
// LAST: projection epilogue writing out[i] = (dec2ᵀ relu(dec1ᵀ y + b1) + b2)
// · out_scale (no Y).  uwp: the layer's B operands [Bu_lo | Bu_hi | Bw_lo |
// Bw_hi] in the swz_off<DP> layout.
template <int DP, bool LAST, typename OutT, int CSR, int KIND = 0>
__device__ __forceinline__ void sell_layer(SellPipe<DP, CSR>& p, const DevCsr& a, const CUtensorMap* mapx,
                                           const CUtensorMap* mapy, const float* __restrict__ X,
                                           const float* __restrict__ axlong, const float* __restrict__ uwp,
                                           const NetView& net, double out_scale, OutT* __restrict__ out,
                                           const TrainIO* tio = nullptr, const CUtensorMap* mapxw = nullptr,
                                           const LiftIO* lio = nullptr) {
  using C = SellCfg<DP, CSR>;
  constexpr int TM = C::TM, G = C::G, R = C::R, NS = C::NS, NW = C::NW, NQ = C::NQ;
  constexpr bool TR = C::TR;
  static_assert(!TR || (!LAST && KIND != 0), "training layers have no projection");
  const int bs = TR ? tio->bs : 1;           // virtual rows per node
  const int nodes = a.n;
  const int n = nodes * bs;                  // (virtual) rows
  const int ntiles = (n + TM - 1) / TM;
  const int npt = TM / bs;                   // nodes per tile (training: bs divides TM)
  const int lbs = __ffs(bs) - 1;             // log2(bs)
  const bool use_mask = KIND == 2 && tio->use_mask;
  const int H = net.hidden;
  float* D1 = p.D1;
  float* B1 = D1 + DP * H;
  float* D2 = B1 + H;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // this layer's operands; every MMA of the previous layer has completed
  // (its epilogues waited for them before the caller's barrier)
  for (int t = tid; t < int(4 * C::BB / 16); t += C::NT)
    reinterpret_cast<float4*>(p.Bs)[t] = reinterpret_cast<const float4*>(uwp)[t];
  // last layer: the projection's first matrix on the tensor cores when its
  // width allows (TCP), as the B operand [D1_lo; D1_hi] (rows h, K = DP:
  // D1op(h, j) = dec1(j, h), split hi = trunc, lo = rest); else dec1 in fp32
  const bool TCP = LAST && C::tc_proj(H);
  if constexpr (LAST) {
    if (TCP) {
      for (int t = tid; t < H * DP; t += C::NT) {
        const int h = t / DP, j = t % DP;
        const float v = net.dec1[j * H + h];
        const float hi = __int_as_float(__float_as_int(v) & 0xffffe000);
        *reinterpret_cast<float*>(p.D1op + tc::swz_off<DP>(h, j)) = v - hi;      // rows 0..H-1: lo
        *reinterpret_cast<float*>(p.D1op + tc::swz_off<DP>(H + h, j)) = hi;      // rows H..2H-1: hi
      }
    } else {
      for (int t = tid; t < DP * H; t += C::NT) D1[t] = net.dec1[t];
    }
    for (int t = tid; t < H; t += C::NT) {
      B1[t] = net.dec1_b[t];
      D2[t] = net.dec2[t];
    }
  }
  if constexpr (C::LIFT) {  // the piecewise-linear lift's tables (k_lift_pw's)
    const int nb = net.nbreak;
    for (int t = tid; t < (nb + 1) * DP; t += C::NT) {
      p.lift[t] = net.lift_a[t];
      p.lift[C::kLiftIv * DP + t] = net.lift_b[t];
    }
    for (int t = tid; t < nb; t += C::NT) p.lift[2 * C::kLiftIv * DP + t] = net.lift_t[t];
  }
  tc::fence_proxy_async();
  __syncthreads();
  // tile schedule: round-robin, or (strip windows) a contiguous chunk of the
  // layout's strip order, so consecutive tiles share X-row windows
  // window-mode arrays: the apply layout (pw) or the training layout (tw)
  const int* w_k = C::TW ? a.tw_k : a.pw_k;
  const int* w_off = C::TW ? a.tw_off : a.pw_off;
  const uint8_t* w_sl = C::TW ? a.tw : a.pw;
  const int w_S = C::TW ? a.tw_S : a.pw_S;
  // rows of halo on either side of a window's own 128 rows: 8 (PW), one node (TW)
  const int w_halo = C::TW ? bs : kPwHalo;
  const int* torder = C::TW ? a.tw_order : (C::PW ? a.pw_order : nullptr);
  const int chunk0 = torder ? static_cast<int>(static_cast<long long>(blockIdx.x) * ntiles / gridDim.x) : 0;
  const int my_tiles =
      torder ? static_cast<int>(static_cast<long long>(blockIdx.x + 1) * ntiles / gridDim.x) - chunk0
             : (blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0);
  // PW: this CTA's chunk of the strip order with each tile's K and slice
  // offset, staged in shared memory once (the control thread would otherwise
  // chase order -> K -> offset through L2 for every tile it issues)
  int* sch_t = p.sched;
  int* sch_k = p.sched + C::KSCHED;
  int* sch_o = p.sched + 2 * C::KSCHED;
  const bool use_sched = C::WINS && my_tiles <= C::KSCHED;
  if (use_sched) {
    for (int j = tid; j < my_tiles; j += C::NT) {
      const int t = __ldg(torder + chunk0 + j);
      sch_t[j] = t;
      sch_k[j] = __ldg(w_k + t);
      sch_o[j] = __ldg(w_off + t);
    }
    __syncthreads();
  }
  auto tile_at = [&](int it) -> int {
    if (use_sched) return sch_t[it];
    return torder ? __ldg(torder + chunk0 + it) : static_cast<int>(blockIdx.x + it * gridDim.x);
  };
  // L2 policies: Â streams evict_first, X gathers evict_last (a.l2hint)
  // (training activations are far larger than L2: normal policy there)
  const bool hint = a.l2hint && !TR;
  const uint64_t pol_stream = hint ? l2_policy_evict_first() : l2_policy_evict_normal();
  const uint64_t pol_keep = hint ? l2_policy_evict_last() : l2_policy_evict_normal();
  const int rb = p.ring_it, mb = p.mma_it, ab = p.af_it, eb = p.ef_it;
  // commits: one per tile, plus the last projection MMA's (TCP)
  const int ncommit = my_tiles;  // (the projection MMAs commit to pbar)
  p.ring_it += my_tiles;
  p.mma_it += ncommit;
  p.af_it += my_tiles > 0 ? my_tiles + 1 : 0;
  p.ef_it += my_tiles;  // one efull completion per tile
  if (my_tiles == 0) return;
#ifdef GNPC_TILE_TRACE
  // (no static shared memory: the layer kernels take all 227 KB dynamically)
  if (tid == 0 && blockIdx.x == 0) g_trace_on = atomicAdd(&g_trace_layer, 1) == GNPC_TILE_TRACE;
  __syncthreads();
  const bool tr_on = blockIdx.x == 0 && *reinterpret_cast<volatile int*>(&g_trace_on) != 0 && warp <= NW;
#endif

  if constexpr (C::LIFT) {
    if (warp >= NW + 2) {
      // ============================================================ lift warps
      // They replay the producer's issue sequence (same gating on the MMA
      // warp's progress counter) and, where the producer of the other modes
      // loads a window by TMA, compute it: window row r of tile u is global
      // row c = 128 u - halo + r, x1[c] = a[p] v + b[p] with v the scaled
      // input and p its kink interval (k_lift_pw's arithmetic, bit for bit);
      // rows outside [0, n) are zero, as the TMA's out-of-bounds fill.
      const int lw = warp - (NW + 2);
      const float* s_a = p.lift;
      const float* s_b = s_a + C::kLiftIv * DP;
      const float* s_t = s_b + C::kLiftIv * DP;
      const int nb = net.nbreak;
      const double in_scale = lio->sc->in_scale;
      constexpr int WR = TM + 2 * kPwHalo;             // 144 rows
      constexpr int NP = (WR + 32 * C::NLIFT - 1) / (32 * C::NLIFT);  // passes per window
      WinSeq ws, wsb;
      int nxt = 0, bcur = 0;
      // lane -> row of a 32-row block and chunk rotation chosen so that both
      // the table reads (lanes of a quarter-warp in different intervals: chunk
      // ch ^ i differs per lane) and the swizzled window stores (physical chunk
      // ch ^ i ^ (r & 7) differs per lane) are free of bank conflicts
      const int li = lane & 7, lg = lane >> 3;
      const int lrow = 8 * (li & 3) + 2 * lg + (li >> 2);
      const size_t esz = lio->f64 ? 8 : 4;
      auto fill = [&](int q, int u) {
        uint8_t* wb = p.win + (q % C::NWIN) * C::WINB;
        float v[NP];
        {  // the next window along the strip into L1 (its loads then skip the L2 round trip)
          const long long c0 = static_cast<long long>(u + w_S) * TM - kPwHalo;
          const long long cp = c0 + 32 * lane;
          if (lane < (WR + 31) / 32 + 1 && cp >= 0 && cp < n)
            asm volatile("prefetch.global.L1 [%0];" ::"l"(static_cast<const char*>(lio->in) + cp * esz));
        }
#pragma unroll
        for (int k = 0; k < NP; ++k) {
          const int r = (k * C::NLIFT + lw) * 32 + lrow;
          const long long c = static_cast<long long>(u) * TM - kPwHalo + r;
          v[k] = 0.f;
          if (r < WR && c >= 0 && c < n) {
            const double x = lio->f64 ? static_cast<const double*>(lio->in)[c]
                                      : static_cast<double>(static_cast<const float*>(lio->in)[c]);
            v[k] = static_cast<float>(in_scale * x);
          }
        }
#pragma unroll
        for (int k = 0; k < NP; ++k) {
          const int r = (k * C::NLIFT + lw) * 32 + lrow;
          if (r >= WR) continue;
          const long long c = static_cast<long long>(u) * TM - kPwHalo + r;
          const bool in_rows = c >= 0 && c < n;
          int lo = 0, hi = nb;  // interval = #kinks <= v
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (s_t[mid] <= v[k]) lo = mid + 1;
            else hi = mid;
          }
          uint8_t* row = wb + r * (DP * 4);
#pragma unroll
          for (int c8 = 0; c8 < DP / 4; ++c8) {
            const int ch = c8 ^ li;
            const float4 al = *reinterpret_cast<const float4*>(s_a + lo * DP + 4 * ch);
            const float4 be = *reinterpret_cast<const float4*>(s_b + lo * DP + 4 * ch);
            const float4 o = in_rows ? make_float4(fmaf(al.x, v[k], be.x), fmaf(al.y, v[k], be.y),
                                                   fmaf(al.z, v[k], be.z), fmaf(al.w, v[k], be.w))
                                     : f4zero();
            *reinterpret_cast<float4*>(row + ((ch ^ (r & 7)) << 4)) = o;
          }
        }
      };
      auto issue_lift = [&](int j) {
        const int t = tile_at(j);
        int sa, sb, sc;
        const int nnew = ws.next(t, w_S, sa, sb, sc);
        if (nnew == 3) {
          fill(sa, t - w_S);
          fill(sb, t);
        }
        fill(sc, t + w_S);
        tc::fence_proxy_async();  // window b is also the MMA's A operand (async proxy)
        __syncwarp();
        if (lane == 0) mbar_arrive(&p.full[(rb + j) % NS]);
      };
      auto issue_more = [&](int it) {
        const int prot = it >= 0 ? bcur : 0;
        while (nxt < my_tiles && nxt <= it + NS - 1 && ws.peek_c(tile_at(nxt), w_S) - prot < C::NWIN)
          issue_lift(nxt++);
      };
      issue_more(-1);
      for (int it = 0; it < my_tiles && nxt < my_tiles; ++it) {
        while (true) {
          int v;
          asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(tc::smem_u32(p.prog)) : "memory");
          if (v > it) break;
          __nanosleep(32);
        }
        int sa, sc;
        wsb.next(tile_at(it), w_S, sa, bcur, sc);
        issue_more(it);
      }
      return;
    }
  }
  if (warp >= NW) {
    // ============================================================ control warp
    // (strip windows: warp NW issues the MMAs and Y stores, warp NW + 1 the
    // ring and window loads, following the MMA warp's progress counter)
    const bool producer = C::NPROD && warp == NW + 1;
    if (lane == 0) {
      if constexpr (!C::LIFT) tc::tma_prefetch_desc(C::WINS ? mapxw : mapx);
      if (!LAST) tc::tma_prefetch_desc(mapy);
      auto issue = [&](int it) {  // tile `it` of this CTA into ring slot (rb + it) % NS
        if (it >= my_tiles) return;
        const int t = tile_at(it);
        const int r = rb + it;
        const int s = r % NS;
        uint8_t* slot = p.ring + s * C::SLOT;
        if constexpr (TR) {
          // the tile's nodes [n0, n0 + npt): full CSR range (padded arrays)
          const int n0 = t * npt;
          const int kb = __ldg(a.rp + n0), ke = __ldg(a.rp + min(n0 + npt, nodes));
          const int a0 = kb & ~3, cnt = ((ke + 3) & ~3) - a0;
          const bool staged = cnt <= C::CAPC;
          tc::mbar_expect_tx(&p.full[s],
                             C::OPB + (use_mask ? C::MASKB : 0) + C::RPB + (staged ? 8 * cnt : 0));
          tc::tma_load_2d(slot, mapx, 0, t * TM, &p.full[s]);
          if (use_mask) {
            if constexpr (C::MBITS)
              tc::bulk_load(slot + C::O_MASK, tio->mask_in + static_cast<size_t>(t) * TM, C::MASKB, &p.full[s]);
            else
              tc::tma_load_2d(slot + C::O_MASK, tio->mapmask, 0, t * TM, &p.full[s]);
          }
          // row_ptr slice from the 16-byte aligned node n0 & ~3 (npt < 4 when bs > 32)
          tc::bulk_load(slot + C::O_RP, a.rp + (n0 & ~3), C::RPB, &p.full[s]);
          if (staged && cnt > 0) {
            tc::bulk_load(slot + C::O_CI, a.ci + a0, 4 * cnt, &p.full[s]);
            tc::bulk_load(slot + C::O_V, a.v + a0, 4 * cnt, &p.full[s]);
          }
        } else if constexpr (CSR == 1) {
          // the tile's short-row CSR range, 16-byte aligned superset [a0, a1)
          const int kb = __ldg(a.rps + t * TM), ke = __ldg(a.rps + min((t + 1) * TM, n));
          const int a0 = kb & ~3, cnt = ((ke + 3) & ~3) - a0;
          const bool staged = cnt <= C::CAPC;
          tc::mbar_expect_tx(&p.full[s], C::OPB + C::RPB + (staged ? 8 * cnt : 0));
          tc::tma_load_2d_hint(slot, mapx, 0, t * TM, &p.full[s], pol_keep);
          tc::bulk_load_hint(slot + C::O_RP, a.rps + t * TM, C::RPB, &p.full[s], pol_stream);
          if (staged && cnt > 0) {
            tc::bulk_load_hint(slot + C::O_CI, a.cis + a0, 4 * cnt, &p.full[s], pol_stream);
            tc::bulk_load_hint(slot + C::O_V, a.vs + a0, 4 * cnt, &p.full[s], pol_stream);
          }
        } else {
          const int K = __ldg((C::PAIR ? a.psell_k : a.sell_k) + t) & 0xffff;
          const bool staged = K > 0 && K <= C::KCAP;
          tc::mbar_expect_tx(&p.full[s], C::OPB + (staged ? K * TM * 8 : 0));
          tc::tma_load_2d_hint(slot, mapx, 0, t * TM, &p.full[s], pol_keep);
          if (staged) {
            const void* src = C::PAIR ? static_cast<const void*>(a.psell + __ldg(a.psell_off + t))
                                      : static_cast<const void*>(a.sell + __ldg(a.sell_off + t));
            tc::bulk_load_hint(slot + C::OPB, src, K * TM * 8, &p.full[s], pol_stream);
          }
        }
      };
      // strip windows (PW): tiles are issued in order while the slice ring
      // has room (j <= it + NS - 1) and the new windows' slots are free: every
      // window older than the current tile's MMA window b(it) is dead
      WinSeq ws;   // issue side
      WinSeq wsb;  // MMA side: b(it) of the current tile
      int nxt = 0, bcur = 0;
      // window box bytes (the TMA map's box: 128 + 2 halo rows)
      const uint32_t winb = static_cast<uint32_t>(TM + 2 * w_halo) * DP * 4;
      auto issue_pw = [&](int j) {
        const int t = tile_at(j);
        int sa, sb, sc;
        const int nnew = ws.next(t, w_S, sa, sb, sc);
        const int s = (rb + j) % NS;
        uint8_t* slot = p.ring + s * C::SLOT;
        const int K = use_sched ? sch_k[j] : __ldg(w_k + t);
        const int off = use_sched ? sch_o[j] : __ldg(w_off + t);
        // slice bytes: pair-union 10 B x 64 pairs per entry; training: the
        // node starts (ST = npt + 1 rounded to 8) plus 6 B per entry
        const uint32_t slb = C::TW ? static_cast<uint32_t>(2 * (((TM / bs) + 1 + 7) & ~7) + 6 * K)
                                   : static_cast<uint32_t>(K * (TM / 2) * 10);
        const bool mk = C::TW && use_mask;
        // (CSR = 9: the lift warps write the windows and arrive for them)
        tc::mbar_expect_tx(&p.full[s], slb + (C::LIFT ? 0 : nnew * winb) + (mk ? C::MASKB : 0));
        tc::bulk_load_hint(slot + (C::TW ? C::O_TWS : 0), w_sl + static_cast<size_t>(off) * 16, slb, &p.full[s],
                           pol_stream);
        if constexpr (C::TW) {
          if (mk) tc::bulk_load(slot + C::O_MASK, tio->mask_in + static_cast<size_t>(t) * TM, C::MASKB, &p.full[s]);
        }
        auto load_win = [&](int q, int u) {
          tc::tma_load_2d_hint(p.win + (q % C::NWIN) * C::WINB, mapxw, 0, u * TM - w_halo, &p.full[s], pol_keep);
        };
        if constexpr (!C::LIFT) {
          if (nnew == 3) {
            load_win(sa, t - w_S);
            load_win(sb, t);
          }
          load_win(sc, t + w_S);
        }
      };
      auto issue_more = [&](int it) {  // after afull(it) (it = -1: prologue)
        const int prot = it >= 0 ? bcur : 0;
        while (nxt < my_tiles && nxt <= it + NS - 1 && ws.peek_c(tile_at(nxt), w_S) - prot < C::NWIN)
          issue_pw(nxt++);
      };
      if constexpr (C::WINS) {
        if (producer) {
          issue_more(-1);
          for (int it = 0; it < my_tiles && nxt < my_tiles; ++it) {
            // MMA(it) issued: tile it's gathers are done, its window b(it) in use
            while (true) {
              int v;
              asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(tc::smem_u32(p.prog)) : "memory");
              if (v > it) break;
              __nanosleep(32);
            }
            int sa, sc;
            wsb.next(tile_at(it), w_S, sa, bcur, sc);
            issue_more(it);
          }
        }
      }
      else if (C::NPROD == 0 || producer) {
        for (int it = 0; it < NS - 1; ++it) issue(it);
        if (producer) {
          for (int it = 0; it < my_tiles; ++it) {  // after MMA(it): its slot's previous tile is done
            while (true) {
              int v;
              asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(tc::smem_u32(p.prog)) : "memory");
              if (v > it) break;
              __nanosleep(32);
            }
            issue(it + NS - 1);
          }
        }
      }
      constexpr uint32_t idesc = tc::idesc_tf32(128, DP);
      constexpr uint32_t idesc2 = tc::idesc_tf32(128, 2 * DP);
      const uint32_t sBstk = tc::smem_u32(p.Bs);
      const uint32_t sA2hi = tc::smem_u32(p.A), sA2lo = sA2hi + C::OPB;
      const uint32_t tAlo = p.tmem + C::alo_col(TCP);
      const uint32_t sXe0 = tc::smem_u32(p.win) + w_halo * DP * 4;
      auto proj_mma = [&](int t1) {  // projection of tile t1 (its relu'd rows hi / lo in TMEM)
        // Dp[:, 0:H] = Y_hi·D1_lo, Dp[:, H:2H] = Y_hi·D1_hi + Y_lo·D1_hi
        const uint32_t tYh = p.tmem + C::ycol((mb + t1) & 1), tYl = tYh + DP;  // A from TMEM
        const uint32_t sD = tc::smem_u32(p.D1op);
        const uint32_t sDh = sD + H * DP * 4;
        const uint32_t iH = tc::idesc_tf32(128, H), i2H = tc::idesc_tf32(128, 2 * H);
        const uint32_t pacc = p.tmem + 2 * DP;
#pragma unroll
        for (int k8 = 0; k8 < DP / 8; ++k8) {
          tc::mma_tf32_ts(pacc, tYh + 8 * k8, tc::make_desc_swz<DP>(sD + k8 * 32), i2H, k8 > 0);
          tc::mma_tf32_ts(pacc + H, tYl + 8 * k8, tc::make_desc_swz<DP>(sDh + k8 * 32), iH, 1);
        }
      };
      for (int it = 0; it <= (producer ? -1 : my_tiles); ++it) {
        if constexpr (C::EARLY) {
          if (it >= 1) {  // epilogue(it-1) and projection epilogue(it-2) have read TMEM
            tc::mbar_wait_dbg(p.efull, (eb + it - 1) & 1, 5, it);
            tc::fence_after();
          }
          GNPC_TR_STAMP(8);
          if (it < my_tiles) {  // X_hi·[U_lo; U_hi] once the tile's rows landed
            const int r = rb + it;
            tc::mbar_wait_dbg(&p.full[r % NS], (r / NS) & 1, 6, it);
            tc::fence_after();
            uint32_t sX = tc::smem_u32(p.ring + (r % NS) * C::SLOT);
            if constexpr (C::WINS) {
              int sa, sc;
              wsb.next(tile_at(it), w_S, sa, bcur, sc);
              sX = sXe0 + (bcur % C::NWIN) * C::WINB;
            }
#pragma unroll
            for (int k8 = 0; k8 < DP / 8; ++k8)
              tc::mma_tf32(p.tmem, tc::make_desc_swz<DP>(sX + k8 * 32), tc::make_desc_swz<DP>(sBstk + k8 * 32),
                           idesc2, k8 > 0);
          }
        }
        GNPC_TR_STAMP(9);
        tc::mbar_wait_dbg(p.afull, (ab + it) & 1, 1, it);
        tc::fence_after();
        GNPC_TR_STAMP(10);
        // stores issued up to the previous iteration have left the Y staging:
        // the buffer the epilogue after this MMA writes is free (waiting
        // after the MMA issue instead measured the same: C2, C4)
        tc::bulk_wait_read0();
        if (KIND == 1 && it < my_tiles && !tio->no_ax) {  // training forward: the tile's ÂX (A2_hi) to HBM
          tc::tma_store_2d(tio->mapax, p.A, 0, tile_at(it) * TM);
          tc::bulk_commit();
        }
        if (it < my_tiles) {
          uint32_t sX = tc::smem_u32(p.ring + ((rb + it) % NS) * C::SLOT);
          if constexpr (C::WINS) {  // the tile's own rows: window b(it) past its halo
            if constexpr (!C::EARLY) {
              int sa, sc;
              wsb.next(tile_at(it), w_S, sa, bcur, sc);
            }
            sX = sXe0 + (bcur % C::NWIN) * C::WINB;
          }
          // 3xTF32 with the two A_hi products stacked along N (A_hi is read
          // once for both): D[:, 0:DP] = A_hi·B_lo, D[:, DP:2DP] = A_hi·B_hi +
          // A_lo·B_hi; the epilogue adds the halves.  Each part's B operands
          // are stored [B_lo | B_hi], i.e. as one 2DP-row operand.  The
          // landed X tile is A_hi of the X·U part (kind::tf32 truncates); its
          // A_lo is in TMEM (TS form).
          uint32_t accf = 0;
#pragma unroll
          for (int part = 0; part < 2; ++part) {
            const uint32_t sah = part == 0 ? sX : sA2hi;
            const uint32_t sbs = sBstk + part * 2 * C::BB;  // [B_lo; B_hi] of this part (2DP rows)
            const uint32_t sbh = sbs + C::BB;                // B_hi rows alone
            // (the A_hi products of a part first, then its A_lo products: the
            // same accumulation order whether or not EARLY issues part 0's
            // A_hi products before afull, so every layout gives the same bits)
#pragma unroll
            for (int k8 = 0; k8 < DP / 8; ++k8) {
              if (!(C::EARLY && part == 0))  // (EARLY: issued before afull)
                tc::mma_tf32(p.tmem, tc::make_desc_swz<DP>(sah + k8 * 32),
                             tc::make_desc_swz<DP>(sbs + k8 * 32), idesc2, accf);
              accf = 1;
            }
#pragma unroll
            for (int k8 = 0; k8 < DP / 8; ++k8) {
              if (part == 0)
                tc::mma_tf32_ts(p.tmem + DP, tAlo + 8 * k8, tc::make_desc_swz<DP>(sbh + k8 * 32), idesc, 1);
              else
                tc::mma_tf32(p.tmem + DP, tc::make_desc_swz<DP>(sA2lo + k8 * 32),
                             tc::make_desc_swz<DP>(sbh + k8 * 32), idesc, 1);
            }
          }
        }
        if (KIND == 1 && it < my_tiles && !tio->no_ax) tc::bulk_wait_read0();  // A2_hi is rewritten after the commit
        if (it < my_tiles) tc::mma_commit(p.mma_bar);
        GNPC_TR_STAMP(11);
        // the projection of tile it-1 after MMA(it), on its own barrier: the
        // epilogues' wait for MMA(it) does not include it
        if (TCP && it >= 1) {
          proj_mma(it - 1);
          tc::mma_commit(p.pbar);
        }
        if (!LAST && it >= 1) {  // tile it-1 is fully staged
          // the layer output streams past this layer's gathers (evict_first:
          // C4 158 -> 155.5 us per layer)
          tc::tma_store_2d_hint(mapy, p.Ystg + ((mb + it - 1) & 1) * C::OPB, 0, tile_at(it - 1) * TM, pol_stream);
          if constexpr (KIND == 1 && C::MBITS) {
            if (tio->mask_out) {
              const int t1 = tile_at(it - 1);
              tc::bulk_store(tio->mask_out + static_cast<size_t>(t1) * TM * 4,
                             p.Ystg + C::O_MST - C::O_Y + ((mb + it - 1) & 1) * TM * 4, TM * 4);
            }
          }
          tc::bulk_commit();
        }
        // every warp passed its wait for MMA(it-1): that slot takes tile it+NS-1
        if constexpr (C::NPROD) {  // the producer warp refills
          if (it < my_tiles)
            asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(tc::smem_u32(p.prog)), "r"(it + 1) : "memory");
        } else {
          issue(it + NS - 1);
        }
      }
      // the layer's output is in global memory before the caller's barrier
      tc::bulk_wait0();
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    __syncwarp();
    return;
  }

  // ================================================================ math warps
  const int gl = tid % G, gid = tid / G;
  float y[LAST ? DP : 1];
  // epilogue of local tile itp (accumulator in TMEM).  Non-last layers:
  // relu'd rows -> Ystg (warp w: lanes 32(w%4).., column group w/4), stored
  // by the control warp's TMA.  Last layer: the projection group of this tile
  // (warps 4*(itp%NQ)..+3, one per lane quarter) pulls whole rows into
  // registers `y` and projects them after arriving — the groups rotate, so
  // no CTA-wide barrier is needed.
  // With the tensor-core projection (TCP) the last layer stages its relu'd
  // rows hi / lo into TMEM (ycol) for the control warp's
  // projection MMA, and the rotating group reads the projection accumulator
  // one tile later (proj_epilogue).
  auto epilogue = [&](int itp) -> bool {
    // (a suspend-time hint on this try_wait measured the same: C5, C2)
    tc::mbar_wait_dbg(p.mma_bar, (mb + itp) & 1, 2, itp);
    tc::fence_after();
    {
      const int it = itp + 1;
      (void)it;
      GNPC_TR_STAMP(3);
    }
    const int q = warp & 3, cq = warp >> 2;  // lane quarter, column group
    const uint32_t trow = p.tmem + (static_cast<uint32_t>(32 * q) << 16);
    if (LAST && !TCP) {
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
      constexpr int CW = DP / NQ;  // columns per warp: 4 or 8
      uint8_t* ys = p.Ystg + ((mb + itp) & 1) * C::OPB;
      float yh[LAST ? CW : 1], ylo[LAST ? CW : 1];
      const uint32_t taddr = trow + cq * CW;
      float v[CW];
      if constexpr (CW == 4) {
        float v2[4];
        tc::tmem_ld4x2(taddr, taddr + DP, v, v2);  // both halves in flight, one wait
#pragma unroll
        for (int c = 0; c < 4; ++c) v[c] += v2[c];
      } else {
#pragma unroll
        for (int c0 = 0; c0 < CW; c0 += 8) {
          float u1[8], u2[8];
          tc::tmem_ld8x2(taddr + c0, taddr + DP + c0, u1, u2);  // both halves in flight, one wait
#pragma unroll
          for (int c = 0; c < 8; ++c) v[c0 + c] = u1[c] + u2[c];
        }
      }
      // training backward: D ⊙ [X_l > 0] from the tile's mask (its ring slot
      // is refilled only after this iteration's arrival), no relu
      const uint8_t* msk = p.ring + ((rb + itp) % NS) * C::SLOT + C::O_MASK;
      uint32_t mword = 0u, mout = 0u;
      if constexpr (KIND == 2 && C::MBITS) {
        if (use_mask) mword = *reinterpret_cast<const uint32_t*>(msk + 4 * m) >> (cq * CW);
      }
#pragma unroll
      for (int c = 0; c < CW; c += 4)
      {
        float4 yv;
        if constexpr (KIND == 2) {
          yv = make_float4(v[c], v[c + 1], v[c + 2], v[c + 3]);
          if (use_mask) {
            if constexpr (C::MBITS) {
              yv.x = (mword >> c) & 1u ? yv.x : 0.f;
              yv.y = (mword >> (c + 1)) & 1u ? yv.y : 0.f;
              yv.z = (mword >> (c + 2)) & 1u ? yv.z : 0.f;
              yv.w = (mword >> (c + 3)) & 1u ? yv.w : 0.f;
            } else {
              const float4 mk = *reinterpret_cast<const float4*>(msk + tc::swz_off<DP>(m, cq * CW + c));
              yv.x = mk.x > 0.f ? yv.x : 0.f;
              yv.y = mk.y > 0.f ? yv.y : 0.f;
              yv.z = mk.z > 0.f ? yv.z : 0.f;
              yv.w = mk.w > 0.f ? yv.w : 0.f;
            }
          }
        } else {
          yv = make_float4(relu(v[c]), relu(v[c + 1]), relu(v[c + 2]), relu(v[c + 3]));
          mout |= (v[c] > 0.f ? 1u : 0u) << c | (v[c + 1] > 0.f ? 1u : 0u) << (c + 1) |
                  (v[c + 2] > 0.f ? 1u : 0u) << (c + 2) | (v[c + 3] > 0.f ? 1u : 0u) << (c + 3);
        }
        if constexpr (LAST) {  // projection operand, kept in TMEM (hi, lo)
          const float4 yl = f4_trunc_lo(yv);
          yh[c] = yv.x; yh[c + 1] = yv.y; yh[c + 2] = yv.z; yh[c + 3] = yv.w;
          ylo[c] = yl.x; ylo[c + 1] = yl.y; ylo[c + 2] = yl.z; ylo[c + 3] = yl.w;
        } else {
          *reinterpret_cast<float4*>(ys + tc::swz_off<DP>(m, cq * CW + c)) = yv;
        }
      }
      if constexpr (LAST) {
        // rows are TMEM lanes as in the accumulator: Y_hi at ycol(buf),
        // Y_lo DP columns on (the projection MMA reads them as its A operand)
        const uint32_t ty = p.tmem + C::ycol((mb + itp) & 1) + (static_cast<uint32_t>(32 * q) << 16) + cq * CW;
        if constexpr (CW == 8) {
          tc::tmem_st8(ty, yh);
          tc::tmem_st8(ty + DP, ylo);
        } else {
          tc::tmem_st4(ty, yh);
          tc::tmem_st4(ty + DP, ylo);
        }
        tc::tmem_wait_st();
      }
      if constexpr (KIND == 1 && C::MBITS) {  // this warp's CW = 8 columns: one byte of the row's word
        p.Ystg[C::O_MST - C::O_Y + ((mb + itp) & 1) * TM * 4 + 4 * m + cq] = static_cast<uint8_t>(mout);
      }
      tc::fence_before();
      return false;
    }
  };
  // TCP: projection epilogue of local tile itp (its projection MMA completed
  // with the commit this iteration waited for): the rotating group reads its
  // rows' 2H accumulator columns, out = (Σ_h relu(z_h + b1_h) dec2_h + b2)·τ/√n
  // The projection epilogue runs on all math warps: warp (lane quarter q,
  // column group cq) reduces relu(z + b1)·dec2 over its H / NQ projection
  // columns for the quarter's 32 rows into PART; one tile later the rotating
  // warp of each quarter adds the NQ partials in a fixed order and writes
  // out[i] (the rotating group alone doing the whole reduction made every
  // tile wait for it: C5 last layer ~19 % of stalls on the MMA barrier).
  float* PART = D2 + H;  // [2][NQ][TM]
  // hidden 32: the warp's 8 projection columns' b1 / dec2 live in registers
  // (they were two shared-memory reads per element: the hottest line of the
  // last layer's profile), and both accumulator halves load under one wait
  float b1r[8], d2r[8];
  const bool proj8 = TCP && H / NQ == 8;
  if (proj8) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      b1r[c] = B1[(warp >> 2) * 8 + c];
      d2r[c] = D2[(warp >> 2) * 8 + c];
    }
  }
  auto proj_epilogue = [&](int itp) {
    tc::mbar_wait_dbg(p.pbar, itp & 1, 7, itp);  // the projection MMA of tile itp
    tc::fence_after();
    const int q = warp & 3, cq = warp >> 2;
    const int hc = H / NQ;  // H % 16 == 0 (tensor-core projection)
    const uint32_t prow = p.tmem + 2 * DP + (static_cast<uint32_t>(32 * q) << 16) + cq * hc;
    float o = 0.f;
    if (proj8) {
      float z1[8], z2[8];
      tc::tmem_ld8x2(prow, prow + H, z1, z2);
#pragma unroll
      for (int c = 0; c < 8; ++c) o = fmaf(relu(z1[c] + z2[c] + b1r[c]), d2r[c], o);
    } else
    for (int h0 = 0; h0 < hc; h0 += 4) {
      float z1[4], z2[4];
      tc::tmem_ld4(prow + h0, z1);
      tc::tmem_ld4(prow + H + h0, z2);
#pragma unroll
      for (int c = 0; c < 4; ++c) o = fmaf(relu(z1[c] + z2[c] + B1[cq * hc + h0 + c]), D2[cq * hc + h0 + c], o);
    }
    tc::fence_before();
    PART[((itp & 1) * NQ + cq) * TM + 32 * q + lane] = o;
  };
  auto proj_final = [&](int itp) {
    const int q = warp & 3, cq = warp >> 2;
    if (cq != itp % NQ) return;
    const float* pp = PART + (itp & 1) * NQ * TM + 32 * q + lane;
    float o = pp[0];
#pragma unroll
    for (int c = 1; c < NQ; ++c) o += pp[c * TM];
    const int i = tile_at(itp) * TM + 32 * q + lane;
    if (i < n) out[i] = static_cast<OutT>(static_cast<double>(o + net.dec2_b) * out_scale);
  };
  auto arrive = [&]() {
    tc::fence_proxy_async();
    __syncwarp();
    if (lane == 0) mbar_arrive(p.afull);
  };
  // LAST: projection MLP (src/gnn.cpp:178-199) of the row this lane holds
  // (row 32*(warp%4) + lane of the tile at row0); dec1 read as warp-uniform
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
      if (i < n) out[i] = static_cast<OutT>(static_cast<double>(o + net.dec2_b) * out_scale);
    }
  };

  // per tile: K_t | has-long << 16 (SELL, pair-union), has-long (CSR)
  const int* tinfo = C::CSRL ? a.tflag : (C::PAIR ? a.psell_k : (C::PW ? a.pw_k : a.sell_k));
  int kw = TR ? 0 : (use_sched ? sch_k[0] : __ldg(tinfo + tile_at(0)));
  const int iters = my_tiles + 1 + (TCP ? 2 : 0);
  WinSeq wsm;                       // strip windows (PW): the control warp's sequence, replayed
  const uint8_t* wtile = nullptr;   // PW: the tile's own rows (window b past its halo)
  for (int it = 0; it < iters; ++it) {
    const bool have = it < my_tiles;
    const int tile = have ? tile_at(it) : 0;
    const int row0 = tile * TM;
    const int r = rb + it;
    uint8_t* slot = p.ring + (r % NS) * C::SLOT;
    float4 acc[R];
    uint32_t wbase = 0;  // PW: shared address of window a; b, c follow (wrapped in the ring)
    const uint32_t wring0 = tc::smem_u32(p.win);
    if constexpr (C::WINS) {
      if (have) {
        int sq[3];
        wsm.next(tile, w_S, sq[0], sq[1], sq[2]);
        wbase = wring0 + (sq[0] % C::NWIN) * C::WINB;
        wtile = p.win + (sq[1] % C::NWIN) * C::WINB + w_halo * DP * 4;
      }
    }
    if (have) {
      const int K = C::CSRL ? 0 : (kw & 0xffff);
      // (strip-window layouts are built only for matrices without long rows)
      const bool haslong = !TR && !C::WINS && (C::CSRL ? kw != 0 : (kw >> 16) != 0);
      const bool staged = K > 0 && K <= C::KCAP;
      if (!TR)  // prefetch
        kw = it + 1 < my_tiles ? (use_sched ? sch_k[it + 1] : __ldg(tinfo + tile_at(it + 1))) : 0;

      // ----------------------------------------------------------- gather
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const int i = row0 + R * gid + j;
        acc[j] = f4zero();
        if (haslong && i < n && __ldg(a.rp + i + 1) - __ldg(a.rp + i) > kLongRow)
          acc[j] = ldg4(axlong + static_cast<size_t>(i) * DP + 4 * gl);
      }
      GNPC_TR_STAMP(0);
      tc::mbar_wait_dbg(&p.full[r % NS], (r / NS) & 1, 3, it);
      GNPC_TR_STAMP(1);
      if constexpr (C::TW) {
        // training strip windows: the group's two rows are samples k0, k0 + 1
        // of one node; each entry names a neighbour node's block (bs rows) in
        // the three windows laid end to end (slot stride WINB), so its rows
        // are at wbase + node * bs * 128 + (k0 + j) * 128, swizzled by row
        const int ST = (npt + 1 + 7) & ~7;
        const int Kt = use_sched ? sch_k[it] : __ldg(a.tw_k + tile);
        const uint16_t* st16 = reinterpret_cast<const uint16_t*>(slot + C::O_TWS);
        const uint16_t* ri = st16 + ST;
        const float* vv = reinterpret_cast<const float*>(slot + C::O_TWS + 2 * ST + 2 * Kt);
        const int v0 = row0 + R * gid;
        const int ln = (v0 >> lbs) - tile * npt, k0 = v0 & (bs - 1);
        const int e0 = st16[ln], e1 = v0 < n ? st16[ln + 1] : e0;
        const uint32_t nb = static_cast<uint32_t>(bs) * DP * 4;
        const uint32_t wlim = wring0 + C::NWIN * C::WINB, wring = C::NWIN * C::WINB;
        uint32_t off[R];
#pragma unroll
        for (int j = 0; j < R; ++j)
          off[j] = (k0 + j) * (DP * 4) + ((gl ^ ((k0 + j) & 7)) << 4);
        for (int e = e0; e < e1; ++e) {
          uint32_t b0 = wbase + ri[e] * nb;
          b0 = b0 >= wlim ? b0 - wring : b0;
          const float w = vv[e];
#pragma unroll
          for (int j = 0; j < R; ++j) fma4(acc[j], w, tc::lds4(b0 + off[j]));
        }
      } else if constexpr (TR) {
        // virtual row v = node*bs + k gathers X rows (col*bs + k) of node's
        // neighbours: one staged (col, val) list serves the node's bs rows
        const int n0 = tile * npt;
        const int* rpt = reinterpret_cast<const int*>(slot + C::O_RP) + (n0 & 3);
        const int kb = rpt[0], ke = rpt[min(npt, nodes - n0)];
        const int a0 = kb & ~3;
        const bool st = ((ke + 3) & ~3) - a0 <= C::CAPC;
        int sj[R], lj[R], self[R];
        const char* xbj[R];
#pragma unroll
        for (int j = 0; j < R; ++j) {
          const int v = row0 + R * gid + j;
          // bs divides 128: a power of two (shift/mask, no integer division)
          const int vv = min(v, n - 1), node = vv >> lbs, k = vv & (bs - 1);
          const int ln = node - n0;
          const int e0 = rpt[ln], e1 = rpt[ln + 1];
          sj[j] = st ? e0 - a0 : e0;
          lj[j] = v < n ? e1 - e0 : 0;
          self[j] = node;
          xbj[j] = reinterpret_cast<const char*>(X + static_cast<size_t>(k) * DP + 4 * gl);
        }
        const unsigned long long stride = static_cast<unsigned long long>(bs) * DP * 4;
        const int* cis = st ? reinterpret_cast<const int*>(slot + C::O_CI) : a.ci;
        const float* vs = st ? reinterpret_cast<const float*>(slot + C::O_V) : a.v;
        if (bs % R == 0)  // the group's rows: consecutive samples of one node
          gather_csr_node<DP, R, C::USC>(xbj[0], stride, cis, vs, sj[0], lj[0], self[0], acc);
        else
          gather_csr_rows<DP, R, C::USC>(xbj, stride, cis, vs, sj, lj, self, acc, pol_keep);
      } else if constexpr (CSR == 1) {
        const int* rpt = reinterpret_cast<const int*>(slot + C::O_RP);
        const int kb = rpt[0], ke = rpt[min(TM, n - row0)];
        const int a0 = kb & ~3;
        const bool st = ((ke + 3) & ~3) - a0 <= C::CAPC;
        int sj[R], lj[R], self[R];
        const char* xbj[R];
#pragma unroll
        for (int j = 0; j < R; ++j) {
          const int rr = R * gid + j;
          const int e0 = rpt[rr], e1 = rpt[rr + 1];
          sj[j] = st ? e0 - a0 : e0;
          lj[j] = row0 + rr < n ? e1 - e0 : 0;
          self[j] = min(row0 + rr, n - 1);
          xbj[j] = reinterpret_cast<const char*>(X + 4 * gl);
        }
        if (st)
          gather_csr_rows<DP, R, C::USC>(xbj, DP * 4ull, reinterpret_cast<const int*>(slot + C::O_CI),
                                         reinterpret_cast<const float*>(slot + C::O_V), sj, lj, self, acc,
                                         pol_keep);
        else
          gather_csr_rows<DP, R, C::USC>(xbj, DP * 4ull, a.cis, a.vs, sj, lj, self, acc, pol_keep);
      } else {
        if constexpr (C::PW) {
          // (a second, wrap-free instance of the gather for the 3 tiles in 5
          // whose windows do not wrap measured slower: C5 layer 331 vs 326 us)
          if constexpr (R == 2)
            gather_pw_rows<C::NG, true>(slot, K, gid, gl, wbase, wring0 + C::NWIN * C::WINB, C::NWIN * C::WINB,
                                        acc);
        } else if constexpr (C::PAIR) {
          if (staged)
            gather_pair_rows<DP, C::US, C::NG, true>(X, gl, reinterpret_cast<const int4*>(slot + C::OPB), K, gid,
                                                     acc, pol_keep);
          else
            gather_pair_rows<DP, C::US, C::NG, false>(X, gl, a.psell + __ldg(a.psell_off + tile), K, gid, acc,
                                                      pol_keep);
        } else if (staged)
          gather_sell_rows<DP, R, C::US, TM, true>(X, gl, reinterpret_cast<const int2*>(slot + C::OPB), K,
                                                   gid, acc, pol_keep);
        else
          gather_sell_rows<DP, R, C::US, TM, false>(X, gl, a.sell + __ldg(a.sell_off + tile), K, gid, acc,
                                                    pol_keep);
      }
    }

    GNPC_TR_STAMP(2);
    // ------------------------------------------- epilogue of the previous tile
    bool proj = false;
    if (it >= 1 && it - 1 < my_tiles) proj = epilogue(it - 1);
    if (TCP && it == my_tiles + 2)  // every warp's last partials are written
      asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory");
    if (TCP && it >= 2 && it - 2 < my_tiles) proj_epilogue(it - 2);
    if (TCP && it >= 3 && it - 3 < my_tiles) proj_final(it - 3);
    if constexpr (C::EARLY) {  // TMEM read for epilogue(it-1): the control warp may issue into it
      if (it >= 1 && it - 1 < my_tiles) {
        __syncwarp();
        if (lane == 0) mbar_arrive(p.efull);
      }
    }

    GNPC_TR_STAMP(4);
    // ---------------------------------------------------------------- split
    if (have) {
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const int rr = R * gid + j;
        const uint32_t o = tc::swz_off<DP>(rr, 4 * gl);
        *reinterpret_cast<float4*>(p.A + o) = acc[j];
        *reinterpret_cast<float4*>(p.A + C::OPB + o) = f4_trunc_lo(acc[j]);
      }
      // X_lo into TMEM, one row per lane: warp (lane quarter q, column group
      // cq) takes columns [cq CW, cq CW + CW) of rows 32q + lane
      {
        constexpr int CW = DP / NQ;
        const int q = warp & 3, cq = warp >> 2, m = 32 * q + lane;
        const uint8_t* xtile = slot;
        if constexpr (C::WINS) xtile = wtile;
        float lo[CW];
#pragma unroll
        for (int c = 0; c < CW; c += 4) {
          const float4 xl = f4_trunc_lo(*reinterpret_cast<const float4*>(xtile + tc::swz_off<DP>(m, cq * CW + c)));
          lo[c] = xl.x;
          lo[c + 1] = xl.y;
          lo[c + 2] = xl.z;
          lo[c + 3] = xl.w;
        }
        const uint32_t ta = p.tmem + C::alo_col(TCP) + (static_cast<uint32_t>(32 * q) << 16) + cq * CW;
        if constexpr (CW == 4) tc::tmem_st4(ta, lo);
        else tc::tmem_st8(ta, lo);
        tc::tmem_wait_st();
        tc::fence_before();
      }
    }
    GNPC_TR_STAMP(5);
    if (it <= my_tiles) arrive();
    GNPC_TR_STAMP(6);
    if (proj) project(tile_at(it - 1) * TM);
  }
}

// One layer as its own launch (norm/lift/layers pipeline of ApplyLaunch).
template <int DP, bool LAST, typename OutT, int CSR = 0>
__global__ void __launch_bounds__(SellCfg<DP, CSR>::NT, 1)
k_layer_sell(DevCsr a, const __grid_constant__ SellMaps maps, const float* __restrict__ X,
             const float* __restrict__ axlong, const float* __restrict__ uwp, NetView net,
             const ApplyScalars* __restrict__ sc, OutT* __restrict__ out, const int* __restrict__ skip) {
  if (skip && *skip) return;
  if (sc->zero) {
    if constexpr (LAST) {
      for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += gridDim.x * blockDim.x)
        out[i] = OutT(0);
    }
    return;
  }
  auto p = sell_setup<DP, CSR>(net.hidden, LAST);
  sell_layer<DP, LAST, OutT, CSR>(p, a, &maps.x, &maps.y, X, axlong, uwp, net, sc->out_scale, out, nullptr,
                                  &maps.xw);
  sell_teardown(p);
}

// The first layer with the lift fused in (CSR = 9): no layer input in HBM.
template <int DP, typename OutT>
__global__ void __launch_bounds__(SellCfg<DP, 9>::NT, 1)
k_layer_sell_lift(DevCsr a, const __grid_constant__ SellMaps maps, const void* __restrict__ in, int in_f64,
                  const float* __restrict__ uwp, NetView net, const ApplyScalars* __restrict__ sc,
                  const int* __restrict__ skip) {
  if (skip && *skip) return;
  if (sc->zero) return;  // the last layer writes M(0) = 0
  auto p = sell_setup<DP, 9>(net.hidden, false);
  const LiftIO lio{in, in_f64, sc};
  sell_layer<DP, false, OutT, 9>(p, a, &maps.x, &maps.y, nullptr, nullptr, uwp, net, sc->out_scale, nullptr, nullptr,
                                 &maps.xw, &lio);
  sell_teardown(p);
}

// Training layer (CSR = 2): KIND 1 forward (Y = relu(XU + ÂXW), ÂX stored
// for the weight gradients), KIND 2 backward over Âᵀ with [Uᵀ; Wᵀ]
// (G_in = [X_l > 0] ⊙ (G U^T + Âᵀ G W^T), unmasked for layer 0).  The bs
// samples of a node are adjacent virtual rows; bs must divide 128.
struct TrainMaps {
  CUtensorMap x, y, ax, mask;
  CUtensorMap xw;  // the gathered input, box {DP, 128 + 2 bs} (training strip windows)
};

template <int DP, int KIND, int CSR = 2>
__global__ void __launch_bounds__(SellCfg<DP, CSR>::NT, 1)
k_train_sell(DevCsr a, const __grid_constant__ TrainMaps maps, const float* __restrict__ X,
             const float* __restrict__ uwp, NetView net, int bs, int use_mask,
             const uint32_t* __restrict__ mask_in, uint8_t* __restrict__ mask_out) {
  auto p = sell_setup<DP, CSR>(net.hidden, false);
  const TrainIO tio{&maps.ax, &maps.mask, bs, KIND == 2 ? use_mask : 0, mask_in, mask_out,
                    KIND == 1 && (use_mask & 2) ? 1 : 0};
  sell_layer<DP, false, float, CSR, KIND>(p, a, &maps.x, &maps.y, X, nullptr, uwp, net, 1.0, nullptr, &tio,
                                          &maps.xw);
  sell_teardown(p);
}

// ---------------------------------------------------------------------------
// The whole apply M(b) in one persistent launch (one CTA per SM, cooperative
// so all CTAs are resident): τ = ‖b‖ (f64 block partials, every CTA sums them
// in the same order), the piecewise-linear lift into X[0], then the L layers,
// with a grid barrier after each phase.  Replaces the 2 + L launches of
// ApplyLaunch for matrices without long rows (src/gnn.cpp:120-201).
struct ApplyFused {
  CUtensorMap x0, x1;           // TMA maps over X[0], X[1]
  CUtensorMap x0w, x1w;         // the same with the strip windows' box (unused at d = 16)
  float* X0;
  float* X1;
  const float* uwp;             // [L][4 DP DP] B operands
  double* partials;             // [gridDim.x]
  unsigned long long* gbar;     // grid-barrier counter (monotonic)
  unsigned long long gbase;     // its value when this launch started
  ApplyScalars* sc;             // τ and scales (written by block 0 for callers)
  unsigned long long* times;    // debug (GNPC_FUSED_TIMES): block 0 phase timestamps, or null
  void* stash;                  // optional device copy of the input (InT[n]): when `in` is host
                                // memory read zero-copy, the norm pass stores it for the lift
};

__device__ __forceinline__ void grid_barrier(unsigned long long* ctr, unsigned long long target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1ull);
    unsigned long long v;
    do {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
      if (v < target) __nanosleep(64);
    } while (v < target);
    __threadfence();  // gpu-scope: invalidates this SM's L1 before re-reading X
  }
  __syncthreads();
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

template <int DP, typename InT, typename OutT, int CSR>
__global__ void __launch_bounds__(SellCfg<DP>::NT, 1)
k_apply_sell(DevCsr a, const __grid_constant__ ApplyFused f, const InT* __restrict__ in, NetView net,
             OutT* __restrict__ out, const int* __restrict__ skip) {
  using C = SellCfg<DP, CSR>;
  // every exit consumes all 1 + L grid-barrier arrivals of this launch so
  // the monotonic counter stays in step with the host's base for the next one
  if (skip && *skip) {
    if (threadIdx.x == 0) atomicAdd(f.gbar, static_cast<unsigned long long>(1 + net.layers));
    return;
  }
  const int n = a.n;
  const int tid = threadIdx.x;
  unsigned long long target = f.gbase;
  int tk = 0;
  auto stamp = [&]() {
    if (f.times && blockIdx.x == 0 && threadIdx.x == 0) f.times[tk] = globaltimer_ns();
    ++tk;
  };
  stamp();
  // ------------------------------------------------------------ τ = ‖b‖₂
  __shared__ double red[32];
  __shared__ double s_scale[2];
  {
    double s = 0.0;
    InT* stash = static_cast<InT*>(f.stash);
    for (int i = blockIdx.x * C::NT + tid; i < n; i += gridDim.x * C::NT) {
      const InT v = in[i];
      if (stash) stash[i] = v;
      const double x = static_cast<double>(v);
      s = fma(x, x, s);
    }
    s = warp_sum(s);
    if ((tid & 31) == 0) red[tid >> 5] = s;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < C::NT / 32; ++w) t += red[w];
      f.partials[blockIdx.x] = t;
    }
    target += gridDim.x;
    grid_barrier(f.gbar, target);
    if (tid < 32) {  // every CTA folds the partials the same way: lane-strided, then a fixed tree
      double t = 0.0;
      for (int b = tid; b < (int)gridDim.x; b += 32) t += reinterpret_cast<volatile double*>(f.partials)[b];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (tid == 0) {
      const double tau = sqrt(t);
      const double sn = sqrt(static_cast<double>(n));
      s_scale[0] = tau == 0.0 ? 0.0 : sn / tau;
      s_scale[1] = tau / sn;
      if (blockIdx.x == 0) {
        f.sc->tau = tau;
        f.sc->zero = tau == 0.0;
        f.sc->in_scale = s_scale[0];
        f.sc->out_scale = s_scale[1];
      }
      }
    }
    __syncthreads();
  }
  const double in_scale = s_scale[0], out_scale = s_scale[1];
  if (in_scale == 0.0) {  // τ = 0: M(0) = 0
    for (int i = blockIdx.x * C::NT + tid; i < n; i += gridDim.x * C::NT) out[i] = OutT(0);
    if (tid == 0) atomicAdd(f.gbar, static_cast<unsigned long long>(net.layers));  // skipped barriers
    return;
  }
  auto p = sell_setup<DP, CSR>(net.hidden, true);
  // ------------------------------------------- lift into X[0] (own tiles' rows)
  {
    const int nb = net.nbreak;
    float* s_a = reinterpret_cast<float*>(p.ring);  // ring is idle until the first layer
    float* s_b = s_a + (nb + 1) * DP;
    float* s_t = s_b + (nb + 1) * DP;
    for (int t = tid; t < (nb + 1) * DP; t += C::NT) {
      s_a[t] = net.lift_a[t];
      s_b[t] = net.lift_b[t];
    }
    for (int t = tid; t < nb; t += C::NT) s_t[t] = net.lift_t[t];
    __syncthreads();
    constexpr int G = DP / 4;
    const int gl = tid % G;
    const int ntiles = (n + C::TM - 1) / C::TM;
    const InT* src = f.stash ? static_cast<const InT*>(f.stash) : in;
    // a thread's rows of up to LT of this CTA's tiles at once: their input
    // loads are in flight together (one tile per pass left the load latency
    // exposed 14 times per apply at C2)
    constexpr int LT = 8;
    for (int r = tid / G; r < C::TM; r += C::NT / G)
    for (int t0 = blockIdx.x; t0 < ntiles; t0 += LT * gridDim.x) {
      float v[LT];
#pragma unroll
      for (int k = 0; k < LT; ++k) {
        const int row = (t0 + k * gridDim.x) * C::TM + r;
        // (length-sorted nodes: row i of the pipeline is node perm[i] of b)
        v[k] = row < n ? static_cast<float>(in_scale * static_cast<double>(src[a.perm ? a.perm[row] : row])) : 0.f;
      }
#pragma unroll
      for (int k = 0; k < LT; ++k) {
        const int row = (t0 + k * gridDim.x) * C::TM + r;
        if (row >= n) continue;
        int lo = 0, hi = nb;  // interval = #kinks <= v
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (s_t[mid] <= v[k]) lo = mid + 1;
          else hi = mid;
        }
        const float4 al = *reinterpret_cast<const float4*>(s_a + lo * DP + 4 * gl);
        const float4 be = *reinterpret_cast<const float4*>(s_b + lo * DP + 4 * gl);
        st4(f.X0 + static_cast<size_t>(row) * DP + 4 * gl,
            make_float4(fmaf(al.x, v[k], be.x), fmaf(al.y, v[k], be.y), fmaf(al.z, v[k], be.z),
                        fmaf(al.w, v[k], be.w)));
      }
    }
    __syncthreads();
    for (int t = tid; t < (2 * (nb + 1) * DP + nb + 3) / 4; t += C::NT)  // restore the zeroed ring
      reinterpret_cast<float4*>(p.ring)[t] = f4zero();
  }
  const int L = net.layers;
  for (int l = 0; l < L; ++l) {
    stamp();
    target += gridDim.x;
    grid_barrier(f.gbar, target);  // layer l's input is complete everywhere
    stamp();
    const float* X = (l & 1) ? f.X1 : f.X0;
    const CUtensorMap* mx = (l & 1) ? &f.x1 : &f.x0;
    const CUtensorMap* my = (l & 1) ? &f.x0 : &f.x1;
    const CUtensorMap* mxw = (l & 1) ? &f.x1w : &f.x0w;
    const float* uw = f.uwp + (size_t)l * 4 * DP * DP;
    if (l + 1 < L)
      sell_layer<DP, false, OutT, CSR>(p, a, mx, my, X, nullptr, uw, net, out_scale, out, nullptr, mxw);
    else
      sell_layer<DP, true, OutT, CSR>(p, a, mx, my, X, nullptr, uw, net, out_scale, out, nullptr, mxw);
  }
  stamp();
  sell_teardown(p);
}

}  // namespace gnpk
