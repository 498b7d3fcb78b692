// Fused Res-GCONV layer with the dense transform on the 5th-gen tensor cores.
//
//   Y = relu([X | ÂX] · [U; W])          (src/gnn.cpp:164-176)
//
// Persistent CTAs walk 128-row tiles in a software pipeline:
//   stage   : the NEXT tile's row_ptr slice and (col, val) range are loaded
//             into registers while the current tile gathers, then parked in
//             a double-buffered smem slot (coalesced, off the critical path);
//   gather  : G = DP/4 lanes per row; each group streams all of its R rows at
//             once, U nonzeros per row per round (R*U independent 128-bit
//             X-row loads in flight per lane), fp32 sums in stored order;
//   epilogue: of the PREVIOUS tile, overlapping its MMA with this gather:
//             tcgen05.ld of the TMEM accumulator (warp w owns lanes
//             32(w%4)..+31; warps w, w+4 split the columns), relu, store Y;
//             LAST: the projection MLP (src/gnn.cpp:178-199) per row;
//   MMA     : [x | ÂX] split into tf32 hi + lo, written in the K-major
//             core-matrix layout; one thread issues 3 x (2DP/8)
//             tcgen05.mma.kind::tf32 (M=128, N=DP, K=8):
//             A_lo·B_hi + A_hi·B_lo + A_hi·B_hi ("3xTF32", ~2^-21 relative per
//             product) into TMEM, committed to an mbarrier.
// [U; W] arrives pre-split (hi/lo) and pre-laid-out by the host (capi.cu).
#pragma once

#include "apply.cuh"
#include "tc.cuh"

namespace gnpk {

template <int DP>
struct TcCfg {
  static constexpr int TM = 128;
  static constexpr int K = 2 * DP;
  static constexpr int KC = K / 4;  // 16-byte chunks per operand row
  static constexpr int KS = K / 8;  // MMA K-steps (8 tf32 per instruction)
  static constexpr int G = DP / 4;
  static constexpr int NG = kThreads / G;
  static constexpr int R = TM / NG;                // rows per gather group
  static constexpr int U = DP == 16 ? 4 : 2;       // nonzeros per row per gather round
  static constexpr int US = DP == 16 ? 7 : 3;      // same, sliced-ELL path (no bounds state)
  static constexpr int CAP = 1536;                 // staged (col, val) entries per tile
  static constexpr int CPT = CAP / kThreads;       // staged entries per thread
  static constexpr int TCOLS = DP < 32 ? 32 : DP;  // TMEM columns (power of two >= 32)
  static constexpr int SST = DP + 4;               // LAST staging row stride (floats)
  static constexpr int RPS = TM + 4;               // staged row_ptr slot
  static constexpr size_t A_FLOATS = (size_t)TM * K;
  static constexpr size_t B_FLOATS = (size_t)DP * K;
  static size_t smem_bytes(bool last, int hidden) {
    size_t f = 2 * A_FLOATS + 2 * B_FLOATS + 2 * (size_t)RPS + 4 * (size_t)CAP;
    if (last) f += (size_t)TM * SST + (size_t)DP * hidden + 2 * (size_t)hidden + 2 * TM;
    return f * 4 + 64 + 1024;  // + mbarrier / tmem slot + 1024-B atom alignment
  }
};

// One group's R rows, U nonzeros per row per round: (col, val) for all R*U
// slots first, then all R*U 128-bit X-row loads, then the FMAs in stored
// column order — so every round keeps R*U independent loads in flight.
// Slots past a row's end read a clamped in-range entry (a real neighbour of
// the tile, so the X row is in bounds) with weight 0: acc + 0*x == acc, and
// no predicated loads or register zeroing sit on the issue path.
template <int DP, int R, int U, typename LD>
__device__ __forceinline__ void gather_rounds(const char* const (&xb)[R], long long rowbytes,
                                              LD load, int last, int (&pos)[R],
                                              const int (&end)[R], float4 (&acc)[R]) {
  while (true) {
    bool more = false;
#pragma unroll
    for (int j = 0; j < R; ++j) more |= pos[j] < end[j];
    if (!more) break;
    int c[R][U];
    float w[R][U];
#pragma unroll
    for (int j = 0; j < R; ++j)
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = pos[j] + u;
        load(min(k, last), c[j][u], w[j][u]);
        w[j][u] = k < end[j] ? w[j][u] : 0.f;
      }
    float4 x[R][U];
#pragma unroll
    for (int j = 0; j < R; ++j)
#pragma unroll
      for (int u = 0; u < U; ++u)
        x[j][u] = ldg4(reinterpret_cast<const float*>(xb[j] + c[j][u] * rowbytes));
#pragma unroll
    for (int j = 0; j < R; ++j) {
#pragma unroll
      for (int u = 0; u < U; ++u) fma4(acc[j], w[j][u], x[j][u]);
      pos[j] += U;
    }
  }
}

// Sliced-ELL gather: every row of the tile has K entries (padding carries
// weight 0 and the row's own column), so the rounds need no bounds checks.
template <int DP, int R, int U, int TM, int NG>
__device__ __forceinline__ void gather_sell(const char* const (&xb)[R], const int2* cv, int K,
                                           int gid, float4 (&acc)[R]) {
  // rounds of U entries; the last round's missing slots are warp-uniformly
  // predicated off, so a tile costs ceil(K/U) dependent load latencies
  for (int k = 0; k < K; k += U) {
    int c[R][U];
    float w[R][U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool on = k + u < K;
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const int2 e = on ? cv[(k + u) * TM + gid + j * NG] : make_int2(0, 0);
        c[j][u] = e.x;
        w[j][u] = __int_as_float(e.y);
      }
    }
    float4 x[R][U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool on = k + u < K;
#pragma unroll
      for (int j = 0; j < R; ++j)
        x[j][u] = on ? ldg4(reinterpret_cast<const float*>(xb[j] + static_cast<long long>(c[j][u]) * (DP * 4)))
                     : f4zero();
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int j = 0; j < R; ++j) fma4(acc[j], w[j][u], x[j][u]);
  }
}

// tf32 hi/lo split by truncation: hi keeps the top 10 mantissa bits, lo = x -
// hi is exact in fp32; the tensor core reads lo's top 10 bits, so the split
// loses < 2^-21 |x| (two integer/fp ops instead of cvt.rna's emulation).
__device__ __forceinline__ void tf32_split(float4 v, float4& hi, float4& lo) {
  hi = make_float4(__int_as_float(__float_as_int(v.x) & 0xffffe000),
                   __int_as_float(__float_as_int(v.y) & 0xffffe000),
                   __int_as_float(__float_as_int(v.z) & 0xffffe000),
                   __int_as_float(__float_as_int(v.w) & 0xffffe000));
  lo = make_float4(v.x - hi.x, v.y - hi.y, v.z - hi.z, v.w - hi.w);
}

// Epilogue modes: relu (forward layer), LAST (forward layer + projection MLP),
// MASK (backward: D ⊙ [mask > 0], identity when mask == nullptr).
enum { kEpiRelu = 0, kEpiLast = 1, kEpiMask = 2 };

// Virtual rows: the GEMM row v = node * bs + k (bs = batch samples resident
// per node, 1 for an apply); a row gathers X rows (col * bs + k) of the
// neighbours of `node`, so one Â row serves all bs samples of the batch.
struct LayerIO {
  const float* X;      // [nodes * bs][DP]
  float* Y;            // [nodes * bs][DP]
  const float* uwtc;   // this layer's pre-split swizzled B operand
  const float* axlong; // bs == 1 only: (ÂX) of long rows
  float* axout;        // optional: (ÂX) rows written out (training forward)
  const float* mask;   // kEpiMask: multiply by [mask > 0]
  int bs;
  int dbg;             // timing experiments only (GNPC_LAYER_DBG): 1 no gather, 2 no MMA, 4 no store
};

// PATH: kPathCsr (any bs), kPathCsr1 (bs == 1, the apply path: node ==
// virtual row), kPathSell (bs == 1, sliced-ELL staging; a.sell required).
enum { kPathCsr = 0, kPathCsr1 = 1, kPathSell = 2 };
template <int DP, int MODE, typename OutT, int PATH = kPathCsr>
__global__ void __launch_bounds__(kThreads, 2)
k_layer_tc(DevCsr a, LayerIO io, NetView net, const ApplyScalars* __restrict__ sc,
           OutT* __restrict__ out, const int* __restrict__ skip) {
  using C = TcCfg<DP>;
  constexpr bool LAST = MODE == kEpiLast;
  constexpr int TM = C::TM, KC = C::KC, KS = C::KS, G = C::G, NG = C::NG, R = C::R;
  constexpr int U = C::U, CAP = C::CAP, CPT = C::CPT, RPS = C::RPS;
  if (skip && *skip) return;
  const float* __restrict__ X = io.X;
  float* __restrict__ Y = io.Y;
  const float* __restrict__ axlong = io.axlong;
  constexpr bool BS1 = PATH != kPathCsr;
  const int bs = BS1 ? 1 : io.bs;
  const int nv = a.n * bs;  // virtual rows
  const int ntiles = (nv + TM - 1) / TM;
  if (sc && sc->zero) {
    if constexpr (LAST) {
      for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += gridDim.x * blockDim.x)
        out[i] = OutT(0);
    }
    return;
  }
  (void)KC;
  // Swizzle atoms need 1024-B alignment in the shared window; pointers are
  // derived from the __shared__ array so they stay in the shared state space.
  extern __shared__ float4 smem_raw[];
  const uint32_t pad = (1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u;
  float* Ahi = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(smem_raw) + pad);
  float* Alo = Ahi + C::A_FLOATS;
  float* Bhi = Alo + C::A_FLOATS;
  float* Blo = Bhi + C::B_FLOATS;
  int* s_rp = reinterpret_cast<int*>(Blo + C::B_FLOATS);  // [2][RPS]
  int2* s_cv = reinterpret_cast<int2*>(s_rp + 2 * RPS);    // [2][CAP] (col, val bits)
  float* Stg = reinterpret_cast<float*>(s_cv + 2 * CAP);   // LAST: [TM][SST]
  float* D1 = Stg + (LAST ? TM * C::SST : 0);              // LAST: [DP][H]
  float* B1 = D1 + (LAST ? DP * net.hidden : 0);
  float* D2 = B1 + (LAST ? net.hidden : 0);
  float* Part = D2 + (LAST ? net.hidden : 0);              // LAST: [2][TM]
  uint64_t* bar = reinterpret_cast<uint64_t*>(Part + (LAST ? 2 * TM : 0) + 4);
  uint64_t* fullb = bar + 1;  // SELL staging barriers [2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 3);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int t = tid; t < int(2 * C::B_FLOATS / 4); t += kThreads)
    reinterpret_cast<float4*>(Bhi)[t] = reinterpret_cast<const float4*>(io.uwtc)[t];
  if constexpr (LAST) {
    const int H = net.hidden;
    for (int t = tid; t < DP * H; t += kThreads) D1[t] = net.dec1[t];
    for (int t = tid; t < H; t += kThreads) {
      B1[t] = net.dec1_b[t];
      D2[t] = net.dec2[t];
    }
  }
  // sliced-ELL staging: one bulk copy per tile (thread 0), completion on fullb
  constexpr bool sell = PATH == kPathSell;
  auto sell_issue = [&](int t, int sl) {
    if (t >= ntiles) return;
    const int K = __ldg(a.sell_k + t) & 0xffff;
    if (K == 0 || K * TM > CAP) return;
    tc::mbar_expect_tx(&fullb[sl], K * TM * 8);
    tc::bulk_load(s_cv + sl * CAP, a.sell + __ldg(a.sell_off + t), K * TM * 8, &fullb[sl]);
  };
  if (tid == 0) {
    tc::mbar_init(bar, 1);
    tc::mbar_init(&fullb[0], 1);
    tc::mbar_init(&fullb[1], 1);
  }
  if (warp == 0) tc::tmem_alloc(tslot, C::TCOLS);

  // ---- staging of a tile's row_ptr slice + (col, val) range (two halves so
  //      the loads can be issued early and the smem stores done late)
  struct Stage {
    int rp;            // row_ptr[n0 + tid] for the tile's nodes n0..n1
    int kb, ke;        // the tile's nonzero range
    int c[CPT];
    float v[CPT];
  };
  auto stage_rp = [&](int tile, Stage& s) {
    if (tile >= ntiles) return;
    const int row0 = tile * TM;
    const int n0 = row0 / bs, n1 = min((row0 + TM - 1) / bs + 1, a.n);
    if (tid <= TM) s.rp = __ldg(a.rp + min(n0 + tid, n1));
    s.kb = __ldg(a.rp + n0);
    s.ke = __ldg(a.rp + n1);
  };
  auto stage_cv = [&](int tile, Stage& s) {
    if (tile >= ntiles || s.ke - s.kb > CAP) return;
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
      const int k = s.kb + tid + q * kThreads;
      if (k < s.ke) {
        s.c[q] = __ldg(a.ci + k);
        s.v[q] = __ldg(a.v + k);
      }
    }
  };
  auto stage_store = [&](int tile, const Stage& s, int slot) {
    if (tile >= ntiles) return;
    if (tid <= TM) s_rp[slot * RPS + tid] = s.rp;
    if (tid == 0) {
      s_rp[slot * RPS + TM + 2] = s.kb;
      s_rp[slot * RPS + TM + 3] = s.ke;
    }
    if (s.ke - s.kb > CAP) return;
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
      const int k = tid + q * kThreads;
      if (s.kb + k < s.ke) s_cv[slot * CAP + k] = make_int2(s.c[q], __float_as_int(s.v[q]));
    }
  };

  int tile = blockIdx.x;
  if constexpr (!sell) {
    Stage s0;
    stage_rp(tile, s0);
    stage_cv(tile, s0);
    stage_store(tile, s0, 0);
  }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (sell && tid == 0) sell_issue(tile, 0);
  uint32_t fph = 0;  // SELL barrier phases (bit per slot)
  const uint32_t tmem = *tslot;
  constexpr uint32_t idesc = tc::idesc_tf32(128, DP);
  const uint32_t sAhi = tc::smem_u32(Ahi), sAlo = tc::smem_u32(Alo);
  const uint32_t sBhi = tc::smem_u32(Bhi), sBlo = tc::smem_u32(Blo);
  const int gl = tid % G, gid = tid / G;
  uint32_t phase = 0;
  int slot = 0;
  int prev_row0 = -1;  // tile whose MMA is in flight

  // ---- epilogue of the tile whose accumulator sits in TMEM
  auto epilogue = [&](int row0) {
    if (io.dbg & 2) return;
    tc::mbar_wait(bar, phase);
    phase ^= 1;
    tc::fence_after();
    constexpr int HC = DP / 2;  // columns per warp half
    const int q = warp & 3, half = warp >> 2;
    const int m = 32 * q + lane;
    const int i = row0 + m;
    float v[HC];
    const uint32_t taddr = tmem + (static_cast<uint32_t>(32 * q) << 16) + half * HC;
    if constexpr (HC == 8) {
      tc::tmem_ld8(taddr, v);
    } else {
      tc::tmem_ld16(taddr, v);
    }
    if constexpr (MODE == kEpiRelu) {
      if (i < nv && !(io.dbg & 4)) {
        float* yrow = Y + static_cast<size_t>(i) * DP + half * HC;
#pragma unroll
        for (int c = 0; c < HC; c += 4)
          st4(yrow + c, make_float4(relu(v[c]), relu(v[c + 1]), relu(v[c + 2]), relu(v[c + 3])));
      }
    } else if constexpr (MODE == kEpiMask) {
      if (i < nv) {
        float* yrow = Y + static_cast<size_t>(i) * DP + half * HC;
        const float* mrow = io.mask ? io.mask + static_cast<size_t>(i) * DP + half * HC : nullptr;
#pragma unroll
        for (int c = 0; c < HC; c += 4) {
          float4 o = make_float4(v[c], v[c + 1], v[c + 2], v[c + 3]);
          if (mrow) {
            const float4 mk = ldg4(mrow + c);
            o.x = mk.x > 0.f ? o.x : 0.f;
            o.y = mk.y > 0.f ? o.y : 0.f;
            o.z = mk.z > 0.f ? o.z : 0.f;
            o.w = mk.w > 0.f ? o.w : 0.f;
          }
          st4(yrow + c, o);
        }
      }
    } else {
#pragma unroll
      for (int c = 0; c < HC; c += 4)
        st4(Stg + m * C::SST + half * HC + c,
            make_float4(relu(v[c]), relu(v[c + 1]), relu(v[c + 2]), relu(v[c + 3])));
    }
    tc::fence_before();
  };
  // LAST: projection MLP of the staged tile (after a barrier)
  // two threads per row, each owning half of the hidden units; dec1 read as
  // warp-uniform float4 broadcasts (4 hidden units per smem wavefront)
  auto project = [&](int row0) {
    if constexpr (LAST) {
      const int H = net.hidden;
      const int r = tid % TM, part = tid / TM;
      const int h0 = part * (H / 2), h1 = part ? H : H / 2;
      float y[DP];
#pragma unroll
      for (int j = 0; j < DP; j += 4) {
        const float4 t = *reinterpret_cast<const float4*>(Stg + r * C::SST + j);
        y[j] = t.x; y[j + 1] = t.y; y[j + 2] = t.z; y[j + 3] = t.w;
      }
      float o = 0.f;
      int h = h0;
      for (; (H & 7) == 0 && h + 4 <= h1; h += 4) {  // float4-aligned dec1 columns
        float4 t = f4zero();
#pragma unroll
        for (int j = 0; j < DP; ++j) fma4(t, y[j], *reinterpret_cast<const float4*>(D1 + j * H + h));
        o = fmaf(relu(t.x + B1[h]), D2[h], o);
        o = fmaf(relu(t.y + B1[h + 1]), D2[h + 1], o);
        o = fmaf(relu(t.z + B1[h + 2]), D2[h + 2], o);
        o = fmaf(relu(t.w + B1[h + 3]), D2[h + 3], o);
      }
      for (; h < h1; ++h) {
        float t = 0.f;
#pragma unroll
        for (int j = 0; j < DP; ++j) t = fmaf(y[j], D1[j * H + h], t);
        o = fmaf(relu(t + B1[h]), D2[h], o);
      }
      Part[part * TM + r] = o;
      __syncthreads();
      if (tid < TM) {
        const int i = row0 + tid;
        if (i < a.n)
          out[i] = static_cast<OutT>(static_cast<double>(Part[tid] + Part[TM + tid] + net.dec2_b) *
                                     sc->out_scale);
      }
    }
  };

  for (; tile < ntiles; tile += gridDim.x) {
    const int row0 = tile * TM;
    const int next = tile + gridDim.x;
    Stage sn;
    float4 acc[R], xs[R];
    if constexpr (sell) {
      // ------------------------------------------------------ gather (SELL)
      if (tid == 0) sell_issue(next, slot ^ 1);  // slot^1 was released by the last barrier
      const int kw = __ldg(a.sell_k + tile);
      const int K = kw & 0xffff;
      const bool staged = K > 0 && K * TM <= CAP;
      const int2* cv = staged ? s_cv + slot * CAP : a.sell + __ldg(a.sell_off + tile);
      const char* xb[R];
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const int i = row0 + gid + j * NG;
        const bool valid = i < nv;
        xb[j] = reinterpret_cast<const char*>(X + 4 * gl);
        acc[j] = f4zero();
        if ((kw >> 16) && valid && __ldg(a.rp + i + 1) - __ldg(a.rp + i) > kLongRow)
          acc[j] = ldg4(axlong + static_cast<size_t>(i) * DP + 4 * gl);
      }
      if (staged) {
        tc::mbar_wait(&fullb[slot], (fph >> slot) & 1);
        fph ^= 1u << slot;
      }
      if (!(io.dbg & 1)) gather_sell<DP, R, C::US, TM, NG>(xb, cv, K, gid, acc);
      // own rows after the gather (registers go to the gather's loads; for
      // stencil-like rows the own row was just gathered and sits in L1)
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const int i = row0 + gid + j * NG;
        xs[j] = (i < nv && !(io.dbg & 16)) ? ldg4(X + static_cast<size_t>(i) * DP + 4 * gl) : f4zero();
      }
    } else {
    stage_rp(next, sn);  // loads only; consumed at the end of the iteration

    // ---------------------------------------------------------------- gather
    const int* rp = s_rp + slot * RPS;
    const int kb = rp[TM + 2], ke = rp[TM + 3];
    const bool staged = ke - kb <= CAP;
    const int n0 = row0 / bs;
    {
      int pos[R], end[R];
      const char* xb[R];
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const int r = gid + j * NG;
        const int i = row0 + r;  // virtual row
        const bool valid = i < nv;
        const int node = valid ? i / bs : n0;
        const int kk = i - node * bs;
        xb[j] = reinterpret_cast<const char*>(X + static_cast<size_t>(kk) * DP + 4 * gl);
        const int s = rp[node - n0], e = rp[node - n0 + 1];
        const bool longrow = axlong != nullptr && e - s > kLongRow;
        pos[j] = s;
        end[j] = (valid && !longrow) ? e : s;
        acc[j] = (valid && longrow) ? ldg4(axlong + static_cast<size_t>(i) * DP + 4 * gl) : f4zero();
        xs[j] = valid ? ldg4(X + static_cast<size_t>(i) * DP + 4 * gl) : f4zero();
      }
      const long long rowbytes = static_cast<long long>(bs) * DP * 4;
      if (staged) {
#pragma unroll
        for (int j = 0; j < R; ++j) {
          pos[j] -= kb;
          end[j] -= kb;
        }
        const int2* cv = s_cv + slot * CAP;
        gather_rounds<DP, R, U>(
            xb, rowbytes,
            [cv](int k, int& c, float& w) {
              const int2 e = cv[k];
              c = e.x;
              w = __int_as_float(e.y);
            },
            ke - kb - 1, pos, end, acc);
      } else {
        gather_rounds<DP, R, U>(
            xb, rowbytes,
            [&a](int k, int& c, float& w) {
              c = __ldg(a.ci + k);
              w = __ldg(a.v + k);
            },
            ke - 1, pos, end, acc);
      }
      if (io.axout != nullptr) {
#pragma unroll
        for (int j = 0; j < R; ++j) {
          const int i = row0 + gid + j * NG;
          if (i < nv) st4(io.axout + static_cast<size_t>(i) * DP + 4 * gl, acc[j]);
        }
      }
    }
    stage_cv(next, sn);
    }

    // ------------------------------------------------ previous tile: epilogue
    if (prev_row0 >= 0) epilogue(prev_row0);

    // ------------------------------------------------ A tile, staging, barrier
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const int r = gid + j * NG;
      const float4 xi = xs[j], ax = acc[j];
      float4 xh, xl, ah, al;
      tf32_split(xi, xh, xl);
      tf32_split(ax, ah, al);
      if (io.dbg & 8) continue;
      const uint32_t ox = tc::sw128_off(r, 4 * gl, TM), oa = tc::sw128_off(r, DP + 4 * gl, TM);
      *reinterpret_cast<float4*>(reinterpret_cast<uint8_t*>(Ahi) + ox) = xh;
      *reinterpret_cast<float4*>(reinterpret_cast<uint8_t*>(Alo) + ox) = xl;
      *reinterpret_cast<float4*>(reinterpret_cast<uint8_t*>(Ahi) + oa) = ah;
      *reinterpret_cast<float4*>(reinterpret_cast<uint8_t*>(Alo) + oa) = al;
    }
    if constexpr (!sell) stage_store(next, sn, slot ^ 1);
    tc::fence_proxy_async();
    __syncthreads();

    if constexpr (LAST) {
      if (prev_row0 >= 0) {
        project(prev_row0);
        __syncthreads();  // Stg is rewritten by the next epilogue
      }
    }

    // ---------------------------------------------------------------- MMA
    if (tid == 0 && !(io.dbg & 2)) {
      tc::fence_after();
      uint32_t accf = 0;
#pragma unroll
      for (int pass = 0; pass < 3; ++pass) {
        const uint32_t sa = pass == 0 ? sAlo : sAhi;
        const uint32_t sb = pass == 1 ? sBlo : sBhi;
#pragma unroll
        for (int s = 0; s < KS; ++s) {
          // K-step s: atom s/4 (atom-major along K), +32 B per step inside it
          const uint64_t ad = tc::make_desc_sw128(sa + (s >> 2) * TM * 128 + (s & 3) * 32, 1024);
          const uint64_t bd = tc::make_desc_sw128(sb + (s >> 2) * DP * 128 + (s & 3) * 32, 1024);
          tc::mma_tf32(tmem, ad, bd, idesc, accf);
          accf = 1;
        }
      }
      tc::mma_commit(bar);
    }
    prev_row0 = row0;
    slot ^= 1;
  }
  if (prev_row0 >= 0) {
    epilogue(prev_row0);
    if constexpr (LAST) {
      __syncthreads();
      project(prev_row0);
    }
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 0) tc::tmem_dealloc(tmem, C::TCOLS);
}

}  // namespace gnpk
