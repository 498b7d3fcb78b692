// Shared device helpers for the sm_100a GNP kernels.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace gnpk {

constexpr int kThreads = 256;     // CTA size used by the streaming kernels
#ifndef GNPC_LONGROW
#define GNPC_LONGROW 32
#endif
constexpr int kLongRow = GNPC_LONGROW;  // rows with more nonzeros take the long-row path

// Device view of Â (or Âᵀ): int32 indices (nnz < 2^31 enforced on upload),
// fp32 values.  long_rows lists the rows with > kLongRow nonzeros.
struct DevCsr {
  int n;
  int nnz;
  const int* __restrict__ rp;
  const int* __restrict__ ci;
  const float* __restrict__ v;
  const int* __restrict__ long_rows;
  int n_long;
  // Apply path on ragged matrices: nodes renumbered by row length; perm[i] =
  // the original index of node i (nullptr: natural order).  With it rp / ci /
  // v and every apply layout below are in the renumbered order.
  const int* __restrict__ perm;
  // Sliced-ELL copy (128-row slices, entry (r, k) of slice t at
  // sell_off[t] + k*128 + r, padding (row, 0.0)); nullptr when the matrix's
  // row lengths are too ragged for it.  sell_k[t] = K_t | (has long row) << 16.
  const int2* __restrict__ sell;
  const int* __restrict__ sell_off;
  const int* __restrict__ sell_k;
  // Short-row CSR (rows with > kLongRow nonzeros emptied; they take the
  // chunked long-row path), padded for 16-byte bulk copies: rps has n+1+132
  // entries (tail = nnz_short), cis/vs nnz_short+4.  tflag[t] = 1 if the
  // 128-row tile t holds a long row.  Aliases the full CSR when n_long == 0.
  const int* __restrict__ rps;
  const int* __restrict__ cis;
  const float* __restrict__ vs;
  const int* __restrict__ tflag;
  // Pair-union sliced-ELL (d = 32 apply, stencil-like matrices without long
  // rows): the two adjacent rows (2g, 2g+1) of a 128-row tile share one entry
  // list, the sorted union of their columns, with one weight per row (0 where
  // a row lacks the column).  Entry (k, g) of tile t at psell_off[t] + 64k + g
  // as {col, w0 bits, w1 bits, 0}; padding {2g, 0, 0, 0}.  psell_k[t] = K_t
  // (union entries of the tile's longest pair).  Each X row the pair shares is
  // gathered once (9-point stencil: 12 loads per pair instead of 18).
  const int4* __restrict__ psell;
  const int* __restrict__ psell_off;
  const int* __restrict__ psell_k;
  // Strip-window pair-union layout (d = 32 apply; stencil-like matrices whose
  // off-tile columns sit at one dominant tile stride S): tiles run in strips
  // t = s0 + S k (pw_order, chunked per CTA) and tile u gathers only from the
  // row windows of tiles u - S, u, u + S, staged in shared memory by TMA (one
  // new window per tile along a strip).  Per tile, the slice at byte
  // 16 pw_off[t] holds K = pw_k[t] (a multiple of 4) pair-union entries per
  // row pair as structure-of-arrays over the 64 pairs: uint16 idx[64][K]
  // (window w in bits 8-9, row within the window in bits 0-7), float
  // w0[64][K], float w1[64][K] (10 bytes per entry).
  const uint8_t* __restrict__ pw;
  const int* __restrict__ pw_off;
  const int* __restrict__ pw_k;
  const int* __restrict__ pw_order;
  int pw_S;
  // Training strip windows (batched layers, bs samples per node, npt = 128/bs
  // nodes per tile): tiles in strips of tw_S (tw_order); tile u gathers from
  // the node windows of tiles u - S, u, u + S extended by one node (npt + 2
  // nodes).  Slice at byte 16 tw_off[t]: uint16 starts[ST] (ST = npt+1
  // rounded to 8: each node's first entry), uint16 node[K] (index in the
  // three windows laid end to end, npt + 2 nodes each), float val[K];
  // K = tw_k[t] (entries rounded to 8).
  const uint8_t* __restrict__ tw;
  const int* __restrict__ tw_off;
  const int* __restrict__ tw_k;
  const int* __restrict__ tw_order;
  int tw_S;
  // L2 policy: 1 = the streamed matrix (slices, CSR ranges) is loaded
  // evict_first and the X-row gathers evict_last, so the layer input stays
  // L2-resident while Â streams past it; 0 = evict_normal everywhere.
  int l2hint;
};
// Row windows of the strip-ordered window mode (d = 32): a window of tile u is
// rows [128u - kPwHalo, 128u + 128 + kPwHalo), one TMA box of kPwRows rows.
constexpr int kPwHalo = 8, kPwRows = 128 + 2 * kPwHalo;
// training strip windows: entries per tile (rounded to 8), window rows max (bs <= 32)
constexpr int kTwKcap = 48, kTwRowsMax = 128 + 2 * 32;

// Per-apply scalars produced by the norm kernel (scale sandwich,
// src/gnn.cpp:128-139,191-199).
struct ApplyScalars {
  double tau;        // ||b||_2
  double in_scale;   // sqrt(n)/tau
  double out_scale;  // tau/sqrt(n)
  int zero;          // tau == 0 → M(b) = 0
  int pad;
};

// ---- device FGMRES state (kernels in krylov.cuh)
struct KState {
  int j;             // next step within the cycle
  int steps;         // completed steps in the cycle
  int stop;          // cycle finished (all later step kernels are no-ops)
  int cycle;         // steps planned for this cycle
  int breakdown;
  int budget_hit;
  int budget_status; // 1 maxiters, 2 timeout
  int iter;          // outer iterations so far (all cycles)
  int maxiters;
  int singular;
  int reorth;        // steps that took the re-orthogonalisation pass
  int pad;
  double rtol, bnorm, beta;
  double tracked_rel;  // after the last step
  double current;      // true relres after the cycle
  long long t0;        // globaltimer at solve start (ns)
  long long deadline;  // < 0: no timeout
  long long t_end;     // globaltimer when the cycle's true residual was formed
};

struct KrylovDev {
  int n, m;                 // restart length m
  double* V;                // n x (m+1)
  double* Z;                // n x m, or nullptr (unpreconditioned: Z = V)
  double* w;                // n
  double* vin;              // n: next preconditioner input (= v_j)
  const double* zout;       // n: preconditioner output z_j
  double* x;                // n
  const double* b;          // n
  double* r;                // n
  double* H;                // (m+1) x m raw Hessenberg, col-major
  double* R;                // (m+1) x m rotated
  double* cs;               // m
  double* sn;               // m
  double* g;                // m+1
  double* y;                // m
  double* partials;         // 2 x grid
  unsigned* ticket;
  double* hist_rel;         // m per cycle
  long long* hist_t;        // m per cycle
  KState* st;
};

__device__ __forceinline__ float4 ldg4(const float* p) {
  return __ldg(reinterpret_cast<const float4*>(p));
}
// L2 cache policies (createpolicy) and a 128-bit read-only load under one.
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_normal() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ int ldg_hint(const int* p, uint64_t pol) {
  int v;
  asm("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float ldg_hint(const float* p, uint64_t pol) {
  float v;
  asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float4 ldg4_hint(const float* p, uint64_t pol) {
  float4 v;
  asm("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
__device__ __forceinline__ float4 f4zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }
__device__ __forceinline__ void fma4(float4& acc, float s, float4 x) {
  acc.x = fmaf(s, x.x, acc.x);
  acc.y = fmaf(s, x.y, acc.y);
  acc.z = fmaf(s, x.z, acc.z);
  acc.w = fmaf(s, x.w, acc.w);
}
__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__device__ __forceinline__ float relu(float x) { return x > 0.f ? x : 0.f; }
__device__ __forceinline__ float4 relu4(float4 a) {
  return make_float4(relu(a.x), relu(a.y), relu(a.z), relu(a.w));
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block sum (fixed shuffle tree + fixed smem order).  All
// threads receive the total.  `scratch` >= 32 entries.
template <typename T>
__device__ __forceinline__ T block_sum(T v, T* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  T t = lane < nw ? scratch[lane] : T(0);
  t = warp_sum(t);
  return t;
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

}  // namespace gnpk
