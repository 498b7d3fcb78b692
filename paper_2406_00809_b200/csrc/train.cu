// Batched GNP training: C ABI entry points (include/gnpc.h, "training").
//
// One step = forward over the B resident samples ([n][B][d] activations),
// L1 residual loss and its Âᵀ gradient, backward through decoder / layers /
// encoder, deterministic weight-gradient reductions, f64 Adam on the flat
// parameter vector, then the fp32 device parameters and tcgen05 operands are
// regenerated on the GPU from the f64 master copy.  Restates
// src/gnn.cpp:208-451 (train_preconditioner's step body) with τ treated as a
// constant of b (SPEC) exactly like the reference.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <chrono>
#include <condition_variable>
#include <exception>
#include <future>
#include <thread>
#include <memory>
#include <mutex>
#include <vector>

#include "capi_common.hpp"
#include "kernels/layer_sell.cuh"
#include "kernels/layer_tc.cuh"
#include "kernels/train.cuh"
#include "kernels/decoder_tc.cuh"
#include "kernels/wgrad_tc.cuh"
#include "kernels/pairs.cuh"
#include "host/pair_stream.hpp"
#include "model.hpp"

using namespace gnpc_impl;

struct gnpc_trainer_s {
  gnpc_model_s* m = nullptr;
  std::unique_ptr<gnpc_csr_s> At;  // Âᵀ (explicit transpose, src/csr.cpp:108-125)
  int B = 0, n = 0, nv = 0, dp = 0, d = 0, H = 0, L = 0;
  double lr = 1e-3;
  std::int64_t t = 0;
  std::int64_t P = 0;
  bool tc = false;
  // forward-only trainer (the monitoring batch of train_preconditioner): the
  // TMA layers skip the ÂX and mask-word stores only a backward would read
  bool fwd_only = false;
  int sms = 0;
  cudaStream_t s = nullptr;
  // flat f64 master parameters, gradient, Adam moments
  DevBuf<double> p64, g64, m1, m2;
  // regeneration maps (see gnpc_model_s::build_maps)
  DevBuf<int> map_view, map_bt_fwd, map_bt_bwd, map_tc_fwd, map_tc_bwd;
  DevBuf<unsigned char> part_tc, part_pair;
  DevBuf<int> map_tc_pair, map_tc_pair_bwd;
  DevBuf<float> BT_fwd, BT_bwd, UWTC_bwd, UWP_bwd;
  // TMA pipeline layers (k_train_sell): maps over the activation and
  // gradient buffers, used when the batch divides the 128-row tile
  bool sell = false;
  std::vector<CUtensorMap> mX, mAX;
  // [X_l > 0] bits of the layer outputs (d = 32: one 32-bit word per row,
  // rows padded to the 128-row tile), written by forward layer l-1 and read
  // by backward layer l instead of the X_l tile
  DevBuf<uint32_t> mbits;
  std::size_t nvpad = 0;
  CUtensorMap mG[2]{};
  // training strip windows (d = 32, DevCsr::tw on Â and Âᵀ): window maps
  // (box 128 + 2B rows) over the gathered inputs X_l (forward) and G (backward)
  bool tw = false;
  std::vector<CUtensorMap> mXw;
  CUtensorMap mGw[2]{};
  // batch
  DevBuf<double> xb, bb, out, sgn, gout, colpart, losspart, tmp;
  // host-batch steps: x is uploaded on a copy stream while the forward runs
  // on b (x is first read by the loss)
  DevBuf<double> tmp2;
  cudaStream_t cs = nullptr;
  cudaEvent_t ev_b = nullptr, ev_x = nullptr;
  ~gnpc_trainer_s() {
    if (ev_b) cudaEventDestroy(ev_b);
    if (ev_x) cudaEventDestroy(ev_x);
    if (cs) cudaStreamDestroy(cs);
  }
  DevBuf<gnpk::SampleScales> scl;
  // activations
  DevBuf<float> Xs, AXs, G[2], vv, hb1, hb2, gyv;
  // reductions
  struct Red {
    gnpk::OuterArgs o;
    DevBuf<int> dst;
    int P4 = 0, Q2 = 0;
    bool tc = false;       // tcgen05 path (k_wgrad_tc): partial layout [64][32]
    gnpk::WgradArgs w{};
    bool tma = false;      // TMA-fed variant (k_wgrad_tma) with its tensor maps
    const float* tma_b = nullptr;
    gnpk::WgradTmaArgs ta{};
    bool colsum = false;   // one-column reduction (k_weighted_colsum)
    const float* cs_A = nullptr;
    const float* cs_w = nullptr;
    int cs_W = 0, cs_nv = 0;
  };
  int colsum_grid = 0;
  int wgrad_grid = 0, wgrad_grid_tma = 0;
  Red red_layer[64], red_dec1, red_dec2, red_enc2, red_enc1;
  DevBuf<double> opart;
  int rowblk = 0;
  int tc_per_sm_fwd = 0, tc_per_sm_bwd = 0;
  int loss_grid = 0;
  std::int64_t nbytes_act = 0;
  // piecewise-linear encoder (H <= 64): tables regenerated on device after
  // every parameter update; backward by per-interval sums (k_enc_buckets)
  bool pw = false;
  DevBuf<float> lt, la, lb;
  DevBuf<unsigned long long> lact;
  DevBuf<int> lnb;
  DevBuf<double> encpart;
  gnpk::LiftTab tab{};
  gnpk::EncOff eoff{};
  int enc_grid = 0, enc_warps = 16, enc_rpb = 0;
  // tensor-core decoder (d = hidden = 32 on the TMA maps): dec2 / dec2_b
  // per-CTA sums folded by k_outer_finish through dec_dst
  bool dec_tc = false;
  int dec_grid = 0, dec_grid_bwd = 0;
  DevBuf<double> decpart, decwpart;
  DevBuf<int> dec_dst;
};

namespace {

constexpr int kTh = gnpk::kThreads;

int grid_for(std::int64_t work, int per_block, int cap) {
  return (int)std::max<std::int64_t>(1, std::min<std::int64_t>((work + per_block - 1) / per_block, cap));
}

void upload_i(DevBuf<int>& b, const std::vector<int>& v) {
  if (!v.empty()) b.upload(v.data(), v.size());
}

// Build one reduction: A = [A1 | A2 | ones], B = Bm, dst map from (p, q).
template <class F>
void make_red(gnpc_trainer_s::Red& r, const float* A1, int P1, int s1, const float* A2, int P2,
              int s2, int ones, const float* Bm, int Q, int sq, int nv, F dstfn) {
  r.o = gnpk::OuterArgs{A1, P1, s1, A2, P2, s2, ones, Bm, Q, sq, nv, nullptr};
  r.P4 = gnpk::outer_P4(r.o);
  r.Q2 = gnpk::outer_Q2(r.o);
  std::vector<int> dst((std::size_t)r.P4 * r.Q2, -1);
  for (int p = 0; p < r.P4; ++p)
    for (int q = 0; q < r.Q2; ++q) dst[(std::size_t)p * r.Q2 + q] = dstfn(p, q);
  upload_i(r.dst, dst);
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link).
// raise a kernel's dynamic shared-memory limit once per (kernel, size)
void set_smem_once(const void* kern, size_t bytes) { set_smem_attr(kern, (int)bytes); }

// [nv][32] fp32 rows viewed as a 2-D tensor, box {32 features, 128 rows}, 128B swizzle.
CUtensorMap rows32_map(const float* base, int nv) {
  return make_rows_map(base, nv, 32, 128, CU_TENSOR_MAP_SWIZZLE_128B);
}

// tcgen05 reduction: A = [A1 | A2 or ones] (<= 32 features each), B (<= 32),
// dst map over the [64][32] partial (m < 32: A1 feature, m >= 32: A2 / bias).
template <class F>
void make_red_tc(gnpc_trainer_s::Red& r, const float* A1, int wa1, int sa1, const float* A2, int wa2,
                 int sa2, int ones, const float* Bm, int wb, int sb, int nv, F dstfn) {
  r.tc = true;
  r.w = gnpk::WgradArgs{A1, wa1, sa1, A2, wa2, sa2, ones, Bm, wb, sb, nv, nullptr};
  r.P4 = 64;
  r.Q2 = 32;
  std::vector<int> dst(64 * 32, -1);
  for (int m = 0; m < 64; ++m)
    for (int q = 0; q < 32; ++q) dst[m * 32 + q] = dstfn(m, q);
  upload_i(r.dst, dst);
}

// one-column reduction (k_weighted_colsum): dst over [out1(32) | out2(32) | out3]
template <class F>
void make_red_colsum(gnpc_trainer_s::Red& r, const float* A, int W, const float* w, int nv, F dstfn) {
  r.colsum = true;
  r.cs_A = A;
  r.cs_W = W;
  r.cs_w = w;
  r.cs_nv = nv;
  std::vector<int> dst(96, -1);
  for (int i = 0; i < 96; ++i) dst[i] = dstfn(i);
  upload_i(r.dst, dst);
}

void run_red(gnpc_trainer_s& T, gnpc_trainer_s::Red& r) {
  if (r.colsum) {
    gnpk::k_weighted_colsum<<<T.colsum_grid, kTh, 0, T.s>>>(r.cs_A, r.cs_W, r.cs_w, r.cs_nv, T.opart.p);
    GNPC_LAUNCHED();
    gnpk::k_outer_finish<<<1, 96, 0, T.s>>>(T.opart.p, T.colsum_grid, 96, r.dst.p, T.g64.p);
    GNPC_LAUNCHED();
    return;
  }
  if (r.tc && r.w.wa1 == 32 && r.w.sa1 == 32 && r.w.wb == 32 && r.w.sb == 32 &&
      (r.w.ones || !r.w.A2 || (r.w.wa2 == 32 && r.w.sa2 == 32))) {
    // TMA-fed variant (32-float rows); tensor maps re-encoded when Bm moves
    const float* Bm = r.o.Bm ? r.o.Bm : r.w.Bm;
    if (!r.tma || r.tma_b != Bm) {
      r.ta.a1 = rows32_map(r.w.A1, r.w.nv);
      r.ta.a2 = r.w.A2 ? rows32_map(r.w.A2, r.w.nv) : r.ta.a1;
      r.ta.a2_mode = r.w.ones ? 2 : (r.w.A2 ? 1 : 0);
      r.ta.b = rows32_map(Bm, r.w.nv);
      r.ta.nv = r.w.nv;
      r.tma = true;
      r.tma_b = Bm;
    }
    r.ta.partials = T.opart.p;
    static const bool tf32 = [] {
      const char* e = std::getenv("GNPC_WGRAD_TF32");
      return e && std::string(e) == "1";
    }();
    if (tf32)
      gnpk::k_wgrad_tma<<<T.wgrad_grid_tma, gnpk::wgt::TH, gnpk::wgt::smem_bytes(), T.s>>>(r.ta);
    else
      gnpk::k_wgrad_bf16<<<T.wgrad_grid_tma, gnpk::wgb::TH, gnpk::wgb::smem_bytes(), T.s>>>(r.ta);
    GNPC_LAUNCHED();
    gnpk::k_outer_finish<<<(64 * 32 + kTh - 1) / kTh, kTh, 0, T.s>>>(T.opart.p, T.wgrad_grid_tma,
                                                                   64 * 32, r.dst.p, T.g64.p);
    GNPC_LAUNCHED();
    return;
  }
  if (r.tc) {
    r.w.partials = T.opart.p;
    r.w.Bm = r.o.Bm ? r.o.Bm : r.w.Bm;
    gnpk::k_wgrad_tc<<<T.wgrad_grid, kTh, gnpk::wg::smem_bytes(), T.s>>>(r.w);
    GNPC_LAUNCHED();
    gnpk::k_outer_finish<<<(64 * 32 + kTh - 1) / kTh, kTh, 0, T.s>>>(T.opart.p, T.wgrad_grid, 64 * 32,
                                                                   r.dst.p, T.g64.p);
    GNPC_LAUNCHED();
    return;
  }
  r.o.partials = T.opart.p;
  const int nblocks = (r.P4 / 4) * (r.Q2 / 2);
  dim3 grid(T.rowblk, (nblocks + kTh - 1) / kTh);
  const size_t smem = (size_t)(32 * r.P4 + 32 * r.Q2) * 4;
  gnpk::k_outer_sum<<<grid, kTh, smem, T.s>>>(r.o);
  GNPC_LAUNCHED();
  const int PQ = r.P4 * r.Q2;
  gnpk::k_outer_finish<<<(PQ + kTh - 1) / kTh, kTh, 0, T.s>>>(T.opart.p, T.rowblk, PQ, r.dst.p,
                                                              T.g64.p);
  GNPC_LAUNCHED();
}

// fp32 device params + layer operands from the f64 master copy
void regenerate(gnpc_trainer_s& T) {
  gnpc_model_s& m = *T.m;
  const int nview = (int)m.map_view.size();
  gnpk::k_gather_params<<<(nview + kTh - 1) / kTh, kTh, 0, T.s>>>(T.p64.p, T.map_view.p, nview, m.P.p);
  GNPC_LAUNCHED();
  if (T.tc) {
    const int c = (int)m.map_tc_fwd.size();
    gnpk::k_gather_split<<<(c + kTh - 1) / kTh, kTh, 0, T.s>>>(T.p64.p, T.map_tc_fwd.p, T.part_tc.p, c,
                                                               m.UWTC.p);
    GNPC_LAUNCHED();
    gnpk::k_gather_split<<<(c + kTh - 1) / kTh, kTh, 0, T.s>>>(T.p64.p, T.map_tc_bwd.p, T.part_tc.p, c,
                                                               T.UWTC_bwd.p);
    GNPC_LAUNCHED();
    if (T.sell) {
      gnpk::k_gather_split<<<(c + kTh - 1) / kTh, kTh, 0, T.s>>>(T.p64.p, T.map_tc_pair_bwd.p, T.part_pair.p,
                                                                 c, T.UWP_bwd.p);
      GNPC_LAUNCHED();
    }
    gnpk::k_gather_split<<<(c + kTh - 1) / kTh, kTh, 0, T.s>>>(T.p64.p, T.map_tc_pair.p, T.part_pair.p, c,
                                                               m.UWP.p);
    GNPC_LAUNCHED();
  } else {
    const int c = (int)m.map_bt_fwd.size();
    gnpk::k_gather_params<<<(c + kTh - 1) / kTh, kTh, 0, T.s>>>(T.p64.p, T.map_bt_fwd.p, c, T.BT_fwd.p);
    GNPC_LAUNCHED();
    gnpk::k_gather_params<<<(c + kTh - 1) / kTh, kTh, 0, T.s>>>(T.p64.p, T.map_bt_bwd.p, c, T.BT_bwd.p);
    GNPC_LAUNCHED();
  }
  if (T.pw) {
    const size_t smem = (size_t)T.H * T.d * 8;
    set_smem_once((const void*)gnpk::k_lift_tables, smem);
    gnpk::k_lift_tables<<<1, 256, smem, T.s>>>(T.p64.p, T.eoff, T.dp, T.tab);
    GNPC_LAUNCHED();
  }
}

template <int DP>
struct TrainLaunch {
  // one Res-GCONV layer over the B-sample batch: forward (relu, ÂX out) or
  // backward data gradient (over Âᵀ, [Uᵀ; Wᵀ], mask by the layer input)
  // in/out: buffer ids for the TMA maps (fwd: X = Xs[l] -> Xs[l+1], ÂX -> AXs[l];
  // bwd: G[gi] -> G[1-gi], mask Xs[l])
  static void layer(gnpc_trainer_s& T, bool fwd, int l, const float* X, float* Y, float* axout,
                    const float* mask, int gi = 0) {
    gnpc_csr_s& A = fwd ? *T.m->a : *T.At;
    gnpk::DevCsr a = A.dev();
    if constexpr (DP == 16 || DP == 32) {
      if constexpr (DP == 32) {
        if (T.tw) {  // strip windows: the gathered rows staged by TMA along strips
          A.bind_tw(T.B, a);
          using S = gnpk::SellCfg<32, 10>;
          const size_t smem = S::smem_bytes(T.H, false);
          auto kern = fwd ? gnpk::k_train_sell<32, 1, 10> : gnpk::k_train_sell<32, 2, 10>;
          set_smem_once((const void*)kern, smem);
          const int tiles = (T.nv + S::TM - 1) / S::TM;
          const int grid = std::max(1, std::min(tiles, T.sms));
          gnpk::TrainMaps maps;
          if (fwd) {
            maps.x = T.mX[l];
            maps.y = T.mX[l + 1];
            maps.ax = T.mAX[l];
            maps.mask = T.mX[l];
            maps.xw = T.mXw[l];
          } else {
            maps.x = T.mG[gi];
            maps.y = T.mG[1 - gi];
            maps.ax = T.mG[gi];
            maps.mask = T.mX[l];
            maps.xw = T.mGw[gi];
          }
          const float* uwp = (fwd ? T.m->UWP.p : T.UWP_bwd.p) + (size_t)l * 4 * DP * DP;
          const uint32_t* min_ = nullptr;
          uint8_t* mout = nullptr;
          if (fwd && l + 1 <= T.L - 1 && !T.fwd_only)
            mout = reinterpret_cast<uint8_t*>(T.mbits.p + (size_t)(l + 1) * T.nvpad);
          if (!fwd && mask != nullptr) min_ = T.mbits.p + (size_t)l * T.nvpad;
          // (forward: bit 1 of the mask argument = no ÂX store)
          kern<<<grid, S::NT, smem, T.s>>>(a, maps, X, uwp, T.m->view, T.B,
                                           fwd ? (T.fwd_only ? 2 : 0) : (mask != nullptr ? 1 : 0), min_, mout);
          GNPC_LAUNCHED();
          return;
        }
      }
      if (T.sell) {
        using S = gnpk::SellCfg<DP, 2>;
        const size_t smem = S::smem_bytes(T.H, false);
        auto kern = fwd ? gnpk::k_train_sell<DP, 1> : gnpk::k_train_sell<DP, 2>;
        set_smem_once((const void*)kern, smem);
        const int tiles = (T.nv + S::TM - 1) / S::TM;
        const int grid = std::max(1, std::min(tiles, T.sms));
        gnpk::TrainMaps maps;
        if (fwd) {
          maps.x = T.mX[l];
          maps.y = T.mX[l + 1];
          maps.ax = T.mAX[l];
          maps.mask = T.mX[l];
        } else {
          maps.x = T.mG[gi];
          maps.y = T.mG[1 - gi];
          maps.ax = T.mG[gi];
          maps.mask = T.mX[l];
        }
        const float* uwp = (fwd ? T.m->UWP.p : T.UWP_bwd.p) + (size_t)l * 4 * DP * DP;
        const uint32_t* min_ = nullptr;
        uint8_t* mout = nullptr;
        if (T.mbits.p) {
          if (fwd && l + 1 <= T.L - 1 && !T.fwd_only)
            mout = reinterpret_cast<uint8_t*>(T.mbits.p + (size_t)(l + 1) * T.nvpad);
          if (!fwd && mask != nullptr) min_ = T.mbits.p + (size_t)l * T.nvpad;
        }
        kern<<<grid, S::NT, smem, T.s>>>(a, maps, X, uwp, T.m->view, T.B,
                                         fwd ? (T.fwd_only ? 2 : 0) : (mask != nullptr ? 1 : 0), min_, mout);
        GNPC_LAUNCHED();
        return;
      }
      if (T.tc) {
        using C = gnpk::TcCfg<DP>;
        const float* uw = (fwd ? T.m->UWTC.p : T.UWTC_bwd.p) + (size_t)l * 2 * C::B_FLOATS;
        auto kern = fwd ? gnpk::k_layer_tc<DP, gnpk::kEpiRelu, float>
                        : gnpk::k_layer_tc<DP, gnpk::kEpiMask, float>;
        const size_t smem = C::smem_bytes(false, T.H);
        int& per_sm = fwd ? T.tc_per_sm_fwd : T.tc_per_sm_bwd;
        if (per_sm == 0) per_sm = tc_ctas_per_sm((const void*)kern, smem, C::TCOLS);
        const int tiles = (T.nv + C::TM - 1) / C::TM;
        const int grid = std::max(1, std::min(tiles, per_sm * T.sms));
        gnpk::LayerIO io{X, Y, uw, nullptr, axout, mask, T.B};
        kern<<<grid, kTh, smem, T.s>>>(a, io, T.m->view, nullptr, (float*)nullptr, nullptr);
        GNPC_LAUNCHED();
        return;
      }
    }
    const float* bt = (fwd ? T.BT_fwd.p : T.BT_bwd.p) + (size_t)l * DP * 2 * DP;
    const int grid = grid_for((std::int64_t)T.nv, kTh / DP, T.sms * 8);
    if (fwd)
      gnpk::k_layer_batched<DP, 0><<<grid, kTh, 0, T.s>>>(a, X, Y, bt, axout, mask, T.B);
    else
      gnpk::k_layer_batched<DP, 2><<<grid, kTh, 0, T.s>>>(a, X, Y, bt, axout, mask, T.B);
    GNPC_LAUNCHED();
  }

  // forward: norms, lift, L layers, decoder -> out (f64 [n][B])
  static void forward(gnpc_trainer_s& T) {
    const gnpk::NetView& net = T.m->view;
    const std::size_t act = (std::size_t)T.nv * DP;
    const int cg = grid_for(T.n, 8, 1024);
    gnpk::k_col_norm_partials<<<cg, kTh, kTh * sizeof(double), T.s>>>(T.bb.p, T.n, T.B, T.colpart.p);
    GNPC_LAUNCHED();
    gnpk::k_col_norm_finish<<<(T.B + 7) / 8, 256, 0, T.s>>>(T.colpart.p, cg, T.n, T.B, T.scl.p);
    GNPC_LAUNCHED();
    if (T.pw) {
      const size_t smem = (size_t)(T.H + 1) * DP * 2 * 4 + 64 * 4;
#ifndef GNPC_LIFT_BPS
#define GNPC_LIFT_BPS 8
#endif
      const int g = grid_for(T.nv, kTh / (DP / 4), T.sms * GNPC_LIFT_BPS);
      gnpk::k_lift_pw_batched<DP><<<g, kTh, smem, T.s>>>(T.bb.p, T.nv, T.B, T.tab, T.H, T.scl.p, T.Xs.p,
                                                          T.vv.p);
      GNPC_LAUNCHED();
    } else {
      const size_t smem = (size_t)T.H * DP * 4 + 2 * (size_t)T.H * 4;
      const int g = grid_for(T.nv, kTh / (DP / 4), T.sms * 8);
      gnpk::k_lift_batched<DP><<<g, kTh, smem, T.s>>>(T.bb.p, T.nv, T.B, net, T.scl.p, T.Xs.p, T.vv.p);
      GNPC_LAUNCHED();
    }
    for (int l = 0; l < T.L; ++l)
      layer(T, true, l, T.Xs.p + l * act, T.Xs.p + (l + 1) * act, T.AXs.p + l * act, nullptr);
    if constexpr (DP == 32) {
      if (T.dec_tc) {
        const size_t smem = gnpk::DecTc<true>::smem_bytes();
        set_smem_once((const void*)gnpk::k_decoder_tc<true>, smem);
        gnpk::k_decoder_tc<true><<<T.dec_grid, gnpk::DecTc<true>::NT, smem, T.s>>>(
            T.mX[T.L], T.Xs.p + T.L * act, T.nv, T.B, net, T.scl.p, nullptr, T.out.p, nullptr, nullptr,
            nullptr);
        GNPC_LAUNCHED();
        return;
      }
    }
    const size_t smem = ((size_t)DP * T.H + 2 * (size_t)T.H + 4 * 32 * (DP + 1)) * 4;
    const int g = grid_for(T.nv, 128, T.sms * 16);
    set_smem_once((const void*)gnpk::k_decoder_fwd<DP>, smem);
    gnpk::k_decoder_fwd<DP><<<g, 128, smem, T.s>>>(T.Xs.p + T.L * act, T.nv, T.B, net, T.scl.p,
                                                   T.out.p);
    GNPC_LAUNCHED();
  }

  static void backward(gnpc_trainer_s& T) {
    const gnpk::NetView& net = T.m->view;
    const std::size_t act = (std::size_t)T.nv * DP;
    GNPC_CUDA(cudaMemsetAsync(T.g64.p, 0, T.P * sizeof(double), T.s));
    bool dec_done = false;
    if constexpr (DP == 32) {
      if (T.dec_tc) {
        const size_t smem = gnpk::DecTc<false>::smem_bytes();
        set_smem_once((const void*)gnpk::k_decoder_tc<false>, smem);
        gnpk::k_decoder_tc<false><<<T.dec_grid_bwd, gnpk::DecTc<false>::NT, smem, T.s>>>(
            T.mX[T.L], T.Xs.p + T.L * act, T.nv, T.B, net, T.scl.p, T.gout.p, nullptr, T.G[0].p, T.decpart.p,
            T.decwpart.p);
        GNPC_LAUNCHED();
        gnpk::k_outer_finish<<<1, 64, 0, T.s>>>(T.decpart.p, T.dec_grid_bwd, 33, T.dec_dst.p, T.g64.p);
        GNPC_LAUNCHED();
        // dec1 / dec1_b from the fused [X_L | 1]ᵀ g_z partials (red_dec1's layout)
        gnpk::k_outer_finish<<<(64 * 32 + kTh - 1) / kTh, kTh, 0, T.s>>>(T.decwpart.p, T.dec_grid_bwd, 64 * 32,
                                                                        T.red_dec1.dst.p, T.g64.p);
        GNPC_LAUNCHED();
        dec_done = true;
      }
    }
    if (!dec_done) {
      const size_t smem = gnpk::mlp_smem_bytes(DP, T.H);
      const int g = grid_for(T.nv, 32 * gnpk::kMlpWarps, T.sms * 16);
      set_smem_once((const void*)gnpk::k_decoder_bwd<DP>, smem);
      gnpk::k_decoder_bwd<DP><<<g, 32 * gnpk::kMlpWarps, smem, T.s>>>(T.Xs.p + T.L * act, T.nv, T.B, net, T.scl.p,
                                                     T.gout.p, T.hb1.p, T.gyv.p, T.hb2.p, T.G[0].p);
      GNPC_LAUNCHED();
    }
    if (!dec_done) {
      run_red(T, T.red_dec2);
      run_red(T, T.red_dec1);
    }
    int cur = 0;
    for (int l = T.L - 1; l >= 0; --l) {
      T.red_layer[l].o.Bm = T.G[cur].p;
      run_red(T, T.red_layer[l]);
      layer(T, false, l, T.G[cur].p, T.G[1 - cur].p, nullptr, l >= 1 ? T.Xs.p + l * act : nullptr, cur);
      cur = 1 - cur;
    }
    if (T.pw) {
      const size_t smem = gnpk::enc_bucket_smem(DP, T.H, T.enc_warps);
      set_smem_once((const void*)gnpk::k_enc_buckets<DP>, smem);
      gnpk::k_enc_buckets<DP><<<T.enc_grid, 32 * T.enc_warps, smem, T.s>>>(T.G[cur].p, T.vv.p, T.nv,
                                                                           T.enc_rpb, T.tab, T.H,
                                                                           T.encpart.p);
      GNPC_LAUNCHED();
      const int per = (T.H + 1) * 2 * DP;
      double* S = T.encpart.p + (size_t)T.enc_grid * per;
      gnpk::k_enc_fold<<<(per + 63) / 64, 64, 0, T.s>>>(T.encpart.p, T.enc_grid, per, S);
      GNPC_LAUNCHED();
      const size_t fs = (size_t)(per + 2 * T.H * T.d) * 8;
      set_smem_once((const void*)gnpk::k_enc_grads, fs);
      gnpk::k_enc_grads<<<1, kTh, fs, T.s>>>(S, DP, T.tab, T.p64.p, T.eoff, T.g64.p);
      GNPC_LAUNCHED();
      return;
    }
    {
      const size_t smem = gnpk::mlp_smem_bytes(DP, T.H);
      const int g = grid_for(T.nv, 32 * gnpk::kMlpWarps, T.sms * 16);
      set_smem_once((const void*)gnpk::k_encoder_bwd<DP>, smem);
      gnpk::k_encoder_bwd<DP><<<g, 32 * gnpk::kMlpWarps, smem, T.s>>>(T.vv.p, T.G[cur].p, T.nv, net, T.hb1.p,
                                                                      T.hb2.p);
      GNPC_LAUNCHED();
    }
    T.red_enc2.o.Bm = T.G[cur].p;
    run_red(T, T.red_enc2);
    run_red(T, T.red_enc1);
  }
};

template <class F>
void dispatch(int dp, F&& f) {
  switch (dp) {
    case 4: f(std::integral_constant<int, 4>{}); break;
    case 8: f(std::integral_constant<int, 8>{}); break;
    case 16: f(std::integral_constant<int, 16>{}); break;
    case 32: f(std::integral_constant<int, 32>{}); break;
    case 64: f(std::integral_constant<int, 64>{}); break;
    default: throw Unsupported("unsupported width");
  }
}

void forward(gnpc_trainer_s& T) {
  dispatch(T.dp, [&](auto c) { TrainLaunch<decltype(c)::value>::forward(T); });
}
void backward(gnpc_trainer_s& T) {
  dispatch(T.dp, [&](auto c) { TrainLaunch<decltype(c)::value>::backward(T); });
}

// loss over the batch (f64, src/gnn.cpp:309-335); also produces gout
double loss_and_grad(gnpc_trainer_s& T, bool want_grad) {
  gnpk::DevCsr a = T.m->a->dev();
  gnpk::k_loss_residual<<<T.loss_grid, kTh, 0, T.s>>>(a, T.B, T.out.p, T.xb.p, T.sgn.p, T.losspart.p);
  GNPC_LAUNCHED();
  if (want_grad) {
    gnpk::DevCsr at = T.At->dev();
    gnpk::k_loss_grad<<<T.loss_grid, kTh, 0, T.s>>>(at, T.B, T.sgn.p, T.gout.p);
    GNPC_LAUNCHED();
  }
  std::vector<double> part(T.loss_grid);
  GNPC_CUDA(cudaMemcpyAsync(part.data(), T.losspart.p, part.size() * 8, cudaMemcpyDeviceToHost, T.s));
  GNPC_CUDA(cudaStreamSynchronize(T.s));
  double acc = 0.0;
  for (double v : part) acc += v;
  return acc / (double)T.B;
}

void adam(gnpc_trainer_s& T) {
  T.t += 1;
  const double bc1 = 1.0 - std::pow(0.9, (double)T.t);
  const double bc2 = 1.0 - std::pow(0.999, (double)T.t);
  gnpk::k_adam<<<(int)((T.P + kTh - 1) / kTh), kTh, 0, T.s>>>(T.p64.p, T.g64.p, T.m1.p, T.m2.p, (int)T.P,
                                                              T.lr, bc1, bc2);
  GNPC_LAUNCHED();
  regenerate(T);
  T.m->trainer_dirty = true;
}

// host n x B column-major f64 -> device [n][B]
void upload_batch(gnpc_trainer_s& T, const double* host, DevBuf<double>& dst) {
  const std::size_t cnt = (std::size_t)T.n * T.B;
  GNPC_CUDA(cudaMemcpyAsync(T.tmp.p, host, cnt * 8, cudaMemcpyHostToDevice, T.s));
  gnpk::k_colmajor_to_nb<<<(int)((cnt + kTh - 1) / kTh), kTh, 0, T.s>>>(T.tmp.p, T.n, T.B, dst.p);
  GNPC_LAUNCHED();
}

void sync_model_params(gnpc_trainer_s& T) {
  GNPC_CUDA(cudaMemcpyAsync(T.m->params.data(), T.p64.p, T.P * 8, cudaMemcpyDeviceToHost, T.s));
  GNPC_CUDA(cudaStreamSynchronize(T.s));
  T.m->build_view();
  T.m->trainer_dirty = false;
}

void need(bool c, const char* msg) {
  if (!c) throw std::invalid_argument(msg);
}

gnpc_trainer_s* create(gnpc_model_s* m, std::int64_t batch, double lr) {
  need(m && batch >= 1, "trainer_create: bad arguments");
  require_device();
  auto T = std::make_unique<gnpc_trainer_s>();
  T->m = m;
  T->B = (int)batch;
  T->lr = lr;
  T->n = (int)m->a->h.n;
  need(T->n >= 1, "trainer_create: empty matrix");
  if ((std::int64_t)T->n * batch >= (std::int64_t(1) << 31))
    throw Unsupported("trainer: n * batch must be < 2^31");
  T->nv = T->n * T->B;
  T->dp = m->dp;
  T->d = (int)m->dims.d;
  T->H = (int)m->dims.hidden;
  T->L = (int)m->dims.layers;
  if (T->L > 64) throw Unsupported("trainer: at most 64 layers");
  T->P = (std::int64_t)m->params.size();
  T->tc = m->use_tc;
  T->sms = num_sms();
  T->s = m->stream;
  m->a->upload();
  T->At = std::make_unique<gnpc_csr_s>();
  T->At->h = gnp_b200::transpose(m->a->h);
  T->At->upload();
  // master params / Adam
  T->p64.upload(m->params.data(), T->P, T->s);
  T->g64.alloc(T->P);
  T->m1.alloc(T->P);
  T->m2.alloc(T->P);
  GNPC_CUDA(cudaMemsetAsync(T->m1.p, 0, T->P * 8, T->s));
  GNPC_CUDA(cudaMemsetAsync(T->m2.p, 0, T->P * 8, T->s));
  m->build_maps();
  upload_i(T->map_view, m->map_view);
  if (T->tc) {
    upload_i(T->map_tc_fwd, m->map_tc_fwd);
    upload_i(T->map_tc_bwd, m->map_tc_bwd);
    T->part_tc.upload(m->part_tc.data(), m->part_tc.size());
    upload_i(T->map_tc_pair, m->map_tc_pair);
    T->part_pair.upload(m->part_pair.data(), m->part_pair.size());
    // TMA pipeline layers when the batch divides the 128-row tile
    static const bool off = [] {
      const char* e = std::getenv("GNPC_NO_TRAIN_SELL");
      return e && std::string(e) == "1";
    }();
    if (!off && 128 % T->B == 0 && (T->dp == 16 || T->dp == 32)) {
      T->sell = true;
      upload_i(T->map_tc_pair_bwd, m->map_tc_pair_bwd);
      T->UWP_bwd.alloc(m->map_tc_pair_bwd.size());
    }
    T->UWTC_bwd.alloc(m->map_tc_bwd.size());
  } else {
    upload_i(T->map_bt_fwd, m->map_bt_fwd);
    upload_i(T->map_bt_bwd, m->map_bt_bwd);
    T->BT_fwd.alloc(m->map_bt_fwd.size());
    T->BT_bwd.alloc(m->map_bt_bwd.size());
  }
  // batch + activations
  const std::size_t nvs = (std::size_t)T->nv, act = nvs * T->dp;
  T->xb.alloc(nvs);
  T->bb.alloc(nvs);
  T->out.alloc(nvs);
  T->sgn.alloc(nvs);
  T->gout.alloc(nvs);
  T->tmp.alloc(nvs);
  T->colpart.alloc((std::size_t)1024 * T->B);
  T->scl.alloc(T->B);
  T->loss_grid = grid_for((std::int64_t)T->n * 32, kTh, T->sms * 8);
  T->losspart.alloc(T->loss_grid + 1);  // + one scratch slot (train_run's step loss)
  T->Xs.alloc(act * (T->L + 1));
  T->AXs.alloc(act * T->L);
  T->G[0].alloc(act);
  T->G[1].alloc(act);
  if (T->sell) {
    const CUtensorMapSwizzle sw = T->dp == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
    for (int l = 0; l <= T->L; ++l) T->mX.push_back(make_rows_map(T->Xs.p + l * act, T->nv, T->dp, 128, sw));
    for (int l = 0; l < T->L; ++l) T->mAX.push_back(make_rows_map(T->AXs.p + l * act, T->nv, T->dp, 128, sw));
    for (int g = 0; g < 2; ++g) T->mG[g] = make_rows_map(T->G[g].p, T->nv, T->dp, 128, sw);
    if (T->dp == 32 && gnpk::SellCfg<32, 10>::MBITS && T->m->a->ensure_tw(T->B) && T->At->ensure_tw(T->B)) {
      T->tw = true;
      const int wr = 128 + 2 * T->B;
      for (int l = 0; l <= T->L; ++l) T->mXw.push_back(make_rows_map(T->Xs.p + l * act, T->nv, T->dp, wr, sw));
      for (int g = 0; g < 2; ++g) T->mGw[g] = make_rows_map(T->G[g].p, T->nv, T->dp, wr, sw);
    }
    if (gnpk::SellCfg<32, 2>::MBITS && T->dp == 32) {
      T->nvpad = ((std::size_t)T->nv + 127) / 128 * 128;
      T->mbits.alloc(T->nvpad * T->L);
      GNPC_CUDA(cudaMemsetAsync(T->mbits.p, 0, T->nvpad * T->L * 4, T->s));
    }
  }
  T->vv.alloc(nvs);
  {
    static const bool off = [] {
      const char* e = std::getenv("GNPC_NO_PW_ENCODER");
      return e && std::string(e) == "1";
    }();
    const gnp_b200::ParamLayout lay = gnp_b200::param_layout(m->dims);
    T->pw = !off && T->H <= 64;
    if (T->pw) {
      const int H = T->H, dp = T->dp;
      T->lt.alloc(64);
      T->la.alloc((std::size_t)(H + 1) * dp);
      T->lb.alloc((std::size_t)(H + 1) * dp);
      T->lact.alloc(H + 1);
      T->lnb.alloc(1);
      T->tab = gnpk::LiftTab{T->lt.p, T->la.p, T->lb.p, T->lact.p, T->lnb.p};
      T->eoff = gnpk::EncOff{(int)lay.enc1, (int)lay.enc1_b, (int)lay.enc2, (int)lay.enc2_b, H, T->d};
      // warps per block: as many as fit the staging ring + accumulator sets
      // (at least 4: a warp walks kEncStg / warps <= 32 rows per stage)
#ifndef GNPC_ENC_WARPS
#define GNPC_ENC_WARPS 8
#endif
      T->enc_warps = GNPC_ENC_WARPS;
      if (gnpk::enc_bucket_smem(dp, H, T->enc_warps) > 220 * 1024) T->enc_warps = 4;
      if (gnpk::enc_bucket_smem(dp, H, T->enc_warps) > 220 * 1024) T->pw = false;
    }
    if (T->pw) {
      const int H = T->H, dp = T->dp;
      T->enc_grid = std::max(1, std::min(T->sms, (T->nv + 4095) / 4096));
      // rows per block: a multiple of the staging block (aligned bulk copies)
      const int stg = gnpk::enc_stage_rows(T->enc_warps);
      T->enc_rpb = ((T->nv + T->enc_grid - 1) / T->enc_grid + stg - 1) / stg * stg;
      T->enc_grid = (T->nv + T->enc_rpb - 1) / T->enc_rpb;
      T->encpart.alloc((std::size_t)(T->enc_grid + 1) * (H + 1) * 2 * dp);
    }
  }
  {
    static const bool off = [] {
      const char* e = std::getenv("GNPC_NO_DEC_TC");
      return e && std::string(e) == "1";
    }();
    T->dec_tc = !off && T->sell && T->tc && T->dp == 32 && T->H == 32;
    if (T->dec_tc) {
      // residency by registers / smem / TMEM (the occupancy API reports 1 CTA
      // per SM for kernels that allocate TMEM; see tc_ctas_per_sm)
      auto ctas = [&](const void* kf, size_t smem, int nt, int tcols) {
        set_smem_once(kf, smem);
        GNPC_CUDA(cudaFuncSetAttribute(kf, cudaFuncAttributePreferredSharedMemoryCarveout,
                                       cudaSharedmemCarveoutMaxShared));
        cudaFuncAttributes fa{};
        GNPC_CUDA(cudaFuncGetAttributes(&fa, kf));
        int dev = 0, smem_sm = 0, regs_sm = 0;
        GNPC_CUDA(cudaGetDevice(&dev));
        GNPC_CUDA(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
        GNPC_CUDA(cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev));
        int per_sm = std::min(regs_sm / (((fa.numRegs + 7) / 8) * 8 * nt),
                              smem_sm / (int)(smem + fa.sharedSizeBytes + 1024));
        per_sm = std::max(1, std::min(per_sm, 512 / tcols));
        return std::max(1, std::min(per_sm * T->sms, (T->nv + 127) / 128));
      };
      T->dec_grid = ctas((const void*)gnpk::k_decoder_tc<true>, gnpk::DecTc<true>::smem_bytes(),
                         gnpk::DecTc<true>::NT, gnpk::DecTc<true>::TCOLS);
      T->dec_grid_bwd = ctas((const void*)gnpk::k_decoder_tc<false>, gnpk::DecTc<false>::smem_bytes(),
                             gnpk::DecTc<false>::NT, gnpk::DecTc<false>::TCOLS);
      T->decpart.alloc((std::size_t)T->dec_grid_bwd * 33);
      T->decwpart.alloc((std::size_t)T->dec_grid_bwd * 64 * 32);
      const gnp_b200::ParamLayout lay = gnp_b200::param_layout(m->dims);
      std::vector<int> dst(33);
      for (int h = 0; h < 32; ++h) dst[h] = (int)(lay.dec2 + h);
      dst[32] = (int)lay.dec2_b;
      upload_i(T->dec_dst, dst);
    }
  }
  T->hb1.alloc(nvs * T->H);
  T->hb2.alloc(nvs * T->H);
  T->gyv.alloc(nvs);
  T->nbytes_act = (std::int64_t)(act * (2 * T->L + 3) + nvs * (2 * T->H + 2)) * 4;
  // reductions (destinations in the flat reference layout)
  const gnp_b200::ParamLayout lay = gnp_b200::param_layout(m->dims);
  const int d = T->d, H = T->H, dp = T->dp;
  T->rowblk = std::max(1, std::min(2 * T->sms, (T->nv + 255) / 256));
  int maxpq = 0;
  for (int l = 0; l < T->L; ++l) {
    make_red(T->red_layer[l], T->Xs.p + l * act, dp, dp, T->AXs.p + l * act, dp, dp, 0, nullptr, dp, dp,
             T->nv, [&](int p, int q) -> int {
               if (q >= d) return -1;
               if (p < d) return (int)(lay.u[l] + (std::int64_t)q * d + p);           // U(k=p, j=q)
               if (p >= dp && p - dp < d) return (int)(lay.w[l] + (std::int64_t)q * d + (p - dp));
               return -1;
             });
    maxpq = std::max(maxpq, T->red_layer[l].P4 * T->red_layer[l].Q2);
  }
  make_red(T->red_dec1, T->Xs.p + T->L * act, dp, dp, nullptr, 0, 0, 1, T->hb2.p, H, H, T->nv,
           [&](int p, int q) -> int {
             if (q >= H) return -1;
             if (p < d) return (int)(lay.dec1 + (std::int64_t)q * d + p);  // dec1(j=p, h=q)
             if (p == dp) return (int)(lay.dec1_b + q);
             return -1;
           });
  make_red(T->red_dec2, T->hb1.p, H, H, nullptr, 0, 0, 1, T->gyv.p, 1, 1, T->nv,
           [&](int p, int q) -> int {
             if (q != 0) return -1;
             if (p < H) return (int)(lay.dec2 + p);
             if (p == H) return (int)lay.dec2_b;
             return -1;
           });
  make_red(T->red_enc2, T->hb1.p, H, H, nullptr, 0, 0, 1, nullptr, dp, dp, T->nv,
           [&](int p, int q) -> int {
             if (q >= d) return -1;
             if (p < H) return (int)(lay.enc2 + (std::int64_t)q * H + p);  // enc2(h=p, j=q)
             if (p == H) return (int)(lay.enc2_b + q);
             return -1;
           });
  make_red(T->red_enc1, T->vv.p, 1, 1, nullptr, 0, 0, 1, T->hb2.p, H, H, T->nv,
           [&](int p, int q) -> int {
             if (q >= H) return -1;
             if (p == 0) return (int)(lay.enc1 + q);
             if (p == 1) return (int)(lay.enc1_b + q);
             return -1;
           });
  for (auto* r : {&T->red_dec1, &T->red_dec2, &T->red_enc2, &T->red_enc1})
    maxpq = std::max(maxpq, r->P4 * r->Q2);
  // tcgen05 reductions whenever every operand fits one 32-feature atom
  const char* no_tc = std::getenv("GNPC_NO_TC");
  if (dp <= 32 && H <= 32 && !(no_tc && no_tc[0] == '1')) {
    for (int l = 0; l < T->L; ++l)
      make_red_tc(T->red_layer[l], T->Xs.p + l * act, dp, dp, T->AXs.p + l * act, dp, dp, 0, nullptr, dp,
                  dp, T->nv, [&](int m_, int q) -> int {
                    if (q >= d) return -1;
                    if (m_ < d) return (int)(lay.u[l] + (std::int64_t)q * d + m_);
                    if (m_ >= 32 && m_ - 32 < d) return (int)(lay.w[l] + (std::int64_t)q * d + (m_ - 32));
                    return -1;
                  });
    make_red_tc(T->red_dec1, T->Xs.p + T->L * act, dp, dp, nullptr, 0, 0, 1, T->hb2.p, H, H, T->nv,
                [&](int m_, int q) -> int {
                  if (q >= H) return -1;
                  if (m_ < d) return (int)(lay.dec1 + (std::int64_t)q * d + m_);
                  if (m_ == 32) return (int)(lay.dec1_b + q);
                  return -1;
                });
    make_red_tc(T->red_dec2, T->hb1.p, H, H, nullptr, 0, 0, 1, T->gyv.p, 1, 1, T->nv,
                [&](int m_, int q) -> int {
                  if (q != 0) return -1;
                  if (m_ < H) return (int)(lay.dec2 + m_);
                  if (m_ == 32) return (int)lay.dec2_b;
                  return -1;
                });
    make_red_tc(T->red_enc2, T->hb1.p, H, H, nullptr, 0, 0, 1, nullptr, dp, dp, T->nv,
                [&](int m_, int q) -> int {
                  if (q >= d) return -1;
                  if (m_ < H) return (int)(lay.enc2 + (std::int64_t)q * H + m_);
                  if (m_ == 32) return (int)(lay.enc2_b + q);
                  return -1;
                });
    make_red_tc(T->red_enc1, T->vv.p, 1, 1, nullptr, 0, 0, 1, T->hb2.p, H, H, T->nv,
                [&](int m_, int q) -> int {
                  if (q >= H) return -1;
                  if (m_ == 0) return (int)(lay.enc1 + q);
                  if (m_ == 32) return (int)(lay.enc1_b + q);
                  return -1;
                });
    GNPC_CUDA(cudaFuncSetAttribute(gnpk::k_wgrad_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)gnpk::wg::smem_bytes()));
    const int per_sm = tc_ctas_per_sm((const void*)gnpk::k_wgrad_tc, gnpk::wg::smem_bytes(), 32);
    T->wgrad_grid = std::max(1, std::min(per_sm * T->sms, (T->nv + 127) / 128));
    GNPC_CUDA(cudaFuncSetAttribute(gnpk::k_wgrad_bf16, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)gnpk::wgb::smem_bytes()));
    GNPC_CUDA(cudaFuncSetAttribute(gnpk::k_wgrad_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)gnpk::wgt::smem_bytes()));
    T->wgrad_grid_tma = std::max(1, std::min(T->sms, (T->nv + 127) / 128));
    T->wgrad_grid = std::max(T->wgrad_grid, T->wgrad_grid_tma);
    maxpq = std::max(maxpq, 64 * 32 * T->wgrad_grid / std::max(T->rowblk, 1) + 64 * 32);
  }
  // the two one-column reductions as weighted column sums
  if (H <= 32) {
    make_red_colsum(T->red_dec2, T->hb1.p, H, T->gyv.p, T->nv, [&](int i) -> int {
      if (i < H) return (int)(lay.dec2 + i);  // Σ post_h gy
      if (i == 64) return (int)lay.dec2_b;    // Σ gy
      return -1;
    });
    make_red_colsum(T->red_enc1, T->hb2.p, H, T->vv.p, T->nv, [&](int i) -> int {
      if (i < H) return (int)(lay.enc1 + i);                 // Σ gp0_h vv
      if (i >= 32 && i < 32 + H) return (int)(lay.enc1_b + i - 32);  // Σ gp0_h
      return -1;
    });
    T->colsum_grid = std::max(1, std::min(4 * T->sms, (T->nv + 1023) / 1024));
  }
  T->opart.alloc(std::max({(std::size_t)T->rowblk * maxpq, (std::size_t)T->wgrad_grid * 64 * 32,
                           (std::size_t)T->colsum_grid * 96}));
  for (auto* r : {&T->red_dec1, &T->red_dec2, &T->red_enc2, &T->red_enc1}) {
    const size_t smem = (size_t)(32 * r->P4 + 32 * r->Q2) * 4;
    if (smem > 48 * 1024)
      GNPC_CUDA(cudaFuncSetAttribute(gnpk::k_outer_sum, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
  }
  if ((std::size_t)(32 * T->red_layer[0].P4 + 32 * T->red_layer[0].Q2) * 4 > 48 * 1024)
    GNPC_CUDA(cudaFuncSetAttribute(gnpk::k_outer_sum, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   96 * 1024));
  regenerate(*T);
  GNPC_CUDA(cudaStreamSynchronize(T->s));
  return T.release();
}

// x, b host n x B column-major: forward + loss (+ grad + backward)
double step_fb(gnpc_trainer_s& T, const double* x, const double* b, bool bwd) {
  // b first (the forward starts on it); x follows on the copy stream, behind
  // b on the link, and lands while the forward runs: the loss is its first reader
  upload_batch(T, b, T.bb);
  if (!T.cs) {
    GNPC_CUDA(cudaStreamCreateWithFlags(&T.cs, cudaStreamNonBlocking));
    GNPC_CUDA(cudaEventCreateWithFlags(&T.ev_b, cudaEventDisableTiming));
    GNPC_CUDA(cudaEventCreateWithFlags(&T.ev_x, cudaEventDisableTiming));
  }
  const std::size_t cnt = (std::size_t)T.n * T.B;
  T.tmp2.ensure(cnt);
  GNPC_CUDA(cudaEventRecord(T.ev_b, T.s));  // after b's copy and every earlier reader of xb
  GNPC_CUDA(cudaStreamWaitEvent(T.cs, T.ev_b, 0));
  GNPC_CUDA(cudaMemcpyAsync(T.tmp2.p, x, cnt * 8, cudaMemcpyHostToDevice, T.cs));
  gnpk::k_colmajor_to_nb<<<(int)((cnt + kTh - 1) / kTh), kTh, 0, T.cs>>>(T.tmp2.p, T.n, T.B, T.xb.p);
  GNPC_LAUNCHED();
  GNPC_CUDA(cudaEventRecord(T.ev_x, T.cs));
  forward(T);
  GNPC_CUDA(cudaStreamWaitEvent(T.s, T.ev_x, 0));
  const double loss = loss_and_grad(T, bwd);
  if (bwd) backward(T);
  return loss;
}

}  // namespace

extern "C" {

int gnpc_trainer_create(gnpc_model m, int64_t batch, double lr, gnpc_trainer* out) {
  return guarded([&] {
    need(out != nullptr, "trainer_create: null out");
    *out = create(m, batch, lr);
  });
}

int gnpc_trainer_destroy(gnpc_trainer t) {
  return guarded([&] {
    if (!t) return;
    // the model (and its stream) may already be gone at interpreter teardown
    cudaDeviceSynchronize();
    delete t;
  });
}

int gnpc_forward_backward(gnpc_trainer t, const double* x, const double* b, double* loss,
                          double* grads, double* out) {
  return guarded([&] {
    need(t && x && b, "forward_backward: null argument");
    const double l = step_fb(*t, x, b, true);
    if (loss) *loss = l;
    if (grads) {
      GNPC_CUDA(cudaMemcpyAsync(grads, t->g64.p, t->P * 8, cudaMemcpyDeviceToHost, t->s));
    }
    if (out) {
      const std::size_t cnt = (std::size_t)t->n * t->B;
      gnpk::k_nb_to_colmajor<<<(int)((cnt + kTh - 1) / kTh), kTh, 0, t->s>>>(t->out.p, t->n, t->B,
                                                                            t->tmp.p);
      GNPC_LAUNCHED();
      GNPC_CUDA(cudaMemcpyAsync(out, t->tmp.p, cnt * 8, cudaMemcpyDeviceToHost, t->s));
    }
    GNPC_CUDA(cudaStreamSynchronize(t->s));
  });
}

int gnpc_train_step(gnpc_trainer t, const double* x, const double* b, double* loss) {
  return guarded([&] {
    need(t && x && b, "train_step: null argument");
    const double l = step_fb(*t, x, b, true);
    adam(*t);
    GNPC_CUDA(cudaStreamSynchronize(t->s));
    if (loss) *loss = l;
  });
}

namespace {
// device pairs x ~ N(0, I) (Philox keyed by seed and the Adam step), b = A x,
// then forward + loss + backward into g64
double synthetic_fb(gnpc_trainer_s& T, uint64_t seed) {
  const std::size_t cnt = (std::size_t)T.n * T.B;
  gnpk::k_philox_normal<<<(int)((cnt / 4 + kTh) / kTh), kTh, 0, T.s>>>(seed, (unsigned long long)T.t, cnt,
                                                                      T.xb.p);
  GNPC_LAUNCHED();
  gnpk::DevCsr a = T.m->a->dev();
  gnpk::k_spmm_nb<<<T.loss_grid, kTh, 0, T.s>>>(a, T.B, T.xb.p, T.bb.p);
  GNPC_LAUNCHED();
  forward(T);
  const double l = loss_and_grad(T, true);
  backward(T);
  return l;
}
}  // namespace

int gnpc_train_step_synthetic(gnpc_trainer t, uint64_t seed, double* loss) {
  return guarded([&] {
    need(t != nullptr, "train_step_synthetic: null trainer");
    const double l = synthetic_fb(*t, seed);
    adam(*t);
    if (loss) *loss = l;
  });
}

int gnpc_train_backward_synthetic(gnpc_trainer t, uint64_t seed, double* loss) {
  return guarded([&] {
    need(t != nullptr, "train_backward_synthetic: null trainer");
    const double l = synthetic_fb(*t, seed);
    GNPC_CUDA(cudaStreamSynchronize(t->s));
    if (loss) *loss = l;
  });
}

int gnpc_monitor_loss(gnpc_trainer t, const double* x, const double* b, int64_t batch, double* loss) {
  return guarded([&] {
    need(t && x && b && loss, "monitor_loss: null argument");
    if (batch != t->B)
      throw std::invalid_argument("monitor_loss: batch must equal the trainer batch");
    *loss = step_fb(*t, x, b, false);
  });
}

int gnpc_trainer_grad_buffer(gnpc_trainer t, double** dev_ptr, int64_t* count) {
  return guarded([&] {
    need(t && dev_ptr && count, "null argument");
    *dev_ptr = t->g64.p;
    *count = t->P;
  });
}

int gnpc_trainer_stream(gnpc_trainer t, void** stream) {
  return guarded([&] {
    need(t && stream, "null argument");
    *stream = static_cast<void*>(t->s);
  });
}

int gnpc_train_backward_only(gnpc_trainer t, const double* x, const double* b, double* loss) {
  return guarded([&] {
    need(t && x && b, "train_backward_only: null argument");
    const double l = step_fb(*t, x, b, true);
    GNPC_CUDA(cudaStreamSynchronize(t->s));
    if (loss) *loss = l;
  });
}

int gnpc_train_apply_grads(gnpc_trainer t) {
  return guarded([&] {
    need(t != nullptr, "null trainer");
    adam(*t);
    GNPC_CUDA(cudaStreamSynchronize(t->s));
  });
}

int gnpc_trainer_adam_state(gnpc_trainer t, double* m1, double* m2, int64_t* step) {
  return guarded([&] {
    need(t != nullptr, "null trainer");
    if (m1) GNPC_CUDA(cudaMemcpyAsync(m1, t->m1.p, t->P * 8, cudaMemcpyDeviceToHost, t->s));
    if (m2) GNPC_CUDA(cudaMemcpyAsync(m2, t->m2.p, t->P * 8, cudaMemcpyDeviceToHost, t->s));
    GNPC_CUDA(cudaStreamSynchronize(t->s));
    if (step) *step = t->t;
  });
}

int gnpc_trainer_params(gnpc_trainer t, double* params) {
  return guarded([&] {
    need(t && params, "null argument");
    GNPC_CUDA(cudaMemcpyAsync(params, t->p64.p, t->P * 8, cudaMemcpyDeviceToHost, t->s));
    GNPC_CUDA(cudaStreamSynchronize(t->s));
  });
}

int gnpc_trainer_sync_model(gnpc_trainer t) {
  return guarded([&] {
    need(t != nullptr, "null trainer");
    sync_model_params(*t);
  });
}

// train_preconditioner (src/gnn.cpp:401-451), device-resident.
//
// Seeds as the reference: init `seed`, sampler seed+1 (built also when
// spectral_count == 0), monitor seed+2, training stream seed+3.  Per step:
//   pairs   a host thread advances the reference Mersenne Twister for the
//           next batch (raw words, pair_stream.hpp) into a pinned slot; the
//           slot crosses on a copy stream while the device runs the current
//           step; k_pairs_x tempers + Box-Muller (or x = V coef for spectral
//           columns) into the trainer's [n][B] batch and k_spmm_nb_f64 forms
//           b = A x with the f64 matrix values
//   step    forward, L1 loss (folded on the device), backward, Adam
//   monitor forward of the fixed monitoring batch (uploaded once), its loss
//           into a device loss array, the best snapshot kept on the device
// No host synchronisation inside the loop: losses and the best parameters are
// read back once at the end.
namespace {

struct PinnedBuf {
  unsigned char* p = nullptr;
  std::size_t bytes = 0;
  explicit PinnedBuf(std::size_t b) : bytes(b) {
    if (cudaHostAlloc(reinterpret_cast<void**>(&p), b ? b : 1, cudaHostAllocDefault) != cudaSuccess) {
      cudaGetLastError();
      p = nullptr;
      throw std::bad_alloc();
    }
  }
  ~PinnedBuf() {
    if (p) cudaFreeHost(p);
  }
  PinnedBuf(const PinnedBuf&) = delete;
  PinnedBuf& operator=(const PinnedBuf&) = delete;
};

struct EvPair {
  cudaEvent_t a = nullptr, b = nullptr;
};

// loss over the batch into *dst on the device (no host read)
void loss_device(gnpc_trainer_s& T, bool want_grad, double* dst) {
  gnpk::DevCsr a = T.m->a->dev();
  gnpk::k_loss_residual<<<T.loss_grid, kTh, 0, T.s>>>(a, T.B, T.out.p, T.xb.p, T.sgn.p, T.losspart.p);
  GNPC_LAUNCHED();
  if (want_grad) {
    gnpk::DevCsr at = T.At->dev();
    gnpk::k_loss_grad<<<T.loss_grid, kTh, 0, T.s>>>(at, T.B, T.sgn.p, T.gout.p);
    GNPC_LAUNCHED();
  }
  gnpk::k_loss_fold<<<1, 32, 0, T.s>>>(T.losspart.p, T.loss_grid, T.B, dst);
  GNPC_LAUNCHED();
}

void train_run(gnpc_csr_s* a, const gnpc_train_config* cfg, double* best, double* losses,
               double* best_loss, double* timing) {
  need(a && cfg && best && losses && best_loss, "train_preconditioner: null argument");
  if (cfg->batch < cfg->spectral_count)
    throw std::invalid_argument("train: batch must be >= spectral_count");
  if (cfg->batch < 1) throw std::invalid_argument("assemble_batch: empty batch");
  if (cfg->monitor_batch < 1) throw std::invalid_argument("assemble_batch: empty batch");
  const gnp_b200::Dims dims{cfg->d, cfg->hidden, cfg->layers};
  std::vector<double> p0 = gnp_b200::init_params(dims, cfg->seed);
  gnpc_model mm = nullptr;
  if (gnpc_model_create(a, dims.d, dims.hidden, dims.layers, p0.data(), &mm))
    throw std::runtime_error(gnpc_last_error());
  std::unique_ptr<gnpc_model_s, void (*)(gnpc_model_s*)> model(mm, [](gnpc_model_s* q) {
    gnpc_model_destroy(q);
  });
  const std::unique_ptr<gnpc_sampler_s> sampler = build_sampler(*a, cfg->arnoldi_m, cfg->seed + 1);
  const gnp_b200::SpectralSampler* sp = &sampler->s;
  const std::int64_t n = a->h.n, B = cfg->batch, MB = cfg->monitor_batch, S = cfg->spectral_count;
  std::unique_ptr<gnpc_trainer_s> tr(create(model.get(), B, cfg->lr));
  std::unique_ptr<gnpc_trainer_s> mon(MB == B ? nullptr : create(model.get(), MB, cfg->lr));
  gnpc_trainer_s& M = mon ? *mon : *tr;
  if (mon) mon->fwd_only = true;  // the monitoring trainer never runs a backward
  cudaStream_t s = tr->s;  // every trainer of a model runs on the model's stream
  // the monitoring batch: drawn once on the host (Rng(seed+2)), resident
  DevBuf<double> mxd, mbd;
  {
    std::vector<double> mx(n * MB), mb(n * MB);
    gnp_b200::Rng monitor_rng(cfg->seed + 2);
    gnp_b200::assemble_batch(sp, a->h, MB, std::min(S, MB), monitor_rng, mx.data(), mb.data());
    upload_batch(M, mx.data(), M.xb);
    upload_batch(M, mb.data(), M.bb);
    if (!mon) {  // shared trainer: keep the monitor batch aside, swap it in
      mxd.alloc(M.xb.count);
      mbd.alloc(M.bb.count);
      std::swap(mxd, M.xb);
      std::swap(mbd, M.bb);
      GNPC_CUDA(cudaStreamSynchronize(s));
    }
  }
  // f64 matrix values for b = A x (the reference's pairs use the f64 Â)
  DevBuf<double> a64;
  a64.upload(a->h.values.data(), a->h.values.size(), s);
  DevBuf<double> vdev;
  if (S > 0) vdev.upload(sp->v.data(), sp->v.size(), s);
  const std::int64_t steps = cfg->steps;
  DevBuf<double> dloss(steps + 1), dbest(1), dbestp(tr->P);
  auto monitoring = [&](std::int64_t k) {
    if (mon) {  // the monitor trainer reads the current params
      GNPC_CUDA(cudaMemcpyAsync(M.p64.p, tr->p64.p, tr->P * 8, cudaMemcpyDeviceToDevice, s));
      regenerate(M);
    } else {
      std::swap(mxd, M.xb);
      std::swap(mbd, M.bb);
    }
    forward(M);
    loss_device(M, false, dloss.p + k);
    if (!mon) {
      std::swap(mxd, M.xb);
      std::swap(mbd, M.bb);
    }
  };
  monitoring(0);
  GNPC_CUDA(cudaMemcpyAsync(dbest.p, dloss.p, 8, cudaMemcpyDeviceToDevice, s));
  GNPC_CUDA(cudaMemcpyAsync(dbestp.p, tr->p64.p, tr->P * 8, cudaMemcpyDeviceToDevice, s));

  // ---- pair stream: host producer thread, two pinned + two device slots
  gnp_b200::PairStream ps(cfg->seed + 3, n, B, S, sp);
  const gnp_b200::PairBatchLayout& lay = ps.layout();
  std::unique_ptr<PinnedBuf> hslot[2];
  DevBuf<unsigned char> dslot[2];
  cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_used[2] = {nullptr, nullptr};
  cudaStream_t cs = nullptr;
  if (steps > 0) {
    for (int q = 0; q < 2; ++q) {
      hslot[q] = std::make_unique<PinnedBuf>(lay.bytes);
      dslot[q].alloc(lay.bytes);
      GNPC_CUDA(cudaEventCreateWithFlags(&ev_copied[q], cudaEventDisableTiming));
      GNPC_CUDA(cudaEventCreateWithFlags(&ev_used[q], cudaEventDisableTiming));
    }
    GNPC_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  }
  struct Cleanup {
    cudaEvent_t* e1;
    cudaEvent_t* e2;
    cudaStream_t* cs;
    ~Cleanup() {
      for (int q = 0; q < 2; ++q) {
        if (e1[q]) cudaEventDestroy(e1[q]);
        if (e2[q]) cudaEventDestroy(e2[q]);
      }
      if (*cs) cudaStreamDestroy(*cs);
    }
  } cleanup{ev_copied, ev_used, &cs};
  std::mutex mu;
  std::condition_variable cv;
  std::int64_t ready = 0, enqueued = 0;
  bool abort = false;
  std::exception_ptr perr;
  std::thread producer;
  if (steps > 0)
    producer = std::thread([&] {
      try {
        for (std::int64_t t = 0; t < steps; ++t) {
          const int q = (int)(t & 1);
          {
            std::unique_lock<std::mutex> lk(mu);
            cv.wait(lk, [&] { return abort || enqueued >= t - 1; });
            if (abort) return;
          }
          if (t >= 2 && cudaEventSynchronize(ev_copied[q]) != cudaSuccess)
            throw std::runtime_error("pair stream: copy failed");
          ps.fill(hslot[q]->p);
          {
            std::lock_guard<std::mutex> lk(mu);
            ready = t + 1;
          }
          cv.notify_all();
        }
      } catch (...) {
        std::lock_guard<std::mutex> lk(mu);
        perr = std::current_exception();
        abort = true;
        cv.notify_all();
      }
    });
  struct Joiner {
    std::thread& t;
    std::mutex& mu;
    std::condition_variable& cv;
    bool& abort;
    ~Joiner() {
      {
        std::lock_guard<std::mutex> lk(mu);
        abort = true;
      }
      cv.notify_all();
      if (t.joinable()) t.join();
    }
  } joiner{producer, mu, cv, abort};

  std::vector<EvPair> evp, evm;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (timing) {
    evp.resize(steps);
    evm.resize(steps);
    for (std::int64_t t = 0; t < steps; ++t)
      for (cudaEvent_t* e : {&evp[t].a, &evp[t].b, &evm[t].a, &evm[t].b}) GNPC_CUDA(cudaEventCreate(e));
    GNPC_CUDA(cudaEventCreate(&e0));
    GNPC_CUDA(cudaEventCreate(&e1));
    GNPC_CUDA(cudaEventRecord(e0, s));
  }
  double host_wait_ms = 0.0;
  const int pgrid = (int)((n * B + kTh - 1) / kTh);
  const gnpk::DevCsr adev = a->dev();
  for (std::int64_t t = 0; t < steps; ++t) {
    const int q = (int)(t & 1);
    {
      const auto w0 = std::chrono::steady_clock::now();
      std::unique_lock<std::mutex> lk(mu);
      cv.wait(lk, [&] { return abort || ready >= t + 1; });
      if (perr) std::rethrow_exception(perr);
      if (abort) throw std::runtime_error("pair stream stopped");
      host_wait_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - w0).count();
    }
    GNPC_CUDA(cudaStreamWaitEvent(cs, ev_used[q], 0));
    GNPC_CUDA(cudaMemcpyAsync(dslot[q].p, hslot[q]->p, lay.bytes, cudaMemcpyHostToDevice, cs));
    GNPC_CUDA(cudaEventRecord(ev_copied[q], cs));
    {
      std::lock_guard<std::mutex> lk(mu);
      enqueued = t + 1;
    }
    cv.notify_all();
    GNPC_CUDA(cudaStreamWaitEvent(s, ev_copied[q], 0));
    if (timing) GNPC_CUDA(cudaEventRecord(evp[t].a, s));
    const unsigned char* ds = dslot[q].p;
    gnpk::k_pairs_x<<<pgrid, kTh, 0, s>>>(
        reinterpret_cast<const gnpk::PairColDev*>(ds + lay.cols_off),
        reinterpret_cast<const double*>(ds + lay.coef_off),
        reinterpret_cast<const unsigned long long*>(ds + lay.words_off), vdev.p, (int)lay.m, (int)n, (int)B,
        tr->xb.p);
    GNPC_LAUNCHED();
    gnpk::k_spmm_nb_f64<<<tr->loss_grid, kTh, 0, s>>>(adev, a64.p, (int)B, tr->xb.p, tr->bb.p);
    GNPC_LAUNCHED();
    GNPC_CUDA(cudaEventRecord(ev_used[q], s));
    if (timing) GNPC_CUDA(cudaEventRecord(evp[t].b, s));
    forward(*tr);
    loss_device(*tr, true, tr->losspart.p + tr->loss_grid);  // scratch slot past the partials
    backward(*tr);
    adam(*tr);
    if (timing) GNPC_CUDA(cudaEventRecord(evm[t].a, s));
    monitoring(t + 1);
    gnpk::k_best_keep<<<1, kTh, 0, s>>>(dloss.p + t + 1, dbest.p, M.p64.p, dbestp.p, (int)tr->P);
    GNPC_LAUNCHED();
    if (timing) GNPC_CUDA(cudaEventRecord(evm[t].b, s));
  }
  if (timing) GNPC_CUDA(cudaEventRecord(e1, s));
  GNPC_CUDA(cudaMemcpyAsync(losses, dloss.p, (steps + 1) * 8, cudaMemcpyDeviceToHost, s));
  GNPC_CUDA(cudaMemcpyAsync(best, dbestp.p, tr->P * 8, cudaMemcpyDeviceToHost, s));
  GNPC_CUDA(cudaMemcpyAsync(best_loss, dbest.p, 8, cudaMemcpyDeviceToHost, s));
  GNPC_CUDA(cudaStreamSynchronize(s));
  if (timing) {
    float tot = 0.f, pm = 0.f, mm2 = 0.f, x = 0.f;
    GNPC_CUDA(cudaEventElapsedTime(&tot, e0, e1));
    for (std::int64_t t = 0; t < steps; ++t) {
      GNPC_CUDA(cudaEventElapsedTime(&x, evp[t].a, evp[t].b));
      pm += x;
      GNPC_CUDA(cudaEventElapsedTime(&x, evm[t].a, evm[t].b));
      mm2 += x;
      for (cudaEvent_t e : {evp[t].a, evp[t].b, evm[t].a, evm[t].b}) cudaEventDestroy(e);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    timing[0] = tot;
    timing[1] = pm;
    timing[2] = mm2;
    timing[3] = host_wait_ms;
  }
}

// One batch of training pairs from the DEVICE generator train_run uses
// (host MT19937-64 words -> device tempering / Box-Muller; spectral columns
// x = V coef as a device tall-skinny product; b = A x in f64 on the device),
// after dropping skip_batches batches; returned as n x batch col-major like
// assemble_batch (src/sampler.cpp:68-83), for parity tests against it.
void device_pairs(gnpc_csr_s* a, const gnpc_sampler_s* smp, std::uint64_t seed, std::int64_t skip_batches,
                  std::int64_t B, std::int64_t S, double* x, double* b) {
  need(a && x && b, "device_pairs: null argument");
  if (B < 1) throw std::invalid_argument("assemble_batch: empty batch");
  if (S < 0 || S > B) throw std::invalid_argument("device_pairs: spectral_count must be in [0, batch]");
  if (S > 0 && !smp) throw std::invalid_argument("device_pairs: spectral columns need a sampler");
  if (skip_batches < 0) throw std::invalid_argument("device_pairs: skip_batches must be >= 0");
  require_device();
  const gnp_b200::SpectralSampler* sp = smp ? &smp->s : nullptr;
  const std::int64_t n = a->h.n;
  gnp_b200::PairStream ps(seed, n, B, S, sp);
  const gnp_b200::PairBatchLayout& lay = ps.layout();
  PinnedBuf hs(lay.bytes);
  for (std::int64_t q = 0; q <= skip_batches; ++q) ps.fill(hs.p);
  cudaStream_t s = nullptr;
  DevBuf<unsigned char> ds(lay.bytes);
  DevBuf<double> a64, vdev, xd((std::size_t)n * B), bd((std::size_t)n * B);
  a64.upload(a->h.values.data(), a->h.values.size(), s);
  if (S > 0) vdev.upload(sp->v.data(), sp->v.size(), s);
  GNPC_CUDA(cudaMemcpyAsync(ds.p, hs.p, lay.bytes, cudaMemcpyHostToDevice, s));
  const gnpk::DevCsr adev = a->dev();
  const int pgrid = (int)((n * B + kTh - 1) / kTh);
  gnpk::k_pairs_x<<<pgrid, kTh, 0, s>>>(reinterpret_cast<const gnpk::PairColDev*>(ds.p + lay.cols_off),
                                        reinterpret_cast<const double*>(ds.p + lay.coef_off),
                                        reinterpret_cast<const unsigned long long*>(ds.p + lay.words_off), vdev.p,
                                        (int)lay.m, (int)n, (int)B, xd.p);
  GNPC_LAUNCHED();
  const int grid = grid_for(n * 32, kTh, num_sms() * 8);
  gnpk::k_spmm_nb_f64<<<grid, kTh, 0, s>>>(adev, a64.p, (int)B, xd.p, bd.p);
  GNPC_LAUNCHED();
  std::vector<double> hx((std::size_t)n * B), hb((std::size_t)n * B);
  GNPC_CUDA(cudaMemcpyAsync(hx.data(), xd.p, hx.size() * 8, cudaMemcpyDeviceToHost, s));
  GNPC_CUDA(cudaMemcpyAsync(hb.data(), bd.p, hb.size() * 8, cudaMemcpyDeviceToHost, s));
  GNPC_CUDA(cudaStreamSynchronize(s));
  for (std::int64_t i = 0; i < n; ++i)  // [n][B] -> col-major n x B
    for (std::int64_t c = 0; c < B; ++c) {
      x[c * n + i] = hx[i * B + c];
      b[c * n + i] = hb[i * B + c];
    }
}

}  // namespace

int gnpc_device_pairs(gnpc_sampler s, gnpc_csr a, uint64_t seed, int64_t skip_batches, int64_t batch,
                      int64_t spectral_count, double* x, double* b) {
  return guarded([&] { device_pairs(a, s, seed, skip_batches, batch, spectral_count, x, b); });
}

int gnpc_train_preconditioner(gnpc_csr a, const gnpc_train_config* cfg, double* best,
                              double* losses, double* best_loss) {
  return guarded([&] { train_run(a, cfg, best, losses, best_loss, nullptr); });
}

int gnpc_train_preconditioner_timed(gnpc_csr a, const gnpc_train_config* cfg, double* best,
                                    double* losses, double* best_loss, double* timing_ms4) {
  return guarded([&] { train_run(a, cfg, best, losses, best_loss, timing_ms4); });
}

}  // extern "C"
