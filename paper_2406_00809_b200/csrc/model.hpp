// gnpc_model_s: GnnParams bound to a device Â (the GnnOperator of
// src/gnn.cpp:455-467, with the parameters uploaded once as padded fp32).
#pragma once

#include "capi_common.hpp"
#include "kernels/apply.cuh"

// Optional per-kernel CUDA-event marks around the apply pipeline (bench
// roofline).  kind: 0 norm, 1 lift, 2 long-row ÂX, 3 layer, 4 last layer+projection.
struct ApplyProf {
  std::vector<cudaEvent_t> ev;
  std::vector<int> kind;
  void mark(int k, cudaStream_t s) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    ev.push_back(e);
    kind.push_back(k);
  }
};

struct gnpc_model_s {
  gnpc_csr_s* a = nullptr;  // borrowed, like GnnOperator::ahat_
  gnp_b200::Dims dims;
  int dp = 16;                 // d padded to a power of two >= 4 (zero weights)
  std::vector<double> params;  // reference layout, f64
  gnpc_impl::DevBuf<float> P;  // device fp32 params (NetView points into it)
  gnpc_impl::DevBuf<float> LIFT;  // piecewise-linear lift tables (kinks, alpha, beta)
  gnpc_impl::DevBuf<float> UWTC;  // per layer [U;W]^T split tf32 hi/lo, tcgen05 layout
  gnpc_impl::DevBuf<float> UWP;   // per layer [Bu_hi|Bw_hi|Bu_lo|Bw_lo], k_layer_sell layout
  // set by a trainer's Adam step (it rewrites P/UWTC/UWP on the device but
  // not the host params or the lift tables); applies refuse to run on the
  // mixed state until gnpc_trainer_sync_model or gnpc_model_set_params
  bool trainer_dirty = false;
  bool use_tc = true;             // DP 16/32: tcgen05 transform (GNPC_NO_TC=1: CUDA cores)
  int tc_per_sm[8] = {};  // cached occupancy per (last, OutT, path) tcgen05 kernel
  gnpk::NetView view{};
  // apply workspace
  gnpc_impl::DevBuf<float> X[2], AXL, LPART;  // LPART: long-row chunk partials
  gnpc_impl::DevBuf<double> partials, io_in, io_out;
  gnpc_impl::DevBuf<unsigned> ticket;
  // grid-barrier counter of the persistent apply (monotonic; the host mirrors
  // its value so each launch knows its base; launches are stream-ordered)
  gnpc_impl::DevBuf<unsigned long long> gbar;
  unsigned long long gbar_host = 0;
  gnpc_impl::DevBuf<unsigned long long> phase_times;  // GNPC_FUSED_TIMES (debug)
  void* fused_stash = nullptr;  // gnpc_apply zero-copy: device copy of the host input
  bool fused_eligible();        // the apply runs as the single persistent launch
  gnpc_impl::DevBuf<gnpk::ApplyScalars> sc;
  // M(b) in the apply path's length-sorted node order (ragged matrices), before the scatter
  gnpc_impl::DevBuf<double> POUT;
  int sms = 0, norm_grid = 0;
  cudaStream_t stream = nullptr;

  // flat-parameter index maps (see capi.cu build_maps)
  std::vector<int> map_view, map_bt_fwd, map_bt_bwd, map_tc_fwd, map_tc_bwd;
  std::vector<unsigned char> part_tc;
  std::vector<int> map_tc_pair;  // flat param -> UWP (same entries as map_tc_fwd, permuted)
  std::vector<int> map_tc_pair_bwd;  // same layout for the backward operands [Uᵀ; Wᵀ]
  std::vector<unsigned char> part_pair;
  // TMA maps over the two activation buffers (k_layer_sell)
  CUtensorMap tmX[2]{};
  CUtensorMap tmXw[2]{};  // box {DP, kPwRows}: the strip windows' halo-extended tiles (d = 32)
  const float* tm_base[2] = {nullptr, nullptr};
  std::size_t o_enc1 = 0, o_enc1b = 0, o_enc2 = 0, o_enc2b = 0, o_uw = 0, o_dec1 = 0,
              o_dec1b = 0, o_dec2 = 0, o_dec2b = 0;
  void build_maps();
  void build_view();
  void ensure_workspace();
  template <typename InT, typename OutT>
  void launch_apply(const InT* in, OutT* out, cudaStream_t s, const int* skip,
                    ApplyProf* prof = nullptr);
};
