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
  gnpc_impl::DevBuf<float> UWTC;  // per layer [U;W]^T split tf32 hi/lo, tcgen05 layout
  bool use_tc = true;             // DP 16/32: tcgen05 transform (GNPC_NO_TC=1: CUDA cores)
  int tc_per_sm[4] = {0, 0, 0, 0};  // cached occupancy per (last, OutT) tcgen05 kernel
  gnpk::NetView view{};
  // apply workspace
  gnpc_impl::DevBuf<float> X[2], AXL;
  gnpc_impl::DevBuf<double> partials, io_in, io_out;
  gnpc_impl::DevBuf<unsigned> ticket;
  gnpc_impl::DevBuf<gnpk::ApplyScalars> sc;
  int sms = 0, norm_grid = 0;
  cudaStream_t stream = nullptr;

  void build_view();
  void ensure_workspace();
  template <typename InT, typename OutT>
  void launch_apply(const InT* in, OutT* out, cudaStream_t s, const int* skip,
                    ApplyProf* prof = nullptr);
};
