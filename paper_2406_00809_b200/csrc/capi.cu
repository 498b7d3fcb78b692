// C ABI (include/gnpc.h) implementation: CSR handles, GNP model upload and the
// apply pipeline launcher, device FGMRES driver, checkpoints.  Training lives
// in train.cu.  No exception crosses the boundary; no CPU fallback exists for
// any device entry point (no device => GNPC_ENODEV).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <mutex>
#include <new>
#include <sstream>
#include <vector>

#include "capi_common.hpp"
#include "kernels/apply.cuh"
#include "kernels/krylov.cuh"
#include "kernels/layer_sell.cuh"
#include "kernels/layer_tc.cuh"
#include "model.hpp"

namespace gnpc_impl {
bool sell_kernel_off();
bool fused_apply_off();
}  // namespace gnpc_impl

using namespace gnpc_impl;
using gnp_b200::CsrHost;

namespace gnpc_impl {

thread_local std::string g_error;
std::atomic<std::int64_t> g_launches{0};

void set_error(const std::string& msg) { g_error = msg; }

void require_device() {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    cudaGetLastError();
    throw NoDevice("no CUDA device available (the GNP device path has no CPU fallback)");
  }
}

int num_sms() {
  int dev = 0, sms = 0;
  GNPC_CUDA(cudaGetDevice(&dev));
  GNPC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  return sms;
}

void need(bool cond, const char* msg) {
  if (!cond) throw std::invalid_argument(msg);
}

// CTAs per SM for a tcgen05 kernel.  The occupancy API reports 1 CTA/SM for
// kernels that allocate TMEM; each CTA here holds only `tcols` of the 512 TMEM
// columns, so residency is bounded by registers / smem / warps / TMEM instead.
// Also raises the kernel's dynamic-smem limit to `smem`.
int tc_ctas_per_sm(const void* kern, size_t smem, int tcols) {
  GNPC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaFuncAttributes fa{};
  GNPC_CUDA(cudaFuncGetAttributes(&fa, kern));
  int dev = 0, smem_sm = 0, regs_sm = 0;
  GNPC_CUDA(cudaGetDevice(&dev));
  GNPC_CUDA(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
  GNPC_CUDA(cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev));
  const int regs_cta = ((fa.numRegs + 7) / 8) * 8 * gnpk::kThreads;
  const int by_regs = regs_sm / std::max(regs_cta, 1);
  const int by_smem = smem_sm / (int)(smem + fa.sharedSizeBytes + 1024);
  const int by_warps = 64 / (gnpk::kThreads / 32);
  const int by_tmem = 512 / tcols;
  const int per_sm = std::min(std::min(by_regs, by_smem), std::min(by_warps, by_tmem));
  if (const char* dbg = std::getenv("GNPC_DEBUG"); dbg && dbg[0] == '1')
    fprintf(stderr, "[gnpc] tcgen05 kernel smem=%zu regs=%d ctas/SM=%d\n", smem, fa.numRegs, per_sm);
  return std::max(per_sm, 1);
}

// ------------------------------------------------------------------ apply launcher
template <int DP>
struct ApplyLaunch {
  template <typename InT, typename OutT>
  // Ragged matrices: the pipeline runs on length-sorted nodes (DevCsr::perm);
  // the lift reads b through the permutation (the norm reads b as it is, so τ
  // has the natural order's bits) and the result is scattered back at the end.
  static void run(gnpc_model_s& m, const InT* in, OutT* out, cudaStream_t s, const int* skip,
                  ApplyProf* prof) {
    gnpc_csr_s& A = *m.a;
    if (!A.has_perm) return run_ordered<InT, OutT>(m, in, out, s, skip, prof);
    const int n = (int)A.h.n;
    m.POUT.ensure((std::size_t)n);
    OutT* pout = reinterpret_cast<OutT*>(m.POUT.p);
    const int grid = std::max(1, std::min((n + gnpk::kThreads - 1) / gnpk::kThreads, m.sms * 8));
    run_ordered<InT, OutT>(m, in, pout, s, skip, prof);
    gnpk::k_perm_scatter<OutT><<<grid, gnpk::kThreads, 0, s>>>(pout, A.perm.p, n, out, skip);
    GNPC_LAUNCHED();
  }
  template <typename InT, typename OutT>
  static void run_ordered(gnpc_model_s& m, const InT* in, OutT* out, cudaStream_t s, const int* skip,
                          ApplyProf* prof) {
    using namespace gnpk;
    gnpc_csr_s& A = *m.a;
    DevCsr a = A.dev_apply();
    const int n = a.n;
    const NetView& net = m.view;
    const int sms = m.sms;
    auto mark = [&](int k) {
      if (prof) prof->mark(k, s);
    };
    const bool sell_off = sell_kernel_off();
    const bool fused_off = fused_apply_off();
    if constexpr (DP == 16 || DP == 32) {
      // the whole apply as one persistent cooperative launch (no long rows:
      // those need their chunk kernels between layers).  The per-kernel
      // profile keeps the per-layer launches so each phase can be timed.
      // DP=16 only: at DP=32 the in-kernel layers measured slower than
      // separate launches (C5: 499 vs 450 us per layer) while DP=16 gains
      // (C2: 17 vs 24 us per layer: no launch gap or prologue per layer)
      // pipeline mode: 0 sliced-ELL, 1 CSR ranges
      const int mode = a.sell ? 0 : 1;
      auto smem_of = [&](int md, bool last) -> size_t {
        return md == 0 ? SellCfg<DP, 0>::smem_bytes(net.hidden, last) : SellCfg<DP, 1>::smem_bytes(net.hidden, last);
      };
      const bool fits = smem_of(mode, true) <= 226 * 1024;
      if (DP == 16 && fits && m.use_tc && !sell_off && !fused_off && A.n_long == 0 && prof == nullptr &&
          n > 0) {
        using S = SellCfg<DP, false>;
        const size_t smem = smem_of(mode, true);
        auto kern = mode == 1 ? k_apply_sell<DP, InT, OutT, 1> : k_apply_sell<DP, InT, OutT, 0>;
        {
          cudaFuncAttributes fa{};
          GNPC_CUDA(cudaFuncGetAttributes(&fa, (const void*)kern));  // static smem counts against 227 KB
          set_smem_attr((const void*)kern, 227 * 1024 - (int)fa.sharedSizeBytes);
        }
        const int tiles = (n + S::TM - 1) / S::TM;
        const int grid = std::max(1, std::min(tiles, sms));
        static const bool times = std::getenv("GNPC_FUSED_TIMES") != nullptr;
        gnpc_impl::DevBuf<unsigned long long>& tbuf = m.phase_times;  // GNPC_FUSED_TIMES debug only
        if (times && !tbuf.p) tbuf.alloc(64);
        ApplyFused fa{m.tmX[0], m.tmX[1], m.tmXw[0], m.tmXw[1], m.X[0].p, m.X[1].p, m.UWP.p, m.partials.p,
                      m.gbar.p, m.gbar_host, m.sc.p, times ? tbuf.p : nullptr, m.fused_stash};
        void* args[] = {(void*)&a, (void*)&fa, (void*)&in, (void*)&net, (void*)&out, (void*)&skip};
        GNPC_CUDA(cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(S::NT), args, smem, s));
        // the grid barriers' base advances only for a launch that happened (a
        // failed cooperative launch must not leave the host count ahead of
        // the device counter)
        m.gbar_host += (unsigned long long)grid * (1 + net.layers);
        GNPC_LAUNCHED();
        if (times) {
          unsigned long long h[64];
          GNPC_CUDA(cudaMemcpyAsync(h, tbuf.p, sizeof(h), cudaMemcpyDeviceToHost, s));
          GNPC_CUDA(cudaStreamSynchronize(s));
          std::fprintf(stderr, "fused phases (us):");
          for (int k = 1; k < 2 * net.layers + 2; ++k) std::fprintf(stderr, " %.1f", (h[k] - h[k - 1]) * 1e-3);
          std::fprintf(stderr, "\n");
        }
        return;
      }
    }
    // τ
    mark(0);
    k_apply_norm<InT><<<m.norm_grid, kThreads, 0, s>>>(in, n, m.partials.p, m.ticket.p, m.sc.p, skip);
    GNPC_LAUNCHED();
    // d = 32 strip windows: the lift is fused into the first layer (its lift
    // warps compute the row windows; x1 never crosses HBM).  GNPC_NO_LIFT_FUSE=1
    // keeps the separate lift kernel.
    bool fuse_lift = false;
    if constexpr (DP == 32) {
      const char* off = std::getenv("GNPC_NO_LIFT_FUSE");  // (read per apply: tests toggle it)
      fuse_lift = !(off && off[0] == '1') && a.pw && m.use_tc && !sell_off && A.n_long == 0 && net.layers >= 2 && net.nbreak <= 32 &&
                  SellCfg<32, 8>::smem_bytes(net.hidden, true) <= 227 * 1024 &&
                  SellCfg<32, 9>::smem_bytes(net.hidden, false) <= 227 * 1024;
    }
    // lift
    if (!fuse_lift) {
      const size_t smem = (size_t)(net.nbreak + 1) * DP * 8 + (size_t)net.nbreak * 4 + 16;
      auto kern = k_lift_pw<DP, InT>;
      set_smem_attr((const void*)kern, 160 * 1024);
      mark(1);
      const int ng = kThreads / (DP / 4);
      int grid = std::min((n + ng - 1) / ng, sms * 8);
      grid = std::max(grid, 1);
      kern<<<grid, kThreads, smem, s>>>(in, n, net, m.sc.p, m.X[0].p, skip, a.perm);
      GNPC_LAUNCHED();
    }
    using Cfg = LayerCfg<DP>;
    const int tiles = (n + Cfg::TM - 1) / Cfg::TM;
    int cur = 0;
    for (int l = 0; l < net.layers; ++l) {
      const float* X = m.X[cur].p;
      const float* uw = net.uw + (size_t)l * 2 * DP * DP;
      const float* axl = nullptr;
      if (A.n_long > 0) {
        mark(2);
        LongPlan lp{A.n_chunks, A.ch_row.p, A.ch_k0.p, A.ch_k1.p, A.n_long,
                    A.long_rows.p, A.long_c0.p, m.LPART.p};
        const int wpb = kThreads / 32;
        k_long_chunks<DP><<<(A.n_chunks + wpb - 1) / wpb, kThreads, 0, s>>>(a, lp, X, m.sc.p, skip);
        GNPC_LAUNCHED();
        const int thr = A.n_long * (DP / 4);
        k_long_combine<DP><<<(thr + kThreads - 1) / kThreads, kThreads, 0, s>>>(lp, m.AXL.p, m.sc.p,
                                                                              skip);
        GNPC_LAUNCHED();
        axl = m.AXL.p;
      }
      const bool last = l + 1 == net.layers;
      // (profile: the fused lift + first layer is timed in the lift's slot, so
      // slot 3 stays the per-launch time of the plain layer kernel)
      mark(last ? 4 : (l == 0 && fuse_lift ? 1 : 3));
      if constexpr (DP == 32) {
        // strip windows (stencil-like d = 32 matrices with a dominant tile
        // stride): X rows staged in shared memory, one new window per tile
        if (l == 0 && fuse_lift) {
          using S = SellCfg<DP, 9>;
          auto kern = k_layer_sell_lift<DP, OutT>;
          set_smem_attr((const void*)kern, 227 * 1024);
          const int tiles_s = (n + S::TM - 1) / S::TM;
          const int grid = std::max(1, std::min(tiles_s, sms));
          SellMaps maps{m.tmX[cur], m.tmX[1 - cur], m.tmXw[cur]};
          kern<<<grid, S::NT, S::smem_bytes(net.hidden, false), s>>>(a, maps, (const void*)in, sizeof(InT) == 8 ? 1 : 0,
                                                                      m.UWP.p, net, m.sc.p, skip);
          GNPC_LAUNCHED();
          cur = 1 - cur;
          continue;
        }
        if (a.pw && m.use_tc && !sell_off && SellCfg<32, 8>::smem_bytes(net.hidden, true) <= 227 * 1024) {
          using S = SellCfg<DP, 7>;
          auto kern = last ? k_layer_sell<DP, true, OutT, 8> : k_layer_sell<DP, false, OutT, 7>;
          const size_t smem_l = last ? SellCfg<DP, 8>::smem_bytes(net.hidden, true)
                                     : SellCfg<DP, 7>::smem_bytes(net.hidden, false);
          set_smem_attr((const void*)kern, 227 * 1024);
          const int tiles_s = (n + S::TM - 1) / S::TM;
          const int grid = std::max(1, std::min(tiles_s, sms));
          SellMaps maps{m.tmX[cur], m.tmX[1 - cur], m.tmXw[cur]};
          const float* uwp = m.UWP.p + (size_t)l * 4 * DP * DP;
          kern<<<grid, S::NT, smem_l, s>>>(a, maps, X, axl, uwp, net, m.sc.p, out, skip);
          GNPC_LAUNCHED();
          cur = 1 - cur;
          continue;
        }
        // pair-union slices (stencil-like d = 32 matrices): 4-deep ring for
        // the non-last layers, 3 deep for the last
        if (a.psell && m.use_tc && !sell_off &&
            SellCfg<32, 6>::smem_bytes(net.hidden, true) <= 227 * 1024) {
          using S = SellCfg<DP, 5>;
          auto kern = last ? k_layer_sell<DP, true, OutT, 6> : k_layer_sell<DP, false, OutT, 5>;
          const size_t smem_l = last ? SellCfg<DP, 6>::smem_bytes(net.hidden, true)
                                     : SellCfg<DP, 5>::smem_bytes(net.hidden, false);
          set_smem_attr((const void*)kern, 227 * 1024);
          const int tiles_s = (n + S::TM - 1) / S::TM;
          const int grid = std::max(1, std::min(tiles_s, sms));
          SellMaps maps{m.tmX[cur], m.tmX[1 - cur], m.tmXw[cur]};
          const float* uwp = m.UWP.p + (size_t)l * 4 * DP * DP;
          kern<<<grid, S::NT, smem_l, s>>>(a, maps, X, axl, uwp, net, m.sc.p, out, skip);
          GNPC_LAUNCHED();
          cur = 1 - cur;
          continue;
        }
      }
      if constexpr (DP == 16 || DP == 32) {
        const int lmode = a.sell ? 0 : 1;
        const size_t smem = lmode == 0 ? SellCfg<DP, 0>::smem_bytes(net.hidden, last)
                                       : SellCfg<DP, 1>::smem_bytes(net.hidden, last);
        const bool sell_fits = smem <= 227 * 1024;
        if (m.use_tc && !sell_off && sell_fits) {
          // TMA pipeline, one 544-thread CTA per SM: sliced-ELL slices on
          // regular matrices, the short-row CSR ranges on ragged ones
          using S = SellCfg<DP, false>;
          // d = 32 non-last sliced-ELL layers: the 4-deep ring (mode 4)
          constexpr int D4 = DP == 32 ? 4 : 0;
          const bool deep = DP == 32 && lmode == 0 && !last;
          auto kern = lmode == 1 ? (last ? k_layer_sell<DP, true, OutT, 1> : k_layer_sell<DP, false, OutT, 1>)
                                 : (last ? k_layer_sell<DP, true, OutT>
                                         : (deep ? k_layer_sell<DP, false, OutT, D4> : k_layer_sell<DP, false, OutT>));
          const size_t smem_l = deep ? SellCfg<DP, D4>::smem_bytes(net.hidden, false) : smem;
          set_smem_attr((const void*)kern, 227 * 1024);
          const int tiles_s = (n + S::TM - 1) / S::TM;
          const int grid = std::max(1, std::min(tiles_s, sms));
          SellMaps maps{m.tmX[cur], m.tmX[1 - cur], m.tmXw[cur]};
          const float* uwp = m.UWP.p + (size_t)l * 4 * DP * DP;
          kern<<<grid, S::NT, smem_l, s>>>(a, maps, X, axl, uwp, net, m.sc.p, out, skip);
          GNPC_LAUNCHED();
          cur = 1 - cur;
          continue;
        }
        if (m.use_tc) {
          using T = TcCfg<DP>;
          const float* uwtc = m.UWTC.p + (size_t)l * 2 * T::B_FLOATS;
          auto kern = a.sell ? (last ? k_layer_tc<DP, kEpiLast, OutT, kPathSell>
                                     : k_layer_tc<DP, kEpiRelu, OutT, kPathSell>)
                             : (last ? k_layer_tc<DP, kEpiLast, OutT, kPathCsr1>
                                     : k_layer_tc<DP, kEpiRelu, OutT, kPathCsr1>);
          const size_t smem = T::smem_bytes(last, net.hidden);
          // launch geometry is computed once per model (host queries would
          // otherwise starve the GPU between the 8 layer launches)
          int& per_sm = m.tc_per_sm[(last ? 2 : 0) + (sizeof(OutT) == 8 ? 1 : 0) + (a.sell ? 4 : 0)];
          if (per_sm == 0) per_sm = tc_ctas_per_sm((const void*)kern, smem, T::TCOLS);
          const int tiles_tc = (n + T::TM - 1) / T::TM;
          const int grid = std::max(1, std::min(tiles_tc, per_sm * sms));
          static const int dbg = [] {
            const char* e = std::getenv("GNPC_LAYER_DBG");
            return e ? std::atoi(e) : 0;
          }();
          LayerIO io{X, last ? nullptr : m.X[1 - cur].p, uwtc, axl, nullptr, nullptr, 1, dbg};
          kern<<<grid, kThreads, smem, s>>>(a, io, net, m.sc.p, out, skip);
          GNPC_LAUNCHED();
          cur = 1 - cur;
          continue;
        }
      }
      if (!last) {
        auto kern = k_layer<DP, false, OutT>;
        const size_t smem = Cfg::smem_bytes(false, net.hidden);
        set_smem_attr((const void*)kern, 200 * 1024);
        kern<<<tiles, kThreads, smem, s>>>(a, X, m.X[1 - cur].p, uw, axl, net, m.sc.p, out, skip);
        GNPC_LAUNCHED();
        cur = 1 - cur;
      } else {
        auto kern = k_layer<DP, true, OutT>;
        const size_t smem = Cfg::smem_bytes(true, net.hidden);
        set_smem_attr((const void*)kern, 200 * 1024);
        kern<<<tiles, kThreads, smem, s>>>(a, X, nullptr, uw, axl, net, m.sc.p, out, skip);
        GNPC_LAUNCHED();
      }
    }
    mark(-1);
  }
};

}  // namespace gnpc_impl

// ====================================================================== TMA maps
namespace gnpc_impl {
static bool env_on(const char* name) {
  const char* e = std::getenv(name);
  return e && std::string(e) == "1";
}
bool sell_kernel_off() {  // GNPC_NO_SELL_KERNEL=1: register-staged tcgen05 layers instead
  static const bool v = env_on("GNPC_NO_SELL_KERNEL");
  return v;
}
bool fused_apply_off() {  // GNPC_NO_FUSED_APPLY=1: per-layer launches instead of one
  static const bool v = env_on("GNPC_NO_FUSED_APPLY");
  return v;
}
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q{};
    void* p = nullptr;
    GNPC_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) throw CudaError("cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

CUtensorMap make_rows_map(const float* base, std::int64_t rows, int width, int box_rows,
                          CUtensorMapSwizzle swizzle) {
  CUtensorMap m{};
  const cuuint64_t dims[2] = {(cuuint64_t)width, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)width * sizeof(float)};
  const cuuint32_t box[2] = {(cuuint32_t)width, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = tensor_map_encoder()(
      &m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
      CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed");
  return m;
}
}  // namespace gnpc_impl

// ====================================================================== CSR
void gnpc_csr_s::upload() {
  if (dev_ready) return;
  require_device();
  if (h.nnz() >= (std::int64_t(1) << 31) || h.n >= (std::int64_t(1) << 31) - 1)
    throw Unsupported("device CSR uses int32 indices: n and nnz must be < 2^31");
  std::vector<int> hrp(h.n + 1), hci(h.nnz());
  std::vector<float> hv(h.nnz());
  std::vector<int> longs;
  max_row = 0;
  for (std::int64_t i = 0; i <= h.n; ++i) hrp[i] = static_cast<int>(h.row_ptr[i]);
  for (std::int64_t k = 0; k < h.nnz(); ++k) {
    hci[k] = static_cast<int>(h.col_idx[k]);
    hv[k] = static_cast<float>(h.values[k]);
  }
  for (std::int64_t i = 0; i < h.n; ++i) max_row = std::max(max_row, hrp[i + 1] - hrp[i]);
  // padded copies (row_ptr + 132 entries of nnz, col/val + 4 zeros): the
  // training TMA layers bulk-copy 16-byte-aligned supersets of a tile's range
  {
    std::vector<int> prp(hrp);
    prp.resize(hrp.size() + 132, hrp.back());
    std::vector<int> pci(hci);
    pci.resize(hci.size() + 4, 0);
    std::vector<float> pv(hv);
    pv.resize(hv.size() + 4, 0.f);
    rp.upload(prp.data(), prp.size());
    ci.upload(pci.data(), pci.size());
    v.upload(pv.data(), pv.size());
  }
  // Ragged matrices (the natural order pads a sliced-ELL copy by > 25 %): the
  // apply path renumbers the nodes by row length (stable sort, ascending; a
  // symmetric permutation of Â), so every 128-row tile holds rows of one
  // length — no lane idles behind a longer neighbour, the sliced-ELL layout
  // applies, and the long rows fill the last tiles.  Each row keeps its
  // entries in stored order, so every sum and the output are bit-identical to
  // the natural order's; M(b) gathers b and scatters its result through
  // `perm`.  The FGMRES SpMV and the training kernels keep the natural order
  // (rp / ci / v above).  GNPC_NO_ROWSORT=1 disables it.
  has_perm = false;
  build_sell(hrp, hci, hv);
  {
    const char* e = std::getenv("GNPC_NO_ROWSORT");
    const char* ns = std::getenv("GNPC_NO_SELL");
    if (!has_sell && !(e && e[0] == '1') && !(ns && ns[0] == '1') && h.n >= 128) {
      const std::int64_t n = h.n;
      std::vector<int> pm(n), inv(n);
      for (std::int64_t i = 0; i < n; ++i) pm[i] = static_cast<int>(i);
      std::stable_sort(pm.begin(), pm.end(), [&](int x, int y) { return hrp[x + 1] - hrp[x] < hrp[y + 1] - hrp[y]; });
      for (std::int64_t i = 0; i < n; ++i) inv[pm[i]] = static_cast<int>(i);
      std::vector<int> qrp(n + 1), qci(hci.size());
      std::vector<float> qv(hv.size());
      qrp[0] = 0;
      for (std::int64_t i = 0; i < n; ++i) {
        const int s0 = hrp[pm[i]], len = hrp[pm[i] + 1] - s0, d0 = qrp[i];
        for (int k = 0; k < len; ++k) {
          qci[d0 + k] = inv[hci[s0 + k]];
          qv[d0 + k] = hv[s0 + k];
        }
        qrp[i + 1] = d0 + len;
      }
      hrp.swap(qrp);
      hci.swap(qci);
      hv.swap(qv);
      std::vector<int> prp(hrp);
      prp.resize(hrp.size() + 132, hrp.back());
      std::vector<int> pci(hci);
      pci.resize(hci.size() + 4, 0);
      std::vector<float> pv(hv);
      pv.resize(hv.size() + 4, 0.f);
      prm_rp.upload(prp.data(), prp.size());
      prm_ci.upload(pci.data(), pci.size());
      prm_v.upload(pv.data(), pv.size());
      perm.upload(pm.data(), pm.size());
      has_perm = true;
      build_sell(hrp, hci, hv);  // uniform tiles: the padding test passes now
    }
  }
  // (from here on hrp / hci / hv are the apply path's view: permuted when has_perm)
  for (std::int64_t i = 0; i < h.n; ++i)
    if (hrp[i + 1] - hrp[i] > gnpk::kLongRow) longs.push_back(static_cast<int>(i));
  n_long = static_cast<int>(longs.size());
  if (n_long) {
    long_rows.upload(longs.data(), longs.size());
    std::vector<int> crow, ck0, ck1, c0(1, 0);
    for (int i : longs) {
      for (int k = hrp[i]; k < hrp[i + 1]; k += gnpk::kChunk) {
        crow.push_back(i);
        ck0.push_back(k);
        ck1.push_back(std::min(k + gnpk::kChunk, hrp[i + 1]));
      }
      c0.push_back(static_cast<int>(crow.size()));
    }
    n_chunks = static_cast<int>(crow.size());
    ch_row.upload(crow.data(), crow.size());
    ch_k0.upload(ck0.data(), ck0.size());
    ch_k1.upload(ck1.data(), ck1.size());
    long_c0.upload(c0.data(), c0.size());
  }
  build_pairs(hrp, hci, hv);
  build_pw(hrp, hci, hv);
  // short-row CSR (long rows emptied), padded for the TMA pipeline's bulk copies
  {
    const std::int64_t n = h.n;
    std::vector<int> srp(n + 1 + 132), sci, tf((n + 127) / 128, 0);
    std::vector<float> sv;
    sci.reserve(hci.size() + 4);
    sv.reserve(hv.size() + 4);
    srp[0] = 0;
    for (std::int64_t i = 0; i < n; ++i) {
      const int s = hrp[i], e = hrp[i + 1];
      if (e - s > gnpk::kLongRow) {
        tf[i / 128] = 1;
      } else {
        sci.insert(sci.end(), hci.begin() + s, hci.begin() + e);
        sv.insert(sv.end(), hv.begin() + s, hv.begin() + e);
      }
      srp[i + 1] = static_cast<int>(sci.size());
    }
    for (std::size_t i = n + 1; i < srp.size(); ++i) srp[i] = srp[n];
    for (int k = 0; k < 4; ++k) {
      sci.push_back(0);
      sv.push_back(0.f);
    }
    rps.upload(srp.data(), srp.size());
    cis.upload(sci.data(), sci.size());
    vs.upload(sv.data(), sv.size());
    tflag.upload(tf.data(), tf.size());
  }
  GNPC_CUDA(cudaDeviceSynchronize());
  dev_ready = true;
}

// Sliced ELL over 128-row slices (the tensor-core layer's tile): slice t holds
// K_t = max short-row length entries per row, column-major within the slice so
// one bulk copy stages a tile and a warp's (col, val) reads are contiguous.
// Built only when the padding stays small (stencil-like matrices); long rows
// (> kLongRow) keep their chunked path and get padding entries here.
void gnpc_csr_s::build_sell(const std::vector<int>& hrp, const std::vector<int>& hci,
                            const std::vector<float>& hv) {
  constexpr int TM = 128;
  const std::int64_t n = h.n;
  const std::int64_t ntiles = (n + TM - 1) / TM;
  if (n == 0) return;
  if (const char* e = std::getenv("GNPC_NO_SELL"); e && std::string(e) == "1") return;
  std::vector<int> K(ntiles, 0), off(ntiles, 0);
  std::int64_t total = 0, short_nnz = 0;
  for (std::int64_t t = 0; t < ntiles; ++t) {
    int kt = 0;
    bool haslong = false;
    for (std::int64_t i = t * TM; i < std::min(n, (t + 1) * TM); ++i) {
      const int len = hrp[i + 1] - hrp[i];
      if (len > gnpk::kLongRow) {
        haslong = true;
      } else {
        kt = std::max(kt, len);
        short_nnz += len;
      }
    }
    if (total + (std::int64_t)kt * TM >= (std::int64_t(1) << 31)) return;
    off[t] = static_cast<int>(total);
    total += (std::int64_t)kt * TM;
    K[t] = kt | (haslong ? 1 << 16 : 0);
  }
  if ((double)total > 1.25 * (double)short_nnz + 4.0 * TM) return;  // too ragged
  std::vector<int2> ent(std::max<std::int64_t>(total, 1));
  for (std::int64_t t = 0; t < ntiles; ++t) {
    const int kt = K[t] & 0xffff;
    for (int r = 0; r < TM; ++r) {
      const std::int64_t i = t * TM + r;
      int s = 0, len = 0;
      if (i < n) {
        s = hrp[i];
        len = hrp[i + 1] - s;
        if (len > gnpk::kLongRow) len = 0;
      }
      for (int k = 0; k < kt; ++k) {
        int2 e;
        if (k < len) {
          e.x = hci[s + k];
          std::memcpy(&e.y, &hv[s + k], 4);
        } else {
          e.x = i < n ? static_cast<int>(i) : 0;  // own row, weight 0
          e.y = 0;
        }
        ent[off[t] + (std::size_t)k * TM + r] = e;
      }
    }
  }
  sell.upload(ent.data(), ent.size());
  sell_off.upload(off.data(), off.size());
  sell_k.upload(K.data(), K.size());
  has_sell = true;
}

// Pair-union sliced-ELL (see DevCsr::psell).  Built for matrices without long
// rows whose rows are column-sorted and whose adjacent row pairs share enough
// columns that the union gathers are <= 80 % of the sliced-ELL gathers
// (9-point stencil: 12 vs 18 per pair).  GNPC_NO_PAIR=1 disables it.
void gnpc_csr_s::build_pairs(const std::vector<int>& hrp, const std::vector<int>& hci,
                             const std::vector<float>& hv) {
  has_pairs = false;
  if (!has_sell || n_long != 0) return;
  if (const char* e = std::getenv("GNPC_NO_PAIR"); e && std::string(e) == "1") return;
  const std::int64_t n = h.n;
  constexpr int TM = 128, NG = TM / 2;
  const std::int64_t ntiles = (n + TM - 1) / TM;
  for (std::int64_t i = 0; i < n; ++i)
    for (int k = hrp[i] + 1; k < hrp[i + 1]; ++k)
      if (hci[k] <= hci[k - 1]) return;  // unsorted or duplicate columns: stored order not a merge
  auto row_range = [&](std::int64_t i, int& s, int& e) {
    if (i < n) {
      s = hrp[i];
      e = hrp[i + 1];
    } else {
      s = e = 0;
    }
  };
  // union length of each pair, per tile maximum
  std::vector<int> K(ntiles, 0), off(ntiles, 0);
  std::int64_t total = 0, sell_gathers = 0;
  for (std::int64_t t = 0; t < ntiles; ++t) {
    int kt = 0, ks = 0;
    for (int g = 0; g < NG; ++g) {
      int s0, e0, s1, e1;
      row_range(t * TM + 2 * g, s0, e0);
      row_range(t * TM + 2 * g + 1, s1, e1);
      ks = std::max(ks, std::max(e0 - s0, e1 - s1));
      int u = 0;
      while (s0 < e0 || s1 < e1) {
        if (s1 >= e1 || (s0 < e0 && hci[s0] < hci[s1])) ++s0;
        else if (s0 >= e0 || hci[s1] < hci[s0]) ++s1;
        else { ++s0; ++s1; }
        ++u;
      }
      kt = std::max(kt, u);
    }
    off[t] = static_cast<int>(total);
    total += (std::int64_t)kt * NG;
    if (total >= (std::int64_t(1) << 31)) return;
    K[t] = kt;
    sell_gathers += (std::int64_t)ks * TM;
  }
  if ((double)total > 0.8 * (double)sell_gathers) return;  // not enough sharing
  std::vector<int4> ent(std::max<std::int64_t>(total, 1));
  for (std::int64_t t = 0; t < ntiles; ++t) {
    for (int g = 0; g < NG; ++g) {
      const std::int64_t i0 = t * TM + 2 * g;
      int s0, e0, s1, e1;
      row_range(i0, s0, e0);
      row_range(i0 + 1, s1, e1);
      int u = 0;
      auto put = [&](int col, float w0, float w1) {
        int4 e;
        e.x = col;
        std::memcpy(&e.y, &w0, 4);
        std::memcpy(&e.z, &w1, 4);
        e.w = 0;
        ent[off[t] + (std::size_t)u * NG + g] = e;
        ++u;
      };
      while (s0 < e0 || s1 < e1) {
        if (s1 >= e1 || (s0 < e0 && hci[s0] < hci[s1])) {
          put(hci[s0], hv[s0], 0.f);
          ++s0;
        } else if (s0 >= e0 || hci[s1] < hci[s0]) {
          put(hci[s1], 0.f, hv[s1]);
          ++s1;
        } else {
          put(hci[s0], hv[s0], hv[s1]);
          ++s0;
          ++s1;
        }
      }
      const int own = i0 < n ? static_cast<int>(i0) : 0;
      while (u < K[t]) put(own, 0.f, 0.f);
    }
  }
  psell.upload(ent.data(), ent.size());
  psell_off.upload(off.data(), off.size());
  psell_k.upload(K.data(), K.size());
  has_pairs = true;
}

// The tile distance S (>= 2) at which most off-tile columns sit (a row
// window straddles two tiles, so distances S-1..S+1 count for S); 0 when no
// distance holds >= 25 % of a row sample's entries.
int gnpc_csr_s::dominant_tile_stride(const std::vector<int>& hrp, const std::vector<int>& hci, int TM) const {
  const std::int64_t n = h.n;
  // histogram of |tile distance| for off-tile entries of a row sample
  std::vector<std::int64_t> hist(4097, 0);
  std::int64_t total = 0;
  const std::int64_t step = std::max<std::int64_t>(1, n / 65536);
  for (std::int64_t i = 0; i < n; i += step) {
    const std::int64_t ti = i / TM;
    for (int k = hrp[i]; k < hrp[i + 1]; ++k) {
      const std::int64_t d = std::llabs(static_cast<std::int64_t>(hci[k]) / TM - ti);
      ++total;
      if (d >= 2 && d <= 4096) ++hist[d];
    }
  }
  if (total == 0) return 0;
  // the most frequent distance, then the entries within +-1 of it (an exact
  // multiple of the tile is a spike; a stencil row offset of 128 S +- 1 rows
  // spills into S - 1 and S + 1)
  int S = 0;
  for (int d = 2; d <= 4095; ++d)
    if (hist[d] > hist[S]) S = d;
  if (S < 2) return 0;
  const std::int64_t near = hist[S - 1] + hist[S] + hist[S + 1];
  if (4 * near < total) return 0;  // no dominant stride: < 25 % of the entries
  return S;
}

// Training strip windows (see DevCsr::tw): the batched layers' 128-row tile
// holds npt = 128 / bs nodes (bs samples each); tile u gathers from the node
// windows of tiles u - S, u, u + S, each extended by one node on either side
// (npt + 2 nodes = 128 + 2 bs virtual rows).  Built per batch size, for
// bs <= 32 (the window slot is sized for 192 rows).  GNPC_NO_TW=1 disables.
void gnpc_csr_s::bind_tw(int bs, gnpk::DevCsr& d) const {
  auto it = tws.find(bs);
  const TwLayout* L = it != tws.end() && it->second->ok ? it->second.get() : nullptr;
  d.tw = L ? L->sl.p : nullptr;
  d.tw_off = L ? L->off.p : nullptr;
  d.tw_k = L ? L->k.p : nullptr;
  d.tw_order = L ? L->order.p : nullptr;
  d.tw_S = L ? L->S : 0;
}

bool gnpc_csr_s::ensure_tw(int bs) {
  if (auto it = tws.find(bs); it != tws.end()) return it->second->ok;
  auto& L = tws[bs];
  L = std::make_unique<TwLayout>();
  if (const char* e = std::getenv("GNPC_NO_TW"); e && std::string(e) == "1") return false;
  if (bs < 1 || bs > 32 || 128 % bs != 0) return false;
  const std::int64_t n = h.n;
  const int npt = 128 / bs, WN = npt + 2;  // nodes per window
  const std::int64_t T = (n + npt - 1) / npt;
  if (T < 4 * 148 || n >= (std::int64_t(1) << 31)) return false;
  std::vector<int> hrp(n + 1), hci(h.nnz());
  for (std::int64_t i = 0; i <= n; ++i) hrp[i] = static_cast<int>(h.row_ptr[i]);
  for (std::int64_t k = 0; k < h.nnz(); ++k) hci[k] = static_cast<int>(h.col_idx[k]);
  const int S = dominant_tile_stride(hrp, hci, npt);
  if (S < 2) return false;
  // node index in the windows (a, b, c) laid end to end at the ring's slot
  // stride (kTwRowsMax rows = WS nodes per slot)
  const int WS = gnpk::kTwRowsMax / bs;
  auto widx = [&](std::int64_t t, std::int64_t c) -> int {
    for (int w : {1, 0, 2}) {
      const std::int64_t b0 = (t + (w - 1) * (std::int64_t)S) * npt - 1;
      if (c >= b0 && c < b0 + WN) return w * WS + static_cast<int>(c - b0);
    }
    return -1;
  };
  constexpr int KMAX = gnpk::kTwKcap;
  const int ST = (npt + 1 + 7) & ~7;  // int16 entry starts, padded to 16 bytes
  std::vector<int> K(T), off(T);
  std::int64_t total16 = 0;
  for (std::int64_t t = 0; t < T; ++t) {
    const std::int64_t n0 = t * npt, n1 = std::min(n, n0 + npt);
    const int m = hrp[n1] - hrp[n0];
    const int kr = (m + 7) & ~7;
    if (kr > KMAX) return false;
    for (int k = hrp[n0]; k < hrp[n1]; ++k)
      if (widx(t, hci[k]) < 0) return false;
    K[t] = kr;
    off[t] = static_cast<int>(total16);
    total16 += (2 * ST + 6 * kr) / 16;
  }
  std::vector<uint8_t> buf(std::max<std::int64_t>(total16 * 16, 16), 0);
  for (std::int64_t t = 0; t < T; ++t) {
    uint8_t* sl = buf.data() + (std::size_t)off[t] * 16;
    uint16_t* st = reinterpret_cast<uint16_t*>(sl);
    uint16_t* ri = st + ST;
    float* vv = reinterpret_cast<float*>(sl + 2 * ST + 2 * K[t]);
    const std::int64_t n0 = t * npt;
    const int kb = hrp[n0];
    for (int i = 0; i <= npt; ++i) st[i] = static_cast<uint16_t>(hrp[std::min(n, n0 + i)] - kb);
    for (int k = kb; k < hrp[std::min(n, n0 + npt)]; ++k) {
      ri[k - kb] = static_cast<uint16_t>(widx(t, hci[k]));
      vv[k - kb] = static_cast<float>(h.values[k]);
    }
  }
  std::vector<int> ord;
  ord.reserve(T);
  for (int s0 = 0; s0 < S; ++s0)
    for (std::int64_t t = s0; t < T; t += S) ord.push_back(static_cast<int>(t));
  L->sl.upload(buf.data(), buf.size());
  L->off.upload(off.data(), off.size());
  L->k.upload(K.data(), K.size());
  L->order.upload(ord.data(), ord.size());
  L->S = S;
  L->ok = true;
  has_tw = true;
  return true;
}

// Strip-window pair-union layout (see DevCsr::pw): tiles ordered in strips
// of stride S, every column of tile u inside the halo-extended row windows of
// tiles u - S, u, u + S, at most GNPC_KCAPPW union entries per row pair.
// GNPC_NO_PW=1 disables it.
void gnpc_csr_s::build_pw(const std::vector<int>& hrp, const std::vector<int>& hci, const std::vector<float>& hv) {
  has_pw = false;
  if (!has_pairs || n_long != 0) return;
  if (const char* e = std::getenv("GNPC_NO_PW"); e && std::string(e) == "1") return;
  const std::int64_t n = h.n;
  constexpr int TM = 128, NG = TM / 2, H = gnpk::kPwHalo, WR = gnpk::kPwRows;
  constexpr int KMAX = gnpk::SellCfg<32, 7>::KCAP;
  const std::int64_t T = (n + TM - 1) / TM;
  // short strips make most tiles chunk starts (three fresh windows each):
  // at least 4 tiles per SM (GNPC_PW_MIN_TILES overrides, for tests)
  std::int64_t min_tiles = 4 * 148;
  if (const char* e = std::getenv("GNPC_PW_MIN_TILES")) min_tiles = std::atoll(e);
  if (T < min_tiles) return;
  const int S = dominant_tile_stride(hrp, hci, 128);
  if (S < 2) return;
  // entry index: the row R = 144 w + r of the windows (a, b, c) laid end to
  // end, as the byte offset 128 R with the SWIZZLE_128B chunk bits of lane
  // group 0 (16 (R & 7)); -1 if the column is outside the three windows
  auto enc = [](int R) { return 128 * R + 16 * (R & 7); };
  auto widx = [&](std::int64_t t, int c) -> int {
    const std::int64_t b1 = t * TM - H;
    if (c >= b1 && c < b1 + WR) return enc(WR + static_cast<int>(c - b1));
    const std::int64_t b0 = (t - S) * TM - H;
    if (c >= b0 && c < b0 + WR) return enc(static_cast<int>(c - b0));
    const std::int64_t b2 = (t + S) * TM - H;
    if (c >= b2 && c < b2 + WR) return enc(2 * WR + static_cast<int>(c - b2));
    return -1;
  };
  // per tile: union entries per pair, padded to a multiple of 4
  std::vector<int> K(T, 0), off(T, 0);
  std::int64_t total16 = 0;
  for (std::int64_t t = 0; t < T; ++t) {
    int kt = 0;
    for (int g = 0; g < NG; ++g) {
      const std::int64_t i0 = t * TM + 2 * g;
      int s0 = i0 < n ? hrp[i0] : 0, e0 = i0 < n ? hrp[i0 + 1] : 0;
      int s1 = i0 + 1 < n ? hrp[i0 + 1] : 0, e1 = i0 + 1 < n ? hrp[i0 + 2] : 0;
      int u = 0;
      while (s0 < e0 || s1 < e1) {
        int c;
        if (s1 >= e1 || (s0 < e0 && hci[s0] < hci[s1])) c = hci[s0++];
        else if (s0 >= e0 || hci[s1] < hci[s0]) c = hci[s1++];
        else { c = hci[s0++]; ++s1; }
        if (widx(t, c) < 0) return;  // a column outside the three windows
        ++u;
      }
      kt = std::max(kt, u);
    }
    kt = (kt + 3) & ~3;
    if (kt > KMAX) return;
    K[t] = kt;
    off[t] = static_cast<int>(total16);
    total16 += (std::int64_t)kt * NG * 10 / 16;  // kt % 4 == 0: 640-byte multiples
  }
  std::vector<uint8_t> buf(std::max<std::int64_t>(total16 * 16, 16), 0);
  for (std::int64_t t = 0; t < T; ++t) {
    const int kt = K[t];
    uint8_t* sl = buf.data() + (std::size_t)off[t] * 16;
    uint16_t* idx = reinterpret_cast<uint16_t*>(sl);
    float* w0 = reinterpret_cast<float*>(sl + NG * kt * 2);
    float* w1 = w0 + NG * kt;
    for (int g = 0; g < NG; ++g) {
      const std::int64_t i0 = t * TM + 2 * g;
      int s0 = i0 < n ? hrp[i0] : 0, e0 = i0 < n ? hrp[i0 + 1] : 0;
      int s1 = i0 + 1 < n ? hrp[i0 + 1] : 0, e1 = i0 + 1 < n ? hrp[i0 + 2] : 0;
      int u = 0;
      auto put = [&](int c, float a0, float a1) {
        idx[g * kt + u] = static_cast<uint16_t>(widx(t, c));
        w0[g * kt + u] = a0;
        w1[g * kt + u] = a1;
        ++u;
      };
      while (s0 < e0 || s1 < e1) {
        if (s1 >= e1 || (s0 < e0 && hci[s0] < hci[s1])) {
          put(hci[s0], hv[s0], 0.f);
          ++s0;
        } else if (s0 >= e0 || hci[s1] < hci[s0]) {
          put(hci[s1], 0.f, hv[s1]);
          ++s1;
        } else {
          put(hci[s0], hv[s0], hv[s1]);
          ++s0;
          ++s1;
        }
      }
      for (; u < kt; ++u) {  // padding: the pair's first row in its own window, weight 0
        idx[g * kt + u] = static_cast<uint16_t>(enc(WR + H + 2 * g));
        w0[g * kt + u] = 0.f;
        w1[g * kt + u] = 0.f;
      }
    }
  }
  std::vector<int> ord;
  ord.reserve(T);
  for (int s0 = 0; s0 < S; ++s0)
    for (std::int64_t t = s0; t < T; t += S) ord.push_back(static_cast<int>(t));
  pw.upload(buf.data(), buf.size());
  pw_off.upload(off.data(), off.size());
  pw_k.upload(K.data(), K.size());
  pw_order.upload(ord.data(), ord.size());
  pw_S = S;
  has_pw = true;
}

// The apply path's view: the length-sorted renumbering when it was built
// (has_perm), else dev() itself.
gnpk::DevCsr gnpc_csr_s::dev_apply() {
  gnpk::DevCsr d = dev();
  if (has_perm) {
    d.rp = prm_rp.p;
    d.ci = prm_ci.p;
    d.v = prm_v.p;
    d.perm = perm.p;
  }
  return d;
}

gnpk::DevCsr gnpc_csr_s::dev() {
  upload();
  gnpk::DevCsr d;
  d.n = static_cast<int>(h.n);
  d.nnz = static_cast<int>(h.nnz());
  d.rp = rp.p;
  d.ci = ci.p;
  d.v = v.p;
  d.perm = nullptr;
  d.long_rows = n_long ? long_rows.p : nullptr;
  d.n_long = n_long;
  d.rps = rps.p;
  d.cis = cis.p;
  d.vs = vs.p;
  d.tflag = tflag.p;
  d.sell = has_sell ? sell.p : nullptr;
  d.sell_off = has_sell ? sell_off.p : nullptr;
  d.sell_k = has_sell ? sell_k.p : nullptr;
  d.tw = nullptr;  // training layouts are per batch size: bind_tw
  d.tw_off = nullptr;
  d.tw_k = nullptr;
  d.tw_order = nullptr;
  d.tw_S = 0;
  d.pw = has_pw ? pw.p : nullptr;
  d.pw_off = has_pw ? pw_off.p : nullptr;
  d.pw_k = has_pw ? pw_k.p : nullptr;
  d.pw_order = has_pw ? pw_order.p : nullptr;
  d.pw_S = has_pw ? pw_S : 0;
  d.psell = has_pairs ? psell.p : nullptr;
  d.psell_off = has_pairs ? psell_off.p : nullptr;
  d.psell_k = has_pairs ? psell_k.p : nullptr;
  static const bool hint_off = [] {
    const char* e = std::getenv("GNPC_L2HINT");
    return e && std::string(e) == "0";
  }();
  d.l2hint = (l2hint && !hint_off) ? 1 : 0;
  return d;
}

// ====================================================================== model
// Index maps from the flat f64 parameter vector (reference order,
// src/gnn.cpp:40-55) into the device fp32 layout and the per-layer operands.
// The host uses them here; the trainer uploads them and regenerates the device
// copies on the GPU after every Adam step (k_gather_params / k_gather_split).
void gnpc_model_s::build_maps() {
  if (!map_view.empty()) return;
  const std::int64_t d = dims.d, H = dims.hidden, L = dims.layers;
  const gnp_b200::ParamLayout lay = gnp_b200::param_layout(dims);
  // every section starts on a 16-byte boundary (float4 loads)
  auto al = [](std::size_t x) { return (x + 3) & ~std::size_t(3); };
  const std::size_t Ha = al(H);
  o_enc1 = 0;
  o_enc1b = Ha;
  o_enc2 = 2 * Ha;
  o_enc2b = o_enc2 + Ha * dp;
  o_uw = o_enc2b + dp;
  o_dec1 = o_uw + (std::size_t)L * 2 * dp * dp;
  o_dec1b = o_dec1 + al((std::size_t)dp * H);
  o_dec2 = o_dec1b + Ha;
  o_dec2b = o_dec2 + Ha;
  const std::size_t total = o_dec2b + 4;
  map_view.assign(total, -1);
  for (std::int64_t h = 0; h < H; ++h) {
    map_view[o_enc1 + h] = (int)(lay.enc1 + h);
    map_view[o_enc1b + h] = (int)(lay.enc1_b + h);
    map_view[o_dec1b + h] = (int)(lay.dec1_b + h);
    map_view[o_dec2 + h] = (int)(lay.dec2 + h);
    for (std::int64_t j = 0; j < d; ++j) {
      map_view[o_enc2 + h * dp + j] = (int)(lay.enc2 + j * H + h);  // enc2 (h, j), col-major H x d
      map_view[o_dec1 + j * H + h] = (int)(lay.dec1 + h * d + j);   // dec1 (j, h), col-major d x H
    }
  }
  for (std::int64_t j = 0; j < d; ++j) map_view[o_enc2b + j] = (int)(lay.enc2_b + j);
  map_view[o_dec2b] = (int)lay.dec2_b;
  // per-layer B operands, element (output j, input k), k < DP: x part, DP.. : ÂX part
  //   forward  : [U; W](k, j)   = U(k, j), W(k - DP, j)
  //   backward : [Uᵀ; Wᵀ](k, j) = U(j, k), W(j, k - DP)   (gX = gpre Uᵀ + Âᵀgpre Wᵀ)
  auto fwd_src = [&](std::int64_t l, int j, int k) -> int {
    if (j >= d) return -1;
    if (k < d) return (int)(lay.u[l] + j * d + k);
    if (k >= dp && k - dp < d) return (int)(lay.w[l] + j * d + (k - dp));
    return -1;
  };
  auto bwd_src = [&](std::int64_t l, int j, int k) -> int {
    if (j >= d) return -1;
    if (k < d) return (int)(lay.u[l] + k * d + j);
    if (k >= dp && k - dp < d) return (int)(lay.w[l] + (k - dp) * d + j);
    return -1;
  };
  const int K = 2 * dp;
  const std::size_t bf = (std::size_t)dp * K;
  for (std::int64_t l = 0; l < L; ++l)
    for (int k = 0; k < K; ++k)
      for (int j = 0; j < dp; ++j) map_view[o_uw + (std::size_t)l * 2 * dp * dp + (std::size_t)k * dp + j] =
          fwd_src(l, j, k);
  map_bt_fwd.assign((std::size_t)L * bf, -1);
  map_bt_bwd.assign((std::size_t)L * bf, -1);
  for (std::int64_t l = 0; l < L; ++l)
    for (int j = 0; j < dp; ++j)
      for (int k = 0; k < K; ++k) {
        map_bt_fwd[(std::size_t)l * bf + (std::size_t)j * K + k] = fwd_src(l, j, k);
        map_bt_bwd[(std::size_t)l * bf + (std::size_t)j * K + k] = bwd_src(l, j, k);
      }
  if (dp == 16 || dp == 32) {
    map_tc_fwd.assign((std::size_t)L * 2 * bf, -1);
    map_tc_bwd.assign((std::size_t)L * 2 * bf, -1);
    part_tc.assign((std::size_t)L * 2 * bf, 0);
    for (std::int64_t l = 0; l < L; ++l)
      for (int j = 0; j < dp; ++j)
        for (int k = 0; k < K; ++k) {
          const std::size_t off = gnpk::tc::sw128_off(j, k, dp) / 4;
          const std::size_t hi = (std::size_t)l * 2 * bf + off, lo = hi + bf;
          map_tc_fwd[hi] = map_tc_fwd[lo] = fwd_src(l, j, k);
          map_tc_bwd[hi] = map_tc_bwd[lo] = bwd_src(l, j, k);
          part_tc[lo] = 1;
        }
    // k_layer_sell: per layer four DP x DP operands, block b = 2*part + hi
    // ([Bu_lo | Bu_hi | Bw_lo | Bw_hi]) in the DP-wide swizzle; element (j, k)
    // of part p = [U; W](k + p*DP, j)
    const std::size_t pb = (std::size_t)dp * dp;
    map_tc_pair.assign((std::size_t)L * 4 * pb, -1);
    map_tc_pair_bwd.assign((std::size_t)L * 4 * pb, -1);
    part_pair.assign((std::size_t)L * 4 * pb, 0);
    for (std::int64_t l = 0; l < L; ++l)
      for (int b = 0; b < 4; ++b)
        for (int j = 0; j < dp; ++j)
          for (int k = 0; k < dp; ++k) {
            const std::size_t off = (dp == 32 ? gnpk::tc::swz_off<32>(j, k) : gnpk::tc::swz_off<16>(j, k)) / 4;
            const std::size_t i = (std::size_t)l * 4 * pb + b * pb + off;
            map_tc_pair[i] = fwd_src(l, j, k + (b >> 1) * dp);
            map_tc_pair_bwd[i] = bwd_src(l, j, k + (b >> 1) * dp);
            part_pair[i] = (b & 1) ? 0 : 1;  // 1 = lo part
          }
  }
}

static float tf32_rna(float x) {
  std::uint32_t u;
  std::memcpy(&u, &x, 4);
  u = (u + 0x1000u) & ~0x1FFFu;  // cvt.rna: round half away from zero on the magnitude
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}

void gnpc_model_s::build_view() {
  build_maps();
  const std::int64_t d = dims.d, H = dims.hidden, L = dims.layers;
  const gnp_b200::ParamLayout lay = gnp_b200::param_layout(dims);
  auto al = [](std::size_t x) { return (x + 3) & ~std::size_t(3); };
  const double* p = params.data();
  std::vector<float> f(map_view.size());
  for (std::size_t i = 0; i < f.size(); ++i) f[i] = map_view[i] >= 0 ? (float)p[map_view[i]] : 0.f;
  P.upload(f.data(), f.size());
  GNPC_CUDA(cudaDeviceSynchronize());
  view.enc1 = P.p + o_enc1;
  view.enc1_b = P.p + o_enc1b;
  view.enc2 = P.p + o_enc2;
  view.enc2_b = P.p + o_enc2b;
  view.uw = P.p + o_uw;
  view.dec1 = P.p + o_dec1;
  view.dec1_b = P.p + o_dec1b;
  view.dec2 = P.p + o_dec2;
  view.dec2_bp = P.p + o_dec2b;
  view.dec2_b = (float)p[lay.dec2_b];
  view.hidden = (int)H;
  view.layers = (int)L;
  // Lift as an exact piecewise-linear function of the scalar v (f64 tables):
  // kinks t_h = -b1_h/enc1_h; on each interval the active hidden set is fixed,
  // so x1 = (Σ_active enc1_h enc2_h) v + (Σ_active b1_h enc2_h + enc2_b).
  {
    std::vector<double> kinks;
    for (std::int64_t h = 0; h < H; ++h)
      if (p[lay.enc1 + h] != 0.0) kinks.push_back(-p[lay.enc1_b + h] / p[lay.enc1 + h]);
    std::sort(kinks.begin(), kinks.end());
    kinks.erase(std::unique(kinks.begin(), kinks.end()), kinks.end());
    const int nb = (int)kinks.size();
    std::vector<float> lt(std::max(nb, 1)), la((std::size_t)(nb + 1) * dp, 0.f),
        lb((std::size_t)(nb + 1) * dp, 0.f);
    for (int k = 0; k < nb; ++k) lt[k] = (float)kinks[k];
    for (int k = 0; k <= nb; ++k) {
      // representative point strictly inside interval k
      double vr;
      if (nb == 0) vr = 0.0;
      else if (k == 0) vr = kinks[0] - 1.0 - std::abs(kinks[0]);
      else if (k == nb) vr = kinks[nb - 1] + 1.0 + std::abs(kinks[nb - 1]);
      else vr = 0.5 * (kinks[k - 1] + kinks[k]);
      for (std::int64_t j = 0; j < d; ++j) {
        double a_ = 0.0, b_ = p[lay.enc2_b + j];
        for (std::int64_t h = 0; h < H; ++h) {
          const double w = p[lay.enc1 + h], bb = p[lay.enc1_b + h];
          if (w * vr + bb > 0.0) {
            const double e = p[lay.enc2 + j * H + h];
            a_ += w * e;
            b_ += bb * e;
          }
        }
        la[(std::size_t)k * dp + j] = (float)a_;
        lb[(std::size_t)k * dp + j] = (float)b_;
      }
    }
    std::vector<float> lift;
    lift.insert(lift.end(), lt.begin(), lt.end());
    const std::size_t oa = al(lift.size());
    lift.resize(oa, 0.f);
    lift.insert(lift.end(), la.begin(), la.end());
    const std::size_t ob = al(lift.size());
    lift.resize(ob, 0.f);
    lift.insert(lift.end(), lb.begin(), lb.end());
    LIFT.upload(lift.data(), lift.size());
    GNPC_CUDA(cudaDeviceSynchronize());
    view.lift_t = LIFT.p;
    view.lift_a = LIFT.p + oa;
    view.lift_b = LIFT.p + ob;
    view.nbreak = nb;
  }
  // tcgen05 B operands (forward): [U; W]ᵀ split into tf32 hi (round-to-nearest)
  // and lo = v - hi, 128-byte-swizzled K-major.
  if (!map_tc_fwd.empty()) {
    std::vector<float> t(map_tc_fwd.size());
    for (std::size_t i = 0; i < t.size(); ++i) {
      const float v = map_tc_fwd[i] >= 0 ? (float)p[map_tc_fwd[i]] : 0.f;
      const float h = tf32_rna(v);
      t[i] = part_tc[i] ? v - h : h;
    }
    UWTC.upload(t.data(), t.size());
    std::vector<float> u(map_tc_pair.size());
    for (std::size_t i = 0; i < u.size(); ++i) {
      const float v = map_tc_pair[i] >= 0 ? (float)p[map_tc_pair[i]] : 0.f;
      const float h = tf32_rna(v);
      u[i] = part_pair[i] ? v - h : h;
    }
    UWP.upload(u.data(), u.size());
    GNPC_CUDA(cudaDeviceSynchronize());
  }
  (void)L;
}

void gnpc_model_s::ensure_workspace() {
  const std::size_t n = (std::size_t)a->h.n;
  X[0].ensure(n * dp);
  X[1].ensure(n * dp);
  if (a->n_long) {
    AXL.ensure(n * dp);
    LPART.ensure((std::size_t)a->n_chunks * dp);
  }
  if (sms == 0) sms = num_sms();
  norm_grid = 2 * sms;
  partials.ensure(std::max(norm_grid, sms));
  if (!gbar.p) {
    gbar.alloc(1);
    GNPC_CUDA(cudaMemset(gbar.p, 0, sizeof(unsigned long long)));
    gbar_host = 0;
  }
  if (!ticket.p) {
    ticket.alloc(1);
    GNPC_CUDA(cudaMemset(ticket.p, 0, sizeof(unsigned)));
  }
  sc.ensure(1);
  if ((dp == 16 || dp == 32) && n > 0) {
    for (int c = 0; c < 2; ++c)
      if (tm_base[c] != X[c].p) {
        tmX[c] = make_rows_map(X[c].p, (std::int64_t)n, dp, 128,
                               dp == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B);
        // the strip windows' halo-extended tiles (d = 32; unused at d = 16)
        tmXw[c] = make_rows_map(X[c].p, (std::int64_t)n, dp, dp == 32 ? gnpk::kPwRows : 128,
                                dp == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B);
        tm_base[c] = X[c].p;
      }
  }
}

bool gnpc_model_s::fused_eligible() {
  a->upload();
  // (length-sorted nodes: the input gather / output scatter would touch host
  // memory at random; those applies stage through device buffers)
  if (dp != 16 || !use_tc || a->n_long != 0 || a->h.n == 0 || a->has_perm) return false;
  if (gnpc_impl::sell_kernel_off() || gnpc_impl::fused_apply_off()) return false;
  const size_t smem = a->has_sell ? gnpk::SellCfg<16, 0>::smem_bytes(dims.hidden, true)
                                  : gnpk::SellCfg<16, 1>::smem_bytes(dims.hidden, true);
  return smem <= 226 * 1024;
}

template <typename InT, typename OutT>
void gnpc_model_s::launch_apply(const InT* in, OutT* out, cudaStream_t s, const int* skip,
                                ApplyProf* prof) {
  if (trainer_dirty)
    throw std::logic_error("model parameters were updated by a trainer: call gnpc_trainer_sync_model "
                           "before applying the model");
  a->upload();
  ensure_workspace();
  switch (dp) {
    case 4: ApplyLaunch<4>::run(*this, in, out, s, skip, prof); break;
    case 8: ApplyLaunch<8>::run(*this, in, out, s, skip, prof); break;
    case 16: ApplyLaunch<16>::run(*this, in, out, s, skip, prof); break;
    case 32: ApplyLaunch<32>::run(*this, in, out, s, skip, prof); break;
    case 64: ApplyLaunch<64>::run(*this, in, out, s, skip, prof); break;
    default: throw Unsupported("unsupported padded width");
  }
}
template void gnpc_model_s::launch_apply<float, float>(const float*, float*, cudaStream_t,
                                                      const int*, ApplyProf*);
template void gnpc_model_s::launch_apply<double, double>(const double*, double*, cudaStream_t,
                                                        const int*, ApplyProf*);

// ====================================================================== FGMRES driver
namespace {

using gnpk::KrylovDev;
using gnpk::KState;

struct HostOp {
  gnpc_host_operator fn;
  void* ctx;
};

void* ortho_kernel_for(int ept) {
  switch (ept) {
    case 0: return (void*)gnpk::k_krylov_ortho<0>;
    case 1: return (void*)gnpk::k_krylov_ortho<1>;
    case 2: return (void*)gnpk::k_krylov_ortho<2>;
    case 4: return (void*)gnpk::k_krylov_ortho<4>;
    case 8: return (void*)gnpk::k_krylov_ortho<8>;
    case 16: return (void*)gnpk::k_krylov_ortho<16>;
  }
  return nullptr;
}

struct OrthoPlan {
  void* kern;
  int grid;
  int block = gnpk::kThreads;
  size_t smem = 0;
  int chunk = 0;  // on-chip variant: rows per CTA
};

// The MGS sweep is one grid barrier per basis vector, so the barrier's cost
// (which grows with the CTA count) is paid j+1 times per pass: prefer few
// CTAs (1, then 2 per SM) holding w in registers with a larger EPT, and only
// then more CTAs.  (C2: ~1180 CTAs at EPT 1 -> 148 CTAs at EPT 8.)  Vectors
// too long for that keep w in registers + shared memory of one 1024-thread
// CTA per SM (k_krylov_ortho_onchip, C5) before falling back to w in HBM.
OrthoPlan plan_ortho(int n) {
  const int sms = num_sms();
  static const bool onchip_off = [] {
    const char* e = std::getenv("GNPC_NO_ONCHIP_MGS");
    return e && std::string(e) == "1";
  }();
  static const bool force_onchip = [] {  // test hook: exercise the on-chip variant at small n
    const char* e = std::getenv("GNPC_FORCE_ONCHIP_MGS");
    return e && std::string(e) == "1";
  }();
  for (int per : {1, 2, 4}) {
    for (int ept : {1, 2, 4, 8, 16}) {
      if (force_onchip) break;
      int per_sm = 0;
      GNPC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ortho_kernel_for(ept),
                                                              gnpk::kThreads, 0));
      if (per_sm < per) continue;
      const long long cap = (long long)per * sms * gnpk::kThreads * ept;
      if (n <= cap) return {ortho_kernel_for(ept), per * sms};
    }
  }
  if (!onchip_off) {
    constexpr int NR = 4;
    auto kern = (const void*)gnpk::k_krylov_ortho_onchip<NR>;
    cudaFuncAttributes fa{};
    GNPC_CUDA(cudaFuncGetAttributes(&fa, kern));
    const int smem_cap = 227 * 1024 - (int)fa.sharedSizeBytes - 1024;
    const long long chunk = ((long long)n + sms - 1) / sms;
    const long long need_smem = std::max<long long>(0, chunk - (long long)NR * gnpk::kOnchipThreads) * 8;
    if (need_smem <= smem_cap) {
      set_smem_attr(kern, (int)std::max<long long>(need_smem, 8));
      int per_sm = 0;
      GNPC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, gnpk::kOnchipThreads,
                                                              (size_t)std::max<long long>(need_smem, 8)));
      if (per_sm >= 1)
        return {(void*)kern, sms, gnpk::kOnchipThreads, (size_t)std::max<long long>(need_smem, 8), (int)chunk};
    }
  }
  for (int ept : {1, 2, 4, 8, 16}) {
    int per_sm = 0;
    GNPC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ortho_kernel_for(ept),
                                                            gnpk::kThreads, 0));
    const long long cap = (long long)per_sm * sms * gnpk::kThreads * ept;
    if (per_sm > 0 && n <= cap) return {ortho_kernel_for(ept), per_sm * sms};
  }
  int per_sm = 0;
  GNPC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ortho_kernel_for(0),
                                                          gnpk::kThreads, 0));
  return {ortho_kernel_for(0), std::max(1, per_sm) * sms};
}

__global__ void k_init_state(const double* __restrict__ b, int n, double* partials,
                             unsigned* ticket, KState* st, double rtol, int maxiters,
                             double timeout_secs) {
  __shared__ double scratch[32];
  __shared__ bool last;
  double p = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    p = fma(b[i], b[i], p);
  p = gnpk::block_sum(p, scratch);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = p;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double t = 0.0;
  for (int z = threadIdx.x; z < (int)gridDim.x; z += blockDim.x)
    t += reinterpret_cast<volatile double*>(partials)[z];
  t = gnpk::block_sum(t, scratch);
  if (threadIdx.x == 0) {
    const long long now = (long long)gnpk::globaltimer_ns();
    st->bnorm = sqrt(t);
    st->rtol = rtol;
    st->maxiters = maxiters;
    st->iter = 0;
    st->reorth = 0;
    st->t0 = now;
    st->deadline = timeout_secs < 0.0 ? -1 : now + (long long)(timeout_secs * 1e9);
    st->stop = 0;
    *ticket = 0u;
  }
}

struct HistSink {
  gnpc_history* h;
  std::int64_t len = 0;
  void push(std::int64_t it, double rel, double t) {
    if (h && len < h->capacity) {
      h->iteration[len] = it;
      h->relres[len] = rel;
      h->elapsed[len] = t;
    }
    ++len;
  }
  void set_last(std::int64_t it, double rel, double t) {
    if (h && len - 1 < h->capacity && len > 0) {
      h->iteration[len - 1] = it;
      h->relres[len - 1] = rel;
      h->elapsed[len - 1] = t;
    }
  }
};

// Core of fgmres_solve (src/krylov.cpp:175-277) on device-resident b/x.
int fgmres_core(gnpc_csr_s& A, gnpc_model_s* M, const HostOp* hop, const double* b_dev,
                double* x_dev, const gnpc_solve_config& cfg, gnpc_history* hist,
                cudaStream_t s) {
  need(cfg.restart >= 1, "fgmres: restart must be >= 1");
  need(cfg.maxiters >= 0, "fgmres: maxiters must be >= 0");
  gnpk::DevCsr a = A.dev();
  const int n = a.n;
  const int m = (int)cfg.restart;
  if (!A.kws || A.kws->n != n || A.kws->m != m) {
    auto w = std::make_unique<KrylovWs>();
    w->n = n;
    w->m = m;
    w->V.alloc((size_t)n * (m + 1));
    if (M || hop) w->Z.alloc((size_t)n * m);
    w->w.alloc(n);
    w->vin.alloc(n);
    w->zout.alloc(n);
    w->r.alloc(n);
    w->H.alloc((size_t)(m + 1) * m);
    w->R.alloc((size_t)(m + 1) * m);
    w->cs.alloc(m);
    w->sn.alloc(m);
    w->g.alloc(m + 1);
    w->y.alloc(m);
    w->partials.alloc(2 * 2048);
    w->hist_rel.alloc(m);
    w->hist_t.alloc(m);
    w->ticket.alloc(1);
    GNPC_CUDA(cudaMemset(w->ticket.p, 0, sizeof(unsigned)));
    w->st.alloc(1);
    A.kws = std::move(w);
  }
  KrylovWs& W = *A.kws;
  if ((M || hop) && !W.Z.p) W.Z.alloc((size_t)n * m);
  KrylovDev k{};
  k.n = n;
  k.m = m;
  k.V = W.V.p;
  k.Z = (M || hop) ? W.Z.p : nullptr;
  k.w = W.w.p;
  k.vin = W.vin.p;
  k.zout = W.zout.p;
  k.x = x_dev;
  k.b = b_dev;
  k.r = W.r.p;
  k.H = W.H.p;
  k.R = W.R.p;
  k.cs = W.cs.p;
  k.sn = W.sn.p;
  k.g = W.g.p;
  k.y = W.y.p;
  k.partials = W.partials.p;
  k.ticket = W.ticket.p;
  k.hist_rel = W.hist_rel.p;
  k.hist_t = W.hist_t.p;
  k.st = W.st.p;
  const int sms = num_sms();
  const int vgrid = std::max(1, std::min((n + 255) / 256, sms * 8));
  const int rgrid = std::max(1, std::min((n + 63) / 64, sms * 8));  // 8 rows per warp

  gnpk::KState hs{};
  auto pull_state = [&] {
    GNPC_CUDA(cudaMemcpyAsync(&hs, W.st.p, sizeof(KState), cudaMemcpyDeviceToHost, s));
    GNPC_CUDA(cudaStreamSynchronize(s));
  };

  k_init_state<<<std::min(rgrid, 2048), gnpk::kThreads, 0, s>>>(
      b_dev, n, W.partials.p, W.ticket.p, W.st.p, cfg.rtol, (int)cfg.maxiters,
      cfg.timeout_secs);
  GNPC_LAUNCHED();
  pull_state();
  if (hs.bnorm == 0.0) throw std::invalid_argument("fgmres: zero right-hand side");

  HistSink H{hist};
  gnpk::k_residual<<<std::min(rgrid, 2048), gnpk::kThreads, 0, s>>>(a, k);
  GNPC_LAUNCHED();
  pull_state();
  H.push(0, hs.current, 0.0);
  int status = GNPC_MAXITERS;
  if (hs.current <= cfg.rtol) {
    status = GNPC_CONVERGED;
  } else {
    const OrthoPlan op = plan_ortho(n);
    std::vector<double> hrel(m);
    std::vector<long long> ht(m);
    std::int64_t iter = 0;
    bool done = false;
    std::vector<double> hv_in, hv_out;
    if (hop) {
      hv_in.resize(n);
      hv_out.resize(n);
    }
    while (iter < cfg.maxiters && !done) {
      if (hs.beta == 0.0) throw std::invalid_argument("arnoldi: zero start vector");
      const int cycle = (int)std::min<std::int64_t>(cfg.restart, cfg.maxiters - iter);
      gnpk::k_cycle_begin<<<vgrid, gnpk::kThreads, 0, s>>>(k, cycle);
      GNPC_LAUNCHED();
      for (int j = 0; j < cycle; ++j) {
        if (hop) {
          // host FlexibleOperator: z_j = M(v_j) on host vectors
          pull_state();
          if (hs.stop) break;
          GNPC_CUDA(cudaMemcpyAsync(hv_in.data(), W.vin.p, n * sizeof(double),
                                    cudaMemcpyDeviceToHost, s));
          GNPC_CUDA(cudaStreamSynchronize(s));
          if (hop->fn(hop->ctx, hv_in.data(), hv_out.data(), n) != 0)
            throw std::runtime_error("host preconditioner failed");
          GNPC_CUDA(cudaMemcpyAsync(W.zout.p, hv_out.data(), n * sizeof(double),
                                    cudaMemcpyHostToDevice, s));
        } else if (M) {
          M->launch_apply<double, double>(W.vin.p, W.zout.p, s, &W.st.p->stop);
        }
        gnpk::k_krylov_spmv<<<rgrid, gnpk::kThreads, 0, s>>>(a, k);
        GNPC_LAUNCHED();
        int chunk = op.chunk;
        void* args[] = {&k, &chunk};
        GNPC_CUDA(cudaLaunchCooperativeKernel(op.kern, op.grid, op.block, args, op.smem, s));
        GNPC_LAUNCHED();
      }
      gnpk::k_cycle_solve<<<1, 32, 0, s>>>(k);
      GNPC_LAUNCHED();
      gnpk::k_update_x<<<vgrid, gnpk::kThreads, 0, s>>>(k);
      GNPC_LAUNCHED();
      gnpk::k_residual<<<std::min(rgrid, 2048), gnpk::kThreads, 0, s>>>(a, k);
      GNPC_LAUNCHED();
      pull_state();
      GNPC_CUDA(cudaMemcpyAsync(hrel.data(), W.hist_rel.p, m * sizeof(double),
                                cudaMemcpyDeviceToHost, s));
      GNPC_CUDA(cudaMemcpyAsync(ht.data(), W.hist_t.p, m * sizeof(long long),
                                cudaMemcpyDeviceToHost, s));
      GNPC_CUDA(cudaStreamSynchronize(s));
      for (int q = 0; q < hs.steps; ++q) H.push(iter + q + 1, hrel[q], 1e-9 * (double)ht[q]);
      iter += hs.steps;
      if (hs.singular) {
        status = GNPC_SOLUTION_FAILURE;
        break;
      }
      const double tracked_rel = hs.tracked_rel;
      const double current = hs.current;
      H.set_last(iter, current, 1e-9 * (double)hs.t_end);
      if (current > 10.0 * tracked_rel && current - tracked_rel > 1e-10) {
        status = GNPC_SOLUTION_FAILURE;
        done = true;
      } else if (current <= cfg.rtol) {
        status = GNPC_CONVERGED;
        done = true;
      } else if (hs.breakdown) {
        status = GNPC_BREAKDOWN_EXACT;
        done = true;
      } else if (hs.budget_hit) {
        status = hs.budget_status;
        done = true;
      } else if (hs.deadline >= 0 && hs.t_end + hs.t0 >= hs.deadline) {
        status = GNPC_TIMEOUT;
        done = true;
      }
      if (!done && hs.steps == 0) throw std::runtime_error("fgmres: cycle made no progress");
    }
    if (!done && status != GNPC_SOLUTION_FAILURE) status = GNPC_MAXITERS;
  }
  if (hist) {
    hist->length = H.len;
    hist->reorth = hs.reorth;
  }
  return status;
}

int fgmres_host(gnpc_csr a, gnpc_model m, const HostOp* hop, const double* b, const double* x0,
                const gnpc_solve_config* cfg, double* x, gnpc_history* hist, int* status) {
  return guarded([&] {
    need(a && b && x && cfg && status, "fgmres: null argument");
    require_device();
    if (m) need(m->a->h.n == a->h.n, "fgmres: preconditioner dimension mismatch");
    const std::size_t n = (std::size_t)a->h.n;
    DevBuf<double> db(n), dx(n);
    cudaStream_t s = m ? m->stream : nullptr;
    GNPC_CUDA(cudaMemcpyAsync(db.p, b, n * 8, cudaMemcpyHostToDevice, s));
    if (x0) {
      GNPC_CUDA(cudaMemcpyAsync(dx.p, x0, n * 8, cudaMemcpyHostToDevice, s));
    } else {
      GNPC_CUDA(cudaMemsetAsync(dx.p, 0, n * 8, s));
    }
    *status = fgmres_core(*a, m, hop, db.p, dx.p, *cfg, hist, s);
    GNPC_CUDA(cudaMemcpyAsync(x, dx.p, n * 8, cudaMemcpyDeviceToHost, s));
    GNPC_CUDA(cudaStreamSynchronize(s));
  });
}

}  // namespace

namespace gnpc_impl {
// build_spectral_sampler (src/sampler.cpp:10-39).  The Arnoldi cycle is the
// device FGMRES machinery run for one unpreconditioned cycle of m steps with
// no convergence test (rtol < 0): r0 = b - A·0 = start exactly, V and the raw
// Hessenberg stay in the Krylov workspace and are read back once.
std::unique_ptr<gnpc_sampler_s> build_sampler(gnpc_csr_s& A, std::int64_t m, std::uint64_t seed) {
  if (A.h.n < 2) throw std::invalid_argument("spectral sampler: n must be >= 2");
  if (m < 1) throw std::invalid_argument("spectral sampler: m must be >= 1");
  require_device();
  const std::int64_t n = A.h.n;
  gnp_b200::Rng rng(seed);
  const std::vector<double> start = rng.gaussian_vector(n);
  DevBuf<double> db(n), dx(n);
  GNPC_CUDA(cudaMemcpy(db.p, start.data(), n * 8, cudaMemcpyHostToDevice));
  GNPC_CUDA(cudaMemset(dx.p, 0, n * 8));
  gnpc_solve_config cfg{-1.0, m, m, -1.0};
  (void)fgmres_core(A, nullptr, nullptr, db.p, dx.p, cfg, nullptr, nullptr);
  KrylovWs& W = *A.kws;
  gnpk::KState st{};
  GNPC_CUDA(cudaMemcpy(&st, W.st.p, sizeof st, cudaMemcpyDeviceToHost));
  const std::int64_t k = st.steps;
  if (k < 1 || k > m) throw std::runtime_error("spectral sampler: Arnoldi cycle made no progress");
  std::vector<double> v(n * k), hfull((m + 1) * m), hk((k + 1) * k);
  GNPC_CUDA(cudaMemcpy(v.data(), W.V.p, n * k * 8, cudaMemcpyDeviceToHost));
  GNPC_CUDA(cudaMemcpy(hfull.data(), W.H.p, hfull.size() * 8, cudaMemcpyDeviceToHost));
  for (std::int64_t c = 0; c < k; ++c)
    for (std::int64_t i = 0; i <= k; ++i) hk[c * (k + 1) + i] = hfull[c * (m + 1) + i];
  auto out = std::make_unique<gnpc_sampler_s>();
  out->s = gnp_b200::spectral_from_arnoldi(n, k, std::move(v), hk);
  return out;
}
}  // namespace gnpc_impl

// ====================================================================== C ABI
extern "C" {

int gnpc_abi_version(void) { return GNPC_ABI_VERSION; }
const char* gnpc_last_error(void) { return g_error.c_str(); }

int gnpc_device_count(int* count) {
  return guarded([&] {
    need(count, "null count");
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) {
      cudaGetLastError();
      c = 0;
    }
    *count = c;
  });
}
int gnpc_set_device(int device) {
  return guarded([&] {
    require_device();
    GNPC_CUDA(cudaSetDevice(device));
  });
}
int gnpc_synchronize(void) {
  return guarded([&] {
    require_device();
    GNPC_CUDA(cudaDeviceSynchronize());
  });
}
#ifdef GNPC_TILE_TRACE
extern "C" int gnpc_debug_tile_trace(unsigned long long* out) {  // 64 x 16 stamps (debug builds only)
  return cudaMemcpyFromSymbol(out, gnpk::g_trace, sizeof(unsigned long long) * 64 * 16) == cudaSuccess ? 0 : 1;
}
#endif
int gnpc_launch_count(int64_t* count) {
  return guarded([&] {
    need(count, "null count");
    *count = g_launches.load();
  });
}

// ---------------------------------------------------------------- CSR
int gnpc_csr_from_triplets(int64_t n, int64_t m, const int64_t* rows, const int64_t* cols,
                           const double* vals, gnpc_csr* out) {
  return guarded([&] {
    need(out && m >= 0 && (m == 0 || (rows && cols && vals)), "csr_from_triplets: bad arguments");
    std::vector<std::int64_t> r(rows, rows + m), c(cols, cols + m);
    std::vector<double> v(vals, vals + m);
    auto h = std::make_unique<gnpc_csr_s>();
    h->h = gnp_b200::csr_from_triplets(n, r, c, v);
    *out = h.release();
  });
}

int gnpc_csr_create(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                    const double* values, gnpc_csr* out) {
  return guarded([&] {
    need(out && n >= 0 && row_ptr, "csr_create: bad arguments");
    auto h = std::make_unique<gnpc_csr_s>();
    h->h.n = n;
    h->h.row_ptr.assign(row_ptr, row_ptr + n + 1);
    const std::int64_t nnz = row_ptr[n];
    need(nnz >= 0 && (nnz == 0 || (col_idx && values)), "csr_create: bad arrays");
    h->h.col_idx.assign(col_idx, col_idx + nnz);
    h->h.values.assign(values, values + nnz);
    gnp_b200::csr_validate(h->h);
    *out = h.release();
  });
}

int gnpc_csr_generate(const char* kind, int64_t size, double p0, double p1, uint64_t seed,
                      gnpc_csr* out) {
  return guarded([&] {
    need(kind && out, "csr_generate: bad arguments");
    const std::string k(kind);
    auto h = std::make_unique<gnpc_csr_s>();
    if (k == "convection_diffusion") h->h = gnp_b200::gen_convection_diffusion(size, p0);
    else if (k == "random_nonsymmetric")
      h->h = gnp_b200::gen_random_nonsymmetric(size, (std::int64_t)p0, p1, seed);
    else if (k == "c2_convdiff3d") h->h = gnp_b200::gen_convection_diffusion_3d(size, p0);
    else if (k == "c3_varcoeff2d") h->h = gnp_b200::gen_varcoeff_diffusion_2d(size, p0, seed);
    else if (k == "c4_powerlaw") h->h = gnp_b200::gen_powerlaw_random(size, p0, 4, 2048, seed);
    else if (k == "c5_aniso9pt") h->h = gnp_b200::gen_anisotropic_9pt(size, p0, p1);
    else throw std::invalid_argument("csr_generate: unknown kind " + k);
    *out = h.release();
  });
}

int gnpc_csr_read_matrix_market(const char* path, gnpc_csr* out) {
  return guarded([&] {
    need(path && out, "read_matrix_market: bad arguments");
    auto h = std::make_unique<gnpc_csr_s>();
    h->h = gnp_b200::read_matrix_market_file(path);
    *out = h.release();
  });
}

int gnpc_csr_info(gnpc_csr a, int64_t* n, int64_t* nnz) {
  return guarded([&] {
    need(a, "null csr");
    if (n) *n = a->h.n;
    if (nnz) *nnz = a->h.nnz();
  });
}

int gnpc_csr_device_layout(gnpc_csr a, int* uploaded, int* sliced_ell, int* long_rows) {
  return guarded([&] {
    need(a, "null csr");
    if (uploaded) *uploaded = a->dev_ready ? 1 : 0;
    if (sliced_ell)
      *sliced_ell = (a->has_sell ? 1 : 0) | (a->has_pairs ? 2 : 0) | (a->has_pw ? 4 : 0) | (a->has_perm ? 32 : 0) |
                    (a->has_tw ? 16 : 0);
    if (long_rows) *long_rows = a->n_long;
  });
}

int gnpc_csr_export(gnpc_csr a, int64_t* row_ptr, int64_t* col_idx, double* values) {
  return guarded([&] {
    need(a, "null csr");
    if (row_ptr) std::copy(a->h.row_ptr.begin(), a->h.row_ptr.end(), row_ptr);
    if (col_idx) std::copy(a->h.col_idx.begin(), a->h.col_idx.end(), col_idx);
    if (values) std::copy(a->h.values.begin(), a->h.values.end(), values);
  });
}

int gnpc_csr_gershgorin_gamma(gnpc_csr a, double* gamma) {
  return guarded([&] {
    need(a && gamma, "null argument");
    *gamma = gnp_b200::gershgorin_gamma(a->h);
  });
}

int gnpc_csr_prescale(gnpc_csr a, double gamma, gnpc_csr* out) {
  return guarded([&] {
    need(a && out, "null argument");
    auto h = std::make_unique<gnpc_csr_s>();
    h->h = gnp_b200::prescale(a->h, gamma);
    *out = h.release();
  });
}

int gnpc_csr_transpose(gnpc_csr a, gnpc_csr* out) {
  return guarded([&] {
    need(a && out, "null argument");
    auto h = std::make_unique<gnpc_csr_s>();
    h->h = gnp_b200::transpose(a->h);
    *out = h.release();
  });
}

int gnpc_csr_hash(gnpc_csr a, uint64_t* hash) {
  return guarded([&] {
    need(a && hash, "null argument");
    *hash = gnp_b200::csr_content_hash(a->h);
  });
}

int gnpc_csr_destroy(gnpc_csr a) {
  return guarded([&] { delete a; });
}

int gnpc_spmv(gnpc_csr a, const double* x, double* y) {
  return guarded([&] {
    need(a && x && y, "spmv: null argument");
    gnpk::DevCsr d = a->dev();
    const std::size_t n = (std::size_t)a->h.n;
    DevBuf<double> dx(n), dy(n);
    GNPC_CUDA(cudaMemcpy(dx.p, x, n * 8, cudaMemcpyHostToDevice));
    const int grid = std::max(1, std::min((int)((n + 63) / 64), num_sms() * 8));
    gnpk::k_spmv_f64<<<grid, gnpk::kThreads>>>(d, dx.p, dy.p);
    GNPC_LAUNCHED();
    GNPC_CUDA(cudaMemcpy(y, dy.p, n * 8, cudaMemcpyDeviceToHost));
  });
}

int gnpc_gaussian_vector(uint64_t seed, int64_t n, double* out) {
  return guarded([&] {
    need(out && n >= 0, "gaussian_vector: bad arguments");
    gnp_b200::Rng rng(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = rng.gaussian();
  });
}

// ---------------------------------------------------------------- model
int gnpc_param_count(int64_t d, int64_t hidden, int64_t layers, int64_t* count) {
  return guarded([&] {
    need(count, "null count");
    need(d >= 1 && hidden >= 1 && layers >= 1, "init_params: dims must be >= 1");
    *count = gnp_b200::param_layout({d, hidden, layers}).total;
  });
}

int gnpc_init_params(int64_t d, int64_t hidden, int64_t layers, uint64_t seed, double* params) {
  return guarded([&] {
    need(params, "null params");
    const auto p = gnp_b200::init_params({d, hidden, layers}, seed);
    std::copy(p.begin(), p.end(), params);
  });
}

int gnpc_model_create(gnpc_csr ahat, int64_t d, int64_t hidden, int64_t layers,
                      const double* params, gnpc_model* out) {
  return guarded([&] {
    need(ahat && params && out, "model_create: null argument");
    need(d >= 1 && hidden >= 1 && layers >= 1, "model_create: dims must be >= 1");
    if (d > 64) throw Unsupported("model_create: d > 64 is not supported by the device kernels");
    if (hidden > 256) throw Unsupported("model_create: hidden > 256 is not supported");
    require_device();
    auto m = std::make_unique<gnpc_model_s>();
    m->a = ahat;
    m->dims = {d, hidden, layers};
    m->dp = 4;
    while (m->dp < d) m->dp *= 2;
    const char* no_tc = std::getenv("GNPC_NO_TC");
    m->use_tc = (m->dp == 16 || m->dp == 32) && !(no_tc && no_tc[0] == '1');
    m->params.assign(params, params + gnp_b200::param_layout(m->dims).total);
    GNPC_CUDA(cudaStreamCreateWithFlags(&m->stream, cudaStreamNonBlocking));
    m->build_view();
    *out = m.release();
  });
}

int gnpc_model_set_params(gnpc_model m, const double* params) {
  return guarded([&] {
    need(m && params, "null argument");
    m->params.assign(params, params + m->params.size());
    GNPC_CUDA(cudaStreamSynchronize(m->stream));
    m->build_view();
    m->trainer_dirty = false;
  });
}

int gnpc_model_get_params(gnpc_model m, double* params) {
  return guarded([&] {
    need(m && params, "null argument");
    if (m->trainer_dirty)
      throw std::logic_error("model parameters were updated by a trainer: call gnpc_trainer_sync_model "
                             "first");
    std::copy(m->params.begin(), m->params.end(), params);
  });
}

int gnpc_model_dims(gnpc_model m, int64_t* d, int64_t* hidden, int64_t* layers) {
  return guarded([&] {
    need(m, "null model");
    if (d) *d = m->dims.d;
    if (hidden) *hidden = m->dims.hidden;
    if (layers) *layers = m->dims.layers;
  });
}

int gnpc_model_destroy(gnpc_model m) {
  return guarded([&] {
    if (!m) return;
    if (m->stream) cudaStreamSynchronize(m->stream);
    cudaStream_t s = m->stream;
    delete m;
    if (s) cudaStreamDestroy(s);
  });
}

int gnpc_apply(gnpc_model m, const double* b, double* out) {
  return guarded([&] {
    need(m && b && out, "apply: null argument");
    const std::size_t n = (std::size_t)m->a->h.n;
    m->io_in.ensure(n);
    m->io_out.ensure(n);
    // pinned (page-locked) caller buffers and the one-launch apply: the
    // kernel reads b and writes M(b) through their device aliases
    // (zero-copy), so the transfers overlap the norm pass and the last layer
    cudaPointerAttributes pa{}, po{};
    if (m->fused_eligible() && cudaPointerGetAttributes(&pa, b) == cudaSuccess &&
        cudaPointerGetAttributes(&po, out) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
        po.type == cudaMemoryTypeHost && pa.devicePointer != nullptr && po.devicePointer != nullptr) {
      m->fused_stash = m->io_in.p;
      m->launch_apply<double, double>(static_cast<const double*>(pa.devicePointer),
                                      static_cast<double*>(po.devicePointer), m->stream, nullptr);
      m->fused_stash = nullptr;
      GNPC_CUDA(cudaStreamSynchronize(m->stream));
      return;
    }
    cudaGetLastError();  // cudaPointerGetAttributes on unregistered memory is not an error to keep
    GNPC_CUDA(cudaMemcpyAsync(m->io_in.p, b, n * 8, cudaMemcpyHostToDevice, m->stream));
    // per-layer apply with a pinned output buffer: the last layer writes M(b)
    // through its device alias, so the device->host transfer overlaps that
    // layer instead of following it (C5: 33.5 MB of f64 over PCIe)
    if (!m->a->has_perm && cudaPointerGetAttributes(&po, out) == cudaSuccess && po.type == cudaMemoryTypeHost &&
        po.devicePointer != nullptr) {
      m->launch_apply<double, double>(m->io_in.p, static_cast<double*>(po.devicePointer), m->stream, nullptr);
      GNPC_CUDA(cudaStreamSynchronize(m->stream));
      return;
    }
    cudaGetLastError();
    m->launch_apply<double, double>(m->io_in.p, m->io_out.p, m->stream, nullptr);
    GNPC_CUDA(cudaMemcpyAsync(out, m->io_out.p, n * 8, cudaMemcpyDeviceToHost, m->stream));
    GNPC_CUDA(cudaStreamSynchronize(m->stream));
  });
}

int gnpc_apply_device_f32(gnpc_model m, const float* b, float* out, void* stream) {
  return guarded([&] {
    need(m && b && out, "apply: null argument");
    m->launch_apply<float, float>(b, out, (cudaStream_t)stream, nullptr);
  });
}

int gnpc_apply_device_f64(gnpc_model m, const double* b, double* out, void* stream) {
  return guarded([&] {
    need(m && b && out, "apply: null argument");
    m->launch_apply<double, double>(b, out, (cudaStream_t)stream, nullptr);
  });
}

int gnpc_apply_profile(gnpc_model m, const float* b, float* out, void* stream, double* ms_by_kind,
                       int64_t* count_by_kind) {
  return guarded([&] {
    need(m && b && out && ms_by_kind && count_by_kind, "apply_profile: null argument");
    ApplyProf prof;
    cudaStream_t s = (cudaStream_t)stream;
    m->launch_apply<float, float>(b, out, s, nullptr, &prof);
    GNPC_CUDA(cudaStreamSynchronize(s));
    for (std::size_t i = 0; i + 1 < prof.ev.size(); ++i) {
      float ms = 0.f;
      GNPC_CUDA(cudaEventElapsedTime(&ms, prof.ev[i], prof.ev[i + 1]));
      ms_by_kind[prof.kind[i]] += ms;
      count_by_kind[prof.kind[i]] += 1;
    }
    for (cudaEvent_t e : prof.ev) cudaEventDestroy(e);
  });
}

// ---------------------------------------------------------------- checkpoints
int gnpc_checkpoint_save(const char* path, int64_t d, int64_t hidden, int64_t layers,
                         const double* params, gnpc_csr a) {
  return guarded([&] {
    need(path && params && a, "checkpoint_save: null argument");
    const gnp_b200::Dims dm{d, hidden, layers};
    std::vector<double> p(params, params + gnp_b200::param_layout(dm).total);
    gnp_b200::MatrixMeta meta{a->h.n, a->h.nnz(), gnp_b200::csr_content_hash(a->h)};
    const std::string bytes = gnp_b200::checkpoint_bytes(dm, p, meta);
    std::ofstream f(path, std::ios::binary);
    if (!f) throw std::runtime_error(std::string("cannot open ") + path + " for writing");
    f.write(bytes.data(), (std::streamsize)bytes.size());
  });
}

int gnpc_checkpoint_load(const char* path, int64_t* dims3, uint64_t* meta3, double* params) {
  return guarded([&] {
    need(path, "checkpoint_load: null path");
    std::ifstream f(path, std::ios::binary);
    if (!f) throw std::runtime_error(std::string("cannot open ") + path);
    std::stringstream ss;
    ss << f.rdbuf();
    gnp_b200::Dims dm;
    std::vector<double> p;
    gnp_b200::MatrixMeta meta;
    gnp_b200::checkpoint_parse(ss.str(), &dm, &p, &meta);
    if (dims3) {
      dims3[0] = dm.d;
      dims3[1] = dm.hidden;
      dims3[2] = dm.layers;
    }
    if (meta3) {
      meta3[0] = (uint64_t)meta.n;
      meta3[1] = (uint64_t)meta.nnz;
      meta3[2] = meta.hash;
    }
    if (params) std::copy(p.begin(), p.end(), params);
  });
}

// ---------------------------------------------------------------- FGMRES
int gnpc_fgmres(gnpc_csr a, gnpc_model m, const double* b, const double* x0,
                const gnpc_solve_config* cfg, double* x, gnpc_history* hist, int* status) {
  return fgmres_host(a, m, nullptr, b, x0, cfg, x, hist, status);
}

int gnpc_fgmres_host_operator(gnpc_csr a, gnpc_host_operator op, void* ctx, const double* b,
                              const double* x0, const gnpc_solve_config* cfg, double* x,
                              gnpc_history* hist, int* status) {
  if (!op) {
    set_error("fgmres_host_operator: null operator");
    return GNPC_EINVAL;
  }
  HostOp h{op, ctx};
  return fgmres_host(a, nullptr, &h, b, x0, cfg, x, hist, status);
}

int gnpc_fgmres_device(gnpc_csr a, gnpc_model m, const double* b_dev, double* x_dev,
                       const gnpc_solve_config* cfg, gnpc_history* hist, int* status,
                       void* stream) {
  return guarded([&] {
    need(a && b_dev && x_dev && cfg && status, "fgmres_device: null argument");
    require_device();
    if (m) need(m->a->h.n == a->h.n, "fgmres: preconditioner dimension mismatch");
    *status = fgmres_core(*a, m, nullptr, b_dev, x_dev, *cfg, hist, (cudaStream_t)stream);
  });
}


int gnpc_sampler_create(gnpc_csr a, int64_t m, uint64_t seed, gnpc_sampler* out) {
  return guarded([&] {
    need(a && out, "sampler_create: null argument");
    *out = build_sampler(*a, m, seed).release();
  });
}

int gnpc_sampler_from_arnoldi(int64_t n, int64_t k, const double* v, const double* hbar,
                              gnpc_sampler* out) {
  return guarded([&] {
    need(v && hbar && out, "sampler_from_arnoldi: null argument");
    if (n < 2) throw std::invalid_argument("spectral sampler: n must be >= 2");
    if (k < 1) throw std::invalid_argument("spectral sampler: m must be >= 1");
    auto s = std::make_unique<gnpc_sampler_s>();
    s->s = gnp_b200::spectral_from_arnoldi(n, k, std::vector<double>(v, v + n * k),
                                           std::vector<double>(hbar, hbar + (k + 1) * k));
    *out = s.release();
  });
}

int gnpc_sampler_destroy(gnpc_sampler s) {
  delete s;
  return GNPC_OK;
}

int gnpc_sampler_info(gnpc_sampler s, int64_t* k, int64_t* m_eff) {
  return guarded([&] {
    need(s != nullptr, "sampler_info: null sampler");
    if (k) *k = s->s.m;
    if (m_eff) *m_eff = s->s.m_eff;
  });
}

int gnpc_sampler_export(gnpc_sampler s, double* v, double* zsv, double* sv) {
  return guarded([&] {
    need(s != nullptr, "sampler_export: null sampler");
    if (v) std::copy(s->s.v.begin(), s->s.v.end(), v);
    if (zsv) std::copy(s->s.zm_sv.begin(), s->s.zm_sv.end(), zsv);
    if (sv) std::copy(s->s.s.begin(), s->s.s.end(), sv);
  });
}

int gnpc_assemble_batch(gnpc_sampler s, gnpc_csr a, uint64_t seed, int64_t skip_batches,
                        int64_t batch, int64_t spectral_count, double* x, double* b) {
  return guarded([&] {
    need(a && x && b, "assemble_batch: null argument");
    need(skip_batches >= 0, "assemble_batch: skip_batches must be >= 0");
    if (spectral_count < 0) throw std::invalid_argument("assemble_batch: spectral_count < 0");
    gnp_b200::Rng rng(seed);
    const gnp_b200::SpectralSampler* sp = s ? &s->s : nullptr;
    for (int64_t q = 0; q < skip_batches; ++q)
      gnp_b200::assemble_batch(sp, a->h, batch, spectral_count, rng, x, b);
    gnp_b200::assemble_batch(sp, a->h, batch, spectral_count, rng, x, b);
  });
}

}  // extern "C"
