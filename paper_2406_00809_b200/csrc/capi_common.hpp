// Internal C++ side of the C ABI: error plumbing, device buffers, handle
// structs.  Not part of the public boundary (include/gnpc.h is).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <tuple>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/gnpc.h"
#include "host/gnp_host.hpp"
#include "kernels/common.cuh"

namespace gnpc_impl {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct Unsupported : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NoDevice : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void set_error(const std::string& msg);

// [rows][width] fp32 rows as a 2-D TMA tensor, box {width, box_rows}.
CUtensorMap make_rows_map(const float* base, std::int64_t rows, int width, int box_rows,
                          CUtensorMapSwizzle swizzle);
extern std::atomic<std::int64_t> g_launches;

#define GNPC_CUDA(expr)                                                                  \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess)                                                               \
      throw ::gnpc_impl::CudaError(std::string(#expr) + ": " + cudaGetErrorString(_e));  \
  } while (0)

#define GNPC_LAUNCHED()                                           \
  do {                                                            \
    ::gnpc_impl::g_launches.fetch_add(1, std::memory_order_relaxed); \
    GNPC_CUDA(cudaGetLastError());                                \
  } while (0)

// Runs f and maps any exception onto a gnpc_status (nothing escapes the ABI).
template <class F>
int guarded(F&& f) {
  try {
    f();
    return GNPC_OK;
  } catch (const NoDevice& e) {
    set_error(e.what());
    return GNPC_ENODEV;
  } catch (const Unsupported& e) {
    set_error(e.what());
    return GNPC_EUNSUPPORTED;
  } catch (const CudaError& e) {
    set_error(e.what());
    cudaGetLastError();  // do not leave a stale error for the next launch check
    return GNPC_ECUDA;
  } catch (const std::bad_alloc&) {
    set_error("device or host allocation failed");
    return GNPC_ENOMEM;
  } catch (const std::out_of_range& e) {
    set_error(e.what());
    return GNPC_ERANGE;
  } catch (const std::invalid_argument& e) {
    set_error(e.what());
    return GNPC_EINVAL;
  } catch (const std::exception& e) {
    set_error(e.what());
    return GNPC_ERUNTIME;
  } catch (...) {
    set_error("unknown error");
    return GNPC_ERUNTIME;
  }
}

void require_device();
int num_sms();
int tc_ctas_per_sm(const void* kern, size_t smem, int tcols);

// Raise a kernel's dynamic shared-memory limit on the CURRENT device, once
// per (device, kernel, size): the attribute is per device, so a process that
// drives several devices sets it on each.
inline void set_smem_attr(const void* kern, int bytes) {
  static std::mutex mu;
  static std::vector<std::tuple<int, const void*, int>> done;
  int dev = 0;
  GNPC_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  for (const auto& [d, k, b] : done)
    if (d == dev && k == kern && b >= bytes) return;
  GNPC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done.emplace_back(dev, kern, bytes);
}

template <typename T>
struct DevBuf {
  T* p = nullptr;
  std::size_t count = 0;
  DevBuf() = default;
  explicit DevBuf(std::size_t n) { alloc(n); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), count(o.count) { o.p = nullptr; o.count = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p; count = o.count;
      o.p = nullptr; o.count = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(std::size_t n) {
    release();
    if (n == 0) n = 1;
    cudaError_t e = cudaMalloc(&p, n * sizeof(T));
    if (e != cudaSuccess) {
      p = nullptr;
      cudaGetLastError();
      throw std::bad_alloc();
    }
    count = n;
  }
  void ensure(std::size_t n) {
    if (count < n || p == nullptr) alloc(n);
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    count = 0;
  }
  void upload(const T* h, std::size_t n, cudaStream_t s = nullptr) {
    ensure(n);
    GNPC_CUDA(cudaMemcpyAsync(p, h, n * sizeof(T), cudaMemcpyHostToDevice, s));
  }
};

// Krylov workspace, cached per (n, restart) on the matrix handle.
struct KrylovWs {
  int n = 0, m = 0;
  DevBuf<double> V, Z, w, vin, zout, x, b, r, H, R, cs, sn, g, y, partials, hist_rel;
  DevBuf<long long> hist_t;
  DevBuf<unsigned> ticket;
  DevBuf<gnpk::KState> st;
};

}  // namespace gnpc_impl

struct gnpc_csr_s {
  gnp_b200::CsrHost h;
  // device copy (lazy): int32 row_ptr / col_idx, fp32 values, long-row list
  bool dev_ready = false;
  gnpc_impl::DevBuf<int> rp, ci, long_rows;
  gnpc_impl::DevBuf<float> v;
  int n_long = 0;
  int max_row = 0;
  // long-row chunk plan (kChunk nonzeros per warp)
  gnpc_impl::DevBuf<int> ch_row, ch_k0, ch_k1, long_c0;
  int n_chunks = 0;
  // sliced-ELL copy for the tensor-core layer (see DevCsr)
  gnpc_impl::DevBuf<int2> sell;
  gnpc_impl::DevBuf<int> sell_off, sell_k;
  bool has_sell = false;
  // length-sorted renumbering of the apply path (ragged matrices; see upload())
  gnpc_impl::DevBuf<int> perm, prm_rp, prm_ci;
  gnpc_impl::DevBuf<float> prm_v;
  bool has_perm = false;
  // padded short-row CSR + per-tile long flags for the TMA CSR layer (see DevCsr)
  gnpc_impl::DevBuf<int> rps, cis, tflag;
  gnpc_impl::DevBuf<float> vs;
  // pair-union sliced-ELL (see DevCsr::psell)
  gnpc_impl::DevBuf<int4> psell;
  gnpc_impl::DevBuf<int> psell_off, psell_k;
  bool has_pairs = false;
  // strip-window pair-union layout (see DevCsr::pw)
  gnpc_impl::DevBuf<uint8_t> pw;
  gnpc_impl::DevBuf<int> pw_off, pw_k, pw_order;
  int pw_S = 0;
  bool has_pw = false;
  // training strip windows (see DevCsr::tw), one layout per batch size (a
  // training run's trainer and its monitor trainer may differ)
  struct TwLayout {
    gnpc_impl::DevBuf<uint8_t> sl;
    gnpc_impl::DevBuf<int> off, k, order;
    int S = 0;
    bool ok = false;
  };
  std::map<int, std::unique_ptr<TwLayout>> tws;
  bool has_tw = false;  // any batch size (introspection)
  bool ensure_tw(int bs);
  // the layout for batch size bs into d (null fields when not built)
  void bind_tw(int bs, gnpk::DevCsr& d) const;
  bool l2hint = true;
  std::unique_ptr<gnpc_csr_s> tr;  // Âᵀ (lazy, for training backward)
  std::unique_ptr<gnpc_impl::KrylovWs> kws;
  void upload();
  void build_sell(const std::vector<int>& hrp, const std::vector<int>& hci,
                  const std::vector<float>& hv);
  void build_pairs(const std::vector<int>& hrp, const std::vector<int>& hci, const std::vector<float>& hv);
  void build_pw(const std::vector<int>& hrp, const std::vector<int>& hci, const std::vector<float>& hv);
  int dominant_tile_stride(const std::vector<int>& hrp, const std::vector<int>& hci, int TM) const;
  gnpk::DevCsr dev();
  gnpk::DevCsr dev_apply();
};

// build_spectral_sampler (src/sampler.cpp:10-39): Arnoldi on the device,
// Jacobi SVD of the small Hessenberg on the host.
struct gnpc_sampler_s {
  gnp_b200::SpectralSampler s;
};
namespace gnpc_impl {
std::unique_ptr<gnpc_sampler_s> build_sampler(gnpc_csr_s& a, std::int64_t m, std::uint64_t seed);
}
