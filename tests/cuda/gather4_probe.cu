// Probe: TMA tile::gather4 (cp.async.bulk.tensor.2d...tile::gather4) on a
// row-major [rows][16] fp32 tensor.  Which tensor-map box is accepted, how
// many bytes complete the transaction, and where the four rows land in
// shared memory.  Prints one line per box configuration.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "kernels/tc.cuh"

using namespace gnpk;

__global__ void probe(const __grid_constant__ CUtensorMap tm, int r0, int r1, int r2, int r3, uint32_t tx,
                      float* out, int nout) {
  __shared__ alignas(1024) float buf[1024];
  __shared__ uint64_t bar;
  const int tid = threadIdx.x;
  for (int i = tid; i < 1024; i += blockDim.x) buf[i] = -1.f;
  if (tid == 0) tc::mbar_init(&bar, 1);
  tc::fence_proxy_async();
  __syncthreads();
  if (tid == 0) {
    tc::mbar_expect_tx(&bar, tx);
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
        "%4, %5, %6}], [%7];" ::"r"(tc::smem_u32(buf)),
        "l"(&tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(tc::smem_u32(&bar))
        : "memory");
  }
  // bounded wait: report instead of hanging if the tx count is wrong
  bool ok = false;
  for (int k = 0; k < 2000000 && !ok; ++k) ok = tc::mbar_test(&bar, 0);
  __syncthreads();
  for (int i = tid; i < nout; i += blockDim.x) out[i] = ok ? buf[i] : -7.f;
}

int main() {
  const int rows = 1000, W = 16;
  std::vector<float> h(rows * W);
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < W; ++c) h[r * W + c] = r + c / 100.f;
  float *d, *o;
  cudaMalloc(&d, h.size() * 4);
  cudaMalloc(&o, 1024 * 4);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  cudaDriverEntryPointQueryResult q{};
  void* fp = nullptr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
  const int boxes[][2] = {{16, 1}, {16, 4}, {8, 1}};
  for (auto& bx : boxes) {
    CUtensorMap tm{};
    const cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)W * 4};
    const cuuint32_t box[2] = {(cuuint32_t)bx[0], (cuuint32_t)bx[1]};
    const cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      printf("box {%d,%d}: encode failed %d\n", bx[0], bx[1], (int)r);
      continue;
    }
    const uint32_t tx = 4u * bx[0] * 4u;  // four rows of box width
    probe<<<1, 128>>>(tm, 7, 500, 3, 999, tx, o, 64);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> ho(64);
    cudaMemcpy(ho.data(), o, 64 * 4, cudaMemcpyDeviceToHost);
    printf("box {%d,%d} tx %u: %s |", bx[0], bx[1], tx, cudaGetErrorString(e));
    for (int i = 0; i < 64; i += 4) printf(" %.2f", ho[i]);
    printf("\n");
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
