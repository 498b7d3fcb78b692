// Probe: tcgen05.mma.kind::tf32 with A in tensor memory.  Is row m in lane m
// and K element k in column a_tmem + k (one 32-bit column per element), and
// does it truncate A like the shared-memory form?  D = A·B^T, M=128, N=32,
// K=32 as four K=8 steps at a_tmem + 8*k8; compared with a CPU product of the
// truncated operands.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "kernels/tc.cuh"

using namespace gnpk;

__global__ void probe(const float* A, const float* B, float* out) {
  extern __shared__ float4 smem_raw[];
  const uint32_t pad = (1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* base = reinterpret_cast<uint8_t*>(smem_raw) + pad;
  uint8_t* Bs = base;  // 32 rows (n) x 32 fp32 (k), SW128 K-major
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + 4096);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 32 * 32; i += blockDim.x) {
    const int r = i / 32, k = i % 32;
    *reinterpret_cast<float*>(Bs + tc::sw128_off(r, k, 32)) = B[i];
  }
  if (tid == 0) tc::mbar_init(bar, 1);
  if (warp == 0) tc::tmem_alloc(tslot, 128);
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t tA = tmem + 64;
  if (warp < 4) {
    const int m = 32 * warp + lane;
    for (int c0 = 0; c0 < 32; c0 += 8) {
      float v[8];
      for (int c = 0; c < 8; ++c) v[c] = A[m * 32 + c0 + c];
      tc::tmem_st8(tA + (static_cast<uint32_t>(32 * warp) << 16) + c0, v);
    }
    tc::tmem_wait_st();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (tid == 0) {
    for (int k8 = 0; k8 < 4; ++k8)
      tc::mma_tf32_ts(tmem, tA + 8 * k8, tc::make_desc_sw128(tc::smem_u32(Bs) + 32 * k8, 1024),
                      tc::idesc_tf32(128, 32), k8 > 0);
    tc::mma_commit(bar);
  }
  tc::mbar_wait(bar, 0);
  tc::fence_after();
  if (warp < 4) {
    const int m = 32 * warp + lane;
    for (int c0 = 0; c0 < 32; c0 += 8) {
      float v[8];
      tc::tmem_ld8(tmem + (static_cast<uint32_t>(32 * warp) << 16) + c0, v);
      for (int c = 0; c < 8; ++c) out[m * 32 + c0 + c] = v[c];
    }
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 0) tc::tmem_dealloc(tmem, 128);
}

static float trunc13(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u &= 0xffffe000u;
  std::memcpy(&f, &u, 4);
  return f;
}

int main() {
  std::vector<float> A(128 * 32), B(32 * 32);
  unsigned s = 12345;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return (s >> 8) * (1.0f / 16777216.f) * 2.f - 1.f; };
  for (auto& x : A) x = rnd();
  for (auto& x : B) x = rnd();
  float *dA, *dB, *dO;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dO, 128 * 32 * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const size_t smem = 4096 + 64 + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  probe<<<1, 128, smem>>>(dA, dB, dO);
  printf("sync: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  std::vector<float> O(128 * 32);
  cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
  double e_tr = 0, e_raw = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 32; ++n) {
      double rt = 0, rr = 0;
      for (int k = 0; k < 32; ++k) {
        rt += double(trunc13(A[m * 32 + k])) * trunc13(B[n * 32 + k]);
        rr += double(A[m * 32 + k]) * B[n * 32 + k];
      }
      e_tr = std::fmax(e_tr, std::fabs(O[m * 32 + n] - rt));
      e_raw = std::fmax(e_raw, std::fabs(O[m * 32 + n] - rr));
    }
  printf("max |D - trunc-product| = %.3e, max |D - fp32 product| = %.3e\n", e_tr, e_raw);
  printf("%s\n", e_tr < 1e-5 ? "TS_LAYOUT_OK" : "TS_LAYOUT_MISMATCH");
  return 0;
}
