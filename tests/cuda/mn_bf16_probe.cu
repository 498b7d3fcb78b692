// Probe: tcgen05.mma.kind::f16 (bf16 in, f32 accumulate) with BOTH operands
// MN-major in shared memory (A: [K][M=64] rows of 128 B, SWIZZLE_128B;
// B: [K][N=32] rows of 64 B, SWIZZLE_64B), M=64 N=32 K=16.  Checks that the
// weight-gradient form D[m][n] = sum_k A[k][m] B[k][n] works without a
// transpose.  Prints the nonzero TMEM lanes and a max error.
#include <cstdio>
#include <cstring>
#include <vector>
#include <cuda_bf16.h>

#include "kernels/tc.cuh"

using namespace gnpk;

__device__ __forceinline__ uint64_t desc_mn(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;
  d |= (uint64_t)layout << 61;
  return d;
}

__global__ void probe(const __nv_bfloat16* A, const __nv_bfloat16* B, float* dump, uint32_t lboA, uint32_t sboA,
                      uint32_t lboB, uint32_t sboB) {
  extern __shared__ float4 smem_raw[];
  const uint32_t pad = (1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* base = reinterpret_cast<uint8_t*>(smem_raw) + pad;
  uint8_t* As = base;          // 16 rows x 128 B
  uint8_t* Bs = base + 4096;   // 16 rows x 64 B
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + 8192);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 16 * 64; i += blockDim.x) {  // A[k][m]
    const int k = i / 64, m = i % 64;
    const uint32_t off = (k >> 3) * 1024 + (k & 7) * 128 + ((((m >> 3) ^ (k & 7))) << 4) + (m & 7) * 2;
    *reinterpret_cast<__nv_bfloat16*>(As + off) = A[i];
  }
  for (int i = tid; i < 16 * 32; i += blockDim.x) {  // B[k][n]
    const int k = i / 32, n = i % 32;
    const uint32_t off = (k >> 3) * 512 + (k & 7) * 64 + ((((n >> 3) ^ ((k & 7) >> 1)) & 3) << 4) + (n & 7) * 2;
    *reinterpret_cast<__nv_bfloat16*>(Bs + off) = B[i];
  }
  if (tid == 0) tc::mbar_init(bar, 1);
  if (warp == 0) tc::tmem_alloc(tslot, 32);
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;
  if (tid == 0) {
    // kind::f16: c F32 (bit 4), a BF16 (bits 7-9 = 1), b BF16 (bits 10-12 = 1),
    // a MN-major (bit 15), b MN-major (bit 16), N>>3 @17, M>>4 @24
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) | ((32u >> 3) << 17) |
                           ((64u >> 4) << 24);
    const uint64_t ad = desc_mn(tc::smem_u32(As), lboA, sboA, 2);
    const uint64_t bd = desc_mn(tc::smem_u32(Bs), lboB, sboB, 4);
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
        "l"(ad), "l"(bd), "r"(idesc), "r"(0));
    tc::mma_commit(bar);
  }
  tc::mbar_wait(bar, 0);
  tc::fence_after();
  if (warp < 4) {
    float v[16];
    tc::tmem_ld16(tmem + (static_cast<uint32_t>(32 * warp) << 16), v);
    for (int i = 0; i < 16; ++i) dump[(32 * warp + lane) * 32 + i] = v[i];
    tc::tmem_ld16(tmem + (static_cast<uint32_t>(32 * warp) << 16) + 16, v);
    for (int i = 0; i < 16; ++i) dump[(32 * warp + lane) * 32 + 16 + i] = v[i];
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 0) tc::tmem_dealloc(tmem, 32);
}

int main() {
  std::vector<__nv_bfloat16> A(16 * 64), B(16 * 32);
  std::vector<float> Af(16 * 64), Bf(16 * 32);
  for (int k = 0; k < 16; ++k) {
    for (int m = 0; m < 64; ++m) Af[k * 64 + m] = (float)((m * 7 + k * 3) % 11) - 5.f;
    for (int n = 0; n < 32; ++n) Bf[k * 32 + n] = (float)((n * 5 + k) % 9) - 4.f;
  }
  for (int i = 0; i < 16 * 64; ++i) A[i] = __float2bfloat16(Af[i]);
  for (int i = 0; i < 16 * 32; ++i) B[i] = __float2bfloat16(Bf[i]);
  __nv_bfloat16 *dA, *dB;
  float* dD;
  cudaMalloc(&dA, A.size() * 2);
  cudaMalloc(&dB, B.size() * 2);
  cudaMalloc(&dD, 128 * 32 * 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  const size_t smem = 8192 + 64 + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const uint32_t var[][4] = {{0, 1024, 0, 512}, {1024, 0, 512, 0}, {16, 1024, 16, 512}};
  for (auto& vv : var) {
    cudaMemset(dD, 0, 128 * 32 * 4);
    probe<<<1, 128, smem>>>(dA, dB, dD, vv[0], vv[1], vv[2], vv[3]);
    const cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> D(128 * 32);
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    // expected D[m][n] = sum_k A[k][m] B[k][n]; M=64 rows live in lanes 32(m/16) + m%16
    double maxerr = 0, maxref = 0;
    int nz = 0;
    for (int m = 0; m < 64; ++m)
      for (int n = 0; n < 32; ++n) {
        double ref = 0;
        for (int k = 0; k < 16; ++k) ref += (double)Af[k * 64 + m] * Bf[k * 32 + n];
        const int lane = 32 * (m / 16) + m % 16;
        const double got = D[lane * 32 + n];
        maxerr = std::max(maxerr, std::abs(got - ref));
        maxref = std::max(maxref, std::abs(ref));
        nz += got != 0.0;
      }
    printf("lboA %u sboA %u lboB %u sboB %u: %s  nonzero %d  maxerr %.3g (max |ref| %.3g)\n", vv[0], vv[1], vv[2],
           vv[3], cudaGetErrorString(e), nz, maxerr, maxref);
  }
  return 0;
}
