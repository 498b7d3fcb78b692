// Debug probe: one 128-row tile, M=64 MN-major tf32 MMA (hi only), dump all
// 128 TMEM lanes x 32 columns.  Mode 1: MN-major A and B (wgrad); mode 0:
// K-major A/B layouts of the same data (forward-style) for comparison.
#include <cstdio>
#include <vector>

#include "kernels/tc.cuh"
#include "kernels/common.cuh"

using namespace gnpk;

__global__ void probe(const float* A, const float* B, float* dump, int mode, int M, uint32_t lbo, uint32_t sbo) {
  extern __shared__ float4 smem_raw[];
  const uint32_t pad = (1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* base = reinterpret_cast<uint8_t*>(smem_raw) + pad;
  uint8_t* As = base;                // 2 atoms
  uint8_t* Bs = base + 2 * 16384;    // 1 atom
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + 3 * 16384);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // A: 128 rows x 64 features (row-major in global), B: 128 rows x 32
  for (int c = tid; c < 128 * 16; c += 256) {
    const int r = c / 16, ch = c % 16;
    float4 x = *reinterpret_cast<const float4*>(A + r * 64 + 4 * ch);
    const uint32_t off = mode == 2 ? ch * sbo + (r / 8) * lbo + (r % 8) * 16 : tc::sw128_off(r, 4 * ch, 128);
    *reinterpret_cast<float4*>(As + off) = x;
  }
  for (int c = tid; c < 128 * 8; c += 256) {
    const int r = c / 8, ch = c % 8;
    float4 x = *reinterpret_cast<const float4*>(B + r * 32 + 4 * ch);
    const uint32_t off = mode == 2 ? ch * sbo + (r / 8) * (lbo / 2) + (r % 8) * 16 : tc::sw128_off(r, 4 * ch, 128);
    *reinterpret_cast<float4*>(Bs + off) = x;
  }
  if (tid == 0) tc::mbar_init(bar, 1);
  if (warp == 0) tc::tmem_alloc(tslot, 32);
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;
  if (tid == 0) {
    const uint32_t idesc = mode >= 1 ? tc::idesc_tf32_mn(M, 32) : tc::idesc_tf32(M, 32);
    for (int s = 0; s < 16; ++s) {
      uint64_t ad, bd;
      if (mode == 2) {
        ad = tc::make_desc(tc::smem_u32(As) + s * lbo, lbo, sbo);
        bd = tc::make_desc(tc::smem_u32(Bs) + s * (lbo / 2), lbo / 2, sbo);
      } else if (mode == 1) {
        ad = tc::make_desc_sw128_mn(tc::smem_u32(As) + s * 1024, lbo, sbo);
        bd = tc::make_desc_sw128_mn(tc::smem_u32(Bs) + s * 1024, lbo, sbo);
      } else {
        ad = tc::make_desc_sw128(tc::smem_u32(As) + (s >> 2) * 16384 + (s & 3) * 32, 1024);
        bd = tc::make_desc_sw128(tc::smem_u32(Bs) + (s >> 2) * 16384 + (s & 3) * 32, 1024);
      }
      tc::mma_tf32(tmem, ad, bd, idesc, s > 0);
      if (mode == 0 && s == 1) break;  // K-major: only 64 K values exist in the A tile rows
    }
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
  std::vector<float> A(128 * 64), B(128 * 32);
  for (int r = 0; r < 128; ++r) {
    for (int f = 0; f < 64; ++f) A[r * 64 + f] = (f == r % 64) ? 1.0f : 0.0f;
    for (int f = 0; f < 32; ++f) B[r * 32 + f] = (float)(r * 100 + f);
  }
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, 128 * 32 * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const size_t smem = 3 * 16384 + 64 + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  // mode 2: lbo = K-group stride (16 M-cores x 128 B = 2048 for A), sbo = M-core stride
  const uint32_t var[][2] = {{2048, 128}, {128, 2048}};
  for (int vi = 0; vi < 2; ++vi)
    for (int M : {64}) {
      const int mode = 2;
      cudaMemset(dD, 0, 128 * 32 * 4);
      probe<<<1, 256, smem>>>(dA, dB, dD, mode, M, var[vi][0], var[vi][1]);
      printf("mode %d M=%d lbo=%u sbo=%u: %s\n", mode, M, var[vi][0], var[vi][1], cudaGetErrorString(cudaDeviceSynchronize()));
      std::vector<float> D(128 * 32);
      cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
      int nz = 0;
      for (int l = 0; l < 128; ++l) {
        bool any = false;
        for (int c = 0; c < 32; ++c) any |= D[l * 32 + c] != 0.f;
        if (any && nz++ < 6)
          printf("  lane %3d: %g %g %g ... %g\n", l, D[l * 32], D[l * 32 + 1], D[l * 32 + 2], D[l * 32 + 31]);
      }
      printf("  nonzero lanes: %d\n", nz);
    }
  return 0;
}
