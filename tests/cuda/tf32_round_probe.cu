// Probe: how does tcgen05.mma.kind::tf32 treat the low 13 mantissa bits of
// an fp32 operand (truncate / round-nearest-even / round-away)?  One M=128,
// N=16, K=8 MMA; A row m holds value a_m in column 0 (zeros elsewhere), B is
// 1.0 in column 0 of every row, so D[m][n] = tf32(a_m).
#include <cstdio>
#include <cstring>
#include <vector>

#include "kernels/tc.cuh"

using namespace gnpk;

__global__ void probe(const float* A, const float* B, float* out) {
  extern __shared__ float4 smem_raw[];
  const uint32_t pad = (1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* base = reinterpret_cast<uint8_t*>(smem_raw) + pad;
  uint8_t* As = base;          // 128 rows x 32 fp32 (one SW128 atom column)
  uint8_t* Bs = base + 16384;  // 16 rows x 32 fp32
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + 16384 + 2048);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 128 * 32; i += blockDim.x) {
    const int r = i / 32, k = i % 32;
    *reinterpret_cast<float*>(As + tc::sw128_off(r, k, 128)) = A[i];
  }
  for (int i = tid; i < 16 * 32; i += blockDim.x) {
    const int r = i / 32, k = i % 32;
    *reinterpret_cast<float*>(Bs + tc::sw128_off(r, k, 16)) = B[i];
  }
  if (tid == 0) tc::mbar_init(bar, 1);
  if (warp == 0) tc::tmem_alloc(tslot, 32);
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;
  if (tid == 0) {
    tc::mma_tf32(tmem, tc::make_desc_sw128(tc::smem_u32(As), 1024), tc::make_desc_sw128(tc::smem_u32(Bs), 1024),
                 tc::idesc_tf32(128, 16), 0);
    tc::mma_commit(bar);
  }
  tc::mbar_wait(bar, 0);
  tc::fence_after();
  if (warp < 4) {
    float v[8];
    tc::tmem_ld8(tmem + (static_cast<uint32_t>(32 * warp) << 16), v);
    out[32 * warp + lane] = v[0];
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 0) tc::tmem_dealloc(tmem, 32);
}

static float bits(uint32_t u) { float f; std::memcpy(&f, &u, 4); return f; }
static uint32_t ubits(float f) { uint32_t u; std::memcpy(&u, &f, 4); return u; }

int main() {
  std::vector<float> A(128 * 32, 0.f), B(16 * 32, 0.f);
  // mantissa tails below tf32 precision: 0x3f800000 + t for t in a table
  const uint32_t tails[] = {0x0000, 0x0800, 0x1000, 0x1001, 0x1fff, 0x2000, 0x3000, 0x2fff, 0x1800};
  const int nt = sizeof(tails) / sizeof(tails[0]);
  for (int m = 0; m < nt; ++m) A[m * 32] = bits(0x3f800000u + tails[m]);
  for (int m = 0; m < nt; ++m) A[(64 + m) * 32] = -bits(0x3f800000u + tails[m]);
  for (int r = 0; r < 16; ++r) B[r * 32] = 1.f;
  float *dA, *dB, *dO;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dO, 128 * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const size_t smem = 16384 + 2048 + 64 + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  probe<<<1, 128, smem>>>(dA, dB, dO);
  printf("sync: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  std::vector<float> O(128);
  cudaMemcpy(O.data(), dO, 128 * 4, cudaMemcpyDeviceToHost);
  for (int m = 0; m < nt; ++m)
    printf("tail 0x%04x: in %08x -> %08x | neg -> %08x\n", tails[m], 0x3f800000u + tails[m], ubits(O[m]),
           ubits(O[64 + m]));
  return 0;
}
