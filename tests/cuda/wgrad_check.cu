// Standalone check of k_wgrad_tc against a CPU f64 reference (debug harness,
// built and run on the GPU box: nvcc ... tests/cuda/wgrad_check.cu).
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "kernels/wgrad_tc.cuh"

int main(int argc, char** argv) {
  const int nv = argc > 1 ? atoi(argv[1]) : 1000;
  const int wa = argc > 2 ? atoi(argv[2]) : 32;
  const int wb = argc > 3 ? atoi(argv[3]) : 32;
  const int ones = argc > 4 ? atoi(argv[4]) : 0;
  std::vector<float> A1((size_t)nv * wa), A2((size_t)nv * wa), Bm((size_t)nv * wb);
  srand(1);
  for (auto& x : A1) x = (rand() / (float)RAND_MAX) - 0.5f;
  for (auto& x : A2) x = (rand() / (float)RAND_MAX) - 0.5f;
  for (auto& x : Bm) x = (rand() / (float)RAND_MAX) - 0.5f;
  float *dA1, *dA2, *dB;
  double* dP;
  cudaMalloc(&dA1, A1.size() * 4);
  cudaMalloc(&dA2, A2.size() * 4);
  cudaMalloc(&dB, Bm.size() * 4);
  const int grid = 4;
  cudaMalloc(&dP, (size_t)grid * 64 * 32 * 8);
  cudaMemcpy(dA1, A1.data(), A1.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dA2, A2.data(), A2.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, Bm.data(), Bm.size() * 4, cudaMemcpyHostToDevice);
  gnpk::WgradArgs g{dA1, wa, wa, ones ? nullptr : dA2, wa, wa, ones, dB, wb, wb, nv, dP};
  cudaFuncSetAttribute(gnpk::k_wgrad_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)gnpk::wg::smem_bytes());
  gnpk::k_wgrad_tc<<<grid, gnpk::kThreads, gnpk::wg::smem_bytes()>>>(g);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<double> P((size_t)grid * 64 * 32);
  cudaMemcpy(P.data(), dP, P.size() * 8, cudaMemcpyDeviceToHost);
  double maxerr = 0, maxref = 0;
  int shown = 0;
  for (int m = 0; m < 64; ++m)
    for (int n = 0; n < 32; ++n) {
      double ref = 0;
      for (int v = 0; v < nv; ++v) {
        double a = 0;
        if (m < 32) a = m < wa ? A1[(size_t)v * wa + m] : 0;
        else a = ones ? (m == 32 ? 1.0 : 0.0) : (m - 32 < wa ? A2[(size_t)v * wa + m - 32] : 0);
        const double b = n < wb ? Bm[(size_t)v * wb + n] : 0;
        ref += a * b;
      }
      double got = 0;
      for (int q = 0; q < grid; ++q) got += P[(size_t)q * 2048 + m * 32 + n];
      maxerr = std::fmax(maxerr, std::fabs(got - ref));
      maxref = std::fmax(maxref, std::fabs(ref));
      if (std::fabs(got - ref) > 1e-3 * (1 + std::fabs(ref)) && shown++ < 8)
        printf("m=%d n=%d got=%g ref=%g\n", m, n, got, ref);
    }
  printf("nv=%d wa=%d wb=%d ones=%d maxerr=%.3e maxref=%.3e rel=%.3e\n", nv, wa, wb, ones, maxerr,
         maxref, maxerr / maxref);
  return 0;
}
