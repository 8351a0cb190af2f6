// phase profile of the v5 elimination (clock64 per phase, lane 0 of every warp)
#define MCS_V5_PROF 1
#include "../paper_2207_08481_b200/csrc/condense.cu"
#include <cstdio>
#include <vector>
template <int W, int MB>
void run(double* dA, double* dB, double* dS, int* info, long cnt) {
  using G = MicroGeo5<60, 36, W>;
  auto kern = spd_schur_v5<60, 36, W, MB>;
  const size_t smem = G::SMEM * 8;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 32 * W, smem);
  kern<<<per * 148, 32 * W, smem>>>(dA, dB, dS, info, cnt);
  unsigned long long z[16] = {0};
  cudaMemcpyToSymbol(v5::g_v5prof, z, sizeof z);
  kern<<<per * 148, 32 * W, smem>>>(dA, dB, dS, info, cnt);
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(z, v5::g_v5prof, sizeof z);
  const char* nm[9] = {"issue-load", "wait-load", "prologue", "owner-chains", "chol8", "nonowner-tiles", "trailing", "barrier", "end"};
  double tot = 0; for (int i = 0; i < 9; ++i) tot += z[i];
  printf("W=%d ctas/sm=%d per element, summed over warps (clk):", W, per);
  for (int i = 0; i < 9; ++i) printf("  %s %.0f", nm[i], (double)z[i] / cnt);
  printf("  | per-warp total %.0f\n", tot / cnt / W);
}
int main() {
  long cnt = 148 * 5 * 40;
  double *dA, *dB, *dS; int* info;
  cudaMalloc(&dA, cnt * 1830 * 8); cudaMalloc(&dB, cnt * 2160 * 8); cudaMalloc(&dS, cnt * 666 * 8);
  cudaMalloc(&info, cnt * 4);
  std::vector<double> A(1830), B(2160);
  for (int i = 0; i < 60; ++i) for (int j = 0; j <= i; ++j) A[i * (i + 1) / 2 + j] = (i == j ? 70.0 : 0.0) + 1.0 / (1 + i + j);
  for (int q = 0; q < 2160; ++q) B[q] = 0.01 * (q % 17);
  cudaMemcpy(dA, A.data(), 1830 * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), 2160 * 8, cudaMemcpyHostToDevice);
  for (long e = 1; e < cnt; e *= 2) {
    cudaMemcpy(dA + e * 1830, dA, std::min(e, cnt - e) * 1830 * 8, cudaMemcpyDeviceToDevice);
    cudaMemcpy(dB + e * 2160, dB, std::min(e, cnt - e) * 2160 * 8, cudaMemcpyDeviceToDevice);
  }
  run<4, 5>(dA, dB, dS, info, cnt);
  run<2, 8>(dA, dB, dS, info, cnt);
  return 0;
}
