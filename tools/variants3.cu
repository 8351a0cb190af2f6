// timing + cross-check of the v5 elimination kernels against the v2 engine
#include "../paper_2207_08481_b200/csrc/condense.cu"
#include <cstdio>
#include <vector>
#include <cmath>
template <int W, int MB>
void run5(double* dA, double* dB, double* dS, int* info, long cnt, const std::vector<double>& ref) {
  using G = MicroGeo5<60, 36, W>;
  auto kern = spd_schur_v5<60, 36, W, MB>;
  const size_t smem = G::SMEM * 8;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 32 * W, smem);
  int grid = per * 148;
  cudaMemset(dS, 0, cnt * 666 * 8);
  for (int rep = 0; rep < 2; ++rep) kern<<<grid, 32 * W, smem>>>(dA, dB, dS, info, cnt);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<<<grid, 32 * W, smem>>>(dA, dB, dS, info, cnt);
  cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, kern);
  std::vector<double> S(cnt * 666); cudaMemcpy(S.data(), dS, S.size() * 8, cudaMemcpyDeviceToHost);
  std::vector<int> inf(cnt); cudaMemcpy(inf.data(), info, cnt * 4, cudaMemcpyDeviceToHost);
  long nbad = 0; for (long e = 0; e < cnt; ++e) nbad += inf[e] != 0;
  double err = 0; for (size_t q = 0; q < S.size(); ++q) err = fmax(err, fabs(S[q] - ref[q]) / (fabs(ref[q]) + 1e-3));
  double tf = 279360.0 * cnt / (ms * 1e-3) / 1e12;
  printf("v5 W=%d minB=%d regs=%3d local=%zu smem=%zu ctas/sm=%d : %.3f ms  %.2f TF/s  maxrel %.1e bad %ld (%s)\n", W, MB, fa.numRegs, fa.localSizeBytes, smem, per, ms, tf, err, nbad, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  const int n = 60, m = 36; const long cnt = 1 << 17;
  std::vector<double> A(cnt * 1830), B(cnt * 2160);
  unsigned s = 1;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return (s >> 8) / 16777216.0 - 0.5; };
  for (long e = 0; e < cnt; ++e) {
    for (int i = 0; i < n; ++i) for (int j = 0; j <= i; ++j) A[e * 1830 + i * (i + 1) / 2 + j] = (i == j ? 60.0 : 0.0) + 0.1 * rnd();
    for (int q = 0; q < n * m; ++q) B[e * 2160 + q] = rnd();
  }
  double *dA, *dB, *dS; int* info;
  cudaMalloc(&dA, A.size() * 8); cudaMalloc(&dB, B.size() * 8); cudaMalloc(&dS, cnt * 666 * 8); cudaMalloc(&info, cnt * 4);
  cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice); cudaMemcpy(dB, B.data(), B.size() * 8, cudaMemcpyHostToDevice);
  launch_spd_schur<60, 36, 8, 2>(dA, dB, dS, info, cnt, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventRecord(e0);
  launch_spd_schur<60, 36, 8, 2>(dA, dB, dS, info, cnt, 0);
  cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("v2 W=8 minB=2: %.3f ms %.2f TF/s\n", ms, 279360.0 * cnt / (ms * 1e-3) / 1e12);
  std::vector<double> ref(cnt * 666); cudaMemcpy(ref.data(), dS, ref.size() * 8, cudaMemcpyDeviceToHost);
  run5<2, 8>(dA, dB, dS, info, cnt, ref);
  run5<4, 4>(dA, dB, dS, info, cnt, ref);
  run5<4, 5>(dA, dB, dS, info, cnt, ref);
  run5<8, 2>(dA, dB, dS, info, cnt, ref);
  run5<4, 1>(dA, dB, dS, info, cnt, ref);
  return 0;
}
