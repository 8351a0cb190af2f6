// timing of elimination-kernel variants (warps per CTA, min CTAs per SM)
#include "../paper_2207_08481_b200/csrc/condense.cu"
#include <cstdio>
#include <vector>
template <int W, int MB>
void run_micro(double* dA, double* dB, double* dS, int* info, long cnt) {
  for (int rep = 0; rep < 2; ++rep) launch_spd_schur<60, 36, W, MB>(dA, dB, dS, info, cnt, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  launch_spd_schur<60, 36, W, MB>(dA, dB, dS, info, cnt, 0);
  cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
  int per = 0; cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, spd_schur_kernel<60, 36, W, MB>);
  using P = Pad<60, 36, W>;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, spd_schur_kernel<60, 36, W, MB>, 32 * W, (1830 + 2160 + P::E::SMEM_WORK) * 8);
  double tf = 279360.0 * cnt / (ms * 1e-3) / 1e12;
  printf("micro W=%2d minB=%d regs=%3d ctas/sm=%d : %.3f ms  %.2f TF/s  (%s)\n", W, MB, fa.numRegs, per, ms, tf, cudaGetErrorString(cudaGetLastError()));
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
  run_micro<8, 1>(dA, dB, dS, info, cnt);
  run_micro<8, 2>(dA, dB, dS, info, cnt);
  run_micro<16, 1>(dA, dB, dS, info, cnt);
  run_micro<4, 1>(dA, dB, dS, info, cnt);
  run_micro<4, 3>(dA, dB, dS, info, cnt);
  run_micro<2, 2>(dA, dB, dS, info, cnt);
  run_micro<2, 3>(dA, dB, dS, info, cnt);
  return 0;
}
