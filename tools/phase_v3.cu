#define MCS_PHASE_PROF
#include "../paper_2207_08481_b200/csrc/condense.cu"
#include <cstdio>
#include <vector>
int main() {
  const int n = 60, m = 36; const long cnt = 1 << 15;
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
  launch_spd_schur_v3<60, 36, 2, 4>(dA, dB, dS, info, cnt, 0);
  unsigned long long z[64] = {0};
  cudaMemcpyToSymbol(mcs::v3::g_v3prof, z, sizeof(z));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  launch_spd_schur_v3<60, 36, 2, 4>(dA, dB, dS, info, cnt, 0);
  cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
  cudaMemcpyFromSymbol(z, mcs::v3::g_v3prof, sizeof(z));
  long per_cta = cnt / (148 * 4);
  printf("ms %.3f, elements per CTA %ld, clk per element per CTA %.0f\n", ms, per_cta, ms * 1e-3 * 1.965e9 / per_cta);
  const char* nm[7] = {"load", "prolog", "C1", "diaginv", "C2", "panelZ", "barrier"};
  for (int w = 0; w < 2; ++w) { printf("warp %d:", w); for (int q = 0; q < 7; ++q) printf("  %s %6.0f", nm[q], (double)z[8 * w + q] / per_cta); printf("\n"); }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
