// Per-phase clocks of the config-5 kernel (micro.cu built with MCS_MICRO_PROF):
//   nvcc ... -DMCS_MICRO_PROF tools/micro_prof.cu paper_2207_08481_b200/csrc/micro.cu
#include <cstdio>
#include <vector>
#include <random>
#include "../paper_2207_08481_b200/csrc/common.cuh"
namespace mcs {
template <int NS, int NC>
int launch_spd_schur_w2(const double*, const double*, double*, int*, int64_t, cudaStream_t);
namespace micro { extern __device__ unsigned long long g_prof[2][8]; }
}
int main() {
  const int n = 60, m = 36, la = n * (n + 1) / 2;
  const long long cnt = 148 * 6 * 40;
  std::vector<double> A(cnt * la), B(cnt * n * m);
  std::mt19937_64 r(1);
  std::normal_distribution<double> N;
  for (long long e = 0; e < cnt; ++e) {
    for (int i = 0; i < n; ++i)
      for (int j = 0; j <= i; ++j) A[e * la + i * (i + 1) / 2 + j] = (i == j ? 2.0 * n : 0.01 * N(r));
    for (int i = 0; i < n * m; ++i) B[e * n * m + i] = N(r);
  }
  double *dA, *dB, *dS; int* info;
  cudaMalloc(&dA, A.size() * 8); cudaMalloc(&dB, B.size() * 8);
  cudaMalloc(&dS, cnt * 666 * 8); cudaMalloc(&info, cnt * 4);
  cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 8, cudaMemcpyHostToDevice);
  mcs::launch_spd_schur_w2<60, 36>(dA, dB, dS, info, cnt, 0);
  unsigned long long z[16] = {0};
  cudaMemcpyToSymbol(mcs::micro::g_prof, z, sizeof(z));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mcs::launch_spd_schur_w2<60, 36>(dA, dB, dS, info, cnt, 0);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[16];
  cudaMemcpyFromSymbol(h, mcs::micro::g_prof, sizeof(h));
  const char* nm[6] = {"B loads", "mbar wait", "unpack", "phase 1", "phase 2", "tail"};
  printf("%lld elements, %.3f ms, %.1f clk/element/SM (6 in flight)\n", cnt, ms,
         ms * 1.965e6 * 148 / cnt);
  for (int w = 0; w < 2; ++w) {
    printf("warp %d:", w);
    for (int i = 0; i < 6; ++i) printf("  %s %.0f", nm[i], (double)h[w * 8 + i] / cnt);
    printf("  [6] %.0f [7] %.0f", (double)h[w * 8 + 6] / cnt, (double)h[w * 8 + 7] / cnt);
    printf("\n");
  }
}
