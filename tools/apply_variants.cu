// timing of elem_apply / ext_restrict / ext_prolong (W warps, NST stages)
#include "../paper_2207_08481_b200/csrc/apply.cu"
#include <cstdio>
#include <vector>
template <int N, int STRIDE, int W, int NST>
float time_apply(const double* M, const int* codes, const double* x, double* y, long nt) {
  auto kern = elem_apply_kernel<N, STRIDE, W, NST>;
  size_t smem = (size_t)W * NST * STRIDE * 8;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, W * 32, smem);
  long want = (nt + W - 1) / W, g = (long)per * 148; int grid = (int)(want < g ? want : g);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    kern<<<grid, W * 32, smem>>>(M, codes, x, y, nt);
    cudaEventRecord(e0); kern<<<grid, W * 32, smem>>>(M, codes, x, y, nt); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  double bytes = (double)nt * STRIDE * 8;
  printf("apply N=%d W=%2d NST=%d ctas/sm=%d: %.1f us  %.0f GB/s\n", N, W, NST, per, best * 1e3, bytes / (best * 1e-3) / 1e9);
  return best;
}
template <int K, int W, int NST>
void time_restrict(const double* ext, const int* bidx, const int* cc, const double* r, double* bub, double* acc, long nt) {
  constexpr int LEN = ExtLen<K>::len;
  auto kern = ext_restrict_kernel<K, LEN, W, NST>;
  size_t smem = (size_t)W * NST * LEN * 8;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, W * 32, smem);
  long want = (nt + W - 1) / W, g = (long)per * 148; int grid = (int)(want < g ? want : g);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9;
  for (int q = 0; q < 5; ++q) {
    kern<<<grid, W * 32, smem>>>(ext, bidx, cc, r, bub, acc, nt);
    cudaEventRecord(e0); kern<<<grid, W * 32, smem>>>(ext, bidx, cc, r, bub, acc, nt); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  printf("restrict k=%d W=%2d NST=%d ctas/sm=%d: %.1f us  %.0f GB/s\n", K, W, NST, per, best * 1e3, (double)nt * LEN * 8 / (best * 1e-3) / 1e9);
}
int main() {
  const long nt4 = 32768, nt6 = 131072;
  double *M, *x, *y; int* codes;
  cudaMalloc(&M, nt6 * 2776 * 8); cudaMalloc(&x, 8000000 * 8); cudaMalloc(&y, 8000000 * 8); cudaMalloc(&codes, nt6 * 74 * 4);
  cudaMemset(M, 0, nt6 * 2776 * 8); cudaMemset(x, 0, 8000000 * 8);
  std::vector<int> hc(nt6 * 74);
  for (long e = 0; e < nt6; ++e) for (int j = 0; j < 74; ++j) hc[e * 74 + j] = 2 * (int)((e * 53 + j * 7) % 7000000);
  cudaMemcpy(codes, hc.data(), hc.size() * 4, cudaMemcpyHostToDevice);
  time_apply<42, 904, 4, 2>(M, codes, x, y, nt4);
  time_apply<42, 904, 8, 2>(M, codes, x, y, nt4);
  time_apply<42, 904, 8, 1>(M, codes, x, y, nt4);
  time_apply<42, 904, 16, 1>(M, codes, x, y, nt4);
  time_apply<42, 904, 12, 1>(M, codes, x, y, nt4);
  time_apply<74, 2776, 8, 1>(M, codes, x, y, nt6);
  time_apply<74, 2776, 4, 2>(M, codes, x, y, nt6);
  time_apply<74, 2776, 6, 1>(M, codes, x, y, nt6);
  double *bub, *acc; int* bidx; cudaMalloc(&bub, nt6 * 35 * 8); cudaMalloc(&acc, 8000000 * 8); cudaMalloc(&bidx, nt6 * 35 * 4);
  cudaMemset(bidx, 0, nt6 * 35 * 4);
  time_restrict<4, 8, 2>(M, bidx, codes, x, bub, acc, nt4);
  time_restrict<4, 16, 1>(M, bidx, codes, x, bub, acc, nt4);
  time_restrict<6, 8, 1>(M, bidx, codes, x, bub, acc, nt6);
  time_restrict<6, 12, 1>(M, bidx, codes, x, bub, acc, nt6);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
