// MCS sigma/omega condensation: production kernel (mcs_condense) vs the v5
// engine for every k, on synthetic well-posed element records.
#include "../paper_2207_08481_b200/csrc/condense.cu"
#include <cstdio>
#include <vector>
#include <cmath>

template <int K>
double flops() {
  using Z = Sizes<K>;
  const double ns = Z::ns, nw = Z::nw, nl = Z::nloc;
  return ns * ns * ns / 3 + ns * ns * (nl + nw) + nw * nw * ns + nw * nw * nw / 3 + 2 * nw * ns * nl +
         nw * nw * nl + nl * nl * ns + nl * nl * nw;
}

template <int K, int W, int MB>
void run5(const double* recs, double* ST, int* info, long nt, const std::vector<double>& ref) {
  using R = Record<K>;
  using G = McsGeo5<K, W>;
  auto kern = condense_v5<K, W, MB>;
  size_t smem = G::SMEM * 8;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 32 * W, smem);
  if (per == 0) { printf("v5 k=%d W=%d: does not fit\n", K, W); return; }
  int grid = per * 148;
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, kern);
  cudaMemset(ST, 0, nt * R::st_len * 8);
  kern<<<grid, 32 * W, smem>>>(recs, ST, info, nt);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); kern<<<grid, 32 * W, smem>>>(recs, ST, info, nt); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  std::vector<double> S(nt * R::st_len); cudaMemcpy(S.data(), ST, S.size() * 8, cudaMemcpyDeviceToHost);
  std::vector<int> hi(nt); cudaMemcpy(hi.data(), info, nt * 4, cudaMemcpyDeviceToHost);
  int nbad = 0; for (int v : hi) nbad += v != 0;
  double num = 0, den = 0;
  for (size_t q = 0; q < S.size(); ++q) { num += (S[q] - ref[q]) * (S[q] - ref[q]); den += ref[q] * ref[q]; }
  printf("v5 k=%d W=%2d minB=%d regs=%3d local=%zu smem=%zu ctas/sm=%d: %.3f ms  %.2f TF/s  relF %.1e bad %d (%s)\n", K, W, MB,
         fa.numRegs, fa.localSizeBytes, smem, per, ms, flops<K>() * nt / (ms * 1e-3) / 1e12, sqrt(num / den), nbad,
         cudaGetErrorString(cudaGetLastError()));
}

template <int K>
void sweep(long nt) {
  using Z = Sizes<K>;
  using R = Record<K>;
  std::vector<double> rec(nt * R::len, 0.0);
  unsigned s = 7;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return (s >> 8) / 16777216.0 - 0.5; };
  for (long e = 0; e < nt; ++e) {
    double* r = rec.data() + e * R::len;
    for (int i = 0; i < Z::ns; ++i) for (int j = 0; j <= i; ++j) { double v = (i == j ? 2.0 * Z::ns : 0.0) + rnd(); r[R::o_msig + i * Z::ns + j] = v; r[R::o_msig + j * Z::ns + i] = v; }
    for (int q = 0; q < Z::nw * Z::ns; ++q) r[R::o_bws + q] = rnd();
    for (int q = 0; q < Z::nu * Z::ns; ++q) r[R::o_bus + q] = rnd();
    for (int q = 0; q < Z::nh * Z::ns; ++q) r[R::o_bhs + q] = rnd();
    for (int i = 0; i < Z::nu; ++i) for (int j = 0; j <= i; ++j) { double v = (i == j ? 1.0 : 0.0) + 0.01 * rnd(); r[R::o_adiv + i * Z::nu + j] = v; r[R::o_adiv + j * Z::nu + i] = v; }
  }
  double *drec, *dST; int* info;
  cudaMalloc(&drec, rec.size() * 8); cudaMalloc(&dST, nt * R::st_len * 8); cudaMalloc(&info, nt * 4);
  cudaMemcpy(drec, rec.data(), rec.size() * 8, cudaMemcpyHostToDevice);
  mcs_condense(K, nt, drec, dST, info, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); mcs_condense(K, nt, drec, dST, info, 0); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("prod k=%d: %.3f ms %.2f TF/s\n", K, ms, flops<K>() * nt / (ms * 1e-3) / 1e12);
  std::vector<double> ref(nt * R::st_len); cudaMemcpy(ref.data(), dST, ref.size() * 8, cudaMemcpyDeviceToHost);
  run5<K, 2, 8>(drec, dST, info, nt, ref);
  run5<K, 4, 4>(drec, dST, info, nt, ref);
  run5<K, 4, 5>(drec, dST, info, nt, ref);
  run5<K, 8, 2>(drec, dST, info, nt, ref);
  if (K >= 5) { run5<K, 8, 1>(drec, dST, info, nt, ref); run5<K, 16, 1>(drec, dST, info, nt, ref); }
  cudaFree(drec); cudaFree(dST); cudaFree(info);
}

int main() {
  sweep<2>(131072);
  sweep<3>(131072);
  sweep<4>(65536);
  sweep<5>(32768);
  sweep<6>(32768);
}
