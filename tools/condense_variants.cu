// k=6 condensation kernel variants on synthetic well-posed element records
#include "../paper_2207_08481_b200/csrc/condense.cu"
#include <cstdio>
#include <vector>
#include <cmath>
constexpr int K = 6;
using Z = Sizes<K>;
using R = Record<K>;
template <int W, int MB>
void run_v3(const double* recs, double* ST, int* info, long nt, const std::vector<double>& ref) {
  using P = Pad<Z::ns + Z::nw, Z::nloc, W>;
  using G = v3::Geo<P::NB, P::NPB, W>;
  auto kern = condense_v3<K, W, MB>;
  size_t smem = G::SMEM * 8;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 32 * W, smem);
  int grid = per * 148;
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, kern);
  kern<<<grid, 32 * W, smem>>>(recs, ST, info, nt);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); kern<<<grid, 32 * W, smem>>>(recs, ST, info, nt); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  std::vector<double> S(nt * R::st_len); cudaMemcpy(S.data(), ST, S.size() * 8, cudaMemcpyDeviceToHost);
  double err = 0; for (size_t q = 0; q < S.size(); ++q) err = fmax(err, fabs(S[q] - ref[q]) / (fabs(ref[q]) + 1e-6));
  printf("v3 k=6 W=%2d minB=%d regs=%3d local=%zu ctas/sm=%d: %.2f ms  %.2f TF/s  maxrel %.1e (%s)\n", W, MB, fa.numRegs, fa.localSizeBytes, per, ms,
         1682184.0 * nt / (ms * 1e-3) / 1e12, err, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  const long nt = 16384;
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
  launch_condense<6, 16>(drec, dST, info, nt, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); launch_condense<6, 16>(drec, dST, info, nt, 0); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("v2 k=6 W=16: %.2f ms %.2f TF/s\n", ms, 1682184.0 * nt / (ms * 1e-3) / 1e12);
  std::vector<double> ref(nt * R::st_len); cudaMemcpy(ref.data(), dST, ref.size() * 8, cudaMemcpyDeviceToHost);
  std::vector<int> hi(nt); cudaMemcpy(hi.data(), info, nt * 4, cudaMemcpyDeviceToHost);
  int nbad = 0; for (int v : hi) nbad += v != 0; printf("bad elements (v2): %d\n", nbad);
  run_v3<8, 1>(drec, dST, info, nt, ref);
  run_v3<12, 1>(drec, dST, info, nt, ref);
  run_v3<16, 1>(drec, dST, info, nt, ref);
  run_v3<6, 1>(drec, dST, info, nt, ref);
}
