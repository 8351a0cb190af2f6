// Latency of one 8x8 pivot-block inverse (micro.cu pivot_inverse: FP32 seed +
// 3 DMMA Newton steps), alone on the SM and next to warps streaming DMMAs or
// scalar FP64 FMAs.  Measured: tools/chol8_lat -> profiles.
#include <cstdio>
#include "../paper_2207_08481_b200/csrc/micro.cu"
using namespace mcs;
__global__ void probe(double* out, long long* clk, int busy_warps, int kind) {
  __shared__ __align__(16) double tile[64];
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64; i += blockDim.x) tile[i] = (i / 8 == i % 8) ? -20.0 : -0.1;
  __syncthreads();
  if (warp == 0) {
    long long t0 = clock64();
    int b = 0;
    double2 acc = make_double2(0, 0);
    for (int it = 0; it < 16; ++it) {
      double2 x;
      b += micro::pivot_inverse(tile, micro::ld2(tile), x);
      acc.x += x.x;
      acc.y += x.y;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { clk[blockIdx.x] = (t1 - t0) / 16; out[0] = acc.x + acc.y + b; }
  } else if (warp <= busy_warps) {
    double2 c[4] = {};
    if (kind == 0) {
      for (int i = 0; i < 4000; ++i)
#pragma unroll
        for (int k = 0; k < 4; ++k) micro::dmma(c[k], 1.0000001, 1e-9);
    } else {
      for (int i = 0; i < 16000; ++i)
#pragma unroll
        for (int k = 0; k < 4; ++k) c[k].x = fma(c[k].x, 1.0000001, 1e-9);
    }
    out[1 + threadIdx.x] = c[0].x + c[1].x + c[2].x + c[3].y;
  }
}
int main() {
  double* d; long long* c; cudaMalloc(&d, 4096 * 8); cudaMalloc(&c, 1024 * 8);
  for (int kind = 0; kind < 2; ++kind)
    for (int bw : {0, 3, 7, 11}) {
      probe<<<148, 32 * 12>>>(d, c, bw, kind);
      probe<<<148, 32 * 12>>>(d, c, bw, kind);
      long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
      printf("pivot_inverse, %2d %s-streaming warps on the SM: %lld clk\n", bw,
             kind == 0 ? "DMMA" : "DFMA", h);
    }
}
