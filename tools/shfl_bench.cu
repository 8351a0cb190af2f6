#include <cstdio>
__global__ void k(long long* out, double x) {
  int lane = threadIdx.x;
  double v = x + lane;
  long long t0 = clock64();
  for (int i = 0; i < 1000; ++i) v = __shfl_sync(0xffffffffu, v, (lane + 1) & 31);
  long long t1 = clock64();
  double a[6]; for (int q = 0; q < 6; ++q) a[q] = v + q;
  long long t2 = clock64();
  for (int i = 0; i < 1000; ++i) {
#pragma unroll
    for (int q = 0; q < 6; ++q) a[q] = __shfl_sync(0xffffffffu, a[q], (lane + q) & 31);
  }
  long long t3 = clock64();
  float f = lane;
  long long t4 = clock64();
  for (int i = 0; i < 1000; ++i) f = __shfl_sync(0xffffffffu, f, (lane + 1) & 31);
  long long t5 = clock64();
  double s = v + f; for (int q = 0; q < 6; ++q) s += a[q];
  if (lane == 0) { out[0] = t1 - t0; out[1] = t3 - t2; out[2] = t5 - t4; }
  if (s == 1.2345) out[3] = 1;
}
int main() {
  long long* d; cudaMalloc(&d, 64); k<<<1, 32>>>(d, 1.0); k<<<1, 32>>>(d, 1.0);
  long long h[4]; cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
  printf("dependent shfl(double): %.1f clk; 6 independent shfl(double) per iter: %.1f clk/iter; dependent shfl(float): %.1f\n", h[0] / 1000.0, h[1] / 1000.0, h[2] / 1000.0);
}
