// Single-warp latency / throughput probes on B200 (clock64):
// dependent DMMA m8n8k4, DFMA, shfl (f64), rcp.approx.f64, 8 independent DMMA
// chains in one warp, and DMMA throughput with 1/2/4/8 warps per SMSP.
#include <cstdio>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
__global__ void lat(long long* out, double a, double b) {
  double c0 = threadIdx.x, c1 = 1;
  long long t0 = clock64();
  for (int i = 0; i < 1000; ++i) dmma(c0, c1, a, b);
  long long t1 = clock64();
  double x = c0;
  long long t2 = clock64();
  for (int i = 0; i < 1000; ++i) x = fma(x, a, b);
  long long t3 = clock64();
  double d[8][2];
  for (int k = 0; k < 8; ++k) d[k][0] = d[k][1] = k;
  long long t4 = clock64();
  for (int i = 0; i < 250; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) dmma(d[k][0], d[k][1], a, b);
  long long t5 = clock64();
  double y = x;
  long long t6 = clock64();
  for (int i = 0; i < 1000; ++i) y = __shfl_sync(0xffffffffu, y, (threadIdx.x + 1) & 31) + 1e-30;
  long long t7 = clock64();
  double r = y + 1.5;
  long long t8 = clock64();
  for (int i = 0; i < 1000; ++i) asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(r));
  long long t9 = clock64();
  double s = x + c1 + y + r;
  for (int k = 0; k < 8; ++k) s += d[k][0] + d[k][1];
  if (threadIdx.x == 0) {
    out[0] = t1 - t0; out[1] = t3 - t2; out[2] = t5 - t4; out[3] = t7 - t6; out[4] = t9 - t8;
  }
  if (s == 1234.5) out[7] = 1;
}
// W warps per CTA, 1 CTA per SM, each warp: CH independent chains
template <int CH>
__global__ void thr(long long* out, double a, double b) {
  double d[CH][2];
  for (int k = 0; k < CH; ++k) d[k][0] = d[k][1] = k + threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < 2000 / CH; ++i)
#pragma unroll
    for (int k = 0; k < CH; ++k) dmma(d[k][0], d[k][1], a, b);
  long long t1 = clock64();
  double s = 0;
  for (int k = 0; k < CH; ++k) s += d[k][0] + d[k][1];
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  if (s == 1234.5) out[7] = 1;
}
int main() {
  long long* d; cudaMalloc(&d, 64);
  lat<<<1, 32>>>(d, 1.0000001, 1e-9); lat<<<1, 32>>>(d, 1.0000001, 1e-9);
  long long h[8]; cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
  printf("dependent DMMA %.1f clk; dependent DFMA %.1f; 8 indep DMMA chains %.1f clk/DMMA; "
         "shfl.f64 %.1f; rcp.approx.f64 %.1f\n", h[0] / 1000.0, h[1] / 1000.0, h[2] / 2000.0,
         h[3] / 1000.0, h[4] / 1000.0);
  for (int w : {4, 8, 16}) {
    for (int ch : {1, 2, 4, 8}) {
      auto k = ch == 1 ? thr<1> : ch == 2 ? thr<2> : ch == 4 ? thr<4> : thr<8>;
      k<<<148, 32 * w>>>(d, 1.0000001, 1e-9);
      k<<<148, 32 * w>>>(d, 1.0000001, 1e-9);
      cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
      // per-SMSP: w/4 warps x 2000 DMMA each
      printf("warps/SM %2d chains %d: %.2f clk per DMMA per SMSP\n", w, ch,
             h[0] / (2000.0 * w / 4));
    }
  }
}
