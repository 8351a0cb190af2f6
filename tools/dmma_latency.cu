// DMMA / DFMA latency and per-warp throughput on B200 (single warp, clock64)
#include <cstdio>
__global__ void lat(long long* out, double a, double b) {
  double c0 = threadIdx.x, c1 = 1;
  long long t0 = clock64();
  for (int i = 0; i < 1000; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  long long t1 = clock64();
  double x = c0;
  long long t2 = clock64();
  for (int i = 0; i < 1000; ++i) x = fma(x, a, b);
  long long t3 = clock64();
  // 8 independent DMMA chains
  double d[8][2];
  for (int k = 0; k < 8; ++k) d[k][0] = d[k][1] = k;
  long long t4 = clock64();
  for (int i = 0; i < 250; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(d[k][0]), "+d"(d[k][1]) : "d"(a), "d"(b));
  long long t5 = clock64();
  double s = x + c1;
  for (int k = 0; k < 8; ++k) s += d[k][0] + d[k][1];
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t3 - t2; out[2] = t5 - t4; }
  if (s == 1234.5) out[3] = 1;
}
int main() {
  long long* d; cudaMalloc(&d, 64);
  lat<<<1, 32>>>(d, 1.0000001, 1e-9); lat<<<1, 32>>>(d, 1.0000001, 1e-9);
  long long h[4]; cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
  printf("dependent DMMA: %.1f clk each; dependent DFMA: %.1f clk each; 8 indep DMMA chains: %.1f clk per DMMA\n",
         h[0] / 1000.0, h[1] / 1000.0, h[2] / 2000.0);
}
