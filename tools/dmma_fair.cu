// DMMA arbitration on one SMSP: latency of a dependent chain of 12 DMMAs in
// warp 0 while other warps stream DMMAs with CH independent chains each.
#include <cstdio>
__device__ __forceinline__ void dmma(double2& c, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c.x), "+d"(c.y) : "d"(a), "d"(b));
}
template <int CH>
__global__ void probe(double* out, long long* clk, int busy, double a) {
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    double2 c = make_double2(threadIdx.x, 1);
    long long tot = 0;
    for (int it = 0; it < 64; ++it) {
      long long t0 = clock64();
#pragma unroll
      for (int k = 0; k < 12; ++k) dmma(c, c.x * 1e-30 + a, c.y * 1e-30 + a);
      tot += clock64() - t0;
      c.x += 1e-300;
    }
    if (threadIdx.x == 0) { clk[blockIdx.x] = tot / 64; out[0] = c.x + c.y; }
  } else if (warp <= busy) {
    double2 c[CH];
    for (int k = 0; k < CH; ++k) c[k] = make_double2(k, threadIdx.x);
    for (int i = 0; i < 20000 / CH; ++i)
#pragma unroll
      for (int k = 0; k < CH; ++k) dmma(c[k], a, 1e-9);
    double s = 0;
    for (int k = 0; k < CH; ++k) s += c[k].x;
    out[1 + threadIdx.x] = s;
  }
}
int main() {
  double* d; long long* c; cudaMalloc(&d, 4096 * 8); cudaMalloc(&c, 1024 * 8);
  for (int ch : {1, 2, 4, 8})
    for (int bw : {0, 4, 8}) {
      auto k = ch == 1 ? probe<1> : ch == 2 ? probe<2> : ch == 4 ? probe<4> : probe<8>;
      k<<<148, 32 * 12>>>(d, c, bw, 1.0000001);
      k<<<148, 32 * 12>>>(d, c, bw, 1.0000001);
      long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
      printf("12 dependent DMMAs: %5lld clk with %d streaming warps on the SMSP (%d chains each)\n",
             h, bw / 4, ch);
    }
}
