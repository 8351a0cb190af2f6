// FP64-pipe arbitration on one SMSP, part 2: does the POSITION of the
// latency-critical warp matter?  A 12-warp CTA; warps 0, 4, 8 share SMSP 0
// (tools/smsp_map.cu).  One of them (the victim) runs a dependent chain
// (DMMA -> DFMA -> DMMA ..., or a shuffle + DFMA chain like the 8x8 Cholesky
// pivots); the other two stream DMMAs with CH independent chains.  Modes:
//   yield 0: plain streamers; 1: streamers __nanosleep(0) after every group of
//   CH DMMAs; 2: streamers issue a dependent integer op chain between groups.
// Prints the victim's latency and the streamers' DMMA rate.
#include <cstdio>
__device__ __forceinline__ void dmma(double2& c, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c.x), "+d"(c.y) : "d"(a), "d"(b));
}
template <int CH, int YIELD, int KIND>
__global__ void probe(double* out, long long* clk, int victim, int nstream, double a, int iters) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if ((warp & 3) != 0) return;                 // SMSP 0 only
  const int slot = warp >> 2;                   // 0, 1, 2
  if (slot == victim) {
    double2 c = make_double2(threadIdx.x, 1);
    double x = 1.0 + lane * 1e-3;
    long long tot = 0;
    for (int it = 0; it < 64; ++it) {
      long long t0 = clock64();
      if (KIND == 0) {
#pragma unroll
        for (int k = 0; k < 12; ++k) dmma(c, c.x * 1e-30 + a, c.y * 1e-30 + a);
      } else {                                  // 8 "pivots": shfl, rsqrt-like chain of 4 DFMA, shfl, fma
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          double d = __shfl_sync(0xffffffffu, x, k);
          double r = d * a;
          r = fma(r, 1e-9, r); r = fma(r, 1e-9, r); r = fma(r, 1e-9, r);
          x = fma(__shfl_sync(0xffffffffu, x * r, k + 1), 1e-9, x);
        }
      }
      tot += clock64() - t0;
      c.x += 1e-300;
    }
    if (lane == 0) { clk[blockIdx.x * 4] = tot / 64; out[0] = c.x + c.y + x; }
  } else {
    int rank = slot - (slot > victim ? 1 : 0);
    if (rank >= nstream) return;
    double2 c[CH];
    for (int k = 0; k < CH; ++k) c[k] = make_double2(k, threadIdx.x);
    unsigned z = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters / CH; ++i) {
#pragma unroll
      for (int k = 0; k < CH; ++k) dmma(c[k], a, 1e-9);
      if (YIELD == 1) __nanosleep(0);
      if (YIELD == 2) { z = z * 1664525u + 1013904223u; z ^= z >> 7; z = z * 22695477u + 1u; }
    }
    long long t1 = clock64();
    double s = z;
    for (int k = 0; k < CH; ++k) s += c[k].x;
    out[1 + threadIdx.x] = s;
    if (lane == 0) clk[blockIdx.x * 4 + 1 + rank] = (t1 - t0);
  }
}
template <int CH, int YIELD, int KIND>
void run(double* d, long long* c, int victim, int nstream) {
  const int iters = 20000;
  probe<CH, YIELD, KIND><<<148, 32 * 12>>>(d, c, victim, nstream, 1.0000001, iters);
  probe<CH, YIELD, KIND><<<148, 32 * 12>>>(d, c, victim, nstream, 1.0000001, iters);
  long long h[4]; cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
  printf("kind %d victim slot %d, %d streamers x %d chains, yield %d: victim %6lld clk; streamer clk/DMMA %.1f %.1f\n",
         KIND, victim, nstream, CH, YIELD, h[0], nstream > 0 ? (double)h[1] / iters : 0.0,
         nstream > 1 ? (double)h[2] / iters : 0.0);
}
int main() {
  double* d; long long* c; cudaMalloc(&d, 4096 * 8); cudaMalloc(&c, 1024 * 8);
  cudaMemset(c, 0, 1024 * 8);
  for (int victim = 0; victim < 3; ++victim)
    for (int ns = 0; ns <= 2; ++ns) {
      run<1, 0, 0>(d, c, victim, ns);
      run<2, 0, 0>(d, c, victim, ns);
      run<8, 0, 0>(d, c, victim, ns);
      run<2, 1, 0>(d, c, victim, ns);
      run<8, 1, 0>(d, c, victim, ns);
      run<2, 2, 0>(d, c, victim, ns);
      run<2, 0, 1>(d, c, victim, ns);
      run<8, 0, 1>(d, c, victim, ns);
      run<8, 1, 1>(d, c, victim, ns);
    }
}
