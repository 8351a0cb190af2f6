// Which SM sub-partition does warp w of a CTA run on?  %warpid % 4 for every
// warp of 64- and 128-thread CTAs, several CTAs per SM.
#include <cstdio>
__global__ void probe(int* out) {
  unsigned wid, smid;
  asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if ((threadIdx.x & 31) == 0) {
    const int w = threadIdx.x >> 5;
    out[(blockIdx.x * 8 + w) * 2] = wid;
    out[(blockIdx.x * 8 + w) * 2 + 1] = smid;
  }
  long long t = clock64();
  while (clock64() - t < 2000000) {}
}
int main() {
  int* d; cudaMalloc(&d, 148 * 16 * 8 * 2 * 4);
  for (int threads : {64, 128}) {
    const int blocks = 148 * 6;
    probe<<<blocks, threads>>>(d);
    int h[148 * 6 * 8 * 2];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    int hist[8][4] = {};
    for (int b = 0; b < blocks; ++b)
      for (int w = 0; w < threads / 32; ++w) hist[w][h[(b * 8 + w) * 2] % 4]++;
    printf("%d-thread CTAs: warp -> SMSP histogram (%%warpid %% 4)\n", threads);
    for (int w = 0; w < threads / 32; ++w)
      printf("  warp %d: %d %d %d %d\n", w, hist[w][0], hist[w][1], hist[w][2], hist[w][3]);
  }
}
