// FP64 peak microbenchmark for the roofline denominator (DFMA pipe and DMMA).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void dmma_m8n8k4_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int k = 0; k < 8; ++k) { c[k][0] = 0; c[k][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void dmma_m16n8k16_kernel(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3 + k;
#pragma unroll
  for (int k = 0; k < 4; ++k) b[k] = 1.0 - threadIdx.x * 1e-4 - k;
  double c[4][4];
#pragma unroll
  for (int k = 0; k < 4; ++k) { c[k][0] = c[k][1] = c[k][2] = c[k][3] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
  if (s == 12345.678) out[threadIdx.x] = s;
}

int main() {
  int dev = 0, nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  double* out; cudaMalloc(&out, 4096 * sizeof(double));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  double best_dfma = 0, best_m884 = 0, best_m16816 = 0;
  for (int rep = 0; rep < 5; ++rep) {
    // DFMA: 8 chains per thread, 256 threads, 8 CTAs per SM
    int iters = 20000, threads = 256, blocks = nsm * 8;
    dfma_kernel<8><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e0);
    dfma_kernel<8><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * (double)iters * threads * blocks;
    if (fl / (ms * 1e-3) > best_dfma) best_dfma = fl / (ms * 1e-3);
    // DMMA m8n8k4: 8x8x4 = 256 FMA per warp-instruction
    iters = 4000;
    dmma_m8n8k4_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e0);
    dmma_m8n8k4_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 256 * 8 * (double)iters * (threads / 32) * blocks;
    if (fl / (ms * 1e-3) > best_m884) best_m884 = fl / (ms * 1e-3);
    iters = 1000;
    dmma_m16n8k16_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e0);
    dmma_m16n8k16_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 16 * 8 * 16 * 4 * (double)iters * (threads / 32) * blocks;
    if (fl / (ms * 1e-3) > best_m16816) best_m16816 = fl / (ms * 1e-3);
  }
  cudaError_t err = cudaGetLastError();
  printf("{\"sms\": %d, \"dfma_tflops\": %.3f, \"dmma_m8n8k4_tflops\": %.3f, \"dmma_m16n8k16_tflops\": %.3f, \"err\": \"%s\"}\n",
         nsm, best_dfma / 1e12, best_m884 / 1e12, best_m16816 / 1e12, cudaGetErrorString(err));
  return err == cudaSuccess ? 0 : 1;
}
