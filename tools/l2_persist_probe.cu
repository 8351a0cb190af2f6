// Probe: can the coarse top inverse (t x t doubles, read once per
// preconditioner application) stay resident in L2 across the ~500 MB of
// streaming traffic of a PCG iteration, via a persisting access-policy window?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2_persist_probe tools/l2_persist_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void gemv(int t, int ld, const double* __restrict__ S, const double* g, double* y) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= t) return;
  const double* row = S + (size_t)w * ld;
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  int j = lane;
  for (; j + 96 < t; j += 128) {
    s0 = fma(__ldg(row + j), g[j], s0);
    s1 = fma(__ldg(row + j + 32), g[j + 32], s1);
    s2 = fma(__ldg(row + j + 64), g[j + 64], s2);
    s3 = fma(__ldg(row + j + 96), g[j + 96], s3);
  }
  for (; j < t; j += 32) s0 = fma(__ldg(row + j), g[j], s0);
  double s = (s0 + s1) + (s2 + s3);
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(~0u, s, o);
  if (!lane) y[w] = s;
}

// CTA per row, double2 loads, U x NT loads in flight per CTA before any FMA
template <int NT, int U>
__global__ void __launch_bounds__(NT) gemv2(int ld2, const double2* __restrict__ S, const double2* g, double* y) {
  const double2* row = S + (size_t)blockIdx.x * ld2;
  double s = 0;
  for (int base = 0; base < ld2; base += NT * U) {
    double2 a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = base + u * NT + threadIdx.x;
      if (j < ld2) { a[u] = __ldg(row + j); b[u] = g[j]; } else { a[u] = b[u] = make_double2(0, 0); }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) s = fma(a[u].y, b[u].y, fma(a[u].x, b[u].x, s));
  }
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(~0u, s, o);
  __shared__ double red[NT / 32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = 0;
    for (int w = 0; w < NT / 32; ++w) v += red[w];
    y[blockIdx.x] = v;
  }
}

__global__ void stream_rw(size_t n, const double* __restrict__ a, double* __restrict__ b) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    b[i] = a[i] * 1.0000001;
}

int main(int argc, char** argv) {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  printf("l2 %d persistingL2CacheMaxSize %d accessPolicyMaxWindowSize %d\n", p.l2CacheSize,
         p.persistingL2CacheMaxSize, p.accessPolicyMaxWindowSize);
  const size_t nstream = (size_t)256 << 20;   // 2 x 256 MB streamed per "iteration"
  double *a, *b, *S, *g, *y;
  CK(cudaMalloc(&a, nstream));
  CK(cudaMalloc(&b, nstream));
  CK(cudaMemset(a, 0, nstream));
  const int ts[] = {2800, 3940, 4096};
  for (int ti = 0; ti < 3; ++ti) {
    const int t = ts[ti];
    const size_t bytes = (size_t)t * t * 8;
    CK(cudaMalloc(&S, bytes + 8 * t + 8));
    CK(cudaMalloc(&g, t * 8 + 8));
    CK(cudaMalloc(&y, t * 8));
    CK(cudaMemset(S, 0, bytes));
    CK(cudaMemset(g, 0, t * 8 + 8));
    for (int kv = 0; kv < 4; ++kv)
    for (int mode = 0; mode < 2; ++mode) {
      cudaStream_t st;
      CK(cudaStreamCreate(&st));
      if (mode) {
        size_t carve = bytes < (size_t)p.persistingL2CacheMaxSize ? bytes : p.persistingL2CacheMaxSize;
        CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, carve));
        cudaStreamAttrValue v = {};
        v.accessPolicyWindow.base_ptr = S;
        v.accessPolicyWindow.num_bytes = bytes < (size_t)p.accessPolicyMaxWindowSize ? bytes : p.accessPolicyMaxWindowSize;
        v.accessPolicyWindow.hitRatio = (float)carve / (float)v.accessPolicyWindow.num_bytes;
        if (v.accessPolicyWindow.hitRatio > 1.f) v.accessPolicyWindow.hitRatio = 1.f;
        v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        CK(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &v));
      }
      cudaEvent_t e0, e1;
      CK(cudaEventCreate(&e0));
      CK(cudaEventCreate(&e1));
      float tot = 0;
      const int it = 30;
      for (int i = 0; i < it + 3; ++i) {
        stream_rw<<<148 * 8, 256, 0, st>>>(nstream / 8, a, b);
        CK(cudaEventRecord(e0, st));
        if (kv == 0) gemv<<<(t * 32 + 255) / 256, 256, 0, st>>>(t, t, S, g, y);
        if (kv == 1) gemv2<128, 16><<<t, 128, 0, st>>>((t + 1) / 2, (const double2*)S, (const double2*)g, y);
        if (kv == 2) gemv2<256, 8><<<t, 256, 0, st>>>((t + 1) / 2, (const double2*)S, (const double2*)g, y);
        if (kv == 3) gemv2<64, 16><<<t, 64, 0, st>>>((t + 1) / 2, (const double2*)S, (const double2*)g, y);
        CK(cudaEventRecord(e1, st));
        CK(cudaStreamSynchronize(st));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (i >= 3) tot += ms;
      }
      printf("kv=%d t=%d (%.1f MB) persist=%d gemv %.2f us (%.0f GB/s)\n", kv, t, bytes / 1e6, mode,
             1e3 * tot / it, bytes / (1e-3 * tot / it) / 1e9);
      if (mode) {
        CK(cudaCtxResetPersistingL2Cache());
        CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0));
      }
      CK(cudaStreamDestroy(st));
    }
    CK(cudaFree(S));
    CK(cudaFree(g));
    CK(cudaFree(y));
  }
  return 0;
}
