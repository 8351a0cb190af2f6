// Achievable HBM read bandwidth on this B200 for the access patterns of the
// element operators: (a) plain 16-byte vector loads, grid-stride; (b) 1-D
// bulk copies (cp.async.bulk) of REC-byte records into a per-warp ring, no
// compute; (c) the same through a CTA-wide ring with one producer thread.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/read_bw_probe tools/read_bw_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c)); }
__device__ __forceinline__ void mb_tx(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(d)), "l"(s), "r"(n), "r"(sa(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(sa(b)), "r"(ph) : "memory");
}

__global__ void rd_vec(const double2* __restrict__ a, size_t n, double* out) {
  double s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double2 v = __ldg(a + i);
    s += v.x + v.y;
  }
  if (s == 123.456) *out = s;
}

// per-warp ring of NST records
template <int NST>
__global__ void rd_bulk_warp(const double* __restrict__ a, int64_t nrec, int rec, double* out) {
  extern __shared__ __align__(128) double sm[];
  __shared__ uint64_t bar[32][NST];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x >> 5;
  double* st = sm + (size_t)w * NST * rec;
  const int64_t gw = (int64_t)blockIdx.x * W + w, nw = (int64_t)gridDim.x * W;
  if (lane == 0) {
    for (int q = 0; q < NST; ++q) mb_init(&bar[w][q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int q = 0; q < NST; ++q)
      if (gw + q * nw < nrec) { mb_tx(&bar[w][q], rec * 8); bulk(st + q * rec, a + (gw + q * nw) * rec, rec * 8, &bar[w][q]); }
  }
  __syncwarp();
  double s = 0;
  int it = 0;
  for (int64_t e = gw; e < nrec; e += nw, ++it) {
    const int q = it % NST;
    mb_wait(&bar[w][q], (it / NST) & 1);
    s += st[q * rec + lane];
    __syncwarp();
    if (lane == 0 && e + NST * nw < nrec) { mb_tx(&bar[w][q], rec * 8); bulk(st + q * rec, a + (e + NST * nw) * rec, rec * 8, &bar[w][q]); }
  }
  if (s == 123.456) *out = s;
}

int main() {
  const size_t bytes = (size_t)256 << 20;
  double *a, *out, *fl;
  CK(cudaMalloc(&a, bytes));
  CK(cudaMalloc(&fl, bytes));
  CK(cudaMalloc(&out, 8));
  CK(cudaMemset(a, 0, bytes));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double* fl2;
  CK(cudaMalloc(&fl2, bytes));
  CK(cudaMemset(fl2, 0, bytes));
  int clean = 0;   // 1: after the write flush, read another 256 MB so L2 holds no dirty lines
  auto timeit = [&](auto launch, const char* name, double nbytes) {
    float best = 1e9, tot = 0;
    for (int i = 0; i < 12; ++i) {
      cudaMemsetAsync(fl, i, bytes);   // L2 flush
      if (clean) rd_vec<<<148 * 8, 256>>>((const double2*)fl2, bytes / 16, out);
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (i >= 2) { tot += ms; best = ms < best ? ms : best; }
    }
    printf("clean=%d %-40s mean %7.2f us  %6.0f GB/s   best %6.0f GB/s\n", clean, name, tot / 10 * 1e3, nbytes / (tot / 10 * 1e-3) / 1e9, nbytes / (best * 1e-3) / 1e9);
  };
  for (clean = 0; clean < 2; ++clean) {
  for (int g : {148 * 4, 148 * 8, 148 * 16})
    timeit([&] { rd_vec<<<g, 256>>>((const double2*)a, bytes / 16, out); }, g == 592 ? "vec2 loads grid 592x256" : g == 1184 ? "vec2 loads grid 1184x256" : "vec2 loads grid 2368x256", bytes);
  const int recs[] = {904, 526, 378};
  for (int rec : recs) {
    const int64_t nrec = bytes / (rec * 8);
    for (int W : {4, 8}) {
      const int NST = 1;
      size_t smem = (size_t)W * NST * rec * 8;
      cudaFuncSetAttribute(rd_bulk_warp<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      int per = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, rd_bulk_warp<1>, W * 32, smem);
      char nm[96];
      snprintf(nm, sizeof nm, "bulk rec %d B W=%d NST=1 (%d CTA/SM)", rec * 8, W, per);
      timeit([&] { rd_bulk_warp<1><<<per * 148, W * 32, smem>>>(a, nrec, rec, out); }, nm, (double)nrec * rec * 8);
    }
    for (int W : {2, 4}) {
      size_t smem = (size_t)W * 2 * rec * 8;
      cudaFuncSetAttribute(rd_bulk_warp<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      int per = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, rd_bulk_warp<2>, W * 32, smem);
      char nm[96];
      snprintf(nm, sizeof nm, "bulk rec %d B W=%d NST=2 (%d CTA/SM)", rec * 8, W, per);
      timeit([&] { rd_bulk_warp<2><<<per * 148, W * 32, smem>>>(a, nrec, rec, out); }, nm, (double)nrec * rec * 8);
    }
  }
  }
  return 0;
}
