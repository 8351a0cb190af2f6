// Exact coarse solve: GPU triangular solves of a host multifrontal Cholesky
// factorisation (the reference uses SuperLU,
// preconditioners.py:111-118,165-171).
//
// Per separator-tree node the factor is stored as dense explicit blocks:
// Linv = L_SS^-1 (packed lower, row-major), Linv^T (packed upper,
// row-major), W = F_BS L_SS^-T (nb x ns) and W^T.  One CTA per node and one
// kernel per tree level and direction:
//   forward   t = b_S - (child updates), y_S = Linv t,
//             out_B = W y_S + (child updates passing through)
//   backward  s = y_S - W^T x_B,  x_S = Linv^T s
// Child contributions are gathered through precomputed source indices in a
// fixed order (deterministic, no atomics); every GEMV is warp-per-row over
// contiguous rows (coalesced).
//
// node table (int64 x 10): s0, ns, nb, off_Linv, off_LinvT, off_W, off_WT, off_out, off_B, 0
#include "common.cuh"

namespace mcs {

constexpr int MF_THREADS = 256;

struct NodeRec {
  int64_t s0, ns, nb, oL, oLT, oW, oWT, oo, ob, pad;
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// shared layout per node: [t or s : ns][ys : ns][pass or xb : nb]
__global__ void __launch_bounds__(MF_THREADS)
    mf_forward(const int* __restrict__ level_nodes, const NodeRec* __restrict__ nodes,
               const double* __restrict__ mats, const int* __restrict__ src_t,
               const int* __restrict__ src_o, const int* __restrict__ perm,
               const double* __restrict__ b, double* __restrict__ y, double* __restrict__ out,
               int max_ns) {
  extern __shared__ double sm[];
  const NodeRec nd = nodes[level_nodes[blockIdx.x]];
  const int ns = (int)nd.ns, nb = (int)nd.nb;
  double* t = sm;
  double* ys = sm + max_ns;
  double* pass = sm + 2 * max_ns;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // all gathers up front, in parallel: own right-hand side and the child
  // updates that pass through to the boundary
  for (int j = threadIdx.x; j < ns + nb; j += MF_THREADS) {
    if (j < ns) {
      const int64_t p = nd.s0 + j;
      double v = __ldg(b + __ldg(perm + p));
      const int a = __ldg(src_t + 2 * p), c = __ldg(src_t + 2 * p + 1);
      if (a >= 0) v -= out[a];
      if (c >= 0) v -= out[c];
      t[j] = v;
    } else {
      const int64_t q = nd.oo + (j - ns);
      const int a = __ldg(src_o + 2 * q), c = __ldg(src_o + 2 * q + 1);
      double v = 0.0;
      if (a >= 0) v += out[a];
      if (c >= 0) v += out[c];
      pass[j - ns] = v;
    }
  }
  __syncthreads();
  const double* L = mats + nd.oL;
  for (int r = warp; r < ns; r += MF_THREADS / 32) {
    const double* row = L + (int64_t)r * (r + 1) / 2;
    double s = 0.0;
    for (int j = lane; j <= r; j += 32) s = fma(__ldg(row + j), t[j], s);
    s = warp_sum(s);
    if (lane == 0) {
      y[nd.s0 + r] = s;
      ys[r] = s;
    }
  }
  __syncthreads();
  const double* W = mats + nd.oW;
  for (int r = warp; r < nb; r += MF_THREADS / 32) {
    const double* row = W + (int64_t)r * ns;
    double s = 0.0;
    for (int j = lane; j < ns; j += 32) s = fma(__ldg(row + j), ys[j], s);
    s = warp_sum(s);
    if (lane == 0) out[nd.oo + r] = s + pass[r];
  }
}

__global__ void __launch_bounds__(MF_THREADS)
    mf_backward(const int* __restrict__ level_nodes, const NodeRec* __restrict__ nodes,
                const double* __restrict__ mats, const int* __restrict__ B,
                const int* __restrict__ perm, const double* __restrict__ y,
                double* __restrict__ xp, double* __restrict__ x, int max_ns) {
  extern __shared__ double sm[];
  const NodeRec nd = nodes[level_nodes[blockIdx.x]];
  const int ns = (int)nd.ns, nb = (int)nd.nb;
  double* s = sm;
  double* xb = sm + 2 * max_ns;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int* Bp = B + nd.ob;
  for (int j = threadIdx.x; j < nb; j += MF_THREADS) xb[j] = xp[__ldg(Bp + j)];
  __syncthreads();
  const double* WT = mats + nd.oWT;
  for (int r = warp; r < ns; r += MF_THREADS / 32) {
    const double* row = WT + (int64_t)r * nb;
    double a = 0.0;
    for (int j = lane; j < nb; j += 32) a = fma(__ldg(row + j), xb[j], a);
    a = warp_sum(a);
    if (lane == 0) s[r] = __ldg(y + nd.s0 + r) - a;
  }
  __syncthreads();
  const double* LT = mats + nd.oLT;     // packed upper, row r holds columns r..ns-1
  for (int r = warp; r < ns; r += MF_THREADS / 32) {
    const double* row = LT + (int64_t)r * ns - (int64_t)r * (r - 1) / 2 - r;
    double a = 0.0;
    for (int j = r + lane; j < ns; j += 32) a = fma(__ldg(row + j), s[j], a);
    a = warp_sum(a);
    if (lane == 0) {
      xp[nd.s0 + r] = a;
      x[perm[nd.s0 + r]] = a;
    }
  }
}

}  // namespace mcs

using namespace mcs;

MCS_API int mcs_mf_forward(int nnodes, const int* level_nodes, const void* nodes,
                           const double* mats, const int* src_t, const int* src_o,
                           const int* perm, const double* b, double* y, double* out, int max_ns,
                           int max_nb, void* stream) {
  if (nnodes <= 0) return 0;
  auto st = static_cast<cudaStream_t>(stream);
  const size_t smem = (2 * (size_t)max_ns + max_nb) * sizeof(double);
  cudaFuncSetAttribute(mf_forward, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  mf_forward<<<nnodes, MF_THREADS, smem, st>>>(level_nodes, static_cast<const NodeRec*>(nodes),
                                               mats, src_t, src_o, perm, b, y, out, max_ns);
  return launch_status();
}

MCS_API int mcs_mf_backward(int nnodes, const int* level_nodes, const void* nodes,
                            const double* mats, const int* B, const int* perm, const double* y,
                            double* xp, double* x, int max_ns, int max_nb, void* stream) {
  if (nnodes <= 0) return 0;
  auto st = static_cast<cudaStream_t>(stream);
  const size_t smem = (2 * (size_t)max_ns + max_nb) * sizeof(double);
  cudaFuncSetAttribute(mf_backward, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  mf_backward<<<nnodes, MF_THREADS, smem, st>>>(level_nodes, static_cast<const NodeRec*>(nodes),
                                                mats, B, perm, y, xp, x, max_ns);
  return launch_status();
}

// ---- top of the separator tree: dense explicit inverse of its Schur complement
namespace mcs {

// g[q] = b[perm[T[q]]] - sum_{p in src[ptr[q]..ptr[q+1])} out[p]   (fixed order)
__global__ void mf_top_gather(int t, const int* __restrict__ T, const int* __restrict__ perm,
                              const double* __restrict__ b, const int* __restrict__ ptr,
                              const int* __restrict__ src, const double* __restrict__ out,
                              double* __restrict__ g) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= t) return;
  double v = b[perm[T[q]]];
  for (int k = ptr[q]; k < ptr[q + 1]; ++k) v -= out[src[k]];
  g[q] = v;
}

// x_T = Sinv g (dense t x t, warp per row), scattered to xp[T[q]] and x[perm[T[q]]]
__global__ void mf_top_solve(int t, const double* __restrict__ Sinv, const double* __restrict__ g,
                             const int* __restrict__ T, const int* __restrict__ perm,
                             double* __restrict__ xp, double* __restrict__ x) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= t) return;
  const double* row = Sinv + (int64_t)w * t;
  double s = 0.0;
  for (int j = lane; j < t; j += 32) s = fma(row[j], g[j], s);
  s = warp_sum(s);
  if (lane == 0) {
    xp[T[w]] = s;
    x[perm[T[w]]] = s;
  }
}

}  // namespace mcs

MCS_API int mcs_mf_top(int t, const int* T, const int* perm, const double* b, const int* ptr,
                       const int* src, const double* out, double* g, const double* Sinv,
                       double* xp, double* x, void* stream) {
  if (t <= 0) return 0;
  auto st = static_cast<cudaStream_t>(stream);
  mf_top_gather<<<(t + 127) / 128, 128, 0, st>>>(t, T, perm, b, ptr, src, out, g);
  int rc = launch_status();
  if (rc) return rc;
  const int64_t threads = (int64_t)t * 32;
  mf_top_solve<<<(int)((threads + 255) / 256), 256, 0, st>>>(t, Sinv, g, T, perm, xp, x);
  return launch_status();
}
