// Exact coarse solve: GPU triangular solves of a host multifrontal Cholesky
// factorisation (the reference uses SuperLU,
// preconditioners.py:111-118,165-171).  Per separator-tree node the factor
// is stored as dense explicit blocks (Linv = L_SS^-1, its transpose, W and
// W^T), so each solve phase is a set of independent dense GEMVs, one warp
// per row, over a task list (node, row range) per tree level.  Child
// contributions are gathered through precomputed source indices in a fixed
// order (deterministic, no atomics).
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

// y_S = Linv (b_S - sum_children out)
__global__ void __launch_bounds__(MF_THREADS)
    mf_forward_own(const int* __restrict__ tasks, const NodeRec* __restrict__ nodes,
                   const double* __restrict__ mats, const int* __restrict__ src_t,
                   const double* __restrict__ out, const int* __restrict__ perm,
                   const double* __restrict__ b, double* __restrict__ y) {
  extern __shared__ double t[];
  const int* tk = tasks + 3 * blockIdx.x;
  const NodeRec nd = nodes[tk[0]];
  const int r0 = tk[1], r1 = tk[2];
  const int ns = (int)nd.ns;
  for (int j = threadIdx.x; j < ns; j += MF_THREADS) {
    const int64_t p = nd.s0 + j;
    double v = b[perm[p]];
    const int a = src_t[2 * p], c = src_t[2 * p + 1];
    if (a >= 0) v -= out[a];
    if (c >= 0) v -= out[c];
    t[j] = v;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* L = mats + nd.oL;
  for (int r = r0 + warp; r < r1; r += MF_THREADS / 32) {
    double s = 0.0;
    for (int j = lane; j <= r; j += 32) s = fma(L[(int64_t)r * ns + j], t[j], s);
    s = warp_sum(s);
    if (lane == 0) y[nd.s0 + r] = s;
  }
}

// out_B = W y_S + pass-through of children's updates
__global__ void __launch_bounds__(MF_THREADS)
    mf_forward_out(const int* __restrict__ tasks, const NodeRec* __restrict__ nodes,
                   const double* __restrict__ mats, const int* __restrict__ src_o,
                   const double* __restrict__ y, double* __restrict__ out) {
  const int* tk = tasks + 3 * blockIdx.x;
  const NodeRec nd = nodes[tk[0]];
  const int r0 = tk[1], r1 = tk[2];
  const int ns = (int)nd.ns;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* W = mats + nd.oW;
  const double* ys = y + nd.s0;
  for (int r = r0 + warp; r < r1; r += MF_THREADS / 32) {
    double s = 0.0;
    for (int j = lane; j < ns; j += 32) s = fma(W[(int64_t)r * ns + j], ys[j], s);
    s = warp_sum(s);
    if (lane == 0) {
      const int64_t q = nd.oo + r;
      const int a = src_o[2 * q], c = src_o[2 * q + 1];
      if (a >= 0) s += out[a];
      if (c >= 0) s += out[c];
      out[q] = s;
    }
  }
}

// s_S = y_S - W^T x_B
__global__ void __launch_bounds__(MF_THREADS)
    mf_backward(const int* __restrict__ tasks, const NodeRec* __restrict__ nodes,
                const double* __restrict__ mats, const int* __restrict__ B,
                const double* __restrict__ y, const double* __restrict__ xp,
                double* __restrict__ s) {
  const int* tk = tasks + 3 * blockIdx.x;
  const NodeRec nd = nodes[tk[0]];
  const int r0 = tk[1], r1 = tk[2];
  const int nb = (int)nd.nb;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* WT = mats + nd.oWT;
  const int* Bp = B + nd.ob;
  for (int r = r0 + warp; r < r1; r += MF_THREADS / 32) {
    double a = 0.0;
    for (int j = lane; j < nb; j += 32) a = fma(WT[(int64_t)r * nb + j], xp[Bp[j]], a);
    a = warp_sum(a);
    if (lane == 0) s[nd.s0 + r] = y[nd.s0 + r] - a;
  }
}

// x_S = Linv^T s_S ; scatter to the caller's ordering
__global__ void __launch_bounds__(MF_THREADS)
    mf_backward2(const int* __restrict__ tasks, const NodeRec* __restrict__ nodes,
                 const double* __restrict__ mats, const double* __restrict__ s,
                 const int* __restrict__ perm, double* __restrict__ xp, double* __restrict__ x) {
  extern __shared__ double ss[];
  const int* tk = tasks + 3 * blockIdx.x;
  const NodeRec nd = nodes[tk[0]];
  const int r0 = tk[1], r1 = tk[2];
  const int ns = (int)nd.ns;
  for (int j = threadIdx.x; j < ns; j += MF_THREADS) ss[j] = s[nd.s0 + j];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* LT = mats + nd.oLT;
  for (int r = r0 + warp; r < r1; r += MF_THREADS / 32) {
    double a = 0.0;
    for (int j = r + lane; j < ns; j += 32) a = fma(LT[(int64_t)r * ns + j], ss[j], a);
    a = warp_sum(a);
    if (lane == 0) {
      xp[nd.s0 + r] = a;
      x[perm[nd.s0 + r]] = a;
    }
  }
}

static int g_max_ns = 0;

}  // namespace mcs

using namespace mcs;

// shared memory is sized from the largest node (set once per factor)
MCS_API int mcs_mf_set_max_own(int max_ns) {
  if (max_ns > g_max_ns) g_max_ns = max_ns;
  const int bytes = g_max_ns * (int)sizeof(double);
  cudaFuncSetAttribute(mf_forward_own, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(mf_backward2, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  return launch_status();
}

MCS_API int mcs_mf_forward_own(int ntasks, const int* tasks, const void* nodes, const double* mats,
                               const int* src_t, const double* out, const int* perm, const double* b,
                               double* y, void* stream) {
  auto st = static_cast<cudaStream_t>(stream);
  mf_forward_own<<<ntasks, MF_THREADS, g_max_ns * sizeof(double), st>>>(
      tasks, static_cast<const NodeRec*>(nodes), mats, src_t, out, perm, b, y);
  return launch_status();
}

MCS_API int mcs_mf_forward_out(int ntasks, const int* tasks, const void* nodes, const double* mats,
                               const int* src_o, const double* y, double* out, void* stream) {
  auto st = static_cast<cudaStream_t>(stream);
  mf_forward_out<<<ntasks, MF_THREADS, 0, st>>>(tasks, static_cast<const NodeRec*>(nodes), mats,
                                                src_o, y, out);
  return launch_status();
}

MCS_API int mcs_mf_backward(int ntasks, const int* tasks, const void* nodes, const double* mats,
                            const int* B, const double* y, const double* xp, double* s,
                            void* stream) {
  auto st = static_cast<cudaStream_t>(stream);
  mf_backward<<<ntasks, MF_THREADS, 0, st>>>(tasks, static_cast<const NodeRec*>(nodes), mats, B,
                                             y, xp, s);
  return launch_status();
}

MCS_API int mcs_mf_backward2(int ntasks, const int* tasks, const void* nodes, const double* mats,
                             const double* s, const int* perm, double* xp, double* x,
                             void* stream) {
  auto st = static_cast<cudaStream_t>(stream);
  mf_backward2<<<ntasks, MF_THREADS, g_max_ns * sizeof(double), st>>>(
      tasks, static_cast<const NodeRec*>(nodes), mats, s, perm, xp, x);
  return launch_status();
}
