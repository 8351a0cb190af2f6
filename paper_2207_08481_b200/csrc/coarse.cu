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
// fixed order (deterministic, no atomics).  Every GEMV is warp-per-row over
// contiguous rows (coalesced), RPW rows per warp walked together so that
// several independent loads per lane are in flight (one row at a time
// serialises a memory latency plus a shuffle tree per row: ~20 us levels).
//
// node table (int64 x 10): s0, ns, nb, off_Linv, off_LinvT, off_W, off_WT, off_out, off_B, 0
#include "common.cuh"

namespace mcs {

constexpr int MF_THREADS = 256;

struct NodeRec {
  int64_t s0, ns, nb, oL, oLT, oW, oWT, oo, ob, nslot;   // nslot: gather sources per entry (>= 2)
};

// start of row j of a packed-upper row-major n x n matrix, minus j (so that
// element (j, c), c >= j, sits at upk_row(j, n) + c)
__device__ __forceinline__ int64_t upk_row(int j, int n) {
  return (int64_t)j * n - (int64_t)j * (j - 1) / 2 - j;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Warp-cooperative GEMV rows: for r in [0, nrows), v_r = sum_{j in [lo, hi)}
// row_r[j] x[j] with (row_r, lo, hi) = ROW(r); each warp takes RPW rows at a
// time and walks them together 32 columns per step, so RPW coalesced loads
// per lane are in flight instead of one; then EMIT(r, v_r) on lane 0.
constexpr int RPW = 4;
template <class ROW, class EMIT>
__device__ __forceinline__ void warp_rows(int nrows, const double* __restrict__ x, ROW row,
                                          EMIT emit) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int NW = MF_THREADS / 32;
  for (int r0 = warp * RPW; r0 < nrows; r0 += NW * RPW) {
    const double* p[RPW];
    int lo[RPW], hi[RPW];
    int jmin = 1 << 30, jmax = 0;
#pragma unroll
    for (int u = 0; u < RPW; ++u) {
      lo[u] = 0;
      hi[u] = 0;
      p[u] = x;
      if (r0 + u < nrows) row(r0 + u, p[u], lo[u], hi[u]);
      jmin = min(jmin, lo[u]);
      jmax = max(jmax, hi[u]);
    }
    double acc[RPW];
#pragma unroll
    for (int u = 0; u < RPW; ++u) acc[u] = 0.0;
    // JU column steps per batch, all RPW x JU loads issued before the first FMA
    // (issue is in order: a consumer waiting on a load blocks the next loads)
    constexpr int JU = 4;
    for (int j0 = jmin + lane; j0 < jmax; j0 += 32 * JU) {
      double v[RPW][JU], xv[JU];
#pragma unroll
      for (int c = 0; c < JU; ++c) {
        const int j = j0 + 32 * c;
        xv[c] = j < jmax ? x[j] : 0.0;
#pragma unroll
        for (int u = 0; u < RPW; ++u) v[u][c] = (j >= lo[u] && j < hi[u]) ? __ldg(p[u] + j) : 0.0;
      }
#pragma unroll
      for (int c = 0; c < JU; ++c)
#pragma unroll
        for (int u = 0; u < RPW; ++u) acc[u] = fma(v[u][c], xv[c], acc[u]);
    }
#pragma unroll
    for (int u = 0; u < RPW; ++u) acc[u] = warp_sum(acc[u]);
    if (lane == 0) {
#pragma unroll
      for (int u = 0; u < RPW; ++u)
        if (r0 + u < nrows) emit(r0 + u, acc[u]);
    }
  }
}

// Thread-per-row GEMV for narrow rows (width <= THREAD_ROW_MAX): every row of
// the node is in flight at once (one memory round trip instead of one per
// 32 rows per warp); each thread reads its row's contiguous span, 4 partial
// sums in a fixed order (deterministic).
constexpr int THREAD_ROW_MAX = 48;
template <class ROW, class EMIT>
__device__ __forceinline__ void thread_rows(int nrows, const double* __restrict__ x, ROW row,
                                            EMIT emit) {
  for (int r = threadIdx.x; r < nrows; r += MF_THREADS) {
    const double* p;
    int lo, hi;
    row(r, p, lo, hi);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int j = lo;
    for (; j + 3 < hi; j += 4) {
      a0 = fma(__ldg(p + j), x[j], a0);
      a1 = fma(__ldg(p + j + 1), x[j + 1], a1);
      a2 = fma(__ldg(p + j + 2), x[j + 2], a2);
      a3 = fma(__ldg(p + j + 3), x[j + 3], a3);
    }
    for (; j < hi; ++j) a0 = fma(__ldg(p + j), x[j], a0);
    emit(r, (a0 + a1) + (a2 + a3));
  }
}

template <class ROW, class EMIT>
__device__ __forceinline__ void node_rows(int nrows, int width, const double* __restrict__ x,
                                          ROW row, EMIT emit) {
  if (width <= THREAD_ROW_MAX) thread_rows(nrows, x, row, emit);
  else warp_rows(nrows, x, row, emit);
}

// shared layout per node: [t or s : ns][ys : ns][pass or xb : nb]
__global__ void __launch_bounds__(MF_THREADS)
    mf_forward(const int* __restrict__ level_nodes, const NodeRec* __restrict__ nodes,
               const double* __restrict__ mats, const int* __restrict__ src_t,
               const int* __restrict__ src_o, const int* __restrict__ perm,
               const double* b, double* __restrict__ y, double* out, int max_ns) {
  extern __shared__ double sm[];
  const NodeRec nd = nodes[level_nodes[blockIdx.x]];
  {   // static factors -> L2 while the previous level finishes
    const char* c0 = reinterpret_cast<const char*>(mats + nd.oL);
    const char* c1 = reinterpret_cast<const char*>(mats + nd.oW);
    const int64_t n0 = 8 * nd.ns * (nd.ns + 1) / 2, n1 = 8 * nd.nb * nd.ns;
    for (int64_t o = threadIdx.x * 128; o < n0; o += MF_THREADS * 128)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(c0 + o));
    for (int64_t o = threadIdx.x * 128; o < n1; o += MF_THREADS * 128)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(c1 + o));
  }
  pdl_wait();
  pdl_trigger();
  const int ns = (int)nd.ns, nb = (int)nd.nb;
  double* t = sm;
  double* ys = sm + max_ns;
  double* pass = sm + 2 * max_ns;
  // all gathers up front, in parallel: own right-hand side and the child
  // updates that pass through to the boundary
  for (int j = threadIdx.x; j < ns + nb; j += MF_THREADS) {
    const int S = (int)nd.nslot;
    if (j < ns) {
      const int64_t p = nd.s0 + j;
      double v = b[__ldg(perm + p)];
      const int* sp = src_t + S * p;
      for (int q = 0; q < S; ++q) {      // fixed order: deterministic
        const int a = __ldg(sp + q);
        if (a >= 0) v -= out[a];
      }
      t[j] = v;
    } else {
      const int* sp = src_o + S * (nd.oo + (j - ns));
      double v = 0.0;
      for (int q = 0; q < S; ++q) {
        const int a = __ldg(sp + q);
        if (a >= 0) v += out[a];
      }
      pass[j - ns] = v;
    }
  }
  __syncthreads();
  // y_S = Linv t (packed lower, row-major), then out_B = W y_S + pass
  const double* L = mats + nd.oL;
  node_rows(
      ns, ns, t,
      [&](int r, const double*& p, int& lo, int& hi) {
        p = L + (int64_t)r * (r + 1) / 2;
        lo = 0;
        hi = r + 1;
      },
      [&](int r, double v) {
        y[nd.s0 + r] = v;
        ys[r] = v;
      });
  __syncthreads();
  const double* W = mats + nd.oW;
  node_rows(
      nb, ns, ys,
      [&](int r, const double*& p, int& lo, int& hi) {
        p = W + (int64_t)r * ns;
        lo = 0;
        hi = ns;
      },
      [&](int r, double v) { out[nd.oo + r] = v + pass[r]; });
}

__global__ void __launch_bounds__(MF_THREADS)
    mf_backward(const int* __restrict__ level_nodes, const NodeRec* __restrict__ nodes,
                const double* __restrict__ mats, const int* __restrict__ B,
                const int* __restrict__ perm, const double* y,
                double* xp, double* __restrict__ x, int max_ns) {
  extern __shared__ double sm[];
  const NodeRec nd = nodes[level_nodes[blockIdx.x]];
  {   // static factors -> L2 while the previous level finishes
    const char* c0 = reinterpret_cast<const char*>(mats + nd.oWT);
    const char* c1 = reinterpret_cast<const char*>(mats + nd.oLT);
    const int64_t n0 = 8 * nd.nb * nd.ns, n1 = 8 * nd.ns * (nd.ns + 1) / 2;
    for (int64_t o = threadIdx.x * 128; o < n0; o += MF_THREADS * 128)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(c0 + o));
    for (int64_t o = threadIdx.x * 128; o < n1; o += MF_THREADS * 128)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(c1 + o));
  }
  pdl_wait();
  pdl_trigger();
  const int ns = (int)nd.ns, nb = (int)nd.nb;
  double* s = sm;
  double* xb = sm + 2 * max_ns;
  const int* Bp = B + nd.ob;
  for (int j = threadIdx.x; j < nb; j += MF_THREADS) xb[j] = xp[__ldg(Bp + j)];
  __syncthreads();
  // s = y_S - W^T x_B (W^T row-major ns x nb), then x_S = Linv^T s (packed upper)
  const double* WT = mats + nd.oWT;
  node_rows(
      ns, nb, xb,
      [&](int r, const double*& p, int& lo, int& hi) {
        p = WT + (int64_t)r * nb;
        lo = 0;
        hi = nb;
      },
      [&](int r, double v) { s[r] = y[nd.s0 + r] - v; });
  __syncthreads();
  const double* LT = mats + nd.oLT;  // packed upper, row r holds columns r..ns-1
  node_rows(
      ns, ns, s,
      [&](int r, const double*& p, int& lo, int& hi) {
        p = LT + upk_row(r, ns);
        lo = r;
        hi = ns;
      },
      [&](int r, double v) {
        xp[nd.s0 + r] = v;
        x[perm[nd.s0 + r]] = v;
      });
}

// ---- shared-memory staged variants (the default when a level's blocks fit) --
// Each node's factor blocks are contiguous in `mats`, 16-byte aligned:
//   forward block  [Linv packed lower | W (nb x ns)]    at off_Linv
//   backward block [W^T (ns x nb) | Linv^T packed upper] at off_WT
// One bulk copy (TMA engine) per CTA moves the block into shared memory and
// the static gather indices go to registers, both before pdl_wait(): the
// factor fetch overlaps the previous level, and after the wait a level costs
// one dependent global round trip (the gathered right-hand side) plus
// shared-memory GEMVs.

// Rows r in [0, nrows) of a matrix in shared memory: v_r = sum_{j in [lo, hi)}
// p_r[j] x[j], G lanes per row (G a power of two <= 8, chosen so that the
// rows of one pass cover the block), fixed-order shuffle reduction.
template <class ROW, class EMIT>
__device__ __forceinline__ void smem_rows(int nrows, int width, const double* x, ROW row,
                                          EMIT emit) {
  int G = 1;
  while (G < 8 && nrows * G * 2 <= MF_THREADS && G * 8 < width) G *= 2;
  const int sub = threadIdx.x & (G - 1);
  for (int r0 = 0; r0 < nrows; r0 += MF_THREADS / G) {
    const int r = r0 + threadIdx.x / G;
    double a0 = 0.0, a1 = 0.0;
    if (r < nrows) {
      const double* p;
      int lo, hi;
      row(r, p, lo, hi);
      int j = lo + sub;
      for (; j + G < hi; j += 2 * G) {
        a0 = fma(p[j], x[j], a0);
        a1 = fma(p[j + G], x[j + G], a1);
      }
      if (j < hi) a0 = fma(p[j], x[j], a0);
    }
    double v = a0 + a1;
    for (int o = G >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (r < nrows && sub == 0) emit(r, v);
  }
}

constexpr int MF_PRE = 2;   // gather indices preloaded per thread (ns + nb <= 512)

__global__ void __launch_bounds__(MF_THREADS)
    mf_forward_s(const int* __restrict__ level_nodes, const NodeRec* __restrict__ nodes,
                 const double* __restrict__ mats, const int* __restrict__ src_t,
                 const int* __restrict__ src_o, const int* __restrict__ perm, const double* b,
                 double* __restrict__ y, double* out, int blk_max, int max_ns) {
  extern __shared__ __align__(16) double sm[];
  __shared__ uint64_t bar;
  const NodeRec nd = nodes[level_nodes[blockIdx.x]];
  const int ns = (int)nd.ns, nb = (int)nd.nb;
  double* F = sm;
  double* t = sm + blk_max;
  double* ys = t + max_ns;
  double* pass = ys + max_ns;
  if (threadIdx.x == 0) {
    const int len = even(npk(ns) + nb * ns);
    mbar_init(&bar, 1);
    fence_barrier_init();
    mbar_expect_tx(&bar, len * 8);
    if (len) bulk_g2s(F, mats + nd.oL, len * 8, &bar);
  }
  const int S = (int)nd.nslot;    // gather sources per entry: two preloaded, the rest (amalgamated nodes) at gather time
  int ia[MF_PRE], ib[MF_PRE], ic[MF_PRE];
#pragma unroll
  for (int u = 0; u < MF_PRE; ++u) {
    const int j = threadIdx.x + u * MF_THREADS;
    ia[u] = ib[u] = ic[u] = -1;
    if (j < ns) {
      const int64_t p = nd.s0 + j;
      ia[u] = __ldg(perm + p);
      ib[u] = __ldg(src_t + S * p);
      ic[u] = __ldg(src_t + S * p + 1);
    } else if (j < ns + nb) {
      const int64_t q = nd.oo + (j - ns);
      ib[u] = __ldg(src_o + S * q);
      ic[u] = __ldg(src_o + S * q + 1);
    }
  }
  pdl_wait();
  pdl_trigger();
  auto gather = [&](int j, int pv, int a, int c) {
    if (j < ns) {
      double v = b[pv];
      if (a >= 0) v -= out[a];
      if (c >= 0) v -= out[c];
      const int* sp = src_t + S * (nd.s0 + j);
      for (int q = 2; q < S; ++q) {
        const int e = __ldg(sp + q);
        if (e >= 0) v -= out[e];
      }
      t[j] = v;
    } else {
      double v = 0.0;
      if (a >= 0) v += out[a];
      if (c >= 0) v += out[c];
      const int* sp = src_o + S * (nd.oo + (j - ns));
      for (int q = 2; q < S; ++q) {
        const int e = __ldg(sp + q);
        if (e >= 0) v += out[e];
      }
      pass[j - ns] = v;
    }
  };
#pragma unroll
  for (int u = 0; u < MF_PRE; ++u) {
    const int j = threadIdx.x + u * MF_THREADS;
    if (j < ns + nb) gather(j, ia[u], ib[u], ic[u]);
  }
  for (int j = threadIdx.x + MF_PRE * MF_THREADS; j < ns + nb; j += MF_THREADS) {
    if (j < ns) {
      const int64_t p = nd.s0 + j;
      gather(j, __ldg(perm + p), __ldg(src_t + S * p), __ldg(src_t + S * p + 1));
    } else {
      const int64_t q = nd.oo + (j - ns);
      gather(j, -1, __ldg(src_o + S * q), __ldg(src_o + S * q + 1));
    }
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  smem_rows(
      ns, ns, t,
      [&](int r, const double*& p, int& lo, int& hi) {
        p = F + r * (r + 1) / 2;
        lo = 0;
        hi = r + 1;
      },
      [&](int r, double v) {
        y[nd.s0 + r] = v;
        ys[r] = v;
      });
  __syncthreads();
  const double* W = F + npk(ns);
  smem_rows(
      nb, ns, ys,
      [&](int r, const double*& p, int& lo, int& hi) {
        p = W + r * ns;
        lo = 0;
        hi = ns;
      },
      [&](int r, double v) { out[nd.oo + r] = v + pass[r]; });
}

__global__ void __launch_bounds__(MF_THREADS)
    mf_backward_s(const int* __restrict__ level_nodes, const NodeRec* __restrict__ nodes,
                  const double* __restrict__ mats, const int* __restrict__ B,
                  const int* __restrict__ perm, const double* y, double* xp,
                  double* __restrict__ x, int blk_max, int max_ns) {
  extern __shared__ __align__(16) double sm[];
  __shared__ uint64_t bar;
  const NodeRec nd = nodes[level_nodes[blockIdx.x]];
  const int ns = (int)nd.ns, nb = (int)nd.nb;
  double* F = sm;
  double* s = sm + blk_max;
  int* ps = reinterpret_cast<int*>(s + max_ns);   // perm of the own rows
  double* xb = s + 2 * max_ns;
  if (threadIdx.x == 0) {
    const int len = even(npk(ns) + nb * ns);
    mbar_init(&bar, 1);
    fence_barrier_init();
    mbar_expect_tx(&bar, len * 8);
    if (len) bulk_g2s(F, mats + nd.oWT, len * 8, &bar);
  }
  int bi[MF_PRE];
  const int* Bp = B + nd.ob;
#pragma unroll
  for (int u = 0; u < MF_PRE; ++u) {
    const int j = threadIdx.x + u * MF_THREADS;
    bi[u] = j < nb ? __ldg(Bp + j) : 0;
  }
  for (int j = threadIdx.x; j < ns; j += MF_THREADS) ps[j] = __ldg(perm + nd.s0 + j);
  pdl_wait();
  pdl_trigger();
#pragma unroll
  for (int u = 0; u < MF_PRE; ++u) {
    const int j = threadIdx.x + u * MF_THREADS;
    if (j < nb) xb[j] = xp[bi[u]];
  }
  for (int j = threadIdx.x + MF_PRE * MF_THREADS; j < nb; j += MF_THREADS) xb[j] = xp[__ldg(Bp + j)];
  __syncthreads();
  mbar_wait(&bar, 0);
  smem_rows(
      ns, nb, xb,
      [&](int r, const double*& p, int& lo, int& hi) {
        p = F + r * nb;
        lo = 0;
        hi = nb;
      },
      [&](int r, double v) { s[r] = y[nd.s0 + r] - v; });
  __syncthreads();
  const double* LT = F + ns * nb;   // packed upper, row r holds columns r..ns-1
  smem_rows(
      ns, ns, s,
      [&](int r, const double*& p, int& lo, int& hi) {
        p = LT + upk_row(r, ns);
        lo = r;
        hi = ns;
      },
      [&](int r, double v) {
        xp[nd.s0 + r] = v;
        x[ps[r]] = v;
      });
}

// shared bytes of the staged kernels for a level (0: use the global variants)
static size_t mf_stage_smem(int max_ns, int max_nb, int& blk_max) {
  blk_max = even(npk(max_ns) + max_ns * max_nb);
  // forward [block | t : max_ns | ys : max_ns | pass : max_nb],
  // backward [block | s : max_ns | perm (ints) : max_ns | xb : max_nb]
  const size_t bytes = ((size_t)blk_max + 2 * (size_t)max_ns + max_nb) * sizeof(double);
  return bytes <= 224 * 1024 ? bytes : 0;   // of the 227 KB a CTA can have
}

}  // namespace mcs

using namespace mcs;

MCS_API int mcs_mf_forward(int nnodes, const int* level_nodes, const void* nodes,
                           const double* mats, const int* src_t, const int* src_o,
                           const int* perm, const double* b, double* y, double* out, int max_ns,
                           int max_nb, void* stream) {
  if (nnodes <= 0) return 0;
  auto st = static_cast<cudaStream_t>(stream);
  int blk_max = 0;
  const size_t staged = mf_stage_smem(max_ns, max_nb, blk_max);
  if (staged) {
    cudaFuncSetAttribute(mf_forward_s, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)staged);
    return launch_pdl_g(PDL_COARSE, mf_forward_s, nnodes, MF_THREADS, staged, st, level_nodes,
                        static_cast<const NodeRec*>(nodes), mats, src_t, src_o, perm, b, y, out,
                        blk_max, max_ns);
  }
  const size_t smem = (2 * (size_t)max_ns + max_nb) * sizeof(double);
  cudaFuncSetAttribute(mf_forward, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  return launch_pdl_g(PDL_COARSE, mf_forward, nnodes, MF_THREADS, smem, st, level_nodes,
                    static_cast<const NodeRec*>(nodes), mats, src_t, src_o, perm, b, y, out, max_ns);
}

MCS_API int mcs_mf_backward(int nnodes, const int* level_nodes, const void* nodes,
                            const double* mats, const int* B, const int* perm, const double* y,
                            double* xp, double* x, int max_ns, int max_nb, void* stream) {
  if (nnodes <= 0) return 0;
  auto st = static_cast<cudaStream_t>(stream);
  int blk_max = 0;
  const size_t staged = mf_stage_smem(max_ns, max_nb, blk_max);
  if (staged) {
    cudaFuncSetAttribute(mf_backward_s, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)staged);
    return launch_pdl_g(PDL_COARSE, mf_backward_s, nnodes, MF_THREADS, staged, st, level_nodes,
                        static_cast<const NodeRec*>(nodes), mats, B, perm, y, xp, x, blk_max,
                        max_ns);
  }
  const size_t smem = (2 * (size_t)max_ns + max_nb) * sizeof(double);
  cudaFuncSetAttribute(mf_backward, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  return launch_pdl_g(PDL_COARSE, mf_backward, nnodes, MF_THREADS, smem, st, level_nodes,
                    static_cast<const NodeRec*>(nodes), mats, B, perm, y, xp, x, max_ns);
}

// ---- top of the separator tree: dense explicit inverse of its Schur complement
namespace mcs {

// g[q] = b[perm[T[q]]] - sum_{p in src[ptr[q]..ptr[q+1])} out[p]   (fixed order)
__global__ void mf_top_gather(int t, const int* __restrict__ T, const int* __restrict__ perm,
                              const double* b, const int* __restrict__ ptr,
                              const int* __restrict__ src, const double* out,
                              double* __restrict__ g) {
  pdl_wait();
  pdl_trigger();
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= t) return;
  double v = b[perm[T[q]]];
  for (int k = ptr[q]; k < ptr[q + 1]; ++k) v -= out[src[k]];
  g[q] = v;
}

// x_T = Sinv g (dense t x ld, ld = t rounded up to 32, zero padded; g zero
// padded to ld): CTA per row, 16-byte loads.  The row's first TOP_NT x TOP_U
// pairs (the whole row for t <= 4096) are loaded before pdl_wait(): Sinv is
// static, so its fetch overlaps the gather kernel and the launch latency.
// The result goes to xp[T[r]] and x[perm[T[r]]].  Fixed-order reduction.
constexpr int TOP_NT = 256, TOP_U = 8;

__global__ void __launch_bounds__(TOP_NT)
    mf_top_solve(int ld2, const double2* __restrict__ Sinv, const double* g,
                 const int* __restrict__ T, const int* __restrict__ perm, double* __restrict__ xp,
                 double* __restrict__ x) {
  const int r = blockIdx.x;
  const double2* row = Sinv + (int64_t)r * ld2;
  const double2* g2 = reinterpret_cast<const double2*>(g);
  double2 a[TOP_U];
#pragma unroll
  for (int u = 0; u < TOP_U; ++u) {
    const int j = u * TOP_NT + threadIdx.x;
    a[u] = j < ld2 ? __ldg(row + j) : make_double2(0.0, 0.0);
  }
  pdl_wait();
  pdl_trigger();
  double s = 0.0;
  for (int base = 0;;) {
#pragma unroll
    for (int u = 0; u < TOP_U; ++u) {
      const int j = base + u * TOP_NT + threadIdx.x;
      if (j < ld2) {
        const double2 b = g2[j];
        s = fma(a[u].y, b.y, fma(a[u].x, b.x, s));
      }
    }
    base += TOP_NT * TOP_U;
    if (base >= ld2) break;
#pragma unroll
    for (int u = 0; u < TOP_U; ++u) {
      const int j = base + u * TOP_NT + threadIdx.x;
      a[u] = j < ld2 ? __ldg(row + j) : make_double2(0.0, 0.0);
    }
  }
  s = warp_sum(s);
  __shared__ double red[TOP_NT / 32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < TOP_NT / 32; ++w) v += red[w];
    xp[T[r]] = v;
    x[perm[T[r]]] = v;
  }
}

}  // namespace mcs

MCS_API int mcs_mf_top_ld(int t) { return (t + 31) / 32 * 32; }

MCS_API int mcs_mf_top(int t, const int* T, const int* perm, const double* b, const int* ptr,
                       const int* src, const double* out, double* g, const double* Sinv,
                       double* xp, double* x, void* stream) {
  if (t <= 0) return 0;
  auto st = static_cast<cudaStream_t>(stream);
  int rc = launch_pdl_g(PDL_COARSE, mf_top_gather, (t + 127) / 128, 128, 0, st, t, T, perm, b, ptr, src, out, g);
  if (rc) return rc;
  const int ld = mcs_mf_top_ld(t);
  return launch_pdl_g(PDL_COARSE, mf_top_solve, t, TOP_NT, 0, st, ld / 2,
                      reinterpret_cast<const double2*>(Sinv), static_cast<const double*>(g), T,
                      perm, xp, x);
}
