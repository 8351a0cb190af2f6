// Element-batched matrix-free operators of the PCG iteration.
//
//  A6  y = sum_T P_T^T D_T S_T D_T P_T x       (condensed operator S, and the
//      same kernel for S_d on coupling dofs; driver.py:138-144 applies the
//      assembled CSR instead)
//  A8  ExtendedAsp outer factors (preconditioners.py:353-378):
//      restrict:  bubble_T = S_oo^-1 r_o,   acc_c += X^T r_o   (signed scatter)
//      prolong:   out_o = bubble_T - X z_c
//
// One warp per element.  The element's packed matrix (or ext record) moves
// HBM -> shared memory with a 1-D bulk async copy into a per-warp stage ring
// (one stage at k = 4: measured best, see launch_apply) while the next
// element's indices and gathered values are prefetched into registers.  Each
// lane owns rows l, l+32, ...; the symmetric packed entry (i, j) is read at
// pk(max, min) (triangular-number addressing is bank-conflict free for 32
// consecutive rows).  Scatter targets are free-dof indices with the sign in
// bit 0 (`code = 2*idx + neg`, -1 = constrained).  Every output dof receives
// at most two contributions, added with atomicAdd onto a zeroed vector:
// 0 + a + b == 0 + b + a exactly, so the result is bitwise deterministic.
#include "common.cuh"

namespace mcs {

// Signed gather x_loc[j] = sign * x[idx] (0 for constrained dofs).
__device__ __forceinline__ double gather_signed(const double* x, int c) {
  return c >= 0 ? code_sign(c) * x[code_index(c)] : 0.0;   // x: produced upstream (no ld.nc)
}

// y = sum_T P^T D M_T D P x, warp per element, W warps per CTA, NST bulk-copy
// stages per warp.  The dof codes and x values of the next elements are
// prefetched into registers two / one element ahead, so neither the
// 1-D bulk copy of the packed matrix nor the dependent index -> x gather is
// on the per-element critical path.
template <int N, int STRIDE, int W, int NST>
__global__ void __launch_bounds__(W * 32)
    elem_apply_kernel(const double* __restrict__ M, const int* __restrict__ codes,
                      const double* x, double* __restrict__ y, int64_t nt,
                      double* __restrict__ dpart, unsigned* __restrict__ dcount,
                      double* __restrict__ dout) {
  constexpr int R = (N + 31) / 32;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bars[W][NST];
  __shared__ double xs[W][N];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* stage = sm + (size_t)warp * NST * STRIDE;
  uint64_t* bar = bars[warp];
  const int64_t gw = (int64_t)blockIdx.x * W + warp;
  const int64_t nw = (int64_t)gridDim.x * W;
  if (lane == 0) {
    for (int q = 0; q < NST; ++q) mbar_init(&bar[q], 1);
    fence_barrier_init();
  }
  __syncwarp();
  if (lane == 0) {
    for (int q = 0; q < NST; ++q) {
      const int64_t e = gw + q * nw;
      if (e < nt) {
        mbar_expect_tx(&bar[q], STRIDE * 8);
        bulk_g2s(stage + q * STRIDE, M + e * STRIDE, STRIDE * 8, &bar[q]);
      }
    }
  }
  // prefetch pipeline: codes of e and e+nw, x values of e
  int cd0[R], cd1[R];
  double xv[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int j = lane + 32 * r;
    const int64_t e0 = gw, e1 = gw + nw;
    cd0[r] = (j < N && e0 < nt) ? __ldg(codes + e0 * N + j) : -1;
    cd1[r] = (j < N && e1 < nt) ? __ldg(codes + e1 * N + j) : -1;
  }
  pdl_wait();   // static data (matrix bulk copies, codes) is in flight; x may now be read
  pdl_trigger();
#pragma unroll
  for (int r = 0; r < R; ++r) xv[r] = gather_signed(x, cd0[r]);
  int it = 0;
  double energy = 0.0;
  for (int64_t e = gw; e < nt; e += nw, ++it) {
    const int s = it % NST;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int j = lane + 32 * r;
      if (j < N) xs[warp][j] = xv[r];
    }
    int cd[R];
#pragma unroll
    for (int r = 0; r < R; ++r) cd[r] = cd0[r];
    // next element's x gather and the codes two ahead
    const int64_t e2 = e + 2 * nw;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int j = lane + 32 * r;
      xv[r] = gather_signed(x, cd1[r]);
      cd0[r] = cd1[r];
      cd1[r] = (j < N && e2 < nt) ? __ldg(codes + e2 * N + j) : -1;
    }
    __syncwarp();
    mbar_wait(&bar[s], (it / NST) & 1);
    const double* P = stage + s * STRIDE;
    // packed entry (i, j) sits at pk(i, 0) + j for j <= i and pk(j, 0) + i
    // for j > i: walked incrementally (+1 while j < i, then + j + 1)
    double acc[R];
    int ad[R], ir[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      acc[r] = 0.0;
      ir[r] = min(lane + 32 * r, N - 1);
      ad[r] = pk(ir[r], 0);
    }
#pragma unroll 2
    for (int j = 0; j < N; ++j) {
      const double xj = xs[warp][j];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        acc[r] = fma(P[ad[r]], xj, acc[r]);
        ad[r] += j < ir[r] ? 1 : j + 1;
      }
    }
    __syncwarp();
    const int64_t nxt = e + NST * nw;
    if (lane == 0 && nxt < nt) {
      mbar_expect_tx(&bar[s], STRIDE * 8);
      bulk_g2s(stage + s * STRIDE, M + nxt * STRIDE, STRIDE * 8, &bar[s]);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = lane + 32 * r;
      if (i < N && cd[r] >= 0) atomicAdd(&y[code_index(cd[r])], code_sign(cd[r]) * acc[r]);
      if (i < N) energy = fma(acc[r], xs[warp][i], energy);
    }
  }
  if (dout) {   // x . (A x) = sum_T x_T^T S_T x_T, fixed-order reduction
    __shared__ double wsum[W];
    __shared__ bool last;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) energy += __shfl_xor_sync(0xffffffffu, energy, o);
    if (lane == 0) wsum[warp] = energy;
    __syncthreads();
    if (threadIdx.x == 0) {
      double b = 0.0;
      for (int w = 0; w < W; ++w) b += wsum[w];
      dpart[blockIdx.x] = b;
      __threadfence();
      last = atomicAdd(dcount, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last && warp == 0) {
      __threadfence();
      double t = 0.0;
      for (int b = lane; b < (int)gridDim.x; b += 32) t += __ldcg(dpart + b);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (lane == 0) {
        *dout = t;
        *dcount = 0u;
      }
    }
  }
}

// ExtendedAsp F1^-1 (restrict) and F2^-1 (prolong); ext record = [X | Soo^-1 packed].
// Same pipeline as the apply: bulk-copied records, register prefetch of the
// next element's indices and gathered vector entries.
template <int K, int LEN, int W, int NST>
__global__ void __launch_bounds__(W * 32)
    ext_restrict_kernel(const double* __restrict__ ext, const int* __restrict__ bidx,
                        const int* __restrict__ ccodes, const double* r,
                        double* __restrict__ bubble, double* __restrict__ acc, int64_t nt) {
  using Z = Sizes<K>;
  constexpr int NI = Z::n_int, NC = Z::ncpl, XL = NI * NC;
  constexpr int RI = (NI + 31) / 32, RC = (NC + 31) / 32;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bars[W][NST];
  __shared__ double ro[W][NI];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* stage = sm + (size_t)warp * NST * LEN;
  uint64_t* bar = bars[warp];
  const int64_t gw = (int64_t)blockIdx.x * W + warp;
  const int64_t nw = (int64_t)gridDim.x * W;
  if (lane == 0) {
    for (int q = 0; q < NST; ++q) mbar_init(&bar[q], 1);
    fence_barrier_init();
  }
  __syncwarp();
  if (lane == 0) {
    for (int q = 0; q < NST; ++q) {
      const int64_t e = gw + q * nw;
      if (e < nt) {
        mbar_expect_tx(&bar[q], LEN * 8);
        bulk_g2s(stage + q * LEN, ext + e * LEN, LEN * 8, &bar[q]);
      }
    }
  }
  int b1[RI], cc0[RC];
  double rv[RI];
#pragma unroll
  for (int q = 0; q < RI; ++q) {
    const int j = lane + 32 * q;
    const int b0 = (j < NI && gw < nt) ? __ldg(bidx + gw * NI + j) : -1;
    rv[q] = (double)b0;   // index parked until r may be read
    b1[q] = (j < NI && gw + nw < nt) ? __ldg(bidx + (gw + nw) * NI + j) : -1;
  }
  pdl_wait();
  pdl_trigger();
#pragma unroll
  for (int q = 0; q < RI; ++q) {
    const int b0 = (int)rv[q];
    rv[q] = b0 >= 0 ? r[b0] : 0.0;
  }
#pragma unroll
  for (int q = 0; q < RC; ++q) {
    const int c = lane + 32 * q;
    cc0[q] = (c < NC && gw < nt) ? __ldg(ccodes + gw * NC + c) : -1;
  }
  int it = 0;
  for (int64_t e = gw; e < nt; e += nw, ++it) {
    const int s = it % NST;
#pragma unroll
    for (int q = 0; q < RI; ++q) {
      const int j = lane + 32 * q;
      if (j < NI) ro[warp][j] = rv[q];
    }
    int cd[RC];
#pragma unroll
    for (int q = 0; q < RC; ++q) cd[q] = cc0[q];
    const int64_t e1 = e + nw, e2 = e + 2 * nw;
#pragma unroll
    for (int q = 0; q < RI; ++q) {
      const int j = lane + 32 * q;
      rv[q] = b1[q] >= 0 ? r[b1[q]] : 0.0;
      b1[q] = (j < NI && e2 < nt) ? __ldg(bidx + e2 * NI + j) : -1;
    }
#pragma unroll
    for (int q = 0; q < RC; ++q) {
      const int c = lane + 32 * q;
      cc0[q] = (c < NC && e1 < nt) ? __ldg(ccodes + e1 * NC + c) : -1;
    }
    __syncwarp();
    mbar_wait(&bar[s], (it / NST) & 1);
    const double* X = stage + s * LEN;
    const double* Sinv = X + XL;
    double a[RI];
    int ad[RI], ir[RI];
#pragma unroll
    for (int q = 0; q < RI; ++q) {
      a[q] = 0.0;
      ir[q] = min(lane + 32 * q, NI - 1);
      ad[q] = pk(ir[q], 0);
    }
#pragma unroll 2
    for (int j = 0; j < NI; ++j) {   // packed walk as in elem_apply_kernel
      const double xj = ro[warp][j];
#pragma unroll
      for (int q = 0; q < RI; ++q) {
        a[q] = fma(Sinv[ad[q]], xj, a[q]);
        ad[q] += j < ir[q] ? 1 : j + 1;
      }
    }
    double c[RC];
#pragma unroll
    for (int q = 0; q < RC; ++q) c[q] = 0.0;
#pragma unroll 5
    for (int i = 0; i < NI; ++i) {
      const double xi = ro[warp][i];
#pragma unroll
      for (int q = 0; q < RC; ++q) c[q] = fma(X[i * NC + min(lane + 32 * q, NC - 1)], xi, c[q]);
    }
    __syncwarp();
    const int64_t nxt = e + NST * nw;
    if (lane == 0 && nxt < nt) {
      mbar_expect_tx(&bar[s], LEN * 8);
      bulk_g2s(stage + s * LEN, ext + nxt * LEN, LEN * 8, &bar[s]);
    }
#pragma unroll
    for (int q = 0; q < RI; ++q) {
      const int i = lane + 32 * q;
      if (i < NI) bubble[e * NI + i] = a[q];
    }
#pragma unroll
    for (int q = 0; q < RC; ++q) {
      const int cc = lane + 32 * q;
      if (cc < NC && cd[q] >= 0) atomicAdd(&acc[code_index(cd[q])], code_sign(cd[q]) * c[q]);
    }
  }
}

template <int K, int LEN, int W, int NST>
__global__ void __launch_bounds__(W * 32)
    ext_prolong_kernel(const double* __restrict__ ext, const int* __restrict__ bidx,
                       const int* __restrict__ ccodes, const double* zc,
                       const double* bubble, const int* __restrict__ c2v,
                       double* __restrict__ out, int64_t nt) {
  using Z = Sizes<K>;
  constexpr int NI = Z::n_int, NC = Z::ncpl, XL = NI * NC;
  constexpr int XLE = even(XL);
  constexpr int RI = (NI + 31) / 32, RC = (NC + 31) / 32;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bars[W][NST];
  __shared__ double zl[W][NC];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* stage = sm + (size_t)warp * NST * XLE;
  uint64_t* bar = bars[warp];
  const int64_t gw = (int64_t)blockIdx.x * W + warp;
  const int64_t nw = (int64_t)gridDim.x * W;
  if (lane == 0) {
    for (int q = 0; q < NST; ++q) mbar_init(&bar[q], 1);
    fence_barrier_init();
  }
  __syncwarp();
  if (lane == 0) {
    for (int q = 0; q < NST; ++q) {
      const int64_t e = gw + q * nw;
      if (e < nt) {
        mbar_expect_tx(&bar[q], XLE * 8);
        bulk_g2s(stage + q * XLE, ext + e * LEN, XLE * 8, &bar[q]);
      }
    }
  }
  int c0[RC], c1[RC];
  double zv[RC];
#pragma unroll
  for (int q = 0; q < RC; ++q) {
    const int c = lane + 32 * q;
    c0[q] = (c < NC && gw < nt) ? __ldg(ccodes + gw * NC + c) : -1;
    c1[q] = (c < NC && gw + nw < nt) ? __ldg(ccodes + (gw + nw) * NC + c) : -1;
  }
  // static indices of the first element before the wait: bubble targets
  // and the scatter targets of the coupling dofs
  int bin[RI], cvn[RC];
#pragma unroll
  for (int q = 0; q < RI; ++q) {
    const int i = lane + 32 * q;
    bin[q] = (i < NI && gw < nt) ? __ldg(bidx + gw * NI + i) : 0;
  }
#pragma unroll
  for (int q = 0; q < RC; ++q) cvn[q] = c0[q] >= 0 ? __ldg(c2v + code_index(c0[q])) : 0;
  pdl_wait();
  pdl_trigger();
  double bubn[RI];
#pragma unroll
  for (int q = 0; q < RC; ++q) zv[q] = gather_signed(zc, c0[q]);
#pragma unroll
  for (int q = 0; q < RI; ++q) {
    const int i = lane + 32 * q;
    bubn[q] = (i < NI && gw < nt) ? bubble[gw * NI + i] : 0.0;
  }
  int it = 0;
  for (int64_t e = gw; e < nt; e += nw, ++it) {
    const int s = it % NST;
    double bub[RI];
    int bi[RI];
#pragma unroll
    for (int q = 0; q < RI; ++q) {
      bub[q] = bubn[q];
      bi[q] = bin[q];
    }
#pragma unroll
    for (int q = 0; q < RC; ++q) {
      const int c = lane + 32 * q;
      if (c < NC) zl[warp][c] = zv[q];
      // the coupling part of out = z_c (the ExtendedAsp scatter, fused):
      // a dof shared by two elements receives the same value twice
      if (c0[q] >= 0) out[cvn[q]] = code_sign(c0[q]) * zv[q];
    }
    // next element's gathers, bubble entries and indices one element ahead
    const int64_t e1 = e + nw, e2 = e + 2 * nw;
#pragma unroll
    for (int q = 0; q < RC; ++q) {
      const int c = lane + 32 * q;
      zv[q] = gather_signed(zc, c1[q]);
      cvn[q] = c1[q] >= 0 ? __ldg(c2v + code_index(c1[q])) : 0;
      c0[q] = c1[q];
      c1[q] = (c < NC && e2 < nt) ? __ldg(ccodes + e2 * NC + c) : -1;
    }
#pragma unroll
    for (int q = 0; q < RI; ++q) {
      const int i = lane + 32 * q;
      bubn[q] = (i < NI && e1 < nt) ? bubble[e1 * NI + i] : 0.0;
      bin[q] = (i < NI && e1 < nt) ? __ldg(bidx + e1 * NI + i) : 0;
    }
    __syncwarp();
    mbar_wait(&bar[s], (it / NST) & 1);
    const double* X = stage + s * XLE;
    double a[RI];
#pragma unroll
    for (int q = 0; q < RI; ++q) a[q] = 0.0;
#pragma unroll 3
    for (int c = 0; c < NC; ++c) {
      const double zcv = zl[warp][c];
#pragma unroll
      for (int q = 0; q < RI; ++q) a[q] = fma(X[min(lane + 32 * q, NI - 1) * NC + c], zcv, a[q]);
    }
    __syncwarp();
    const int64_t nxt = e + NST * nw;
    if (lane == 0 && nxt < nt) {
      mbar_expect_tx(&bar[s], XLE * 8);
      bulk_g2s(stage + s * XLE, ext + nxt * LEN, XLE * 8, &bar[s]);
    }
#pragma unroll
    for (int q = 0; q < RI; ++q) {
      const int i = lane + 32 * q;
      if (i < NI) out[bi[q]] = bub[q] - a[q];
    }
  }
}

// w_c[j] = r[map[j]] - acc[j]
__global__ void gather_sub_kernel(const double* r, const int* __restrict__ map,
                                  const double* acc, double* __restrict__ w, int n) {
  pdl_wait();
  pdl_trigger();
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
    w[j] = r[map[j]] - acc[j];
}

// out[map[j]] = z[j]
__global__ void scatter_kernel(const double* z, const int* __restrict__ map,
                               double* __restrict__ out, int n) {
  pdl_wait();
  pdl_trigger();
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
    out[map[j]] = z[j];
}


template <int N, int STRIDE>
static int launch_apply(const double* M, const int* codes, const double* x, double* y, int64_t nt,
                        double* dpart, unsigned* dcount, double* dout, cudaStream_t st) {
  // one bulk stage per warp when a stage is large (k = 5, 6), two otherwise;
  // aim for ~64-96 KB of bulk copies in flight per SM
  // measured on B200 (tools/apply_variants.cu): warps in flight matter more
  // than per-warp ring depth; one stage per warp, 8 warps, fills the SM
  // (3 CTAs/SM at k = 4: 66% of HBM; k = 6: 69%).  A CTA-wide ring with one
  // producer thread and 16 consumer warps (28 records in flight per SM) was
  // measured slower (62.5 vs 58.4 us at cfg2); so was 2-stage x 4 warps.
  constexpr int W = 8;
  constexpr int NST = 1;
  auto kern = elem_apply_kernel<N, STRIDE, W, NST>;
  const size_t smem = (size_t)W * NST * STRIDE * sizeof(double);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, W * 32, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t want = (nt + W - 1) / W;
  int64_t g = (int64_t)per_sm * sm_count();
  // the fused p'Ap writes one partial per CTA: stay inside the workspace
  // (mcs_reduce_workspace_len; the grid-stride loop covers the rest)
  if (dpart && g > mcs_reduce_workspace_len()) g = mcs_reduce_workspace_len();
  return launch_pdl_g(PDL_APPLY, kern, (int)(want < g ? want : g), W * 32, smem, st, M, codes, x, y, nt,
                      dpart, dcount, dout);
}

template <int K>
struct ExtLen {
  using Z = Sizes<K>;
  static constexpr int len = even(Z::n_int * Z::ncpl + npk(Z::n_int));
};

template <int K>
static int launch_restrict(const double* ext, const int* bidx, const int* cc, const double* r,
                           double* bubble, double* acc, int64_t nt, cudaStream_t st) {
  constexpr int LEN = ExtLen<K>::len;
  constexpr int W = 8, NST = 1;
  auto kern = ext_restrict_kernel<K, LEN, W, NST>;
  const size_t smem = (size_t)W * NST * LEN * sizeof(double);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, W * 32, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t want = (nt + W - 1) / W, g = (int64_t)per_sm * sm_count();
  return launch_pdl_g(PDL_ELEM, kern, (int)(want < g ? want : g), W * 32, smem, st, ext, bidx, cc, r, bubble,
                    acc, nt);
}

template <int K>
static int launch_prolong(const double* ext, const int* bidx, const int* cc, const double* zc,
                          const double* bubble, const int* c2v, double* out, int64_t nt,
                          cudaStream_t st) {
  constexpr int LEN = ExtLen<K>::len;
  using Z = Sizes<K>;
  constexpr int XLE = even(Z::n_int * Z::ncpl);
  constexpr int W = 8, NST = 1;
  auto kern = ext_prolong_kernel<K, LEN, W, NST>;
  const size_t smem = (size_t)W * NST * XLE * sizeof(double);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, W * 32, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t want = (nt + W - 1) / W, g = (int64_t)per_sm * sm_count();
  return launch_pdl_g(PDL_ELEM, kern, (int)(want < g ? want : g), W * 32, smem, st, ext, bidx, cc, zc, bubble,
                    c2v, out, nt);
}

}  // namespace mcs

using namespace mcs;

static int apply_elem(int k, int which, int64_t nt, const double* M_packed, const int* codes,
                      const double* x, double* y, int64_t ny, double* dpart, unsigned* dcount,
                      double* dout, cudaStream_t st) {
  int rc = err_code(cudaMemsetAsync(y, 0, ny * sizeof(double), st));
  if (rc || nt <= 0) return rc;
#define MCS_APPLY_CASE(KK)                                                                  \
  case KK: {                                                                                \
    using Z = Sizes<KK>;                                                                    \
    if (which == 0)                                                                         \
      return launch_apply<Z::nloc, even(npk(Z::nloc))>(M_packed, codes, x, y, nt, dpart,    \
                                                       dcount, dout, st);                   \
    return launch_apply<Z::ncpl, even(npk(Z::ncpl))>(M_packed, codes, x, y, nt, dpart,      \
                                                     dcount, dout, st);                     \
  }
  switch (k) {
    MCS_APPLY_CASE(2)
    MCS_APPLY_CASE(3)
    MCS_APPLY_CASE(4)
    MCS_APPLY_CASE(5)
    MCS_APPLY_CASE(6)
  }
#undef MCS_APPLY_CASE
  return -1000;
}

// which = 0: S (nloc, stride st_stride);  which = 1: S_d (ncpl, stride sd_stride)
MCS_API int mcs_apply_elem(int k, int which, int64_t nt, const double* M_packed, const int* codes,
                           const double* x, double* y, int64_t ny, void* stream) {
  return apply_elem(k, which, nt, M_packed, codes, x, y, ny, nullptr, nullptr, nullptr,
                    static_cast<cudaStream_t>(stream));
}

// the same apply, plus *out = x . y = sum_T x_T^T M_T x_T (deterministic)
MCS_API int mcs_apply_elem_dot(int k, int which, int64_t nt, const double* M_packed,
                               const int* codes, const double* x, double* y, int64_t ny,
                               double* partials, unsigned* counter, double* out, void* stream) {
  return apply_elem(k, which, nt, M_packed, codes, x, y, ny, partials, counter, out,
                    static_cast<cudaStream_t>(stream));
}

MCS_API int mcs_ext_restrict(int k, int64_t nt, const double* ext, const int* bidx, const int* ccodes,
                             const double* r, double* bubble, double* acc, int64_t nacc,
                             void* stream) {
  auto st = static_cast<cudaStream_t>(stream);
  int rc = err_code(cudaMemsetAsync(acc, 0, nacc * sizeof(double), st));
  if (rc || nt <= 0) return rc;
  switch (k) {
    case 2: return launch_restrict<2>(ext, bidx, ccodes, r, bubble, acc, nt, st);
    case 3: return launch_restrict<3>(ext, bidx, ccodes, r, bubble, acc, nt, st);
    case 4: return launch_restrict<4>(ext, bidx, ccodes, r, bubble, acc, nt, st);
    case 5: return launch_restrict<5>(ext, bidx, ccodes, r, bubble, acc, nt, st);
    case 6: return launch_restrict<6>(ext, bidx, ccodes, r, bubble, acc, nt, st);
  }
  return -1000;
}

MCS_API int mcs_ext_prolong(int k, int64_t nt, const double* ext, const int* bidx, const int* ccodes,
                            const double* zc, const double* bubble, const int* c2v, double* out,
                            void* stream) {
  auto st = static_cast<cudaStream_t>(stream);
  if (nt <= 0) return 0;
  switch (k) {
    case 2: return launch_prolong<2>(ext, bidx, ccodes, zc, bubble, c2v, out, nt, st);
    case 3: return launch_prolong<3>(ext, bidx, ccodes, zc, bubble, c2v, out, nt, st);
    case 4: return launch_prolong<4>(ext, bidx, ccodes, zc, bubble, c2v, out, nt, st);
    case 5: return launch_prolong<5>(ext, bidx, ccodes, zc, bubble, c2v, out, nt, st);
    case 6: return launch_prolong<6>(ext, bidx, ccodes, zc, bubble, c2v, out, nt, st);
  }
  return -1000;
}

MCS_API int mcs_gather_sub(int n, const double* r, const int* map, const double* acc, double* w,
                           void* stream) {
  if (n <= 0) return 0;
  auto st = static_cast<cudaStream_t>(stream);
  const int grid = (n + 255) / 256 < 4 * sm_count() ? (n + 255) / 256 : 4 * sm_count();
  return launch_pdl_g(PDL_ELEM, gather_sub_kernel, grid, 256, 0, st, r, map, acc, w, n);
}

MCS_API int mcs_scatter(int n, const double* z, const int* map, double* out, void* stream) {
  if (n <= 0) return 0;
  auto st = static_cast<cudaStream_t>(stream);
  const int grid = (n + 255) / 256 < 4 * sm_count() ? (n + 255) / 256 : 4 * sm_count();
  return launch_pdl_g(PDL_ELEM, scatter_kernel, grid, 256, 0, st, z, map, out, n);
}
