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
// HBM -> shared memory with a 1-D bulk async copy into a 2-stage per-warp ring
// so the next element streams in while the current one is multiplied.  Each
// lane owns rows l, l+32, ...; the symmetric packed entry (i, j) is read at
// pk(max, min) (triangular-number addressing is bank-conflict free for 32
// consecutive rows).  Scatter targets are free-dof indices with the sign in
// bit 0 (`code = 2*idx + neg`, -1 = constrained).  Every output dof receives
// at most two contributions, added with atomicAdd onto a zeroed vector:
// 0 + a + b == 0 + b + a exactly, so the result is bitwise deterministic.
#include "common.cuh"

namespace mcs {

constexpr int WARPS = 4;

struct WarpRing {
  uint64_t bar[2];
};

template <int N, int STRIDE>
__global__ void __launch_bounds__(WARPS * 32)
    elem_apply_kernel(const double* __restrict__ M, const int* __restrict__ codes,
                      const double* __restrict__ x, double* __restrict__ y, int64_t nt) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) WarpRing ring[WARPS];
  __shared__ double xs[WARPS][N];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* stage = sm + (size_t)warp * 2 * STRIDE;
  uint64_t* bar = ring[warp].bar;
  const int64_t gw = (int64_t)blockIdx.x * WARPS + warp;
  const int64_t nw = (int64_t)gridDim.x * WARPS;
  if (lane == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  __syncwarp();
  if (lane == 0) {
    for (int s = 0; s < 2; ++s) {
      const int64_t e = gw + s * nw;
      if (e < nt) {
        mbar_expect_tx(&bar[s], STRIDE * 8);
        bulk_g2s(stage + s * STRIDE, M + e * STRIDE, STRIDE * 8, &bar[s]);
      }
    }
  }
  int it = 0;
  for (int64_t e = gw; e < nt; e += nw, ++it) {
    const int s = it & 1;
    int cd[(N + 31) / 32];
#pragma unroll
    for (int r = 0; r < (N + 31) / 32; ++r) {
      const int j = lane + 32 * r;
      if (j < N) {
        const int c = codes[e * N + j];
        cd[r] = c;
        xs[warp][j] = c >= 0 ? code_sign(c) * x[code_index(c)] : 0.0;
      }
    }
    __syncwarp();
    mbar_wait(&bar[s], (it >> 1) & 1);
    const double* P = stage + s * STRIDE;
    constexpr int R = (N + 31) / 32;
    double acc[R];
    int rowb[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      acc[r] = 0.0;
      const int i = min(lane + 32 * r, N - 1);
      rowb[r] = pk(i, 0);
    }
#pragma unroll 2
    for (int j = 0; j < N; ++j) {
      const double xj = xs[warp][j];
      const int cb = pk(j, 0);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = min(lane + 32 * r, N - 1);
        acc[r] = fma(P[j <= i ? rowb[r] + j : cb + i], xj, acc[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = lane + 32 * r;
      if (i < N) {
        const int c = cd[r];
        if (c >= 0) atomicAdd(&y[code_index(c)], code_sign(c) * acc[r]);
      }
    }
    __syncwarp();
    const int64_t nxt = e + 2 * nw;
    if (lane == 0 && nxt < nt) {
      mbar_expect_tx(&bar[s], STRIDE * 8);
      bulk_g2s(stage + s * STRIDE, M + nxt * STRIDE, STRIDE * 8, &bar[s]);
    }
  }
}

// ExtendedAsp F1^-1 (restrict) and F2^-1 (prolong); ext record = [X | Soo^-1 packed]
template <int K, int LEN>
__global__ void __launch_bounds__(WARPS * 32)
    ext_restrict_kernel(const double* __restrict__ ext, const int* __restrict__ bidx,
                        const int* __restrict__ ccodes, const double* __restrict__ r,
                        double* __restrict__ bubble, double* __restrict__ acc, int64_t nt) {
  using Z = Sizes<K>;
  constexpr int NI = Z::n_int, NC = Z::ncpl, XL = NI * NC;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) WarpRing ring[WARPS];
  __shared__ double ro[WARPS][NI];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* stage = sm + (size_t)warp * 2 * LEN;
  uint64_t* bar = ring[warp].bar;
  const int64_t gw = (int64_t)blockIdx.x * WARPS + warp;
  const int64_t nw = (int64_t)gridDim.x * WARPS;
  if (lane == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  __syncwarp();
  if (lane == 0) {
    for (int s = 0; s < 2; ++s) {
      const int64_t e = gw + s * nw;
      if (e < nt) {
        mbar_expect_tx(&bar[s], LEN * 8);
        bulk_g2s(stage + s * LEN, ext + e * LEN, LEN * 8, &bar[s]);
      }
    }
  }
  int it = 0;
  for (int64_t e = gw; e < nt; e += nw, ++it) {
    const int s = it & 1;
    for (int j = lane; j < NI; j += 32) ro[warp][j] = r[bidx[e * NI + j]];
    __syncwarp();
    mbar_wait(&bar[s], (it >> 1) & 1);
    const double* X = stage + s * LEN;
    const double* Sinv = X + XL;
    for (int i = lane; i < NI; i += 32) {
      double a = 0.0;
      const int rowb = pk(i, 0);
      for (int j = 0; j < NI; ++j) a = fma(Sinv[j <= i ? rowb + j : pk(j, i)], ro[warp][j], a);
      bubble[e * NI + i] = a;
    }
    for (int c = lane; c < NC; c += 32) {
      double a = 0.0;
#pragma unroll 5
      for (int i = 0; i < NI; ++i) a = fma(X[i * NC + c], ro[warp][i], a);
      const int cd = ccodes[e * NC + c];
      if (cd >= 0) atomicAdd(&acc[code_index(cd)], code_sign(cd) * a);
    }
    __syncwarp();
    const int64_t nxt = e + 2 * nw;
    if (lane == 0 && nxt < nt) {
      mbar_expect_tx(&bar[s], LEN * 8);
      bulk_g2s(stage + s * LEN, ext + nxt * LEN, LEN * 8, &bar[s]);
    }
  }
}

template <int K, int LEN>
__global__ void __launch_bounds__(WARPS * 32)
    ext_prolong_kernel(const double* __restrict__ ext, const int* __restrict__ bidx,
                       const int* __restrict__ ccodes, const double* __restrict__ zc,
                       const double* __restrict__ bubble, double* __restrict__ out, int64_t nt) {
  using Z = Sizes<K>;
  constexpr int NI = Z::n_int, NC = Z::ncpl, XL = NI * NC;
  constexpr int XLE = even(XL);
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) WarpRing ring[WARPS];
  __shared__ double zl[WARPS][NC];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* stage = sm + (size_t)warp * 2 * XLE;
  uint64_t* bar = ring[warp].bar;
  const int64_t gw = (int64_t)blockIdx.x * WARPS + warp;
  const int64_t nw = (int64_t)gridDim.x * WARPS;
  if (lane == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  __syncwarp();
  if (lane == 0) {
    for (int s = 0; s < 2; ++s) {
      const int64_t e = gw + s * nw;
      if (e < nt) {
        mbar_expect_tx(&bar[s], XLE * 8);
        bulk_g2s(stage + s * XLE, ext + e * LEN, XLE * 8, &bar[s]);
      }
    }
  }
  int it = 0;
  for (int64_t e = gw; e < nt; e += nw, ++it) {
    const int s = it & 1;
    for (int c = lane; c < NC; c += 32) {
      const int cd = ccodes[e * NC + c];
      zl[warp][c] = cd >= 0 ? code_sign(cd) * zc[code_index(cd)] : 0.0;
    }
    __syncwarp();
    mbar_wait(&bar[s], (it >> 1) & 1);
    const double* X = stage + s * XLE;
    for (int i = lane; i < NI; i += 32) {
      double a = 0.0;
      for (int c = 0; c < NC; ++c) a = fma(X[i * NC + c], zl[warp][c], a);
      out[bidx[e * NI + i]] = bubble[e * NI + i] - a;
    }
    __syncwarp();
    const int64_t nxt = e + 2 * nw;
    if (lane == 0 && nxt < nt) {
      mbar_expect_tx(&bar[s], XLE * 8);
      bulk_g2s(stage + s * XLE, ext + nxt * LEN, XLE * 8, &bar[s]);
    }
  }
}

// w_c[j] = r[map[j]] - acc[j]
__global__ void gather_sub_kernel(const double* __restrict__ r, const int* __restrict__ map,
                                  const double* __restrict__ acc, double* __restrict__ w, int n) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
    w[j] = r[map[j]] - acc[j];
}

// out[map[j]] = z[j]
__global__ void scatter_kernel(const double* __restrict__ z, const int* __restrict__ map,
                               double* __restrict__ out, int n) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
    out[map[j]] = z[j];
}

static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

template <class Kern>
static int warp_grid(Kern k, size_t smem, int64_t nt) {
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, WARPS * 32, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t want = (nt + WARPS - 1) / WARPS;
  const int64_t g = (int64_t)per_sm * sm_count();
  return (int)(want < g ? want : g);
}

template <int N, int STRIDE>
static int launch_apply(const double* M, const int* codes, const double* x, double* y, int64_t nt,
                        cudaStream_t st) {
  auto kern = elem_apply_kernel<N, STRIDE>;
  const size_t smem = (size_t)WARPS * 2 * STRIDE * sizeof(double);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<warp_grid(kern, smem, nt), WARPS * 32, smem, st>>>(M, codes, x, y, nt);
  return launch_status();
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
  auto kern = ext_restrict_kernel<K, LEN>;
  const size_t smem = (size_t)WARPS * 2 * LEN * sizeof(double);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<warp_grid(kern, smem, nt), WARPS * 32, smem, st>>>(ext, bidx, cc, r, bubble, acc, nt);
  return launch_status();
}

template <int K>
static int launch_prolong(const double* ext, const int* bidx, const int* cc, const double* zc,
                          const double* bubble, double* out, int64_t nt, cudaStream_t st) {
  constexpr int LEN = ExtLen<K>::len;
  using Z = Sizes<K>;
  auto kern = ext_prolong_kernel<K, LEN>;
  const size_t smem = (size_t)WARPS * 2 * even(Z::n_int * Z::ncpl) * sizeof(double);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<warp_grid(kern, smem, nt), WARPS * 32, smem, st>>>(ext, bidx, cc, zc, bubble, out, nt);
  return launch_status();
}

}  // namespace mcs

using namespace mcs;

// which = 0: S (nloc, stride st_stride);  which = 1: S_d (ncpl, stride sd_stride)
MCS_API int mcs_apply_elem(int k, int which, int64_t nt, const double* M_packed, const int* codes,
                           const double* x, double* y, int64_t ny, void* stream) {
  auto st = static_cast<cudaStream_t>(stream);
  int rc = err_code(cudaMemsetAsync(y, 0, ny * sizeof(double), st));
  if (rc || nt <= 0) return rc;
#define MCS_APPLY_CASE(KK)                                                                 \
  case KK: {                                                                               \
    using Z = Sizes<KK>;                                                                   \
    if (which == 0) return launch_apply<Z::nloc, even(npk(Z::nloc))>(M_packed, codes, x, y, nt, st); \
    return launch_apply<Z::ncpl, even(npk(Z::ncpl))>(M_packed, codes, x, y, nt, st);      \
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
                            const double* zc, const double* bubble, double* out, void* stream) {
  auto st = static_cast<cudaStream_t>(stream);
  if (nt <= 0) return 0;
  switch (k) {
    case 2: return launch_prolong<2>(ext, bidx, ccodes, zc, bubble, out, nt, st);
    case 3: return launch_prolong<3>(ext, bidx, ccodes, zc, bubble, out, nt, st);
    case 4: return launch_prolong<4>(ext, bidx, ccodes, zc, bubble, out, nt, st);
    case 5: return launch_prolong<5>(ext, bidx, ccodes, zc, bubble, out, nt, st);
    case 6: return launch_prolong<6>(ext, bidx, ccodes, zc, bubble, out, nt, st);
  }
  return -1000;
}

MCS_API int mcs_gather_sub(int n, const double* r, const int* map, const double* acc, double* w,
                           void* stream) {
  if (n <= 0) return 0;
  auto st = static_cast<cudaStream_t>(stream);
  const int grid = (n + 255) / 256 < 4 * sm_count() ? (n + 255) / 256 : 4 * sm_count();
  gather_sub_kernel<<<grid, 256, 0, st>>>(r, map, acc, w, n);
  return launch_status();
}

MCS_API int mcs_scatter(int n, const double* z, const int* map, double* out, void* stream) {
  if (n <= 0) return 0;
  auto st = static_cast<cudaStream_t>(stream);
  const int grid = (n + 255) / 256 < 4 * sm_count() ? (n + 255) / 256 : 4 * sm_count();
  scatter_kernel<<<grid, 256, 0, st>>>(z, map, out, n);
  return launch_status();
}
