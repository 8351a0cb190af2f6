// Per-element static condensation on B200.
//
// One CTA owns one element at a time (persistent over elements).  The
// element's symmetric augmented saddle matrix lives in REGISTERS: the lower
// triangle is cut into TBxTB tiles, one tile per thread, and eliminated
// right-looking without pivoting.  Each pivot step broadcasts the current
// pivot column through shared memory (double buffered, one __syncthreads per
// pivot) and every thread applies the rank-1 update to its register tile
// with TB*TB DFMAs against 2*TB shared-memory (broadcast) loads.
//
//   microbench (A5):   K = [[A, B], [B^T, 0]]  -> eliminate the n_s (positive)
//                      pivots -> trailing block = -B^T A^-1 B = -S
//   MCS (A3):          K = [[msig, bws^T, Bsig^T], [bws, 0, 0], [Bsig, 0, -adiv]]
//                      -> n_s positive then n_w negative pivots -> trailing
//                      block = -S_T, the reference's S_T of
//                      condensation.py:161-176 (LU of [[-msig, bws^T],
//                      [bws, 0]] then adiv - Bsig M^-1 Bsig^T), proved equal in
//                      DESIGN.md §3.
//
// The next element's input is prefetched into shared memory with one 1-D
// bulk async copy (TMA engine, cp.async.bulk + mbarrier) issued as soon as
// the current element's tiles are in registers, so HBM traffic overlaps the
// FP64 elimination of the current element.
#include "common.cuh"

namespace mcs {

template <int N, int TB>
struct Grid2 {
  static constexpr int NB = (N + TB - 1) / TB;
  static constexpr int NT = NB * (NB + 1) / 2;
  static constexpr int THREADS = (NT + 31) / 32 * 32;
  static constexpr int NPAD = NB * TB;
};

__device__ __forceinline__ void tile_of(int t, int& bi, int& bj) {
  int i = 0;
  while ((i + 1) * (i + 2) / 2 <= t) ++i;
  bi = i;
  bj = t - i * (i + 1) / 2;
}

// Eliminate pivots [P0, P1); pivots < PSIGN must be > 0, the rest < 0.
// Records the first offending pivot (1-based) in *bad (shared).
template <int N, int TB, int P0, int P1, int PSIGN>
__device__ __forceinline__ void eliminate(double (&a)[TB][TB], int bi, int bj, bool act,
                                          double (*col)[Grid2<N, TB>::NPAD], int* bad) {
  for (int pb = P0 / TB; pb <= (P1 - 1) / TB; ++pb) {
#pragma unroll
    for (int cj = 0; cj < TB; ++cj) {
      const int j = pb * TB + cj;
      if (j < P0 || j >= P1) continue;
      double* cb = col[j & 1];
      if (act && bj == pb) {
#pragma unroll
        for (int r = 0; r < TB; ++r) cb[bi * TB + r] = a[r][cj];
      }
      __syncthreads();
      const double d = cb[j];
      if (threadIdx.x == 0) {
        const bool ok = (j < PSIGN) ? (d > 0.0) : (d < 0.0);
        if (!ok && *bad == 0) *bad = j + 1;
      }
      if (act && bj >= pb) {
        const double inv = 1.0 / d;
        double li[TB], lc[TB];
        const double2* rp = reinterpret_cast<const double2*>(cb + bi * TB);
        const double2* cp = reinterpret_cast<const double2*>(cb + bj * TB);
#pragma unroll
        for (int r = 0; r < TB / 2; ++r) {
          double2 v = rp[r];
          li[2 * r] = v.x * inv;
          li[2 * r + 1] = v.y * inv;
          double2 w = cp[r];
          lc[2 * r] = w.x;
          lc[2 * r + 1] = w.y;
        }
        if (bj > pb) {
#pragma unroll
          for (int r = 0; r < TB; ++r)
#pragma unroll
            for (int c = 0; c < TB; ++c) a[r][c] = fma(-li[r], lc[c], a[r][c]);
        } else {
#pragma unroll
          for (int r = 0; r < TB; ++r)
#pragma unroll
            for (int c = cj + 1; c < TB; ++c) a[r][c] = fma(-li[r], lc[c], a[r][c]);
        }
      }
    }
  }
}

// --------------------------------------------------------------- A5: microbench

template <int NS, int NC, int TB>
__global__ void __launch_bounds__(Grid2<NS + NC, TB>::THREADS)
    spd_schur_kernel(const double* __restrict__ A, const double* __restrict__ B,
                     double* __restrict__ S, int* __restrict__ info, int64_t batch) {
  constexpr int N = NS + NC;
  using G = Grid2<N, TB>;
  constexpr int LA = npk(NS), LB = NS * NC, LS = npk(NC);
  static_assert((LA % 2) == 0 && (LB % 2) == 0, "16-byte bulk copies");
  extern __shared__ __align__(128) double smem[];
  double* sA = smem;
  double* sB = smem + LA;
  __shared__ __align__(16) double col[2][G::NPAD];
  __shared__ __align__(8) uint64_t bar;
  __shared__ int bad;

  int bi = 0, bj = 0;
  const bool act = threadIdx.x < G::NT;
  if (act) tile_of(threadIdx.x, bi, bj);

  int64_t e = blockIdx.x;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0 && e < batch) {
    mbar_expect_tx(&bar, (LA + LB) * 8);
    bulk_g2s(sA, A + e * LA, LA * 8, &bar);
    bulk_g2s(sB, B + e * LB, LB * 8, &bar);
  }
  uint32_t phase = 0;
  for (; e < batch; e += gridDim.x) {
    mbar_wait(&bar, phase);
    phase ^= 1;
    double a[TB][TB];
#pragma unroll
    for (int r = 0; r < TB; ++r)
#pragma unroll
      for (int c = 0; c < TB; ++c) {
        const int i = bi * TB + r, j = bj * TB + c;
        double v = 0.0;
        if (act && i < N && j <= i) {
          if (i < NS) v = sA[pk(i, j)];
          else if (j < NS) v = sB[j * NC + (i - NS)];
        }
        a[r][c] = v;
      }
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    const int64_t nxt = e + gridDim.x;
    if (threadIdx.x == 0 && nxt < batch) {   // prefetch the next element
      mbar_expect_tx(&bar, (LA + LB) * 8);
      bulk_g2s(sA, A + nxt * LA, LA * 8, &bar);
      bulk_g2s(sB, B + nxt * LB, LB * 8, &bar);
    }
    eliminate<N, TB, 0, NS, NS>(a, bi, bj, act, col, &bad);
    // trailing block holds -S
    double* out = S + e * LS;
#pragma unroll
    for (int r = 0; r < TB; ++r)
#pragma unroll
      for (int c = 0; c < TB; ++c) {
        const int i = bi * TB + r, j = bj * TB + c;
        if (act && i < N && j >= NS && j <= i) out[pk(i - NS, j - NS)] = -a[r][c];
      }
    __syncthreads();
    if (threadIdx.x == 0 && info) info[e] = bad;
  }
}

// ------------------------------------------------------- A3: MCS condensation

// element record: [msig ns*ns | bws nw*ns | bus nu*ns | bhs nh*ns | adiv nu*nu],
// every segment padded to an even number of doubles (16-byte bulk copies)
template <int K>
struct Record {
  using Z = Sizes<K>;
  static constexpr int o_msig = 0;
  static constexpr int o_bws = even(Z::ns * Z::ns);
  static constexpr int o_bus = o_bws + even(Z::nw * Z::ns);
  static constexpr int o_bhs = o_bus + even(Z::nu * Z::ns);
  static constexpr int o_adiv = o_bhs + even(Z::nh * Z::ns);
  static constexpr int len = o_adiv + even(Z::nu * Z::nu);
  static constexpr int st_len = even(npk(Z::nloc));   // packed S_T stride
};

template <int K>
__device__ __forceinline__ double mcs_entry(const double* rec, int i, int j) {
  using Z = Sizes<K>;
  using R = Record<K>;
  constexpr int ns = Z::ns, nw = Z::nw, nu = Z::nu, c0 = Z::ns + Z::nw;
  if (i < ns) return rec[R::o_msig + i * ns + j];
  if (i < c0) return j < ns ? rec[R::o_bws + (i - ns) * ns + j] : 0.0;
  const int l = i - c0;
  if (j < ns) return l < nu ? rec[R::o_bus + l * ns + j] : rec[R::o_bhs + (l - nu) * ns + j];
  if (j < c0) return 0.0;
  const int m = j - c0;
  return (l < nu && m < nu) ? -rec[R::o_adiv + l * nu + m] : 0.0;
}

template <int K, int TB>
__global__ void __launch_bounds__(Grid2<Sizes<K>::naug, TB>::THREADS)
    condense_kernel(const double* __restrict__ recs, double* __restrict__ ST,
                    int* __restrict__ info, int64_t nt) {
  using Z = Sizes<K>;
  using R = Record<K>;
  constexpr int N = Z::naug, NP = Z::ns + Z::nw;
  using G = Grid2<N, TB>;
  extern __shared__ __align__(128) double srec[];
  __shared__ __align__(16) double col[2][G::NPAD];
  __shared__ __align__(8) uint64_t bar;
  __shared__ int bad;

  int bi = 0, bj = 0;
  const bool act = threadIdx.x < G::NT;
  if (act) tile_of(threadIdx.x, bi, bj);
  int64_t e = blockIdx.x;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0 && e < nt) {
    mbar_expect_tx(&bar, R::len * 8);
    bulk_g2s(srec, recs + e * R::len, R::len * 8, &bar);
  }
  uint32_t phase = 0;
  for (; e < nt; e += gridDim.x) {
    mbar_wait(&bar, phase);
    phase ^= 1;
    double a[TB][TB];
#pragma unroll
    for (int r = 0; r < TB; ++r)
#pragma unroll
      for (int c = 0; c < TB; ++c) {
        const int i = bi * TB + r, j = bj * TB + c;
        a[r][c] = (act && i < N && j <= i) ? mcs_entry<K>(srec, i, j) : 0.0;
      }
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    const int64_t nxt = e + gridDim.x;
    if (threadIdx.x == 0 && nxt < nt) {
      mbar_expect_tx(&bar, R::len * 8);
      bulk_g2s(srec, recs + nxt * R::len, R::len * 8, &bar);
    }
    eliminate<N, TB, 0, NP, Z::ns>(a, bi, bj, act, col, &bad);
    double* out = ST + e * R::st_len;
#pragma unroll
    for (int r = 0; r < TB; ++r)
#pragma unroll
      for (int c = 0; c < TB; ++c) {
        const int i = bi * TB + r, j = bj * TB + c;
        if (act && i < N && j >= NP && j <= i) out[pk(i - NP, j - NP)] = -a[r][c];
      }
    __syncthreads();
    if (threadIdx.x == 0 && info) info[e] = bad;
  }
}

// ---------------------------------------------- A1: element blocks on the GPU
// rec[e][q] = sum_{p in prog[q]} W[e][widx[p]] * coef[p]   (refblocks.py)
__global__ void element_blocks_kernel(const double* __restrict__ W, int nwgt,
                                      const int* __restrict__ ptr, const int* __restrict__ widx,
                                      const double* __restrict__ coef, int reclen,
                                      double* __restrict__ recs, int64_t nt) {
  extern __shared__ double sw[];
  for (int64_t e = blockIdx.x; e < nt; e += gridDim.x) {
    for (int r = threadIdx.x; r < nwgt; r += blockDim.x) sw[r] = W[e * nwgt + r];
    __syncthreads();
    for (int q = threadIdx.x; q < reclen; q += blockDim.x) {
      double s = 0.0;
      for (int p = ptr[q]; p < ptr[q + 1]; ++p) s = fma(sw[widx[p]], coef[p], s);
      recs[e * reclen + q] = s;
    }
    __syncthreads();
  }
}

static int g_num_sms = 0;
static int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return g_num_sms;
}

template <class Kern>
static int persistent_grid(Kern k, int threads, size_t smem, int64_t n) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, threads, smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  int64_t g = static_cast<int64_t>(per_sm) * num_sms();
  return static_cast<int>(n < g ? n : g);
}

template <int NS, int NC, int TB>
static int launch_spd_schur(const double* A, const double* B, double* S, int* info, int64_t batch,
                            cudaStream_t st) {
  using G = Grid2<NS + NC, TB>;
  auto kern = spd_schur_kernel<NS, NC, TB>;
  const size_t smem = (npk(NS) + NS * NC) * sizeof(double);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = persistent_grid(kern, G::THREADS, smem, batch);
  kern<<<grid, G::THREADS, smem, st>>>(A, B, S, info, batch);
  return launch_status();
}

template <int K, int TB>
static int launch_condense(const double* recs, double* ST, int* info, int64_t nt, cudaStream_t st) {
  using G = Grid2<Sizes<K>::naug, TB>;
  auto kern = condense_kernel<K, TB>;
  const size_t smem = Record<K>::len * sizeof(double);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = persistent_grid(kern, G::THREADS, smem, nt);
  kern<<<grid, G::THREADS, smem, st>>>(recs, ST, info, nt);
  return launch_status();
}

}  // namespace mcs

using namespace mcs;

MCS_API int mcs_spd_schur_batched(int n, int m, int64_t batch, const double* A_packed_lower,
                                  const double* B, double* S_packed, int* info, void* stream) {
  if (batch <= 0) return 0;
  auto st = static_cast<cudaStream_t>(stream);
  if (n == 60 && m == 36) return launch_spd_schur<60, 36, 8>(A_packed_lower, B, S_packed, info, batch, st);
  if (n == 8 && m == 4) return launch_spd_schur<8, 4, 4>(A_packed_lower, B, S_packed, info, batch, st);
  return -1000;  // unsupported shape (compiled instantiations only)
}

MCS_API int mcs_record_len(int k) {
  switch (k) {
    case 2: return Record<2>::len;
    case 3: return Record<3>::len;
    case 4: return Record<4>::len;
    case 5: return Record<5>::len;
    case 6: return Record<6>::len;
  }
  return -1;
}

MCS_API int mcs_st_stride(int k) {
  switch (k) {
    case 2: return Record<2>::st_len;
    case 3: return Record<3>::st_len;
    case 4: return Record<4>::st_len;
    case 5: return Record<5>::st_len;
    case 6: return Record<6>::st_len;
  }
  return -1;
}

MCS_API int mcs_condense(int k, int64_t nt, const double* records, double* S_packed, int* info,
                         void* stream) {
  if (nt <= 0) return 0;
  auto st = static_cast<cudaStream_t>(stream);
  switch (k) {
    case 2: return launch_condense<2, 4>(records, S_packed, info, nt, st);
    case 3: return launch_condense<3, 8>(records, S_packed, info, nt, st);
    case 4: return launch_condense<4, 8>(records, S_packed, info, nt, st);
    case 5: return launch_condense<5, 8>(records, S_packed, info, nt, st);
    case 6: return launch_condense<6, 8>(records, S_packed, info, nt, st);
  }
  return -1000;
}

MCS_API int mcs_element_blocks(int64_t nt, int nwgt, const double* W, int reclen, const int* prog_ptr,
                               const int* prog_widx, const double* prog_coef, double* records,
                               void* stream) {
  if (nt <= 0) return 0;
  auto st = static_cast<cudaStream_t>(stream);
  const int grid = static_cast<int>(nt < 148 * 16 ? nt : 148 * 16);
  element_blocks_kernel<<<grid, 256, nwgt * sizeof(double), st>>>(W, nwgt, prog_ptr, prog_widx,
                                                                   prog_coef, reclen, records, nt);
  return launch_status();
}
