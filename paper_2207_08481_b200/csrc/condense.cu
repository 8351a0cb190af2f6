// Per-element static condensation on B200.
//
// One CTA owns one element at a time (persistent over elements).  The
// element's symmetric augmented saddle matrix, padded to a multiple of 8, is
// eliminated on the FP64 tensor cores by the left-looking signed-Cholesky
// engine of elim_v5.cuh (panel in shared memory, trailing block in
// registers, one look-ahead diagonal per column):
//
//   microbench (A5):   K = [[A, B], [B^T, 0]]  -> eliminate the n_s (positive)
//                      pivots -> S = B^T A^-1 B
//   MCS (A3):          K = [[msig, bws^T, Bsig^T], [bws, 0, 0], [Bsig, 0, -adiv]]
//                      -> n_s positive then n_w negative pivots -> S_T, the
//                      reference's S_T of condensation.py:161-176 (LU of
//                      [[-msig, bws^T], [bws, 0]] then adiv - Bsig M^-1
//                      Bsig^T), proved equal in DESIGN.md §3.
//
// Raw block entries are read once, straight from the element record in HBM
// into the DMMA accumulators that consume them.  (The MCS element blocks of
// the solver path take the structured kernels of condense_struct.cu /
// condense_fused.cu; this dense engine serves the config-5 microbench and
// user-supplied blocks without the MCS structure.)
#include <cstdlib>

#include "elim_v5.cuh"

namespace mcs {

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

template <class Kern>
static int persistent_grid(Kern k, int threads, size_t smem, int64_t n);

// ------------------------------- v5 kernels (Crout signed Cholesky, elim_v5.cuh)

__device__ __forceinline__ void init_signs(signed char* ex, int npp, int npos, int np) {
  for (int i = threadIdx.x; i < npp; i += blockDim.x) ex[i] = (i < npos || i >= np) ? 1 : -1;
}

template <int NS, int NC, int W>
using MicroGeo5 = v5::Geo<((NS + 7) / 8 * 8 + (NC + 7) / 8 * 8) / 8, (NS + 7) / 8, W, NS, NS>;

template <int NS, int NC, int W, int MINB>
__global__ void __launch_bounds__(32 * W, MINB)
    spd_schur_v5(const double* __restrict__ A, const double* __restrict__ B,
                 double* __restrict__ S, int* __restrict__ info, int64_t batch) {
  using G = MicroGeo5<NS, NC, W>;
  constexpr int NPP = 8 * G::NPB;
  constexpr int LA = npk(NS), LB = NS * NC, LS = npk(NC);
  extern __shared__ __align__(128) double smem[];
  __shared__ int bad;
  __shared__ signed char expect[NPP];
  init_signs(expect, NPP, NS, NS);
  for (int64_t e = blockIdx.x; e < batch; e += gridDim.x) {
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    const double* Ae = A + e * LA;
    const double* Be = B + e * LB;
    double* Se = S + e * LS;
    auto entry = [&](int i, int j) -> const double* {  // padded (i, j), j < NPP
      if (i < NS) return j <= i ? Ae + pk(i, j) : v5::zero_src();
      if (i < NPP) return i == j ? v5::one_src() : v5::zero_src();
      return (i - NPP < NC && j < NS) ? Be + j * NC + (i - NPP) : v5::zero_src();
    };
    auto fetch = [&](int bi, int bj) {
      const int lane = threadIdx.x & 31, i = 8 * bi + (lane >> 2), j = 8 * bj + 2 * (lane & 3);
      return make_double2(__ldg(entry(i, j)), __ldg(entry(i, j + 1)));
    };
    auto trail = [](int, int) { return 0.0; };
    auto store = [&](int i, int j, double v) {
      i -= NPP;
      if (i < NC) Se[pk(i, j - NPP)] = v;
    };
    v5::eliminate<G>(fetch, trail, store, smem, expect, &bad);
    __syncthreads();
    if (threadIdx.x == 0 && info) info[e] = bad;
  }
}

template <int NS, int NC, int W, int MINB>
static int launch_spd_schur_v5(const double* A, const double* B, double* S, int* info,
                               int64_t batch, cudaStream_t st) {
  using G = MicroGeo5<NS, NC, W>;
  auto kern = spd_schur_v5<NS, NC, W, MINB>;
  const size_t smem = G::SMEM * sizeof(double);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = persistent_grid(kern, 32 * W, smem, batch);
  kern<<<grid, 32 * W, smem, st>>>(A, B, S, info, batch);
  return launch_status();
}

template <int K, int W>
using McsGeo5 = v5::Geo<((Sizes<K>::ns + Sizes<K>::nw + 7) / 8 * 8 + (Sizes<K>::nloc + 7) / 8 * 8) / 8,
                        (Sizes<K>::ns + Sizes<K>::nw + 7) / 8, W, Sizes<K>::ns + Sizes<K>::nw,
                        Sizes<K>::ns>;

template <int K, int W, int MINB>
__global__ void __launch_bounds__(32 * W, MINB)
    condense_v5(const double* __restrict__ recs, double* __restrict__ ST, int* __restrict__ info,
                int64_t nt) {
  using Z = Sizes<K>;
  using R = Record<K>;
  using G = McsGeo5<K, W>;
  constexpr int ns = Z::ns, nu = Z::nu, NP = Z::ns + Z::nw, NPP = 8 * G::NPB;
  extern __shared__ __align__(128) double smem[];
  __shared__ int bad;
  __shared__ signed char expect[NPP];
  for (int i = threadIdx.x; i < NPP; i += blockDim.x) expect[i] = i < ns ? 1 : -1;
  for (int64_t e = blockIdx.x; e < nt; e += gridDim.x) {
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    const double* rec = recs + e * R::len;
    double* Se = ST + e * R::st_len;
    auto entry = [&](int i, int j) -> const double* {  // padded (i, j), j < NPP
      if (i < ns) return j <= i ? rec + R::o_msig + i * ns + j : v5::zero_src();
      if (i < NP) return j < ns ? rec + R::o_bws + (i - ns) * ns + j : v5::zero_src();
      if (i < NPP) return i == j ? v5::minus_one_src() : v5::zero_src();  // padding: -1 pivots
      const int l = i - NPP;
      if (l >= Z::nloc || j >= ns) return v5::zero_src();
      return l < nu ? rec + R::o_bus + l * ns + j : rec + R::o_bhs + (l - nu) * ns + j;
    };
    auto fetch = [&](int bi, int bj) {
      const int lane = threadIdx.x & 31, i = 8 * bi + (lane >> 2), j = 8 * bj + 2 * (lane & 3);
      return make_double2(__ldg(entry(i, j)), __ldg(entry(i, j + 1)));
    };
    auto trail = [&](int i, int j) {
      const int l = i - NPP, m = j - NPP;
      return (l < nu && m < nu) ? __ldg(rec + R::o_adiv + l * nu + m) : 0.0;
    };
    auto store = [&](int i, int j, double v) {
      i -= NPP;
      if (i < Z::nloc) Se[pk(i, j - NPP)] = v;
    };
    v5::eliminate<G>(fetch, trail, store, smem, expect, &bad);
    __syncthreads();
    if (threadIdx.x == 0 && info) info[e] = bad;
  }
}

template <int K, int W, int MINB>
static int launch_condense_v5(const double* recs, double* ST, int* info, int64_t nt,
                              cudaStream_t st) {
  using G = McsGeo5<K, W>;
  auto kern = condense_v5<K, W, MINB>;
  const size_t smem = G::SMEM * sizeof(double);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = persistent_grid(kern, 32 * W, smem, nt);
  kern<<<grid, 32 * W, smem, st>>>(recs, ST, info, nt);
  return launch_status();
}

// ---------------------------------------------- A1: element blocks on the GPU
// rec[e][q] = sum_{p in prog[q]} W[e][widx[p]] * coef[p]   (refblocks.py)
// A CTA handles EB elements at once so every program entry fetched from
// L1/L2 serves EB elements; record writes are coalesced along q.
constexpr int EB = 8;

__global__ void __launch_bounds__(256)
    element_blocks_kernel(const double* __restrict__ W, int nwgt, const int* __restrict__ ptr,
                          const int* __restrict__ widx, const double* __restrict__ coef,
                          int reclen, double* __restrict__ recs, int64_t nt) {
  extern __shared__ double sw[];          // [EB][nwgt]
  for (int64_t base = (int64_t)blockIdx.x * EB; base < nt; base += (int64_t)gridDim.x * EB) {
    for (int r = threadIdx.x; r < EB * nwgt; r += blockDim.x) {
      const int64_t e = base + r / nwgt;
      sw[r] = e < nt ? W[e * nwgt + r % nwgt] : 0.0;
    }
    __syncthreads();
    for (int q = threadIdx.x; q < reclen; q += blockDim.x) {
      double acc[EB];
#pragma unroll
      for (int b = 0; b < EB; ++b) acc[b] = 0.0;
      const int p1 = __ldg(ptr + q + 1);
      for (int p = __ldg(ptr + q); p < p1; ++p) {
        const int w = __ldg(widx + p);
        const double c = __ldg(coef + p);
#pragma unroll
        for (int b = 0; b < EB; ++b) acc[b] = fma(sw[b * nwgt + w], c, acc[b]);
      }
#pragma unroll
      for (int b = 0; b < EB; ++b)
        if (base + b < nt) recs[(base + b) * reclen + q] = acc[b];
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
  // (declared above for the v3 launchers)
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, threads, smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  int64_t g = static_cast<int64_t>(per_sm) * num_sms();
  return static_cast<int>(n < g ? n : g);
}

template <int NS, int NC>
int launch_spd_schur_w2(const double* A, const double* B, double* S, int* info, int64_t batch,
                        cudaStream_t st);   // micro.cu

}  // namespace mcs

using namespace mcs;

MCS_API int mcs_spd_schur_batched(int n, int m, int64_t batch, const double* A_packed_lower,
                                  const double* B, double* S_packed, int* info, void* stream) {
  if (batch <= 0) return 0;
  auto st = static_cast<cudaStream_t>(stream);
  // default: the one-warp register-resident kernel of micro.cu (MCS_MICRO=2: its
  // two-warp kernel, 3: one warp per element with pair barriers); MCS_MICRO=5: the v5 engine
  static const int which = getenv("MCS_MICRO") ? atoi(getenv("MCS_MICRO")) : 1;
  if (n == 60 && m == 36) {
    if (which == 5) return launch_spd_schur_v5<60, 36, 4, 5>(A_packed_lower, B, S_packed, info, batch, st);
    return launch_spd_schur_w2<60, 36>(A_packed_lower, B, S_packed, info, batch, st);
  }
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
    // v5 engine (elim_v5.cuh); warps / CTAs per SM from tools/condense_v5_sweep.cu
    case 2: return launch_condense_v5<2, 2, 8>(records, S_packed, info, nt, st);
    case 3: return launch_condense_v5<3, 2, 8>(records, S_packed, info, nt, st);
    case 4: return launch_condense_v5<4, 4, 4>(records, S_packed, info, nt, st);
    case 5: return launch_condense_v5<5, 8, 2>(records, S_packed, info, nt, st);
    case 6: return launch_condense_v5<6, 8, 2>(records, S_packed, info, nt, st);
  }
  return -1000;
}

MCS_API int mcs_element_blocks(int64_t nt, int nwgt, const double* W, int reclen, const int* prog_ptr,
                               const int* prog_widx, const double* prog_coef, double* records,
                               void* stream) {
  if (nt <= 0) return 0;
  auto st = static_cast<cudaStream_t>(stream);
  const int64_t want = (nt + EB - 1) / EB;
  const int grid = static_cast<int>(want < 148 * 8 ? want : 148 * 8);
  element_blocks_kernel<<<grid, 256, EB * nwgt * sizeof(double), st>>>(
      W, nwgt, prog_ptr, prog_widx, prog_coef, reclen, records, nt);
  return launch_status();
}
