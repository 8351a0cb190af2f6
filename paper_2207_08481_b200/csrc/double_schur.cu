// Double Schur complement per element, the batched
// restatement of condensation.py:207-226 on the element-local S_T:
//   S_oo = S_T[iint, iint],  X = S_oo^-1 S_T[iint, icpl],
//   Sd_T = S_T[icpl, icpl] - S_T[icpl, iint] X.
// Interior rows are element-private, so this equals the reference's
// extraction from the assembled S (signs square away).
//
// One CTA per element (persistent): S_T (packed) arrives in shared memory by
// one 1-D bulk async copy; Gauss-Jordan without pivoting on the SPD block
// [S_oo | S_oc | I] yields [I | X | S_oo^-1]; Sd_T follows as a small
// SYRK-like product.  Outputs:
//   ext record  [X (n_int x ncpl, row-major) | S_oo^-1 (lower packed)]  (even stride)
//   Sd_T        lower packed (even stride)
#include "elim_v3.cuh"
#include "elim_v5.cuh"

namespace mcs {

template <int K>
__device__ __forceinline__ double sym_at(const double* P, int a, int b) {
  return a >= b ? P[pk(a, b)] : P[pk(b, a)];
}

template <int K, int THREADS>
__global__ void __launch_bounds__(THREADS)
    double_schur_kernel(const double* __restrict__ ST, double* __restrict__ ext,
                        double* __restrict__ Sd, int* __restrict__ info, int64_t nt) {
  using Z = Sizes<K>;
  using L = ExtLayout<K>;
  constexpr int NI = Z::n_int, NC = Z::ncpl, WC = 2 * NI + NC;
  extern __shared__ __align__(128) double sm[];
  double* sS = sm;                        // packed S_T
  double* W = sm + L::st_len;             // NI x WC
  double* mcol = W + NI * WC;             // NI
  double* prow = mcol + NI;               // WC
  __shared__ __align__(8) uint64_t bar;
  __shared__ int bad;
  const int tid = threadIdx.x;

  int64_t e = blockIdx.x;
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (tid == 0 && e < nt) {
    mbar_expect_tx(&bar, L::st_len * 8);
    bulk_g2s(sS, ST + e * L::st_len, L::st_len * 8, &bar);
  }
  uint32_t phase = 0;
  for (; e < nt; e += gridDim.x) {
    mbar_wait(&bar, phase);
    phase ^= 1;
    if (tid == 0) bad = 0;
    for (int q = tid; q < NI * WC; q += THREADS) {
      const int i = q / WC, c = q % WC;
      const int li = Z::n_em + i;
      double v;
      if (c < NI) v = sym_at<K>(sS, li, Z::n_em + c);
      else if (c < NI + NC) v = sym_at<K>(sS, li, cpl_local<K>(c - NI));
      else v = (c - NI - NC == i) ? 1.0 : 0.0;
      W[q] = v;
    }
    __syncthreads();
    for (int j = 0; j < NI; ++j) {
      const double piv = W[j * WC + j];
      if (tid == 0 && !(piv > 0.0) && bad == 0) bad = j + 1;
      const double inv = 1.0 / piv;
      for (int q = tid; q < NI + WC; q += THREADS) {
        if (q < NI) mcol[q] = W[q * WC + j];
        else prow[q - NI] = W[j * WC + (q - NI)] * inv;
      }
      __syncthreads();
      // columns <= j are already unit vectors: update c in (j, WC)
      const int ncols = WC - j - 1;
      for (int q = tid; q < NI * ncols; q += THREADS) {
        const int i = q / ncols, c = j + 1 + q % ncols;
        W[i * WC + c] = (i == j) ? prow[c] : fma(-mcol[i], prow[c], W[i * WC + c]);
      }
      __syncthreads();
    }
    // outputs
    double* xo = ext + e * L::len;
    for (int q = tid; q < NI * NC; q += THREADS) {
      const int i = q / NC, c = q % NC;
      xo[q] = W[i * WC + NI + c];
    }
    for (int q = tid; q < npk(NI); q += THREADS) {
      int i = 0;
      while (pk(i + 1, 0) <= q) ++i;
      const int c = q - pk(i, 0);
      xo[L::x_len + q] = 0.5 * (W[i * WC + NI + NC + c] + W[c * WC + NI + NC + i]);
    }
    double* so = Sd + e * L::sd_len;
    for (int q = tid; q < npk(NC); q += THREADS) {
      int a = 0;
      while (pk(a + 1, 0) <= q) ++a;
      const int b = q - pk(a, 0);
      const int la = cpl_local<K>(a), lb = cpl_local<K>(b);
      double s = 0.0;
#pragma unroll 5
      for (int i = 0; i < NI; ++i) s = fma(sym_at<K>(sS, la, Z::n_em + i), W[i * WC + NI + b], s);
      so[q] = sym_at<K>(sS, la, lb) - s;
    }
    __syncthreads();
    const int64_t nxt = e + gridDim.x;
    if (tid == 0 && nxt < nt) {
      mbar_expect_tx(&bar, L::st_len * 8);
      bulk_g2s(sS, ST + nxt * L::st_len, L::st_len * 8, &bar);
    }
    if (tid == 0 && info) info[e] = bad;
  }
}

// ---- v3: the same DMMA blocked elimination engine as the condensation, on
// K = [[S_oo, S_oc, I], [S_co, S_cc, 0], [I, 0, 0]]  (o = interior bubbles,
// c = coupling dofs).  Eliminating the n_int (positive) o pivots leaves
//   [[S_cc - S_co S_oo^-1 S_oc, -(S_oo^-1 S_oc)^T], [-S_oo^-1 S_oc, -S_oo^-1]]
// = [[Sd_T, -X^T], [-X, -S_oo^-1]] as the trailing block, i.e. all three
// outputs of the reference's double_schur in one elimination.
template <int K, int W, int MINB>
__global__ void __launch_bounds__(32 * W, MINB)
    double_schur_v3(const double* __restrict__ ST, double* __restrict__ ext,
                    double* __restrict__ Sd, int* __restrict__ info, int64_t nt) {
  using Z = Sizes<K>;
  using L = ExtLayout<K>;
  constexpr int NI = Z::n_int, NC = Z::ncpl, NP = NI, NTR = NC + NI;
  constexpr int NPP = (NP + 7) / 8 * 8, NCP = (NTR + 7) / 8 * 8;
  using G = v3::Geo<(NPP + NCP) / 8, NPP / 8, W>;
  extern __shared__ __align__(128) double smem[];
  __shared__ int bad;
  __shared__ signed char expect[NPP];
  for (int i = threadIdx.x; i < NPP; i += blockDim.x) expect[i] = i < NP ? 1 : 0;
  const v3::Smem<G> sm{smem};
  const int warp = threadIdx.x >> 5;
  for (int64_t e = blockIdx.x; e < nt; e += gridDim.x) {
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    const double* S = ST + e * L::st_len;
    double* xo = ext + e * L::len;
    double* so = Sd + e * L::sd_len;
    // real index -> local S_T index: o rows, then c rows; E rows return -1
    auto loc = [](int r) { return r < NI ? Z::n_em + r : (r < NI + NC ? cpl_local<K>(r - NI) : -1); };
    auto load = [&](int i, int j) {
      return v3::padded_entry<NP, NTR, NPP>(i, j, [&](int ri, int rj) {
        const int li = loc(ri), lj = loc(rj);
        if (li >= 0 && lj >= 0) return __ldg(S + (li >= lj ? pk(li, lj) : pk(lj, li)));
        // E rows: identity against the o columns
        if (li < 0 && lj >= 0) return (rj < NI && ri - NI - NC == rj) ? 1.0 : 0.0;
        return 0.0;
      });
    };
    auto store = [&](int i, int j, double v) {
      i -= NPP;
      j -= NPP;
      if (j > i || i >= NTR) return;
      if (i < NC) so[pk(i, j)] = v;                                  // Sd_T
      else if (j < NC) xo[(i - NC) * NC + j] = -v;                    // X
      else xo[L::x_len + pk(i - NC, j - NC)] = -v;                    // S_oo^-1
    };
    v3::dispatch<G>(warp, load, store, sm, expect, &bad);
    __syncthreads();
    if (threadIdx.x == 0 && info) info[e] = bad;
  }
}

template <int K, int W, int MINB>
static int launch_double_schur_v3(const double* ST, double* ext, double* Sd, int* info, int64_t nt,
                                  cudaStream_t st) {
  using Z = Sizes<K>;
  constexpr int NPP = (Z::n_int + 7) / 8 * 8, NCP = (Z::ncpl + Z::n_int + 7) / 8 * 8;
  using G = v3::Geo<(NPP + NCP) / 8, NPP / 8, W>;
  auto kern = double_schur_v3<K, W, MINB>;
  const size_t smem = G::SMEM * sizeof(double);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 1, dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * W, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t g = (int64_t)per_sm * nsm;
  kern<<<(int)(nt < g ? nt : g), 32 * W, smem, st>>>(ST, ext, Sd, info, nt);
  return launch_status();
}

// ---- v5: the left-looking signed-Cholesky engine of elim_v5.cuh on the same
// K = [[S_oo, S_oc, I], [S_co, S_cc, 0], [I, 0, 0]] (n_int positive pivots).
// The engine's STORE receives minus the trailing block:
//   [[-Sd_T, X^T], [X, S_oo^-1]].
template <int K, int W>
using DsGeo5 = v5::Geo<((Sizes<K>::n_int + 7) / 8 * 8 + (Sizes<K>::ncpl + Sizes<K>::n_int + 7) / 8 * 8) / 8,
                       (Sizes<K>::n_int + 7) / 8, W, Sizes<K>::n_int, Sizes<K>::n_int>;

template <int K, int W, int MINB>
__global__ void __launch_bounds__(32 * W, MINB)
    double_schur_v5(const double* __restrict__ ST, double* __restrict__ ext,
                    double* __restrict__ Sd, int* __restrict__ info, int64_t nt) {
  using Z = Sizes<K>;
  using L = ExtLayout<K>;
  using G = DsGeo5<K, W>;
  constexpr int NI = Z::n_int, NC = Z::ncpl, NEM = Z::n_em, NPP = 8 * G::NPB;
  extern __shared__ __align__(128) double smem[];
  __shared__ int bad;
  __shared__ signed char expect[NPP];
  for (int i = threadIdx.x; i < NPP; i += blockDim.x) expect[i] = 1;
  for (int64_t e = blockIdx.x; e < nt; e += gridDim.x) {
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    const double* S = ST + e * L::st_len;
    double* xo = ext + e * L::len;
    double* so = Sd + e * L::sd_len;
    auto sym = [&](int a, int b) { return __ldg(S + (a >= b ? pk(a, b) : pk(b, a))); };
    auto entry = [&](int i, int j) -> double {   // padded (i, j), j < NPP (pivot columns)
      if (i < NPP) {
        if (i < NI && j < NI) return sym(NEM + i, NEM + j);
        return i == j ? 1.0 : 0.0;
      }
      if (j >= NI) return 0.0;
      const int r = i - NPP;
      if (r < NC) return sym(cpl_local<K>(r), NEM + j);
      return (r - NC == j) ? 1.0 : 0.0;              // identity rows (r < NC + NI), padding 0
    };
    auto fetch = [&](int bi, int bj) {
      const int lane = threadIdx.x & 31, i = 8 * bi + (lane >> 2), j = 8 * bj + 2 * (lane & 3);
      return make_double2(entry(i, j), entry(i, j + 1));
    };
    auto trail = [&](int i, int j) {                 // -K_tt: -S_cc, zero elsewhere
      const int r = i - NPP, c = j - NPP;
      return (r < NC && c < NC) ? -sym(cpl_local<K>(r), cpl_local<K>(c)) : 0.0;
    };
    auto store = [&](int i, int j, double v) {
      const int r = i - NPP, c = j - NPP;
      if (r < NC) so[pk(r, c)] = -v;
      else if (r < NC + NI) {
        if (c < NC) xo[(r - NC) * NC + c] = v;
        else xo[L::x_len + pk(r - NC, c - NC)] = v;
      }
    };
    v5::eliminate<G>(fetch, trail, store, smem, expect, &bad);
    __syncthreads();
    if (threadIdx.x == 0 && info) info[e] = bad;
  }
}

template <int K, int W, int MINB>
static int launch_double_schur_v5(const double* ST, double* ext, double* Sd, int* info, int64_t nt,
                                  cudaStream_t st) {
  using G = DsGeo5<K, W>;
  auto kern = double_schur_v5<K, W, MINB>;
  const size_t smem = G::SMEM * sizeof(double);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 1, dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * W, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t g = (int64_t)per_sm * nsm;
  kern<<<(int)(nt < g ? nt : g), 32 * W, smem, st>>>(ST, ext, Sd, info, nt);
  return launch_status();
}

template <int K>
static int launch_double_schur(const double* ST, double* ext, double* Sd, int* info, int64_t nt,
                               cudaStream_t st) {
  using Z = Sizes<K>;
  using L = ExtLayout<K>;
  constexpr int THREADS = 128;
  auto kern = double_schur_kernel<K, THREADS>;
  const size_t smem =
      (L::st_len + Z::n_int * (2 * Z::n_int + Z::ncpl) + Z::n_int + 2 * Z::n_int + Z::ncpl) *
      sizeof(double);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 1, dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, THREADS, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t g = (int64_t)per_sm * nsm;
  kern<<<(int)(nt < g ? nt : g), THREADS, smem, st>>>(ST, ext, Sd, info, nt);
  return launch_status();
}

}  // namespace mcs

using namespace mcs;

MCS_API int mcs_ext_stride(int k) {
  switch (k) {
    case 2: return ExtLayout<2>::len;
    case 3: return ExtLayout<3>::len;
    case 4: return ExtLayout<4>::len;
    case 5: return ExtLayout<5>::len;
    case 6: return ExtLayout<6>::len;
  }
  return -1;
}

MCS_API int mcs_sd_stride(int k) {
  switch (k) {
    case 2: return ExtLayout<2>::sd_len;
    case 3: return ExtLayout<3>::sd_len;
    case 4: return ExtLayout<4>::sd_len;
    case 5: return ExtLayout<5>::sd_len;
    case 6: return ExtLayout<6>::sd_len;
  }
  return -1;
}

MCS_API int mcs_double_schur(int k, int64_t nt, const double* S_packed, double* ext, double* Sd_packed,
                             int* info, void* stream) {
  if (nt <= 0) return 0;
  auto st = static_cast<cudaStream_t>(stream);
  switch (k) {
    case 2: return launch_double_schur_v3<2, 2, 6>(S_packed, ext, Sd_packed, info, nt, st);
    case 3: return launch_double_schur_v3<3, 2, 4>(S_packed, ext, Sd_packed, info, nt, st);
    case 4: return launch_double_schur_v3<4, 2, 4>(S_packed, ext, Sd_packed, info, nt, st);
    case 5: return launch_double_schur_v5<5, 4, 4>(S_packed, ext, Sd_packed, info, nt, st);
    case 6: return launch_double_schur_v5<6, 8, 2>(S_packed, ext, Sd_packed, info, nt, st);
  }
  return -1000;
}
