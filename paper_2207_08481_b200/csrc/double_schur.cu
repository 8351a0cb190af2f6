// Double Schur complement per element, the batched
// restatement of condensation.py:207-226 on the element-local S_T:
//   S_oo = S_T[iint, iint],  X = S_oo^-1 S_T[iint, icpl],
//   Sd_T = S_T[icpl, icpl] - S_T[icpl, iint] X.
// Interior rows are element-private, so this equals the reference's
// extraction from the assembled S (signs square away).
//
// (For k <= 4 the fused condensation kernel computes these outputs itself;
// this kernel serves k = 5, 6 and user-supplied blocks.)  One CTA per
// element (persistent), the signed-Cholesky DMMA engine of elim_v5.cuh.
// Outputs:
//   ext record  [X (n_int x ncpl, row-major) | S_oo^-1 (lower packed)]  (even stride)
//   Sd_T        lower packed (even stride)
#include <cstdlib>

#include "ds_reg.cuh"
#include "ds_warp.cuh"
#include "elim_v5.cuh"

namespace mcs {

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

// ---- warp per element (default for every k): the reference's own sequence
// (condensation.py:207-226) on registers, shared memory and the FP64 tensor
// cores, no inter-warp barrier:
//   S_oo = L L^T   lane-per-row Cholesky with shuffles for the pivots (rows
//                  32.. of k = 6 in shared memory, updated by lanes 0..2);
//   L^-1           lane-per-column forward substitution, blocked by 8 rows
//                  (an 8-wide independent update, then an 8-step chain);
//   W = L^-1 S_oc, X = L^-T W, S_oo^-1 = L^-T L^-1, Sd_T = S_cc - W^T W
//                  m8n8k4 DMMA over 8x8 output tiles (k steps of 4 rows).
// S_T is read from global memory (it was written by the condensation kernel
// just before, so mostly from L2); per warp shared memory holds L, then W,
// and L^-1.  (The v5 CTA engine above is kept as MCS_DS=5 for A/B.)
// standalone layout (one warp per element): L, then W over it | L^-1 | rd
template <int K>
struct DswLayout {
  using G = dsw::Geo<K>;
  static constexpr int o_L = 0;
  static constexpr int LW = G::L_LEN > G::W_LEN ? G::L_LEN : G::W_LEN;
  static constexpr int o_LI = LW;
  static constexpr int o_rd = o_LI + G::LI_LEN;
  static constexpr int PER_WARP = even(o_rd + G::NI);
};

template <int K, int WPB, int YM>
__global__ void __launch_bounds__(32 * WPB)
    double_schur_warp(const double* __restrict__ ST, double* __restrict__ ext,
                      double* __restrict__ Sd, int* __restrict__ info, int64_t nt) {
  using G = dsw::Geo<K>;
  using Y = DswLayout<K>;
  using L = ExtLayout<K>;
  extern __shared__ __align__(128) double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* base = smem + warp * Y::PER_WARP;
  double* Ls = base + Y::o_L;
  double* Wd = base + Y::o_L;      // W replaces L once L^-1 exists
  double* LI = base + Y::o_LI;
  double* rd = base + Y::o_rd;
  const int64_t nw = (int64_t)gridDim.x * WPB;
#pragma unroll 1
  for (int64_t e = (int64_t)blockIdx.x * WPB + warp; e < nt; e += nw) {
    const double* S = ST + e * L::st_len;
    auto Sg = [&](int a, int b) { return __ldg(S + (a >= b ? pk(a, b) : pk(b, a))); };
    // pull the next element's S_T into L2 while this one is eliminated
    if (e + nw < nt) {
      const char* nx = reinterpret_cast<const char*>(ST + (e + nw) * L::st_len);
      for (int off = lane * 128; off < L::st_len * 8; off += 32 * 128)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(nx + off));
    }
    const bool ok = dsw::chol_soo<K>(Sg, Ls, rd);
    __syncwarp();
    dsw::linv<K>(Ls, rd, LI);
    __syncwarp();
    dsw::stage_soc<K>(Sg, Wd, lane, 32);
    __syncwarp();
#pragma unroll 1
    for (int J = 0; J < G::NCB; ++J) dsw::w_block<K, YM>(LI, Wd, J);
    dsw::out_tiles<K, decltype(Sg), YM>(Sg, LI, Wd, ext + e * L::len, Sd + e * L::sd_len, 0, 1);
    if (lane == 0 && info) info[e] = ok ? 0 : 1;
    __syncwarp();
  }
}

template <int K, int WPB, int YM>
static int launch_dsw(const double* ST, double* ext, double* Sd, int* info,
                      int64_t nt, cudaStream_t st) {
  auto kern = double_schur_warp<K, WPB, YM>;
  const size_t smem = (size_t)WPB * DswLayout<K>::PER_WARP * sizeof(double);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * WPB, smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  const int64_t want = (nt + WPB - 1) / WPB, cap = (int64_t)per_sm * sm_count();
  kern<<<(int)(want < cap ? want : cap), 32 * WPB, smem, st>>>(ST, ext, Sd, info, nt);
  return launch_status();
}

template <int K, int WPB>
static int launch_double_schur_warp(const double* ST, double* ext, double* Sd, int* info,
                                    int64_t nt, cudaStream_t st) {
  // MCS_DS_YIELD: throttle mask (1 after every W column block, 2 after every
  // output tile, 4 after every 4th output tile); A/B measurements
  static const int ym = getenv("MCS_DS_YIELD") ? atoi(getenv("MCS_DS_YIELD")) : 0;
  switch (ym) {
    case 1: return launch_dsw<K, WPB, 1>(ST, ext, Sd, info, nt, st);
    case 2: return launch_dsw<K, WPB, 2>(ST, ext, Sd, info, nt, st);
    case 3: return launch_dsw<K, WPB, 3>(ST, ext, Sd, info, nt, st);
    case 4: return launch_dsw<K, WPB, 4>(ST, ext, Sd, info, nt, st);
    case 5: return launch_dsw<K, WPB, 5>(ST, ext, Sd, info, nt, st);
  }
  return launch_dsw<K, WPB, 0>(ST, ext, Sd, info, nt, st);
}

// ---- register-resident warp-per-element kernel (ds_reg.cuh).  PAIR: one
// 8-warp CTA per SM, warps w and w + 4 (same SM sub-partition) in lockstep
// through a named barrier before every pivot tile (dsr::sweep).
template <int K, int WPB, int MINB, bool PAIR>
__global__ void __launch_bounds__(32 * WPB, MINB)
    double_schur_reg(const double* __restrict__ ST, double* __restrict__ ext,
                     double* __restrict__ Sd, int* __restrict__ info, int64_t nt, int pf) {
  using G = dsr::Geo<K>;
  using L = ExtLayout<K>;
  static_assert(!PAIR || WPB == 8, "pairs: warps w, w + 4 of an 8-warp CTA");
  extern __shared__ __align__(128) double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* T = smem + warp * G::PER_WARP;
  const int64_t nw = (int64_t)gridDim.x * WPB;
  // every warp of the CTA runs the same number of rounds (the pair barriers);
  // a warp past the end repeats the last element into its own scratch-free
  // outputs (same values, harmless rewrite)
  const int64_t e0 = (int64_t)blockIdx.x * WPB;
  const int64_t rounds = e0 < nt ? (nt - e0 + nw - 1) / nw : 0;
#pragma unroll 1
  for (int64_t rd = 0; rd < rounds; ++rd) {
    const int64_t ew = e0 + warp + rd * nw;
    const int64_t e = ew < nt ? ew : nt - 1;
    if (pf && e + nw < nt) {               // the next element's S_T into L2
      const char* nx = reinterpret_cast<const char*>(ST + (e + nw) * L::st_len);
      for (int off = lane * 128; off < L::st_len * 8; off += 32 * 128)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(nx + off));
    }
    const double* S = ST + e * L::st_len;
    auto sym = [&](int a, int b) { return __ldg(S + (a >= b ? pk(a, b) : pk(b, a))); };
    bool ok;
    if constexpr (PAIR)
      ok = dsr::element_pm<K, decltype(sym), dsr::PairSync0, (K >= 5), false, true>(sym, T, ext + e * L::len, Sd + e * L::sd_len,
                                                                  dsr::PairSync0{1 + (warp & 3)});
    else
      ok = dsr::element_pm<K, decltype(sym), dsr::NoSync, (K >= 5), false, true>(sym, T, ext + e * L::len, Sd + e * L::sd_len);
    if (lane == 0 && info) info[e] = ok ? 0 : 1;
  }
}

template <int K, int WPB, int MINB, bool PAIR>
static int launch_double_schur_reg(const double* ST, double* ext, double* Sd, int* info,
                                   int64_t nt, cudaStream_t st) {
  auto kern = double_schur_reg<K, WPB, MINB, PAIR>;
  const size_t smem = (size_t)WPB * dsr::Geo<K>::PER_WARP * sizeof(double);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * WPB, smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  const int64_t want = (nt + WPB - 1) / WPB, cap = (int64_t)per_sm * sm_count();
  static const int pf = getenv("MCS_DSR_PF") ? atoi(getenv("MCS_DSR_PF")) : 0;   // 1: L2 prefetch of the next S_T (same time, 1.4x the DRAM reads)
  kern<<<(int)(want < cap ? want : cap), 32 * WPB, smem, st>>>(ST, ext, Sd, info, nt, pf);
  return launch_status();
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
  // default: the register-resident warp-per-element kernel (ds_reg.cuh);
  // MCS_DS=1: the shared-memory warp kernel (ds_warp.cuh), MCS_DS=5: the v5 CTA engine
  static const int ds = getenv("MCS_DS") ? atoi(getenv("MCS_DS")) : 2;
  if (ds == 2) {                            // register-resident kernel (ds_reg.cuh)
    // MCS_DSR_PAIR=0: k = 5, 6 without the pair barriers (A/B measurements)
    static const int pair = getenv("MCS_DSR_PAIR") ? atoi(getenv("MCS_DSR_PAIR")) : 1;
    switch (k) {
      case 2: return launch_double_schur_reg<2, 4, 1, false>(S_packed, ext, Sd_packed, info, nt, st);
      case 3: return launch_double_schur_reg<3, 4, 1, false>(S_packed, ext, Sd_packed, info, nt, st);
      case 4: return launch_double_schur_reg<4, 4, 1, false>(S_packed, ext, Sd_packed, info, nt, st);
      case 5:
        if (pair) return launch_double_schur_reg<5, 8, 1, true>(S_packed, ext, Sd_packed, info, nt, st);
        return launch_double_schur_reg<5, 4, 2, false>(S_packed, ext, Sd_packed, info, nt, st);
      case 6:
        if (pair) return launch_double_schur_reg<6, 8, 1, true>(S_packed, ext, Sd_packed, info, nt, st);
        return launch_double_schur_reg<6, 4, 2, false>(S_packed, ext, Sd_packed, info, nt, st);
    }
    return -1000;
  }
  if (ds != 5) {
    switch (k) {
      case 2: return launch_double_schur_warp<2, 4>(S_packed, ext, Sd_packed, info, nt, st);
      case 3: return launch_double_schur_warp<3, 4>(S_packed, ext, Sd_packed, info, nt, st);
      case 4: return launch_double_schur_warp<4, 4>(S_packed, ext, Sd_packed, info, nt, st);
      case 5: return launch_double_schur_warp<5, 1>(S_packed, ext, Sd_packed, info, nt, st);
      case 6: return launch_double_schur_warp<6, 1>(S_packed, ext, Sd_packed, info, nt, st);
    }
    return -1000;
  }
  switch (k) {
    case 2: return launch_double_schur_v5<2, 2, 8>(S_packed, ext, Sd_packed, info, nt, st);
    case 3: return launch_double_schur_v5<3, 2, 6>(S_packed, ext, Sd_packed, info, nt, st);
    case 4: return launch_double_schur_v5<4, 4, 4>(S_packed, ext, Sd_packed, info, nt, st);
    case 5: return launch_double_schur_v5<5, 4, 4>(S_packed, ext, Sd_packed, info, nt, st);
    case 6: {
      // MCS_DS6 = 0..3 selects the (warps, CTAs/SM) variant (A/B measurements)
      static const int v = getenv("MCS_DS6") ? atoi(getenv("MCS_DS6")) : 0;
      switch (v) {
        case 1: return launch_double_schur_v5<6, 2, 6>(S_packed, ext, Sd_packed, info, nt, st);
        case 2: return launch_double_schur_v5<6, 4, 4>(S_packed, ext, Sd_packed, info, nt, st);
        case 3: return launch_double_schur_v5<6, 4, 6>(S_packed, ext, Sd_packed, info, nt, st);
        default: return launch_double_schur_v5<6, 8, 2>(S_packed, ext, Sd_packed, info, nt, st);
      }
    }
  }
  return -1000;
}
