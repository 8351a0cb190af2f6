// Warp-level building blocks of the per-element double Schur complement
// (the reference's sequence condensation.py:207-226 on the
// element-local S_T):
//   S_oo = L L^T       chol_soo   lane-per-row Cholesky with shuffles for the
//                                 pivots; k = 6 has n_int = 35 > 32 rows: block
//                                 Cholesky, the 3 extra rows via L21 = A21 L11^-T
//                                 (lanes 0..2) and L22 = chol(A22 - L21 L21^T)
//   L^-1               linv       lane-per-column blocked forward substitution
//   W = L^-1 S_oc      stage_soc + w_block   (m8n8k4 DMMA, in place per column block)
//   X = L^-T W, S_oo^-1 = L^-T L^-1, Sd_T = S_cc - W^T W
//                      out_tiles  (DMMA over 8x8 output tiles)
// Used by the standalone warp-per-element kernel (double_schur.cu) and as the
// last phase of the generation-fused condensation for k = 5, 6
// (condense_struct.cu), where the four warps of an element's CTA split it.
// S_T is read through a functor Sg(a, b) (packed lower, symmetric access).
#pragma once
#include "common.cuh"

namespace mcs {
namespace dsw {

template <int K>
struct Geo {
  using Z = Sizes<K>;
  static constexpr int NI = Z::n_int, NC = Z::ncpl, NEM = Z::n_em;
  static constexpr int NR = NI < 32 ? NI : 32, NX = NI - NR;   // register rows / extra rows
  static constexpr int NIK = (NI + 3) / 4;                 // k steps over the interior rows
  static constexpr int NIT = (NI + 7) / 8;                 // 8-row tiles of X / S_oo^-1
  // padded rows of W / L^-1: the k steps read rows < 4 NIK, the 8-row tiles < 8 NIT
  static constexpr int NIR = 8 * NIT > 4 * NIK ? 8 * NIT : 4 * NIK;
  static constexpr int NCB = (NC + 7) / 8;                 // 8-column tiles of W / Sd
  // row strides == 4 or 12 mod 16 (doubles): the DMMA operand loads
  // (4ks + t) * ST + 8J + g of a half-warp hit 16 distinct 8-byte banks
  static constexpr int st_(int n) { return (n % 16 == 4 || n % 16 == 12) ? n : st_(n + 1); }
  static constexpr int WST = st_(8 * NCB);
  static constexpr int LST = st_(8 * NIT);
  static constexpr int NWR = 4 * NIK;                      // rows of W the k steps read
  static constexpr int L_LEN = NI * NI, LI_LEN = NIR * LST, W_LEN = NWR * WST;
  static constexpr int NTX = NIT * NCB, NTS = NIT * (NIT + 1) / 2, NTD = NCB * (NCB + 1) / 2;
  static constexpr int NTILES = NTX + NTS + NTD;           // output tiles of out_tiles
  static_assert(NX <= 8 && NC <= 64, "lane-per-row factor: at most 8 extra rows");
};

// S_oo = L L^T into Ls (row-major NI x NI, lower significant) and rd[j] =
// 1 / L_jj.  Warp-level; returns false if a pivot is not positive.
template <int K, class SG>
__device__ __forceinline__ bool chol_soo(SG Sg, double* Ls, double* rd) {
  using G = Geo<K>;
  constexpr int NI = G::NI, NEM = G::NEM, NR = G::NR, NX = G::NX;
  const int lane = threadIdx.x & 31;
  bool ok = true;
  const int r0 = lane < NR ? lane : 0;
  double a[NR];
#pragma unroll
  for (int c = 0; c < NR; ++c) a[c] = Sg(NEM + r0, NEM + c);
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    const double d = __shfl_sync(0xffffffffu, a[j], j);
    ok &= d > 0.0;
    const double r = rsqrt_nr(d);
    if (lane == 0) rd[j] = r;
    a[j] *= r;
#pragma unroll
    for (int c = j + 1; c < NR; ++c) a[c] = fma(-a[j], __shfl_sync(0xffffffffu, a[j], c), a[c]);
  }
  if (lane < NR) {
#pragma unroll
    for (int c = 0; c < NR; ++c) Ls[lane * NI + c] = a[c];
  }
  if constexpr (NX > 0) {
    __syncwarp();
    if (lane < NX) {
      const int i = NR + lane;
      double y[NR];
#pragma unroll
      for (int jb = 0; jb < NR; jb += 8) {
        double acc[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u] = Sg(NEM + i, NEM + jb + u);
#pragma unroll
        for (int q = 0; q < jb; ++q)
#pragma unroll
          for (int u = 0; u < 8; ++u) acc[u] = fma(-Ls[(jb + u) * NI + q], y[q], acc[u]);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int j = jb + u;
          double v = acc[u];
#pragma unroll
          for (int q = jb; q < j; ++q) v = fma(-Ls[j * NI + q], y[q], v);
          y[j] = v * rd[j];
        }
      }
#pragma unroll
      for (int q = 0; q < NR; ++q) Ls[i * NI + q] = y[q];
      __syncwarp((1u << NX) - 1);          // the other extra rows of L21 are read below
      // A22 - L21 L21^T, row i, columns NR..i
#pragma unroll
      for (int u = 0; u < NX; ++u) {
        double v = Sg(NEM + i, NEM + NR + u);
#pragma unroll
        for (int q = 0; q < NR; ++q) v = fma(-y[q], Ls[(NR + u) * NI + q], v);
        if (u <= lane) Ls[i * NI + NR + u] = v;
      }
    }
    __syncwarp();
    if (lane == 0) {                       // L22 = chol of the NX x NX remainder (in place)
#pragma unroll
      for (int j = 0; j < NX; ++j) {
        double* Lj = Ls + (NR + j) * NI + NR;
        const double d = Lj[j];
        ok &= d > 0.0;
        const double r = rsqrt_nr(d);
        rd[NR + j] = r;
        Lj[j] = d * r;
#pragma unroll
        for (int i2 = j + 1; i2 < NX; ++i2) {
          double* Li2 = Ls + (NR + i2) * NI + NR;
          Li2[j] *= r;
#pragma unroll
          for (int c = j + 1; c <= i2; ++c) Li2[c] = fma(-Li2[j], Ls[(NR + c) * NI + NR + j], Li2[c]);
        }
      }
    }
    ok = __shfl_sync(0xffffffffu, ok, 0) && ok;
  }
  return __all_sync(0xffffffffu, ok);
}

// L^-1 into LI (NIR x LST, zero padded), lane per column.  Warp-level.
template <int K>
__device__ __forceinline__ void linv(const double* Ls, const double* rd, double* LI) {
  using G = Geo<K>;
  constexpr int NI = G::NI, NIR = G::NIR, LST = G::LST, NX = G::NX;
  const int lane = threadIdx.x & 31;
  for (int q = lane; q < NIR * LST; q += 32) {
    const int j = q / LST, c = q % LST;
    if (j >= NI || c >= NI) LI[q] = 0.0;
  }
  const int c = lane;                         // column c < min(NI, 32)
  if (c < NI) {
    double x[NI];
#pragma unroll
    for (int jb = 0; jb < NI; jb += 8) {
      double acc[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) acc[u] = (jb + u == c) ? 1.0 : 0.0;
#pragma unroll
      for (int q = 0; q < jb; ++q)            // rows of earlier blocks: independent FMAs
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (jb + u < NI) acc[u] = fma(-Ls[(jb + u) * NI + q], x[q], acc[u]);
#pragma unroll
      for (int u = 0; u < 8; ++u) {            // the diagonal block: an 8-step chain
        const int j = jb + u;
        if (j < NI) {
          double v = acc[u];
#pragma unroll
          for (int q = jb; q < j; ++q) v = fma(-Ls[j * NI + q], x[q], v);
          x[j] = v * rd[j];
        }
      }
    }
#pragma unroll
    for (int j = 0; j < NI; ++j) LI[j * LST + c] = (j >= c) ? x[j] : 0.0;
  }
  if constexpr (NX > 0) {                     // columns 32.. : nonzero only in rows >= 32
    if (lane < NX) {
      const int cc = 32 + lane;
#pragma unroll
      for (int j = 0; j < 32; ++j) LI[j * LST + cc] = 0.0;   // upper triangle
      double y[NX];
#pragma unroll
      for (int u = 0; u < NX; ++u) {
        const int j = 32 + u;
        double v = (j == cc) ? 1.0 : 0.0;
#pragma unroll
        for (int q = 0; q < u; ++q) v = fma(-Ls[j * NI + 32 + q], y[q], v);
        y[u] = v * rd[j];
        LI[j * LST + cc] = (j >= cc) ? y[u] : 0.0;
      }
    }
  }
}

// S_oc (rows NIR x WST, zero padded) into Wd by threads tid, tid + nthr, ...
template <int K, class SG>
__device__ __forceinline__ void stage_soc(SG Sg, double* Wd, int tid, int nthr) {
  using G = Geo<K>;
  constexpr int NI = G::NI, NC = G::NC, NEM = G::NEM, WST = G::WST, NIR = G::NIR;
  // (loads batched 16 deep: each is an L2 round trip)
#pragma unroll 16
  for (int q = tid; q < G::NWR * WST; q += nthr) {
    const int j = q / WST, c = q % WST;
    Wd[q] = (j < NI && c < NC) ? Sg(NEM + j, cpl_local<K>(c)) : 0.0;
  }
}

// W column block J = L^-1 S_oc[:, block J], in place over the staged S_oc.
// YM: FP64-pipe throttle (tools/dmma_prio.cu): __nanosleep(0) after a DMMA
// burst lets the dependent chains of the co-resident warps through.
template <int K, int YM = 0>
__device__ __forceinline__ void w_block(const double* LI, double* Wd, int J) {
  using G = Geo<K>;
  constexpr int WST = G::WST, LST = G::LST, NIR = G::NIR;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double cacc[G::NIT][2];
#pragma unroll
  for (int I = 0; I < G::NIT; ++I) {
    cacc[I][0] = cacc[I][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < G::NIK; ++ks)
      dmma884(cacc[I][0], cacc[I][1], LI[(8 * I + g) * LST + 4 * ks + t],
              Wd[(4 * ks + t) * WST + 8 * J + g]);
  }
  __syncwarp();                                // every lane has read column block J
#pragma unroll
  for (int I = 0; I < G::NIT; ++I)
    if (8 * I + g < G::NWR)                    // rows >= 4 NIK are zero and never read
      *reinterpret_cast<double2*>(Wd + (8 * I + g) * WST + 8 * J + 2 * t) =
          make_double2(cacc[I][0], cacc[I][1]);
  __syncwarp();
  if constexpr (YM & 1) __nanosleep(0);
}

// Output tiles q = tile0, tile0 + step, ... of [X (NIT x NCB) | S_oo^-1
// (lower NIT) | Sd_T (lower NCB)] into the ext record xo and Sd_T so.
template <int K, class SG, int YM = 0>
__device__ __forceinline__ void out_tiles(SG Sg, const double* LI, const double* Wd, double* xo,
                                          double* so, int tile0, int step) {
  using G = Geo<K>;
  using L = ExtLayout<K>;
  constexpr int NI = G::NI, NC = G::NC, WST = G::WST, LST = G::LST;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll 1
  for (int q = tile0; q < G::NTILES; q += step) {
    if constexpr (YM & 2) __nanosleep(0);
    if constexpr (YM & 4) { if ((q & 3) == 3) __nanosleep(0); }
    if (q < G::NTX) {                          // X = L^-T W
      const int I = q / G::NCB, J = q % G::NCB;
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int ks = 0; ks < G::NIK; ++ks)
        dmma884(c0, c1, LI[(4 * ks + t) * LST + 8 * I + g], Wd[(4 * ks + t) * WST + 8 * J + g]);
      const int i = 8 * I + g, c = 8 * J + 2 * t;
      if (i < NI) {
        if (c < NC) xo[i * NC + c] = c0;
        if (c + 1 < NC) xo[i * NC + c + 1] = c1;
      }
    } else if (q < G::NTX + G::NTS) {          // S_oo^-1 = L^-T L^-1 (lower packed)
      int I = 0, r = q - G::NTX;
      while (r > I) { r -= I + 1; ++I; }
      const int J = r;
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int ks = 0; ks < G::NIK; ++ks)
        dmma884(c0, c1, LI[(4 * ks + t) * LST + 8 * I + g], LI[(4 * ks + t) * LST + 8 * J + g]);
      const int i = 8 * I + g, j = 8 * J + 2 * t;
      if (i < NI) {
        if (j <= i) xo[L::x_len + pk(i, j)] = c0;
        if (j + 1 <= i) xo[L::x_len + pk(i, j + 1)] = c1;
      }
    } else {                                   // Sd_T = S_cc - W^T W (lower tiles)
      int I = 0, r = q - G::NTX - G::NTS;
      while (r > I) { r -= I + 1; ++I; }
      const int J = r;
      // the S_cc entries first: their L2 round trip overlaps the DMMA chain
      const int a = 8 * I + g, b = 8 * J + 2 * t;
      double s0 = 0.0, s1 = 0.0;
      if (a < NC) {
        if (b <= a) s0 = Sg(cpl_local<K>(a), cpl_local<K>(b));
        if (b + 1 <= a) s1 = Sg(cpl_local<K>(a), cpl_local<K>(b + 1));
      }
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int ks = 0; ks < G::NIK; ++ks) {
        const double* wr = Wd + (4 * ks + t) * WST;
        dmma884(c0, c1, wr[8 * I + g], wr[8 * J + g]);
      }
      if (a < NC) {
        if (b <= a) so[pk(a, b)] = s0 - c0;
        if (b + 1 <= a) so[pk(a, b + 1)] = s1 - c1;
      }
    }
  }
}

}  // namespace dsw
}  // namespace mcs
