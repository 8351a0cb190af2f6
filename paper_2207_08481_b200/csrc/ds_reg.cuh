// Register-resident double Schur complement, one warp per element (SURVEY
// §8a row A4; the reference's sequence condensation.py:207-226 on the
// element-local S_T):
//   S_oo = L L^T,  X = S_oo^-1 S_oc,  S_oo^-1,  Sd_T = S_cc - S_co X.
//
// Every matrix is cut into 8x8 tiles held in the DMMA "row layout" (lane
// (g, t) owns entries [g][2t], [g][2t+1]), which is at once the m8n8k4
// accumulator layout and a valid operand layout of C += X Y^T (two m8n8k4
// steps over the k slots 2t and 2t+1).  With S_co (coupling x interior) and
// an identity block as right-hand sides, ONE right-looking sweep over the
// pivot tiles j of S_oo produces, in registers,
//   W^T  = S_co L^-T        (bt[c][j],  NCB x NP tiles)
//   L^-T = I    L^-T        (it[J][I],  I >= J)
// and then
//   Sd_T   = S_cc - W^T W          (X Y^T of bt rows)
//   X      = L^-T W     = it bt^T  (row tile I, sum over I' >= I)
//   S_oo^-1 = L^-T L^-1 = it it^T.
// Per step j: the 8x8 diagonal tile is factorised with shuffles (chol8m,
// which returns M_j^-1), the panel L_ij = A_ij M_j^-T and every trailing
// update are DMMA pairs on register operands.  The trailing part of S_oo
// lives in per-lane private shared-memory slots (lane l only ever touches
// bytes [16 l, 16 l + 16) of a tile, so no warp synchronisation is needed);
// nothing else leaves the registers: no W / L^-1 staging, no operand
// reloads, ~770 DMMAs and ~3k instructions per element at k = 6 against
// 864 DMMAs and 12.4k instructions for the shared-memory kernel of
// ds_warp.cuh.
#pragma once
#include "common.cuh"

namespace mcs {
namespace dsr {

template <int K>
struct Geo {
  using Z = Sizes<K>;
  static constexpr int NI = Z::n_int, NC = Z::ncpl, NEM = Z::n_em;
  static constexpr int NP = (NI + 7) / 8;                  // pivot tiles of S_oo
  static constexpr int NCB = (NC + 7) / 8;                 // row tiles of S_co / Sd
  static constexpr int NT = NP * (NP + 1) / 2;             // lower tiles of S_oo
  static constexpr int PER_WARP = NT * 64;                 // doubles of shared memory per warp
  __host__ __device__ static constexpr int q(int i, int j) { return i * (i + 1) / 2 + j; }
};

__device__ __forceinline__ void mma_xyt(double2& c, double2 x, double2 y) {
  dmma884(c.x, c.y, x.x, y.x);
  dmma884(c.x, c.y, x.y, y.y);
}
// the first m8n8k4 step only (k slots 0, 2, 4, 6): a k tile whose odd columns are zero
__device__ __forceinline__ void mma_xyt_even(double2& c, double2 x, double2 y) {
  dmma884(c.x, c.y, x.x, y.x);
}
// HALF ? even k slots only : both steps
template <bool HALF>
__device__ __forceinline__ void mma_tile(double2& c, double2 x, double2 y) {
  if constexpr (HALF) mma_xyt_even(c, x, y);
  else mma_xyt(c, x, y);
}

// Positions of the N pivot dofs in NP = ceil(N / 8) tiles.  When the last
// tile holds REM <= 4 dofs (k = 6: 35 = 4 * 8 + 3; the microbench: 60 =
// 7 * 8 + 4) they sit on its EVEN slots and the odd slots are padding
// (identity rows): every product that contracts over that tile then needs
// only the first of its two m8n8k4 steps (HALF).
template <int N>
struct PivMap {
  static constexpr int NP = (N + 7) / 8, REM = N - 8 * (NP - 1);
  static constexpr bool HALF = REM <= 4 && NP > 1;
  // dof at slot s of tile `tile`, -1 for padding
  __host__ __device__ static constexpr int dof(int tile, int s) {
    if (tile < NP - 1) return 8 * tile + s;          // full tiles: no padding
    if (HALF) return (s % 2 == 0 && s / 2 < REM) ? 8 * tile + s / 2 : -1;
    return s < REM ? 8 * tile + s : -1;
  }
};

// Cholesky M M^T = Y of one SPD 8x8 tile in the row layout (lower triangle
// significant), returned as M^-1 in the row layout.  With Y = Lu D Lu^T (Lu
// unit lower), M^-1 = D^-1/2 Lu^-1: the elimination of the tile and the
// forward elimination of an identity (-> Lu^-1) share the multipliers
// w = Y[g][p] / d_p, so a pivot costs one reciprocal, one multiply and four
// fmas per lane; the row scaling d_g^-1/2 is ONE rsqrt per lane at the end
// (lane (g, t) keeps the pivot of its own row).  The NEXT pivot
// d' = Y[p+1][p+1] - Y[p+1][p]^2 / d is formed ahead of the tile update from
// two extra shuffles (the same fma the update performs, so the value is
// bitwise the one the update leaves in the tile): the reciprocal chain
// (fma -> rcp) and the update chain (shuffle -> fma) run side by side
// instead of end to end.
// bad: first non-positive pivot (1-based, offset by base), 0 if none yet.
__device__ __forceinline__ double2 chol8m(double y0, double y1, int& bad, int base) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double x0 = (g == 2 * t) ? 1.0 : 0.0, x1 = (g == 2 * t + 1) ? 1.0 : 0.0;
  double d = __shfl_sync(0xffffffffu, y0, 0);
  double r = rcp64(d);
  double dg = 1.0;                                         // the pivot of row g
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const int sp = p >> 1;
    const double yp = (p & 1) ? y1 : y0;                   // Y[g][p] in lanes t == sp
    const double yg = __shfl_sync(0xffffffffu, yp, 4 * g + sp);
    const double yc0 = __shfl_sync(0xffffffffu, yp, 8 * t + sp);
    const double yc1 = __shfl_sync(0xffffffffu, yp, 8 * t + 4 + sp);
    double dn = 1.0, rn = 1.0;
    if (p < 7) {
      const double e = __shfl_sync(0xffffffffu, yp, 4 * (p + 1) + sp);
      const double f = __shfl_sync(0xffffffffu, ((p + 1) & 1) ? y1 : y0, 4 * (p + 1) + ((p + 1) >> 1));
      dn = fma(-(e * r), e, f);
      rn = rcp64(dn);
    }
    if (!(d > 0.0) && bad == 0) bad = base + p + 1;
    dg = (g == p) ? d : dg;
    const double w = yg * r;                               // Lu[g][p]
    y0 = fma(-w, yc0, y0);
    y1 = fma(-w, yc1, y1);
    const double xp0 = __shfl_sync(0xffffffffu, x0, 4 * p + t);
    const double xp1 = __shfl_sync(0xffffffffu, x1, 4 * p + t);
    if (g > p) {
      x0 = fma(-w, xp0, x0);
      x1 = fma(-w, xp1, x1);
    }
    d = dn;
    r = rn;
  }
  const double sc = rsqrt_nr(dg);
  return make_double2(x0 * sc, x1 * sc);
}

// Variant with the scaling d^-1/2 taken per pivot inside the loop (eight
// rsqrt per tile, twice the FP64 instructions, but no rsqrt after the last
// pivot): measured faster in the k = 5, 6 double Schur, slower in the fused
// kernel and the microbench.
__device__ __forceinline__ double2 chol8m_rs(double y0, double y1, int& bad, int base) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double x0 = (g == 2 * t) ? 1.0 : 0.0, x1 = (g == 2 * t + 1) ? 1.0 : 0.0;
  double d = __shfl_sync(0xffffffffu, y0, 0);
  double r = rcp64(d);
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const int sp = p >> 1;
    const double yp = (p & 1) ? y1 : y0;                   // Y[g][p] in lanes t == sp
    const double yg = __shfl_sync(0xffffffffu, yp, 4 * g + sp);
    const double yc0 = __shfl_sync(0xffffffffu, yp, 8 * t + sp);
    const double yc1 = __shfl_sync(0xffffffffu, yp, 8 * t + 4 + sp);
    double dn = 1.0, rn = 1.0;
    if (p < 7) {
      const double e = __shfl_sync(0xffffffffu, yp, 4 * (p + 1) + sp);
      const double f = __shfl_sync(0xffffffffu, ((p + 1) & 1) ? y1 : y0, 4 * (p + 1) + ((p + 1) >> 1));
      dn = fma(-(e * r), e, f);
      rn = rcp64(dn);
    }
    if (!(d > 0.0) && bad == 0) bad = base + p + 1;
    const double w = yg * r;
    y0 = fma(-w, yc0, y0);
    y1 = fma(-w, yc1, y1);
    const double sc = rsqrt_nr(d);
    const double mg = yg * sc;                             // M[g][p]
    const double xp0 = __shfl_sync(0xffffffffu, x0, 4 * p + t) * sc;
    const double xp1 = __shfl_sync(0xffffffffu, x1, 4 * p + t) * sc;
    if (g == p) {
      x0 = xp0;
      x1 = xp1;
    } else if (g > p) {
      x0 = fma(-mg, xp0, x0);
      x1 = fma(-mg, xp1, x1);
    }
    d = dn;
    r = rn;
  }
  return make_double2(x0, x1);
}

// no-op step hook of sweep()
struct NoSync {
  __device__ __forceinline__ void operator()(int) const {}
};

// The right-looking sweep over the NP pivot tiles of the SPD matrix A whose
// lower tiles sit NEGATED in this lane's private slots Tl + q(i, j) * 64
// (padding: -1 on the diagonal): with -A stored, the panel product yields
// -L_ij, the only form the updates need, and no operand is ever negated.  bt[c][j]: the NCB x NP right-hand-side tiles, replaced by
// W^T = B L^-T.  IT: also it[J][I] = (L^-T) tiles (I >= J) from an identity
// right-hand side.  bad: first non-positive pivot (1-based), 0 if none.
// named barrier over a pair of warps (ids 1..15; 0 is __syncthreads)
struct PairSync {
  int id;
  __device__ __forceinline__ void operator()(int) const {
    asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory");
  }
};

// the same barrier before the first pivot tile only (the pair starts every
// element together and drifts afterwards)
struct PairSync0 {
  int id;
  __device__ __forceinline__ void operator()(int j) const {
    if (j == 0) asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory");
  }
};

// sync(j) runs before pivot tile j is factorised: the kernels pair the two
// warps of an SM sub-partition with a named barrier there, so that their
// latency-bound factorisations coincide and their DMMA bursts share the
// FP64 pipe (a warp streaming DMMAs starves a co-resident warp's dependent
// FP64 chain: tools/dmma_prio.cu; unsynchronised, two warps serialise).
// HALF: the last pivot tile's odd slots are padding (PivMap): its diagonal
// products take one m8n8k4 step.
template <int NP, int NCB, bool IT, class SY = NoSync, bool RS = false, bool HALF = false>
__device__ __forceinline__ void sweep(double* __restrict__ Tl, double2 (&bt)[NCB][NP],
                                      double2 (&it)[IT ? NP : 1][IT ? NP : 1], int& bad,
                                      SY sync = SY()) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  auto q = [](int i, int j) { return i * (i + 1) / 2 + j; };
  if constexpr (IT) {
#pragma unroll
    for (int a = 0; a < NP; ++a)
#pragma unroll
      for (int b = 0; b < NP; ++b) it[a][b] = make_double2(0.0, 0.0);
  }
  const double2 eye = make_double2(g == 2 * t ? 1.0 : 0.0, g == 2 * t + 1 ? 1.0 : 0.0);
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    sync(j);
    const double2 dj = *reinterpret_cast<const double2*>(Tl + q(j, j) * 64);
    const double2 mi = RS ? chol8m_rs(-dj.x, -dj.y, bad, 8 * j)
                          : chol8m(-dj.x, -dj.y, bad, 8 * j);   // M_j^-1
    // panel: -L_ij = (-A_ij) M_j^-T
    double2 ln[NP];
#pragma unroll
    for (int i = j + 1; i < NP; ++i) {
      double2 o = make_double2(0.0, 0.0);
      mma_xyt(o, *reinterpret_cast<const double2*>(Tl + q(i, j) * 64), mi);
      ln[i] = o;
    }
    // the next diagonal tile first: its factorisation heads the critical path
    if (j + 1 < NP) {
      double2 c = *reinterpret_cast<const double2*>(Tl + q(j + 1, j + 1) * 64);
      mma_xyt(c, ln[j + 1], ln[j + 1]);
      *reinterpret_cast<double2*>(Tl + q(j + 1, j + 1) * 64) = c;
    }
    // right-hand sides: W^T_cj = B_cj M_j^-T, (L^-T)_Jj likewise (J <= j)
#pragma unroll
    for (int c = 0; c < NCB; ++c) {
      double2 o = make_double2(0.0, 0.0);
      if (HALF && j == NP - 1) mma_xyt_even(o, bt[c][j], mi);
      else mma_xyt(o, bt[c][j], mi);
      bt[c][j] = o;
    }
    if constexpr (IT) {
#pragma unroll
      for (int J = 0; J <= j; ++J) {
        double2 o = make_double2(0.0, 0.0);
        // (HALF, J == j: the padding rows of this tile come out zero instead
        // of unit rows; they are never stored nor multiplied into stored ones)
        if (HALF && j == NP - 1) mma_xyt_even(o, J == j ? eye : it[J][j], mi);
        else mma_xyt(o, J == j ? eye : it[J][j], mi);
        it[J][j] = o;
      }
    }
    // trailing updates with column j: -A_ik += (-L_ij) (-L_kj)^T
#pragma unroll
    for (int i = j + 1; i < NP; ++i) {
#pragma unroll
      for (int k = j + 1; k <= i; ++k) {
        if (i == j + 1 && k == j + 1) continue;            // done above
        double2 c = *reinterpret_cast<const double2*>(Tl + q(i, k) * 64);
        mma_xyt(c, ln[i], ln[k]);
        *reinterpret_cast<double2*>(Tl + q(i, k) * 64) = c;
      }
#pragma unroll
      for (int c = 0; c < NCB; ++c) mma_xyt(bt[c][i], bt[c][j], ln[i]);
      if constexpr (IT) {
#pragma unroll
        for (int J = 0; J <= j; ++J) mma_xyt(it[J][i], it[J][j], ln[i]);
      }
    }
  }
}

// One element.  sym(a, b): entry (a, b) of the symmetric S_T (global or
// shared memory); T: this warp's NT private tile slots (16-byte aligned).
// Returns false if S_oo is not positive definite.
// ALIAS: the tile slots T overlap memory that sym() reads for S_oo and S_co
// (the fused k = 5, 6 kernel puts them over the interior rows of the packed
// S_T): every such entry is loaded into registers before the first slot is
// written.  The S_cc entries read at the end must lie outside T.
template <int K, class SYM, class SY = NoSync, bool RS = false, bool ALIAS = false, bool SDLAST = false>
__device__ __forceinline__ bool element(SYM sym, double* __restrict__ T,
                                        double* __restrict__ xo, double* __restrict__ so,
                                        SY sync = SY()) {
  using G = Geo<K>;
  using L = ExtLayout<K>;
  constexpr int NI = G::NI, NC = G::NC, NEM = G::NEM, NP = G::NP, NCB = G::NCB;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double* Tl = T + 2 * lane;
  // ---- loads: S_co tiles into registers, S_oo lower tiles into the slots
  double2 bt[NCB][NP];
#pragma unroll
  for (int c = 0; c < NCB; ++c) {
    const int row = 8 * c + g, a = cpl_local<K>(row);
#pragma unroll
    for (int i = 0; i < NP; ++i) {
      const int col = 8 * i + 2 * t;
      double2 v = make_double2(0.0, 0.0);
      if (row < NC) {
        if (col < NI) v.x = sym(a, NEM + col);
        if (col + 1 < NI) v.y = sym(a, NEM + col + 1);
      }
      bt[c][i] = v;
    }
  }
  if constexpr (ALIAS) {
    double2 a0[G::NT];
#pragma unroll
    for (int i = 0; i < NP; ++i)
#pragma unroll
      for (int j = 0; j <= i; ++j) {
        const int r = 8 * i + g, c0 = 8 * j + 2 * t;
        double2 v;
        v.x = (r < NI && c0 < NI) ? -sym(NEM + r, NEM + c0) : (r == c0 ? -1.0 : 0.0);
        v.y = (r < NI && c0 + 1 < NI) ? -sym(NEM + r, NEM + c0 + 1) : (r == c0 + 1 ? -1.0 : 0.0);
        a0[G::q(i, j)] = v;
      }
    __syncwarp();                          // every lane holds its S_co and S_oo entries
#pragma unroll
    for (int q = 0; q < G::NT; ++q) *reinterpret_cast<double2*>(Tl + q * 64) = a0[q];
  } else {
#pragma unroll
  for (int i = 0; i < NP; ++i)
#pragma unroll
    for (int j = 0; j <= i; ++j) {
      const int r = 8 * i + g, c0 = 8 * j + 2 * t;
      double2 v;
      v.x = (r < NI && c0 < NI) ? -sym(NEM + r, NEM + c0) : (r == c0 ? -1.0 : 0.0);
      v.y = (r < NI && c0 + 1 < NI) ? -sym(NEM + r, NEM + c0 + 1) : (r == c0 + 1 ? -1.0 : 0.0);
      *reinterpret_cast<double2*>(Tl + G::q(i, j) * 64) = v;
    }

  }
  double2 it[NP][NP];
  int bad = 0;
  sweep<NP, NCB, true, SY, RS>(Tl, bt, it, bad, sync);

  if constexpr (!SDLAST) {
  // ---- Sd_T = S_cc - W^T W (lower tiles), S_cc loaded ahead of each chain
#pragma unroll
  for (int c = 0; c < NCB; ++c) {
    const int row = 8 * c + g, a = cpl_local<K>(row);
#pragma unroll
    for (int d = 0; d <= c; ++d) {
      const int col = 8 * d + 2 * t;
      double s0 = 0.0, s1 = 0.0;
      if (row < NC) {
        if (col <= row) s0 = sym(a, cpl_local<K>(col));
        if (col + 1 <= row) s1 = sym(a, cpl_local<K>(col + 1));
      }
      double2 o = make_double2(0.0, 0.0);
#pragma unroll
      for (int j = 0; j < NP; ++j) mma_xyt(o, bt[c][j], bt[d][j]);
      if (row < NC) {
        if (col <= row) so[pk(row, col)] = s0 - o.x;
        if (col + 1 <= row) so[pk(row, col + 1)] = s1 - o.y;
      }
    }
  }
  }
  // ---- X = L^-T W (row tile I: sum over I' >= I), row-major n_int x ncpl
#pragma unroll
  for (int I = 0; I < NP; ++I) {
    const int row = 8 * I + g;
#pragma unroll
    for (int c = 0; c < NCB; ++c) {
      double2 o = make_double2(0.0, 0.0);
#pragma unroll
      for (int Ip = I; Ip < NP; ++Ip) mma_xyt(o, it[I][Ip], bt[c][Ip]);
      const int col = 8 * c + 2 * t;
      if (row < NI) {
        if constexpr (NC % 2 == 0) {
          if (col < NC) *reinterpret_cast<double2*>(xo + row * NC + col) = o;
        } else {
          if (col < NC) xo[row * NC + col] = o.x;
          if (col + 1 < NC) xo[row * NC + col + 1] = o.y;
        }
      }
    }
  }
  // ---- S_oo^-1 = L^-T L^-1 (lower packed)
#pragma unroll
  for (int I = 0; I < NP; ++I) {
    const int row = 8 * I + g;
#pragma unroll
    for (int Iq = 0; Iq <= I; ++Iq) {
      double2 o = make_double2(0.0, 0.0);
#pragma unroll
      for (int Ip = I; Ip < NP; ++Ip) mma_xyt(o, it[I][Ip], it[Iq][Ip]);
      const int col = 8 * Iq + 2 * t;
      if (row < NI) {
        if (col <= row) xo[L::x_len + pk(row, col)] = o.x;
        if (col + 1 <= row) xo[L::x_len + pk(row, col + 1)] = o.y;
      }
    }
  }
  // ---- SDLAST (S_T in global memory): Sd_T = S_cc - W^T W last: `it` is
  // dead by now, and the S_cc entries of tile row c + 1 are requested before
  // the DMMA chains of row c (a single chain, ~260 clk, does not cover an L2
  // round trip).  With S_T in shared memory (fused phase D) Sd_T first is
  // 1.5% faster.
  if constexpr (SDLAST) {
    double2 cur[NCB], nxt[NCB];
    auto load_row = [&](int c, double2 (&dst)[NCB]) {
      const int row = 8 * c + g, a = cpl_local<K>(row);
#pragma unroll
      for (int d = 0; d < NCB; ++d) {
        if (d > c) continue;
        const int col = 8 * d + 2 * t;
        double2 v = make_double2(0.0, 0.0);
        if (row < NC) {
          if (col <= row) v.x = sym(a, cpl_local<K>(col));
          if (col + 1 <= row) v.y = sym(a, cpl_local<K>(col + 1));
        }
        dst[d] = v;
      }
    };
    load_row(0, cur);
#pragma unroll
    for (int c = 0; c < NCB; ++c) {
      if (c + 1 < NCB) load_row(c + 1, nxt);
      const int row = 8 * c + g;
#pragma unroll
      for (int d = 0; d <= c; ++d) {
        double2 o = make_double2(0.0, 0.0);
#pragma unroll
        for (int j = 0; j < NP; ++j) mma_xyt(o, bt[c][j], bt[d][j]);
        const int col = 8 * d + 2 * t;
        if (row < NC) {
          if (col <= row) so[pk(row, col)] = cur[d].x - o.x;
          if (col + 1 <= row) so[pk(row, col + 1)] = cur[d].y - o.y;
        }
      }
#pragma unroll
      for (int d = 0; d < NCB; ++d) cur[d] = nxt[d];
    }
  }
  return __all_sync(0xffffffffu, bad == 0);
}

// The same with the pivot dofs placed by PivMap (k = 6: the three interior
// dofs of the last tile on its even slots, products over it in one m8n8k4
// step).  Kept apart from element(): the fused k <= 4 kernel is sensitive to
// the code around its phase D (+-1-2% from equivalent index arithmetic).
// ALIAS: the tile slots T overlap memory that sym() reads for S_oo and S_co
// (the fused k = 5, 6 kernel puts them over the interior rows of the packed
// S_T): every such entry is loaded into registers before the first slot is
// written.  The S_cc entries read at the end must lie outside T.
template <int K, class SYM, class SY = NoSync, bool RS = false, bool ALIAS = false, bool SDLAST = false>
__device__ __forceinline__ bool element_pm(SYM sym, double* __restrict__ T,
                                        double* __restrict__ xo, double* __restrict__ so,
                                        SY sync = SY()) {
  using G = Geo<K>;
  using L = ExtLayout<K>;
  using PM = PivMap<G::NI>;
  constexpr int NC = G::NC, NEM = G::NEM, NP = G::NP, NCB = G::NCB;
  constexpr bool HALF = PM::HALF;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double* Tl = T + 2 * lane;
  // ---- loads: S_co tiles into registers, S_oo lower tiles into the slots
  // (interior dof of row g / columns 2t, 2t + 1 of pivot tile i: PivMap)
  double2 bt[NCB][NP];
#pragma unroll
  for (int c = 0; c < NCB; ++c) {
    const int row = 8 * c + g, a = cpl_local<K>(row);
#pragma unroll
    for (int i = 0; i < NP; ++i) {
      const int d0 = PM::dof(i, 2 * t), d1 = PM::dof(i, 2 * t + 1);
      double2 v = make_double2(0.0, 0.0);
      if (row < NC) {
        if (d0 >= 0) v.x = sym(a, NEM + d0);
        if (d1 >= 0) v.y = sym(a, NEM + d1);
      }
      bt[c][i] = v;
    }
  }
  auto soo_tile = [&](int i, int j) {
    const int rd = PM::dof(i, g), c0 = PM::dof(j, 2 * t), c1 = PM::dof(j, 2 * t + 1);
    double2 v;
    v.x = (rd >= 0 && c0 >= 0) ? -sym(NEM + rd, NEM + c0) : ((i == j && g == 2 * t) ? -1.0 : 0.0);
    v.y = (rd >= 0 && c1 >= 0) ? -sym(NEM + rd, NEM + c1) : ((i == j && g == 2 * t + 1) ? -1.0 : 0.0);
    return v;
  };
  if constexpr (ALIAS) {
    double2 a0[G::NT];
#pragma unroll
    for (int i = 0; i < NP; ++i)
#pragma unroll
      for (int j = 0; j <= i; ++j) a0[G::q(i, j)] = soo_tile(i, j);
    __syncwarp();                          // every lane holds its S_co and S_oo entries
#pragma unroll
    for (int q = 0; q < G::NT; ++q) *reinterpret_cast<double2*>(Tl + q * 64) = a0[q];
  } else {
#pragma unroll
    for (int i = 0; i < NP; ++i)
#pragma unroll
      for (int j = 0; j <= i; ++j) *reinterpret_cast<double2*>(Tl + G::q(i, j) * 64) = soo_tile(i, j);
  }
  double2 it[NP][NP];
  int bad = 0;
  sweep<NP, NCB, true, SY, RS, HALF>(Tl, bt, it, bad, sync);

  // products that contract over the last pivot tile take one m8n8k4 step when
  // its odd slots are padding
  auto mma_p = [&](double2& o, double2 x, double2 y, int ktile) {
    if (HALF && ktile == NP - 1) mma_xyt_even(o, x, y);
    else mma_xyt(o, x, y);
  };
  if constexpr (!SDLAST) {
  // ---- Sd_T = S_cc - W^T W (lower tiles), S_cc loaded ahead of each chain
#pragma unroll
  for (int c = 0; c < NCB; ++c) {
    const int row = 8 * c + g, a = cpl_local<K>(row);
#pragma unroll
    for (int d = 0; d <= c; ++d) {
      const int col = 8 * d + 2 * t;
      double s0 = 0.0, s1 = 0.0;
      if (row < NC) {
        if (col <= row) s0 = sym(a, cpl_local<K>(col));
        if (col + 1 <= row) s1 = sym(a, cpl_local<K>(col + 1));
      }
      double2 o = make_double2(0.0, 0.0);
#pragma unroll
      for (int j = 0; j < NP; ++j) mma_p(o, bt[c][j], bt[d][j], j);
      if (row < NC) {
        if (col <= row) so[pk(row, col)] = s0 - o.x;
        if (col + 1 <= row) so[pk(row, col + 1)] = s1 - o.y;
      }
    }
  }
  }
  // ---- X = L^-T W (row tile I: sum over I' >= I), row-major n_int x ncpl
#pragma unroll
  for (int I = 0; I < NP; ++I) {
    const int row = PM::dof(I, g);
#pragma unroll
    for (int c = 0; c < NCB; ++c) {
      double2 o = make_double2(0.0, 0.0);
#pragma unroll
      for (int Ip = I; Ip < NP; ++Ip) mma_p(o, it[I][Ip], bt[c][Ip], Ip);
      const int col = 8 * c + 2 * t;
      if (row >= 0) {
        if constexpr (NC % 2 == 0) {
          if (col < NC) *reinterpret_cast<double2*>(xo + row * NC + col) = o;
        } else {
          if (col < NC) xo[row * NC + col] = o.x;
          if (col + 1 < NC) xo[row * NC + col + 1] = o.y;
        }
      }
    }
  }
  // ---- S_oo^-1 = L^-T L^-1 (lower packed)
#pragma unroll
  for (int I = 0; I < NP; ++I) {
    const int row = PM::dof(I, g);
#pragma unroll
    for (int Iq = 0; Iq <= I; ++Iq) {
      double2 o = make_double2(0.0, 0.0);
#pragma unroll
      for (int Ip = I; Ip < NP; ++Ip) mma_p(o, it[I][Ip], it[Iq][Ip], Ip);
      const int c0 = PM::dof(Iq, 2 * t), c1 = PM::dof(Iq, 2 * t + 1);
      if (row >= 0) {
        if (c0 >= 0 && c0 <= row) xo[L::x_len + pk(row, c0)] = o.x;
        if (c1 >= 0 && c1 <= row) xo[L::x_len + pk(row, c1)] = o.y;
      }
    }
  }
  // ---- SDLAST (S_T in global memory): Sd_T = S_cc - W^T W last: `it` is
  // dead by now, and the S_cc entries of tile row c + 1 are requested before
  // the DMMA chains of row c (a single chain, ~260 clk, does not cover an L2
  // round trip).  With S_T in shared memory (fused phase D) Sd_T first is
  // 1.5% faster.
  if constexpr (SDLAST) {
    double2 cur[NCB], nxt[NCB];
    auto load_row = [&](int c, double2 (&dst)[NCB]) {
      const int row = 8 * c + g, a = cpl_local<K>(row);
#pragma unroll
      for (int d = 0; d < NCB; ++d) {
        if (d > c) continue;
        const int col = 8 * d + 2 * t;
        double2 v = make_double2(0.0, 0.0);
        if (row < NC) {
          if (col <= row) v.x = sym(a, cpl_local<K>(col));
          if (col + 1 <= row) v.y = sym(a, cpl_local<K>(col + 1));
        }
        dst[d] = v;
      }
    };
    load_row(0, cur);
#pragma unroll
    for (int c = 0; c < NCB; ++c) {
      if (c + 1 < NCB) load_row(c + 1, nxt);
      const int row = 8 * c + g;
#pragma unroll
      for (int d = 0; d <= c; ++d) {
        double2 o = make_double2(0.0, 0.0);
#pragma unroll
        for (int j = 0; j < NP; ++j) mma_p(o, bt[c][j], bt[d][j], j);
        const int col = 8 * d + 2 * t;
        if (row < NC) {
          if (col <= row) so[pk(row, col)] = cur[d].x - o.x;
          if (col + 1 <= row) so[pk(row, col + 1)] = cur[d].y - o.y;
        }
      }
#pragma unroll
      for (int d = 0; d < NCB; ++d) cur[d] = nxt[d];
    }
  }
  return __all_sync(0xffffffffu, bad == 0);
}

}  // namespace dsr
}  // namespace mcs
