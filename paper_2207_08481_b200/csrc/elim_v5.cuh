// Left-looking (Crout) block signed-Cholesky elimination of one element's
// saddle matrix on the FP64 tensor cores (v5).
//
//   K = L J L^T,  L block lower triangular, J = diag(+-1) (the known pivot
//   signs: +1 for sigma, -1 for omega, +1 for padding)
//
// The element matrix is cut into 8x8 tiles (row-major, 64 B rows).  Only the
// PANEL (tile columns j < NPB, i.e. the pivot columns) lives in shared
// memory; the trailing block, which becomes the Schur complement, lives in
// REGISTERS of its owner warps as DMMA accumulators and goes straight to
// global memory at the end.  Per pivot column j:
//
//   panel tile  acc_ij = -K_ij + sum_{k<j} L_ik J_k L_jk^T   (one DMMA chain,
//               C in registers, 2 DMMA per k tile), then L_ij = acc_ij (-Q_j)
//               with Q_j = M_j^-T J_j, and written over K_ij in place;
//   diagonal    Y_jj = -acc_jj = M_j J_j M_j^T: signed Cholesky of the 8x8
//               tile in registers (one warp, shuffles), M_j^-1 alongside;
//   trailing    acc_ab += L_aj J_j L_bj^T for every trailing tile (a, b).
//
// Look-ahead: the warp that owns diagonal j+1 computes L_{j+1,j} first and
// goes straight on to Y_{j+1,j+1} and its Cholesky while the other warps
// finish column j, so the serial 8x8 factorisations overlap the DMMA work.
// One __syncthreads per pivot column.
//
// DMMA k-permutation: lane (g, t) feeds entries (g, 2t) and (g, 2t+1) of the
// A and B tiles to two consecutive m8n8k4 steps (k slots {2t} then {2t+1}).
// Both operands use the same permutation, so C += X Y^T is exact, operands
// come in as one 128-bit shared load per lane, and the accumulator layout
// (g, 2t..2t+1) is directly the A operand of the next product.  With 64 B
// tile rows these 128-bit loads are bank-conflict free.
#pragma once
#include "common.cuh"

namespace mcs {
namespace v5 {

#ifdef MCS_V5_PROF
__device__ unsigned long long g_v5prof[16];
#define V5T0() long long _tp = clock64()
#define V5T(i)                                                              \
  do {                                                                      \
    if ((threadIdx.x & 31) == 0) {                                          \
      long long _t = clock64();                                             \
      atomicAdd(&g_v5prof[i], (unsigned long long)(_t - _tp));              \
      _tp = _t;                                                             \
    }                                                                       \
  } while (0)
#else
#define V5T0()
#define V5T(i)
#endif

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ double rsqrt64(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  // two Newton steps: y <- y + y (1 - x y^2) / 2
  double r = fma(-x * y, y, 1.0);
  y = fma(0.5 * y, r, y);
  r = fma(-x * y, y, 1.0);
  return fma(0.5 * y, r, y);
}

__device__ __forceinline__ double flip(double v, unsigned m) {
  return __hiloint2double(__double2hiint(v) ^ (int)m, __double2loint(v));
}

// constant sources for padding entries (loads stay unconditional, so a
// prefetched value is never waited on by a select)
__device__ const double kConstants[3] = {0.0, 1.0, -1.0};
__device__ __forceinline__ const double* zero_src() { return &kConstants[0]; }
__device__ __forceinline__ const double* one_src() { return &kConstants[1]; }
__device__ __forceinline__ const double* minus_one_src() { return &kConstants[2]; }

// Row source of the panel: entries (i, j0 .. j0 + n - 1) are p[q * stride],
// the others zero (padding diagonals are set by the engine).
struct Row {
  const double* p;
  int stride;
  int n;
};

// NB tile rows, NPB pivot tile columns, W warps, NPIV real pivots (the rest of
// the 8*NPB are unit padding, +1 or -1 see PADNEG), NNEG0..NPIV-1 are the
// negative pivots.
template <int NB_, int NPB_, int W_, int NPIV_, int NNEG0_>
struct Geo {
  static constexpr int NB = NB_, NPB = NPB_, W = W_, NPIV = NPIV_, NNEG0 = NNEG0_;
  // padding pivots take the sign of the last real pivot, so that at most one
  // pivot tile (the sigma/omega boundary) has mixed signs
  static constexpr bool PADNEG = NNEG0 < NPIV;
  static constexpr int NEG_HI = PADNEG ? 8 * NPB : NPIV;
  static constexpr int THREADS = 32 * W;
  static constexpr int NTP = NPB * NB - NPB * (NPB - 1) / 2;  // panel tiles
  static constexpr int NC8 = NB - NPB;
  static constexpr int NTT = NC8 * (NC8 + 1) / 2;  // trailing tiles
  static constexpr int TPW = (NTT + W - 1) / W;
  static constexpr int SMEM = NTP * 64 + 2 * 64;   // doubles: panel + Rneg[2]
  // Crout tiles one warp takes in one column (rounded up to pairs)
  static constexpr int KA = (NB - 2 + W - 2) / (W - 1), KB = (NB - NPB + W - 1) / W;
  static constexpr int KMAX = ((KA > KB ? KA : KB) + 1) / 2 * 2;
  // sign type of pivot tile kb: 0 all +1, 1 all -1, 2 mixed
  __host__ __device__ static constexpr int ptype(int kb) {
    const int lo = 8 * kb, hi = 8 * kb + 8;
    const int nlo = lo > NNEG0 ? lo : NNEG0, nhi = hi < NEG_HI ? hi : NEG_HI;  // negatives in tile
    if (nhi <= nlo) return 0;
    return (nlo == lo && nhi == hi) ? 1 : 2;
  }
  // panel tiles in row-major order: row i holds min(i + 1, NPB) tiles
  __device__ static constexpr int rb(int i) {
    const int m = i < NPB ? i : NPB;
    return m * (m + 1) / 2 + (i - m) * NPB;
  }
  __device__ static constexpr int gp(int i, int j) { return rb(i) + j; }
  __host__ __device__ static constexpr int nmixed() {
    int n = 0;
    for (int q = 0; q < NPB; ++q) n += ptype(q) == 2;
    return n;
  }
};

template <class G>
__device__ __forceinline__ double2 ld2(const double* tile) {
  const int lane = threadIdx.x & 31;
  return *reinterpret_cast<const double2*>(tile + (lane >> 2) * 8 + 2 * (lane & 3));
}
__device__ __forceinline__ void st2(double* tile, double a, double b) {
  const int lane = threadIdx.x & 31;
  *reinterpret_cast<double2*>(tile + (lane >> 2) * 8 + 2 * (lane & 3)) = make_double2(a, b);
}

// B operand of pivot tile kb with the pivot signs J applied
template <class G>
__device__ __forceinline__ void signed_b(int kb, double2& b, unsigned m0, unsigned m1) {
  if constexpr (G::NNEG0 < G::NPIV) {
    // uniform per kb: all-negative tiles flip both, the mixed tile per lane
    bool allneg = false, mixed = false;
#pragma unroll
    for (int q = 0; q < G::NPB; ++q) {
      if (G::ptype(q) == 1) allneg |= (kb == q);
      if (G::ptype(q) == 2) mixed |= (kb == q);
    }
    if (allneg) {
      b.x = -b.x;
      b.y = -b.y;
    } else if (mixed) {
      b.x = flip(b.x, m0);
      b.y = flip(b.y, m1);
    }
  }
}

// acc (+)= sum_{k < kend} X_k J_k Y_k^T over the panel tiles X_k = L(i, k),
// Y_k = L(j, k) (two independent rows i1, i2 sharing Y when i2 >= 0)
template <class G>
__device__ __forceinline__ void chain2(const double* T, int i1, int i2, int j, int kend, double* a1,
                                       double* a2, unsigned m0, unsigned m1) {
  const double* py = T + G::rb(j) * 64;
  const double* p1 = T + G::rb(i1) * 64;
  const double* p2 = T + G::rb(i2 >= 0 ? i2 : i1) * 64;
#pragma unroll 2
  for (int kb = 0; kb < kend; ++kb) {
    double2 y = ld2<G>(py + kb * 64);
    const double2 x1 = ld2<G>(p1 + kb * 64);
    const double2 x2 = ld2<G>(p2 + kb * 64);
    signed_b<G>(kb, y, m0, m1);
    dmma(a1[0], a1[1], x1.x, y.x);
    dmma(a2[0], a2[1], x2.x, y.x);
    dmma(a1[0], a1[1], x1.y, y.y);
    dmma(a2[0], a2[1], x2.y, y.y);
  }
}

// signed Cholesky of the 8x8 tile Y (lane (g,t) holds Y[g][2t], Y[g][2t+1],
// lower triangle significant):  Y = M J M^T.  Writes Rn = -J M^-1 (row g =
// -J_g row g of M^-1) to shared memory and returns 0 or the 1-based failing
// pivot (sign different from `expect`, or zero).
// The elimination chain only needs 1/d (Y -= y_g y_c / d); the scaling
// s = |d|^-1/2 feeds the M^-1 recurrence, which runs alongside.
__device__ __forceinline__ int chol8(double y0, double y1, const signed char* expect, double* Rn) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#if defined(MCS_V5_DBG) && MCS_V5_DBG == 2
  st2(Rn, y0 * 1e-3, y1 * 1e-3);
  return 0;
#endif
  double x0 = (g == 2 * t) ? 1.0 : 0.0, x1 = (g == 2 * t + 1) ? 1.0 : 0.0;  // -> M^-1
  int bad = 0;
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const int sp = p >> 1;
    const double yp = (p & 1) ? y1 : y0;  // Y[g][p] in lanes t == sp
    const double d = __shfl_sync(0xffffffffu, yp, 4 * p + sp);
    const double yg = __shfl_sync(0xffffffffu, yp, 4 * g + sp);
    const double yc0 = __shfl_sync(0xffffffffu, yp, 8 * t + sp);
    const double yc1 = __shfl_sync(0xffffffffu, yp, 8 * t + 4 + sp);
    const double J = (double)expect[p];
    if (!(d * J > 0.0) && bad == 0) bad = p + 1;
    const double w = yg * rcp64(d);
    y0 = fma(-w, yc0, y0);
    y1 = fma(-w, yc1, y1);
    // M[g][p] = Y[g][p] J s;  M^-1 by forward elimination:
    // row p <- row p * s (1 / M[p][p] = s), rows g > p -= M[g][p] row p
    const double sc = rsqrt64(fabs(d));
    const double mg = yg * (J * sc);
    const double xp0 = __shfl_sync(0xffffffffu, x0, 4 * p + t) * sc;
    const double xp1 = __shfl_sync(0xffffffffu, x1, 4 * p + t) * sc;
    if (g == p) {
      x0 = xp0;
      x1 = xp1;
    } else if (g > p) {
      x0 = fma(-mg, xp0, x0);
      x1 = fma(-mg, xp1, x1);
    }
  }
  const double Jg = -(double)expect[g];
  st2(Rn, Jg * x0, Jg * x1);
  return bad;
}

// FETCH(bi, bj) -> this lane's two raw entries (8 bi + g, 8 bj + 2t + {0,1})
// of K in padded coordinates (diagonal tiles: lower triangle significant;
// padding: unit pivots, zero couplings).  Every raw panel entry is read once,
// straight from global memory into the DMMA accumulator that consumes it,
// so there is no copy-in phase: loads are issued at the start of a phase and
// consumed at the end of the chain they seed.
// TRAIL(i, j) -> -K_ij for the trailing block; STORE(i, j, v) receives
// v = -(K_tt - sum) = the trailing accumulator, i >= j (padded coordinates).
template <class G, class FETCH, class TRAIL, class STORE>
__device__ __forceinline__ void eliminate(FETCH fetch, TRAIL trail, STORE store, double* smem,
                                          const signed char* expect, int* bad) {
  static_assert(G::W >= 2, "v5 needs at least two warps");
  static_assert(G::nmixed() <= 1, "at most one pivot tile with mixed signs");
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  V5T0();
  double* T = smem;
  double* Rb = smem + G::NTP * 64;
  auto R = [&](int j) { return Rb + (j & 1) * 64; };
  auto tileptr = [&](int i, int j) { return T + G::gp(i, j) * 64; };

  // sign masks of the mixed pivot tile (if any) for k slots 2t, 2t+1
  unsigned m0 = 0, m1 = 0;
#pragma unroll
  for (int q = 0; q < G::NPB; ++q)
    if (G::ptype(q) == 2) {
      m0 = expect[8 * q + 2 * t] < 0 ? 0x80000000u : 0u;
      m1 = expect[8 * q + 2 * t + 1] < 0 ? 0x80000000u : 0u;
    }

  // Crout rows of column j for this warp: i0 + n nw, n = 0, 1, ... (< NB);
  // pairs (n, n+1) share a pass.  The owner of diagonal j+1 takes none.
  auto crout_rows = [&](int j, int& i0, int& nw) {
    const bool look = j + 1 < G::NPB;
    const int owner = (j + 1) % G::W;
    nw = look ? G::W - 1 : G::W;
    i0 = (look ? j + 2 : j + 1) + (look ? (warp - owner - 1 + G::W) % G::W : warp);
    if (look && warp == owner) i0 = G::NB;
  };
  // ---- prologue: diagonal 0 (warp 0), accumulators of the other warps
  if (warp == 0) {
    const double2 y = fetch(0, 0);
    const int b = chol8(y.x, y.y, expect, R(0));
    if (lane == 0 && b) atomicCAS(bad, 0, b);
  }

  // trailing accumulators acc = -K (registers); slots past NTT compute a
  // dummy copy of tile 0 so that no DMMA is predicated
  double acc[G::TPW][2];
  int ta[G::TPW], tb[G::TPW];
#pragma unroll
  for (int m = 0; m < G::TPW; ++m) {
    const int q0 = warp + m * G::W, q = q0 < G::NTT ? q0 : 0;
    int a = 0, b = 0, s = 0;
    while (s + (G::NC8 - b) <= q) {
      s += G::NC8 - b;
      ++b;
    }
    a = b + (q - s);
    ta[m] = G::NPB + a;
    tb[m] = G::NPB + b;
    acc[m][0] = trail(8 * ta[m] + g, 8 * tb[m] + 2 * t);
    acc[m][1] = trail(8 * ta[m] + g, 8 * tb[m] + 2 * t + 1);
    if (q0 >= G::NTT) ta[m] = -ta[m];  // dummy slot: computed, never stored
  }

  // look-ahead accumulators of this warp's future diagonals c = warp + m W
  // (right-looking): D_c = -K_cc + sum L_ck J L_ck^T,
  // S_c = -K_c,c-1 + sum L_ck J L_c-1,k^T, brought up to date each column
  constexpr int MW = (G::NPB + G::W - 1) / G::W;
  double D[MW][2], S[MW][2];
#pragma unroll
  for (int m = 0; m < MW; ++m) {
    const int c = warp + m * G::W;
    D[m][0] = D[m][1] = S[m][0] = S[m][1] = 0.0;
    if (c >= 1 && c < G::NPB) {
      const double2 kd = fetch(c, c), ks = fetch(c, c - 1);
      D[m][0] = -kd.x;
      D[m][1] = -kd.y;
      S[m][0] = -ks.x;
      S[m][1] = -ks.y;
    }
  }
  auto pair_update = [&](double* a, int i, int jrow, int k) {  // a += L_ik J L_jrow,k^T
    const double2 x = ld2<G>(tileptr(i, k));
    double2 y = ld2<G>(tileptr(jrow, k));
    signed_b<G>(k, y, m0, m1);
    dmma(a[0], a[1], x.x, y.x);
    dmma(a[0], a[1], x.y, y.y);
  };
  __syncthreads();
  V5T(2);

#pragma unroll 1
  for (int j = 0; j < G::NPB; ++j) {
    const bool look = j + 1 < G::NPB;
    const int owner = (j + 1) % G::W;
    if (look && warp == owner) {
      // critical path: S_{j+1}, D_{j+1} <- column j-1; L_{j+1,j} = S (-Q_j);
      // D_{j+1} += L J L^T; Cholesky -> Rn_{j+1}
      double s[2] = {0.0, 0.0}, d[2] = {0.0, 0.0};
#pragma unroll
      for (int m = 0; m < MW; ++m)
        if (warp + m * G::W == j + 1) {
          s[0] = S[m][0];
          s[1] = S[m][1];
          d[0] = D[m][0];
          d[1] = D[m][1];
        }
      if (j >= 1) {
        pair_update(s, j + 1, j, j - 1);
        pair_update(d, j + 1, j + 1, j - 1);
      }
      const double2 q = ld2<G>(R(j));
      double o0 = 0.0, o1 = 0.0;
      dmma(o0, o1, s[0], q.x);
      dmma(o0, o1, s[1], q.y);
      st2(tileptr(j + 1, j), o0, o1);
      double2 bb = make_double2(o0, o1);
      signed_b<G>(j, bb, m0, m1);
      dmma(d[0], d[1], o0, bb.x);
      dmma(d[0], d[1], o1, bb.y);
      V5T(3);
      const int b = chol8(-d[0], -d[1], expect + 8 * (j + 1), R(j + 1));
      if (lane == 0 && b) atomicCAS(bad, 0, 8 * (j + 1) + b);
      V5T(4);
    } else {
      // Crout panel tiles i >= j+2 (all of column j after the last look-ahead),
      // two rows per pass sharing the L_jk operand
      const double2 q = ld2<G>(R(j));
      int i1, nw;
      crout_rows(j, i1, nw);
#pragma unroll 1
      for (; i1 < G::NB; i1 += 2 * nw) {
        const bool two = i1 + nw < G::NB;
        const int i2 = two ? i1 + nw : i1;
        const double2 k1 = fetch(i1, j), k2 = fetch(i2, j);
        double a1[2] = {0.0, 0.0}, a2[2] = {0.0, 0.0};
        chain2<G>(T, i1, i2, j, j, a1, a2, m0, m1);
        double o0 = 0.0, o1 = 0.0, p0 = 0.0, p1 = 0.0;
        dmma(o0, o1, a1[0] - k1.x, q.x);
        dmma(p0, p1, a2[0] - k2.x, q.x);
        dmma(o0, o1, a1[1] - k1.y, q.y);
        dmma(p0, p1, a2[1] - k2.y, q.y);
        st2(tileptr(i1, j), o0, o1);
        if (two) st2(tileptr(i2, j), p0, p1);
      }
      V5T(5);
    }
    if (j >= 1) {
      // off the critical path: future look-ahead accumulators and the trailing block
#pragma unroll
      for (int m = 0; m < MW; ++m) {
        const int c = warp + m * G::W;
        if (c >= j + 2 && c < G::NPB) {
          pair_update(D[m], c, c, j - 1);
          pair_update(S[m], c, c - 1, j - 1);
        }
      }
#pragma unroll
      for (int m = 0; m < G::TPW; ++m) pair_update(acc[m], abs(ta[m]), tb[m], j - 1);
    }
    V5T(6);
    __syncthreads();
    V5T(7);
  }
#pragma unroll
  for (int m = 0; m < G::TPW; ++m) pair_update(acc[m], abs(ta[m]), tb[m], G::NPB - 1);

  // ---- trailing block out
#pragma unroll
  for (int m = 0; m < G::TPW; ++m)
    if (ta[m] >= 0) {
      const int i = 8 * ta[m] + g, jj = 8 * tb[m] + 2 * t;
      if (jj <= i) store(i, jj, acc[m][0]);
      if (jj + 1 <= i) store(i, jj + 1, acc[m][1]);
    }
  V5T(8);
}

}  // namespace v5
}  // namespace mcs
