// Blocked symmetric elimination of one element's saddle matrix on the FP64
// tensor cores (DMMA, mma.sync.m8n8k4.f64).
//
// The (padded) augmented matrix K of size 8*NB is cut into 8x8 tiles; the
// lower-triangular tiles are distributed over the W warps of the CTA
// (column-major tile order, cyclic) and live in REGISTERS in the DMMA
// accumulator layout (lane = 4*row + col/2, two doubles per lane and tile).
// Pivots are eliminated one 8x8 block at a time (block LDL^T without
// pivoting, the order the reference's factorisations imply):
//
//   A  the owner warp of the diagonal tile P inverts it (Gauss-Jordan on
//      shared memory, pivot signs checked)                       -> Pinv
//   B  every panel tile R_i = K[i, p] (i > p) is published raw to shared
//      memory together with Z_i = R_i Pinv (2 DMMA)
//   C  every trailing tile K[i, j] (i >= j > p) takes
//      K[i, j] -= Z_i R_j^T                                    (2 DMMA)
//
// two __syncthreads per 8 pivots.  After NPB pivot blocks the trailing tiles
// hold the Schur complement with the opposite sign: -S.
#pragma once
#include "common.cuh"

namespace mcs {

constexpr int TROW = 12;              // shared-memory row stride of an 8x8 tile (bank spread)
constexpr int TSZ = 8 * TROW;         // doubles per shared tile

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int NB_, int NPB_, int W_>
struct Elim {
  static constexpr int NB = NB_, NPB = NPB_, W = W_;
  static constexpr int NT = NB * (NB + 1) / 2;
  static constexpr int TPW = (NT + W - 1) / W;
  static constexpr int THREADS = 32 * W;
  // dynamic shared memory (doubles) besides the input stage
  static constexpr int SMEM_WORK = 4 * NB * TSZ + 2 * TSZ + 8 * 18;

  // column-major lower tile order: g -> (bi, bj)
  __device__ static void tile_of(int g, int& bi, int& bj) {
    int j = 0, start = 0;
    while (start + (NB - j) <= g) {
      start += NB - j;
      ++j;
    }
    bj = j;
    bi = j + (g - start);
  }
  __device__ static constexpr int gindex(int bi, int bj) { return bj * NB - bj * (bj - 1) / 2 + (bi - bj); }
};

// named CTA barriers (bar.arrive / bar.sync): the diagonal owner releases the
// other warps without anybody spinning on shared memory
__device__ __forceinline__ void named_arrive(int id, int nthreads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ double rcp64(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  y = fma(fma(-x, y, 1.0), y, y);
  return fma(fma(-x, y, 1.0), y, y);
}

// Invert the 8x8 diagonal block held by one warp in the DMMA accumulator
// layout (v0, v1 = entries (lane/4, 2*(lane%4) + {0,1})).  Gauss-Jordan on
// the augmented [Q | I] in the fraction-free (Bareiss) form
//     R_i <- (p_j R_i - R_i[j] R_j) / p_{j-1}      (i != j),
// lane = row r and a quarter of the 16 columns, rows exchanged through a
// small padded shared-memory scratch W (8 x GJS doubles).  The dependency
// chain per pivot is load -> FMA -> multiply -> store: the reciprocal of p_j
// is formed one step ahead, off the chain, and the pivot-sign checks run
// after the loop.  The pivot ratios p_j / p_{j-1} are the LDL^T pivots
// (checked against expect[j] in {+1, -1, 0}); at the end the left block is
// p_7 I and Q^-1 = right / p_7.  Writes Q^-1 to P (stride TROW); returns the
// first offending pivot (1-based) or 0.
constexpr int GJS = 18;   // scratch row stride (doubles)

__device__ __forceinline__ int warp_inverse8(double v0, double v1, double* W, double* P,
                                             const signed char* expect) {
  const int lane = threadIdx.x & 31;
  const int r = lane >> 2, qd = lane & 3, c0 = 4 * qd;
  // C layout -> scratch (left block), identity on the right
  W[r * GJS + 2 * qd] = v0;
  W[r * GJS + 2 * qd + 1] = v1;
  W[r * GJS + 8 + 2 * qd] = (2 * qd == r) ? 1.0 : 0.0;
  W[r * GJS + 8 + 2 * qd + 1] = (2 * qd + 1 == r) ? 1.0 : 0.0;
  __syncwarp();
  double m[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) m[q] = W[r * GJS + c0 + q];
  double piv[8];
  double inv_prev = 1.0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const double p = W[j * GJS + j];
    const double mr = W[r * GJS + j];
    double rj[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) rj[q] = W[j * GJS + c0 + q];
    piv[j] = p;
    __syncwarp();
    const bool keep = (r == j);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double u = fma(p, m[q], -mr * rj[q]) * inv_prev;
      m[q] = keep ? m[q] : u;
      W[r * GJS + c0 + q] = m[q];
    }
    inv_prev = rcp64(p);
    __syncwarp();
  }
  int badj = 0;
  bool neg_prev = false;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const bool neg = piv[j] < 0.0;
    const bool pos_ratio = (neg == neg_prev) && piv[j] != 0.0;
    const int s = expect[j];
    const bool ok = s > 0 ? pos_ratio : (s < 0 ? (!pos_ratio && piv[j] != 0.0) : piv[j] != 0.0);
    if (!ok && badj == 0) badj = j + 1;
    neg_prev = neg;
  }
  if (qd >= 2) {
#pragma unroll
    for (int q = 0; q < 4; ++q) P[r * TROW + c0 - 8 + q] = m[q] * inv_prev;
  }
  __syncwarp();
  return badj;
}

#ifdef MCS_PHASE_PROF
__device__ unsigned long long g_phase_prof[8 * 32];
__device__ __forceinline__ long long pclock() {
  long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)::"memory");
  return t;
}
#define PT(i) do { long long _t = pclock(); prof[i] += _t - tprev; tprev = _t; } while (0)
#else
#define PT(i) do {} while (0)
#endif

__device__ __forceinline__ void publish(double* dst, double v0, double v1) {
  const int lane = threadIdx.x & 31;
  dst[(lane >> 2) * TROW + 2 * (lane & 3)] = v0;
  dst[(lane >> 2) * TROW + 2 * (lane & 3) + 1] = v1;
}

// The elimination itself, right-looking with a one-panel look-ahead.
// `acc` holds the warp's tiles (loaded by the caller); on return the
// trailing tiles (bi, bj >= NPB) hold -S.  Per pivot block p:
//   C1  update column p+1 with (Z_p, R_p); publish R_{p+1}; the diagonal
//       owner inverts K[p+1,p+1] right away and raises `flag`
//   C2  update the remaining trailing tiles with (Z_p, R_p)
//   B   panel owners wait for the flag and form Z_{p+1} = R_{p+1} Pinv_{p+1}
//   one __syncthreads
// so the serial 8x8 inversion overlaps the bulk of the trailing update.
template <class E>
__device__ __forceinline__ void eliminate_tiles(double (&acc)[E::TPW][2], const int (&tij)[E::TPW],
                                                double* work, const signed char* expect_all,
                                                int* bad, volatile int* flag) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gr = lane >> 2, tg = lane & 3;
  double* Rb = work;                       // [2][NB] tiles
  double* Zb = work + 2 * E::NB * TSZ;     // [2][NB] tiles
  double* Pb = Zb + 2 * E::NB * TSZ;       // [2] tiles
  double* Gw = Pb + 2 * TSZ;               // 8 x GJS Gauss-Jordan scratch
#ifdef MCS_PHASE_PROF
  long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tprev = pclock();
#endif
  auto R_ = [&](int p, int i) { return Rb + ((p & 1) * E::NB + i) * TSZ; };
  auto Z_ = [&](int p, int i) { return Zb + ((p & 1) * E::NB + i) * TSZ; };
  auto P_ = [&](int p) { return Pb + (p & 1) * TSZ; };

  // the diagonal tile of column c, kept aside by its owner until inversion
  double dv0 = 0.0, dv1 = 0.0;
  auto stage_diag = [&](double v0, double v1) {
    dv0 = v0;
    dv1 = v1;
  };
  // owner warp: invert the diagonal tile, publish Pinv_c, release the others
  auto diag_inverse = [&](int c) {
    const int b = warp_inverse8(dv0, dv1, Gw, P_(c), expect_all + 8 * c);
    if (lane == 0 && b && *bad == 0) *bad = 8 * c + b;
    __threadfence_block();
    named_arrive(1, E::THREADS);       // Pinv_c published
  };
  // Z_c[i] = R_c[i] Pinv_c for the panel tiles this warp owns
  auto panel_z = [&](int c) {
    const int gd = E::gindex(c, c);
    if (warp != gd % E::W) named_sync(1, E::THREADS);   // wait for Pinv_c
    PT(6);
    for (int bi = c + 1; bi < E::NB; ++bi) {
      if ((gd + (bi - c)) % E::W != warp) continue;
      const double* R = R_(c, bi);
      const double* P = P_(c);
      double z0 = 0.0, z1 = 0.0;
#pragma unroll
      for (int kk = 0; kk < 8; kk += 4) dmma(z0, z1, R[gr * TROW + kk + tg], P[(kk + tg) * TROW + gr]);
      publish(Z_(c, bi), z0, z1);
    }
  };

  // prologue: pivot block 0
  {
    const int gd = 0;
#pragma unroll
    for (int t = 0; t < E::TPW; ++t) {
      const int g = warp + t * E::W;
      if (g == gd) stage_diag(acc[t][0], acc[t][1]);
      else if (g > gd && g < E::NB) publish(R_(0, g), acc[t][0], acc[t][1]);
    }
    if (warp == 0) diag_inverse(0);
    __syncwarp();
    panel_z(0);
    PT(7);
    __syncthreads();
    PT(1);
  }
  for (int pb = 0; pb < E::NPB; ++pb) {
    const int nx = pb + 1;                         // next pivot column
    const int g1 = E::gindex(nx, nx);              // first tile of column nx
    const int c1_end = g1 + (E::NB - nx);           // column nx = [g1, c1_end)
    const bool look = nx < E::NPB;
    PT(5);
    // ---- C1: column nx first
#pragma unroll
    for (int t = 0; t < E::TPW; ++t) {
      const int g = warp + t * E::W;
      if (g >= g1 && g < c1_end) {
        const int bi = tij[t] & 0xff, bj = tij[t] >> 8;
        const double* Z = Z_(pb, bi);
        const double* R = R_(pb, bj);
#pragma unroll
        for (int kk = 0; kk < 8; kk += 4)
          dmma(acc[t][0], acc[t][1], -Z[gr * TROW + kk + tg], R[gr * TROW + kk + tg]);
        if (look) {
          if (g == g1) stage_diag(acc[t][0], acc[t][1]);
          else publish(R_(nx, bi), acc[t][0], acc[t][1]);
        }
      }
    }
    PT(2);
    if (look && warp == g1 % E::W) diag_inverse(nx);
    PT(0);
    // ---- C2: the rest of the trailing matrix
#pragma unroll
    for (int t = 0; t < E::TPW; ++t) {
      const int g = warp + t * E::W;
      if (g >= c1_end && g < E::NT) {
        const int bi = tij[t] & 0xff, bj = tij[t] >> 8;
        const double* Z = Z_(pb, bi);
        const double* R = R_(pb, bj);
#pragma unroll
        for (int kk = 0; kk < 8; kk += 4)
          dmma(acc[t][0], acc[t][1], -Z[gr * TROW + kk + tg], R[gr * TROW + kk + tg]);
      }
    }
    PT(3);
    if (look) {
      __syncwarp();
      panel_z(nx);
    }
    PT(4);
    __syncthreads();
    PT(1);
  }
#ifdef MCS_PHASE_PROF
  if (lane == 0 && blockIdx.x == 0)
    for (int q = 0; q < 8; ++q) atomicAdd(&g_phase_prof[8 * warp + q], (unsigned long long)prof[q]);
#endif
}

}  // namespace mcs
