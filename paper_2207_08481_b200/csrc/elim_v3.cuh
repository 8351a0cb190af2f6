// Blocked symmetric elimination of one element's saddle matrix on the FP64
// tensor cores (DMMA, mma.sync.m8n8k4.f64) -- compile-time tile ownership.
//
// The padded matrix (8*NB) is cut into 8x8 tiles; the lower tiles are dealt
// cyclically (column-major order) over the W warps of a small CTA.  Every
// warp runs its own ROLE instantiation, so each tile's coordinates are
// compile-time constants: no per-tile metadata lives in registers and all
// shared-memory offsets are immediates.  That keeps a whole element in
// ~125 registers/thread at W = 4, i.e. four elements in flight per SM, which
// is what hides the per-element dependency chain (one 8x8 pivot-block
// inversion per panel).
//
// Per 8-pivot panel p (look-ahead by one panel):
//   C1  update column p+1 with (Z_p, R_p); publish R_{p+1}; the diagonal
//       owner inverts K[p+1,p+1] (Bareiss Gauss-Jordan) and releases the
//       others through a named barrier
//   C2  update the remaining trailing tiles with (Z_p, R_p)
//   B   panel owners form Z_{p+1} = R_{p+1} Pinv_{p+1} (2 DMMA per tile)
//   one CTA barrier
// After NPB panels the trailing tiles hold -S.
#pragma once
#include "elim_dmma.cuh"

namespace mcs {
namespace v3 {

constexpr int TR = 8;                 // shared tile row stride (doubles), XOR-swizzled
constexpr int TS = 64;                // doubles per shared tile

// swizzled offset of (row, col) inside a shared 8x8 tile: rows 2,3,6,7 swap
// the column halves so a DMMA fragment load (8 rows x 4 cols) hits 16
// distinct bank pairs
__device__ __forceinline__ int sw(int row, int col) { return row * TR + (col ^ ((row & 2) << 1)); }

__host__ __device__ constexpr int gcol_start(int NB, int j) { return j * NB - j * (j - 1) / 2; }
__host__ __device__ constexpr int tile_bj(int NB, int g) {
  int j = 0;
  while (gcol_start(NB, j + 1) <= g) ++j;
  return j;
}
__host__ __device__ constexpr int tile_bi(int NB, int g) {
  const int j = tile_bj(NB, g);
  return j + (g - gcol_start(NB, j));
}

template <int NB_, int NPB_, int W_>
struct Geo {
  static constexpr int NB = NB_, NPB = NPB_, W = W_;
  static constexpr int NT = NB * (NB + 1) / 2;
  static constexpr int TPW = (NT + W - 1) / W;
  static constexpr int THREADS = 32 * W;
  // shared: R[2][NB] + Z[2][NB] + P[2] tiles + GJ scratch
  static constexpr int SMEM = (4 * NB + 2) * TS + 8 * GJS;
};

// Bareiss Gauss-Jordan inverse of the 8x8 block in C layout (see
// elim_dmma.cuh); writes Q^-1 into a swizzled shared tile.
__device__ __forceinline__ int inverse8_to(double v0, double v1, double* W, double* P,
                                           const signed char* expect) {
  const int lane = threadIdx.x & 31;
  const int r = lane >> 2, qd = lane & 3, c0 = 4 * qd;
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
    for (int q = 0; q < 4; ++q) P[sw(r, c0 - 8 + q)] = m[q] * inv_prev;
  }
  __syncwarp();
  return badj;
}

#ifdef MCS_PHASE_PROF
__device__ unsigned long long g_v3prof[8 * 8];
#define V3T(i) do { long long _t = pclock(); vprof[i] += _t - tprev; tprev = _t; } while (0)
#else
#define V3T(i) do {} while (0)
#endif

// one warp role: tiles g = ROLE + t*W
template <class G, int ROLE>
struct Role {
  static constexpr int cnt() {
    int n = 0;
    for (int g = ROLE; g < G::NT; g += G::W) ++n;
    return n;
  }
  static constexpr int T = cnt();
  static constexpr int g(int t) { return ROLE + t * G::W; }
  static constexpr int bi(int t) { return tile_bi(G::NB, g(t)); }
  static constexpr int bj(int t) { return tile_bj(G::NB, g(t)); }
};

template <class G>
struct Smem {
  double* base;
  __device__ double* R(int p, int i) const { return base + ((p & 1) * G::NB + i) * TS; }
  __device__ double* Z(int p, int i) const { return base + ((2 + (p & 1)) * G::NB + i) * TS; }
  __device__ double* P(int p) const { return base + (4 * G::NB + (p & 1)) * TS; }
  __device__ double* GJ() const { return base + (4 * G::NB + 2) * TS; }
};

__device__ __forceinline__ void put(double* tile, double v0, double v1) {
  const int lane = threadIdx.x & 31, gr = lane >> 2, tg = lane & 3;
  tile[sw(gr, 2 * tg)] = v0;
  tile[sw(gr, 2 * tg + 1)] = v1;
}

// predicated DMMA (no branch around it, so tile updates stay straight-line
// code the compiler can software-pipeline); not volatile: a pure function
__device__ __forceinline__ void dmma_if(bool on, double& c0, double& c1, double a, double b) {
  asm("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "@p mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n}\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b), "r"((int)on));
}

// acc[t] -= Z_i R_j^T  (i = bi(t), j = bj(t)) when `on`
__device__ __forceinline__ void upd(bool on, double& c0, double& c1, const double* Z,
                                    const double* R) {
  const int lane = threadIdx.x & 31, gr = lane >> 2, tg = lane & 3;
#pragma unroll
  for (int kk = 0; kk < 8; kk += 4) dmma_if(on, c0, c1, -Z[sw(gr, kk + tg)], R[sw(gr, kk + tg)]);
}

// The elimination for warp role ROLE.  LOAD(i, j) returns padded entry (i, j)
// (any order); STORE(i, j, v) receives the trailing block (real rows, j <= i).
template <class G, int ROLE, class LOAD>
__device__ __forceinline__ void run_role(double (&acc)[Role<G, ROLE>::T][2], LOAD load,
                                         const Smem<G>& sm, const signed char* expect, int* bad) {
  using RL = Role<G, ROLE>;
  constexpr int T = RL::T;
  const int lane = threadIdx.x & 31, gr = lane >> 2, tg = lane & 3;
#ifdef MCS_PHASE_PROF
  long long vprof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tprev = pclock();
#endif
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const int i = RL::bi(t) * 8 + gr;
#pragma unroll
    for (int q = 0; q < 2; ++q) acc[t][q] = load(i, RL::bj(t) * 8 + 2 * tg + q);
  }
  V3T(0);
  double dv0 = 0.0, dv1 = 0.0;
  auto diag_inverse = [&](int c) {
    const int b = inverse8_to(dv0, dv1, sm.GJ(), sm.P(c), expect + 8 * c);
    if (lane == 0 && b && *bad == 0) *bad = 8 * c + b;
    __threadfence_block();
    named_arrive(1, G::THREADS);
  };
  auto panel_z = [&](int c) {
    const int owner = (c * G::NB - c * (c - 1) / 2) % G::W;
    if (ROLE != owner) named_sync(1, G::THREADS);
#pragma unroll
    for (int t = 0; t < T; ++t) {
      if (RL::bj(t) == c && RL::bi(t) > c) {
        const double* R = sm.R(c, RL::bi(t));
        const double* P = sm.P(c);
        double z0 = 0.0, z1 = 0.0;
#pragma unroll
        for (int kk = 0; kk < 8; kk += 4) dmma(z0, z1, R[sw(gr, kk + tg)], P[sw(kk + tg, gr)]);
        put(sm.Z(c, RL::bi(t)), z0, z1);
      }
    }
  };
  // prologue: pivot block 0
#pragma unroll
  for (int t = 0; t < T; ++t) {
    if (RL::bj(t) == 0) {
      if (RL::bi(t) == 0) {
        dv0 = acc[t][0];
        dv1 = acc[t][1];
      } else {
        put(sm.R(0, RL::bi(t)), acc[t][0], acc[t][1]);
      }
    }
  }
  if (ROLE == 0) diag_inverse(0);
  __syncwarp();
  panel_z(0);
  __syncthreads();
  V3T(1);
  for (int pb = 0; pb < G::NPB; ++pb) {
    const int nx = pb + 1;
    const bool look = nx < G::NPB;
    // C1: column nx (its diagonal tile is first in column-major order, so
    // the owner starts the inversion before updating the rest)
#pragma unroll
    for (int t = 0; t < T; ++t) {
      if (RL::bj(t) == nx) {
        upd(true, acc[t][0], acc[t][1], sm.Z(pb, RL::bi(t)), sm.R(pb, RL::bj(t)));
        if (look) {
          if (RL::bi(t) == nx) {
            dv0 = acc[t][0];
            dv1 = acc[t][1];
            diag_inverse(nx);
          } else {
            put(sm.R(nx, RL::bi(t)), acc[t][0], acc[t][1]);
          }
        }
      }
    }
    V3T(2);
    V3T(3);
    // C2: the rest of the trailing matrix, k-split outer so the two DMMAs of
    // a tile are far apart (no accumulator dependency stalls)
#pragma unroll
    for (int kk = 0; kk < 8; kk += 4) {
#pragma unroll
      for (int t = 0; t < T; ++t) {
        if (RL::bj(t) > nx) {
          const double* Z = sm.Z(pb, RL::bi(t));
          const double* R = sm.R(pb, RL::bj(t));
          dmma(acc[t][0], acc[t][1], -Z[sw(gr, kk + tg)], R[sw(gr, kk + tg)]);
        }
      }
    }
    V3T(4);
    if (look) {
      __syncwarp();
      panel_z(nx);
    }
    V3T(5);
    __syncthreads();
    V3T(6);
  }
#ifdef MCS_PHASE_PROF
  if (lane == 0 && blockIdx.x == 0)
    for (int q = 0; q < 8; ++q) atomicAdd(&g_v3prof[8 * ROLE + q], (unsigned long long)vprof[q]);
#endif
}

template <class G, int ROLE, class STORE>
__device__ __forceinline__ void store_role(const double (&acc)[Role<G, ROLE>::T][2], STORE store) {
  using RL = Role<G, ROLE>;
  const int lane = threadIdx.x & 31, gr = lane >> 2, tg = lane & 3;
#pragma unroll
  for (int t = 0; t < RL::T; ++t) {
    if (RL::bj(t) >= G::NPB) {
#pragma unroll
      for (int q = 0; q < 2; ++q) store(RL::bi(t) * 8 + gr, RL::bj(t) * 8 + 2 * tg + q, acc[t][q]);
    }
  }
}

// padded index -> real entry (real_entry called with ri >= rj); dummy pivots
// are unit, dummy trailing rows zero
template <int NP, int NC, int NPP, class F>
__device__ __forceinline__ double padded_entry(int i, int j, F real_entry) {
  if (i < j) { const int s = i; i = j; j = s; }
  const bool di = (i < NPP) ? (i >= NP) : (i - NPP >= NC);
  const bool dj = (j < NPP) ? (j >= NP) : (j - NPP >= NC);
  if (di || dj) return (i == j && i < NPP) ? 1.0 : 0.0;
  return real_entry(i < NPP ? i : NP + (i - NPP), j < NPP ? j : NP + (j - NPP));
}

// run warp role `warp` (compile-time dispatch over 0..W-1)
template <class G, int R = 0, class LOAD, class STORE>
__device__ __forceinline__ void dispatch(int warp, LOAD load, STORE store, const Smem<G>& sm,
                                         const signed char* expect, int* bad) {
  if constexpr (R < G::W) {
    if (warp == R) {
      double acc[Role<G, R>::T][2];
      run_role<G, R>(acc, load, sm, expect, bad);
      store_role<G, R>(acc, store);
    } else {
      dispatch<G, R + 1>(warp, load, store, sm, expect, bad);
    }
  }
}

}  // namespace v3
}  // namespace mcs
