// Batched SPD Schur complement S = B^T A^-1 B on the FP64 tensor cores
// (BASELINE config 5: n = 60, m = 36; the reference
// idiom is cho_factor / cho_solve / B^T X, condensation.py:216-224).
//
// Two warps per element (one 64-thread CTA, persistent over elements), two
// phases, every matrix cut into 8x8 tiles (n padded to 8*NP with unit
// diagonal, m to 8*NCB with zero columns):
//
//  1. Cholesky of A, right-looking, in shared memory (36 lower tiles at
//     n = 60).  Per pivot column j: the diagonal tile is factorised by a
//     register-redundant 8x8 Cholesky (chol8r), which leaves
//     R_j = -M_j^-1 in place of the tile; the panel L_ij = A_ij M_j^-T is
//     one DMMA pair per tile; the trailing update A_ik -= L_ij L_kj^T is
//     one DMMA pair per tile.  Look-ahead: warp 0 updates the next diagonal
//     tile first and factorises it while warp 1 finishes the trailing
//     block, so the serial 8x8 factorisation overlaps the tensor-core work.
//  2. W^T = B^T L^-T and S = W^T W with B^T held in REGISTERS (warp 0 owns
//     column blocks c < C1, warp 1 the rest): per block row j,
//     W^T_cj = B^T_cj M_j^-T, S_cd += W^T_cj (W^T_dj)^T, and the
//     right-looking update B^T_ci -= W^T_cj L_ij^T for i > j.  The DMMA
//     accumulator layout (lane (g,t) owns row g, columns 2t, 2t+1) is the
//     operand layout of every product here (both operands take k slots 2t,
//     2t+1 in two m8n8k4 steps), so W^T, S and B^T never leave registers;
//     warp 0 publishes its W^T_j tiles in shared memory for the cross
//     blocks S_cd (c >= C1 > d) that warp 1 accumulates.
//
// The next element's packed A (14.6 KB at n = 60) arrives by one 1-D bulk
// copy (TMA engine) during phase 2 and its B^T is loaded into registers
// during phase 1, so the HBM traffic overlaps the arithmetic.
#include <cstdlib>

#include "ds_reg.cuh"
#include "elim_v5.cuh"

#ifndef MCS_MICRO_YM
#define MCS_MICRO_YM 0
#endif

namespace mcs {
namespace micro {

#ifdef MCS_MICRO_PROF
// per-phase clock accounting (tools/micro_prof.cu): [warp][phase]
__device__ unsigned long long g_prof[2][8];
#define MP0() long long _tp = clock64()
#define MP(w, i)                                                           \
  do {                                                                     \
    if ((threadIdx.x & 31) == 0) {                                         \
      long long _t = clock64();                                            \
      atomicAdd(&g_prof[w][i], (unsigned long long)(_t - _tp));            \
      _tp = _t;                                                            \
    }                                                                      \
  } while (0)
#else
#define MP0()
#define MP(w, i)
#endif

__device__ __forceinline__ void dmma(double2& c, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c.x), "+d"(c.y)
      : "d"(a), "d"(b));
}
// c += X Y^T over one 8-wide k tile: X, Y in the row layout (k slots 2t, 2t+1)
__device__ __forceinline__ void mma_xyt(double2& c, double2 x, double2 y) {
  dmma(c, x.x, y.x);
  dmma(c, x.y, y.y);
}
__device__ __forceinline__ double2 neg(double2 v) { return make_double2(-v.x, -v.y); }
__device__ __forceinline__ double2 ld2(const double* tile) {
  const int lane = threadIdx.x & 31;
  return *reinterpret_cast<const double2*>(tile + (lane >> 2) * 8 + 2 * (lane & 3));
}
__device__ __forceinline__ void st2(double* tile, double2 v) {
  const int lane = threadIdx.x & 31;
  *reinterpret_cast<double2*>(tile + (lane >> 2) * 8 + 2 * (lane & 3)) = v;
}
// Cholesky + inverse of one 8x8 SPD tile with NO lane exchange: every lane
// reads the whole lower tile (broadcast shared loads) and computes the
// factorisation redundantly in registers (a pivot step is one rsqrt chain;
// the shuffle-based v5::chol8 pays ~4x its latency here).  The tile is then
// overwritten with R = -M^-1 in the row layout (M = chol(tile), lower).
// Returns 0 or the 1-based first non-positive pivot.
__device__ __forceinline__ int chol8r(double* tile) {
  double a[36];                                   // packed lower, row-major
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j <= i; ++j) a[i * (i + 1) / 2 + j] = tile[i * 8 + j];
  int bad = 0;
  double s[8];
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const double d = a[p * (p + 1) / 2 + p];
    bad = (bad == 0 && !(d > 0.0)) ? p + 1 : bad;
    s[p] = rsqrt_nr(d);                           // 1 / M_pp
#pragma unroll
    for (int i = p + 1; i < 8; ++i) a[i * (i + 1) / 2 + p] *= s[p];
#pragma unroll
    for (int i = p + 1; i < 8; ++i)
#pragma unroll
      for (int k = p + 1; k <= i; ++k)
        a[i * (i + 1) / 2 + k] = fma(-a[i * (i + 1) / 2 + p], a[k * (k + 1) / 2 + p],
                                     a[i * (i + 1) / 2 + k]);
  }
  // in-place inverse of the unit-scaled factor, last column first:
  // X[j][j] = s_j, X[i][j] = -s_j sum_{k=j+1..i} X[i][k] M[k][j]  (i > j)
#pragma unroll
  for (int j = 7; j >= 0; --j) {
    double col[8];
#pragma unroll
    for (int i = j + 1; i < 8; ++i) {
      double acc = 0.0;
#pragma unroll
      for (int k = j + 1; k <= i; ++k) acc = fma(a[i * (i + 1) / 2 + k], a[k * (k + 1) / 2 + j], acc);
      col[i] = acc;
    }
#pragma unroll
    for (int i = j + 1; i < 8; ++i) a[i * (i + 1) / 2 + j] = -s[j] * col[i];
    a[j * (j + 1) / 2 + j] = s[j];
  }
  __syncwarp();                                   // every lane has read the tile
  const int lane = threadIdx.x & 31, g = lane >> 2, t2 = 2 * (lane & 3);
  double2 r = make_double2(0.0, 0.0);
#pragma unroll
  for (int gg = 0; gg < 8; ++gg)
#pragma unroll
    for (int c = 0; c <= gg; ++c) {
      const double v = -a[gg * (gg + 1) / 2 + c];
      r.x = (g == gg && c == t2) ? v : r.x;
      r.y = (g == gg && c == t2 + 1) ? v : r.y;
    }
  st2(tile, r);
  return bad;
}

#ifndef MCS_CHOL
#define MCS_CHOL 1
#endif
// the 8x8 diagonal factorisation used by phase 1 (MCS_CHOL 1: the shuffle
// variant of elim_v5.cuh, fewer FP64 instructions -> less contention with
// the DMMA streams of the co-resident warps, which share the FP64 pipe)
__device__ __forceinline__ int chol_diag(double* tile, const signed char* ones) {
#if MCS_CHOL == 1
  const double2 y = ld2(tile);
  __syncwarp();
  return v5::chol8(y.x, y.y, ones, tile);
#else
  return chol8r(tile);
#endif
}

// named barrier over the CTA's two warps (id 0 doubles as __syncthreads)
__device__ __forceinline__ void bar(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }

template <int NS, int NC>
struct Geo {
  static constexpr int NP = (NS + 7) / 8;                 // pivot tile rows of A
  static constexpr int NCB = (NC + 7) / 8;                // tile rows of B^T / S
  static constexpr int C1 = (NCB + 1) / 2;                // warp 0 owns c < C1
  static constexpr int NT = NP * (NP + 1) / 2;            // lower tiles of A
  static constexpr int LA = NS * (NS + 1) / 2;            // packed A (doubles)
  static constexpr int LA2 = (LA + 1) & ~1;               // staging (16-byte multiple)
  static constexpr int SMEM = (NT * 64 + 2 * C1 * 64 + LA2) * 8 + 16;
  static constexpr int NSEG = 8 * NP * (NP + 1) / 2;      // tile-row segments
  __host__ __device__ static constexpr int q(int i, int j) { return i * (i + 1) / 2 + j; }
};

// B^T tile (c, i) of element e into the row layout: lane (g, t) gets
// B[8i + 2t + s][8c + g], zero outside n x m
template <int NS, int NC>
__device__ __forceinline__ double2 load_bt(const double* __restrict__ Be, int c, int i) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int col = 8 * c + g, r0 = 8 * i + 2 * t;
  double2 v = make_double2(0.0, 0.0);
  if (col < NC) {
    if (r0 < NS) v.x = __ldg(Be + r0 * NC + col);
    if (r0 + 1 < NS) v.y = __ldg(Be + (r0 + 1) * NC + col);
  }
  return v;
}

// packed-lower staging -> 8x8 lower tiles, one 8-wide row segment of a
// tile per step (row r of tile (r/8, j): up to 8 consecutive doubles of the
// packed row).  The padding rows of the last diagonal tile are reset to the
// identity (phase 1 leaves -M^-1 there); the other padding entries stay
// zero from the one-time clear (every update keeps them zero).
template <int NS, int NC>
__device__ __forceinline__ void unpack_a(const double* __restrict__ P, double* __restrict__ T) {
  using G = Geo<NS, NC>;
  constexpr int NSEG = G::NSEG;
  for (int sgi = threadIdx.x; sgi < NSEG; sgi += 64) {
    // segment -> (row, tile column): rows 8b..8b+7 carry b+1 segments each
    int b = 0, base = 0;
#pragma unroll
    for (int q = 0; q < G::NP; ++q)
      if (sgi >= base + 8 * (q + 1) && q + 1 < G::NP) {
        base += 8 * (q + 1);
        b = q + 1;
      }
    const int off = sgi - base, r = 8 * b + off / (b + 1), j = off % (b + 1);
    if (r >= NS) continue;
    const double* src = P + r * (r + 1) / 2 + 8 * j;
    double* dst = T + G::q(b, j) * 64 + (r & 7) * 8;
    const int len = j < b ? 8 : (r & 7) + 1;
    double v[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) v[c] = c < len ? src[c] : 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (c < len) dst[c] = v[c];
  }
  if constexpr (NS % 8 != 0) {
    constexpr int R0 = NS % 8;
    double* D = T + G::q(G::NP - 1, G::NP - 1) * 64;
    for (int x = threadIdx.x; x < (8 - R0) * 8; x += 64) {
      const int r = R0 + x / 8, c = x % 8;
      D[r * 8 + c] = r == c ? 1.0 : 0.0;
    }
  }
}

// Phase 2 for the column blocks [CB, CE) of one warp.  X: warp 0's W^T_j
// tiles (double-buffered by j parity) for the cross blocks of warp 1.
// YM: FP64-pipe throttle mask (tools/dmma_prio.cu): a warp that streams DMMAs
// delays every dependent FP64 op of the co-resident warps by hundreds of
// cycles; __nanosleep(0) after a burst lets their chains through.
// bit 0: after every trailing-update tile, 1: after every trailing row,
// 2: after every phase-2 pivot block, 3: after every phase-2 B^T row update.
template <int YM, int BIT>
__device__ __forceinline__ void yield_fp64() {
  if constexpr ((YM >> BIT) & 1) __nanosleep(0);
}

template <int NS, int NC, int CB, int CE, int YM>
__device__ __forceinline__ void phase2(const double* T, double* X, double2 (&bt)[CE - CB][Geo<NS, NC>::NP],
                                       double* __restrict__ Se) {
  using G = Geo<NS, NC>;
  constexpr int NW = CE - CB, NP = G::NP, C1 = G::C1;
  constexpr bool CROSS = CB >= C1 && C1 > 0;              // warp 1: S_cd, d < C1
  double2 s_own[NW][NW];
  double2 s_x[CROSS ? NW : 1][C1];
#pragma unroll
  for (int a = 0; a < NW; ++a) {
#pragma unroll
    for (int b = 0; b < NW; ++b) s_own[a][b] = make_double2(0.0, 0.0);
#pragma unroll
    for (int d = 0; d < C1; ++d) s_x[CROSS ? a : 0][d] = make_double2(0.0, 0.0);
  }
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    const double2 r = ld2(T + G::q(j, j) * 64);           // R_j = -M_j^-1
    double2 wt[NW];
#pragma unroll
    for (int a = 0; a < NW; ++a) {                        // W^T_cj = -(B^T_cj R_j^T)
      wt[a] = make_double2(0.0, 0.0);
      mma_xyt(wt[a], neg(bt[a][j]), r);
    }
    if constexpr (!CROSS) {
#pragma unroll
      for (int a = 0; a < NW; ++a) st2(X + ((j & 1) * C1 + a) * 64, wt[a]);
    }
#pragma unroll
    for (int a = 0; a < NW; ++a)
#pragma unroll
      for (int b = 0; b <= a; ++b) mma_xyt(s_own[a][b], wt[a], wt[b]);
#pragma unroll
    for (int i = j + 1; i < NP; ++i) {                    // B^T_ci -= W^T_cj L_ij^T
      const double2 l = ld2(T + G::q(i, j) * 64);
#pragma unroll
      for (int a = 0; a < NW; ++a) mma_xyt(bt[a][i], neg(wt[a]), l);
      yield_fp64<YM, 3>();
    }
    yield_fp64<YM, 2>();
    bar(2);
    if constexpr (CROSS) {
#pragma unroll
      for (int d = 0; d < C1; ++d) {
        const double2 x = ld2(X + ((j & 1) * C1 + d) * 64);
#pragma unroll
        for (int a = 0; a < NW; ++a) mma_xyt(s_x[a][d], wt[a], x);
      }
    }
  }
  // S out (packed lower, rows < NC)
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  auto put = [&](int c, int d, double2 v) {
    const int row = 8 * c + g, col = 8 * d + 2 * t;
    if (row < NC) {
      if (col <= row) Se[row * (row + 1) / 2 + col] = v.x;
      if (col + 1 <= row) Se[row * (row + 1) / 2 + col + 1] = v.y;
    }
  };
#pragma unroll
  for (int a = 0; a < NW; ++a) {
#pragma unroll
    for (int b = 0; b <= a; ++b) put(CB + a, CB + b, s_own[a][b]);
    if constexpr (CROSS) {
#pragma unroll
      for (int d = 0; d < C1; ++d) put(CB + a, d, s_x[a][d]);
    }
  }
}

// One element, from the point of view of warp WARP (0 or 1).  The two warps
// run the same barrier sequence; each instantiation only keeps its own B^T
// column blocks live.
template <int NS, int NC, int WARP, int YM>
__device__ __forceinline__ void element(const double* __restrict__ A, const double* __restrict__ B,
                                        double* __restrict__ S, int* __restrict__ info,
                                        int64_t batch, int64_t e, double* T, double* X, double* P,
                                        uint64_t* mbar, uint32_t phase, const signed char* ones,
                                        int* bad) {
  using G = Geo<NS, NC>;
  constexpr int NP = G::NP, NCB = G::NCB, C1 = G::C1;
  constexpr int CB = WARP == 0 ? 0 : C1, CE = WARP == 0 ? C1 : NCB;
  const int lane = threadIdx.x & 31;
  MP0();
  const double* Be = B + e * (int64_t)(NS * NC);
  // this warp's B^T tiles into registers (consumed in phase 2)
  double2 bt[CE - CB > 0 ? CE - CB : 1][NP];
#pragma unroll
  for (int a = 0; a < CE - CB; ++a)
#pragma unroll
    for (int i = 0; i < NP; ++i) bt[a][i] = load_bt<NS, NC>(Be, CB + a, i);
  if (threadIdx.x == 0) *bad = 0;
  MP(WARP, 0);
  mbar_wait(mbar, phase);
  MP(WARP, 1);
  unpack_a<NS, NC>(P, T);
  bar(0);
  MP(WARP, 2);
  // the next element's A streams in while this one is eliminated
  if (threadIdx.x == 0 && e + gridDim.x < batch) {
    mbar_expect_tx(mbar, G::LA * 8);
    bulk_g2s(P, A + (e + gridDim.x) * G::LA, G::LA * 8, mbar);
  }
  // ---- phase 1: Cholesky of A (R_j = -M_j^-1 left in the diagonal tiles).
  // Warp 0 factorises the diagonal tiles, warp 1 updates the rest of the
  // trailing block.  The loops stay rolled: unrolled, batched trailing
  // updates stream DMMAs harder and starve the diagonal chain of the
  // co-resident elements (tools/dmma_fair.cu), measured slower.
  if (WARP == 0) {
    const int b = chol_diag(T, ones);
    if (lane == 0 && b) atomicCAS(bad, 0, b);
  }
  bar(1);
#pragma unroll 1
  for (int j = 0; j < NP; ++j) {
    const double2 r = ld2(T + G::q(j, j) * 64);
    // panel L_ij = A_ij M_j^-T = -(A_ij R_j^T), rows split between the warps
    for (int i = j + 1 + WARP; i < NP; i += 2) {
      double2 o = make_double2(0.0, 0.0);
      mma_xyt(o, neg(ld2(T + G::q(i, j) * 64)), r);
      st2(T + G::q(i, j) * 64, o);
    }
    bar(1);
    if (j + 1 < NP) {
      if (WARP == 0) {
        // look-ahead: the next diagonal tile, then its factorisation
        double* D = T + G::q(j + 1, j + 1) * 64;
        double2 c = ld2(D);
        const double2 l = ld2(T + G::q(j + 1, j) * 64);
        mma_xyt(c, neg(l), l);
        st2(D, c);
        __syncwarp();
        const int b = chol_diag(D, ones);
        if (lane == 0 && b) atomicCAS(bad, 0, 8 * (j + 1) + b);
      } else {
        // the rest of the trailing block: A_ik -= L_ij L_kj^T, j < k <= i
        for (int i = j + 1; i < NP; ++i) {
          const double2 li = neg(ld2(T + G::q(i, j) * 64));
          for (int k = (i == j + 1 ? j + 2 : j + 1); k <= i; ++k) {
            double* C = T + G::q(i, k) * 64;
            double2 c = ld2(C);
            mma_xyt(c, li, ld2(T + G::q(k, j) * 64));
            st2(C, c);
            yield_fp64<YM, 0>();
          }
          yield_fp64<YM, 1>();
        }
      }
      bar(1);
    }
  }
  MP(WARP, 3);
  // ---- phase 2: W^T = B^T L^-T, S = W^T W (registers)
  double* Se = S + e * (int64_t)(NC * (NC + 1) / 2);
  if constexpr (CE > CB)
    phase2<NS, NC, CB, CE, YM>(T, X, bt, Se);
  else
    for (int j = 0; j < NP; ++j) bar(2);
  MP(WARP, 4);
  bar(0);
  if (threadIdx.x == 0 && info) info[e] = *bad;
  MP(WARP, 5);
}

template <int NS, int NC, int YM>
__global__ void __launch_bounds__(64, 6)
    spd_schur_w2(const double* __restrict__ A, const double* __restrict__ B,
                 double* __restrict__ S, int* __restrict__ info, int64_t batch) {
  using G = Geo<NS, NC>;
  extern __shared__ __align__(128) double smem[];
  double* T = smem;                                      // NT tiles
  double* X = T + G::NT * 64;                            // 2 x C1 tiles
  double* P = X + 2 * G::C1 * 64;                        // packed A staging
  uint64_t* mbar = reinterpret_cast<uint64_t*>(P + G::LA2);
  __shared__ signed char ones[8];
  __shared__ int bad;
  if (threadIdx.x < 8) ones[threadIdx.x] = 1;
  for (int x = threadIdx.x; x < G::NT * 64; x += 64) T[x] = 0.0;   // padding stays zero
  if (threadIdx.x == 0) {
    mbar_init(mbar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  int64_t e = blockIdx.x;
  if (threadIdx.x == 0 && e < batch) {
    mbar_expect_tx(mbar, G::LA * 8);
    bulk_g2s(P, A + e * G::LA, G::LA * 8, mbar);
  }
  uint32_t phase = 0;
  const bool w0 = threadIdx.x < 32;
  for (; e < batch; e += gridDim.x, phase ^= 1) {
    if (w0)
      element<NS, NC, 0, YM>(A, B, S, info, batch, e, T, X, P, mbar, phase, ones, &bad);
    else
      element<NS, NC, 1, YM>(A, B, S, info, batch, e, T, X, P, mbar, phase, ones, &bad);
  }
}

// ---- one warp per element, register resident (the sweep of ds_reg.cuh):
// B^T lives in registers in the DMMA row layout and becomes W^T = B^T L^-T
// under the right-looking sweep over the 8x8 pivot tiles of A; the trailing
// part of A sits in per-lane private shared-memory slots (no barrier, no
// warp synchronisation); S = W^T W is formed from the register tiles.
// PAIR: warps w and w + 4 of the 8-warp CTA (same SM sub-partition) meet at
// a named barrier before every pivot tile, so their 8x8 factorisations run
// together and their DMMA bursts share the pipe (see dsr::sweep).
using dsr::PairSync;

template <int NS, int NC, int WPB, int MINB, int PAIR>
__global__ void __launch_bounds__(32 * WPB, MINB)
    spd_schur_w1(const double* __restrict__ A, const double* __restrict__ B,
                 double* __restrict__ S, int* __restrict__ info, int64_t batch, int pf) {
  using G = Geo<NS, NC>;
  constexpr int NP = G::NP, NCB = G::NCB, LA = G::LA;
  extern __shared__ __align__(128) double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double* Tl = smem + warp * (G::NT * 64) + 2 * lane;
  static_assert(!PAIR || WPB == 8, "pairs: warps w, w + 4 of an 8-warp CTA");
  const int64_t nw = (int64_t)gridDim.x * WPB;
  // every warp of the CTA runs the same number of rounds (the pair barriers);
  // a warp past the end repeats the last element without storing
  const int64_t e0 = (int64_t)blockIdx.x * WPB;
  const int64_t rounds = e0 < batch ? (batch - e0 + nw - 1) / nw : 0;
#pragma unroll 1
  for (int64_t rd = 0; rd < rounds; ++rd) {
    const int64_t ew = e0 + warp + rd * nw;
    const bool live = ew < batch;
    const int64_t e = live ? ew : batch - 1;
    if (pf && e + nw < batch) {
      const char* na = reinterpret_cast<const char*>(A + (e + nw) * LA);
      for (int off = lane * 128; off < LA * 8; off += 32 * 128)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(na + off));
      const char* nb = reinterpret_cast<const char*>(B + (e + nw) * (int64_t)(NS * NC));
      for (int off = lane * 128; off < NS * NC * 8; off += 32 * 128)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(nb + off));
    }
    const double* Ae = A + e * LA;
    const double* Be = B + e * (int64_t)(NS * NC);
    // pivot dofs by tile slot (dsr::PivMap: n = 60 puts the four dofs of the
    // last tile on its even slots, so products over that tile take one DMMA)
    using PM = dsr::PivMap<NS>;
    auto asym = [&](int r, int c) { return __ldg(Ae + (r >= c ? pk(r, c) : pk(c, r))); };
#pragma unroll
    for (int i = 0; i < NP; ++i)
#pragma unroll
      for (int j = 0; j <= i; ++j) {
        const int rd = PM::dof(i, g), c0 = PM::dof(j, 2 * t), c1 = PM::dof(j, 2 * t + 1);
        double2 v;   // the slots hold -A (padding: -1 on the diagonal)
        v.x = (rd >= 0 && c0 >= 0) ? -asym(rd, c0) : ((i == j && g == 2 * t) ? -1.0 : 0.0);
        v.y = (rd >= 0 && c1 >= 0) ? -asym(rd, c1) : ((i == j && g == 2 * t + 1) ? -1.0 : 0.0);
        *reinterpret_cast<double2*>(Tl + G::q(i, j) * 64) = v;
      }
    double2 bt[NCB][NP];   // B^T tile (c, i): lane (g, t) gets B[dof(i, 2t + s)][8c + g]
#pragma unroll
    for (int c = 0; c < NCB; ++c)
#pragma unroll
      for (int i = 0; i < NP; ++i) {
        const int col = 8 * c + g, r0 = PM::dof(i, 2 * t), r1 = PM::dof(i, 2 * t + 1);
        double2 v = make_double2(0.0, 0.0);
        if (col < NC) {
          if (r0 >= 0) v.x = __ldg(Be + r0 * NC + col);
          if (r1 >= 0) v.y = __ldg(Be + r1 * NC + col);
        }
        bt[c][i] = v;
      }
    int bad = 0;
    double2 none[1][1];
    if constexpr (PAIR == 1)
      dsr::sweep<NP, NCB, false, PairSync, false, PM::HALF>(Tl, bt, none, bad, PairSync{1 + (warp & 3)});
    else if constexpr (PAIR == 2)
      dsr::sweep<NP, NCB, false, dsr::PairSync0, false, PM::HALF>(Tl, bt, none, bad,
                                                                 dsr::PairSync0{1 + (warp & 3)});
    else
      dsr::sweep<NP, NCB, false, dsr::NoSync, false, PM::HALF>(Tl, bt, none, bad);
    if (!live) continue;
    double* Se = S + e * (int64_t)(NC * (NC + 1) / 2);
#pragma unroll
    for (int c = 0; c < NCB; ++c) {
      const int row = 8 * c + g;
#pragma unroll
      for (int d = 0; d <= c; ++d) {
        double2 o = make_double2(0.0, 0.0);
#pragma unroll
        for (int j = 0; j < NP; ++j) {
          if (PM::HALF && j == NP - 1) dsr::mma_xyt_even(o, bt[c][j], bt[d][j]);
          else dsr::mma_xyt(o, bt[c][j], bt[d][j]);
        }
        const int col = 8 * d + 2 * t;
        if (row < NC) {
          if (col <= row) Se[row * (row + 1) / 2 + col] = o.x;
          if (col + 1 <= row) Se[row * (row + 1) / 2 + col + 1] = o.y;
        }
      }
    }
    if (lane == 0 && info) info[e] = bad;
  }
}

}  // namespace micro

template <int NS, int NC, int YM>
static int launch_w2(const double* A, const double* B, double* S, int* info, int64_t batch,
                     cudaStream_t st) {
  using G = micro::Geo<NS, NC>;
  auto kern = micro::spd_schur_w2<NS, NC, YM>;
  const size_t smem = G::SMEM;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 64, smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  const int64_t g = (int64_t)per_sm * sm_count();
  kern<<<(int)(batch < g ? batch : g), 64, smem, st>>>(A, B, S, info, batch);
  return launch_status();
}

template <int NS, int NC>
int launch_spd_schur_w2(const double* A, const double* B, double* S, int* info, int64_t batch,
                        cudaStream_t st) {
  // MCS_MICRO_YIELD = throttle mask (A/B measurements; default MCS_MICRO_YM)
  // default: one warp per element, register resident; MCS_MICRO=2: the
  // two-warp kernel (and its MCS_MICRO_YIELD throttle variants)
  static const int mv = getenv("MCS_MICRO") ? atoi(getenv("MCS_MICRO")) : 1;
  if (mv != 2) {
    // default: the pair meets once per element (22.3 ms); 3: before every
    // pivot tile (22.9 ms); 4: never (22.75 ms)
    auto kern = mv == 3 ? micro::spd_schur_w1<NS, NC, 8, 1, 1>
                        : (mv == 4 ? micro::spd_schur_w1<NS, NC, 8, 1, 0> : micro::spd_schur_w1<NS, NC, 8, 1, 2>);
    const size_t smem = (size_t)8 * micro::Geo<NS, NC>::NT * 64 * sizeof(double);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem) != cudaSuccess ||
        per_sm < 1)
      per_sm = 1;
    const int64_t want = (batch + 7) / 8, cap = (int64_t)per_sm * sm_count();
    static const int pf = getenv("MCS_MICRO_PF") ? atoi(getenv("MCS_MICRO_PF")) : 0;   // 1: L2 prefetch of the next element (measured slower: L2 thrash, 1.6x the DRAM reads)
    kern<<<(int)(want < cap ? want : cap), 256, smem, st>>>(A, B, S, info, batch, pf);
    return launch_status();
  }
  static const int ym = getenv("MCS_MICRO_YIELD") ? atoi(getenv("MCS_MICRO_YIELD")) : MCS_MICRO_YM;
  switch (ym) {
    case 1: return launch_w2<NS, NC, 1>(A, B, S, info, batch, st);
    case 2: return launch_w2<NS, NC, 2>(A, B, S, info, batch, st);
    case 4: return launch_w2<NS, NC, 4>(A, B, S, info, batch, st);
    case 8: return launch_w2<NS, NC, 8>(A, B, S, info, batch, st);
    case 5: return launch_w2<NS, NC, 5>(A, B, S, info, batch, st);
    case 6: return launch_w2<NS, NC, 6>(A, B, S, info, batch, st);
    case 9: return launch_w2<NS, NC, 9>(A, B, S, info, batch, st);
    case 10: return launch_w2<NS, NC, 10>(A, B, S, info, batch, st);
  }
  return launch_w2<NS, NC, 0>(A, B, S, info, batch, st);
}

template int launch_spd_schur_w2<60, 36>(const double*, const double*, double*, int*, int64_t,
                                         cudaStream_t);

}  // namespace mcs
