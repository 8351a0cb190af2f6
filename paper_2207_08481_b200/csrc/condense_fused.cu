// Fused element pipeline: geometry weights -> element blocks -> sigma/omega
// condensation -> double Schur, ONE WARP PER ELEMENT (SURVEY §8a rows
// A1 + A3 + A4, §8f-1).  k <= 4: Y whole in registers, one pass.  k = 5, 6:
// Y is produced CPP column chunks at a time (passes), the partial S_T sums
// live in the warp's packed shared-memory copy between passes, the
// lane-ordered Bsig tables are read from a global (L2-resident) buffer with
// coalesced loads instead of a per-CTA shared-memory copy.
//
// Algebra (csrc/condense_struct.cu): with the block
// structure of the MCS element spaces
//     S_T = adiv + Y Y^T,   Y = [B_m F_m (m < ml) | B_b L_b^-T],
// B = Bsig = [bus; bhs] generated on the fly from the reference-cell tables
// (refblocks.py; B[i] = base[i] + sum_a w[i][a] T_a[i], w = the element's
// bus-edge / bhs weights of the edge row i belongs to), then the reference's
// double_schur (condensation.py:207-226) on the element-local S_T:
//     S_oo = L L^T, X = S_oo^-1 S_oc, Sd_T = S_cc - (L^-1 S_oc)^T (L^-1 S_oc),
//     S_oo^-1 = L^-T L^-1.
//
// Why a warp per element: every step is a short dependency chain (12- and
// 15-pivot Cholesky factorisations, triangular solves) that a CTA-wide
// pipeline would serialise behind barriers.  A warp needs no barrier, and
// 12 resident warps per SM keep 12 elements in flight.  Y lives in REGISTERS
// in the DMMA operand layout: lane (g, t) holds rows 8I + g, columns
// (8 kc + 2t, 8 kc + 2t + 1) of every 8x8 chunk, so S_T = Y Y^T (m8n8k4
// FP64 MMA) takes A = Y_I and B = Y_J straight from the same lane's
// registers (no shared-memory operand traffic).  Columns of Y are ordered
// so that each 8-column chunk is uniform across lanes except one "mixed"
// chunk: low blocks m = 4 kc + t (2 columns per lane), then the bubble
// columns, produced by a DMMA of the bubble part of B with L_b^-T whose
// accumulator layout IS the operand layout.
#include <cstdlib>

#include "common.cuh"
#include "ds_reg.cuh"

namespace mcs {

// optional per-phase clock accounting (tools/fused_prof.py builds a copy of
// this file with MCS_FUSED_PROF defined; the library never does)
#ifdef MCS_FUSED_PROF
__device__ unsigned long long g_fz_prof[8];
#define FZ_T0() long long _fz_t = clock64()
#define FZ_T(i)                                                              \
  do {                                                                       \
    __syncwarp();                                                            \
    if ((threadIdx.x & 31) == 0) {                                           \
      const long long _n = clock64();                                        \
      atomicAdd(&g_fz_prof[i], (unsigned long long)(_n - _fz_t));            \
      _fz_t = _n;                                                            \
    }                                                                        \
  } while (0)
#else
#define FZ_T0()
#define FZ_T(i)
#endif

#ifndef MCS_FZ_CPP4
#define MCS_FZ_CPP4 4   // Y column chunks per pass at k = 4 (4 = one pass; tools/fused_prof.py sweeps it)
#endif

namespace fz {

constexpr int W_MSIG = 0, W_ADIV = 27, NWS = 36;   // weight slots (refblocks.py), 30.. = 0

// Row classification of Bsig and the per-tile formats of the lane-ordered
// shared-memory tables (a separate struct: Geo uses these in its own
// constant expressions).
template <int K>
struct Rows {
  using Z = Sizes<K>;
  static constexpr int NEM = Z::n_em, nu = Z::nu, nloc = Z::nloc;
  // Bsig row i: 0 facet (bus volume + edge term of edge i/(k+1)), 1 interior
  // bubble (volume only), 2 Vhat (bhs of edge (i-nu)/k), 3 padding
  __host__ __device__ static constexpr int row_type(int i) {
    return i < NEM ? 0 : (i < nu ? 1 : (i < nloc ? 2 : 3));
  }
  // weight slot of row i's three edge weights (refblocks.py W_BUSE / W_BHS)
  __host__ __device__ static constexpr int row_woff(int i) {
    return i < NEM ? 9 + 3 * (i / (K + 1)) : ((i >= nu && i < nloc) ? 18 + 3 * ((i - nu) / K) : 30);
  }
  // Row types present in the 8-row tile I (bit 0 facet, 1 interior, 2 Vhat).
  __host__ __device__ static constexpr int tile_types(int I) {
    int m = 0;
    for (int rr = 0; rr < 8; ++rr) {
      const int ty = row_type(8 * I + rr);
      if (ty < 3) m |= 1 << ty;
    }
    return m;
  }
  // Per-CTA shared-memory tables of Bsig, stored IN THE ORDER THE LANES READ
  // THEM (lane (g, t) of tile I owns row 8I + g): every lane generates exactly
  // the entries its Y registers need, so Bsig is never staged.
  //
  // Low blocks (dof 3m + a = Dubiner function m x generator a): the edge
  // terms act on generator a only, T_a[i][3m + a'] = delta_aa' Ehat[i][m]
  // (engine.fused_tables checks it), hence per (row, m = 4 kc + t) the four
  // values (base_0, base_1, base_2, Ehat) and
  //   y_s = sum_a base_a F_m[a][s] + Ehat * G_s,  G_s = sum_a w_a F_m[a][s]
  // (G per element and edge group, precomputed once per element).
  // Format of tile I: 4 = (b0, b1 | b2, Ehat) as two conflict-free 16-byte
  // planes, 3 = interior rows only (b0, b1, b2), 1 = Vhat rows only (Ehat).
  __host__ __device__ static constexpr int fmt_low(int I) {
    const int m = tile_types(I);
    return m == 2 ? 3 : (m == 4 ? 1 : 4);
  }
  // Bubble columns (A operand of the bubble DMMA, column nl + 4 ks + t): 4 =
  // (base, T0 | T1, T2), 1 = interior rows only (base), 3 = Vhat only (T0, T1, T2).
  __host__ __device__ static constexpr int fmt_bub(int I) {
    const int m = tile_types(I);
    return m == 2 ? 1 : (m == 4 ? 3 : 4);
  }
  __host__ __device__ static constexpr int lo_off(int I, int nlow) {
    int o = 0;
    for (int q = 0; q < I; ++q) o += 32 * nlow * fmt_low(q);
    return o;
  }
  __host__ __device__ static constexpr int bu_off(int I, int nks) {
    int o = 0;
    for (int q = 0; q < I; ++q) o += 32 * nks * fmt_bub(q);
    return o;
  }
};

template <int K>
struct Geo {
  using Z = Sizes<K>;
  using T = FTab<K>;
  static constexpr int ml = T::ml, nb = T::nb, nl = T::nl, ns = Z::ns, nu = Z::nu;
  static constexpr int nloc = Z::nloc, NI = Z::n_int, NC = Z::ncpl, NEM = Z::n_em;
  static constexpr int r = ml % 4;                    // low blocks in the mixed chunk
  static constexpr int NLF = ml / 4;                  // full low chunks
  static constexpr int MIX = r > 0 ? 1 : 0;
  static constexpr int NLOW = NLF + MIX;
  static constexpr int BMIX = MIX ? 8 - 2 * r : 0;    // bubble columns in the mixed chunk
  static constexpr int BREST = nb > BMIX ? nb - BMIX : 0;
  static constexpr int NBP = (BREST + 7) / 8;         // pure bubble chunks
  static constexpr int NBT = MIX + NBP;               // bubble DMMA n-tiles
  static constexpr int NKC = NLF + MIX + NBP;         // 8-column chunks of Y
  static constexpr int NKS = (nb + 3) / 4;            // k-steps of the bubble DMMA
  static constexpr int NR = T::NR, NRB = NR / 8;
  static constexpr int TAIL = nloc - 8 * (NRB - 1);   // real rows of the last 8-row tile
#ifndef MCS_FZ_NO_STAIL
  // TAIL == 1 (k = 5): that row's S_T entries as dot products in phase C
  // (measured: k = 5 1.89 -> 1.75 ms; with TAIL == 2 at k = 4 the shuffles
  // cost more than the 48 DMMAs they replace: 0.324 -> 0.329 ms)
  static constexpr bool STAIL = TAIL <= 1;
#else
  static constexpr bool STAIL = false;
#endif
  static_assert(!STAIL || 8 * (NRB - 1) >= nu, "tail rows are Vhat rows (no adiv term)");
  static constexpr int st_len = ExtLayout<K>::st_len;
  // k >= 5 (BIG): Y in passes of CPP chunks, tables in global memory, the
  // phase-A factors alias the packed S_T (dead until the first pass ends),
  // G has its own slot (it lives across the passes)
  static constexpr bool BIG = K >= 5;
  static constexpr int CPP = BIG ? 3 : (K == 4 ? MCS_FZ_CPP4 : NKC);
  static constexpr int NPASS = (NKC + CPP - 1) / CPP;
  static constexpr int NG = 6 * ml * 2;               // G[edge group][m][s]
  // per-warp shared memory (doubles)
  static constexpr int o_w = 0;
  static constexpr int o_F = NWS;                     // F_m, 6 per block
  static constexpr int o_G = o_F + even(6 * ml);      // G (BIG only)
  static constexpr int o_S = o_G + (BIG ? even(NG) : 0);   // packed S_T
  static constexpr int UA = 2 * nb * nb + even(nb);   // Ls | Li | 1/diag
  static constexpr int UB = even(6 * ml * 2);         // G[edge group][m][s] (phase B)
  static constexpr int o_U = BIG ? o_S : o_S + st_len;     // phase-dependent union
  static constexpr int UD = dsr::Geo<K>::PER_WARP;    // phase D: private tile slots of S_oo
  static constexpr int UMAX = UA > UB ? (UA > UD ? UA : UD) : (UB > UD ? UB : UD);
  static constexpr int PER_WARP = BIG ? o_S + (st_len > even(UA) ? st_len : even(UA)) : o_U + even(UMAX);
  static_assert(nb <= 32 && ml <= 32, "lane-per-row factorisations");
  static_assert(6 * ml * 2 <= nb * nb, "G fits over Ls");
  using RW = Rows<K>;
  __host__ __device__ static constexpr int row_type(int i) { return RW::row_type(i); }
  __host__ __device__ static constexpr int row_woff(int i) { return RW::row_woff(i); }
  __host__ __device__ static constexpr int fmt_low(int I) { return RW::fmt_low(I); }
  __host__ __device__ static constexpr int fmt_bub(int I) { return RW::fmt_bub(I); }
  __host__ __device__ static constexpr int lo_off(int I) { return RW::lo_off(I, NLOW); }
  __host__ __device__ static constexpr int bu_off(int I) { return RW::bu_off(I, NKS); }
  static constexpr int TAB_LO = 0;
  static constexpr int TAB_BU = TAB_LO + RW::lo_off(NRB, NLOW);
  static constexpr int TAB_MB = TAB_BU + RW::bu_off(NRB, NKS);        // MbRef [6][nb][nb]
  static constexpr int TAB_A = TAB_MB + even(6 * nb * nb);   // ARef [6][ml][9]
  static constexpr int TAB_SMEM = TAB_A + even(6 * 9 * ml);
  // bubble column of DMMA n-tile bt, output column n (-1: none)
  // HALF: the last pure bubble chunk holds <= 4 columns: they sit on the even
  // columns (the k slots of the first m8n8k4 step of Y Y^T), the odd ones are
  // zero and phase C skips the second step for that chunk (k = 6)
  static constexpr int BLAST = NBP > 0 ? BREST - 8 * (NBP - 1) : 0;
  static constexpr bool HALF = NBP > 0 && BLAST <= 4;
  __host__ __device__ static constexpr int jmap(int bt, int n) {
    if (MIX && bt == 0) return (n >= 2 * r && n - 2 * r < nb) ? n - 2 * r : -1;
    if (HALF && bt == NBT - 1) {
      const int j = BMIX + 8 * (bt - MIX) + n / 2;
      return (n % 2 == 0 && n / 2 < BLAST) ? j : -1;
    }
    const int j = BMIX + 8 * (bt - MIX) + n;
    return j < nb ? j : -1;
  }
};

// signed-free Cholesky of an n x n SPD matrix held one row per lane
// (a[c] = row lane, c < n; lanes >= n carry a copy of row 0).  On return
// l[c] = L[lane][c] (c <= lane significant) and rd[j] = 1 / L[j][j] (same on
// every lane, written to rd_out by lane 0).  ok = false if a pivot is not
// positive.
template <int N>
__device__ __forceinline__ bool chol_rows(double (&a)[N], double (&l)[N], double* rd_out) {
  const int lane = threadIdx.x & 31;
  bool ok = true;
#pragma unroll
  for (int j = 0; j < N; ++j) {
    const double d = __shfl_sync(0xffffffffu, a[j], j);
    ok &= d > 0.0;
    const double r = rsqrt_nr(d);
    if (lane == 0) rd_out[j] = r;
    l[j] = a[j] * r;
#pragma unroll
    for (int c = j + 1; c < N; ++c) a[c] = fma(-l[j], __shfl_sync(0xffffffffu, l[j], c), a[c]);
  }
  return ok;
}

// Column `col` of L^-1 for the n x n lower L in shared memory (row stride
// ls, 1/diag in rd): forward substitution blocked by 8 rows -- the rows of
// earlier blocks enter as 8 independent accumulations, only the 8 rows of a
// diagonal block form a dependent chain (an n-step chain otherwise).
template <int N>
__device__ __forceinline__ void linv_col(const double* Ls, int ls, const double* rd, int col,
                                         double (&x)[N]) {
#pragma unroll
  for (int jb = 0; jb < N; jb += 8) {
    double acc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = (jb + u == col) ? 1.0 : 0.0;
#pragma unroll
    for (int q = 0; q < jb; ++q)
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (jb + u < N) acc[u] = fma(-Ls[(jb + u) * ls + q], x[q], acc[u]);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int j = jb + u;
      if (j < N) {
        double v = acc[u];
#pragma unroll
        for (int q = jb; q < j; ++q) v = fma(-Ls[j * ls + q], x[q], v);
        x[j] = v * rd[j];
      }
    }
  }
}

}  // namespace fz

// Lane-ordered Bsig tables (layout: fz::Rows / fz::Geo) plus the MbRef and
// ARef segments, from the FTab tables.  Threads tid, tid + nthr, ...
template <int K>
__device__ __forceinline__ void build_lane_tables(const double* __restrict__ tab,
                                                  double* __restrict__ stab, int tid, int nthr) {
  using G = fz::Geo<K>;
  using T = FTab<K>;
  constexpr int ml = G::ml, nb = G::nb, nl = G::nl, ns = G::ns, nloc = G::nloc, NRB = G::NRB;
  for (int q = tid; q < 6 * nb * nb; q += nthr) stab[G::TAB_MB + q] = tab[T::o_Mb + q];
  for (int q = tid; q < 6 * 9 * ml; q += nthr) stab[G::TAB_A + q] = tab[T::o_A + q];
  for (int q = tid; q < 32 * G::NLOW * NRB; q += nthr) {
    const int ln = q & 31, kc = (q >> 5) % G::NLOW, I = (q >> 5) / G::NLOW;
    const int i = 8 * I + (ln >> 2), m = 4 * kc + (ln & 3);
    double b0 = 0.0, b1 = 0.0, b2 = 0.0, eh = 0.0;
    if (i < nloc && m < ml) {
      const double* src = tab + T::o_G4 + 4 * (i * ns + 3 * m);
      b0 = src[0];
      b1 = src[4];
      b2 = src[8];
      eh = src[1];   // T_0 of column 3m (= T_1 of 3m + 1 = T_2 of 3m + 2)
    }
    double* dst = stab + G::TAB_LO + G::lo_off(I);
    const int fmt = G::fmt_low(I);
    if (fmt == 4) {
      dst[(2 * kc) * 64 + 2 * ln] = b0;
      dst[(2 * kc) * 64 + 2 * ln + 1] = b1;
      dst[(2 * kc + 1) * 64 + 2 * ln] = b2;
      dst[(2 * kc + 1) * 64 + 2 * ln + 1] = eh;
    } else if (fmt == 3) {
      dst[(3 * kc) * 32 + ln] = b0;
      dst[(3 * kc + 1) * 32 + ln] = b1;
      dst[(3 * kc + 2) * 32 + ln] = b2;
    } else {
      dst[kc * 32 + ln] = eh;
    }
  }
  for (int q = tid; q < 32 * G::NKS * NRB; q += nthr) {
    const int ln = q & 31, ks = (q >> 5) % G::NKS, I = (q >> 5) / G::NKS;
    const int i = 8 * I + (ln >> 2), c = 4 * ks + (ln & 3);
    double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
    if (i < nloc && c < nb) {
      const double* src = tab + T::o_G4 + 4 * (i * ns + nl + c);
      v0 = src[0];
      v1 = src[1];
      v2 = src[2];
      v3 = src[3];
    }
    double* dst = stab + G::TAB_BU + G::bu_off(I);
    const int fmt = G::fmt_bub(I);
    if (fmt == 4) {
      dst[(2 * ks) * 64 + 2 * ln] = v0;
      dst[(2 * ks) * 64 + 2 * ln + 1] = v1;
      dst[(2 * ks + 1) * 64 + 2 * ln] = v2;
      dst[(2 * ks + 1) * 64 + 2 * ln + 1] = v3;
    } else if (fmt == 3) {
      dst[(3 * ks) * 32 + ln] = v1;
      dst[(3 * ks + 1) * 32 + ln] = v2;
      dst[(3 * ks + 2) * 32 + ln] = v3;
    } else {
      dst[ks * 32 + ln] = v0;
    }
  }
}

// k >= 5: the tables once per call into a global buffer (stays in L2)
template <int K>
__global__ void fused_lane_tables_kernel(const double* __restrict__ tab, double* __restrict__ gtab) {
  build_lane_tables<K>(tab, gtab, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
}

template <int N>
struct IC {
  static constexpr int value = N;
};

// DS: the double Schur as phase D (ext, Sd written); otherwise S_T only.
// PAIR: the WPB / 4 warps of an SM sub-partition (w, w + 4, ...) start every
// element together (named barrier), so that their chain-bound phase A runs
// side by side and their DMMA-bound phases share the pipe (a warp streaming
// DMMAs starves a co-resident warp's dependent FP64 chain).
// Measured: k = 6 3.72 -> 3.48 ms; k = 5 1.75 -> 1.86 ms (off).
template <int K, int WPB, int MINB, bool DS, bool PAIR = false>
__global__ void __launch_bounds__(32 * WPB, MINB)
    condense_fused_kernel(const double* __restrict__ Wg, int nwgt, const double* __restrict__ tab,
                          const double* __restrict__ gtab, double* __restrict__ ST,
                          double* __restrict__ ext, double* __restrict__ Sd,
                          int* __restrict__ info, int64_t nt) {
  using G = fz::Geo<K>;
  using T = FTab<K>;
  using L = ExtLayout<K>;
  constexpr int ml = G::ml, nb = G::nb, nu = G::nu, nloc = G::nloc;
  constexpr int NRB = G::NRB, NKC = G::NKC, CPP = G::CPP, NPASS = G::NPASS;
  constexpr bool BIG = G::BIG;
  extern __shared__ __align__(16) double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const double* stab;                                    // lane-ordered Bsig tables
  double* sw;
  if constexpr (BIG) {
    stab = gtab;
    sw = smem + warp * G::PER_WARP;
  } else {
    build_lane_tables<K>(tab, smem, threadIdx.x, 32 * WPB);   // compact copy per CTA
    __syncthreads();
    stab = smem;
    sw = smem + G::TAB_SMEM + warp * G::PER_WARP;
  }
  double* wts = sw + G::o_w;
  double* Fs = sw + G::o_F;
  double* Spk = sw + G::o_S;
  double* U = sw + G::o_U;

  if (lane < fz::NWS - 30) wts[30 + lane] = 0.0;        // zero weight slots
  const int64_t nw = static_cast<int64_t>(gridDim.x) * WPB;
  int64_t e = static_cast<int64_t>(blockIdx.x) * WPB + warp;
  const int nwl = nwgt < 30 ? nwgt : 30;
  double wnext = (e < nt && lane < nwl) ? __ldg(Wg + e * nwgt + lane) : 0.0;

  static_assert(!PAIR || WPB % 4 == 0, "groups: the warps w, w + 4, ... of one CTA");
  const int64_t e0 = static_cast<int64_t>(blockIdx.x) * WPB;
  int64_t rounds = e0 < nt ? (nt - e0 + nw - 1) / nw : 0;   // PAIR: the same trip count for the CTA
#pragma unroll 1
  for (; PAIR ? rounds > 0 : e < nt; e += nw, --rounds) {
    if constexpr (PAIR) {
      asm volatile("bar.sync %0, %1;" ::"r"(1 + (warp & 3)), "n"(32 * (WPB / 4)) : "memory");
      if (e >= nt) continue;
    }
    if (lane < nwl) wts[lane] = wnext;
    if (e + nw < nt && lane < nwl) wnext = __ldg(Wg + (e + nw) * nwgt + lane);   // prefetch
    __syncwarp();
    int bad = 0;

    FZ_T0();
    // ---------------- A: bubble block factor and the 3x3 block factors
    double* Ls = U;
    double* Li = U + nb * nb;
    double* Rd = U + 2 * nb * nb;
    {
      const int i = lane < nb ? lane : 0;
      double a[nb], l[nb];
#pragma unroll
      for (int c = 0; c < nb; ++c) a[c] = 0.0;
#pragma unroll
      for (int r = 0; r < 6; ++r) {
        const double w = wts[fz::W_MSIG + r];
        const double* mr = stab + G::TAB_MB + (r * nb + i) * nb;
#pragma unroll
        for (int c = 0; c < nb; ++c) a[c] = fma(w, mr[c], a[c]);
      }
      if (!fz::chol_rows<nb>(a, l, Rd)) bad |= 1;
      if (lane < nb) {
#pragma unroll
        for (int c = 0; c < nb; ++c) Ls[lane * nb + c] = l[c];
      }
    }
    if (lane < ml) {
      double A[9];
#pragma unroll
      for (int q = 0; q < 9; ++q) A[q] = 0.0;
#pragma unroll
      for (int r = 0; r < 6; ++r) {
        const double w = wts[fz::W_MSIG + r];
        const double* ar = stab + G::TAB_A + (r * ml + lane) * 9;
#pragma unroll
        for (int q = 0; q < 9; ++q) A[q] = fma(w, ar[q], A[q]);
      }
      // s = detJ skew(T_a): the bws weights (refblocks.py W_BWS)
      const double s0 = wts[6], s1 = wts[7], s2 = wts[8];
      const double a00 = A[0], a10 = A[3], a11 = A[4], a20 = A[6], a21 = A[7], a22 = A[8];
      const double d11p = a11 - (a10 * a10) / a00;
      const bool okA = a00 > 0.0 && d11p > 0.0;
      const double i00 = rsqrt_nr(a00);
      const double l10 = a10 * i00, l20 = a20 * i00;
      const double d11 = a11 - l10 * l10;
      const double i11 = rsqrt_nr(d11);
      const double l21 = (a21 - l20 * l10) * i11;
      const double d22 = a22 - l20 * l20 - l21 * l21;
      const double i22 = rsqrt_nr(d22);
      if (!(okA && d22 > 0.0)) bad |= 1;
      const double v0 = s0 * i00;
      const double v1 = (s1 - l10 * v0) * i11;
      const double v2 = (s2 - l20 * v0 - l21 * v1) * i22;
      const double vn = rsqrt_nr(v0 * v0 + v1 * v1 + v2 * v2);
      const double u0 = v0 * vn, u1 = v1 * vn, u2 = v2 * vn;
      const double au0 = fabs(u0), au1 = fabs(u1), au2 = fabs(u2);
      const int ax = (au0 <= au1 && au0 <= au2) ? 0 : (au1 <= au2 ? 1 : 2);
      const double ua = ax == 0 ? u0 : (ax == 1 ? u1 : u2);
      double q10 = -ua * u0, q11 = -ua * u1, q12 = -ua * u2;
      if (ax == 0) q10 += 1.0;
      else if (ax == 1) q11 += 1.0;
      else q12 += 1.0;
      const double qn = rsqrt_nr(q10 * q10 + q11 * q11 + q12 * q12);
      q10 *= qn;
      q11 *= qn;
      q12 *= qn;
      const double q20 = u1 * q12 - u2 * q11, q21 = u2 * q10 - u0 * q12, q22 = u0 * q11 - u1 * q10;
      const double f20 = q12 * i22, f21 = q22 * i22;
      const double f10 = (q11 - l21 * f20) * i11, f11 = (q21 - l21 * f21) * i11;
      const double f00 = (q10 - l10 * f10 - l20 * f20) * i00;
      const double f01 = (q20 - l10 * f11 - l20 * f21) * i00;
      double* Fm = Fs + 6 * lane;
      Fm[0] = f00;
      Fm[1] = f01;
      Fm[2] = f10;
      Fm[3] = f11;
      Fm[4] = f20;
      Fm[5] = f21;
    }
    __syncwarp();
    if (lane < nb) {   // column `lane` of L_b^-1 (blocked forward substitution)
      double x[nb];
      fz::linv_col<nb>(Ls, nb, Rd, lane, x);
#pragma unroll
      for (int j = 0; j < nb; ++j) Li[j * nb + lane] = x[j];
    }
    __syncwarp();
    // B operands of the bubble DMMA: (L_b^-T)[q][j] = Li[j][q], q = 4 ks + t, j = jmap(bt, g)
    double LiR[G::NBT][G::NKS];
#pragma unroll
    for (int bt = 0; bt < G::NBT; ++bt) {
      const int j = G::jmap(bt, g);
#pragma unroll
      for (int ks = 0; ks < G::NKS; ++ks) {
        const int q = 4 * ks + t;
        LiR[bt][ks] = (j >= 0 && q < nb) ? Li[j * nb + q] : 0.0;
      }
    }
    __syncwarp();
    // G[grp][m][s] = sum_a w[9 + 3 grp + a] F_m[a][s]: the edge weights of
    // the three bus edges (grp 0..2) and the three bhs edges (3..5) folded
    // into F (k <= 4: over Ls, which is dead once L_b^-1 is formed)
    double* Gs = BIG ? sw + G::o_G : U;
    for (int q = lane; q < G::NG; q += 32) {
      const int sI = q & 1, m = (q >> 1) % ml, grp = (q >> 1) / ml;
      const double* w = wts + 9 + 3 * grp;
      const double* Fm = Fs + 6 * m + sI;
      Gs[q] = fma(w[0], Fm[0], fma(w[1], Fm[2], w[2] * Fm[4]));
    }
    if (lane == 0) Spk[G::st_len - 1] = 0.0;              // packed padding (never written)
    __syncwarp();

    FZ_T(0);
    const double wad = wts[fz::W_ADIV];
    // ---------------- passes over the column chunks [k0, k1) of Y
    auto pass = [&](auto PSc) {
      constexpr int PS = decltype(PSc)::value;
      // executed from the last chunks down: the bubble chunks (and with them
      // the L_b^-T operands) belong to pass 0 only
      constexpr int k1 = NKC - PS * CPP, k0 = (k1 > CPP) ? k1 - CPP : 0, NCH = k1 - k0;
      static_assert(!BIG || PS == 0 || k1 <= G::NLF, "bubble chunks in pass 0 only");
      // ---- B: Y chunks in registers, every lane generating exactly the Bsig
      // entries its registers need from the lane-ordered tables
      double2 Yf[NRB][NCH];
#pragma unroll
      for (int kc = k0; kc < k1; ++kc) {
        if (kc >= G::NLOW) {
#pragma unroll
          for (int I = 0; I < NRB; ++I) Yf[I][kc - k0] = make_double2(0.0, 0.0);
          continue;
        }
        const int m = 4 * kc + t;
        const int mm = m < ml ? m : ml - 1;       // padding lanes: zero table entries
        const double2 F0 = *reinterpret_cast<const double2*>(Fs + 6 * mm);
        const double2 F1 = *reinterpret_cast<const double2*>(Fs + 6 * mm + 2);
        const double2 F2 = *reinterpret_cast<const double2*>(Fs + 6 * mm + 4);
#pragma unroll
        for (int I = 0; I < NRB; ++I) {
          const double* tl = stab + G::TAB_LO + G::lo_off(I);
          const int fmt = G::fmt_low(I);
          double y0 = 0.0, y1 = 0.0, eh4 = 0.0;
          if (fmt != 1) {
            double b0, b1, b2;
            if (fmt == 4) {
              const double2 p = *reinterpret_cast<const double2*>(tl + (2 * kc) * 64 + 2 * lane);
              const double2 q = *reinterpret_cast<const double2*>(tl + (2 * kc + 1) * 64 + 2 * lane);
              b0 = p.x;
              b1 = p.y;
              b2 = q.x;
              eh4 = q.y;
            } else {
              b0 = tl[(3 * kc) * 32 + lane];
              b1 = tl[(3 * kc + 1) * 32 + lane];
              b2 = tl[(3 * kc + 2) * 32 + lane];
            }
            y0 = fma(b0, F0.x, fma(b1, F1.x, b2 * F2.x));
            y1 = fma(b0, F0.y, fma(b1, F1.y, b2 * F2.y));
          }
          if (fmt != 3) {
            const double eh = fmt == 4 ? eh4 : tl[kc * 32 + lane];
            const int wo = G::row_woff(8 * I + g);
            const int grp = wo < 30 ? (wo - 9) / 3 : 0;      // interior / padding rows: Ehat = 0
            const double2 Gm = *reinterpret_cast<const double2*>(Gs + 2 * (grp * ml + mm));
            y0 = fma(eh, Gm.x, y0);
            y1 = fma(eh, Gm.y, y1);
          }
          Yf[I][kc - k0] = make_double2(y0, y1);
        }
      }
      // bubble n-tiles bt whose chunk NLF + bt lies in this pass
      constexpr int b0t = (k0 > G::NLF ? k0 - G::NLF : 0);
      constexpr int b1t = (k1 - G::NLF < G::NBT ? k1 - G::NLF : G::NBT);
      if constexpr (b1t > b0t) {
#pragma unroll
        for (int I = 0; I < NRB; ++I) {
          const double* tb = stab + G::TAB_BU + G::bu_off(I);
          const int fmt = G::fmt_bub(I);
          double w0 = 0.0, w1 = 0.0, w2 = 0.0;
          if (fmt != 1) {
            const int wo = G::row_woff(8 * I + g);
            w0 = wts[wo];
            w1 = wts[wo + 1];
            w2 = wts[wo + 2];
          }
          double a[G::NKS];
#pragma unroll
          for (int ks = 0; ks < G::NKS; ++ks) {
            if (fmt == 4) {
              const double2 p = *reinterpret_cast<const double2*>(tb + (2 * ks) * 64 + 2 * lane);
              const double2 q = *reinterpret_cast<const double2*>(tb + (2 * ks + 1) * 64 + 2 * lane);
              a[ks] = fma(w2, q.y, fma(w1, q.x, fma(w0, p.y, p.x)));
            } else if (fmt == 3) {
              a[ks] = fma(w2, tb[(3 * ks + 2) * 32 + lane],
                          fma(w1, tb[(3 * ks + 1) * 32 + lane], w0 * tb[(3 * ks) * 32 + lane]));
            } else {
              a[ks] = tb[ks * 32 + lane];
            }
          }
#pragma unroll
          for (int bt = b0t; bt < b1t; ++bt) {
            double c0 = 0.0, c1 = 0.0;
#pragma unroll
            for (int ks = 0; ks < G::NKS; ++ks) dmma884(c0, c1, a[ks], LiR[bt][ks]);
            const int kc = G::NLF + bt - k0;
            Yf[I][kc].x += c0;
            Yf[I][kc].y += c1;
          }
        }
      }
      if constexpr (PS == 0) {
        __syncwarp();          // BIG: every lane is done with the factors aliased by Spk
        FZ_T(1);
      }
      // ---- C: S_T (+)= Y Y^T over this pass's chunks (DMMA); the packed
      // shared-memory copy carries the partial sums between passes (each
      // lane re-reads exactly the entries it stored)
      // one tile row I at a time: the I + 1 independent accumulator chains of
      // the row interleave (k outer, J inner) and share the A operand Y_I
#pragma unroll
      for (int I = 0; I < NRB - (G::STAIL ? 1 : 0); ++I) {
        const int i = 8 * I + g;
        double acc[NRB][2];
#pragma unroll
        for (int J = 0; J <= I; ++J) {
          acc[J][0] = acc[J][1] = 0.0;
          if constexpr (PS > 0) {
            const int j = 8 * J + 2 * t;
            if (i < nloc) {
              if (j <= i) acc[J][0] = Spk[pk(i, j)];
              if (j + 1 <= i) acc[J][1] = Spk[pk(i, j + 1)];
            }
          }
        }
#pragma unroll
        for (int kc = 0; kc < NCH; ++kc) {
#pragma unroll
          for (int J = 0; J <= I; ++J) dmma884(acc[J][0], acc[J][1], Yf[I][kc].x, Yf[J][kc].x);
          if (G::HALF && k0 + kc == NKC - 1) continue;     // odd columns of the last chunk are zero
#pragma unroll
          for (int J = 0; J <= I; ++J) dmma884(acc[J][0], acc[J][1], Yf[I][kc].y, Yf[J][kc].y);
        }
#pragma unroll
        for (int J = 0; J <= I; ++J) {
          const int j = 8 * J + 2 * t;
          double c0 = acc[J][0], c1 = acc[J][1];
          if constexpr (PS == NPASS - 1) {
            if (i < nu && j < nu) c0 = fma(wad, __ldg(tab + T::o_adiv + i * nu + j), c0);
            if (i < nu && j + 1 < nu) c1 = fma(wad, __ldg(tab + T::o_adiv + i * nu + j + 1), c1);
          }
          if (i < nloc) {
            if (j <= i) Spk[pk(i, j)] = c0;
            if (j + 1 <= i) Spk[pk(i, j + 1)] = c1;
          }
        }
        asm volatile("" ::: "memory");   // keep the epilogue loads row by row (registers)
      }
      // the last tile row holds TAIL real rows (Vhat rows: no adiv term):
      // NRB tiles of DMMAs for them would be mostly padding, so their entries
      // S[i0][j] = Y[i0] . Y[j] are plain dot products -- row i0 of Y is
      // broadcast from the lanes g == rr of the last tile (same t: same
      // columns), every lane dots it with its own rows, the four t lanes of
      // a row add up
      if constexpr (G::STAIL) {
#pragma unroll
        for (int rr = 0; rr < G::TAIL; ++rr) {
          const int i0 = 8 * (NRB - 1) + rr;
          double2 yt[NCH];
#pragma unroll
          for (int kc = 0; kc < NCH; ++kc) {
            yt[kc].x = __shfl_sync(0xffffffffu, Yf[NRB - 1][kc].x, 4 * rr + t);
            yt[kc].y = __shfl_sync(0xffffffffu, Yf[NRB - 1][kc].y, 4 * rr + t);
          }
#pragma unroll
          for (int I = 0; I < NRB; ++I) {
            double pd = 0.0;
#pragma unroll
            for (int kc = 0; kc < NCH; ++kc) {
              pd = fma(Yf[I][kc].x, yt[kc].x, pd);
              if (G::HALF && k0 + kc == NKC - 1) continue;
              pd = fma(Yf[I][kc].y, yt[kc].y, pd);
            }
            pd += __shfl_xor_sync(0xffffffffu, pd, 1);
            pd += __shfl_xor_sync(0xffffffffu, pd, 2);
            const int j = 8 * I + g;
            if (t == 0 && j <= i0) {
              if constexpr (PS > 0) pd += Spk[pk(i0, j)];
              Spk[pk(i0, j)] = pd;
            }
          }
        }
      }
    };
    pass(IC<0>{});
    if constexpr (NPASS > 1) pass(IC<1>{});
    if constexpr (NPASS > 2) pass(IC<2>{});
    if constexpr (NPASS > 3) pass(IC<3>{});
    static_assert(NPASS <= 4, "passes");
    __syncwarp();
    {
      const double2* src = reinterpret_cast<const double2*>(Spk);
      double2* dst = reinterpret_cast<double2*>(ST + e * G::st_len);
      for (int q = lane; q < G::st_len / 2; q += 32) dst[q] = src[q];
    }

    FZ_T(2);
    // ---------------- D: double Schur on the element-local S_T, register
    // resident (ds_reg.cuh): one sweep over the 8x8 pivot tiles of S_oo with
    // S_co and an identity block as right-hand sides, then Sd_T, X and
    // S_oo^-1 as X Y^T products of register tiles
    if constexpr (DS) {
      auto S = [&](int a, int b) { return a >= b ? Spk[pk(a, b)] : Spk[pk(b, a)]; };
      if constexpr (BIG) {
        // the tile slots over the interior rows of the packed S_T: S_oo and
        // S_co are in registers before the first slot is written, S_cc (read
        // last) lies in the rows before and after them
        constexpr int T0 = even(pk(G::NEM, 0));
        static_assert(T0 + dsr::Geo<K>::PER_WARP <= pk(G::NEM + G::NI, 0), "slots inside the interior rows");
        if (!dsr::element_pm<K, decltype(S), dsr::NoSync, true, true>(S, Spk + T0, ext + e * L::len,
                                                                   Sd + e * L::sd_len))
          bad |= 2;
      } else {
        if (!dsr::element<K>(S, U, ext + e * L::len, Sd + e * L::sd_len)) bad |= 2;
      }
    }
    FZ_T(3);
    if (lane == 0 && info) info[e] = bad;
    __syncwarp();
  }
}

#ifndef MCS_FZ_PAIR4
#define MCS_FZ_PAIR4 false   // k = 4: the three warps of a sub-partition in lockstep per element (A/B)
#endif
#ifndef MCS_FZ_WPB4
#define MCS_FZ_WPB4 12   // warps per CTA at k = 4 (tools/fused_prof.py sweeps it)
#endif

template <int K, int WPB, int MINB, bool DS, bool PAIR = false>
static int launch_condense_fused(int64_t nt, const double* W, int nwgt, const double* tab,
                                 double* ST, double* ext, double* Sd, int* info,
                                 cudaStream_t st) {
  using G = fz::Geo<K>;
  auto kern = condense_fused_kernel<K, WPB, MINB, DS, PAIR>;
  const size_t smem =
      ((G::BIG ? 0 : G::TAB_SMEM) + static_cast<size_t>(WPB) * G::PER_WARP) * sizeof(double);
  double* gtab = nullptr;
  if constexpr (G::BIG) {
    // lane-ordered tables in a library-owned global buffer, rebuilt on the
    // caller's stream at every call (concurrent calls with DIFFERENT tables
    // for the same k on different streams are not supported)
    static double* buf = nullptr;
    if (!buf && cudaMalloc(&buf, G::TAB_SMEM * sizeof(double)) != cudaSuccess) return launch_status();
    gtab = buf;
    fused_lane_tables_kernel<K><<<16, 256, 0, st>>>(tab, gtab);
  }
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0, dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * WPB, smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  const int64_t want = (nt + WPB - 1) / WPB, cap = static_cast<int64_t>(per_sm) * nsm;
  const int grid = static_cast<int>(want < cap ? want : cap);
  kern<<<grid, 32 * WPB, smem, st>>>(W, nwgt, tab, gtab, ST, ext, Sd, info, nt);
  return launch_status();
}

// k = 5, 6 without the double Schur (mcs_condense_gen routes here)
int launch_condense_fused_big(int k, int64_t nt, const double* W, int nwgt, const double* tab,
                              double* ST, int* info, cudaStream_t st) {
  // pairs of warps start every element together: default at k = 6 only
  // (MCS_FZ_PAIR=0 / 1 forces it off / on for k = 5, 6)
  static const int pair = getenv("MCS_FZ_PAIR") ? atoi(getenv("MCS_FZ_PAIR")) : -1;
  switch (k) {
    case 5:
      if (pair == 1) return launch_condense_fused<5, 8, 1, false, true>(nt, W, nwgt, tab, ST, nullptr, nullptr, info, st);
      return launch_condense_fused<5, 4, 2, false>(nt, W, nwgt, tab, ST, nullptr, nullptr, info, st);
    case 6:
      if (pair != 0) return launch_condense_fused<6, 8, 1, false, true>(nt, W, nwgt, tab, ST, nullptr, nullptr, info, st);
      return launch_condense_fused<6, 4, 2, false>(nt, W, nwgt, tab, ST, nullptr, nullptr, info, st);
  }
  return -1000;
}

}  // namespace mcs

using namespace mcs;

MCS_API int mcs_fused_table_len(int k) {
  switch (k) {
    case 2: return FTab<2>::len;
    case 3: return FTab<3>::len;
    case 4: return FTab<4>::len;
    case 5: return FTab<5>::len;
    case 6: return FTab<6>::len;
  }
  return -1;
}

MCS_API int mcs_condense_fused(int k, int64_t nt, const double* W, int nwgt, const double* tables,
                               double* S_packed, double* ext,
                               double* Sd_packed, int* info, void* stream) {
  if (nt <= 0) return 0;
  if (nwgt < 30) return -1000;
  auto st = static_cast<cudaStream_t>(stream);
  switch (k) {
    // one CTA per SM: the compact tables once per CTA, one element per warp
    case 2: return launch_condense_fused<2, 16, 1, true>(nt, W, nwgt, tables, S_packed, ext, Sd_packed, info, st);
    case 3: return launch_condense_fused<3, 12, 1, true>(nt, W, nwgt, tables, S_packed, ext, Sd_packed, info, st);
    case 4: return launch_condense_fused<4, MCS_FZ_WPB4, 1, true, MCS_FZ_PAIR4>(nt, W, nwgt, tables, S_packed, ext, Sd_packed, info, st);
    // k = 5, 6: the passes pipeline with the double Schur as phase D
    case 5: return launch_condense_fused<5, 4, 2, true>(nt, W, nwgt, tables, S_packed, ext, Sd_packed, info, st);
    case 6: return launch_condense_fused<6, 4, 2, true>(nt, W, nwgt, tables, S_packed, ext, Sd_packed, info, st);
  }
  return -1000;
}

#ifdef MCS_FUSED_PROF
extern "C" __attribute__((visibility("default"))) int fz_prof_gen(int k, int64_t nt, const double* W, int nwgt,
                                                                  const double* tables, double* S_packed,
                                                                  int* info, void* stream) {
  return mcs::launch_condense_fused_big(k, nt, W, nwgt, tables, S_packed, info,
                                        static_cast<cudaStream_t>(stream));
}
extern "C" __attribute__((visibility("default"))) void fz_prof_read(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, mcs::g_fz_prof, 8 * sizeof(unsigned long long));
}
#endif
