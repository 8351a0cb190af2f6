// Structured sigma/omega condensation on B200.
//
// The reference eliminates (sigma, omega) with a dense LU of
// M = [[-msig, bws^T], [bws, 0]] per element (condensation.py:161-176):
//
//     S_T = adiv - Bsig M^-1 Bsig^T,   Bsig = [bus; bhs]   (nloc x ns).
//
// The MCS element spaces make M far from dense (basis.py:288-337):
//   * the stress basis is Dubiner(P^{k-1}) x {3 trace-free generators}
//     (dof 3m + a) plus 3k nt-bubbles built from the degree-k Dubiner
//     functions; the Dubiner basis is L2-orthonormal on the reference cell
//     and sigma = J^-T sigma_hat J^T maps each generator on its own, so
//     msig = blockdiag(A_0, ..., A_{ml-1}, Mb): ml 3x3 blocks and one
//     3k x 3k bubble block;
//   * omega is P^{k-1} and the bubbles are orthogonal to P^{k-1}, so
//     bws = [Phi (x) s | 0] with a fixed invertible Phi (ml x ml) and one
//     3-vector s = detJ skew(T_a) per element.
// (Checked on the reference's own blocks: off-structure entries <= 3e-15
// relative, tests/test_struct_condense.py.)
// With that structure the (1,1) block of M^-1 is block diagonal (Phi
// cancels exactly):  -[M^-1]_11 = blockdiag(Pi_0, ..., Pi_{ml-1}, Mb^-1),
//     Pi_m = A_m^-1 - A_m^-1 s s^T A_m^-1 / (s^T A_m^-1 s)   (rank 2, PSD),
// hence
//     S_T = adiv + Y Y^T,   Y = [B_m F_m (m < ml) | B_b L_b^-T]  (nloc x k(k+4))
// with Pi_m = F_m F_m^T (F_m = L_m^-T Q_m, L_m = chol(A_m), Q_m an
// orthonormal basis of (L_m^-1 s)^perp) and Mb = L_b L_b^T.
//
// Kernel (one CTA per element at a time, persistent, 2-stage ring of 1-D
// bulk async copies (TMA engine) bringing in the next element's compact
// record while the current one is processed):
//   A  warp 0: Cholesky of Mb in registers (lane = row, shuffles) and L_b^-1;
//      warp 1: F_m for every 3x3 block (lane = block);
//   B  thread per row of Bsig: Y row = (B_m F_m | L_b^-1 b_bubble);
//   C  S_T = adiv + Y Y^T on the FP64 tensor cores (DMMA m8n8k4, 8x8 output
//      tiles of the lower triangle spread over the warps), written packed.
#include <cstdlib>

#include "ds_warp.cuh"

namespace mcs {

// compact element record of the structured path (doubles, even segments):
//   [s (3) + pad | A_m 3x3 row-major (ml blocks) | Mb (nb x nb) |
//    Bsig = [bus; bhs] (nloc x ns) | adiv (nu x nu)]
template <int K>
struct SRec {
  using Z = Sizes<K>;
  static constexpr int ml = K * (K + 1) / 2;
  static constexpr int nl = 3 * ml;
  static constexpr int nb = 3 * K;
  static constexpr int ny = 2 * ml + nb;
  static constexpr int o_s = 0;
  static constexpr int o_A = 4;
  static constexpr int o_Mb = o_A + even(9 * ml);
  static constexpr int o_B = o_Mb + even(nb * nb);
  static constexpr int o_adiv = o_B + even(Z::nloc * Z::ns);
  static constexpr int len = o_adiv + even(Z::nu * Z::nu);
  static_assert(nl + nb == Z::ns, "stress space = low part + nt-bubbles");
  static_assert(Z::nw == ml, "omega space = P^{k-1}");
};

namespace cs {

template <int K, int W>
struct Geo {
  using Z = Sizes<K>;
  using R = SRec<K>;
  static constexpr int NYP = (R::ny + 7) / 8 * 8;                // Y columns, padded
  static constexpr int YST = (NYP % 16 == 8) ? NYP : NYP + 8;    // conflict-free 128-bit rows
  static constexpr int NR = (Z::nloc + 7) / 8 * 8;               // Y rows, padded
  static constexpr int NRB = NR / 8;
  static constexpr int NTILE = NRB * (NRB + 1) / 2;
  static constexpr int o_Y = 2 * R::len;
  static constexpr int o_F = o_Y + NR * YST;
  static constexpr int o_L = o_F + even(6 * R::ml);
  static constexpr int o_Li = o_L + even(R::nb * R::nb);
  static constexpr int SMEM = o_Li + even(R::nb * R::nb);        // doubles
  static_assert(W >= 2, "warp 0: bubble Cholesky, warp 1: 3x3 blocks");
  static_assert(R::ml <= 32 && R::nb <= 32, "one lane per block / bubble row");
};

}  // namespace cs

template <int K, int W, int MINB>
__global__ void __launch_bounds__(32 * W, MINB)
    condense_struct_kernel(const double* __restrict__ recs, double* __restrict__ ST,
                           int* __restrict__ info, int64_t nt) {
  using Z = Sizes<K>;
  using R = SRec<K>;
  using G = cs::Geo<K, W>;
  constexpr int ns = Z::ns, nu = Z::nu, nloc = Z::nloc, ml = R::ml, nl = R::nl, nb = R::nb;
  constexpr int T = 32 * W, YST = G::YST, NYP = G::NYP;
  constexpr int st_len = even(npk(nloc));
  extern __shared__ __align__(128) double smem[];
  double* Y = smem + G::o_Y;
  double* F = smem + G::o_F;
  double* Ls = smem + G::o_L;
  double* Li = smem + G::o_Li;
  __shared__ __align__(8) uint64_t full[2];
  __shared__ int bad[2];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;

  for (int i = tid; i < G::NR * YST; i += T) Y[i] = 0.0;   // padding rows stay zero
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    fence_barrier_init();
    bad[0] = bad[1] = 0;
  }
  __syncthreads();
  int64_t e = blockIdx.x;
  if (tid == 0 && e < nt) {
    mbar_expect_tx(&full[0], R::len * 8);
    bulk_g2s(smem, recs + e * R::len, R::len * 8, &full[0]);
  }
#pragma unroll 1
  for (int it = 0; e < nt; ++it, e += gridDim.x) {
    const int s = it & 1;
    const double* rec = smem + s * R::len;
    if (tid == 0) {
      bad[s ^ 1] = 0;
      const int64_t nx = e + gridDim.x;
      if (nx < nt) {   // the other stage was released by the previous iteration's barrier
        mbar_expect_tx(&full[s ^ 1], R::len * 8);
        bulk_g2s(smem + (s ^ 1) * R::len, recs + nx * R::len, R::len * 8, &full[s ^ 1]);
      }
    }
    mbar_wait(&full[s], (it >> 1) & 1);

    // ---- A: bubble Cholesky + inverse (warp 0), 3x3 block factors (warp 1)
    if (warp == 0) {
      const int i = lane < nb ? lane : 0;
      double a[nb], l[nb];
#pragma unroll
      for (int c = 0; c < nb; ++c) a[c] = rec[R::o_Mb + i * nb + c];
      bool ok = true;
#pragma unroll
      for (int j = 0; j < nb; ++j) {
        const double d = __shfl_sync(0xffffffffu, a[j], j);
        ok &= d > 0.0;
        const double r = rsqrt_nr(d);
        l[j] = (lane == j) ? d * r : a[j] * r;          // L[i][j] (i >= j significant)
#pragma unroll
        for (int c = j + 1; c < nb; ++c) a[c] = fma(-l[j], __shfl_sync(0xffffffffu, l[j], c), a[c]);
      }
      if (lane < nb) {
#pragma unroll
        for (int c = 0; c < nb; ++c) Ls[lane * nb + c] = l[c];
      }
      if (lane == 0 && !ok) bad[s] = 1;
      __syncwarp();
      if (lane < nb) {   // column `lane` of L^-1 by forward substitution
        double x[nb];
#pragma unroll
        for (int j = 0; j < nb; ++j) {
          double acc = (j == lane) ? 1.0 : 0.0;
#pragma unroll
          for (int q = 0; q < j; ++q) acc = fma(-Ls[j * nb + q], x[q], acc);
          x[j] = acc / Ls[j * nb + j];
        }
#pragma unroll
        for (int j = 0; j < nb; ++j) Li[j * nb + lane] = x[j];
      }
    } else if (warp == 1 && lane < ml) {
      const double* A = rec + R::o_A + 9 * lane;
      const double s0 = rec[R::o_s], s1 = rec[R::o_s + 1], s2 = rec[R::o_s + 2];
      const double a00 = A[0], a10 = A[3], a11 = A[4], a20 = A[6], a21 = A[7], a22 = A[8];
      // L = chol(A)
      const double l00 = sqrt(a00), i00 = 1.0 / l00;
      const double l10 = a10 * i00, l20 = a20 * i00;
      const double d11 = a11 - l10 * l10;
      const double l11 = sqrt(d11), i11 = 1.0 / l11;
      const double l21 = (a21 - l20 * l10) * i11;
      const double d22 = a22 - l20 * l20 - l21 * l21;
      const double l22 = sqrt(d22), i22 = 1.0 / l22;
      if (!(a00 > 0.0 && d11 > 0.0 && d22 > 0.0)) bad[s] = 1;
      // u = L^-1 s / |L^-1 s|
      const double v0 = s0 * i00;
      const double v1 = (s1 - l10 * v0) * i11;
      const double v2 = (s2 - l20 * v0 - l21 * v1) * i22;
      const double vn = rsqrt_nr(v0 * v0 + v1 * v1 + v2 * v2);
      const double u0 = v0 * vn, u1 = v1 * vn, u2 = v2 * vn;
      // Q = [q1 q2], orthonormal basis of u^perp: q1 from the axis least
      // aligned with u, q2 = u x q1
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
      // F = L^-T Q  (back substitution with L^T)
      const double f20 = q12 * i22, f21 = q22 * i22;
      const double f10 = (q11 - l21 * f20) * i11, f11 = (q21 - l21 * f21) * i11;
      const double f00 = (q10 - l10 * f10 - l20 * f20) * i00;
      const double f01 = (q20 - l10 * f11 - l20 * f21) * i00;
      double* Fm = F + 6 * lane;
      Fm[0] = f00;
      Fm[1] = f01;
      Fm[2] = f10;
      Fm[3] = f11;
      Fm[4] = f20;
      Fm[5] = f21;
    }
    __syncthreads();

    // ---- B: Y rows (thread per row of Bsig)
    for (int i = tid; i < nloc; i += T) {
      const double* b = rec + R::o_B + i * ns;
      double* y = Y + i * YST;
#pragma unroll
      for (int m = 0; m < ml; ++m) {
        const double b0 = b[3 * m], b1 = b[3 * m + 1], b2 = b[3 * m + 2];
        const double* Fm = F + 6 * m;
        y[2 * m] = fma(b0, Fm[0], fma(b1, Fm[2], b2 * Fm[4]));
        y[2 * m + 1] = fma(b0, Fm[1], fma(b1, Fm[3], b2 * Fm[5]));
      }
      double xb[nb];
#pragma unroll
      for (int q = 0; q < nb; ++q) xb[q] = b[nl + q];
#pragma unroll
      for (int j = 0; j < nb; ++j) {
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q <= j; ++q) acc = fma(Li[j * nb + q], xb[q], acc);
        y[2 * ml + j] = acc;
      }
#pragma unroll
      for (int c = R::ny; c < NYP; ++c) y[c] = 0.0;
    }
    __syncthreads();

    // ---- C: S_T = adiv + Y Y^T, lower 8x8 tiles on the FP64 tensor cores
    double* Se = ST + e * st_len;
#pragma unroll 1
    for (int q = warp; q < G::NTILE; q += W) {
      int I = 0, rem = q;
      while (rem > I) {
        rem -= I + 1;
        ++I;
      }
      const int J = rem;
      const double* ya = Y + (8 * I + g) * YST + 2 * t;
      const double* yb = Y + (8 * J + g) * YST + 2 * t;
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int kc = 0; kc < NYP / 8; ++kc) {
        const double2 a = *reinterpret_cast<const double2*>(ya + 8 * kc);
        const double2 bb = *reinterpret_cast<const double2*>(yb + 8 * kc);
        dmma884(c0, c1, a.x, bb.x);
        dmma884(c0, c1, a.y, bb.y);
      }
      const int i = 8 * I + g, j = 8 * J + 2 * t;
      if (i < nloc) {
        if (j <= i) Se[pk(i, j)] = c0 + ((i < nu && j < nu) ? rec[R::o_adiv + i * nu + j] : 0.0);
        if (j + 1 <= i)
          Se[pk(i, j + 1)] = c1 + ((i < nu && j + 1 < nu) ? rec[R::o_adiv + i * nu + j + 1] : 0.0);
      }
    }
    __syncthreads();
    if (tid == 0 && info) info[e] = bad[s];
  }
}

// ---- generation fused (k = 5, 6, where Y does not fit a warp's registers):
// the compact record is never written; each CTA regenerates Bsig rows from
// the L2-resident reference tables (FTab, the fused kernel's tables) and the
// element's geometry weights, so the per-element HBM traffic is the 240-byte
// weight row in and S_T out.  Same phases as condense_struct_kernel, with
// shared memory only for Y and the factors (4 CTAs per SM).
namespace cs {
template <int K, int W>
struct GeoGen {
  using Z = Sizes<K>;
  using R = SRec<K>;
  static constexpr int NYP = (R::ny + 7) / 8 * 8;
  static constexpr int YST = (NYP % 16 == 8) ? NYP : NYP + 8;
  static constexpr int NR = (Z::nloc + 7) / 8 * 8;
  static constexpr int NRB = NR / 8;
  static constexpr int NTILE = NRB * (NRB + 1) / 2;
  static constexpr int o_Y = 0;
  static constexpr int o_F = o_Y + NR * YST;
  static constexpr int o_L = o_F + even(6 * R::ml);
  static constexpr int o_Li = o_L + even(R::nb * R::nb);
  static constexpr int o_Rd = o_Li + even(R::nb * R::nb);
  static constexpr int o_w = o_Rd + even(R::nb);
  static constexpr int SMEM = o_w + 36;
};

// Bsig row i: 0 facet, 1 interior bubble, 2 Vhat, 3 padding (refblocks.py)
template <int K>
__device__ __forceinline__ int gen_row_woff(int i) {
  using Z = Sizes<K>;
  return i < Z::n_em ? 9 + 3 * (i / (K + 1))
                     : ((i >= Z::nu && i < Z::nloc) ? 18 + 3 * ((i - Z::nu) / K) : 30);
}
}  // namespace cs

template <int K, int W, int MINB, bool DS>
__global__ void __launch_bounds__(32 * W, MINB)
    condense_gen_kernel(const double* __restrict__ Wg, int nwgt, const double* __restrict__ tab,
                        double* __restrict__ ST, double* __restrict__ ext,
                        double* __restrict__ Sd, int* __restrict__ info, int64_t nt) {
  using Z = Sizes<K>;
  using R = SRec<K>;
  using TB = FTab<K>;
  using G = cs::GeoGen<K, W>;
  constexpr int ns = Z::ns, nu = Z::nu, nloc = Z::nloc, ml = R::ml, nl = R::nl, nb = R::nb;
  constexpr int T = 32 * W, YST = G::YST, NYP = G::NYP;
  constexpr int st_len = even(npk(nloc));
  extern __shared__ __align__(128) double smem[];
  double* Y = smem + G::o_Y;
  double* F = smem + G::o_F;
  double* Ls = smem + G::o_L;
  double* Li = smem + G::o_Li;
  double* Rd = smem + G::o_Rd;
  double* wts = smem + G::o_w;
  __shared__ int bad;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  for (int i = tid; i < G::NR * YST; i += T) Y[i] = 0.0;
  if (tid < 6) wts[30 + tid] = 0.0;
  const double2* G4 = reinterpret_cast<const double2*>(tab + TB::o_G4);
#pragma unroll 1
  for (int64_t e = blockIdx.x; e < nt; e += gridDim.x) {
    if (tid < 30) wts[tid] = __ldg(Wg + e * nwgt + tid);
    if (tid == 0) bad = 0;
    __syncthreads();
    // ---- A: bubble block (warp 0), 3x3 block factors (warp 1)
    if (warp == 0) {
      const int i = lane < nb ? lane : 0;
      double a[nb], l[nb];
#pragma unroll
      for (int c = 0; c < nb; ++c) a[c] = 0.0;
#pragma unroll
      for (int r = 0; r < 6; ++r) {
        const double w = wts[r];
#pragma unroll
        for (int c = 0; c < nb; ++c) a[c] = fma(w, __ldg(tab + TB::o_Mb + (r * nb + i) * nb + c), a[c]);
      }
      bool ok = true;
#pragma unroll
      for (int j = 0; j < nb; ++j) {
        const double d = __shfl_sync(0xffffffffu, a[j], j);
        ok &= d > 0.0;
        const double rr = rsqrt_nr(d);
        if (lane == 0) Rd[j] = rr;
        l[j] = a[j] * rr;
#pragma unroll
        for (int c = j + 1; c < nb; ++c) a[c] = fma(-l[j], __shfl_sync(0xffffffffu, l[j], c), a[c]);
      }
      if (lane < nb) {
#pragma unroll
        for (int c = 0; c < nb; ++c) Ls[lane * nb + c] = l[c];
      }
      if (lane == 0 && !ok) bad = 1;
      __syncwarp();
      if (lane < nb) {   // column `lane` of L_b^-1
        double x[nb];
#pragma unroll
        for (int j = 0; j < nb; ++j) {
          double acc = (j == lane) ? 1.0 : 0.0;
#pragma unroll
          for (int q = 0; q < j; ++q) acc = fma(-Ls[j * nb + q], x[q], acc);
          x[j] = acc * Rd[j];
          Li[j * nb + lane] = x[j];
        }
      }
    } else if (warp == 1 && lane < ml) {
      double A[9];
#pragma unroll
      for (int q = 0; q < 9; ++q) A[q] = 0.0;
#pragma unroll
      for (int r = 0; r < 6; ++r) {
        const double w = wts[r];
#pragma unroll
        for (int q = 0; q < 9; ++q) A[q] = fma(w, __ldg(tab + TB::o_A + (r * ml + lane) * 9 + q), A[q]);
      }
      const double s0 = wts[6], s1 = wts[7], s2 = wts[8];
      const double a00 = A[0], a10 = A[3], a11 = A[4], a20 = A[6], a21 = A[7], a22 = A[8];
      const double i00 = rsqrt_nr(a00);
      const double l10 = a10 * i00, l20 = a20 * i00;
      const double d11 = a11 - l10 * l10;
      const double i11 = rsqrt_nr(d11);
      const double l21 = (a21 - l20 * l10) * i11;
      const double d22 = a22 - l20 * l20 - l21 * l21;
      const double i22 = rsqrt_nr(d22);
      if (!(a00 > 0.0 && d11 > 0.0 && d22 > 0.0)) bad = 1;
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
      double* Fm = F + 6 * lane;
      Fm[0] = (q10 - l10 * f10 - l20 * f20) * i00;
      Fm[1] = (q20 - l10 * f11 - l20 * f21) * i00;
      Fm[2] = f10;
      Fm[3] = f11;
      Fm[4] = f20;
      Fm[5] = f21;
    }
    __syncthreads();
    // ---- B: Y rows (thread per row), Bsig entries generated on the fly
    for (int i = tid; i < nloc; i += T) {
      const int wo = cs::gen_row_woff<K>(i);
      const double w0 = wts[wo], w1 = wts[wo + 1], w2 = wts[wo + 2];
      const double2* rowp = G4 + 2 * i * ns;
      auto gen = [&](int c) {
        const double2 v01 = __ldg(rowp + 2 * c), v23 = __ldg(rowp + 2 * c + 1);
        return fma(w2, v23.y, fma(w1, v23.x, fma(w0, v01.y, v01.x)));
      };
      double* y = Y + i * YST;
#pragma unroll 2
      for (int m = 0; m < ml; ++m) {
        const double b0 = gen(3 * m), b1 = gen(3 * m + 1), b2 = gen(3 * m + 2);
        const double* Fm = F + 6 * m;
        y[2 * m] = fma(b0, Fm[0], fma(b1, Fm[2], b2 * Fm[4]));
        y[2 * m + 1] = fma(b0, Fm[1], fma(b1, Fm[3], b2 * Fm[5]));
      }
      double xb[nb];
#pragma unroll
      for (int q = 0; q < nb; ++q) xb[q] = gen(nl + q);
#pragma unroll
      for (int j = 0; j < nb; ++j) {
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q <= j; ++q) acc = fma(Li[j * nb + q], xb[q], acc);
        y[2 * ml + j] = acc;
      }
#pragma unroll
      for (int c = R::ny; c < NYP; ++c) y[c] = 0.0;
    }
    __syncthreads();
    // ---- C: S_T = adiv + Y Y^T (DMMA), packed lower
    double* Se = ST + e * st_len;
    const double wad = wts[27];
#pragma unroll 1
    for (int q = warp; q < G::NTILE; q += W) {
      int I = 0, rem = q;
      while (rem > I) {
        rem -= I + 1;
        ++I;
      }
      const int J = rem;
      const double* ya = Y + (8 * I + g) * YST + 2 * t;
      const double* yb = Y + (8 * J + g) * YST + 2 * t;
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int kc = 0; kc < NYP / 8; ++kc) {
        const double2 a = *reinterpret_cast<const double2*>(ya + 8 * kc);
        const double2 bb = *reinterpret_cast<const double2*>(yb + 8 * kc);
        dmma884(c0, c1, a.x, bb.x);
        dmma884(c0, c1, a.y, bb.y);
      }
      const int i = 8 * I + g, j = 8 * J + 2 * t;
      if (i < nloc) {
        if (j <= i)
          Se[pk(i, j)] = c0 + ((i < nu && j < nu) ? wad * __ldg(tab + TB::o_adiv + i * nu + j) : 0.0);
        if (j + 1 <= i)
          Se[pk(i, j + 1)] =
              c1 + ((i < nu && j + 1 < nu) ? wad * __ldg(tab + TB::o_adiv + i * nu + j + 1) : 0.0);
      }
    }
    __syncthreads();
    if constexpr (DS) {
      // ---- D: the double Schur of this element (condensation.py:207-226),
      // fused: S_T is read back from global memory just written by this CTA
      // (L2; plain loads, not the non-coherent path), the four warps split the
      // work (ds_warp.cuh), Y's shared memory holds L, L^-1 and W.
      using DG = dsw::Geo<K>;
      static_assert(even(DG::L_LEN) + DG::LI_LEN + DG::W_LEN + DG::NI <= G::NR * YST,
                    "double-Schur buffers fit in Y");
      double* Ls = Y;
      double* LIs = Ls + even(DG::L_LEN);
      double* Wd = LIs + DG::LI_LEN;
      double* rdd = Wd + DG::W_LEN;
      const double* Sp = Se;
      auto Sg = [&](int a, int b) { return Sp[a >= b ? pk(a, b) : pk(b, a)]; };
      if (warp == 0) {
        if (!dsw::chol_soo<K>(Sg, Ls, rdd) && lane == 0) atomicOr(&bad, 2);
      } else {
        dsw::stage_soc<K>(Sg, Wd, tid - 32, T - 32);
      }
      __syncthreads();
      if (warp == 0) dsw::linv<K>(Ls, rdd, LIs);
      __syncthreads();
      for (int J = warp; J < DG::NCB; J += W) dsw::w_block<K>(LIs, Wd, J);
      __syncthreads();
      using EL = ExtLayout<K>;
      dsw::out_tiles<K>(Sg, LIs, Wd, ext + e * EL::len, Sd + e * EL::sd_len, warp, W);
      __syncthreads();
    }
    if (tid == 0 && info) info[e] = bad;
  }
}

static int cs_num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

template <int K, int W, int MINB>
static int launch_condense_struct(const double* recs, double* ST, int* info, int64_t nt,
                                  cudaStream_t st) {
  using G = cs::Geo<K, W>;
  auto kern = condense_struct_kernel<K, W, MINB>;
  const size_t smem = G::SMEM * sizeof(double);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * W, smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  const int64_t cap = static_cast<int64_t>(per_sm) * cs_num_sms();
  const int grid = static_cast<int>(nt < cap ? nt : cap);
  kern<<<grid, 32 * W, smem, st>>>(recs, ST, info, nt);
  return launch_status();
}

template <int K, int W, int MINB, bool DS = false>
static int launch_condense_gen(const double* Wg, int nwgt, const double* tab, double* ST, int* info,
                               int64_t nt, cudaStream_t st, double* ext = nullptr,
                               double* Sd = nullptr) {
  using G = cs::GeoGen<K, W>;
  auto kern = condense_gen_kernel<K, W, MINB, DS>;
  const size_t smem = G::SMEM * sizeof(double);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * W, smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  const int64_t cap = static_cast<int64_t>(per_sm) * cs_num_sms();
  const int grid = static_cast<int>(nt < cap ? nt : cap);
  kern<<<grid, 32 * W, smem, st>>>(Wg, nwgt, tab, ST, ext, Sd, info, nt);
  return launch_status();
}

}  // namespace mcs

using namespace mcs;

namespace mcs {
int launch_condense_fused_big(int k, int64_t nt, const double* W, int nwgt, const double* tab,
                              double* ST, int* info, cudaStream_t st);
}

MCS_API int mcs_condense_gen(int k, int64_t nt, const double* W, int nwgt, const double* tables,
                             double* S_packed, int* info, void* stream) {
  if (nt <= 0) return 0;
  if (nwgt < 30) return -1000;
  auto st = static_cast<cudaStream_t>(stream);
  // k = 5, 6: the warp-per-element fused pipeline in passes (condense_fused.cu);
  // MCS_GEN=1: the CTA-per-element kernel of this file (A/B measurements)
  static const int gen = getenv("MCS_GEN") ? atoi(getenv("MCS_GEN")) : 2;
  if (k >= 5 && gen != 1) return launch_condense_fused_big(k, nt, W, nwgt, tables, S_packed, info, st);
  switch (k) {
    case 2: return launch_condense_gen<2, 4, 4>(W, nwgt, tables, S_packed, info, nt, st);
    case 3: return launch_condense_gen<3, 4, 4>(W, nwgt, tables, S_packed, info, nt, st);
    case 4: return launch_condense_gen<4, 4, 4>(W, nwgt, tables, S_packed, info, nt, st);
    case 5: return launch_condense_gen<5, 4, 4>(W, nwgt, tables, S_packed, info, nt, st);
    case 6: return launch_condense_gen<6, 4, 4>(W, nwgt, tables, S_packed, info, nt, st);
  }
  return -1000;
}

MCS_API int mcs_condense_gen_ds(int k, int64_t nt, const double* W, int nwgt, const double* tables,
                                double* S_packed, double* ext, double* Sd_packed, int* info,
                                void* stream) {
  if (nt <= 0) return 0;
  if (nwgt < 30) return -1000;
  auto st = static_cast<cudaStream_t>(stream);
  switch (k) {
    case 5: return launch_condense_gen<5, 4, 4, true>(W, nwgt, tables, S_packed, info, nt, st, ext, Sd_packed);
    case 6: {
      static const int v = getenv("MCS_GENDS6") ? atoi(getenv("MCS_GENDS6")) : 4;
      if (v == 3) return launch_condense_gen<6, 4, 3, true>(W, nwgt, tables, S_packed, info, nt, st, ext, Sd_packed);
      return launch_condense_gen<6, 4, 4, true>(W, nwgt, tables, S_packed, info, nt, st, ext, Sd_packed);
    }
  }
  return -1000;
}

MCS_API int mcs_srec_len(int k) {
  switch (k) {
    case 2: return SRec<2>::len;
    case 3: return SRec<3>::len;
    case 4: return SRec<4>::len;
    case 5: return SRec<5>::len;
    case 6: return SRec<6>::len;
  }
  return -1;
}

MCS_API int mcs_condense_struct(int k, int64_t nt, const double* srecords, double* S_packed,
                                int* info, void* stream) {
  if (nt <= 0) return 0;
  auto st = static_cast<cudaStream_t>(stream);
  switch (k) {
    case 2: return launch_condense_struct<2, 4, 1>(srecords, S_packed, info, nt, st);
    case 3: return launch_condense_struct<3, 4, 1>(srecords, S_packed, info, nt, st);
    case 4: return launch_condense_struct<4, 4, 1>(srecords, S_packed, info, nt, st);
    case 5: return launch_condense_struct<5, 4, 1>(srecords, S_packed, info, nt, st);
    case 6: return launch_condense_struct<6, 8, 1>(srecords, S_packed, info, nt, st);
  }
  return -1000;
}
