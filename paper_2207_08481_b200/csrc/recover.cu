// Element-wise stress recovery (reference
// CondensedSystem.recover_stress, condensation.py:64-74):
//     (sigma_T, omega_T) = -R_T u_T,   R_T = M^-1 [Bsig^T; 0],
//     M = [[-msig, bws^T], [bws, 0]].
// With the block structure of DESIGN.md §3.2 (msig = blockdiag(A_m, M_b),
// bws = [Phi (x) s | 0]) and f = Bsig^T u_T:
//     sigma_m = Pi_m f_m = A_m^-1 f_m - q_m d_m / c_m,
//         q_m = A_m^-1 s, c_m = s . q_m, d_m = q_m . f_m,
//     sigma_b = M_b^-1 f_b,
//     omega   = -Phi^-T (d / c),
// so no element stores R (the reference keeps (ns + nw) x nloc doubles per
// element, 572 MB at cfg2); the recovery regenerates Bsig from the geometry
// weights like the fused condensation kernel.  One warp per element.
#include "common.cuh"

namespace mcs {

template <int K>
struct RTab {   // = FTab<K> (condense_fused.cu) followed by Phi^-T [nw][ml]
  using Z = Sizes<K>;
  static constexpr int ml = K * (K + 1) / 2, nl = 3 * ml, nb = 3 * K;
  static constexpr int NR = (Z::nloc + 7) / 8 * 8;
  static constexpr int o_G4 = 0;
  static constexpr int o_adiv = o_G4 + 4 * NR * Z::ns;
  static constexpr int o_Mb = o_adiv + even(Z::nu * Z::nu);
  static constexpr int o_A = o_Mb + even(6 * nb * nb);
  static constexpr int o_PhiT = o_A + even(6 * 9 * ml);
  static constexpr int len = o_PhiT + even(ml * ml);
};

template <int K>
__device__ __forceinline__ int rc_row_woff(int i) {
  using Z = Sizes<K>;
  return i < Z::n_em ? 9 + 3 * (i / (K + 1))
                     : ((i >= Z::nu && i < Z::nloc) ? 18 + 3 * ((i - Z::nu) / K) : 30);
}

constexpr int RC_WARPS = 4;

template <int K>
__global__ void __launch_bounds__(32 * RC_WARPS)
    recover_kernel(const double* __restrict__ Wg, int nwgt, const double* __restrict__ tab,
                   const int* __restrict__ codes, const double* __restrict__ x,
                   double* __restrict__ sig, double* __restrict__ om, int* __restrict__ info,
                   int64_t nt) {
  using Z = Sizes<K>;
  using T = RTab<K>;
  constexpr int ns = Z::ns, nloc = Z::nloc, ml = T::ml, nl = T::nl, nb = T::nb, nw = Z::nw;
  constexpr int PER = 36 + even(nloc) + even(ns) + 2 * nb * nb + 2 * even(nb) + even(ml);
  extern __shared__ __align__(16) double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* w = smem + warp * PER;         // weights, slots 30.. = 0
  double* u = w + 36;                    // local velocity (signed)
  double* f = u + even(nloc);            // Bsig^T u
  double* Ls = f + even(ns);             // bubble Cholesky rows
  double* Li = Ls + nb * nb;             // L_b^-1
  double* Rd = Li + nb * nb;             // 1 / diag(L_b)
  double* dc = Rd + even(nb);            // d_m / c_m
  double* yb = dc + even(ml);            // L_b^-1 f_b (nb)
  if (lane < 6) w[30 + lane] = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * RC_WARPS + warp; e < nt;
       e += (int64_t)gridDim.x * RC_WARPS) {
    if (lane < 30) w[lane] = __ldg(Wg + e * nwgt + lane);
    for (int j = lane; j < nloc; j += 32) {
      const int c = __ldg(codes + e * nloc + j);
      u[j] = code_sign(c) * __ldg(x + code_index(c));
    }
    __syncwarp();
    // f = Bsig^T u, Bsig rows generated from the tables (lane = column)
    for (int c = lane; c < ns; c += 32) {
      double acc = 0.0;
      for (int i = 0; i < nloc; ++i) {
        const int wo = rc_row_woff<K>(i);
        const double2* p = reinterpret_cast<const double2*>(tab + T::o_G4) + 2 * (i * ns + c);
        const double2 v01 = __ldg(p), v23 = __ldg(p + 1);
        double b = fma(w[wo], v01.y, v01.x);
        b = fma(w[wo + 1], v23.x, b);
        b = fma(w[wo + 2], v23.y, b);
        acc = fma(b, u[i], acc);
      }
      f[c] = acc;
    }
    int bad = 0;
    // bubble block: M_b = sum_r w_r MbRef_r, Cholesky (lane = row)
    {
      const int i = lane < nb ? lane : 0;
      double a[nb], l[nb];
#pragma unroll
      for (int c = 0; c < nb; ++c) a[c] = 0.0;
#pragma unroll
      for (int r = 0; r < 6; ++r) {
        const double wr = w[r];
#pragma unroll
        for (int c = 0; c < nb; ++c) a[c] = fma(wr, __ldg(tab + T::o_Mb + (r * nb + i) * nb + c), a[c]);
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
      if (!ok) bad = 1;
      if (lane < nb) {
#pragma unroll
        for (int c = 0; c < nb; ++c) Ls[lane * nb + c] = l[c];
      }
    }
    __syncwarp();   // f, Ls, Rd visible
    double* so = sig + e * ns;
    if (lane < ml) {   // 3x3 block m = lane: sigma_m = Pi_m f_m, d_m / c_m
      double A[9];
#pragma unroll
      for (int q = 0; q < 9; ++q) A[q] = 0.0;
#pragma unroll
      for (int r = 0; r < 6; ++r) {
        const double wr = w[r];
#pragma unroll
        for (int q = 0; q < 9; ++q) A[q] = fma(wr, __ldg(tab + T::o_A + (r * ml + lane) * 9 + q), A[q]);
      }
      const double s0 = w[6], s1 = w[7], s2 = w[8];
      const double f0 = f[3 * lane], f1 = f[3 * lane + 1], f2 = f[3 * lane + 2];
      // Cholesky A = L L^T, solves with L L^T
      const double a00 = A[0], a10 = A[3], a11 = A[4], a20 = A[6], a21 = A[7], a22 = A[8];
      const double i00 = rsqrt_nr(a00);
      const double l10 = a10 * i00, l20 = a20 * i00;
      const double d11 = a11 - l10 * l10;
      const double i11 = rsqrt_nr(d11);
      const double l21 = (a21 - l20 * l10) * i11;
      const double d22 = a22 - l20 * l20 - l21 * l21;
      const double i22 = rsqrt_nr(d22);
      if (!(a00 > 0.0 && d11 > 0.0 && d22 > 0.0)) bad = 1;
      auto solve = [&](double b0, double b1, double b2, double& x0, double& x1, double& x2) {
        const double y0 = b0 * i00, y1 = (b1 - l10 * y0) * i11, y2 = (b2 - l20 * y0 - l21 * y1) * i22;
        x2 = y2 * i22;
        x1 = (y1 - l21 * x2) * i11;
        x0 = (y0 - l10 * x1 - l20 * x2) * i00;
      };
      double a0, a1, a2, q0, q1, q2;
      solve(f0, f1, f2, a0, a1, a2);
      solve(s0, s1, s2, q0, q1, q2);
      const double c = s0 * q0 + s1 * q1 + s2 * q2;
      const double d = s0 * a0 + s1 * a1 + s2 * a2;
      const double r = d / c;
      so[3 * lane] = a0 - q0 * r;
      so[3 * lane + 1] = a1 - q1 * r;
      so[3 * lane + 2] = a2 - q2 * r;
      dc[lane] = r;
    } else if (lane >= 32 - nb) {   // column j of L_b^-1 (lanes 32-nb .. 31)
      const int j0 = lane - (32 - nb);
      double xv[nb];
#pragma unroll
      for (int j = 0; j < nb; ++j) {
        double acc = (j == j0) ? 1.0 : 0.0;
#pragma unroll
        for (int q = 0; q < j; ++q) acc = fma(-Ls[j * nb + q], xv[q], acc);
        xv[j] = acc * Rd[j];
        Li[j * nb + j0] = xv[j];
      }
    }
    if (ml + nb > 32) {   // not enough lanes for both: second pass for L_b^-1
      __syncwarp();
      if (lane < nb) {
        double xv[nb];
#pragma unroll
        for (int j = 0; j < nb; ++j) {
          double acc = (j == lane) ? 1.0 : 0.0;
#pragma unroll
          for (int q = 0; q < j; ++q) acc = fma(-Ls[j * nb + q], xv[q], acc);
          xv[j] = acc * Rd[j];
          Li[j * nb + lane] = xv[j];
        }
      }
    }
    __syncwarp();
    // sigma_b = L_b^-T (L_b^-1 f_b)
    if (lane < nb) {
      double acc = 0.0;
      for (int q = 0; q <= lane; ++q) acc = fma(Li[lane * nb + q], f[nl + q], acc);
      yb[lane] = acc;
    }
    __syncwarp();
    if (lane < nb) {
      double acc = 0.0;
      for (int q = lane; q < nb; ++q) acc = fma(Li[q * nb + lane], yb[q], acc);
      so[nl + lane] = acc;
    }
    // omega = -Phi^-T (d / c)
    if (lane < nw) {
      double acc = 0.0;
      for (int m = 0; m < ml; ++m) acc = fma(__ldg(tab + T::o_PhiT + lane * ml + m), dc[m], acc);
      om[e * nw + lane] = -acc;
    }
    if (lane == 0 && info) info[e] = bad;
    __syncwarp();
  }
}

template <int K>
static int launch_recover(int64_t nt, const double* W, int nwgt, const double* tab,
                          const int* codes, const double* x, double* sig, double* om, int* info,
                          cudaStream_t st) {
  using Z = Sizes<K>;
  using T = RTab<K>;
  constexpr int PER = 36 + even(Z::nloc) + even(Z::ns) + 2 * T::nb * T::nb + 2 * even(T::nb) +
                      even(T::ml);
  const size_t smem = (size_t)RC_WARPS * PER * sizeof(double);
  auto kern = recover_kernel<K>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t want = (nt + RC_WARPS - 1) / RC_WARPS;
  const int grid = (int)(want < 148 * 16 ? want : 148 * 16);
  kern<<<grid, 32 * RC_WARPS, smem, st>>>(W, nwgt, tab, codes, x, sig, om, info, nt);
  return launch_status();
}

}  // namespace mcs

using namespace mcs;

MCS_API int mcs_recover_table_len(int k) {
  switch (k) {
    case 2: return RTab<2>::len;
    case 3: return RTab<3>::len;
    case 4: return RTab<4>::len;
    case 5: return RTab<5>::len;
    case 6: return RTab<6>::len;
  }
  return -1;
}

MCS_API int mcs_recover_stress(int k, int64_t nt, const double* W, int nwgt, const double* tables,
                               const int* vv_codes, const double* x_full, double* sigma,
                               double* omega, int* info, void* stream) {
  if (nt <= 0) return 0;
  if (nwgt < 30) return -1000;
  auto st = static_cast<cudaStream_t>(stream);
  switch (k) {
    case 2: return launch_recover<2>(nt, W, nwgt, tables, vv_codes, x_full, sigma, omega, info, st);
    case 3: return launch_recover<3>(nt, W, nwgt, tables, vv_codes, x_full, sigma, omega, info, st);
    case 4: return launch_recover<4>(nt, W, nwgt, tables, vv_codes, x_full, sigma, omega, info, st);
    case 5: return launch_recover<5>(nt, W, nwgt, tables, vv_codes, x_full, sigma, omega, info, st);
    case 6: return launch_recover<6>(nt, W, nwgt, tables, vv_codes, x_full, sigma, omega, info, st);
  }
  return -1000;
}
