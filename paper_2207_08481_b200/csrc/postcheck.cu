// Post-solve structural checks on the GPU (reference
// driver.py:183-218 post_checks):
//   max_div      = max_{T, p} |div u(x_p)|,  div u = (tab_div^T u_T) / detJ
//   grad_sq      = sum_T int_T |grad u|^2,    grad u = J grad_hat(u) J^-1 / detJ
//   nt jump      = max over interior facets and edge points of
//                  |t_F^T sigma n_F (side 0) - the same on side 1|, with the
//                  point order reversed on flipped edges (driver.py:206-207)
//   nt scale     = max |t_F^T sigma n_F| on side 0
// For the nt values, t_F^T (J^-T sigma_hat J^T) n_F = (J^-1 t_F)^T sigma_hat
// (J^T n_F), so the reference stress tables are contracted with two
// per-element 2-vectors.  One warp per element / per interior facet.
// Maxima of non-negative doubles use atomicMax on their bit patterns (order
// independent); the gradient sum is a fixed-order per-warp / per-slot sum.
#include "common.cuh"

namespace mcs {

constexpr int PC_WARPS = 4;

__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  atomicMax(reinterpret_cast<unsigned long long*>(addr), __double_as_longlong(v));
}

// geo: [nt][10] = J (row-major 2x2), J^-1 (row-major 2x2), detJ, pad
__global__ void __launch_bounds__(32 * PC_WARPS)
    pc_element_kernel(int64_t nt, int nu, int nq, const double* __restrict__ geo,
                      const int* __restrict__ vcodes, const double* __restrict__ u,
                      const double* __restrict__ tab_div, const double* __restrict__ tab_grad,
                      const double* __restrict__ wq, double* __restrict__ max_div,
                      double* __restrict__ part) {
  extern __shared__ double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* ul = sm + warp * nu;
  const int64_t gw = (int64_t)blockIdx.x * PC_WARPS + warp;
  const int64_t nw = (int64_t)gridDim.x * PC_WARPS;
  double gsum = 0.0, dmax = 0.0;
  for (int64_t e = gw; e < nt; e += nw) {
    for (int j = lane; j < nu; j += 32) {
      const int c = __ldg(vcodes + e * nu + j);
      ul[j] = code_sign(c) * __ldg(u + code_index(c));
    }
    __syncwarp();
    const double* G = geo + e * 10;
    const double J00 = G[0], J01 = G[1], J10 = G[2], J11 = G[3];
    const double I00 = G[4], I01 = G[5], I10 = G[6], I11 = G[7], det = G[8];
    const double idet = 1.0 / det;
    for (int p = lane; p < nq; p += 32) {
      double dv = 0.0, g00 = 0.0, g01 = 0.0, g10 = 0.0, g11 = 0.0;
      for (int a = 0; a < nu; ++a) {
        const double ua = ul[a];
        dv = fma(ua, __ldg(tab_div + a * nq + p), dv);
        const double* tg = tab_grad + ((int64_t)a * nq + p) * 4;
        g00 = fma(ua, __ldg(tg), g00);
        g01 = fma(ua, __ldg(tg + 1), g01);
        g10 = fma(ua, __ldg(tg + 2), g10);
        g11 = fma(ua, __ldg(tg + 3), g11);
      }
      dmax = fmax(dmax, fabs(dv * idet));
      // grad u = J g J^-1 / detJ
      const double h00 = J00 * g00 + J01 * g10, h01 = J00 * g01 + J01 * g11;
      const double h10 = J10 * g00 + J11 * g10, h11 = J10 * g01 + J11 * g11;
      const double m00 = (h00 * I00 + h01 * I10) * idet, m01 = (h00 * I01 + h01 * I11) * idet;
      const double m10 = (h10 * I00 + h11 * I10) * idet, m11 = (h10 * I01 + h11 * I11) * idet;
      gsum = fma((m00 * m00 + m01 * m01) + (m10 * m10 + m11 * m11), __ldg(wq + p) * det, gsum);
    }
    __syncwarp();
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    gsum += __shfl_xor_sync(0xffffffffu, gsum, o);
    dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  }
  if (lane == 0) {
    part[gw] = gsum;
    atomic_max_nonneg(max_div, dmax);
  }
}

// fac: [nif][4] = (t0, le0, t1, le1); frame: [nif][4] = (t_F, n_F);
// flip: [nt][3]; tab_se: [ns][3][nqe][2][2] reference stress at edge points
__global__ void __launch_bounds__(32 * PC_WARPS)
    pc_facet_kernel(int nif, int ns, int nqe, const int* __restrict__ fac,
                    const double* __restrict__ frame, const double* __restrict__ geo,
                    const signed char* __restrict__ flip, const double* __restrict__ sigma,
                    const double* __restrict__ tab_se, double* __restrict__ max_jump,
                    double* __restrict__ max_scale) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * PC_WARPS + warp;
  const int64_t nw = (int64_t)gridDim.x * PC_WARPS;
  double jmax = 0.0, smax = 0.0;
  for (int64_t f = gw; f < nif; f += nw) {
    const double tx = frame[f * 4], ty = frame[f * 4 + 1];
    const double nx = frame[f * 4 + 2], ny = frame[f * 4 + 3];
    double nt_side[2][8];
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      const int t = fac[f * 4 + 2 * side], le = fac[f * 4 + 2 * side + 1];
      const double* G = geo + (int64_t)t * 10;
      // a = J^-1 t_F, b = J^T n_F
      const double a0 = G[4] * tx + G[5] * ty, a1 = G[6] * tx + G[7] * ty;
      const double b0 = G[0] * nx + G[2] * ny, b1 = G[1] * nx + G[3] * ny;
      const bool fl = flip[t * 3 + le] != 0;
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        double v = 0.0;
        if (p < nqe) {
          for (int s = lane; s < ns; s += 32) {
            const double* S = tab_se + (((int64_t)s * 3 + le) * nqe + p) * 4;
            const double q = a0 * (S[0] * b0 + S[1] * b1) + a1 * (S[2] * b0 + S[3] * b1);
            v = fma(__ldg(sigma + (int64_t)t * ns + s), q, v);
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        }
        // reference: the point order is reversed on flipped edges
        const int pp = (fl && p < nqe) ? nqe - 1 - p : p;
#pragma unroll
        for (int r = 0; r < 8; ++r)
          if (r == pp) nt_side[side][r] = v;
      }
    }
#pragma unroll
    for (int p = 0; p < 8; ++p)
      if (p < nqe) {
        jmax = fmax(jmax, fabs(nt_side[0][p] - nt_side[1][p]));
        smax = fmax(smax, fabs(nt_side[0][p]));
      }
  }
  if (lane == 0) {
    atomic_max_nonneg(max_jump, jmax);
    atomic_max_nonneg(max_scale, smax);
  }
}

}  // namespace mcs

using namespace mcs;

MCS_API int mcs_post_checks(int64_t nt, int nu, int nq, const double* geo, const int* vcodes,
                            const double* u, const double* tab_div, const double* tab_grad,
                            const double* wq, int nif, int ns, int nqe, const int* fac,
                            const double* frame, const signed char* flip, const double* sigma,
                            const double* tab_se, double* out, double* part, int nparts,
                            void* stream) {
  auto st = static_cast<cudaStream_t>(stream);
  if (nqe > 8) return -1000;
  int rc = err_code(cudaMemsetAsync(out, 0, 4 * sizeof(double), st));
  if (rc) return rc;
  const int grid = nparts / PC_WARPS;
  if (grid < 1) return -1000;
  rc = err_code(cudaMemsetAsync(part, 0, (size_t)nparts * sizeof(double), st));
  if (rc) return rc;
  if (nt > 0) {
    pc_element_kernel<<<grid, 32 * PC_WARPS, PC_WARPS * nu * sizeof(double), st>>>(
        nt, nu, nq, geo, vcodes, u, tab_div, tab_grad, wq, out, part);
    rc = launch_status();
    if (rc) return rc;
  }
  if (nif > 0) {
    const int fg = (nif + PC_WARPS - 1) / PC_WARPS;
    pc_facet_kernel<<<fg < 4 * 148 ? fg : 4 * 148, 32 * PC_WARPS, 0, st>>>(
        nif, ns, nqe, fac, frame, geo, flip, sigma, tab_se, out + 1, out + 2);
    rc = launch_status();
  }
  return rc;
}
