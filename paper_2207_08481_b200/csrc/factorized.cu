// CondensedSystem methods of the drop-in boundary that act on
// vectors over ALL (V, Vhat) dofs, constrained ones included:
//
//   mcs_apply_S_factorized   y = S x through the exact block factorisation
//                            (reference condensation.py:104-122):
//                              z_o = x_o + X x_c,  d_o = S_oo z_o,
//                              y_c = Sd_T x_c + X^T d_o,  y_o = d_o
//                            summed over elements (Sd = sum_T Sd_T, so the
//                            global Sd @ x_c of the reference is the sum of
//                            the per-element Sd_T x_c).
//   mcs_harmonic_extend      out = x, out_o = -X x_c per element
//                            (reference condensation.py:93-102).
//   mcs_block_inverse        packed SPD inverses of caller-supplied dense
//                            facet blocks (FacetBlockSmoother built from a
//                            CSR matrix and a block list, preconditioners.py:
//                            177-200), in the SoA layout of jacobi_apply.
//
// One warp per element, lanes over local rows; every coupling dof receives
// at most two contributions into a zeroed vector (0 + a + b == 0 + b + a),
// bubble dofs one, so the atomics are deterministic.
#include "common.cuh"

namespace mcs {

constexpr int FZ_WARPS = 4;

template <int K>
__global__ void __launch_bounds__(32 * FZ_WARPS)
    apply_factorized_kernel(const double* __restrict__ ST, const double* __restrict__ ext,
                            const double* __restrict__ Sd, const int* __restrict__ codes,
                            const double* __restrict__ x, double* __restrict__ y, int64_t nt) {
  using Z = Sizes<K>;
  using L = ExtLayout<K>;
  constexpr int nloc = Z::nloc, ni = Z::n_int, nc = Z::ncpl, nem = Z::n_em;
  __shared__ double sh[FZ_WARPS][even(nloc) + 2 * even(ni)];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* loc = sh[warp];
  double* zo = loc + even(nloc);
  double* d_o = zo + even(ni);
  for (int64_t e = (int64_t)blockIdx.x * FZ_WARPS + warp; e < nt;
       e += (int64_t)gridDim.x * FZ_WARPS) {
    const int* ce = codes + e * nloc;
    for (int j = lane; j < nloc; j += 32) {
      const int c = ce[j];
      loc[j] = code_sign(c) * x[code_index(c)];
    }
    __syncwarp();
    const double* X = ext + e * L::len;
    const double* S = ST + e * L::st_len;
    for (int i = lane; i < ni; i += 32) {           // z_o = x_o + X x_c
      double s = loc[nem + i];
      for (int c = 0; c < nc; ++c) s = fma(X[i * nc + c], loc[cpl_local<K>(c)], s);
      zo[i] = s;
    }
    __syncwarp();
    for (int i = lane; i < ni; i += 32) {           // d_o = S_oo z_o
      const int li = nem + i;
      double s = 0.0;
      for (int j = 0; j < ni; ++j) {
        const int lj = nem + j;
        s = fma(li >= lj ? S[pk(li, lj)] : S[pk(lj, li)], zo[j], s);
      }
      d_o[i] = s;
    }
    __syncwarp();
    const double* D = Sd + e * L::sd_len;
    for (int c = lane; c < nc; c += 32) {           // y_c = Sd_T x_c + X^T d_o
      double s = 0.0;
      for (int b = 0; b < nc; ++b)
        s = fma(c >= b ? D[pk(c, b)] : D[pk(b, c)], loc[cpl_local<K>(b)], s);
      for (int i = 0; i < ni; ++i) s = fma(X[i * nc + c], d_o[i], s);
      const int code = ce[cpl_local<K>(c)];
      atomicAdd(y + code_index(code), code_sign(code) * s);
    }
    for (int i = lane; i < ni; i += 32) {
      const int code = ce[nem + i];
      atomicAdd(y + code_index(code), code_sign(code) * d_o[i]);
    }
    __syncwarp();
  }
}

template <int K>
__global__ void __launch_bounds__(32 * FZ_WARPS)
    harmonic_extend_kernel(const double* __restrict__ ext, const int* __restrict__ codes,
                           const double* __restrict__ x, double* __restrict__ out, int64_t nt) {
  using Z = Sizes<K>;
  using L = ExtLayout<K>;
  constexpr int nloc = Z::nloc, ni = Z::n_int, nc = Z::ncpl, nem = Z::n_em;
  __shared__ double sh[FZ_WARPS][even(nc)];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* xc = sh[warp];
  for (int64_t e = (int64_t)blockIdx.x * FZ_WARPS + warp; e < nt;
       e += (int64_t)gridDim.x * FZ_WARPS) {
    const int* ce = codes + e * nloc;
    for (int c = lane; c < nc; c += 32) {
      const int code = ce[cpl_local<K>(c)];
      xc[c] = code_sign(code) * x[code_index(code)];
    }
    __syncwarp();
    const double* X = ext + e * L::len;
    for (int i = lane; i < ni; i += 32) {
      double s = 0.0;
      for (int c = 0; c < nc; ++c) s = fma(X[i * nc + c], xc[c], s);
      const int code = ce[nem + i];
      out[code_index(code)] = -s * code_sign(code);
    }
    __syncwarp();
  }
}

// blocks: [nblk][B][B] row-major (entries beyond bsize[b] ignored),
// idx: [nblk][B] free coupling index or -1.  Output as jacobi_setup_kernel:
// binv [npk(B)][nblk], bidx [B][nblk].  Gauss-Jordan without pivoting (SPD);
// info[b] = 1 + first non-positive pivot.
template <int B>
__global__ void block_inverse_kernel(const double* __restrict__ blocks,
                                     const int* __restrict__ idx, const int* __restrict__ bsize,
                                     int nblk, double* __restrict__ binv, int* __restrict__ bidx,
                                     int* __restrict__ info) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nblk) return;
  const int n = bsize[b];
  double A[B][2 * B];
  for (int a = 0; a < n; ++a)
    for (int c = 0; c < 2 * n; ++c)
      A[a][c] = c < n ? blocks[((int64_t)b * B + a) * B + c] : ((c - n == a) ? 1.0 : 0.0);
  int bad = 0;
  for (int j = 0; j < n; ++j) {
    const double piv = A[j][j];
    if (!(piv > 0.0) && !bad) bad = j + 1;
    const double inv = 1.0 / piv;
    for (int c = 0; c < 2 * n; ++c) A[j][c] *= inv;
    for (int i = 0; i < n; ++i) {
      if (i == j) continue;
      const double m = A[i][j];
      for (int c = 0; c < 2 * n; ++c) A[i][c] = fma(-m, A[j][c], A[i][c]);
    }
  }
  for (int i = 0; i < B; ++i) {
    bidx[(int64_t)i * nblk + b] = i < n ? idx[(int64_t)b * B + i] : -1;
    for (int j = 0; j <= i; ++j)
      binv[(int64_t)pk(i, j) * nblk + b] = (i < n) ? 0.5 * (A[i][n + j] + A[j][n + i]) : 0.0;
  }
  info[b] = bad;
}

template <int K>
static int launch_factorized(const double* ST, const double* ext, const double* Sd,
                             const int* codes, const double* x, double* y, int64_t nt,
                             cudaStream_t st) {
  const int64_t want = (nt + FZ_WARPS - 1) / FZ_WARPS;
  const int grid = (int)(want < 16 * 148 ? want : 16 * 148);
  apply_factorized_kernel<K><<<grid, 32 * FZ_WARPS, 0, st>>>(ST, ext, Sd, codes, x, y, nt);
  return launch_status();
}

template <int K>
static int launch_extend(const double* ext, const int* codes, const double* x, double* out,
                         int64_t nt, cudaStream_t st) {
  const int64_t want = (nt + FZ_WARPS - 1) / FZ_WARPS;
  const int grid = (int)(want < 16 * 148 ? want : 16 * 148);
  harmonic_extend_kernel<K><<<grid, 32 * FZ_WARPS, 0, st>>>(ext, codes, x, out, nt);
  return launch_status();
}

}  // namespace mcs

using namespace mcs;

#define MCS_K_SWITCH(CALL)   \
  switch (k) {               \
    case 2: return CALL(2);  \
    case 3: return CALL(3);  \
    case 4: return CALL(4);  \
    case 5: return CALL(5);  \
    case 6: return CALL(6);  \
    default: return -1000;   \
  }

MCS_API int mcs_apply_S_factorized(int k, int64_t nt, const double* ST, const double* ext,
                                   const double* Sd, const int* codes, const double* x, double* y,
                                   void* stream) {
  if (nt <= 0) return 0;
  auto st = static_cast<cudaStream_t>(stream);
#define C(K) launch_factorized<K>(ST, ext, Sd, codes, x, y, nt, st)
  MCS_K_SWITCH(C)
#undef C
}

MCS_API int mcs_harmonic_extend(int k, int64_t nt, const double* ext, const int* codes,
                                const double* x, double* out, void* stream) {
  if (nt <= 0) return 0;
  auto st = static_cast<cudaStream_t>(stream);
#define C(K) launch_extend<K>(ext, codes, x, out, nt, st)
  MCS_K_SWITCH(C)
#undef C
}

MCS_API int mcs_block_inverse(int k, int nblk, const double* blocks, const int* idx,
                              const int* bsize, double* binv, int* bidx, int* info, void* stream) {
  if (nblk <= 0) return 0;
  auto st = static_cast<cudaStream_t>(stream);
  const int grid = (nblk + 127) / 128;
  switch (k) {
    case 2: block_inverse_kernel<5><<<grid, 128, 0, st>>>(blocks, idx, bsize, nblk, binv, bidx, info); break;
    case 3: block_inverse_kernel<7><<<grid, 128, 0, st>>>(blocks, idx, bsize, nblk, binv, bidx, info); break;
    case 4: block_inverse_kernel<9><<<grid, 128, 0, st>>>(blocks, idx, bsize, nblk, binv, bidx, info); break;
    case 5: block_inverse_kernel<11><<<grid, 128, 0, st>>>(blocks, idx, bsize, nblk, binv, bidx, info); break;
    case 6: block_inverse_kernel<13><<<grid, 128, 0, st>>>(blocks, idx, bsize, nblk, binv, bidx, info); break;
    default: return -1000;
  }
  return launch_status();
}
