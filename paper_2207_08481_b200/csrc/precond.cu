// Auxiliary-space preconditioner pieces.
//
//  A9  facet-block Jacobi on S_d (preconditioners.py:177-206, variant
//      "jacobi", blocks of facet_blocks_schur :266-280).  Setup assembles
//      every facet block from the Sd_T of its <= 2 incident elements and
//      inverts it (Gauss-Jordan, SPD, no pivoting); apply is one thread per
//      facet over structure-of-arrays packed inverses (coalesced), scaled by
//      1/jacobi_scale.  Blocks are disjoint, so x[blk] = Binv r[blk] exactly.
//  A10 CSR SpMV y = alpha*A x + beta*y for E_c and its explicitly stored
//      transpose (preconditioners.py:316-317); a sub-warp per row with a
//      fixed-order shuffle reduction (deterministic).
#include <cstdlib>

#include "common.cuh"

namespace mcs {

// fpos[f][p] : local coupling index of facet-position p in element t of slot s
// blocks: per facet block b: facet id, up to 2 (element, local edge) slots
// dof codes from the element's cpl codes (2*cplfree + neg, -1 constrained)
template <int K>
__global__ void jacobi_setup_kernel(const double* __restrict__ Sd, int sd_stride,
                                    const int* __restrict__ ccodes, const int* __restrict__ slots,
                                    int nblk, double* __restrict__ binv, int* __restrict__ bidx,
                                    int* __restrict__ bsize, int* __restrict__ info) {
  using Z = Sizes<K>;
  constexpr int B = 2 * K + 1, NC = Z::ncpl;
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nblk) return;
  double A[B][2 * B];
  int pos[B];
  int n = 0;
  const int t0 = slots[4 * b + 0], le0 = slots[4 * b + 1];
  // facet position p -> local cpl index within element with local edge le
  auto cl = [](int le, int p) { return p <= K ? le * (K + 1) + p : Z::n_em + le * K + (p - K - 1); };
  for (int p = 0; p < B; ++p) {
    const int c = ccodes[(int64_t)t0 * NC + cl(le0, p)];
    if (c >= 0) pos[n++] = p;
  }
  for (int a = 0; a < n; ++a)
    for (int c = 0; c < 2 * n; ++c) A[a][c] = (c - n == a) ? 1.0 : 0.0;
  for (int s = 0; s < 2; ++s) {
    const int t = slots[4 * b + 2 * s], le = slots[4 * b + 2 * s + 1];
    if (t < 0) continue;
    const double* P = Sd + (int64_t)t * sd_stride;
    for (int a = 0; a < n; ++a) {
      const int ca = cl(le, pos[a]);
      const double sa = code_sign(ccodes[(int64_t)t * NC + ca]);
      for (int c = 0; c < n; ++c) {
        const int cc = cl(le, pos[c]);
        const double sc = code_sign(ccodes[(int64_t)t * NC + cc]);
        A[a][c] += sa * sc * (ca >= cc ? P[pk(ca, cc)] : P[pk(cc, ca)]);
      }
    }
  }
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
    int code = -1;
    if (i < n) code = code_index(ccodes[(int64_t)t0 * NC + cl(le0, pos[i])]);
    bidx[(int64_t)i * nblk + b] = code;
    for (int j = 0; j <= i; ++j)
      binv[(int64_t)pk(i, j) * nblk + b] =
          (i < n) ? 0.5 * (A[i][n + j] + A[j][n + i]) : 0.0;
  }
  bsize[b] = n;
  if (info) info[b] = bad;
}

// Thread per facet block, all loads issued before the first FMA.
template <int B>
__global__ void __launch_bounds__(64)
    jacobi_apply_kernel(const double* __restrict__ binv, const int* __restrict__ bidx, int nblk,
                        const double* r, double* __restrict__ x, double scale_inv) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  constexpr int NP = B * (B + 1) / 2;
  int id[B];
  double rl[B], a[NP];
  const int bb = b < nblk ? b : nblk - 1;
#pragma unroll
  for (int j = 0; j < B; ++j) id[j] = __ldg(bidx + (int64_t)j * nblk + bb);
#pragma unroll
  for (int p = 0; p < NP; ++p) a[p] = __ldg(binv + (int64_t)p * nblk + bb);
  pdl_wait();   // the block inverses and indices are in flight; r may now be read
  pdl_trigger();
  if (b >= nblk) return;
#pragma unroll
  for (int j = 0; j < B; ++j) rl[j] = id[j] >= 0 ? r[id[j]] : 0.0;
#pragma unroll
  for (int i = 0; i < B; ++i) {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < B; ++j) s = fma(a[i >= j ? pk(i, j) : pk(j, i)], rl[j], s);
    if (id[i] >= 0) x[id[i]] = s * scale_inv;
  }
}

// Thread per (facet, block row): a CTA of B warps covers 32 facets, warp w
// computes row w of every facet's x[blk] = Binv r[blk].  Nine times the
// threads of the facet-per-thread kernel (each with 9 + 9 + 9 independent
// loads); the shared packed entries, indices and gathered r come from L1/L2.
// Kept as an A/B variant (MCS_JAC_VARIANT=2): slower than one thread per
// facet at cfg2 (14.3 vs 10.2 us event time).
template <int B>
__global__ void __launch_bounds__(32 * B)
    jacobi_rows_kernel(const double* __restrict__ binv, const int* __restrict__ bidx, int nblk,
                       const double* r, double* __restrict__ x, double scale_inv) {
  const int row = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int f = blockIdx.x * 32 + lane;
  const int ff = f < nblk ? f : nblk - 1;
  double a[B];
  int id[B];
#pragma unroll
  for (int j = 0; j < B; ++j) {
    a[j] = __ldg(binv + (int64_t)(row >= j ? pk(row, j) : pk(j, row)) * nblk + ff);
    id[j] = __ldg(bidx + (int64_t)j * nblk + ff);
  }
  pdl_wait();   // the block inverses and indices are in flight; r may now be read
  pdl_trigger();
  if (f >= nblk) return;
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < B; ++j) s = fma(a[j], id[j] >= 0 ? r[id[j]] : 0.0, s);
  if (id[row] >= 0) x[id[row]] = s * scale_inv;
}

template <int LANES>
__global__ void csr_spmv_kernel(int nrows, const int* __restrict__ ptr, const int* __restrict__ col,
                                const double* __restrict__ val, const double* x,
                                double* __restrict__ y, double alpha, double beta) {
  pdl_wait();
  pdl_trigger();
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int row = tid / LANES, sub = tid % LANES;
  double s = 0.0;
  if (row < nrows)
    for (int p = ptr[row] + sub; p < ptr[row + 1]; p += LANES) s = fma(val[p], x[col[p]], s);
#pragma unroll
  for (int o = LANES / 2; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o, LANES);
  if (row < nrows && sub == 0) y[row] = (beta == 0.0 ? 0.0 : beta * y[row]) + alpha * s;
}

}  // namespace mcs

using namespace mcs;

MCS_API int mcs_jacobi_setup(int k, int nblk, const double* Sd_packed, int sd_stride, const int* ccodes,
                             const int* slots, double* binv, int* bidx, int* bsize, int* info,
                             void* stream) {
  if (nblk <= 0) return 0;
  auto st = static_cast<cudaStream_t>(stream);
  const int grid = (nblk + 127) / 128;
  switch (k) {
    case 2: jacobi_setup_kernel<2><<<grid, 128, 0, st>>>(Sd_packed, sd_stride, ccodes, slots, nblk, binv, bidx, bsize, info); break;
    case 3: jacobi_setup_kernel<3><<<grid, 128, 0, st>>>(Sd_packed, sd_stride, ccodes, slots, nblk, binv, bidx, bsize, info); break;
    case 4: jacobi_setup_kernel<4><<<grid, 128, 0, st>>>(Sd_packed, sd_stride, ccodes, slots, nblk, binv, bidx, bsize, info); break;
    case 5: jacobi_setup_kernel<5><<<grid, 128, 0, st>>>(Sd_packed, sd_stride, ccodes, slots, nblk, binv, bidx, bsize, info); break;
    case 6: jacobi_setup_kernel<6><<<grid, 128, 0, st>>>(Sd_packed, sd_stride, ccodes, slots, nblk, binv, bidx, bsize, info); break;
    default: return -1000;
  }
  return launch_status();
}

// binv: [npk(2k+1)][nblk] packed inverses (SoA), bidx: [2k+1][nblk] (-1 padding)
MCS_API int mcs_jacobi_apply(int k, int nblk, const double* binv, const int* bidx,
                             const double* r, double* x, double scale_inv, void* stream) {
  if (nblk <= 0) return 0;
  auto st = static_cast<cudaStream_t>(stream);
  // default: thread per facet.  MCS_JAC_VARIANT=2: thread per (facet, row),
  // measured slower at cfg2 (14.3 vs 10.2 us, profiles/r02/jacobi_variants.txt)
  static const int variant = getenv("MCS_JAC_VARIANT") ? atoi(getenv("MCS_JAC_VARIANT")) : 1;
  if (variant == 2) {
    const int gr = (nblk + 31) / 32;
    switch (k) {
      case 2: return launch_pdl_g(PDL_PREC, jacobi_rows_kernel<5>, gr, 32 * 5, 0, st, binv, bidx, nblk, r, x, scale_inv);
      case 3: return launch_pdl_g(PDL_PREC, jacobi_rows_kernel<7>, gr, 32 * 7, 0, st, binv, bidx, nblk, r, x, scale_inv);
      case 4: return launch_pdl_g(PDL_PREC, jacobi_rows_kernel<9>, gr, 32 * 9, 0, st, binv, bidx, nblk, r, x, scale_inv);
      case 5: return launch_pdl_g(PDL_PREC, jacobi_rows_kernel<11>, gr, 32 * 11, 0, st, binv, bidx, nblk, r, x, scale_inv);
      case 6: return launch_pdl_g(PDL_PREC, jacobi_rows_kernel<13>, gr, 32 * 13, 0, st, binv, bidx, nblk, r, x, scale_inv);
      default: return -1000;
    }
  }
  const int grid = (nblk + 63) / 64;
  switch (k) {
    case 2: return launch_pdl_g(PDL_PREC, jacobi_apply_kernel<5>, grid, 64, 0, st, binv, bidx, nblk, r, x, scale_inv);
    case 3: return launch_pdl_g(PDL_PREC, jacobi_apply_kernel<7>, grid, 64, 0, st, binv, bidx, nblk, r, x, scale_inv);
    case 4: return launch_pdl_g(PDL_PREC, jacobi_apply_kernel<9>, grid, 64, 0, st, binv, bidx, nblk, r, x, scale_inv);
    case 5: return launch_pdl_g(PDL_PREC, jacobi_apply_kernel<11>, grid, 64, 0, st, binv, bidx, nblk, r, x, scale_inv);
    case 6: return launch_pdl_g(PDL_PREC, jacobi_apply_kernel<13>, grid, 64, 0, st, binv, bidx, nblk, r, x, scale_inv);
    default: return -1000;
  }
  return launch_status();
}

MCS_API int mcs_csr_spmv(int nrows, const int* ptr, const int* col, const double* val, const double* x,
                         double* y, double alpha, double beta, int lanes, void* stream) {
  if (nrows <= 0) return 0;
  auto st = static_cast<cudaStream_t>(stream);
  const int64_t threads = (int64_t)nrows * lanes;
  const int grid = (int)((threads + 255) / 256);
  switch (lanes) {
    case 1: return launch_pdl_g(PDL_PREC, csr_spmv_kernel<1>, grid, 256, 0, st, nrows, ptr, col, val, x, y, alpha, beta);
    case 4: return launch_pdl_g(PDL_PREC, csr_spmv_kernel<4>, grid, 256, 0, st, nrows, ptr, col, val, x, y, alpha, beta);
    case 8: return launch_pdl_g(PDL_PREC, csr_spmv_kernel<8>, grid, 256, 0, st, nrows, ptr, col, val, x, y, alpha, beta);
    case 32: return launch_pdl_g(PDL_PREC, csr_spmv_kernel<32>, grid, 256, 0, st, nrows, ptr, col, val, x, y, alpha, beta);
    default: return -1000;
  }
  return launch_status();
}

// y = A x for a dense row-major n x n matrix (small exact coarse solves); warp per row
__global__ void dense_gemv_kernel(int n, const double* __restrict__ A, const double* x,
                                  double* __restrict__ y) {
  pdl_wait();
  pdl_trigger();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= n) return;
  const double* row = A + (int64_t)warp * n;
  double s = 0.0;
  for (int j = lane; j < n; j += 32) s = fma(row[j], x[j], s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if (lane == 0) y[warp] = s;
}

MCS_API int mcs_dense_gemv(int n, const double* A, const double* x, double* y, void* stream) {
  if (n <= 0) return 0;
  auto st = static_cast<cudaStream_t>(stream);
  const int64_t threads = (int64_t)n * 32;
  return launch_pdl_g(PDL_PREC, dense_gemv_kernel, (int)((threads + 255) / 256), 256, 0, st, n, A, x, y);
}
