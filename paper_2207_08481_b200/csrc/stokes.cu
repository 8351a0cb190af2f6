// Stokes (saddle-point) mode (reference driver.py:148-160,
// krylov.py:25-100 gmres, preconditioners.py:384-420 PressureMassPrecond /
// SaddlePreconditioner).
//
//   B apply    y_p[t nq + q] = sum_u Bpu[q][u] s_tu x[g_tu]        (thread per row)
//   B^T apply  y[g_tu] = sum_t s_tu sum_q Bpu[q][u] p[t nq + q]     (atomics onto a
//              zeroed vector: <= 2 contributions per dof, 0 + a + b == 0 + b + a,
//              bitwise deterministic)
//   GMRES      h = V w for the Krylov basis V (m x n, row-major) in two
//              deterministic passes (fixed chunking, partials summed in order),
//              w = beta w + alpha V^T h (thread per entry, fixed order over rows).
// Bpu (nq x nu) is J-invariant (refblocks.py), so it lives in shared memory.
#include "common.cuh"

namespace mcs {

constexpr int SK_THREADS = 256;

__global__ void __launch_bounds__(SK_THREADS)
    apply_B_kernel(int nq, int nu, int nloc, int64_t nt, const double* __restrict__ Bpu,
                   const int* __restrict__ codes, const double* __restrict__ x,
                   double* __restrict__ y) {
  extern __shared__ double sB[];
  for (int i = threadIdx.x; i < nq * nu; i += SK_THREADS) sB[i] = Bpu[i];
  __syncthreads();
  const int64_t n = nt * nq;
  for (int64_t r = (int64_t)blockIdx.x * SK_THREADS + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * SK_THREADS) {
    const int64_t t = r / nq;
    const int q = (int)(r - t * nq);
    const int* cd = codes + t * nloc;
    double acc = 0.0;
    for (int u = 0; u < nu; ++u) {
      const int c = __ldg(cd + u);
      if (c >= 0) acc = fma(sB[q * nu + u], code_sign(c) * __ldg(x + code_index(c)), acc);
    }
    y[r] = acc;
  }
}

__global__ void __launch_bounds__(SK_THREADS)
    apply_BT_kernel(int nq, int nu, int nloc, int64_t nt, const double* __restrict__ Bpu,
                    const int* __restrict__ codes, const double* __restrict__ p,
                    double* __restrict__ y) {
  extern __shared__ double sB[];
  for (int i = threadIdx.x; i < nq * nu; i += SK_THREADS) sB[i] = Bpu[i];
  __syncthreads();
  const int64_t n = nt * nu;
  for (int64_t r = (int64_t)blockIdx.x * SK_THREADS + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * SK_THREADS) {
    const int64_t t = r / nu;
    const int u = (int)(r - t * nu);
    const int c = __ldg(codes + t * nloc + u);
    if (c < 0) continue;
    const double* pt = p + t * nq;
    double acc = 0.0;
    for (int q = 0; q < nq; ++q) acc = fma(sB[q * nu + u], __ldg(pt + q), acc);
    atomicAdd(y + code_index(c), code_sign(c) * acc);
  }
}

constexpr int MD_CHUNKS = 64;

// partial[i][c] = sum over chunk c of V[i] . w
__global__ void __launch_bounds__(SK_THREADS)
    mdot_partial_kernel(int64_t n, int64_t ld, const double* __restrict__ V,
                        const double* __restrict__ w, double* __restrict__ partial,
                        const double* __restrict__ gate) {
  if (gate && *gate != 0.0) return;
  const int i = blockIdx.y, c = blockIdx.x;
  const int64_t len = (n + MD_CHUNKS - 1) / MD_CHUNKS;
  const int64_t lo = c * len, hi = lo + len < n ? lo + len : n;
  const double* v = V + i * ld;
  double s = 0.0;
  for (int64_t k = lo + threadIdx.x; k < hi; k += SK_THREADS) s = fma(v[k], w[k], s);
  __shared__ double red[SK_THREADS / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < SK_THREADS / 32; ++q) t += red[q];
    partial[i * MD_CHUNKS + c] = t;
  }
}

__global__ void mdot_final_kernel(int m, const double* __restrict__ partial,
                                  double* __restrict__ h, const double* __restrict__ gate) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  if (gate && *gate != 0.0) {
    h[i] = 0.0;
    return;
  }
  double s = 0.0;
  for (int c = 0; c < MD_CHUNKS; ++c) s += partial[i * MD_CHUNKS + c];
  h[i] = s;
}

// w[k] = beta w[k] + alpha sum_{i < m} h[i] V[i][k]   (rows in order)
__global__ void __launch_bounds__(SK_THREADS)
    gemv_acc_kernel(int m, int64_t n, int64_t ld, const double* __restrict__ V,
                    const double* __restrict__ h, double alpha, double beta,
                    double* __restrict__ w, const double* __restrict__ gate) {
  if (gate && *gate != 0.0) return;
  for (int64_t k = (int64_t)blockIdx.x * SK_THREADS + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * SK_THREADS) {
    double s = 0.0;
    for (int i = 0; i < m; ++i) s = fma(__ldg(h + i), V[i * ld + k], s);
    w[k] = beta == 0.0 ? alpha * s : fma(alpha, s, beta * w[k]);
  }
}

// DGKS test of classical Gram-Schmidt on the device (krylov.py gmres): the
// second pass is skipped (sc[g] = 1) when ||w_after|| > ||w_before|| / sqrt(2),
// the host's comparison with the same IEEE operations.
__global__ void gs_gate_kernel(double* sc, int before, int after, int g) {
  sc[g] = (sqrt(sc[after]) > 0.7071067811865476 * sqrt(sc[before])) ? 1.0 : 0.0;
}

// ---- fused classical Gram-Schmidt pass (krylov.py gmres): given the first
// pass's h1 = V^T w, one read of the basis V produces
//   w' = w - V h1               (the first pass's update, in place),
//   h2 partials = V^T w' and ||w'||^2 partials
// per CTA column range; gs_final sums them in fixed order, evaluates the DGKS
// gate and leaves h2 (zero when the gate skips the second pass).  Each CTA
// stages a tile of SUB basis columns x m rows in shared memory, so every V
// entry leaves HBM once for both products (three basis reads per step
// instead of four).  Deterministic: fixed column ranges, fixed row order,
// fixed reduction trees.
constexpr int GS_THREADS = 256, GS_SMEM = 64 * 1024;

__global__ void __launch_bounds__(GS_THREADS)
    gs_fused_kernel(int m, int64_t n, int64_t ld, int sub, const double* __restrict__ V,
                    double* __restrict__ w, const double* __restrict__ h1,
                    double* __restrict__ ph2, double* __restrict__ pnrm) {
  extern __shared__ double tile[];            // [m][sub], then R x sub partials, sub w'
  const int tid = threadIdx.x;
  const int R = GS_THREADS / sub;              // row groups of pass a
  double* part = tile + m * sub;
  double* wp = part + R * sub;
  const int64_t span = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = (int64_t)blockIdx.x * span, hi = lo + span < n ? lo + span : n;
  double h2acc[4] = {0.0, 0.0, 0.0, 0.0};      // rows tid + 256 q (m <= 1024)
  double nrm = 0.0;
  const int c = tid % sub, r = tid / sub;
  for (int64_t c0 = lo; c0 < hi; c0 += sub) {
    const int cw = (int)(hi - c0 < sub ? hi - c0 : sub);
    for (int q = tid; q < m * sub; q += GS_THREADS) {
      const int i = q / sub, cc = q % sub;
      tile[q] = cc < cw ? V[i * ld + c0 + cc] : 0.0;
    }
    __syncthreads();
    // pass a: column c, rows r, r + R, ... (in order), then the R partials in order
    double s = 0.0;
    for (int i = r; i < m; i += R) s = fma(__ldg(h1 + i), tile[i * sub + c], s);
    part[r * sub + c] = s;
    __syncthreads();
    if (tid < sub) {
      double t = 0.0;
      for (int q = 0; q < R; ++q) t += part[q * sub + tid];
      double v = 0.0;
      if (tid < cw) {
        v = w[c0 + tid] - t;
        w[c0 + tid] = v;
      }
      wp[tid] = v;
      nrm = fma(v, v, nrm);
    }
    __syncthreads();
    // pass b: row i, the sub columns in order
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = tid + GS_THREADS * q;
      if (i < m) {
        double a = h2acc[q];
        for (int cc = 0; cc < sub; ++cc) a = fma(tile[i * sub + cc], wp[cc], a);
        h2acc[q] = a;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int i = tid + GS_THREADS * q;
    if (i < m) ph2[(int64_t)i * gridDim.x + blockIdx.x] = h2acc[q];
  }
  // ||w'||^2 of this CTA: the sub column threads in order
  __syncthreads();
  if (tid < sub) part[tid] = nrm;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int q = 0; q < sub; ++q) t += part[q];
    pnrm[blockIdx.x] = t;
  }
}

// h2[i] = sum_cta ph2[i][cta] (in order); sc[after] = sum_cta pnrm; the DGKS
// gate sc[g] as gs_gate_kernel; h2 = 0 when the gate skips the second pass.
__global__ void gs_final_kernel(int m, int nblk, const double* __restrict__ ph2,
                                const double* __restrict__ pnrm, double* __restrict__ h2,
                                double* sc, int before, int after, int g) {
  __shared__ double gate;
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int b = 0; b < nblk; ++b) t += pnrm[b];
    sc[after] = t;
    gate = (sqrt(t) > 0.7071067811865476 * sqrt(sc[before])) ? 1.0 : 0.0;
    sc[g] = gate;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nblk; ++b) s += ph2[(int64_t)i * nblk + b];
    h2[i] = gate != 0.0 ? 0.0 : s;
  }
}

static int sk_grid(int64_t n) {
  const int64_t g = (n + SK_THREADS - 1) / SK_THREADS;
  return (int)(g < 8 * 148 ? (g < 1 ? 1 : g) : 8 * 148);
}

}  // namespace mcs

using namespace mcs;

MCS_API int mcs_apply_B(int nq, int nu, int nloc, int64_t nt, const double* Bpu, const int* codes,
                        const double* x, double* y, void* stream) {
  if (nt <= 0) return 0;
  auto st = static_cast<cudaStream_t>(stream);
  apply_B_kernel<<<sk_grid(nt * nq), SK_THREADS, nq * nu * sizeof(double), st>>>(
      nq, nu, nloc, nt, Bpu, codes, x, y);
  return launch_status();
}

MCS_API int mcs_apply_BT(int nq, int nu, int nloc, int64_t nt, const double* Bpu, const int* codes,
                         const double* p, double* y, void* stream) {
  if (nt <= 0) return 0;
  auto st = static_cast<cudaStream_t>(stream);
  apply_BT_kernel<<<sk_grid(nt * nu), SK_THREADS, nq * nu * sizeof(double), st>>>(
      nq, nu, nloc, nt, Bpu, codes, p, y);
  return launch_status();
}

MCS_API int mcs_mdot_len(void) { return MD_CHUNKS; }

MCS_API int mcs_mdot_gated(int m, int64_t n, int64_t ld, const double* V, const double* w,
                           double* partial, double* h, const double* gate, void* stream) {
  if (m <= 0) return 0;
  auto st = static_cast<cudaStream_t>(stream);
  mdot_partial_kernel<<<dim3(MD_CHUNKS, m), SK_THREADS, 0, st>>>(n, ld, V, w, partial, gate);
  int rc = launch_status();
  if (rc) return rc;
  mdot_final_kernel<<<(m + 127) / 128, 128, 0, st>>>(m, partial, h, gate);
  return launch_status();
}

MCS_API int mcs_mdot(int m, int64_t n, int64_t ld, const double* V, const double* w,
                     double* partial, double* h, void* stream) {
  return mcs_mdot_gated(m, n, ld, V, w, partial, h, nullptr, stream);
}

MCS_API int mcs_gemv_acc_gated(int m, int64_t n, int64_t ld, const double* V, const double* h,
                               double alpha, double beta, double* w, const double* gate,
                               void* stream) {
  if (n <= 0) return 0;
  auto st = static_cast<cudaStream_t>(stream);
  gemv_acc_kernel<<<(int)((n + SK_THREADS - 1) / SK_THREADS), SK_THREADS, 0, st>>>(m, n, ld, V, h, alpha, beta, w, gate);
  return launch_status();
}

MCS_API int mcs_gemv_acc(int m, int64_t n, int64_t ld, const double* V, const double* h,
                         double alpha, double beta, double* w, void* stream) {
  return mcs_gemv_acc_gated(m, n, ld, V, h, alpha, beta, w, nullptr, stream);
}

MCS_API int mcs_gs_gate(double* sc, int before, int after, int gate, void* stream) {
  gs_gate_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(sc, before, after, gate);
  return launch_status();
}

// sub-tile width for m basis vectors (64 KB of shared memory per CTA); 0 =
// the fused pass is not available (m > 1024: use the unfused kernels)
static int gs_sub(int m) {
  const int need = m + 2;                     // tile rows + partial / w' slack
  if (m > 1024) return 0;
  for (int sub = 32; sub >= 8; sub /= 2)
    if ((int64_t)need * sub * 8 + (GS_THREADS / sub) * sub * 8 <= GS_SMEM) return sub;
  return 0;
}

MCS_API int mcs_gs_fused_blocks(void) { return 2 * 148; }

MCS_API int mcs_gs_fused(int m, int64_t n, int64_t ld, const double* V, double* w, const double* h1,
                         double* ph2, double* pnrm, double* h2, double* sc, int before, int after,
                         int gate, void* stream) {
  const int sub = gs_sub(m);
  if (sub == 0 || m <= 0) return -1000;
  auto st = static_cast<cudaStream_t>(stream);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gs_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, GS_SMEM);
    attr = true;
  }
  const int nblk = mcs_gs_fused_blocks();
  const size_t smem = ((size_t)m * sub + (GS_THREADS / sub) * sub + sub) * sizeof(double);
  gs_fused_kernel<<<nblk, GS_THREADS, smem, st>>>(m, n, ld, sub, V, w, h1, ph2, pnrm);
  int rc = launch_status();
  if (rc) return rc;
  gs_final_kernel<<<1, 256, 0, st>>>(m, nblk, ph2, pnrm, h2, sc, before, after, gate);
  return launch_status();
}
