// PCG vector algebra (krylov.py:103-137).
//
// Scalars stay on the device (`sc[]`): alpha = rz/pAp and beta = rz_new/rz
// are formed inside the kernels that consume them, so one iteration needs a
// single 16-byte device->host read (pAp, ||r||^2) for the reference's
// stopping test and negative-curvature check.  Reductions are deterministic:
// a fixed grid, fixed per-thread strides, a fixed shuffle tree per block and
// the last-arriving block summing the block partials in index order.
#include <cstdlib>

#include "common.cuh"

namespace mcs {

constexpr int RED_BLOCKS = 1184;  // 8 x 148 SMs: enough loads in flight for HBM
constexpr int RED_THREADS = 256;

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double ws[RED_THREADS / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) ws[w] = v;
  __syncthreads();
  double s = 0.0;
  if (w == 0) {
    s = l < RED_THREADS / 32 ? ws[l] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  }
  return s;  // valid in thread 0
}

// last block: sum partials[0..gridDim) -> *out with all its threads (fixed
// strided assignment + the fixed block_sum tree: deterministic).  Partials
// are read through L2 (ld.global.cg) after the fence, batched, instead of
// one volatile round trip at a time.
// Returns true in thread 0 of the last block, after *out is written.
__device__ __forceinline__ bool finish(double part, double* partials, unsigned* counter,
                                       double* out) {
  __shared__ bool last;
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = part;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
  double s = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += RED_THREADS) s += __ldcg(partials + b);
  s = block_sum(s);
  if (threadIdx.x == 0) {
    *out = s;
    *counter = 0u;
    return true;
  }
  return false;
}

__global__ void __launch_bounds__(RED_THREADS)
    dot_kernel(int64_t n, const double* __restrict__ x, const double* __restrict__ y,
               double* partials, unsigned* counter, double* out) {
  pdl_wait();
  pdl_trigger();
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * RED_THREADS + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * RED_THREADS)
    s = fma(x[i], y[i], s);
  s = block_sum(s);
  finish(s, partials, counter, out);
}

// alpha = sc[rz]/sc[pap];  x += alpha p;  r -= alpha Ap;  sc[rr] = r.r
// Gating (several PCG steps per CUDA graph, krylov.py): gate_in >= 0 and
// sc[gate_in] != 0 -> the step is a no-op (the previous step stopped the
// loop); gate_out >= 0 -> sc[gate_out] = 1 when this step stops the loop,
// with the host's own test: pAp <= 0 or sqrt(rr) / bnorm <= rtol (IEEE
// sqrt and division, so device and host decide identically; a NaN passes
// both, as in the reference loop, which then runs on to maxit).
__global__ void __launch_bounds__(RED_THREADS)
    cg_update_kernel(int64_t n, double* __restrict__ x, double* __restrict__ r,
                     const double* __restrict__ p, const double* __restrict__ Ap, double* sc,
                     int rz, int pap, int rr, int gate_in, int gate_out, int bnorm_i, int rtol_i,
                     double* partials, unsigned* counter) {
  pdl_wait();
  pdl_trigger();
  if (gate_in >= 0 && sc[gate_in] != 0.0) return;
  const double alpha = sc[rz] / sc[pap];
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * RED_THREADS + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * RED_THREADS) {
    x[i] = fma(alpha, p[i], x[i]);
    const double ri = fma(-alpha, Ap[i], r[i]);
    r[i] = ri;
    s = fma(ri, ri, s);
  }
  s = block_sum(s);
  if (finish(s, partials, counter, sc + rr) && gate_out >= 0) {
    const double rrv = sc[rr], pv = sc[pap];
    sc[gate_out] = (pv <= 0.0 || __dsqrt_rn(rrv) / sc[bnorm_i] <= sc[rtol_i]) ? 1.0 : 0.0;
  }
}

// p = z + (sc[num]/sc[den]) p
__global__ void xpby_kernel(int64_t n, const double* __restrict__ z, double* __restrict__ p,
                            const double* sc, int num, int den) {
  pdl_wait();
  pdl_trigger();
  const double beta = sc[num] / sc[den];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = fma(beta, p[i], z[i]);
}

// y = a x + b y
__global__ void axpby_kernel(int64_t n, double a, const double* __restrict__ x, double b,
                             double* __restrict__ y) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = b == 0.0 ? a * x[i] : fma(a, x[i], b * y[i]);
}

// y = x / d (elementwise, IEEE division: the reference's r / diag)
__global__ void vdiv_kernel(int64_t n, const double* __restrict__ x, const double* __restrict__ d,
                            double* __restrict__ y) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = x[i] / d[i];
}

static int grid_for(int64_t n);

}  // namespace mcs

bool mcs::pdl_enabled(int group) {
  static int mask = -1;
  if (mask < 0) {
    const char* e = getenv("MCS_NO_PDL");
    const char* m = getenv("MCS_PDL_MASK");
    // default 29: every group but the ExtendedAsp element kernels (launched
    // early they pin 3 CTAs/SM of shared memory while they wait: measured
    // ~1% slower on the multiplicative PCG; the S / S_d apply keeps PDL,
    // 60.4 vs 62.4 us standalone)
    mask = (e && e[0] == '1') ? 0 : (m ? atoi(m) : 29);
  }
  return (mask & group) != 0;
}

namespace mcs {

static int grid_for(int64_t n) {
  const int64_t g = (n + 255) / 256;
  return (int)(g < 16 * 148 ? (g < 1 ? 1 : g) : 16 * 148);
}

}  // namespace mcs

using namespace mcs;

// Partials slots: the fixed reduction grid, and one per CTA of the fused
// p'Ap element apply (apply.cu; at most 8 CTAs of 256 threads per SM).
MCS_API int mcs_reduce_workspace_len() {
  const int a = 8 * sm_count();
  return a > RED_BLOCKS ? a : RED_BLOCKS;
}

MCS_API int mcs_dot(int64_t n, const double* x, const double* y, double* partials, unsigned* counter,
                    double* out, void* stream) {
  auto st = static_cast<cudaStream_t>(stream);
  return launch_pdl_g(PDL_BLAS, dot_kernel, RED_BLOCKS, RED_THREADS, 0, st, n, x, y, partials, counter, out);
}

MCS_API int mcs_cg_update(int64_t n, double* x, double* r, const double* p, const double* Ap, double* sc,
                          int rz, int pap, int rr, double* partials, unsigned* counter, void* stream) {
  auto st = static_cast<cudaStream_t>(stream);
  return launch_pdl_g(PDL_BLAS, cg_update_kernel, RED_BLOCKS, RED_THREADS, 0, st, n, x, r, p, Ap, sc, rz, pap,
                    rr, -1, -1, 0, 0, partials, counter);
}

MCS_API int mcs_cg_update_gated(int64_t n, double* x, double* r, const double* p, const double* Ap,
                                double* sc, int rz, int pap, int rr, int gate_in, int gate_out,
                                int bnorm_i, int rtol_i, double* partials, unsigned* counter,
                                void* stream) {
  auto st = static_cast<cudaStream_t>(stream);
  return launch_pdl_g(PDL_BLAS, cg_update_kernel, RED_BLOCKS, RED_THREADS, 0, st, n, x, r, p, Ap, sc, rz, pap,
                    rr, gate_in, gate_out, bnorm_i, rtol_i, partials, counter);
}

MCS_API int mcs_xpby(int64_t n, const double* z, double* p, const double* sc, int num, int den,
                     void* stream) {
  auto st = static_cast<cudaStream_t>(stream);
  return launch_pdl_g(PDL_BLAS, xpby_kernel, grid_for(n), 256, 0, st, n, z, p, sc, num, den);
}

MCS_API int mcs_axpby(int64_t n, double a, const double* x, double b, double* y, void* stream) {
  if (n <= 0) return 0;
  auto st = static_cast<cudaStream_t>(stream);
  return launch_pdl_g(PDL_BLAS, axpby_kernel, grid_for(n), 256, 0, st, n, a, x, b, y);
}

MCS_API int mcs_vdiv(int64_t n, const double* x, const double* d, double* y, void* stream) {
  if (n <= 0) return 0;
  auto st = static_cast<cudaStream_t>(stream);
  return launch_pdl_g(PDL_BLAS, vdiv_kernel, grid_for(n), 256, 0, st, n, x, d, y);
}

// zero n doubles with a memset node (no kernel launch)
MCS_API int mcs_zero(int64_t n, double* y, void* stream) {
  if (n <= 0) return 0;
  return err_code(cudaMemsetAsync(y, 0, (size_t)n * sizeof(double), static_cast<cudaStream_t>(stream)));
}
