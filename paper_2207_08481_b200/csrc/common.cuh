// Shared helpers for the MCS condensation / PCG kernels (sm_100a only).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "mcs_abi.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "this library targets sm_100a (B200) only"
#endif

#define MCS_API extern "C" __attribute__((visibility("default")))

namespace mcs {

// SMs of the current device (cached; 148 on B200)
inline int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}


// lower-packed, row-major: (i, j) with j <= i  ->  i(i+1)/2 + j
__host__ __device__ constexpr int pk(int i, int j) { return i * (i + 1) / 2 + j; }
__host__ __device__ constexpr int npk(int n) { return n * (n + 1) / 2; }
__host__ __device__ constexpr int even(int n) { return (n + 1) & ~1; }

// local sizes of the MCS element at degree k
template <int K>
struct Sizes {
  static constexpr int k = K;
  static constexpr int ns = 3 * (K + 1) * (K + 2) / 2 - 3;
  static constexpr int nw = K * (K + 1) / 2;
  static constexpr int nu = (K + 1) * (K + 2);
  static constexpr int nh = 3 * K;
  static constexpr int nloc = nu + nh;
  static constexpr int n_em = 3 * (K + 1);
  static constexpr int n_int = (K + 1) * (K - 1);
  static constexpr int ncpl = nloc - n_int;
  static constexpr int naug = ns + nw + nloc;   // augmented saddle size
};

inline int err_code(cudaError_t e) { return e == cudaSuccess ? 0 : -static_cast<int>(e); }

// ---- programmatic dependent launch (PDL) for the PCG kernel chain --------
// Kernels launched with launch_pdl_g() may start while their predecessor in
// the stream is still running: each calls pdl_wait() before it reads anything
// an earlier kernel wrote or writes any global memory, and pdl_trigger()
// right after it (so at most one kernel waits ahead of the running one: a
// trigger at kernel entry lets a cascade of waiting grids pin SM slots that
// multi-wave predecessors still need).  Before pdl_wait()
// only static data is touched (element matrices, index maps, factors), so
// index loads, bulk copies and L2 prefetches overlap the predecessor's tail
// and the launch latency.  Stream capture turns the attribute into
// programmatic graph edges.  MCS_NO_PDL=1 launches normally.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// kernel groups (MCS_PDL_MASK bit): 1 vector kernels, 2 ExtendedAsp element
// kernels, 4 smoother / SpMV, 8 coarse solve, 16 the S / S_d element apply
enum PdlGroup { PDL_BLAS = 1, PDL_ELEM = 2, PDL_PREC = 4, PDL_COARSE = 8, PDL_APPLY = 16 };
bool pdl_enabled(int group);

template <class... KArgs, class... Args>
inline int launch_pdl_g(int group, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                        cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled(group) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return err_code(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
}

// Return the pending launch error (if any) as a negative code.
inline int launch_status() { return err_code(cudaGetLastError()); }

// per-element outputs of the double Schur (condensation.py:207-226):
//   ext record  [X (n_int x ncpl, row-major) | S_oo^-1 (lower packed)]  (even stride)
//   Sd_T        lower packed (even stride)
template <int K>
struct ExtLayout {
  using Z = Sizes<K>;
  static constexpr int x_len = Z::n_int * Z::ncpl;
  static constexpr int len = even(x_len + npk(Z::n_int));
  static constexpr int sd_len = even(npk(Z::ncpl));
  static constexpr int st_len = even(npk(Z::nloc));
};

// local index of coupling dof c (facet BDM dofs, then Vhat)
template <int K>
__device__ __forceinline__ int cpl_local(int c) {
  using Z = Sizes<K>;
  return c < Z::n_em ? c : c + Z::n_int;
}

// reference-cell tables of the fused kernel (doubles):
//   G4 [NR][ns][4] = (base, T_0, T_1, T_2) per Bsig entry | Adiv [nu][nu] |
//   MbRef [6][nb][nb] | ARef [6][ml][9]      (rows >= nloc zero; segments even)
template <int K>
struct FTab {
  using Z = Sizes<K>;
  static constexpr int ml = K * (K + 1) / 2, nl = 3 * ml, nb = 3 * K;
  static constexpr int NR = (Z::nloc + 7) / 8 * 8;
  static constexpr int o_G4 = 0;
  static constexpr int o_adiv = o_G4 + 4 * NR * Z::ns;
  static constexpr int o_Mb = o_adiv + even(Z::nu * Z::nu);
  static constexpr int o_A = o_Mb + even(6 * nb * nb);
  static constexpr int len = o_A + even(6 * 9 * ml);
};

// FP64 tensor-core MMA, m8n8k4: lane (g, t) supplies A[g][t], B[t][g] and
// owns C[g][2t], C[g][2t+1]
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// 1/x to full double precision: hardware approximation + 2 Newton steps
__device__ __forceinline__ double rcp64(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  y = fma(fma(-x, y, 1.0), y, y);
  return fma(fma(-x, y, 1.0), y, y);
}

// 1/sqrt(x) to full double precision: hardware approximation + 2 Newton steps
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double r = fma(-x * y, y, 1.0);
  y = fma(0.5 * y, r, y);
  r = fma(-x * y, y, 1.0);
  return fma(0.5 * y, r, y);
}

// dof code: 2*index + (sign < 0), or -1 for a constrained dof (reads 0, no write)
__device__ __forceinline__ double code_sign(int c) { return (c & 1) ? -1.0 : 1.0; }
__device__ __forceinline__ int code_index(int c) { return c >> 1; }

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- 1-D bulk async copy (TMA engine, cp.async.bulk) global -> shared ----
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(phase)
      : "memory");
}

}  // namespace mcs
