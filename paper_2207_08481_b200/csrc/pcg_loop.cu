// A13 PCG: the whole iteration loop as ONE CUDA graph launch.
//
// The captured two-step PCG graph (krylov.py `_PcgState.capture`: A p with
// p'Ap, the gated x/r update with ||r||^2, z = M r, r'z, the p update, twice)
// becomes the body of a conditional WHILE node.  After each pair a one-thread
// record kernel appends (p'Ap, ||r||^2) of the steps that ran to a device
// history and evaluates the host loop's stopping test (krylov.py `cg`,
// reference krylov.py:103-137: stop when p'Ap <= 0 (a NaN does not stop), or
// sqrt(rr) / ||b|| <= rtol, the same IEEE operations) plus the maxit cap; the
// conditional handle keeps looping while neither fires.  The host then reads
// the history once and replays the reference's control flow over it, so the
// residual history and iteration count are those of the pair-per-launch loop,
// without a host round trip every two iterations.
//
// history layout (float64): [0] steps recorded, [1] maxit, then (p'Ap, rr)
// per step.
#include "common.cuh"

namespace mcs {

__global__ void pcg_loop_init_kernel(double* hist, int maxit) {
  hist[0] = 0.0;
  hist[1] = (double)maxit;
}

__global__ void pcg_record_kernel(const double* __restrict__ sc, double* __restrict__ hist, int pap,
                                  int rr, int pap2, int rr2, int bnorm_i, int rtol_i, int cap,
                                  cudaGraphConditionalHandle h) {
  int c = (int)hist[0];
  const int maxit = min((int)hist[1], cap);
  const double bn = sc[bnorm_i], rt = sc[rtol_i];
  bool stop = false;
  for (int s = 0; s < 2 && !stop; ++s) {
    const double a = sc[s == 0 ? pap : pap2], b = sc[s == 0 ? rr : rr2];
    hist[2 + 2 * c] = a;
    hist[3 + 2 * c] = b;
    ++c;
    stop = a <= 0.0 || sqrt(b) / bn <= rt;   // the gate's test (cg_update_kernel)
  }
  hist[0] = (double)c;
  cudaGraphSetConditional(h, (!stop && c + 2 <= maxit) ? 1u : 0u);
}

}  // namespace mcs

using namespace mcs;

MCS_API int mcs_pcg_loop_build(void* pair_graph, const double* sc, double* hist, int pap, int rr,
                               int pap2, int rr2, int bnorm_i, int rtol_i, int cap,
                               void** exec_out) {
  if (!pair_graph || !exec_out || cap < 2) return -1000;
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaGraphCreate(&g, 0);
  if (e != cudaSuccess) return err_code(e);
  cudaGraphConditionalHandle h;
  cudaGraphExec_t ex = nullptr;
  cudaGraphNode_t wn, child, kn;
  cudaGraphNodeParams cp = {};
  cudaKernelNodeParams kp = {};
  void* args[] = {&sc, &hist, &pap, &rr, &pap2, &rr2, &bnorm_i, &rtol_i, &cap, &h};
  e = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
  if (e != cudaSuccess) goto done;
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  e = cudaGraphAddNode(&wn, g, nullptr, 0, &cp);
  if (e != cudaSuccess) goto done;
  e = cudaGraphAddChildGraphNode(&child, cp.conditional.phGraph_out[0], nullptr, 0,
                                 static_cast<cudaGraph_t>(pair_graph));
  if (e != cudaSuccess) goto done;
  kp.func = (void*)pcg_record_kernel;
  kp.gridDim = dim3(1);
  kp.blockDim = dim3(1);
  kp.kernelParams = args;
  e = cudaGraphAddKernelNode(&kn, cp.conditional.phGraph_out[0], &child, 1, &kp);
  if (e != cudaSuccess) goto done;
  e = cudaGraphInstantiate(&ex, g, 0);
done:
  cudaGraphDestroy(g);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return err_code(e);
  }
  *exec_out = ex;
  return 0;
}

MCS_API int mcs_pcg_loop_launch(void* exec, double* hist, int maxit, void* stream) {
  auto st = static_cast<cudaStream_t>(stream);
  pcg_loop_init_kernel<<<1, 1, 0, st>>>(hist, maxit);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return err_code(e);
  return err_code(cudaGraphLaunch(static_cast<cudaGraphExec_t>(exec), st));
}

MCS_API int mcs_pcg_loop_destroy(void* exec) {
  return exec ? err_code(cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(exec))) : 0;
}
