/* mcs_abi.h -- C ABI of libmcsgpu.so, the B200 (sm_100a) kernels behind the
 * condensed MCS Stokes hot path (arXiv 2207.08481; reference package
 * `mcstokes`, pure NumPy/SciPy).
 *
 * Conventions
 *   - every pointer is a DEVICE pointer owned by the caller (torch tensors);
 *   - `stream` is a cudaStream_t; every call is asynchronous on it;
 *   - return 0 = ok, < 0 = CUDA error (-cudaError_t) or unsupported
 *     arguments (-1000); per-element failures go to `info[e]` (0 = ok,
 *     otherwise the 1-based failing pivot), mapped to the reference's
 *     exceptions by the Python layer;
 *   - float64 everywhere; int32 index arrays;
 *   - packed symmetric = lower triangle, row-major, (i,j) at i(i+1)/2 + j,
 *     per-element stride padded to an even number of doubles;
 *   - dof codes: 2*free_index + (sign < 0), or -1 for a constrained dof.
 *
 * No function keeps global mutable state.  There is no CPU fallback.
 */
#ifndef MCS_ABI_H
#define MCS_ABI_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- element blocks (replaces assembly.py:49-96 assemble_element_blocks /
 *      all_element_blocks): rec[e][q] = sum_p W[e][widx[p]] * coef[p] over the
 *      CSR program of refblocks.py.  W: [nt][nwgt] geometry weights. */
int mcs_element_blocks(int64_t nt, int nwgt, const double* W, int reclen, const int* prog_ptr,
                       const int* prog_widx, const double* prog_coef, double* records,
                       void* stream);

/* record layout / packed strides for degree k (2..6) */
int mcs_record_len(int k);
int mcs_st_stride(int k);
int mcs_ext_stride(int k);
int mcs_sd_stride(int k);

/* ---- sigma/omega condensation (replaces condensation.py:159-177, the LU of
 *      [[-msig, bws^T],[bws, 0]] and S_T = adiv - Bsig M^-1 Bsig^T per element).
 *      records: [nt][mcs_record_len(k)], S_packed: [nt][mcs_st_stride(k)]. */
int mcs_condense(int k, int64_t nt, const double* records, double* S_packed, int* info,
                 void* stream);

/* ---- structured sigma/omega condensation (same result as mcs_condense,
 *      exploiting the block structure of the MCS element spaces, DESIGN.md
 *      §3.2): S_T = adiv + Y Y^T, Y = [B_m F_m | B_b L_b^-T].  srecords:
 *      [nt][mcs_srec_len(k)] = [s | A_m 3x3 blocks | Mb | Bsig | adiv]. */
int mcs_srec_len(int k);
int mcs_condense_struct(int k, int64_t nt, const double* srecords, double* S_packed, int* info,
                        void* stream);

/* ---- generation-fused structured condensation for any k (used for k = 5, 6,
 *      where Y does not fit a warp's registers): S_T from the geometry weights
 *      W [nt][nwgt >= 30] and the tables [mcs_fused_table_len(k)]; the compact
 *      record never reaches HBM.  k = 5, 6: the warp-per-element pipeline of
 *      mcs_condense_fused in passes over the columns of Y (the lane-ordered
 *      tables live in a library-owned device buffer rebuilt on `stream` at
 *      every call: concurrent calls for the same k with DIFFERENT tables on
 *      different streams are not supported); k <= 4 (and MCS_GEN=1): CTA per
 *      element, Y in shared memory. */
int mcs_condense_gen(int k, int64_t nt, const double* W, int nwgt, const double* tables,
                     double* S_packed, int* info, void* stream);
/* k = 5, 6: mcs_condense_gen plus the double Schur outputs in the same kernel
 *      (replaces condensation.py:159-177 AND :207-226 per element): ext and
 *      Sd_packed as mcs_double_schur; info bit 0: singular stress block,
 *      bit 1: S_oo not SPD. */
int mcs_condense_gen_ds(int k, int64_t nt, const double* W, int nwgt, const double* tables,
                        double* S_packed, double* ext, double* Sd_packed, int* info, void* stream);

/* ---- fused element pipeline, k = 2..6 (replaces assembly.py:49-91 +
 *      condensation.py:159-177 + condensation.py:207-226 per element): one
 *      warp per element generates Bsig from the reference-cell tables and the
 *      element's geometry weights W [nt][nwgt >= 30], forms S_T = adiv + Y Y^T
 *      and the double Schur outputs (ext, Sd_packed as mcs_double_schur).
 *      (The package uses it for k <= 4; at k = 5, 6 mcs_condense_gen followed
 *      by mcs_double_schur gives bitwise the same outputs and is faster.)
 *      tables: [mcs_fused_table_len(k)] (engine.fused_tables).  info bit 0:
 *      singular stress block, bit 1: S_oo not SPD. */
int mcs_fused_table_len(int k);
int mcs_condense_fused(int k, int64_t nt, const double* W, int nwgt, const double* tables,
                       double* S_packed, double* ext, double* Sd_packed, int* info, void* stream);

/* ---- stress recovery (replaces CondensedSystem.recover_stress,
 *      condensation.py:64-74: (sigma, omega)_T = -M^-1 [Bsig^T; 0] u_T): one
 *      warp per element regenerates Bsig from the weights W [nt][nwgt >= 30]
 *      and the tables [mcs_recover_table_len(k)], solves with the block
 *      structure of msig / bws.  vv_codes: [nt][nloc] codes over ALL (V, Vhat)
 *      dofs (2*global + (sign < 0)); x_full: all (V, Vhat) dofs; sigma:
 *      [nt][ns], omega: [nt][nw] (element-major, the reference numbering).
 *      info[e] != 0: singular local stress block. */
int mcs_recover_table_len(int k);
int mcs_recover_stress(int k, int64_t nt, const double* W, int nwgt, const double* tables,
                       const int* vv_codes, const double* x_full, double* sigma, double* omega,
                       int* info, void* stream);

/* ---- post-solve structural checks (replaces driver.py:183-218 post_checks):
 *      out[0] = max |div u| over elements and quadrature points, out[1] / out[2]
 *      = max nt jump / max |nt| over interior facets and edge points; part:
 *      [nparts] per-warp partial sums of int |grad u|^2 (sum them in order).
 *      geo: [nt][10] = (J, J^-1 row-major, detJ, pad); vcodes: [nt][nu] V-dof
 *      codes over all V dofs; tab_div [nu][nq], tab_grad [nu][nq][2][2], wq [nq];
 *      fac: [nif][4] = (t0, le0, t1, le1), frame: [nif][4] = (t_F, n_F),
 *      flip: [nt][3], sigma: [nt][ns], tab_se: [ns][3][nqe][2][2], nqe <= 8. */
int mcs_post_checks(int64_t nt, int nu, int nq, const double* geo, const int* vcodes,
                    const double* u, const double* tab_div, const double* tab_grad,
                    const double* wq, int nif, int ns, int nqe, const int* fac,
                    const double* frame, const signed char* flip, const double* sigma,
                    const double* tab_se, double* out, double* part, int nparts, void* stream);

/* ---- double Schur (replaces condensation.py:207-226 double_schur per
 *      element): ext = [X = S_oo^-1 S_oc (n_int x ncpl) | S_oo^-1 packed],
 *      Sd_packed = S_cc - S_co X. */
int mcs_double_schur(int k, int64_t nt, const double* S_packed, double* ext, double* Sd_packed,
                     int* info, void* stream);

/* ---- config-5 microbench SPD Schur S = B^T A^-1 B (reference idiom
 *      condensation.py:216-224, cho_factor / cho_solve / B^T X).
 *      A_packed_lower: [batch][n(n+1)/2], B: [batch][n][m], S: [batch][m(m+1)/2].
 *      Compiled shapes: (60, 36), (8, 4). */
int mcs_spd_schur_batched(int n, int m, int64_t batch, const double* A_packed_lower,
                          const double* B, double* S_packed, int* info, void* stream);

/* ---- condensed operator apply (replaces driver.py:138,144 `S_free @ v`, and
 *      the S_d CSR of driver.py:96): y = sum_T P^T D S_T D P x over free dofs.
 *      which = 0: S_T (codes [nt][nloc]); which = 1: Sd_T (codes [nt][ncpl]).
 *      y (length ny) is overwritten. */
int mcs_apply_elem(int k, int which, int64_t nt, const double* M_packed, const int* codes,
                   const double* x, double* y, int64_t ny, void* stream);
/* the same apply fused with the CG curvature: *out = x . y =
 * sum_T x_T^T M_T x_T (fixed-order reduction over partials[grid] with the
 * last-block counter; partials: >= 8 * number of SMs doubles) */
int mcs_apply_elem_dot(int k, int which, int64_t nt, const double* M_packed, const int* codes,
                       const double* x, double* y, int64_t ny, double* partials,
                       unsigned* counter, double* out, void* stream);

/* ---- ExtendedAsp outer factors (replaces preconditioners.py:353-378):
 *      restrict: bubble[e] = S_oo^-1 r_o, acc = sum X^T r_o (signed; acc
 *      overwritten, length nacc); prolong: out[bubble dofs] = bubble - X z_c and
 *      out[c2v[j]] = z_c[j] for the coupling dofs (the scatter, fused). */
int mcs_ext_restrict(int k, int64_t nt, const double* ext, const int* bubble_idx,
                     const int* cpl_codes, const double* r, double* bubble, double* acc,
                     int64_t nacc, void* stream);
int mcs_ext_prolong(int k, int64_t nt, const double* ext, const int* bubble_idx,
                    const int* cpl_codes, const double* zc, const double* bubble, const int* c2v,
                    double* out, void* stream);
/* w[j] = r[map[j]] - acc[j];  out[map[j]] = z[j] */
int mcs_gather_sub(int n, const double* r, const int* map, const double* acc, double* w,
                   void* stream);
int mcs_scatter(int n, const double* z, const int* map, double* out, void* stream);

/* ---- facet-block Jacobi on S_d (replaces preconditioners.py:177-206 variant
 *      "jacobi" with facet_blocks_schur :266-280).  slots: [nblk][4] =
 *      (t0, le0, t1, le1); binv: [npk(2k+1)][nblk] SoA; bidx: [2k+1][nblk]. */
int mcs_jacobi_setup(int k, int nblk, const double* Sd_packed, int sd_stride, const int* cpl_codes,
                     const int* slots, double* binv, int* bidx, int* bsize, int* info,
                     void* stream);
int mcs_jacobi_apply(int k, int nblk, const double* binv, const int* bidx, const double* r,
                     double* x, double scale_inv, void* stream);

/* ---- CSR SpMV y = alpha A x + beta y (replaces the E_c / E_c^T products of
 *      preconditioners.py:316-317); lanes in {1, 4, 8, 32} per row. */
int mcs_csr_spmv(int nrows, const int* ptr, const int* col, const double* val, const double* x,
                 double* y, double alpha, double beta, int lanes, void* stream);

/* ---- exact coarse solve (replaces CoarseSolver.solve, SuperLU,
 *      preconditioners.py:111-118,165-171): dense explicit inverse (small)
 *      or multifrontal triangular solves (per tree level, see coarse.py). */
int mcs_dense_gemv(int n, const double* A, const double* x, double* y, void* stream);
/* one kernel per separator-tree level and direction, one CTA per node
 * (node table, packed factors and gather sources built by coarse.py) */
int mcs_mf_forward(int nnodes, const int* level_nodes, const void* nodes, const double* mats,
                   const int* src_t, const int* src_o, const int* perm, const double* b,
                   double* y, double* out, int max_ns, int max_nb, void* stream);
int mcs_mf_backward(int nnodes, const int* level_nodes, const void* nodes, const double* mats,
                    const int* B, const int* perm, const double* y, double* xp, double* x,
                    int max_ns, int max_nb, void* stream);
/* top of the tree (t dofs): g = b_T - frontier updates, x_T = Sinv g with the
 * dense inverse of the top Schur complement (= (A^-1)_TT).  Sinv is t rows of
 * ld = mcs_mf_top_ld(t) doubles (zero padded), g holds ld doubles whose
 * padding is zero (only g[0..t) is written). */
int mcs_mf_top_ld(int t);
int mcs_mf_top(int t, const int* T, const int* perm, const double* b, const int* ptr,
               const int* src, const double* out, double* g, const double* Sinv, double* xp,
               double* x, void* stream);

/* ---- Stokes (saddle) mode (replaces the B / B^T products of driver.py:148-151
 *      and preconditioners.py:405-420, and the Gram-Schmidt products of the
 *      GMRES of krylov.py:25-100).  Bpu: [nq][nu] reference matrix (J-invariant);
 *      codes: the free (V, Vhat) dof codes [nt][nloc] (first nu = V dofs);
 *      pressure dofs element-major [nt][nq].  B^T accumulates into y (zero it). */
int mcs_apply_B(int nq, int nu, int nloc, int64_t nt, const double* Bpu, const int* codes,
                const double* x, double* y, void* stream);
int mcs_apply_BT(int nq, int nu, int nloc, int64_t nt, const double* Bpu, const int* codes,
                 const double* p, double* y, void* stream);
/* h[i] = V[i] . w for i < m (V row-major, leading dimension ld); partial:
 * [m][mcs_mdot_len()] scratch.  w = beta w + alpha V^T h.  Deterministic. */
int mcs_mdot_len(void);
int mcs_mdot(int m, int64_t n, int64_t ld, const double* V, const double* w, double* partial,
             double* h, void* stream);
int mcs_gemv_acc(int m, int64_t n, int64_t ld, const double* V, const double* h, double alpha,
                 double beta, double* w, void* stream);
/* the same, skipped (h = 0, w unchanged) when *gate != 0; mcs_gs_gate sets
 * sc[gate] = 1 when sqrt(sc[after]) > sqrt(sc[before]) / sqrt(2) (the DGKS
 * test of krylov.py gmres), so the second Gram-Schmidt pass needs no host
 * decision (replaces the reorthogonalisation branch of krylov.py:25-100) */
int mcs_mdot_gated(int m, int64_t n, int64_t ld, const double* V, const double* w,
                   double* partial, double* h, const double* gate, void* stream);
int mcs_gemv_acc_gated(int m, int64_t n, int64_t ld, const double* V, const double* h,
                       double alpha, double beta, double* w, const double* gate, void* stream);
int mcs_gs_gate(double* sc, int before, int after, int gate, void* stream);
/* One basis read for the second Gram-Schmidt pass (replaces, per GMRES step,
 * the gemv w -= V h1, the dot ||w||^2, mcs_gs_gate and the gated mdot):
 * w <- w - V h1 in place, h2 = V^T w (0 when the gate skips the second pass),
 * sc[after] = ||w||^2, sc[gate] as mcs_gs_gate.  ph2: [m][mcs_gs_fused_blocks()],
 * pnrm: [mcs_gs_fused_blocks()].  Returns -1000 when m exceeds the shared-
 * memory tile (m > 990): the caller then uses the unfused kernels. */
int mcs_gs_fused_blocks(void);
int mcs_gs_fused(int m, int64_t n, int64_t ld, const double* V, double* w, const double* h1,
                 double* ph2, double* pnrm, double* h2, double* sc, int before, int after,
                 int gate, void* stream);

/* ---- PCG vector algebra (replaces krylov.py:103-137 NumPy ops); deterministic
 *      reductions into device scalars sc[]. */
int mcs_reduce_workspace_len(void);
int mcs_dot(int64_t n, const double* x, const double* y, double* partials, unsigned* counter,
            double* out, void* stream);
int mcs_cg_update(int64_t n, double* x, double* r, const double* p, const double* Ap, double* sc,
                  int rz, int pap, int rr, double* partials, unsigned* counter, void* stream);
/* the same with a stop gate, for several PCG steps per CUDA graph: a no-op
 * when sc[gate_in] != 0 (gate_in >= 0); sets sc[gate_out] = 1 when
 * sc[pap] <= 0 or sqrt(sc[rr]) / sc[bnorm_i] <= sc[rtol_i] (gate_out >= 0; a NaN
 * sets neither, as in the reference loop krylov.py:121-131) */
int mcs_cg_update_gated(int64_t n, double* x, double* r, const double* p, const double* Ap,
                        double* sc, int rz, int pap, int rr, int gate_in, int gate_out,
                        int bnorm_i, int rtol_i, double* partials, unsigned* counter,
                        void* stream);
int mcs_xpby(int64_t n, const double* z, double* p, const double* sc, int num, int den,
             void* stream);
int mcs_axpby(int64_t n, double a, const double* x, double b, double* y, void* stream);
/* y = x / d elementwise (PressureMassPrecond.apply, preconditioners.py:400-401) */
int mcs_vdiv(int64_t n, const double* x, const double* d, double* y, void* stream);
/* y[0..n) = 0 as a memset node (accumulation targets of the atomic scatters) */
int mcs_zero(int64_t n, double* y, void* stream);

/* ---- A13 PCG loop as one CUDA graph (csrc/pcg_loop.cu) ------------------
 * Replaces the host iteration loop of krylov.py:103-137 (one Python
 * iteration per step) with a conditional WHILE graph around the captured
 * two-step PCG graph `pair_graph` (a cudaGraph_t).  After each pair a record
 * kernel appends (sc[pap], sc[rr]) of the steps that ran to `hist`
 * ([0] steps, [1] maxit, then two doubles per step, room for `cap` steps) and
 * stops the loop on p'Ap <= 0, sqrt(rr) / sc[bnorm_i] <= sc[rtol_i], or
 * maxit.  build: *exec_out = the instantiated graph (cudaGraphExec_t). */
int mcs_pcg_loop_build(void* pair_graph, const double* sc, double* hist, int pap, int rr,
                       int pap2, int rr2, int bnorm_i, int rtol_i, int cap, void** exec_out);
int mcs_pcg_loop_launch(void* exec, double* hist, int maxit, void* stream);
int mcs_pcg_loop_destroy(void* exec);

/* ---- CondensedSystem vector methods over ALL (V, Vhat) dofs (csrc/factorized.cu)
 *      vv_codes: [nt][nloc] = 2*global + (sign < 0), as mcs_recover_stress.
 *  mcs_apply_S_factorized  replaces condensation.py:104-122
 *      (CondensedSystem.apply_S_factorized): y += S x through
 *      [I X^T; 0 I] [Sd 0; 0 S_oo] [I 0; X I] per element, from S_packed
 *      (S_oo block), ext (X) and Sd_packed; y must be zeroed by the caller.
 *  mcs_harmonic_extend     replaces condensation.py:93-102
 *      (CondensedSystem.harmonic_extend): out[bubble dofs] = -X x_c; the
 *      caller copies x into out first (out keeps the coupling dofs). */
int mcs_apply_S_factorized(int k, int64_t nt, const double* S_packed, const double* ext,
                           const double* Sd_packed, const int* vv_codes, const double* x,
                           double* y, void* stream);
int mcs_harmonic_extend(int k, int64_t nt, const double* ext, const int* vv_codes,
                        const double* x, double* out, void* stream);
/* ---- packed inverses of caller-supplied SPD blocks for the facet Jacobi
 *      apply (replaces the per-block cho_factor of FacetBlockSmoother.__init__,
 *      preconditioners.py:186-200, when the smoother is built from a CSR
 *      matrix and a block list): blocks [nblk][B][B] row-major, idx [nblk][B]
 *      (-1 padding), bsize [nblk], B = 2k+1; outputs as mcs_jacobi_setup.
 *      info[b] = 1 + first non-positive pivot. */
int mcs_block_inverse(int k, int nblk, const double* blocks, const int* idx, const int* bsize,
                      double* binv, int* bidx, int* info, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MCS_ABI_H */
