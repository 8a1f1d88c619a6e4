/*
 * alefsi_b200 — C ABI of the B200-native linear-solve path of the
 * approximated-Newton ALE-FSI solver (arXiv 1904.02401).
 *
 * This is the boundary a Python ctypes binding of the reference package
 * (pkg/src/alefsi) uses to replace its CPU solver objects; see
 * INTEGRATION.md for the binding.  Every entry point returns 0 on success or
 * an ALEFSI_ERR_* code; alefsi_last_error() describes the failure.
 * Plain pointers and sizes only.  Unless stated otherwise vector arguments
 * of the alefsi_mg_* calls are DEVICE pointers enqueued on the handle's
 * stream; functions with a host_ptrs flag accept host buffers when it is 1
 * and then synchronise before returning.
 *
 * Index conventions follow the reference: a level's dofs are node-major,
 * dof = node * nc + component with nc = dim + 1 (p, v_1..v_d); level 0 is
 * the coarsest level.
 *
 * Hard limits (violations return ALEFSI_ERR_ARG with a message):
 *   - GMRES max_iter in [1, 510] (Hessenberg columns staged in 512-entry
 *     shared arrays of the Krylov kernels);
 *   - coarsest level at most 4096 dofs (dense explicit inverse, one n x 16
 *     panel per cluster of CTAs);
 *   - Vanka patch sizes with compiled kernels: nc = 3 with 27 / 75 / 81 dofs
 *     per patch, nc = 4 with 108 / 500, nc = 2 with 18 (2D/3D Q2 one-element
 *     and 2x2(x2)-cell macro patches of the reference's PatchSet);
 *   - device assembly (asm_*): fewer than 2^31 blocks per level, dim 2 or 3,
 *     nq == 3^dim Gauss points; the shape tables of one dim are loaded once
 *     per process and later calls must pass the same tables.
 */
#ifndef ALEFSI_B200_H
#define ALEFSI_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ALEFSI_OK 0
#define ALEFSI_ERR_ARG 1
#define ALEFSI_ERR_CUDA 2
#define ALEFSI_ERR_SINGULAR 3       /* linsolve.py:132-133 "singular Vanka patch block" */
#define ALEFSI_ERR_NOT_CONVERGED 4  /* linsolve.py:110-114 GMRES stalled -> SolverError */
#define ALEFSI_ERR_STATE 5
#define ALEFSI_ERR_INTERNAL 6

typedef struct alefsi_mg_opaque* alefsi_mg;

const char* alefsi_last_error(void);
int alefsi_abi_version(void);
int alefsi_device_count(int32_t* count);

/* ---- host-side index structures (no GPU needed) ------------------------ */

/* Row-sorted union of element stencils; replaces BlockPattern's key
 * construction (reference fem.py:119-133).  Call once with indices == NULL
 * to fill indptr[n_nodes+1], then again with indices[indptr[n_nodes]]. */
int alefsi_pattern_build(int64_t n_nodes, int64_t n_elem, const int64_t* elem_ptr,
                         const int64_t* elem_nodes, int64_t* indptr, int32_t* indices);

/* slots[e][a][b] of the pair (elem[e][a], elem[e][b]) or -1; replaces
 * BlockPattern.slots_for (reference fem.py:138-146). */
int alefsi_pattern_slots(int64_t n_nodes, const int64_t* indptr, const int32_t* indices,
                         int64_t n_elem, int32_t npe, const int64_t* elem_nodes, int64_t* slots);

/* data[slot(e,a,b)] += local[e][a][b] (bs doubles per pair) in flattened
 * order; replaces BlockPattern.scatter / scatter_subset np.add.at
 * (reference fem.py:151-155, 166-169). */
int alefsi_scatter_add_blocks(int64_t n_nodes, const int64_t* indptr, const int32_t* indices,
                              int64_t n_elem, int32_t npe, const int64_t* elem_nodes, int32_t bs,
                              const double* local, double* data, int32_t skip_missing);

/* slot_in_a[s] = slot of entry s of row-sorted pattern B in pattern A, or -1
 * (splits the LPS macro pattern against the cell pattern; fem.py:79-90). */
int alefsi_pattern_match(int64_t n_nodes, const int64_t* a_ptr, const int32_t* a_idx,
                         const int64_t* b_ptr, const int32_t* b_idx, int64_t* slot_in_a);

/* Entries of the LPS macro pattern outside the cell pattern (to_cell < 0):
 * the scalar pressure-extension pattern pp_indptr / pp_indices and, per macro
 * entry, its extension slot to_pp (-1 when it has a cell slot).  Completes
 * the split of reference problem.py:79-90 (the LPS operator on the union
 * pattern) into cell blocks + pressure extension. */
int alefsi_split_extension(int64_t n_nodes, const int64_t* mptr, const int32_t* mind,
                           const int64_t* to_cell, int64_t* pp_indptr, int32_t* pp_indices,
                           int64_t* to_pp);

/* Greedy first-fit patch coloring; replaces color_patches
 * (reference mesh.py:522-556).  patch_size is the dof count per patch. */
int alefsi_color_patches(int64_t n_patches, const int64_t* patch_ptr, const int64_t* patch_nodes,
                         const int64_t* patch_size, int64_t n_nodes, int64_t* color,
                         int64_t* n_colors);

/* ---- device multigrid hierarchy ----------------------------------------- */

/* MgSolver(levels, nu_pre, nu_post) + VankaSmoother(omega)
 * (reference linsolve.py:229-236, 147-161). */
int alefsi_mg_create(int32_t n_levels, int32_t nc, int32_t nu_pre, int32_t nu_post, double omega,
                     alefsi_mg* out);
int alefsi_mg_destroy(alefsi_mg h);
/* Enqueue on a caller-owned cudaStream_t (e.g. torch's current stream). */
int alefsi_mg_set_stream(alefsi_mg h, void* stream);
/* Capture the V-cycle once as a CUDA graph and replay it. */
int alefsi_mg_use_graph(alefsi_mg h, int32_t on);

/* Level operator MgLevel.matrix (reference linsolve.py:223; assembled by
 * model.momentum_jacobian_data, model.py:297-381) in the split layout:
 * nc x nc blocks on the Q2 cell-stencil pattern plus scalar
 * pressure-pressure entries on the LPS macro pattern outside it.  A
 * reference BlockPattern/data pair maps onto it exactly.
 * HOST pointers; copied to HBM. */
int alefsi_mg_set_matrix(alefsi_mg h, int32_t level, int64_t n_nodes, int64_t nnzb,
                         const int64_t* indptr, const int32_t* indices, const double* data,
                         int64_t nnz_pp, const int64_t* pp_indptr, const int32_t* pp_indices,
                         const double* pp_data);

/* Operator structure only (data zeroed on the device), for device assembly. */
int alefsi_mg_set_pattern(alefsi_mg h, int32_t level, int64_t n_nodes, int64_t nnzb,
                          const int64_t* indptr, const int32_t* indices, int64_t nnz_pp,
                          const int64_t* pp_indptr, const int32_t* pp_indices);

/* Device assembly of the condensed Jacobian (model.momentum_jacobian_data,
 * reference model.py:297-381).  asm_setup (once per level): Q2 cell nodes
 * (n_cells, 3^dim) int32, node coordinates (n_nodes, dim), cells grouped by
 * colour (group_kind 0 fluid / 1 solid; a colour's cells share no node), the
 * LPS macro entries as (cell slot | -1, pp slot | -1, value) triples
 * (problem.py:79-90) and the Dirichlet row mask (n_nodes*nc bytes).
 * asm_tables: Q2 basis N (nq,nb), gradients dN (nq,nb,dim), weights (nq);
 * nq must equal nb = 3^dim; one constant bank per dim, loaded by the first
 * call for that dim (later calls must pass identical tables).
 * asm_momentum: params = {rho_f, mu_f, rho_s, mu_s, lam_s, k, theta}; U and
 * U_prev host (n_nodes, 1+2dim); extra = host-reduced outflow-facet blocks
 * (unique slots; pass n_extra = 0 once asm_outflow has been called for the
 * level).  The matrix must be re-factorised afterwards.  Assembling level 0
 * also starts that level's dense inverse on a side stream, so that it runs
 * under the assembly of the finer levels; alefsi_mg_factorize joins it (any
 * later change of level 0 before the factorisation discards it).
 * asm_outflow (once per level): the do-nothing outflow facets
 * (model._outflow_blocks, reference model.py:363-375) for assembly on the
 * device: owner-cell nodes conn (n_facets, 3^dim) and cell ids, facet
 * quadrature N (n_facets, nq, 3^dim), G (n_facets, nq, 3^dim, dim), dS
 * (n_facets, nq), normal (n_facets, nq, dim), and the slot reduction plan:
 * n_unique matrix slots, and per slot u the flat (facet, b, a) block indices
 * contrib[uptr[u]:uptr[u+1]] in ascending order. */
int alefsi_mg_asm_setup(alefsi_mg h, int32_t level, int32_t dim, int64_t n_cells,
                        const int32_t* cell_nodes, const double* coords, int32_t n_groups,
                        const int64_t* group_ptr, const int32_t* group_kind,
                        const int32_t* group_cells, int64_t n_lps, const int64_t* lps_cell_slot,
                        const int64_t* lps_pp_slot, const double* lps_vals,
                        const uint8_t* dirichlet);
int alefsi_mg_asm_tables(alefsi_mg h, int32_t dim, int32_t nq, const double* N, const double* dN,
                         const double* w);
int alefsi_mg_asm_momentum(alefsi_mg h, int32_t level, const double* params, const double* U,
                           const double* U_prev, int64_t n_extra, const int64_t* extra_slots,
                           const double* extra_vals);
int alefsi_mg_asm_outflow(alefsi_mg h, int32_t level, int64_t n_facets, int32_t nq,
                          const int32_t* conn, const int64_t* cells, const double* N,
                          const double* G, const double* dS, const double* normal,
                          int64_t n_unique, const int64_t* slots, const int64_t* uptr,
                          const int64_t* contrib);
/* Cell parts of the theta-step residual (which = 0, model.theta_residual,
 * reference model.py:208-275, out (n_nodes, 1+2dim)) or of the explicit
 * previous-state forces (which = 1, model.explicit_forces, model.py:159-185,
 * out (n_nodes, dim)) on the device; params = {rho_f, mu_f, rho_s, mu_s,
 * lam_s, k, theta, f0, f1, f2, ext_model (0 harmonic, 1 linear elasticity),
 * ext_mu, ext_lam, ext_volume_scaling}.  Host arrays; U may be NULL for
 * which = 1. */
int alefsi_mg_asm_residual(alefsi_mg h, int32_t level, const double* params, const double* U,
                           const double* U_prev, int32_t which, double* out);
/* Residual tail on the device (reference model.py:191-205 and 277-283):
 * after this call asm_residual also adds the do-nothing outflow rows
 * (which = 0: scaled by k*theta into R[:, 1:1+dim]; which = 1: into the
 * explicit forces) and, for which = 0, k * (L @ p) into R[:, 0] with the
 * scalar LPS operator L given as CSR (n_nodes rows).  The outflow rows are
 * reduced per node: onodes (unique facet nodes), and per node u the flat
 * (facet, b) indices ocontrib[ouptr[u]:ouptr[u+1]] in ascending order.
 * Requires asm_outflow when n_onodes > 0. */
int alefsi_mg_asm_residual_tables(alefsi_mg h, int32_t level, const int64_t* lps_indptr,
                                  const int32_t* lps_indices, const double* lps_vals,
                                  int64_t n_onodes, const int64_t* onodes, const int64_t* ouptr,
                                  const int64_t* ocontrib);
/* Copy a level's operator data (blocks, pp entries) to host memory. */
int alefsi_mg_get_matrix(alefsi_mg h, int32_t level, double* data, double* pp_data);

/* PatchSet groups (reference mesh.py:446-480): n_groups homogeneous groups,
 * patch_nodes concatenated group after group (node ids, patch-major).
 * HOST pointers. */
int alefsi_mg_set_patches(alefsi_mg h, int32_t level, int32_t n_groups,
                          const int64_t* group_n_patches, const int32_t* group_nodes_per_patch,
                          const int64_t* patch_nodes);

/* MgLevel.P, scalar Q2 interpolation from level-1 to level as CSR over fine
 * nodes (reference linsolve.py:183-216).  HOST pointers. */
int alefsi_mg_set_prolongation(alefsi_mg h, int32_t level, int64_t n_fine, int64_t n_coarse,
                               int64_t nnz, const int64_t* indptr, const int32_t* indices,
                               const double* vals);

/* MgLevel.constrained, one byte per dof (reference linsolve.py:226). HOST. */
int alefsi_mg_set_constrained(alefsi_mg h, int32_t level, const uint8_t* mask);

/* VankaSmoother.factorize / patch_factorize on every level >= 1 and the
 * coarse-level factorisation of MgSolver.__init__ (reference
 * linsolve.py:120-134, 163-165, 236).  Coarsest level <= 4096 dofs;
 * ALEFSI_ERR_SINGULAR names the first singular patch (or the coarse
 * block).  Scratch is kept in the handle across re-factorisations. */
int alefsi_mg_factorize(alefsi_mg h);

/* z = one V-cycle applied to b (MgSolver.dot, reference linsolve.py:238-255). */
int alefsi_mg_apply(alefsi_mg h, const double* b, double* z, int32_t host_ptrs);

/* y = A x (b == NULL) or y = b - A x on one level (DEVICE). */
int alefsi_mg_spmv(alefsi_mg h, int32_t level, const double* x, const double* b, double* y);

/* Layout of a 2D (nc = 3) level's SpMV copy: sliced ELL with lanes_per_row
 * = 1, 2 or 4 lanes per block row (slices of 32 / lanes rows), or 0 for the
 * CSR half-warp kernel.  The default is chosen by level size at
 * set_pattern / set_matrix; this call re-lays a level out (tuning,
 * measurements).  No effect on other nc. */
int alefsi_mg_set_sell(alefsi_mg h, int32_t level, int32_t lanes_per_row);

/* Form of a level's Vanka apply kernel: -1 (default) column-split patches
 * (4 thread groups per patch, partials combined in fixed order) for launches
 * of fewer than 8,192 patches, one thread group per patch otherwise; 0 / 1
 * force the unsplit / split form (tuning, measurements; patches <= 108 dofs). */
int alefsi_mg_set_apply_split(alefsi_mg h, int32_t level, int32_t split);

/* x <- one damped additive Vanka sweep (VankaSmoother.sweep,
 * reference linsolve.py:167-178) (DEVICE). */
int alefsi_mg_vanka_sweep(alefsi_mg h, int32_t level, double* x, const double* b);

/* b_coarse = P^T r_fine with coarse constraints zeroed (MgSolver._restrict,
 * reference linsolve.py:260-264) (DEVICE). */
int alefsi_mg_restrict(alefsi_mg h, int32_t level, const double* r_fine, double* b_coarse);

/* x_fine += P x_coarse with fine constraints zeroed (MgSolver._prolong +
 * the update of linsolve.py:252, 266-270) (DEVICE). */
int alefsi_mg_prolong_add(alefsi_mg h, int32_t level, const double* x_coarse, double* x_fine);

/* x = A_0^{-1} b on the coarsest level (coarse_lu.solve, linsolve.py:246). */
int alefsi_mg_coarse_solve(alefsi_mg h, const double* b, double* x);

/* Copy the stored patch inverses of one group to host memory:
 * (n_patches, np, ld) column-major with ld = np rounded up to even. */
int alefsi_mg_get_inverses(alefsi_mg h, int32_t level, int32_t group, double* out);

/* info[0..7] = n_nodes, ndof, nnzb, nnz_pp, n_groups, Y size, inverse doubles, ld. */
int alefsi_mg_info(alefsi_mg h, int32_t level, int64_t* info);

/* Right-preconditioned, unrestarted GMRES with the V-cycle as
 * preconditioner (gmres, reference linsolve.py:41-115): classical
 * Gram-Schmidt with the conditional second pass, Givens rotations,
 * residuals[0..iterations] = the reference's stats.residuals (max_iter + 1
 * doubles).  max_iter must be in [1, 510].  Returns
 * ALEFSI_ERR_NOT_CONVERGED (x and residuals still written) when max_iter is
 * reached above tolerance. */
int alefsi_gmres(alefsi_mg h, const double* b, double* x, double rel_tol, double abs_tol,
                 int32_t max_iter, int32_t host_ptrs, double* residuals, int32_t* iterations,
                 int32_t* converged);
/* Pre-allocate the Krylov basis for max_iter iterations. */
int alefsi_gmres_workspace(alefsi_mg h, int32_t max_iter);
/* Number of device kernels this handle has enqueued (graph replays excluded). */
int alefsi_kernel_stats(alefsi_mg h, int64_t* launches);

/* Live per-kernel timing with CUDA events on the launch stream (disables the
 * graph path while on).  profile_read fills counts[14] and ms[14]: index
 * kind + 7 * finest with kind 0 spmv, 1 vanka_apply, 2 vanka_gather,
 * 3 restrict, 4 prolong, 5 coarse solve, 6 Krylov orthogonalisation. */
int alefsi_mg_profile(alefsi_mg h, int32_t on);
int alefsi_mg_profile_read(alefsi_mg h, int64_t* counts, double* ms, int32_t reset);

#ifdef __cplusplus
}
#endif

#endif /* ALEFSI_B200_H */
