// Device kernels of the MG-GMRES / Vanka path (sm_100a, FP64).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace alefsi {

// ---- operator: A = B (nc x nc blocks, cell pattern) + L (scalar pp extension)
struct DevMatrix {
  int nc = 0;
  int64_t n_nodes = 0, nnzb = 0, nnz_pp = 0;
  const int64_t* indptr = nullptr;
  const int32_t* indices = nullptr;
  const double* data = nullptr;
  const int64_t* pp_indptr = nullptr;
  const int32_t* pp_indices = nullptr;
  const double* pp_data = nullptr;
  // optional sliced-ELL copy used by the SpMV (nc == 3): slices of R
  // consecutive block rows, slice s holds its rows' k-th blocks in slot
  // off[s] + k, a slot = nc*nc element planes of R doubles (one per row)
  // (R = 32 / sell_lanes rows per slice; a row's slots are split
  // round-robin over its sell_lanes lanes)
  int64_t n_slices = 0;
  int sell_lanes = 0;
  const int64_t* sell_off = nullptr;    // n_slices + 1 (slot units)
  const int32_t* sell_col = nullptr;    // slots * R block columns
  const double* sell_val = nullptr;     // slots * nc*nc * R
  const int64_t* sell_poff = nullptr;   // pressure extension, same scheme (nullptr: none)
  const int32_t* sell_pcol = nullptr;
  const double* sell_pval = nullptr;
};

// refresh the sliced-ELL values from the CSR data: map[pos] = CSR block (or
// entry) index of slot position pos, -1 for padding (stored as zero)
void launch_sell_pack(int64_t n_pos, int R, int nc2, const int64_t* map, const double* data,
                      double* val, cudaStream_t s);

// y = A x (mode 0) or y = b - A x (mode 1)
void launch_spmv(const DevMatrix& A, const double* x, const double* b, double* y, int mode,
                 cudaStream_t s);

// ---- Vanka smoother
struct DevPatchGroup {
  int npn = 0;          // nodes per patch
  int np = 0;           // dofs per patch (npn * nc)
  int ld = 0;           // padded column length of the stored inverse (even)
  int64_t n_patches = 0;
  const int32_t* nodes = nullptr;   // (n_patches, npn)
  double* inv = nullptr;            // (n_patches, np, ld) column-major inverses
  int64_t y_offset = 0;             // start of this group's rows in Y
  double* work = nullptr;           // factorisation scratch, vanka_factorize_work doubles
  const int32_t* slots = nullptr;   // (n_patches, npn, npn) operator slots (vanka_uses_slots)
};

// (nc, dofs per patch) combinations with compiled Vanka kernels
bool vanka_supported(int nc, int np);
// patch sizes whose factorisation kernel reads a per-patch operator-slot table
// (launch_patch_slots, rebuilt when the sparsity pattern or the patches change)
bool vanka_uses_slots(int np);
void launch_patch_slots(const DevMatrix& A, const DevPatchGroup& g, int32_t* slots,
                        cudaStream_t s);
// factorisation scratch of a patch group in doubles (0: none needed)
int64_t vanka_factorize_work(int np, int64_t n_patches);
// gather A_i = R_i A R_i^T and invert (Gauss-Jordan, partial pivoting);
// singular patches set *status to 1 + patch index (first one wins)
void launch_vanka_factorize(const DevMatrix& A, const DevPatchGroup& g, int64_t* status,
                            cudaStream_t s);
// Y[p] = A_p^{-1} d[dofs_p] for every patch of the groups (consecutive groups
// of one patch size share a launch); split: -1 default (column-split kernel
// below 8,192 patches per launch), 0 never, 1 always; returns the number of
// launches
int launch_vanka_apply(const DevPatchGroup* groups, int n_groups, int nc, const double* d,
                       double* Y, int split, cudaStream_t s);
// x[dof] = (init_zero ? 0 : x[dof]) + omega * sum_{p ∋ dof} w[node] * Y[p, dof]
void launch_vanka_gather(int64_t n_nodes, int nc, const int64_t* gptr, const int64_t* goff,
                         const double* weight, const double* Y, double* x, double omega,
                         int init_zero, cudaStream_t s);

// ---- grid transfer (scalar CSR applied per component)
void launch_restrict(int64_t n_coarse, int nc, const int64_t* ptr, const int32_t* idx,
                     const double* val, const double* r_fine, const uint8_t* constrained_coarse,
                     double* b_coarse, cudaStream_t s);
void launch_prolong_add(int64_t n_fine, int nc, const int64_t* ptr, const int32_t* idx,
                        const double* val, const double* x_coarse,
                        const uint8_t* constrained_fine, double* x_fine, cudaStream_t s);

// ---- coarse level: dense inverse and apply
// work: dense_inverse_work(n) doubles
int dense_inverse(double* M, int64_t n, double* work, int64_t* status, cudaStream_t s);
inline int64_t dense_inverse_work(int64_t n) { return 2 * n + 2 + 64 * n; }
// y = M x, M n x n stored with row stride ld (a multiple of 4)
void launch_dense_matvec(int64_t n, const double* M, int64_t ld, const double* x, double* y,
                         cudaStream_t s);
// P[i, j] = M[i, j] (row stride n -> ld), padding zero
void launch_pad_rows(int64_t n, const double* M, int64_t ld, double* P, cudaStream_t s);

// ---- GMRES (reference linsolve.py:41-115) with its state on the device, so
// that a whole solve can run as one CUDA graph (conditional while node).
// Every launcher returns the number of kernels it enqueued.
struct GmresCtl {
  int k;            // current Arnoldi step (0-based)
  int its;          // completed iterations
  int done;         // stop (converged or max_iter)
  int converged;
  int flag;         // second Gram-Schmidt pass needed (Kahan test)
  int max_iter;
  int hstride;      // Hessenberg row length (workspace capacity)
  int pad;
  double beta, tol, rel_tol, abs_tol;
};
constexpr int kRedBlocks = 592;   // 4 x 148 SMs
// hcol[j] = v_j . w (j <= k), hcol[k+1] = w . w; deterministic two-stage sums;
// flag (optional): skip unless *flag != 0; max_nvec bounds k + 1
int launch_multi_dot(GmresCtl* ctl, int max_nvec, const double* V, int64_t ldv, const double* w,
                     int64_t n, double* partial, double* out, const int* flag, cudaStream_t s);
// w -= sum_{j<=k} h[j] v_j; out[0] = w . w (after)
int launch_multi_axpy(GmresCtl* ctl, const double* V, int64_t ldv, const double* h, double* w,
                      int64_t n, double* partial, double* out, const int* flag, cudaStream_t s);
int launch_arnoldi_finish(GmresCtl* ctl, double* hcol, double* h2, const double* na2, int stage,
                          cudaStream_t s);
// v_{k+1} = w / hcol[k+1] into V and into the V-cycle input buffer vin
int launch_scale_copy_slot(const GmresCtl* ctl, const double* w, double* V, int64_t ldv,
                           const double* hcol, double* vin, int64_t n, cudaStream_t s);
// beta, tol, early exit, v_0 = b / beta (into V and vin); sets the condition
int launch_gmres_init(GmresCtl* ctl, const double* b, int64_t n, double* partial, double* scal,
                      double* res, double* g, double* v0, double* vin,
                      cudaGraphConditionalHandle cond, int use_cond, cudaStream_t s);
// Givens update of column k, residual estimate, stopping test; k += 1
int launch_givens(GmresCtl* ctl, const double* hcol, double* H, double* cs, double* sn, double* g,
                  double* res, cudaGraphConditionalHandle cond, int use_cond, cudaStream_t s);
// out = V triu(H)^{-1} g over the completed iterations
int launch_gmres_solution(const GmresCtl* ctl, const double* H, const double* g, double* y,
                          const double* V, int64_t ldv, double* out, int64_t n, cudaStream_t s);

}  // namespace alefsi
