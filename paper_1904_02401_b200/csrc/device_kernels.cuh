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
};

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
};

// (nc, dofs per patch) combinations with compiled Vanka kernels
bool vanka_supported(int nc, int np);
// factorisation scratch of a patch group in doubles (0: none needed)
int64_t vanka_factorize_work(int np, int64_t n_patches);
// gather A_i = R_i A R_i^T and invert (Gauss-Jordan, partial pivoting);
// singular patches set *status to 1 + patch index (first one wins)
void launch_vanka_factorize(const DevMatrix& A, const DevPatchGroup& g, int64_t* status,
                            cudaStream_t s);
// Y[p] = A_p^{-1} d[dofs_p] for every patch of the groups (consecutive groups
// of one patch size share a launch); returns the number of launches
int launch_vanka_apply(const DevPatchGroup* groups, int n_groups, int nc, const double* d,
                       double* Y, cudaStream_t s);
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
void launch_dense_matvec(int64_t n, const double* M, const double* x, double* y,
                         cudaStream_t s);

// ---- Krylov vector kernels (deterministic fixed-order reductions)
constexpr int kRedBlocks = 592;   // 4 x 148 SMs
// out[j] = sum_i V[j*ldv + i] * w[i] for j < nvec; out[nvec] = sum_i w[i]^2
// flag (optional): skip unless *flag != 0
void launch_multi_dot(int nvec, const double* V, int64_t ldv, const double* w, int64_t n,
                      double* partial, double* out, const int* flag, cudaStream_t s);
// w[i] -= sum_j h[j] V[j*ldv + i]; out[0] = sum_i w[i]^2 (after update)
void launch_multi_axpy(int nvec, const double* V, int64_t ldv, const double* h, double* w,
                       int64_t n, double* partial, double* out, const int* flag,
                       cudaStream_t s);
// Arnoldi bookkeeping on device (see mg.cu)
void launch_arnoldi_finish(int k, double* hcol, double* h2, const double* nb2, double* na2,
                           int* flag, int stage, cudaStream_t s);
void launch_scale_copy(const double* w, double* v, const double* hkk1, int64_t n,
                       cudaStream_t s);
void launch_scale(const double* x, double* y, double alpha, int64_t n, cudaStream_t s);
// y = sum_j c[j] V[j*ldv + i]  (c on device)
void launch_combine(int nvec, const double* V, int64_t ldv, const double* c, double* y,
                    int64_t n, cudaStream_t s);
void launch_sumsq(const double* x, int64_t n, double* partial, double* out, cudaStream_t s);

}  // namespace alefsi
