// Device assembly of the condensed Jacobian (see assembly_kernels.cu).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace alefsi {

struct AsmArgs {
  const int32_t* cell_nodes = nullptr;   // (n_cells, 3^d)
  const double* coords = nullptr;        // (n_nodes, d)
  const double* U = nullptr;             // (n_nodes, 1 + 2d) current state
  const double* Up = nullptr;            // previous time step
  const int32_t* cell_slots = nullptr;   // (n_cells, 3^d, 3^d) block slot of (row node, column node)
  double* data = nullptr;                // (nnzb, d+1, d+1) output, accumulated
  int64_t* status = nullptr;             // 1 + first inverted cell
  double rho_f = 0, mu_f = 0, rho_s = 0, mu_s = 0, lam_s = 0, k = 0, theta = 0;
};

struct ResArgs {
  const int32_t* cell_nodes = nullptr;
  const double* coords = nullptr;
  const double* U = nullptr;
  const double* Up = nullptr;
  int64_t* status = nullptr;
  double rho_f = 0, mu_f = 0, rho_s = 0, mu_s = 0, lam_s = 0, k = 0, theta = 0;
  double f[3] = {0, 0, 0};
  int ext_model = 0;          // 0 harmonic, 1 linear elasticity
  double ext_mu = 1, ext_lam = 0;
  int ext_volume_scaling = 0;
};

struct OutflowArgs {
  int64_t n_facets = 0;
  int nq = 0;                            // facet quadrature points
  const int32_t* conn = nullptr;         // (n_facets, 3^d) owner-cell nodes
  const int64_t* cell_of_facet = nullptr;
  const double* N = nullptr;             // (n_facets, nq, 3^d)
  const double* G = nullptr;             // (n_facets, nq, 3^d, d)
  const double* dS = nullptr;            // (n_facets, nq)
  const double* normal = nullptr;        // (n_facets, nq, d)
  const double* U = nullptr;             // (n_nodes, 1 + 2d) state
  int64_t* status = nullptr;
  double mu_f = 0, k = 0, theta = 0;
};

// do-nothing outflow blocks of the Jacobian: per-facet local blocks into
// `local`, then a fixed-order reduction per unique matrix slot into data
void launch_outflow(const OutflowArgs& a, int dim, int64_t n_unique, const int64_t* slots,
                    const int64_t* uptr, const int64_t* contrib, double* local, double* data,
                    cudaStream_t s);

// do-nothing outflow term of the residual: per-facet rows into `local`
// (n_facets, 3^d, d), reduced per node in fixed order into out[:, off:off+d]
void launch_outflow_residual(const OutflowArgs& a, int dim, double scale, int64_t n_unique,
                             const int64_t* nodes, const int64_t* uptr, const int64_t* contrib,
                             double* local, double* out, int no, int off, cudaStream_t s);
// out[:, 0] += k * (L @ U[:, 0]) for the scalar LPS operator L (CSR)
void launch_lps_residual(int64_t n, const int64_t* indptr, const int32_t* indices,
                         const double* vals, const double* U, int nf, double k, double* out,
                         int no, cudaStream_t s);

// cell contributions of the theta residual (kind 0 fluid, 1 solid) or of the
// explicit previous-state forces (kind 2 fluid, 3 solid), added into out
void launch_residual_cells(const ResArgs& a, int dim, int kind, const int32_t* cells,
                           int64_t n_cells, double* out, cudaStream_t s);

// Q2 tables at the Gauss points: N (nq, nb), dN (nq, nb, dim), weights (nq)
// 0 ok; 1 bad shape (nq != nb or dim not 2/3); 2 tables differ from those
// already loaded for this dim; 3 CUDA error
int set_assembly_tables(const double* N, const double* dN, const double* w, int nq, int nb,
                        int dim);
// kind 0: fluid cells, 1: solid cells; cells of one colour (no shared nodes)
void launch_assemble_cells(const AsmArgs& a, int dim, int kind, const int32_t* cells,
                           int64_t n_cells, cudaStream_t s);
void launch_add_blocks(double* data, int bs, int64_t n, const int64_t* slots, const double* vals,
                       cudaStream_t s);
void launch_lps(double* data, int nc, double* pp, int64_t n, const int64_t* cell_slot,
                const int64_t* pp_slot, const double* vals, double k, cudaStream_t s);
void launch_dirichlet(double* data, int nc, double* pp, int64_t n_nodes, const int64_t* indptr,
                      const int32_t* indices, const int64_t* pp_indptr, const uint8_t* mask,
                      cudaStream_t s);

}  // namespace alefsi
