// Device-resident multigrid hierarchy, V-cycle and right-preconditioned
// GMRES behind the C ABI of include/alefsi_b200.h.
//
// Mirrors the reference solver objects (reference pkg/src/alefsi/linsolve.py):
//   gmres                 linsolve.py:41-115   -> alefsi_gmres
//   patch_factorize       linsolve.py:120-134  -> alefsi_mg_factorize
//   VankaSmoother.sweep   linsolve.py:167-178  -> alefsi_mg_vanka_sweep
//   MgSolver._cycle       linsolve.py:243-255  -> alefsi_mg_apply
//   MgSolver._restrict    linsolve.py:260-264  -> alefsi_mg_restrict
//   MgSolver._prolong     linsolve.py:266-270  -> alefsi_mg_prolong_add
//   coarse_lu.solve       linsolve.py:236,246  -> alefsi_mg_coarse_solve
// The per-level operators, patch inverses, transfer operators and Krylov
// basis live in HBM for the lifetime of the handle; the host only runs the
// Givens rotations of the (max_iter+1) x max_iter Hessenberg matrix.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "alefsi_common.h"
#include "alefsi_b200.h"
#include "assembly_kernels.cuh"
#include "device_kernels.cuh"

namespace alefsi {
namespace {

// dense (n*nc)^2 copy of a split operator (coarse level), warp per node row
__global__ void split_to_dense_kernel(DevMatrix A, double* M) {
  const int lane = threadIdx.x & 31;
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (row >= A.n_nodes) return;
  const int nc = A.nc;
  const int64_t n = A.n_nodes * nc;
  for (int64_t s = A.indptr[row] + lane; s < A.indptr[row + 1]; s += 32) {
    const int64_t col = A.indices[s];
    for (int i = 0; i < nc; ++i)
      for (int j = 0; j < nc; ++j)
        M[(row * nc + i) * n + col * nc + j] += A.data[s * nc * nc + i * nc + j];
  }
  if (A.pp_indptr != nullptr)
    for (int64_t s = A.pp_indptr[row] + lane; s < A.pp_indptr[row + 1]; s += 32)
      M[(row * nc) * n + (int64_t)A.pp_indices[s] * nc] += A.pp_data[s];
}

void launch_split_to_dense(const DevMatrix& A, double* M, cudaStream_t s) {
  split_to_dense_kernel<<<(unsigned)((A.n_nodes * 32 + 255) / 256), 256, 0, s>>>(A, M);
}

#define CK(expr)                                                                  \
  do {                                                                            \
    cudaError_t _e = (expr);                                                      \
    if (_e != cudaSuccess)                                                        \
      return fail(ALEFSI_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) {
    o.p = nullptr;
    o.n = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      reset();
      p = o.p;
      n = o.n;
      o.p = nullptr;
      o.n = 0;
    }
    return *this;
  }
  ~DevBuf() { reset(); }
  void reset() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  cudaError_t alloc(size_t count) {
    reset();
    n = count;
    if (count == 0) return cudaSuccess;
    return cudaMalloc(&p, count * sizeof(T));
  }
  // keep the allocation when the size is unchanged (re-factorisation)
  cudaError_t ensure(size_t count) {
    if (p != nullptr && n == count) return cudaSuccess;
    return alloc(count);
  }
  // stream-ordered copy into a buffer kept across calls of the same size
  // (no cudaFree, which would synchronise the device, per call)
  cudaError_t upload(const T* host, size_t count, cudaStream_t s) {
    cudaError_t e = ensure(count);
    if (e != cudaSuccess || count == 0) return e;
    return cudaMemcpyAsync(p, host, count * sizeof(T), cudaMemcpyHostToDevice, s);
  }
};

struct Group {
  int npn = 0, np = 0, ld = 0;
  int64_t n_patches = 0, y_offset = 0;
  DevBuf<int32_t> nodes;
  DevBuf<double> inv;
  DevBuf<double> fwork;   // factorisation scratch (500 x 500 macro patches), kept
  DevBuf<int32_t> slots;  // operator slots of the patches' node pairs (75 / 108)
  int64_t slots_epoch = -1;   // pattern epoch the table was built for
};

struct Level {
  int64_t n_nodes = 0;
  int nc = 0;
  bool has_matrix = false;
  int64_t pattern_epoch = 0;   // bumped whenever indptr / indices are (re)loaded
  int64_t nnzb = 0, nnz_pp = 0;
  DevBuf<int64_t> indptr, pp_indptr;
  DevBuf<int32_t> indices, pp_indices;
  DevBuf<double> data, pp_data;
  std::vector<double> host_dense;   // level 0 only: dense copy for the coarse inverse
  std::vector<std::unique_ptr<Group>> groups;
  DevBuf<double> Y;
  DevBuf<int64_t> gptr, goff;
  DevBuf<double> weight;
  bool has_P = false;
  int64_t n_coarse = 0;
  DevBuf<int64_t> P_ptr, R_ptr;
  DevBuf<int32_t> P_idx, R_idx;
  DevBuf<double> P_val, R_val;
  DevBuf<uint8_t> constrained;
  DevBuf<double> x, b, d;
  // device assembly of the condensed Jacobian (assembly_kernels.cu)
  bool has_asm = false;
  int dim = 0;
  DevBuf<int32_t> asm_cell_nodes, asm_group_cells;
  DevBuf<int32_t> asm_cell_slots;    // (n_cells, nb, nb) block slots of the cells' node pairs
  int64_t asm_n_cells = 0, asm_slots_epoch = -1;
  DevBuf<double> asm_coords, asm_U, asm_Up, res_out, asm_extra_vals;
  DevBuf<int64_t> asm_extra_slots;
  // do-nothing outflow facets assembled on the device
  int64_t of_nf = 0, of_nu = 0;
  int of_nq = 0;
  DevBuf<int32_t> of_conn;
  DevBuf<int64_t> of_cells, of_slots, of_uptr, of_contrib;
  DevBuf<double> of_N, of_G, of_dS, of_n, of_local;
  // residual tail on the device: outflow rows reduced per node, LPS operator
  bool rt_ready = false;
  int64_t rt_nodes_n = 0;
  DevBuf<int64_t> rt_nodes, rt_uptr, rt_contrib, lps_indptr;
  DevBuf<int32_t> lps_indices;
  DevBuf<double> lps_vals, rt_local;
  std::vector<int64_t> asm_group_ptr;
  std::vector<int> asm_group_kind;
  int64_t n_lps = 0;
  DevBuf<int64_t> lps_cell, lps_pp;
  DevBuf<double> lps_val;
  DevBuf<uint8_t> dir_mask;

  // sliced-ELL copy of the operator for the SpMV (nc == 3), see DevMatrix
  int64_t n_slices = 0, sell_slots = 0, sell_pslots = 0;
  int sell_lanes = 0;     // lanes per row (slice height 32 / lanes); 0: none
  int apply_split = -1;   // Vanka apply form: -1 by patch count, 0 / 1 forced
  bool sell_dirty = false;
  DevBuf<int64_t> sell_off, sell_poff, sell_map, sell_pmap;
  DevBuf<int32_t> sell_col, sell_pcol;
  DevBuf<double> sell_val, sell_pval;

  int64_t ndof() const { return n_nodes * nc; }
  DevMatrix mat() const {
    DevMatrix m;
    m.nc = nc;
    m.n_nodes = n_nodes;
    m.nnzb = nnzb;
    m.nnz_pp = nnz_pp;
    m.indptr = indptr.p;
    m.indices = indices.p;
    m.data = data.p;
    m.pp_indptr = nnz_pp > 0 ? pp_indptr.p : nullptr;
    m.pp_indices = pp_indices.p;
    m.pp_data = pp_data.p;
    if (n_slices > 0) {
      m.n_slices = n_slices;
      m.sell_lanes = sell_lanes;
      m.sell_off = sell_off.p;
      m.sell_col = sell_col.p;
      m.sell_val = sell_val.p;
      if (sell_pslots > 0) {
        m.sell_poff = sell_poff.p;
        m.sell_pcol = sell_pcol.p;
        m.sell_pval = sell_pval.p;
      }
    }
    return m;
  }
};

// Lanes per block row of the sliced-ELL SpMV by level size (0: the
// half-warp CSR kernel).  Measured per level of configs 0 and 1
// (scripts/spmv_layout.py, profiles/r2f_spmv_layout.log): 1,051,137 nodes
// lanes 1: 247 us (CSR 369); 263,425 nodes lanes 2: 61 us (lanes 1: 107,
// CSR 87); 66,177 nodes and below the CSR kernel is fastest (25 us vs 26).
int default_sell_lanes(int nc, int64_t n_nodes) {
  if (nc != 3) return 0;
  if (n_nodes >= (int64_t)1 << 20) return 1;
  if (n_nodes >= (int64_t)1 << 17) return 2;
  return 0;
}

// Sliced-ELL index of a CSR pattern: slices of R = 32 / lanes consecutive
// rows, no row permutation (the Q2 node numbering keeps the rows of a slice
// at nearly equal length — config 1 finest level: 0.25 % block padding).
// pos = slot * R + row-in-slice.
void sell_index(int64_t n, int R, const int64_t* ptr, const int32_t* idx, std::vector<int64_t>& off,
                std::vector<int32_t>& col, std::vector<int64_t>& map) {
  const int64_t ns = (n + R - 1) / R;
  off.assign(ns + 1, 0);
  for (int64_t sl = 0; sl < ns; ++sl) {
    int64_t w = 0;
    for (int64_t r = sl * R; r < std::min(n, sl * R + R); ++r) w = std::max(w, ptr[r + 1] - ptr[r]);
    off[sl + 1] = off[sl] + w;
  }
  col.assign((size_t)off[ns] * R, 0);
  map.assign((size_t)off[ns] * R, -1);
  for (int64_t sl = 0; sl < ns; ++sl)
    for (int q = 0; q < R; ++q) {
      const int64_t r = sl * R + q;
      const int64_t len = r < n ? ptr[r + 1] - ptr[r] : 0;
      for (int64_t k = 0; k < off[sl + 1] - off[sl]; ++k) {
        const size_t pos = (size_t)(off[sl] + k) * R + q;
        // padding: zero value on a valid column (the row itself, else 0)
        col[pos] = k < len ? idx[ptr[r] + k] : (int32_t)(r < n ? r : 0);
        map[pos] = k < len ? ptr[r] + k : -1;
      }
    }
}

int build_sell(Level& L, int lanes, const int64_t* indptr, const int32_t* indices,
               const int64_t* pp_indptr, const int32_t* pp_indices, cudaStream_t s) {
  L.n_slices = 0;
  L.sell_lanes = 0;
  L.sell_slots = L.sell_pslots = 0;
  if (L.nc != 3 || L.n_nodes == 0 || lanes == 0) return ALEFSI_OK;
  if (lanes != 1 && lanes != 2 && lanes != 4)
    return fail(ALEFSI_ERR_ARG, "sliced ELL: 1, 2 or 4 lanes per row");
  const int R = 32 / lanes;
  std::vector<int64_t> off, map;
  std::vector<int32_t> col;
  sell_index(L.n_nodes, R, indptr, indices, off, col, map);
  const int64_t ns = (int64_t)off.size() - 1;
  CK(L.sell_off.upload(off.data(), off.size(), s));
  CK(L.sell_col.upload(col.data(), col.size(), s));
  CK(L.sell_map.upload(map.data(), map.size(), s));
  CK(L.sell_val.ensure((size_t)off[ns] * R * 9));
  L.sell_slots = off[ns];
  if (L.nnz_pp > 0) {
    std::vector<int64_t> poff, pmap;
    std::vector<int32_t> pcol;
    sell_index(L.n_nodes, R, pp_indptr, pp_indices, poff, pcol, pmap);
    CK(L.sell_poff.upload(poff.data(), poff.size(), s));
    CK(L.sell_pcol.upload(pcol.data(), pcol.size(), s));
    CK(L.sell_pmap.upload(pmap.data(), pmap.size(), s));
    CK(L.sell_pval.ensure((size_t)poff[ns] * R));
    L.sell_pslots = poff[ns];
  }
  CK(cudaStreamSynchronize(s));     // host index vectors go out of scope
  L.n_slices = ns;
  L.sell_lanes = lanes;
  L.sell_dirty = true;
  return ALEFSI_OK;
}

// refresh the sliced-ELL values after the CSR data changed
void refresh_sell(Level& L, cudaStream_t s) {
  if (L.n_slices == 0 || !L.sell_dirty) return;
  const int R = 32 / L.sell_lanes;
  launch_sell_pack(L.sell_slots * R, R, 9, L.sell_map.p, L.data.p, L.sell_val.p, s);
  if (L.sell_pslots > 0)
    launch_sell_pack(L.sell_pslots * R, R, 1, L.sell_pmap.p, L.pp_data.p, L.sell_pval.p, s);
  L.sell_dirty = false;
}

}  // namespace

struct MgHandle {
  int n_levels = 0, nc = 0, nu_pre = 2, nu_post = 2;
  double omega = 0.8;
  std::vector<Level> lv;
  DevBuf<double> coarse_inv, coarse_work;
  // the inverse with rows padded to a multiple of 4 doubles for the
  // 32-byte loads of the coarse matvec
  DevBuf<double> coarse_pad;
  int64_t coarse_ld = 0;
  DevBuf<int64_t> status, coarse_status;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  // the coarse inverse is computed on a side stream, concurrently with the
  // patch factorisations of the finer levels
  cudaStream_t side_stream = nullptr;
  cudaEvent_t side_in = nullptr, side_out = nullptr;
  bool factorized = false;
  // the coarse inverse of the freshly assembled level 0 is already running
  // on the side stream (started by alefsi_mg_asm_momentum(level 0), so that
  // it overlaps the assembly of the finer levels)
  bool coarse_inflight = false;
  // graph-captured V-cycle (fixed in/out buffers)
  bool use_graph = false;
  bool graph_valid = false;
  cudaGraphExec_t graph_exec = nullptr;
  cudaStream_t cap_stream = nullptr;
  cudaEvent_t cap_in = nullptr, cap_out = nullptr;
  int64_t graph_kernels = 0;
  DevBuf<double> g_in, g_out;
  // GMRES workspace
  int v_cap = 0;
  DevBuf<double> V, w, xb, bb, vin, vout, partial, tmp, tmp2, scal;
  // device-resident GMRES state: control block, Hessenberg (v_cap x
  // v_cap-1), rotations, g, residual history, back-substitution result
  DevBuf<GmresCtl> ctl;
  DevBuf<double> Hd, csd, snd, gd, resd, yd;
  GmresCtl* ctl_host = nullptr;     // pinned
  // one CUDA graph per solve: init -> while (Arnoldi step) -> solution
  bool solve_valid = false;
  cudaGraphExec_t solve_exec = nullptr;
  int64_t n_init = 0, n_body = 0, n_fin = 0;
  double* pinned = nullptr;
  int64_t kernel_launches = 0;

  // Optional live per-kernel timing with CUDA events on the launch stream.
  // kind: 0 spmv, 1 vanka_apply, 2 vanka_gather, 3 restrict, 4 prolong,
  //       5 coarse, 6 krylov; slot = kind + kKinds * (level is finest).
  static constexpr int kKinds = 7;
  bool prof_on = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  std::vector<int> ev_slot;
  int64_t prof_count[2 * kKinds] = {0};
  double prof_ms[2 * kKinds] = {0};

  ~MgHandle() {
    if (graph_exec) cudaGraphExecDestroy(graph_exec);
    if (solve_exec) cudaGraphExecDestroy(solve_exec);
    if (ctl_host) cudaFreeHost(ctl_host);
    if (cap_stream) cudaStreamDestroy(cap_stream);
    if (cap_in) cudaEventDestroy(cap_in);
    if (cap_out) cudaEventDestroy(cap_out);
    if (pinned) cudaFreeHost(pinned);
    for (auto e : ev_pool) cudaEventDestroy(e);
    if (side_stream) cudaStreamDestroy(side_stream);
    if (side_in) cudaEventDestroy(side_in);
    if (side_out) cudaEventDestroy(side_out);
    if (own_stream && stream) cudaStreamDestroy(stream);
  }

  Level& fine() { return lv.back(); }

  // returns the event-pair index or -1
  int prof_begin(int kind, int level) {
    if (!prof_on) return -1;
    if (ev_used + 2 > ev_pool.size()) {
      for (int i = 0; i < 256; ++i) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return -1;
        ev_pool.push_back(e);
      }
      ev_slot.resize(ev_pool.size() / 2);
    }
    const int pair = (int)(ev_used / 2);
    cudaEventRecord(ev_pool[ev_used], stream);
    ev_used += 2;
    ev_slot[pair] = kind + kKinds * (level == n_levels - 1 ? 1 : 0);
    return pair;
  }
  void prof_end(int pair) {
    if (pair >= 0) cudaEventRecord(ev_pool[2 * pair + 1], stream);
  }
  // fold recorded pairs into the totals (stream must be idle)
  void prof_collect() {
    for (size_t p = 0; p < ev_used / 2; ++p) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, ev_pool[2 * p], ev_pool[2 * p + 1]) == cudaSuccess) {
        prof_ms[ev_slot[p]] += ms;
        prof_count[ev_slot[p]] += 1;
      }
    }
    ev_used = 0;
  }

  // ---------------------------------------------------------------- V-cycle
  void sweep(Level& L, int l, const double* b, double* x, bool zero) {
    const double* d = b;
    if (!zero) {
      int pr = prof_begin(0, l);
      launch_spmv(L.mat(), x, b, L.d.p, 1, stream);
      prof_end(pr);
      ++kernel_launches;
      d = L.d.p;
    }
    {
      std::vector<DevPatchGroup> dg(L.groups.size());
      const int ng = (int)dg.size();
      for (int i = 0; i < ng; ++i) {
        const auto& g = L.groups[i];
        dg[i].npn = g->npn;
        dg[i].np = g->np;
        dg[i].ld = g->ld;
        dg[i].n_patches = g->n_patches;
        dg[i].nodes = g->nodes.p;
        dg[i].inv = g->inv.p;
        dg[i].y_offset = g->y_offset;
      }
      int pr = prof_begin(1, l);
      kernel_launches += launch_vanka_apply(dg.data(), ng, L.nc, d, L.Y.p, L.apply_split, stream);
      prof_end(pr);
    }
    int pr = prof_begin(2, l);
    launch_vanka_gather(L.n_nodes, L.nc, L.gptr.p, L.goff.p, L.weight.p, L.Y.p, x, omega,
                        zero ? 1 : 0, stream);
    prof_end(pr);
    ++kernel_launches;
  }

  void cycle(int l, const double* b, double* x) {
    Level& L = lv[l];
    if (l == 0) {
      int pr = prof_begin(5, l);
      launch_dense_matvec(L.ndof(), coarse_pad.p, coarse_ld, b, x, stream);
      prof_end(pr);
      ++kernel_launches;
      return;
    }
    bool zero = true;
    for (int s = 0; s < nu_pre; ++s) {
      sweep(L, l, b, x, zero);
      zero = false;
    }
    if (zero) cudaMemsetAsync(x, 0, sizeof(double) * L.ndof(), stream);
    int pr = prof_begin(0, l);
    launch_spmv(L.mat(), x, b, L.d.p, 1, stream);
    prof_end(pr);
    Level& C = lv[l - 1];
    pr = prof_begin(3, l);
    launch_restrict(C.n_nodes, C.nc, L.R_ptr.p, L.R_idx.p, L.R_val.p, L.d.p, C.constrained.p,
                    C.b.p, stream);
    prof_end(pr);
    kernel_launches += 2;
    cycle(l - 1, C.b.p, C.x.p);
    pr = prof_begin(4, l);
    launch_prolong_add(L.n_nodes, L.nc, L.P_ptr.p, L.P_idx.p, L.P_val.p, C.x.p,
                       L.constrained.p, x, stream);
    prof_end(pr);
    ++kernel_launches;
    for (int s = 0; s < nu_post; ++s) sweep(L, l, b, x, false);
  }

  int apply(const double* b, double* x) {
    if (!factorized) return fail(ALEFSI_ERR_STATE, "mg_apply before mg_factorize");
    const int64_t n = fine().ndof();
    if (!use_graph || prof_on) {
      cycle(n_levels - 1, b, x);
      CK(cudaGetLastError());
      return ALEFSI_OK;
    }
    // The V-cycle is captured and replayed on a private stream (the caller's
    // stream may be the legacy default stream, which cannot be captured),
    // ordered against the caller's stream with events.
    if (!cap_stream) {
      CK(cudaStreamCreateWithFlags(&cap_stream, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&cap_in, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&cap_out, cudaEventDisableTiming));
    }
    if (!graph_valid) {
      CK(g_in.alloc(n));
      CK(g_out.alloc(n));
      if (graph_exec) {
        cudaGraphExecDestroy(graph_exec);
        graph_exec = nullptr;
      }
      cudaGraph_t graph;
      cudaStream_t user = stream;
      stream = cap_stream;
      const int64_t before = kernel_launches;
      cudaError_t e = cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal);
      if (e == cudaSuccess) {
        cycle(n_levels - 1, g_in.p, g_out.p);
        e = cudaStreamEndCapture(stream, &graph);
      }
      stream = user;
      CK(e);
      graph_kernels = kernel_launches - before;
      kernel_launches = before;
      CK(cudaGraphInstantiate(&graph_exec, graph, 0));
      cudaGraphDestroy(graph);
      graph_valid = true;
    }
    CK(cudaMemcpyAsync(g_in.p, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, stream));
    CK(cudaEventRecord(cap_in, stream));
    CK(cudaStreamWaitEvent(cap_stream, cap_in, 0));
    CK(cudaGraphLaunch(graph_exec, cap_stream));
    CK(cudaEventRecord(cap_out, cap_stream));
    CK(cudaStreamWaitEvent(stream, cap_out, 0));
    CK(cudaMemcpyAsync(x, g_out.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, stream));
    kernel_launches += graph_kernels;
    return ALEFSI_OK;
  }

  // ------------------------------------------------------------ factorize
  // buffers the captured V-cycle graph reads; a re-factorisation that keeps
  // them (same sizes: ensure() does not reallocate) keeps the graph valid
  std::vector<const void*> graph_buffers() const {
    std::vector<const void*> v{coarse_inv.p, coarse_pad.p};
    for (const auto& L : lv) {
      v.push_back(L.x.p);
      v.push_back(L.b.p);
      v.push_back(L.d.p);
      for (const auto& g : L.groups) v.push_back(g->inv.p);
    }
    return v;
  }

  // coarse level: dense inverse, enqueued on the side stream after the work
  // already on the main stream (the operator's assembly)
  int start_coarse_inverse() {
    Level& C = lv[0];
    if (!C.has_matrix) return fail(ALEFSI_ERR_STATE, "coarse matrix missing");
    if (!side_stream) {
      // high priority: the serial chain of panel steps gets an SM as soon as
      // one frees up instead of queueing behind the patch factorisations
      int lo = 0, hi = 0;
      CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      CK(cudaStreamCreateWithPriority(&side_stream, cudaStreamNonBlocking, hi));
      CK(cudaEventCreateWithFlags(&side_in, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&side_out, cudaEventDisableTiming));
    }
    if (!coarse_status.p) CK(coarse_status.alloc(1));
    CK(cudaEventRecord(side_in, stream));
    CK(cudaStreamWaitEvent(side_stream, side_in, 0));
    const int64_t n0 = C.ndof();
    if (!C.host_dense.empty()) {
      CK(coarse_inv.upload(C.host_dense.data(), (size_t)n0 * n0, side_stream));
    } else {   // device-assembled coarse operator
      CK(coarse_inv.ensure((size_t)n0 * n0));
      CK(cudaMemsetAsync(coarse_inv.p, 0, sizeof(double) * n0 * n0, side_stream));
      launch_split_to_dense(C.mat(), coarse_inv.p, side_stream);
    }
    CK(coarse_work.ensure((size_t)dense_inverse_work(n0)));
    if (dense_inverse(coarse_inv.p, n0, coarse_work.p, coarse_status.p, side_stream) != 0)
      return fail(ALEFSI_ERR_ARG, "coarse level too large for the dense inverse (" +
                                      std::to_string(n0) + " > 4096 dofs)");
    coarse_ld = (n0 + 3) / 4 * 4;
    CK(coarse_pad.ensure((size_t)n0 * coarse_ld));
    launch_pad_rows(n0, coarse_inv.p, coarse_ld, coarse_pad.p, side_stream);
    CK(cudaGetLastError());
    CK(cudaEventRecord(side_out, side_stream));
    return ALEFSI_OK;
  }

  // level 0's operator is about to change: let an early-started inverse drain
  void cancel_coarse_inflight() {
    if (coarse_inflight && side_stream) cudaStreamSynchronize(side_stream);
    coarse_inflight = false;
  }

  int finish_coarse_inverse() {
    CK(cudaStreamWaitEvent(stream, side_out, 0));
    int64_t st = 0;
    CK(cudaMemcpyAsync(&st, coarse_status.p, sizeof(int64_t), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    if (st != 0) return fail(ALEFSI_ERR_SINGULAR, "singular coarse-level matrix");
    return ALEFSI_OK;
  }

  int factorize() {
    const std::vector<const void*> before = graph_buffers();
    for (auto& L : lv) refresh_sell(L, stream);
    int rc = coarse_inflight ? ALEFSI_OK : start_coarse_inverse();
    coarse_inflight = false;
    if (rc) {
      if (side_stream) cudaStreamSynchronize(side_stream);
      return rc;
    }
    for (int l = 1; l < n_levels; ++l) {
      Level& L = lv[l];
      auto bail = [&](int code, const std::string& msg) {
        cudaStreamSynchronize(side_stream);
        return fail(code, msg);
      };
      if (!L.has_matrix) return bail(ALEFSI_ERR_STATE, "level matrix missing");
      if (!L.has_P) return bail(ALEFSI_ERR_STATE, "level prolongation missing");
      if (L.groups.empty()) return bail(ALEFSI_ERR_STATE, "level patches missing");
      if (!L.constrained.p || !lv[l - 1].constrained.p)
        return bail(ALEFSI_ERR_STATE, "constrained mask missing");
      CK(cudaMemsetAsync(status.p, 0, sizeof(int64_t), stream));
      int64_t off = 0;
      for (auto& g : L.groups) {
        CK(g->inv.ensure((size_t)g->n_patches * g->np * g->ld));
        const int64_t wn = vanka_factorize_work(g->np, g->n_patches);
        if (wn > 0) CK(g->fwork.ensure((size_t)wn));
        DevPatchGroup dg;
        dg.work = g->fwork.p;
        dg.npn = g->npn;
        dg.np = g->np;
        dg.ld = g->ld;
        dg.n_patches = g->n_patches;
        dg.nodes = g->nodes.p;
        dg.inv = g->inv.p;
        if (vanka_uses_slots(g->np)) {
          if (g->slots_epoch != L.pattern_epoch) {
            CK(g->slots.ensure((size_t)g->n_patches * g->npn * g->npn));
            launch_patch_slots(L.mat(), dg, g->slots.p, stream);
            g->slots_epoch = L.pattern_epoch;
          }
          dg.slots = g->slots.p;
        }
        launch_vanka_factorize(L.mat(), dg, status.p, stream);
        CK(cudaGetLastError());
        int64_t st = 0;
        CK(cudaMemcpyAsync(&st, status.p, sizeof(int64_t), cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        if (st != 0)
          return bail(ALEFSI_ERR_SINGULAR,
                      "singular Vanka patch block: level " + std::to_string(l) + " patch " +
                          std::to_string(off + st - 1));
        off += g->n_patches;
      }
    }
    rc = finish_coarse_inverse();
    if (rc) return rc;
    for (int l = 0; l < n_levels; ++l) {
      Level& L = lv[l];
      CK(L.x.ensure(L.ndof()));
      CK(L.b.ensure(L.ndof()));
      CK(L.d.ensure(L.ndof()));
    }
    factorized = true;
    if (graph_buffers() != before) graph_valid = solve_valid = false;
    return ALEFSI_OK;
  }

  // ----------------------------------------------------------------- GMRES
  int ensure_workspace(int max_iter) {
    const int64_t n = fine().ndof();
    if (v_cap < max_iter + 1) {
      CK(V.alloc((size_t)(max_iter + 1) * n));
      v_cap = max_iter + 1;
      const int m = v_cap - 1;
      CK(Hd.alloc((size_t)(m + 1) * m));
      CK(csd.alloc(m));
      CK(snd.alloc(m));
      CK(gd.alloc(m + 1));
      CK(resd.alloc(m + 1));
      CK(yd.alloc(m + 1));
      CK(tmp.alloc(m + 2));
      CK(tmp2.alloc(m + 2));
      CK(partial.alloc((size_t)kRedBlocks * (m + 2)));
      solve_valid = false;
    }
    if (w.n != (size_t)n) {
      CK(w.alloc(n));
      CK(xb.alloc(n));
      CK(bb.alloc(n));
      CK(vin.alloc(n));
      CK(vout.alloc(n));
      solve_valid = false;
    }
    if (!scal.p) CK(scal.alloc(4));
    if (!ctl.p) CK(ctl.alloc(1));
    if (!ctl_host) CK(cudaMallocHost(&ctl_host, sizeof(GmresCtl)));
    if (!pinned) CK(cudaMallocHost(&pinned, sizeof(double) * 1024));
    return ALEFSI_OK;
  }

  // The three phases of a solve (reference linsolve.py:41-115), enqueued on
  // `stream`: init (||b||, tolerance, v_0), one Arnoldi step (V-cycle on
  // vin -> vout, w = A vout, classical Gram-Schmidt with the conditional
  // second pass, v_{k+1}, Givens update and stopping test), and the
  // solution x = M(V y).  Each returns the number of kernels it enqueued.
  int64_t enqueue_init(cudaGraphConditionalHandle cond, int use_cond) {
    return launch_gmres_init(ctl.p, bb.p, fine().ndof(), partial.p, scal.p, resd.p, gd.p, V.p,
                             vin.p, cond, use_cond, stream);
  }

  int64_t enqueue_step(cudaGraphConditionalHandle cond, int use_cond) {
    Level& F = fine();
    const int64_t n = F.ndof();
    const int64_t before = kernel_launches;
    cycle(n_levels - 1, vin.p, vout.p);
    int64_t c = kernel_launches - before;
    kernel_launches = before;
    int pr = prof_begin(0, n_levels - 1);
    launch_spmv(F.mat(), vout.p, nullptr, w.p, 0, stream);
    prof_end(pr);
    pr = prof_begin(6, n_levels - 1);
    int* flag = &ctl.p->flag;
    const int mx = v_cap;     // k + 1 <= v_cap - 1
    // first classical Gram-Schmidt pass: tmp[0..k] = V w, tmp[k+1] = w.w
    c += 1 + launch_multi_dot(ctl.p, mx, V.p, n, w.p, n, partial.p, tmp.p, nullptr, stream);
    c += launch_multi_axpy(ctl.p, V.p, n, tmp.p, w.p, n, partial.p, scal.p, nullptr, stream);
    c += launch_arnoldi_finish(ctl.p, tmp.p, tmp2.p, scal.p, 0, stream);
    // conditional second pass (device flag)
    c += launch_multi_dot(ctl.p, mx, V.p, n, w.p, n, partial.p, tmp2.p, flag, stream);
    c += launch_multi_axpy(ctl.p, V.p, n, tmp2.p, w.p, n, partial.p, scal.p, flag, stream);
    c += launch_arnoldi_finish(ctl.p, tmp.p, tmp2.p, scal.p, 1, stream);
    c += launch_scale_copy_slot(ctl.p, w.p, V.p, n, tmp.p, vin.p, n, stream);
    c += launch_givens(ctl.p, tmp.p, Hd.p, csd.p, snd.p, gd.p, resd.p, cond, use_cond, stream);
    prof_end(pr);
    return c;
  }

  int64_t enqueue_solution() {
    const int64_t n = fine().ndof();
    int64_t c = launch_gmres_solution(ctl.p, Hd.p, gd.p, yd.p, V.p, n, vin.p, n, stream);
    const int64_t before = kernel_launches;
    cycle(n_levels - 1, vin.p, vout.p);
    c += kernel_launches - before;
    kernel_launches = before;
    return c;
  }

  // capture init -> while(step) -> solution as one graph (conditional while
  // node; the body's last kernel sets the condition)
  int build_solve_graph() {
    if (!cap_stream) {
      CK(cudaStreamCreateWithFlags(&cap_stream, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&cap_in, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&cap_out, cudaEventDisableTiming));
    }
    if (solve_exec) {
      cudaGraphExecDestroy(solve_exec);
      solve_exec = nullptr;
    }
    cudaGraph_t graph = nullptr;
    CK(cudaGraphCreate(&graph, 0));
    cudaGraphConditionalHandle cond;
    CK(cudaGraphConditionalHandleCreate(&cond, graph, 0, 0));
    cudaStream_t user = stream;
    stream = cap_stream;
    auto restore = [&](cudaError_t e) {
      stream = user;
      if (e != cudaSuccess) cudaGraphDestroy(graph);
      return e;
    };
    CK(restore(cudaStreamBeginCaptureToGraph(stream, graph, nullptr, nullptr, 0,
                                             cudaStreamCaptureModeThreadLocal)));
    stream = cap_stream;
    n_init = enqueue_init(cond, 1);
    cudaStreamCaptureStatus st;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    cudaGraph_t cg = nullptr;
    cudaError_t e = cudaStreamGetCaptureInfo(stream, &st, nullptr, &cg, &deps, &ndeps);
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = cond;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t wnode;
    if (e == cudaSuccess) e = cudaGraphAddNode(&wnode, cg, deps, ndeps, &cp);
    if (e == cudaSuccess)
      e = cudaStreamUpdateCaptureDependencies(stream, &wnode, 1, cudaStreamSetCaptureDependencies);
    if (e != cudaSuccess) {
      cudaGraph_t junk;
      cudaStreamEndCapture(stream, &junk);
      return fail(ALEFSI_ERR_CUDA, std::string("solve graph: ") + cudaGetErrorString(restore(e)));
    }
    // body: one Arnoldi step, captured from a second (private) stream
    cudaStream_t body_stream;
    e = cudaStreamCreateWithFlags(&body_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess)
      e = cudaStreamBeginCaptureToGraph(body_stream, cp.conditional.phGraph_out[0], nullptr,
                                        nullptr, 0, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
      stream = body_stream;
      n_body = enqueue_step(cond, 1);
      stream = cap_stream;
      e = cudaStreamEndCapture(body_stream, nullptr);
    }
    cudaStreamDestroy(body_stream);
    if (e != cudaSuccess) {
      cudaGraph_t junk;
      cudaStreamEndCapture(stream, &junk);
      return fail(ALEFSI_ERR_CUDA, std::string("solve graph body: ") + cudaGetErrorString(restore(e)));
    }
    n_fin = enqueue_solution();
    e = cudaStreamEndCapture(stream, &graph);
    CK(restore(e));
    e = cudaGraphInstantiate(&solve_exec, graph, 0);
    cudaGraphDestroy(graph);
    CK(e);
    solve_valid = true;
    return ALEFSI_OK;
  }

  int gmres(const double* b_in, double* x_out, double rel_tol, double abs_tol, int max_iter,
            int host_ptrs, double* residuals, int* iterations, int* converged) {
    if (!factorized) return fail(ALEFSI_ERR_STATE, "gmres before mg_factorize");
    if (max_iter < 1 || max_iter > 510) return fail(ALEFSI_ERR_ARG, "max_iter must be in [1, 510]");
    int rc = ensure_workspace(max_iter);
    if (rc) return rc;
    const int64_t n = fine().ndof();
    GmresCtl& hc = *ctl_host;
    hc = GmresCtl{};
    hc.rel_tol = rel_tol;
    hc.abs_tol = abs_tol;
    hc.max_iter = max_iter;
    hc.hstride = v_cap - 1;
    CK(cudaMemcpyAsync(ctl.p, &hc, sizeof(GmresCtl), cudaMemcpyHostToDevice, stream));
    CK(cudaMemcpyAsync(bb.p, b_in, sizeof(double) * n,
                       host_ptrs ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, stream));
    if (use_graph && !prof_on) {
      if (!solve_valid) {
        rc = build_solve_graph();
        if (rc) return rc;
      }
      CK(cudaGraphLaunch(solve_exec, stream));
      CK(cudaMemcpyAsync(&hc, ctl.p, sizeof(GmresCtl), cudaMemcpyDeviceToHost, stream));
      CK(cudaStreamSynchronize(stream));
      kernel_launches += n_init + (int64_t)hc.its * n_body + n_fin;
    } else {
      // the same kernels, stepped from the host (per-kernel profiling, or
      // graphs off): one control-block read per Arnoldi step
      cudaGraphConditionalHandle none = 0;
      kernel_launches += enqueue_init(none, 0);
      CK(cudaMemcpyAsync(&hc, ctl.p, sizeof(GmresCtl), cudaMemcpyDeviceToHost, stream));
      CK(cudaStreamSynchronize(stream));
      while (!hc.done) {
        kernel_launches += enqueue_step(none, 0);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(&hc, ctl.p, sizeof(GmresCtl), cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        prof_collect();
      }
      kernel_launches += enqueue_solution();
    }
    CK(cudaGetLastError());
    const int its = hc.its;
    if (its == 0) {       // ||b|| <= tol: x = 0 (linsolve.py:58-61)
      if (host_ptrs) std::fill(x_out, x_out + n, 0.0);
      else CK(cudaMemsetAsync(x_out, 0, sizeof(double) * n, stream));
    } else {
      CK(cudaMemcpyAsync(x_out, vout.p, sizeof(double) * n,
                         host_ptrs ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, stream));
    }
    CK(cudaMemcpyAsync(residuals, resd.p, sizeof(double) * (its + 1), cudaMemcpyDeviceToHost,
                       stream));
    CK(cudaStreamSynchronize(stream));
    prof_collect();
    *iterations = its;
    *converged = hc.converged;
    if (!hc.converged) return fail(ALEFSI_ERR_NOT_CONVERGED, "GMRES did not reach the tolerance");
    return ALEFSI_OK;
  }
};

}  // namespace alefsi

using alefsi::MgHandle;
using alefsi::fail;

#define CKAPI(expr)                                                               \
  do {                                                                            \
    cudaError_t _e = (expr);                                                      \
    if (_e != cudaSuccess)                                                        \
      return fail(ALEFSI_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

static MgHandle* H(alefsi_mg h) { return reinterpret_cast<MgHandle*>(h); }

static int check_level(MgHandle* m, int level) {
  if (!m) return fail(ALEFSI_ERR_ARG, "null handle");
  if (level < 0 || level >= m->n_levels) return fail(ALEFSI_ERR_ARG, "level out of range");
  return ALEFSI_OK;
}

extern "C" {

int alefsi_device_count(int32_t* count) {
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  *count = (e == cudaSuccess) ? c : 0;
  return ALEFSI_OK;
}

int alefsi_mg_create(int32_t n_levels, int32_t nc, int32_t nu_pre, int32_t nu_post, double omega,
                     alefsi_mg* out) {
  ALEFSI_TRY_BEGIN
  if (n_levels < 1 || nc < 1 || nc > 4 || nu_pre < 0 || nu_post < 0)
    return fail(ALEFSI_ERR_ARG, "mg_create: bad arguments");
  auto* m = new MgHandle();
  m->n_levels = n_levels;
  m->nc = nc;
  m->nu_pre = nu_pre;
  m->nu_post = nu_post;
  m->omega = omega;
  m->lv.resize(n_levels);
  for (auto& L : m->lv) L.nc = nc;
  cudaError_t e = cudaStreamCreateWithFlags(&m->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete m;
    return fail(ALEFSI_ERR_CUDA, std::string("stream create: ") + cudaGetErrorString(e));
  }
  m->own_stream = true;
  e = m->status.alloc(1);
  if (e != cudaSuccess) {
    delete m;
    return fail(ALEFSI_ERR_CUDA, std::string("alloc: ") + cudaGetErrorString(e));
  }
  *out = reinterpret_cast<alefsi_mg>(m);
  return ALEFSI_OK;
  ALEFSI_TRY_END
}

int alefsi_mg_destroy(alefsi_mg h) {
  ALEFSI_TRY_BEGIN
  MgHandle* m = H(h);
  if (m) {
    cudaStreamSynchronize(m->stream);
    delete m;
  }
  return ALEFSI_OK;
  ALEFSI_TRY_END
}

int alefsi_mg_set_stream(alefsi_mg h, void* stream) {
  MgHandle* m = H(h);
  if (!m) return fail(ALEFSI_ERR_ARG, "null handle");
  cudaStreamSynchronize(m->stream);
  if (m->own_stream) cudaStreamDestroy(m->stream);
  m->stream = reinterpret_cast<cudaStream_t>(stream);
  m->own_stream = false;
  m->graph_valid = false;
  m->solve_valid = false;
  return ALEFSI_OK;
}

int alefsi_mg_use_graph(alefsi_mg h, int32_t on) {
  MgHandle* m = H(h);
  if (!m) return fail(ALEFSI_ERR_ARG, "null handle");
  m->use_graph = on != 0;
  m->graph_valid = false;
  m->solve_valid = false;
  return ALEFSI_OK;
}

int alefsi_mg_set_matrix(alefsi_mg h, int32_t level, int64_t n_nodes, int64_t nnzb,
                         const int64_t* indptr, const int32_t* indices, const double* data,
                         int64_t nnz_pp, const int64_t* pp_indptr, const int32_t* pp_indices,
                         const double* pp_data) {
  ALEFSI_TRY_BEGIN
  MgHandle* m = H(h);
  int rc = check_level(m, level);
  if (rc) return rc;
  auto& L = m->lv[level];
  const int nc = m->nc;
  if (indptr[0] != 0 || indptr[n_nodes] != nnzb) return fail(ALEFSI_ERR_ARG, "bad indptr");
  if (nnz_pp > 0 && (pp_indptr[0] != 0 || pp_indptr[n_nodes] != nnz_pp))
    return fail(ALEFSI_ERR_ARG, "bad pp_indptr");
  L.n_nodes = n_nodes;
  L.nnzb = nnzb;
  L.nnz_pp = nnz_pp;
  if (level == 0) m->cancel_coarse_inflight();
  ++L.pattern_epoch;
  CKAPI(L.indptr.upload(indptr, n_nodes + 1, m->stream));
  CKAPI(L.indices.upload(indices, nnzb, m->stream));
  CKAPI(L.data.upload(data, (size_t)nnzb * nc * nc, m->stream));
  if (nnz_pp > 0) {
    CKAPI(L.pp_indptr.upload(pp_indptr, n_nodes + 1, m->stream));
    CKAPI(L.pp_indices.upload(pp_indices, nnz_pp, m->stream));
    CKAPI(L.pp_data.upload(pp_data, nnz_pp, m->stream));
  }
  L.nc = nc;
  rc = alefsi::build_sell(L, alefsi::default_sell_lanes(nc, n_nodes), indptr, indices, pp_indptr,
                         pp_indices, m->stream);
  if (rc) return rc;
  if (level == 0) {
    const int64_t n0 = n_nodes * nc;
    if (n0 > 20000) return fail(ALEFSI_ERR_ARG, "coarse level too large for a dense inverse");
    L.host_dense.assign((size_t)n0 * n0, 0.0);
    for (int64_t r = 0; r < n_nodes; ++r) {
      for (int64_t s = indptr[r]; s < indptr[r + 1]; ++s) {
        const int64_t c = indices[s];
        for (int i = 0; i < nc; ++i)
          for (int j = 0; j < nc; ++j)
            L.host_dense[(size_t)(r * nc + i) * n0 + c * nc + j] +=
                data[(size_t)s * nc * nc + i * nc + j];
      }
      if (nnz_pp > 0)
        for (int64_t s = pp_indptr[r]; s < pp_indptr[r + 1]; ++s)
          L.host_dense[(size_t)(r * nc) * n0 + (int64_t)pp_indices[s] * nc] += pp_data[s];
    }
  }
  CKAPI(cudaStreamSynchronize(m->stream));
  L.has_matrix = true;
  m->factorized = false;
  m->graph_valid = false;
  m->solve_valid = false;
  return ALEFSI_OK;
  ALEFSI_TRY_END
}

int alefsi_mg_set_pattern(alefsi_mg h, int32_t level, int64_t n_nodes, int64_t nnzb,
                          const int64_t* indptr, const int32_t* indices, int64_t nnz_pp,
                          const int64_t* pp_indptr, const int32_t* pp_indices) {
  ALEFSI_TRY_BEGIN
  MgHandle* m = H(h);
  int rc = check_level(m, level);
  if (rc) return rc;
  auto& L = m->lv[level];
  const int nc = m->nc;
  if (indptr[0] != 0 || indptr[n_nodes] != nnzb) return fail(ALEFSI_ERR_ARG, "bad indptr");
  if (nnzb >= (int64_t)1 << 31) return fail(ALEFSI_ERR_ARG, "pattern too large for int32 slots");
  L.n_nodes = n_nodes;
  L.nnzb = nnzb;
  L.nnz_pp = nnz_pp;
  if (level == 0) m->cancel_coarse_inflight();
  ++L.pattern_epoch;
  CKAPI(L.indptr.upload(indptr, n_nodes + 1, m->stream));
  CKAPI(L.indices.upload(indices, nnzb, m->stream));
  CKAPI(L.data.alloc((size_t)nnzb * nc * nc));
  CKAPI(cudaMemsetAsync(L.data.p, 0, sizeof(double) * nnzb * nc * nc, m->stream));
  if (nnz_pp > 0) {
    CKAPI(L.pp_indptr.upload(pp_indptr, n_nodes + 1, m->stream));
    CKAPI(L.pp_indices.upload(pp_indices, nnz_pp, m->stream));
    CKAPI(L.pp_data.alloc(nnz_pp));
    CKAPI(cudaMemsetAsync(L.pp_data.p, 0, sizeof(double) * nnz_pp, m->stream));
  }
  L.nc = nc;
  rc = alefsi::build_sell(L, alefsi::default_sell_lanes(nc, n_nodes), indptr, indices, pp_indptr,
                         pp_indices, m->stream);
  if (rc) return rc;
  L.host_dense.clear();
  CKAPI(cudaStreamSynchronize(m->stream));
  L.has_matrix = true;
  m->factorized = false;
  m->graph_valid = false;
  m->solve_valid = false;
  return ALEFSI_OK;
  ALEFSI_TRY_END
}

int alefsi_mg_asm_setup(alefsi_mg h, int32_t level, int32_t dim, int64_t n_cells,
                        const int32_t* cell_nodes, const double* coords, int32_t n_groups,
                        const int64_t* group_ptr, const int32_t* group_kind,
                        const int32_t* group_cells, int64_t n_lps, const int64_t* lps_cell_slot,
                        const int64_t* lps_pp_slot, const double* lps_vals,
                        const uint8_t* dirichlet) {
  ALEFSI_TRY_BEGIN
  MgHandle* m = H(h);
  int rc = check_level(m, level);
  if (rc) return rc;
  auto& L = m->lv[level];
  if (!L.has_matrix) return fail(ALEFSI_ERR_STATE, "set_pattern before asm_setup");
  if (dim + 1 != m->nc || (dim != 2 && dim != 3)) return fail(ALEFSI_ERR_ARG, "asm: bad dim");
  // the cell kernels keep block slots as 32-bit ints in shared memory
  if (L.nnzb >= ((int64_t)1 << 31))
    return fail(ALEFSI_ERR_ARG, "asm: device assembly needs fewer than 2^31 blocks per level");
  const int nb = dim == 3 ? 27 : 9;
  L.dim = dim;
  CKAPI(L.asm_cell_nodes.upload(cell_nodes, (size_t)n_cells * nb, m->stream));
  L.asm_n_cells = n_cells;
  L.asm_slots_epoch = -1;
  CKAPI(L.asm_coords.upload(coords, (size_t)L.n_nodes * dim, m->stream));
  L.asm_group_ptr.assign(group_ptr, group_ptr + n_groups + 1);
  L.asm_group_kind.assign(group_kind, group_kind + n_groups);
  CKAPI(L.asm_group_cells.upload(group_cells, group_ptr[n_groups], m->stream));
  L.n_lps = n_lps;
  if (n_lps > 0) {
    CKAPI(L.lps_cell.upload(lps_cell_slot, n_lps, m->stream));
    CKAPI(L.lps_pp.upload(lps_pp_slot, n_lps, m->stream));
    CKAPI(L.lps_val.upload(lps_vals, n_lps, m->stream));
  }
  CKAPI(L.dir_mask.upload(dirichlet, L.ndof(), m->stream));
  CKAPI(L.asm_U.alloc((size_t)L.n_nodes * (1 + 2 * dim)));
  CKAPI(L.asm_Up.alloc((size_t)L.n_nodes * (1 + 2 * dim)));
  CKAPI(cudaStreamSynchronize(m->stream));
  L.has_asm = true;
  return ALEFSI_OK;
  ALEFSI_TRY_END
}

int alefsi_mg_asm_tables(alefsi_mg h, int32_t dim, int32_t nq, const double* N, const double* dN,
                         const double* w) {
  MgHandle* m = H(h);
  if (!m) return fail(ALEFSI_ERR_ARG, "null handle");
  const int nb = dim == 3 ? 27 : 9;
  if (dim != 2 && dim != 3) return fail(ALEFSI_ERR_ARG, "asm: dim must be 2 or 3");
  if (nq != nb)
    return fail(ALEFSI_ERR_ARG, "asm: the Q2 kernels integrate with nq == nb quadrature points");
  const int rc = alefsi::set_assembly_tables(N, dN, w, nq, nb, dim);
  if (rc == 2)
    return fail(ALEFSI_ERR_ARG, "asm: shape tables differ from those already loaded for dim " +
                                    std::to_string(dim));
  if (rc != 0) return fail(ALEFSI_ERR_CUDA, "asm: loading the shape tables failed");
  return ALEFSI_OK;
}

// params = rho_f, mu_f, rho_s, mu_s, lam_s, k, theta; U, Up host (n_nodes, 1+2d);
// extra = host-reduced facet blocks (unique slots) added after the cells
int alefsi_mg_asm_momentum(alefsi_mg h, int32_t level, const double* params, const double* U,
                           const double* Up, int64_t n_extra, const int64_t* extra_slots,
                           const double* extra_vals) {
  ALEFSI_TRY_BEGIN
  MgHandle* m = H(h);
  int rc = check_level(m, level);
  if (rc) return rc;
  auto& L = m->lv[level];
  if (!L.has_asm) return fail(ALEFSI_ERR_STATE, "asm_setup missing");
  if (level == 0) m->cancel_coarse_inflight();
  const int nc = m->nc, nf = 1 + 2 * L.dim;
  cudaStream_t s = m->stream;
  CKAPI(cudaMemcpyAsync(L.asm_U.p, U, sizeof(double) * L.n_nodes * nf, cudaMemcpyHostToDevice, s));
  CKAPI(cudaMemcpyAsync(L.asm_Up.p, Up, sizeof(double) * L.n_nodes * nf, cudaMemcpyHostToDevice, s));
  CKAPI(cudaMemsetAsync(L.data.p, 0, sizeof(double) * L.nnzb * nc * nc, s));
  if (L.nnz_pp > 0) CKAPI(cudaMemsetAsync(L.pp_data.p, 0, sizeof(double) * L.nnz_pp, s));
  CKAPI(cudaMemsetAsync(m->status.p, 0, sizeof(int64_t), s));
  L.sell_dirty = true;
  if (L.asm_slots_epoch != L.pattern_epoch) {
    // block slots of every cell's node pairs, once per sparsity pattern
    const int nb = L.dim == 3 ? 27 : 9;
    CKAPI(L.asm_cell_slots.ensure((size_t)L.asm_n_cells * nb * nb));
    alefsi::DevPatchGroup cg;
    cg.npn = nb;
    cg.n_patches = L.asm_n_cells;
    cg.nodes = L.asm_cell_nodes.p;
    alefsi::launch_patch_slots(L.mat(), cg, L.asm_cell_slots.p, s);
    L.asm_slots_epoch = L.pattern_epoch;
  }
  alefsi::AsmArgs a;
  a.cell_nodes = L.asm_cell_nodes.p;
  a.cell_slots = L.asm_cell_slots.p;
  a.coords = L.asm_coords.p;
  a.U = L.asm_U.p;
  a.Up = L.asm_Up.p;
  a.data = L.data.p;
  a.status = m->status.p;
  a.rho_f = params[0];
  a.mu_f = params[1];
  a.rho_s = params[2];
  a.mu_s = params[3];
  a.lam_s = params[4];
  a.k = params[5];
  a.theta = params[6];
  for (size_t g = 0; g + 1 < L.asm_group_ptr.size(); ++g) {
    const int64_t b = L.asm_group_ptr[g], e = L.asm_group_ptr[g + 1];
    alefsi::launch_assemble_cells(a, L.dim, L.asm_group_kind[g], L.asm_group_cells.p + b, e - b, s);
    ++m->kernel_launches;
  }
  CKAPI(cudaGetLastError());
  if (L.of_nf > 0) {
    alefsi::OutflowArgs o;
    o.n_facets = L.of_nf;
    o.nq = L.of_nq;
    o.conn = L.of_conn.p;
    o.cell_of_facet = L.of_cells.p;
    o.N = L.of_N.p;
    o.G = L.of_G.p;
    o.dS = L.of_dS.p;
    o.normal = L.of_n.p;
    o.U = L.asm_U.p;
    o.status = m->status.p;
    o.mu_f = a.mu_f;
    o.k = a.k;
    o.theta = a.theta;
    alefsi::launch_outflow(o, L.dim, L.of_nu, L.of_slots.p, L.of_uptr.p, L.of_contrib.p,
                           L.of_local.p, L.data.p, s);
    m->kernel_launches += 2;
  }
  if (n_extra > 0) {
    CKAPI(L.asm_extra_slots.upload(extra_slots, n_extra, s));
    CKAPI(L.asm_extra_vals.upload(extra_vals, (size_t)n_extra * nc * nc, s));
    alefsi::launch_add_blocks(L.data.p, nc * nc, n_extra, L.asm_extra_slots.p,
                              L.asm_extra_vals.p, s);
  }
  alefsi::launch_lps(L.data.p, nc, L.pp_data.p, L.n_lps, L.lps_cell.p, L.lps_pp.p, L.lps_val.p,
                     a.k, s);
  alefsi::launch_dirichlet(L.data.p, nc, L.pp_data.p, L.n_nodes, L.indptr.p, L.indices.p,
                           L.nnz_pp > 0 ? L.pp_indptr.p : nullptr, L.dir_mask.p, s);
  m->kernel_launches += 2;
  int64_t st = 0;
  CKAPI(cudaMemcpyAsync(&st, m->status.p, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CKAPI(cudaStreamSynchronize(s));
  if (st != 0)
    return fail(ALEFSI_ERR_SINGULAR, "inverted element in device assembly: cell " +
                                         std::to_string(st - 1));
  // operator values change in place: the V-cycle graph (pointers only) stays
  m->factorized = false;
  if (level == 0 && m->n_levels > 1) {
    // the coarse inverse is a serial chain of ~n/16 panel steps: start it now,
    // under the assembly of the finer levels (alefsi_mg_factorize joins it)
    rc = m->start_coarse_inverse();
    if (rc) {
      if (m->side_stream) cudaStreamSynchronize(m->side_stream);
      return rc;
    }
    m->coarse_inflight = true;
  }
  return ALEFSI_OK;
  ALEFSI_TRY_END
}

int alefsi_mg_asm_outflow(alefsi_mg h, int32_t level, int64_t n_facets, int32_t nq,
                          const int32_t* conn, const int64_t* cells, const double* N,
                          const double* G, const double* dS, const double* normal,
                          int64_t n_unique, const int64_t* slots, const int64_t* uptr,
                          const int64_t* contrib) {
  ALEFSI_TRY_BEGIN
  MgHandle* m = H(h);
  int rc = check_level(m, level);
  if (rc) return rc;
  auto& L = m->lv[level];
  if (!L.has_asm) return fail(ALEFSI_ERR_STATE, "asm_setup missing");
  const int d = L.dim, nb = d == 2 ? 9 : 27;
  if (n_facets < 0 || n_unique < 0 || nq < 1 || nq > (d == 2 ? 3 : 9))
    return fail(ALEFSI_ERR_ARG, "bad outflow facet sizes");
  cudaStream_t s = m->stream;
  const size_t nfq = (size_t)n_facets * nq;
  CKAPI(L.of_conn.upload(conn, (size_t)n_facets * nb, s));
  CKAPI(L.of_cells.upload(cells, (size_t)n_facets, s));
  CKAPI(L.of_N.upload(N, nfq * nb, s));
  CKAPI(L.of_G.upload(G, nfq * nb * d, s));
  CKAPI(L.of_dS.upload(dS, nfq, s));
  CKAPI(L.of_n.upload(normal, nfq * d, s));
  CKAPI(L.of_slots.upload(slots, (size_t)n_unique, s));
  CKAPI(L.of_uptr.upload(uptr, (size_t)n_unique + 1, s));
  CKAPI(L.of_contrib.upload(contrib, (size_t)n_facets * nb * nb, s));
  CKAPI(L.of_local.ensure((size_t)n_facets * nb * nb * d * d));
  CKAPI(cudaStreamSynchronize(s));
  L.of_nf = n_facets;
  L.of_nq = nq;
  L.of_nu = n_unique;
  return ALEFSI_OK;
  ALEFSI_TRY_END
}

int alefsi_mg_asm_residual_tables(alefsi_mg h, int32_t level, const int64_t* lps_indptr,
                                  const int32_t* lps_indices, const double* lps_vals,
                                  int64_t n_onodes, const int64_t* onodes, const int64_t* ouptr,
                                  const int64_t* ocontrib) {
  ALEFSI_TRY_BEGIN
  MgHandle* m = H(h);
  int rc = check_level(m, level);
  if (rc) return rc;
  auto& L = m->lv[level];
  if (!L.has_asm) return fail(ALEFSI_ERR_STATE, "asm_setup missing");
  const int d = L.dim, nb = d == 2 ? 9 : 27;
  if (n_onodes > 0 && L.of_nf == 0) return fail(ALEFSI_ERR_STATE, "asm_outflow missing");
  cudaStream_t s = m->stream;
  const int64_t nnz = lps_indptr[L.n_nodes];
  CKAPI(L.lps_indptr.upload(lps_indptr, (size_t)L.n_nodes + 1, s));
  CKAPI(L.lps_indices.upload(lps_indices, (size_t)nnz, s));
  CKAPI(L.lps_vals.upload(lps_vals, (size_t)nnz, s));
  if (n_onodes > 0) {
    CKAPI(L.rt_nodes.upload(onodes, (size_t)n_onodes, s));
    CKAPI(L.rt_uptr.upload(ouptr, (size_t)n_onodes + 1, s));
    CKAPI(L.rt_contrib.upload(ocontrib, (size_t)L.of_nf * nb, s));
    CKAPI(L.rt_local.ensure((size_t)L.of_nf * nb * d));
  }
  CKAPI(cudaStreamSynchronize(s));
  L.rt_nodes_n = n_onodes;
  L.rt_ready = true;
  return ALEFSI_OK;
  ALEFSI_TRY_END
}

// params = rho_f, mu_f, rho_s, mu_s, lam_s, k, theta, f0, f1, f2, ext_model
// (0 harmonic / 1 linear elasticity), ext_mu, ext_lam, ext_volume_scaling.
// which = 0: cell parts of the theta residual -> out (n_nodes, 1+2d);
// which = 1: cell parts of the explicit forces of U_prev -> out (n_nodes, d).
// U, U_prev, out are host arrays.
int alefsi_mg_asm_residual(alefsi_mg h, int32_t level, const double* params, const double* U,
                           const double* Up, int32_t which, double* out) {
  ALEFSI_TRY_BEGIN
  MgHandle* m = H(h);
  int rc = check_level(m, level);
  if (rc) return rc;
  auto& L = m->lv[level];
  if (!L.has_asm) return fail(ALEFSI_ERR_STATE, "asm_setup missing");
  const int d = L.dim, nf = 1 + 2 * d;
  const int no = which == 0 ? nf : d;
  cudaStream_t s = m->stream;
  if (U) CKAPI(cudaMemcpyAsync(L.asm_U.p, U, sizeof(double) * L.n_nodes * nf, cudaMemcpyHostToDevice, s));
  CKAPI(cudaMemcpyAsync(L.asm_Up.p, Up, sizeof(double) * L.n_nodes * nf, cudaMemcpyHostToDevice, s));
  if (L.res_out.n != (size_t)L.n_nodes * nf) CKAPI(L.res_out.alloc((size_t)L.n_nodes * nf));
  CKAPI(cudaMemsetAsync(L.res_out.p, 0, sizeof(double) * L.n_nodes * no, s));
  CKAPI(cudaMemsetAsync(m->status.p, 0, sizeof(int64_t), s));
  alefsi::ResArgs a;
  a.cell_nodes = L.asm_cell_nodes.p;
  a.coords = L.asm_coords.p;
  a.U = L.asm_U.p;
  a.Up = L.asm_Up.p;
  a.status = m->status.p;
  a.rho_f = params[0];
  a.mu_f = params[1];
  a.rho_s = params[2];
  a.mu_s = params[3];
  a.lam_s = params[4];
  a.k = params[5];
  a.theta = params[6];
  a.f[0] = params[7];
  a.f[1] = params[8];
  a.f[2] = params[9];
  a.ext_model = (int)params[10];
  a.ext_mu = params[11];
  a.ext_lam = params[12];
  a.ext_volume_scaling = (int)params[13];
  for (size_t g = 0; g + 1 < L.asm_group_ptr.size(); ++g) {
    const int64_t b = L.asm_group_ptr[g], e = L.asm_group_ptr[g + 1];
    const int kind = L.asm_group_kind[g] + (which == 1 ? 2 : 0);
    alefsi::launch_residual_cells(a, d, kind, L.asm_group_cells.p + b, e - b, L.res_out.p, s);
    ++m->kernel_launches;
  }
  if (L.rt_ready) {
    if (L.of_nf > 0) {
      alefsi::OutflowArgs o;
      o.n_facets = L.of_nf;
      o.nq = L.of_nq;
      o.conn = L.of_conn.p;
      o.cell_of_facet = L.of_cells.p;
      o.N = L.of_N.p;
      o.G = L.of_G.p;
      o.dS = L.of_dS.p;
      o.normal = L.of_n.p;
      o.U = which == 0 ? L.asm_U.p : L.asm_Up.p;
      o.status = m->status.p;
      o.mu_f = a.mu_f;
      const double scale = which == 0 ? a.k * a.theta : 1.0;
      alefsi::launch_outflow_residual(o, d, scale, L.rt_nodes_n, L.rt_nodes.p, L.rt_uptr.p,
                                      L.rt_contrib.p, L.rt_local.p, L.res_out.p, no,
                                      which == 0 ? 1 : 0, s);
      m->kernel_launches += 2;
    }
    if (which == 0) {
      alefsi::launch_lps_residual(L.n_nodes, L.lps_indptr.p, L.lps_indices.p, L.lps_vals.p,
                                  L.asm_U.p, nf, a.k, L.res_out.p, no, s);
      ++m->kernel_launches;
    }
  }
  CKAPI(cudaGetLastError());
  CKAPI(cudaMemcpyAsync(out, L.res_out.p, sizeof(double) * L.n_nodes * no, cudaMemcpyDeviceToHost, s));
  int64_t st = 0;
  CKAPI(cudaMemcpyAsync(&st, m->status.p, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CKAPI(cudaStreamSynchronize(s));
  if (st != 0)
    return fail(ALEFSI_ERR_SINGULAR, "inverted element in device residual: cell " +
                                         std::to_string(st - 1));
  return ALEFSI_OK;
  ALEFSI_TRY_END
}

int alefsi_mg_get_matrix(alefsi_mg h, int32_t level, double* data, double* pp_data) {
  ALEFSI_TRY_BEGIN
  MgHandle* m = H(h);
  int rc = check_level(m, level);
  if (rc) return rc;
  auto& L = m->lv[level];
  CKAPI(cudaMemcpyAsync(data, L.data.p, sizeof(double) * L.nnzb * m->nc * m->nc,
                        cudaMemcpyDeviceToHost, m->stream));
  if (L.nnz_pp > 0 && pp_data)
    CKAPI(cudaMemcpyAsync(pp_data, L.pp_data.p, sizeof(double) * L.nnz_pp,
                          cudaMemcpyDeviceToHost, m->stream));
  CKAPI(cudaStreamSynchronize(m->stream));
  return ALEFSI_OK;
  ALEFSI_TRY_END
}

int alefsi_mg_set_patches(alefsi_mg h, int32_t level, int32_t n_groups,
                          const int64_t* group_n_patches, const int32_t* group_nodes_per_patch,
                          const int64_t* patch_nodes) {
  ALEFSI_TRY_BEGIN
  MgHandle* m = H(h);
  int rc = check_level(m, level);
  if (rc) return rc;
  auto& L = m->lv[level];
  if (L.n_nodes == 0) return fail(ALEFSI_ERR_STATE, "set_matrix before set_patches");
  const int nc = m->nc;
  L.groups.clear();
  int64_t y_size = 0, flat_off = 0;
  std::vector<int64_t> mult(L.n_nodes, 0);
  // node -> (Y offset) gather entries in ascending global patch order
  std::vector<int64_t> count(L.n_nodes + 1, 0);
  for (int gi = 0; gi < n_groups; ++gi) {
    const int npn = group_nodes_per_patch[gi];
    const int64_t np_ = group_n_patches[gi];
    for (int64_t s = 0; s < np_ * npn; ++s) {
      const int64_t nd = patch_nodes[flat_off + s];
      if (nd < 0 || nd >= L.n_nodes) return fail(ALEFSI_ERR_ARG, "patch node out of range");
      count[nd + 1]++;
    }
    flat_off += np_ * npn;
  }
  for (int64_t i = 0; i < L.n_nodes; ++i) count[i + 1] += count[i];
  std::vector<int64_t> goff(count[L.n_nodes]);
  std::vector<int64_t> fill(count.begin(), count.end() - 1);
  flat_off = 0;
  for (int gi = 0; gi < n_groups; ++gi) {
    auto g = std::make_unique<alefsi::Group>();
    g->npn = group_nodes_per_patch[gi];
    g->np = g->npn * nc;
    if (!alefsi::vanka_supported(nc, g->np))
      return fail(ALEFSI_ERR_ARG, "unsupported Vanka patch size " + std::to_string(g->np) +
                                      " for nc=" + std::to_string(nc));
    g->ld = (g->np + 1) / 2 * 2;
    g->n_patches = group_n_patches[gi];
    g->y_offset = y_size;
    std::vector<int32_t> nodes32((size_t)g->n_patches * g->npn);
    for (int64_t p = 0; p < g->n_patches; ++p)
      for (int a = 0; a < g->npn; ++a) {
        const int64_t nd = patch_nodes[flat_off + p * g->npn + a];
        nodes32[(size_t)p * g->npn + a] = (int32_t)nd;
        goff[fill[nd]++] = y_size + p * g->ld + (int64_t)a * nc;
      }
    CKAPI(g->nodes.upload(nodes32.data(), nodes32.size(), m->stream));
    CKAPI(cudaStreamSynchronize(m->stream));
    flat_off += g->n_patches * g->npn;
    y_size += g->n_patches * g->ld;
    L.groups.push_back(std::move(g));
  }
  // weights 1 / multiplicity (linsolve.py:156-161)
  std::vector<double> wts(L.n_nodes);
  for (int64_t i = 0; i < L.n_nodes; ++i) {
    const int64_t c = count[i + 1] - count[i];
    wts[i] = 1.0 / (double)(c == 0 ? 1 : c);
  }
  CKAPI(L.Y.alloc(y_size));
  CKAPI(L.gptr.upload(count.data(), count.size(), m->stream));
  CKAPI(L.goff.upload(goff.data(), goff.size(), m->stream));
  CKAPI(L.weight.upload(wts.data(), wts.size(), m->stream));
  CKAPI(cudaStreamSynchronize(m->stream));
  m->factorized = false;
  m->graph_valid = false;
  m->solve_valid = false;
  return ALEFSI_OK;
  ALEFSI_TRY_END
}

int alefsi_mg_set_prolongation(alefsi_mg h, int32_t level, int64_t n_fine, int64_t n_coarse,
                               int64_t nnz, const int64_t* indptr, const int32_t* indices,
                               const double* vals) {
  ALEFSI_TRY_BEGIN
  MgHandle* m = H(h);
  int rc = check_level(m, level);
  if (rc) return rc;
  if (level == 0) return fail(ALEFSI_ERR_ARG, "level 0 has no prolongation");
  auto& L = m->lv[level];
  if (indptr[0] != 0 || indptr[n_fine] != nnz) return fail(ALEFSI_ERR_ARG, "bad P indptr");
  CKAPI(L.P_ptr.upload(indptr, n_fine + 1, m->stream));
  CKAPI(L.P_idx.upload(indices, nnz, m->stream));
  CKAPI(L.P_val.upload(vals, nnz, m->stream));
  // transpose (coarse rows, fine columns ascending)
  std::vector<int64_t> rp(n_coarse + 1, 0);
  for (int64_t e = 0; e < nnz; ++e) {
    if (indices[e] < 0 || indices[e] >= n_coarse) return fail(ALEFSI_ERR_ARG, "P column out of range");
    rp[indices[e] + 1]++;
  }
  for (int64_t i = 0; i < n_coarse; ++i) rp[i + 1] += rp[i];
  std::vector<int32_t> ri(nnz);
  std::vector<double> rv(nnz);
  std::vector<int64_t> fill(rp.begin(), rp.end() - 1);
  for (int64_t r = 0; r < n_fine; ++r)
    for (int64_t e = indptr[r]; e < indptr[r + 1]; ++e) {
      const int64_t pos = fill[indices[e]]++;
      ri[pos] = (int32_t)r;
      rv[pos] = vals[e];
    }
  CKAPI(L.R_ptr.upload(rp.data(), rp.size(), m->stream));
  CKAPI(L.R_idx.upload(ri.data(), ri.size(), m->stream));
  CKAPI(L.R_val.upload(rv.data(), rv.size(), m->stream));
  CKAPI(cudaStreamSynchronize(m->stream));
  L.n_coarse = n_coarse;
  L.has_P = true;
  m->graph_valid = false;
  m->solve_valid = false;
  return ALEFSI_OK;
  ALEFSI_TRY_END
}

int alefsi_mg_set_constrained(alefsi_mg h, int32_t level, const uint8_t* mask) {
  ALEFSI_TRY_BEGIN
  MgHandle* m = H(h);
  int rc = check_level(m, level);
  if (rc) return rc;
  auto& L = m->lv[level];
  if (L.n_nodes == 0) return fail(ALEFSI_ERR_STATE, "set_matrix before set_constrained");
  CKAPI(L.constrained.upload(mask, L.ndof(), m->stream));
  CKAPI(cudaStreamSynchronize(m->stream));
  m->graph_valid = false;
  m->solve_valid = false;
  return ALEFSI_OK;
  ALEFSI_TRY_END
}

int alefsi_mg_factorize(alefsi_mg h) {
  ALEFSI_TRY_BEGIN
  MgHandle* m = H(h);
  if (!m) return fail(ALEFSI_ERR_ARG, "null handle");
  return m->factorize();
  ALEFSI_TRY_END
}

int alefsi_mg_apply(alefsi_mg h, const double* b, double* z, int32_t host_ptrs) {
  ALEFSI_TRY_BEGIN
  MgHandle* m = H(h);
  if (!m) return fail(ALEFSI_ERR_ARG, "null handle");
  if (!host_ptrs) return m->apply(b, z);
  const int64_t n = m->fine().ndof();
  int rc = m->ensure_workspace(1);
  if (rc) return rc;
  CKAPI(cudaMemcpyAsync(m->bb.p, b, sizeof(double) * n, cudaMemcpyHostToDevice, m->stream));
  rc = m->apply(m->bb.p, m->xb.p);
  if (rc) return rc;
  CKAPI(cudaMemcpyAsync(z, m->xb.p, sizeof(double) * n, cudaMemcpyDeviceToHost, m->stream));
  CKAPI(cudaStreamSynchronize(m->stream));
  return ALEFSI_OK;
  ALEFSI_TRY_END
}

int alefsi_mg_set_sell(alefsi_mg h, int32_t level, int32_t lanes_per_row) {
  ALEFSI_TRY_BEGIN
  MgHandle* m = H(h);
  int rc = check_level(m, level);
  if (rc) return rc;
  auto& L = m->lv[level];
  if (!L.has_matrix) return fail(ALEFSI_ERR_STATE, "set_sell before the level's pattern");
  std::vector<int64_t> ip(L.n_nodes + 1), pp;
  std::vector<int32_t> ix(L.nnzb), px;
  CKAPI(cudaMemcpy(ip.data(), L.indptr.p, sizeof(int64_t) * ip.size(), cudaMemcpyDeviceToHost));
  CKAPI(cudaMemcpy(ix.data(), L.indices.p, sizeof(int32_t) * ix.size(), cudaMemcpyDeviceToHost));
  if (L.nnz_pp > 0) {
    pp.resize(L.n_nodes + 1);
    px.resize(L.nnz_pp);
    CKAPI(cudaMemcpy(pp.data(), L.pp_indptr.p, sizeof(int64_t) * pp.size(), cudaMemcpyDeviceToHost));
    CKAPI(cudaMemcpy(px.data(), L.pp_indices.p, sizeof(int32_t) * px.size(), cudaMemcpyDeviceToHost));
  }
  rc = alefsi::build_sell(L, lanes_per_row, ip.data(), ix.data(), pp.data(), px.data(), m->stream);
  if (rc) return rc;
  alefsi::refresh_sell(L, m->stream);
  CKAPI(cudaStreamSynchronize(m->stream));
  m->graph_valid = false;
  m->solve_valid = false;
  return ALEFSI_OK;
  ALEFSI_TRY_END
}

int alefsi_mg_set_apply_split(alefsi_mg h, int32_t level, int32_t split) {
  MgHandle* m = H(h);
  int rc = check_level(m, level);
  if (rc) return rc;
  if (split < -1 || split > 1) return fail(ALEFSI_ERR_ARG, "apply split: -1, 0 or 1");
  m->lv[level].apply_split = split;
  m->graph_valid = false;
  m->solve_valid = false;
  return ALEFSI_OK;
}

int alefsi_mg_spmv(alefsi_mg h, int32_t level, const double* x, const double* b, double* y) {
  ALEFSI_TRY_BEGIN
  MgHandle* m = H(h);
  int rc = check_level(m, level);
  if (rc) return rc;
  alefsi::refresh_sell(m->lv[level], m->stream);
  alefsi::launch_spmv(m->lv[level].mat(), x, b, y, b ? 1 : 0, m->stream);
  CKAPI(cudaGetLastError());
  return ALEFSI_OK;
  ALEFSI_TRY_END
}

int alefsi_mg_vanka_sweep(alefsi_mg h, int32_t level, double* x, const double* b) {
  ALEFSI_TRY_BEGIN
  MgHandle* m = H(h);
  int rc = check_level(m, level);
  if (rc) return rc;
  if (!m->factorized) return fail(ALEFSI_ERR_STATE, "sweep before factorize");
  if (level == 0) return fail(ALEFSI_ERR_ARG, "level 0 has no smoother");
  m->sweep(m->lv[level], level, b, x, false);
  CKAPI(cudaGetLastError());
  return ALEFSI_OK;
  ALEFSI_TRY_END
}

int alefsi_mg_restrict(alefsi_mg h, int32_t level, const double* r_fine, double* b_coarse) {
  ALEFSI_TRY_BEGIN
  MgHandle* m = H(h);
  int rc = check_level(m, level);
  if (rc) return rc;
  if (level == 0) return fail(ALEFSI_ERR_ARG, "level 0 has no coarser level");
  auto& L = m->lv[level];
  auto& C = m->lv[level - 1];
  alefsi::launch_restrict(C.n_nodes, C.nc, L.R_ptr.p, L.R_idx.p, L.R_val.p, r_fine,
                          C.constrained.p, b_coarse, m->stream);
  CKAPI(cudaGetLastError());
  return ALEFSI_OK;
  ALEFSI_TRY_END
}

int alefsi_mg_prolong_add(alefsi_mg h, int32_t level, const double* x_coarse, double* x_fine) {
  ALEFSI_TRY_BEGIN
  MgHandle* m = H(h);
  int rc = check_level(m, level);
  if (rc) return rc;
  if (level == 0) return fail(ALEFSI_ERR_ARG, "level 0 has no coarser level");
  auto& L = m->lv[level];
  alefsi::launch_prolong_add(L.n_nodes, L.nc, L.P_ptr.p, L.P_idx.p, L.P_val.p, x_coarse,
                             L.constrained.p, x_fine, m->stream);
  CKAPI(cudaGetLastError());
  return ALEFSI_OK;
  ALEFSI_TRY_END
}

int alefsi_mg_coarse_solve(alefsi_mg h, const double* b, double* x) {
  ALEFSI_TRY_BEGIN
  MgHandle* m = H(h);
  if (!m) return fail(ALEFSI_ERR_ARG, "null handle");
  if (!m->factorized) return fail(ALEFSI_ERR_STATE, "coarse solve before factorize");
  alefsi::launch_dense_matvec(m->lv[0].ndof(), m->coarse_pad.p, m->coarse_ld, b, x, m->stream);
  CKAPI(cudaGetLastError());
  return ALEFSI_OK;
  ALEFSI_TRY_END
}

int alefsi_mg_get_inverses(alefsi_mg h, int32_t level, int32_t group, double* out) {
  ALEFSI_TRY_BEGIN
  MgHandle* m = H(h);
  int rc = check_level(m, level);
  if (rc) return rc;
  auto& L = m->lv[level];
  if (group < 0 || group >= (int)L.groups.size()) return fail(ALEFSI_ERR_ARG, "bad group");
  auto& g = *L.groups[group];
  CKAPI(cudaMemcpyAsync(out, g.inv.p, sizeof(double) * g.inv.n, cudaMemcpyDeviceToHost,
                        m->stream));
  CKAPI(cudaStreamSynchronize(m->stream));
  return ALEFSI_OK;
  ALEFSI_TRY_END
}

// info[0..7] = n_nodes, ndof, nnzb, nnz_pp, n_groups, y_size, inverse doubles, ld of group 0
int alefsi_mg_info(alefsi_mg h, int32_t level, int64_t* info) {
  MgHandle* m = H(h);
  int rc = check_level(m, level);
  if (rc) return rc;
  auto& L = m->lv[level];
  int64_t inv = 0;
  for (auto& g : L.groups) inv += g->n_patches * g->np * g->ld;
  info[0] = L.n_nodes;
  info[1] = L.ndof();
  info[2] = L.nnzb;
  info[3] = L.nnz_pp;
  info[4] = (int64_t)L.groups.size();
  info[5] = (int64_t)L.Y.n;
  info[6] = inv;
  info[7] = L.groups.empty() ? 0 : L.groups[0]->ld;
  return ALEFSI_OK;
}

int alefsi_gmres(alefsi_mg h, const double* b, double* x, double rel_tol, double abs_tol,
                 int32_t max_iter, int32_t host_ptrs, double* residuals, int32_t* iterations,
                 int32_t* converged) {
  ALEFSI_TRY_BEGIN
  MgHandle* m = H(h);
  if (!m) return fail(ALEFSI_ERR_ARG, "null handle");
  int its = 0, conv = 0;
  int rc = m->gmres(b, x, rel_tol, abs_tol, max_iter, host_ptrs, residuals, &its, &conv);
  *iterations = its;
  *converged = conv;
  return rc;
  ALEFSI_TRY_END
}

int alefsi_gmres_workspace(alefsi_mg h, int32_t max_iter) {
  ALEFSI_TRY_BEGIN
  MgHandle* m = H(h);
  if (!m) return fail(ALEFSI_ERR_ARG, "null handle");
  return m->ensure_workspace(max_iter);
  ALEFSI_TRY_END
}

int alefsi_mg_profile(alefsi_mg h, int32_t on) {
  MgHandle* m = H(h);
  if (!m) return fail(ALEFSI_ERR_ARG, "null handle");
  cudaStreamSynchronize(m->stream);
  m->prof_collect();
  m->prof_on = on != 0;
  return ALEFSI_OK;
}

int alefsi_mg_profile_read(alefsi_mg h, int64_t* counts, double* ms, int32_t reset) {
  MgHandle* m = H(h);
  if (!m) return fail(ALEFSI_ERR_ARG, "null handle");
  cudaStreamSynchronize(m->stream);
  m->prof_collect();
  for (int i = 0; i < 2 * MgHandle::kKinds; ++i) {
    counts[i] = m->prof_count[i];
    ms[i] = m->prof_ms[i];
    if (reset) {
      m->prof_count[i] = 0;
      m->prof_ms[i] = 0.0;
    }
  }
  return ALEFSI_OK;
}

int alefsi_kernel_stats(alefsi_mg h, int64_t* launches) {
  MgHandle* m = H(h);
  if (!m) return fail(ALEFSI_ERR_ARG, "null handle");
  *launches = m->kernel_launches;
  return ALEFSI_OK;
}

}  // extern "C"
