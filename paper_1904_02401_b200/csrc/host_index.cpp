// Host-side (native) index structures for the linear-solve path.
//
// These are the integer/byte parts of the path that must be bit-exact with
// the reference: the block sparsity pattern (reference fem.py:116-146,
// BlockPattern), the element-block scatter-add (fem.py:151-155 / 166-169,
// np.add.at in flattened order), and the greedy first-fit patch coloring
// (reference mesh.py:522-556, color_patches).  They run on the host CPU during
// setup; none of them is on the per-iteration device path.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <vector>

#include "alefsi_common.h"

namespace {

// node -> element adjacency (CSR), elements visited in ascending order
void node_element_adjacency(int64_t n_nodes, int64_t n_elem, const int64_t* elem_ptr,
                            const int64_t* elem_nodes, std::vector<int64_t>& ptr,
                            std::vector<int64_t>& adj) {
  ptr.assign(n_nodes + 1, 0);
  for (int64_t e = 0; e < n_elem; ++e)
    for (int64_t s = elem_ptr[e]; s < elem_ptr[e + 1]; ++s) ptr[elem_nodes[s] + 1]++;
  for (int64_t i = 0; i < n_nodes; ++i) ptr[i + 1] += ptr[i];
  adj.assign(ptr[n_nodes], 0);
  std::vector<int64_t> fill(ptr.begin(), ptr.end() - 1);
  for (int64_t e = 0; e < n_elem; ++e)
    for (int64_t s = elem_ptr[e]; s < elem_ptr[e + 1]; ++s) adj[fill[elem_nodes[s]]++] = e;
}

bool check_nodes(int64_t n_nodes, int64_t n_elem, const int64_t* elem_ptr,
                 const int64_t* elem_nodes) {
  for (int64_t e = 0; e < n_elem; ++e)
    for (int64_t s = elem_ptr[e]; s < elem_ptr[e + 1]; ++s)
      if (elem_nodes[s] < 0 || elem_nodes[s] >= n_nodes) return false;
  return true;
}

template <typename F>
void parallel_rows(int64_t n, F&& f) {
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t i = 0; i < n; ++i) f(i);
}

}  // namespace

extern "C" {

// Union of the element stencils: row i holds every node sharing an element
// with node i, sorted ascending (same order as the reference's sorted
// rows*n+cols keys).  Two-phase: count (indices == nullptr) then fill.
int alefsi_pattern_build(int64_t n_nodes, int64_t n_elem, const int64_t* elem_ptr,
                         const int64_t* elem_nodes, int64_t* indptr, int32_t* indices) {
  ALEFSI_TRY_BEGIN
  if (!check_nodes(n_nodes, n_elem, elem_ptr, elem_nodes))
    return alefsi::fail(ALEFSI_ERR_ARG, "pattern_build: element node out of range");
  std::vector<int64_t> ptr, adj;
  node_element_adjacency(n_nodes, n_elem, elem_ptr, elem_nodes, ptr, adj);
  std::vector<int64_t> counts(n_nodes, 0);
  const bool fill = indices != nullptr;  // fill phase: indptr is an input
  parallel_rows(n_nodes, [&](int64_t i) {
    std::vector<int64_t> row;
    for (int64_t s = ptr[i]; s < ptr[i + 1]; ++s) {
      int64_t e = adj[s];
      for (int64_t t = elem_ptr[e]; t < elem_ptr[e + 1]; ++t) row.push_back(elem_nodes[t]);
    }
    std::sort(row.begin(), row.end());
    row.erase(std::unique(row.begin(), row.end()), row.end());
    if (fill) {
      int32_t* out = indices + indptr[i];
      for (size_t k = 0; k < row.size(); ++k) out[k] = (int32_t)row[k];
    } else {
      counts[i] = (int64_t)row.size();
    }
  });
  if (!fill) {
    indptr[0] = 0;
    for (int64_t i = 0; i < n_nodes; ++i) indptr[i + 1] = indptr[i] + counts[i];
  }
  return ALEFSI_OK;
  ALEFSI_TRY_END
}

// Slot of (row, col) in a sorted CSR row, or -1.
static inline int64_t find_slot(const int64_t* indptr, const int32_t* indices, int64_t row,
                                int64_t col) {
  const int32_t* b = indices + indptr[row];
  const int32_t* e = indices + indptr[row + 1];
  const int32_t* p = std::lower_bound(b, e, (int32_t)col);
  if (p == e || *p != (int32_t)col) return -1;
  return indptr[row] + (p - indices - indptr[row]);
}

// Slots of every (node_a, node_b) pair of homogeneous elements:
// slots[e, a, b] = slot of (elem[e,a], elem[e,b]) or -1 (reference
// fem.py:138-146, slots_for, with -1 instead of the sentinel nnzb).
int alefsi_pattern_slots(int64_t n_nodes, const int64_t* indptr, const int32_t* indices,
                         int64_t n_elem, int32_t npe, const int64_t* elem_nodes,
                         int64_t* slots) {
  ALEFSI_TRY_BEGIN
  parallel_rows(n_elem, [&](int64_t e) {
    const int64_t* nd = elem_nodes + e * npe;
    int64_t* out = slots + e * (int64_t)npe * npe;
    for (int a = 0; a < npe; ++a)
      for (int b = 0; b < npe; ++b) {
        int64_t r = nd[a], c = nd[b];
        out[a * npe + b] = (r < 0 || r >= n_nodes) ? -1 : find_slot(indptr, indices, r, c);
      }
  });
  return ALEFSI_OK;
  ALEFSI_TRY_END
}

// data[slot(elem[e,a], elem[e,b])] += local[e, a, b] (blocks of bs doubles),
// elements and pairs visited in flattened order exactly like np.add.at in
// the reference (fem.py:151-155).  Pairs missing from the pattern are an
// error unless skip_missing is set.
int alefsi_scatter_add_blocks(int64_t n_nodes, const int64_t* indptr, const int32_t* indices,
                              int64_t n_elem, int32_t npe, const int64_t* elem_nodes,
                              int32_t bs, const double* local, double* data,
                              int32_t skip_missing) {
  ALEFSI_TRY_BEGIN
  // Parallel over block rows: every slot of row r is only touched by the
  // elements containing r, visited in ascending element order, so each slot
  // receives its contributions in exactly the sequential (np.add.at) order.
  std::vector<int64_t> eptr(n_elem + 1);
  for (int64_t e = 0; e <= n_elem; ++e) eptr[e] = e * npe;
  if (!check_nodes(n_nodes, n_elem, eptr.data(), elem_nodes))
    return alefsi::fail(ALEFSI_ERR_ARG, "scatter_add_blocks: element node out of range");
  std::vector<int64_t> ptr, adj;
  node_element_adjacency(n_nodes, n_elem, eptr.data(), elem_nodes, ptr, adj);
  int missing = 0;
#pragma omp parallel for schedule(dynamic, 256) reduction(| : missing)
  for (int64_t r = 0; r < n_nodes; ++r) {
    for (int64_t s = ptr[r]; s < ptr[r + 1]; ++s) {
      const int64_t e = adj[s];
      const int64_t* nd = elem_nodes + e * npe;
      const double* loc = local + e * (int64_t)npe * npe * bs;
      for (int a = 0; a < npe; ++a) {
        if (nd[a] != r) continue;
        for (int b = 0; b < npe; ++b) {
          const int64_t slot = find_slot(indptr, indices, r, nd[b]);
          if (slot < 0) {
            missing |= 1;
            continue;
          }
          const double* src = loc + ((int64_t)a * npe + b) * bs;
          double* dst = data + slot * bs;
          for (int k = 0; k < bs; ++k) dst[k] += src[k];
        }
      }
    }
  }
  if (missing && !skip_missing)
    return alefsi::fail(ALEFSI_ERR_ARG, "scatter_add_blocks: pair outside pattern");
  return ALEFSI_OK;
  ALEFSI_TRY_END
}

// For every entry of pattern B (rows sorted): its slot in pattern A or -1.
int alefsi_pattern_match(int64_t n_nodes, const int64_t* a_ptr, const int32_t* a_idx,
                         const int64_t* b_ptr, const int32_t* b_idx, int64_t* slot_in_a) {
  ALEFSI_TRY_BEGIN
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t r = 0; r < n_nodes; ++r) {
    int64_t i = a_ptr[r];
    const int64_t ie = a_ptr[r + 1];
    for (int64_t s = b_ptr[r]; s < b_ptr[r + 1]; ++s) {
      while (i < ie && a_idx[i] < b_idx[s]) ++i;
      slot_in_a[s] = (i < ie && a_idx[i] == b_idx[s]) ? i : -1;
    }
  }
  return ALEFSI_OK;
  ALEFSI_TRY_END
}

// Split of the LPS macro pattern against the cell pattern: entries without a
// cell slot (to_cell < 0) form the pressure-extension pattern, row by row in
// macro order.  pp_indptr (n+1), pp_indices (count), to_pp (len(mind), -1 for
// entries that have a cell slot).  Two parallel passes over the rows.
int alefsi_split_extension(int64_t n_nodes, const int64_t* mptr, const int32_t* mind,
                           const int64_t* to_cell, int64_t* pp_indptr, int32_t* pp_indices,
                           int64_t* to_pp) {
  ALEFSI_TRY_BEGIN
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t r = 0; r < n_nodes; ++r) {
    int64_t c = 0;
    for (int64_t s = mptr[r]; s < mptr[r + 1]; ++s) c += to_cell[s] < 0;
    pp_indptr[r + 1] = c;
  }
  pp_indptr[0] = 0;
  for (int64_t r = 0; r < n_nodes; ++r) pp_indptr[r + 1] += pp_indptr[r];
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t r = 0; r < n_nodes; ++r) {
    int64_t o = pp_indptr[r];
    for (int64_t s = mptr[r]; s < mptr[r + 1]; ++s) {
      if (to_cell[s] < 0) {
        pp_indices[o] = mind[s];
        to_pp[s] = o++;
      } else {
        to_pp[s] = -1;
      }
    }
  }
  return ALEFSI_OK;
  ALEFSI_TRY_END
}

// Greedy first-fit coloring, reference mesh.py:522-556: repeated passes over
// the patches in stored order; in pass c the first unlabeled, unblocked patch
// fixes the color's patch size, every later unlabeled unblocked patch of that
// size receives color c and blocks all patches sharing one of its nodes.
int alefsi_color_patches(int64_t n_patches, const int64_t* patch_ptr, const int64_t* patch_nodes,
                         const int64_t* patch_size, int64_t n_nodes, int64_t* color,
                         int64_t* n_colors) {
  ALEFSI_TRY_BEGIN
  if (!check_nodes(n_nodes, n_patches, patch_ptr, patch_nodes))
    return alefsi::fail(ALEFSI_ERR_ARG, "color_patches: patch node out of range");
  std::vector<int64_t> ptr, adj;
  node_element_adjacency(n_nodes, n_patches, patch_ptr, patch_nodes, ptr, adj);
  for (int64_t i = 0; i < n_patches; ++i) color[i] = -1;
  std::vector<uint8_t> blocked(n_patches);
  int64_t remaining = n_patches, c = 0;
  while (remaining > 0) {
    std::fill(blocked.begin(), blocked.end(), 0);
    bool have_size = false;
    int64_t size_of_color = 0;
    for (int64_t i = 0; i < n_patches; ++i) {
      if (color[i] >= 0 || blocked[i]) continue;
      if (!have_size) {
        size_of_color = patch_size[i];
        have_size = true;
      }
      if (patch_size[i] != size_of_color) continue;
      color[i] = c;
      --remaining;
      for (int64_t s = patch_ptr[i]; s < patch_ptr[i + 1]; ++s) {
        int64_t nd = patch_nodes[s];
        for (int64_t t = ptr[nd]; t < ptr[nd + 1]; ++t) blocked[adj[t]] = 1;
      }
    }
    ++c;
  }
  *n_colors = c;
  return ALEFSI_OK;
  ALEFSI_TRY_END
}

}  // extern "C"
