// Device kernels of the MG-GMRES / Vanka linear-solve path, sm_100a, FP64.
//
// Every kernel here is HBM- (or L2-) bandwidth bound: the operator is a
// block-sparse FEM stencil and the smoother is a batch of distinct small
// dense inverses, so there is no GEMM-shaped work for the tensor cores.
// Design rules followed throughout: coalesced 16-byte streaming loads with
// evict-first hints for data read once per sweep (operator blocks, patch
// inverses), read-only-path loads for vectors reused from L2, and fixed-order
// reductions so that every result is bitwise reproducible run to run.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <algorithm>
#include <cstdlib>

#include "device_kernels.cuh"

namespace alefsi {

namespace {

constexpr int kWarp = 32;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Fixed-shape block reduction (blockDim.x == 256): deterministic.
__device__ __forceinline__ double block_sum_256(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double r = 0.0;
  if (w == 0) {
    r = l < 8 ? red[l] : 0.0;
    r = warp_sum(r);
  }
  return r;  // valid in thread 0
}

// 32-byte quads usable: length and stride multiples of 4, aligned base
inline bool vec4_ok(const double* p, int64_t ld, int64_t n) {
  return n % 4 == 0 && ld % 4 == 0 && reinterpret_cast<uintptr_t>(p) % 32 == 0;
}

// levels below this many nodes are L2 resident and latency bound
constexpr int64_t kSmallLevelNodes = 65536;
// patch launches below this many patches use the column-split apply
constexpr int64_t kSmallPatchCount = 8192;

inline int grid_for(int64_t n, int per_block) { return (int)((n + per_block - 1) / per_block); }

// Programmatic dependent launch: kernels of the solve path are launched with
// programmaticStreamSerialization, so a kernel's CTAs may be scheduled while
// its predecessor on the stream (or graph edge) drains.  pdl_entry() lets the
// next kernel launch early and then waits until the predecessor's grid has
// completed and its memory is visible — before this kernel reads or writes
// anything — so the ordering is the plain stream order minus the launch gap.
__device__ __forceinline__ void pdl_entry() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, Args... args) {
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// --------------------------------------------------------------------------
// Block-sparse matrix-vector product.  One warp per block row (mesh node).
// NC = 4: lane = 4*blk + r, each lane streams one 32-byte block row
// (2 x 16-byte loads), 8 blocks = 1 KiB per warp iteration; rows are summed
// with xor-shuffles over lanes sharing r.  NC = 3: lane = 3*blk + r over 30
// lanes, 8-byte loads (blocks are 72 bytes), per-r butterfly reductions.
// The scalar pressure extension L is swept by the same warp afterwards.
// --------------------------------------------------------------------------
template <int NC, int MODE>
__global__ void __launch_bounds__(256) spmv_kernel(int64_t n, const int64_t* __restrict__ indptr,
                                                   const int32_t* __restrict__ indices,
                                                   const double* __restrict__ data,
                                                   const int64_t* __restrict__ pp_ptr,
                                                   const int32_t* __restrict__ pp_idx,
                                                   const double* __restrict__ pp_val,
                                                   const double* __restrict__ x,
                                                   const double* __restrict__ b,
                                                   double* __restrict__ y) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (row >= n) return;
  constexpr int BPI = kWarp / NC;  // blocks per warp iteration
  const int r = lane % NC;
  const int sub = lane / NC;
  const int64_t beg = indptr[row], end = indptr[row + 1];
  double acc = 0.0;
  // (a 4-way manually unrolled variant measured 16% slower: the extra
  // registers cost occupancy, and 64 warps/SM already cover the latency)
  if (sub < BPI) {
    for (int64_t blk = beg + sub; blk < end; blk += BPI) {
      const int64_t col = __ldcs(indices + blk);
      const double* v = data + blk * (NC * NC) + r * NC;
      const double* xv = x + col * NC;
      if constexpr (NC % 2 == 0) {
#pragma unroll
        for (int c = 0; c < NC / 2; ++c) {
          const double2 vv = __ldcs(reinterpret_cast<const double2*>(v) + c);
          const double2 xx = __ldg(reinterpret_cast<const double2*>(xv) + c);
          acc = fma(vv.x, xx.x, acc);
          acc = fma(vv.y, xx.y, acc);
        }
      } else {
#pragma unroll
        for (int c = 0; c < NC; ++c) acc = fma(__ldcs(v + c), __ldg(xv + c), acc);
      }
    }
  }
  // pressure extension: sum_e L[row, e] * x[col_e, 0]
  double accp = 0.0;
  if (pp_ptr != nullptr) {
    const int64_t pb = pp_ptr[row], pe = pp_ptr[row + 1];
    for (int64_t e = pb + lane; e < pe; e += kWarp)
      accp = fma(__ldcs(pp_val + e), __ldg(x + (int64_t)__ldcs(pp_idx + e) * NC), accp);
    accp = warp_sum(accp);
  }
  double out[NC];
  if constexpr (kWarp % NC == 0) {
#pragma unroll
    for (int o = NC; o < kWarp; o <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    // lanes 0..NC-1 now hold rows 0..NC-1
    if (lane < NC) {
      double v = acc + (lane == 0 ? accp : 0.0);
      const int64_t o = row * NC + lane;
      y[o] = MODE == 1 ? b[o] - v : v;
    }
  } else {
#pragma unroll
    for (int rr = 0; rr < NC; ++rr) out[rr] = warp_sum((r == rr && sub < BPI) ? acc : 0.0);
    if (lane < NC) {
      double v = out[0];
#pragma unroll
      for (int rr = 1; rr < NC; ++rr)
        if (lane == rr) v = out[rr];
      if (lane == 0) v += accp;
      const int64_t o = row * NC + lane;
      y[o] = MODE == 1 ? b[o] - v : v;
    }
  }
}

// Even block size with 32-bit block/entry offsets (nnzb * NC^2 < 2^31): same
// lane mapping as spmv_kernel, fewer integer instructions per byte streamed —
// the kernel is partly issue-limited when the 1 kW power cap lowers SM clocks.
template <int NC, int MODE>
__global__ void __launch_bounds__(256) spmv32_kernel(int64_t n, const int64_t* __restrict__ indptr,
                                                     const int32_t* __restrict__ indices,
                                                     const double* __restrict__ data,
                                                     const int64_t* __restrict__ pp_ptr,
                                                     const int32_t* __restrict__ pp_idx,
                                                     const double* __restrict__ pp_val,
                                                     const double* __restrict__ x,
                                                     const double* __restrict__ b,
                                                     double* __restrict__ y) {
  pdl_entry();
  static_assert(NC % 2 == 0 && kWarp % NC == 0, "even block size");
  constexpr int BPI = kWarp / NC, H = NC / 2;
  const int lane = threadIdx.x & 31;
  const int row = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (row >= n) return;
  const int r = lane % NC, sub = lane / NC;
  const int beg = (int)indptr[row], end = (int)indptr[row + 1];
  const double2* d2 = reinterpret_cast<const double2*>(data) + r * H;
  const double2* x2 = reinterpret_cast<const double2*>(x);
  double acc = 0.0;
  for (int blk = beg + sub; blk < end; blk += BPI) {
    const int col = __ldcs(indices + blk);
#pragma unroll
    for (int c = 0; c < H; ++c) {
      const double2 vv = __ldcs(d2 + blk * (NC * H) + c);
      const double2 xx = __ldg(x2 + col * H + c);
      acc = fma(vv.x, xx.x, acc);
      acc = fma(vv.y, xx.y, acc);
    }
  }
  double accp = 0.0;
  if (pp_ptr != nullptr) {
    const int pb = (int)pp_ptr[row], pe = (int)pp_ptr[row + 1];
    for (int e = pb + lane; e < pe; e += kWarp)
      accp = fma(__ldcs(pp_val + e), __ldg(x + __ldcs(pp_idx + e) * NC), accp);
    accp = warp_sum(accp);
  }
#pragma unroll
  for (int o = NC; o < kWarp; o <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane < NC) {
    const double v = acc + (lane == 0 ? accp : 0.0);
    const int o = row * NC + lane;
    y[o] = MODE == 1 ? b[o] - v : v;
  }
}

// 256-bit global loads (sm_100): one LDG.256 per block row and per x block.
struct d4 {
  double x, y, z, w;
};
__device__ __forceinline__ d4 ld256_stream(const double* p) {   // streamed: evict-first in L2
  d4 v;
  asm("ld.global.L1::no_allocate.L2::evict_first.v4.f64 {%0,%1,%2,%3}, [%4];"
      : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ d4 ld256_ro(const double* p) {       // read-only path
  d4 v;
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
      : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}

// NC = 4 with 32-bit offsets: lane = 4*blk + r loads its whole 32-byte block
// row and the 32-byte x block with one instruction each (half the load
// instructions of spmv32_kernel; same FMA order, bitwise-equal results).
//
// Block columns are fetched 32 at a time with one coalesced load and handed
// out by shuffle, so the x gather of an iteration waits on L2 only.
//
// UNR: the four column steps of a 32-block chunk are unrolled so their loads
// are in flight together.  Used on small, L2-resident levels, where a
// warp's chain of dependent L2 round trips (not resident warps) sets the
// time; the large levels keep one step at a time for 32 registers and full
// occupancy.  Same FMA order either way: bitwise-equal results.
template <int MODE, bool UNR = false>
__global__ void __launch_bounds__(256) spmv4_kernel(int64_t n, const int64_t* __restrict__ indptr,
                                                       const int32_t* __restrict__ indices,
                                                       const double* __restrict__ data,
                                                       const int64_t* __restrict__ pp_ptr,
                                                       const int32_t* __restrict__ pp_idx,
                                                       const double* __restrict__ pp_val,
                                                       const double* __restrict__ x,
                                                       const double* __restrict__ b,
                                                       double* __restrict__ y) {
  pdl_entry();
  constexpr int NC = 4, BPI = kWarp / NC;
  const int lane = threadIdx.x & 31;
  const int row = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (row >= n) return;
  const int r = lane % NC, sub = lane / NC;
  const int beg = (int)indptr[row], end = (int)indptr[row + 1];
  const double* dr = data + r * NC;
  double acc = 0.0;
  for (int base = beg; base < end; base += kWarp) {
    const int cidx = base + lane < end ? __ldcs(indices + base + lane) : 0;
#pragma unroll (UNR ? 4 : 1)
    for (int j = 0; j < kWarp / BPI; ++j) {
      const int col = __shfl_sync(0xffffffffu, cidx, j * BPI + sub);
      const int blk = base + j * BPI + sub;
      if (blk < end) {
        const d4 vv = ld256_stream(dr + blk * (NC * NC));
        const d4 xx = ld256_ro(x + col * NC);
        acc = fma(vv.x, xx.x, acc);
        acc = fma(vv.y, xx.y, acc);
        acc = fma(vv.z, xx.z, acc);
        acc = fma(vv.w, xx.w, acc);
      }
    }
  }
  double accp = 0.0;
  if (pp_ptr != nullptr) {
    const int pb = (int)pp_ptr[row], pe = (int)pp_ptr[row + 1];
    for (int e = pb + lane; e < pe; e += kWarp)
      accp = fma(__ldcs(pp_val + e), __ldg(x + __ldcs(pp_idx + e) * NC), accp);
    accp = warp_sum(accp);
  }
#pragma unroll
  for (int o = NC; o < kWarp; o <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane < NC) {
    const double v = acc + (lane == 0 ? accp : 0.0);
    const int o = row * NC + lane;
    y[o] = MODE == 1 ? b[o] - v : v;
  }
}

// Half-warp per block row for the short 2D rows (NC = 3, ~16 blocks + ~19
// pressure-extension entries): lane = 3*blk + r over 15 of 16 lanes, two
// independent rows per warp double the loads in flight per warp.
template <int NC, int MODE>
__global__ void __launch_bounds__(256) spmv_half_kernel(int64_t n, const int64_t* __restrict__ indptr,
                                                        const int32_t* __restrict__ indices,
                                                        const double* __restrict__ data,
                                                        const int64_t* __restrict__ pp_ptr,
                                                        const int32_t* __restrict__ pp_idx,
                                                        const double* __restrict__ pp_val,
                                                        const double* __restrict__ x,
                                                        const double* __restrict__ b,
                                                        double* __restrict__ y) {
  pdl_entry();
  constexpr int HL = 16, BPI = HL / NC;
  const int lane = threadIdx.x & 31, hl = lane & (HL - 1);
  const unsigned hmask = (lane < HL) ? 0x0000ffffu : 0xffff0000u;
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 4;
  if (row >= n) return;     // both halves of a warp exit together only at the tail
  const int r = hl % NC, sub = hl / NC;
  const int64_t beg = indptr[row], end = indptr[row + 1];
  double acc = 0.0;
  if (sub < BPI) {
    for (int64_t blk = beg + sub; blk < end; blk += BPI) {
      const int64_t col = __ldcs(indices + blk);
      const double* v = data + blk * (NC * NC) + r * NC;
      const double* xv = x + col * NC;
#pragma unroll
      for (int c = 0; c < NC; ++c) acc = fma(__ldcs(v + c), __ldg(xv + c), acc);
    }
  }
  double accp = 0.0;
  if (pp_ptr != nullptr)
    for (int64_t e = pp_ptr[row] + hl; e < pp_ptr[row + 1]; e += HL)
      accp = fma(__ldcs(pp_val + e), __ldg(x + (int64_t)__ldcs(pp_idx + e) * NC), accp);
  double out[NC];
#pragma unroll
  for (int rr = 0; rr < NC; ++rr) {
    double v = (r == rr && sub < BPI) ? acc : 0.0;
    if (rr == 0) v += accp;
#pragma unroll
    for (int o = HL / 2; o > 0; o >>= 1) v += __shfl_xor_sync(hmask, v, o, HL);
    out[rr] = v;
  }
  if (hl < NC) {
    double v = out[0];
#pragma unroll
    for (int rr = 1; rr < NC; ++rr)
      if (hl == rr) v = out[rr];
    const int64_t o = row * NC + hl;
    y[o] = MODE == 1 ? b[o] - v : v;
  }
}

// 2D (NC = 3) operator in sliced-ELL form: warp = one slice of R = 32 / T
// consecutive block rows, T lanes per row taking the row's slots round-robin
// (T = 1: lane = row, slots in pattern order).  Every element plane of a
// slot is one coalesced R*8-byte segment (a warp load covers T consecutive
// slots, evict-first), the columns an R*4-byte segment; x is read through
// the read-only path (x stays L2-resident).  A lane sums its slots in order,
// its row's pressure-extension entries likewise; the T partial sums are
// combined by xor-shuffles.  Padding slots hold zeros and a valid column.
template <int MODE, int T>
__global__ void __launch_bounds__(256) spmv3_sell_kernel(int64_t n, int64_t n_slices,
                                                         const int64_t* __restrict__ off,
                                                         const int32_t* __restrict__ col,
                                                         const double* __restrict__ val,
                                                         const int64_t* __restrict__ poff,
                                                         const int32_t* __restrict__ pcol,
                                                         const double* __restrict__ pval,
                                                         const double* __restrict__ x,
                                                         const double* __restrict__ b,
                                                         double* __restrict__ y) {
  pdl_entry();
  constexpr int NC = 3, R = 32 / T;
  const int lane = threadIdx.x & 31, q = lane % R, h = lane / R;
  const int64_t sl = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (sl >= n_slices) return;
  const int64_t row = sl * R + q;
  const int64_t g0 = off[sl], g1 = off[sl + 1];
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll 2
  for (int64_t g = g0 + h; g < g1; g += T) {
    const int c = __ldcs(col + g * R + q);
    const double* v = val + g * (NC * NC * R) + q;
    double e[NC * NC];
#pragma unroll
    for (int k = 0; k < NC * NC; ++k) e[k] = __ldcs(v + k * R);
    const double x0 = __ldg(x + (int64_t)c * NC), x1 = __ldg(x + (int64_t)c * NC + 1),
                 x2 = __ldg(x + (int64_t)c * NC + 2);
    a0 = fma(e[0], x0, a0); a0 = fma(e[1], x1, a0); a0 = fma(e[2], x2, a0);
    a1 = fma(e[3], x0, a1); a1 = fma(e[4], x1, a1); a1 = fma(e[5], x2, a1);
    a2 = fma(e[6], x0, a2); a2 = fma(e[7], x1, a2); a2 = fma(e[8], x2, a2);
  }
  if (poff != nullptr) {
    double ap = 0.0;
    const int64_t p0 = poff[sl], p1 = poff[sl + 1];
#pragma unroll 4
    for (int64_t g = p0 + h; g < p1; g += T)
      ap = fma(__ldcs(pval + g * R + q), __ldg(x + (int64_t)__ldcs(pcol + g * R + q) * NC), ap);
    a0 += ap;
  }
#pragma unroll
  for (int o = R; o < 32; o <<= 1) {
    a0 += __shfl_xor_sync(0xffffffffu, a0, o);
    a1 += __shfl_xor_sync(0xffffffffu, a1, o);
    a2 += __shfl_xor_sync(0xffffffffu, a2, o);
  }
  if (h != 0 || row >= n) return;
  const int64_t o = row * NC;
  if (MODE == 1) {
    y[o] = b[o] - a0;
    y[o + 1] = b[o + 1] - a1;
    y[o + 2] = b[o + 2] - a2;
  } else {
    y[o] = a0;
    y[o + 1] = a1;
    y[o + 2] = a2;
  }
}

__global__ void sell_pack_kernel(int64_t n_pos, int R, int nc2, const int64_t* __restrict__ map,
                                 const double* __restrict__ data, double* __restrict__ val) {
  for (int64_t pos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pos < n_pos;
       pos += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = map[pos];
    const int64_t g = pos / R, q = pos - g * R;
    double* out = val + g * nc2 * R + q;
    for (int k = 0; k < nc2; ++k) out[k * R] = m >= 0 ? data[m * nc2 + k] : 0.0;
  }
}

// --------------------------------------------------------------------------
// Vanka apply: Y[p] = A_p^{-1} d[dofs_p].  Inverses are stored column-major
// with an even column length LD, so thread t of a patch owns rows
// RPT*t .. RPT*t+RPT-1 and streams one 16-byte (RPT = 2) or 32-byte (RPT = 4,
// LD % 4 == 0, 32-byte aligned storage) piece per column: a patch column is
// one contiguous LD*8-byte run, read exactly once per sweep with evict-first
// loads.  The patch defect is staged in shared memory and broadcast.
// --------------------------------------------------------------------------
template <int LD, int RPT>
struct ApplyShape {
  static constexpr int TPP = ((LD / RPT + 31) / 32) * 32;  // threads per patch
  static constexpr int BLK = TPP > 128 ? TPP : 128;        // CTA size
  static constexpr int PPC = BLK / TPP;                    // patches per CTA
};

// Up to two patch groups of the same shape (the fluid and the solid patches
// of a level) in one launch: CTAs [0, blocks0) serve group 0, the rest group
// 1, so the small solid group runs alongside the fluid group instead of as
// its own latency-bound launch.
struct ApplyGroups {
  int64_t n_patches[2];
  const int32_t* nodes[2];
  const double* inv[2];
  double* y[2];
  int blocks0;
};

template <int NP, int LD, int NC, int RPT>
__global__ void __launch_bounds__(ApplyShape<LD, RPT>::BLK) vanka_apply_kernel(
    ApplyGroups G, const double* __restrict__ d) {
  pdl_entry();
  constexpr int NPN = NP / NC;
  constexpr int TPP = ApplyShape<LD, RPT>::TPP;
  constexpr int PPC = ApplyShape<LD, RPT>::PPC;
  static_assert(PPC >= 1, "patch too large for one CTA");
  static_assert(LD % RPT == 0 && (RPT == 2 || RPT == 4), "row split");
  __shared__ double ds[PPC][LD];
  const int gi = blockIdx.x >= (unsigned)G.blocks0 ? 1 : 0;
  const int64_t n_patches = G.n_patches[gi];
  const int32_t* __restrict__ nodes = G.nodes[gi];
  const double* __restrict__ inv = G.inv[gi];
  double* __restrict__ Y = G.y[gi];
  const int sub = threadIdx.x / TPP, t = threadIdx.x % TPP;
  const int64_t p = (int64_t)(blockIdx.x - (gi ? G.blocks0 : 0)) * PPC + sub;
  const bool valid = p < n_patches;
  if (valid) {
    for (int j = t; j < NP; j += TPP) {
      const int a = j / NC, c = j - a * NC;
      ds[sub][j] = __ldg(d + (int64_t)__ldg(nodes + p * NPN + a) * NC + c);
    }
  }
  __syncthreads();
  if (!valid || RPT * t >= LD) return;
  const double* col = inv + p * (int64_t)(NP * LD) + RPT * t;
  double* out = Y + p * (int64_t)LD + RPT * t;
  if constexpr (RPT == 2) {
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll 12
    for (int j = 0; j < NP; ++j) {
      const double2 v = __ldcs(reinterpret_cast<const double2*>(col + j * LD));
      const double dj = ds[sub][j];
      acc.x = fma(v.x, dj, acc.x);
      acc.y = fma(v.y, dj, acc.y);
    }
    *reinterpret_cast<double2*>(out) = acc;
  } else {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll 12
    for (int j = 0; j < NP; ++j) {
      const d4 v = ld256_stream(col + j * LD);
      const double dj = ds[sub][j];
      a0 = fma(v.x, dj, a0);
      a1 = fma(v.y, dj, a1);
      a2 = fma(v.z, dj, a2);
      a3 = fma(v.w, dj, a3);
    }
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(out), "d"(a0), "d"(a1), "d"(a2),
                 "d"(a3)
                 : "memory");
  }
}

// Small patch groups (coarse levels): S thread groups per patch split the
// column range, partial results combined in fixed order through shared
// memory — a quarter of the dependent load rounds per thread when there are
// too few patches to fill the GPU.
template <int NP, int LD, int NC, int RPT, int S>
__global__ void __launch_bounds__(ApplyShape<LD, RPT>::TPP * S) vanka_apply_split_kernel(
    ApplyGroups G, const double* __restrict__ d) {
  pdl_entry();
  constexpr int NPN = NP / NC;
  constexpr int TPP = ApplyShape<LD, RPT>::TPP;
  constexpr int CPS = (NP + S - 1) / S;   // columns per split
  __shared__ double ds[LD];
  __shared__ double part[S][LD];
  const int gi = blockIdx.x >= (unsigned)G.blocks0 ? 1 : 0;
  const int32_t* __restrict__ nodes = G.nodes[gi];
  const double* __restrict__ inv = G.inv[gi];
  double* __restrict__ Y = G.y[gi];
  const int64_t p = (int64_t)(blockIdx.x - (gi ? G.blocks0 : 0));
  if (p >= G.n_patches[gi]) return;
  for (int j = threadIdx.x; j < NP; j += TPP * S) {
    const int a = j / NC, c = j - a * NC;
    ds[j] = __ldg(d + (int64_t)__ldg(nodes + p * NPN + a) * NC + c);
  }
  __syncthreads();
  const int sp = threadIdx.x / TPP, t = threadIdx.x % TPP;
  const bool rows_ok = RPT * t < LD;
  double acc[RPT];
#pragma unroll
  for (int r = 0; r < RPT; ++r) acc[r] = 0.0;
  if (rows_ok) {
    const double* col = inv + p * (int64_t)(NP * LD) + RPT * t;
    const int j0 = sp * CPS, j1 = min(NP, j0 + CPS);
#pragma unroll 9
    for (int j = j0; j < j1; ++j) {
      const double dj = ds[j];
      if constexpr (RPT == 4) {
        const d4 v = ld256_stream(col + j * LD);
        acc[0] = fma(v.x, dj, acc[0]);
        acc[1] = fma(v.y, dj, acc[1]);
        acc[2] = fma(v.z, dj, acc[2]);
        acc[3] = fma(v.w, dj, acc[3]);
      } else {
        const double2 v = __ldcs(reinterpret_cast<const double2*>(col + j * LD));
        acc[0] = fma(v.x, dj, acc[0]);
        acc[1] = fma(v.y, dj, acc[1]);
      }
    }
#pragma unroll
    for (int r = 0; r < RPT; ++r) part[sp][RPT * t + r] = acc[r];
  }
  __syncthreads();
  if (sp != 0 || !rows_ok) return;
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    double v = part[0][RPT * t + r];
#pragma unroll
    for (int q = 1; q < S; ++q) v += part[q][RPT * t + r];
    Y[p * (int64_t)LD + RPT * t + r] = v;
  }
}

// Deterministic scatter-add of the weighted patch corrections: each dof sums
// its patches' rows in ascending patch order (the reference's np.add.at
// order, linsolve.py:171-178) and applies x + omega * upd.
__global__ void vanka_gather_kernel(int64_t ndof, int nc, const int64_t* __restrict__ gptr,
                                    const int64_t* __restrict__ goff,
                                    const double* __restrict__ w, const double* __restrict__ Y,
                                    double* __restrict__ x, double omega, int init_zero) {
  pdl_entry();
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ndof) return;
  const int64_t n = t / nc;
  const int c = (int)(t - n * nc);
  const double wn = __ldg(w + n);
  double acc = 0.0;
  for (int64_t s = gptr[n]; s < gptr[n + 1]; ++s)
    acc = __dadd_rn(acc, __dmul_rn(wn, __ldg(Y + goff[s] + c)));
  const double base = init_zero ? 0.0 : x[t];
  x[t] = __dadd_rn(base, __dmul_rn(omega, acc));
}

// NC = 4: one thread per node sums the node's 4 components together — one
// 32-byte load of Y per (patch, local node) slot (slots are 4-aligned: every
// patch column length and group offset is a multiple of 4) and one 32-byte
// load / store of x.  Per component the same operations in the same order
// as vanka_gather_kernel: bitwise-identical x.
__global__ void vanka_gather4_kernel(int64_t n_nodes, const int64_t* __restrict__ gptr,
                                     const int64_t* __restrict__ goff,
                                     const double* __restrict__ w, const double* __restrict__ Y,
                                     double* __restrict__ x, double omega, int init_zero) {
  pdl_entry();
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= n_nodes) return;
  const double wn = __ldg(w + n);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  const int64_t sb = gptr[n], se = gptr[n + 1];
  // four slots' offsets, then their four Y loads, in flight together
  for (int64_t s = sb; s < se; s += 4) {
    d4 y[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      y[u] = d4{0.0, 0.0, 0.0, 0.0};
      if (s + u < se) y[u] = ld256_ro(Y + __ldg(goff + s + u));
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (s + u < se) {
        a0 = __dadd_rn(a0, __dmul_rn(wn, y[u].x));
        a1 = __dadd_rn(a1, __dmul_rn(wn, y[u].y));
        a2 = __dadd_rn(a2, __dmul_rn(wn, y[u].z));
        a3 = __dadd_rn(a3, __dmul_rn(wn, y[u].w));
      }
    }
  }
  double* xn = x + 4 * n;
  d4 base{0.0, 0.0, 0.0, 0.0};
  if (!init_zero) base = ld256_ro(xn);
  const double o0 = __dadd_rn(base.x, __dmul_rn(omega, a0));
  const double o1 = __dadd_rn(base.y, __dmul_rn(omega, a1));
  const double o2 = __dadd_rn(base.z, __dmul_rn(omega, a2));
  const double o3 = __dadd_rn(base.w, __dmul_rn(omega, a3));
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(xn), "d"(o0), "d"(o1), "d"(o2),
               "d"(o3)
               : "memory");
}

template <int I>
struct IntC {
  static constexpr int value = I;
};

// Gauss-Jordan inversion of every patch matrix with implicit partial
// pivoting, one CTA of W warps per NPAT patches.  Rows are never swapped:
// step k pivots on the largest unused row p_k of column k (the pivot LAPACK's
// getrf would choose, lowest index on ties), and at the end
//     inv[q(r)][p_c] = R[r][c],   q = p^{-1},
// which is written directly in the column-major (ld) layout.
// Warp w owns the strided column set {w + W*j} of every row ty + 32*i (lane
// ty), in registers.  The warp owning column k+1 publishes it and picks the
// next pivot with a warp-local argmax right after its own share of the
// step-k elimination, overlapped with the other warps' eliminations: two
// block barriers per pivot step, no single-warp phase on the critical path.
// Used for the small patch sizes (18, 27, 81); 75 and 108 use the second form
// below.
template <int NP, int NC, int W, int NPAT>
__global__ void __launch_bounds__(32 * W) vanka_factorize_cw_kernel(
    DevMatrix A, int64_t n_patches, const int32_t* __restrict__ nodes, double* __restrict__ inv,
    int ld, int64_t* status) {
  constexpr int NPN = NP / NC, RT = (NP + 31) / 32, CT = (NP + W - 1) / W, NT = 32 * W;
  static_assert(RT <= 4, "pivot-row scaling covers up to 4 register rows");
  constexpr int NR = 32 * RT, NCOL = W * CT;               // padded row / column counts
  __shared__ int32_t slotB[NPAT][NPN * NPN], slotP[NPAT][NPN * NPN];
  __shared__ double colk[NPAT][2][NR], prow[NPAT][NCOL], pivval[NPAT];
  __shared__ int used[NPAT][NP], piv_of_step[NPAT][NP], step_of_row[NPAT][NP];
  const int tid = threadIdx.x, ty = tid & 31, w = tid >> 5;
  for (int i = tid; i < NPAT * 2 * NR; i += NT) (&colk[0][0][0])[i] = 0.0;
  for (int i = tid; i < NPAT * NCOL; i += NT) (&prow[0][0])[i] = 0.0;
  int64_t pid[NPAT];
  bool live[NPAT];
#pragma unroll
  for (int q = 0; q < NPAT; ++q) {
    pid[q] = (int64_t)blockIdx.x * NPAT + q;
    live[q] = pid[q] < n_patches;
  }
#pragma unroll
  for (int q = 0; q < NPAT; ++q) {
    if (!live[q]) continue;
    const int32_t* pn = nodes + pid[q] * NPN;
    for (int t = tid; t < NPN * NPN; t += NT) {
      const int a = t / NPN, b = t - a * NPN;
      const int64_t ra = pn[a];
      const int32_t cb = pn[b];
      int64_t lo = A.indptr[ra], hi = A.indptr[ra + 1];
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (A.indices[mid] < cb) lo = mid + 1; else hi = mid;
      }
      slotB[q][t] = (lo < A.indptr[ra + 1] && A.indices[lo] == cb) ? (int32_t)lo : -1;
      int64_t sp = -1;
      if (slotB[q][t] < 0 && A.pp_indptr != nullptr) {
        lo = A.pp_indptr[ra];
        hi = A.pp_indptr[ra + 1];
        while (lo < hi) {
          const int64_t mid = (lo + hi) >> 1;
          if (A.pp_indices[mid] < cb) lo = mid + 1; else hi = mid;
        }
        if (lo < A.pp_indptr[ra + 1] && A.pp_indices[lo] == cb) sp = lo;
      }
      slotP[q][t] = (int32_t)sp;
    }
  }
  for (int i = tid; i < NPAT * NP; i += NT) used[i / NP][i % NP] = 0;
  __syncthreads();
  double M[NPAT][RT][CT];
#pragma unroll
  for (int q = 0; q < NPAT; ++q)
#pragma unroll
    for (int i = 0; i < RT; ++i)
#pragma unroll
      for (int j = 0; j < CT; ++j) {
        const int r = ty + 32 * i, c = w + W * j;
        double v = (r == c) ? 1.0 : 0.0;          // identity for a missing tail patch
        if (live[q] && r < NP && c < NP) {
          const int a = r / NC, ci = r - a * NC, b = c / NC, cj = c - b * NC;
          const int t = a * NPN + b;
          v = 0.0;
          if (slotB[q][t] >= 0) v = A.data[(int64_t)slotB[q][t] * (NC * NC) + ci * NC + cj];
          else if (ci == 0 && cj == 0 && slotP[q][t] >= 0) v = A.pp_data[slotP[q][t]];
        }
        M[q][i][j] = v;
      }
  // owner warp of column k: publish it and choose its pivot (largest |.| of
  // the unused rows, lowest index on ties)
  auto owner_step = [&](int k) {
    if (w != k % W) return;
    const int jk = k / W;
#pragma unroll
    for (int q = 0; q < NPAT; ++q) {
      double best = -1.0;
      int bi = NP;
#pragma unroll
      for (int i = 0; i < RT; ++i) {
        const int r = ty + 32 * i;
        double v = 0.0;
#pragma unroll
        for (int j = 0; j < CT; ++j) {
          if (j == jk) v = M[q][i][j];
          // column k restarts from 0: the elimination's fma then yields
          // -f * (1/pivot) there, with no per-element select
          M[q][i][j] = (j == jk) ? 0.0 : M[q][i][j];
        }
        if (r < NP) {
          colk[q][k & 1][r] = v;
          const double a = used[q][r] ? -1.0 : fabs(v);
          if (a > best) { best = a; bi = r; }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      __syncwarp();
      if (ty == 0) {
        used[q][bi] = 1;
        piv_of_step[q][k] = bi;
        step_of_row[q][bi] = k;
        // the pivot leaves the published column: f = 0 on the pivot row
        // makes the elimination below select-free
        pivval[q] = colk[q][k & 1][bi];
        colk[q][k & 1][bi] = 0.0;
      }
    }
  };
  owner_step(0);
  for (int k = 0; k < NP; ++k) {
    __syncthreads();
    int pr[NPAT];
    double rp[NPAT];
#pragma unroll
    for (int q = 0; q < NPAT; ++q) {
      pr[q] = piv_of_step[q][k];
      const double piv = pivval[q];
      if (piv == 0.0 && live[q] && tid == 0)
        atomicCAS(reinterpret_cast<unsigned long long*>(status), 0ull,
                  (unsigned long long)(pid[q] + 1));
      rp[q] = piv != 0.0 ? 1.0 / piv : 0.0;   // singular: reported, result unused
      // one lane per warp holds the pivot row's elements of its columns; a
      // branch per register row keeps the scaling straight-line code
      if (ty == (pr[q] & 31)) {
        auto scale = [&](auto I) {
          constexpr int i = decltype(I)::value;
#pragma unroll
          for (int j = 0; j < CT; ++j) {
            const int c = w + W * j;
            const double v = (c == k) ? rp[q] : M[q][i][j] * rp[q];
            M[q][i][j] = v;
            if (c < NP) prow[q][c] = v;
          }
        };
        switch (pr[q] >> 5) {
          case 0: scale(IntC<0>{}); break;
          case 1: if constexpr (RT > 1) scale(IntC<1>{}); break;
          case 2: if constexpr (RT > 2) scale(IntC<2>{}); break;
          default: if constexpr (RT > 3) scale(IntC<3>{}); break;
        }
      }
    }
    __syncthreads();
    // branch-free elimination: padded rows hold f = 0 (colk zero-padded),
    // padded columns multiply a zero prow entry, the pivot row keeps its
    // scaled values through f = 0 (its colk entry is cleared by the owner),
    // and column k (zeroed by its owner, pivot entry 1/pivot in prow)
    // becomes -f/pivot
#pragma unroll
    for (int q = 0; q < NPAT; ++q) {
      const double* ck = colk[q][k & 1];
      double pv[CT];
#pragma unroll
      for (int j = 0; j < CT; ++j) pv[j] = prow[q][w + W * j];
#pragma unroll
      for (int i = 0; i < RT; ++i) {
        const double nf = -ck[ty + 32 * i];
#pragma unroll
        for (int j = 0; j < CT; ++j) M[q][i][j] = fma(nf, pv[j], M[q][i][j]);
      }
    }
    if (k + 1 < NP) owner_step(k + 1);
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NPAT; ++q) {
    if (!live[q]) continue;
    double* out = inv + pid[q] * (int64_t)NP * ld;
#pragma unroll
    for (int i = 0; i < RT; ++i)
#pragma unroll
      for (int j = 0; j < CT; ++j) {
        const int r = ty + 32 * i, c = w + W * j;
        if (r < NP && c < NP)
          out[(int64_t)piv_of_step[q][c] * ld + step_of_row[q][r]] = M[q][i][j];
      }
    if (ld > NP)
      for (int col = tid; col < NP; col += NT)
        for (int r = NP; r < ld; ++r) out[(int64_t)col * ld + r] = 0.0;
  }
}


// Operator slots of every (row node, column node) pair of every patch, found
// once per sparsity pattern: >= 0 block slot, <= -2 pressure-extension entry
// -(v + 2), -1 structurally zero (the reference's pattern.slots_for,
// linsolve.py:124-126).  The factorisation kernels read their patch's table
// with one coalesced load instead of npn^2 binary searches per factorisation.
__global__ void patch_slots_kernel(DevMatrix A, int64_t n_patches, int npn,
                                   const int32_t* __restrict__ nodes,
                                   int32_t* __restrict__ slots) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t per = (int64_t)npn * npn;
  if (t >= n_patches * per) return;
  const int64_t p = t / per;
  const int r = (int)(t - p * per), a = r / npn, b = r - a * npn;
  const int64_t ra = nodes[p * npn + a];
  const int32_t cb = nodes[p * npn + b];
  int64_t lo = A.indptr[ra], hi = A.indptr[ra + 1];
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (A.indices[mid] < cb) lo = mid + 1; else hi = mid;
  }
  int32_t v = -1;
  if (lo < A.indptr[ra + 1] && A.indices[lo] == cb) {
    v = (int32_t)lo;
  } else if (A.pp_indptr != nullptr) {
    lo = A.pp_indptr[ra];
    hi = A.pp_indptr[ra + 1];
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (A.pp_indices[mid] < cb) lo = mid + 1; else hi = mid;
    }
    if (lo < A.pp_indptr[ra + 1] && A.pp_indices[lo] == cb) v = -(int32_t)lo - 2;
  }
  slots[t] = v;
}

// --------------------------------------------------------------------------
// Gauss-Jordan inversion, second form: warp w owns the columns {w + W*j} of
// every row (rows ty + 32*i in registers, the NP - 32*RTR tail rows in shared
// memory, one per lane), ONE rolled loop over the pivot steps with one block
// barrier per step:
//  * the pivot row is scaled and handed round inside each warp (the lane
//    holding it writes the warp's segment to shared memory, __syncwarp), so
//    the only block-wide exchange is the pivot column;
//  * the owner of column k+1 applies step k to that column first, publishes
//    it and chooses pivot k+1 while the other warps eliminate; the choice is
//    two warp-wide integer max reductions over a key (|value| with its low 7
//    mantissa bits replaced by 127 - row: largest |value|, lowest row among
//    values equal in the upper 45 mantissa bits — the getrf pivot up to
//    last-bits ties);
//  * after its elimination the owner resets the published column to the unit
//    vector of the pivot row, so step k+1 needs no special case: the scaled
//    pivot row carries 1/pivot there and the elimination writes -f/pivot.
// --------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@p bra DONE_%=;\n"
      "bra WAIT_%=;\n"
      "DONE_%=:\n"
      "}\n" ::"r"(a), "r"(parity) : "memory");
}

struct alignas(16) GjPivot {
  double rp;      // 1 / pivot (0 for a reported zero pivot)
  int row, pad;
};

template <int NP, int NC, int W, int MINB>
__global__ void __launch_bounds__(32 * W, MINB) vanka_factorize_pw_kernel(
    DevMatrix A, int64_t n_patches, const int32_t* __restrict__ slots, double* __restrict__ inv,
    int ld, int64_t* status) {
  constexpr int NPN = NP / NC, CT = NP / W, RTR = NP / 32, TAIL = NP - 32 * RTR, NT = 32 * W;
  constexpr int CTP = (CT + 1) & ~1;                        // 16-byte aligned warp segments
  // tail rows: the row stride keeps the 16-byte accesses of 8 consecutive
  // lanes on distinct banks
  constexpr int TS = (W * CTP + 1) / 4 * 4 + 2;
  constexpr int CS = 32 * RTR + 32;
  static_assert(NP % W == 0 && NP < 128 && RTR >= 1 && TS % 2 == 0, "layout");
  __shared__ __align__(16) double prow[W][CTP];
  __shared__ __align__(16) double Mt[TAIL > 0 ? TAIL : 1][TS];
  // No block barrier in the pivot loop.  The published column / pivot of step
  // k sits in ring slot k % D; full[slot] is completed by the owner warp's 32
  // arrivals after publication, empty[slot] by one arrival per warp once its
  // lanes have read the slot: nobody waits for the owner's own elimination
  // (deeper rings measured equal: the chain of pivot choices sets the pace).
  constexpr int D = 2;
  __shared__ __align__(16) double colk[D][CS];
  __shared__ GjPivot pivot[D];
  __shared__ uint64_t full_bar[D], empty_bar[D];
  __shared__ int piv_of_step[NP], step_of_row[NP];
  __shared__ double rp_of_row[NP];                         // pending row factors
  __shared__ int32_t slotB[NPN * NPN], slotP[NPN * NPN];
  const int tid = threadIdx.x, ty = tid & 31, w = tid >> 5;
  const int64_t pid = blockIdx.x;
  {
    const int32_t* ps = slots + pid * (NPN * NPN);
    for (int t = tid; t < NPN * NPN; t += NT) {
      const int32_t v = ps[t];
      slotB[t] = v >= 0 ? v : -1;
      slotP[t] = v <= -2 ? -(v + 2) : -1;
    }
    for (int i = tid; i < D * CS; i += NT) (&colk[0][0])[i] = 0.0;
    for (int i = tid; i < W * CTP; i += NT) (&prow[0][0])[i] = 0.0;
    if (tid < D) {
      mbar_init(&full_bar[tid], 32);
      mbar_init(&empty_bar[tid], W);
    }
  }
  __syncthreads();
  auto entry = [&](int r, int c) -> double {
    const int a = r / NC, ci = r - a * NC, b = c / NC, cj = c - b * NC;
    const int t = a * NPN + b;
    if (slotB[t] >= 0) return A.data[(int64_t)slotB[t] * (NC * NC) + ci * NC + cj];
    if (ci == 0 && cj == 0 && slotP[t] >= 0) return A.pp_data[slotP[t]];
    return 0.0;
  };
  const bool tl = TAIL > 0 && ty < TAIL;                    // this lane carries a tail row
  double* const mt = &Mt[tl ? ty : 0][w * CTP];             // its segment of that row
  double* const myrow = prow[w];
  double M[RTR][CT];
#pragma unroll
  for (int i = 0; i < RTR; ++i)
#pragma unroll
    for (int j = 0; j < CT; ++j) M[i][j] = entry(ty + 32 * i, j * W + w);
  if (tl) {
#pragma unroll
    for (int j = 0; j < CTP; ++j) mt[j] = j < CT ? entry(32 * RTR + ty, j * W + w) : 0.0;
  }
  unsigned usedmask = 0;
  // publication + pivot choice of column kk by its owner warp: c / ct are the
  // column's current values in this lane's rows; returns the pivot row
  auto pick = [&](int kk, const double (&c)[RTR], double ct) -> int {
    const int slot = kk & (D - 1);
    if (kk >= D) mbar_wait(&empty_bar[slot], ((kk / D) - 1) & 1);
    double* cn = colk[slot];
    unsigned long long key = 0ull;
#pragma unroll
    for (int i = 0; i < RTR; ++i) {
      cn[ty + 32 * i] = c[i];
      const unsigned long long kb =
          ((unsigned long long)__double_as_longlong(fabs(c[i])) & ~127ull) |
          (unsigned long long)(127 - (ty + 32 * i));
      if (!(usedmask >> i & 1u) && kb > key) key = kb;
    }
    if (tl) {
      cn[32 * RTR + ty] = ct;
      const unsigned long long kb =
          ((unsigned long long)__double_as_longlong(fabs(ct)) & ~127ull) |
          (unsigned long long)(127 - (32 * RTR + ty));
      if (!(usedmask >> RTR & 1u) && kb > key) key = kb;
    }
    const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
    const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
    const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
    const int bi = min(127 - (int)(ml & 127u), NP - 1);
    __syncwarp();
    const double val = cn[bi];
    // zero, NaN or infinite pivot: reported like the reference's singular block
    const bool bad = val == 0.0 || mh >= 0x7ff00000u;
    const double rp = bad ? 0.0 : 1.0 / val;
    __syncwarp();
    if (ty == 0) {
      cn[bi] = 0.0;                              // f = 0 on the pivot row
      GjPivot pn;
      pn.rp = rp;
      pn.row = bi;
      pn.pad = 0;
      pivot[slot] = pn;
      piv_of_step[kk] = bi;
      step_of_row[bi] = kk;
      rp_of_row[bi] = rp;
      if (bad)
        atomicCAS(reinterpret_cast<unsigned long long*>(status), 0ull,
                  (unsigned long long)(pid + 1));
    }
    mbar_arrive(&full_bar[slot]);                // every lane after its own writes
    return bi;
  };
#define ALEFSI_GJ_CASES(X)                                                                   \
  X(0) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15)           \
  X(16) X(17) X(18) X(19) X(20) X(21) X(22) X(23) X(24) X(25) X(26) X(27)
  static_assert(CT <= 28, "column switch");
  // the published column becomes the unit vector of its pivot row
  auto reset_column = [&](int jn, int bi) {
    switch (jn) {
#define ALEFSI_GJ_RESET(J)                                                                   \
  case J:                                                                                    \
    if constexpr (J < CT) {                                                                  \
      _Pragma("unroll") for (int i = 0; i < RTR; ++i)                                        \
          M[i][J] = (ty + 32 * i == bi) ? 1.0 : 0.0;                                         \
    }                                                                                        \
    break;
      ALEFSI_GJ_CASES(ALEFSI_GJ_RESET)
#undef ALEFSI_GJ_RESET
      default: break;
    }
    if (tl) mt[jn] = (32 * RTR + ty == bi) ? 1.0 : 0.0;
  };
  if (w == 0) {
    double c[RTR];
#pragma unroll
    for (int i = 0; i < RTR; ++i) c[i] = M[i][0];
    const int bi = pick(0, c, tl ? mt[0] : 0.0);
    reset_column(0, bi);
  }
  // iteration kk: elimination step k = kk - 1 and, by its owner, publication
  // + pivot choice of column kk (kk < NP)
#pragma unroll 1
  for (int kk = 1; kk <= NP; ++kk) {
    const int wn = kk % W, jn = kk / W;
    const int cs = (kk - 1) & (D - 1);
    __syncwarp();            // the warp is done with its pivot-row segment of the last step
    mbar_wait(&full_bar[cs], ((kk - 1) / D) & 1);
    const GjPivot pv = pivot[cs];
    const double* ck = colk[cs];
    const int pl = pv.row & 31, pi = pv.row >> 5;
    if (pl == ty) {
      usedmask |= 1u << pi;
      // the lane holding the pivot row hands this warp's segment of it to the
      // warp's other lanes, unscaled: 1/pivot goes into the multipliers, and
      // the row keeps its own factor 1/pivot pending until the write-out (a
      // row with a pending factor updates itself consistently: its published
      // column entries are unscaled too)
      if (pi < RTR) {
#pragma unroll
        for (int i = 0; i < RTR; ++i) {
          if (pi == i) {
#pragma unroll
            for (int jj = 0; jj < CT; ++jj) myrow[jj] = M[i][jj];
          }
        }
      } else {
#pragma unroll
        for (int jj = 0; jj + 1 < CTP; jj += 2)
          *reinterpret_cast<double2*>(myrow + jj) = *reinterpret_cast<const double2*>(mt + jj);
      }
    }
    double f[RTR];
#pragma unroll
    for (int i = 0; i < RTR; ++i) f[i] = -ck[ty + 32 * i] * pv.rp;
    const double ft = -ck[32 * RTR + (tl ? ty : 0)] * pv.rp;
    __syncwarp();
    if (ty == 0) mbar_arrive(&empty_bar[cs]);
    int bi = -1;
    if (w == wn && kk < NP) {
      // next pivot column first: apply step k to it, publish it, choose its pivot
      double c[RTR];
      const double pvn = myrow[jn];
      switch (jn) {
#define ALEFSI_GJ_COL(J)                                                                     \
  case J:                                                                                    \
    if constexpr (J < CT) {                                                                  \
      _Pragma("unroll") for (int i = 0; i < RTR; ++i) c[i] = fma(f[i], pvn, M[i][J]);        \
    }                                                                                        \
    break;
        ALEFSI_GJ_CASES(ALEFSI_GJ_COL)
#undef ALEFSI_GJ_COL
        default: break;
      }
      bi = pick(kk, c, tl ? fma(ft, pvn, mt[jn]) : 0.0);
    }
#pragma unroll
    for (int jj = 0; jj + 1 < CTP; jj += 2) {
      const double2 p2 = *reinterpret_cast<const double2*>(myrow + jj);
#pragma unroll
      for (int i = 0; i < RTR; ++i) {
        M[i][jj] = fma(f[i], p2.x, M[i][jj]);
        if (jj + 1 < CT) M[i][jj + 1] = fma(f[i], p2.y, M[i][jj + 1]);
      }
      if (tl) {
        double2 t2 = *reinterpret_cast<double2*>(mt + jj);
        t2.x = fma(ft, p2.x, t2.x);
        t2.y = fma(ft, p2.y, t2.y);       // padding column: stays 0 (p2.y = 0)
        *reinterpret_cast<double2*>(mt + jj) = t2;
      }
    }
    if (bi >= 0) reset_column(jn, bi);
  }
#undef ALEFSI_GJ_CASES
  __syncthreads();
  double* out = inv + pid * (int64_t)NP * ld;
#pragma unroll
  for (int i = 0; i < RTR; ++i)
#pragma unroll
    for (int j = 0; j < CT; ++j)
      out[(int64_t)piv_of_step[j * W + w] * ld + step_of_row[ty + 32 * i]] =
          M[i][j] * rp_of_row[ty + 32 * i];
  if (tl) {
#pragma unroll
    for (int j = 0; j < CT; ++j)
      out[(int64_t)piv_of_step[j * W + w] * ld + step_of_row[32 * RTR + ty]] =
          mt[j] * rp_of_row[32 * RTR + ty];
  }
  if (ld > NP)
    for (int col = tid; col < NP; col += NT)
      for (int r = NP; r < ld; ++r) out[(int64_t)col * ld + r] = 0.0;
}

// --------------------------------------------------------------------------
// Large patches (2x2x2-cell macros in 3D: 500 x 500, the reference's default
// solid blocking, newton.py:53-56): batched blocked Gauss-Jordan.  Each patch
// matrix is gathered row-major into its own slot of the group's inverse
// storage (ld == np), then every 16-column panel is factorised by one CTA per
// patch (gj_panel_kernel, panel in shared memory) and applied to the rest of
// all patches' matrices by one 3D-grid gj_update_kernel launch; the row
// permutation is undone (gj_unscramble_kernel) and each inverse transposed in
// place to the column-major storage of the apply kernels.  Pivot choice of
// partial pivoting (largest |value| among the remaining rows, reference
// linsolve.py:131 np.linalg.inv -> getrf); ~64 launches per factorisation
// instead of one launch pair per pivot step.
// --------------------------------------------------------------------------
__global__ void big_gather_kernel(DevMatrix A, int np_, int npn, const int32_t* nodes,
                                  double* M) {
  const int64_t p = blockIdx.y;
  const int32_t* pn = nodes + p * npn;
  double* Mp = M + p * (int64_t)np_ * np_;
  const int nc = A.nc;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (int64_t)np_ * np_;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / np_), j = (int)(e - (int64_t)i * np_);
    const int a = i / nc, ci = i - a * nc, b = j / nc, cj = j - b * nc;
    const int64_t ra = pn[a];
    const int32_t cb = pn[b];
    int64_t lo = A.indptr[ra], hi = A.indptr[ra + 1];
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (A.indices[mid] < cb) lo = mid + 1; else hi = mid;
    }
    double v = 0.0;
    if (lo < A.indptr[ra + 1] && A.indices[lo] == cb) {
      v = A.data[lo * nc * nc + ci * nc + cj];
    } else if (ci == 0 && cj == 0 && A.pp_indptr != nullptr) {
      lo = A.pp_indptr[ra];
      hi = A.pp_indptr[ra + 1];
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (A.pp_indices[mid] < cb) lo = mid + 1; else hi = mid;
      }
      if (lo < A.pp_indptr[ra + 1] && A.pp_indices[lo] == cb) v = A.pp_data[lo];
    }
    Mp[e] = v;
  }
}

// row-major inverse -> column-major (in place, n x n per patch); a failed
// patch reports 1 + its index in the group status (first one wins)
__global__ void big_finish_kernel(int np_, double* M, const int64_t* pstatus, int64_t* status) {
  const int64_t p = blockIdx.y;
  if (pstatus[p] != 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0)
      atomicCAS(reinterpret_cast<unsigned long long*>(status), 0ull,
                (unsigned long long)(p + 1));
    return;
  }
  double* Mp = M + p * (int64_t)np_ * np_;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (int64_t)np_ * np_;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / np_), j = (int)(e - (int64_t)i * np_);
    if (i < j) {
      const double t = Mp[e];
      Mp[e] = Mp[(int64_t)j * np_ + i];
      Mp[(int64_t)j * np_ + i] = t;
    }
  }
}

// --------------------------------------------------------------------------
// Grid transfer: Q2 interpolation P (fine rows) and its transpose (coarse
// rows), applied per component with the constrained-dof masks of
// linsolve.py:260-270.  Summation order follows the stored column order
// (fine-node order for the transpose, as in scipy's CSC matvec).
// --------------------------------------------------------------------------
__global__ void transfer_kernel(int64_t nrows, int nc, const int64_t* __restrict__ ptr,
                                const int32_t* __restrict__ idx, const double* __restrict__ val,
                                const double* __restrict__ src,
                                const uint8_t* __restrict__ constrained,
                                double* __restrict__ dst, int add) {
  pdl_entry();
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nrows * nc) return;
  const int64_t row = t / nc;
  const int c = (int)(t - row * nc);
  double acc = 0.0;
  const int64_t end = ptr[row + 1];
  int64_t e = ptr[row];
  // loads of four entries in flight, sums in stored order (long restriction rows)
  for (; e + 4 <= end; e += 4) {
    const double v0 = __ldg(val + e), v1 = __ldg(val + e + 1), v2 = __ldg(val + e + 2),
                 v3 = __ldg(val + e + 3);
    const double x0 = __ldg(src + (int64_t)__ldg(idx + e) * nc + c);
    const double x1 = __ldg(src + (int64_t)__ldg(idx + e + 1) * nc + c);
    const double x2 = __ldg(src + (int64_t)__ldg(idx + e + 2) * nc + c);
    const double x3 = __ldg(src + (int64_t)__ldg(idx + e + 3) * nc + c);
    acc = __dadd_rn(acc, __dmul_rn(v0, x0));
    acc = __dadd_rn(acc, __dmul_rn(v1, x1));
    acc = __dadd_rn(acc, __dmul_rn(v2, x2));
    acc = __dadd_rn(acc, __dmul_rn(v3, x3));
  }
  for (; e < end; ++e)
    acc = __dadd_rn(acc, __dmul_rn(__ldg(val + e), __ldg(src + (int64_t)__ldg(idx + e) * nc + c)));
  if (constrained[t]) acc = 0.0;
  dst[t] = add ? __dadd_rn(dst[t], acc) : acc;
}

// Restriction on small levels: 8 lanes per (coarse node, component), lane k
// summing entries k, k+8, ... of the row, combined by a fixed xor-shuffle
// tree (deterministic; a different association than the sequential sum).
// The long rows (~100 fine nodes per coarse node) otherwise make every
// thread a chain of dependent L2 round trips.
__global__ void __launch_bounds__(256) transfer_split_kernel(
    int64_t nrows, int nc, const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
    const double* __restrict__ val, const double* __restrict__ src,
    const uint8_t* __restrict__ constrained, double* __restrict__ dst, int add) {
  pdl_entry();
  const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  const int k = threadIdx.x & 7;
  const bool live = g < nrows * nc;
  const int64_t row = live ? g / nc : 0;
  const int c = live ? (int)(g - row * nc) : 0;
  double acc = 0.0;
  if (live) {
    const int64_t end = ptr[row + 1];
    for (int64_t e = ptr[row] + k; e < end; e += 8)
      acc = __dadd_rn(acc, __dmul_rn(__ldg(val + e), __ldg(src + (int64_t)__ldg(idx + e) * nc + c)));
  }
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o, 8));
  if (!live || k != 0) return;
  if (constrained[g]) acc = 0.0;
  dst[g] = add ? __dadd_rn(dst[g], acc) : acc;
}

// NC = 4: one thread per row applies the row's (val, idx) run to all four
// components (one 32-byte load of the source block per entry), four entries
// in flight per step.  Per component the products and sums are those of
// transfer_kernel in the same order: bitwise identical.
__global__ void transfer4_kernel(int64_t nrows, const int64_t* __restrict__ ptr,
                                 const int32_t* __restrict__ idx, const double* __restrict__ val,
                                 const double* __restrict__ src,
                                 const uint8_t* __restrict__ constrained,
                                 double* __restrict__ dst, int add) {
  pdl_entry();
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= nrows) return;
  const int64_t beg = ptr[row], end = ptr[row + 1];
  d4 acc = {0.0, 0.0, 0.0, 0.0};
  auto step = [&](double v, const d4& x) {
    acc.x = __dadd_rn(acc.x, __dmul_rn(v, x.x));
    acc.y = __dadd_rn(acc.y, __dmul_rn(v, x.y));
    acc.z = __dadd_rn(acc.z, __dmul_rn(v, x.z));
    acc.w = __dadd_rn(acc.w, __dmul_rn(v, x.w));
  };
  int64_t e = beg;
  for (; e + 4 <= end; e += 4) {
    const double v0 = __ldg(val + e), v1 = __ldg(val + e + 1), v2 = __ldg(val + e + 2),
                 v3 = __ldg(val + e + 3);
    const int c0 = __ldg(idx + e), c1 = __ldg(idx + e + 1), c2 = __ldg(idx + e + 2),
              c3 = __ldg(idx + e + 3);
    const d4 x0 = ld256_ro(src + (int64_t)c0 * 4), x1 = ld256_ro(src + (int64_t)c1 * 4);
    const d4 x2 = ld256_ro(src + (int64_t)c2 * 4), x3 = ld256_ro(src + (int64_t)c3 * 4);
    step(v0, x0);
    step(v1, x1);
    step(v2, x2);
    step(v3, x3);
  }
  for (; e < end; ++e) step(__ldg(val + e), ld256_ro(src + (int64_t)__ldg(idx + e) * 4));
  const uchar4 m = reinterpret_cast<const uchar4*>(constrained)[row];
  double2* o = reinterpret_cast<double2*>(dst + row * 4);
  double2 a = {m.x ? 0.0 : acc.x, m.y ? 0.0 : acc.y}, b = {m.z ? 0.0 : acc.z, m.w ? 0.0 : acc.w};
  if (add) {
    const double2 a0 = o[0], b0 = o[1];
    a = {__dadd_rn(a0.x, a.x), __dadd_rn(a0.y, a.y)};
    b = {__dadd_rn(b0.x, b.x), __dadd_rn(b0.y, b.y)};
  }
  o[0] = a;
  o[1] = b;
}

// --------------------------------------------------------------------------
// Coarse level: dense Gauss-Jordan inverse (one pivot step per launch pair)
// and a warp-per-row dense matvec.
// --------------------------------------------------------------------------
// Pivot step k: one pass over column k (all rows, staged in shared memory)
// finds the pivot among rows >= k; rows k and p are swapped, column k is
// published with the swap applied, and the pivot row is scaled.
constexpr int kGjMaxN = 4096;
__global__ void __launch_bounds__(1024) gj_pivot_kernel(double* M, int64_t n, int64_t k,
                                                        int64_t* perm, double* colk,
                                                        double* rp_out, int64_t* status) {
  __shared__ double sb[32];
  __shared__ int64_t si[32];
  __shared__ int64_t prow;
  __shared__ double cs[kGjMaxN];
  const int tid = threadIdx.x;
  double best = -1.0;
  int64_t bi = k;
  for (int64_t i = tid; i < n; i += blockDim.x) {
    const double v = M[i * n + k];
    cs[i] = v;
    if (i >= k && fabs(v) > best) { best = fabs(v); bi = i; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
  }
  if ((tid & 31) == 0) { sb[tid >> 5] = best; si[tid >> 5] = bi; }
  __syncthreads();
  if (tid < 32) {
    best = tid < (int)(blockDim.x >> 5) ? sb[tid] : -2.0;
    bi = tid < (int)(blockDim.x >> 5) ? si[tid] : n;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    if (tid == 0) { prow = bi; perm[k] = bi; }
  }
  __syncthreads();
  const int64_t pr = prow;
  const double piv = cs[pr];
  if (piv == 0.0) {
    if (tid == 0 && *status == 0) *status = k + 1;
    if (tid == 0) *rp_out = 0.0;
    return;
  }
  const double rp = 1.0 / piv;
  for (int64_t i = tid; i < n; i += blockDim.x)
    colk[i] = cs[i == k ? pr : (i == pr ? k : i)];
  // swap rows k and pr, scale the new pivot row
  for (int64_t j = tid; j < n; j += blockDim.x) {
    const double vk = M[k * n + j], vp = M[pr * n + j];
    if (pr != k) M[pr * n + j] = vk;
    M[k * n + j] = (j == k) ? rp : vp * rp;
  }
  if (tid == 0) *rp_out = rp;
}

// Elimination of column k from every row but k: row i = blockIdx.y, two
// columns per thread (n even) with 16-byte accesses.
__global__ void gj_eliminate_kernel(double* M, int64_t n, int64_t k, const double* colk,
                                    const double* rp_in) {
  const int64_t i = blockIdx.y;
  if (i == k) return;
  const double rp = *rp_in;
  if (rp == 0.0) return;
  const double f = colk[i];
  const double* pk = M + k * n;
  double* row = M + i * n;
  if ((n & 1) == 0) {
    const int64_t j2 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (2 * j2 >= n) return;
    const double2 p = reinterpret_cast<const double2*>(pk)[j2];
    double2 v = reinterpret_cast<double2*>(row)[j2];
    v.x = (2 * j2 == k) ? -f * rp : v.x - f * p.x;
    v.y = (2 * j2 + 1 == k) ? -f * rp : v.y - f * p.y;
    reinterpret_cast<double2*>(row)[j2] = v;
  } else {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x)
      row[j] = (j == k) ? -f * rp : row[j] - f * pk[j];
  }
}

// Blocked Gauss-Jordan: panels of nb pivot columns.  The panel kernel (one
// CTA, the n x nb panel in shared memory) runs the nb pivot steps of the
// unblocked algorithm on the panel only (same pivot choice: largest |value|
// among rows >= k, lowest row on ties), records the composed row
// permutation src[] and snapshots the rows it moved or pivots on.  The
// update kernel then applies the whole panel to the other columns as one
// rank-nb product:
//   rows k0..k0+nb-1 :  M[i, j] = sum_s X[i, s] * M_old[src(k0+s), j]   (X = A^-1)
//   other rows       :  M[i, j] = M_old[src(i), j] + sum_s L[i, s] * M_old[src(k0+s), j]
// (L = -B A^-1; both stored in the panel columns), i.e. nb pivot steps per
// pass over the matrix instead of one.
template <int KB>
__global__ void __launch_bounds__(512) gj_panel_kernel(double* M, int n, int k0, int kb,
                                                        int64_t* perm, int* src_out,
                                                        double* slab, int* rowslot,
                                                        int64_t* status) {
  extern __shared__ __align__(16) unsigned char gj_smem[];
  double* P = reinterpret_cast<double*>(gj_smem);        // column-major: P[t * n + i]
  int* src = reinterpret_cast<int*>(P + (size_t)n * kb);  // n
  __shared__ int s_pr, s_stop, s_ntouch;
  __shared__ int touched[64], srows[64];
  // per-warp pivot candidates (|value|, row) of the next pivot column: each
  // step's row update also scans the column the next step pivots on, so the
  // pivot search is spread over all warps instead of a 32-lane scan of n rows
  // between two barriers (same choice: largest |value|, lowest row on ties)
  __shared__ double cand_v[32];
  __shared__ int cand_i[32];
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;
  auto warp_argmax = [&](double& best, int& bi) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
  };
  {   // batched use (Vanka macro patches): matrix blockIdx.x of a batch
    const int64_t bat = blockIdx.x;
    M += bat * n * n;
    perm += bat * n;
    src_out += bat * n;
    rowslot += bat * n;
    slab += bat * 2 * KB * n;
    status += bat;
  }
  if (*status != 0) return;   // an earlier panel hit a zero pivot
  for (int e = tid; e < n * kb; e += nt) {
    const int i = e / kb, t = e - i * kb;
    P[t * n + i] = M[(int64_t)i * n + k0 + t];
  }
  for (int i = tid; i < n; i += nt) src[i] = i;
  if (tid == 0) { s_stop = 0; s_ntouch = 0; }
  __syncthreads();
  {
    double best = -1.0;
    int bi = n;
    for (int i = k0 + tid; i < n; i += nt) {
      const double v = fabs(P[i]);
      if (v > best) { best = v; bi = i; }
    }
    warp_argmax(best, bi);
    if (lane == 0) { cand_v[wid] = best; cand_i[wid] = bi; }
  }
  __syncthreads();
  __shared__ double s_piv[KB], s_rk[KB];
#pragma unroll
  for (int t = 0; t < KB; ++t) {
    if (t >= kb) break;
    const int k = k0 + t;
    const double* Pt = P + t * n;
    // warp 0: pivot of column t (rows >= k) from the warps' candidates, the
    // swap bookkeeping and copies of the pivot row and old row k
    if (tid < 32) {
      double best = lane < nt / 32 ? cand_v[lane] : -1.0;
      int bi = lane < nt / 32 ? cand_i[lane] : n;
      warp_argmax(best, bi);
      const int pr = bi < n ? bi : k;
      if (tid < kb) {
        s_piv[tid] = P[tid * n + pr];
        s_rk[tid] = P[tid * n + k];
      }
      if (tid == 0) {
        s_pr = pr;
        perm[k] = pr;
        if (Pt[pr] == 0.0) {
          s_stop = 1;
          if (*status == 0) *status = k + 1;
        }
        if (s_ntouch < 64) touched[s_ntouch++] = k;
        if (pr != k && s_ntouch < 64) touched[s_ntouch++] = pr;
        const int a2 = src[k];
        src[k] = src[pr];
        src[pr] = a2;
      }
    }
    __syncthreads();
    if (s_stop) return;
    const int pr = s_pr;
    double piv[KB], rk[KB];
#pragma unroll
    for (int s2 = 0; s2 < KB; ++s2) {
      piv[s2] = s2 < kb ? s_piv[s2] : 0.0;
      rk[s2] = s2 < kb ? s_rk[s2] : 0.0;
    }
    const double rp = 1.0 / piv[t];
    // rows after the swap: row k <- old row pr (scaled), row pr <- old row k;
    // one thread per row, reading its multiplier before writing the row
    double nbest = -1.0;
    int nbi = n;
    for (int i = tid; i < n; i += nt) {
      if (i == k) {
#pragma unroll
        for (int s2 = 0; s2 < KB; ++s2)
          if (s2 < kb) P[s2 * n + k] = (s2 == t) ? rp : piv[s2] * rp;
        continue;
      }
      double row[KB];
#pragma unroll
      for (int s2 = 0; s2 < KB; ++s2) row[s2] = s2 < kb ? (i == pr ? rk[s2] : P[s2 * n + i]) : 0.0;
      const double f = row[t];
#pragma unroll
      for (int s2 = 0; s2 < KB; ++s2)
        if (s2 < kb) {
          const double v = (s2 == t) ? -f * rp : row[s2] - f * (piv[s2] * rp);
          P[s2 * n + i] = v;
          // next pivot column: rows >= k + 1, ascending within the thread
          if (s2 == t + 1 && i > k) {
            const double a = fabs(v);
            if (a > nbest) { nbest = a; nbi = i; }
          }
        }
    }
    if (t + 1 < kb) {
      warp_argmax(nbest, nbi);
      if (lane == 0) { cand_v[wid] = nbest; cand_i[wid] = nbi; }
    }
    __syncthreads();
  }
  // panel columns in their final form
  for (int e = tid; e < n * kb; e += nt) {
    const int i = e / kb, t = e - i * kb;
    M[(int64_t)i * n + k0 + t] = P[t * n + i];
  }
  for (int i = tid; i < n; i += nt) {
    src_out[i] = src[i];
    rowslot[i] = -1;
  }
  __syncthreads();
  // rows read through the permutation: sources of the pivot positions and of
  // every moved row, snapshot before the update kernel overwrites them
  if (tid == 0) {
    int q = 0;
    for (int a = 0; a < s_ntouch; ++a) {
      const int r = src[touched[a]];
      bool seen = false;
      for (int c = 0; c < q; ++c) seen = seen || srows[c] == r;
      if (!seen) {
        rowslot[r] = q;
        srows[q++] = r;
      }
    }
    s_ntouch = q;
  }
  __syncthreads();
  const int ncopy = s_ntouch * n;
  for (int e = tid; e < ncopy; e += nt) {
    const int q = e / n, j = e - q * n;
    slab[e] = M[(int64_t)srows[q] * n + j];
  }
}

// The same panel factorisation spread over a thread-block cluster of C CTAs
// (distributed shared memory): CTA c holds rows [c*R, (c+1)*R) of the
// n x kb panel, so the panel load, the row updates and the per-step pivot
// scans run on C SMs instead of one.  Per pivot step: every CTA publishes its
// best candidate, all CTAs pick the same pivot from the C candidates (largest
// |value|, lowest row on ties: the single-CTA choice), the owners of the
// pivot row and of row k publish their old values, and every CTA updates its
// rows with the single-CTA kernel's arithmetic.  Each CTA's candidate
// carries its row and the owner of the next row k publishes it, both in the
// CTA's own shared memory, double-buffered by step parity: one cluster
// barrier per step, remote loads only; bitwise-equal panels.  Rank 0 keeps the permutation bookkeeping and
// the snapshot rows exactly as gj_panel_kernel does.
template <int KB>
__global__ void __launch_bounds__(256) gj_panel_cluster_kernel(double* M, int n, int k0, int kb,
                                                               int R, int64_t* perm,
                                                               int* src_out, double* slab,
                                                               int* rowslot, int64_t* status) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int C = (int)cluster.num_blocks(), cr = (int)cluster.block_rank();
  extern __shared__ __align__(16) unsigned char gjc_smem[];
  double* P = reinterpret_cast<double*>(gjc_smem);        // column-major: P[t * R + local row]
  int* src = reinterpret_cast<int*>(P + (size_t)R * kb);  // n (rank 0)
  // per-CTA publication for the next step, double-buffered by step parity
  // (read remotely by every CTA after one cluster barrier): the CTA's best
  // candidate of the step's pivot column with that row's old values, and old
  // row k from its owner
  __shared__ double cand_v[8], cta_v[2], candrow[2][KB], rkrow[2][KB], lp[KB], lk[KB];
  __shared__ int cand_i[8], cta_i[2], s_pr, s_ntouch;
  __shared__ int touched[64], srows[64];
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;
  const int r0 = cr * R, r1 = min(n, r0 + R), nr = max(0, r1 - r0);
  auto warp_argmax = [&](double& best, int& bi) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
  };
  // per-warp candidates -> this CTA's candidate for step t with its row
  // (warp 0), old row k0 + t from its owner (warp 1), after a CTA barrier
  auto cta_publish = [&](int t) {
    __syncthreads();
    const int bf = t & 1;
    if (tid < 32) {
      double best = lane < nt / 32 ? cand_v[lane] : -1.0;
      int bi = lane < nt / 32 ? cand_i[lane] : n;
      warp_argmax(best, bi);
      if (lane == 0) { cta_v[bf] = best; cta_i[bf] = bi; }
      if (lane < kb) candrow[bf][lane] = bi < n ? P[lane * R + bi - r0] : 0.0;
    } else if (tid < 64) {
      const int k = k0 + t;
      if (k >= r0 && k < r1 && lane < kb) rkrow[bf][lane] = P[lane * R + k - r0];
    }
  };
  if (*status != 0) return;   // an earlier panel hit a zero pivot (every CTA sees it)
  constexpr int LB = 8;         // global loads in flight per thread in the copies
  for (int e0 = tid; e0 < nr * kb; e0 += LB * nt) {
    double v[LB];
#pragma unroll
    for (int u = 0; u < LB; ++u) {
      const int e = e0 + u * nt;
      if (e < nr * kb) {
        const int il = e / kb, t = e - il * kb;
        v[u] = M[(int64_t)(r0 + il) * n + k0 + t];
      }
    }
#pragma unroll
    for (int u = 0; u < LB; ++u) {
      const int e = e0 + u * nt;
      if (e < nr * kb) {
        const int il = e / kb, t = e - il * kb;
        P[t * R + il] = v[u];
      }
    }
  }
  if (cr == 0) {
    for (int i = tid; i < n; i += nt) src[i] = i;
    if (tid == 0) s_ntouch = 0;
  }
  __syncthreads();
  {
    double best = -1.0;
    int bi = n;
    for (int il = tid; il < nr; il += nt)
      if (r0 + il >= k0) {
        const double v = fabs(P[il]);
        if (v > best) { best = v; bi = r0 + il; }
      }
    warp_argmax(best, bi);
    if (lane == 0) { cand_v[wid] = best; cand_i[wid] = bi; }
  }
  cta_publish(0);
  cluster.sync();
  // the step loop stays rolled (an unrolled body of KB steps overflowed the
  // instruction cache: "no instruction" was the top stall); column t is
  // picked from the unrolled register rows by compare-and-select
#pragma unroll 1
  for (int t = 0; t < kb; ++t) {
    const int k = k0 + t, bf = t & 1;
    if (tid < 32) {
      double best = -1.0;
      int bi = n;
      if (lane < C) {
        best = *cluster.map_shared_rank(&cta_v[bf], lane);
        bi = *cluster.map_shared_rank(&cta_i[bf], lane);
      }
      warp_argmax(best, bi);
      const int pr = bi < n ? bi : k;
      if (lane == 0) s_pr = pr;
      // old pivot row: the winning CTA's candidate row (pr == k: old row k)
      if (lane < kb) {
        lk[lane] = *cluster.map_shared_rank(&rkrow[bf][lane], k / R);
        lp[lane] = bi < n ? *cluster.map_shared_rank(&candrow[bf][lane], pr / R) : lk[lane];
      }
    }
    __syncthreads();
    const int pr = s_pr;
    const double pivt = lp[t];
    if (pivt == 0.0) {     // same value in every CTA: all leave together
      if (cr == 0 && tid == 0) {
        perm[k] = pr;
        if (*status == 0) *status = k + 1;
      }
      // no CTA may exit while another still reads its shared memory
      cluster.sync();
      return;
    }
    if (cr == 0 && tid == 0) {
      perm[k] = pr;
      if (s_ntouch < 64) touched[s_ntouch++] = k;
      if (pr != k && s_ntouch < 64) touched[s_ntouch++] = pr;
      const int a2 = src[k];
      src[k] = src[pr];
      src[pr] = a2;
    }
    const double rp = 1.0 / pivt;
    double nbest = -1.0;
    int nbi = n;
    // rows streamed element by element (old pivot row and old row k from
    // shared memory): the same expressions as gj_panel_kernel, few registers
    for (int il = tid; il < nr; il += nt) {
      const int i = r0 + il;
      if (i == k) {
        for (int s2 = 0; s2 < kb; ++s2) P[s2 * R + il] = (s2 == t) ? rp : lp[s2] * rp;
        continue;
      }
      const bool isp = i == pr;
      const double f = isp ? lk[t] : P[t * R + il];
#pragma unroll 4
      for (int s2 = 0; s2 < kb; ++s2) {
        const double old = isp ? lk[s2] : P[s2 * R + il];
        const double v = (s2 == t) ? -f * rp : old - f * (lp[s2] * rp);
        P[s2 * R + il] = v;
        if (s2 == t + 1 && i > k) {
          const double a = fabs(v);
          if (a > nbest) { nbest = a; nbi = i; }
        }
      }
    }
    warp_argmax(nbest, nbi);
    if (lane == 0) { cand_v[wid] = nbest; cand_i[wid] = nbi; }
    if (t + 1 < kb) cta_publish(t + 1);
    cluster.sync();   // next step's publication complete; this step's reads done
  }
  for (int e = tid; e < nr * kb; e += nt) {
    const int il = e / kb, t = e - il * kb;
    M[(int64_t)(r0 + il) * n + k0 + t] = P[t * R + il];
  }
  cluster.sync();     // panel columns of M complete before the row snapshots
  if (cr == 0) {
    for (int i = tid; i < n; i += nt) {
      src_out[i] = src[i];
      rowslot[i] = -1;
    }
    __syncthreads();
    if (tid == 0) {
      int q = 0;
      for (int a = 0; a < s_ntouch; ++a) {
        const int r = src[touched[a]];
        bool seen = false;
        for (int c = 0; c < q; ++c) seen = seen || srows[c] == r;
        if (!seen) {
          rowslot[r] = q;
          srows[q++] = r;
        }
      }
      s_ntouch = q;
    }
  }
  cluster.sync();     // snapshot row list ready in rank 0
  // every CTA copies its share of the snapshot rows, eight loads in flight
  const int nsr = *cluster.map_shared_rank(&s_ntouch, 0);
  if (tid < nsr) touched[tid] = *cluster.map_shared_rank(&srows[tid], 0);
  __syncthreads();
  const int64_t ncopy = (int64_t)nsr * n;
  const int64_t gstride = (int64_t)C * nt;
  for (int64_t e0 = (int64_t)cr * nt + tid; e0 < ncopy; e0 += LB * gstride) {
    double v[LB];
#pragma unroll
    for (int u = 0; u < LB; ++u) {
      const int64_t e = e0 + u * gstride;
      if (e < ncopy) {
        const int q = (int)(e / n), j = (int)(e - (int64_t)q * n);
        v[u] = M[(int64_t)touched[q] * n + j];
      }
    }
#pragma unroll
    for (int u = 0; u < LB; ++u)
      if (e0 + u * gstride < ncopy) slab[e0 + u * gstride] = v[u];
  }
  cluster.sync();     // rank 0's shared memory stays valid until every CTA has read it
}

// rank-kb application of a factorised panel to the other columns (see
// gj_panel_kernel).  CTA tile: 32 rows x 128 columns, thread = one column x
// 16 rows (coalesced row segments); the tile's permutation sources, panel
// coefficients and pivot-row segments are staged in shared memory.
template <int KBM>
__global__ void __launch_bounds__(256) gj_update_kernel(double* M, int n, int k0, int kb,
                                                        const int* __restrict__ src,
                                                        const double* __restrict__ slab,
                                                        const int* __restrict__ rowslot,
                                                        const int64_t* status) {
  __shared__ double sK[KBM][128];
  __shared__ double cf[32][KBM + 1];
  __shared__ int kslot[KBM], rsrc[32];
  {   // batched use: matrix blockIdx.z
    const int64_t bat = blockIdx.z;
    M += bat * n * n;
    src += bat * n;
    rowslot += bat * n;
    slab += bat * 2 * KBM * n;
    status += bat;
  }
  if (*status != 0) return;
  const int i0 = blockIdx.y * 32, j0 = blockIdx.x * 128, tid = threadIdx.x;
  if (tid < kb) kslot[tid] = rowslot[src[k0 + tid]];
  if (tid >= 64 && tid < 96) {
    const int i = i0 + tid - 64;
    // -2: pivot position (no base term), -1: unmoved row, else slab row
    rsrc[tid - 64] = i >= n ? -2 : (i >= k0 && i < k0 + kb) ? -2
                                 : (src[i] == i ? -1 : rowslot[src[i]]);
  }
  for (int e = tid; e < 32 * kb; e += 256) {
    const int r = e / kb, s2 = e - r * kb, i = i0 + r;
    cf[r][s2] = i < n ? M[(int64_t)i * n + k0 + s2] : 0.0;
  }
  __syncthreads();
  for (int e = tid; e < kb * 128; e += 256) {
    const int s2 = e >> 7, jj = e & 127, j = j0 + jj;
    sK[s2][jj] = j < n ? slab[(int64_t)kslot[s2] * n + j] : 0.0;
  }
  __syncthreads();
  const int jj = tid & 127, j = j0 + jj;
  if (j >= n || (j >= k0 && j < k0 + kb)) return;
  // this thread's column of the pivot-row segments, reused for its 16 rows
  double sk[KBM];
#pragma unroll
  for (int s2 = 0; s2 < KBM; ++s2) sk[s2] = s2 < kb ? sK[s2][jj] : 0.0;
#pragma unroll 4
  for (int r = tid >> 7; r < 32; r += 2) {
    const int i = i0 + r;
    if (i >= n) break;
    const int rs = rsrc[r];
    double acc = rs == -2 ? 0.0 : (rs == -1 ? M[(int64_t)i * n + j] : slab[(int64_t)rs * n + j]);
#pragma unroll
    for (int s2 = 0; s2 < KBM; ++s2)
      if (s2 < kb) acc = fma(cf[r][s2], sk[s2], acc);
    M[(int64_t)i * n + j] = acc;
  }
}

// (skipped after a zero pivot: the pivot list is then incomplete)
__global__ void gj_unscramble_kernel(double* M, int64_t n, const int64_t* perm,
                                     const int64_t* status) {
  M += (int64_t)blockIdx.y * n * n;     // batched use: matrix blockIdx.y
  perm += (int64_t)blockIdx.y * n;
  status += blockIdx.y;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || *status != 0) return;
  double* row = M + i * n;
  for (int64_t k = n - 1; k >= 0; --k) {
    const int64_t p = perm[k];
    if (p != k) {
      const double t = row[k];
      row[k] = row[p];
      row[p] = t;
    }
  }
}

// warp per row; lane j sums columns j, j + 32, ... (fixed order: this
// order is part of the parity — a two-accumulator variant moved the 3d_tiny
// GMRES history from ~1e-12 to 1.03e-10 of the reference's, whose own
// BLAS-thread spread there is 6e-11).  Rows padded to ld % 4 == 0 are read
// as 32-byte quads, 128 columns per warp step, and handed to the lanes in
// that order through a 1 KiB shared-memory transpose: the same FMA sequence
// with a quarter of the load instructions.
__global__ void __launch_bounds__(256) dense_matvec_kernel(int64_t n, const double* __restrict__ M,
                                                           int64_t ld,
                                                           const double* __restrict__ x,
                                                           double* __restrict__ y) {
  pdl_entry();
  __shared__ double sq[8][128];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (row >= n) return;
  const double* r = M + row * ld;
  double acc = 0.0;
  for (int64_t c0 = 0; c0 < n; c0 += 128) {
    const int64_t q = c0 + 4 * lane;
    d4 v = {0.0, 0.0, 0.0, 0.0};
    if (q < ld) v = ld256_ro(r + q);
    sq[w][4 * lane] = v.x;
    sq[w][4 * lane + 1] = v.y;
    sq[w][4 * lane + 2] = v.z;
    sq[w][4 * lane + 3] = v.w;
    __syncwarp();
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int64_t j = c0 + lane + 32 * m;
      if (j < n) acc = fma(sq[w][lane + 32 * m], __ldg(x + j), acc);
    }
    __syncwarp();
  }
  acc = warp_sum(acc);
  if (lane == 0) y[row] = acc;
}

__global__ void pad_rows_kernel(int64_t n, const double* __restrict__ M, int64_t ld,
                                double* __restrict__ P) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * ld;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / ld, j = e - i * ld;
    P[e] = j < n ? M[i * n + j] : 0.0;
  }
}

// --------------------------------------------------------------------------
// Krylov vector kernels.  Two-stage fixed-order reductions: kRedBlocks
// partial sums per output, then one CTA per output sums its partials.
// --------------------------------------------------------------------------
constexpr int kBatch = 8;

// VW = 4: every thread streams 32-byte quads (one LDG.256 per vector) so
// that a warp keeps (nvec + 1) KiB in flight per iteration; w.w is folded
// into the first pass.  VW = 1: scalar path for lengths that are not a
// multiple of 4 (2D).  Fixed element-to-thread map: deterministic.
template <int VW>
__global__ void __launch_bounds__(256) multi_dot_kernel(const GmresCtl* __restrict__ ctl,
                                                        const double* __restrict__ V,
                                                        int64_t ldv, const double* __restrict__ w,
                                                        int64_t n, double* __restrict__ partial,
                                                        const int* flag) {
  pdl_entry();
  if (flag != nullptr && *flag == 0) return;
  __shared__ double red[8];
  const int nvec = ctl->k + 1;            // basis vectors v_0 .. v_k
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gs = (int64_t)gridDim.x * blockDim.x;
  const int nout = nvec + 1;
  const int64_t nv = n / VW;
  double sq = 0.0;
  for (int j0 = 0; j0 < nvec || j0 == 0; j0 += kBatch) {
    double acc[kBatch];
#pragma unroll
    for (int q = 0; q < kBatch; ++q) acc[q] = 0.0;
    for (int64_t i = gt; i < nv; i += gs) {
      if constexpr (VW == 4) {
        const d4 wi = ld256_ro(w + 4 * i);
        if (j0 == 0) {
          sq = fma(wi.x, wi.x, sq);
          sq = fma(wi.y, wi.y, sq);
          sq = fma(wi.z, wi.z, sq);
          sq = fma(wi.w, wi.w, sq);
        }
#pragma unroll
        for (int q = 0; q < kBatch; ++q)
          if (j0 + q < nvec) {
            const d4 v = ld256_ro(V + (int64_t)(j0 + q) * ldv + 4 * i);
            acc[q] = fma(v.x, wi.x, acc[q]);
            acc[q] = fma(v.y, wi.y, acc[q]);
            acc[q] = fma(v.z, wi.z, acc[q]);
            acc[q] = fma(v.w, wi.w, acc[q]);
          }
      } else {
        const double wi = __ldg(w + i);
        if (j0 == 0) sq = fma(wi, wi, sq);
#pragma unroll
        for (int q = 0; q < kBatch; ++q)
          if (j0 + q < nvec) acc[q] = fma(__ldg(V + (int64_t)(j0 + q) * ldv + i), wi, acc[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < kBatch; ++q) {
      if (j0 + q >= nvec) break;
      const double s = block_sum_256(acc[q], red);
      if (threadIdx.x == 0) partial[(int64_t)blockIdx.x * nout + j0 + q] = s;
    }
  }
  const double s = block_sum_256(sq, red);
  if (threadIdx.x == 0) partial[(int64_t)blockIdx.x * nout + nvec] = s;
}

// out[j] = sum of the blocks' partials j, one CTA per output; nout = k + 2
// (multi_dot) when ctl is given, else the fixed count
__global__ void __launch_bounds__(256) reduce_partials_kernel(int nout, int nblocks,
                                                              const double* __restrict__ partial,
                                                              double* __restrict__ out,
                                                              const int* flag,
                                                              const GmresCtl* ctl) {
  pdl_entry();
  if (flag != nullptr && *flag == 0) return;
  if (ctl != nullptr) nout = ctl->k + 2;
  const int j = blockIdx.x;
  if (j >= nout) return;
  __shared__ double red[8];
  double acc = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += blockDim.x) acc += partial[(int64_t)b * nout + j];
  const double s = block_sum_256(acc, red);
  if (threadIdx.x == 0) out[j] = s;
}

template <int VW>
__global__ void __launch_bounds__(256) multi_axpy_kernel(const GmresCtl* __restrict__ ctl,
                                                         const double* __restrict__ V,
                                                         int64_t ldv, const double* __restrict__ h,
                                                         double* __restrict__ w, int64_t n,
                                                         double* __restrict__ partial,
                                                         const int* flag) {
  pdl_entry();
  if (flag != nullptr && *flag == 0) return;
  __shared__ double hs[512];
  __shared__ double red[8];
  const int nvec = ctl->k + 1;
  for (int j = threadIdx.x; j < nvec; j += blockDim.x) hs[j] = h[j];
  __syncthreads();
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gs = (int64_t)gridDim.x * blockDim.x;
  double sq = 0.0;
  if constexpr (VW == 4) {
    for (int64_t i = gt; i < n / 4; i += gs) {
      d4 acc = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 4
      for (int j = 0; j < nvec; ++j) {
        const double hj = hs[j];
        const d4 v = ld256_ro(V + (int64_t)j * ldv + 4 * i);
        acc.x = fma(hj, v.x, acc.x);
        acc.y = fma(hj, v.y, acc.y);
        acc.z = fma(hj, v.z, acc.z);
        acc.w = fma(hj, v.w, acc.w);
      }
      double2* wp = reinterpret_cast<double2*>(w + 4 * i);
      double2 a = wp[0], b = wp[1];
      a.x -= acc.x;
      a.y -= acc.y;
      b.x -= acc.z;
      b.y -= acc.w;
      wp[0] = a;
      wp[1] = b;
      sq = fma(a.x, a.x, sq);
      sq = fma(a.y, a.y, sq);
      sq = fma(b.x, b.x, sq);
      sq = fma(b.y, b.y, sq);
    }
  } else {
    for (int64_t i = gt; i < n; i += gs) {
      double acc = 0.0;
      for (int j = 0; j < nvec; ++j) acc = fma(hs[j], __ldg(V + (int64_t)j * ldv + i), acc);
      const double wi = w[i] - acc;
      w[i] = wi;
      sq = fma(wi, wi, sq);
    }
  }
  const double s = block_sum_256(sq, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// stage 0: decide re-orthogonalisation (Kahan test of linsolve.py:79-83,
// ||w|| after the first pass vs hcol[k+1] = ||w||^2 before it);
// stage 1: fold the second projection into the Hessenberg column and set
// H[k+1, k] = ||w||.
__global__ void arnoldi_finish_kernel(GmresCtl* ctl, double* hcol, const double* h2,
                                      const double* na2, int stage) {
  pdl_entry();
  const int k = ctl->k;
  if (stage == 0) {
    if (threadIdx.x == 0) ctl->flag = (sqrt(*na2) < 0.7071 * sqrt(hcol[k + 1])) ? 1 : 0;
    return;
  }
  if (ctl->flag)
    for (int j = threadIdx.x; j <= k; j += blockDim.x) hcol[j] += h2[j];
  __syncthreads();
  if (threadIdx.x == 0) hcol[k + 1] = sqrt(*na2);
}

// v_{k+1} = w / H[k+1, k] (linsolve.py:85-86), also into the V-cycle's input
// buffer for the next Arnoldi step
__global__ void scale_copy_slot_kernel(const GmresCtl* __restrict__ ctl,
                                       const double* __restrict__ w, double* __restrict__ V,
                                       int64_t ldv, const double* __restrict__ hcol,
                                       double* __restrict__ vin, int64_t n) {
  pdl_entry();
  const int k = ctl->k;
  const double h = hcol[k + 1];
  if (!(h > 0.0)) return;
  double* v = V + (int64_t)(k + 1) * ldv;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double t = w[i] / h;
    v[i] = t;
    vin[i] = t;
  }
}

// beta = ||b||, tolerance, early exit (linsolve.py:55-60); v_0 = b / beta
__global__ void gmres_init_kernel(GmresCtl* ctl, const double* bb, double* res, double* g,
                                  cudaGraphConditionalHandle cond, int use_cond) {
  pdl_entry();
  const double beta = sqrt(*bb);
  const double tol = fmax(ctl->rel_tol * beta, ctl->abs_tol);
  const int stop = (beta == 0.0 || beta <= tol) ? 1 : 0;
  ctl->beta = beta;
  ctl->tol = tol;
  ctl->k = 0;
  ctl->its = 0;
  ctl->done = stop;
  ctl->converged = 1;
  res[0] = beta;
  g[0] = beta;
  if (use_cond) cudaGraphSetConditional(cond, stop ? 0u : 1u);
}

__global__ void scale_dual_kernel(const GmresCtl* __restrict__ ctl, const double* __restrict__ b,
                                  double* __restrict__ v0, double* __restrict__ vin, int64_t n) {
  pdl_entry();
  if (ctl->done) return;
  const double beta = ctl->beta;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double t = b[i] / beta;
    v0[i] = t;
    vin[i] = t;
  }
}

// Hessenberg column k, accumulated Givens rotations and the new one, the
// residual estimate |g[k+1]| and the stopping test (linsolve.py:88-102);
// H is (hstride + 1) x hstride row-major.  Sets the while-node condition.
__global__ void givens_kernel(GmresCtl* ctl, const double* __restrict__ hcol, double* H,
                              double* cs, double* sn, double* g, double* res,
                              cudaGraphConditionalHandle cond, int use_cond) {
  pdl_entry();
  const int k = ctl->k, m = ctl->hstride;
  auto Hat = [&](int i, int j) -> double& { return H[(int64_t)i * m + j]; };
  for (int i = 0; i <= k + 1; ++i) Hat(i, k) = hcol[i];
  for (int i = 0; i < k; ++i) {
    const double t = cs[i] * Hat(i, k) + sn[i] * Hat(i + 1, k);
    Hat(i + 1, k) = -sn[i] * Hat(i, k) + cs[i] * Hat(i + 1, k);
    Hat(i, k) = t;
  }
  const double r = hypot(Hat(k, k), Hat(k + 1, k));
  cs[k] = Hat(k, k) / r;
  sn[k] = Hat(k + 1, k) / r;
  Hat(k, k) = r;
  Hat(k + 1, k) = 0.0;
  g[k + 1] = -sn[k] * g[k];
  g[k] = cs[k] * g[k];
  const double rr = fabs(g[k + 1]);
  res[k + 1] = rr;
  const int conv = rr <= ctl->tol ? 1 : 0;
  const int stop = conv || k + 1 >= ctl->max_iter;
  ctl->its = k + 1;
  ctl->converged = conv;
  ctl->done = stop;
  ctl->k = k + 1;
  if (use_cond) cudaGraphSetConditional(cond, stop ? 0u : 1u);
}

// y = triu(H)^{-1} g (linsolve.py:107), column-oriented back substitution
__global__ void backsolve_kernel(const GmresCtl* ctl, const double* H, const double* g,
                                 double* y) {
  pdl_entry();
  const int its = ctl->its, m = ctl->hstride;
  for (int j = 0; j < its; ++j) y[j] = g[j];
  for (int j = its - 1; j >= 0; --j) {
    y[j] /= H[(int64_t)j * m + j];
    for (int i = 0; i < j; ++i) y[i] -= y[j] * H[(int64_t)i * m + j];
  }
}

// out = sum_j c[j] V[j] over the its basis vectors (V y of linsolve.py:108)
__global__ void combine_kernel(const GmresCtl* __restrict__ ctl, const double* __restrict__ V,
                               int64_t ldv, const double* __restrict__ c, double* __restrict__ y,
                               int64_t n) {
  pdl_entry();
  __shared__ double cs[512];
  const int nvec = ctl->its;
  for (int j = threadIdx.x; j < nvec; j += blockDim.x) cs[j] = c[j];
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int j = 0; j < nvec; ++j) acc = fma(cs[j], __ldg(V + (int64_t)j * ldv + i), acc);
    y[i] = acc;
  }
}

__global__ void __launch_bounds__(256) sumsq_kernel(const double* __restrict__ x, int64_t n,
                                                    double* __restrict__ partial) {
  pdl_entry();
  __shared__ double red[8];
  double sq = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    sq = fma(x[i], x[i], sq);
  const double s = block_sum_256(sq, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

template <int NC>
void spmv_dispatch(const DevMatrix& A, const double* x, const double* b, double* y, int mode,
                   cudaStream_t s) {
  const int grid = grid_for(A.n_nodes * 32, 256);
  if constexpr (NC == 3) {
    if (A.sell_off != nullptr) {
      const int sgrid = grid_for(A.n_slices * 32, 256);
      auto k = A.sell_lanes == 4 ? (mode == 0 ? spmv3_sell_kernel<0, 4> : spmv3_sell_kernel<1, 4>)
             : A.sell_lanes == 2 ? (mode == 0 ? spmv3_sell_kernel<0, 2> : spmv3_sell_kernel<1, 2>)
                                 : (mode == 0 ? spmv3_sell_kernel<0, 1> : spmv3_sell_kernel<1, 1>);
      launch_pdl(k, sgrid, 256, 0, s, A.n_nodes, A.n_slices, A.sell_off, A.sell_col, A.sell_val,
                 A.sell_poff, A.sell_pcol, A.sell_pval, x, b, y);
      return;
    }
    const int hgrid = grid_for(A.n_nodes * 16, 256);
    if (mode == 0)
      launch_pdl(spmv_half_kernel<NC, 0>, hgrid, 256, 0, s, A.n_nodes, A.indptr, A.indices, A.data,
                                                    A.pp_indptr, A.pp_indices, A.pp_data, x, b, y);
    else
      launch_pdl(spmv_half_kernel<NC, 1>, hgrid, 256, 0, s, A.n_nodes, A.indptr, A.indices, A.data,
                                                    A.pp_indptr, A.pp_indices, A.pp_data, x, b, y);
    return;
  }
  if constexpr (NC % 2 == 0) {
    const bool idx32 = A.nnzb * NC * NC < ((int64_t)1 << 31) && A.nnz_pp < ((int64_t)1 << 31) &&
                       A.n_nodes * NC < ((int64_t)1 << 31);
    if (idx32 && NC == 4) {
      const bool unr = A.n_nodes < kSmallLevelNodes;
      auto k = unr ? (mode == 0 ? spmv4_kernel<0, true> : spmv4_kernel<1, true>)
                   : (mode == 0 ? spmv4_kernel<0, false> : spmv4_kernel<1, false>);
      launch_pdl(k, grid, 256, 0, s, A.n_nodes, A.indptr, A.indices, A.data, A.pp_indptr, A.pp_indices,
                             A.pp_data, x, b, y);
      return;
    }
    if (idx32) {
      if (mode == 0)
        launch_pdl(spmv32_kernel<NC, 0>, grid, 256, 0, s, A.n_nodes, A.indptr, A.indices, A.data,
                                                  A.pp_indptr, A.pp_indices, A.pp_data, x, b, y);
      else
        launch_pdl(spmv32_kernel<NC, 1>, grid, 256, 0, s, A.n_nodes, A.indptr, A.indices, A.data,
                                                  A.pp_indptr, A.pp_indices, A.pp_data, x, b, y);
      return;
    }
  }
  if (mode == 0)
    launch_pdl(spmv_kernel<NC, 0>, grid, 256, 0, s, A.n_nodes, A.indptr, A.indices, A.data, A.pp_indptr,
                                            A.pp_indices, A.pp_data, x, b, y);
  else
    launch_pdl(spmv_kernel<NC, 1>, grid, 256, 0, s, A.n_nodes, A.indptr, A.indices, A.data, A.pp_indptr,
                                            A.pp_indices, A.pp_data, x, b, y);
}

template <int NP, int LD, int NC>
void apply_dispatch(const DevPatchGroup* g, int ng, const double* d, double* Y, int split,
                    cudaStream_t s) {
  bool v4 = false;
  if constexpr (LD % 4 == 0) {
    v4 = true;
    for (int i = 0; i < ng; ++i)
      v4 = v4 && reinterpret_cast<uintptr_t>(g[i].inv) % 32 == 0 &&
           reinterpret_cast<uintptr_t>(Y + g[i].y_offset) % 32 == 0;
  }
  ApplyGroups G{};
  const int ppc = v4 ? ApplyShape<LD, 4>::PPC : ApplyShape<LD, 2>::PPC;
  int grid = 0;
  for (int i = 0; i < 2; ++i) {
    const DevPatchGroup& gg = g[i < ng ? i : 0];
    G.n_patches[i] = i < ng ? gg.n_patches : 0;
    G.nodes[i] = gg.nodes;
    G.inv[i] = gg.inv;
    G.y[i] = Y + gg.y_offset;
    const int b = i < ng ? grid_for(gg.n_patches, ppc) : 0;
    if (i == 0) G.blocks0 = b;
    grid += b;
  }
  if (grid == 0) return;
  const int64_t total = G.n_patches[0] + G.n_patches[1];
  // column-split form: by default for launches of < kSmallPatchCount patches
  // (L2-resident levels); split = 0 / 1 forces the choice (tuning)
  const bool use_split = NP <= 108 && (split < 0 ? total < kSmallPatchCount : split > 0);
  if (use_split) {
    // one CTA per patch, 4 column splits
    G.blocks0 = (int)G.n_patches[0];
    const int sgrid = (int)total;
    if constexpr (LD % 4 == 0) {
      if (v4) {
        launch_pdl(vanka_apply_split_kernel<NP, LD, NC, 4, 4>, sgrid, ApplyShape<LD, 4>::TPP * 4, 0, s, G, d);
        return;
      }
    }
    launch_pdl(vanka_apply_split_kernel<NP, LD, NC, 2, 4>, sgrid, ApplyShape<LD, 2>::TPP * 4, 0, s, G, d);
    return;
  }
  if constexpr (LD % 4 == 0) {
    if (v4) {
      launch_pdl(vanka_apply_kernel<NP, LD, NC, 4>, grid, ApplyShape<LD, 4>::BLK, 0, s, G, d);
      return;
    }
  }
  launch_pdl(vanka_apply_kernel<NP, LD, NC, 2>, grid, ApplyShape<LD, 2>::BLK, 0, s, G, d);
}

// batched blocked Gauss-Jordan for the 500 x 500 macro patches (big_* and gj_*
// kernels).  work: vanka_factorize_work(np, n_patches) doubles from the handle
// (perm | src | rowslot | panel slabs | per-patch status), no allocation,
// no synchronisation.
constexpr int kBigKB = 16;

void factorize_big(const DevMatrix& A, const DevPatchGroup& g, int64_t* status, cudaStream_t s) {
  const int n = g.np;
  const int64_t P = g.n_patches;
  double* M = g.inv;                                   // ld == np (checked by the caller)
  int64_t* perm = reinterpret_cast<int64_t*>(g.work);
  int* src = reinterpret_cast<int*>(perm + P * n);
  int* rowslot = src + P * n;
  double* slab = reinterpret_cast<double*>(rowslot + P * n);
  int64_t* pstatus = reinterpret_cast<int64_t*>(slab + P * 2 * kBigKB * n);
  static bool attr = [] {
    cudaFuncSetAttribute(gj_panel_kernel<kBigKB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         225 * 1024);
    return true;
  }();
  (void)attr;
  cudaMemsetAsync(pstatus, 0, sizeof(int64_t) * P, s);
  big_gather_kernel<<<dim3(32, (unsigned)P), 256, 0, s>>>(A, n, g.npn, g.nodes, M);
  const size_t smem = (size_t)n * kBigKB * 8 + (size_t)n * 4;
  const dim3 ug((unsigned)grid_for(n, 128), (unsigned)grid_for(n, 32), (unsigned)P);
  for (int k0 = 0; k0 < n; k0 += kBigKB) {
    const int kb = std::min(kBigKB, n - k0);
    gj_panel_kernel<kBigKB><<<(unsigned)P, 512, smem, s>>>(M, n, k0, kb, perm, src, slab,
                                                           rowslot, pstatus);
    gj_update_kernel<kBigKB><<<ug, 256, 0, s>>>(M, n, k0, kb, src, slab, rowslot, pstatus);
  }
  gj_unscramble_kernel<<<dim3((unsigned)grid_for(n, 128), (unsigned)P), 128, 0, s>>>(
      M, n, perm, pstatus);
  big_finish_kernel<<<dim3(32, (unsigned)P), 256, 0, s>>>(n, M, pstatus, status);
}

template <int NP, int NC, int W, int NPAT>
void factorize_cw_dispatch(const DevMatrix& A, const DevPatchGroup& g, int64_t* status,
                           cudaStream_t s) {
  const unsigned grid = (unsigned)((g.n_patches + NPAT - 1) / NPAT);
  vanka_factorize_cw_kernel<NP, NC, W, NPAT><<<grid, 32 * W, 0, s>>>(
      A, g.n_patches, g.nodes, g.inv, g.ld, status);
}

template <int NP, int NC, int W, int MINB>
void factorize_pw_dispatch(const DevMatrix& A, const DevPatchGroup& g, int64_t* status,
                           cudaStream_t s) {
  vanka_factorize_pw_kernel<NP, NC, W, MINB><<<(unsigned)g.n_patches, 32 * W, 0, s>>>(
      A, g.n_patches, g.slots, g.inv, g.ld, status);
}

}  // namespace

void launch_spmv(const DevMatrix& A, const double* x, const double* b, double* y, int mode,
                 cudaStream_t s) {
  if (A.n_nodes == 0) return;
  if (A.nc == 4) spmv_dispatch<4>(A, x, b, y, mode, s);
  else if (A.nc == 3) spmv_dispatch<3>(A, x, b, y, mode, s);
  else if (A.nc == 2) spmv_dispatch<2>(A, x, b, y, mode, s);
}

void launch_sell_pack(int64_t n_pos, int R, int nc2, const int64_t* map, const double* data,
                      double* val, cudaStream_t s) {
  if (n_pos == 0) return;
  sell_pack_kernel<<<(int)std::min<int64_t>(grid_for(n_pos, 256), 4 * 148 * 8), 256, 0, s>>>(
      n_pos, R, nc2, map, data, val);
}

bool vanka_uses_slots(int np) { return np == 75 || np == 108; }

void launch_patch_slots(const DevMatrix& A, const DevPatchGroup& g, int32_t* slots,
                        cudaStream_t s) {
  const int64_t n = g.n_patches * g.npn * g.npn;
  if (n == 0) return;
  patch_slots_kernel<<<(unsigned)grid_for(n, 256), 256, 0, s>>>(A, g.n_patches, g.npn, g.nodes,
                                                               slots);
}

int64_t vanka_factorize_work(int np, int64_t n_patches) {
  if (np != 500) return 0;   // register kernels need no scratch
  // perm (int64) + src, rowslot (int) + 2 KB slab rows + status, in doubles
  return n_patches * ((int64_t)np * (2 + 2 * kBigKB) + 1);
}

bool vanka_supported(int nc, int np) {
  return (nc == 3 && (np == 27 || np == 75 || np == 81)) ||
         (nc == 4 && (np == 108 || np == 500)) || (nc == 2 && np == 18);
}

void launch_vanka_factorize(const DevMatrix& A, const DevPatchGroup& g, int64_t* status,
                            cudaStream_t s) {
  if (g.n_patches == 0) return;
  if (A.nc == 3 && g.np == 27) factorize_cw_dispatch<27, 3, 3, 2>(A, g, status, s);
  // 75x75 and 108x108: the second form (fat warps, mbarrier ring).  Config 3
  // Vanka + coarse factorisation 103.3 -> 61.2 ms, config 1 50.3 -> 43.1 ms
  // against the column-strided kernel with two block barriers per step.
  else if (A.nc == 3 && g.np == 75) factorize_pw_dispatch<75, 3, 5, 3>(A, g, status, s);
  else if (A.nc == 4 && g.np == 108) factorize_pw_dispatch<108, 4, 6, 2>(A, g, status, s);
  else if (A.nc == 2 && g.np == 18) factorize_cw_dispatch<18, 2, 2, 2>(A, g, status, s);
  else if (A.nc == 3 && g.np == 81) factorize_cw_dispatch<81, 3, 9, 2>(A, g, status, s);
  else if (A.nc == 4 && g.np == 500 && g.ld == g.np && g.work != nullptr)
    factorize_big(A, g, status, s);
}

// one launch per pair of consecutive groups with the same patch size;
// returns the number of launches
int launch_vanka_apply(const DevPatchGroup* groups, int n_groups, int nc, const double* d,
                       double* Y, int split, cudaStream_t s) {
  int launches = 0;
  for (int i = 0; i < n_groups;) {
    const DevPatchGroup& g = groups[i];
    const int ng = (i + 1 < n_groups && groups[i + 1].np == g.np && groups[i + 1].ld == g.ld)
                       ? 2 : 1;
    const DevPatchGroup* gp = groups + i;
    i += ng;
    if (g.n_patches == 0 && (ng == 1 || gp[1].n_patches == 0)) continue;
    if (nc == 3 && g.np == 27) apply_dispatch<27, 28, 3>(gp, ng, d, Y, split, s);
    else if (nc == 3 && g.np == 75) apply_dispatch<75, 76, 3>(gp, ng, d, Y, split, s);
    else if (nc == 4 && g.np == 108) apply_dispatch<108, 108, 4>(gp, ng, d, Y, split, s);
    else if (nc == 2 && g.np == 18) apply_dispatch<18, 18, 2>(gp, ng, d, Y, split, s);
    else if (nc == 3 && g.np == 81) apply_dispatch<81, 82, 3>(gp, ng, d, Y, split, s);
    else if (nc == 4 && g.np == 500) apply_dispatch<500, 500, 4>(gp, ng, d, Y, split, s);
    else continue;
    ++launches;
  }
  return launches;
}

void launch_vanka_gather(int64_t n_nodes, int nc, const int64_t* gptr, const int64_t* goff,
                         const double* weight, const double* Y, double* x, double omega,
                         int init_zero, cudaStream_t s) {
  const int64_t ndof = n_nodes * nc;
  if (ndof == 0) return;
  // large levels only: up to ~10^5 nodes a thread per dof (4x the threads)
  // is as fast or faster (140k nodes: 0.0114 vs 0.0121 ms)
  if (nc == 4 && n_nodes >= 4 * kSmallLevelNodes &&
      reinterpret_cast<uintptr_t>(Y) % 32 == 0 &&
      reinterpret_cast<uintptr_t>(x) % 32 == 0) {
    launch_pdl(vanka_gather4_kernel, grid_for(n_nodes, 256), 256, 0, s, n_nodes, gptr, goff, weight, Y,
                                                                 x, omega, init_zero);
    return;
  }
  launch_pdl(vanka_gather_kernel, grid_for(ndof, 256), 256, 0, s, ndof, nc, gptr, goff, weight, Y, x,
                                                           omega, init_zero);
}

void launch_restrict(int64_t n_coarse, int nc, const int64_t* ptr, const int32_t* idx,
                     const double* val, const double* r_fine, const uint8_t* constrained_coarse,
                     double* b_coarse, cudaStream_t s) {
  // restriction rows are long (a coarse node collects ~100 fine nodes): a
  // thread per (row, component), or 8 lanes per (row, component) on small levels
  if (n_coarse < kSmallLevelNodes)
    launch_pdl(transfer_split_kernel, grid_for(n_coarse * nc * 8, 256), 256, 0, s, 
        n_coarse, nc, ptr, idx, val, r_fine, constrained_coarse, b_coarse, 0);
  else
    launch_pdl(transfer_kernel, grid_for(n_coarse * nc, 256), 256, 0, s, 
        n_coarse, nc, ptr, idx, val, r_fine, constrained_coarse, b_coarse, 0);
}

void launch_prolong_add(int64_t n_fine, int nc, const int64_t* ptr, const int32_t* idx,
                        const double* val, const double* x_coarse,
                        const uint8_t* constrained_fine, double* x_fine, cudaStream_t s) {
  if (nc == 4 && vec4_ok(x_coarse, 0, 4) && vec4_ok(x_fine, 0, 4))
    launch_pdl(transfer4_kernel, grid_for(n_fine, 128), 128, 0, s, n_fine, ptr, idx, val, x_coarse,
                                                           constrained_fine, x_fine, 1);
  else
    launch_pdl(transfer_kernel, grid_for(n_fine * nc, 256), 256, 0, s, 
        n_fine, nc, ptr, idx, val, x_coarse, constrained_fine, x_fine, 1);
}

// panel width of the blocked Gauss-Jordan: n x nb panel + n ints in shared memory
int gj_panel_width(int64_t n) {
  for (int nb = 16; nb >= 4; nb >>= 1)
    if (n * nb * 8 + n * 4 <= 225 * 1024 && n >= 4 * nb) return nb;
  return 0;
}

// CTAs per cluster panel: 16 (non-portable size, 2d config 0 39.5 -> 37 ms
// vs 8) where the device can co-schedule it, else 8, else 0 = the single-CTA
// panel kernel
int gj_cluster_size() {
  static const int c = [] {
    cudaFuncSetAttribute(gj_panel_cluster_kernel<16>,
                         cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(gj_panel_cluster_kernel<16>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024);
    // largest cluster the device co-schedules with the largest panel share
    // (kGjMaxN rows); none (e.g. no cluster support): single-CTA panels
    for (int cs = 16; cs >= 8; cs /= 2) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute cat[1];
      cat[0].id = cudaLaunchAttributeClusterDimension;
      cat[0].val.clusterDim.x = cs;
      cat[0].val.clusterDim.y = 1;
      cat[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(cs);
      cfg.blockDim = dim3(256);
      cfg.dynamicSmemBytes = (size_t)(kGjMaxN / cs) * 32 * 8 + (size_t)kGjMaxN * 4;
      cfg.attrs = cat;
      cfg.numAttrs = 1;
      int nclusters = 0;
      const bool ok = cudaOccupancyMaxActiveClusters(&nclusters, gj_panel_cluster_kernel<16>,
                                                     &cfg) == cudaSuccess && nclusters > 0;
      cudaGetLastError();   // a refused query leaves no sticky error
      if (ok) return cs;
    }
    return 0;
  }();
  return c;
}
bool gj_cluster_enabled() { return gj_cluster_size() > 0; }

int dense_inverse(double* M, int64_t n, double* work, int64_t* status, cudaStream_t s) {
  // cluster panels: the n x 16 panel spread over 8-16 SMs fits for every n <= kGjMaxN
  // (32-column cluster panels measured slower: config 2 18.2 -> 18.9 ms)
  const bool clus = gj_cluster_enabled() && n >= 128;
  const int nb = clus ? 16 : gj_panel_width(n);
  if (nb > 0 && n <= kGjMaxN) {
    // work: perm (n int64) | src (n int) | rowslot (n int) | slab (2 nb x n)
    int64_t* perm = reinterpret_cast<int64_t*>(work);
    int* src = reinterpret_cast<int*>(work + n);
    int* rowslot = src + n;
    double* slab = work + 2 * n;
    const size_t smem = (size_t)n * nb * 8 + (size_t)n * 4;
    // dynamic + static shared memory must stay within the 227 KB per CTA
    static bool attr = [] {
      cudaFuncSetAttribute(gj_panel_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           225 * 1024);
      cudaFuncSetAttribute(gj_panel_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           225 * 1024);
      cudaFuncSetAttribute(gj_panel_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           225 * 1024);
      return true;
    }();
    (void)attr;
    cudaMemsetAsync(status, 0, sizeof(int64_t), s);
    const dim3 ug((unsigned)grid_for(n, 128), (unsigned)grid_for(n, 32));
    const int kGjCluster = gj_cluster_size() > 0 ? gj_cluster_size() : 8;   // CTAs per panel
    const int R = (int)((n + kGjCluster - 1) / kGjCluster);
    const size_t csmem = (size_t)R * nb * 8 + (size_t)n * 4;
    static bool cattr = [] {
      cudaFuncSetAttribute(gj_panel_cluster_kernel<16>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024);
      cudaFuncSetAttribute(gj_panel_cluster_kernel<16>,
                           cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      return true;
    }();
    (void)cattr;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute cat[1];
    cat[0].id = cudaLaunchAttributeClusterDimension;
    cat[0].val.clusterDim.x = kGjCluster;
    cat[0].val.clusterDim.y = 1;
    cat[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(kGjCluster);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = csmem;
    cfg.stream = s;
    cfg.attrs = cat;
    cfg.numAttrs = 1;
    for (int64_t k0 = 0; k0 < n; k0 += nb) {
      const int kb = (int)std::min<int64_t>(nb, n - k0);
      if (clus)
        cudaLaunchKernelEx(&cfg, gj_panel_cluster_kernel<16>, M, (int)n, (int)k0, kb, R, perm, src,
                           slab, rowslot, status);
      else if (nb == 16)
        gj_panel_kernel<16><<<1, 512, smem, s>>>(M, (int)n, (int)k0, kb, perm, src, slab,
                                                 rowslot, status);
      else if (nb == 8)
        gj_panel_kernel<8><<<1, 512, smem, s>>>(M, (int)n, (int)k0, kb, perm, src, slab,
                                                rowslot, status);
      else
        gj_panel_kernel<4><<<1, 512, smem, s>>>(M, (int)n, (int)k0, kb, perm, src, slab,
                                                rowslot, status);
      gj_update_kernel<16><<<ug, 256, 0, s>>>(M, (int)n, (int)k0, kb, src, slab, rowslot,
                                                status);
    }
    gj_unscramble_kernel<<<grid_for(n, 128), 128, 0, s>>>(M, n, perm, status);
    return 0;
  }
  // work: colk (n doubles) | rp (1 double) | perm (n int64)
  double* colk = work;
  double* rp = work + n;
  int64_t* perm = reinterpret_cast<int64_t*>(work + n + 1);
  cudaMemsetAsync(status, 0, sizeof(int64_t), s);
  if (n > kGjMaxN) return (int)cudaErrorInvalidValue;
  const dim3 grid((unsigned)grid_for((n + 1) / 2, 128), (unsigned)n);
  for (int64_t k = 0; k < n; ++k) {
    gj_pivot_kernel<<<1, 1024, 0, s>>>(M, n, k, perm, colk, rp, status);
    gj_eliminate_kernel<<<grid, 128, 0, s>>>(M, n, k, colk, rp);
  }
  gj_unscramble_kernel<<<grid_for(n, 128), 128, 0, s>>>(M, n, perm, status);
  return 0;
}

void launch_dense_matvec(int64_t n, const double* M, int64_t ld, const double* x, double* y,
                         cudaStream_t s) {
  launch_pdl(dense_matvec_kernel, grid_for(n * 32, 256), 256, 0, s, n, M, ld, x, y);
}

void launch_pad_rows(int64_t n, const double* M, int64_t ld, double* P, cudaStream_t s) {
  pad_rows_kernel<<<(int)std::min<int64_t>(grid_for(n * ld, 256), 4096), 256, 0, s>>>(n, M, ld, P);
}

int launch_multi_dot(GmresCtl* ctl, int max_nvec, const double* V, int64_t ldv, const double* w,
                     int64_t n, double* partial, double* out, const int* flag, cudaStream_t s) {
  if (vec4_ok(V, ldv, n) && vec4_ok(w, 0, n))
    launch_pdl(multi_dot_kernel<4>, kRedBlocks, 256, 0, s, ctl, V, ldv, w, n, partial, flag);
  else
    launch_pdl(multi_dot_kernel<1>, kRedBlocks, 256, 0, s, ctl, V, ldv, w, n, partial, flag);
  launch_pdl(reduce_partials_kernel, max_nvec + 1, 256, 0, s, 0, kRedBlocks, partial, out, flag, ctl);
  return 2;
}

int launch_multi_axpy(GmresCtl* ctl, const double* V, int64_t ldv, const double* h, double* w,
                      int64_t n, double* partial, double* out, const int* flag, cudaStream_t s) {
  if (vec4_ok(V, ldv, n) && vec4_ok(w, 0, n))
    launch_pdl(multi_axpy_kernel<4>, kRedBlocks, 256, 0, s, ctl, V, ldv, h, w, n, partial, flag);
  else
    launch_pdl(multi_axpy_kernel<1>, kRedBlocks, 256, 0, s, ctl, V, ldv, h, w, n, partial, flag);
  launch_pdl(reduce_partials_kernel, 1, 256, 0, s, 1, kRedBlocks, partial, out, flag, nullptr);
  return 2;
}

int launch_arnoldi_finish(GmresCtl* ctl, double* hcol, double* h2, const double* na2, int stage,
                          cudaStream_t s) {
  launch_pdl(arnoldi_finish_kernel, 1, 256, 0, s, ctl, hcol, h2, na2, stage);
  return 1;
}

int launch_scale_copy_slot(const GmresCtl* ctl, const double* w, double* V, int64_t ldv,
                           const double* hcol, double* vin, int64_t n, cudaStream_t s) {
  launch_pdl(scale_copy_slot_kernel, kRedBlocks, 256, 0, s, ctl, w, V, ldv, hcol, vin, n);
  return 1;
}

int launch_gmres_init(GmresCtl* ctl, const double* b, int64_t n, double* partial, double* scal,
                      double* res, double* g, double* v0, double* vin,
                      cudaGraphConditionalHandle cond, int use_cond, cudaStream_t s) {
  launch_pdl(sumsq_kernel, kRedBlocks, 256, 0, s, b, n, partial);
  launch_pdl(reduce_partials_kernel, 1, 256, 0, s, 1, kRedBlocks, partial, scal, nullptr, nullptr);
  launch_pdl(gmres_init_kernel, 1, 1, 0, s, ctl, scal, res, g, cond, use_cond);
  launch_pdl(scale_dual_kernel, kRedBlocks, 256, 0, s, ctl, b, v0, vin, n);
  return 4;
}

int launch_givens(GmresCtl* ctl, const double* hcol, double* H, double* cs, double* sn, double* g,
                  double* res, cudaGraphConditionalHandle cond, int use_cond, cudaStream_t s) {
  launch_pdl(givens_kernel, 1, 1, 0, s, ctl, hcol, H, cs, sn, g, res, cond, use_cond);
  return 1;
}

int launch_gmres_solution(const GmresCtl* ctl, const double* H, const double* g, double* y,
                          const double* V, int64_t ldv, double* out, int64_t n, cudaStream_t s) {
  launch_pdl(backsolve_kernel, 1, 1, 0, s, ctl, H, g, y);
  launch_pdl(combine_kernel, kRedBlocks, 256, 0, s, ctl, V, ldv, y, out, n);
  return 2;
}

}  // namespace alefsi
