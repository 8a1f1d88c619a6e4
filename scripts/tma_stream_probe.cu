// Bulk-copy (cp.async.bulk) streaming probe: GB/s of a persistent
// one-CTA-per-SM global->shared ring as a function of copy size, copies per
// stage and stages in flight.  Development tool (run on the GPU box):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probe scripts/tma_stream_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void wait_bar(uint64_t* bar, uint32_t par, int wmode) {
  if (wmode == 0) {
    asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}" ::"r"(su(bar)), "r"(par) : "memory");
  } else if (wmode == 1) {
    asm volatile("{\n.reg .pred P;\nW: mbarrier.test_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}" ::"r"(su(bar)), "r"(par) : "memory");
  } else {
    asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1, 20;\n@!P bra W;\n}" ::"r"(su(bar)), "r"(par) : "memory");
  }
}

__global__ void __launch_bounds__(288, 1) probe(const char* src, int64_t bytes_per_cta, int stage_bytes,
                                                int nstages, int splits, double* sink, int wmode) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + 196608);
  uint64_t* empty = full + 64;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nstages; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(full + i)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(su(empty + i)));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t n = bytes_per_cta / stage_bytes;
  const char* base = src + blockIdx.x * bytes_per_cta;
  if (warp == 8) {
    if (lane != 0) return;
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    for (int64_t t = 0; t < n; ++t) {
      const int s = (int)(t % nstages);
      if (t >= nstages) {
        const uint32_t par = (uint32_t)(((t / nstages) - 1) & 1);
        wait_bar(empty + s, par, wmode);
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(full + s)), "r"(stage_bytes) : "memory");
      const int piece = stage_bytes / splits;
      for (int q = 0; q < splits; ++q)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                     ::"r"(su(smem + s * stage_bytes + q * piece)), "l"(base + t * stage_bytes + q * piece), "r"(piece),
                     "r"(su(full + s)), "l"(pol) : "memory");
    }
    return;
  }
  double acc = 0.0;
  for (int64_t t = 0; t < n; ++t) {
    const int s = (int)(t % nstages);
    const uint32_t par = (uint32_t)((t / nstages) & 1);
    wait_bar(full + s, par, wmode);
    const double* d = reinterpret_cast<const double*>(smem + s * stage_bytes);
    for (int i = warp * 32 + lane; i < stage_bytes / 8; i += 256) acc += d[i];
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(empty + s)) : "memory");
  }
  if (acc == 12345.0) sink[0] = acc;
}

__global__ void ldg_stream(const double* src, int64_t n4, double* sink) {
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    double a, b, c, d;
    asm volatile("ld.global.L1::no_allocate.L2::evict_first.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(src + 4 * i));
    acc += a + b + c + d;
  }
  if (acc == 12345.0) sink[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t per_cta = (int64_t)48 << 20;   // 48 MiB per CTA -> ~7 GB total
  char* src;
  double* sink;
  cudaMalloc(&src, per_cta * sms);
  cudaMalloc(&sink, 8);
  cudaMemset(src, 0, per_cta * sms);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 196608 + 1024);
  const int sizes[] = {2048, 4096, 8192, 16384, 32768, 49152, 65536};
  const int splits_list[] = {1, 4};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int wm = 0; wm < 3; ++wm)
  for (int sp : splits_list)
    for (int S : sizes) {
      int nst = 196608 / S;
      if (nst > 64) nst = 64;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        probe<<<sms, 288, 196608 + 1024>>>(src, per_cta, S, nst, sp, sink, wm);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep == 1)
          printf("wait %d stage %6d B x %2d stages, %d copies/stage: %.3f ms  %.0f GB/s  (%s)\n", wm, S, nst, sp, ms,
                 (double)per_cta * sms / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
      }
    }
  for (int blocks_per_sm : {4, 8, 16, 32}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      ldg_stream<<<sms * blocks_per_sm, 256>>>((const double*)src, per_cta * sms / 32, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 1) printf("LDG.256 stream, %d CTAs/SM: %.3f ms %.0f GB/s\n", blocks_per_sm, ms, (double)per_cta * sms / ms / 1e6);
    }
  }
  return 0;
}
