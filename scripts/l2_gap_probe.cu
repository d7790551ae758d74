// Probe: does an L2 prefetch issued while HBM is otherwise idle make a later TMA stream faster?
// Kernel A prefetches the first `pre` bytes of a weight matrix into L2 (bulk prefetch, many CTAs);
// kernel B then TMA-streams `total` bytes starting at the same address.  Compare B's time with and
// without A.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/l2_gap_probe scripts/l2_gap_probe.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2512_23858_b200/csrc/common.cuh"
using namespace ygg;

__global__ void prefetch_k(const char* base, size_t bytes, int mode) {
  const size_t per = (bytes / gridDim.x) & ~size_t(255);
  const char* p = base + per * blockIdx.x;
  if (mode == 0) {  // bulk prefetch in 64 KB pieces by one thread
    if (threadIdx.x == 0)
      for (size_t o = 0; o < per; o += 65536) {
        const uint32_t n = (per - o) < 65536 ? static_cast<uint32_t>(per - o) : 65536u;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p + o), "r"(n) : "memory");
      }
  } else {  // per-line prefetch from all threads
    for (size_t o = threadIdx.x * 128; o < per; o += blockDim.x * 128)
      asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p + o) : "memory");
  }
}

__global__ void stream_k(const __grid_constant__ CUtensorMap map, long long per_cta, int kgroups, int stages) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(base + stages * 16384);
  uint64_t* empty = full + stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_barrier_init();
  }
  __syncthreads();
  const long long u0 = per_cta * blockIdx.x;
  if (threadIdx.x == 0) {
    int st = 0; uint32_t ph = 0;
    for (long long i = 0; i < per_cta; ++i) {
      mbar_wait(&empty[st], ph ^ 1u);
      const long long u = u0 + i;
      mbar_arrive_expect_tx(&full[st], 16384);
      tma_load_2d(base + st * 16384, &map, &full[st], static_cast<int>(u % kgroups) * 64, static_cast<int>(u / kgroups) * 128,
                  policy_evict_first());
      if (++st == stages) { st = 0; ph ^= 1u; }
    }
  } else if (threadIdx.x == 32) {
    int st = 0; uint32_t ph = 0;
    for (long long i = 0; i < per_cta; ++i) {
      mbar_wait(&full[st], ph);
      mbar_arrive(&empty[st]);
      if (++st == stages) { st = 0; ph ^= 1u; }
    }
  }
}

int main() {
  const int N = 28672, K = 4096;  // an 8B gate|up matrix: 235 MB
  void* W; cudaMalloc(&W, (size_t)N * K * 2); cudaMemset(W, 1, (size_t)N * K * 2);
  void* F; cudaMalloc(&F, 512ull << 20);  // L2 flush buffer
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  printf("enc=%p W=%p F=%p err=%s\n", fn, W, F, cudaGetErrorString(cudaGetLastError()));
  fflush(stdout);
  alignas(64) CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)N}; cuuint64_t str[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {64, 128}; cuuint32_t es[2] = {1, 1};
  enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, W, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encoded\n"); fflush(stdout);
  cudaFuncSetAttribute(stream_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int stages = 6, sms = 148, kg = K / 64;
  // stream the first 48 MB (a GEMM's opening window) — each CTA its contiguous share, tile-major
  for (int mb : {16, 48}) {
    const long long units = (long long)mb * (1 << 20) / 16384;
    const long long per = units / sms;
    for (int mode : {-1, 0, 1}) {
      float best = 1e9;
      for (int it = 0; it < 5; ++it) {
        if (it == 0) { printf("mb %d mode %d\n", mb, mode); fflush(stdout); }
        cudaMemset(F, it, 512ull << 20);  // flush L2
        if (mode >= 0) {
          // prefetch exactly the region the stream reads: units are tile-major (128 rows x 64 k)
          // -> rows [0, units/kg*128) x all k: contiguous bytes = rows * K * 2
          const size_t bytes = (size_t)(units / kg + 1) * 128 * K * 2;
          prefetch_k<<<sms, 128>>>((const char*)W, bytes, mode);
          cudaDeviceSynchronize();
          // emulate an idle gap long enough for the prefetch to land
        }
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        stream_k<<<sms, 64, 1024 + stages * 16384 + 2 * stages * 8>>>(map, per, kg, stages);
        if (it == 0) { printf("launched %s\n", cudaGetErrorString(cudaGetLastError())); fflush(stdout); }
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      printf("window %d MB prefetch mode %2d: stream %.1f us (%.0f GB/s)\n", mb, mode, best * 1e3,
             (double)per * sms * 16384 / (best * 1e-3) / 1e9);
    }
  }
  return 0;
}
