// Microbenchmark: HBM streaming rate of a TMA ring (no MMA), to find the per-SM limit that the
// persistent forward's weight stream runs into.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -std=c++17 -o /tmp/tma_probe scripts/tma_probe.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2512_23858_b200/csrc/common.cuh"

using namespace ygg;

YGG_DEV void tma3(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// Each CTA streams `per_cta` boxes (box = kbox k-blocks x 128 rows x 64 cols bf16).
__global__ void probe(const __grid_constant__ CUtensorMap map, int stages, int kbox, long long per_cta, int kb_total,
                      int n_tiles) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t box_bytes = 128 * 128 * kbox;
  uint64_t* full = reinterpret_cast<uint64_t*>(base + stages * box_bytes);
  uint64_t* empty = full + stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const uint64_t pol = policy_evict_first();
  const long long u0 = per_cta * blockIdx.x;
  const int kgroups = kb_total / kbox;
  if (threadIdx.x == 0) {
    int st = 0;
    uint32_t ph = 0;
    for (long long i = 0; i < per_cta; ++i) {
      mbar_wait(&empty[st], ph ^ 1u);
      const long long u = u0 + i;
      const int kg = static_cast<int>(u % kgroups);
      const int nt = static_cast<int>((u / kgroups) % n_tiles);
      mbar_arrive_expect_tx(&full[st], box_bytes);
      if (kbox == 1)
        tma_load_2d(base + st * box_bytes, &map, &full[st], kg * 64, nt * 128, pol);
      else
        tma3(base + st * box_bytes, &map, &full[st], 0, nt * 128, kg * kbox);
      if (++st == stages) { st = 0; ph ^= 1u; }
    }
  } else if (threadIdx.x == 32) {
    int st = 0;
    uint32_t ph = 0;
    for (long long i = 0; i < per_cta; ++i) {
      mbar_wait(&full[st], ph);
      mbar_arrive(&empty[st]);
      if (++st == stages) { st = 0; ph ^= 1u; }
    }
  }
}

int main() {
  const int N = 128256, K = 4096;  // lm_head-sized weight: 1.05 GB
  void* W;
  cudaMalloc(&W, static_cast<size_t>(N) * K * 2);
  cudaMemset(W, 0, static_cast<size_t>(N) * K * 2);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  const int kb_total = K / 64, n_tiles = N / 128;
  const long long units = static_cast<long long>(kb_total) * n_tiles;
  for (int kbox : {1, 2, 4}) {
    CUtensorMap map;
    if (kbox == 1) {
      cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)N};
      cuuint64_t str[1] = {(cuuint64_t)K * 2};
      cuuint32_t box[2] = {64, 128};
      cuuint32_t es[2] = {1, 1};
      enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, W, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
      // [N][K/64][64] viewed as (64 cols, N rows, K/64 kblocks)
      cuuint64_t dims[3] = {64, (cuuint64_t)N, (cuuint64_t)(K / 64)};
      cuuint64_t str[2] = {(cuuint64_t)K * 2, 128};
      cuuint32_t box[3] = {64, 128, (cuuint32_t)kbox};
      cuuint32_t es[3] = {1, 1, 1};
      CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, W, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) { printf("encode kbox=%d failed %d\n", kbox, (int)r); continue; }
    }
    for (int ctas_per_sm : {1, 2}) {
      for (int stages : {2, 4, 6, 8, 12}) {
        const size_t smem = 1024 + static_cast<size_t>(stages) * 16384 * kbox + 2 * stages * 8;
        if (smem * ctas_per_sm > 228 * 1024 - 2048 * ctas_per_sm) continue;
        const int grid = sms * ctas_per_sm;
        const long long per_cta = units / kbox / grid;
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int it = 0; it < 2; ++it) probe<<<grid, 64, smem>>>(map, stages, kbox, per_cta, kb_total, n_tiles);
        cudaEventRecord(a);
        const int reps = 5;
        for (int it = 0; it < reps; ++it) probe<<<grid, 64, smem>>>(map, stages, kbox, per_cta, kb_total, n_tiles);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double bytes = static_cast<double>(per_cta) * grid * 16384 * kbox;
        printf("kbox=%d ctas/sm=%d stages=%2d  %.0f GB/s  (%.1f KB in flight/SM) err=%s\n", kbox, ctas_per_sm, stages,
               bytes / (ms / reps * 1e-3) / 1e9, stages * 16.0 * kbox * ctas_per_sm, cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
