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
                      int n_tiles, int pf_mode, int look, int stall_every, int stall_ns, const char* Wbase, int K,
                      const __grid_constant__ CUtensorMap xmap, int xrows) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t box_bytes = 128 * 128 * kbox;
  const uint32_t xbytes = xrows * 128;
  unsigned char* xbase = base + stages * box_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(xbase + stages * xbytes);
  uint64_t* empty = full + stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_barrier_init();
  }
  if (threadIdx.x == 0) *reinterpret_cast<volatile long long*>(empty + stages) = 0;
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
      if (pf_mode && kbox == 1 && i + look < per_cta) {
        const long long v = u0 + i + look;
        const int pk = static_cast<int>(v % kgroups);
        const int pn = static_cast<int>((v / kgroups) % n_tiles);
        if (pf_mode == 1 || pf_mode == 5) {
          asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(&map)),
                       "r"(pk * 64), "r"(pn * 128) : "memory");
        }
      }
      mbar_arrive_expect_tx(&full[st], box_bytes + xbytes);
      if (xrows) tma_load_2d(xbase + st * xbytes, &xmap, &full[st], kg * 64, 0, policy_evict_last());
      if (pf_mode == 5) {  // tensor prefetch + demand load without a cache hint
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
            ::"r"(smem_u32(base + st * box_bytes)), "l"(reinterpret_cast<uint64_t>(&map)), "r"(smem_u32(&full[st])),
            "r"(kg * 64), "r"(nt * 128) : "memory");
      } else if (kbox == 1)
        tma_load_2d(base + st * box_bytes, &map, &full[st], kg * 64, nt * 128, pol);
      else
        tma3(base + st * box_bytes, &map, &full[st], 0, nt * 128, kg * kbox);
      if (++st == stages) { st = 0; ph ^= 1u; }
    }
  } else if (threadIdx.x >= 64 && pf_mode >= 2) {
    // helper warp: prefetch units up to (consumer progress + look) into L2, independent of the ring
    volatile long long* prog = reinterpret_cast<volatile long long*>(empty + stages);
    const int lane = threadIdx.x & 31;
    for (long long j = 0; j < per_cta; ++j) {
      while (j > *prog + look) {}
      const long long v = u0 + j;
      const int pk = static_cast<int>(v % kgroups);
      const int pn = static_cast<int>((v / kgroups) % n_tiles);
      for (int r = lane; r < 128; r += 32) {
        const char* row = Wbase + (static_cast<size_t>(pn) * 128 + r) * K * 2 + pk * 128;
        if (pf_mode == 2) asm volatile("cp.async.bulk.prefetch.L2.global [%0], 128;" ::"l"(row) : "memory");
        else asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(row) : "memory");
      }
    }
  } else if (threadIdx.x == 32) {
    volatile long long* prog = reinterpret_cast<volatile long long*>(empty + stages);
    int st = 0;
    uint32_t ph = 0;
    for (long long i = 0; i < per_cta; ++i) {
      if (stall_every && i % stall_every == 0 && i) {
        const long long t0 = clock64();
        while (clock64() - t0 < static_cast<long long>(stall_ns) * 19 / 10) {}
      }
      mbar_wait(&full[st], ph);
      mbar_arrive(&empty[st]);
      *prog = i;
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
  void* X;
  cudaMalloc(&X, 64 * K * 2);
  cudaMemset(X, 0, 64 * K * 2);
  CUtensorMap xmaps[3];
  for (int xi = 0; xi < 3; ++xi) {
    const int xr = xi == 0 ? 16 : (xi == 1 ? 16 : 64);
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)50};
    cuuint64_t str[1] = {(cuuint64_t)K * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)xr};
    cuuint32_t es[2] = {1, 1};
    enc(&xmaps[xi], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, X, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  const long long units = static_cast<long long>(kb_total) * n_tiles;
  for (int kbox : {1}) {
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
    for (int ctas_per_sm : {1}) {
      for (int stages : {6}) {
       for (int xrows : {0}) for (int st2 : {6}) for (int mode : {0, 1, 5}) for (int look : {0, 16, 48}) for (int stall : {0, 64}) {
        if (mode == 0 && look) continue;
        const int stages_ = st2;
        const size_t smem = 1024 + static_cast<size_t>(st2) * (16384 * kbox + xrows * 128) + 2 * st2 * 8 + 64;
        if (smem * ctas_per_sm > 228 * 1024 - 2048 * ctas_per_sm) continue;
        const int grid = sms * ctas_per_sm;
        const long long per_cta = units / kbox / grid;
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int it = 0; it < 2; ++it) probe<<<grid, 96, smem>>>(map, stages_, kbox, per_cta, kb_total, n_tiles, mode, look, stall, 10000, (const char*)W, K, xmaps[xrows == 64 ? 2 : 1], xrows);
        cudaEventRecord(a);
        const int reps = 5;
        for (int it = 0; it < reps; ++it) probe<<<grid, 96, smem>>>(map, stages_, kbox, per_cta, kb_total, n_tiles, mode, look, stall, 10000, (const char*)W, K, xmaps[xrows == 64 ? 2 : 1], xrows);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double bytes = static_cast<double>(per_cta) * grid * 16384 * kbox;
        printf("xrows=%d stages=%d mode=%d look=%2d stall=%d %2d  %.0f GB/s  %.1f us err=%s\n", xrows, st2, mode, look, stall, stages,
               bytes / (ms / reps * 1e-3) / 1e9, ms / reps * 1e3, cudaGetErrorString(cudaGetLastError()));
       }
      }
    }
  }
  return 0;
}
