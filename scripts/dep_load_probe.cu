// Probe: latency of a dependent load right after griddepcontrol.wait — TMA 2D box (16 KB, mbarrier)
// vs plain 16-byte loads by all threads (ld.global.cg) — of data the previous kernel just wrote.
// Kernel A (148 CTAs) writes the 16 KB buffer; kernel B (PDL, 148 CTAs) waits, then loads it and
// stamps %globaltimer at wait-return and at data-ready.  Prints the median ready - release over CTAs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/dep_load_probe scripts/dep_load_probe.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

#include "../paper_2512_23858_b200/csrc/common.cuh"

using namespace ygg;

__global__ void writer(uint4* buf, int n16, int iter) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += gridDim.x * blockDim.x)
    buf[i] = make_uint4(i + iter, i, iter, 1);
}

__global__ void reader(const __grid_constant__ CUtensorMap map, const uint4* buf, int mode,
                       unsigned long long* out, uint4* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
    tma_prefetch_desc(&map);
  }
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const unsigned long long t0 = gtimer();
  uint4 acc = make_uint4(0, 0, 0, 0);
  if (mode == 0) {  // TMA: 64 rows x 256 B box of a [64][256 B] tensor
    if (threadIdx.x == 0) {
      mbar_arrive_expect_tx(&bar, 16384);
      tma_load_2d(sm, &map, &bar, 0, 0, policy_evict_last());
    }
    mbar_wait(&bar, 0);
    acc = reinterpret_cast<const uint4*>(sm)[threadIdx.x];
  } else {  // every thread: 4 x 16 B loads (1024 threads x 16 B = 16 KB)
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint4 v = __ldcg(buf + threadIdx.x + k * 256);
      acc.x += v.x;
      acc.y ^= v.y;
    }
  }
  __syncthreads();
  const unsigned long long t1 = gtimer();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc.x == 0xdeadbeef) sink[0] = acc;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

int main() {
  uint4* buf;
  uint4* sink;
  unsigned long long* out;
  cudaMalloc(&buf, 16384);
  cudaMalloc(&sink, 64);
  cudaMalloc(&out, 148 * 8);
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
  CUtensorMap map;
  cuuint64_t dims[2] = {128, 64};  // bf16 elements: 256 B rows, 64 rows
  cuuint64_t str[1] = {256};
  cuuint32_t box[2] = {128, 64};
  cuuint32_t es[2] = {1, 1};
  enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(reader, cudaFuncAttributeMaxDynamicSharedMemorySize, 20480);
  cudaStream_t s;
  cudaStreamCreate(&s);
  for (int mode : {0, 1, 0, 1}) {
    std::vector<unsigned long long> all;
    for (int it = 0; it < 50; ++it) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cfg.stream = s;
      cfg.gridDim = dim3(148);
      cfg.blockDim = dim3(256);
      cudaLaunchKernelEx(&cfg, writer, buf, 1024, it);
      cfg.dynamicSmemBytes = 20480;
      cudaLaunchKernelEx(&cfg, reader, map, (const uint4*)buf, mode, out, sink);
      std::vector<unsigned long long> h(148);
      cudaMemcpyAsync(h.data(), out, 148 * 8, cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      if (it >= 5) all.insert(all.end(), h.begin(), h.end());
    }
    std::sort(all.begin(), all.end());
    printf("mode %s: median %.0f ns, p90 %.0f ns (%s)\n", mode == 0 ? "TMA " : "LDG ", double(all[all.size() / 2]),
           double(all[all.size() * 9 / 10]), cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
