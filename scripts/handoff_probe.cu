// Probe: kernel-to-kernel dependency latency on a chain of short 148-CTA kernels (profiling only).
//   mode 0: programmatic dependent launch, consumer waits with griddepcontrol.wait (grid completion)
//   big 1: every other kernel takes 190 KB of dynamic shared memory (the verify GEMM's footprint)
//   mode 1: consumer launched early by PDL, but waits on a per-launch arrival counter that every
//           producer CTA releases after its stores (acquire-poll), no griddepcontrol.wait
// Each kernel: every CTA reads 4 KB of the previous kernel's output, writes 4 KB.  Reports us per kernel.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/handoff_probe scripts/handoff_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void step(const float* in, float* out, unsigned* ctr, int idx, int mode) {
  extern __shared__ float dyn[];
  if (threadIdx.x == 1023) dyn[0] = 0.f;
  if (mode == 0) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
  } else {
    if (threadIdx.x == 0 && idx > 0) {
      const unsigned target = gridDim.x;
      while (ld_acquire(ctr + idx - 1) < target) {
      }
    }
    __syncthreads();
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  float v = 0.f;
  for (int r = 0; r < 4; ++r) v += __ldcg(in + (i * 4 + r) % (148 * 256 * 4));
  out[i] = v * 0.5f + 1.f;
  if (mode == 1) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(ctr + idx, 1u);
    }
  }
}

int main() {
  const int n = 148 * 256, K = 200;
  float *a, *b;
  unsigned* ctr;
  cudaMalloc(&a, n * 4 * 4);
  cudaMalloc(&b, n * 4 * 4);
  cudaMalloc(&ctr, K * 4);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaFuncSetAttribute(step, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int big : {0, 1})
  for (int mode : {0, 1, 0, 1}) {
    float best = 1e9;
    for (int it = 0; it < 5; ++it) {
      cudaMemsetAsync(ctr, 0, K * 4, s);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0, s);
      for (int k = 0; k < K; ++k) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(148);
        cfg.blockDim = dim3(256);
        cfg.stream = s;
        cfg.dynamicSmemBytes = (big && (k & 1)) ? 190 * 1024 : 0;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, step, (const float*)((k & 1) ? b : a), (k & 1) ? a : b, ctr, k, mode);
      }
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("big %d mode %d: %.3f us per kernel (%s)\n", big, mode, best * 1e3 / K, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
