// Probe: dependency gap (last CTA end of a small "epilogue" kernel -> griddepcontrol.wait release of the
// next "GEMM" kernel) as a function of the epilogue's CTA count and the GEMM's shared-memory footprint.
// Chain G E G E ... under programmatic dependent launch; every kernel stamps %globaltimer (atomicMax of
// CTA ends, atomicMin of releases).  Profiling only.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/gap_probe scripts/gap_probe.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// stamps[k][0] = min release, [1] = max end
__global__ void gemm_like(unsigned long long* st, float* buf, int spin_ns) {
  extern __shared__ float sm[];
  if (threadIdx.x == 0) sm[0] = 0.f;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) atomicMin(st + 0, gt());
  const unsigned long long t0 = gt();
  while (gt() - t0 < static_cast<unsigned long long>(spin_ns)) {
  }
  buf[blockIdx.x * blockDim.x + threadIdx.x] += 1.f;
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(st + 1, gt());
}

__global__ void epi_like(unsigned long long* st, float* buf, int n) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x == 0) atomicMin(st + 0, gt());
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) buf[i] = buf[i] * 0.5f + 1.f;
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(st + 1, gt());
}

int main() {
  float* buf;
  unsigned long long* st;
  const int K = 40;
  cudaMalloc(&buf, 64 << 20);
  cudaMemset(buf, 0, 64 << 20);
  cudaMalloc(&st, K * 2 * 8);
  cudaFuncSetAttribute(gemm_like, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaStream_t s;
  cudaStreamCreate(&s);
  for (int smem_kb : {190, 0}) {
    for (int ectas : {50, 148, 300, 700}) {
      std::vector<double> gaps_g, gaps_e;
      for (int it = 0; it < 5; ++it) {
        std::vector<unsigned long long> init(K * 2);
        for (int k = 0; k < K; ++k) { init[2 * k] = ~0ull; init[2 * k + 1] = 0; }
        cudaMemcpy(st, init.data(), K * 16, cudaMemcpyHostToDevice);
        for (int k = 0; k < K; ++k) {
          cudaLaunchConfig_t cfg = {};
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          at[0].val.programmaticStreamSerializationAllowed = 1;
          cfg.attrs = at;
          cfg.numAttrs = 1;
          cfg.stream = s;
          if (k % 2 == 0) {
            cfg.gridDim = dim3(148);
            cfg.blockDim = dim3(192);
            cfg.dynamicSmemBytes = smem_kb * 1024;
            cudaLaunchKernelEx(&cfg, gemm_like, st + 2 * k, buf, 5000);
          } else {
            cfg.gridDim = dim3(ectas);
            cfg.blockDim = dim3(128);
            cfg.dynamicSmemBytes = 0;
            cudaLaunchKernelEx(&cfg, epi_like, st + 2 * k, buf, ectas * 128);
          }
        }
        cudaStreamSynchronize(s);
        std::vector<unsigned long long> h(K * 2);
        cudaMemcpy(h.data(), st, K * 16, cudaMemcpyDeviceToHost);
        for (int k = 2; k < K; ++k) {
          const double gap = (double(h[2 * k]) - double(h[2 * (k - 1) + 1])) / 1e3;
          (k % 2 == 0 ? gaps_g : gaps_e).push_back(gap);
        }
      }
      std::sort(gaps_g.begin(), gaps_g.end());
      std::sort(gaps_e.begin(), gaps_e.end());
      printf("gemm smem %3d KB, epi CTAs %3d: epi->gemm gap median %.2f us, gemm->epi gap median %.2f us (%s)\n",
             smem_kb, ectas, gaps_g[gaps_g.size() / 2], gaps_e[gaps_e.size() / 2], cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
