// mma.sync m16n8k16 bf16 throughput / latency probe on sm_100a (profiling only).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/mma_probe scripts/mma_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void probe(int iters, float* out, long long* cycles) {
  float d[CHAINS][4] = {};
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
          "{%0, %1, %2, %3};"
          : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cycles = t1 - t0;
}

template <int CHAINS>
void run(int warps, int iters) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 8);
  probe<CHAINS><<<148, 32 * warps>>>(iters, out, cyc);
  cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double mmas = static_cast<double>(iters) * CHAINS;
  printf("chains %d warps/SM %2d: %.1f cycles per mma per warp, %.0f FMA/clk/SM\n", CHAINS, warps, c / mmas,
         mmas * warps * 2048.0 / c);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<1>(1, 4096);
  run<8>(1, 1024);
  run<8>(4, 1024);
  run<8>(8, 1024);
  run<8>(16, 1024);
  run<4>(8, 2048);
  return 0;
}
