// Host-side helpers shared by every translation unit of libygg.so: thread-local error text,
// argument checks that map to the reference's ValueError convention, and a launch macro
// that always enables programmatic dependent launch (PDL) so consecutive kernels of a step
// overlap their prologues with the previous kernel's tail.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>

#include "../../include/ygg.h"

namespace ygg {

int ygg_fail(int code, const char* fmt, ...);

// Next slot of the armed kernel-timeline buffer (ygg_trace_arm), tagged with kernel_id, or nullptr.
unsigned long long* trace_next(int kernel_id);

// Every launch uses programmatic dependent launch (griddepcontrol in the kernels).
inline int pdl_enabled() { return 1; }

template <typename Kernel, typename... Args>
int launch_pdl(Kernel kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t stream, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled();
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t err = cudaLaunchKernelEx(&cfg, kernel, args...);
  if (err != cudaSuccess) return ygg_fail(YGG_ERR_CUDA, "launch failed: %s", cudaGetErrorString(err));
  return YGG_OK;
}

template <typename Kernel, typename... Args>
int launch_pdl_cluster(Kernel kernel, dim3 grid, dim3 block, int cluster_x, cudaStream_t stream, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled();
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = cluster_x;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cudaError_t err = cudaLaunchKernelEx(&cfg, kernel, args...);
  if (err != cudaSuccess) return ygg_fail(YGG_ERR_CUDA, "cluster launch failed: %s", cudaGetErrorString(err));
  return YGG_OK;
}

// PDL launch with a (cluster_x, 1, 1) thread-block cluster and dynamic shared memory.
template <typename Kernel, typename... Args>
int launch_pdl_cluster_x(Kernel kernel, dim3 grid, dim3 block, size_t smem, int cluster_x, cudaStream_t stream,
                         Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled();
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = cluster_x;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cudaError_t err = cudaLaunchKernelEx(&cfg, kernel, args...);
  if (err != cudaSuccess) return ygg_fail(YGG_ERR_CUDA, "cluster launch failed: %s", cudaGetErrorString(err));
  return YGG_OK;
}

// PDL launch with a (1, 1, cluster_z) thread-block cluster and dynamic shared memory.
template <typename Kernel, typename... Args>
int launch_pdl_cluster_z(Kernel kernel, dim3 grid, dim3 block, size_t smem, int cluster_z, cudaStream_t stream,
                         Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled();
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = 1;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = cluster_z;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cudaError_t err = cudaLaunchKernelEx(&cfg, kernel, args...);
  if (err != cudaSuccess) return ygg_fail(YGG_ERR_CUDA, "cluster launch failed: %s", cudaGetErrorString(err));
  return YGG_OK;
}

}  // namespace ygg

#define YGG_LAUNCH_PDL_CLUSTER(kernel, grid, block, cx, stream, ...)                              \
  do {                                                                                            \
    int _rc = ::ygg::launch_pdl_cluster(kernel, grid, block, cx, stream, __VA_ARGS__);            \
    if (_rc) return _rc;                                                                          \
  } while (0)

#define YGG_CHECK_ARG(cond, msg)                                   \
  do {                                                             \
    if (!(cond)) return ::ygg::ygg_fail(YGG_ERR_VALUE, "%s", msg); \
  } while (0)

#define YGG_LAUNCH_PDL(kernel, grid, block, smem, stream, ...)                                    \
  do {                                                                                            \
    int _rc = ::ygg::launch_pdl(kernel, grid, block, smem, stream, __VA_ARGS__);                  \
    if (_rc) return _rc;                                                                          \
  } while (0)
