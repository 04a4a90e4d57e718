// Host-side runtime shared by the translation units of libsfft2d_b200.so:
// error handling, the PDL launch helper, and the context services (workspace,
// per-launch profiling hooks, shared-memory opt-in) that capi.cu defines.
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <utility>

#include "../../include/sfft2d_b200.h"

namespace sfft {

struct SfftError {
  int code;
  std::string msg;
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw SfftError{code, msg}; }

inline void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(SFFT2D_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

constexpr int kHostNumSMs = 148;   // B200

// CTAs for `work` items at `per_block` per CTA, capped (grid-stride kernels)
inline unsigned grid_for(long long work, int per_block = 256, int cap = kHostNumSMs * 16) {
  long long b = (work + per_block - 1) / per_block;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return (unsigned)b;
}

inline bool is_pow2(long long v) { return v >= 1 && (v & (v - 1)) == 0; }
inline int ilog2(long long v) {
  int l = 0;
  while ((1LL << l) < v) ++l;
  return l;
}

// ---- context services (capi.cu)
// named stream-ordered workspace of at least `bytes` (grow-only)
void* ws(sfft2d_ctx* c, const char* name, size_t bytes);
// bracket every launch: count it, check it, and when profiling record an
// event pair with the launch's algorithmic bytes
void pre(sfft2d_ctx* c, cudaStream_t st);
void post(sfft2d_ctx* c, const char* what, cudaStream_t st, double bytes);
// raise the kernel's dynamic shared-memory limit (once per device and kernel)
void allow_smem_ptr(const void* kernel);
template <typename K>
inline void allow_smem(K kernel) {
  allow_smem_ptr((const void*)kernel);
}

// resident CTAs per SM of `kernel` at (threads, dynamic smem), queried once
// per device/kernel/shape from the occupancy calculator (so grid sizing
// follows the compiled register count instead of a hard-coded assumption)
int ctas_per_sm_ptr(const void* kernel, int threads, size_t smem);
template <typename K>
inline int ctas_per_sm(K kernel, int threads, size_t smem) {
  if (smem > 0) allow_smem(kernel);
  return ctas_per_sm_ptr((const void*)kernel, threads, smem);
}

// Launch with programmatic stream serialisation (PDL): the kernel may be
// scheduled while its predecessor in the stream drains; it waits in pdl_wait()
// before touching memory.  Launch errors throw.  Kernels launched with dynamic
// shared memory get their limit raised first (the 48 KB default bounds static
// + dynamic together; the opt-in is cached per device and kernel).
template <typename... KArgs, typename... Args>
void kl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
        Args&&... args) {
  if (smem > 0) allow_smem(kernel);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  ck(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...), "cudaLaunchKernelEx");
}

// kl() for a kernel launched in thread-block clusters of `cluster_x` CTAs
// (grid.x a multiple of cluster_x), also with PDL.
template <typename... KArgs, typename... Args>
void klc(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
         int cluster_x, Args&&... args) {
  if (smem > 0) allow_smem(kernel);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = (unsigned)cluster_x;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  ck(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...), "cudaLaunchKernelEx(cluster)");
}

}  // namespace sfft
