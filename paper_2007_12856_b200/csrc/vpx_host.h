// Host-side helpers shared by every C-ABI entry point: status codes, the
// thread-local last-error message and TMA tensor-map encoding.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <utility>

#include "../../include/vpx.h"

namespace vpx {

void set_error(const char* fmt, ...);
int precision();
// Number of kernels this library has launched (vpx_launch_count()).
extern std::atomic<long long> g_launches;
// Conv passes that ran on the generic CUDA-core kernels (conv_simt.cu) while the
// library is in TF32 tensor-core mode: no tcgen05 kernel covers that shape.
extern std::atomic<long long> g_fallbacks;
inline void note_fallback() {
  if (precision() == 0) g_fallbacks.fetch_add(1, std::memory_order_relaxed);
}

#define VPX_FAIL(code, ...)        \
  do {                             \
    ::vpx::set_error(__VA_ARGS__); \
    return (code);                 \
  } while (0)

#define VPX_CHECK_CUDA(expr)                                                                \
  do {                                                                                      \
    cudaError_t _e = (expr);                                                                \
    if (_e != cudaSuccess) VPX_FAIL(VPX_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(_e)); \
  } while (0)

#define VPX_LAUNCH_CHECK()                                                           \
  do {                                                                               \
    ::vpx::g_launches.fetch_add(1, std::memory_order_relaxed);                       \
    cudaError_t _e = cudaGetLastError();                                             \
    if (_e != cudaSuccess) VPX_FAIL(VPX_ERR_CUDA, "launch: %s", cudaGetErrorString(_e)); \
  } while (0)

// Programmatic dependent launch for the deep-layer conv chain: the kernel may
// be scheduled while its predecessor in the stream drains, runs its prologue
// (barrier init, TMEM alloc, tensor-map prefetch) and then blocks in
// vpx::pdl_wait() until the predecessor has completed and its writes are
// visible.  Only kernels that call pdl_wait() before touching global memory
// are launched this way.  VPX_NO_PDL=1 launches them with plain serialization.
inline bool pdl_enabled() {
  static const bool on = std::getenv("VPX_NO_PDL") == nullptr;
  return on;
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Encode a tiled TMA map. dims/box are innermost-first; strides_bytes has
// rank-1 entries (stride of dims 1..rank-1).  Returns 0 or VPX_ERR_CUDA.
int encode_tiled(CUtensorMap* map, CUtensorMapDataType dtype, int rank, void* gaddr,
                 const uint64_t* dims, const uint64_t* strides_bytes, const uint32_t* box,
                 CUtensorMapSwizzle swizzle);
// Same with per-dimension element (traversal) strides.
int encode_tiled_strided(CUtensorMap* map, CUtensorMapDataType dtype, int rank, void* gaddr,
                         const uint64_t* dims, const uint64_t* strides_bytes, const uint32_t* box,
                         const uint32_t* elem_strides, CUtensorMapSwizzle swizzle);

}  // namespace vpx
