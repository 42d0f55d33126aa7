// Host plumbing: error state, version tag, TMA tensor-map encoding.
#include "vpx_host.h"

namespace vpx {

static thread_local char g_err[1024] = {0};
std::atomic<long long> g_launches{0};
std::atomic<long long> g_fallbacks{0};
static int g_precision = 0;
int precision() { return g_precision; }

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

int encode_tiled(CUtensorMap* map, CUtensorMapDataType dtype, int rank, void* gaddr,
                 const uint64_t* dims, const uint64_t* strides_bytes, const uint32_t* box,
                 CUtensorMapSwizzle swizzle) {
  const uint32_t ones[5] = {1, 1, 1, 1, 1};
  return encode_tiled_strided(map, dtype, rank, gaddr, dims, strides_bytes, box, ones, swizzle);
}

int encode_tiled_strided(CUtensorMap* map, CUtensorMapDataType dtype, int rank, void* gaddr,
                         const uint64_t* dims, const uint64_t* strides_bytes, const uint32_t* box,
                         const uint32_t* elem_strides, CUtensorMapSwizzle swizzle) {
  auto fn = encode_fn();
  if (!fn) VPX_FAIL(VPX_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  for (int i = 0; i < rank; ++i) estr[i] = elem_strides[i];
  CUresult r = fn(map, dtype, rank, gaddr, reinterpret_cast<const cuuint64_t*>(dims),
                  reinterpret_cast<const cuuint64_t*>(strides_bytes),
                  reinterpret_cast<const cuuint32_t*>(box), estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    VPX_FAIL(VPX_ERR_CUDA,
             "cuTensorMapEncodeTiled failed (%d): rank %d dims %llu,%llu,%llu,%llu,%llu box "
             "%u,%u,%u,%u,%u",
             int(r), rank, (unsigned long long)dims[0], (unsigned long long)(rank > 1 ? dims[1] : 0),
             (unsigned long long)(rank > 2 ? dims[2] : 0),
             (unsigned long long)(rank > 3 ? dims[3] : 0),
             (unsigned long long)(rank > 4 ? dims[4] : 0), box[0], rank > 1 ? box[1] : 0,
             rank > 2 ? box[2] : 0, rank > 3 ? box[3] : 0, rank > 4 ? box[4] : 0);
  }
  return VPX_OK;
}

}  // namespace vpx

#ifndef VPX_GIT_REV
#define VPX_GIT_REV "unknown"
#endif

extern "C" const char* vpx_last_error(void) { return vpx::g_err; }
extern "C" const char* vpx_version(void) { return "libvpx sm_100a " VPX_GIT_REV; }
extern "C" long long vpx_launch_count(void) { return vpx::g_launches.load(); }
extern "C" long long vpx_fallback_count(void) { return vpx::g_fallbacks.load(); }
extern "C" int vpx_set_precision(int mode) {
  if (mode != 0 && mode != 1) VPX_FAIL(VPX_ERR_UNSUPPORTED, "precision mode %d", mode);
  vpx::g_precision = mode;
  return VPX_OK;
}
extern "C" int vpx_get_precision(void) { return vpx::g_precision; }
