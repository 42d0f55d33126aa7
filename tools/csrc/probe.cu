// Test-only probes that pin UMMA descriptor and TMA box semantics on the
// device (used by tests/test_probe_gpu.py).  vpx_probe_umma copies a host-built
// shared-memory image into smem, issues a list of tcgen05.mma operations and
// dumps the TMEM accumulator; vpx_probe_tma loads one 5D box and dumps smem.
#include "vpx_host.h"
#include "vpx_ptx.cuh"

namespace {

constexpr int kProbeSmem = 200 * 1024;

// op layout (4 x u64): adesc (start = offset into image), bdesc (same),
// idesc | (d_col << 32), accumulate flag | 2 if A comes from TMEM (then the
// adesc word is the TMEM column of A).  ta[128][ta_cols] (optional) is stored
// to TMEM columns [256, 256 + ta_cols) before the ops run.
__global__ void __launch_bounds__(128, 1)
    probe_umma_kernel(const uint4* __restrict__ img, int img_bytes,
                      const uint64_t* __restrict__ ops, int n_ops, float* __restrict__ out,
                      int ncols, const float* __restrict__ ta, int ta_cols) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  uint4* s4 = reinterpret_cast<uint4*>(smem);
  for (int i = tid; i < img_bytes / 16; i += blockDim.x) s4[i] = img[i];
  vpx::fence_proxy_async_smem();
  if (warp == 0) vpx::tmem_alloc<512>(&tmem_base);
  if (tid == 0) {
    vpx::mbar_init(&bar, 1);
    vpx::fence_barrier_init();
  }
  vpx::tc_fence_before();
  __syncthreads();
  vpx::tc_fence_after();
  const uint32_t tbase = tmem_base;
  if (ta != nullptr) {
    const int row = 32 * (warp & 3) + (tid & 31);
    for (int c = 0; c < ta_cols; c += 16) {
      float v[16];
      for (int j = 0; j < 16; ++j) v[j] = ta[row * ta_cols + c + j];
      vpx::tmem_st16(tbase + (static_cast<uint32_t>(32 * (warp & 3)) << 16) + 256 + c, v);
    }
    vpx::tmem_st_wait();
  }
  vpx::tc_fence_before();
  __syncthreads();
  vpx::tc_fence_after();
  const uint64_t sbase = static_cast<uint64_t>(vpx::smem_u32(smem) >> 4);
  if (tid == 0) {
    for (int i = 0; i < n_ops; ++i) {
      uint64_t b = ops[4 * i + 1] + sbase;
      uint64_t w = ops[4 * i + 2];
      uint32_t idesc = static_cast<uint32_t>(w & 0xffffffffu);
      uint32_t dcol = static_cast<uint32_t>(w >> 32);
      uint32_t acc = static_cast<uint32_t>(ops[4 * i + 3]) & 1u;
      if (ops[4 * i + 3] & 2u)
        vpx::umma_tf32_ta(tbase + dcol, tbase + static_cast<uint32_t>(ops[4 * i + 0]), b, idesc, acc);
      else
        vpx::umma_tf32(tbase + dcol, ops[4 * i + 0] + sbase, b, idesc, acc);
    }
    vpx::umma_commit(&bar);
  }
  __syncwarp();
  vpx::mbar_wait(&bar, 0);
  vpx::tc_fence_after();
  const int lane_base = 32 * (warp & 3);
  for (int c = 0; c < ncols; c += 16) {
    float v[16];
    vpx::tmem_ld16(tbase + (static_cast<uint32_t>(lane_base) << 16) + c, v);
    const int row = lane_base + (tid & 31);
    for (int j = 0; j < 16 && c + j < ncols; ++j) out[row * ncols + c + j] = v[j];
  }
  vpx::tc_fence_before();
  __syncthreads();
  if (warp == 0) vpx::tmem_dealloc<512>(tbase);
}

__global__ void __launch_bounds__(128, 1)
    probe_tma_kernel(const __grid_constant__ CUtensorMap map, int c0, int c1, int c2, int c3,
                     int c4, uint32_t bytes, uint4* __restrict__ out, int* __restrict__ ok) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  const int tid = threadIdx.x;
  if (tid == 0) {
    vpx::mbar_init(&bar, 1);
    vpx::fence_barrier_init();
  }
  __syncthreads();
  if (tid == 0) {
    vpx::mbar_arrive_expect_tx(&bar, bytes);
    vpx::tma_load_5d(smem, &map, &bar, c0, c1, c2, c3, c4);
  }
  // bounded wait: a wrong byte count must not hang the probe
  bool done = false;
  for (long long it = 0; it < (1LL << 22) && !done; ++it) done = vpx::mbar_try_wait(&bar, 0);
  if (tid == 0) ok[0] = done ? 1 : 0;
  if (!done) return;
  const uint4* s4 = reinterpret_cast<const uint4*>(smem);
  for (uint32_t i = tid; i < bytes / 16; i += blockDim.x) out[i] = s4[i];
}

// Back-to-back MMA issue rate: n_iter x (M=128, N, K=8) tf32 MMAs on fixed
// operands; reports the cycles from first issue to commit completion.
__global__ void __launch_bounds__(128, 1)
    probe_rate_kernel(int N, int n_iter, int a_layout, int n_acc, int bf16,
                      long long* __restrict__ cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 100 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 1.0f;
  vpx::fence_proxy_async_smem();
  if (warp == 0) vpx::tmem_alloc<512>(&tmem_base);
  if (tid == 0) {
    vpx::mbar_init(&bar, 1);
    vpx::fence_barrier_init();
  }
  vpx::tc_fence_before();
  __syncthreads();
  vpx::tc_fence_after();
  const uint32_t tbase = tmem_base;
  const uint32_t s0 = vpx::smem_u32(smem);
  if (tid == 0) {
    // a_layout 0: no-swizzle K-major, aligned core matrices (LBO 2048); 1: SW128;
    // 3: no-swizzle with LBO 16 (the conv_c1fwd.cu shifted-window A, core
    // matrices overlapping at 16-byte offsets); 4: SW32 K-major (SBO 256)
    uint64_t a = a_layout == 0 ? vpx::make_sdesc(s0, 2048, 128, 0)
               : a_layout == 3 ? vpx::make_sdesc(s0 + 16, 16, 128, 0)
               : a_layout == 4 ? vpx::make_sdesc(s0, 16, 256, 6)
                               : vpx::make_sdesc(s0, 16, 1024, 2);
    uint64_t b = (a_layout == 0 || a_layout == 3) ? vpx::make_sdesc(s0 + 32768, 4096, 128, 0)
                                                   : vpx::make_sdesc(s0 + 32768, 16, 1024, 2);
    uint32_t idesc = vpx::make_idesc(bf16 ? 1 : 2, 128, N, false, false);
    long long t0 = clock64();
    if (a_layout == 2) {
      for (int i = 0; i < n_iter; ++i)
        vpx::umma_tf32_ta(tbase + (i % n_acc) * N, tbase + 256 + 8 * (i & 7), b, idesc, i >= n_acc);
    } else if (bf16) {
      for (int i = 0; i < n_iter; ++i)
        vpx::umma_f16(tbase + (i % n_acc) * N, a, b, idesc, i >= n_acc);
    } else {
      for (int i = 0; i < n_iter; ++i)
        vpx::umma_tf32(tbase + (i % n_acc) * N, a, b, idesc, i >= n_acc);
    }
    vpx::umma_commit(&bar);
    vpx::mbar_wait(&bar, 0);
    long long t1 = clock64();
    cycles[0] = t1 - t0;
  }
  __syncwarp();
  vpx::tc_fence_before();
  __syncthreads();
  if (warp == 0) vpx::tmem_dealloc<512>(tbase);
}

// Same, with the issue loop in the canonical warp-uniform form (whole warp 1
// iterates; one elected lane issues an unrolled burst of NACC MMAs).
// MODE 0 tf32, 1 bf16, 2 tf32 with A in TMEM (cols 256..), 3 = 2 with B MN-major
// SWIZZLE_128B_BASE32B (LBO 128 B, SBO 512 B: the voxel-row operand of conv_c1bwd.cu)
template <int N, int NACC, int MODE>
__global__ void __launch_bounds__(128, 1) probe_rate2_kernel(int n_iter, long long* cycles) {
  constexpr bool BF16 = MODE == 1;
  static_assert(MODE != 10 || N % 16 == 0, "");
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  // MODE 9 = MODE 8 with pseudo-random operands in smem and TMEM
  for (int i = tid; i < 100 * 1024 / 4; i += blockDim.x)
    reinterpret_cast<float*>(smem)[i] = MODE == 9 ? __uint_as_float((i * 2654435761u) & 0xbfffe000u | 0x3e000000u) : 1.0f;
  vpx::fence_proxy_async_smem();
  if (warp == 0) vpx::tmem_alloc<512>(&tmem_base);
  if (tid == 0) {
    vpx::mbar_init(&bar, 1);
    vpx::mbar_init(&bar2, 1);
    vpx::fence_barrier_init();
  }
  vpx::tc_fence_before();
  __syncthreads();
  vpx::tc_fence_after();
  if (MODE == 9) {
    float v[16];
    for (int c = 0; c < 512; c += 16) {
      for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(((tid * 977 + c * 131 + j * 7919) * 2654435761u) & 0xbfffe000u | 0x3e000000u);
      vpx::tmem_st16(tmem_base + (static_cast<uint32_t>(32 * warp) << 16) + c, v);
    }
    vpx::tmem_st_wait();
    vpx::tc_fence_before();
    __syncthreads();
    vpx::tc_fence_after();
  }
  const uint32_t tbase = tmem_base;
  if (warp == 1) {
    const uint32_t s0 = vpx::smem_u32(smem);
    const uint64_t a = vpx::make_sdesc(s0, 2048, 128, 0);
    const uint64_t b = vpx::make_sdesc(s0 + 32768, 4096, 128, 0);
    constexpr uint32_t idesc = vpx::make_idesc(BF16 ? 1 : 2, 128, N, false, false);
    constexpr uint32_t idesc_mn = vpx::make_idesc(2, 128, N, false, true);
    const uint64_t bmn = vpx::make_sdesc(s0 + 32768, 128, 512, 1);
    const uint64_t bmn9 = vpx::make_sdesc(s0, 128, 512, 1);
    long long t0 = clock64();
    for (int i = 0; i < n_iter; i += NACC) {
      if (MODE == 6) vpx::tc_fence_after();
      if (vpx::elect_one()) {
#pragma unroll
        for (int j = 0; j < NACC; ++j) {
          if (MODE == 2)
            vpx::umma_tf32_ta(tbase + (j * N) % 256, tbase + 256 + 8 * (j & 7), b, idesc, i > 0);
          else if (MODE == 7)
            vpx::umma_tf32_ta(tbase + j * N, tbase + 432 + 8 * (j & 7), bmn + 64 * (j & 3), idesc_mn, i > 0);
          else if (MODE == 8 || MODE == 9)  // 9 B rows 10 KB apart, as in conv_c1bwd.cu
            vpx::umma_tf32_ta(tbase + j * N, tbase + 432 + 8 * (i & 7), bmn9 + 640 * j, idesc_mn, i > 0);
          else if (MODE >= 3 && MODE != 10)
            vpx::umma_tf32_ta(tbase + (j * N) % 256, tbase + 256 + 8 * (j & 7), bmn + 64 * (j & 3), idesc_mn,
                              i > 0);
          else if (MODE == 10)  // no-swizzle, LBO 16: the c1 forward's shifted 16-byte-pitch window
            vpx::umma_tf32(tbase + j * N, vpx::make_sdesc(s0 + 16 * (j & 1), 16, 128, 0), b, idesc, i > 0);
          else if (BF16)
            vpx::umma_f16(tbase + j * N, a + 2 * (j & 1), b, idesc, i > 0);
          else
            vpx::umma_tf32(tbase + j * N, a + 2 * (j & 1), b, idesc, i > 0);
        }
        if (MODE == 5) vpx::umma_commit(&bar2);
      }
      __syncwarp();
    }
    if (vpx::elect_one()) vpx::umma_commit(&bar);
    __syncwarp();
    vpx::mbar_wait(&bar, 0);
    long long t1 = clock64();
    if ((tid & 31) == 0) cycles[0] = t1 - t0;
  }
  vpx::tc_fence_before();
  __syncthreads();
  if (warp == 0) vpx::tmem_dealloc<512>(tbase);
}

template <int N, int NACC, int MODE>
static int launch_rate2(int n_iter, long long* cycles, cudaStream_t st) {
  VPX_CHECK_CUDA(cudaFuncSetAttribute(probe_rate2_kernel<N, NACC, MODE>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024 + 1024));
  probe_rate2_kernel<N, NACC, MODE><<<1, 128, 100 * 1024 + 1024, st>>>(n_iter, cycles);
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}

}  // namespace

extern "C" int vpx_probe_mma_rate2(int N, int n_acc, int bf16, int n_iter, long long* cycles,
                                   void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
#define RATE_CASE(n, a)                                                         \
  if (N == n && n_acc == a)                                                     \
    return bf16 == 10 ? launch_rate2<n, a, 10>(n_iter, cycles, st)              \
           : bf16 == 9 ? launch_rate2<n, a, 9>(n_iter, cycles, st)              \
           : bf16 == 8 ? launch_rate2<n, a, 8>(n_iter, cycles, st)              \
           : bf16 == 7 ? launch_rate2<n, a, 7>(n_iter, cycles, st)              \
           : bf16 == 6 ? launch_rate2<n, a, 6>(n_iter, cycles, st)              \
           : bf16 == 5 ? launch_rate2<n, a, 5>(n_iter, cycles, st)              \
           : bf16 == 3 ? launch_rate2<n, a, 3>(n_iter, cycles, st)              \
           : bf16 == 2 ? launch_rate2<n, a, 2>(n_iter, cycles, st)              \
           : bf16    ? launch_rate2<n, a, 1>(n_iter, cycles, st)                \
                     : launch_rate2<n, a, 0>(n_iter, cycles, st);
  RATE_CASE(16, 1) RATE_CASE(16, 4) RATE_CASE(16, 8) RATE_CASE(32, 1) RATE_CASE(32, 4)
  RATE_CASE(32, 8) RATE_CASE(48, 1) RATE_CASE(48, 2) RATE_CASE(48, 4) RATE_CASE(48, 8) RATE_CASE(48, 9) RATE_CASE(96, 1) RATE_CASE(96, 2) RATE_CASE(64, 1) RATE_CASE(64, 4) RATE_CASE(64, 8) RATE_CASE(128, 1)
  RATE_CASE(128, 2) RATE_CASE(256, 1) RATE_CASE(256, 2)
#undef RATE_CASE
  VPX_FAIL(VPX_ERR_UNSUPPORTED, "rate2 case");
}

extern "C" int vpx_probe_mma_rate(int N, int n_iter, int a_layout, int n_acc, int bf16,
                                  long long* cycles, void* stream) {
  VPX_CHECK_CUDA(cudaFuncSetAttribute(probe_rate_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024 + 1024));
  probe_rate_kernel<<<1, 128, 100 * 1024 + 1024, static_cast<cudaStream_t>(stream)>>>(N, n_iter, a_layout,
                                                                               n_acc, bf16, cycles);
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}

extern "C" int vpx_probe_umma(const void* img, int img_bytes, const uint64_t* ops, int n_ops,
                              float* out, int ncols, void* stream) {
  if (img_bytes > kProbeSmem || img_bytes % 16) VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "image size");
  if (ncols % 16 || ncols > 512) VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "ncols");
  VPX_CHECK_CUDA(cudaFuncSetAttribute(probe_umma_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, kProbeSmem));
  probe_umma_kernel<<<1, 128, kProbeSmem, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint4*>(img), img_bytes, ops, n_ops, out, ncols, nullptr, 0);
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}

extern "C" int vpx_probe_umma_ta(const void* img, int img_bytes, const uint64_t* ops, int n_ops,
                                 const float* ta, int ta_cols, float* out, int ncols, void* stream) {
  if (img_bytes > kProbeSmem || img_bytes % 16) VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "image size");
  if (ncols % 16 || ncols > 256 || ta_cols % 16 || ta_cols > 256) VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "cols");
  VPX_CHECK_CUDA(cudaFuncSetAttribute(probe_umma_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, kProbeSmem));
  probe_umma_kernel<<<1, 128, kProbeSmem, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint4*>(img), img_bytes, ops, n_ops, out, ncols, ta, ta_cols);
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}

extern "C" int vpx_probe_tma(const void* gsrc, const uint64_t* dims5, const uint64_t* strides4,
                             const uint32_t* box5, const uint32_t* estr5, int swizzle,
                             const int32_t* coords5, void* out, int out_bytes, int* ok,
                             void* stream) {
  CUtensorMap map;
  CUtensorMapSwizzle sw = swizzle == 1282 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B
                          : swizzle == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                          : swizzle == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                          : swizzle == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                          : CU_TENSOR_MAP_SWIZZLE_NONE;
  int rc = vpx::encode_tiled_strided(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5,
                                     const_cast<void*>(gsrc), dims5, strides4, box5, estr5, sw);
  if (rc) return rc;
  if (out_bytes > kProbeSmem || out_bytes % 16) VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "out size");
  VPX_CHECK_CUDA(cudaFuncSetAttribute(probe_tma_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, kProbeSmem));
  probe_tma_kernel<<<1, 128, kProbeSmem, static_cast<cudaStream_t>(stream)>>>(
      map, coords5[0], coords5[1], coords5[2], coords5[3], coords5[4],
      static_cast<uint32_t>(out_bytes), static_cast<uint4*>(out), ok);
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}
