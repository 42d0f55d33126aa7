// Filter gradient of the k2s2 transposed convolution on tcgen05:
//   wg[ci][co][P] = sum_q x[q][ci] * u[2q + P][co]     (P = (a, b, c) in {0,1}^3)
// reference pkg/src/voxpar/layers/reference.py:134-144.
//
// The reduction runs over coarse voxels q, so both operands are voxel-major
// tiles exactly as the NDHWC frames hold them: MN-major UMMA operands in the
// SWIZZLE_128B_BASE32B form (128-byte rows = 32 fp32 channels, one row per
// voxel, 4-row atoms), K = 8 coarse voxels per MMA.
//   A (M = 128) = four 32-lane blocks, block i = the fine gradient sampled at
//     parity P = P0 + i (u[2q + P], a TMA box with element stride 2 along W),
//     channels past Cout are TMA zero fill; blocks sit one tile apart (LBO).
//   B (N = 32) = the coarse input x[q], channels past Cin zero fill.
// Two MMAs per K step (P0 = 0 and 4) into two 32-column TMEM accumulators.
// Split-K over row ranges: CTA p owns rows [p*R/P, (p+1)*R/P) of the coarse
// grid (n, d, h, W segment), writes partial[p][ci][co][8] once, and a
// fixed-order sum over p (reduce_partials) makes the result deterministic.
#include "conv_common.h"
#include "conv_simt.h"
#include "vpx_host.h"
#include "vpx_ptx.cuh"

namespace {

constexpr int kRow = 128;   // bytes per smem row: 32 fp32 channels
constexpr int kSeg = 32;    // coarse voxels per W segment (multiple of 8)
constexpr int kTile = kSeg * kRow;
constexpr int kStage = 9 * kTile;  // 8 parity tiles of u + 1 tile of x (36 KB)
constexpr int kStages = 4;

struct DwParams {
  int n, d, h, w;       // coarse extents (x interior)
  int cin, cout;
  int nseg;             // W segments per row
  long long rows;       // n * d * h * nseg
  int P;                // row ranges (CTAs)
  int x_off_d, x_off_h, x_off_w;  // x frame margins
  int u_off_d, u_off_h, u_off_w;  // u frame margins
  float* part;          // [P][cin][cout][8]
};

__global__ void __launch_bounds__(256, 1)
    deconv_wgrad_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap umap,
                        const DwParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages], tfull;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long r0 = p.rows * blockIdx.x / p.P, r1 = p.rows * (blockIdx.x + 1) / p.P;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      vpx::mbar_init(&full[s], 1);
      vpx::mbar_init(&empty[s], 1);
    }
    vpx::mbar_init(&tfull, 1);
    vpx::fence_barrier_init();
    vpx::tma_prefetch_desc(&xmap);
    vpx::tma_prefetch_desc(&umap);
  }
  if (warp == 2) vpx::tmem_alloc<64>(&tmem_base);
  vpx::tc_fence_before();
  __syncthreads();
  vpx::tc_fence_after();
  const uint32_t tbase = tmem_base;

  if (warp == 0) {
    if (vpx::elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (long long r = r0; r < r1; ++r) {
        long long t = r;
        const int sg = static_cast<int>(t % p.nseg);
        t /= p.nseg;
        const int y = static_cast<int>(t % p.h);
        t /= p.h;
        const int z = static_cast<int>(t % p.d);
        const int n = static_cast<int>(t / p.d);
        const int x0 = sg * kSeg;
        vpx::mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* st = smem + stage * kStage;
        vpx::mbar_arrive_expect_tx(&full[stage], kStage);
#pragma unroll
        for (int P = 0; P < 8; ++P) {
          const int a = (P >> 2) & 1, b = (P >> 1) & 1, c = P & 1;
          vpx::tma_load_5d(st + P * kTile, &umap, &full[stage], 0, 2 * x0 + c + p.u_off_w, 2 * y + b + p.u_off_h,
                           2 * z + a + p.u_off_d, n);
        }
        vpx::tma_load_5d(st + 8 * kTile, &xmap, &full[stage], 0, x0 + p.x_off_w, y + p.x_off_h, z + p.x_off_d, n);
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = vpx::make_idesc(2, 128, 32, true, true);
    int stage = 0;
    uint32_t phase = 0;
    for (long long r = r0; r < r1; ++r) {
      vpx::mbar_wait(&full[stage], phase);
      vpx::tc_fence_after();
      if (vpx::elect_one()) {
        const uint32_t sb = vpx::smem_u32(smem + stage * kStage);
        // base descriptors + address-field offsets (8 voxel rows = 1024 B per K step)
        const uint64_t b0 = vpx::make_sdesc(sb + 8 * kTile, kTile, 512, 1);
        const uint64_t a0 = vpx::make_sdesc(sb, kTile, 512, 1);
#pragma unroll
        for (int k = 0; k < kSeg; k += 8) {
          const uint32_t first = (r == r0 && k == 0) ? 0u : 1u;
#pragma unroll
          for (int h = 0; h < 2; ++h)
            vpx::umma_tf32(tbase + 32 * h, a0 + (4 * h * kTile + k * kRow) / 16, b0 + k * kRow / 16, idesc, first);
        }
        vpx::umma_commit(&empty[stage]);
        if (r == r1 - 1) vpx::umma_commit(&tfull);
      }
      __syncwarp();
      if (++stage == kStages) {
        stage = 0;
        phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    const int q = warp - 4;           // TMEM lane quarter = parity block i
    const int co = lane;              // lane within the block = output channel
    const bool have = r1 > r0;
    if (have) {
      vpx::mbar_wait(&tfull, 0);
      vpx::tc_fence_after();
    }
    float* base = p.part + static_cast<long long>(blockIdx.x) * p.cin * p.cout * 8;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int P = 4 * h + q;
#pragma unroll
      for (int cb = 0; cb < 32; cb += 16) {
        float v[16];
        if (have) {
          vpx::tmem_ld16(tbase + (static_cast<uint32_t>(q * 32) << 16) + 32 * h + cb, v);
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = 0.f;
        }
        if (co < p.cout) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int ci = cb + j;
            if (ci < p.cin) base[(static_cast<long long>(ci) * p.cout + co) * 8 + P] = v[j];
          }
        }
      }
    }
  }
  vpx::tc_fence_before();
  __syncthreads();
  if (warp == 2) vpx::tmem_dealloc<64>(tbase);
}

int encode_ch32(CUtensorMap* map, const float* base, const vpx::Frame& f, int box_w, int w_stride) {
  const uint64_t Wf = f.w + 2 * f.mw, Hf = f.h + 2 * f.mh, Df = f.d + 2 * f.md;
  uint64_t dims[5] = {(uint64_t)f.c, Wf, Hf, Df, (uint64_t)f.n};
  uint64_t strides[4] = {(uint64_t)f.c * 4, Wf * f.c * 4, Hf * Wf * f.c * 4, Df * Hf * Wf * f.c * 4};
  uint32_t box[5] = {32, (uint32_t)(box_w * w_stride), 1, 1, 1};
  uint32_t estr[5] = {1, (uint32_t)w_stride, 1, 1, 1};
  return vpx::encode_tiled_strided(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(base), dims,
                                   strides, box, estr, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
}

}  // namespace

namespace vpx {

// Cin, Cout <= 32 (one 32-channel block each; channel rows must be 16-byte
// multiples for TMA), coarse W a multiple of the 32-voxel segment.
int deconv_wgrad_tc_supported(const Frame& xf, const Frame& uf) {
  return xf.c <= 32 && uf.c <= 32 && xf.c % 4 == 0 && uf.c % 4 == 0 && xf.w % kSeg == 0 && uf.w == 2 * xf.w &&
         uf.h == 2 * xf.h && uf.d == 2 * xf.d && uf.n == xf.n;
}

int deconv_wgrad_tc_parts(const Frame& xf) {
  const long long rows = (long long)xf.n * xf.d * xf.h * (xf.w / kSeg);
  return static_cast<int>(rows < num_sms() ? rows : num_sms());
}

int deconv_wgrad_tc(const float* x, const Frame& xf, const float* u, const Frame& uf, float* part,
                    cudaStream_t st) {
  DwParams p{};
  p.n = xf.n;
  p.d = xf.d;
  p.h = xf.h;
  p.w = xf.w;
  p.cin = xf.c;
  p.cout = uf.c;
  p.nseg = xf.w / kSeg;
  p.rows = (long long)xf.n * xf.d * xf.h * p.nseg;
  p.P = deconv_wgrad_tc_parts(xf);
  p.x_off_d = xf.md;
  p.x_off_h = xf.mh;
  p.x_off_w = xf.mw;
  p.u_off_d = uf.md;
  p.u_off_h = uf.mh;
  p.u_off_w = uf.mw;
  p.part = part;
  CUtensorMap xm, um;
  if (int rc = encode_ch32(&xm, x, xf, kSeg, 1)) return rc;
  if (int rc = encode_ch32(&um, u, uf, kSeg, 2)) return rc;
  const int smem = kStages * kStage + 1024;
  VPX_CHECK_CUDA(cudaFuncSetAttribute(deconv_wgrad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  deconv_wgrad_kernel<<<p.P, 256, smem, st>>>(xm, um, p);
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}

}  // namespace vpx
