// Filter gradient of the 4-input-channel first layer (CosmoFlow c1:
// 4 -> 16 channels over 512^3 voxels, a 1728-entry reduction over 134M
// voxels) on tcgen05 with dense operands.
//
// x (NDHWC, 16 bytes per voxel) is read as 128-byte rows of 8 voxels x 4
// channels; u comes in a 4-channel-blocked layout [C/4][n][d][h][w][4] (written
// that way by the LeakyReLU backward that produces it) so it too forms 8-voxel
// rows per 4-channel group.  One MMA (M=128, N=128, K=8 rows = 64 voxels):
//   A rows m = (gs, j, ci): x voxel 8*(k + gs - 1) + j, channel ci (gs = 0..3,
//     four M blocks at LBO = one 128-byte row, i.e. x shifted by -8..+16 voxels)
//   B rows n = (g, j', co4): u voxel 8*k + j', channel 4g + co4
//   D[m][n] = sum_k x[...] u[...]: every (x, u) voxel pair whose W distance
//   s = 8(gs-1) + j - j' is -1, 0 or +1 is a tap c = s + 1 of the filter
//   gradient; all other entries are discarded.
// Depth tap a is the CTA's sub-task, H tap b is one MMA per b into its own
// 128-column accumulator.  The epilogue folds D into wg[co][ci][a][b][c]
// (8 entries per output) through shared memory and writes a split-K partial.
// Reference semantics: reference pkg/src/voxpar/kernels/_hot.pyx:70-93.
#include "conv_common.h"
#include "conv_simt.h"
#include "vpx_host.h"
#include "vpx_ptx.cuh"

namespace {

struct WgC4Params {
  int n, d, h, w;
  int cout;            // 16 (4 groups)
  long long rows;      // n * d * h output rows
  int P;               // row ranges (split-K)
  int x_off_d, x_off_h;
  float* part;         // [P][cout][4][27]
};

constexpr int kRowB = 128;

template <int W, int S>
__global__ void __launch_bounds__(256, 1)
    wgrad_c4_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap umap,
                    const WgC4Params p) {
  constexpr int XR = W / 8 + 4;           // x rows (of 8 voxels) per H line in the box
  constexpr int XB = (3 * XR * kRowB + 1023) / 1024 * 1024;  // three H lines (b = 0..2)
  constexpr int UPL = (W / 8) * kRowB;    // one 4-channel group plane
  constexpr int UB = 4 * UPL;
  constexpr int STAGE = (XB + UB + 1023) / 1024 * 1024;
  constexpr int KSTEPS = W / 64;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[S], empty[S], tfull;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int a = blockIdx.x % 3, pidx = blockIdx.x / 3;
  const long long r0 = p.rows * pidx / p.P, r1 = p.rows * (pidx + 1) / p.P;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      vpx::mbar_init(&full[s], 1);
      vpx::mbar_init(&empty[s], 1);
    }
    vpx::mbar_init(&tfull, 1);
    vpx::fence_barrier_init();
    vpx::tma_prefetch_desc(&xmap);
    vpx::tma_prefetch_desc(&umap);
  }
  if (warp == 2) vpx::tmem_alloc<512>(&tmem_base);
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
        const int y = t % p.h;
        t /= p.h;
        const int z = t % p.d;
        const int n = static_cast<int>(t / p.d);
        vpx::mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* sx = smem + stage * STAGE;
        vpx::mbar_arrive_expect_tx(&full[stage], 3 * XR * kRowB + UB);
        // x: rows -1 .. W/8+2 (8-voxel units) of H lines y-1..y+1 at depth z+a-1
        vpx::tma_load_5d(sx, &xmap, &full[stage], 0, -1, y - 1 + p.x_off_h, z - 1 + a + p.x_off_d, n);
#pragma unroll
        for (int g = 0; g < 4; ++g)
          vpx::tma_load_5d(sx + XB + g * UPL, &umap, &full[stage], 0, 0, y, z, g * p.n + n);
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = vpx::make_idesc(2, 128, 128, true, true);
    int stage = 0;
    uint32_t phase = 0;
    for (long long r = r0; r < r1; ++r) {
      vpx::mbar_wait(&full[stage], phase);
      vpx::tc_fence_after();
      if (vpx::elect_one()) {
        const uint32_t xb = vpx::smem_u32(smem + stage * STAGE);
        const uint32_t ub = xb + XB;
#pragma unroll
        for (int kk = 0; kk < KSTEPS; ++kk) {
          const uint64_t bdesc = vpx::make_sdesc(ub + kk * 8 * kRowB, UPL, 512, 1);
#pragma unroll
          for (int b = 0; b < 3; ++b) {
            const uint64_t adesc = vpx::make_sdesc(xb + (b * XR + kk * 8) * kRowB, kRowB, 512, 1);
            vpx::umma_tf32(tbase + b * 128, adesc, bdesc, idesc, (r > r0 || kk > 0) ? 1u : 0u);
          }
        }
        vpx::umma_commit(&empty[stage]);
        if (r == r1 - 1) vpx::umma_commit(&tfull);
      }
      __syncwarp();
      if (++stage == S) {
        stage = 0;
        phase ^= 1;
      }
    }
  }
  // ---------------------------------------------------------------- epilogue
  // all roles join: fold D_b into the 16x4x3 outputs of each (a, b)
  const bool have = r1 > r0;
  float* sD = reinterpret_cast<float*>(smem);  // [128][129], reuses the (drained) stages
  float* base = p.part + static_cast<long long>(pidx) * p.cout * 4 * 27;
  if (warp >= 4 && have) {
    vpx::mbar_wait(&tfull, 0);
    vpx::tc_fence_after();
  }
  __syncthreads();
  for (int b = 0; b < 3; ++b) {
    if (warp >= 4) {
      const int q = warp - 4, m = q * 32 + lane;
#pragma unroll 1
      for (int col = 0; col < 128; col += 16) {
        float v[16];
        if (have) {
          vpx::tmem_ld16(tbase + (static_cast<uint32_t>(q * 32) << 16) + b * 128 + col, v);
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = 0.f;
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) sD[m * 129 + col + i] = v[i];
      }
    }
    __syncthreads();
    for (int o = threadIdx.x; o < p.cout * 4 * 3; o += blockDim.x) {
      const int c = o % 3, ci = (o / 3) % 4, co = o / 12;
      const int g = co >> 2, co4 = co & 3;
      float s = 0.f;
#pragma unroll
      for (int jp = 0; jp < 8; ++jp) {
        const int t = jp + c + 7;  // = 8(gs-1) + j + 8 with s = c - 1
        const int gs = t >> 3, j = t & 7;
        s += sD[(gs * 32 + j * 4 + ci) * 129 + g * 32 + jp * 4 + co4];
      }
      base[(co * 4 + ci) * 27 + (a * 3 + b) * 3 + c] = s;
    }
    __syncthreads();
  }
  vpx::tc_fence_before();
  __syncthreads();
  if (warp == 2) vpx::tmem_dealloc<512>(tbase);
}

template <int W>
int launch_c4(const CUtensorMap& xm, const CUtensorMap& um, const WgC4Params& p, cudaStream_t st) {
  constexpr int XB = (3 * (W / 8 + 4) * 128 + 1023) / 1024 * 1024, UB = 4 * (W / 8) * 128;
  constexpr int STAGE = (XB + UB + 1023) / 1024 * 1024;
  constexpr int S0 = (200 * 1024) / STAGE;
  constexpr int S = S0 > 4 ? 4 : S0;
  static_assert(S >= 2, "stage");
  auto kern = wgrad_c4_kernel<W, S>;
  constexpr int SCRATCH = 128 * 129 * 4;  // epilogue reuses the stage buffers
  const int smem = (S * STAGE > SCRATCH ? S * STAGE : SCRATCH) + 1024;
  VPX_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  kern<<<3 * p.P, 256, smem, st>>>(xm, um, p);
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}

}  // namespace

namespace vpx {

int wgrad_c4_supported(const Frame& xf, const Frame& uf) {
  return xf.c == 4 && uf.c == 16 && xf.mw == 0 && (uf.w == 512 || uf.w == 256 || uf.w == 128 || uf.w == 64) &&
         uf.md == 0 && uf.mh == 0 && uf.mw == 0;
}

int wgrad_c4_parts(const Frame& uf) {
  const long long rows = (long long)uf.n * uf.d * uf.h;
  long long P = num_sms() / 3;
  if (P > rows) P = rows;
  return static_cast<int>(P < 1 ? 1 : P);
}

// x: NDHWC frame (C=4, no W margin); ub: u in [4][n][d][h][w][4] blocked layout.
int conv_wgrad_c4(const float* x, const Frame& xf, const float* ub, const Frame& uf, float* part,
                  cudaStream_t st) {
  WgC4Params p{};
  p.n = uf.n;
  p.d = uf.d;
  p.h = uf.h;
  p.w = uf.w;
  p.cout = uf.c;
  p.rows = (long long)uf.n * uf.d * uf.h;
  p.P = wgrad_c4_parts(uf);
  p.x_off_d = xf.md;
  p.x_off_h = xf.mh;
  p.part = part;
  const int W = uf.w;
  CUtensorMap xm, um;
  {
    const uint64_t Hf = xf.h + 2 * xf.mh, Df = xf.d + 2 * xf.md;
    uint64_t dims[5] = {32, (uint64_t)W / 8, Hf, Df, (uint64_t)xf.n};
    uint64_t strides[4] = {128, (uint64_t)W * 16, Hf * W * 16, Df * Hf * W * 16};
    uint32_t box[5] = {32, (uint32_t)(W / 8 + 4), 3, 1, 1};
    if (int rc = encode_tiled(&xm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(x), dims, strides, box,
                              CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B))
      return rc;
  }
  {
    uint64_t dims[5] = {32, (uint64_t)W / 8, (uint64_t)uf.h, (uint64_t)uf.d, (uint64_t)uf.n * 4};
    uint64_t strides[4] = {128, (uint64_t)W * 16, (uint64_t)uf.h * W * 16, (uint64_t)uf.d * uf.h * W * 16};
    uint32_t box[5] = {32, (uint32_t)(W / 8), 1, 1, 1};
    if (int rc = encode_tiled(&um, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(ub), dims, strides, box,
                              CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B))
      return rc;
  }
  switch (W) {
    case 512: return launch_c4<512>(xm, um, p, st);
    case 256: return launch_c4<256>(xm, um, p, st);
    case 128: return launch_c4<128>(xm, um, p, st);
    case 64: return launch_c4<64>(xm, um, p, st);
  }
  VPX_FAIL(VPX_ERR_UNSUPPORTED, "wgrad c4: W=%d", W);
}

}  // namespace vpx
