// Filter gradient of a stride-1 3x3x3 convolution with equal, small channel
// counts (Cin = Cout = CH in {8, 16, 32}: the U-Net levels), on tcgen05:
//   wg[co][ci][a][b][c] = sum_v u[v][co] * x[v + (a,b,c) - 1][ci]
//
// A CH-channel row viewed as 128-byte rows holds G = 32 / CH consecutive
// voxels, so both operands are the activations exactly as they lie in HBM
// (NDHWC), loaded by TMA as "group rows" (MN-major SWIZZLE_128B_BASE32B), K =
// 8 voxel groups per MMA:
//   A (M = 128) = four 32-lane blocks at LBO = one u row in shared memory:
//       block j = u row (z, y' - 1 + j) (j = 3 is padding), lane (d, co) of
//       group k = u[G k + d][co];
//   B (N = 96)  = x row (z + a - 1, y') as groups k - 1, k, k + 1 (LBO = 128 B),
//       column (e, ci) = x[G (k - 1) + e][ci].
// D_a[(j, d, co)][(e, ci)] accumulates the tap (a, b = 2 - j, c = e - d - G + 1)
// for every valid c in 0..2, so one MMA covers all 9 (b, c) taps of a depth tap
// a for G voxels x CH channels; the three depth taps are three MMAs with the
// same A into three 96-column accumulators.  u rows live in a 12-slot ring
// (plus mirrored copies of slots 0..2, so the 4 rows of A are always
// contiguous); x rows stream through 3 stages.  Compared with the generic
// mode-A kernel (32-channel slots, 1 voxel per row) this removes the
// channel padding: 8x less MMA work at CH = 8.
//
// Split-K over row ranges, per-CTA partials, fixed-order reduction afterwards
// (deterministic).  Reference semantics: reference pkg/src/voxpar/kernels/_hot.pyx:70-93.
#include <cstdlib>

#include "conv_common.h"
#include "conv_simt.h"
#include "vpx_host.h"
#include "vpx_ptx.cuh"

namespace {

struct WgParams {
  int n, d, h, w;           // u extents (= x interior extents)
  int hs;                   // x rows per plane: h + 2 * x_off_h (margin rows hold halos)
  long long rows;           // n * d * hs  (one step per x row (n, z, y'))
  int P;
  int x_off_d, x_off_h;     // x frame margins (W margin must be 0)
  float* part;              // [P][CH][CH][27]
};

constexpr int kRing = 12;   // u ring slots (+3 mirrored)
constexpr int kStages = 3;  // x stages (3 rows each)
constexpr int kN = 96;      // B columns: x groups k-1, k, k+1

template <int CH, int W>
struct WgCfg {
  static constexpr int G = 32 / CH;
  static constexpr int GROUPS = W / G;
  static constexpr int KS = GROUPS / 8;
  static constexpr int USL = (GROUPS * 128 + 1023) / 1024 * 1024;
  static constexpr int XROW = ((GROUPS + 2) * 128 + 1023) / 1024 * 1024;
  static constexpr int XST = 3 * XROW;
  static constexpr int UBYTES = (kRing + 3) * USL;
  static constexpr int PIPE = UBYTES + kStages * XST;
  static constexpr int SCRATCH = 3 * G * CH * CH * 9 * 4;
  static constexpr int SMEM = PIPE > SCRATCH ? PIPE : SCRATCH;
  static_assert(GROUPS % 8 == 0 && GROUPS <= 64, "rows of 8..64 groups");
};

template <int CH, int W>
__global__ void __launch_bounds__(256, 1)
    wgrad_g_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap umap,
                   const WgParams p) {
  using Cfg = WgCfg<CH, W>;
  constexpr int G = Cfg::G;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* su = smem;
  uint8_t* sx = smem + Cfg::UBYTES;
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages], tfull;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pidx = blockIdx.x;
  const long long r0 = p.rows * pidx / p.P, r1 = p.rows * (pidx + 1) / p.P;

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
  if (warp == 2) vpx::tmem_alloc<512>(&tmem_base);
  vpx::tc_fence_before();
  __syncthreads();
  vpx::tc_fence_after();
  const uint32_t tbase = tmem_base;

  if (warp == 0) {
    if (vpx::elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      int q = 0;  // ring position of A block 0 (u row y' - 1)
      for (long long r = r0; r < r1; ++r) {
        long long t = r;
        const int y = static_cast<int>(t % p.hs) - p.x_off_h;
        t /= p.hs;
        const int z = static_cast<int>(t % p.d);
        const int n = static_cast<int>(t / p.d);
        const bool fresh = r == r0 || y == -p.x_off_h;
        if (r != r0) q += fresh ? 4 : 1;
        vpx::mbar_wait(&empty[stage], phase ^ 1);
        const int nu = fresh ? 4 : 1;
        int ncopy = 0;
        for (int i = 4 - nu; i < 4; ++i) ncopy += ((q + i) % kRing) < 3;
        vpx::mbar_arrive_expect_tx(&full[stage], (nu + ncopy) * Cfg::GROUPS * 128 + 3 * (Cfg::GROUPS + 2) * 128);
        for (int i = 4 - nu; i < 4; ++i) {
          const int slot = (q + i) % kRing;
          const int yy = y - 1 + i;  // rows outside [0, h) are TMA zero fill
          vpx::tma_load_5d(su + slot * Cfg::USL, &umap, &full[stage], 0, 0, yy, z, n);
          if (slot < 3) vpx::tma_load_5d(su + (kRing + slot) * Cfg::USL, &umap, &full[stage], 0, 0, yy, z, n);
        }
        uint8_t* xs = sx + stage * Cfg::XST;
#pragma unroll
        for (int a = 0; a < 3; ++a)
          vpx::tma_load_5d(xs + a * Cfg::XROW, &xmap, &full[stage], 0, -1, y + p.x_off_h, z - 1 + a + p.x_off_d, n);
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (vpx::elect_one()) {
      constexpr uint32_t idesc = vpx::make_idesc(2, 128, kN, true, true);
      int stage = 0;
      uint32_t phase = 0;
      int q = 0;
      const uint32_t ubase = vpx::smem_u32(su), xbase = vpx::smem_u32(sx);
      for (long long r = r0; r < r1; ++r) {
        const int y = static_cast<int>(r % p.hs);
        if (r != r0) q += (y == 0) ? 4 : 1;
        vpx::mbar_wait(&full[stage], phase);
        vpx::tc_fence_after();
        const uint32_t ua = ubase + (q % kRing) * Cfg::USL;
        const uint32_t xa = xbase + stage * Cfg::XST;
        const uint32_t first = r == r0 ? 0u : 1u;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          uint64_t adesc = vpx::make_sdesc(ua, Cfg::USL, 512, 1);
          uint64_t bdesc = vpx::make_sdesc(xa + a * Cfg::XROW, 128, 512, 1);
#pragma unroll 1
          for (int j = 0; j < Cfg::KS; ++j) {
            vpx::umma_tf32(tbase + a * kN, adesc, bdesc, idesc, (j == 0) ? first : 1u);
            adesc += 1024 >> 4;  // next 8 groups
            bdesc += 1024 >> 4;
          }
        }
        vpx::umma_commit(&empty[stage]);
        if (r == r1 - 1) vpx::umma_commit(&tfull);
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    __syncwarp();
  }
  // epilogue: warps 4..7 own TMEM lanes 32 (warp - 4) .. +31 = A block j
  const bool have = r1 > r0;
  float* scratch = reinterpret_cast<float*>(smem);  // [j][d][co][ci][a][c], after all MMAs
  if (warp >= 4) {
    if (have) {
      vpx::mbar_wait(&tfull, 0);
      vpx::tc_fence_after();
    }
    const int j = warp - 4;
    const int d = lane / CH, co = lane % CH;
#pragma unroll 1
    for (int a = 0; a < 3; ++a) {
#pragma unroll 1
      for (int col = 0; col < kN; col += 16) {
        float v[16];
        if (have) {
          vpx::tmem_ld16(tbase + (static_cast<uint32_t>(j * 32) << 16) + a * kN + col, v);
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = 0.f;
        }
        if (j < 3) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int nn = col + i;
            const int e = (nn >> 5) * G + (nn & 31) / CH, ci = nn % CH;
            const int c = e - d - G + 1;
            if (c >= 0 && c <= 2) scratch[((((j * G + d) * CH + co) * CH + ci) * 3 + a) * 3 + c] = v[i];
          }
        }
      }
    }
  }
  vpx::tc_fence_before();
  __syncthreads();
  float* out = p.part + static_cast<long long>(pidx) * CH * CH * 27;
  for (int o = threadIdx.x; o < CH * CH * 27; o += blockDim.x) {
    const int tap = o % 27, ci = (o / 27) % CH, co = o / (27 * CH);
    const int a = tap / 9, b = (tap / 3) % 3, c = tap % 3, j = 2 - b;
    float s = 0.f;
#pragma unroll
    for (int d = 0; d < G; ++d) s += scratch[((((j * G + d) * CH + co) * CH + ci) * 3 + a) * 3 + c];
    out[o] = s;
  }
  if (warp == 2) vpx::tmem_dealloc<512>(tbase);
}

// Group-row view of a CH-channel NDHWC frame (W margin 0): rows of 32 floats.
int encode_group_map(CUtensorMap* map, const float* base, const vpx::Frame& f, int box_groups) {
  const int G = 32 / f.c;
  const uint64_t Hf = f.h + 2 * f.mh, Df = f.d + 2 * f.md;
  const uint64_t row = (uint64_t)f.w * f.c * 4;
  uint64_t dims[5] = {32, (uint64_t)(f.w / G), Hf, Df, (uint64_t)f.n};
  uint64_t strides[4] = {128, row, Hf * row, Df * Hf * row};
  uint32_t box[5] = {32, (uint32_t)box_groups, 1, 1, 1};
  return vpx::encode_tiled(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(base), dims, strides, box,
                           CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
}

template <int CH, int W>
int launch_wg(const CUtensorMap& xm, const CUtensorMap& um, const WgParams& p, cudaStream_t st) {
  using Cfg = WgCfg<CH, W>;
  auto kern = wgrad_g_kernel<CH, W>;
  const int smem = Cfg::SMEM + 1024;
  VPX_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  kern<<<p.P, 256, smem, st>>>(xm, um, p);
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}

}  // namespace

namespace vpx {

int wgrad_g_supported(const Frame& xf, const Frame& uf, int stride) {
  if (stride != 1 || xf.c != uf.c || xf.mw || uf.md || uf.mh || uf.mw) return 0;
  if (xf.c != 8 && xf.c != 16 && xf.c != 32) return 0;
  const int G = 32 / xf.c, g = uf.w / G;
  return uf.w % G == 0 && (g == 8 || g == 16 || g == 32 || g == 64);
}

int wgrad_g_parts(const Frame& uf) {
  const long long rows = (long long)uf.n * uf.d * uf.h;
  const long long P = num_sms();
  return static_cast<int>(rows < P ? rows : P);
}

int conv_wgrad_g(const float* x, const Frame& xf, const float* u, const Frame& uf, float* part, cudaStream_t st) {
  if (!wgrad_g_supported(xf, uf, 1)) VPX_FAIL(VPX_ERR_UNSUPPORTED, "grouped wgrad: shape");
  const int CH = xf.c, G = 32 / CH, groups = uf.w / G;
  WgParams p;
  p.n = uf.n;
  p.d = uf.d;
  p.h = uf.h;
  p.w = uf.w;
  p.hs = uf.h + 2 * xf.mh;
  p.rows = (long long)uf.n * uf.d * p.hs;
  p.P = wgrad_g_parts(uf);
  p.x_off_d = xf.md;
  p.x_off_h = xf.mh;
  p.part = part;
  CUtensorMap xm, um;
  if (int rc = encode_group_map(&xm, x, xf, groups + 2)) return rc;
  if (int rc = encode_group_map(&um, u, uf, groups)) return rc;
#define WG_CASE(ch, g)                                          \
  if (CH == ch && groups == g) return launch_wg<ch, g * (32 / ch)>(xm, um, p, st);
  WG_CASE(8, 64) WG_CASE(8, 32) WG_CASE(8, 16) WG_CASE(8, 8)
  WG_CASE(16, 64) WG_CASE(16, 32) WG_CASE(16, 16) WG_CASE(16, 8)
  WG_CASE(32, 64) WG_CASE(32, 32) WG_CASE(32, 16) WG_CASE(32, 8)
#undef WG_CASE
  VPX_FAIL(VPX_ERR_UNSUPPORTED, "grouped wgrad: %d channels, %d groups", CH, groups);
}

}  // namespace vpx
