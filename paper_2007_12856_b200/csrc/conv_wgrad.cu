// Filter gradient of a stride-1 3x3x3 convolution on tcgen05:
//   wg[co][ci][a][b][c] = sum_v u[v][co] * x[v + (a,b,c) - 1][ci]
// The reduction runs over voxels, so both operands are voxel-major tiles in
// the NDHWC layout they already have: MN-major UMMA operands (the only TF32
// MN-major smem form is SWIZZLE_128B_BASE32B: 128-byte rows of 32 channels,
// 4-row atoms), K = 8 voxels per MMA, accumulators in TMEM.
//
//   A (M = 128 rows) = x: four 32-channel "M-blocks" at a uniform LBO.
//     mode A (Cin <= 32): block i = x shifted by i voxels (LBO = one 128-byte
//       row), i.e. M = (W tap 0..3) x (32 channel slots; slots >= Cin are TMA
//       zero-fill), so one MMA covers the three W taps at once.
//     mode B (Cin % 128 == 0): block i = channel block i of a 128-channel
//       tile (LBO = plane stride); W taps are separate MMAs.
//     mode B, Cin = 64 (tap pairs): blocks 0-1 = the 64 channels at tap t,
//       blocks 2-3 = the same channels at tap t + 1 (each tap applied in the
//       TMA coordinates), so all 128 rows are useful: 14 sub-tasks instead of
//       27 half-empty ones, every element summed in the same K order.
//   B (N = Cout tile <= 256) = u: 32-channel blocks at LBO = plane stride.
//
// Split-K: CTA (sub, p) owns sub-task `sub` (mode A: depth tap a, the three H
// taps are three MMAs into three TMEM column blocks; mode B: (tap, ci tile,
// co tile)) over the p-th contiguous range of output rows, accumulates in TMEM
// and writes its slice of partial[p][cout][cin][27] once.  A fixed-order sum
// over p (reduce_partials) makes the result deterministic.
//
// Reference semantics: reference pkg/src/voxpar/kernels/_hot.pyx:70-93.
#include "conv_common.h"
#include "conv_simt.h"
#include "vpx_host.h"
#include "vpx_ptx.cuh"

namespace {

struct WgradParams {
  int n, d, h, w;     // u extents (= x interior extents, stride 1)
  int cin, cout;
  int wseg, nxseg;    // W segment (<=128, multiple of 8) and count
  long long rows;     // n * d * h * nxseg row tasks
  int nsub, P;        // sub-tasks, row ranges
  int x_off_d, x_off_h, x_off_w;  // x frame margins
  int stride;                     // 1 or 2 (mode B only): x voxel = stride*o + tap - 1
  int ci_tiles, co_tiles;         // mode B tiling
  int pair;                       // mode B, Cin = 64: two taps per 128-row tile
  float* part;                    // [P][cout][cin][27]
};

constexpr int kRow = 128;  // bytes per smem row (32 fp32 channels)

template <bool MODE_A, int NCOUT, int S, int WMAX>
__global__ void __launch_bounds__(256, 1)
    wgrad_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap umap,
                 const WgradParams p) {
  constexpr int NCO = (NCOUT + 31) / 32;
  constexpr int XROWS = MODE_A ? 3 : 1;  // x rows (H taps) per stage
  constexpr int XPL = MODE_A ? 1 : 4;    // x channel planes per stage
  constexpr int XPLANE = XROWS * (WMAX + 4) * kRow;
  constexpr int UPLANE = WMAX * kRow;
  constexpr int XB = XPL * XPLANE, UB = NCO * UPLANE;
  constexpr int STAGE = ((XB + UB) + 1023) / 1024 * 1024;
  constexpr int COLS = MODE_A ? 3 * NCOUT : NCOUT;
  constexpr int TCOLS = COLS <= 32 ? 32 : COLS <= 64 ? 64 : COLS <= 128 ? 128 : COLS <= 256 ? 256 : 512;
  static_assert(COLS <= 512, "TMEM");

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[S], empty[S], tfull;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // sub-task and row range of this CTA
  const int sub = blockIdx.x % p.nsub, pidx = blockIdx.x / p.nsub;
  const long long r0 = p.rows * pidx / p.P, r1 = p.rows * (pidx + 1) / p.P;
  int a, b = 0, c = 0, cit = 0, cot = 0;
  int t0 = 0, t1 = -1;  // pair mode: taps of M rows 0-63 / 64-127 (-1: none)
  if (MODE_A) {
    a = sub;
  } else if (p.pair) {
    cot = sub % p.co_tiles;
    t0 = 2 * (sub / p.co_tiles);
    t1 = t0 + 1 < 27 ? t0 + 1 : -1;
    a = t0 / 9;
    b = (t0 / 3) % 3;
    c = t0 % 3;
  } else {
    cot = sub % p.co_tiles;
    int t = sub / p.co_tiles;
    cit = t % p.ci_tiles;
    t /= p.ci_tiles;
    c = t % 3;
    b = (t / 3) % 3;
    a = t / 9;
  }
  const int wseg = p.wseg;
  const int xpitch = (wseg + 4) * kRow;  // bytes between the x rows of one plane

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
  if (warp == 2) vpx::tmem_alloc<TCOLS>(&tmem_base);
  vpx::tc_fence_before();
  __syncthreads();
  vpx::tc_fence_after();
  const uint32_t tbase = tmem_base;
  vpx::pdl_wait();

  if (warp == 0) {
    if (vpx::elect_one()) {
      // mode B: channel planes actually present in this 128-channel tile (the
      // rest stay stale and only feed discarded D rows); stride-2 boxes walk
      // every second voxel (TMA element stride), so the W tap is applied in the
      // coordinate instead of as a shared-memory offset
      const int npl = MODE_A ? XPL : min(XPL, (p.cin - 128 * cit) / 32);
      const int xrows = (MODE_A || p.stride == 1) ? wseg + 4 : wseg;
      const int xw0 = (MODE_A || p.stride == 1) ? -1 : c - 1;
      const int nplx = (!MODE_A && p.pair) ? (t1 >= 0 ? 4 : 2) : npl;
      const uint32_t tx = nplx * XROWS * xrows * kRow + NCO * wseg * kRow;
      int stage = 0;
      uint32_t phase = 0;
      for (long long r = r0; r < r1; ++r) {
        long long t = r;
        const int xs = t % p.nxseg;
        t /= p.nxseg;
        const int y = t % p.h;
        t /= p.h;
        const int z = t % p.d;
        const int n = static_cast<int>(t / p.d);
        const int x0 = xs * wseg;
        vpx::mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* sx = smem + stage * STAGE;
        uint8_t* su = sx + XB;
        vpx::mbar_arrive_expect_tx(&full[stage], tx);
        const int s = MODE_A ? 1 : p.stride;
        if (!MODE_A && p.pair) {
          for (int pl = 0; pl < nplx; ++pl) {  // planes 0-1: tap t0, planes 2-3: tap t1
            const int t = pl < 2 ? t0 : t1;
            vpx::tma_load_5d(sx + pl * XPLANE, &xmap, &full[stage], 32 * (pl & 1), s * x0 + t % 3 - 1 + p.x_off_w,
                             s * y - 1 + (t / 3) % 3 + p.x_off_h, s * z - 1 + t / 9 + p.x_off_d, n);
          }
        } else {
          for (int pl = 0; pl < npl; ++pl)
            vpx::tma_load_5d(sx + pl * XPLANE, &xmap, &full[stage], 32 * (cit * 4 + pl), s * x0 + xw0 + p.x_off_w,
                             s * y - 1 + b + p.x_off_h, s * z - 1 + a + p.x_off_d, n);
        }
#pragma unroll
        for (int cb = 0; cb < NCO; ++cb)
          vpx::tma_load_5d(su + cb * UPLANE, &umap, &full[stage], 32 * (cot * NCO + cb), x0, y, z, n);
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = vpx::make_idesc(2, 128, NCOUT, true, true);
    int stage = 0;
    uint32_t phase = 0;
    for (long long r = r0; r < r1; ++r) {
      vpx::mbar_wait(&full[stage], phase);
      vpx::tc_fence_after();
      if (vpx::elect_one()) {
        const uint32_t xb = vpx::smem_u32(smem + stage * STAGE);
        const uint32_t ub = xb + XB;
        // descriptors advanced by 8 rows (1024 B = 64 in the address field)
        // per K step instead of rebuilt for every MMA by the issuing thread
        uint64_t bdesc = vpx::make_sdesc(ub, UPLANE, 512, 1);
        uint64_t adesc[MODE_A ? 3 : 1];
        if (MODE_A) {
#pragma unroll
          for (int bb = 0; bb < (MODE_A ? 3 : 1); ++bb) adesc[bb] = vpx::make_sdesc(xb + bb * xpitch, kRow, 512, 1);
        } else {
          adesc[0] = vpx::make_sdesc(xb + (p.stride == 1 && !p.pair ? c : 0) * kRow, XPLANE, 512, 1);
        }
        for (int k = 0; k < wseg; k += 8) {
          const uint32_t first = (r == r0 && k == 0) ? 0u : 1u;
#pragma unroll
          for (int bb = 0; bb < (MODE_A ? 3 : 1); ++bb) {
            vpx::umma_tf32(tbase + bb * NCOUT, adesc[bb], bdesc, idesc, first);
            adesc[bb] += 8 * kRow / 16;
          }
          bdesc += 8 * kRow / 16;
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
  } else if (warp >= 4) {
    const int q = warp - 4;
    const int m = q * 32 + lane;  // TMEM lane = M row
    const bool have = r1 > r0;
    if (have) {
      vpx::mbar_wait(&tfull, 0);
      vpx::tc_fence_after();
    }
    int ci, cc, tap = 0;
    if (MODE_A) {
      cc = m >> 5;
      ci = m & 31;
    } else if (p.pair) {
      ci = m & 63;
      tap = m < 64 ? t0 : t1;
      cc = tap < 0 ? 3 : 0;
    } else {
      cc = c;
      ci = cit * 128 + m;
      tap = (a * 3 + b) * 3 + c;
    }
    const bool valid = ci < p.cin && cc < 3;
    float* base = p.part + static_cast<long long>(pidx) * p.cout * p.cin * 27;
#pragma unroll 1
    for (int col = 0; col < COLS; col += 16) {
      float v[16];
      if (have) {
        vpx::tmem_ld16(tbase + (static_cast<uint32_t>(q * 32) << 16) + col, v);
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = 0.f;
      }
      if (valid) {
        if (MODE_A) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int nn = col + j;
            const int bb = nn / NCOUT, co = nn % NCOUT;
            if (co < p.cout) base[(static_cast<long long>(co) * p.cin + ci) * 27 + (a * 3 + bb) * 3 + cc] = v[j];
          }
        } else {
          // mode B: tap-major partials [tap][co][ci], so a warp's 32 input
          // channels are one contiguous 128-byte run (the [co][ci][tap] order
          // scattered every store 108 bytes apart: ~40 us per deep-layer
          // filter gradient); reduce_partials_tapmajor transposes back
          float* tb = base + static_cast<long long>(tap) * p.cout * p.cin;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int co = cot * NCOUT + col + j;
            if (co < p.cout) tb[static_cast<long long>(co) * p.cin + ci] = v[j];
          }
        }
      }
    }
  }
  vpx::tc_fence_before();
  __syncthreads();
  if (warp == 2) vpx::tmem_dealloc<TCOLS>(tbase);
}

int encode_ch32_map(CUtensorMap* map, const float* base, const vpx::Frame& f, int box_w, int box_h,
                    int w_stride = 1) {
  const uint64_t Wf = f.w + 2 * f.mw, Hf = f.h + 2 * f.mh, Df = f.d + 2 * f.md;
  uint64_t dims[5] = {(uint64_t)f.c, Wf, Hf, Df, (uint64_t)f.n};
  uint64_t strides[4] = {(uint64_t)f.c * 4, Wf * f.c * 4, Hf * Wf * f.c * 4, Df * Hf * Wf * f.c * 4};
  uint32_t box[5] = {32, (uint32_t)(box_w * w_stride), (uint32_t)box_h, 1, 1};
  uint32_t estr[5] = {1, (uint32_t)w_stride, 1, 1, 1};
  return vpx::encode_tiled_strided(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(base), dims,
                                   strides, box, estr, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
}

template <bool MODE_A, int NCOUT>
int launch_wgrad(const CUtensorMap& xm, const CUtensorMap& um, const WgradParams& p, cudaStream_t st) {
  constexpr int WMAX = MODE_A ? 128 : 32;
  constexpr int NCO = (NCOUT + 31) / 32;
  constexpr int XROWS = MODE_A ? 3 : 1;
  constexpr int XPL = MODE_A ? 1 : 4;
  constexpr int STAGE = ((XPL * XROWS * (WMAX + 4) * 128 + NCO * WMAX * 128) + 1023) / 1024 * 1024;
  constexpr int S = (200 * 1024) / STAGE >= 4 ? 4 : (200 * 1024) / STAGE;
  static_assert(S >= 2, "stage size");
  auto kern = wgrad_kernel<MODE_A, NCOUT, S, WMAX>;
  const int smem = S * STAGE + 1024;
  VPX_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  VPX_CHECK_CUDA(vpx::launch_pdl(kern, p.nsub * p.P, 256, smem, st, xm, um, p));
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}

// mode B with 64 input channels: two taps share the 128-row tile
bool pair_mode(const vpx::Frame& xf) {
  return xf.c == 64 && getenv("VPX_WGRAD_NOPAIR") == nullptr;
}

int nsub_of(const vpx::Frame& xf, const vpx::Frame& uf) {
  if (xf.c <= 32) return 3;
  const int nco = uf.c == 128 ? 128 : 256;
  return (pair_mode(xf) ? 14 : 27 * ((xf.c + 127) / 128)) * (uf.c / nco);
}

}  // namespace

namespace vpx {

// 1 if the tcgen05 wgrad handles this layer (k = 3 checked by the caller).
// stride 2 is handled in mode B only (Cin >= 64, the CosmoFlow c4 shape).
int wgrad_tc_supported(const Frame& xf, const Frame& uf, int stride) {
  if (uf.mw || uf.md || uf.mh) return 0;  // upstream gradients are margin-free
  const int cin = xf.c, cout = uf.c;
  // W < 8 (CosmoFlow-512 c7 at 4^3): one 8-voxel K step per row, the u rows
  // past W are TMA zero fill, so they add nothing (mode B only)
  if (uf.w < 8)
    return cin % 32 == 0 && cin >= 64 && (stride == 1 || stride == 2) && (cout == 128 || cout % 256 == 0);
  if (uf.w % 8 || (uf.w > 128 && uf.w % 128)) return 0;
  if (stride == 1 && cin <= 32 && cin % 4 == 0) return cout == 8 || cout == 16 || cout == 32 || cout == 64;
  if (cin % 32 == 0 && cin >= 64 && uf.w <= 32 && (stride == 1 || stride == 2))
    return cout == 128 || cout % 256 == 0;
  return 0;
}

// 1: the partial slices are tap-major ([tap][cout][cin], mode B) and need
// reduce_partials_tapmajor; 0: [cout][cin][tap] (mode A).
int wgrad_tc_tapmajor(const Frame& xf) { return xf.c > 32; }

// Number of partial slices the split-K reduction produces.
int wgrad_tc_parts(const Frame& xf, const Frame& uf) {
  const int nsub = nsub_of(xf, uf);
  const long long rows = (long long)uf.n * uf.d * uf.h * (uf.w < 8 ? 1 : uf.w / (uf.w < 128 ? uf.w : 128));
  // one CTA per SM (smem-limited): nsub * P must not exceed the SM count, or the
  // leftover CTAs run as a second wave and double the kernel time
  long long P = num_sms() / nsub;
  // deep layers (c6, c7 at 8^3 / 4^3): with only a few hundred voxels of K
  // per CTA the kernel is bound by writing the P partial filter gradients
  // (7 MB each at 256x256x27), not by the MMAs -- keep >= 256 voxels per slice
  const long long kvox = rows * (uf.w < 8 ? 8 : uf.w < 128 ? uf.w : 128);
  if (P > kvox / 256) P = kvox / 256;
  if (P < 1) P = 1;
  if (P > rows) P = rows;
  return static_cast<int>(P);
}

int conv_wgrad_tc(const float* x, const Frame& xf, const float* u, const Frame& uf, int stride, float* part,
                  cudaStream_t st) {
  WgradParams p{};
  p.stride = stride;
  p.n = uf.n;
  p.d = uf.d;
  p.h = uf.h;
  p.w = uf.w;
  p.cin = xf.c;
  p.cout = uf.c;
  p.wseg = uf.w < 8 ? 8 : uf.w < 128 ? uf.w : 128;
  p.nxseg = uf.w < 8 ? 1 : uf.w / p.wseg;
  p.rows = (long long)uf.n * uf.d * uf.h * p.nxseg;
  p.nsub = nsub_of(xf, uf);
  p.P = wgrad_tc_parts(xf, uf);
  p.x_off_d = xf.md;
  p.x_off_h = xf.mh;
  p.x_off_w = xf.mw;
  p.part = part;
  const bool modeA = xf.c <= 32;
  if (!modeA) {
    p.ci_tiles = (xf.c + 127) / 128;
    p.co_tiles = uf.c / (uf.c == 128 ? 128 : 256);
    p.pair = pair_mode(xf) ? 1 : 0;
  }
  CUtensorMap xm, um;
  if (modeA || stride == 1) {
    if (int rc = encode_ch32_map(&xm, x, xf, p.wseg + 4, modeA ? 3 : 1)) return rc;
  } else {
    if (int rc = encode_ch32_map(&xm, x, xf, p.wseg, 1, stride)) return rc;
  }
  if (int rc = encode_ch32_map(&um, u, uf, p.wseg, 1)) return rc;
  if (modeA) {
    switch (uf.c) {
      case 8:   // 32-wide N tile, channels beyond cout are TMA zero-fill
      case 16:
      case 32: return launch_wgrad<true, 32>(xm, um, p, st);
      case 64: return launch_wgrad<true, 64>(xm, um, p, st);
    }
  } else {
    if (uf.c == 128) return launch_wgrad<false, 128>(xm, um, p, st);
    return launch_wgrad<false, 256>(xm, um, p, st);
  }
  VPX_FAIL(VPX_ERR_UNSUPPORTED, "wgrad cout %d", uf.c);
}

}  // namespace vpx
