// Filter gradient of a stride-1 3x3x3 convolution with 16 input and 32 output
// channels (CosmoFlow c2), with the upstream gradient u as the MMA's A operand
// in TMEM:
//   wg[co][ci][a][b][c] = sum_v u[v][co] * x[v + (a,b,c) - 1][ci]
//
// A (128 TMEM lanes) = u of TWO consecutive rows y, y+1 at two W-shifts each:
//   lane (r, d, co), column k  ->  u[row y+r][2k + d + 1][co]      (r, d in {0,1})
// B = an input row X as 128-byte chunks of 2 voxels x 16 channels (MN-major
//   SWIZZLE_128B_BASE32B), N = 64: chunks k and k+1 (LBO = one chunk row).
// One MMA per input row X in y-1 .. y+2 (4 MMAs per K step) accumulates
//   D_X[(r, d, co)][(j, e, ci)] += u[y+r][2k+d+1][co] * x[X][2k+2j+e][ci],
// i.e. height tap b = X - y - r + 1 and width tap c = 2j + e - d whenever both
// are in 0..2: six of the eight lane halves and 3 of 4 voxel slots are useful
// (56%), against 37.5% for the shared-memory-A kernel (conv_wgrad.cu mode A),
// and the MMA reads only B (N = 64 -> 32 cycles) from shared memory.
// Depth tap a is the CTA's sub-task (4 x 64 accumulator columns + an 8-slot A
// ring fit in TMEM; 9 taps would not).  The input rows of depth z+a-1 stay in
// an 8-row shared-memory ring, so consecutive row pairs reuse them; u arrives
// in 4 KB TMA boxes per K step and four producer warps copy it into TMEM.
// Split-K over row pairs, partial slices reduced in a fixed order.
// Reference semantics: reference pkg/src/voxpar/kernels/_hot.pyx:70-93.
#include "conv_common.h"
#include "conv_simt.h"
#include "vpx_host.h"
#include "vpx_ptx.cuh"

namespace {

struct UtParams {
  int n, d, h;               // u extents (h even); W is the template parameter
  long long pairs;           // n * d * h / 2 row pairs
  int P;                     // row-pair ranges (split-K)
  int x_off_d, x_off_h;      // x frame margins
  float* part;               // [P][32][16][27]
};

constexpr int kAcc = 64;          // N per accumulator
constexpr int kACol = 4 * kAcc;   // A ring starts at TMEM column 256
constexpr int kSlots = 8;         // A slots in TMEM, 16 columns (two K=8 steps) each
constexpr int kUSt = 8;           // u stages in shared memory (TMA lookahead)

template <int W>
struct UtCfg {
  static constexpr int KS = (W / 2 + 1 + 15) / 16;        // 16-row slots per row pair (k = -1 .. 16KS-2)
  static constexpr int XCH = 16 * KS + 1;                 // x chunks -1 .. 16KS-1
  static constexpr int XROW = (XCH * 128 + 1023) / 1024 * 1024;
  static constexpr int XS = 8 * XROW;                     // 8-row ring of input rows
  static constexpr int UST = 2 * 32 * 32 * 4;             // u box: 2 rows x 32 voxels x 32 ch (8 KB)
  static constexpr int PIPE = XS + kUSt * UST;
  static constexpr int SCRATCH = 4 * 32 * 16 * 9 * 4;    // epilogue fold
  static constexpr int SMEM = PIPE > SCRATCH ? PIPE : SCRATCH;
};

template <int W>
__global__ void __launch_bounds__(384, 1)
    wgrad_ut_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap umap,
                    const UtParams p) {
  using Cfg = UtCfg<W>;
  constexpr int KS = Cfg::KS, XROW = Cfg::XROW;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* xs = smem;
  uint8_t* us = smem + Cfg::XS;
  __shared__ __align__(8) uint64_t xfull[4], rowdone[4], ufull[kUSt], uempty[kUSt], fullA[kSlots],
      emptyA[kSlots], tfull;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int a = blockIdx.x % 3, pidx = blockIdx.x / 3;
  const long long r0 = p.pairs * pidx / p.P, r1 = p.pairs * (pidx + 1) / p.P;
  const int hp = p.h / 2;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) {
      vpx::mbar_init(&xfull[i], 1);
      vpx::mbar_init(&rowdone[i], 1);
    }
    for (int i = 0; i < kUSt; ++i) {
      vpx::mbar_init(&ufull[i], 1);
      vpx::mbar_init(&uempty[i], 4);
    }
    for (int i = 0; i < kSlots; ++i) {
      vpx::mbar_init(&fullA[i], 4);
      vpx::mbar_init(&emptyA[i], 1);
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

  auto decode = [&](long long pr, int& n, int& z, int& y) {
    y = 2 * static_cast<int>(pr % hp);
    pr /= hp;
    z = static_cast<int>(pr % p.d);
    n = static_cast<int>(pr / p.d);
  };

  if (warp == 0) {
    // ---------------------------------------------- input rows (8-row ring)
    if (vpx::elect_one()) {
      for (long long pr = r0; pr < r1; ++pr) {
        const int i = static_cast<int>(pr - r0);
        int n, z, y;
        decode(pr, n, z, y);
        const bool reset = (i == 0) || (y == 0);
        // ring slot of row X is X & 7; rows y+1, y+2 overwrite y-7, y-6, last
        // read by pair i-3; a reset reloads four rows and waits for pair i-1
        if (reset && i >= 1) vpx::mbar_wait_sleep(&rowdone[(i - 1) & 3], ((i - 1) >> 2) & 1, 20);
        else if (i >= 3) vpx::mbar_wait_sleep(&rowdone[(i - 3) & 3], ((i - 3) >> 2) & 1, 20);
        const int first = reset ? y - 1 : y + 1;
        const int nrow = reset ? 4 : 2;
        vpx::mbar_arrive_expect_tx(&xfull[i & 3], nrow * Cfg::XCH * 128);
        for (int j = 0; j < nrow; ++j) {
          const int X = first + j;
          vpx::tma_load_5d(xs + (X & 7) * XROW, &xmap, &xfull[i & 3], 0, -1, X + p.x_off_h, z - 1 + a + p.x_off_d,
                           n);
        }
      }
    }
  } else if (warp == 3) {
    // ---------------------------------------------- u boxes, one per K step
    if (vpx::elect_one()) {
      uint32_t g = 0;
      for (long long pr = r0; pr < r1; ++pr) {
        int n, z, y;
        decode(pr, n, z, y);
        for (int s = 0; s < KS; ++s, ++g) {
          const int st = g & (kUSt - 1);
          vpx::mbar_wait_sleep(&uempty[st], ((g / kUSt) & 1) ^ 1, 20);
          vpx::mbar_arrive_expect_tx(&ufull[st], Cfg::UST);
          vpx::tma_load_5d(us + st * Cfg::UST, &umap, &ufull[st], 0, 32 * s - 1, y, z, n);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA
    constexpr uint32_t idesc = vpx::make_idesc(2, 128, kAcc, false, true);
    if (vpx::elect_one()) {  // one thread issues everything
      const uint32_t xb = vpx::smem_u32(xs);
      uint32_t g = 0;
      int y = 2 * static_cast<int>(r0 % hp);
      for (long long pr = r0; pr < r1; ++pr) {
        const int i = static_cast<int>(pr - r0);
        vpx::mbar_wait(&xfull[i & 3], (i >> 2) & 1);
        uint64_t bd[4];  // input rows y-1 .. y+2 at K step 0
#pragma unroll
        for (int X = 0; X < 4; ++X) bd[X] = vpx::make_sdesc(xb + ((y - 1 + X) & 7) * XROW, 128, 512, 1);
        for (int s = 0; s < KS; ++s, ++g) {
          const int slot = g & (kSlots - 1);
          vpx::mbar_wait(&fullA[slot], (g / kSlots) & 1);
          vpx::tc_fence_after();
          const uint32_t acol = tbase + kACol + slot * 16;
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {  // two K=8 steps per slot; 8 chunk rows (1024 B) each
            const uint32_t acc = (i > 0 || s > 0 || hh > 0) ? 1u : 0u;
#pragma unroll
            for (int X = 0; X < 4; ++X)
              vpx::umma_tf32_ta(tbase + X * kAcc, acol + 8 * hh, bd[X] + static_cast<uint64_t>((2 * s + hh) * 64),
                                idesc, acc);
          }
          vpx::umma_commit(&emptyA[slot]);
        }
        vpx::umma_commit(&rowdone[i & 3]);
        if (pr == r1 - 1) vpx::umma_commit(&tfull);
        y = (y + 2 == p.h) ? 0 : y + 2;
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------ u -> TMEM (A operand)
    // two warps per TMEM lane quarter (warps 4..7, 8..11) take alternate K
    // steps; each loads its next slot while the previous tcgen05.st drains
    const int q = warp & 3, h = (warp - 4) >> 2;  // lane quarter = (r, d) = (q >> 1, q & 1); lane = co
    const int r = q >> 1, dsh = q & 1;
    const uint32_t lane_addr = tbase + (static_cast<uint32_t>(q * 32) << 16) + kACol;
    const uint32_t ub = vpx::smem_u32(us) + (r * 32 + dsh) * 128 + lane * 4;
    const uint32_t total = static_cast<uint32_t>((r1 - r0) * KS);
    auto load = [&](uint32_t g, float (&v)[16]) {
      const int st = g & (kUSt - 1);
      vpx::mbar_wait(&ufull[st], (g / kUSt) & 1);
      const uint32_t base = ub + st * Cfg::UST;  // column kk: box voxel 2kk + d
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) v[kk] = vpx::lds_f32(base + kk * 256);
      __syncwarp();
      if (lane == 0) vpx::mbar_arrive(&uempty[st]);
    };
    float v[16];
    uint32_t g = h;
    if (g < total) load(g, v);
    for (; g < total; g += 2) {
      const int st = g & (kSlots - 1);
      vpx::mbar_wait(&emptyA[st], ((g / kSlots) & 1) ^ 1);
      vpx::tmem_st16(lane_addr + st * 16, v);
      if (g + 2 < total) load(g + 2, v);  // overlaps the store
      vpx::tmem_st_wait();
      vpx::tc_fence_before();
      __syncwarp();
      if (lane == 0) vpx::mbar_arrive(&fullA[st]);
    }
  }

  // ---------------------------------------------------------------- epilogue
  const bool have = r1 > r0;
  if (warp >= 4 && warp < 8 && have) {
    vpx::mbar_wait_sleep(&tfull, 0, 256);
    vpx::tc_fence_after();
  }
  __syncthreads();  // all TMA landed and consumed, all MMAs retired: reuse the ring
  float* red = reinterpret_cast<float*>(smem);  // [q][co][ci][9 (b,c)]
  if (warp >= 4 && warp < 8) {
    const int q = warp - 4, r = q >> 1, dsh = q & 1;
    float* rq = red + (q * 32 + lane) * 16 * 9;
    for (int t = 0; t < 16 * 9; ++t) rq[t] = 0.f;
#pragma unroll 1
    for (int X = 0; X < 4; ++X) {
      const int b = X - r;  // height tap of this accumulator for u row y+r
      if (b < 0 || b > 2) continue;
      float v[kAcc];
      if (have) {
#pragma unroll
        for (int c16 = 0; c16 < kAcc / 16; ++c16) {
          float t16[16];
          vpx::tmem_ld16(tbase + (static_cast<uint32_t>(q * 32) << 16) + X * kAcc + 16 * c16, t16);
#pragma unroll
          for (int j = 0; j < 16; ++j) v[16 * c16 + j] = t16[j];
        }
      } else {
#pragma unroll
        for (int j = 0; j < kAcc; ++j) v[j] = 0.f;
      }
      // column n = 32 j + 16 e + ci holds x voxel offset t = 2j + e; width tap c = t - d
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int c = t - dsh;
        if (c >= 0 && c <= 2) {
#pragma unroll
          for (int ci = 0; ci < 16; ++ci) rq[ci * 9 + b * 3 + c] = v[(t >> 1) * 32 + (t & 1) * 16 + ci];
        }
      }
    }
  }
  __syncthreads();
  float* base = p.part + static_cast<long long>(pidx) * 32 * 16 * 27;
  for (int o = threadIdx.x; o < 32 * 16 * 9; o += blockDim.x) {
    const int co = o / (16 * 9), rem = o % (16 * 9), ci = rem / 9, bc = rem % 9;
    float s = 0.f;
#pragma unroll
    for (int q = 0; q < 4; ++q) s += red[(q * 32 + co) * 16 * 9 + rem];
    base[(co * 16 + ci) * 27 + a * 9 + bc] = s;
  }
  vpx::tc_fence_before();
  __syncthreads();
  if (warp == 2) vpx::tmem_dealloc<512>(tbase);
}

template <int W>
int launch_ut(const CUtensorMap& xm, const CUtensorMap& um, const UtParams& p, cudaStream_t st) {
  constexpr int smem = UtCfg<W>::SMEM + 1024;
  static_assert(smem <= 227 * 1024, "smem");
  auto kern = wgrad_ut_kernel<W>;
  VPX_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  kern<<<3 * p.P, 384, smem, st>>>(xm, um, p);
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}

}  // namespace

namespace vpx {

int wgrad_ut_supported(const Frame& xf, const Frame& uf, int stride) {
  if (precision() != 0 || stride != 1) return 0;
  if (xf.c != 16 || uf.c != 32 || xf.mw || uf.md || uf.mh || uf.mw) return 0;
  if (!(uf.w == 128 || uf.w == 256) || uf.h % 2) return 0;
  return xf.n == uf.n && xf.d == uf.d && xf.h == uf.h && xf.w == uf.w;
}

int wgrad_ut_parts(const Frame& uf) {
  const long long pairs = (long long)uf.n * uf.d * uf.h / 2;
  long long P = num_sms() / 3;
  if (P > pairs) P = pairs;
  return static_cast<int>(P < 1 ? 1 : P);
}

int conv_wgrad_ut(const float* x, const Frame& xf, const float* u, const Frame& uf, float* part, cudaStream_t st) {
  UtParams p{};
  p.n = uf.n;
  p.d = uf.d;
  p.h = uf.h;
  p.pairs = (long long)uf.n * uf.d * uf.h / 2;
  p.P = wgrad_ut_parts(uf);
  p.x_off_d = xf.md;
  p.x_off_h = xf.mh;
  p.part = part;
  const int W = uf.w;
  const int xch = W == 256 ? UtCfg<256>::XCH : UtCfg<128>::XCH;
  CUtensorMap xm, um;
  {
    const uint64_t Hf = xf.h + 2 * xf.mh, Df = xf.d + 2 * xf.md;
    uint64_t dims[5] = {32, (uint64_t)W / 2, Hf, Df, (uint64_t)xf.n};
    uint64_t strides[4] = {128, (uint64_t)W * 64, Hf * W * 64, Df * Hf * W * 64};
    uint32_t box[5] = {32, (uint32_t)xch, 1, 1, 1};
    if (int rc = encode_tiled(&xm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(x), dims, strides, box,
                              CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B))
      return rc;
  }
  {
    uint64_t dims[5] = {32, (uint64_t)W, (uint64_t)uf.h, (uint64_t)uf.d, (uint64_t)uf.n};
    uint64_t strides[4] = {128, (uint64_t)W * 128, (uint64_t)uf.h * W * 128, (uint64_t)uf.d * uf.h * W * 128};
    uint32_t box[5] = {32, 32, 2, 1, 1};
    if (int rc = encode_tiled(&um, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(u), dims, strides, box,
                              CU_TENSOR_MAP_SWIZZLE_NONE))
      return rc;
  }
  if (W == 256) return launch_ut<256>(xm, um, p, st);
  return launch_ut<128>(xm, um, p, st);
}

}  // namespace vpx
