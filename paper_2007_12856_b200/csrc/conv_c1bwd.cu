// Backward of the first CosmoFlow block (Conv3d 4 -> 16, LeakyReLU, 2^3 average
// pool) in ONE kernel: the filter gradient is computed straight from the pooled
// gradient, without materialising the 16-channel full-resolution gradient.
//
//   u[v][co]  = leaky'(y[v][co]) * up[v/2][co] / 8        (pool + LeakyReLU bwd)
//   wg[co][ci][a][b][c] = sum_v u[v][co] * x[v + (a,b,c) - 1][ci]
//
// tcgen05 with the A operand in TMEM: the producer warps compute u for 64
// voxels at a time and store it with tcgen05.st as A[m = (d, co)][k] =
// u[8k + d + 1][co] (8 W-shifts d x 16 channels = 128 lanes, one column per
// 8-voxel group k); B is the input row as 128-byte rows of 8 voxels x 4
// channels (MN-major SWIZZLE_128B_BASE32B, N = 48: rows k and k+1).  Entry
// (d, co) x (e, ci) of D_ab accumulates u[8k+d+1][co] * x[8k+e][ci], i.e. W tap
// c = e - d of the filter gradient when 0 <= c <= 2 (the rest is discarded).
// Each of the 9 (depth, height) taps is one MMA on its own x row into its own
// 48-column accumulator (432 TMEM columns); A cycles through an 8-slot ring
// in the remaining 64 columns.  The MMA reads only B from shared memory, so a
// K=8 step costs ~N/2 cycles instead of the (A + B)/128 B/clk of a
// shared-memory A operand.
//
// Warp roles: w0 TMA (x rows into a 4-row ring per depth tap, y and pooled
// gradient rows), w1 MMA issuer, w2 TMEM owner, w4..w11 u producers (w4..w7 also the
// epilogue: fold D into wg, split-K partial per CTA, fixed-order reduction
// afterwards -> deterministic).
// Reference semantics: reference pkg/src/voxpar/kernels/_hot.pyx:70-93 (filter
// gradient), layers/reference.py:170-173 (avg pool bwd), :231-236 (leaky bwd).
#include <cstdlib>

#include "conv_common.h"
#include "conv_simt.h"
#include "vpx_host.h"
#include "vpx_ptx.cuh"
#include "vpx_round.cuh"

namespace {

__device__ __forceinline__ long long globaltimer_ns() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

struct C1Params {
  int n, d, h;              // u (= y) interior extents, W is the template parameter
  long long rows;           // n * d * h
  int P;                    // CTAs (row ranges)
  int x_off_d, x_off_h;     // x frame margins
  int y_off_d, y_off_h;     // y frame margins
  int up_off_d, up_off_h;   // pooled-gradient frame margins
  float slope;
  int dbg;                  // profiling switch (VPX_C1_DEBUG): 1 skip u math, 2 skip TMEM stores
  float* part;              // [P][16][4][27]
};

constexpr int kNA = 48;          // N per tap (x chunks k, k+1: 64 > 48 used columns)
constexpr int kACol = 9 * kNA;   // first A column (432)
constexpr int kASlots = 8;       // A ring: 8 slots x 8 columns
constexpr int kRowBlock = 16;    // rows per round-robin block of the CTA row assignment
constexpr int kProdGroups = 4;   // u producer warps per TMEM lane quarter (power of 2)
constexpr int kProdWarps = 4 * kProdGroups;

// SRC: 0 = u from the LeakyReLU output y and the pooled gradient, 1 = from the
// sign mask and the pooled gradient, 2 = u itself (any conv 4 -> 16 whose
// upstream gradient is already materialised, e.g. after BatchNorm)
template <int W, int SRC = 0>
struct C1Cfg {
  static constexpr int KS = (W / 8 + 1 + 7) / 8;           // K-steps per row (k = -1 .. 8KS-2)
  static constexpr int XCH = 8 * KS + 1;                   // x chunks per row (-1 .. 8KS-1)
  static constexpr int XROW = (XCH * 128 + 1023) / 1024 * 1024;
  static constexpr int XS = 12 * XROW;                     // 3 depth taps x 4-row ring
  static constexpr int YB = SRC == 1 ? W * 2 : W * 16 * 4; // y / u row, or its 16-bit sign-mask row
  static constexpr int UB = SRC == 2 ? 0 : W / 2 * 16 * 4;  // pooled-gradient row
  static constexpr int PIPE = XS + 2 * YB + 2 * UB;
  static constexpr int SCRATCH = 128 * 108 * 4;            // epilogue fold, reuses the pipeline buffers
  static constexpr int SMEM = PIPE > SCRATCH ? PIPE : SCRATCH;
};

template <int W, int SRC>
__global__ void __launch_bounds__(128 + 32 * kProdWarps, 1)
    c1_pooled_wgrad_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap ymap,
                           const __grid_constant__ CUtensorMap upmap, const C1Params p) {
  using Cfg = C1Cfg<W, SRC>;
  constexpr bool MASK = SRC == 1;
  constexpr int KS = Cfg::KS, XROW = Cfg::XROW;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* xs = smem;
  uint8_t* ys = smem + Cfg::XS;
  uint8_t* us = ys + 2 * Cfg::YB;
  __shared__ __align__(8) uint64_t xfull[2], yfull[2], yempty[2], rowdone[2], fullA[kASlots], emptyA[kASlots],
      tfull;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pidx = blockIdx.x;
  // Rows go to CTAs in round-robin blocks of kRowBlock (not one contiguous
  // range each): all CTAs then work inside a window of a few depth planes, so
  // the x rows every depth tap re-reads come from L2 instead of HBM (a
  // contiguous range per CTA re-read each x plane from DRAM for the next depth).
  const long long nblk = (p.rows + kRowBlock - 1) / kRowBlock;
  const long long myblk = pidx < nblk ? (nblk - 1 - pidx) / p.P + 1 : 0;
  long long nseq = myblk * kRowBlock;
  if (myblk > 0) {
    const long long lastend = (pidx + (myblk - 1) * p.P + 1) * kRowBlock;
    if (lastend > p.rows) nseq -= lastend - p.rows;
  }
  auto row_of = [&](long long i) -> long long {
    return (pidx + (i / kRowBlock) * p.P) * kRowBlock + i % kRowBlock;
  };

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      vpx::mbar_init(&xfull[i], 1);
      vpx::mbar_init(&yfull[i], 1);
      vpx::mbar_init(&yempty[i], kProdWarps);
      vpx::mbar_init(&rowdone[i], 1);
    }
    for (int i = 0; i < kASlots; ++i) {
      vpx::mbar_init(&fullA[i], 4);
      vpx::mbar_init(&emptyA[i], 1);
    }
    vpx::mbar_init(&tfull, 1);
    vpx::fence_barrier_init();
    vpx::tma_prefetch_desc(&xmap);
    vpx::tma_prefetch_desc(&ymap);
    vpx::tma_prefetch_desc(&upmap);
  }
  if (warp == 2) vpx::tmem_alloc<512>(&tmem_base);
  vpx::tc_fence_before();
  __syncthreads();
  vpx::tc_fence_after();
  const uint32_t tbase = tmem_base;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (p.dbg < 4 && vpx::elect_one()) {
      for (long long ii = 0; ii < nseq; ++ii) {
        const int i = static_cast<int>(ii);
        const long long r = row_of(ii);
        long long t = r;
        const int y = t % p.h;
        t /= p.h;
        const int z = t % p.d;
        const int n = static_cast<int>(t / p.d);
        const bool reset = (i % kRowBlock == 0) || (y == 0);
        // warm L2 with the x rows two steps ahead (the ring only holds one
        // row of lookahead per depth tap)
        if (i % kRowBlock + 2 < kRowBlock && ii + 2 < nseq && y + 3 < p.h + p.x_off_h)
          for (int a = 0; a < 3; ++a) vpx::tma_prefetch_5d(&xmap, 0, -1, y + 3 + p.x_off_h, z - 1 + a + p.x_off_d, n);
        // the x ring slot of row y+1 last served u row i-2; a reset reloads all
        // three rows per depth tap, so u row i-1 must be done
        if (reset && i >= 1) vpx::mbar_wait_sleep(&rowdone[(i - 1) & 1], ((i - 1) >> 1) & 1);
        else if (i >= 2) vpx::mbar_wait_sleep(&rowdone[i & 1], ((i - 2) >> 1) & 1);
        const int nrow = reset ? 3 : 1;
        vpx::mbar_arrive_expect_tx(&xfull[i & 1], 3 * nrow * Cfg::XCH * 128);
#pragma unroll 1
        for (int a = 0; a < 3; ++a) {
          for (int j = 0; j < nrow; ++j) {
            const int yy = reset ? y - 1 + j : y + 1;
            vpx::tma_load_5d(xs + (a * 4 + (yy & 3)) * XROW, &xmap, &xfull[i & 1], 0, -1, yy + p.x_off_h,
                             z - 1 + a + p.x_off_d, n);
          }
        }
      }
    }
  } else if (warp == 3) {
    // ------------------------------------- y / pooled-gradient rows (2 stages)
    if (p.dbg < 4 && vpx::elect_one()) {
      for (long long ii = 0; ii < nseq; ++ii) {
        const int i = static_cast<int>(ii);
        long long t = row_of(ii);
        const int y = t % p.h;
        t /= p.h;
        const int z = t % p.d;
        const int n = static_cast<int>(t / p.d);
        vpx::mbar_wait_sleep(&yempty[i & 1], ((i >> 1) & 1) ^ 1);
        vpx::mbar_arrive_expect_tx(&yfull[i & 1], Cfg::YB + Cfg::UB);
        if (MASK)
          vpx::tma_load_5d(ys + (i & 1) * Cfg::YB, &ymap, &yfull[i & 1], 0, y, z, n, 0);
        else
          vpx::tma_load_5d(ys + (i & 1) * Cfg::YB, &ymap, &yfull[i & 1], 0, 0, y + p.y_off_h, z + p.y_off_d, n);
        if (SRC != 2)
          vpx::tma_load_5d(us + (i & 1) * Cfg::UB, &upmap, &yfull[i & 1], 0, 0, (y >> 1) + p.up_off_h,
                           (z >> 1) + p.up_off_d, n);
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA
    // The issue loop must stay well under the ~25 cycles an N=48 MMA takes:
    // descriptors are built once per row and advanced by one add per K-step,
    // the K-step loop is fully unrolled (KS is a compile-time constant).
    constexpr uint32_t idesc = vpx::make_idesc(2, 128, kNA, false, true);
    const uint32_t xb = vpx::smem_u32(xs);
    const bool skip_waits = p.dbg >= 4;
    const long long tclk0 = clock64();
    const long long tgl0 = globaltimer_ns();
    if (vpx::elect_one()) {  // one thread issues everything (no per-step warp sync)
      int g = 0;
      for (long long ii = 0; ii < nseq; ++ii) {
        const int i = static_cast<int>(ii);
        const int y = static_cast<int>(row_of(ii) % p.h);
        if (!skip_waits) vpx::mbar_wait(&xfull[i & 1], (i >> 1) & 1);
        uint64_t bd[9];  // B descriptors of the 9 (depth, height) taps at K-step 0
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b)
            bd[a * 3 + b] = vpx::make_sdesc(xb + (a * 4 + ((y - 1 + b) & 3)) * XROW, 128, 512, 1);
#pragma unroll
        for (int s = 0; s < KS; ++s, ++g) {
          const int slot = g & (kASlots - 1);
          if (!skip_waits) vpx::mbar_wait(&fullA[slot], (g >> 3) & 1);
          vpx::tc_fence_after();
          const uint32_t acol = tbase + kACol + slot * 8;
          const uint32_t acc = (i > 0 || s > 0) ? 1u : 0u;
#pragma unroll
          for (int ab = 0; ab < 9; ++ab)  // K-step s starts 8 chunk rows (1024 B) further
            vpx::umma_tf32_ta(tbase + ab * kNA, acol, bd[ab] + static_cast<uint64_t>(s * 64), idesc, acc);
          vpx::umma_commit(&emptyA[slot]);
        }
        vpx::umma_commit(&rowdone[i & 1]);
        if (ii == nseq - 1) vpx::umma_commit(&tfull);
      }
    }
    __syncwarp();
    if (p.dbg && pidx == 0 && lane == 0) {
      vpx::mbar_wait(&tfull, 0);
      const long long c = clock64() - tclk0, ns = globaltimer_ns() - tgl0;
      printf("c1 dbg %d: CTA0 %lld MMAs, %.1f cycles/MMA, %.2f GHz\n", p.dbg, nseq * KS * 9,
             double(c) / double(nseq * KS * 9), double(c) / double(ns));
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------- u producers
    // kProdGroups producer warps per TMEM lane quarter (warps 4..7, 8..11, ...)
    // take K-step slots round robin; each computes its next slot while the
    // previous tcgen05.st drains.  The u math is latency-bound, so more warps
    // in flight is what makes it keep up with the MMAs (2 -> 4 per quarter:
    // c1 filter gradient 3.16 -> see DESIGN.md).
    const int q = warp & 3, h = (warp - 4) >> 2, m = q * 32 + lane, dd = m >> 4, co = m & 15;
    const uint32_t lane_addr = tbase + (static_cast<uint32_t>(q * 32) << 16) + kACol;
    const float slope = p.slope;
    // sign of the stored activation at u voxel b + 8 kk: from y, or one bit of the mask
    auto pos = [&](uint32_t ya, int kk) -> bool {
      if constexpr (MASK)
        return (vpx::lds_u16(ya + kk * 16) >> co) & 1u;
      else
        return vpx::lds_f32(ya + kk * 512) >= 0.f;
    };
    auto make_u = [&](int s, uint32_t ya0, uint32_t ua0, float (&v)[8]) {
      // u voxel of column kk: 8k + d + 1 with k = 8s + kk - 1  ->  b + 8 kk
      const int b = 64 * s - 7 + dd;
      const uint32_t ya = ya0 + b * (MASK ? 2 : 64), ua = ua0 + (b >> 1) * 64;
      auto val = [&](int kk) -> float {
        if constexpr (SRC == 2) {
          return vpx::lds_f32(ya + kk * 512);  // u as stored (already TF32)
        } else {
          const float gp = vpx::lds_f32(ua + kk * 256) * 0.125f;
          return vpx::tf32_rn(pos(ya, kk) ? gp : slope * gp);
        }
      };
      if (s > 0 && 64 * s + 56 < W) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) v[kk] = val(kk);
      } else {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          v[kk] = 0.f;
          if (static_cast<unsigned>(b + 8 * kk) < static_cast<unsigned>(W)) v[kk] = val(kk);
        }
      }
    };
    for (long long ii = 0; ii < (p.dbg >= 4 ? 0 : nseq); ++ii) {
      const int i = static_cast<int>(ii);
      vpx::mbar_wait_sleep(&yfull[i & 1], (i >> 1) & 1, 64);
      const uint32_t ya0 = vpx::smem_u32(ys + (i & 1) * Cfg::YB) + (MASK ? 0 : co * 4);
      const uint32_t ua0 = vpx::smem_u32(us + (i & 1) * Cfg::UB) + co * 4;
      int s = (h - i * KS) & (kProdGroups - 1);  // first K-step g = i KS + s of this row with g = h mod groups
      float v[8];
      if (s < KS) {
        if (p.dbg) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) v[kk] = 0.f;
        } else {
          make_u(s, ya0, ua0, v);
        }
      }
#pragma unroll 1
      for (; s < KS; s += kProdGroups) {
        const int g = i * KS + s, slot = g & (kASlots - 1);
        vpx::mbar_wait_sleep(&emptyA[slot], ((g >> 3) & 1) ^ 1);
        if (p.dbg != 2) vpx::tmem_st8(lane_addr + slot * 8, v);
        if (s + kProdGroups < KS && !p.dbg) make_u(s + kProdGroups, ya0, ua0, v);  // overlaps the store
        if (p.dbg != 2) vpx::tmem_st_wait();
        vpx::tc_fence_before();
        __syncwarp();
        if (lane == 0) vpx::mbar_arrive(&fullA[slot]);
      }
      __syncwarp();
      if (lane == 0) vpx::mbar_arrive(&yempty[i & 1]);
    }
  }

  // ---------------------------------------------------------------- epilogue
  const bool have = nseq > 0;
  if (warp >= 4 && warp < 8 && have) {
    vpx::mbar_wait_sleep(&tfull, 0, 256);
    vpx::tc_fence_after();
  }
  __syncthreads();  // all TMA landed and consumed, all MMAs retired: reuse the x ring
  float* red = reinterpret_cast<float*>(smem);  // [d][co][ci][27]
  if (warp >= 4 && warp < 8) {
    const int q = warp - 4, m = q * 32 + lane, dd = m >> 4;
#pragma unroll 1
    for (int ab = 0; ab < 9; ++ab) {
      float v[kNA];
      if (have) {
#pragma unroll
        for (int c16 = 0; c16 < kNA / 16; ++c16) {
          float t16[16];
          vpx::tmem_ld16(tbase + (static_cast<uint32_t>(q * 32) << 16) + ab * kNA + 16 * c16, t16);
#pragma unroll
          for (int j = 0; j < 16; ++j) v[16 * c16 + j] = t16[j];
        }
      } else {
#pragma unroll
        for (int j = 0; j < kNA; ++j) v[j] = 0.f;
      }
      // x voxel offset t = e (+8 for chunk k+1) = d + c; compile-time column
      // indices keep v[] in registers
#pragma unroll
      for (int t = 0; t < 10; ++t) {
        const int c = t - dd;
        if (c >= 0 && c <= 2) {
#pragma unroll
          for (int ci = 0; ci < 4; ++ci) red[(m * 4 + ci) * 27 + ab * 3 + c] = v[(t >> 3) * 32 + (t & 7) * 4 + ci];
        }
      }
    }
  }
  __syncthreads();
  float* base = p.part + static_cast<long long>(pidx) * 16 * 4 * 27;
  for (int o = threadIdx.x; o < 16 * 4 * 27; o += blockDim.x) {
    const int co = o / 108, rem = o % 108;
    float s = 0.f;
#pragma unroll
    for (int dd = 0; dd < 8; ++dd) s += red[(dd * 16 + co) * 108 + rem];
    base[o] = s;
  }
  vpx::tc_fence_before();
  __syncthreads();
  if (warp == 2) vpx::tmem_dealloc<512>(tbase);
}

template <int W, int SRC>
int launch_c1(const CUtensorMap& xm, const CUtensorMap& ym, const CUtensorMap& um, const C1Params& p,
              cudaStream_t st) {
  constexpr int smem = C1Cfg<W, SRC>::SMEM + 1024;
  static_assert(smem <= 227 * 1024, "smem");
  auto kern = c1_pooled_wgrad_kernel<W, SRC>;
  VPX_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  kern<<<p.P, 128 + 32 * kProdWarps, smem, st>>>(xm, ym, um, p);
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}

}  // namespace

namespace vpx {

int c1_pooled_supported(const Frame& xf, const Frame& yf, const Frame& uf) {
  if (precision() != 0) return 0;
  if (xf.c != 4 || yf.c != 16 || uf.c != 16) return 0;
  if (xf.mw || yf.mw || uf.mw) return 0;
  if (!(yf.w == 64 || yf.w == 128 || yf.w == 256 || yf.w == 512)) return 0;
  if (xf.n != yf.n || xf.d != yf.d || xf.h != yf.h || xf.w != yf.w) return 0;
  if (yf.d % 2 || yf.h % 2 || uf.n != yf.n || uf.d * 2 != yf.d || uf.h * 2 != yf.h || uf.w * 2 != yf.w) return 0;
  return 1;
}

// c1 filter gradient from a materialised u (conv 4 -> 16, stride 1, TF32)
int c1_direct_supported(const Frame& xf, const Frame& uf) {
  if (precision() != 0 || xf.c != 4 || uf.c != 16 || xf.mw || uf.md || uf.mh || uf.mw) return 0;
  if (!(uf.w == 64 || uf.w == 128 || uf.w == 256 || uf.w == 512)) return 0;
  return xf.n == uf.n && xf.d == uf.d && xf.h == uf.h && xf.w == uf.w;
}

int c1_pooled_parts(const Frame& yf) {
  const long long rows = (long long)yf.n * yf.d * yf.h;
  long long P = getenv("VPX_C1_P") ? atoi(getenv("VPX_C1_P")) : num_sms();
  if (P > rows) P = rows;
  return static_cast<int>(P < 1 ? 1 : P);
}

int conv_wgrad_c1_pooled(const float* x, const Frame& xf, const float* y, const Frame& yf, const float* up,
                         const Frame& uf, float slope, float* part, cudaStream_t st, const uint16_t* mask,
                         bool u_direct) {
  C1Params p{};
  p.n = yf.n;
  p.d = yf.d;
  p.h = yf.h;
  p.rows = (long long)yf.n * yf.d * yf.h;
  p.P = c1_pooled_parts(yf);
  p.x_off_d = xf.md;
  p.x_off_h = xf.mh;
  p.y_off_d = yf.md;
  p.y_off_h = yf.mh;
  p.up_off_d = uf.md;
  p.up_off_h = uf.mh;
  p.slope = slope;
  p.dbg = getenv("VPX_C1_DEBUG") ? atoi(getenv("VPX_C1_DEBUG")) : 0;
  p.part = part;
  const int W = yf.w;
  int xch = 0;
  switch (W) {
    case 512: xch = C1Cfg<512, 0>::XCH; break;
    case 256: xch = C1Cfg<256, 0>::XCH; break;
    case 128: xch = C1Cfg<128, 0>::XCH; break;
    case 64: xch = C1Cfg<64, 0>::XCH; break;
  }
  CUtensorMap xm, ym, um;
  {
    const uint64_t Hf = xf.h + 2 * xf.mh, Df = xf.d + 2 * xf.md;
    uint64_t dims[5] = {32, (uint64_t)W / 8, Hf, Df, (uint64_t)xf.n};
    uint64_t strides[4] = {128, (uint64_t)W * 16, Hf * W * 16, Df * Hf * W * 16};
    uint32_t box[5] = {32, (uint32_t)xch, 1, 1, 1};
    if (int rc = encode_tiled(&xm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(x), dims, strides, box,
                              CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B))
      return rc;
  }
  if (mask) {
    // [n][d][h][w] 16-bit signs viewed as 32-bit pairs: one row per box
    uint64_t dims[5] = {(uint64_t)W / 2, (uint64_t)yf.h, (uint64_t)yf.d, (uint64_t)yf.n, 1};
    uint64_t strides[4] = {(uint64_t)W * 2, (uint64_t)yf.h * W * 2, (uint64_t)yf.d * yf.h * W * 2,
                           (uint64_t)yf.n * yf.d * yf.h * W * 2};
    uint32_t box[5] = {(uint32_t)(W / 2), 1, 1, 1, 1};
    if (int rc = encode_tiled(&ym, CU_TENSOR_MAP_DATA_TYPE_UINT32, 5, const_cast<uint16_t*>(mask), dims, strides,
                              box, CU_TENSOR_MAP_SWIZZLE_NONE))
      return rc;
  } else {
    const uint64_t Hf = yf.h + 2 * yf.mh, Df = yf.d + 2 * yf.md;
    uint64_t dims[5] = {64, (uint64_t)W / 4, Hf, Df, (uint64_t)yf.n};
    uint64_t strides[4] = {256, (uint64_t)W * 64, Hf * W * 64, Df * Hf * W * 64};
    uint32_t box[5] = {64, (uint32_t)(W / 4), 1, 1, 1};
    if (int rc = encode_tiled(&ym, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(y), dims, strides, box,
                              CU_TENSOR_MAP_SWIZZLE_NONE))
      return rc;
  }
  if (u_direct) {
    um = ym;  // unused
  } else {
    const uint64_t Wu = uf.w, Hf = uf.h + 2 * uf.mh, Df = uf.d + 2 * uf.md;
    uint64_t dims[5] = {64, Wu / 4, Hf, Df, (uint64_t)uf.n};
    uint64_t strides[4] = {256, Wu * 64, Hf * Wu * 64, Df * Hf * Wu * 64};
    uint32_t box[5] = {64, (uint32_t)(Wu / 4), 1, 1, 1};
    if (int rc = encode_tiled(&um, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(up), dims, strides, box,
                              CU_TENSOR_MAP_SWIZZLE_NONE))
      return rc;
  }
  if (u_direct) {
    switch (W) {
      case 512: return launch_c1<512, 2>(xm, ym, um, p, st);
      case 256: return launch_c1<256, 2>(xm, ym, um, p, st);
      case 128: return launch_c1<128, 2>(xm, ym, um, p, st);
      case 64: return launch_c1<64, 2>(xm, ym, um, p, st);
    }
  }
  if (mask) {
    switch (W) {
      case 512: return launch_c1<512, 1>(xm, ym, um, p, st);
      case 256: return launch_c1<256, 1>(xm, ym, um, p, st);
      case 128: return launch_c1<128, 1>(xm, ym, um, p, st);
      case 64: return launch_c1<64, 1>(xm, ym, um, p, st);
    }
  }
  switch (W) {
    case 512: return launch_c1<512, 0>(xm, ym, um, p, st);
    case 256: return launch_c1<256, 0>(xm, ym, um, p, st);
    case 128: return launch_c1<128, 0>(xm, ym, um, p, st);
    case 64: return launch_c1<64, 0>(xm, ym, um, p, st);
  }
  VPX_FAIL(VPX_ERR_UNSUPPORTED, "c1 pooled filter gradient: W=%d", W);
}

}  // namespace vpx

