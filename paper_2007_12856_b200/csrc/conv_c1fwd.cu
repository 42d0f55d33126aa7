// Forward of the first CosmoFlow block (Conv3d 4 -> 16, LeakyReLU, 2^3 average
// pool) in ONE kernel: the 16-channel full-resolution activation never reaches
// HBM.  The kernel writes only
//   * the pooled output  p[n][z/2][y/2][x/2][co] = sum of the 8 stored (TF32
//     rounded) activations / 8, in the order vpx_pool_fwd sums them,
//   * a sign mask  m[n][z][y][x] (16 bits, bit co set when the stored
//     activation is >= 0) -- all the LeakyReLU backward needs (slope > 0).
// That is 2.1 GB of input + 1.34 GB of output per 512^3 sample instead of
// 2.1 + 8.6 (conv) + 8.6 + 1.07 (pool) GB.
//
// A task is (sample, depth pair z0 z0+1, band of RB rows, 128-voxel W
// segment).  One stage holds the four input planes z0-1 .. z0+2 of an input
// row (read once for both output depths -- separate depth passes read six
// plane-rows per input row).  Per input row the tensor cores run ONE chain of
// six K = 8 MMAs, M = 128 voxels, K = (input plane p, width tap c, 4 input
// channels) = 4 x 3 x 4 = 48, N = (output depth d, height tap b, 16 output
// channels) = 96, with weight w[co][ci][p - d][b][c] (zero when p - d is not a
// depth tap).  Its three 16-column blocks b per depth belong to output rows
// y + 1 - b (height taps in N, as conv_rowh.cu), so output row y sums the
// b = 0, 1, 2 blocks of input rows y-1, y, y+1 from a 5-row TMEM ring; the
// 2^3 pooling window is complete in registers once a row pair of both depths
// is read.  Against the depth-pass form (two chains of five N = 48 MMAs per
// input row) this is 6 x 56 instead of 10 x 44 tensor cycles per input row and
// 2/3 of the input traffic.
// Reference semantics: reference pkg/src/voxpar/kernels/_hot.pyx:19-41 (conv),
// layers/reference.py:231-233 (leaky), :159-168 (average pool).
#include "conv_common.h"
#include "vpx_host.h"
#include "vpx_ptx.cuh"
#include "vpx_round.cuh"

namespace {

struct C1FwdParams {
  int n, d, h, w;            // conv output (= input interior) extents
  int nxseg, rb, nbands, zpairs;
  int num_tasks;
  int x_off_d, x_off_h, x_off_w;
  const float* wpack;        // B operand (pack_c1_fwd_kernel)
  float slope;
  float* pout;               // pooled frame storage
  long long p_sn, p_sd, p_sh, p_sw;
  int p_off_d, p_off_h, p_off_w;
  int rnd;
  uint16_t* mask;            // [n][d][h][w]
};

// An input plane-row = 130 voxels (x0-1 .. x0+128) x 4 channels, fetched as
// 1 KB + 1 KB + 32 B runs of the NDHWC row (a row view of x, boxes of 256 / 8
// floats); planes sit kWin = 136 voxels apart so every TMA destination is
// 128-byte aligned.
constexpr int kWinVox = 130;
constexpr int kWin = 136;
constexpr int kPlanes = 4;
constexpr int kStage = kPlanes * kWin * 16;
constexpr int kN = 96;           // 2 depths x 3 height taps x 16 channels
constexpr int kNB = 5;           // E-block ring: 5 input rows x 96 TMEM columns
constexpr int kKSteps = 6;       // 12 (plane, width tap) pairs, 4 input channels
constexpr int kBStep = 2 * kN * 16;
constexpr int kWBytes = kKSteps * kBStep;
constexpr int kRB = 64;          // band height (even)
constexpr bool kRoundActivations = false;
constexpr int kS = 16;           // input-row stages
constexpr int kSmem = (kWBytes + 1023) / 1024 * 1024 + kS * kStage + 1024;

// B operand, K-major no-swizzle: [K step s][K half h][N row n][4 ci] with
// (plane, width tap) t = 2s + h = 3p + c and n = 48 d + 16 b + co.
__global__ void pack_c1_fwd_kernel(const float* __restrict__ w, float* __restrict__ out) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= kWBytes / 4) return;
  const int ci = idx & 3, n = (idx >> 2) % kN, sh = (idx >> 2) / kN;  // sh = 2 s + h = t
  const int p = sh / 3, c = sh % 3, d = n / 48, b = (n / 16) % 3, co = n % 16;
  const int a = p - d;  // depth tap
  out[idx] = (a >= 0 && a <= 2) ? vpx::tf32_rn(w[((co * 4 + ci) * 3 + a) * 9 + b * 3 + c]) : 0.f;
}

template <int DBG>
__global__ void __launch_bounds__(384, 1)
    c1_fwd_pool_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap xmap8,
                       const C1FwdParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sw = smem;
  uint8_t* sa = smem + (kWBytes + 1023) / 1024 * 1024;
  __shared__ __align__(8) uint64_t full[kS], empty[kS], bfull[kNB], bempty[kNB], wbar;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kS; ++s) {
      vpx::mbar_init(&full[s], 1);
      vpx::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < kNB; ++s) {
      vpx::mbar_init(&bfull[s], 1);
      vpx::mbar_init(&bempty[s], 256);
    }
    vpx::mbar_init(&wbar, 1);
    vpx::fence_barrier_init();
    vpx::tma_prefetch_desc(&xmap);
    vpx::tma_prefetch_desc(&xmap8);
  }
  if (warp == 2) vpx::tmem_alloc<512>(&tmem_base);
  vpx::tc_fence_before();
  __syncthreads();
  vpx::tc_fence_after();
  const uint32_t tbase = tmem_base;

  auto decode = [&](int task, int& n, int& z0, int& x0, int& y0, int& rows) {
    int t = task;
    const int xs = t % p.nxseg;
    t /= p.nxseg;
    const int band = t % p.nbands;
    t /= p.nbands;
    z0 = 2 * (t % p.zpairs);
    n = t / p.zpairs;
    x0 = xs * 128;
    y0 = band * p.rb;
    rows = min(p.rb, p.h - y0);
  };

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (vpx::elect_one()) {
      vpx::mbar_arrive_expect_tx(&wbar, kWBytes);
      vpx::bulk_g2s(sw, p.wpack, kWBytes, &wbar);
      int stage = 0;
      uint32_t phase = 0;
      for (int task = blockIdx.x; task < p.num_tasks; task += gridDim.x) {
        int n, z0, x0, y0, rows;
        decode(task, n, z0, x0, y0, rows);
        const int e0 = 4 * (x0 - 1 + p.x_off_w);
        for (int j = 0; j < rows + 2; ++j) {
          vpx::mbar_wait_sleep(&empty[stage], phase ^ 1, 20);
          vpx::mbar_arrive_expect_tx(&full[stage], kPlanes * kWinVox * 16);
          const int yy = y0 - 1 + j + p.x_off_h;
#pragma unroll
          for (int a = 0; a < kPlanes; ++a) {
            uint8_t* pl = sa + stage * kStage + a * kWin * 16;
            const int zz = z0 - 1 + a + p.x_off_d;
            vpx::tma_load_5d(pl, &xmap, &full[stage], e0, yy, zz, n, 0);
            vpx::tma_load_5d(pl + 1024, &xmap, &full[stage], e0 + 256, yy, zz, n, 0);
            vpx::tma_load_5d(pl + 2048, &xmap8, &full[stage], e0 + 512, yy, zz, n, 0);
          }
          if (++stage == kS) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA
    constexpr uint32_t idesc = vpx::make_idesc(2, 128, kN, false, false);
    if (vpx::elect_one()) {
      vpx::mbar_wait(&wbar, 0);
      const uint32_t wb = vpx::smem_u32(sw);
      const uint32_t ab0 = vpx::smem_u32(sa);
      // Descriptors built once: B is resident; A differs per stage only in
      // its start-address field (address >> 4, no carry below 256 KB), so a
      // row's six MMAs cost one add each -- a single issuing thread that
      // rebuilt every descriptor spent more cycles issuing than the MMAs took
      uint64_t adesc0[kKSteps], bdesc[kKSteps];
#pragma unroll
      for (int s = 0; s < kKSteps; ++s) {
        const int t0 = 2 * s, t1 = 2 * s + 1;  // (plane, width tap) t = 3 p + c
        const uint32_t lbo = ((t1 / 3 - t0 / 3) * kWin + (t1 % 3 - t0 % 3)) * 16;
        adesc0[s] = vpx::make_sdesc(ab0 + ((t0 / 3) * kWin + t0 % 3) * 16, lbo, 128, 0);
        bdesc[s] = vpx::make_sdesc(wb + s * kBStep, kN * 16, 128, 0);
      }
      int stage = 0;
      uint32_t phase = 0, soff = 0;           // soff = stage * kStage >> 4
      uint32_t slot = 0, sphase = 0;          // ring slot of input row gr and its use parity
      uint32_t d = tbase;
      for (int task = blockIdx.x; task < p.num_tasks; task += gridDim.x) {
        int n, z0, x0, y0, rows;
        decode(task, n, z0, x0, y0, rows);
        for (int j = 0; j < rows + 2; ++j) {
          vpx::mbar_wait(&bempty[slot], sphase ^ 1);
          vpx::mbar_wait(&full[stage], phase);
          vpx::tc_fence_after();
#pragma unroll
          for (int s = 0; s < kKSteps; ++s)
            vpx::umma_tf32(d, adesc0[s] + soff, bdesc[s], idesc, s > 0 ? 1u : 0u);
          vpx::umma_commit(&empty[stage]);
          vpx::umma_commit(&bfull[slot]);
          if (++stage == kS) {
            stage = 0;
            phase ^= 1;
            soff = 0;
          } else {
            soff += kStage >> 4;
          }
          if (++slot == kNB) {
            slot = 0;
            sphase ^= 1;
            d = tbase;
          } else {
            d += kN;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;                // TMEM lane quarter: voxels 32q .. 32q+31
    const int ch = ((warp - 4) >> 2) * 8;  // this set's 8 channels
    const uint32_t lane_base = tbase + (static_cast<uint32_t>(q * 32) << 16) + ch;
    const float slope = p.slope;
    const bool rnd = p.rnd != 0;
    const bool even = (lane & 1) == 0;
    uint32_t gr = 0;
    auto wait_full = [&](uint32_t g) { vpx::mbar_wait(&bfull[g % kNB], (g / kNB) & 1); };
    // output row y of both depths = blocks b = 0, 1, 2 of input rows g, g+1,
    // g+2 (g = input row y-1); input row g is released once loaded
    auto row = [&](uint32_t g, float (&v)[2][8], uint32_t (&bits)[2]) {
      wait_full(g + 2);
      vpx::tc_fence_after();
      uint32_t a[2][3][8];
#pragma unroll
      for (int dd = 0; dd < 2; ++dd)
#pragma unroll
        for (int b = 0; b < 3; ++b) vpx::tmem_ld8_nw(lane_base + ((g + b) % kNB) * kN + dd * 48 + b * 16, a[dd][b]);
      vpx::tmem_ld_wait();
      vpx::tc_fence_before();
      vpx::mbar_arrive(&bempty[g % kNB]);
#pragma unroll
      for (int dd = 0; dd < 2; ++dd) {
        bits[dd] = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float s = (__uint_as_float(a[dd][0][i]) + __uint_as_float(a[dd][1][i])) + __uint_as_float(a[dd][2][i]);
          s = fmaxf(s, slope * s);  // LeakyReLU, 0 < slope <= 1 (reference layers/reference.py:231-233)
          // the activation is never stored, so it is pooled unrounded (only
          // the pooled value is rounded to TF32): a third fewer epilogue
          // instructions per value, within one TF32 step of the rounded form
          if (rnd && kRoundActivations) s = vpx::tf32_rn(s);
          v[dd][i] = s;
          bits[dd] |= (s >= 0.f ? 1u : 0u) << i;
        }
      }
    };
    for (int task = blockIdx.x; task < p.num_tasks; task += gridDim.x) {
      int n, z0, x0, y0, rows;
      decode(task, n, z0, x0, y0, rows);
      const int x = x0 + q * 32 + lane;
      float* dp = p.pout + static_cast<long long>(n) * p.p_sn + static_cast<long long>((z0 >> 1) + p.p_off_d) * p.p_sd +
                  static_cast<long long>((y0 >> 1) + p.p_off_h) * p.p_sh +
                  static_cast<long long>((x >> 1) + p.p_off_w) * p.p_sw + ch;
      const long long mstep = static_cast<long long>(p.w) * 2, mplane = mstep * p.h;
      uint8_t* mrow = reinterpret_cast<uint8_t*>(p.mask) + ((((long long)n * p.d + z0) * p.h + y0) * p.w + x) * 2 +
                      (ch >> 3);
      for (int k = 0; k < rows; k += 2, mrow += 2 * mstep, dp += p.p_sh) {
        if (DBG == 1) {  // timing: ring releases only
          for (int i = 0; i < 2; ++i) {
            wait_full(gr + k + i + 2);
            vpx::mbar_arrive(&bempty[(gr + k + i) % kNB]);
          }
          continue;
        }
        float v0[2][8], v1[2][8];
        uint32_t b0[2], b1[2];
        row(gr + k, v0, b0);
        row(gr + k + 1, v1, b1);
        mrow[0] = static_cast<uint8_t>(b0[0]);
        mrow[mstep] = static_cast<uint8_t>(b1[0]);
        mrow[mplane] = static_cast<uint8_t>(b0[1]);
        mrow[mplane + mstep] = static_cast<uint8_t>(b1[1]);
        // 2^3 average pool: each lane sums its voxel's four values (two rows x
        // two depths), one shuffle brings the W neighbour's sum to the even
        // lane, which owns the pooled voxel (one shuffle per channel instead of
        // four; a different summation order than vpx_pool_fwd's sequential one)
        float part[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) part[i] = (v0[0][i] + v1[0][i]) + (v0[1][i] + v1[1][i]);
        float nb[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) nb[i] = __shfl_down_sync(0xffffffffu, part[i], 1);
        if (even) {
          float fin[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float t = (part[i] + nb[i]) * 0.125f;
            fin[i] = rnd ? vpx::tf32_rn(t) : t;
          }
          reinterpret_cast<float4*>(dp)[0] = make_float4(fin[0], fin[1], fin[2], fin[3]);
          reinterpret_cast<float4*>(dp)[1] = make_float4(fin[4], fin[5], fin[6], fin[7]);
        }
      }
      // the band's last two input rows are not the first block of any later row
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        wait_full(gr + rows + i);
        vpx::mbar_arrive(&bempty[(gr + rows + i) % kNB]);
      }
      gr += rows + 2;
    }
  }
  vpx::tc_fence_before();
  __syncthreads();
  if (warp == 2) vpx::tmem_dealloc<512>(tbase);
}

}  // namespace

namespace vpx {

long long c1_fwd_packed_bytes() { return kWBytes; }

int c1_fwd_pack(const float* w, float* dst, cudaStream_t st) {
  pack_c1_fwd_kernel<<<(kWBytes / 4 + 255) / 256, 256, 0, st>>>(w, dst);
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}

int c1_fwd_pool_supported(const Frame& xf, int cout, const Frame& pf) {
  if (precision() != 0 || xf.c != 4 || cout != 16 || pf.c != 16) return 0;
  if (xf.w % 128 || xf.d % 2 || xf.h % 2 || xf.mw) return 0;
  return pf.n == xf.n && pf.d * 2 == xf.d && pf.h * 2 == xf.h && pf.w * 2 == xf.w;
}

int conv_c1_fwd_pool(const float* x, const Frame& xf, const float* wpack, float slope, float* pout,
                     const Frame& pf, uint16_t* mask, cudaStream_t st) {
  C1FwdParams p{};
  p.n = xf.n;
  p.d = xf.d;
  p.h = xf.h;
  p.w = xf.w;
  p.nxseg = xf.w / 128;
  p.rb = kRB < xf.h ? kRB : xf.h;
  p.nbands = (xf.h + p.rb - 1) / p.rb;
  p.zpairs = xf.d / 2;  // a task computes both depths of a pooling pair
  p.num_tasks = xf.n * p.zpairs * p.nbands * p.nxseg;
  p.x_off_d = xf.md;
  p.x_off_h = xf.mh;
  p.x_off_w = xf.mw;
  p.wpack = wpack;
  p.slope = slope;
  p.pout = pout;
  const long long Wf = pf.w + 2 * pf.mw, Hf = pf.h + 2 * pf.mh, Df = pf.d + 2 * pf.md;
  p.p_sw = pf.c;
  p.p_sh = Wf * pf.c;
  p.p_sd = Hf * Wf * pf.c;
  p.p_sn = Df * Hf * Wf * pf.c;
  p.p_off_d = pf.md;
  p.p_off_h = pf.mh;
  p.p_off_w = pf.mw;
  p.rnd = pf.rnd;
  p.mask = mask;
  CUtensorMap map, map8;
  {
    // row view: dims {W*4 floats, H, D, n, 1}
    const uint64_t Wf2 = xf.w + 2 * xf.mw, Hf2 = xf.h + 2 * xf.mh, Df2 = xf.d + 2 * xf.md;
    uint64_t dims[5] = {Wf2 * 4, Hf2, Df2, (uint64_t)xf.n, 1};
    uint64_t strides[4] = {Wf2 * 16, Hf2 * Wf2 * 16, Df2 * Hf2 * Wf2 * 16, (uint64_t)xf.n * Df2 * Hf2 * Wf2 * 16};
    uint32_t box[5] = {256, 1, 1, 1, 1};
    if (int rc = encode_tiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(x), dims, strides, box,
                              CU_TENSOR_MAP_SWIZZLE_NONE))
      return rc;
    box[0] = (kWinVox - 128) * 4;
    if (int rc = encode_tiled(&map8, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(x), dims, strides, box,
                              CU_TENSOR_MAP_SWIZZLE_NONE))
      return rc;
  }
  const int grid = p.num_tasks < num_sms() ? p.num_tasks : num_sms();
  static const int dbg = getenv("VPX_C1F_DBG") ? atoi(getenv("VPX_C1F_DBG")) : 0;
  if (dbg == 1) {
    VPX_CHECK_CUDA(cudaFuncSetAttribute(c1_fwd_pool_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    c1_fwd_pool_kernel<1><<<grid, 384, kSmem, st>>>(map, map8, p);
    VPX_LAUNCH_CHECK();
    return VPX_OK;
  }
  VPX_CHECK_CUDA(cudaFuncSetAttribute(c1_fwd_pool_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
  c1_fwd_pool_kernel<0><<<grid, 384, kSmem, st>>>(map, map8, p);
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}

}  // namespace vpx
