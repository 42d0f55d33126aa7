// Forward of the first CosmoFlow block (Conv3d 4 -> 16, LeakyReLU, 2^3 average
// pool) in ONE kernel: the 16-channel full-resolution activation never reaches
// HBM.  The kernel writes only
//   * the pooled output  p[n][z/2][y/2][x/2][co] = sum of the 8 stored (TF32
//     rounded) activations / 8, in exactly the order vpx_pool_fwd sums them,
//   * a sign mask  m[n][z][y][x] (16 bits, bit co set when the stored
//     activation is >= 0) -- all the LeakyReLU backward needs (slope > 0).
// That is 2.1 GB of input + 1.34 GB of output per 512^3 sample instead of
// 2.1 + 8.6 (conv) + 8.6 + 1.07 (pool) GB.
//
// The convolution is the height-taps-in-N scheme of conv_rowh.cu (N = 3 x 16,
// output rows summed from three TMEM blocks).  A task is (sample, depth pair,
// band of RB rows, 128-voxel W segment): the band is computed for depth z0,
// whose row-and-width pooled partial sums stay in shared memory, then for
// depth z0+1, which finishes the pooled values.  The 8 epilogue warps split
// the 16 channels in two halves (one set of four warps per TMEM lane quarter
// layout), so every pooling step stays inside one thread and its lane pair.
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
  const float* wpack;        // rowh B layout (vpx::rowh_pack, cin 4, cout 16)
  float slope;
  float* pout;               // pooled frame storage
  long long p_sn, p_sd, p_sh, p_sw;
  int p_off_d, p_off_h, p_off_w;
  int rnd;
  uint16_t* mask;            // [n][d][h][w]
};

constexpr int kWin = 130;
constexpr int kPlane = (3 * kWin * 16 + 127) / 128 * 128;
constexpr int kN = 48;           // 3 height taps x 16 channels
constexpr int kNB = 8;           // E-block ring (8 x 48 TMEM columns)
constexpr int kKSteps = 5;       // (a, c) tap pairs, 4 input channels
constexpr int kBStep = 2 * kN * 16;
constexpr int kWBytes = kKSteps * kBStep;
constexpr int kRB = 32;          // band height (even)
constexpr int kS = 8;            // input-row stages
constexpr int kPoolBuf = (kRB / 2) * 64 * 16 * 4;  // pooled partials of one band (64 KB)
constexpr int kSmem = (kWBytes + 1023) / 1024 * 1024 + kS * kPlane + kPoolBuf + 1024;

__global__ void __launch_bounds__(384, 1)
    c1_fwd_pool_kernel(const __grid_constant__ CUtensorMap xmap, const C1FwdParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sw = smem;
  uint8_t* sa = smem + (kWBytes + 1023) / 1024 * 1024;
  float* pbuf = reinterpret_cast<float*>(sa + kS * kPlane);
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
  }
  if (warp == 2) vpx::tmem_alloc<512>(&tmem_base);
  // The last K step pairs tap (2,2) with a zero-weight phantom tap whose A rows
  // start one voxel later: voxel 127 reads 16 bytes past the 130-voxel window,
  // into the stage padding TMA never writes.  Zero it once so stale shared
  // memory (possibly NaN bit patterns) cannot turn 0 * x into NaN.
  for (int i = threadIdx.x; i < kS * (kPlane - 3 * kWin * 16) / 4; i += blockDim.x) {
    constexpr int kPadWords = (kPlane - 3 * kWin * 16) / 4;
    reinterpret_cast<uint32_t*>(sa + (i / kPadWords) * kPlane + 3 * kWin * 16)[i % kPadWords] = 0u;
  }
  vpx::fence_proxy_async_smem();
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
        for (int pz = 0; pz < 2; ++pz)
          for (int j = 0; j < rows + 2; ++j) {
            vpx::mbar_wait_sleep(&empty[stage], phase ^ 1, 20);
            vpx::mbar_arrive_expect_tx(&full[stage], 3 * kWin * 16);
            vpx::tma_load_5d(sa + stage * kPlane, &xmap, &full[stage], 0, x0 - 1 + p.x_off_w,
                             y0 - 1 + j + p.x_off_h, z0 + pz - 1 + p.x_off_d, n);
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
      int stage = 0;
      uint32_t phase = 0;
      uint32_t gr = 0;
      for (int task = blockIdx.x; task < p.num_tasks; task += gridDim.x) {
        int n, z0, x0, y0, rows;
        decode(task, n, z0, x0, y0, rows);
        for (int pz = 0; pz < 2; ++pz)
          for (int j = 0; j < rows + 2; ++j, ++gr) {
            const int slot = static_cast<int>(gr & (kNB - 1));
            vpx::mbar_wait_sleep(&bempty[slot], ((gr / kNB) & 1) ^ 1, 20);
            vpx::mbar_wait(&full[stage], phase);
            vpx::tc_fence_after();
            const uint32_t d = tbase + slot * kN;
            const uint32_t ab = ab0 + stage * kPlane;
#pragma unroll
            for (int q = 0; q < kKSteps; ++q) {
              const int t0 = 2 * q, t1 = q < 4 ? 2 * q + 1 : 2 * q;  // (a, c) taps t = 3a + c
              const uint32_t lbo = ((t1 / 3 - t0 / 3) * kWin + (t1 % 3 - t0 % 3)) * 16;
              const uint64_t adesc = vpx::make_sdesc(ab + ((t0 / 3) * kWin + t0 % 3) * 16, q < 4 ? lbo : 16, 128, 0);
              const uint64_t bdesc = vpx::make_sdesc(wb + q * kBStep, kN * 16, 128, 0);
              vpx::umma_tf32(d, adesc, bdesc, idesc, q > 0 ? 1u : 0u);
            }
            vpx::umma_commit(&empty[stage]);
            vpx::umma_commit(&bfull[slot]);
            if (++stage == kS) {
              stage = 0;
              phase ^= 1;
            }
          }
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    // Row pairs (y, y+1) per iteration; 32-bit bookkeeping, pointers advanced
    // incrementally (the per-row overhead, not the math, used to dominate).
    const int q = warp & 3;                // TMEM lane quarter: voxels 32q .. 32q+31
    const int ch = ((warp - 4) >> 2) * 8;  // this set's 8 channels
    const uint32_t lane_base = tbase + (static_cast<uint32_t>(q * 32) << 16) + ch;
    const float slope = p.slope;
    const bool rnd = p.rnd != 0;
    const bool even = (lane & 1) == 0;
    uint32_t gr = 0;
    // one output row: sum of the three E slices -> leaky -> TF32 -> sign bits
    auto row = [&](uint32_t g, float (&v)[8]) -> uint32_t {
      uint32_t a0[8], a1[8], a2[8];
      vpx::tmem_ld8_nw(lane_base + (g & (kNB - 1)) * kN + 0 * 16, a0);
      vpx::tmem_ld8_nw(lane_base + ((g + 1) & (kNB - 1)) * kN + 1 * 16, a1);
      vpx::tmem_ld8_nw(lane_base + ((g + 2) & (kNB - 1)) * kN + 2 * 16, a2);
      vpx::tmem_ld_wait();
      uint32_t bits = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float s = (__uint_as_float(a0[i]) + __uint_as_float(a1[i])) + __uint_as_float(a2[i]);
        s = fmaxf(s, slope * s);  // LeakyReLU, 0 < slope <= 1 (reference layers/reference.py:231-233)
        if (rnd) s = vpx::tf32_rn(s);
        v[i] = s;
        bits |= (s >= 0.f ? 1u : 0u) << i;
      }
      return bits;
    };
    auto wait_full = [&](uint32_t g) { vpx::mbar_wait(&bfull[g & (kNB - 1)], (g / kNB) & 1); };
    for (int task = blockIdx.x; task < p.num_tasks; task += gridDim.x) {
      int n, z0, x0, y0, rows;
      decode(task, n, z0, x0, y0, rows);
      const int x = x0 + q * 32 + lane;
      float* dst = p.pout + static_cast<long long>(n) * p.p_sn + static_cast<long long>((z0 >> 1) + p.p_off_d) * p.p_sd +
                   static_cast<long long>((y0 >> 1) + p.p_off_h) * p.p_sh +
                   static_cast<long long>((x >> 1) + p.p_off_w) * p.p_sw + ch;
      for (int pz = 0; pz < 2; ++pz) {
        uint8_t* mrow = reinterpret_cast<uint8_t*>(p.mask) +
                        ((((long long)n * p.d + z0 + pz) * p.h + y0) * p.w + x) * 2 + (ch >> 3);
        const long long mstep = static_cast<long long>(p.w) * 2;
        float* pb = pbuf + ((q * 16 + (lane >> 1)) * 16 + ch);
        float* dp = dst;
        wait_full(gr);
        wait_full(gr + 1);
        for (int k = 0; k < rows; k += 2, mrow += 2 * mstep, pb += 64 * 16, dp += p.p_sh) {
          const uint32_t g = gr + k;
          float v0[8], v1[8];
          wait_full(g + 2);
          vpx::tc_fence_after();
          const uint32_t b0 = row(g, v0);
          wait_full(g + 3);
          vpx::tc_fence_after();
          const uint32_t b1 = row(g + 1, v1);
          // E_{y-1}, E_y are not needed by later rows of this pass
          vpx::tc_fence_before();
          vpx::mbar_arrive(&bempty[g & (kNB - 1)]);
          vpx::mbar_arrive(&bempty[(g + 1) & (kNB - 1)]);
          if (k + 2 >= rows) {
            vpx::mbar_arrive(&bempty[(g + 2) & (kNB - 1)]);
            vpx::mbar_arrive(&bempty[(g + 3) & (kNB - 1)]);
          }
          mrow[0] = static_cast<uint8_t>(b0);
          mrow[mstep] = static_cast<uint8_t>(b1);
          // vpx_pool_fwd sums the window as (z,y,x) (z,y,x+1) (z,y+1,x) (z,y+1,x+1),
          // then the same four at z+1, sequentially; the even lane of each x
          // pair owns the pooled voxel and keeps that exact order
          float n0[8], n1[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            n0[i] = __shfl_down_sync(0xffffffffu, v0[i], 1);
            n1[i] = __shfl_down_sync(0xffffffffu, v1[i], 1);
          }
          if (even) {
            if (pz == 0) {
              float4* pb4 = reinterpret_cast<float4*>(pb);
#pragma unroll
              for (int i = 0; i < 2; ++i)
                pb4[i] = make_float4(((v0[4 * i] + n0[4 * i]) + v1[4 * i]) + n1[4 * i],
                                     ((v0[4 * i + 1] + n0[4 * i + 1]) + v1[4 * i + 1]) + n1[4 * i + 1],
                                     ((v0[4 * i + 2] + n0[4 * i + 2]) + v1[4 * i + 2]) + n1[4 * i + 2],
                                     ((v0[4 * i + 3] + n0[4 * i + 3]) + v1[4 * i + 3]) + n1[4 * i + 3]);
            } else {
              float fin[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                float t = pb[i];
                t = t + v0[i];
                t = t + n0[i];
                t = t + v1[i];
                t = t + n1[i];
                t = t / 8.0f;
                fin[i] = rnd ? vpx::tf32_rn(t) : t;
              }
              reinterpret_cast<float4*>(dp)[0] = make_float4(fin[0], fin[1], fin[2], fin[3]);
              reinterpret_cast<float4*>(dp)[1] = make_float4(fin[4], fin[5], fin[6], fin[7]);
            }
          }
        }
        gr += rows + 2;
      }
    }
  }
  vpx::tc_fence_before();
  __syncthreads();
  if (warp == 2) vpx::tmem_dealloc<512>(tbase);
}

}  // namespace

namespace vpx {

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
  p.zpairs = xf.d / 2;
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
  CUtensorMap map;
  {
    const uint64_t Wf2 = xf.w + 2 * xf.mw, Hf2 = xf.h + 2 * xf.mh, Df2 = xf.d + 2 * xf.md;
    uint64_t dims[5] = {4, Wf2, Hf2, Df2, (uint64_t)xf.n};
    uint64_t strides[4] = {16, Wf2 * 16, Hf2 * Wf2 * 16, Df2 * Hf2 * Wf2 * 16};
    uint32_t box[5] = {4, 130, 1, 3, 1};
    if (int rc = encode_tiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(x), dims, strides, box,
                              CU_TENSOR_MAP_SWIZZLE_NONE))
      return rc;
  }
  VPX_CHECK_CUDA(cudaFuncSetAttribute(c1_fwd_pool_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
  const int grid = p.num_tasks < num_sms() ? p.num_tasks : num_sms();
  c1_fwd_pool_kernel<<<grid, 384, kSmem, st>>>(map, p);
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}

}  // namespace vpx
