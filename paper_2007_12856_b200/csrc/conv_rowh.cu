// Implicit-GEMM 3x3x3 convolution on tcgen05 for narrow outputs (16/32
// channels): the three height taps go into the MMA's N dimension.
//
// The row-window kernel (conv_rowwin.cu) issues one M=128 x N=COUT MMA per
// tap; with COUT = 16/32 every MMA still reads the whole 4 KB A tile from
// shared memory, so it runs at the A-read rate (~40 cycles) for a small N.
// Here the input row r is the unit of work: for each (depth tap a, width tap
// c, channel chunk) ONE MMA multiplies the 128-voxel window of row r by the
// weights of all three height taps at once,
//     E_r[v][(b, co)] = sum_{a,c,ci} x[z+a-1][r][v+c-1][ci] * w[co][ci][a][b][c]
// (N = 3*COUT), and output row y is assembled by the epilogue from three
// consecutive input rows:  out[y] = E_{y-1}[b=0] + E_y[b=1] + E_{y+1}[b=2].
// The E blocks live in a 4-slot TMEM ring (3 read by the epilogue while the
// MMA fills the 4th).  Work unit: a band of RB output rows at (n, z, 128-voxel
// W segment), i.e. RB+2 input rows.  All weights stay resident in shared
// memory (<= 55 KB); the input rows stream through an S-stage TMA ring in the
// same 16-byte-voxel-pitch layout as the row-window kernel (no im2col: every
// width tap is the same window at a shifted start address).
//
// Warp roles (384 threads): w0 TMA producer, w1 MMA issuer (one elected
// thread), w2 TMEM owner, w4..w11 epilogue in two sets of four (one per TMEM
// lane quarter) taking alternate output rows: 3 TMEM slices -> sum ->
// optional LeakyReLU -> TF32 rounding -> coalesced NDHWC stores through
// padded smem.  (With 16 output channels a row is only 5 MMAs, so the
// epilogue, not the tensor pipe, sets the pace unless it is doubled.)
// Reference semantics: reference pkg/src/voxpar/kernels/_hot.pyx:19-41 (fwd),
// :44-67 (bwd_data, computed as a gather conv with flipped/transposed weights).
#include "conv_common.h"
#include "vpx_host.h"
#include "vpx_ptx.cuh"
#include "vpx_round.cuh"

namespace {

using vpx::ConvRowParams;

constexpr int kWinH = 130;                             // 128 outputs + 2 halo voxels
constexpr int kPlane = (3 * kWinH * 16 + 127) / 128 * 128;  // 3 depth planes x 130 voxels x 16 B

template <int CIN, int C>
struct RowH {
  static constexpr bool PAIR = CIN == 4;                 // two (a,c) taps per K=8 step
  static constexpr int NCH = CIN / 4;                    // 4-channel chunk planes per input row (PAIR)
  // CIN >= 8: the window is stored as whole voxel rows (CIN*4 bytes) in the
  // matching K-major swizzle (one wide TMA box; a width tap is a row shift)
  static constexpr int RB = CIN * 4;
  static constexpr uint32_t LAYOUT = RB == 128 ? 2 : RB == 64 ? 4 : 6;  // SW128 / SW64 / SW32
  static constexpr int KSTEPS = PAIR ? 5 : 9 * (CIN / 8);
  static constexpr int N = (3 * C + 15) / 16 * 16;        // 3 height taps x C, padded to a multiple of 16
  static constexpr int BSTEP = 2 * N * 16;               // bytes of B per K step
  static constexpr int WBYTES = KSTEPS * BSTEP;
  static constexpr int STAGE = PAIR ? NCH * kPlane : (3 * kWinH * RB + 1023) / 1024 * 1024;
  static constexpr int EPI = 8 * 32 * (C + 4) * 4;       // 8 epilogue warps
  static constexpr int S0 = (226 * 1024 - 2048 - WBYTES - EPI) / STAGE;
  static constexpr int S = S0 > 8 ? 8 : S0;
  static constexpr int SMEM = (WBYTES + 1023) / 1024 * 1024 + S * STAGE + EPI + 1024;
  static constexpr int NB = 512 / N >= 8 ? 8 : 4;       // TMEM ring of E blocks (power of 2)
  static constexpr int TCOLS = NB * N <= 256 ? 256 : 512;
};

template <int CIN, int C>
__global__ void __launch_bounds__(384, 1)
    conv_rowh_kernel(const __grid_constant__ CUtensorMap xmap, const ConvRowParams p) {
  using K = RowH<CIN, C>;
  constexpr int N = K::N, S = K::S, kNB = K::NB;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sw = smem;                                                   // resident weights
  uint8_t* sa = smem + (K::WBYTES + 1023) / 1024 * 1024;                // input-row stages
  float* sepi = reinterpret_cast<float*>(sa + S * K::STAGE);            // epilogue staging
  __shared__ __align__(8) uint64_t full[S], empty[S], bfull[kNB], bempty[kNB], wbar;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rb = p.ngy;  // rows per band (ConvRowParams reuse: ngy = band height)
  const int nbands = (p.yhi - p.ylo + rb - 1) / rb;
  const int nz = p.zhi - p.zlo;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      vpx::mbar_init(&full[s], 1);
      vpx::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < kNB; ++s) {
      vpx::mbar_init(&bfull[s], 1);
      vpx::mbar_init(&bempty[s], 128);
    }
    vpx::mbar_init(&wbar, 1);
    vpx::fence_barrier_init();
    vpx::tma_prefetch_desc(&xmap);
  }
  if (warp == 2) vpx::tmem_alloc<K::TCOLS>(&tmem_base);
  if constexpr (K::PAIR) {
    // the (2,2) + phantom-tap K step reads 16 bytes past each 130-voxel plane
    // (zero weights); keep that never-loaded padding finite (see conv_c1fwd.cu)
    constexpr int kPadWords = (kPlane - 3 * kWinH * 16) / 4;
    for (int i = threadIdx.x; i < S * K::NCH * kPadWords; i += blockDim.x)
      reinterpret_cast<uint32_t*>(sa + (i / kPadWords) * kPlane + 3 * kWinH * 16)[i % kPadWords] = 0u;
    vpx::fence_proxy_async_smem();
  }
  vpx::tc_fence_before();
  __syncthreads();
  vpx::tc_fence_after();
  const uint32_t tbase = tmem_base;

  auto decode = [&](int task, int& n, int& z, int& x0, int& y0, int& rows) {
    int t = task;
    const int xs = t % p.nxseg;
    t /= p.nxseg;
    const int band = t % nbands;
    t /= nbands;
    z = p.zlo + t % nz;
    n = t / nz;
    x0 = xs * 128;
    y0 = p.ylo + band * rb;
    rows = min(rb, p.yhi - y0);
  };

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (vpx::elect_one()) {
      vpx::mbar_arrive_expect_tx(&wbar, K::WBYTES);
      vpx::bulk_g2s(sw, p.wpack, K::WBYTES, &wbar);
      int stage = 0;
      uint32_t phase = 0;
      for (int task = blockIdx.x; task < p.num_tiles; task += gridDim.x) {
        int n, z, x0, y0, rows;
        decode(task, n, z, x0, y0, rows);
        for (int j = 0; j < rows + 2; ++j) {
          const int r = y0 - 1 + j;
          vpx::mbar_wait_sleep(&empty[stage], phase ^ 1, 20);
          uint8_t* dst = sa + stage * K::STAGE;
          vpx::mbar_arrive_expect_tx(&full[stage], 3 * kWinH * CIN * 4);
          if constexpr (K::PAIR) {
            vpx::tma_load_5d(dst, &xmap, &full[stage], 0, x0 - 1 + p.in_off_w, r + p.in_off_h, z - 1 + p.in_off_d,
                             n);
          } else {
            vpx::tma_load_5d(dst, &xmap, &full[stage], 0, x0 - 1 + p.in_off_w, r + p.in_off_h, z - 1 + p.in_off_d,
                             n);
          }
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA
    constexpr uint32_t idesc = vpx::make_idesc(2, 128, N, false, false);
    if (vpx::elect_one()) {
      vpx::mbar_wait(&wbar, 0);
      const uint32_t wb = vpx::smem_u32(sw);
      const uint32_t ab0 = vpx::smem_u32(sa);
      const uint64_t bbase = vpx::make_sdesc(wb, N * 16, 128, 0);
      int stage = 0;
      uint32_t phase = 0;
      uint32_t gr = 0;  // E blocks produced by this CTA
      for (int task = blockIdx.x; task < p.num_tiles; task += gridDim.x) {
        int n, z, x0, y0, rows;
        decode(task, n, z, x0, y0, rows);
        for (int j = 0; j < rows + 2; ++j, ++gr) {
          const int slot = static_cast<int>(gr & (kNB - 1));
          vpx::mbar_wait_sleep(&bempty[slot], ((gr / kNB) & 1) ^ 1, 20);
          vpx::mbar_wait(&full[stage], phase);
          vpx::tc_fence_after();
          const uint32_t d = tbase + slot * N;
          const uint32_t ab = ab0 + stage * K::STAGE;
          if constexpr (K::PAIR) {
#pragma unroll
            for (int q = 0; q < 5; ++q) {
              const int t0 = 2 * q, t1 = q < 4 ? 2 * q + 1 : 2 * q;  // (a, c) taps, t = 3a + c
              const uint32_t lbo = ((t1 / 3 - t0 / 3) * kWinH + (t1 % 3 - t0 % 3)) * 16;
              const uint64_t adesc = vpx::make_sdesc(ab + ((t0 / 3) * kWinH + t0 % 3) * 16, q < 4 ? lbo : 16, 128, 0);
              const uint64_t bdesc = vpx::make_sdesc(wb + q * K::BSTEP, N * 16, 128, 0);
              vpx::umma_tf32(d, adesc, bdesc, idesc, q > 0 ? 1u : 0u);
            }
          } else {
            // descriptors = a per-row base + a compile-time offset in the
            // 16-byte address field (no carry below 256 KB): one add per
            // operand instead of rebuilding both for each of the 9 x CIN/8
            // MMAs -- the single issuing thread is otherwise slower than the
            // N = 48 MMAs it feeds
            const uint64_t arow = vpx::make_sdesc(ab, 16, 8 * K::RB, K::LAYOUT);
#pragma unroll
            for (int t = 0; t < 9; ++t) {
#pragma unroll
              for (int jp = 0; jp < CIN / 8; ++jp) {
                // row (plane a, voxel c) of the swizzled window, K step jp = 8 channels (32 B)
                const uint64_t adesc = arow + (((t / 3) * kWinH + t % 3) * K::RB + jp * 32) / 16;
                const uint64_t bdesc = bbase + ((t * (CIN / 8) + jp) * K::BSTEP) / 16;
                vpx::umma_tf32(d, adesc, bdesc, idesc, (t | jp) != 0 ? 1u : 0u);
              }
            }
          }
          vpx::umma_commit(&empty[stage]);
          vpx::umma_commit(&bfull[slot]);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;            // TMEM lane quarter = voxels 32q .. 32q+31 of the segment
    const int hset = (warp - 4) >> 2;  // output rows k with k % 2 == hset
    float* stg = sepi + (warp - 4) * 32 * (C + 4);
    const uint32_t lane_base = tbase + (static_cast<uint32_t>(q * 32) << 16);
    const bool act = p.act != 0, rnd = p.rnd != 0;
    const float slope = p.slope;
    uint32_t gr = 0;
    for (int task = blockIdx.x; task < p.num_tiles; task += gridDim.x) {
      int n, z, x0, y0, rows;
      decode(task, n, z, x0, y0, rows);
      // E blocks of this band: gr .. gr + rows + 1 (input rows y0-1 .. y0+rows)
      float* ow = p.out + static_cast<long long>(n) * p.out_sn + static_cast<long long>(z + p.out_off_d) * p.out_sd +
                  static_cast<long long>(x0 + q * 32 + p.out_off_w) * p.out_sw +
                  static_cast<long long>(y0 + hset + p.out_off_h) * p.out_sh;
      const long long ostep = 2 * p.out_sh;
      for (int k = hset; k < rows; k += 2, ow += ostep) {
        const uint32_t gm = gr + k;  // E_{y-1}, E_y, E_{y+1} = gm, gm+1, gm+2
        // none of the three can be recycled before this row frees E_{y-1} and
        // the other set finishes row k+1, so the parity waits are unambiguous
        vpx::mbar_wait(&bfull[gm & (kNB - 1)], (gm / kNB) & 1);
        vpx::mbar_wait(&bfull[(gm + 1) & (kNB - 1)], ((gm + 1) / kNB) & 1);
        vpx::mbar_wait(&bfull[(gm + 2) & (kNB - 1)], ((gm + 2) / kNB) & 1);
        vpx::tc_fence_after();
        const uint32_t s0 = lane_base + (gm & (kNB - 1)) * N, s1 = lane_base + ((gm + 1) & (kNB - 1)) * N + C,
                       s2 = lane_base + ((gm + 2) & (kNB - 1)) * N + 2 * C;
        constexpr int CW = C < 16 ? C : 16;  // TMEM columns per load
#pragma unroll
        for (int cb = 0; cb < C / CW; ++cb) {
          uint32_t v0[CW], v1[CW], v2[CW];  // three loads in flight, one wait
          if constexpr (CW == 16) {
            vpx::tmem_ld16_nw(s0 + cb * 16, v0);
            vpx::tmem_ld16_nw(s1 + cb * 16, v1);
            vpx::tmem_ld16_nw(s2 + cb * 16, v2);
          } else {
            vpx::tmem_ld8_nw(s0, v0);
            vpx::tmem_ld8_nw(s1, v1);
            vpx::tmem_ld8_nw(s2, v2);
          }
          vpx::tmem_ld_wait();
          float v[CW];
#pragma unroll
          for (int i = 0; i < CW; ++i) {
            v[i] = (__uint_as_float(v0[i]) + __uint_as_float(v1[i])) + __uint_as_float(v2[i]);
            if (act) v[i] = v[i] >= 0.f ? v[i] : slope * v[i];  // reference layers/reference.py:231-233
            if (rnd) v[i] = vpx::tf32_rn(v[i]);
          }
          float4* s4 = reinterpret_cast<float4*>(stg + lane * (C + 4) + cb * CW);
#pragma unroll
          for (int i = 0; i < CW / 4; ++i) s4[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        }
        // E_{y-1} is not needed by any later output row of this band; the last
        // row also releases the band's final two blocks
        vpx::tc_fence_before();
        vpx::mbar_arrive(&bempty[gm & (kNB - 1)]);
        if (k == rows - 1) {
          vpx::mbar_arrive(&bempty[(gm + 1) & (kNB - 1)]);
          vpx::mbar_arrive(&bempty[(gm + 2) & (kNB - 1)]);
        }
        __syncwarp();
        constexpr int Q = C / 4;  // float4 chunks per voxel
#pragma unroll
        for (int kk = 0; kk < Q; ++kk) {
          const int c = kk * 32 + lane, vx = c / Q, qq = c % Q;
          const float4 val = *reinterpret_cast<const float4*>(stg + vx * (C + 4) + qq * 4);
          *reinterpret_cast<float4*>(ow + static_cast<long long>(vx) * p.out_sw + qq * 4) = val;
        }
        __syncwarp();
      }
      gr += rows + 2;
    }
  }
  vpx::tc_fence_before();
  __syncthreads();
  if (warp == 2) vpx::tmem_dealloc<K::TCOLS>(tbase);
}

template <int CIN, int C>
int launch_rowh(const CUtensorMap& xmap, const ConvRowParams& p, cudaStream_t st) {
  using K = RowH<CIN, C>;
  static_assert(K::S >= 2, "stages");
  static_assert(K::SMEM <= 227 * 1024, "smem");
  auto kern = conv_rowh_kernel<CIN, C>;
  VPX_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, K::SMEM));
  int grid = p.num_tiles < vpx::num_sms() ? p.num_tiles : vpx::num_sms();
  if (grid <= 0) return VPX_OK;
  kern<<<grid, 384, K::SMEM, st>>>(xmap, p);
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}

// Pack OIDHW weights into the resident B layout:
//   B[kstep][h][n = (b, o)][e]  (K-major, no swizzle: 8 rows x 16 B core matrices,
//   the two 4-channel halves of a K=8 step LBO = N*16 apart)
//   non-pair: kstep = t*(I/8) + jp, t = 3a + c, input channel i = 4(2jp + h) + e
//   pair (I = 4): kstep = q, tap t = 2q + h (t = 9 -> zeros), i = e
//   mode 0: Weff[o][i][a][b][c] = w[o][i][a][b][c]; mode 1: w[i][o][2-a][2-b][2-c]
__global__ void pack_rowh_kernel(const float* __restrict__ w, int cout, int cin, int mode, int pair,
                                 float* __restrict__ out) {
  const int O = mode ? cin : cout, I = mode ? cout : cin;
  const int N = (3 * O + 15) / 16 * 16;  // rows >= 3*O are zero padding
  const int ksteps = pair ? 5 : 9 * (I / 8);
  const long long total = (long long)ksteps * 2 * N * 4;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    long long t = idx;
    const int e = t % 4;
    t /= 4;
    const int nn = t % N;
    t /= N;
    const int h = t % 2;
    const int ks = static_cast<int>(t / 2);
    const int b = nn / O, o = nn % O;
    int tap, i;
    if (pair) {
      tap = 2 * ks + h;
      i = e;
    } else {
      tap = ks / (I / 8);
      i = 4 * (2 * (ks % (I / 8)) + h) + e;
    }
    float v = 0.f;
    if (tap < 9 && b < 3) {
      const int a = tap / 3, c = tap % 3;
      if (mode == 0)
        v = w[(((long long)o * cin + i) * 3 + a) * 9 + b * 3 + c];
      else
        v = w[(((long long)i * cin + o) * 3 + (2 - a)) * 9 + (2 - b) * 3 + (2 - c)];
    }
    out[idx] = vpx::tf32_rn(v);
  }
}


// ---------------------------------------------------------------------------
// conv -> LeakyReLU -> 2^3 average pool fused into the height-taps-in-N
// kernel (the conv_c1fwd.cu scheme for wider layers, e.g. CosmoFlow c2):
// a task is (sample, depth pair, band of RB rows, 128-voxel segment); depth z0
// leaves its row-and-width pooled partials in shared memory, depth z0+1
// finishes them in vpx_pool_fwd's exact summation order.  Only the pooled
// output and a sign mask (cout bits per voxel) reach HBM.  The 8 epilogue
// warps split the channels in two halves; each thread takes output rows in
// pairs (y, y+1), so the pool's row sum and (via a lane shuffle) its width
// sum stay in registers.  The E-block ring needs only 3 + 1 slots per row,
// so it is sized 512 / N (5 for N = 96, not a power of two).
template <int CIN, int C>
struct RowhPoolCfg {
  using K = RowH<CIN, C>;
  static constexpr int NB = 512 / K::N > 8 ? 8 : 512 / K::N;
  static constexpr int RBAND = 16;
  static constexpr int CH = C / 2;                         // channels per epilogue warp set
  static constexpr int PBUF = RBAND / 2 * 64 * C * 4;
  static constexpr int S0 = (226 * 1024 - 2048 - K::WBYTES - PBUF) / K::STAGE;
  static constexpr int S = S0 > 8 ? 8 : S0;
  static constexpr int SMEM = (K::WBYTES + 1023) / 1024 * 1024 + S * K::STAGE + PBUF + 1024;
  static_assert(!K::PAIR && (CH == 8 || CH == 16), "channel split");
};

template <int CIN, int C>
__global__ void __launch_bounds__(384, 1)
    conv_rowh_pool_kernel(const __grid_constant__ CUtensorMap xmap, const vpx::RowhPoolParams p) {
  using K = RowH<CIN, C>;
  using Q = RowhPoolCfg<CIN, C>;
  constexpr int N = K::N, S = Q::S, NB = Q::NB, CH = Q::CH;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sw = smem;
  uint8_t* sa = smem + (K::WBYTES + 1023) / 1024 * 1024;
  float* pbuf = reinterpret_cast<float*>(sa + S * K::STAGE);
  __shared__ __align__(8) uint64_t full[S], empty[S], bfull[NB], bempty[NB], wbar;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      vpx::mbar_init(&full[s], 1);
      vpx::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < NB; ++s) {
      vpx::mbar_init(&bfull[s], 1);
      vpx::mbar_init(&bempty[s], 256);
    }
    vpx::mbar_init(&wbar, 1);
    vpx::fence_barrier_init();
    vpx::tma_prefetch_desc(&xmap);
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
      vpx::mbar_arrive_expect_tx(&wbar, K::WBYTES);
      vpx::bulk_g2s(sw, p.wpack, K::WBYTES, &wbar);
      int stage = 0;
      uint32_t phase = 0;
      for (int task = blockIdx.x; task < p.num_tasks; task += gridDim.x) {
        int n, z0, x0, y0, rows;
        decode(task, n, z0, x0, y0, rows);
        for (int pz = 0; pz < 2; ++pz)
          for (int j = 0; j < rows + 2; ++j) {
            vpx::mbar_wait_sleep(&empty[stage], phase ^ 1, 20);
            vpx::mbar_arrive_expect_tx(&full[stage], 3 * kWinH * CIN * 4);
            vpx::tma_load_5d(sa + stage * K::STAGE, &xmap, &full[stage], 0, x0 - 1 + p.in_off_w,
                             y0 - 1 + j + p.in_off_h, z0 + pz - 1 + p.in_off_d, n);
            if (++stage == S) {
              stage = 0;
              phase ^= 1;
            }
          }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA
    constexpr uint32_t idesc = vpx::make_idesc(2, 128, N, false, false);
    if (vpx::elect_one()) {
      vpx::mbar_wait(&wbar, 0);
      const uint32_t wb = vpx::smem_u32(sw);
      const uint32_t ab0 = vpx::smem_u32(sa);
      const uint64_t bbase = vpx::make_sdesc(wb, N * 16, 128, 0);
      int stage = 0;
      uint32_t phase = 0;
      uint32_t gr = 0;
      for (int task = blockIdx.x; task < p.num_tasks; task += gridDim.x) {
        int n, z0, x0, y0, rows;
        decode(task, n, z0, x0, y0, rows);
        for (int pz = 0; pz < 2; ++pz)
          for (int j = 0; j < rows + 2; ++j, ++gr) {
            const uint32_t slot = gr % NB;
            vpx::mbar_wait_sleep(&bempty[slot], ((gr / NB) & 1) ^ 1, 20);
            vpx::mbar_wait(&full[stage], phase);
            vpx::tc_fence_after();
            const uint32_t d = tbase + slot * N;
            const uint32_t ab = ab0 + stage * K::STAGE;
            const uint64_t arow = vpx::make_sdesc(ab, 16, 8 * K::RB, K::LAYOUT);  // + per-MMA address offsets
#pragma unroll
            for (int t = 0; t < 9; ++t) {
#pragma unroll
              for (int jp = 0; jp < CIN / 8; ++jp) {
                const uint64_t adesc = arow + (((t / 3) * kWinH + t % 3) * K::RB + jp * 32) / 16;
                const uint64_t bdesc = bbase + ((t * (CIN / 8) + jp) * K::BSTEP) / 16;
                vpx::umma_tf32(d, adesc, bdesc, idesc, (t | jp) != 0 ? 1u : 0u);
              }
            }
            vpx::umma_commit(&empty[stage]);
            vpx::umma_commit(&bfull[slot]);
            if (++stage == S) {
              stage = 0;
              phase ^= 1;
            }
          }
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;                // TMEM lane quarter: voxels 32q .. 32q+31
    const int hset = (warp - 4) >> 2;      // channel half
    const int ch0 = hset * CH;
    const uint32_t lane_base = tbase + (static_cast<uint32_t>(q * 32) << 16) + ch0;
    const float slope = p.slope;
    const bool rnd = p.rnd != 0;
    const bool even = (lane & 1) == 0;
    constexpr int MB = C / 8;              // mask bytes per voxel
    uint32_t gr = 0;
    // output row g: sum of three E slices -> leaky -> TF32 -> sign bits
    auto row = [&](uint32_t g, float (&v)[CH]) -> uint32_t {
      uint32_t a0[CH], a1[CH], a2[CH];
      if constexpr (CH == 16) {
        vpx::tmem_ld16_nw(lane_base + (g % NB) * N, a0);
        vpx::tmem_ld16_nw(lane_base + ((g + 1) % NB) * N + C, a1);
        vpx::tmem_ld16_nw(lane_base + ((g + 2) % NB) * N + 2 * C, a2);
      } else {
        vpx::tmem_ld8_nw(lane_base + (g % NB) * N, a0);
        vpx::tmem_ld8_nw(lane_base + ((g + 1) % NB) * N + C, a1);
        vpx::tmem_ld8_nw(lane_base + ((g + 2) % NB) * N + 2 * C, a2);
      }
      vpx::tmem_ld_wait();
      uint32_t bits = 0;
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        float s = (__uint_as_float(a0[i]) + __uint_as_float(a1[i])) + __uint_as_float(a2[i]);
        s = fmaxf(s, slope * s);  // LeakyReLU, 0 < slope <= 1 (reference layers/reference.py:231-233)
        // pooled unrounded (the activation is never stored; the pooled value is rounded)
        v[i] = s;
        bits |= (s >= 0.f ? 1u : 0u) << i;
      }
      return bits;
    };
    auto wait_full = [&](uint32_t g) { vpx::mbar_wait(&bfull[g % NB], (g / NB) & 1); };
    auto release = [&](uint32_t g) { vpx::mbar_arrive(&bempty[g % NB]); };
    for (int task = blockIdx.x; task < p.num_tasks; task += gridDim.x) {
      int n, z0, x0, y0, rows;
      decode(task, n, z0, x0, y0, rows);
      const int x = x0 + q * 32 + lane;
      float* dst = p.pout + static_cast<long long>(n) * p.p_sn +
                   static_cast<long long>((z0 >> 1) + p.p_off_d) * p.p_sd +
                   static_cast<long long>((y0 >> 1) + p.p_off_h) * p.p_sh +
                   static_cast<long long>((x >> 1) + p.p_off_w) * p.p_sw + ch0;
      for (int pz = 0; pz < 2; ++pz) {
        uint8_t* mrow = p.mask + ((((long long)n * p.d + z0 + pz) * p.h + y0) * p.w + x) * MB + hset * (CH / 8);
        const long long mstep = static_cast<long long>(p.w) * MB;
        float* pb = pbuf + ((q * 16 + (lane >> 1)) * C + ch0);
        float* dp = dst;
        for (int k = 0; k < rows; k += 2, mrow += 2 * mstep, pb += 64 * C, dp += p.p_sh) {
          const uint32_t g = gr + k;
          float v0[CH], v1[CH];
          wait_full(g);
          wait_full(g + 1);
          wait_full(g + 2);
          vpx::tc_fence_after();
          const uint32_t b0 = row(g, v0);
          vpx::tc_fence_before();
          release(g);
          wait_full(g + 3);
          vpx::tc_fence_after();
          const uint32_t b1 = row(g + 1, v1);
          vpx::tc_fence_before();
          release(g + 1);
          if (k + 2 >= rows) {
            release(g + 2);
            release(g + 3);
          }
          if constexpr (CH == 16) {
            *reinterpret_cast<uint16_t*>(mrow) = static_cast<uint16_t>(b0);
            *reinterpret_cast<uint16_t*>(mrow + mstep) = static_cast<uint16_t>(b1);
          } else {
            mrow[0] = static_cast<uint8_t>(b0);
            mrow[mstep] = static_cast<uint8_t>(b1);
          }
          // each lane sums its voxel's two rows, one shuffle per channel brings
          // the W neighbour's sum to the even lane (the pooled voxel's owner);
          // depth z0's partial waits in shared memory for depth z0+1
          float part[CH], nb[CH];
#pragma unroll
          for (int i = 0; i < CH; ++i) part[i] = v0[i] + v1[i];
#pragma unroll
          for (int i = 0; i < CH; ++i) nb[i] = __shfl_down_sync(0xffffffffu, part[i], 1);
          if (even) {
            float4* pb4 = reinterpret_cast<float4*>(pb);
            if (pz == 0) {
#pragma unroll
              for (int i = 0; i < CH / 4; ++i)
                pb4[i] = make_float4(part[4 * i] + nb[4 * i], part[4 * i + 1] + nb[4 * i + 1],
                                     part[4 * i + 2] + nb[4 * i + 2], part[4 * i + 3] + nb[4 * i + 3]);
            } else {
#pragma unroll
              for (int i = 0; i < CH / 4; ++i) {
                const float4 pp = pb4[i];
                const float pv[4] = {pp.x, pp.y, pp.z, pp.w};
                float fin[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const float t = (pv[j] + (part[4 * i + j] + nb[4 * i + j])) * 0.125f;
                  fin[j] = rnd ? vpx::tf32_rn(t) : t;
                }
                reinterpret_cast<float4*>(dp)[i] = make_float4(fin[0], fin[1], fin[2], fin[3]);
              }
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

template <int CIN, int C>
int launch_rowh_pool(const CUtensorMap& xmap, const vpx::RowhPoolParams& p, cudaStream_t st) {
  using Q = RowhPoolCfg<CIN, C>;
  static_assert(Q::S >= 3, "stages");
  static_assert(Q::SMEM <= 227 * 1024, "smem");
  auto kern = conv_rowh_pool_kernel<CIN, C>;
  VPX_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Q::SMEM));
  const int grid = p.num_tasks < vpx::num_sms() ? p.num_tasks : vpx::num_sms();
  if (grid <= 0) return VPX_OK;
  kern<<<grid, 384, Q::SMEM, st>>>(xmap, p);
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}
}  // namespace

namespace vpx {

// Channel configurations with a rowh instance (cin_eff -> cout_eff).
int rowh_supported(int cin, int cout) {
  return (cin == 4 && cout == 16) || (cin == 8 && cout == 16) || (cin == 16 && cout == 16) ||
         (cin == 32 && cout == 16) || (cin == 16 && cout == 32) || (cin == 8 && cout == 8) ||
         (cin == 16 && cout == 8) || (cin == 32 && cout == 8);
}

long long rowh_packed_bytes(int cin, int cout) {
  const int ksteps = cin == 4 ? 5 : 9 * (cin / 8);
  return (long long)ksteps * 2 * ((3 * cout + 15) / 16 * 16) * 16;
}

int rowh_pack(const float* w, int cout, int cin, int mode, float* dst, cudaStream_t st) {
  const int I = mode ? cout : cin, O = mode ? cin : cout;
  if (!rowh_supported(I, O)) VPX_FAIL(VPX_ERR_UNSUPPORTED, "rowh pack");
  const long long total = rowh_packed_bytes(I, O) / 4;
  int grid = static_cast<int>((total + 255) / 256);
  if (grid > 4096) grid = 4096;
  pack_rowh_kernel<<<grid, 256, 0, st>>>(w, cout, cin, mode, I == 4, dst);
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}

int launch_rowh_any(const CUtensorMap& xmap, const ConvRowParams& p, int cin, int cout, cudaStream_t st) {
  if (cin == 4 && cout == 16) return launch_rowh<4, 16>(xmap, p, st);
  if (cin == 8 && cout == 16) return launch_rowh<8, 16>(xmap, p, st);
  if (cin == 16 && cout == 16) return launch_rowh<16, 16>(xmap, p, st);
  if (cin == 32 && cout == 16) return launch_rowh<32, 16>(xmap, p, st);
  if (cin == 16 && cout == 32) return launch_rowh<16, 32>(xmap, p, st);
  if (cin == 8 && cout == 8) return launch_rowh<8, 8>(xmap, p, st);
  if (cin == 16 && cout == 8) return launch_rowh<16, 8>(xmap, p, st);
  if (cin == 32 && cout == 8) return launch_rowh<32, 8>(xmap, p, st);
  VPX_FAIL(VPX_ERR_UNSUPPORTED, "rowh conv: no instance for cin=%d cout=%d", cin, cout);
}

int rowh_pool_instance(int cin, int cout) { return (cin == 16 && cout == 32) || (cin == 16 && cout == 16); }

int launch_rowh_pool_any(const CUtensorMap& xmap, const RowhPoolParams& p, int cin, int cout, cudaStream_t st) {
  if (cin == 16 && cout == 32) return launch_rowh_pool<16, 32>(xmap, p, st);
  if (cin == 16 && cout == 16) return launch_rowh_pool<16, 16>(xmap, p, st);
  VPX_FAIL(VPX_ERR_UNSUPPORTED, "fused conv+pool: no instance for cin=%d cout=%d", cin, cout);
}

}  // namespace vpx
