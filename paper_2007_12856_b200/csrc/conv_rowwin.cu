// Implicit-GEMM 3x3x3 convolution on tcgen05 for rows of 128 output voxels
// ("row-window" kernel).  Used for the forward pass and, with flipped and
// transposed weights, for backward-data (stride-1 layers).
//
// Work unit (tile): R consecutive output rows y0..y0+R-1 at depth z of sample
// n, W-segment x0..x0+127.  Each output row is one UMMA M=128 accumulator of
// COUT fp32 columns in TMEM.  The input window for the tile -- 3 depth planes x
// (R+2) rows x 130 voxels x 4 channels per 16-byte chunk -- lands in shared
// memory by TMA (out-of-bounds taps read as zero = "same" padding at the walls,
// frame margins hold neighbour halos).  Because a window row is stored at a
// 16-byte voxel pitch, the A operand for tap (a,b,c) of row r is the same
// window addressed from a shifted start: no im2col copy.  The K dimension
// runs over (tap, channel chunk pair); for Cin=4 two taps share one K=8 step.
//
// Warp roles (256 threads): w0 TMA producer, w1 MMA issuer, w2 TMEM owner,
// w4..w7 epilogue (TMEM -> registers -> global NDHWC fp32).  Persistent CTAs,
// S-stage smem ring, double-buffered accumulators.
//
// Reference semantics: reference pkg/src/voxpar/kernels/_hot.pyx:19-41 (fwd),
// :44-67 (bwd_data as the adjoint scatter; here computed as a gather conv).
#include "conv_common.h"
#include "vpx_host.h"
#include "vpx_ptx.cuh"
#include "vpx_round.cuh"

namespace {

using vpx::ConvRowParams;

constexpr int kWin = 130;  // 128 outputs + 2 halo voxels along W

template <int R>
__host__ __device__ constexpr int plane_raw() {
  return 3 * (R + 2) * kWin * 16;
}
template <int R>
__host__ __device__ constexpr int plane_bytes() {
  return (plane_raw<R>() + 127) / 128 * 128;
}
// non-pair instances: 8-channel planes stored as 32-byte voxel rows in the
// K-major SWIZZLE_32B layout (one TMA box per plane instead of two 16-byte ones)
template <int R>
__host__ __device__ constexpr int plane8_bytes() {
  return (2 * plane_raw<R>() + 1023) / 1024 * 1024;
}
template <int COUT, int CG, bool PAIR>
__host__ __device__ constexpr int b_bytes() {
  return (PAIR ? 28 : 27 * CG) * COUT * 16;
}
template <int COUT, int R, int CG, bool PAIR>
__host__ __device__ constexpr int stage_bytes() {
  return ((PAIR ? CG * plane_bytes<R>() : (CG / 2) * plane8_bytes<R>()) + b_bytes<COUT, CG, PAIR>() + 1023) /
         1024 * 1024;
}
__host__ __device__ constexpr int pow2_cols(int c) {
  return c <= 32 ? 32 : c <= 64 ? 64 : c <= 128 ? 128 : c <= 256 ? 256 : 512;
}

// Epilogue staging for coalesced stores (COUT <= 32): 4 warps x 32 voxels x
// (COUT + 4) floats, padded so the per-lane 16-byte stores are conflict free.
template <int COUT>
__host__ __device__ constexpr int epi_bytes() {
  return COUT <= 32 ? 4 * 32 * (COUT + 4) * 4 : 0;
}

template <int COUT, int R, int CG, bool PAIR, int S>
__global__ void __launch_bounds__(256, 1)
    conv_rowwin_kernel(const __grid_constant__ CUtensorMap xmap, const ConvRowParams p) {
  constexpr bool kStaged = epi_bytes<COUT>() > 0;
  constexpr int PLANE = PAIR ? plane_bytes<R>() : plane8_bytes<R>();
  constexpr int ABYTES = PAIR ? CG * PLANE : (CG / 2) * PLANE;
  constexpr int BBYTES = b_bytes<COUT, CG, PAIR>();
  constexpr int STAGE = stage_bytes<COUT, R, CG, PAIR>();
  constexpr int ACC = R * COUT;
  constexpr int TCOLS = pow2_cols(2 * ACC);
  constexpr uint32_t TX = CG * plane_raw<R>() + BBYTES;
  static_assert(2 * ACC <= 512, "accumulators exceed TMEM");

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[S], empty[S], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      vpx::mbar_init(&full[s], 1);
      vpx::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      vpx::mbar_init(&tfull[s], 1);
      vpx::mbar_init(&tempty[s], 128);
    }
    vpx::fence_barrier_init();
    vpx::tma_prefetch_desc(&xmap);
  }
  if (warp == 2) vpx::tmem_alloc<TCOLS>(&tmem_base);
  vpx::tc_fence_before();
  __syncthreads();
  vpx::tc_fence_after();
  const uint32_t tbase = tmem_base;

  const int nz = p.zhi - p.zlo;
  const int ngroups = p.n_groups;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (vpx::elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
        int t = tile;
        const int xs = t % p.nxseg;
        t /= p.nxseg;
        const int yg = t % p.ngy;
        t /= p.ngy;
        const int z = p.zlo + t % nz;
        const int n = t / nz;
        const int x0 = xs * 128, y0 = p.ylo + yg * R;
        for (int g = 0; g < ngroups; ++g) {
          vpx::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sA = smem + stage * STAGE;
          vpx::mbar_arrive_expect_tx(&full[stage], TX);
          if constexpr (PAIR) {
#pragma unroll
            for (int c = 0; c < CG; ++c)
              vpx::tma_load_5d(sA + c * PLANE, &xmap, &full[stage], 4 * (g * CG + c), x0 - 1 + p.in_off_w,
                               y0 - 1 + p.in_off_h, z - 1 + p.in_off_d, n);
          } else {
#pragma unroll
            for (int c = 0; c < CG / 2; ++c)
              vpx::tma_load_5d(sA + c * PLANE, &xmap, &full[stage], 4 * (g * CG + 2 * c), x0 - 1 + p.in_off_w,
                               y0 - 1 + p.in_off_h, z - 1 + p.in_off_d, n);
          }
          vpx::bulk_g2s(sA + ABYTES, p.wpack + static_cast<size_t>(g) * (BBYTES / 4), BBYTES,
                        &full[stage]);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = vpx::make_idesc(2, 128, COUT, false, false);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t aphase = 0;
    for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
      vpx::mbar_wait(&tempty[acc], aphase ^ 1);
      vpx::tc_fence_after();
      const uint32_t dacc = tbase + acc * ACC;
      for (int g = 0; g < ngroups; ++g) {
        vpx::mbar_wait(&full[stage], phase);
        vpx::tc_fence_after();
        if (vpx::elect_one()) {
          const uint32_t aBase = vpx::smem_u32(smem + stage * STAGE);
          const uint32_t bBase = aBase + ABYTES;
          if constexpr (PAIR) {
#pragma unroll 1
            for (int q = 0; q < 14; ++q) {
              const int t0 = 2 * q;
              const int a0 = t0 / 9, b0 = (t0 / 3) % 3, c0 = t0 % 3;
              int lbo = 16;
              if (q < 13) {
                const int t1 = t0 + 1;
                const int a1 = t1 / 9, b1 = (t1 / 3) % 3, c1 = t1 % 3;
                lbo = (((a1 - a0) * (R + 2) + (b1 - b0)) * kWin + (c1 - c0)) * 16;
              }
              const uint64_t bdesc = vpx::make_sdesc(bBase + q * 2 * COUT * 16, COUT * 16, 128, 0);
#pragma unroll
              for (int r = 0; r < R; ++r) {
                const uint32_t as = aBase + ((a0 * (R + 2) + r + b0) * kWin + c0) * 16;
                vpx::umma_tf32(dacc + r * COUT, vpx::make_sdesc(as, lbo, 128, 0), bdesc, idesc,
                               (g | q) != 0);
              }
            }
          } else {
            // fully unrolled: every descriptor is the stage's base descriptor
            // plus a compile-time offset in the 16-byte address field (one add)
            // -- rebuilding them per MMA kept the single issuing thread behind
            // the N = 32 / 64 MMAs
            const uint64_t a0desc = vpx::make_sdesc(aBase, 16, 256, 6);
            const uint64_t b0desc = vpx::make_sdesc(bBase, COUT * 16, 128, 0);
#pragma unroll
            for (int t = 0; t < 27; ++t) {
              const int a = t / 9, b = (t / 3) % 3, c = t % 3;
#pragma unroll
              for (int jp = 0; jp < CG / 2; ++jp) {
                const uint64_t bdesc = b0desc + (t * CG + 2 * jp) * COUT;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                  // 8-channel plane jp, voxel row (a, r+b, c): 32-byte SW32 rows, 8-row atoms
                  const uint64_t adesc = a0desc + (jp * PLANE + ((a * (R + 2) + r + b) * kWin + c) * 32) / 16;
                  vpx::umma_tf32(dacc + r * COUT, adesc, bdesc, idesc, (g | t | jp) != 0);
                }
              }
            }
          }
          vpx::umma_commit(&empty[stage]);
          if (g == ngroups - 1) vpx::umma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
      acc ^= 1;
      if (acc == 0) aphase ^= 1;
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const int q = warp - 4;  // TMEM lane quarter
    float* stg = reinterpret_cast<float*>(smem + S * STAGE) + q * 32 * (COUT + 4);
    int acc = 0;
    uint32_t aphase = 0;
    for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
      int t = tile;
      const int xs = t % p.nxseg;
      t /= p.nxseg;
      const int yg = t % p.ngy;
      t /= p.ngy;
      const int z = p.zlo + t % nz;
      const int n = t / nz;
      const int x = xs * 128 + q * 32 + lane;
      const int y0 = p.ylo + yg * R;
      vpx::mbar_wait(&tfull[acc], aphase);
      vpx::tc_fence_after();
      float* orow = p.out + static_cast<long long>(n) * p.out_sn +
                    static_cast<long long>(z + p.out_off_d) * p.out_sd +
                    static_cast<long long>(x + p.out_off_w) * p.out_sw;
      // warp's first voxel of the row segment (for the coalesced write-out)
      float* orow_w = orow - static_cast<long long>(lane) * p.out_sw;
#pragma unroll 1
      for (int r = 0; r < R; ++r) {
        const int y = y0 + r;
        float* o = orow + static_cast<long long>(y + p.out_off_h) * p.out_sh;
#pragma unroll
        for (int cb = 0; cb < COUT / 16; ++cb) {
          float v[16];
          vpx::tmem_ld16(tbase + (static_cast<uint32_t>(q * 32) << 16) + acc * ACC + r * COUT + cb * 16, v);
          if (p.act) {  // fused LeakyReLU (reference layers/reference.py:231-233)
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = v[i] >= 0.f ? v[i] : p.slope * v[i];
          }
          if (p.rnd) {
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = vpx::tf32_rn(v[i]);
          }
          if constexpr (kStaged) {
            // this lane's voxel row -> padded smem (conflict-free 16-byte stores)
            float4* s4 = reinterpret_cast<float4*>(stg + lane * (COUT + 4) + cb * 16);
#pragma unroll
            for (int i = 0; i < 4; ++i) s4[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
          } else if (y < p.yhi) {
            float4* o4 = reinterpret_cast<float4*>(o + cb * 16);
#pragma unroll
            for (int i = 0; i < 4; ++i) o4[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
          }
        }
        if constexpr (kStaged) {
          // 32 voxels x COUT channels are contiguous in global memory: write
          // them out as consecutive 16-byte chunks (fully coalesced)
          __syncwarp();
          if (y < p.yhi) {
            float* ow = orow_w + static_cast<long long>(y + p.out_off_h) * p.out_sh;
            constexpr int Q = COUT / 4;  // float4 chunks per voxel
#pragma unroll
            for (int k = 0; k < Q; ++k) {
              const int c = k * 32 + lane, vx = c / Q, qq = c % Q;
              const float4 val = *reinterpret_cast<const float4*>(stg + vx * (COUT + 4) + qq * 4);
              *reinterpret_cast<float4*>(ow + static_cast<long long>(vx) * p.out_sw + qq * 4) = val;
            }
          }
          __syncwarp();
        }
      }
      vpx::tc_fence_before();
      vpx::mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) aphase ^= 1;
    }
  }
  vpx::tc_fence_before();
  __syncthreads();
  if (warp == 2) vpx::tmem_dealloc<TCOLS>(tbase);
}

template <int COUT, int R, int CG, bool PAIR>
int launch_rowwin(const CUtensorMap& xmap, const ConvRowParams& p, cudaStream_t st) {
  constexpr int STAGE = stage_bytes<COUT, R, CG, PAIR>();
  constexpr int BUDGET = 226 * 1024 - epi_bytes<COUT>();
  constexpr int S = (BUDGET - 1024) / STAGE >= 4 ? 4 : (BUDGET - 1024) / STAGE;
  static_assert(S >= 2, "stage too large");
  constexpr int SMEM = S * STAGE + epi_bytes<COUT>() + 1024;
  auto kern = conv_rowwin_kernel<COUT, R, CG, PAIR, S>;
  VPX_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
  int grid = p.num_tiles < vpx::num_sms() ? p.num_tiles : vpx::num_sms();
  if (grid <= 0) return VPX_OK;
  kern<<<grid, 256, SMEM, st>>>(xmap, p);
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}

}  // namespace

namespace vpx {

// Pick the (R, CG) instance for a channel configuration; 0 if unsupported.
int rowwin_config(int cin, int cout, int* R, int* CG) {
  if (cin == 4 && cout == 16) { *R = 8; *CG = 1; return 1; }
  if (cin == 16 && cout == 32) { *R = 4; *CG = 2; return 1; }
  if (cin == 32 && cout == 16) { *R = 4; *CG = 2; return 1; }   // c2 dgrad
  if (cin == 32 && cout == 64) { *R = 2; *CG = 2; return 1; }
  if (cin == 64 && cout == 32) { *R = 4; *CG = 2; return 1; }   // c3 dgrad
  if (cin == 16 && cout == 16) { *R = 4; *CG = 2; return 1; }
  if (cin == 8 && cout == 16) { *R = 4; *CG = 2; return 1; }
  if (cin == 16 && cout == 8) { return 0; }
  return 0;
}

int launch_rowwin_any(const CUtensorMap& xmap, const ConvRowParams& p, int cin, int cout,
                      cudaStream_t st) {
  if (cin == 4 && cout == 16) return launch_rowwin<16, 8, 1, true>(xmap, p, st);
  if (cin == 16 && cout == 32) return launch_rowwin<32, 4, 2, false>(xmap, p, st);
  if (cin == 32 && cout == 16) return launch_rowwin<16, 4, 2, false>(xmap, p, st);
  if (cin == 32 && cout == 64) return launch_rowwin<64, 2, 2, false>(xmap, p, st);
  if (cin == 64 && cout == 32) return launch_rowwin<32, 4, 2, false>(xmap, p, st);
  if (cin == 16 && cout == 16) return launch_rowwin<16, 4, 2, false>(xmap, p, st);
  if (cin == 8 && cout == 16) return launch_rowwin<16, 4, 2, false>(xmap, p, st);
  VPX_FAIL(VPX_ERR_UNSUPPORTED, "row-window conv: no instance for cin=%d cout=%d", cin, cout);
}

}  // namespace vpx
