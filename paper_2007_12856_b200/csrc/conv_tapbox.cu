// Implicit-GEMM convolution on tcgen05 for layers whose rows are too short
// for the row-window kernel (W < 128: CosmoFlow c4..c7, U-Net deep levels,
// any W-partitioned grid) and for stride 2.
//
// M tile = a box of 128 output voxels (Wb x Hb x Db, W fastest).  For each
// K entry (tap offset, 32-channel chunk) one TMA box of the input lands in
// shared memory as 128-byte rows (SWIZZLE_128B K-major): the "im2col" is done
// by the TMA unit, out-of-bounds taps read zeros (= "same" padding), frame
// margins supply neighbour halos.  Stride-2 forward uses TMA element strides
// (the box walks every second input voxel).  Stride-2 backward-data is run as
// eight parity classes of output voxels (p = 2q + P); each class is a
// stride-1 gather over u with its own list of taps (ConvTapParams.cls_*).
// B = packed weights [entry][N_total][32] by 2D TMA, N tile <= 256.
// Reference semantics: reference pkg/src/voxpar/kernels/_hot.pyx:19-67.
#include <cuda_bf16.h>

#include <cstdlib>

#include "conv_common.h"
#include <algorithm>

#include "conv_simt.h"
#include "vpx_host.h"
#include "vpx_ptx.cuh"
#include "vpx_round.cuh"

namespace vpx {

constexpr int kMaxEntries = 256;

struct ConvTapParams {
  int n;                        // samples
  int qd, qh, qw;               // q-grid origin offsets: q = q0 + tile coords
  int QD, QH, QW;               // q-grid extents
  int Db, Hb, Wb;               // tile box (Db*Hb*Wb <= 128)
  int td, th, tw;               // tiles per dim
  int ncls;                     // parity classes (1 or 8)
  int ntn;                      // N tiles
  int num_tiles;
  int in_stride;                // 1 or 2 (input coordinate = s*q + off + margin)
  int in_off_d, in_off_h, in_off_w;
  int ntot;                     // total N (rows of each packed weight entry)
  // per K entry: (od+1) | (oh+1)<<2 | (ow+1)<<4 | chunk<<8 | tap<<16
  int entries[kMaxEntries];
  int cls_start[9];             // entry ranges per parity class
  int balance;                  // 1: tiles handed out heaviest class first, serpentine over CTAs
  int cls_order[8];             // balance: classes by descending K entries
  float* out;
  long long out_sn, out_sd, out_sh, out_sw;
  int out_off_d, out_off_h, out_off_w;  // frame margins of the output
  int out_stride;                       // 1 or 2 (p = s*q + P)
  int pd_lo, pd_hi, ph_lo, ph_hi, pw_lo, pw_hi;  // valid output range (interior coords incl. margins)
  int act;
  float slope;
  int rnd;
  int nvalid;                   // output channels actually stored (< NT only for an 8-channel deconv output)
  int dcout;                    // > 0: transposed-conv forward with all 8 parities in N (n = P*dcout + co)
  int out_bf16;                 // 1: the output frame stores bf16 (BF16 path)
  int ksplit;                   // split of each tile's K entries across CTAs (1 = none)
  int base_tiles;               // tiles without the split
  float* part;                  // ksplit > 1: raw partial tiles [ks][base_tiles][128][NT]
};

}  // namespace vpx

namespace {

using vpx::ConvTapParams;

// Destination of output columns [col, col+4) of the voxel q = (qz, qy, qx):
// the class-P output p = s*q + P, or (merged transposed conv) the parity of
// the column's block.  nullptr when the position is outside the valid range.
__device__ __forceinline__ float* tapbox_dst(const ConvTapParams& p, int n, int qz, int qy, int qx, int cls, int col) {
  int P = cls, c = col;
  if (p.dcout) {
    P = col / p.dcout;
    c = col % p.dcout;
  }
  const int pz = p.out_stride * qz + ((P >> 2) & 1), py = p.out_stride * qy + ((P >> 1) & 1),
            px = p.out_stride * qx + (P & 1);
  if (pz < p.pd_lo || pz >= p.pd_hi || py < p.ph_lo || py >= p.ph_hi || px < p.pw_lo || px >= p.pw_hi) return nullptr;
  return p.out + static_cast<long long>(n) * p.out_sn + static_cast<long long>(pz + p.out_off_d) * p.out_sd +
         static_cast<long long>(py + p.out_off_h) * p.out_sh + static_cast<long long>(px + p.out_off_w) * p.out_sw + c;
}

// Store 16 consecutive output channels at element offset `off` of the output
// (fp32, or bf16 on the BF16 path: round to nearest even).
__device__ __forceinline__ void tapbox_store16(const ConvTapParams& p, long long off, const float (&v)[16], int nmax) {
  if (p.out_bf16) {
    uint16_t* o = reinterpret_cast<uint16_t*>(p.out) + off;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (4 * i < nmax) {
        const __nv_bfloat162 lo = __floats2bfloat162_rn(v[4 * i], v[4 * i + 1]);
        const __nv_bfloat162 hi = __floats2bfloat162_rn(v[4 * i + 2], v[4 * i + 3]);
        uint2 w;
        w.x = *reinterpret_cast<const uint32_t*>(&lo);
        w.y = *reinterpret_cast<const uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(o + 4 * i) = w;
      }
    return;
  }
  float4* o4 = reinterpret_cast<float4*>(p.out + off);
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (4 * i < nmax) o4[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
}

// Fixed-order sum of the split-K partial tiles for (base tile tb, row r,
// channels 4 c4 .. 4 c4 + 3), then the epilogue (LeakyReLU, TF32 rounding,
// frame store) the single-pass kernel would have applied.
template <int NT>
__device__ __forceinline__ void tapbox_reduce_elem(const ConvTapParams& p, int tb, int r, int c4) {
  int tile = tb;
  const int nt = tile % p.ntn;
  tile /= p.ntn;
  const int cls = tile % p.ncls;
  tile /= p.ncls;
  const int xt = tile % p.tw;
  tile /= p.tw;
  const int yt = tile % p.th;
  tile /= p.th;
  const int zt = tile % p.td;
  const int n = tile / p.td;
  const int dx = r % p.Wb, dy = (r / p.Wb) % p.Hb, dz = r / (p.Wb * p.Hb);
  const int qz = p.qd + zt * p.Db + dz, qy = p.qh + yt * p.Hb + dy, qx = p.qw + xt * p.Wb + dx;
  const int Pd = (cls >> 2) & 1, Ph = (cls >> 1) & 1, Pw = cls & 1;
  const int pz = p.out_stride * qz + Pd, py = p.out_stride * qy + Ph, px = p.out_stride * qx + Pw;
  const bool valid = dz < p.Db && qz < p.qd + p.QD && qy < p.qh + p.QH && qx < p.qw + p.QW &&
                     (p.dcout || (pz >= p.pd_lo && pz < p.pd_hi && py >= p.ph_lo && py < p.ph_hi &&
                                  px >= p.pw_lo && px < p.pw_hi));
  if (!valid || nt * NT + 4 * c4 >= p.nvalid) return;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  const float4* src = reinterpret_cast<const float4*>(p.part + (static_cast<long long>(tb) * 128 + r) * NT) + c4;
  const long long kstride = static_cast<long long>(p.base_tiles) * 128 * NT / 4;
  int ks = 0;
  for (; ks + 16 <= p.ksplit; ks += 16) {  // deep splits: 16 loads in flight, summed in order
    float4 v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = src[(ks + j) * kstride];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      acc.x += v[j].x;
      acc.y += v[j].y;
      acc.z += v[j].z;
      acc.w += v[j].w;
    }
  }
  for (; ks + 4 <= p.ksplit; ks += 4) {  // four independent loads in flight, summed in order
    float4 v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = src[(ks + j) * kstride];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      acc.x += v[j].x;
      acc.y += v[j].y;
      acc.z += v[j].z;
      acc.w += v[j].w;
    }
  }
  for (; ks < p.ksplit; ++ks) {
    const float4 v = src[ks * kstride];
    acc.x += v.x;
    acc.y += v.y;
    acc.z += v.z;
    acc.w += v.w;
  }
  float o[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (p.act) o[j] = o[j] >= 0.f ? o[j] : p.slope * o[j];
    if (p.rnd && !p.out_bf16) o[j] = vpx::tf32_rn(o[j]);
  }
  float* dst = p.dcout ? tapbox_dst(p, n, qz, qy, qx, cls, nt * NT + 4 * c4)
                       : p.out + static_cast<long long>(n) * p.out_sn +
                             static_cast<long long>(pz + p.out_off_d) * p.out_sd +
                             static_cast<long long>(py + p.out_off_h) * p.out_sh +
                             static_cast<long long>(px + p.out_off_w) * p.out_sw + nt * NT + 4 * c4;
  if (dst && p.out_bf16) {
    const __nv_bfloat162 lo = __floats2bfloat162_rn(o[0], o[1]), hi = __floats2bfloat162_rn(o[2], o[3]);
    uint2 w;
    w.x = *reinterpret_cast<const uint32_t*>(&lo);
    w.y = *reinterpret_cast<const uint32_t*>(&hi);
    *reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(p.out) + (dst - p.out)) = w;
  } else if (dst) {
    *reinterpret_cast<float4*>(dst) = make_float4(o[0], o[1], o[2], o[3]);
  }
}

template <int NT>
__global__ void tapbox_reduce_kernel(const __grid_constant__ ConvTapParams p) {
  const long long total = (long long)p.base_tiles * 128 * (NT / 4);
  vpx::pdl_wait();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int c4 = static_cast<int>(i % (NT / 4));
    const int r = static_cast<int>((i / (NT / 4)) % 128);
    tapbox_reduce_elem<NT>(p, static_cast<int>(i / (NT / 4) / 128), r, c4);
  }
}

// BF16 = true: kind::f16 MMAs on bf16 operands (64-channel K chunks = the same
// 128-byte SWIZZLE_128B rows, K = 16 per MMA instead of 8), fp32 accumulation.
template <int NT, int S, bool BF16>
__global__ void __launch_bounds__(256, 1)
    conv_tapbox_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap wmap,
                       const ConvTapParams p) {
  constexpr int ABYTES = 128 * 128;  // 128 voxel rows x 128 bytes (32 fp32 / 64 bf16 channels)
  constexpr int CW = BF16 ? 64 : 32; // channels per K chunk
  constexpr int BBYTES = NT * 128;
  constexpr int STAGE = ABYTES + BBYTES;  // multiple of 1024
  constexpr int TCOLS = NT <= 32 ? 32 : NT <= 64 ? 64 : NT <= 128 ? 128 : 256;
  static_assert(2 * TCOLS <= 512, "TMEM");

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[S], empty[S], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
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
    vpx::tma_prefetch_desc(&wmap);
  }
  if (warp == 2) vpx::tmem_alloc<2 * TCOLS>(&tmem_base);
  vpx::tc_fence_before();
  __syncthreads();
  vpx::tc_fence_after();
  const uint32_t tbase = tmem_base;
  vpx::pdl_wait();

  // tile -> (k split, n-tile, class, n, zt, yt, xt)
  auto decode = [&](int tile, int& nt, int& cls, int& n, int& zt, int& yt, int& xt) {
    tile %= p.base_tiles;
    nt = tile % p.ntn;
    tile /= p.ntn;
    cls = tile % p.ncls;
    tile /= p.ncls;
    xt = tile % p.tw;
    tile /= p.tw;
    yt = tile % p.th;
    tile /= p.th;
    zt = tile % p.td;
    n = tile / p.td;
  };
  // j-th tile of this CTA.  Plain: round robin.  Balanced (stride-2 backward
  // data: the 8 parity classes carry 1..8 taps, and round robin gave every
  // CTA the same two classes -- up to 4x the work of the lightest CTAs): the
  // tiles sorted heaviest class first, dealt out serpentine.  Every tile is
  // still computed whole by one CTA, so the results are the same bits.
  auto tile_of = [&](int j) -> int {
    const int G = gridDim.x, b = blockIdx.x;
    if (!p.balance) return b + j * G;
    const int q = j * G + ((j & 1) ? G - 1 - b : b);
    if (q >= p.num_tiles) return p.num_tiles;
    const int per = p.num_tiles / p.ncls, rem = q % per;
    return ((rem / p.ntn) * p.ncls + p.cls_order[q / per]) * p.ntn + rem % p.ntn;
  };
  // K entries of this tile's class, restricted to its split
  auto krange = [&](int tile, int cls, int& e0, int& e1) {
    const int c0 = p.cls_start[cls], len = p.cls_start[cls + 1] - c0, ks = tile / p.base_tiles;
    e0 = c0 + len * ks / p.ksplit;
    e1 = c0 + len * (ks + 1) / p.ksplit;
  };

  if (warp == 0) {
    if (vpx::elect_one()) {
      const uint32_t a_tx = p.Db * p.Hb * p.Wb * 128;
      int stage = 0;
      uint32_t phase = 0;
      for (int j = 0, tile = tile_of(0); tile < p.num_tiles; tile = tile_of(++j)) {
        int nt, cls, n, zt, yt, xt;
        decode(tile, nt, cls, n, zt, yt, xt);
        const int qz = p.qd + zt * p.Db, qy = p.qh + yt * p.Hb, qx = p.qw + xt * p.Wb;
        int e0, e1;
        krange(tile, cls, e0, e1);
        for (int e = e0; e < e1; ++e) {
          const int ent = p.entries[e];
          const int od = (ent & 3) - 1, oh = ((ent >> 2) & 3) - 1, ow = ((ent >> 4) & 3) - 1;
          const int chunk = (ent >> 8) & 0xff;
          vpx::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE;
          vpx::mbar_arrive_expect_tx(&full[stage], a_tx + BBYTES);
          vpx::tma_load_5d(sa, &xmap, &full[stage], CW * chunk, p.in_stride * qx + ow + p.in_off_w,
                           p.in_stride * qy + oh + p.in_off_h, p.in_stride * qz + od + p.in_off_d, n);
          vpx::tma_load_2d(sa + ABYTES, &wmap, &full[stage], 0, e * p.ntot + nt * NT);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = vpx::make_idesc(BF16 ? 1 : 2, 128, NT, false, false);
    int stage = 0, acc = 0;
    uint32_t phase = 0, aphase = 0;
    for (int j = 0, tile = tile_of(0); tile < p.num_tiles; tile = tile_of(++j)) {
      int nt, cls, n, zt, yt, xt;
      decode(tile, nt, cls, n, zt, yt, xt);
      int e0, e1;
      krange(tile, cls, e0, e1);
      vpx::mbar_wait(&tempty[acc], aphase ^ 1);
      vpx::tc_fence_after();
      const uint32_t d = tbase + acc * TCOLS;
      for (int e = e0; e < e1; ++e) {
        vpx::mbar_wait(&full[stage], phase);
        vpx::tc_fence_after();
        if (vpx::elect_one()) {
          const uint32_t a = vpx::smem_u32(smem + stage * STAGE);
          const uint32_t b = a + ABYTES;
          const uint64_t ad0 = vpx::make_sdesc(a, 16, 1024, 2), bd0 = vpx::make_sdesc(b, 16, 1024, 2);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t ad = ad0 + 2 * k, bd = bd0 + 2 * k;  // +32 B per K step
            if constexpr (BF16)
              vpx::umma_f16(d, ad, bd, idesc, (e > e0 || k > 0) ? 1u : 0u);
            else
              vpx::umma_tf32(d, ad, bd, idesc, (e > e0 || k > 0) ? 1u : 0u);
          }
          vpx::umma_commit(&empty[stage]);
          if (e == e1 - 1) vpx::umma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (e1 == e0 && vpx::elect_one()) vpx::umma_commit(&tfull[acc]);  // empty class: no MMAs
      __syncwarp();
      acc ^= 1;
      if (acc == 0) aphase ^= 1;
    }
  } else if (warp >= 4) {
    const int q = warp - 4;
    const int r = q * 32 + lane;  // row of the M tile
    int acc = 0;
    uint32_t aphase = 0;
    for (int j = 0, tile = tile_of(0); tile < p.num_tiles; tile = tile_of(++j)) {
      int nt, cls, n, zt, yt, xt;
      decode(tile, nt, cls, n, zt, yt, xt);
      int e0, e1;
      krange(tile, cls, e0, e1);
      const bool empty_cls = e1 == e0;
      vpx::mbar_wait(&tfull[acc], aphase);
      vpx::tc_fence_after();
      const int dx = r % p.Wb, dy = (r / p.Wb) % p.Hb, dz = r / (p.Wb * p.Hb);
      const int qz = p.qd + zt * p.Db + dz, qy = p.qh + yt * p.Hb + dy, qx = p.qw + xt * p.Wb + dx;
      const int Pd = (cls >> 2) & 1, Ph = (cls >> 1) & 1, Pw = cls & 1;
      const int pz = p.out_stride * qz + Pd, py = p.out_stride * qy + Ph, px = p.out_stride * qx + Pw;
      const bool valid = dz < p.Db && qz < p.qd + p.QD && qy < p.qh + p.QH && qx < p.qw + p.QW &&
                         (p.dcout || (pz >= p.pd_lo && pz < p.pd_hi && py >= p.ph_lo && py < p.ph_hi &&
                                      px >= p.pw_lo && px < p.pw_hi));
      float* o = p.out + static_cast<long long>(n) * p.out_sn + static_cast<long long>(pz + p.out_off_d) * p.out_sd +
                 static_cast<long long>(py + p.out_off_h) * p.out_sh + static_cast<long long>(px + p.out_off_w) * p.out_sw +
                 nt * NT;
      // split K: raw partial accumulators, summed in order by tapbox_reduce_kernel
      float* prow = p.part + (static_cast<long long>(tile) * 128 + r) * NT;
#pragma unroll 1
      for (int cb = 0; cb < NT; cb += 16) {
        float v[16];
        vpx::tmem_ld16(tbase + (static_cast<uint32_t>(q * 32) << 16) + acc * TCOLS + cb, v);
        if (p.ksplit > 1) {
          if (!valid) continue;  // tapbox_reduce_elem skips these rows too
          float4* o4 = reinterpret_cast<float4*>(prow + cb);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            o4[i] = empty_cls ? make_float4(0.f, 0.f, 0.f, 0.f)
                              : make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        } else if (valid) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            if (empty_cls) v[i] = 0.f;
            if (p.act) v[i] = v[i] >= 0.f ? v[i] : p.slope * v[i];
            if (p.rnd && !p.out_bf16) v[i] = vpx::tf32_rn(v[i]);
          }
          if (p.dcout) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              float* d4 = tapbox_dst(p, n, qz, qy, qx, cls, nt * NT + cb + 4 * i);
              if (d4) *reinterpret_cast<float4*>(d4) = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
            }
          } else {
            tapbox_store16(p, (o - p.out) + cb, v, p.nvalid - (nt * NT + cb));
          }
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
  if (warp == 2) vpx::tmem_dealloc<2 * TCOLS>(tbase);
}

template <int NT, bool BF16 = false>
int launch_tapbox(const CUtensorMap& xm, const CUtensorMap& wm, const ConvTapParams& p, cudaStream_t st) {
  constexpr int STAGE = 128 * 128 + NT * 128;
  constexpr int S = (200 * 1024) / STAGE >= 6 ? 6 : (200 * 1024) / STAGE;
  auto kern = conv_tapbox_kernel<NT, S, BF16>;
  const int smem = S * STAGE + 1024;
  VPX_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int grid = p.num_tiles < vpx::num_sms() ? p.num_tiles : vpx::num_sms();
  VPX_CHECK_CUDA(vpx::launch_pdl(kern, grid, 256, smem, st, xm, wm, p));
  VPX_LAUNCH_CHECK();
  if (p.ksplit > 1) {
    const long long total = (long long)p.base_tiles * 128 * (NT / 4);
    const int rg = static_cast<int>((total + 255) / 256 < 4096 ? (total + 255) / 256 : 4096);
    VPX_CHECK_CUDA(vpx::launch_pdl(tapbox_reduce_kernel<NT>, rg, 256, 0, st, p));
    VPX_LAUNCH_CHECK();
  }
  return VPX_OK;
}

// Packed B: [entry][ntot][32]; value = Weff(o = row, i = 32*chunk + j, tap)
//   mode 0 fwd:   w[o][i][tap]        (ntot = cout, i over cin)
//   mode 1 dgrad: w[i][o][tap]        (ntot = cin,  i over cout)
//   kind 1 (k2s2 transposed conv, w = (cin, cout, 8)):
//   mode 1 fwd:   w[i][o][P]          (ntot = cout, i over cin)
//   mode 0 dgrad: w[o][i][P]          (ntot = cin,  i over cout)
__global__ void pack_tapbox_kernel(const float* __restrict__ w, int cout, int cin, int mode, int kind,
                                   const __grid_constant__ ConvTapParams tp, int n_entries, int ntot,
                                   float* __restrict__ out) {
  const long long total = (long long)n_entries * ntot * 32;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int j = idx % 32;
    const int o = (idx / 32) % ntot;
    const int e = static_cast<int>(idx / (32LL * ntot));
    const int i = 32 * ((tp.entries[e] >> 8) & 0xff) + j;
    const int tap = tp.entries[e] >> 16;
    float v = 0.f;
    if (o < tp.nvalid) {
      if (kind == 2) {  // merged transposed-conv forward: row o = P * cout + co
        if (i < cin) v = w[((long long)i * cout + o % cout) * 8 + o / cout];
      } else if (kind == 1) {
        if (mode == 1) {
          if (i < cin) v = w[((long long)i * cout + o) * 8 + tap];
        } else {
          if (i < cout) v = w[((long long)o * cout + i) * 8 + tap];
        }
      } else if (mode == 0) {
        if (i < cin) v = w[((long long)o * cin + i) * 27 + tap];
      } else {
        if (i < cout) v = w[((long long)i * cin + o) * 27 + tap];
      }
    }
    out[idx] = vpx::tf32_rn(v);
  }
}

// Same packing, one block per packed row o: the row's K x T source weights
// are staged in shared memory (one contiguous run for the forward layout),
// then each warp writes whole 128-byte entry segments.  The thread-per-element
// form above reads w with a 27- or 27*cin-float stride between neighbouring
// threads: 14 vs 9 us per CosmoFlow c6/c7 pass (tools/small_pass.py), where
// the pack is a third of the pass.  Row stride Tp = T rounded up to odd keeps
// the segment reads conflict-free.
__global__ void __launch_bounds__(256) pack_tapbox_row_kernel(const float* __restrict__ w, int cout, int cin,
                                                              int mode, int kind,
                                                              const __grid_constant__ ConvTapParams tp,
                                                              int n_entries, int ntot, int kchan,
                                                              float* __restrict__ out) {
  extern __shared__ float srow2[];
  const int o = blockIdx.x;
  const int T = kind == 0 ? 27 : kind == 1 ? 8 : 1, Tp = T | 1;
  const int kpad = (kchan + 31) / 32 * 32;
  const bool live = o < tp.nvalid;
  if (kind == 0 && mode == 0) {  // w[o][i][tap]: one contiguous run of cin * 27 floats
    const float* src = w + (long long)o * cin * 27;
    for (int idx = threadIdx.x; idx < kpad * 27; idx += blockDim.x) {
      const int i = idx / 27, t = idx - i * 27;
      srow2[i * Tp + t] = (live && i < kchan) ? src[idx] : 0.f;
    }
  } else {
    for (int idx = threadIdx.x; idx < kpad * T; idx += blockDim.x) {
      const int i = idx / T, t = idx % T;
      float v = 0.f;
      if (live && i < kchan) {
        if (kind == 2) v = w[((long long)i * cout + o % cout) * 8 + o / cout];
        else if (kind == 1) v = mode == 1 ? w[((long long)i * cout + o) * 8 + t] : w[((long long)o * cout + i) * 8 + t];
        else v = w[((long long)i * cin + o) * 27 + t];
      }
      srow2[i * Tp + t] = v;
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
#pragma unroll 4
  for (int e = threadIdx.x >> 5; e < n_entries; e += blockDim.x >> 5) {
    const int ent = tp.entries[e];
    const int chunk = (ent >> 8) & 0xff, tap = kind == 2 ? 0 : ent >> 16;
    out[((long long)e * ntot + o) * 32 + lane] = vpx::tf32_rn(srow2[(32 * chunk + lane) * Tp + tap]);
  }
}

// BF16 path: packed B [entry][ntot][64] bf16 (128-byte rows), 3x3x3 conv only.
__global__ void pack_tapbox_bf16_kernel(const float* __restrict__ w, int cout, int cin, int mode,
                                        const __grid_constant__ ConvTapParams tp, int n_entries, int ntot,
                                        __nv_bfloat16* __restrict__ out) {
  const long long total = (long long)n_entries * ntot * 64;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int j = idx % 64;
    const int o = (idx / 64) % ntot;
    const int e = static_cast<int>(idx / (64LL * ntot));
    const int i = 64 * ((tp.entries[e] >> 8) & 0xff) + j;
    const int tap = tp.entries[e] >> 16;
    float v = 0.f;
    if (o < tp.nvalid) {
      if (mode == 0) {
        if (i < cin) v = w[((long long)o * cin + i) * 27 + tap];
      } else {
        if (i < cout) v = w[((long long)i * cin + o) * 27 + tap];
      }
    }
    out[idx] = __float2bfloat16_rn(v);
  }
}

int encode_in_map(CUtensorMap* map, const float* base, const vpx::Frame& f, int Db, int Hb, int Wb, int s,
                  bool bf16 = false) {
  const uint64_t Wf = f.w + 2 * f.mw, Hf = f.h + 2 * f.mh, Df = f.d + 2 * f.md;
  const uint64_t eb = bf16 ? 2 : 4;  // bytes per element
  uint64_t dims[5] = {(uint64_t)f.c, Wf, Hf, Df, (uint64_t)f.n};
  uint64_t strides[4] = {(uint64_t)f.c * eb, Wf * f.c * eb, Hf * Wf * f.c * eb, Df * Hf * Wf * f.c * eb};
  uint32_t box[5] = {bf16 ? 64u : 32u, (uint32_t)(s * Wb), (uint32_t)(s * Hb), (uint32_t)(s * Db), 1};
  uint32_t estr[5] = {1, (uint32_t)s, (uint32_t)s, (uint32_t)s, 1};
  return vpx::encode_tiled_strided(map, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5,
                                   const_cast<float*>(base), dims, strides, box, estr, CU_TENSOR_MAP_SWIZZLE_128B);
}

int encode_w_map(CUtensorMap* map, const float* base, long long rows, int NT, bool bf16 = false) {
  uint64_t dims[2] = {bf16 ? 64u : 32u, (uint64_t)rows};
  uint64_t strides[1] = {128};
  uint32_t box[2] = {bf16 ? 64u : 32u, (uint32_t)NT};
  return vpx::encode_tiled(map, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                           const_cast<float*>(base), dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
}

void tile_shape(int D, int H, int W, int* Db, int* Hb, int* Wb) {
  *Wb = W < 128 ? W : 128;
  *Hb = H < 128 / *Wb ? H : 128 / *Wb;
  int rest = 128 / (*Wb * *Hb);
  *Db = D < rest ? D : rest;
}

}  // namespace

namespace vpx {

// Workspace: the packed weights, [entry <= 256][ntot][32] fp32.
long long tapbox_workspace_bytes(int cin, int cout) {
  const long long ntot = cin > cout ? cin : cout;
  return (long long)kMaxEntries * ntot * 32 * 4;
}

int tapbox_supported(int cin, int cout, int mode, int kind) {
  int ntot = (mode == 0) == (kind == 0) ? cout : cin;
  if (kind == 1 && ntot == 8) ntot = 16;  // 8-channel deconv outputs: N tile 16, stores masked
  // N tiles with a kernel instance: 16/32/64/128/256, or a multiple of 256
  return ntot == 16 || ntot == 32 || ntot == 64 || ntot == 128 || ntot % 256 == 0;
}

// mode 0: forward (stride 1 or 2); mode 1: backward-data (stride 1 or 2).
// in: input frame (x for fwd, u for dgrad); out: output frame.
// kind 0: 3x3x3 conv, mode 0 forward (stride 1 or 2), mode 1 backward-data.
// kind 1: k2s2 transposed conv (reference layers/reference.py:99-131, weights
//   (cin, cout, 2, 2, 2)), stride 2 implied: mode 1 = its forward (eight
//   parity classes P of the fine output p = 2q + P, one tap each, reading the
//   coarse input at q), mode 0 = its backward-data (the coarse gradient
//   gathers the fine one at 2q + P, eight taps, TMA element stride 2).
// in: the tensor streamed along K; out: the tensor written.
int conv_tapbox(int mode, const float* in, const Frame& inf, const float* w, int cin, int cout, int stride,
                float* out, const Frame& of, int act, float slope, void* ws, cudaStream_t st, long long ws_bytes,
                int kind, int bf16, const float* wpre, bool pack_only) {
  // transposed-conv forward as ONE GEMM per coarse-voxel tile: N = 8 parities x Cout,
  // the epilogue scatters column block P to the fine voxel 2q + P
  const bool merged = kind == 1 && mode == 1 && (8 * cout == 64 || 8 * cout == 128 || 8 * cout == 256);
  const int nvalid = merged ? 8 * cout : (mode == 0) == (kind == 0) ? cout : cin;
  const int ntot = (kind == 1 && nvalid == 8) ? 16 : nvalid;
  const int kchan = (mode == 0) == (kind == 0) ? cin : cout;  // channels along K
  const int cw = (bf16 & 1) ? 64 : 32;                         // channels per K chunk (one 128-byte row)
  const int nchunks = (kchan + cw - 1) / cw;
  if ((bf16 & 1) && kind != 0) VPX_FAIL(VPX_ERR_UNSUPPORTED, "tapbox bf16: 3x3x3 conv only");
  ConvTapParams p{};
  p.nvalid = nvalid;
  p.dcout = merged ? cout : 0;
  int ne = 0;
  if (kind == 1) stride = 2;
  const int ncls = (mode == 1 && stride == 2 && !merged) ? 8 : 1;
  for (int cls = 0; cls < ncls; ++cls) {
    p.cls_start[cls] = ne;
    if (merged) {
      for (int ch = 0; ch < nchunks; ++ch) p.entries[ne++] = 1 | (1 << 2) | (1 << 4) | (ch << 8);
      continue;
    }
    if (kind == 1) {
      for (int P = 0; P < 8; ++P) {
        if (mode == 1 && P != cls) continue;  // forward: class P uses tap P at offset 0
        const int off[3] = {mode == 0 ? (P >> 2) & 1 : 0, mode == 0 ? (P >> 1) & 1 : 0, mode == 0 ? P & 1 : 0};
        for (int ch = 0; ch < nchunks; ++ch) {
          if (ne >= kMaxEntries) VPX_FAIL(VPX_ERR_UNSUPPORTED, "tapbox: more than %d K entries", kMaxEntries);
          p.entries[ne++] = (off[0] + 1) | ((off[1] + 1) << 2) | ((off[2] + 1) << 4) | (ch << 8) | (P << 16);
        }
      }
      continue;
    }
    for (int tap = 0; tap < 27; ++tap) {
      const int t[3] = {tap / 9, (tap / 3) % 3, tap % 3};
      int off[3];
      bool ok = true;
      for (int dd = 0; dd < 3; ++dd) {
        if (mode == 0) {
          off[dd] = t[dd] - 1;  // input = s*q + t - 1
        } else if (stride == 1) {
          off[dd] = 1 - t[dd];  // u index = p + 1 - t
        } else {
          const int P = (cls >> (2 - dd)) & 1;
          const int num = P + 1 - t[dd];
          if (num & 1) ok = false;
          off[dd] = num / 2;  // u index = q + (P + 1 - t)/2, in {0, 1}
        }
      }
      if (!ok) continue;
      for (int ch = 0; ch < nchunks; ++ch) {
        if (ne >= kMaxEntries) VPX_FAIL(VPX_ERR_UNSUPPORTED, "tapbox: more than %d K entries", kMaxEntries);
        p.entries[ne++] = (off[0] + 1) | ((off[1] + 1) << 2) | ((off[2] + 1) << 4) | (ch << 8) | (tap << 16);
      }
    }
  }
  p.cls_start[ncls] = ne;
  // wpre: weights packed earlier (vpx_prepack_all); pack_only: just the pack, into ws
  float* wpack = wpre ? const_cast<float*>(wpre) : static_cast<float*>(ws);
  if (!wpre) {
    const long long total = (long long)ne * ntot * cw;
    int grid = static_cast<int>((total + 255) / 256);
    if (grid > 8192) grid = 8192;
    if (bf16 & 1)
      pack_tapbox_bf16_kernel<<<grid, 256, 0, st>>>(w, cout, cin, mode, p, ne, ntot,
                                                    reinterpret_cast<__nv_bfloat16*>(wpack));
    // the row-staged form wins once there are >= 256 packed rows (one block
    // each); below that the element-wise form's parallelism wins (c4, c5 dgrad)
    else if (ntot < 256 || getenv("VPX_PACK_ELEMWISE"))  // tests compare the two bit for bit
      pack_tapbox_kernel<<<grid, 256, 0, st>>>(w, cout, cin, mode, merged ? 2 : kind, p, ne, ntot, wpack);
    else {
      const int kk = merged ? 2 : kind, T = kk == 0 ? 27 : kk == 1 ? 8 : 1;
      const int smem = (kchan + 31) / 32 * 32 * (T | 1) * 4;
      if (smem > 48 * 1024)
        VPX_CHECK_CUDA(cudaFuncSetAttribute(pack_tapbox_row_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      pack_tapbox_row_kernel<<<ntot, 256, smem, st>>>(w, cout, cin, mode, kk, p, ne, ntot, kchan, wpack);
    }
    VPX_LAUNCH_CHECK();
  }
  if (pack_only) return VPX_OK;
  p.n = of.n;
  // q grid
  const int s_in = (mode == 0) ? stride : 1;
  const int s_out = (mode == 1) ? stride : 1;
  int QD, QH, QW, q0d = 0, q0h = 0, q0w = 0;
  if (mode == 0) {
    QD = of.d;
    QH = of.h;
    QW = of.w;
  } else if (kind == 1) {  // transposed conv: every coarse input voxel, interior outputs only
    QD = inf.d;
    QH = inf.h;
    QW = inf.w;
  } else {
    // cover output positions [-m, e+m) of the xg frame: q in [(-m - 1)/s .. ]
    const int lo[3] = {-of.md, -of.mh, -of.mw};
    const int hi[3] = {of.d + of.md, of.h + of.mh, of.w + of.mw};
    int qlo[3], qhi[3];
    for (int dd = 0; dd < 3; ++dd) {
      if (s_out == 1) {
        qlo[dd] = lo[dd];
        qhi[dd] = hi[dd];
      } else {  // p = 2q + P, P in {0,1}: q in [ceil((lo-1)/2), floor((hi-1)/2)]
        qlo[dd] = -((1 - lo[dd]) / 2);
        qhi[dd] = (hi[dd] - 1) / 2 + 1;
      }
    }
    q0d = qlo[0];
    q0h = qlo[1];
    q0w = qlo[2];
    QD = qhi[0] - qlo[0];
    QH = qhi[1] - qlo[1];
    QW = qhi[2] - qlo[2];
  }
  int Db, Hb, Wb;
  tile_shape(QD, QH, QW, &Db, &Hb, &Wb);
  p.qd = q0d;
  p.qh = q0h;
  p.qw = q0w;
  p.QD = QD;
  p.QH = QH;
  p.QW = QW;
  p.Db = Db;
  p.Hb = Hb;
  p.Wb = Wb;
  p.td = (QD + Db - 1) / Db;
  p.th = (QH + Hb - 1) / Hb;
  p.tw = (QW + Wb - 1) / Wb;
  p.ncls = ncls;
  const int NT = ntot <= 256 ? ntot : 256;
  p.ntn = ntot / NT;
  p.base_tiles = of.n * p.td * p.th * p.tw * ncls * p.ntn;
  // few tiles (deep layers): split each tile's K entries over otherwise idle
  // SMs; partial tiles go after the packed weights in the workspace.  At most
  // 16 ways (VPX_KSPLIT_MAX): on the 4^3/8^3 CosmoFlow layers a 64-way split
  // saved less in the conv than its partial tiles cost the reduce (c7 forward
  // 24.8 -> 21.7 us per pass, tools/small_pass.py)
  p.ksplit = 1;
  p.part = nullptr;
  {
    const long long wbytes = (tapbox_workspace_bytes(cin, cout) + 255) / 256 * 256;
    int ks = 2 * p.base_tiles <= num_sms() ? num_sms() / p.base_tiles : 1;
    const int min_entries = ne / ncls;
    if (ks > min_entries / 2) ks = min_entries / 2 > 1 ? min_entries / 2 : 1;
    static const int ks_cap = getenv("VPX_KSPLIT_MAX") ? atoi(getenv("VPX_KSPLIT_MAX")) : 16;
    if (ks > ks_cap) ks = ks_cap > 1 ? ks_cap : 1;
    const int NTc = ntot <= 256 ? ntot : 256;
    if (getenv("VPX_NO_KSPLIT")) ks = 1;
    // the split depends on the shape only (never on how large a workspace the
    // caller happens to pass), so results are reproducible run to run;
    // vpx_conv3d_workspace_bytes covers ks * base_tiles <= num_sms partial tiles
    if (ks > 1 && wbytes + (long long)ks * p.base_tiles * 128 * NTc * 4 > ws_bytes)
      VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "tapbox: workspace %lld B < %lld B (vpx_conv3d_workspace_bytes)", ws_bytes,
               wbytes + (long long)ks * p.base_tiles * 128 * NTc * 4);
    if (ks > 1) {
      p.ksplit = ks;
      p.part = reinterpret_cast<float*>(static_cast<char*>(ws) + wbytes);
    }
  }
  p.num_tiles = p.base_tiles * p.ksplit;
  p.balance = (ncls == 8 && p.ksplit == 1 && !getenv("VPX_TAPBOX_RR")) ? 1 : 0;
  for (int c = 0; c < 8; ++c) p.cls_order[c] = c < ncls ? c : 0;
  if (p.balance)  // stable: classes with equal entry counts keep their order
    std::stable_sort(p.cls_order, p.cls_order + ncls, [&](int a, int b) {
      return p.cls_start[a + 1] - p.cls_start[a] > p.cls_start[b + 1] - p.cls_start[b];
    });
  p.in_stride = s_in;
  p.in_off_d = inf.md;
  p.in_off_h = inf.mh;
  p.in_off_w = inf.mw;
  p.ntot = ntot;
  p.out = out;
  const long long Wf = of.w + 2 * of.mw, Hf = of.h + 2 * of.mh, Df = of.d + 2 * of.md;
  p.out_sw = of.c;
  p.out_sh = Wf * of.c;
  p.out_sd = Hf * Wf * of.c;
  p.out_sn = Df * Hf * Wf * of.c;
  p.out_off_d = of.md;
  p.out_off_h = of.mh;
  p.out_off_w = of.mw;
  p.out_stride = s_out;
  if (mode == 0 || kind == 1) {
    p.pd_lo = 0, p.pd_hi = of.d, p.ph_lo = 0, p.ph_hi = of.h, p.pw_lo = 0, p.pw_hi = of.w;
  } else {
    p.pd_lo = -of.md, p.pd_hi = of.d + of.md, p.ph_lo = -of.mh, p.ph_hi = of.h + of.mh;
    p.pw_lo = -of.mw, p.pw_hi = of.w + of.mw;
  }
  p.act = act;
  p.slope = slope;
  p.rnd = of.rnd;
  p.out_bf16 = bf16 >> 1;  // bit 1: bf16 output storage (bit 0: bf16 operands)
  CUtensorMap xm, wm;
  if (int rc = encode_in_map(&xm, in, inf, Db, Hb, Wb, s_in, bf16 & 1)) return rc;
  if (int rc = encode_w_map(&wm, wpack, (long long)ne * ntot, NT, bf16 & 1)) return rc;
  if (bf16 & 1) {
    switch (NT) {
      case 16: return launch_tapbox<16, true>(xm, wm, p, st);
      case 32: return launch_tapbox<32, true>(xm, wm, p, st);
      case 64: return launch_tapbox<64, true>(xm, wm, p, st);
      case 128: return launch_tapbox<128, true>(xm, wm, p, st);
      case 256: return launch_tapbox<256, true>(xm, wm, p, st);
    }
  }
  switch (NT) {
    case 16: return launch_tapbox<16>(xm, wm, p, st);
    case 32: return launch_tapbox<32>(xm, wm, p, st);
    case 64: return launch_tapbox<64>(xm, wm, p, st);
    case 128: return launch_tapbox<128>(xm, wm, p, st);
    case 256: return launch_tapbox<256>(xm, wm, p, st);
  }
  VPX_FAIL(VPX_ERR_UNSUPPORTED, "tapbox N tile %d", NT);
}

}  // namespace vpx
