// CUDA-core convolutions for the two U-Net layers whose channel counts are too
// small for a tensor-core tile (reference networks.py U-Net-mini):
//   * the 1x1x1 head (8 -> 2 channels): forward, input gradient, filter gradient;
//   * the first 3x3x3 layer on the 1-channel input (1 -> 8): forward (+ fused
//     LeakyReLU) and filter gradient.
// Both are HBM- or LSU-bound; what matters is one index decode per row (not per
// element), float4 channel loads, weights broadcast from shared memory, and for
// the filter gradients a persistent grid whose per-block partials are summed in
// fixed order by reduce_partials (deterministic).
// Arithmetic order of the forward / input-gradient kernels equals the generic
// direct kernels in conv_simt.cu (taps ascending, channels ascending, fmaf), so
// swapping paths does not change a single bit of those outputs.
#include "conv_simt.h"
#include "vpx_host.h"
#include <cstdlib>

#include "vpx_round.cuh"

namespace vpx {

namespace {

__device__ __forceinline__ long long fidx(const Frame& f, int n, int z, int y, int x) {
  return ((((long long)n * (f.d + 2 * f.md) + (z + f.md)) * (f.h + 2 * f.mh) + (y + f.mh)) *
              (f.w + 2 * f.mw) +
          (x + f.mw)) *
         f.c;
}
// first interior voxel of interior row `row` = (n, z, y)
__device__ __forceinline__ long long frow(const Frame& f, long long row) {
  const int y = static_cast<int>(row % f.h);
  row /= f.h;
  const int z = static_cast<int>(row % f.d);
  const int n = static_cast<int>(row / f.d);
  return fidx(f, n, z, y, 0);
}
__device__ __forceinline__ bool finside(const Frame& f, int z, int y, int x) {
  return z >= -f.md && z < f.d + f.md && y >= -f.mh && y < f.h + f.mh && x >= -f.mw && x < f.w + f.mw;
}

template <int C>
__device__ __forceinline__ void load_c(const float* p, float (&v)[C]) {
  if constexpr (C % 4 == 0) {
#pragma unroll
    for (int i = 0; i < C / 4; ++i) {
      const float4 t = *reinterpret_cast<const float4*>(p + 4 * i);
      v[4 * i] = t.x;
      v[4 * i + 1] = t.y;
      v[4 * i + 2] = t.z;
      v[4 * i + 3] = t.w;
    }
  } else if constexpr (C % 2 == 0) {
#pragma unroll
    for (int i = 0; i < C / 2; ++i) {
      const float2 t = *reinterpret_cast<const float2*>(p + 2 * i);
      v[2 * i] = t.x;
      v[2 * i + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < C; ++i) v[i] = p[i];
  }
}

// ------------------------------------------------------------ 1x1x1 conv
// y[v][co] = sum_ci x[v][ci] w[co][ci]; blocks stride over interior rows.
template <int CI, int CO>
__global__ void __launch_bounds__(256) pw_fwd_kernel(const float* __restrict__ x, Frame xf,
                                                     const float* __restrict__ w, float* __restrict__ y,
                                                     Frame yf, int act, float slope) {
  __shared__ float ws[CO * CI];
  for (int i = threadIdx.x; i < CO * CI; i += blockDim.x) ws[i] = rnd(yf, w[i]);  // TF32 mode: TF32 operands
  __syncthreads();
  const long long nrows = (long long)xf.n * xf.d * xf.h;
  for (long long row = blockIdx.x; row < nrows; row += gridDim.x) {
    const float* xr = x + frow(xf, row);
    float* yr = y + frow(yf, row);
    for (int i = threadIdx.x; i < xf.w; i += blockDim.x) {
      float xv[CI];
      load_c<CI>(xr + (long long)i * CI, xv);
#pragma unroll
      for (int co = 0; co < CO; ++co) {
        float acc = 0.f;
#pragma unroll
        for (int ci = 0; ci < CI; ++ci) acc = fmaf(xv[ci], ws[co * CI + ci], acc);
        yr[(long long)i * CO + co] = rnd(yf, (act && acc < 0.f) ? slope * acc : acc);
      }
    }
  }
}

// g[v][ci] = sum_co u[v][co] w[co][ci] (gradient frame without margins)
template <int CI, int CO>
__global__ void __launch_bounds__(256) pw_dgrad_kernel(const float* __restrict__ u, Frame uf,
                                                       const float* __restrict__ w, float* __restrict__ g,
                                                       Frame gf) {
  __shared__ float ws[CO * CI];
  for (int i = threadIdx.x; i < CO * CI; i += blockDim.x) ws[i] = rnd(gf, w[i]);
  __syncthreads();
  const long long nrows = (long long)uf.n * uf.d * uf.h;
  for (long long row = blockIdx.x; row < nrows; row += gridDim.x) {
    const float* ur = u + frow(uf, row);
    float* gr = g + frow(gf, row);
    for (int i = threadIdx.x; i < uf.w; i += blockDim.x) {
      float uv[CO];
      load_c<CO>(ur + (long long)i * CO, uv);
      float acc[CI];
#pragma unroll
      for (int ci = 0; ci < CI; ++ci) acc[ci] = 0.f;
#pragma unroll
      for (int co = 0; co < CO; ++co)
#pragma unroll
        for (int ci = 0; ci < CI; ++ci) acc[ci] = fmaf(uv[co], ws[co * CI + ci], acc[ci]);
      float* gp = gr + (long long)i * CI;
      if constexpr (CI % 4 == 0) {
#pragma unroll
        for (int q = 0; q < CI / 4; ++q)
          *reinterpret_cast<float4*>(gp + 4 * q) =
              rnd4(gf, make_float4(acc[4 * q], acc[4 * q + 1], acc[4 * q + 2], acc[4 * q + 3]));
      } else {
#pragma unroll
        for (int ci = 0; ci < CI; ++ci) gp[ci] = rnd(gf, acc[ci]);
      }
    }
  }
}

// Block-level fixed-order reduction of NV per-thread values into out[0..NV).
template <int NV>
__device__ __forceinline__ void block_reduce_store(float (&acc)[NV], float* red, float* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    float v = acc[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp * NV + j] = v;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < NV; j += blockDim.x) {
    float s = 0.f;
    for (int q = 0; q < nw; ++q) s += red[q * NV + j];
    out[j] = s;
  }
}

// part[block][co][ci] = sum over the block's rows of u[v][co] x[v][ci]
template <int CI, int CO>
__global__ void __launch_bounds__(256) pw_wgrad_kernel(const float* __restrict__ x, Frame xf,
                                                       const float* __restrict__ u, Frame uf,
                                                       float* __restrict__ part) {
  __shared__ float red[8 * CO * CI];
  float acc[CO * CI];
#pragma unroll
  for (int j = 0; j < CO * CI; ++j) acc[j] = 0.f;
  const long long nrows = (long long)uf.n * uf.d * uf.h;
  for (long long row = blockIdx.x; row < nrows; row += gridDim.x) {
    const float* xr = x + frow(xf, row);
    const float* ur = u + frow(uf, row);
    for (int i = threadIdx.x; i < uf.w; i += blockDim.x) {
      float xv[CI], uv[CO];
      load_c<CI>(xr + (long long)i * CI, xv);
      load_c<CO>(ur + (long long)i * CO, uv);
#pragma unroll
      for (int co = 0; co < CO; ++co)
#pragma unroll
        for (int ci = 0; ci < CI; ++ci) acc[co * CI + ci] = fmaf(uv[co], xv[ci], acc[co * CI + ci]);
    }
  }
  block_reduce_store<CO * CI>(acc, red, part + (long long)blockIdx.x * CO * CI);
}

// ------------------------------------------------ 3x3x3 conv, 1 input channel
constexpr int kTX = 64, kTY = 4;  // output tile: 4 rows x 64 voxels of one plane

struct C1Tile {
  int n, z, y0, x0;
};
__device__ __forceinline__ C1Tile c1_tile(const Frame& of, long long t) {
  const int tx = (of.w + kTX - 1) / kTX, ty = (of.h + kTY - 1) / kTY;
  C1Tile r;
  r.x0 = static_cast<int>(t % tx) * kTX;
  t /= tx;
  r.y0 = static_cast<int>(t % ty) * kTY;
  t /= ty;
  r.z = static_cast<int>(t % of.d);
  r.n = static_cast<int>(t / of.d);
  return r;
}
// xs[a][yy][xx] = x[z + a - 1][y0 + yy - 1][x0 + xx - 1] (0 outside the frame)
__device__ __forceinline__ void c1_load_x(const float* __restrict__ x, const Frame& xf, const C1Tile& t,
                                          float* xs) {
  constexpr int PY = kTY + 2, PX = kTX + 2;
  for (int i = threadIdx.x; i < 3 * PY * PX; i += blockDim.x) {
    const int xx = i % PX, yy = (i / PX) % PY, a = i / (PX * PY);
    const int iz = t.z + a - 1, iy = t.y0 + yy - 1, ix = t.x0 + xx - 1;
    xs[i] = finside(xf, iz, iy, ix) ? __ldg(x + fidx(xf, t.n, iz, iy, ix)) : 0.f;
  }
}

template <int CO>
__global__ void __launch_bounds__(256) c1k3_fwd_kernel(const float* __restrict__ x, Frame xf,
                                                       const float* __restrict__ w, float* __restrict__ y,
                                                       Frame yf, int act, float slope) {
  constexpr int PY = kTY + 2, PX = kTX + 2;
  __shared__ float xs[3 * PY * PX];
  __shared__ __align__(16) float ws[27 * CO];  // ws[tap][co] = w[co][0][tap]
  for (int i = threadIdx.x; i < 27 * CO; i += blockDim.x) ws[i] = rnd(yf, w[(i % CO) * 27 + i / CO]);
  const C1Tile t = c1_tile(yf, blockIdx.x);
  c1_load_x(x, xf, t, xs);
  __syncthreads();
  const int tx = threadIdx.x % kTX, ty = threadIdx.x / kTX;
  const int ox = t.x0 + tx, oy = t.y0 + ty;
  if (ox >= yf.w || oy >= yf.h) return;
  float acc[CO];
#pragma unroll
  for (int co = 0; co < CO; ++co) acc[co] = 0.f;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const float xv = xs[(a * PY + ty + b) * PX + tx + c];
        const float* wt = ws + ((a * 3 + b) * 3 + c) * CO;
#pragma unroll
        for (int co = 0; co < CO; ++co) acc[co] = fmaf(xv, wt[co], acc[co]);
      }
  float* yp = y + fidx(yf, t.n, t.z, oy, ox);
#pragma unroll
  for (int j = 0; j < CO; ++j) acc[j] = (act && acc[j] < 0.f) ? slope * acc[j] : acc[j];
#pragma unroll
  for (int q = 0; q < CO / 4; ++q)
    *reinterpret_cast<float4*>(yp + 4 * q) =
        rnd4(yf, make_float4(acc[4 * q], acc[4 * q + 1], acc[4 * q + 2], acc[4 * q + 3]));
}

// Same conv, register-blocked: a block computes 4 planes x 4 rows x 64
// voxels; a thread owns 4 consecutive voxels of one row and all CO channels,
// so per (depth, height) tap row it reads 6 input values once and reuses each
// for 3 width taps x 4 voxels, and each tap's CO weights (broadcast float4s)
// for its 4 voxels: 12 FMAs per shared-memory load instead of ~3 (the
// one-voxel-per-thread kernel above ran at 14 TF/s, bound by its loads).
constexpr int kF4Z = 4, kF4Y = 4, kF4X = 64, kF4P = kF4X + 4;  // row pitch 68 floats: 16-byte aligned rows

template <int CO>
__global__ void __launch_bounds__(256) c1k3_fwd4_kernel(const float* __restrict__ x, Frame xf,
                                                        const float* __restrict__ w, float* __restrict__ y,
                                                        Frame yf, int act, float slope) {
  constexpr int RZ = kF4Z + 2, RY = kF4Y + 2;
  __shared__ __align__(16) float xs[RZ * RY * kF4P];
  __shared__ __align__(16) float ws[27 * CO];  // ws[tap][co] = w[co][0][tap]
  for (int i = threadIdx.x; i < 27 * CO; i += blockDim.x) ws[i] = rnd(yf, w[(i % CO) * 27 + i / CO]);
  long long t = blockIdx.x;
  const int ntx = (yf.w + kF4X - 1) / kF4X, nty = (yf.h + kF4Y - 1) / kF4Y, ntz = (yf.d + kF4Z - 1) / kF4Z;
  const int x0 = static_cast<int>(t % ntx) * kF4X;
  t /= ntx;
  const int y0 = static_cast<int>(t % nty) * kF4Y;
  t /= nty;
  const int z0 = static_cast<int>(t % ntz) * kF4Z;
  const int n = static_cast<int>(t / ntz);
  // stage input rows (z0-1 .. z0+4) x (y0-1 .. y0+4), voxels x0-1 .. x0+kF4X+2; one warp per row
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int r = warp; r < RZ * RY; r += blockDim.x >> 5) {
    const int iz = z0 + r / RY - 1, iy = y0 + r % RY - 1;
    const bool rowin = iz >= -xf.md && iz < xf.d + xf.md && iy >= -xf.mh && iy < xf.h + xf.mh;
    const float* src = x + fidx(xf, n, rowin ? iz : 0, rowin ? iy : 0, 0);
    for (int i = lane; i < kF4P; i += 32) {
      const int ix = x0 + i - 1;
      xs[r * kF4P + i] = rowin && ix >= -xf.mw && ix < xf.w + xf.mw ? __ldg(src + (long long)ix * xf.c) : 0.f;
    }
  }
  __syncthreads();
  const int q = threadIdx.x % (kF4X / 4), ty = (threadIdx.x / (kF4X / 4)) % kF4Y, tz = threadIdx.x / (kF4X / 4 * kF4Y);
  const int oz = z0 + tz, oy = y0 + ty, ox = x0 + 4 * q;
  if (oz >= yf.d || oy >= yf.h || ox >= yf.w) return;
  float acc[4][CO];
#pragma unroll
  for (int v = 0; v < 4; ++v)
#pragma unroll
    for (int co = 0; co < CO; ++co) acc[v][co] = 0.f;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const float* xr = xs + ((tz + a) * RY + ty + b) * kF4P + 4 * q;  // voxel ox + i - 1 is xr[i]
      const float4 lo = *reinterpret_cast<const float4*>(xr);
      const float2 hi = *reinterpret_cast<const float2*>(xr + 4);
      const float xw[6] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y};
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const float* wt = ws + ((a * 3 + b) * 3 + c) * CO;
#pragma unroll
        for (int g = 0; g < CO / 4; ++g) {
          const float4 w4 = *reinterpret_cast<const float4*>(wt + 4 * g);
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const float xv = xw[v + c];
            acc[v][4 * g] = fmaf(xv, w4.x, acc[v][4 * g]);
            acc[v][4 * g + 1] = fmaf(xv, w4.y, acc[v][4 * g + 1]);
            acc[v][4 * g + 2] = fmaf(xv, w4.z, acc[v][4 * g + 2]);
            acc[v][4 * g + 3] = fmaf(xv, w4.w, acc[v][4 * g + 3]);
          }
        }
      }
    }
  float* yp = y + fidx(yf, n, oz, oy, ox);
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    if (ox + v >= yf.w) break;
#pragma unroll
    for (int g = 0; g < CO / 4; ++g) {
      float4 o = make_float4(acc[v][4 * g], acc[v][4 * g + 1], acc[v][4 * g + 2], acc[v][4 * g + 3]);
      if (act) {
        o.x = o.x < 0.f ? slope * o.x : o.x;
        o.y = o.y < 0.f ? slope * o.y : o.y;
        o.z = o.z < 0.f ? slope * o.z : o.z;
        o.w = o.w < 0.f ? slope * o.w : o.w;
      }
      *reinterpret_cast<float4*>(yp + (long long)v * yf.c + 4 * g) = rnd4(yf, o);
    }
  }
}

// part[block][co][tap] = sum over the block's tiles of u[v][co] x[v + tap - 1].
// Thread roles: ((a, b) tap row, 4-channel group q) x VG voxel groups.  A role
// slides along W over 4-voxel segments: per voxel one float4 of u and one new
// x value feed 12 FMAs (the three width taps of its row x 4 channels), instead
// of one LDS.128 per FMA quad when every tap re-read u (the kernel was
// shared-memory bound at 10x its HBM roofline).  Tiles are staged row by row
// (one index decode per row, not per element).
template <int CO>
__global__ void __launch_bounds__(256) c1k3_wgrad_kernel(const float* __restrict__ x, Frame xf,
                                                         const float* __restrict__ u, Frame uf,
                                                         long long ntiles, float* __restrict__ part) {
  constexpr int PY = kTY + 2, PX = kTX + 2, NQ = CO / 4, ROLES = 9 * NQ, VG = 256 / ROLES;
  constexpr int SEG = 4, ITEMS = kTY * (kTX / SEG);
  __shared__ float xs[3 * PY * PX];
  __shared__ __align__(16) float us[kTX * kTY * CO];
  __shared__ __align__(16) float red[VG * 27 * CO];
  const int role = threadIdx.x % ROLES, vg = threadIdx.x / ROLES;
  const int ab = role / NQ, q = role % NQ;
  const int a = ab / 3, b = ab % 3;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float acc[3][4] = {};
  for (long long ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
    const C1Tile t = c1_tile(uf, ti);
    for (int rr = warp; rr < 3 * PY; rr += 8) {  // x patch rows (depth a, row yy), voxels t.x0-1 .. t.x0+kTX
      const int aa = rr / PY, yy = rr % PY;
      const int iz = t.z + aa - 1, iy = t.y0 + yy - 1;
      const bool rowin = iz >= -xf.md && iz < xf.d + xf.md && iy >= -xf.mh && iy < xf.h + xf.mh;
      const float* src = x + fidx(xf, t.n, rowin ? iz : 0, rowin ? iy : 0, 0);
      for (int xx = lane; xx < PX; xx += 32) {
        const int ix = t.x0 + xx - 1;
        xs[rr * PX + xx] = rowin && ix >= -xf.mw && ix < xf.w + xf.mw ? __ldg(src + (long long)ix * xf.c) : 0.f;
      }
    }
    for (int r = warp; r < kTY; r += 8) {  // u rows: kTX voxels x CO channels, contiguous in the frame
      const int oy = t.y0 + r;
      const float4* src = oy < uf.h ? reinterpret_cast<const float4*>(u + fidx(uf, t.n, t.z, oy, t.x0)) : nullptr;
      for (int i = lane; i < kTX * NQ; i += 32) {
        float4 val = make_float4(0.f, 0.f, 0.f, 0.f);
        if (src != nullptr && t.x0 + i / NQ < uf.w) val = src[i];
        reinterpret_cast<float4*>(us + r * kTX * CO)[i] = val;
      }
    }
    __syncthreads();
    if (vg < VG) {
      for (int it = vg; it < ITEMS; it += VG) {
        const int r = it / (kTX / SEG), x0 = (it % (kTX / SEG)) * SEG;
        const float* xb = xs + (a * PY + r + b) * PX + x0;  // x[v + c - 1] for voxel x0 + i is xb[i + c]
        float xw[SEG + 2];
#pragma unroll
        for (int i = 0; i < SEG + 2; ++i) xw[i] = xb[i];
#pragma unroll
        for (int i = 0; i < SEG; ++i) {
          const float4 uv = *reinterpret_cast<const float4*>(us + (r * kTX + x0 + i) * CO + 4 * q);
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            acc[c][0] = fmaf(uv.x, xw[i + c], acc[c][0]);
            acc[c][1] = fmaf(uv.y, xw[i + c], acc[c][1]);
            acc[c][2] = fmaf(uv.z, xw[i + c], acc[c][2]);
            acc[c][3] = fmaf(uv.w, xw[i + c], acc[c][3]);
          }
        }
      }
    }
    __syncthreads();
  }
  if (vg < VG) {
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int j = 0; j < 4; ++j) red[(vg * CO + 4 * q + j) * 27 + ab * 3 + c] = acc[c][j];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 27 * CO; i += blockDim.x) {
    float s = 0.f;
    for (int g = 0; g < VG; ++g) s += red[g * 27 * CO + i];
    part[(long long)blockIdx.x * 27 * CO + i] = s;  // [co][ci = 0][tap]
  }
}

int rows_grid(const Frame& f, int cap_per_sm) {
  const long long rows = (long long)f.n * f.d * f.h;
  const long long cap = (long long)num_sms() * cap_per_sm;
  return static_cast<int>(rows < 1 ? 1 : (rows > cap ? cap : rows));
}

}  // namespace

// ------------------------------------------------------------------- host
#define PW_CASES(X) X(4, 1) X(4, 2) X(4, 4) X(8, 1) X(8, 2) X(8, 4) X(16, 1) X(16, 2) X(16, 4) X(32, 1) X(32, 2)

int small_conv_supported(int which, const Frame& xf, const Frame& of, int k, int s) {
  // which: 0 fwd (xf input, of output), 1 bwd-data (xf = upstream, of = gradient), 2 bwd-filter
  if (s != 1) return 0;
  if (k == 1) {
    const int ci = which == 1 ? of.c : xf.c, co = which == 1 ? xf.c : of.c;
#define PW_OK(a, b) if (ci == a && co == b) return which != 1 || (of.md == 0 && of.mh == 0 && of.mw == 0);
    PW_CASES(PW_OK)
#undef PW_OK
    return 0;
  }
  if (k == 3 && which != 1) {
    const int co = of.c;
    return xf.c == 1 && (co == 4 || co == 8 || co == 16);
  }
  return 0;
}

int small_wgrad_parts(const Frame& uf, int k) {
  if (k == 1) return rows_grid(uf, 4);
  const long long ntiles = (long long)uf.n * uf.d * ((uf.h + kTY - 1) / kTY) * ((uf.w + kTX - 1) / kTX);
  // one wave of resident blocks (each loops over tiles): 8 per SM asked for
  // more than fit (5 by registers for CO = 8), leaving a 0.6-wave tail that
  // every block's equal share of tiles turned into a second full wave
  int per_sm = 8;
  const int co = uf.c;
  int occ = 0;
  if (co == 4) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, c1k3_wgrad_kernel<4>, 256, 0);
  if (co == 8) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, c1k3_wgrad_kernel<8>, 256, 0);
  if (co == 16) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, c1k3_wgrad_kernel<16>, 256, 0);
  if (occ > 0 && occ < per_sm) per_sm = occ;
  const long long cap = (long long)per_sm * num_sms();
  return static_cast<int>(ntiles < cap ? ntiles : cap);
}

int small_conv_fwd(const float* x, const Frame& xf, const float* w, int k, float* y, const Frame& yf, int act,
                   float slope, cudaStream_t st) {
  if (k == 1) {
#define PW_F(a, b)                                                                           \
  if (xf.c == a && yf.c == b) {                                                              \
    pw_fwd_kernel<a, b><<<rows_grid(xf, 16), 256, 0, st>>>(x, xf, w, y, yf, act, slope);     \
    VPX_LAUNCH_CHECK();                                                                      \
    return VPX_OK;                                                                           \
  }
    PW_CASES(PW_F)
#undef PW_F
  } else {
    if (!getenv("VPX_C1K3_V1")) {
      const long long ntiles = (long long)yf.n * ((yf.d + kF4Z - 1) / kF4Z) * ((yf.h + kF4Y - 1) / kF4Y) *
                               ((yf.w + kF4X - 1) / kF4X);
      if (ntiles > 0x7fffffffLL) VPX_FAIL(VPX_ERR_UNSUPPORTED, "too many tiles");
      const int g = static_cast<int>(ntiles);
      switch (yf.c) {
        case 4: c1k3_fwd4_kernel<4><<<g, 256, 0, st>>>(x, xf, w, y, yf, act, slope); break;
        case 8: c1k3_fwd4_kernel<8><<<g, 256, 0, st>>>(x, xf, w, y, yf, act, slope); break;
        case 16: c1k3_fwd4_kernel<16><<<g, 256, 0, st>>>(x, xf, w, y, yf, act, slope); break;
        default: VPX_FAIL(VPX_ERR_UNSUPPORTED, "small conv fwd: %d channels", yf.c);
      }
      VPX_LAUNCH_CHECK();
      return VPX_OK;
    }
    const long long ntiles = (long long)yf.n * yf.d * ((yf.h + kTY - 1) / kTY) * ((yf.w + kTX - 1) / kTX);
    if (ntiles > 0x7fffffffLL) VPX_FAIL(VPX_ERR_UNSUPPORTED, "too many tiles");
    const int g = static_cast<int>(ntiles);
    switch (yf.c) {
      case 4: c1k3_fwd_kernel<4><<<g, 256, 0, st>>>(x, xf, w, y, yf, act, slope); break;
      case 8: c1k3_fwd_kernel<8><<<g, 256, 0, st>>>(x, xf, w, y, yf, act, slope); break;
      case 16: c1k3_fwd_kernel<16><<<g, 256, 0, st>>>(x, xf, w, y, yf, act, slope); break;
      default: VPX_FAIL(VPX_ERR_UNSUPPORTED, "small conv fwd: %d channels", yf.c);
    }
    VPX_LAUNCH_CHECK();
    return VPX_OK;
  }
  VPX_FAIL(VPX_ERR_UNSUPPORTED, "small conv fwd: %d -> %d channels", xf.c, yf.c);
}

int small_conv_bwd_data(const float* u, const Frame& uf, const float* w, float* g, const Frame& gf,
                        cudaStream_t st) {
#define PW_D(a, b)                                                                   \
  if (gf.c == a && uf.c == b) {                                                      \
    pw_dgrad_kernel<a, b><<<rows_grid(uf, 16), 256, 0, st>>>(u, uf, w, g, gf);       \
    VPX_LAUNCH_CHECK();                                                              \
    return VPX_OK;                                                                   \
  }
  PW_CASES(PW_D)
#undef PW_D
  VPX_FAIL(VPX_ERR_UNSUPPORTED, "small conv bwd_data: %d -> %d channels", gf.c, uf.c);
}

// Partials only: part[P][cout][cin][k^3], P = small_wgrad_parts(uf, k).
int small_conv_wgrad(const float* x, const Frame& xf, const float* u, const Frame& uf, int k, float* part,
                     cudaStream_t st) {
  const int P = small_wgrad_parts(uf, k);
  if (k == 1) {
#define PW_W(a, b)                                                              \
  if (xf.c == a && uf.c == b) {                                                 \
    pw_wgrad_kernel<a, b><<<P, 256, 0, st>>>(x, xf, u, uf, part);               \
    VPX_LAUNCH_CHECK();                                                         \
    return VPX_OK;                                                              \
  }
    PW_CASES(PW_W)
#undef PW_W
    VPX_FAIL(VPX_ERR_UNSUPPORTED, "small conv wgrad: %d -> %d channels", xf.c, uf.c);
  }
  const long long ntiles = (long long)uf.n * uf.d * ((uf.h + kTY - 1) / kTY) * ((uf.w + kTX - 1) / kTX);
  switch (uf.c) {
    case 4: c1k3_wgrad_kernel<4><<<P, 256, 0, st>>>(x, xf, u, uf, ntiles, part); break;
    case 8: c1k3_wgrad_kernel<8><<<P, 256, 0, st>>>(x, xf, u, uf, ntiles, part); break;
    case 16: c1k3_wgrad_kernel<16><<<P, 256, 0, st>>>(x, xf, u, uf, ntiles, part); break;
    default: VPX_FAIL(VPX_ERR_UNSUPPORTED, "small conv wgrad: %d channels", uf.c);
  }
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}

}  // namespace vpx
