// Direct (CUDA-core) 3D convolution kernels for the shapes the tcgen05 paths
// do not cover: odd kernel sizes other than 3 (the U-Net 1x1x1 head), stride-2
// backward-data, frame-margin faces.  Same arithmetic contract as the
// reference's direct loops (reference pkg/src/voxpar/kernels/_hot.pyx:19-93):
// fp32 inputs, fp32 accumulation, "same" zero padding r = (k-1)/2, output
// extent ceil(e/stride).  Tensors are NDHWC halo frames (see include/vpx.h).
#include "conv_simt.h"
#include "vpx_host.h"
#include "vpx_ptx.cuh"
#include "vpx_round.cuh"

namespace vpx {

__device__ __forceinline__ long long fr_index(const Frame& f, int n, int z, int y, int x) {
  return ((((long long)n * (f.d + 2 * f.md) + (z + f.md)) * (f.h + 2 * f.mh) + (y + f.mh)) *
              (f.w + 2 * f.mw) +
          (x + f.mw)) *
         f.c;
}
__device__ __forceinline__ bool fr_inside(const Frame& f, int z, int y, int x) {
  return z >= -f.md && z < f.d + f.md && y >= -f.mh && y < f.h + f.mh && x >= -f.mw &&
         x < f.w + f.mw;
}

// y[n,o,co] = sum_{tap,ci} x[n, s*o + tap - r, ci] * w[co,ci,tap]; CPT output channels per thread.
template <int CPT>
__global__ void conv_fwd_simt_kernel(const float* __restrict__ x, Frame xf,
                                     const float* __restrict__ w, int k, int s,
                                     float* __restrict__ y, Frame yf, int act, float slope) {
  const int cq = yf.c / CPT;
  const long long total = (long long)yf.n * yf.d * yf.h * yf.w * cq;
  const int r = (k - 1) / 2;
  const int k3 = k * k * k;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    long long t = idx;
    const int c4 = t % cq;
    t /= cq;
    const int ox = t % yf.w;
    t /= yf.w;
    const int oy = t % yf.h;
    t /= yf.h;
    const int oz = t % yf.d;
    const int n = t / yf.d;
    float acc[CPT];
#pragma unroll
    for (int j = 0; j < CPT; ++j) acc[j] = 0.f;
    for (int a = 0; a < k; ++a) {
      const int iz = s * oz + a - r;
      for (int b = 0; b < k; ++b) {
        const int iy = s * oy + b - r;
        for (int c = 0; c < k; ++c) {
          const int ix = s * ox + c - r;
          if (!fr_inside(xf, iz, iy, ix)) continue;
          const float* xp = x + fr_index(xf, n, iz, iy, ix);
          const int tap = (a * k + b) * k + c;
          for (int ci = 0; ci < xf.c; ++ci) {
            const float xv = __ldg(xp + ci);
#pragma unroll
            for (int j = 0; j < CPT; ++j)
              acc[j] = fmaf(xv, rnd(yf, __ldg(w + ((long long)(CPT * c4 + j) * xf.c + ci) * k3 + tap)), acc[j]);
          }
        }
      }
    }
    float* yp = y + fr_index(yf, n, oz, oy, ox) + CPT * c4;
#pragma unroll
    for (int j = 0; j < CPT; ++j) yp[j] = rnd(yf, (act && acc[j] < 0.f) ? slope * acc[j] : acc[j]);
  }
}

// Input gradient as a gather over the adjoint: xg[n,p,ci] = sum u[n,o,co] w[co,ci,tap]
// over (o, tap) with s*o + tap - r == p.  Covers every position of the xg frame
// (interior and margins).  One input channel per thread.
__global__ void conv_bwd_data_simt_kernel(const float* __restrict__ u, Frame uf,
                                          const float* __restrict__ w, int k, int s,
                                          float* __restrict__ xg, Frame gf) {
  const int Dz = gf.d + 2 * gf.md, Hy = gf.h + 2 * gf.mh, Wx = gf.w + 2 * gf.mw;
  const long long total = (long long)gf.n * Dz * Hy * Wx * gf.c;
  const int r = (k - 1) / 2;
  const int k3 = k * k * k;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    long long t = idx;
    const int ci = t % gf.c;
    t /= gf.c;
    const int px = t % Wx - gf.mw;
    t /= Wx;
    const int py = t % Hy - gf.mh;
    t /= Hy;
    const int pz = t % Dz - gf.md;
    const int n = t / Dz;
    float acc = 0.f;
    for (int a = 0; a < k; ++a) {
      const int qz = pz + r - a;
      if (qz < 0 || qz % s) continue;
      const int oz = qz / s;
      if (oz >= uf.d) continue;
      for (int b = 0; b < k; ++b) {
        const int qy = py + r - b;
        if (qy < 0 || qy % s) continue;
        const int oy = qy / s;
        if (oy >= uf.h) continue;
        for (int c = 0; c < k; ++c) {
          const int qx = px + r - c;
          if (qx < 0 || qx % s) continue;
          const int ox = qx / s;
          if (ox >= uf.w) continue;
          const float* up = u + fr_index(uf, n, oz, oy, ox);
          const int tap = (a * k + b) * k + c;
          for (int co = 0; co < uf.c; ++co)
            acc = fmaf(__ldg(up + co), rnd(gf, __ldg(w + ((long long)co * gf.c + ci) * k3 + tap)), acc);
        }
      }
    }
    xg[idx] = rnd(gf, acc);
  }
}

// Filter gradient partials: block (kt, ct, p) computes a 32 (tap,ci) x 32 co tile
// over voxel chunk p and writes it to part[p][co][ci][tap] (OIDHW order).
__global__ void __launch_bounds__(256) conv_wgrad_simt_kernel(
    const float* __restrict__ x, Frame xf, const float* __restrict__ u, Frame uf, int k, int s,
    long long chunk, float* __restrict__ part) {
  __shared__ float su[32][33];
  __shared__ float sx[32][33];
  const int r = (k - 1) / 2;
  const int k3 = k * k * k;
  const int KT = k3 * xf.c;  // (tap, ci) extent
  const int kt0 = blockIdx.x * 32, co0 = blockIdx.y * 32;
  const long long nvox = (long long)uf.n * uf.d * uf.h * uf.w;
  const long long v0 = blockIdx.z * chunk;
  const long long v1 = min(nvox, v0 + chunk);
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // ty: 0..7
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (long long vb = v0; vb < v1; vb += 32) {
    // load u[v][co0..co0+31] and x[v + tap][ci] for kt in tile
    for (int i = threadIdx.x; i < 32 * 32; i += 256) {
      const int vi = i >> 5, j = i & 31;
      const long long v = vb + vi;
      float uv = 0.f, xv = 0.f;
      if (v < v1) {
        long long tt = v;
        const int ox = tt % uf.w;
        tt /= uf.w;
        const int oy = tt % uf.h;
        tt /= uf.h;
        const int oz = tt % uf.d;
        const int n = tt / uf.d;
        if (co0 + j < uf.c) uv = __ldg(u + fr_index(uf, n, oz, oy, ox) + co0 + j);
        const int kt = kt0 + j;
        if (kt < KT) {
          const int tap = kt / xf.c, ci = kt % xf.c;
          const int a = tap / (k * k), b = (tap / k) % k, c = tap % k;
          const int iz = s * oz + a - r, iy = s * oy + b - r, ix = s * ox + c - r;
          if (fr_inside(xf, iz, iy, ix)) xv = __ldg(x + fr_index(xf, n, iz, iy, ix) + ci);
        }
      }
      su[vi][j] = uv;
      sx[vi][j] = xv;
    }
    __syncthreads();
#pragma unroll 8
    for (int vi = 0; vi < 32; ++vi) {
      const float xv = sx[vi][tx];
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[j] = fmaf(su[vi][ty * 4 + j], xv, acc[j]);
    }
    __syncthreads();
  }
  const int kt = kt0 + tx;
  if (kt < KT) {
    const int tap = kt / xf.c, ci = kt % xf.c;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int co = co0 + ty * 4 + j;
      if (co < uf.c)
        part[(long long)blockIdx.z * uf.c * xf.c * k3 + ((long long)co * xf.c + ci) * k3 + tap] = acc[j];
    }
  }
}

// Fixed-order sum of P partial slices part[p][len] (split-K / per-block
// partials of every filter gradient).  A block takes 32 consecutive outputs
// (coalesced rows) x 32 lanes over p: lane l sums p = l, l + 32, ... in order,
// then lane 0 adds the 32 lane sums in order -- deterministic, and a chain of
// P / 32 loads instead of P (one thread per output walking all P partials
// took 0.19 ms for P = 1184).  Output element i goes to
// out[(i / inner) * out_stride + out_off + i % inner] (inner = len: plain).
__global__ void __launch_bounds__(1024) reduce_partials_kernel(const float* __restrict__ part, int P, long long len,
                                                               int inner, long long out_stride, long long out_off,
                                                               float* __restrict__ out, int accumulate) {
  __shared__ float red[32][33];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const long long i = blockIdx.x * 32LL + tx;
  float s = 0.f;
  if (i < len) {
#pragma unroll 4
    for (int p = ty; p < P; p += 32) s += part[(long long)p * len + i];
  }
  red[ty][tx] = s;
  __syncthreads();
  if (ty == 0 && i < len) {
    float t = red[0][tx];
    for (int l = 1; l < 32; ++l) t += red[l][tx];
    float* o = out + (i / inner) * out_stride + out_off + i % inner;
    *o = accumulate ? *o + t : t;
  }
}

static int grid_for(long long total, int block) {
  long long g = (total + block - 1) / block;
  long long cap = (long long)num_sms() * 16;
  return static_cast<int>(g < cap ? (g > 0 ? g : 1) : cap);
}

int conv_fwd_simt(const float* x, const Frame& xf, const float* w, int k, int s, float* y,
                  const Frame& yf, cudaStream_t st, int act, float slope) {
  if (yf.c % 4 == 0) {
    long long total = (long long)yf.n * yf.d * yf.h * yf.w * (yf.c / 4);
    conv_fwd_simt_kernel<4><<<grid_for(total, 256), 256, 0, st>>>(x, xf, w, k, s, y, yf, act, slope);
  } else {
    long long total = (long long)yf.n * yf.d * yf.h * yf.w * yf.c;
    conv_fwd_simt_kernel<1><<<grid_for(total, 256), 256, 0, st>>>(x, xf, w, k, s, y, yf, act, slope);
  }
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}

int conv_bwd_data_simt(const float* u, const Frame& uf, const float* w, int k, int s, float* xg,
                       const Frame& gf, cudaStream_t st) {
  long long total = (long long)gf.n * (gf.d + 2 * gf.md) * (gf.h + 2 * gf.mh) *
                    (gf.w + 2 * gf.mw) * gf.c;
  conv_bwd_data_simt_kernel<<<grid_for(total, 256), 256, 0, st>>>(u, uf, w, k, s, xg, gf);
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}

long long wgrad_simt_parts(const Frame& uf) {
  const long long nvox = (long long)uf.n * uf.d * uf.h * uf.w;
  long long P = (nvox + 4095) / 4096;
  return P < 256 ? P : 256;
}

// Few partials (P <= 64): one thread per output walks them in order.
// Contiguous destination (inner == len, out_off == 0), float4 lanes, P summed
// in order -- the same sums as reduce_partials_seq_kernel.
__global__ void reduce_partials_seq4_kernel(const float4* __restrict__ part, int P, long long len4,
                                            float4* __restrict__ out, int accumulate) {
  vpx::pdl_wait();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < len4;
       i += (long long)gridDim.x * blockDim.x) {
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    int p = 0;
    for (; p + 8 <= P; p += 8) {  // eight loads in flight, summed in order
      float4 v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = part[(long long)(p + j) * len4 + i];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        s.x += v[j].x;
        s.y += v[j].y;
        s.z += v[j].z;
        s.w += v[j].w;
      }
    }
    for (; p < P; ++p) {
      const float4 v = part[(long long)p * len4 + i];
      s.x += v.x;
      s.y += v.y;
      s.z += v.z;
      s.w += v.w;
    }
    if (accumulate) {
      const float4 o = out[i];
      s = make_float4(o.x + s.x, o.y + s.y, o.z + s.z, o.w + s.w);
    }
    out[i] = s;
  }
}

__global__ void reduce_partials_seq_kernel(const float* __restrict__ part, int P, long long len, int inner,
                                           long long out_stride, long long out_off, float* __restrict__ out,
                                           int accumulate) {
  vpx::pdl_wait();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < len;
       i += (long long)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int p = 0; p < P; ++p) s += part[(long long)p * len + i];
    float* o = out + (i / inner) * out_stride + out_off + i % inner;
    *o = accumulate ? *o + s : s;
  }
}

// out[co][ci0 + ci][tap] (=|+=) sum_p part[p][tap][co][ci], p in order: one
// block per (co, 32 input channels) sums the 27 taps' 128-byte runs into
// shared memory and writes the 32 x 27 result as one contiguous run.
__global__ void reduce_partials_tapmajor_kernel(const float* __restrict__ part, int P, int cout, int cin,
                                                long long out_co_stride, int ci0, float* __restrict__ out,
                                                int accumulate) {
  __shared__ float t[32 * 27];
  const int co = blockIdx.y, cb = blockIdx.x * 32;
  const long long slice = 27LL * cout * cin;
  vpx::pdl_wait();
  for (int i = threadIdx.x; i < 32 * 27; i += blockDim.x) {
    const int tap = i >> 5, c = i & 31;
    float s = 0.f;
    if (cb + c < cin) {
      const float* src = part + ((long long)tap * cout + co) * cin + cb + c;
      int p = 0;
      for (; p + 8 <= P; p += 8) {  // eight loads in flight, summed in order
        float v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = src[(p + j) * slice];
#pragma unroll
        for (int j = 0; j < 8; ++j) s += v[j];
      }
      for (; p < P; ++p) s += src[p * slice];
    }
    t[c * 27 + tap] = s;
  }
  __syncthreads();
  const int nc = cin - cb < 32 ? cin - cb : 32;
  float* o = out + co * out_co_stride + (long long)(ci0 + cb) * 27;
  for (int i = threadIdx.x; i < nc * 27; i += blockDim.x) o[i] = accumulate ? o[i] + t[i] : t[i];
}

int reduce_partials_tapmajor(const float* part, int P, int cout, int cin, long long out_co_stride, int ci0,
                             float* out, int accumulate, cudaStream_t st) {
  VPX_CHECK_CUDA(vpx::launch_pdl(reduce_partials_tapmajor_kernel, dim3((cin + 31) / 32, cout), 256, 0, st, part, P,
                                 cout, cin, out_co_stride, ci0, out, accumulate));
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}

int reduce_partials_slice(const float* part, int P, long long len, int inner, long long out_stride,
                          long long out_off, float* out, int accumulate, cudaStream_t st) {
  if (len <= 0) return VPX_OK;
  if (P <= 64 && inner == len && out_off == 0 && len % 4 == 0 &&
      (reinterpret_cast<uintptr_t>(part) | reinterpret_cast<uintptr_t>(out)) % 16 == 0) {
    VPX_CHECK_CUDA(vpx::launch_pdl(reduce_partials_seq4_kernel, grid_for(len / 4, 256), 256, 0, st,
                                   reinterpret_cast<const float4*>(part), P, len / 4, reinterpret_cast<float4*>(out),
                                   accumulate));
    VPX_LAUNCH_CHECK();
    return VPX_OK;
  }
  if (P <= 64) {
    VPX_CHECK_CUDA(vpx::launch_pdl(reduce_partials_seq_kernel, grid_for(len, 256), 256, 0, st, part, P, len, inner,
                                   out_stride, out_off, out, accumulate));
    VPX_LAUNCH_CHECK();
    return VPX_OK;
  }
  reduce_partials_kernel<<<static_cast<unsigned>((len + 31) / 32), dim3(32, 32), 0, st>>>(
      part, P, len, inner, out_stride, out_off, out, accumulate);
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}

int reduce_partials(const float* part, int P, long long len, float* out, int accumulate,
                    cudaStream_t st) {
  return reduce_partials_slice(part, P, len, static_cast<int>(len), 0, 0, out, accumulate, st);
}

int conv_wgrad_simt(const float* x, const Frame& xf, const float* u, const Frame& uf, int k, int s,
                    float* wg, int accumulate, float* part, cudaStream_t st) {
  const int k3 = k * k * k;
  const long long nvox = (long long)uf.n * uf.d * uf.h * uf.w;
  const long long P = wgrad_simt_parts(uf);
  const long long chunk = ((nvox + P - 1) / P + 31) / 32 * 32;
  const int Pn = static_cast<int>((nvox + chunk - 1) / chunk);
  dim3 grid((k3 * xf.c + 31) / 32, (uf.c + 31) / 32, Pn);
  conv_wgrad_simt_kernel<<<grid, 256, 0, st>>>(x, xf, u, uf, k, s, chunk, part);
  VPX_LAUNCH_CHECK();
  const long long len = (long long)uf.c * xf.c * k3;
  return reduce_partials(part, Pn, len, wg, accumulate, st);
}

}  // namespace vpx
