// Memory-bound kernels of the training step: LeakyReLU, 2^3 pooling, batch
// norm statistics/apply/backward, channel concat, k2s2 transposed conv, halo
// pack/unpack, the pinned splitmix64 PRNG, Adam/SGD, losses, layout moves.
//
// All activations are NDHWC halo frames (Frame = {n,c,d,h,w,md,mh,mw}); every
// kernel reads/writes frame interiors through fr_off() so producers can write
// straight into their consumer's halo-wide frame (no reference-style _wrap
// copy, reference layers/distributed.py:31-33).  Reductions are deterministic:
// fixed block partition + fixed-order final sum, accumulated in fp64.
#include <cstdlib>

#include "conv_common.h"
#include "conv_simt.h"
#include "ops_vec.h"
#include "vpx_round.cuh"
#include "vpx_host.h"

namespace vpx {

struct VoxIdx {
  int n, z, y, x;
};

__device__ __forceinline__ VoxIdx vox_decode(long long v, const Frame& f) {
  VoxIdx r;
  r.x = v % f.w;
  v /= f.w;
  r.y = v % f.h;
  v /= f.h;
  r.z = v % f.d;
  r.n = static_cast<int>(v / f.d);
  return r;
}
// Element offset of interior voxel (n,z,y,x) channel 0 in frame f.
__device__ __forceinline__ long long fr_off(const Frame& f, int n, int z, int y, int x) {
  return ((((long long)n * (f.d + 2 * f.md) + (z + f.md)) * (f.h + 2 * f.mh) + (y + f.mh)) *
              (f.w + 2 * f.mw) +
          (x + f.mw)) *
         f.c;
}
__device__ __forceinline__ long long vox_count(const Frame& f) {
  return (long long)f.n * f.d * f.h * f.w;
}

static int grid1d(long long total, int block = 256) {
  long long g = (total + block - 1) / block;
  long long cap = (long long)num_sms() * 32;
  if (g < 1) g = 1;
  return static_cast<int>(g < cap ? g : cap);
}

#define GRID_STRIDE(i, total)                                                         \
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (total); \
       i += (long long)gridDim.x * blockDim.x)

// ------------------------------------------------------------------ leaky
// reference layers/reference.py:231-236: x >= 0 ? x : slope*x; bwd passes u at x == 0.
__global__ void leaky_fwd_kernel(const float* __restrict__ x, Frame xf, float* __restrict__ y,
                                 Frame yf, float slope) {
  const long long total = vox_count(xf) * xf.c;
  GRID_STRIDE(i, total) {
    const int c = i % xf.c;
    const VoxIdx v = vox_decode(i / xf.c, xf);
    const float a = x[fr_off(xf, v.n, v.z, v.y, v.x) + c];
    y[fr_off(yf, v.n, v.z, v.y, v.x) + c] = rnd(yf, a >= 0.f ? a : slope * a);
  }
}
__global__ void leaky_bwd_kernel(const float* __restrict__ x, Frame xf, const float* __restrict__ u,
                                 Frame uf, float* __restrict__ g, Frame gf, float slope) {
  const long long total = vox_count(xf) * xf.c;
  GRID_STRIDE(i, total) {
    const int c = i % xf.c;
    const VoxIdx v = vox_decode(i / xf.c, xf);
    const float a = x[fr_off(xf, v.n, v.z, v.y, v.x) + c];
    const float b = u[fr_off(uf, v.n, v.z, v.y, v.x) + c];
    g[fr_off(gf, v.n, v.z, v.y, v.x) + c] = rnd(gf, a >= 0.f ? b : slope * b);
  }
}

// ------------------------------------------------------------------- pool
// reference layers/reference.py:149-183: 2^3 stride 2, window flattened in
// (d,h,w) C order, max ties -> lowest linear index; avg bwd = u/8 broadcast.
__global__ void pool_fwd_kernel(const float* __restrict__ x, Frame xf, float* __restrict__ y,
                                Frame yf, int is_max) {
  const long long total = vox_count(yf) * yf.c;
  GRID_STRIDE(i, total) {
    const int c = i % yf.c;
    const VoxIdx o = vox_decode(i / yf.c, yf);
    float best = 0.f, sum = 0.f;
    int first = 1;
    for (int w8 = 0; w8 < 8; ++w8) {
      const int a = w8 >> 2, b = (w8 >> 1) & 1, cc = w8 & 1;
      const float val = x[fr_off(xf, o.n, 2 * o.z + a, 2 * o.y + b, 2 * o.x + cc) + c];
      if (first || val > best) best = val;
      first = 0;
      sum += val;
    }
    y[fr_off(yf, o.n, o.z, o.y, o.x) + c] = rnd(yf, is_max ? best : sum / 8.0f);
  }
}
__global__ void pool_bwd_kernel(const float* __restrict__ x, Frame xf, const float* __restrict__ u,
                                Frame uf, float* __restrict__ g, Frame gf, int is_max) {
  const long long total = vox_count(uf) * uf.c;
  GRID_STRIDE(i, total) {
    const int c = i % uf.c;
    const VoxIdx o = vox_decode(i / uf.c, uf);
    const float uv = u[fr_off(uf, o.n, o.z, o.y, o.x) + c];
    int arg = 0;
    if (is_max) {
      float best = 0.f;
      for (int w8 = 0; w8 < 8; ++w8) {
        const int a = w8 >> 2, b = (w8 >> 1) & 1, cc = w8 & 1;
        const float val = x[fr_off(xf, o.n, 2 * o.z + a, 2 * o.y + b, 2 * o.x + cc) + c];
        if (w8 == 0 || val > best) {
          best = val;
          arg = w8;
        }
      }
    }
    const float avg = uv / 8.0f;
    for (int w8 = 0; w8 < 8; ++w8) {
      const int a = w8 >> 2, b = (w8 >> 1) & 1, cc = w8 & 1;
      g[fr_off(gf, o.n, 2 * o.z + a, 2 * o.y + b, 2 * o.x + cc) + c] =
          rnd(gf, is_max ? (w8 == arg ? uv : 0.f) : avg);
    }
  }
}

// -------------------------------------------------------------- batchnorm
// Per-channel partial sums over a fixed voxel partition (deterministic).
// mode 0: (sum x, sum x^2); mode 1: (sum u, sum u*xhat) with xhat=(x-mean)*inv.
constexpr int kBnParts = 1184;  // 8 blocks per SM: enough loads in flight for HBM

__global__ void bn_partial_kernel(const float* __restrict__ x, Frame xf, const float* __restrict__ u,
                                  Frame uf, const float* __restrict__ mean,
                                  const float* __restrict__ inv, int mode,
                                  double* __restrict__ part) {
  // block p handles voxels [p*chunk, (p+1)*chunk); threads stride channels x voxels
  const int C = xf.c;
  const long long nv = vox_count(xf);
  const long long chunk = (nv + gridDim.x - 1) / gridDim.x;
  const long long v0 = blockIdx.x * chunk, v1 = min(nv, v0 + chunk);
  extern __shared__ double sh[];  // [2][blockDim.x]
  const int lanes_per_c = blockDim.x / C > 0 ? blockDim.x / C : 1;
  const int c = threadIdx.x % C;
  const int lane = threadIdx.x / C;
  double s1 = 0.0, s2 = 0.0;
  if (threadIdx.x < lanes_per_c * C) {
    for (long long v = v0 + lane; v < v1; v += lanes_per_c) {
      const VoxIdx q = vox_decode(v, xf);
      const float a = x[fr_off(xf, q.n, q.z, q.y, q.x) + c];
      if (mode == 0) {
        s1 += a;
        s2 += (double)a * a;
      } else {
        const float b = u[fr_off(uf, q.n, q.z, q.y, q.x) + c];
        const float xh = (a - mean[c]) * inv[c];
        s1 += b;
        s2 += (double)b * xh;
      }
    }
  }
  sh[threadIdx.x] = s1;
  sh[blockDim.x + threadIdx.x] = s2;
  __syncthreads();
  if (threadIdx.x < C) {
    double t1 = 0.0, t2 = 0.0;
    for (int l = 0; l < lanes_per_c; ++l) {
      t1 += sh[l * C + threadIdx.x];
      t2 += sh[blockDim.x + l * C + threadIdx.x];
    }
    part[(long long)blockIdx.x * 2 * C + threadIdx.x] = t1;
    part[(long long)blockIdx.x * 2 * C + C + threadIdx.x] = t2;
  }
}
// One block per statistic (2C blocks): 256 strided partial sums, then a
// fixed-order shared-memory tree -- deterministic, and the P partials are
// read in parallel instead of by one thread per statistic in sequence (that
// serial walk over P = 1184 partials used to cost ~0.2 ms per BN call).
__global__ void __launch_bounds__(256) bn_finish_kernel(const double* __restrict__ part, int P, int C,
                                                        float* __restrict__ out2c) {
  __shared__ double sh[256];
  const int i = blockIdx.x;
  double s = 0.0;
  for (int p = threadIdx.x; p < P; p += 256) s += part[(long long)p * 2 * C + i];
  sh[threadIdx.x] = s;
  __syncthreads();
#pragma unroll
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out2c[i] = static_cast<float>(sh[0]);
}
// y = gamma*(x-mean)*inv + beta (reference layers/reference.py:206-214)
__global__ void bn_apply_kernel(const float* __restrict__ x, Frame xf, const float* __restrict__ mean,
                                const float* __restrict__ inv, const float* __restrict__ gamma,
                                const float* __restrict__ beta, float* __restrict__ y, Frame yf) {
  const long long total = vox_count(xf) * xf.c;
  GRID_STRIDE(i, total) {
    const int c = i % xf.c;
    const VoxIdx v = vox_decode(i / xf.c, xf);
    const float xh = (x[fr_off(xf, v.n, v.z, v.y, v.x) + c] - mean[c]) * inv[c];
    y[fr_off(yf, v.n, v.z, v.y, v.x) + c] = rnd(yf, gamma[c] * xh + beta[c]);
  }
}
// dx = gamma*inv*(u - (sum_u + xhat*sum_uxhat)/count) (reference layers/reference.py:217-226)
__global__ void bn_bwd_apply_kernel(const float* __restrict__ x, Frame xf, const float* __restrict__ u,
                                    Frame uf, const float* __restrict__ mean,
                                    const float* __restrict__ inv, const float* __restrict__ gamma,
                                    const float* __restrict__ sums, float inv_count,
                                    float* __restrict__ g, Frame gf) {
  const int C = xf.c;
  const long long total = vox_count(xf) * C;
  GRID_STRIDE(i, total) {
    const int c = i % C;
    const VoxIdx v = vox_decode(i / C, xf);
    const float xh = (x[fr_off(xf, v.n, v.z, v.y, v.x) + c] - mean[c]) * inv[c];
    const float b = u[fr_off(uf, v.n, v.z, v.y, v.x) + c];
    g[fr_off(gf, v.n, v.z, v.y, v.x) + c] =
        rnd(gf, gamma[c] * inv[c] * (b - (sums[c] + xh * sums[C + c]) * inv_count));
  }
}
// mean/var from allreduced sums; running stats update (reference layers/reference.py:188-204)
__global__ void bn_stats_kernel(const float* __restrict__ sums, int C, double count, float eps,
                                float momentum, float* __restrict__ mean, float* __restrict__ inv,
                                float* __restrict__ run_mean, float* __restrict__ run_var) {
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    const double m = (double)sums[c] / count;
    double var = (double)sums[C + c] / count - m * m;
    if (var < 0) var = 0;
    mean[c] = static_cast<float>(m);
    inv[c] = static_cast<float>(1.0 / sqrt(var + eps));
    if (run_mean) run_mean[c] = momentum * run_mean[c] + (1.f - momentum) * static_cast<float>(m);
    if (run_var) run_var[c] = momentum * run_var[c] + (1.f - momentum) * static_cast<float>(var);
  }
}

// ----------------------------------------------------------------- concat
__global__ void concat_kernel(const float* __restrict__ a, Frame af, const float* __restrict__ b,
                              Frame bf, float* __restrict__ y, Frame yf) {
  const long long total = vox_count(yf) * yf.c;
  GRID_STRIDE(i, total) {
    const int c = i % yf.c;
    const VoxIdx v = vox_decode(i / yf.c, yf);
    const float val = c < af.c ? a[fr_off(af, v.n, v.z, v.y, v.x) + c]
                               : b[fr_off(bf, v.n, v.z, v.y, v.x) + c - af.c];
    y[fr_off(yf, v.n, v.z, v.y, v.x) + c] = rnd(yf, val);
  }
}
// split gradient of a concat: ga (+)= u[:, :ca], gb (+)= u[:, ca:]
__global__ void split_kernel(const float* __restrict__ u, Frame uf, float* __restrict__ ga, Frame gaf,
                             float* __restrict__ gb, Frame gbf, int acc_b) {
  const long long total = vox_count(uf) * uf.c;
  GRID_STRIDE(i, total) {
    const int c = i % uf.c;
    const VoxIdx v = vox_decode(i / uf.c, uf);
    const float val = u[fr_off(uf, v.n, v.z, v.y, v.x) + c];
    if (c < gaf.c) {
      ga[fr_off(gaf, v.n, v.z, v.y, v.x) + c] = val;
    } else {
      float* p = gb + fr_off(gbf, v.n, v.z, v.y, v.x) + c - gaf.c;
      *p = rnd(gbf, acc_b ? *p + val : val);
    }
  }
}
// y (+)= x over frame interiors
__global__ void add_kernel(const float* __restrict__ x, Frame xf, float* __restrict__ y, Frame yf) {
  const long long total = vox_count(xf) * xf.c;
  GRID_STRIDE(i, total) {
    const int c = i % xf.c;
    const VoxIdx v = vox_decode(i / xf.c, xf);
    float* q = y + fr_off(yf, v.n, v.z, v.y, v.x) + c;
    *q = rnd(yf, *q + x[fr_off(xf, v.n, v.z, v.y, v.x) + c]);
  }
}
__global__ void copy_kernel(const float* __restrict__ x, Frame xf, float* __restrict__ y, Frame yf) {
  const long long total = vox_count(xf) * xf.c;
  GRID_STRIDE(i, total) {
    const int c = i % xf.c;
    const VoxIdx v = vox_decode(i / xf.c, xf);
    y[fr_off(yf, v.n, v.z, v.y, v.x) + c] = x[fr_off(xf, v.n, v.z, v.y, v.x) + c];
  }
}

// ------------------------------------------------- transposed conv k2 s2
// reference layers/reference.py:99-144; w is (cin, cout, 2,2,2).
__global__ void deconv_fwd_kernel(const float* __restrict__ x, Frame xf, const float* __restrict__ w,
                                  float* __restrict__ y, Frame yf) {
  const long long total = vox_count(yf) * yf.c;
  GRID_STRIDE(i, total) {
    const int co = i % yf.c;
    const VoxIdx o = vox_decode(i / yf.c, yf);
    const int k = ((o.z & 1) * 2 + (o.y & 1)) * 2 + (o.x & 1);
    const float* xp = x + fr_off(xf, o.n, o.z >> 1, o.y >> 1, o.x >> 1);
    float acc = 0.f;
    for (int ci = 0; ci < xf.c; ++ci) acc = fmaf(xp[ci], rnd(yf, w[((long long)ci * yf.c + co) * 8 + k]), acc);
    y[fr_off(yf, o.n, o.z, o.y, o.x) + co] = rnd(yf, acc);
  }
}
__global__ void deconv_bwd_data_kernel(const float* __restrict__ u, Frame uf,
                                       const float* __restrict__ w, float* __restrict__ g, Frame gf) {
  const long long total = vox_count(gf) * gf.c;
  GRID_STRIDE(i, total) {
    const int ci = i % gf.c;
    const VoxIdx p = vox_decode(i / gf.c, gf);
    float acc = 0.f;
    for (int k = 0; k < 8; ++k) {
      const int a = k >> 2, b = (k >> 1) & 1, c = k & 1;
      const float* up = u + fr_off(uf, p.n, 2 * p.z + a, 2 * p.y + b, 2 * p.x + c);
      for (int co = 0; co < uf.c; ++co) acc = fmaf(up[co], rnd(gf, w[((long long)ci * uf.c + co) * 8 + k]), acc);
    }
    g[fr_off(gf, p.n, p.z, p.y, p.x) + ci] = rnd(gf, acc);
  }
}
// wg[ci][co][k] partial over voxel chunks -> part[p][ci][co][k]
__global__ void deconv_wgrad_kernel(const float* __restrict__ x, Frame xf, const float* __restrict__ u,
                                    Frame uf, long long chunk, float* __restrict__ part) {
  const int len = xf.c * uf.c * 8;
  const long long nv = vox_count(xf);
  const long long v0 = blockIdx.y * chunk, v1 = min(nv, v0 + chunk);
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < len; e += gridDim.x * blockDim.x) {
    const int k = e % 8, co = (e / 8) % uf.c, ci = e / (8 * uf.c);
    const int a = k >> 2, b = (k >> 1) & 1, c = k & 1;
    float acc = 0.f;
    for (long long v = v0; v < v1; ++v) {
      const VoxIdx q = vox_decode(v, xf);
      acc = fmaf(x[fr_off(xf, q.n, q.z, q.y, q.x) + ci],
                 u[fr_off(uf, q.n, 2 * q.z + a, 2 * q.y + b, 2 * q.x + c) + co], acc);
    }
    part[(long long)blockIdx.y * len + e] = acc;
  }
}
__global__ void reduce_parts_kernel(const float* __restrict__ part, int P, long long len,
                                    float* __restrict__ out, int accumulate) {
  GRID_STRIDE(i, len) {
    float s = 0.f;
    for (int p = 0; p < P; ++p) s += part[(long long)p * len + i];
    out[i] = accumulate ? out[i] + s : s;
  }
}

// ------------------------------------------------------------------- halo
// Copy a box of a frame (frame coordinates, i.e. margins included; samples
// n0..n0+en) to/from a dense buffer in (n, z, y, x, c) C order.
// mode 0: pack, 1: unpack, 2: unpack-add.
__global__ void halo_copy_kernel(float* __restrict__ fr, Frame f, int n0, int z0, int y0, int x0,
                                 int en, int ez, int ey, int ex, float* __restrict__ buf, int mode) {
  const long long total = (long long)en * ez * ey * ex * f.c;
  const long long Wf = f.w + 2 * f.mw, Hf = f.h + 2 * f.mh, Df = f.d + 2 * f.md;
  GRID_STRIDE(i, total) {
    long long t = i;
    const int c = t % f.c;
    t /= f.c;
    const int x = t % ex;
    t /= ex;
    const int y = t % ey;
    t /= ey;
    const int z = t % ez;
    const int n = n0 + static_cast<int>(t / ez);
    const long long off = ((((long long)n * Df + z0 + z) * Hf + y0 + y) * Wf + x0 + x) * f.c + c;
    if (mode == 0)
      buf[i] = fr[off];
    else if (mode == 1)
      fr[off] = buf[i];
    else
      fr[off] += buf[i];
  }
}

// -------------------------------------------------------------------- prng
// splitmix64 counter streams (reference prng.py:28-90).  uniform in fp64:
// lo + (hi-lo) * ((u64 >> 11) * 2^-53), computed with explicit non-fused ops so
// the result is bit-identical to numpy's.
__device__ __forceinline__ uint64_t sm_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
__global__ void prng_uniform_kernel(uint64_t key, long long n, double lo, double hi,
                                    float* __restrict__ out32, double* __restrict__ out64) {
  GRID_STRIDE(i, n) {
    const uint64_t r = sm_mix(key + (static_cast<uint64_t>(i) + 1ULL) * 0x9E3779B97F4A7C15ULL);
    const double u01 = __dmul_rn(static_cast<double>(r >> 11), 1.1102230246251565e-16);
    const double v = __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), u01));
    if (out32) out32[i] = static_cast<float>(v);
    if (out64) out64[i] = v;
  }
}
// keep-mask (uniform01 < keep) for counters base + i
__global__ void prng_mask_kernel(uint64_t key, long long n, double keep, uint8_t* __restrict__ out) {
  GRID_STRIDE(i, n) {
    const uint64_t r = sm_mix(key + (static_cast<uint64_t>(i) + 1ULL) * 0x9E3779B97F4A7C15ULL);
    const double u01 = __dmul_rn(static_cast<double>(r >> 11), 1.1102230246251565e-16);
    out[i] = u01 < keep ? 1 : 0;
  }
}
// y = lo + (hi-lo)*uniform placed into an NDHWC frame from an NCDHW-ordered stream
__global__ void prng_volume_kernel(uint64_t key, Frame f, long long counter_base, double lo, double hi,
                                   float* __restrict__ fr) {
  const long long total = vox_count(f) * f.c;
  GRID_STRIDE(i, total) {
    // i enumerates NCDHW order of the interior: (n, c, z, y, x)
    long long t = i;
    const int x = t % f.w;
    t /= f.w;
    const int y = t % f.h;
    t /= f.h;
    const int z = t % f.d;
    t /= f.d;
    const int c = t % f.c;
    const int n = t / f.c;
    const uint64_t ctr = static_cast<uint64_t>(counter_base + i);
    const uint64_t r = sm_mix(key + (ctr + 1ULL) * 0x9E3779B97F4A7C15ULL);
    const double u01 = __dmul_rn(static_cast<double>(r >> 11), 1.1102230246251565e-16);
    const double v = __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), u01));
    fr[fr_off(f, n, z, y, x) + c] = rnd(f, static_cast<float>(v));
  }
}

// --------------------------------------------------------------- optimizer
// In-place bias-corrected Adam (reference model/optim.py:71-88), fp32 like the
// reference's fp32 path; c1 = 1-b1^t, c2 = 1-b2^t precomputed on the host.
__global__ void adam_kernel(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                            float* __restrict__ v, long long n, float lr, float b1, float b2,
                            float c1, float c2, float eps) {
  GRID_STRIDE(i, n) {
    const float gi = g[i];
    float mi = m[i] * b1;
    mi = mi + (1.f - b1) * gi;
    float vi = v[i] * b2;
    vi = vi + (1.f - b2) * (gi * gi);
    m[i] = mi;
    v[i] = vi;
    p[i] = p[i] - lr * (mi / c1) / (sqrtf(vi / c2) + eps);
  }
}
// Same update with lr, 1-b1^t, 1-b2^t read from device memory (hyper = {lr, c1,
// c2}): the step can be captured once in a CUDA graph and replayed with the
// per-step scalars rewritten in place.
__global__ void adam_dev_kernel(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                                float* __restrict__ v, long long n, const float* __restrict__ hyper, float b1,
                                float b2, float eps) {
  const float lr = hyper[0], c1 = hyper[1], c2 = hyper[2];
  GRID_STRIDE(i, n) {
    const float gi = g[i];
    float mi = m[i] * b1;
    mi = mi + (1.f - b1) * gi;
    float vi = v[i] * b2;
    vi = vi + (1.f - b2) * (gi * gi);
    m[i] = mi;
    v[i] = vi;
    p[i] = p[i] - lr * (mi / c1) / (sqrtf(vi / c2) + eps);
  }
}
__global__ void prng_mask_dev_kernel(const uint64_t* __restrict__ keyp, long long n, double keep,
                                     uint8_t* __restrict__ out) {
  const uint64_t key = *keyp;
  GRID_STRIDE(i, n) {
    const uint64_t r = sm_mix(key + (static_cast<uint64_t>(i) + 1ULL) * 0x9E3779B97F4A7C15ULL);
    const double u01 = __dmul_rn(static_cast<double>(r >> 11), 1.1102230246251565e-16);
    out[i] = u01 < keep ? 1 : 0;
  }
}
// ---- peer-memory halo mailboxes (comm.py PeerHalo) -------------------------
// The sender packs its face straight into the neighbour's mailbox over NVLink
// (vpx_halo_copy with a peer pointer), then bumps the neighbour's arrival
// counter; the receiver waits for its counter and unpacks from local memory.
__global__ void peer_signal_kernel(unsigned long long* peer_flag) {
  __threadfence_system();
  atomicAdd_system(peer_flag, 1ULL);
}
__global__ void peer_wait_kernel(const unsigned long long* flag, unsigned long long* expected,
                                 long long timeout_ns, int* error) {
  const unsigned long long want = *expected + 1ULL;
  long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
    if (v >= want) break;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > timeout_ns) {  // the neighbour never arrived: fail loudly instead of hanging
      *error = 1;
      __threadfence_system();
      asm volatile("trap;");
    }
    __nanosleep(64);
  }
  *expected = want;
  __threadfence_system();
}
__global__ void sgd_kernel(float* __restrict__ p, const float* __restrict__ g, long long n, float lr) {
  GRID_STRIDE(i, n) p[i] = p[i] - lr * g[i];
}

// ------------------------------------------------------------------ losses
// per-voxel softmax cross entropy over K channels; labels int64 (n, d, h, w).
// writes dlogits = (softmax - onehot) / count into g and per-block loss partials.
__global__ void xent_kernel(const float* __restrict__ logits, Frame lf, const long long* __restrict__ lab,
                            double inv_count, float* __restrict__ g, Frame gf, double* __restrict__ part) {
  const long long nv = vox_count(lf);
  const int K = lf.c;
  double local = 0.0;
  GRID_STRIDE(v, nv) {
    const VoxIdx q = vox_decode(v, lf);
    const float* lp = logits + fr_off(lf, q.n, q.z, q.y, q.x);
    float mx = lp[0];
    for (int k = 1; k < K; ++k) mx = fmaxf(mx, lp[k]);
    float se = 0.f;
    for (int k = 0; k < K; ++k) se += expf(lp[k] - mx);
    const float lse = logf(se);
    const long long y = lab[v];
    local -= (double)(lp[y] - mx - lse);
    float* gp = g + fr_off(gf, q.n, q.z, q.y, q.x);
    for (int k = 0; k < K; ++k) {
      const float pr = expf(lp[k] - mx - lse);
      gp[k] = rnd(gf, static_cast<float>((pr - (k == y ? 1.f : 0.f)) * inv_count));
    }
  }
  __shared__ double sh[256];
  sh[threadIdx.x] = local;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

// Two classes on margin-free frames (the U-Net head): two voxels per thread
// as one float4 of logits, one 16-byte label pair and one float4 of
// gradients -- no per-voxel index decode, same per-voxel arithmetic (and bits)
// as xent_kernel.
__global__ void xent2_flat_kernel(const float4* __restrict__ logits, const longlong2* __restrict__ lab,
                                  long long npairs, double inv_count, float4* __restrict__ g, Frame gf,
                                  double* __restrict__ part) {
  double local = 0.0;
  GRID_STRIDE(i, npairs) {
    const float4 l = logits[i];
    const longlong2 y = lab[i];
    float out[4];
    const float lv[2][2] = {{l.x, l.y}, {l.z, l.w}};
    const long long yv[2] = {y.x, y.y};
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const float mx = fmaxf(lv[v][0], lv[v][1]);
      float se = 0.f;
      se += expf(lv[v][0] - mx);
      se += expf(lv[v][1] - mx);
      const float lse = logf(se);
      local -= (double)(lv[v][yv[v]] - mx - lse);
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const float pr = expf(lv[v][k] - mx - lse);
        out[2 * v + k] = rnd(gf, static_cast<float>((pr - (k == yv[v] ? 1.f : 0.f)) * inv_count));
      }
    }
    g[i] = make_float4(out[0], out[1], out[2], out[3]);
  }
  __shared__ double sh[256];
  sh[threadIdx.x] = local;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

// ------------------------------------------------------------------ layout
// NCDHW dense <-> NDHWC frame interior.
__global__ void ncdhw_to_frame_kernel(const float* __restrict__ src, Frame f, float* __restrict__ fr) {
  const long long total = vox_count(f) * f.c;
  GRID_STRIDE(i, total) {
    long long t = i;
    const int x = t % f.w;
    t /= f.w;
    const int y = t % f.h;
    t /= f.h;
    const int z = t % f.d;
    t /= f.d;
    const int c = t % f.c;
    const int n = t / f.c;
    fr[fr_off(f, n, z, y, x) + c] = rnd(f, src[i]);
  }
}
// int16 NCDHW (the HSB1 storage dtype, reference datastore.py:10-19) -> fp32
// frame interior: the datastore's conversion to the training dtype
// (reference datastore.py:429-444) fused into the layout change.  Blocks
// stride over (n, z, y) rows; a thread takes 4 consecutive voxels: one 4-wide
// vector load per channel plane, a 4x4 register transpose, four 16-byte
// stores of 4 channels (C % 4 == 0, W % 4 == 0; the scalar loop otherwise).
// One voxel per thread with scalar loads left this HBM-bound kernel at
// ~1.75 TB/s (1.5 ms per 512^3 x 4 sample, the e2e step's largest addition).
template <typename T> struct Vec4;
template <> struct Vec4<int8_t> { using type = char4; };
template <> struct Vec4<int16_t> { using type = short4; };
template <> struct Vec4<float> { using type = float4; };

template <typename T>  // int16 (HSB1 storage), int8 (the datastore's narrowed transfer copy) or fp32
__global__ void ncdhw_vec_to_frame_kernel(const T* __restrict__ src, Frame f, float* __restrict__ fr) {
  using V = typename Vec4<T>::type;
  const long long nrows = (long long)f.n * f.d * f.h;
  const long long plane = (long long)f.d * f.h * f.w;
  const int w4 = f.w / 4;
  for (long long row = blockIdx.x; row < nrows; row += gridDim.x) {
    const int y = static_cast<int>(row % f.h);
    const long long t = row / f.h;
    const int z = static_cast<int>(t % f.d);
    const int n = static_cast<int>(t / f.d);
    const T* s = src + (((long long)n * f.c * f.d + z) * f.h + y) * f.w;
    float* dst = fr + fr_off(f, n, z, y, 0);
    for (int q = threadIdx.x; q < w4; q += blockDim.x) {
      for (int c = 0; c < f.c; c += 4) {
        V v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = reinterpret_cast<const V*>(s + (c + k) * plane)[q];
        float* d = dst + (long long)(4 * q) * f.c + c;
        *reinterpret_cast<float4*>(d) = rnd4(f, make_float4(v[0].x, v[1].x, v[2].x, v[3].x));
        *reinterpret_cast<float4*>(d + f.c) = rnd4(f, make_float4(v[0].y, v[1].y, v[2].y, v[3].y));
        *reinterpret_cast<float4*>(d + 2 * f.c) = rnd4(f, make_float4(v[0].z, v[1].z, v[2].z, v[3].z));
        *reinterpret_cast<float4*>(d + 3 * f.c) = rnd4(f, make_float4(v[0].w, v[1].w, v[2].w, v[3].w));
      }
    }
  }
}

template <typename T>  // the general shape (C or W not a multiple of 4)
__global__ void ncdhw_int_to_frame_kernel(const T* __restrict__ src, Frame f, float* __restrict__ fr) {
  const long long nrows = (long long)f.n * f.d * f.h;
  const long long plane = (long long)f.d * f.h * f.w;
  for (long long row = blockIdx.x; row < nrows; row += gridDim.x) {
    const int y = static_cast<int>(row % f.h);
    const long long t = row / f.h;
    const int z = static_cast<int>(t % f.d);
    const int n = static_cast<int>(t / f.d);
    const T* s = src + (((long long)n * f.c * f.d + z) * f.h + y) * f.w;
    float* dst = fr + fr_off(f, n, z, y, 0);
    for (int x = threadIdx.x; x < f.w; x += blockDim.x)
      for (int c = 0; c < f.c; ++c) dst[(long long)x * f.c + c] = rnd(f, static_cast<float>(s[c * plane + x]));
  }
}

// Lane `src` of the warp holds 4 consecutive voxels of one channel plane in a
// packed vector; return voxel j of it (all lanes take part in the shuffles).
__device__ __forceinline__ float shfl_voxel(char4 v, int src, int j) {
  const int w = __shfl_sync(0xffffffffu, *reinterpret_cast<int*>(&v), src);
  return static_cast<float>(static_cast<signed char>(w >> (8 * j)));
}
__device__ __forceinline__ float shfl_voxel(short4 v, int src, int j) {
  const int lo = __shfl_sync(0xffffffffu, *reinterpret_cast<int*>(&v.x), src);
  const int hi = __shfl_sync(0xffffffffu, *reinterpret_cast<int*>(&v.z), src);
  return static_cast<float>(static_cast<short>((j < 2 ? lo : hi) >> (16 * (j & 1))));
}

// C == 4 (the CosmoFlow input, reference datastore.py:10-19 channels), int8 or
// int16: a warp loads 128 consecutive voxels as one 4-wide vector per lane and
// channel plane, then writes them back as four fully coalesced 512-byte runs
// of float4 (lane L of run k stores voxel 32k + L, gathered with shuffles), so
// every 32-byte sector is written whole by one instruction.
template <typename T>
__global__ void ncdhw_c4_to_frame_kernel(const T* __restrict__ src, Frame f, float* __restrict__ fr) {
  using V = typename Vec4<T>::type;
  const long long nrows = (long long)f.n * f.d * f.h;
  const long long plane = (long long)f.d * f.h * f.w;
  const int w4 = f.w / 4, lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  for (long long row = blockIdx.x; row < nrows; row += gridDim.x) {
    const int y = static_cast<int>(row % f.h);
    const long long t = row / f.h;
    const int z = static_cast<int>(t % f.d);
    const int n = static_cast<int>(t / f.d);
    const T* s = src + (((long long)n * 4 * f.d + z) * f.h + y) * f.w;
    float4* dst = reinterpret_cast<float4*>(fr + fr_off(f, n, z, y, 0));
    for (int q0 = 32 * warp; q0 < w4; q0 += 32 * nwarps) {
      const int q = q0 + lane;
      V v[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (q < w4) {
          v[c] = reinterpret_cast<const V*>(s + c * plane)[q];
        } else {
          v[c] = V{};
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int sl = 8 * k + (lane >> 2), j = lane & 3;
        const float4 o = make_float4(shfl_voxel(v[0], sl, j), shfl_voxel(v[1], sl, j), shfl_voxel(v[2], sl, j),
                                     shfl_voxel(v[3], sl, j));
        const int x = 4 * q0 + 32 * k + lane;
        if (x < f.w) dst[x] = rnd4(f, o);
      }
    }
  }
}

// C == 1 (the U-Net input): NCDHW and NDHWC coincide, a vectorised convert.
template <typename T>
__global__ void ncdhw_c1_to_frame_kernel(const T* __restrict__ src, Frame f, float* __restrict__ fr) {
  using V = typename Vec4<T>::type;
  const long long nrows = (long long)f.n * f.d * f.h;
  const int w4 = f.w / 4;
  for (long long row = blockIdx.x; row < nrows; row += gridDim.x) {
    const int y = static_cast<int>(row % f.h);
    const long long t = row / f.h;
    const int z = static_cast<int>(t % f.d);
    const int n = static_cast<int>(t / f.d);
    const V* s = reinterpret_cast<const V*>(src + (((long long)n * f.d + z) * f.h + y) * f.w);
    float4* dst = reinterpret_cast<float4*>(fr + fr_off(f, n, z, y, 0));
    for (int q = threadIdx.x; q < w4; q += blockDim.x) {
      const V v = s[q];
      dst[q] = rnd4(f, make_float4(v.x, v.y, v.z, v.w));
    }
  }
}

template <typename T>
static int layout_to_frame(const T* src, const Frame& f, float* fr, cudaStream_t st) {
  const long long rows = (long long)f.n * f.d * f.h;
  const long long cap = (long long)num_sms() * 16;
  const int grid = static_cast<int>(rows < cap ? rows : cap);
  const bool vec = f.c % 4 == 0 && f.w % 4 == 0 && (reinterpret_cast<uintptr_t>(src) % (4 * sizeof(T))) == 0;
  static const bool plain = getenv("VPX_LAYOUT_PLAIN") != nullptr;  // A/B switch (tools/e2e_probe.py)
  if constexpr (sizeof(T) < 4) {
    if (vec && f.c == 4 && !plain) {
      ncdhw_c4_to_frame_kernel<T><<<grid, 128, 0, st>>>(src, f, fr);
      VPX_LAUNCH_CHECK();
      return VPX_OK;
    }
  }
  if (vec)
    ncdhw_vec_to_frame_kernel<T><<<grid, 128, 0, st>>>(src, f, fr);
  else if (f.c == 1 && f.w % 4 == 0 && f.mw % 4 == 0 && (reinterpret_cast<uintptr_t>(src) % (4 * sizeof(T))) == 0)
    ncdhw_c1_to_frame_kernel<T><<<grid, 128, 0, st>>>(src, f, fr);
  else
    ncdhw_int_to_frame_kernel<T><<<grid, 256, 0, st>>>(src, f, fr);
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}
__global__ void i16_to_i64_kernel(const int16_t* __restrict__ src, long long n, long long* __restrict__ dst) {
  GRID_STRIDE(i, n) dst[i] = src[i];
}
__global__ void frame_to_ncdhw_kernel(const float* __restrict__ fr, Frame f, float* __restrict__ dst) {
  const long long total = vox_count(f) * f.c;
  GRID_STRIDE(i, total) {
    long long t = i;
    const int x = t % f.w;
    t /= f.w;
    const int y = t % f.h;
    t /= f.h;
    const int z = t % f.d;
    t /= f.d;
    const int c = t % f.c;
    const int n = t / f.c;
    dst[i] = fr[fr_off(f, n, z, y, x) + c];
  }
}

static Frame F(const int* f) {
  return Frame{f[0], f[1], f[2], f[3], f[4], f[5], f[6], f[7], precision() == 0 ? 1 : 0};
}
static long long VC(const Frame& f) { return (long long)f.n * f.d * f.h * f.w; }
static cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

}  // namespace vpx

using namespace vpx;

#define LAUNCH_TAIL \
  VPX_LAUNCH_CHECK(); \
  return VPX_OK

extern "C" int vpx_leaky_fwd(const float* x, const int* xf, float* y, const int* yf, float slope,
                             void* st) {
  Frame a = F(xf), b = F(yf);
  if (a.c % 4 == 0) return leaky_fwd_vec(x, a, y, b, slope, S(st));
  leaky_fwd_kernel<<<grid1d(VC(a) * a.c), 256, 0, S(st)>>>(x, a, y, b, slope);
  LAUNCH_TAIL;
}
extern "C" int vpx_leaky_bwd(const float* x, const int* xf, const float* u, const int* uf, float* g,
                             const int* gf, float slope, void* st) {
  Frame a = F(xf), b = F(uf), c = F(gf);
  if (a.c % 4 == 0) return leaky_bwd_vec(x, a, u, b, g, c, slope, S(st));
  leaky_bwd_kernel<<<grid1d(VC(a) * a.c), 256, 0, S(st)>>>(x, a, u, b, g, c, slope);
  LAUNCH_TAIL;
}
extern "C" int vpx_pool_fwd(const float* x, const int* xf, float* y, const int* yf, int is_max,
                            void* st) {
  Frame a = F(xf), b = F(yf);
  if (a.d % 2 || a.h % 2 || a.w % 2) VPX_FAIL(VPX_ERR_NON_DIVISIBLE, "pool3d needs even extents");
  if (b.d * 2 != a.d || b.h * 2 != a.h || b.w * 2 != a.w || a.c != b.c || a.n != b.n)
    VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "pool output extents");
  if (a.c % 4 == 0) return pool_fwd_vec(x, a, y, b, is_max, S(st));
  pool_fwd_kernel<<<grid1d(VC(b) * b.c), 256, 0, S(st)>>>(x, a, y, b, is_max);
  LAUNCH_TAIL;
}
extern "C" int vpx_pool_bwd(const float* x, const int* xf, const float* u, const int* uf, float* g,
                            const int* gf, int is_max, void* st) {
  Frame a = F(xf), b = F(uf), c = F(gf);
  if (a.c % 4 == 0) return pool_bwd_vec(x, a, u, b, g, c, is_max, S(st));
  pool_bwd_kernel<<<grid1d(VC(b) * b.c), 256, 0, S(st)>>>(x, a, u, b, g, c, is_max);
  LAUNCH_TAIL;
}
extern "C" long long vpx_bn_workspace_bytes(int c) { return (long long)kBnParts * 2 * c * 8; }
extern "C" int vpx_bn_sums(const float* x, const int* xf, const float* u, const int* uf,
                           const float* mean, const float* inv, int mode, float* out2c, void* ws,
                           void* st) {
  Frame a = F(xf), b = uf ? F(uf) : F(xf);
  if (a.c % 4 == 0 && a.c / 4 <= 256 && 256 % (a.c / 4) == 0) {
    if (int rc = bn_sums_vec(x, a, u ? u : x, b, mean, inv, mode, static_cast<double*>(ws), kBnParts, S(st)))
      return rc;
    bn_finish_kernel<<<2 * a.c, 256, 0, S(st)>>>(static_cast<double*>(ws), kBnParts, a.c, out2c);
    LAUNCH_TAIL;
  }
  const int threads = a.c >= 256 ? a.c : (256 / a.c) * a.c;
  if (threads > 1024) VPX_FAIL(VPX_ERR_UNSUPPORTED, "bn channels %d", a.c);
  bn_partial_kernel<<<kBnParts, threads, 2 * threads * sizeof(double), S(st)>>>(
      x, a, u ? u : x, b, mean, inv, mode, static_cast<double*>(ws));
  VPX_LAUNCH_CHECK();
  bn_finish_kernel<<<2 * a.c, 256, 0, S(st)>>>(static_cast<double*>(ws), kBnParts, a.c, out2c);
  LAUNCH_TAIL;
}
extern "C" int vpx_bn_stats(const float* sums, int c, double count, float eps, float momentum,
                            float* mean, float* inv, float* run_mean, float* run_var, void* st) {
  bn_stats_kernel<<<1, 256, 0, S(st)>>>(sums, c, count, eps, momentum, mean, inv, run_mean, run_var);
  LAUNCH_TAIL;
}
extern "C" int vpx_bn_apply(const float* x, const int* xf, const float* mean, const float* inv,
                            const float* gamma, const float* beta, float* y, const int* yf, void* st) {
  Frame a = F(xf), b = F(yf);
  if (a.c % 4 == 0) return bn_apply_vec(x, a, mean, inv, gamma, beta, y, b, S(st));
  bn_apply_kernel<<<grid1d(VC(a) * a.c), 256, 0, S(st)>>>(x, a, mean, inv, gamma, beta, y, b);
  LAUNCH_TAIL;
}
extern "C" int vpx_bn_apply_leaky(const float* x, const int* xf, const float* mean, const float* inv,
                                  const float* gamma, const float* beta, float slope, float* y, const int* yf,
                                  void* st) {
  Frame a = F(xf), b = F(yf);
  if (a.c % 4) VPX_FAIL(VPX_ERR_UNSUPPORTED, "bn_apply_leaky needs C % 4 == 0");
  return bn_apply_vec(x, a, mean, inv, gamma, beta, y, b, S(st), true, slope);
}
extern "C" int vpx_bn_bwd_apply(const float* x, const int* xf, const float* u, const int* uf,
                                const float* mean, const float* inv, const float* gamma,
                                const float* sums, double count, float* g, const int* gf, void* st) {
  Frame a = F(xf), b = F(uf), c = F(gf);
  if (a.c % 4 == 0)
    return bn_bwd_apply_vec(x, a, u, b, mean, inv, gamma, sums, static_cast<float>(1.0 / count), g, c, S(st));
  bn_bwd_apply_kernel<<<grid1d(VC(a) * a.c), 256, 0, S(st)>>>(
      x, a, u, b, mean, inv, gamma, sums, static_cast<float>(1.0 / count), g, c);
  LAUNCH_TAIL;
}
extern "C" int vpx_concat(const float* a, const int* af, const float* b, const int* bf, float* y,
                          const int* yf, void* st) {
  Frame A = F(af), B = F(bf), Y = F(yf);
  if (A.c + B.c != Y.c) VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "concat channels");
  if (A.c % 4 == 0 && B.c % 4 == 0) return vpx::concat_vec(a, A, b, B, y, Y, S(st));
  concat_kernel<<<grid1d(VC(Y) * Y.c), 256, 0, S(st)>>>(a, A, b, B, y, Y);
  LAUNCH_TAIL;
}
extern "C" int vpx_split(const float* u, const int* uf, float* ga, const int* gaf, float* gb,
                         const int* gbf, int acc_b, void* st) {
  Frame U = F(uf), A = F(gaf), B = F(gbf);
  if (A.c + B.c != U.c) VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "split channels");
  if (A.c % 4 == 0 && B.c % 4 == 0) return vpx::split_vec(u, U, ga, A, gb, B, acc_b, S(st));
  split_kernel<<<grid1d(VC(U) * U.c), 256, 0, S(st)>>>(u, U, ga, A, gb, B, acc_b);
  LAUNCH_TAIL;
}
extern "C" int vpx_add(const float* x, const int* xf, float* y, const int* yf, void* st) {
  Frame A = F(xf), B = F(yf);
  add_kernel<<<grid1d(VC(A) * A.c), 256, 0, S(st)>>>(x, A, y, B);
  LAUNCH_TAIL;
}
extern "C" int vpx_copy(const float* x, const int* xf, float* y, const int* yf, void* st) {
  Frame A = F(xf), B = F(yf);
  copy_kernel<<<grid1d(VC(A) * A.c), 256, 0, S(st)>>>(x, A, y, B);
  LAUNCH_TAIL;
}
static int deconv_shape_check(const Frame& coarse, const Frame& fine, const char* what) {
  if (coarse.n != fine.n || fine.d != 2 * coarse.d || fine.h != 2 * coarse.h || fine.w != 2 * coarse.w)
    VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "%s: fine (%d,%d,%d,%d) is not twice coarse (%d,%d,%d,%d)", what, fine.n,
             fine.d, fine.h, fine.w, coarse.n, coarse.d, coarse.h, coarse.w);
  return VPX_OK;
}
// TF32 mode: the transposed conv runs on tcgen05 through the tap-box implicit
// GEMM (conv_tapbox.cu kind 1); FP32 mode (and channel counts without a
// tensor-core tile) on the CUDA-core kernels.
static bool deconv_tc(int cin, int cout, int mode) {
  return vpx::precision() == 0 && cin % 4 == 0 && cout % 4 == 0 && vpx::tapbox_supported(cin, cout, mode, 1) &&
         !getenv("VPX_NO_DECONV_TC");
}
extern "C" int vpx_deconv_fwd(const float* x, const int* xf, const float* w, float* y, const int* yf, void* ws,
                              long long ws_bytes, void* st) {
  Frame A = F(xf), B = F(yf);
  if (int rc = deconv_shape_check(A, B, "deconv fwd")) return rc;
  if (deconv_tc(A.c, B.c, 1))
    return vpx::conv_tapbox(1, x, A, w, A.c, B.c, 2, y, B, 0, 0.f, ws, S(st), ws_bytes, 1);
  vpx::note_fallback();
  if (vpx::deconv_vec_supported(A.c, B.c)) return vpx::deconv_fwd_vec(x, A, w, y, B, S(st));
  deconv_fwd_kernel<<<grid1d(VC(B) * B.c), 256, 0, S(st)>>>(x, A, w, y, B);
  LAUNCH_TAIL;
}
extern "C" int vpx_deconv_bwd_data(const float* u, const int* uf, const float* w, float* g, const int* gf,
                                   void* ws, long long ws_bytes, void* st) {
  Frame A = F(uf), B = F(gf);
  if (int rc = deconv_shape_check(B, A, "deconv bwd_data")) return rc;
  if (deconv_tc(B.c, A.c, 0))
    return vpx::conv_tapbox(0, u, A, w, B.c, A.c, 2, g, B, 0, 0.f, ws, S(st), ws_bytes, 1);
  vpx::note_fallback();
  if (vpx::deconv_vec_supported(B.c, A.c)) return vpx::deconv_dgrad_vec(u, A, w, g, B, S(st));
  deconv_bwd_data_kernel<<<grid1d(VC(B) * B.c), 256, 0, S(st)>>>(u, A, w, g, B);
  LAUNCH_TAIL;
}
// partial slices for the filter gradient: 8 per SM for the vectorised kernel
// (its tile loop is latency-bound), at least 256 for the generic one
static long long deconv_parts_cap() { return 8LL * num_sms() > 256 ? 8LL * num_sms() : 256; }
extern "C" long long vpx_deconv_workspace_bytes(int cin, int cout) {
  const long long parts = deconv_parts_cap() * cin * cout * 8 * 4;
  // tap-box path: packed weights + split-K partial tiles (conv_tapbox.cu)
  const int nmax = cin > cout ? cin : cout;
  const long long tb = (vpx::tapbox_workspace_bytes(cin, cout) + 255) / 256 * 256 +
                       (long long)num_sms() * 128 * (nmax < 16 ? 16 : nmax) * 4;
  return parts > tb ? parts : tb;
}
extern "C" int vpx_deconv_bwd_filter(const float* x, const int* xf, const float* u, const int* uf,
                                     float* wg, int accumulate, void* ws, void* st) {
  Frame A = F(xf), B = F(uf);
  const long long nv = VC(A);
  const int P = static_cast<int>(nv < 256 ? nv : 256);
  const long long chunk = (nv + P - 1) / P;
  const int len = A.c * B.c * 8;
  if (vpx::precision() == 0 && vpx::deconv_wgrad_tc_supported(A, B) && !getenv("VPX_NO_DECONV_TC")) {
    if (int rc = vpx::deconv_wgrad_tc(x, A, u, B, static_cast<float*>(ws), S(st))) return rc;
    return vpx::reduce_partials(static_cast<float*>(ws), vpx::deconv_wgrad_tc_parts(A), len, wg, accumulate, S(st));
  }
  vpx::note_fallback();
  if (vpx::deconv_vec_supported(A.c, B.c)) {
    int Pv = 0;
    if (int rc = vpx::deconv_wgrad_vec(x, A, u, B, static_cast<float*>(ws), static_cast<int>(deconv_parts_cap()),
                                       &Pv, S(st)))
      return rc;
    return vpx::reduce_partials(static_cast<float*>(ws), Pv, len, wg, accumulate, S(st));
  }
  dim3 grid((len + 255) / 256, P);
  deconv_wgrad_kernel<<<grid, 256, 0, S(st)>>>(x, A, u, B, chunk, static_cast<float*>(ws));
  VPX_LAUNCH_CHECK();
  reduce_parts_kernel<<<grid1d(len), 256, 0, S(st)>>>(static_cast<float*>(ws), P, len, wg, accumulate);
  LAUNCH_TAIL;
}
extern "C" int vpx_halo_copy(float* fr, const int* ff, const int* box8, float* buf, int mode,
                             void* st) {
  Frame f = F(ff);
  const int* b = box8;
  if (b[0] < 0 || b[4] < 0 || b[0] + b[4] > f.n || b[1] < 0 || b[1] + b[5] > f.d + 2 * f.md ||
      b[2] < 0 || b[2] + b[6] > f.h + 2 * f.mh || b[3] < 0 || b[3] + b[7] > f.w + 2 * f.mw)
    VPX_FAIL(VPX_ERR_OUT_OF_BOUNDS, "halo box outside frame");
  const long long total = (long long)b[4] * b[5] * b[6] * b[7] * f.c;
  if (total == 0) return VPX_OK;
  halo_copy_kernel<<<grid1d(total), 256, 0, S(st)>>>(fr, f, b[0], b[1], b[2], b[3], b[4], b[5],
                                                     b[6], b[7], buf, mode);
  LAUNCH_TAIL;
}
extern "C" int vpx_prng_uniform(unsigned long long key, long long n, double lo, double hi,
                                float* out32, double* out64, void* st) {
  prng_uniform_kernel<<<grid1d(n), 256, 0, S(st)>>>(key, n, lo, hi, out32, out64);
  LAUNCH_TAIL;
}
extern "C" int vpx_prng_mask(unsigned long long key, long long n, double keep, unsigned char* out,
                             void* st) {
  prng_mask_kernel<<<grid1d(n), 256, 0, S(st)>>>(key, n, keep, out);
  LAUNCH_TAIL;
}
extern "C" int vpx_prng_volume(unsigned long long key, const int* ff, long long counter_base,
                               double lo, double hi, float* fr, void* st) {
  Frame f = F(ff);
  prng_volume_kernel<<<grid1d(VC(f) * f.c), 256, 0, S(st)>>>(key, f, counter_base, lo, hi, fr);
  LAUNCH_TAIL;
}
extern "C" int vpx_adam(float* p, const float* g, float* m, float* v, long long n, float lr,
                        float b1, float b2, float c1, float c2, float eps, void* st) {
  adam_kernel<<<grid1d(n), 256, 0, S(st)>>>(p, g, m, v, n, lr, b1, b2, c1, c2, eps);
  LAUNCH_TAIL;
}
extern "C" int vpx_adam_dev(float* p, const float* g, float* m, float* v, long long n, const float* hyper,
                            float b1, float b2, float eps, void* st) {
  adam_dev_kernel<<<grid1d(n), 256, 0, S(st)>>>(p, g, m, v, n, hyper, b1, b2, eps);
  LAUNCH_TAIL;
}
extern "C" int vpx_prng_mask_dev(const unsigned long long* key, long long n, double keep, unsigned char* out,
                                 void* st) {
  prng_mask_dev_kernel<<<grid1d(n), 256, 0, S(st)>>>(reinterpret_cast<const uint64_t*>(key), n, keep, out);
  LAUNCH_TAIL;
}
extern "C" int vpx_peer_signal(unsigned long long* peer_flag, void* st) {
  peer_signal_kernel<<<1, 1, 0, S(st)>>>(peer_flag);
  LAUNCH_TAIL;
}
extern "C" int vpx_peer_wait(const unsigned long long* flag, unsigned long long* expected, long long timeout_ns,
                             int* error, void* st) {
  peer_wait_kernel<<<1, 1, 0, S(st)>>>(flag, expected, timeout_ns, error);
  LAUNCH_TAIL;
}
extern "C" int vpx_sgd(float* p, const float* g, long long n, float lr, void* st) {
  sgd_kernel<<<grid1d(n), 256, 0, S(st)>>>(p, g, n, lr);
  LAUNCH_TAIL;
}
extern "C" int vpx_xent(const float* logits, const int* lf, const long long* labels, double count,
                        float* g, const int* gf, double* part, int nparts, void* st) {
  Frame A = F(lf), B = F(gf);
  const bool flat = A.md == 0 && A.mh == 0 && A.mw == 0 && B.md == 0 && B.mh == 0 && B.mw == 0;
  const bool aligned = (reinterpret_cast<uintptr_t>(logits) | reinterpret_cast<uintptr_t>(labels) |
                        reinterpret_cast<uintptr_t>(g)) % 16 == 0;
  if (A.c == 2 && B.c == 2 && flat && aligned && VC(A) % 2 == 0) {
    xent2_flat_kernel<<<nparts, 256, 0, S(st)>>>(reinterpret_cast<const float4*>(logits),
                                                 reinterpret_cast<const longlong2*>(labels), VC(A) / 2,
                                                 1.0 / count, reinterpret_cast<float4*>(g), B, part);
    LAUNCH_TAIL;
  }
  xent_kernel<<<nparts, 256, 0, S(st)>>>(logits, A, labels, 1.0 / count, g, B, part);
  LAUNCH_TAIL;
}
extern "C" int vpx_layout_ncdhw_to_frame(const float* src, const int* ff, float* fr, void* st) {
  Frame f = F(ff);
  if ((f.c % 4 == 0 || f.c == 1) && f.w % 4 == 0 && reinterpret_cast<uintptr_t>(src) % 16 == 0)
    return layout_to_frame<float>(src, f, fr, S(st));
  ncdhw_to_frame_kernel<<<grid1d(VC(f) * f.c), 256, 0, S(st)>>>(src, f, fr);
  LAUNCH_TAIL;
}
extern "C" int vpx_layout_ncdhw_i16_to_frame(const int16_t* src, const int* ff, float* fr, void* st) {
  return layout_to_frame<int16_t>(src, F(ff), fr, S(st));
}
extern "C" int vpx_layout_ncdhw_i8_to_frame(const int8_t* src, const int* ff, float* fr, void* st) {
  return layout_to_frame<int8_t>(src, F(ff), fr, S(st));
}
extern "C" int vpx_convert_i16_to_i64(const int16_t* src, long long n, long long* dst, void* st) {
  if (n <= 0) return VPX_OK;
  i16_to_i64_kernel<<<grid1d(n), 256, 0, S(st)>>>(src, n, dst);
  LAUNCH_TAIL;
}
extern "C" int vpx_layout_frame_to_ncdhw(const float* fr, const int* ff, float* dst, void* st) {
  Frame f = F(ff);
  frame_to_ncdhw_kernel<<<grid1d(VC(f) * f.c), 256, 0, S(st)>>>(fr, f, dst);
  LAUNCH_TAIL;
}
