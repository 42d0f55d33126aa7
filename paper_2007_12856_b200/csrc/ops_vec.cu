// Vectorised (float4 over channels) variants of the memory-bound kernels in
// ops.cu, used whenever C % 4 == 0.  Work is enumerated per float4 of an
// interior row: a row (n, z, y) of every frame is contiguous (margins only sit
// at the row ends), so one index decode serves 4 channels and all loads and
// stores are 16-byte and coalesced.
#include "conv_simt.h"
#include "ops_vec.h"
#include "vpx_round.cuh"
#include "vpx_host.h"

namespace vpx {

namespace {

__device__ __forceinline__ long long row_base(const Frame& f, long long row) {
  const int y = row % f.h;
  row /= f.h;
  const int z = row % f.d;
  const int n = static_cast<int>(row / f.d);
  return ((((long long)n * (f.d + 2 * f.md) + (z + f.md)) * (f.h + 2 * f.mh) + (y + f.mh)) *
              (f.w + 2 * f.mw) +
          f.mw) *
         f.c;
}

__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void st4(const Frame& f, float* p, float4 v) {
  *reinterpret_cast<float4*>(p) = rnd4(f, v);
}
__device__ __forceinline__ float lk(float v, float s) { return v >= 0.f ? v : s * v; }

#define ROW_LOOP(f)                                                                          \
  const long long per_row = (long long)(f).w * (f).c / 4;                                    \
  const long long total = (long long)(f).n * (f).d * (f).h * per_row;                        \
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;          \
       i += (long long)gridDim.x * blockDim.x)

// Two-level loop for one-to-one pointwise kernels: blocks stride over the
// interior rows (n, z, y), threads over a row's float4s -- no 64-bit divide per
// element (which otherwise costs more than the memory traffic).
#define ROWS2_LOOP(f)                                                                     \
  const int per_row = (f).w * (f).c / 4;                                                  \
  const long long nrows = (long long)(f).n * (f).d * (f).h;                               \
  for (long long row = blockIdx.x; row < nrows; row += gridDim.x)                         \
    for (int jj = threadIdx.x; jj < per_row; jj += blockDim.x)

__global__ void leaky_fwd_v(const float* __restrict__ x, Frame xf, float* __restrict__ y, Frame yf, float s) {
  ROWS2_LOOP(xf) {
    const int off = 4 * jj;
    float4 v = ld4(x + row_base(xf, row) + off);
    v = make_float4(lk(v.x, s), lk(v.y, s), lk(v.z, s), lk(v.w, s));
    st4(yf, y + row_base(yf, row) + off, v);
  }
}

__global__ void leaky_bwd_v(const float* __restrict__ x, Frame xf, const float* __restrict__ u, Frame uf,
                            float* __restrict__ g, Frame gf, float s) {
  ROWS2_LOOP(xf) {
    const int off = 4 * jj;
    const float4 a = ld4(x + row_base(xf, row) + off);
    const float4 b = ld4(u + row_base(uf, row) + off);
    st4(gf, g + row_base(gf, row) + off, make_float4(a.x >= 0.f ? b.x : s * b.x, a.y >= 0.f ? b.y : s * b.y,
                                                 a.z >= 0.f ? b.z : s * b.z, a.w >= 0.f ? b.w : s * b.w));
  }
}

__device__ __forceinline__ void mx(float4& best, const float4 v) {
  // strict '>' keeps the first (lowest window index) maximum on ties
  best.x = v.x > best.x ? v.x : best.x;
  best.y = v.y > best.y ? v.y : best.y;
  best.z = v.z > best.z ? v.z : best.z;
  best.w = v.w > best.w ? v.w : best.w;
}

// output row (n, zo, yo) of the pooled frame reads input rows (2zo+a, 2yo+b)
__global__ void pool_fwd_v(const float* __restrict__ x, Frame xf, float* __restrict__ y, Frame yf,
                           int is_max) {
  const int C = yf.c;
  const long long in_row_stride = (long long)(xf.w + 2 * xf.mw) * C;
  const long long in_plane_stride = (long long)(xf.h + 2 * xf.mh) * in_row_stride;
  ROW_LOOP(yf) {
    const long long orow = i / per_row, off = i % per_row;
    const int xo = static_cast<int>(off / (C / 4)), c4 = static_cast<int>(off % (C / 4));
    long long t = orow;
    const int yo = t % yf.h;
    t /= yf.h;
    const int zo = t % yf.d;
    const int n = static_cast<int>(t / yf.d);
    const float* p = x + ((((long long)n * (xf.d + 2 * xf.md) + (2 * zo + xf.md)) * (xf.h + 2 * xf.mh) +
                           (2 * yo + xf.mh)) * (xf.w + 2 * xf.mw) + (2 * xo + xf.mw)) * C + 4 * c4;
    float4 acc = ld4(p);
    float4 sum = acc;
#pragma unroll
    for (int w8 = 1; w8 < 8; ++w8) {
      const int a = w8 >> 2, b = (w8 >> 1) & 1, cc = w8 & 1;
      const float4 v = ld4(p + a * in_plane_stride + b * in_row_stride + cc * C);
      if (is_max) mx(acc, v);
      sum.x += v.x;
      sum.y += v.y;
      sum.z += v.z;
      sum.w += v.w;
    }
    if (!is_max) acc = make_float4(sum.x / 8.0f, sum.y / 8.0f, sum.z / 8.0f, sum.w / 8.0f);
    st4(yf, y + row_base(yf, orow) + 4 * off, acc);
  }
}

// g[input window] from u[pooled voxel]; max: one-hot at the first maximum
__global__ void pool_bwd_v(const float* __restrict__ x, Frame xf, const float* __restrict__ u, Frame uf,
                           float* __restrict__ g, Frame gf, int is_max) {
  const int C = uf.c;
  ROW_LOOP(uf) {
    const long long orow = i / per_row, off = i % per_row;
    const int xo = static_cast<int>(off / (C / 4)), c4 = static_cast<int>(off % (C / 4));
    long long t = orow;
    const int yo = t % uf.h;
    t /= uf.h;
    const int zo = t % uf.d;
    const int n = static_cast<int>(t / uf.d);
    const float4 uv = ld4(u + row_base(uf, orow) + 4 * off);
    auto foff = [&](const Frame& f, int a, int b, int cc) {
      return ((((long long)n * (f.d + 2 * f.md) + (2 * zo + a + f.md)) * (f.h + 2 * f.mh) + (2 * yo + b + f.mh)) *
                  (f.w + 2 * f.mw) + (2 * xo + cc + f.mw)) * C + 4 * c4;
    };
    if (!is_max) {
      const float4 gv = make_float4(uv.x / 8.0f, uv.y / 8.0f, uv.z / 8.0f, uv.w / 8.0f);
#pragma unroll
      for (int w8 = 0; w8 < 8; ++w8) st4(gf, g + foff(gf, w8 >> 2, (w8 >> 1) & 1, w8 & 1), gv);
    } else {
      float4 best = ld4(x + foff(xf, 0, 0, 0));
      int ax = 0, ay = 0, az = 0, aw = 0;
#pragma unroll
      for (int w8 = 1; w8 < 8; ++w8) {
        const float4 v = ld4(x + foff(xf, w8 >> 2, (w8 >> 1) & 1, w8 & 1));
        if (v.x > best.x) { best.x = v.x; ax = w8; }
        if (v.y > best.y) { best.y = v.y; ay = w8; }
        if (v.z > best.z) { best.z = v.z; az = w8; }
        if (v.w > best.w) { best.w = v.w; aw = w8; }
      }
#pragma unroll
      for (int w8 = 0; w8 < 8; ++w8)
        st4(gf, g + foff(gf, w8 >> 2, (w8 >> 1) & 1, w8 & 1),
            make_float4(w8 == ax ? uv.x : 0.f, w8 == ay ? uv.y : 0.f, w8 == az ? uv.z : 0.f, w8 == aw ? uv.w : 0.f));
    }
  }
}

// LEAKY: BatchNorm followed by LeakyReLU in one pass (the normalised value is
// rounded as its own frame would store it, then activated and rounded again:
// the same bits as bn_apply + leaky_fwd, without the intermediate tensor).
template <bool LEAKY>
__global__ void bn_apply_v(const float* __restrict__ x, Frame xf, const float* __restrict__ mean,
                           const float* __restrict__ inv, const float* __restrict__ gamma,
                           const float* __restrict__ beta, float* __restrict__ y, Frame yf, float s) {
  const int C = xf.c;
  ROWS2_LOOP(xf) {
    const int off = 4 * jj;
    const int c = off % C;
    const float4 v = ld4(x + row_base(xf, row) + off);
    float r[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      r[j] = gamma[c + j] * ((r[j] - mean[c + j]) * inv[c + j]) + beta[c + j];
      if (LEAKY) {
        r[j] = rnd(yf, r[j]);
        r[j] = r[j] >= 0.f ? r[j] : s * r[j];
      }
    }
    st4(yf, y + row_base(yf, row) + off, make_float4(r[0], r[1], r[2], r[3]));
  }
}

__global__ void bn_bwd_apply_v(const float* __restrict__ x, Frame xf, const float* __restrict__ u, Frame uf,
                               const float* __restrict__ mean, const float* __restrict__ inv,
                               const float* __restrict__ gamma, const float* __restrict__ sums,
                               float inv_count, float* __restrict__ g, Frame gf) {
  const int C = xf.c;
  ROWS2_LOOP(xf) {
    const int off = 4 * jj;
    const int c = off % C;
    const float4 a = ld4(x + row_base(xf, row) + off);
    const float4 b = ld4(u + row_base(uf, row) + off);
    const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
    float r[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float xh = (av[j] - mean[c + j]) * inv[c + j];
      r[j] = gamma[c + j] * inv[c + j] * (bv[j] - (sums[c + j] + xh * sums[C + c + j]) * inv_count);
    }
    st4(gf, g + row_base(gf, row) + off, make_float4(r[0], r[1], r[2], r[3]));
  }
}

// Margin-free frames: the interior is one contiguous NDHWC array, so the
// pointwise kernels run a flat float4 loop with no index decode at all.  The
// grid stride is a multiple of 256 float4s and C/4 divides 256, so a thread's
// channel quad is fixed (per-channel constants live in registers).
#define FLAT_LOOP(n4)                                                                       \
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (n4);          \
       i += (long long)gridDim.x * blockDim.x)

__global__ void leaky_fwd_flat(const float4* __restrict__ x, float4* __restrict__ y, long long n4, float s,
                               Frame yf) {
  FLAT_LOOP(n4) {
    const float4 v = x[i];
    y[i] = rnd4(yf, make_float4(lk(v.x, s), lk(v.y, s), lk(v.z, s), lk(v.w, s)));
  }
}
__global__ void leaky_bwd_flat(const float4* __restrict__ x, const float4* __restrict__ u, float4* __restrict__ g,
                               long long n4, float s, Frame gf) {
  FLAT_LOOP(n4) {
    const float4 a = x[i], b = u[i];
    g[i] = rnd4(gf, make_float4(a.x >= 0.f ? b.x : s * b.x, a.y >= 0.f ? b.y : s * b.y,
                                a.z >= 0.f ? b.z : s * b.z, a.w >= 0.f ? b.w : s * b.w));
  }
}
template <bool LEAKY>
__global__ void bn_apply_flat(const float4* __restrict__ x, const float* __restrict__ mean,
                              const float* __restrict__ inv, const float* __restrict__ gamma,
                              const float* __restrict__ beta, float4* __restrict__ y, long long n4, int C4,
                              Frame yf, float s) {
  const int c = 4 * (threadIdx.x % C4);
  float mu[4], iv[4], ga[4], be[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    mu[j] = mean[c + j];
    iv[j] = inv[c + j];
    ga[j] = gamma[c + j];
    be[j] = beta[c + j];
  }
  FLAT_LOOP(n4) {
    const float4 v = x[i];
    const float r[4] = {v.x, v.y, v.z, v.w};
    float o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      o[j] = ga[j] * ((r[j] - mu[j]) * iv[j]) + be[j];
      if (LEAKY) {
        o[j] = rnd(yf, o[j]);
        o[j] = o[j] >= 0.f ? o[j] : s * o[j];
      }
    }
    y[i] = rnd4(yf, make_float4(o[0], o[1], o[2], o[3]));
  }
}
__global__ void bn_bwd_apply_flat(const float4* __restrict__ x, const float4* __restrict__ u,
                                  const float* __restrict__ mean, const float* __restrict__ inv,
                                  const float* __restrict__ gamma, const float* __restrict__ sums, float inv_count,
                                  float4* __restrict__ g, long long n4, int C4, Frame gf) {
  const int C = 4 * C4, c = 4 * (threadIdx.x % C4);
  float mu[4], iv[4], gi[4], s0[4], s1[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    mu[j] = mean[c + j];
    iv[j] = inv[c + j];
    gi[j] = gamma[c + j] * inv[c + j];
    s0[j] = sums[c + j];
    s1[j] = sums[C + c + j];
  }
  FLAT_LOOP(n4) {
    const float4 a = x[i], b = u[i];
    const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
    float r[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float xh = (av[j] - mu[j]) * iv[j];
      r[j] = gi[j] * (bv[j] - (s0[j] + xh * s1[j]) * inv_count);
    }
    g[i] = rnd4(gf, make_float4(r[0], r[1], r[2], r[3]));
  }
}

bool flat_ok(const Frame& f) { return f.md == 0 && f.mh == 0 && f.mw == 0 && f.c % 4 == 0 && 256 % (f.c / 4) == 0; }
long long n4_of(const Frame& f) { return (long long)f.n * f.d * f.h * f.w * f.c / 4; }

int grid_v(const Frame& f) {
  const long long total = (long long)f.n * f.d * f.h * f.w * f.c / 4;
  long long g = (total + 255) / 256;
  const long long cap = (long long)num_sms() * 16;
  return static_cast<int>(g < 1 ? 1 : (g > cap ? cap : g));
}
// grid for ROWS2_LOOP kernels: one block per row, capped
int grid_rows(const Frame& f) {
  const long long rows = (long long)f.n * f.d * f.h;
  const long long cap = (long long)num_sms() * 16;
  return static_cast<int>(rows < 1 ? 1 : (rows > cap ? cap : rows));
}

}  // namespace

int leaky_fwd_vec(const float* x, const Frame& xf, float* y, const Frame& yf, float s, cudaStream_t st) {
  if (flat_ok(xf) && flat_ok(yf)) {
    leaky_fwd_flat<<<grid_v(xf), 256, 0, st>>>(reinterpret_cast<const float4*>(x), reinterpret_cast<float4*>(y),
                                                n4_of(xf), s, yf);
    VPX_LAUNCH_CHECK();
    return VPX_OK;
  }
  leaky_fwd_v<<<grid_rows(xf), 256, 0, st>>>(x, xf, y, yf, s);
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}
int leaky_bwd_vec(const float* x, const Frame& xf, const float* u, const Frame& uf, float* g, const Frame& gf,
                  float s, cudaStream_t st) {
  if (flat_ok(xf) && flat_ok(uf) && flat_ok(gf)) {
    leaky_bwd_flat<<<grid_v(xf), 256, 0, st>>>(reinterpret_cast<const float4*>(x), reinterpret_cast<const float4*>(u),
                                                reinterpret_cast<float4*>(g), n4_of(xf), s, gf);
    VPX_LAUNCH_CHECK();
    return VPX_OK;
  }
  leaky_bwd_v<<<grid_rows(xf), 256, 0, st>>>(x, xf, u, uf, g, gf, s);
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}
int pool_fwd_vec(const float* x, const Frame& xf, float* y, const Frame& yf, int is_max, cudaStream_t st) {
  pool_fwd_v<<<grid_v(yf), 256, 0, st>>>(x, xf, y, yf, is_max);
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}
int pool_bwd_vec(const float* x, const Frame& xf, const float* u, const Frame& uf, float* g, const Frame& gf,
                 int is_max, cudaStream_t st) {
  pool_bwd_v<<<grid_v(uf), 256, 0, st>>>(x, xf, u, uf, g, gf, is_max);
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}
int bn_apply_vec(const float* x, const Frame& xf, const float* mean, const float* inv, const float* gamma,
                 const float* beta, float* y, const Frame& yf, cudaStream_t st, bool leaky, float slope) {
  if (flat_ok(xf) && flat_ok(yf)) {
    auto k = leaky ? bn_apply_flat<true> : bn_apply_flat<false>;
    k<<<grid_v(xf), 256, 0, st>>>(reinterpret_cast<const float4*>(x), mean, inv, gamma, beta,
                                  reinterpret_cast<float4*>(y), n4_of(xf), xf.c / 4, yf, slope);
    VPX_LAUNCH_CHECK();
    return VPX_OK;
  }
  auto k = leaky ? bn_apply_v<true> : bn_apply_v<false>;
  k<<<grid_rows(xf), 256, 0, st>>>(x, xf, mean, inv, gamma, beta, y, yf, slope);
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}
int bn_bwd_apply_vec(const float* x, const Frame& xf, const float* u, const Frame& uf, const float* mean,
                     const float* inv, const float* gamma, const float* sums, float inv_count, float* g,
                     const Frame& gf, cudaStream_t st) {
  if (flat_ok(xf) && flat_ok(uf) && flat_ok(gf)) {
    bn_bwd_apply_flat<<<grid_v(xf), 256, 0, st>>>(reinterpret_cast<const float4*>(x),
                                                   reinterpret_cast<const float4*>(u), mean, inv, gamma, sums,
                                                   inv_count, reinterpret_cast<float4*>(g), n4_of(xf), xf.c / 4, gf);
    VPX_LAUNCH_CHECK();
    return VPX_OK;
  }
  bn_bwd_apply_v<<<grid_rows(xf), 256, 0, st>>>(x, xf, u, uf, mean, inv, gamma, sums, inv_count, g, gf);
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}

}  // namespace vpx

// Fused 2^3 pool backward + LeakyReLU backward of the first conv block,
// writing the conv-output gradient in the 4-channel-blocked layout
// [C/4][n][d][h][w][4] that conv_wgrad_c4.cu consumes.  y is the LeakyReLU
// output (= pool input; its sign is the pre-activation's sign), up the pooled
// gradient.  Saves the full-resolution pool-backward tensor (write + read).
namespace vpx {
namespace {
__global__ void pool_leaky_bwd_blocked_v(const float* __restrict__ y, Frame yf, const float* __restrict__ up,
                                         Frame uf, float* __restrict__ gb, float s, int is_max) {
  const int C = uf.c;
  const long long vox_full = (long long)yf.n * yf.d * yf.h * yf.w;
  ROW_LOOP(uf) {
    const long long orow = i / per_row, off = i % per_row;
    const int xo = static_cast<int>(off / (C / 4)), c4 = static_cast<int>(off % (C / 4));
    long long t = orow;
    const int yo = t % uf.h;
    t /= uf.h;
    const int zo = t % uf.d;
    const int n = static_cast<int>(t / uf.d);
    const float4 uv = ld4(up + row_base(uf, orow) + 4 * off);
    float4 vals[8];
#pragma unroll
    for (int w8 = 0; w8 < 8; ++w8) {
      const int a = w8 >> 2, b = (w8 >> 1) & 1, cc = w8 & 1;
      vals[w8] = ld4(y + ((((long long)n * (yf.d + 2 * yf.md) + (2 * zo + a + yf.md)) * (yf.h + 2 * yf.mh) +
                           (2 * yo + b + yf.mh)) * (yf.w + 2 * yf.mw) + (2 * xo + cc + yf.mw)) * C + 4 * c4);
    }
    int ax = 0, ay = 0, az = 0, aw = 0;
    if (is_max) {
      float4 best = vals[0];
#pragma unroll
      for (int w8 = 1; w8 < 8; ++w8) {
        if (vals[w8].x > best.x) { best.x = vals[w8].x; ax = w8; }
        if (vals[w8].y > best.y) { best.y = vals[w8].y; ay = w8; }
        if (vals[w8].z > best.z) { best.z = vals[w8].z; az = w8; }
        if (vals[w8].w > best.w) { best.w = vals[w8].w; aw = w8; }
      }
    }
    const float4 avg = make_float4(uv.x / 8.0f, uv.y / 8.0f, uv.z / 8.0f, uv.w / 8.0f);
#pragma unroll
    for (int w8 = 0; w8 < 8; ++w8) {
      const int a = w8 >> 2, b = (w8 >> 1) & 1, cc = w8 & 1;
      float4 g = is_max ? make_float4(w8 == ax ? uv.x : 0.f, w8 == ay ? uv.y : 0.f, w8 == az ? uv.z : 0.f,
                                      w8 == aw ? uv.w : 0.f)
                        : avg;
      const float4 v = vals[w8];
      g = make_float4(v.x >= 0.f ? g.x : s * g.x, v.y >= 0.f ? g.y : s * g.y, v.z >= 0.f ? g.z : s * g.z,
                      v.w >= 0.f ? g.w : s * g.w);
      const long long vox = (((long long)n * yf.d + 2 * zo + a) * yf.h + 2 * yo + b) * yf.w + 2 * xo + cc;
      float* dst = gb + ((long long)c4 * vox_full + vox) * 4;
      *reinterpret_cast<float4*>(dst) = rnd4(yf, g);
    }
  }
}

// Same fused pool + LeakyReLU backward, writing the gradient frame gf (NDHWC,
// any margins): replaces the pool-backward write + leaky-backward read/write.
__global__ void pool_leaky_bwd_v(const float* __restrict__ y, Frame yf, const float* __restrict__ up, Frame uf,
                                 float* __restrict__ g, Frame gf, float s, int is_max) {
  const int C = uf.c;
  ROW_LOOP(uf) {
    const long long orow = i / per_row, off = i % per_row;
    const int xo = static_cast<int>(off / (C / 4)), c4 = static_cast<int>(off % (C / 4));
    long long t = orow;
    const int yo = t % uf.h;
    t /= uf.h;
    const int zo = t % uf.d;
    const int n = static_cast<int>(t / uf.d);
    auto foff = [&](const Frame& f, int a, int b, int cc) {
      return ((((long long)n * (f.d + 2 * f.md) + (2 * zo + a + f.md)) * (f.h + 2 * f.mh) + (2 * yo + b + f.mh)) *
                  (f.w + 2 * f.mw) + (2 * xo + cc + f.mw)) * C + 4 * c4;
    };
    const float4 uv = ld4(up + row_base(uf, orow) + 4 * off);
    float4 vals[8];
#pragma unroll
    for (int w8 = 0; w8 < 8; ++w8) vals[w8] = ld4(y + foff(yf, w8 >> 2, (w8 >> 1) & 1, w8 & 1));
    int ax = 0, ay = 0, az = 0, aw = 0;
    if (is_max) {
      float4 best = vals[0];
#pragma unroll
      for (int w8 = 1; w8 < 8; ++w8) {
        if (vals[w8].x > best.x) { best.x = vals[w8].x; ax = w8; }
        if (vals[w8].y > best.y) { best.y = vals[w8].y; ay = w8; }
        if (vals[w8].z > best.z) { best.z = vals[w8].z; az = w8; }
        if (vals[w8].w > best.w) { best.w = vals[w8].w; aw = w8; }
      }
    }
    const float4 avg = make_float4(uv.x / 8.0f, uv.y / 8.0f, uv.z / 8.0f, uv.w / 8.0f);
#pragma unroll
    for (int w8 = 0; w8 < 8; ++w8) {
      float4 gg = is_max ? make_float4(w8 == ax ? uv.x : 0.f, w8 == ay ? uv.y : 0.f, w8 == az ? uv.z : 0.f,
                                       w8 == aw ? uv.w : 0.f)
                         : avg;
      const float4 v = vals[w8];
      gg = make_float4(v.x >= 0.f ? gg.x : s * gg.x, v.y >= 0.f ? gg.y : s * gg.y, v.z >= 0.f ? gg.z : s * gg.z,
                       v.w >= 0.f ? gg.w : s * gg.w);
      st4(gf, g + foff(gf, w8 >> 2, (w8 >> 1) & 1, w8 & 1), gg);
    }
  }
}
// Average-pool + LeakyReLU backward from the forward's sign mask (the fused
// conv+pool forward never stores the activation): g = (bit ? 1 : s) * up / 8,
// the same operations in the same order as pool_leaky_bwd_v.  mask: MB bytes
// per voxel, [n][d][h][w], no margins.
template <int MB>
__global__ void pool_leaky_bwd_mask_v(const uint8_t* __restrict__ mask, const float* __restrict__ up, Frame uf,
                                      float* __restrict__ g, Frame gf, float s) {
  const int C = uf.c;
  const int Dm = 2 * uf.d, Hm = 2 * uf.h, Wm = 2 * uf.w;
  ROW_LOOP(uf) {
    const long long orow = i / per_row, off = i % per_row;
    const int xo = static_cast<int>(off / (C / 4)), c4 = static_cast<int>(off % (C / 4));
    long long t = orow;
    const int yo = t % uf.h;
    t /= uf.h;
    const int zo = t % uf.d;
    const int n = static_cast<int>(t / uf.d);
    const float4 uv = ld4(up + row_base(uf, orow) + 4 * off);
    const float4 avg = make_float4(uv.x / 8.0f, uv.y / 8.0f, uv.z / 8.0f, uv.w / 8.0f);
#pragma unroll
    for (int w8 = 0; w8 < 8; ++w8) {
      const int a = w8 >> 2, b = (w8 >> 1) & 1, cc = w8 & 1;
      const long long vox = (((long long)n * Dm + 2 * zo + a) * Hm + 2 * yo + b) * Wm + 2 * xo + cc;
      uint32_t bits;
      if constexpr (MB == 4) bits = reinterpret_cast<const uint32_t*>(mask)[vox];
      else if constexpr (MB == 2) bits = reinterpret_cast<const uint16_t*>(mask)[vox];
      else bits = mask[vox];
      bits >>= 4 * c4;
      const float4 gg = make_float4((bits & 1u) ? avg.x : s * avg.x, (bits & 2u) ? avg.y : s * avg.y,
                                    (bits & 4u) ? avg.z : s * avg.z, (bits & 8u) ? avg.w : s * avg.w);
      st4(gf, g + ((((long long)n * (gf.d + 2 * gf.md) + (2 * zo + a + gf.md)) * (gf.h + 2 * gf.mh) +
                    (2 * yo + b + gf.mh)) * (gf.w + 2 * gf.mw) + (2 * xo + cc + gf.mw)) * C + 4 * c4,
          gg);
    }
  }
}
}  // namespace

// BatchNorm per-channel sums, float4 over channels and whole interior rows
// per block (no per-voxel index decode).  Block p owns rows
// [rows*p/P, rows*(p+1)/P); lanes with the same channel quad are combined in
// a fixed order, so the fp64 partials are deterministic.
// mode 0: (sum x, sum x^2); mode 1: (sum u, sum u*xhat), xhat = (x-mean)*inv.
template <int MODE>
__global__ void bn_sums_v(const float* __restrict__ x, Frame xf, const float* __restrict__ u, Frame uf,
                          const float* __restrict__ mean, const float* __restrict__ inv, double* __restrict__ part,
                          int flat) {
  extern __shared__ double shd[];  // [8][blockDim.x]
  const int C = xf.c, C4 = C / 4;
  const int lanes = blockDim.x / C4, c4 = threadIdx.x % C4, lane = threadIdx.x / C4;
  const long long rows = (long long)xf.n * xf.d * xf.h;
  const long long r0 = rows * blockIdx.x / gridDim.x, r1 = rows * (blockIdx.x + 1) / gridDim.x;
  double s1[4] = {0.0, 0.0, 0.0, 0.0}, s2[4] = {0.0, 0.0, 0.0, 0.0};
  float4 mu = make_float4(0.f, 0.f, 0.f, 0.f), iv = mu;
  if (MODE == 1) {
    mu = ld4(mean + 4 * c4);
    iv = ld4(inv + 4 * c4);
  }
  if (flat) {
    // contiguous interior: rows [r0, r1) are one float4 range; c4 = threadIdx.x % C4
    const long long per_row4 = (long long)xf.w * C4;
    const float4* xp = reinterpret_cast<const float4*>(x) + r0 * per_row4;
    const float4* up = reinterpret_cast<const float4*>(u) + r0 * per_row4;
    const long long n4 = (r1 - r0) * per_row4;
#pragma unroll 4
    for (long long i = threadIdx.x; i < n4; i += blockDim.x) {
      const float4 a = xp[i];
      if (MODE == 0) {
        s1[0] += a.x; s1[1] += a.y; s1[2] += a.z; s1[3] += a.w;
        s2[0] += (double)a.x * a.x; s2[1] += (double)a.y * a.y;
        s2[2] += (double)a.z * a.z; s2[3] += (double)a.w * a.w;
      } else {
        const float4 b = up[i];
        s1[0] += b.x; s1[1] += b.y; s1[2] += b.z; s1[3] += b.w;
        s2[0] += (double)b.x * ((a.x - mu.x) * iv.x);
        s2[1] += (double)b.y * ((a.y - mu.y) * iv.y);
        s2[2] += (double)b.z * ((a.z - mu.z) * iv.z);
        s2[3] += (double)b.w * ((a.w - mu.w) * iv.w);
      }
    }
  } else if (lane < lanes) {
    for (long long row = r0; row < r1; ++row) {
      const float* xb = x + row_base(xf, row) + 4 * c4;
      const float* ub = MODE == 1 ? u + row_base(uf, row) + 4 * c4 : nullptr;
      for (int v = lane; v < xf.w; v += lanes) {
        const float4 a = ld4(xb + (long long)v * C);
        if (MODE == 0) {
          s1[0] += a.x; s1[1] += a.y; s1[2] += a.z; s1[3] += a.w;
          s2[0] += (double)a.x * a.x; s2[1] += (double)a.y * a.y;
          s2[2] += (double)a.z * a.z; s2[3] += (double)a.w * a.w;
        } else {
          const float4 b = ld4(ub + (long long)v * uf.c);
          s1[0] += b.x; s1[1] += b.y; s1[2] += b.z; s1[3] += b.w;
          s2[0] += (double)b.x * ((a.x - mu.x) * iv.x);
          s2[1] += (double)b.y * ((a.y - mu.y) * iv.y);
          s2[2] += (double)b.z * ((a.z - mu.z) * iv.z);
          s2[3] += (double)b.w * ((a.w - mu.w) * iv.w);
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    shd[j * blockDim.x + threadIdx.x] = s1[j];
    shd[(4 + j) * blockDim.x + threadIdx.x] = s2[j];
  }
  __syncthreads();
  if (threadIdx.x < C4) {  // lane 0 of every channel quad folds the lanes in order
    double t1[4] = {0.0, 0.0, 0.0, 0.0}, t2[4] = {0.0, 0.0, 0.0, 0.0};
    for (int l = 0; l < lanes; ++l)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        t1[j] += shd[j * blockDim.x + l * C4 + threadIdx.x];
        t2[j] += shd[(4 + j) * blockDim.x + l * C4 + threadIdx.x];
      }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      part[(long long)blockIdx.x * 2 * C + 4 * threadIdx.x + j] = t1[j];
      part[(long long)blockIdx.x * 2 * C + C + 4 * threadIdx.x + j] = t2[j];
    }
  }
}

int bn_sums_vec(const float* x, const Frame& xf, const float* u, const Frame& uf, const float* mean,
                const float* inv, int mode, double* part, int P, cudaStream_t st) {
  const int C4 = xf.c / 4;
  if (xf.c % 4 || C4 > 256 || 256 % C4) return VPX_ERR_UNSUPPORTED;
  const size_t sh = 8 * 256 * sizeof(double);
  const int flat = flat_ok(xf) && (mode == 0 || flat_ok(uf));
  if (mode == 0)
    bn_sums_v<0><<<P, 256, sh, st>>>(x, xf, x, xf, mean, inv, part, flat);
  else
    bn_sums_v<1><<<P, 256, sh, st>>>(x, xf, u, uf, mean, inv, part, flat);
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}

int pool_leaky_bwd(const float* y, const Frame& yf, const float* up, const Frame& uf, float* g, const Frame& gf,
                   float s, int is_max, cudaStream_t st) {
  pool_leaky_bwd_v<<<grid_v(uf), 256, 0, st>>>(y, yf, up, uf, g, gf, s, is_max);
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}

int pool_leaky_bwd_mask(const uint8_t* mask, const float* up, const Frame& uf, float* g, const Frame& gf, float s,
                        cudaStream_t st) {
  switch (uf.c / 8) {
    case 1: pool_leaky_bwd_mask_v<1><<<grid_v(uf), 256, 0, st>>>(mask, up, uf, g, gf, s); break;
    case 2: pool_leaky_bwd_mask_v<2><<<grid_v(uf), 256, 0, st>>>(mask, up, uf, g, gf, s); break;
    case 4: pool_leaky_bwd_mask_v<4><<<grid_v(uf), 256, 0, st>>>(mask, up, uf, g, gf, s); break;
    default: return VPX_ERR_UNSUPPORTED;
  }
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}

int pool_leaky_bwd_blocked(const float* y, const Frame& yf, const float* up, const Frame& uf, float* gb,
                           float s, int is_max, cudaStream_t st) {
  pool_leaky_bwd_blocked_v<<<grid_v(uf), 256, 0, st>>>(y, yf, up, uf, gb, s, is_max);
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}
}  // namespace vpx
