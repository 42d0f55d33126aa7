// U-Net decoder ops with small channel counts, row-structured and float4-wide:
//   * k2 s2 transposed conv (reference layers/reference.py:99-144): forward and
//     input gradient with one thread per coarse voxel (its 8 children), weights
//     broadcast from shared memory; filter gradient as a persistent, staged
//     outer-product reduction with fixed-order per-block partials;
//   * channel concat / split of the skip connections.
// The forward and input-gradient kernels keep the arithmetic order of the
// generic kernels in ops.cu (fmaf over ci ascending / over (k, co) ascending),
// so their outputs are bit-identical to those.
#include "conv_simt.h"
#include "ops_vec.h"
#include "vpx_host.h"
#include "vpx_round.cuh"

namespace vpx {

namespace {

__device__ __forceinline__ long long fidx(const Frame& f, int n, int z, int y, int x) {
  return ((((long long)n * (f.d + 2 * f.md) + (z + f.md)) * (f.h + 2 * f.mh) + (y + f.mh)) *
              (f.w + 2 * f.mw) +
          (x + f.mw)) *
         f.c;
}
struct Row {
  int n, z, y;
};
__device__ __forceinline__ Row row_of(const Frame& f, long long row) {
  Row r;
  r.y = static_cast<int>(row % f.h);
  row /= f.h;
  r.z = static_cast<int>(row % f.d);
  r.n = static_cast<int>(row / f.d);
  return r;
}
template <int C>
__device__ __forceinline__ void ld_c(const float* p, float (&v)[C]) {
  static_assert(C % 4 == 0, "float4 channels");
#pragma unroll
  for (int i = 0; i < C / 4; ++i) {
    const float4 t = *reinterpret_cast<const float4*>(p + 4 * i);
    v[4 * i] = t.x;
    v[4 * i + 1] = t.y;
    v[4 * i + 2] = t.z;
    v[4 * i + 3] = t.w;
  }
}
template <int C>
__device__ __forceinline__ void st_c(const Frame& f, float* p, const float (&v)[C]) {
#pragma unroll
  for (int i = 0; i < C / 4; ++i)
    *reinterpret_cast<float4*>(p + 4 * i) = rnd4(f, make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]));
}

// y[2p + k][co] = sum_ci x[p][ci] w[ci][co][k]
template <int CI, int CO>
__global__ void __launch_bounds__(128) deconv_fwd_v(const float* __restrict__ x, Frame xf,
                                                    const float* __restrict__ w, float* __restrict__ y, Frame yf) {
  __shared__ __align__(16) float ws[8 * CI * CO];  // [k][ci][co]
  for (int i = threadIdx.x; i < 8 * CI * CO; i += blockDim.x) {
    const int k = i % 8, co = (i / 8) % CO, ci = i / (8 * CO);
    ws[(k * CI + ci) * CO + co] = rnd(yf, w[i]);  // TF32 mode: TF32 operands
  }
  __syncthreads();
  const long long nrows = (long long)xf.n * xf.d * xf.h;
  for (long long row = blockIdx.x; row < nrows; row += gridDim.x) {
    const Row r = row_of(xf, row);
    const float* xr = x + fidx(xf, r.n, r.z, r.y, 0);
    for (int px = threadIdx.x; px < xf.w; px += blockDim.x) {
      float xv[CI];
      ld_c<CI>(xr + (long long)px * CI, xv);
#pragma unroll 1
      for (int k = 0; k < 8; ++k) {
        const int a = k >> 2, b = (k >> 1) & 1, c = k & 1;
        float acc[CO];
#pragma unroll
        for (int co = 0; co < CO; ++co) acc[co] = 0.f;
        const float* wk = ws + k * CI * CO;
#pragma unroll
        for (int ci = 0; ci < CI; ++ci) {
#pragma unroll
          for (int q = 0; q < CO / 4; ++q) {
            const float4 wv = *reinterpret_cast<const float4*>(wk + ci * CO + 4 * q);
            acc[4 * q] = fmaf(xv[ci], wv.x, acc[4 * q]);
            acc[4 * q + 1] = fmaf(xv[ci], wv.y, acc[4 * q + 1]);
            acc[4 * q + 2] = fmaf(xv[ci], wv.z, acc[4 * q + 2]);
            acc[4 * q + 3] = fmaf(xv[ci], wv.w, acc[4 * q + 3]);
          }
        }
        st_c<CO>(yf, y + fidx(yf, r.n, 2 * r.z + a, 2 * r.y + b, 2 * px + c), acc);
      }
    }
  }
}

// g[p][ci] = sum_{k, co} u[2p + k][co] w[ci][co][k]
template <int CI, int CO>
__global__ void __launch_bounds__(128) deconv_dgrad_v(const float* __restrict__ u, Frame uf,
                                                      const float* __restrict__ w, float* __restrict__ g, Frame gf) {
  __shared__ __align__(16) float ws[8 * CO * CI];  // [k][co][ci]
  for (int i = threadIdx.x; i < 8 * CI * CO; i += blockDim.x) {
    const int k = i % 8, co = (i / 8) % CO, ci = i / (8 * CO);
    ws[(k * CO + co) * CI + ci] = rnd(gf, w[i]);
  }
  __syncthreads();
  const long long nrows = (long long)gf.n * gf.d * gf.h;
  for (long long row = blockIdx.x; row < nrows; row += gridDim.x) {
    const Row r = row_of(gf, row);
    for (int px = threadIdx.x; px < gf.w; px += blockDim.x) {
      float acc[CI];
#pragma unroll
      for (int ci = 0; ci < CI; ++ci) acc[ci] = 0.f;
#pragma unroll 1
      for (int k = 0; k < 8; ++k) {
        const int a = k >> 2, b = (k >> 1) & 1, c = k & 1;
        float uv[CO];
        ld_c<CO>(u + fidx(uf, r.n, 2 * r.z + a, 2 * r.y + b, 2 * px + c), uv);
        const float* wk = ws + k * CO * CI;
#pragma unroll
        for (int co = 0; co < CO; ++co) {
#pragma unroll
          for (int q = 0; q < CI / 4; ++q) {
            const float4 wv = *reinterpret_cast<const float4*>(wk + co * CI + 4 * q);
            acc[4 * q] = fmaf(uv[co], wv.x, acc[4 * q]);
            acc[4 * q + 1] = fmaf(uv[co], wv.y, acc[4 * q + 1]);
            acc[4 * q + 2] = fmaf(uv[co], wv.z, acc[4 * q + 2]);
            acc[4 * q + 3] = fmaf(uv[co], wv.w, acc[4 * q + 3]);
          }
        }
      }
      st_c<CI>(gf, g + fidx(gf, r.n, r.z, r.y, px), acc);
    }
  }
}

// part[block][ci][co][k] = sum over the block's tiles of x[p][ci] u[2p + k][co].
// A tile is 32 consecutive coarse voxels of one row; thread = (k, ci, CB-wide
// co block), 256 threads cover all 8*CI*CO outputs.
constexpr int kDTV = 32;
template <int CI, int CO>
__global__ void __launch_bounds__(256) deconv_wgrad_v(const float* __restrict__ x, Frame xf,
                                                      const float* __restrict__ u, Frame uf, long long ntiles,
                                                      float* __restrict__ part) {
  constexpr int CB = CI * CO * 8 / 256;
  static_assert(CB % 4 == 0 && CB <= CO && CO % CB == 0, "co block");
  __shared__ __align__(16) float xs[kDTV * CI];
  __shared__ __align__(16) float us[kDTV * 8 * CO];  // [v][k][co]
  const int t = threadIdx.x;
  const int cb = t % (CO / CB), ci = (t / (CO / CB)) % CI, k = t / (CI * (CO / CB));
  const int tiles_per_row = (xf.w + kDTV - 1) / kDTV;
  float acc[CB];
#pragma unroll
  for (int j = 0; j < CB; ++j) acc[j] = 0.f;
  for (long long ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
    const Row r = row_of(xf, ti / tiles_per_row);
    const int x0 = static_cast<int>(ti % tiles_per_row) * kDTV;
    const int nv = xf.w - x0 < kDTV ? xf.w - x0 : kDTV;
    for (int i = t; i < kDTV * CI / 4; i += blockDim.x) {
      const int v = i / (CI / 4), q = i % (CI / 4);
      float4 val = make_float4(0.f, 0.f, 0.f, 0.f);
      if (v < nv) val = *reinterpret_cast<const float4*>(x + fidx(xf, r.n, r.z, r.y, x0 + v) + 4 * q);
      *reinterpret_cast<float4*>(xs + v * CI + 4 * q) = val;
    }
    // children rows (2z + a, 2y + b), fine x in [2 x0, 2 x0 + 64)
    for (int i = t; i < 4 * 2 * kDTV * CO / 4; i += blockDim.x) {
      const int q = i % (CO / 4);
      const int fx = (i / (CO / 4)) % (2 * kDTV);
      const int ab = i / (CO / 4 * 2 * kDTV);
      const int a = ab >> 1, b = ab & 1, v = fx >> 1, c = fx & 1;
      float4 val = make_float4(0.f, 0.f, 0.f, 0.f);
      if (v < nv)
        val = *reinterpret_cast<const float4*>(u + fidx(uf, r.n, 2 * r.z + a, 2 * r.y + b, 2 * x0 + fx) + 4 * q);
      *reinterpret_cast<float4*>(us + (v * 8 + (ab * 2 + c)) * CO + 4 * q) = val;
    }
    __syncthreads();
#pragma unroll 4
    for (int v = 0; v < kDTV; ++v) {
      const float xv = xs[v * CI + ci];
      const float* up = us + (v * 8 + k) * CO + cb * CB;
#pragma unroll
      for (int q = 0; q < CB / 4; ++q) {
        const float4 uv = *reinterpret_cast<const float4*>(up + 4 * q);
        acc[4 * q] = fmaf(xv, uv.x, acc[4 * q]);
        acc[4 * q + 1] = fmaf(xv, uv.y, acc[4 * q + 1]);
        acc[4 * q + 2] = fmaf(xv, uv.z, acc[4 * q + 2]);
        acc[4 * q + 3] = fmaf(xv, uv.w, acc[4 * q + 3]);
      }
    }
    __syncthreads();
  }
  float* out = part + (long long)blockIdx.x * 8 * CI * CO;
#pragma unroll
  for (int j = 0; j < CB; ++j) out[(ci * CO + cb * CB + j) * 8 + k] = acc[j];
}

// concat / split over float4 channel groups (both parts' channel counts % 4 == 0)
__global__ void concat_v(const float* __restrict__ a, Frame af, const float* __restrict__ b, Frame bf,
                         float* __restrict__ y, Frame yf) {
  const int qa = af.c / 4, qy = yf.c / 4;
  const long long nrows = (long long)yf.n * yf.d * yf.h;
  const int per_row = yf.w * qy;
  for (long long row = blockIdx.x; row < nrows; row += gridDim.x) {
    const Row r = row_of(yf, row);
    const float* ar = a + fidx(af, r.n, r.z, r.y, 0);
    const float* br = b + fidx(bf, r.n, r.z, r.y, 0);
    float* yr = y + fidx(yf, r.n, r.z, r.y, 0);
    for (int j = threadIdx.x; j < per_row; j += blockDim.x) {
      const int px = j / qy, q = j - px * qy;
      const float4 v = q < qa ? *reinterpret_cast<const float4*>(ar + (long long)px * af.c + 4 * q)
                              : *reinterpret_cast<const float4*>(br + (long long)px * bf.c + 4 * (q - qa));
      *reinterpret_cast<float4*>(yr + 4 * j) = rnd4(yf, v);
    }
  }
}
__global__ void split_v(const float* __restrict__ u, Frame uf, float* __restrict__ ga, Frame gaf,
                        float* __restrict__ gb, Frame gbf, int acc_b) {
  const int qa = gaf.c / 4, qu = uf.c / 4;
  const long long nrows = (long long)uf.n * uf.d * uf.h;
  const int per_row = uf.w * qu;
  for (long long row = blockIdx.x; row < nrows; row += gridDim.x) {
    const Row r = row_of(uf, row);
    const float* ur = u + fidx(uf, r.n, r.z, r.y, 0);
    float* ar = ga + fidx(gaf, r.n, r.z, r.y, 0);
    float* br = gb + fidx(gbf, r.n, r.z, r.y, 0);
    for (int j = threadIdx.x; j < per_row; j += blockDim.x) {
      const int px = j / qu, q = j - px * qu;
      const float4 v = *reinterpret_cast<const float4*>(ur + 4 * j);
      if (q < qa) {
        *reinterpret_cast<float4*>(ar + (long long)px * gaf.c + 4 * q) = v;
      } else {
        float4* p = reinterpret_cast<float4*>(br + (long long)px * gbf.c + 4 * (q - qa));
        float4 o = v;
        if (acc_b) {
          const float4 old = *p;
          o = make_float4(old.x + v.x, old.y + v.y, old.z + v.z, old.w + v.w);
        }
        *p = rnd4(gbf, o);
      }
    }
  }
}

int rows_grid_u(const Frame& f, int per_sm) {
  const long long rows = (long long)f.n * f.d * f.h;
  const long long cap = (long long)num_sms() * per_sm;
  return static_cast<int>(rows < 1 ? 1 : (rows > cap ? cap : rows));
}

}  // namespace

#define DECONV_CASES(X) X(16, 8) X(32, 16) X(32, 8) X(16, 16) X(32, 32)

int deconv_vec_supported(int cin, int cout) {
#define D_OK(a, b) if (cin == a && cout == b) return 1;
  DECONV_CASES(D_OK)
#undef D_OK
  return 0;
}

int deconv_fwd_vec(const float* x, const Frame& xf, const float* w, float* y, const Frame& yf, cudaStream_t st) {
#define D_F(a, b)                                                               \
  if (xf.c == a && yf.c == b) {                                                 \
    deconv_fwd_v<a, b><<<rows_grid_u(xf, 16), 128, 0, st>>>(x, xf, w, y, yf);   \
    VPX_LAUNCH_CHECK();                                                         \
    return VPX_OK;                                                              \
  }
  DECONV_CASES(D_F)
#undef D_F
  VPX_FAIL(VPX_ERR_UNSUPPORTED, "deconv %d -> %d", xf.c, yf.c);
}

int deconv_dgrad_vec(const float* u, const Frame& uf, const float* w, float* g, const Frame& gf, cudaStream_t st) {
#define D_D(a, b)                                                               \
  if (gf.c == a && uf.c == b) {                                                 \
    deconv_dgrad_v<a, b><<<rows_grid_u(gf, 16), 128, 0, st>>>(u, uf, w, g, gf); \
    VPX_LAUNCH_CHECK();                                                         \
    return VPX_OK;                                                              \
  }
  DECONV_CASES(D_D)
#undef D_D
  VPX_FAIL(VPX_ERR_UNSUPPORTED, "deconv %d -> %d", gf.c, uf.c);
}

// Partials part[P][ci][co][k]; returns P through *parts (P <= max_parts).
int deconv_wgrad_vec(const float* x, const Frame& xf, const float* u, const Frame& uf, float* part, int max_parts,
                     int* parts, cudaStream_t st) {
  const long long ntiles = (long long)xf.n * xf.d * xf.h * ((xf.w + kDTV - 1) / kDTV);
  long long P = 8LL * num_sms();  // 8 resident blocks per SM hide the per-tile load latency
  if (P > max_parts) P = max_parts;
  if (P > ntiles) P = ntiles;
  if (P < 1) P = 1;
  *parts = static_cast<int>(P);
#define D_W(a, b)                                                                          \
  if (xf.c == a && uf.c == b) {                                                            \
    deconv_wgrad_v<a, b><<<static_cast<int>(P), 256, 0, st>>>(x, xf, u, uf, ntiles, part); \
    VPX_LAUNCH_CHECK();                                                                    \
    return VPX_OK;                                                                         \
  }
  DECONV_CASES(D_W)
#undef D_W
  VPX_FAIL(VPX_ERR_UNSUPPORTED, "deconv %d -> %d", xf.c, uf.c);
}

int concat_vec(const float* a, const Frame& af, const float* b, const Frame& bf, float* y, const Frame& yf,
               cudaStream_t st) {
  concat_v<<<rows_grid_u(yf, 16), 256, 0, st>>>(a, af, b, bf, y, yf);
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}

int split_vec(const float* u, const Frame& uf, float* ga, const Frame& gaf, float* gb, const Frame& gbf, int acc_b,
              cudaStream_t st) {
  split_v<<<rows_grid_u(uf, 16), 256, 0, st>>>(u, uf, ga, gaf, gb, gbf, acc_b);
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}

}  // namespace vpx
