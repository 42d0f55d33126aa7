// CUDA-core convolution kernels (shapes outside the tcgen05 fast paths).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace vpx {

// NDHWC halo frame: interior extents (n,c,d,h,w) and margins (md,mh,mw).
// Allocation is [n][d+2md][h+2mh][w+2mw][c], contiguous.
struct Frame {
  int n, c, d, h, w, md, mh, mw;
  int rnd;  // 1: values stored into this frame are rounded to nearest TF32
};

// Numeric mode of the library (vpx_set_precision): 0 = TF32 tensor cores with
// round-to-nearest TF32 storage of activations/gradients, 1 = FP32 everywhere
// (CUDA-core direct kernels, no rounding; the strict-parity mode).
int precision();

int num_sms();
int conv_fwd_simt(const float* x, const Frame& xf, const float* w, int k, int s, float* y,
                  const Frame& yf, cudaStream_t st, int act = 0, float slope = 0.f);
int conv_bwd_data_simt(const float* u, const Frame& uf, const float* w, int k, int s, float* xg,
                       const Frame& gf, cudaStream_t st);
long long wgrad_simt_parts(const Frame& uf);
int reduce_partials(const float* part, int P, long long len, float* out, int accumulate,
                    cudaStream_t st);
int reduce_partials_slice(const float* part, int P, long long len, int inner, long long out_stride,
                          long long out_off, float* out, int accumulate, cudaStream_t st);
int wgrad_tc_supported(const Frame& xf, const Frame& uf, int stride);
int wgrad_tc_parts(const Frame& xf, const Frame& uf);
int wgrad_tc_tapmajor(const Frame& xf);
int reduce_partials_tapmajor(const float* part, int P, int cout, int cin, long long out_co_stride, int ci0,
                             float* out, int accumulate, cudaStream_t st);
int conv_wgrad_tc(const float* x, const Frame& xf, const float* u, const Frame& uf, int stride, float* part,
                  cudaStream_t st);
int wgrad_ut_supported(const Frame& xf, const Frame& uf, int stride);
int wgrad_ut_parts(const Frame& uf);
int conv_wgrad_ut(const float* x, const Frame& xf, const float* u, const Frame& uf, float* part, cudaStream_t st);
int wgrad_g_supported(const Frame& xf, const Frame& uf, int stride);
int wgrad_g_parts(const Frame& uf);
int conv_wgrad_g(const float* x, const Frame& xf, const float* u, const Frame& uf, float* part, cudaStream_t st);
int c1_pooled_supported(const Frame& xf, const Frame& yf, const Frame& uf);
int c1_pooled_parts(const Frame& yf);
int conv_wgrad_c1_pooled(const float* x, const Frame& xf, const float* y, const Frame& yf, const float* up,
                         const Frame& uf, float slope, float* part, cudaStream_t st,
                         const uint16_t* mask = nullptr, bool u_direct = false);
int c1_direct_supported(const Frame& xf, const Frame& uf);
int c1_fwd_pool_supported(const Frame& xf, int cout, const Frame& pf);
long long c1_fwd_packed_bytes();
int c1_fwd_pack(const float* w, float* dst, cudaStream_t st);
int conv_c1_fwd_pool(const float* x, const Frame& xf, const float* wpack, float slope, float* pout,
                     const Frame& pf, uint16_t* mask, cudaStream_t st);
// conv_small.cu: 1x1x1 convs and 3x3x3 convs on 1 input channel (U-Net edges)
int small_conv_supported(int which, const Frame& xf, const Frame& of, int k, int s);
int small_wgrad_parts(const Frame& uf, int k);
int small_conv_fwd(const float* x, const Frame& xf, const float* w, int k, float* y, const Frame& yf, int act,
                   float slope, cudaStream_t st);
int small_conv_bwd_data(const float* u, const Frame& uf, const float* w, float* g, const Frame& gf,
                        cudaStream_t st);
int small_conv_wgrad(const float* x, const Frame& xf, const float* u, const Frame& uf, int k, float* part,
                     cudaStream_t st);
int conv_wgrad_simt(const float* x, const Frame& xf, const float* u, const Frame& uf, int k, int s,
                    float* wg, int accumulate, float* part, cudaStream_t st);

}  // namespace vpx
