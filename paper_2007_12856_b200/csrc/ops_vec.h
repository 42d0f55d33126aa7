// float4-vectorised memory-bound kernels (C % 4 == 0), see ops_vec.cu.
#pragma once
#include <cuda_runtime.h>

#include "conv_simt.h"

namespace vpx {
int leaky_fwd_vec(const float* x, const Frame& xf, float* y, const Frame& yf, float s, cudaStream_t st);
int leaky_bwd_vec(const float* x, const Frame& xf, const float* u, const Frame& uf, float* g, const Frame& gf,
                  float s, cudaStream_t st);
int pool_fwd_vec(const float* x, const Frame& xf, float* y, const Frame& yf, int is_max, cudaStream_t st);
int pool_bwd_vec(const float* x, const Frame& xf, const float* u, const Frame& uf, float* g, const Frame& gf,
                 int is_max, cudaStream_t st);
int bn_apply_vec(const float* x, const Frame& xf, const float* mean, const float* inv, const float* gamma,
                 const float* beta, float* y, const Frame& yf, cudaStream_t st, bool leaky = false, float slope = 0.f);
int bn_bwd_apply_vec(const float* x, const Frame& xf, const float* u, const Frame& uf, const float* mean,
                     const float* inv, const float* gamma, const float* sums, float inv_count, float* g,
                     const Frame& gf, cudaStream_t st);
int bn_sums_vec(const float* x, const Frame& xf, const float* u, const Frame& uf, const float* mean,
                const float* inv, int mode, double* part, int P, cudaStream_t st);
int pool_leaky_bwd(const float* y, const Frame& yf, const float* up, const Frame& uf, float* g, const Frame& gf,
                   float s, int is_max, cudaStream_t st);
int pool_leaky_bwd_mask(const uint8_t* mask, const float* up, const Frame& uf, float* g, const Frame& gf, float s,
                        cudaStream_t st);
int pool_leaky_bwd_blocked(const float* y, const Frame& yf, const float* up, const Frame& uf, float* gb,
                           float s, int is_max, cudaStream_t st);
int wgrad_c4_supported(const Frame& xf, const Frame& uf);
int wgrad_c4_parts(const Frame& uf);
int conv_wgrad_c4(const float* x, const Frame& xf, const float* ub, const Frame& uf, float* part,
                  cudaStream_t st);
// ops_unet.cu
int deconv_vec_supported(int cin, int cout);
int deconv_fwd_vec(const float* x, const Frame& xf, const float* w, float* y, const Frame& yf, cudaStream_t st);
int deconv_dgrad_vec(const float* u, const Frame& uf, const float* w, float* g, const Frame& gf, cudaStream_t st);
int deconv_wgrad_vec(const float* x, const Frame& xf, const float* u, const Frame& uf, float* part, int max_parts,
                     int* parts, cudaStream_t st);
int concat_vec(const float* a, const Frame& af, const float* b, const Frame& bf, float* y, const Frame& yf,
               cudaStream_t st);
int split_vec(const float* u, const Frame& uf, float* ga, const Frame& gaf, float* gb, const Frame& gbf, int acc_b,
              cudaStream_t st);
}  // namespace vpx
