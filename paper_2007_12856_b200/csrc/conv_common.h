// Shared declarations for the convolution kernels.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace vpx {

// Parameters of one row-window launch (see conv_rowwin.cu).
struct ConvRowParams {
  int zlo, zhi;  // output depth range (may extend to -1 / D for dgrad frame margins)
  int ylo, yhi;  // output row range
  int nxseg;     // W_out / 128
  int ngy;       // ceil((yhi - ylo) / R)
  int num_tiles;
  int n_groups;  // channel-chunk groups along K
  // map coordinate of input voxel for output voxel o and tap offset t in {0,1,2}:
  //   coord = o - 1 + t + in_off
  int in_off_d, in_off_h, in_off_w;
  const float* wpack;  // packed B operand, n_groups blocks
  float* out;
  long long out_sn, out_sd, out_sh, out_sw;  // element strides of the output frame
  int out_off_d, out_off_h, out_off_w;       // output voxel o lands at frame index o + off
  int act;                                   // 1: fused LeakyReLU epilogue
  float slope;
  int rnd;                                   // 1: round stores to nearest TF32
};

// Fused conv -> LeakyReLU -> 2^3 average pool on the height-taps-in-N kernel
// (conv_rowh.cu, conv_rowh_pool_kernel): pooled output + per-voxel sign mask.
struct RowhPoolParams {
  int n, d, h, w;            // conv output (= input interior) extents
  int nxseg, rb, nbands, zpairs, num_tasks;
  int in_off_d, in_off_h, in_off_w;
  const float* wpack;        // rowh B layout (rowh_pack mode 0)
  float slope;               // 0 < slope <= 1
  float* pout;               // pooled frame storage
  long long p_sn, p_sd, p_sh, p_sw;
  int p_off_d, p_off_h, p_off_w;
  int rnd;
  uint8_t* mask;             // [n][d][h][w] x cout/8 bytes, bit co = stored activation >= 0
};
int rowh_pool_instance(int cin, int cout);
int launch_rowh_pool_any(const CUtensorMap& xmap, const RowhPoolParams& p, int cin, int cout, cudaStream_t st);

int num_sms();
int rowwin_config(int cin, int cout, int* R, int* CG);
struct Frame;
long long tapbox_workspace_bytes(int cin, int cout);
int tapbox_supported(int cin, int cout, int mode, int kind = 0);
// k2s2 transposed-conv filter gradient on tcgen05 (deconv_wgrad.cu)
int deconv_wgrad_tc_supported(const Frame& xf, const Frame& uf);
int deconv_wgrad_tc_parts(const Frame& xf);
int deconv_wgrad_tc(const float* x, const Frame& xf, const float* u, const Frame& uf, float* part, cudaStream_t st);
int conv_tapbox(int mode, const float* in, const Frame& inf, const float* w, int cin, int cout, int stride,
                float* out, const Frame& of, int act, float slope, void* ws, cudaStream_t st, long long ws_bytes,
                int kind = 0, int bf16 = 0, const float* wpre = nullptr, bool pack_only = false);
// Packed-weight cache (conv_host.cu): the pack a conv pass would do, made
// ahead of time by vpx_prepack_all; nullptr when there is no current one.
enum PackPath { kPackRowh = 1, kPackRowwin = 2, kPackTapbox = 3 };
const float* packcache_get(const float* w, int mode, int path, int cin, int cout, int stride, cudaStream_t st);
int rowh_supported(int cin, int cout);
long long rowh_packed_bytes(int cin, int cout);
int rowh_pack(const float* w, int cout, int cin, int mode, float* dst, cudaStream_t st);
int launch_rowh_any(const CUtensorMap& xmap, const ConvRowParams& p, int cin, int cout, cudaStream_t st);
int launch_rowwin_any(const CUtensorMap& xmap, const ConvRowParams& p, int cin, int cout,
                      cudaStream_t st);

}  // namespace vpx
