// C-ABI entry points for the convolution passes (include/vpx.h) and the
// weight-packing kernel that arranges the UMMA B operand for conv_rowwin.cu.
//
// Replaces the reference's kernel boundary voxpar.kernels.conv3d_{fwd,
// bwd_data,bwd_filter} (reference pkg/src/voxpar/kernels/__init__.py:63-72,
// cyext.py:20-45): same math, device-resident NDHWC halo frames instead of
// host NCDHW arrays, explicit workspace instead of internal allocation.
#include <climits>
#include <cstdlib>
#include <vector>

#include "conv_common.h"
#include "conv_simt.h"
#include "ops_vec.h"
#include "vpx_host.h"
#include "vpx_round.cuh"

namespace vpx {

static int g_sm_limit = 0;  // vpx_set_sm_limit: 0 = every SM

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return g_sm_limit > 0 && g_sm_limit < n ? g_sm_limit : n;
}

// Pack OIDHW weights into the row-window B layout.
//   mode 0 (forward):  Weff[o][i][t] = w[o][i][t]            (O=cout, I=cin)
//   mode 1 (bwd data): Weff[o][i][t] = w[i][o][26 - t]       (O=cin,  I=cout)
// non-pair layout [g][t][c<CG][O][4]; pair layout (I == 4) [q<14][h<2][O][4], tap 2q+h.
__global__ void pack_rowwin_kernel(const float* __restrict__ w, int cout, int cin, int mode,
                                   int CG, int pair, float* __restrict__ out) {
  const int O = mode ? cin : cout;
  const int I = mode ? cout : cin;
  const long long total = pair ? 28LL * O * 4 : 27LL * I * O;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    long long t = idx;
    const int e = t % 4;
    t /= 4;
    const int o = t % O;
    t /= O;
    int tap, i;
    if (pair) {
      tap = static_cast<int>(t);  // t = 2q + h
      i = e;
    } else {
      const int c = t % CG;
      t /= CG;
      tap = t % 27;
      const int g = static_cast<int>(t / 27);
      i = 4 * (g * CG + c) + e;
    }
    float v = 0.f;
    if (tap < 27) {
      if (mode == 0)
        v = w[((long long)o * cin + i) * 27 + tap];
      else
        v = w[((long long)i * cin + o) * 27 + (26 - tap)];
    }
    out[idx] = tf32_rn(v);
  }
}

static Frame to_frame(const int* f) {
  return Frame{f[0], f[1], f[2], f[3], f[4], f[5], f[6], f[7], precision() == 0 ? 1 : 0};
}

static int check_frame(const int* f, const char* what) {
  for (int i = 0; i < 5; ++i)
    if (f[i] < 1) VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "%s: extent %d is %d", what, i, f[i]);
  for (int i = 5; i < 8; ++i)
    if (f[i] < 0 || f[i] > 1) VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "%s: margin %d is %d", what, i - 5, f[i]);
  return VPX_OK;
}

static long long packed_floats(int cin, int cout) {
  long long a = 27LL * cin * cout, b = 28LL * 4 * (cin > cout ? cin : cout);
  return a > b ? a : b;
}

static int encode_frame_map(CUtensorMap* map, const float* base, const Frame& f, int R, bool pair) {
  const uint64_t Wf = f.w + 2 * f.mw, Hf = f.h + 2 * f.mh, Df = f.d + 2 * f.md;
  uint64_t dims[5] = {(uint64_t)f.c, Wf, Hf, Df, (uint64_t)f.n};
  uint64_t strides[4] = {(uint64_t)f.c * 4, Wf * f.c * 4, Hf * Wf * f.c * 4, Df * Hf * Wf * f.c * 4};
  // pair (cin 4): 16-byte voxel rows; otherwise 8 channels as 32-byte SW32 rows
  uint32_t box[5] = {pair ? 4u : 8u, 130, (uint32_t)(R + 2), 3, 1};
  return encode_tiled(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(base), dims,
                      strides, box, pair ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_32B);
}

// One row-window launch: output frame region z in [zlo,zhi), y in [ylo,yhi),
// x in [0, wout) (wout % 128 == 0), input frame `in` (channels cin_eff).
static int rowwin_run(const float* in, const Frame& inf, const float* wpack, int cin_eff,
                      int cout_eff, float* out, const Frame& of, int zlo, int zhi, int ylo,
                      int yhi, int wout, cudaStream_t st, int act = 0, float slope = 0.f) {
  int R, CG;
  if (!rowwin_config(cin_eff, cout_eff, &R, &CG)) VPX_FAIL(VPX_ERR_UNSUPPORTED, "rowwin config");
  CUtensorMap map;
  int rc = encode_frame_map(&map, in, inf, R, cin_eff == 4);
  if (rc) return rc;
  ConvRowParams p{};
  p.zlo = zlo;
  p.zhi = zhi;
  p.ylo = ylo;
  p.yhi = yhi;
  p.nxseg = wout / 128;
  p.ngy = (yhi - ylo + R - 1) / R;
  p.n_groups = cin_eff == 4 ? 1 : cin_eff / (4 * CG);
  p.num_tiles = inf.n * (zhi - zlo) * p.ngy * p.nxseg;
  p.in_off_d = inf.md;
  p.in_off_h = inf.mh;
  p.in_off_w = inf.mw;
  p.wpack = wpack;
  p.out = out;
  const long long Wf = of.w + 2 * of.mw, Hf = of.h + 2 * of.mh, Df = of.d + 2 * of.md;
  p.out_sw = of.c;
  p.out_sh = Wf * of.c;
  p.out_sd = Hf * Wf * of.c;
  p.out_sn = Df * Hf * Wf * of.c;
  p.out_off_d = of.md;
  p.out_off_h = of.mh;
  p.out_off_w = of.mw;
  p.act = act;
  p.slope = slope;
  p.rnd = of.rnd;
  return launch_rowwin_any(map, p, cin_eff, cout_eff, st);
}

// Same launch for the height-taps-in-N kernel (conv_rowh.cu): bands of RB
// output rows, each streaming RB + 2 input rows.
static int rowh_run(const float* in, const Frame& inf, const float* wpack, int cin_eff, int cout_eff, float* out,
                    const Frame& of, int zlo, int zhi, int ylo, int yhi, int wout, cudaStream_t st, int act = 0,
                    float slope = 0.f) {
  CUtensorMap map;
  {
    const uint64_t Wf = inf.w + 2 * inf.mw, Hf = inf.h + 2 * inf.mh, Df = inf.d + 2 * inf.md;
    uint64_t dims[5] = {(uint64_t)inf.c, Wf, Hf, Df, (uint64_t)inf.n};
    uint64_t strides[4] = {(uint64_t)inf.c * 4, Wf * inf.c * 4, Hf * Wf * inf.c * 4, Df * Hf * Wf * inf.c * 4};
    // cin 4: one 16-byte voxel row per box row (interleaved layout); cin 8/16/32:
    // whole voxel rows in the K-major swizzle of matching width (conv_rowh.cu)
    const uint32_t ci = static_cast<uint32_t>(cin_eff);
    uint32_t box[5] = {ci, 130, 1, 3, 1};
    const CUtensorMapSwizzle sw = ci == 32   ? CU_TENSOR_MAP_SWIZZLE_128B
                                  : ci == 16 ? CU_TENSOR_MAP_SWIZZLE_64B
                                  : ci == 8  ? CU_TENSOR_MAP_SWIZZLE_32B
                                             : CU_TENSOR_MAP_SWIZZLE_NONE;
    if (int rc = encode_tiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(in), dims, strides, box,
                              sw))
      return rc;
  }
  ConvRowParams p{};
  p.zlo = zlo;
  p.zhi = zhi;
  p.ylo = ylo;
  p.yhi = yhi;
  p.nxseg = wout / 128;
  const long long cols = (long long)inf.n * (zhi - zlo) * p.nxseg;
  const int H = yhi - ylo;
  int rb = 64;  // band height: long bands (edge rows cost 2/(rb+2)) but >= 8 tasks per SM
  while (rb > 16 && cols * ((H + rb - 1) / rb) < 8LL * num_sms()) rb /= 2;
  if (rb > H) rb = H;
  p.ngy = rb;
  p.num_tiles = static_cast<int>(cols * ((H + rb - 1) / rb));
  p.in_off_d = inf.md;
  p.in_off_h = inf.mh;
  p.in_off_w = inf.mw;
  p.wpack = wpack;
  p.out = out;
  const long long Wf = of.w + 2 * of.mw, Hf = of.h + 2 * of.mh, Df = of.d + 2 * of.md;
  p.out_sw = of.c;
  p.out_sh = Wf * of.c;
  p.out_sd = Hf * Wf * of.c;
  p.out_sn = Df * Hf * Wf * of.c;
  p.out_off_d = of.md;
  p.out_off_h = of.mh;
  p.out_off_w = of.mw;
  p.act = act;
  p.slope = slope;
  p.rnd = of.rnd;
  return launch_rowh_any(map, p, cin_eff, cout_eff, st);
}

static bool rowh_off() {
  static int v = -1;
  if (v < 0) v = getenv("VPX_NO_ROWH") != nullptr;
  return v != 0;
}

static int pack(const float* w, int cout, int cin, int mode, float* dst, cudaStream_t st) {
  const int I = mode ? cout : cin, O = mode ? cin : cout;
  int R, CG;
  if (!rowwin_config(I, O, &R, &CG)) VPX_FAIL(VPX_ERR_UNSUPPORTED, "pack config");
  const int pair = I == 4;
  const long long total = pair ? 28LL * O * 4 : 27LL * I * O;
  int grid = static_cast<int>((total + 255) / 256);
  if (grid > 4096) grid = 4096;
  pack_rowwin_kernel<<<grid, 256, 0, st>>>(w, cout, cin, mode, CG, pair, dst);
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}

// ---------------------------------------------------------- packed weights
// Every conv pass packs its weights into the kernel's B layout.  The engine
// opts in to doing those packs ahead of the step, on a side stream that
// overlaps the first layer (vpx_prepack_begin / vpx_prepack_all /
// vpx_prepack_end): a pass whose (weights, direction, kernel, shape) entry
// was packed under the current weights version reads that buffer and skips
// its own pack.  Entries are recorded by the passes themselves (outside graph
// capture), so the engine needs no knowledge of which kernel a pass picks.
struct PackEntry {
  const float* w;
  int mode, path, cin, cout, stride;
  float* buf;
  unsigned long long ver;
};
static std::vector<PackEntry> g_packs;
static unsigned long long g_wver = 1;  // entries start at 0: never current
static int g_pack_on = 0;
static unsigned long long g_pack_owner = 0;

static long long pack_entry_bytes(int path, int mode, int cin, int cout) {
  if (path == kPackRowh) return mode ? rowh_packed_bytes(cout, cin) : rowh_packed_bytes(cin, cout);
  if (path == kPackRowwin) return packed_floats(cin, cout) * 4;
  return tapbox_workspace_bytes(cin, cout);
}

static int pack_entry(const PackEntry& e, cudaStream_t st) {
  if (e.path == kPackRowh) return rowh_pack(e.w, e.cout, e.cin, e.mode, e.buf, st);
  if (e.path == kPackRowwin) return pack(e.w, e.cout, e.cin, e.mode, e.buf, st);
  Frame dummy{};
  return conv_tapbox(e.mode, nullptr, dummy, e.w, e.cin, e.cout, e.stride, nullptr, dummy, 0, 0.f, e.buf, st,
                     tapbox_workspace_bytes(e.cin, e.cout), 0, 0, nullptr, true);
}

static void packcache_clear() {
  for (auto& e : g_packs) cudaFree(e.buf);
  g_packs.clear();
}

const float* packcache_get(const float* w, int mode, int path, int cin, int cout, int stride, cudaStream_t st) {
  if (!g_pack_on) return nullptr;
  for (const auto& e : g_packs)
    if (e.w == w && e.mode == mode && e.path == path && e.cin == cin && e.cout == cout && e.stride == stride)
      return e.ver == g_wver ? e.buf : nullptr;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return nullptr;
  PackEntry e{w, mode, path, cin, cout, stride, nullptr, 0};
  if (cudaMalloc(&e.buf, pack_entry_bytes(path, mode, cin, cout)) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  g_packs.push_back(e);
  return nullptr;
}


}  // namespace vpx

using vpx::Frame;

// Grid budget of the persistent kernels launched after this call (0 = all
// SMs).  Leaving a few SMs free lets communication kernels (NCCL) run next to
// a convolution instead of after it.

// Weight pre-packing (see packcache_get): begin a step for the weights
// owned by `owner` (the flat parameter buffer; a new owner drops every entry)
// and make a new weights version current; pack every recorded entry; end the
// step (the optimizer has changed the weights: no entry is current).
extern "C" int vpx_prepack_begin(unsigned long long owner, long long owner_numel) {
  const unsigned long long tok = owner ^ (static_cast<unsigned long long>(owner_numel) << 1);
  if (tok != vpx::g_pack_owner) {
    vpx::packcache_clear();
    vpx::g_pack_owner = tok;
  }
  vpx::g_pack_on = 1;
  ++vpx::g_wver;
  return VPX_OK;
}

extern "C" int vpx_prepack_all(void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  for (auto& e : vpx::g_packs) {
    if (int rc = vpx::pack_entry(e, st)) return rc;
    e.ver = vpx::g_wver;
  }
  return VPX_OK;
}

extern "C" int vpx_prepack_end(void) {
  ++vpx::g_wver;
  return VPX_OK;
}

extern "C" int vpx_prepack_entries(void) { return static_cast<int>(vpx::g_packs.size()); }

extern "C" int vpx_set_sm_limit(int n) {
  vpx::g_sm_limit = n < 0 ? 0 : n;
  return VPX_OK;
}

extern "C" long long vpx_conv3d_workspace_bytes(int cin, int cout, int k, const int* ufr) {
  Frame uf = vpx::to_frame(ufr);
  const long long k3 = (long long)k * k * k;
  long long packed = vpx::packed_floats(cin, cout) * 4;
  long long parts = vpx::wgrad_simt_parts(uf) * cout * cin * k3 * 4;
  const long long tc = (long long)vpx::num_sms() * cout * cin * 27 * 4;
  if (tc > parts) parts = tc;
  if (k == 1 || cin == 1) {  // conv_small.cu partials
    const long long sm = 8LL * vpx::num_sms() * cout * cin * k3 * 4;
    if (sm > parts) parts = sm;
  }
  const long long tb = vpx::tapbox_workspace_bytes(cin, cout);
  if (tb > packed) packed = tb;
  {  // tap-box split-K partial tiles: ks * base_tiles <= num_sms tiles of 128 x min(N, 256) (conv_tapbox.cu)
    const int nmax = cin > cout ? cin : cout;
    const long long tbp = (long long)vpx::num_sms() * 128 * (nmax < 256 ? nmax : 256) * 4;
    if (tbp > parts) parts = tbp;
  }
  const long long rh = vpx::rowh_packed_bytes(cin, cout) > vpx::rowh_packed_bytes(cout, cin)
                           ? vpx::rowh_packed_bytes(cin, cout)
                           : vpx::rowh_packed_bytes(cout, cin);
  if (rh > packed) packed = rh;
  if (cin == 4 && cout == 16 && vpx::c1_fwd_packed_bytes() > packed) packed = vpx::c1_fwd_packed_bytes();
  return ((packed + 255) / 256) * 256 + ((parts + 255) / 256) * 256;
}

// Output planes [zlo, zhi) only (zlo = INT_MIN: all).  Partial ranges are
// implemented by the row kernels; other paths report VPX_ERR_UNSUPPORTED so
// the caller runs the whole layer instead (halo overlap, layers.py).
static int conv_fwd_impl(const float* x, const int* xfr, const float* w, int k, int stride, float* y,
                         const int* yfr, int act, float slope, int zlo, int zhi, void* ws, long long ws_bytes,
                         void* stream) {
  if (int rc = vpx::check_frame(xfr, "conv fwd input")) return rc;
  if (int rc = vpx::check_frame(yfr, "conv fwd output")) return rc;
  Frame xf = vpx::to_frame(xfr), yf = vpx::to_frame(yfr);
  if (k < 1 || k % 2 == 0) VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "conv kernels must be odd, got %d", k);
  if (stride < 1 || stride > 2) VPX_FAIL(VPX_ERR_UNSUPPORTED, "stride %d", stride);
  if (yf.n != xf.n || yf.d != (xf.d + stride - 1) / stride || yf.h != (xf.h + stride - 1) / stride ||
      yf.w != (xf.w + stride - 1) / stride)
    VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "conv fwd: output (%d,%d,%d,%d) does not match input (%d,%d,%d,%d) stride %d",
             yf.n, yf.d, yf.h, yf.w, xf.n, xf.d, xf.h, xf.w, stride);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int cin = xf.c, cout = yf.c;
  int R, CG;
  const bool tc = vpx::precision() == 0;
  const bool full = zlo == INT_MIN;
  if (full) {
    zlo = 0;
    zhi = yf.d;
  } else if (zlo < 0 || zhi > yf.d || zlo >= zhi) {
    VPX_FAIL(VPX_ERR_OUT_OF_BOUNDS, "conv fwd: plane range [%d, %d) outside [0, %d)", zlo, zhi, yf.d);
  }
  if (tc && k == 3 && stride == 1 && yf.w % 128 == 0 && vpx::rowh_supported(cin, cout) && !vpx::rowh_off()) {
    if (ws_bytes < vpx::rowh_packed_bytes(cin, cout)) VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "workspace too small");
    const float* wpack = vpx::packcache_get(w, 0, vpx::kPackRowh, cin, cout, 1, st);
    if (!wpack) {
      if (int rc = vpx::rowh_pack(w, cout, cin, 0, static_cast<float*>(ws), st)) return rc;
      wpack = static_cast<float*>(ws);
    }
    return vpx::rowh_run(x, xf, wpack, cin, cout, y, yf, zlo, zhi, 0, yf.h, yf.w, st, act, slope);
  }
  if (tc && k == 3 && stride == 1 && yf.w % 128 == 0 && vpx::rowwin_config(cin, cout, &R, &CG) &&
      !getenv("VPX_NO_ROWWIN")) {
    if (ws_bytes < vpx::packed_floats(cin, cout) * 4) VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "workspace too small");
    const float* wpack = vpx::packcache_get(w, 0, vpx::kPackRowwin, cin, cout, 1, st);
    if (!wpack) {
      if (int rc = vpx::pack(w, cout, cin, 0, static_cast<float*>(ws), st)) return rc;
      wpack = static_cast<float*>(ws);
    }
    return vpx::rowwin_run(x, xf, wpack, cin, cout, y, yf, zlo, zhi, 0, yf.h, yf.w, st, act, slope);
  }
  if (!full && (zlo != 0 || zhi != yf.d)) VPX_FAIL(VPX_ERR_UNSUPPORTED, "conv fwd: plane ranges need a row kernel");
  if (tc && k == 3 && cin % 4 == 0 && vpx::tapbox_supported(cin, cout, 0)) {
    if (ws_bytes < vpx::tapbox_workspace_bytes(cin, cout)) VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "workspace too small");
    return vpx::conv_tapbox(0, x, xf, w, cin, cout, stride, y, yf, act, slope, ws, st, ws_bytes, 0, 0,
                            vpx::packcache_get(w, 0, vpx::kPackTapbox, cin, cout, stride, st));
  }
  if (vpx::small_conv_supported(0, xf, yf, k, stride) && !getenv("VPX_NO_SMALL"))
    return vpx::small_conv_fwd(x, xf, w, k, y, yf, act, slope, st);
  vpx::note_fallback();
  return vpx::conv_fwd_simt(x, xf, w, k, stride, y, yf, st, act, slope);
}

extern "C" int vpx_conv3d_fwd_act(const float* x, const int* xfr, const float* w, int k, int stride,
                                  float* y, const int* yfr, int act, float slope, void* ws,
                                  long long ws_bytes, void* stream) {
  return conv_fwd_impl(x, xfr, w, k, stride, y, yfr, act, slope, INT_MIN, 0, ws, ws_bytes, stream);
}

extern "C" int vpx_conv3d_fwd_act_range(const float* x, const int* xfr, const float* w, int k, int stride,
                                        float* y, const int* yfr, int act, float slope, int zlo, int zhi,
                                        void* ws, long long ws_bytes, void* stream) {
  return conv_fwd_impl(x, xfr, w, k, stride, y, yfr, act, slope, zlo, zhi, ws, ws_bytes, stream);
}

extern "C" int vpx_conv3d_fwd(const float* x, const int* xfr, const float* w, int k, int stride,
                              float* y, const int* yfr, void* ws, long long ws_bytes,
                              void* stream) {
  return vpx_conv3d_fwd_act(x, xfr, w, k, stride, y, yfr, 0, 0.f, ws, ws_bytes, stream);
}

static int conv_bwd_data_impl(const float* u, const int* ufr, const float* w, int k, int stride, float* xg,
                              const int* gfr, int zlo, int zhi, void* ws, long long ws_bytes, void* stream) {
  if (int rc = vpx::check_frame(ufr, "conv bwd_data upstream")) return rc;
  if (int rc = vpx::check_frame(gfr, "conv bwd_data output")) return rc;
  Frame uf = vpx::to_frame(ufr), gf = vpx::to_frame(gfr);
  if (k < 1 || k % 2 == 0) VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "conv kernels must be odd, got %d", k);
  if (uf.n != gf.n || uf.d != (gf.d + stride - 1) / stride || uf.h != (gf.h + stride - 1) / stride ||
      uf.w != (gf.w + stride - 1) / stride)
    VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "conv bwd_data: upstream does not match input extents");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int cout = uf.c, cin = gf.c;
  int R, CG;
  const bool tc = vpx::precision() == 0;
  // output planes of the gradient frame, margins included: [-md, d + md)
  const bool full = zlo == INT_MIN;
  if (full) {
    zlo = -gf.md;
    zhi = gf.d + gf.md;
  } else if (zlo < -gf.md || zhi > gf.d + gf.md || zlo >= zhi) {
    VPX_FAIL(VPX_ERR_OUT_OF_BOUNDS, "conv bwd_data: plane range [%d, %d) outside the frame", zlo, zhi);
  }
  if (tc && k == 3 && stride == 1 && gf.mw == 0 && gf.w % 128 == 0 && vpx::rowh_supported(cout, cin) &&
      !vpx::rowh_off()) {
    if (ws_bytes < vpx::rowh_packed_bytes(cout, cin)) VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "workspace too small");
    const float* wpack = vpx::packcache_get(w, 1, vpx::kPackRowh, cin, cout, 1, st);
    if (!wpack) {
      if (int rc = vpx::rowh_pack(w, cout, cin, 1, static_cast<float*>(ws), st)) return rc;
      wpack = static_cast<float*>(ws);
    }
    return vpx::rowh_run(u, uf, wpack, cout, cin, xg, gf, zlo, zhi, -gf.mh, gf.h + gf.mh, gf.w, st);
  }
  if (tc && k == 3 && stride == 1 && gf.mw == 0 && gf.w % 128 == 0 &&
      vpx::rowwin_config(cout, cin, &R, &CG) && !getenv("VPX_NO_ROWWIN")) {
    if (ws_bytes < vpx::packed_floats(cin, cout) * 4) VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "workspace too small");
    const float* wpack = vpx::packcache_get(w, 1, vpx::kPackRowwin, cin, cout, 1, st);
    if (!wpack) {
      if (int rc = vpx::pack(w, cout, cin, 1, static_cast<float*>(ws), st)) return rc;
      wpack = static_cast<float*>(ws);
    }
    return vpx::rowwin_run(u, uf, wpack, cout, cin, xg, gf, zlo, zhi, -gf.mh, gf.h + gf.mh, gf.w, st);
  }
  if (!full) VPX_FAIL(VPX_ERR_UNSUPPORTED, "conv bwd_data: plane ranges need a row kernel");
  if (tc && k == 3 && cout % 4 == 0 && vpx::tapbox_supported(cin, cout, 1)) {
    if (ws_bytes < vpx::tapbox_workspace_bytes(cin, cout)) VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "workspace too small");
    return vpx::conv_tapbox(1, u, uf, w, cin, cout, stride, xg, gf, 0, 0.f, ws, st, ws_bytes, 0, 0,
                            vpx::packcache_get(w, 1, vpx::kPackTapbox, cin, cout, stride, st));
  }
  if (k == 1 && vpx::small_conv_supported(1, uf, gf, k, stride) && !getenv("VPX_NO_SMALL"))
    return vpx::small_conv_bwd_data(u, uf, w, xg, gf, st);
  vpx::note_fallback();
  return vpx::conv_bwd_data_simt(u, uf, w, k, stride, xg, gf, st);
}

// Filter gradient; cin_total > 0 selects slice mode: x holds input channels
// [ci0, ci0 + xf.c) of a weight tensor with cin_total input channels and only
// that slice of wg is written (a conv whose input is a channel concat).
static int conv_bwd_filter_impl(const float* x, const int* xfr, const float* u, const int* ufr, int k, int stride,
                                float* wg, int accumulate, int ci0, int cin_total, void* ws, long long ws_bytes,
                                void* stream) {
  if (int rc = vpx::check_frame(xfr, "conv bwd_filter input")) return rc;
  if (int rc = vpx::check_frame(ufr, "conv bwd_filter upstream")) return rc;
  Frame xf = vpx::to_frame(xfr), uf = vpx::to_frame(ufr);
  if (k < 1 || k % 2 == 0) VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "conv kernels must be odd, got %d", k);
  if (uf.n != xf.n || uf.d != (xf.d + stride - 1) / stride || uf.h != (xf.h + stride - 1) / stride ||
      uf.w != (xf.w + stride - 1) / stride)
    VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "conv bwd_filter: upstream does not match input extents");
  const bool slice = cin_total > 0;
  if (slice && (ci0 < 0 || ci0 + xf.c > cin_total))
    VPX_FAIL(VPX_ERR_OUT_OF_BOUNDS, "conv bwd_filter: channel slice [%d, %d) outside %d", ci0, ci0 + xf.c, cin_total);
  long long need = vpx_conv3d_workspace_bytes(xf.c, uf.c, k, ufr);
  if (ws_bytes < need) VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "workspace too small (%lld < %lld)", ws_bytes, need);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  float* part = reinterpret_cast<float*>(static_cast<char*>(ws) +
                                         ((vpx::packed_floats(xf.c, uf.c) * 4 + 255) / 256) * 256);
  const int k3 = k * k * k;
  const long long len = (long long)uf.c * xf.c * k3;
  auto finish = [&](int P) {
    if (!slice) return vpx::reduce_partials(part, P, len, wg, accumulate, st);
    return vpx::reduce_partials_slice(part, P, len, xf.c * k3, (long long)cin_total * k3, (long long)ci0 * k3, wg,
                                      accumulate, st);
  };
  if (k == 3 && stride == 1 && vpx::c1_direct_supported(xf, uf)) {
    // 4 -> 16 channels: u in TMEM, x as dense 8-voxel rows (conv_c1bwd.cu, SRC 2)
    if (int rc = vpx::conv_wgrad_c1_pooled(x, xf, u, uf, u, uf, 0.f, part, st, nullptr, true)) return rc;
    return finish(vpx::c1_pooled_parts(uf));
  }
  if (k == 3 && vpx::wgrad_ut_supported(xf, uf, stride) && !getenv("VPX_NO_WGRAD_UT")) {
    if (int rc = vpx::conv_wgrad_ut(x, xf, u, uf, part, st)) return rc;
    return finish(vpx::wgrad_ut_parts(uf));
  }
  if (vpx::precision() == 0 && k == 3 && vpx::wgrad_g_supported(xf, uf, stride) && !getenv("VPX_NO_WGRAD_G")) {
    if (int rc = vpx::conv_wgrad_g(x, xf, u, uf, part, st)) return rc;
    return finish(vpx::wgrad_g_parts(uf));
  }
  if (vpx::precision() == 0 && k == 3 && vpx::wgrad_tc_supported(xf, uf, stride)) {
    if (int rc = vpx::conv_wgrad_tc(x, xf, u, uf, stride, part, st)) return rc;
    if (k3 == 27 && vpx::wgrad_tc_tapmajor(xf))
      return vpx::reduce_partials_tapmajor(part, vpx::wgrad_tc_parts(xf, uf), uf.c, xf.c,
                                           (long long)(slice ? cin_total : xf.c) * 27, slice ? ci0 : 0, wg, accumulate,
                                           st);
    return finish(vpx::wgrad_tc_parts(xf, uf));
  }
  if (vpx::small_conv_supported(2, xf, uf, k, stride) && !getenv("VPX_NO_SMALL")) {
    if (int rc = vpx::small_conv_wgrad(x, xf, u, uf, k, part, st)) return rc;
    return finish(vpx::small_wgrad_parts(uf, k));
  }
  if (slice) VPX_FAIL(VPX_ERR_UNSUPPORTED, "conv bwd_filter: channel slices need a partial-sum kernel");
  vpx::note_fallback();
  return vpx::conv_wgrad_simt(x, xf, u, uf, k, stride, wg, accumulate, part, st);
}

extern "C" int vpx_conv3d_bwd_filter(const float* x, const int* xfr, const float* u,
                                     const int* ufr, int k, int stride, float* wg, int accumulate,
                                     void* ws, long long ws_bytes, void* stream) {
  return conv_bwd_filter_impl(x, xfr, u, ufr, k, stride, wg, accumulate, 0, 0, ws, ws_bytes, stream);
}

extern "C" int vpx_conv3d_bwd_filter_cslice(const float* x, const int* xfr, const float* u, const int* ufr, int k,
                                            int stride, float* wg, int ci0, int cin_total, int accumulate,
                                            void* ws, long long ws_bytes, void* stream) {
  if (cin_total < 1) VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "cin_total %d", cin_total);
  return conv_bwd_filter_impl(x, xfr, u, ufr, k, stride, wg, accumulate, ci0, cin_total, ws, ws_bytes, stream);
}

extern "C" int vpx_conv3d_bwd_data(const float* u, const int* ufr, const float* w, int k, int stride, float* xg,
                                   const int* gfr, void* ws, long long ws_bytes, void* stream) {
  return conv_bwd_data_impl(u, ufr, w, k, stride, xg, gfr, INT_MIN, 0, ws, ws_bytes, stream);
}

extern "C" int vpx_conv3d_bwd_data_range(const float* u, const int* ufr, const float* w, int k, int stride,
                                         float* xg, const int* gfr, int zlo, int zhi, void* ws, long long ws_bytes,
                                         void* stream) {
  return conv_bwd_data_impl(u, ufr, w, k, stride, xg, gfr, zlo, zhi, ws, ws_bytes, stream);
}

extern "C" int vpx_pool_leaky_bwd_blocked(const float* y, const int* yfr, const float* up, const int* upfr,
                                          float* gb, float slope, int is_max, void* stream) {
  Frame yf = vpx::to_frame(yfr), uf = vpx::to_frame(upfr);
  if (yf.c % 4 || uf.c != yf.c || uf.d * 2 != yf.d || uf.h * 2 != yf.h || uf.w * 2 != yf.w)
    VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "pool/leaky blocked backward: extents");
  return vpx::pool_leaky_bwd_blocked(y, yf, up, uf, gb, slope, is_max, static_cast<cudaStream_t>(stream));
}

extern "C" int vpx_conv3d_fwd_leaky_pool_c4(const float* x, const int* xfr, const float* w, float slope,
                                            float* pout, const int* pfr, uint16_t* mask, void* ws, long long ws_bytes,
                                            void* stream) {
  if (int rc = vpx::check_frame(xfr, "first block input")) return rc;
  if (int rc = vpx::check_frame(pfr, "first block pooled output")) return rc;
  Frame xf = vpx::to_frame(xfr), pf = vpx::to_frame(pfr);
  if (!vpx::c1_fwd_pool_supported(xf, pf.c, pf)) VPX_FAIL(VPX_ERR_UNSUPPORTED, "fused first block: shape/mode");
  if (!(slope > 0.f && slope <= 1.f)) VPX_FAIL(VPX_ERR_UNSUPPORTED, "fused first block: slope must be in (0, 1]");
  if (ws_bytes < vpx::c1_fwd_packed_bytes()) VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  float* wpack = static_cast<float*>(ws);
  if (int rc = vpx::c1_fwd_pack(w, wpack, st)) return rc;
  return vpx::conv_c1_fwd_pool(x, xf, wpack, slope, pout, pf, mask, st);
}

// conv(k3 s1) -> LeakyReLU -> 2^3 average pool in one kernel for any layer
// with a fused instance: Cin 4 -> 16 (conv_c1fwd.cu) or the height-taps-in-N
// instances (conv_rowh.cu: 16 -> 32, 16 -> 16).  mask: cout/8 bytes per voxel.
extern "C" int vpx_conv3d_fwd_leaky_pool(const float* x, const int* xfr, const float* w, float slope, float* pout,
                                         const int* pfr, void* mask, void* ws, long long ws_bytes, void* stream) {
  if (int rc = vpx::check_frame(xfr, "fused conv+pool input")) return rc;
  if (int rc = vpx::check_frame(pfr, "fused conv+pool output")) return rc;
  Frame xf = vpx::to_frame(xfr), pf = vpx::to_frame(pfr);
  const int cin = xf.c, cout = pf.c;
  if (cin == 4 && cout == 16)
    return vpx_conv3d_fwd_leaky_pool_c4(x, xfr, w, slope, pout, pfr, static_cast<uint16_t*>(mask), ws, ws_bytes,
                                        stream);
  if (vpx::precision() != 0 || !vpx::rowh_pool_instance(cin, cout))
    VPX_FAIL(VPX_ERR_UNSUPPORTED, "fused conv+pool: %d -> %d channels / mode", cin, cout);
  if (xf.w % 128 || xf.d % 2 || xf.h % 2 || xf.mw || pf.n != xf.n || pf.d * 2 != xf.d || pf.h * 2 != xf.h ||
      pf.w * 2 != xf.w)
    VPX_FAIL(VPX_ERR_UNSUPPORTED, "fused conv+pool: extents");
  if (!(slope > 0.f && slope <= 1.f)) VPX_FAIL(VPX_ERR_UNSUPPORTED, "fused conv+pool: slope must be in (0, 1]");
  if (ws_bytes < vpx::rowh_packed_bytes(cin, cout)) VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const float* wpack = vpx::packcache_get(w, 0, vpx::kPackRowh, cin, cout, 1, st);
  if (!wpack) {
    if (int rc = vpx::rowh_pack(w, cout, cin, 0, static_cast<float*>(ws), st)) return rc;
    wpack = static_cast<float*>(ws);
  }
  CUtensorMap map;
  {
    const uint64_t Wf = xf.w + 2 * xf.mw, Hf = xf.h + 2 * xf.mh, Df = xf.d + 2 * xf.md;
    uint64_t dims[5] = {(uint64_t)cin, Wf, Hf, Df, (uint64_t)xf.n};
    uint64_t strides[4] = {(uint64_t)cin * 4, Wf * cin * 4, Hf * Wf * cin * 4, Df * Hf * Wf * cin * 4};
    uint32_t box[5] = {(uint32_t)cin, 130, 1, 3, 1};
    const CUtensorMapSwizzle sw = cin == 32   ? CU_TENSOR_MAP_SWIZZLE_128B
                                  : cin == 16 ? CU_TENSOR_MAP_SWIZZLE_64B
                                              : CU_TENSOR_MAP_SWIZZLE_32B;
    if (int rc = vpx::encode_tiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(x), dims, strides,
                                   box, sw))
      return rc;
  }
  vpx::RowhPoolParams p{};
  p.n = xf.n;
  p.d = xf.d;
  p.h = xf.h;
  p.w = xf.w;
  p.nxseg = xf.w / 128;
  p.rb = 16 < xf.h ? 16 : xf.h;
  p.nbands = (xf.h + p.rb - 1) / p.rb;
  p.zpairs = xf.d / 2;
  p.num_tasks = xf.n * p.zpairs * p.nbands * p.nxseg;
  p.in_off_d = xf.md;
  p.in_off_h = xf.mh;
  p.in_off_w = xf.mw;
  p.wpack = wpack;
  p.slope = slope;
  p.pout = pout;
  const long long Wf = pf.w + 2 * pf.mw, Hf = pf.h + 2 * pf.mh, Df = pf.d + 2 * pf.md;
  p.p_sw = pf.c;
  p.p_sh = Wf * pf.c;
  p.p_sd = Hf * Wf * pf.c;
  p.p_sn = Df * Hf * Wf * pf.c;
  p.p_off_d = pf.md;
  p.p_off_h = pf.mh;
  p.p_off_w = pf.mw;
  p.rnd = pf.rnd;
  p.mask = static_cast<uint8_t*>(mask);
  return vpx::launch_rowh_pool_any(map, p, cin, cout, st);
}

extern "C" int vpx_conv3d_bwd_filter_c4_pooled_mask(const float* x, const int* xfr, const uint16_t* mask,
                                                    const int* mfr, const float* up, const int* upfr, float slope,
                                                    float* wg, int accumulate, void* ws, long long ws_bytes,
                                                    void* stream) {
  Frame xf = vpx::to_frame(xfr), mf = vpx::to_frame(mfr), uf = vpx::to_frame(upfr);
  if (mf.md || mf.mh || mf.mw || !vpx::c1_pooled_supported(xf, mf, uf))
    VPX_FAIL(VPX_ERR_UNSUPPORTED, "pooled c1 filter gradient (mask): shape/mode");
  const int P = vpx::c1_pooled_parts(mf);
  const long long need = (long long)P * 16 * 4 * 27 * 4;
  if (ws_bytes < need) VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  float* part = static_cast<float*>(ws);
  if (int rc = vpx::conv_wgrad_c1_pooled(x, xf, nullptr, mf, up, uf, slope, part, st, mask)) return rc;
  return vpx::reduce_partials(part, P, 16 * 4 * 27, wg, accumulate, st);
}

extern "C" int vpx_pool_leaky_bwd(const float* y, const int* yfr, const float* up, const int* upfr, float* g,
                                  const int* gfr, float slope, int is_max, void* stream) {
  Frame yf = vpx::to_frame(yfr), uf = vpx::to_frame(upfr), gf = vpx::to_frame(gfr);
  if (yf.c % 4 || uf.c != yf.c || gf.c != yf.c || uf.d * 2 != yf.d || uf.h * 2 != yf.h || uf.w * 2 != yf.w ||
      gf.d != yf.d || gf.h != yf.h || gf.w != yf.w || gf.n != yf.n || uf.n != yf.n)
    VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "pool/leaky backward: extents");
  return vpx::pool_leaky_bwd(y, yf, up, uf, g, gf, slope, is_max, static_cast<cudaStream_t>(stream));
}

// Same backward (average pool only) from the fused forward's sign mask
// (mfr = {n, C, d, h, w, 0, 0, 0}: the mask's voxel grid, C/8 bytes per voxel).
extern "C" int vpx_pool_leaky_bwd_mask(const void* mask, const int* mfr, const float* up, const int* upfr, float* g,
                                       const int* gfr, float slope, void* stream) {
  Frame mf = vpx::to_frame(mfr), uf = vpx::to_frame(upfr), gf = vpx::to_frame(gfr);
  if (mf.md || mf.mh || mf.mw || uf.c != mf.c || gf.c != mf.c || uf.d * 2 != mf.d || uf.h * 2 != mf.h ||
      uf.w * 2 != mf.w || gf.d != mf.d || gf.h != mf.h || gf.w != mf.w || gf.n != mf.n || uf.n != mf.n)
    VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "pool/leaky backward (mask): extents");
  if (mf.c != 8 && mf.c != 16 && mf.c != 32) VPX_FAIL(VPX_ERR_UNSUPPORTED, "mask of %d channels", mf.c);
  return vpx::pool_leaky_bwd_mask(static_cast<const uint8_t*>(mask), up, uf, g, gf, slope,
                                  static_cast<cudaStream_t>(stream));
}

extern "C" int vpx_conv3d_bwd_filter_c4(const float* x, const int* xfr, const float* ub, const int* ufr,
                                        float* wg, int accumulate, void* ws, long long ws_bytes,
                                        void* stream) {
  Frame xf = vpx::to_frame(xfr), uf = vpx::to_frame(ufr);
  if (!vpx::wgrad_c4_supported(xf, uf)) VPX_FAIL(VPX_ERR_UNSUPPORTED, "blocked c4 filter gradient: shape");
  if (uf.n != xf.n || uf.d != xf.d || uf.h != xf.h || uf.w != xf.w)
    VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "blocked c4 filter gradient: extents");
  const int P = vpx::wgrad_c4_parts(uf);
  const long long need = (long long)P * uf.c * 4 * 27 * 4;
  if (ws_bytes < need) VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  float* part = static_cast<float*>(ws);
  if (int rc = vpx::conv_wgrad_c4(x, xf, ub, uf, part, st)) return rc;
  return vpx::reduce_partials(part, P, (long long)uf.c * 4 * 27, wg, accumulate, st);
}

// First-block filter gradient straight from the pooled gradient (avg pool).
extern "C" int vpx_conv3d_bwd_filter_c4_pooled(const float* x, const int* xfr, const float* y, const int* yfr,
                                               const float* up, const int* upfr, float slope, int is_max,
                                               float* wg, int accumulate, void* ws, long long ws_bytes,
                                               void* stream) {
  Frame xf = vpx::to_frame(xfr), yf = vpx::to_frame(yfr), uf = vpx::to_frame(upfr);
  if (is_max || !vpx::c1_pooled_supported(xf, yf, uf))
    VPX_FAIL(VPX_ERR_UNSUPPORTED, "pooled c1 filter gradient: shape/mode");
  const int P = vpx::c1_pooled_parts(yf);
  const long long need = (long long)P * 16 * 4 * 27 * 4;
  if (ws_bytes < need) VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  float* part = static_cast<float*>(ws);
  if (int rc = vpx::conv_wgrad_c1_pooled(x, xf, y, yf, up, uf, slope, part, st)) return rc;
  return vpx::reduce_partials(part, P, 16 * 4 * 27, wg, accumulate, st);
}

// ------------------------------------------------------------------ BF16 path
// 3x3x3 convolution forward / backward-data with bf16 operands on tcgen05
// kind::f16 (fp32 accumulation): input frame and output frame in bf16
// (NDHWC, channel rows of 2-byte elements), weights fp32 OIDHW rounded to
// bf16 by the pack kernel.  The tap-box implicit GEMM, 64-channel K chunks.
extern "C" int vpx_conv3d_fwd_bf16(const void* x, const int* xfr, const float* w, int k, int stride, void* y,
                                   const int* yfr, void* ws, long long ws_bytes, void* stream) {
  if (int rc = vpx::check_frame(xfr, "bf16 conv fwd input")) return rc;
  if (int rc = vpx::check_frame(yfr, "bf16 conv fwd output")) return rc;
  Frame xf = vpx::to_frame(xfr), yf = vpx::to_frame(yfr);
  if (k != 3 || stride < 1 || stride > 2) VPX_FAIL(VPX_ERR_UNSUPPORTED, "bf16 conv: k=3, stride 1/2 only");
  if (xf.c % 8 || !vpx::tapbox_supported(xf.c, yf.c, 0))
    VPX_FAIL(VPX_ERR_UNSUPPORTED, "bf16 conv fwd: channels %d -> %d", xf.c, yf.c);
  if (yf.n != xf.n || yf.d != (xf.d + stride - 1) / stride || yf.h != (xf.h + stride - 1) / stride ||
      yf.w != (xf.w + stride - 1) / stride)
    VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "bf16 conv fwd: output extents");
  if (ws_bytes < vpx::tapbox_workspace_bytes(xf.c, yf.c)) VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "workspace too small");
  return vpx::conv_tapbox(0, static_cast<const float*>(x), xf, w, xf.c, yf.c, stride, static_cast<float*>(y), yf, 0,
                          0.f, ws, static_cast<cudaStream_t>(stream), ws_bytes, 0, 3);
}

extern "C" int vpx_conv3d_bwd_data_bf16(const void* u, const int* ufr, const float* w, int k, int stride, void* g,
                                        const int* gfr, void* ws, long long ws_bytes, void* stream) {
  if (int rc = vpx::check_frame(ufr, "bf16 conv bwd_data input")) return rc;
  if (int rc = vpx::check_frame(gfr, "bf16 conv bwd_data output")) return rc;
  Frame uf = vpx::to_frame(ufr), gf = vpx::to_frame(gfr);
  if (k != 3 || stride < 1 || stride > 2) VPX_FAIL(VPX_ERR_UNSUPPORTED, "bf16 conv: k=3, stride 1/2 only");
  if (uf.c % 8 || !vpx::tapbox_supported(gf.c, uf.c, 1))
    VPX_FAIL(VPX_ERR_UNSUPPORTED, "bf16 conv bwd_data: channels %d <- %d", gf.c, uf.c);
  if (ws_bytes < vpx::tapbox_workspace_bytes(gf.c, uf.c)) VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "workspace too small");
  return vpx::conv_tapbox(1, static_cast<const float*>(u), uf, w, gf.c, uf.c, stride, static_cast<float*>(g), gf, 0,
                          0.f, ws, static_cast<cudaStream_t>(stream), ws_bytes, 0, 3);
}
