/* vpx.h -- C ABI of the B200-native voxpar hot path (libvpx.so).
 *
 * Every entry point takes plain device pointers, extents and a cudaStream_t
 * (passed as void*), launches stream-ordered asynchronous work with no hidden
 * synchronisation, never allocates or frees caller buffers, and returns an int
 * status: 0 on success, a negative VPX_ERR_* code otherwise, with a message
 * available from vpx_last_error().  The status codes map 1:1 onto the
 * reference's exception taxonomy (reference pkg/src/voxpar/errors.py:4-77).
 *
 * Layout conventions:
 *   activations  NDHWC fp32, stored in a halo frame [N][D+2md][H+2mh][W+2mw][C]
 *                whose margins m* are 1 in partitioned dims and 0 elsewhere;
 *   conv weights OIDHW fp32 exactly as the reference keeps them
 *                (reference layers/reference.py:68); packed per pass internally.
 *
 * The reference's kernel boundary this replaces is
 *   voxpar.kernels.conv3d_fwd / conv3d_bwd_data / conv3d_bwd_filter
 *   (reference pkg/src/voxpar/kernels/__init__.py:63-72) and its native
 *   Cython ABI _hot.conv3d_* (reference pkg/src/voxpar/kernels/_hot.pyx:19-93).
 */
#ifndef VPX_H_
#define VPX_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (errors.py names) */
#define VPX_OK 0
#define VPX_ERR_SHAPE_MISMATCH -1   /* errors.ShapeMismatch  (errors.py:23) */
#define VPX_ERR_NON_DIVISIBLE -2    /* errors.NonDivisible   (errors.py:8)  */
#define VPX_ERR_OUT_OF_BOUNDS -3    /* errors.OutOfBounds    (errors.py:19) */
#define VPX_ERR_LENGTH_MISMATCH -4  /* errors.LengthMismatch (errors.py:27) */
#define VPX_ERR_UNSUPPORTED -5      /* shape outside what the sm_100a kernels implement */
#define VPX_ERR_CUDA -6             /* CUDA runtime / driver failure */

/* Message for the last non-zero status returned on this thread. */
const char* vpx_last_error(void);
/* Library build tag (architecture, git revision). */
const char* vpx_version(void);
/* Total number of CUDA kernels this library has launched in this process. */
long long vpx_launch_count(void);
/* Conv passes that fell back to the generic CUDA-core kernels while in TF32
 * mode (no tcgen05 kernel covers the shape); bench.py reports it per step. */
long long vpx_fallback_count(void);
/* Numeric mode.  0 (default) = TF32: convolutions on tcgen05 tensor cores,
 * activations/gradients stored rounded to nearest TF32 so the MMA operands
 * are exact and the rounding unbiased (north-star tolerance rtol 1e-3).
 * 1 = FP32: every conv pass on CUDA-core direct kernels in fp32, no rounding
 * (the reference's own fp32 verify tolerance, rel 1e-5, reference cli.py:186). */
int vpx_set_precision(int mode);
/* Persistent-kernel grid budget for subsequent launches (0 = every SM): lets
 * NCCL kernels run beside an overlapped convolution. */
int vpx_set_sm_limit(int n);
int vpx_get_precision(void);

/* ------------------------------------------------------------ convolution --
 * Frames are described by int[8] = {n, c, d, h, w, md, mh, mw}: interior extents
 * and per-dimension halo margins (0 or 1); storage [n][d+2md][h+2mh][w+2mw][c].
 * Weights are OIDHW fp32 [cout][cin][k][k][k] exactly as the reference holds them
 * (reference layers/reference.py:68). Odd k, stride 1 or 2, "same" padding. */

/* Workspace bytes needed by the three passes for this layer (packed B operand
 * + filter-gradient partials). ufr describes the upstream-gradient frame. */
long long vpx_conv3d_workspace_bytes(int cin, int cout, int k, const int* ufr);

/* y = conv(x, w): replaces voxpar.kernels.conv3d_fwd(xpad, w, stride)
 * (reference kernels/__init__.py:63, _hot.pyx:19-41).  Writes the interior of
 * the y frame; margins of y are left untouched. */
int vpx_conv3d_fwd(const float* x, const int* xfr, const float* w, int k, int stride, float* y,
                   const int* yfr, void* ws, long long ws_bytes, void* stream);
/* Same, with the layer's LeakyReLU fused into the epilogue when act == 1:
 * y = leaky(conv(x, w), slope).  Because slope > 0, leaky(y) keeps the sign
 * of its input, so the backward pass needs only y (vpx_leaky_bwd(y, ...)). */
int vpx_conv3d_fwd_act(const float* x, const int* xfr, const float* w, int k, int stride, float* y,
                       const int* yfr, int act, float slope, void* ws, long long ws_bytes,
                       void* stream);

/* Same on output planes [zlo, zhi) only (row kernels; VPX_ERR_UNSUPPORTED
 * otherwise): lets the caller overlap a halo exchange with the planes that do
 * not read the halo. */
int vpx_conv3d_fwd_act_range(const float* x, const int* xfr, const float* w, int k, int stride, float* y,
                             const int* yfr, int act, float slope, int zlo, int zhi, void* ws, long long ws_bytes,
                             void* stream);

/* xg = adjoint scatter of u through w, over EVERY position of the xg frame
 * (interior and margins): replaces voxpar.kernels.conv3d_bwd_data(u, w,
 * stride, pad_spatial) (reference kernels/__init__.py:67, _hot.pyx:44-67). */
int vpx_conv3d_bwd_data(const float* u, const int* ufr, const float* w, int k, int stride,
                        float* xg, const int* gfr, void* ws, long long ws_bytes, void* stream);

/* bwd_data on gradient-frame planes [zlo, zhi), margins included (-md .. d+md). */
int vpx_conv3d_bwd_data_range(const float* u, const int* ufr, const float* w, int k, int stride, float* xg,
                              const int* gfr, int zlo, int zhi, void* ws, long long ws_bytes, void* stream);

/* Weight pre-packing (no reference counterpart: the reference convolves from
 * the OIDHW weights directly).  Every conv pass packs its weights into its
 * kernel's operand layout; between vpx_prepack_begin and vpx_prepack_end a
 * pass whose pack was recorded on an earlier step and redone by
 * vpx_prepack_all reads that buffer instead (the engine runs prepack_all on a
 * side stream beside the first layer).  owner/owner_numel: the flat weight
 * buffer (a new owner drops every recorded pack).  prepack_end: the weights
 * changed, no pack is current.  prepack_entries: the recorded packs. */
int vpx_prepack_begin(unsigned long long owner, long long owner_numel);
int vpx_prepack_all(void* stream);
int vpx_prepack_end(void);
int vpx_prepack_entries(void);

/* wg (=|+=) sum over voxels of u (x) x-patches; x frame margins must hold the
 * exchanged halos.  Replaces voxpar.kernels.conv3d_bwd_filter(xpad, u, stride,
 * kernel) (reference kernels/__init__.py:71, _hot.pyx:70-93).  Deterministic. */
int vpx_conv3d_bwd_filter(const float* x, const int* xfr, const float* u, const int* ufr, int k,
                          int stride, float* wg, int accumulate, void* ws, long long ws_bytes,
                          void* stream);

/* The filter gradient of input channels [ci0, ci0 + xf.c) of a weight tensor
 * (cout, cin_total, k, k, k): x is one operand of a channel concat (reference
 * engine.py:432-438 concatenates the U-Net skip before the conv), so the conv
 * after a concat can take its filter gradient from the concat's sources
 * instead of the concatenated frame.  Only that slice of wg is written. */
int vpx_conv3d_bwd_filter_cslice(const float* x, const int* xfr, const float* u, const int* ufr, int k,
                                 int stride, float* wg, int ci0, int cin_total, int accumulate, void* ws,
                                 long long ws_bytes, void* stream);

/* First-layer fast path (Cin = 4, Cout = 16, the CosmoFlow c1 block):
 * vpx_pool_leaky_bwd_blocked fuses the 2^3 pool backward and the LeakyReLU
 * backward (y = LeakyReLU output = pool input) and writes the conv-output
 * gradient in the 4-channel-blocked layout [C/4][n][d][h][w][4];
 * vpx_conv3d_bwd_filter_c4 computes the filter gradient from it on tcgen05.
 * ufr describes the logical (unblocked) gradient: {n, 16, d, h, w, 0, 0, 0}. */
int vpx_pool_leaky_bwd_blocked(const float* y, const int* yf, const float* up, const int* upf, float* gb,
                               float slope, int is_max, void* stream);
/* Fused 2^3 pool backward + LeakyReLU backward of a conv -> leaky -> pool block
 * (reference layers/reference.py:170-182 then :234-236): g = leaky'(y) *
 * pool_bwd(y, up), written into the frame gf; y is the LeakyReLU output (= pool
 * input).  One pass instead of pool-bwd write + leaky-bwd read/write. */
int vpx_pool_leaky_bwd(const float* y, const int* yf, const float* up, const int* upf, float* g, const int* gf,
                       float slope, int is_max, void* stream);
int vpx_conv3d_bwd_filter_c4(const float* x, const int* xfr, const float* ub, const int* ufr, float* wg,
                             int accumulate, void* ws, long long ws_bytes, void* stream);
/* The same filter gradient computed straight from the POOLED gradient `up`
 * (average pool only): u = leaky'(y) * up/8 is produced inside the kernel
 * (into TMEM, the MMA's A operand) and never written to memory; replaces the
 * pair above for TF32 mode (conv_c1bwd.cu).  y: LeakyReLU output frame,
 * up: pooled-gradient frame (half extents).  Frames may carry D/H margins,
 * not W margins.  VPX_ERR_UNSUPPORTED for max pooling or FP32 mode. */
int vpx_conv3d_bwd_filter_c4_pooled(const float* x, const int* xfr, const float* y, const int* yfr,
                                    const float* up, const int* upfr, float slope, int is_max, float* wg,
                                    int accumulate, void* ws, long long ws_bytes, void* stream);

/* Fused first-block forward (conv 4 -> 16, LeakyReLU, 2^3 average pool, TF32
 * mode, conv_c1fwd.cu): writes only the pooled frame pout (pfr: half extents)
 * and the sign mask[n][d][h][w] (bit co set when the stored activation is
 * >= 0); the full-resolution activation never reaches memory.  ws holds the
 * packed weights (vpx_conv3d_workspace_bytes(4, 16, 3, .) suffices). */
int vpx_conv3d_fwd_leaky_pool_c4(const float* x, const int* xfr, const float* w, float slope, float* pout,
                                 const int* pfr, uint16_t* mask, void* ws, long long ws_bytes, void* stream);
/* The same fusion for every conv -> LeakyReLU -> average-pool block with an
 * instance (Cin 4 -> 16 as above; 16 -> 32 and 16 -> 16 on the height-taps-in-N
 * kernel, e.g. CosmoFlow c2): pooled output + sign mask (cout/8 bytes per
 * voxel, [n][d][h][w]).  TF32 mode, 0 < slope <= 1, even D/H, W % 128 == 0. */
int vpx_conv3d_fwd_leaky_pool(const float* x, const int* xfr, const float* w, float slope, float* pout,
                              const int* pfr, void* mask, void* ws, long long ws_bytes, void* stream);
/* Average-pool + LeakyReLU backward from that mask (reference
 * layers/reference.py:170-173 then :234-236): g = leaky'(mask) * up / 8. */
int vpx_pool_leaky_bwd_mask(const void* mask, const int* mfr, const float* up, const int* upfr, float* g,
                            const int* gfr, float slope, void* stream);
/* Its backward: the c1 filter gradient from the pooled gradient and the sign
 * mask (mfr = {n, 16, d, h, w, 0, 0, 0} describes the mask's voxel grid). */
int vpx_conv3d_bwd_filter_c4_pooled_mask(const float* x, const int* xfr, const uint16_t* mask, const int* mfr,
                                         const float* up, const int* upfr, float slope, float* wg, int accumulate,
                                         void* ws, long long ws_bytes, void* stream);

/* ------------------------------------------------------- pointwise / pool --
 * reference layers/reference.py:149-236, layers/distributed.py:132-214.
 * All read/write frame interiors; is_max selects max (ties -> lowest index in
 * (d,h,w) C order) vs average 2^3 stride-2 pooling. */
int vpx_leaky_fwd(const float* x, const int* xf, float* y, const int* yf, float slope, void* stream);
int vpx_leaky_bwd(const float* x, const int* xf, const float* u, const int* uf, float* g,
                  const int* gf, float slope, void* stream);
int vpx_pool_fwd(const float* x, const int* xf, float* y, const int* yf, int is_max, void* stream);
int vpx_pool_bwd(const float* x, const int* xf, const float* u, const int* uf, float* g,
                 const int* gf, int is_max, void* stream);
int vpx_concat(const float* a, const int* af, const float* b, const int* bf, float* y, const int* yf,
               void* stream);
int vpx_split(const float* u, const int* uf, float* ga, const int* gaf, float* gb, const int* gbf,
              int acc_b, void* stream);
int vpx_add(const float* x, const int* xf, float* y, const int* yf, void* stream);
int vpx_copy(const float* x, const int* xf, float* y, const int* yf, void* stream);

/* -------------------------------------------------------------- batchnorm --
 * reference layers/reference.py:188-226, layers/distributed.py:152-201.
 * vpx_bn_sums: mode 0 -> out2c = [sum x, sum x^2]; mode 1 -> [sum u, sum u*xhat]
 * (xhat recomputed from x, mean, inv).  Local partials only: the caller
 * allreduces out2c over the tensor's rank group.  ws >= vpx_bn_workspace_bytes. */
long long vpx_bn_workspace_bytes(int c);
int vpx_bn_sums(const float* x, const int* xf, const float* u, const int* uf, const float* mean,
                const float* inv, int mode, float* out2c, void* ws, void* stream);
int vpx_bn_stats(const float* sums, int c, double count, float eps, float momentum, float* mean,
                 float* inv, float* run_mean, float* run_var, void* stream);
int vpx_bn_apply(const float* x, const int* xf, const float* mean, const float* inv,
                 const float* gamma, const float* beta, float* y, const int* yf, void* stream);
/* BatchNorm apply + LeakyReLU in one pass (C % 4 == 0); same bits as
 * vpx_bn_apply then vpx_leaky_fwd into frames with y's rounding (reference
 * layers/reference.py:209-214 then :231-233). */
int vpx_bn_apply_leaky(const float* x, const int* xf, const float* mean, const float* inv, const float* gamma,
                       const float* beta, float slope, float* y, const int* yf, void* stream);
int vpx_bn_bwd_apply(const float* x, const int* xf, const float* u, const int* uf, const float* mean,
                     const float* inv, const float* gamma, const float* sums, double count, float* g,
                     const int* gf, void* stream);

/* ------------------------------------------------- transposed conv k2 s2 --
 * reference layers/reference.py:99-144 (w is (cin, cout, 2, 2, 2)). */
long long vpx_deconv_workspace_bytes(int cin, int cout);
/* TF32 mode: tcgen05 implicit GEMMs (forward: per fine parity class P a
 * coarse-voxel x Cout GEMM over Cin with a stride-2 scatter epilogue;
 * backward-data: a coarse-voxel x Cin GEMM over (P, Cout) gathering the fine
 * gradient with TMA element stride 2).  ws: vpx_deconv_workspace_bytes. */
int vpx_deconv_fwd(const float* x, const int* xf, const float* w, float* y, const int* yf, void* ws,
                   long long ws_bytes, void* stream);
int vpx_deconv_bwd_data(const float* u, const int* uf, const float* w, float* g, const int* gf, void* ws,
                        long long ws_bytes, void* stream);
int vpx_deconv_bwd_filter(const float* x, const int* xf, const float* u, const int* uf, float* wg,
                          int accumulate, void* ws, void* stream);

/* -------------------------------------------------------------- BF16 path --
 * 3x3x3 conv forward / backward-data with bf16 storage (input and output
 * frames NDHWC bf16, channel counts % 8 == 0) on tcgen05 kind::f16 with fp32
 * accumulation; weights fp32 OIDHW (rounded to bf16 when packed).  Same
 * semantics as vpx_conv3d_fwd / vpx_conv3d_bwd_data (reference _hot.pyx:19-67);
 * north-star tolerance rtol 2e-2 against the fp32 reference.  ws:
 * vpx_conv3d_workspace_bytes. */
int vpx_conv3d_fwd_bf16(const void* x, const int* xf, const float* w, int k, int stride, void* y, const int* yf,
                        void* ws, long long ws_bytes, void* stream);
int vpx_conv3d_bwd_data_bf16(const void* u, const int* uf, const float* w, int k, int stride, void* g,
                             const int* gf, void* ws, long long ws_bytes, void* stream);

/* ------------------------------------------------------------------- halo --
 * Copy the box {n0,z0,y0,x0,en,ez,ey,ex} (frame coordinates, margins included)
 * of a frame to a dense (n,z,y,x,c) buffer (mode 0, pack), back (mode 1,
 * unpack) or accumulate into the frame (mode 2, adjoint unpack).  Replaces the
 * slab copies of reference fabric.py:404-410,436-442 / tensor.py:388-409 and
 * the block moves of redistribute (reference layers/distributed.py:298-368). */
int vpx_halo_copy(float* frame, const int* ff, const int* box8, float* buf, int mode, void* stream);

/* Peer-memory halo mailboxes (CUDA IPC over NVLink, comm.py PeerHalo): after
 * packing a face into the neighbour's mailbox with vpx_halo_copy(peer ptr),
 * vpx_peer_signal bumps the neighbour's arrival counter (system-scope
 * atomic); vpx_peer_wait blocks the stream until the local counter exceeds
 * *expected, then increments *expected (device-side, graph-replayable).  A
 * neighbour that never arrives within timeout_ns sets *error and traps. */
int vpx_peer_signal(unsigned long long* peer_flag, void* stream);
int vpx_peer_wait(const unsigned long long* flag, unsigned long long* expected, long long timeout_ns, int* error,
                  void* stream);

/* One halo round (one partitioned dim, both sides) in ONE kernel over the same
 * mailboxes: pack each face straight into the neighbour's mailbox (peer
 * stores), release it with a system-scope increment of the neighbour's flag
 * once every block has packed, wait (acquire) for the neighbours' faces and
 * unpack (mode 1) or accumulate (mode 2, adjoint round) them into the frame.
 * Replaces pack + vpx_peer_signal + vpx_peer_wait + unpack per side; one
 * dimension step of reference fabric.py:380-411 (forward) / :414-443
 * (reverse).  `faces` = 2 x 32 int64 per face (side -1, side +1):
 *   [0] send?  [1..8] send box {n0,z0,y0,x0,en,ez,ey,ex}  [9] peer mailbox
 *   [10] peer flag  [11] recv?  [12..19] recv box  [20] local mailbox
 *   [21] local flag  [22] local expected count  [23] (face 0 only) three u32
 *   zero-initialised block counters for the round  [24] recv mode (1|2).
 * Channels must be a multiple of 4.  A neighbour that never arrives within
 * timeout_ns sets *error and traps. */
int vpx_halo_round_peer(float* frame, const int* ff, const long long* faces, long long mailbox_bytes,
                        long long timeout_ns, int* error, void* stream);

/* ------------------------------------------------------------------- prng --
 * Pinned splitmix64 streams (reference prng.py:28-90), bit-exact with numpy:
 * value i = lo + (hi-lo) * ((mix(key + (i+1)*golden) >> 11) * 2^-53). */
int vpx_prng_uniform(unsigned long long key, long long n, double lo, double hi, float* out32,
                     double* out64, void* stream);
int vpx_prng_mask(unsigned long long key, long long n, double keep, unsigned char* out, void* stream);
/* Fill a frame interior from the stream whose counter runs over the NCDHW order
 * of the interior, starting at counter_base (synthetic batches, cli.py:112-125). */
int vpx_prng_volume(unsigned long long key, const int* ff, long long counter_base, double lo,
                    double hi, float* frame, void* stream);

/* -------------------------------------------------------------- optimizer --
 * reference model/optim.py:63-88; c1 = 1-b1^t, c2 = 1-b2^t. */
int vpx_adam(float* p, const float* g, float* m, float* v, long long n, float lr, float b1, float b2,
             float c1, float c2, float eps, void* stream);
int vpx_sgd(float* p, const float* g, long long n, float lr, void* stream);
/* Graph-replayable variants: per-step scalars read from device memory
 * (hyper = {lr, 1-b1^t, 1-b2^t}; key = the folded dropout key). */
int vpx_adam_dev(float* p, const float* g, float* m, float* v, long long n, const float* hyper, float b1,
                 float b2, float eps, void* stream);
int vpx_prng_mask_dev(const unsigned long long* key, long long n, double keep, unsigned char* out, void* stream);

/* ----------------------------------------------------------------- losses --
 * Per-voxel softmax cross entropy (reference layers/reference.py:282-307):
 * g = (softmax - onehot)/count, part[b] = per-block sums of -log p[label]. */
int vpx_xent(const float* logits, const int* lf, const long long* labels, double count, float* g,
             const int* gf, double* part, int nparts, void* stream);

/* ----------------------------------------------------------------- layout -- */
int vpx_layout_ncdhw_to_frame(const float* src, const int* ff, float* frame, void* stream);
int vpx_layout_frame_to_ncdhw(const float* frame, const int* ff, float* dst, void* stream);
/* Datastore ingest (reference datastore.py:429-444, HSB1 int16 storage):
 * int16 NCDHW block -> fp32 frame interior (conversion fused into the layout
 * change; TF32-rounded in TF32 mode), and int16 label slab -> int64 class ids. */
int vpx_layout_ncdhw_i16_to_frame(const int16_t* src, const int* ff, float* frame, void* stream);
/* Same from the datastore's int8 transfer copy (an int16 hyperslab whose
 * values fit int8: half the host->device bytes, identical fp32 values). */
int vpx_layout_ncdhw_i8_to_frame(const int8_t* src, const int* ff, float* frame, void* stream);
int vpx_convert_i16_to_i64(const int16_t* src, long long n, long long* dst, void* stream);


#ifdef __cplusplus
}
#endif
#endif /* VPX_H_ */
