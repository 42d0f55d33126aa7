// One halo round (one partitioned dim, both sides) over CUDA-IPC peer memory
// in ONE kernel: pack both boundary faces straight into the neighbours'
// mailboxes over NVLink, signal each neighbour once its face is complete
// (last-block detection, system-scope release), wait for the neighbours'
// faces, unpack (or accumulate, for the adjoint round) them into the frame
// margins.  Replaces pack + signal + wait + unpack (four launches per side)
// of the round in comm.PeerHalo, i.e. one dimension step of the reference's
// halo_exchange / reverse_halo_exchange (reference fabric.py:380-443).
//
// Deadlock freedom: a block waits only for the neighbour's face, never for
// another block of this kernel, and the grid is at most one block per SM
// (256 threads, no shared memory) so every block is resident and finishes its
// pack before it spins.  Counters live in device memory and return to their
// initial state at the end of every launch, so the round replays in a CUDA
// graph.
#include "conv_simt.h"
#include "vpx_host.h"

namespace vpx {
int num_sms();
}

namespace {

using vpx::Frame;

// int64 fields of one face in the descriptor (include/vpx.h)
enum : int {
  kSendValid = 0,
  kSendBox = 1,  // 8 fields
  kPeerBuf = 9,
  kPeerFlag = 10,
  kRecvValid = 11,
  kRecvBox = 12,  // 8 fields
  kLocalBuf = 20,
  kLocalFlag = 21,
  kLocalExpected = 22,
  kCounters = 23,
  kMode = 24,
  kFaceFields = 32,
};

struct Box {
  int n0, z0, y0, x0, en, ez, ey, ex;
};

struct Face {
  int send, recv, mode;
  Box sb, rb;
  float4* peer_buf;
  unsigned long long* peer_flag;
  const float4* local_buf;
  const unsigned long long* local_flag;
  unsigned long long* expected;
};

struct RoundParams {
  Face f[2];
  unsigned int* counters;  // [0], [1]: blocks done packing face 0 / 1; [2]: blocks done with the round
  Frame fr;
  long long timeout_ns;
  int* error;
};

// float4 index i of a dense (n, z, y, x, c) box -> float offset in the frame
// (32-bit index math: a face never exceeds the mailbox, far below 2^31 float4s)
__device__ __forceinline__ long long box_off(const Frame& f, const Box& b, unsigned int i, unsigned int c4) {
  unsigned int t = i;
  const int c = static_cast<int>(t % c4) * 4;
  t /= c4;
  const int x = static_cast<int>(t % static_cast<unsigned int>(b.ex));
  t /= static_cast<unsigned int>(b.ex);
  const int y = static_cast<int>(t % static_cast<unsigned int>(b.ey));
  t /= static_cast<unsigned int>(b.ey);
  const int z = static_cast<int>(t % static_cast<unsigned int>(b.ez));
  const int n = b.n0 + static_cast<int>(t / static_cast<unsigned int>(b.ez));
  const long long Wf = f.w + 2 * f.mw, Hf = f.h + 2 * f.mh, Df = f.d + 2 * f.md;
  return ((((long long)n * Df + b.z0 + z) * Hf + b.y0 + y) * Wf + b.x0 + x) * f.c + c;
}

__device__ __forceinline__ long long box_vec4(const Frame& f, const Box& b) {
  return (long long)b.en * b.ez * b.ey * b.ex * (f.c / 4);
}

__device__ __forceinline__ long long now_ns() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(256) halo_round_peer_kernel(float* __restrict__ frame, const RoundParams p) {
  __shared__ unsigned long long want[2];
  __shared__ int last;
  const Frame& f = p.fr;
  const unsigned int c4 = f.c / 4;
  if (threadIdx.x < 2) {
    const Face& F = p.f[threadIdx.x];
    want[threadIdx.x] = F.recv ? *F.expected + 1ULL : 0ULL;  // read before any block can update it
  }
  __syncthreads();
  // ---- pack both faces into the neighbours' mailboxes (peer stores)
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const Face& F = p.f[s];
    if (!F.send) continue;
    const unsigned int n = static_cast<unsigned int>(box_vec4(f, F.sb));
    for (unsigned int i = blockIdx.x * 256u + threadIdx.x; i < n; i += gridDim.x * 256u)
      F.peer_buf[i] = *reinterpret_cast<const float4*>(frame + box_off(f, F.sb, i, c4));
  }
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const Face& F = p.f[s];
    if (!F.send) continue;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      // the last block to finish this face releases it to the neighbour
      if (atomicInc(&p.counters[s], gridDim.x - 1) == gridDim.x - 1) {
        __threadfence_system();
        atomicAdd_system(F.peer_flag, 1ULL);
      }
    }
  }
  // ---- wait for the neighbours' faces, unpack / accumulate into the margins
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const Face& F = p.f[s];
    if (!F.recv) continue;
    if (threadIdx.x == 0) {
      const long long t0 = now_ns();
      for (;;) {
        unsigned long long v;
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(F.local_flag) : "memory");
        if (v >= want[s]) break;
        if (now_ns() - t0 > p.timeout_ns) {  // the neighbour never arrived: fail loudly
          *p.error = 1;
          __threadfence_system();
          asm volatile("trap;");
        }
        __nanosleep(64);
      }
      __threadfence();
    }
    __syncthreads();
    const unsigned int n = static_cast<unsigned int>(box_vec4(f, F.rb));
    for (unsigned int i = blockIdx.x * 256u + threadIdx.x; i < n; i += gridDim.x * 256u) {
      const float4 v = __ldcg(F.local_buf + i);  // written by the peer: bypass L1
      float4* dst = reinterpret_cast<float4*>(frame + box_off(f, F.rb, i, c4));
      if (F.mode == 2) {
        float4 o = *dst;
        o.x += v.x;
        o.y += v.y;
        o.z += v.z;
        o.w += v.w;
        *dst = o;
      } else {
        *dst = v;
      }
    }
  }
  // ---- the last block to finish advances the expected arrival counts
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicInc(&p.counters[2], gridDim.x - 1) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x < 2 && p.f[threadIdx.x].recv) {
    *p.f[threadIdx.x].expected = want[threadIdx.x];
    __threadfence_system();
  }
}

Box read_box(const long long* d) {
  return Box{static_cast<int>(d[0]), static_cast<int>(d[1]), static_cast<int>(d[2]), static_cast<int>(d[3]),
             static_cast<int>(d[4]), static_cast<int>(d[5]), static_cast<int>(d[6]), static_cast<int>(d[7])};
}

bool box_ok(const Frame& f, const Box& b) {
  return b.n0 >= 0 && b.en >= 0 && b.n0 + b.en <= f.n && b.z0 >= 0 && b.z0 + b.ez <= f.d + 2 * f.md && b.y0 >= 0 &&
         b.y0 + b.ey <= f.h + 2 * f.mh && b.x0 >= 0 && b.x0 + b.ex <= f.w + 2 * f.mw;
}

}  // namespace

extern "C" int vpx_halo_round_peer(float* frame, const int* ff, const long long* faces, long long mailbox_bytes,
                                   long long timeout_ns, int* error, void* stream) {
  RoundParams p{};
  p.fr = Frame{ff[0], ff[1], ff[2], ff[3], ff[4], ff[5], ff[6], ff[7], 0};
  if (p.fr.c % 4) VPX_FAIL(VPX_ERR_UNSUPPORTED, "peer halo round: channels must be a multiple of 4");
  long long most = 0;
  bool any = false;
  for (int s = 0; s < 2; ++s) {
    const long long* d = faces + s * kFaceFields;
    Face& F = p.f[s];
    F.send = d[kSendValid] != 0;
    F.recv = d[kRecvValid] != 0;
    F.mode = static_cast<int>(d[kMode]);
    F.sb = read_box(d + kSendBox);
    F.rb = read_box(d + kRecvBox);
    F.peer_buf = reinterpret_cast<float4*>(d[kPeerBuf]);
    F.peer_flag = reinterpret_cast<unsigned long long*>(d[kPeerFlag]);
    F.local_buf = reinterpret_cast<const float4*>(d[kLocalBuf]);
    F.local_flag = reinterpret_cast<const unsigned long long*>(d[kLocalFlag]);
    F.expected = reinterpret_cast<unsigned long long*>(d[kLocalExpected]);
    if (s == 0) p.counters = reinterpret_cast<unsigned int*>(d[kCounters]);
    any = any || F.send || F.recv;
    if (F.recv && F.mode != 1 && F.mode != 2) VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "peer halo round: mode must be 1 or 2");
    for (int k = 0; k < 2; ++k) {
      const bool on = k ? F.recv : F.send;
      const Box& b = k ? F.rb : F.sb;
      if (!on) continue;
      if (!box_ok(p.fr, b)) VPX_FAIL(VPX_ERR_OUT_OF_BOUNDS, "peer halo round: box outside frame");
      const long long bytes = (long long)b.en * b.ez * b.ey * b.ex * p.fr.c * 4;
      if (bytes > mailbox_bytes || bytes / 16 >= (1ll << 31)) VPX_FAIL(VPX_ERR_OUT_OF_BOUNDS, "peer halo round: face larger than the mailbox");
      most = bytes > most ? bytes : most;
    }
  }
  if (!any) return VPX_OK;
  if (!p.counters) VPX_FAIL(VPX_ERR_SHAPE_MISMATCH, "peer halo round: no counters (face 0, field %d)", kCounters);
  p.timeout_ns = timeout_ns;
  p.error = error;
  long long blocks = (most / 16 + 255) / 256;
  blocks = blocks < 1 ? 1 : blocks;
  const int sms = vpx::num_sms();
  if (blocks > sms) blocks = sms;
  halo_round_peer_kernel<<<static_cast<int>(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(frame, p);
  VPX_LAUNCH_CHECK();
  return VPX_OK;
}
