/* vpx_probe.h -- measurement scaffolding (NOT part of the product ABI).
 * tcgen05 / TMA probes used by tools/probe_*.py to measure MMA issue rates
 * and operand layouts; built into tools/libvpx_probe.so by tools/probe_lib.py,
 * linked against libvpx.so.  Nothing in paper_2007_12856_b200/ loads it. */
#pragma once
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
/* ---------------------------------------------------------------- probes --
 * Test-only entry points used to pin UMMA/TMA semantics on the device. */
int vpx_probe_umma(const void* img, int img_bytes, const uint64_t* ops, int n_ops, float* out,
                   int ncols, void* stream);
/* Same as vpx_probe_umma, with ta[128][ta_cols] stored to TMEM columns 256.. first;
 * op flag 2 selects A from TMEM (adesc word = TMEM column). */
int vpx_probe_umma_ta(const void* img, int img_bytes, const uint64_t* ops, int n_ops, const float* ta,
                      int ta_cols, float* out, int ncols, void* stream);
int vpx_probe_tma(const void* gsrc, const uint64_t* dims5, const uint64_t* strides4,
                  const uint32_t* box5, const uint32_t* estr5, int swizzle, const int32_t* coords5,
                  void* out, int out_bytes, int* ok, void* stream);
int vpx_probe_mma_rate(int N, int n_iter, int a_layout, int n_acc, int bf16, long long* cycles,
                       void* stream);
int vpx_probe_mma_rate2(int N, int n_acc, int bf16, int n_iter, long long* cycles, void* stream);
#ifdef __cplusplus
}
#endif
