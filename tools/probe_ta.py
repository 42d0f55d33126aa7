"""Probe tcgen05.mma with the A operand in TMEM (kind::tf32) on a B200.

1. correctness: A[128][K] stored to TMEM columns 256.., B K-major SWIZZLE_128B
   rows in smem, D = A @ B^T for N = 64 / 256, K = 8 and 32 (4 MMAs,
   A columns advancing by 8).
2. issue rate: back-to-back MMAs, A in TMEM vs A in smem, N = 16..256.
Run on the GPU box: python tools/probe_ta.py
"""

import ctypes
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
from paper_2007_12856_b200 import _lib
import probe_lib  # noqa: E402
from probe_umma import Img, check, idesc, sdesc, swz, tf32, RESULTS  # noqa: E402

rng = np.random.default_rng(1)


def run_ta(img_bytes, ops, ta, ncols):
    img = torch.from_numpy(np.ascontiguousarray(img_bytes).view(np.uint8)).cuda()
    ops_arr = np.array(ops, dtype=np.uint64).reshape(-1)
    ops_t = torch.from_numpy(ops_arr.view(np.int64)).cuda()
    ta_t = torch.from_numpy(np.ascontiguousarray(ta, dtype=np.float32)).cuda()
    out = torch.zeros(128 * ncols, dtype=torch.float32, device="cuda")
    probe_lib.call("vpx_probe_umma_ta", img.data_ptr(), img.numel(), ops_t.data_ptr(), len(ops), ta_t.data_ptr(),
              ta.shape[1], out.data_ptr(), ncols, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return out.cpu().numpy().reshape(128, ncols)


def t_correct():
    for N in (64, 256):
        for K in (8, 32):
            A = tf32(rng.standard_normal((128, 32)))
            A[:, K:] = 0
            Bm = tf32(rng.standard_normal((N, 32)))
            img = Img(65536)
            for r in range(N):
                for k in range(32):
                    img.put_f32(swz(r * 128 + k * 4, 128), Bm[r, k])
            ops = []
            for kk in range(K // 8):
                b = sdesc(32 * kk, 16, 1024, 2)
                ops.append((256 + 8 * kk, b, idesc(128, N) | (0 << 32), (1 if kk else 0) | 2))
            D = run_ta(img.b, ops, A, N)
            check(f"ta_N{N}_K{K}", D[:, :N], A[:, :K] @ Bm[:, :K].T)
    # A sub-columns: start the A operand at column 256 + 4 (not a multiple of 8)
    A = tf32(rng.standard_normal((128, 16)))
    Bm = tf32(rng.standard_normal((64, 32)))
    img = Img(65536)
    for r in range(64):
        for k in range(32):
            img.put_f32(swz(r * 128 + k * 4, 128), Bm[r, k])
    ops = [(260, sdesc(0, 16, 1024, 2), idesc(128, 64), 2)]
    D = run_ta(img.b, ops, A, 64)
    check("ta_col_offset4", D[:, :64], A[:, 4:12] @ Bm[:, :8].T)


def swz32b(addr):
    return addr ^ (((addr >> 7) & 3) << 5)


def t_mn_rows():
    """A (u) in TMEM, B = x rows of 128 B (8 voxels x 4 ch) MN-major SW128_BASE32B,
    N = 48: block 0 = chunk k, block 1 = chunk k+1 (LBO = one 128-byte row)."""
    nch = 40
    X = tf32(rng.standard_normal((nch, 32)))
    img = Img(65536)
    flat = X.reshape(-1)
    for i in range(flat.size):
        img.put_f32(swz32b(i * 4), flat[i])
    for N in (48, 64):
        for s in (0, 1, 3):
            A = tf32(rng.standard_normal((128, 16)))
            Bm = np.zeros((N, 8), np.float32)
            for n in range(N):
                for k in range(8):
                    Bm[n, k] = X[8 * s + k + n // 32, n % 32]
            ops = [(256, sdesc(8 * s * 128, 128, 512, 1), idesc(128, N, False, True), 2)]
            D = run_ta(img.b, ops, A, N)
            check(f"ta_mnrows_N{N}_s{s}", D[:, :N], A[:, :8] @ Bm.T)


def t_rate():
    cyc = torch.zeros(1, dtype=torch.int64, device="cuda")
    res = {}
    for N, n_acc in ((16, 8), (32, 8), (48, 8), (48, 9), (64, 4), (96, 2), (128, 2), (256, 1)):
        for mode in ((0, 2, 3, 5, 6, 7, 8, 9) if (N, n_acc) == (48, 9) else (0, 2, 3)):
            probe_lib.call("vpx_probe_mma_rate2", N, n_acc, mode, 4096, cyc.data_ptr(),
                      torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            c = int(cyc.item()) / 4096
            tag = {0: "smemA", 2: "tmemA", 3: "tmemA_mnB", 5: "tmemA_mnB_commit", 6: "tmemA_mnB_fence",
                   7: "tmemA_mnB_acc0-431", 8: "tmemA_mnB_9rows", 9: "tmemA_mnB_9rows_random"}[mode]
            res[f"N{N}_acc{n_acc}_{tag}"] = c
            print(f"N={N:3d} acc={n_acc} {tag}: {c:.1f} cycles/MMA")
    RESULTS["rate"] = res


if __name__ == "__main__":
    t_correct()
    t_mn_rows()
    t_rate()
    out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/probe_ta.json"
    json.dump(RESULTS, open(out, "w"), indent=1)
