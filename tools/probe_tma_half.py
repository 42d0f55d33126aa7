"""Probe: TMA box whose inner dimension is 32 bytes (8 fp32 channels of a
16-channel row) under SWIZZLE_128B_ATOM_32B -- is the box packed densely
(4 voxels per 128-byte smem row) with the swizzle applied by address?"""
import ctypes

import numpy as np
import torch

from paper_2007_12856_b200 import _lib
import probe_lib  # noqa: E402

W, C = 64, 16
X = np.zeros((W, C), np.float32)
for v in range(W):
    for c in range(C):
        X[v, c] = v * 100 + c
g = torch.from_numpy(X).cuda()
ONES = (ctypes.c_uint32 * 5)(1, 1, 1, 1, 1)
for sw in (1282, 128, 32):
    for half in (0, 1):
        dims = (ctypes.c_uint64 * 5)(8, 2, W, 1, 1)
        strides = (ctypes.c_uint64 * 4)(32, C * 4, W * C * 4, W * C * 4)
        box = (ctypes.c_uint32 * 5)(8, 1, 32, 1, 1)
        coords = (ctypes.c_int32 * 5)(0, half, -1, 0, 0)
        nbytes = 32 * 32  # box bytes: 8 floats x 32 voxels
        out = torch.full((nbytes // 4,), -1.0, dtype=torch.float32, device="cuda")
        ok = torch.zeros(1, dtype=torch.int32, device="cuda")
        try:
            probe_lib.call("vpx_probe_tma", g.data_ptr(), ctypes.addressof(dims), ctypes.addressof(strides),
                      ctypes.addressof(box), ctypes.addressof(ONES), sw, ctypes.addressof(coords), out.data_ptr(),
                      nbytes, ok.data_ptr(), torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
        except Exception as e:  # encode may reject the box
            print(f"sw={sw} half={half}: {e}")
            continue
        o = out.cpu().numpy().reshape(-1, 4)  # 16-byte chunks
        print(f"sw={sw} half={half} ok={ok.item()}")
        for row in range(len(o) // 8):
            print("  row", row, [f"{int(o[row * 8 + k][0])}" for k in range(8)])
