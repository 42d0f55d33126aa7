"""tcgen05 MMA throughput (M=128, K=8, tf32, warp-uniform issue, NACC
independent accumulators) with A in shared memory: aligned no-swizzle core
matrices (mode 0, LBO 2048) vs the c1 forward's shifted 16-byte-pitch window
(mode 10, LBO 16, core matrices overlapping).  python tools/probe_alayout.py"""
import json
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import probe_lib  # noqa: E402

cyc = torch.zeros(1, dtype=torch.int64, device="cuda")
out = {}
for mode in (0, 10):
    for N, nacc in ((16, 8), (32, 8), (48, 8), (64, 8), (128, 2)):
        it = 4096
        probe_lib.call("vpx_probe_mma_rate2", N, nacc, mode, it, cyc.data_ptr(), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        out[f"mode{mode}_N{N}"] = int(cyc.item()) / it
        print(f"mode {mode} N={N} nacc={nacc}: {int(cyc.item()) / it:.1f} cyc/mma", flush=True)
print(json.dumps(out))
