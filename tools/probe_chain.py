"""tcgen05 MMA rate when successive MMAs accumulate into the SAME TMEM
accumulator (n_acc = 1: a dependent chain, as a conv row's K steps) versus
n_acc independent accumulators issued round-robin.  M=128, K=8, tf32, A in
shared memory (mode 0 aligned no-swizzle, mode 10 the c1 forward's shifted
16-byte-pitch window).  python tools/probe_chain.py"""
import json
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import probe_lib  # noqa: E402

cyc = torch.zeros(1, dtype=torch.int64, device="cuda")
out = {}
for mode in (0, 10):
    for N, nacc in ((16, 1), (16, 4), (16, 8), (32, 1), (32, 4), (32, 8), (48, 1), (48, 2), (48, 4), (48, 8),
                    (64, 1), (64, 4), (96, 1), (96, 2), (128, 1), (128, 2), (256, 1)):
        it = 4096
        probe_lib.call("vpx_probe_mma_rate2", N, nacc, mode, it, cyc.data_ptr(), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        out[f"mode{mode}_N{N}_acc{nacc}"] = int(cyc.item()) / it
        print(f"mode {mode} N={N} nacc={nacc}: {int(cyc.item()) / it:.1f} cyc/mma", flush=True)
print(json.dumps(out))
