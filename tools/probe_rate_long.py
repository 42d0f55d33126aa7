import sys, torch
sys.path.insert(0, ".")
from paper_2007_12856_b200 import _lib
import probe_lib  # noqa: E402
cyc = torch.zeros(1, dtype=torch.int64, device="cuda")
for n in (4095*9//9*9, 65536*9//9, 1 << 20):
    n = (n // 9) * 9
    for mode in (9, 0):
        N, acc = 48, 9
        probe_lib.call("vpx_probe_mma_rate2", N, acc, mode, n, cyc.data_ptr(), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        print(f"n_iter={n} mode={mode}: {int(cyc.item())/n:.1f} cycles/MMA", flush=True)
