"""Concurrent host->device copy bandwidth with one process per GPU (run under
torchrun): each rank copies a 134 MB pinned int8 block (its 1x4x1x1 share of
the 512^3 x 4 e2e input) repeatedly; pinned memory allocated with the
process unbound vs bound to the GPU's NUMA-local CPUs (nvmlDeviceSetCpuAffinity,
first touch).  Prints per-rank GB/s and the NUMA node of each GPU."""
import os
import time

import pynvml
import torch
import torch.distributed as dist

rank = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(rank)
dist.init_process_group("gloo")
n = 134217728 * int(os.environ.get("H2D_SCALE", "1"))
mode = os.environ.get("H2D_MODE", "default")
orig = os.sched_getaffinity(0)
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(rank)
busid = pynvml.nvmlDeviceGetPciInfo(h).busId
busid = busid.decode() if isinstance(busid, bytes) else busid
try:
    node = open(f"/sys/bus/pci/devices/{busid.lower()[4:] if busid.count(':') == 2 and len(busid) > 12 else busid.lower()}/numa_node").read().strip()
except OSError:
    node = "?"
if mode == "bound":
    pynvml.nvmlDeviceSetCpuAffinity(h)
src = torch.empty(n, dtype=torch.int8).pin_memory()
src.fill_(1)  # first touch
os.sched_setaffinity(0, orig)
dst = torch.empty(n, dtype=torch.int8, device="cuda")
for _ in range(3):
    dst.copy_(src, non_blocking=True)
torch.cuda.synchronize()
dist.barrier()
t0 = time.perf_counter()
for _ in range(20):
    dst.copy_(src, non_blocking=True)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
dist.barrier()
print(f"rank {rank} bus {busid} numa {node} mode {mode}: {20 * n / dt / 1e9:.1f} GB/s", flush=True)
