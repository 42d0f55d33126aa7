"""Host->device copy bandwidth of a 0.54 GB pinned block (the e2e input path):
one copy vs chunked copies on one / two streams.  python tools/h2d_probe.py"""
import torch

n = 512 ** 3 * 4
src = torch.empty(n, dtype=torch.int8).pin_memory()
dst = torch.empty(n, dtype=torch.int8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]


def run(chunks, nstreams):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    step = n // chunks
    cur = torch.cuda.current_stream()
    for s in streams[:nstreams]:
        s.wait_stream(cur)
    for i in range(chunks):
        with torch.cuda.stream(streams[i % nstreams]):
            dst[i * step:(i + 1) * step].copy_(src[i * step:(i + 1) * step], non_blocking=True)
    for s in streams[:nstreams]:
        cur.wait_stream(s)
    b.record()
    b.synchronize()
    return n / (a.elapsed_time(b) * 1e-3) / 1e9


for chunks, ns in ((1, 1), (4, 1), (4, 2), (8, 4), (16, 4)):
    best = max(run(chunks, ns) for _ in range(5))
    print(f"chunks={chunks} streams={ns}: {best:.1f} GB/s", flush=True)
