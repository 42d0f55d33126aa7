"""Loss per step through the bench's three phases (eager, graph replay, host
input pipeline with the datastore int16 block) -- a divergence/NaN probe.

    python tools/loss_trace.py [--width 512] [--steps 6]
"""
import argparse
import math
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2007_12856_b200 import engine  # noqa: E402
from paper_2007_12856_b200.comm import RankCtx  # noqa: E402
from paper_2007_12856_b200.geometry import ProcessGrid  # noqa: E402
from paper_2007_12856_b200.networks import build_cosmoflow  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--width", type=int, default=512)
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--lr", type=float, default=1e-4)
    ap.add_argument("--eager-after-capture", type=int, default=0)
    ap.add_argument("--freed", action="store_true",
                    help="after capture, list freed default-pool blocks with the stack that allocated them")
    ap.add_argument("--poison", action="store_true",
                    help="fill all free (cached + device) memory with NaN after the eager steps: exposes "
                         "graph pointers into freed memory")
    a = ap.parse_args()
    import bench

    if a.freed:
        torch.cuda.memory._record_memory_history(max_entries=200000)
    ctx = RankCtx.from_env()
    grid = ProcessGrid(1, 1, 1, 1)
    net = build_cosmoflow(a.width)
    plan = engine.make_plan(net, grid, 1, a.width)
    state = engine.make_state(net, 0)
    x, y, ids = engine.synthetic_batch_full(net, a.width, 1, 0)
    batch = engine.scatter_batch(plan, x, y, ids, 0)
    del x

    def report(tag, loss):
        p = state.params.flat if hasattr(state.params, "flat") else None
        g = state.params.grad
        gn = float(g.norm())
        pn = float(p.norm()) if p is not None else float("nan")
        print(f"{tag}: loss {float(loss.item()):.6g} |grad| {gn:.4g} |param| {pn:.4g}", flush=True)

    for i in range(a.steps):
        report(f"eager {i}", engine.train_step(ctx, plan, state, batch, a.lr, as_tensor=True))
    cap = engine.CapturedStep(ctx, plan, state, batch, a.lr)
    for i in range(a.eager_after_capture):
        report(f"eager-after-capture {i}", engine.train_step(ctx, plan, state, batch, a.lr, as_tensor=True))
    if a.freed:
        snap = torch.cuda.memory._snapshot()
        last = {}
        for tr in snap.get("device_traces", [[]])[0]:
            if tr["action"] in ("alloc", "free_completed", "free_requested"):
                last.setdefault(tr["addr"], []).append(tr)
        for seg in snap["segments"]:
            if tuple(seg.get("segment_pool_id", (0, 0))) != (0, 0):
                continue
            for blk in seg["blocks"]:
                if blk["state"] != "inactive":
                    continue
                evs = last.get(blk["address"], [])
                allocs = [e for e in evs if e["action"] == "alloc"]
                fr = []
                if allocs:
                    fr = [f"{f['filename'].split('/')[-1]}:{f['line']}:{f['name']}" for f in allocs[-1]["frames"]
                          if "paper_2007" in f["filename"] or "loss_trace" in f["filename"] or "bench" in f["filename"]]
                print(f"freed block {blk['size'] / 2**20:.1f} MiB stream {seg.get('stream')} "
                      f"(allocs {len(allocs)}): {' < '.join(fr[:8])}")
    if a.poison:
        free, _ = torch.cuda.mem_get_info()
        reserved_free = torch.cuda.memory_reserved() - torch.cuda.memory_allocated()
        junk = []
        for nb in (reserved_free, free - (2 << 30)):
            if nb > (64 << 20):
                try:
                    junk.append(torch.full((nb // 4 - (16 << 20),), float("nan"), device="cuda"))
                except RuntimeError as exc:
                    print("poison alloc failed", exc)
        print("poisoned GB", sum(j.numel() * 4 for j in junk) / 1e9, flush=True)
        del junk
    for i in range(a.steps):
        report(f"graph {i}", cap(a.lr))
    x_host = batch.x_block.to_ncdhw().cpu().pin_memory()
    print("fp32 input absmax", float(x_host.abs().max()))

    class Args:
        pass
    ds = bench.datastore_block(Args(), net, grid, plan, ctx, a.width)
    print("int16 block", tuple(ds.shape), ds.dtype, int(ds.abs().max()))
    pipe = engine.HostInputPipeline(ds)
    pipe.start()
    for i in range(a.steps):
        pipe.load(batch, prefetch_next=i + 1 < a.steps)
        xb = batch.x_block
        report(f"ds {i} (x absmax {float(xb.data.abs().max()) if hasattr(xb, 'data') else math.nan:.3g})", cap(a.lr))


if __name__ == "__main__":
    main()
