"""Find a captured kernel that reads memory outside the graph's pool.

Captures forward (graph 1) and loss+backward (graph 2) in one private pool,
fills every free default-pool / device block with NaN, replays, and reports
the first stashed activation / gradient that went non-finite.

    python tools/graph_bisect.py [--width 128]
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2007_12856_b200 import engine  # noqa: E402
from paper_2007_12856_b200.comm import RankCtx  # noqa: E402
from paper_2007_12856_b200.geometry import ProcessGrid  # noqa: E402
from paper_2007_12856_b200.networks import build_cosmoflow  # noqa: E402


def tensors_of(obj):
    if obj is None:
        return []
    if isinstance(obj, torch.Tensor):
        return [obj]
    if isinstance(obj, (list, tuple)):
        return [t for o in obj for t in tensors_of(o)]
    t = getattr(obj, "t", None)
    return [t] if isinstance(t, torch.Tensor) else []


def bad(obj):
    for t in tensors_of(obj):
        if t.is_floating_point() and not torch.isfinite(t).all():
            return True
    return False


def poison():
    free, _ = torch.cuda.mem_get_info()
    reserved_free = torch.cuda.memory_reserved() - torch.cuda.memory_allocated()
    junk = []
    for nb in (reserved_free, free - (2 << 30)):
        if nb > (64 << 20):
            try:
                junk.append(torch.full((nb // 4 - (16 << 20),), float("nan"), device="cuda"))
            except RuntimeError:
                pass
    torch.cuda.synchronize()
    print("poisoned GB", sum(j.numel() * 4 for j in junk) / 1e9, flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--width", type=int, default=128)
    a = ap.parse_args()
    ctx = RankCtx.from_env()
    net = build_cosmoflow(a.width)
    plan = engine.make_plan(net, ProcessGrid(1, 1, 1, 1), 1, a.width)
    state = engine.make_state(net, 0)
    x, y, ids = engine.synthetic_batch_full(net, a.width, 1, 0)
    batch = engine.scatter_batch(plan, x, y, ids, 0)
    sc = engine.StepScalars(net, batch.sample_ids)
    sc.set(state, 1e-4, (0, 0, 0))

    def fwd():
        return engine.forward(ctx, plan, state, batch, "train", 0, scalars=sc)

    def bwd(pred, stash):
        loss, dpred = engine.loss_and_grad(ctx, plan, pred, batch)
        state.params.grad.zero_()
        engine.backward(ctx, plan, state, stash, dpred)
        return loss

    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(2):
            p, s = fwd()
            bwd(p, s)
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    del p, s
    from paper_2007_12856_b200 import _lib
    calls = []
    orig = _lib.call

    def logged(name, *args):
        calls.append((name, [a for a in args if isinstance(a, int) and a > (1 << 32)]))
        return orig(name, *args)
    _lib.call = logged
    g1, g2 = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    with torch.cuda.graph(g1):
        pred, stash = fwd()
    with torch.cuda.graph(g2, pool=g1.pool()):
        loss = bwd(pred, stash)
    torch.cuda.synchronize()
    _lib.call = orig
    snap = torch.cuda.memory._snapshot()
    freed = []
    for seg in snap["segments"]:
        addr = seg["address"]
        for blk in seg["blocks"]:
            if blk["state"] == "inactive":
                freed.append((addr, addr + blk["size"], tuple(seg.get("segment_pool_id", (0, 0)))))
            addr += blk["size"]
    print(f"{len(calls)} captured calls, {len(freed)} free blocks", flush=True)
    for name, ptrs in calls:
        for p in ptrs:
            for lo, hi, pool in freed:
                if lo <= p < hi:
                    print(f"  {name}: pointer {p:#x} inside a FREE block [{lo:#x},{hi:#x}) pool {pool}", flush=True)
    g1.replay()
    g2.replay()
    torch.cuda.synchronize()
    print("clean replay: loss", float(loss.item()), "stash bad", [i for i, s in enumerate(stash) if bad(s)],
          "grad finite", bool(torch.isfinite(state.params.grad).all()), flush=True)
    poison()
    g1.replay()
    torch.cuda.synchronize()
    badf = [(i, net.layers[i].name) for i, s in enumerate(stash) if bad(s)]
    print("after poison, forward: non-finite stash entries", badf, "pred bad", bad(pred), flush=True)
    from paper_2007_12856_b200 import layers as L
    for nm, t in (("x_block", batch.x_block.t), ("WS", L.WS._t), ("params", state.params.flat)):
        print(f"  {nm}: finite {bool(torch.isfinite(t).all()) if t is not None else None}", flush=True)
    for i, s_ in enumerate(stash[:8]):
        for t in tensors_of(s_):
            if t.is_floating_point():
                nf = ~torch.isfinite(t)
                idx = nf.nonzero()
                print(f"  stash[{i}] {net.layers[i].name} shape {tuple(t.shape)} non-finite {int(nf.sum())}"
                      f" first {idx[:3].tolist()} last {idx[-3:].tolist()}", flush=True)
            else:
                print(f"  stash[{i}] {net.layers[i].name} {t.dtype} {tuple(t.shape)}", flush=True)
    g2.replay()
    torch.cuda.synchronize()
    G = state.params.grads
    print("after poison, backward: loss", float(loss.item()), "non-finite grads",
          [k for k, v in G.items() if not torch.isfinite(v).all()], flush=True)


if __name__ == "__main__":
    main()
