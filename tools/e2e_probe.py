"""Where the end-to-end step loses time against the device-only step
(CosmoFlow-512, one GPU): replay only / + layout kernel from a staged int8
block / + H2D copy pipeline / + loss.item() per step.  python tools/e2e_probe.py"""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2007_12856_b200 import engine  # noqa: E402
from paper_2007_12856_b200.comm import RankCtx  # noqa: E402
from paper_2007_12856_b200.geometry import ProcessGrid  # noqa: E402
from paper_2007_12856_b200.networks import build_cosmoflow  # noqa: E402

W, K = 512, 10
net = build_cosmoflow(W)
ctx = RankCtx(0, 1)
plan = engine.make_plan(net, ProcessGrid(1, 1, 1, 1), 1, W)
state = engine.make_state(net, 0)
x, y, ids = engine.synthetic_batch_full(net, W, 1, 0)
batch = engine.scatter_batch(plan, x, y, ids, 0)
host = torch.floor(x.clamp(-1, 1) * 8).to(torch.int8).cpu().pin_memory()
dev_block = host.cuda()
del x
cap = engine.CapturedStep(ctx, plan, state, batch, 1e-4)
for _ in range(3):
    cap(1e-4)
torch.cuda.synchronize()


def timed(name, body):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    body()
    b.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3 / K
    print(f"{name:48s} device {a.elapsed_time(b) / K:7.3f} ms/step  wall {wall:7.3f}", flush=True)


def replay():
    for _ in range(K):
        cap(1e-4)


def replay_sync():
    for _ in range(K):
        float(cap(1e-4).item())


def layout_only():
    for _ in range(K):
        batch.x_block.load_ncdhw(dev_block)


def layout_replay():
    for _ in range(K):
        batch.x_block.load_ncdhw(dev_block)
        cap(1e-4)


def pipeline(sync):
    def body():
        pipe = engine.HostInputPipeline(host)
        pipe.start()
        for i in range(K):
            pipe.load(batch, prefetch_next=i + 1 < K)
            loss = cap(1e-4)
            if sync:
                float(loss.item())
    return body


timed("graph replay", replay)
timed("graph replay + loss.item() each step", replay_sync)
timed("layout kernel only (int8 on device)", layout_only)
timed("layout (int8 on device) + replay", layout_replay)
timed("H2D pipeline + layout + replay", pipeline(False))
timed("H2D pipeline + layout + replay + loss.item()", pipeline(True))
