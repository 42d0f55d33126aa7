"""Multi-GPU parity check (run under torchrun, one process per GPU).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/check_dist.py GRID [WIDTH] [N] [PREC]

Every rank runs one hybrid-parallel training step of CosmoFlow-WIDTH on GRID
(GxPDxPHxPW) over NCCL; rank 0 runs the serial CPU oracle on the full batch
and compares the loss, the allreduced gradient bucket and the updated
parameters.  fp32 mode must match to 1e-5 (the reference's own fp32
tolerance); tf32 mode prints the errors.  Exit status 0 = pass.
"""

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, ".")
import paper_2007_12856_b200 as pkg  # noqa: E402
from paper_2007_12856_b200 import engine  # noqa: E402
from paper_2007_12856_b200.comm import RankCtx  # noqa: E402
from paper_2007_12856_b200.geometry import ProcessGrid  # noqa: E402
from paper_2007_12856_b200.networks import build_cosmoflow  # noqa: E402


def main():
    grid = ProcessGrid.parse(sys.argv[1])
    W = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    prec = sys.argv[4] if len(sys.argv) > 4 else "fp32"
    bn = len(sys.argv) > 5 and sys.argv[5] == "bn"
    ctx = RankCtx.from_env()
    pkg.set_precision(prec)
    net = build_cosmoflow(W, with_bn=bn)
    plan = engine.make_plan(net, grid, n, W)
    ctx.prepare_groups([plan.leads])
    x, y, ids = engine.synthetic_batch_full(net, W, n, 0)
    state = engine.make_state(net, 0)
    batch = engine.scatter_batch(plan, x, y, ids, ctx.rank)
    lr = 1e-3
    ctx.ensure_peer_halo(plan)  # CUDA-IPC mailboxes unless VPX_NCCL_HALO=1
    state.params.grad.zero_()
    pred, stash = engine.forward(ctx, plan, state, batch, "train", 0)
    loss, dpred = engine.loss_and_grad(ctx, plan, pred, batch)
    engine.backward(ctx, plan, state, stash, dpred)
    engine.gradient_allreduce(ctx, state)
    grads = state.params.grad.clone()
    engine.optimizer_step(state, lr)
    torch.cuda.synchronize()
    # every rank must hold the identical loss and replicated parameters
    lt = loss.clone()
    dist.all_reduce(lt, op=dist.ReduceOp.MAX)
    lmin = loss.clone()
    dist.all_reduce(lmin, op=dist.ReduceOp.MIN)
    pmax = state.params.flat.clone()
    dist.all_reduce(pmax, op=dist.ReduceOp.MAX)
    replicated = bool(torch.equal(pmax, state.params.flat)) and float(lt) == float(lmin)
    ok = True
    if ctx.rank == 0:
        from oracle import serial as O

        xo, yo, _ = O.synthetic_batch(net, W, n, 0, np.float32)
        po = O.init_params(net, 0, np.float32)
        go = {}
        loss_o = O.train_step(net, po, O.make_bn_states(net, po, np.float32), O.Adam(po), lr, xo, yo, ids,
                              (0, 0, 0), grads_out=go)
        tol = 1e-5 if prec == "fp32" else 2e-2
        worst = 0.0
        for name, (pos, cnt) in state.params.offsets.items():
            g = grads[pos:pos + cnt].cpu().numpy().astype(np.float64)
            r = go[name].reshape(-1).astype(np.float64)
            e = float(np.linalg.norm(g - r) / max(np.linalg.norm(r), 1e-300)) if prec != "fp32" else \
                float(np.max(np.abs(g - r)) / max(np.max(np.abs(r)), 1e-300))
            worst = max(worst, e)
            if e > tol:
                print(f"  grad {name}: err {e:.3e}")
                ok = False
        le = abs(float(loss.item()) - loss_o) / abs(loss_o)
        ok = ok and le < (1e-5 if prec == "fp32" else 1e-3) and replicated
        print(f"[check_dist] halo path: {ctx.halo_path}")
        print(f"[check_dist] grid {sys.argv[1]} W={W} n={n} {prec}{' bn' if bn else ''}: loss {float(loss.item())!r} "
              f"oracle {loss_o!r} (rel {le:.2e}); worst grad err {worst:.2e}; replicated={replicated}; "
              f"{'PASS' if ok else 'FAIL'}", flush=True)
    flag = torch.tensor([0 if ok else 1], device="cuda")
    dist.all_reduce(flag)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(int(flag.item() > 0))


if __name__ == "__main__":
    main()
