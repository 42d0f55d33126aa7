"""Multi-GPU parity worker (TEST INFRASTRUCTURE; run under torchrun, one
process per GPU, by tests/test_multigpu.py):

    torchrun --nproc-per-node N tests/dist_worker.py halo KEY
    torchrun --nproc-per-node N tests/dist_worker.py step GRID NET WIDTH N PREC
    torchrun --nproc-per-node N tests/dist_worker.py replay GRID WIDTH N
    torchrun --nproc-per-node N tests/dist_worker.py pipelined GRID WIDTH N

halo    device halo rounds on the golden frames the REFERENCE fabric produced
        (tests/golden/halo.npz): every exchange path (fused peer round, split
        peer send/recv, NCCL send/recv) forward and adjoint, bit-exact
        (reference fabric.py:380-443, tests/test_fabric.py:119-226).
step    one hybrid-parallel training step on GRID over NCCL; the traces of all
        ranks are gathered on rank 0 and compared, tensor by tensor in the
        reference metric, with the serial oracle of the same numerics (fp32:
        1e-5; tf32: the TF32-emulating oracle, device branch decisions within
        one TF32 ulp followed, end-to-end tolerance as in
        tests/test_gpu_engine.py), plus every parameter gradient, the loss and
        replication of the updated parameters (reference
        tests/test_model.py:227-283).
replay  CapturedStep graph replays over the peer-memory halo path (replays
        queued without host synchronisation) against eager steps over the
        NCCL halo path: parameters, moments and loss bit-identical.
pipelined  engine.PipelinedSteps (two step graphs, two input frames, the
        next block's H2D + layout on a copy stream) over the peer halo against
        eager steps on the same per-step host blocks: losses and parameters
        bit-identical.

Rank 0 prints one line "[dist_worker] {json}"; exit status 0 = pass.
"""

import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2007_12856_b200 as pkg  # noqa: E402
from paper_2007_12856_b200 import engine  # noqa: E402
from paper_2007_12856_b200.comm import PeerHalo, RankCtx, halo_exchange, reverse_halo_exchange  # noqa: E402
from paper_2007_12856_b200 import comm as C  # noqa: E402
from paper_2007_12856_b200.frames import DistTensor  # noqa: E402
from paper_2007_12856_b200.geometry import ProcessGrid, Shape5D, make_partition  # noqa: E402
from paper_2007_12856_b200.networks import build_cosmoflow, build_unet_mini  # noqa: E402


def _report(ctx, ok, **info):
    flag = torch.tensor([0 if ok else 1], device="cuda")
    dist.all_reduce(flag)
    if ctx.rank == 0:
        info["pass"] = bool(flag.item() == 0)
        print("[dist_worker] " + json.dumps(info), flush=True)
    dist.barrier()
    return int(flag.item() > 0)


# ---------------------------------------------------------------- halo
class _Plan:
    def __init__(self, meta):
        self.in_meta = [meta]


def _ref_to_device(ref_frame, meta):
    """Reference NCDHW frame (margins in every dim) -> NDHWC device frame."""
    fm = meta.margins()
    sl = [slice(None), slice(None)]
    for r, m, e in zip(meta.radii, fm, ref_frame.shape[2:]):
        sl.append(slice(r - m, e - (r - m)))
    return np.ascontiguousarray(ref_frame[tuple(sl)].transpose(0, 2, 3, 4, 1))


def run_halo(ctx, key):
    A = np.load(os.path.join(ROOT, "tests", "golden", "halo.npz"))
    shape, radii = tuple(int(v) for v in A[f"{key}_shape"]), tuple(int(v) for v in A[f"{key}_radii"])
    grid = ProcessGrid(*map(int, key.split("x")))
    meta = make_partition(Shape5D(*shape), grid, radii)
    r = ctx.rank
    loc, fm = meta.local_shape(r), meta.margins()
    inner = (slice(None), slice(fm[0], fm[0] + loc.d), slice(fm[1], fm[1] + loc.h), slice(fm[2], fm[2] + loc.w))
    want_fwd = _ref_to_device(A[f"{key}_r{r}_fwd"], meta).astype(np.float32)
    rev_in = A[f"{key}_r{r}_rev"]
    g0 = _ref_to_device(np.arange(rev_in.size, dtype=np.float64).reshape(rev_in.shape) * 0.25 - 3.0,
                        meta).astype(np.float32)
    want_rev = _ref_to_device(rev_in, meta).astype(np.float32)[inner]
    results = {}
    peer = PeerHalo(ctx, _Plan(meta))
    paths = [("nccl", None, None), ("peer_split", peer, False)]
    if loc.c % 4 == 0:
        paths.append(("peer_fused_round", peer, True))
    ok = True
    for name, pr, fused in paths:
        ctx.peer = pr
        if fused is not None:
            C._FUSED_ROUND = fused
        for rep in range(3):  # repeated rounds: mailbox parities alternate
            start = np.zeros_like(want_fwd)
            start[inner] = want_fwd[inner]
            t = DistTensor(meta, r, zero=True)
            t.t.copy_(torch.from_numpy(start).cuda())
            halo_exchange(ctx, t)
            g = DistTensor(meta, r, zero=True)
            g.t.copy_(torch.from_numpy(g0).cuda())
            reverse_halo_exchange(ctx, meta, r, g)
            torch.cuda.synchronize()
            f_ok = np.array_equal(t.t.cpu().numpy(), want_fwd)
            r_ok = np.array_equal(g.t.cpu().numpy()[inner], want_rev)
            ok = ok and f_ok and r_ok
            results.setdefault(name, []).append([f_ok, r_ok])
    C._FUSED_ROUND = True
    ctx.peer = None
    peer.close()
    return _report(ctx, ok, mode="halo", grid=key, shape=list(shape), radii=list(radii), rank0_results=results)


# ---------------------------------------------------------------- step
def _gather_trace(ctx, plan, trace):
    """Assemble every traced tensor into its global array on rank 0."""
    mine = {}
    for k, v in trace.items():
        if v is None:
            continue
        if isinstance(v, DistTensor):
            m, gr = v.meta, v.grid_rank
            reg = m.region(gr)
            lo, _ = m.sample_range(m.group_of(gr))
            gs = m.global_shape
            mine[k] = ("5d", (gs.n, gs.c, gs.d, gs.h, gs.w), lo, tuple(reg.offset), v.numpy())
        else:  # flat (n_local, features) on a group lead
            g = plan.grid.coords(ctx.rank)[0]
            mine[k] = ("flat", None, g * (plan.n_global // plan.grid.groups), None, v.detach().cpu().numpy())
    parts = [None] * ctx.size if ctx.rank == 0 else None
    dist.gather_object(mine, parts, dst=0)
    if ctx.rank != 0:
        return None
    out = {}
    for part in parts:
        for k, (kind, gshape, lo, off, a) in part.items():
            if kind == "5d":
                dst = out.setdefault(k, np.zeros(gshape, dtype=np.float32))
                n, c, d, h, w = a.shape
                dst[lo:lo + n, :, off[0]:off[0] + d, off[1]:off[1] + h, off[2]:off[2] + w] = a
            else:
                if k not in out:
                    out[k] = np.zeros((plan.n_global,) + a.shape[1:], dtype=np.float32)
                out[k][lo:lo + a.shape[0]] = a
    return out


def _rel(got, ref):
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.max(np.abs(np.asarray(got, np.float64) - ref)) / max(np.max(np.abs(ref)), 1e-30))


def run_step(ctx, grid_s, net_s, width, n, prec):
    from oracle import serial as O

    grid = ProcessGrid.parse(grid_s)
    pkg.set_precision(prec)
    net = build_unet_mini(width) if net_s == "unet" else build_cosmoflow(width, with_bn=net_s == "cosmoflow_bn")
    plan = engine.make_plan(net, grid, n, width)
    ctx.prepare_groups([plan.leads])
    x, y, ids = engine.synthetic_batch_full(net, width, n, 0)
    state = engine.make_state(net, 0)
    batch = engine.scatter_batch(plan, x, y, ids, ctx.rank)
    lr = 1e-3
    ctx.ensure_peer_halo(plan)
    trace = {}
    state.params.grad.zero_()
    pred, stash = engine.forward(ctx, plan, state, batch, "train", 0, trace=trace)
    loss, dpred = engine.loss_and_grad(ctx, plan, pred, batch)
    engine.backward(ctx, plan, state, stash, dpred, trace=trace)
    engine.gradient_allreduce(ctx, state)
    grads = state.params.grad.clone()
    engine.optimizer_step(state, lr)
    torch.cuda.synchronize()
    lmax, lmin = loss.clone(), loss.clone()
    dist.all_reduce(lmax, op=dist.ReduceOp.MAX)
    dist.all_reduce(lmin, op=dist.ReduceOp.MIN)
    pmax = state.params.flat.clone()
    dist.all_reduce(pmax, op=dist.ReduceOp.MAX)
    replicated = bool(torch.equal(pmax, state.params.flat)) and float(lmax) == float(lmin)
    dev = _gather_trace(ctx, plan, trace)
    ok, info = True, {}
    if ctx.rank == 0:
        xo, yo, _ = O.synthetic_batch(net, width, n, 0, np.float32)
        # fp32: the reference's own semantics with fp64 accumulation and the device's branch within
        # 2^-17 of a LeakyReLU / max-pool branch point (fp32 accumulation noise; tie-breaks counted)
        num = O.TF32(device=dev) if prec == "tf32" else O.TF32(device=dev, tau=2.0 ** -17, tf32=False)
        po = O.init_params(net, 0, np.float32)
        tr, go = {}, {}
        loss_o = O.train_step(net, po, O.make_bn_states(net, po, np.float32), O.Adam(po), lr, xo, yo, ids,
                              (0, 0, 0), trace=tr, grads_out=go, num=num)
        p32 = O.init_params(net, 0, np.float32)
        loss_32 = O.train_step(
            net, p32, O.make_bn_states(net, p32, np.float32), O.Adam(p32), lr, xo, yo, ids, (0, 0, 0))
        if prec == "fp32":
            tol = 1e-5
        else:
            # end to end: compounded TF32 rounding noise (tests/test_gpu_engine.py), plus the spatial
            # partials' summation order (BN statistics, filter gradients) -- the per-layer bound is
            # the teacher-forced 1e-3 below
            tol = 3e-3
        worst_t, worst_g = (0.0, None), (0.0, None)
        missing = [k for k in tr if k not in dev]
        for k, ref in tr.items():
            if k in dev:
                e = _rel(dev[k], ref)
                worst_t = max(worst_t, (e, str(k)))
        for name, (pos, cnt) in state.params.offsets.items():
            e = _rel(grads[pos:pos + cnt].cpu().numpy(), go[name].reshape(-1))
            worst_g = max(worst_g, (e, name))
        le = abs(float(loss.item()) - loss_o) / abs(loss_o)
        le32 = abs(float(loss.item()) - loss_32) / abs(loss_32)
        flips = num.flips_outside_band() if num is not None else {}
        worst_l = (0.0, None)
        if prec == "tf32":  # per layer: each layer on the device's own (gathered) inputs, rtol 1e-3
            pl = O.init_params(net, 0, np.float32)
            lt, lg = O.layerwise(net, pl, O.make_bn_states(net, pl, np.float32), xo, yo, dev, ids, (0, 0, 0),
                                 num=O.TF32())
            for k, ref in lt.items():
                if k in dev:
                    worst_l = max(worst_l, (_rel(dev[k], ref), str(k)))
            for name, (pos, cnt) in state.params.offsets.items():
                worst_l = max(worst_l, (_rel(grads[pos:pos + cnt].cpu().numpy(), lg[name].reshape(-1)),
                                        "grad " + name))
        ok = (le <= (1e-5 if prec == "fp32" else 1e-3) and le32 <= 1e-3 and worst_t[0] < tol and worst_g[0] < tol
              and worst_l[0] < 1e-3 and replicated and not flips and not missing)
        info = dict(loss=float(loss.item()), oracle_loss=loss_o, loss_rel=le, loss_rel_vs_fp32_oracle=le32,
                    worst_trace=worst_t, worst_grad=worst_g, tol=tol, worst_layerwise=worst_l, tensors_compared=len(tr) - len(missing),
                    missing=[str(k) for k in missing], flips_outside_band=flips,
                    branch_followed_in_band=sum(v["flips_in_band"] for v in num.branches.values()))
    return _report(ctx, ok, mode="step", grid=grid_s, net=net_s, width=width, n=n, precision=prec,
                   halo_path=ctx.halo_path, replicated=replicated, **info)


# ---------------------------------------------------------------- replay
def run_replay(ctx, grid_s, width, n):
    grid = ProcessGrid.parse(grid_s)
    net = build_cosmoflow(width)
    plan = engine.make_plan(net, grid, n, width)
    ctx.prepare_groups([plan.leads])
    x, y, ids = engine.synthetic_batch_full(net, width, n, 0)
    lrs = [1e-3 * (1.0 - 0.07 * i) for i in range(6)]
    runs = {}
    for name, captured, nccl in (("eager_nccl", False, True), ("eager_peer", False, False),
                                 ("replay_peer", True, False), ("replay_nccl", True, True)):
        ctx._peer_plan = None
        if nccl:
            os.environ["VPX_NCCL_HALO"] = "1"
        else:
            os.environ.pop("VPX_NCCL_HALO", None)
        ctx.ensure_peer_halo(plan)
        path = ctx.halo_path
        state = engine.make_state(net, 0)
        batch = engine.scatter_batch(plan, x, y, ids, ctx.rank)
        if captured:
            cap = engine.CapturedStep(ctx, plan, state, batch, lrs[0], warmup=2)
            for i in range(2, 6):
                loss = cap(lrs[i], iteration=i)
        else:
            for i in range(6):
                batch.iteration = i if i >= 2 else 0
                loss = engine.train_step(ctx, plan, state, batch, lrs[i] if i >= 2 else lrs[0], as_tensor=True)
        torch.cuda.synchronize()
        runs[name] = (state.params.flat.clone(), state.opt.m.clone(), state.opt.v.clone(), float(loss.item()), path)
    os.environ.pop("VPX_NCCL_HALO", None)
    p0, m0, v0, l0, h0 = runs["eager_nccl"]
    eq = {}
    for name, (p1, m1, v1, l1, h1) in runs.items():
        eq[name] = dict(equal=bool(torch.equal(p0, p1) and torch.equal(m0, m1) and torch.equal(v0, v1) and l0 == l1),
                        loss=l1, halo=h1, max_param_diff=float((p0 - p1).abs().max()))
    ok = all(v["equal"] for v in eq.values()) and "PeerHalo" in runs["replay_peer"][4]
    return _report(ctx, ok, mode="replay", grid=grid_s, width=width, n=n, runs=eq)


def _poison_free_memory():
    free, _ = torch.cuda.mem_get_info()
    cached = torch.cuda.memory_reserved() - torch.cuda.memory_allocated()
    junk = []
    for nb in (cached, free - (4 << 30)):
        if nb > (64 << 20):
            try:
                junk.append(torch.full((nb // 4 - (16 << 20),), float("nan"), device="cuda"))
            except RuntimeError:
                pass
    torch.cuda.synchronize()
    del junk
    torch.cuda.empty_cache()


def run_stale(ctx, grid_s, width, n):
    """The traced step twice in one process, the second after NaN-filling all
    free device memory: every traced tensor and the gradient bucket must be
    bit-identical (a kernel reading memory it never wrote shows here)."""
    grid = ProcessGrid.parse(grid_s)
    net = build_cosmoflow(width)
    plan = engine.make_plan(net, grid, n, width)
    ctx.prepare_groups([plan.leads])
    x, y, ids = engine.synthetic_batch_full(net, width, n, 0)
    ctx.ensure_peer_halo(plan)
    runs = []
    for k in range(2):
        if k:
            _poison_free_memory()
        state = engine.make_state(net, 0)
        batch = engine.scatter_batch(plan, x, y, ids, ctx.rank)
        trace = {}
        state.params.grad.zero_()
        pred, stash = engine.forward(ctx, plan, state, batch, "train", 0, trace=trace)
        loss, dpred = engine.loss_and_grad(ctx, plan, pred, batch)
        engine.backward(ctx, plan, state, stash, dpred, trace=trace)
        engine.gradient_allreduce(ctx, state)
        torch.cuda.synchronize()
        tr = {}
        for key, v in trace.items():
            if v is None:
                continue
            tr[key] = v.numpy() if isinstance(v, DistTensor) else v.detach().cpu().numpy()
        xin = batch.x_block.t.detach().cpu().numpy()  # input frame incl. the margins the exchange filled
        runs.append((tr, state.params.grad.clone(), float(loss.item()), xin))
        del trace, stash, pred, dpred, batch, state
    (t0, g0, l0, x0), (t1, g1, l1, x1) = runs
    order = [k for k in t0]
    diff = [str(k) for k in order if not np.array_equal(t0[k], t1[k], equal_nan=False)]
    xeq = bool(np.array_equal(x0, x1))
    first_diff = None
    if diff:
        k0 = next(k for k in order if str(k) == diff[0])
        a, b = t0[k0], t1[k0]
        bad = np.argwhere(a != b)
        first_diff = dict(n=int(len(bad)), of=int(a.size), shape=list(a.shape), lo=bad.min(axis=0).tolist(),
                          hi=bad.max(axis=0).tolist(), maxabs=float(np.nanmax(np.abs(a - b))),
                          nan0=int(np.isnan(a).sum()), nan1=int(np.isnan(b).sum()),
                          sample=[[int(v) for v in bad[i]] + [float(a[tuple(bad[i])]), float(b[tuple(bad[i])])]
                                  for i in range(min(4, len(bad)))])
    where = None
    if not xeq:
        bad = np.argwhere(x0 != x1)
        where = [bad.min(axis=0).tolist(), bad.max(axis=0).tolist(), int(len(bad)), list(x0.shape)]
    ok = not diff and torch.equal(g0, g1) and l0 == l1 and xeq
    info = dict(rank=ctx.rank, first_differing=diff[:6], grads_equal=bool(torch.equal(g0, g1)), loss=[l0, l1],
                input_frame_equal=xeq, input_frame_diff=where, first_diff=first_diff)
    allinfo = [None] * ctx.size if ctx.rank == 0 else None
    dist.gather_object(info, allinfo, dst=0)
    return _report(ctx, ok, mode="stale", grid=grid_s, width=width, n=n, per_rank=allinfo)


def run_pipelined(ctx, grid_s, width, n):
    """engine.PipelinedSteps over the peer-halo path (two graphs, two input
    frames, next block's H2D + layout on a copy stream) against eager steps
    on the same per-step host blocks: losses and parameters bit-equal."""
    grid = ProcessGrid.parse(grid_s)
    net = build_cosmoflow(width)
    plan = engine.make_plan(net, grid, n, width)
    ctx.prepare_groups([plan.leads])
    x, y, ids = engine.synthetic_batch_full(net, width, n, 0)
    ctx.ensure_peer_halo(plan)
    K, warm = 5, 1
    runs = []
    for pipelined in (False, True):
        state = engine.make_state(net, 0)
        batch = engine.scatter_batch(plan, x, y, ids, ctx.rank)
        shape = (batch.x_block.n, batch.x_block.c) + batch.x_block.spatial if batch.x_block is not None else None
        g = torch.Generator().manual_seed(11 + ctx.rank)
        blocks = [torch.randint(-8, 9, shape, generator=g).to(torch.int8).pin_memory() for _ in range(K)] \
            if shape is not None else None
        losses = []
        if pipelined:
            pipe = engine.PipelinedSteps(ctx, plan, state, batch, (lambda i: blocks[i]) if blocks else None, 1e-3,
                                         warmup=warm)
            pipe.start()
            for i in range(K):
                prev = pipe.step(1e-3, prefetch_next=i + 1 < K)
                if prev is not None:
                    losses.append(prev)
            losses.append(pipe.finish())
        else:
            for _ in range(2 * warm):
                engine.train_step(ctx, plan, state, batch, 1e-3)
            for i in range(K):
                if blocks is not None:
                    batch.x_block.load_ncdhw(blocks[i].cuda())
                losses.append(engine.train_step(ctx, plan, state, batch, 1e-3))
        torch.cuda.synchronize()
        runs.append((losses, state.params.flat.clone()))
    (l0, p0), (l1, p1) = runs
    ok = l0 == l1 and bool(torch.equal(p0, p1)) and all(np.isfinite(l1))
    return _report(ctx, ok, mode="pipelined", grid=grid_s, width=width, n=n, losses=[l0, l1],
                   halo=ctx.halo_path, max_param_diff=float((p0 - p1).abs().max()))


def main():
    ctx = RankCtx.from_env()
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    mode = sys.argv[1]
    if mode == "halo":
        rc = run_halo(ctx, sys.argv[2])
    elif mode == "step":
        rc = run_step(ctx, sys.argv[2], sys.argv[3], int(sys.argv[4]), int(sys.argv[5]), sys.argv[6])
    elif mode == "stale":
        rc = run_stale(ctx, sys.argv[2], int(sys.argv[3]), int(sys.argv[4]))
    elif mode == "replay":
        rc = run_replay(ctx, sys.argv[2], int(sys.argv[3]), int(sys.argv[4]))
    elif mode == "pipelined":
        rc = run_pipelined(ctx, sys.argv[2], int(sys.argv[3]), int(sys.argv[4]))
    else:
        raise SystemExit(f"unknown mode {mode}")
    dist.destroy_process_group()
    sys.exit(rc)


if __name__ == "__main__":
    main()
