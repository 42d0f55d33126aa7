"""Hybrid data x spatial parallel training step on B200s.

Public API mirrors the reference engine (reference
pkg/src/voxpar/model/engine.py): ``make_plan`` / ``Plan``, ``Batch``,
``RankState``, ``forward``, ``loss_and_grad``, ``backward``,
``train_step`` and ``scatter_batch``.  One process drives one GPU; the
per-rank program is the reference's, with device DistTensors, libvpx
kernels and NCCL collectives underneath.

Layout decisions (make_plan, reference engine.py:62-176): every layer is
"spatial" until the redistribution point -- the first layer that cannot run
partitioned on the grid, or the flatten -- after which it is "collapsed"
(full spatial extent on one lead rank per data-parallel group) and, past
the flatten, "flat".  Each edge's partition carries the halo radii its
consumer needs.

Gradients: every parameter's gradient is written straight into a view of one
flat fp32 bucket (param_entries order, reference networks.py:133-153), which
is allreduced once over all ranks (reference engine.py:446-462) -- that sum
both completes spatial partial sums and averages data-parallel groups,
because the loss is normalised by the global batch.  Adam then runs as one
kernel over the flat parameter / moment buffers.
"""

from __future__ import annotations

import contextlib
import os
from dataclasses import dataclass, field

import torch
import torch.distributed as dist

from . import _lib, prng
from .accounting import out_shape
from .comm import RankCtx
from .errors import NonDivisible, ShapeMismatch
from .frames import DistTensor, stream_ptr
from .geometry import DistTensorMeta, ProcessGrid, Shape5D, make_partition
from . import layers as D
from .networks import NetworkSpec, param_entries
from .timing import region

NO_HALO = (0, 0, 0)


# --------------------------------------------------------------------- plan

@dataclass(frozen=True)
class Plan:
    net: NetworkSpec
    grid: ProcessGrid
    n_global: int
    w_i: int
    placement: tuple   # per layer: "spatial" | "collapsed" | "flat"
    in_meta: tuple     # per layer: DistTensorMeta of its 5D input (None past flatten)
    out_radii: tuple   # per layer: halo radii of its output
    redist_idx: int    # layer the redistribution precedes; -1 = never
    redist_src_meta: DistTensorMeta
    leads: tuple       # process rank of each group's lead
    label_meta: DistTensorMeta  # xent label layout; None for mse

    @property
    def input_meta(self) -> DistTensorMeta:
        return self.in_meta[0]


def _consumer_radii(layer):
    return layer.params.radii if layer.kind == "conv" else NO_HALO


def _why_not_spatial(layer, in_shape, parts):
    """None if `layer` can run partitioned on `parts`, else the reason
    (reference engine.py:62-81)."""
    ext = in_shape[2:]
    for name, e, p in zip("dhw", ext, parts):
        if e % p:
            return f"extent {name}={e} not divisible by {p} partitions"
    if layer.kind == "conv":
        for name, e, p, r, s in zip("dhw", ext, parts, layer.params.radii, layer.params.stride):
            loc = e // p
            if p > 1 and r > loc:
                return f"halo radius {r} exceeds local extent {loc} in {name}"
            if p > 1 and loc % s:
                return f"local extent {name}={loc} not divisible by stride {s}"
    elif layer.kind == "pool":
        for name, e, p in zip("dhw", ext, parts):
            if (e // p) % 2:
                return f"local extent {name}={e // p} is odd"
    return None


def make_plan(net: NetworkSpec, grid: ProcessGrid, n_global: int, w_i: int,
              redistribute_before: str = None) -> Plan:
    shapes = [(n_global, net.in_channels, w_i, w_i, w_i)]
    by_name = {}
    for layer in net.layers:
        skip = by_name.get(layer.skip) if layer.kind == "concat" else None
        nxt = out_shape(layer, shapes[-1], skip_shape=skip)
        by_name[layer.name] = nxt
        shapes.append(nxt)

    parts = grid.spatial_parts
    redist, reasons = -1, {}
    for i, layer in enumerate(net.layers):
        if layer.kind == "flatten":
            if redist < 0:
                redist = i
            break
        why = _why_not_spatial(layer, shapes[i], parts)
        if why is not None and redist < 0:
            redist, reasons[i] = i, why
    if redistribute_before is not None:
        forced = net.layer_index(redistribute_before)
        if redist >= 0 and forced > redist:
            bad = net.layers[redist]
            raise NonDivisible(f"layer {bad.name!r} cannot run spatially on grid {parts}: "
                               f"{reasons.get(redist, 'needs flat layout')}")
        redist = forced
    if redist == 0 and grid.spatial_size > 1:
        raise NonDivisible(f"layer {net.layers[0].name!r} cannot run spatially on grid {parts}: "
                           f"{reasons.get(0)}")
    if redist >= 0:
        for i, layer in enumerate(net.layers):
            if layer.kind == "concat" and net.layer_index(layer.skip) < redist <= i:
                raise NonDivisible(f"redistribution before {net.layers[redist].name!r} would split the "
                                   f"{layer.name!r} skip connection across layouts")

    leads = tuple(grid.rank_of(g, 0, 0, 0) for g in range(grid.groups))
    collapsed_grid = ProcessGrid(grid.groups, 1, 1, 1)

    def meta_for(shape, spatial, radii):
        s5 = Shape5D(*shape)
        if spatial:
            return make_partition(s5, grid, radii)
        return make_partition(s5, collapsed_grid, radii, rank_map=leads)

    placement, in_meta, out_radii = [], [], []
    flat = False
    for i, layer in enumerate(net.layers):
        if layer.kind == "flatten":
            placement.append("flat")
            in_meta.append(meta_for(shapes[i], False, NO_HALO))
            out_radii.append(NO_HALO)
            flat = True
            continue
        if flat:
            placement.append("flat")
            in_meta.append(None)
            out_radii.append(NO_HALO)
            continue
        spatial = redist < 0 or i < redist
        placement.append("spatial" if spatial else "collapsed")
        in_meta.append(meta_for(shapes[i], spatial, _consumer_radii(layer)))
        nxt = net.layers[i + 1] if i + 1 < len(net.layers) else None
        if nxt is None or nxt.kind == "flatten" or (redist >= 0 and i + 1 == redist):
            out_radii.append(NO_HALO)
        else:
            out_radii.append(_consumer_radii(nxt))
    redist_src = meta_for(shapes[redist], True, NO_HALO) if redist >= 0 else None
    label_meta = None
    if net.loss == "xent":
        o = shapes[-1]
        label_meta = meta_for((o[0], 1) + tuple(o[2:]), placement[-1] == "spatial", NO_HALO)
    return Plan(net, grid, n_global, w_i, tuple(placement), tuple(in_meta), tuple(out_radii),
                redist, redist_src, leads, label_meta)


def _meta_like(meta: DistTensorMeta, radii=NO_HALO):
    return make_partition(meta.global_shape, meta.grid, radii, meta.rank_map)


def _grid_rank(meta: DistTensorMeta, rank: int):
    return meta.rank_map.index(rank) if rank in meta.rank_map else None


# -------------------------------------------------------------------- state

@dataclass
class Batch:
    """One rank's share of a global batch (reference engine.py:179-194).

    x_block: DistTensor (or NCDHW array) of this rank's input block, None when
    it holds none.  target: (n_local, out_dim) CUDA tensor (mse).  y_block:
    int64 CUDA tensor (n_local, d, h, w) labels (xent).
    """

    x_block: object = None
    target: torch.Tensor = None
    y_block: torch.Tensor = None
    sample_ids: tuple = ()
    epoch: int = 0
    iteration: int = 0


class FlatParams:
    """All trainable tensors as views of one flat fp32 buffer (plus a twin
    gradient bucket and Adam moments), in param_entries order."""

    def __init__(self, net: NetworkSpec, device="cuda"):
        self.entries = param_entries(net)
        total = sum(_numel(s) for _, s, _ in self.entries)
        self.flat = torch.zeros(total, dtype=torch.float32, device=device)
        self.grad = torch.zeros(total, dtype=torch.float32, device=device)
        self.views, self.grads, self.offsets = {}, {}, {}
        pos = 0
        for name, shape, _ in self.entries:
            n = _numel(shape)
            self.views[name] = self.flat[pos:pos + n].view(shape)
            self.grads[name] = self.grad[pos:pos + n].view(shape)
            self.offsets[name] = (pos, n)
            pos += n
        self.numel = total

    # the reference's RankState.params is a dict name -> array (reference
    # engine.py:197-203); the same read/write access by name, on views
    def __getitem__(self, name):
        return self.views[name]

    def __setitem__(self, name, value):
        self.views[name].copy_(torch.as_tensor(value, dtype=torch.float32))

    def __iter__(self):
        return iter(self.views)

    def __len__(self):
        return len(self.views)

    def __contains__(self, name):
        return name in self.views

    def keys(self):
        return self.views.keys()

    def values(self):
        return self.views.values()

    def items(self):
        return self.views.items()


def _numel(shape):
    n = 1
    for s in shape:
        n *= s
    return n


@dataclass
class OptimizerState:
    kind: str = "adam"
    m: torch.Tensor = None
    v: torch.Tensor = None
    t: int = 0
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8


@dataclass
class RankState:
    """Per-rank replica of everything training mutates (reference engine.py:197-203)."""

    params: FlatParams
    bn_states: dict
    opt: OptimizerState


def init_params(net: NetworkSpec, seed: int = 0) -> FlatParams:
    """Kaiming-uniform U(+-sqrt(6/fan_in)) drawn from prng [seed,-1,i] in fp64
    on the device then cast; gamma 1, beta/bias 0 (reference optim.py:97-113).
    Bit-identical to the reference's fp32 initialisation."""
    fp = FlatParams(net)
    for i, (name, shape, fan_in) in enumerate(fp.entries):
        view = fp.views[name]
        if fan_in == 0:
            view.fill_(1.0 if name.endswith(".gamma") else 0.0)
        else:
            b = (6.0 / fan_in) ** 0.5
            prng.uniform_device([seed, -1, i], view.numel(), -b, b, out=view.view(-1))
    return fp


def make_state(net: NetworkSpec, seed: int = 0, kind: str = "adam") -> RankState:
    fp = init_params(net, seed)
    bn = {}
    for layer in net.layers:
        if layer.kind == "bn":
            bn[layer.name] = D.BNState(fp.views[f"{layer.name}.gamma"], fp.views[f"{layer.name}.beta"])
    opt = OptimizerState(kind)
    if kind == "adam":
        opt.m = torch.zeros_like(fp.flat)
        opt.v = torch.zeros_like(fp.flat)
    return RankState(fp, bn, opt)


def lr_at(lr0: float, epoch: int, horizon: int = 100, terminal: float = 0.01) -> float:
    """Linear decay schedule (reference optim.py:20-31)."""
    e = min(max(epoch, 0), horizon)
    return lr0 * (1.0 - (1.0 - terminal) * e / horizon)


def optimizer_step(state: RankState, lr: float, scalars: "StepScalars" = None):
    """Adam (bias corrected, sqrt(v_hat)+eps) or SGD over the flat buffers
    (reference optim.py:63-93).  With `scalars` the step count, lr and bias
    corrections come from device memory (graph replay; StepScalars owns t)."""
    p, opt = state.params, state.opt
    st = stream_ptr()
    if scalars is not None:
        if opt.kind != "adam":
            raise ShapeMismatch("graph-captured steps support Adam only")
        _lib.call("vpx_adam_dev", p.flat.data_ptr(), p.grad.data_ptr(), opt.m.data_ptr(), opt.v.data_ptr(),
                  p.numel, scalars.hyper_ptr, opt.beta1, opt.beta2, opt.eps, st)
        return
    opt.t += 1
    if opt.kind == "adam":
        c1 = 1.0 - opt.beta1 ** opt.t
        c2 = 1.0 - opt.beta2 ** opt.t
        _lib.call("vpx_adam", p.flat.data_ptr(), p.grad.data_ptr(), opt.m.data_ptr(), opt.v.data_ptr(),
                  p.numel, float(lr), opt.beta1, opt.beta2, float(c1), float(c2), opt.eps, st)
    else:
        _lib.call("vpx_sgd", p.flat.data_ptr(), p.grad.data_ptr(), p.numel, float(lr), st)


# ------------------------------------------------------------------ forward

def _flat_mask(layer_idx, step_key, sample_ids, features, keep, scalars=None):
    seed, epoch, it = step_key
    if scalars is not None:  # keys live in device memory, rewritten per replay
        rows = []
        for s in sample_ids:
            out = torch.empty(features, dtype=torch.uint8, device="cuda")
            _lib.call("vpx_prng_mask_dev", scalars.key_ptr(layer_idx, int(s)), features, float(keep),
                      out.data_ptr(), stream_ptr())
            rows.append(out)
    else:
        rows = [prng.keep_mask_device([seed, epoch, it, int(s), layer_idx], features, keep) for s in sample_ids]
    if not rows:
        return torch.zeros((0, features), dtype=torch.uint8, device="cuda")
    return torch.stack(rows)


def _apply_mask(x, mask, keep):
    return x * (mask.to(x.dtype) / keep)


def _flatten(t: DistTensor):
    """NCDHW-order flatten of a lead-local block (reference engine.py:249-258)."""
    return t.to_ncdhw().reshape(t.n, -1)


def _no_fused_pool() -> bool:
    return os.environ.get("VPX_NO_FUSED_POOL", "") == "1"


def forward(ctx: RankCtx, plan: Plan, state: RankState, batch: Batch, mode: str, seed: int = 0,
            trace: dict = None, scalars: "StepScalars" = None, pack_wait: torch.cuda.Event = None):
    net = plan.net
    P, bn = state.params.views, state.bn_states
    me = ctx.rank
    step_key = (seed, batch.epoch, batch.iteration)
    cur = None
    gr0 = _grid_rank(plan.input_meta, me)
    if gr0 is not None:
        if batch.x_block is None:
            raise ShapeMismatch(f"rank {me} holds an input block but the batch has none")
        cur = batch.x_block if isinstance(batch.x_block, DistTensor) else \
            DistTensor(plan.input_meta, gr0, batch.x_block)
    outputs, stash = {}, []
    fused_act = False
    skip_to = -1
    for i, layer in enumerate(net.layers):
        if i < skip_to:
            continue
        fused_block = (trace is None and cur is not None and layer.kind == "conv" and i + 3 < len(net.layers)
                and net.layers[i + 1].kind == "leaky" and net.layers[i + 2].kind == "pool"
                and len({plan.placement[i], plan.placement[i + 1], plan.placement[i + 2]}) == 1
                and plan.placement[i] != "flat" and plan.redist_idx not in (i, i + 1, i + 2)
                and not any(getattr(l, "skip", None) in (layer.name, net.layers[i + 1].name)
                            for l in net.layers)
                and (D.first_block_fwd_supported(cur, layer.params, net.layers[i + 2].pool_kind,
                                                 net.layers[i + 1].slope) if i == 0 else
                     D.block_fwd_pool_supported(cur, layer.params, net.layers[i + 2].pool_kind,
                                                net.layers[i + 1].slope))
                and not _no_fused_pool())
        if pack_wait is not None and (i > 0 or not fused_block):
            # weights packed ahead on the side stream (train_step); the fused
            # first block packs its own and runs while they are being made
            torch.cuda.current_stream().wait_event(pack_wait)
            pack_wait = None
        if fused_block:
            # conv -> leaky -> avg pool in one kernel: pooled output + sign mask
            pooled, mask = D.first_block_fwd(ctx, cur, P[f"{layer.name}.w"], layer.params,
                                             net.layers[i + 1].slope, plan.out_radii[i + 2], tag=layer.name)
            stash.extend([cur, mask, mask])
            outputs[layer.name] = outputs[net.layers[i + 1].name] = None
            outputs[net.layers[i + 2].name] = pooled
            cur = pooled
            skip_to = i + 3
            continue
        if i == plan.redist_idx and plan.placement[i] != "flat":
            cur = D.redistribute(ctx, cur, plan.redist_src_meta, plan.in_meta[i])
        if plan.placement[i] == "flat":
            if layer.kind == "flatten":
                if plan.redist_idx == i:
                    cur = D.redistribute(ctx, cur, plan.redist_src_meta, plan.in_meta[i])
                stash.append(None)
                if cur is not None:
                    cur = _flatten(cur)
            elif cur is None:
                stash.append(None)
            elif layer.kind == "fc":
                stash.append(cur)
                cur = torch.addmm(P[f"{layer.name}.b"], cur, P[f"{layer.name}.w"])
            elif layer.kind == "leaky":
                stash.append(cur)
                cur = torch.where(cur >= 0, cur, cur * layer.slope)
            elif layer.kind == "dropout":
                if mode == "train":
                    m = _flat_mask(i, step_key, batch.sample_ids, cur.shape[1], layer.keep, scalars)
                    cur = _apply_mask(cur, m, layer.keep)
                    stash.append(m)
                else:
                    stash.append(None)
            else:
                raise ShapeMismatch(f"layer kind {layer.kind!r} after flatten")
            outputs[layer.name] = cur
            continue
        if cur is None:
            stash.append(None)
            outputs[layer.name] = None
            continue
        radii = plan.out_radii[i]
        if fused_act:
            # this LeakyReLU already ran in the previous conv's epilogue; its
            # backward only needs the activation output (sign-preserving)
            fused_act = False
            stash.append(cur)
            outputs[layer.name] = cur
            continue
        if layer.kind == "conv":
            stash.append(cur)
            nxt = net.layers[i + 1] if i + 1 < len(net.layers) else None
            fused_act = (trace is None and nxt is not None and nxt.kind == "leaky"
                         and plan.placement[i + 1] == plan.placement[i] and plan.redist_idx != i + 1)
            cur = D.dist_conv3d(ctx, cur, P[f"{layer.name}.w"], layer.params,
                                plan.out_radii[i + 1] if fused_act else radii, tag=layer.name,
                                leaky_slope=nxt.slope if fused_act else None)
        elif layer.kind == "deconv":
            stash.append(cur)
            cur = D.dist_deconv3d(ctx, cur, P[f"{layer.name}.w"], radii, tag=layer.name)
        elif layer.kind == "pool":
            stash.append(cur)
            cur = D.dist_pool3d(ctx, cur, layer.pool_kind, radii, tag=layer.name)
        elif layer.kind == "bn":
            nxt = net.layers[i + 1] if i + 1 < len(net.layers) else None
            fused_act = (trace is None and nxt is not None and nxt.kind == "leaky" and cur.c % 4 == 0
                         and plan.placement[i + 1] == plan.placement[i] and plan.redist_idx != i + 1)
            cur, cache = D.dist_batchnorm(ctx, cur, bn[layer.name], mode,
                                          plan.out_radii[i + 1] if fused_act else radii, tag=layer.name,
                                          leaky_slope=nxt.slope if fused_act else None)
            stash.append(cache)
        elif layer.kind == "leaky":
            stash.append(cur)
            cur = D.dist_leaky_relu(cur, layer.slope, radii, tag=layer.name)
        elif layer.kind == "concat":
            skip = outputs[layer.skip]
            stash.append((cur.c, skip.c, cur, skip))
            cur = D.dist_concat_channels(cur, skip, radii, tag=layer.name)
        elif layer.kind == "dropout":
            raise ShapeMismatch("spatial dropout is not part of either network")
        else:
            raise ShapeMismatch(f"unknown layer kind {layer.kind!r}")
        outputs[layer.name] = cur
    if trace is not None:
        for name, value in outputs.items():
            trace[("fwd", name)] = value
    return cur, stash


def loss_and_grad(ctx: RankCtx, plan: Plan, pred, batch: Batch):
    """(loss as a 1-element fp64 CUDA tensor, identical on every rank; dpred)."""
    net = plan.net
    if net.loss == "mse":
        size = plan.n_global * net.out_dim
        return D.dist_mse(ctx, pred, batch.target, size, None)
    gs = plan.label_meta.global_shape
    count = gs.n * gs.d * gs.h * gs.w
    if pred is None:
        local = torch.zeros(1, dtype=torch.float64, device="cuda")
        ctx.allreduce_sum_(local)
        return local / count, None
    loss, g = D.dist_cross_entropy(ctx, pred, batch.y_block, count, None)
    return loss, g


def backward(ctx: RankCtx, plan: Plan, state: RankState, stash, dpred, trace: dict = None,
             buckets: "GradBuckets" = None):
    """Backward pass writing gradient partials into the flat bucket; with
    `buckets`, finished buckets are all-reduced while lower layers run."""
    net = plan.net
    P, G, bn = state.params.views, state.params.grads, state.bn_states
    u = dpred
    extra = {}
    skip_below = None
    skip_one = None
    if buckets is not None:
        buckets.start()
    for i in range(len(net.layers) - 1, -1, -1):
        layer = net.layers[i]
        if buckets is not None:
            buckets.layers_done_above(i)
        kept = stash[i]
        if skip_below is not None and i >= skip_below:
            continue
        if (trace is None and u is not None and layer.kind == "pool" and i == 2
                and D.first_block_fast_path(net.layers[0], net.layers[1], kept, u, plan.in_meta[0])):
            # conv(Cin=4) -> leaky -> pool: fused pool/leaky backward in the
            # blocked layout + the dense c1 filter-gradient kernel; nothing
            # consumes the network input's gradient
            D.first_block_wgrad(ctx, stash[0], kept, u, net.layers[1].slope, layer.pool_kind,
                                G[f"{net.layers[0].name}.w"], tag=net.layers[0].name)
            u = None
            skip_below = 0
            continue
        if (trace is None and u is not None and layer.kind == "pool" and i >= 1
                and net.layers[i - 1].kind == "leaky" and stash[i - 1] is kept and kept.c % 4 == 0
                and layer.name not in extra and net.layers[i - 1].name not in extra
                and plan.redist_idx not in (i, i - 1) and plan.placement[i] != "flat"):
            # leaky -> pool backward fused into one pass over the block
            act = net.layers[i - 1]
            u = D.dist_pool_leaky_bwd(kept, u, act.slope, layer.pool_kind, plan.in_meta[i - 1], tag=act.name)
            skip_below = None
            skip_one = i - 1
            continue
        if skip_one == i:
            continue
        if plan.placement[i] == "flat":
            if layer.kind == "flatten":
                if u is not None:
                    m = _meta_like(plan.in_meta[i])
                    gr = _grid_rank(m, ctx.rank)
                    ls = m.local_shape(gr)
                    u = DistTensor(m, gr, u.reshape(ls.n, ls.c, ls.d, ls.h, ls.w))
                if plan.redist_idx == i:
                    u = D.redistribute(ctx, u, _meta_like(plan.in_meta[i]), plan.redist_src_meta)
            elif u is None:
                pass
            elif layer.kind == "fc":
                w = P[f"{layer.name}.w"]
                torch.mm(kept.t(), u, out=G[f"{layer.name}.w"])
                torch.sum(u, dim=0, out=G[f"{layer.name}.b"])
                u = u @ w.t()
            elif layer.kind == "leaky":
                u = torch.where(kept >= 0, u, u * layer.slope)
            elif layer.kind == "dropout":
                if kept is not None:
                    u = _apply_mask(u, kept, layer.keep)
            if trace is not None:
                trace[("bwd", layer.name)] = u
            continue
        if u is not None and layer.name in extra:
            # in place, unless a trace holds on to u
            u = D.add_into(u.clone() if trace is not None else u, extra.pop(layer.name))
        if u is None:
            if i == plan.redist_idx:
                u = D.redistribute(ctx, None, _meta_like(plan.in_meta[i]), plan.redist_src_meta)
            if trace is not None:
                trace[("bwd", layer.name)] = u
            continue
        in_meta = plan.in_meta[i]
        if layer.kind == "conv":
            srcs = None
            if trace is None and i > 0 and net.layers[i - 1].kind == "concat":
                srcs = D.concat_wgrad_sources(kept, stash[i - 1][2:], u, layer.params)
            if srcs is not None:
                D.dist_conv3d_bwd_filter_slices(ctx, srcs, u, layer.params, G[f"{layer.name}.w"], tag=layer.name)
            else:
                D.dist_conv3d_bwd_filter(ctx, kept, u, layer.params, reduce=False, out=G[f"{layer.name}.w"],
                                         tag=layer.name)
            if i == 0 and trace is None:
                u = None  # nothing consumes the network input's gradient
            else:
                u = D.dist_conv3d_bwd_data(ctx, u, P[f"{layer.name}.w"], layer.params, in_meta, tag=layer.name)
        elif layer.kind == "deconv":
            D.dist_deconv3d_bwd_filter(ctx, kept, u, reduce=False, out=G[f"{layer.name}.w"], tag=layer.name)
            u = D.dist_deconv3d_bwd_data(ctx, u, P[f"{layer.name}.w"], in_meta, tag=layer.name)
        elif layer.kind == "pool":
            u = D.dist_pool3d_bwd(ctx, kept, u, layer.pool_kind, in_meta, tag=layer.name)
        elif layer.kind == "bn":
            u, _, _ = D.dist_batchnorm_bwd(ctx, u, bn[layer.name], kept, in_meta, tag=layer.name,
                                           dgamma=G[f"{layer.name}.gamma"], dbeta=G[f"{layer.name}.beta"])
        elif layer.kind == "leaky":
            u = D.dist_leaky_relu_bwd(kept, u, layer.slope, in_meta, tag=layer.name)
        elif layer.kind == "concat":
            c_main = kept[0]
            main, sk = D.dist_concat_bwd(u, c_main, _meta_like(in_meta),
                                         _skip_meta(plan, layer), extra.get(layer.skip), tag=layer.name)
            extra[layer.skip] = sk
            u = main
        if u is not None and i == plan.redist_idx:
            u = D.redistribute(ctx, u, _meta_like(in_meta), plan.redist_src_meta)
        if trace is not None:
            trace[("bwd", layer.name)] = u
    return G


def _skip_meta(plan: Plan, concat_layer):
    """Layout of the skip source's output (the concat's second operand)."""
    net = plan.net
    j = net.layer_index(concat_layer.skip)
    src_in = plan.in_meta[j]
    gs = src_in.global_shape
    o = out_shape(net.layers[j], (gs.n, gs.c, gs.d, gs.h, gs.w))
    return make_partition(Shape5D(*o), src_in.grid, NO_HALO, src_in.rank_map)


BUCKET_BYTES = int(os.environ.get("VPX_BUCKET_MB", "4")) << 20


class GradBuckets:
    """The flat gradient all-reduce (reference engine.py:446-462: one sum over
    all ranks of the bucket in param_entries order) split into contiguous
    buckets of >= BUCKET_BYTES at parameter boundaries and overlapped with the
    backward pass: backward() visits layers last to first, so once it reaches
    layer i every parameter of layers > i is final, and each bucket whose
    parameters all belong to finished layers is reduced at once, on a
    communication stream and a communicator of its own, while the lower
    layers' kernels run.  The sum is the same (each element is reduced exactly
    once over the same ranks); finish() joins the stream before the optimizer."""

    def __init__(self, ctx: RankCtx, net: NetworkSpec, params: "FlatParams"):
        self.ctx, self.params = ctx, params
        owner = {name: net.layer_index(name.rsplit(".", 1)[0]) for name, _, _ in params.entries}
        self.buckets = []  # (lo, hi, lowest owning layer)
        lo, low = 0, None
        for name, _, _ in params.entries:
            pos, cnt = params.offsets[name]
            low = owner[name] if low is None else min(low, owner[name])
            if 4 * (pos + cnt - lo) >= BUCKET_BYTES:
                self.buckets.append((lo, pos + cnt, low))
                lo, low = pos + cnt, None
        if lo < params.numel:
            self.buckets.append((lo, params.numel, low))
        self.pending = []
        self.group = ctx.grad_group()
        self.stream = ctx.grad_stream()

    def start(self):
        self.pending = sorted(range(len(self.buckets)), key=lambda b: -self.buckets[b][2])

    def layers_done_above(self, i: int):
        """Every layer with index > i has its gradients final: launch the
        buckets they complete."""
        while self.pending and self.buckets[self.pending[0]][2] > i:
            self._launch(self.pending.pop(0))

    def _launch(self, b):
        lo, hi, _ = self.buckets[b]
        cur = torch.cuda.current_stream()
        self.stream.wait_stream(cur)
        with torch.cuda.stream(self.stream):
            view = self.params.grad[lo:hi]
            with region("comm.allreduce_grad", 0, 4 * (hi - lo)):
                dist.all_reduce(view, op=dist.ReduceOp.SUM, group=self.group)

    def finish(self):
        self.layers_done_above(-1)
        torch.cuda.current_stream().wait_stream(self.stream)


def gradient_allreduce(ctx: RankCtx, state: RankState, buckets: "GradBuckets" = None):
    """Sum of the gradient bucket over all ranks (reference engine.py:446-462):
    the buckets backward() has not launched yet, then the join; without
    buckets (single rank or a caller-driven backward) one flat all-reduce."""
    if buckets is not None:
        buckets.finish()
        return
    ctx.allreduce_sum_(state.params.grad, None)


def train_step(ctx: RankCtx, plan: Plan, state: RankState, batch: Batch, lr: float, seed: int = 0,
               scalars: "StepScalars" = None, as_tensor: bool = False):
    """One hybrid-parallel training step (reference engine.py:465-473).
    Returns the loss as a float, identical on every rank, like the reference
    -- which reads it back, i.e. synchronises with the device.  With
    as_tensor=True it returns the 1-element fp64 CUDA tensor instead and the
    step queues without any host synchronisation (except once per plan, when
    the halo mailboxes are set up); CapturedStep and the bench use that."""
    ctx.ensure_peer_halo(plan)
    buckets = _buckets(ctx, plan, state)
    pack_wait = _prepack(state)
    state.params.grad.zero_()
    pred, stash = forward(ctx, plan, state, batch, "train", seed, scalars=scalars, pack_wait=pack_wait)
    loss, dpred = loss_and_grad(ctx, plan, pred, batch)
    backward(ctx, plan, state, stash, dpred, buckets=buckets)
    gradient_allreduce(ctx, state, buckets)
    optimizer_step(state, lr, scalars)
    if pack_wait is not None:
        _lib.call("vpx_prepack_end")  # the optimizer changed the weights: no pack is current
    return loss if as_tensor else float(loss.item())


_PACK_STREAM = {}


def _prepack(state: RankState):
    """Pack every conv pass's weights for this step on a side stream, in
    parallel with the first layer (vpx_prepack_*, csrc/conv_host.cu): the
    passes recorded their packs on earlier steps and now read the packed
    buffers instead of packing inline (~10 us per deep-layer pass).  The
    returned event is what forward() waits on before its first conv that may
    read them.  VPX_NO_PREPACK=1 keeps every pack inline."""
    if os.environ.get("VPX_NO_PREPACK") == "1" or not torch.cuda.is_available():
        return None
    _lib.call("vpx_prepack_begin", state.params.flat.data_ptr(), state.params.flat.numel())
    dev = torch.cuda.current_device()
    side = _PACK_STREAM.get(dev)
    if side is None:
        side = _PACK_STREAM[dev] = torch.cuda.Stream()
    cur = torch.cuda.current_stream()
    side.wait_stream(cur)
    with torch.cuda.stream(side):
        _lib.call("vpx_prepack_all", stream_ptr())
        ev = torch.cuda.Event()
        ev.record(side)
    return ev


def _buckets(ctx: RankCtx, plan: Plan, state: RankState):
    """The overlapped bucketed all-reduce (GradBuckets) for multi-rank steps,
    built once per (plan, state); VPX_FLAT_ALLREDUCE=1 keeps one flat
    all-reduce after the backward pass."""
    if ctx.size == 1 or os.environ.get("VPX_FLAT_ALLREDUCE") == "1":
        return None
    b = getattr(state, "_buckets", None)
    if b is None or b[0] is not plan:
        state._buckets = (plan, GradBuckets(ctx, plan.net, state.params))
    return state._buckets[1]


class StepScalars:
    """Per-step scalars that a captured step reads from device memory: Adam's
    {lr, 1-b1^t, 1-b2^t} and one folded dropout key per (dropout layer,
    sample).  `set(...)` recomputes them on the host (same formulas as the
    eager step: reference optim.py:71-88, engine.py:314-320) and queues one
    pinned host->device copy on the current stream.

    The host side is a ring of pinned slots, each guarded by an event recorded
    after its copy: a slot is rewritten only once the copy that read it has
    completed, so the host may queue any number of replays without
    synchronising and every replay still sees its own step's scalars."""

    RING = 4

    def __init__(self, net: NetworkSpec, sample_ids):
        self.slots = {}
        for i, layer in enumerate(net.layers):
            if layer.kind == "dropout":
                for s in sample_ids:
                    self.slots[(i, int(s))] = len(self.slots)
        self.dev = torch.zeros(4 + 2 * max(1, len(self.slots)), dtype=torch.float32, device="cuda")
        self._ring = [torch.zeros_like(self.dev, device="cpu").pin_memory() for _ in range(self.RING)]
        self._done = [None] * self.RING
        self._next = 0
        self.hyper_ptr = self.dev.data_ptr()

    def key_ptr(self, layer_idx: int, sample_id: int) -> int:
        return self.dev.data_ptr() + 16 + 8 * self.slots[(layer_idx, sample_id)]

    def set(self, state: RankState, lr: float, step_key):
        k = self._next
        self._next = (k + 1) % self.RING
        if self._done[k] is not None:
            self._done[k].synchronize()  # the copy that last read this slot has finished
        host = self._ring[k]
        keys = host[4:].view(torch.int64)
        opt = state.opt
        opt.t += 1
        host[0] = float(lr)
        host[1] = float(1.0 - opt.beta1 ** opt.t)
        host[2] = float(1.0 - opt.beta2 ** opt.t)
        seed, epoch, it = step_key
        for (i, s), j in self.slots.items():
            v = prng.key_fold([seed, epoch, it, s, i])
            keys[j] = v - (1 << 64) if v >= (1 << 63) else v
        self.dev.copy_(host, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self._done[k] = ev


class CapturedStep:
    """train_step captured once in a CUDA graph and replayed (no per-kernel
    launch cost, no Python on the hot path).  Shapes, buffers and the batch's
    device frames are fixed at capture; per-step scalars (lr, Adam bias
    corrections, dropout keys) go through StepScalars, the input block is
    refreshed in place (e.g. HostInputPipeline.load) before each call.  The
    loss tensor returned is the graph's static output."""

    def __init__(self, ctx: RankCtx, plan: Plan, state: RankState, batch: Batch, lr: float, seed: int = 0,
                 warmup: int = 2, recorder=None):
        self.ctx, self.plan, self.state, self.batch, self.seed = ctx, plan, state, batch, seed
        self.scalars = StepScalars(plan.net, batch.sample_ids)
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(warmup):  # real steps: settles workspaces and allocator state
                self.scalars.set(state, lr, (seed, batch.epoch, batch.iteration))
                train_step(ctx, plan, state, batch, lr, seed, scalars=self.scalars, as_tensor=True)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        # recorder: a timing.Recorder(graph=True) active during the capture only
        # (its regions become event nodes re-timed by every replay)
        with torch.cuda.graph(self.graph), (recorder if recorder is not None else contextlib.nullcontext()):
            self.loss = train_step(ctx, plan, state, batch, lr, seed, scalars=self.scalars, as_tensor=True)

    def __call__(self, lr: float, epoch: int = None, iteration: int = None):
        b = self.batch
        if epoch is not None:
            b.epoch = epoch
        if iteration is not None:
            b.iteration = iteration
        self.scalars.set(self.state, lr, (self.seed, b.epoch, b.iteration))
        self.graph.replay()
        return self.loss


# ------------------------------------------------------------------ batches

def synthetic_batch_full(net: NetworkSpec, w_i: int, n: int, seed: int = 0):
    """The reference's deterministic verify batch (reference cli.py:112-125):
    x = prng.uniform([seed,-3,0], N*C*W^3, -1, 1) as NCDHW, targets
    uniform([seed,-3,1]) (mse) or labels randint([seed,-3,1], 0, K) (xent).
    Generated on the device; bit-identical to the reference's values."""
    shape = (n, net.in_channels, w_i, w_i, w_i)
    numel = shape[0] * shape[1] * shape[2] * shape[3] * shape[4]
    x = prng.uniform_device([seed, -3, 0], numel, -1.0, 1.0).reshape(shape)
    if net.loss == "mse":
        y = prng.uniform_device([seed, -3, 1], n * net.out_dim, -1.0, 1.0).reshape(n, net.out_dim)
    else:
        y = randint_device([seed, -3, 1], n * w_i ** 3, 0, net.out_dim).reshape(n, w_i, w_i, w_i)
    return x, y, tuple(range(n))


def randint_device(key, n, lo, hi):
    """prng.randint (modulo-mapped u64) on the host stream; labels are small."""
    import numpy as np

    from .prng import resolve, GOLDEN, MASK

    k = np.uint64(resolve(key))
    ctr = np.arange(n, dtype=np.uint64)
    z = k + (ctr + np.uint64(1)) * np.uint64(GOLDEN)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    z = z ^ (z >> np.uint64(31))
    vals = (z % np.uint64(hi - lo)).astype(np.int64) + lo
    return torch.from_numpy(vals).cuda()


def scatter_batch(plan: Plan, x, y, sample_ids, rank: int, epoch: int = 0, iteration: int = 0) -> Batch:
    """This rank's Batch from a global NCDHW batch (device or host tensors).
    Group g owns rows [g*n_local, (g+1)*n_local) (reference engine.py:482-513)."""
    n_local = plan.n_global // plan.grid.groups
    g = plan.grid.coords(rank)[0]
    rows = slice(g * n_local, (g + 1) * n_local)
    ids = tuple(int(s) for s in sample_ids)[rows]
    b = Batch(sample_ids=ids, epoch=epoch, iteration=iteration)
    gin = _grid_rank(plan.input_meta, rank)
    if gin is not None:
        meta = plan.input_meta
        reg = meta.region(gin)
        lo, hi = meta.sample_range(meta.group_of(gin))
        sl = (slice(lo, hi), slice(None)) + reg.slices()
        b.x_block = DistTensor(meta, gin, torch.as_tensor(x)[sl])
    if plan.net.loss == "mse":
        b.target = torch.as_tensor(y)[rows].to("cuda", torch.float32)
    else:
        gl = _grid_rank(plan.label_meta, rank)
        if gl is not None:
            reg = plan.label_meta.region(gl)
            lo, hi = plan.label_meta.sample_range(plan.label_meta.group_of(gl))
            b.y_block = torch.as_tensor(y)[(slice(lo, hi),) + reg.slices()].to("cuda", torch.int64).contiguous()
    return b


class HostInputPipeline:
    """Streams per-step input blocks from pinned host memory into a Batch.

    The reference reads each step's block from its datastore on the host
    (reference data/datastore.py:156-179) and hands numpy arrays to the step.
    Here the block is copied host->device on a dedicated copy stream into one
    of two staging buffers while the previous step computes; `load(batch)`
    makes the compute stream wait for that copy, converts the staged NCDHW
    block into the batch's halo frame (vpx_layout_ncdhw_to_frame) and queues
    the next copy.  Copies therefore overlap compute and the step itself sees
    no host synchronisation.

    host_blocks: a callable step -> pinned NCDHW host tensor (this rank's
    block), or a single tensor reused every step.
    """

    def __init__(self, host_blocks, device=None):
        self._src = host_blocks if callable(host_blocks) else (lambda i, t=host_blocks: t)
        first = self._src(0)
        self.shape = tuple(first.shape)
        self.bytes_per_step = first.numel() * first.element_size()
        self.copy_stream = torch.cuda.Stream(device=device)
        self._buf = [torch.empty(self.shape, dtype=first.dtype, device="cuda") for _ in range(2)]
        self._ready = [torch.cuda.Event() for _ in range(2)]
        self._free = [torch.cuda.Event() for _ in range(2)]
        self._free_recorded = [False, False]
        self._step = 0
        self._issued = -1

    def _issue(self, i):
        slot = i % 2
        with torch.cuda.stream(self.copy_stream):
            if self._free_recorded[slot]:
                self.copy_stream.wait_event(self._free[slot])
            blk = self._src(i)
            if blk.dtype != self._buf[slot].dtype or tuple(blk.shape) != self.shape:
                raise ShapeMismatch(f"input block {i}: {blk.dtype} {tuple(blk.shape)}, pipeline staged "
                                    f"{self._buf[slot].dtype} {self.shape}")
            self._buf[slot].copy_(blk, non_blocking=True)
            self._ready[slot].record(self.copy_stream)
        self._issued = i

    def start(self, after: torch.cuda.Event = None):
        """Queue the first copy (optionally after `after` on the copy stream)."""
        if after is not None:
            self.copy_stream.wait_event(after)
        self._issue(self._step)

    def load(self, batch: "Batch", prefetch_next: bool = True) -> "Batch":
        i = self._step
        if self._issued < i:
            self._issue(i)
        slot = i % 2
        cur = torch.cuda.current_stream()
        cur.wait_event(self._ready[slot])
        batch.x_block.load_ncdhw(self._buf[slot])
        self._free[slot].record(cur)
        self._free_recorded[slot] = True
        self._step += 1
        if prefetch_next:
            self._issue(self._step)
        return batch


class PipelinedSteps:
    """Training-loop driver over host-resident input blocks: the end-to-end
    path (HSB1 datastore -> pinned host block -> device -> step -> loss on
    the host) with no host->device work on the compute stream.

    Two input frames, each with its own captured step graph (CapturedStep on
    a twin of `batch` whose x_block is a second DistTensor).  While step i
    replays from frame i % 2, a copy stream moves step i+1's pinned block to
    a device staging buffer and converts it into frame (i+1) % 2 with the
    int -> fp32 layout kernel (vpx_layout_ncdhw_i8/i16_to_frame), so both the
    PCIe copy and the layout overlap compute; a frame is rewritten only after
    the graph that read it has finished (an event per frame).  Each step's
    loss is copied to pinned host memory asynchronously; `step()` returns the
    PREVIOUS step's loss as a float (its copy completed while this step was
    queued), `finish()` the last one.  The reference reads each step's block
    from its datastore on the host and calls train_step (reference
    data/datastore.py:156-179, model/engine.py:465-473).

    host_blocks: a callable step -> pinned NCDHW host tensor (this rank's
    block) or one tensor reused every step.  Ranks holding no input block
    (batch.x_block is None) replay without input traffic.
    """

    def __init__(self, ctx: RankCtx, plan: Plan, state: RankState, batch: Batch, host_blocks, lr: float,
                 seed: int = 0, warmup: int = 2, layout_sms: int = None):
        self.layout_sms = int(os.environ.get("VPX_PIPE_LAYOUT_SMS", "0")) if layout_sms is None else layout_sms
        twin = Batch(x_block=batch.x_block.clone() if batch.x_block is not None else None, target=batch.target,
                     y_block=batch.y_block, sample_ids=batch.sample_ids, epoch=batch.epoch,
                     iteration=batch.iteration)
        self.batches = (batch, twin)
        self.caps = tuple(CapturedStep(ctx, plan, state, b, lr, seed, warmup=warmup) for b in self.batches)
        self.has_input = batch.x_block is not None and host_blocks is not None
        self._src = host_blocks if callable(host_blocks) else (lambda i, t=host_blocks: t)
        self.copy_stream = torch.cuda.Stream()
        self.bytes_per_step = 0
        if self.has_input:
            first = self._src(0)
            self.shape, self.dtype = tuple(first.shape), first.dtype
            self.bytes_per_step = first.numel() * first.element_size()
            self._stage = [torch.empty(self.shape, dtype=self.dtype, device="cuda") for _ in range(2)]
        self._ready = [torch.cuda.Event() for _ in range(2)]
        self._free = [None, None]
        self._loss_host = None  # pinned, allocated with the loss dtype at the first step
        self._loss_ev = [torch.cuda.Event() for _ in range(2)]
        self.i = 0
        self._prepared = -1

    def _prepare(self, i: int):
        f = i % 2
        cs = self.copy_stream
        with torch.cuda.stream(cs):
            if self.has_input:
                blk = self._src(i)
                if blk.dtype != self.dtype or tuple(blk.shape) != self.shape:
                    raise ShapeMismatch(f"input block {i}: {blk.dtype} {tuple(blk.shape)}, pipeline staged "
                                        f"{self.dtype} {self.shape}")
                # the PCIe copy needs only the staging buffer (last read by
                # the previous layout on this stream), so it may start while
                # the step before the previous one still runs
                self._stage[f].copy_(blk, non_blocking=True)
            if self._free[f] is not None:  # the frame: once the graph that read it is done
                cs.wait_event(self._free[f])
            if self.has_input:
                # layout_sms: optionally confine the layout kernel to a few
                # SMs' worth of blocks (vpx_set_sm_limit) while it runs beside the step
                if self.layout_sms:
                    _lib.call("vpx_set_sm_limit", self.layout_sms)
                try:
                    self.batches[f].x_block.load_ncdhw(self._stage[f])
                finally:
                    if self.layout_sms:
                        _lib.call("vpx_set_sm_limit", 0)
            self._ready[f].record(cs)
        self._prepared = i

    def start(self, after: torch.cuda.Event = None):
        """Queue step 0's input (optionally after `after` on the copy stream)."""
        if after is not None:
            self.copy_stream.wait_event(after)
        self._prepare(self.i)

    def step(self, lr: float, prefetch_next: bool = True):
        i, f = self.i, self.i % 2
        if self._prepared < i:
            self._prepare(i)
        cur = torch.cuda.current_stream()
        cur.wait_event(self._ready[f])
        loss = self.caps[f](lr)
        done = torch.cuda.Event()
        done.record(cur)
        self._free[f] = done
        if self._loss_host is None:
            self._loss_host = torch.zeros(2, dtype=loss.dtype).pin_memory()
        self._loss_host[f:f + 1].copy_(loss.reshape(1), non_blocking=True)
        self._loss_ev[f].record(cur)
        if prefetch_next:
            self._prepare(i + 1)
        prev = None
        if i > 0:
            self._loss_ev[1 - f].synchronize()
            prev = float(self._loss_host[1 - f])
        self.i += 1
        return prev

    def finish(self) -> float:
        """The last step's loss (waits for it)."""
        f = (self.i - 1) % 2
        self._loss_ev[f].synchronize()
        return float(self._loss_host[f])
