"""Generate golden fixtures by running the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
Writes tests/golden/{prng.json, geometry.json, plans.json, kernels.npz,
layers.npz, nets.npz, halo.npz}.  The GPU box never runs this (it has no
/root/reference); the committed fixtures travel with the repo.
"""

from __future__ import annotations

import json
import math
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

from voxpar import prng  # noqa: E402
from voxpar import kernels  # noqa: E402
from voxpar.fabric import halo_exchange, reverse_halo_exchange, run_ranks  # noqa: E402
from voxpar.layers import reference as R  # noqa: E402
from voxpar.model import engine, serial  # noqa: E402
from voxpar.model.networks import build_cosmoflow, build_unet_mini, param_entries, total_params  # noqa: E402
from voxpar.model.optim import OptimizerState, init_params  # noqa: E402
from voxpar.tensor import (DistTensor, ProcessGrid, Region, Shape5D, gather,  # noqa: E402
                           halo_faces, hyperslab_byte_ranges, make_partition, round_slices, scatter,
                           split_extent)
from voxpar.layers.accounting import network_flops  # noqa: E402

GRIDS = [(1, 1, 1, 1), (1, 2, 1, 1), (1, 4, 1, 1), (1, 8, 1, 1), (1, 2, 2, 1), (1, 1, 2, 2),
         (2, 2, 1, 1), (1, 2, 2, 2), (2, 4, 1, 1), (4, 2, 1, 1), (1, 4, 2, 1)]


def sl(s):
    return [s.start, s.stop]


def prng_fixture():
    keys = [[0, -1, 0], [0, -3, 0], [0, -3, 1], [7, 1, 2, 3, 4], [123456789, -2], [0]]
    out = {"key_fold": {}, "u64": {}, "uniform": {}, "randint": {}, "permutation": {}}
    for k in keys:
        s = json.dumps(k)
        out["key_fold"][s] = str(prng.key_fold(k))
        out["u64"][s] = [str(v) for v in prng.u64(k, 16)]
        out["uniform"][s] = [float(v) for v in prng.uniform(k, 16, -0.5, 2.0)]
        out["randint"][s] = [int(v) for v in prng.randint(k, 16, 0, 7)]
        out["permutation"][s] = [int(v) for v in prng.permutation(k, 12)]
    # long stream checksums (device generator vs reference at scale)
    big = prng.uniform([0, -3, 0], 1 << 20, -1.0, 1.0)
    out["uniform_1M_sum"] = float(big.sum())
    out["uniform_1M_head"] = [float(v) for v in big[:8]]
    out["uniform_1M_f32_bytes_sha"] = __import__("hashlib").sha256(big.astype(np.float32).tobytes()).hexdigest()
    (OUT / "prng.json").write_text(json.dumps(out, indent=1))


def geometry_fixture():
    cases = []
    for g in GRIDS:
        grid = ProcessGrid(*g)
        for shape, radii in (((g[0] * 2, 3, 16, 8, 8), (1, 1, 1)), ((g[0], 2, 8, 16, 16), (1, 0, 1)),
                             ((g[0] * 1, 1, 32, 32, 32), (2, 2, 2))):
            try:
                meta = make_partition(Shape5D(*shape), grid, radii)
            except Exception as e:  # noqa: BLE001
                cases.append({"grid": g, "shape": shape, "radii": radii, "error": type(e).__name__})
                continue
            ranks = []
            for r in range(grid.size):
                reg = meta.region(r)
                faces = [{"dim": f.dim, "side": f.side, "neighbor": f.neighbor, "face_id": f.face_id,
                          "send": [list(f.send.offset), list(f.send.extent)],
                          "recv": [list(f.recv.offset), list(f.recv.extent)]} for f in halo_faces(meta, r)]
                rounds = {}
                for dim in range(3):
                    for side in (-1, 1):
                        b, m = round_slices(meta, r, dim, side)
                        rounds[f"{dim},{side}"] = [[sl(s) for s in b[2:]], [sl(s) for s in m[2:]]]
                ranks.append({"coords": list(grid.coords(r)), "offset": list(reg.offset),
                              "extent": list(reg.extent), "faces": faces, "rounds": rounds,
                              "neighbors": [[meta.neighbor(r, d, s) for s in (-1, 1)] for d in range(3)]})
            cases.append({"grid": g, "shape": shape, "radii": radii, "ranks": ranks})
    errs = []
    for args in ((10, 3), (512, 8), (64, 1), (7, 0)):
        try:
            errs.append([list(args), [list(x) for x in split_extent(*args)]])
        except Exception as e:  # noqa: BLE001
            errs.append([list(args), type(e).__name__])
    slabs = []
    for fs, reg in (((2, 8, 8, 8), Region((0, 2, 0), (8, 3, 8))), ((1, 16, 16, 16), Region((4, 0, 0), (4, 16, 16))),
                    ((3, 4, 6, 5), Region((1, 1, 1), (2, 3, 2)))):
        slabs.append([list(fs), [list(reg.offset), list(reg.extent)], [list(r) for r in hyperslab_byte_ranges(fs, reg, 2)]])
    (OUT / "geometry.json").write_text(json.dumps({"cases": cases, "split": errs, "hyperslab": slabs}))


def plans_fixture():
    out = []
    for net_name, wi, n, with_bn in (("cosmoflow", 512, 1, False), ("cosmoflow", 256, 8, False),
                                     ("cosmoflow", 128, 8, False), ("cosmoflow", 64, 2, False),
                                     ("cosmoflow", 32, 2, True), ("unet", 16, 2, False), ("unet", 64, 1, False)):
        net = build_cosmoflow(wi, with_bn=with_bn) if net_name == "cosmoflow" else build_unet_mini(wi)
        for g in GRIDS:
            grid = ProcessGrid(*g)
            rec = {"net": net_name, "wi": wi, "n": n, "bn": with_bn, "grid": g}
            try:
                plan = engine.make_plan(net, grid, n, wi)
                rec.update(placement=list(plan.placement), redist=plan.redist_idx, leads=list(plan.leads),
                           out_radii=[list(r) for r in plan.out_radii],
                           in_radii=[list(m.radii) if m is not None else None for m in plan.in_meta])
            except Exception as e:  # noqa: BLE001
                rec["error"] = type(e).__name__
            out.append(rec)
    nets = {}
    for wi in (32, 64, 128, 256, 512):
        net = build_cosmoflow(wi)
        _, fwd, tot = network_flops(net, (1, 4, wi, wi, wi))
        nets[f"cosmoflow{wi}"] = {"params": total_params(net), "conv_fwd": fwd, "conv_total": tot,
                                  "layers": [l.name for l in net.layers],
                                  "entries": [[a, list(b), c] for a, b, c in param_entries(net)]}
    for wi in (16, 32, 64):
        net = build_unet_mini(wi)
        nets[f"unet{wi}"] = {"params": total_params(net), "layers": [l.name for l in net.layers],
                             "entries": [[a, list(b), c] for a, b, c in param_entries(net)]}
    (OUT / "plans.json").write_text(json.dumps({"plans": out, "nets": nets}))


def kernels_fixture():
    rng = np.random.default_rng(1234)
    arrs = {}
    for dt in (np.float32, np.float64):
        for case, (n, cin, cout, d, h, w, k, s) in enumerate(
                [(2, 3, 4, 9, 9, 9, 3, 1), (1, 4, 16, 6, 8, 10, 3, 2), (1, 2, 3, 5, 5, 5, 1, 1)]):
            x = rng.standard_normal((n, cin, d, h, w)).astype(dt)
            wt = rng.standard_normal((cout, cin, k, k, k)).astype(dt)
            p = R.ConvParams(cin, cout, (k,) * 3, (s,) * 3)
            y = R.conv3d_ref(x, wt, p)
            u = rng.standard_normal(y.shape).astype(dt)
            xg = R.conv3d_bwd_data_ref(u, wt, p, x.shape[2:])
            wg = R.conv3d_bwd_filter_ref(x, u, p)
            tag = f"{np.dtype(dt).name}_{case}"
            arrs.update({f"x_{tag}": x, f"w_{tag}": wt, f"u_{tag}": u, f"y_{tag}": y, f"xg_{tag}": xg,
                         f"wg_{tag}": wg, f"meta_{tag}": np.array([n, cin, cout, d, h, w, k, s])})
    np.savez_compressed(OUT / "kernels.npz", **arrs, backend=np.array(kernels.backend_name()))


def layers_fixture():
    rng = np.random.default_rng(99)
    A = {}
    x = rng.standard_normal((2, 3, 4, 6, 8))
    x[0, 0, 0:2, 0:2, 0:2] = 1.5  # ties: lowest index wins
    A["pool_x"] = x
    for kind in ("average", "max"):
        y = R.pool3d_ref(x, kind)
        u = rng.standard_normal(y.shape)
        A[f"pool_{kind}_y"], A[f"pool_{kind}_u"], A[f"pool_{kind}_g"] = y, u, R.pool3d_bwd_ref(x, u, kind)
    bx = rng.standard_normal((2, 5, 3, 4, 4)) * 2 + 0.5
    st = R.BNState.fresh(5)
    st.gamma[...] = rng.standard_normal(5)
    st.beta[...] = rng.standard_normal(5)
    A["bn_x"], A["bn_gamma"], A["bn_beta"] = bx, st.gamma.copy(), st.beta.copy()
    y, cache = R.batchnorm_fwd_ref(bx, st)
    bu = rng.standard_normal(bx.shape)
    dx, dg, db = R.batchnorm_bwd_ref(bu, st, cache)
    A.update(bn_y=y, bn_u=bu, bn_dx=dx, bn_dg=dg, bn_db=db, bn_rm=st.running_mean, bn_rv=st.running_var)
    lx = rng.standard_normal((3, 7))
    lx[0, 0] = 0.0
    lu = rng.standard_normal((3, 7))
    A.update(leaky_x=lx, leaky_u=lu, leaky_y=R.leaky_relu(lx, 0.3), leaky_g=R.leaky_relu_bwd(lx, lu, 0.3))
    dx_ = rng.standard_normal((2, 3, 2, 3, 4))
    dw_ = rng.standard_normal((3, 5, 2, 2, 2))
    dy = R.deconv3d_ref(dx_, dw_)
    du = rng.standard_normal(dy.shape)
    A.update(deconv_x=dx_, deconv_w=dw_, deconv_y=dy, deconv_u=du, deconv_g=R.deconv3d_bwd_data_ref(du, dw_),
             deconv_wg=R.deconv3d_bwd_filter_ref(dx_, du))
    lg = rng.standard_normal((2, 2, 3, 4, 5))
    lab = rng.integers(0, 2, (2, 3, 4, 5))
    loss, g = R.cross_entropy_ref(lg, lab)
    A.update(xent_logits=lg, xent_labels=lab, xent_loss=np.array(loss), xent_g=g)
    pr, tg = rng.standard_normal((4, 4)), rng.standard_normal((4, 4))
    ml, mg = R.mse_loss(pr, tg)
    A.update(mse_pred=pr, mse_target=tg, mse_loss=np.array(ml), mse_g=mg)
    A["dropout_mask"] = R.dropout_mask([0, 1, 2, 3, 4], 64, 0.8)
    np.savez_compressed(OUT / "layers.npz", **A)


def _sample(a, k=48):
    a = np.asarray(a).ravel()
    idx = np.linspace(0, a.size - 1, num=min(k, a.size)).astype(np.int64)
    return np.concatenate([[a.sum(), (a * a).sum(), np.abs(a).max()], a[idx]])


def nets_fixture():
    A = {}
    for tag, net, wi, n, dt in (("cf32_f64", build_cosmoflow(32), 32, 2, np.float64),
                                ("cf32bn_f64", build_cosmoflow(32, with_bn=True), 32, 2, np.float64),
                                ("un16_f64", build_unet_mini(16), 16, 2, np.float64),
                                ("cf64_f32", build_cosmoflow(64), 64, 2, np.float32)):
        x, y = _batch(net, wi, n, 0, dt)
        params = init_params(net, 0, dt)
        states = serial.make_bn_states(net, params, dt)
        trace = {}
        pred, stash = serial.forward(net, params, states, x, "train", (0, 0, 0), tuple(range(n)), trace=trace)
        loss, dpred = serial.loss_and_grad(net, pred, y)
        grads = serial.backward(net, params, states, stash, dpred, trace=trace)
        A[f"{tag}_loss"] = np.array(loss)
        for (ph, name), v in trace.items():
            A[f"{tag}_tr_{ph}_{name}"] = _sample(v)
        for name, g in grads.items():
            A[f"{tag}_grad_{name}"] = _sample(g)
        opt = OptimizerState.for_params("adam", params)
        from voxpar.model.optim import adam_step

        adam_step(params, grads, opt, 1e-3)
        for name, p in params.items():
            A[f"{tag}_param1_{name}"] = _sample(p)
    # distributed reference: 1 step on grid 1x2x1x1 and 2x2x1x1 (loss + gathered bwd input grads)
    net = build_cosmoflow(32)
    for g in ((1, 2, 1, 1), (2, 2, 1, 1)):
        grid = ProcessGrid(*g)
        plan = engine.make_plan(net, grid, 2, 32)
        x, y = _batch(net, 32, 2, 0, np.float64)
        params = init_params(net, 0, np.float64)
        batches = engine.scatter_batch(plan, x, y, tuple(range(2)))

        def fn(ctx):
            p = {k: v.copy() for k, v in params.items()}
            st = engine.RankState(p, serial.make_bn_states(net, p, np.float64), OptimizerState.for_params("adam", p))
            loss = engine.train_step(ctx, plan, st, batches[ctx.rank], 1e-3)
            return loss, {k: v.copy() for k, v in p.items()}

        res = run_ranks(grid.size, fn)
        A[f"dist_{'x'.join(map(str, g))}_loss"] = np.array([r[0] for r in res])
        for name, p in res[0][1].items():
            A[f"dist_{'x'.join(map(str, g))}_param1_{name}"] = _sample(p)
    np.savez_compressed(OUT / "nets.npz", **A)


def _batch(net, wi, n, seed, dt):
    shape = (n, net.in_channels, wi, wi, wi)
    x = prng.uniform([seed, -3, 0], math.prod(shape), -1.0, 1.0).reshape(shape).astype(dt)
    if net.loss == "mse":
        y = prng.uniform([seed, -3, 1], n * net.out_dim, -1.0, 1.0).reshape(n, net.out_dim).astype(dt)
    else:
        y = prng.randint([seed, -3, 1], n * wi ** 3, 0, net.out_dim).reshape(n, wi, wi, wi)
    return x, y


def halo_fixture():
    """Frames after halo_exchange / reverse_halo_exchange on the reference fabric
    (global-coordinate ramp), for bit-exact comparison of the device exchange."""
    A = {}
    for g, shape, radii in (((1, 2, 2, 1), (2, 3, 8, 8, 6), (1, 1, 1)), ((1, 2, 2, 2), (1, 2, 8, 8, 8), (1, 1, 1)),
                            ((1, 4, 1, 1), (1, 2, 16, 4, 4), (1, 1, 1)), ((2, 2, 1, 1), (2, 2, 8, 4, 4), (1, 0, 0)),
                            # 2-rank grids and channel counts % 4 == 0 (the device's fused peer round)
                            ((1, 2, 1, 1), (1, 4, 8, 6, 6), (1, 1, 1)), ((1, 1, 2, 1), (2, 8, 6, 8, 6), (1, 1, 1)),
                            ((1, 1, 1, 2), (1, 4, 6, 6, 8), (1, 1, 1)), ((2, 1, 2, 1), (2, 4, 6, 8, 6), (1, 1, 1))):
        grid = ProcessGrid(*g)
        meta = make_partition(Shape5D(*shape), grid, radii)
        full = np.arange(np.prod(shape), dtype=np.float64).reshape(shape) * 0.5 + 1.0
        blocks = scatter(meta, full)

        def fn(ctx):
            t = DistTensor(meta, ctx.rank, blocks[ctx.rank])
            halo_exchange(ctx, t)
            fr = t.padded().copy()
            grad = np.arange(fr.size, dtype=np.float64).reshape(fr.shape) * 0.25 - 3.0
            reverse_halo_exchange(ctx, meta, ctx.rank, grad)
            return fr, grad

        res = run_ranks(grid.size, fn)
        key = "x".join(map(str, g))
        for r, (fr, grad) in enumerate(res):
            A[f"{key}_r{r}_fwd"] = fr
            A[f"{key}_r{r}_rev"] = grad
        A[f"{key}_shape"] = np.array(shape)
        A[f"{key}_radii"] = np.array(radii)
    np.savez_compressed(OUT / "halo.npz", **A)


if __name__ == "__main__":
    which = sys.argv[1:] or ["prng", "geometry", "plans", "kernels", "layers", "halo", "nets"]
    for w in which:
        globals()[f"{w}_fixture"]()
        print("wrote", w)
