"""Calibrate the performance model (paper_2007_12856_b200/perfmodel.py) on B200.

1. Communication (run under torchrun on 4 GPUs of one box):
       python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \
           tools/calibrate_perfmodel.py comm --out gpurun_out
   * pingpong.csv  `bytes,seconds`: one fused peer-memory halo round
     (vpx_halo_round_peer) between ranks 0 and 1 over NVLink, one face each
     way; seconds = round time / 2 so the model's 2*SR(b) is the round.
   * allreduce.csv `elements,ranks,seconds`: NCCL all_reduce (fp32 sum) of
     1e3..1e7 elements over 2 and 4 ranks.
   Times are CUDA events around one replay of a CUDA graph holding R
   back-to-back repetitions (after warm-up), max over ranks.

2. Model (CPU): kernel table from bench.py's per-layer CUDA-event breakdown
   at 1/2/4 GPUs (rank 0's local blocks under 1xNx1x1), fits from step 1,
   predicted vs measured step time per GPU count, prediction for 8:
       python tools/calibrate_perfmodel.py model --bench gpurun_out/bench_{1,2,4}gpu.json \
           --comm gpurun_out --out profiles/perfmodel
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

# ------------------------------------------------------------------ comm


def measure_comm(out: Path, reps: int = 50):
    import torch
    import torch.distributed as dist

    from paper_2007_12856_b200 import engine
    from paper_2007_12856_b200.comm import PeerHalo, RankCtx
    from paper_2007_12856_b200.frames import Frame
    from paper_2007_12856_b200.geometry import ProcessGrid
    from paper_2007_12856_b200.networks import build_cosmoflow

    ctx = RankCtx.from_env()
    rank, world = ctx.rank, ctx.size
    if world < 2:
        raise SystemExit("comm calibration needs >= 2 ranks")
    dev = torch.cuda.current_device()

    def timed(fn, n):
        # n calls captured in one CUDA graph (as inside the training step), so
        # the host's per-call cost does not enter the measurement; n is even
        # so the mailbox parities at replay start match the capture's
        for _ in range(4):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            for _ in range(n):
                fn()
        torch.cuda.synchronize()
        dist.barrier()
        g.replay()
        torch.cuda.synchronize()
        dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        g.replay()
        e.record()
        torch.cuda.synchronize()
        t = torch.tensor([s.elapsed_time(e) / n * 1e-3], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- halo-round ping-pong between ranks 0 and 1 (mailboxes of a 1x{world}x1x1 CosmoFlow-512 plan)
    net = build_cosmoflow(512)
    plan = engine.make_plan(net, ProcessGrid(1, world, 1, 1), 1, 512)
    peer = PeerHalo(ctx, plan)
    rows = []
    for c, h, w in [(4, 16, 16), (4, 32, 32), (4, 64, 64), (4, 128, 128), (4, 256, 256), (16, 128, 256),
                    (4, 512, 512), (16, 256, 256)]:
        nbytes = c * h * w * 4
        if nbytes > peer.slab:
            continue
        fr = Frame(1, c, 1, h, w, (1, 0, 0), zero=True)
        fr.interior.normal_()
        side = 1 if rank == 0 else -1
        send = (1, 0, 0, 1, h, w)
        recv = (2, 0, 0, 1, h, w) if side == 1 else (0, 0, 0, 1, h, w)

        def one():
            if rank < 2:
                peer.round(0, [side], fr, [send], [recv], 1)

        t = timed(one, reps)
        rows.append((nbytes, t / 2))
        if rank == 0:
            print(f"[calib] halo round {nbytes} B: {t * 1e6:.2f} us", flush=True)
    # ---- NCCL all-reduce over 2 and 4 ranks
    groups = {p: dist.new_group(list(range(p))) for p in (2, 4) if p <= world}
    ar = []
    for p, g in groups.items():
        for m in (1_000, 10_000, 100_000, 1_000_000, 10_000_000):
            buf = torch.ones(m, dtype=torch.float32, device=dev)

            def one():
                if rank < p:
                    dist.all_reduce(buf, group=g)

            t = timed(one, 20)
            ar.append((m, p, t))
            if rank == 0:
                print(f"[calib] allreduce {m} x fp32 over {p}: {t * 1e6:.1f} us", flush=True)
    if rank == 0:
        out.mkdir(parents=True, exist_ok=True)
        (out / "pingpong.csv").write_text("bytes,seconds\n" + "".join(f"{b},{t!r}\n" for b, t in rows))
        (out / "allreduce.csv").write_text("elements,ranks,seconds\n" + "".join(f"{m},{p},{t!r}\n" for m, p, t in ar))
    dist.barrier()


# ------------------------------------------------------------------ model

# bench.py region tag suffix -> model phase
_PHASE = {"fwd": "fwd", "dgrad": "bwd_data", "wgrad": "bwd_filter", "bwd": "bwd_data"}
_TINY = 1e-9  # a phase fused into another kernel: the table needs a positive entry


def kernel_rows(net, w: int, parts: int, bench: dict):
    """(kind, phase, local out shape, seconds, source) rows from one bench line."""
    from paper_2007_12856_b200 import perfmodel as pm

    geos = {g.name: g for g in pm.network_geometry(net, w, 1, (parts, 1, 1))}
    names = [l.name for l in net.layers]
    kern = bench["kernels"]
    rows = []
    for name, g in geos.items():
        if min(g.out_local) < 1:
            continue  # block smaller than the partition (the planner gathers these layers to the lead)
        i = names.index(name)
        for phase in ("fwd", "bwd_data", "bwd_filter"):
            if g.kind == "pool" and phase == "bwd_filter":
                continue
            secs, src = 0.0, []
            for tag, v in kern.items():
                layer, _, suffix = tag.rpartition(".")
                if _PHASE.get(suffix) != phase:
                    continue
                if layer == name:
                    secs += v["ms_per_step"] * 1e-3
                    src.append(tag)
                elif g.kind == "pool" and layer == names[i - 1] and net.layers[i - 1].kind == "leaky" \
                        and suffix == "bwd":
                    secs += v["ms_per_step"] * 1e-3  # fused LeakyReLU + pool backward (one kernel)
                    src.append(tag)
            if secs <= 0:
                secs, src = _TINY, ["fused into the neighbouring conv kernel"]
            rows.append((g.kind, phase, g.out_local, secs, "+".join(src)))
            if g.main_local != g.out_local and min(g.main_local) > 0:
                # the halo-free interior, in proportion to its voxels, so the
                # model's Comp(D_main) lookup is an exact hit on this layer
                import math
                share = math.prod(g.main_local) / math.prod(g.out_local)
                rows.append((g.kind, phase, g.main_local, max(secs * share, _TINY), f"interior share of {name}"))
                # and the boundary shell (the model looks it up by voxel count)
                shell = g.out_local[:2] + (g.out_local[2] - g.main_local[2],) + g.out_local[3:]
                rows.append((g.kind, phase, shell, max(secs * (1 - share), _TINY), f"interior share of {name} (shell)"))
    return rows


def model(bench_paths, comm_dir: Path, out: Path, width: int = 512):
    from paper_2007_12856_b200 import perfmodel as pm
    from paper_2007_12856_b200.geometry import ProcessGrid
    from paper_2007_12856_b200.networks import build_cosmoflow

    net = build_cosmoflow(width)
    measured = {}
    table = pm.KernelTimeTable()
    sources = []
    for p in bench_paths:
        line = json.loads(Path(p).read_text().strip().splitlines()[-1])
        n = line["n_gpus"]
        measured[n] = line["ms_per_step"] * 1e-3
        for kind, phase, shape, secs, src in kernel_rows(net, width, n, line):
            if table.exact(kind, phase, shape) is None:
                table.add_row(kind, phase, shape, secs)
                sources.append((kind, phase, shape, secs, src))
    # 8-way rows (no 8-GPU box here): each layer/phase's 4-way time times its
    # own measured 2 -> 4 ratio (clamped to [0.5, 1]), so latency-bound layers
    # stop shrinking while bandwidth/compute-bound ones keep halving
    per = {}
    for kind, phase, shape, secs, src in sources:
        if src.startswith("interior"):
            continue
        per.setdefault((kind, phase, shape[1], shape[3], shape[4]), {})[shape[2]] = (secs, src, shape)
    for (kind, phase, c, h, w), by_d in per.items():
        ds = sorted(by_d)
        if len(ds) < 3 or ds[0] * 4 != ds[-1]:
            continue
        (t4, src4, s4), (t2, _, _) = by_d[ds[0]], by_d[ds[1]]
        if s4[2] % 2:
            continue
        ratio = 1.0 if src4.startswith("fused") else min(1.0, max(0.5, t4 / t2))
        s8 = (s4[0], c, s4[2] // 2, h, w)
        t8 = t4 * ratio
        extra = [(s8, t8)]
        if kind == "conv" and s8[2] > 2:
            # depth split, radius 1, stride 1 layers: one boundary plane per side
            extra += [((s8[0], c, s8[2] - 2, h, w), t8 * (s8[2] - 2) / s8[2]), ((s8[0], c, 2, h, w), t8 * 2 / s8[2])]
        for shp, t in extra:
            if table.exact(kind, phase, shp) is None:
                table.add_row(kind, phase, shp, max(t, _TINY))
                sources.append((kind, phase, shp, max(t, _TINY), f"extrapolated: 4-way x {ratio:.2f} (2->4 ratio)"))
    link = pm.fit_link(pm.load_pingpong(comm_dir / "pingpong.csv"))
    coll = pm.fit_allreduce(pm.load_allreduce(comm_dir / "allreduce.csv"))
    out.mkdir(parents=True, exist_ok=True)
    pm.write_kernel_table(out / "kernel_table.csv", table)
    for f in ("pingpong.csv", "allreduce.csv"):
        (out / f).write_text((comm_dir / f).read_text())
    lines = ["# Performance model calibrated on B200 (CosmoFlow 512^3, batch 1, 1xNx1x1)", "",
             "Model: reference perfmodel.py restated in `paper_2007_12856_b200/perfmodel.py` (cost reports "
             "bit-identical to the reference's, `tests/test_perfmodel.py`).  Inputs measured here:",
             "", f"* kernel table `kernel_table.csv` ({len(table)} rows): per-layer CUDA-event times of "
             "bench.py's eager pass at 1/2/4 GPUs (rank 0's local block), phases fused into one kernel "
             f"carry {_TINY:g} s;",
             f"* link fit from `pingpong.csv` (fused peer-memory halo round over NVLink): alpha = "
             f"{link.alpha * 1e6:.2f} us, beta = {link.beta * 1e12:.3f} ps/B ({1 / link.beta / 1e9 if link.beta else 0:.0f} GB/s);",
             f"* all-reduce fit from `allreduce.csv` (NCCL, 2 and 4 ranks): c0 = {coll.c0:.3f}, c1 = {coll.c1:.3f}, "
             f"c2 = {coll.c2:.3f}, rms log residual {coll.residual:.3f}.", "",
             "| GPUs | grid | predicted ms/step | measured ms/step (bench.py, graph replay) | predicted / measured | "
             "predicted samples/s |", "|---|---|---|---|---|---|"]
    preds = {}
    for n in (1, 2, 4, 8):
        grid = ProcessGrid(1, n, 1, 1)
        bd = pm.total_cost(net, width, grid, 1, table, link, coll)
        preds[n] = bd
        meas = measured.get(n)
        lines.append(f"| {n} | 1x{n}x1x1 | {bd.total * 1e3:.3f} | "
                     f"{'%.3f' % (meas * 1e3) if meas else '—'} | "
                     f"{'%.2f' % (bd.total / meas) if meas else '—'} | {1 / bd.total:.1f} |")
        (out / f"report_1x{n}x1x1.csv").write_text(bd.report() + "\n")
    base = preds[1].total
    gaps = {n: measured[n] / preds[n].total for n in measured if n > 1}
    if gaps:
        worst = max(gaps.items(), key=lambda kv: kv[1])
        lines += ["", f"The model leaves out what it does not cost (flatten/fc/dropout/loss/Adam, redistribution, "
                  f"neighbour-to-neighbour skew at every halo round): measured/predicted is "
                  + ", ".join(f"{v:.2f} at {n} GPUs" for n, v in sorted(gaps.items()))
                  + f"; applying the {worst[0]}-GPU factor to the 8-GPU prediction gives "
                  f"{preds[8].total * worst[1] * 1e3:.2f} ms/step "
                  f"({base / (8 * preds[8].total * worst[1]) * 100:.0f}% of ideal vs the model's 1-GPU time)."]
    lines += ["", "Predicted strong-scaling efficiency vs 1 GPU: " +
              ", ".join(f"{n} GPUs {base / (n * preds[n].total) * 100:.0f}%" for n in (2, 4, 8)) + ".",
              "8-GPU kernel rows are extrapolated per layer from the measured 2 -> 4 GPU ratio (no 8-GPU box "
              "was available to this calibration); interior/shell splits are the model's own voxel-count "
              "interpolation (notes in `report_1x8x1x1.csv`).", "",
              "Kernel-table sources (bench.py region tags summed per row):", "",
              "| kind | phase | local out shape | seconds | from |", "|---|---|---|---|---|"]
    lines += [f"| {k} | {ph} | {s} | {v:.3e} | {src} |" for k, ph, s, v, src in sources]
    (out / "calibration.md").write_text("\n".join(lines) + "\n")
    print("\n".join(lines[:20]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["comm", "model"])
    ap.add_argument("--out", default="gpurun_out")
    ap.add_argument("--bench", nargs="*", default=[])
    ap.add_argument("--comm", default="gpurun_out")
    ap.add_argument("--width", type=int, default=512)
    a = ap.parse_args()
    if a.mode == "comm":
        measure_comm(Path(a.out))
    else:
        model(a.bench, Path(a.comm), Path(a.out), a.width)


if __name__ == "__main__":
    main()
