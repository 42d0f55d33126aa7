"""Golden outputs of the reference performance model (run here, where the
reference exists):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_perfmodel_golden.py
Writes tests/golden/perfmodel.json: cost reports (exact float reprs) for a
few network / partition / table / link / collective combinations, comp_time
lookups and fits, all computed by reference perfmodel.py itself."""
import json
import math
from pathlib import Path

from voxpar import perfmodel as pm
from voxpar.model.networks import build_cosmoflow, build_unet_mini
from voxpar.tensor import ProcessGrid

here = Path(__file__).resolve().parent
COLL_PTS = [(m, p, 2e-6 * m ** 0.8 * p ** 0.35 + 1e-5) for m in (1e3, 1e5, 1e7) for p in (2, 4, 8)]
LINK_PTS = [(4096, 9.1e-6), (1 << 20, 1.3e-5), (4 << 20, 2.2e-5), (16 << 20, 5.0e-5)]

CASES = [
    # name, net, w_i, grid, n_global, table kind, table parts
    ("cosmo128_1x2", ("cosmoflow", 128, False), (1, 2, 1, 1), 2, "flop", [(1, 1, 1), (2, 1, 1)]),
    ("cosmo512_1x8_extrap", ("cosmoflow", 512, False), (1, 8, 1, 1), 1, "ideal", [(1, 1, 1)]),
    ("cosmo64bn_2x2x2x1", ("cosmoflow", 64, True), (2, 2, 2, 1), 4, "flop", [(2, 2, 1)]),
    ("unet64_1x2x2x1", ("unet", 64, False), (1, 2, 2, 1), 2, "ideal", [(2, 2, 1), (1, 1, 1)]),
]


def build(spec):
    kind, w, bn = spec
    return build_cosmoflow(w, with_bn=bn) if kind == "cosmoflow" else build_unet_mini(w)


def main():
    out = {"link_pts": LINK_PTS, "coll_pts": COLL_PTS}
    link = pm.fit_link(LINK_PTS)
    coll = pm.fit_allreduce(COLL_PTS)
    out["link"] = [link.alpha, link.beta]
    out["coll"] = [coll.c0, coll.c1, coll.c2, coll.residual]
    out["cases"] = {}
    for name, spec, g, n, kind, parts in CASES:
        net = build(spec)
        grid = ProcessGrid(*g)
        nl = n // grid.groups
        if kind == "flop":
            table = pm.flop_proportional_table(net, spec[1], nl, parts, 1e-12, 2.0)
        else:
            table = pm.ideal_table(net, spec[1], nl, parts)
        bd = pm.total_cost(net, spec[1], grid, n, table, link, coll)
        out["cases"][name] = {"report": bd.report(), "total": bd.total, "rows": len(table)}
    # comp_time: exact hits, interpolation, both extrapolations, raw voxel counts
    t = pm.KernelTimeTable()
    for shape, secs in [((1, 4, 2, 2, 2), 1e-6), ((1, 4, 4, 4, 4), 3e-6), ((1, 4, 8, 8, 8), 1.7e-5),
                        ((2, 4, 4, 4, 4), 5e-6)]:
        t.add_row("conv", "fwd", shape, secs)
    out["comp_time"] = {str(d): list(pm.comp_time(t, "conv", "fwd", d))
                        for d in [(1, 4, 4, 4, 4), (1, 1, 16, 16, 2), 100, 300, 1, 5000, 512, 256, 32]}
    (here / "perfmodel.json").write_text(json.dumps(out))
    print("wrote", here / "perfmodel.json", math.fsum(c["total"] for c in out["cases"].values()))


if __name__ == "__main__":
    main()
