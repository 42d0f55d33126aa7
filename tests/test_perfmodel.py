"""Performance model (CPU): the reference's own known-answer checks for the
fits and lookups (reference tests/test_perfmodel.py), plus golden cost
reports written by the reference model itself (tests/golden/
make_perfmodel_golden.py) compared as exact text -- every float repr equal."""

import json
import math
from pathlib import Path

import pytest

from paper_2007_12856_b200 import perfmodel as pm
from paper_2007_12856_b200.errors import ConfigError, DegenerateFit, InsufficientData, NoComparableEntry
from paper_2007_12856_b200.geometry import ProcessGrid
from paper_2007_12856_b200.networks import build_cosmoflow, build_unet_mini

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "perfmodel.json").read_text())


def test_fit_link_two_points_exact():
    link = pm.fit_link([(2048, 1.5e-5), (1048576, 5.125e-3)])
    assert abs(link.alpha - 5e-6) <= 1e-18 and abs(link.beta - 4.8828125e-9) <= 1e-21
    assert abs(link.sr(2048) - 1.5e-5) <= 1e-18


def test_fit_errors():
    with pytest.raises(InsufficientData):
        pm.fit_link([(1024, 1e-5)])
    with pytest.raises(DegenerateFit):
        pm.fit_link([(1024, 1e-5), (1024, 2e-5)])
    with pytest.raises(DegenerateFit):
        pm.fit_link([(1024, 2e-5), (2048, 1e-5)])
    with pytest.raises(InsufficientData):
        pm.fit_allreduce([(10, 2, 1e-3), (20, 2, 2e-3)])
    with pytest.raises(DegenerateFit):
        pm.fit_allreduce([(10, 2, 1e-3), (10, 2, 2e-3), (10, 2, 3e-3)])
    with pytest.raises(DegenerateFit):
        pm.fit_allreduce([(10, 2, -1e-3), (20, 4, 2e-3), (30, 8, 3e-3)])


def test_fit_allreduce_recovers_powerlaw():
    c0, c1, c2 = 2.0, 0.9, 0.3
    pts = [(m, p, math.exp(c0 + c1 * math.log(m) + c2 * math.log(p))) for m in (1e3, 1e4, 1e5) for p in (2, 4, 8)]
    coll = pm.fit_allreduce(pts)
    assert max(abs(coll.c0 - c0), abs(coll.c1 - c1), abs(coll.c2 - c2)) <= 1e-6 and coll.residual <= 1e-9
    assert coll.time(100, 1) == 0.0 and coll.time(0, 8) == 0.0


def test_fits_match_reference():
    link = pm.fit_link(GOLD["link_pts"])
    coll = pm.fit_allreduce(GOLD["coll_pts"])
    assert [link.alpha, link.beta] == pytest.approx(GOLD["link"], rel=1e-12, abs=1e-24)
    assert [coll.c0, coll.c1, coll.c2, coll.residual] == pytest.approx(GOLD["coll"], rel=1e-10, abs=1e-14)


def test_comp_time_matches_reference():
    t = pm.KernelTimeTable()
    for shape, secs in [((1, 4, 2, 2, 2), 1e-6), ((1, 4, 4, 4, 4), 3e-6), ((1, 4, 8, 8, 8), 1.7e-5),
                        ((2, 4, 4, 4, 4), 5e-6)]:
        t.add_row("conv", "fwd", shape, secs)
    for key, want in GOLD["comp_time"].items():
        d = eval(key)  # noqa: S307 - golden keys are tuples/ints written by the generator
        assert list(pm.comp_time(t, "conv", "fwd", d)) == want, key
    with pytest.raises(NoComparableEntry):
        pm.comp_time(t, "pool", "fwd", (1, 1, 1, 1, 1))
    assert pm.comp_time(t, "conv", "fwd", 0) == (0.0, None)


def test_kernel_table_parse_errors_and_round_trip(tmp_path):
    with pytest.raises(ConfigError):
        pm.parse_kernel_table(["kind,phase,n,c,d,h,w"])
    with pytest.raises(ConfigError):
        pm.parse_kernel_table([pm.TABLE_COLUMNS, "conv,sideways,1,1,1,1,1,1e-3"])
    with pytest.raises(ConfigError):
        pm.parse_kernel_table([pm.TABLE_COLUMNS, "conv,fwd,1,1,1,1,1,0"])
    with pytest.raises(ConfigError):
        pm.parse_kernel_table([pm.TABLE_COLUMNS, "conv,fwd,1,1,1,1,1,1e-3", "conv,fwd,1,1,1,1,1,2e-3"])
    t = pm.flop_proportional_table(build_cosmoflow(64), 64, 1, [(1, 1, 1), (2, 1, 1)])
    p = tmp_path / "t.csv"
    pm.write_kernel_table(p, t)
    t2 = pm.parse_kernel_table(str(p))
    assert t2.rows() == t.rows() and len(t2) == len(t)


def _net(spec):
    kind, w, bn = spec
    return build_cosmoflow(w, with_bn=bn) if kind == "cosmoflow" else build_unet_mini(w)


CASES = {
    "cosmo128_1x2": (("cosmoflow", 128, False), (1, 2, 1, 1), 2, "flop", [(1, 1, 1), (2, 1, 1)]),
    "cosmo512_1x8_extrap": (("cosmoflow", 512, False), (1, 8, 1, 1), 1, "ideal", [(1, 1, 1)]),
    "cosmo64bn_2x2x2x1": (("cosmoflow", 64, True), (2, 2, 2, 1), 4, "flop", [(2, 2, 1)]),
    "unet64_1x2x2x1": (("unet", 64, False), (1, 2, 2, 1), 2, "ideal", [(2, 2, 1), (1, 1, 1)]),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_cost_report_equals_reference(name):
    spec, g, n, kind, parts = CASES[name]
    net, grid = _net(spec), ProcessGrid(*g)
    nl = n // grid.groups
    table = (pm.flop_proportional_table(net, spec[1], nl, parts, 1e-12, 2.0) if kind == "flop"
             else pm.ideal_table(net, spec[1], nl, parts))
    link, coll = pm.fit_link(GOLD["link_pts"]), pm.fit_allreduce(GOLD["coll_pts"])
    bd = pm.total_cost(net, spec[1], grid, n, table, link, coll)
    want = GOLD["cases"][name]
    assert len(table) == want["rows"]
    assert bd.report() == want["report"]
    assert bd.total == want["total"]


def test_fp_structure():
    """FP = max(main, 2 SR) + shell: compute-bound and link-bound regimes, and
    an unpartitioned layer is pure compute."""
    net = build_cosmoflow(64)
    table = pm.ideal_table(net, 64, 1, [(2, 1, 1), (1, 1, 1)])
    geo = [g for g in pm.network_geometry(net, 64, 1, (2, 1, 1)) if g.name == "c2"][0]
    main, _ = pm.comp_time(table, "conv", "fwd", geo.main_local)
    shell, _ = pm.comp_time(table, "conv", "fwd", geo.halo_voxels)
    slow = pm.LinkModel(1.0, 0.0)
    assert pm.layer_fp_cost(table, geo, pm.ZERO_LINK, pm.ZERO_COLLECTIVE, 2) == main + shell
    assert pm.layer_fp_cost(table, geo, slow, pm.ZERO_COLLECTIVE, 2) == 2.0 + shell
    geo1 = [g for g in pm.network_geometry(net, 64, 1, (1, 1, 1)) if g.name == "c2"][0]
    assert geo1.sr_bytes == (0, 0, 0) and geo1.halo_voxels == 0
