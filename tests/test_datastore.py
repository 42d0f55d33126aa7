"""Datastore (HSB1 files, schedules, owner map, distributed cache) against
golden vectors written by the reference itself (tests/golden/
make_datastore_golden.py, reference datastore.py); CPU only except the
device materialisation test."""

import json
import os
import socket
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2007_12856_b200 import datastore as D
from paper_2007_12856_b200 import prng
from paper_2007_12856_b200.errors import BadBatch, BadMagic, BadVersion, CacheNotEmpty, IoError, MissingSample
from paper_2007_12856_b200.geometry import ProcessGrid, Region, hyperslab_byte_ranges

GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def golden():
    return json.loads((GOLD / "datastore.json").read_text())


def test_schedule_owner_map_fixture_match_reference(golden):
    for k, perm in golden["perm"].items():
        s, e, t = (int(v) for v in k.split(","))
        assert list(D.epoch_schedule(s, e, t, 2, 1).perm) == perm
    man = D.load_manifest(GOLD / "ds_fixture" / "mse" / "manifest.json")
    sched = D.epoch_schedule(0, 0, 8, 4, 2)
    owners = D.build_owner_map(man, ProcessGrid(2, 1, 1, 1), sched)
    assert {str(k): v for k, v in owners.items()} == golden["owner_map_8_4_2"]
    assert np.array_equal(man.targets(), np.array(golden["targets"]))
    vox = D._fixture_voxels(7, 3, (2, 3, 4, 5))
    assert vox.dtype == np.int16 and vox.reshape(-1).tolist() == golden["fixture_7_3"]
    # files written by the reference read back bit-identically, targets recomputed
    for sid in range(man.size):
        pay = D.read_payload(man.path(sid))
        assert np.array_equal(pay, D._fixture_voxels(5, sid, (2, 4, 6, 8)))
        assert np.allclose(D.fixture_target(pay), man.samples[sid].target, rtol=0, atol=0)


def test_hsb1_round_trip_and_errors(tmp_path):
    v = np.arange(2 * 3 * 4 * 5, dtype=np.float32).reshape(2, 3, 4, 5) - 7.5
    p = tmp_path / "a.hsb"
    D.write_sample(p, v.shape, "fp32", v)
    hdr = D.read_header(p)
    assert hdr.dims == (2, 3, 4, 5) and hdr.dtype_name == "fp32" and hdr.payload_bytes == v.nbytes
    assert np.array_equal(D.read_payload(p), v)
    raw = bytearray(p.read_bytes())
    bad = tmp_path / "bad.hsb"
    bad.write_bytes(b"XSB1" + raw[4:])
    with pytest.raises(BadMagic):
        D.read_header(bad)
    bad.write_bytes(raw[:4] + bytes([2]) + raw[5:])
    with pytest.raises(BadVersion):
        D.read_header(bad)
    bad.write_bytes(raw[:-4])
    with pytest.raises(IoError):
        D.read_header(bad)
    with pytest.raises(IoError):
        D.write_sample(tmp_path / "c.hsb", v.shape, "bf16", v)
    with pytest.raises(IoError):
        D.read_header(tmp_path / "missing.hsb")


def test_hyperslab_reads_exact_region_and_counts_bytes(tmp_path):
    rng = np.random.default_rng(0)
    v = rng.integers(-8, 9, (3, 8, 6, 10)).astype(np.int16)
    p = tmp_path / "s.hsb"
    D.write_sample(p, v.shape, "int16", v)
    for reg in (Region((2, 0, 0), (4, 6, 10)), Region((0, 3, 2), (8, 3, 5)), Region((5, 1, 7), (3, 2, 3))):
        c = D.IoCounters()
        got = D.read_hyperslab(p, reg, c, epoch=1)
        (od, oh, ow), (ed, eh, ew) = reg.offset, reg.extent
        assert np.array_equal(got, v[:, od:od + ed, oh:oh + eh, ow:ow + ew])
        assert c.file_bytes_read == sum(n for _, n in hyperslab_byte_ranges(v.shape, reg, 2))
        assert c.epoch_file_bytes(1) == c.file_bytes_read and c.file_opens == 1
        dst = torch.empty(got.shape, dtype=torch.int16)
        D.read_hyperslab(p, reg, out=dst)
        assert np.array_equal(dst.numpy(), got)


def test_schedule_and_store_errors(tmp_path):
    with pytest.raises(BadBatch):
        D.epoch_schedule(0, 0, 10, 3, 2)
    with pytest.raises(BadBatch):
        D.epoch_schedule(0, 0, 3, 4, 1)
    man = D.load_manifest(GOLD / "ds_fixture" / "mse" / "manifest.json")
    with pytest.raises(BadBatch):
        D.build_owner_map(man, ProcessGrid(1, 1, 1, 1), D.epoch_schedule(0, 0, 8, 4, 2))
    st = D.DataStore(man, ProcessGrid(2, 2, 1, 1), 1, pin=False)
    with pytest.raises(MissingSample):
        D.exchange_for_iteration(None, st, D.epoch_schedule(0, 1, 8, 4, 2), 0, device=False)
    D.ingest_epoch0(st, D.epoch_schedule(0, 0, 8, 4, 2))
    with pytest.raises(CacheNotEmpty):
        D.ingest_epoch0(st, D.epoch_schedule(0, 0, 8, 4, 2))
    (tmp_path / "m.json").write_text('{"format": "other"}')
    with pytest.raises(IoError):
        D.load_manifest(tmp_path / "m.json")


def _exchange_worker(rank, size, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(size))
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        man = D.load_manifest(GOLD / "ds_fixture" / "mse" / "manifest.json")
        grid = ProcessGrid(2, 1, 1, 1)
        st = D.DataStore(man, grid, rank, pin=False)
        D.ingest_epoch0(st, D.epoch_schedule(0, 0, 8, 4, 2))
        res = {"epoch0_bytes": st.counters.epoch_file_bytes(0), "owned": sorted(st.cache)}
        sched = D.epoch_schedule(0, 1, 8, 4, 2)
        got = []
        for it in range(sched.iterations):
            dl = D.exchange_for_iteration(None, st, sched, it, device=False)
            for sid, blk, _ in dl:
                got.append((sid, bool(np.array_equal(blk.numpy(), D.read_payload(man.path(sid))))))
            x, t, _ = D.materialize_batch(st, dl)
            res.setdefault("x_ok", True)
            ref = np.stack([D.read_payload(man.path(s)) for s, _, _ in dl]).astype(np.float32)
            res["x_ok"] &= bool(np.array_equal(x, ref)) and t.shape == (2, 4)
        res["got"] = got
        res["exchange"] = st.counters.exchange_bytes
        # the narrowed exchange (agreed int8 transfer dtype) delivers the same values
        import torch

        res["agreed"] = str(st.agree_transfer_dtype())
        res["narrow_ok"] = True
        for it in range(sched.iterations):
            dl = D.exchange_for_iteration(None, st, sched, it, device=False, narrow=True)
            x, t, _ = D.materialize_batch(st, dl)
            ref = np.stack([D.read_payload(man.path(s)) for s, _, _ in dl]).astype(np.float32)
            res["narrow_ok"] &= bool(np.array_equal(x, ref)) and all(b.dtype == torch.int8 for _, b, _ in dl)
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_two_group_exchange_gloo():
    """2 data-parallel groups: epoch 0 reads every payload byte once across
    ranks; epoch 1 ships the slabs a group does not own (reference
    datastore.py:384-426)."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_exchange_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    man = D.load_manifest(GOLD / "ds_fixture" / "mse" / "manifest.json")
    total = sum(D.read_header(man.path(i)).payload_bytes for i in range(man.size))
    assert res[0]["epoch0_bytes"] + res[1]["epoch0_bytes"] == total
    assert sorted(res[0]["owned"] + res[1]["owned"]) == list(range(8))
    sched = D.epoch_schedule(0, 1, 8, 4, 2)
    for r in (0, 1):
        want = [sid for it in range(sched.iterations) for sid in sched.group_samples(it, r)]
        assert [sid for sid, _ in res[r]["got"]] == want
        assert all(ok for _, ok in res[r]["got"]) and res[r]["x_ok"]
    assert res[0]["exchange"] + res[1]["exchange"] > 0
    assert res[0]["agreed"] == res[1]["agreed"] == "torch.int8"  # the fixture range [-8, 8] fits int8
    assert res[0]["narrow_ok"] and res[1]["narrow_ok"]


@pytest.mark.gpu
def test_materialize_into_device_frame_and_labels():
    from paper_2007_12856_b200.frames import DistTensor
    from paper_2007_12856_b200.geometry import Shape5D, make_partition

    man = D.load_manifest(GOLD / "ds_fixture" / "xent" / "manifest.json")
    grid = ProcessGrid(1, 1, 1, 1)
    st = D.DataStore(man, grid, 0)
    D.ingest_epoch0(st, D.epoch_schedule(0, 0, 2, 2, 1))
    dl = D.exchange_for_iteration(None, st, D.epoch_schedule(0, 0, 2, 2, 1), 0, device=False)
    meta = make_partition(Shape5D(2, 1, 4, 4, 4), grid, (1, 1, 1))
    xb = DistTensor(meta, 0, zero=True)
    x, t, lab = D.materialize_batch(st, dl, x_block=xb)
    ref_x = np.stack([D.read_payload(man.path(s)) for s, _, _ in dl]).astype(np.float32)
    assert np.array_equal(x.to_ncdhw().cpu().numpy(), ref_x)
    ref_l = np.stack([D.read_payload(man.label_path(s)) for s, _, _ in dl])[:, 0].astype(np.int64)
    assert lab.dtype == torch.int64 and np.array_equal(lab.cpu().numpy(), ref_l)


def _two_sample_store(tmp_path, vals):
    from paper_2007_12856_b200 import datastore as DS
    from paper_2007_12856_b200.geometry import ProcessGrid

    dims = (1, 4, 4, 4)
    entries = []
    for sid, v in vals.items():
        DS.write_sample(tmp_path / f"s{sid}.hsb", dims, "int16", v.reshape(dims))
        entries.append(DS.SampleEntry(sid, f"s{sid}.hsb", target=(0.0, 0.0, 0.0, 0.0)))
    man = DS.Manifest(root=str(tmp_path), dtype="int16", dims=dims, loss="mse", samples=tuple(entries))
    store = DS.DataStore(man, ProcessGrid(1, 1, 1, 1), 0, pin=False)
    DS.ingest_epoch0(store, DS.epoch_schedule(0, 0, len(vals), len(vals), 1))
    return store


def test_transfer_block_narrows_losslessly(tmp_path):
    """DataStore.transfer_block: an int8 copy (same values) when every cached
    int16 voxel of the store fits int8; forcing int16 returns the cache."""
    import torch

    vals = {0: np.arange(64, dtype=np.int16) - 8, 1: np.arange(64, dtype=np.int16) - 127}
    store = _two_sample_store(tmp_path, vals)
    assert store.transfer_dtype() == torch.int8
    t0, t1 = store.transfer_block(0), store.transfer_block(1)
    for sid, t in ((0, t0), (1, t1)):
        assert t.dtype == torch.int8 and np.array_equal(t.numpy().astype(np.int16).ravel(), vals[sid])
    assert store.transfer_block(0) is t0  # made once
    assert store.transfer_block(0, dtype=torch.int16).dtype == torch.int16


def test_transfer_dtype_is_one_decision_per_dataset(tmp_path):
    """Regression (advisor r1): sample 0 fits int8, sample 1 does not.  Every
    block must then travel as int16 -- a per-sample choice would stage sample
    0 as int8 and wrap sample 1's voxels in the same staging buffer."""
    import torch

    from paper_2007_12856_b200.errors import ShapeMismatch

    vals = {0: np.arange(64, dtype=np.int16) - 8, 1: np.full(64, 300, dtype=np.int16)}
    store = _two_sample_store(tmp_path, vals)
    assert store.transfer_dtype() == torch.int16
    assert store.transfer_block(0).dtype == store.transfer_block(1).dtype == torch.int16
    with pytest.raises(ShapeMismatch):
        store.transfer_block(0, dtype=torch.int8)
