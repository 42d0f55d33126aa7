"""Multi-process (world size 2 and 4, gloo, CPU) check of the halo exchange
host logic: dimension-ordered rounds, neighbour pairing and the adjoint.
The device pack/unpack kernels are replaced by torch slicing here; the
frames must equal the reference fabric's results bit for bit (golden)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2007_12856_b200.comm import RankCtx, halo_exchange, reverse_halo_exchange
from paper_2007_12856_b200.geometry import ProcessGrid, Shape5D, make_partition


class CpuFrame:
    """Minimal stand-in for a DistTensor on the CPU (NDHWC frame)."""

    def __init__(self, meta, rank, t):
        self.meta, self.grid_rank, self.t = meta, rank, t
        loc = meta.local_shape(rank)
        self.n, self.c = loc.n, loc.c
        self.m = meta.margins()


def _view(fr, box):
    z0, y0, x0, ez, ey, ex = box
    return fr.t[:, z0:z0 + ez, y0:y0 + ey, x0:x0 + ex, :]


def cpu_pack(fr, box, buf):
    buf.copy_(_view(fr, box).reshape(-1))


def cpu_unpack(fr, box, buf, accumulate):
    v = _view(fr, box)
    if accumulate:
        v += buf.reshape(v.shape)
    else:
        v.copy_(buf.reshape(v.shape))


def _ref_to_device_frame(ref_frame, meta):
    """Reference NCDHW frame (margins in every dim) -> NDHWC device frame
    (margins only in partitioned dims)."""
    fm = meta.margins()
    sl = [slice(None), slice(None)]
    for r, m, e in zip(meta.radii, fm, ref_frame.shape[2:]):
        sl.append(slice(r - m, e - (r - m)))
    return np.ascontiguousarray(ref_frame[tuple(sl)].transpose(0, 2, 3, 4, 1))


def _worker(rank, size, port, key, A, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(size))
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        shape, radii = tuple(A[f"{key}_shape"]), tuple(A[f"{key}_radii"])
        grid = ProcessGrid(*map(int, key.split("x")))
        meta = make_partition(Shape5D(*shape), grid, radii)
        ref_fwd = A[f"{key}_r{rank}_fwd"]
        # start from the reference frame with its margins cleared (interior only)
        dev = _ref_to_device_frame(ref_fwd, meta).astype(np.float64)
        fm = meta.margins()
        start = np.zeros_like(dev)
        loc = meta.local_shape(rank)
        inner = (slice(None), slice(fm[0], fm[0] + loc.d), slice(fm[1], fm[1] + loc.h), slice(fm[2], fm[2] + loc.w))
        start[inner] = dev[inner]
        fr = CpuFrame(meta, rank, torch.from_numpy(start).float())
        ctx = RankCtx(rank, size)
        halo_exchange(ctx, fr, pack=cpu_pack, unpack=cpu_unpack)
        ok_fwd = np.array_equal(fr.t.numpy(), dev.astype(np.float32))
        # adjoint: reference gradient frame restricted to the device frame
        rev_in = A[f"{key}_r{rank}_rev"]
        init = np.arange(rev_in.size, dtype=np.float64).reshape(rev_in.shape) * 0.25 - 3.0
        g0 = _ref_to_device_frame(init, meta)
        gexp = _ref_to_device_frame(rev_in, meta)
        gf = CpuFrame(meta, rank, torch.from_numpy(g0.copy()))
        reverse_halo_exchange(ctx, meta, rank, gf, pack=cpu_pack, unpack=cpu_unpack)
        ok_rev = np.array_equal(gf.t.numpy()[inner], gexp[inner])
        q.put((rank, ok_fwd, ok_rev))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("key", ["1x2x2x1", "1x2x2x2", "1x4x1x1", "2x2x1x1", "1x2x1x1", "1x1x2x1", "1x1x1x2", "2x1x2x1"])
def test_halo_rounds_bit_exact_vs_reference_fabric(golden, key):
    A = dict(np.load(golden / "halo.npz"))
    size = int(np.prod([int(v) for v in key.split("x")]))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, size, port, key, A, q)) for r in range(size)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok_f for _, ok_f, _ in res), res
    assert all(ok_r for _, _, ok_r in res), res
