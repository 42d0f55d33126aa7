"""Inter-GPU communication for the hybrid-parallel step (one process per GPU).

Replaces the reference's simulated message fabric (reference
pkg/src/voxpar/fabric.py: threads + per-(src,dst,tag) deques + a binomial
tree allreduce) with torch.distributed over NCCL on NVLink/NVSwitch:

* ``RankCtx`` keeps the reference's per-rank handle API (rank, send, recv,
  allreduce_sum; reference fabric.py:111-128), backed by NCCL P2P and
  all-reduce on device tensors.
* ``halo_exchange`` / ``reverse_halo_exchange`` follow the reference's
  dimension-ordered rounds (reference fabric.py:380-443, tensor.py:354-385):
  ascending dims forward, descending dims for the adjoint, each round's slab
  spanning the margins already exchanged so edges and corners propagate.
  Slabs are packed/unpacked by vpx_halo_copy and both faces of a round go in
  one NCCL group (batch_isend_irecv).  Contents are bit-exact (pure copies);
  the only difference from the reference is that unpartitioned dims carry no
  zero margins in the messages (frames.py), so payloads are smaller.
* Reductions are NCCL sums, so reduced values are tolerance-equal, not
  bit-equal, to the reference's binomial tree.

World size 1 needs no process group: every collective is the identity.
The host-side geometry is exercised on CPU with the gloo backend
(tests/test_comm_gloo.py), where pack/unpack are torch slicing callables.
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist

from . import _lib
from .errors import OutOfBounds
from .geometry import round_boxes
from .timing import region


class RankCtx:
    """Per-process handle (reference fabric.py:111-128 API)."""

    def __init__(self, rank: int = 0, size: int = 1, device=None):
        self.rank = rank
        self.size = size
        self.device = device
        self._groups = {}
        self._bufs = {}

    # -------------------------------------------------------------- setup
    @classmethod
    def from_env(cls, backend: str = None):
        """Initialise from torchrun's env (RANK/WORLD_SIZE/LOCAL_RANK/MASTER_*)."""
        size = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        if size > 1 and not dist.is_initialized():
            local = int(os.environ.get("LOCAL_RANK", rank))
            if backend is None:
                backend = "nccl" if torch.cuda.is_available() else "gloo"
            if backend == "nccl":
                torch.cuda.set_device(local)
                dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            else:
                dist.init_process_group(backend)
        dev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else None
        return cls(rank, size, dev)

    def group(self, members):
        """Process group for a sorted member tuple; None = world.  Creation is
        collective over the world: call prepare_groups() in the same order on
        every rank before use."""
        members = tuple(sorted(members))
        if self.size == 1 or len(members) == self.size:
            return None
        if members not in self._groups:
            self._groups[members] = dist.new_group(list(members))
        return self._groups[members]

    def prepare_groups(self, member_sets):
        for m in member_sets:
            self.group(m)

    # ------------------------------------------------------------- p2p
    def send(self, dst: int, tag: int, tensor: torch.Tensor):
        if dst == self.rank:
            raise OutOfBounds("send to self")
        dist.send(tensor.contiguous(), dst)

    def recv(self, src: int, tag: int, like: torch.Tensor) -> torch.Tensor:
        dist.recv(like, src)
        return like

    def exchange(self, ops):
        """ops: list of ("send"|"recv", peer, tensor); one NCCL group."""
        if not ops:
            return
        p2p = [dist.P2POp(dist.isend if kind == "send" else dist.irecv, t, peer)
               for kind, peer, t in ops]
        nbytes = sum(4 * t.numel() for kind, _, t in ops if kind == "send")
        with region("comm.p2p", 0, nbytes):
            for req in dist.batch_isend_irecv(p2p):
                req.wait()

    # ------------------------------------------------------- collectives
    def allreduce_sum_(self, tensor: torch.Tensor, members=None) -> torch.Tensor:
        """In-place sum over `members` (default all ranks)."""
        if self.size == 1:
            return tensor
        if members is not None and self.rank not in members:
            raise OutOfBounds(f"rank {self.rank} not in allreduce group {sorted(members)}")
        if members is not None and len(members) == 1:
            return tensor
        tag = "comm.allreduce_grad" if tensor.numel() > 65536 else "comm.allreduce_small"
        with region(tag, 0, tensor.numel() * tensor.element_size()):
            dist.all_reduce(tensor, op=dist.ReduceOp.SUM, group=self.group(members or range(self.size)))
        return tensor

    def allreduce_sum(self, vec, group=None):
        """Reference-style (returns the reduced vector; reference fabric.py:274-312)."""
        t = vec if isinstance(vec, torch.Tensor) else torch.as_tensor(vec)
        return self.allreduce_sum_(t.clone(), group)

    def barrier(self):
        if self.size > 1:
            dist.barrier()

    def comm_stream(self):
        """Side stream for exchanges overlapped with compute (one per process)."""
        st = getattr(self, "_comm_stream", None)
        if st is None:
            st = self._comm_stream = torch.cuda.Stream()
        return st

    def buffer(self, key, numel, device):
        b = self._bufs.get(key)
        if b is None or b.numel() < numel:
            b = torch.empty(numel, dtype=torch.float32, device=device)
            self._bufs[key] = b
        return b[:numel]


def _box_numel(frame, box):
    """box = (z0, y0, x0, ez, ey, ex) over all samples, or an 8-tuple with samples."""
    if len(box) == 6:
        return frame.n * box[3] * box[4] * box[5] * frame.c
    return box[4] * box[5] * box[6] * box[7] * frame.c


def _box8(frame, box):
    if len(box) == 6:
        return (0, box[0], box[1], box[2], frame.n, box[3], box[4], box[5])
    return tuple(box)


def copy_box(frame, box, buf, mode):
    """vpx_halo_copy: mode 0 pack, 1 unpack, 2 unpack-add."""
    _lib.call("vpx_halo_copy", frame.ptr, frame.desc, _box_arg(_box8(frame, box)), buf.data_ptr(),
              mode, torch.cuda.current_stream().cuda_stream)


def _cuda_pack(frame, box, buf):
    copy_box(frame, box, buf, 0)


def _cuda_unpack(frame, box, buf, accumulate):
    copy_box(frame, box, buf, 2 if accumulate else 1)


_BOX_CACHE = {}


def _box_arg(box8):
    import ctypes

    arr = _BOX_CACHE.get(box8)
    if arr is None:
        arr = (ctypes.c_int * 8)(*box8)
        _BOX_CACHE[box8] = arr
    return ctypes.addressof(arr)


def halo_exchange(ctx: RankCtx, tensor, pack=_cuda_pack, unpack=_cuda_unpack):
    """Fill the frame margins of `tensor` (a DistTensor) with neighbour
    boundary data, one round per partitioned dim in ascending order.  Outer
    walls keep their zeros.  Collective over the tensor's rank map."""
    meta, gr = tensor.meta, tensor.grid_rank
    if meta.fabric_rank(gr) != ctx.rank:
        raise OutOfBounds(f"rank {ctx.rank} exchanging a tensor owned by {meta.fabric_rank(gr)}")
    for dim in range(3):
        if meta.radii[dim] == 0 or meta.grid.spatial_parts[dim] == 1:
            continue
        ops, unpacks = [], []
        for side in (-1, 1):
            nbr = meta.neighbor(gr, dim, side)
            if nbr is None:
                continue
            bbox, mbox = round_boxes(meta, gr, dim, side)
            n = _box_numel(tensor, bbox)
            sbuf = ctx.buffer(("hs", dim, side), n, tensor.t.device)
            rbuf = ctx.buffer(("hr", dim, side), n, tensor.t.device)
            pack(tensor, bbox, sbuf)
            peer = meta.fabric_rank(nbr)
            ops.append(("send", peer, sbuf))
            ops.append(("recv", peer, rbuf))
            unpacks.append((mbox, rbuf))
        ctx.exchange(ops)
        for mbox, rbuf in unpacks:
            unpack(tensor, mbox, rbuf, False)
    return tensor


def reverse_halo_exchange(ctx: RankCtx, meta, grid_rank: int, frame, pack=_cuda_pack,
                          unpack=_cuda_unpack):
    """Adjoint of halo_exchange on a gradient frame: descending dims, send
    the margin slab, accumulate what arrives into the boundary; wall margins
    are dropped (reference fabric.py:414-443)."""
    if meta.fabric_rank(grid_rank) != ctx.rank:
        raise OutOfBounds(f"rank {ctx.rank} exchanging a frame owned by {meta.fabric_rank(grid_rank)}")
    for dim in (2, 1, 0):
        if meta.radii[dim] == 0 or meta.grid.spatial_parts[dim] == 1:
            continue
        ops, unpacks = [], []
        for side in (-1, 1):
            nbr = meta.neighbor(grid_rank, dim, side)
            if nbr is None:
                continue
            bbox, mbox = round_boxes(meta, grid_rank, dim, side)
            n = _box_numel(frame, mbox)
            sbuf = ctx.buffer(("rs", dim, side), n, frame.t.device)
            rbuf = ctx.buffer(("rr", dim, side), n, frame.t.device)
            pack(frame, mbox, sbuf)
            peer = meta.fabric_rank(nbr)
            ops.append(("send", peer, sbuf))
            ops.append(("recv", peer, rbuf))
            unpacks.append((bbox, rbuf))
        ctx.exchange(ops)
        for bbox, rbuf in unpacks:
            unpack(frame, bbox, rbuf, True)
    return frame
