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


# Profiling switch only (results are wrong with it): VPX_SKIP_HALO=1 skips the
# halo exchanges to measure what they cost inside a step.
_SKIP_HALO = os.environ.get("VPX_SKIP_HALO") == "1"
# PeerHalo rounds as one fused kernel (vpx_halo_round_peer); VPX_HALO_SPLIT=1
# selects the four-launch pack / signal / wait / unpack sequence per side.
_FUSED_ROUND = os.environ.get("VPX_HALO_SPLIT") != "1"


class RankCtx:
    """Per-process handle (reference fabric.py:111-128 API)."""

    def __init__(self, rank: int = 0, size: int = 1, device=None):
        self.rank = rank
        self.size = size
        self.device = device
        self._groups = {}
        self._bufs = {}
        self.peer = None

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
    _DTYPES = (torch.float32, torch.float64, torch.int64, torch.int32, torch.int16, torch.int8, torch.uint8)

    def send(self, dst: int, tag: int, tensor: torch.Tensor):
        """Point-to-point send (reference fabric.py:111-119).  A small header
        (dtype code, ndim, dims) precedes the payload so recv() can allocate
        the message like the reference's fabric hands over the array."""
        if dst == self.rank:
            raise OutOfBounds("send to self")
        t = tensor.contiguous()
        if t.dim() > 8:
            raise OutOfBounds(f"send of a {t.dim()}-d tensor (at most 8 dims)")
        hdr = torch.zeros(10, dtype=torch.int64, device=t.device)
        hdr[0], hdr[1] = self._DTYPES.index(t.dtype), t.dim()
        if t.dim():
            hdr[2:2 + t.dim()] = torch.tensor(t.shape, dtype=torch.int64)
        dist.send(hdr, dst)
        dist.send(t, dst)

    def recv(self, src: int, tag: int, like: torch.Tensor = None) -> torch.Tensor:
        """Receive the next message from `src` (reference fabric.py:120-121);
        `like` optionally supplies the destination buffer."""
        dev = like.device if like is not None else (self.device or torch.device("cpu"))
        hdr = torch.empty(10, dtype=torch.int64, device=dev)
        dist.recv(hdr, src)
        shape = tuple(int(v) for v in hdr[2:2 + int(hdr[1])].tolist())
        dt = self._DTYPES[int(hdr[0])]
        if like is None:
            like = torch.empty(shape, dtype=dt, device=dev)
        elif tuple(like.shape) != shape or like.dtype != dt:
            raise OutOfBounds(f"recv buffer {tuple(like.shape)} {like.dtype} != message {shape} {dt}")
        dist.recv(like, src)
        return like

    def exchange(self, ops, tag: str = "comm.p2p"):
        """ops: list of ("send"|"recv", peer, tensor); one NCCL group."""
        if not ops:
            return
        p2p = [dist.P2POp(dist.isend if kind == "send" else dist.irecv, t, peer)
               for kind, peer, t in ops]
        nbytes = sum(4 * t.numel() for kind, _, t in ops if kind == "send")
        with region(tag, 0, nbytes):
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

    def ensure_peer_halo(self, plan):
        """Set up CUDA-IPC halo mailboxes (PeerHalo) once per plan; collective.
        Falls back to NCCL P2P when IPC is unavailable or VPX_NCCL_HALO=1."""
        if self.size == 1 or getattr(self, "_peer_plan", None) is plan:
            return
        self._peer_plan = plan
        if os.environ.get("VPX_NCCL_HALO") == "1" or not torch.cuda.is_available():
            self.close_peer_halo()
            return
        need = PeerHalo.requirements(self, plan)
        if need is None:  # nothing spatially partitioned: no halos to exchange
            self.close_peer_halo()
            self.halo_error = None
            self.no_halo = True
            return
        self.no_halo = False
        if self.peer is not None and self.peer.satisfies(need):
            return  # same neighbours, mailboxes large enough: keep the mappings
        self.close_peer_halo()
        ok = 1
        try:
            peer = PeerHalo(self, plan)
        except Exception as exc:  # pragma: no cover - reported through halo_path
            peer, ok = None, 0
            self.halo_error = f"{type(exc).__name__}: {exc}"
        flag = torch.tensor([ok], dtype=torch.int32, device="cuda")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) != 1 and peer is not None:
            peer.close()
            peer = None
        self.peer = peer

    def close_peer_halo(self):
        """Release the peer-halo mailboxes and IPC mappings (collective when a
        PeerHalo is open: every rank closes together)."""
        if self.peer is not None:
            self.peer.close()
            self.peer = None

    @property
    def halo_path(self) -> str:
        if self.size == 1:
            return "none (single rank)"
        if getattr(self, "no_halo", False):
            return "none (no spatially partitioned tensor)"
        if self.peer is not None:
            return "CUDA-IPC mailboxes over NVLink (PeerHalo)"
        return "NCCL send/recv" + (f" (IPC setup failed: {self.halo_error})" if getattr(self, "halo_error", None) else "")

    def grad_group(self):
        """A communicator of its own for the bucketed gradient all-reduce, so
        its kernels (on grad_stream) never queue behind or interleave with the
        halo / BatchNorm collectives of the world group.  Collective on first
        use."""
        g = getattr(self, "_grad_group", None)
        if g is None and self.size > 1:
            g = self._grad_group = dist.new_group(list(range(self.size)))
        return g

    def grad_stream(self):
        st = getattr(self, "_grad_stream", None)
        if st is None:
            st = self._grad_stream = torch.cuda.Stream()
        return st

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


class PeerHalo:
    """Halo faces through CUDA-IPC mailboxes over NVLink instead of NCCL P2P.

    Every rank allocates, once, two mailboxes per (dim, side) it receives
    from plus an arrival counter, and opens its neighbours' allocations via
    CUDA IPC.  A face is packed by vpx_halo_copy straight into the
    neighbour's mailbox (peer stores), vpx_peer_signal bumps the neighbour's
    counter; the receiver's vpx_peer_wait holds its stream until the face has
    arrived and unpacks locally.  No NCCL kernel, no rendezvous: each round is
    a pack kernel, a one-thread signal and a one-thread wait.  Mailboxes
    alternate per exchange; a rank writes mailbox p again only after it has
    received the neighbour's next face, which the neighbour sends after
    unpacking p (exchanges with a neighbour are always two-way), and steps are
    separated by the gradient all-reduce.  Counters live in device memory, so
    the exchange replays inside a CUDA graph.
    """

    TIMEOUT_NS = 10_000_000_000

    def __init__(self, ctx: "RankCtx", plan):
        from cuda.bindings import runtime as rt

        self.rt = rt
        need = self.requirements(ctx, plan)
        if need is None:
            raise OutOfBounds("no spatially partitioned tensors")
        meta, gr, slab, self.neighbours = need
        self.slab = slab
        self.flags_off = 12 * self.slab
        total = self.flags_off + 4096
        err, ptr = rt.cudaMalloc(total)
        if err != rt.cudaError_t.cudaSuccess:
            raise OutOfBounds(f"peer mailbox allocation failed: {err}")
        rt.cudaMemset(ptr, 0, total)
        rt.cudaDeviceSynchronize()
        self.base = int(ptr)
        self.opened = {}
        err, handle = rt.cudaIpcGetMemHandle(ptr)
        if err != rt.cudaError_t.cudaSuccess:
            raise OutOfBounds(f"cudaIpcGetMemHandle failed: {err}")
        handles = [None] * ctx.size
        dist.all_gather_object(handles, bytes(handle.reserved))
        self.peer_base, opened = {}, {}
        for dim in range(3):
            for side in (-1, 1):
                nbr = meta.neighbor(gr, dim, side)
                if nbr is None:
                    continue
                peer = meta.fabric_rank(nbr)
                if peer not in opened:  # one mapping per peer process
                    h = rt.cudaIpcMemHandle_t()
                    h.reserved = handles[peer]
                    err, pptr = rt.cudaIpcOpenMemHandle(h, rt.cudaIpcMemLazyEnablePeerAccess)
                    if err != rt.cudaError_t.cudaSuccess:
                        raise OutOfBounds(f"cudaIpcOpenMemHandle({peer}) failed: {err}")
                    opened[peer] = int(pptr)
                self.peer_base[(dim, side)] = opened[peer]
        self.opened = opened
        self.count = {}
        self.ctx = ctx
        ctx.barrier()

    @staticmethod
    def requirements(ctx: "RankCtx", plan):
        """(first partitioned meta, its grid rank, mailbox bytes, neighbour
        set) a plan needs, or None when nothing is spatially partitioned."""
        metas = [m for m in plan.in_meta if m is not None and any(p > 1 for p in m.grid.spatial_parts)]
        if not metas:
            return None
        meta = metas[0]
        gr = meta.grid_rank_of(ctx.rank)
        # largest face any round can carry: whole frame cross-section, all channels
        slab = 0
        for m in metas:
            try:
                g = m.grid_rank_of(ctx.rank)
            except OutOfBounds:
                continue
            ls, mg = m.local_shape(g), m.margins()
            ext = (ls.d + 2 * mg[0], ls.h + 2 * mg[1], ls.w + 2 * mg[2])
            for dim in range(3):
                slab = max(slab, ls.n * ls.c * ext[(dim + 1) % 3] * ext[(dim + 2) % 3] * max(1, m.radii[dim]) * 4)
        nbrs = tuple((dim, side, meta.fabric_rank(meta.neighbor(gr, dim, side)))
                     for dim in range(3) for side in (-1, 1) if meta.neighbor(gr, dim, side) is not None)
        return meta, gr, (slab + 4095) // 4096 * 4096, nbrs

    def satisfies(self, need) -> bool:
        return need is not None and need[3] == self.neighbours and need[2] <= self.slab

    def close(self):
        """Close the neighbours' IPC mappings and free this rank's mailbox.
        Collective: a neighbour may still be writing into our mailbox until
        every rank has drained its stream, hence the barrier first."""
        if self.base is None:
            return
        torch.cuda.synchronize()
        self.ctx.barrier()
        for p in self.opened.values():
            self.rt.cudaIpcCloseMemHandle(p)
        self.opened = {}
        self.ctx.barrier()
        self.rt.cudaFree(self.base)
        self.base = None

    @staticmethod
    def _chan(dim, side):
        return 2 * dim + (side + 1) // 2

    def _parity(self, key):
        c = self.count.get(key, 0)
        self.count[key] = c + 1
        return c & 1

    def send(self, dim, side, frame, box, mode):
        """Face `box` of `frame` -> the neighbour on `side` (its channel (dim, -side))."""
        ch = self._chan(dim, -side)
        par = self._parity(("s", dim, side))
        dst = self.peer_base[(dim, side)] + (2 * ch + par) * self.slab
        if _box_numel(frame, box) * 4 > self.slab:
            raise OutOfBounds("halo face larger than the mailbox")
        st = torch.cuda.current_stream().cuda_stream
        _lib.call("vpx_halo_copy", frame.ptr, frame.desc, _box_arg(_box8(frame, box)), dst, mode, st)
        _lib.call("vpx_peer_signal", self.peer_base[(dim, side)] + self.flags_off + 8 * ch, st)

    def round(self, dim, sides, frame, send_boxes, recv_boxes, mode):
        """One whole round (both sides of `dim`) in one kernel
        (vpx_halo_round_peer): faces packed into the neighbours' mailboxes,
        released, awaited and unpacked (mode 1) / accumulated (mode 2).  Same
        mailboxes, flags and parities as send()/recv()."""
        import ctypes

        desc = [0] * 64
        desc[23] = self.base + self.flags_off + 256  # three u32 block counters (zero at rest)
        for side, sbox, rbox in zip(sides, send_boxes, recv_boxes):
            d = 32 * ((side + 1) // 2)
            ch_s = self._chan(dim, -side)
            par_s = self._parity(("s", dim, side))
            ch_r = self._chan(dim, side)
            par_r = self._parity(("r", dim, side))
            desc[d + 0] = 1
            desc[d + 1:d + 9] = _box8(frame, sbox)
            desc[d + 9] = self.peer_base[(dim, side)] + (2 * ch_s + par_s) * self.slab
            desc[d + 10] = self.peer_base[(dim, side)] + self.flags_off + 8 * ch_s
            desc[d + 11] = 1
            desc[d + 12:d + 20] = _box8(frame, rbox)
            desc[d + 20] = self.base + (2 * ch_r + par_r) * self.slab
            desc[d + 21] = self.base + self.flags_off + 8 * ch_r
            desc[d + 22] = self.base + self.flags_off + 64 + 8 * ch_r
            desc[d + 24] = mode
        arr = (ctypes.c_longlong * 64)(*desc)
        st = torch.cuda.current_stream().cuda_stream
        _lib.call("vpx_halo_round_peer", frame.ptr, frame.desc, ctypes.addressof(arr), self.slab, self.TIMEOUT_NS,
                  self.base + self.flags_off + 128, st)

    def recv(self, dim, side, frame, box, mode):
        """Face from the neighbour on `side` (my channel (dim, side)) -> `box` of `frame`."""
        ch = self._chan(dim, side)
        par = self._parity(("r", dim, side))
        st = torch.cuda.current_stream().cuda_stream
        _lib.call("vpx_peer_wait", self.base + self.flags_off + 8 * ch, self.base + self.flags_off + 64 + 8 * ch,
                  self.TIMEOUT_NS, self.base + self.flags_off + 128, st)
        src = self.base + (2 * ch + par) * self.slab
        _lib.call("vpx_halo_copy", frame.ptr, frame.desc, _box_arg(_box8(frame, box)), src, mode, st)


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
    if _SKIP_HALO:
        return tensor
    meta, gr = tensor.meta, tensor.grid_rank
    if meta.fabric_rank(gr) != ctx.rank:
        raise OutOfBounds(f"rank {ctx.rank} exchanging a tensor owned by {meta.fabric_rank(gr)}")
    peer = ctx.peer if (pack is _cuda_pack and getattr(ctx, "peer", None) is not None) else None
    for dim in range(3):
        if meta.radii[dim] == 0 or meta.grid.spatial_parts[dim] == 1:
            continue
        if peer is not None:
            sides = [s for s in (-1, 1) if meta.neighbor(gr, dim, s) is not None]
            nbytes = sum(4 * _box_numel(tensor, round_boxes(meta, gr, dim, side)[0]) for side in sides)
            with region("comm.halo", 0, nbytes):
                if _FUSED_ROUND and tensor.c % 4 == 0:
                    boxes = [round_boxes(meta, gr, dim, side) for side in sides]
                    peer.round(dim, sides, tensor, [b[0] for b in boxes], [b[1] for b in boxes], 1)
                else:
                    for side in sides:
                        peer.send(dim, side, tensor, round_boxes(meta, gr, dim, side)[0], 0)
                    for side in sides:
                        peer.recv(dim, side, tensor, round_boxes(meta, gr, dim, side)[1], 1)
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
            other = meta.fabric_rank(nbr)
            ops.append(("send", other, sbuf))
            ops.append(("recv", other, rbuf))
            unpacks.append((mbox, rbuf))
        ctx.exchange(ops, "comm.halo")
        for mbox, rbuf in unpacks:
            unpack(tensor, mbox, rbuf, False)
    return tensor


def reverse_halo_exchange(ctx: RankCtx, meta, grid_rank: int, frame, pack=_cuda_pack,
                          unpack=_cuda_unpack):
    """Adjoint of halo_exchange on a gradient frame: descending dims, send
    the margin slab, accumulate what arrives into the boundary; wall margins
    are dropped (reference fabric.py:414-443)."""
    if _SKIP_HALO:
        return frame
    if meta.fabric_rank(grid_rank) != ctx.rank:
        raise OutOfBounds(f"rank {ctx.rank} exchanging a frame owned by {meta.fabric_rank(grid_rank)}")
    peer = ctx.peer if (pack is _cuda_pack and getattr(ctx, "peer", None) is not None) else None
    for dim in (2, 1, 0):
        if meta.radii[dim] == 0 or meta.grid.spatial_parts[dim] == 1:
            continue
        if peer is not None:
            sides = [s for s in (-1, 1) if meta.neighbor(grid_rank, dim, s) is not None]
            nbytes = sum(4 * _box_numel(frame, round_boxes(meta, grid_rank, dim, side)[1]) for side in sides)
            with region("comm.halo", 0, nbytes):
                if _FUSED_ROUND and frame.c % 4 == 0:
                    boxes = [round_boxes(meta, grid_rank, dim, side) for side in sides]
                    peer.round(dim, sides, frame, [b[1] for b in boxes], [b[0] for b in boxes], 2)
                else:
                    for side in sides:
                        peer.send(dim, side, frame, round_boxes(meta, grid_rank, dim, side)[1], 0)
                    for side in sides:
                        peer.recv(dim, side, frame, round_boxes(meta, grid_rank, dim, side)[0], 2)
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
            other = meta.fabric_rank(nbr)
            ops.append(("send", other, sbuf))
            ops.append(("recv", other, rbuf))
            unpacks.append((bbox, rbuf))
        ctx.exchange(ops, "comm.halo")
        for bbox, rbuf in unpacks:
            unpack(frame, bbox, rbuf, True)
    return frame
