"""Device-resident distributed tensors (NDHWC halo frames in HBM).

A DistTensor holds one rank's block of a partitioned 5D tensor as a single
fp32 CUDA tensor of shape (n_local, D+2md, H+2mh, W+2mw, C): channels
innermost (each voxel is one contiguous 16..1024-byte row, the unit the
tcgen05 kernels load with TMA), margins m = the consumer's halo radius in
partitioned dimensions only.  Outer walls and unpartitioned dimensions get
their zero padding from TMA out-of-bounds fill, so they cost no memory.

Reference counterpart: DistTensor (reference pkg/src/voxpar/tensor.py:294-351)
keeps an NCDHW numpy frame with margins in every dimension and is re-copied
by every op (_wrap, reference layers/distributed.py:31-33); here producers
write straight into their consumer's frame.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .errors import ShapeMismatch
from .geometry import DistTensorMeta


def frame_desc(n, c, d, h, w, md=0, mh=0, mw=0):
    """int[8] frame descriptor for the C ABI (include/vpx.h)."""
    return (ctypes.c_int * 8)(n, c, d, h, w, md, mh, mw)


def stream_ptr():
    return torch.cuda.current_stream().cuda_stream


class Frame:
    """A plain device frame (no partition metadata): storage + descriptor."""

    __slots__ = ("t", "n", "c", "d", "h", "w", "m", "_desc")

    def __init__(self, n, c, d, h, w, margins=(0, 0, 0), zero=None, tensor=None):
        md, mh, mw = margins
        self.n, self.c, self.d, self.h, self.w, self.m = n, c, d, h, w, tuple(margins)
        shape = (n, d + 2 * md, h + 2 * mh, w + 2 * mw, c)
        if tensor is not None:
            if tuple(tensor.shape) != shape:
                raise ShapeMismatch(f"frame storage {tuple(tensor.shape)} != {shape}")
            self.t = tensor
        elif zero if zero is not None else any(margins):
            self.t = torch.zeros(shape, dtype=torch.float32, device="cuda")
        else:
            self.t = torch.empty(shape, dtype=torch.float32, device="cuda")
        self._desc = frame_desc(n, c, d, h, w, md, mh, mw)

    @property
    def desc(self):
        return ctypes.addressof(self._desc)

    @property
    def ptr(self):
        return self.t.data_ptr()

    @property
    def interior(self):
        md, mh, mw = self.m
        return self.t[:, md:md + self.d, mh:mh + self.h, mw:mw + self.w, :]

    @property
    def spatial(self):
        return (self.d, self.h, self.w)

    def voxels(self):
        return self.n * self.d * self.h * self.w

    def to_ncdhw(self) -> torch.Tensor:
        """Dense NCDHW copy of the interior (device)."""
        out = torch.empty((self.n, self.c, self.d, self.h, self.w), dtype=torch.float32, device="cuda")
        _lib.call("vpx_layout_frame_to_ncdhw", self.ptr, self.desc, out.data_ptr(), stream_ptr())
        return out

    def load_ncdhw(self, src) -> "Frame":
        """Fill the interior from an NCDHW array/tensor (host or device)."""
        if isinstance(src, np.ndarray):
            if src.dtype in (np.int16, np.int8):
                src = torch.from_numpy(np.ascontiguousarray(src))
            else:
                src = torch.from_numpy(np.ascontiguousarray(src, dtype=np.float32))
        if tuple(src.shape) != (self.n, self.c, self.d, self.h, self.w):
            raise ShapeMismatch(f"block shape {tuple(src.shape)} != {(self.n, self.c) + self.spatial}")
        if src.dtype in (torch.int16, torch.int8):
            # HSB1 storage dtype (or the datastore's int8 transfer copy):
            # converted to fp32 inside the layout kernel
            src = src.to(device="cuda").contiguous()
            fn = "vpx_layout_ncdhw_i16_to_frame" if src.dtype == torch.int16 else "vpx_layout_ncdhw_i8_to_frame"
            _lib.call(fn, src.data_ptr(), self.desc, self.ptr, stream_ptr())
            return self
        src = src.to(device="cuda", dtype=torch.float32).contiguous()
        _lib.call("vpx_layout_ncdhw_to_frame", src.data_ptr(), self.desc, self.ptr, stream_ptr())
        return self


class DistTensor(Frame):
    """One rank's block of a partitioned tensor (API of reference tensor.py:294-351)."""

    __slots__ = ("meta", "grid_rank")

    def __init__(self, meta: DistTensorMeta, grid_rank: int, data=None, zero=None):
        loc = meta.local_shape(grid_rank)
        super().__init__(loc.n, loc.c, loc.d, loc.h, loc.w, meta.margins(), zero=zero)
        self.meta = meta
        self.grid_rank = grid_rank
        if data is not None:
            self.load_ncdhw(data)

    def clone(self) -> "DistTensor":
        out = DistTensor.__new__(DistTensor)
        Frame.__init__(out, self.n, self.c, self.d, self.h, self.w, self.m, tensor=self.t.clone())
        out.meta, out.grid_rank = self.meta, self.grid_rank
        return out

    @property
    def region(self):
        return self.meta.region(self.grid_rank)

    @property
    def data(self):
        """Interior (n, d, h, w, c) view, writable."""
        return self.interior

    def padded(self):
        return self.t

    def numpy(self) -> np.ndarray:
        """Interior as an NCDHW float32 numpy array (parity / trace dumps)."""
        return self.to_ncdhw().cpu().numpy()
