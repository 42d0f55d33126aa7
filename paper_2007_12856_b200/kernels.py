"""Kernel backend with the reference's kernel boundary (drop-in for voxpar.kernels).

The reference selects between two interchangeable modules exporting
``NAME`` + ``conv3d_fwd(xpad, w, stride)``, ``conv3d_bwd_data(u, w, stride,
pad_spatial)``, ``conv3d_bwd_filter(xpad, u, stride, kernel)`` (reference
pkg/src/voxpar/kernels/__init__.py:63-72, cyext.py:9-45, fallback.py:14-72).
This module is a third such backend ("b200") over libvpx.so, with the same
contracts:

* ``xpad`` is the pre-padded NCDHW input (``np.pad`` "same" padding, or a
  halo frame whose margins hold neighbour data, reference
  layers/distributed.py:57-65); ``u`` the NCDHW upstream gradient; ``w`` OIDHW.
* out spatial = (pad - k) // s + 1 (reference fallback.py:17-18);
  ``conv3d_bwd_data`` returns the gradient over the whole padded frame
  (margins included: the caller crops or reverse-exchanges it).
* Arguments may be numpy arrays (host buffers: copied to the device, computed,
  copied back; the result is a numpy array) or CUDA torch tensors (the result
  stays on the device).  Only float32 is accepted (``TypeError`` otherwise,
  like the reference's dtype check, cyext.py:14-17); kernels must be cubic
  with k in {1, 3} (the halo frames hold margins of 0 or 1), else
  ``Unsupported``.

Numerics follow the library's precision mode (``set_precision``): "tf32"
(tensor cores; inputs are rounded to nearest TF32 on upload) or "fp32"
(CUDA-core direct kernels).  No CPU path exists: without a CUDA device every
call raises ``DeviceError``.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .errors import ShapeMismatch, Unsupported
from .frames import frame_desc as _frame_desc, stream_ptr

NAME = "b200"

_ws = {"t": None}
_keep = []


def frame_desc(*v):
    """Address of an int[8] frame descriptor, kept alive until the next call."""
    arr = _frame_desc(*v)
    _keep.append(arr)
    del _keep[:-16]
    return ctypes.addressof(arr)


def _workspace(nbytes):
    t = _ws["t"]
    if t is None or t.numel() * 4 < nbytes:
        t = torch.empty(max(1, (nbytes + 3) // 4), dtype=torch.float32, device="cuda")
        _ws["t"] = t
    return t


def _check_dtype(*arrays):
    for a in arrays:
        dt = a.dtype
        if dt not in (np.float32, torch.float32):
            raise TypeError(f"b200 kernels support float32 only, got {dt}")


def _triple(v):
    v = tuple(int(x) for x in (v if hasattr(v, "__len__") else (v, v, v)))
    if len(v) != 3:
        raise ShapeMismatch(f"expected 3 spatial values, got {v}")
    return v


def _cube(vals, what):
    if len(set(vals)) != 1:
        raise Unsupported(f"non-cubic {what} {vals}")
    return vals[0]


def _to_device(a):
    """(cuda tensor, was_host)"""
    if isinstance(a, torch.Tensor):
        if not a.is_cuda:
            return a.contiguous().cuda(non_blocking=True), True
        return a.contiguous(), False
    return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().cuda(non_blocking=True), True


def _framed(src, n, c, d, h, w, m):
    """NCDHW device tensor covering the whole padded frame -> NDHWC frame storage
    with interior (d, h, w) and margin m (the padded array is the frame)."""
    buf = torch.empty((n, d + 2 * m, h + 2 * m, w + 2 * m, c), dtype=torch.float32, device="cuda")
    whole = frame_desc(n, c, d + 2 * m, h + 2 * m, w + 2 * m)
    _lib.call("vpx_layout_ncdhw_to_frame", src.data_ptr(), whole, buf.data_ptr(), stream_ptr())
    return buf


def _unframed(buf, n, c, d, h, w, m):
    out = torch.empty((n, c, d + 2 * m, h + 2 * m, w + 2 * m), dtype=torch.float32, device="cuda")
    whole = frame_desc(n, c, d + 2 * m, h + 2 * m, w + 2 * m)
    _lib.call("vpx_layout_frame_to_ncdhw", buf.data_ptr(), whole, out.data_ptr(), stream_ptr())
    return out


def _result(t, host):
    if host:
        return t.cpu().numpy()
    return t


def _geometry(pad_spatial, k, stride):
    if k not in (1, 3):
        raise Unsupported(f"kernel size {k}: the halo frames support k in (1, 3)")
    m = (k - 1) // 2
    s = _cube(stride, "stride")
    if s not in (1, 2):
        raise Unsupported(f"stride {s}")
    interior = tuple(p - 2 * m for p in pad_spatial)
    if min(interior) < 1:
        raise ShapeMismatch(f"padded extent {pad_spatial} too small for kernel {k}")
    out = tuple((p - k) // s + 1 for p in pad_spatial)
    return m, s, interior, out


def conv3d_fwd(xpad, w, stride):
    """y = conv(xpad, w) (reference kernels/__init__.py:63, _hot.pyx:19-41)."""
    _check_dtype(xpad, w)
    n, cin = xpad.shape[:2]
    cout, wcin = w.shape[:2]
    if wcin != cin:
        raise ShapeMismatch(f"weight cin {wcin} != input channels {cin}")
    k = _cube(tuple(w.shape[2:]), "kernel")
    m, s, (d, h, wd), (od, oh, ow) = _geometry(tuple(xpad.shape[2:]), k, _triple(stride))
    x_d, host = _to_device(xpad)
    w_d, _ = _to_device(w)
    xf = _framed(x_d, n, cin, d, h, wd, m)
    y = torch.empty((n, od, oh, ow, cout), dtype=torch.float32, device="cuda")
    ydesc = frame_desc(n, cout, od, oh, ow)
    nb = _lib.load().vpx_conv3d_workspace_bytes(cin, cout, k, ydesc)
    ws = _workspace(nb)
    _lib.call("vpx_conv3d_fwd", xf.data_ptr(), frame_desc(n, cin, d, h, wd, m, m, m), w_d.data_ptr(), k, s,
              y.data_ptr(), ydesc, ws.data_ptr(), ws.numel() * 4, stream_ptr())
    return _result(_unframed(y, n, cout, od, oh, ow, 0), host)


def conv3d_bwd_data(u, w, stride, pad_spatial):
    """Gradient w.r.t. the padded input frame (reference kernels/__init__.py:67,
    _hot.pyx:44-67): every position of the (n, cin) + pad_spatial frame."""
    _check_dtype(u, w)
    n, cout = u.shape[:2]
    wcout, cin = w.shape[:2]
    if wcout != cout:
        raise ShapeMismatch(f"weight cout {wcout} != gradient channels {cout}")
    k = _cube(tuple(w.shape[2:]), "kernel")
    pad_spatial = _triple(pad_spatial)
    m, s, (d, h, wd), out = _geometry(pad_spatial, k, _triple(stride))
    if tuple(u.shape[2:]) != out:
        raise ShapeMismatch(f"gradient spatial {tuple(u.shape[2:])} != conv output {out}")
    u_d, host = _to_device(u)
    w_d, _ = _to_device(w)
    od, oh, ow = out
    uf = _framed(u_d, n, cout, od, oh, ow, 0)
    g = torch.empty((n, d + 2 * m, h + 2 * m, wd + 2 * m, cin), dtype=torch.float32, device="cuda")
    udesc = frame_desc(n, cout, od, oh, ow)
    nb = _lib.load().vpx_conv3d_workspace_bytes(cin, cout, k, udesc)
    ws = _workspace(nb)
    _lib.call("vpx_conv3d_bwd_data", uf.data_ptr(), udesc, w_d.data_ptr(), k, s, g.data_ptr(),
              frame_desc(n, cin, d, h, wd, m, m, m), ws.data_ptr(), ws.numel() * 4, stream_ptr())
    return _result(_unframed(g, n, cin, d, h, wd, m), host)


def conv3d_bwd_filter(xpad, u, stride, kernel):
    """wg[co][ci][a][b][c] = sum u * shifted xpad (reference kernels/__init__.py:71,
    _hot.pyx:70-93).  Deterministic."""
    _check_dtype(xpad, u)
    n, cin = xpad.shape[:2]
    cout = u.shape[1]
    if u.shape[0] != n:
        raise ShapeMismatch(f"gradient batch {u.shape[0]} != input batch {n}")
    k = _cube(_triple(kernel), "kernel")
    m, s, (d, h, wd), out = _geometry(tuple(xpad.shape[2:]), k, _triple(stride))
    if tuple(u.shape[2:]) != out:
        raise ShapeMismatch(f"gradient spatial {tuple(u.shape[2:])} != conv output {out}")
    x_d, host = _to_device(xpad)
    u_d, _ = _to_device(u)
    od, oh, ow = out
    xf = _framed(x_d, n, cin, d, h, wd, m)
    uf = _framed(u_d, n, cout, od, oh, ow, 0)
    udesc = frame_desc(n, cout, od, oh, ow)
    wg = torch.empty((cout, cin, k, k, k), dtype=torch.float32, device="cuda")
    nb = _lib.load().vpx_conv3d_workspace_bytes(cin, cout, k, udesc)
    ws = _workspace(nb)
    _lib.call("vpx_conv3d_bwd_filter", xf.data_ptr(), frame_desc(n, cin, d, h, wd, m, m, m), uf.data_ptr(),
              udesc, k, s, wg.data_ptr(), 0, ws.data_ptr(), ws.numel() * 4, stream_ptr())
    return _result(wg, host)
