"""Serial numpy oracle of the training step -- TEST INFRASTRUCTURE ONLY.

Each function restates one reference routine (file:line cited) with the same
arithmetic in numpy; the three conv loops run in oracle/conv_oracle.c (same
accumulation order as the reference's Cython, -ffp-contract=off), or in the
reference's own compiled kernels when oracle/_ref is built and
VOX_ORACLE_REF=1.  Works in float32 or float64 (dtype of the inputs).
"""

from __future__ import annotations

import ctypes
import importlib.util
import math
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent

# ----------------------------------------------------------------- prng
# reference prng.py:28-90 (splitmix64 key fold + counter stream)
_MASK = (1 << 64) - 1
_G, _M1, _M2, _F0 = 0x9E3779B97F4A7C15, 0xBF58476D1CE4E5B9, 0x94D049BB133111EB, 0x243F6A8885A308D3


def _mix(z: int) -> int:
    z &= _MASK
    z = ((z ^ (z >> 30)) * _M1) & _MASK
    z = ((z ^ (z >> 27)) * _M2) & _MASK
    return z ^ (z >> 31)


def key_fold(parts) -> int:
    acc = _F0
    for p in parts:
        acc = _mix(acc ^ _mix((int(p) & _MASK) + _G))
    return acc


def u64(key, n=None, counters=None):
    k = key if isinstance(key, int) else key_fold(key)
    c = np.arange(n, dtype=np.uint64) if counters is None else np.asarray(counters).astype(np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(k) + (c + np.uint64(1)) * np.uint64(_G)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(_M1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(_M2)
    return z ^ (z >> np.uint64(31))


def uniform01(key, n=None, counters=None):
    return (u64(key, n, counters) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def uniform(key, n, lo, hi):
    return lo + (hi - lo) * uniform01(key, n)


def randint(key, n, lo, hi):
    return (u64(key, n) % np.uint64(hi - lo)).astype(np.int64) + lo


def permutation(key, size):
    perm = np.arange(size, dtype=np.int64)
    draws = u64(key, size)
    for i in range(size - 1, 0, -1):
        j = int(draws[i] % np.uint64(i + 1))
        perm[i], perm[j] = perm[j], perm[i]
    return perm


# --------------------------------------------------------------- conv C
_C = None
_REF = None


def _clib():
    global _C
    if _C is None:
        so = HERE / "conv_oracle.so"
        if not so.exists():
            from . import build_oracle

            build_oracle.build_conv_oracle()
        _C = ctypes.CDLL(str(so))
    return _C


def ref_kernels():
    """The reference's own compiled _hot module (oracle/_ref), or None."""
    global _REF
    if _REF is None:
        from .build_oracle import ref_module_path

        p = ref_module_path()
        if not p.exists():
            return None
        spec = importlib.util.spec_from_file_location("_hot", p)
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        _REF = mod
    return _REF


def _threads():
    return int(os.environ.get("VOX_ORACLE_THREADS", os.cpu_count() or 1))


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _suffix(a):
    if a.dtype == np.float32:
        return "f32"
    if a.dtype == np.float64:
        return "f64"
    raise TypeError(f"oracle conv supports fp32/fp64, got {a.dtype}")


def _use_ref():
    return os.environ.get("VOX_ORACLE_REF") == "1" and ref_kernels() is not None


def k_conv3d_fwd(xpad, w, stride):
    """reference kernels/cyext.py:20-27 + _hot.pyx:19-41"""
    xpad, w = np.ascontiguousarray(xpad), np.ascontiguousarray(w, dtype=xpad.dtype)
    n, cin, pd, ph, pw = xpad.shape
    cout, _, kd, kh, kw = w.shape
    od, oh, ow = ((p - k) // s + 1 for p, k, s in zip((pd, ph, pw), (kd, kh, kw), stride))
    y = np.zeros((n, cout, od, oh, ow), dtype=xpad.dtype)
    if _use_ref():
        ref_kernels().conv3d_fwd(xpad, w, *stride, y)
        return y
    getattr(_clib(), "vox_conv3d_fwd_" + _suffix(xpad))(
        _ptr(xpad), ctypes.c_longlong(n), ctypes.c_longlong(cin), ctypes.c_longlong(pd),
        ctypes.c_longlong(ph), ctypes.c_longlong(pw), _ptr(w), ctypes.c_longlong(cout),
        ctypes.c_longlong(kd), ctypes.c_longlong(kh), ctypes.c_longlong(kw),
        *(ctypes.c_longlong(s) for s in stride), _ptr(y), ctypes.c_longlong(od),
        ctypes.c_longlong(oh), ctypes.c_longlong(ow), ctypes.c_int(_threads()))
    return y


def k_conv3d_bwd_data(u, w, stride, pad_spatial):
    """reference kernels/cyext.py:30-36 + _hot.pyx:44-67"""
    u, w = np.ascontiguousarray(u), np.ascontiguousarray(w, dtype=u.dtype)
    n, cout, od, oh, ow = u.shape
    _, cin, kd, kh, kw = w.shape
    xg = np.zeros((n, cin) + tuple(pad_spatial), dtype=u.dtype)
    if _use_ref():
        ref_kernels().conv3d_bwd_data(u, w, *stride, xg)
        return xg
    getattr(_clib(), "vox_conv3d_bwd_data_" + _suffix(u))(
        _ptr(u), ctypes.c_longlong(n), ctypes.c_longlong(cout), ctypes.c_longlong(od),
        ctypes.c_longlong(oh), ctypes.c_longlong(ow), _ptr(w), ctypes.c_longlong(cin),
        ctypes.c_longlong(kd), ctypes.c_longlong(kh), ctypes.c_longlong(kw),
        *(ctypes.c_longlong(s) for s in stride), _ptr(xg),
        *(ctypes.c_longlong(p) for p in pad_spatial), ctypes.c_int(_threads()))
    return xg


def k_conv3d_bwd_filter(xpad, u, stride, kernel):
    """reference kernels/cyext.py:39-45 + _hot.pyx:70-93"""
    xpad, u = np.ascontiguousarray(xpad), np.ascontiguousarray(u, dtype=xpad.dtype)
    n, cin, pd, ph, pw = xpad.shape
    _, cout, od, oh, ow = u.shape
    wg = np.zeros((cout, cin) + tuple(kernel), dtype=xpad.dtype)
    if _use_ref():
        ref_kernels().conv3d_bwd_filter(xpad, u, *stride, wg)
        return wg
    getattr(_clib(), "vox_conv3d_bwd_filter_" + _suffix(xpad))(
        _ptr(xpad), ctypes.c_longlong(n), ctypes.c_longlong(cin), ctypes.c_longlong(pd),
        ctypes.c_longlong(ph), ctypes.c_longlong(pw), _ptr(u), ctypes.c_longlong(cout),
        ctypes.c_longlong(od), ctypes.c_longlong(oh), ctypes.c_longlong(ow),
        *(ctypes.c_longlong(k) for k in kernel), *(ctypes.c_longlong(s) for s in stride),
        _ptr(wg), ctypes.c_int(_threads()))
    return wg


# --------------------------------------------------------------- layers
def tf32_round(a):
    """Round fp32 to the nearest TF32 value, ties away from zero: the same bits
    as the device's vpx::tf32_rn (csrc/vpx_round.cuh) and cvt.rna.tf32.f32."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    return ((a.view(np.uint32) + np.uint32(0x1000)) & np.uint32(0xFFFFE000)).view(np.float32)


class TF32:
    """TF32-mode numerics of the device path, restated for the oracle.

    The device in TF32 mode (the measured mode) (1) rounds every value it
    stores into an activation/gradient frame to the nearest TF32, (2) feeds
    conv/deconv weights to the products rounded the same way, and (3)
    accumulates the exact TF32 x TF32 products in fp32.  This oracle rounds at
    the same points and accumulates in fp64 (then casts to fp32), so what
    remains between the two is fp32 accumulation order.

    LeakyReLU and max-pool backward are discontinuous in their forward input:
    a pre-activation within a few TF32 ulps of zero (or a max-pool window
    whose two largest values are that close) may legitimately land on the
    other side on the device.  With `device` (the device's forward trace,
    NCDHW arrays keyed ("fwd", layer)), decisions whose oracle margin is at
    most `tau` x max|input| take the device's branch; every decision is
    recorded in `self.branches`, and `flips_outside_band()` lists any
    disagreement OUTSIDE that band (which is a real bug)."""

    def __init__(self, device=None, tau=2.0 ** -11, tf32=True):
        self.device = device
        self.tau = tau
        self.branches = {}
        # tf32=False: the fp32 path's oracle -- no rounding, fp64 accumulation,
        # the same tie-breaks with a band at fp32 accumulation noise (large
        # volumes meet pre-activations that close to zero even in fp32)
        self.r = tf32_round if tf32 else (lambda a: np.asarray(a, dtype=np.float32))

    def dev(self, layer_name):
        if self.device is None:
            return None
        v = self.device.get(("fwd", layer_name))
        return None if v is None else np.asarray(v)

    def leaky_mask(self, name, x, dev_x):
        mask = x >= 0
        amb = np.abs(x) <= self.tau * max(float(np.max(np.abs(x))), 1e-30)
        rec = {"ambiguous": int(amb.sum()), "flips_in_band": 0, "flips_outside": 0}
        if dev_x is not None:
            dmask = dev_x >= 0
            rec["flips_in_band"] = int((amb & (dmask != mask)).sum())
            rec["flips_outside"] = int((~amb & (dmask != mask)).sum())
            mask = np.where(amb, dmask, mask)
        self.branches[name] = rec
        return mask

    def argmax_windows(self, name, x, dev_x):
        win = _windows(x)
        arg = win.argmax(axis=-1)
        top2 = np.sort(win, axis=-1)[..., -2:]
        amb = (top2[..., 1] - top2[..., 0]) <= self.tau * max(float(np.max(np.abs(x))), 1e-30)
        rec = {"ambiguous": int(amb.sum()), "flips_in_band": 0, "flips_outside": 0}
        if dev_x is not None:
            darg = _windows(dev_x).argmax(axis=-1)
            rec["flips_in_band"] = int((amb & (darg != arg)).sum())
            rec["flips_outside"] = int((~amb & (darg != arg)).sum())
            arg = np.where(amb, darg, arg)
        self.branches[name] = rec
        return arg

    def flips_outside_band(self):
        return {k: v["flips_outside"] for k, v in self.branches.items() if v["flips_outside"]}


def _f64(fn, *arrays_and_rest, nargs=2):
    """Run an oracle contraction in fp64 on fp32 operands, return fp32."""
    args = [np.asarray(a, dtype=np.float64) for a in arrays_and_rest[:nargs]] + list(arrays_and_rest[nargs:])
    return fn(*args).astype(np.float32)


def _pad(x, radii):
    rd, rh, rw = radii
    return np.pad(x, ((0, 0), (0, 0), (rd, rd), (rh, rh), (rw, rw)))


def _radii(kernel):
    return tuple((k - 1) // 2 for k in kernel)


def conv3d(x, w, kernel, stride):
    """reference layers/reference.py:72-75"""
    return k_conv3d_fwd(_pad(x, _radii(kernel)), w, stride)


def conv3d_bwd_data(u, w, kernel, stride, in_spatial):
    """reference layers/reference.py:78-87"""
    r = _radii(kernel)
    full = k_conv3d_bwd_data(u, w, stride, tuple(e + 2 * q for e, q in zip(in_spatial, r)))
    return full[:, :, r[0]:r[0] + in_spatial[0], r[1]:r[1] + in_spatial[1], r[2]:r[2] + in_spatial[2]]


def conv3d_bwd_filter(x, u, kernel, stride):
    """reference layers/reference.py:90-94"""
    return k_conv3d_bwd_filter(_pad(x, _radii(kernel)), u, stride, kernel)


def deconv3d(x, w):
    """reference layers/reference.py:99-117: y[n,co,2i+k] = sum_ci x[n,ci,i] w[ci,co,k]"""
    n, cin, d, h, ww = x.shape
    cout = w.shape[1]
    y = np.zeros((n, cout, 2 * d, 2 * h, 2 * ww), dtype=x.dtype)
    for a in range(2):
        for b in range(2):
            for c in range(2):
                y[:, :, a::2, b::2, c::2] = np.einsum("nidhw,io->nodhw", x, w[:, :, a, b, c])
    return y


def deconv3d_bwd_data(u, w):
    """reference layers/reference.py:120-131"""
    xg = 0
    for a in range(2):
        for b in range(2):
            for c in range(2):
                xg = xg + np.einsum("nodhw,io->nidhw", u[:, :, a::2, b::2, c::2], w[:, :, a, b, c])
    return xg.astype(u.dtype)


def deconv3d_bwd_filter(x, u):
    """reference layers/reference.py:134-144"""
    wg = np.zeros((x.shape[1], u.shape[1], 2, 2, 2), dtype=x.dtype)
    for a in range(2):
        for b in range(2):
            for c in range(2):
                wg[:, :, a, b, c] = np.einsum("nidhw,nodhw->io", x, u[:, :, a::2, b::2, c::2])
    return wg


def _windows(x):
    """2^3 windows flattened in (d,h,w) C order (reference layers/reference.py:149-156)"""
    n, c, d, h, w = x.shape
    if d % 2 or h % 2 or w % 2:
        raise ValueError(f"pool3d needs even extents, got {(d, h, w)}")
    v = x.reshape(n, c, d // 2, 2, h // 2, 2, w // 2, 2)
    return v.transpose(0, 1, 2, 4, 6, 3, 5, 7).reshape(n, c, d // 2, h // 2, w // 2, 8)


def pool3d(x, kind):
    """reference layers/reference.py:159-165"""
    win = _windows(x)
    return win.max(axis=-1) if kind == "max" else win.mean(axis=-1)


def pool3d_bwd(x, u, kind, arg=None):
    """reference layers/reference.py:168-183 (avg: u/8 broadcast; max: one-hot at
    the first maximum, or at `arg` when given)"""
    n, c, d, h, w = x.shape
    if kind == "average":
        g = u / u.dtype.type(8)
        return g.repeat(2, axis=2).repeat(2, axis=3).repeat(2, axis=4)
    win = _windows(x)
    hot = np.zeros(win.shape, dtype=u.dtype)
    np.put_along_axis(hot, (win.argmax(axis=-1) if arg is None else arg)[..., None], 1.0, axis=-1)
    g = (hot * u[..., None]).reshape(n, c, d // 2, h // 2, w // 2, 2, 2, 2)
    return g.transpose(0, 1, 2, 5, 3, 6, 4, 7).reshape(n, c, d, h, w)


class BN:
    """reference layers/reference.py:39-57"""

    def __init__(self, gamma, beta, dtype):
        self.gamma, self.beta = gamma, beta
        c = gamma.shape[0]
        self.running_mean = np.zeros(c, dtype=dtype)
        self.running_var = np.ones(c, dtype=dtype)
        self.eps, self.momentum = 1e-5, 0.9


def batchnorm_fwd(x, st: BN, mode="train"):
    """reference layers/reference.py:188-214 (biased var from one-pass sums)"""
    c = x.shape[1]
    ax = (0, 2, 3, 4)
    if mode == "train":
        cnt = x.size // c
        mean = x.sum(axis=ax) / cnt
        var = np.maximum((x * x).sum(axis=ax) / cnt - mean * mean, 0.0)
        st.running_mean[...] = st.momentum * st.running_mean + (1 - st.momentum) * mean
        st.running_var[...] = st.momentum * st.running_var + (1 - st.momentum) * var
    else:
        mean, var, cnt = st.running_mean, st.running_var, 0
    inv = 1.0 / np.sqrt(var + st.eps)
    col = lambda v: np.asarray(v).reshape(1, c, 1, 1, 1).astype(x.dtype)
    xhat = (x - col(mean)) * col(inv)
    return col(st.gamma) * xhat + col(st.beta), (xhat, inv, cnt)


def batchnorm_bwd(u, st: BN, cache):
    """reference layers/reference.py:217-226"""
    xhat, inv, cnt = cache
    c = u.shape[1]
    ax = (0, 2, 3, 4)
    db = u.sum(axis=ax)
    dg = (u * xhat).sum(axis=ax)
    col = lambda v: np.asarray(v).reshape(1, c, 1, 1, 1).astype(u.dtype)
    return col(st.gamma * inv) * (u - (col(db) + xhat * col(dg)) / cnt), dg, db


def leaky(x, slope):
    """reference layers/reference.py:231-233"""
    return np.where(x >= 0, x, x.dtype.type(slope) * x)


def leaky_bwd(x, u, slope, mask=None):
    """reference layers/reference.py:234-236 (`mask`: precomputed x >= 0)"""
    return np.where(x >= 0 if mask is None else mask, u, u.dtype.type(slope) * u)


def dropout_mask(key_parts, n, keep):
    """reference layers/reference.py:239-246"""
    return uniform01(list(key_parts), n) < keep


def dropout_apply(x, mask, keep):
    """reference layers/reference.py:249-253"""
    return x * (mask.astype(x.dtype) / x.dtype.type(keep))


def mse(pred, target):
    """reference layers/reference.py:273-279"""
    d = pred - target
    return float((d * d).sum() / d.size), (2.0 / d.size) * d


def log_softmax(z):
    m = z.max(axis=1, keepdims=True)
    z = z - m
    return z - np.log(np.exp(z).sum(axis=1, keepdims=True))


def cross_entropy(logits, labels):
    """reference layers/reference.py:282-307"""
    lp = log_softmax(logits)
    cnt = labels.size
    lab = labels[:, None].astype(np.int64)
    loss = float(-np.take_along_axis(lp, lab, axis=1).sum() / cnt)
    g = np.exp(lp)
    np.put_along_axis(g, lab, np.take_along_axis(g, lab, axis=1) - 1.0, axis=1)
    return loss, g / cnt


# ---------------------------------------------------------------- model
def param_entries(net):
    """reference model/networks.py:133-153 (order of the gradient bucket)"""
    out = []
    for l in net.layers:
        if l.kind == "conv":
            p = l.params
            out.append((f"{l.name}.w", (p.cout, p.cin) + tuple(p.kernel), p.cin * math.prod(p.kernel)))
        elif l.kind == "deconv":
            out.append((f"{l.name}.w", (l.cin, l.cout, 2, 2, 2), l.cin * 8))
        elif l.kind == "bn":
            out.append((f"{l.name}.gamma", (l.channels,), 0))
            out.append((f"{l.name}.beta", (l.channels,), 0))
        elif l.kind == "fc":
            out.append((f"{l.name}.w", (l.fin, l.fout), l.fin))
            out.append((f"{l.name}.b", (l.fout,), 0))
    return out


def init_params(net, seed, dtype=np.float64):
    """reference model/optim.py:97-113"""
    params = {}
    for i, (name, shape, fan_in) in enumerate(param_entries(net)):
        if fan_in == 0:
            params[name] = np.full(shape, 1.0 if name.endswith(".gamma") else 0.0, dtype=dtype)
        else:
            b = math.sqrt(6.0 / fan_in)
            params[name] = uniform([seed, -1, i], math.prod(shape), -b, b).reshape(shape).astype(dtype)
    return params


def make_bn_states(net, params, dtype):
    """reference model/serial.py:19-30"""
    return {l.name: BN(params[f"{l.name}.gamma"], params[f"{l.name}.beta"], dtype)
            for l in net.layers if l.kind == "bn"}


def synthetic_batch(net, wi, n, seed, dtype):
    """reference cli.py:112-125"""
    shape = (n, net.in_channels, wi, wi, wi)
    x = uniform([seed, -3, 0], math.prod(shape), -1.0, 1.0).reshape(shape).astype(dtype)
    if net.loss == "mse":
        y = uniform([seed, -3, 1], n * net.out_dim, -1.0, 1.0).reshape(n, net.out_dim).astype(dtype)
    else:
        y = randint([seed, -3, 1], n * wi ** 3, 0, net.out_dim).reshape(n, wi, wi, wi)
    return x, y, tuple(range(n))


def _fwd_layer(l, idx, cur, params, states, mode, step_key, sample_ids, outs, num):
    """One layer of reference model/serial.py:42-89: returns (output, stash entry)."""
    R = num.r if num is not None else (lambda a: a)
    k = l.kind
    if k == "conv":
        w = params[f"{l.name}.w"]
        if num is None:
            return conv3d(cur, w, l.params.kernel, l.params.stride), cur
        return R(_f64(conv3d, cur, R(w), l.params.kernel, l.params.stride)), cur
    if k == "deconv":
        w = params[f"{l.name}.w"]
        return (deconv3d(cur, w) if num is None else R(_f64(deconv3d, cur, R(w)))), cur
    if k == "pool":
        return (pool3d(cur, l.pool_kind) if num is None else R(_f64(pool3d, cur, l.pool_kind, nargs=1))), cur
    if k == "bn":
        if num is None:
            return batchnorm_fwd(cur, states[l.name], mode)
        y, cache = batchnorm_fwd(cur.astype(np.float64), states[l.name], mode)
        return R(y.astype(np.float32)), cache
    if k == "leaky":
        return (R(leaky(cur, l.slope)) if cur.ndim == 5 else leaky(cur, l.slope)), cur
    if k == "dropout":
        if mode != "train":
            return cur, None
        s, e, it = step_key
        m = np.stack([dropout_mask([s, e, it, int(sid), idx], cur.shape[1], l.keep) for sid in sample_ids])
        return dropout_apply(cur, m, l.keep), m
    if k == "flatten":
        return cur.reshape(cur.shape[0], -1), cur.shape
    if k == "fc":
        return cur @ params[f"{l.name}.w"] + params[f"{l.name}.b"], cur
    if k == "concat":
        skip = outs[l.skip]
        return np.concatenate([cur, skip], axis=1), (cur.shape[1], skip.shape[1])
    raise ValueError(k)


def forward(net, params, states, x, mode, step_key=(0, 0, 0), sample_ids=(), trace=None, num=None):
    """reference model/serial.py:42-89 (num: TF32 numerics of the device, or None)"""
    cur, outs, stash = (num.r(x) if num is not None else x), {}, []
    for idx, l in enumerate(net.layers):
        cur, kept = _fwd_layer(l, idx, cur, params, states, mode, step_key, sample_ids, outs, num)
        stash.append(kept)
        outs[l.name] = cur
        if trace is not None:
            trace[("fwd", l.name)] = cur
    return cur, stash


def loss_and_grad(net, pred, target, num=None):
    if net.loss == "mse":
        return mse(pred, target)
    loss, g = cross_entropy(pred, target)
    return loss, (g if num is None else num.r(g.astype(np.float32)))


def _bwd_layer(l, u, kept, params, states, grads, num, prev_name):
    """One layer of reference model/serial.py:100-150: returns (input gradient,
    skip gradient or None); parameter gradients go into `grads`."""
    R = num.r if num is not None else (lambda a: a)
    k = l.kind
    if k == "conv":
        w = params[f"{l.name}.w"]
        kk, st = l.params.kernel, l.params.stride
        if num is None:
            grads[f"{l.name}.w"] = conv3d_bwd_filter(kept, u, kk, st)
            return conv3d_bwd_data(u, w, kk, st, kept.shape[2:]), None
        grads[f"{l.name}.w"] = _f64(conv3d_bwd_filter, kept, u, kk, st)
        return R(_f64(conv3d_bwd_data, u, R(w), kk, st, kept.shape[2:])), None
    if k == "deconv":
        w = params[f"{l.name}.w"]
        if num is None:
            grads[f"{l.name}.w"] = deconv3d_bwd_filter(kept, u)
            return deconv3d_bwd_data(u, w), None
        grads[f"{l.name}.w"] = _f64(deconv3d_bwd_filter, kept, u)
        return R(_f64(deconv3d_bwd_data, u, R(w))), None
    if k == "pool":
        arg = None
        if num is not None and l.pool_kind == "max":
            arg = num.argmax_windows(l.name, kept, num.dev(prev_name))
        return R(pool3d_bwd(kept, u, l.pool_kind, arg)), None
    if k == "bn":
        if num is None:
            u, grads[f"{l.name}.gamma"], grads[f"{l.name}.beta"] = batchnorm_bwd(u, states[l.name], kept)
            return u, None
        g, dg, db = batchnorm_bwd(u.astype(np.float64), states[l.name], kept)
        grads[f"{l.name}.gamma"], grads[f"{l.name}.beta"] = dg.astype(np.float32), db.astype(np.float32)
        return R(g.astype(np.float32)), None
    if k == "leaky":
        mask = None if num is None else num.leaky_mask(l.name, kept, num.dev(prev_name))
        g = leaky_bwd(kept, u, l.slope, mask)
        return (R(g) if kept.ndim == 5 else g), None
    if k == "dropout":
        return (dropout_apply(u, kept, l.keep) if kept is not None else u), None
    if k == "flatten":
        return R(u.reshape(kept)), None
    if k == "fc":
        w = params[f"{l.name}.w"]
        grads[f"{l.name}.w"], grads[f"{l.name}.b"] = kept.T @ u, u.sum(axis=0)
        return u @ w.T, None
    if k == "concat":
        c_main, _ = kept
        return u[:, :c_main], u[:, c_main:]
    raise ValueError(k)


def backward(net, params, states, stash, dpred, trace=None, num=None):
    """reference model/serial.py:100-150 (num: TF32 numerics of the device, or None)"""
    R = num.r if num is not None else (lambda a: a)
    grads, u, extra = {}, dpred, {}
    for idx in range(len(net.layers) - 1, -1, -1):
        l = net.layers[idx]
        if l.name in extra:
            u = R(u + extra.pop(l.name))
        prev = net.layers[idx - 1].name if idx > 0 else None
        u, sk = _bwd_layer(l, u, stash[idx], params, states, grads, num, prev)
        if sk is not None:
            extra[l.skip] = extra.get(l.skip, 0) + sk
        if trace is not None:
            trace[("bwd", l.name)] = u
    return grads


def layerwise(net, params, states, x, target, dev, sample_ids=(), step_key=(0, 0, 0), num=None):
    """Teacher-forced per-layer oracle: every layer is evaluated on the
    DEVICE's own inputs -- forward on the device output of the layer before it
    (the first on the network input), backward on the device gradient arriving
    from the layer after it (plus, at a skip source, the device gradient the
    concat split off) and on the device forward input -- so each layer's
    result isolates that layer's kernels from the rounding noise compounded
    upstream.  `dev`: the device trace {("fwd"|"bwd", name): NCDHW/flat array}.
    Returns (trace, grads) in the shapes of forward/backward's."""
    R = num.r if num is not None else (lambda a: a)
    layers = net.layers
    trace, stash, outs = {}, [], {}
    for idx, l in enumerate(layers):
        cur = R(x) if idx == 0 else dev[("fwd", layers[idx - 1].name)]
        outs_dev = {k[1]: v for k, v in dev.items() if k[0] == "fwd"}
        y, kept = _fwd_layer(l, idx, cur, params, states, "train", step_key, sample_ids, outs_dev, num)
        stash.append(kept)
        trace[("fwd", l.name)] = y
    _, dpred = loss_and_grad(net, dev[("fwd", layers[-1].name)], target, num)
    grads = {}
    skips = {}
    for idx, l in enumerate(layers):
        if l.kind == "concat":
            c_main = stash[idx][0]
            after = dev[("bwd", layers[idx + 1].name)] if idx + 1 < len(layers) else dpred
            skips[l.skip] = skips.get(l.skip, 0) + after[:, c_main:]
    for idx in range(len(layers) - 1, -1, -1):
        l = layers[idx]
        u = dpred if idx == len(layers) - 1 else dev[("bwd", layers[idx + 1].name)]
        if l.name in skips:
            u = R(u + skips[l.name])
        prev = layers[idx - 1].name if idx > 0 else None
        g, _ = _bwd_layer(l, u, stash[idx], params, states, grads, None if num is None else _NoTie(num), prev)
        trace[("bwd", l.name)] = g
    return trace, grads


class _NoTie:
    """TF32 numerics without device tie-breaks (a teacher-forced layer sees the
    device's own pre-activations, so its branch decisions are the device's)."""

    def __init__(self, num):
        self.r = num.r
        self.branches = {}

    def dev(self, _name):
        return None

    def leaky_mask(self, name, x, _dev):
        return x >= 0

    def argmax_windows(self, name, x, _dev):
        return _windows(x).argmax(axis=-1)


class Adam:
    """reference model/optim.py:34-52, 71-88"""

    def __init__(self, params, kind="adam"):
        self.kind, self.t = kind, 0
        self.m = {k: np.zeros_like(v) for k, v in params.items()}
        self.v = {k: np.zeros_like(v) for k, v in params.items()}
        self.b1, self.b2, self.eps = 0.9, 0.999, 1e-8

    def step(self, params, grads, lr):
        self.t += 1
        if self.kind == "sgd":
            for k, p in params.items():
                p -= lr * grads[k]
            return
        c1, c2 = 1.0 - self.b1 ** self.t, 1.0 - self.b2 ** self.t
        for k, p in params.items():
            g, m, v = grads[k], self.m[k], self.v[k]
            m *= self.b1
            m += (1 - self.b1) * g
            v *= self.b2
            v += (1 - self.b2) * (g * g)
            p -= lr * (m / c1) / (np.sqrt(v / c2) + self.eps)


def train_step(net, params, states, opt, lr, x, target, sample_ids, step_key, trace=None, grads_out=None,
               num=None):
    """reference model/serial.py:153-161 (num: TF32 numerics of the device, or None)"""
    pred, stash = forward(net, params, states, x, "train", step_key, sample_ids, trace=trace, num=num)
    loss, dpred = loss_and_grad(net, pred, target, num)
    grads = backward(net, params, states, stash, dpred, trace=trace, num=num)
    if grads_out is not None:
        grads_out.update({k: v.copy() for k, v in grads.items()})
    opt.step(params, grads, lr)
    return loss
