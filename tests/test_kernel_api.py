"""The b200 kernel backend behind the reference's kernel boundary
(reference pkg/tests/test_kernels.py, kernels/__init__.py:63-72): same
call signatures, host (numpy) and device (torch) buffers, checked against the
oracle (the reference's own Cython kernels when oracle/_ref is built)."""

import numpy as np
import pytest

from paper_2007_12856_b200 import kernels as K

from oracle import serial as O


def _cases(dtype=np.float32):
    """reference tests/test_kernels.py:9-16 plus tensor-core-sized shapes."""
    rng = np.random.default_rng(3)
    out = []
    for stride in ((1, 1, 1), (2, 2, 2)):
        xpad = rng.normal(size=(2, 3, 9, 9, 9)).astype(dtype)
        w = rng.normal(size=(4, 3, 3, 3, 3)).astype(dtype)
        out.append((xpad, w, stride))
    # row-window (W = 128) and tap-box (W < 128, stride 2) shapes
    out.append((rng.normal(size=(1, 16, 6, 6, 130)).astype(dtype),
                rng.normal(size=(32, 16, 3, 3, 3)).astype(dtype) * 0.1, (1, 1, 1)))
    out.append((rng.normal(size=(1, 64, 10, 10, 10)).astype(dtype),
                rng.normal(size=(128, 64, 3, 3, 3)).astype(dtype) * 0.05, (2, 2, 2)))
    out.append((rng.normal(size=(2, 32, 10, 6, 18)).astype(dtype),
                rng.normal(size=(64, 32, 3, 3, 3)).astype(dtype) * 0.05, (1, 1, 1)))
    return out


def _scaled_err(got, want):
    return float(np.max(np.abs(got - want)) / np.max(np.abs(want)))


def test_backend_name_and_dtype_check():
    assert K.NAME == "b200"
    x = np.zeros((1, 1, 3, 3, 3))
    with pytest.raises(TypeError, match="float32"):
        K.conv3d_fwd(x, np.ones((1, 1, 1, 1, 1)), (1, 1, 1))


def test_unsupported_kernel_size():
    from paper_2007_12856_b200.errors import Unsupported

    x = np.zeros((1, 1, 7, 7, 7), np.float32)
    with pytest.raises(Unsupported):
        K.conv3d_fwd(x, np.ones((1, 1, 5, 5, 5), np.float32), (1, 1, 1))


@pytest.fixture(params=["fp32", "tf32"])
def precision(request):
    import paper_2007_12856_b200 as pkg

    pkg.set_precision(request.param)
    yield request.param
    pkg.set_precision("tf32")


@pytest.mark.gpu
def test_fwd_known_value(precision):
    """reference tests/test_kernels.py:73-79: 1x1x1 identity kernel."""
    xpad = np.arange(27, dtype=np.float32).reshape(1, 1, 3, 3, 3)
    w = np.ones((1, 1, 1, 1, 1), np.float32)
    np.testing.assert_array_equal(K.conv3d_fwd(xpad, w, (1, 1, 1)), xpad)


@pytest.mark.gpu
def test_backend_agrees_with_oracle(precision):
    """fp32 mode: within 1e-5 of the reference kernels (their fwd/bwd
    cross-backend tolerance is 1e-6 on reductions of identical order; ours
    accumulates in a different order).  tf32 mode: the north-star rtol 1e-3
    against the TF32-emulating oracle (operands rounded to nearest TF32 as the
    device frames and weight packs do, fp64 accumulation, the data gradient
    stored rounded), and 1e-3 against the plain fp32 kernels as well."""
    tol = 1e-5 if precision == "fp32" else 1e-3
    R = O.tf32_round

    def emu(fn, a, b, *rest, rnd_out=True):
        out = fn(R(a).astype(np.float64), R(b).astype(np.float64), *rest).astype(np.float32)
        return R(out) if rnd_out else out

    for xpad, w, stride in _cases():
        y_o = O.k_conv3d_fwd(xpad, w, stride)
        y = K.conv3d_fwd(xpad, w, stride)
        assert y.shape == y_o.shape and y.dtype == np.float32
        assert _scaled_err(y, y_o) < tol, ("fwd", xpad.shape, stride, _scaled_err(y, y_o))

        u = (y_o + np.float32(0.5)).astype(np.float32)
        g_o = O.k_conv3d_bwd_data(u, w, stride, xpad.shape[2:])
        g = K.conv3d_bwd_data(u, w, stride, xpad.shape[2:])
        assert g.shape == g_o.shape
        assert _scaled_err(g, g_o) < tol, ("bwd_data", xpad.shape, stride, _scaled_err(g, g_o))

        f_o = O.k_conv3d_bwd_filter(xpad, u, stride, w.shape[2:])
        f = K.conv3d_bwd_filter(xpad, u, stride, w.shape[2:])
        assert f.shape == f_o.shape
        assert _scaled_err(f, f_o) < tol, ("bwd_filter", xpad.shape, stride, _scaled_err(f, f_o))
        if precision == "tf32":
            for name, got, ref in (
                    ("fwd", y, emu(O.k_conv3d_fwd, xpad, w, stride)),
                    ("bwd_data", g, emu(O.k_conv3d_bwd_data, u, w, stride, xpad.shape[2:])),
                    ("bwd_filter", f, emu(O.k_conv3d_bwd_filter, xpad, u, stride, w.shape[2:], rnd_out=False))):
                assert _scaled_err(got, ref) < 1e-3, (name, "tf32-emulated", xpad.shape, stride,
                                                      _scaled_err(got, ref))


@pytest.mark.gpu
def test_device_buffers_stay_on_device():
    import torch

    xpad, w, stride = _cases()[0]
    y_host = K.conv3d_fwd(xpad, w, stride)
    y_dev = K.conv3d_fwd(torch.from_numpy(xpad).cuda(), torch.from_numpy(w).cuda(), stride)
    assert y_dev.is_cuda
    np.testing.assert_array_equal(y_dev.cpu().numpy(), y_host)
