"""Pin the CPU oracle against the reference (golden vectors + the reference's
own compiled kernels).  CPU only."""

import json

import numpy as np
import pytest

from oracle import build_oracle, serial as O


def _load(golden, name):
    return np.load(golden / name, allow_pickle=False)


def test_prng_matches_reference(golden):
    g = json.loads((golden / "prng.json").read_text())
    for k, v in g["key_fold"].items():
        key = json.loads(k)
        assert O.key_fold(key) == int(v)
        assert [int(x) for x in O.u64(key, 16)] == [int(x) for x in g["u64"][k]]
        assert O.uniform(key, 16, -0.5, 2.0).tolist() == g["uniform"][k]
        assert O.randint(key, 16, 0, 7).tolist() == g["randint"][k]
        assert O.permutation(key, 12).tolist() == g["permutation"][k]
    big = O.uniform([0, -3, 0], 1 << 20, -1.0, 1.0)
    assert big[:8].tolist() == g["uniform_1M_head"]
    import hashlib

    assert hashlib.sha256(big.astype(np.float32).tobytes()).hexdigest() == g["uniform_1M_f32_bytes_sha"]


@pytest.mark.parametrize("dt", ["float32", "float64"])
@pytest.mark.parametrize("case", [0, 1, 2])
def test_oracle_conv_matches_reference_vectors(golden, dt, case):
    A = _load(golden, "kernels.npz")
    t = f"{dt}_{case}"
    n, cin, cout, d, h, w, k, s = A[f"meta_{t}"]
    x, wt, u = A[f"x_{t}"], A[f"w_{t}"], A[f"u_{t}"]
    y = O.conv3d(x, wt, (k,) * 3, (s,) * 3)
    # forward: same accumulation order as the reference -> bit-identical
    assert np.array_equal(y, A[f"y_{t}"])
    xg = O.conv3d_bwd_data(u, wt, (k,) * 3, (s,) * 3, x.shape[2:])
    wg = O.conv3d_bwd_filter(x, u, (k,) * 3, (s,) * 3)
    tol = 1e-5 if dt == "float32" else 1e-12  # fixtures came from the BLAS (numpy) backend
    for got, ref in ((xg, A[f"xg_{t}"]), (wg, A[f"wg_{t}"])):
        assert np.max(np.abs(got - ref)) <= tol * np.max(np.abs(ref))


@pytest.mark.skipif(build_oracle.build_reference_kernels() is None, reason="reference kernels not built")
@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_oracle_conv_bitwise_equals_reference_cython(dt):
    """oracle/conv_oracle.c == the reference's own _hot.pyx build, bit for bit."""
    ref = O.ref_kernels()
    rng = np.random.default_rng(5)
    for (n, cin, cout, d, h, w, k, s) in [(2, 3, 5, 7, 6, 9, 3, 1), (1, 4, 4, 8, 8, 8, 3, 2), (1, 2, 3, 4, 5, 6, 1, 1)]:
        xp = rng.standard_normal((n, cin, d + k - 1, h + k - 1, w + k - 1)).astype(dt)
        wt = rng.standard_normal((cout, cin, k, k, k)).astype(dt)
        y = O.k_conv3d_fwd(xp, wt, (s,) * 3)
        y2 = np.zeros_like(y)
        ref.conv3d_fwd(xp, wt, s, s, s, y2)
        assert np.array_equal(y, y2)
        u = rng.standard_normal(y.shape).astype(dt)
        g = O.k_conv3d_bwd_data(u, wt, (s,) * 3, xp.shape[2:])
        g2 = np.zeros_like(xp)
        ref.conv3d_bwd_data(u, wt, s, s, s, g2)
        assert np.array_equal(g, g2)
        wg = O.k_conv3d_bwd_filter(xp, u, (s,) * 3, (k,) * 3)
        wg2 = np.zeros_like(wt)
        ref.conv3d_bwd_filter(xp, u, s, s, s, wg2)
        assert np.array_equal(wg, wg2)


def test_oracle_layers_match_reference(golden):
    A = _load(golden, "layers.npz")
    x = A["pool_x"]
    for kind in ("average", "max"):
        assert np.array_equal(O.pool3d(x, kind), A[f"pool_{kind}_y"])
        assert np.allclose(O.pool3d_bwd(x, A[f"pool_{kind}_u"], kind), A[f"pool_{kind}_g"], rtol=0, atol=1e-15)
    st = O.BN(A["bn_gamma"].copy(), A["bn_beta"].copy(), np.float64)
    y, cache = O.batchnorm_fwd(A["bn_x"], st)
    assert np.allclose(y, A["bn_y"], rtol=1e-13, atol=1e-13)
    dx, dg, db = O.batchnorm_bwd(A["bn_u"], st, cache)
    for a, b in ((dx, "bn_dx"), (dg, "bn_dg"), (db, "bn_db"), (st.running_mean, "bn_rm"), (st.running_var, "bn_rv")):
        assert np.allclose(a, A[b], rtol=1e-12, atol=1e-12)
    assert np.array_equal(O.leaky(A["leaky_x"], 0.3), A["leaky_y"])
    assert np.array_equal(O.leaky_bwd(A["leaky_x"], A["leaky_u"], 0.3), A["leaky_g"])
    assert np.allclose(O.deconv3d(A["deconv_x"], A["deconv_w"]), A["deconv_y"], rtol=1e-12, atol=1e-12)
    assert np.allclose(O.deconv3d_bwd_data(A["deconv_u"], A["deconv_w"]), A["deconv_g"], rtol=1e-12, atol=1e-12)
    assert np.allclose(O.deconv3d_bwd_filter(A["deconv_x"], A["deconv_u"]), A["deconv_wg"], rtol=1e-12, atol=1e-12)
    loss, g = O.cross_entropy(A["xent_logits"], A["xent_labels"])
    assert abs(loss - float(A["xent_loss"])) < 1e-14 and np.allclose(g, A["xent_g"], rtol=1e-13, atol=1e-15)
    ml, mg = O.mse(A["mse_pred"], A["mse_target"])
    assert ml == float(A["mse_loss"]) and np.array_equal(mg, A["mse_g"])
    assert np.array_equal(O.dropout_mask([0, 1, 2, 3, 4], 64, 0.8), A["dropout_mask"])


def _sample(a, k=48):
    a = np.asarray(a).ravel()
    idx = np.linspace(0, a.size - 1, num=min(k, a.size)).astype(np.int64)
    return np.concatenate([[a.sum(), (a * a).sum(), np.abs(a).max()], a[idx]])


@pytest.mark.parametrize("tag", ["cf32_f64", "cf32bn_f64", "un16_f64"])
def test_oracle_network_step_matches_reference(golden, tag):
    """Serial oracle train step == reference serial step (fp64: 1e-10 rel)."""
    from paper_2007_12856_b200.networks import build_cosmoflow, build_unet_mini

    A = _load(golden, "nets.npz")
    net = {"cf32_f64": build_cosmoflow(32), "cf32bn_f64": build_cosmoflow(32, with_bn=True),
           "un16_f64": build_unet_mini(16)}[tag]
    wi = 16 if tag.startswith("un") else 32
    x, y, ids = O.synthetic_batch(net, wi, 2, 0, np.float64)
    params = O.init_params(net, 0, np.float64)
    states = O.make_bn_states(net, params, np.float64)
    trace, grads = {}, {}
    opt = O.Adam(params)
    loss = O.train_step(net, params, states, opt, 1e-3, x, y, ids, (0, 0, 0), trace=trace, grads_out=grads)
    assert abs(loss - float(A[f"{tag}_loss"])) <= 1e-12 * abs(float(A[f"{tag}_loss"]))
    for (ph, name), v in trace.items():
        ref = A[f"{tag}_tr_{ph}_{name}"]
        got = _sample(v)
        assert np.max(np.abs(got - ref)) <= 1e-10 * max(1e-300, np.max(np.abs(ref))), (ph, name)
    for name, g in grads.items():
        ref = A[f"{tag}_grad_{name}"]
        assert np.max(np.abs(_sample(g) - ref)) <= 1e-10 * max(1e-300, np.max(np.abs(ref))), name
    for name, p in params.items():
        ref = A[f"{tag}_param1_{name}"]
        assert np.max(np.abs(_sample(p) - ref)) <= 1e-10 * max(1e-300, np.max(np.abs(ref))), name


def test_tf32_round_matches_device_rule():
    """oracle.serial.tf32_round is the device's vpx::tf32_rn: nearest TF32,
    ties away from zero, carry into the exponent."""
    bits = np.array([0x3F800000, 0x3F800FFF, 0x3F801000, 0x3F802000, 0xBF801000, 0x3FFFF000, 0x00000000,
                     0x7F7FF000], dtype=np.uint32)
    got = O.tf32_round(bits.view(np.float32)).view(np.uint32)
    want = np.array([0x3F800000, 0x3F800000, 0x3F802000, 0x3F802000, 0xBF802000, 0x40000000, 0x00000000,
                     0x7F800000], dtype=np.uint32)
    np.testing.assert_array_equal(got, want)
    x = np.random.default_rng(0).normal(size=4096).astype(np.float32)
    r = O.tf32_round(x)
    assert np.all(r.view(np.uint32) & 0x1FFF == 0)
    assert np.max(np.abs(r - x) / np.abs(x)) <= 2.0 ** -11


@pytest.mark.parametrize("which", ["cosmoflow32bn", "unet16"])
@pytest.mark.parametrize("tf32", [False, True])
def test_layerwise_oracle_reproduces_its_own_trace(which, tf32):
    """Teacher forcing (oracle.serial.layerwise) fed the oracle's OWN trace
    must give that trace back bit for bit, layer by layer and for every
    parameter gradient: the per-layer GPU parity test relies on it."""
    from paper_2007_12856_b200.networks import build_cosmoflow, build_unet_mini

    net, wi = (build_unet_mini(16), 16) if which == "unet16" else (build_cosmoflow(32, with_bn=True), 32)
    x, y, ids = O.synthetic_batch(net, wi, 2, 0, np.float32)
    runs = []
    for _ in range(2):
        p = O.init_params(net, 0, np.float32)
        runs.append((p, O.make_bn_states(net, p, np.float32)))
    num = O.TF32() if tf32 else None
    tr, gr = {}, {}
    pred, stash = O.forward(net, runs[0][0], runs[0][1], x, "train", (0, 0, 0), ids, trace=tr, num=num)
    _, dpred = O.loss_and_grad(net, pred, y, num)
    gr = O.backward(net, runs[0][0], runs[0][1], stash, dpred, trace=tr, num=num)
    lt, lg = O.layerwise(net, runs[1][0], runs[1][1], x, y, tr, ids, (0, 0, 0), num=num)
    assert set(lt) == set(tr) and set(lg) == set(gr)
    for k in tr:
        np.testing.assert_array_equal(np.asarray(lt[k]), np.asarray(tr[k]), err_msg=str(k))
    for k in gr:
        np.testing.assert_array_equal(lg[k], gr[k], err_msg=k)
