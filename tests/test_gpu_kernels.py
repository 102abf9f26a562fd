"""Kernel-level parity of every C-ABI entry point against the float64 oracle
(numpy), on the edge cases the reference tests: ragged clients, tail
batches, zero epochs, proximal term, norm exactly at the bound, non-finite
updates, noise statistics and determinism."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import port
from paper_2404_06430_b200 import native
from tests.conftest import assert_close_fp32

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


_KEEP: list = []  # device copies must outlive the (async) kernel launches that use them


def dev(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    t = t.cuda()
    _KEEP.append(t)
    return t


@pytest.fixture(autouse=True)
def _release_kept():
    yield
    torch.cuda.synchronize()
    _KEEP.clear()


def S():
    return native.stream_handle()


def cohort(rng, sizes, dim, k, epochs, seed0=0):
    X = rng.normal(size=(sum(sizes), dim))
    y = rng.integers(0, k, size=sum(sizes))
    starts = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
    perms = [np.concatenate([np.random.default_rng(seed0 + i * 7 + e).permutation(n) for e in range(epochs)])
             if epochs else np.zeros(0, np.int64) for i, n in enumerate(sizes)]
    perm_off = np.concatenate([[0], np.cumsum([len(p) for p in perms])[:-1]]).astype(np.int64)
    flat = np.concatenate(perms).astype(np.int32) if epochs else np.zeros(1, np.int32)
    return X, y, starts, np.array(sizes, np.int32), flat, perm_off, perms


def fit_sgd(kind, dims, theta, X, y, starts, sizes, flat, perm_off, epochs, B, lr, mu=0.0):
    C = len(sizes)
    D = theta.size
    ld = (D + 3) & ~3
    delta = torch.zeros(C, ld, device="cuda")
    bad = torch.zeros(C, dtype=torch.int32, device="cuda")
    tX, ty = dev(X.astype(np.float32)), dev(y.astype(np.int32))
    native.call(f"fb_local_sgd_{kind}_f32", dev(theta.astype(np.float32)).data_ptr(), *dims, tX.data_ptr(),
                ty.data_ptr(), dev(starts).data_ptr(), dev(sizes).data_ptr(), dev(flat).data_ptr(),
                dev(perm_off).data_ptr(), C, epochs, B, lr, mu, None, 0, delta.data_ptr(), ld, bad.data_ptr(), S())
    return delta[:, :D].double().cpu().numpy(), bad.cpu().numpy()


@pytest.mark.parametrize("kind", ["linear", "mlp"])
@pytest.mark.parametrize("epochs,B,mu", [(1, 10, 0.0), (2, 7, 0.0), (0, 5, 0.0), (1, 4, 0.3), (3, 64, 0.0)])
def test_local_sgd_matches_oracle(kind, epochs, B, mu):
    rng = np.random.default_rng(epochs * 10 + B)
    dim, h, k = 32, 64, 10
    sizes = [1, 7, 23, 50, 13, 64]
    X, y, starts, nrows, flat, perm_off, perms = cohort(rng, sizes, dim, k, epochs)
    model = port.Mlp(dim, h, k) if kind == "mlp" else port.Linear(dim, k)
    theta_d = model.init(5) if kind == "mlp" else {n: rng.normal(scale=0.1, size=s) for n, s in model.dims.items()}
    theta = port.flat(theta_d, model.dims)
    dims = (dim, h, k) if kind == "mlp" else (dim, k)
    X32 = X.astype(np.float32).astype(np.float64)  # both sides see fp32-rounded features
    got, bad = fit_sgd(kind, dims, theta, X, y, starts, nrows, flat, perm_off, epochs, B, 0.1, mu)
    assert not bad.any()
    for c, n in enumerate(sizes):
        rows = slice(starts[c], starts[c] + n)
        pm = perms[c].reshape(epochs, n) if epochs else np.zeros((0, n), np.int64)
        after = port.fit_local(model, theta_d, X32[rows], y[rows], pm, 0.1, B, mu=mu)
        ref = theta - port.flat(after, model.dims)
        if epochs == 0:
            assert np.all(got[c] == 0)
        else:
            assert_close_fp32(got[c], ref, rtol=1e-4, what=f"{kind} client {c} n={n}")


@pytest.mark.parametrize("kind", ["linear", "mlp"])
def test_eval_matches_oracle(kind):
    rng = np.random.default_rng(3)
    dim, h, k = 32, 64, 10
    sizes = [1, 31, 32, 33, 100, 5]
    X, y, starts, nrows, *_ = cohort(rng, sizes, dim, k, 0)
    model = port.Mlp(dim, h, k) if kind == "mlp" else port.Linear(dim, k)
    theta_d = {n: rng.normal(scale=0.3, size=s) for n, s in model.dims.items()}
    theta = port.flat(theta_d, model.dims)
    C = len(sizes)
    loss = torch.zeros(C, dtype=torch.float64, device="cuda")
    corr = torch.zeros(C, dtype=torch.int32, device="cuda")
    dims = (dim, h, k) if kind == "mlp" else (dim, k)
    native.call(f"fb_eval_{kind}_f32", dev(theta.astype(np.float32)).data_ptr(), *dims,
                dev(X.astype(np.float32)).data_ptr(), dev(y.astype(np.int32)).data_ptr(), dev(starts).data_ptr(),
                dev(nrows).data_ptr(), C, loss.data_ptr(), corr.data_ptr(), S())
    X32 = X.astype(np.float32).astype(np.float64)
    for c, n in enumerate(sizes):
        rows = slice(starts[c], starts[c] + n)
        ls, cr = model.eval_counts(theta_d, X32[rows], y[rows])
        assert loss[c].item() == pytest.approx(ls, rel=1e-5)
        assert abs(corr[c].item() - cr) <= 1  # argmax may flip on a near-tie in fp32


def _clip_call(delta, w, bound, ld=None):
    C, D = delta.shape
    ld = ld or D
    buf = torch.zeros(C, ld, device="cuda")
    buf[:, :D] = dev(delta.astype(np.float32))
    norm = torch.zeros(C, dtype=torch.float64, device="cuda")
    coef = torch.zeros(C, device="cuda")
    clipped = torch.zeros(C, dtype=torch.int32, device="cuda")
    bad = torch.zeros(C, dtype=torch.int32, device="cuda")
    wsb = native.call("fb_clip_workspace_bytes", C, D)
    ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device="cuda")
    native.call("fb_delta_norm_clip_f32", buf.data_ptr(), ld, C, D, dev(w.astype(np.float32)).data_ptr(), bound,
                norm.data_ptr(), coef.data_ptr(), clipped.data_ptr(), bad.data_ptr(), ws.data_ptr(), ws.numel(), S())
    return buf, norm.cpu().numpy(), coef.cpu().numpy(), clipped.cpu().numpy(), bad.cpu().numpy()


@pytest.mark.parametrize("D,ld", [(1, 4), (330, 332), (2762, 2764), (100_003, 100_004), (1_626_442, 1_626_444)])
def test_delta_norm_clip_and_weighted_sum(D, ld):
    rng = np.random.default_rng(D)
    C = 37
    delta = rng.normal(size=(C, D)) * np.where(rng.random(C) < 0.5, 1e-4, 1.0)[:, None] / np.sqrt(D)
    w = rng.integers(1, 60, size=C).astype(np.float64)
    bound = 0.9
    buf, norm, coef, clipped, bad = _clip_call(delta, w, bound, ld)
    d32 = delta.astype(np.float32).astype(np.float64)
    ref_norm = np.linalg.norm(w[:, None] * d32, axis=1)
    np.testing.assert_allclose(norm, ref_norm, rtol=1e-9)
    ref_clip = ref_norm > bound
    np.testing.assert_array_equal(clipped.astype(bool), ref_clip)
    ref_coef = w * np.where(ref_clip, bound / ref_norm, 1.0)
    np.testing.assert_allclose(coef, ref_coef, rtol=1e-6)
    assert not bad.any()
    agg = torch.zeros(D, device="cuda")
    wsb = native.call("fb_weighted_sum_workspace_bytes", C, D)
    ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device="cuda")
    native.call("fb_weighted_sum_f32", buf.data_ptr(), ld, C, D, dev(coef.astype(np.float32)).data_ptr(),
                agg.data_ptr(), 0, ws.data_ptr(), ws.numel(), S())
    ref = (ref_coef[:, None] * d32).sum(axis=0)
    assert_close_fp32(agg.double().cpu().numpy(), ref)


def test_clip_exactly_at_bound_is_not_clipped():
    """clip only if norm > S (fedsim/privacy/clipping.py:49)."""
    delta = np.array([[0.5, 0.5, 0.5, 0.5], [3.0, 4.0, 0.0, 0.0], [0.0, 0.0, 0.0, 0.0]])  # exact in fp32
    _, norm, coef, clipped, _ = _clip_call(delta, np.ones(3), 1.0)
    np.testing.assert_array_equal(clipped, [0, 1, 0])
    np.testing.assert_allclose(coef, [1.0, 0.2, 1.0], rtol=1e-7)
    np.testing.assert_allclose(norm, [1.0, 5.0, 0.0], rtol=1e-7)


def test_nonfinite_delta_flagged():
    delta = np.ones((3, 10))
    delta[1, 4] = np.inf
    delta[2, 0] = np.nan
    *_, bad = _clip_call(delta, np.ones(3), 1.0)
    np.testing.assert_array_equal(bad, [0, 1, 1])


def test_weighted_sum_accumulate_and_empty():
    D = 1000
    agg = torch.ones(D, device="cuda")
    native.call("fb_weighted_sum_f32", None, D, 0, D, None, agg.data_ptr(), 1, None, 0, S())
    assert torch.all(agg == 1)
    native.call("fb_weighted_sum_f32", None, D, 0, D, None, agg.data_ptr(), 0, None, 0, S())
    assert torch.all(agg == 0)


def test_sumsq():
    x = np.random.default_rng(0).normal(size=3_000_001).astype(np.float32)
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    ws = torch.empty(8192, dtype=torch.uint8, device="cuda")
    native.call("fb_sumsq_f32", dev(x).data_ptr(), x.size, out.data_ptr(), ws.data_ptr(), ws.numel(), S())
    assert out.item() == pytest.approx(float((x.astype(np.float64) ** 2).sum()), rel=1e-12)


def test_gaussian_statistics_and_determinism():
    n = 4_000_000
    out = torch.empty(n, device="cuda")
    std = 0.02
    native.call("fb_gaussian_f32", out.data_ptr(), n, std, 12345, 0, 0, S())
    z = out.double().cpu().numpy()
    assert abs(z.mean()) <= 3 * std / np.sqrt(n)
    assert abs(z.std() - std) <= 3 * std / np.sqrt(2 * n)
    # higher moments of a normal: kurtosis 3
    assert abs(((z / std) ** 4).mean() - 3.0) < 0.02
    again = torch.empty(n, device="cuda")
    native.call("fb_gaussian_f32", again.data_ptr(), n, std, 12345, 0, 0, S())
    assert torch.equal(out, again)
    # counter-based: a slice drawn at an offset equals the same slice of the full draw
    part = torch.empty(1000, device="cuda")
    native.call("fb_gaussian_f32", part.data_ptr(), 1000, std, 12345, 4000, 0, S())
    assert torch.equal(part, out[4000:5000])
    other = torch.empty(n, device="cuda")
    native.call("fb_gaussian_f32", other.data_ptr(), n, std, 12346, 0, 0, S())
    assert abs(np.corrcoef(z[:100000], other.double().cpu().numpy()[:100000])[0, 1]) < 0.02


@pytest.mark.parametrize("D", [5, 2762, 1_626_442])
def test_noise_avg_sgd(D):
    rng = np.random.default_rng(D)
    theta = rng.normal(size=D).astype(np.float32)
    agg = rng.normal(size=D).astype(np.float32)
    inj = rng.normal(scale=0.1, size=D).astype(np.float32)
    t = dev(theta)
    native.call("fb_noise_avg_sgd_f32", t.data_ptr(), dev(agg).data_ptr(), D, 0.0, 0, dev(inj).data_ptr(),
                1.0 / 50, 0.7, None, S())
    ref = theta.astype(np.float64) - 0.7 * (agg.astype(np.float64) + inj) / 50
    assert_close_fp32(t.double().cpu().numpy(), ref)
    # philox path: fused result == materialized noise + same step
    t2 = dev(theta)
    out_agg = torch.empty(D, device="cuda")
    native.call("fb_noise_avg_sgd_f32", t2.data_ptr(), dev(agg).data_ptr(), D, 0.05, 99, None, 1.0 / 50, 0.7,
                out_agg.data_ptr(), S())
    noise = torch.empty(D, device="cuda")
    native.call("fb_gaussian_f32", noise.data_ptr(), D, 0.05, 99, 0, 0, S())
    a2 = dev(agg)
    native.call("fb_gaussian_f32", a2.data_ptr(), D, 0.05, 99, 0, 1, S())
    assert torch.equal(out_agg, a2)
    ref2 = theta.astype(np.float64) - 0.7 * out_agg.double().cpu().numpy() / 50
    assert_close_fp32(t2.double().cpu().numpy(), ref2)


@pytest.mark.parametrize("D", [7, 2762, 1_626_442])
def test_noise_avg_adam_matches_oracle(D):
    """fb_noise_avg_adam_f32 over 4 steps vs the float64 AdamOptimizer
    restatement (fedsim/models/optimizers.py:24-68), injected noise."""
    from oracle import port

    rng = np.random.default_rng(D + 1)
    theta = rng.normal(size=D).astype(np.float32)
    t, m, v = dev(theta), torch.zeros(D, device="cuda"), torch.zeros(D, device="cuda")
    ref, st = theta.astype(np.float64), {}
    for k in range(1, 5):
        agg = rng.normal(size=D).astype(np.float32)
        inj = rng.normal(scale=0.1, size=D).astype(np.float32)
        native.call("fb_noise_avg_adam_f32", t.data_ptr(), m.data_ptr(), v.data_ptr(), dev(agg).data_ptr(), D, 0.0, 0,
                    dev(inj).data_ptr(), 1.0 / 20, 0.05, 0.9, 0.99, 0.1, k, None, S())
        ref = port.central_adam(ref, agg.astype(np.float64), 20.0, 0.05, st, 0.9, 0.99, 0.1,
                                noise=inj.astype(np.float64))
        assert_close_fp32(t.double().cpu().numpy(), ref, what=f"adam step {k}")
    with pytest.raises(ValueError, match="step >= 1"):
        native.call("fb_noise_avg_adam_f32", t.data_ptr(), m.data_ptr(), v.data_ptr(), t.data_ptr(), D, 0.0, 0, None,
                    1.0, 0.1, 0.9, 0.99, 0.1, 0, None, S())


def test_scaffold_kernels():
    """correction / payload / scatter against numpy (fedsim/algorithms/scaffold.py:46-79)."""
    rng = np.random.default_rng(3)
    C, D, ld, lds = 5, 37, 40, 44
    server = rng.normal(size=D).astype(np.float32)
    store = rng.normal(size=(4, lds)).astype(np.float32)
    rows = np.array([2, -1, 0, 3, -1], dtype=np.int32)
    u = np.where(rows[:, None] >= 0, store[np.maximum(rows, 0), :D], 0.0)
    corr = torch.zeros(C, ld, device="cuda")
    d_store, d_rows = dev(store), dev(rows)
    native.call("fb_scaffold_correction_f32", dev(server).data_ptr(), d_store.data_ptr(), lds, d_rows.data_ptr(), C, D,
                corr.data_ptr(), ld, S())
    np.testing.assert_array_equal(corr.cpu().numpy()[:, :D], (server[None, :] - u).astype(np.float32))
    delta = rng.normal(size=(C, ld)).astype(np.float32)
    scale = rng.uniform(1, 3, size=C).astype(np.float32)
    pay = torch.zeros(C, 2 * D + 2, device="cuda")
    newc = torch.zeros(C, ld, device="cuda")
    native.call("fb_scaffold_payload_f32", dev(delta).data_ptr(), ld, dev(server).data_ptr(), d_store.data_ptr(), lds,
                d_rows.data_ptr(), dev(scale).data_ptr(), C, D, pay.data_ptr(), 2 * D + 2, newc.data_ptr(), ld, S())
    ds = delta[:, :D] * scale[:, None]
    np.testing.assert_allclose(pay.cpu().numpy()[:, :D], delta[:, :D])
    np.testing.assert_allclose(pay.cpu().numpy()[:, D:2 * D], ds - server[None, :], rtol=1e-6, atol=1e-6)
    np.testing.assert_allclose(newc.cpu().numpy()[:, :D], (u - server[None, :]) + ds, rtol=1e-6, atol=1e-6)
    tgt = torch.zeros(6, lds, device="cuda")
    native.call("fb_scatter_rows_f32", tgt.data_ptr(), lds, dev(np.array([4, 1], dtype=np.int32)).data_ptr(),
                newc.data_ptr(), ld, 2, D, S())
    np.testing.assert_array_equal(tgt.cpu().numpy()[[4, 1], :D], newc.cpu().numpy()[:2, :D])


def test_delta_norm_clip_ex_matches_full_scan():
    """K2 with a skipped column range plus its precomputed squares == the full scan."""
    rng = np.random.default_rng(11)
    C, D, ld = 37, 5003, 5004
    lo, hi = 1000, 4000
    delta = rng.normal(size=(C, ld)).astype(np.float32)
    w = rng.uniform(0.5, 2.0, size=C).astype(np.float32)
    d = dev(delta)
    extra = dev(np.square(delta[:, lo:hi].astype(np.float64)).sum(axis=1))
    outs = []
    for ex in (False, True):
        norm = torch.zeros(C, dtype=torch.float64, device="cuda")
        coef = torch.zeros(C, device="cuda")
        clipped = torch.zeros(C, dtype=torch.int32, device="cuda")
        bad = torch.zeros(C, dtype=torch.int32, device="cuda")
        wsb = native.call("fb_clip_workspace_bytes", C, D) + 16 * C
        ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
        if ex:
            native.call("fb_delta_norm_clip_ex_f32", d.data_ptr(), ld, C, D, lo, hi, extra.data_ptr(), dev(w).data_ptr(),
                        50.0, norm.data_ptr(), coef.data_ptr(), clipped.data_ptr(), bad.data_ptr(), ws.data_ptr(), wsb,
                        S())
        else:
            native.call("fb_delta_norm_clip_f32", d.data_ptr(), ld, C, D, dev(w).data_ptr(), 50.0, norm.data_ptr(),
                        coef.data_ptr(), clipped.data_ptr(), bad.data_ptr(), ws.data_ptr(), wsb, S())
        outs.append((norm.cpu().numpy(), coef.cpu().numpy(), clipped.cpu().numpy()))
    np.testing.assert_allclose(outs[1][0], outs[0][0], rtol=1e-13)
    np.testing.assert_allclose(outs[1][1], outs[0][1], rtol=1e-6)
    np.testing.assert_array_equal(outs[1][2], outs[0][2])
    with pytest.raises(ValueError, match="skip"):
        native.call("fb_delta_norm_clip_ex_f32", d.data_ptr(), ld, C, D, 10, 5, None, dev(w).data_ptr(), 1.0,
                    None, None, None, None, None, 0, S())


def test_bad_arguments_raise_value_error():
    with pytest.raises(ValueError, match="bad shape"):
        native.call("fb_delta_norm_clip_f32", None, 2, 1, 4, None, 1.0, None, None, None, None, None, 0, S())
