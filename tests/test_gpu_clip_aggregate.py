"""Fused K2 + K3 (fb_clip_aggregate_f32: norm, clip factor and weighted sum in
one HBM pass) against float64 numpy and against the two-kernel path
(fb_delta_norm_clip_f32 + fb_weighted_sum_f32), on the reference's clip
semantics (fedsim/privacy/clipping.py:37-56: norm of the weight-premultiplied
update, strict >, factor S/norm) and aggregation (fedsim/engine/aggregator.py:
39-44).  Shapes cover a ragged tail column quad, one client, the 64-client
fp32 block boundary (63/64/65/130), the CNN's D and configs[4]'s D = 10M."""

from __future__ import annotations

import numpy as np
import pytest

from paper_2404_06430_b200 import native
from tests.conftest import assert_close_fp32

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def S():
    return native.stream_handle()


def fused(buf, ld, C, D, w, bound, agg=None, accumulate=0):
    norm = torch.zeros(C, dtype=torch.float64, device="cuda")
    coef = torch.zeros(C, device="cuda")
    clipped = torch.zeros(C, dtype=torch.int32, device="cuda")
    bad = torch.zeros(C, dtype=torch.int32, device="cuda")
    if agg is None:
        agg = torch.full((D,), float("nan"), device="cuda")  # overwritten, never read (accumulate=0)
    ws = torch.empty(max(native.call("fb_clip_aggregate_workspace_bytes", C, D), 16), dtype=torch.uint8,
                     device="cuda")
    native.call("fb_clip_aggregate_f32", buf.data_ptr(), ld, C, D, w.data_ptr(), bound, norm.data_ptr(),
                coef.data_ptr(), clipped.data_ptr(), bad.data_ptr(), agg.data_ptr(), accumulate, ws.data_ptr(),
                ws.numel(), S())
    torch.cuda.synchronize()
    return (agg.double().cpu().numpy(), norm.cpu().numpy(), coef.cpu().numpy(), clipped.cpu().numpy(),
            bad.cpu().numpy())


def two_pass(buf, ld, C, D, w, bound):
    norm = torch.zeros(C, dtype=torch.float64, device="cuda")
    coef = torch.zeros(C, device="cuda")
    clipped = torch.zeros(C, dtype=torch.int32, device="cuda")
    bad = torch.zeros(C, dtype=torch.int32, device="cuda")
    ws = torch.empty(max(native.call("fb_clip_workspace_bytes", C, D), 16), dtype=torch.uint8, device="cuda")
    native.call("fb_delta_norm_clip_f32", buf.data_ptr(), ld, C, D, w.data_ptr(), bound, norm.data_ptr(),
                coef.data_ptr(), clipped.data_ptr(), bad.data_ptr(), ws.data_ptr(), ws.numel(), S())
    agg = torch.zeros(D, device="cuda")
    ws2 = torch.empty(max(native.call("fb_weighted_sum_workspace_bytes", C, D), 16), dtype=torch.uint8,
                      device="cuda")
    native.call("fb_weighted_sum_f32", buf.data_ptr(), ld, C, D, coef.data_ptr(), agg.data_ptr(), 0,
                ws2.data_ptr(), ws2.numel(), S())
    torch.cuda.synchronize()
    return agg.double().cpu().numpy(), norm.cpu().numpy(), coef.cpu().numpy(), clipped.cpu().numpy()


def make(C, D, seed, ld=None):
    ld = ld or (D + 3) & ~3
    g = torch.Generator(device="cuda").manual_seed(seed)
    buf = torch.randn(C, ld, device="cuda", generator=g) * (1.0 / np.sqrt(D))
    scale = torch.where(torch.rand(C, device="cuda", generator=g) < 0.5, 1e-4, 1.0)
    buf *= scale[:, None]
    if ld > D:
        buf[:, D:] = float("nan")  # padding columns must never be read into a result
    w = torch.randint(1, 60, (C,), device="cuda", generator=g).float()
    return buf, ld, w


@pytest.mark.parametrize("C,D", [(1, 5), (3, 2049), (63, 2762), (64, 100_003), (65, 100_003), (130, 331_777),
                                 (37, 1_626_442)])
def test_fused_matches_float64(C, D):
    buf, ld, w = make(C, D, seed=C * 7 + D)
    bound = 0.9
    agg, norm, coef, clipped, bad = fused(buf, ld, C, D, w, bound)
    d = buf[:, :D].double().cpu().numpy()
    wn = w.double().cpu().numpy()
    ref_norm = np.linalg.norm(wn[:, None] * d, axis=1)
    np.testing.assert_allclose(norm, ref_norm, rtol=1e-9)
    ref_clip = ref_norm > bound
    np.testing.assert_array_equal(clipped.astype(bool), ref_clip)
    ref_coef = wn * np.where(ref_clip, bound / ref_norm, 1.0)
    np.testing.assert_allclose(coef, ref_coef, rtol=1e-6)
    assert not bad.any()
    assert_close_fp32(agg, (coef.astype(np.float64)[:, None] * d).sum(axis=0), what="fused aggregate")
    # and the same decisions / near-identical sums as the two-kernel path (fp64 norms
    # summed in a different order: equal to ~1 ulp)
    agg2, norm2, coef2, clipped2 = two_pass(buf, ld, C, D, w, bound)
    np.testing.assert_allclose(norm, norm2, rtol=1e-14)
    np.testing.assert_allclose(coef, coef2, rtol=1.2e-7)
    np.testing.assert_array_equal(clipped, clipped2)
    assert_close_fp32(agg, agg2, what="fused vs two-pass")


def test_fused_at_configs4_shape_and_deterministic():
    """D = 10M (configs[4]), 96 clients (one fp64 block flush): float64 check
    by a column sample, bitwise rerun equality."""
    C, D = 96, 10_000_000
    buf, ld, w = make(C, D, seed=4)
    w.fill_(1.0)
    agg, norm, coef, clipped, _ = fused(buf, ld, C, D, w, 1.0)
    agg_b, *_ = fused(buf, ld, C, D, w, 1.0)
    np.testing.assert_array_equal(agg, agg_b)
    cols = np.sort(np.random.default_rng(0).choice(D, 200_000, replace=False))
    cols = np.concatenate([cols, np.arange(D - 4099, D)])  # the last CTA's slice and the ragged tail
    d = buf[:, torch.from_numpy(cols).cuda()].double().cpu().numpy()
    full_norm = torch.linalg.vector_norm(buf[:, :D].double(), dim=1).cpu().numpy()
    np.testing.assert_allclose(norm, full_norm, rtol=1e-9)
    assert_close_fp32(agg[cols], (coef.astype(np.float64)[:, None] * d).sum(axis=0), what="configs[4] aggregate")
    assert 0 < clipped.sum() < C


def test_fused_exact_bound_nonfinite_and_accumulate():
    D = 4100
    rows = np.zeros((4, D), np.float32)
    rows[0, :4] = 0.5          # norm exactly 1.0 = bound: not clipped (strict >)
    rows[1, :2] = [3.0, 4.0]   # norm 5: clipped to factor 0.2
    rows[2, 7] = np.inf        # non-finite: flagged, coef 0
    rows[3, D - 1] = 2.0       # last column (the ragged tail of the last slice row)
    ld = D + 4
    buf = torch.zeros(4, ld, device="cuda")
    buf[:, :D] = torch.from_numpy(rows).cuda()
    w = torch.ones(4, device="cuda")
    base = torch.full((D,), 0.25, device="cuda")
    agg, norm, coef, clipped, bad = fused(buf, ld, 4, D, w, 1.0, agg=base.clone(), accumulate=1)
    np.testing.assert_array_equal(clipped, [0, 1, 0, 1])
    np.testing.assert_array_equal(bad, [0, 0, 1, 0])
    np.testing.assert_allclose(norm[[0, 1, 3]], [1.0, 5.0, 2.0], rtol=1e-7)
    np.testing.assert_allclose(coef, [1.0, 0.2, 0.0, 0.5], rtol=1e-7)
    # column 7 holds coef 0 * inf = nan, exactly as the two-kernel path (the engine raises on nonfinite)
    assert np.isnan(agg[7])
    keep = np.ones(D, bool)
    keep[7] = False
    want = 0.25 + np.array([1.0, 0.2, 0.0, 0.5]) @ np.where(np.isfinite(rows), rows, 0.0)
    np.testing.assert_allclose(agg[keep], want[keep], rtol=1e-7)


def test_fused_unsupported_shapes():
    assert native.call("fb_clip_aggregate_max_columns") >= 10_000_000
    too_big = native.call("fb_clip_aggregate_max_columns") + 1
    with pytest.raises(native.NativeError):
        native.call("fb_clip_aggregate_f32", None, too_big, 1, too_big, None, 1.0, None, None, None, None, None, 0,
                    None, 0, S())


@pytest.mark.parametrize("name", ["mlp_dp", "logistic_dp", "mlp_noclip"])
def test_engine_through_fused_path_matches_reference_run(name, golden, monkeypatch):
    """The engine routed through fb_clip_aggregate_f32 (threshold lowered so the
    reference-sized models take it) reproduces the reference's own runs."""
    from paper_2404_06430_b200 import engine
    from tests.test_gpu_engine import run_engine
    from tests.helpers import CONFIGS, golden_rows

    monkeypatch.setattr(engine, "FUSED_CLIP_AGGREGATE_MIN_D", 0)
    calls = []
    real = native.call

    def spy(fn, *args):
        calls.append(fn)
        return real(fn, *args)

    monkeypatch.setattr(native, "call", spy)
    g = golden(name)
    res, thetas = run_engine(CONFIGS[name])
    assert "fb_clip_aggregate_f32" in calls and "fb_weighted_sum_f32" not in calls
    assert res.cohort_digest == str(g["digest"])
    for t in range(len(thetas)):
        assert_close_fp32(thetas[t], g["thetas"][t], what=f"{name} theta after iteration {t}")
    got, ref = res.metrics_rows, golden_rows(g)
    assert [r[:3] for r in got] == [r[:3] for r in ref]
    np.testing.assert_allclose([r[3] for r in got], [r[3] for r in ref], rtol=2e-5)


def test_fused_rows_gather_matches_two_pass():
    """fb_clip_aggregate_rows_f32: client c reads delta row rows[c] -- a permuted queue with
    repeats (a pool of 5 rows for 150 clients, crossing two fp32 blocks) equals the
    two-kernel path over the materialised gathered matrix."""
    P, C, D = 5, 150, 70_001
    buf, ld, _ = make(P, D, seed=9)
    rows = torch.tensor(np.random.default_rng(1).integers(0, P, C), dtype=torch.int32, device="cuda")
    w = torch.rand(C, device="cuda") + 0.5
    norm = torch.zeros(C, dtype=torch.float64, device="cuda")
    coef = torch.zeros(C, device="cuda")
    clipped = torch.zeros(C, dtype=torch.int32, device="cuda")
    bad = torch.zeros(C, dtype=torch.int32, device="cuda")
    agg = torch.zeros(D, device="cuda")
    ws = torch.empty(native.call("fb_clip_aggregate_workspace_bytes", C, D), dtype=torch.uint8, device="cuda")
    native.call("fb_clip_aggregate_rows_f32", buf.data_ptr(), rows.data_ptr(), ld, C, D, w.data_ptr(), 0.9,
                norm.data_ptr(), coef.data_ptr(), clipped.data_ptr(), bad.data_ptr(), agg.data_ptr(), 0,
                ws.data_ptr(), ws.numel(), S())
    torch.cuda.synchronize()
    gathered = buf[rows.long()].contiguous()
    agg2, norm2, coef2, clipped2 = two_pass(gathered, ld, C, D, w, 0.9)
    np.testing.assert_allclose(norm.cpu().numpy(), norm2, rtol=1e-14)
    np.testing.assert_array_equal(clipped.cpu().numpy(), clipped2)
    assert_close_fp32(agg.double().cpu().numpy(), agg2, what="gathered fused vs two-pass")
