"""Config D (FLAIR-shaped ResNet-18, GroupNorm, multi-label BCE): the sm_100a
local-SGD and eval entry points (csrc/resnet.cu, through the C ABI) against the
float64 oracle (oracle/port.py ResNet18, itself pinned to float64 autograd in
tests/test_oracle_resnet.py) at a narrow shape, at the full 64-wide network on
32 x 32 images and at the full 224 x 224 config D shape, plus one end-to-end
FedAvg + clip + Gaussian-DP central iteration through GpuSimulationEngine with
central Adam.

Tolerance: fp32 against float64; per-client update relative L2 error <= 1e-5,
eval loss rtol 1e-5, exact-match counts exact (+-1 at the wide shapes, where a
logit within rounding of 0 can flip)."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2404_06430_b200 as fb
from oracle import port
from paper_2404_06430_b200 import native
from paper_2404_06430_b200 import resnet as rn_glue
from tests.conftest import assert_close_fp32

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

NARROW = dict(num_classes=5, width=8, groups=4, image=32)
WIDE32 = dict(num_classes=17, width=64, groups=32, image=32)  # the full network on small images (tcgen05 tiles)


@pytest.fixture(params=[1, 0], ids=["tcgen05", "simt"])
def gemm_impl(request):
    native.call("fb_lm_set_gemm_impl", request.param)
    yield request.param
    native.call("fb_lm_set_gemm_impl", 1)


def cohort(shape, n_users, seed, max_images=20):
    m = port.ResNet18(**shape)
    ds = fb.make_synthetic_images(n_users, image=m.image, num_classes=m.num_classes, max_images=max_images,
                                  seed=seed)
    return m, list(ds.users.values())


def pack(users):
    X = np.concatenate([u.features for u in users]).astype(np.float32)
    n = np.array([u.num_points for u in users], dtype=np.int32)
    start = np.concatenate([[0], np.cumsum(n)[:-1]]).astype(np.int64)
    return X, n, start


def d(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def run_local_sgd(model, theta, users, ctx_seed, E, B, lr, mu=0.0, wave=None, eval_out=None):
    X, n, start = pack(users)
    perms = [port.user_perms(ctx_seed, u.user_id, u.num_points, E).astype(np.int32).ravel() for u in users]
    off = np.concatenate([[0], np.cumsum([len(p) for p in perms])[:-1]]).astype(np.int64)
    C, D = len(users), model.num_params
    ld = (D + 3) & ~3
    dims = rn_glue.dims_of(model)
    W = wave or C
    ws = torch.empty(native.call("fb_resnet_workspace_bytes", dims.ctypes.data, B, W), dtype=torch.uint8,
                     device="cuda")
    delta = torch.zeros(C, ld, device="cuda")
    bad = torch.zeros(C, dtype=torch.int32, device="cuda")
    th, Xd, sd, nd, pd, od = d(theta.astype(np.float32)), d(X), d(start), d(n), d(np.concatenate(perms)), d(off)
    native.call("fb_local_sgd_resnet_f32", th.data_ptr(), dims.ctypes.data, Xd.data_ptr(), X.shape[1],
                sd.data_ptr(), nd.data_ptr(), n.ctypes.data, pd.data_ptr(), od.data_ptr(), C, E, B, lr, mu, None, 0,
                delta.data_ptr(), ld, bad.data_ptr(), W, ws.data_ptr(), ws.numel(),
                native.ptr(eval_out[0]) if eval_out else None, native.ptr(eval_out[1]) if eval_out else None,
                native.stream_handle())
    torch.cuda.synchronize()
    return delta[:, :D].double().cpu().numpy(), bad.cpu().numpy()


def run_eval(model, theta, users, groups=3, B=4, skip_first=None):
    """skip_first=(ctx_seed, E, skip): evaluate only epoch 0's images past the first skip."""
    X, n, start = pack(users)
    C = len(users)
    dims = rn_glue.dims_of(model)
    ws = torch.empty(native.call("fb_resnet_workspace_bytes", dims.ctypes.data, B, groups), dtype=torch.uint8,
                     device="cuda")
    loss = torch.zeros(C, dtype=torch.float64, device="cuda")
    corr = torch.zeros(C, dtype=torch.int32, device="cuda")
    th, Xd, sd, nd = d(theta.astype(np.float32)), d(X), d(start), d(n)
    pd = od = None
    skip = 0
    if skip_first is not None:
        seed, E, skip = skip_first
        perms = [port.user_perms(seed, u.user_id, u.num_points, E).astype(np.int32).ravel() for u in users]
        pd = d(np.concatenate(perms))
        od = d(np.concatenate([[0], np.cumsum([len(p) for p in perms])[:-1]]).astype(np.int64))
    native.call("fb_eval_resnet_f32", th.data_ptr(), dims.ctypes.data, Xd.data_ptr(), X.shape[1], sd.data_ptr(),
                nd.data_ptr(), n.ctypes.data, C, loss.data_ptr(), corr.data_ptr(), B, groups, ws.data_ptr(),
                ws.numel(), native.ptr(pd), native.ptr(od), skip, native.stream_handle())
    torch.cuda.synchronize()
    return loss.cpu().numpy(), corr.cpu().numpy()


def oracle_deltas(m, p0, users, ctx_seed, E, B, lr, mu=0.0, margins=None):
    """Float64 local training per client; ``margins`` (a list) receives each client's
    smallest decision margin along its trajectory: min over every ReLU input of |z| /
    rms(z) and every maxpool window's top-two gap / rms (port.TRACK_MARGINS)."""
    out = []
    for u in users:
        X = u.features.astype(np.float64)
        port.MARGINS.clear()
        port.TRACK_MARGINS = margins is not None
        try:
            after = port.fit_local(m, p0, X, u.labels, port.user_perms(ctx_seed, u.user_id, u.num_points, E), lr,
                                   B, mu=mu)
        finally:
            port.TRACK_MARGINS = False
        if margins is not None:
            margins.append(min(port.MARGINS, default=np.inf))
        out.append(port.flat(p0, m.dims) - port.flat(after, m.dims))
    return np.array(out)


# a decision closer than this (relative to its tensor's rms) to its threshold may flip in
# fp32: the pre-activations carry ~1e-7 relative rounding amplified through the layers
# (a 7e-7 margin flipped in the narrow E=2 case, 1.2e-6 did not)
FLIP_MARGIN = 2e-6


def assert_updates(got, want, margins, what):
    """Per-client relative L2 error <= 1e-5, except clients whose float64 trajectory
    passes a ReLU / maxpool decision within FLIP_MARGIN of its threshold: fp32 rounding
    can flip that decision and reroute one gradient (a discrete ~1e-3 .. 1e-2 change on
    a narrow network), so those are only held to 5e-2 -- and counted."""
    err = rel_err(got, want)
    prone = np.array(margins) < FLIP_MARGIN
    print(f"{what}: errors {np.array2string(err, precision=2)}, min margins "
          f"{np.array2string(np.array(margins), precision=1)}, flip-prone {int(prone.sum())}/{len(err)}")
    assert (err[~prone] <= 1e-5).all(), (err, margins)
    assert (err[prone] <= 5e-2).all(), (err, margins)


def rel_err(a, b):
    return np.linalg.norm(a - b, axis=-1) / np.maximum(np.linalg.norm(b, axis=-1), 1e-30)


def product_model(shape):
    return fb.ResNet18(**shape) if shape else fb.ResNet18()


@pytest.mark.parametrize("E,B,lr,mu", [(1, 4, 0.05, 0.0), (2, 3, 0.02, 0.0), (1, 5, 0.05, 0.1)])
def test_resnet_narrow_local_sgd_matches_oracle(E, B, lr, mu, gemm_impl):
    """Ragged clients (1 .. 12 images), tail batches, two epochs, FedProx term;
    clients trained in waves of 3 (largest first) to cover the wave loop."""
    m, users = cohort(NARROW, 7, seed=11, max_images=12)
    model = product_model(NARROW)
    p0 = m.init(3)
    theta = port.flat(p0, m.dims)
    got, bad = run_local_sgd(model, theta, users, 99, E, B, lr, mu, wave=3)
    margins = []
    want = oracle_deltas(m, p0, users, 99, E, B, lr, mu, margins=margins)
    assert not bad.any()
    assert_updates(got, want, margins, f"narrow E={E} B={B} mu={mu}")


@pytest.mark.parametrize("B,max_images", [(4, 10), (16, 40)], ids=["B4", "B16-splitK"])
def test_resnet_wide32_local_sgd_and_eval_match_oracle(gemm_impl, B, max_images):
    """The full 64-wide ResNet-18 (every conv GEMM on the tcgen05 tiles) on 32 x 32 images;
    at B = 16 the stem's weight gradient (K = 16 x 256 rows) runs split-K in 2 chunks."""
    m, users = cohort(WIDE32, 4, seed=21, max_images=max_images)
    model = product_model(WIDE32)
    p0 = m.init(7)
    theta = port.flat(p0, m.dims)
    got, bad = run_local_sgd(model, theta, users, 5, 1, B, 0.05)
    margins = []
    want = oracle_deltas(m, p0, users, 5, 1, B, 0.05, margins=margins)
    assert not bad.any()
    assert_updates(got, want, margins, f"wide32 B={B}")
    loss, corr = run_eval(model, theta, users, groups=2, B=4)
    for c, u in enumerate(users):
        ls, k = m.eval_counts(p0, u.features.astype(np.float64))
        assert loss[c] == pytest.approx(ls, rel=1e-5)
        assert abs(int(corr[c]) - k) <= 1


def test_resnet_eval_narrow_matches_oracle():
    m, users = cohort(NARROW, 9, seed=5, max_images=15)
    p0 = m.init(2)
    loss, corr = run_eval(product_model(NARROW), port.flat(p0, m.dims), users, groups=3, B=4)
    for c, u in enumerate(users):
        ls, k = m.eval_counts(p0, u.features.astype(np.float64))
        assert loss[c] == pytest.approx(ls, rel=1e-5)
        assert corr[c] == k


def test_resnet_configD_matches_oracle():
    """The full config D shape: 224 x 224 images, 17 labels, B = 16, local lr 0.01
    (PAPER.md:1133-1135); one full batch and one tail batch of 7.

    Forward (evaluation loss): ReLU / maxpool are continuous, so the forward matches the
    float64 oracle to fp32 rounding -- rtol 1e-5.  Backward: at this size a few ReLU /
    maxpool decisions sit within fp32 rounding of their threshold, and flipping one
    reroutes a gradient, so NO fp32 implementation meets 1e-5 on the whole update:
    PyTorch's own fp32 arithmetic (same network and inputs) is 4e-5 .. 2.4e-4 from the
    oracle (printed here; tools/rn_diag.py per layer: 2.5e-3 on the stem, 1e-7 on the
    head).  Gates: the fc block (downstream of every decision) at 1e-5, the whole update
    at 1e-3 (a few flips' worth); the exact backward is pinned at 1e-5 by the 64-wide
    network on 32 x 32 images above."""
    from tests.test_oracle_resnet import torch_resnet_loss

    m = port.ResNet18()
    model = product_model({})
    ds = fb.make_synthetic_images(6, image=224, num_classes=17, max_images=40, seed=2)
    big = [u for u in ds.users.values() if u.num_points >= 16]
    u16 = fb.UserDataset(big[0].user_id, big[0].features[:16], big[0].labels[:16])
    u7 = fb.UserDataset(big[1].user_id, big[1].features[:7], big[1].labels[:7])
    users = [u16, u7]
    p0 = m.init(1)
    theta = port.flat(p0, m.dims)
    lr = 0.01
    loss, corr = run_eval(model, theta, users, groups=2, B=8)
    got, bad = run_local_sgd(model, theta, users, 8, 1, 16, lr)
    assert not bad.any()
    fc = slice(sum(k for n, k in m.dims.items() if not n.startswith("fc.")), None)
    for c, u in enumerate(users):
        X = u.features.astype(np.float64)
        ls, k = m.eval_counts(p0, X)
        assert loss[c] == pytest.approx(ls, rel=1e-5), c
        assert abs(int(corr[c]) - k) <= 1
        perm = port.user_perms(8, u.user_id, u.num_points, 1)[0]
        _, g = m.loss_and_grad(p0, X[perm])
        want = port.flat(g, m.dims) * lr
        loss32, t = torch_resnet_loss(m, p0, X[perm], dtype=torch.float32)
        loss32.backward()
        floor = np.concatenate([t[n].grad.numpy().ravel().astype(np.float64) for n in m.dims]) * lr
        e_gpu = np.linalg.norm(got[c] - want) / np.linalg.norm(want)
        e_floor = np.linalg.norm(floor - want) / np.linalg.norm(want)
        e_fc = np.linalg.norm(got[c][fc] - want[fc]) / np.linalg.norm(want[fc])
        print(f"config D client {c} ({u.num_points} images): GPU {e_gpu:.2e} (fc {e_fc:.2e}), "
              f"torch fp32 {e_floor:.2e}")
        assert e_fc <= 1e-5 and e_gpu <= 1e-3, (e_fc, e_gpu, e_floor)


@pytest.mark.parametrize("shape,B,E", [("narrow", 3, 2), ("wide32", 4, 1)])
def test_resnet_first_batch_eval_shared_with_local_sgd(shape, B, E):
    """Split evaluation (fb_eval_resnet_f32 perms/skip + fb_local_sgd_resnet_f32
    eval_loss / eval_correct) equals the full evaluation and the oracle's."""
    shp = NARROW if shape == "narrow" else WIDE32
    m, users = cohort(shp, 6, seed=17, max_images=9)
    model = product_model(shp)
    p0 = m.init(6)
    theta = port.flat(p0, m.dims)
    full_loss, full_corr = run_eval(model, theta, users, groups=3)
    loss, corr = run_eval(model, theta, users, groups=3, skip_first=(41, E, B))
    lt = torch.from_numpy(loss).cuda()
    ct = torch.from_numpy(corr).cuda()
    run_local_sgd(model, theta, users, 41, E, B, 0.02, wave=2, eval_out=(lt, ct))
    loss, corr = lt.cpu().numpy(), ct.cpu().numpy()
    for c, u in enumerate(users):
        ls, k = m.eval_counts(p0, u.features.astype(np.float64))
        assert loss[c] == pytest.approx(ls, rel=1e-5), c
        assert loss[c] == pytest.approx(full_loss[c], rel=1e-5), c
        assert abs(int(corr[c]) - k) <= 1 and abs(int(corr[c]) - int(full_corr[c])) <= 1, c


def test_resnet_deterministic_rerun():
    m, users = cohort(NARROW, 5, seed=3)
    theta = port.flat(m.init(1), m.dims)
    a, _ = run_local_sgd(product_model(NARROW), theta, users, 7, 1, 4, 0.05, wave=2)
    b, _ = run_local_sgd(product_model(NARROW), theta, users, 7, 1, 4, 0.05, wave=2)
    np.testing.assert_array_equal(a, b)


def test_resnet_engine_central_iteration_with_adam_matches_oracle():
    """FedAvg + ClippingPostprocessor (bound 0.1) + GaussianCentralMechanism
    (reference noise injected) + central Adam (lr 0.1, betas 0.9 / 0.99, eps 0.1), one
    iteration through GpuSimulationEngine."""
    m = port.ResNet18(**NARROW)
    model = product_model(NARROW)
    train = fb.make_synthetic_images(10, image=m.image, num_classes=m.num_classes, max_images=14, seed=8,
                                     id_prefix="train")
    clip = fb.ClippingPostprocessor(0.1)
    mech = fb.GaussianCentralMechanism(clip, sigma=1.0, r=0.1, noise_base_seed=7, noise_source="numpy")
    alg = fb.FedAvg(model, fb.AdamOptimizer(0.1, beta1=0.9, beta2=0.99, adaptivity_degree=0.1), total_iterations=1,
                    cohort_size=5, local_learning_rate=0.01, local_num_epochs=2, local_batch_size=4,
                    eval_frequency=10, eval_cohort_size=1, weighting="datapoints", run_seed=3, init_seed=4)
    eng = fb.GpuSimulationEngine({fb.Population.TRAIN: train, fb.Population.VAL: train}, postprocessors=[clip, mech])
    state = alg.initial_state()
    ctxs = alg.get_next_central_contexts(state, 0)[:1]
    res = eng.run_iteration(alg, state, ctxs)
    state = alg.process_aggregated_statistics_all_contexts(state, ctxs, res.aggregates, res.metrics, [])
    got = state.params.flat_host()
    users = {u.user_id: (u.features.astype(np.float64), u.labels) for u in train.users.values()}
    theta0 = m.init(4)
    ref = port.run_context(m, theta0, users, 5, ctxs[0].seed, train=(0.01, 2, 4), weighting="datapoints", bound=0.1,
                           sigma=1.0, r=0.1, noise_base=7, t=0, pop="train")
    want = port.central_adam(port.flat(theta0, m.dims), ref.aggregate, ref.weight, 0.1, {}, noise=ref.noise,
                             beta1=0.9, beta2=0.99, eps=0.1)
    assert_close_fp32(got, want, what="theta after one ResNet central iteration")
    mt = res.metrics[0] if isinstance(res.metrics, list) else res.metrics
    assert mt is not None


def test_resnet_bench_shape_cohort_matches_oracle():
    """Parity at the benchmarked configuration (bench.py --workload resnet): the bench's own
    synthetic population, cohort 200 drawn by the engine's sampler, E = 2, B = 16, local lr
    0.01, every client trained in the bench's largest-first waves; the float64 oracle
    replays a sample of three clients (~0.5 s per image step on the host).

    Over several local steps at 224 px, fp32 decision flips (see
    test_resnet_configD_matches_oracle) also perturb every later step, so the reference
    point is PyTorch's own fp32 training of the same clients (same batches, same update
    rule): the gate is max(1e-3, 3 x that fp32 error) per client (both printed)."""
    import bench

    wl = bench.WORKLOADS["resnet"]
    ds = bench.build(wl)[fb.Population.TRAIN]
    m = port.ResNet18()
    model = product_model({})
    cohort_ids = port.sample_cohort(ds.user_ids, wl["cohort"], port.cohort_seed(0, 0, "train"))
    users = [ds.users[u] for u in cohort_ids]
    p0 = m.init(0)
    theta = port.flat(p0, m.dims)
    got, bad = run_local_sgd(model, theta, users, 17, wl["epochs"], wl["batch"], wl["lr"],
                             wave=rn_glue.wave_size(model, wl["batch"], len(users)))
    assert not bad.any()
    sizes = np.array([u.num_points for u in users])
    order = np.argsort(sizes)
    sample = [int(order[0]), int(order[len(order) // 2]), int(order[int(0.8 * len(order))])]  # small / median / large
    want = oracle_deltas(m, p0, [users[i] for i in sample], 17, wl["epochs"], wl["batch"], wl["lr"])
    err = rel_err(got[sample], want)
    floor = rel_err(np.array([torch_fp32_deltas(m, p0, users[i], 17, wl["epochs"], wl["batch"], wl["lr"])
                              for i in sample]), want)
    print(f"bench-shape ResNet parity: clients {sample} with {sizes[sample].tolist()} images: GPU errors "
          f"{np.array2string(err, precision=2)}, torch fp32 {np.array2string(floor, precision=2)}")
    assert (err <= np.maximum(1e-3, 3 * floor)).all(), (err, floor)


def torch_fp32_deltas(m, p0, u, ctx_seed, E, B, lr):
    """PyTorch fp32 (CPU) local training with the reference's update rule and batches."""
    from tests.test_oracle_resnet import torch_resnet_loss

    X = u.features.astype(np.float64)
    perms = port.user_perms(ctx_seed, u.user_id, u.num_points, E)
    p = {k: v.astype(np.float32) for k, v in p0.items()}
    for e in range(E):
        for s0 in range(0, u.num_points, B):
            loss, t = torch_resnet_loss(m, p, X[perms[e, s0:s0 + B]], dtype=torch.float32)
            loss.backward()
            p = {k: (torch.from_numpy(p[k]) - lr * t[k].grad.reshape(-1)).numpy() for k in p}
    return port.flat(p0, m.dims) - port.flat({k: v.astype(np.float64) for k, v in p.items()}, m.dims)


@pytest.mark.parametrize("algo", [dict(kind="scaffold", num_train_users=10), dict(kind="fedprox", mu=0.1)],
                         ids=["scaffold", "fedprox"])
def test_resnet_engine_algorithms_match_oracle(algo):
    """SCAFFOLD and FedProx on config D's model through
    GpuSimulationEngine, 3 central iterations with clip + injected noise + central Adam and
    evaluation, against the oracle's run_fedavg (fedsim/algorithms/scaffold.py:28-120,
    fedsim/algorithms/fedavg.py:201-296).  Per-iteration theta at rtol 1e-5 (atol 1e-6
    max|ref|) unless the oracle's trajectory passed a decision within FLIP_MARGIN of its
    threshold (then relative L2 <= 1e-2; printed)."""
    from tests.conftest import assert_close_fp32
    from tests.helpers import run_sim

    m = port.ResNet18(**NARROW)
    model = product_model(NARROW)
    train = fb.make_synthetic_images(10, image=m.image, num_classes=m.num_classes, max_images=14, seed=8,
                                     id_prefix="train")
    val = fb.make_synthetic_images(4, image=m.image, num_classes=m.num_classes, max_images=6, seed=9,
                                   population=fb.Population.VAL, id_prefix="val")
    clip = fb.ClippingPostprocessor(0.1)
    noise_base = 7
    mech = fb.GaussianCentralMechanism(clip, sigma=1.0, r=0.2, noise_base_seed=noise_base, noise_source="numpy")
    opt = fb.AdamOptimizer(0.05, beta1=0.9, beta2=0.99, adaptivity_degree=0.1)
    weighting = "uniform" if algo["kind"] == "scaffold" else "datapoints"  # (SCAFFOLD averages uniformly)
    kw = dict(total_iterations=3, cohort_size=5, local_learning_rate=0.01, local_num_epochs=2, local_batch_size=4,
              eval_frequency=2, eval_cohort_size=3, weighting=weighting, run_seed=3, init_seed=4)
    alg = (fb.Scaffold(model, opt, num_train_users=algo["num_train_users"], **kw) if algo["kind"] == "scaffold"
           else fb.FedProx(model, opt, mu=algo["mu"], **kw))
    eng = fb.GpuSimulationEngine({fb.Population.TRAIN: train, fb.Population.VAL: val}, postprocessors=[clip, mech])
    thetas = []
    res = run_sim(alg, eng, callbacks=[lambda p, rows, t: thetas.append(p.flat_host()) and False])
    users = lambda ds: {u.user_id: (u.features.astype(np.float64), u.labels) for u in ds.users.values()}
    port.MARGINS.clear()
    port.TRACK_MARGINS = True
    try:
        want, rows, digest = port.run_fedavg(
            m, users(train), users(val), iterations=3, cohort=5, eval_cohort=3, eval_every=2, lr=0.01, epochs=2,
            batch=4, clr=0.05, weighting=weighting, bound=0.1, sigma=1.0, r=0.2, noise_base=noise_base,
            run_seed=3, init_seed=4, algorithm=algo,
            optimizer=dict(kind="adam", lr=0.05, beta1=0.9, beta2=0.99, eps=0.1))
    finally:
        port.TRACK_MARGINS = False
    margin = min(port.MARGINS, default=np.inf)
    assert res.cohort_digest == digest
    got = np.array(thetas)[:, :want.shape[1]]
    errs = np.linalg.norm(got - want, axis=1) / np.linalg.norm(want, axis=1)
    print(f"ResNet {algo['kind']}: theta errors per iteration {np.array2string(errs, precision=2)}, "
          f"min decision margin {margin:.1e}")
    if margin >= FLIP_MARGIN:
        for t in range(len(want)):
            assert_close_fp32(got[t], want[t], what=f"ResNet {algo['kind']} theta after iteration {t}")
    else:
        assert errs.max() <= 1e-2, errs
