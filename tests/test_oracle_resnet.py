"""Pins the config D ResNet-18 oracle (oracle/port.py ResNet18: GroupNorm, multi-label
sigmoid BCE), which has no reference implementation, against float64 torch autograd of
the same network written with torch ops (CPU, test-only) -- at a narrow shape and at
the full 64-wide ResNet-18 on small images -- plus eval / loss consistency, the maxpool
tie rule and the parameter count of the FLAIR configuration."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import port

torch = pytest.importorskip("torch")
F = torch.nn.functional


def torch_resnet_loss(m: port.ResNet18, p: dict, X: np.ndarray, dtype=None):
    """(loss, {name: leaf tensor}) of the network written with torch ops; float64 by
    default, float32 for the fp32 floor the GPU parity tests compare against."""
    dtype = dtype or torch.float64
    t = {k: torch.tensor(v, dtype=dtype, requires_grad=True) for k, v in p.items()}
    S, K, w = m.image, m.num_classes, m.width
    x = torch.tensor(X[:, :3 * S * S].reshape(-1, 3, S, S), dtype=dtype)
    lab = torch.tensor(X[:, 3 * S * S:3 * S * S + K], dtype=dtype)
    gn = lambda h, name: F.group_norm(h, m.groups, t[name + ".weight"], t[name + ".bias"], m.eps)
    h = F.conv2d(x, t["conv1.weight"].reshape(w, 3, 7, 7), stride=2, padding=3)
    h = F.max_pool2d(torch.relu(gn(h, "gn1")), 3, 2, 1)
    for name, ci, co, st, ds in m.blocks():
        u = torch.relu(gn(F.conv2d(h, t[f"{name}.conv1.weight"].reshape(co, ci, 3, 3), stride=st, padding=1),
                          f"{name}.gn1"))
        v = gn(F.conv2d(u, t[f"{name}.conv2.weight"].reshape(co, co, 3, 3), padding=1), f"{name}.gn2")
        sc = h
        if ds:
            sc = gn(F.conv2d(h, t[f"{name}.downsample.0.weight"].reshape(co, ci, 1, 1), stride=st),
                    f"{name}.downsample.1")
        h = torch.relu(v + sc)
    feat = h.mean(dim=(2, 3))
    z = feat @ t["fc.weight"].reshape(K, -1).T + t["fc.bias"]
    return F.binary_cross_entropy_with_logits(z, lab), t


def images(m, n, seed):
    rng = np.random.default_rng(seed)
    S, K = m.image, m.num_classes
    pix = rng.normal(size=(n, 3 * S * S))
    lab = (rng.random((n, K)) < 0.3).astype(np.float64)
    return np.concatenate([pix, lab], axis=1)


def perturbed(m, seed):
    p = m.init(seed)
    rng = np.random.default_rng(seed + 1)
    for k in p:  # non-trivial norm gains / biases
        if k.endswith("bias") or ".gn" in k or k.startswith("gn") or "downsample.1" in k:
            p[k] = p[k] + 0.1 * rng.normal(size=p[k].shape)
    return p


@pytest.mark.parametrize("shape", [dict(num_classes=5, width=8, groups=4, image=32),
                                   dict(num_classes=17, width=64, groups=32, image=32)], ids=["narrow", "full-32px"])
def test_resnet_oracle_gradient_matches_autograd(shape):
    m = port.ResNet18(**shape)
    p = perturbed(m, 3)
    X = images(m, 3, seed=4)
    loss, g = m.loss_and_grad(p, X)
    ref, t = torch_resnet_loss(m, p, X)
    ref.backward()
    assert abs(loss - ref.item()) <= 1e-12 * abs(ref.item())
    for name in m.dims:
        np.testing.assert_allclose(g[name], t[name].grad.numpy().ravel(), rtol=1e-8,
                                   atol=1e-12 * np.abs(t[name].grad.numpy()).max(), err_msg=name)


def test_resnet_maxpool_ties_follow_torch():
    """All-negative stem pre-activations: every pooled window is a tie of zeros after the
    ReLU; the gradient must still route like PyTorch's (first maximum, row-major)."""
    m = port.ResNet18(num_classes=3, width=8, groups=2, image=16)
    p = m.init(1)
    p["gn1.bias"] = p["gn1.bias"] - 0.5  # many zero (tied) post-ReLU stem outputs
    X = images(m, 2, seed=9)
    loss, g = m.loss_and_grad(p, X)
    ref, t = torch_resnet_loss(m, p, X)
    ref.backward()
    for name in m.dims:
        np.testing.assert_allclose(g[name], t[name].grad.numpy().ravel(), rtol=1e-8,
                                   atol=1e-12 * max(np.abs(t[name].grad.numpy()).max(), 1e-300), err_msg=name)


def test_resnet_parameter_count():
    m = port.ResNet18()
    assert sum(m.dims.values()) == 11_185_233  # torchvision resnet18 (GN for BN), 17-way fc


def test_resnet_eval_counts_consistent_with_loss():
    m = port.ResNet18(num_classes=4, width=8, groups=4, image=32)
    p = m.init(2)
    X = images(m, 5, seed=1)
    loss_mean, _ = m.loss_and_grad(p, X)
    loss_sum, correct = m.eval_counts(p, X)
    assert np.isclose(loss_sum, 5 * loss_mean, rtol=1e-12)
    assert 0 <= correct <= 5
