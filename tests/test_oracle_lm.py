"""Pins the config C transformer-LM oracle (oracle/port.py TransformerLM), which
has no reference implementation, the way the reference pins its own models
(tests/test_models.py:27-63 finite differences) -- here against float64 torch
autograd of the same network (CPU, test-only), at a tiny shape and at the
full config C shape, plus eval / loss consistency and the parameter count
the paper quotes."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2404_06430_b200 as fb
from oracle import port

torch = pytest.importorskip("torch")


def torch_lm_loss(m: port.TransformerLM, p: dict, X: np.ndarray):
    """The same network written with torch ops (float64), for autograd."""
    import torch.nn.functional as F

    t = {k: torch.tensor(v, dtype=torch.float64, requires_grad=True) for k, v in p.items()}
    N, L, d, H = X.shape[0], m.seq, m.d, m.heads
    dh = d // H
    tok = torch.tensor(X[:, :L].astype(np.int64))
    tgt = torch.tensor(X[:, 1:L + 1].astype(np.int64))
    E = t["embedding"].reshape(m.vocab, d)
    x = E[tok] * np.sqrt(d) + torch.tensor(port.lm_positions(L, d))
    causal = torch.triu(torch.ones(L, L, dtype=torch.bool), 1)
    for l in range(m.layers):
        q = lambda n: t[f"layer{l}/{n}"]
        qkv = x @ q("in_proj_weight").reshape(3 * d, d).T + q("in_proj_bias")
        Q, K, V = (qkv[..., i * d:(i + 1) * d].reshape(N, L, H, dh).transpose(1, 2) for i in range(3))
        s = (Q @ K.transpose(-1, -2) / np.sqrt(dh)).masked_fill(causal, float("-inf"))
        o = (torch.softmax(s, -1) @ V).transpose(1, 2).reshape(N, L, d)
        a = o @ q("out_proj_weight").reshape(d, d).T + q("out_proj_bias")
        x1 = F.layer_norm(x + a, (d,), q("norm1_weight"), q("norm1_bias"), m.eps)
        f = torch.relu(x1 @ q("linear1_weight").reshape(m.ff, d).T + q("linear1_bias"))
        f = f @ q("linear2_weight").reshape(d, m.ff).T + q("linear2_bias")
        x = F.layer_norm(x1 + f, (d,), q("norm2_weight"), q("norm2_bias"), m.eps)
    logits = x @ E.T
    loss = F.cross_entropy(logits.reshape(-1, m.vocab), tgt.reshape(-1), ignore_index=port.LM_PAD)
    return loss, t


def sentences(m, n, seed):
    ds = fb.make_synthetic_sentences(1, vocab=m.vocab, seq=m.seq, max_sentences=64, seed=seed)
    X = next(iter(ds.users.values())).features
    reps = -(-n // X.shape[0])
    return np.concatenate([X] * reps)[:n]


@pytest.mark.parametrize("shape", [dict(vocab=13, d=8, heads=2, ff=16, layers=2, seq=6),
                                   dict()], ids=["tiny", "configC"])
def test_lm_oracle_gradient_matches_autograd(shape):
    m = port.TransformerLM(**shape)
    p = m.init(5)
    rng = np.random.default_rng(0)
    for k in p:  # non-trivial LayerNorm gains / biases
        if k.endswith("_bias") or "norm" in k:
            p[k] = p[k] + 0.1 * rng.normal(size=p[k].shape)
    X = sentences(m, 3, seed=2)
    loss, g = m.loss_and_grad(p, X)
    ref, t = torch_lm_loss(m, p, X)
    ref.backward()
    assert abs(loss - ref.item()) <= 1e-12 * abs(ref.item())
    for name in m.dims:
        np.testing.assert_allclose(g[name], t[name].grad.numpy().ravel(), rtol=1e-8, atol=1e-14, err_msg=name)


def test_lm_parameter_count_and_layout():
    m = port.TransformerLM()
    assert sum(m.dims.values()) == 1_962_912
    assert fb.TransformerLM().param_dims == m.dims
    assert fb.TransformerLM().num_params == 1_962_912


def test_lm_eval_counts_consistent_with_loss():
    m = port.TransformerLM(vocab=29, d=16, heads=4, ff=32, layers=1, seq=8)
    p = m.init(1)
    X = sentences(m, 7, seed=3)
    loss_mean, _ = m.loss_and_grad(p, X)
    loss_sum, correct = m.eval_counts(p, X)
    nv = int((X[:, 1:] != port.LM_PAD).sum())
    assert np.isclose(loss_sum, nv * loss_mean, rtol=1e-12)
    assert 0 <= correct <= nv


def test_lm_all_pad_batch_has_zero_gradient():
    m = port.TransformerLM(vocab=11, d=8, heads=2, ff=8, layers=1, seq=4)
    p = m.init(0)
    X = np.zeros((2, 5))
    loss, g = m.loss_and_grad(p, X)
    assert loss == 0.0 and all(not v.any() for v in g.values())


def test_synthetic_sentences_shape():
    ds = fb.make_synthetic_sentences(50, seed=7)
    sizes = np.array([u.num_points for u in ds.users.values()])
    assert sizes.min() >= 1 and sizes.max() <= 64
    for u in ds.users.values():
        X = u.features
        assert X.shape[1] == 21 and (X[:, 0] == 1).all()
        np.testing.assert_array_equal((X[:, 1:] != 0).sum(axis=1), u.labels)
        assert X.max() < 10004
