"""Float64 numpy restatement of the reference central iteration.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Every function cites
the reference code it restates; paths are relative to
/root/reference/pkg/src/.  Self-contained: numpy + hashlib only, so it can
check the product without sharing its code.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import numpy as np

# ------------------------------------------------------------------ seeds
# fedsim/core/seeds.py:18-42


def derive_seed(*parts) -> int:
    h = hashlib.sha256()
    for p in parts:
        h.update(repr(p).encode())
        h.update(b"\x1f")
    return int.from_bytes(h.digest()[:8], "little") & ((1 << 63) - 1)


def user_seed(ctx_seed: int, uid: str) -> int:
    return derive_seed(ctx_seed, "user", uid)


def cohort_seed(run_seed: int, t: int, pop: str) -> int:
    return derive_seed(run_seed, "cohort", t, pop)


def noise_seed(base: int, t: int, pop: str) -> int:
    return derive_seed(base, "noise", t, pop)


# --------------------------------------------------------------- sampling
# fedsim/feddata/sampling.py:25-34 (fixed mode)


def sample_cohort(user_ids, cohort_size: int, seed: int) -> tuple:
    picks = np.random.default_rng(seed).choice(len(user_ids), size=cohort_size, replace=False)
    return tuple(user_ids[i] for i in picks)


# fedsim/engine/scheduling.py:34-78


def lower_median(ws) -> float:
    s = sorted(ws)
    return float(s[(len(s) - 1) // 2])


def lpt_queues(weights: dict, m: int, base: float):
    order = sorted(weights.items(), key=lambda kv: (-kv[1], kv[0]))
    queues = [[] for _ in range(m)]
    loads = [0.0] * m
    for uid, w in order:
        k = min(range(m), key=loads.__getitem__)
        queues[k].append(uid)
        loads[k] += w + base
    return [tuple(q) for q in queues], loads


# fedsim/models/models.py:231-264


def user_perms(ctx_seed: int, uid: str, n: int, epochs: int) -> np.ndarray:
    rng = np.random.default_rng(user_seed(ctx_seed, uid))
    return np.stack([rng.permutation(n) for _ in range(epochs)]).astype(np.int64)


# ---------------------------------------------------------------- models


def _xent(logits: np.ndarray, y: np.ndarray):
    """Mean CE and d(mean CE)/dlogits (fedsim/models/models.py:115-124)."""
    n = logits.shape[0]
    z = logits - logits.max(axis=1, keepdims=True)
    p = np.exp(z)
    p /= p.sum(axis=1, keepdims=True)
    loss = -np.mean(np.log(p[np.arange(n), y]))
    p[np.arange(n), y] -= 1.0
    return float(loss), p / n


def _eval_rows(logits: np.ndarray, y: np.ndarray):
    """Summed CE and first-argmax hits (fedsim/models/kernels.py:70-83)."""
    m = logits.max(axis=1, keepdims=True)
    lse = np.log(np.exp(logits - m).sum(axis=1))
    loss = -(logits[np.arange(len(y)), y] - m[:, 0] - lse)
    return float(loss.sum()), int((np.argmax(logits, axis=1) == y).sum())


@dataclass(frozen=True)
class Linear:
    dim: int
    k: int

    @property
    def dims(self):
        return {"weights": self.dim * self.k, "bias": self.k}

    def init(self, seed):
        return {n: np.zeros(s) for n, s in self.dims.items()}

    def loss_and_grad(self, p, X, y):  # fedsim/models/models.py:110-124
        W = p["weights"].reshape(self.dim, self.k)
        loss, dl = _xent(X @ W + p["bias"], y)
        return loss, {"weights": (X.T @ dl).ravel(), "bias": dl.sum(axis=0)}

    def eval_counts(self, p, X, y):
        W = p["weights"].reshape(self.dim, self.k)
        return _eval_rows(X @ W + p["bias"], y)


@dataclass(frozen=True)
class Mlp:
    dim: int
    h: int
    k: int

    @property
    def dims(self):
        return {"layer1/weights": self.dim * self.h, "layer1/bias": self.h,
                "layer2/weights": self.h * self.k, "layer2/bias": self.k}

    def init(self, seed):  # fedsim/models/models.py:162-175
        rng = np.random.default_rng(seed)
        b1, b2 = 1.0 / np.sqrt(self.dim), 1.0 / np.sqrt(self.h)
        return {"layer1/weights": rng.uniform(-b1, b1, self.dim * self.h),
                "layer1/bias": rng.uniform(-b1, b1, self.h),
                "layer2/weights": rng.uniform(-b2, b2, self.h * self.k),
                "layer2/bias": rng.uniform(-b2, b2, self.k)}

    def loss_and_grad(self, p, X, y):  # fedsim/models/models.py:185-205
        W1 = p["layer1/weights"].reshape(self.dim, self.h)
        W2 = p["layer2/weights"].reshape(self.h, self.k)
        z1 = X @ W1 + p["layer1/bias"]
        h = np.maximum(z1, 0.0)
        loss, dl = _xent(h @ W2 + p["layer2/bias"], y)
        dz1 = (dl @ W2.T) * (z1 > 0.0)
        return loss, {"layer1/weights": (X.T @ dz1).ravel(), "layer1/bias": dz1.sum(axis=0),
                      "layer2/weights": (h.T @ dl).ravel(), "layer2/bias": dl.sum(axis=0)}

    def eval_counts(self, p, X, y):
        W1 = p["layer1/weights"].reshape(self.dim, self.h)
        W2 = p["layer2/weights"].reshape(self.h, self.k)
        h = np.maximum(X @ W1 + p["layer1/bias"], 0.0)
        return _eval_rows(h @ W2 + p["layer2/bias"], y)


# Decision margins of the last CNN forwards (test instrumentation): fp32 vs
# float64 can only disagree on a ReLU sign or a max-pool winner when the
# float64 value sits within ~1e-6 (relative) of that decision boundary.
MARGINS: list[float] = []
TRACK_MARGINS = False


def _record_margin(*vals):
    if TRACK_MARGINS:
        MARGINS.append(min(vals))


def _relu_margin(z: np.ndarray) -> float:
    scale = float(np.sqrt(np.mean(z * z))) or 1.0
    return float(np.abs(z).min()) / scale


def _im2col3(x: np.ndarray) -> np.ndarray:
    """NHWC [N, H, W, C] -> [N*(H-2)*(W-2), C*9] with (c, kh, kw) column order
    (the OIHW weight flattening)."""
    win = np.lib.stride_tricks.sliding_window_view(x, (3, 3), axis=(1, 2))  # N,Ho,Wo,C,3,3
    n, ho, wo, c = win.shape[:4]
    return win.reshape(n * ho * wo, c * 9)


@dataclass(frozen=True)
class Cnn:
    """conv3x3(3->32)+ReLU, conv3x3(32->64)+ReLU, maxpool2, fc 12544->128
    +ReLU, fc 128->10; valid convs, CHW inputs, OIHW conv weights, [in,out]
    fc weights (paper_2404_06430_b200/models.py).  No reference
    implementation exists (SURVEY.md section 8 "Assumed CNN")."""

    c0: int = 3
    s: int = 32
    c1: int = 32
    c2: int = 64
    hid: int = 128
    k: int = 10

    @property
    def flat(self):
        return self.c2 * ((self.s - 4) // 2) ** 2

    @property
    def dims(self):
        return {"conv1/weights": self.c1 * self.c0 * 9, "conv1/bias": self.c1,
                "conv2/weights": self.c2 * self.c1 * 9, "conv2/bias": self.c2,
                "fc1/weights": self.flat * self.hid, "fc1/bias": self.hid,
                "fc2/weights": self.hid * self.k, "fc2/bias": self.k}

    def init(self, seed):
        fan = {"conv1": self.c0 * 9, "conv2": self.c1 * 9, "fc1": self.flat, "fc2": self.hid}
        rng = np.random.default_rng(seed)
        out = {}
        for name, n in self.dims.items():
            b = 1.0 / np.sqrt(fan[name.split("/")[0]])
            out[name] = rng.uniform(-b, b, n)
        return out

    def _forward(self, p, X):
        N, s = X.shape[0], self.s
        s1, s2, sp = s - 2, s - 4, (s - 4) // 2
        x = X.reshape(N, self.c0, s, s).transpose(0, 2, 3, 1)             # NHWC
        cols1 = _im2col3(x)                                                # N*s1*s1, c0*9
        z1 = cols1 @ p["conv1/weights"].reshape(self.c1, -1).T + p["conv1/bias"]
        a1 = np.maximum(z1, 0.0).reshape(N, s1, s1, self.c1)
        cols2 = _im2col3(a1)                                               # N*s2*s2, c1*9
        z2 = cols2 @ p["conv2/weights"].reshape(self.c2, -1).T + p["conv2/bias"]
        a2 = np.maximum(z2, 0.0).reshape(N, sp, 2, sp, 2, self.c2)
        win = a2.transpose(0, 5, 1, 3, 2, 4).reshape(N, self.c2, sp, sp, 4)  # (dy, dx) window order
        arg = win.argmax(axis=4)  # first maximum in (0,0),(0,1),(1,0),(1,1) order
        pooled = np.take_along_axis(win, arg[..., None], axis=4)[..., 0]
        if TRACK_MARGINS:
            srt = np.sort(win, axis=4)
            live = srt[..., 3] > 0
            gap = (srt[..., 3] - srt[..., 2])[live]
            scale = float(np.sqrt(np.mean(z2 * z2))) or 1.0
            pool_gap = float(gap.min()) / scale if gap.size else np.inf
            _record_margin(_relu_margin(z1), _relu_margin(z2), pool_gap)
        flat = pooled.reshape(N, -1)                                       # CHW flatten order
        z3 = flat @ p["fc1/weights"].reshape(self.flat, self.hid) + p["fc1/bias"]
        a3 = np.maximum(z3, 0.0)
        _record_margin(_relu_margin(z3))
        logits = a3 @ p["fc2/weights"].reshape(self.hid, self.k) + p["fc2/bias"]
        return dict(cols1=cols1, z1=z1, cols2=cols2, z2=z2, arg=arg, flat=flat, z3=z3, a3=a3), logits

    def loss_and_grad(self, p, X, y):
        N = X.shape[0]
        s1, s2, sp = self.s - 2, self.s - 4, (self.s - 4) // 2
        c, logits = self._forward(p, X)
        loss, dl = _xent(logits, y)
        Wf2 = p["fc2/weights"].reshape(self.hid, self.k)
        Wf1 = p["fc1/weights"].reshape(self.flat, self.hid)
        g = {"fc2/weights": (c["a3"].T @ dl).ravel(), "fc2/bias": dl.sum(axis=0)}
        dz3 = (dl @ Wf2.T) * (c["z3"] > 0.0)
        g["fc1/weights"] = (c["flat"].T @ dz3).ravel()
        g["fc1/bias"] = dz3.sum(axis=0)
        dpool = (dz3 @ Wf1.T).reshape(N, self.c2, sp, sp)
        dwin = np.zeros((N, self.c2, sp, sp, 4))
        np.put_along_axis(dwin, c["arg"][..., None], dpool[..., None], axis=4)
        da2 = dwin.reshape(N, self.c2, sp, sp, 2, 2).transpose(0, 2, 4, 3, 5, 1).reshape(N * s2 * s2, self.c2)
        dz2 = da2 * (c["z2"] > 0.0)                                        # N*s2*s2, c2
        g["conv2/weights"] = (dz2.T @ c["cols2"]).ravel()
        g["conv2/bias"] = dz2.sum(axis=0)
        # conv-transpose per tap: da1[y+a, x+b, :] += dz2[y, x, :] @ W2[:, :, a, b]
        W2t = p["conv2/weights"].reshape(self.c2, self.c1, 3, 3)
        dzi = dz2.reshape(N, s2, s2, self.c2)
        da1 = np.zeros((N, s1, s1, self.c1))
        for a in range(3):
            for b in range(3):
                da1[:, a:a + s2, b:b + s2, :] += dzi @ W2t[:, :, a, b]
        da1 = da1.reshape(N * s1 * s1, self.c1)
        dz1 = da1 * (c["z1"] > 0.0)
        g["conv1/weights"] = (dz1.T @ c["cols1"]).ravel()
        g["conv1/bias"] = dz1.sum(axis=0)
        return loss, {n: g[n] for n in self.dims}

    def eval_counts(self, p, X, y):
        _, logits = self._forward(p, X)
        return _eval_rows(logits, y)


# ---------------------------------------------------- config C: transformer LM
# StackOverflow-shaped next-word model (BASELINE configs[2]; /root/reference/PAPER.md:
# 1052 "transformer model with 1962912 parameters", 1071-1085: embedding 96, 8 heads,
# feed-forward 1536, 3 layers, sequence length 20).  The reference ships no LM, so this
# oracle DEFINES the arithmetic (like Cnn above) and is pinned to float64 torch
# autograd (tests/test_oracle_lm.py).  1 962 912 = 10 004 * 96 (tied input / output
# embedding, no output bias) + 3 * 334 176 (PyTorch nn.TransformerEncoderLayer(96, 8,
# 1536) parameter set: in_proj, out_proj, linear1, linear2, norm1, norm2).
#   * post-norm encoder layers (norm_first=False), ReLU feed-forward, LayerNorm eps 1e-5;
#   * causal self-attention, sinusoidal positions, embedding scaled by sqrt(d_model);
#   * dropout off (the reference has no RNG stream for it, SURVEY.md section 8 Config A note);
#   * a datapoint is ONE sentence: features = L + 1 token ids (0 = pad), inputs
#     tokens[:L], targets tokens[1:]; pad targets are ignored;
#   * batch loss = mean cross-entropy over the batch's non-pad targets (0 if none);
#     eval_counts = (summed CE over non-pad targets, correct non-pad targets).
LM_PAD = 0


def lm_positions(L: int, d: int) -> np.ndarray:
    pos = np.arange(L, dtype=np.float64)[:, None]
    div = np.exp(np.arange(0, d, 2, dtype=np.float64) * (-np.log(10000.0) / d))
    pe = np.zeros((L, d))
    pe[:, 0::2] = np.sin(pos * div)
    pe[:, 1::2] = np.cos(pos * div[: d // 2])
    return pe


@dataclass(frozen=True)
class TransformerLM:
    vocab: int = 10004
    d: int = 96
    heads: int = 8
    ff: int = 1536
    layers: int = 3
    seq: int = 20
    eps: float = 1e-5

    @property
    def dims(self):
        d, f, out = self.d, self.ff, {"embedding": self.vocab * self.d}
        for l in range(self.layers):
            out.update({f"layer{l}/in_proj_weight": 3 * d * d, f"layer{l}/in_proj_bias": 3 * d,
                        f"layer{l}/out_proj_weight": d * d, f"layer{l}/out_proj_bias": d,
                        f"layer{l}/linear1_weight": f * d, f"layer{l}/linear1_bias": f,
                        f"layer{l}/linear2_weight": d * f, f"layer{l}/linear2_bias": d,
                        f"layer{l}/norm1_weight": d, f"layer{l}/norm1_bias": d,
                        f"layer{l}/norm2_weight": d, f"layer{l}/norm2_bias": d})
        return out

    def init(self, seed):
        """Weights N(0, 0.02^2) in dims order (one generator), biases 0, LayerNorm gains 1."""
        rng = np.random.default_rng(seed)
        out = {}
        for name, n in self.dims.items():
            if name.endswith("_bias"):
                out[name] = np.zeros(n)
            elif "norm" in name:
                out[name] = np.ones(n)
            else:
                out[name] = rng.normal(0.0, 0.02, n)
        return out

    def _ln(self, y, g, b):
        mu = y.mean(axis=-1, keepdims=True)
        var = ((y - mu) ** 2).mean(axis=-1, keepdims=True)
        rstd = 1.0 / np.sqrt(var + self.eps)
        xh = (y - mu) * rstd
        return xh * g + b, xh, rstd

    def _ln_back(self, dout, xh, rstd, g):
        dxh = dout * g
        return rstd * (dxh - dxh.mean(axis=-1, keepdims=True) - xh * (dxh * xh).mean(axis=-1, keepdims=True))

    def _forward(self, p, X):
        N, L, d, H = X.shape[0], self.seq, self.d, self.heads
        dh = d // H
        tok = X[:, :L].astype(np.int64)
        E = p["embedding"].reshape(self.vocab, d)
        x = E[tok] * np.sqrt(d) + lm_positions(L, d)
        causal = np.triu(np.ones((L, L), dtype=bool), 1)
        cache = []
        for l in range(self.layers):
            q = lambda n: p[f"layer{l}/{n}"]
            Wqkv, bqkv = q("in_proj_weight").reshape(3 * d, d), q("in_proj_bias")
            qkv = x @ Wqkv.T + bqkv                                             # N, L, 3d
            Q, K, V = (qkv[..., i * d:(i + 1) * d].reshape(N, L, H, dh).transpose(0, 2, 1, 3) for i in range(3))
            s = Q @ K.transpose(0, 1, 3, 2) / np.sqrt(dh)                      # N, H, L, L
            s = np.where(causal, -np.inf, s)
            P = np.exp(s - s.max(axis=-1, keepdims=True))
            P /= P.sum(axis=-1, keepdims=True)
            o = (P @ V).transpose(0, 2, 1, 3).reshape(N, L, d)
            a = o @ q("out_proj_weight").reshape(d, d).T + q("out_proj_bias")
            x1, xh1, r1 = self._ln(x + a, q("norm1_weight"), q("norm1_bias"))
            z = x1 @ q("linear1_weight").reshape(self.ff, d).T + q("linear1_bias")
            h = np.maximum(z, 0.0)
            f = h @ q("linear2_weight").reshape(d, self.ff).T + q("linear2_bias")
            x2, xh2, r2 = self._ln(x1 + f, q("norm2_weight"), q("norm2_bias"))
            cache.append(dict(x=x, Q=Q, K=K, V=V, P=P, o=o, x1=x1, xh1=xh1, r1=r1, z=z, h=h, xh2=xh2, r2=r2))
            x = x2
        logits = x @ E.T                                                        # N, L, V
        return tok, x, cache, logits

    def _targets(self, X):
        tgt = X[:, 1:self.seq + 1].astype(np.int64)
        return tgt, tgt != LM_PAD

    def loss_and_grad(self, p, X, y=None):
        N, L, d, H = X.shape[0], self.seq, self.d, self.heads
        dh = d // H
        tok, xL, cache, logits = self._forward(p, X)
        tgt, mask = self._targets(X)
        nv = int(mask.sum())
        z = logits - logits.max(axis=-1, keepdims=True)
        P = np.exp(z)
        P /= P.sum(axis=-1, keepdims=True)
        lp = np.log(np.take_along_axis(P, tgt[..., None], axis=-1)[..., 0])
        loss = float(-(lp * mask).sum() / nv) if nv else 0.0
        dl = P
        np.put_along_axis(dl, tgt[..., None], np.take_along_axis(dl, tgt[..., None], axis=-1) - 1.0, axis=-1)
        dl *= (mask / nv)[..., None] if nv else 0.0
        E = p["embedding"].reshape(self.vocab, d)
        g = {"embedding": np.einsum("nlv,nld->vd", dl, xL)}
        dx = dl @ E
        for l in reversed(range(self.layers)):
            c = cache[l]
            q = lambda n: p[f"layer{l}/{n}"]
            G = {}
            dy2 = dx
            G["norm2_weight"] = (dy2 * c["xh2"]).sum(axis=(0, 1))
            G["norm2_bias"] = dy2.sum(axis=(0, 1))
            dx1 = self._ln_back(dy2, c["xh2"], c["r2"], q("norm2_weight"))    # into x1 (both branches)
            W2 = q("linear2_weight").reshape(d, self.ff)
            G["linear2_weight"] = np.einsum("nld,nlf->df", dx1, c["h"])
            G["linear2_bias"] = dx1.sum(axis=(0, 1))
            dz = (dx1 @ W2) * (c["z"] > 0.0)
            W1 = q("linear1_weight").reshape(self.ff, d)
            G["linear1_weight"] = np.einsum("nlf,nld->fd", dz, c["x1"])
            G["linear1_bias"] = dz.sum(axis=(0, 1))
            dx1 = dx1 + dz @ W1
            G["norm1_weight"] = (dx1 * c["xh1"]).sum(axis=(0, 1))
            G["norm1_bias"] = dx1.sum(axis=(0, 1))
            dy1 = self._ln_back(dx1, c["xh1"], c["r1"], q("norm1_weight"))   # into x and a
            Wo = q("out_proj_weight").reshape(d, d)
            G["out_proj_weight"] = np.einsum("nli,nlj->ij", dy1, c["o"])
            G["out_proj_bias"] = dy1.sum(axis=(0, 1))
            do = (dy1 @ Wo).reshape(N, L, H, dh).transpose(0, 2, 1, 3)
            Pm = c["P"]
            dP = do @ c["V"].transpose(0, 1, 3, 2)
            dV = Pm.transpose(0, 1, 3, 2) @ do
            ds = Pm * (dP - (dP * Pm).sum(axis=-1, keepdims=True)) / np.sqrt(dh)
            dQ = ds @ c["K"]
            dK = ds.transpose(0, 1, 3, 2) @ c["Q"]
            dqkv = np.concatenate([t.transpose(0, 2, 1, 3).reshape(N, L, d) for t in (dQ, dK, dV)], axis=-1)
            Wqkv = q("in_proj_weight").reshape(3 * d, d)
            G["in_proj_weight"] = np.einsum("nlo,nli->oi", dqkv, c["x"])
            G["in_proj_bias"] = dqkv.sum(axis=(0, 1))
            dx = dy1 + dqkv @ Wqkv
            for k, v in G.items():
                g[f"layer{l}/{k}"] = v
        gE = g["embedding"]
        np.add.at(gE, tok.ravel(), dx.reshape(-1, d) * np.sqrt(d))
        return loss, {n: np.asarray(g[n]).ravel() for n in self.dims}

    def eval_counts(self, p, X, y=None):
        _, _, _, logits = self._forward(p, X)
        tgt, mask = self._targets(X)
        m = logits.max(axis=-1, keepdims=True)
        lse = np.log(np.exp(logits - m).sum(axis=-1))
        ce = -(np.take_along_axis(logits, tgt[..., None], axis=-1)[..., 0] - m[..., 0] - lse)
        hit = np.argmax(logits, axis=-1) == tgt
        return float((ce * mask).sum()), int((hit & mask).sum())


# ------------------------------------------------ config D: ResNet-18, multi-label
# FLAIR-shaped image model (BASELINE configs[3]; /root/reference/PAPER.md:1104-1138:
# ResNet-18, 17 coarse multi-label classes, cohort 200, E = 2, B = 16, central Adam).
# The reference ships no ResNet, so this oracle DEFINES the arithmetic and is pinned
# to float64 torch autograd (tests/test_oracle_resnet.py):
#   * torchvision's ResNet-18 layout (He et al. 2016): conv7x7/2 (pad 3) -> norm -> ReLU
#     -> maxpool 3x3/2 (pad 1) -> 4 stages x 2 BasicBlocks (widths w, 2w, 4w, 8w; stage
#     strides 1, 2, 2, 2; 1x1/stride conv + norm shortcut where the shape changes) ->
#     global average pool -> fc (8w -> K, with bias); convs without bias;
#   * GroupNorm(groups, C), eps 1e-5, in place of BatchNorm (the FLAIR benchmark's
#     choice for federated training: no cross-client batch statistics);
#   * maxpool ties go to the first maximum in row-major window order (PyTorch's);
#   * a datapoint is ONE image: features = 3 x S x S pixels in CHW order followed by K
#     label indicators (0 / 1);
#   * loss = sigmoid binary cross-entropy, per image the mean over its K labels, the
#     batch loss the mean over the batch's images (BCEWithLogits, reduction "mean");
#     eval_counts = (summed per-image loss, images whose K thresholded logits (z > 0)
#     all equal their labels -- exact-match accuracy).
def _conv_cols(x: np.ndarray, k: int, stride: int, pad: int):
    """NCHW x -> im2col [N*Ho*Wo, C*k*k] in (c, ky, kx) column order (OIHW flattening)."""
    N, C, H, W = x.shape
    xp = np.pad(x, ((0, 0), (0, 0), (pad, pad), (pad, pad))) if pad else x
    win = np.lib.stride_tricks.sliding_window_view(xp, (k, k), axis=(2, 3))[:, :, ::stride, ::stride]
    Ho, Wo = win.shape[2], win.shape[3]
    return win.transpose(0, 2, 3, 1, 4, 5).reshape(N * Ho * Wo, C * k * k), Ho, Wo


def _conv_back_input(dcols: np.ndarray, shape, k: int, stride: int, pad: int, Ho: int, Wo: int):
    N, C, H, W = shape
    d = dcols.reshape(N, Ho, Wo, C, k, k)
    dxp = np.zeros((N, C, H + 2 * pad, W + 2 * pad))
    for i in range(k):
        for j in range(k):
            dxp[:, :, i:i + stride * (Ho - 1) + 1:stride, j:j + stride * (Wo - 1) + 1:stride] += \
                d[:, :, :, :, i, j].transpose(0, 3, 1, 2)
    return dxp[:, :, pad:pad + H, pad:pad + W]


@dataclass(frozen=True)
class ResNet18:
    num_classes: int = 17
    width: int = 64
    groups: int = 32
    image: int = 224
    eps: float = 1e-5

    def blocks(self):
        """(name, c_in, c_out, stride, has_downsample) per BasicBlock."""
        out, cin = [], self.width
        for s in range(4):
            cout = self.width << s
            for b in range(2):
                stride = 2 if (s > 0 and b == 0) else 1
                out.append((f"layer{s + 1}.{b}", cin, cout, stride, stride != 1 or cin != cout))
                cin = cout
        return out

    @property
    def dims(self):
        w = self.width
        out = {"conv1.weight": w * 3 * 49, "gn1.weight": w, "gn1.bias": w}
        for name, ci, co, _, ds in self.blocks():
            out.update({f"{name}.conv1.weight": co * ci * 9, f"{name}.gn1.weight": co, f"{name}.gn1.bias": co,
                        f"{name}.conv2.weight": co * co * 9, f"{name}.gn2.weight": co, f"{name}.gn2.bias": co})
            if ds:
                out.update({f"{name}.downsample.0.weight": co * ci, f"{name}.downsample.1.weight": co,
                            f"{name}.downsample.1.bias": co})
        out.update({"fc.weight": self.num_classes * 8 * w, "fc.bias": self.num_classes})
        return out

    def init(self, seed):
        """Convs N(0, 2 / (c_out k^2)) (kaiming fan-out, torchvision), fc N(0, 1 / fan_in),
        norm gains 1, biases 0; one generator in dims order."""
        rng = np.random.default_rng(seed)
        out = {}
        for name, n in self.dims.items():
            if name.endswith("bias"):
                out[name] = np.zeros(n)
            elif ".gn" in name or name.startswith("gn") or "downsample.1" in name:
                out[name] = np.ones(n)
            elif name == "fc.weight":
                out[name] = rng.normal(0.0, 1.0 / np.sqrt(8 * self.width), n)
            else:
                k2 = 49 if name == "conv1.weight" else (1 if "downsample" in name else 9)
                out[name] = rng.normal(0.0, np.sqrt(2.0 / (self._cout(name) * k2)), n)
        return out

    def _cout(self, name):
        if name == "conv1.weight":
            return self.width
        blk = name.split(".conv")[0].split(".downsample")[0]
        return {b[0]: b[2] for b in self.blocks()}[blk]

    def _gn(self, x, g, b):
        N, C, H, W = x.shape
        G = self.groups
        xg = x.reshape(N, G, -1)
        mu = xg.mean(axis=-1, keepdims=True)
        var = ((xg - mu) ** 2).mean(axis=-1, keepdims=True)
        rstd = 1.0 / np.sqrt(var + self.eps)
        xh = ((xg - mu) * rstd).reshape(N, C, H, W)
        return xh * g[None, :, None, None] + b[None, :, None, None], xh, rstd

    def _gn_back(self, dy, xh, rstd, g):
        N, C, H, W = dy.shape
        G = self.groups
        dxh = (dy * g[None, :, None, None]).reshape(N, G, -1)
        xg = xh.reshape(N, G, -1)
        dx = rstd * (dxh - dxh.mean(axis=-1, keepdims=True) - xg * (dxh * xg).mean(axis=-1, keepdims=True))
        return dx.reshape(N, C, H, W), (dy * xh).sum(axis=(0, 2, 3)), dy.sum(axis=(0, 2, 3))

    def _conv(self, x, w, k, stride, pad):
        cols, Ho, Wo = _conv_cols(x, k, stride, pad)
        co = w.size // cols.shape[1]
        y = (cols @ w.reshape(co, -1).T).reshape(x.shape[0], Ho, Wo, co).transpose(0, 3, 1, 2)
        return y, cols

    def _conv_back(self, dy, cols, x_shape, w, k, stride, pad, need_dx=True):
        N, co, Ho, Wo = dy.shape
        d2 = dy.transpose(0, 2, 3, 1).reshape(-1, co)
        gw = (d2.T @ cols).ravel()
        if not need_dx:
            return None, gw
        return _conv_back_input(d2 @ w.reshape(co, -1), x_shape, k, stride, pad, Ho, Wo), gw

    def _split(self, X):
        S, K = self.image, self.num_classes
        return X[:, :3 * S * S].reshape(-1, 3, S, S), X[:, 3 * S * S:3 * S * S + K]

    def _forward(self, p, X):
        x, _ = self._split(X)
        N = x.shape[0]
        cache = {}
        c1, cols = self._conv(x, p["conv1.weight"], 7, 2, 3)
        a, xh, r = self._gn(c1, p["gn1.weight"], p["gn1.bias"])
        if TRACK_MARGINS:
            _record_margin(_relu_margin(a))
        a = np.maximum(a, 0.0)
        cache["stem"] = (x.shape, cols, xh, r, a)
        # maxpool 3x3/2 pad 1: first maximum in row-major window order
        ap = np.pad(a, ((0, 0), (0, 0), (1, 1), (1, 1)), constant_values=-np.inf)
        win = np.lib.stride_tricks.sliding_window_view(ap, (3, 3), axis=(2, 3))[:, :, ::2, ::2]
        Ho, Wo = win.shape[2], win.shape[3]
        win = win.reshape(N, a.shape[1], Ho, Wo, 9)
        arg = win.argmax(axis=-1)
        x = np.take_along_axis(win, arg[..., None], axis=-1)[..., 0]
        if TRACK_MARGINS:  # gap between a window's two largest values (exact ties of zeros excluded)
            srt = np.sort(win, axis=-1)
            live = srt[..., -1] > 0
            gap = (srt[..., -1] - srt[..., -2])[live]
            scale = float(np.sqrt(np.mean(a * a))) or 1.0
            _record_margin(float(gap.min()) / scale if gap.size else np.inf)
        cache["pool"] = (a.shape, arg, Ho, Wo)
        for name, ci, co, st, ds in self.blocks():
            q = lambda n: p[f"{name}.{n}"]
            t1, cols1 = self._conv(x, q("conv1.weight"), 3, st, 1)
            u1, xh1, r1 = self._gn(t1, q("gn1.weight"), q("gn1.bias"))
            if TRACK_MARGINS:
                _record_margin(_relu_margin(u1))
            u1 = np.maximum(u1, 0.0)
            t2, cols2 = self._conv(u1, q("conv2.weight"), 3, 1, 1)
            v2, xh2, r2 = self._gn(t2, q("gn2.weight"), q("gn2.bias"))
            if ds:
                td, colsd = self._conv(x, q("downsample.0.weight"), 1, st, 0)
                sc, xhd, rd = self._gn(td, q("downsample.1.weight"), q("downsample.1.bias"))
            else:
                sc, colsd, xhd, rd = x, None, None, None
            if TRACK_MARGINS:
                _record_margin(_relu_margin(v2 + sc))
            out = np.maximum(v2 + sc, 0.0)
            cache[name] = (x.shape, cols1, xh1, r1, u1, cols2, xh2, r2, colsd, xhd, rd, out)
            x = out
        feat = x.mean(axis=(2, 3))
        logits = feat @ p["fc.weight"].reshape(self.num_classes, -1).T + p["fc.bias"]
        cache["head"] = (x.shape, feat)
        return cache, logits

    @staticmethod
    def _bce(z, y):
        """per-element BCE with logits, stable form."""
        return np.maximum(z, 0.0) - z * y + np.log1p(np.exp(-np.abs(z)))

    def loss_and_grad(self, p, X, y=None):
        cache, z = self._forward(p, X)
        _, lab = self._split(X)
        N, K = z.shape
        loss = float(self._bce(z, lab).mean())
        dz = (1.0 / (1.0 + np.exp(-z)) - lab) / (N * K)
        g = {}
        shape4, feat = cache["head"]
        g["fc.weight"] = (dz.T @ feat).ravel()
        g["fc.bias"] = dz.sum(axis=0)
        dx = np.broadcast_to((dz @ p["fc.weight"].reshape(K, -1))[:, :, None, None], shape4) / (shape4[2] * shape4[3])
        for name, ci, co, st, ds in reversed(self.blocks()):
            q = lambda n: p[f"{name}.{n}"]
            xs, cols1, xh1, r1, u1, cols2, xh2, r2, colsd, xhd, rd, out = cache[name]
            dv = dx * (out > 0.0)
            dt2, g[f"{name}.gn2.weight"], g[f"{name}.gn2.bias"] = self._gn_back(dv, xh2, r2, q("gn2.weight"))
            if ds:
                dtd, g[f"{name}.downsample.1.weight"], g[f"{name}.downsample.1.bias"] = \
                    self._gn_back(dv, xhd, rd, q("downsample.1.weight"))
                dsc, g[f"{name}.downsample.0.weight"] = self._conv_back(dtd, colsd, xs, q("downsample.0.weight"),
                                                                       1, st, 0)
            else:
                dsc = dv
            du1, g[f"{name}.conv2.weight"] = self._conv_back(dt2, cols2, u1.shape, q("conv2.weight"), 3, 1, 1)
            du1 = du1 * (u1 > 0.0)
            dt1, g[f"{name}.gn1.weight"], g[f"{name}.gn1.bias"] = self._gn_back(du1, xh1, r1, q("gn1.weight"))
            dxin, g[f"{name}.conv1.weight"] = self._conv_back(dt1, cols1, xs, q("conv1.weight"), 3, st, 1)
            dx = dxin + dsc
        ashape, arg, Ho, Wo = cache["pool"]
        Nn, C, H, W = ashape
        dwin = np.zeros((Nn, C, Ho, Wo, 9))
        np.put_along_axis(dwin, arg[..., None], dx[..., None], axis=-1)
        dap = np.zeros((Nn, C, H + 2, W + 2))
        dwin = dwin.reshape(Nn, C, Ho, Wo, 3, 3)
        for i in range(3):
            for j in range(3):
                dap[:, :, i:i + 2 * (Ho - 1) + 1:2, j:j + 2 * (Wo - 1) + 1:2] += dwin[..., i, j]
        da = dap[:, :, 1:1 + H, 1:1 + W]
        xshape, cols, xh, r, a = cache["stem"]
        da = da * (a > 0.0)
        dc1, g["gn1.weight"], g["gn1.bias"] = self._gn_back(da, xh, r, p["gn1.weight"])
        _, g["conv1.weight"] = self._conv_back(dc1, cols, xshape, p["conv1.weight"], 7, 2, 3, need_dx=False)
        return loss, {n: np.asarray(g[n]).ravel() for n in self.dims}

    def eval_counts(self, p, X, y=None):
        _, z = self._forward(p, X)
        _, lab = self._split(X)
        per = self._bce(z, lab).mean(axis=1)
        hit = ((z > 0.0) == (lab > 0.5)).all(axis=1)
        return float(per.sum()), int(hit.sum())


# ------------------------------------------------------------ local work


def fit_local(model, params, X, y, perms, lr, batch_size, mu=0.0, control=None):
    """Generic Model.fit_local (fedsim/models/models.py:53-79): batches in
    perms order, tail batch kept, all entries updated after the gradient."""
    p = {n: v.copy() for n, v in params.items()}
    E, n = perms.shape
    for e in range(E):
        for s in range(0, n, batch_size):
            idx = perms[e, s:s + batch_size]
            _, g = model.loss_and_grad(p, X[idx], y[idx])
            for name in p:
                step = g[name]
                if mu != 0.0:
                    step = step + mu * (p[name] - params[name])
                if control is not None:
                    step = step + control[name]
                p[name] = p[name] - lr * step
    return p


def flat(params, dims) -> np.ndarray:
    return np.concatenate([np.asarray(params[n], dtype=np.float64).ravel() for n in dims])


@dataclass
class ContextResult:
    cohort: tuple
    queue: tuple
    loss_sum: np.ndarray          # per queue user
    correct: np.ndarray
    n: np.ndarray
    delta: np.ndarray | None = None   # [C, D] weighted (w_u * (theta_t - theta_u))
    norm: np.ndarray | None = None
    clipped: np.ndarray | None = None
    aggregate: np.ndarray | None = None   # clipped sum, before noise
    weight: float = 0.0
    noise: np.ndarray | None = None
    metrics: dict = field(default_factory=dict)
    user_updates: list = field(default_factory=list)


def run_context(model, theta: dict, users: dict, cohort_size: int, ctx_seed: int, *, train=None,
                weighting="datapoints", bound=None, sigma=0.0, r=1.0, noise_base=0, t=0, pop="train",
                world=1, rank=0, base_policy="median", noise=True, mu=0.0, scaffold=None):
    """One context of SimulationEngine._run_context (fedsim/engine/runtime.py:106-171)
    with FedAvg users (fedsim/algorithms/fedavg.py:127-180), ClippingPostprocessor
    (fedsim/privacy/clipping.py:105-146) and GaussianCentralMechanism
    (fedsim/privacy/mechanisms.py:146-193).  ``train`` = (lr, epochs, batch).
    ``mu``: FedProx proximal term (fedsim/algorithms/fedavg.py:218-227).
    ``scaffold``: dict(server=flat control, users={uid: flat control}) for
    Scaffold users (fedsim/algorithms/scaffold.py:46-79): the payload is
    [model delta | control delta] and ``res.user_updates`` the new controls."""
    ids = tuple(users)
    cohort = sample_cohort(ids, cohort_size, ctx_seed)
    w_all = {u: float(users[u][0].shape[0]) for u in cohort}
    base = lower_median(list(w_all.values())) if base_policy == "median" else 0.0
    queue = lpt_queues(w_all, world, base)[0][rank]
    dims = model.dims
    res = ContextResult(cohort, queue, np.zeros(len(queue)), np.zeros(len(queue), dtype=np.int64),
                        np.array([users[u][0].shape[0] for u in queue], dtype=np.int64))
    deltas, norms, clips = [], [], []
    for i, uid in enumerate(queue):
        X, y = users[uid]
        res.loss_sum[i], res.correct[i] = model.eval_counts(theta, X, y)
        if train is None:
            continue
        lr, E, B = train
        control = None
        if scaffold is not None:
            Dm = int(sum(dims.values()))
            uc = scaffold["users"].get(uid, np.zeros(Dm))
            control = _unflat(scaffold["server"] - uc, dims)
        after = (fit_local(model, theta, X, y, user_perms(ctx_seed, uid, X.shape[0], E), lr, B, mu=mu,
                           control=control) if E else theta)
        w = float(X.shape[0]) if weighting == "datapoints" else 1.0
        d = w * (flat(theta, dims) - flat(after, dims))       # fedsim/models/params.py:32-45
        if scaffold is not None:                              # fedsim/algorithms/scaffold.py:63-79
            steps = E * (-(-X.shape[0] // B))
            new_c = uc - scaffold["server"] + d * (1.0 / (steps * lr))
            res.user_updates.append((uid, new_c))
            d = np.concatenate([d, new_c - uc])
        nrm = float(np.linalg.norm(d))
        c = bound is not None and nrm > bound                 # fedsim/privacy/clipping.py:49
        if c:
            d = d * (bound / nrm)
        deltas.append(d)
        norms.append(nrm)
        clips.append(c)
        res.weight += w
    n = res.n.astype(np.float64)
    res.metrics = {"loss": (res.loss_sum.sum(), n.sum()), "accuracy": (float(res.correct.sum()), n.sum()),
                   "per_user_accuracy": ((res.correct / n).sum(), float(len(queue)))}
    if train is None:
        return res
    res.delta = np.array(deltas)
    res.norm = np.array(norms)
    res.clipped = np.array(clips)
    res.aggregate = res.delta.sum(axis=0)
    if bound is not None:
        std = r * sigma * bound
        res.metrics.update({"clip_fraction": (float(res.clipped.sum()), float(len(queue))),
                            "update_norm": (float(res.norm.sum()), float(len(queue))),
                            "clipping_bound": (bound, 1.0), "noise_std": (std, 1.0)})
        sig = float(np.linalg.norm(res.aggregate))
        if std > 0:
            res.metrics["snr"] = (sig / np.sqrt(res.aggregate.size * std**2), 1.0)
        if std > 0 and noise:
            rng = np.random.default_rng(noise_seed(noise_base, t, pop))
            groups = 2 if scaffold is not None else 1   # model/* entries, then control/*
            res.noise = np.concatenate([rng.normal(0.0, std, k) for _ in range(groups) for k in dims.values()])
    return res


def _unflat(v, dims):
    off = np.cumsum([0] + list(dims.values()))
    return {n: v[off[i]:off[i + 1]] for i, n in enumerate(dims)}


def central_sgd(theta_flat: np.ndarray, aggregate: np.ndarray, weight: float, lr: float, noise=None):
    """average -> SGD (fedsim/core/statistics.py:105-113, fedsim/models/optimizers.py:13-21);
    noise is added to the SUM first."""
    agg = aggregate if noise is None else aggregate + noise
    return theta_flat - lr * (agg * (1.0 / weight))


def central_adam(theta_flat: np.ndarray, aggregate: np.ndarray, weight: float, lr: float, state: dict,
                 beta1: float = 0.9, beta2: float = 0.99, eps: float = 0.1, noise=None):
    """average -> AdamOptimizer.step (fedsim/models/optimizers.py:24-68, float64).
    ``state`` carries m, v and the step count between calls (zero at start)."""
    g = (aggregate if noise is None else aggregate + noise) * (1.0 / weight)
    m = beta1 * state.get("m", np.zeros_like(g)) + (1 - beta1) * g
    v = beta2 * state.get("v", np.zeros_like(g)) + (1 - beta2) * g * g
    t = state.get("t", 0) + 1
    state.update(m=m, v=v, t=t)
    return theta_flat - lr * (m / (1 - beta1**t)) / (np.sqrt(v / (1 - beta2**t)) + eps)


def adafedprox_update_mu(mu, previous, current, dec=0.9, inc=1.1, floor=1e-4, cap=1.0):
    """fedsim/algorithms/fedavg.py:230-245."""
    if current < previous:
        return max(mu * dec, floor)
    if current > previous:
        return min(mu * inc, cap)
    return mu


def run_fedavg(model, train_users: dict, val_users: dict, *, iterations, cohort, eval_cohort, eval_every,
               lr, epochs, batch, clr, weighting, bound, sigma, r, noise_base, run_seed, init_seed, world=1,
               algorithm=None, optimizer=None):
    """run_simulation (fedsim/engine/loop.py:45-88) over FedAvg contexts
    (fedsim/algorithms/fedavg.py:97-125,183-198).  Returns per-iteration
    flat thetas, metric rows sorted by (population, name), cohort digest.
    ``algorithm``: None / dict(kind="fedprox"|"adafedprox", mu) /
    dict(kind="scaffold", num_train_users) (fedsim/algorithms/fedavg.py:201-296,
    fedsim/algorithms/scaffold.py:28-120); ``optimizer``: None (SGD at clr) or
    dict(kind="adam", lr, beta1, beta2, eps) (fedsim/models/optimizers.py:24-68)."""
    dims = model.dims
    theta = model.init(init_seed)
    algo = algorithm or dict(kind="fedavg")
    mu = float(algo.get("mu", 0.0)) if algo["kind"] in ("fedprox", "adafedprox") else 0.0
    prev_loss = None
    Dm = int(sum(dims.values()))
    scaffold = dict(server=np.zeros(Dm), users={}) if algo["kind"] == "scaffold" else None
    adam = {}
    thetas, rows = [], []
    digest = hashlib.sha256()
    for t in range(iterations):
        metrics = {}
        cohorts = []
        ctxs = [("train", train_users, cohort, True)]
        if t % eval_every == 0:
            ctxs.append(("val", val_users, eval_cohort, False))
        agg_state = None
        for pop, users, csize, train in ctxs:
            parts = [run_context(model, theta, users, csize, cohort_seed(run_seed, t, pop),
                                 train=(lr, epochs, batch) if train else None, weighting=weighting,
                                 bound=bound, sigma=sigma, r=r, noise_base=noise_base, t=t, pop=pop,
                                 world=world, rank=k, mu=mu, scaffold=scaffold if train else None)
                     for k in range(world)]
            cohorts.append((pop, parts[0].cohort))
            for k, v in _merge_parts(parts).items():
                metrics[(pop, k)] = v
            if train:
                agg = sum(p.aggregate for p in parts if len(p.queue))
                weight = sum(p.weight for p in parts)
                agg_state = (agg, weight, parts[0].noise)  # one draw per context (rank-independent)
            if train and scaffold is not None:
                for p in parts:
                    for uid, c in p.user_updates:
                        scaffold["users"][uid] = c
        if agg_state is not None:
            agg, weight, nz = agg_state
            ctrl = None
            if scaffold is not None:   # split the [model | control] payload
                ctrl = (agg[Dm:] + (nz[Dm:] if nz is not None else 0.0)) * (1.0 / weight)
                agg, nz = agg[:Dm], (nz[:Dm] if nz is not None else None)
            if optimizer is not None and optimizer["kind"] == "adam":
                new = central_adam(flat(theta, dims), agg, weight, optimizer["lr"], adam, optimizer["beta1"],
                                   optimizer["beta2"], optimizer["eps"], nz)
            else:
                new = central_sgd(flat(theta, dims), agg, weight, clr, nz)
            theta = _unflat(new, dims)
            if ctrl is not None:
                scaffold["server"] = scaffold["server"] + (weight / algo["num_train_users"]) * ctrl
        if algo["kind"] == "adafedprox" and ("train", "loss") in metrics:
            num, den = metrics[("train", "loss")]
            cur = num / den
            if prev_loss is not None:
                mu = adafedprox_update_mu(mu, prev_loss, cur)
            prev_loss = cur
        thetas.append(flat(theta, dims))
        for pop, c in cohorts:
            digest.update(repr((t, pop, c)).encode())
        rows.extend((t, pop, name, num / den, den) for (pop, name), (num, den) in sorted(metrics.items()))
    return np.array(thetas), rows, digest.hexdigest()


def _merge_parts(parts):
    """Sum per-rank metric (num, den) pairs; snr / noise_std / bound are
    computed once on the reduced aggregate."""
    out = {}
    for p in parts:
        for k, (num, den) in p.metrics.items():
            if k in ("snr", "noise_std", "clipping_bound"):
                continue
            a = out.get(k, (0.0, 0.0))
            out[k] = (a[0] + num, a[1] + den)
    ref = parts[0].metrics
    for k in ("noise_std", "clipping_bound"):
        if k in ref:
            out[k] = ref[k]
    if "noise_std" in ref and ref["noise_std"][0] > 0:
        agg = sum(p.aggregate for p in parts if len(p.queue))
        out["snr"] = (float(np.linalg.norm(agg)) / np.sqrt(agg.size * ref["noise_std"][0] ** 2), 1.0)
    return out
