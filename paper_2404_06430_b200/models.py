"""Model layouts and central optimizers for the GPU path.

A model here is a *layout*: ordered parameter entries (the payload order
of every flat device buffer), an initialiser that replays the reference's
numpy draws, and the geometry the sm_100a kernels need.  The arithmetic
lives in ``csrc/`` -- there is no host forward/backward (no CPU fallback).

* ``LogisticRegression`` -- fedsim/models/models.py:88-142 (zeros init).
* ``MLP``                -- fedsim/models/models.py:145-228
                            (U(+-1/sqrt(fan_in)) in entry order).
* ``CNN``                -- the BASELINE "small CIFAR-10 CNN", absent from
  the reference ("Assumed CNN"): conv3x3(3->32)+ReLU,
  conv3x3(32->64)+ReLU, maxpool 2x2, flatten(12544), fc128+ReLU, fc10,
  valid convolutions, no dropout.  D = 1,626,442.  Conv weights are
  [out][in][kh][kw], fc weights [in][out] (the reference's ``X @ W``
  convention); inputs are CHW rows of 3*32*32.  Initialised like the
  reference MLP: U(+-1/sqrt(fan_in)) drawn in entry order.
* ``TransformerLM``      -- config C's StackOverflow-shaped next-word model
  (1,962,912 parameters), also absent from the reference; see its docstring.
* ``ResNet18``           -- config D's FLAIR-shaped multi-label image model
  (11,185,233 parameters), also absent from the reference; see its docstring.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Mapping

import numpy as np

from .core import HyperParam, make_rng, resolve


class Model:
    """Layout contract shared by every model (fedsim/models/models.py:21-51)."""

    kind: str = ""

    @property
    def param_dims(self) -> dict[str, int]:
        raise NotImplementedError

    @property
    def num_params(self) -> int:
        return sum(self.param_dims.values())

    def init_params(self, seed: int) -> dict[str, np.ndarray]:
        raise NotImplementedError

    def _uniform_init(self, seed: int, fan_in: Mapping[str, int]) -> dict[str, np.ndarray]:
        rng = make_rng(seed)
        out = {}
        for name, n in self.param_dims.items():
            bound = 1.0 / np.sqrt(fan_in[name])
            out[name] = rng.uniform(-bound, bound, n)
        return out


@dataclass(frozen=True)
class LogisticRegression(Model):
    dim: int
    num_classes: int
    kind = "linear"

    @property
    def param_dims(self) -> dict[str, int]:
        return {"weights": self.dim * self.num_classes, "bias": self.num_classes}

    def init_params(self, seed: int) -> dict[str, np.ndarray]:
        return {n: np.zeros(k) for n, k in self.param_dims.items()}

    @property
    def input_dim(self) -> int:
        return self.dim


@dataclass(frozen=True)
class MLP(Model):
    dim: int
    hidden_units: int
    num_classes: int
    kind = "mlp"

    @property
    def param_dims(self) -> dict[str, int]:
        return {
            "layer1/weights": self.dim * self.hidden_units,
            "layer1/bias": self.hidden_units,
            "layer2/weights": self.hidden_units * self.num_classes,
            "layer2/bias": self.num_classes,
        }

    def init_params(self, seed: int) -> dict[str, np.ndarray]:
        # entries are drawn W1, b1, W2, b2 from one stream
        # (fedsim/models/models.py:162-175)
        d, h = self.dim, self.hidden_units
        return self._uniform_init(
            seed, {"layer1/weights": d, "layer1/bias": d, "layer2/weights": h, "layer2/bias": h}
        )

    @property
    def input_dim(self) -> int:
        return self.dim


@dataclass(frozen=True)
class CNN(Model):
    in_channels: int = 3
    image_size: int = 32
    conv1_channels: int = 32
    conv2_channels: int = 64
    hidden_units: int = 128
    num_classes: int = 10
    kind = "cnn"

    @property
    def conv1_out(self) -> int:  # spatial side after conv1 (valid 3x3)
        return self.image_size - 2

    @property
    def conv2_out(self) -> int:
        return self.image_size - 4

    @property
    def pool_out(self) -> int:
        return self.conv2_out // 2

    @property
    def flat_dim(self) -> int:
        return self.conv2_channels * self.pool_out * self.pool_out

    @property
    def input_dim(self) -> int:
        return self.in_channels * self.image_size * self.image_size

    @property
    def param_dims(self) -> dict[str, int]:
        c0, c1, c2 = self.in_channels, self.conv1_channels, self.conv2_channels
        return {
            "conv1/weights": c1 * c0 * 9,
            "conv1/bias": c1,
            "conv2/weights": c2 * c1 * 9,
            "conv2/bias": c2,
            "fc1/weights": self.flat_dim * self.hidden_units,
            "fc1/bias": self.hidden_units,
            "fc2/weights": self.hidden_units * self.num_classes,
            "fc2/bias": self.num_classes,
        }

    def init_params(self, seed: int) -> dict[str, np.ndarray]:
        c0, c1 = self.in_channels, self.conv1_channels
        fan = {
            "conv1/weights": c0 * 9, "conv1/bias": c0 * 9,
            "conv2/weights": c1 * 9, "conv2/bias": c1 * 9,
            "fc1/weights": self.flat_dim, "fc1/bias": self.flat_dim,
            "fc2/weights": self.hidden_units, "fc2/bias": self.hidden_units,
        }
        return self._uniform_init(seed, fan)

    def forward_flops_per_sample(self) -> int:
        """2 x MACs of one forward pass (33.67 MFLOP)."""
        s1, s2 = self.conv1_out, self.conv2_out
        macs = (
            s1 * s1 * self.conv1_channels * self.in_channels * 9
            + s2 * s2 * self.conv2_channels * self.conv1_channels * 9
            + self.flat_dim * self.hidden_units
            + self.hidden_units * self.num_classes
        )
        return 2 * macs


@dataclass(frozen=True)
class TransformerLM(Model):
    """Config C (BASELINE configs[2]): the StackOverflow-shaped next-word
    transformer -- vocabulary
    10 004, d_model 96, 8 heads, feed-forward 1536, 3 post-norm causal
    encoder layers, sequence length 20, tied input/output embedding without
    output bias: 1 962 912 parameters.  ReLU feed-forward, LayerNorm eps
    1e-5, sinusoidal positions added to the sqrt(d)-scaled embedding, no
    dropout.  Weight layouts are PyTorch's ([out, in] row-major).  A
    datapoint is one sentence of ``seq + 1`` token ids (0 = pad): inputs
    ids[:seq], targets ids[1:]; pad targets are ignored, the batch loss is
    the mean cross-entropy over the batch's non-pad targets.  The reference
    has no LM; the arithmetic is defined (and pinned to float64 autograd) by
    the oracle's TransformerLM.  Weights init N(0, 0.02^2) in entry order
    from one generator, biases 0, LayerNorm gains 1."""

    vocab: int = 10004
    d_model: int = 96
    heads: int = 8
    ff: int = 1536
    layers: int = 3
    seq: int = 20
    kind = "lm"

    @property
    def input_dim(self) -> int:
        return self.seq + 1

    @property
    def param_dims(self) -> dict[str, int]:
        d, f = self.d_model, self.ff
        out = {"embedding": self.vocab * d}
        for l in range(self.layers):
            out.update({f"layer{l}/in_proj_weight": 3 * d * d, f"layer{l}/in_proj_bias": 3 * d,
                        f"layer{l}/out_proj_weight": d * d, f"layer{l}/out_proj_bias": d,
                        f"layer{l}/linear1_weight": f * d, f"layer{l}/linear1_bias": f,
                        f"layer{l}/linear2_weight": d * f, f"layer{l}/linear2_bias": d,
                        f"layer{l}/norm1_weight": d, f"layer{l}/norm1_bias": d,
                        f"layer{l}/norm2_weight": d, f"layer{l}/norm2_bias": d})
        return out

    def init_params(self, seed: int) -> dict[str, np.ndarray]:
        rng = make_rng(seed)
        out = {}
        for name, n in self.param_dims.items():
            if name.endswith("_bias"):
                out[name] = np.zeros(n)
            elif "norm" in name:
                out[name] = np.ones(n)
            else:
                out[name] = rng.normal(0.0, 0.02, n)
        return out

    def forward_flops_per_token(self) -> int:
        """2 x MACs of one token's forward pass: projections, attention over the
        causal prefix (mean length (seq + 1) / 2) and the tied output layer."""
        d, f, L = self.d_model, self.ff, self.seq
        per_layer = 3 * d * d + d * d + 2 * d * f + d * (L + 1)  # (QK^T + PV: 2 * d * (L + 1) / 2)
        return 2 * (self.layers * per_layer + self.vocab * d)


@dataclass(frozen=True)
class ResNet18(Model):
    """Config D (BASELINE configs[3]): the FLAIR-shaped multi-label image model
    (ResNet-18, 17 coarse labels).
    torchvision's ResNet-18 layout -- conv7x7/2 -> norm -> ReLU -> maxpool
    3x3/2 -> 4 stages x 2 BasicBlocks (widths w, 2w, 4w, 8w) -> global average
    pool -> fc(8w -> K) -- with GroupNorm(``groups``, eps 1e-5) for BatchNorm
    (no cross-client batch statistics in federated training), no conv biases.
    Weight layouts are PyTorch's (OIHW convs, [out, in] fc).  A datapoint is
    one image: features = 3 x S x S CHW pixels then the K label indicators;
    the loss is the sigmoid BCE, per image the mean over its K labels, the batch
    loss the mean over its images; accuracy is exact-match.  The reference has
    no ResNet; the arithmetic is defined (and pinned to float64 autograd) by the
    oracle's ResNet18.  Init: convs N(0, 2 / (c_out k^2)) (kaiming fan-out), fc
    N(0, 1 / fan_in), norm gains 1, biases 0, one generator in entry order."""

    num_classes: int = 17
    width: int = 64
    groups: int = 32
    image: int = 224
    kind = "resnet"

    @property
    def input_dim(self) -> int:
        return 3 * self.image * self.image + self.num_classes

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
    def param_dims(self) -> dict[str, int]:
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

    def init_params(self, seed: int) -> dict[str, np.ndarray]:
        rng = make_rng(seed)
        cout = {b[0]: b[2] for b in self.blocks()}
        out = {}
        for name, n in self.param_dims.items():
            if name.endswith("bias"):
                out[name] = np.zeros(n)
            elif ".gn" in name or name.startswith("gn") or "downsample.1" in name:
                out[name] = np.ones(n)
            elif name == "fc.weight":
                out[name] = rng.normal(0.0, 1.0 / np.sqrt(8 * self.width), n)
            else:
                k2 = 49 if name == "conv1.weight" else (1 if "downsample" in name else 9)
                co = self.width if name == "conv1.weight" else cout[name.split(".conv")[0].split(".downsample")[0]]
                out[name] = rng.normal(0.0, np.sqrt(2.0 / (co * k2)), n)
        return out

    def forward_flops_per_image(self) -> int:
        """2 x MACs of one image's forward pass (convolutions and fc; norms,
        pooling and activations not counted)."""
        def conv(ci, co, k, hout):
            return ci * co * k * k * hout * hout
        S = self.image
        h = (S + 6 - 7) // 2 + 1
        macs = conv(3, self.width, 7, h)
        h = (h + 2 - 3) // 2 + 1
        for _, ci, co, st, ds in self.blocks():
            ho = (h + 2 - 3) // st + 1
            macs += conv(ci, co, 3, ho) + conv(co, co, 3, ho) + (conv(ci, co, 1, ho) if ds else 0)
            h = ho
        return 2 * (macs + 8 * self.width * self.num_classes)


def count_local_steps(num_points: int, local_params) -> int:
    """E * ceil(n / B) (fedsim/models/models.py:267-272)."""
    if num_points == 0:
        return 0
    return local_params.num_epochs * (-(-num_points // local_params.batch_size))


# --------------------------------------------------------------------------
# central optimizers (fedsim/models/optimizers.py:13-87)


class SGDOptimizer:
    """theta <- theta - lr * averaged_delta (fedsim/models/optimizers.py:13-21).

    On the GPU path the step is one fused kernel that also adds the
    pending central DP noise and divides by the total weight."""

    def __init__(self, learning_rate: "float | HyperParam"):
        self.learning_rate = learning_rate

    def step(self, params, direction, iteration: int):
        lr = resolve(self.learning_rate, iteration)
        if hasattr(direction, "apply_sgd"):
            return direction.apply_sgd(params, lr)
        return {n: params[n] - lr * direction[n] for n in params}


class AdamOptimizer:
    """Adam with bias correction, treating the averaged delta as gradient
    (fedsim/models/optimizers.py:24-68); ``adaptivity_degree`` is the epsilon
    added to the root of the bias-corrected second moment.

    On the GPU path the step is one fused kernel (fb_noise_avg_adam_f32) that
    also adds the pending central DP noise and divides by the total weight;
    the moments are flat fp32 device vectors."""

    def __init__(self, learning_rate: "float | HyperParam", beta1: float = 0.9, beta2: float = 0.99,
                 adaptivity_degree: float = 0.1):
        if not 0.0 <= beta1 < 1.0 or not 0.0 <= beta2 < 1.0:
            raise ValueError("betas must be in [0, 1)")
        if adaptivity_degree <= 0.0:
            raise ValueError("adaptivity_degree must be > 0")
        self.learning_rate = learning_rate
        self.beta1 = beta1
        self.beta2 = beta2
        self.adaptivity_degree = adaptivity_degree
        self.step_count = 0
        self.first_moment = None
        self.second_moment = None

    def step(self, params, direction, iteration: int):
        lr = resolve(self.learning_rate, iteration)
        if hasattr(direction, "apply_adam"):
            return direction.apply_adam(params, self, lr)
        # host dicts (unit tests of the mirror): the reference's float64 update
        if self.first_moment is None:
            self.first_moment = {n: np.zeros_like(v) for n, v in params.items()}
            self.second_moment = {n: np.zeros_like(v) for n, v in params.items()}
        self.step_count += 1
        t = self.step_count
        out = {}
        for name, theta in params.items():
            g = direction[name]
            m = self.beta1 * self.first_moment[name] + (1 - self.beta1) * g
            v = self.beta2 * self.second_moment[name] + (1 - self.beta2) * g * g
            self.first_moment[name] = m
            self.second_moment[name] = v
            m_hat = m / (1 - self.beta1**t)
            v_hat = v / (1 - self.beta2**t)
            out[name] = theta - lr * m_hat / (np.sqrt(v_hat) + self.adaptivity_degree)
        return out


CentralOptimizer = SGDOptimizer | AdamOptimizer


def central_step(optimizer, params, averaged_delta, iteration: int):
    """Apply one central update from an averaged delta (weight 1)
    (fedsim/models/optimizers.py:74-87)."""
    if averaged_delta.weight != 1.0:
        raise ValueError(
            "central_step expects an averaged delta (weight 1), "
            f"got weight {averaged_delta.weight}"
        )
    if hasattr(averaged_delta, "apply_sgd"):
        return optimizer.step(params, averaged_delta, iteration)
    return optimizer.step(params, averaged_delta.entries, iteration)
