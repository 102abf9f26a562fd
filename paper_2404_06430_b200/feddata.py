"""User datasets, cohort sampling and the synthetic data generator.

Host-side mirror of fedsim/feddata/{datasets,sampling,partition,
synthetic,io}.py.  Cohort sampling must be bit-exact with the reference
(north_star), so ``sample_cohort`` issues exactly the same numpy
``Generator`` calls as fedsim/feddata/sampling.py:25-39.  The generators
(synthetic data, IID split) also replay the reference's numpy call
sequence, so the same seeds give the same users on both sides.
"""

from __future__ import annotations

import csv
import logging
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .core import Population, make_rng
from .errors import CohortTooLarge, DataError, TooFewPoints

log = logging.getLogger(__name__)


@dataclass(frozen=True)
class UserDataset:
    """One user's rows: features [n, dim] and int labels [n]; weight = n
    (fedsim/feddata/datasets.py:12-40)."""

    user_id: str
    features: np.ndarray
    labels: np.ndarray

    def __post_init__(self) -> None:
        if self.features.ndim != 2:
            raise ValueError("features must be a (num_points, dim) array")
        if self.labels.shape != (self.features.shape[0],):
            raise ValueError("labels must be a vector aligned with features")
        if self.features.shape[0] < 1:
            raise ValueError("a user needs at least one datapoint")
        if not np.isfinite(self.features).all():
            raise ValueError("features contain non-finite values")

    @property
    def num_points(self) -> int:
        return int(self.features.shape[0])

    @property
    def weight(self) -> float:
        return float(self.num_points)


@dataclass(frozen=True)
class FederatedDataset:
    """Ordered users of one population (fedsim/feddata/datasets.py:43-65)."""

    users: dict[str, UserDataset]
    population: Population

    def __post_init__(self) -> None:
        for key, user in self.users.items():
            if key != user.user_id:
                raise ValueError(f"key {key!r} does not match user_id {user.user_id!r}")

    @property
    def num_users(self) -> int:
        return len(self.users)

    @property
    def user_ids(self) -> tuple[str, ...]:
        return tuple(self.users)

    @property
    def total_points(self) -> int:
        return sum(u.num_points for u in self.users.values())


def sample_cohort(
    dataset: FederatedDataset,
    cohort_size: int,
    seed: int,
    mode: str = "fixed",
    poisson_rate: float | None = None,
) -> tuple[str, ...]:
    """Cohort for one context, in seeded draw order.

    ``fixed``: ``default_rng(seed).choice(N, C, replace=False)``;
    ``poisson``: independent Bernoulli(rate) inclusion, possibly empty
    (fedsim/feddata/sampling.py:12-40).
    """
    ids = dataset.user_ids
    rng = make_rng(seed)
    if mode == "fixed":
        if cohort_size > len(ids):
            raise CohortTooLarge(f"cohort of {cohort_size} from {len(ids)} users")
        return tuple(ids[int(i)] for i in rng.choice(len(ids), size=cohort_size, replace=False))
    if mode == "poisson":
        if poisson_rate is None or not 0.0 < poisson_rate <= 1.0:
            raise ValueError("poisson mode needs a rate in (0, 1]")
        keep = rng.random(len(ids)) < poisson_rate
        return tuple(uid for uid, k in zip(ids, keep) if k)
    raise ValueError(f"unknown sampling mode {mode!r}")


def make_synthetic_classification(
    num_points: int, dim: int, num_classes: int, margin: float, seed: int
) -> tuple[np.ndarray, np.ndarray]:
    """Gaussian blobs: class centres ~ N(0, I) rescaled so the closest
    pair is ``margin`` apart, points = centre + N(0, I), balanced labels in
    shuffled order (fedsim/feddata/synthetic.py:10-51; same draw order)."""
    if dim < 1 or num_classes < 1:
        raise ValueError("dim and num_classes must be >= 1")
    if margin <= 0.0:
        raise ValueError("margin must be > 0")
    rng = make_rng(seed)
    if num_points == 0:
        return np.zeros((0, dim)), np.zeros(0, dtype=np.int64)

    def closest_pair(c: np.ndarray) -> float:
        d2 = ((c[:, None, :] - c[None, :, :]) ** 2).sum(axis=2)
        iu = np.triu_indices(num_classes, k=1)
        return float(np.sqrt(d2)[iu].min())

    centres = rng.normal(size=(num_classes, dim))
    if num_classes > 1:
        gap = closest_pair(centres)
        while gap < 1e-9:
            centres = rng.normal(size=(num_classes, dim))
            gap = closest_pair(centres)
        centres *= margin / gap
    per, extra = divmod(num_points, num_classes)
    counts = np.full(num_classes, per)
    counts[:extra] += 1
    labels = np.repeat(np.arange(num_classes, dtype=np.int64), counts)
    labels = labels[rng.permutation(num_points)]
    features = centres[labels] + rng.normal(size=(num_points, dim))
    return features, labels


LM_PAD, LM_BOS, LM_EOS, LM_OOV = 0, 1, 2, 3


def make_synthetic_sentences(
    num_users: int,
    *,
    vocab: int = 10004,
    seq: int = 20,
    max_sentences: int = 64,
    seed: int = 0,
    population: Population = Population.TRAIN,
    id_prefix: str = "u",
) -> FederatedDataset:
    """StackOverflow-shaped users for the config C language model (BASELINE
    configs[2]; <= 64 sentences per user,
    sequence length 20).  There is no dataset offline, so the shape is
    synthesised: sentences per user max(1, round(lognormal(3, 1))) capped at
    ``max_sentences`` (the ragged draw of fedsim/cli/bench.py:61-63); each
    sentence is [BOS, w_1 .. w_k, EOS] padded with PAD to ``seq + 1`` ids,
    k ~ U[1, seq - 1], words Zipf(1.2)-ranked over ids 4 .. vocab - 1 (OOV
    beyond).  A datapoint is one sentence: features = the seq + 1 ids (as
    float64, exact), label = its number of non-pad targets."""
    if num_users < 0 or seq < 2 or vocab < 5 or max_sentences < 1:
        raise ValueError("need num_users >= 0, seq >= 2, vocab >= 5, max_sentences >= 1")
    rng = make_rng(seed)
    sizes = np.clip(np.round(rng.lognormal(3.0, 1.0, size=num_users)), 1, max_sentences).astype(np.int64)
    users = {}
    for i, n in enumerate(sizes):
        k = rng.integers(1, seq, size=n)                       # real words per sentence
        ranks = rng.zipf(1.2, size=(n, seq - 1))
        words = np.where(ranks <= vocab - 4, ranks + 3, LM_OOV)
        X = np.full((n, seq + 1), LM_PAD, dtype=np.int64)
        X[:, 0] = LM_BOS
        for r in range(n):
            X[r, 1:k[r] + 1] = words[r, :k[r]]
            X[r, k[r] + 1] = LM_EOS
        uid = f"{id_prefix}{i:05d}"
        users[uid] = UserDataset(uid, X.astype(np.float64), (k + 1).astype(np.int64))
    return FederatedDataset(users=users, population=population)


def make_synthetic_images(
    num_users: int,
    *,
    image: int = 224,
    num_classes: int = 17,
    max_images: int = 500,
    seed: int = 0,
    population: Population = Population.TRAIN,
    id_prefix: str = "u",
) -> FederatedDataset:
    """FLAIR-shaped users for the config D ResNet-18 (BASELINE configs[3];
    /root/reference/PAPER.md:1104-1138: 1 - 500 (max 512) images per user, 17
    coarse multi-label classes).  There is no dataset offline, so the shape is
    synthesised: images per user max(1, round(lognormal(3, 1))) capped at
    ``max_images`` (the ragged draw of fedsim/cli/bench.py:61-63), pixels N(0, 1)
    (already normalised), each label present with probability 2 / K.  A datapoint
    is one image: features = its 3 x S x S CHW pixels followed by the K label
    indicators (float32), label = its number of positive labels."""
    if num_users < 0 or image < 32 or num_classes < 1 or max_images < 1:
        raise ValueError("need num_users >= 0, image >= 32, num_classes >= 1, max_images >= 1")
    rng = make_rng(seed)
    sizes = np.clip(np.round(rng.lognormal(3.0, 1.0, size=num_users)), 1, max_images).astype(np.int64)
    npx = 3 * image * image
    users = {}
    for i, n in enumerate(sizes):
        X = np.empty((n, npx + num_classes), dtype=np.float32)
        X[:, :npx] = rng.standard_normal((n, npx), dtype=np.float32)
        lab = rng.random((n, num_classes)) < 2.0 / num_classes
        X[:, npx:] = lab
        uid = f"{id_prefix}{i:05d}"
        users[uid] = UserDataset(uid, X, lab.sum(axis=1).astype(np.int64))
    return FederatedDataset(users=users, population=population)


def _users_from_chunks(features, labels, chunks, population, prefix) -> FederatedDataset:
    users = {}
    for i, idx in enumerate(chunks):
        uid = f"{prefix}{i:05d}"
        users[uid] = UserDataset(uid, features[idx], labels[idx].astype(np.int64))
    return FederatedDataset(users=users, population=population)


def partition_iid(
    features: np.ndarray,
    labels: np.ndarray,
    points_per_user: int,
    seed: int,
    population: Population = Population.TRAIN,
    id_prefix: str = "u",
) -> FederatedDataset:
    """Shuffle once and deal equal slices (fedsim/feddata/partition.py:28-57)."""
    if points_per_user < 1:
        raise ValueError("points_per_user must be >= 1")
    total = features.shape[0]
    num_users = total // points_per_user
    if num_users == 0:
        raise TooFewPoints(f"{total} points cannot fill a user of {points_per_user}")
    if total % points_per_user:
        log.warning("dropping %d points that do not fill a full user", total % points_per_user)
    order = make_rng(seed).permutation(total)
    chunks = [order[i * points_per_user:(i + 1) * points_per_user] for i in range(num_users)]
    return _users_from_chunks(features, labels, chunks, population, id_prefix)


def load_partition(path: str | Path, population: Population) -> FederatedDataset:
    """Read ``user_id,f0..f{d-1},label`` rows (fedsim/feddata/io.py:30-60)."""
    path = Path(path)
    if not path.exists():
        raise DataError(f"partition file not found: {path}")
    rows: dict[str, tuple[list, list]] = {}
    with path.open(newline="") as fh:
        reader = csv.reader(fh)
        header = next(reader, None)
        if header is None:
            raise DataError(f"partition file is empty: {path}")
        if header[0] != "user_id" or header[-1] != "label":
            raise DataError(f"unexpected partition header in {path}: {header}")
        dim = len(header) - 2
        for lineno, row in enumerate(reader, start=2):
            if len(row) != dim + 2:
                raise DataError(f"{path}:{lineno}: expected {dim + 2} columns")
            f, l = rows.setdefault(row[0], ([], []))
            f.append([float(x) for x in row[1:-1]])
            l.append(int(row[-1]))
    if not rows:
        raise DataError(f"partition file has no rows: {path}")
    users = {
        uid: UserDataset(uid, np.array(f, dtype=np.float64).reshape(len(l), dim),
                         np.array(l, dtype=np.int64))
        for uid, (f, l) in rows.items()
    }
    return FederatedDataset(users=users, population=population)


def save_partition(dataset: FederatedDataset, path: str | Path) -> None:
    with Path(path).open("w", newline="") as fh:
        w = csv.writer(fh)
        dim = next(iter(dataset.users.values())).features.shape[1]
        w.writerow(["user_id", *(f"f{i}" for i in range(dim)), "label"])
        for user in dataset.users.values():
            for feat, lab in zip(user.features, user.labels):
                w.writerow([user.user_id, *(repr(float(x)) for x in feat), int(lab)])
