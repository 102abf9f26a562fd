"""Device-resident forms of the path's value types.

* :class:`DeviceParams` -- model parameters as ONE flat fp32 HBM vector in
  entry order (the reference's ``ModelParams`` dict, fedsim/models/params.py:17).
* :class:`DeviceStatistics` -- the reduced cohort aggregate: the payload as a
  flat fp32 HBM vector, the ``_clip/*`` bookkeeping sums as host scalars,
  the total weight, and any *pending* central noise / averaging, which the
  central SGD step applies in one fused kernel (fb_noise_avg_sgd_f32).
* :class:`DevicePopulation` -- a FederatedDataset packed once into HBM:
  features fp32 [rows, dim] (users contiguous, dataset order), labels int32.
* :class:`Workspace` -- grow-only scratch buffers keyed by purpose (the C
  ABI never allocates).
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace
from typing import Iterator, Mapping, Sequence

import numpy as np

from . import native
from .core import Statistics
from .errors import IncompatibleShapes, ZeroWeight


def _torch():
    import torch

    return torch


class Workspace:
    """Named, grow-only device scratch (one per engine / device)."""

    def __init__(self, device):
        self.device = device
        self._bufs: dict[str, object] = {}

    def get(self, name: str, nbytes: int):
        torch = _torch()
        nbytes = max(int(nbytes), 16)
        buf = self._bufs.get(name)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            self._bufs[name] = buf
        return buf

    def tensor(self, name: str, shape, dtype):
        torch = _torch()
        n = int(np.prod(shape)) if len(shape) else 1
        esize = torch.empty((), dtype=dtype).element_size()
        return self.get(name, n * esize)[: n * esize].view(dtype).view(*shape)


def _offsets(dims: Mapping[str, int]) -> dict[str, tuple[int, int]]:
    out, o = {}, 0
    for n, k in dims.items():
        out[n] = (o, o + int(k))
        o += int(k)
    return out


class DeviceParams(Mapping):
    """Flat fp32 parameter vector with named views (entry order = dims order)."""

    def __init__(self, flat, dims: Mapping[str, int]):
        self.flat = flat
        self.dims = dict(dims)
        self._off = _offsets(self.dims)
        if flat.numel() != sum(self.dims.values()):
            raise IncompatibleShapes(f"flat has {flat.numel()} values, layout needs {sum(self.dims.values())}")

    @classmethod
    def from_host(cls, params: Mapping[str, np.ndarray], device) -> "DeviceParams":
        torch = _torch()
        dims = {n: int(np.asarray(v).size) for n, v in params.items()}
        host = np.concatenate([np.asarray(v, dtype=np.float64).ravel() for v in params.values()])
        return cls(torch.from_numpy(host.astype(np.float32)).to(device), dims)

    def __getitem__(self, name: str):
        lo, hi = self._off[name]
        return self.flat[lo:hi]

    def __iter__(self) -> Iterator[str]:
        return iter(self.dims)

    def __len__(self) -> int:
        return len(self.dims)

    @property
    def num_params(self) -> int:
        return self.flat.numel()

    def to_host(self) -> dict[str, np.ndarray]:
        host = self.flat.detach().to("cpu", dtype=_torch().float64).numpy()
        return {n: host[lo:hi].copy() for n, (lo, hi) in self._off.items()}

    def flat_host(self) -> np.ndarray:
        return self.flat.detach().to("cpu", dtype=_torch().float64).numpy()

    def clone(self) -> "DeviceParams":
        return DeviceParams(self.flat.clone(), self.dims)


@dataclass
class PendingNoise:
    std: float
    seed: int                      # Philox key (the reference's noise_seed value)
    injected: object | None = None  # device fp32 [D]: the reference's own draws (parity)


@dataclass
class Comm:
    """How the central epilogue is distributed (set by the engine)."""

    rank: int = 0
    world_size: int = 1
    group: object | None = None
    epilogue: str = "rank0"   # "rank0": step on rank 0 + broadcast; "replicated"

    def root(self) -> int:
        """Global rank of the group's rank 0 (broadcast takes global ranks)."""
        if self.group is None:
            return 0
        return _torch().distributed.get_global_rank(self.group, 0)


@dataclass
class DeviceStatistics:
    """Reduced aggregate.  ``flat`` holds the payload sum (un-averaged,
    un-noised); averaging and noise are recorded and applied lazily."""

    flat: object
    dims: dict[str, int]
    weight: float
    bookkeeping: dict[str, np.ndarray] = field(default_factory=dict)
    noise: PendingNoise | None = None
    scale: float = 1.0
    workspace: Workspace | None = None
    comm: Comm = field(default_factory=Comm)

    # ---- reference-compatible surface (fedsim/core/statistics.py:21-80)
    @property
    def entries(self) -> dict:
        out = {}
        for n, (lo, hi) in _offsets(self.dims).items():
            out[n] = self.flat[lo:hi]
        out.update(self.bookkeeping)
        return out

    @property
    def names(self) -> tuple[str, ...]:
        return tuple(self.dims) + tuple(self.bookkeeping)

    @property
    def payload_names(self) -> tuple[str, ...]:
        return tuple(self.dims)

    @property
    def num_dims(self) -> int:
        return self.flat.numel() + sum(int(v.size) for v in self.bookkeeping.values())

    # ---- device operations
    def device_norm(self, order: float, names) -> float:
        """L2 norm of the selected payload entries of the (un-noised, unscaled)
        aggregate, fp64 accumulation on the device."""
        if order != 2.0:
            raise ValueError("device aggregates support the L2 norm only")
        names = tuple(names)
        if names != tuple(self.dims):
            raise ValueError("device norm is defined over the whole payload")
        torch = _torch()
        ws = self.workspace or Workspace(self.flat.device)
        out = ws.tensor("sumsq_out", (1,), torch.float64)
        scratch = ws.get("sumsq_ws", 8192)
        native.call("fb_sumsq_f32", native.ptr(self.flat), self.flat.numel(), native.ptr(out),
                    native.ptr(scratch), scratch.numel(), native.stream_handle())
        return float(np.sqrt(out.item())) * abs(self.scale)

    def with_noise(self, std: float, seed: int, injected=None) -> "DeviceStatistics":
        if self.noise is not None:
            raise ValueError("aggregate already carries pending noise")
        return replace(self, noise=PendingNoise(float(std), int(seed), injected))

    def without_bookkeeping(self) -> "DeviceStatistics":
        return replace(self, bookkeeping={})

    def averaged(self) -> "DeviceStatistics":
        if self.weight == 0.0:
            raise ZeroWeight("cannot average statistics with zero total weight")
        return replace(self, scale=self.scale / self.weight, weight=1.0)

    def apply_sgd(self, params: DeviceParams, lr: float) -> DeviceParams:
        """theta_{t+1} = theta_t - lr * scale * (sum + noise): K4+K5 in one kernel.

        With a multi-rank engine the step runs on rank 0 and theta is
        broadcast (``epilogue="rank0"``), or identically on every rank from
        the counter-based noise (``"replicated"``)."""
        if params.num_params != self.flat.numel():
            raise IncompatibleShapes("aggregate and parameters differ in size")
        torch = _torch()
        out = params.flat.clone()
        comm = self.comm
        run_here = comm.world_size == 1 or comm.epilogue == "replicated" or comm.rank == 0
        if run_here:
            nz = self.noise
            native.call(
                "fb_noise_avg_sgd_f32", native.ptr(out), native.ptr(self.flat), self.flat.numel(),
                nz.std if nz else 0.0, nz.seed if nz else 0,
                native.ptr(nz.injected) if nz is not None and nz.injected is not None else None,
                float(self.scale), float(lr), None, native.stream_handle(),
            )
        if comm.world_size > 1 and comm.epilogue == "rank0":
            torch.distributed.broadcast(out, src=comm.root(), group=comm.group)
        return DeviceParams(out, params.dims)

    def apply_adam(self, params: DeviceParams, opt, lr: float) -> DeviceParams:
        """One central Adam step (fedsim/models/optimizers.py:24-68) on the
        averaged noised aggregate: K4 + Adam in one kernel.  The moments live
        on the device in ``opt`` (lazily zero on the first step, as the
        reference); multi-rank as :meth:`apply_sgd`."""
        if params.num_params != self.flat.numel():
            raise IncompatibleShapes("aggregate and parameters differ in size")
        torch = _torch()
        if opt.first_moment is None:
            opt.first_moment = torch.zeros_like(params.flat)
            opt.second_moment = torch.zeros_like(params.flat)
        opt.step_count += 1
        out = params.flat.clone()
        comm = self.comm
        run_here = comm.world_size == 1 or comm.epilogue == "replicated" or comm.rank == 0
        if run_here:
            nz = self.noise
            native.call(
                "fb_noise_avg_adam_f32", native.ptr(out), native.ptr(opt.first_moment), native.ptr(opt.second_moment),
                native.ptr(self.flat), self.flat.numel(), nz.std if nz else 0.0, nz.seed if nz else 0,
                native.ptr(nz.injected) if nz is not None and nz.injected is not None else None,
                float(self.scale), float(lr), float(opt.beta1), float(opt.beta2), float(opt.adaptivity_degree),
                int(opt.step_count), None, native.stream_handle(),
            )
        if comm.world_size > 1 and comm.epilogue == "rank0":
            torch.distributed.broadcast(out, src=comm.root(), group=comm.group)
        return DeviceParams(out, params.dims)

    def split_payload(self, sizes: Sequence[int]) -> list["DeviceStatistics"]:
        """Consecutive payload groups of an (averaged) aggregate as separate
        device statistics sharing its scale and weight; the pending noise is
        sliced the same way (Philox draws are materialised once for the whole
        vector so every element keeps its counter)."""
        torch = _torch()
        nz = self.noise
        full = None
        if nz is not None and nz.std != 0.0:
            full = nz.injected
            if full is None:
                full = torch.empty_like(self.flat)
                native.call("fb_gaussian_f32", native.ptr(full), full.numel(), nz.std, nz.seed, 0, 0,
                            native.stream_handle())
        out, lo = [], 0
        names = list(self.dims)
        for k in sizes:
            sub, acc = {}, 0
            while names and acc < k:
                n = names.pop(0)
                sub[n] = self.dims[n]
                acc += self.dims[n]
            if acc != k:
                raise IncompatibleShapes("payload groups do not align with the entries")
            noise = None if nz is None else PendingNoise(nz.std, nz.seed, None if full is None else full[lo:lo + k])
            out.append(replace(self, flat=self.flat[lo:lo + k], dims=sub, bookkeeping={}, noise=noise))
            lo += k
        return out

    def materialize(self):
        """Device fp32 payload with pending noise and scale applied."""
        torch = _torch()
        x = self.flat.clone()
        nz = self.noise
        if nz is not None:
            if nz.injected is not None:
                x += nz.injected
            elif nz.std != 0.0:
                native.call("fb_gaussian_f32", native.ptr(x), x.numel(), nz.std, nz.seed, 0, 1,
                            native.stream_handle())
        if self.scale != 1.0:
            x = (x.double() * self.scale).float()
        return x

    @classmethod
    def from_host(cls, stats, device, workspace: Workspace | None = None, comm: Comm | None = None) -> "DeviceStatistics":
        """Host statistics (entries name -> vector, ``_``-prefixed bookkeeping
        kept on the host) as a device aggregate with nothing pending."""
        torch = _torch()
        dims = {n: int(np.asarray(v).size) for n, v in stats.entries.items() if not n.startswith("_")}
        book = {n: np.asarray(v, dtype=np.float64) for n, v in stats.entries.items() if n.startswith("_")}
        host = (np.concatenate([np.asarray(stats.entries[n], dtype=np.float64).ravel() for n in dims])
                if dims else np.zeros(0))
        flat = torch.from_numpy(host.astype(np.float32)).to(device)
        return cls(flat=flat, dims=dims, weight=float(stats.weight), bookkeeping=book, workspace=workspace,
                   comm=comm if comm is not None else Comm())

    def to_host(self) -> Statistics:
        host = self.materialize().to("cpu", dtype=_torch().float64).numpy()
        entries = {n: host[lo:hi].copy() for n, (lo, hi) in _offsets(self.dims).items()}
        entries.update({n: np.array(v, dtype=np.float64) for n, v in self.bookkeeping.items()})
        return Statistics(entries=entries, weight=self.weight)


class DevicePopulation:
    """A FederatedDataset packed once (features fp32, labels int32).

    ``residency="device"`` keeps the packed arrays in HBM; ``"host"`` keeps
    them in pinned host memory and the engine gathers each context's cohort
    rows to the device (one fb_gather_rows launch reading host memory), the
    end-to-end data path."""

    def __init__(self, dataset, device, residency: str = "device"):
        if residency not in ("device", "host"):
            raise ValueError("residency must be 'device' or 'host'")
        self.residency = residency
        torch = _torch()
        users = list(dataset.users.values())
        if not users:
            raise ValueError("cannot pack an empty dataset")
        dims = {u.features.shape[1] for u in users}
        if len(dims) != 1:
            raise ValueError(f"users disagree on feature dim: {sorted(dims)}")
        self.dim = dims.pop()
        counts = np.array([u.num_points for u in users], dtype=np.int64)
        starts = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int64)
        self.index = {u.user_id: i for i, u in enumerate(users)}
        self.row_start = starts
        self.num_rows = counts.astype(np.int32)
        total = int(counts.sum())
        X = np.empty((total, self.dim), dtype=np.float32)
        y = np.empty(total, dtype=np.int32)
        for u, s in zip(users, starts):
            X[s:s + u.num_points] = u.features
            y[s:s + u.num_points] = u.labels
        if residency == "device":
            self.X = torch.from_numpy(X).to(device)
            self.y = torch.from_numpy(y).to(device)
        else:
            self.X = torch.from_numpy(X).pin_memory()
            self.y = torch.from_numpy(y).pin_memory()
        self.total_rows = total
        self.max_label = int(y.max()) if total else 0
        self.min_label = int(y.min()) if total else 0
        self._feature_range = None

    def _features(self):
        """(integral, min, max) of the features -- token-id datasets (the LM) index the
        embedding with them; computed once, on first use, where the rows live."""
        if self._feature_range is None:
            if self.total_rows == 0:
                self._feature_range = (True, 0.0, 0.0)
            else:
                X = self.X
                self._feature_range = (bool(_torch().equal(X, X.floor())), float(X.min()), float(X.max()))
        return self._feature_range

    @property
    def integral(self) -> bool:
        return self._features()[0]

    @property
    def min_feature(self) -> float:
        return self._features()[1]

    @property
    def max_feature(self) -> float:
        return self._features()[2]


class ControlStore:
    """Per-user SCAFFOLD control vectors on the device (the reference keeps
    them server-side keyed by user id, fedsim/algorithms/scaffold.py:34-57):
    one [capacity, ld] fp32 matrix plus a host user -> row map; a user
    without a row has the zero control."""

    def __init__(self, D: int, device):
        self.D = int(D)
        self.ld = (self.D + 3) & ~3
        self.device = device
        self.index: dict[str, int] = {}
        self.mat = None

    def __len__(self) -> int:
        return len(self.index)

    def __contains__(self, uid) -> bool:
        return uid in self.index

    def _reserve(self, n: int) -> None:
        torch = _torch()
        cap = 0 if self.mat is None else self.mat.shape[0]
        if n <= cap:
            return
        new = torch.zeros((max(n, 2 * cap, 16), self.ld), dtype=torch.float32, device=self.device)
        if self.mat is not None:
            new[:cap].copy_(self.mat)
        self.mat = new

    def rows_of(self, uids: Sequence[str]) -> np.ndarray:
        return np.fromiter((self.index.get(u, -1) for u in uids), dtype=np.int32, count=len(uids))

    def matrix(self):
        self._reserve(1)
        return self.mat

    def set_rows(self, uids: Sequence[str], src) -> None:
        """store[uid] = src[c] for every user (one scatter kernel)."""
        for u in uids:
            if u not in self.index:
                self.index[u] = len(self.index)
        self._reserve(len(self.index))
        torch = _torch()
        rows = torch.from_numpy(self.rows_of(uids)).to(self.device)
        native.call("fb_scatter_rows_f32", native.ptr(self.mat), self.ld, native.ptr(rows), native.ptr(src),
                    src.stride(0), len(uids), self.D, native.stream_handle())

    def get(self, uid: str) -> np.ndarray:
        """Host copy of one user's control (tests / inspection)."""
        if uid not in self.index:
            return np.zeros(self.D)
        return self.mat[self.index[uid], : self.D].double().cpu().numpy()


class ControlUpdates(list):
    """The engine's SCAFFOLD user updates: a list of (user_id, device row)
    pairs as the reference's ``user_updates`` (fedsim/algorithms/scaffold.py:79),
    with the batched [C, ld] matrix kept for a one-kernel store update."""

    def __init__(self, uids: Sequence[str], matrix):
        super().__init__((u, matrix[c]) for c, u in enumerate(uids))
        self.uids = list(uids)
        self.matrix = matrix
