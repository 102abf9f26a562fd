"""GpuSimulationEngine -- drop-in for fedsim's SimulationEngine.

Same constructor keywords and the same ``run_iteration(algorithm, state,
contexts) -> IterationResult`` as fedsim/engine/runtime.py:36-104 (the only
call the outer loop makes, fedsim/engine/loop.py:62).  Per context:

  host  sample_cohort -> compute_base_weight -> schedule_users(world)   bit-exact
        per-user seeds -> minibatch permutations (this rank's queue)     bit-exact
  H2D   one packed copy of the cohort descriptor
  GPU   eval at theta_t (K0) -> local SGD (K1) -> delta/norm/clip (K2)
        -> weighted sum (K3)                               [one stream]
  NCCL  all-reduce of the flat payload + fp64 all-reduce of the sums (N>1)
  D2H   per-client loss/correct/norm/clipped/non-finite flags (one copy)
  host  metrics, provenance errors, server postprocessors (reversed order)

The central step (noise + /W + SGD, K4+K5) runs when the algorithm folds
the aggregate back (``FedAvg.process_aggregated_statistics_all_contexts``)
because the returned DeviceStatistics carries the pending noise.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Any, Mapping, Sequence

import numpy as np

from . import cnn, interop, lm, native, resnet
from .core import CentralContext, MetricKind, MetricValue, Population, merge_metrics, user_seed
from .algorithms import CONTROL_PREFIX, MODEL_PREFIX
from .device import Comm, ControlStore, ControlUpdates, DeviceParams, DevicePopulation, DeviceStatistics, Workspace
from .errors import EngineError
from .feddata import FederatedDataset, sample_cohort
from .models import CNN, MLP, LogisticRegression, ResNet18, TransformerLM
from .privacy import CLIPPED_KEY, COUNT_KEY, NORM_KEY, validate_pipeline
from .scheduling import compute_base_weight, schedule_users


@dataclass
class IterationResult:
    aggregates: tuple
    metrics: dict[tuple[str, str], MetricValue]
    user_updates: list = field(default_factory=list)
    cohorts: tuple[tuple[str, tuple[str, ...]], ...] = ()


def _torch():
    import torch

    return torch


def client_permutations(ctx_seed: int, user_ids: Sequence[str], sizes: Sequence[int], epochs: int) -> list[np.ndarray]:
    """Per-user epoch shuffles: default_rng(user_seed(ctx, uid)).permutation(n)
    per epoch (fedsim/models/models.py:252-255 with fedsim/core/seeds.py:31)."""
    out = []
    for uid, n in zip(user_ids, sizes):
        rng = np.random.default_rng(user_seed(ctx_seed, uid))
        out.append(np.concatenate([rng.permutation(n) for _ in range(epochs)]) if epochs else
                   np.zeros(0, dtype=np.int64))
    return out


def plan_queues(dataset, ctx: CentralContext, world_size: int, *, cohort_mode: str = "fixed",
                poisson_rate: float | None = None, base_policy: str = "median", base_value: float = 0.0):
    """The cohort (identical on every rank: same seed, fedsim/feddata/sampling.py:12-40)
    and every rank's LPT queue over ``world_size`` workers
    (fedsim/engine/scheduling.py:34-78) -- the reference's worker assignment with
    num_workers = world_size."""
    cohort = sample_cohort(dataset, ctx.cohort_size, ctx.seed, mode=cohort_mode, poisson_rate=poisson_rate)
    if not cohort:
        return cohort, tuple(() for _ in range(world_size))
    weights = {uid: float(dataset.users[uid].weight) for uid in cohort}
    base = compute_base_weight(list(weights.values()), base_policy, base_value)
    return cohort, tuple(schedule_users(weights, world_size, base).queues)


def plan_shard(dataset, ctx: CentralContext, rank: int, world_size: int, **kw):
    """Host half of a context on one rank: the cohort and this rank's queue (:func:`plan_queues`)."""
    cohort, queues = plan_queues(dataset, ctx, world_size, **kw)
    return cohort, queues[rank]


# thread blocks of the prefetch gather kernel (each keeps 4 x 16 B x 256 threads in flight over PCIe)
PREFETCH_BLOCKS = 48
# cohorts whose rows form at most this many contiguous host runs are prefetched by the copy engines
PREFETCH_MAX_RUNS = 64
# largest single memcpy of a run (measured e2e: one copy per run 18.7 it/s, 8 MB chunks 18.5)
PREFETCH_CHUNK_BYTES = 1 << 30

# per-context sums reduced across ranks (FB_SUM_* in include/fedsim_b200.h), carried as fp32
# (hi, lo) pairs in the tail of the one buffer that is all-reduced
SUM_FIELDS = ("loss", "correct", "points", "per_user_acc", "users", "clipped", "count", "norm", "weight",
              "nonfinite")
NUM_SUMS = len(SUM_FIELDS)
TAIL = 2 * NUM_SUMS


def pack_sums(sums: np.ndarray) -> np.ndarray:
    """fp64 sums -> the fp32 (hi, lo) tail fb_context_sums writes."""
    s = np.asarray(sums, dtype=np.float64)
    hi = s.astype(np.float32)
    lo = (s - hi.astype(np.float64)).astype(np.float32)
    return np.stack([hi, lo], axis=1).ravel()


def unpack_sums(tail: np.ndarray) -> np.ndarray:
    t = np.asarray(tail, dtype=np.float32).astype(np.float64).reshape(-1, 2)
    return t[:, 0] + t[:, 1]


# Materialised payloads at least this wide go through the fused one-pass K2 + K3
# (clip_aggregate_fused.cu); below it the per-client grid handshake costs more than the
# second HBM pass it saves (aggregation microbench: fused 0.58 vs two-pass 0.49 of the
# roofline at D = 4 M, 0.37 vs 0.44 at 2 M).
FUSED_CLIP_AGGREGATE_MIN_D = 3_000_000

# CNN: evaluate each client's first local batch inside the first local-SGD step (same
# forward at theta_t) instead of a second time in the evaluation pass
SHARE_FIRST_BATCH_EVAL = True


def fused_clip_aggregate(D: int, ld: int, deferred: bool) -> bool:
    return (not deferred and D >= FUSED_CLIP_AGGREGATE_MIN_D and ld % 4 == 0
            and D <= native.call("fb_clip_aggregate_max_columns"))


def reduce_across_ranks(buf, group=None) -> None:
    """worker_reduce across ranks (fedsim/engine/aggregator.py:46-62): ONE
    all-reduce(SUM) of the flat fp32 buffer [payload | sums tail] (NCCL over
    NVLink on GPUs), in place.  No host synchronisation before it: the tail
    is written on the device by fb_context_sums."""
    _torch().distributed.all_reduce(buf, group=group)


def first_bad_user(local_pos: int, rank: int, world_size: int, group=None) -> tuple[int, int]:
    """(rank, queue position) of the first client with a non-finite update in
    rank-then-queue order -- the error the reference raises first (its worker
    futures are read in worker-index order, fedsim/engine/runtime.py:139-147).
    Collective over the group (error path only); local_pos < 0 = none here."""
    torch = _torch()
    big = (1 << 62)
    key = big if local_pos < 0 else (rank << 32) + local_pos
    if world_size > 1:
        dist = torch.distributed
        dev = (torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl"
               else torch.device("cpu"))
        t = torch.tensor([key], dtype=torch.int64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
        key = int(t.item())
    if key >= big:
        return -1, -1
    return key >> 32, key & 0xFFFFFFFF


def native_permutations(ctx_seed: int, user_ids: Sequence[str], num_rows: np.ndarray, epochs: int,
                        perm_off: np.ndarray, repr_cache: dict | None = None) -> np.ndarray:
    """Same draws as :func:`client_permutations`, computed by the library's
    native SHA-256 / SeedSequence / PCG64 restatement (fb_user_permutations):
    ~2 us per user instead of ~20 us through numpy."""
    cache = repr_cache if repr_cache is not None else {}
    reprs = []
    for uid in user_ids:
        r = cache.get(uid)
        if r is None:
            r = cache[uid] = repr(uid).encode()
        reprs.append(r)
    blob = np.frombuffer(b"".join(reprs) or b"\0", dtype=np.uint8)
    id_off = np.zeros(len(reprs) + 1, dtype=np.int64)
    np.cumsum([len(r) for r in reprs], out=id_off[1:])
    rows = np.ascontiguousarray(num_rows, dtype=np.int32)
    out = np.empty(max(int(rows.astype(np.int64).sum()) * epochs, 1), dtype=np.int32)
    native.check(native.load_library().fb_user_permutations(
        int(ctx_seed), blob.ctypes.data, id_off.ctypes.data, len(reprs), rows.ctypes.data, int(epochs),
        out.ctypes.data, np.ascontiguousarray(perm_off, dtype=np.int64).ctypes.data), "fb_user_permutations")
    return out[: int(rows.astype(np.int64).sum()) * epochs]


class _Staging:
    """Packs host arrays into one pinned buffer, one H2D copy, device views."""

    def __init__(self, device):
        self.device = device
        self._host = None
        self._dev = None

    def upload(self, arrays: Sequence[np.ndarray]):
        torch = _torch()
        offs, total = [], 0
        for a in arrays:
            offs.append(total)
            total += (a.nbytes + 15) & ~15
        total = max(total, 16)
        if self._host is None or self._host.numel() < total:
            self._host = torch.empty(total * 2, dtype=torch.uint8, pin_memory=True)
            self._dev = torch.empty(total * 2, dtype=torch.uint8, device=self.device)
        hv = self._host.numpy()
        for a, o in zip(arrays, offs):
            hv[o:o + a.nbytes] = np.ascontiguousarray(a).view(np.uint8).ravel()
        # read by a kernel from the pinned buffer (not a copy-engine memcpy; see fb_upload_pinned)
        native.call("fb_upload_pinned", native.ptr(self._host), native.ptr(self._dev), total, native.stream_handle())
        views = []
        for a, o in zip(arrays, offs):
            dt = {np.dtype(np.int64): torch.int64, np.dtype(np.int32): torch.int32,
                  np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64}[a.dtype]
            views.append(self._dev[o:o + a.nbytes].view(dt))
        return views


@dataclass
class _GatheredPopulation:
    """This context's cohort rows, gathered to the device in cohort order."""

    X: Any
    y: Any
    dim: int


class _ModelRunner:
    """Dispatches eval / local SGD to the model's fb_* entry points."""

    def __init__(self, model, ws: Workspace):
        self.model = model
        self.ws = ws
        if isinstance(model, MLP):
            self.kind, self.dims = "mlp", (model.dim, model.hidden_units, model.num_classes)
        elif isinstance(model, LogisticRegression):
            self.kind, self.dims = "linear", (model.dim, model.num_classes)
        elif isinstance(model, TransformerLM):
            self.kind, self.dims = "lm", ()
        elif isinstance(model, ResNet18):
            self.kind, self.dims = "resnet", ()
            if native.call("fb_resnet_num_params", resnet.dims_of(model).ctypes.data) != model.num_params:
                raise ValueError(f"GpuSimulationEngine: unsupported ResNet18 shape {model} (width a power of two "
                                 "in [4, 64], groups dividing it, image side in [32, 1024], classes <= 256)")
        elif isinstance(model, CNN):
            if model != CNN():  # csrc/cnn.cu is compiled for exactly this geometry
                raise ValueError(f"GpuSimulationEngine: the CNN kernels are compiled for {CNN()}, got {model}")
            self.kind, self.dims = "cnn", ()
        else:
            raise ValueError(f"GpuSimulationEngine: unsupported model {type(model).__name__}")
        self.D = model.num_params
        self.ld = (self.D + 3) & ~3  # 16-byte aligned client rows

    def eval(self, theta, pop: DevicePopulation, row_start, num_rows, C, loss, correct, stream, h_num_rows,
             skip_first=None):
        if self.kind == "cnn":
            return cnn.eval_cohort(self, theta, pop, row_start, num_rows, C, loss, correct, stream, h_num_rows,
                                   skip_first=skip_first)
        if self.kind == "lm":
            return lm.eval_cohort(self, theta, pop, row_start, num_rows, C, loss, correct, stream, h_num_rows,
                                  skip_first=skip_first)
        if self.kind == "resnet":
            return resnet.eval_cohort(self, theta, pop, row_start, num_rows, C, loss, correct, stream, h_num_rows,
                                      skip_first=skip_first)
        fn = f"fb_eval_{self.kind}_f32"
        native.call(fn, native.ptr(theta), *self.dims, native.ptr(pop.X), native.ptr(pop.y),
                    native.ptr(row_start), native.ptr(num_rows), C, native.ptr(loss), native.ptr(correct),
                    stream)

    def local_sgd(self, theta, pop, row_start, num_rows, perms, perm_off, C, tp, prox_mu, delta, nonfinite, stream,
                  h_num_rows, control=None, defer_fc1=False, eval_out=None):
        if self.kind == "cnn":  # returns the fc1-block sum of squares when the factored path made it
            return cnn.local_sgd_cohort(self, theta, pop, row_start, num_rows, perms, perm_off, C, tp,
                                        prox_mu, delta, nonfinite, stream, h_num_rows, control=control,
                                        defer_fc1=defer_fc1, eval_out=eval_out)
        if self.kind == "lm":
            return lm.local_sgd_cohort(self, theta, pop, row_start, num_rows, perms, perm_off, C, tp, prox_mu, delta,
                                       nonfinite, stream, h_num_rows, control=control, eval_out=eval_out)
        if self.kind == "resnet":
            return resnet.local_sgd_cohort(self, theta, pop, row_start, num_rows, perms, perm_off, C, tp, prox_mu,
                                           delta, nonfinite, stream, h_num_rows, control=control, eval_out=eval_out)
        fn = f"fb_local_sgd_{self.kind}_f32"
        native.call(fn, native.ptr(theta), *self.dims, native.ptr(pop.X), native.ptr(pop.y),
                    native.ptr(row_start), native.ptr(num_rows), native.ptr(perms), native.ptr(perm_off), C,
                    tp.num_epochs, tp.batch_size, float(tp.learning_rate), float(prox_mu),
                    native.ptr(control) if control is not None else None,
                    control.stride(0) if control is not None else 0,
                    native.ptr(delta), self.ld, native.ptr(nonfinite), stream)


class GpuSimulationEngine:
    """Runs central iterations with the whole cohort batched on B200(s).

    Multi-GPU: one process per GPU (torchrun); if ``torch.distributed`` is
    initialised, the cohort is sharded with the reference's LPT scheduler
    over ``world_size`` workers and rank r simulates ``queues[r]``.
    ``central_epilogue``: "rank0" (noise + step on rank 0, broadcast theta)
    or "replicated" (every rank applies the same counter-based noise).
    ``factored_aggregate`` (CNN): the fc1 block of the aggregate is formed from
    the clients' low-rank fc1 histories instead of materialised per-client
    deltas (``fb_cnn_fc1_aggregate_f32``); False keeps the materialising path.
    """

    def __init__(
        self,
        datasets: Mapping[Population, FederatedDataset],
        *,
        num_workers: int = 1,
        postprocessors: Sequence = (),
        aggregator=None,
        base_policy: str = "median",
        base_value: float = 0.0,
        cohort_mode: str = "fixed",
        poisson_rate: float | None = None,
        device=None,
        process_group=None,
        central_epilogue: str = "rank0",
        data_residency: str = "device",
        prefetch: bool = True,
        factored_aggregate: bool = True,
    ):
        if num_workers < 1:
            raise ValueError("num_workers must be >= 1")
        validate_pipeline(postprocessors)
        interop.check_postprocessors(postprocessors)   # the reference's own objects or this package's
        interop.check_aggregator(aggregator)
        if central_epilogue not in ("rank0", "replicated"):
            raise ValueError("central_epilogue must be 'rank0' or 'replicated'")
        if data_residency not in ("device", "host"):
            raise ValueError("data_residency must be 'device' or 'host'")
        self.data_residency = data_residency
        torch = _torch()
        native.lib()  # fail loudly: no CUDA device / no library => no engine
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        dist = torch.distributed
        if dist.is_available() and dist.is_initialized():
            self.rank = dist.get_rank(process_group)
            self.world_size = dist.get_world_size(process_group)
        else:
            self.rank, self.world_size = 0, 1
        self.group = process_group
        self._comm = Comm(self.rank, self.world_size, process_group, central_epilogue)
        self._datasets = dict(datasets)
        self._num_workers = int(num_workers)
        self._postprocessors = tuple(postprocessors)
        self._clip = next((p for p in postprocessors if interop.is_clipping(p)), None)
        self._aggregator = aggregator  # None or a SumAggregator: run as K3 + the rank all-reduce
        self._base_policy = base_policy
        self._base_value = float(base_value)
        self._cohort_mode = cohort_mode
        self._poisson_rate = poisson_rate
        self.ws = Workspace(self.device)
        self._staging = _Staging(self.device)
        self._pops: dict[Population, DevicePopulation] = {}
        self._runners: dict[int, _ModelRunner] = {}
        self._repr_cache: dict[str, bytes] = {}
        self.stream = torch.cuda.current_stream(self.device)
        self.io_bytes = {"h2d": 0, "d2h": 0}  # cumulative host<->device traffic of run_iteration
        # host-resident data: the next iteration's cohort rows are gathered on a copy
        # stream while this iteration computes (prefetching t+1 during t)
        self._prefetch = bool(prefetch) and data_residency == "host"
        # CNN: aggregate the fc1 block from the clients' low-rank histories (no per-client materialisation)
        self._factored_aggregate = bool(factored_aggregate)
        self._copy_stream = torch.cuda.Stream(self.device) if self._prefetch else None
        self._pf: dict = {}
        self._pf_bufs: dict = {}
        self._pf_done: dict = {}
        self._pf_pending = None
        self._plans: dict = {}      # host plans computed ahead (key: population, seed, cohort size, epochs)
        self._planned: set = set()
        # record_clients: keep this rank's queue and its per-client eval / norm / clip results of
        # the last context of each population (one extra D2H copy; tests and diagnostics)
        self.record_clients = False
        self.last_client_results: dict = {}
        self._theta_cache = None  # (host params object, its DeviceParams) for the reference's host params

    @property
    def num_workers(self) -> int:
        return self._num_workers

    @property
    def postprocessors(self) -> tuple:
        return self._postprocessors

    def population(self, pop: Population) -> DevicePopulation:
        if pop not in self._pops:
            self._pops[pop] = DevicePopulation(self._datasets[pop], self.device, self.data_residency)
        return self._pops[pop]

    def _runner(self, model) -> _ModelRunner:
        key = model  # frozen dataclass layouts: equal layouts share a runner
        if key not in self._runners:
            self._runners[key] = _ModelRunner(model, self.ws)
        return self._runners[key]

    # ------------------------------------------------------------------ API
    def run_iteration(self, algorithm, state, contexts: Sequence[CentralContext]) -> IterationResult:
        own = interop.is_own(algorithm)
        if not own and "FedAvg" not in interop.class_names(algorithm):
            raise ValueError(f"GpuSimulationEngine: unsupported algorithm {type(algorithm).__name__}")
        if own and not isinstance(state.params, DeviceParams):
            state.params = DeviceParams.from_host(state.params, self.device)
        aggregates, metrics, cohorts, updates = [], {}, [], []
        if self._prefetch and contexts:
            # iteration t+1's cohort-row copy is issued by the first context once its own
            # kernels are queued (the host work then overlaps them), so it runs beside this
            # iteration's kernels (run_iteration blocks on its per-client results further down)
            self._pf_pending = (algorithm, state, contexts[0].iteration + 1)
        for ctx in contexts:
            agg, ctx_metrics, cohort, ctx_updates = self._run_context(algorithm, state, ctx)
            if ctx_updates:
                updates = ctx_updates if not updates else updates + list(ctx_updates)
            aggregates.append(agg)
            pop = ctx.population.value
            for name, val in ctx_metrics.items():
                key = (pop, name)
                metrics[key] = metrics[key] + val if key in metrics else val
            cohorts.append((pop, cohort))
        self._issue_prefetch()
        if self._prefetch and contexts:
            done = _torch().cuda.Event()
            done.record(self.stream)  # every kernel of iteration t that reads its prefetched rows is before this
            self._pf_done[contexts[0].iteration & 1] = done
            self._pf.pop(contexts[0].iteration, None)
        return IterationResult(tuple(aggregates), metrics, updates, tuple(cohorts))

    def _issue_prefetch(self) -> None:
        pending, self._pf_pending = self._pf_pending, None
        if pending is not None:
            self._prefetch_next(*pending)

    def _prefetch_next(self, algorithm, state, t: int) -> None:
        """Gather iteration t's cohort rows (host-resident dataset) on the copy
        stream, overlapping the current iteration's kernels.  Used by
        _run_context only if the context it is given has the same population,
        seed and cohort size (so a mispredicted plan just falls back to the
        synchronous gather)."""
        torch = _torch()
        try:
            nxt = algorithm.get_next_central_contexts(state, t)
        except Exception:  # noqa: BLE001 -- prediction only
            return
        # buffers of this parity were last read by iteration t-2 (its end-of-iteration event)
        prev = self._pf_done.get(t & 1)
        if prev is not None:
            self._copy_stream.wait_event(prev)
        new = {}
        for k, ctx in enumerate(nxt):
            if ctx.population not in self._datasets:
                continue
            queue = self._peek_plan(ctx)["queue"]
            if not queue:
                continue
            pop = self.population(ctx.population)
            idx = np.fromiter((pop.index[u] for u in queue), dtype=np.int64, count=len(queue))
            num_rows = pop.num_rows[idx].astype(np.int32)
            # device layout in HOST order (users sorted by their rows' address): users adjacent in
            # the pinned dataset become one contiguous run, copied by the DMA engines with no SMs
            src = pop.row_start[idx].astype(np.int64)
            order = np.argsort(src, kind="stable")
            n_sorted = num_rows[order].astype(np.int64)
            dst = np.empty(len(queue), dtype=np.int64)
            dst[order] = np.concatenate([[0], np.cumsum(n_sorted[:-1])]) if len(queue) else n_sorted
            brk = np.flatnonzero(src[order][1:] != src[order][:-1] + n_sorted[:-1]) + 1
            run_lo = np.concatenate([[0], brk])
            run_hi = np.concatenate([brk, [len(queue)]])
            rows = int(num_rows.astype(np.int64).sum())
            key = (k, t & 1)
            bufs = self._pf_bufs.get(key)
            if bufs is None or bufs[0].shape[0] < rows or bufs[0].shape[1] != pop.dim:
                bufs = (torch.empty((max(rows, 1), pop.dim), dtype=torch.float32, device=self.device),
                        torch.empty((max(rows, 1),), dtype=torch.int32, device=self.device))
                self._pf_bufs[key] = bufs
            keep = None
            with torch.cuda.stream(self._copy_stream):
                if len(run_lo) <= PREFETCH_MAX_RUNS:  # copy engines: cudaMemcpyAsync per run (no SMs);
                    # the compute stream's own uploads go through fb_upload_pinned, so they never
                    # queue behind these copies
                    step = max(1, PREFETCH_CHUNK_BYTES // (4 * pop.dim))
                    for a, b in zip(run_lo, run_hi):
                        s0 = int(src[order[a]])
                        d0 = int(dst[order[a]])
                        n = int(n_sorted[a:b].sum())
                        for o in range(0, n, step):
                            m = min(step, n - o)
                            bufs[0][d0 + o:d0 + o + m].copy_(pop.X[s0 + o:s0 + o + m], non_blocking=True)
                        bufs[1][d0:d0 + n].copy_(pop.y[s0:s0 + n], non_blocking=True)
                    self.io_bytes["h2d"] += rows * (4 * pop.dim + 4)
                else:  # many scattered users: a few-block gather kernel beside the compute kernels
                    meta_h = torch.from_numpy(np.concatenate([src, dst, num_rows.astype(np.int64)])).pin_memory()
                    meta = meta_h.to(self.device, non_blocking=True)
                    C = len(queue)
                    src_d, dst_d = meta[:C], meta[C:2 * C]
                    nr_d = meta[2 * C:].to(torch.int32)
                    cs = native.stream_handle(self._copy_stream)
                    native.call("fb_gather_rows_lite", native.ptr(pop.X), 4 * pop.dim, native.ptr(src_d),
                                native.ptr(nr_d), C, native.ptr(dst_d), native.ptr(bufs[0]), PREFETCH_BLOCKS, cs)
                    native.call("fb_gather_rows_lite", native.ptr(pop.y), 4, native.ptr(src_d), native.ptr(nr_d), C,
                                native.ptr(dst_d), native.ptr(bufs[1]), PREFETCH_BLOCKS, cs)
                    keep = (meta_h, meta, nr_d)
                    self.io_bytes["h2d"] += int(meta_h.numel()) * 8 + rows * (4 * pop.dim + 4)
                ev = torch.cuda.Event()
                ev.record(self._copy_stream)
            new[(ctx.population, ctx.seed, ctx.cohort_size)] = dict(queue=tuple(queue), X=bufs[0], y=bufs[1],
                                                                    dst=dst, event=ev, keep=keep)
        self._pf[t] = new

    # ------------------------------------------------------------ internals
    def _gather_controls(self, queues, local, ld: int):
        """SCAFFOLD across ranks: all-gather the new per-user controls of every
        rank's shard (padded to the longest queue) so each rank's replicated
        control store sees the whole cohort's updates, in rank-then-queue order
        (the reference merges its workers' user_updates,
        fedsim/engine/runtime.py:95-104)."""
        torch = _torch()
        cmax = max(max((len(q) for q in queues), default=0), 1)
        buf = torch.zeros((cmax, ld), dtype=torch.float32, device=self.device)
        if local is not None and len(local):
            buf[: len(local)].copy_(local.matrix[: len(local)])
        outs = [torch.empty_like(buf) for _ in range(self.world_size)]
        torch.distributed.all_gather(outs, buf, group=self.group)
        uids = [u for q in queues for u in q]
        if not uids:
            return None
        return ControlUpdates(uids, torch.cat([o[: len(q)] for o, q in zip(outs, queues)]))

    def _host_plan(self, ctx: CentralContext) -> dict:
        """Cohort, this rank's LPT queue and (training) the minibatch permutations of
        one context -- computed ahead by _plan_ahead when possible."""
        epochs = ctx.local_params.num_epochs if ctx.do_training and ctx.local_params is not None else 0
        key = (ctx.population, ctx.seed, ctx.cohort_size, epochs)
        hp = self._plans.pop(key, None)
        if hp is not None:
            return hp
        dataset = self._datasets[ctx.population]
        cohort, queues = plan_queues(dataset, ctx, self.world_size, cohort_mode=self._cohort_mode,
                                     poisson_rate=self._poisson_rate, base_policy=self._base_policy,
                                     base_value=self._base_value)
        return {"cohort": cohort, "queue": queues[self.rank], "queues": queues}

    def _peek_plan(self, ctx: CentralContext) -> dict:
        """The context's host plan, computed now if needed and kept for _run_context."""
        epochs = ctx.local_params.num_epochs if ctx.do_training and ctx.local_params is not None else 0
        key = (ctx.population, ctx.seed, ctx.cohort_size, epochs)
        if key not in self._plans:
            self._plans[key] = self._host_plan(ctx)
        return self._plans[key]

    def _plan_ahead(self, algorithm, state, t: int) -> None:
        """Prefetch the host work of iteration t: same seeds, same calls."""
        if t in self._planned:
            return
        self._planned = {t}
        try:
            nxt = algorithm.get_next_central_contexts(state, t)
        except Exception:  # noqa: BLE001 -- prediction only
            return
        for ctx in nxt:
            if ctx.population not in self._datasets:
                continue
            hp = self._peek_plan(ctx)
            epochs = ctx.local_params.num_epochs if ctx.do_training and ctx.local_params is not None else 0
            if epochs and hp["queue"] and "perms" not in hp:
                pop = self.population(ctx.population)
                idx = np.fromiter((pop.index[u] for u in hp["queue"]), dtype=np.int64, count=len(hp["queue"]))
                num_rows = pop.num_rows[idx]
                perm_off = np.zeros(len(idx), dtype=np.int64)
                if len(idx) > 1:
                    perm_off[1:] = np.cumsum(num_rows[:-1].astype(np.int64) * epochs)
                hp["perms"] = native_permutations(ctx.seed, hp["queue"], num_rows, epochs, perm_off,
                                                  self._repr_cache)

    def _theta(self, state) -> DeviceParams:
        """theta_t on the device.  This package's algorithms keep it there; the
        reference's keep host float64 ModelParams (fedsim/models/params.py:17),
        uploaded once per new params object (one per iteration)."""
        if isinstance(state.params, DeviceParams):
            return state.params
        cached = self._theta_cache
        if cached is None or cached[0] is not state.params:
            cached = self._theta_cache = (state.params, DeviceParams.from_host(state.params, self.device))
        return cached[1]

    def _clip_bound(self) -> float:
        return float(self._clip.current_bound) if self._clip is not None else 0.0

    def _host_controls(self, state, queue, D: int):
        """The reference's Scaffold keeps controls on the host (fedsim/algorithms/
        scaffold.py:34-57): server control and the queue's user controls are
        uploaded into a transient device store for the correction / payload kernels."""
        torch = _torch()
        names = list(state.params)
        server_h = state.extra["server_control"]
        server = torch.from_numpy(np.concatenate([np.asarray(server_h[n], dtype=np.float64).ravel()
                                                  for n in names]).astype(np.float32)).to(self.device)
        store = ControlStore(D, self.device)
        users = state.extra["user_controls"]
        known = [u for u in queue if u in users]
        if known:
            mat = np.stack([np.concatenate([np.asarray(users[u][n], dtype=np.float64).ravel() for n in names])
                            for u in known]).astype(np.float32)
            store.set_rows(known, torch.from_numpy(mat).to(self.device))
        return server, store

    def _host_updates(self, updates, state):
        """ControlUpdates -> the reference's user_updates: (uid, {name: float64 vector})."""
        if updates is None:
            return []
        names = list(state.params)
        offs = np.cumsum([0] + [int(np.asarray(state.params[n]).size) for n in names])
        mat = updates.matrix[:, : offs[-1]].double().cpu().numpy() if len(updates.uids) else None
        return [(u, {n: mat[c, offs[i]:offs[i + 1]].copy() for i, n in enumerate(names)})
                for c, u in enumerate(updates.uids)]

    def _controls(self, state, D: int):
        """SCAFFOLD server control (flat fp32) and per-user control store,
        created on the device on first use (zero, as the reference)."""
        torch = _torch()
        if state.extra.get("server_control") is None:
            state.extra["server_control"] = torch.zeros(D, dtype=torch.float32, device=self.device)
        if state.extra.get("user_controls") is None:
            state.extra["user_controls"] = ControlStore(D, self.device)
        return state.extra["server_control"], state.extra["user_controls"]

    def _run_context(self, algorithm, state, ctx: CentralContext):
        torch = _torch()
        pop_key = ctx.population
        dataset = self._datasets.get(pop_key)
        if dataset is None:
            raise EngineError(f"iteration {ctx.iteration}: no dataset for population {pop_key.value!r}")
        hp = self._host_plan(ctx)
        cohort, queue = hp["cohort"], hp["queue"]
        if not cohort:
            return None, {}, cohort, None

        plan = interop.cohort_plan(algorithm, state, ctx)
        own = interop.is_own(algorithm)
        runner = self._runner(plan.model)
        scaffold = bool(getattr(plan, "scaffold", False)) and plan.train is not None
        pop = self.population(pop_key)
        if pop.dim != plan.model.input_dim:
            raise ValueError(f"dataset dim {pop.dim} != model input dim {plan.model.input_dim}")
        if runner.kind == "lm":  # sentences of token ids: the kernels index the embedding with them
            if pop.total_rows and (not pop.integral or pop.min_feature < 0 or pop.max_feature >= plan.model.vocab):
                raise ValueError(f"population {pop_key.value!r}: token ids must be integers in "
                                 f"[0, {plan.model.vocab}), got [{pop.min_feature}, {pop.max_feature}]")
        elif runner.kind == "resnet":  # (multi-label: the K label indicators ride at the end of each row)
            pass
        elif pop.total_rows and (pop.min_label < 0 or pop.max_label >= plan.model.num_classes):
            raise ValueError(f"labels of population {pop_key.value!r} lie in [{pop.min_label}, {pop.max_label}], "
                             f"outside the model's {plan.model.num_classes} classes")
        theta = self._theta(state)
        C = len(queue)
        stream = native.stream_handle(self.stream)
        idx = np.fromiter((pop.index[u] for u in queue), dtype=np.int64, count=C)
        row_start = pop.row_start[idx]
        num_rows = pop.num_rows[idx]
        train = plan.train is not None
        gathered = pop.residency == "host"
        pf = None
        if gathered:  # kernels see the cohort's rows packed on the device (prefetch layout or cohort order)
            src_start = row_start
            pf = self._pf.get(ctx.iteration, {}).pop((pop_key, ctx.seed, ctx.cohort_size), None)
            if pf is not None and pf["queue"] != tuple(queue):
                pf = None
            if pf is not None:
                row_start = pf["dst"].copy()
            else:
                row_start = np.zeros(C, dtype=np.int64)
                if C > 1:
                    row_start[1:] = np.cumsum(num_rows[:-1].astype(np.int64))
        host = [row_start, num_rows]
        if train:
            tp = plan.train
            perm_off = np.zeros(C, dtype=np.int64)
            if C > 1:
                perm_off[1:] = np.cumsum(num_rows[:-1].astype(np.int64) * tp.num_epochs)
            perm_flat = hp.get("perms")
            if perm_flat is None or len(perm_flat) != int(num_rows.astype(np.int64).sum()) * tp.num_epochs:
                perm_flat = native_permutations(ctx.seed, queue, num_rows, tp.num_epochs, perm_off, self._repr_cache)
            w = (num_rows.astype(np.float32) if plan.weighting == "datapoints"
                 else np.ones(C, dtype=np.float32))
            host += [perm_flat, perm_off, w]
            if scaffold:  # control update scale 1 / (steps * lr) (fedsim/algorithms/scaffold.py:46-70)
                # checked over every rank's queue (in rank order) so all ranks raise together
                for q in hp.get("queues", (queue,)):
                    n_q = np.fromiter((dataset.users[u].num_points for u in q), dtype=np.int64, count=len(q))
                    steps_q = tp.num_epochs * (-(-n_q // tp.batch_size))
                    bad = np.flatnonzero(steps_q.astype(np.float64) * float(tp.learning_rate) == 0.0)
                    if len(bad):
                        raise EngineError(
                            f"iteration {ctx.iteration}, population {pop_key.value!r}, user {q[int(bad[0])]!r}: "
                            f"control update divides by steps * learning_rate; got {int(steps_q[bad[0]])} steps "
                            f"at lr {tp.learning_rate}")
                steps = tp.num_epochs * (-(-num_rows.astype(np.int64) // tp.batch_size))
                denom = steps.astype(np.float64) * float(tp.learning_rate)
                ctrl_scale = (1.0 / denom).astype(np.float32) if C else np.zeros(0, dtype=np.float32)
        if gathered:
            host.append(src_start)
        dev = self._staging.upload(host)
        self.io_bytes["h2d"] += sum(int(a.nbytes) for a in host)
        d_row_start, d_num_rows = dev[0], dev[1]
        if pf is not None:  # rows already on the device (copy stream)
            self.stream.wait_event(pf["event"])
            pop = _GatheredPopulation(pf["X"], pf["y"], pop.dim)
        elif gathered:
            rows = int(num_rows.sum())
            gX = self.ws.tensor("gather_X", (max(rows, 1), pop.dim), torch.float32)
            gy = self.ws.tensor("gather_y", (max(rows, 1),), torch.int32)
            mx = int(num_rows.max()) if C else 0
            native.call("fb_gather_rows", native.ptr(pop.X), 4 * pop.dim, native.ptr(dev[-1]), native.ptr(d_num_rows),
                        C, native.ptr(d_row_start), native.ptr(gX), mx, stream)
            native.call("fb_gather_rows", native.ptr(pop.y), 4, native.ptr(dev[-1]), native.ptr(d_num_rows), C,
                        native.ptr(d_row_start), native.ptr(gy), mx, stream)
            self.io_bytes["h2d"] += rows * (4 * pop.dim + 4)
            pop = _GatheredPopulation(gX, gy, pop.dim)

        # per-client result block: loss f64, norm f64 | correct, clipped, nonfinite i32
        Cp = max(C, 1)
        res = self.ws.get("client_results", 8 * Cp * 2 + 4 * Cp * 3)
        loss = res[: 8 * Cp].view(torch.float64)
        norm = res[8 * Cp: 16 * Cp].view(torch.float64)
        ints = res[16 * Cp: 16 * Cp + 12 * Cp].view(torch.int32)
        correct, clipped, nonfinite = ints[:Cp], ints[Cp:2 * Cp], ints[2 * Cp:3 * Cp]
        # CNN / LM training contexts: the first local step runs at theta_t, so its forward IS the
        # evaluation of the first batch (fedsim/algorithms/fedavg.py:165 evaluates every row at
        # theta_t before training): evaluate only epoch 0's remaining rows here and let the
        # local-SGD call add the first batch's loss / hits
        share0 = bool(train and C and runner.kind in ("cnn", "lm", "resnet") and plan.train is not None
                      and plan.train.num_epochs >= 1 and SHARE_FIRST_BATCH_EVAL)
        if C:
            runner.eval(theta.flat, pop, d_row_start, d_num_rows, C, loss, correct, stream, num_rows,
                        skip_first=(dev[2], dev[3], plan.train.batch_size) if share0 else None)
        self._issue_prefetch()  # next iteration's rows: host work now overlaps the queued kernels

        agg_flat = None
        updates = None
        d_w = None
        if train:
            d_perms, d_perm_off, d_w = dev[2], dev[3], dev[4]
            # SCAFFOLD: the payload is [model delta | control delta] (fedsim/algorithms/scaffold.py:63-79)
            Dp = 2 * runner.D if scaffold else runner.D
            # one flat buffer [payload | sums tail]: the only thing the ranks all-reduce
            red = torch.empty(Dp + TAIL, dtype=torch.float32, device=self.device)
            agg_flat = red[:Dp]
            if scaffold:  # every rank owns a store, also with an empty shard (its queue may be empty)
                server, store = (self._controls(state, runner.D) if own
                                 else self._host_controls(state, queue, runner.D))
            if C:
                delta = self.ws.tensor("delta", (C, runner.ld), torch.float32)
                control = None
                if scaffold:
                    d_rows = torch.from_numpy(store.rows_of(queue)).to(self.device, non_blocking=True)
                    control = self.ws.tensor("scaffold_correction", (C, runner.ld), torch.float32)
                    native.call("fb_scaffold_correction_f32", native.ptr(server), native.ptr(store.matrix()),
                                store.ld, native.ptr(d_rows), C, runner.D, native.ptr(control), runner.ld, stream)
                fc1_sq = runner.local_sgd(theta.flat, pop, d_row_start, d_num_rows, d_perms, d_perm_off, C,
                                          plan.train, plan.prox_mu, delta, nonfinite, stream, num_rows,
                                          control=control, defer_fc1=self._factored_aggregate and not scaffold,
                                          eval_out=(loss, correct) if share0 else None)
                deferred = getattr(runner, "fc1_pending", None) is not None
                payload, ldp = delta, runner.ld
                if scaffold:
                    ldp = (Dp + 3) & ~3
                    payload = self.ws.tensor("scaffold_payload", (C, ldp), torch.float32)
                    new_control = torch.empty((C, runner.ld), dtype=torch.float32, device=self.device)
                    d_scale = torch.from_numpy(ctrl_scale).to(self.device, non_blocking=True)
                    native.call("fb_scaffold_payload_f32", native.ptr(delta), runner.ld, native.ptr(server),
                                native.ptr(store.matrix()), store.ld, native.ptr(d_rows), native.ptr(d_scale), C,
                                runner.D, native.ptr(payload), ldp, native.ptr(new_control), runner.ld, stream)
                    updates = ControlUpdates(queue, new_control)
                coef = self.ws.tensor("coef", (Cp,), torch.float32)
                bound = self._clip_bound()
                wsb = native.call("fb_clip_workspace_bytes", C, Dp) + 16 * C  # (+ the two-range K2 variant)
                kws = self.ws.get("clip_ws", wsb)
                nf2 = self.ws.tensor("nonfinite2", (Cp,), torch.int32)
                if fc1_sq is not None and not scaffold:  # fc1 block's squares came with its materialisation
                    native.call("fb_delta_norm_clip_ex_f32", native.ptr(payload), ldp, C, Dp, cnn.FC1_LO,
                                cnn.FC1_HI, native.ptr(fc1_sq), native.ptr(d_w), float(bound), native.ptr(norm),
                                native.ptr(coef), native.ptr(clipped), native.ptr(nf2), native.ptr(kws), kws.numel(),
                                stream)
                elif fused_clip_aggregate(Dp, ldp, deferred):  # K2 + K3 in one HBM pass
                    fws = self.ws.get("fused_ws", native.call("fb_clip_aggregate_workspace_bytes", C, Dp))
                    native.call("fb_clip_aggregate_f32", native.ptr(payload), ldp, C, Dp, native.ptr(d_w),
                                float(bound), native.ptr(norm), native.ptr(coef), native.ptr(clipped),
                                native.ptr(nf2), native.ptr(agg_flat), 0, native.ptr(fws), fws.numel(), stream)
                else:
                    native.call("fb_delta_norm_clip_f32", native.ptr(payload), ldp, C, Dp, native.ptr(d_w),
                                float(bound), native.ptr(norm), native.ptr(coef), native.ptr(clipped),
                                native.ptr(nf2), native.ptr(kws), kws.numel(), stream)
                torch.bitwise_or(nonfinite[:C], nf2[:C], out=nonfinite[:C])
                wsb = native.call("fb_weighted_sum_workspace_bytes", C, Dp)
                if deferred:  # (a narrow column range may use more client slices)
                    wsb = max(wsb, native.call("fb_weighted_sum_workspace_bytes", C, cnn.FC1_LO),
                              native.call("fb_weighted_sum_workspace_bytes", C, Dp - cnn.FC1_HI))
                sws = self.ws.get("sum_ws", wsb)
                if deferred:  # K3 around the CNN's fc1 block, which comes from the low-rank history
                    lo, hi = cnn.FC1_LO, cnn.FC1_HI
                    native.call("fb_weighted_sum_f32", native.ptr(payload), ldp, C, lo, native.ptr(coef),
                                native.ptr(agg_flat), 0, native.ptr(sws), sws.numel(), stream)
                    native.call("fb_weighted_sum_f32", native.ptr(payload) + 4 * hi, ldp, C, Dp - hi,
                                native.ptr(coef), native.ptr(agg_flat) + 4 * hi, 0, native.ptr(sws), sws.numel(),
                                stream)
                    cnn.fc1_aggregate(runner, coef, agg_flat[lo:hi], stream)
                elif not fused_clip_aggregate(Dp, ldp, deferred):
                    native.call("fb_weighted_sum_f32", native.ptr(payload), ldp, C, Dp, native.ptr(coef),
                                native.ptr(agg_flat), 0, native.ptr(sws), sws.numel(), stream)
            else:
                agg_flat.zero_()
            if scaffold and self.world_size > 1:  # every rank's store takes the whole cohort's controls
                updates = self._gather_controls(hp["queues"], updates, runner.ld)
        else:
            red = torch.empty(TAIL, dtype=torch.float32, device=self.device)
        native.call("fb_context_sums", native.ptr(loss), native.ptr(correct), native.ptr(d_num_rows),
                    native.ptr(norm), native.ptr(clipped), native.ptr(nonfinite), native.ptr(d_w), C, int(train),
                    native.ptr(red) + 4 * (red.numel() - TAIL), stream)
        if self.world_size > 1:
            reduce_across_ranks(red, self.group)

        # the host half of the next iteration (sampling, LPT shard, permutations) runs here,
        # while the GPU works through this context, instead of between iterations
        if train:
            self._plan_ahead(algorithm, state, ctx.iteration + 1)
        # one small D2H copy: the reduced sums (waits for this context's kernels and the reduce)
        sums = unpack_sums(red[-TAIL:].to("cpu").numpy())
        self.io_bytes["d2h"] += 4 * TAIL
        if self.record_clients or (train and sums[9] > 0):
            host_res = res[: 16 * Cp + 12 * Cp].to("cpu")
            self.io_bytes["d2h"] += int(host_res.numel())
            h_ints = host_res[16 * Cp:].view(torch.int32).numpy()
            h_bad = h_ints[2 * Cp:2 * Cp + C]
            if self.record_clients:
                self.last_client_results[pop_key.value] = dict(
                    queue=tuple(queue), loss=host_res[: 8 * Cp].view(torch.float64).numpy()[:C].copy(),
                    norm=host_res[8 * Cp: 16 * Cp].view(torch.float64).numpy()[:C].copy(),
                    correct=h_ints[:C].copy(), clipped=h_ints[Cp:Cp + C].copy())
            if train and sums[9] > 0:  # raised on EVERY rank (the count came through the all-reduce)
                bad = np.flatnonzero(h_bad)
                r, pos = first_bad_user(int(bad[0]) if len(bad) else -1, self.rank, self.world_size, self.group)
                uid = hp.get("queues", (queue,))[r][pos]
                raise EngineError(
                    f"iteration {ctx.iteration}, population {pop_key.value!r}, user {uid!r}: "
                    "entry contains non-finite values"
                )
        metrics: dict[str, MetricValue] = {}
        if sums[4] > 0:
            metrics = {
                "loss": MetricValue(MetricKind.CENTRAL, float(sums[0]), float(sums[2])),
                "accuracy": MetricValue(MetricKind.CENTRAL, float(sums[1]), float(sums[2])),
                "per_user_accuracy": MetricValue(MetricKind.PER_USER, float(sums[3]), float(sums[4])),
            }
        if not train:
            return None, metrics, cohort, None

        book = {}
        if self._clip is not None:
            book = {CLIPPED_KEY: np.array([sums[5]]), COUNT_KEY: np.array([sums[6]]),
                    NORM_KEY: np.array([sums[7]])}
        dims = dict(plan.model.param_dims)
        if scaffold:
            dims = {**{MODEL_PREFIX + n: k for n, k in dims.items()}, **{CONTROL_PREFIX + n: k for n, k in dims.items()}}
        aggregate = DeviceStatistics(flat=agg_flat, dims=dims, weight=float(sums[8]),
                                     bookkeeping=book, workspace=self.ws, comm=self._comm)
        for proc in reversed(self._postprocessors):
            try:
                if not interop.is_own(proc) and isinstance(aggregate, DeviceStatistics):
                    aggregate = aggregate.to_host()  # the reference's own server half runs on host Statistics
                aggregate, server_metrics = proc.postprocess_server(aggregate, ctx)
            except Exception as exc:
                raise EngineError(
                    f"iteration {ctx.iteration}, population {pop_key.value!r}: server postprocessor "
                    f"{type(proc).__name__} failed: {exc}"
                ) from exc
            metrics = merge_metrics(metrics, server_metrics)
        if not own:  # the reference's central step consumes host Statistics and host user_updates
            if isinstance(aggregate, DeviceStatistics):
                aggregate = aggregate.to_host()
            updates = self._host_updates(updates, state) if scaffold else updates
        elif not isinstance(aggregate, DeviceStatistics):
            aggregate = DeviceStatistics.from_host(aggregate, self.device, workspace=self.ws, comm=self._comm)
        return aggregate, metrics, cohort, updates
