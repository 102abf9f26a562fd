"""N > 1 path on CPU: world_size-2 process group over gloo (127.0.0.1).

Each rank plans its shard exactly as GpuSimulationEngine does (same cohort,
LPT queue over world_size workers), produces its queue's clipped weighted
deltas and metric sums (the oracle stands in for the device kernels here --
test-only), packs them as the engine does (fp32 payload, then the sums as
fp32 hi/lo pairs, the layout fb_context_sums writes) and reduces the ONE
buffer with the engine's own reduce_across_ranks.  The reduced result must
equal the single-process run of the whole cohort, and the shard map must be
the reference's 2-worker assignment (golden fixture)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

WORLD = 2


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank: int, port: int, name: str):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        import paper_2404_06430_b200 as fb
        from oracle import port as oport
        from paper_2404_06430_b200.engine import SUM_FIELDS, TAIL, pack_sums, plan_shard, reduce_across_ranks, unpack_sums
        from tests.conftest import load_golden
        from tests.helpers import CONFIGS, oracle_model, product_datasets, users_of

        cfg = CONFIGS[name]
        ds = product_datasets(cfg)
        alg, _ = __import__("tests.helpers", fromlist=["product_run_parts"]).product_run_parts(cfg)
        state = alg.initial_state()
        ctx = alg.get_next_central_contexts(state, 0)[0]
        cohort, queue = plan_shard(ds[fb.Population.TRAIN], ctx, rank, WORLD)

        # the shard map: union is the cohort, disjoint, == the reference's 2-worker queues
        queues = [None] * WORLD
        dist.all_gather_object(queues, list(queue))
        assert sorted(sum(queues, [])) == sorted(cohort)
        assert len(set(queues[0]) & set(queues[1])) == 0
        g = load_golden(name)
        if cfg["workers"] == WORLD:
            assert ["|".join(q) for q in queues] == [str(q) for q in g["queues0"]]

        m = oracle_model(cfg)
        users = users_of(ds[fb.Population.TRAIN])
        theta = m.init(cfg["init_seed"])
        train = (cfg["lr"], cfg["epochs"], cfg["batch"])
        part = oport.run_context(m, theta, users, cfg["cohort"], ctx.seed, train=train, weighting=cfg["weighting"],
                                 bound=cfg["bound"], sigma=0.0, world=WORLD, rank=rank)
        assert list(part.queue) == list(queue)
        n = part.n.astype(np.float64)
        local = np.array([part.loss_sum.sum(), float(part.correct.sum()), n.sum(), (part.correct / n).sum(),
                          float(len(queue)), float(part.clipped.sum()), float(len(queue)), float(part.norm.sum()),
                          part.weight, 0.0])
        buf = torch.from_numpy(np.concatenate([part.aggregate.astype(np.float32), pack_sums(local)]))
        reduce_across_ranks(buf)
        agg, sums = buf[:-TAIL].double(), unpack_sums(buf[-TAIL:].numpy())

        whole = oport.run_context(m, theta, users, cfg["cohort"], ctx.seed, train=train, weighting=cfg["weighting"],
                                  bound=cfg["bound"], sigma=0.0)
        nw = whole.n.astype(np.float64)
        want = np.array([whole.loss_sum.sum(), float(whole.correct.sum()), nw.sum(), (whole.correct / nw).sum(),
                         float(len(cohort)), float(whole.clipped.sum()), float(len(cohort)), float(whole.norm.sum()),
                         whole.weight, 0.0])
        assert len(SUM_FIELDS) == len(want)
        integral = [1, 2, 4, 5, 6, 8, 9]   # counts: exact through the fp32 hi word
        np.testing.assert_array_equal(sums[integral], want[integral])
        # real-valued sums (loss, per-user accuracy, norm): the fp32 (hi, lo) pair sums round once
        # per rank in the hi word, ~2^-24 relative (per-client values are fp32-computed anyway)
        np.testing.assert_allclose(sums, want, rtol=2e-7)
        np.testing.assert_allclose(agg.numpy(), whole.aggregate, rtol=2e-6, atol=1e-7 * np.abs(whole.aggregate).max())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["logistic_dp", "mlp_dp"])
def test_two_rank_shard_and_reduce_matches_single_process(name):
    mp.spawn(_rank_main, args=(_free_port(), name), nprocs=WORLD, join=True)
