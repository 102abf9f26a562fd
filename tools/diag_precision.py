"""Per-block precision of the CNN local-SGD deltas at the bench shape.

Runs fb_local_sgd_cnn_f32 for the whole 1000-user bench cohort (so the timed
per-CTA kernel variants run) under several kernel settings, and compares the
first K clients' deltas with the float64 oracle -- next to the error of the
same oracle evaluated in float32 numpy (the fp32 floor: ReLU / max-pool
decision flips and fp32 rounding).  Diagnostic tool, not a test.

    python tools/diag_precision.py [K]
"""

from __future__ import annotations

import multiprocessing as mp
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
import paper_2404_06430_b200 as fb  # noqa: E402
from oracle import port  # noqa: E402

WL = bench.WORKLOADS["cnn"]
JOB: dict = {}


def _oracle(uid):
    from threadpoolctl import threadpool_limits

    threadpool_limits(1)
    m, th, users = JOB["m"], JOB["th"], JOB["users"]
    X, y = users[uid]
    perms = port.user_perms(JOB["seed"], uid, X.shape[0], 1)
    a64 = port.fit_local(m, th, X.astype(np.float64), y, perms, WL["lr"], WL["batch"])
    th32 = {k: v.astype(np.float32) for k, v in th.items()}
    a32 = port.fit_local(m, th32, X.astype(np.float32), y, perms, np.float32(WL["lr"]), WL["batch"])
    d64 = port.flat(th, m.dims) - port.flat(a64, m.dims)
    d32 = (port.flat(th32, m.dims).astype(np.float32) - port.flat(a32, m.dims).astype(np.float32)).astype(np.float64)
    return d64, d32


def blocks(m):
    off, out = 0, []
    for n, k in m.dims.items():
        out.append((n, off, off + k))
        off += k
    return out


def report(tag, got, ref, m):
    rel = np.linalg.norm(got - ref, axis=1) / np.linalg.norm(ref, axis=1)
    line = f"{tag:28s} all: med {np.median(rel):.2e} p90 {np.quantile(rel, .9):.2e} max {rel.max():.2e} |"
    for n, a, b in blocks(m):
        r = np.linalg.norm(got[:, a:b] - ref[:, a:b], axis=1) / np.maximum(np.linalg.norm(ref[:, a:b], axis=1), 1e-300)
        line += f" {n} {np.median(r):.1e}"
    print(line, flush=True)


def main():
    import torch

    from paper_2404_06430_b200 import cnn, native

    K = int(sys.argv[1]) if len(sys.argv) > 1 else 48
    ds = bench.build(WL)
    train = ds[fb.Population.TRAIN]
    uids = list(train.users)
    users = {u: (np.asarray(train.users[u].features), train.users[u].labels) for u in uids}
    om = port.Cnn()
    th = om.init(0)
    seed = 12345
    JOB.update(m=om, th=th, users=users, seed=seed)
    with mp.get_context("fork").Pool(16) as pool:
        res = pool.map(_oracle, uids[:K])
    ref = np.array([r[0] for r in res])
    f32 = np.array([r[1] for r in res])
    report("numpy float32 oracle", f32, ref, om)

    dev = torch.device("cuda")
    theta = torch.from_numpy(port.flat(th, om.dims).astype(np.float32)).to(dev)
    pop = fb.DevicePopulation(train, dev)
    C = len(uids)
    num_rows = pop.num_rows
    perms = np.concatenate([port.user_perms(seed, u, int(n), 1)[0] for u, n in zip(uids, num_rows)]).astype(np.int32)
    perm_off = np.concatenate([[0], np.cumsum(num_rows.astype(np.int64))[:-1]]).astype(np.int64)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    args = (d(pop.row_start), d(num_rows), d(perms), d(perm_off))
    tp = fb.LocalTrainParams(WL["lr"], 1, WL["batch"])
    for impl, fact in ((1, True), (1, False), (0, False)):
        native.call("fb_cnn_set_conv_impl", impl)
        cnn.FACTORED_FC1 = fact
        runner = fb.engine._ModelRunner(fb.CNN(), fb.device.Workspace(dev))
        delta = torch.zeros(C, runner.ld, device=dev)
        bad = torch.zeros(C, dtype=torch.int32, device=dev)
        runner.local_sgd(theta, pop, *args, C, tp, 0.0, delta, bad, 0, num_rows)
        got = delta[:K, :runner.D].double().cpu().numpy()
        report(f"gpu conv_impl={impl} fc1={'factored' if fact else 'dense'}", got, ref, om)
        del delta
        torch.cuda.empty_cache()
    native.call("fb_cnn_set_conv_impl", 1)


if __name__ == "__main__":
    main()
