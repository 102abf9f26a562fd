"""Host glue for the CNN entry points (fb_eval_cnn_f32 / fb_local_sgd_cnn_f32).

Chooses the slot count per layer launch (every client's step-s minibatch in
one wave when it fits the memory budget) and sizes the workspace.
"""

from __future__ import annotations

import numpy as np

from . import native

# samples per layer launch; ~0.35 MB of activations per slot -> <= ~6 GB
MAX_SLOTS = 16384
EVAL_GROUP = 16


# factored fc1 (fb_local_sgd_cnn_f32 hist_steps): history rows per client
FC1_RANK_MAX = 64
FACTORED_FC1 = True


def hist_steps(max_steps: int, B: int) -> int:
    """History depth for the factored fc1 update, 0 = dense (too many steps)."""
    return max_steps if FACTORED_FC1 and 0 < max_steps * B <= FC1_RANK_MAX else 0


def _slots(C: int, B: int) -> int:
    per_wave = max(1, min(C, MAX_SLOTS // B))
    return per_wave * B


def _eval_slots(total_rows: int) -> int:
    n = min(MAX_SLOTS, max(EVAL_GROUP, int(total_rows)))
    return (n + EVAL_GROUP - 1) // EVAL_GROUP * EVAL_GROUP


def eval_cohort(runner, theta, pop, row_start, num_rows, C, loss, correct, stream, h_num_rows, skip_first=None):
    """``skip_first=(perms, perm_off, B)``: evaluate only epoch 0's rows past each client's
    first batch of B -- the local-SGD call that follows evaluates that batch at theta_t in its
    first step (its forward IS the evaluation) and adds it to ``loss`` / ``correct``."""
    n = np.asarray(h_num_rows, dtype=np.int64)
    if skip_first is not None:
        perms, perm_off, B = skip_first
        total = int((n - np.minimum(n, B)).sum())
    else:
        perms, perm_off, B = None, None, 0
        total = int(n.sum())
    slots = _eval_slots(max(total, 1))
    nbytes = native.call("fb_cnn_workspace_bytes", slots, C, 0)
    ws = runner.ws.get("cnn_ws", nbytes)
    native.call("fb_eval_cnn_f32", native.ptr(theta), native.ptr(pop.X), native.ptr(pop.y), native.ptr(row_start),
                native.ptr(num_rows), C, total, native.ptr(loss), native.ptr(correct), slots, native.ptr(ws),
                ws.numel(), native.ptr(perms), native.ptr(perm_off), int(B), stream)


# (row range of the fc1 weight block in the flat parameter vector: models.CNN.param_dims order)
FC1_LO, FC1_HI = 19392, 19392 + 12544 * 128


def local_sgd_cohort(runner, theta, pop, row_start, num_rows, perms, perm_off, C, tp, prox_mu, delta, nonfinite,
                     stream, h_num_rows, control=None, defer_fc1=False, eval_out=None):
    """Returns the per-client fc1-block sum of squares (fp64 device [C]) when the
    factored tcgen05 path produced it, else None (K2 then scans the whole row).
    ``control`` ([C, ld] device, c - c_i per client; SCAFFOLD) selects the dense
    fc1 form: a per-client dense control term has no low-rank history.
    ``defer_fc1``: when the factored form runs in one wave, leave the clients'
    fc1 blocks unmaterialised and record the call in ``runner.fc1_pending`` for
    :func:`fc1_aggregate` (the engine's K3 for that block)."""
    B = tp.batch_size
    n = np.asarray(h_num_rows, dtype=np.int64)
    steps = np.ascontiguousarray(tp.num_epochs * ((n + B - 1) // B), dtype=np.int32)  # host, per client
    max_steps = int(steps.max()) if len(n) else 0
    slots = _slots(C, B)
    hist = hist_steps(max_steps, B) if control is None else 0
    nbytes = native.call("fb_cnn_workspace_bytes", slots, slots // B, hist)
    ws = runner.ws.get("cnn_ws", nbytes)
    sq = None
    if hist > 0 and max_steps > 0:
        import torch

        sq = runner.ws.tensor("cnn_fc1_sumsq", (max(C, 1),), torch.float64)
    defer = bool(defer_fc1 and sq is not None and 0 < C <= slots // B)
    runner.fc1_pending = (dict(C=C, B=B, max_steps=max_steps, lr=float(tp.learning_rate), mu=float(prox_mu),
                               slots=slots, hist=hist, ws=ws) if defer else None)
    native.call("fb_local_sgd_cnn_f32", native.ptr(theta), native.ptr(pop.X), native.ptr(pop.y),
                native.ptr(row_start), native.ptr(num_rows), native.ptr(perms), native.ptr(perm_off), C,
                tp.num_epochs, B, max_steps, float(tp.learning_rate), float(prox_mu), native.ptr(delta),
                runner.ld, native.ptr(nonfinite), slots, hist, native.ptr(ws), ws.numel(),
                native.ptr(sq) if sq is not None else None,
                native.ptr(control) if control is not None else None,
                control.stride(0) if control is not None else 0, steps.ctypes.data, 0 if defer else 1,
                native.ptr(eval_out[0]) if eval_out is not None else None,
                native.ptr(eval_out[1]) if eval_out is not None else None, stream)
    return sq


def fc1_aggregate(runner, coef, agg_fc1, stream) -> None:
    """agg_fc1[k, h] = sum_c coef[c] * delta_c[k, h] over the fc1 weight block of the
    deferred local-SGD call (runner.fc1_pending), from its low-rank history."""
    p = runner.fc1_pending
    runner.fc1_pending = None
    native.call("fb_cnn_fc1_aggregate_f32", native.ptr(coef), p["C"], p["B"], p["max_steps"], p["lr"], p["mu"],
                p["slots"], p["hist"], native.ptr(p["ws"]), p["ws"].numel(), native.ptr(agg_fc1), stream)
