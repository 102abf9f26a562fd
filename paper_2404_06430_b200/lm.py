"""Host glue for the config C language model (fb_eval_lm_f32 / fb_local_sgd_lm_f32,
csrc/lm.cu): the model's dims vector, the wave size (clients trained side by
side, bounded by an activation-memory budget) and the workspace."""

from __future__ import annotations

import numpy as np

from . import native

# activations + per-client weight / gradient rows of one wave stay under this
WAVE_BYTES = 24 << 30
EVAL_GROUPS = 256  # sentence groups of B per evaluation chunk


def dims_of(model) -> np.ndarray:
    return np.array([model.vocab, model.d_model, model.heads, model.ff, model.layers, model.seq], dtype=np.int32)


def wave_size(model, B: int, C: int) -> int:
    dims = dims_of(model)
    one = native.call("fb_lm_workspace_bytes", dims.ctypes.data, B, 1, 1)
    two = native.call("fb_lm_workspace_bytes", dims.ctypes.data, B, 2, 1)
    per = max(two - one, 1)
    return int(max(1, min(C, (WAVE_BYTES - one) // per + 1)))


def eval_cohort(runner, theta, pop, row_start, num_rows, C, loss, correct, stream, h_num_rows, skip_first=None):
    """``skip_first=(perms, perm_off, B)``: as cnn.eval_cohort -- only epoch 0's sentences past
    each client's first batch are evaluated here; local_sgd_cohort(eval_out=...) adds that batch."""
    perms, perm_off, skip = skip_first if skip_first is not None else (None, None, 0)
    model = runner.model
    dims = dims_of(model)
    B = 16
    nbytes = native.call("fb_lm_workspace_bytes", dims.ctypes.data, B, 1, EVAL_GROUPS)
    ws = runner.ws.get("lm_ws", nbytes)
    h = np.ascontiguousarray(h_num_rows, dtype=np.int32)
    native.call("fb_eval_lm_f32", native.ptr(theta), dims.ctypes.data, native.ptr(pop.X), native.ptr(row_start),
                native.ptr(num_rows), h.ctypes.data, C, native.ptr(loss), native.ptr(correct), B, EVAL_GROUPS,
                native.ptr(ws), ws.numel(), native.ptr(perms), native.ptr(perm_off), int(skip), stream)


def local_sgd_cohort(runner, theta, pop, row_start, num_rows, perms, perm_off, C, tp, prox_mu, delta, nonfinite,
                     stream, h_num_rows, control=None, eval_out=None):
    model = runner.model
    dims = dims_of(model)
    B = int(tp.batch_size)
    W = wave_size(model, B, max(C, 1))
    nbytes = native.call("fb_lm_workspace_bytes", dims.ctypes.data, B, W, EVAL_GROUPS)
    ws = runner.ws.get("lm_ws", nbytes)
    h = np.ascontiguousarray(h_num_rows, dtype=np.int32)
    native.call("fb_local_sgd_lm_f32", native.ptr(theta), dims.ctypes.data, native.ptr(pop.X), native.ptr(row_start),
                native.ptr(num_rows), h.ctypes.data, native.ptr(perms), native.ptr(perm_off), C, tp.num_epochs, B,
                float(tp.learning_rate), float(prox_mu), native.ptr(control) if control is not None else None,
                control.stride(0) if control is not None else 0, native.ptr(delta), runner.ld, native.ptr(nonfinite),
                W, native.ptr(ws), ws.numel(), native.ptr(eval_out[0]) if eval_out is not None else None,
                native.ptr(eval_out[1]) if eval_out is not None else None, stream)
    return None
