"""Host glue for the config D ResNet-18 (fb_eval_resnet_f32 / fb_local_sgd_resnet_f32,
csrc/resnet.cu): the model's dims vector, the wave size (clients trained side by
side, bounded by an activation-memory budget) and the workspace.  Evaluation runs
in chunks of one wave's worth of images through the same workspace."""

from __future__ import annotations

import numpy as np

from . import native

# activations + per-client weight / gradient rows of one wave stay under this
WAVE_BYTES = 40 << 30
MAX_WAVE = 64


def dims_of(model) -> np.ndarray:
    return np.array([model.num_classes, model.width, model.groups, model.image], dtype=np.int32)


def wave_size(model, B: int, C: int) -> int:
    dims = dims_of(model)
    one = native.call("fb_resnet_workspace_bytes", dims.ctypes.data, B, 1)
    two = native.call("fb_resnet_workspace_bytes", dims.ctypes.data, B, 2)
    per = max(two - one, 1)
    return int(max(1, min(C, MAX_WAVE, (WAVE_BYTES - one) // per + 1)))


def _workspace(runner, B: int, W: int):
    dims = dims_of(runner.model)
    return runner.ws.get("resnet_ws", native.call("fb_resnet_workspace_bytes", dims.ctypes.data, B, W))


def _batch(runner) -> int:
    return getattr(runner, "resnet_batch", 16)


def eval_cohort(runner, theta, pop, row_start, num_rows, C, loss, correct, stream, h_num_rows, skip_first=None):
    """``skip_first=(perms, perm_off, B)``: as cnn.eval_cohort -- only epoch 0's images past
    each client's first batch are evaluated here; local_sgd_cohort(eval_out=...) adds that batch."""
    perms, perm_off, skip = skip_first if skip_first is not None else (None, None, 0)
    model = runner.model
    dims = dims_of(model)
    B = _batch(runner)
    W = wave_size(model, B, 1 << 16)  # evaluation chunks of a full wave (the training workspace)
    ws = _workspace(runner, B, W)
    h = np.ascontiguousarray(h_num_rows, dtype=np.int32)
    native.call("fb_eval_resnet_f32", native.ptr(theta), dims.ctypes.data, native.ptr(pop.X), pop.dim,
                native.ptr(row_start), native.ptr(num_rows), h.ctypes.data, C, native.ptr(loss), native.ptr(correct),
                B, W, native.ptr(ws), ws.numel(), native.ptr(perms), native.ptr(perm_off), int(skip), stream)


def local_sgd_cohort(runner, theta, pop, row_start, num_rows, perms, perm_off, C, tp, prox_mu, delta, nonfinite,
                     stream, h_num_rows, control=None, eval_out=None):
    model = runner.model
    dims = dims_of(model)
    B = int(tp.batch_size)
    runner.resnet_batch = B
    W = wave_size(model, B, 1 << 16)
    ws = _workspace(runner, B, W)
    Wc = min(W, max(C, 1))
    h = np.ascontiguousarray(h_num_rows, dtype=np.int32)
    native.call("fb_local_sgd_resnet_f32", native.ptr(theta), dims.ctypes.data, native.ptr(pop.X), pop.dim,
                native.ptr(row_start), native.ptr(num_rows), h.ctypes.data, native.ptr(perms), native.ptr(perm_off), C,
                tp.num_epochs, B, float(tp.learning_rate), float(prox_mu),
                native.ptr(control) if control is not None else None,
                control.stride(0) if control is not None else 0, native.ptr(delta), runner.ld, native.ptr(nonfinite),
                Wc, native.ptr(ws), ws.numel(), native.ptr(eval_out[0]) if eval_out is not None else None,
                native.ptr(eval_out[1]) if eval_out is not None else None, stream)
    return None
