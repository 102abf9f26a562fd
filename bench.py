#!/usr/bin/env python
"""Central-iteration throughput of the B200 engine (BASELINE.json metric:
central iterations/sec and clients/sec at cohort N) and the CPU reference arm.

Default workload (BASELINE configs[1], single-GPU form): FedAvg + central
Gaussian DP (L2 clip 1.0), the CIFAR-10 CNN, cohort 1000 of 1000 users x 50
synthetic CIFAR-shaped points (3x32x32), 1 local epoch, batch 10, local lr
0.1, central SGD lr 1.0, uniform weighting, sigma 0.8025 (the reference's
calibration for eps=2, delta=1e-6, q=0.001, T=1500), r = C / C~ = 1,
validation context (100 users) every 10 iterations.

A step = one central iteration (host sampling + LPT shard + permutations,
eval + local SGD + clip + aggregate on the GPU, all-reduce for N>1, noise +
average + central SGD).  ``value`` has the dataset resident in HBM; ``e2e``
keeps it in pinned host memory and moves each iteration's cohort rows to the
device inside the timed region (plus the per-client results back).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "central iterations/sec and clients/sec at cohort N, 1/2/4/8 B200 vs host-CPU ref"
SIGMA_T1500 = 0.802516171110736  # reference calibrate_sigma(2.0, 1e-6, 0.001, 1500)

WORKLOADS = {
    "cnn": dict(model="cnn", dim=3072, users=1000, val_users=100, ppu=50, cohort=1000, eval_cohort=100,
                epochs=1, batch=10, lr=0.1, clr=1.0, bound=1.0, sigma=SIGMA_T1500, noise_cohort=1000,
                eval_every=10, name="cifar10-cnn fedavg+gaussian-dp cohort1000 (BASELINE configs[1])"),
    "mlp": dict(model="mlp", dim=32, hidden=64, users=1000, val_users=100, ppu=50, cohort=1000, eval_cohort=100,
                epochs=1, batch=10, lr=0.1, clr=1.0, bound=1.0, sigma=SIGMA_T1500, noise_cohort=1000,
                eval_every=10, name="mlp(64) fedavg+gaussian-dp cohort1000 (reference-native shape)"),
    "logistic": dict(model="logistic", dim=32, users=1000, val_users=100, ppu=50, cohort=1000, eval_cohort=100,
                     epochs=1, batch=10, lr=0.1, clr=1.0, bound=1.0, sigma=SIGMA_T1500, noise_cohort=1000,
                     eval_every=10, name="logistic fedavg+gaussian-dp cohort1000 (reference-native shape)"),
    # ragged clients (the reference-native shapes): per-user sizes drawn like
    # fedsim/cli/bench.py:61-63 -- lognormal(mean 3, sigma 1), rounded, clipped to [1, 500]
    "mlp-ragged": dict(model="mlp", dim=32, hidden=64, users=1000, val_users=100, ppu=None, ragged=True, cohort=400,
                       eval_cohort=100, epochs=1, batch=10, lr=0.1, clr=1.0, bound=1.0, sigma=SIGMA_T1500,
                       noise_cohort=1000, eval_every=10,
                       name="mlp(64) fedavg+gaussian-dp cohort400, ragged users (StackOverflow-shaped sizes)"),
    "cnn-ragged": dict(model="cnn", dim=3072, users=1000, val_users=100, ppu=None, ragged=True, cohort=200,
                       eval_cohort=100, epochs=1, batch=10, lr=0.1, clr=1.0, bound=1.0, sigma=SIGMA_T1500,
                       noise_cohort=1000, eval_every=10,
                       name="cifar10-cnn fedavg+gaussian-dp cohort200, ragged users 1-500 (FLAIR-shaped sizes)"),
    # BASELINE configs[2] / SURVEY.md 8(f) row 3: StackOverflow-shaped next-word transformer
    # (/root/reference/PAPER.md:1052,1071-1085): cohort 400, 1 epoch, B=16, local lr 0.3,
    # central Adam (lr 0.1, betas 0.9/0.99, adaptivity 0.1), clip 1.0, noise cohort 5000,
    # evaluation every 20; <= 64 sentences of 20 tokens per user (synthetic, ragged)
    "lm": dict(model="lm", users=4000, val_users=200, ppu=None, sentences=True, cohort=400, eval_cohort=100,
               epochs=1, batch=16, lr=0.3, clr=0.1, adam=(0.9, 0.99, 0.1), bound=1.0, sigma=1.0, noise_cohort=5000,
               eval_every=20, name="stackoverflow-transformer-lm fedavg+gaussian-dp+adam cohort400 (BASELINE configs[2])"),
    # BASELINE configs[3] / SURVEY.md 8(f) row 3: FLAIR-shaped ResNet-18 (GroupNorm), 17-label
    # multi-label BCE: cohort 200, 2 epochs, B=16, local lr
    # 0.01, central Adam (lr 0.1, betas 0.9/0.99, adaptivity 0.1), clip 0.1, noise cohort 5000,
    # evaluation every 20; 1 - 500 224 x 224 images per user (synthetic, ragged)
    "resnet": dict(model="resnet", users=400, val_users=40, ppu=None, images=True, cohort=200, eval_cohort=40,
                   epochs=2, batch=16, lr=0.01, clr=0.1, adam=(0.9, 0.99, 0.1), bound=0.1, sigma=1.0,
                   noise_cohort=5000, eval_every=20,
                   name="flair-resnet18-gn multilabel fedavg+gaussian-dp+adam cohort200 (BASELINE configs[3])"),
}

# FP32 FFMA peak: 148 SMs x 128 lanes x 2 x 1.965 GHz
FP32_FFMA_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12

# algorithmic FLOPs per processed sample for the CNN kernels (2 x MACs of the
# dense operation the kernel implements)
CNN_MACS = {"conv1": 30 * 30 * 32 * 27, "conv2": 28 * 28 * 64 * 288, "fc1": 12544 * 128, "fc2": 128 * 10}


def _torch():
    import torch

    return torch


# ------------------------------------------------------------------ setup


def ragged_sizes(n_users: int, seed: int) -> np.ndarray:
    """fedsim/cli/bench.py:61-63: max(1, round(lognormal(3, 1))), capped at 500."""
    raw = np.random.default_rng(seed).lognormal(mean=3.0, sigma=1.0, size=n_users)
    return np.clip(np.maximum(1, np.round(raw)), 1, 500).astype(np.int64)


def build_ragged(wl: dict):
    import paper_2404_06430_b200 as fb
    from paper_2404_06430_b200.feddata import FederatedDataset, UserDataset

    sizes = {"train": ragged_sizes(wl["users"], 1), "val": ragged_sizes(wl["val_users"], 2)}
    total = int(sizes["train"].sum() + sizes["val"].sum())
    X, y = fb.make_synthetic_classification(total, dim=wl["dim"], num_classes=10, margin=6.0,
                                            seed=fb.derive_seed(0, "pool"))
    X = X.astype(np.float32)
    out, off = {}, 0
    for pop, key in ((fb.Population.TRAIN, "train"), (fb.Population.VAL, "val")):
        users = {}
        for i, n in enumerate(sizes[key]):
            uid = f"{key}{i:05d}"
            users[uid] = UserDataset(uid, X[off:off + n], y[off:off + n])
            off += int(n)
        out[pop] = FederatedDataset(users=users, population=pop)
    return out


def build(wl: dict):
    import paper_2404_06430_b200 as fb

    if wl.get("images"):
        return {fb.Population.TRAIN: fb.make_synthetic_images(wl["users"], seed=fb.derive_seed(0, "train", "resnet"),
                                                              id_prefix="train"),
                fb.Population.VAL: fb.make_synthetic_images(wl["val_users"], seed=fb.derive_seed(0, "val", "resnet"),
                                                            population=fb.Population.VAL, id_prefix="val")}
    if wl.get("sentences"):
        return {fb.Population.TRAIN: fb.make_synthetic_sentences(wl["users"], seed=fb.derive_seed(0, "train", "lm"),
                                                                 population=fb.Population.TRAIN, id_prefix="train"),
                fb.Population.VAL: fb.make_synthetic_sentences(wl["val_users"], seed=fb.derive_seed(0, "val", "lm"),
                                                               population=fb.Population.VAL, id_prefix="val")}
    if wl.get("ragged"):
        return build_ragged(wl)
    ppu = wl["ppu"]
    ntr, nva = wl["users"] * ppu, wl["val_users"] * ppu
    X, y = fb.make_synthetic_classification(ntr + nva, dim=wl["dim"], num_classes=10, margin=6.0,
                                            seed=fb.derive_seed(0, "pool"))
    X = X.astype(np.float32)  # features are cast to fp32 once and fed to both sides
    train = fb.partition_iid(X[:ntr], y[:ntr], ppu, seed=fb.derive_seed(0, "train", "split"),
                             population=fb.Population.TRAIN, id_prefix="train")
    val = fb.partition_iid(X[ntr:], y[ntr:], ppu, seed=fb.derive_seed(0, "val", "split"),
                           population=fb.Population.VAL, id_prefix="val")
    return {fb.Population.TRAIN: train, fb.Population.VAL: val}


def make_model(wl):
    import paper_2404_06430_b200 as fb

    if wl["model"] == "cnn":
        return fb.CNN()
    if wl["model"] == "lm":
        return fb.TransformerLM()
    if wl["model"] == "resnet":
        return fb.ResNet18()
    if wl["model"] == "mlp":
        return fb.MLP(wl["dim"], wl["hidden"], 10)
    return fb.LogisticRegression(wl["dim"], 10)


def make_algorithm(wl, iterations):
    import paper_2404_06430_b200 as fb

    opt = (fb.AdamOptimizer(wl["clr"], beta1=wl["adam"][0], beta2=wl["adam"][1], adaptivity_degree=wl["adam"][2])
           if wl.get("adam") else fb.SGDOptimizer(wl["clr"]))
    alg = fb.FedAvg(make_model(wl), opt, total_iterations=iterations,
                    cohort_size=wl["cohort"], local_learning_rate=wl["lr"], local_num_epochs=wl["epochs"],
                    local_batch_size=wl["batch"], eval_frequency=wl["eval_every"],
                    eval_cohort_size=wl["eval_cohort"], weighting="uniform", run_seed=0, init_seed=0)
    clip = fb.ClippingPostprocessor(wl["bound"])
    r = wl["cohort"] / wl["noise_cohort"]
    mech = fb.GaussianCentralMechanism(clip, sigma=wl["sigma"], r=r,
                                       noise_base_seed=fb.derive_seed(0, "noise-stream", 0))
    return alg, [clip, mech]


# ----------------------------------------------------------------- clocks


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = Path(tempfile.mkstemp(suffix=".csv")[1])

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=self.path.open("w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait(timeout=10)

    def summary(self) -> dict:
        rows = []
        for line in self.path.read_text().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) == 6 and f[0].isdigit():
                rows.append(f)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(float(r[0]) for r in rows), "sm_max_mhz": float(rows[0][1]),
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------- GPU arm


def run_iterations(engine, alg, state, t0, k):
    for t in range(t0, t0 + k):
        ctxs = alg.get_next_central_contexts(state, t)
        res = engine.run_iteration(alg, state, ctxs)
        state = alg.process_aggregated_statistics_all_contexts(state, ctxs, res.aggregates, res.metrics,
                                                               res.user_updates)
    return state


def timed(engine, alg, state, t0, k, dist, world):
    """K iterations bracketed by barrier + synchronize; CUDA-event device time,
    max over ranks."""
    torch = _torch()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    ev0.record(engine.stream)
    state = run_iterations(engine, alg, state, t0, k)
    ev1.record(engine.stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    wall = time.perf_counter() - w0
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device=engine.device, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return state, ms, wall


def kernel_work(wl: dict, counts: dict) -> dict:
    """Algorithmic work per kernel over the timed window (this rank):
    name -> (bound, amount, unit-note).  FLOPs count the dense operation the
    kernel implements once (2 x MACs); bytes count
    compulsory HBM traffic (per-client fc1 deltas read / written, activations)."""
    conv2 = 2 * CNN_MACS["conv2"]
    fc1_bytes = 12544 * 128 * 4
    fwd, train, steps = counts["fwd"], counts["train"], counts["client_steps"]
    return {
        "conv2_fwd_tc_kernel": ("tensor", conv2 * fwd, "3-term fp16 tcgen05"),
        "conv2_fwd_pool_kernel": ("tensor", conv2 * fwd, "FP32 FFMA"),
        "conv2_bwd_x_tc_kernel": ("tensor", conv2 * train, "3-term fp16 tcgen05"),
        "conv2_bwd_x_kernel": ("tensor", conv2 * train, "FP32 FFMA"),
        "conv2_bwd_w_tc_kernel": ("tensor", conv2 * train, "3-term fp16 tcgen05"),
        "conv2_bwd_w_kernel": ("tensor", conv2 * train, "FP32 FFMA"),
        "conv1_fwd_kernel": ("tensor", 2 * CNN_MACS["conv1"] * fwd, "FP32 FFMA"),
        "conv1_bwd_w_kernel": ("tensor", 2 * CNN_MACS["conv1"] * train, "FP32 FFMA"),
        "conv1_fwd_tc_kernel": ("tensor", 2 * CNN_MACS["conv1"] * fwd, "3xTF32 tcgen05 (hi/lo weights stacked along N)"),
        "conv1_bwd_w_tc_kernel": ("tensor", 2 * CNN_MACS["conv1"] * train, "3xTF32 tcgen05 (hi/lo in operand rows)"),
        "conv1_bwd_w_ffma_kernel": ("fp32", 2 * CNN_MACS["conv1"] * train, "FP32 FFMA (register-blocked 8 x 7 tiles)"),
        # implicit-GEMM conv1 forward: the tensor work is ~1% of the tcgen05 rate; the kernel is
        # bound by writing a1 (fp16 hi + lo NHWC, 115,200 B per slot) after reading the image
        "conv1_fwd_ig_kernel": ("hbm", fwd * (2 * 2 * 28800 + 4 * 3072), "bytes (a1 hi+lo written, image read)"),
        # factored fc1 (squares-only materialisation and the factored aggregate): each reads the
        # client's fp16 hi/lo pooled history once, 4 B per history row element (steps x batch rows)
        "fc1_mat_tc_kernel": ("hbm", counts["client_steps"] * wl["batch"] * 12544 * 4, "bytes"),
        "fc1_agg_tc_kernel": ("hbm", counts["client_steps"] * wl["batch"] * 12544 * 4, "bytes"),
        # per client-step: read the client's fc1 delta (fwd); read + write it (bwd)
        "fc1_fwd_kernel": ("hbm", steps * fc1_bytes + fwd * 12544 * 4, "bytes"),
        "fc1_bwd_kernel": ("hbm", steps * 2 * fc1_bytes + 2 * train * 12544 * 4, "bytes"),
        "row_sumsq_partial_kernel": ("hbm", counts["clients"] * counts["D_dense"] * 4, "bytes"),
        # K3 reads the columns around the factored fc1 block (that block comes from fc1_agg_tc)
        "weighted_sum_kernel": ("hbm", counts["clients"] * counts["D_dense"] * 4 + counts["D_dense"] * 4 * counts["iters"],
                                "bytes"),
        "zero_delta_kernel": ("hbm", counts["clients"] * counts["D_dense"] * 4, "bytes"),
    }


def lm_kernel_work(counts: dict) -> dict:
    """Config C: every grouped GEMM flavour does the same dense work per processed
    token row -- 2 x (3d^2 + d^2 + 2 d F) x layers + 2 V d FLOPs (3.91 MFLOP at the
    config C shape): forward Y = X W^T (NT), backward dX = dY W (NN), dW = dY^T X (TN).
    Rows = slot rows processed (B x seq per active client step, eval chunks of
    256 x 16 sentences), padding included."""
    import paper_2404_06430_b200 as fb

    m = fb.TransformerLM()
    per_row = 2 * ((3 * m.d_model**2 + m.d_model**2 + 2 * m.d_model * m.ff) * m.layers + m.vocab * m.d_model)
    note = "FP32 FFMA (SIMT tiled GEMM)"
    tc = "3xTF32 tcgen05 (grouped persistent GEMM)"
    return {"lm_gemm_nt_kernel": ("fp32", per_row * counts["fwd_rows"], note),
            "lm_gemm_nn_kernel": ("fp32", per_row * counts["train_rows"], note),
            "lm_gemm_tn_kernel": ("fp32", per_row * counts["train_rows"], note),
            "lm_gemm_tc_nt_kernel": ("tensor", per_row * counts["fwd_rows"], tc),
            "lm_gemm_tc_nn_kernel": ("tensor", per_row * counts["train_rows"], tc),
            "lm_gemm_tc_tn_kernel": ("tensor", per_row * counts["train_rows"], tc)}


def resnet_kernel_work(counts: dict) -> dict:
    """Config D: algorithmic conv + fc FLOPs per image (2 x MACs, models.ResNet18
    .forward_flops_per_image: 3.63 GFLOP at 224 x 224) -- forward Y = col W^T (NT) for
    every forward pass, dW = dY^T col (TN) and dcol = dY W (NN, no stem: its input needs
    no gradient) per trained image.  Images = real images only: the zero slots of tail
    batches are work the kernels do but the algorithm does not."""
    import paper_2404_06430_b200 as fb

    m = fb.ResNet18()
    f = m.forward_flops_per_image()
    h = (m.image + 6 - 7) // 2 + 1
    stem = 2 * 3 * m.width * 49 * h * h
    tc = "3xTF32 tcgen05 (grouped persistent GEMM over im2col)"
    note = "FP32 FFMA (SIMT tiled GEMM)"
    return {"rn_gemm_tc_nt_kernel": ("tensor", f * counts["fwd"], tc),
            "rn_gemm_tc_tn_kernel": ("tensor", f * counts["train"], tc),
            "rn_gemm_tc_nn_kernel": ("tensor", (f - stem) * counts["train"], tc),
            "rn_gemm_nt_kernel": ("fp32", 0, note), "rn_gemm_nn_kernel": ("fp32", 0, note),
            "rn_gemm_tn_kernel": ("fp32", 0, note)}


def _ncu_kernel(name: str) -> dict | None:
    try:
        return json.loads((ROOT / "profiles" / "ncu_traffic.json").read_text())["kernels"][name]
    except (OSError, KeyError, ValueError):
        return None


def _ncu_traffic(name: str):
    """DRAM bytes (read + write) of one launch of `name` from the committed
    ncu --set full capture (profiles/ncu_traffic.json), with the launch size."""
    k = _ncu_kernel(name)
    if k is None or "dram_bytes" not in k:
        return None
    if "slots" not in k:  # (grouped-GEMM entries: bytes summed over the captured launches)
        return {"dram_bytes_captured": k["dram_bytes"], "launches_captured": k.get("launches"),
                "source": "profiles/ncu_traffic.json"}
    return {"dram_bytes_per_launch": k["dram_bytes"], "slots_per_launch": k["slots"],
            "algorithmic_bytes_per_launch": k.get("algorithmic_bytes"), "source": "profiles/ncu_traffic.json"}


def _tensor_evidence(name: str, frac: float) -> dict:
    """ncu tensor-pipe utilisation and issued-MMA-op accounting of a tcgen05
    kernel (profiles/ncu_traffic.json): the issued fraction counts every
    product the hi/lo operand split and the M padding make the pipe execute."""
    k = _ncu_kernel(name) or {}
    out = {}
    if "tensor_pipe_pct" in k:
        out["tensor_pipe_active_pct"] = k["tensor_pipe_pct"]
    if "tensor_ops_pct_of_peak" in k:
        out["tensor_ops_pct_of_tf32_or_f16_peak"] = k["tensor_ops_pct_of_peak"]
    if "mma_ops_per_algorithmic" in k:
        out["issued_ops_per_algorithmic"] = k["mma_ops_per_algorithmic"]
        out["issued_frac"] = round(frac * k["mma_ops_per_algorithmic"], 4)
    return out


def roofline(report: dict, wl: dict, counts: dict, peaks: dict) -> tuple[dict, dict]:
    """Dominant kernel's achieved throughput vs the measured peak, plus the
    same figure for every kernel with a defined algorithmic work."""
    if not report:
        return {}, {}
    work = (kernel_work(wl, counts) if wl["model"] == "cnn" else
            lm_kernel_work(counts) if wl["model"] == "lm" else
            resnet_kernel_work(counts) if wl["model"] == "resnet" else {})
    total = sum(v[0] for v in report.values())
    per = {}
    for name, (ms, launches) in report.items():
        if name not in work:
            continue
        bound, amount, note = work[name]
        if bound == "fp32":
            ach = amount / (ms * 1e-3) / 1e12
            per[name] = {"bound": "tensor", "achieved": round(ach, 2), "unit": "TFLOP/s",
                         "frac": round(ach / FP32_FFMA_TFLOPS, 4), "ms": round(ms, 2), "share": round(ms / total, 4),
                         "math": note, "peak": round(FP32_FFMA_TFLOPS, 1)}
        elif bound == "tensor":
            ach = amount / (ms * 1e-3) / 1e12
            peak = peaks.get("bf16_tflops", 1590.0)
            per[name] = {"bound": "tensor", "achieved": round(ach, 2), "unit": "TFLOP/s", "frac": round(ach / peak, 4),
                         "ms": round(ms, 2), "share": round(ms / total, 4), "math": note,
                         **_tensor_evidence(name, ach / peak)}
        else:
            ach = amount / (ms * 1e-3) / 1e9
            peak = peaks.get("hbm_gbs", 6650.0)
            per[name] = {"bound": "hbm", "achieved": round(ach, 1), "unit": "GB/s", "frac": round(ach / peak, 4),
                         "ms": round(ms, 2), "share": round(ms / total, 4)}
    name, (ms, launches) = max(report.items(), key=lambda kv: kv[1][0])
    out = {"kernel": name, "share_of_gpu_time": ms / total if total else None}
    if name in per and "peak" in per[name]:  # FP32 SIMT kernels: against the FFMA peak
        k = per[name]
        out.update(bound="tensor", achieved=k["achieved"], peak=k["peak"], unit="TFLOP/s", frac=k["frac"],
                   traffic=None, peak_source="FP32 FFMA peak 148 SMs x 128 lanes x 2 x 1.965 GHz (SURVEY.md 8(d)); "
                   "the kernel is a SIMT FP32 tiled GEMM, not tcgen05",
                   algorithmic=f"{work[name][1]:.4g} FLOP over {launches} launches")
    elif name in per:
        k = per[name]
        peak = peaks.get("bf16_tflops", 1590.0) if k["bound"] == "tensor" else peaks.get("hbm_gbs", 6650.0)
        out.update(bound=k["bound"], achieved=k["achieved"], peak=peak, unit=k["unit"], frac=k["frac"],
                   traffic=_ncu_traffic(name),
                   **{key: k[key] for key in ("tensor_pipe_active_pct", "issued_ops_per_algorithmic", "issued_frac",
                                              "tensor_ops_pct_of_tf32_or_f16_peak") if key in k},
                   peak_source=(("MEASURED_PEAKS.json bf16_tflops (dense bf16 cuBLAS); the kernel's own math is "
                                 + k.get("math", "") + ": three kind::tf32 MMAs per algorithmic product at half the "
                                 "bf16 rate -> at most 1/6 of this peak") if "TF32" in k.get("math", "") and
                                wl["model"] in ("lm", "resnet") else
                                ("MEASURED_PEAKS.json bf16_tflops (dense bf16 cuBLAS); the kernel's own math is "
                                + k.get("math", "") + ": per algorithmic product one N=128 MMA (hi*[Whi;Wlo]) + one "
                                "N=64 MMA (lo*Whi) -> at most 1/3 of the fp16/bf16 dense rate, and the N=64 half is "
                                "bound by shared-memory operand reads (tools/microbench/README.md)"))
                   if k["bound"] == "tensor" else "MEASURED_PEAKS.json hbm_gbs",
                   algorithmic=f"{work[name][1]:.4g} {'FLOP' if k['bound'] == 'tensor' else 'bytes'} over {launches} launches")
    else:
        out.update(bound="hbm", achieved=None, peak=peaks.get("hbm_gbs", 6650.0), unit="GB/s", frac=None, traffic=None)
    return out, per


def gpu_arm(args, wl):
    torch = _torch()
    import paper_2404_06430_b200 as fb
    from paper_2404_06430_b200 import native
    if os.environ.get("FB_CNN_CONV_IMPL"):  # experiments only: kernel variants (fb_cnn_set_conv_impl)
        native.call("fb_cnn_set_conv_impl", int(os.environ["FB_CNN_CONV_IMPL"]))

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = torch.distributed
    local = local % max(torch.cuda.device_count(), 1)  # (ranks share a device only in the gloo test mode)
    torch.cuda.set_device(local)
    if world > 1:
        backend = os.environ.get("FB_DIST_BACKEND", "nccl")  # "gloo": N ranks on one GPU (flow test only)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}

    ds = build(wl)
    K, W = args.steps, args.warmup
    alg, post = make_algorithm(wl, W + K + args.profile_steps + max(args.e2e_warmup, wl["eval_every"]) +
                               args.e2e_steps + 1)
    engine = fb.GpuSimulationEngine(ds, postprocessors=post)
    state = alg.initial_state()
    state = run_iterations(engine, alg, state, 0, W)
    n0 = native.lib().fb_launch_count()
    native.lib().fb_timing_enable(0)  # the headline carries no per-launch instrumentation
    with ClockSampler(local) as clk:
        state, ms, wall = timed(engine, alg, state, W, K, dist, world)
    launches = native.lib().fb_launch_count() - n0
    clocks = clk.summary()
    # second pass, per-kernel device times (every launch bracketed by CUDA events on its
    # stream): the roofline's kernel durations, not the headline
    KP = max(1, min(K, args.profile_steps))
    native.lib().fb_timing_enable(1)
    state, ms_prof, _ = timed(engine, alg, state, W + K, KP, dist, world)
    report = native.timing_report()
    native.lib().fb_timing_enable(0)

    # samples processed by the forward / training kernels in the timed window (this rank)
    C = wl["cohort"]
    per_rank = C / world
    val_iters = sum(1 for t in range(W + K, W + K + KP) if t % wl["eval_every"] == 0)
    ppu = wl["ppu"] or float(np.mean([u.num_points for u in ds[fb.Population.TRAIN].users.values()]))
    steps = wl["epochs"] * -(-int(round(ppu)) // wl["batch"])  # (ragged: at the mean size; approximate)
    train_samples = per_rank * ppu * wl["epochs"] * KP
    fwd_samples = train_samples + per_rank * ppu * KP + val_iters * (wl["eval_cohort"] / world) * ppu
    D = make_model(wl).num_params
    # columns the dense per-client passes (zero_delta, K2) touch: the factored CNN fc1
    # block is written by fc1_mat_tc and its squares come out of that kernel
    from paper_2404_06430_b200 import cnn as cnn_mod
    dense_D = (D + 3) & ~3
    if wl["model"] == "cnn" and cnn_mod.hist_steps(max(int(steps), 1), wl["batch"]):
        dense_D -= cnn_mod.FC1_HI - cnn_mod.FC1_LO
    counts = {"train": train_samples, "fwd": fwd_samples, "client_steps": per_rank * steps * KP,
              "clients": per_rank * KP, "D": (D + 3) & ~3, "D_dense": dense_D, "iters": KP}
    if wl["model"] == "lm":  # slot rows the GEMMs process (B x seq per client step; eval chunks padded)
        from paper_2404_06430_b200 import lm as lm_mod
        seq, B = 20, wl["batch"]
        sizes = np.array([u.num_points for u in ds[fb.Population.TRAIN].users.values()], dtype=np.float64)
        mean_steps = float(np.mean(wl["epochs"] * np.ceil(sizes / B)))
        chunk = lm_mod.EVAL_GROUPS * B
        ev_rows = lambda nsent: np.ceil(nsent / chunk) * chunk * seq
        counts["train_rows"] = per_rank * mean_steps * B * seq * KP
        counts["fwd_rows"] = (counts["train_rows"] + ev_rows(per_rank * float(sizes.mean())) * KP
                              + val_iters * ev_rows((wl["eval_cohort"] / world) * float(sizes.mean())))
        steps = mean_steps
    if wl["model"] == "resnet":  # real images through the forward / training passes (tail slots excluded)
        sizes = np.array([u.num_points for u in ds[fb.Population.TRAIN].users.values()], dtype=np.float64)
        B = wl["batch"]
        mean_n = float(sizes.mean())
        shared = float(np.mean(np.minimum(sizes, B)))  # the first batch's eval rides on local step 0
        counts["train"] = per_rank * mean_n * wl["epochs"] * KP
        counts["fwd"] = (counts["train"] + per_rank * (mean_n - shared) * KP
                         + val_iters * (wl["eval_cohort"] / world) * mean_n)
        steps = float(np.mean(wl["epochs"] * np.ceil(sizes / B)))

    # end-to-end: dataset in pinned host memory, cohort rows moved every iteration
    e2e = None
    if args.e2e_steps > 0:
        eng2 = fb.GpuSimulationEngine(ds, postprocessors=post, data_residency="host")
        # warm-up covers a validation iteration too (every context kind has allocated its
        # prefetch buffers once before the timed window)
        e2e_warmup = max(args.e2e_warmup, wl["eval_every"])
        t0 = W + K + KP
        state = run_iterations(eng2, alg, state, t0, e2e_warmup)
        eng2.io_bytes = {"h2d": 0, "d2h": 0}
        state, ms2, wall2 = timed(eng2, alg, state, t0 + e2e_warmup, args.e2e_steps, dist, world)
        e2e = {"value": args.e2e_steps / (ms2 / 1e3), "unit": "iterations/s",
               "clients_per_sec": C * args.e2e_steps / (ms2 / 1e3),
               "h2d_bytes_per_step": int(eng2.io_bytes["h2d"] / args.e2e_steps),
               "d2h_bytes_per_step": int(eng2.io_bytes["d2h"] / args.e2e_steps),
               "data": "dataset in pinned host memory; cohort rows gathered to HBM each iteration"}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:  # (config D: ~0.5 s per image pass on the host -> one client)
        cpu = cpu_baseline(wl, ds, 1 if wl["model"] == "resnet" else args.cpu_clients)

    rf, per_kernel = roofline(report, wl, counts, peaks)
    if rank == 0:
        ips = K / (ms / 1e3)
        line = {
            "metric": METRIC, "value": ips, "unit": "iterations/s", "clients_per_sec": ips * C,
            "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": ms / K, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": wl["name"], "model": wl["model"], "cohort": C, "users": wl["users"],
                       "points_per_user": wl["ppu"] or (f"ragged lognormal(3,1) in [1,64] sentences of 20 tokens, "
                                                        f"mean {ppu:.1f}" if wl["model"] == "lm" else
                                                        f"ragged lognormal(3,1) in [1,500] 224x224 images, 17 "
                                                        f"labels, mean {ppu:.1f}" if wl["model"] == "resnet" else
                                                        f"ragged lognormal(3,1) in [1,500], mean {ppu:.1f}"),
                       "local_epochs": wl["epochs"], "batch": wl["batch"],
                       "local_steps_per_client": steps, "sigma": wl["sigma"], "clip_bound": wl["bound"],
                       "eval_every": wl["eval_every"], "parallelism": f"cohort-dp{world}",
                       "l2": "inputs larger than L2 (dataset 614 MB + per-iteration working set of GBs)"},
            "wall_s": wall, "clocks": clocks, "gpu_launches": int(launches), "e2e": e2e,
            "profile_pass": {"steps": KP, "ms_per_step": ms_prof / KP,
                             "note": "per-kernel times come from this second pass (fb_timing_enable(1)); the "
                                     "headline window above runs without instrumentation"},
            "roofline": rf,
            "kernels": per_kernel,
            "kernels_ms": {k: round(v[0], 3) for k, v in sorted(report.items(), key=lambda kv: -kv[1][0])},
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------------- CPU arms


def _cores() -> int:
    try:
        from threadpoolctl import threadpool_info

        n = max((i.get("num_threads", 1) for i in threadpool_info()), default=1)
        return int(n)
    except Exception:
        return len(os.sched_getaffinity(0))


def cpu_iteration_seconds(wl, ds, n_clients: int, t: int = 0) -> tuple[float, str]:
    """Time the oracle port (the reference algorithm, numpy float64) on a
    bounded sample of the train cohort and extrapolate one central
    iteration: C x per-client time + amortised validation eval."""
    import paper_2404_06430_b200 as fb
    from oracle import port

    model = {"cnn": lambda: port.Cnn(), "lm": lambda: port.TransformerLM(), "resnet": lambda: port.ResNet18(),
             "mlp": lambda: port.Mlp(wl["dim"], wl["hidden"], 10),
             "logistic": lambda: port.Linear(wl["dim"], 10)}[wl["model"]]()
    theta = model.init(0)
    train = ds[fb.Population.TRAIN]
    ctx = port.cohort_seed(0, t, "train")
    cohort = port.sample_cohort(train.user_ids, wl["cohort"], ctx)[:n_clients]
    users = {u: (train.users[u].features.astype(np.float64), train.users[u].labels) for u in cohort}
    t0 = time.perf_counter()
    port.run_context(model, theta, users, len(cohort), ctx, train=(wl["lr"], wl["epochs"], wl["batch"]),
                     weighting="uniform", bound=wl["bound"], sigma=wl["sigma"], r=1.0, noise=False)
    per_client = (time.perf_counter() - t0) / len(cohort)
    val = ds[fb.Population.VAL]
    vu = val.user_ids[:max(1, n_clients // 4)]
    t1 = time.perf_counter()
    for u in vu:
        model.eval_counts(theta, val.users[u].features, val.users[u].labels)
    per_val = (time.perf_counter() - t1) / len(vu)
    it = wl["cohort"] * per_client + wl["eval_cohort"] * per_val / wl["eval_every"]
    sample = (f"{len(cohort)} train clients (eval + {wl['epochs']} epoch local SGD + clip) and {len(vu)} val users "
              f"of iteration {t}, extrapolated to cohort {wl['cohort']} + validation every {wl['eval_every']}")
    return it, sample


def cpu_baseline(wl, ds, n_clients):
    it, sample = cpu_iteration_seconds(wl, ds, n_clients)
    return {"value": 1.0 / it, "unit": "iterations/s", "cores": _cores(), "kind": "port", "sample": sample,
            "seconds_per_iteration": it}


_REF: dict = {}  # fork-inherited by the reference arm's worker processes


def _ref_queue_worker(span):
    """One worker of the reference engine, in its own process: fedsim's own
    SimulationEngine._run_queue (simulate_one_user -> postprocess_one_user ->
    SumAggregator.accumulate over the queue; fedsim/engine/runtime.py:173-209)
    on a slice of the cohort, one BLAS thread."""
    from threadpoolctl import threadpool_limits

    lo, hi = span
    with threadpool_limits(1):
        return _REF["engine"]._run_queue(_REF["alg"], _REF["state"], _REF["dataset"], _REF["ctx"],
                                         _REF["queue"][lo:hi])


def _reference_setup(wl):
    """The reference's own objects (fedsim from baseline/_ref): datasets, the
    oracle CNN in fedsim's generic Model contract (fedsim has no CNN; its own
    fit_local loop drives it), a FedAvg factory (cohort size -> algorithm) and
    ClippingPostprocessor + GaussianCentralMechanism at the bench's settings."""
    REF = ROOT / "baseline" / "_ref"
    if wl.get("ppu") is None:  # ragged / sentence / image populations: the port's own data path
        raise ValueError(f"the reference arm's fedsim datasets cover fixed-size users only ({wl['model']})")
    if not (REF / "fedsim" / "__init__.py").exists():
        raise ImportError("fedsim not installed in baseline/_ref")
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "fedsim_numba_cache"))
    sys.path.append(str(REF))
    from fedsim.algorithms import FedAvg
    from fedsim.core import Population, derive_seed
    from fedsim.feddata import make_synthetic_classification, partition_iid
    from fedsim.models import MLP, LogisticRegression, Model, SGDOptimizer
    from fedsim.privacy import ClippingPostprocessor, GaussianCentralMechanism

    from oracle.port import Cnn

    class RefCNN(Model):
        def __init__(self):
            self.impl = Cnn()

        @property
        def param_dims(self):
            return self.impl.dims

        def init_params(self, seed):
            return self.impl.init(seed)

        def loss_and_grad(self, params, X, y):
            return self.impl.loss_and_grad(params, X, y)

        def eval_counts(self, params, X, y, backend=None):
            return self.impl.eval_counts(params, X, y)

    ppu = wl["ppu"]
    ntr, nva = wl["users"] * ppu, wl["val_users"] * ppu
    X, y = make_synthetic_classification(ntr + nva, dim=wl["dim"], num_classes=10, margin=6.0,
                                         seed=derive_seed(0, "pool"))
    X = X.astype(np.float32).astype(np.float64)  # the same fp32-representable features the GPU arm sees
    ds = {Population.TRAIN: partition_iid(X[:ntr], y[:ntr], ppu, seed=derive_seed(0, "train", "split"),
                                          population=Population.TRAIN, id_prefix="train"),
          Population.VAL: partition_iid(X[ntr:], y[ntr:], ppu, seed=derive_seed(0, "val", "split"),
                                        population=Population.VAL, id_prefix="val")}
    model = {"cnn": RefCNN, "mlp": lambda: MLP(wl["dim"], wl["hidden"], 10),
             "logistic": lambda: LogisticRegression(wl["dim"], 10)}[wl["model"]]()
    def make_alg(cohort):
        return FedAvg(model, SGDOptimizer(wl["clr"]), total_iterations=1 << 30, cohort_size=cohort,
                      local_learning_rate=wl["lr"], local_num_epochs=wl["epochs"], local_batch_size=wl["batch"],
                      eval_frequency=wl["eval_every"], eval_cohort_size=wl["eval_cohort"], weighting="uniform",
                      run_seed=0, init_seed=0)

    clip = ClippingPostprocessor(wl["bound"])
    mech = GaussianCentralMechanism(clip, sigma=wl["sigma"], r=wl["cohort"] / wl["noise_cohort"],
                                    noise_base_seed=derive_seed(0, "noise-stream", 0))
    return ds, make_alg, [clip, mech]


def _reference_iteration(setting, ds, alg, post, state, t, ncores):
    """Seconds for one central iteration of the reference (train context only)
    at ``alg.cohort_size`` users, in one of BASELINE.md section 2.3's settings:
    "blas"    SimulationEngine(num_workers=1), BLAS threads = ncores;
    "threads" SimulationEngine(num_workers=ncores), BLAS threads = 1;
    "procs"   the engine's per-worker _run_queue in ncores forked processes
              (BLAS 1 each) + its own worker_reduce / server postprocessors."""
    import multiprocessing as mp

    from fedsim.engine import SimulationEngine
    from fedsim.engine.scheduling import compute_base_weight, schedule_users
    from fedsim.feddata import sample_cohort
    from threadpoolctl import threadpool_limits

    ctx = alg.get_next_central_contexts(state, t)[0]
    t0 = time.perf_counter()
    if setting in ("blas", "threads"):
        workers = 1 if setting == "blas" else ncores
        with threadpool_limits(ncores if setting == "blas" else 1):
            eng = SimulationEngine(ds, num_workers=workers, postprocessors=post)
            res = eng.run_iteration(alg, state, (ctx,))
            state = alg.process_aggregated_statistics_all_contexts(state, (ctx,), res.aggregates, res.metrics,
                                                                   res.user_updates)
        return time.perf_counter() - t0, state
    eng = SimulationEngine(ds, num_workers=ncores, postprocessors=post)
    dataset = ds[ctx.population]
    cohort = sample_cohort(dataset, ctx.cohort_size, ctx.seed)
    w = {u: float(dataset.users[u].weight) for u in cohort}
    queues = schedule_users(w, ncores, compute_base_weight(list(w.values()), "median")).queues
    flat = [u for q in queues for u in q]
    bounds = np.cumsum([0] + [len(q) for q in queues])
    _REF.update(engine=eng, alg=alg, state=state, dataset=dataset, ctx=ctx, queue=flat)
    with mp.get_context("fork").Pool(ncores) as pool:
        outs = pool.map(_ref_queue_worker, [(int(a), int(b)) for a, b in zip(bounds[:-1], bounds[1:])])
    agg = eng._aggregator.worker_reduce([o[0] for o in outs])
    for proc in reversed(post):
        agg, _ = proc.postprocess_server(agg, ctx)
    state = alg.process_aggregated_statistics_all_contexts(state, (ctx,), (agg,), {}, [])
    return time.perf_counter() - t0, state


def reference_arm(args, wl):
    """The reference's own CPU implementation of the path on this box's host
    cores: fedsim's SimulationEngine / FedAvg / ClippingPostprocessor /
    GaussianCentralMechanism / SumAggregator from baseline/_ref, with the
    oracle CNN as the model (the reference has none).  Each step is one
    reference central iteration at a bounded cohort sample (3 x ncores users)
    in the fastest of BASELINE.md section 2.3's settings; the per-iteration
    cost at cohort C is a + C * b from a two-size fit (fixed cost a: noise
    over D, the server step; b: per user), plus the validation context
    amortised over eval_every.  Falls back to the oracle port's timing if
    baseline/_ref is absent."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    ncores = len(os.sched_getaffinity(0))
    C = wl["cohort"]
    try:
        ds, make_alg, post = _reference_setup(wl)
    except (ImportError, ValueError) as exc:
        return _reference_arm_port(args, wl, str(exc))
    small, big = ncores, 3 * ncores
    alg_small, alg_big = make_alg(small), make_alg(big)
    cpu = {"model": _cpu_model(), "affinity": ncores}
    # settings on the small sample (one iteration each, after a warm-up of the fastest)
    st = alg_small.initial_state()
    settings = {}
    for setting in ("procs", "threads", "blas"):
        if setting == "blas" and args.steps > 0:
            sec, st = _reference_iteration(setting, ds, alg_small, post, st, 1, ncores)
        else:
            _reference_iteration(setting, ds, alg_small, post, st, 1, ncores)
            sec, st = _reference_iteration(setting, ds, alg_small, post, st, 2, ncores)
        settings[setting] = sec
    best = min(settings, key=settings.get)
    st_big = alg_big.initial_state()
    for k in range(args.warmup):
        _, st_big = _reference_iteration(best, ds, alg_big, post, st_big, 1 + k, ncores)
    t_small = settings[best]
    times = []
    for k in range(args.steps):
        sec, st_big = _reference_iteration(best, ds, alg_big, post, st_big, 1 + args.warmup + k, ncores)
        times.append(sec)
    t_big = float(np.median(times))
    b = max((t_big - t_small) / (big - small), 1e-9)
    a = max(t_small - small * b, 0.0)
    # validation context (eval of eval_cohort users at theta_t), amortised over eval_every
    from fedsim.core import CentralContext, EvalParams
    from fedsim.engine import SimulationEngine
    from threadpoolctl import threadpool_limits

    vctx = CentralContext(iteration=0, population=next(p for p in ds if p.value == "val"),
                          cohort_size=wl["eval_cohort"], seed=0, do_training=False, eval_params=EvalParams())
    t0 = time.perf_counter()
    with threadpool_limits(1):
        SimulationEngine(ds, num_workers=ncores, postprocessors=post).run_iteration(alg_big, st_big, (vctx,))
    t_val = time.perf_counter() - t0
    it = a + C * b + t_val / wl["eval_every"]
    value = 1.0 / it
    sample = (f"reference SimulationEngine iterations at cohort {small} and {big} (median of {args.steps}), "
              f"setting '{best}'; fit a + C*b with a={a:.3f}s b={b:.4f}s/user -> cohort {C}, plus the "
              f"{wl['eval_cohort']}-user validation context ({t_val:.2f}s) / {wl['eval_every']}")
    line = {
        "metric": METRIC, "impl": "reference", "value": value, "unit": "iterations/s", "clients_per_sec": value * C,
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * it, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl["name"], "model": wl["model"], "cohort": C, "parallelism": "host-cpu"},
        "cpu_baseline": {"value": value, "unit": "iterations/s", "cores": ncores,
                         "kind": "reference", "sample": sample, "cpu": cpu,
                         "settings_s_per_iteration_at_small_cohort": {k: round(v, 3) for k, v in settings.items()},
                         "fastest": best},
        "e2e": {"value": value, "unit": "iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _reference_arm_port(args, wl, why):
    ds = build(wl)
    cpu_iteration_seconds(wl, ds, 1)  # warm-up (BLAS thread pools, page-in)
    its = []
    for k in range(args.steps):
        it, sample = cpu_iteration_seconds(wl, ds, args.ref_clients, t=k)
        its.append(it)
    value = 1.0 / float(np.mean(its))
    C = wl["cohort"]
    line = {
        "metric": METRIC, "impl": "reference", "value": value, "unit": "iterations/s", "clients_per_sec": value * C,
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 / value, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl["name"], "model": wl["model"], "cohort": C, "parallelism": "host-cpu"},
        "cpu_baseline": {"value": value, "unit": "iterations/s", "cores": _cores(), "kind": "port",
                         "sample": sample + f" (oracle port: {why})"},
        "e2e": {"value": value, "unit": "iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def aggregation_microbench(args):
    """BASELINE configs[4]: clip / aggregate / noise over a 10M-parameter
    update for cohort C on one GPU.  Client deltas come from a pool of P
    materialised [P, D] fp32 buffers (P * 40 MB >> L2, so every pass streams
    HBM); a step = K2 (norm + clip factor) and K3 (weighted sum) over all C
    clients in chunks of P, then K4+K5 (Philox noise + /W + SGD) once."""
    torch = _torch()
    from paper_2404_06430_b200 import native

    D, P, C = args.micro_dim, args.micro_pool, args.cohort or 1000
    ld = (D + 3) & ~3
    g = torch.Generator(device="cuda").manual_seed(0)
    pool = torch.randn(P, ld, device="cuda", generator=g) * (1.0 / np.sqrt(D))
    pool[P // 2:] *= 1e-4                      # half the pool below the bound: a clip mix
    w = torch.ones(P, device="cuda")
    norm = torch.empty(P, dtype=torch.float64, device="cuda")
    coef = torch.empty(P, device="cuda")
    clipped = torch.empty(P, dtype=torch.int32, device="cuda")
    bad = torch.empty(P, dtype=torch.int32, device="cuda")
    cws = torch.empty(max(native.call("fb_clip_workspace_bytes", P, D), 16), dtype=torch.uint8, device="cuda")
    sws = torch.empty(max(native.call("fb_weighted_sum_workspace_bytes", P, D), 16), dtype=torch.uint8, device="cuda")
    agg = torch.empty(D, device="cuda")
    theta = torch.zeros(D, device="cuda")
    s = native.stream_handle()

    fused = args.micro_impl == "fused"
    if fused:  # all C clients in ONE launch, client c reading pool row c % P
        fws = torch.empty(max(native.call("fb_clip_aggregate_workspace_bytes", C, D), 16), dtype=torch.uint8,
                          device="cuda")
        rows = torch.arange(C, device="cuda", dtype=torch.int32) % P
        wC = torch.ones(C, device="cuda")
        normC = torch.empty(C, dtype=torch.float64, device="cuda")
        coefC = torch.empty(C, device="cuda")
        clipC = torch.empty(C, dtype=torch.int32, device="cuda")
        badC = torch.empty(C, dtype=torch.int32, device="cuda")

    def step():
        if fused:  # K2 + K3 in one HBM pass (clip_aggregate_fused.cu)
            native.call("fb_clip_aggregate_rows_f32", pool.data_ptr(), rows.data_ptr(), ld, C, D, wC.data_ptr(), 1.0,
                        normC.data_ptr(), coefC.data_ptr(), clipC.data_ptr(), badC.data_ptr(), agg.data_ptr(), 0,
                        fws.data_ptr(), fws.numel(), s)
        for c0 in range(0, C if not fused else 0, P):
            n = min(P, C - c0)
            native.call("fb_delta_norm_clip_f32", pool.data_ptr(), ld, n, D, w.data_ptr(), 1.0, norm.data_ptr(),
                        coef.data_ptr(), clipped.data_ptr(), bad.data_ptr(), cws.data_ptr(), cws.numel(), s)
            native.call("fb_weighted_sum_f32", pool.data_ptr(), ld, n, D, coef.data_ptr(), agg.data_ptr(),
                        int(c0 > 0), sws.data_ptr(), sws.numel(), s)
        native.call("fb_noise_avg_sgd_f32", theta.data_ptr(), agg.data_ptr(), D, 0.1, 1234, None, 1.0 / C, 1.0,
                    None, s)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        step()
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    # per-kernel times from a second, instrumented pass (the headline window above has none)
    native.lib().fb_timing_enable(1)
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    rep = native.timing_report()
    native.lib().fb_timing_enable(0)
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm = peaks.get("hbm_gbs", 6650.0)
    b_alg = 4.0 * D * C + 12.0 * D   # each client read once + aggregate + theta r/w
    kern = {}
    chunks = -(-C // P)
    for name, bytes_per_step in (("row_sumsq_partial_kernel", 4.0 * D * C),
                                 ("weighted_sum_kernel", 4.0 * D * C + 4.0 * D * chunks),
                                 # one read per client + the aggregate written once (one launch)
                                 ("clip_aggregate_fused_kernel", 4.0 * D * C + 4.0 * D),
                                 ("noise_avg_sgd_kernel", 12.0 * D)):
        if name in rep:
            t = rep[name][0] / args.steps
            kern[name] = {"ms": round(t, 3), "GB/s": round(bytes_per_step / (t * 1e-3) / 1e9, 1),
                          "frac": round(bytes_per_step / (t * 1e-3) / 1e9 / hbm, 4)}
    print(json.dumps({
        "metric": "aggregation microbench (BASELINE configs[4]): clip + aggregate + noise, 10M-param update",
        "value": 1e3 / ms, "unit": "iterations/s", "clients_per_sec": C * 1e3 / ms, "ms_per_step": ms,
        "steps": args.steps, "warmup": args.warmup, "n_gpus": 1, "higher_is_better": True, "dtype": "f32",
        "config": {"workload": "aggmicro", "D": D, "cohort": C, "pool": P, "impl": args.micro_impl,
                   "l2": f"pool of {P} x {4 * ld / 1e6:.0f} MB client deltas >> L2"},
        "roofline": {"bound": "hbm", "achieved": round(b_alg / (ms * 1e-3) / 1e9, 1), "peak": hbm, "unit": "GB/s",
                     "frac": round(b_alg / (ms * 1e-3) / 1e9 / hbm, 4),
                     "algorithmic_bytes_per_step": b_alg,
                     "note": ("fused K2+K3: each client read once from HBM (re-read from L2)" if fused else
                              "K2 reads every client once more than B_alg counts")},
        "kernels": kern}), flush=True)


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS) + ["aggmicro"], default="cnn")
    ap.add_argument("--micro-dim", type=int, default=10_000_000)
    ap.add_argument("--micro-pool", type=int, default=64)
    ap.add_argument("--micro-impl", choices=["fused", "twopass"], default="fused")
    ap.add_argument("--cohort", type=int, default=None)
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--e2e-warmup", type=int, default=2)
    ap.add_argument("--cpu-clients", type=int, default=16)
    ap.add_argument("--profile-steps", type=int, default=5)
    ap.add_argument("--ref-clients", type=int, default=4)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args(argv)
    if args.warmup < 3 and args.impl == "ours":
        ap.error("--warmup must be >= 3")
    if args.workload == "aggmicro":
        aggregation_microbench(args)
        return
    wl = dict(WORKLOADS[args.workload])
    if args.cohort:
        wl["cohort"] = args.cohort
        wl["name"] += f" (cohort {args.cohort})"
    if args.impl == "reference":
        reference_arm(args, wl)
    else:
        gpu_arm(args, wl)


if __name__ == "__main__":
    main()
