"""Diagnostic: per-entry relative error of one ResNet-18 local step at the config D
shape (GPU tcgen05 / SIMT vs float64 oracle, and torch fp32 on the host as the fp32 floor)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2404_06430_b200 as fb  # noqa: E402
from oracle import port  # noqa: E402
from paper_2404_06430_b200 import native  # noqa: E402
from tests.test_gpu_resnet import run_local_sgd  # noqa: E402
from tests.test_oracle_resnet import torch_resnet_loss  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 224
n = int(sys.argv[2]) if len(sys.argv) > 2 else 16
m = port.ResNet18(image=S)
model = fb.ResNet18(image=S)
ds = fb.make_synthetic_images(1, image=S, num_classes=17, max_images=n, seed=2)
u = next(iter(ds.users.values()))
import dataclasses  # noqa: E402
X = u.features[:n].astype(np.float64)
u = dataclasses.replace(u, features=u.features[:n], labels=u.labels[:n]) if dataclasses.is_dataclass(u) else u
p0 = m.init(1)
theta = port.flat(p0, m.dims)
lr = 0.01
perm = port.user_perms(8, u.user_id, u.num_points, 1)
loss, g = m.loss_and_grad(p0, X[perm[0]])
want = port.flat(g, m.dims) * lr
# torch fp32 floor
p32 = {k: v.astype(np.float32).astype(np.float64) for k, v in p0.items()}
ref, t = torch_resnet_loss(m, p0, X[perm[0]])


def t32(m, p, Xb):
    import torch.nn.functional as F
    tt = {k: torch.tensor(v, dtype=torch.float32, requires_grad=True) for k, v in p.items()}
    Sx, K, w = m.image, m.num_classes, m.width
    x = torch.tensor(Xb[:, :3 * Sx * Sx].reshape(-1, 3, Sx, Sx), dtype=torch.float32)
    lab = torch.tensor(Xb[:, 3 * Sx * Sx:], dtype=torch.float32)
    gn = lambda h, name: F.group_norm(h, m.groups, tt[name + ".weight"], tt[name + ".bias"], m.eps)
    h = F.conv2d(x, tt["conv1.weight"].reshape(w, 3, 7, 7), stride=2, padding=3)
    h = F.max_pool2d(torch.relu(gn(h, "gn1")), 3, 2, 1)
    for name, ci, co, st, dsm in m.blocks():
        uu = torch.relu(gn(F.conv2d(h, tt[f"{name}.conv1.weight"].reshape(co, ci, 3, 3), stride=st, padding=1),
                           f"{name}.gn1"))
        v = gn(F.conv2d(uu, tt[f"{name}.conv2.weight"].reshape(co, co, 3, 3), padding=1), f"{name}.gn2")
        sc = h
        if dsm:
            sc = gn(F.conv2d(h, tt[f"{name}.downsample.0.weight"].reshape(co, ci, 1, 1), stride=st),
                    f"{name}.downsample.1")
        h = torch.relu(v + sc)
    z = h.mean(dim=(2, 3)) @ tt["fc.weight"].reshape(K, -1).T + tt["fc.bias"]
    l = F.binary_cross_entropy_with_logits(z, lab)
    l.backward()
    return np.concatenate([tt[k].grad.numpy().ravel().astype(np.float64) for k in m.dims]) * lr


floor = t32(m, p0, X[perm[0]])
res = {"torch_fp32": floor}
for impl in (1, 0):
    native.call("fb_lm_set_gemm_impl", impl)
    got, _ = run_local_sgd(model, theta, [u], 8, 1, n, lr)
    res["tc" if impl else "simt"] = got[0]
off = 0
rows = []
for name, k in m.dims.items():
    wv = want[off:off + k]
    line = [name[:28].ljust(28)]
    for key, v in res.items():
        e = np.linalg.norm(v[off:off + k] - wv) / max(np.linalg.norm(wv), 1e-30)
        line.append(f"{key} {e:.1e}")
    rows.append("  ".join(line))
    off += k
print("\n".join(rows))
for key, v in res.items():
    print(key, "total", np.linalg.norm(v - want) / np.linalg.norm(want))
