import sys, numpy as np
sys.path.insert(0, '.')
import paper_2404_06430_b200 as fb
from paper_2404_06430_b200 import native
from tests.fedsim_ref import build
from tests.helpers import CONFIGS
from tests.conftest import load_golden
g = load_golden("cnn_dp")
for impl in (1, 4):
    native.call("fb_cnn_set_conv_impl", impl)
    cfg = CONFIGS["cnn_dp"]
    fs, ds, alg, post = build(cfg)
    from fedsim.engine import SumAggregator, run_simulation
    eng = fb.GpuSimulationEngine(ds, postprocessors=post, aggregator=SumAggregator())
    names = list(alg.model.param_dims); dims = alg.model.param_dims
    thetas = []
    res = run_simulation(alg, eng, callbacks=[lambda p, rows, t: thetas.append(np.concatenate([np.asarray(p[n]) for n in names])) and False])
    keep = g["keep"]
    # map kept indices to parameter names
    offs = np.cumsum([0] + [int(np.prod(dims[n])) for n in names])
    idx = np.arange(offs[-1])[keep]
    for t, th in enumerate(thetas):
        a = th[keep].astype(np.float64); e = g["thetas"][t]
        atol = 1e-6 * np.abs(e).max(); err = np.abs(a - e); lim = 1e-5 * np.abs(e) + atol
        bad = np.where(err > lim)[0]
        where = {}
        for b in bad:
            k = np.searchsorted(offs, idx[b], side='right') - 1
            where[names[k]] = where.get(names[k], 0) + 1
        print(f"impl {impl} iter {t}: violations {len(bad)} max err/lim {(err/lim).max():.2f} where {where}")
native.call("fb_cnn_set_conv_impl", 1)
