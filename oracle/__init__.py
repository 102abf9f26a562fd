"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

A float64 numpy restatement of the reference's central-iteration path
(fedsim 0.1.0 under /root/reference/pkg/src/fedsim), used as the parity
checker by ``tests/``, by ``__graft_entry__.smoke()`` and as the timed
CPU baseline (``bench.py`` cpu_baseline leg and ``--impl reference``).
Nothing in ``paper_2404_06430_b200/`` imports it; the product path runs on
the GPU or fails loudly.

Pinning: the logistic / MLP arithmetic, sampling, scheduling, clipping,
aggregation, noise stream and central step are checked against golden
vectors dumped from the reference itself (tests/golden/make_golden.py,
run in the container where /root/reference is importable).  The CNN has
no reference implementation; its oracle is pinned by finite differences
and by running it through the reference's own generic ``Model.fit_local``
loop (also in the golden fixtures).
"""
