"""CSV partitions (`user_id,f0..f{d-1},label`) in the
reference's format (fedsim/feddata/io.py:19-60).

* files written by the package are byte-identical to the reference's
  `save_partition` of the same dataset, and each side loads the other's file
  back losslessly (shortest round-trip float repr, io.py:1-5);
* the reference's error conventions (DataError for a missing / empty /
  header-less / ragged / row-less file, io.py:31-58);
* GPU: an engine fed the loaded partition produces the same iteration as one
  fed the in-memory partition (bitwise), and matches the reference run."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2404_06430_b200 as fb
from tests.fedsim_ref import fedsim


def _dataset(n_users=7, ppu=5, dim=6, seed=11):
    X, y = fb.make_synthetic_classification(n_users * ppu, dim=dim, num_classes=4, margin=3.0, seed=seed)
    return fb.partition_iid(X, y, ppu, seed=seed + 1, population=fb.Population.TRAIN, id_prefix="train")


def _assert_same_dataset(a_users, b_users):
    assert list(a_users) == list(b_users)
    for uid in a_users:
        a, b = a_users[uid], b_users[uid]
        assert a.features.dtype == b.features.dtype == np.float64
        assert a.labels.dtype == b.labels.dtype == np.int64
        np.testing.assert_array_equal(a.features, b.features)
        np.testing.assert_array_equal(a.labels, b.labels)


def test_round_trip_lossless(tmp_path):
    ds = _dataset()
    path = tmp_path / "part.csv"
    fb.save_partition(ds, path)
    back = fb.load_partition(path, fb.Population.TRAIN)
    assert back.population == fb.Population.TRAIN
    _assert_same_dataset(ds.users, back.users)


def test_byte_identical_to_reference_writer(tmp_path):
    fs = fedsim()
    from fedsim.core import Population
    from fedsim.feddata.datasets import FederatedDataset, UserDataset
    from fedsim.feddata.io import load_partition, save_partition

    ds = _dataset()
    ref_ds = FederatedDataset(users={u.user_id: UserDataset(u.user_id, u.features, u.labels)
                                     for u in ds.users.values()}, population=Population.TRAIN)
    ours, theirs = tmp_path / "ours.csv", tmp_path / "theirs.csv"
    fb.save_partition(ds, ours)
    save_partition(ref_ds, theirs)
    assert ours.read_bytes() == theirs.read_bytes()
    # each side reads the other's file back exactly
    _assert_same_dataset(fb.load_partition(theirs, fb.Population.TRAIN).users, ds.users)
    _assert_same_dataset(load_partition(ours, Population.TRAIN).users, ds.users)
    assert fs is not None


def test_ragged_users_and_row_order(tmp_path):
    """Rows of one user need not be contiguous; users keep first-seen order
    and rows keep file order (io.py:44-47)."""
    path = tmp_path / "p.csv"
    path.write_text("user_id,f0,f1,label\n"
                    "b,1.0,2.0,1\n"
                    "a,0.1,0.2,0\n"
                    "b,3.5,-4.25,2\n")
    ds = fb.load_partition(path, fb.Population.VAL)
    assert list(ds.users) == ["b", "a"]
    np.testing.assert_array_equal(ds.users["b"].features, [[1.0, 2.0], [3.5, -4.25]])
    np.testing.assert_array_equal(ds.users["b"].labels, [1, 2])
    assert ds.users["a"].num_points == 1


@pytest.mark.parametrize("content,match", [
    (None, "partition file not found"),
    ("", "partition file is empty"),
    ("uid,f0,label\nu,1.0,0\n", "unexpected partition header"),
    ("user_id,f0,f1,label\nu,1.0,0\n", r"p\.csv:2: expected 4 columns"),
    ("user_id,f0,label\n", "partition file has no rows"),
])
def test_errors_match_reference(tmp_path, content, match):
    fedsim()
    from fedsim.core import Population
    from fedsim.errors import DataError as RefDataError
    from fedsim.feddata.io import load_partition

    path = tmp_path / "p.csv"
    if content is not None:
        path.write_text(content)
    with pytest.raises(fb.DataError, match=match) as ours:
        fb.load_partition(path, fb.Population.TRAIN)
    with pytest.raises(RefDataError) as theirs:
        load_partition(path, Population.TRAIN)
    assert str(ours.value) == str(theirs.value)


@pytest.mark.gpu
def test_engine_on_loaded_partition(tmp_path, golden):
    """The GPU engine on a CSV partition written by the REFERENCE's
    save_partition gives bitwise the same model as on the in-memory
    partition, and matches the reference run (mlp_dp golden)."""
    fedsim()
    from fedsim.core import Population
    from fedsim.feddata.datasets import FederatedDataset, UserDataset
    from fedsim.feddata.io import save_partition

    from tests.conftest import assert_close_fp32
    from tests.helpers import CONFIGS, product_datasets, product_run_parts, run_sim

    cfg = CONFIGS["mlp_dp"]
    g = golden("mlp_dp")
    ds = product_datasets(cfg)
    loaded = {}
    for pop, part in ds.items():
        path = tmp_path / f"{pop.value}.csv"
        save_partition(FederatedDataset(users={u.user_id: UserDataset(u.user_id, u.features, u.labels)
                                               for u in part.users.values()},
                                        population=Population(pop.value)), path)
        loaded[pop] = fb.load_partition(path, pop)

    def run(datasets):
        alg, post = product_run_parts(cfg)
        thetas = []
        res = run_sim(alg, fb.GpuSimulationEngine(datasets, postprocessors=post),
                      callbacks=[lambda p, rows, t: thetas.append(p.flat_host()) and False])
        return res, thetas

    res_mem, th_mem = run(ds)
    res_csv, th_csv = run(loaded)
    assert res_csv.cohort_digest == res_mem.cohort_digest == str(g["digest"])
    for t in range(len(th_mem)):
        np.testing.assert_array_equal(th_csv[t], th_mem[t])
        assert_close_fp32(th_csv[t], g["thetas"][t], what=f"theta after iteration {t}")
