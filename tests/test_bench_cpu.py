"""bench.py host logic without a GPU: every workload builds its seeded inputs with consistent
shapes, and the traffic lookup reads the committed ncu record."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

CONFIGS = ["trifocal", "fourview", "fivepoint", "p3p", "cyclic7", "cyclic7ph", "katsura6", "eco12"]


@pytest.mark.parametrize("name", CONFIGS)
def test_workload_shapes(name):
    d, start, p0, p1s, _, meta = bench.make_workload(name, 0, 2)
    assert meta["workload"]
    if start is None:   # total-degree single instance: the library builds start and parameters
        assert d.n_params == 0
        return
    assert start.ndim == 2 and start.shape[1] == d.n_vars and start.shape[0] >= 1
    assert p0.shape == (d.n_params,)
    assert p1s.ndim == 2 and p1s.shape[1] == d.n_params and p1s.shape[0] in (1, 2)
    assert np.all(np.isfinite(start)) and np.all(np.isfinite(p1s))


def test_rank_instance_blocks():
    """Each rank's instances come from distributed.shard_range: weak scaling gives every rank its own
    --instances block, strong scaling splits --total-instances (uneven totals too); instance b is the
    same input whichever rank (and block size) builds it."""
    import argparse
    weak = argparse.Namespace(instances=3, total_instances=0)
    strong = argparse.Namespace(instances=3, total_instances=7)
    assert [bench.instance_range(weak, r, 2) for r in range(2)] == [(0, 3), (3, 6)]
    assert [bench.instance_range(strong, r, 2) for r in range(2)] == [(0, 4), (4, 7)]
    assert [bench.instance_range(strong, r, 3) for r in range(3)] == [(0, 3), (3, 5), (5, 7)]
    whole = bench.make_workload("fourview", 0, 7)[3]
    parts = np.concatenate([bench.make_workload("fourview", *bench.instance_range(strong, r, 3))[3] for r in range(3)])
    assert np.array_equal(whole, parts)
    a = bench.make_workload("fourview", 0, 2)[3]
    b = bench.make_workload("fourview", 2, 4)[3]
    assert not np.allclose(a, b)


def test_traffic_lookup():
    assert bench.traffic_bytes("fourview", 1024, 296) > 0
    assert bench.traffic_bytes("trifocal", 7, 5344) is None
