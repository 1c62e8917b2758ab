"""The two round schedules of packed models (kernels.cuh): the eventless loop
(kPacked, every record every round: RCPSP30's default) and filtered rounds
(kPackedF: only the records reading a start or plane word changed in the
previous round, by segment: RCPSP120's default).  Both must give the
reference's fixed points per node and its optima, whichever a model gets by
default, so every check here runs under both (PCCP_PACKED_FILTER=0/1, read at
load)."""
import os

import numpy as np
import pytest

from oracle.port import Oracle
from test_gpu_node_audit import audited, check_samples
from test_gpu_parity import build

pytestmark = pytest.mark.gpu

RCPSP30_OPTIMA = {1: 84, 2: 77, 5: 73, 7: 60, 9: 61, 11: 99}


@pytest.fixture(params=["0", "1"], ids=["eventless", "filtered"])
def schedule(request, monkeypatch):
    monkeypatch.setenv("PCCP_PACKED_FILTER", request.param)
    return request.param


def test_rcpsp30_optima(schedule):
    from paper_2207_12116_b200 import Engine, Model
    for seed, opt in RCPSP30_OPTIMA.items():
        m = Model.rcpsp_random(seed, 30, 4)
        with Engine(0) as e:
            r = e.load(m).solve(timeout_s=60)
        assert r.status == "OPTIMAL" and r.objective == opt and m.check_solution(r.best_words), (schedule, seed)


@pytest.mark.parametrize("seed", [1, 7])
def test_rcpsp30_nodes(seed, schedule, golden):
    m, s, pre, post, failed = audited(f"rcpsp30_s{seed}", 48, 10, lambda e: e.solve(timeout_s=60))
    assert s.status == "OPTIMAL" and s.objective == golden[f"rcpsp30_s{seed}"]["optimum"]["value"]
    check_samples(m, pre, post, failed)


def test_rcpsp120_reference_order_nodes(schedule):
    """The reference's order (no incumbent): 2^12-th nodes of a 200k-node search."""
    m, s, pre, post, failed = audited("rcpsp120_s1", 40, 12, lambda e: e.solve(node_limit=200000))
    assert s.status == "UNKNOWN"
    check_samples(m, pre, post, failed)


def test_rcpsp_fixed_points_of_random_boxes(schedule):
    """propagate_batch on random sub-boxes of RCPSP30/120 roots (the first round
    evaluates everything, later ones only what changed)."""
    from paper_2207_12116_b200 import Engine, Model
    rng = np.random.default_rng(11)
    for n in (30, 120):
        m = Model.rcpsp_random(1, n, 4)
        t = m.tables()
        o = Oracle(t)
        _, root, _, _ = o.run_sequential(m.bottom())
        starts = [int(t.slot_word[s]) for s in m.starts()]
        stores = []
        for _ in range(24):
            s = root.copy()
            for w in rng.choice(starts, size=6, replace=False):
                lo, hi = int(s[w]), int(s[w + 1])
                if hi > lo:
                    cut = int(rng.integers(lo, hi + 1))
                    if rng.integers(0, 2):
                        s[w] = cut
                    else:
                        s[w + 1] = cut
            stores.append(s)
        with Engine(0) as e:
            out, failed, _ = e.load(m).propagate_batch(np.stack(stores))
        for s, w, f in zip(stores, out, failed):
            fo, wo, _, _ = o.run_sequential(s)
            assert f == fo
            if not f:
                assert np.array_equal(w, wo)
