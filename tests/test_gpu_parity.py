"""Parity of the CUDA path against the reference (golden fixtures generated from
the reference library by tests/golden/make_golden.py) and the C oracle.

Integer work: every comparison is bit-exact.  Node counts of the optimisation
runs differ from the reference only through search order (incumbent timing);
those tests compare optima and check every solution independently."""
import numpy as np
import pytest

from conftest import load_micro_csps, load_micro_rcpsps
from oracle.port import Oracle, store_hash

pytestmark = pytest.mark.gpu

CONFIG_BUILDERS = {}


def build(name):
    from paper_2207_12116_b200 import Model
    if name.startswith("nqueens"):
        return Model.nqueens(int(name[len("nqueens"):]))
    if name == "csp1":
        return Model.random_csp(1)
    if name.startswith("csp_small"):
        return Model.random_csp(int(name[len("csp_small"):]), n_vars=60, n_cons=200)
    if name.startswith("rcpsp30_s"):
        return Model.rcpsp_random(int(name[len("rcpsp30_s"):]), 30, 4)
    if name.startswith("rcpsp10_s"):
        return Model.rcpsp_random(int(name[len("rcpsp10_s"):]), 10, 2)
    if name.startswith("rcpsp120_s"):
        return Model.rcpsp_random(int(name[len("rcpsp120_s"):]), 120, 4)
    return None


@pytest.fixture(scope="module")
def engine():
    from paper_2207_12116_b200 import Engine
    with Engine(0) as e:
        yield e


@pytest.fixture(scope="module")
def hengine():
    from paper_2207_12116_b200 import Engine
    with Engine(0, hash=True) as e:
        yield e


def config_names(golden, prefix=None):
    return [n for n in golden if build(n) is not None and (prefix is None or n.startswith(prefix))]


def test_root_fixpoints_all_configs(golden, engine):
    """run_sequential on the bottom store of every configuration (K1)."""
    for name in config_names(golden):
        g = golden[name]
        m = build(name)
        assert m.tables().n_cmds == g["n_cmds"], name
        engine.load(m)
        failed, words, rounds = engine.run_sequential()
        assert failed == g["root"]["failed"], name
        if not failed:
            assert store_hash(words) == g["root"]["hash"], name


@pytest.mark.parametrize("tag", ["micro_csp_s2", "micro_csp_s4242"])
def test_micro_csp_fixpoints(tag, engine):
    """The reference acceptance confluence instances (acceptance_main.cpp:170-174)
    and test_engine.cpp:94-114's: GPU fixed point == run_sequential's."""
    for i, (t, failed, fix, _) in enumerate(load_micro_csps(tag)):
        engine.load(t)
        f, w, _ = engine.run_sequential()
        assert f == failed, (tag, i)
        if not failed:
            assert np.array_equal(w, fix), (tag, i)


def test_micro_csp_batch_random_stores(engine):
    """Batched K1 on random sub-boxes of every micro CSP vs the C oracle."""
    rng = np.random.default_rng(7)
    for t, _, _, _ in load_micro_csps("micro_csp_s2")[:200]:
        o = Oracle(t)
        engine.load(t)
        base = o.bottom()
        stores = []
        for _ in range(8):
            s = base.copy()
            for k, w in zip(t.slot_kind, t.slot_word):
                if k == 4:
                    a, b = sorted(rng.integers(-1, 10, 2))
                    s[w], s[w + 1] = a, b + int(rng.integers(0, 3))
            stores.append(s)
        out, failed, _ = engine.propagate_batch(np.stack(stores))
        for s, w, f in zip(stores, out, failed):
            fo, wo, _, _ = o.run_sequential(s)
            assert f == fo
            if not f:
                assert np.array_equal(w, wo)


def _strip_init(m, n_init):
    from paper_2207_12116_b200.model import Tables
    t = m.tables()
    off = (t.cmd_off[n_init:] - t.cmd_off[n_init]).astype(np.uint32)
    return Tables(t.slot_kind, t.slot_word, t.n_words, off, t.cmd_code[t.cmd_off[n_init]:], t.cands, t.obj_slot)


@pytest.mark.parametrize("shift", [0, 2**30 - 4, -(2**30) + 2, 2**31 - 12, -(2**31) + 12])
@pytest.mark.parametrize("n", [8, 14])
def test_sentinel_and_wide_arithmetic(n, shift, engine):
    """H1: +-inf sentinels and values beyond +-2^30 (the 32-bit fast path's
    range) must follow the reference's widened int64 arithmetic exactly.
    N-Queens commands without their init tells, random stores with infinite
    and shifted bounds, GPU == C oracle."""
    t = _strip_init(build(f"nqueens{n}"), n)
    o = Oracle(t)
    engine.load(t)
    rng = np.random.default_rng(n * 1000 + (shift % 997))
    MIN, MAX = -(2**31), 2**31 - 1
    stores = []
    for _ in range(512):
        s = o.bottom()
        for w in t.slot_word:
            r = rng.random()
            a, b = sorted(int(v) + shift for v in rng.integers(-3, n + 1, 2))
            a, b = min(max(a, MIN + 1), MAX - 1), min(max(b, MIN + 1), MAX - 1)
            if r < 0.5:
                s[w], s[w + 1] = a, b
            elif r < 0.7:
                s[w], s[w + 1] = MIN, b
            elif r < 0.9:
                s[w], s[w + 1] = a, MAX
        stores.append(s)
    out, failed, _ = engine.propagate_batch(np.stack(stores))
    for s, w, f in zip(stores, out, failed):
        fo, wo, _, _ = o.run_sequential(s)
        assert f == fo
        if not f:
            assert np.array_equal(w, wo)


@pytest.mark.parametrize("shift", [0, 5000, 2**29 - 40000, -(2**29) + 3])
@pytest.mark.parametrize("n", [8, 14])
def test_ne_fast_path_finite_boxes(n, shift, engine):
    """Finite stores: the host's value-range analysis (ne_fast_ok) admits the
    check-free NE path for small boxes and refuses it near 2^29; either way the
    fixed points equal the oracle's (and the same run with PCCP_NO_NE_FAST)."""
    import os
    t = _strip_init(build(f"nqueens{n}"), n)
    o = Oracle(t)
    engine.load(t)
    rng = np.random.default_rng(n * 7919 + (shift % 1009))
    stores = []
    for _ in range(512):
        s = o.bottom()
        for w in t.slot_word:
            a, b = sorted(int(v) + shift for v in rng.integers(-3, n + 1, 2))
            s[w], s[w + 1] = a, b + int(rng.integers(0, 2))
        stores.append(s)
    out, failed, _ = engine.propagate_batch(np.stack(stores))
    os.environ["PCCP_NO_NE_FAST"] = "1"
    try:
        out2, failed2, _ = engine.propagate_batch(np.stack(stores))
    finally:
        del os.environ["PCCP_NO_NE_FAST"]
    assert np.array_equal(failed, failed2)
    for s, w, w2, f in zip(stores, out, out2, failed):
        fo, wo, _, _ = o.run_sequential(s)
        assert f == fo
        if not f:
            assert np.array_equal(w, wo) and np.array_equal(w2, wo)


@pytest.mark.parametrize("seed", [1, 3])
def test_rows_fast_path_random_boxes(seed, engine):
    """RCPSP30 stores with random start windows and random 0/1 overlap booleans
    (after the init tells): the rows' 32-bit path (rows_fast_ok) and the
    widened path (PCCP_NO_FAST) both equal the C oracle, fixed point and
    failure; a store with an unbounded boolean must take the widened path."""
    import os
    m = build(f"rcpsp30_s{seed}")
    t = m.tables()
    o = Oracle(t)
    engine.load(m)
    root = o.run_sequential(m.bottom())[1]
    starts = set(int(t.slot_word[s]) for s in m.starts())
    rng = np.random.default_rng(seed)
    stores = []
    sw = sorted(starts)
    for k in range(64):
        s = root.copy()
        for w in rng.choice(sw, size=int(rng.integers(1, 8)), replace=False):
            lo, hi = int(s[w]), int(s[w + 1])
            a = int(rng.integers(lo, min(hi, lo + 10) + 1))
            b = int(rng.integers(a, min(hi, a + 12) + 1))
            s[w], s[w + 1] = a, b
        for w in range(0, t.n_words, 2):
            if w not in starts and s[w] == 0 and s[w + 1] == 1 and rng.random() < 0.003:
                v = int(rng.integers(0, 2))
                s[w], s[w + 1] = v, v
        stores.append(s)
    out, failed, _ = engine.propagate_batch(np.stack(stores))
    os.environ["PCCP_NO_FAST"] = "1"
    try:
        out2, failed2, _ = engine.propagate_batch(np.stack(stores))
    finally:
        del os.environ["PCCP_NO_FAST"]
    assert failed.any() and not failed.all()
    for s, w, w2, f, f2 in zip(stores, out, out2, failed, failed2):
        fo, wo, _, _ = o.run_sequential(s)
        assert f == fo == f2
        if not f:
            assert np.array_equal(w, wo) and np.array_equal(w2, wo)


@pytest.mark.parametrize("n", [8, 10])
def test_enumerate_nqueens_without_fast_path(n, golden):
    import os
    from paper_2207_12116_b200 import Engine
    g = golden[f"nqueens{n}"]["enumerate"]
    os.environ["PCCP_NO_NE_FAST"] = "1"
    try:
        with Engine(0, hash=True) as e:
            res = e.load(build(f"nqueens{n}")).enumerate()
    finally:
        del os.environ["PCCP_NO_NE_FAST"]
    for k in ("nodes", "failures", "solutions", "hash_sum"):
        assert res[k] == g[k], (n, k)


def test_replayed_paths(golden, engine):
    """materialize() of sampled decision paths (with objective bounds) == reference."""
    for name in config_names(golden):
        g = golden[name]
        reps = g.get("replays")
        if not reps:
            continue
        engine.load(build(name))
        paths = [r["decisions"] for r in reps]
        best = [r["best"] for r in reps]
        out, failed = engine.replay(paths, best)
        for r, w, f in zip(reps, out, failed):
            assert f == r["failed"], name
            if not f:
                assert store_hash(w) == r["hash"], name


@pytest.mark.parametrize("n", [4, 5, 6, 8, 10])
def test_enumerate_nqueens(n, golden, hengine):
    g = golden[f"nqueens{n}"]["enumerate"]
    res = hengine.load(build(f"nqueens{n}")).enumerate()
    for k in ("nodes", "failures", "solutions", "open_leaves", "hash_sum"):
        assert res[k] == g[k], (n, k)
    assert res["exhausted"]


def test_enumerate_csp_depth12(golden, hengine):
    g = golden["csp1"]["enumerate_d12"]
    res = hengine.load(build("csp1")).enumerate(depth_cap=12)
    for k in ("nodes", "failures", "solutions", "open_leaves", "hash_sum"):
        assert res[k] == g[k], k


@pytest.mark.parametrize("group_threads", [0, 32, 128, 512])
def test_enumerate_csp_depth22_repeatable(group_threads, golden):
    """Config 3 at the benchmark depth, under warp- and CTA-sized groups, three
    times each: chaotic parallel rounds must still give identical counts."""
    from paper_2207_12116_b200 import Engine
    g = golden["csp1"]["enumerate_d22"]
    with Engine(0, hash=True, group_threads=group_threads) as e:
        e.load(build("csp1"))
        for _ in range(3):
            res = e.enumerate(depth_cap=22)
            for k in ("nodes", "failures", "solutions", "open_leaves", "hash_sum"):
                assert res[k] == g[k], (group_threads, k, res[k], g[k])


@pytest.mark.parametrize("group_threads", [64, 256])
def test_enumerate_nqueens_cta_groups(group_threads, golden):
    from paper_2207_12116_b200 import Engine
    g = golden["nqueens10"]["enumerate"]
    with Engine(0, hash=True, group_threads=group_threads) as e:
        e.load(build("nqueens10"))
        for _ in range(3):
            res = e.enumerate()
            for k in ("nodes", "failures", "solutions", "hash_sum"):
                assert res[k] == g[k], (group_threads, k)


@pytest.mark.parametrize("seed", [2, 3])
def test_enumerate_small_csp(seed, golden, hengine):
    g = golden[f"csp_small{seed}"]["enumerate_d10"]
    res = hengine.load(build(f"csp_small{seed}")).enumerate(depth_cap=10)
    for k in ("nodes", "failures", "solutions", "open_leaves", "hash_sum"):
        assert res[k] == g[k], k


@pytest.mark.parametrize("seed", [1, 5, 11])
def test_rcpsp30_optimum(seed, golden, engine):
    m = build(f"rcpsp30_s{seed}")
    res = engine.load(m).solve(timeout_s=120)
    assert res.status == "OPTIMAL"
    assert res.objective == golden[f"rcpsp30_s{seed}"]["optimum"]["value"]
    assert m.check_solution(res.best_words)
    incs = [v for v, _ in res.improvements]
    assert all(a > b for a, b in zip(incs, incs[1:]))  # strictly decreasing (test_solver.cpp:247-261)


@pytest.mark.parametrize("seed", range(1, 9))
def test_rcpsp10_optimum(seed, golden, engine):
    g = golden[f"rcpsp10_s{seed}"]["solve_dfs"]
    m = build(f"rcpsp10_s{seed}")
    res = engine.load(m).solve()
    assert res.status == {0: "OPTIMAL", 2: "UNSAT"}[g["status"]]
    assert res.objective == g["objective"]
    if res.objective is not None:
        assert m.check_solution(res.best_words)


def test_micro_rcpsp_optimality(engine):
    """200 micro RCPSPs of the optimality criterion (acceptance_main.cpp:243-287):
    GPU optimum == brute-force enumeration, UNSAT where the reference proves it."""
    for t, rec in load_micro_rcpsps():
        engine.load(t)
        res = engine.solve()
        if rec["brute_force"] is None:
            assert res.status == "UNSAT"
        else:
            assert res.status == "OPTIMAL" and res.objective == rec["brute_force"]


def test_node_limit_zero_is_unknown(engine):
    from paper_2207_12116_b200 import Model
    m = Model.rcpsp([0, 2, 3, 0], [[0], [1], [1], [0]], [1], [(0, 1), (0, 2), (1, 2), (1, 3), (2, 3)], 5)
    engine.load(m)
    assert engine.solve(node_limit=0).status == "UNKNOWN"
    r = engine.solve()
    assert r.status == "OPTIMAL" and r.objective == 5  # test_solver.cpp:70-79


def test_unsat_below_healthy_root(engine):
    """test_solver.cpp:105-126: three unit tasks on capacity one cannot fit horizon 5."""
    from paper_2207_12116_b200 import Model
    prec = []
    for i in (1, 2, 3):
        prec += [(0, i), (i, 4)]
    m = Model.rcpsp([0, 2, 2, 2, 0], [[0], [1], [1], [1], [0]], [1], prec, 5)
    engine.load(m)
    failed, _, _ = engine.run_sequential()
    assert not failed
    assert engine.solve().status == "UNSAT"


@pytest.mark.parametrize("dom_hi", [100, 10**6, 10**8, 2**30])
def test_value_range_analysis_large_domains(dom_hi, hengine):
    """Random linear CSPs whose domains grow until the value-range analysis must
    refuse the 32-bit row path (|sum| would pass 2^30) and then past the
    reference's own 2^30 fast range: depth-capped enumeration counts and
    hash-sums equal the C oracle's in every case."""
    from paper_2207_12116_b200 import Model
    m = Model.random_csp(5, n_vars=40, n_cons=120, dom_hi=dom_hi)
    t = m.tables()
    want = Oracle(t).enumerate(m.bottom(), depth_cap=9)
    got = hengine.load(m).enumerate(depth_cap=9)
    for k in ("nodes", "failures", "solutions", "open_leaves", "hash_sum"):
        assert got[k] == want[k], (dom_hi, k, got[k], want[k])


def test_enumerate_csp_depth12_without_fast_paths(golden):
    """Config 3 through the widened unit/row/reification paths (PCCP_NO_FAST):
    the same golden counts and hash-sum as the 32-bit paths."""
    import os
    from paper_2207_12116_b200 import Engine
    g = golden["csp1"]["enumerate_d12"]
    os.environ["PCCP_NO_FAST"] = "1"
    try:
        with Engine(0, hash=True) as e:
            res = e.load(build("csp1")).enumerate(depth_cap=12)
    finally:
        del os.environ["PCCP_NO_FAST"]
    for k in ("nodes", "failures", "solutions", "open_leaves", "hash_sum"):
        assert res[k] == g[k], k


@pytest.mark.parametrize("limit", [1, 7, 500, 5000])
def test_node_limit_bounds_materialisations(limit, golden):
    """SharedControl's node limit (solver.cpp:68-76) counts every materialisation,
    the root and the decomposition's included: the search stops after about
    `limit` nodes (groups overshoot by at most one node each) and reports a
    non-exhausted run; a limit above the tree size changes nothing."""
    from paper_2207_12116_b200 import Engine
    with Engine(0) as e:
        e.load(build("nqueens10"))
        r = e.enumerate(node_limit=limit)
        assert not r["exhausted"]
        assert r["nodes"] <= limit + 2 * 4736, (limit, r["nodes"])
        full = e.enumerate(node_limit=10**9)
        assert full["exhausted"] and full["nodes"] == golden["nqueens10"]["enumerate"]["nodes"]
        m = build("rcpsp30_s1")
        e.load(m)
        s = e.solve(node_limit=limit)
        assert s.status in ("SAT", "UNKNOWN")
        assert s.stats["nodes"] <= limit + 2 * 4736
        if s.objective is not None:
            assert m.check_solution(s.best_words)


@pytest.mark.parametrize("seed", [1, 2])
def test_interleaved_scalar_cells(seed, hengine):
    """A store whose scalar cells (sum accumulators) sit between interval
    cells: the failure scan cannot walk the intervals by index (lower.cpp
    iv_prefix) and reads the interval and scalar lists.  Enumeration counts and
    hash-sum, GPU == C oracle."""
    from paper_2207_12116_b200 import Model
    from paper_2207_12116_b200.model import Kind, leq_offset, linear_leq
    rng = np.random.default_rng(seed)
    m = Model()
    xs = []
    for blk in range(4):
        for _ in range(4):
            x = m.add_cell()
            m.tell(x, 0, 6)
            xs.append(x)
        # sums over the cells so far: their accumulators follow this block
        for _ in range(2):
            idx = rng.choice(len(xs), size=3, replace=False)
            terms = [(int(rng.integers(1, 4)), xs[i]) for i in idx]
            m.post(linear_leq(terms, int(rng.integers(6, 14))))
        i, j = sorted(rng.choice(len(xs), size=2, replace=False))
        m.post(leq_offset(xs[i], 1, xs[j]))
    t = m.tables()
    scal = [w for k, w in zip(t.slot_kind, t.slot_word) if k != Kind.Interval]
    assert scal and min(scal) < max(t.slot_word), "scalars must be interleaved"
    o = Oracle(t)
    g = o.enumerate(o.bottom(), depth_cap=24)
    assert g["nodes"] > 1000 and g["exhausted"]
    res = hengine.load(m).enumerate(depth_cap=24)
    for k in ("nodes", "failures", "solutions", "open_leaves", "hash_sum"):
        assert res[k] == g[k], k


@pytest.mark.parametrize("group_threads,groups_per_cta,ctas_per_sm,eps_factor", [
    (32, 3, 0, 0),    # warp groups, 3 per CTA: ownership windows of a non-power-of-two width
    (32, 8, 1, 64),   # one CTA per SM, a deep frontier: small levels, then chunked ones
    (128, 0, 0, 4),   # CTA groups with a decomposition (one group per CTA)
    (256, 0, 1, 1),   # CTA groups, a frontier of one node per group
])
def test_decomposition_shapes_enumerate_exactly(group_threads, groups_per_cta, ctas_per_sm, eps_factor, golden):
    """The EPS decomposition's barrier-free small levels (every CTA compacting
    the flags itself, children on their own groups) and its chunked large
    levels, under grid shapes the defaults do not use: Q10 and the CSP at
    depth 12 must give the golden counts and hash-sums."""
    from paper_2207_12116_b200 import Engine
    with Engine(0, hash=True, group_threads=group_threads, groups_per_cta=groups_per_cta, ctas_per_sm=ctas_per_sm,
                eps_factor=eps_factor) as e:
        g = golden["nqueens10"]["enumerate"]
        res = e.load(build("nqueens10")).enumerate()
        for k in ("nodes", "failures", "solutions", "hash_sum"):
            assert res[k] == g[k], (k, res[k], g[k])
        g = golden["csp1"]["enumerate_d12"]
        res = e.load(build("csp1")).enumerate(depth_cap=12)
        for k in ("nodes", "failures", "solutions", "open_leaves", "hash_sum"):
            assert res[k] == g[k], (k, res[k], g[k])
