"""Bit-plane 0/1 cells beyond RCPSP (lower.cpp lower_packed): small random
models built through the model API with reified overlaps over 0/1 cells,
capacity sums over them and precedences.  Each variant takes a different
device path — word-parallel bit rows with the kPacked kernel (coefficients
< 8), per-term bit rows in the all-families kernel (a coefficient of 9), and
the plain layout (a 0/1 cell also read by a precedence, so nothing packs) —
and every one must give the C oracle's enumeration counts and hash-sums (the
hash is over the reference layout, so it checks the decoding too) and its
optima."""
import numpy as np
import pytest

from oracle.port import Oracle

pytestmark = pytest.mark.gpu


def build(seed, n=6, horizon=9, big_coef=False, leak=False):
    from paper_2207_12116_b200.model import Model, and_c, leq, leq_offset, linear_leq, precedes
    rng = np.random.default_rng(seed)
    m = Model()
    x = [m.add_cell() for _ in range(n)]
    b = [[m.add_cell() for _ in range(n)] for _ in range(n)]
    d = [int(v) for v in rng.integers(1, 4, n)]
    for i in range(n):
        m.tell(x[i], 0, horizon)
    for i in range(n):
        for j in range(n):
            m.tell(b[i][j], 0, 1)
    for i in range(n):
        m.tell(b[i][i], 1, 1)
    for j in range(n):
        for i in range(n):
            if i != j:
                m.post_reified(b[i][j], and_c(leq(x[i], x[j]), leq_offset(x[j], 1 - d[i], x[i])))
    for j in range(n):
        use = [int(u) for u in rng.integers(0, 5, n)]
        if big_coef:
            use[0] = 9
        terms = [(use[i], b[i][j]) for i in range(n) if use[i] > 0]
        if terms:
            m.post(linear_leq(terms, int(rng.integers(2, 6)) if not big_coef else 10))
    for _ in range(2):
        i, j = sorted(int(v) for v in rng.choice(n, 2, replace=False))
        m.post(precedes(x[i], d[i], x[j]))
    if leak:  # a 0/1 cell read by a precedence: it cannot leave the word store
        m.post(precedes(b[0][1], 0, x[2]))
    m.set_candidates(x)
    m.set_objective(x[n - 1])
    return m


@pytest.mark.parametrize("group_threads", [0, 64])  # warp groups (these stores are small), CTA groups
@pytest.mark.parametrize("variant", ["wrows", "brows", "plain"])
def test_packed_paths_match_the_oracle(variant, group_threads):
    from paper_2207_12116_b200 import Engine
    from paper_2207_12116_b200._native import STATUS_NAMES
    kw = {"wrows": {}, "brows": {"big_coef": True}, "plain": {"leak": True}}[variant]
    for seed in range(6):
        m = build(seed, **kw)
        t = m.tables()
        o = Oracle(t)
        with Engine(0, hash=True, group_threads=group_threads) as e:
            e.load(m)
            info = e.lowering_info()
            assert (info["packed_cells"] > 0) == (variant != "plain"), (variant, seed)
            got = e.enumerate(depth_cap=10)
            want = o.enumerate(m.bottom(), depth_cap=10)
            for k in ("nodes", "failures", "solutions", "open_leaves", "hash_sum"):
                assert got[k] == want[k], (variant, seed, k)
            r = e.solve(timeout_s=30)
        s = o.solve_dfs(m.bottom())
        assert r.status == STATUS_NAMES[s["status"]] and r.objective == s["objective"], (variant, seed, r.status, s)
