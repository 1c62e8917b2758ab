"""The product's host model builder (csrc/host) against the reference's model
API: identical flat tables (slot numbering, command order, word indices) for
every benchmark configuration, and the reference's own propagation unit
cases (test_propagation.cpp, test_engine.cpp, test_solver.cpp) replayed on
product-built tables through the C oracle."""
import hashlib

import numpy as np
import pytest

from oracle import refh
from oracle.port import Oracle
from paper_2207_12116_b200 import (Kind, Model, ModelError, Operand, and_c, iff_c, leq, leq_offset, linear_leq, lt,
                                   not_c, precedes)


def digest(t):
    h = hashlib.sha256()
    for a in (np.asarray(t.slot_kind, np.uint8), np.asarray(t.slot_word, np.uint32), np.asarray(t.cmd_off, np.uint32),
              np.asarray(t.cmd_code, np.int32), np.asarray(t.cands, np.int32)):
        h.update(a.tobytes())
    h.update(np.int32(t.n_words).tobytes())
    h.update(np.int32(t.obj_slot).tobytes())
    return h.hexdigest()


def build(name):
    if name.startswith("nqueens"):
        return Model.nqueens(int(name[7:]))
    if name == "csp1":
        return Model.random_csp(1)
    if name.startswith("csp_small"):
        return Model.random_csp(int(name[9:]), n_vars=60, n_cons=200)
    if name.startswith("rcpsp30_s"):
        return Model.rcpsp_random(int(name[9:]), 30, 4)
    if name.startswith("rcpsp10_s"):
        return Model.rcpsp_random(int(name[9:]), 10, 2)
    if name.startswith("rcpsp120_s"):
        return Model.rcpsp_random(int(name[10:]), 120, 4)
    return None


def test_tables_identical_to_reference(golden):
    n = 0
    for name, g in golden.items():
        m = build(name)
        if m is None:
            continue
        t = m.tables()
        assert (t.n_slots, t.n_words, t.n_cmds) == (g["n_slots"], g["n_words"], g["n_cmds"]), name
        assert digest(t) == g["tables_sha256"], name
        n += 1
    assert n >= 30


def test_survey_config_sizes():
    """SURVEY 8(a) sizes: Q8 16 words / 344 cmds ... RCPSP120 30,500 / 219,276."""
    for m, words, cmds in ((Model.nqueens(8), 16, 344), (Model.nqueens(14), 28, 1106),
                           (Model.random_csp(1), 1090, 4567), (Model.rcpsp_random(1, 30, 4), 2240, 14340)):
        t = m.tables()
        assert (t.n_words, t.n_cmds) == (words, cmds)


def xy(x0, x1, y0, y1, c=5):
    m = Model()
    x, y = m.add_cell(Kind.Interval), m.add_cell(Kind.Interval)
    m.tell(x, x0, x1)
    m.tell(y, y0, y1)
    m.post(linear_leq([(1, x), (1, y)], c))
    return m, x, y


def fix(m):
    o = Oracle(m.tables())
    return o.run_sequential(o.bottom())


def interval(words, m, s):
    w = m.tables().slot_word[s]
    return int(words[w]), int(words[w + 1])


def test_x_plus_y_leq_5():
    m, x, y = xy(0, 10, 0, 10)  # test_engine.cpp:48-55
    f, w, _, _ = fix(m)
    assert not f and interval(w, m, x) == (0, 5) and interval(w, m, y) == (0, 5)
    m, x, y = xy(4, 10, 3, 10)  # test_engine.cpp:57-62
    f, w, _, _ = fix(m)
    assert f


def test_sum_rule_zeroes_overloaded_boolean():
    """test_propagation.cpp:40-58: 2b1 + 2b2 <= 3, b2 = 1 => lsum = 2, b1 = 0."""
    m = Model()
    b1, b2 = m.add_cell(), m.add_cell()
    m.post(linear_leq([(2, b1), (2, b2)], 3))
    t = m.tables()
    assert t.n_slots == 3 and t.slot_kind[2] == Kind.ZInc
    m.tell(b1, 0, 1)
    m.tell(b2, 1, 1)
    f, w, _, _ = fix(m)
    assert not f
    assert w[t.slot_word[2]] == 2
    assert interval(w, m, b1) == (0, 0) and interval(w, m, b2) == (1, 1)


@pytest.mark.parametrize("case", ["entailed", "activated", "negated"])
def test_reification(case):
    """test_propagation.cpp:104-130."""
    m = Model()
    x, y, b = m.add_cell(), m.add_cell(), m.add_cell()
    m.post_reified(b, leq(Operand.v(x), Operand.v(y)))
    if case == "entailed":
        m.tell(x, 0, 2)
        m.tell(y, 5, 9)
        m.tell(b, 0, 1)
    else:
        m.tell(x, 0, 9)
        m.tell(y, 0, 9)
        m.tell(b, *((1, 1) if case == "activated" else (0, 0)))
    f, w, _, _ = fix(m)
    assert not f
    if case == "entailed":
        assert interval(w, m, b) == (1, 1)
    elif case == "activated":
        assert interval(w, m, x) == (0, 9) and interval(w, m, y) == (0, 9)
    else:
        assert interval(w, m, y) == (0, 8) and interval(w, m, x) == (1, 9)


def test_compile_errors_and_rollback():
    """test_propagation.cpp:132-146: sums cannot be negated; constants; coefficients."""
    m = Model()
    b, v = m.add_cell(), m.add_cell()
    n = m.tables().n_slots
    with pytest.raises(ModelError):
        m.post(not_c(linear_leq([(2, v)], 3)))
    with pytest.raises(ModelError):
        m.post_reified(b, linear_leq([(2, v)], 3))
    with pytest.raises(ModelError):
        m.post(leq(Operand.c(1), Operand.c(2)))
    with pytest.raises(ModelError):
        linear_leq([(-1, 0)], 3)
    with pytest.raises(ModelError):
        m.post(iff_c(leq(Operand.v(b), Operand.v(v)), linear_leq([(1, v), (2, b)], 4)))
    with pytest.raises(ModelError):
        m.post(leq(Operand.v(99), Operand.v(v)))
    assert m.tables().n_slots == n  # failed compiles leave no lsum cells behind


def test_two_task_chain_optimum():
    """test_solver.cpp:70-79 / test_cli.cpp:56-65: makespan 5."""
    m = Model.rcpsp([0, 2, 3, 0], [[0], [1], [1], [0]], [1], [(0, 1), (0, 2), (1, 2), (1, 3), (2, 3)], 5)
    o = Oracle(m.tables())
    r = o.solve_dfs(o.bottom())
    assert r["status"] == 0 and r["objective"] == 5
    assert m.check_solution(r["best_words"])
    bad = r["best_words"].copy()
    bad[m.tables().slot_word[m.starts()[2]]] = 0  # task 2 over task 1
    assert not m.check_solution(bad)


def test_rcpsp_instances_and_errors():
    # test_rcpsp.cpp:99-110: root propagation fixes the diagonal overlaps
    toy = "3 1\n1\n0 0 1 2\n4 1 1 3\n0 0 0\n"
    m = Model.rcpsp_patterson(toy)
    o = Oracle(m.tables())
    f, w, _, _ = o.run_sequential(o.bottom())
    assert not f
    assert m.tables().obj_slot == m.starts()[-1]
    with pytest.raises(ModelError):
        Model.rcpsp_patterson("2 0\n\n1 1 2\n1 1 1\n")  # cyclic
    with pytest.raises(ModelError):
        Model.rcpsp_patterson("3 1\n1\n0 0 1 2\n")  # truncated
    empty = Model.rcpsp([], [], [], [], 0)  # the degenerate instance: makespan 0
    o = Oracle(empty.tables())
    assert o.solve_dfs(o.bottom())["objective"] == 0


def test_not_and_and_iff_shapes():
    m = Model()
    a, b = m.add_cell(), m.add_cell()
    m.tell(a, 0, 3)
    m.tell(b, 0, 3)
    m.post(not_c(and_c(leq_offset(Operand.v(a), 0, Operand.v(b)), leq_offset(Operand.v(b), 0, Operand.v(a)))))
    m.post(iff_c(lt(Operand.v(a), Operand.c(2)), precedes(Operand.v(b), 1, Operand.c(3))))
    # 2 tells + not(and): 2 asks x 2 tells + iff: 4 asks x 1 tell (propagation.cpp:350-373)
    assert m.tables().n_cmds == 10
    f, w, _, _ = fix(m)
    assert not f
    m.tell(a, 1, 1)
    f, w, _, _ = fix(m)
    # a=1 < 2 entails the left side, so b+1 <= 3; b != a cannot cut the middle of [0,2]
    assert not f and interval(w, m, b) == (0, 2)
    m.tell(a, 0, 0)  # now a = 0 and 1 together: failure
    assert fix(m)[0]
