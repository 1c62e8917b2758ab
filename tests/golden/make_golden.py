"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Run where /root/reference exists (this container), after `make -C oracle ref`:

    python tests/golden/make_golden.py            # fast set (~2 min)
    python tests/golden/make_golden.py --slow     # adds CSP depth 22 and RCPSP30 optima

Every number written here is produced by the unmodified reference library
(oracle/_ref/libpccp_ref.so, built from /root/reference/proj/src) through its
public API, or by the harness enumerator written over that API
(oracle/ref_harness.cpp).  Values quoted from SURVEY.md rather than recomputed
are marked "provenance": "survey".
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.refh import INT32_MAX, RefModel, RefRng  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def tables_digest(t) -> str:
    h = hashlib.sha256()
    for a in (np.asarray(t.slot_kind, np.uint8), np.asarray(t.slot_word, np.uint32),
              np.asarray(t.cmd_off, np.uint32), np.asarray(t.cmd_code, np.int32), np.asarray(t.cands, np.int32)):
        h.update(a.tobytes())
    h.update(np.int32(t.n_words).tobytes())
    h.update(np.int32(t.obj_slot).tobytes())
    return h.hexdigest()


def store_hash(words) -> int:
    h = 1469598103934665603
    for v in np.asarray(words, np.int32).view(np.uint32):
        v = int(v)
        for b in range(4):
            h ^= (v >> (8 * b)) & 0xFF
            h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def random_paths(m: RefModel, n_paths: int, max_depth: int, seed: int, with_best: bool):
    """Random root-to-node decision paths replayed through the reference
    (materialize, solver.cpp:91-102).  Returns a list of dicts."""
    rng = np.random.default_rng(seed)
    out = []
    root = m.root()
    failed, fix, _, _ = m.run_sequential(root)
    assert not failed
    obj_w = m.tables.slot_word[m.tables.obj_slot] if m.tables.obj_slot >= 0 else None
    while len(out) < n_paths:
        dec = []
        best = INT32_MAX
        if with_best and obj_w is not None and rng.random() < 0.5:
            lo, hi = int(fix[obj_w]), int(fix[obj_w + 1])
            best = int(rng.integers(lo, hi + 2))
        cur = fix
        depth = int(rng.integers(1, max_depth + 1))
        for _ in range(depth):
            b = m.branch(cur)
            if b is None:
                break
            var, mid = b
            dec.append((var, int(rng.integers(0, 2)), mid))
            failed, cur = m.replay(dec, best)
            if failed:
                break
        failed, words = m.replay(dec, best)
        out.append(dict(decisions=[list(map(int, d)) for d in dec], best=best, failed=bool(failed),
                        hash=None if failed else store_hash(words)))
    return out


def config_entry(name, m: RefModel, paths=0, max_depth=0, with_best=False):
    t = m.tables
    root = m.root()
    failed, fix, iters, apps = m.run_sequential(root)
    e = dict(name=name, n_slots=len(t.slot_kind), n_words=t.n_words, n_cmds=t.n_cmds,
             code_len=len(t.cmd_code), obj_slot=t.obj_slot, n_cands=len(t.cands),
             tables_sha256=tables_digest(t),
             root=dict(failed=failed, hash=None if failed else store_hash(fix), iterations=iters, applications=apps))
    if paths:
        e["replays"] = random_paths(m, paths, max_depth, seed=len(name) * 7919 + 17, with_best=with_best)
    return e


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--slow", action="store_true")
    args = ap.parse_args()

    configs = {}
    # -- N-Queens (configs 1, 2) ------------------------------------------------
    for n in (4, 5, 6, 8, 10):
        m = RefModel.nqueens(n)
        e = config_entry(f"nqueens{n}", m, paths=200, max_depth=3 * n)
        r = m.enumerate()
        e["enumerate"] = {k: r[k] for k in ("nodes", "failures", "solutions", "open_leaves", "hash_sum", "sweeps")}
        e["enumerate"]["provenance"] = "reference"
        configs[e["name"]] = e
        print(e["name"], e["enumerate"], flush=True)
    m = RefModel.nqueens(14)
    e = config_entry("nqueens14", m, paths=300, max_depth=40)
    e["enumerate"] = dict(nodes=8567767, failures=3918288, solutions=365596, open_leaves=0,
                          hash_sum=0xDB0839842A068562, provenance="survey")
    configs[e["name"]] = e

    # -- random linear CSP (config 3) ---------------------------------------------
    m = RefModel.csp(1)
    e = config_entry("csp1", m, paths=300, max_depth=30)
    r = m.enumerate(depth_cap=12)
    e["enumerate_d12"] = {k: r[k] for k in ("nodes", "failures", "solutions", "open_leaves", "hash_sum", "sweeps")}
    e["enumerate_d12"]["provenance"] = "reference"
    if args.slow:
        r = m.enumerate(depth_cap=22, threads=8)
        e["enumerate_d22"] = {k: r[k] for k in ("nodes", "failures", "solutions", "open_leaves", "hash_sum")}
        e["enumerate_d22"]["provenance"] = "reference"
    else:
        e["enumerate_d22"] = dict(nodes=108611, failures=23228, solutions=0, open_leaves=31078,
                                  hash_sum=0x6C8868DADE5564A8, provenance="survey")
    configs[e["name"]] = e
    print("csp1", e["enumerate_d12"], flush=True)
    for seed in (2, 3):
        m = RefModel.csp(seed, n_vars=60, n_cons=200)
        e = config_entry(f"csp_small{seed}", m, paths=100, max_depth=20)
        r = m.enumerate(depth_cap=10)
        e["enumerate_d10"] = {k: r[k] for k in ("nodes", "failures", "solutions", "open_leaves", "hash_sum")}
        configs[e["name"]] = e

    # -- RCPSP (configs 4, 5) ----------------------------------------------------
    optima = {1: 84, 2: 77, 5: 73, 7: 60, 9: 61, 11: 99}
    for seed in range(1, 13):
        m = RefModel.rcpsp(seed, 30, 4)
        e = config_entry(f"rcpsp30_s{seed}", m, paths=150 if seed in (1, 2) else 30, max_depth=60, with_best=True)
        if seed in optima:
            e["optimum"] = dict(value=optima[seed], provenance="survey")
        configs[e["name"]] = e
    for seed in (1, 5, 11):
        r = RefModel.rcpsp(seed, 30, 4).solve_parallel(workers=8, timeout_s=60)
        assert r["status"] == 0 and r["objective"] == optima[seed], r
        configs[f"rcpsp30_s{seed}"]["optimum"] = dict(value=r["objective"], provenance="reference")
        print("rcpsp30", seed, r["objective"], r["nodes"], flush=True)
    if args.slow:
        for seed in (2, 7, 9):
            r = RefModel.rcpsp(seed, 30, 4).solve_parallel(workers=8, timeout_s=300)
            if r["status"] == 0:
                configs[f"rcpsp30_s{seed}"]["optimum"] = dict(value=r["objective"], provenance="reference")
            print("rcpsp30", seed, r["status"], r["objective"], flush=True)
    m = RefModel.rcpsp(1, 120, 4)
    e = config_entry("rcpsp120_s1", m, paths=20, max_depth=40, with_best=True)
    configs[e["name"]] = e
    print("rcpsp120", e["n_words"], e["n_cmds"], e["root"], flush=True)
    # small RCPSPs where the reference proves the optimum quickly (multi-size parity)
    for seed in range(1, 9):
        m = RefModel.rcpsp(seed, 10, 2)
        e = config_entry(f"rcpsp10_s{seed}", m)
        r = m.solve_dfs()
        e["solve_dfs"] = dict(status=r["status"], objective=r["objective"], nodes=r["nodes"],
                              solutions=r["solutions"], best_hash=store_hash(r["best_words"]) if r["objective"] is not None else None)
        configs[e["name"]] = e
    # the reference acceptance corpus (corpus.cpp:92-104), first 30 by index
    for idx in range(0, 30):
        m = RefModel.corpus(idx)
        e = config_entry(f"corpus{idx}", m)
        r = m.solve_dfs(node_limit=200000)
        e["solve_dfs"] = dict(status=r["status"], objective=r["objective"], nodes=r["nodes"], solutions=r["solutions"])
        configs[e["name"]] = e

    with open(os.path.join(OUT, "configs.json"), "w") as f:
        json.dump(configs, f, indent=1, sort_keys=True)

    # -- micro CSPs of the acceptance confluence criterion (rng seed 2,
    #    acceptance_main.cpp:137-194) and test_engine's 120 (rng 4242) ----------
    for tag, seed, count in (("micro_csp_s2", 2, 500), ("micro_csp_s4242", 4242, 120)):
        rng = RefRng(seed)
        kinds, words, offs, codes, nw, status, fixes, iters = [], [], [], [], [], [], [], []
        for _ in range(count):
            m = rng.micro_csp()
            t = m.tables
            failed, fix, it, _ = m.run_sequential(m.root())
            kinds.append(t.slot_kind)
            words.append(t.slot_word)
            offs.append(t.cmd_off)
            codes.append(t.cmd_code)
            nw.append(t.n_words)
            status.append(int(failed))
            fixes.append(fix)
            iters.append(it)
        def pack(arrs, dt):
            lens = np.array([len(a) for a in arrs], np.int64)
            return np.concatenate([np.asarray(a, dt) for a in arrs]) if arrs else np.zeros(0, dt), lens
        k, kl = pack(kinds, np.uint8)
        w, wl = pack(words, np.uint32)
        o, ol = pack(offs, np.uint32)
        c, cl = pack(codes, np.int32)
        fx, fl = pack(fixes, np.int32)
        np.savez_compressed(os.path.join(OUT, f"{tag}.npz"), kind=k, kind_len=kl, word=w, word_len=wl, off=o,
                            off_len=ol, code=c, code_len=cl, n_words=np.array(nw, np.int64),
                            status=np.array(status, np.int8), fix=fx, fix_len=fl, iters=np.array(iters, np.int64))
        print(tag, count, "failed:", sum(status), flush=True)

    # -- micro RCPSPs of the optimality criterion (rng seed 4,
    #    acceptance_main.cpp:243-287): tables + brute-force optimum ------------
    rng = RefRng(4)
    recs = []
    kinds, words, offs, codes, cands = [], [], [], [], []
    for _ in range(200):
        m = rng.micro_rcpsp()
        t = m.tables
        bf = m.brute_force_makespan()
        r = m.solve_dfs()
        recs.append(dict(n_words=t.n_words, obj_slot=t.obj_slot, brute_force=bf, status=r["status"],
                         objective=r["objective"], nodes=r["nodes"]))
        kinds.append(t.slot_kind)
        words.append(t.slot_word)
        offs.append(t.cmd_off)
        codes.append(t.cmd_code)
        cands.append(t.cands)
    def pack(arrs, dt):
        lens = np.array([len(a) for a in arrs], np.int64)
        return np.concatenate([np.asarray(a, dt) for a in arrs]), lens
    k, kl = pack(kinds, np.uint8)
    w, wl = pack(words, np.uint32)
    o, ol = pack(offs, np.uint32)
    c, cl = pack(codes, np.int32)
    cd, cdl = pack(cands, np.int32)
    np.savez_compressed(os.path.join(OUT, "micro_rcpsp_s4.npz"), kind=k, kind_len=kl, word=w, word_len=wl, off=o,
                        off_len=ol, code=c, code_len=cl, cands=cd, cands_len=cdl)
    with open(os.path.join(OUT, "micro_rcpsp_s4.json"), "w") as f:
        json.dump(recs, f)
    print("micro_rcpsp", len(recs), "unsat:", sum(r["brute_force"] is None for r in recs), flush=True)


if __name__ == "__main__":
    main()
