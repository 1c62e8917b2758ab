"""Ad-hoc exploration on the GPU box: per-config timings and launch plans.

    python scripts/explore.py q14 csp rcpsp30 rcpsp120 [--gt 32 --gpc 8 ...]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2207_12116_b200 import Engine, Model  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what", nargs="+")
    ap.add_argument("--gt", type=int, default=0)
    ap.add_argument("--gpc", type=int, default=0)
    ap.add_argument("--cps", type=int, default=0)
    ap.add_argument("--eps", type=int, default=0)
    ap.add_argument("--hash", action="store_true")
    ap.add_argument("--timeout", type=float, default=60)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--vo", type=int, default=-1, help="value order")
    ap.add_argument("--var", type=int, default=0, help="var order (1: smallest lb)")
    ap.add_argument("--primal", type=int, default=0, help="primal phase ms")
    a = ap.parse_args()
    eng = Engine(0, group_threads=a.gt, groups_per_cta=a.gpc, ctas_per_sm=a.cps, eps_factor=a.eps, hash=a.hash,
                 value_order=a.vo, var_order=a.var, primal_ms=a.primal)
    for w in a.what:
        if w.startswith("q"):
            m = Model.nqueens(int(w[1:]))
            eng.load(m)
            info = eng.lowering_info()
            for _ in range(a.reps):
                t = time.time()
                r = eng.enumerate()
                dt = time.time() - t
            print(w, json.dumps(info))
            print(w, f"nodes={r['nodes']} sols={r['solutions']} kernel={r['kernel_ms']:.2f}ms dec={r['decompose_ms']:.2f}ms "
                     f"levels={r['bfs_levels']} don={r['donations']} rounds={r['rounds']} wall={dt:.4f}s nodes/s={r['nodes'] / dt:.3e}")
        elif w.startswith("csp"):
            d = int(w[3:]) if len(w) > 3 else 22
            m = Model.random_csp(1)
            eng.load(m)
            info = eng.lowering_info()
            for _ in range(a.reps):
                t = time.time()
                r = eng.enumerate(depth_cap=d)
                dt = time.time() - t
            print(w, json.dumps(info))
            print(w, json.dumps(r), f"wall {dt:.4f}s nodes/s {r['nodes'] / dt:.3e}")
        elif w.startswith("rcpsp30") or w.startswith("rcpsp120"):
            n = 30 if w.startswith("rcpsp30") else 120
            seeds = [int(s) for s in w.split("_")[1:]] or [1]
            for s in seeds:
                m = Model.rcpsp_random(s, n, 4)
                eng.load(m)
                info = eng.lowering_info()
                t = time.time()
                r = eng.solve(timeout_s=a.timeout)
                dt = time.time() - t
                ok = m.check_solution(r.best_words) if r.best_words is not None else None
                st = r.stats
                last = r.improvements[-1][1] if r.improvements else None
                print(f"{w} seed={s} {r.status} obj={r.objective} valid={ok} nodes={st['nodes']} rounds={st['rounds']} "
                      f"wall={dt:.3f}s kernel={st['kernel_ms']:.1f}ms t_best={last} nodes/s={st['nodes'] / dt:.3e} "
                      f"evals/s={st['evals'] / dt:.3e} sub={st['subproblems']} cta={info['group_threads']}"
                      f" smem_table={info['table_in_smem']} levels={st['bfs_levels']} dec={st['decompose_ms']:.1f}ms don={st['donations']}"
                      f" primal={r.primal} impr={[(v, round(t, 1)) for v, t in r.improvements[:4]]}..{[(v, round(t, 1)) for v, t in r.improvements[-4:]]}")
        sys.stdout.flush()


if __name__ == "__main__":
    main()
