"""The ownership rules of the barrier-free EPS compaction (search.cuh
small_compact / expand_level), restated on the host: every index entry a group
reads in the next level must have been written by that group's own CTA, since
small levels have no grid barrier between the compaction and the next
expansion.  Pure integer arithmetic, no GPU."""
import random


def reads(G, per_cta, n_par):
    """expand_level: parent p -> the CTAs whose groups read idx[p]."""
    ng = G * per_cta
    out = {}
    if 2 * n_par <= ng:  # split level: children 2p and 2p+1 on their own groups
        for j in range(2 * n_par):
            out.setdefault(j >> 1, set()).add((j % ng) // per_cta)
    else:
        for p in range(n_par):
            out.setdefault(p, set()).add((p % ng) // per_cta)
    return out


def writes(G, per_cta, total, B):
    """small_compact on CTA B: the positions it writes, by the device formulas."""
    got = set()
    if 2 * total <= G * per_cta:
        plo, phi = (B * per_cta) >> 1, ((B + 1) * per_cta - 1) >> 1
        got = {p for p in range(total) if plo <= p <= phi}
    else:
        # windows [ws, ws + per_cta), q = p // per_cta = B + m G, walked from
        # any thread's first position p0 (here every p0 in turn)
        for p0 in range(total):
            q = p0 // per_cta
            r = (B - q) % G
            ws = (q + r) * per_cta
            p = p0
            if p >= ws + per_cta:
                ws += G * per_cta
            if p >= ws:
                got.add(p)
    return got


def test_every_read_entry_is_written_by_the_readers_cta():
    rng = random.Random(7)
    cases = [(888, 8), (296, 1), (148, 1), (5, 3), (7, 8), (1, 1), (2, 4)]
    cases += [(rng.randint(1, 40), rng.choice([1, 2, 3, 4, 8])) for _ in range(30)]
    for G, per_cta in cases:
        ng = G * per_cta
        for total in sorted({1, 2, ng // 2, ng // 2 + 1, ng, ng + 1, 3 * ng + 5, rng.randint(1, 4 * ng)}):
            if total < 1:
                continue
            need = reads(G, per_cta, total)
            # every CTA of small grids; a sample of the large ones (the union check needs all)
            bs = range(G) if G <= 64 else sorted(rng.sample(range(G), 12))
            have = {B: writes(G, per_cta, total, B) for B in bs}
            for p, ctas in need.items():
                for B in ctas:
                    if B in have:
                        assert p in have[B], (G, per_cta, total, p, B)
            if G <= 64:  # together the CTAs write every position (the search reads them all)
                assert set().union(*have.values()) == set(range(total)), (G, per_cta, total)


def test_window_walk_matches_the_modulo_rule():
    # the thread-local window walk in small_compact equals (p / per_cta) % G == B
    for G, per_cta in [(888, 8), (3, 2), (7, 1), (5, 5)]:
        ng = G * per_cta
        total = 3 * ng + 7
        for B in range(G):
            want = {p for p in range(total) if (p // per_cta) % G == B}
            got = set()
            for p0 in range(0, total, 13):  # a thread's run of consecutive positions
                q = p0 // per_cta
                r = (B - q) % G
                ws = (q + r) * per_cta
                for p in range(p0, min(total, p0 + 32)):
                    if p >= ws + per_cta:
                        ws += G * per_cta
                    if p >= ws:
                        got.add(p)
            assert got == {p for p in want if any(p0 <= p < p0 + 32 for p0 in range(0, total, 13))}
