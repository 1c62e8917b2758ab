/* pccp_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference propagate-and-search path,
 * operating on the flat command tables of include/pccp_gpu.h.  It is the
 * checker for the CUDA path (tests/, __graft_entry__.smoke) and the "port"
 * CPU baseline in bench.py; the product never links it.  Each function cites
 * the reference code it restates (paths relative to /root/reference/proj).
 *
 * Parity is pinned: tests/test_oracle.py checks this restatement against the
 * reference library itself (oracle/_ref, built from the reference sources by
 * oracle/Makefile) and against the committed goldens in tests/golden/.
 */
#include "pccp_oracle.h"

#include <stdlib.h>
#include <string.h>

#define WIDE_INF ((int64_t)1 << 40) /* kWideInf, command.cpp:9 / lattice.cpp:10 */

/* term_value, command.cpp:11-19: coef 0 contributes nothing even on a
 * sentinel; sentinels widen to +-2^40 with the coefficient's sign; finite
 * products clamp to +-2^40. */
static int64_t term_value(int32_t coef, int32_t v) {
  if (coef == 0) return 0;
  if (v == INT32_MAX) return coef > 0 ? WIDE_INF : -WIDE_INF;
  if (v == INT32_MIN) return coef > 0 ? -WIDE_INF : WIDE_INF;
  int64_t p = (int64_t)coef * (int64_t)v;
  if (p > WIDE_INF) p = WIDE_INF;
  if (p < -WIDE_INF) p = -WIDE_INF;
  return p;
}

/* LinExpr::eval, command.cpp:21-27: int64 accumulation, narrow to sentinels. */
int32_t orc_lin_eval(const int32_t* e, const int32_t* words) {
  int64_t acc = e[0];
  const int32_t n = e[1];
  for (int32_t i = 0; i < n; ++i) acc += term_value(e[2 + 2 * i], words[e[3 + 2 * i]]);
  if (acc >= INT32_MAX) return INT32_MAX;
  if (acc <= INT32_MIN) return INT32_MIN;
  return (int32_t)acc;
}

static int expr_len(const int32_t* e) { return 2 + 2 * e[1]; }

/* scalar_top, lattice.hpp:53-61 */
static int32_t scalar_top(int kind) {
  switch (kind) {
    case PCCP_ZINC: return INT32_MAX;
    case PCCP_ZDEC: return INT32_MIN;
    case PCCP_BINC: return 1;
    case PCCP_BDEC: return 0;
    default: return 0;
  }
}

/* kind_is_up, lattice.hpp:35; the Interval lb word is up, ub word down (store.cpp:12-14). */
static int word_is_up(const pccp_model* m, uint32_t w, const uint8_t* up) {
  (void)m;
  return up[w];
}

static uint8_t* make_word_up(const pccp_model* m) {
  uint8_t* up = (uint8_t*)calloc(m->n_words ? m->n_words : 1, 1);
  for (uint32_t s = 0; s < m->n_slots; ++s) {
    const uint32_t w = m->slot_word[s];
    if (m->slot_kind[s] == PCCP_INTERVAL) {
      up[w] = 1;
      up[w + 1] = 0;
    } else {
      up[w] = (m->slot_kind[s] == PCCP_ZINC || m->slot_kind[s] == PCCP_BINC);
    }
  }
  return up;
}

/* Store::join_word, store.hpp:90-98: max on up words, min on down words;
 * true iff the word strictly increased in its lattice. */
static int join_word(int32_t* words, uint32_t w, int32_t v, int up) {
  if (up ? v > words[w] : v < words[w]) {
    words[w] = v;
    return 1;
  }
  return 0;
}

/* Store::is_failed, store.cpp:65-75 */
int orc_is_failed(const pccp_model* m, const int32_t* words) {
  for (uint32_t s = 0; s < m->n_slots; ++s) {
    const uint32_t w = m->slot_word[s];
    if (m->slot_kind[s] == PCCP_INTERVAL) {
      if (words[w] > words[w + 1]) return 1;
    } else if (words[w] == scalar_top(m->slot_kind[s])) {
      return 1;
    }
  }
  return 0;
}

/* GuardedCommand::guards_hold + Pred::eval, command.cpp:29-33,93-98. */
static int guards_hold(const int32_t* c, const int32_t* words, const int32_t** fn_out) {
  const int32_t ng = c[0];
  const int32_t* p = c + 5;
  int ok = 1;
  for (int32_t g = 0; g < ng; ++g) {
    const int32_t rel = p[0], rhs = p[1];
    if (ok) {
      const int32_t v = orc_lin_eval(p + 2, words);
      ok = rel == PCCP_LEQ ? v <= rhs : v > rhs;
    }
    p += 2 + expr_len(p + 2);
  }
  *fn_out = p;
  return ok;
}

/* GuardedCommand::apply fast paths, command.cpp:100-113.  Returns the bx
 * change flag, or -1 for a scalar tell without a scalar expression
 * (MonotoneFn::eval throws ModelError, command.cpp:63). */
static int apply_fn(const int32_t* c, const int32_t* fn, int32_t* words, const uint8_t* up,
                    const pccp_model* m) {
  const int32_t kind = c[2], mask = c[4];
  const uint32_t tw = (uint32_t)c[3];
  const int32_t* e = fn;
  const int32_t *sc = 0, *lb = 0, *ub = 0;
  if (mask & PCCP_FN_SCALAR) { sc = e; e += expr_len(e); }
  if (mask & PCCP_FN_LB) { lb = e; e += expr_len(e); }
  if (mask & PCCP_FN_UB) { ub = e; e += expr_len(e); }
  if (kind == PCCP_INTERVAL) {
    int changed = 0;
    if (lb) changed |= join_word(words, tw, orc_lin_eval(lb, words), 1);
    if (ub) changed |= join_word(words, tw + 1, orc_lin_eval(ub, words), 0);
    return changed;
  }
  if (!sc) return -1;
  return join_word(words, tw, orc_lin_eval(sc, words), word_is_up(m, tw, up));
}

static int run_seq(const pccp_model* m, const uint8_t* up, int32_t* words, uint64_t* iterations,
                   uint64_t* applications) {
  uint64_t it = 0, apps = 0;
  int changed = 1;
  while (changed) { /* engine.cpp:17-31 */
    changed = 0;
    ++it;
    for (uint32_t i = 0; i < m->n_cmds; ++i) {
      const int32_t* c = m->cmd_code + m->cmd_off[i];
      const int32_t* fn;
      if (!guards_hold(c, words, &fn)) continue;
      ++apps;
      const int r = apply_fn(c, fn, words, up, m);
      if (r < 0) return -1;
      changed |= r;
    }
    if (orc_is_failed(m, words)) {
      if (iterations) *iterations = it;
      if (applications) *applications = apps;
      return 1;
    }
  }
  if (iterations) *iterations = it;
  if (applications) *applications = apps;
  return 0;
}

int orc_run_sequential(const pccp_model* m, int32_t* words, uint64_t* iterations,
                       uint64_t* applications) {
  uint8_t* up = make_word_up(m);
  const int r = run_seq(m, up, words, iterations, applications);
  free(up);
  return r;
}

/* branch, solver.cpp:19-47: narrowest unfixed candidate (Interval, lo < hi),
 * first in candidate order on ties; mid = floor((lo+hi)/2) in int64. */
int orc_branch(const pccp_model* m, const int32_t* words, int32_t* var, int32_t* mid) {
  int32_t best = -1;
  int64_t best_w = 0;
  const uint32_t n = m->n_cands ? m->n_cands : m->n_slots;
  for (uint32_t k = 0; k < n; ++k) {
    const int32_t s = m->n_cands ? m->cands[k] : (int32_t)k;
    if (m->slot_kind[s] != PCCP_INTERVAL) continue;
    const int32_t lo = words[m->slot_word[s]], hi = words[m->slot_word[s] + 1];
    if (lo >= hi) continue;
    const int64_t width = (int64_t)hi - (int64_t)lo + 1;
    if (best < 0 || width < best_w) {
      best = s;
      best_w = width;
    }
  }
  if (best < 0) return 0;
  const int32_t lo = words[m->slot_word[best]], hi = words[m->slot_word[best] + 1];
  if (lo == INT32_MIN || hi == INT32_MAX) return -1; /* ModelError: unbounded */
  *var = best;
  *mid = (int32_t)(((int64_t)lo + (int64_t)hi) >> 1);
  return 1;
}

/* Decision::as_join + Store::join_in_place on an Interval, solver.hpp:20-23, store.cpp:51-63 */
static void join_decision(const pccp_model* m, int32_t* words, int32_t var, int32_t upper,
                          int32_t mid) {
  const uint32_t w = m->slot_word[var];
  if (upper) join_word(words, w, mid + 1, 1);
  else join_word(words, w + 1, mid, 0);
}

static int materialise(const pccp_model* m, const uint8_t* up, const int32_t* root, int n_dec,
                       const int32_t* dec, int32_t best, int32_t* out, uint64_t* sweeps) {
  memcpy(out, root, sizeof(int32_t) * m->n_words); /* Store::copy_from, store.cpp:84-92 */
  for (int i = 0; i < n_dec; ++i) join_decision(m, out, dec[3 * i], dec[3 * i + 1], dec[3 * i + 2]);
  if (best != INT32_MAX && m->obj_slot >= 0) /* solver.cpp:96-99 */
    join_word(out, m->slot_word[m->obj_slot] + 1, best - 1, 0);
  uint64_t it = 0;
  const int r = run_seq(m, up, out, &it, 0);
  if (sweeps) *sweeps += it;
  return r;
}

int orc_replay(const pccp_model* m, const int32_t* root, int n_dec, const int32_t* dec, int32_t best,
               int32_t* out) {
  uint8_t* up = make_word_up(m);
  const int r = materialise(m, up, root, n_dec, dec, best, out, 0);
  free(up);
  return r;
}

uint64_t orc_store_hash(uint32_t n_words, const int32_t* words) {
  uint64_t h = 1469598103934665603ull;
  for (uint32_t i = 0; i < n_words; ++i) {
    const uint32_t v = (uint32_t)words[i];
    for (int b = 0; b < 4; ++b) {
      h ^= (v >> (8 * b)) & 0xffu;
      h *= 1099511628211ull;
    }
  }
  return h;
}

/* ---- explicit DFS stack of decision paths (SearchNode, solver.hpp:28-30) ---- */
typedef struct {
  int32_t* dec; /* triples */
  int n;
} path_t;

typedef struct {
  path_t* v;
  size_t n, cap;
} pstack_t;

static void ps_push(pstack_t* s, const int32_t* dec, int n, const int32_t* extra) {
  if (s->n == s->cap) {
    s->cap = s->cap ? 2 * s->cap : 64;
    s->v = (path_t*)realloc(s->v, s->cap * sizeof(path_t));
  }
  path_t p;
  p.n = n + (extra ? 1 : 0);
  p.dec = (int32_t*)malloc(sizeof(int32_t) * 3 * (size_t)(p.n ? p.n : 1));
  if (n) memcpy(p.dec, dec, sizeof(int32_t) * 3 * (size_t)n);
  if (extra) memcpy(p.dec + 3 * n, extra, sizeof(int32_t) * 3);
  s->v[s->n++] = p;
}

static void ps_free(pstack_t* s) {
  for (size_t i = 0; i < s->n; ++i) free(s->v[i].dec);
  free(s->v);
}

/* Enumeration over dfs() order (solver.cpp:122-146): pop, materialise
 * (full recomputation from the root, solver.cpp:91-102), then push right
 * before left so the left branch (x <= mid) is explored first. */
int orc_enumerate(const pccp_model* m, const int32_t* root, int depth_cap, uint64_t node_budget,
                  uint64_t* out) {
  uint8_t* up = make_word_up(m);
  int32_t* cur = (int32_t*)malloc(sizeof(int32_t) * (m->n_words ? m->n_words : 1));
  uint64_t nodes = 0, fails = 0, sols = 0, open = 0, hash = 0, sweeps = 0;
  int exhausted = 1, err = 0;
  if (node_budget == 0) node_budget = UINT64_MAX;
  pstack_t st = {0, 0, 0};
  ps_push(&st, 0, 0, 0);
  while (st.n) {
    if (nodes >= node_budget) {
      exhausted = 0;
      break;
    }
    path_t p = st.v[--st.n];
    ++nodes;
    const int r = materialise(m, up, root, p.n, p.dec, INT32_MAX, cur, &sweeps);
    if (r < 0) { err = 1; free(p.dec); break; }
    if (r == 1) {
      ++fails;
      free(p.dec);
      continue;
    }
    hash += orc_store_hash(m->n_words, cur);
    int32_t var, mid;
    const int b = orc_branch(m, cur, &var, &mid);
    if (b < 0) { err = 1; free(p.dec); break; }
    if (b == 0) {
      ++sols;
    } else if (depth_cap >= 0 && p.n >= depth_cap) {
      ++open;
    } else {
      const int32_t right[3] = {var, 1, mid}, left[3] = {var, 0, mid};
      ps_push(&st, p.dec, p.n, right);
      ps_push(&st, p.dec, p.n, left);
    }
    free(p.dec);
  }
  ps_free(&st);
  free(cur);
  free(up);
  out[0] = nodes; out[1] = fails; out[2] = sols; out[3] = open;
  out[4] = hash; out[5] = sweeps; out[6] = (uint64_t)exhausted;
  return err ? -1 : 0;
}

/* solve_dfs + dfs + record_solution + finish, solver.cpp:104-173. */
int orc_solve_dfs(const pccp_model* m, const int32_t* root, uint64_t node_limit, int32_t* out,
                  uint64_t* st_out, int32_t* best_words) {
  uint8_t* up = make_word_up(m);
  int32_t* cur = (int32_t*)malloc(sizeof(int32_t) * (m->n_words ? m->n_words : 1));
  uint64_t nodes = 0, sols = 0;
  int32_t best = INT32_MAX;
  int exhausted = 1, err = 0;
  pstack_t st = {0, 0, 0};
  ps_push(&st, 0, 0, 0);
  while (st.n) {
    if (nodes >= node_limit) { /* SharedControl::should_stop, solver.cpp:68-76 */
      exhausted = 0;
      break;
    }
    path_t p = st.v[--st.n];
    ++nodes;
    const int r = materialise(m, up, root, p.n, p.dec, best, cur, 0);
    if (r < 0) { err = 1; free(p.dec); break; }
    if (r == 1) { free(p.dec); continue; }
    int32_t var, mid;
    const int b = orc_branch(m, cur, &var, &mid);
    if (b < 0) { err = 1; free(p.dec); break; }
    if (b == 0) {
      const int32_t value = cur[m->slot_word[m->obj_slot]]; /* obj.lo, solver.cpp:106-107 */
      if (value < best) {                                   /* Objective::improve */
        best = value;
        ++sols;
        if (best_words) memcpy(best_words, cur, sizeof(int32_t) * m->n_words);
      }
    } else {
      const int32_t right[3] = {var, 1, mid}, left[3] = {var, 0, mid};
      ps_push(&st, p.dec, p.n, right);
      ps_push(&st, p.dec, p.n, left);
    }
    free(p.dec);
  }
  ps_free(&st);
  free(cur);
  free(up);
  const int has = best != INT32_MAX;
  out[0] = has ? (exhausted ? PCCP_OPTIMAL : PCCP_SAT) : (exhausted ? PCCP_UNSAT : PCCP_UNKNOWN);
  out[1] = has;
  out[2] = has ? best : 0;
  st_out[0] = nodes;
  st_out[1] = sols;
  return err ? -1 : 0;
}
