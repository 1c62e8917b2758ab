// ref_harness.cpp — TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// A C-ABI harness over the *unmodified* reference library compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libpccp_ref.so.
// It exists to
//   (1) build the five benchmark configurations through the reference's own
//       model API and serialise them into the flat tables of
//       include/pccp_gpu.h (so the product's host builder can be checked
//       table-for-table against the reference),
//   (2) run the reference engine / solver on them (goldens, CPU baseline),
//   (3) host the all-solutions DFS enumerator the reference lacks, written
//       over the reference public API (branch, run_sequential, Store) in the
//       node order of dfs() (solver.cpp:122-146), as SURVEY 8(c) prescribes.
// Only tests/, bench.py's cpu_baseline / --impl reference arm and the golden
// generator load it.

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <deque>
#include <mutex>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "corpus.hpp"
#include "generators.hpp"
#include "pccp/engine.hpp"
#include "pccp/propagation.hpp"
#include "pccp/rcpsp.hpp"
#include "pccp/solver.hpp"

using namespace pccp;

namespace {

thread_local std::string g_err;

struct RefModel {
  std::shared_ptr<const Schema> schema;
  std::vector<GuardedCommand> props;
  std::vector<Slot> cands;
  Slot obj = -1;
  bool is_rcpsp = false;
  rcpsp::RcpspInstance inst;
  rcpsp::RcpspModel rmodel;
  // flat tables (include/pccp_gpu.h)
  std::vector<uint8_t> kind;
  std::vector<uint32_t> word;
  std::vector<uint32_t> off;
  std::vector<int32_t> code;
};

void put_expr(std::vector<int32_t>& code, const LinExpr& e) {
  code.push_back(e.k);
  code.push_back(static_cast<int32_t>(e.terms.size()));
  for (const Term& t : e.terms) {
    code.push_back(t.coef);
    code.push_back(static_cast<int32_t>(t.word));
  }
}

void serialise(RefModel& m) {
  const Schema& s = *m.schema;
  m.kind.clear();
  m.word.clear();
  for (Slot i = 0; i < s.slot_count(); ++i) {
    m.kind.push_back(static_cast<uint8_t>(s.kind(i)));
    m.word.push_back(s.first_word(i));
  }
  m.off.assign(1, 0);
  m.code.clear();
  for (const GuardedCommand& gc : m.props) {
    if (gc.fn.generic) throw ModelError("generic fn cannot be serialised");
    m.code.push_back(static_cast<int32_t>(gc.guards.size()));
    m.code.push_back(gc.target);
    m.code.push_back(static_cast<int32_t>(gc.target_kind));
    m.code.push_back(static_cast<int32_t>(gc.target_word));
    int mask = 0;
    if (gc.fn.scalar) mask |= 1;
    if (gc.fn.lb) mask |= 2;
    if (gc.fn.ub) mask |= 4;
    m.code.push_back(mask);
    for (const Pred& p : gc.guards) {
      if (p.generic) throw ModelError("generic pred cannot be serialised");
      m.code.push_back(p.rel == Pred::Rel::Leq ? 0 : 1);
      m.code.push_back(p.rhs);
      put_expr(m.code, p.lhs);
    }
    if (gc.fn.scalar) put_expr(m.code, *gc.fn.scalar);
    if (gc.fn.lb) put_expr(m.code, *gc.fn.lb);
    if (gc.fn.ub) put_expr(m.code, *gc.fn.ub);
    m.off.push_back(static_cast<uint32_t>(m.code.size()));
  }
}

RefModel* finish_model(RefModel* m) {
  try {
    serialise(*m);
  } catch (const std::exception& e) {
    g_err = e.what();
    delete m;
    return nullptr;
  }
  return m;
}

void append(std::vector<GuardedCommand>& props, Propagator p) {
  props.insert(props.end(), std::make_move_iterator(p.commands.begin()),
               std::make_move_iterator(p.commands.end()));
}

RefModel* from_rcpsp(const rcpsp::RcpspInstance& inst) {
  auto* m = new RefModel;
  m->is_rcpsp = true;
  m->inst = inst;
  m->rmodel = rcpsp::build_model(inst);
  m->schema = m->rmodel.schema;
  m->props = m->rmodel.props;
  m->cands = m->rmodel.search_vars;
  m->obj = m->rmodel.objective;
  return finish_model(m);
}

void load_words(Store& s, const int32_t* w) {
  if (!w) return;
  for (Word i = 0; i < s.schema().word_count(); ++i) s.store_word(i, w[i]);
}
void save_words(const Store& s, int32_t* w) {
  if (!w) return;
  for (Word i = 0; i < s.schema().word_count(); ++i) w[i] = s.load_word(i);
}

uint64_t store_hash(const Store& s) {
  uint64_t h = 1469598103934665603ull;
  for (Word i = 0; i < s.schema().word_count(); ++i) {
    const uint32_t v = static_cast<uint32_t>(s.load_word(i));
    for (int b = 0; b < 4; ++b) {
      h ^= (v >> (8 * b)) & 0xffu;
      h *= 1099511628211ull;
    }
  }
  return h;
}

using Clock = std::chrono::steady_clock;

struct EnumCounters {
  std::atomic<uint64_t> nodes{0}, failures{0}, solutions{0}, open{0}, hash{0}, sweeps{0};
  std::atomic<bool> stop{false};
};

enum class Kind3 { Failed, Solution, Open, Expand };

// materialize() of solver.cpp:91-102 without the objective: copy root, replay
// the decision path, run the sequential engine.
Kind3 materialise(const RefModel& m, const Store& root, Store& cur, const SearchNode& node,
                  int depth_cap, bool count, EnumCounters& c, const BranchStrategy& strat,
                  std::optional<std::pair<Decision, Decision>>* out_dec) {
  cur.copy_from(root);
  for (const Decision& d : node.decisions) cur.join_in_place(d.var, d.as_join());
  const EngineResult r = run_sequential(m.props, cur);
  if (count) {
    c.nodes.fetch_add(1, std::memory_order_relaxed);
    c.sweeps.fetch_add(r.iterations, std::memory_order_relaxed);
  }
  if (r.failed()) {
    if (count) c.failures.fetch_add(1, std::memory_order_relaxed);
    return Kind3::Failed;
  }
  if (count) c.hash.fetch_add(store_hash(cur), std::memory_order_relaxed);
  auto dec = branch(cur, strat);
  if (!dec) {
    if (count) c.solutions.fetch_add(1, std::memory_order_relaxed);
    return Kind3::Solution;
  }
  if (depth_cap >= 0 && static_cast<int>(node.decisions.size()) >= depth_cap) {
    if (count) c.open.fetch_add(1, std::memory_order_relaxed);
    return Kind3::Open;
  }
  if (out_dec) *out_dec = dec;
  return Kind3::Expand;
}

// dfs() order (solver.cpp:122-146): LIFO stack, left (x <= mid) popped first.
void dfs_enum(const RefModel& m, const Store& root, const SearchNode& start, bool count_start,
              int depth_cap, EnumCounters& c, const BranchStrategy& strat,
              Clock::time_point deadline, uint64_t node_budget) {
  Store cur(root.schema_ptr());
  std::vector<std::pair<SearchNode, bool>> stack;
  stack.push_back({start, count_start});
  while (!stack.empty()) {
    if (c.stop.load(std::memory_order_relaxed)) return;
    if (Clock::now() >= deadline || c.nodes.load(std::memory_order_relaxed) >= node_budget) {
      c.stop.store(true);
      return;
    }
    auto [node, cnt] = std::move(stack.back());
    stack.pop_back();
    std::optional<std::pair<Decision, Decision>> dec;
    if (materialise(m, root, cur, node, depth_cap, cnt, c, strat, &dec) != Kind3::Expand) continue;
    SearchNode right = node;
    right.decisions.push_back(dec->second);
    stack.push_back({std::move(right), true});
    node.decisions.push_back(dec->first);
    stack.push_back({std::move(node), true});
  }
}

}  // namespace

extern "C" {

const char* refh_last_error() { return g_err.c_str(); }

void refh_free(void* h) { delete static_cast<RefModel*>(h); }

// ---- model builders ------------------------------------------------------

// N-Queens as SURVEY 8(d) config 1/2: q_i != q_j + d as not(and(leq_offset,leq_offset)).
void* refh_model_nqueens(int n) {
  auto* m = new RefModel;
  SchemaBuilder sb;
  std::vector<Slot> q;
  for (int i = 0; i < n; ++i) q.push_back(sb.add_cell("q" + std::to_string(i), Kind::Interval));
  std::vector<Process> init;
  for (int i = 0; i < n; ++i) init.push_back(tell_const(q[i], LatticeValue::interval(0, n - 1)));
  m->props = gnf(par(std::move(init)), sb.peek());
  for (int i = 0; i < n; ++i) {
    for (int j = i + 1; j < n; ++j) {
      for (int d : {0, j - i, i - j}) {
        append(m->props, compile(not_c(and_c(leq_offset(Operand::v(q[i]), -d, Operand::v(q[j])),
                                             leq_offset(Operand::v(q[j]), d, Operand::v(q[i])))),
                                 sb));
      }
    }
  }
  m->schema = sb.share();
  finalize_all(m->props, *m->schema);
  return finish_model(m);
}

// Random linear CSP of SURVEY 8(d) config 3.  `variant` selects the order of
// the two draws per sum term (0: coefficient then variable, 1: the reverse).
void* refh_model_csp(uint64_t seed, int n_vars, int n_cons, int dom_hi, int variant) {
  auto* m = new RefModel;
  std::mt19937_64 rng(seed);
  auto pick = [&rng](int lo, int hi) { return std::uniform_int_distribution<int>(lo, hi)(rng); };
  SchemaBuilder sb;
  std::vector<Slot> x;
  for (int i = 0; i < n_vars; ++i) x.push_back(sb.add_cell("x" + std::to_string(i), Kind::Interval));
  std::vector<Process> init;
  for (int i = 0; i < n_vars; ++i) init.push_back(tell_const(x[i], LatticeValue::interval(0, dom_hi)));
  m->props = gnf(par(std::move(init)), sb.peek());
  for (int c = 0; c < n_cons; ++c) {
    if (std::uniform_real_distribution<double>(0.0, 1.0)(rng) < 0.3) {
      const int i = pick(0, n_vars - 2);
      const int j = pick(i + 1, n_vars - 1);
      const int d = pick(1, 2);
      append(m->props, compile(precedes(Operand::v(x[i]), d, Operand::v(x[j])), sb));
    } else {
      const int k = pick(2, 5);
      std::vector<std::pair<int32_t, Slot>> terms;
      int64_t sum_a = 0;
      for (int t = 0; t < k; ++t) {
        int a, v;
        if (variant == 0) {
          a = pick(1, 9);
          v = pick(0, n_vars - 1);
        } else {
          v = pick(0, n_vars - 1);
          a = pick(1, 9);
        }
        terms.emplace_back(a, x[v]);
        sum_a += a;
      }
      const int32_t cap = static_cast<int32_t>(sum_a * dom_hi / 4);
      append(m->props, compile(linear_leq(std::move(terms), cap), sb));
    }
  }
  m->schema = sb.share();
  finalize_all(m->props, *m->schema);
  return finish_model(m);
}

void* refh_model_rcpsp(uint64_t seed, int n_real, int resources) {
  try {
    std::mt19937_64 rng(seed);
    return from_rcpsp(testsupport::random_patterson(rng, n_real, resources));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void* refh_model_corpus(int idx) {
  static const auto corpus = testsupport::corpus_instances();
  return from_rcpsp(corpus.at(static_cast<size_t>(idx)));
}

void* refh_model_patterson(const char* text) {
  try {
    return from_rcpsp(rcpsp::parse_patterson_text(text));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void* refh_rng_new(uint64_t seed) { return new std::mt19937_64(seed); }
void refh_rng_free(void* r) { delete static_cast<std::mt19937_64*>(r); }

// The reference's random_micro_csp (generators.cpp:15-96), drawn from `rng`.
void* refh_model_micro_csp(void* rng) {
  auto* m = new RefModel;
  testsupport::MicroCsp csp = testsupport::random_micro_csp(*static_cast<std::mt19937_64*>(rng));
  m->schema = csp.schema;
  m->props = std::move(csp.props);
  return finish_model(m);
}

// The reference's random_micro_rcpsp (generators.cpp:280-322).
void* refh_model_micro_rcpsp(void* rng) {
  return from_rcpsp(testsupport::random_micro_rcpsp(*static_cast<std::mt19937_64*>(rng)));
}

// brute_force_makespan (generators.cpp:324-361); returns INT32_MIN if unsat.
int32_t refh_brute_force_makespan(void* h) {
  auto* m = static_cast<RefModel*>(h);
  auto r = testsupport::brute_force_makespan(m->inst);
  return r ? *r : INT32_MIN;
}

// ---- table access ----------------------------------------------------------

uint32_t refh_n_slots(void* h) { return static_cast<uint32_t>(static_cast<RefModel*>(h)->kind.size()); }
uint32_t refh_n_words(void* h) { return static_cast<RefModel*>(h)->schema->word_count(); }
uint32_t refh_n_cmds(void* h) { return static_cast<uint32_t>(static_cast<RefModel*>(h)->props.size()); }
uint32_t refh_code_len(void* h) { return static_cast<uint32_t>(static_cast<RefModel*>(h)->code.size()); }
uint32_t refh_n_cands(void* h) { return static_cast<uint32_t>(static_cast<RefModel*>(h)->cands.size()); }
int32_t refh_obj_slot(void* h) { return static_cast<RefModel*>(h)->obj; }

void refh_tables(void* h, uint8_t* kind, uint32_t* word, uint32_t* off, int32_t* code,
                 int32_t* cands) {
  auto* m = static_cast<RefModel*>(h);
  std::memcpy(kind, m->kind.data(), m->kind.size());
  std::memcpy(word, m->word.data(), m->word.size() * 4);
  std::memcpy(off, m->off.data(), m->off.size() * 4);
  std::memcpy(code, m->code.data(), m->code.size() * 4);
  for (size_t i = 0; i < m->cands.size(); ++i) cands[i] = m->cands[i];
}

// Bottom store (Store::reset, store.cpp:29-39).
void refh_root(void* h, int32_t* words) {
  auto* m = static_cast<RefModel*>(h);
  Store s(m->schema);
  save_words(s, words);
}

// ---- engine ----------------------------------------------------------------

// run_sequential (engine.cpp:13-32) on `in` (NULL: bottom store). Returns
// 1 if failed, 0 at a fixed point, -1 on error.
int refh_run_sequential(void* h, const int32_t* in, int32_t* out, uint64_t* iters,
                        uint64_t* apps) {
  auto* m = static_cast<RefModel*>(h);
  try {
    Store s(m->schema);
    load_words(s, in);
    const EngineResult r = run_sequential(m->props, s);
    save_words(s, out);
    if (iters) *iters = r.iterations;
    if (apps) *apps = r.applications;
    return r.failed() ? 1 : 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int refh_run_parallel(void* h, const int32_t* in, int32_t* out, unsigned workers,
                      uint64_t* iters) {
  auto* m = static_cast<RefModel*>(h);
  try {
    Store s(m->schema);
    load_words(s, in);
    const EngineResult r = run_parallel(m->props, s, workers);
    save_words(s, out);
    if (iters) *iters = r.iterations;
    return r.failed() ? 1 : 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// materialize (solver.cpp:91-102) of one decision path: (var, upper, mid)
// triples; best == INT32_MAX means no objective bound.
int refh_replay(void* h, const int32_t* root, int n_dec, const int32_t* dec, int32_t best,
                int32_t* out, uint64_t* iters) {
  auto* m = static_cast<RefModel*>(h);
  try {
    Store s(m->schema);
    load_words(s, root);
    for (int i = 0; i < n_dec; ++i) {
      Decision d{dec[3 * i], dec[3 * i + 1] != 0, dec[3 * i + 2]};
      s.join_in_place(d.var, d.as_join());
    }
    if (best != kPosInf && m->obj >= 0) {
      s.join_in_place(m->obj, LatticeValue::interval(kNegInf, best - 1));
    }
    const EngineResult r = run_sequential(m->props, s);
    save_words(s, out);
    if (iters) *iters = r.iterations;
    return r.failed() ? 1 : 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// branch (solver.cpp:19-47): returns 0 none, 1 found, -1 error (unbounded).
int refh_branch(void* h, const int32_t* words, int32_t* var, int32_t* mid) {
  auto* m = static_cast<RefModel*>(h);
  try {
    Store s(m->schema);
    load_words(s, words);
    auto d = branch(s, BranchStrategy{m->cands});
    if (!d) return 0;
    *var = d->first.var;
    *mid = d->first.mid;
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// ---- all-solutions enumeration (harness over the reference API) ------------
// out[0..6] = nodes, failures, solutions, open_leaves, hash_sum, sweeps, exhausted
// threads <= 1: plain dfs from the root; else a BFS frontier of 8*threads
// open nodes (each counted once) drained by `threads` std::threads.
int refh_enumerate(void* h, int depth_cap, int threads, double budget_s, uint64_t node_budget,
                   uint64_t* out, double* elapsed_ms) {
  auto* m = static_cast<RefModel*>(h);
  try {
    EnumCounters c;
    const BranchStrategy strat{m->cands};
    Store root(m->schema);
    const auto t0 = Clock::now();
    const auto deadline =
        budget_s > 0 ? t0 + std::chrono::duration_cast<Clock::duration>(
                                std::chrono::duration<double>(budget_s))
                     : Clock::time_point::max();
    if (node_budget == 0) node_budget = UINT64_MAX;
    if (threads <= 1) {
      dfs_enum(*m, root, SearchNode{}, true, depth_cap, c, strat, deadline, node_budget);
    } else {
      std::deque<SearchNode> open;
      Store cur(m->schema);
      std::optional<std::pair<Decision, Decision>> dec;
      if (materialise(*m, root, cur, SearchNode{}, depth_cap, true, c, strat, &dec) ==
          Kind3::Expand) {
        open.push_back(SearchNode{});
      }
      const size_t target = static_cast<size_t>(8) * threads;
      while (!open.empty() && open.size() < target) {
        SearchNode node = std::move(open.front());
        open.pop_front();
        materialise(*m, root, cur, node, depth_cap, false, c, strat, &dec);
        const auto d = *dec;
        for (const Decision& dd : {d.first, d.second}) {
          SearchNode child = node;
          child.decisions.push_back(dd);
          if (materialise(*m, root, cur, child, depth_cap, true, c, strat, nullptr) ==
              Kind3::Expand) {
            open.push_back(std::move(child));
          }
        }
      }
      std::vector<SearchNode> frontier(open.begin(), open.end());
      std::atomic<size_t> cursor{0};
      auto worker = [&]() {
        while (true) {
          const size_t i = cursor.fetch_add(1);
          if (i >= frontier.size() || c.stop.load()) break;
          dfs_enum(*m, root, frontier[i], false, depth_cap, c, strat, deadline, node_budget);
        }
      };
      std::vector<std::thread> pool;
      for (int w = 0; w < threads; ++w) pool.emplace_back(worker);
      for (auto& t : pool) t.join();
    }
    out[0] = c.nodes;
    out[1] = c.failures;
    out[2] = c.solutions;
    out[3] = c.open;
    out[4] = c.hash;
    out[5] = c.sweeps;
    out[6] = c.stop.load() ? 0 : 1;
    if (elapsed_ms)
      *elapsed_ms = std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// ---- branch and bound --------------------------------------------------------
// out: [status, has_obj, obj] ; st: [nodes, solutions] ; best_words optional.
static void fill_solve(RefModel* m, const SolveResult& r, int32_t* out, uint64_t* st,
                       double* elapsed_ms, int32_t* best_words) {
  out[0] = static_cast<int32_t>(r.status);
  out[1] = r.objective ? 1 : 0;
  out[2] = r.objective ? *r.objective : 0;
  st[0] = r.stats.nodes;
  st[1] = r.stats.solutions;
  if (elapsed_ms) *elapsed_ms = static_cast<double>(r.stats.elapsed.count());
  if (best_words && !r.best_store.empty()) {
    const Schema& s = *m->schema;
    for (Slot i = 0; i < s.slot_count(); ++i) {
      const LatticeValue& v = r.best_store[static_cast<size_t>(i)];
      best_words[s.first_word(i)] = v.lo;
      if (v.kind == Kind::Interval) best_words[s.first_word(i) + 1] = v.hi;
    }
  }
}

int refh_solve_parallel(void* h, unsigned workers, double timeout_s, uint64_t node_limit,
                        unsigned eps_factor, int32_t* out, uint64_t* st, double* elapsed_ms,
                        int32_t* best_words) {
  auto* m = static_cast<RefModel*>(h);
  try {
    Store root(m->schema);
    SolveLimits lim;
    if (timeout_s > 0)
      lim.timeout = std::chrono::duration_cast<Clock::duration>(std::chrono::duration<double>(timeout_s));
    lim.node_limit = node_limit;
    const SolveResult r = solve_parallel(root, m->props, m->obj, workers, lim, {}, eps_factor,
                                         nullptr, BranchStrategy{m->cands});
    fill_solve(m, r, out, st, elapsed_ms, best_words);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int refh_solve_dfs(void* h, double timeout_s, uint64_t node_limit, int32_t* out, uint64_t* st,
                   double* elapsed_ms, int32_t* best_words) {
  auto* m = static_cast<RefModel*>(h);
  try {
    Store root(m->schema);
    SolveLimits lim;
    if (timeout_s > 0)
      lim.timeout = std::chrono::duration_cast<Clock::duration>(std::chrono::duration<double>(timeout_s));
    lim.node_limit = node_limit;
    Objective obj(m->obj);
    const SolveResult r = solve_dfs(root, m->props, obj, lim, {}, nullptr, BranchStrategy{m->cands});
    fill_solve(m, r, out, st, elapsed_ms, best_words);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// check_solution (rcpsp.cpp:275-300) on the start lower bounds of `words`.
int refh_check_solution(void* h, const int32_t* words) {
  auto* m = static_cast<RefModel*>(h);
  if (!m->is_rcpsp) return -1;
  std::vector<int32_t> starts;
  for (Slot s : m->rmodel.starts) starts.push_back(words[m->schema->first_word(s)]);
  return rcpsp::check_solution(m->inst, starts) ? 1 : 0;
}

}  // extern "C"
