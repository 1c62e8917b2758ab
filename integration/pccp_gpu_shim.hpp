// pccp_gpu_shim.hpp — the reference-side binding of the B200 engine.
//
// A header a maintainer of the reference (/root/reference/proj) drops into
// its include path to route search through the GPU: it serialises the
// reference's own Schema + std::vector<GuardedCommand> into the flat tables
// of include/pccp_gpu.h and exposes entry points with the reference's
// signatures:
//
//   pccp::gpu::solve_gpu            ~ pccp::solve_parallel  (solver.hpp:124-128; `workers` -> GpuConfig)
//   pccp::gpu::run_gpu              ~ pccp::run_sequential  (engine.hpp:27-28)
//   pccp::gpu::propagate_batch_gpu  ~ run_sequential over many stores at once (engine.hpp:27-41)
//   pccp::gpu::enumerate_gpu          (new: all-solutions counting)
//   pccp::gpu::GpuEngine              a persistent engine: the model is lowered and uploaded
//                                     once, then solved / enumerated / propagated repeatedly
//
// GpuConfig::devices lists one context per entry: {0} is one GPU, {0,1,...,7}
// the eight GPUs of a box, and a repeated ordinal ({0,0}) runs two shards on
// one device.  The shards split one bound-free EPS frontier (i mod N) and
// share the incumbent through peer memory (pccp_gpu_link_peers); the result
// follows finish() (solver.cpp:148-162) over their union.
//
// Error behaviour: PCCP_EMODEL -> pccp::ModelError (lattice.hpp:29-32), any
// other failure -> std::runtime_error.  Generic (std::function) predicates and
// functions cannot run on the device and raise ModelError here, never silently.
//
// Deviation (documented in INTEGRATION.md): the SolutionCallback runs once,
// after the search, with the best store — the device cannot call back into
// host code mid-search (the reference calls it on worker threads).
#pragma once

#include <chrono>
#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "pccp/engine.hpp"
#include "pccp/solver.hpp"
#include "pccp_gpu.h"

namespace pccp::gpu {

struct FlatModel {
  std::vector<std::uint8_t> kind;
  std::vector<std::uint32_t> word;
  std::vector<std::uint32_t> off{0};
  std::vector<std::int32_t> code;
  std::vector<std::int32_t> cands;
  pccp_model view{};
};

inline void put_expr(std::vector<std::int32_t>& code, const LinExpr& e) {
  code.push_back(e.k);
  code.push_back(static_cast<std::int32_t>(e.terms.size()));
  for (const Term& t : e.terms) {
    code.push_back(t.coef);
    code.push_back(static_cast<std::int32_t>(t.word));
  }
}

// Schema + finalized GuardedCommands -> flat tables (include/pccp_gpu.h).
inline FlatModel serialise(const Schema& schema, std::span<const GuardedCommand> props,
                           const BranchStrategy& strategy = {}, Slot objective = -1) {
  FlatModel f;
  for (Slot s = 0; s < schema.slot_count(); ++s) {
    f.kind.push_back(static_cast<std::uint8_t>(schema.kind(s)));
    f.word.push_back(schema.first_word(s));
  }
  for (const GuardedCommand& gc : props) {
    if (gc.fn.generic) throw ModelError("GPU engine: generic MonotoneFn cannot be lowered");
    f.code.push_back(static_cast<std::int32_t>(gc.guards.size()));
    f.code.push_back(gc.target);
    f.code.push_back(static_cast<std::int32_t>(gc.target_kind));
    f.code.push_back(static_cast<std::int32_t>(gc.target_word));
    f.code.push_back((gc.fn.scalar ? PCCP_FN_SCALAR : 0) | (gc.fn.lb ? PCCP_FN_LB : 0) |
                     (gc.fn.ub ? PCCP_FN_UB : 0));
    for (const Pred& p : gc.guards) {
      if (p.generic) throw ModelError("GPU engine: generic Pred cannot be lowered");
      f.code.push_back(p.rel == Pred::Rel::Leq ? PCCP_LEQ : PCCP_GT);
      f.code.push_back(p.rhs);
      put_expr(f.code, p.lhs);
    }
    if (gc.fn.scalar) put_expr(f.code, *gc.fn.scalar);
    if (gc.fn.lb) put_expr(f.code, *gc.fn.lb);
    if (gc.fn.ub) put_expr(f.code, *gc.fn.ub);
    f.off.push_back(static_cast<std::uint32_t>(f.code.size()));
  }
  f.cands.assign(strategy.candidates.begin(), strategy.candidates.end());
  f.view.n_slots = static_cast<std::uint32_t>(f.kind.size());
  f.view.slot_kind = f.kind.data();
  f.view.slot_word = f.word.data();
  f.view.n_words = schema.word_count();
  f.view.n_cmds = static_cast<std::uint32_t>(props.size());
  f.view.cmd_off = f.off.data();
  f.view.cmd_code = f.code.data();
  f.view.n_cands = static_cast<std::uint32_t>(f.cands.size());
  f.view.cands = f.cands.data();
  f.view.obj_slot = objective;
  return f;
}

// solve_parallel's `workers` and `eps_factor` arguments, for GPUs.
struct GpuConfig {
  std::vector<int> devices{0};  // one shard per entry (a device may repeat)
  int ctas_per_sm = 0;          // 0: occupancy
  int group_threads = 0;        // threads per subproblem: 32 (warp) .. 1024; 0: by store size
  int groups_per_cta = 0;       // warp groups per CTA; 0: auto
  int eps_factor = 0;           // EPS subproblems per resident group; 0: engine default
  int primal_ms = 0;            // > 0: primal dives before the reference-order search (include/pccp_gpu.h)
};

inline void check(int rc) {
  if (rc == PCCP_OK) return;
  const std::string msg = pccp_gpu_last_error();
  if (rc == PCCP_EMODEL) throw ModelError(msg);
  throw std::runtime_error("pccp_gpu: " + msg);
}

inline std::vector<std::int32_t> words_of(const Store& s) {
  std::vector<std::int32_t> w(s.schema().word_count());
  for (Word i = 0; i < w.size(); ++i) w[i] = s.load_word(i);
  return w;
}

struct EnumerateResult {
  std::uint64_t nodes = 0, failures = 0, solutions = 0, open_leaves = 0, hash_sum = 0;
  bool exhausted = true;
};

// A persistent engine: one context per GpuConfig::devices entry, the model
// lowered and uploaded once.  Not re-entrant (one caller thread).
class GpuEngine {
 public:
  GpuEngine(const Schema& schema, std::span<const GuardedCommand> props, const BranchStrategy& strategy = {},
            Slot objective = -1, const GpuConfig& cfg = {})
      : flat_(serialise(schema, props, strategy, objective)), n_words_(schema.word_count()) {
    if (cfg.devices.empty()) throw std::invalid_argument("GpuConfig: no devices");
    const int n = static_cast<int>(cfg.devices.size());
    try {
      for (int i = 0; i < n; ++i) {
        pccp_gpu_cfg c{};
        c.device = cfg.devices[static_cast<std::size_t>(i)];
        c.ctas_per_sm = cfg.ctas_per_sm;
        c.group_threads = cfg.group_threads;
        c.groups_per_cta = cfg.groups_per_cta;
        c.eps_factor = cfg.eps_factor;
        c.primal_ms = cfg.primal_ms;
        c.shard_index = i;
        c.shard_count = n;
        pccp_gpu_ctx* ctx = nullptr;
        check(pccp_gpu_open(&c, &ctx));
        ctx_.push_back(ctx);
        check(pccp_gpu_load(ctx, &flat_.view));
      }
      if (n > 1) check(pccp_gpu_link_peers(ctx_.data(), n));
    } catch (...) {
      close();
      throw;
    }
  }
  ~GpuEngine() { close(); }
  GpuEngine(const GpuEngine&) = delete;
  GpuEngine& operator=(const GpuEngine&) = delete;

  std::size_t shards() const { return ctx_.size(); }

  // solve_parallel (solver.cpp:229-283) over the shards: same result type and
  // status rules (finish, solver.cpp:148-162) over the union of the shards;
  // a primal dive that exhausted the whole tree on one shard is the proof.
  SolveResult solve(const Store& root, const SolveLimits& limits = {}, const SolutionCallback& on_solution = nullptr) {
    const std::vector<std::int32_t> rw = words_of(root);
    const std::size_t n = ctx_.size();
    for (pccp_gpu_ctx* c : ctx_) check(pccp_gpu_reset_shared(c));  // every shard before any starts
    std::vector<pccp_solve_result> res(n);
    std::vector<std::vector<std::int32_t>> best(n, std::vector<std::int32_t>(std::max<std::size_t>(n_words_, 1)));
    const pccp_limits lim{std::chrono::duration<double>(limits.timeout).count(), limits.node_limit};
    run_all([&](std::size_t k) { return pccp_gpu_solve(ctx_[k], rw.data(), &lim, &res[k], best[k].data()); });
    bool exhausted = true, proved = false, has = false;
    std::int32_t obj = 0;
    SolveResult out;
    double ms = 0;
    for (const pccp_solve_result& r : res) {
      exhausted = exhausted && (r.status == PCCP_OPTIMAL || r.status == PCCP_UNSAT);
      proved = proved || r.primal_proved;
      out.stats.nodes += r.stats.nodes;
      out.stats.solutions += r.stats.solutions;
      ms = std::max(ms, r.stats.elapsed_ms);
      if (r.has_objective && (!has || r.objective < obj)) {
        has = true;
        obj = r.objective;
      }
    }
    exhausted = exhausted || proved;
    out.status = has ? (exhausted ? SolveStatus::Optimal : SolveStatus::Sat)
                     : (exhausted ? SolveStatus::Unsat : SolveStatus::Unknown);
    out.stats.elapsed = std::chrono::milliseconds(static_cast<long long>(ms));
    if (has) {
      out.objective = obj;
      for (std::size_t k = 0; k < n; ++k) {
        if (res[k].has_objective != 1 || res[k].objective != obj) continue;
        Store s(root.schema_ptr());
        for (Word i = 0; i < n_words_; ++i) s.store_word(i, best[k][i]);
        out.best_store = s.snapshot();
        if (on_solution) on_solution(s, obj);
        break;
      }
    }
    return out;
  }

  // All-solutions enumeration below `root`: the shards' counters summed
  // (the hash-sum mod 2^64 by unsigned wrap-around).
  EnumerateResult enumerate(const Store& root, int depth_cap = -1, const SolveLimits& limits = {}) {
    const std::vector<std::int32_t> rw = words_of(root);
    std::vector<pccp_enum_result> res(ctx_.size());
    const pccp_limits lim{std::chrono::duration<double>(limits.timeout).count(), limits.node_limit};
    run_all([&](std::size_t k) { return pccp_gpu_enumerate(ctx_[k], rw.data(), depth_cap, &lim, &res[k]); });
    EnumerateResult e;
    for (const pccp_enum_result& r : res) {
      e.nodes += r.stats.nodes;
      e.failures += r.stats.failures;
      e.solutions += r.stats.solutions;
      e.open_leaves += r.stats.open_leaves;
      e.hash_sum += r.stats.hash_sum;
      e.exhausted = e.exhausted && r.exhausted != 0;
    }
    return e;
  }

  // run_sequential (engine.cpp:13-32) on every store, one device launch
  // (shard 0's context).  The stores are updated in place.
  std::vector<EngineResult> propagate_batch(std::span<Store> stores) {
    const std::size_t n = stores.size();
    std::vector<std::int32_t> w(n * n_words_);
    for (std::size_t k = 0; k < n; ++k)
      for (Word i = 0; i < n_words_; ++i) w[k * n_words_ + i] = stores[k].load_word(i);
    std::vector<std::uint8_t> st(n);
    std::vector<std::uint32_t> rounds(n);
    check(pccp_gpu_propagate_batch(ctx_.front(), w.data(), static_cast<std::uint32_t>(n), w.data(), st.data(),
                                   rounds.data()));
    std::vector<EngineResult> out(n);
    for (std::size_t k = 0; k < n; ++k) {
      for (Word i = 0; i < n_words_; ++i) stores[k].store_word(i, w[k * n_words_ + i]);
      out[k].status = st[k] ? Status::Failed : Status::Fixpoint;
      out[k].iterations = rounds[k];
    }
    return out;
  }

  EngineResult propagate(Store& s) { return propagate_batch(std::span<Store>(&s, 1)).front(); }

 private:
  template <class F>
  void run_all(F&& f) {
    const std::size_t n = ctx_.size();
    std::vector<int> rc(n, PCCP_OK);
    std::vector<std::string> err(n);
    if (n == 1) {
      rc[0] = f(std::size_t{0});
      if (rc[0] != PCCP_OK) err[0] = pccp_gpu_last_error();
    } else {  // one host thread per context (contexts are not re-entrant)
      std::vector<std::thread> th;
      for (std::size_t k = 0; k < n; ++k)
        th.emplace_back([&, k] {
          rc[k] = f(k);
          if (rc[k] != PCCP_OK) err[k] = pccp_gpu_last_error();
        });
      for (auto& t : th) t.join();
    }
    for (std::size_t k = 0; k < n; ++k) {
      if (rc[k] == PCCP_OK) continue;
      if (rc[k] == PCCP_EMODEL) throw ModelError(err[k]);
      throw std::runtime_error("pccp_gpu: " + err[k]);
    }
  }
  void close() {
    for (pccp_gpu_ctx* c : ctx_) pccp_gpu_close(c);
    ctx_.clear();
  }

  FlatModel flat_;
  Word n_words_;
  std::vector<pccp_gpu_ctx*> ctx_;
};

// Device counterpart of solve_parallel (solver.cpp:229-283): same result type
// and status rules; `workers` (and eps_factor) become a GpuConfig.
inline SolveResult solve_gpu(const Store& root, std::span<const GuardedCommand> props, Slot obj_var,
                             const GpuConfig& cfg = {}, const SolveLimits& limits = {},
                             const SolutionCallback& on_solution = nullptr, const BranchStrategy& strategy = {}) {
  GpuEngine e(root.schema(), props, strategy, obj_var, cfg);
  return e.solve(root, limits, on_solution);
}

// Device counterpart of run_sequential (engine.cpp:13-32) on one store.
inline EngineResult run_gpu(std::span<const GuardedCommand> gc, Store& s, const GpuConfig& cfg = {}) {
  GpuConfig one = cfg;
  one.devices.resize(1);
  GpuEngine e(s.schema(), gc, {}, -1, one);
  return e.propagate(s);
}

// run_sequential on many stores of one schema in one launch (parity checks,
// the GPU column of `pccp verify`).
inline std::vector<EngineResult> propagate_batch_gpu(std::span<const GuardedCommand> gc, std::span<Store> stores,
                                                     const GpuConfig& cfg = {}) {
  if (stores.empty()) return {};
  GpuConfig one = cfg;
  one.devices.resize(1);
  GpuEngine e(stores.front().schema(), gc, {}, -1, one);
  return e.propagate_batch(stores);
}

inline EnumerateResult enumerate_gpu(const Store& root, std::span<const GuardedCommand> props,
                                     const BranchStrategy& strategy = {}, int depth_cap = -1,
                                     const GpuConfig& cfg = {}, const SolveLimits& limits = {}) {
  GpuEngine e(root.schema(), props, strategy, -1, cfg);
  return e.enumerate(root, depth_cap, limits);
}

}  // namespace pccp::gpu
