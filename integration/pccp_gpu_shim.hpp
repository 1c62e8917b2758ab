// pccp_gpu_shim.hpp — the reference-side binding of the B200 engine.
//
// A header a maintainer of the reference (/root/reference/proj) drops into
// its include path to route search through the GPU: it serialises the
// reference's own Schema + std::vector<GuardedCommand> into the flat tables
// of include/pccp_gpu.h and exposes entry points with the reference's
// signatures:
//
//   pccp::gpu::solve_gpu   ~ pccp::solve_parallel   (solver.hpp:124-128)
//   pccp::gpu::run_gpu     ~ pccp::run_sequential   (engine.hpp:27-28)
//   pccp::gpu::enumerate_gpu  (new: all-solutions counting)
//
// Error behaviour: PCCP_EMODEL -> pccp::ModelError (lattice.hpp:29-32), any
// other failure -> std::runtime_error.  Generic (std::function) predicates and
// functions cannot run on the device and raise ModelError here, never silently.
//
// Deviation (documented in INTEGRATION.md): the SolutionCallback runs once,
// after the search, with the best store — the device cannot call back into
// host code mid-search (the reference calls it on worker threads).
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
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

struct GpuConfig {
  int device = 0;
  int eps_factor = 0;  // 0: engine default
  int shard_index = 0, shard_count = 1;
};

inline void check(int rc) {
  if (rc == PCCP_OK) return;
  const std::string msg = pccp_gpu_last_error();
  if (rc == PCCP_EMODEL) throw ModelError(msg);
  throw std::runtime_error("pccp_gpu: " + msg);
}

class Context {
 public:
  explicit Context(const GpuConfig& cfg) {
    pccp_gpu_cfg c{};
    c.device = cfg.device;
    c.eps_factor = cfg.eps_factor;
    c.shard_index = cfg.shard_index;
    c.shard_count = cfg.shard_count;
    check(pccp_gpu_open(&c, &ctx_));
  }
  ~Context() { pccp_gpu_close(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  pccp_gpu_ctx* get() const { return ctx_; }

 private:
  pccp_gpu_ctx* ctx_ = nullptr;
};

inline std::vector<std::int32_t> words_of(const Store& s) {
  std::vector<std::int32_t> w(s.schema().word_count());
  for (Word i = 0; i < w.size(); ++i) w[i] = s.load_word(i);
  return w;
}

// Device counterpart of solve_parallel (solver.cpp:229-283): same result type
// and status rules; `workers` becomes a GpuConfig.
inline SolveResult solve_gpu(const Store& root, std::span<const GuardedCommand> props, Slot obj_var,
                             const GpuConfig& cfg = {}, const SolveLimits& limits = {},
                             const SolutionCallback& on_solution = nullptr, const BranchStrategy& strategy = {}) {
  const Schema& schema = root.schema();
  FlatModel f = serialise(schema, props, strategy, obj_var);
  Context ctx(cfg);
  check(pccp_gpu_load(ctx.get(), &f.view));
  pccp_limits lim{std::chrono::duration<double>(limits.timeout).count(), limits.node_limit};
  pccp_solve_result r{};
  const std::vector<std::int32_t> rw = words_of(root);
  std::vector<std::int32_t> best(schema.word_count());
  check(pccp_gpu_solve(ctx.get(), rw.data(), &lim, &r, best.data()));
  SolveResult out;
  out.status = static_cast<SolveStatus>(r.status);
  out.stats.nodes = r.stats.nodes;
  out.stats.solutions = r.stats.solutions;
  out.stats.elapsed = std::chrono::milliseconds(static_cast<long long>(r.stats.elapsed_ms));
  if (r.has_objective) {
    out.objective = r.objective;
    Store s(root.schema_ptr());
    for (Word i = 0; i < best.size(); ++i) s.store_word(i, best[i]);
    out.best_store = s.snapshot();
    if (on_solution) on_solution(s, r.objective);
  }
  return out;
}

// Device counterpart of run_sequential (engine.cpp:13-32) on one store.
inline EngineResult run_gpu(std::span<const GuardedCommand> gc, Store& s, const GpuConfig& cfg = {}) {
  FlatModel f = serialise(s.schema(), gc);
  Context ctx(cfg);
  check(pccp_gpu_load(ctx.get(), &f.view));
  std::vector<std::int32_t> w = words_of(s);
  std::uint8_t status = 0;
  std::uint32_t rounds = 0;
  check(pccp_gpu_propagate_batch(ctx.get(), w.data(), 1, w.data(), &status, &rounds));
  for (Word i = 0; i < w.size(); ++i) s.store_word(i, w[i]);
  EngineResult r;
  r.status = status ? Status::Failed : Status::Fixpoint;
  r.iterations = rounds;
  return r;
}

struct EnumerateResult {
  std::uint64_t nodes = 0, failures = 0, solutions = 0, open_leaves = 0, hash_sum = 0;
  bool exhausted = true;
};

inline EnumerateResult enumerate_gpu(const Store& root, std::span<const GuardedCommand> props,
                                     const BranchStrategy& strategy = {}, int depth_cap = -1,
                                     const GpuConfig& cfg = {}, const SolveLimits& limits = {}) {
  FlatModel f = serialise(root.schema(), props, strategy);
  Context ctx(cfg);
  check(pccp_gpu_load(ctx.get(), &f.view));
  pccp_limits lim{std::chrono::duration<double>(limits.timeout).count(), limits.node_limit};
  pccp_enum_result r{};
  const std::vector<std::int32_t> rw = words_of(root);
  check(pccp_gpu_enumerate(ctx.get(), rw.data(), depth_cap, &lim, &r));
  return {r.stats.nodes, r.stats.failures, r.stats.solutions, r.stats.open_leaves, r.stats.hash_sum,
          r.exhausted != 0};
}

}  // namespace pccp::gpu
