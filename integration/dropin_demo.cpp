// dropin_demo.cpp — the reference library calling the B200 engine through
// integration/pccp_gpu_shim.hpp, exactly as a maintainer would wire it.
//
// Built by `make -C oracle dropin` (links the reference objects of oracle/_ref
// and paper_2207_12116_b200/libpccp_b200.so).  TEST INFRASTRUCTURE: run by
// tests/test_gpu_dropin.py on the GPU box.  Prints one JSON object.
#include <cstdio>
#include <random>
#include <string>

#include "corpus.hpp"
#include "pccp/propagation.hpp"
#include "pccp/rcpsp.hpp"
#include "pccp_gpu_shim.hpp"

using namespace pccp;

int main() {
  int ok = 1;
  // 1. run_sequential vs run_gpu on the RCPSP30 seed-1 root.
  std::mt19937_64 rng(1);
  const auto inst = testsupport::random_patterson(rng, 30, 4);
  const auto model = rcpsp::build_model(inst);
  Store a(model.schema), b(model.schema);
  const EngineResult ra = run_sequential(model.props, a);
  const EngineResult rb = gpu::run_gpu(model.props, b);
  const bool fix_eq = ra.status == rb.status && snapshots_equal(a.snapshot(), b.snapshot());
  ok &= fix_eq;

  // 2. solve_parallel vs solve_gpu: same optimum, checker-valid schedule.
  Store root(model.schema);
  const SolveResult cpu = solve_parallel(root, model.props, model.objective, 4, {}, {}, 8, nullptr,
                                         BranchStrategy{model.search_vars});
  int callbacks = 0;
  const SolveResult dev = gpu::solve_gpu(root, model.props, model.objective, {}, {},
                                         [&](const Store&, std::int32_t) { ++callbacks; },
                                         BranchStrategy{model.search_vars});
  const bool opt_eq = cpu.status == dev.status && cpu.objective == dev.objective;
  const bool valid = dev.objective && rcpsp::check_solution(inst, rcpsp::extract_starts(model, dev.best_store));
  ok &= opt_eq && valid && callbacks == 1;

  // 3. a generic (std::function) command is rejected with ModelError, never dropped.
  bool rejected = false;
  try {
    std::vector<GuardedCommand> g = model.props;
    GuardedCommand gc;
    gc.target = model.starts[1];
    GenericFn fn;
    fn.eval = [](const Store&) { return LatticeValue::interval(0, 1); };
    gc.fn = MonotoneFn::make_generic(fn);
    finalize(gc, *model.schema);
    g.push_back(gc);
    Store s(model.schema);
    gpu::run_gpu(g, s);
  } catch (const ModelError&) {
    rejected = true;
  }
  ok &= rejected;

  // 4. N-Queens 8 enumeration through the shim (92 solutions, 779 nodes).
  SchemaBuilder sb;
  std::vector<Slot> q;
  for (int i = 0; i < 8; ++i) q.push_back(sb.add_cell("q" + std::to_string(i), Kind::Interval));
  std::vector<Process> init;
  for (int i = 0; i < 8; ++i) init.push_back(tell_const(q[i], LatticeValue::interval(0, 7)));
  std::vector<GuardedCommand> props = gnf(par(std::move(init)), sb.peek());
  for (int i = 0; i < 8; ++i)
    for (int j = i + 1; j < 8; ++j)
      for (int d : {0, j - i, i - j}) {
        Propagator p = compile(not_c(and_c(leq_offset(Operand::v(q[i]), -d, Operand::v(q[j])),
                                           leq_offset(Operand::v(q[j]), d, Operand::v(q[i])))),
                               sb);
        props.insert(props.end(), p.commands.begin(), p.commands.end());
      }
  auto schema = sb.share();
  finalize_all(props, *schema);
  Store qroot(schema);
  const auto e = gpu::enumerate_gpu(qroot, props);
  const bool q8 = e.solutions == 92 && e.nodes == 779 && e.failures == 298;
  ok &= q8;

  // 5. solve_gpu over two shards (GpuConfig{devices = {0, 0}}: two contexts on
  //    device 0 splitting one EPS frontier, incumbent linked through peer
  //    memory) against solve_parallel, on RCPSP30 seeds 1 and 7.
  bool sharded_eq = true;
  std::string sharded_txt;
  for (std::uint64_t seed : {1ull, 7ull}) {
    std::mt19937_64 r2(seed);
    const auto inst2 = testsupport::random_patterson(r2, 30, 4);
    const auto m2 = rcpsp::build_model(inst2);
    Store root2(m2.schema);
    const SolveResult c2 = solve_parallel(root2, m2.props, m2.objective, 4, {}, {}, 8, nullptr,
                                          BranchStrategy{m2.search_vars});
    gpu::GpuConfig two;
    two.devices = {0, 0};
    const SolveResult d2 = gpu::solve_gpu(root2, m2.props, m2.objective, two, {}, nullptr,
                                          BranchStrategy{m2.search_vars});
    const bool v2 = d2.objective && rcpsp::check_solution(inst2, rcpsp::extract_starts(m2, d2.best_store));
    sharded_eq &= c2.status == d2.status && c2.objective == d2.objective && v2;
    sharded_txt += (sharded_txt.empty() ? "" : ", ") + std::to_string(c2.objective ? *c2.objective : -1) + "/" +
                   std::to_string(d2.objective ? *d2.objective : -1);
  }
  ok &= sharded_eq;

  // 6. A persistent GpuEngine: lowered once, solved three times, same optimum.
  gpu::GpuEngine eng(*model.schema, model.props, BranchStrategy{model.search_vars}, model.objective);
  bool persistent = true;
  for (int k = 0; k < 3; ++k) {
    const SolveResult rk = eng.solve(root);
    persistent &= rk.status == SolveStatus::Optimal && rk.objective == cpu.objective;
  }
  ok &= persistent;

  // 7. propagate_batch_gpu on random sub-boxes of the RCPSP30 root fixed point
  //    against run_sequential on each (engine.cpp:13-32).
  std::mt19937 pick(5);
  std::vector<Store> batch;
  std::vector<Store> cpu_batch;
  for (int k = 0; k < 64; ++k) {
    batch.emplace_back(model.schema);
    cpu_batch.emplace_back(model.schema);
    for (Word i = 0; i < a.schema().word_count(); ++i) {
      batch.back().store_word(i, a.load_word(i));
      cpu_batch.back().store_word(i, a.load_word(i));
    }
    for (int d = 0; d < 3; ++d) {  // tighten a few start windows
      const Slot st = model.starts[pick() % model.starts.size()];
      const LatticeValue v = a.get(st);
      if (v.hi <= v.lo) continue;
      const std::int32_t mid = v.lo + static_cast<std::int32_t>(pick() % static_cast<unsigned>(v.hi - v.lo));
      const LatticeValue j = (pick() & 1) ? LatticeValue::interval(v.lo, mid) : LatticeValue::interval(mid + 1, v.hi);
      batch.back().join_in_place(st, j);
      cpu_batch.back().join_in_place(st, j);
    }
  }
  const auto gr = gpu::propagate_batch_gpu(model.props, std::span<Store>(batch));
  int batch_eq = 0, batch_failed = 0;
  for (std::size_t k = 0; k < batch.size(); ++k) {
    const EngineResult cr = run_sequential(model.props, cpu_batch[k]);
    const bool same = cr.status == gr[k].status &&
                      (cr.status == Status::Failed || snapshots_equal(cpu_batch[k].snapshot(), batch[k].snapshot()));
    batch_eq += same ? 1 : 0;
    batch_failed += cr.status == Status::Failed ? 1 : 0;
  }
  ok &= batch_eq == static_cast<int>(batch.size());

  std::printf(
      "{\"fixpoint_equal\": %s, \"cpu_status\": %d, \"gpu_status\": %d, \"cpu_objective\": %d, "
      "\"gpu_objective\": %d, \"valid\": %s, \"callbacks\": %d, \"generic_rejected\": %s, \"q8\": [%llu, %llu, %llu], "
      "\"sharded_equal\": %s, \"sharded_optima\": \"%s\", \"persistent\": %s, \"batch_equal\": %d, "
      "\"batch_failed\": %d, \"ok\": %s}\n",
      fix_eq ? "true" : "false", (int)cpu.status, (int)dev.status, cpu.objective ? *cpu.objective : -1,
      dev.objective ? *dev.objective : -1, valid ? "true" : "false", callbacks, rejected ? "true" : "false",
      (unsigned long long)e.nodes, (unsigned long long)e.solutions, (unsigned long long)e.failures,
      sharded_eq ? "true" : "false", sharded_txt.c_str(), persistent ? "true" : "false", batch_eq, batch_failed,
      ok ? "true" : "false");
  return ok ? 0 : 1;
}
