// dropin_demo.cpp — the reference library calling the B200 engine through
// integration/pccp_gpu_shim.hpp, exactly as a maintainer would wire it.
//
// Built by `make -C oracle dropin` (links the reference objects of oracle/_ref
// and paper_2207_12116_b200/libpccp_b200.so).  TEST INFRASTRUCTURE: run by
// tests/test_gpu_dropin.py on the GPU box.  Prints one JSON object.
#include <cstdio>
#include <random>

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

  std::printf(
      "{\"fixpoint_equal\": %s, \"cpu_status\": %d, \"gpu_status\": %d, \"cpu_objective\": %d, "
      "\"gpu_objective\": %d, \"valid\": %s, \"callbacks\": %d, \"generic_rejected\": %s, \"q8\": [%llu, %llu, %llu], "
      "\"ok\": %s}\n",
      fix_eq ? "true" : "false", (int)cpu.status, (int)dev.status, cpu.objective ? *cpu.objective : -1,
      dev.objective ? *dev.objective : -1, valid ? "true" : "false", callbacks, rejected ? "true" : "false",
      (unsigned long long)e.nodes, (unsigned long long)e.solutions, (unsigned long long)e.failures,
      ok ? "true" : "false");
  return ok ? 0 : 1;
}
