// verify_gpu.cpp — the reference's confluence check (`pccp verify`,
// tools/pccp.cpp:97-188) with the B200 engine's fixed points in the set.
//
// For every instance it root-propagates with the reference's own engines —
// run_sequential, run_fair x 10 seeds, run_parallel x {1, 2, 4, 8} workers —
// and with the device engine through integration/pccp_gpu_shim.hpp under
// several launch shapes (warp groups, CTA groups of 128 / 512 / 1024
// threads), and passes iff every run agrees with `seq` cell for cell (status
// only when failed, as the reference compares).  It also checks that the
// reference's non-monotone PCCP_VERIFY_MUTANT command (a generic
// std::function tell) is rejected by the device path with ModelError instead
// of being dropped.
//
// Instances: the 110-instance stand-in corpus (tests/support/corpus.cpp:92-104)
// and the RCPSP 30x4 parity seeds.  Built by `make -C oracle verify` from the
// unmodified reference sources.  TEST INFRASTRUCTURE: run by
// tests/test_gpu_dropin.py on the GPU box.  Prints one JSON object.
#include <cstdio>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "corpus.hpp"
#include "pccp/engine.hpp"
#include "pccp/propagation.hpp"
#include "pccp/rcpsp.hpp"
#include "pccp_gpu_shim.hpp"

using namespace pccp;

namespace {

struct Run {
  std::string name;
  std::vector<LatticeValue> snap;
  Status status;
};

// The reference's mutant hook (tools/pccp.cpp:114-143), restated: a generic
// tell whose value shrinks as the store grows.
std::vector<GuardedCommand> with_mutant(const rcpsp::RcpspInstance& inst, const rcpsp::RcpspModel& model) {
  std::vector<GuardedCommand> props = model.props;
  const std::size_t n = inst.task_count();
  std::vector<Slot> diagonals;
  for (std::size_t i = 0; i < n && diagonals.size() < 2; ++i)
    if (inst.tasks[i].duration > 0) diagonals.push_back(model.overlaps[i * n + i]);
  std::size_t first_real = 0;
  for (std::size_t i = 0; i < n; ++i)
    if (inst.tasks[i].duration > 0) {
      first_real = i;
      break;
    }
  GuardedCommand gc;
  gc.target = model.starts[first_real];
  GenericFn f;
  for (Slot d : diagonals) f.reads.push_back(lb_of(d));
  f.eval = [diagonals](const Store& s) {
    std::int32_t raised = 0;
    for (Slot d : diagonals) raised += std::max(0, s.get(d).lo);
    return LatticeValue::interval(raised <= 0 ? 1 : kNegInf, kPosInf);
  };
  gc.fn = MonotoneFn::make_generic(std::move(f));
  finalize(gc, *model.schema);
  props.insert(props.begin(), std::move(gc));
  return props;
}

// One instance: every reference engine and every device shape against seq.
// Returns "" on PASS, else the reference's FAIL text.
std::string verify(const rcpsp::RcpspModel& model, int& gpu_runs, int& runs_total) {
  std::vector<Run> runs;
  auto add_run = [&](const std::string& name, const std::function<EngineResult(Store&)>& f) {
    Store s(model.schema);
    const EngineResult r = f(s);
    runs.push_back(Run{name, s.snapshot(), r.status});
  };
  const auto& props = model.props;
  add_run("seq", [&](Store& s) { return run_sequential(props, s); });
  for (std::uint64_t seed = 1; seed <= 10; ++seed)
    add_run("fair/" + std::to_string(seed), [&](Store& s) { return run_fair(props, s, seed); });
  for (unsigned w : {1u, 2u, 4u, 8u})
    add_run("par/" + std::to_string(w), [&](Store& s) { return run_parallel(props, s, w); });
  for (int t : {32, 128, 512, 1024}) {
    gpu::GpuConfig cfg;
    cfg.group_threads = t;
    try {
      gpu::GpuEngine eng(*model.schema, props, {}, -1, cfg);
      add_run(t == 32 ? std::string("gpu/warp") : "gpu/cta" + std::to_string(t),
              [&](Store& s) { return eng.propagate(s); });
      ++gpu_runs;
    } catch (const std::runtime_error& e) {
      // a launch shape the store does not fit (shared memory) is not an engine of this model
      if (std::string(e.what()).find("exceeds shared memory") == std::string::npos &&
          std::string(e.what()).find("does not fit") == std::string::npos)
        throw;
    }
  }
  runs_total += static_cast<int>(runs.size());
  const Run& ref = runs.front();
  for (const Run& run : runs) {
    if (run.status != ref.status)
      return "FAIL: " + run.name + " ended " + (run.status == Status::Failed ? "Failed" : "Fixpoint") + " but " +
             ref.name + " ended " + (ref.status == Status::Failed ? "Failed" : "Fixpoint");
    if (ref.status == Status::Failed) continue;  // failed stores are all top
    for (Slot i = 0; i < model.schema->slot_count(); ++i)
      if (!equal(run.snap[static_cast<std::size_t>(i)], ref.snap[static_cast<std::size_t>(i)]))
        return "FAIL: cell '" + model.schema->name(i) + "' differs: " + run.name + " has " +
               to_string(run.snap[static_cast<std::size_t>(i)]) + ", " + ref.name + " has " +
               to_string(ref.snap[static_cast<std::size_t>(i)]);
  }
  return "";
}

}  // namespace

int main() {
  std::vector<std::pair<std::string, rcpsp::RcpspInstance>> instances;
  const auto corpus = testsupport::corpus_instances();
  for (std::size_t i = 0; i < corpus.size(); ++i) instances.emplace_back("corpus" + std::to_string(i), corpus[i]);
  for (std::uint64_t seed : {1ull, 2ull, 5ull, 7ull, 9ull, 11ull}) {
    std::mt19937_64 rng(seed);
    instances.emplace_back("rcpsp30_s" + std::to_string(seed), testsupport::random_patterson(rng, 30, 4));
  }
  int pass = 0, gpu_runs = 0, runs_total = 0, mutant_rejected = 0, mutant_checked = 0;
  std::string fails;
  for (const auto& [name, inst] : instances) {
    const auto model = rcpsp::build_model(inst);
    const std::string r = verify(model, gpu_runs, runs_total);
    if (r.empty()) ++pass;
    else fails += (fails.empty() ? "" : " | ") + name + ": " + r;
    if (mutant_checked < 10 && !model.overlaps.empty()) {
      ++mutant_checked;
      try {
        gpu::GpuEngine eng(*model.schema, with_mutant(inst, model), {}, -1, {});
      } catch (const ModelError&) {
        ++mutant_rejected;
      }
    }
  }
  for (char& c : fails)
    if (c == '"') c = '\'';
  const bool ok = pass == static_cast<int>(instances.size()) && mutant_rejected == mutant_checked && mutant_checked > 0;
  std::printf(
      "{\"instances\": %zu, \"pass\": %d, \"runs\": %d, \"gpu_runs\": %d, \"mutant_checked\": %d, "
      "\"mutant_rejected\": %d, \"fails\": \"%s\", \"ok\": %s}\n",
      instances.size(), pass, runs_total, gpu_runs, mutant_checked, mutant_rejected, fails.c_str(),
      ok ? "true" : "false");
  return ok ? 0 : 1;
}
