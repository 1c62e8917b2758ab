// rcpsp.cpp — RCPSP instances, the decomposed cumulative model and the
// independent checker.  See rcpsp.hpp; citations are to /root/reference/proj.
#include "rcpsp.hpp"

#include <algorithm>
#include <random>
#include <set>
#include <sstream>

namespace pccp_b200 {

void validate(const RcpspInstance& inst) {
  const std::size_t n = inst.tasks();
  if (inst.usage.size() != n) throw ModelError("usage table does not match the task count");
  for (std::size_t i = 0; i < n; ++i) {
    if (inst.usage[i].size() != inst.resources()) throw ModelError("task usage arity does not match resource count");
    if (inst.duration[i] < 0) throw ModelError("negative duration");
    for (std::int32_t u : inst.usage[i])
      if (u < 0) throw ModelError("negative resource usage");
  }
  std::vector<int> indeg(n, 0);
  for (const auto& [i, j] : inst.precedences) {
    if (i < 0 || j < 0 || static_cast<std::size_t>(i) >= n || static_cast<std::size_t>(j) >= n)
      throw ModelError("precedence endpoint out of range");
    if (i == j) throw ModelError("self precedence");
    ++indeg[static_cast<std::size_t>(j)];
  }
  // Kahn's algorithm: every task must be removable.
  std::vector<std::size_t> ready;
  for (std::size_t i = 0; i < n; ++i)
    if (indeg[i] == 0) ready.push_back(i);
  std::size_t seen = 0;
  while (!ready.empty()) {
    const std::size_t i = ready.back();
    ready.pop_back();
    ++seen;
    for (const auto& [a, b] : inst.precedences)
      if (static_cast<std::size_t>(a) == i && --indeg[static_cast<std::size_t>(b)] == 0)
        ready.push_back(static_cast<std::size_t>(b));
  }
  if (seen != n) throw ModelError("precedence graph is cyclic");
}

// The generator of the reference's synthetic Patterson-style corpus
// (tests/support/corpus.cpp:32-90): capacities U[4,7]; real tasks get a
// duration U[1,9] and usages U[0, 2c/3]; tasks fill layers of width U{2,3};
// each task of layer l>0 takes 1-2 random predecessors in layer l-1; tasks
// without predecessor (successor) hang off the source (sink) dummy.  The draw
// order is the reference's, so seeds give the same instances.
RcpspInstance random_patterson(std::uint64_t seed, int n_real, int resources) {
  std::mt19937_64 rng(seed);
  auto draw = [&rng](int lo, int hi) { return std::uniform_int_distribution<int>(lo, hi)(rng); };
  RcpspInstance inst;
  const std::size_t n = static_cast<std::size_t>(n_real) + 2;
  for (int k = 0; k < resources; ++k) inst.capacity.push_back(draw(4, 7));
  inst.duration.assign(n, 0);
  inst.usage.assign(n, std::vector<std::int32_t>(static_cast<std::size_t>(resources), 0));
  for (std::size_t t = 1; t + 1 < n; ++t) {
    inst.duration[t] = draw(1, 9);
    for (int k = 0; k < resources; ++k)
      inst.usage[t][static_cast<std::size_t>(k)] = draw(0, (2 * inst.capacity[static_cast<std::size_t>(k)]) / 3);
  }
  const std::size_t width = static_cast<std::size_t>(draw(2, 3));
  std::vector<std::vector<std::size_t>> layer;
  for (std::size_t t = 1; t + 1 < n; ++t) {
    if (layer.empty() || layer.back().size() >= width) layer.emplace_back();
    layer.back().push_back(t);
  }
  std::set<std::pair<std::size_t, std::size_t>> arcs;  // sorted, de-duplicated
  for (std::size_t l = 1; l < layer.size(); ++l) {
    const auto& prev = layer[l - 1];
    for (std::size_t t : layer[l]) {
      const int preds = draw(1, 2);
      for (int p = 0; p < preds; ++p)
        arcs.emplace(prev[static_cast<std::size_t>(draw(0, static_cast<int>(prev.size()) - 1))], t);
    }
  }
  std::vector<char> has_pred(n, 0), has_succ(n, 0);
  for (const auto& [a, b] : arcs) {
    inst.precedences.emplace_back(static_cast<std::int32_t>(a), static_cast<std::int32_t>(b));
    has_pred[b] = 1;
    has_succ[a] = 1;
  }
  for (std::size_t t = 1; t + 1 < n; ++t) {
    if (!has_pred[t]) inst.precedences.emplace_back(0, static_cast<std::int32_t>(t));
    if (!has_succ[t]) inst.precedences.emplace_back(static_cast<std::int32_t>(t), static_cast<std::int32_t>(n - 1));
  }
  std::int32_t h = 0;
  for (std::int32_t d : inst.duration) h += d;
  inst.horizon = h;
  validate(inst);
  return inst;
}

RcpspInstance parse_patterson(const std::string& text) {
  std::istringstream in(text);
  auto next = [&in](const char* what) -> std::int32_t {
    long long v;
    if (!(in >> v)) throw ModelError(std::string("truncated instance: expected ") + what);
    if (v < 0 || v > kPosInf - 1) throw ModelError(std::string(what) + " out of range");
    return static_cast<std::int32_t>(v);
  };
  RcpspInstance inst;
  const std::int32_t jobs = next("job count");
  const std::int32_t res = next("resource count");
  for (std::int32_t k = 0; k < res; ++k) inst.capacity.push_back(next("capacity"));
  std::vector<std::vector<std::int32_t>> succ(static_cast<std::size_t>(jobs));
  for (std::int32_t j = 0; j < jobs; ++j) {
    inst.duration.push_back(next("duration"));
    std::vector<std::int32_t> u;
    for (std::int32_t k = 0; k < res; ++k) u.push_back(next("usage"));
    inst.usage.push_back(std::move(u));
    const std::int32_t ns = next("successor count");
    for (std::int32_t s = 0; s < ns; ++s) {
      const std::int32_t id = next("successor id");
      if (id < 1 || id > jobs) throw ModelError("successor id out of range");
      succ[static_cast<std::size_t>(j)].push_back(id - 1);
    }
  }
  for (std::size_t i = 0; i < succ.size(); ++i)
    for (std::int32_t j : succ[i]) inst.precedences.emplace_back(static_cast<std::int32_t>(i), j);
  std::int64_t h = 0;
  for (std::int32_t d : inst.duration) h += d;
  inst.horizon = static_cast<std::int32_t>(std::min<std::int64_t>(h, kPosInf - 2));
  validate(inst);
  return inst;
}

RcpspModel build_rcpsp(const RcpspInstance& inst) {
  const std::size_t n = inst.tasks();
  RcpspModel out;
  out.model = std::make_unique<Model>();
  Model& m = *out.model;
  if (n == 0) {  // degenerate: one zero makespan (rcpsp.cpp:182-191)
    m.objective = m.add_cell(Kind::Interval, "makespan");
    m.tell_interval(m.objective, 0, 0);
    return out;
  }
  const std::int32_t h = inst.horizon;
  for (std::size_t i = 0; i < n; ++i) out.starts.push_back(m.add_cell(Kind::Interval, "s" + std::to_string(i + 1)));
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t j = 0; j < n; ++j)
      out.overlaps.push_back(m.add_cell(Kind::Interval, "b" + std::to_string(i + 1) + "_" + std::to_string(j + 1)));
  auto b = [&](std::size_t i, std::size_t j) { return out.overlaps[i * n + j]; };

  // Domains, then the diagonal: a running task overlaps its own start; a
  // zero-duration task overlaps nothing (rcpsp.cpp:205-227).
  for (std::size_t i = 0; i < n; ++i) m.tell_interval(out.starts[i], 0, h);
  for (std::size_t i = 0; i < n * n; ++i) m.tell_interval(out.overlaps[i], 0, 1);
  for (std::size_t i = 0; i < n; ++i) {
    if (inst.duration[i] > 0) {
      m.tell_interval(b(i, i), 1, 1);
    } else {
      for (std::size_t j = 0; j < n; ++j) m.tell_interval(b(i, j), 0, 0);
    }
  }
  for (const auto& [i, j] : inst.precedences)
    m.append(compile(precedes(Operand::v(out.starts[static_cast<std::size_t>(i)]),
                              inst.duration[static_cast<std::size_t>(i)],
                              Operand::v(out.starts[static_cast<std::size_t>(j)])),
                     m));
  // b_ij <-> (s_i <= s_j and s_j < s_i + d_i) for i != j, running i (rcpsp.cpp:239-250).
  for (std::size_t j = 0; j < n; ++j) {
    for (std::size_t i = 0; i < n; ++i) {
      if (i == j || inst.duration[i] == 0) continue;
      const Operand si = Operand::v(out.starts[i]), sj = Operand::v(out.starts[j]);
      m.append(compile_reified(b(i, j), and_c(leq(si, sj), leq_offset(sj, 1 - inst.duration[i], si)), m));
    }
  }
  // Per resource and task: the tasks overlapping j's start fit the capacity.
  for (std::size_t k = 0; k < inst.resources(); ++k) {
    for (std::size_t j = 0; j < n; ++j) {
      std::vector<std::pair<std::int32_t, std::int32_t>> terms;
      for (std::size_t i = 0; i < n; ++i)
        if (inst.usage[i][k] > 0) terms.emplace_back(inst.usage[i][k], b(i, j));
      if (!terms.empty()) m.append(compile(linear_leq(std::move(terms), inst.capacity[k]), m));
    }
  }
  m.objective = out.starts[n - 1];  // the sink's start is the makespan
  m.candidates = out.starts;        // branch on starts; propagation fixes the rest
  return out;
}

bool check_solution(const RcpspInstance& inst, const std::vector<std::int32_t>& starts) {
  const std::size_t n = inst.tasks();
  if (starts.size() != n) throw ModelError("check_solution: one start per task required");
  for (std::int32_t s : starts)
    if (s < 0) return false;
  for (const auto& [i, j] : inst.precedences)
    if (std::int64_t{starts[static_cast<std::size_t>(i)]} + inst.duration[static_cast<std::size_t>(i)] >
        starts[static_cast<std::size_t>(j)])
      return false;
  std::int64_t end = 0;
  for (std::size_t i = 0; i < n; ++i) end = std::max<std::int64_t>(end, std::int64_t{starts[i]} + inst.duration[i]);
  // Sweep time points with an event list instead of re-scanning all tasks.
  for (std::size_t k = 0; k < inst.resources(); ++k) {
    std::vector<std::int64_t> delta(static_cast<std::size_t>(end) + 1, 0);
    for (std::size_t i = 0; i < n; ++i) {
      if (inst.duration[i] == 0 || inst.usage[i][k] == 0) continue;
      delta[static_cast<std::size_t>(starts[i])] += inst.usage[i][k];
      delta[static_cast<std::size_t>(starts[i] + inst.duration[i])] -= inst.usage[i][k];
    }
    std::int64_t load = 0;
    for (std::int64_t t = 0; t < end; ++t) {
      load += delta[static_cast<std::size_t>(t)];
      if (load > inst.capacity[k]) return false;
    }
  }
  return true;
}

}  // namespace pccp_b200
