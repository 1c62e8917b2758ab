// rcpsp.cpp — RCPSP instances, the decomposed cumulative model and the
// independent checker.  See rcpsp.hpp; citations are to /root/reference/proj.
#include "rcpsp.hpp"

#include <algorithm>
#include <cctype>
#include <climits>
#include <cstdint>
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

namespace {

// A small JSON reader: just enough of RFC 8259 for instance files (objects,
// arrays, integers, strings, true/false/null).  Values are kept as a tree.
struct JVal {
  enum class T { Null, Bool, Num, Str, Arr, Obj } t = T::Null;
  long long num = 0;
  bool real = false;  // a number with a fraction or exponent
  std::string str;
  std::vector<JVal> arr;
  std::vector<std::pair<std::string, JVal>> obj;
  const JVal* get(const std::string& k) const {
    for (const auto& [key, v] : obj)
      if (key == k) return &v;
    return nullptr;
  }
};

class JParser {
 public:
  explicit JParser(const std::string& s) : s_(s) {}
  JVal document() {
    JVal v = value(0);
    ws();
    if (i_ != s_.size()) fail("trailing characters");
    return v;
  }

 private:
  [[noreturn]] void fail(const std::string& what) const {
    throw ModelError("bad json instance: " + what + " at offset " + std::to_string(i_));
  }
  void ws() {
    while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\t' || s_[i_] == '\n' || s_[i_] == '\r')) ++i_;
  }
  bool lit(const char* w) {
    const std::size_t n = std::char_traits<char>::length(w);
    if (s_.compare(i_, n, w) != 0) return false;
    i_ += n;
    return true;
  }
  std::string string() {
    std::string out;
    ++i_;  // opening quote
    while (i_ < s_.size() && s_[i_] != '"') {
      char c = s_[i_++];
      if (c == '\\') {
        if (i_ >= s_.size()) fail("unterminated escape");
        c = s_[i_++];
        switch (c) {
          case 'n': c = '\n'; break;
          case 't': c = '\t'; break;
          case 'r': c = '\r'; break;
          case 'b': c = '\b'; break;
          case 'f': c = '\f'; break;
          case 'u':
            if (i_ + 4 > s_.size()) fail("bad unicode escape");
            i_ += 4;  // keys of interest are ASCII; keep a placeholder
            c = '?';
            break;
          default: break;  // \" \\ \/
        }
      }
      out.push_back(c);
    }
    if (i_ >= s_.size()) fail("unterminated string");
    ++i_;
    return out;
  }
  JVal value(int depth) {
    if (depth > 64) fail("nesting too deep");
    ws();
    if (i_ >= s_.size()) fail("unexpected end");
    JVal v;
    const char c = s_[i_];
    if (c == '{') {
      v.t = JVal::T::Obj;
      ++i_;
      ws();
      if (i_ < s_.size() && s_[i_] == '}') {
        ++i_;
        return v;
      }
      for (;;) {
        ws();
        if (i_ >= s_.size() || s_[i_] != '"') fail("expected a key");
        std::string k = string();
        ws();
        if (i_ >= s_.size() || s_[i_] != ':') fail("expected ':'");
        ++i_;
        v.obj.emplace_back(std::move(k), value(depth + 1));
        ws();
        if (i_ < s_.size() && s_[i_] == ',') {
          ++i_;
          continue;
        }
        if (i_ < s_.size() && s_[i_] == '}') {
          ++i_;
          return v;
        }
        fail("expected ',' or '}'");
      }
    }
    if (c == '[') {
      v.t = JVal::T::Arr;
      ++i_;
      ws();
      if (i_ < s_.size() && s_[i_] == ']') {
        ++i_;
        return v;
      }
      for (;;) {
        v.arr.push_back(value(depth + 1));
        ws();
        if (i_ < s_.size() && s_[i_] == ',') {
          ++i_;
          continue;
        }
        if (i_ < s_.size() && s_[i_] == ']') {
          ++i_;
          return v;
        }
        fail("expected ',' or ']'");
      }
    }
    if (c == '"') {
      v.t = JVal::T::Str;
      v.str = string();
      return v;
    }
    if (lit("true")) {
      v.t = JVal::T::Bool;
      v.num = 1;
      return v;
    }
    if (lit("false")) {
      v.t = JVal::T::Bool;
      return v;
    }
    if (lit("null")) return v;
    if (c == '-' || (c >= '0' && c <= '9')) {
      const std::size_t b = i_;
      if (s_[i_] == '-') ++i_;
      while (i_ < s_.size() && std::isdigit(static_cast<unsigned char>(s_[i_]))) ++i_;
      while (i_ < s_.size() && (s_[i_] == '.' || s_[i_] == 'e' || s_[i_] == 'E' || s_[i_] == '+' || s_[i_] == '-' ||
                                std::isdigit(static_cast<unsigned char>(s_[i_])))) {
        v.real = true;
        ++i_;
      }
      const std::string tok = s_.substr(b, i_ - b);
      if (tok == "-" || tok.size() > 19) fail("bad number");
      v.t = JVal::T::Num;
      v.num = v.real ? static_cast<long long>(std::stod(tok)) : std::stoll(tok);
      return v;
    }
    fail("unexpected character");
  }
  const std::string& s_;
  std::size_t i_ = 0;
};

std::int32_t jint(const JVal& v, const char* what) {
  if (v.t != JVal::T::Num || v.real || v.num < INT32_MIN || v.num > INT32_MAX)
    throw ModelError(std::string("bad json instance: ") + what + " must be a 32-bit integer");
  return static_cast<std::int32_t>(v.num);
}

std::vector<std::int32_t> jints(const JVal& v, const char* what) {
  if (v.t != JVal::T::Arr) throw ModelError(std::string("bad json instance: ") + what + " must be an array");
  std::vector<std::int32_t> out;
  for (const JVal& x : v.arr) out.push_back(jint(x, what));
  return out;
}

}  // namespace

RcpspInstance parse_json(const std::string& text) {
  const JVal j = JParser(text).document();
  if (j.t != JVal::T::Obj) throw ModelError("bad json instance: the document must be an object");
  const JVal* tasks = j.get("tasks");
  if (!tasks || tasks->t != JVal::T::Arr) throw ModelError("bad json instance: key 'tasks' not found");
  RcpspInstance inst;
  if (const JVal* c = j.get("capacities")) inst.capacity = jints(*c, "capacities");
  for (const JVal& t : tasks->arr) {
    if (t.t != JVal::T::Obj) throw ModelError("bad json instance: a task must be an object");
    const JVal* d = t.get("duration");
    if (!d) throw ModelError("bad json instance: key 'duration' not found");
    inst.duration.push_back(jint(*d, "duration"));
    std::vector<std::int32_t> u;
    if (const JVal* us = t.get("usages")) u = jints(*us, "usages");
    u.resize(inst.capacity.size(), 0);  // rcpsp.cpp:155: usages padded/truncated to the resources
    inst.usage.push_back(std::move(u));
  }
  if (const JVal* ps = j.get("precedences")) {
    if (ps->t != JVal::T::Arr) throw ModelError("bad json instance: precedences must be an array");
    for (const JVal& p : ps->arr) {
      const std::vector<std::int32_t> ij = jints(p, "precedence");
      if (ij.size() != 2) throw ModelError("precedence entries must be pairs");
      if (ij[0] < 0 || ij[1] < 0) throw ModelError("precedence endpoint out of range");
      inst.precedences.emplace_back(ij[0], ij[1]);
    }
  }
  if (const JVal* h = j.get("horizon")) {
    inst.horizon = jint(*h, "horizon");
  } else {
    std::int64_t sum = 0;
    for (std::int32_t d : inst.duration) sum += d;
    inst.horizon = static_cast<std::int32_t>(std::min<std::int64_t>(sum, kPosInf - 2));
  }
  validate(inst);
  return inst;
}

std::string patterson_text(const RcpspInstance& inst) {
  std::ostringstream o;
  const std::size_t n = inst.tasks();
  o << n << ' ' << inst.resources() << '\n';
  for (std::size_t k = 0; k < inst.resources(); ++k) o << (k ? " " : "") << inst.capacity[k];
  o << '\n';
  std::vector<std::vector<std::int32_t>> succ(n);
  for (const auto& [i, j] : inst.precedences) succ[static_cast<std::size_t>(i)].push_back(j + 1);
  for (std::size_t i = 0; i < n; ++i) {
    o << inst.duration[i];
    for (std::int32_t u : inst.usage[i]) o << ' ' << u;
    o << ' ' << succ[i].size();
    for (std::int32_t j : succ[i]) o << ' ' << j;
    o << '\n';
  }
  return o.str();
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
