// model.cpp — schema, indexical compiler and benchmark models (host side).
// See model.hpp.  Reference citations are to /root/reference/proj.
#include "model.hpp"

#include <random>

namespace pccp_b200 {

namespace {
constexpr std::int64_t kWide = std::int64_t{1} << 40;

std::int64_t widen(std::int32_t v) {
  return v == kPosInf ? kWide : v == kNegInf ? -kWide : static_cast<std::int64_t>(v);
}
std::int32_t narrow(std::int64_t v) {
  return v >= kPosInf ? kPosInf : v <= kNegInf ? kNegInf : static_cast<std::int32_t>(v);
}

Lin constant(std::int32_t k) { return Lin{k, {}}; }
Lin single(std::int32_t coef, std::int32_t slot, Part p, std::int32_t k = 0) {
  return Lin{k, {Term{coef, slot, p}}};
}

// tell_const of an interval value (MonotoneFn::const_value, command.cpp:82-91):
// an infinite bound tells nothing.
Cmd interval_tell(std::int32_t slot, std::int32_t lo, std::int32_t hi) {
  Cmd c;
  c.target = slot;
  if (lo != kNegInf) c.lb = constant(lo);
  if (hi != kPosInf) c.ub = constant(hi);
  return c;
}

void push_all(Gnf& out, Gnf more) {
  for (Cmd& c : more) out.push_back(std::move(c));
}

// ask(g1, ask(g2, ... body)) over a GNF body: guards accumulate outermost
// first (gnf_rec, process.cpp:117-147).
Gnf under_guards(const std::vector<Guard>& pre, const Gnf& body) {
  Gnf out = body;
  for (Cmd& c : out) c.guards.insert(c.guards.begin(), pre.begin(), pre.end());
  return out;
}

using Dnf = std::vector<std::vector<Guard>>;

// ask_dnf (propagation.cpp:255-264): one guarded copy of the body per disjunct.
Gnf ask_dnf(const Dnf& dnf, const Gnf& body) {
  Gnf out;
  for (const auto& disjunct : dnf) push_all(out, under_guards(disjunct, body));
  return out;
}

// ---- entailment predicates (propagation.cpp:133-201) -----------------------------
Guard ent_leq(const Constraint& c) {  // ub(x) - lb(y) <= -offset
  Guard g;
  if (!c.x.is_const) g.lhs.terms.push_back(Term{1, c.x.var, Part::Ub});
  else g.lhs.k = sat_add(g.lhs.k, c.x.value);
  if (!c.y.is_const) g.lhs.terms.push_back(Term{-1, c.y.var, Part::Lb});
  else g.lhs.k = sat_add(g.lhs.k, -c.y.value);
  g.gt = false;
  g.rhs = -c.offset;
  return g;
}
Guard ent_not_leq(const Constraint& c) {  // lb(x) - ub(y) > -offset
  Guard g;
  if (!c.x.is_const) g.lhs.terms.push_back(Term{1, c.x.var, Part::Lb});
  else g.lhs.k = sat_add(g.lhs.k, c.x.value);
  if (!c.y.is_const) g.lhs.terms.push_back(Term{-1, c.y.var, Part::Ub});
  else g.lhs.k = sat_add(g.lhs.k, -c.y.value);
  g.gt = true;
  g.rhs = -c.offset;
  return g;
}
Guard ent_sum(const Constraint& c, bool negated) {
  Guard g;
  for (const auto& [coef, var] : c.terms) g.lhs.terms.push_back(Term{coef, var, negated ? Part::Lb : Part::Ub});
  g.gt = negated;
  g.rhs = c.c;
  return g;
}

Dnf ent_guards(const Constraint& c);
Dnf ent_not_guards(const Constraint& c);

Dnf ent_guards(const Constraint& c) {
  switch (c.tag) {
    case Constraint::Tag::Leq: return {{ent_leq(c)}};
    case Constraint::Tag::Sum: return {{ent_sum(c, false)}};
    case Constraint::Tag::And: {  // product of the two DNFs
      const Dnf l = ent_guards(*c.a), r = ent_guards(*c.b);
      Dnf out;
      for (const auto& dl : l)
        for (const auto& dr : r) {
          std::vector<Guard> d = dl;
          d.insert(d.end(), dr.begin(), dr.end());
          out.push_back(std::move(d));
        }
      return out;
    }
    case Constraint::Tag::Not: return ent_not_guards(*c.a);
    default: throw CompileError("entailment guard of an iff constraint is not supported");
  }
}

Dnf ent_not_guards(const Constraint& c) {
  switch (c.tag) {
    case Constraint::Tag::Leq: return {{ent_not_leq(c)}};
    case Constraint::Tag::Sum: return {{ent_sum(c, true)}};
    case Constraint::Tag::And: {  // union
      Dnf out = ent_not_guards(*c.a);
      const Dnf r = ent_not_guards(*c.b);
      out.insert(out.end(), r.begin(), r.end());
      return out;
    }
    case Constraint::Tag::Not: return ent_guards(*c.a);
    default: throw CompileError("entailment guard of an iff constraint is not supported");
  }
}

// negate (propagation.cpp:111-131): not(x + k <= y) = y + (1-k) <= x.
Constraint negate(const Constraint& c) {
  switch (c.tag) {
    case Constraint::Tag::Leq: return leq_offset(c.y, 1 - c.offset, c.x);
    case Constraint::Tag::Not: return *c.a;
    case Constraint::Tag::Sum: throw CompileError("negation of a sum constraint is not supported");
    case Constraint::Tag::And: return not_c(c);
    default: throw CompileError("negation of an iff constraint is not supported");
  }
}

// Indexical compiler (propagation.cpp:266-373).  Cells for sum locals are
// appended to `m` in depth-first order, which is the order erase_locals
// numbers them (process.cpp:78-115).
struct Compiler {
  Model& m;

  Gnf leq(const Constraint& c) {  // compile_leq, propagation.cpp:266-290
    if (c.x.is_const && c.y.is_const)
      throw CompileError("leq with two constant operands");
    Gnf out;
    if (!c.x.is_const) {  // x <- (bot, ub(y) - offset)
      Cmd t;
      t.target = c.x.var;
      t.ub = c.y.is_const ? constant(sat_add(c.y.value, -c.offset))
                          : single(1, c.y.var, Part::Ub, -c.offset);
      out.push_back(std::move(t));
    }
    if (!c.y.is_const) {  // y <- (lb(x) + offset, top)
      Cmd t;
      t.target = c.y.var;
      t.lb = c.x.is_const ? constant(sat_add(c.x.value, c.offset))
                          : single(1, c.x.var, Part::Lb, c.offset);
      out.push_back(std::move(t));
    }
    return out;
  }

  Gnf binary_sum(const Constraint& c) {  // propagation.cpp:294-305
    const std::int32_t x = c.terms[0].second, y = c.terms[1].second;
    Cmd tx, ty;
    tx.target = x;
    tx.ub = single(-1, y, Part::Lb, c.c);
    ty.target = y;
    ty.ub = single(-1, x, Part::Lb, c.c);
    return {tx, ty};
  }

  Gnf general_sum(const Constraint& c) {  // propagation.cpp:314-335
    const std::int32_t lsum = m.add_cell(Kind::ZInc, "lsum");
    Gnf out;
    Cmd sum;
    sum.target = lsum;
    sum.scalar = Lin{};
    for (const auto& [coef, var] : c.terms) sum.scalar->terms.push_back(Term{coef, var, Part::Lb});
    out.push_back(std::move(sum));
    Cmd overload;  // [lsum > c] => lsum <- +inf
    overload.guards.push_back(Guard{single(1, lsum, Part::Scalar), true, c.c});
    overload.target = lsum;
    overload.scalar = constant(kPosInf);
    out.push_back(std::move(overload));
    for (const auto& [coef, var] : c.terms) {  // [coef + lsum - coef*lb(x) > c] => x <- (0,0)
      Cmd z = interval_tell(var, 0, 0);
      Guard g;
      g.lhs.k = coef;
      g.lhs.terms = {Term{1, lsum, Part::Scalar}, Term{-coef, var, Part::Lb}};
      g.gt = true;
      g.rhs = c.c;
      z.guards.push_back(std::move(g));
      out.push_back(std::move(z));
    }
    return out;
  }

  Gnf rec(const Constraint& c) {  // compile_rec, propagation.cpp:337-373
    switch (c.tag) {
      case Constraint::Tag::Leq: return leq(c);
      case Constraint::Tag::Sum:
        if (c.terms.size() == 2 && c.terms[0].first == 1 && c.terms[1].first == 1) return binary_sum(c);
        return general_sum(c);
      case Constraint::Tag::And: {
        Gnf out = rec(*c.a);
        push_all(out, rec(*c.b));
        return out;
      }
      case Constraint::Tag::Not: {
        const Constraint& inner = *c.a;
        if (inner.tag == Constraint::Tag::And) {
          // not(a and b): once one side is entailed, propagate the other's negation.
          const Gnf na = rec(negate(*inner.a));
          const Gnf nb = rec(negate(*inner.b));
          Gnf out = ask_dnf(ent_guards(*inner.a), nb);
          push_all(out, ask_dnf(ent_guards(*inner.b), na));
          return out;
        }
        return rec(negate(inner));
      }
      case Constraint::Tag::Iff: {
        const Constraint& a = *c.a;
        const Constraint& b = *c.b;
        const Gnf cb = rec(b), ca = rec(a), ncb = rec(not_c(b)), nca = rec(not_c(a));
        Gnf out = ask_dnf(ent_guards(a), cb);
        push_all(out, ask_dnf(ent_guards(b), ca));
        push_all(out, ask_dnf(ent_not_guards(a), ncb));
        push_all(out, ask_dnf(ent_not_guards(b), nca));
        return out;
      }
    }
    return {};
  }
};

}  // namespace

std::int32_t sat_add(std::int32_t a, std::int32_t b) { return narrow(widen(a) + widen(b)); }

// ---- Model -------------------------------------------------------------------------

std::int32_t Model::add_cell(Kind k, std::string name) {
  kinds_.push_back(k);
  words_.push_back(n_words_);
  names_.push_back(std::move(name));
  n_words_ += (k == Kind::Interval) ? 2u : 1u;
  return static_cast<std::int32_t>(kinds_.size()) - 1;
}

void Model::truncate_cells(std::int32_t n) {
  while (slot_count() > n) {
    n_words_ -= kinds_.back() == Kind::Interval ? 2u : 1u;
    kinds_.pop_back();
    words_.pop_back();
    names_.pop_back();
  }
}

void Model::append(Gnf cmds) { push_all(cmds_, std::move(cmds)); }

void Model::tell_interval(std::int32_t slot, std::int32_t lo, std::int32_t hi) {
  cmds_.push_back(interval_tell(slot, lo, hi));
}

std::vector<std::int32_t> Model::bottom() const {
  std::vector<std::int32_t> w(n_words_);
  for (std::size_t s = 0; s < kinds_.size(); ++s) {
    switch (kinds_[s]) {
      case Kind::Interval: w[words_[s]] = kNegInf; w[words_[s] + 1] = kPosInf; break;
      case Kind::ZInc: w[words_[s]] = kNegInf; break;
      case Kind::ZDec: w[words_[s]] = kPosInf; break;
      case Kind::BInc: w[words_[s]] = 0; break;
      case Kind::BDec: w[words_[s]] = 1; break;
    }
  }
  return w;
}

FlatTables Model::flatten() const {
  FlatTables t;
  for (std::size_t s = 0; s < kinds_.size(); ++s) {
    t.slot_kind.push_back(static_cast<std::uint8_t>(kinds_[s]));
    t.slot_word.push_back(words_[s]);
  }
  t.n_words = n_words_;
  auto word_of = [this](const Term& tm) -> std::int32_t {
    if (tm.slot < 0 || tm.slot >= slot_count()) throw ModelError("term reads an unknown cell");
    const bool interval = kind(tm.slot) == Kind::Interval;
    switch (tm.part) {
      case Part::Scalar:
        if (interval) throw ModelError("scalar read of interval cell");
        return static_cast<std::int32_t>(first_word(tm.slot));
      case Part::Lb:
        if (!interval) throw ModelError("lb read of scalar cell");
        return static_cast<std::int32_t>(first_word(tm.slot));
      case Part::Ub:
        if (!interval) throw ModelError("ub read of scalar cell");
        return static_cast<std::int32_t>(first_word(tm.slot) + 1);
    }
    return 0;
  };
  auto put = [&](const Lin& e) {
    t.cmd_code.push_back(e.k);
    t.cmd_code.push_back(static_cast<std::int32_t>(e.terms.size()));
    for (const Term& tm : e.terms) {
      t.cmd_code.push_back(tm.coef);
      t.cmd_code.push_back(word_of(tm));
    }
  };
  t.cmd_off.push_back(0);
  for (const Cmd& c : cmds_) {
    if (c.target < 0 || c.target >= slot_count()) throw ModelError("tell targets an unknown cell");
    t.cmd_code.push_back(static_cast<std::int32_t>(c.guards.size()));
    t.cmd_code.push_back(c.target);
    t.cmd_code.push_back(static_cast<std::int32_t>(kind(c.target)));
    t.cmd_code.push_back(static_cast<std::int32_t>(first_word(c.target)));
    t.cmd_code.push_back((c.scalar ? 1 : 0) | (c.lb ? 2 : 0) | (c.ub ? 4 : 0));
    for (const Guard& g : c.guards) {
      t.cmd_code.push_back(g.gt ? 1 : 0);
      t.cmd_code.push_back(g.rhs);
      put(g.lhs);
    }
    if (c.scalar) put(*c.scalar);
    if (c.lb) put(*c.lb);
    if (c.ub) put(*c.ub);
    t.cmd_off.push_back(static_cast<std::uint32_t>(t.cmd_code.size()));
  }
  t.cands = candidates;
  t.obj_slot = objective;
  return t;
}

// ---- constraint constructors -------------------------------------------------------

Constraint linear_leq(std::vector<std::pair<std::int32_t, std::int32_t>> terms, std::int32_t c) {
  for (const auto& tc : terms)
    if (tc.first < 0) throw CompileError("linear_leq: coefficients must be nonnegative");
  Constraint k;
  k.tag = Constraint::Tag::Sum;
  k.terms = std::move(terms);
  k.c = c;
  return k;
}
Constraint leq_offset(Operand x, std::int32_t offset, Operand y) {
  Constraint k;
  k.tag = Constraint::Tag::Leq;
  k.x = x;
  k.y = y;
  k.offset = offset;
  return k;
}
Constraint and_c(Constraint a, Constraint b) {
  Constraint k;
  k.tag = Constraint::Tag::And;
  k.a = std::make_shared<const Constraint>(std::move(a));
  k.b = std::make_shared<const Constraint>(std::move(b));
  return k;
}
Constraint iff_c(Constraint a, Constraint b) {
  Constraint k;
  k.tag = Constraint::Tag::Iff;
  k.a = std::make_shared<const Constraint>(std::move(a));
  k.b = std::make_shared<const Constraint>(std::move(b));
  return k;
}
Constraint not_c(Constraint a) {
  Constraint k;
  k.tag = Constraint::Tag::Not;
  k.a = std::make_shared<const Constraint>(std::move(a));
  return k;
}

// Cells appended by a compile that then throws are rolled back, matching the
// reference where locals are only erased after the whole tree compiled.
Gnf compile(const Constraint& c, Model& m) {
  const std::int32_t n = m.slot_count();
  try {
    Compiler comp{m};
    return comp.rec(c);
  } catch (...) {
    m.truncate_cells(n);
    throw;
  }
}

Gnf compile_reified(std::int32_t b, const Constraint& c, Model& m) {
  if (b < 0 || b >= m.slot_count() || m.kind(b) != Kind::Interval)
    throw CompileError("compile_reified: reification variable must be a 0/1 interval");
  const std::int32_t n = m.slot_count();
  Gnf when_true, when_false;
  try {
    Compiler comp{m};
    when_true = comp.rec(c);
    when_false = comp.rec(not_c(c));
  } catch (...) {
    m.truncate_cells(n);
    throw;
  }
  Gnf out = ask_dnf(ent_guards(c), Gnf{interval_tell(b, 1, 1)});
  push_all(out, ask_dnf(ent_not_guards(c), Gnf{interval_tell(b, 0, 0)}));
  push_all(out, under_guards({Guard{single(1, b, Part::Lb), true, 0}}, when_true));    // lb(b) >= 1
  push_all(out, under_guards({Guard{single(1, b, Part::Ub), false, 0}}, when_false));  // ub(b) <= 0
  return out;
}

// ---- benchmark models ----------------------------------------------------------------

// Config 1/2: N-Queens, q_i != q_j + d for d in {0, j-i, i-j} as
// not(and(q_i - d <= q_j, q_j + d <= q_i)).
std::unique_ptr<Model> build_nqueens(int n) {
  auto m = std::make_unique<Model>();
  std::vector<std::int32_t> q;
  for (int i = 0; i < n; ++i) q.push_back(m->add_cell(Kind::Interval, "q" + std::to_string(i)));
  for (int i = 0; i < n; ++i) m->tell_interval(q[i], 0, n - 1);
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j)
      for (int d : {0, j - i, i - j})
        m->append(compile(not_c(and_c(leq_offset(Operand::v(q[i]), -d, Operand::v(q[j])),
                                      leq_offset(Operand::v(q[j]), d, Operand::v(q[i])))),
                          *m));
  return m;
}

// Config 3: random linear integer CSP: n_vars interval
// variables in [0, dom_hi]; each constraint is, with probability 0.3, a
// precedence x_i + d <= x_j, else a sum of 2..5 terms a*x (a in 1..9) bounded
// by floor(dom_hi/4 * sum a).  libstdc++ distributions over mt19937_64.
std::unique_ptr<Model> build_random_csp(std::uint64_t seed, int n_vars, int n_cons, int dom_hi) {
  auto m = std::make_unique<Model>();
  std::mt19937_64 rng(seed);
  auto draw = [&rng](int lo, int hi) { return std::uniform_int_distribution<int>(lo, hi)(rng); };
  std::vector<std::int32_t> x;
  for (int i = 0; i < n_vars; ++i) x.push_back(m->add_cell(Kind::Interval, "x" + std::to_string(i)));
  for (int i = 0; i < n_vars; ++i) m->tell_interval(x[i], 0, dom_hi);
  std::uniform_real_distribution<double> coin(0.0, 1.0);
  for (int c = 0; c < n_cons; ++c) {
    if (coin(rng) < 0.3) {
      const int i = draw(0, n_vars - 2);
      const int j = draw(i + 1, n_vars - 1);
      const int d = draw(1, 2);
      m->append(compile(precedes(Operand::v(x[i]), d, Operand::v(x[j])), *m));
      continue;
    }
    const int k = draw(2, 5);
    std::vector<std::pair<std::int32_t, std::int32_t>> terms;
    std::int64_t sum_a = 0;
    for (int t = 0; t < k; ++t) {
      const int a = draw(1, 9);
      const int v = draw(0, n_vars - 1);
      terms.emplace_back(a, x[v]);
      sum_a += a;
    }
    m->append(compile(linear_leq(std::move(terms), static_cast<std::int32_t>(sum_a * dom_hi / 4)), *m));
  }
  return m;
}

}  // namespace pccp_b200
