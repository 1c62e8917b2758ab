// lower.cpp — flat reference tables -> device tables (see lower.hpp).
#include "lower.hpp"

#include <algorithm>
#include <functional>
#include <map>
#include <cstdlib>
#include <optional>
#include <stdexcept>
#include <tuple>

namespace pccp_b200 {

namespace {

struct Expr {
  std::int32_t k = 0;
  std::vector<std::pair<std::int32_t, std::uint32_t>> terms;  // (coef, word)
};
struct GuardP {
  int rel;
  std::int32_t rhs;
  Expr lhs;
};
struct CmdP {
  std::int32_t target;
  int kind;
  std::uint32_t tw;
  std::vector<GuardP> guards;
  std::optional<Expr> sc, lb, ub;
};

[[noreturn]] void bad(const std::string& why) { throw std::runtime_error(why); }

std::vector<CmdP> parse(const pccp_model& m) {
  std::vector<CmdP> out;
  out.reserve(m.n_cmds);
  const std::int32_t* code = m.cmd_code;
  for (std::uint32_t i = 0; i < m.n_cmds; ++i) {
    const std::uint32_t beg = m.cmd_off[i], end = m.cmd_off[i + 1];
    if (end < beg + 5) bad("command " + std::to_string(i) + ": truncated header");
    std::uint32_t p = beg;
    auto take = [&]() -> std::int32_t {
      if (p >= end) bad("command " + std::to_string(i) + ": truncated");
      return code[p++];
    };
    auto expr = [&]() {
      Expr e;
      e.k = take();
      const std::int32_t n = take();
      if (n < 0) bad("negative term count");
      for (std::int32_t t = 0; t < n; ++t) {
        const std::int32_t coef = take();
        const std::int32_t w = take();
        if (w < 0 || static_cast<std::uint32_t>(w) >= m.n_words) bad("term word out of range");
        e.terms.emplace_back(coef, static_cast<std::uint32_t>(w));
      }
      return e;
    };
    CmdP c;
    const std::int32_t ng = take();
    c.target = take();
    c.kind = take();
    const std::int32_t tw = take();
    const std::int32_t mask = take();
    if (ng < 0) bad("negative guard count");
    if (c.target < 0 || static_cast<std::uint32_t>(c.target) >= m.n_slots) bad("tell target out of range");
    if (c.kind != m.slot_kind[c.target]) bad("target kind does not match the schema");
    if (static_cast<std::uint32_t>(tw) != m.slot_word[c.target]) bad("target word does not match the schema");
    c.tw = static_cast<std::uint32_t>(tw);
    for (std::int32_t g = 0; g < ng; ++g) {
      GuardP gp;
      gp.rel = take();
      gp.rhs = take();
      if (gp.rel != PCCP_LEQ && gp.rel != PCCP_GT) bad("bad guard relation");
      gp.lhs = expr();
      c.guards.push_back(std::move(gp));
    }
    if (mask & PCCP_FN_SCALAR) c.sc = expr();
    if (mask & PCCP_FN_LB) c.lb = expr();
    if (mask & PCCP_FN_UB) c.ub = expr();
    if (p != end) bad("command " + std::to_string(i) + ": trailing words");
    if (c.kind != PCCP_INTERVAL && !c.sc)
      bad("scalar tell without a scalar expression");  // MonotoneFn::eval, command.cpp:63
    out.push_back(std::move(c));
  }
  return out;
}

bool fits_term(std::int32_t coef, std::uint32_t word) {
  return coef >= -2048 && coef <= 2047 && word <= kTermWordMask;
}
std::int32_t pack(std::int32_t coef, std::uint32_t word) {
  return static_cast<std::int32_t>((static_cast<std::uint32_t>(coef) << kTermWordBits) | word);
}

// Normalised guard: sum tv(c_i, v_i) <= T.  Returns false if not expressible.
//   narrow(k + S) <= rhs  <=>  rhs == +inf || S <= rhs - k
//   narrow(k + S) >  rhs  <=>  rhs != +inf && -S <= k - rhs - 1,  tv(-c, v) = -tv(c, v)
struct NormGuard {
  bool always = false, never = false;
  std::int32_t T = 0;
  std::vector<std::pair<std::int32_t, std::uint32_t>> terms;
};
std::optional<NormGuard> normalise(const GuardP& g) {
  NormGuard n;
  if (g.rhs == INT32_MAX) {
    if (g.rel == PCCP_LEQ) n.always = true;
    else n.never = true;
    return n;
  }
  std::int64_t T;
  if (g.rel == PCCP_LEQ) {
    T = std::int64_t{g.rhs} - g.lhs.k;
    n.terms = g.lhs.terms;
  } else {
    T = std::int64_t{g.lhs.k} - g.rhs - 1;
    for (auto [c, w] : g.lhs.terms) {
      if (c == INT32_MIN) return std::nullopt;
      n.terms.emplace_back(-c, w);
    }
  }
  if (T < INT32_MIN || T > INT32_MAX) return std::nullopt;
  n.T = static_cast<std::int32_t>(T);
  return n;
}

std::uint32_t align4(std::uint32_t x) { return (x + 3u) & ~3u; }

}  // namespace

namespace {
Lowered lower_impl(const pccp_model& m, bool want_bits);
}

Lowered lower_model(const pccp_model& m) { return lower_impl(m, false); }
Lowered lower_packed(const pccp_model& m) { return lower_impl(m, true); }

namespace {

Lowered lower_impl(const pccp_model& m, bool want_bits) {
  if (m.n_slots && (!m.slot_kind || !m.slot_word)) bad("null slot tables");
  if (m.n_cmds && (!m.cmd_off || !m.cmd_code)) bad("null command tables");
  Lowered out;
  DeviceLayout& L = out.L;
  L.n_words = m.n_words;
  L.n_ref_cmds = m.n_cmds;

  // Schema: word directions and owners.
  out.word_up.assign(m.n_words, 0);
  out.slot_of_word.assign(m.n_words, -1);
  std::vector<std::uint8_t> is_lb(m.n_words, 0);
  for (std::uint32_t s = 0; s < m.n_slots; ++s) {
    const std::uint32_t w = m.slot_word[s];
    const int k = m.slot_kind[s];
    if (k < 0 || k > 4) bad("bad slot kind");
    const std::uint32_t span = k == PCCP_INTERVAL ? 2 : 1;
    if (w + span > m.n_words) bad("slot word out of range");
    if (k == PCCP_INTERVAL) {
      out.word_up[w] = 1;
      out.word_up[w + 1] = 0;
      is_lb[w] = 1;
      out.slot_of_word[w] = out.slot_of_word[w + 1] = static_cast<std::int32_t>(s);
    } else {
      out.word_up[w] = (k == PCCP_ZINC || k == PCCP_BINC);
      out.slot_of_word[w] = static_cast<std::int32_t>(s);
    }
  }

  const std::vector<CmdP> cmds = parse(m);

  // Value-range classes of the words (lower.hpp, fast_paths):
  //   0: written only by finite constant tells — holds its entry value or a constant;
  //   1: an interval bound written only by constants and affine tells (k +- one
  //      word whose class is <= 1): NE, reification and precedence tells;
  //   2: anything else (sums, scaled terms, sentinel constants, scalar cells
  //      written affinely, generic code).
  std::vector<std::uint8_t>& cls = out.word_cls;
  cls.assign(m.n_words, 0);
  std::vector<std::vector<std::uint32_t>> aff_src(m.n_words);
  std::vector<std::uint8_t>& read_fast = out.word_read_fast;
  read_fast.assign(m.n_words, 0);
  for (const CmdP& c : cmds) {
    auto part = [&](const std::optional<Expr>& e, std::uint32_t w, bool interval) {
      if (!e || w >= m.n_words) return;
      if (e->terms.empty()) {
        if (e->k == INT32_MIN || e->k == INT32_MAX) cls[w] = 2;
        else out.kconst = std::max(out.kconst, std::abs(std::int64_t{e->k}));
      } else if (interval && e->terms.size() == 1 && std::abs(e->terms[0].first) == 1 &&
                 e->k != INT32_MIN && e->k != INT32_MAX && e->terms[0].second < m.n_words) {
        cls[w] = std::max<std::uint8_t>(cls[w], 1);
        aff_src[w].push_back(e->terms[0].second);
        read_fast[e->terms[0].second] = 1;
        out.kaff = std::max(out.kaff, std::abs(std::int64_t{e->k}));
        ++out.r_aff;
      } else {
        cls[w] = 2;
      }
    };
    if (c.kind == PCCP_INTERVAL) {
      part(c.lb, c.tw, true);
      part(c.ub, c.tw + 1, true);
    } else {
      part(c.sc, c.tw, false);
    }
  }
  for (bool changed = true; changed;) {  // an affine word reading an unbounded word is unbounded
    changed = false;
    for (std::uint32_t w = 0; w < m.n_words; ++w) {
      if (cls[w] != 1) continue;
      for (std::uint32_t src : aff_src[w]) {
        if (cls[src] == 2) {
          cls[w] = 2;
          changed = true;
          break;
        }
      }
    }
  }
  out.word_partner.assign(m.n_words, -1);
  for (std::uint32_t sl = 0; sl < m.n_slots; ++sl) {
    if (m.slot_kind[sl] != PCCP_INTERVAL) continue;
    const std::uint32_t w = m.slot_word[sl];
    out.word_partner[w] = static_cast<std::int32_t>(w + 1);
    out.word_partner[w + 1] = static_cast<std::int32_t>(w);
  }

  // B_alg of SURVEY 8(d): 4*(guard terms) + 4*(fn terms + target words).
  {
    double total = 0;
    for (const CmdP& c : cmds) {
      std::size_t b = 0;
      for (const GuardP& g : c.guards) b += 4 * g.lhs.terms.size();
      if (c.kind == PCCP_INTERVAL) {
        if (c.lb) b += 4 * (c.lb->terms.size() + 1);
        if (c.ub) b += 4 * (c.ub->terms.size() + 1);
      } else {
        b += 4 * (c.sc->terms.size() + 1);
      }
      total += static_cast<double>(b);
    }
    out.alg_bytes_per_eval = cmds.empty() ? 0.0 : total / static_cast<double>(cmds.size());
  }

  // Word reference counts, to prove an lsum cell is private to its row.
  std::vector<std::uint32_t> refs(m.n_words, 0);
  for (const CmdP& c : cmds) {
    ++refs[c.tw];
    for (const GuardP& g : c.guards)
      for (auto& t : g.lhs.terms) ++refs[t.second];
    for (const auto* e : {&c.sc, &c.lb, &c.ub})
      if (*e)
        for (auto& t : (*e)->terms) ++refs[t.second];
  }

  std::vector<std::int32_t> fold_w, fold_v;
  struct Small {
    std::int32_t g[4] = {0, 0, 0, 0};
    std::int32_t T[2] = {INT32_MAX, INT32_MAX};
    std::int32_t lbk = INT32_MIN, lbt = 0, ubk = INT32_MAX, ubt = 0;
    std::int32_t tw = 0;
    std::uint32_t shape = 0;
  };
  std::vector<Small> smalls;
  struct Row {
    std::uint32_t lsum;
    std::int32_t c;
    std::vector<std::int32_t> terms;
  };
  std::vector<Row> rows;
  std::vector<std::uint32_t> generic;

  const bool no_rows = std::getenv("PCCP_NO_ROWS") != nullptr;  // diagnostics: interpret sums
  // compile_sum pattern (propagation.cpp:314-335) starting at command i.
  auto match_row = [&](std::size_t i) -> std::size_t {
    const CmdP& s = cmds[i];
    if (no_rows) return 0;
    if (!s.guards.empty() || s.kind != PCCP_ZINC || !s.sc || s.lb || s.ub || s.sc->k != 0) return 0;
    const auto& terms = s.sc->terms;
    const std::size_t n = terms.size();
    if (n == 0 || i + 2 + n > cmds.size()) return 0;
    const std::uint32_t lw = s.tw;
    for (auto [coef, w] : terms)
      if (coef < 0 || !is_lb[w] || !fits_term(coef, w)) return 0;
    const CmdP& o = cmds[i + 1];  // [lsum > c] => lsum <- +inf
    if (o.target != s.target || o.guards.size() != 1 || !o.sc || o.lb || o.ub) return 0;
    if (o.sc->k != INT32_MAX || !o.sc->terms.empty()) return 0;
    const GuardP& og = o.guards[0];
    if (og.rel != PCCP_GT || og.lhs.k != 0 || og.lhs.terms.size() != 1 || og.lhs.terms[0].first != 1 ||
        og.lhs.terms[0].second != lw)
      return 0;
    const std::int32_t c = og.rhs;
    for (std::size_t t = 0; t < n; ++t) {  // [coef + lsum - coef*lb(x) > c] => x <- (0,0)
      const CmdP& z = cmds[i + 2 + t];
      const auto [coef, w] = terms[t];
      if (z.guards.size() != 1 || z.kind != PCCP_INTERVAL || z.tw != w || z.sc) return 0;
      if (!z.lb || !z.ub || z.lb->k != 0 || z.ub->k != 0 || !z.lb->terms.empty() || !z.ub->terms.empty())
        return 0;
      const GuardP& g = z.guards[0];
      if (g.rel != PCCP_GT || g.rhs != c || g.lhs.k != coef || g.lhs.terms.size() != 2) return 0;
      if (g.lhs.terms[0] != std::make_pair(std::int32_t{1}, lw)) return 0;
      if (coef == INT32_MIN || g.lhs.terms[1] != std::make_pair(-coef, w)) return 0;
    }
    // lsum must be private: 1 + n reads in zero guards, 1 in overload guard,
    // 2 as a target (tell + overload).
    if (refs[lw] != n + 3) return 0;
    Row r;
    r.lsum = lw;
    r.c = c;
    for (auto [coef, w] : terms) r.terms.push_back(pack(coef, w));
    rows.push_back(std::move(r));
    return 2 + n;
  };

  // Unit records (kernels.cuh eval_unit): every guard in the canonical form
  // S[a] - S[b] <= T (an absent term reads the constant-zero word Z =
  // n_words), one bound tell `k +- S[f]` per record; a command telling both
  // bounds becomes two records (same guards, same fixed points).
  const std::uint32_t Z = m.n_words;
  const bool unit_ok = Z < 0x7fffu && !std::getenv("PCCP_NO_UNIT");
  L.zero_word = Z;
  struct U1 {
    std::int32_t x, y, z, w;
  };
  std::vector<U1> unit1;
  std::vector<std::pair<U1, std::pair<std::int32_t, std::int32_t>>> unit2;
  auto unit_guard = [&](const NormGuard& n, std::int32_t& x) {
    std::uint32_t a = Z, b = Z;
    for (auto [coef, w] : n.terms) {
      if (w >= 0xffffu) return false;
      if (coef == 1 && a == Z) a = w;
      else if (coef == -1 && b == Z) b = w;
      else return false;
    }
    x = static_cast<std::int32_t>(a | (b << 16));
    return true;
  };
  auto try_unit = [&](const CmdP& c, const std::vector<NormGuard>& gs) {
    std::int32_t gx[2] = {static_cast<std::int32_t>(Z | (Z << 16)), 0}, gT[2] = {0, 0};
    for (std::size_t k = 0; k < gs.size(); ++k) {
      if (!unit_guard(gs[k], gx[k])) return false;
      gT[k] = gs[k].T;
    }
    std::vector<U1> recs;
    for (int part = 0; part < 2; ++part) {
      const std::optional<Expr>& e = part == 0 ? c.lb : c.ub;
      if (!e) continue;
      const std::uint32_t tw = c.tw + static_cast<std::uint32_t>(part);
      if (tw >= 0x7fffu || e->terms.size() > 1 || e->k <= -(1 << 30) || e->k >= (1 << 30)) return false;
      std::uint32_t f = Z, neg = 0;
      if (e->terms.size() == 1) {
        const auto [coef, w] = e->terms[0];
        if ((coef != 1 && coef != -1) || w >= 0x7fffu) return false;
        f = w;
        neg = coef < 0 ? 1u : 0u;
      }
      recs.push_back(U1{gx[0], gT[0], e->k,
                        static_cast<std::int32_t>(tw | (f << 15) | (neg << 30) | (part == 0 ? 1u << 31 : 0u))});
    }
    for (const U1& r : recs) {
      if (gs.size() <= 1) unit1.push_back(r);
      else unit2.push_back({r, {gx[1], gT[1]}});
    }
    return true;
  };

  // not(and(x + a <= y, y + b <= x)) compiles (propagation.cpp:350-360) to
  //   [ub x - lb y <= -a] => ub x <- ub y + b - 1      [same] => lb y <- lb x + 1 - b
  //   [ub y - lb x <= -b] => ub y <- ub x + a - 1      [same] => lb x <- lb y + 1 - a
  struct NE {
    std::int32_t x, a, b;
  };
  std::vector<NE> nes;
  const bool ne_ok = !std::getenv("PCCP_NO_NE");
  auto match_ne = [&](std::size_t i) -> bool {
    if (!ne_ok || i + 4 > cmds.size()) return false;
    auto guard_of = [](const CmdP& c, std::uint32_t plus, std::uint32_t minus, std::int32_t& rhs) {
      if (c.guards.size() != 1) return false;
      const GuardP& g = c.guards[0];
      if (g.rel != PCCP_LEQ || g.lhs.k != 0 || g.lhs.terms.size() != 2) return false;
      if (g.lhs.terms[0] != std::make_pair(std::int32_t{1}, plus)) return false;
      if (g.lhs.terms[1] != std::make_pair(std::int32_t{-1}, minus)) return false;
      rhs = g.rhs;
      return true;
    };
    auto tell_of = [](const CmdP& c, bool upper, std::uint32_t lbw, std::uint32_t src, std::int64_t& k) {
      if (c.kind != PCCP_INTERVAL || c.tw != lbw || c.sc) return false;
      const std::optional<Expr>& e = upper ? c.ub : c.lb;
      const std::optional<Expr>& other = upper ? c.lb : c.ub;
      if (!e || other || e->terms.size() != 1 || e->terms[0] != std::make_pair(std::int32_t{1}, src)) return false;
      k = e->k;
      return true;
    };
    const std::uint32_t lx = cmds[i].tw, ly = cmds[i + 1].tw;
    if (cmds[i].kind != PCCP_INTERVAL || cmds[i + 1].kind != PCCP_INTERVAL) return false;
    if (lx >= 0xffffu || ly >= 0xffffu) return false;
    std::int32_t r0, r1, r2, r3;
    std::int64_t k0, k1, k2, k3;
    if (!guard_of(cmds[i], lx + 1, ly, r0) || !tell_of(cmds[i], true, lx, ly + 1, k0)) return false;
    if (!guard_of(cmds[i + 1], lx + 1, ly, r1) || r1 != r0 || !tell_of(cmds[i + 1], false, ly, lx, k1)) return false;
    if (!guard_of(cmds[i + 2], ly + 1, lx, r2) || !tell_of(cmds[i + 2], true, ly, lx + 1, k2)) return false;
    if (!guard_of(cmds[i + 3], ly + 1, lx, r3) || r3 != r2 || !tell_of(cmds[i + 3], false, lx, ly, k3)) return false;
    const std::int64_t a = -std::int64_t{r0}, b = -std::int64_t{r2};
    if (k0 != b - 1 || k1 != 1 - b || k2 != a - 1 || k3 != 1 - a) return false;
    const std::int64_t lim = (1 << 30) - 2;
    if (a < -lim || a > lim || b < -lim || b > lim) return false;
    nes.push_back(NE{static_cast<std::int32_t>(lx | (ly << 16)), static_cast<std::int32_t>(a),
                     static_cast<std::int32_t>(b)});
    return true;
  };

  // compile_reified(b, and(x + p <= y, y + q <= x)) (propagation.cpp:415-431,
  // rcpsp.cpp:239-250 with p = 0, q = 1 - d) emits, in order:
  //   [eA, eB] => b <- (1,1)   [nA] => b <- (0,0)   [nB] => b <- (0,0)
  //   [lb b > 0] => ub x <- ub y - p, lb y <- lb x + p, ub y <- ub x - q, lb x <- lb y + q
  //   [ub b <= 0, eA] => ub x <- ub y - (1-q), lb y <- lb x + (1-q)
  //   [ub b <= 0, eB] => ub y <- ub x - (1-p), lb x <- lb y + (1-p)
  // with eA: ub x - lb y <= -p, eB: ub y - lb x <= -q, nA: lb x - ub y > -p, nB: lb y - ub x > -q.
  struct Reif {
    std::int32_t xy, b, p, q;
  };
  std::vector<Reif> reifs;
  const bool reif_ok = !std::getenv("PCCP_NO_REIF");
  auto match_reif = [&](std::size_t i) -> bool {
    if (!reif_ok || i + 11 > cmds.size()) return false;
    using P = std::pair<std::int32_t, std::uint32_t>;
    auto guard2 = [](const GuardP& g, int rel, std::int32_t rhs, P t0, P t1) {
      return g.rel == rel && g.rhs == rhs && g.lhs.k == 0 && g.lhs.terms.size() == 2 && g.lhs.terms[0] == t0 &&
             g.lhs.terms[1] == t1;
    };
    auto guard1 = [](const GuardP& g, int rel, std::uint32_t w) {
      return g.rel == rel && g.rhs == 0 && g.lhs.k == 0 && g.lhs.terms.size() == 1 &&
             g.lhs.terms[0] == P{1, w};
    };
    auto const_b = [](const CmdP& c, std::uint32_t bw, std::int32_t v) {
      return c.kind == PCCP_INTERVAL && c.tw == bw && !c.sc && c.lb && c.ub && c.lb->k == v && c.ub->k == v &&
             c.lb->terms.empty() && c.ub->terms.empty();
    };
    auto tell = [](const CmdP& c, std::uint32_t lbw, bool upper, std::int64_t k, std::uint32_t src) {
      if (c.kind != PCCP_INTERVAL || c.tw != lbw || c.sc) return false;
      const std::optional<Expr>& e = upper ? c.ub : c.lb;
      const std::optional<Expr>& o = upper ? c.lb : c.ub;
      return e && !o && e->k == k && e->terms.size() == 1 && e->terms[0] == P{1, src};
    };
    const CmdP& c0 = cmds[i];
    if (c0.guards.size() != 2 || c0.kind != PCCP_INTERVAL) return false;
    const GuardP& gA = c0.guards[0];
    const GuardP& gB = c0.guards[1];
    if (gA.lhs.terms.size() != 2 || gB.lhs.terms.size() != 2) return false;
    const std::uint32_t ux = gA.lhs.terms[0].second, ly = gA.lhs.terms[1].second;
    if (ux == 0 || ly + 1 >= m.n_words || !is_lb[ux - 1] || !is_lb[ly]) return false;
    const std::uint32_t lx = ux - 1, uy = ly + 1, bw = c0.tw;
    const std::int64_t p = -std::int64_t{gA.rhs}, q = -std::int64_t{gB.rhs};
    const std::int64_t lim = (1 << 29);
    if (p < -lim || p > lim || q < -lim || q > lim) return false;
    if (lx >= 0xffffu || ly >= 0xffffu || bw >= 0xffffu) return false;
    const std::int32_t rp = gA.rhs, rq = gB.rhs;
    if (!guard2(gA, PCCP_LEQ, rp, P{1, ux}, P{-1, ly}) || !guard2(gB, PCCP_LEQ, rq, P{1, uy}, P{-1, lx})) return false;
    if (!const_b(c0, bw, 1)) return false;
    const CmdP &c1 = cmds[i + 1], &c2 = cmds[i + 2];
    if (c1.guards.size() != 1 || !guard2(c1.guards[0], PCCP_GT, rp, P{1, lx}, P{-1, uy}) || !const_b(c1, bw, 0))
      return false;
    if (c2.guards.size() != 1 || !guard2(c2.guards[0], PCCP_GT, rq, P{1, ly}, P{-1, ux}) || !const_b(c2, bw, 0))
      return false;
    for (int k = 3; k <= 6; ++k) {
      const CmdP& c = cmds[i + k];
      if (c.guards.size() != 1 || !guard1(c.guards[0], PCCP_GT, bw)) return false;
    }
    if (!tell(cmds[i + 3], lx, true, -p, uy) || !tell(cmds[i + 4], ly, false, p, lx) ||
        !tell(cmds[i + 5], ly, true, -q, ux) || !tell(cmds[i + 6], lx, false, q, ly))
      return false;
    for (int k = 7; k <= 10; ++k) {
      const CmdP& c = cmds[i + k];
      if (c.guards.size() != 2 || !guard1(c.guards[0], PCCP_LEQ, bw + 1)) return false;
      const GuardP& g = c.guards[1];
      if (k <= 8 ? !guard2(g, PCCP_LEQ, rp, P{1, ux}, P{-1, ly}) : !guard2(g, PCCP_LEQ, rq, P{1, uy}, P{-1, lx}))
        return false;
    }
    if (!tell(cmds[i + 7], lx, true, -(1 - q), uy) || !tell(cmds[i + 8], ly, false, 1 - q, lx) ||
        !tell(cmds[i + 9], ly, true, -(1 - p), ux) || !tell(cmds[i + 10], lx, false, 1 - p, ly))
      return false;
    reifs.push_back(Reif{static_cast<std::int32_t>(lx | (ly << 16)), static_cast<std::int32_t>(bw),
                         static_cast<std::int32_t>(p), static_cast<std::int32_t>(q)});
    return true;
  };

  for (std::size_t i = 0; i < cmds.size();) {
    if (match_reif(i)) {
      i += 11;
      continue;
    }
    if (match_ne(i)) {
      i += 4;
      continue;
    }
    if (const std::size_t used = match_row(i)) {
      i += used;
      continue;
    }
    const CmdP& c = cmds[i];
    // fold: unguarded constant tells
    bool constant = c.guards.empty();
    for (const auto* e : {&c.sc, &c.lb, &c.ub})
      if (*e && !(*e)->terms.empty()) constant = false;
    if (constant) {
      if (c.kind == PCCP_INTERVAL) {
        if (c.lb) { fold_w.push_back(static_cast<std::int32_t>(c.tw | 0x80000000u)); fold_v.push_back(c.lb->k); }
        if (c.ub) { fold_w.push_back(static_cast<std::int32_t>(c.tw + 1)); fold_v.push_back(c.ub->k); }
      } else {
        fold_w.push_back(static_cast<std::int32_t>(c.tw | (out.word_up[c.tw] ? 0x80000000u : 0u)));
        fold_v.push_back(c.sc->k);
      }
      ++i;
      continue;
    }
    // small: interval target, <= 2 guards of <= 2 terms, <= 1 term per bound
    bool ok = c.kind == PCCP_INTERVAL && c.guards.size() <= 2 && c.tw + 1 <= kTermWordMask;
    Small s;
    bool never = false;
    int ng = 0;
    std::uint32_t shape = 0;
    std::vector<NormGuard> kept;
    if (ok) {
      for (const GuardP& g : c.guards) {
        auto n = normalise(g);
        if (!n || n->terms.size() > 2) { ok = false; break; }
        if (n->never) { never = true; break; }
        if (n->always) continue;
        for (std::size_t t = 0; t < n->terms.size(); ++t) {
          if (!fits_term(n->terms[t].first, n->terms[t].second)) { ok = false; break; }
          s.g[2 * ng + t] = pack(n->terms[t].first, n->terms[t].second);
        }
        s.T[ng] = n->T;
        shape |= static_cast<std::uint32_t>(n->terms.size()) << (4 * ng);
        kept.push_back(*n);
        ++ng;
      }
    }
    if (never) {  // can never fire: dropped (still counted as a reference command)
      ++out.n_dropped;
      ++i;
      continue;
    }
    if (ok && unit_ok && try_unit(c, kept)) {
      ++i;
      continue;
    }
    if (ok) {
      for (const auto* e : {&c.lb, &c.ub}) {
        if (*e && ((*e)->terms.size() > 1 ||
                   ((*e)->terms.size() == 1 && !fits_term((*e)->terms[0].first, (*e)->terms[0].second))))
          ok = false;
      }
    }
    if (!ok) {
      generic.push_back(static_cast<std::uint32_t>(i));
      ++i;
      continue;
    }
    if (c.lb) {
      s.lbk = c.lb->k;
      if (!c.lb->terms.empty()) s.lbt = pack(c.lb->terms[0].first, c.lb->terms[0].second);
      shape |= 1u << 8 | (c.lb->terms.empty() ? 0u : 1u << 9);
    }
    if (c.ub) {
      s.ubk = c.ub->k;
      if (!c.ub->terms.empty()) s.ubt = pack(c.ub->terms[0].first, c.ub->terms[0].second);
      shape |= 1u << 10 | (c.ub->terms.empty() ? 0u : 1u << 11);
    }
    s.tw = static_cast<std::int32_t>(c.tw);
    s.shape = shape | static_cast<std::uint32_t>(ng) << 12;
    smalls.push_back(s);
    ++i;
  }
  // Group shapes so a warp walks a homogeneous segment (fewer divergent paths).
  std::stable_sort(smalls.begin(), smalls.end(), [](const Small& a, const Small& b) { return a.shape < b.shape; });

  // ---- bit-plane 0/1 cells (lower_packed, lower.hpp) -----------------------------
  const std::uint32_t NW = m.n_words;
  std::vector<std::int32_t> bitof(NW, -1);  // lb word of a packed slot -> its bit
  std::vector<std::uint8_t> brow(rows.size(), 0);  // rows over packed cells only
  std::uint32_t n_bits = 0;
  std::vector<std::int32_t> flb(NW, INT32_MIN), fub(NW, INT32_MAX);  // folded constants per word
  bool packed = false;
  if (want_bits && !std::getenv("PCCP_NO_PACK")) {
    std::vector<std::uint8_t> other(NW, 0), fold_bad(NW, 0);
    auto touch = [&](std::uint32_t w) {
      if (w < NW) other[w] = 1;
    };
    auto touch_iv = [&](std::uint32_t w) {
      touch(w);
      touch(w + 1);
    };
    for (const NE& e : nes) {
      touch_iv(static_cast<std::uint32_t>(e.x) & 0xffffu);
      touch_iv(static_cast<std::uint32_t>(e.x) >> 16);
    }
    for (const Reif& r : reifs) {
      touch_iv(static_cast<std::uint32_t>(r.xy) & 0xffffu);
      touch_iv(static_cast<std::uint32_t>(r.xy) >> 16);
    }
    auto touch_unit = [&](const U1& r) {
      const std::uint32_t x = static_cast<std::uint32_t>(r.x), w = static_cast<std::uint32_t>(r.w);
      touch(x & 0xffffu);
      touch(x >> 16);
      touch(w & 0x7fffu);
      touch((w >> 15) & 0x7fffu);
    };
    for (const U1& r : unit1) touch_unit(r);
    for (const auto& r : unit2) {
      touch_unit(r.first);
      touch(static_cast<std::uint32_t>(r.second.first) & 0xffffu);
      touch(static_cast<std::uint32_t>(r.second.first) >> 16);
    }
    auto tw_of = [](std::int32_t t) { return static_cast<std::uint32_t>(t) & kTermWordMask; };
    for (const Small& s : smalls) {
      for (int k = 0; k < 4; ++k)
        if (s.g[k]) touch(tw_of(s.g[k]));
      if (s.lbt) touch(tw_of(s.lbt));
      if (s.ubt) touch(tw_of(s.ubt));
      touch_iv(static_cast<std::uint32_t>(s.tw));
    }
    for (std::uint32_t gi : generic) {
      const CmdP& c = cmds[gi];
      touch(c.tw);
      if (c.kind == PCCP_INTERVAL) touch(c.tw + 1);
      for (const GuardP& g : c.guards)
        for (auto& t : g.lhs.terms) touch(t.second);
      for (const auto* e : {&c.sc, &c.lb, &c.ub})
        if (*e)
          for (auto& t : (*e)->terms) touch(t.second);
    }
    for (const Row& r : rows) touch(r.lsum);
    if (m.n_cands == 0) {  // every interval slot is a candidate: nothing packs
      std::fill(other.begin(), other.end(), 1);
    } else if (m.cands) {
      for (std::uint32_t i = 0; i < m.n_cands; ++i) {
        const std::int32_t s = m.cands[i];
        if (s >= 0 && static_cast<std::uint32_t>(s) < m.n_slots) touch_iv(m.slot_word[s]);
      }
    }
    if (m.obj_slot >= 0 && static_cast<std::uint32_t>(m.obj_slot) < m.n_slots) touch_iv(m.slot_word[m.obj_slot]);
    for (std::size_t i = 0; i < fold_w.size(); ++i) {
      const std::uint32_t w = static_cast<std::uint32_t>(fold_w[i]) & 0x7fffffffu;
      const std::int32_t v = fold_v[i];
      if (w >= NW) continue;
      if (v != 0 && v != 1) fold_bad[w] = 1;
      if (fold_w[i] < 0) {
        if (is_lb[w]) flb[w] = std::max(flb[w], v);
        else other[w] = 1;  // an up scalar
      } else if (w > 0 && is_lb[w - 1]) {
        fub[w] = std::min(fub[w], v);
      } else {
        other[w] = 1;
      }
    }
    std::vector<std::uint8_t> pk(NW, 0);  // lb words of packable slots
    for (std::uint32_t s = 0; s < m.n_slots; ++s) {
      if (m.slot_kind[s] != PCCP_INTERVAL) continue;
      const std::uint32_t w = m.slot_word[s];
      pk[w] = !other[w] && !other[w + 1] && !fold_bad[w] && !fold_bad[w + 1] && flb[w] != INT32_MIN &&
              fub[w + 1] != INT32_MAX;
    }
    // A row sums packed bits only if every term is packed (else it stays a
    // word row and its terms stay words); its bit sum must fit 2^29.
    for (bool ch = true; ch;) {
      ch = false;
      for (const Row& r : rows) {
        std::size_t cnt = 0;
        std::int64_t sum = 0;
        for (std::int32_t x : r.terms) {
          cnt += pk[tw_of(x)] ? 1 : 0;
          sum += std::abs(std::int64_t{x >> kTermWordBits});
        }
        if (cnt && (cnt < r.terms.size() || sum >= (1 << 29) || r.c <= -(1 << 30) || (r.c >= (1 << 30) && r.c != INT32_MAX))) {
          for (std::int32_t x : r.terms)
            if (pk[tw_of(x)]) {
              pk[tw_of(x)] = 0;
              ch = true;
            }
        }
      }
    }
    bool all_reif = true;
    for (const Reif& r : reifs) all_reif &= pk[static_cast<std::uint32_t>(r.b)] != 0;
    std::size_t n_pk = 0;
    for (std::uint32_t w = 0; w < NW; ++w) n_pk += pk[w];
    packed = all_reif && n_pk > 0 && n_pk < (1u << 20);
    if (packed) {
      // Bit order: cells summed by the same rows are neighbours (union-find
      // over each row's terms; RCPSP: one column b_{., j} per component), so a
      // row reads a few consecutive plane words.  Components in order of first
      // appearance in the rows, cells by reference word inside a component.
      std::vector<std::int32_t> par(NW, -1);
      std::function<std::int32_t(std::int32_t)> find = [&](std::int32_t w) {
        while (par[w] != w) w = par[w] = par[par[w]];
        return w;
      };
      for (std::uint32_t w = 0; w < NW; ++w)
        if (pk[w]) par[w] = static_cast<std::int32_t>(w);
      for (std::size_t r = 0; r < rows.size(); ++r) {
        if (rows[r].terms.empty() || !pk[tw_of(rows[r].terms[0])]) continue;
        brow[r] = 1;
        const std::int32_t a = find(static_cast<std::int32_t>(tw_of(rows[r].terms[0])));
        for (std::int32_t x : rows[r].terms) {
          const std::int32_t b = find(static_cast<std::int32_t>(tw_of(x)));
          if (a != b) par[b] = a;
        }
      }
      // reifications of one y join their cells' components too (RCPSP: a
      // task that uses no resource has no row terms, but its b_{i,j} belongs
      // to column j), so the records of one y are one range of bits
      // (filtered rounds: lower.cpp r_y)
      {
        std::map<std::uint32_t, std::int32_t> first_of_y;
        for (const Reif& r : reifs) {
          const std::uint32_t y = static_cast<std::uint32_t>(r.xy) >> 16;
          const std::int32_t b = find(r.b);
          auto it = first_of_y.find(y);
          if (it == first_of_y.end()) {
            first_of_y.emplace(y, b);
          } else {
            const std::int32_t a = find(it->second);
            if (a != b) par[b] = a;
          }
        }
      }
      std::vector<std::int64_t> rank(NW, -1);
      std::int64_t next = 0;
      for (std::size_t r = 0; r < rows.size(); ++r)
        if (brow[r])
          for (std::int32_t x : rows[r].terms) {
            const std::int32_t c = find(static_cast<std::int32_t>(tw_of(x)));
            if (rank[c] < 0) rank[c] = next++;
          }
      std::vector<std::uint32_t> order;
      for (std::uint32_t w = 0; w < NW; ++w)
        if (pk[w]) {
          const std::int32_t c = find(static_cast<std::int32_t>(w));
          if (rank[c] < 0) rank[c] = next++;
          order.push_back(w);
        }
      std::stable_sort(order.begin(), order.end(), [&](std::uint32_t a, std::uint32_t b) {
        return rank[find(static_cast<std::int32_t>(a))] < rank[find(static_cast<std::int32_t>(b))];
      });
      for (std::uint32_t w : order) bitof[w] = static_cast<std::int32_t>(n_bits++);
    }
  }
  // Reference word -> device word (packed cells: -1), and the device zero word.
  std::vector<std::int32_t> dmap(NW, -1);
  std::uint32_t n_int = 0;
  for (std::uint32_t w = 0; w < NW; ++w) {
    const bool in_bits = bitof[w] >= 0 || (w > 0 && bitof[w - 1] >= 0 && is_lb[w - 1]);
    if (!in_bits) dmap[w] = static_cast<std::int32_t>(n_int++);
  }
  const std::uint32_t n_pairs = (n_bits + 31) / 32;
  const std::uint32_t plane = packed ? (n_int + 1) & ~1u : n_int;
  // + one zero pair after the planes: a row's 32-bit window may read the
  // pair after its last bit (eval_wrows)
  const std::uint32_t DW = packed ? plane + 2 * n_pairs + 2 : NW;  // device store words
  out.dev_words = DW;
  auto W = [&](std::uint32_t w) -> std::uint32_t {  // device word of a reference word (Z -> the device Z)
    if (w >= NW) return DW;
    if (dmap[w] < 0) bad("internal: a packed cell read as a word");
    return static_cast<std::uint32_t>(dmap[w]);
  };
  auto WT = [&](std::int32_t t) -> std::int32_t {  // a packed term (coef << 20 | word), 0 = none
    if (!t) return 0;
    return static_cast<std::int32_t>((static_cast<std::uint32_t>(t) & ~kTermWordMask) |
                                     W(static_cast<std::uint32_t>(t) & kTermWordMask));
  };
  if (packed) {
    L.packed = 1;
    L.plane = plane;
    L.n_pairs = n_pairs;
    L.ref_words = NW;
    L.n_words = DW;
    L.zero_word = DW;
    for (NE& e : nes) e.x = static_cast<std::int32_t>(W(e.x & 0xffff) | (W(static_cast<std::uint32_t>(e.x) >> 16) << 16));
    for (Reif& r : reifs) {
      r.xy = static_cast<std::int32_t>(W(r.xy & 0xffff) | (W(static_cast<std::uint32_t>(r.xy) >> 16) << 16));
      r.b = bitof[static_cast<std::uint32_t>(r.b)];
    }
    auto unit_map = [&](U1& r) {
      const std::uint32_t x = static_cast<std::uint32_t>(r.x), w = static_cast<std::uint32_t>(r.w);
      r.x = static_cast<std::int32_t>(W(x & 0xffffu) | (W(x >> 16) << 16));
      r.w = static_cast<std::int32_t>((w & 0xc0000000u) | W(w & 0x7fffu) | (W((w >> 15) & 0x7fffu) << 15));
    };
    for (U1& r : unit1) unit_map(r);
    for (auto& r : unit2) {
      unit_map(r.first);
      const std::uint32_t g2 = static_cast<std::uint32_t>(r.second.first);
      r.second.first = static_cast<std::int32_t>(W(g2 & 0xffffu) | (W(g2 >> 16) << 16));
    }
    for (Small& s : smalls) {
      for (int k = 0; k < 4; ++k) s.g[k] = WT(s.g[k]);
      s.lbt = WT(s.lbt);
      s.ubt = WT(s.ubt);
      s.tw = static_cast<std::int32_t>(W(static_cast<std::uint32_t>(s.tw)));
    }
    for (std::size_t r = 0; r < rows.size(); ++r) {
      rows[r].lsum = W(rows[r].lsum);
      if (!brow[r])
        for (std::int32_t& x : rows[r].terms) x = WT(x);
    }
    // device folds: word cells only (the packed cells' folds are applied by to_device)
    std::vector<std::int32_t> fw2, fv2;
    for (std::size_t i = 0; i < fold_w.size(); ++i) {
      const std::uint32_t w = static_cast<std::uint32_t>(fold_w[i]) & 0x7fffffffu;
      if (w < NW && dmap[w] < 0) continue;
      fw2.push_back(static_cast<std::int32_t>((static_cast<std::uint32_t>(fold_w[i]) & 0x80000000u) | W(w)));
      fv2.push_back(fold_v[i]);
    }
    fold_w.swap(fw2);
    fold_v.swap(fv2);
    out.bit_lbw.assign(n_bits, 0);
    out.bit_fold_lb.assign(n_bits, 0);
    out.bit_fold_ub.assign(n_bits, 1);
    for (std::uint32_t w = 0; w < NW; ++w)
      if (bitof[w] >= 0) {
        out.bit_lbw[static_cast<std::uint32_t>(bitof[w])] = static_cast<std::int32_t>(w);
        out.bit_fold_lb[static_cast<std::uint32_t>(bitof[w])] = flb[w];
        out.bit_fold_ub[static_cast<std::uint32_t>(bitof[w])] = fub[w + 1];
      }
    out.dec.assign(NW, 0);
    for (std::uint32_t w = 0; w < NW; ++w) {
      if (dmap[w] >= 0) out.dec[w] = dmap[w];
      else if (bitof[w] >= 0) out.dec[w] = -1 - 2 * bitof[w];
      else out.dec[w] = -1 - (2 * bitof[w - 1] + 1);
    }
  }

  // ---- blob ----------------------------------------------------------------------
  std::vector<std::int32_t>& B = out.blob;
  auto reserve_arr = [&B](std::uint32_t n) {
    const std::uint32_t off = align4(static_cast<std::uint32_t>(B.size()));
    B.resize(off + n, 0);
    return off;
  };
  // Record order within a round: the records of one variable pair (compile
  // order keeps them adjacent: not(x = y + d) for d = 0, j - i, i - j in
  // N-Queens) are spread apart, k-th record of every pair first, so a later
  // record sees what an earlier one of its pair joined in the same round
  // instead of reading the same snapshot in the same warp instruction
  // (Q14: 56.3 -> 50.2 M rounds).  Any order reaches the same fixed point.
  {
    const char* o = std::getenv("PCCP_NE_ORDER");
    const int mode = o ? std::atoi(o) : 2;
    if (mode >= 1) {
      std::map<std::int32_t, int> seen;
      std::vector<std::pair<int, std::size_t>> key(nes.size());
      for (std::size_t i = 0; i < nes.size(); ++i) key[i] = {seen[nes[i].x]++, i};
      std::vector<std::size_t> idx(nes.size());
      for (std::size_t i = 0; i < idx.size(); ++i) idx[i] = i;
      // ties: by the distance of the two lb words (measured on Q14: 50.2 -> 49.0 M rounds)
      auto dist = [&](std::size_t i) {
        return std::abs((long)(nes[i].x & 0xffff) - (long)((unsigned)nes[i].x >> 16));
      };
      std::stable_sort(idx.begin(), idx.end(), [&](std::size_t a2, std::size_t b2) {
        if (key[a2].first != key[b2].first) return key[a2].first < key[b2].first;
        return dist(a2) < dist(b2);
      });
      std::vector<NE> t;
      for (std::size_t i : idx) t.push_back(nes[i]);
      if (mode == 2) std::reverse(t.begin(), t.end());
      nes = t;
    }
  }
  L.n_ne = static_cast<std::uint32_t>(nes.size());
  L.ne = reserve_arr(4 * L.n_ne);
  L.ne_even = 1;
  for (std::uint32_t i = 0; i < L.n_ne; ++i) {  // {4 lbx, a - 1, b - 1, 4 lby}: byte offsets into the store
    const std::uint32_t lx = static_cast<std::uint32_t>(nes[i].x) & 0xffffu, ly = static_cast<std::uint32_t>(nes[i].x) >> 16;
    B[L.ne + 4 * i + 0] = static_cast<std::int32_t>(4 * lx);
    B[L.ne + 4 * i + 1] = nes[i].a - 1;
    B[L.ne + 4 * i + 2] = nes[i].b - 1;
    B[L.ne + 4 * i + 3] = static_cast<std::int32_t>(4 * ly);
    if ((lx | ly) & 1u) L.ne_even = 0;
  }
  // Order the reifications x-major: a warp then reads one x (broadcast) and
  // consecutive y / b words (2-way bank conflicts).  RCPSP compiles them
  // j-major (rcpsp.cpp:241-242), which puts b_ij of a warp n words apart —
  // the same bank for every lane when n = 32.
  // Packed: by bit instead (y-major, RCPSP's compile order): a warp's b
  // cells then share one plane pair (a broadcast) and x varies by word.
  std::stable_sort(reifs.begin(), reifs.end(), [packed](const Reif& a, const Reif& b) {
    if (packed) return a.b < b.b;
    const std::uint32_t ax = static_cast<std::uint32_t>(a.xy) & 0xffffu, bx = static_cast<std::uint32_t>(b.xy) & 0xffffu;
    if (ax != bx) return ax < bx;
    return (static_cast<std::uint32_t>(a.xy) >> 16) < (static_cast<std::uint32_t>(b.xy) >> 16);
  });
  L.n_reif = static_cast<std::uint32_t>(reifs.size());
  // Packed layouts: 8-byte records {lx | ly << 16, bit | p << 18 | q << 25}
  // (7-bit signed p, q; RCPSP: p = 0, q = 1 - d) when every record fits.
  L.reif8 = packed ? 1u : 0u;
  for (const Reif& r : reifs)
    if (r.b < 0 || r.b >= (1 << 18) || r.p < -64 || r.p > 63 || r.q < -64 || r.q > 63) L.reif8 = 0;
  if (std::getenv("PCCP_NO_REIF8")) L.reif8 = 0;
  L.reif = reserve_arr((L.reif8 ? 2 : 4) * L.n_reif);
  for (std::uint32_t i = 0; i < L.n_reif; ++i) {
    if (L.reif8) {
      B[L.reif + 2 * i + 0] = reifs[i].xy;
      B[L.reif + 2 * i + 1] = static_cast<std::int32_t>(static_cast<std::uint32_t>(reifs[i].b) |
                                                        ((static_cast<std::uint32_t>(reifs[i].p) & 0x7fu) << 18) |
                                                        ((static_cast<std::uint32_t>(reifs[i].q) & 0x7fu) << 25));
      continue;
    }
    B[L.reif + 4 * i + 0] = reifs[i].xy;
    B[L.reif + 4 * i + 1] = reifs[i].b;
    B[L.reif + 4 * i + 2] = reifs[i].p;
    B[L.reif + 4 * i + 3] = reifs[i].q;
  }
  // Segments of the filtered kPacked rounds (kernels.cuh packed_round): the
  // records that read start k as y (a contiguous range: records are sorted by
  // b's bit, and a component of bits is one y), as x (CSR of record indices),
  // and the records whose b lies in plane word p (a range).
  if (packed && L.reif8 && L.n_reif) {
    std::uint32_t ns = 0;
    for (const Reif& r : reifs)
      ns = std::max({ns, ((static_cast<std::uint32_t>(r.xy) & 0xffffu) >> 1) + 1,
                     ((static_cast<std::uint32_t>(r.xy) >> 16) >> 1) + 1});
    std::vector<std::int32_t> yb(ns, 0), ye(ns, 0), xoff(ns + 1, 0), xrec(L.n_reif), pb(n_pairs + 1, 0);
    std::vector<std::uint8_t> seen(ns, 0);
    bool contiguous = true;
    for (std::uint32_t i = 0; i < L.n_reif; ++i) {
      const std::uint32_t ky = (static_cast<std::uint32_t>(reifs[i].xy) >> 16) >> 1;
      if (!seen[ky]) {
        seen[ky] = 1;
        yb[ky] = ye[ky] = static_cast<std::int32_t>(i);
      } else if (ye[ky] != static_cast<std::int32_t>(i)) {
        contiguous = false;
      }
      ye[ky] = static_cast<std::int32_t>(i + 1);
      ++xoff[((static_cast<std::uint32_t>(reifs[i].xy) & 0xffffu) >> 1) + 1];
    }
    for (std::uint32_t k = 0; k < ns; ++k) xoff[k + 1] += xoff[k];
    {
      std::vector<std::int32_t> fill(xoff.begin(), xoff.end() - 1);
      for (std::uint32_t i = 0; i < L.n_reif; ++i)
        xrec[static_cast<std::uint32_t>(fill[(static_cast<std::uint32_t>(reifs[i].xy) & 0xffffu) >> 1]++)] =
            static_cast<std::int32_t>(i);
    }
    for (std::uint32_t p = 0, i = 0; p <= n_pairs; ++p) {
      while (i < L.n_reif && static_cast<std::uint32_t>(reifs[i].b) < 32 * p) ++i;
      pb[p] = static_cast<std::int32_t>(i);
    }
    pb[n_pairs] = static_cast<std::int32_t>(L.n_reif);
    if (contiguous) {
      L.rfilt = 1;
      L.r_ns = ns;
      L.r_y = reserve_arr(2 * ns);
      L.r_xoff = reserve_arr(ns + 1);
      L.r_xrec = reserve_arr(L.n_reif);
      L.r_p = reserve_arr(n_pairs + 1);
      for (std::uint32_t k = 0; k < ns; ++k) {
        B[L.r_y + 2 * k] = yb[k];
        B[L.r_y + 2 * k + 1] = ye[k];
      }
      std::copy(xoff.begin(), xoff.end(), B.begin() + L.r_xoff);
      std::copy(xrec.begin(), xrec.end(), B.begin() + L.r_xrec);
      std::copy(pb.begin(), pb.end(), B.begin() + L.r_p);
    }
  }
  L.n_unit1 = static_cast<std::uint32_t>(unit1.size());
  L.unit1 = reserve_arr(4 * L.n_unit1);
  for (std::uint32_t i = 0; i < L.n_unit1; ++i) {
    const U1& r = unit1[i];
    B[L.unit1 + 4 * i + 0] = r.x;
    B[L.unit1 + 4 * i + 1] = r.y;
    B[L.unit1 + 4 * i + 2] = r.z;
    B[L.unit1 + 4 * i + 3] = r.w;
  }
  L.n_unit2 = static_cast<std::uint32_t>(unit2.size());
  L.unit2 = reserve_arr(4 * L.n_unit2);
  L.unit2g = reserve_arr(2 * L.n_unit2);
  for (std::uint32_t i = 0; i < L.n_unit2; ++i) {
    const U1& r = unit2[i].first;
    B[L.unit2 + 4 * i + 0] = r.x;
    B[L.unit2 + 4 * i + 1] = r.y;
    B[L.unit2 + 4 * i + 2] = r.z;
    B[L.unit2 + 4 * i + 3] = r.w;
    B[L.unit2g + 2 * i + 0] = unit2[i].second.first;
    B[L.unit2g + 2 * i + 1] = unit2[i].second.second;
  }
  // Per-word reader lists for the filtered rounds (opt-in, PCCP_FILTERED=1:
  // with fused NE records the eventless loop needs ~30% fewer rounds and wins).
  L.filtered = (!packed && m.n_words <= 64 && smalls.empty() && rows.empty() && generic.empty() && reifs.empty() &&
                std::getenv("PCCP_FILTERED") != nullptr)
                   ? 1u
                   : 0u;
  {
    std::vector<std::vector<std::int32_t>> readers(m.n_words);
    auto note = [&](std::int32_t entry, std::uint32_t x, std::uint32_t w) {
      std::uint32_t ws[3] = {x & 0xffffu, x >> 16, (w >> 15) & 0x7fffu};
      for (int k = 0; k < 3; ++k) {
        if (ws[k] >= m.n_words) continue;  // the zero word never changes
        bool dup = false;
        for (int j = 0; j < k; ++j) dup |= ws[j] == ws[k];
        if (!dup) readers[ws[k]].push_back(entry);
      }
    };
    if (L.filtered) {
      for (std::uint32_t i = 0; i < unit1.size(); ++i)
        note(static_cast<std::int32_t>(i), static_cast<std::uint32_t>(unit1[i].x), static_cast<std::uint32_t>(unit1[i].w));
      for (std::uint32_t i = 0; i < unit2.size(); ++i) {
        const std::int32_t e = static_cast<std::int32_t>(i | 0x80000000u);
        note(e, static_cast<std::uint32_t>(unit2[i].first.x), static_cast<std::uint32_t>(unit2[i].first.w));
        const std::uint32_t g2 = static_cast<std::uint32_t>(unit2[i].second.first);
        for (std::uint32_t w2 : {g2 & 0xffffu, g2 >> 16}) {
          if (w2 >= m.n_words) continue;
          if (readers[w2].empty() || readers[w2].back() != e) readers[w2].push_back(e);
        }
      }
      for (std::uint32_t i = 0; i < nes.size(); ++i) {  // entry tag 01: fused not(and)
        const std::int32_t e = static_cast<std::int32_t>(i | 0x40000000u);
        const std::uint32_t lx = static_cast<std::uint32_t>(nes[i].x) & 0xffffu;
        const std::uint32_t ly = static_cast<std::uint32_t>(nes[i].x) >> 16;
        for (std::uint32_t w : {lx, lx + 1, ly, ly + 1})
          if (readers[w].empty() || readers[w].back() != e) readers[w].push_back(e);
      }
    }
    std::uint32_t total = 0;
    for (const auto& r : readers) total += static_cast<std::uint32_t>(r.size());
    L.wl_off = reserve_arr(L.filtered ? m.n_words + 1 : 1);
    L.wl = reserve_arr(total);
    std::uint32_t p = 0;
    if (L.filtered) {
      for (std::uint32_t w = 0; w < m.n_words; ++w) {
        B[L.wl_off + w] = static_cast<std::int32_t>(p);
        for (std::int32_t e : readers[w]) B[L.wl + p++] = e;
      }
      B[L.wl_off + m.n_words] = static_cast<std::int32_t>(p);
    }
  }
  const std::uint32_t ns = static_cast<std::uint32_t>(smalls.size());
  L.n_small = ns;
  for (int k = 0; k < 4; ++k) L.small_g[k] = reserve_arr(ns);
  for (int k = 0; k < 2; ++k) L.small_T[k] = reserve_arr(ns);
  L.small_lbk = reserve_arr(ns);
  L.small_lbt = reserve_arr(ns);
  L.small_ubk = reserve_arr(ns);
  L.small_ubt = reserve_arr(ns);
  L.small_tw = reserve_arr(ns);
  for (std::uint32_t i = 0; i < ns; ++i) {
    const Small& s = smalls[i];
    for (int k = 0; k < 4; ++k) B[L.small_g[k] + i] = s.g[k];
    for (int k = 0; k < 2; ++k) B[L.small_T[k] + i] = s.T[k];
    B[L.small_lbk + i] = s.lbk;
    B[L.small_lbt + i] = s.lbt;
    B[L.small_ubk + i] = s.ubk;
    B[L.small_ubt + i] = s.ubt;
    B[L.small_tw + i] = s.tw;
  }
  std::vector<Row> bit_rows;  // packed: rows over bit cells
  if (packed) {
    std::vector<Row> word_rows;
    for (std::size_t r = 0; r < rows.size(); ++r) (brow[r] ? bit_rows : word_rows).push_back(std::move(rows[r]));
    rows.swap(word_rows);
  }
  L.n_rows = static_cast<std::uint32_t>(rows.size());
  std::uint32_t n_terms = 0, max_terms = 0;
  for (const Row& r : rows) {
    n_terms += static_cast<std::uint32_t>(r.terms.size());
    max_terms = std::max<std::uint32_t>(max_terms, static_cast<std::uint32_t>(r.terms.size()));
  }
  L.n_row_terms = n_terms;
  // ~8 terms per lane: few lanes per row keeps a warp's loads on many rows of
  // consecutive words (kernels.cuh eval_rows) at a modest serial cost.
  L.row_lanes = 1;
  while (L.row_lanes < 32 && L.row_lanes * 8 < max_terms) L.row_lanes <<= 1;
  if (const char* rl = std::getenv("PCCP_ROW_LANES")) {
    const unsigned v = static_cast<unsigned>(std::atoi(rl));
    if (v >= 1 && v <= 32 && (v & (v - 1)) == 0) L.row_lanes = v;
  }
  L.row_lg = 0;
  while ((1u << L.row_lg) < L.row_lanes) ++L.row_lg;
  L.row_tl = (max_terms + L.row_lanes - 1) / L.row_lanes;
  L.row_off = reserve_arr(L.n_rows + 1);
  L.row_lsum = reserve_arr(L.n_rows);
  L.row_c = reserve_arr(L.n_rows);
  L.row_terms = reserve_arr(n_terms);
  {
    std::uint32_t t = 0;
    for (std::uint32_t r = 0; r < L.n_rows; ++r) {
      B[L.row_off + r] = static_cast<std::int32_t>(t);
      B[L.row_lsum + r] = static_cast<std::int32_t>(rows[r].lsum);
      B[L.row_c + r] = rows[r].c;
      for (std::int32_t x : rows[r].terms) B[L.row_terms + t++] = x;
    }
    B[L.row_off + L.n_rows] = static_cast<std::int32_t>(t);
    // Paired (lb, ub) loads pay when neighbouring lanes read neighbouring
    // intervals (RCPSP: term k of rows t and t+1 is b_{i,t}, b_{i,t+1}); on
    // scattered terms (random CSP) the 8-byte loads only add bank conflicts.
    L.row_even = 1;
    std::uint64_t contig = 0;
    auto tw = [](std::int32_t x) { return static_cast<std::uint32_t>(x) & kTermWordMask; };
    for (std::size_t r = 0; r < rows.size(); ++r) {
      const auto& ts = rows[r].terms;
      for (std::size_t k = 0; k < ts.size(); ++k) {
        if ((tw(ts[k]) & 1u) || tw(ts[k]) + 1 >= DW) L.row_even = 0;
        if (k + 1 < ts.size() && tw(ts[k + 1]) == tw(ts[k]) + 2) ++contig;
        if (r + 1 < rows.size() && rows[r + 1].terms.size() == ts.size() && tw(rows[r + 1].terms[k]) == tw(ts[k]) + 2)
          ++contig;
      }
    }
    if (2 * contig < t) L.row_even = 0;
    if (std::getenv("PCCP_ROW_PAIR") && std::atoi(std::getenv("PCCP_ROW_PAIR")) == 0) L.row_even = 0;
    // the same per row as one int4 {first term, end, c, lsum word} (eval_rows_fast)
    L.row_meta = reserve_arr(4 * L.n_rows);
    for (std::uint32_t r = 0; r < L.n_rows; ++r) {
      B[L.row_meta + 4 * r + 0] = B[L.row_off + r];
      B[L.row_meta + 4 * r + 1] = B[L.row_off + r + 1];
      B[L.row_meta + 4 * r + 2] = rows[r].c;
      B[L.row_meta + 4 * r + 3] = static_cast<std::int32_t>(rows[r].lsum);
    }
  }
  // Bit rows: each row's terms as offsets from its first bit; rows with the
  // same (coef, offset) list share one pattern (RCPSP: one per resource).
  {
    std::map<std::vector<std::int32_t>, std::pair<std::uint32_t, std::uint32_t>> pat_of;
    std::vector<std::int32_t> pat_terms, base(bit_rows.size());
    std::vector<std::pair<std::uint32_t, std::uint32_t>> range(bit_rows.size());
    std::uint32_t max_pt = 0;
    for (std::size_t r = 0; r < bit_rows.size(); ++r) {
      std::int32_t b0 = INT32_MAX;
      for (std::int32_t x : bit_rows[r].terms)
        b0 = std::min(b0, bitof[static_cast<std::uint32_t>(x) & kTermWordMask]);
      std::vector<std::int32_t> pt;
      for (std::int32_t x : bit_rows[r].terms)
        pt.push_back(pack(x >> kTermWordBits,
                          static_cast<std::uint32_t>(bitof[static_cast<std::uint32_t>(x) & kTermWordMask] - b0)));
      auto it = pat_of.find(pt);
      if (it == pat_of.end()) {
        const std::uint32_t beg = static_cast<std::uint32_t>(pat_terms.size());
        pat_terms.insert(pat_terms.end(), pt.begin(), pt.end());
        it = pat_of.emplace(pt, std::make_pair(beg, static_cast<std::uint32_t>(pat_terms.size()))).first;
      }
      base[r] = b0;
      range[r] = it->second;
      max_pt = std::max<std::uint32_t>(max_pt, static_cast<std::uint32_t>(pt.size()));
    }
    L.n_brows = static_cast<std::uint32_t>(bit_rows.size());
    L.brow_lanes = 1;
    while (L.brow_lanes < 32 && L.brow_lanes * 8 < max_pt) L.brow_lanes <<= 1;
    L.brow_meta = reserve_arr(4 * L.n_brows);
    L.brow_base = reserve_arr(L.n_brows);
    L.bpat = reserve_arr(static_cast<std::uint32_t>(pat_terms.size()));
    for (std::uint32_t r = 0; r < L.n_brows; ++r) {
      B[L.brow_meta + 4 * r + 0] = static_cast<std::int32_t>(range[r].first);
      B[L.brow_meta + 4 * r + 1] = static_cast<std::int32_t>(range[r].second);
      B[L.brow_meta + 4 * r + 2] = bit_rows[r].c;
      B[L.brow_meta + 4 * r + 3] = static_cast<std::int32_t>(bit_rows[r].lsum);
      B[L.brow_base + r] = base[r];
    }
    std::copy(pat_terms.begin(), pat_terms.end(), B.begin() + L.bpat);
    // Word-parallel form (kernels.cuh eval_wrows) when every bit row has
    // coefficients in [0, 8) and no repeated cell: per 32-bit chunk of the
    // row's bit window, the term mask T and the coefficient bit-planes U0..U2,
    // so a chunk's sum is popc arithmetic and its zeroing mask (coef > c - s)
    // a bit-sliced comparison.
    bool wok = L.n_brows > 0 && !std::getenv("PCCP_NO_WROWS");
    std::uint32_t max_ch = 1;
    for (std::size_t r = 0; r < bit_rows.size() && wok; ++r) {
      std::vector<std::uint8_t> seen;
      for (std::uint32_t k = range[r].first; k < range[r].second; ++k) {
        const std::int32_t coef = pat_terms[k] >> kTermWordBits;
        const std::uint32_t off = static_cast<std::uint32_t>(pat_terms[k]) & kTermWordMask;
        if (coef < 0 || coef > 7 || off >= 32 * 32) wok = false;
        if (!wok) break;
        if (seen.size() <= off) seen.resize(off + 1, 0);
        if (seen[off]++) wok = false;
        max_ch = std::max<std::uint32_t>(max_ch, off / 32 + 1);
      }
    }
    if (wok) {
      L.wrows = 1;
      L.wrow_lg = 0;
      while ((1u << L.wrow_lg) < max_ch) ++L.wrow_lg;
      const std::uint32_t chunks = 1u << L.wrow_lg;
      std::map<std::pair<std::uint32_t, std::uint32_t>, std::uint32_t> wpat_of;  // pattern range -> first int4
      std::vector<std::int32_t> wpat;
      std::vector<std::uint32_t> wfirst(bit_rows.size());
      for (std::size_t r = 0; r < bit_rows.size(); ++r) {
        auto it = wpat_of.find(range[r]);
        if (it == wpat_of.end()) {
          const std::uint32_t first = static_cast<std::uint32_t>(wpat.size() / 4);
          std::vector<std::uint32_t> q(4 * chunks, 0);
          for (std::uint32_t k = range[r].first; k < range[r].second; ++k) {
            const std::uint32_t coef = static_cast<std::uint32_t>(pat_terms[k] >> kTermWordBits);
            const std::uint32_t off = static_cast<std::uint32_t>(pat_terms[k]) & kTermWordMask;
            const std::uint32_t m = 1u << (off & 31), c4 = 4 * (off / 32);
            q[c4] |= m;
            for (int b = 0; b < 3; ++b)
              if ((coef >> b) & 1u) q[c4 + 1 + b] |= m;
          }
          for (std::uint32_t v : q) wpat.push_back(static_cast<std::int32_t>(v));
          it = wpat_of.emplace(range[r], first).first;
        }
        wfirst[r] = it->second;
      }
      L.wrow_meta = reserve_arr(4 * L.n_brows);
      L.wpat = reserve_arr(static_cast<std::uint32_t>(wpat.size()));
      for (std::uint32_t r = 0; r < L.n_brows; ++r) {
        B[L.wrow_meta + 4 * r + 0] = static_cast<std::int32_t>(wfirst[r]);
        B[L.wrow_meta + 4 * r + 1] = bit_rows[r].c;
        B[L.wrow_meta + 4 * r + 2] = static_cast<std::int32_t>(bit_rows[r].lsum);
        B[L.wrow_meta + 4 * r + 3] = base[r];
      }
      std::copy(wpat.begin(), wpat.end(), B.begin() + L.wpat);
    }
    L.brow_lg = 0;
    while ((1u << L.brow_lg) < L.brow_lanes) ++L.brow_lg;
  }
  // Value-range analysis over the reference words (plain layouts only: a
  // packed layout takes the plain lowering's per-launch flags, engine.cu).
  if (!packed) {
    // Rows whose terms all read class <= 1 words can be summed in 32 bits once
    // the entry values are known to be small (fast_paths).
    {
      bool ok = L.n_rows > 0;
      for (const Row& r : rows) {
        std::int64_t s0 = 0, s1 = 0;
        for (std::int32_t x : r.terms) {
          const std::uint32_t w = static_cast<std::uint32_t>(x) & kTermWordMask;
          const std::int64_t coef = std::abs(std::int64_t{x >> kTermWordBits});
          if (w >= m.n_words || cls[w] == 2) {
            ok = false;
            continue;
          }
          read_fast[w] = 1;
          (cls[w] == 0 ? s0 : s1) += coef;
        }
        out.row_sum0.push_back(s0);
        out.row_sum1.push_back(s1);
      }
      out.rows_ok = ok;
    }
    out.ne_ok = L.n_ne > 0 && L.ne_even;
    for (std::uint32_t i = 0; i < L.n_ne && out.ne_ok; ++i) {
      for (std::uint32_t o : {0u, 3u}) {
        const std::uint32_t lbw = static_cast<std::uint32_t>(B[L.ne + 4 * i + o]) / 4;
        if (cls[lbw] == 2 || cls[lbw + 1] == 2) out.ne_ok = false;
        read_fast[lbw] = read_fast[lbw + 1] = 1;
      }
    }
    // unit records: guard words a, b (and the second guard's), tell source f
    out.unit_ok = L.n_unit1 + L.n_unit2 > 0;
    {
      auto ok_word = [&](std::uint32_t w) {  // the constant-zero word Z = n_words is always fine
        if (w == m.n_words) return true;
        if (w > m.n_words || cls[w] == 2) return false;
        read_fast[w] = 1;
        return true;
      };
      auto scan = [&](std::uint32_t off, std::uint32_t n) {
        for (std::uint32_t i = 0; i < n && out.unit_ok; ++i) {
          const std::uint32_t x = static_cast<std::uint32_t>(B[off + 4 * i]);
          const std::uint32_t w = static_cast<std::uint32_t>(B[off + 4 * i + 3]);
          if (!ok_word(x & 0xffffu) || !ok_word(x >> 16) || !ok_word((w >> 15) & 0x7fffu)) out.unit_ok = false;
          out.unit_k = std::max(out.unit_k, std::abs(std::int64_t{B[off + 4 * i + 2]}));
        }
      };
      scan(L.unit1, L.n_unit1);
      scan(L.unit2, L.n_unit2);
      for (std::uint32_t i = 0; i < L.n_unit2 && out.unit_ok; ++i) {
        const std::uint32_t x = static_cast<std::uint32_t>(B[L.unit2g + 2 * i]);
        if (!ok_word(x & 0xffffu) || !ok_word(x >> 16)) out.unit_ok = false;
      }
    }
    out.reif_ok = L.n_reif > 0;
    for (std::uint32_t i = 0; i < L.n_reif && out.reif_ok; ++i) {
      const std::uint32_t xy = static_cast<std::uint32_t>(B[L.reif + 4 * i]);
      for (std::uint32_t lbw : {xy & 0xffffu, xy >> 16}) {
        if (lbw + 1 >= m.n_words || cls[lbw] == 2 || cls[lbw + 1] == 2) out.reif_ok = false;
        else read_fast[lbw] = read_fast[lbw + 1] = 1;
      }
      out.reif_k = std::max({out.reif_k, std::abs(std::int64_t{B[L.reif + 4 * i + 2]}),
                             std::abs(std::int64_t{B[L.reif + 4 * i + 3]})});
    }
  }
  L.n_gen = static_cast<std::uint32_t>(generic.size());
  L.gen_off = reserve_arr(L.n_gen + 1);
  std::uint32_t gen_len = 0;
  for (std::uint32_t g : generic) gen_len += m.cmd_off[g + 1] - m.cmd_off[g];
  L.gen_code = reserve_arr(gen_len);
  {
    std::uint32_t p = 0;
    for (std::uint32_t k = 0; k < L.n_gen; ++k) {
      const std::uint32_t i = generic[k];
      B[L.gen_off + k] = static_cast<std::int32_t>(p);
      const std::uint32_t c0 = p;
      for (std::uint32_t x = m.cmd_off[i]; x < m.cmd_off[i + 1]; ++x) B[L.gen_code + p++] = m.cmd_code[x];
      if (packed) {  // the stream's words in the device layout (parse() checked its shape)
        std::int32_t* q = &B[L.gen_code + c0];
        const std::int32_t ng = q[0], mask = q[4];
        q[3] = static_cast<std::int32_t>(W(static_cast<std::uint32_t>(q[3])));
        std::int32_t* e = q + 5;
        auto remap_expr = [&](std::int32_t* x) {  // [k, n, (coef, word) * n]
          for (std::int32_t t = 0; t < x[1]; ++t) x[3 + 2 * t] = static_cast<std::int32_t>(W(static_cast<std::uint32_t>(x[3 + 2 * t])));
          return x + 2 + 2 * x[1];
        };
        for (std::int32_t g = 0; g < ng; ++g) e = remap_expr(e + 2);  // [rel, rhs, expr]
        for (std::int32_t f : {PCCP_FN_SCALAR, PCCP_FN_LB, PCCP_FN_UB})
          if (mask & f) e = remap_expr(e);
      }
    }
    B[L.gen_off + L.n_gen] = static_cast<std::int32_t>(p);
  }

  std::vector<std::int32_t> iv, scw, sct;
  for (std::uint32_t s = 0; s < m.n_slots; ++s) {
    const int k = m.slot_kind[s];
    if (k == PCCP_INTERVAL) {
      if (dmap[m.slot_word[s]] >= 0) iv.push_back(static_cast<std::int32_t>(W(m.slot_word[s])));  // not a bit cell
    } else {
      scw.push_back(static_cast<std::int32_t>(W(m.slot_word[s])));
      sct.push_back(k == PCCP_ZINC ? INT32_MAX : k == PCCP_ZDEC ? INT32_MIN : k == PCCP_BINC ? 1 : 0);
    }
  }
  L.n_iv = static_cast<std::uint32_t>(iv.size());
  L.iv_lb = reserve_arr(L.n_iv);
  std::copy(iv.begin(), iv.end(), B.begin() + L.iv_lb);
  // Dense interval stores (every word belongs to an interval, lb words 0, 2,
  // 4, ...): the failure scan reads (lb, ub) pairs by index, no table.
  L.iv_prefix = 1;
  for (std::uint32_t i = 0; i < L.n_iv && L.iv_prefix; ++i)
    if (iv[i] != static_cast<std::int32_t>(2 * i)) L.iv_prefix = 0;
  L.iv_dense = !packed && L.iv_prefix && L.n_iv * 2 == m.n_words ? 1 : 0;
  L.n_sc = static_cast<std::uint32_t>(scw.size());
  // Every scalar a row's lsum cell, and every row reporting its overload
  // (kernels.cuh eval_rows, eval_wrows; not the per-term bit rows): the
  // failure scan skips the scalars.  A row's lsum is private to it
  // (match_row), so the overload rule is its only way to top.
  if (!scw.empty() && (bit_rows.empty() || L.wrows) && !std::getenv("PCCP_SCALAR_SCAN")) {
    std::vector<std::uint8_t> is_lsum(DW + 1, 0);
    for (const Row& r : bit_rows) is_lsum[r.lsum] = 1;
    for (const Row& r : rows) is_lsum[r.lsum] = 1;
    L.sc_in_rows = 1;
    for (std::int32_t w : scw)
      if (!is_lsum[static_cast<std::uint32_t>(w)]) L.sc_in_rows = 0;
  }
  L.sc_w = reserve_arr(L.n_sc);
  L.sc_top = reserve_arr(L.n_sc);
  std::copy(scw.begin(), scw.end(), B.begin() + L.sc_w);
  std::copy(sct.begin(), sct.end(), B.begin() + L.sc_top);

  std::vector<std::int32_t> cand;
  if (m.n_cands == 0) {
    for (std::uint32_t s = 0; s < m.n_slots; ++s)
      if (m.slot_kind[s] == PCCP_INTERVAL) cand.push_back(static_cast<std::int32_t>(W(m.slot_word[s])));
  } else {
    if (!m.cands) bad("null candidate table");
    for (std::uint32_t i = 0; i < m.n_cands; ++i) {
      const std::int32_t s = m.cands[i];
      if (s < 0 || static_cast<std::uint32_t>(s) >= m.n_slots) bad("candidate slot out of range");
      if (m.slot_kind[s] == PCCP_INTERVAL) cand.push_back(static_cast<std::int32_t>(W(m.slot_word[s])));
    }
  }
  L.n_cand = static_cast<std::uint32_t>(cand.size());
  L.cand_lbw = reserve_arr(L.n_cand);
  std::copy(cand.begin(), cand.end(), B.begin() + L.cand_lbw);

  if (m.obj_slot >= 0) {
    if (static_cast<std::uint32_t>(m.obj_slot) >= m.n_slots || m.slot_kind[m.obj_slot] != PCCP_INTERVAL)
      bad("objective must be an interval slot");
    L.obj_lbw = static_cast<std::int32_t>(W(m.slot_word[m.obj_slot]));
  } else {
    L.obj_lbw = -1;
  }
  // Everything above is read per round or per node (staged into shared memory
  // when it fits); the folds (node entry of a root) and the decode table
  // (hash-sums of packed stores) stay in global memory.
  L.hot_words = static_cast<std::uint32_t>(B.size());
  L.n_fold = static_cast<std::uint32_t>(fold_w.size());
  L.fold_w = reserve_arr(L.n_fold);
  L.fold_v = reserve_arr(L.n_fold);
  for (std::uint32_t i = 0; i < L.n_fold; ++i) {
    B[L.fold_w + i] = fold_w[i];
    B[L.fold_v + i] = fold_v[i];
  }

  // Byte model of one round (lower.hpp): per record, the store words its
  // evaluation reads and its table entry.
  {
    double sb = 0, tb = 0;
    sb += 16.0 * L.n_ne, tb += 16.0 * L.n_ne;      // (lb, ub) of x and y; int4
    sb += 24.0 * L.n_reif, tb += (L.reif8 ? 8.0 : 16.0) * L.n_reif;  // x, y, b intervals (or x, y, b's plane pair); int4 / int2
    auto unit_words = [&](std::uint32_t x, std::uint32_t w) {
      int k = 1;  // the target
      for (std::uint32_t v : {x & 0xffffu, x >> 16, (w >> 15) & 0x7fffu}) k += v != Z ? 1 : 0;
      return 4.0 * k;
    };
    for (const U1& r : unit1) sb += unit_words(static_cast<std::uint32_t>(r.x), static_cast<std::uint32_t>(r.w));
    tb += 16.0 * unit1.size();
    for (const auto& r : unit2) {
      sb += unit_words(static_cast<std::uint32_t>(r.first.x), static_cast<std::uint32_t>(r.first.w));
      const std::uint32_t g2 = static_cast<std::uint32_t>(r.second.first);
      for (std::uint32_t v : {g2 & 0xffffu, g2 >> 16}) sb += v != Z ? 4.0 : 0.0;
    }
    tb += 24.0 * unit2.size();
    for (const Small& sm : smalls) {
      int k = 1 + ((sm.shape >> 10) & 1);  // target word(s)
      for (int j = 0; j < 4; ++j) k += sm.g[j] ? 1 : 0;
      k += sm.lbt ? 1 : 0;
      k += sm.ubt ? 1 : 0;
      sb += 4.0 * k;
    }
    tb += 44.0 * smalls.size();
    sb += 4.0 * L.n_rows + (L.row_even ? 8.0 : 4.0) * n_terms;  // lsum + each term's lb (or (lb, ub))
    tb += 16.0 * L.n_rows + 4.0 * n_terms;
    for (std::uint32_t g : generic) {
      const CmdP& c = cmds[g];
      for (const GuardP& gp : c.guards) sb += 4.0 * gp.lhs.terms.size();
      for (const auto* e : {&c.sc, &c.lb, &c.ub})
        if (*e) sb += 4.0 * ((*e)->terms.size() + 1);
      tb += 4.0 * (m.cmd_off[g + 1] - m.cmd_off[g]);
    }
    sb += 8.0 * L.n_iv + 4.0 * L.n_sc;  // the failure scan
    if (L.wrows) {  // per row: lsum + two plane pairs per 32-bit chunk; meta + one int4 per chunk
      sb += (4.0 + 16.0 * (1u << L.wrow_lg)) * L.n_brows;
      tb += (16.0 + 16.0 * (1u << L.wrow_lg)) * L.n_brows;
    } else {
      for (const Row& r : bit_rows) sb += 4.0 + 8.0 * r.terms.size();  // lsum + each term's plane pair
      tb += 20.0 * bit_rows.size();
      for (std::uint32_t r = 0; r < L.n_brows; ++r) tb += 4.0 * (B[L.brow_meta + 4 * r + 1] - B[L.brow_meta + 4 * r]);
    }
    sb += 8.0 * L.n_pairs;  // the planes' failure scan
    out.store_bytes_per_round = sb;
    out.table_bytes_per_round = tb;
  }
  if (packed) {
    L.dec = reserve_arr(NW);
    std::copy(out.dec.begin(), out.dec.end(), B.begin() + L.dec);
  }
  L.blob_words = static_cast<std::uint32_t>(B.size());
  if (B.empty()) B.push_back(0);
  return out;
}

}  // namespace

void to_device(const Lowered& d, const std::int32_t* ref, std::int32_t* dev) {
  const DeviceLayout& L = d.L;
  if (!L.packed) {
    std::copy(ref, ref + L.n_words, dev);
    return;
  }
  std::fill(dev, dev + L.n_words, 0);  // the pad word and the planes start at 0
  for (std::uint32_t w = 0; w < L.ref_words; ++w)
    if (d.dec[w] >= 0) dev[d.dec[w]] = ref[w];
  for (std::size_t b = 0; b < d.bit_lbw.size(); ++b) {
    const std::uint32_t w = static_cast<std::uint32_t>(d.bit_lbw[b]);
    // the folded constants every entry point applies (lower_packed): lb >= 0,
    // ub <= 1, so lb <= ub leaves (0,0), (0,1) or (1,1); anything else is the
    // empty interval, kept as both bits (failed)
    const std::int32_t lb = std::max(ref[w], d.bit_fold_lb[b]), ub = std::min(ref[w + 1], d.bit_fold_ub[b]);
    const std::uint32_t m = 1u << (b & 31), k = L.plane + 2 * static_cast<std::uint32_t>(b >> 5);
    if (lb > ub || lb >= 1) dev[k] |= static_cast<std::int32_t>(m);
    if (lb > ub || ub <= 0) dev[k + 1] |= static_cast<std::int32_t>(m);
  }
}

void to_reference(const Lowered& d, const std::int32_t* dev, std::int32_t* ref) {
  const DeviceLayout& L = d.L;
  if (!L.packed) {
    std::copy(dev, dev + L.n_words, ref);
    return;
  }
  for (std::uint32_t w = 0; w < L.ref_words; ++w) {
    const std::int32_t e = d.dec[w];
    if (e >= 0) {
      ref[w] = dev[e];
    } else {
      const std::uint32_t code = static_cast<std::uint32_t>(-1 - e), b = code >> 1;
      const std::uint32_t bits = static_cast<std::uint32_t>(dev[L.plane + 2 * (b >> 5) + (code & 1u)]);
      const bool set = (bits >> (b & 31)) & 1u;
      ref[w] = (code & 1u) ? (set ? 0 : 1) : (set ? 1 : 0);  // UB bit: ub <= 0; LB bit: lb >= 1
    }
  }
}

// The value-range analysis at run time.  Outside a failed round every
// interval stays inside its entry box (lb only rises, ub only falls), so at
// every round start a class-1 word is bounded by B1, the largest entry value
// of the intervals it belongs to; a class-0 word holds its entry value or a
// constant (B0).  Inside a round a class-1 value is an entry value plus one
// affine offset (<= kaff) per link of a dependency chain of affine joins, and
// a round performs at most r_aff of them: |v| <= max(B0, B1) + r_aff * kaff.
// Decisions and the objective bound stay inside the box (+-1).
void fast_paths(const Lowered& low, const std::int32_t* stores, std::size_t n_stores, std::size_t stride,
                bool& ne_fast, bool& rows_fast, bool& reif_fast, bool& unit_fast) {
  ne_fast = rows_fast = reif_fast = unit_fast = false;
  if ((!low.ne_ok && !low.rows_ok && !low.reif_ok && !low.unit_ok) || !stores || !n_stores) return;
  const DeviceLayout& L = low.L;
  const std::uint32_t nw = L.n_words;
  std::vector<std::int32_t> w(nw);
  std::int64_t b0 = low.kconst, b1 = 0;
  for (std::size_t s = 0; s < n_stores; ++s) {
    std::copy(stores + s * stride, stores + s * stride + nw, w.begin());
    for (std::uint32_t i = 0; i < L.n_fold; ++i) {
      const std::int32_t wf = low.blob[L.fold_w + i], v = low.blob[L.fold_v + i];
      std::int32_t& x = w[static_cast<std::uint32_t>(wf) & 0x7fffffffu];
      x = wf < 0 ? std::max(x, v) : std::min(x, v);
    }
    for (std::uint32_t i = 0; i < nw; ++i) {
      const std::uint8_t c = low.word_cls[i];
      if (c == 2 || !(low.word_read_fast[i] || c == 1)) continue;
      auto finite = [](std::int32_t v) { return v != INT32_MIN && v != INT32_MAX; };
      if (c == 0) {
        if (!finite(w[i])) return;
        b0 = std::max(b0, std::abs(std::int64_t{w[i]}));
      } else {  // class 1: the interval's box must be finite on both sides
        const std::int32_t p = low.word_partner[i];
        if (p < 0 || !finite(w[i]) || !finite(w[static_cast<std::uint32_t>(p)])) return;
        b1 = std::max({b1, std::abs(std::int64_t{w[i]}), std::abs(std::int64_t{w[static_cast<std::uint32_t>(p)]})});
      }
    }
  }
  const std::int64_t lim = std::int64_t{1} << 30;
  const std::int64_t bound1 = std::max(b0, b1) + 1 + low.r_aff * low.kaff;
  if (bound1 >= lim) return;
  ne_fast = low.ne_ok && bound1 + low.kaff + 2 < lim;
  reif_fast = low.reif_ok && bound1 + low.reif_k + 2 < lim;
  unit_fast = low.unit_ok && bound1 + low.unit_k + 2 < lim;
  if (low.rows_ok) {
    // |sum| <= S; the zeroing guard coef + sum - coef * v is <= 2 S + |coef|
    std::int64_t worst = 0;
    for (std::size_t r = 0; r < low.row_sum0.size(); ++r)
      worst = std::max(worst, low.row_sum0[r] * (b0 + 1) + low.row_sum1[r] * bound1);
    rows_fast = 3 * worst + 3 < lim;
  }
}

void host_join_decision(const pccp_model& m, std::int32_t* words, const pccp_decision& d) {
  if (d.var < 0 || static_cast<std::uint32_t>(d.var) >= m.n_slots || m.slot_kind[d.var] != PCCP_INTERVAL)
    throw std::runtime_error("decision on a non-interval slot");
  const std::uint32_t w = m.slot_word[d.var];
  if (d.upper) {
    const std::int32_t lo = d.mid + 1;
    if (lo > words[w]) words[w] = lo;
  } else if (d.mid < words[w + 1]) {
    words[w + 1] = d.mid;
  }
}

}  // namespace pccp_b200
