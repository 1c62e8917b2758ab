// capi_host.cpp — extern "C" wrapper of the host model builder (include/pccp_host.h).
#include <cstring>
#include <string>

#include "../../../include/pccp_host.h"
#include "model.hpp"
#include "rcpsp.hpp"

using namespace pccp_b200;

struct pccp_host_model {
  std::unique_ptr<Model> model;
  bool is_rcpsp = false;
  RcpspInstance inst;
  std::vector<std::int32_t> starts;
  FlatTables flat;  // cache behind pccp_host_view
};

namespace {
thread_local std::string g_err;

template <class F>
auto guarded(F&& f, decltype(f()) on_error) -> decltype(f()) {
  try {
    return f();
  } catch (const std::exception& e) {
    g_err = e.what();
  } catch (...) {
    g_err = "unknown error";
  }
  return on_error;
}

pccp_host_model* wrap(std::unique_ptr<Model> m) {
  auto* h = new pccp_host_model;
  h->model = std::move(m);
  return h;
}

pccp_host_model* wrap_rcpsp(const RcpspInstance& inst) {
  RcpspModel rm = build_rcpsp(inst);
  auto* h = new pccp_host_model;
  h->model = std::move(rm.model);
  h->is_rcpsp = true;
  h->inst = inst;
  h->starts = rm.starts;
  return h;
}

// Parses one prefix-encoded constraint starting at expr[pos].
Constraint parse(const std::int32_t* e, std::int32_t len, std::int32_t& pos) {
  auto at = [&](std::int32_t i) -> std::int32_t {
    if (i >= len) throw ModelError("constraint expression truncated");
    return e[i];
  };
  const std::int32_t tag = at(pos++);
  switch (tag) {
    case PCCP_C_SUM: {
      const std::int32_t n = at(pos++);
      if (n < 0) throw ModelError("negative term count");
      std::vector<std::pair<std::int32_t, std::int32_t>> terms;
      for (std::int32_t i = 0; i < n; ++i) {
        const std::int32_t coef = at(pos++);
        const std::int32_t slot = at(pos++);
        terms.emplace_back(coef, slot);
      }
      const std::int32_t c = at(pos++);
      return linear_leq(std::move(terms), c);
    }
    case PCCP_C_LEQ: {
      const std::int32_t xc = at(pos++), x = at(pos++), off = at(pos++), yc = at(pos++), y = at(pos++);
      return leq_offset(xc ? Operand::c(x) : Operand::v(x), off, yc ? Operand::c(y) : Operand::v(y));
    }
    case PCCP_C_AND: {
      Constraint a = parse(e, len, pos);
      Constraint b = parse(e, len, pos);
      return and_c(std::move(a), std::move(b));
    }
    case PCCP_C_IFF: {
      Constraint a = parse(e, len, pos);
      Constraint b = parse(e, len, pos);
      return iff_c(std::move(a), std::move(b));
    }
    case PCCP_C_NOT: return not_c(parse(e, len, pos));
    default: throw ModelError("unknown constraint tag " + std::to_string(tag));
  }
}

Constraint parse_all(const std::int32_t* e, std::int32_t len) {
  std::int32_t pos = 0;
  Constraint c = parse(e, len, pos);
  if (pos != len) throw ModelError("trailing words after the constraint expression");
  return c;
}

// Operand slots must exist and be intervals (op_lb / op_ub, propagation.cpp:95-106).
void check_slots(const Constraint& c, const Model& m) {
  auto var = [&](std::int32_t s) {
    if (s < 0 || s >= m.slot_count()) throw ModelError("constraint references unknown slot " + std::to_string(s));
    if (m.kind(s) != Kind::Interval) throw ModelError("constraint operand is not an interval");
  };
  switch (c.tag) {
    case Constraint::Tag::Sum:
      for (const auto& t : c.terms) var(t.second);
      break;
    case Constraint::Tag::Leq:
      if (!c.x.is_const) var(c.x.var);
      if (!c.y.is_const) var(c.y.var);
      break;
    case Constraint::Tag::Not: check_slots(*c.a, m); break;
    default:
      check_slots(*c.a, m);
      check_slots(*c.b, m);
  }
}
}  // namespace

extern "C" {

const char* pccp_host_last_error(void) { return g_err.c_str(); }

pccp_host_model* pccp_host_new(void) { return wrap(std::make_unique<Model>()); }
void pccp_host_free(pccp_host_model* m) { delete m; }

pccp_host_model* pccp_host_nqueens(int32_t n) {
  return guarded([&] { return n < 1 ? throw ModelError("n must be >= 1"), nullptr : wrap(build_nqueens(n)); },
                 (pccp_host_model*)nullptr);
}

pccp_host_model* pccp_host_random_csp(uint64_t seed, int32_t n_vars, int32_t n_cons, int32_t dom_hi) {
  return guarded(
      [&] {
        if (n_vars < 2 || n_cons < 0 || dom_hi < 0) throw ModelError("bad csp parameters");
        return wrap(build_random_csp(seed, n_vars, n_cons, dom_hi));
      },
      (pccp_host_model*)nullptr);
}

pccp_host_model* pccp_host_rcpsp_random(uint64_t seed, int32_t n_real, int32_t resources) {
  return guarded([&] { return wrap_rcpsp(random_patterson(seed, n_real, resources)); }, (pccp_host_model*)nullptr);
}

pccp_host_model* pccp_host_rcpsp_patterson(const char* text) {
  return guarded([&] { return wrap_rcpsp(parse_patterson(text ? text : "")); }, (pccp_host_model*)nullptr);
}

pccp_host_model* pccp_host_rcpsp(int32_t n_tasks, const int32_t* duration, int32_t n_res, const int32_t* usage,
                                 const int32_t* capacity, int32_t n_prec, const int32_t* prec, int32_t horizon) {
  return guarded(
      [&] {
        if (n_tasks < 0 || n_res < 0 || n_prec < 0) throw ModelError("negative size");
        RcpspInstance inst;
        for (int32_t i = 0; i < n_tasks; ++i) {
          inst.duration.push_back(duration[i]);
          inst.usage.emplace_back(usage + static_cast<std::ptrdiff_t>(i) * n_res,
                                  usage + static_cast<std::ptrdiff_t>(i + 1) * n_res);
        }
        for (int32_t k = 0; k < n_res; ++k) inst.capacity.push_back(capacity[k]);
        for (int32_t p = 0; p < n_prec; ++p) inst.precedences.emplace_back(prec[2 * p], prec[2 * p + 1]);
        inst.horizon = horizon;
        validate(inst);
        return wrap_rcpsp(inst);
      },
      (pccp_host_model*)nullptr);
}

int32_t pccp_host_add_cell(pccp_host_model* m, int32_t kind) {
  return guarded(
      [&] {
        if (kind < 0 || kind > 4) throw ModelError("bad lattice kind");
        return m->model->add_cell(static_cast<Kind>(kind));
      },
      int32_t{-1});
}

int pccp_host_tell(pccp_host_model* m, int32_t slot, int32_t lo, int32_t hi) {
  return guarded(
      [&] {
        if (slot < 0 || slot >= m->model->slot_count() || m->model->kind(slot) != Kind::Interval)
          throw ModelError("tell: slot is not an interval");
        m->model->tell_interval(slot, lo, hi);
        return int{PCCP_OK};
      },
      int{PCCP_EMODEL});
}

int pccp_host_post(pccp_host_model* m, const int32_t* expr, int32_t len) {
  return guarded(
      [&] {
        const Constraint c = parse_all(expr, len);
        check_slots(c, *m->model);
        m->model->append(compile(c, *m->model));
        return int{PCCP_OK};
      },
      int{PCCP_EMODEL});
}

int pccp_host_post_reified(pccp_host_model* m, int32_t b, const int32_t* expr, int32_t len) {
  return guarded(
      [&] {
        const Constraint c = parse_all(expr, len);
        check_slots(c, *m->model);
        m->model->append(compile_reified(b, c, *m->model));
        return int{PCCP_OK};
      },
      int{PCCP_EMODEL});
}

int pccp_host_set_objective(pccp_host_model* m, int32_t slot) {
  return guarded(
      [&] {
        if (slot >= m->model->slot_count() || (slot >= 0 && m->model->kind(slot) != Kind::Interval))
          throw ModelError("objective must be an interval cell");
        m->model->objective = slot;
        return int{PCCP_OK};
      },
      int{PCCP_EMODEL});
}

int pccp_host_set_candidates(pccp_host_model* m, const int32_t* slots, int32_t n) {
  return guarded(
      [&] {
        std::vector<std::int32_t> c(slots, slots + n);
        for (std::int32_t s : c)
          if (s < 0 || s >= m->model->slot_count()) throw ModelError("candidate slot out of range");
        m->model->candidates = std::move(c);
        return int{PCCP_OK};
      },
      int{PCCP_EMODEL});
}

int pccp_host_view(pccp_host_model* m, pccp_model* out) {
  return guarded(
      [&] {
        m->flat = m->model->flatten();
        const FlatTables& t = m->flat;
        out->n_slots = static_cast<uint32_t>(t.slot_kind.size());
        out->slot_kind = t.slot_kind.data();
        out->slot_word = t.slot_word.data();
        out->n_words = t.n_words;
        out->n_cmds = static_cast<uint32_t>(t.cmd_off.size() - 1);
        out->cmd_off = t.cmd_off.data();
        out->cmd_code = t.cmd_code.data();
        out->n_cands = static_cast<uint32_t>(t.cands.size());
        out->cands = t.cands.data();
        out->obj_slot = t.obj_slot;
        return int{PCCP_OK};
      },
      int{PCCP_EMODEL});
}

int pccp_host_bottom(const pccp_host_model* m, int32_t* words) {
  const auto w = m->model->bottom();
  if (!w.empty()) std::memcpy(words, w.data(), w.size() * sizeof(int32_t));
  return PCCP_OK;
}

int32_t pccp_host_rcpsp_tasks(const pccp_host_model* m) {
  return m->is_rcpsp ? static_cast<int32_t>(m->inst.tasks()) : -1;
}

int pccp_host_rcpsp_starts(const pccp_host_model* m, int32_t* slots) {
  if (!m->is_rcpsp) return PCCP_EARG;
  for (size_t i = 0; i < m->starts.size(); ++i) slots[i] = m->starts[i];
  return PCCP_OK;
}

int pccp_host_rcpsp_check(const pccp_host_model* m, const int32_t* words) {
  if (!m->is_rcpsp) return -1;
  return guarded(
      [&] {
        std::vector<std::int32_t> s;
        for (std::int32_t slot : m->starts) s.push_back(words[m->model->first_word(slot)]);
        return check_solution(m->inst, s) ? 1 : 0;
      },
      -1);
}

}  // extern "C"
