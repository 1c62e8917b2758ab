// model.hpp — host-side model construction for the B200 engine.
//
// This is the product's own C++ restatement of the reference's model API
// (lattice.hpp, store.hpp Schema, command.hpp, process.hpp gnf,
// propagation.hpp compile / compile_reified), reduced to what the device
// path needs: a schema of cells and a *flat, ordered list of guarded
// commands*.  The reference builds PCCP process trees, erases locals and
// lowers to guarded normal form; here the compiler emits the GNF list
// directly in the same depth-first order, so slot numbering (H7) and the
// command sequence come out identical — tests/test_host_model.py checks the
// flat tables byte-for-byte against the reference library's own output.
#pragma once

#include <cstdint>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

namespace pccp_b200 {

// ---- lattice (lattice.hpp:16-97) --------------------------------------------
enum class Kind : std::uint8_t { ZInc = 0, ZDec = 1, BInc = 2, BDec = 3, Interval = 4 };

inline constexpr std::int32_t kNegInf = INT32_MIN;
inline constexpr std::int32_t kPosInf = INT32_MAX;

struct ModelError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CompileError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// sat_add (lattice.cpp:110-112): sentinels widen to +-2^40, sum narrows back.
std::int32_t sat_add(std::int32_t a, std::int32_t b);

// ---- expressions -------------------------------------------------------------
enum class Part : std::uint8_t { Scalar, Lb, Ub };

struct Term {
  std::int32_t coef;
  std::int32_t slot;
  Part part;
};

// k + sum coef*cell (LinExpr, command.hpp:35-46)
struct Lin {
  std::int32_t k = 0;
  std::vector<Term> terms;
};

// lhs <= rhs (leq) or lhs > rhs (gt)  (Pred, command.hpp:58-87)
struct Guard {
  Lin lhs;
  bool gt = true;
  std::int32_t rhs = 0;
};

// One command of guarded normal form: guards => target <- fn.
struct Cmd {
  std::vector<Guard> guards;
  std::int32_t target = 0;
  std::optional<Lin> scalar, lb, ub;
};

using Gnf = std::vector<Cmd>;

// ---- schema + command list -----------------------------------------------------
struct FlatTables {
  std::vector<std::uint8_t> slot_kind;
  std::vector<std::uint32_t> slot_word;
  std::uint32_t n_words = 0;
  std::vector<std::uint32_t> cmd_off;
  std::vector<std::int32_t> cmd_code;
  std::vector<std::int32_t> cands;
  std::int32_t obj_slot = -1;
};

class Model {
 public:
  std::int32_t add_cell(Kind k, std::string name = {});
  std::int32_t slot_count() const { return static_cast<std::int32_t>(kinds_.size()); }
  Kind kind(std::int32_t s) const { return kinds_.at(static_cast<std::size_t>(s)); }
  std::uint32_t first_word(std::int32_t s) const { return words_.at(static_cast<std::size_t>(s)); }
  std::uint32_t word_count() const { return n_words_; }
  const std::string& name(std::int32_t s) const { return names_.at(static_cast<std::size_t>(s)); }

  void append(Gnf cmds);
  void truncate_cells(std::int32_t n);  // roll back cells added by a failed compile
  const Gnf& commands() const { return cmds_; }

  // Unguarded constant tell of an interval / scalar value (tell_const + gnf).
  void tell_interval(std::int32_t slot, std::int32_t lo, std::int32_t hi);

  std::vector<std::int32_t> candidates;  // BranchStrategy (empty: every interval)
  std::int32_t objective = -1;

  // Serialise to the flat tables of include/pccp_gpu.h; resolves words
  // (resolve_word, command.cpp:135-156) and throws ModelError on misuse.
  FlatTables flatten() const;

  // Store::reset (store.cpp:29-39).
  std::vector<std::int32_t> bottom() const;

 private:
  std::vector<Kind> kinds_;
  std::vector<std::uint32_t> words_;
  std::vector<std::string> names_;
  std::uint32_t n_words_ = 0;
  Gnf cmds_;
};

// ---- constraints (propagation.hpp:17-66) -------------------------------------------
struct Operand {
  std::int32_t var = -1;
  std::int32_t value = 0;
  bool is_const = false;
  static Operand v(std::int32_t s) { return {s, 0, false}; }
  static Operand c(std::int32_t k) { return {-1, k, true}; }
};

struct Constraint {
  enum class Tag : std::uint8_t { Sum, Leq, And, Iff, Not } tag = Tag::Leq;
  std::vector<std::pair<std::int32_t, std::int32_t>> terms;  // Sum: (coef, slot)
  std::int32_t c = 0;                                        // Sum bound
  Operand x, y;                                              // Leq: x + offset <= y
  std::int32_t offset = 0;
  std::shared_ptr<const Constraint> a, b;  // And / Iff / Not
};

Constraint linear_leq(std::vector<std::pair<std::int32_t, std::int32_t>> terms, std::int32_t c);
Constraint leq_offset(Operand x, std::int32_t offset, Operand y);
inline Constraint leq(Operand x, Operand y) { return leq_offset(x, 0, y); }
inline Constraint lt(Operand x, Operand y) { return leq_offset(x, 1, y); }
inline Constraint precedes(Operand x, std::int32_t d, Operand y) { return leq_offset(x, d, y); }
Constraint and_c(Constraint a, Constraint b);
Constraint iff_c(Constraint a, Constraint b);
Constraint not_c(Constraint a);

// compile (propagation.cpp:408-413): appends cells (one lsum per general sum)
// to `m` and returns the guarded commands, without appending them.
Gnf compile(const Constraint& c, Model& m);
// compile_reified (propagation.cpp:415-431).
Gnf compile_reified(std::int32_t b, const Constraint& c, Model& m);

// ---- benchmark models ----------------------------------------------
std::unique_ptr<Model> build_nqueens(int n);
std::unique_ptr<Model> build_random_csp(std::uint64_t seed, int n_vars, int n_cons, int dom_hi);

}  // namespace pccp_b200
