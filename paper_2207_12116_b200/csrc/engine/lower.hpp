// lower.hpp — flat reference tables -> device tables.
//
// The reference executes every GuardedCommand through one generic
// interpreter (GuardedCommand::apply, command.cpp:100-113).  The device path
// instead splits the command list into shape families, each a structure of
// arrays that a warp walks with coalesced loads:
//
//   fold    unguarded constant tells (init domains).  Idempotent after their
//           first application, so they are joined once at node entry instead
//           of every round (exact: the store only grows).
//   small   interval tells with <= 2 guards of <= 2 terms and <= 1 term per
//           bound: every reified / not(and) / offset / binary-sum command.
//           Guards are normalised to `sum tv(c_i, v_i) <= T` (H1 arithmetic).
//   row     a general sum compiled by compile_sum (propagation.cpp:314-335):
//           lsum tell + overload rule + one zeroing guard per term, fused
//           into one row evaluated by a sub-warp from one read of the lbs (H2).
//   generic anything else, interpreted from the flat stream on the device.
//
// Word indices are the reference's (H7), so stores round-trip unchanged;
// lower_packed's layout moves 0/1 cells into bit planes (to_device / to_reference).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../../include/pccp_gpu.h"

namespace pccp_b200 {

// Packed term: (coef << 20) | word, coef in [-2048, 2047], word < 2^20.
constexpr int kTermWordBits = 20;
constexpr std::uint32_t kTermWordMask = (1u << kTermWordBits) - 1;

struct DeviceLayout {
  // offsets (int32 units) into the blob
  std::uint32_t unit1, n_unit1;          // int4 records: guard (a | b<<16, T), tell (k, tw | f<<15 | neg<<30 | up<<31)
  std::uint32_t unit2, unit2g, n_unit2;  // same + int2 second guard
  std::uint32_t zero_word;               // constant-zero word Z = n_words (store_stride > n_words)
  // Fused not(and(x + a <= y, y + b <= x)) groups: the 4 commands compile_rec
  // emits for it (propagation.cpp:350-360) read and write only lb/ub of x and y.
  std::uint32_t ne, n_ne;                // int4 {4 lbx, a - 1, b - 1, 4 lby} (byte offsets of the lb words)
  std::uint32_t ne_even;                 // every NE lb word is even: (lb, ub) is one 8-byte load
  // Fused compile_reified(b, and(x + p <= y, y + q <= x)): the 11 commands of
  // propagation.cpp:415-431 over lb/ub of x, y and b (RCPSP overlaps).
  std::uint32_t reif, n_reif;            // int4 {lbx | lby << 16, lbb, p, q}
  // Filtered rounds (stores of <= 64 words made only of unit records): a
  // round re-evaluates just the records that read a word changed in the
  // previous round (CSR lists per word, entry = record | unit2 << 31).
  std::uint32_t filtered;
  std::uint32_t wl_off, wl;
  std::uint32_t small_g[4], small_T[2], small_lbk, small_lbt, small_ubk, small_ubt, small_tw;
  std::uint32_t n_small;
  std::uint32_t fold_w, fold_v;  // fold_w: word | (up << 31)
  std::uint32_t n_fold;
  std::uint32_t row_off, row_lsum, row_c, row_terms;
  std::uint32_t row_meta;  // int4 per row: {first term, end, c, lsum word}
  std::uint32_t n_rows, n_row_terms, row_lanes;  // lanes per row (power of two <= 32)
  std::uint32_t row_lg;                           // log2 row_lanes
  std::uint32_t row_tl;                           // the most terms one lane reads (ceil(max terms / row_lanes))
  std::uint32_t row_even;                         // every row term's lb word is even: (lb, ub) is one 8-byte load
  std::uint32_t gen_off;                          // offsets into gen_code
  std::uint32_t gen_code;
  std::uint32_t n_gen;
  std::uint32_t iv_lb;  // lb words of interval slots (failure scan)
  std::uint32_t iv_dense;  // the store is intervals only, lb words 0, 2, 4, ... (scan by index)
  std::uint32_t iv_prefix;  // the intervals are words [0, 2 n_iv), scalars after (RCPSP: the sums)
  std::uint32_t n_iv;
  std::uint32_t sc_w, sc_top;  // scalar slots: word, top value
  std::uint32_t n_sc;
  std::uint32_t cand_lbw;  // lb word of each branching candidate, priority order
  std::uint32_t n_cand;
  std::int32_t obj_lbw;  // -1: no objective
  std::uint32_t n_words;
  std::uint32_t n_ref_cmds;
  std::uint32_t blob_words;
  std::uint32_t hot_words;  // prefix of the blob read per round or per node (staged to smem); folds, decode after
  std::uint32_t var_order;  // set per launch: 0 first-fail (branch, solver.cpp:19-47), 1-3 smallest lb
  std::uint32_t var_seed;   // set per launch: var_order 3 tie-break seed
  std::uint32_t ne_fast;    // set per launch: value-range analysis proved the 32-bit NE path exact
  std::uint32_t rows_fast;  // set per launch: the same for the sum rows (fast_paths)
  std::uint32_t reif_fast;  // set per launch: the same for the reification records (fast_paths)
  std::uint32_t unit_fast;  // set per launch: the same for the unit records (fast_paths)
  // Bit-plane 0/1 cells (lower_packed).  The 0/1 interval slots (RCPSP's
  // overlap booleans, rcpsp.cpp:197-213) leave the word store: each becomes
  // one bit of an (LB, UB) plane pair, LB bit = [lb >= 1], UB bit = [ub <= 0],
  // both joined with red.shared.or (both only ever set: lb rises, ub falls);
  // both set = the empty interval (failed).  The other words keep their
  // reference order at device words [0, plane).
  std::uint32_t packed;       // 1: this layout has bit planes
  std::uint32_t plane;        // device word of plane pair 0 (even); pair k = words plane+2k (LB), plane+2k+1 (UB)
  std::uint32_t n_pairs;      // plane pairs (32 cells each)
  std::uint32_t ref_words;    // words of the reference store
  std::uint32_t dec;          // per reference word: device word (>= 0) or -1 - (2 * bit + is_ub)
  // Bit rows: compile_sum rows (propagation.cpp:314-335) over packed cells.
  // Row r reads bits brow_base[r] + off for each term (coef << 20 | off) of
  // its pattern [meta.x, meta.y) — RCPSP rows of one resource share a pattern.
  std::uint32_t brow_meta;    // int4 per row: {pattern begin, pattern end, c, lsum word}
  std::uint32_t brow_base;    // first bit of each row
  std::uint32_t bpat;         // pattern terms
  std::uint32_t n_brows, brow_lanes;
  std::uint32_t reif8;        // packed reification records are int2 {lx | ly << 16, bit | p << 18 | q << 25}
  std::uint32_t brow_lg;      // log2 brow_lanes
  // Word-parallel bit rows (eval_wrows): 2^wrow_lg lanes per row, one per
  // 32-bit chunk of the row's bit window.
  std::uint32_t wrows, wrow_lg;
  std::uint32_t wrow_meta;    // int4 per row: {first chunk (int4 index into wpat), c, lsum word, first bit}
  std::uint32_t wpat;         // int4 per chunk: {term mask, coefficient bit-planes 0, 1, 2}
  std::uint32_t sc_in_rows;   // every scalar slot is the lsum cell of a word-parallel bit row
  // Filtered kPacked rounds (kernels.cuh propagate_packed), set per launch:
  // dirty masks of dm_s words (one bit per start interval) + dm_p words (one
  // bit per plane word) per round buffer.
  std::uint32_t pfilter, dm_s, dm_p;
  // Reification segments for those rounds (lower.cpp): by y start (int2 [begin,
  // end) ranges), by x start (CSR r_xoff / r_xrec of record indices), by plane
  // word (r_p: begin of each word's range); r_ns starts.
  std::uint32_t rfilt, r_ns, r_y, r_xoff, r_xrec, r_p;
};


struct Lowered {
  DeviceLayout L{};
  std::vector<std::int32_t> blob;
  std::uint32_t n_dropped = 0;  // commands that can never fire (guard rhs = +inf with '>')
  double alg_bytes_per_eval = 0;  // SURVEY 8(d) B_alg over the reference commands
  // The byte model of one fixed-point round over the LOWERED records (what a
  // fused record actually reads, engine roofline): store words read
  // (shared memory) and table bytes read (shared memory when the tables fit,
  // else L2).  Joins are not counted: a round writes a few words at most.
  double store_bytes_per_round = 0, table_bytes_per_round = 0;
  std::vector<std::uint8_t> word_up;
  // value-range analysis (fast_paths)
  std::vector<std::uint8_t> word_cls;        // 0 constant-only, 1 affine interval bound, 2 unbounded
  std::vector<std::uint8_t> word_read_fast;  // read by a row term, an NE record or an affine tell
  std::vector<std::int32_t> word_partner;    // the other bound of an interval word, -1 for scalars
  std::int64_t kconst = 0, kaff = 0;         // max |k| over constant / affine tells
  std::int64_t r_aff = 0;                    // affine tells per round (one per command part)
  bool rows_ok = false, ne_ok = false;       // every row term / NE word has class <= 1
  bool reif_ok = false;                      // every reification x/y bound has class <= 1
  std::int64_t reif_k = 0;                   // max |p|, |q| over the reifications
  bool unit_ok = false;                      // every unit-record word read has class <= 1
  std::int64_t unit_k = 0;                   // max |k| over the unit tells
  std::vector<std::int64_t> row_sum0, row_sum1;  // per row: sum |coef| over class-0 / class-1 terms
  std::vector<std::int32_t> slot_of_word;  // for diagnostics
  // Packed layouts (L.packed): the host side of the bit planes.
  std::vector<std::int32_t> dec;          // L.dec on the host
  std::vector<std::int32_t> bit_lbw;      // reference lb word of each bit
  std::vector<std::int32_t> bit_fold_lb;  // max of the folded lb constants of each bit's cell (0 or 1)
  std::vector<std::int32_t> bit_fold_ub;  // min of the folded ub constants (0 or 1)
  std::uint32_t dev_words = 0;            // device store words (the reference's n_words when not packed)
};

// Throws std::runtime_error (mapped to PCCP_EMODEL) on malformed tables.
Lowered lower_model(const pccp_model& m);

// The device layout with bit-plane 0/1 cells when the model has them
// (L.packed = 1), else the plain lowering.  A slot is packed when it is an
// interval whose lb and ub are both folded to constants in {0, 1} (so every
// store that reaches the device holds it at 0/1, or failed), whose only
// writers are those folds, fused reifications (b <- (1,1) / (0,0)) and
// compile_sum zeroing (b <- (0,0)), and whose only readers are reifications
// and sum rows whose terms are all packed.  Every value such a cell can hold
// is one of (0,1), (1,1), (0,0) or failed: the two bits are exact.
Lowered lower_packed(const pccp_model& m);

// Reference store -> packed device store (folding the packed cells' constant
// tells, as every entry point folds) and back.  Plain layouts copy.
void to_device(const Lowered& d, const std::int32_t* ref, std::int32_t* dev);
void to_reference(const Lowered& d, const std::int32_t* dev, std::int32_t* ref);

// Value-range analysis for the exact 32-bit paths (engine.cu sets
// DeviceLayout::ne_fast / rows_fast per launch from the input stores): true
// when no NE evaluation can read a value outside (-2^30, 2^30), resp. every
// row sum and zeroing guard fits in 32 bits.  lower.cpp states the argument.
void fast_paths(const Lowered& low, const std::int32_t* stores, std::size_t n_stores, std::size_t stride,
                bool& ne_fast, bool& rows_fast, bool& reif_fast, bool& unit_fast);

// Host-side join of a decision into a store (Decision::as_join +
// Store::join_in_place on an Interval, solver.hpp:20-23, store.cpp:51-63).
void host_join_decision(const pccp_model& m, std::int32_t* words, const pccp_decision& d);

}  // namespace pccp_b200
