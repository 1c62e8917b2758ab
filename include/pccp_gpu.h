/*
 * pccp_gpu.h — C ABI of the B200 propagate-and-search engine.
 *
 * This is the drop-in boundary for the reference's search entry points
 * (/root/reference/proj/include/pccp/solver.hpp:99-128 and
 * /root/reference/proj/include/pccp/engine.hpp:27-41).  Everything that
 * crosses it is a plain pointer, a size or a POD struct; no C++ types, no
 * exceptions.  A model arrives as *flat command tables* — the serialised form
 * of the reference's `std::vector<GuardedCommand>` (command.hpp:119-140) plus
 * its `Schema` (store.hpp:29-43) — and is lowered to device tables inside
 * pccp_gpu_load().  INTEGRATION.md shows the ~60-line serialiser a
 * maintainer adds on the reference side.
 *
 * Entry points and the reference interface each one replaces:
 *   pccp_gpu_propagate_batch  run_sequential / run_parallel   engine.hpp:27-41, engine.cpp:13-133
 *   pccp_gpu_enumerate        (new: all-solutions counting; the reference has only
 *                              branch-and-bound, solver.cpp:122-146 gives the DFS order)
 *   pccp_gpu_solve            solve_parallel / solve_dfs        solver.hpp:105-128, solver.cpp:229-283
 *                             (its EPS phase restates eps_decompose, solver.cpp:180-227,
 *                              and every node runs branch, solver.cpp:19-47, on the device)
 *   pccp_gpu_replay           materialize                       solver.cpp:91-102
 *
 * Return codes: PCCP_OK, PCCP_EMODEL (ModelError/SchemaError/CompileError,
 * lattice.hpp:24-32), PCCP_ECUDA, PCCP_ELIMIT, PCCP_EARG.  The message of the
 * last failure on the calling thread is pccp_gpu_last_error().
 *
 * Threading: one context per host thread; a context is not re-entrant.
 */
#ifndef PCCP_GPU_H
#define PCCP_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- return codes ------------------------------------------------------ */
enum {
  PCCP_OK = 0,
  PCCP_EMODEL = 1, /* model/lowering error (reference: ModelError, SchemaError) */
  PCCP_ECUDA = 2,  /* CUDA runtime / launch failure, no device */
  PCCP_ELIMIT = 3, /* model exceeds a device capacity limit */
  PCCP_EARG = 4    /* bad argument */
};

/* ---- lattice kinds: same order as pccp::Kind (lattice.hpp:16) ----------- */
enum { PCCP_ZINC = 0, PCCP_ZDEC = 1, PCCP_BINC = 2, PCCP_BDEC = 3, PCCP_INTERVAL = 4 };

/* ---- predicate relation: same order as Pred::Rel (command.hpp:64) ------- */
enum { PCCP_LEQ = 0, PCCP_GT = 1 };

/* ---- monotone function parts present in a command (MonotoneFn, command.hpp:98-101) */
enum { PCCP_FN_SCALAR = 1, PCCP_FN_LB = 2, PCCP_FN_UB = 4 };

/* ---- solve status: same order as SolveStatus (solver.hpp:56) ------------ */
enum { PCCP_OPTIMAL = 0, PCCP_SAT = 1, PCCP_UNSAT = 2, PCCP_UNKNOWN = 3 };

/* ---- engine status: same order as pccp::Status (engine.hpp:12) ---------- */
enum { PCCP_FIXPOINT = 0, PCCP_FAILED = 1 };

/*
 * Flat command tables.
 *
 * Slots: slot s has kind slot_kind[s] and first word slot_word[s]; an Interval
 * owns words (w, w+1) = (lb, ub), a scalar owns one word (store.cpp:5-21).
 *
 * Command i is the int32 stream cmd_code[cmd_off[i] .. cmd_off[i+1]):
 *   [0] n_guards  [1] target_slot  [2] target_kind  [3] target_word  [4] fn_mask
 *   then per guard   : rel, rhs, k, n_terms, (coef, word) x n_terms
 *   then per fn part present, in the order scalar, lb, ub:
 *                      k, n_terms, (coef, word) x n_terms
 * A guard reads `k + sum coef*word  rel  rhs` (Pred::eval, command.cpp:29-33);
 * a fn part is the saturating linear form LinExpr::eval (command.cpp:11-27).
 * Generic (std::function) predicates or functions are not representable:
 * the serialiser must reject them (they are test-only escape hatches).
 */
typedef struct pccp_model {
  uint32_t n_slots;
  const uint8_t* slot_kind;  /* n_slots */
  const uint32_t* slot_word; /* n_slots */
  uint32_t n_words;
  uint32_t n_cmds;
  const uint32_t* cmd_off; /* n_cmds + 1 */
  const int32_t* cmd_code; /* cmd_off[n_cmds] int32 */
  uint32_t n_cands;        /* 0: every Interval slot (BranchStrategy{}, solver.hpp:89-91) */
  const int32_t* cands;    /* candidate slots, in priority order */
  int32_t obj_slot;        /* objective Interval slot for minimisation, or -1 */
} pccp_model;

/* One branching decision (solver.hpp:16-24): upper=0 joins (-inf, mid),
 * upper=1 joins (mid+1, +inf) into slot `var`. */
typedef struct pccp_decision {
  int32_t var;
  int32_t upper;
  int32_t mid;
} pccp_decision;

/* Device execution configuration; zero fields take automatic values. */
typedef struct pccp_gpu_cfg {
  int32_t device;        /* CUDA ordinal */
  int32_t group_threads; /* threads owning one subproblem: 32 (warp) .. 1024; 0 = auto */
  int32_t groups_per_cta;/* warp-groups sharing one CTA (and its smem command table); 0 = auto */
  int32_t ctas_per_sm;   /* 0 = auto (occupancy) */
  int32_t eps_factor;    /* EPS subproblems per resident group; 0 = auto (warp groups 8; CTA groups
                            start from the root alone and spread by donations) */
  int32_t shard_index;   /* this GPU's share of the EPS frontier: i mod shard_count == shard_index */
  int32_t shard_count;   /* 0/1 = unsharded */
  int32_t hash;          /* 1: accumulate the order-independent fixed-point hash-sum */
  int32_t verbose;       /* 1: one summary line per device search on stderr (layout, grid, times, counters) */
  int32_t value_order;   /* DFS branch order: 0 left (x <= mid) first, as dfs() (solver.cpp:139-143);
                            1 right first; 2 mixed (odd groups right first); -1 = 0.
                            The explored tree is the same,
                            so counts, optima and proofs are unchanged; only node order differs. */
  int32_t var_order;     /* variable selection: 0 = branch() (solver.cpp:19-47), the narrowest
                            candidate; 1 = smallest lower bound (ties: candidate order).  Not in
                            the reference (BranchStrategy, solver.hpp:89-91, has candidates only):
                            a different tree, so node counts differ; optima and UNSAT do not. */
  int32_t primal_ms;     /* pccp_gpu_solve only, > 0: a primal phase of at most this many ms with
                            var_order 2 runs first, restarted from the root under obj <= best-1
                            whenever it improved and then stalled (env PCCP_PRIMAL_STALL_MS,
                            default max(100, primal_ms/20)); its incumbent (and, if one segment
                            exhausts its tree, its proof) carries into the exact phase, which
                            searches the cfg's var_order tree under obj <= best-1.  0 = off. */
  int32_t audit_nodes;   /* > 0: the persistent search records the store before and after the
                            fixed point of up to this many nodes (every 2^audit_shift-th
                            materialisation), for pccp_gpu_audit.  0 = off. */
  int32_t audit_shift;
  int32_t record_frontier; /* 1: keep the hashes of the last search's shared EPS frontier and of this
                              shard's share of it (pccp_gpu_frontier; tests of the partition) */
  int32_t mix_order;     /* minimisation, a portfolio of branching orders: every mix_order-th search
                            group branches in var_order 2 (smallest lb, latest start on ties) inside
                            whatever box it explores, the others in the cfg's var_order.  Every box
                            is still searched completely, so optima and proofs are unchanged; node
                            counts differ.  0 = auto (the measured default), -1 = off. */
} pccp_gpu_cfg;

typedef struct pccp_limits {
  double timeout_s;    /* <= 0: none */
  uint64_t node_limit; /* 0 is honoured (immediate UNKNOWN, solver.cpp:68-76); UINT64_MAX: none */
} pccp_limits;

/* Counters returned by every search call. `nodes` counts materialised tree
 * nodes (one propagation fixed point each, solver.cpp:100); `evals` counts
 * propagator evaluations in reference-command units (rounds x commands). */
typedef struct pccp_stats {
  uint64_t nodes;
  uint64_t failures;
  uint64_t solutions;
  uint64_t open_leaves; /* depth-capped enumeration only */
  uint64_t hash_sum;    /* sum over non-failed nodes of the FNV-style store hash */
  uint64_t rounds;      /* fixed-point rounds over all nodes */
  uint64_t evals;       /* rounds x reference commands */
  uint64_t subproblems; /* EPS frontier size handed to the persistent search */
  uint64_t max_depth;
  double elapsed_ms;    /* whole call, host clock */
  double kernel_ms;     /* device time of the search kernels (CUDA events) */
  double decompose_ms;  /* device+host time of the EPS phase */
  uint64_t launches;    /* kernels launched by this call */
  uint64_t search_evals;/* evals inside the persistent search kernel only */
  uint64_t h2d_bytes;   /* host->device bytes moved by this call */
  uint64_t d2h_bytes;   /* device->host bytes moved by this call */
  double device_ms;     /* device time of the whole call (CUDA events on the engine stream): root
                           propagation + decomposition + search; host-side buffer sizing between
                           them (first calls) is in elapsed_ms only */
  uint64_t bfs_levels;  /* EPS decomposition levels */
  uint64_t donations;   /* subtrees handed from busy to idle groups (dynamic load balancing) */
  uint64_t rematerialised; /* nodes materialised a second time: EPS frontier nodes re-propagated under
                              the current bound, as solve_parallel's workers re-materialise their
                              subproblem roots (solver.cpp:266-268); distinct tree nodes = nodes -
                              rematerialised */
  uint64_t stolen;      /* N linked shards: frontier subproblems this shard took from peers' shares */
  uint64_t remote_in;   /* N linked shards: pending branches donated to this GPU by peers */
  uint64_t remote_out;  /* ... and by this GPU to peers */
} pccp_stats;

typedef struct pccp_enum_result {
  pccp_stats stats;
  int32_t exhausted; /* 1: every subtree explored; 0: stopped by a limit */
} pccp_enum_result;

typedef struct pccp_solve_result {
  pccp_stats stats;
  int32_t status;        /* PCCP_OPTIMAL .. PCCP_UNKNOWN */
  int32_t has_objective;
  int32_t objective;
  int32_t n_improvements;      /* incumbent log length (<= 64 kept) */
  int32_t improvements[64];    /* objective values, in improvement order */
  double improvement_ms[64];   /* device time since search start */
  int32_t phases;              /* 1, or 2 with a primal phase (cfg.primal_ms) */
  int32_t primal_proved;       /* the primal phase exhausted its tree: its result is the proof.  The
                                  primal dives of an N-shard solve cover the WHOLE tree on every GPU,
                                  so one GPU's primal proof is the job's proof (peers are told to stop) */
  uint64_t primal_nodes;       /* nodes of the primal phase (included in stats.nodes) */
  double primal_device_ms;     /* device time of the primal phase */
  int32_t primal_restarts;     /* primal segments restarted from the root under a better bound */
} pccp_solve_result;

typedef struct pccp_gpu_ctx pccp_gpu_ctx;

const char* pccp_gpu_last_error(void);
const char* pccp_gpu_version(void);

int pccp_gpu_device_count(int32_t* out);
int pccp_gpu_open(const pccp_gpu_cfg* cfg, pccp_gpu_ctx** out);
void pccp_gpu_close(pccp_gpu_ctx* ctx);

/* Lowers the flat tables to device tables and uploads them (deep copy). */
int pccp_gpu_load(pccp_gpu_ctx* ctx, const pccp_model* model);

/* Fixed point of every one of `n` input stores (n x n_words, host memory),
 * independently: the device form of run_sequential (engine.cpp:13-32).
 * out_words may alias in_words.  status[i] is PCCP_FIXPOINT/PCCP_FAILED;
 * rounds (optional) receives the rounds each store took. */
int pccp_gpu_propagate_batch(pccp_gpu_ctx* ctx, const int32_t* in_words, uint32_t n,
                             int32_t* out_words, uint8_t* status, uint32_t* rounds);

/* Replays decision paths on top of `root` and propagates, like materialize
 * (solver.cpp:91-102): copy root, join each decision, join obj <= best-1
 * (best == INT32_MAX: no bound), run to the fixed point.  Path p is
 * decisions[path_off[p] .. path_off[p+1]). */
int pccp_gpu_replay(pccp_gpu_ctx* ctx, const int32_t* root_words, uint32_t n_paths,
                    const uint32_t* path_off, const pccp_decision* decisions,
                    const int32_t* best, int32_t* out_words, uint8_t* status);

/* All-solutions enumeration below `root_words` (host memory, n_words):
 * depth-first left-first search in the order of dfs() (solver.cpp:122-146),
 * nodes with >= depth_cap decisions are propagated and counted but not
 * expanded (depth_cap < 0: unlimited).  EPS-decomposed over the device. */
int pccp_gpu_enumerate(pccp_gpu_ctx* ctx, const int32_t* root_words, int32_t depth_cap,
                       const pccp_limits* limits, pccp_enum_result* out);

/* Branch-and-bound minimisation of model->obj_slot: the device form of
 * solve_parallel (solver.cpp:229-283).  best_words (optional, n_words) gets
 * the best solution store.  Status rules of finish() (solver.cpp:148-162). */
int pccp_gpu_solve(pccp_gpu_ctx* ctx, const int32_t* root_words, const pccp_limits* limits,
                   pccp_solve_result* out, int32_t* best_words);

/* Multi-GPU incumbent sharing (optimisation only).  Each process exports the
 * IPC handle of its device incumbent cell (<= 64 bytes); after all handles
 * are exchanged (e.g. torch.distributed.all_gather_object) every process
 * attaches its peers, and improving solutions are pushed with system-scope
 * atomicMin into every peer replica over NVLink. */
int pccp_gpu_incumbent_handle(pccp_gpu_ctx* ctx, uint8_t* out64);
int pccp_gpu_attach_peers(pccp_gpu_ctx* ctx, const uint8_t* handles64, int32_t n_handles,
                          int32_t self_index);

/* The same for contexts of one process (one host thread per device, e.g. the
 * pccp_gpu CLI with --gpus N): peer access is enabled between their devices
 * and each context pushes improvements into every other context's cell.
 * Contexts on the same device are linked directly. */
int pccp_gpu_link_peers(pccp_gpu_ctx* const* ctxs, int32_t n);

/* Cross-rank cells.  Once peers are attached or linked, a search never
 * resets the incumbent cell, the best-store lock and the `done` flag (a
 * peer's push may land before this rank's search starts, and must not be
 * lost); they are reset by pccp_gpu_open, pccp_gpu_load and this call.  A
 * multi-rank caller resets every rank, then barriers, then solves
 * (paper_2207_12116_b200/distributed.py run_solve). */
int pccp_gpu_reset_shared(pccp_gpu_ctx* ctx);

/* Offers an objective value to the incumbent cell (atomicMin): the value of a
 * known solution, e.g. a warm start.  The search then looks for strictly
 * better solutions only (solver.cpp:96-99); a value below the optimum makes
 * the solve report that value with no store (has_objective = 2). */
int pccp_gpu_offer_incumbent(pccp_gpu_ctx* ctx, int32_t value);

/* With cfg.record_frontier: the FNV store hashes of the last
 * search's shared EPS frontier (phase A, identical on every shard) and of the
 * positions i = shard_index (mod shard_count) this context kept.  Each array
 * receives at most `cap` entries; *n_all / *n_share get the full sizes. */
int pccp_gpu_frontier(pccp_gpu_ctx* ctx, uint64_t* all, uint32_t* n_all, uint64_t* share,
                      uint32_t* n_share, uint32_t cap);

/* The node audit of the last enumerate/solve call (cfg.audit_nodes > 0):
 * pre[k] is a node's store as materialised (parent fixed point + decision +
 * objective bound), post[k] the engine's result for it and failed[k] its
 * status, so a caller can recompute run_sequential(pre[k]) (engine.cpp:13-32)
 * and compare.  pre/post hold cfg.audit_nodes x n_words int32; *n_out gets
 * the number of samples taken. */
int pccp_gpu_audit(pccp_gpu_ctx* ctx, int32_t* pre, int32_t* post, uint8_t* failed, uint32_t* n_out);

/* Information about the lowered model (device tables), for roofline accounting. */
typedef struct pccp_lowering_info {
  uint32_t n_words;
  uint32_t n_cmds;          /* reference commands */
  uint32_t n_folded;        /* unguarded constant tells folded into node entry */
  uint32_t n_small;         /* fixed-shape small commands */
  uint32_t n_rows;          /* fused sum rows (lsum tell + overload + zeroing guards) */
  uint32_t n_row_terms;
  uint32_t n_generic;       /* interpreted fallback commands */
  uint32_t table_bytes;     /* device table bytes read per round */
  uint32_t store_bytes;
  uint32_t group_threads;
  uint32_t groups_per_cta;
  uint32_t ctas;
  uint32_t smem_bytes;
  uint32_t table_in_smem;
  uint32_t stack_in_smem;
  uint32_t stack_depth;
  double alg_bytes_per_eval; /* 4*(guard terms) + 4*(fn terms + target words), per
                                reference command: counts a word once per command that reads it */
  double store_bytes_per_round; /* the lowered records' byte model: store bytes one fixed-point round
                                   reads (fused records read each word once for several commands) */
  double table_bytes_per_round; /* table bytes one round reads (shared memory if table_in_smem, else L2) */
  uint32_t packed_cells;  /* 0/1 interval cells held as bits of (lb, ub) bit planes (0: plain layout) */
  uint32_t device_words;  /* words of one device store (= n_words in the plain layout) */
} pccp_lowering_info;

int pccp_gpu_lowering_info(pccp_gpu_ctx* ctx, pccp_lowering_info* out);

/* Host-only: lowers the tables without a device (validation / diagnostics).
 * shape_counts (optional, 6 entries): unit records with <= 1 guard, unit
 * records with 2 guards, commands dropped as never-firing, fused not(and)
 * constraints, filtered-rounds flag, fused reifications. */
int pccp_lower_only(const pccp_model* model, pccp_lowering_info* out, uint32_t* shape_counts);

/* Host-only: the value-range analysis (lower.cpp fast_paths) for `n` input
 * stores of the lowered model: *mask gets bit 0 NE, bit 1 sum rows, bit 2
 * reifications, bit 3 unit records = the families whose 32-bit path the
 * engine would take for these inputs (diagnostics and tests). */
int pccp_lower_fast_paths(const pccp_model* model, const int32_t* stores, uint32_t n, uint32_t* mask);

/* Host-only: the device store layout the engine picks for this model (bit
 * planes for its 0/1 cells, lower.hpp lower_packed).  *dev_words gets the
 * device store size; when dev / back are non-null the n reference stores in
 * `stores` are converted to it (dev: n * dev_words) and back (back: n *
 * n_words).  The conversion folds the packed cells' constant tells, as every
 * entry point does, and keeps an empty 0/1 cell empty (tests, diagnostics). */
int pccp_lower_layout(const pccp_model* model, const int32_t* stores, uint32_t n, int32_t* dev, int32_t* back,
                      uint32_t* dev_words);

#ifdef __cplusplus
}
#endif

#endif /* PCCP_GPU_H */
