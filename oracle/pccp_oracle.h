/* pccp_oracle.h — TEST INFRASTRUCTURE ONLY: plain-C restatement of the
 * reference propagate-and-search path over the flat tables of
 * include/pccp_gpu.h.  Used by tests/ and bench.py's cpu_baseline as the
 * checker; never linked into the product. */
#ifndef PCCP_ORACLE_H
#define PCCP_ORACLE_H

#include <stdint.h>

#include "pccp_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Saturating linear form (command.cpp:11-27). `e` points at [k, n, (coef, word)*n]. */
int32_t orc_lin_eval(const int32_t* e, const int32_t* words);

/* Store failure test (store.cpp:65-75). */
int orc_is_failed(const pccp_model* m, const int32_t* words);

/* run_sequential (engine.cpp:13-32) in place; returns 1 if failed. */
int orc_run_sequential(const pccp_model* m, int32_t* words, uint64_t* iterations,
                       uint64_t* applications);

/* branch (solver.cpp:19-47): 0 = no candidate (solution), 1 = decision, -1 = unbounded (ModelError). */
int orc_branch(const pccp_model* m, const int32_t* words, int32_t* var, int32_t* mid);

/* materialize (solver.cpp:91-102); decisions are (var, upper, mid) triples; best == INT32_MAX: no bound. */
int orc_replay(const pccp_model* m, const int32_t* root, int n_dec, const int32_t* dec, int32_t best,
               int32_t* out);

/* Hash of SURVEY 8(c): FNV-style over the 4 little-endian bytes of every word. */
uint64_t orc_store_hash(uint32_t n_words, const int32_t* words);

/* All-solutions DFS with depth cap, node order of dfs() (solver.cpp:122-146).
 * out: nodes, failures, solutions, open_leaves, hash_sum, sweeps, exhausted. Returns -1 on ModelError. */
int orc_enumerate(const pccp_model* m, const int32_t* root, int depth_cap, uint64_t node_budget,
                  uint64_t* out);

/* solve_dfs (solver.cpp:166-173): out = status, has_obj, obj; st = nodes, solutions. */
int orc_solve_dfs(const pccp_model* m, const int32_t* root, uint64_t node_limit, int32_t* out,
                  uint64_t* st, int32_t* best_words);

#ifdef __cplusplus
}
#endif

#endif
