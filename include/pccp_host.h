/*
 * pccp_host.h — C ABI of the host-side model builder shipped with the B200
 * engine (paper_2207_12116_b200/csrc/host).  It restates the reference's model
 * construction API (store.hpp SchemaBuilder::add_cell, propagation.hpp
 * compile / compile_reified, rcpsp.hpp build_model / check_solution) and
 * produces the flat tables pccp_gpu_load() consumes (include/pccp_gpu.h).
 *
 * A caller that already has the reference library does not need this: it
 * serialises its own std::vector<GuardedCommand>.  This
 * builder lets the engine, its tests and its benchmark construct the five
 * benchmark configurations without the reference present.
 *
 * Constraint expressions are prefix int32 streams:
 *   PCCP_C_SUM  n (coef slot)*n c      sum coef*x <= c, coef >= 0   (linear_leq)
 *   PCCP_C_LEQ  xc x offset yc y       x + offset <= y; xc/yc = 1 marks a constant operand
 *   PCCP_C_AND  <a> <b>
 *   PCCP_C_IFF  <a> <b>
 *   PCCP_C_NOT  <a>
 */
#ifndef PCCP_HOST_H
#define PCCP_HOST_H

#include <stdint.h>

#include "pccp_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

enum { PCCP_C_SUM = 0, PCCP_C_LEQ = 1, PCCP_C_AND = 2, PCCP_C_IFF = 3, PCCP_C_NOT = 4 };

typedef struct pccp_host_model pccp_host_model;

const char* pccp_host_last_error(void);

pccp_host_model* pccp_host_new(void);
void pccp_host_free(pccp_host_model* m);

/* Benchmark configurations. */
pccp_host_model* pccp_host_nqueens(int32_t n);
pccp_host_model* pccp_host_random_csp(uint64_t seed, int32_t n_vars, int32_t n_cons, int32_t dom_hi);
pccp_host_model* pccp_host_rcpsp_random(uint64_t seed, int32_t n_real, int32_t resources);
pccp_host_model* pccp_host_rcpsp_patterson(const char* text);
/* usage is n_tasks x n_res row-major; prec is n_prec (i, j) pairs. */
pccp_host_model* pccp_host_rcpsp(int32_t n_tasks, const int32_t* duration, int32_t n_res,
                                 const int32_t* usage, const int32_t* capacity, int32_t n_prec,
                                 const int32_t* prec, int32_t horizon);

/* Generic construction. Return the new slot / PCCP_OK, or -1 / PCCP_EMODEL on error. */
int32_t pccp_host_add_cell(pccp_host_model* m, int32_t kind);
int pccp_host_tell(pccp_host_model* m, int32_t slot, int32_t lo, int32_t hi);
int pccp_host_post(pccp_host_model* m, const int32_t* expr, int32_t len);
int pccp_host_post_reified(pccp_host_model* m, int32_t b, const int32_t* expr, int32_t len);
int pccp_host_set_objective(pccp_host_model* m, int32_t slot);
int pccp_host_set_candidates(pccp_host_model* m, const int32_t* slots, int32_t n);

/* Borrowed view of the flat tables; valid until the model is mutated or freed. */
int pccp_host_view(pccp_host_model* m, pccp_model* out);
/* Bottom store (Store::reset): n_words int32. */
int pccp_host_bottom(const pccp_host_model* m, int32_t* words);

/* RCPSP models only: number of tasks, their start slots, and
 * check_solution on the start lower bounds of a store (1 valid, 0 invalid, -1 error). */
int32_t pccp_host_rcpsp_tasks(const pccp_host_model* m);
int pccp_host_rcpsp_starts(const pccp_host_model* m, int32_t* slots);
int pccp_host_rcpsp_check(const pccp_host_model* m, const int32_t* words);

#ifdef __cplusplus
}
#endif

#endif
