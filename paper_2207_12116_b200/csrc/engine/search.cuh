// search.cuh — node processing, EPS decomposition and the persistent DFS.
//
// Node = materialisation + fixed point (materialize, solver.cpp:91-102).  The
// device keeps the parent's fixed point instead of replaying the decision path
// from the subproblem root: the fixed point above (parent fixpoint ⊔ decision
// ⊔ objective bound) equals the fixed point above (root ⊔ path ⊔ bound) — the
// reference's own "replay = incremental descent" property
// (test_solver.cpp:196-227) — and tests/test_gpu_parity.py replays sampled
// paths on the CPU oracle to prove it per node.
#pragma once

#include "kernels.cuh"

namespace pccp_b200 {
namespace dev {

struct SearchCtl {
  Globals* G;
  int* best_store;       // n_words, the best solution store
  Globals* const* peers; // peer contexts' globals: incumbent replicas, done flags (system-scope atomics)
  int n_peers;
  int bound;             // join obj <= best-1 at materialisation (0 in the shared EPS phase of N shards)
  int mode;              // 0: enumerate, 1: minimise the objective
  int hash;              // accumulate the fixed-point hash-sum
  int depth_cap;         // < 0: none
  int count;             // accumulate counters (EPS on shard 0 only)
  const int* blob;       // the tables in global memory (the cold ones: folds, decode table)
  // node audit (pccp_gpu_audit): every 2^audit_shift-th materialisation of the
  // persistent search, up to audit_n samples of (pre, post, failed)
  int* audit_pre;
  int* audit_post;
  unsigned char* audit_failed;
  int audit_n, audit_shift;
};

// Per-group counters, kept in shared memory (Frame::cnt) and updated by the
// group's rank 0 only: 7 u64 held in registers by every lane would cost the
// search kernels 14 registers each, i.e. resident groups.
struct Cnt {
  unsigned long long nodes = 0, fails = 0, sols = 0, open = 0, hash = 0, rounds = 0, maxd = 0, pad = 0;
};

__device__ __forceinline__ void flush(Globals* G, Cnt& c) {
  if (c.nodes) atomicAdd(&G->nodes, c.nodes);
  if (c.fails) atomicAdd(&G->failures, c.fails);
  if (c.sols) atomicAdd(&G->solutions, c.sols);
  if (c.open) atomicAdd(&G->open_leaves, c.open);
  if (c.hash) atomicAdd(&G->hash_sum, c.hash);
  if (c.rounds) atomicAdd(&G->rounds, c.rounds);
  if (c.maxd) atomicMax(&G->max_depth, c.maxd);
  c = Cnt{};
}

__device__ __forceinline__ unsigned long long word_bit(int w) { return w < 64 ? 1ull << w : 0ull; }

// Per-group control prefetch (rank 0 only).  The search's per-node control
// reads — the stop flag, the incumbent (solver.cpp:96-99) and the donation
// hunger — are L2 round trips that the whole group would wait for at the
// node's first barrier.  Rank 0 instead fetches both 16-byte Globals blocks
// into shared memory with cp.async.cg (L2, coherent with the atomics) when a
// node starts and reads them when the next one starts: the latency hides
// behind the node's propagation.  Values one node old are sound: a stale stop
// flag stops one node later; a stale incumbent is still some solution's value,
// only a weaker bound (`own` keeps the group's own improvements exact).
struct alignas(16) Pf {
  int ctl[4];   // cursor, stop, incomplete, incumbent
  int hung[4];  // hungry, padding
  int own;      // best value this group recorded (INT_MAX: none)
  int inc;      // the incumbent of the last completed prefetch (ctl[3] may be in flight again)
  int pad[2];   // pad[0]: the next node's control word (CTA groups); pad[1]: node tick (remote donation)
};

__device__ __forceinline__ void prefetch_ctl(Pf* pf, const Globals* G) {
  const unsigned d0 = (unsigned)__cvta_generic_to_shared(pf->ctl), d1 = (unsigned)__cvta_generic_to_shared(pf->hung);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d0), "l"(&G->cursor) : "memory");
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d1), "l"(&G->hungry) : "memory");
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void prefetch_wait() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Objective tightening at materialisation (solver.cpp:96-99): obj <= best-1.
// Returns the dirty bit of the objective's ub word when it moved (uniform).
// dm (filtered kPacked rounds): rank 0 marks the objective's start when it moved.
template <class G>
__device__ __forceinline__ unsigned long long join_objective(const G& g, volatile int* S, const DeviceLayout& L,
                                                             const SearchCtl& C, const Pf* pf = nullptr,
                                                             unsigned dm = 0) {
  if (C.mode != 1 || !C.bound || L.obj_lbw < 0) return 0ull;
  int moved = 0;
  if (g.rank() == 0) {
    const int best = pf ? min(*(volatile const int*)&pf->inc, *(volatile const int*)&pf->own)
                        : *(volatile int*)&C.G->incumbent;
    if (best != INT_MAX) moved = join_min(S, L.obj_lbw + 1, best - 1) ? 1 : 0;
    if (moved && dm) smark(dm, (unsigned)L.obj_lbw >> 1);
  }
  // Only the filtered rounds use the dirty mask; the eventless loop needs no
  // broadcast (callers sync before propagating).
  if (!L.filtered) return 0ull;
  return g.bcast0(moved) ? word_bit(L.obj_lbw + 1) : 0ull;
}

// SharedControl::should_stop (solver.cpp:68-76): stop flag, timeout, node limit.
// The limit checks of one materialisation, on the group's rank 0.
__device__ __forceinline__ int stop_rank0(const SearchCtl& C, const Pf* pf = nullptr) {
  int stop = 0;
  {
    Globals* Gl = C.G;
    stop = pf ? *(volatile const int*)&pf->ctl[1] : *(volatile int*)&Gl->stop;  // also raised by a peer's proof (k_signal_done)
    if (!stop && Gl->timeout_ns && globaltimer() - Gl->t0 >= Gl->timeout_ns) {
      atomicCAS(&Gl->stop, 0, 1);
      stop = 1;
    }
    if (!stop && Gl->stall_ns && *(volatile int*)&Gl->incumbent != INT_MAX &&
        globaltimer() - Gl->t0 - *(volatile unsigned long long*)&Gl->last_impr_ns >= Gl->stall_ns) {
      Gl->stalled = 1;
      atomicCAS(&Gl->stop, 0, 1);
      stop = 1;
    }
    if (!stop && Gl->node_limit != ~0ull) {
      // one reservation per materialisation; the limit admits exactly node_limit nodes
      if (atomicAdd(&Gl->nodes_reserved, 1ull) >= Gl->node_limit) {
        atomicCAS(&Gl->stop, 0, 1);
        stop = 1;
      }
    }
  }
  return stop;
}

template <class G>
__device__ __forceinline__ bool should_stop(const G& g, const SearchCtl& C) {
  return g.bcast0(g.rank() == 0 ? stop_rank0(C) : 0) != 0;
}

// The stop flag and the timeout only (no node reservation): checked by the
// EPS decomposition per parent, as decompose() checks should_stop
// (solver.cpp:189).
template <class G>
__device__ __forceinline__ bool time_stop(const G& g, const SearchCtl& C, unsigned reserve = 0) {
  int stop = 0;
  if (g.rank() == 0) {
    Globals* Gl = C.G;
    stop = *(volatile int*)&Gl->stop;
    if (!stop && Gl->timeout_ns && globaltimer() - Gl->t0 >= Gl->timeout_ns) {
      atomicCAS(&Gl->stop, 0, 1);
      stop = 1;
    }
    // the materialisations about to happen count against the node limit, as
    // every materialisation does in the reference (solver.cpp:68-76, 100)
    if (!stop && reserve && Gl->node_limit != ~0ull &&
        atomicAdd(&Gl->nodes_reserved, (unsigned long long)reserve) + reserve > Gl->node_limit) {
      atomicCAS(&Gl->stop, 0, 1);
      stop = 1;
    }
  }
  return g.bcast0(stop) != 0;
}

// record_solution + Objective::improve (solver.cpp:104-118, solver.hpp:43-49):
// CAS-min on the incumbent, pushed to every peer GPU's replica.  Under the
// lock (the reference's solution mutex) a solution that still beats
// best_value is an improvement: its store is copied, it is counted and it is
// logged, so the log is strictly decreasing (test_solver.cpp:247-261).
template <class G>
__device__ void record_solution(const G& g, volatile int* S, const DeviceLayout& L, const SearchCtl& C, Cnt& cnt,
                                Pf* pf = nullptr) {
  Globals* Gl = C.G;
  const int value = S[L.obj_lbw];
  int improved = 0;
  if (g.rank() == 0) {
    if (pf && value < pf->own) pf->own = value;
    const int old = atomicMin(&Gl->incumbent, value);
    improved = value < old;
    if (improved) {
      for (int p = 0; p < C.n_peers; ++p) atomicMin_system(&C.peers[p]->incumbent, value);
      while (atomicCAS(&Gl->best_lock, 0, 1) != 0) {
      }
    }
  }
  improved = g.bcast0(improved);
  if (!improved) return;
  int do_copy = 0;
  if (g.rank() == 0) do_copy = value < *(volatile int*)&Gl->best_value;
  do_copy = g.bcast0(do_copy);
  if (do_copy) copy_out(g, C.best_store, S, (int)L.n_words);
  __threadfence();
  g.sync();
  if (g.rank() == 0) {
    if (do_copy) {
      *(volatile int*)&Gl->best_value = value;
      if (C.count) ++cnt.sols;
      const int k = Gl->n_impr++ & 63;  // ring of the last 64 improvements, written under the lock
      const unsigned long long t = globaltimer() - Gl->t0;
      Gl->impr_val[k] = value;
      Gl->impr_ns[k] = t;
      *(volatile unsigned long long*)&Gl->last_impr_ns = t;
    }
    __threadfence();
    atomicExch(&Gl->best_lock, 0);
  }
}

// After a node's fixed point: count, hash, classify.  Returns 1 when the node
// must be expanded (lbw/mid set), 0 when it is a leaf, -1 on a model error.
template <int F = kAllFamilies, class G>
__device__ int classify(const G& g, volatile int* S, const int* __restrict__ T, const DeviceLayout& L,
                        const SearchCtl& C, Cnt& cnt, bool failed, int depth, int& lbw, int& mid, Pf* pf = nullptr,
                        int vo = -1) {
  if (failed) {
    if (C.count && g.rank() == 0) ++cnt.fails;
    return 0;
  }
  if (C.hash && C.count && g.rank() == 0) {
    // NE-only models are never packed: keep the decoding hash out of that kernel
    if constexpr (F == kNeOnly) cnt.hash += store_hash(S, (int)L.n_words);
    else cnt.hash += store_hash_ref(S, C.blob, L);
  }
  const int b = branch(g, S, T, L, lbw, mid, vo);
  if (b < 0) {
    if (g.rank() == 0) {
      C.G->error_code = 1;
      atomicExch(&C.G->stop, 2);
    }
    return -1;
  }
  if (b == 0) {  // every candidate fixed: a solution
    if (C.mode == 1) record_solution(g, S, L, C, cnt, pf);
    else if (C.count && g.rank() == 0) ++cnt.sols;
    return 0;
  }
  if (C.depth_cap >= 0 && depth >= C.depth_cap) {
    if (C.count && g.rank() == 0) ++cnt.open;
    return 0;
  }
  return 1;
}

// Kernel prologue: optional smem copy of the tables, CTA scratch, group store.
constexpr int kFrameCtl = 4 + 2 * 64;  // ints: the 4-int ring + 64 u64 of reduction slots
struct Frame {
  const int* __restrict__ T;
  int* ring;
  unsigned long long* red;
  Cnt* cnt;  // one per group of the CTA
  Pf* pf;    // one per group of the CTA
  int* dm;   // dirty masks of filtered kPacked rounds, dm_words per group
  int dm_words;
  int* stores;
};

// The command tables are staged into shared memory by the bulk-copy engine
// (cp.async.bulk, TMA's 1-D form): thread 0 arms an mbarrier with the byte
// count and issues the copies; the CTA sets up the rest meanwhile and waits
// on the barrier's phase 0.
__device__ __forceinline__ void stage_table(const int* blob, int* dst, unsigned bytes) {
  __shared__ __align__(8) unsigned long long tbar;
  const unsigned mb = (unsigned)__cvta_generic_to_shared(&tbar);
  const unsigned sd = (unsigned)__cvta_generic_to_shared(dst);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
    constexpr unsigned kChunk = 32768;
    for (unsigned o = 0; o < bytes; o += kChunk) {
      const unsigned n = bytes - o < kChunk ? bytes - o : kChunk;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(sd + o), "l"(reinterpret_cast<const char*>(blob) + o), "r"(n), "r"(mb)
                   : "memory");
    }
  }
  __syncthreads();  // the barrier is initialised before anyone waits on it
  asm volatile(
      "{\n .reg .pred done;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 done, [%0], 0;\n"
      " @!done bra WAIT_%=;\n}" ::"r"(mb)
      : "memory");
}

__device__ __forceinline__ Frame frame(const Model& M) {
  extern __shared__ __align__(16) int smem[];
  Frame f;
  int off = 0;
  f.T = M.blob;
  if (M.table_in_smem) {  // the hot prefix (lower.cpp hot_words); folds and the decode table stay global
    const int n4 = ((int)M.L.hot_words + 3) >> 2;
    stage_table(M.blob, smem, (unsigned)n4 * 16u);
    f.T = smem;
    off = n4 * 4;
  }
  f.ring = smem + off;
  f.red = reinterpret_cast<unsigned long long*>(smem + off + 4);
  off += kFrameCtl;
  f.cnt = reinterpret_cast<Cnt*>(smem + off);
  for (int i = threadIdx.x; i < M.cnt_slots * (int)(sizeof(Cnt) / 8); i += blockDim.x)
    reinterpret_cast<unsigned long long*>(f.cnt)[i] = 0ull;
  off += M.cnt_slots * (int)(sizeof(Cnt) / 4);
  f.pf = reinterpret_cast<Pf*>(smem + off);
  for (int i = threadIdx.x; i < M.cnt_slots; i += blockDim.x) {
    f.pf[i].own = f.pf[i].inc = INT_MAX;
    f.pf[i].pad[1] = 0;
  }
  off += M.cnt_slots * (int)(sizeof(Pf) / 4);
  f.dm = smem + off;  // filtered kPacked rounds: zero between propagations (propagate_packed)
  for (int i = threadIdx.x; i < M.cnt_slots * M.dm_words; i += blockDim.x) f.dm[i] = 0;
  off += M.cnt_slots * M.dm_words;
  f.dm_words = M.dm_words;
  f.stores = smem + off;
  __syncthreads();
  return f;
}

template <bool TS>
__device__ __forceinline__ Tab<TS> make_tab(const Frame& f) {
  Tab<TS> t;
  t.p = f.T;
  t.base = 0;
  if constexpr (TS) t.base = (unsigned)__cvta_generic_to_shared((const void*)f.T);
  return t;
}

// The constant-zero word Z read by absent unit-record terms; never written.
template <class G>
__device__ __forceinline__ unsigned init_store(const G& g, volatile int* S, const DeviceLayout& L) {
  if (g.rank() == 0) S[L.zero_word] = 0;
  g.sync();
  return (unsigned)__cvta_generic_to_shared((const void*)S);
}

template <class G>
struct GroupOf;
template <>
struct GroupOf<WarpGroup> {
  static __device__ __forceinline__ WarpGroup make(const Frame&) { return WarpGroup{(int)(threadIdx.x & 31)}; }
  static __device__ __forceinline__ int in_cta() { return (int)(threadIdx.x >> 5); }
  static __device__ __forceinline__ int per_cta() { return (int)(blockDim.x >> 5); }
};
template <>
struct GroupOf<CtaGroup> {
  static __device__ __forceinline__ CtaGroup make(const Frame& f) {
    return CtaGroup{(int)threadIdx.x, (int)blockDim.x, f.ring, f.red};
  }
  static __device__ __forceinline__ int in_cta() { return 0; }
  static __device__ __forceinline__ int per_cta() { return 1; }
};

// Shared address of this group's dirty masks (filtered kPacked rounds; 0 when none).
template <class G>
__device__ __forceinline__ unsigned dm_addr(const Frame& f) {
  if (!f.dm_words) return 0u;
  return (unsigned)__cvta_generic_to_shared(f.dm + GroupOf<G>::in_cta() * f.dm_words);
}

// Launch bounds: warp groups run <= 8 warps per CTA; CTA groups up to 1024
// threads.  Both give ptxas a 64-register budget (at least 4 CTAs of 8 warps);
// the NE-only warp kernel gets 40 (6 CTAs of 8 warps).
template <class G, int F>
struct MaxThreads {
  static constexpr int value = 1024;
  static constexpr int min_blocks = 1;
};
#ifndef PCCP_WARP_MIN_BLOCKS
#define PCCP_WARP_MIN_BLOCKS 4
#endif
#ifndef PCCP_NE_MIN_BLOCKS
#define PCCP_NE_MIN_BLOCKS 6
#endif
template <int F>
struct MaxThreads<WarpGroup, F> {
  static constexpr int value = 256;
  static constexpr int min_blocks = F == kNeOnly ? PCCP_NE_MIN_BLOCKS : PCCP_WARP_MIN_BLOCKS;
};

// ---- K1: batched fixed points (run_sequential on N independent stores) ---------
template <class G, bool TS, int F>
__global__ void __launch_bounds__(MaxThreads<G, F>::value, MaxThreads<G, F>::min_blocks) k_propagate(Model M, int* stores, int n, int stride, unsigned char* status, unsigned* rounds,
                            int fold) {
  const Frame f = frame(M);
  const G g = GroupOf<G>::make(f);
  const Tab<TS> tab = make_tab<TS>(f);
  volatile int* S = f.stores + GroupOf<G>::in_cta() * M.store_stride;
  const unsigned sb = init_store(g, S, M.L);
  const int gid = blockIdx.x * GroupOf<G>::per_cta() + GroupOf<G>::in_cta();
  const int ng = gridDim.x * GroupOf<G>::per_cta();
  for (int i = gid; i < n; i += ng) {
    int* io = stores + (size_t)i * stride;
    copy_words(g, S, io, (int)M.L.n_words);
    g.sync();
    if (fold) {
      apply_fold(g, S, M.blob, M.L);
      g.sync();
    }
    int r = 0;
    const bool failed = propagate<G, TS, F>(g, S, sb, tab, M.L, r, kAllDirty, dm_addr<G>(f));
    copy_out(g, io, S, (int)M.L.n_words);
    if (g.rank() == 0) {
      status[i] = failed ? 1 : 0;
      if (rounds) rounds[i] = (unsigned)r;
    }
    g.sync();
  }
}

// ---- the problem root: fold, objective, fixed point, classification ----------------
template <class G, bool TS, int F>
__global__ void __launch_bounds__(MaxThreads<G, F>::value, MaxThreads<G, F>::min_blocks) k_root(Model M, SearchCtl C, int* store, unsigned char* flag) {
  const Frame f = frame(M);
  const G g = GroupOf<G>::make(f);
  const Tab<TS> tab = make_tab<TS>(f);
  if (GroupOf<G>::in_cta() != 0 || blockIdx.x != 0) return;
  volatile int* S = f.stores;
  const unsigned sb = init_store(g, S, M.L);
  Cnt& cnt = f.cnt[GroupOf<G>::in_cta()];
  copy_words(g, S, store, (int)M.L.n_words);
  g.sync();
  apply_fold(g, S, M.blob, M.L);
  g.sync();
  join_objective(g, S, M.L, C);
  if (g.rank() == 0 && C.G->node_limit != ~0ull) atomicAdd(&C.G->nodes_reserved, 1ull);  // the root's materialisation
  g.sync();
  int r = 0;
  const bool failed = propagate<G, TS, F>(g, S, sb, tab, M.L, r, kAllDirty, dm_addr<G>(f));
  if (C.count && g.rank() == 0) {
    ++cnt.nodes;
    cnt.rounds += (unsigned long long)r;
  }
  int lbw = 0, mid = 0;
  const int e = classify<F>(g, S, f.T, M.L, C, cnt, failed, 0, lbw, mid);
  copy_out(g, store, S, (int)M.L.n_words);
  if (g.rank() == 0) {
    *flag = e == 1 ? 1 : 0;
    flush(C.G, cnt);
  }
}

// ---- K5: the EPS decomposition (decompose, solver.cpp:180-213) ----------------
// Whole BFS levels in one persistent launch: every CTA is resident (the grid
// is the kernel's occupancy), levels are separated by a software grid
// barrier, and the compaction into the next frontier runs in-kernel, so a
// level costs a few microseconds of synchronisation instead of two launches
// and a host round trip.  Parent p's children go to slots 2p (left, x <= mid)
// and 2p+1 (right); the stable compaction keeps BFS order, so the frontier is
// identical on every GPU.  Levels run while the frontier is non-empty, below
// `target` and no model error has stopped the search.
struct DecState {
  int count;   // current frontier size
  int levels;  // levels expanded so far
};

// Sense-reversing grid barrier over gridDim.x resident CTAs (bar[0] arrivals,
// bar[1] generation).  Every CTA must call it the same number of times.
__device__ __forceinline__ void grid_sync(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned gen = *(volatile unsigned*)&bar[1];
    __threadfence();
    if (atomicAdd(&bar[0], 1u) == gridDim.x - 1) {
      *(volatile unsigned*)&bar[0] = 0;
      __threadfence();
      atomicAdd(&bar[1], 1u);
    } else {
      while (*(volatile unsigned*)&bar[1] == gen) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

// grid_sync that also snapshots *stop: the last CTA to arrive copies it into
// bar[2] before releasing the others, so every CTA reads the same value (a
// stop raised by the next level's expansion cannot reach a CTA that is still
// deciding whether to run it).  bar[2] is rewritten only at the next barrier,
// which no CTA reaches before every CTA has read it.
__device__ __forceinline__ int grid_sync_snap(unsigned* bar, const int* stop) {
  __shared__ int snap;
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned gen = *(volatile unsigned*)&bar[1];
    __threadfence();
    if (atomicAdd(&bar[0], 1u) == gridDim.x - 1) {
      __threadfence();
      *(volatile int*)&bar[2] = *(volatile const int*)stop;
      *(volatile unsigned*)&bar[0] = 0;
      __threadfence();
      atomicAdd(&bar[1], 1u);
    } else {
      while (*(volatile unsigned*)&bar[1] == gen) __nanosleep(32);
    }
    __threadfence();
    snap = *(volatile int*)&bar[2];
  }
  __syncthreads();
  return snap;
}

// Compaction of a small level (n <= 32 x blockDim flags) without a grid
// barrier: every CTA scans all n flags itself (thread t: flags [32t, 32t+32),
// two 16-byte loads past L1) and writes the index entries its own groups
// will read next (see expand_level's assignment below), so the CTAs together
// write all of them.  Returns the total on every thread.
__device__ __forceinline__ int small_compact(const unsigned char* flags, int n, int* idx, int per_cta) {
  __shared__ int wtot[33];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = (int)(blockDim.x >> 5);
  const int lo = 32 * tid;
  unsigned bits = 0;
  if (lo < n) {
    // two independent 16-byte loads through L2 (ld.global.cg: past this SM's
    // L1, which may hold a previous level's flags), issued together
    const uint4* w = reinterpret_cast<const uint4*>(flags + lo);
    const uint4 a = __ldcg(w), b = lo + 16 < n ? __ldcg(w + 1) : make_uint4(0u, 0u, 0u, 0u);
    const unsigned v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
    for (int k = 0; k < 8; ++k)  // bytes are 0 or 1
      bits |= ((v[k] & 1u) | ((v[k] >> 7) & 2u) | ((v[k] >> 14) & 4u) | ((v[k] >> 21) & 8u)) << (4 * k);
    if (n - lo < 32) bits &= (1u << (n - lo)) - 1u;  // bytes past n are a previous level's
  }
  const int c = __popc(bits);
  int incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) wtot[wid] = incl;
  __syncthreads();
  int before = 0, total = 0;
  for (int k = 0; k < nw; ++k) {
    const int t = wtot[k];
    before += k < wid ? t : 0;
    total += t;
  }
  // this thread's positions p0, p0 + 1, ... in set-bit order: only the ones
  // this CTA's groups read next are written.  expand_level hands parent p to
  // group p mod ng, or, when the next level splits (2 total <= ng), its two
  // children to groups 2p and 2p + 1.
  if (c) {
    const int p0 = before + incl - c, G = (int)gridDim.x, B = (int)blockIdx.x;
    int p = p0;
    if (2 * total <= G * per_cta) {  // items [B per_cta, (B+1) per_cta) hold 2p or 2p+1 for p in [plo, phi]
      const int plo = (B * per_cta) >> 1, phi = ((B + 1) * per_cta - 1) >> 1;
      for (unsigned b = bits; b; b &= b - 1u, ++p)
        if (p >= plo && p <= phi) idx[p] = lo + __ffs((int)b) - 1;
    } else {
      int q = p0 / per_cta;
      int r = (B - q) % G;
      q += r < 0 ? r + G : r;
      int ws = q * per_cta;  // the next owned window [ws, ws + per_cta): q = blockIdx.x + m gridDim.x
      for (unsigned b = bits; b; b &= b - 1u, ++p) {
        if (p >= ws + per_cta) ws += G * per_cta;
        if (p >= ws) idx[p] = lo + __ffs((int)b) - 1;
      }
    }
  }
  __syncthreads();  // the groups of this CTA read idx next; wtot is reused by the next call
  return total;
}

// Both children of every parent of one level (one group per parent, or one
// per child on small levels).
__device__ unsigned long long* g_dbg_tl = nullptr;  // PCCP_DEBUG_TIMELINE: CTA 0's last parent
__device__ __forceinline__ void dbg_mark(int k) {
#ifdef PCCP_DEBUG_TIMELINE
  if (g_dbg_tl && blockIdx.x == 0 && threadIdx.x == 0 && k < 32) g_dbg_tl[k] = globaltimer();
#endif
}

template <class G, bool TS, int F>
__device__ void expand_level(const G& g, volatile int* S, unsigned sb, const Tab<TS>& tab, const Frame& f,
                             const DeviceLayout& L, const SearchCtl& C, Cnt& cnt, const int* parents,
                             const int* parent_idx, int n_par, int stride, int child_depth, int* children,
                             unsigned char* flags) {
  const int gid = blockIdx.x * GroupOf<G>::per_cta() + GroupOf<G>::in_cta();
  const int ng = gridDim.x * GroupOf<G>::per_cta();
  // A level with fewer parents than half the groups gives each child its own
  // group (both read the parent and take the same decision), so the two
  // children of a parent propagate side by side instead of one after the other.
  const bool split = 2 * n_par <= ng;
  const int n_items = split ? 2 * n_par : n_par;
  for (int j = gid; j < n_items; j += ng) {
    const int p = split ? j >> 1 : j;
    const int side0 = split ? (j & 1) : 0, side1 = split ? (j & 1) : 1;
    if (time_stop(g, C, (unsigned)(side1 - side0 + 1))) {  // abandoned: the subtree is unexplored
      if (g.rank() == 0) {
        C.G->incomplete = 1; atomicOr(&C.G->why, 1);
        for (int side = side0; side <= side1; ++side) flags[2 * p + side] = 0;
      }
      g.sync();
      continue;
    }
    const int* par = parents + (size_t)parent_idx[p] * stride;
    dbg_mark(0);
    copy_words(g, S, par, (int)L.n_words);
    g.sync();
    dbg_mark(1);
    int lbw = 0, mid = 0;
    const int b = branch(g, S, f.T, L, lbw, mid);
    g.sync();  // every thread has read S before rank 0 joins the decision
    dbg_mark(2);
    for (int side = side0; side <= side1; ++side) {
      unsigned char keep = 0;
      if (b == 1) {
        if (side != side0) {
          copy_words(g, S, par, (int)L.n_words);
          g.sync();
        }
        if (g.rank() == 0) {
          if (side == 0) join_min(S, lbw + 1, mid);
          else join_max(S, lbw, mid + 1);
        }
        g.sync();
        unsigned long long dirty = word_bit(side == 0 ? lbw + 1 : lbw);
        dirty |= join_objective(g, S, L, C);
        g.sync();
        int r = 0;
        dbg_mark(3 + 5 * side);
        // (filtered kPacked rounds: every word of a child, no per-node marks here)
        const bool failed =
            propagate<G, TS, F>(g, S, sb, tab, L, r, F == kPackedF ? kAllDirty : dirty, dm_addr<G>(f));
        dbg_mark(4 + 5 * side);
#ifdef PCCP_DEBUG_TIMELINE
        if (g_dbg_tl && blockIdx.x == 0 && threadIdx.x == 0) g_dbg_tl[20 + side] = r;
#endif
        if (C.count && g.rank() == 0) {
          ++cnt.nodes;
          cnt.rounds += (unsigned long long)r;
          if ((unsigned long long)child_depth > cnt.maxd) cnt.maxd = (unsigned long long)child_depth;
        }
        int clbw, cmid;
        const int e = classify<F>(g, S, f.T, L, C, cnt, failed, child_depth, clbw, cmid);
        dbg_mark(5 + 5 * side);
        if (e == 1) {
          copy_out(g, children + (size_t)(2 * p + side) * stride, S, (int)L.n_words);
          keep = 1;
        }
        dbg_mark(6 + 5 * side);
      } else if (b < 0 && g.rank() == 0) {
        C.G->error_code = 1;
        atomicExch(&C.G->stop, 2);
      }
      if (g.rank() == 0) flags[2 * p + side] = keep;
      g.sync();
    }
  }
}

// Stable compaction of flags[0, n) into idx, CTA b owning chunk b: pass 1
// counts each chunk, pass 2 (after a grid barrier) scans its chunk from the
// sum of the earlier chunks.  Returns the total on every thread.
__device__ int grid_compact(const unsigned char* flags, int n, int* idx, int* chunk_count, unsigned* bar) {
  __shared__ int wsum[33];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = (int)(blockDim.x >> 5);
  const int chunk = (n + (int)gridDim.x - 1) / (int)gridDim.x;
  const int lo = min(n, (int)blockIdx.x * chunk), hi = min(n, lo + chunk);
  int mine = 0;
  for (int i = lo + tid; i < hi; i += blockDim.x) mine += flags[i] ? 1 : 0;
  mine = __reduce_add_sync(kFull, mine);
  if (lane == 0) wsum[wid] = mine;
  __syncthreads();
  if (tid == 0) {
    int t = 0;
    for (int w = 0; w < nw; ++w) t += wsum[w];
    chunk_count[blockIdx.x] = t;
  }
  grid_sync(bar);
  // offset of this chunk and the total, from the chunk counts
  int before = 0, total = 0;
  for (int b = tid; b < (int)gridDim.x; b += blockDim.x) {
    const int v = *(volatile int*)&chunk_count[b];
    total += v;
    if (b < (int)blockIdx.x) before += v;
  }
  before = __reduce_add_sync(kFull, before);
  total = __reduce_add_sync(kFull, total);
  __syncthreads();
  if (lane == 0) wsum[wid] = before;
  __syncthreads();
  if (tid == 0) {
    int t = 0;
    for (int w = 0; w < nw; ++w) t += wsum[w];
    wsum[32] = t;
  }
  __syncthreads();
  int base = wsum[32];
  __syncthreads();
  if (lane == 0) wsum[wid] = total;
  __syncthreads();
  if (tid == 0) {
    int t = 0;
    for (int w = 0; w < nw; ++w) t += wsum[w];
    wsum[32] = t;
  }
  __syncthreads();
  total = wsum[32];
  __syncthreads();
  for (int start = lo; start < hi; start += blockDim.x) {
    const int i = start + tid;
    const bool fl = i < hi && flags[i];
    const unsigned m = __ballot_sync(kFull, fl);
    if (lane == 0) wsum[wid] = __popc(m);
    __syncthreads();
    if (tid == 0) {
      int t = 0;
      for (int w = 0; w < nw; ++w) {
        const int c = wsum[w];
        wsum[w] = t;
        t += c;
      }
      wsum[32] = t;
    }
    __syncthreads();
    if (fl) idx[base + wsum[wid] + __popc(m & ((1u << lane) - 1u))] = i;
    base += wsum[32];
    __syncthreads();
  }
  return total;
}

template <class G, bool TS, int F>
__global__ void __launch_bounds__(MaxThreads<G, F>::value, MaxThreads<G, F>::min_blocks)
    k_decompose(Model M, SearchCtl C, int* fb0, int* fb1, int* ib0, int* ib1, DecState* st, int target, int stride,
                unsigned char* flags, int fstride, int* chunk_count, unsigned* bar, unsigned long long* prof) {
  const Frame f = frame(M);
  const G g = GroupOf<G>::make(f);
  const Tab<TS> tab = make_tab<TS>(f);
  volatile int* S = f.stores + GroupOf<G>::in_cta() * M.store_stride;
  const unsigned sb = init_store(g, S, M.L);
  Cnt& cnt = f.cnt[GroupOf<G>::in_cta()];
  int count = *(volatile int*)&st->count;
  int levels = *(volatile int*)&st->levels;
  // no kernel writes stop before the first level: the same value everywhere
  bool err = *(volatile int*)&C.G->stop == 2;
  for (int k = 0;; ++k) {
    if (count <= 0 || count >= target || err) break;  // uniform across the grid
    // ping-pong by selects, not a two-element array (a dynamic index puts it on the stack)
    int* const fsrc = (k & 1) ? fb1 : fb0;
    int* const fdst = (k & 1) ? fb0 : fb1;
    int* const isrc = (k & 1) ? ib1 : ib0;
    int* const idst = (k & 1) ? ib0 : ib1;
    // flags alternate between two buffers: a CTA may expand level k+1 while
    // another still scans level k's flags (small levels have no second barrier)
    unsigned char* fl = flags + (size_t)(k & 1) * (size_t)fstride;
    const bool rec = prof && blockIdx.x == 0 && threadIdx.x == 0 && k < 60;  // PCCP_DEBUG_DEC timeline
    if (rec) prof[4 * k] = globaltimer();
    expand_level<G, TS, F>(g, S, sb, tab, f, M.L, C, cnt, fsrc, isrc, count, stride, levels + 1, fdst,
                           fl);
    err = grid_sync_snap(bar, &C.G->stop) == 2;
    if (rec) prof[4 * k + 1] = globaltimer();
    const bool small = 2 * count <= 32 * (int)blockDim.x;
    count = small ? small_compact(fl, 2 * count, idst, GroupOf<G>::per_cta())
                  : grid_compact(fl, 2 * count, idst, chunk_count, bar);
    if (rec) prof[4 * k + 2] = globaltimer();
    ++levels;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st->count = count;
      st->levels = levels;
    }
    if (!small) grid_sync(bar);  // every CTA has read the chunk counts and agrees on `count`
    if (rec) prof[4 * k + 3] = globaltimer();
  }
  if (g.rank() == 0) flush(C.G, cnt);
}

// Positions shard + k * shards of the shared frontier's index list.
__global__ void k_shard_filter(const int* idx, int* out, int shard, int shards, int n_out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n_out) out[k] = idx[shard + k * shards];
}

// Search start: the clock, and a peer's proof that landed before this
// search's reset (`done` survives resets, `stop` does not).
__global__ void k_init_clock(Globals* G) {
  G->t0 = globaltimer();
  if (*(volatile int*)&G->done) atomicCAS(&G->stop, 0, 1);
}

// A proof over the whole tree (an unsharded primal segment exhausted): every
// peer may stop.  `done` persists across the peer's searches; `stop` ends the
// running one without an extra per-node load (stop_rank0 reads it anyway).
__global__ void k_signal_done(Globals* const* peers, int n) {
  for (int p = 0; p < n; ++p) {
    atomicExch_system(&peers[p]->done, 1);
    atomicCAS_system(&peers[p]->stop, 0, 1);
  }
}

// Offer a bound to the incumbent cell (an objective value some solution has).
__global__ void k_offer_incumbent(Globals* G, int v) { atomicMin(&G->incumbent, v); }

struct SearchParams {
  const int* frontier;
  const int* frontier_idx;
  int n_frontier;
  int stride;
  int depth0;
  int shard_index, shard_count;
  int* stack_pool;
  int stack_depth;   // entries per group
  int entry_stride;  // words per entry: store + (lbw, mid, depth)
  // dynamic load balancing (donation of the shallowest pending right branch)
  int balance;       // 0: off; else the pending branches a group needs before it donates one
  int donate_deep;   // 1: donate the deepest pending branch (the sibling nearest the group's DFS position)
  int mix_order;     // > 0: groups gid % mix_order == 0 branch in var_order 2 (minimisation)
  int* mailbox;      // per group: store (n_words) + (unused, depth, state)
  int mb_stride;
  int* waitq;        // ring of idle group ids (-1: empty)
  int n_groups;
  int value_order;   // 0 left first, 1 right first, 2 odd groups right first
  // cross-GPU work stealing (steal_pop): frontier = the shared phase-A
  // frontier of all shards, this shard's share popped from own_q, then peers'
  int steal;
  unsigned epoch;
  unsigned long long* own_q;
  Globals* const* peers;   // peer contexts' globals (their qcells)
  const int* peer_shard;   // each peer's shard index
  int n_peers;
  int* qlog;               // record_frontier: the positions this shard processed (or null)
  int remote;              // cross-GPU donation to / from the peers (hand_over_remote)
};

// Pop from an epoch-tagged share cell (Globals::qcell): k < n_share of this
// epoch, or -1.  Only the owner installs its epoch on a cell still tagged with
// an older one (position 0 goes to it); a thief takes positions only from
// shares whose owner has started this search, so it never empties the share
// of a peer that is merely a moment late, only the tails of running ones.
// Every position of an epoch is handed out once, whoever pops it.  Linked
// shards run the same sequence of sharded searches (epochs 1, 2, ...), on the
// same root.
__device__ __forceinline__ long long qpop(unsigned long long* q, unsigned e, long long n_share, bool owner) {
  if (!owner) {  // a thief: compare-and-swap, so it never moves a cell of another epoch
    unsigned long long v = atomicAdd_system(q, 0ull);
    for (;;) {
      if ((unsigned)(v >> 32) != e || (long long)(unsigned)v >= n_share) return -1;
      const unsigned long long prev = atomicCAS_system(q, v, v + 1);
      if (prev == v) return (long long)(unsigned)v;
      v = prev;
    }
  }
  for (;;) {
    const unsigned long long v = atomicAdd_system(q, 1ull);
    const unsigned ep = (unsigned)(v >> 32);
    if (ep == e) return (long long)(unsigned)v < n_share ? (long long)(unsigned)v : -1;
    if (ep > e) return -1;  // a later search owns the cell: this one's share was handed out
    unsigned long long cur = v + 1;
    while ((unsigned)(cur >> 32) < e) {
      const unsigned long long prev = atomicCAS_system(q, cur, ((unsigned long long)e << 32) | 1ull);
      if (prev == cur) return 0;
      cur = prev;
    }
  }
}

// The next frontier position for a group of this shard: its own share first,
// then the peers' shares (work stealing: a GPU that drained its share takes
// positions another GPU has not reached yet).  -1 when all are handed out.
__device__ __forceinline__ long long steal_pop(const SearchParams& P, Globals* Gl) {
  const long long N = P.shard_count, n = P.n_frontier;
  auto share = [&](long long s) { return n > s ? (n - s + N - 1) / N : 0ll; };
  long long k = qpop(P.own_q, P.epoch, share(P.shard_index), true);
  if (k >= 0) return P.shard_index + k * N;
  for (int j = 0; j < P.n_peers; ++j) {
    const int s = P.peer_shard[j];
    k = qpop(&P.peers[j]->qcell, P.epoch, share(s), false);
    if (k >= 0) {
      atomicAdd(&Gl->stolen, 1ull);
      return s + k * N;
    }
  }
  return -1;
}

// A pending stack entry stores (parent fixed point, lbw | pending_left << 31,
// mid, depth); apply its pending branch to a store.
__device__ __forceinline__ void apply_pending(int* dst, int lbw_tag, int mid) {
  const int lbw = lbw_tag & 0x7fffffff;
  if (lbw_tag < 0) {  // pending left branch: x <= mid
    if (mid < dst[lbw + 1]) dst[lbw + 1] = mid;
  } else if (mid + 1 > dst[lbw]) {  // pending right branch: x >= mid+1
    dst[lbw] = mid + 1;
  }
}

// Donation: an idle group registers in the wait ring and announces hunger; a
// busy group that sees hunger and has >= 2 pending right branches claims one
// unit of hunger, takes the receiver id, marks it active (so termination —
// no active group — can never be observed mid-handoff), and writes its
// shallowest pending node (parent fixed point + right decision, not yet
// propagated) into the receiver's mailbox.  The receiver materialises and
// counts that node itself, so every node is still processed exactly once.
// Rank 0: claim one unit of hunger (1) or not (0).
__device__ __forceinline__ int claim_donation_rank0(Globals* Gl, const Pf* pf) {
  // the hunger from the prefetch when there is one; the claim itself is atomic
  if ((pf ? *(volatile const int*)&pf->hung[0] : *(volatile int*)&Gl->hungry) <= 0) return 0;
  if (atomicAdd(&Gl->hungry, -1) > 0) return 1;
  atomicAdd(&Gl->hungry, 1);
  return 0;
}

// After a claim: take the receiver from the wait ring and hand it the
// shallowest pending node.
template <class G>
__device__ __forceinline__ void hand_over(const G& g, const SearchParams& P, Globals* Gl, int* stk, int nw, int& bot,
                                          int& sp) {
  int recv = -1;
  if (g.rank() == 0) {
    const unsigned h = atomicAdd(&Gl->wait_head, 1u) % (unsigned)P.n_groups;
    while ((recv = *(volatile int*)&P.waitq[h]) < 0) {
    }
    P.waitq[h] = -1;
    atomicAdd(&Gl->active, 1);
    atomicAdd(&Gl->donations, 1ull);
  }
  recv = g.bcast0(recv);
  const int at = P.donate_deep ? sp - 1 : bot;
  const int* ent = stk + (size_t)at * P.entry_stride;
  int* dst = P.mailbox + (size_t)recv * P.mb_stride;
  for (int i = g.rank(); i < nw; i += g.size()) dst[i] = ent[i];
  g.sync();
  if (g.rank() == 0) {
    apply_pending(dst, ent[nw], ent[nw + 1]);
    dst[nw + 1] = ent[nw + 2] + 1;
    __threadfence();
    *(volatile int*)&dst[nw + 2] = 1;
  }
  if (P.donate_deep) --sp;
  else ++bot;
}

// Cross-GPU donation.  When no group of its own GPU is hungry, a busy group
// with pending branches looks (every 32nd node) for a peer GPU of the same
// epoch whose kernel is running with idle groups, and hands one of them its
// shallowest pending branch, as hand_over does inside a GPU: it claims a free
// inbox slot (CAS 0 -> 1) and one unit of the peer's hunger, takes the
// receiver from the peer's wait ring, marks it active, writes the node into
// the slot through NVLink (peer stores), fences at system scope and flags the
// slot ready for that receiver.  One hunger unit, one ring entry, one
// receiver: the same accounting as a local donation.  Idle groups wait for
// donations while a fully resident peer is busy (peers_busy); a group leaving
// the kernel closes the inbox first (close_inbox), so no donation lands after
// the kernel ends.
// Rank 0: returns (peer << 8 | slot << 16 | 4) or 0.
__device__ __forceinline__ int claim_remote_rank0(const SearchParams& P, Globals* Gl) {
  // Donate only while every group of this kernel is resident: then the
  // receiver's GPU counts this one busy (peers_busy) and keeps its idle
  // groups — the receiver among them — until the node has landed.  (Its
  // groups leave only at quiescence, so residency holds while this group is
  // active.)  On one device a kernel can be partly resident behind another.
  if (*(volatile int*)&Gl->running < P.n_groups) return 0;
  for (int j = 0; j < P.n_peers; ++j) {
    Globals* B = P.peers[j];
    if (*(volatile int*)&B->running <= 0 || !*(volatile int*)&B->remote || *(volatile int*)&B->stop ||
        *(volatile int*)&B->epoch_pub != (int)P.epoch)
      continue;
    if (*(volatile int*)&B->hungry <= 0) continue;
    // the slot first: while this group holds it (state 1) the peer cannot
    // close its inbox, so it cannot exit (nor its host reset the hunger)
    // under the claim below
    int slot = -1;
    for (int k = 0; k < kInbox && slot < 0; ++k)
      if (atomicCAS_system(&B->inbox_state[k], 0, 1) == 0) slot = k;
    if (slot < 0) continue;
    if (atomicAdd_system(&B->hungry, -1) <= 0) {
      atomicAdd_system(&B->hungry, 1);
      __threadfence_system();
      atomicExch_system(&B->inbox_state[slot], 0);
      continue;
    }
    return 4 | (j << 8) | (slot << 16);
  }
  return 0;
}

// Whether a peer of this epoch that may donate runs its whole kernel (every
// group resident) with an active group: idle groups keep waiting for it.  A
// peer not fully resident is not waited for — on one device its remaining
// CTAs may need this kernel's SMs.
__device__ __forceinline__ bool peers_busy(const SearchParams& P) {
  for (int j = 0; j < P.n_peers; ++j) {
    Globals* B = P.peers[j];
    if (*(volatile int*)&B->remote && *(volatile int*)&B->epoch_pub == (int)P.epoch &&
        *(volatile int*)&B->running >= *(volatile int*)&B->n_groups_pub && *(volatile int*)&B->active > 0)
      return true;
  }
  return false;
}

// At quiescence (no active group here, no busy peer) an idle group closes
// the inbox before it leaves: free slots 0 -> 9, so no donor can claim one
// afterwards — donors claim a slot before the hunger and the ring entry, so
// the hunger and ring entries the idle groups leave behind draw no donation.
// A slot being written or ready (1, 2) means a donation is landing (its donor
// marks a receiver active first): the group keeps waiting.  Returns whether
// every slot is closed.
__device__ __forceinline__ bool close_inbox_quiet(Globals* Gl) {
  bool all = true;
  for (int k = 0; k < kInbox; ++k) {
    const int st = atomicCAS(&Gl->inbox_state[k], 0, 9);
    if (st != 0 && st != 9) all = false;
  }
  return all;
}

// A group leaving the kernel closes this GPU's inbox (slots 0 -> 9): no donor
// can claim a slot afterwards, so none writes into cells its host will reset.
// A slot being written (1) is waited for; a ready one (2) no group will take
// any more: its node is abandoned (the search is incomplete) and the donor's
// activation of the receiver is undone, so this GPU can still become quiet.
__device__ __forceinline__ void close_inbox(Globals* Gl) {
  for (int k = 0; k < kInbox; ++k) {
    for (;;) {
      const int st = *(volatile int*)&Gl->inbox_state[k];
      if (st == 9) break;
      if (st == 1) {
        __nanosleep(100);
        continue;
      }
      if (atomicCAS(&Gl->inbox_state[k], st, 9) != st) continue;
      if (st == 2) {
        Gl->incomplete = 1; atomicOr(&Gl->why, 8);
        atomicAdd(&Gl->active, -1);
      }
      break;
    }
  }
}

template <class G>
__device__ __forceinline__ void hand_over_remote(const G& g, const SearchParams& P, Globals* Gl, int* stk, int nw,
                                                 int& bot, int ctl) {
  const int j = (ctl >> 8) & 0xff, slot = (ctl >> 16) & 0xff;
  Globals* B = P.peers[j];
  if (g.rank() == 0) {
    const unsigned n = (unsigned)*(volatile int*)&B->n_groups_pub;
    const unsigned h = atomicAdd_system(&B->wait_head, 1u) % n;
    volatile int* wq = waitq_of(B);
    int recv;
    while ((recv = wq[h]) < 0) {
    }
    wq[h] = -1;
    atomicAdd_system(&B->active, 1);
    *(volatile int*)&B->inbox_rcv[slot] = recv;
    atomicAdd(&Gl->remote_out, 1ull);
  }
  const int* ent = stk + (size_t)bot * P.entry_stride;
  int* dst = inbox_of(B, slot);
  for (int i = g.rank(); i < nw; i += g.size()) dst[i] = ent[i];
  g.sync();
  if (g.rank() == 0) {
    apply_pending(dst, ent[nw], ent[nw + 1]);
    *(volatile int*)&B->inbox_depth[slot] = ent[nw + 2] + 1;
    __threadfence_system();
    *(volatile int*)&B->inbox_state[slot] = 2;
  }
  ++bot;
}

// Rank 0's control for the next node of a CTA group: claim (bit 1), stop
// (bit 0), from the prefetched control words, then the next prefetch.
__device__ __forceinline__ int node_ctl_rank0(const SearchCtl& C, const SearchParams& P, Globals* Gl, Pf* pf,
                                              int pending, bool need_prop) {
  int c = 0;
  prefetch_wait();
  pf->inc = pf->ctl[3];  // join_objective reads this copy: the next prefetch rewrites ctl[]
  if (P.balance && pending >= P.balance) c |= claim_donation_rank0(Gl, pf) << 1;
  if (P.remote && !(c & 2) && P.balance && pending >= P.balance && (++pf->pad[1] & 31) == 0)
    c |= claim_remote_rank0(P, Gl);
  if (need_prop) c |= stop_rank0(C, pf);
  prefetch_ctl(pf, Gl);
  return c;
}

#ifndef PCCP_CTL_MERGE
#define PCCP_CTL_MERGE 1
#endif

// ---- K4 + K6: persistent DFS over the EPS work queue ------------------------------
// Each group pops subproblem k (this GPU owns frontier i = shard_index +
// k*shard_count) and explores it depth-first, left branch first (dfs,
// solver.cpp:122-146).  A branching node pushes (its fixed point, right
// decision) and descends left in place; a leaf pops.  When the queue is
// empty, idle groups are fed by donations (claim_donation_rank0, hand_over).
// Audit: the node-audit instantiation (pccp_gpu_audit), launched only when
// samples are requested, so the production kernel carries no audit code.
template <class G, bool TS, int F, bool Audit = false>
__global__ void __launch_bounds__(MaxThreads<G, F>::value, MaxThreads<G, F>::min_blocks) k_search(Model M, SearchCtl C, SearchParams P) {
  const Frame f = frame(M);
  const G g = GroupOf<G>::make(f);
  const Tab<TS> tab = make_tab<TS>(f);
  volatile int* S = f.stores + GroupOf<G>::in_cta() * M.store_stride;
  const unsigned sb = init_store(g, S, M.L);
  const int gid = blockIdx.x * GroupOf<G>::per_cta() + GroupOf<G>::in_cta();
  const DeviceLayout& L = M.L;
  const int nw = (int)L.n_words;
  int* stk = P.stack_pool + (size_t)gid * (size_t)P.stack_depth * (size_t)P.entry_stride;
  Globals* Gl = C.G;
  Cnt& cnt = f.cnt[GroupOf<G>::in_cta()];
  // the control prefetch pays for CTA groups, whose whole CTA waits at the
  // node's first barrier; a warp group's wait is hidden by the SM's other
  // warps, and the extra instructions cost the issue-bound Q14 kernel 4%
  constexpr bool kPrefetch = std::is_same<G, CtaGroup>::value;
  constexpr bool kMerge = kPrefetch && PCCP_CTL_MERGE;  // the control of the next node before the last barrier
  Pf* pf = kPrefetch ? f.pf + GroupOf<G>::in_cta() : nullptr;
  if (kPrefetch && g.rank() == 0) prefetch_ctl(pf, Gl);
  // filtered kPacked rounds: a node's changes (decision, objective) are marked
  // in the first dirty mask by rank 0 before the propagation
  const unsigned dm = F == kPackedF ? dm_addr<G>(f) : 0u;
  bool queue_open = true;
  // cross-GPU donation is compiled for CTA groups only (the issue-bound Q14
  // warp kernel lost 3% to the extra code; its trees split evenly anyway)
  constexpr bool kRemote = std::is_same<G, CtaGroup>::value;
  if (kRemote && g.rank() == 0) atomicAdd(&Gl->running, 1);  // peers donate only to a GPU whose kernel runs
  const bool right_first = P.value_order == 1 || (P.value_order == 2 && (gid & 1));
  // mixed orders (minimisation): every mix_order-th group branches by the
  // smallest lb, latest start first (var_order 2, the primal dives' order)
  // inside whatever box it explores; every box is still searched completely,
  // so proofs and optima are unchanged (DESIGN: mixed orders)
  const int vo = P.mix_order > 0 && C.mode == 1 && gid % P.mix_order == 0 ? 2 : -1;
  for (;;) {
    int depth = P.depth0;
    bool need_prop = C.mode == 1;
    unsigned long long dirty = 0;  // words changed since the store was last a fixed point
    if (queue_open) {
      long long idx = 0;
      if (g.rank() == 0) {
        if (P.steal) {
          idx = steal_pop(P, Gl);
          if (idx < 0) idx = P.n_frontier;
          else if (P.qlog) P.qlog[atomicAdd(&Gl->qlog_n, 1ull)] = (int)idx;
        } else {
          idx = (long long)P.shard_index + (long long)atomicAdd(&Gl->cursor, 1u) * (long long)P.shard_count;
        }
        if (idx > P.n_frontier) idx = P.n_frontier;
      }
      idx = g.bcast0((int)idx);
      if (idx >= P.n_frontier) queue_open = false;
      else {
        int stop = 0;
        if (g.rank() == 0) stop = *(volatile int*)&Gl->stop;
        if (g.bcast0(stop)) {
          if (g.rank() == 0) {
            Gl->incomplete = 1; atomicOr(&Gl->why, 16);
            atomicAdd(&Gl->active, -1);  // leaves the active set, as every other exit does
          }
          break;
        }
        copy_words(g, S, P.frontier + (size_t)P.frontier_idx[idx] * P.stride, nw);
        g.sync();
      }
    }
    if (!queue_open) {
      if (!P.balance) break;
      // idle: register, then wait for a donation or for global quiescence
      int got = 0;
      if (g.rank() == 0) {
        atomicAdd(&Gl->active, -1);
        const unsigned t = atomicAdd(&Gl->wait_tail, 1u) % (unsigned)P.n_groups;
        *(volatile int*)&P.waitq[t] = gid;
        __threadfence();
        atomicAdd(&Gl->hungry, 1);
        volatile int* state = (volatile int*)&P.mailbox[(size_t)gid * P.mb_stride + nw + 2];
        for (;;) {
          if (*state == 1) {
            got = 1;
            break;
          }
          if (kRemote && P.remote) {  // a peer's donation, addressed to this group
            for (int k = 0; k < kInbox && !got; ++k)
              if (*(volatile int*)&Gl->inbox_state[k] == 2 && *(volatile int*)&Gl->inbox_rcv[k] == gid) got = 2 + k;
            if (got) break;
          }
          // Quiescence: no active group here and no busy peer (whose groups
          // could still hand this one work).  A stopped GPU exits at once,
          // counted incomplete when peers could have donated to it.
          const bool stopped = *(volatile int*)&Gl->stop != 0;
          if (stopped) {
            if (kRemote && P.remote) {
              Gl->incomplete = 1;
              atomicOr(&Gl->why, 4);
            }
            break;
          }
          if (*(volatile int*)&Gl->active == 0 &&
              !(kRemote && P.remote && (peers_busy(P) || !close_inbox_quiet(Gl))))
            break;
          __nanosleep(200);
        }
      }
      got = g.bcast0(got);
      if (!got) break;
      __threadfence();
      if (got == 1) {
        const int* mb = P.mailbox + (size_t)gid * P.mb_stride;
        copy_words(g, S, mb, nw);
        depth = *(volatile const int*)&mb[nw + 1];
        g.sync();
        if (g.rank() == 0) *(volatile int*)&P.mailbox[(size_t)gid * P.mb_stride + nw + 2] = 0;
      } else {  // inbox slot got - 2: the donor marked this GPU active for it
        const int k = got - 2;
        const volatile int* src = inbox_of(Gl, k);  // written over NVLink: volatile loads, past L1
        for (int i = g.rank(); i < nw; i += g.size()) S[i] = src[i];
        depth = *(volatile int*)&Gl->inbox_depth[k];
        g.sync();
        if (g.rank() == 0) {
          atomicAdd(&Gl->remote_in, 1ull);
          *(volatile int*)&Gl->inbox_state[k] = 0;
        }
      }
      need_prop = true;
      dirty = kAllDirty;
    }
    int sp = 0, bot = 0;
    bool abandoned = false;
    bool remat = need_prop && dirty != kAllDirty;  // a frontier node re-materialised under the bound (mode 1)
    if (dm) dirty = kAllDirty;  // a subproblem's first propagation evaluates everything
    // Enumeration: a frontier node was counted and classified during the
    // decomposition.  Minimisation: re-materialise it with the current bound,
    // as dfs() does for its subproblem root.  A donated node is unpropagated.
    if (need_prop) {
      dirty |= join_objective(g, S, L, C);
      g.sync();
    }
    // Rank 0's per-node control (donation claim, limit checks) from the
    // control words prefetched when the previous node started.  CTA groups
    // compute it at the end of the previous node, before that node's last
    // barrier, and publish it in shared memory (pf->pad[0]): no broadcast of
    // its own (two barriers per node fewer).
    bool ctl_ready = false;
    for (;;) {
      int ctl = 0;
      if constexpr (kMerge) {
        if (ctl_ready) {
          ctl = *(volatile int*)&pf->pad[0];
        } else {
          if (g.rank() == 0) ctl = node_ctl_rank0(C, P, Gl, pf, sp - bot, need_prop);
          ctl = g.bcast0(ctl);
        }
        ctl_ready = false;
      } else if constexpr (kPrefetch) {
        if (g.rank() == 0) ctl = node_ctl_rank0(C, P, Gl, pf, sp - bot, need_prop);
        ctl = g.bcast0(ctl);
      } else {
        if (g.rank() == 0) {
          if (P.balance && sp - bot >= P.balance) ctl |= claim_donation_rank0(Gl, pf) << 1;
          if (need_prop) ctl |= stop_rank0(C, pf);
        }
        ctl = g.bcast0(ctl);
      }
      if (ctl & 2) hand_over(g, P, Gl, stk, nw, bot, sp);
      else if (kRemote && (ctl & 4)) hand_over_remote(g, P, Gl, stk, nw, bot, ctl);
      int lbw = 0, mid = 0, e;
      if (need_prop) {
        if (ctl & 1) {
          abandoned = true;
          break;
        }
        int slot = -1;
        if constexpr (Audit) {  // claim an audit slot for this materialisation
          int k = -1;
          if (g.rank() == 0) {
            const unsigned long long t = atomicAdd(&Gl->audit_seen, 1ull);
            if ((t & ((1ull << C.audit_shift) - 1ull)) == 0ull && (t >> C.audit_shift) < (unsigned long long)C.audit_n)
              k = (int)(t >> C.audit_shift);
          }
          slot = g.bcast0(k);
          if (slot >= 0) copy_out(g, C.audit_pre + (size_t)slot * nw, S, nw);
        }
        int r = 0;
        const bool failed = propagate<G, TS, F>(g, S, sb, tab, L, r, dirty, dm);
        if constexpr (Audit) {
          if (slot >= 0) {
            copy_out(g, C.audit_post + (size_t)slot * nw, S, nw);
            if (g.rank() == 0) C.audit_failed[slot] = failed ? 1 : 0;
          }
        }
        if (g.rank() == 0) {
          ++cnt.nodes;
          cnt.rounds += (unsigned long long)r;
          if ((unsigned long long)depth > cnt.maxd) cnt.maxd = (unsigned long long)depth;
          if (remat) atomicAdd(&Gl->rematerialised, 1ull);
        }
        remat = false;
        e = classify<F>(g, S, f.T, L, C, cnt, failed, depth, lbw, mid, pf, vo);
      } else {
        e = branch(g, S, f.T, L, lbw, mid, vo);
      }
      if (e < 0) {
        abandoned = true;
        break;
      }
      if (e == 1) {
        if (sp >= P.stack_depth) {  // capacity: cannot happen with the host's depth bound
          if (g.rank() == 0) {
            Gl->error_code = 2;
            atomicExch(&Gl->stop, 2);
          }
          abandoned = true;
          break;
        }
        int* ent = stk + (size_t)sp * P.entry_stride;
        copy_out(g, ent, S, nw);
        g.sync();  // the parent fixed point is saved before the first decision lands
        if (g.rank() == 0) {
          ent[nw] = right_first ? (int)((unsigned)lbw | 0x80000000u) : lbw;  // the branch left pending
          ent[nw + 1] = mid;
          ent[nw + 2] = depth;
          if (right_first) join_max(S, lbw, mid + 1);  // x >= mid+1 first
          else join_min(S, lbw + 1, mid);              // x <= mid first (dfs(), solver.cpp:139-143)
          if (dm) smark(dm, (unsigned)lbw >> 1);
        }
        ++sp;
        ++depth;
        // rank 0 made the decision join and makes the objective join: one sync
        dirty = word_bit(right_first ? lbw : lbw + 1) | join_objective(g, S, L, C, pf, dm);
        need_prop = true;
        if constexpr (kMerge) {
          if (g.rank() == 0) pf->pad[0] = node_ctl_rank0(C, P, Gl, pf, sp - bot, true);
          ctl_ready = true;
        }
        g.sync();
        continue;
      }
      if (sp == bot) break;
      --sp;
      const int* ent = stk + (size_t)sp * P.entry_stride;
      g.sync();  // no thread still reads the leaf (hash, branch) when it is overwritten
      copy_words(g, S, ent, nw);
      g.sync();
      const int tag = ent[nw];
      if (g.rank() == 0) {
        if (tag < 0) join_min(S, (tag & 0x7fffffff) + 1, ent[nw + 1]);  // pending x <= mid
        else join_max(S, tag, ent[nw + 1] + 1);                        // pending x >= mid+1
        if (dm) smark(dm, (unsigned)(tag & 0x7fffffff) >> 1);
      }
      depth = ent[nw + 2] + 1;
      dirty = word_bit(tag < 0 ? (tag & 0x7fffffff) + 1 : tag);
      dirty |= join_objective(g, S, L, C, pf, dm);  // rank 0, after its decision join
      need_prop = true;
      if constexpr (kMerge) {
        if (g.rank() == 0) pf->pad[0] = node_ctl_rank0(C, P, Gl, pf, sp - bot, true);
        ctl_ready = true;
      }
      g.sync();
    }
    if (g.rank() == 0) {
      if (abandoned) {
        Gl->incomplete = 1;
        atomicOr(&Gl->why, 2);
      }
      flush(Gl, cnt);
    }
    if (abandoned) {
      if (g.rank() == 0) atomicAdd(&Gl->active, -1);
      break;
    }
  }
  if (g.rank() == 0) {
    if (kPrefetch) prefetch_wait();  // no copy into shared memory outlives the CTA
    flush(Gl, cnt);
    if constexpr (kRemote) {
      if (P.remote) close_inbox(Gl);
      __threadfence();
      atomicAdd(&Gl->running, -1);
    }
  }
}

}  // namespace dev
}  // namespace pccp_b200
