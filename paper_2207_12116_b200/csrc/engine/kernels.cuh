// kernels.cuh — sm_100a propagate-and-search kernels.
//
// One *group* of threads owns one search subproblem: either a single warp
// (small stores: many independent subproblems per SM, fixed point detected
// with warp votes) or a whole CTA (large stores: the fixed point detected
// with __syncthreads_or over a 3-slot change ring, engine.cpp:86-116).  The
// group's interval store lives in shared memory; propagators tighten it with
// atomicMax (lb / ZInc words) and atomicMin (ub / ZDec words), the
// lock-free lattice joins of Store::join_word (store.hpp:90-98).  Reads of
// the store go through `volatile` so no word is cached in a register across
// a round (the erratum of PAPER.md:459-460).
//
// Arithmetic is the reference's, bit for bit (H1): term values widen the
// sentinels to +-2^40 and clamp finite products to +-2^40, sums accumulate in
// int64 and narrow back to the int32 sentinels (command.cpp:11-27).
#pragma once

#include <climits>
#include <cstdint>
#include <type_traits>

#include "lower.hpp"

namespace pccp_b200 {
namespace dev {

constexpr long long kWide = 1LL << 40;
constexpr unsigned kFull = 0xffffffffu;

struct Model {
  DeviceLayout L;
  const int* __restrict__ blob;  // global copy of the tables
  int table_in_smem;             // copy the blob into shared memory at kernel start
  int store_stride;              // words per group store in smem (>= n_words, multiple of 4)
  int cnt_slots;                 // groups per CTA (one Cnt each in smem)
  int dm_words;                  // per group: the dirty masks of filtered kPacked rounds (3 x (starts + pairs) words)
};

// Counters and control shared by all groups of one search (global memory).
struct Globals {
  unsigned long long nodes, failures, solutions, open_leaves, hash_sum, rounds, max_depth;
  unsigned long long node_limit;   // ~0: none
  unsigned long long nodes_reserved;  // materialisations admitted against node_limit
  unsigned long long t0;           // %globaltimer at search start
  unsigned long long timeout_ns;   // 0: none
  // {cursor, stop, incomplete, incumbent} and {hungry, active, wait_head,
  // wait_tail} are 16-byte blocks: the search prefetches both per node with
  // cp.async (search.cuh prefetch_ctl)
  alignas(16) unsigned int cursor;  // EPS work queue
  int stop;                        // 1: limit reached, 2: model error
  int incomplete;                  // a subproblem was abandoned
  // [incumbent, n_impr): the cross-rank cells.  With peers linked they are
  // never rewritten by a search's reset (engine.cu reset_globals), only by
  // pccp_gpu_reset_shared / a model load, so a peer's push is never lost.
  int incumbent;                   // best objective, INT_MAX: none (local replica)
  int best_lock;
  int best_value;
  int done;                        // a peer proved optimality over the whole tree: stop
  // Cross-GPU work stealing (search.cuh steal_pop): this shard's share of the
  // shared EPS frontier, popped as qcell = epoch << 32 | k (the k-th position
  // of the share, shard + k * shards) with system-scope atomics by this GPU
  // and, once their own share is exhausted, by its peers.  Kept across
  // searches like the cells above (the epoch tags each sharded search); its
  // own 128-byte line, away from the per-node reads of the cells above.
  alignas(128) unsigned long long qcell;
  unsigned long long qcell_pad[15];
  int n_impr;
  int impr_val[64];
  unsigned long long impr_ns[64];
  int error_code;
  // dynamic load balancing (search.cuh maybe_donate)
  // hungry is read by every busy group each node: its own 128-byte line,
  // away from the idle groups' atomics on active / wait_* (sharing the line
  // cost Q14 0.6%, measured); the prefetch copies its first 16 bytes
  alignas(128) int hungry;      // idle groups waiting for a donation
  int hungry_pad[31];
  int active;                   // groups exploring, or promised a donation
  unsigned wait_head, wait_tail;
  unsigned long long donations;
  // primal restarts (engine.cu pccp_gpu_solve): stop once an incumbent exists
  // and none improved it for stall_ns; `stalled` says the stop was this one
  unsigned long long stall_ns;     // 0: off
  unsigned long long last_impr_ns; // since t0
  int stalled;
  unsigned long long audit_seen;   // materialisations offered to the node audit
  unsigned long long rematerialised;  // frontier nodes materialised again by the search (mode 1)
  unsigned long long qlog_n;          // record_frontier: frontier positions this shard processed
  unsigned long long stolen;          // frontier positions taken from peers' shares
  // Cross-GPU donation (search.cuh hand_over_remote): a peer's busy group
  // hands a pending branch to one of this GPU's idle groups through an inbox
  // slot of this allocation (the wait ring and the slots follow Globals in
  // the same cudaMalloc, so the IPC handle of Globals maps them too).
  int running;                        // groups of this GPU's search kernel inside k_search
  int n_groups_pub;                   // groups of the running search (the wait ring's modulus)
  int remote;                         // this search receives cross-GPU donations
  int epoch_pub;                      // its sharded-search epoch: donations only within one epoch
  int inbox_state[4];                 // 0 free, 1 being written, 2 ready for inbox_rcv, 9 closed
  int inbox_rcv[4];                   // the receiving group (popped from this GPU's wait ring)
  int inbox_depth[4];
  unsigned long long remote_in, remote_out;  // donations received from / sent to peers
  int why;                            // incomplete: 1 decomposition, 2 abandoned, 4 stopped idle, 8 inbox, 16 pop stop
};

// The allocation behind a context's Globals: Globals, then the wait ring of
// idle groups (kMaxGroups ints), then kInbox inbox slots of kSlotWords each.
constexpr int kMaxGroups = 16384, kInbox = 4, kSlotWords = 16384;
constexpr size_t kWaitqOffset = (sizeof(Globals) + 255) & ~size_t(255);
constexpr size_t kInboxOffset = kWaitqOffset + sizeof(int) * kMaxGroups;
constexpr size_t kGlobalsBytes = kInboxOffset + sizeof(int) * (size_t)kInbox * kSlotWords;
__host__ __device__ __forceinline__ int* waitq_of(Globals* G) { return (int*)((char*)G + kWaitqOffset); }
__host__ __device__ __forceinline__ int* inbox_of(Globals* G, int s) {
  return (int*)((char*)G + kInboxOffset) + (size_t)s * kSlotWords;
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// term_value, command.cpp:11-19
__device__ __forceinline__ long long tv(int c, int v) {
  if (v == INT_MAX) return c > 0 ? kWide : (c < 0 ? -kWide : 0);
  if (v == INT_MIN) return c > 0 ? -kWide : (c < 0 ? kWide : 0);
  long long p = (long long)c * (long long)v;
  return p > kWide ? kWide : (p < -kWide ? -kWide : p);
}
__device__ __forceinline__ int narrow(long long a) {
  return a >= INT_MAX ? INT_MAX : (a <= INT_MIN ? INT_MIN : (int)a);
}
__device__ __forceinline__ int tcoef(int x) { return x >> kTermWordBits; }
__device__ __forceinline__ int tword(int x) { return x & (int)kTermWordMask; }

// Store::join_word, store.hpp:90-98: read first, only issue the atomic when
// the value would strictly improve; returns the strict-change flag (bx).
__device__ __forceinline__ bool join_max(volatile int* S, int w, int v) {
  if (v > S[w]) return atomicMax((int*)(S + w), v) < v;
  return false;
}
__device__ __forceinline__ bool join_min(volatile int* S, int w, int v) {
  if (v < S[w]) return atomicMin((int*)(S + w), v) > v;
  return false;
}

// ---- groups --------------------------------------------------------------------

struct WarpGroup {
  int lane;
  __device__ __forceinline__ int rank() const { return lane; }
  __device__ __forceinline__ int size() const { return 32; }
  __device__ __forceinline__ int warp() const { return 0; }
  __device__ __forceinline__ int warps() const { return 1; }
  __device__ __forceinline__ void sync() const { __syncwarp(); }
  __device__ __forceinline__ void round_begin() const {}
  // End of a fixed-point round: one vote per flag.
  __device__ __forceinline__ void round_end(bool ch, bool fl, bool& any_ch, bool& any_fl, int) const {
    __syncwarp();
    any_ch = __any_sync(kFull, ch);
    any_fl = __any_sync(kFull, fl);
  }
  __device__ __forceinline__ bool any(bool p) const { return __any_sync(kFull, p); }
  __device__ __forceinline__ unsigned long long min_u64(unsigned long long v, int = 0) const {
    // all keys below 2^32 (small widths / bounds, or none): one redux.min
    if (__all_sync(kFull, (v >> 32) == 0ull || v == ~0ull)) {
      const unsigned m = __reduce_min_sync(kFull, v == ~0ull ? 0xffffffffu : (unsigned)v);
      return m == 0xffffffffu ? ~0ull : (unsigned long long)m;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long u = __shfl_xor_sync(kFull, v, o);
      v = u < v ? u : v;
    }
    return v;
  }
  __device__ __forceinline__ int bcast0(int v) const { return __shfl_sync(kFull, v, 0); }
  __device__ __forceinline__ unsigned uid() const { return blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); }
};

struct CtaGroup {
  int tid, n;
  int* ring;                 // 4 ints of smem: 3-slot change ring + spare
  unsigned long long* red;   // 64 u64 of smem (two slots of 32 warps)
  __device__ __forceinline__ int rank() const { return tid; }
  __device__ __forceinline__ int size() const { return n; }
  __device__ __forceinline__ int warp() const { return tid >> 5; }
  __device__ __forceinline__ int warps() const { return n >> 5; }
  __device__ __forceinline__ unsigned uid() const { return blockIdx.x; }
  __device__ __forceinline__ void sync() const { __syncthreads(); }
  __device__ __forceinline__ void round_begin() const {
    if (tid < 3) ring[tid] = 0;
    __syncthreads();
  }
  // One barrier per round: round i sets ring[i%3] on change and clears
  // ring[(i+1)%3]; after the barrier everybody reads ring[i%3] (the
  // past/present/future ring of run_parallel, engine.cpp:86-116).
  __device__ __forceinline__ void round_end(bool ch, bool fl, bool& any_ch, bool& any_fl, int i) const {
    if (ch) ring[i % 3] = 1;
    if (tid == 0) ring[(i + 1) % 3] = 0;
    any_fl = __syncthreads_or(fl) != 0;
    any_ch = *(volatile int*)&ring[i % 3] != 0;
  }
  __device__ __forceinline__ bool any(bool p) const { return __syncthreads_or(p) != 0; }
  __device__ __forceinline__ unsigned long long min_u64(unsigned long long v, int = 0) const {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long u = __shfl_xor_sync(kFull, v, o);
      v = u < v ? u : v;
    }
    if ((tid & 31) == 0) red[tid >> 5] = v;
    __syncthreads();
    if (tid < 32) {
      v = tid < (n >> 5) ? red[tid] : ~0ull;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long u = __shfl_xor_sync(kFull, v, o);
        v = u < v ? u : v;
      }
      if (tid == 0) red[32] = v;
    }
    __syncthreads();
    v = red[32];
    __syncthreads();
    return v;
  }
  __device__ __forceinline__ int bcast0(int v) const {
    if (tid == 0) ring[3] = v;
    __syncthreads();
    v = ring[3];
    __syncthreads();
    return v;
  }
};

// ---- table access ------------------------------------------------------------------
// TS = true: the tables were copied into shared memory at kernel start.
template <bool TS>
struct Tab;
template <>
struct Tab<true> {
  const int* p;   // generic view (legacy paths)
  unsigned base;  // shared address of table word 0
  __device__ __forceinline__ int4 ld4(unsigned off, int i) const {
    int4 r;
    asm("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
        : "r"(base + 4u * off + 16u * (unsigned)i));
    return r;
  }
  __device__ __forceinline__ int2 ld2(unsigned off, int i) const {
    int2 r;
    asm("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "r"(base + 4u * off + 8u * (unsigned)i));
    return r;
  }
  __device__ __forceinline__ int ld1(unsigned off, int i) const {
    int r;
    asm("ld.shared.b32 %0, [%1];" : "=r"(r) : "r"(base + 4u * (off + (unsigned)i)));
    return r;
  }
};
template <>
struct Tab<false> {
  const int* p;
  unsigned base;
  __device__ __forceinline__ int4 ld4(unsigned off, int i) const {
    return __ldg(reinterpret_cast<const int4*>(p + off) + i);
  }
  __device__ __forceinline__ int2 ld2(unsigned off, int i) const {
    return __ldg(reinterpret_cast<const int2*>(p + off) + i);
  }
  __device__ __forceinline__ int ld1(unsigned off, int i) const { return __ldg(p + off + i); }
};

// ---- store access by 32-bit shared address -------------------------------------------
// asm volatile keeps these loads in program order with the atomics below
// (no "memory" clobber, so loop-invariant table arithmetic can still hoist).
__device__ __forceinline__ int sld(unsigned a) {
  int v;
  asm volatile("ld.volatile.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
// (lb, ub) of an interval whose lb word is even: one 8-byte load.
__device__ __forceinline__ int2 sld2(unsigned a) {
  int2 v;
  asm volatile("ld.volatile.shared.v2.b32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ int satom_max(unsigned a, int v) {
  int old;
  asm volatile("atom.shared.max.s32 %0, [%1], %2;" : "=r"(old) : "r"(a), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ int satom_min(unsigned a, int v) {
  int old;
  asm volatile("atom.shared.min.s32 %0, [%1], %2;" : "=r"(old) : "r"(a), "r"(v) : "memory");
  return old;
}
// -2^30 <= v < 2^30.  Unsigned arithmetic: a signed `v + 2^30` overflows for
// v near INT_MAX (UB), which lets the compiler drop the upper check.
__device__ __forceinline__ bool small30(int v) { return (unsigned)v + 0x40000000u < 0x80000000u; }
__device__ __forceinline__ long long widen(int v) {
  return v == INT_MAX ? kWide : (v == INT_MIN ? -kWide : (long long)v);
}

// Unit guard `S[a] - S[b] <= T` (a, b packed in x).  Both reads in
// (-2^30, 2^30): exact in 32 bits; otherwise the reference's widened int64
// arithmetic (tv(+1, a) + tv(-1, b), command.cpp:11-27).
__device__ __forceinline__ bool unit_guard(unsigned sb, int x, int T) {
  const int va = sld(sb + (((unsigned)x & 0xffffu) << 2));
  const int vb = sld(sb + (((unsigned)x >> 16) << 2));
  if (small30(va) & small30(vb)) return va - vb <= T;
  return widen(va) - widen(vb) <= (long long)T;
}

// Unit tell: target word tw <- k +- S[f], joined up (lb) or down (ub).
// |k| < 2^30 is guaranteed by the lowering, so a small read needs no narrow.
__device__ __forceinline__ bool unit_tell(unsigned sb, int k, int w) {
  const unsigned tw = (unsigned)w & 0x7fffu, f = ((unsigned)w >> 15) & 0x7fffu;
  const int vf = sld(sb + (f << 2));
  const bool neg = (w & 0x40000000) != 0;
  int val;
  if (small30(vf)) val = neg ? k - vf : k + vf;
  else val = narrow((long long)k + (neg ? -widen(vf) : widen(vf)));
  const unsigned a = sb + (tw << 2);
  const int cur = sld(a);
  if (w < 0) return val > cur && satom_max(a, val) < val;
  return val < cur && satom_min(a, val) > val;
}

// Shared-memory joins without a return value.
__device__ __forceinline__ void sred_min(unsigned a, int v) {
  asm volatile("red.shared.min.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void sred_max(unsigned a, int v) {
  asm volatile("red.shared.max.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// Dirty masks of filtered kPacked rounds (packed_round_f): bit i of a mask
// in shared memory.
__device__ __forceinline__ void smark(unsigned m, unsigned i) {  // bit i of a shared mask
  asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(m + 4u * (i >> 5)), "r"(1u << (i & 31u)) : "memory");
}
__device__ __forceinline__ unsigned sldu(unsigned a) {
  unsigned v;
  asm volatile("ld.volatile.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sst(unsigned a, int v) {
  asm volatile("st.volatile.shared.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned stest(unsigned m, unsigned i) {
  unsigned v;
  asm volatile("ld.volatile.shared.b32 %0, [%1];" : "=r"(v) : "r"(m + 4u * (i >> 5)));
  return (v >> (i & 31u)) & 1u;
}

// Unit record under L.unit_fast (the value-range analysis bounds every word
// it reads): all four words loaded at once, 32-bit arithmetic, and the tell
// joined without a return value when it beats the target's snapshot (a
// change this round, as in eval_ne_fast).  g2 (unit2 records) is the second
// guard {a | b << 16, T}, or T = INT_MAX for none.
template <bool Marks = false>
__device__ __forceinline__ void eval_unit_fast(unsigned sb, int4 q, int2 g2, unsigned& ch, unsigned ms = 0) {
  const unsigned tw = (unsigned)q.w & 0x7fffu, f = ((unsigned)q.w >> 15) & 0x7fffu;
  const unsigned at = sb + (tw << 2);
  const int va = sld(sb + (((unsigned)q.x & 0xffffu) << 2)), vb = sld(sb + (((unsigned)q.x >> 16) << 2));
  const int vf = sld(sb + (f << 2)), cur = sld(at);
  const int wa = sld(sb + (((unsigned)g2.x & 0xffffu) << 2)), wb = sld(sb + (((unsigned)g2.x >> 16) << 2));
  if (va - vb <= q.y && wa - wb <= g2.y) {
    const int val = (q.w & 0x40000000) ? q.z - vf : q.z + vf;
    if (q.w < 0 ? val > cur : val < cur) {
      if (q.w < 0) sred_max(at, val);
      else sred_min(at, val);
      ch = 1u;
      if constexpr (Marks) smark(ms, tw >> 1);
    }
  }
}

__device__ __forceinline__ bool sjoin_max(unsigned a, int v) {
  const int cur = sld(a);
  return v > cur && satom_max(a, v) < v;
}
__device__ __forceinline__ bool sjoin_min(unsigned a, int v) {
  const int cur = sld(a);
  return v < cur && satom_min(a, v) > v;
}

// Fused not(and(x + a <= y, y + b <= x)): the four commands of
// propagation.cpp:350-360 over lb/ub of x and y, from one read of the four
// words.  Returns the mask of changed words (bit w of the word index, words
// >= 64 unmasked: callers that track masks only use stores of <= 64 words).
__device__ __forceinline__ unsigned long long eval_ne(unsigned sb, int4 q) {
  const unsigned wx = (unsigned)q.x >> 2, wy = (unsigned)q.w >> 2;
  const unsigned ax = sb + (unsigned)q.x, ay = sb + (unsigned)q.w;
  const int lx = sld(ax), ux = sld(ax + 4), ly = sld(ay), uy = sld(ay + 4);
  const int a = q.y + 1, b = q.z + 1;
  unsigned long long m = 0;
  auto bit = [](unsigned w) { return 1ull << (w & 63u); };  // any bit flags a change past 64 words
  if (small30(lx) & small30(ux) & small30(ly) & small30(uy)) {
    // Branch-free up to the joins.  The snapshot doubles as the pre-join
    // check: a bound only moves toward top, so a value that does not beat
    // the snapshot cannot beat the current word either.
    const bool g1 = ux - ly <= -a;  // x + a <= y entailed: enforce not(y + b <= x), i.e. x + 1 - b <= y
    const bool g2 = uy - lx <= -b;  // y + b <= x entailed: enforce y + 1 - a <= x
    const int v1 = uy + b - 1, v2 = lx + 1 - b, v3 = ux + a - 1, v4 = ly + 1 - a;
    const bool c1 = g1 & (v1 < ux), c2 = g1 & (v2 > ly), c3 = g2 & (v3 < uy), c4 = g2 & (v4 > lx);
    if (c1 | c2 | c3 | c4) {
      if (c1 && satom_min(ax + 4, v1) > v1) m |= bit(wx + 1);
      if (c2 && satom_max(ay, v2) < v2) m |= bit(wy);
      if (c3 && satom_min(ay + 4, v3) > v3) m |= bit(wy + 1);
      if (c4 && satom_max(ax, v4) < v4) m |= bit(wx);
    }
  } else {  // widened int64 arithmetic of command.cpp:11-27
    if (widen(ux) - widen(ly) <= -(long long)a) {
      if (sjoin_min(ax + 4, narrow((long long)(b - 1) + widen(uy)))) m |= bit(wx + 1);
      if (sjoin_max(ay, narrow((long long)(1 - b) + widen(lx)))) m |= bit(wy);
    }
    if (widen(uy) - widen(lx) <= -(long long)b) {
      if (sjoin_min(ay + 4, narrow((long long)(a - 1) + widen(ux)))) m |= bit(wy + 1);
      if (sjoin_max(ax, narrow((long long)(1 - a) + widen(ly)))) m |= bit(wx);
    }
  }
  return m;
}

// eval_ne when the host's value-range analysis (fast_paths, lower.cpp) has
// proved every value read stays inside (-2^30, 2^30): the 32-bit path is then
// exact with no range checks, and (lb, ub) pairs load as one 8-byte word.
//
// With A = a - 1, B = b - 1 (the table's form): x + a <= y is entailed iff
// ub x + A < lb y, i.e. v3 < lb y; y + b <= x iff v1 < lb x.  The joins need
// no return value: a candidate that beats the round's snapshot proves the
// word changed during this round (it was worse when read and is no worse than
// the candidate after the join), and every change comes from such a join, so
// "some candidate beat its snapshot" flags exactly the rounds that changed a
// word — the flag the fixed-point loop needs.
// Joins without a return value.  When any of a record's four candidates
// beats its snapshot, all four are issued, the others as the join identity
// (min with INT_MAX, max with INT_MIN): one branch region per record
// instead of one per join.
// Sets ch when a candidate beat its snapshot (inside the join branch, so
// the flag costs nothing on the common no-change path).
__device__ __forceinline__ void eval_ne_fast(unsigned sb, int4 q, unsigned& ch) {
  const unsigned ax = sb + (unsigned)q.x, ay = sb + (unsigned)q.w;
  const int2 X = sld2(ax), Y = sld2(ay);
  const int A = q.y, B = q.z;
  const int v1 = Y.y + B, v2 = X.x - B, v3 = X.y + A, v4 = Y.x - A;
  const bool g1 = v3 < Y.x, g2 = v1 < X.x;
  const bool c1 = g1 & (v1 < X.y), c2 = g1 & (v2 > Y.x), c3 = g2 & (v3 < Y.y), c4 = g2 & (v4 > X.x);
  if (c1 | c2 | c3 | c4) {
    sred_min(ax + 4, c1 ? v1 : INT_MAX);
    sred_max(ay, c2 ? v2 : INT_MIN);
    sred_min(ay + 4, c3 ? v3 : INT_MAX);
    sred_max(ax, c4 ? v4 : INT_MIN);
    ch = 1u;
  }
}

__device__ __forceinline__ int4 lds128(unsigned a) {
  int4 r;
  asm("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a));
  return r;
}

// One eventless round over the NE records.  With the table in shared memory
// the loop walks record addresses directly (one add and one compare per
// record).
template <class G, bool TS>
__device__ __forceinline__ bool ne_round(const G& g, unsigned sb, const Tab<TS>& tab, const DeviceLayout& L) {
  const int n = (int)L.n_ne;
  const unsigned off = L.ne;
  unsigned ch = 0;
  if (L.ne_fast) {
    if constexpr (TS) {
      const unsigned step = 16u * (unsigned)g.size();
      const unsigned end = tab.base + 4u * off + 16u * (unsigned)n;
      unsigned a = tab.base + 4u * off + 16u * (unsigned)g.rank();
      for (; a + step < end; a += 2 * step) {  // two records per trip: loads of both issued first
        const int4 q0 = lds128(a), q1 = lds128(a + step);
        eval_ne_fast(sb, q0, ch);
        eval_ne_fast(sb, q1, ch);
      }
      if (a < end) eval_ne_fast(sb, lds128(a), ch);
    } else {
      for (int i = g.rank(); i < n; i += g.size()) eval_ne_fast(sb, tab.ld4(off, i), ch);
    }
  } else {
    for (int i = g.rank(); i < n; i += g.size()) ch |= eval_ne(sb, tab.ld4(off, i)) != 0ull;
  }
  return ch != 0;
}

// Fused reification b <-> (x + p <= y and y + q <= x): the 11 commands of
// compile_reified (propagation.cpp:415-431) from one read of the 6 words.
// q = {lbx | lby << 16, lbb, p, q}.  Returns true iff a word changed.
// Fast: the host's value-range analysis (fast_paths) proved every x/y value
// read stays inside (-2^30, 2^30), so the 32-bit branch is taken unchecked.
template <bool Fast>
__device__ __forceinline__ void reif_core(int lx, int ux, int ly, int uy, int lb, int ub, int p, int q, int& nlb,
                                          int& nub, int& nux, int& nly, int& nuy, int& nlx) {
  const bool bt = lb > 0, bf = ub <= 0;  // [lb b > 0], [ub b <= 0]
  nlb = INT_MIN, nub = INT_MAX, nux = INT_MAX, nly = INT_MIN, nuy = INT_MAX, nlx = INT_MIN;
  if (Fast || (small30(lx) & small30(ux) & small30(ly) & small30(uy))) {
    const bool eA = ux - ly <= -p, eB = uy - lx <= -q;  // entailment of x + p <= y, y + q <= x
    const bool nA = lx - uy > -p, nB = ly - ux > -q;    // entailment of their negations
    if (eA & eB) nlb = nub = 1;
    if (nA | nB) {
      nlb = max(nlb, 0);
      nub = min(nub, 0);
    }
    if (bt) {  // b = 1 activates x + p <= y and y + q <= x
      nux = uy - p;
      nly = lx + p;
      nuy = ux - q;
      nlx = ly + q;
    }
    if (bf & eA) {  // b = 0 and x + p <= y entailed: y + q <= x must fail, x + 1 - q <= y
      nux = min(nux, uy - 1 + q);
      nly = max(nly, lx + 1 - q);
    }
    if (bf & eB) {  // symmetric: y + 1 - p <= x
      nuy = min(nuy, ux - 1 + p);
      nlx = max(nlx, ly + 1 - p);
    }
  } else {  // widened int64 arithmetic of command.cpp:11-27
    const long long wlx = widen(lx), wux = widen(ux), wly = widen(ly), wuy = widen(uy);
    const bool eA = wux - wly <= -(long long)p, eB = wuy - wlx <= -(long long)q;
    const bool nA = wlx - wuy > -(long long)p, nB = wly - wux > -(long long)q;
    if (eA & eB) nlb = nub = 1;
    if (nA | nB) {
      nlb = max(nlb, 0);
      nub = min(nub, 0);
    }
    if (bt) {
      nux = narrow(wuy - p);
      nly = narrow(wlx + p);
      nuy = narrow(wux - q);
      nlx = narrow(wly + q);
    }
    if (bf & eA) {
      nux = min(nux, narrow(wuy - 1 + q));
      nly = max(nly, narrow(wlx + 1 - q));
    }
    if (bf & eB) {
      nuy = min(nuy, narrow(wux - 1 + p));
      nlx = max(nlx, narrow(wly + 1 - p));
    }
  }
}

template <bool Fast>
__device__ __forceinline__ bool eval_reif(unsigned sb, int4 r) {
  const unsigned ax = sb + (((unsigned)r.x & 0xffffu) << 2), ay = sb + (((unsigned)r.x >> 16) << 2);
  const unsigned ab = sb + ((unsigned)r.y << 2);
  const int lx = sld(ax), ux = sld(ax + 4), ly = sld(ay), uy = sld(ay + 4), lb = sld(ab), ub = sld(ab + 4);
  int nlb, nub, nux, nly, nuy, nlx;
  reif_core<Fast>(lx, ux, ly, uy, lb, ub, r.z, r.w, nlb, nub, nux, nly, nuy, nlx);
  // Joins; the snapshot is the pre-check (bounds only move toward top).  As in
  // eval_ne_fast, a candidate that beats its snapshot proves a change this
  // round, so the joins need no return value: all six are issued under one
  // branch, the non-improving ones as the join identity.
  const bool c1 = nlb > lb, c2 = nub < ub, c3 = nux < ux, c4 = nly > ly, c5 = nuy < uy, c6 = nlx > lx;
  if (c1 | c2 | c3 | c4 | c5 | c6) {
    sred_max(ab, c1 ? nlb : INT_MIN);
    sred_min(ab + 4, c2 ? nub : INT_MAX);
    sred_min(ax + 4, c3 ? nux : INT_MAX);
    sred_max(ay, c4 ? nly : INT_MIN);
    sred_min(ay + 4, c5 ? nuy : INT_MAX);
    sred_max(ax, c6 ? nlx : INT_MIN);
    return true;
  }
  return false;
}

__device__ __forceinline__ void sred_or(unsigned a, unsigned v) {
  asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// eval_reif with b a bit-plane cell (L.packed, lower_packed): r.y is b's bit;
// sp is the shared address of plane pair 0.  lb b = LB bit, ub b = 1 - UB bit;
// the joins b <- 1 / b <- 0 set the LB / UB bit (red.or), the only moves a
// 0/1 cell has (nlb > lb only for nlb = 1, lb = 0; nub < ub only for 0 < 1).
// Even: x's and y's lb words are even (kPacked: every interval sits at words
// [0, 2 n_iv)), so each (lb, ub) pair is one 8-byte load.
// Marks: filtered kPacked rounds — a join that beats its snapshot marks its
// start (ms, bit = start index = lb word / 2) or its plane word (mp, bit =
// cell / 32) in the next round's dirty masks.
template <bool Fast, bool Even = false, bool Marks = false>
__device__ __forceinline__ bool eval_reif_bits(unsigned sb, unsigned sp, int4 r, unsigned ms = 0, unsigned mp = 0) {
  const unsigned ax = sb + (((unsigned)r.x & 0xffffu) << 2), ay = sb + (((unsigned)r.x >> 16) << 2);
  const unsigned bit = (unsigned)r.y, ap = sp + ((bit >> 5) << 3), mk = 1u << (bit & 31u);
  int lx, ux, ly, uy;
  if constexpr (Even) {
    const int2 X = sld2(ax), Y = sld2(ay);
    lx = X.x, ux = X.y, ly = Y.x, uy = Y.y;
  } else {
    lx = sld(ax), ux = sld(ax + 4), ly = sld(ay), uy = sld(ay + 4);
  }
  const int2 P = sld2(ap);
  const int lb = ((unsigned)P.x & mk) ? 1 : 0, ub = ((unsigned)P.y & mk) ? 0 : 1;
  int nlb, nub, nux, nly, nuy, nlx;
  reif_core<Fast>(lx, ux, ly, uy, lb, ub, r.z, r.w, nlb, nub, nux, nly, nuy, nlx);
  const bool c1 = nlb > lb, c2 = nub < ub, c3 = nux < ux, c4 = nly > ly, c5 = nuy < uy, c6 = nlx > lx;
  if (c1 | c2 | c3 | c4 | c5 | c6) {
    if (c1) sred_or(ap, mk);
    if (c2) sred_or(ap + 4, mk);
    sred_min(ax + 4, c3 ? nux : INT_MAX);
    sred_max(ay, c4 ? nly : INT_MIN);
    sred_min(ay + 4, c5 ? nuy : INT_MAX);
    sred_max(ax, c6 ? nlx : INT_MIN);
    if constexpr (Marks) {
      if (c1 | c2) smark(mp, bit >> 5);
      if (c3 | c6) smark(ms, ((unsigned)r.x & 0xffffu) >> 1);
      if (c4 | c5) smark(ms, ((unsigned)r.x >> 16) >> 1);
    }
    return true;
  }
  return false;
}

// ---- propagators -----------------------------------------------------------------

// LinExpr::eval over a flat [k, n, (coef, word)*n] expression (command.cpp:21-27).
__device__ __forceinline__ int lin_eval(const int* __restrict__ e, volatile int* S) {
  long long acc = e[0];
  const int n = e[1];
  for (int t = 0; t < n; ++t) acc += tv(e[2 + 2 * t], S[e[3 + 2 * t]]);
  return narrow(acc);
}

// Interpreted fallback: GuardedCommand::apply (command.cpp:93-113) on the flat stream.
__device__ bool eval_generic(volatile int* S, const int* __restrict__ c) {
  const int ng = c[0], kind = c[2], tw = c[3], mask = c[4];
  const int* p = c + 5;
  for (int g = 0; g < ng; ++g) {
    const int rel = p[0], rhs = p[1];
    const int v = lin_eval(p + 2, S);
    if (rel == PCCP_LEQ ? !(v <= rhs) : !(v > rhs)) return false;
    p += 4 + 2 * p[3];
  }
  const int *sc = nullptr, *lb = nullptr, *ub = nullptr;
  if (mask & PCCP_FN_SCALAR) { sc = p; p += 2 + 2 * p[1]; }
  if (mask & PCCP_FN_LB) { lb = p; p += 2 + 2 * p[1]; }
  if (mask & PCCP_FN_UB) { ub = p; }
  bool ch = false;
  if (kind == PCCP_INTERVAL) {
    if (lb) ch |= join_max(S, tw, lin_eval(lb, S));
    if (ub) ch |= join_min(S, tw + 1, lin_eval(ub, S));
  } else {
    const int v = lin_eval(sc, S);
    ch |= (kind == PCCP_ZINC || kind == PCCP_BINC) ? join_max(S, tw, v) : join_min(S, tw, v);
  }
  return ch;
}

// Small command i: up to two normalised guards `tv + tv <= T`, then the lb
// and/or ub tell, each `narrow(k + tv)`.
__device__ __forceinline__ bool eval_small(volatile int* S, const int* __restrict__ T, const DeviceLayout& L,
                                           int i) {
  const int a0 = T[L.small_g[0] + i], a1 = T[L.small_g[1] + i];
  long long s = 0;
  if (a0) s += tv(tcoef(a0), S[tword(a0)]);
  if (a1) s += tv(tcoef(a1), S[tword(a1)]);
  if (s > (long long)T[L.small_T[0] + i]) return false;
  const int T1 = T[L.small_T[1] + i];
  const int a2 = T[L.small_g[2] + i], a3 = T[L.small_g[3] + i];
  if (a2 | a3) {
    s = 0;
    if (a2) s += tv(tcoef(a2), S[tword(a2)]);
    if (a3) s += tv(tcoef(a3), S[tword(a3)]);
    if (s > (long long)T1) return false;
  } else if (T1 < 0) {
    return false;  // 0 <= T1 fails
  }
  const int tw = T[L.small_tw + i];
  bool ch = false;
  const int lbk = T[L.small_lbk + i], lbt = T[L.small_lbt + i];
  if (lbt) ch |= join_max(S, tw, narrow((long long)lbk + tv(tcoef(lbt), S[tword(lbt)])));
  else if (lbk != INT_MIN) ch |= join_max(S, tw, lbk);
  const int ubk = T[L.small_ubk + i], ubt = T[L.small_ubt + i];
  if (ubt) ch |= join_min(S, tw + 1, narrow((long long)ubk + tv(tcoef(ubt), S[tword(ubt)])));
  else if (ubk != INT_MAX) ch |= join_min(S, tw + 1, ubk);
  return ch;
}

// Fused sum rows (H2).  A sub-warp of L.row_lanes lanes owns a row: it reads
// every lb once, reduces S = sum tv(coef, lb), joins lsum <- narrow(S) (and
// +inf when S > c, the overload rule), then evaluates each zeroing guard
// `coef + lsum - coef*lb(x) > c` with lsum taken from the same reduction.
// The second read of lb(x) can only be newer than the one summed, which
// makes the guard weaker, never unsound; at the quiet round both reads agree.
// Lane mapping: consecutive rows (RCPSP: consecutive tasks j of one resource,
// whose rows share their term list) go to consecutive sub-warps, so one load
// instruction touches b_{i,j} for a few i and many consecutive j — stride-2
// words, ~2-way bank conflicts — instead of one column b_{.,j} (n words
// apart: a single bank when n = 32).
//
// L.rows_fast (fast_paths on the host): every term reads a word whose values
// the value-range analysis bounds, so that sums and guards stay inside
// (-2^30, 2^30): the same rows in plain 32-bit arithmetic, no sentinel tests.
// An overloaded row (cell = +inf) makes every zeroing guard hold, as tv(1,
// +inf) does in the widened form.
//
// Latency: a lane's terms (at most kRowTerms, lower.cpp sizes row_lanes so)
// are loaded in two batches — every table entry, then every store word —
// instead of a dependent load chain per term, and the zeroing guards reuse
// the values summed.  That is sound (the summed values are lower bounds of
// the current ones, so a guard that holds on them holds now) and it is the
// fixed point's: at the quiet round every read is of the final store.
//
// Pair (L.row_even: every term's lb word is even): each term is read as one
// 8-byte (lb, ub) load, so the zeroing join b <- (0, 0) needs no second read:
// it is due only when the snapshot has lb < 0 or ub > 0 (bounds only
// tighten, so a snapshot already at 0 stays there), and a due join proves a
// change this round, issued return-free like eval_ne_fast's.
constexpr int kRowTerms = 8;
template <class G, bool TS, bool Pair, int T = kRowTerms>
__device__ bool eval_rows_fast(const G& g, unsigned sb, const Tab<TS>& tab, const DeviceLayout& L, bool& fl) {
  const int R = (int)L.row_lanes, lg = (int)L.row_lg;  // R = 2^lg: shifts, not divisions (CSP: 10% of instructions)
  const int sub = g.rank() & (R - 1);
  const int per_pass = g.size() >> lg;
  const int my = g.rank() >> lg;
  const int n_rows = (int)L.n_rows;
  const unsigned off_meta = L.row_meta, off_terms = L.row_terms;
  unsigned ch = 0;
  for (int base = 0; base < n_rows; base += per_pass) {
    const int row = base + my;
    const bool act = row < n_rows;
    int s = 0;
    int x[T], v[T], u[T];
    const int4 meta = act ? tab.ld4(off_meta, row) : make_int4(0, 0, INT_MAX, 0);  // {beg, end, c, lsum}
    const int j0 = meta.x + sub, end = meta.y, c = meta.z;
    const unsigned alsum = sb + ((unsigned)meta.w << 2);
    const int n_my = end > j0 ? (end - j0 + R - 1) >> lg : 0;  // this lane's terms (<= T)
#pragma unroll
    for (int t = 0; t < T; ++t) x[t] = t < n_my ? tab.ld1(off_terms, j0 + t * R) : 0;
    const int lsum_now = act && sub == 0 ? sld(alsum) : INT_MAX;  // snapshot for the lsum join
#pragma unroll
    for (int t = 0; t < T; ++t) {
      if constexpr (Pair) {
        const int2 p = t < n_my ? sld2(sb + ((unsigned)tword(x[t]) << 2)) : make_int2(0, 0);
        v[t] = p.x;
        u[t] = p.y;
      } else {
        v[t] = t < n_my ? sld(sb + ((unsigned)tword(x[t]) << 2)) : 0;
      }
    }
    // m: the largest coef - coef * lb of this lane's terms, so that no term's
    // zeroing guard coef + s - coef * lb > c holds unless m + s > c: lanes
    // (and, at run time, whole warps) skip the guard loop on quiet rows.
    int m = 0;
#pragma unroll
    for (int t = 0; t < T; ++t) {
      s += tcoef(x[t]) * v[t];
      const int a = tcoef(x[t]) - tcoef(x[t]) * v[t];
      m = t == 0 || a > m ? a : m;
    }
    for (int o = R >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o, R);
    if (act) {
      const bool over = s > c;
      const int cell = over ? INT_MAX : s;  // [lsum > c] => lsum <- +inf
      if (sub == 0 && cell > lsum_now) {     // beats the snapshot: a change this round (eval_ne_fast)
        sred_max(alsum, cell);
        ch = 1u;
      }
      if (sub == 0 && (over || lsum_now == INT_MAX)) fl = true;  // the cell is (or becomes) top: failed
      if (c != INT_MAX && (over || (n_my > 0 && m + s > c))) {
#pragma unroll
        for (int t = 0; t < T; ++t) {
          const int coef = tcoef(x[t]);
          if (t < n_my && (over || coef + s - coef * v[t] > c)) {
            const unsigned a = sb + ((unsigned)tword(x[t]) << 2);
            if constexpr (Pair) {
              if (v[t] < 0) {
                sred_max(a, 0);
                ch = 1u;
              }
              if (u[t] > 0) {
                sred_min(a + 4, 0);
                ch = 1u;
              }
            } else {
              ch |= sjoin_max(a, 0);
              ch |= sjoin_min(a + 4, 0);
            }
          }
        }
      }
    }
  }
  return ch != 0;
}

// fl: set when a row's lsum cell is (or becomes) top (the overload rule), the
// failure the scalar scan would find (skipped when every scalar is a row's cell).
template <class G, bool TS>
__device__ bool eval_rows(const G& g, unsigned sb, const Tab<TS>& tab, const DeviceLayout& L, bool& fl) {
  if (L.rows_fast) {
    if (L.row_even) return eval_rows_fast<G, TS, true>(g, sb, tab, L, fl);
    // short rows (random CSP: <= 5 terms per lane): 5 unrolled term slots, not 8
    if (L.row_tl <= 5) return eval_rows_fast<G, TS, false, 5>(g, sb, tab, L, fl);
    return eval_rows_fast<G, TS, false>(g, sb, tab, L, fl);
  }
  const int R = (int)L.row_lanes, lg = (int)L.row_lg;
  const int sub = g.rank() & (R - 1);
  const int per_pass = g.size() >> lg;
  const int my = g.rank() >> lg;
  bool ch = false;
  for (int base = 0; base < (int)L.n_rows; base += per_pass) {
    const int row = base + my;
    const bool act = row < (int)L.n_rows;
    long long s = 0;
    int beg = 0, end = 0;
    if (act) {
      beg = tab.ld1(L.row_off, row);
      end = tab.ld1(L.row_off, row + 1);
      for (int j = beg + sub; j < end; j += R) {
        const int x = tab.ld1(L.row_terms, j);
        s += tv(tcoef(x), sld(sb + ((unsigned)tword(x) << 2)));
      }
    }
    for (int o = R >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o, R);
    if (act) {
      const int c = tab.ld1(L.row_c, row);
      const int lsum = narrow(s);
      const int cell = lsum > c ? INT_MAX : lsum;  // [lsum > c] => lsum <- +inf
      if (sub == 0) {
        const unsigned al = sb + ((unsigned)tab.ld1(L.row_lsum, row) << 2);
        ch |= sjoin_max(al, cell);
        if (cell == INT_MAX || sld(al) == INT_MAX) fl = true;
      }
      if (c != INT_MAX) {
        const long long wl = tv(1, cell);
        for (int j = beg + sub; j < end; j += R) {
          const int x = tab.ld1(L.row_terms, j);
          const int coef = tcoef(x);
          const unsigned a = sb + ((unsigned)tword(x) << 2);
          if ((long long)coef + wl + tv(-coef, sld(a)) > (long long)c) {
            ch |= sjoin_max(a, 0);
            ch |= sjoin_min(a + 4, 0);
          }
        }
      }
    }
  }
  return ch;
}

// Sum rows over bit-plane cells (L.packed): the row of eval_rows_fast with
// each term's lb read as its LB bit (lb in {0, 1}) and the zeroing join
// b <- (0, 0) as setting its UB bit (lb >= 0 already holds).  A term's pair
// (LB, UB) is one 8-byte load; the terms of a row are consecutive bits
// (lower_packed orders them so), so a sub-warp's loads hit a few words.
// Sums are exact in 32 bits: lower_packed bounds sum |coef| by 2^29.
template <class G, bool TS>
__device__ bool eval_brows(const G& g, unsigned sb, const Tab<TS>& tab, const DeviceLayout& L) {
  const int R = (int)L.brow_lanes, lg = (int)L.brow_lg;
  const int sub = g.rank() & (R - 1);
  const int per_pass = g.size() >> lg;
  const int my = g.rank() >> lg;
  const int n_rows = (int)L.n_brows;
  const unsigned sp = sb + 4u * L.plane;
  unsigned ch = 0;
  for (int base = 0; base < n_rows; base += per_pass) {
    const int row = base + my;
    const bool act = row < n_rows;
    const int4 meta = act ? tab.ld4(L.brow_meta, row) : make_int4(0, 0, INT_MAX, 0);  // {beg, end, c, lsum}
    const int b0 = act ? tab.ld1(L.brow_base, row) : 0;
    const int j0 = meta.x + sub, end = meta.y, c = meta.z;
    const unsigned alsum = sb + ((unsigned)meta.w << 2);
    const int n_my = end > j0 ? (end - j0 + R - 1) >> lg : 0;
    int x[kRowTerms];
    unsigned v = 0, z = 0;  // this lane's terms: LB bits, UB bits
#pragma unroll
    for (int t = 0; t < kRowTerms; ++t) x[t] = t < n_my ? tab.ld1(L.bpat, j0 + t * R) : 0;
    const int lsum_now = act && sub == 0 ? sld(alsum) : INT_MAX;
    int s = 0;
#pragma unroll
    for (int t = 0; t < kRowTerms; ++t) {
      if (t < n_my) {
        const unsigned bit = (unsigned)(b0 + tword(x[t]));
        const int2 P = sld2(sp + ((bit >> 5) << 3));
        const unsigned lbb = ((unsigned)P.x >> (bit & 31u)) & 1u, ubb = ((unsigned)P.y >> (bit & 31u)) & 1u;
        v |= lbb << t;
        z |= ubb << t;
        s += tcoef(x[t]) * (int)lbb;
      }
    }
    for (int o = R >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o, R);
    if (act) {
      const bool over = s > c;
      const int cell = over ? INT_MAX : s;  // [lsum > c] => lsum <- +inf
      if (sub == 0 && cell > lsum_now) {
        sred_max(alsum, cell);
        ch = 1u;
      }
      if (c != INT_MAX) {
#pragma unroll
        for (int t = 0; t < kRowTerms; ++t) {
          const int coef = tcoef(x[t]);
          const int vb = (int)((v >> t) & 1u);
          if (t < n_my && !((z >> t) & 1u) && (over || coef + s - coef * vb > c)) {
            const unsigned bit = (unsigned)(b0 + tword(x[t]));
            sred_or(sp + ((bit >> 5) << 3) + 4u, 1u << (bit & 31u));
            ch = 1u;
          }
        }
      }
    }
  }
  return ch != 0;
}

// Bit rows, word-parallel (L.wrows, lower.cpp): lane q of a row's 2^wrow_lg
// lanes takes the 32-bit chunk q of the row's bit window, funnel-shifted out
// of two plane pairs: lb bits & term mask T.  The chunk's sum is
// popc(lb & U0) + 2 popc(lb & U1) + 4 popc(lb & U2) (U_b: the terms whose
// coefficient has bit b).  Zeroing, [coef + s - coef * lb > c] => b <- (0, 0):
// every term when s > c (overload), else the terms with lb = 0 and coef >
// c - s, a bit-sliced comparison of the planes against c - s.  A new UB bit
// (not in the snapshot) is a change; the joins are red.or on the two words.
__device__ __forceinline__ unsigned coef_gt(const int4& P, int thr) {  // terms with coef > thr >= 0
  if (thr >= 8) return 0u;
  unsigned gt = 0u, eq = (unsigned)P.x;
  const unsigned U[3] = {(unsigned)P.y, (unsigned)P.z, (unsigned)P.w};
#pragma unroll
  for (int b = 2; b >= 0; --b) {
    if ((thr >> b) & 1) {
      eq &= U[b];
    } else {
      gt |= eq & U[b];
      eq &= ~U[b];
    }
  }
  return gt;
}

// `rank` may be a rotation of g.rank() by a multiple of 32 (lane groups stay
// aligned for the shuffles).  fl: set when a row is (or becomes) overloaded —
// its lsum cell is (or is joined to) top, the failure the scan would find
// next (kPacked kernels skip the scalar scan: every scalar is such a cell).
// Filt (filtered kPacked rounds): a warp whose rows' windows hold no plane
// word marked in `cp` skips the pass (warp-uniform: the shuffles below need
// every lane); zeroing joins mark the plane words they write in `np`.
template <class G, bool TS, bool Filt = false>
__device__ bool eval_wrows(const G& g, unsigned sb, const Tab<TS>& tab, const DeviceLayout& L, int rank, bool& fl,
                           unsigned cp = 0, unsigned np = 0) {
  const int lg = (int)L.wrow_lg, Q = 1 << lg;
  const int q = rank & (Q - 1);
  const int per_pass = g.size() >> lg;
  const int my = rank >> lg;
  const int n_rows = (int)L.n_brows;
  const unsigned sp = sb + 4u * L.plane;
  unsigned ch = 0;
  for (int base = 0; base < n_rows; base += per_pass) {
    const int row = base + my;
    const bool act = row < n_rows;
    const int4 meta = act ? tab.ld4(L.wrow_meta, row) : make_int4(0, INT_MAX, 0, 0);  // {chunk0, c, lsum, bit0}
    const unsigned bit = (unsigned)meta.w + 32u * (unsigned)q, sh = bit & 31u;
    const unsigned a = sp + ((bit >> 5) << 3);
    if constexpr (Filt) {  // before the chunk's table entry is fetched
      const bool d = act && (stest(cp, bit >> 5) | (sh ? stest(cp, (bit >> 5) + 1u) : 0u));
      if (!__any_sync(kFull, d)) continue;
    }
    const int4 P = act ? tab.ld4(L.wpat, meta.x + q) : make_int4(0, 0, 0, 0);  // {T, U0, U1, U2}
    const unsigned alsum = sb + ((unsigned)meta.z << 2);
    const int lsum_now = act && q == 0 ? sld(alsum) : INT_MAX;
    unsigned lbw = 0u, ubw = 0u;
    if (P.x) {
      const int2 w0 = sld2(a), w1 = sld2(a + 8u);
      lbw = __funnelshift_r((unsigned)w0.x, (unsigned)w1.x, sh) & (unsigned)P.x;
      ubw = __funnelshift_r((unsigned)w0.y, (unsigned)w1.y, sh) & (unsigned)P.x;
    }
    int s = __popc(lbw & (unsigned)P.y) + 2 * __popc(lbw & (unsigned)P.z) + 4 * __popc(lbw & (unsigned)P.w);
    for (int o = Q >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o, Q);
    if (act) {
      const int c = meta.y;
      const bool over = s > c;
      const int cell = over ? INT_MAX : s;  // [lsum > c] => lsum <- +inf
      if (q == 0 && cell > lsum_now) {
        sred_max(alsum, cell);
        ch = 1u;
      }
      if (q == 0 && (over || lsum_now == INT_MAX)) fl = true;
      if (c != INT_MAX && P.x) {
        const unsigned z = (over ? (unsigned)P.x : coef_gt(P, c - s) & ~lbw) & ~ubw;
        if (z) {
          sred_or(a + 4u, z << sh);
          if (sh && (z >> (32u - sh))) sred_or(a + 12u, z >> (32u - sh));
          ch = 1u;
          if constexpr (Filt) {
            if (z << sh) smark(np, bit >> 5);
            if (sh && (z >> (32u - sh))) smark(np, (bit >> 5) + 1u);
          }
        }
      }
    }
  }
  return ch != 0;
}

// Unguarded constant tells, joined once at node entry.
template <class G>
__device__ __forceinline__ void apply_fold(const G& g, volatile int* S, const int* __restrict__ T,
                                           const DeviceLayout& L) {
  for (int i = g.rank(); i < (int)L.n_fold; i += g.size()) {
    const int wf = T[L.fold_w + i];
    const int v = T[L.fold_v + i];
    const int w = wf & 0x7fffffff;
    if (wf < 0) join_max(S, w, v);
    else join_min(S, w, v);
  }
}

// The eventless fixed-point loop (run_sequential / run_parallel,
// engine.cpp:13-133): every round evaluates every command, joins with
// atomics, and scans a strided slice of the store for failure (an empty
// interval or a scalar at top, store.cpp:65-75).  Failure is monotone, so a
// scan of any intermediate state is valid; it runs every round (H8).
// Returns true iff the store failed.
constexpr unsigned long long kAllDirty = ~0ull;

// Filtered rounds for stores of <= 64 words (one bit per word, one register):
// round r evaluates only the records that read a word changed in round r-1
// (or at node entry, `dirty`).  A record whose inputs are unchanged since its
// last evaluation would join the same value again — a no-op — so skipping it
// leaves the fixed point, the failure status and the node set unchanged; the
// loop ends when a round changes nothing, exactly as the eventless loop.
// Failure is checked on the intervals touched since the previous check.
template <bool TS>
__device__ bool propagate_filtered(const WarpGroup& g, volatile int* S, unsigned sb, const Tab<TS>& tab,
                                   const DeviceLayout& L, unsigned long long dirty, int& rounds) {
  const int* __restrict__ T = tab.p;
  const int nw = (int)L.n_words;
  if (nw < 64) dirty &= (1ull << nw) - 1ull;
  int r = 0;
  bool failed = false;
  unsigned long long D = dirty;
  for (;;) {
    unsigned long long mine = 0;
    unsigned long long todo = D;
    while (todo) {
      const int w = __ffsll((long long)todo) - 1;
      todo &= todo - 1ull;
      const int beg = tab.ld1(L.wl_off, w), end = tab.ld1(L.wl_off, w + 1);
      for (int j = beg + g.lane; j < end; j += 32) {
        const int e = tab.ld1(L.wl, j);
        if (e & 0x40000000) {
          mine |= eval_ne(sb, tab.ld4(L.ne, e & 0x3fffffff));
          continue;
        }
        int4 q;
        bool ok;
        if (e >= 0) {
          q = tab.ld4(L.unit1, e);
          ok = unit_guard(sb, q.x, q.y);
        } else {
          const int i = e & 0x7fffffff;
          q = tab.ld4(L.unit2, i);
          ok = unit_guard(sb, q.x, q.y);
          if (ok) {
            const int2 q2 = tab.ld2(L.unit2g, i);
            ok = unit_guard(sb, q2.x, q2.y);
          }
        }
        if (ok && unit_tell(sb, q.z, q.w)) mine |= 1ull << ((unsigned)q.w & 0x7fffu);
      }
    }
    __syncwarp();
    const unsigned lo = __reduce_or_sync(kFull, (unsigned)mine);
    const unsigned hi = __reduce_or_sync(kFull, (unsigned)(mine >> 32));
    const unsigned long long changed = ((unsigned long long)hi << 32) | lo;
    const unsigned long long touched = changed | D;
    bool fl = false;
    for (int i = g.lane; i < (int)L.n_iv; i += 32) {
      const int w = T[L.iv_lb + i];
      if ((touched >> w) & 3ull) fl |= S[w] > S[w + 1];
    }
    for (int i = g.lane; i < (int)L.n_sc; i += 32) fl |= S[T[L.sc_w + i]] == T[L.sc_top + i];
    ++r;
    if (__any_sync(kFull, fl)) {
      failed = true;
      break;
    }
    if (!changed) break;
    D = changed;
  }
  rounds = r;
  return failed;
}

// Build with -DPCCP_DEBUG_TIMELINE (PCCP_NVFLAGS) for the PCCP_DEBUG_DEC timelines.
__device__ unsigned long long* g_dbg_round = nullptr;  // one round's timeline (CTA 0)
__device__ __forceinline__ void dbg_r(int k) {
#ifdef PCCP_DEBUG_TIMELINE
  if (g_dbg_round && blockIdx.x == 0 && threadIdx.x == 0) g_dbg_round[k] = globaltimer();
#endif
}

// One round of every family but NE (propagate below).
template <class G, bool TS>
__device__ __forceinline__ bool eval_other_families(const G& g, volatile int* S, unsigned sb, const Tab<TS>& tab,
                                                    const DeviceLayout& L, bool& fl) {
    const int* __restrict__ T = tab.p;
    bool ch = false;
    if (L.reif8) {  // packed, 8-byte records
      const unsigned sp = sb + 4u * L.plane;
      auto rec = [&](int i) {
        const int2 q = tab.ld2(L.reif, i);
        return make_int4(q.x, q.y & 0x3ffff, (q.y << 7) >> 25, q.y >> 25);
      };
      if (L.reif_fast) {
        for (int i = g.rank(); i < (int)L.n_reif; i += g.size()) ch |= eval_reif_bits<true>(sb, sp, rec(i));
      } else {
        for (int i = g.rank(); i < (int)L.n_reif; i += g.size()) ch |= eval_reif_bits<false>(sb, sp, rec(i));
      }
    } else if (L.packed) {
      const unsigned sp = sb + 4u * L.plane;
      if (L.reif_fast) {
        for (int i = g.rank(); i < (int)L.n_reif; i += g.size()) ch |= eval_reif_bits<true>(sb, sp, tab.ld4(L.reif, i));
      } else {
        for (int i = g.rank(); i < (int)L.n_reif; i += g.size()) ch |= eval_reif_bits<false>(sb, sp, tab.ld4(L.reif, i));
      }
    } else if (L.reif_fast) {
      for (int i = g.rank(); i < (int)L.n_reif; i += g.size()) ch |= eval_reif<true>(sb, tab.ld4(L.reif, i));
    } else {
      for (int i = g.rank(); i < (int)L.n_reif; i += g.size()) ch |= eval_reif<false>(sb, tab.ld4(L.reif, i));
    }
    dbg_r(0);
    // unit records from the last warp down: the rows' last, partial pass
    // falls on the first warps, so the two remainders land on different warps
    const int ru = (g.size() - 32 * (g.rank() >> 5) - 32) + (g.rank() & 31);
    if (L.unit_fast) {
      unsigned uch = 0;
      const int2 none = make_int2(0, INT_MAX);  // S[0] - S[0] <= INT_MAX: no second guard
      for (int i = ru; i < (int)L.n_unit1; i += g.size()) eval_unit_fast(sb, tab.ld4(L.unit1, i), none, uch);
      for (int i = ru; i < (int)L.n_unit2; i += g.size())
        eval_unit_fast(sb, tab.ld4(L.unit2, i), tab.ld2(L.unit2g, i), uch);
      ch |= uch != 0;
    } else {
      for (int i = ru; i < (int)L.n_unit1; i += g.size()) {
        const int4 q = tab.ld4(L.unit1, i);
        if (unit_guard(sb, q.x, q.y)) ch |= unit_tell(sb, q.z, q.w);
      }
      for (int i = ru; i < (int)L.n_unit2; i += g.size()) {
        const int4 q = tab.ld4(L.unit2, i);
        if (unit_guard(sb, q.x, q.y)) {
          const int2 q2 = tab.ld2(L.unit2g, i);
          if (unit_guard(sb, q2.x, q2.y)) ch |= unit_tell(sb, q.z, q.w);
        }
      }
    }
    dbg_r(1);
    for (int i = g.rank(); i < (int)L.n_small; i += g.size()) ch |= eval_small(S, T, L, i);
    dbg_r(2);
    if (L.n_rows) ch |= eval_rows(g, sb, tab, L, fl);
    if (L.n_brows) ch |= L.wrows ? eval_wrows(g, sb, tab, L, g.rank(), fl) : eval_brows(g, sb, tab, L);
    dbg_r(3);
    for (int i = g.rank(); i < (int)L.n_gen; i += g.size())
      ch |= eval_generic(S, T + L.gen_code + T[L.gen_off + i]);
    return ch;
}

// F selects the command families compiled into the loop: kAllFamilies, or
// kNeOnly for models lowered to NE records alone (N-Queens): a smaller
// kernel, fewer registers, more resident groups (engine.cu dispatch); or
// kPacked for packed models made of 8-byte bit reifications, unit records and
// word-parallel bit rows only, whose scalars are all row sums (RCPSP).
constexpr int kAllFamilies = 0, kNeOnly = 1, kPacked = 2, kPackedF = 3;  // kPackedF: kPacked, filtered rounds

// One round of a kPacked model.  The reifications go from rank 0 up; unit
// records, rows and the scans from the last warp down (a rotation by whole
// warps), so the warps carrying one reification more than the others are
// not the ones carrying the rows.  Failure: the start intervals (the words
// [0, 2 n_iv)), the bit planes, and overloaded rows (eval_wrows).
//
// Filt (L.pfilter, propagate_packed): a record is evaluated only when a start
// or plane word it reads is marked in this round's dirty masks (cs, cp): one
// whose inputs did not change since it was last evaluated would join the
// same values again, a no-op.  Its joins mark the next round's masks (ns, np).
template <class G, bool TS, bool Filt = false>
__device__ __forceinline__ bool packed_round(const G& g, unsigned sb, const Tab<TS>& tab, const DeviceLayout& L,
                                             bool& fl, unsigned cs = 0, unsigned cp = 0, unsigned ns = 0,
                                             unsigned np = 0, bool full = false) {
  const unsigned sp = sb + 4u * L.plane;
  const unsigned n2 = 2u * L.n_iv;  // the start words
  auto rec = [&](int i) {
    const int2 q = tab.ld2(L.reif, i);
    return make_int4(q.x, q.y & 0x3ffff, (q.y << 7) >> 25, q.y >> 25);
  };
  auto clean = [&](const int4& q) {  // reification inputs: x, y starts and b's plane word
    if constexpr (Filt) {
      return !(stest(cs, ((unsigned)q.x & 0xffffu) >> 1) | stest(cs, ((unsigned)q.x >> 16) >> 1) |
               stest(cp, (unsigned)q.y >> 5));
    }
    return false;
  };
  auto wdirty = [&](unsigned w) { return w < n2 ? stest(cs, w >> 1) : 0u; };  // the zero word never changes
  bool ch = false;
  auto reif = [&](int i) {
    const int4 q = rec(i);
    if (L.reif_fast) ch |= eval_reif_bits<true, true, Filt>(sb, sp, q, ns, np);
    else ch |= eval_reif_bits<false, true, Filt>(sb, sp, q, ns, np);
  };
  bool segs = false;
  if constexpr (Filt) {
    // The reifications that read a marked start or plane word, by segment
    // (lower.cpp: the y range, the x list and the plane word's range of each),
    // cut into 32-record chunks dealt to the warps in turn: every warp walks
    // the same marked bits, so the loops stay uniform, and a warp's lanes
    // evaluate records that are all due.  A round whose marks are everything
    // (`full`: a subproblem's first round) walks all records instead.
    segs = L.rfilt && !full;
    if (segs) {
      const int nwarps = g.warps(), wid = g.warp(), lane = g.rank() & 31;
      int turn = 0;  // the warp that takes the next chunk (the same sequence in every warp)
      // Chunk j of a segment goes to warp (turn + j) mod nwarps: a warp visits
      // only its own chunks, then every warp advances turn by the chunk count.
      auto seg = [&](int b, int e, bool indirect) {
        if (e <= b) return;
        const int nc = (e - b + 31) >> 5;
        int j = wid - turn;
        if (j < 0) j += nwarps;
        for (; j < nc; j += nwarps) {
          const int i = b + 32 * j + lane;
          if (i < e) reif(indirect ? tab.ld1(L.r_xrec, i) : i);
        }
        turn += nc;  // a few chunks per segment: subtract rather than divide
        while (turn >= nwarps) turn -= nwarps;
      };
      // The marked bits of a mask of n words, in order: the lanes read 32 words
      // at once and the warp walks the nonzero ones (a ballot), not every word.
      auto walk = [&](unsigned m, unsigned n, auto&& fn) {
        for (unsigned w0 = 0; w0 < n; w0 += 32) {
          const unsigned val = w0 + (unsigned)lane < n ? sldu(m + 4u * (w0 + (unsigned)lane)) : 0u;
          for (unsigned nz = __ballot_sync(kFull, val != 0u); nz; nz &= nz - 1u) {
            const int k = __ffs((int)nz) - 1;
            for (unsigned bits = __shfl_sync(kFull, val, k); bits; bits &= bits - 1u)
              fn(32u * (w0 + (unsigned)k) + (unsigned)(__ffs((int)bits) - 1));
          }
        }
      };
      walk(cs, L.dm_s, [&](unsigned k) {
        if (k >= L.r_ns) return;
        const int2 yr = tab.ld2(L.r_y, (int)k);
        seg(yr.x, yr.y, false);
        seg(tab.ld1(L.r_xoff, (int)k), tab.ld1(L.r_xoff, (int)k + 1), true);
      });
      walk(cp, L.dm_p, [&](unsigned p) {
        if (p >= L.n_pairs) return;
        seg(tab.ld1(L.r_p, (int)p), tab.ld1(L.r_p, (int)p + 1), false);
      });
    }
  }
  if (!segs) {
    for (int i = g.rank(); i < (int)L.n_reif; i += g.size()) {
      if (Filt && !full && clean(rec(i))) continue;
      reif(i);
    }
  }
  const int rr = (g.size() - 32 * (g.rank() >> 5 ) - 32) + (g.rank() & 31);  // warps in reverse order
  auto unit_clean = [&](const int4& q, const int2& g2) {
    if constexpr (Filt) {
      const unsigned x = (unsigned)q.x, f = ((unsigned)q.w >> 15) & 0x7fffu, y = (unsigned)g2.x;
      return !(wdirty(x & 0xffffu) | wdirty(x >> 16) | wdirty(f) | wdirty(y & 0xffffu) | wdirty(y >> 16));
    }
    return false;
  };
  const int2 none = make_int2((int)(L.zero_word | (L.zero_word << 16)), INT_MAX);  // Z - Z <= INT_MAX: no second guard
  if (L.unit_fast) {
    unsigned uch = 0;
    for (int i = rr; i < (int)L.n_unit1; i += g.size()) {
      const int4 q = tab.ld4(L.unit1, i);
      if (!unit_clean(q, none)) eval_unit_fast<Filt>(sb, q, none, uch, ns);
    }
    for (int i = rr; i < (int)L.n_unit2; i += g.size()) {
      const int4 q = tab.ld4(L.unit2, i);
      const int2 q2 = tab.ld2(L.unit2g, i);
      if (!unit_clean(q, q2)) eval_unit_fast<Filt>(sb, q, q2, uch, ns);
    }
    ch |= uch != 0;
  } else {
    for (int i = rr; i < (int)L.n_unit1; i += g.size()) {
      const int4 q = tab.ld4(L.unit1, i);
      if (unit_clean(q, none)) continue;
      if (unit_guard(sb, q.x, q.y) && unit_tell(sb, q.z, q.w)) {
        ch = true;
        if constexpr (Filt) smark(ns, ((unsigned)q.w & 0x7fffu) >> 1);
      }
    }
    for (int i = rr; i < (int)L.n_unit2; i += g.size()) {
      const int4 q = tab.ld4(L.unit2, i);
      const int2 q2 = tab.ld2(L.unit2g, i);
      if (unit_clean(q, q2)) continue;
      if (unit_guard(sb, q.x, q.y) && unit_guard(sb, q2.x, q2.y) && unit_tell(sb, q.z, q.w)) {
        ch = true;
        if constexpr (Filt) smark(ns, ((unsigned)q.w & 0x7fffu) >> 1);
      }
    }
  }
  ch |= eval_wrows<G, TS, Filt>(g, sb, tab, L, rr, fl, cp, np);
  for (int i = rr; i < (int)L.n_iv; i += g.size()) {
    const int2 v = sld2(sb + 8u * (unsigned)i);
    fl |= v.x > v.y;
  }
  for (int i = rr; i < (int)L.n_pairs; i += g.size()) {
    const int2 P = sld2(sp + 8u * (unsigned)i);
    fl |= (P.x & P.y) != 0;
  }
  return ch;
}

// Filtered rounds of a kPacked model (F = kPackedF): three rotating dirty masks
// D[r % 3] (read by round r), D[(r+1) % 3] (marked by round r's joins),
// D[(r+2) % 3] (cleared during round r: round r-1 read it, round r+1 marks
// it).  Each mask is `starts` bits then `plane words` bits (DeviceLayout
// dm_s, dm_p words).  On entry D[0] holds the node's changes — every start
// and plane word when dirty == kAllDirty, else the marks the caller made (the
// decision's start and the objective's); D[1] and D[2] are zero, and all three
// are zero again on return.  A record whose inputs are unmarked is skipped:
// its inputs are unchanged since it was last evaluated, so it would join the
// same values again.  The loop ends, as the eventless one, at the first round
// without a change or with a failure.
template <class G, bool TS>
__device__ bool propagate_packed(const G& g, unsigned sb, const Tab<TS>& tab, const DeviceLayout& L, int& rounds,
                                 unsigned long long dirty, unsigned dm) {
  const int W = (int)(L.dm_s + L.dm_p);
  if (dirty == kAllDirty)
    for (int i = g.rank(); i < W; i += g.size()) sst(dm + 4u * i, -1);
  g.round_begin();
  int r = 0;
  bool failed = false;
  for (;;) {
    const unsigned cur = dm + 4u * (unsigned)(W * (r % 3)), nxt = dm + 4u * (unsigned)(W * ((r + 1) % 3)),
                   clr = dm + 4u * (unsigned)(W * ((r + 2) % 3));
    for (int i = g.rank(); i < W; i += g.size()) sst(clr + 4u * i, 0);
    bool fl = false;
    const bool ch = packed_round<G, TS, true>(g, sb, tab, L, fl, cur, cur + 4u * L.dm_s, nxt, nxt + 4u * L.dm_s,
                                              r == 0 && dirty == kAllDirty);
    bool any_ch, any_fl;
    g.round_end(ch, fl, any_ch, any_fl, r);
    ++r;
    if (any_fl) {
      failed = true;
      break;
    }
    if (!any_ch) break;
  }
  for (int i = g.rank(); i < 3 * W; i += g.size()) sst(dm + 4u * i, 0);
  rounds = r;
  return failed;
}

template <class G, bool TS, int F = kAllFamilies>
__device__ bool propagate(const G& g, volatile int* S, unsigned sb, const Tab<TS>& tab, const DeviceLayout& L,
                          int& rounds, unsigned long long dirty = kAllDirty, unsigned dm = 0) {
  if constexpr (std::is_same<G, WarpGroup>::value && F == kAllFamilies) {
    if (L.filtered) return propagate_filtered(g, S, sb, tab, L, dirty, rounds);
  }
  if constexpr (F == kPackedF) return propagate_packed(g, sb, tab, L, rounds, dirty, dm);
  const int* __restrict__ T = tab.p;
  g.round_begin();
  int r = 0;
  bool failed = false;
  for (;;) {
    bool ch, fl = false;
    if constexpr (F == kPacked) {
      ch = packed_round(g, sb, tab, L, fl);
    } else {
    ch = ne_round(g, sb, tab, L);
    if constexpr (F == kAllFamilies) ch |= eval_other_families(g, S, sb, tab, L, fl);
    // The scan may see an intermediate state: failure is monotone, and a join
    // after it changed a word, so the next round scans again (H8).
    // NE-only kernels keep the plain test (iv_dense): the extra scalar branch
    // costs Q14 3% in code generation.
    if (F == kAllFamilies ? L.iv_prefix : L.iv_dense) {  // intervals by index; scalars (if any) from their list
      const int n_iv = (int)L.n_iv;
      if (n_iv <= g.size()) {  // one interval per rank at most: no loop
        if (g.rank() < n_iv) {
          const int2 v = sld2(sb + 8u * (unsigned)g.rank());
          fl = v.x > v.y;
        }
      } else {
        for (int i = g.rank(); i < n_iv; i += g.size()) {
          const int2 v = sld2(sb + 8u * (unsigned)i);
          fl |= v.x > v.y;
        }
      }
      if (F == kAllFamilies && !L.iv_dense && !L.sc_in_rows)  // (every scalar a row's cell: the rows report it)
        for (int i = g.rank(); i < (int)L.n_sc; i += g.size())
          fl |= sld(sb + 4u * (unsigned)tab.ld1(L.sc_w, i)) == tab.ld1(L.sc_top, i);
      if (F == kAllFamilies && L.packed)  // bit cells: empty = both bits
        for (int i = g.rank(); i < (int)L.n_pairs; i += g.size()) {
          const int2 P = sld2(sb + 4u * (L.plane + 2u * (unsigned)i));
          fl |= (P.x & P.y) != 0;
        }
    } else {
      for (int i = g.rank(); i < (int)L.n_iv; i += g.size()) {
        const unsigned a = sb + 4u * (unsigned)tab.ld1(L.iv_lb, i);
        fl |= sld(a) > sld(a + 4);
      }
      if (!L.sc_in_rows)
        for (int i = g.rank(); i < (int)L.n_sc; i += g.size())
          fl |= sld(sb + 4u * (unsigned)tab.ld1(L.sc_w, i)) == tab.ld1(L.sc_top, i);
      if (F == kAllFamilies && L.packed)
        for (int i = g.rank(); i < (int)L.n_pairs; i += g.size()) {
          const int2 P = sld2(sb + 4u * (L.plane + 2u * (unsigned)i));
          fl |= (P.x & P.y) != 0;
        }
    }
    }  // F != kPacked
    dbg_r(4);
    bool any_ch, any_fl;
    g.round_end(ch, fl, any_ch, any_fl, r);
    dbg_r(5);
    ++r;
    if (any_fl) { failed = true; break; }
    if (!any_ch) break;
  }
  rounds = r;
  return failed;
}


// branch (solver.cpp:19-47): narrowest candidate with lo < hi, first in
// candidate order on ties (key = width << 24 | position), mid = floor((lo+hi)/2).
// Returns 0: none (a solution), 1: decision, -1: unbounded (ModelError).
// L.var_order > 0 selects by smallest lb instead (the primal-dive extension,
// not in the reference); ties go to candidate order (1), the smallest ub
// (2: latest start first, the LST rule of schedule generation), or a
// pseudo-random priority per group and per L.var_seed (3).  The split, mid
// and the unbounded check are the reference's in every order.
__device__ __forceinline__ unsigned mix24(unsigned x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x & 0xffffffu;
}
template <class G>
__device__ int branch(const G& g, volatile int* S, const int* __restrict__ T, const DeviceLayout& L, int& lbw,
                      int& mid, int vo_group = -1) {
  unsigned long long best = ~0ull;
  const unsigned vo = vo_group >= 0 ? (unsigned)vo_group : L.var_order;
  if (vo <= 1) {
    for (int i = g.rank(); i < (int)L.n_cand; i += g.size()) {
      const int w = T[L.cand_lbw + i];
      const int lo = S[w], hi = S[w + 1];
      if (lo < hi) {
        const unsigned long long width = (unsigned long long)((long long)hi - (long long)lo + 1);
        const unsigned long long k = vo ? (unsigned long long)((unsigned)lo ^ 0x80000000u) : width;
        const unsigned long long key = (k << 24) | (unsigned long long)i;
        best = key < best ? key : best;
      }
    }
  } else {
    unsigned long long m = ~0ull;
    for (int i = g.rank(); i < (int)L.n_cand; i += g.size()) {
      const int w = T[L.cand_lbw + i];
      const int lo = S[w], hi = S[w + 1];
      const unsigned long long k = (unsigned)lo ^ 0x80000000u;
      if (lo < hi && k < m) m = k;
    }
    m = g.min_u64(m, 1);
    if (m == ~0ull) return 0;
    const unsigned salt = mix24(L.var_seed * 0x9e3779b9u + g.uid()) << 8;
    for (int i = g.rank(); i < (int)L.n_cand; i += g.size()) {
      const int w = T[L.cand_lbw + i];
      const int lo = S[w], hi = S[w + 1];
      if (lo < hi && ((unsigned)lo ^ 0x80000000u) == m) {
        const unsigned long long k =
            vo == 2 ? (unsigned long long)((unsigned)hi ^ 0x80000000u) : (unsigned long long)mix24(salt ^ (unsigned)i);
        const unsigned long long key = (k << 24) | (unsigned long long)i;
        best = key < best ? key : best;
      }
    }
  }
  best = g.min_u64(best);
  if (best == ~0ull) return 0;
  const int w = T[L.cand_lbw + (int)(best & 0xffffffull)];
  const int lo = S[w], hi = S[w + 1];
  if (lo == INT_MIN || hi == INT_MAX) return -1;
  lbw = w;
  mid = (int)(((long long)lo + (long long)hi) >> 1);
  return 1;
}

// SURVEY 8(c) hash: FNV-style over the 4 little-endian bytes of each word.
__device__ __forceinline__ unsigned long long store_hash(volatile int* S, int n) {
  unsigned long long h = 1469598103934665603ull;
  for (int w = 0; w < n; ++w) {
    const unsigned v = (unsigned)S[w];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      h ^= (v >> (8 * b)) & 0xffu;
      h *= 1099511628211ull;
    }
  }
  return h;
}

// The hash over the reference layout: a packed store decodes its bit cells
// (lower.hpp L.dec) back to the reference's (lb, ub) words on the fly.
__device__ __forceinline__ unsigned long long store_hash_ref(volatile int* S, const int* __restrict__ T,
                                                             const DeviceLayout& L) {
  if (!L.packed) return store_hash(S, (int)L.n_words);
  unsigned long long h = 1469598103934665603ull;
  for (unsigned w = 0; w < L.ref_words; ++w) {
    const int e = T[L.dec + w];
    unsigned v;
    if (e >= 0) {
      v = (unsigned)S[e];
    } else {
      const unsigned code = (unsigned)(-1 - e), b = code >> 1;
      const unsigned set = ((unsigned)S[L.plane + 2u * (b >> 5) + (code & 1u)] >> (b & 31u)) & 1u;
      v = (code & 1u) ? 1u - set : set;  // UB bit: ub = 0; LB bit: lb = 1
    }
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      h ^= (v >> (8 * b)) & 0xffu;
      h *= 1099511628211ull;
    }
  }
  return h;
}

template <class G>
__device__ __forceinline__ void copy_words(const G& g, volatile int* dst, const int* __restrict__ src, int n) {
  for (int i = g.rank(); i < n; i += g.size()) dst[i] = src[i];
}
template <class G>
__device__ __forceinline__ void copy_out(const G& g, int* __restrict__ dst, volatile int* src, int n) {
  for (int i = g.rank(); i < n; i += g.size()) dst[i] = src[i];
}

}  // namespace dev
}  // namespace pccp_b200
