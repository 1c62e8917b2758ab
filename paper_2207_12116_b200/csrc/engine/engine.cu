// engine.cu — host side of the B200 engine: contexts, launch planning, the
// EPS driver and the C ABI of include/pccp_gpu.h.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstddef>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../include/pccp_gpu.h"
#include "search.cuh"

using namespace pccp_b200;

namespace {

thread_local std::string g_err;

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct LimitError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ArgError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define CK(x)                                                                                     \
  do {                                                                                            \
    const cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess) throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_));      \
  } while (0)

template <class F>
int api(F&& f) {
  try {
    return f();
  } catch (const CudaError& e) {
    g_err = e.what();
    return PCCP_ECUDA;
  } catch (const LimitError& e) {
    g_err = e.what();
    return PCCP_ELIMIT;
  } catch (const ArgError& e) {
    g_err = e.what();
    return PCCP_EARG;
  } catch (const std::exception& e) {
    g_err = e.what();
    return PCCP_EMODEL;
  }
}

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  void ensure(size_t k) {
    if (k <= n && p) return;
    release();
    k = std::max<size_t>(k, 1);
    if (cudaMalloc(&p, k * sizeof(T)) != cudaSuccess) {
      cudaGetLastError();
      p = nullptr;
      n = 0;
      throw LimitError("device allocation of " + std::to_string(k * sizeof(T)) + " bytes failed");
    }
    n = k;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

std::uint32_t align4(std::uint32_t x) { return (x + 3u) & ~3u; }

// cfg.mix_order = 0: every kMixOrder-th group of a minimisation branches in
// var_order 2 (measured: the six RCPSP30 parity seeds, DESIGN "Mixed orders").
constexpr int kMixOrder = 48;

double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

struct pccp_gpu_ctx {
  pccp_gpu_cfg cfg{};
  int device = 0;
  int n_sm = 0;
  size_t smem_optin = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[6] = {};
  bool loaded = false;
  bool low_valid = false;            // low/dl hold the lowering of the model whose key is low_key
  std::vector<std::int32_t> low_key;

  Lowered low;  // the plain lowering (reference words): value-range analysis, byte models
  Lowered dl;   // the device layout: bit-plane 0/1 cells when the model has them (lower_packed), else = low
  std::vector<std::uint8_t> slot_kind;
  std::vector<std::uint32_t> slot_word;
  pccp_model view{};  // host copy of the slot tables (commands not kept)
  DBuf<int> blob;

  // launch plan
  bool warp = true;
  int block = 256;
  int gpc = 8;  // groups per CTA
  int ctas = 0;
  size_t smem = 0;
  int store_stride = 4;
  int table_in_smem = 0;
  int ne_only = 0;  // lowered to NE records (and fold tells) only: the kNeOnly kernels
  int packed_only = 0;  // packed reifications, unit records and word-parallel bit rows only: kPacked
  int packed_filter = 0;  // ... with filtered rounds (kPackedF)
  int dec_ctas = 0;  // grid of the persistent decomposition kernel
  long long plan_key = -1;  // last plan's (variant, block, smem) and its occupancies
  int plan_occ = 0, plan_occ_dec = 0;
  std::uint32_t audit_taken = 0;  // node-audit samples of the last search

  DBuf<int> fa, fb, ia, ib, stack, best, io, mailbox, dec, chunk, audit;  // (the wait ring lives behind Globals)
  DBuf<unsigned char> flags, st;
  DBuf<unsigned> rnd;
  dev::Globals* G = nullptr;
  std::vector<void*> opened;
  DBuf<dev::Globals*> d_peers;  // peer contexts' globals (incumbent replicas, done flags, share cells)
  DBuf<int> d_peer_shard;       // each peer's shard index
  int n_peers = 0;
  unsigned epoch = 0;           // sharded searches with work stealing run so far (Globals::qcell tags)
  DBuf<int> qlog;               // record_frontier in stealing searches: positions processed here
  // cfg.record_frontier: FNV hashes of the shared EPS frontier (phase A) and of
  // this shard's share of it, from the last search (pccp_gpu_frontier)
  std::vector<std::uint64_t> frontier_all, frontier_share;
  std::uint64_t launches = 0;

  int groups() const { return ctas * (warp ? gpc : 1); }
  // Per group: three dirty masks of (starts + plane words) bits, in ints (x4 for alignment).
  int dm_words() const {
    const DeviceLayout& L = dl.L;
    return (int)align4(3u * ((L.n_iv + 31) / 32 + (L.n_pairs + 31) / 32));
  }

  // Per-launch layout: branching order, and the value-range analyses of the
  // input stores (lower.cpp fast_paths) that admit the 32-bit
  // paths (PCCP_NO_FAST=1 disables both, for parity tests).
  dev::Model model(int var_order = 0, unsigned var_seed = 0, const std::int32_t* stores = nullptr,
                   std::size_t n_stores = 0, std::size_t stride = 0) const {
    dev::Model M;
    M.L = dl.L;
    M.L.var_order = (std::uint32_t)var_order;
    M.L.var_seed = var_seed;
    bool ne = false, rows = false, reif = false, unit = false;
    if (!std::getenv("PCCP_NO_FAST")) fast_paths(low, stores, n_stores, stride, ne, rows, reif, unit);
    M.L.unit_fast = unit ? 1u : 0u;
    M.L.ne_fast = ne && !std::getenv("PCCP_NO_NE_FAST") ? 1u : 0u;
    M.L.rows_fast = rows ? 1u : 0u;
    M.L.reif_fast = reif ? 1u : 0u;
    M.blob = blob.p;
    M.table_in_smem = table_in_smem;
    M.store_stride = store_stride;
    M.cnt_slots = warp ? gpc : 1;
    // filtered kPacked rounds (kernels.cuh propagate_packed); PCCP_EVENTLESS=1
    // keeps the eventless loop (every record every round)
    M.L.dm_s = (dl.L.n_iv + 31) / 32;
    M.L.dm_p = (dl.L.n_pairs + 31) / 32;
    M.L.pfilter = packed_filter ? 1u : 0u;
    M.dm_words = packed_filter ? dm_words() : 0;
    return M;
  }
};

namespace {

template <class Gp, bool TS, int F>
void set_smem_attrs(size_t smem) {
  CK(cudaFuncSetAttribute(dev::k_propagate<Gp, TS, F>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(dev::k_root<Gp, TS, F>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(dev::k_decompose<Gp, TS, F>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(dev::k_search<Gp, TS, F>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(dev::k_search<Gp, TS, F, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
}

template <class Gp, bool TS, int F>
int occupancy(int block, size_t smem) {
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, dev::k_search<Gp, TS, F>, block, smem));
  return occ;
}

template <class Gp, bool TS, int F>
int occupancy_decompose(int block, size_t smem) {
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, dev::k_decompose<Gp, TS, F>, block, smem));
  return occ;
}

// Calls f.template operator()<Group, TableInSmem, Families>() for the
// context's plan: warp or CTA groups, tables in shared or global memory, and
// the NE-only kernel for models lowered to NE records alone (warp groups).
template <class Fn>
void dispatch(const pccp_gpu_ctx* c, Fn&& f) {
  using dev::kAllFamilies;
  using dev::kNeOnly;
  using dev::kPacked;
  using dev::kPackedF;
  if (c->packed_only && c->packed_filter) {  // CTA groups only (plan)
    if (c->table_in_smem) f.template operator()<dev::CtaGroup, true, kPackedF>();
    else f.template operator()<dev::CtaGroup, false, kPackedF>();
  } else if (c->packed_only) {
    if (c->warp) {
      if (c->table_in_smem) f.template operator()<dev::WarpGroup, true, kPacked>();
      else f.template operator()<dev::WarpGroup, false, kPacked>();
    } else {
      if (c->table_in_smem) f.template operator()<dev::CtaGroup, true, kPacked>();
      else f.template operator()<dev::CtaGroup, false, kPacked>();
    }
  } else if (c->warp && c->ne_only) {
    if (c->table_in_smem) f.template operator()<dev::WarpGroup, true, kNeOnly>();
    else f.template operator()<dev::WarpGroup, false, kNeOnly>();
  } else if (c->warp) {
    if (c->table_in_smem) f.template operator()<dev::WarpGroup, true, kAllFamilies>();
    else f.template operator()<dev::WarpGroup, false, kAllFamilies>();
  } else {
    if (c->table_in_smem) f.template operator()<dev::CtaGroup, true, kAllFamilies>();
    else f.template operator()<dev::CtaGroup, false, kAllFamilies>();
  }
}

void plan(pccp_gpu_ctx* c) {
  const DeviceLayout& L = c->dl.L;
  c->store_stride = (int)align4(L.n_words + 1);  // + the constant-zero word
  c->packed_only = L.packed && L.reif8 && L.wrows && L.sc_in_rows && L.iv_prefix && !L.n_ne && !L.n_small &&
                           !L.n_rows && !L.n_gen && !L.filtered && !std::getenv("PCCP_NO_PACKED_KERNEL")
                       ? 1
                       : 0;
  // Filtered rounds (kPackedF) for packed models whose tables stream from L2
  // (RCPSP120), CTA groups; PCCP_PACKED_FILTER=0/1 forces the choice.
  {
    const size_t hot = (size_t)align4(L.hot_words) * 4;
    bool f = c->packed_only && L.rfilt && hot > 96 * 1024;
    if (const char* pf = std::getenv("PCCP_PACKED_FILTER")) f = c->packed_only && L.rfilt && std::atoi(pf) != 0;
    c->packed_filter = f ? 1 : 0;
  }
  // per group in shared memory: the store, counters, control prefetch, dirty masks
  const size_t per_group = (size_t)c->store_stride * 4 + sizeof(dev::Cnt) + sizeof(dev::Pf) +
                           (c->packed_filter ? (size_t)c->dm_words() * 4 : 0);
  const int gt = c->cfg.group_threads;
  // warp groups for small models: judged on the reference store (a packed
  // RCPSP30 store is 256 words, but its 14k commands want a CTA per node:
  // warp groups explored 12x the nodes and took 13x longer, measured)
  c->warp = gt == 32 || (gt == 0 && (L.packed ? L.ref_words : L.n_words) <= 256);
  if (c->warp) c->packed_filter = 0;  // kPackedF has CTA groups only
  if (c->warp) {
    c->gpc = c->cfg.groups_per_cta > 0 ? std::min(c->cfg.groups_per_cta, 8) : 8;  // MaxThreads<WarpGroup>
    c->block = 32 * c->gpc;
  } else {
    int t = gt;
    if (t <= 0) {
      // ~16 reference commands per thread, up to 1024; but tables streamed
      // from L2 (too large for shared memory) want more resident groups per
      // SM to hide that latency: 256 (RCPSP120: 6.95 M nodes/s at 256 threads,
      // 6.48 at 512, 5.34 at 1024, measured)
      const size_t base1 = dev::kFrameCtl * 4 + per_group;
      const bool l2_tables = base1 + (size_t)align4(L.hot_words) * 4 > 100 * 1024 && !std::getenv("PCCP_TABLE_SMEM");
      t = 128;
      while (t < (l2_tables ? 256 : 1024) && (std::uint32_t)(2 * t) <= L.n_ref_cmds / 16) t *= 2;
    }
    if (t < 64 || t > 1024 || (t & 31)) throw ArgError("group_threads must be 32 or a multiple of 32 in [64, 1024]");
    c->gpc = 1;
    c->block = t;
  }
  const size_t base = dev::kFrameCtl * 4 + (size_t)(c->warp ? c->gpc : 1) * per_group;
  const size_t table = (size_t)align4(L.hot_words) * 4;  // the staged (hot) prefix of the tables
  if (base > c->smem_optin) throw LimitError("store of " + std::to_string(L.n_words) + " words exceeds shared memory");
  c->ne_only = L.n_ne > 0 && !L.n_reif && !L.n_unit1 && !L.n_unit2 && !L.n_small && !L.n_rows && !L.n_gen &&
                       !L.filtered && !std::getenv("PCCP_NO_NE_KERNEL")
                   ? 1
                   : 0;
  const char* env = std::getenv("PCCP_TABLE_SMEM");
  bool in_smem = base + table <= 100 * 1024;
  if (env) in_smem = std::atoi(env) != 0 && base + table <= c->smem_optin;
  c->table_in_smem = in_smem ? 1 : 0;
  c->smem = base + (in_smem ? table : 0);
  int occ = 0;
  int occ_dec = 0;
  // the attributes and occupancies depend only on (kernel variant, block,
  // smem): a reload of a model with the same plan reuses them
  const long long key = ((long long)c->warp << 62) ^ ((long long)c->ne_only << 61) ^ ((long long)c->packed_only << 59) ^ ((long long)c->packed_filter << 58) ^
                        ((long long)c->table_in_smem << 60) ^ ((long long)c->block << 40) ^ (long long)c->smem;
  if (c->plan_key == key) {
    occ = c->plan_occ;
    occ_dec = c->plan_occ_dec;
  } else {
    dispatch(c, [&]<class Gp, bool TS, int F>() {
      set_smem_attrs<Gp, TS, F>(c->smem);
      occ = occupancy<Gp, TS, F>(c->block, c->smem);
      occ_dec = occupancy_decompose<Gp, TS, F>(c->block, c->smem);
    });
    c->plan_key = key;
    c->plan_occ = occ;
    c->plan_occ_dec = occ_dec;
  }
  if (occ_dec < 1) throw LimitError("decomposition kernel does not fit on an SM");
  if ((long long)c->n_sm * std::max(occ, 1) * (c->warp ? c->gpc : 1) > dev::kMaxGroups)
    throw LimitError("more search groups than the wait ring holds");
  if (occ < 1) throw LimitError("kernel does not fit on an SM (smem " + std::to_string(c->smem) + " B)");
  if (c->cfg.ctas_per_sm > 0) occ = std::min(occ, c->cfg.ctas_per_sm);
  c->ctas = c->n_sm * occ;
  c->dec_ctas = c->n_sm * std::min(occ_dec, std::max(1, occ));  // co-resident (cooperative launch)
}

// keep_incumbent: leave the incumbent cell, the best-store lock and
// best_value as they are (the exact phase after a primal phase; peers may be
// pushing into the cell meanwhile, so it is not rewritten from the host).
// EPS subproblems per resident group: warp groups (tiny stores) 8; CTA groups
// 2, since their decomposition levels are latency-bound and donations balance
// the tail (CSP depth 22: 5.1 -> 4.9 ms).
int eps_factor(const pccp_gpu_ctx* c) { return c->cfg.eps_factor > 0 ? c->cfg.eps_factor : (c->warp ? 8 : 2); }

// The cross-rank cells of Globals (incumbent, best_lock, best_value, done):
// INT_MAX / unlocked / no proof.  At open, at load and on request
// (pccp_gpu_reset_shared): with peers linked a search never rewrites them, so
// a push that lands before this rank's search starts is kept.
void reset_shared(pccp_gpu_ctx* c) {
  const int cells[4] = {INT32_MAX, 0, INT32_MAX, 0};
  static_assert(offsetof(dev::Globals, done) - offsetof(dev::Globals, incumbent) == 3 * sizeof(int), "layout");
  CK(cudaMemcpyAsync(reinterpret_cast<char*>(c->G) + offsetof(dev::Globals, incumbent), cells, sizeof(cells),
                     cudaMemcpyHostToDevice, c->stream));
  CK(cudaStreamSynchronize(c->stream));
}

void reset_globals(pccp_gpu_ctx* c, const pccp_limits* lim, bool keep_incumbent = false,
                   unsigned long long stall_ns = 0) {
  if (c->n_peers > 0) keep_incumbent = true;  // peers push into the cells at any time
  dev::Globals h;
  std::memset(&h, 0, sizeof(h));
  h.stall_ns = stall_ns;
  h.incumbent = INT32_MAX;
  h.best_value = INT32_MAX;
  h.node_limit = lim ? lim->node_limit : ~0ull;
  h.timeout_ns = (lim && lim->timeout_s > 0) ? (unsigned long long)(lim->timeout_s * 1e9) : 0ull;
  if (keep_incumbent) {
    constexpr size_t a = offsetof(dev::Globals, incumbent), b = offsetof(dev::Globals, n_impr);
    const char* hp = reinterpret_cast<const char*>(&h);
    char* dp = reinterpret_cast<char*>(c->G);
    CK(cudaMemcpyAsync(dp, hp, a, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(dp + b, hp + b, sizeof(h) - b, cudaMemcpyHostToDevice, c->stream));
  } else {
    CK(cudaMemcpyAsync(c->G, &h, sizeof(h), cudaMemcpyHostToDevice, c->stream));
  }
  dev::k_init_clock<<<1, 1, 0, c->stream>>>(c->G);
  CK(cudaGetLastError());
  ++c->launches;
}

// Depth bound for the DFS stacks: a variable of width w can be bisected at
// most ceil(log2 w) times along one path (solver.cpp:44-46).
// `root` is in the device layout.
int depth_bound(const pccp_gpu_ctx* c, const std::vector<std::int32_t>& root) {
  const DeviceLayout& L = c->dl.L;
  long long d = 2;
  for (std::uint32_t i = 0; i < L.n_cand; ++i) {
    const int w = c->dl.blob[L.cand_lbw + i];
    const long long lo = root[w], hi = root[w + 1];
    if (lo == INT32_MIN || hi == INT32_MAX) {
      d += 33;
    } else if (hi > lo) {
      d += (long long)std::ceil(std::log2((double)(hi - lo + 1))) + 1;
    }
  }
  return (int)std::min<long long>(d, 1 << 20);
}

struct RunOut {
  dev::Globals g{};
  double decompose_ms = 0, kernel_ms = 0, elapsed_ms = 0;
  std::uint64_t subproblems = 0;
  std::uint64_t bfs_rounds = 0, launches = 0, h2d = 0, d2h = 0, levels = 0;
  double device_ms = 0;
  double root_ms = 0, gap_ms = 0;  // root propagation; host gap (buffer sizing) before the decomposition
};

std::uint64_t host_store_hash(const std::int32_t* w, std::uint32_t n) {
  std::uint64_t h = 1469598103934665603ull;
  for (std::uint32_t i = 0; i < n; ++i) {
    const std::uint32_t v = static_cast<std::uint32_t>(w[i]);
    for (int b = 0; b < 4; ++b) {
      h ^= (v >> (8 * b)) & 0xffu;
      h *= 1099511628211ull;
    }
  }
  return h;
}

// cfg.record_frontier: hashes of the frontier in (fa, ia) and of the share
// this GPU processes: positions i = shard (mod shards), or, with work
// stealing, the positions it popped (`taken`, read after the search).
void record_frontier(pccp_gpu_ctx* c, int count, int stride, int shard, int shards,
                     const std::vector<int>* taken = nullptr) {
  const std::uint32_t nw = c->low.L.n_words;  // hashed in the reference layout
  std::vector<std::int32_t> ref(nw);
  std::vector<int> idx((size_t)count);
  CK(cudaMemcpyAsync(idx.data(), c->ia.p, (size_t)count * 4, cudaMemcpyDeviceToHost, c->stream));
  std::vector<std::int32_t> st((size_t)c->fa.n);
  CK(cudaMemcpyAsync(st.data(), c->fa.p, c->fa.n * 4, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  std::vector<std::uint64_t> h((size_t)count);
  for (int i = 0; i < count; ++i) {
    to_reference(c->dl, st.data() + (size_t)idx[(size_t)i] * (size_t)stride, ref.data());
    h[(size_t)i] = host_store_hash(ref.data(), nw);
  }
  c->frontier_all.assign(h.begin(), h.end());
  c->frontier_share.clear();
  if (taken) {
    for (int i : *taken)
      if (i >= 0 && i < count) c->frontier_share.push_back(h[(size_t)i]);
  } else {
    for (int i = shard; i < count; i += shards) c->frontier_share.push_back(h[(size_t)i]);
  }
}

template <class Gp, bool TS, int F>
void run_search(pccp_gpu_ctx* c, int mode, const int32_t* root_words, int depth_cap, const pccp_limits* lim,
                RunOut& out, int var_order = 0, bool keep_incumbent = false, unsigned long long stall_ns = 0,
                unsigned var_seed = 0, bool sharded = true) {
  const double t_start = now_ms();
  const std::uint64_t launches0 = c->launches;
  const DeviceLayout& L = c->dl.L;
  const int nw = (int)L.n_words;  // device store words
  const int stride = c->store_stride;
  // sharded = false: this search covers the whole tree on this GPU (the
  // primal segments of an N-shard solve), counted by it alone
  const int shard_count = sharded ? std::max(1, c->cfg.shard_count) : 1;
  const int shard_index = sharded ? c->cfg.shard_index : 0;
  if (shard_index < 0 || shard_index >= shard_count) throw ArgError("shard_index out of range");
  // Linked shards steal from each other's shares of the shared phase-A
  // frontier (search.cuh steal_pop); unlinked ones keep the static i mod N
  // split and expand their share (phase B below).
  const bool steal = shard_count > 1 && c->n_peers > 0 && !std::getenv("PCCP_NO_STEAL");
  const unsigned epoch = steal ? ++c->epoch : 0u;
  const dev::Model M = c->model(var_order, var_seed, root_words, 1, (size_t)c->low.L.n_words);
  dev::SearchCtl C{};
  C.G = c->G;
  C.blob = c->blob.p;
  C.n_peers = mode == 1 ? c->n_peers : 0;
  C.peers = c->d_peers.p;
  C.mode = mode;
  C.hash = c->cfg.hash;
  C.depth_cap = depth_cap;
  C.count = shard_index == 0 ? 1 : 0;  // the decomposition runs on every GPU, counted once
  // With N shards the root and the shared phase A must be the same on every
  // GPU, whatever incumbent each has seen (peers push at any time): they run
  // without the objective join, so the frontier depends on the model and the
  // root alone and positions i = shard (mod N) partition it.  Phase B and the
  // search re-materialise under the bound (sound: the bound is a solution's).
  C.bound = shard_count > 1 ? 0 : 1;
  c->best.ensure((size_t)std::max(nw, 1));
  C.best_store = c->best.p;
  if (c->cfg.audit_nodes > 0) {
    const size_t k = (size_t)c->cfg.audit_nodes;
    c->audit.ensure(2 * k * (size_t)std::max(nw, 1) + (k + 3) / 4);
    C.audit_pre = c->audit.p;
    C.audit_post = c->audit.p + k * (size_t)std::max(nw, 1);
    C.audit_failed = reinterpret_cast<unsigned char*>(c->audit.p + 2 * k * (size_t)std::max(nw, 1));
    C.audit_n = c->cfg.audit_nodes;
    C.audit_shift = std::clamp(c->cfg.audit_shift, 0, 40);
  }

  // EPS targets (see below), known before anything is allocated
  const int eps = eps_factor(c);
  // CTA groups (stores of hundreds of words and more) skip phase B by default:
  // the root goes to one group and donations spread the tree (a donation per
  // node of every busy group doubles the busy groups per node time), which
  // beats BFS levels of whole-grid barriers (RCPSP30 proofs 3.5-4.5 -> 2.6-3.9
  // ms, CSP depth 22 4.75 -> 4.3 ms).  Warp groups keep eps x groups (Q14:
  // 17.33 ms vs 17.44 ms without).
  long long target_ll = (c->warp || c->cfg.eps_factor > 0) ? (long long)eps * c->groups() : 1;
  if (const char* dt = std::getenv("PCCP_DEC_TARGET")) target_ll = std::max(1, std::atoi(dt));
  const long long target_a_ll = shard_count > 1 ? (long long)c->groups() * shard_count : 0;
  if (std::max(target_ll, target_a_ll) > (1ll << 28)) throw LimitError("EPS target too large");
  const int cap = (int)std::max(target_ll, target_a_ll);
  // the root store is frontier buffer 0 of the decomposition (capacity 2*cap:
  // odd levels write their children there), allocated before the device
  // clock starts (reset_globals)
  c->fa.ensure((size_t)stride * (size_t)std::max(2 * (size_t)cap, (size_t)1));
  c->ia.ensure(1);
  c->flags.ensure(2);
  reset_globals(c, lim, keep_incumbent, stall_ns);
  std::vector<std::int32_t> root((size_t)nw);
  to_device(c->dl, root_words, root.data());
  CK(cudaMemcpyAsync(c->fa.p, root.data(), (size_t)nw * 4, cudaMemcpyHostToDevice, c->stream));
  const int zero = 0;
  CK(cudaMemcpyAsync(c->ia.p, &zero, 4, cudaMemcpyHostToDevice, c->stream));
  out.h2d += sizeof(dev::Globals) + (std::uint64_t)nw * 4 + 4;
  CK(cudaEventRecord(c->ev[0], c->stream));
  dev::k_root<Gp, TS, F><<<1, c->block, c->smem, c->stream>>>(M, C, c->fa.p, c->flags.p);
  CK(cudaGetLastError());
  ++c->launches;
  unsigned char rflag = 0;
  CK(cudaMemcpyAsync(&rflag, c->flags.p, 1, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(root.data(), c->fa.p, (size_t)nw * 4, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaEventRecord(c->ev[3], c->stream));
  CK(cudaStreamSynchronize(c->stream));
  out.d2h += 1 + (std::uint64_t)nw * 4;
  // Device buffers for the decomposition and the search are sized here, while
  // the GPU is idle, and the device clock restarts after them (ev[4]): a first
  // call's allocations are host time, not device time (they are in elapsed_ms).
  const int dmax = [&] {
    const int d = depth_bound(c, root);
    return depth_cap >= 0 ? std::min(d, depth_cap + 2) : d;
  }();
  const int entry = (int)align4((std::uint32_t)nw + 3);
  const int mb_stride = (int)align4((std::uint32_t)nw + 3);
  if (rflag) {
    c->stack.ensure((size_t)c->groups() * (size_t)dmax * (size_t)entry);
    c->mailbox.ensure((size_t)c->groups() * (size_t)mb_stride);
  }

  // EPS decomposition: whole BFS levels until the frontier holds target nodes.
  // Levels are enqueued in batches without host round trips: each level's
  // size lives on the device (dev::DecState) and a level past the target is a
  // no-op; within a phase, level L reads ping-pong buffer L&1 and writes
  // (L+1)&1.  Children of fewer than `target` parents need 2*target slots.
  //
  // With N shards the decomposition has two phases.  Phase A is identical on
  // every GPU (counted on shard 0 only) and stops at `groups * N` nodes; each
  // GPU keeps the positions i = shard (mod N) of that frontier, and phase B
  // expands only those (counted by their owner) to `eps * groups` nodes.  So
  // each GPU expands its own share, not the whole job's frontier, and every
  // tree node is still materialised exactly once across the GPUs.
  int count = rflag ? 1 : 0;
  int level = 0;
  // two flag buffers of 2 cap bytes (k_decompose), 16-byte aligned for the
  // small levels' word loads
  const int fstride = (int)((2 * (size_t)cap + 15) / 16 * 16);
  if (count > 0) {
    c->fb.ensure(2 * (size_t)cap * stride);
    c->ib.ensure(2 * (size_t)cap);
    c->ia.ensure(2 * (size_t)cap);  // may reallocate: index 0 of the root frontier is rewritten
    CK(cudaMemcpyAsync(c->ia.p, &zero, 4, cudaMemcpyHostToDevice, c->stream));
    c->flags.ensure(2 * (size_t)fstride);
    c->dec.ensure(2);
    c->chunk.ensure((size_t)c->dec_ctas + 3);
  }
  CK(cudaEventRecord(c->ev[4], c->stream));
  dev::DecState* d_st = reinterpret_cast<dev::DecState*>(c->dec.p);
  // Expand the frontier in (fa, ia) until it holds `target` nodes, in one
  // cooperative launch of the persistent decomposition kernel; the result is
  // left in (fa, ia).  Returns false after a model error.
  auto expand_until = [&](int target) -> bool {
    if (count <= 0 || count >= target) return true;
    const int grid = c->dec_ctas;
    c->chunk.ensure((size_t)grid + 3);
    const dev::DecState st0{count, level};
    CK(cudaMemcpyAsync(c->dec.p, &st0, sizeof(st0), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemsetAsync(c->chunk.p + grid, 0, 3 * sizeof(int), c->stream));  // grid barrier words, stop snapshot
    int* fb0 = c->fa.p;
    int* fb1 = c->fb.p;
    int* ib0 = c->ia.p;
    int* ib1 = c->ib.p;
    unsigned char* flags = c->flags.p;
    int* chunk_count = c->chunk.p;
    unsigned* bar = reinterpret_cast<unsigned*>(c->chunk.p + grid);
    int tgt = target, strd = stride, fstr = fstride;
    const bool dbg = std::getenv("PCCP_DEBUG_DEC") != nullptr;
    DBuf<unsigned long long> profbuf;
    unsigned long long* prof = nullptr;
    if (dbg) {
      profbuf.ensure(240 + 32);
      CK(cudaMemsetAsync(profbuf.p, 0, (240 + 32) * 8, c->stream));
      prof = profbuf.p;
      unsigned long long* tl = profbuf.p + 240;
      CK(cudaMemcpyToSymbolAsync(dev::g_dbg_tl, &tl, sizeof(tl), 0, cudaMemcpyHostToDevice, c->stream));
      unsigned long long* tr = profbuf.p + 240 + 24;
      CK(cudaMemcpyToSymbolAsync(dev::g_dbg_round, &tr, sizeof(tr), 0, cudaMemcpyHostToDevice, c->stream));
    }
    void* args[] = {(void*)&M, (void*)&C, (void*)&fb0, (void*)&fb1, (void*)&ib0, (void*)&ib1, (void*)&d_st,
                    (void*)&tgt, (void*)&strd, (void*)&flags, (void*)&fstr, (void*)&chunk_count, (void*)&bar,
                    (void*)&prof};
    const int level0 = level;
    CK(cudaLaunchCooperativeKernel((const void*)dev::k_decompose<Gp, TS, F>, dim3(grid), dim3(c->block), args,
                                   c->smem, c->stream));
    ++c->launches;
    dev::DecState st;
    int stop = 0;
    CK(cudaMemcpyAsync(&st, d_st, sizeof(st), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(&stop, &c->G->stop, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    out.d2h += sizeof(st) + 4;
    count = st.count;
    level = st.levels;
    if (dbg) {
      fprintf(stderr, "decompose: level=%d count=%d t=%.3f ms grid=%d\n", level, count, now_ms() - t_start, grid);
      unsigned long long h[240];
      CK(cudaMemcpy(h, prof, sizeof(h), cudaMemcpyDeviceToHost));
      unsigned long long tl[32];
      CK(cudaMemcpy(tl, prof + 240, sizeof(tl), cudaMemcpyDeviceToHost));
      fprintf(stderr, "  last parent of CTA 0: copy %.1f branch %.1f | L: join %.1f prop %.1f (r=%llu) classify %.1f out %.1f"
                      " | R: join %.1f prop %.1f (r=%llu) classify %.1f out %.1f us\n",
              (tl[1] - tl[0]) * 1e-3, (tl[2] - tl[1]) * 1e-3, (tl[3] - tl[2]) * 1e-3, (tl[4] - tl[3]) * 1e-3, tl[20],
              (tl[5] - tl[4]) * 1e-3, (tl[6] - tl[5]) * 1e-3, (tl[8] - tl[6]) * 1e-3, (tl[9] - tl[8]) * 1e-3, tl[21],
              (tl[10] - tl[9]) * 1e-3, (tl[11] - tl[10]) * 1e-3);
      fprintf(stderr, "  last round of CTA 0: reif+ne %.2f unit1 %.2f small %.2f rows %.2f gen+scan %.2f end %.2f us\n",
              0.0, (tl[25] - tl[24]) * 1e-3, (tl[26] - tl[25]) * 1e-3, (tl[27] - tl[26]) * 1e-3,
              (tl[28] - tl[27]) * 1e-3, (tl[29] - tl[28]) * 1e-3);
      unsigned long long* zero = nullptr;
      CK(cudaMemcpyToSymbol(dev::g_dbg_tl, &zero, sizeof(zero)));
      CK(cudaMemcpyToSymbol(dev::g_dbg_round, &zero, sizeof(zero)));
      for (int k = 0; k < 60 && h[4 * k]; ++k)
        fprintf(stderr, "  level %2d: expand %7.1f us  compact %6.1f us  barrier %5.1f us\n", k,
                (h[4 * k + 1] - h[4 * k]) * 1e-3, (h[4 * k + 2] - h[4 * k + 1]) * 1e-3,
                (h[4 * k + 3] - h[4 * k + 2]) * 1e-3);
    }
    if ((level - level0) & 1) {  // the frontier is in buffer (levels of this phase) & 1
      std::swap(c->fa, c->fb);
      std::swap(c->ia, c->ib);
    }
    return stop != 2;
  };
  c->frontier_all.clear();
  c->frontier_share.clear();
  int steal_count = 0;  // stealing: the shared frontier's size (every position is popped once)
  if (shard_count > 1 && steal) {
    if (expand_until((int)target_a_ll) && count > 0) steal_count = count;
    C.count = 1;  // the search below counts what this GPU processes
  } else if (shard_count > 1) {
    if (expand_until((int)target_a_ll) && count > 0) {
      if (c->cfg.record_frontier) record_frontier(c, count, stride, shard_index, shard_count);
      const int mine = count > shard_index ? (count - shard_index + shard_count - 1) / shard_count : 0;
      if (mine > 0) {
        dev::k_shard_filter<<<(mine + 255) / 256, 256, 0, c->stream>>>(c->ia.p, c->ib.p, shard_index, shard_count, mine);
        CK(cudaGetLastError());
        ++c->launches;
        std::swap(c->ia, c->ib);
      }
      count = mine;
      C.count = 1;  // phase B and the search: every node below here is this GPU's alone
      C.bound = 1;  // and is re-materialised under the bound
      expand_until((int)target_ll);
    }
  } else {
    expand_until((int)target_ll);
    if (c->cfg.record_frontier && count > 0) record_frontier(c, count, stride, 0, 1);
  }
  C.bound = 1;
  CK(cudaEventRecord(c->ev[1], c->stream));
  CK(cudaMemcpyAsync(&out.bfs_rounds, &c->G->rounds, 8, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  out.d2h += 8;
  out.subproblems = (std::uint64_t)count;

  bool searched = false;
  if (count > 0) {
    dev::SearchParams P{};
    P.frontier = c->fa.p;
    P.frontier_idx = c->ia.p;
    P.n_frontier = count;
    P.stride = stride;
    P.depth0 = level;
    P.shard_index = 0;  // the frontier is already this GPU's share (phase B)
    P.shard_count = 1;
    P.stack_pool = c->stack.p;
    P.stack_depth = dmax;
    P.entry_stride = entry;
    // dynamic load balancing: per-group mailboxes + the wait ring
    P.balance = std::getenv("PCCP_NO_BALANCE") ? 0 : 2;
    if (const char* dm = std::getenv("PCCP_DONATE_MIN")) P.balance = std::max(1, std::atoi(dm));
    if (const char* dd = std::getenv("PCCP_DONATE_DEEP")) P.donate_deep = std::atoi(dd) != 0 ? 1 : 0;
    // a portfolio of branching orders for minimisation (cfg.mix_order; kMixOrder
    // measured on the RCPSP30 parity seeds, DESIGN "Mixed orders")
    P.mix_order = c->cfg.mix_order > 0 ? c->cfg.mix_order : (c->cfg.mix_order == 0 ? kMixOrder : 0);
    if (const char* mo = std::getenv("PCCP_MIX_ORDER")) P.mix_order = std::max(0, std::atoi(mo));
    P.n_groups = c->groups();
    P.mb_stride = mb_stride;
    CK(cudaMemsetAsync(c->mailbox.p, 0, (size_t)P.n_groups * P.mb_stride * 4, c->stream));
    CK(cudaMemsetAsync(dev::waitq_of(c->G), 0xff, (size_t)P.n_groups * 4, c->stream));
    const int active = P.n_groups;
    CK(cudaMemcpyAsync(&c->G->active, &active, sizeof(int), cudaMemcpyHostToDevice, c->stream));
    P.mailbox = c->mailbox.p;
    P.value_order = c->cfg.value_order >= 0 ? std::min(c->cfg.value_order, 2) : 0;
    if (const char* vo = std::getenv("PCCP_VALUE_ORDER")) P.value_order = std::atoi(vo);
    P.waitq = dev::waitq_of(c->G);
    if (steal) {  // the whole shared frontier; positions come from the share cells
      P.shard_index = shard_index;
      P.shard_count = shard_count;
      P.steal = 1;
      P.epoch = epoch;
      P.own_q = &c->G->qcell;
      P.peers = c->d_peers.p;
      P.peer_shard = c->d_peer_shard.p;
      P.n_peers = c->n_peers;
      if (c->cfg.record_frontier) {
        c->qlog.ensure((size_t)count);
        P.qlog = c->qlog.p;
      }
      // cross-GPU donation of pending branches (search.cuh hand_over_remote)
      P.remote = !c->warp && nw + 3 <= dev::kSlotWords && !std::getenv("PCCP_NO_REMOTE_DONATE") ? 1 : 0;  // CTA groups
    }
    {  // what peers read before they donate: the ring's modulus, whether this search takes donations, its epoch
      const int pub[3] = {P.n_groups, P.remote, (int)P.epoch};
      static_assert(offsetof(dev::Globals, remote) == offsetof(dev::Globals, n_groups_pub) + sizeof(int), "layout");
      static_assert(offsetof(dev::Globals, epoch_pub) == offsetof(dev::Globals, remote) + sizeof(int), "layout");
      CK(cudaMemcpyAsync(&c->G->n_groups_pub, pub, sizeof(pub), cudaMemcpyHostToDevice, c->stream));
    }
    C.count = 1;
    if (C.audit_n > 0) dev::k_search<Gp, TS, F, true><<<c->ctas, c->block, c->smem, c->stream>>>(M, C, P);
    else dev::k_search<Gp, TS, F><<<c->ctas, c->block, c->smem, c->stream>>>(M, C, P);
    CK(cudaGetLastError());
    ++c->launches;
    searched = true;
  }
  CK(cudaEventRecord(c->ev[2], c->stream));
  CK(cudaMemcpyAsync(&out.g, c->G, sizeof(dev::Globals), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  out.d2h += sizeof(dev::Globals);
  if (steal && c->cfg.record_frontier && steal_count > 0) {
    std::vector<int> taken((size_t)std::min<unsigned long long>(out.g.qlog_n, (unsigned long long)steal_count));
    if (!taken.empty())
      CK(cudaMemcpy(taken.data(), c->qlog.p, taken.size() * 4, cudaMemcpyDeviceToHost));
    record_frontier(c, steal_count, stride, shard_index, shard_count, &taken);
  }
  out.launches = c->launches - launches0;
  out.levels = (std::uint64_t)level;
  // device time = root propagation (ev0..ev3) + decomposition and search (ev4..ev2)
  float ms = 0, root_ms = 0;
  CK(cudaEventElapsedTime(&root_ms, c->ev[0], c->ev[3]));
  CK(cudaEventElapsedTime(&ms, c->ev[4], c->ev[2]));
  out.device_ms = root_ms + ms;
  CK(cudaEventElapsedTime(&ms, c->ev[4], c->ev[1]));
  out.decompose_ms = root_ms + ms;
  CK(cudaEventElapsedTime(&ms, c->ev[3], c->ev[4]));
  out.root_ms = root_ms;
  out.gap_ms = ms;
  if (searched) {
    CK(cudaEventElapsedTime(&ms, c->ev[1], c->ev[2]));
    out.kernel_ms = ms;
  }
  out.elapsed_ms = now_ms() - t_start;
  c->audit_taken = c->cfg.audit_nodes > 0
                       ? (std::uint32_t)std::min<unsigned long long>(
                             (out.g.audit_seen + (1ull << std::clamp(c->cfg.audit_shift, 0, 40)) - 1) >>
                                 std::clamp(c->cfg.audit_shift, 0, 40),
                             (unsigned long long)c->cfg.audit_nodes)
                       : 0u;
  if (c->cfg.verbose)
    fprintf(stderr,
            "pccp_gpu[dev %d shard %d/%d]: %s, %d %s groups (%d CTAs x %d threads, smem %zu B, tables in %s), "
            "store %u words%s; root %.3f ms, decompose %.3f ms (%d subproblems, %llu levels), search %.3f ms; "
            "nodes %llu, rounds %llu, donations %llu%s\n",
            c->device, shard_index, shard_count, mode == 1 ? "minimise" : "enumerate", c->groups(),
            c->warp ? "warp" : "CTA", c->ctas, c->block, c->smem, c->table_in_smem ? "smem" : "L2",
            (unsigned)nw, L.packed ? " (bit-plane 0/1 cells)" : "", out.root_ms, out.decompose_ms - out.root_ms, count,
            (unsigned long long)level, out.kernel_ms, out.g.nodes, out.g.rounds, out.g.donations,
            out.g.incomplete ? ", incomplete" : "");
  if (c->cfg.verbose && out.g.incomplete)
    fprintf(stderr, "pccp_gpu[dev %d shard %d/%d]: incomplete causes %d, stop %d, remote in %llu out %llu\n", c->device,
            shard_index, shard_count, out.g.why, out.g.stop, out.g.remote_in, out.g.remote_out);
  if (out.g.stop == 2) {
    if (out.g.error_code == 1) throw std::runtime_error("branch: a candidate variable is unbounded");
    throw LimitError("DFS stack capacity exceeded");
  }
}

void fill_stats(const pccp_gpu_ctx* c, const RunOut& r, pccp_stats& s) {
  std::memset(&s, 0, sizeof(s));
  s.nodes = r.g.nodes;
  s.failures = r.g.failures;
  s.solutions = r.g.solutions;
  s.open_leaves = r.g.open_leaves;
  s.hash_sum = r.g.hash_sum;
  s.rounds = r.g.rounds;
  s.evals = r.g.rounds * (std::uint64_t)c->low.L.n_ref_cmds;
  s.subproblems = r.subproblems;
  s.max_depth = r.g.max_depth;
  s.elapsed_ms = r.elapsed_ms;
  s.kernel_ms = r.kernel_ms;
  s.decompose_ms = r.decompose_ms;
  s.launches = r.launches;
  s.search_evals = (r.g.rounds - r.bfs_rounds) * (std::uint64_t)c->low.L.n_ref_cmds;
  s.h2d_bytes = r.h2d;
  s.d2h_bytes = r.d2h;
  s.device_ms = r.device_ms;
  s.bfs_levels = r.levels;
  s.donations = r.g.donations;
  s.rematerialised = r.g.rematerialised;
  s.stolen = r.g.stolen;
  s.remote_in = r.g.remote_in;
  s.remote_out = r.g.remote_out;
}

// Counters of consecutive searches of one call (primal segments, exact
// phase); the final search's control state (incumbent, stop) wins.
void merge_run(RunOut& acc, const RunOut& r, bool first) {
  if (first) {
    acc = r;
    return;
  }
  dev::Globals g = r.g;
  g.nodes += acc.g.nodes;
  g.failures += acc.g.failures;
  g.solutions += acc.g.solutions;
  g.rounds += acc.g.rounds;
  g.max_depth = std::max(g.max_depth, acc.g.max_depth);
  g.donations += acc.g.donations;
  g.rematerialised += acc.g.rematerialised;
  g.stolen += acc.g.stolen;
  g.remote_in += acc.g.remote_in;
  g.remote_out += acc.g.remote_out;
  acc.g = g;
  acc.bfs_rounds += r.bfs_rounds;
  acc.decompose_ms += r.decompose_ms;
  acc.kernel_ms += r.kernel_ms;
  acc.device_ms += r.device_ms;
  acc.elapsed_ms += r.elapsed_ms;
  acc.launches += r.launches;
  acc.h2d += r.h2d;
  acc.d2h += r.d2h;
  acc.subproblems += r.subproblems;
  acc.levels += r.levels;
}

// The device keeps the last 64 improvements in a ring (record_solution).
// Improvement times are device-clock offsets from the run's start; those after
// the root fixed point exclude the host gap in which the search buffers were sized.
void append_log(const RunOut& r, double offset_ms, std::vector<std::pair<int, double>>& log) {
  const dev::Globals& g = r.g;
  const int n = g.n_impr, first = std::max(0, n - 64);
  for (int k = first; k < n; ++k) {
    double t = (double)g.impr_ns[k & 63] * 1e-6;
    if (t >= r.root_ms + r.gap_ms) t -= r.gap_ms;
    log.emplace_back(g.impr_val[k & 63], offset_ms + t);
  }
}

void check_loaded(const pccp_gpu_ctx* c) {
  if (!c) throw ArgError("null context");
  if (!c->loaded) throw ArgError("no model loaded");
  CK(cudaSetDevice(c->device));
}

}  // namespace

extern "C" {

const char* pccp_gpu_last_error(void) { return g_err.c_str(); }
const char* pccp_gpu_version(void) { return "pccp-b200 0.1 (sm_100a)"; }

int pccp_gpu_device_count(int32_t* out) {
  return api([&] {
    int n = 0;
    const cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    *out = n;
    return n > 0 ? PCCP_OK : (g_err = "no CUDA device", PCCP_ECUDA);
  });
}

int pccp_gpu_open(const pccp_gpu_cfg* cfg, pccp_gpu_ctx** out) {
  return api([&] {
    if (!out) throw ArgError("null output");
    *out = nullptr;
    auto* c = new pccp_gpu_ctx;
    try {
      if (cfg) c->cfg = *cfg;
      c->device = c->cfg.device;
      CK(cudaSetDevice(c->device));
      cudaDeviceProp prop;
      CK(cudaGetDeviceProperties(&prop, c->device));
      if (prop.major < 10) throw CudaError("device is not sm_100 class (compute capability " +
                                           std::to_string(prop.major) + "." + std::to_string(prop.minor) + ")");
      c->n_sm = prop.multiProcessorCount;
      c->smem_optin = prop.sharedMemPerBlockOptin;
      CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      for (auto& e : c->ev) CK(cudaEventCreate(&e));
      // Globals, the wait ring and the inbox slots in one allocation (one IPC handle maps all)
      CK(cudaMalloc(&c->G, dev::kGlobalsBytes));
      CK(cudaMemset(c->G, 0, dev::kGlobalsBytes));
      reset_shared(c);
    } catch (...) {
      pccp_gpu_close(c);
      throw;
    }
    *out = c;
    return PCCP_OK;
  });
}

void pccp_gpu_close(pccp_gpu_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (void* p : c->opened) cudaIpcCloseMemHandle(p);
  c->blob.release();
  c->fa.release();
  c->fb.release();
  c->ia.release();
  c->ib.release();
  c->stack.release();
  c->mailbox.release();
  c->dec.release();
  c->chunk.release();
  c->audit.release();
  c->best.release();
  c->io.release();
  c->flags.release();
  c->st.release();
  c->rnd.release();
  c->d_peers.release();
  c->d_peer_shard.release();
  c->qlog.release();
  if (c->G) cudaFree(c->G);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

// The identity of a model for the lowering cache: every table of the ABI
// struct, and the environment knobs lower.cpp reads.
std::vector<std::int32_t> model_key(const pccp_model& m) {
  std::vector<std::int32_t> k;
  const std::uint32_t nc = m.cmd_off ? m.cmd_off[m.n_cmds] : 0;
  k.reserve(8 + 2 * (size_t)m.n_slots + m.n_cmds + nc + m.n_cands);
  k.push_back((std::int32_t)m.n_slots);
  k.push_back((std::int32_t)m.n_words);
  k.push_back((std::int32_t)m.n_cmds);
  k.push_back((std::int32_t)m.n_cands);
  k.push_back(m.obj_slot);
  for (std::uint32_t i = 0; i < m.n_slots; ++i) k.push_back(m.slot_kind ? m.slot_kind[i] : 0);
  if (m.slot_word) k.insert(k.end(), m.slot_word, m.slot_word + m.n_slots);
  if (m.cmd_off) k.insert(k.end(), m.cmd_off, m.cmd_off + m.n_cmds + 1);
  if (m.cmd_code) k.insert(k.end(), m.cmd_code, m.cmd_code + nc);
  if (m.cands) k.insert(k.end(), m.cands, m.cands + m.n_cands);
  for (const char* e : {"PCCP_FILTERED", "PCCP_NE_ORDER", "PCCP_NO_NE", "PCCP_NO_PACK", "PCCP_NO_REIF",
                        "PCCP_NO_REIF8", "PCCP_NO_ROWS", "PCCP_NO_UNIT", "PCCP_NO_WROWS", "PCCP_ROW_LANES",
                        "PCCP_ROW_PAIR", "PCCP_SCALAR_SCAN"}) {
    k.push_back(-1);
    if (const char* v = std::getenv(e))
      for (; *v; ++v) k.push_back(*v);
  }
  return k;
}

int pccp_gpu_load(pccp_gpu_ctx* c, const pccp_model* m) {
  return api([&] {
    if (!c || !m) throw ArgError("null argument");
    CK(cudaSetDevice(c->device));
    c->loaded = false;
    const bool lt = std::getenv("PCCP_LOAD_TIMING") != nullptr;
    double tl[8] = {now_ms()};
    // A reload of the model already lowered here (same tables, same lowering
    // knobs) keeps its lowering; the tables are still uploaded below.
    std::vector<std::int32_t> key = model_key(*m);
    if (!c->low_valid || key != c->low_key) {
      c->low_valid = false;
      c->low = lower_model(*m);
      if (c->low.L.n_cand >= (1u << 24)) throw LimitError("more than 2^24 branching candidates");
      // bit-plane cells only where the plain lowering found reifications or rows
      c->dl = (c->low.L.n_reif || c->low.L.n_rows) ? lower_packed(*m) : c->low;
      c->low_key = std::move(key);
      c->low_valid = true;
    }
    tl[1] = now_ms();
    reset_shared(c);  // an incumbent of the previous model means nothing for this one
    tl[2] = now_ms();
    c->slot_kind.assign(m->slot_kind, m->slot_kind + m->n_slots);
    c->slot_word.assign(m->slot_word, m->slot_word + m->n_slots);
    c->view = *m;
    c->view.slot_kind = c->slot_kind.data();
    c->view.slot_word = c->slot_word.data();
    c->view.cmd_off = nullptr;
    c->view.cmd_code = nullptr;
    c->view.cands = nullptr;
    c->blob.ensure(c->dl.blob.size() + 4);
    CK(cudaMemcpyAsync(c->blob.p, c->dl.blob.data(), c->dl.blob.size() * 4, cudaMemcpyHostToDevice, c->stream));
    tl[3] = now_ms();
    plan(c);
    tl[4] = now_ms();
    // Size the DFS stacks here rather than in the first solve: the depth bound
    // of the bottom store under the folded constant tells bounds the one of any
    // root reached from it by propagation (bounds only tighten).  Skipped when
    // a candidate is unbounded there (the solve sizes them from its root).
    {
      const DeviceLayout& L = c->low.L;
      std::vector<std::int32_t> r0(L.n_words);
      for (std::uint32_t w = 0; w < L.n_words; ++w) r0[w] = c->low.word_up[w] ? INT32_MIN : INT32_MAX;
      for (std::uint32_t k = 0; k < L.n_fold; ++k) {
        const std::uint32_t fw = static_cast<std::uint32_t>(c->low.blob[L.fold_w + k]);
        const std::int32_t v = c->low.blob[L.fold_v + k];
        const std::uint32_t w = fw & 0x7fffffffu;
        if (w >= L.n_words) continue;
        r0[w] = (fw >> 31) ? std::max(r0[w], v) : std::min(r0[w], v);
      }
      bool bounded = true;
      for (std::uint32_t i = 0; i < L.n_cand; ++i) {
        const int w = c->low.blob[L.cand_lbw + i];
        if (r0[w] == INT32_MIN || r0[w + 1] == INT32_MAX) bounded = false;
      }
      std::vector<std::int32_t> d0(c->dl.L.n_words);
      to_device(c->dl, r0.data(), d0.data());
      const size_t entry = align4(c->dl.L.n_words + 3);
      const size_t bytes = bounded ? (size_t)c->groups() * (size_t)depth_bound(c, d0) * entry * 4 : 0;
      // Best effort: at most a quarter of the free device memory (several
      // contexts may share a device); a solve whose root needs more sizes
      // the stacks itself (run_search), and a failed allocation here only
      // defers that.
      // (cudaMemGetInfo is a driver query that can wait behind a concurrent
      // nvidia-smi for tens of ms: a reload whose stacks already fit skips it)
      const bool fits = bytes / 4 <= c->stack.n && c->stack.p && (size_t)c->groups() * entry <= c->mailbox.n &&
                        c->mailbox.p;
      size_t free_b = 0, total_b = 0;
      tl[5] = now_ms();
      if (bounded && !fits) CK(cudaMemGetInfo(&free_b, &total_b));
      tl[6] = now_ms();
      if (bounded && !fits && bytes <= free_b / 4) {
        try {
          c->stack.ensure(bytes / 4);
          c->mailbox.ensure((size_t)c->groups() * entry);
              } catch (const LimitError&) {
          c->stack.release();
          c->mailbox.release();
        }
      }
    }
    CK(cudaStreamSynchronize(c->stream));
    if (lt)
      fprintf(stderr, "pccp_gpu_load: lower %.3f reset %.3f upload %.3f plan %.3f bound %.3f meminfo %.3f rest %.3f ms\n",
              tl[1] - tl[0], tl[2] - tl[1], tl[3] - tl[2], tl[4] - tl[3], tl[5] - tl[4], tl[6] - tl[5],
              now_ms() - tl[6]);
    c->loaded = true;
    return PCCP_OK;
  });
}

int pccp_gpu_lowering_info(pccp_gpu_ctx* c, pccp_lowering_info* o) {
  return api([&] {
    check_loaded(c);
    const DeviceLayout& L = c->low.L;
    std::memset(o, 0, sizeof(*o));
    o->n_words = L.n_words;
    o->n_cmds = L.n_ref_cmds;
    o->n_folded = L.n_fold;
    o->n_small = L.n_small;
    o->n_rows = L.n_rows;
    o->n_row_terms = L.n_row_terms;
    o->n_generic = L.n_gen;
    o->table_bytes = c->dl.L.hot_words * 4;
    o->store_bytes = c->dl.L.n_words * 4;
    o->packed_cells = (std::uint32_t)c->dl.bit_lbw.size();
    o->device_words = c->dl.L.n_words;
    o->group_threads = c->warp ? 32 : c->block;
    o->groups_per_cta = c->warp ? c->gpc : 1;
    o->ctas = c->ctas;
    o->smem_bytes = (std::uint32_t)c->smem;
    o->table_in_smem = c->table_in_smem;
    o->stack_in_smem = 0;
    o->alg_bytes_per_eval = c->low.alg_bytes_per_eval;
    o->store_bytes_per_round = c->dl.store_bytes_per_round;
    o->table_bytes_per_round = c->dl.table_bytes_per_round;
    o->stack_depth = 0;
    return PCCP_OK;
  });
}

int pccp_lower_only(const pccp_model* m, pccp_lowering_info* o, uint32_t* shape_counts) {
  return api([&] {
    if (!m || !o) throw ArgError("null argument");
    const Lowered low = lower_model(*m);
    const DeviceLayout& L = low.L;
    std::memset(o, 0, sizeof(*o));
    {
      const Lowered pk = lower_packed(*m);
      o->packed_cells = (std::uint32_t)pk.bit_lbw.size();
      o->device_words = pk.L.n_words;
    }
    o->n_words = L.n_words;
    o->n_cmds = L.n_ref_cmds;
    o->n_folded = L.n_fold;
    o->n_small = L.n_small;
    o->n_rows = L.n_rows;
    o->n_row_terms = L.n_row_terms;
    o->n_generic = L.n_gen;
    o->table_bytes = L.hot_words * 4;
    o->store_bytes = L.n_words * 4;
    o->alg_bytes_per_eval = low.alg_bytes_per_eval;
    o->store_bytes_per_round = low.store_bytes_per_round;
    o->table_bytes_per_round = low.table_bytes_per_round;
    if (shape_counts) {
      shape_counts[0] = L.n_unit1;
      shape_counts[1] = L.n_unit2;
      shape_counts[2] = low.n_dropped;
      shape_counts[3] = L.n_ne;
      shape_counts[4] = L.filtered;
      shape_counts[5] = L.n_reif;
    }
    return PCCP_OK;
  });
}

int pccp_lower_fast_paths(const pccp_model* m, const int32_t* stores, uint32_t n, uint32_t* mask) {
  return api([&] {
    if (!m || !mask || (n && !stores)) throw ArgError("null argument");
    const Lowered low = lower_model(*m);
    bool ne = false, rows = false, reif = false, unit = false;
    fast_paths(low, stores, n, low.L.n_words, ne, rows, reif, unit);
    *mask = (ne ? 1u : 0u) | (rows ? 2u : 0u) | (reif ? 4u : 0u) | (unit ? 8u : 0u);
    return PCCP_OK;
  });
}

int pccp_lower_layout(const pccp_model* m, const int32_t* stores, uint32_t n, int32_t* dev, int32_t* back,
                      uint32_t* dev_words) {
  return api([&] {
    if (!m || !dev_words || (n && !stores)) throw ArgError("null argument");
    const Lowered d = lower_packed(*m);
    *dev_words = d.L.n_words;
    const size_t rw = m->n_words, dw = d.L.n_words;
    for (uint32_t i = 0; i < n; ++i) {
      std::vector<std::int32_t> t(dw);
      to_device(d, stores + i * rw, t.data());
      if (dev) std::copy(t.begin(), t.end(), dev + i * dw);
      if (back) to_reference(d, t.data(), back + i * rw);
    }
    return PCCP_OK;
  });
}

int pccp_gpu_propagate_batch(pccp_gpu_ctx* c, const int32_t* in, uint32_t n, int32_t* out, uint8_t* status,
                             uint32_t* rounds) {
  return api([&] {
    check_loaded(c);
    if (n == 0) return PCCP_OK;
    if (!in || !out || !status) throw ArgError("null buffer");
    const size_t rw = c->low.L.n_words, nw = c->dl.L.n_words;  // reference / device words
    c->io.ensure((size_t)n * std::max<size_t>(nw, 1));
    c->st.ensure(n);
    c->rnd.ensure(n);
    std::vector<std::int32_t> dev_in;
    const std::int32_t* src = in;
    if (c->dl.L.packed) {
      dev_in.resize((size_t)n * nw);
      for (uint32_t i = 0; i < n; ++i) to_device(c->dl, in + (size_t)i * rw, dev_in.data() + (size_t)i * nw);
      src = dev_in.data();
    }
    if (nw) CK(cudaMemcpyAsync(c->io.p, src, (size_t)n * nw * 4, cudaMemcpyHostToDevice, c->stream));
    const dev::Model M = c->model(0, 0, in, n, rw);
    const int per = c->warp ? c->gpc : 1;
    const int grid = (int)std::min<long long>(c->ctas, ((long long)n + per - 1) / per);
    dispatch(c, [&]<class Gp, bool TS, int F>() {
      dev::k_propagate<Gp, TS, F><<<grid, c->block, c->smem, c->stream>>>(M, c->io.p, (int)n, (int)nw, c->st.p,
                                                                       c->rnd.p, 1);
    });
    CK(cudaGetLastError());
    ++c->launches;
    if (c->dl.L.packed) {
      CK(cudaMemcpyAsync(dev_in.data(), c->io.p, (size_t)n * nw * 4, cudaMemcpyDeviceToHost, c->stream));
    } else if (nw) {
      CK(cudaMemcpyAsync(out, c->io.p, (size_t)n * nw * 4, cudaMemcpyDeviceToHost, c->stream));
    }
    CK(cudaMemcpyAsync(status, c->st.p, n, cudaMemcpyDeviceToHost, c->stream));
    if (rounds) CK(cudaMemcpyAsync(rounds, c->rnd.p, (size_t)n * 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (c->dl.L.packed)
      for (uint32_t i = 0; i < n; ++i) to_reference(c->dl, dev_in.data() + (size_t)i * nw, out + (size_t)i * rw);
    return PCCP_OK;
  });
}

int pccp_gpu_replay(pccp_gpu_ctx* c, const int32_t* root, uint32_t n_paths, const uint32_t* path_off,
                    const pccp_decision* dec, const int32_t* best, int32_t* out, uint8_t* status) {
  return api([&] {
    check_loaded(c);
    const size_t nw = c->low.L.n_words;
    std::vector<std::int32_t> stores((size_t)n_paths * nw);
    for (uint32_t p = 0; p < n_paths; ++p) {
      std::int32_t* s = stores.data() + (size_t)p * nw;
      std::memcpy(s, root, nw * 4);
      for (uint32_t k = path_off[p]; k < path_off[p + 1]; ++k) host_join_decision(c->view, s, dec[k]);
      const std::int32_t b = best ? best[p] : INT32_MAX;
      if (b != INT32_MAX && c->low.L.obj_lbw >= 0) {
        std::int32_t& ub = s[c->low.L.obj_lbw + 1];
        if (b - 1 < ub) ub = b - 1;
      }
    }
    const int r = pccp_gpu_propagate_batch(c, stores.data(), n_paths, out, status, nullptr);
    if (r != PCCP_OK) throw CudaError(g_err);
    return PCCP_OK;
  });
}

int pccp_gpu_enumerate(pccp_gpu_ctx* c, const int32_t* root, int32_t depth_cap, const pccp_limits* lim,
                       pccp_enum_result* out) {
  return api([&] {
    check_loaded(c);
    if (!root || !out) throw ArgError("null argument");
    std::memset(out, 0, sizeof(*out));
    if (lim && lim->node_limit == 0) return PCCP_OK;
    RunOut r;
    dispatch(c, [&]<class Gp, bool TS, int F>() { run_search<Gp, TS, F>(c, 0, root, depth_cap, lim, r); });
    fill_stats(c, r, out->stats);
    out->exhausted = r.g.incomplete ? 0 : 1;
    return PCCP_OK;
  });
}

int pccp_gpu_solve(pccp_gpu_ctx* c, const int32_t* root, const pccp_limits* lim, pccp_solve_result* out,
                   int32_t* best_words) {
  return api([&] {
    check_loaded(c);
    if (!root || !out) throw ArgError("null argument");
    if (c->low.L.obj_lbw < 0) throw std::runtime_error("solve: the model has no objective");
    std::memset(out, 0, sizeof(*out));
    if (lim && lim->node_limit == 0) {  // should_stop before the root (solver.cpp:240)
      out->status = PCCP_UNKNOWN;
      return PCCP_OK;
    }
    const int var_order = std::clamp(c->cfg.var_order, 0, 3);
    const char* pv = std::getenv("PCCP_PRIMAL_VAR_ORDER");
    const int primal_order = pv ? std::clamp(std::atoi(pv), 1, 3) : 2;
    // Segment 0 uses primal_order; later segments (restarts) alternate
    // randomised ties (var_order 3, a new seed per segment, a different order
    // per group) with primal_order, and keep restarting while time remains
    // even after a segment without improvement.  Opt-in (PCCP_PRIMAL_DIVERSIFY=1):
    // on RCPSP120 it found 257 instead of 258 in 10 s, and 92 instead of 91 on
    // RCPSP30 seed 10; the default is the plain restart-on-improvement loop.
    const char* pdv = std::getenv("PCCP_PRIMAL_DIVERSIFY");
    const bool diversify = pdv && std::atoi(pdv) != 0;
    // With N shards every GPU dives the WHOLE tree in the primal phase
    // (sharded = false below), so a segment that exhausts its tree is a proof
    // by itself, whatever the other GPUs did.  Shard 0 keeps primal_order;
    // the others take randomised ties (var_order 3, seeded by shard and
    // segment), so the N dives differ.
    const int shards = std::max(1, c->cfg.shard_count);
    auto seg_order = [&](int seg) {
      if (shards > 1 && c->cfg.shard_index > 0) return 3;
      return (diversify && (seg & 1)) ? 3 : primal_order;
    };
    std::vector<std::pair<int, double>> log;  // improvement log over all phases
    RunOut r;
    out->phases = 1;
    const double t_call = now_ms();
    auto left = [&](pccp_limits& l, const RunOut& acc) {  // the caller's limits minus what was used
      l = lim ? *lim : pccp_limits{0.0, ~0ull};
      if (l.timeout_s > 0) l.timeout_s -= (now_ms() - t_call) * 1e-3;
      if (l.node_limit != ~0ull) l.node_limit = l.node_limit > acc.g.nodes ? l.node_limit - acc.g.nodes : 0;
      return !(lim && lim->timeout_s > 0 && l.timeout_s <= 0) && l.node_limit > 0;
    };
    bool proved = false;
    if (c->cfg.primal_ms > 0) {
      // Primal phase: smallest-lb dives (complete searches of another tree),
      // restarted from the root under obj <= best-1 whenever a segment stalls
      // (no improvement for stall_ms) after improving; bounded by primal_ms
      // and the caller's limits.
      const double budget_ms = c->cfg.primal_ms;
      const char* se = std::getenv("PCCP_PRIMAL_STALL_MS");
      const double stall_ms = se ? std::atof(se) : std::max(100.0, 0.05 * budget_ms);
      RunOut acc;
      acc.g.incumbent = acc.g.best_value = INT32_MAX;  // nothing ran yet: no incumbent, no proof
      acc.g.incomplete = 1;
      for (int seg = 0;; ++seg) {
        pccp_limits l1;
        if (!left(l1, acc)) break;
        const double spent = now_ms() - t_call;
        if (spent >= budget_ms) break;
        const double p_s = (budget_ms - spent) * 1e-3;
        l1.timeout_s = l1.timeout_s > 0 ? std::min(l1.timeout_s, p_s) : p_s;
        RunOut r1;
        dispatch(c, [&]<class Gp, bool TS, int F>() {
          run_search<Gp, TS, F>(c, 1, root, -1, &l1, r1, seg_order(seg), seg > 0,
                                (unsigned long long)(stall_ms * 1e6), (unsigned)seg + 7919u * (unsigned)c->cfg.shard_index,
                                /*sharded=*/false);
        });
        append_log(r1, acc.device_ms, log);
        merge_run(acc, r1, seg == 0);
        if (r1.g.incomplete == 0) {
          proved = true;
          if (c->n_peers > 0) {  // the whole tree is exhausted: every peer may stop
            dev::k_signal_done<<<1, 1, 0, c->stream>>>(c->d_peers.p, c->n_peers);
            CK(cudaGetLastError());
            CK(cudaStreamSynchronize(c->stream));
          }
          break;
        }
        if (r1.g.done) break;                                  // a peer proved it
        if (!r1.g.stalled) break;                              // out of time or limits
        if (r1.g.n_impr == 0 && !(diversify && seg + 1 < 64)) break;  // nothing new
        out->primal_restarts = seg + 1;
      }
      out->primal_nodes = acc.g.nodes;
      out->primal_device_ms = acc.device_ms;
      out->primal_proved = proved ? 1 : 0;
      r = acc;
    }
    pccp_limits l2;
    if (c->cfg.primal_ms <= 0) {
      dispatch(c, [&]<class Gp, bool TS, int F>() { run_search<Gp, TS, F>(c, 1, root, -1, lim, r, var_order); });
      append_log(r, 0.0, log);
    } else if (!proved && !r.g.done && left(l2, r)) {
      RunOut r2;
      dispatch(c, [&]<class Gp, bool TS, int F>() { run_search<Gp, TS, F>(c, 1, root, -1, &l2, r2, var_order, true); });
      append_log(r2, r.device_ms, log);
      merge_run(r, r2, false);
      out->phases = 2;
    }
    fill_stats(c, r, out->stats);
    const bool exhausted = r.g.incomplete == 0;
    const bool has = r.g.incumbent != INT32_MAX;
    out->has_objective = has ? 1 : 0;
    out->objective = has ? r.g.incumbent : 0;
    out->status = has ? (exhausted ? PCCP_OPTIMAL : PCCP_SAT) : (exhausted ? PCCP_UNSAT : PCCP_UNKNOWN);
    // keep the first 32 and the last 32 improvements (the last one is the incumbent)
    if (log.size() > 64) log.erase(log.begin() + 32, log.end() - 32);
    out->n_improvements = (int32_t)log.size();
    for (int k = 0; k < out->n_improvements; ++k) {
      out->improvements[k] = log[k].first;
      out->improvement_ms[k] = log[k].second;
    }
    if (best_words && has && r.g.best_value == r.g.incumbent) {
      std::vector<std::int32_t> dw(c->dl.L.n_words);
      CK(cudaMemcpy(dw.data(), c->best.p, dw.size() * 4, cudaMemcpyDeviceToHost));
      to_reference(c->dl, dw.data(), best_words);
    }
    else if (best_words && has)
      out->has_objective = 2;  // incumbent found on a peer GPU: its store lives there
    return PCCP_OK;
  });
}

int pccp_gpu_incumbent_handle(pccp_gpu_ctx* c, uint8_t* out64) {
  return api([&] {
    if (!c || !out64) throw ArgError("null argument");
    CK(cudaSetDevice(c->device));
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, c->G));
    static_assert(sizeof(h) <= 64, "IPC handle larger than 64 bytes");
    std::memset(out64, 0, 64);
    std::memcpy(out64, &h, sizeof(h));
    return PCCP_OK;
  });
}

int pccp_gpu_attach_peers(pccp_gpu_ctx* c, const uint8_t* handles, int32_t n, int32_t self) {
  return api([&] {
    if (!c || (n > 0 && !handles)) throw ArgError("null argument");
    CK(cudaSetDevice(c->device));
    std::vector<dev::Globals*> ptrs;
    std::vector<int> shard;  // handle i belongs to shard i (distributed.attach_incumbents gathers by rank)
    for (int i = 0; i < n; ++i) {
      if (i == self) continue;
      cudaIpcMemHandle_t h;
      std::memcpy(&h, handles + 64 * i, sizeof(h));
      void* p = nullptr;
      CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
      c->opened.push_back(p);
      ptrs.push_back(static_cast<dev::Globals*>(p));
      shard.push_back(i);
    }
    c->n_peers = (int)ptrs.size();
    if (!ptrs.empty()) {
      c->d_peers.ensure(ptrs.size());
      CK(cudaMemcpy(c->d_peers.p, ptrs.data(), ptrs.size() * sizeof(dev::Globals*), cudaMemcpyHostToDevice));
      c->d_peer_shard.ensure(shard.size());
      CK(cudaMemcpy(c->d_peer_shard.p, shard.data(), shard.size() * sizeof(int), cudaMemcpyHostToDevice));
    }
    return PCCP_OK;
  });
}

int pccp_gpu_reset_shared(pccp_gpu_ctx* c) {
  return api([&] {
    if (!c) throw ArgError("null context");
    CK(cudaSetDevice(c->device));
    reset_shared(c);
    return PCCP_OK;
  });
}

int pccp_gpu_offer_incumbent(pccp_gpu_ctx* c, int32_t value) {
  return api([&] {
    if (!c) throw ArgError("null context");
    CK(cudaSetDevice(c->device));
    dev::k_offer_incumbent<<<1, 1, 0, c->stream>>>(c->G, value);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(c->stream));
    return PCCP_OK;
  });
}

int pccp_gpu_frontier(pccp_gpu_ctx* c, uint64_t* all, uint32_t* n_all, uint64_t* share, uint32_t* n_share,
                      uint32_t cap) {
  return api([&] {
    if (!c || !n_all || !n_share) throw ArgError("null argument");
    *n_all = (uint32_t)c->frontier_all.size();
    *n_share = (uint32_t)c->frontier_share.size();
    if (all) std::copy_n(c->frontier_all.begin(), std::min<size_t>(cap, c->frontier_all.size()), all);
    if (share) std::copy_n(c->frontier_share.begin(), std::min<size_t>(cap, c->frontier_share.size()), share);
    return PCCP_OK;
  });
}

int pccp_gpu_audit(pccp_gpu_ctx* c, int32_t* pre, int32_t* post, uint8_t* failed, uint32_t* n_out) {
  return api([&] {
    check_loaded(c);
    if (!n_out) throw ArgError("null argument");
    *n_out = 0;
    if (c->cfg.audit_nodes <= 0 || !c->audit.p) return PCCP_OK;
    const size_t nw = std::max<size_t>(c->dl.L.n_words, 1), rw = c->low.L.n_words, k = (size_t)c->cfg.audit_nodes,
                 n = c->audit_taken;
    if (n && (!pre || !post || !failed)) throw ArgError("null buffer");
    if (n) {
      std::vector<std::int32_t> a(n * nw), b(n * nw);
      CK(cudaMemcpy(a.data(), c->audit.p, n * nw * 4, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(b.data(), c->audit.p + k * nw, n * nw * 4, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(failed, c->audit.p + 2 * k * nw, n, cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < n; ++i) {
        to_reference(c->dl, a.data() + i * nw, pre + i * rw);
        to_reference(c->dl, b.data() + i * nw, post + i * rw);
      }
    }
    *n_out = (uint32_t)n;
    return PCCP_OK;
  });
}

int pccp_gpu_link_peers(pccp_gpu_ctx* const* ctxs, int32_t n) {
  return api([&] {
    if (n < 0 || (n > 0 && !ctxs)) throw ArgError("null argument");
    for (int i = 0; i < n; ++i)
      if (!ctxs[i]) throw ArgError("null context");
    for (int i = 0; i < n; ++i) {
      pccp_gpu_ctx* c = ctxs[i];
      CK(cudaSetDevice(c->device));
      std::vector<dev::Globals*> ptrs;
      std::vector<int> shard;
      for (int j = 0; j < n; ++j) {
        if (j == i) continue;
        const int dj = ctxs[j]->device;
        if (dj != c->device) {
          int can = 0;
          CK(cudaDeviceCanAccessPeer(&can, c->device, dj));
          if (!can) throw CudaError("device " + std::to_string(c->device) + " cannot access peer " + std::to_string(dj));
          const cudaError_t e = cudaDeviceEnablePeerAccess(dj, 0);
          if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
          else CK(e);
        }
        ptrs.push_back(ctxs[j]->G);
        shard.push_back(ctxs[j]->cfg.shard_index);
      }
      c->n_peers = (int)ptrs.size();
      if (!ptrs.empty()) {
        c->d_peers.ensure(ptrs.size());
        CK(cudaMemcpy(c->d_peers.p, ptrs.data(), ptrs.size() * sizeof(dev::Globals*), cudaMemcpyHostToDevice));
        c->d_peer_shard.ensure(shard.size());
        CK(cudaMemcpy(c->d_peer_shard.p, shard.data(), shard.size() * sizeof(int), cudaMemcpyHostToDevice));
      }
    }
    return PCCP_OK;
  });
}

}  // extern "C"
