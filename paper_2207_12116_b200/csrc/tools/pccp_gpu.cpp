// pccp_gpu — the reference CLI's `solve` and `verify` (tools/pccp.cpp:43-188)
// on the B200 engine.  Same instance formats (Patterson .rcp, .json), same
// report keys (status, objective, nodes, time_ms, nodes_per_sec), same JSON
// keys and exit codes (0 done, 2 UNKNOWN, 1 error; test_cli.cpp:56-118).
//
//   pccp_gpu solve FILE [--gpus N] [--devices d0,d1,..] [--timeout S] [--eps-factor K]
//                       [--primal-ms MS] [--json] [--stats]
//                       [--engine seq|fair|par] [--workers W] [--seed S]   (accepted, see below)
//   pccp_gpu verify FILE
//   pccp_gpu gen SEED N_REAL RESOURCES   (Patterson text of random_patterson(mt19937_64(SEED), ..),
//                                         the generator of the benchmark configs 4 and 5)
//
// `--gpus N` runs one context per device on its own host thread; the EPS
// frontier is sharded i mod N and the incumbent is shared by peer atomics
// (pccp_gpu_link_peers).  The reference's --engine/--workers/--seed select
// CPU propagation engines and thread counts; the device has one engine (the
// eventless fixed-point loop), so they are validated and otherwise ignored.
// `verify` is the reference's cross-engine confluence check with the device
// configurations as the engines: the root fixed point under warp groups and
// CTA groups of 64..1024 threads, tables in shared or global memory, must
// agree cell for cell.
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "../../../include/pccp_gpu.h"
#include "../host/model.hpp"
#include "../host/rcpsp.hpp"

using namespace pccp_b200;

namespace {

struct Config {
  std::string cmd, instance, engine = "seq";
  int gpus = 1;
  std::vector<int> devices;
  double timeout_s = 300.0;
  int eps_factor = 8;
  int primal_ms = 0;
  unsigned workers = 1;
  std::uint64_t seed = 1;
  bool json = false, stats = false;
  std::vector<double> gen;
};

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

const char* status_name(int s) {
  switch (s) {
    case PCCP_OPTIMAL: return "OPTIMAL";
    case PCCP_SAT: return "SAT";
    case PCCP_UNSAT: return "UNSAT";
    default: return "UNKNOWN";
  }
}

RcpspInstance load_instance(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ModelError("cannot open instance file: " + path);
  std::ostringstream buf;
  buf << in.rdbuf();
  if (path.size() > 5 && path.substr(path.size() - 5) == ".json") return parse_json(buf.str());
  return parse_patterson(buf.str());
}

void check(int rc, const char* what) {
  if (rc != PCCP_OK) throw std::runtime_error(std::string(what) + ": " + pccp_gpu_last_error());
}

pccp_model view_of(const FlatTables& t) {
  pccp_model m{};
  m.n_slots = static_cast<std::uint32_t>(t.slot_kind.size());
  m.slot_kind = t.slot_kind.data();
  m.slot_word = t.slot_word.data();
  m.n_words = t.n_words;
  m.n_cmds = static_cast<std::uint32_t>(t.cmd_off.size() - 1);
  m.cmd_off = t.cmd_off.data();
  m.cmd_code = t.cmd_code.data();
  m.n_cands = static_cast<std::uint32_t>(t.cands.size());
  m.cands = t.cands.data();
  m.obj_slot = t.obj_slot;
  return m;
}

std::string interval_text(const std::int32_t* w) {
  auto one = [](std::int32_t v) {
    if (v == INT32_MIN) return std::string("-inf");
    if (v == INT32_MAX) return std::string("+inf");
    return std::to_string(v);
  };
  return "[" + one(w[0]) + ", " + one(w[1]) + "]";
}

int cmd_solve(const Config& cfg) {
  RcpspInstance inst;
  RcpspModel rm;
  FlatTables tables;
  try {
    inst = load_instance(cfg.instance);
    rm = build_rcpsp(inst);
    tables = rm.model->flatten();
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
  const pccp_model view = view_of(tables);
  const std::vector<std::int32_t> root = rm.model->bottom();
  const int n = cfg.gpus;

  std::vector<pccp_gpu_ctx*> ctx(static_cast<std::size_t>(n), nullptr);
  auto close_all = [&] {
    for (auto* c : ctx) pccp_gpu_close(c);
  };
  std::vector<pccp_solve_result> res(static_cast<std::size_t>(n));
  std::vector<std::vector<std::int32_t>> best(static_cast<std::size_t>(n),
                                              std::vector<std::int32_t>(std::max<std::uint32_t>(view.n_words, 1)));
  std::vector<int> rc(static_cast<std::size_t>(n), PCCP_OK);
  std::vector<std::string> err(static_cast<std::size_t>(n));
  try {
    for (int i = 0; i < n; ++i) {
      pccp_gpu_cfg gc{};
      gc.device = cfg.devices.empty() ? i : cfg.devices[static_cast<std::size_t>(i)];
      gc.shard_index = i;
      gc.shard_count = n;
      gc.eps_factor = cfg.eps_factor;
      gc.primal_ms = cfg.primal_ms;
      check(pccp_gpu_open(&gc, &ctx[static_cast<std::size_t>(i)]), "open");
      check(pccp_gpu_load(ctx[static_cast<std::size_t>(i)], &view), "load");
    }
    if (n > 1) check(pccp_gpu_link_peers(ctx.data(), n), "link peers");
  } catch (const std::exception& e) {
    close_all();
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }

  pccp_limits lim{cfg.timeout_s, ~0ull};
  const auto t0 = std::chrono::steady_clock::now();
  {
    std::vector<std::thread> th;
    for (int i = 0; i < n; ++i) {
      th.emplace_back([&, i] {
        const auto k = static_cast<std::size_t>(i);
        rc[k] = pccp_gpu_solve(ctx[k], root.data(), &lim, &res[k], best[k].data());
        if (rc[k] != PCCP_OK) err[k] = pccp_gpu_last_error();
      });
    }
    for (auto& t : th) t.join();
  }
  const auto ms =
      std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0).count();
  close_all();
  for (int i = 0; i < n; ++i) {
    if (rc[static_cast<std::size_t>(i)] != PCCP_OK) {
      std::cerr << "error: " << err[static_cast<std::size_t>(i)] << "\n";
      return 1;
    }
  }

  // finish() (solver.cpp:148-162) over the union of the shards: every shard
  // exhausted (they partition one bound-free EPS frontier), or one GPU's
  // primal dive exhausted the whole tree.
  bool exhausted = true, has = false, whole_tree = false;
  std::int32_t obj = 0;
  int owner = -1;
  std::uint64_t nodes = 0, primal_nodes = 0, restarts = 0;
  for (int i = 0; i < n; ++i) {
    const pccp_solve_result& r = res[static_cast<std::size_t>(i)];
    exhausted = exhausted && (r.status == PCCP_OPTIMAL || r.status == PCCP_UNSAT);
    whole_tree = whole_tree || r.primal_proved;
    nodes += r.stats.nodes;
    primal_nodes += r.primal_nodes;
    restarts += static_cast<std::uint64_t>(r.primal_restarts);
    if (r.has_objective && (!has || r.objective < obj)) {
      has = true;
      obj = r.objective;
    }
  }
  exhausted = exhausted || whole_tree;
  for (int i = 0; i < n && has; ++i) {
    const pccp_solve_result& r = res[static_cast<std::size_t>(i)];
    if (r.has_objective == 1 && r.objective == obj) {
      owner = i;
      break;
    }
  }
  const int status = has ? (exhausted ? PCCP_OPTIMAL : PCCP_SAT) : (exhausted ? PCCP_UNSAT : PCCP_UNKNOWN);

  if (has && inst.tasks() > 0) {
    if (owner < 0) {
      std::cerr << "error: the best solution's store is missing\n";
      return 1;
    }
    std::vector<std::int32_t> starts;
    for (std::int32_t s : rm.starts) starts.push_back(best[static_cast<std::size_t>(owner)][rm.model->first_word(s)]);
    if (!check_solution(inst, starts)) {
      std::cerr << "error: reported solution failed the independent check\n";
      return 1;
    }
  }

  const std::int64_t nps = ms > 0 ? static_cast<std::int64_t>(nodes) * 1000 / ms : static_cast<std::int64_t>(nodes) * 1000;
  if (cfg.json) {
    // nlohmann::json's default object keeps keys sorted: same text as the reference
    std::cout << "{\"nodes\":" << nodes << ",\"nodes_per_sec\":" << nps
              << ",\"objective\":" << (has ? std::to_string(obj) : std::string("null")) << ",\"status\":\""
              << status_name(status) << "\",\"time_ms\":" << ms;
    if (cfg.stats)
      std::cout << ",\"gpus\":" << n << ",\"primal_nodes\":" << primal_nodes << ",\"primal_restarts\":" << restarts;
    std::cout << "}\n";
  } else {
    std::cout << "status: " << status_name(status) << "\n";
    std::cout << "objective: " << (has ? std::to_string(obj) : std::string("none")) << "\n";
    std::cout << "nodes: " << nodes << "\n";
    std::cout << "time_ms: " << ms << "\n";
    std::cout << "nodes_per_sec: " << nps << "\n";
    if (cfg.stats) {
      std::cout << "gpus: " << n << "\n";
      std::cout << "primal_nodes: " << primal_nodes << "\n";
      std::cout << "primal_restarts: " << restarts << "\n";
    }
  }
  return status == PCCP_UNKNOWN ? 2 : 0;
}

int cmd_verify(const Config& cfg) {
  RcpspInstance inst;
  RcpspModel rm;
  FlatTables tables;
  try {
    inst = load_instance(cfg.instance);
    rm = build_rcpsp(inst);
    tables = rm.model->flatten();
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
  const pccp_model view = view_of(tables);
  const std::vector<std::int32_t> root = rm.model->bottom();
  const int device = cfg.devices.empty() ? 0 : cfg.devices[0];
  struct Run {
    std::string name;
    std::vector<std::int32_t> words;
    int status;
  };
  std::vector<Run> runs;
  const int threads[] = {32, 64, 128, 256, 512, 1024};
  for (int smem = 1; smem >= 0; --smem) {
    for (int t : threads) {
      // table placement is chosen at load time (engine.cu plan, PCCP_TABLE_SMEM)
      setenv("PCCP_TABLE_SMEM", smem ? "1" : "0", 1);
      pccp_gpu_cfg gc{};
      gc.device = device;
      gc.group_threads = t;
      gc.groups_per_cta = 1;
      pccp_gpu_ctx* c = nullptr;
      int r = pccp_gpu_open(&gc, &c);
      if (r == PCCP_OK) r = pccp_gpu_load(c, &view);
      pccp_lowering_info info{};
      if (r == PCCP_OK) r = pccp_gpu_lowering_info(c, &info);
      // a configuration the model does not fit (store or tables beyond shared
      // memory) is not an engine of this model
      if (r == PCCP_ELIMIT || (r == PCCP_OK && static_cast<int>(info.table_in_smem) != smem)) {
        pccp_gpu_close(c);
        continue;
      }
      Run run{(t == 32 ? std::string("warp") : "cta" + std::to_string(t)) + (smem ? "/smem" : "/global"),
              std::vector<std::int32_t>(std::max<std::uint32_t>(view.n_words, 1)), 0};
      std::uint8_t st = 0;
      if (r == PCCP_OK) r = pccp_gpu_propagate_batch(c, root.data(), 1, run.words.data(), &st, nullptr);
      if (r != PCCP_OK) {
        std::cerr << "error: " << run.name << ": " << pccp_gpu_last_error() << "\n";
        pccp_gpu_close(c);
        unsetenv("PCCP_TABLE_SMEM");
        return 1;
      }
      pccp_gpu_close(c);
      run.status = st;
      runs.push_back(std::move(run));
    }
  }
  unsetenv("PCCP_TABLE_SMEM");
  if (runs.empty()) {
    std::cerr << "error: the model fits no device configuration\n";
    return 1;
  }
  const Run& ref = runs.front();
  const Model& m = *rm.model;
  for (const Run& run : runs) {
    if (run.status != ref.status) {
      std::cout << "FAIL: " << run.name << " ended " << (run.status ? "Failed" : "Fixpoint") << " but " << ref.name
                << " ended " << (ref.status ? "Failed" : "Fixpoint") << "\n";
      return 1;
    }
    if (ref.status) continue;  // failed stores are all top
    for (std::int32_t s = 0; s < m.slot_count(); ++s) {
      const std::uint32_t w = m.first_word(s);
      const int nw = m.kind(s) == Kind::Interval ? 2 : 1;
      if (std::memcmp(&run.words[w], &ref.words[w], static_cast<std::size_t>(nw) * 4) != 0) {
        const std::string a = nw == 2 ? interval_text(&run.words[w]) : std::to_string(run.words[w]);
        const std::string b = nw == 2 ? interval_text(&ref.words[w]) : std::to_string(ref.words[w]);
        std::cout << "FAIL: cell '" << m.name(s) << "' differs: " << run.name << " has " << a << ", " << ref.name
                  << " has " << b << "\n";
        return 1;
      }
    }
  }
  std::cout << "PASS: " << runs.size() << " engine runs agree on " << m.slot_count() << " cells\n";
  return 0;
}

void usage(std::ostream& o) {
  o << "PCCP constraint solver (B200 engine)\n"
       "usage: pccp_gpu solve FILE [--gpus N] [--devices d0,d1,..] [--timeout S] [--eps-factor K]\n"
       "                           [--primal-ms MS] [--json] [--stats] [--engine seq|fair|par]\n"
       "                           [--workers W] [--seed S]\n"
       "       pccp_gpu verify FILE\n"
       "       pccp_gpu gen SEED N_REAL RESOURCES\n";
}

Config parse_args(int argc, char** argv) {
  Config cfg;
  if (const char* env = std::getenv("PCCP_WORKERS")) cfg.workers = static_cast<unsigned>(std::max(1, std::atoi(env)));
  if (argc < 2) throw UsageError("a subcommand is required");
  cfg.cmd = argv[1];
  if (cfg.cmd == "gen") {
    if (argc != 5) throw UsageError("gen takes SEED N_REAL RESOURCES");
    for (int i = 2; i < 5; ++i) {
      char* end = nullptr;
      const double x = std::strtod(argv[i], &end);
      if (!end || *end || x < 0 || x > 1.8e19) throw UsageError(std::string("gen: bad value '") + argv[i] + "'");
      cfg.gen.push_back(x);
    }
    return cfg;
  }
  if (cfg.cmd != "solve" && cfg.cmd != "verify") throw UsageError("unknown subcommand: " + cfg.cmd);
  auto num = [](const std::string& flag, const char* v, double lo, double hi) {
    char* end = nullptr;
    const double x = std::strtod(v, &end);
    if (!end || *end || x < lo || x > hi) throw UsageError(flag + ": bad value '" + v + "'");
    return x;
  };
  for (int i = 2; i < argc; ++i) {
    const std::string a = argv[i];
    auto val = [&]() -> const char* {
      if (i + 1 >= argc) throw UsageError(a + " needs a value");
      return argv[++i];
    };
    if (a == "--json" && cfg.cmd == "solve") cfg.json = true;
    else if (a == "--stats" && cfg.cmd == "solve") cfg.stats = true;
    else if (a == "--gpus" && cfg.cmd == "solve") cfg.gpus = static_cast<int>(num(a, val(), 1, 64));
    else if (a == "--timeout" && cfg.cmd == "solve") cfg.timeout_s = num(a, val(), 0, 1e9);
    else if (a == "--eps-factor" && cfg.cmd == "solve") cfg.eps_factor = static_cast<int>(num(a, val(), 1, 1 << 20));
    else if (a == "--primal-ms" && cfg.cmd == "solve") cfg.primal_ms = static_cast<int>(num(a, val(), 0, 2e9));
    else if (a == "--workers" && cfg.cmd == "solve") cfg.workers = static_cast<unsigned>(num(a, val(), 1, 1 << 20));
    else if (a == "--seed" && cfg.cmd == "solve") cfg.seed = static_cast<std::uint64_t>(num(a, val(), 0, 1.8e19));
    else if (a == "--engine" && cfg.cmd == "solve") {
      cfg.engine = val();
      if (cfg.engine != "seq" && cfg.engine != "fair" && cfg.engine != "par")
        throw UsageError("--engine: " + cfg.engine + " not in {seq,fair,par}");
    } else if (a == "--devices") {
      std::stringstream ss(val());
      std::string tok;
      while (std::getline(ss, tok, ',')) cfg.devices.push_back(static_cast<int>(num("--devices", tok.c_str(), 0, 1023)));
    } else if (!a.empty() && a[0] == '-') {
      throw UsageError("unknown option: " + a);
    } else if (cfg.instance.empty()) {
      cfg.instance = a;
    } else {
      throw UsageError("unexpected argument: " + a);
    }
  }
  if (cfg.instance.empty()) throw UsageError("file is required");
  if (!cfg.devices.empty() && cfg.cmd == "solve") {
    if (cfg.gpus != 1 && static_cast<int>(cfg.devices.size()) != cfg.gpus)
      throw UsageError("--devices lists " + std::to_string(cfg.devices.size()) + " devices for --gpus " +
                       std::to_string(cfg.gpus));
    cfg.gpus = static_cast<int>(cfg.devices.size());
  }
  return cfg;
}

}  // namespace

int main(int argc, char** argv) {
  Config cfg;
  try {
    cfg = parse_args(argc, argv);
  } catch (const UsageError& e) {
    std::cerr << "error: " << e.what() << "\n";
    usage(std::cerr);
    return 109;  // CLI11's exit code for argument errors (non-zero, distinct from 1 and 2)
  }
  try {
    if (cfg.cmd == "gen") {
      std::cout << patterson_text(random_patterson(static_cast<std::uint64_t>(cfg.gen[0]),
                                                   static_cast<int>(cfg.gen[1]), static_cast<int>(cfg.gen[2])));
      return 0;
    }
    return cfg.cmd == "solve" ? cmd_solve(cfg) : cmd_verify(cfg);
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
