// rcpsp.hpp — RCPSP front-end of the host model builder (configs 4 and 5).
// Restates rcpsp::build_model / check_solution (rcpsp.cpp:178-300) and the
// reference's instance generator random_patterson (tests/support/corpus.cpp:32-90),
// which defines the benchmark instances.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "model.hpp"

namespace pccp_b200 {

struct RcpspInstance {
  std::vector<std::int32_t> duration;            // per task, dummies included
  std::vector<std::vector<std::int32_t>> usage;  // [task][resource]
  std::vector<std::int32_t> capacity;            // per resource
  std::vector<std::pair<std::int32_t, std::int32_t>> precedences;  // i ends before j starts
  std::int32_t horizon = 0;

  std::size_t tasks() const { return duration.size(); }
  std::size_t resources() const { return capacity.size(); }
};

// Acyclicity and range checks (rcpsp::validate, rcpsp.cpp:60-92); throws ModelError.
void validate(const RcpspInstance& inst);

// random_patterson(mt19937_64(seed), n_real, resources).
RcpspInstance random_patterson(std::uint64_t seed, int n_real, int resources);

// Patterson text (rcpsp::parse_patterson, rcpsp.cpp:94-127); throws ModelError.
RcpspInstance parse_patterson(const std::string& text);

// JSON instance (rcpsp::parse_json_text, rcpsp.cpp:140-168): {"tasks": [{"duration": d,
// "usages": [...]}, ...], "capacities": [...], "precedences": [[i, j], ...],
// "horizon": h}; missing usages are 0, a missing horizon is the duration sum.
// Throws ModelError ("bad json instance: ...").
RcpspInstance parse_json(const std::string& text);

// Patterson text of an instance (the inverse of parse_patterson; the
// reference's testsupport::patterson_text, used for file round trips).
std::string patterson_text(const RcpspInstance& inst);

struct RcpspModel {
  std::unique_ptr<Model> model;
  std::vector<std::int32_t> starts;    // start slot per task
  std::vector<std::int32_t> overlaps;  // b[i*n+j]
};

// The decomposed cumulative model (rcpsp.cpp:178-273): starts in (0,h), 0/1
// overlap booleans, precedences, n^2 overlap reifications, one resource sum
// per (resource, task).  Objective: the sink's start; candidates: the starts.
RcpspModel build_rcpsp(const RcpspInstance& inst);

// Time-indexed validity of concrete starts (rcpsp.cpp:275-300).
bool check_solution(const RcpspInstance& inst, const std::vector<std::int32_t>& starts);

}  // namespace pccp_b200
