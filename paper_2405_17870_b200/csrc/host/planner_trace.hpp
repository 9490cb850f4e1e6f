// Scenario model of nz_planner_run_trace.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "nezha/balancer.hpp"
#include "nezha/collective.hpp"

namespace nz {
void setLastError(const std::string& msg);  // comm.cpp: backs nz_last_error()
}

namespace nezha {

struct TruthLine {
  int rail_id = 0;
  double a_us = 0;
  double b_bps = 1;
  double jitter = 0;
};

struct FaultLine {
  std::uint32_t op = 0;
  int rail = 0;
  std::uint64_t chunk = 0;
};

// Unplanned failure: one rank's link of `rail` dies at
// `chunk` of op `op`; the monitors agree and the planner stops using the rail
// from op `op + 1 + lag` (lag = ops issued before the agreement landed).
struct StallLine {
  std::uint32_t op = 0;
  int rail = 0;
  std::uint64_t chunk = 0;
  std::uint32_t lag = 0;
};

struct ReadmitLine {
  std::uint32_t op = 0;
  int rail = 0;
};

struct Scenario {
  int world = 8;
  Algorithm algorithm = Algorithm::RingChunked;
  BalancerConfig cfg;
  std::vector<RailProfile> rails;
  std::vector<RailProfile> concurrent;  // optional P13 profiles ("concurrent" lines)
  std::vector<TruthLine> truth;
  double truth_sync_us = 0;
  std::uint64_t seed = 0;
  std::vector<std::uint64_t> sizes;
  std::vector<FaultLine> faults;
  std::vector<StallLine> stalls;
  std::vector<ReadmitLine> readmits;
  Bytes wave_bytes = kDefaultWaveBytes;
};

Scenario parseScenario(const std::string& text);
double truthLatency(const Scenario& sc, std::uint32_t op, int rail_id, Bytes len, bool multi);
std::string planJson(std::uint32_t op, Bytes S, const Plan& p);
std::string runTrace(const std::string& text);

inline void setPlannerError(const std::string& msg) { nz::setLastError(msg); }

}  // namespace nezha
