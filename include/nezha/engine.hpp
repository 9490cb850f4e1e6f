// nezha/engine.hpp — the engine-level multi-rail allreduce (SPEC.md:226,
// :353, :416; Fig. 6 flow), B200 edition.
//
// One Engine per rank process. allreduce():
//   split_oversized -> Balancer::allocate -> one CUDA stream per rail forks
//   from the caller's stream -> the rails' sm_100a kernels / DMA run on
//   disjoint segments -> join back into the caller's stream -> Timer.
// The Timer samples op k at op k + kTimerLag (deterministic on every rank)
// and a flush agrees on the per-rail means across ranks (max over ranks)
// before the balancer moves, so all ranks keep identical tables.
// A rail failure (device fault record) is handled inline: health -> Failed,
// HandoffTicket to argmax data_length, the orphan chunks run on the target
// rail's stream after its current task, with the failed rail's geometry.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "nezha/balancer.hpp"
#include "nezha/collective.hpp"
#include "nezha/faults.hpp"
#include "nezha_b200.h"

namespace nezha {

struct RailSpec {
  int rail_id = 0;
  int kind = NZ_RAIL_SM;  // nz_rail_kind_t
  int sm_budget = 0;
  RailProfile profile;
  bool has_profile = false;
};

// Rails config: [[rail]] protocol / t_setup_us / bandwidth_bps /
// calibration = [[size, latency_us], ...] / sm_budget. protocol maps
// sharp|nvls -> NVLS, glex|ce -> CE, tcp|sm -> SM.
std::vector<RailSpec> parseRailsToml(const std::string& text);

// Protocol ceilings of one rail from a startup sweep (engine tunePaths):
// times[3k + v] is the (rank-agreed) time of path v at sizes[k] (v = 0 LL,
// 1 staged one-shot, 2 two-shot; >= 1e30 = not applicable), sizes ascending.
// LL keeps the contiguous run of sizes it won from the smallest (its full
// capacity if it won all, half the smallest size if it won none); one-shot
// the run right after it. Returns {ll_max, oneshot_max}.
std::pair<std::uint64_t, std::uint64_t> choosePathCeilings(const std::vector<std::uint64_t>& sizes,
                                                           const std::vector<double>& times, std::uint64_t ll_cap,
                                                           std::uint64_t os_cap);

}  // namespace nezha
