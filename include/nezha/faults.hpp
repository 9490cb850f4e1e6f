// nezha/faults.hpp — exception handler: health states and segment handoff
// (PAPER.md:455-463).
//
// On B200 a rail failure is reported by the device (a fault record posted by
// the rail's kernel into mapped host memory) instead of a TCP
// channel-down; the monitor thread spins on those records, so detection is
// microseconds rather than the SPEC's 3 x 50 ms heartbeat budget. The
// heartbeat state machine is kept for rails that merely stall.
#pragma once

#include <cstdint>
#include <optional>
#include <vector>

#include "nezha/balancer.hpp"
#include "nezha/core/types.hpp"

namespace nezha {

enum class HealthStatus : std::uint8_t { Healthy = 0, Suspect = 1, Failed = 2 };
const char* toString(HealthStatus s);

/// SPEC.md:370-373, per rail.
struct HealthState {
  int rail_id = 0;
  HealthStatus status = HealthStatus::Healthy;
  double last_heartbeat_us = 0;
  std::uint32_t failure_epoch = 0;
};

/// SPEC.md:374-377.
struct HandoffTicket {
  std::uint32_t op_seq = 0;
  Segment orphan;
  int source_rail = 0;
  int target_rail = 0;
  double issued_us = 0;
  bool operator==(const HandoffTicket&) const = default;
};

/// heartbeats every `interval_us`; `suspect_after` missed
/// beats -> Suspect, `fail_after` -> Failed; channel-down -> Failed at once.
/// Failed is sticky until readmit.
class HealthMonitor {
 public:
  HealthMonitor(std::vector<int> rail_ids, double interval_us = 50'000, int suspect_after = 2, int fail_after = 3);

  void heartbeat(int rail_id, double now_us);
  // Re-evaluates missed beats; returns the rails whose status changed.
  std::vector<int> tick(double now_us);
  void channelDown(int rail_id);
  // only a Failed rail that has been beating for >= hold_us.
  void readmit(int rail_id, double now_us, double hold_us = 1'000'000);

  const HealthState& state(int rail_id) const;
  std::vector<int> healthyRails() const;

 private:
  HealthState& find(int rail_id);
  std::vector<HealthState> states_;
  std::vector<double> healthy_since_;
  double interval_us_;
  int suspect_after_;
  int fail_after_;
};

// P9: the survivor with the largest current data_length in this op's plan
// (ties -> lowest rail_id; rails absent from the plan count 0). nullopt when
// no healthy rail other than `failed_rail` exists.
std::optional<int> chooseHandoffTarget(const Plan& plan, int failed_rail, const std::vector<int>& healthy_rails);

// P10: the orphan of a failure at chunk k of `seg` under chunk size C:
// [seg.offset + k*C, seg.end()); empty when k >= number of chunks.
Segment orphanOf(const Segment& seg, Bytes chunk_bytes, std::uint64_t chunk_k);

}  // namespace nezha
