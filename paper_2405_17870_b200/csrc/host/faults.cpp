// Health monitor and handoff rules (P9/P10).
#include "nezha/faults.hpp"

#include <algorithm>
#include <stdexcept>

namespace nezha {

const char* toString(HealthStatus s) {
  switch (s) {
    case HealthStatus::Healthy:
      return "healthy";
    case HealthStatus::Suspect:
      return "suspect";
    case HealthStatus::Failed:
      return "failed";
  }
  return "unknown";
}

HealthMonitor::HealthMonitor(std::vector<int> rail_ids, double interval_us, int suspect_after, int fail_after)
    : interval_us_(interval_us), suspect_after_(suspect_after), fail_after_(fail_after) {
  if (!(interval_us > 0) || suspect_after < 1 || fail_after <= suspect_after) {
    throw std::invalid_argument("HealthMonitor: bad heartbeat parameters");
  }
  std::sort(rail_ids.begin(), rail_ids.end());
  for (int id : rail_ids) states_.push_back(HealthState{id, HealthStatus::Healthy, 0, 0});
  healthy_since_.assign(states_.size(), -1.0);  // -1: no heartbeat streak yet
}

HealthState& HealthMonitor::find(int rail_id) {
  for (auto& s : states_)
    if (s.rail_id == rail_id) return s;
  throw std::invalid_argument("unknown rail " + std::to_string(rail_id));
}

const HealthState& HealthMonitor::state(int rail_id) const {
  return const_cast<HealthMonitor*>(this)->find(rail_id);
}

void HealthMonitor::heartbeat(int rail_id, double now_us) {
  HealthState& s = find(rail_id);
  const size_t i = &s - states_.data();
  if (healthy_since_[i] < 0) healthy_since_[i] = now_us;  // streak starts at the first beat
  s.last_heartbeat_us = now_us;
  if (s.status == HealthStatus::Suspect) s.status = HealthStatus::Healthy;  // Suspect -> Healthy
}

std::vector<int> HealthMonitor::tick(double now_us) {
  std::vector<int> changed;
  for (size_t i = 0; i < states_.size(); ++i) {
    HealthState& s = states_[i];
    if (s.status == HealthStatus::Failed) continue;
    const double missed = (now_us - s.last_heartbeat_us) / interval_us_;
    HealthStatus next = s.status;
    if (missed >= fail_after_ && s.status == HealthStatus::Suspect)
      next = HealthStatus::Failed;
    else if (missed >= suspect_after_ && s.status == HealthStatus::Healthy)
      next = HealthStatus::Suspect;
    if (next != s.status) {
      s.status = next;
      if (next == HealthStatus::Failed) {
        ++s.failure_epoch;
        healthy_since_[i] = -1.0;
      }
      changed.push_back(s.rail_id);
    }
  }
  return changed;
}

void HealthMonitor::channelDown(int rail_id) {
  HealthState& s = find(rail_id);
  if (s.status == HealthStatus::Failed) return;
  s.status = HealthStatus::Failed;
  ++s.failure_epoch;
  healthy_since_[&s - states_.data()] = -1.0;
}

void HealthMonitor::readmit(int rail_id, double now_us, double hold_us) {
  HealthState& s = find(rail_id);
  const size_t i = &s - states_.data();
  if (s.status != HealthStatus::Failed) throw std::invalid_argument("readmit: rail is not failed");
  if (healthy_since_[i] < 0 || now_us - healthy_since_[i] < hold_us) {
    throw std::invalid_argument("readmit: rail has not been healthy long enough");
  }
  s.status = HealthStatus::Healthy;
}

std::vector<int> HealthMonitor::healthyRails() const {
  std::vector<int> out;
  for (const auto& s : states_)
    if (s.status != HealthStatus::Failed) out.push_back(s.rail_id);
  return out;
}

std::optional<int> chooseHandoffTarget(const Plan& plan, int failed_rail, const std::vector<int>& healthy_rails) {
  std::vector<int> cand;
  for (int r : healthy_rails)
    if (r != failed_rail) cand.push_back(r);
  if (cand.empty()) return std::nullopt;
  std::sort(cand.begin(), cand.end());
  int best = cand[0];
  Bytes best_len = 0;
  bool first = true;
  for (int r : cand) {
    Bytes len = 0;
    for (const auto& rs : plan.segments)
      if (rs.rail_id == r) len += rs.segment.length;
    if (first || len > best_len) {
      best = r;
      best_len = len;
      first = false;
    }
  }
  return best;
}

Segment orphanOf(const Segment& seg, Bytes chunk_bytes, std::uint64_t chunk_k) {
  if (chunk_bytes == 0) throw std::invalid_argument("orphanOf: chunk_bytes must be positive");
  const Bytes begin = chunk_k * chunk_bytes;
  if (begin >= seg.length) return Segment{seg.end(), 0};
  return Segment{seg.offset + begin, seg.length - begin};
}

}  // namespace nezha
