// Core value types and cost model (reference proj/src/core/types.cpp:9-108,
// proj/src/core/math.cpp:7-35). Compiled with -ffp-contract=off so every
// double below rounds exactly as the oracle's restatement does.
#include <algorithm>
#include <stdexcept>
#include <string>

#include "nezha/core/math.hpp"
#include "nezha/core/types.hpp"

namespace nezha {

namespace {
struct KindName {
  ProtocolKind kind;
  const char* name;
};
// Canonical names first (toString uses them), then the B200 rail aliases.
constexpr KindName kKindNames[] = {
    {ProtocolKind::Tcp, "tcp"},     {ProtocolKind::Sharp, "sharp"}, {ProtocolKind::Glex, "glex"},
    {ProtocolKind::Custom, "custom"}, {ProtocolKind::Sharp, "nvls"},  {ProtocolKind::Glex, "ce"},
    {ProtocolKind::Tcp, "sm"},
};

[[noreturn]] void badRail(int id, const char* what) {
  throw std::invalid_argument("rail " + std::to_string(id) + ": " + what);
}
}  // namespace

const char* toString(ProtocolKind kind) {
  for (const auto& kn : kKindNames) {
    if (kn.kind == kind) return kn.name;
  }
  return "unknown";
}

ProtocolKind protocolKindFromString(const std::string& name) {
  for (const auto& kn : kKindNames) {
    if (name == kn.name) return kn.kind;
  }
  throw std::invalid_argument("unknown protocol kind: " + name);
}

void RailProfile::validate() const {
  if (!(t_setup_us >= 0)) badRail(rail_id, "t_setup must be >= 0");
  if (!(bandwidth_bps > 0)) badRail(rail_id, "bandwidth must be > 0");
  if (max_frame_payload == 0) badRail(rail_id, "max_frame_payload must be > 0");
  const auto& pts = efficiency_points;
  for (size_t i = 1; i < pts.size(); ++i) {
    const bool size_up = pts[i].first > pts[i - 1].first;
    const bool lat_up = pts[i].second > pts[i - 1].second;
    if (!size_up || !lat_up) {
      badRail(rail_id, "efficiency_points must be strictly increasing in size and latency");
    }
  }
}

Micros RailProfile::parametricLatency(Bytes size) const {
  return t_setup_us + static_cast<double>(size) / bandwidth_bps * 1e6;
}

Micros RailProfile::messageLatency(Bytes size) const {
  const auto& pts = efficiency_points;
  if (pts.empty()) return parametricLatency(size);
  if (pts.size() == 1 || size <= pts.front().first) return pts.front().second;
  // First sample at or above `size` (or the last one when extrapolating).
  size_t hi = 1;
  while (hi + 1 < pts.size() && pts[hi].first < size) ++hi;
  const double x0 = static_cast<double>(pts[hi - 1].first);
  const double x1 = static_cast<double>(pts[hi].first);
  const double frac = (static_cast<double>(size) - x0) / (x1 - x0);
  return pts[hi - 1].second + frac * (pts[hi].second - pts[hi - 1].second);
}

bool segmentsCoverExactly(std::vector<Segment> segments, Bytes total) {
  std::sort(segments.begin(), segments.end(),
            [](const Segment& a, const Segment& b) { return a.offset < b.offset; });
  Bytes next = 0;
  for (const auto& s : segments) {
    if (s.offset != next) return false;
    next += s.length;
  }
  return next == total;
}

int bucketOf(Bytes size) {
  if (size == 0) throw std::invalid_argument("bucketOf: size must be positive");
  return 63 - __builtin_clzll(size);
}

Bytes bucketFloor(int bucket) {
  if (bucket < 0 || bucket > 63) throw std::invalid_argument("bucketFloor: bucket out of range");
  return Bytes{1} << bucket;
}

Bytes ringVolume(int node_count, Bytes payload) {
  if (node_count < 2) throw std::invalid_argument("ringVolume: node_count must be >= 2");
  // 2(N-1)M/N with round-half-up, exact in 128-bit integers.
  using u128 = unsigned __int128;
  const u128 n = static_cast<u128>(node_count);
  const u128 num = u128{2} * (n - 1) * payload;
  return static_cast<Bytes>((num + n / 2) / n);
}

double networkEfficiency(const RailProfile& profile, Bytes payload) {
  if (payload == 0) throw std::invalid_argument("networkEfficiency: payload must be positive");
  const double transfer_us = static_cast<double>(payload) / profile.bandwidth_bps * 1e6;
  return 1.0 / (1.0 + profile.t_setup_us / transfer_us);
}

double realTimeThroughput(const RailProfile& profile, Bytes payload) {
  if (payload == 0) return 0.0;
  const Micros t = profile.messageLatency(payload);
  if (t <= 0) return 0.0;
  return static_cast<double>(payload) / (t * 1e-6);
}

}  // namespace nezha
