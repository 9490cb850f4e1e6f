// Rails config reader (SPEC.md:526 schema) -> RailSpec list.
#include <stdexcept>

#include "nezha/engine.hpp"
#include "nezha/util/toml.hpp"

namespace nezha {

std::vector<RailSpec> parseRailsToml(const std::string& text) {
  const auto root = toml::parse(text);
  std::vector<RailSpec> out;
  if (!root.contains("rail")) throw std::invalid_argument("rails config: no [[rail]] entries");
  int next_id = 0;
  for (const auto& r : root.at("rail").asArray()) {
    RailSpec s;
    s.rail_id = static_cast<int>(r.intOr("id", next_id));
    next_id = s.rail_id + 1;
    const std::string proto = r.stringOr("protocol", "tcp");
    const ProtocolKind pk = protocolKindFromString(proto);
    s.kind = pk == ProtocolKind::Sharp ? NZ_RAIL_NVLS : (pk == ProtocolKind::Glex ? NZ_RAIL_CE : NZ_RAIL_SM);
    s.sm_budget = static_cast<int>(r.intOr("sm_budget", 0));
    s.profile.rail_id = s.rail_id;
    s.profile.protocol = pk;
    s.profile.t_setup_us = r.doubleOr("t_setup_us", 0.0);
    s.profile.bandwidth_bps = r.doubleOr("bandwidth_bps", 0.0);
    if (r.contains("calibration")) {
      for (const auto& pt : r.at("calibration").asArray()) {
        const auto& a = pt.asArray();
        if (a.size() != 2) throw std::invalid_argument("rails config: calibration points are [size, latency_us]");
        s.profile.efficiency_points.emplace_back(static_cast<Bytes>(a[0].asInt()), a[1].asDouble());
      }
    }
    s.has_profile = s.profile.bandwidth_bps > 0;
    if (s.has_profile) s.profile.validate();
    out.push_back(s);
  }
  return out;
}

std::pair<std::uint64_t, std::uint64_t> choosePathCeilings(const std::vector<std::uint64_t>& sizes,
                                                           const std::vector<double>& times, std::uint64_t ll_cap,
                                                           std::uint64_t os_cap) {
  if (times.size() != 3 * sizes.size()) throw std::invalid_argument("choosePathCeilings: 3 times per size");
  auto best = [&](size_t k) {
    int b = 2;
    for (int v = 0; v < 2; ++v)
      if (times[k * 3 + v] < times[k * 3 + b]) b = v;
    return b;
  };
  std::uint64_t ll_max = 0, os_max = 0;
  size_t k = 0;
  if (ll_cap) {
    ll_max = sizes.empty() ? ll_cap : std::min<std::uint64_t>(ll_cap, sizes[0] / 2);
    for (; k < sizes.size() && best(k) == 0; ++k) ll_max = sizes[k];
    if (k == sizes.size()) ll_max = ll_cap;
  }
  if (os_cap) {
    os_max = ll_max;
    for (; k < sizes.size() && best(k) == 1; ++k) os_max = sizes[k];
    if (k == sizes.size()) os_max = std::max(os_max, os_cap);
  }
  return {ll_max, os_max};
}

}  // namespace nezha
