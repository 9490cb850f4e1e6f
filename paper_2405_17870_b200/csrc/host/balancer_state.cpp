// AllocationTable persistence for warm restarts.
#include <sstream>
#include <stdexcept>

#include "json.hpp"
#include "nezha/balancer.hpp"

namespace nezha {

namespace {

void writeProfile(std::ostringstream& o, const RailProfile& p) {
  o << "{\"rail_id\":" << p.rail_id << ",\"t_setup_us\":" << formatDouble(p.t_setup_us)
    << ",\"bandwidth_bps\":" << formatDouble(p.bandwidth_bps) << ",\"calibration\":[";
  for (size_t j = 0; j < p.efficiency_points.size(); ++j) {
    o << (j ? "," : "") << "[" << p.efficiency_points[j].first << "," << formatDouble(p.efficiency_points[j].second)
      << "]";
  }
  o << "]}";
}

RailProfile readProfile(const toml::Value& v, const RailProfile& like) {
  RailProfile p = like;
  p.rail_id = static_cast<int>(v.at("rail_id").asInt());
  p.t_setup_us = v.at("t_setup_us").asDouble();
  p.bandwidth_bps = v.at("bandwidth_bps").asDouble();
  p.efficiency_points.clear();
  for (const auto& pt : v.at("calibration").asArray()) {
    const auto& a = pt.asArray();
    p.efficiency_points.emplace_back(static_cast<Bytes>(a.at(0).asInt()), a.at(1).asDouble());
  }
  p.validate();
  return p;
}

}  // namespace

std::string Balancer::saveState() const {
  std::ostringstream o;
  o << "{\"version\":1,\"sync_overhead_us\":" << formatDouble(cfg_.sync_overhead_us) << ",\"profiles\":[";
  for (size_t i = 0; i < rails_.size(); ++i) {
    o << (i ? "," : "");
    writeProfile(o, rails_[i]);
  }
  o << "],\"concurrent\":[";
  for (size_t i = 0; i < concurrent_.size(); ++i) {
    o << (i ? "," : "");
    writeProfile(o, concurrent_[i]);
  }
  o << "],\"buckets\":{";
  bool first = true;
  for (const auto& [k, e] : table_.buckets) {
    if (!e.measured && !e.demoted) continue;
    o << (first ? "" : ",") << "\"" << k << "\":{\"alpha\":[";
    for (size_t i = 0; i < e.alpha.size(); ++i) o << (i ? "," : "") << formatDouble(e.alpha[i]);
    o << "],\"measured\":" << (e.measured ? "true" : "false") << ",\"iters\":" << e.iters
      << ",\"converged\":" << (e.converged ? "true" : "false") << ",\"demoted\":" << (e.demoted ? "true" : "false")
      << "}";
    first = false;
  }
  o << "}}";
  return o.str();
}

void Balancer::loadState(const std::string& text) {
  const toml::Value root = json::parse(text);
  if (root.intOr("version", 0) != 1) throw std::invalid_argument("balancer state: unsupported version");
  std::vector<RailProfile> prof;
  for (const auto& v : root.at("profiles").asArray()) prof.push_back(readProfile(v, rails_[railIndex(static_cast<int>(v.at("rail_id").asInt()))]));
  if (prof.size() != rails_.size()) throw std::invalid_argument("balancer state: rail count differs");
  std::vector<RailProfile> conc;
  if (root.contains("concurrent")) {
    for (const auto& v : root.at("concurrent").asArray())
      conc.push_back(readProfile(v, rails_[railIndex(static_cast<int>(v.at("rail_id").asInt()))]));
  }
  rails_ = prof;
  concurrent_ = conc;
  ++profile_version_;
  cfg_.sync_overhead_us = root.doubleOr("sync_overhead_us", cfg_.sync_overhead_us);
  for (auto& [k, e] : table_.buckets) {
    e.measured = false;
    e.demoted = false;
    e.iters = 0;
    e.converged = false;
  }
  if (root.contains("buckets")) {
    for (const auto& [key, v] : root.at("buckets").asTable()) {
      const int k = std::stoi(key);
      if (k < kMinBucket || k > kMaxBucket) throw std::invalid_argument("balancer state: bucket out of range");
      BucketEntry& e = table_.buckets[k];
      e.alpha.assign(rails_.size(), 0.0);
      const auto& a = v.at("alpha").asArray();
      if (a.size() != rails_.size()) throw std::invalid_argument("balancer state: alpha size differs");
      for (size_t i = 0; i < a.size(); ++i) e.alpha[i] = a[i].asDouble();
      e.measured = v.boolOr("measured", false);
      e.iters = static_cast<int>(v.intOr("iters", 0));
      e.converged = v.boolOr("converged", false);
      e.demoted = v.boolOr("demoted", false);
    }
  }
  windows_.clear();
  rebuild();
}

}  // namespace nezha
