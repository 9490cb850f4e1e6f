// nz_planner_run_trace: the balancer + fault decisions driven by an injected
// scenario instead of a GPU. The engine runs the same
// Balancer / chooseHandoffTarget / orphanOf code on measured latencies; this
// entry point feeds it the scenario's latency model so its decision log can
// be diffed byte for byte against oracle/planner.py.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "nezha/balancer.hpp"
#include "nezha/collective.hpp"
#include "nezha/core/error.hpp"
#include "nezha/faults.hpp"
#include "nezha_b200.h"
#include "planner_trace.hpp"

namespace nezha {

namespace {

std::uint64_t splitmix(std::uint64_t& state) {
  std::uint64_t z = (state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

double unit01(std::uint64_t x) { return static_cast<double>(x >> 11) * (1.0 / 9007199254740992.0); }

}  // namespace

Scenario parseScenario(const std::string& text) {
  Scenario sc;
  std::istringstream in(text);
  std::string line;
  int lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    const auto hash = line.find('#');
    if (hash != std::string::npos) line.resize(hash);
    std::istringstream ls(line);
    std::string key;
    if (!(ls >> key)) continue;
    auto bad = [&](const std::string& why) {
      throw std::invalid_argument("scenario line " + std::to_string(lineno) + ": " + why);
    };
    if (key == "world") {
      if (!(ls >> sc.world) || sc.world < 1) bad("world");
    } else if (key == "algorithm") {
      std::string a;
      ls >> a;
      if (a == "ring")
        sc.algorithm = Algorithm::Ring;
      else if (a == "ring_chunked")
        sc.algorithm = Algorithm::RingChunked;
      else
        bad("algorithm");
    } else if (key == "config") {
      std::string k;
      double v;
      while (ls >> k >> v) {
        if (k == "tau") sc.cfg.tau = v;
        else if (k == "eta") sc.cfg.eta = v;
        else if (k == "eps") sc.cfg.convergence_eps = v;
        else if (k == "sync_us") sc.cfg.sync_overhead_us = v;
        else if (k == "window") sc.cfg.window = static_cast<int>(v);
        else if (k == "max_iters") sc.cfg.max_iters = static_cast<int>(v);
        else if (k == "demote_after") sc.cfg.demote_after = static_cast<int>(v);
        else bad("config key " + k);
      }
    } else if (key == "rail" || key == "concurrent") {
      RailProfile p;
      std::string proto;
      if (!(ls >> p.rail_id >> proto >> p.t_setup_us >> p.bandwidth_bps)) bad("rail");
      p.protocol = protocolKindFromString(proto);
      std::string tag;
      if (ls >> tag) {
        if (tag != "cal") bad("expected 'cal'");
        std::string pt;
        while (ls >> pt) {
          const auto colon = pt.find(':');
          if (colon == std::string::npos) bad("calibration point");
          p.efficiency_points.emplace_back(std::stoull(pt.substr(0, colon)), std::stod(pt.substr(colon + 1)));
        }
      }
      (key == "rail" ? sc.rails : sc.concurrent).push_back(p);
    } else if (key == "truth") {
      TruthLine t;
      if (!(ls >> t.rail_id >> t.a_us >> t.b_bps >> t.jitter)) bad("truth");
      sc.truth.push_back(t);
    } else if (key == "truth_sync") {
      if (!(ls >> sc.truth_sync_us)) bad("truth_sync");
    } else if (key == "seed") {
      if (!(ls >> sc.seed)) bad("seed");
    } else if (key == "ops") {
      std::uint64_t n, s;
      if (!(ls >> n >> s) || s == 0) bad("ops");
      for (std::uint64_t i = 0; i < n; ++i) sc.sizes.push_back(s);
    } else if (key == "ops_loguniform") {
      std::uint64_t n, lo, hi;
      if (!(ls >> n >> lo >> hi) || lo < 4 || hi < lo) bad("ops_loguniform");
      std::uint64_t st = sc.seed;
      const double l0 = std::log2(static_cast<double>(lo)), l1 = std::log2(static_cast<double>(hi));
      for (std::uint64_t i = 0; i < n; ++i) {
        const double x = l0 + unit01(splitmix(st)) * (l1 - l0);
        std::uint64_t s = static_cast<std::uint64_t>(std::floor(std::exp2(x))) & ~std::uint64_t{3};
        sc.sizes.push_back(s < 4 ? 4 : s);
      }
    } else if (key == "fail") {
      FaultLine f;
      if (!(ls >> f.op >> f.rail >> f.chunk)) bad("fail");
      sc.faults.push_back(f);
    } else if (key == "stall") {
      StallLine t;
      if (!(ls >> t.op >> t.rail >> t.chunk >> t.lag)) bad("stall");
      sc.stalls.push_back(t);
    } else if (key == "wave_bytes") {
      if (!(ls >> sc.wave_bytes) || sc.wave_bytes == 0) bad("wave_bytes");
    } else if (key == "readmit") {
      ReadmitLine r;
      if (!(ls >> r.op >> r.rail)) bad("readmit");
      sc.readmits.push_back(r);
    } else {
      bad("unknown key " + key);
    }
  }
  if (sc.rails.empty()) throw std::invalid_argument("scenario: no rails");
  return sc;
}

double truthLatency(const Scenario& sc, std::uint32_t op, int rail_id, Bytes len, bool multi) {
  for (const auto& t : sc.truth) {
    if (t.rail_id != rail_id) continue;
    std::uint64_t st = sc.seed ^ (static_cast<std::uint64_t>(op) * 0x9E3779B97F4A7C15ull) ^
                       (static_cast<std::uint64_t>(rail_id + 1) * 0xBF58476D1CE4E5B9ull);
    const double u = 2.0 * unit01(splitmix(st)) - 1.0;
    double us = t.a_us + static_cast<double>(len) / t.b_bps * 1e6;
    us = us * (1.0 + t.jitter * u);
    if (multi) us = us + sc.truth_sync_us;
    return us;
  }
  throw std::invalid_argument("scenario: no truth line for rail " + std::to_string(rail_id));
}

std::string planJson(std::uint32_t op, Bytes S, const Plan& p) {
  std::ostringstream o;
  o << "{\"op\":" << op << ",\"S\":" << S << ",\"bucket\":" << p.bucket << ",\"hot\":" << (p.hot ? "true" : "false")
    << ",\"rho\":" << formatDouble(p.rho) << ",\"gated\":" << (p.gated ? "true" : "false") << ",\"segs\":[";
  for (size_t i = 0; i < p.segments.size(); ++i) {
    const auto& s = p.segments[i];
    o << (i ? "," : "") << "[" << s.rail_id << "," << s.segment.offset << "," << s.segment.length << "]";
  }
  o << "]}";
  return o.str();
}

namespace {

void ticketJson(std::ostringstream& log, const std::optional<HandoffTicket>& ticket, bool unrecoverable) {
  if (ticket) {
    log << "{\"op_seq\":" << ticket->op_seq << ",\"offset\":" << ticket->orphan.offset
        << ",\"length\":" << ticket->orphan.length << ",\"source\":" << ticket->source_rail
        << ",\"target\":" << ticket->target_rail << "}";
  } else {
    log << "null";
  }
  if (unrecoverable) log << ",\"unrecoverable\":true";
}

// P9 over `healthy` for the orphan of `seg` from chunk k: nullopt ticket and
// unrecoverable = true when no survivor exists; nullopt, false when empty.
std::optional<HandoffTicket> handoff(const Plan& plan, std::uint32_t op, int rail, const Segment& seg, Bytes C,
                                     std::uint64_t k, const std::vector<int>& healthy, bool* unrecoverable) {
  *unrecoverable = false;
  const Segment orphan = orphanOf(seg, C, k);
  if (orphan.length == 0) return std::nullopt;
  const auto target = chooseHandoffTarget(plan, rail, healthy);
  if (!target) {
    *unrecoverable = true;
    return std::nullopt;
  }
  return HandoffTicket{op, orphan, rail, *target, 0};
}

}  // namespace

std::string runTrace(const std::string& text) {
  Scenario sc = parseScenario(text);
  Balancer bal(sc.rails, sc.cfg);
  if (!sc.concurrent.empty()) bal.setConcurrentProfiles(sc.concurrent);
  std::ostringstream log;
  std::vector<int> healthy;  // not failed by agreement (P9's survivors)
  for (const auto& r : bal.rails()) healthy.push_back(r.rail_id);
  std::vector<std::pair<std::uint32_t, int>> activations;  // (op, rail): the planner drops the rail there
  std::vector<int> dead;  // links dead on some rank: every launch on them fails at entry
  auto erase = [](std::vector<int>& v, int x) { v.erase(std::remove(v.begin(), v.end(), x), v.end()); };
  for (std::uint32_t op = 0; op < sc.sizes.size(); ++op) {
    for (const auto& r : sc.readmits) {
      if (r.op != op) continue;
      // A rail whose agreed drop has not reached the planner yet is still
      // planned: readmitting it only cancels the drop (as the engine does).
      const auto pending = std::find_if(activations.begin(), activations.end(),
                                        [&](const auto& a) { return a.second == r.rail; });
      if (pending == activations.end()) bal.readmit(r.rail);
      activations.erase(std::remove_if(activations.begin(), activations.end(),
                                       [&](const auto& a) { return a.second == r.rail; }),
                        activations.end());
      if (std::find(healthy.begin(), healthy.end(), r.rail) == healthy.end()) healthy.push_back(r.rail);
      std::sort(healthy.begin(), healthy.end());
      erase(dead, r.rail);
      log << "{\"readmit\":" << r.rail << ",\"op\":" << op << "}\n";
    }
    for (auto it = activations.begin(); it != activations.end();) {
      if (it->first > op) {
        ++it;
        continue;
      }
      if (bal.healthy(it->second)) bal.markFailed(it->second);
      log << "{\"dropped\":" << it->second << ",\"op\":" << op << "}\n";
      it = activations.erase(it);
    }
    const Bytes S = sc.sizes[op];
    Plan plan;
    try {
      plan = bal.allocate(S);
    } catch (const UnrecoverableError&) {
      log << "{\"op\":" << op << ",\"S\":" << S << ",\"unrecoverable\":true}\n";
      continue;
    }
    log << planJson(op, S, plan) << "\n";
    bool failed_this_op = false;
    for (const auto& f : sc.faults) {
      if (f.op != op) continue;
      failed_this_op = true;
      log << "{\"fail\":{\"op\":" << op << ",\"rail\":" << f.rail << ",\"chunk\":" << f.chunk << "},\"ticket\":";
      const Segment* seg = nullptr;
      for (const auto& rs : plan.segments)
        if (rs.rail_id == f.rail) seg = &rs.segment;
      std::optional<HandoffTicket> ticket;
      bool unrecoverable = false;
      if (seg) {
        const Bytes C = defaultChunkBytes(seg->length, sc.world, sc.algorithm);
        ticket = handoff(plan, op, f.rail, *seg, C, f.chunk, healthy, &unrecoverable);
      }
      ticketJson(log, ticket, unrecoverable);
      log << "}\n";
      erase(healthy, f.rail);
      bal.markFailed(f.rail);
    }
    // Launches on a dead link fail at entry on every rank: the monitor
    // reroutes the whole segment (no chunk completed).
    for (const auto& rs : plan.segments) {
      if (std::find(dead.begin(), dead.end(), rs.rail_id) == dead.end()) continue;
      failed_this_op = true;
      const Bytes C = defaultChunkBytes(rs.segment.length, sc.world, sc.algorithm);
      bool unrecoverable = false;
      const auto ticket = handoff(plan, op, rs.rail_id, rs.segment, C, 0, healthy, &unrecoverable);
      log << "{\"lost\":{\"op\":" << op << ",\"rail\":" << rs.rail_id << "},\"ticket\":";
      ticketJson(log, ticket, unrecoverable);
      log << "}\n";
    }
    for (const auto& t : sc.stalls) {
      if (t.op != op) continue;
      const Segment* seg = nullptr;
      for (const auto& rs : plan.segments)
        if (rs.rail_id == t.rail) seg = &rs.segment;
      const bool already = std::find(dead.begin(), dead.end(), t.rail) != dead.end();
      log << "{\"stall\":{\"op\":" << op << ",\"rail\":" << t.rail << ",\"chunk\":" << t.chunk << "}";
      if (!seg || already) {  // the link died where this op never touched it
        log << ",\"fired\":false}\n";
        continue;
      }
      const Bytes C = defaultChunkBytes(seg->length, sc.world, sc.algorithm);
      const std::uint64_t nch = (seg->length + C - 1) / C;
      const std::uint64_t k = completedBeforeStall(C, 0, nch, t.chunk, sc.wave_bytes);
      if (k >= nch) {
        log << ",\"fired\":false}\n";
        continue;
      }
      failed_this_op = true;
      erase(healthy, t.rail);
      dead.push_back(t.rail);
      const std::uint32_t activation = op + 1 + t.lag;
      activations.emplace_back(activation, t.rail);
      bool unrecoverable = false;
      const auto ticket = handoff(plan, op, t.rail, *seg, C, k, healthy, &unrecoverable);
      log << ",\"fired\":true,\"orphan_chunk\":" << k << ",\"activation\":" << activation << ",\"ticket\":";
      ticketJson(log, ticket, unrecoverable);
      log << "}\n";
    }
    if (failed_this_op) continue;  // an op that lost a rail is not a Timer sample
    std::vector<std::pair<int, Micros>> lat;
    const bool multi = plan.segments.size() > 1;
    for (const auto& rs : plan.segments) lat.emplace_back(rs.rail_id, truthLatency(sc, op, rs.rail_id, rs.segment.length, multi));
    auto fe = bal.recordOp(plan, lat);
    if (fe) {
      const auto& e = bal.table().buckets.at(fe->bucket);
      log << "{\"flush\":" << fe->bucket << ",\"op\":" << op << ",\"means\":[";
      for (size_t i = 0; i < fe->means.size(); ++i)
        log << (i ? "," : "") << "[" << fe->means[i].first << "," << formatDouble(fe->means[i].second) << "]";
      log << "],\"epoch\":" << bal.table().epoch << ",\"threshold\":";
      if (bal.table().threshold == kNoThreshold)
        log << "null";
      else
        log << bal.table().threshold;
      log << ",\"alpha\":[";
      for (size_t i = 0; i < e.alpha.size(); ++i) log << (i ? "," : "") << formatDouble(e.alpha[i]);
      log << "],\"hot\":" << (e.hot ? "true" : "false") << ",\"iters\":" << e.iters
          << ",\"converged\":" << (e.converged ? "true" : "false") << ",\"demoted\":" << (e.demoted ? "true" : "false")
          << "}\n";
    }
  }
  log << bal.tableJson() << "\n";
  return log.str();
}

}  // namespace nezha

extern "C" int nz_planner_run_trace(const char* scenario, char* out, size_t cap) {
  if (!scenario || !out) return NZ_ERR_INVALID;
  std::string s;
  try {
    s = nezha::runTrace(scenario);
  } catch (const std::invalid_argument& e) {
    nezha::setPlannerError(e.what());
    return NZ_ERR_INVALID;
  } catch (const std::exception& e) {
    nezha::setPlannerError(e.what());
    return NZ_ERR_SYSTEM;
  }
  if (s.size() + 1 > cap) return NZ_ERR_BUFFER;
  std::memcpy(out, s.c_str(), s.size() + 1);
  return NZ_OK;
}
