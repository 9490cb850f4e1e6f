// Engine: the multi-rail allreduce of one rank (
// PAPER.md:379 Fig. 6). Planner (Balancer) + rails (rails.cu) + Timer +
// fault monitor / handoff. See include/nezha/engine.hpp for the contract;
// startup calibration lives in engine_calibrate.cpp.
#include "engine_impl.h"

using nz::fail;
using nz::guarded;

std::vector<std::pair<int, nezha::Micros>> nz_engine::agree(const std::vector<std::pair<int, nezha::Micros>>& mine) {
  if (comm->world == 1) return mine;
  std::vector<double> v(specs.size(), -1.0);
  for (auto& [id, m] : mine) v[index(id)] = m;
  std::vector<double> all(v.size() * comm->world);
  const auto msgs = nz::exchange(comm, v.data(), v.size() * sizeof(double), {});
  for (int r = 0; r < comm->world; ++r) std::memcpy(all.data() + r * v.size(), msgs[r].data.data(), v.size() * sizeof(double));
  std::vector<std::pair<int, nezha::Micros>> out;
  for (size_t i = 0; i < v.size(); ++i) {
    double m = -1.0;
    for (int r = 0; r < comm->world; ++r) m = std::max(m, all[r * v.size() + i]);
    if (m >= 0) out.emplace_back(specs[i].rail_id, m);
  }
  return out;
}

void nz_engine::harvest(uint32_t upto) {
  while (!pending.empty() && pending.front().op + static_cast<uint32_t>(cfg.timer_lag) <= upto) {
    Pending p = std::move(pending.front());
    pending.pop_front();
    std::vector<std::pair<int, nezha::Micros>> lat;
    for (auto& [id, e] : p.ends) {
      NZ_CUDA(cudaEventSynchronize(e));
      float ms = 0;
      NZ_CUDA(cudaEventElapsedTime(&ms, p.start, e));
      bool found = false;
      for (auto& pr : lat)
        if (pr.first == id) {
          pr.second = std::max(pr.second, static_cast<double>(ms) * 1000.0);
          found = true;
        }
      if (!found) lat.emplace_back(id, static_cast<double>(ms) * 1000.0);
      pool.push_back(e);
    }
    pool.push_back(p.start);
    if (stats.size() != specs.size()) stats.assign(specs.size(), RailStat{});
    for (auto& [id, us] : lat) {
      RailStat& st = stats[index(id)];
      st.ops += 1;
      st.us += us;
      for (const auto& rs : p.plan.segments)
        if (rs.rail_id == id) st.bytes += rs.segment.length;
    }
    if (!p.skip) bal->recordOp(p.plan, lat);
  }
}

void nz_engine::finishFailoverReport() {
  if (!fo_pending) return;
  volatile uint64_t* s = stamps_host;
  if (s[2] == 0) return;
  const double f = static_cast<double>(s[3]);
  fo.detect_us = (static_cast<double>(s[0]) - f) / 1000.0;
  fo.resume_us = (static_cast<double>(s[1]) - f) / 1000.0;
  fo.done_us = (static_cast<double>(s[2]) - f) / 1000.0;
  fo.host_detect_us = (static_cast<double>(host_seen_ns + clock_offset_ns) - f) / 1000.0;
  have_fo = true;
  fo_pending = false;
}

std::vector<nz::ComputeGate> nz_engine::gatesFor(const std::vector<std::pair<int, uint64_t>>& segs, std::string* log) {
  std::vector<nz::ComputeGate> gates(segs.size());
  if (pool_mode == nezha::PoolMode::Off || segs.size() < 2) return gates;
  std::vector<std::pair<int, int>> demands;
  for (const auto& [rid, len] : segs) demands.emplace_back(rid, nz::railComputeCtas(rails[index(rid)], len));
  const auto grants = nezha::planComputeGrants(*cpool, pool_mode, demands);
  std::map<int, cudaEvent_t> released;
  pool_stats.ops += 1;
  std::ostringstream o;
  for (size_t i = 0; i < grants.size(); ++i) {
    const auto& g = grants[i];
    gates[i].max_ctas = g.grant;
    for (int w : g.waits) gates[i].waits.push_back(released.at(w));
    gates[i].release = event();
    released[g.rail_id] = gates[i].release;
    pool_pending.push_back(gates[i].release);
    pool_stats.waits += g.waits.empty() ? 0 : 1;
    pool_stats.shrunk += g.grant < g.demand ? 1 : 0;
    o << (i ? "," : "") << "[" << g.rail_id << "," << g.demand << "," << g.grant << ",[";
    for (size_t j = 0; j < g.waits.size(); ++j) o << (j ? "," : "") << g.waits[j];
    o << "]]";
  }
  if (log) *log = o.str();
  return gates;
}

void nz_engine::recycleGates() {
  for (auto e : pool_pending) pool.push_back(e);
  pool_pending.clear();
}

void nz_engine::op(nz_buf* in, nz_buf* out, uint64_t base, uint64_t len, int dtype, cudaStream_t user) {
  const uint32_t seq = op_seq++;
  // Inside a CUDA graph capture (graph-safe rails only) nothing may wait on
  // the device: no Timer harvest, no Timer sample, no failure injection.
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  NZ_CUDA(cudaStreamIsCapturing(user, &cap));
  const bool capturing = cap != cudaStreamCaptureStatusNone;
  if (capturing) {
    if (!cfg.graph_safe) fail(NZ_ERR_INVALID, "graph capture needs an engine created with graph_safe = 1");
    if (inject.count(seq)) fail(NZ_ERR_INVALID, "failure injection inside a graph capture");
  } else {
    harvest(seq);
  }
  nezha::Plan plan = bal->allocate(len);
  const int world = comm->world;
  if (!plan.hot && inject.find(seq) == inject.end()) {
    // Cold (or rho-gated) op: one rail, launched straight on the caller's
    // stream — no fork/join, no Timer events. A single-rail sample cannot
    // move the table (a cold flush only records telemetry), so skipping it
    // leaves every decision unchanged (P11).
    const auto& rs = plan.segments[0];
    nz_rail* r = rails[index(rs.rail_id)];
    const uint64_t C = nezha::defaultChunkBytes(rs.segment.length, world, algo);
    nz::railAllreduce(r, in, out, base + rs.segment.offset, rs.segment.length, C, 0, UINT64_MAX, dtype, seq, -1,
                      user);
    recordPlan(seq, base, len, std::move(plan));
    return;
  }
  Pending p;
  p.op = seq;
  p.plan = plan;
  p.start = event();
  NZ_CUDA(cudaEventRecord(p.start, user));
  auto inj = inject.find(seq);
  const nezha::Segment* failed_seg = nullptr;
  int failed_rail = -1;
  uint64_t failed_chunk = 0;
  std::vector<std::pair<int, uint64_t>> segs;
  for (const auto& rs : plan.segments) segs.emplace_back(rs.rail_id, rs.segment.length);
  std::string grant_log;
  auto gates = gatesFor(segs, &grant_log);
  for (size_t si = 0; si < plan.segments.size(); ++si) {
    const auto& rs = plan.segments[si];
    nz_rail* r = rails[index(rs.rail_id)];
    NZ_CUDA(cudaStreamWaitEvent(r->stream, p.start, 0));
    const uint64_t C = nezha::defaultChunkBytes(rs.segment.length, world, algo);
    int64_t fail_chunk = -1;
    if (inj != inject.end() && inj->second.first == rs.rail_id) {
      fail_chunk = static_cast<int64_t>(inj->second.second);
      const uint64_t nch = (rs.segment.length + C - 1) / C;
      if (inj->second.second < nch) {
        failed_seg = &rs.segment;
        failed_rail = rs.rail_id;
        failed_chunk = inj->second.second;
      }
    }
    nz::railAllreduce(r, in, out, base + rs.segment.offset, rs.segment.length, C, 0, UINT64_MAX, dtype, seq,
                      fail_chunk, r->stream, &gates[si]);
    cudaEvent_t e = event();
    NZ_CUDA(cudaEventRecord(e, r->stream));
    p.ends.emplace_back(rs.rail_id, e);
  }
  if (inj != inject.end()) {
    const int rid = inj->second.first;
    inject.erase(inj);
    p.skip = true;
    if (failed_seg) {
      handoff(p, plan, *failed_seg, failed_rail, failed_chunk, in, out, base, dtype);
    } else if (health->state(rid).status != nezha::HealthStatus::Failed) {
      // Idle failure: the rail carried nothing at / after that chunk.
      health->channelDown(rid);
      bal->markFailed(rid);
    }
  }
  for (auto& [id, e] : p.ends) NZ_CUDA(cudaStreamWaitEvent(user, e, 0));
  recycleGates();
  if (capturing) {  // the captured records become graph edges: the events are free again
    for (auto& [id, e] : p.ends) pool.push_back(e);
    pool.push_back(p.start);
  } else {
    pending.push_back(std::move(p));
  }
  recordPlan(seq, base, len, std::move(plan), std::move(grant_log));
}

void nz_engine::recordPlan(uint32_t seq, uint64_t base, uint64_t len, nezha::Plan&& plan, std::string&& grants) {
  last_plans.push_back(PlanRecord{seq, base, len, std::move(plan), std::move(grants)});
}

std::string nz_engine::planRecordJson(const PlanRecord& r) const {
  std::ostringstream o;
  o << "{\"op\":" << r.seq << ",\"offset\":" << r.base << ",\"length\":" << r.len
    << ",\"hot\":" << (r.plan.hot ? "true" : "false") << ",\"segs\":[";
  for (size_t i = 0; i < r.plan.segments.size(); ++i) {
    const auto& rs = r.plan.segments[i];
    o << (i ? "," : "") << "[" << rs.rail_id << "," << r.base + rs.segment.offset << "," << rs.segment.length
      << "," << nezha::defaultChunkBytes(rs.segment.length, comm->world, algo) << "]";
  }
  o << "]";
  if (!r.grants.empty()) o << ",\"grants\":[" << r.grants << "]";
  o << "}";
  return o.str();
}

int64_t nz_engine::realtimeNs() {
  timespec ts;
  clock_gettime(CLOCK_REALTIME, &ts);
  return static_cast<int64_t>(ts.tv_sec) * 1000000000LL + ts.tv_nsec;
}

void nz_engine::calibrateClock() {
  int64_t best = INT64_MAX;
  for (int i = 0; i < 5; ++i) {
    stamps_host[0] = 0;
    const int64_t t0 = realtimeNs();
    nz::launchStamp(stamps_dev + 0, ctrl);
    NZ_CUDA(cudaStreamSynchronize(ctrl));
    const int64_t t1 = realtimeNs();
    if (t1 - t0 < best) {
      best = t1 - t0;
      clock_offset_ns = static_cast<int64_t>(stamps_host[0]) - (t0 + t1) / 2;
    }
  }
}

void nz_engine::handoff(Pending& p, const nezha::Plan& plan, const nezha::Segment& seg, int rid, uint64_t k,
                        nz_buf* in, nz_buf* out, uint64_t base, int dtype) {
  nz_rail* fr = rails[index(rid)];
  nz_fault_record_t rec{};
  const auto deadline = std::chrono::steady_clock::now() + std::chrono::seconds(60);
  for (;;) {
    volatile nz_fault_record_t* f = fr->fault_host;
    if (f->valid) {
      __sync_synchronize();
      rec.op_seq = f->op_seq;
      rec.chunk = f->chunk;
      rec.t_fail_ns = f->t_fail_ns;
      f->valid = 0;
      host_seen_ns = realtimeNs();
      break;
    }
    if (*reinterpret_cast<volatile int*>(fr->wd_host)) fail(NZ_ERR_TIMEOUT, "rail watchdog fired while waiting for a fault");
    if (std::chrono::steady_clock::now() > deadline) fail(NZ_ERR_TIMEOUT, "fault record never arrived");
  }
  std::memset(stamps_host, 0, 4 * sizeof(uint64_t));
  stamps_host[3] = rec.t_fail_ns;
  nz::launchStamp(stamps_dev + 0, ctrl);  // detection acknowledged on the device timeline
  health->channelDown(rid);
  bal->markFailed(rid);
  const auto target = nezha::chooseHandoffTarget(plan, rid, healthyIds());
  if (!target) fail(NZ_ERR_UNRECOVERABLE, "no surviving rail to take over the orphaned segment");
  const uint64_t C = nezha::defaultChunkBytes(seg.length, comm->world, algo);
  const nezha::Segment orphan = nezha::orphanOf(seg, C, k);
  nz_rail* tr = rails[index(*target)];
  nz::launchStamp(stamps_dev + 1, tr->stream);
  nz::railAllreduce(tr, in, out, base + seg.offset, seg.length, C, k, UINT64_MAX, dtype, p.op, -1, tr->stream);
  nz::launchStamp(stamps_dev + 2, tr->stream);
  cudaEvent_t e = event();
  NZ_CUDA(cudaEventRecord(e, tr->stream));
  p.ends.emplace_back(*target, e);
  fo = nz_failover_report_t{};
  fo.op_seq = p.op;
  fo.failed_rail = rid;
  fo.target_rail = *target;
  fo.orphan_offset = base + orphan.offset;
  fo.orphan_length = orphan.length;
  fo_pending = true;
}

void nz_engine::staged(const char* src, char* dst, uint64_t bytes, int dtype, cudaMemcpyKind kin,
                       cudaMemcpyKind kout, cudaStream_t user) {
  if (user) {
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    NZ_CUDA(cudaStreamIsCapturing(user, &cap));
    if (cap != cudaStreamCaptureStatusNone) {
      fail(NZ_ERR_INVALID, "staged allreduce cannot be captured: capture nz_engine_allreduce on symmetric buffers");
    }
  }
  ensureUnbound(bytes);
  nz_buf* in = ub_in;
  nz_buf* out = ub_out;
  const int me = comm->rank;
  // The UnboundBuffer is reused call after call: staging waits for the
  // previous call's reductions and copy-outs, and for the caller's stream.
  for (cudaStream_t prev : {io, d2h, user}) {
    if (!prev) continue;
    cudaEvent_t ready = event();
    NZ_CUDA(cudaEventRecord(ready, prev));
    NZ_CUDA(cudaStreamWaitEvent(h2d, ready, 0));
    pool.push_back(ready);
  }
  last_plans.clear();
  for (const auto& piece : nezha::hostPipelinePieces(bytes, nz::elemSizeOf(dtype))) {
    NZ_CUDA(cudaMemcpyAsync(in->ptrs[me] + piece.offset, src + piece.offset, piece.length, kin, h2d));
    cudaEvent_t up = event();
    NZ_CUDA(cudaEventRecord(up, h2d));
    NZ_CUDA(cudaStreamWaitEvent(io, up, 0));
    op(in, out, piece.offset, piece.length, dtype, io);
    cudaEvent_t red = event();
    NZ_CUDA(cudaEventRecord(red, io));
    NZ_CUDA(cudaStreamWaitEvent(d2h, red, 0));
    NZ_CUDA(cudaMemcpyAsync(dst + piece.offset, out->ptrs[me] + piece.offset, piece.length, kout, d2h));
    pool.push_back(up);  // waits are captured at enqueue time: safe to recycle
    pool.push_back(red);
  }
  if (user) {
    cudaEvent_t done = event();
    NZ_CUDA(cudaEventRecord(done, d2h));
    NZ_CUDA(cudaStreamWaitEvent(user, done, 0));
    pool.push_back(done);
  }
}

void nz_engine::synchronize() {
  NZ_CUDA(cudaDeviceSynchronize());  // rail streams and cold ops on callers' streams
  // Asynchronous failure path: a rail kernel whose barrier / LL poll timed
  // out (a peer never arrived) sets its watchdog word and exits. Ranks
  // agree (any rank saw it) and the rail goes Failed everywhere, so the
  // tables stay identical; the caller learns the results since the last
  // synchronize are not to be trusted (ChannelDownError, error.hpp:22-27).
  std::vector<int32_t> flags(rails.size(), 0);
  for (size_t i = 0; i < rails.size(); ++i) {
    volatile int* w = rails[i]->wd_host;
    flags[i] = *w;
    *w = 0;
  }
  if (comm->world > 1) {
    const auto msgs = nz::exchange(comm, flags.data(), flags.size() * sizeof(int32_t), {});
    for (const auto& m : msgs) {
      const int32_t* v = reinterpret_cast<const int32_t*>(m.data.data());
      for (size_t i = 0; i < flags.size(); ++i) flags[i] |= v[i];
    }
  }
  std::string down;
  for (size_t i = 0; i < rails.size(); ++i) {
    if (!flags[i]) continue;
    down += (down.empty() ? "" : ",") + std::to_string(specs[i].rail_id);
    if (health->state(specs[i].rail_id).status != nezha::HealthStatus::Failed) {
      health->channelDown(specs[i].rail_id);
      bal->markFailed(specs[i].rail_id);
    }
  }
  finishFailoverReport();
  drainTimer();  // every rank harvests the same ops here
  if (!down.empty()) {
    fail(NZ_ERR_RAIL_DOWN, "rail watchdog fired on rail(s) " + down +
                               ": marked Failed and excluded; results since the last synchronize are invalid");
  }
}

void nz_engine::ensureUnbound(uint64_t bytes) {
  if (ub_in && ub_in->size >= bytes) return;
  NZ_CUDA(cudaDeviceSynchronize());
  if (ub_in) nz::freeSymmetric(ub_in);
  if (ub_out) nz::freeSymmetric(ub_out);
  ub_in = ub_out = nullptr;
  ub_in = nz::allocSymmetric(comm, bytes);
  ub_out = nz::allocSymmetric(comm, bytes);
}

std::string nz_engine::stateJson() {
  std::ostringstream o;
  o << "{\"op_seq\":" << op_seq << ",\"world\":" << comm->world << ",\"rank\":" << comm->rank
    << ",\"sync_overhead_us\":" << nezha::formatDouble(bal->config().sync_overhead_us) << ",\"rails\":[";
  for (size_t i = 0; i < specs.size(); ++i) {
    const auto& p = bal->rails()[i];
    o << (i ? "," : "") << "{\"rail_id\":" << specs[i].rail_id << ",\"kind\":\""
      << (specs[i].kind == NZ_RAIL_NVLS ? "nvls" : specs[i].kind == NZ_RAIL_CE ? "ce" : "sm")
      << "\",\"sm_budget\":" << rails[i]->sm_budget << ",\"ll_max\":" << rails[i]->ll_max
      << ",\"oneshot_max\":" << rails[i]->os_max << ",\"protocol\":\"" << nezha::toString(p.protocol) << "\",\"health\":\""
      << nezha::toString(health->state(specs[i].rail_id).status) << "\",\"t_setup_us\":"
      << nezha::formatDouble(p.t_setup_us) << ",\"bandwidth_bps\":" << nezha::formatDouble(p.bandwidth_bps)
      << ",\"calibration\":[";
    for (size_t j = 0; j < p.efficiency_points.size(); ++j)
      o << (j ? "," : "") << "[" << p.efficiency_points[j].first << ","
        << nezha::formatDouble(p.efficiency_points[j].second) << "]";
    o << "]}";
  }
  o << "],\"concurrent\":[";
  const auto& conc = bal->concurrentProfiles();
  for (size_t i = 0; i < conc.size(); ++i) {
    o << (i ? "," : "") << "{\"rail_id\":" << conc[i].rail_id << ",\"calibration\":[";
    for (size_t j = 0; j < conc[i].efficiency_points.size(); ++j)
      o << (j ? "," : "") << "[" << conc[i].efficiency_points[j].first << ","
        << nezha::formatDouble(conc[i].efficiency_points[j].second) << "]";
    o << "]}";
  }
  o << "],\"compute_pool\":{\"mode\":" << static_cast<int>(pool_mode) << ",\"tokens\":"
    << (cpool ? cpool->totalTokens() : 0) << ",\"ops\":" << pool_stats.ops << ",\"waits\":" << pool_stats.waits
    << ",\"shrunk\":" << pool_stats.shrunk << "}";
  o << ",\"table\":" << bal->tableJson() << "}";
  return o.str();
}

namespace {
int copyOut(const std::string& s, char* out, size_t cap) {
  if (!out) return NZ_ERR_INVALID;
  if (s.size() + 1 > cap) return NZ_ERR_BUFFER;
  std::memcpy(out, s.c_str(), s.size() + 1);
  return NZ_OK;
}
}  // namespace

extern "C" {

void nz_engine_config_default(nz_engine_config_t* c) {
  if (!c) return;
  *c = nz_engine_config_t{};
  c->num_rails = 3;
  c->kinds[0] = NZ_RAIL_NVLS;
  c->kinds[1] = NZ_RAIL_CE;
  c->kinds[2] = NZ_RAIL_SM;
  c->sm_budget[0] = 0;
  c->sm_budget[1] = 0;
  c->sm_budget[2] = 0;
  c->algorithm = NZ_ALGO_RING_CHUNKED;
  c->tau = 5.0;
  c->eta = 0.05;
  c->convergence_eps = 0.01;
  c->sync_overhead_us = -1.0;
  c->window = 100;
  c->max_iters = 100;
  c->demote_after = 3;
  c->rails_toml = nullptr;
  c->calibrate_iters = 20;
  c->calibrate_max_bytes = uint64_t{1} << 30;
  c->timer_lag = 2;
  c->tune_budgets = 0;  // on once its hardware sweep is recorded in profiles/
}

int nz_engine_create(nz_comm_t* comm, const nz_engine_config_t* cfg, nz_engine_t** out) {
  return guarded([&] {
    if (!comm || !out) fail(NZ_ERR_INVALID, "null argument");
    auto eng = std::make_unique<nz_engine>();
    eng->comm = comm;
    if (cfg) {
      eng->cfg = *cfg;
    } else {
      nz_engine_config_default(&eng->cfg);
    }
    auto& c = eng->cfg;
    if (c.timer_lag < 1) c.timer_lag = 1;
    if (c.compute_pool < 0 || c.compute_pool > 2) fail(NZ_ERR_INVALID, "compute_pool must be 0 (off), 1 (block) or 2 (shrink)");
    if (c.pool_tokens < 0) fail(NZ_ERR_INVALID, "pool_tokens must be >= 0");
    eng->pool_mode = static_cast<nezha::PoolMode>(c.compute_pool);
    eng->cpool = std::make_unique<nezha::ComputePool>(c.pool_tokens > 0 ? c.pool_tokens : std::max(1, comm->sm_count));
    eng->algo = c.algorithm == NZ_ALGO_RING ? nezha::Algorithm::Ring : nezha::Algorithm::RingChunked;
    if (c.rails_toml) {
      eng->specs = nezha::parseRailsToml(c.rails_toml);
    } else {
      if (c.num_rails < 1 || c.num_rails > 3) fail(NZ_ERR_INVALID, "num_rails must be 1..3");
      for (int i = 0; i < c.num_rails; ++i) {
        nezha::RailSpec s;
        s.rail_id = i;
        s.kind = c.kinds[i];
        s.sm_budget = c.sm_budget[i];
        s.profile.rail_id = i;
        s.profile.protocol = s.kind == NZ_RAIL_NVLS ? nezha::ProtocolKind::Sharp
                             : s.kind == NZ_RAIL_CE ? nezha::ProtocolKind::Glex
                                                    : nezha::ProtocolKind::Tcp;
        eng->specs.push_back(s);
      }
    }
    std::sort(eng->specs.begin(), eng->specs.end(), [](auto& a, auto& b) { return a.rail_id < b.rail_id; });
    NZ_CUDA(cudaSetDevice(comm->device));
    for (auto& s : eng->specs) {
      nz_rail_t* r = nullptr;
      const int rc = nz_rail_create_ex(comm, s.kind, s.rail_id, s.sm_budget, c.graph_safe ? NZ_RAIL_FLAG_GRAPH_SAFE : 0,
                                       &r);
      if (rc != NZ_OK) fail(rc, nz_last_error());
      eng->rails.push_back(r);
    }
    std::vector<int> ids;
    std::vector<nezha::RailProfile> profiles;
    bool all_profiles = true;
    for (auto& s : eng->specs) {
      ids.push_back(s.rail_id);
      all_profiles &= s.has_profile;
      nezha::RailProfile p = s.profile;
      if (!s.has_profile) {  // placeholder until calibration replaces it
        p.t_setup_us = 10;
        p.bandwidth_bps = 1e11;
      }
      profiles.push_back(p);
    }
    nezha::BalancerConfig bc;
    bc.tau = c.tau;
    bc.eta = c.eta;
    bc.convergence_eps = c.convergence_eps;
    bc.sync_overhead_us = c.sync_overhead_us < 0 ? 0.0 : c.sync_overhead_us;
    bc.window = c.window;
    bc.max_iters = c.max_iters;
    bc.demote_after = c.demote_after;
    eng->bal = std::make_unique<nezha::Balancer>(profiles, bc);
    nz_engine* raw = eng.get();
    eng->bal->setAgreement([raw](int, const std::vector<std::pair<int, nezha::Micros>>& m) { return raw->agree(m); });
    eng->health = std::make_unique<nezha::HealthMonitor>(ids);
    NZ_CUDA(cudaStreamCreateWithFlags(&eng->ctrl, cudaStreamNonBlocking));
    NZ_CUDA(cudaStreamCreateWithFlags(&eng->io, cudaStreamNonBlocking));
    NZ_CUDA(cudaStreamCreateWithFlags(&eng->h2d, cudaStreamNonBlocking));
    NZ_CUDA(cudaStreamCreateWithFlags(&eng->d2h, cudaStreamNonBlocking));
    NZ_CUDA(cudaHostAlloc(&eng->stamps_host, 4 * sizeof(uint64_t), cudaHostAllocMapped));
    std::memset(eng->stamps_host, 0, 4 * sizeof(uint64_t));
    NZ_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&eng->stamps_dev), eng->stamps_host, 0));
    eng->calibrateClock();
    if (!all_profiles || c.sync_overhead_us < 0) eng->calibrate();
    NZ_CUDA(cudaDeviceSynchronize());
    *out = eng.release();
  });
}

int nz_engine_destroy(nz_engine_t* eng) {
  return guarded([&] {
    if (!eng) return;
    cudaSetDevice(eng->comm->device);
    cudaDeviceSynchronize();
    for (auto e : eng->pool) cudaEventDestroy(e);
    for (auto e : eng->pool_pending) cudaEventDestroy(e);
    for (auto& p : eng->pending) {
      cudaEventDestroy(p.start);
      for (auto& pr : p.ends) cudaEventDestroy(pr.second);
    }
    for (auto* r : eng->rails) nz_rail_destroy(r);
    if (eng->ub_in) nz::freeSymmetric(eng->ub_in);
    if (eng->ub_out) nz::freeSymmetric(eng->ub_out);
    if (eng->ctrl) cudaStreamDestroy(eng->ctrl);
    if (eng->io) cudaStreamDestroy(eng->io);
    if (eng->h2d) cudaStreamDestroy(eng->h2d);
    if (eng->d2h) cudaStreamDestroy(eng->d2h);
    if (eng->stamps_host) cudaFreeHost(eng->stamps_host);
    delete eng;
  });
}

int nz_engine_allreduce(nz_engine_t* eng, nz_buf_t* in, nz_buf_t* out, uint64_t bytes, int dtype, void* stream) {
  return guarded([&] {
    if (!eng || !in || !out) fail(NZ_ERR_INVALID, "null argument");
    const int es = nz::elemSizeOf(dtype);
    if (bytes % es) fail(NZ_ERR_INVALID, "bytes is not a whole number of elements");
    if (bytes > in->size || bytes > out->size) fail(NZ_ERR_INVALID, "payload exceeds the buffers");
    if (bytes == 0) return;
    NZ_CUDA(cudaSetDevice(eng->comm->device));
    // NULL is the legacy default stream; pass it explicitly, since a NULL
    // stream given to a rail means "the rail's own stream" (nz_rail_allreduce)
    // and the cold path would then run unordered with the caller's copies.
    cudaStream_t user = stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy;
    eng->last_plans.clear();
    for (const auto& piece : nezha::splitOversized(bytes)) {
      eng->op(in, out, piece.offset, piece.length, dtype, user);
    }
  });
}

int nz_engine_allreduce_host(nz_engine_t* eng, const void* host_in, void* host_out, uint64_t bytes, int dtype) {
  return guarded([&] {
    if (!eng || !host_in || !host_out) fail(NZ_ERR_INVALID, "null argument");
    if (bytes == 0) return;
    NZ_CUDA(cudaSetDevice(eng->comm->device));
    eng->staged(static_cast<const char*>(host_in), static_cast<char*>(host_out), bytes, dtype, cudaMemcpyHostToDevice,
                cudaMemcpyDeviceToHost, nullptr);
    NZ_CUDA(cudaStreamSynchronize(eng->d2h));
    NZ_CUDA(cudaStreamSynchronize(eng->io));
    eng->finishFailoverReport();
  });
}

int nz_engine_allreduce_device(nz_engine_t* eng, const void* src, void* dst, uint64_t bytes, int dtype,
                               void* stream) {
  return guarded([&] {
    if (!eng || !src || !dst) fail(NZ_ERR_INVALID, "null argument");
    if (bytes == 0) return;
    NZ_CUDA(cudaSetDevice(eng->comm->device));
    cudaStream_t user = stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy;
    eng->staged(static_cast<const char*>(src), static_cast<char*>(dst), bytes, dtype, cudaMemcpyDeviceToDevice,
                cudaMemcpyDeviceToDevice, user);
  });
}

int nz_engine_inject_failure(nz_engine_t* eng, uint32_t op_seq, int rail_id, uint64_t chunk) {
  return guarded([&] {
    if (!eng) fail(NZ_ERR_INVALID, "null engine");
    eng->index(rail_id);
    if (op_seq < eng->op_seq) fail(NZ_ERR_INVALID, "op already issued");
    eng->inject[op_seq] = {rail_id, chunk};
    eng->calibrateClock();  // %globaltimer drifts against the host clock: re-anchor next to the op
  });
}

int nz_engine_readmit(nz_engine_t* eng, int rail_id) {
  return guarded([&] {
    if (!eng) fail(NZ_ERR_INVALID, "null engine");
    eng->synchronize();
    eng->drainTimer();
    eng->health->heartbeat(rail_id, 0);
    eng->health->readmit(rail_id, 0, 0);
    eng->bal->readmit(rail_id);
  });
}

int nz_engine_synchronize(nz_engine_t* eng) {
  return guarded([&] {
    if (!eng) fail(NZ_ERR_INVALID, "null engine");
    NZ_CUDA(cudaSetDevice(eng->comm->device));
    eng->synchronize();
  });
}

uint32_t nz_engine_op_seq(const nz_engine_t* eng) { return eng ? eng->op_seq : 0; }

int nz_engine_last_failover(nz_engine_t* eng, nz_failover_report_t* rep) {
  if (!eng || !rep) return NZ_ERR_INVALID;
  eng->finishFailoverReport();
  if (!eng->have_fo) return NZ_ERR_INVALID;
  *rep = eng->fo;
  return NZ_OK;
}

int nz_engine_state_json(nz_engine_t* eng, char* out, size_t cap) {
  std::string s;
  const int rc = guarded([&] {
    if (!eng) fail(NZ_ERR_INVALID, "null engine");
    s = eng->stateJson();
  });
  return rc != NZ_OK ? rc : copyOut(s, out, cap);
}

int nz_engine_rail_stats(nz_engine_t* eng, int rail_id, uint64_t* ops, double* total_us, uint64_t* total_bytes) {
  return guarded([&] {
    if (!eng || !ops || !total_us || !total_bytes) fail(NZ_ERR_INVALID, "null argument");
    const int i = eng->index(rail_id);
    if (eng->stats.size() != eng->specs.size()) eng->stats.assign(eng->specs.size(), nz_engine::RailStat{});
    *ops = eng->stats[i].ops;
    *total_us = eng->stats[i].us;
    *total_bytes = eng->stats[i].bytes;
  });
}

int nz_engine_save_state(nz_engine_t* eng, char* out, size_t cap) {
  std::string s;
  const int rc = guarded([&] {
    if (!eng) fail(NZ_ERR_INVALID, "null engine");
    s = eng->bal->saveState();
  });
  return rc != NZ_OK ? rc : copyOut(s, out, cap);
}

int nz_engine_load_state(nz_engine_t* eng, const char* json) {
  return guarded([&] {
    if (!eng || !json) fail(NZ_ERR_INVALID, "null argument");
    eng->synchronize();
    eng->bal->loadState(json);
  });
}

int nz_engine_stats_reset(nz_engine_t* eng) {
  if (!eng) return NZ_ERR_INVALID;
  eng->stats.assign(eng->specs.size(), nz_engine::RailStat{});
  return NZ_OK;
}

int nz_engine_last_plan_json(nz_engine_t* eng, char* out, size_t cap) {
  if (!eng) return NZ_ERR_INVALID;
  std::string s = "[";
  for (size_t i = 0; i < eng->last_plans.size(); ++i) s += (i ? "," : "") + eng->planRecordJson(eng->last_plans[i]);
  s += "]";
  return copyOut(s, out, cap);
}

int nz_engine_plan_json(nz_engine_t* eng, uint64_t bytes, char* out, size_t cap) {
  std::string s;
  const int rc = guarded([&] {
    if (!eng || bytes == 0) fail(NZ_ERR_INVALID, "bad argument");
    std::ostringstream o;
    o << "{\"pieces\":[";
    bool first = true;
    for (const auto& piece : nezha::splitOversized(bytes)) {
      const auto plan = eng->bal->allocate(piece.length);
      o << (first ? "" : ",") << "{\"offset\":" << piece.offset << ",\"plan\":"
        << nezha::planJson(0, piece.length, plan) << "}";
      first = false;
    }
    o << "]}";
    s = o.str();
  });
  return rc != NZ_OK ? rc : copyOut(s, out, cap);
}

}  // extern "C"
