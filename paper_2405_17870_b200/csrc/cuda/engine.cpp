// Engine: the multi-rail allreduce of one rank (
// PAPER.md:379 Fig. 6). Planner (Balancer) + rails (rails.cu) + Timer, with
// the failure monitor in engine_monitor.cpp. See include/nezha/engine.hpp for
// the contract; startup calibration lives in engine_calibrate.cpp.
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

// Timer: op k is sampled when op k + timer_lag is issued,
// the same op on every rank, so every flush (and its cross-rank agreement)
// happens at the same point of every rank's op stream. The end events are
// recorded right after each rail's launches, so this never waits on a
// stream gate, i.e. never on the failure monitor.
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
    // A rail whose launches failed (on every rank alike) makes the op a
    // non-sample: its latency is the failure's, not the rail's.
    for (auto& [ri, tag] : p.tags) {
      const volatile nz_rail_status_t* s = rails[ri]->status_host;
      if (static_cast<int32_t>(s->ok_tag - tag) < 0) p.skip = true;
    }
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

void nz_engine::launchSegment(uint32_t seq, const nezha::Plan& plan, const nezha::RailSegment& rs, nz_buf* in,
                              nz_buf* out, uint64_t base, int dtype, cudaStream_t st, nz::ComputeGate* gate,
                              bool capturing, cudaStream_t user, cudaEvent_t* end_out, Pending* p) {
  const int ri = index(rs.rail_id);
  nz_rail* r = rails[ri];
  const uint64_t C = nezha::defaultChunkBytes(rs.segment.length, comm->world, algo);
  nz::RailOp o;
  o.in = in;
  o.out = out;
  o.seg_off = base + rs.segment.offset;
  o.seg_len = rs.segment.length;
  o.chunk_bytes = C;
  o.dtype = dtype;
  o.op_seq = seq;
  o.st = st;
  o.gate = gate;
  o.status = !capturing;
  auto inj = inject.find(seq);
  if (inj != inject.end() && inj->second.first == rs.rail_id) o.stall_chunk = static_cast<int64_t>(inj->second.second);
  const uint32_t tag = nz::railRun(r, o);
  if (end_out) {  // Timer end of a hot op's rail
    *end_out = event();
    NZ_CUDA(cudaEventRecord(*end_out, st));
    NZ_CUDA(cudaStreamWaitEvent(user, *end_out, 0));
  }
  if (!monitored || capturing || tag == 0) return;
  Entry e;
  e.op = seq;
  e.rail = ri;
  e.tag = tag;
  e.in = in;
  e.out = out;
  e.seg_off = o.seg_off;
  e.seg_len = o.seg_len;
  e.chunk = C;
  e.chunk_end = (o.seg_len + C - 1) / C;
  e.dtype = dtype;
  e.ll = nz::railLLPath(r, o.seg_off, o.seg_len);
  e.plan = plan;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!entry_pool.empty()) {
      e.end = entry_pool.back();
      entry_pool.pop_back();
    }
  }
  if (!e.end) NZ_CUDA(cudaEventCreateWithFlags(&e.end, cudaEventDisableTiming));
  NZ_CUDA(cudaEventRecord(e.end, st));  // before the gate: the monitor must see a failed launch retire
  // The caller's stream passes this segment only once its gate word holds
  // the tag: written by the rail's last launch when it succeeded, or by the
  // monitor's reroute when it did not.
  NZ_CU(NZ_DRV(cuStreamWaitValue32)(reinterpret_cast<CUstream>(user), nz::railGateAddr(r), tag,
                                    CU_STREAM_WAIT_VALUE_GEQ));
  if (p) p->tags.emplace_back(ri, tag);
  {
    std::lock_guard<std::mutex> lk(mu);
    inflight.push_back(std::move(e));
  }
  cv.notify_all();
}

void nz_engine::op(nz_buf* in, nz_buf* out, uint64_t base, uint64_t len, int dtype, cudaStream_t user) {
  const uint32_t seq = op_seq++;
  // Inside a CUDA graph capture (graph-safe rails only) nothing may wait on
  // the device: no Timer harvest, no Timer sample, no failure injection, no
  // monitor entries or gates.
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  NZ_CUDA(cudaStreamIsCapturing(user, &cap));
  const bool capturing = cap != cudaStreamCaptureStatusNone;
  if (capturing) {
    if (!cfg.graph_safe) fail(NZ_ERR_INVALID, "graph capture needs an engine created with graph_safe = 1");
    if (inject.count(seq)) fail(NZ_ERR_INVALID, "failure injection inside a graph capture");
  } else {
    harvest(seq);
  }
  applyTableEvents(seq);
  nezha::Plan plan = bal->allocate(len);
  if (!plan.hot) {
    // Cold (or rho-gated) op: one rail, launched straight on the caller's
    // stream — no fork/join, no Timer events. A single-rail sample cannot
    // move the table (a cold flush only records telemetry), so skipping it
    // leaves every decision unchanged (P11).
    launchSegment(seq, plan, plan.segments[0], in, out, base, dtype, user, nullptr, capturing, user, nullptr,
                  nullptr);
    inject.erase(seq);
    recordPlan(seq, base, len, std::move(plan));
    return;
  }
  Pending p;
  p.op = seq;
  p.plan = plan;
  p.start = event();
  NZ_CUDA(cudaEventRecord(p.start, user));
  std::vector<std::pair<int, uint64_t>> segs;
  for (const auto& rs : plan.segments) segs.emplace_back(rs.rail_id, rs.segment.length);
  std::string grant_log;
  auto gates = gatesFor(segs, &grant_log);
  for (size_t si = 0; si < plan.segments.size(); ++si) {
    const auto& rs = plan.segments[si];
    nz_rail* r = rails[index(rs.rail_id)];
    NZ_CUDA(cudaStreamWaitEvent(r->stream, p.start, 0));
    cudaEvent_t e = nullptr;
    launchSegment(seq, plan, rs, in, out, base, dtype, r->stream, &gates[si], capturing, user, &e, &p);
    p.ends.emplace_back(rs.rail_id, e);
  }
  if (inject.erase(seq)) p.skip = true;
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
  NZ_CUDA(cudaDeviceSynchronize());  // rail streams, gated caller streams (the monitor releases them)
  if (monitored) drainMonitor();
  // Without the monitor a rail kernel whose cross-rank wait timed out sets
  // its watchdog word and exits: ranks agree (any rank saw it) and the rail
  // goes Failed everywhere, so the tables stay identical; the caller learns
  // the results since the last synchronize are not to be trusted
  // (ChannelDownError, error.hpp:22-27). With the monitor those launches
  // were rerouted already: the words are just cleared.
  std::vector<int32_t> flags(rails.size(), 0);
  for (size_t i = 0; i < rails.size(); ++i) {
    volatile int* w = rails[i]->wd_host;
    flags[i] = monitored ? 0 : *w;
    *w = 0;
  }
  if (comm->world > 1 && !monitored) {
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
  drainTimer();  // every rank harvests the same ops here
  if (!down.empty()) {
    fail(NZ_ERR_RAIL_DOWN, "rail watchdog fired on rail(s) " + down +
                               ": marked Failed and excluded; results since the last synchronize are invalid");
  }
  std::string err;
  {
    std::lock_guard<std::mutex> lk(mu);
    err.swap(mon_error);
  }
  if (!err.empty()) fail(NZ_ERR_UNRECOVERABLE, "failure monitor: " + err);
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
    << ",\"loopback\":" << (comm->loop ? "true" : "false")
    << ",\"sync_overhead_us\":" << nezha::formatDouble(bal->config().sync_overhead_us) << ",\"rails\":[";
  std::lock_guard<std::mutex> lk(mu);
  for (size_t i = 0; i < specs.size(); ++i) {
    const auto& p = bal->rails()[i];
    o << (i ? "," : "") << "{\"rail_id\":" << specs[i].rail_id << ",\"kind\":\""
      << (specs[i].kind == NZ_RAIL_NVLS ? "nvls" : specs[i].kind == NZ_RAIL_CE ? "ce" : "sm")
      << "\",\"sm_budget\":" << rails[i]->sm_budget << ",\"ll_max\":" << rails[i]->ll_max << ",\"protocol\":\""
      << nezha::toString(p.protocol) << "\",\"health\":\"" << nezha::toString(health->state(specs[i].rail_id).status)
      << "\",\"planned\":" << (bal->healthy(specs[i].rail_id) ? "true" : "false")
      << ",\"t_setup_us\":" << nezha::formatDouble(p.t_setup_us)
      << ",\"bandwidth_bps\":" << nezha::formatDouble(p.bandwidth_bps) << ",\"calibration\":[";
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
  o << ",\"monitor\":{\"on\":" << (monitored ? "true" : "false") << ",\"off_reason\":\"" << mon_off_reason
    << "\",\"failovers\":" << reports.size()
    << ",\"inflight\":" << inflight.size() << ",\"failed\":[";
  bool first = true;
  for (int id : agreed_failed) {
    o << (first ? "" : ",") << id;
    first = false;
  }
  o << "]}";
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
  // Op k is harvested when op k + 16 is issued: the issuing thread (e.g. a
  // DDP hook inside backward) runs up to 16 ops ahead of the device.
  c->timer_lag = 16;
  c->tune_budgets = 0;  // on once its hardware sweep is recorded in profiles/
  c->monitor = 1;
  c->detect_us = 0;
  c->heartbeat_us = 50000;  // SPEC.md:380-388; NEZHA_HEARTBEAT_US overrides the default
  if (const char* h = getenv("NEZHA_HEARTBEAT_US")) {
    const double v = atof(h);
    if (v > 0) c->heartbeat_us = v;
  }
  c->readmit_hold_us = 1e6;
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
    if (!(c.heartbeat_us > 0)) c.heartbeat_us = 50000;
    if (c.readmit_hold_us < 0) c.readmit_hold_us = 0;
    if (c.compute_pool < 0 || c.compute_pool > 2) fail(NZ_ERR_INVALID, "compute_pool must be 0 (off), 1 (block) or 2 (shrink)");
    if (c.pool_tokens < 0) fail(NZ_ERR_INVALID, "pool_tokens must be >= 0");
    if (c.graph_safe && comm->loop && comm->world > 1)
      fail(NZ_ERR_UNSUPPORTED, "graph-safe engines need one process per rank (loopback launches cannot be captured)");
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
    // Destroys whatever was built if a later step throws.
    struct Cleanup {
      std::unique_ptr<nz_engine>* e;
      ~Cleanup() {
        if (*e) nz_engine_destroy(e->release());
      }
    } cleanup{&eng};
    for (auto& s : eng->specs) {
      eng->rails.push_back(nz::railCreate(comm, s.kind, s.rail_id, s.sm_budget, c.graph_safe != 0, false));
      eng->rails.back()->detect_us = c.detect_us;
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
    eng->health = std::make_unique<nezha::HealthMonitor>(ids, c.heartbeat_us);
    NZ_CUDA(cudaStreamCreateWithFlags(&eng->ctrl, cudaStreamNonBlocking));
    NZ_CUDA(cudaStreamCreateWithFlags(&eng->io, cudaStreamNonBlocking));
    NZ_CUDA(cudaStreamCreateWithFlags(&eng->h2d, cudaStreamNonBlocking));
    NZ_CUDA(cudaStreamCreateWithFlags(&eng->d2h, cudaStreamNonBlocking));
    if (comm->loop) {
      NZ_CUDA(cudaStreamCreateWithFlags(&eng->loop_user, cudaStreamNonBlocking));
      NZ_CUDA(cudaEventCreateWithFlags(&eng->loop_ev, cudaEventDisableTiming));
    }
    NZ_CUDA(cudaHostAlloc(&eng->rec_stamps_host, 4 * sizeof(uint64_t), cudaHostAllocMapped));
    std::memset(eng->rec_stamps_host, 0, 4 * sizeof(uint64_t));
    NZ_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&eng->rec_stamps_dev), eng->rec_stamps_host, 0));
    eng->calibrateClock();
    if (!all_profiles || c.sync_overhead_us < 0) eng->calibrate();
    NZ_CUDA(cudaDeviceSynchronize());
    eng->startMonitor();
    *out = eng.release();
  });
}

int nz_engine_destroy(nz_engine_t* eng) {
  return guarded([&] {
    if (!eng) return;
    cudaSetDevice(eng->comm->device);
    cudaDeviceSynchronize();
    eng->stopMonitor();
    for (auto e : eng->pool) cudaEventDestroy(e);
    for (auto e : eng->pool_pending) cudaEventDestroy(e);
    for (auto e : eng->entry_pool) cudaEventDestroy(e);
    for (auto& en : eng->inflight) cudaEventDestroy(en.end);
    for (auto& p : eng->pending) {
      cudaEventDestroy(p.start);
      for (auto& pr : p.ends) cudaEventDestroy(pr.second);
    }
    for (auto* r : eng->twins) nz::railDestroy(r);
    for (auto* r : eng->rails) nz::railDestroy(r);
    if (eng->ub_in) nz::freeSymmetric(eng->ub_in);
    if (eng->ub_out) nz::freeSymmetric(eng->ub_out);
    if (eng->ctrl) cudaStreamDestroy(eng->ctrl);
    if (eng->io) cudaStreamDestroy(eng->io);
    if (eng->h2d) cudaStreamDestroy(eng->h2d);
    if (eng->d2h) cudaStreamDestroy(eng->d2h);
    if (eng->loop_user) cudaStreamDestroy(eng->loop_user);
    if (eng->loop_ev) cudaEventDestroy(eng->loop_ev);
    if (eng->rec_stamps_host) cudaFreeHost(eng->rec_stamps_host);
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
    cudaStream_t user = eng->callerStream(stream);
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
  });
}

int nz_engine_allreduce_device(nz_engine_t* eng, const void* src, void* dst, uint64_t bytes, int dtype,
                               void* stream) {
  return guarded([&] {
    if (!eng || !src || !dst) fail(NZ_ERR_INVALID, "null argument");
    if (bytes == 0) return;
    NZ_CUDA(cudaSetDevice(eng->comm->device));
    cudaStream_t user = eng->callerStream(stream);
    eng->staged(static_cast<const char*>(src), static_cast<char*>(dst), bytes, dtype, cudaMemcpyDeviceToDevice,
                cudaMemcpyDeviceToDevice, user);
  });
}

int nz_engine_inject_failure(nz_engine_t* eng, uint32_t op_seq, int rail_id, uint64_t chunk) {
  return guarded([&] {
    if (!eng) fail(NZ_ERR_INVALID, "null engine");
    eng->index(rail_id);
    if (op_seq < eng->op_seq) fail(NZ_ERR_INVALID, "op already issued");
    if (chunk > static_cast<uint64_t>(INT64_MAX)) fail(NZ_ERR_INVALID, "chunk out of range");
    if (!eng->monitored && eng->comm->world > 1)
      fail(NZ_ERR_INVALID, "failure injection needs the failure monitor (config monitor = 1)");
    eng->inject[op_seq] = {rail_id, chunk};
  });
}

int nz_engine_readmit(nz_engine_t* eng, int rail_id) {
  return guarded([&] {
    if (!eng) fail(NZ_ERR_INVALID, "null engine");
    NZ_CUDA(cudaSetDevice(eng->comm->device));
    eng->readmit(rail_id);
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

nz_rail_t* nz_engine_rail(nz_engine_t* eng, int rail_id) {
  if (!eng) return nullptr;
  for (size_t i = 0; i < eng->specs.size(); ++i)
    if (eng->specs[i].rail_id == rail_id) return eng->rails[i];
  return nullptr;
}

int nz_engine_last_failover(nz_engine_t* eng, nz_failover_report_t* rep) {
  if (!eng || !rep) return NZ_ERR_INVALID;
  std::lock_guard<std::mutex> lk(eng->mu);
  if (eng->reports.empty()) return NZ_ERR_INVALID;
  *rep = eng->reports.back();
  return NZ_OK;
}

int nz_engine_failover_count(nz_engine_t* eng) {
  if (!eng) return NZ_ERR_INVALID;
  std::lock_guard<std::mutex> lk(eng->mu);
  return static_cast<int>(eng->reports.size());
}

int nz_engine_failover_get(nz_engine_t* eng, int i, nz_failover_report_t* rep) {
  if (!eng || !rep) return NZ_ERR_INVALID;
  std::lock_guard<std::mutex> lk(eng->mu);
  if (i < 0 || i >= static_cast<int>(eng->reports.size())) return NZ_ERR_INVALID;
  *rep = eng->reports[i];
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
