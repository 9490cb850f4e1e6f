// Engine: the multi-rail allreduce of one rank (
// PAPER.md:379 Fig. 6). Planner (Balancer) + rails (rails.cu) + Timer +
// fault monitor / handoff. See include/nezha/engine.hpp for the contract.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <deque>
#include <memory>
#include <sstream>
#include <thread>

#include "../host/planner_trace.hpp"
#include "internal.h"
#include "nezha/balancer.hpp"
#include "nezha/calibration.hpp"
#include "nezha/collective.hpp"
#include "nezha/compute_pool.hpp"
#include "nezha/core/error.hpp"
#include "nezha/core/math.hpp"
#include "nezha/engine.hpp"
#include "nezha/faults.hpp"
#include "nezha/util/toml.hpp"


using nz::fail;
using nz::guarded;

struct nz_engine {
  struct Pending {
    uint32_t op = 0;
    nezha::Plan plan;
    cudaEvent_t start = nullptr;
    std::vector<std::pair<int, cudaEvent_t>> ends;
    bool skip = false;  // an op that lost a rail is not a Timer sample
  };

  nz_comm* comm = nullptr;
  nz_engine_config_t cfg{};
  std::vector<nezha::RailSpec> specs;  // sorted by rail_id
  std::vector<nz_rail*> rails;         // parallel to specs
  std::unique_ptr<nezha::Balancer> bal;
  std::unique_ptr<nezha::HealthMonitor> health;
  nezha::Algorithm algo = nezha::Algorithm::RingChunked;
  uint32_t op_seq = 0;
  std::deque<Pending> pending;
  std::vector<cudaEvent_t> pool;
  std::map<uint32_t, std::pair<int, uint64_t>> inject;
  nz_failover_report_t fo{};
  bool have_fo = false;
  bool fo_pending = false;
  uint64_t* stamps_host = nullptr;  // [0] detect, [1] resume, [2] done, [3] fault
  uint64_t* stamps_dev = nullptr;
  cudaStream_t ctrl = nullptr;
  cudaStream_t io = nullptr;
  cudaStream_t h2d = nullptr;  // host path: uploads of the next piece
  cudaStream_t d2h = nullptr;  // host path: downloads of the previous piece
  nz_buf* ub_in = nullptr;
  nz_buf* ub_out = nullptr;
  // Plans of each piece of the last call; rendered to JSON only on request
  // (nz_engine_last_plan_json) so the per-op host path builds no strings.
  struct PlanRecord {
    uint32_t seq = 0;
    uint64_t base = 0, len = 0;
    nezha::Plan plan;
    std::string grants;  // [rail, demand, grant, [waits]]... when the ComputePool is on
  };
  std::vector<PlanRecord> last_plans;
  int64_t clock_offset_ns = 0;          // %globaltimer - CLOCK_REALTIME
  int64_t host_seen_ns = 0;             // host monitor saw the last fault record
  struct RailStat {
    uint64_t ops = 0;
    double us = 0;
    uint64_t bytes = 0;
  };
  std::vector<RailStat> stats;  // parallel to specs
  // ComputePool over this GPU's SMs (P14), driven in stream order.
  std::unique_ptr<nezha::ComputePool> cpool;
  nezha::PoolMode pool_mode = nezha::PoolMode::Off;
  struct PoolStats {
    uint64_t ops = 0;     // hot ops arbitrated
    uint64_t waits = 0;   // computation phases ordered after an earlier holder
    uint64_t shrunk = 0;  // grants below demand
  } pool_stats;

  int index(int rail_id) const {
    for (size_t i = 0; i < specs.size(); ++i)
      if (specs[i].rail_id == rail_id) return static_cast<int>(i);
    fail(NZ_ERR_INVALID, "unknown rail " + std::to_string(rail_id));
  }

  cudaEvent_t event() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    NZ_CUDA(cudaEventCreate(&e));
    return e;
  }

  // Element-wise max over ranks: what every rank applies at a flush.
  std::vector<std::pair<int, nezha::Micros>> agree(const std::vector<std::pair<int, nezha::Micros>>& mine) {
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

  void harvest(uint32_t upto) {
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

  void drainTimer() { harvest(UINT32_MAX - 8); }

  std::vector<int> healthyIds() const { return health->healthyRails(); }

  void finishFailoverReport() {
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

  // Computation-phase gates of one concurrent launch of `segs` (rail_id,
  // length) in rail order; empty when the pool is off. The release events go
  // back to the event pool once the launch is enqueued (waits are captured at
  // cudaStreamWaitEvent time).
  std::vector<nz::ComputeGate> gatesFor(const std::vector<std::pair<int, uint64_t>>& segs, std::string* log) {
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
  std::vector<cudaEvent_t> pool_pending;  // gate events of the launch being enqueued
  void recycleGates() {
    for (auto e : pool_pending) pool.push_back(e);
    pool_pending.clear();
  }

  // One op (piece) of at most 1 GiB at byte offset `base`.
  void op(nz_buf* in, nz_buf* out, uint64_t base, uint64_t len, int dtype, cudaStream_t user) {
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

  void recordPlan(uint32_t seq, uint64_t base, uint64_t len, nezha::Plan&& plan, std::string&& grants = {}) {
    last_plans.push_back(PlanRecord{seq, base, len, std::move(plan), std::move(grants)});
  }

  std::string planRecordJson(const PlanRecord& r) const {
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

  // Exception handler: wait for the device's fault record,
  // mark the rail Failed, pick the target (P9) and run the orphan chunks on
  // it with the failed segment's geometry (P10), after its current task.
  static int64_t realtimeNs() {
    timespec ts;
    clock_gettime(CLOCK_REALTIME, &ts);
    return static_cast<int64_t>(ts.tv_sec) * 1000000000LL + ts.tv_nsec;
  }

  // %globaltimer vs host CLOCK_REALTIME: best of 5 stamp round trips. Lets
  // the report place the host monitor's detection on the device timeline.
  void calibrateClock() {
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

  void handoff(Pending& p, const nezha::Plan& plan, const nezha::Segment& seg, int rid, uint64_t k, nz_buf* in,
               nz_buf* out, uint64_t base, int dtype) {
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

  // Allreduce of memory outside the symmetric heap (host, or device memory
  // the caller owns): a three-stage pipeline over pieces.
  // Piece i+1 is staged into the UnboundBuffer on h2d while the rails reduce
  // piece i on io and piece i-1 is copied out on d2h, so the copies overlap
  // each other and the NVLink work. Each piece is an independent allreduce
  // with its own recorded plan (like split_oversized pieces); the pieces are
  // a function of `bytes` alone, so every rank cuts the same ones. `user`
  // (device variant): the staging waits for it first and it waits for the
  // last copy-out; nullptr (host variant): the caller synchronizes.
  void staged(const char* src, char* dst, uint64_t bytes, int dtype, cudaMemcpyKind kin, cudaMemcpyKind kout,
              cudaStream_t user) {
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

  // Collective point: every rank calls it at the same place in its op stream.
  void synchronize() {
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

  void ensureUnbound(uint64_t bytes) {
    if (ub_in && ub_in->size >= bytes) return;
    NZ_CUDA(cudaDeviceSynchronize());
    if (ub_in) nz::freeSymmetric(ub_in);
    if (ub_out) nz::freeSymmetric(ub_out);
    ub_in = ub_out = nullptr;
    ub_in = nz::allocSymmetric(comm, bytes);
    ub_out = nz::allocSymmetric(comm, bytes);
  }

  // Startup calibration: each rail alone over a size sweep, then the
  // coordination cost of a fork/join over all rails.
  // CTA budget of the SM-driven rails, measured instead of assumed: each
  // candidate grid runs the two-shot path at one large size, ranks agree on
  // the times (max), the fastest wins (ties within 3 % go to the smaller
  // grid). Rails whose budget the config pins are left alone. The chosen
  // grids then hold for calibration and every op, identically on all ranks.
  void tuneBudgets(uint64_t maxb, cudaEvent_t e0, cudaEvent_t e1) {
    if (comm->world == 1) return;
    const uint64_t s = std::min<uint64_t>(uint64_t{64} << 20, maxb) & ~uint64_t{4095};
    if (s <= (uint64_t{4} << 20)) return;  // must be past the one-shot (LL) ceiling
    for (size_t i = 0; i < rails.size(); ++i) {
      nz_rail* r = rails[i];
      if (specs[i].sm_budget > 0) continue;
      std::vector<int> cands;
      if (r->kind == NZ_RAIL_NVLS) cands = {16, 32, 64};
      if (r->kind == NZ_RAIL_SM) cands = {32, 64, 128};
      if (cands.empty()) continue;
      const uint64_t C = nezha::defaultChunkBytes(s, comm->world, algo);
      std::vector<double> t(cands.size());
      for (size_t k = 0; k < cands.size(); ++k) {
        r->sm_budget = std::min(cands[k], comm->sm_count);
        for (int w = 0; w < 2; ++w) nz::railAllreduce(r, ub_in, ub_out, 0, s, C, 0, UINT64_MAX, NZ_F32, 0, -1, r->stream);
        NZ_CUDA(cudaEventRecord(e0, r->stream));
        for (int it = 0; it < 5; ++it) nz::railAllreduce(r, ub_in, ub_out, 0, s, C, 0, UINT64_MAX, NZ_F32, 0, -1, r->stream);
        NZ_CUDA(cudaEventRecord(e1, r->stream));
        NZ_CUDA(cudaEventSynchronize(e1));
        float ms = 0;
        NZ_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        t[k] = ms;
      }
      const auto msgs = nz::exchange(comm, t.data(), t.size() * sizeof(double), {});
      for (int rk = 0; rk < comm->world; ++rk) {
        const double* v = reinterpret_cast<const double*>(msgs[rk].data.data());
        for (size_t k = 0; k < t.size(); ++k) t[k] = std::max(t[k], v[k]);
      }
      size_t best = 0;
      for (size_t k = 1; k < t.size(); ++k)
        if (t[k] < t[best] * 0.97) best = k;
      r->sm_budget = std::min(cands[best], comm->sm_count);
    }
  }

  // Which protocol a rail uses at which size, measured instead of assumed:
  // for rails with more than one path (SM: one-shot LL, optional one-shot
  // staging, two-shot) every path is timed at sizes 64 KiB .. 4 MiB, ranks
  // agree on the times (max), and each ceiling becomes the largest size of
  // the contiguous run of sizes where that path was fastest. Per rail, the
  // same on every rank; the startup profiles are then measured with it.
  void tunePaths(uint64_t maxb, cudaEvent_t e0, cudaEvent_t e1) {
    if (comm->world == 1) return;
    for (size_t i = 0; i < rails.size(); ++i) {
      nz_rail* r = rails[i];
      if (r->ll_cap == 0 && r->os_cap == 0) continue;
      std::vector<uint64_t> sizes;
      for (uint64_t sz = 64 << 10; sz <= std::min<uint64_t>(uint64_t{4} << 20, maxb); sz *= 2) sizes.push_back(sz);
      if (sizes.empty()) continue;
      // times[k][v]: v = 0 LL, 1 one-shot, 2 two-shot; huge when not applicable.
      std::vector<double> t(sizes.size() * 3, 1e30);
      for (size_t k = 0; k < sizes.size(); ++k) {
        const uint64_t s = sizes[k];
        const uint64_t C = nezha::defaultChunkBytes(s, comm->world, algo);
        for (int v = 0; v < 3; ++v) {
          if ((v == 0 && s > r->ll_cap) || (v == 1 && s > r->os_cap)) continue;
          r->ll_max = v == 0 ? r->ll_cap : 0;
          r->os_max = v == 1 ? r->os_cap : 0;
          for (int w = 0; w < 3; ++w) nz::railAllreduce(r, ub_in, ub_out, 0, s, C, 0, UINT64_MAX, NZ_F32, 0, -1, r->stream);
          NZ_CUDA(cudaEventRecord(e0, r->stream));
          for (int it = 0; it < 20; ++it) nz::railAllreduce(r, ub_in, ub_out, 0, s, C, 0, UINT64_MAX, NZ_F32, 0, -1, r->stream);
          NZ_CUDA(cudaEventRecord(e1, r->stream));
          NZ_CUDA(cudaEventSynchronize(e1));
          float ms = 0;
          NZ_CUDA(cudaEventElapsedTime(&ms, e0, e1));
          t[k * 3 + v] = ms;
        }
      }
      const auto msgs = nz::exchange(comm, t.data(), t.size() * sizeof(double), {});
      for (int rk = 0; rk < comm->world; ++rk) {
        const double* v = reinterpret_cast<const double*>(msgs[rk].data.data());
        for (size_t j = 0; j < t.size(); ++j) t[j] = std::max(t[j], v[j]);
      }
      const auto [ll_max, os_max] = nezha::choosePathCeilings(sizes, t, r->ll_cap, r->os_cap);
      r->ll_max = ll_max;
      r->os_max = os_max;
    }
  }

  void calibrate() {
    const uint64_t maxb = std::max<uint64_t>(cfg.calibrate_max_bytes, 1 << 16);
    ensureUnbound(maxb);
    const int world = comm->world;
    std::vector<uint64_t> sizes;
    for (uint64_t s = 4096; s <= maxb; s *= 4) sizes.push_back(s);
    cudaEvent_t e0 = event(), e1 = event();
    if (cfg.tune_budgets) {
      tuneBudgets(maxb, e0, e1);
      tunePaths(maxb, e0, e1);
    }
    std::vector<nezha::RailProfile> profiles;
    bool measured_any = false;
    for (size_t i = 0; i < specs.size(); ++i) {
      if (specs[i].has_profile) {  // given by the rails config: keep it
        profiles.push_back(specs[i].profile);
        continue;
      }
      measured_any = true;
      nz_rail* r = rails[i];
      std::vector<double> lat;
      for (uint64_t s : sizes) {
        const uint64_t C = nezha::defaultChunkBytes(s, world, algo);
        const int iters = s <= (1u << 20) ? std::max(cfg.calibrate_iters, 4) : std::max(cfg.calibrate_iters / 4, 2);
        for (int w = 0; w < 2; ++w) nz::railAllreduce(r, ub_in, ub_out, 0, s, C, 0, UINT64_MAX, NZ_F32, 0, -1, r->stream);
        NZ_CUDA(cudaEventRecord(e0, r->stream));
        for (int it = 0; it < iters; ++it)
          nz::railAllreduce(r, ub_in, ub_out, 0, s, C, 0, UINT64_MAX, NZ_F32, 0, -1, r->stream);
        NZ_CUDA(cudaEventRecord(e1, r->stream));
        NZ_CUDA(cudaEventSynchronize(e1));
        float ms = 0;
        NZ_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        lat.push_back(static_cast<double>(ms) * 1000.0 / iters);
      }
      // Ranks agree (max), then the samples are made strictly increasing so
      // RailProfile::validate accepts them (types.cpp:44-51).
      if (world > 1) {
        const auto msgs = nz::exchange(comm, lat.data(), lat.size() * sizeof(double), {});
        for (int rk = 0; rk < world; ++rk) {
          const double* v = reinterpret_cast<const double*>(msgs[rk].data.data());
          for (size_t j = 0; j < lat.size(); ++j) lat[j] = std::max(lat[j], v[j]);
        }
      }
      for (size_t j = 1; j < lat.size(); ++j) lat[j] = std::max(lat[j], lat[j - 1] + 1e-3);
      nezha::RailProfile p = specs[i].profile;
      p.rail_id = specs[i].rail_id;
      p.efficiency_points.clear();
      for (size_t j = 0; j < sizes.size(); ++j) p.efficiency_points.emplace_back(sizes[j], lat[j]);
      // (t_setup, B) from calibrate(); the measured
      // points stay as the interpolation table messageLatency() uses.
      const nezha::CalibratedProfile cal = nezha::calibrate(p.rail_id, p.protocol, p.efficiency_points);
      p.t_setup_us = cal.profile.t_setup_us;
      p.bandwidth_bps = cal.profile.bandwidth_bps;
      profiles.push_back(p);
      specs[i].profile = p;
      specs[i].has_profile = true;
    }
    bal->setProfiles(profiles);
    if (measured_any && specs.size() > 1) calibrateConcurrent(sizes, e0);
    if (cfg.sync_overhead_us < 0 && specs.size() > 1) {
      // Fork/join of every rail on 4 KiB each vs the slowest rail alone.
      const uint64_t s = 4096;
      const int iters = 50;
      double single = 0;
      for (auto& sp : specs) single = std::max(single, sp.profile.messageLatency(s));
      cudaStream_t user = io;
      NZ_CUDA(cudaEventRecord(e0, user));
      for (int it = 0; it < iters; ++it) {
        cudaEvent_t f = event();
        NZ_CUDA(cudaEventRecord(f, user));
        std::vector<cudaEvent_t> ends;
        for (size_t i = 0; i < rails.size(); ++i) {
          NZ_CUDA(cudaStreamWaitEvent(rails[i]->stream, f, 0));
          nz::railAllreduce(rails[i], ub_in, ub_out, s * i, s, 65536, 0, UINT64_MAX, NZ_F32, 0, -1, rails[i]->stream);
          cudaEvent_t e = event();
          NZ_CUDA(cudaEventRecord(e, rails[i]->stream));
          NZ_CUDA(cudaStreamWaitEvent(user, e, 0));
          ends.push_back(e);
        }
        NZ_CUDA(cudaStreamSynchronize(user));
        pool.push_back(f);
        for (auto e : ends) pool.push_back(e);
      }
      NZ_CUDA(cudaEventRecord(e1, user));
      NZ_CUDA(cudaEventSynchronize(e1));
      float ms = 0;
      NZ_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      double multi = static_cast<double>(ms) * 1000.0 / iters;
      if (world > 1) {
        const auto msgs = nz::exchange(comm, &multi, sizeof(multi), {});
        for (int rk = 0; rk < world; ++rk) multi = std::max(multi, *reinterpret_cast<const double*>(msgs[rk].data.data()));
      }
      bal->setSyncOverhead(std::max(0.0, multi - single));
    }
    pool.push_back(e0);
    pool.push_back(e1);
  }

  // P13: every rail busy at once on a uniform split of S; rail i's latency
  // for its S/R share under that contention becomes its concurrent profile.
  void calibrateConcurrent(const std::vector<uint64_t>& sizes, cudaEvent_t start) {
    const int world = comm->world;
    const size_t R = specs.size();
    std::vector<std::vector<double>> lat(R);
    std::vector<uint64_t> shares;
    std::vector<cudaEvent_t> ends(R);
    for (auto& e : ends) e = event();
    for (uint64_t S : sizes) {
      const uint64_t share = std::max<uint64_t>((S / R) & ~uint64_t{15}, 16);
      shares.push_back(share);
      const int iters = S <= (1u << 20) ? std::max(cfg.calibrate_iters, 4) : std::max(cfg.calibrate_iters / 4, 2);
      std::vector<double> acc(R, 0.0);
      std::vector<std::pair<int, uint64_t>> segs;
      for (size_t i = 0; i < R; ++i) segs.emplace_back(specs[i].rail_id, share);
      for (int it = 0; it < iters + 1; ++it) {
        NZ_CUDA(cudaEventRecord(start, io));
        auto gates = gatesFor(segs, nullptr);  // the profiles see the same SM arbitration as the ops
        for (size_t i = 0; i < R; ++i) {
          NZ_CUDA(cudaStreamWaitEvent(rails[i]->stream, start, 0));
          const uint64_t C = nezha::defaultChunkBytes(share, world, algo);
          nz::railAllreduce(rails[i], ub_in, ub_out, share * i, share, C, 0, UINT64_MAX, NZ_F32, 0, -1,
                            rails[i]->stream, &gates[i]);
          NZ_CUDA(cudaEventRecord(ends[i], rails[i]->stream));
          NZ_CUDA(cudaStreamWaitEvent(io, ends[i], 0));
        }
        recycleGates();
        NZ_CUDA(cudaStreamSynchronize(io));
        if (it == 0) continue;  // warm-up
        for (size_t i = 0; i < R; ++i) {
          float ms = 0;
          NZ_CUDA(cudaEventElapsedTime(&ms, start, ends[i]));
          acc[i] += static_cast<double>(ms) * 1000.0;
        }
      }
      for (size_t i = 0; i < R; ++i) lat[i].push_back(acc[i] / iters);
    }
    for (auto e : ends) pool.push_back(e);
    std::vector<nezha::RailProfile> conc;
    for (size_t i = 0; i < R; ++i) {
      auto& l = lat[i];
      if (world > 1) {
        const auto msgs = nz::exchange(comm, l.data(), l.size() * sizeof(double), {});
        for (int rk = 0; rk < world; ++rk) {
          const double* v = reinterpret_cast<const double*>(msgs[rk].data.data());
          for (size_t j = 0; j < l.size(); ++j) l[j] = std::max(l[j], v[j]);
        }
      }
      for (size_t j = 1; j < l.size(); ++j) l[j] = std::max(l[j], l[j - 1] + 1e-3);
      nezha::RailProfile p = specs[i].profile;
      p.efficiency_points.clear();
      for (size_t j = 0; j < shares.size(); ++j) {
        if (j && shares[j] <= shares[j - 1]) continue;
        p.efficiency_points.emplace_back(shares[j], l[j]);
      }
      p.t_setup_us = l.front();
      p.bandwidth_bps =
          static_cast<double>(shares.back() - shares.front()) / std::max(1e-9, (l.back() - l.front()) * 1e-6);
      conc.push_back(p);
    }
    bal->setConcurrentProfiles(conc);
  }

  std::string stateJson() {
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
};

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
