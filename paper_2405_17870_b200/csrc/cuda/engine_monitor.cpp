// Failure monitor of the engine (the paper's
// Exception Handler).
//
// One thread per rank watches every rail launch sequence the engine issued
// (an Entry per rail per op), strictly in issue order, through the launch
// status the kernels publish into mapped host memory:
//   * retired with its tag in the rail's status: success, heartbeat;
//   * retired without it: the rail failed on this rank for this op — a peer
//     never reached the end barrier (the device gave up after the detection
//     budget), or this rank's link died (injected stall), or the host aborted
//     a wait (below). Every rank sees the same failure, since no rank's
//     launch can succeed without every rank's arrival;
//   * started but not retired for longer than the heartbeat budget
//     (Suspect then Failed): the monitor sets the rail's
//     abort word and the kernel leaves its wait, i.e. the case above.
// On a failure the ranks' monitors agree over their own control channel on
// the orphan — the chunks after the minimum, over ranks, of the chunks each
// rank completed — and on the op index from which the planner
// stops using the rail. Each then re-reduces the orphan on the recovery twin
// of the P9 target (same kernels, own barrier pads and stream, so it cannot
// interleave with the issuing thread's launches on that rail) with the failed
// segment's geometry, and finally writes the failed op's tag into the failed
// rail's gate word: the caller's stream, which waits on that word, resumes.
// The issuing thread never blocks on any of this.
#include "engine_impl.h"

using nz::fail;

namespace {

// Round 1 of an agreement: the entry this rank wants agreed (its failed
// front), or none (it joins a peer's request). The subject is the earliest
// proposed entry in issue order (op, then rail order).
struct Proposal {
  uint32_t op;
  int32_t rail_index;
  int32_t rail_id;
  uint32_t tag;
  int32_t valid;
  int32_t pad;
};

// Round 2: this rank's outcome of the subject.
struct AgreeMsg {
  uint32_t op;
  int32_t rail_id;
  uint32_t tag;
  uint32_t issued;
  uint64_t prog;    // chunks [0, prog) of the segment complete on this rank
  int64_t t_fail;   // host-clock ns of this rank's link death, 0 = none
  int64_t t_det;    // host-clock ns of this rank's device-side detection, 0 = none
  int32_t ok;       // the entry succeeded on this rank (it joined a peer's agreement)
  int32_t pad;
};

double nowUs() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

void nz_engine::calibrateClock() {
  // Only the monitor (or the creating thread before it starts) calls this.
  int64_t best = INT64_MAX;
  volatile uint64_t* slot = rec_stamps_host + 2;
  for (int i = 0; i < 5; ++i) {
    *slot = 0;
    const int64_t t0 = realtimeNs();
    nz::launchStamp(rec_stamps_dev + 2, ctrl);
    NZ_CUDA(cudaStreamSynchronize(ctrl));
    const int64_t t1 = realtimeNs();
    if (t1 - t0 < best) {
      best = t1 - t0;
      clock_offset_ns = static_cast<int64_t>(*slot) - (t0 + t1) / 2;
    }
  }
}

void nz_engine::startMonitor() {
  monitored = cfg.monitor != 0 && comm->world > 1;
  if (!monitored) return;
  if (const char* g = getenv("NEZHA_START_GRACE_US")) start_grace_us = std::max(0.0, atof(g));
  // The stream gates are CUDA stream memory operations: check once that the
  // driver takes them (a wait that is already satisfied, then a write) on
  // every rank; without them the engine runs unmonitored (round-1 behaviour:
  // a failed rail raises ChannelDownError at nz_engine_synchronize).
  int32_t ok = 1;
  {
    nz_rail* r = rails.front();
    const CUstream st = reinterpret_cast<CUstream>(ctrl);
    if (!NZ_DRV(cuStreamWaitValue32) || !NZ_DRV(cuStreamWriteValue32) ||
        NZ_DRV(cuStreamWaitValue32)(st, nz::railGateAddr(r), 0, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS ||
        NZ_DRV(cuStreamWriteValue32)(st, nz::railGateAddr(r), r->tag, 0) != CUDA_SUCCESS ||
        cudaStreamSynchronize(ctrl) != cudaSuccess) {
      ok = 0;
      cudaGetLastError();
    }
  }
  const auto all = nz::exchange(comm, &ok, sizeof(ok), {});
  for (const auto& m : all) ok &= *reinterpret_cast<const int32_t*>(m.data.data());
  if (!ok) {
    monitored = false;
    mon_off_reason = "CUDA stream memory operations unavailable";
    return;
  }
  // Twins run rarely (a reroute) but beside the main rails' kernels: a small
  // CTA budget keeps every spinning kernel of the GPU co-resident (§3).
  for (auto& s : specs)
    twins.push_back(nz::railCreate(comm, s.kind, s.rail_id, s.kind == NZ_RAIL_CE ? s.sm_budget : 32, false, true));
  for (size_t i = 0; i < twins.size(); ++i) twins[i]->detect_us = cfg.detect_us;
  mon = std::thread([this] { monitorLoop(); });
}

void nz_engine::stopMonitor() {
  {
    std::lock_guard<std::mutex> lk(mu);
    mon_stop = true;
  }
  cv.notify_all();
  if (mon.joinable()) mon.join();
}

void nz_engine::applyTableEvents(uint32_t seq) {
  if (!monitored) return;
  std::unique_lock<std::mutex> lk(mu);
  cv.wait(lk, [&] { return !agreeing || mon_stop; });
  issued = seq + 1;
  while (!table_events.empty() && static_cast<int32_t>(table_events.front().activation - seq) <= 0) {
    const TableEvent ev = table_events.front();
    table_events.pop_front();
    if (bal->healthy(ev.rail_id)) bal->markFailed(ev.rail_id);
  }
}

void nz_engine::drainMonitor() {
  std::unique_lock<std::mutex> lk(mu);
  cv.wait(lk, [&] { return inflight.empty() || mon_stop || !mon_error.empty(); });
}

void nz_engine::monitorLoop() {
  cudaSetDevice(comm->device);
  const double hb = cfg.heartbeat_us;
  auto last_clock = std::chrono::steady_clock::now();
  uint64_t beat_key = ~0ull;  // (rail, tag) of the entry whose start was fed to the heartbeat clock
  for (;;) {
    Entry front;
    bool recal = false;
    {
      std::unique_lock<std::mutex> lk(mu);
      if (mon_stop) return;
      if (inflight.empty()) {
        const double now = nowUs();
        for (auto& s : specs)
          if (!agreed_failed.count(s.rail_id)) health->heartbeat(s.rail_id, now);
        recal = std::chrono::steady_clock::now() - last_clock > std::chrono::seconds(1);
      } else {
        front = inflight.front();
      }
    }
    // A peer's agreement request is answered even while this rank is idle
    // (its entries all retired): the peer's failover waits on it.
    try {
      serviceRequests();
    } catch (const std::exception& e) {
      std::lock_guard<std::mutex> lk(mu);
      if (mon_error.empty()) mon_error = e.what();
    }
    if (!front.end) {
      if (recal) {  // idle: re-anchor %globaltimer against the host clock
        try {
          calibrateClock();
        } catch (const std::exception&) {
        }
        last_clock = std::chrono::steady_clock::now();
      } else {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait_for(lk, std::chrono::microseconds(200), [&] { return mon_stop || !inflight.empty(); });
      }
      continue;
    }
    const cudaError_t q = cudaEventQuery(front.end);
    if (q == cudaErrorNotReady) {
      // Heartbeats: every rail beats unless its oldest
      // launch started and has not retired; a rail past the budget is
      // aborted so its kernels leave their waits and the failure path runs.
      const volatile nz_rail_status_t* st = rails[front.rail]->status_host;
      const bool started = st->start_tag == front.tag;
      // Running: this launch passed its start barrier (every rank arrived)
      // after it started, so data is moving and a stop means a broken rail.
      const uint64_t t_start = st->t_start_ns, t_run = st->t_run_ns;
      const bool running = started && st->run_tag == front.tag && static_cast<int64_t>(t_run - t_start) >= 0;
      const double now = nowUs();
      std::vector<int> aborted;
      {
        std::lock_guard<std::mutex> lk(mu);
        for (size_t i = 0; i < specs.size(); ++i) {
          if (agreed_failed.count(specs[i].rail_id)) continue;
          if (static_cast<int>(i) == front.rail && started) {
            // Its last sign of life is the start of the launch it is in, or
            // the moment every rank was in: missed beats count from there,
            // not from queueing time. A launch still waiting for peers at its
            // start barrier is not the rail failing — a peer's host may just
            // be late (stragglers) — so it keeps beating through the start
            // grace and only then starts missing beats.
            const int64_t t0 = static_cast<int64_t>(running ? t_run : t_start) - clock_offset_ns;
            const double age_us = std::max(0.0, static_cast<double>(realtimeNs() - t0) / 1000.0);
            if (!running && age_us < start_grace_us) {
              health->heartbeat(specs[i].rail_id, now);
              continue;
            }
            const uint64_t key = (static_cast<uint64_t>(front.rail) << 33) | (static_cast<uint64_t>(running) << 32) |
                                 front.tag;
            if (key != beat_key) {
              health->heartbeat(specs[i].rail_id, now - (running ? age_us : age_us - start_grace_us));
              beat_key = key;
            }
            continue;
          }
          health->heartbeat(specs[i].rail_id, now);
        }
        // A two-shot launch left by its rank at the start barrier cannot
        // complete anywhere (this rank never reaches the end barrier), so the
        // abort keeps the ranks' outcomes equal; an LL launch is never
        // aborted on a heartbeat (see kernels.cuh ll_body).
        for (int id : health->tick(now))
          if (health->state(id).status == nezha::HealthStatus::Failed && !(id == specs[front.rail].rail_id && front.ll))
            aborted.push_back(id);
      }
      for (int id : aborted) reinterpret_cast<volatile nz_rail_status_t*>(rails[index(id)]->status_host)->abort = 1;
      if (started) {
        std::this_thread::yield();  // a launch is running: poll tightly (detection latency)
      } else {
        std::this_thread::sleep_for(std::chrono::microseconds(20));
      }
      (void)hb;
      continue;
    }
    const int64_t seen = realtimeNs();
    if (q != cudaSuccess) {
      std::lock_guard<std::mutex> lk(mu);
      mon_error = std::string("device error while monitoring: ") + cudaGetErrorString(q);
      mon_stop = true;
      cv.notify_all();
      return;
    }
    const volatile nz_rail_status_t* st = rails[front.rail]->status_host;
    const bool ok = static_cast<int32_t>(st->ok_tag - front.tag) >= 0;
    if (!ok) {
      try {
        // Agreements run in issue order: an earlier entry a peer proposes is
        // settled first, then this one is proposed again.
        while (!failover(&front, seen)) {
        }
      } catch (const std::exception& e) {
        // The caller's stream must not stay gated: release it, report at sync.
        NZ_DRV(cuStreamWriteValue32)(reinterpret_cast<CUstream>(ctrl), nz::railGateAddr(rails[front.rail]), front.tag, 0);
        cudaStreamSynchronize(ctrl);
        std::lock_guard<std::mutex> lk(mu);
        if (mon_error.empty()) mon_error = e.what();
        agreeing = false;
      }
    } else {
      std::lock_guard<std::mutex> lk(mu);
      health->heartbeat(specs[front.rail].rail_id, nowUs());
      retired_ok.push_back(front);
      retired_ok.back().end = nullptr;
      if (retired_ok.size() > 4096) retired_ok.pop_front();
    }
    {
      std::lock_guard<std::mutex> lk(mu);
      inflight.pop_front();
      entry_pool.push_back(front.end);
    }
    cv.notify_all();
  }
}

void nz_engine::serviceRequests() {
  std::vector<std::vector<char>> reqs;
  while (nz::peekExchange(comm, nz::kChanMonitor, &reqs)) {
    // Join only once this rank retired a proposed entry: then it can answer
    // for it and for any earlier entry (all retired here, and every one that
    // failed here was agreed before). Otherwise it reaches the entry in issue
    // order and proposes or joins then.
    bool past = false;
    for (const auto& req : reqs) {
      Proposal m{};
      if (req.size() != sizeof(m)) fail(NZ_ERR_SYSTEM, "monitor agreement: bad request");
      std::memcpy(&m, req.data(), sizeof(m));
      if (!m.valid) continue;
      std::lock_guard<std::mutex> lk(mu);
      for (auto it = retired_ok.rbegin(); it != retired_ok.rend() && !past; ++it)
        past = it->op == m.op && it->rail == m.rail_index && it->tag == m.tag;
    }
    if (!past) return;
    failover(nullptr, realtimeNs());
  }
}

bool nz_engine::failover(const Entry* own, int64_t seen_ns) {
  Proposal prop{};
  if (own) {
    prop.op = own->op;
    prop.rail_index = own->rail;
    prop.rail_id = specs[own->rail].rail_id;
    prop.tag = own->tag;
    prop.valid = 1;
  }
  {
    std::lock_guard<std::mutex> lk(mu);
    agreeing = true;  // planning waits: the table switch lands at an op index every rank agrees on
  }
  const auto props = nz::exchange(comm, &prop, sizeof(prop), {}, nz::kChanMonitor);
  Proposal subj{};
  for (const auto& m : props) {
    Proposal o{};
    if (m.data.size() != sizeof(o)) fail(NZ_ERR_SYSTEM, "monitor agreement: bad proposal");
    std::memcpy(&o, m.data.data(), sizeof(o));
    if (!o.valid) continue;
    if (!subj.valid || static_cast<int32_t>(o.op - subj.op) < 0 || (o.op == subj.op && o.rail_index < subj.rail_index))
      subj = o;
  }
  if (!subj.valid) fail(NZ_ERR_SYSTEM, "monitor agreement: nobody proposed an entry");
  const bool mine_is_subject = own && own->op == subj.op && own->rail == subj.rail_index && own->tag == subj.tag;
  Entry e;
  bool ok_here = false;
  if (mine_is_subject) {
    e = *own;
  } else {
    bool found = false;
    {
      std::lock_guard<std::mutex> lk(mu);
      for (auto it = retired_ok.rbegin(); it != retired_ok.rend() && !found; ++it) {
        if (it->op == subj.op && it->rail == subj.rail_index && it->tag == subj.tag) {
          e = *it;
          found = true;
        }
      }
    }
    if (!found)
      fail(NZ_ERR_SYSTEM, "monitor agreement: op " + std::to_string(subj.op) + " rail " + std::to_string(subj.rail_id) +
                              " is neither this rank's failure nor among its retired successes");
    ok_here = true;
  }
  nz_rail* fr = rails[e.rail];
  const int rail_id = specs[e.rail].rail_id;
  const volatile nz_rail_status_t* st = fr->status_host;
  AgreeMsg mine{};
  mine.op = e.op;
  mine.rail_id = rail_id;
  mine.tag = e.tag;
  mine.ok = ok_here ? 1 : 0;
  if (ok_here) {
    mine.prog = e.chunk_end;
  } else {
    mine.prog = st->prog_tag == e.tag ? std::min<uint64_t>(static_cast<uint64_t>(st->prog_chunk), e.chunk_end) : 0;
    mine.t_fail = st->fail_tag == e.tag && st->t_fail_ns ? static_cast<int64_t>(st->t_fail_ns) - clock_offset_ns : 0;
    mine.t_det = st->det_tag == e.tag && st->t_det_ns ? static_cast<int64_t>(st->t_det_ns) - clock_offset_ns : 0;
  }
  {
    std::lock_guard<std::mutex> lk(mu);
    mine.issued = issued;
  }
  const auto msgs = nz::exchange(comm, &mine, sizeof(mine), {}, nz::kChanMonitor);
  uint64_t k = mine.prog;
  uint32_t activation = mine.issued;
  int64_t t_fail = 0, t_det_first = 0;
  int oks = 0;
  for (const auto& m : msgs) {
    AgreeMsg o{};
    if (m.data.size() != sizeof(o)) fail(NZ_ERR_SYSTEM, "monitor agreement: bad message");
    std::memcpy(&o, m.data.data(), sizeof(o));
    if (o.op != mine.op || o.rail_id != mine.rail_id || o.tag != mine.tag)
      fail(NZ_ERR_SYSTEM, "monitor agreement: ranks disagree on the failed op (op " + std::to_string(mine.op) +
                              " rail " + std::to_string(rail_id) + " vs op " + std::to_string(o.op) + " rail " +
                              std::to_string(o.rail_id) + ")");
    k = std::min(k, o.prog);
    oks += o.ok;
    if (static_cast<int32_t>(o.issued - activation) > 0) activation = o.issued;
    if (o.t_fail && (!t_fail || o.t_fail < t_fail)) t_fail = o.t_fail;
    if (o.t_det && (!t_det_first || o.t_det < t_det_first)) t_det_first = o.t_det;
  }
  // Every rank takes the same decision from the same messages: the rail is
  // failed by agreement from `activation` on, and its launches on this rank
  // stop waiting from now on (abort), so launches already issued on it fail
  // on every rank alike.
  std::vector<int> healthy;
  {
    std::lock_guard<std::mutex> lk(mu);
    agreed_failed.insert(rail_id);
    table_events.push_back(TableEvent{activation, rail_id});
    lost_ops.insert(e.op);
    health->channelDown(rail_id);
    agreeing = false;
    for (auto& s : specs)
      if (!agreed_failed.count(s.rail_id)) healthy.push_back(s.rail_id);
  }
  cv.notify_all();
  reinterpret_cast<volatile nz_rail_status_t*>(fr->status_host)->abort = 1;
  nz_failover_report_t rep{};
  rep.op_seq = e.op;
  rep.failed_rail = rail_id;
  rep.target_rail = -1;
  rep.orphan_offset = e.seg_off + e.seg_len;
  rep.stalled_here = mine.t_fail ? 1 : 0;
  if (oks > 0) {
    // Some rank passed the op's end barrier: every rank had arrived, i.e.
    // every store of the op landed everywhere (two-shot, NVLS, CE). Nothing
    // to reroute; the ranks that gave up early just release their callers.
    // The LL path folds locally after its last wait, so there a rank that
    // gave up still lacks its sum: that mix is reported, not hidden.
    if (!ok_here) {
      NZ_CU(NZ_DRV(cuStreamWriteValue32)(reinterpret_cast<CUstream>(ctrl), nz::railGateAddr(fr), e.tag, 0));
      NZ_CUDA(cudaStreamSynchronize(ctrl));
      if (e.ll)
        fail(NZ_ERR_UNRECOVERABLE, "op " + std::to_string(e.op) + ": LL path on rail " + std::to_string(rail_id) +
                                       " completed on some ranks only (a peer came back after the watchdog)");
    }
    rep.orphan_chunk = e.chunk_end;
    std::lock_guard<std::mutex> lk(mu);
    reports.push_back(rep);
    return mine_is_subject;
  }
  const auto target = nezha::chooseHandoffTarget(e.plan, rail_id, healthy);
  if (!target) fail(NZ_ERR_UNRECOVERABLE, "no surviving rail to take over the orphaned segment");
  nz_rail* tw = twins[index(*target)];
  const nezha::Segment orphan = nezha::orphanOf(nezha::Segment{e.seg_off, e.seg_len}, e.chunk, k);
  // Reroute (P9/P10): the orphan chunks on the target's twin with the failed
  // segment's geometry, so order-controlled rails reproduce the same bits.
  volatile uint64_t* stamps = rec_stamps_host;
  stamps[0] = 0;
  stamps[1] = 0;
  nz::launchStamp(rec_stamps_dev + 0, tw->stream);
  uint32_t tag2 = 0;
  if (orphan.length > 0) {
    nz::RailOp o;
    o.in = e.in;
    o.out = e.out;
    o.seg_off = e.seg_off;
    o.seg_len = e.seg_len;
    o.chunk_bytes = e.chunk;
    o.chunk_begin = k;
    o.chunk_end = e.chunk_end;
    o.dtype = e.dtype;
    o.op_seq = e.op;
    o.st = tw->stream;
    tag2 = nz::railRun(tw, o);
  }
  nz::launchStamp(rec_stamps_dev + 1, tw->stream);
  NZ_CU(NZ_DRV(cuStreamWriteValue32)(reinterpret_cast<CUstream>(tw->stream), nz::railGateAddr(fr), e.tag, 0));
  NZ_CUDA(cudaStreamSynchronize(tw->stream));
  if (tag2 && static_cast<int32_t>(tw->status_host->ok_tag - tag2) < 0)
    fail(NZ_ERR_UNRECOVERABLE, "the reroute of op " + std::to_string(e.op) + " failed on rail " + std::to_string(*target));
  rep.target_rail = *target;
  rep.orphan_offset = orphan.offset;
  rep.orphan_length = orphan.length;
  rep.orphan_chunk = k;
  // All times on the shared host clock (each rank maps its %globaltimer).
  const double f = static_cast<double>(t_fail ? t_fail : (t_det_first ? t_det_first : seen_ns));
  const double resume = static_cast<double>(static_cast<int64_t>(stamps[0]) - clock_offset_ns);
  const double done = static_cast<double>(static_cast<int64_t>(stamps[1]) - clock_offset_ns);
  rep.host_detect_us = (static_cast<double>(seen_ns) - f) / 1000.0;
  rep.detect_us = rep.host_detect_us;
  rep.device_detect_us = mine.t_det ? (static_cast<double>(mine.t_det) - f) / 1000.0 : 0.0;
  rep.resume_us = (resume - f) / 1000.0;
  rep.done_us = (done - f) / 1000.0;
  rep.resume_after_detect_us = (resume - static_cast<double>(seen_ns)) / 1000.0;
  std::lock_guard<std::mutex> lk(mu);
  reports.push_back(rep);
  return mine_is_subject;
}

void nz_engine::readmit(int rail_id) {
  const int idx = index(rail_id);
  synchronize();
  {
    std::lock_guard<std::mutex> lk(mu);
    if (monitored && !agreed_failed.count(rail_id)) fail(NZ_ERR_INVALID, "readmit: rail is not failed");
  }
  if (!monitored && bal->healthy(rail_id)) fail(NZ_ERR_INVALID, "readmit: rail is not failed");
  nz_rail* r = rails[idx];
  nz::railRevive(r, nullptr);  // its twin is the monitor's and never failed with it
  // the rail must keep beating for the hold period before it
  // carries data again. A beat is a probe allreduce on the rail that
  // succeeded on every rank.
  ensureUnbound(1 << 16);
  const double hold = cfg.readmit_hold_us;
  double t_first = -1;  // first successful probe: the start of the healthy streak
  for (;;) {
    nz::RailOp o;
    o.in = ub_in;
    o.out = ub_out;
    o.seg_off = 0;
    o.seg_len = 4096;
    o.chunk_bytes = 4096;
    o.dtype = NZ_I32;
    o.st = r->stream;
    const uint32_t tag = nz::railRun(r, o);
    NZ_CUDA(cudaStreamSynchronize(r->stream));
    int32_t ok = tag == 0 || static_cast<int32_t>(r->status_host->ok_tag - tag) >= 0 ? 1 : 0;
    if (comm->world > 1) {
      const auto msgs = nz::exchange(comm, &ok, sizeof(ok), {});
      for (const auto& m : msgs) ok &= *reinterpret_cast<const int32_t*>(m.data.data());
    }
    if (!ok) fail(NZ_ERR_RAIL_DOWN, "readmit: probe allreduce on rail " + std::to_string(rail_id) + " failed");
    const double now = nowUs();
    if (t_first < 0) t_first = now;
    {
      std::lock_guard<std::mutex> lk(mu);
      health->heartbeat(rail_id, now);
    }
    // Every rank leaves the loop after the same number of probes.
    int32_t done = now - t_first >= hold ? 1 : 0;
    if (comm->world > 1) {
      const auto msgs = nz::exchange(comm, &done, sizeof(done), {});
      for (const auto& m : msgs) done &= *reinterpret_cast<const int32_t*>(m.data.data());
    }
    if (done) break;
    const double left = hold - (now - t_first);
    std::this_thread::sleep_for(
        std::chrono::microseconds(static_cast<int64_t>(std::clamp(left, 0.0, cfg.heartbeat_us / 2))));
  }
  {
    std::lock_guard<std::mutex> lk(mu);
    if (health->state(rail_id).status == nezha::HealthStatus::Failed) {
      // The streak started at the first successful probe (after channelDown).
      const double now = nowUs();
      health->readmit(rail_id, now, std::min(hold, now - t_first));
    }
    agreed_failed.erase(rail_id);
    for (auto it = table_events.begin(); it != table_events.end();)
      it = it->rail_id == rail_id ? table_events.erase(it) : std::next(it);
  }
  if (!bal->healthy(rail_id)) bal->readmit(rail_id);
}
