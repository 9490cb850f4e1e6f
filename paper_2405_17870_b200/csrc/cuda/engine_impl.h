// nz_engine: state and operations of one rank's multi-rail engine, shared by
// engine.cpp (ops, Timer, C ABI), engine_monitor.cpp (failure monitor,
// reroute, readmit) and engine_calibrate.cpp (startup calibration and
// tuning). Flow and contract: include/nezha/engine.hpp.
#pragma once

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <memory>
#include <mutex>
#include <set>
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

struct nz_engine {
  struct Pending {
    uint32_t op = 0;
    nezha::Plan plan;
    cudaEvent_t start = nullptr;
    std::vector<std::pair<int, cudaEvent_t>> ends;
    std::vector<std::pair<int, uint32_t>> tags;  // (rail index, entry tag) of monitored segments
    bool skip = false;  // an op that lost a rail is not a Timer sample
  };

  // One rail's part of one op, watched by the monitor until it retires
  // (DESIGN.md §6b). The geometry is what a reroute re-reduces.
  struct Entry {
    uint32_t op = 0;
    int rail = 0;  // index into rails
    uint32_t tag = 0;
    nz_buf* in = nullptr;
    nz_buf* out = nullptr;
    uint64_t seg_off = 0, seg_len = 0, chunk = 0, chunk_end = 0;
    int dtype = NZ_F32;
    bool ll = false;  // one-shot LL path (no end barrier: a timeout does not imply the others' data)
    nezha::Plan plan;
    cudaEvent_t end = nullptr;
  };

  // A table change agreed by every rank, applied before op `activation` is
  // planned (so every rank plans every op against the same table).
  struct TableEvent {
    uint32_t activation = 0;
    int rail_id = 0;
  };

  nz_comm* comm = nullptr;
  nz_engine_config_t cfg{};
  std::vector<nezha::RailSpec> specs;  // sorted by rail_id
  std::vector<nz_rail*> rails;         // parallel to specs
  std::vector<nz_rail*> twins;         // recovery twin per rail (monitor only), parallel to specs
  std::unique_ptr<nezha::Balancer> bal;  // owned by the issuing thread
  std::unique_ptr<nezha::HealthMonitor> health;  // owned by the monitor thread (under mu)
  nezha::Algorithm algo = nezha::Algorithm::RingChunked;
  uint32_t op_seq = 0;
  std::deque<Pending> pending;
  std::vector<cudaEvent_t> pool;
  std::map<uint32_t, std::pair<int, uint64_t>> inject;
  cudaStream_t ctrl = nullptr;
  cudaStream_t io = nullptr;
  cudaStream_t h2d = nullptr;  // host path: uploads of the next piece
  cudaStream_t d2h = nullptr;  // host path: downloads of the previous piece
  // Loopback ranks share the process's legacy stream, so a NULL caller
  // stream means this rank's own stream instead (a stream gate of one rank
  // must not hold up another rank's work).
  cudaStream_t loop_user = nullptr;
  cudaEvent_t loop_ev = nullptr;
  cudaStream_t callerStream(void* stream) {
    if (stream) return static_cast<cudaStream_t>(stream);
    if (!loop_user) return cudaStreamLegacy;
    // Work this thread put on the legacy stream (e.g. the copy that filled
    // the input) comes first.
    NZ_CUDA(cudaEventRecord(loop_ev, cudaStreamLegacy));
    NZ_CUDA(cudaStreamWaitEvent(loop_user, loop_ev, 0));
    return loop_user;
  }
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
  int64_t clock_offset_ns = 0;  // %globaltimer - CLOCK_REALTIME
  // A launch waiting at its start barrier keeps beating this long (peers'
  // hosts may be late); NEZHA_START_GRACE_US, default 1 s.
  double start_grace_us = 1e6;
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

  // ---- failure monitor (engine_monitor.cpp) ----
  bool monitored = false;  // cfg.monitor and world > 1
  std::string mon_off_reason;
  std::mutex mu;           // everything below, shared by the two threads
  std::condition_variable cv;
  std::deque<Entry> inflight;                 // issue order
  std::vector<cudaEvent_t> entry_pool;        // retired entry events
  std::deque<TableEvent> table_events;        // agreed, not yet applied
  std::set<int> agreed_failed;                // rail ids failed by agreement
  std::set<uint32_t> lost_ops;                // ops whose result needed a reroute
  uint32_t issued = 0;                        // ops planned by the issuing thread
  bool agreeing = false;                      // the monitor is agreeing: planning waits
  bool mon_stop = false;
  std::string mon_error;                      // surfaced at the next synchronize
  std::vector<nz_failover_report_t> reports;  // every failover, in order
  std::deque<Entry> retired_ok;               // recent successes (a peer may ask about them)
  std::thread mon;
  uint64_t* rec_stamps_host = nullptr;  // [0] resume, [1] done of the current reroute
  uint64_t* rec_stamps_dev = nullptr;

  int index(int rail_id) const {
    for (size_t i = 0; i < specs.size(); ++i)
      if (specs[i].rail_id == rail_id) return static_cast<int>(i);
    nz::fail(NZ_ERR_INVALID, "unknown rail " + std::to_string(rail_id));
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
  std::vector<std::pair<int, nezha::Micros>> agree(const std::vector<std::pair<int, nezha::Micros>>& mine);

  void harvest(uint32_t upto);

  void drainTimer() { harvest(UINT32_MAX - 8); }

  // Computation-phase gates of one concurrent launch of `segs` (rail_id,
  // length) in rail order; empty when the pool is off. The release events go
  // back to the event pool once the launch is enqueued (waits are captured at
  // cudaStreamWaitEvent time).
  std::vector<nz::ComputeGate> gatesFor(const std::vector<std::pair<int, uint64_t>>& segs, std::string* log);
  std::vector<cudaEvent_t> pool_pending;  // gate events of the launch being enqueued
  void recycleGates();

  // One op (piece) of at most 1 GiB at byte offset `base`.
  void op(nz_buf* in, nz_buf* out, uint64_t base, uint64_t len, int dtype, cudaStream_t user);
  // One rail segment of an op: launches, entry for the monitor, stream gate.
  void launchSegment(uint32_t seq, const nezha::Plan& plan, const nezha::RailSegment& rs, nz_buf* in, nz_buf* out,
                     uint64_t base, int dtype, cudaStream_t st, nz::ComputeGate* gate, bool capturing,
                     cudaStream_t user, cudaEvent_t* end_out, Pending* p);

  void recordPlan(uint32_t seq, uint64_t base, uint64_t len, nezha::Plan&& plan, std::string&& grants = {});

  std::string planRecordJson(const PlanRecord& r) const;

  static int64_t realtimeNs();

  // %globaltimer vs host CLOCK_REALTIME: best of 5 stamp round trips. Lets
  // the reports place host-side detection on the device timeline.
  void calibrateClock();

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
              cudaStream_t user);

  // Collective point: every rank calls it at the same place in its op stream.
  void synchronize();

  void ensureUnbound(uint64_t bytes);

  // ---- monitor thread (engine_monitor.cpp) ----
  void startMonitor();
  void stopMonitor();
  void monitorLoop();
  // One agreement (two rounds on the monitor channel): the ranks propose
  // their failed front entry (`own`, or nullptr when joining a peer), settle
  // the earliest proposed one — orphan, P9 target, reroute on the target's
  // twin, gate release, report — and return whether it was `own`.
  bool failover(const Entry* own, int64_t seen_ns);
  // Joins a peer's agreement on an entry this rank already retired.
  void serviceRequests();
  // Applies agreed table events due before planning op `seq` (issuing thread).
  void applyTableEvents(uint32_t seq);
  // Waits until every entry issued so far retired or was rerouted.
  void drainMonitor();
  // SPEC.md:398-406 with probes on the rail (collective).
  void readmit(int rail_id);

  // Startup calibration: each rail alone over a size sweep, then the
  // coordination cost of a fork/join over all rails.
  // CTA budget of the SM-driven rails, measured instead of assumed: each
  // candidate grid runs the two-shot path at one large size, ranks agree on
  // the times (max), the fastest wins (ties within 3 % go to the smaller
  // grid). Rails whose budget the config pins are left alone. The chosen
  // grids then hold for calibration and every op, identically on all ranks.
  void tuneBudgets(uint64_t maxb, cudaEvent_t e0, cudaEvent_t e1);

  // Which protocol a rail uses at which size, measured instead of assumed:
  // for rails with an LL path (SM) both paths are timed at sizes 64 KiB ..
  // 4 MiB, ranks agree on the times (max), and the LL ceiling becomes the
  // largest size of the contiguous run of sizes where LL was fastest.
  void tunePaths(uint64_t maxb, cudaEvent_t e0, cudaEvent_t e1);

  void calibrate();

  // P13: every rail busy at once on a uniform split of S; rail i's latency
  // for its S/R share under that contention becomes its concurrent profile.
  void calibrateConcurrent(const std::vector<uint64_t>& sizes, cudaEvent_t start);

  std::string stateJson();
};
