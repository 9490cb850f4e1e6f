// nz_engine: state and operations of one rank's multi-rail engine, shared by
// engine.cpp (ops, Timer, faults, C ABI) and engine_calibrate.cpp (startup
// calibration and tuning). Flow and contract: include/nezha/engine.hpp.
#pragma once

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

  std::vector<int> healthyIds() const { return health->healthyRails(); }

  void finishFailoverReport();

  // Computation-phase gates of one concurrent launch of `segs` (rail_id,
  // length) in rail order; empty when the pool is off. The release events go
  // back to the event pool once the launch is enqueued (waits are captured at
  // cudaStreamWaitEvent time).
  std::vector<nz::ComputeGate> gatesFor(const std::vector<std::pair<int, uint64_t>>& segs, std::string* log);
  std::vector<cudaEvent_t> pool_pending;  // gate events of the launch being enqueued
  void recycleGates();

  // One op (piece) of at most 1 GiB at byte offset `base`.
  void op(nz_buf* in, nz_buf* out, uint64_t base, uint64_t len, int dtype, cudaStream_t user);

  void recordPlan(uint32_t seq, uint64_t base, uint64_t len, nezha::Plan&& plan, std::string&& grants = {});

  std::string planRecordJson(const PlanRecord& r) const;

  // Exception handler: wait for the device's fault record,
  // mark the rail Failed, pick the target (P9) and run the orphan chunks on
  // it with the failed segment's geometry (P10), after its current task.
  static int64_t realtimeNs();

  // %globaltimer vs host CLOCK_REALTIME: best of 5 stamp round trips. Lets
  // the report place the host monitor's detection on the device timeline.
  void calibrateClock();

  void handoff(Pending& p, const nezha::Plan& plan, const nezha::Segment& seg, int rid, uint64_t k, nz_buf* in,
               nz_buf* out, uint64_t base, int dtype);

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

  // Startup calibration: each rail alone over a size sweep, then the
  // coordination cost of a fork/join over all rails.
  // CTA budget of the SM-driven rails, measured instead of assumed: each
  // candidate grid runs the two-shot path at one large size, ranks agree on
  // the times (max), the fastest wins (ties within 3 % go to the smaller
  // grid). Rails whose budget the config pins are left alone. The chosen
  // grids then hold for calibration and every op, identically on all ranks.
  void tuneBudgets(uint64_t maxb, cudaEvent_t e0, cudaEvent_t e1);

  // Which protocol a rail uses at which size, measured instead of assumed:
  // for rails with more than one path (SM: one-shot LL, optional one-shot
  // staging, two-shot) every path is timed at sizes 64 KiB .. 4 MiB, ranks
  // agree on the times (max), and each ceiling becomes the largest size of
  // the contiguous run of sizes where that path was fastest. Per rail, the
  // same on every rank; the startup profiles are then measured with it.
  void tunePaths(uint64_t maxb, cudaEvent_t e0, cudaEvent_t e1);

  void calibrate();

  // P13: every rail busy at once on a uniform split of S; rail i's latency
  // for its S/R share under that contention becomes its concurrent profile.
  void calibrateConcurrent(const std::vector<uint64_t>& sizes, cudaEvent_t start);

  std::string stateJson();
};

