// Internal definitions shared by the CUDA translation units of libnezha_b200.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

#include "nezha_b200.h"

namespace nz {

constexpr int kMaxRanks = 8;     // one NVSwitch box
constexpr int kMaxCtas = 1024;   // barrier slots per rail
constexpr int kThreads = 512;    // CTA size of the data kernels
constexpr size_t kPadBytes = size_t(kMaxCtas) * kMaxRanks * sizeof(uint32_t);  // per rail
constexpr int kMaxRails = 16;    // pads carved from the control buffer

// Error plumbing: C++ exceptions inside, codes + thread-local text outside.
struct ApiError : std::runtime_error {
  ApiError(int code, const std::string& what) : std::runtime_error(what), code(code) {}
  int code;
};
void setLastError(const std::string& msg);
[[noreturn]] void fail(int code, const std::string& msg);
void checkCuda(cudaError_t e, const char* what);
void checkCu(CUresult e, const char* what);

#define NZ_CUDA(x) ::nz::checkCuda((x), #x)
#define NZ_CU(x) ::nz::checkCu((x), #x)

// Driver API entry points, resolved through cudaGetDriverEntryPoint so the
// library itself has no link-time dependency on libcuda (it loads, and its
// exports can be checked, on a machine without a GPU driver).
struct DriverApi {
#define NZ_DRV_FN(name) decltype(&::name) name = nullptr;
#include "driver_fns.inc"
#undef NZ_DRV_FN
};
const DriverApi& drv();
#define NZ_DRV(fn) (::nz::drv().fn)

// Runs `fn`, mapping exceptions to ABI codes.
template <typename F>
int guarded(F&& fn) {
  try {
    fn();
    return NZ_OK;
  } catch (const ApiError& e) {
    setLastError(e.what());
    return e.code;
  } catch (const std::invalid_argument& e) {
    setLastError(e.what());
    return NZ_ERR_INVALID;
  } catch (const std::exception& e) {
    setLastError(e.what());
    return NZ_ERR_SYSTEM;
  }
}

struct Msg {
  std::vector<char> data;
  std::vector<int> fds;
};

// One rendezvous channel of a rank (the FileStore / control-queue analogue):
// every rank contributes a small blob per exchange, in the same order on all
// ranks. Channel 0 is used by the thread that issues ops, channel 1 by the
// engine's failure monitor, so the two never interleave their sequences.
constexpr int kChanMain = 0;
constexpr int kChanMonitor = 1;
constexpr int kChannels = 2;
struct Channel {
  int listen_fd = -1;  // abstract unix socket (multi-process ranks)
  uint64_t seq = 0;
  std::map<std::pair<uint64_t, int>, Msg> stash;  // early messages keyed by (sequence, sender)
};

struct LoopGroup;
struct LoopRail;

}  // namespace nz

// Device-visible description of one symmetric buffer.
struct nz_buf {
  nz_comm* comm = nullptr;
  size_t size = 0;        // bytes requested
  size_t mapped = 0;      // bytes mapped (granularity rounded)
  CUmemGenericAllocationHandle local = 0;
  std::vector<CUmemGenericAllocationHandle> imported;  // per rank (0 for self)
  std::vector<char*> ptrs;                             // per rank VA in this process
  CUmemGenericAllocationHandle mc = 0;
  char* mc_ptr = nullptr;
};

constexpr int kMaxRanksHost = 8;

struct nz_comm {
  int rank = 0;
  int world = 1;
  int device = 0;
  int sm_count = 0;
  bool multicast = false;
  int timeout_ms = 60000;
  std::string session;
  nz::Channel chan[nz::kChannels];
  // Virtual-rank loopback (nz_comm_init_loopback): peers are threads of this
  // process driving the same GPU; exchanges and cross-rank launches meet in
  // the group.
  std::shared_ptr<nz::LoopGroup> loop;
  nz_buf* ctrl = nullptr;  // barrier pads, one kPadBytes region per rail
  int next_pad = 0;
  std::vector<int> free_pads;  // returned by destroyed rails (same order on every rank)
  // Rails alive on this rank, for the loopback co-residency budget
  // (rails.cu combine): live_big = rails whose combined grids are large (SM:
  // two-shot fold, LL); copy-engine rails only combine one-CTA barriers.
  // The engine's monitor runs one recovery (one twin grid) at a time.
  int live_rails = 0;
  int live_big = 0;
  int live_twins = 0;
};

struct nz_rail {
  nz_comm* comm = nullptr;
  int kind = 0;
  int rail_id = 0;
  int sm_budget = 0;
  int pad = 0;
  bool graph_safe = false;
  bool recovery = false;  // the engine monitor's twin of a rail (own pads, stream, status)
  cudaStream_t stream = nullptr;
  std::vector<cudaStream_t> side;  // CE: one per peer so several copy engines run at once
  cudaEvent_t fork = nullptr;
  std::vector<cudaEvent_t> join;
  uint32_t* pad_local = nullptr;
  uint32_t* pad_peer[kMaxRanksHost] = {};
  uint32_t epoch = 0;
  nz_fault_record_t* fault_host = nullptr;
  nz_fault_record_t* fault_dev = nullptr;
  int* wd_host = nullptr;
  int* wd_dev = nullptr;
  // Launch status (kernels.cuh RailCtl): device control words + mapped record.
  uint32_t* ctl_dev = nullptr;
  nz_rail_status_t* status_host = nullptr;
  nz_rail_status_t* status_dev = nullptr;
  uint32_t tag = 0;           // op entries issued on this rail (same on every rank)
  int64_t stall_chunk = -1;   // nz_rail_inject_stall armed for the next call
  double detect_us = 0;       // end-barrier budget override (0: default)
  char* staging = nullptr;  // CE: (world-1) slots of staging_slot bytes
  size_t staging_slot = 0;
  nz_buf* ll = nullptr;     // SM: one-shot LL slots [parity][rank][slot_words] of {data, flag}
  uint64_t ll_slot_words = 0;
  uint32_t ll_flag = 0;
  // LL path ceiling (bytes): LL up to ll_max, two-shot above. ll_cap is the
  // buffer capacity; the engine may re-measure the crossover at startup.
  uint64_t ll_max = 0;
  uint64_t ll_cap = 0;
  // Launch order across streams: a rail's launches share pads, LL slots and
  // the control words, so a launch on a new stream first waits for the
  // previous stream's work ("one executor per rail").
  cudaStream_t last_stream = nullptr;
  cudaEvent_t order_ev = nullptr;  // recorded after every eager launch
  bool order_valid = false;
  // Loopback: the group's combiner for this pad, and this rank's events.
  nz::LoopRail* lr = nullptr;
  cudaEvent_t lr_ready = nullptr;
  cudaEvent_t lr_done = nullptr;
  // C-ABI bookkeeping (nz_rail_inject_failure / _progress / _abort); the
  // engine drives rails through nz::railRun and does not touch these.
  int64_t armed_fail = -1;      // failure armed for the next nz_rail_allreduce
  bool aborted = false;         // nz_rail_abort: the rail takes no more work
  uint32_t last_tag = 0;        // entry of the last nz_rail_allreduce
  uint64_t prog_begin = 0;      // its first chunk
  uint64_t prog_stop = 0;       // its stop chunk
  bool prog_valid = false;
};

namespace nz {

// In-process rendezvous of a loopback job (one per session).
struct LoopGroup {
  int world = 0;
  int device = 0;
  uint32_t joined = 0;  // bitmask of ranks
  std::atomic<bool> aborted{false};  // nz_comm_abort: a rank's host code failed
  std::mutex m;
  std::condition_variable cv;
  std::map<std::tuple<int, uint64_t, int>, std::vector<char>> box;  // (channel, seq, sender)
  std::map<std::pair<int, uint64_t>, int> reads;
  std::map<int, std::unique_ptr<LoopRail>> rails;  // by pad index
  ~LoopGroup();
};

// Combiner of one pad's cross-rank launches: the last virtual rank to arrive
// launches one grid for all of them on the group stream, after every rank's
// stream reached the launch (ready events); each rank's stream then waits for
// the grid (done events).
struct LoopRail {
  std::mutex m;
  std::condition_variable cv;
  uint64_t gen = 0;
  int arrived = 0;
  int kind = -1, dtype = -1, grid = 0;
  std::vector<char> args;
  cudaEvent_t ready[kMaxRanks] = {};
  cudaEvent_t done[kMaxRanks] = {};
  cudaStream_t stream = nullptr;
  std::string error;
  // Optional per-launch timing of the grids on the group stream (the stream
  // the kernels run on): event pairs, summed and recycled on read.
  bool timing = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> tev;
  size_t tev_used = 0;
};

// Host-side exchange: every rank contributes (bytes, fds); returns world
// messages indexed by rank (own message included, fds only from peers).
std::vector<Msg> exchange(nz_comm* c, const void* data, size_t bytes, const std::vector<int>& fds,
                          int channel = kChanMain);
// Non-blocking: true (and the blobs of the peers that did) when a peer
// already entered the channel's next exchange, i.e. waits for this rank.
bool peekExchange(nz_comm* c, int channel, std::vector<std::vector<char>>* blobs);
nz_buf* allocSymmetric(nz_comm* c, size_t bytes);
// Device wait budget at the start of an op (NEZHA_WATCHDOG_MS, 20 s).
uint64_t watchdogNs();

// Collective unless `collective` is false (allocation error paths): waits for
// every rank's kernels before unmapping.
void freeSymmetric(nz_buf* b, bool collective = true);
int elemSizeOf(int dtype);

// rails.cu
// Computation-phase gate from the engine's ComputePool arbitration
// (include/nezha/compute_pool.hpp, P14): the rail's SM-driven
// kernel is capped at `max_ctas`, waits for `waits` (earlier holders' phase
// exits) and records `release` as soon as it retires; the CE rail's DMA
// phases stay outside the gate.
struct ComputeGate {
  int max_ctas = 0;  // 0: no cap
  std::vector<cudaEvent_t> waits;
  cudaEvent_t release = nullptr;
  bool entered = false;
  bool exited = false;
};

// One rail call: chunks [chunk_begin, chunk_end) of the segment geometry.
struct RailOp {
  nz_buf* in = nullptr;
  nz_buf* out = nullptr;
  uint64_t seg_off = 0, seg_len = 0, chunk_bytes = 0;
  uint64_t chunk_begin = 0, chunk_end = UINT64_MAX;
  int dtype = NZ_F32;
  uint32_t op_seq = 0;
  int64_t fail_chunk = -1;   // trace form (every rank): stop before it, post a fault record
  int64_t stall_chunk = -1;  // unplanned: this rank's link dies there
  cudaStream_t st = nullptr; // nullptr: the rail's stream
  ComputeGate* gate = nullptr;
  bool status = true;        // publish progress / gate (off inside graph capture)
};

// Runs one rail call; returns its entry tag when its last launch publishes
// the gate (callers may wait for tag on the gate word), else 0.
uint32_t railRun(nz_rail* r, const RailOp& op);
inline uint32_t railAllreduce(nz_rail* r, nz_buf* in, nz_buf* out, uint64_t seg_off, uint64_t seg_len,
                              uint64_t chunk_bytes, uint64_t chunk_begin, uint64_t chunk_end, int dtype,
                              uint32_t op_seq, int64_t fail_chunk, cudaStream_t st, ComputeGate* gate = nullptr) {
  RailOp o;
  o.in = in;
  o.out = out;
  o.seg_off = seg_off;
  o.seg_len = seg_len;
  o.chunk_bytes = chunk_bytes;
  o.chunk_begin = chunk_begin;
  o.chunk_end = chunk_end;
  o.dtype = dtype;
  o.op_seq = op_seq;
  o.fail_chunk = fail_chunk;
  o.st = st;
  o.gate = gate;
  return railRun(r, o);
}
// Waves of a call: consecutive chunk groups of >= NEZHA_WAVE_BYTES (64 MiB)
// each, one launch sequence apiece, so progress is published between them.
std::vector<std::pair<uint64_t, uint64_t>> railWaves(uint64_t chunk_bytes, uint64_t cb, uint64_t ce);
// CTAs of the rail's computation-phase kernel for a whole segment of
// `seg_len` bytes (the ComputePool demand); 0 when it launches none.
int railComputeCtas(nz_rail* r, uint64_t seg_len);
void launchStamp(uint64_t* dst, cudaStream_t st);
// Rail creation for the engine (twins: recovery = true, no LL path).
nz_rail* railCreate(nz_comm* comm, int kind, int rail_id, int sm_budget, bool graph_safe, bool recovery);
void railDestroy(nz_rail* r);
// The rail's gate word (device memory, for cuStreamWaitValue32 /
// cuStreamWriteValue32) and its reset after a failure (sticky, abort).
CUdeviceptr railGateAddr(nz_rail* r);
// Whether a call over this segment runs the one-shot LL path.
bool railLLPath(nz_rail* r, uint64_t seg_off, uint64_t seg_len);
void railRevive(nz_rail* r, cudaStream_t st);

// rails_vr.cu: the virtual-rank (loopback) grids.
enum LoopKind : int { kLoopFold = 0, kLoopLL = 1, kLoopBarrier = 2 };
void launchLoopGrid(int kind, int world, int dtype, const void* pack, int grid, cudaStream_t st);
int loopOccupancy(int kind, int world, int dtype);

}  // namespace nz
