// Kernel argument blocks of the three rails (passed by value as
// __grid_constant__ parameters; plain C++ so host code can build them
// without the device headers). See kernels.cuh for the kernels.
#pragma once

#include <stdint.h>

#include "nezha_b200.h"

namespace nz {

constexpr int kDevMaxRanks = 8;

struct Geometry {
  uint64_t seg_off;
  uint64_t seg_len;
  uint64_t chunk;
};

// Words of a rail's device control block (RailCtl::dev).
enum : int {
  kCtlRetired = 0,  // CTAs of the current launch that retired
  kCtlFailed = 1,   // a CTA of the current launch failed
  kCtlGate = 2,     // tag of the last op entry completed on this rank
  kCtlSticky = 3,   // the rail failed on this rank: launches exit at once
  kCtlSeq = 4,      // launches retired (graph-safe epochs / LL flags)
  kCtlWords = 8,
};

struct RailCtl {
  uint32_t* dev;              // nullptr: launch without status (emulation, CE reduce)
  nz_rail_status_t* host;     // host-mapped record for the engine's monitor
  uint32_t tag;               // op entry this launch belongs to
  int final_wave;             // last launch of the entry: gate on success
  int stall;                  // injected dead link: stop after the start barrier
  uint64_t prog_chunk;        // chunks complete once this launch succeeds (~0: none)
  uint64_t end_timeout_ns;    // budget of the end barrier (failure detection)
};

// Cross-rank per-CTA barrier pads of one rail: slot [cta][rank] of rank p's
// pad is written only by `rank`, with monotonically increasing epochs.
struct BarrierArgs {
  uint32_t* local;
  uint32_t* peer[kDevMaxRanks];
  uint32_t epoch;
  int* watchdog;                    // host-mapped; set when a wait times out
  uint64_t timeout_ns;              // start-of-op budget (NEZHA_WATCHDOG_MS, default 20 s)
  const uint32_t* seq;              // graph-safe rails: device launch counter; nullptr = host `epoch`
  const volatile uint32_t* abort;   // host-mapped; nonzero = the monitor gave up on this rail
};

struct FaultPost {
  nz_fault_record_t* rec;  // host-mapped, nullptr = nothing to post
  uint32_t op_seq;
  uint64_t chunk;
};

struct FoldArgs {
  const char* src[kDevMaxRanks];  // rank r's element at byte offset x is src[r] + x
  char* dst[kDevMaxRanks];        // outputs written at byte offset x
  uint64_t s, e;                  // this rank's shard [s, e)
  uint64_t range_bytes;           // whole reduced range, sizes the grid identically on every rank
  Geometry g;
  BarrierArgs bar;
  int use_barrier;
  int rank;
  FaultPost post;
  RailCtl ctl;
};

struct NvlsArgs {
  char* mc_in;
  char* mc_out;
  FoldArgs f;  // unicast view for the unaligned head / tail and the barrier
};

// Arguments of every virtual rank of a loopback job, indexed by blockIdx.y.
template <typename A>
struct VPack {
  A a[kDevMaxRanks];
};

// --------------------------------------------------------- LL (one-shot) --
// Small segments on the SM rail: every rank pushes its words, each tagged
// with this op's flag in the same 8-byte store ({data, flag} pairs, the LL
// idea), into slot [rank] of every peer's LL buffer, then polls its own slots
// and folds in ring order (P1). No barrier round trips: one NVLink one-way
// latency. Two parities alternate so a rank at most one op ahead never
// overwrites a slot a peer still reads (stream order on every rank).
struct LLArgs {
  const char* in;  // my input, byte offset x at in + x
  char* out;       // my output
  uint64_t* peer[kDevMaxRanks];  // each rank's LL buffer (8-byte {data, flag} words)
  uint64_t* local;
  uint64_t lo, hi;
  uint64_t words;       // ceil((hi - lo) / 4)
  uint64_t slot_words;  // capacity of one (parity, rank) slot
  Geometry g;
  uint32_t flag;
  int parity;
  int rank;
  int* watchdog;
  uint64_t timeout_ns;
  FaultPost post;
  const uint32_t* seq;              // graph-safe rails: flag / parity from the device launch counter
  const volatile uint32_t* abort;   // host-mapped; set only once the ranks agreed the rail failed
  RailCtl ctl;
};

// CE rail: start / end barriers around the DMA phases (K4). The start
// barrier orders the peers' inputs before this rank's gather DMAs; the end
// barrier orders every peer's scatter into this rank's output before the op
// counts as done, posts the fault record and publishes the launch status.
struct BarrierKArgs {
  BarrierArgs bar;
  int rank;
  int end;  // 0: start barrier, 1: end barrier
  FaultPost post;
  RailCtl ctl;
};

}  // namespace nz
