// Internal definitions shared by the CUDA translation units of libnezha_b200.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
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
  int listen_fd = -1;
  uint64_t xchg_seq = 0;
  // Messages that arrived early, keyed by (exchange sequence, sender).
  struct Msg {
    std::vector<char> data;
    std::vector<int> fds;
  };
  std::map<std::pair<uint64_t, int>, Msg> stash;
  nz_buf* ctrl = nullptr;  // barrier pads, one kPadBytes region per rail
  int next_pad = 0;
};

struct nz_rail {
  nz_comm* comm = nullptr;
  int kind = 0;
  int rail_id = 0;
  int sm_budget = 0;
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
  char* staging = nullptr;  // CE: (world-1) slots of staging_slot bytes
  size_t staging_slot = 0;
  nz_buf* ll = nullptr;     // SM: one-shot LL slots [parity][rank][slot_words] of {data, flag}
  uint64_t ll_slot_words = 0;
  uint32_t ll_flag = 0;
  uint32_t* seq_dev = nullptr;  // graph-safe rails: device [op counter, CTAs retired]
  nz_buf* os = nullptr;         // SM one-shot staging [parity 2][rank N][os_slot bytes] (NEZHA_SM_ONESHOT)
  uint64_t os_slot = 0;
  // Path ceilings (bytes): LL up to ll_max, one-shot up to os_max, two-shot
  // above. Set to the buffer capacities at creation; the engine re-measures
  // the crossovers at startup (same on every rank).
  uint64_t ll_max = 0;
  uint64_t os_max = 0;
  uint64_t ll_cap = 0;
  uint64_t os_cap = 0;
  // C-ABI bookkeeping (nz_rail_inject_failure / _progress / _abort); the
  // engine drives rails through nz::railAllreduce and does not touch these.
  int64_t armed_fail = -1;      // failure armed for the next nz_rail_allreduce
  bool aborted = false;         // nz_rail_abort: the rail takes no more work
  cudaEvent_t done = nullptr;   // end of the last nz_rail_allreduce
  uint64_t prog_begin = 0;      // its first chunk
  uint64_t prog_stop = 0;       // chunks complete once `done` fired
  bool prog_valid = false;
};

namespace nz {
// Host-side exchange: every rank contributes (bytes, fds); returns world
// messages indexed by rank (own message included, fds only from peers).
std::vector<nz_comm::Msg> exchange(nz_comm* c, const void* data, size_t bytes, const std::vector<int>& fds);
nz_buf* allocSymmetric(nz_comm* c, size_t bytes);
void freeSymmetric(nz_buf* b);
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
void railAllreduce(nz_rail* r, nz_buf* in, nz_buf* out, uint64_t seg_off, uint64_t seg_len, uint64_t chunk_bytes,
                   uint64_t chunk_begin, uint64_t chunk_end, int dtype, uint32_t op_seq, int64_t fail_chunk,
                   cudaStream_t st, ComputeGate* gate = nullptr);
// CTAs of the rail's computation-phase kernel for a whole segment of
// `seg_len` bytes (the ComputePool demand); 0 when it launches none.
int railComputeCtas(nz_rail* r, uint64_t seg_len);
void launchStamp(uint64_t* dst, cudaStream_t st);
}  // namespace nz
