// Host side of the three rails: launch configuration, DMA phases of the
// copy-engine rail, launch status and fault records, loopback launches. One
// nz_rail per (rank, rail); each owns a CUDA stream, which is the B200 form of
// the reference's "one collective executor per rail".
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>

#include "internal.h"
#include "kernels.cuh"
#include "nezha/collective.hpp"

namespace nz {

// Every kernel this library launches bumps this (nz_kernel_launch_count).
std::atomic<uint64_t> g_launches{0};

namespace {

int elemSize(int dtype) {
  switch (dtype) {
    case NZ_F32:
    case NZ_I32:
      return 4;
    case NZ_BF16:
      return 2;
  }
  fail(NZ_ERR_INVALID, "unknown dtype " + std::to_string(dtype));
}

// Contiguous shard of [lo, hi) owned by `rank`: interior split at 16-byte
// boundaries, unaligned head to rank 0, tail to rank world-1.
void shardOf(uint64_t lo, uint64_t hi, int rank, int world, uint64_t* s, uint64_t* e) {
  const uint64_t A = (lo + 15) & ~15ull, B = hi & ~15ull;
  if (A >= B) {
    *s = rank == 0 ? lo : hi;
    *e = hi;
    return;
  }
  const uint64_t V = (B - A) / 16;
  *s = rank == 0 ? lo : A + 16 * (V * rank / world);
  *e = rank == world - 1 ? hi : A + 16 * (V * (rank + 1) / world);
}

long long envLL(const char* name, long long def) {
  const char* e = getenv(name);
  return e ? atoll(e) : def;
}

// Device wait budget at the start of an op (ranks may legitimately arrive far
// apart: the caller's stream decides when a launch starts). NEZHA_WATCHDOG_MS
// overrides the 20 s default; past it a kernel gives up instead of hanging.
}  // namespace

uint64_t watchdogNs() {
  static const uint64_t ns = [] {
    const long long ms = envLL("NEZHA_WATCHDOG_MS", 20000);
    return static_cast<uint64_t>(ms > 0 ? ms : 20000) * 1000000ull;
  }();
  return ns;
}

namespace {

// End-barrier budget: every rank passed the start barrier of the same op and
// does the same work, so a peer missing for much longer than the op itself
// takes has lost its link. max(floor, 4 x range / 100 GB/s),
// floor NEZHA_DETECT_US (5000 us) or the rail's / engine's setting: generous
// against a slow-but-alive peer, still far below SPEC's 200 ms.
uint64_t detectNs(const nz_rail* r, uint64_t range_bytes) {
  static const double env_us = static_cast<double>(envLL("NEZHA_DETECT_US", 5000));
  const double floor_us = r->detect_us > 0 ? r->detect_us : env_us;
  const double scaled_us = 4.0 * static_cast<double>(range_bytes) / 100e9 * 1e6;
  return static_cast<uint64_t>(std::max(floor_us, scaled_us) * 1000.0);
}

uint64_t waveBytes() {
  static const uint64_t b = [] {
    const long long v = envLL("NEZHA_WAVE_BYTES", 64ll << 20);
    return static_cast<uint64_t>(v > 0 ? v : (64ll << 20));
  }();
  return b;
}

BarrierArgs barrierArgs(nz_rail* r, uint32_t epoch) {
  BarrierArgs b{};
  b.local = r->pad_local;
  for (int p = 0; p < r->comm->world; ++p) b.peer[p] = r->pad_peer[p];
  b.epoch = epoch;
  b.watchdog = r->wd_dev;
  b.timeout_ns = watchdogNs();
  b.seq = r->graph_safe ? r->ctl_dev + kCtlSeq : nullptr;
  b.abort = &r->status_dev->abort;
  return b;
}

int gridFor(nz_rail* r, uint64_t range_bytes, int world, int unroll) {
  // sm_budget 0 = the rail's measured sweet spot on B200 (profiles/README.md):
  // NVLS saturates the switch path with 32 CTAs, the SM rail with 64; the
  // rest of the GPU stays free for a concurrent rail or the caller's kernels.
  // With one rank every rail is a local copy (HBM-bound): two CTAs per SM.
  const int def = world == 1 ? 2 * r->comm->sm_count
                             : (r->kind == NZ_RAIL_NVLS ? 32 : (r->kind == NZ_RAIL_SM ? 64 : r->comm->sm_count));
  const int budget = world == 1 ? def : std::min(r->sm_budget > 0 ? r->sm_budget : def, r->comm->sm_count);
  const uint64_t per_rank_vec = range_bytes / 16 / static_cast<uint64_t>(world) + 1;
  const uint64_t per_cta = static_cast<uint64_t>(kThreads) * unroll;
  const uint64_t g = (per_rank_vec + per_cta - 1) / per_cta;
  return static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(g, std::min(budget, kMaxCtas))));
}

constexpr uint64_t kLLMaxBytes = 2048 * 1024;  // SM rail one-shot LL path up to this payload

// LL pays 2 wire bytes per payload byte times N receivers; beyond ~4 MiB / N
// the two-shot kernels win (measured crossover, profiles/README.md).
uint64_t llMaxBytes(int world) {
  // NEZHA_LL_MAX (bytes) lowers the ceiling for sweeps; it never raises it
  // (the LL buffers are sized by this function at rail creation).
  static const long long env = envLL("NEZHA_LL_MAX", -1);
  const uint64_t def = std::min<uint64_t>(kLLMaxBytes, (uint64_t{4} << 20) / world);
  return env >= 0 ? std::min<uint64_t>(def, static_cast<uint64_t>(env)) : def;
}

bool llPath(nz_rail* r, uint64_t lo, uint64_t hi) {
  return r->comm->world > 1 && r->kind == NZ_RAIL_SM && r->ll && hi - lo <= r->ll_max && lo % 4 == 0;
}

// One thread per polled word, capped at the rail's CTA budget (default 64,
// as its two-shot path): LL CTAs wait on peers' CTAs of the same index, so the
// rail must stay inside the co-residency budget it shares with the other
// rails' kernels (§3 "CTA budgets"), whichever path it takes.
int llGrid(nz_rail* r, uint64_t lo, uint64_t hi) {
  const uint64_t words = (hi - lo + 3) / 4;
  const int budget = std::min(r->sm_budget > 0 ? r->sm_budget : 64, r->comm->sm_count);
  return static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>((words + kThreads - 1) / kThreads, budget)));
}

int copyGrid(nz_rail* r, uint64_t lo, uint64_t hi) {
  const uint64_t vec = (hi - lo) / 16 + 1;
  return static_cast<int>(
      std::max<uint64_t>(1, std::min<uint64_t>((vec + kThreads * 8 - 1) / (kThreads * 8), 2ull * r->comm->sm_count)));
}

int smGrid(nz_rail* r, uint64_t lo, uint64_t hi) { return gridFor(r, hi - lo, r->comm->world, 2); }

// ------------------------------------------------------------ launches ----
template <typename DT, int N, int NDST>
void launchFoldT(const FoldArgs& a, int grid, cudaStream_t st) {
  fold_kernel<DT, N, NDST><<<grid, kThreads, 0, st>>>(a);
}

template <int N, int NDST>
void dispatchFoldDT(int dtype, const FoldArgs& a, int grid, cudaStream_t st) {
  switch (dtype) {
    case NZ_F32: return launchFoldT<F32, N, NDST>(a, grid, st);
    case NZ_BF16: return launchFoldT<BF16, N, NDST>(a, grid, st);
    case NZ_I32: return launchFoldT<I32, N, NDST>(a, grid, st);
  }
}

template <int NDST_IS_N>
void dispatchFold(int world, int dtype, const FoldArgs& a, int grid, cudaStream_t st) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  switch (world) {
#define NZ_CASE(n) \
  case n: return dispatchFoldDT<n, NDST_IS_N ? n : 1>(dtype, a, grid, st);
    NZ_CASE(1) NZ_CASE(2) NZ_CASE(3) NZ_CASE(4) NZ_CASE(5) NZ_CASE(6) NZ_CASE(7) NZ_CASE(8)
#undef NZ_CASE
  }
}

void dispatchLL(int world, int dtype, const LLArgs& a, int grid, cudaStream_t st) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  switch (world) {
#define NZ_CASE(n)                                                                             \
  case n:                                                                                      \
    if (dtype == NZ_F32) return (void)(ll_kernel<F32, n><<<grid, kThreads, 0, st>>>(a));      \
    if (dtype == NZ_BF16) return (void)(ll_kernel<BF16, n><<<grid, kThreads, 0, st>>>(a));    \
    return (void)(ll_kernel<I32, n><<<grid, kThreads, 0, st>>>(a));
    NZ_CASE(2) NZ_CASE(3) NZ_CASE(4) NZ_CASE(5) NZ_CASE(6) NZ_CASE(7) NZ_CASE(8)
#undef NZ_CASE
  }
}

template <int N>
void launchNvls(int dtype, const NvlsArgs& a, int grid, cudaStream_t st) {
  if (dtype == NZ_F32) return (void)(nvls_kernel<F32, N><<<grid, kThreads, 0, st>>>(a));
  if (dtype == NZ_BF16) return (void)(nvls_kernel<BF16, N><<<grid, kThreads, 0, st>>>(a));
  return (void)(nvls_kernel<I32, N><<<grid, kThreads, 0, st>>>(a));
}

void dispatchNvls(int world, int dtype, const NvlsArgs& a, int grid, cudaStream_t st) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  switch (world) {
#define NZ_CASE(n) \
  case n: return launchNvls<n>(dtype, a, grid, st);
    NZ_CASE(2) NZ_CASE(3) NZ_CASE(4) NZ_CASE(5) NZ_CASE(6) NZ_CASE(7) NZ_CASE(8)
#undef NZ_CASE
  }
}

void dispatchBarrier(int world, const BarrierKArgs& k, cudaStream_t st) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  switch (world) {
#define NZ_CASE(n) \
  case n: barrier_kernel<n><<<1, 32, 0, st>>>(k); break;
    NZ_CASE(1) NZ_CASE(2) NZ_CASE(3) NZ_CASE(4) NZ_CASE(5) NZ_CASE(6) NZ_CASE(7) NZ_CASE(8)
#undef NZ_CASE
  }
}

// Loopback: the last virtual rank to reach this launch runs one grid for all
// of them (blockIdx.y = rank) on the pad's group stream, ordered after every
// rank's stream and before each rank's next work. The grid is capped so that
// every cross-rank grid that can run at once is resident at once — the
// cross-rank waits inside are then between co-resident CTAs, and no grid
// waits on another launch:
//   * copy-engine rails combine only their start / end barriers (N CTAs of
//     32 threads): kLoopReserveSMs hold all of them;
//   * the one recovery twin the monitor may be running gets kLoopTwinSMs;
//   * the SM-kind rails (two-shot fold, LL) share the rest evenly.
// Units are each kernel's own resident CTAs per SM (occupancy x SMs).
constexpr int kLoopReserveSMs = 2;
constexpr int kLoopTwinSMs = 8;

int loopCap(const nz_rail* r, int kind, int dtype) {
  const nz_comm* c = r->comm;
  const int N = c->world;
  const int occ = std::max(1, loopOccupancy(kind, N, dtype));
  if (r->recovery) return std::max(1, occ * kLoopTwinSMs / N);
  const int avail = std::max(1, c->sm_count - kLoopReserveSMs - (c->live_twins ? kLoopTwinSMs : 0));
  return std::max(1, occ * avail / (N * std::max(1, c->live_big)));
}

template <typename A>
void combine(nz_rail* r, int kind, int dtype, const A& a, int grid, cudaStream_t st) {
  nz_comm* c = r->comm;
  LoopRail& L = *r->lr;
  const int me = c->rank, N = c->world;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  NZ_CUDA(cudaStreamIsCapturing(st, &cap));
  if (cap != cudaStreamCaptureStatusNone) fail(NZ_ERR_UNSUPPORTED, "loopback ranks cannot be captured in a CUDA graph");
  NZ_CUDA(cudaEventRecord(r->lr_ready, st));
  std::unique_lock<std::mutex> lk(L.m);
  const uint64_t gen = L.gen;
  if (L.arrived == 0) {
    L.kind = kind;
    L.dtype = dtype;
    L.grid = grid;
    L.args.assign(sizeof(VPack<A>), 0);
    L.error.clear();
  } else if (L.kind != kind || L.dtype != dtype || L.grid != grid || L.args.size() != sizeof(VPack<A>)) {
    L.error = "loopback ranks issued different launches on rail " + std::to_string(r->rail_id);
  }
  if (L.args.size() == sizeof(VPack<A>)) memcpy(L.args.data() + me * sizeof(A), &a, sizeof(A));
  std::string err;
  if (++L.arrived == N) {
    err = L.error;
    if (err.empty()) {
      try {
        for (int p = 0; p < N; ++p) NZ_CUDA(cudaStreamWaitEvent(L.stream, L.ready[p], 0));
        const int cap_ctas = kind == kLoopBarrier ? 1 : loopCap(r, kind, dtype);
        std::pair<cudaEvent_t, cudaEvent_t>* tp = nullptr;
        if (L.timing) {
          if (L.tev_used == L.tev.size()) {
            std::pair<cudaEvent_t, cudaEvent_t> pr;
            NZ_CUDA(cudaEventCreate(&pr.first));
            NZ_CUDA(cudaEventCreate(&pr.second));
            L.tev.push_back(pr);
          }
          tp = &L.tev[L.tev_used++];
          NZ_CUDA(cudaEventRecord(tp->first, L.stream));
        }
        launchLoopGrid(kind, N, dtype, L.args.data(), std::min(grid, cap_ctas), L.stream);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        NZ_CUDA(cudaGetLastError());
        if (tp) NZ_CUDA(cudaEventRecord(tp->second, L.stream));
        for (int p = 0; p < N; ++p) NZ_CUDA(cudaEventRecord(L.done[p], L.stream));
      } catch (const std::exception& e) {
        err = e.what();
      }
    }
    L.arrived = 0;
    L.error = err;
    L.gen++;
    L.cv.notify_all();
  } else {
    const auto deadline = std::chrono::steady_clock::now() + std::chrono::milliseconds(c->timeout_ms);
    while (L.gen == gen) {
      if (c->loop->aborted) fail(NZ_ERR_TIMEOUT, "loopback group aborted: a virtual rank failed");
      if (L.cv.wait_until(lk, deadline) == std::cv_status::timeout && L.gen == gen) {
        fail(NZ_ERR_TIMEOUT, "loopback launch: a virtual rank never reached rail " + std::to_string(r->rail_id));
      }
    }
    err = L.error;
  }
  lk.unlock();
  if (!err.empty()) fail(NZ_ERR_CUDA, err);
  NZ_CUDA(cudaStreamWaitEvent(st, r->lr_done, 0));
}

// Cross-rank launches: direct on a real rank, combined across virtual ranks.
void launchCrossFold(nz_rail* r, int dtype, const FoldArgs& a, int grid, cudaStream_t st) {
  if (r->lr) return combine(r, kLoopFold, dtype, a, grid, st);
  dispatchFold<1>(r->comm->world, dtype, a, grid, st);
}

void launchCrossLL(nz_rail* r, int dtype, const LLArgs& a, int grid, cudaStream_t st) {
  if (r->lr) return combine(r, kLoopLL, dtype, a, grid, st);
  dispatchLL(r->comm->world, dtype, a, grid, st);
}

void launchBarrier(nz_rail* r, uint32_t epoch, bool end, FaultPost post, const RailCtl& ctl, cudaStream_t st) {
  BarrierKArgs k{};
  k.bar = barrierArgs(r, epoch);
  k.rank = r->comm->rank;
  k.end = end ? 1 : 0;
  k.post = post;
  k.ctl = ctl;
  if (r->lr) return combine(r, kLoopBarrier, NZ_F32, k, 1, st);
  dispatchBarrier(r->comm->world, k, st);
}

void ensureStaging(nz_rail* r, size_t slot, cudaStream_t st, std::vector<char*>* retired) {
  if (slot <= r->staging_slot) return;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  NZ_CUDA(cudaStreamIsCapturing(st, &cap));
  if (cap != cudaStreamCaptureStatusNone)
    fail(NZ_ERR_INVALID, "CE staging must grow outside graph capture: run the largest op eagerly first");
  // A captured graph may still reference the old buffer: keep it until the
  // rail is destroyed instead of freeing it under the graph.
  if (r->staging) retired->push_back(r->staging);
  r->staging = nullptr;
  const size_t want = (slot + (1u << 20)) & ~((size_t(1) << 20) - 1);
  NZ_CUDA(cudaMalloc(&r->staging, want * std::max(1, r->comm->world - 1)));
  r->staging_slot = want;
}

// Old staging buffers of every rail, freed at rail destruction.
std::mutex g_retired_mu;
std::map<nz_rail*, std::vector<char*>> g_retired;

void gateEnter(ComputeGate* gate, cudaStream_t st) {
  if (!gate || gate->entered) return;
  for (cudaEvent_t e : gate->waits) NZ_CUDA(cudaStreamWaitEvent(st, e, 0));
  gate->entered = true;
}

void gateExit(ComputeGate* gate, cudaStream_t st) {
  if (!gate || gate->exited) return;
  gateEnter(gate, st);  // a rail with nothing to compute still orders after its waits
  if (gate->release) NZ_CUDA(cudaEventRecord(gate->release, st));
  gate->exited = true;
}

int gated(int grid, const ComputeGate* gate) {
  return gate && gate->max_ctas > 0 ? std::max(1, std::min(grid, gate->max_ctas)) : grid;
}

// Pieces of a CE shard [s, e) pipelined through gather / fold / scatter:
// the gather of piece i+1 (inbound NVLink) overlaps the fold of piece i and
// the scatter of piece i-1 (outbound), so both link directions work at once.
// Under RingChunked the pieces are the chunks (transmission
// of chunk k+1 overlaps reduction of chunk k); nezha::pipelineCuts.
// NEZHA_CE_PIECES forces an equal-piece count (sweeps).
std::vector<uint64_t> cePieces(uint64_t s, uint64_t e, const Geometry& g) {
  static const int forced = static_cast<int>(envLL("NEZHA_CE_PIECES", 0));
  return nezha::pipelineCuts(s, e, nezha::ChunkGeometry{g.seg_off, g.seg_len, g.chunk}, forced);
}

// One launch sequence of a rail over [lo, hi) with order geometry g.
void railWave(nz_rail* r, nz_buf* in, nz_buf* out, uint64_t lo, uint64_t hi, const Geometry& g, int dtype,
              FaultPost post, const RailCtl& ctl, cudaStream_t st, ComputeGate* gate) {
  nz_comm* c = r->comm;
  const int N = c->world;
  const int me = c->rank;
  uint64_t s, e;
  shardOf(lo, hi, me, N, &s, &e);
  const uint32_t epoch = r->epoch + 1;
  r->epoch += 2;  // start + end barrier; identical on every rank

  if (llPath(r, lo, hi)) {
    LLArgs a{};
    a.in = in->ptrs[me];
    a.out = out->ptrs[me];
    for (int p = 0; p < N; ++p) a.peer[p] = reinterpret_cast<uint64_t*>(r->ll->ptrs[p]);
    a.local = reinterpret_cast<uint64_t*>(r->ll->ptrs[me]);
    // Every 16-byte push must be 16-byte aligned.
    if ((r->ll_slot_words & 1u) != 0 || reinterpret_cast<uintptr_t>(r->ll->ptrs[me]) % 16 != 0)
      fail(NZ_ERR_INVALID, "LL slots are not 16-byte aligned");
    a.lo = lo;
    a.hi = hi;
    a.words = (hi - lo + 3) / 4;
    a.slot_words = r->ll_slot_words;
    a.g = g;
    if (++r->ll_flag == 0) r->ll_flag = 1;  // flag 0 means "never written"
    a.flag = r->ll_flag;
    a.parity = static_cast<int>(r->ll_flag & 1u);
    a.rank = me;
    a.watchdog = r->wd_dev;
    a.timeout_ns = watchdogNs();
    a.post = post;
    a.seq = r->graph_safe ? r->ctl_dev + kCtlSeq : nullptr;
    a.abort = &r->status_dev->abort;
    a.ctl = ctl;
    gateEnter(gate, st);
    launchCrossLL(r, dtype, a, gated(llGrid(r, lo, hi), gate), st);
    NZ_CUDA(cudaGetLastError());
    return;
  }

  if (N == 1) {  // identity allreduce: every rail is a local HBM copy
    gateEnter(gate, st);
    copy_kernel<<<gated(copyGrid(r, lo, hi), gate), kThreads, 0, st>>>(in->ptrs[0], out->ptrs[0], lo, hi, post, ctl);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    NZ_CUDA(cudaGetLastError());
    return;
  }

  if (r->kind == NZ_RAIL_SM) {
    FoldArgs a{};
    for (int p = 0; p < N; ++p) {
      a.src[p] = in->ptrs[p];
      a.dst[p] = out->ptrs[p];
    }
    a.s = s;
    a.e = e;
    a.range_bytes = hi - lo;
    a.g = g;
    a.bar = barrierArgs(r, epoch);
    a.use_barrier = 1;
    a.rank = me;
    a.post = post;
    a.ctl = ctl;
    gateEnter(gate, st);
    launchCrossFold(r, dtype, a, gated(smGrid(r, lo, hi), gate), st);
    NZ_CUDA(cudaGetLastError());
    return;
  }

  if (r->kind == NZ_RAIL_NVLS) {
    if (!in->mc_ptr || !out->mc_ptr) fail(NZ_ERR_UNSUPPORTED, "NVLS rail needs multicast-bound buffers");
    if (reinterpret_cast<uintptr_t>(in->mc_ptr) % 16 != 0 || reinterpret_cast<uintptr_t>(out->mc_ptr) % 16 != 0)
      fail(NZ_ERR_INVALID, "multicast windows must be 16-byte aligned");
    NvlsArgs a{};
    a.mc_in = in->mc_ptr;
    a.mc_out = out->mc_ptr;
    for (int p = 0; p < N; ++p) {
      a.f.src[p] = in->ptrs[p];
      a.f.dst[p] = out->ptrs[p];
    }
    a.f.s = s;
    a.f.e = e;
    a.f.range_bytes = hi - lo;
    a.f.g = g;
    a.f.bar = barrierArgs(r, epoch);
    a.f.use_barrier = 1;
    a.f.rank = me;
    a.f.post = post;
    a.f.ctl = ctl;
    gateEnter(gate, st);
    dispatchNvls(N, dtype, a, gated(gridFor(r, hi - lo, N, 4), gate), st);
    NZ_CUDA(cudaGetLastError());
    return;
  }

  // Copy-engine rail: start barrier, then per piece of my shard a DMA gather
  // from every peer, the local ring-order reduce and a DMA scatter of the sum
  // to every peer, pipelined across pieces; end barrier.
  RailCtl start_ctl = ctl;
  start_ctl.final_wave = 0;
  start_ctl.prog_chunk = ~0ull;
  launchBarrier(r, epoch, false, FaultPost{}, start_ctl, st);
  const uint64_t len = e - s;
  if (len > 0) {
    // Staged copies keep the 16-byte phase of the source so the reduce
    // kernel's vector loads stay aligned: copy from s16 = align_down(s, 16).
    const uint64_t s16 = s & ~15ull;
    {
      std::lock_guard<std::mutex> lk(g_retired_mu);
      ensureStaging(r, e - s16, st, &g_retired[r]);
    }
    const std::vector<uint64_t> cut = cePieces(s, e, g);
    const int P = static_cast<int>(cut.size()) - 1;
    const int peers = N - 1;  // side[0 .. peers) gather, side[peers .. 2 peers) scatter
    NZ_CUDA(cudaEventRecord(r->fork, st));
    for (int j = 0; j < 2 * peers; ++j) NZ_CUDA(cudaStreamWaitEvent(r->side[j], r->fork, 0));
    FoldArgs a{};
    for (int p = 0; p < N; ++p) {
      const int j = (p - me + N) % N;
      a.src[p] = j == 0 ? in->ptrs[me] : r->staging + (j - 1) * r->staging_slot - s16;
    }
    a.dst[0] = out->ptrs[me];
    a.range_bytes = hi - lo;
    a.g = g;
    a.use_barrier = 0;
    a.rank = me;
    for (int i = 0; i < P; ++i) {
      const uint64_t ps = cut[i], pe = cut[i + 1];
      if (pe <= ps) continue;
      const uint64_t ps16 = ps & ~15ull;
      for (int j = 1; j < N; ++j) {
        const int p = (me + j) % N;
        cudaStream_t gs = r->side[j - 1];
        NZ_CUDA(cudaMemcpyAsync(r->staging + (j - 1) * r->staging_slot + (ps16 - s16), in->ptrs[p] + ps16, pe - ps16,
                                cudaMemcpyDeviceToDevice, gs));
        NZ_CUDA(cudaEventRecord(r->join[j - 1], gs));
        NZ_CUDA(cudaStreamWaitEvent(st, r->join[j - 1], 0));
      }
      a.s = ps;
      a.e = pe;
      gateEnter(gate, st);  // computation phase: the local folds
      dispatchFold<0>(N, dtype, a, gated(gridFor(r, (pe - ps) * N, N, 2), gate), st);
      NZ_CUDA(cudaGetLastError());
      NZ_CUDA(cudaEventRecord(r->fork, st));
      for (int j = 1; j < N; ++j) {
        const int p = (me + j) % N;
        cudaStream_t ss = r->side[peers + j - 1];
        NZ_CUDA(cudaStreamWaitEvent(ss, r->fork, 0));
        NZ_CUDA(cudaMemcpyAsync(out->ptrs[p] + ps, out->ptrs[me] + ps, pe - ps, cudaMemcpyDeviceToDevice, ss));
      }
    }
    for (int j = 0; j < peers; ++j) {
      NZ_CUDA(cudaEventRecord(r->join[peers + j], r->side[peers + j]));
      NZ_CUDA(cudaStreamWaitEvent(st, r->join[peers + j], 0));
    }
  }
  launchBarrier(r, epoch + 1, true, post, ctl, st);
  NZ_CUDA(cudaGetLastError());
}

// A rail's launches share pads, LL slots and control words, so a launch on a
// stream other than the one the rail's previous launch went to first waits
// for that launch. The event is recorded after every eager launch, so the
// wait never touches the previous stream itself (which the caller may have
// destroyed since); captured launches are ordered by their graph instead.
void orderBefore(nz_rail* r, cudaStream_t st, bool capturing) {
  if (capturing || !r->order_valid || st == r->last_stream) return;
  NZ_CUDA(cudaStreamWaitEvent(st, r->order_ev, 0));
}

void orderAfter(nz_rail* r, cudaStream_t st, bool capturing) {
  if (capturing) return;
  NZ_CUDA(cudaEventRecord(r->order_ev, st));
  r->order_valid = true;
  r->last_stream = st;
}

}  // namespace

int elemSizeOf(int dtype) { return elemSize(dtype); }

__global__ void stamp_kernel(uint64_t* dst) {
  *reinterpret_cast<volatile uint64_t*>(dst) = globaltimer();
  __threadfence_system();
}

void launchStamp(uint64_t* dst, cudaStream_t st) {
  stamp_kernel<<<1, 1, 0, st>>>(dst);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  NZ_CUDA(cudaGetLastError());
}

std::vector<std::pair<uint64_t, uint64_t>> railWaves(uint64_t chunk_bytes, uint64_t cb, uint64_t ce) {
  return nezha::waveRanges(chunk_bytes, cb, ce, waveBytes());
}

uint32_t railRun(nz_rail* r, const RailOp& op) {
  const int es = elemSize(op.dtype);
  if (op.chunk_bytes == 0 || op.chunk_bytes % es || op.seg_off % es || op.seg_len % es) {
    fail(NZ_ERR_INVALID, "segment geometry not element aligned");
  }
  if (op.in->comm != r->comm || op.out->comm != r->comm) fail(NZ_ERR_INVALID, "buffer from another comm");
  if (op.seg_off + op.seg_len > op.in->size || op.seg_off + op.seg_len > op.out->size)
    fail(NZ_ERR_INVALID, "segment exceeds buffer");
  const uint64_t nch = (op.seg_len + op.chunk_bytes - 1) / op.chunk_bytes;
  if (op.chunk_begin > op.chunk_end) fail(NZ_ERR_INVALID, "chunk_begin > chunk_end");
  const uint64_t chunk_end = std::min(op.chunk_end, nch);
  // A window that starts past the segment's last chunk is empty.
  const uint64_t chunk_begin = std::min(op.chunk_begin, chunk_end);
  uint64_t stop = chunk_end;
  FaultPost post{};
  if (op.fail_chunk >= 0 && static_cast<uint64_t>(op.fail_chunk) >= chunk_begin &&
      static_cast<uint64_t>(op.fail_chunk) < chunk_end) {
    stop = static_cast<uint64_t>(op.fail_chunk);
    post.rec = r->fault_dev;
    post.op_seq = op.op_seq;
    post.chunk = stop;
  }
  int64_t stall = op.stall_chunk >= 0 ? op.stall_chunk : r->stall_chunk;
  r->stall_chunk = -1;
  cudaStream_t st = op.st ? op.st : r->stream;
  NZ_CUDA(cudaSetDevice(r->comm->device));
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  NZ_CUDA(cudaStreamIsCapturing(st, &cap));
  const bool capturing = cap != cudaStreamCaptureStatusNone;
  orderBefore(r, st, capturing);
  if (++r->tag == 0) r->tag = 1;
  const uint32_t tag = r->tag;
  const Geometry g{op.seg_off, op.seg_len, op.chunk_bytes};
  const uint64_t lo = op.seg_off + std::min(op.seg_len, chunk_begin * op.chunk_bytes);
  const uint64_t hi = op.seg_off + std::min(op.seg_len, stop * op.chunk_bytes);
  RailCtl ctl{};
  ctl.dev = r->ctl_dev;
  ctl.host = r->status_dev;
  ctl.tag = tag;
  if (hi <= lo) {
    if (!post.rec) {
      gateExit(op.gate, st);  // keeps the pool's ordering chain through an empty segment
      return 0;
    }
    // Nothing to reduce, but the trace-form failure is still posted.
    ctl.final_wave = op.status ? 1 : 0;
    ctl.prog_chunk = op.status ? stop : ~0ull;
    ctl.end_timeout_ns = detectNs(r, 0);
    launchBarrier(r, r->epoch + 1, true, post, ctl, st);
    r->epoch += 2;
    gateExit(op.gate, st);
    orderAfter(r, st, capturing);
    return op.status ? tag : 0;
  }
  std::vector<std::pair<uint64_t, uint64_t>> waves;
  if (llPath(r, lo, hi))
    waves.emplace_back(chunk_begin, stop);
  else
    waves = railWaves(op.chunk_bytes, chunk_begin, stop);
  for (size_t w = 0; w < waves.size(); ++w) {
    const auto [c0, c1] = waves[w];
    const bool last = w + 1 == waves.size();
    const uint64_t wlo = op.seg_off + std::min(op.seg_len, c0 * op.chunk_bytes);
    const uint64_t whi = op.seg_off + std::min(op.seg_len, c1 * op.chunk_bytes);
    ctl.final_wave = last && op.status ? 1 : 0;
    ctl.prog_chunk = op.status ? c1 : ~0ull;
    ctl.stall = stall >= 0 && static_cast<uint64_t>(stall) >= c0 && static_cast<uint64_t>(stall) < c1 ? 1 : 0;
    ctl.end_timeout_ns = detectNs(r, whi - wlo);
    railWave(r, op.in, op.out, wlo, whi, g, op.dtype, last ? post : FaultPost{}, ctl, st, op.gate);
  }
  gateExit(op.gate, st);
  orderAfter(r, st, capturing);
  return op.status ? tag : 0;
}

int railComputeCtas(nz_rail* r, uint64_t seg_len) {
  if (seg_len == 0) return 0;
  if (llPath(r, 0, seg_len)) return llGrid(r, 0, seg_len);
  if (r->comm->world == 1) return copyGrid(r, 0, seg_len);
  if (r->kind == NZ_RAIL_SM) return smGrid(r, 0, seg_len);
  return gridFor(r, seg_len, r->comm->world, r->kind == NZ_RAIL_NVLS ? 4 : 2);
}

bool railLLPath(nz_rail* r, uint64_t seg_off, uint64_t seg_len) { return llPath(r, seg_off, seg_off + seg_len); }

CUdeviceptr railGateAddr(nz_rail* r) { return reinterpret_cast<CUdeviceptr>(r->ctl_dev + kCtlGate); }

void railRevive(nz_rail* r, cudaStream_t st) {
  NZ_CUDA(cudaSetDevice(r->comm->device));
  if (!st) st = r->stream;
  orderBefore(r, st, false);
  NZ_CUDA(cudaMemsetAsync(r->ctl_dev + kCtlRetired, 0, 2 * sizeof(uint32_t), st));
  NZ_CUDA(cudaMemsetAsync(r->ctl_dev + kCtlSticky, 0, sizeof(uint32_t), st));
  NZ_CUDA(cudaStreamSynchronize(st));
  reinterpret_cast<volatile nz_rail_status_t*>(r->status_host)->abort = 0;
  *reinterpret_cast<volatile int*>(r->wd_host) = 0;
  r->stall_chunk = -1;
}

// The comm's live-rail counts (loopback co-residency budget, loopCap).
static void countLive(const nz_rail* r, int d) {
  nz_comm* c = r->comm;
  if (r->recovery) {
    c->live_twins = std::max(0, c->live_twins + d);
    return;
  }
  c->live_rails = std::max(0, c->live_rails + d);
  if (r->kind != NZ_RAIL_CE) c->live_big = std::max(0, c->live_big + d);
}

nz_rail* railCreate(nz_comm* comm, int kind, int rail_id, int sm_budget, bool graph_safe, bool recovery) {
  if (kind < NZ_RAIL_NVLS || kind > NZ_RAIL_SM) fail(NZ_ERR_INVALID, "unknown rail kind");
  if (kind == NZ_RAIL_NVLS && comm->world > 1 && !comm->multicast) {
    fail(NZ_ERR_UNSUPPORTED, comm->loop ? "NVLS rail needs NVSwitch multicast: not available to loopback ranks"
                                        : "NVLS rail requires NVSwitch multicast support");
  }
  NZ_CUDA(cudaSetDevice(comm->device));
  int pad = -1;
  bool reused = false;
  if (!comm->free_pads.empty()) {
    pad = comm->free_pads.front();
    comm->free_pads.erase(comm->free_pads.begin());
    reused = true;
  } else {
    if (comm->next_pad >= kMaxRails) fail(NZ_ERR_INVALID, "too many rails on one comm");
    pad = comm->next_pad++;
  }
  auto* r = new nz_rail();
  r->comm = comm;
  r->kind = kind;
  r->rail_id = rail_id;
  r->sm_budget = sm_budget;
  r->pad = pad;
  r->graph_safe = graph_safe;
  r->recovery = recovery;
  try {
    const size_t pad_off = kPadBytes * pad;
    r->pad_local = reinterpret_cast<uint32_t*>(comm->ctrl->ptrs[comm->rank] + pad_off);
    for (int p = 0; p < comm->world; ++p) r->pad_peer[p] = reinterpret_cast<uint32_t*>(comm->ctrl->ptrs[p] + pad_off);
    if (reused) {  // a recycled pad starts from zero epochs on every rank
      NZ_CUDA(cudaMemset(r->pad_local, 0, kPadBytes));
      NZ_CUDA(cudaDeviceSynchronize());
      exchange(comm, nullptr, 0, {});
    }
    NZ_CUDA(cudaMalloc(&r->ctl_dev, kCtlWords * sizeof(uint32_t)));
    NZ_CUDA(cudaMemset(r->ctl_dev, 0, kCtlWords * sizeof(uint32_t)));
    NZ_CUDA(cudaHostAlloc(&r->status_host, sizeof(nz_rail_status_t), cudaHostAllocMapped));
    memset(r->status_host, 0, sizeof(nz_rail_status_t));
    NZ_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&r->status_dev), r->status_host, 0));
    NZ_CUDA(cudaStreamCreateWithFlags(&r->stream, cudaStreamNonBlocking));
    NZ_CUDA(cudaEventCreateWithFlags(&r->fork, cudaEventDisableTiming));
    NZ_CUDA(cudaEventCreateWithFlags(&r->order_ev, cudaEventDisableTiming));
    if (kind == NZ_RAIL_SM && comm->world > 1 && !recovery) {
      // LL slots: [parity 2][rank N][words] x 8 bytes, zeroed on every rank
      // first. Even word count: every slot starts 16-byte aligned for the v4 pushes.
      r->ll_slot_words = ((llMaxBytes(comm->world) + 7) / 4 + 1) & ~uint64_t{1};
      r->ll = allocSymmetric(comm, 2 * comm->world * r->ll_slot_words * sizeof(uint64_t));
      r->ll_cap = r->ll_max = llMaxBytes(comm->world);
      NZ_CUDA(cudaMemset(r->ll->ptrs[comm->rank], 0, r->ll->mapped));
      NZ_CUDA(cudaDeviceSynchronize());
      exchange(comm, nullptr, 0, {});
    }
    if (kind == NZ_RAIL_CE) {
      for (int j = 0; j < 2 * (comm->world - 1); ++j) {  // gather streams, then scatter streams
        cudaStream_t s;
        cudaEvent_t e;
        NZ_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        NZ_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        r->side.push_back(s);
        r->join.push_back(e);
      }
    }
    NZ_CUDA(cudaHostAlloc(&r->fault_host, sizeof(nz_fault_record_t), cudaHostAllocMapped));
    memset(r->fault_host, 0, sizeof(nz_fault_record_t));
    NZ_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&r->fault_dev), r->fault_host, 0));
    NZ_CUDA(cudaHostAlloc(&r->wd_host, sizeof(int), cudaHostAllocMapped));
    *r->wd_host = 0;
    NZ_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&r->wd_dev), r->wd_host, 0));
    if (comm->loop && comm->world > 1) {
      NZ_CUDA(cudaEventCreateWithFlags(&r->lr_ready, cudaEventDisableTiming));
      NZ_CUDA(cudaEventCreateWithFlags(&r->lr_done, cudaEventDisableTiming));
      std::lock_guard<std::mutex> lk(comm->loop->m);
      auto& slot = comm->loop->rails[pad];
      if (!slot) {
        slot = std::make_unique<LoopRail>();
        NZ_CUDA(cudaStreamCreateWithFlags(&slot->stream, cudaStreamNonBlocking));
      }
      slot->ready[comm->rank] = r->lr_ready;
      slot->done[comm->rank] = r->lr_done;
      r->lr = slot.get();
    }
  } catch (...) {
    countLive(r, +1);  // railDestroy returns the pad and the counts
    railDestroy(r);
    throw;
  }
  countLive(r, +1);
  return r;
}

void railDestroy(nz_rail* r) {
  if (!r) return;
  nz_comm* comm = r->comm;
  cudaSetDevice(comm->device);
  if (r->stream) cudaStreamSynchronize(r->stream);
  for (auto s : r->side) {
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
  }
  for (auto e : r->join) cudaEventDestroy(e);
  if (r->lr) {
    // The group stream may still run this rank's last combined grid.
    cudaStreamSynchronize(r->lr->stream);
  }
  if (r->fork) cudaEventDestroy(r->fork);
  if (r->order_ev) cudaEventDestroy(r->order_ev);
  if (r->lr_ready) cudaEventDestroy(r->lr_ready);
  if (r->lr_done) cudaEventDestroy(r->lr_done);
  if (r->stream) cudaStreamDestroy(r->stream);
  if (r->staging) cudaFree(r->staging);
  {
    std::lock_guard<std::mutex> lk(g_retired_mu);
    auto it = g_retired.find(r);
    if (it != g_retired.end()) {
      for (char* p : it->second) cudaFree(p);
      g_retired.erase(it);
    }
  }
  if (r->ll) freeSymmetric(r->ll);
  if (r->fault_host) cudaFreeHost(r->fault_host);
  if (r->wd_host) cudaFreeHost(r->wd_host);
  if (r->status_host) cudaFreeHost(r->status_host);
  if (r->ctl_dev) cudaFree(r->ctl_dev);
  comm->free_pads.push_back(r->pad);
  countLive(r, -1);
  delete r;
}

}  // namespace nz

using nz::fail;
using nz::guarded;

extern "C" {

int nz_has_cuda_kernels(void) { return 1; }

uint64_t nz_kernel_launch_count(void) { return nz::g_launches.load(); }

int nz_rail_create(nz_comm_t* comm, int kind, int rail_id, int sm_budget, nz_rail_t** out) {
  return nz_rail_create_ex(comm, kind, rail_id, sm_budget, 0, out);
}

int nz_rail_create_ex(nz_comm_t* comm, int kind, int rail_id, int sm_budget, int flags, nz_rail_t** out) {
  return guarded([&] {
    if (!comm || !out) fail(NZ_ERR_INVALID, "null argument");
    if (flags & ~NZ_RAIL_FLAG_GRAPH_SAFE) fail(NZ_ERR_INVALID, "unknown rail flags");
    if ((flags & NZ_RAIL_FLAG_GRAPH_SAFE) && comm->loop && comm->world > 1)
      fail(NZ_ERR_UNSUPPORTED, "graph-safe rails need one process per rank (loopback launches cannot be captured)");
    *out = nz::railCreate(comm, kind, rail_id, sm_budget, (flags & NZ_RAIL_FLAG_GRAPH_SAFE) != 0, false);
  });
}

int nz_rail_destroy(nz_rail_t* r) {
  return guarded([&] { nz::railDestroy(r); });
}

int nz_rail_kind(const nz_rail_t* r) { return r ? r->kind : NZ_ERR_INVALID; }

int nz_rail_synchronize(nz_rail_t* r) {
  return guarded([&] {
    if (!r) fail(NZ_ERR_INVALID, "null rail");
    NZ_CUDA(cudaSetDevice(r->comm->device));
    for (auto s : r->side) NZ_CUDA(cudaStreamSynchronize(s));
    NZ_CUDA(cudaStreamSynchronize(r->stream));
    if (r->order_valid) NZ_CUDA(cudaEventSynchronize(r->order_ev));
  });
}
void* nz_rail_stream(const nz_rail_t* r) { return r ? static_cast<void*>(r->stream) : nullptr; }

int nz_rail_allreduce(nz_rail_t* rail, nz_buf_t* in, nz_buf_t* out, uint64_t seg_off, uint64_t seg_len,
                      uint64_t chunk_bytes, uint64_t chunk_begin, uint64_t chunk_end, int dtype, uint32_t op_seq,
                      int64_t fail_chunk, void* stream) {
  return guarded([&] {
    if (!rail || !in || !out) fail(NZ_ERR_INVALID, "null argument");
    if (rail->aborted) fail(NZ_ERR_RAIL_DOWN, "rail " + std::to_string(rail->rail_id) + " was aborted");
    if (fail_chunk < 0 && rail->armed_fail >= 0) fail_chunk = rail->armed_fail;
    rail->armed_fail = -1;
    nz::RailOp o;
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
    o.st = stream ? static_cast<cudaStream_t>(stream) : rail->stream;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    NZ_CUDA(cudaStreamIsCapturing(o.st, &cap));
    o.status = cap == cudaStreamCaptureStatusNone;
    nz::railRun(rail, o);
    const uint64_t nch = chunk_bytes ? (seg_len + chunk_bytes - 1) / chunk_bytes : 0;
    const uint64_t end = std::min(chunk_end, nch);
    rail->last_tag = rail->tag;
    rail->prog_begin = std::min(chunk_begin, end);
    rail->prog_stop = fail_chunk >= 0 && static_cast<uint64_t>(fail_chunk) >= rail->prog_begin &&
                              static_cast<uint64_t>(fail_chunk) < end
                          ? static_cast<uint64_t>(fail_chunk)
                          : end;
    rail->prog_valid = o.status;
  });
}

int nz_rail_inject_failure(nz_rail_t* rail, uint64_t chunk) {
  return guarded([&] {
    if (!rail) fail(NZ_ERR_INVALID, "null rail");
    if (chunk > static_cast<uint64_t>(INT64_MAX)) fail(NZ_ERR_INVALID, "chunk out of range");
    rail->armed_fail = static_cast<int64_t>(chunk);
  });
}

int nz_rail_inject_stall(nz_rail_t* rail, uint64_t chunk) {
  return guarded([&] {
    if (!rail) fail(NZ_ERR_INVALID, "null rail");
    if (chunk > static_cast<uint64_t>(INT64_MAX)) fail(NZ_ERR_INVALID, "chunk out of range");
    rail->stall_chunk = static_cast<int64_t>(chunk);
  });
}

int nz_rail_revive(nz_rail_t* rail) {
  return guarded([&] {
    if (!rail) fail(NZ_ERR_INVALID, "null rail");
    nz::railRevive(rail, nullptr);
  });
}

int nz_rail_set_detect_us(nz_rail_t* rail, double us) {
  return guarded([&] {
    if (!rail || !(us >= 0)) fail(NZ_ERR_INVALID, "bad argument");
    rail->detect_us = us;
  });
}

int nz_rail_loop_timing(nz_rail_t* rail, int enable) {
  return guarded([&] {
    if (!rail) fail(NZ_ERR_INVALID, "null rail");
    if (!rail->lr) fail(NZ_ERR_INVALID, "not a loopback rail");
    std::lock_guard<std::mutex> lk(rail->lr->m);
    rail->lr->timing = enable != 0;
  });
}

int nz_rail_loop_time(nz_rail_t* rail, uint64_t* launches, double* total_us) {
  return guarded([&] {
    if (!rail || !launches || !total_us) fail(NZ_ERR_INVALID, "null argument");
    if (!rail->lr) fail(NZ_ERR_INVALID, "not a loopback rail");
    nz::LoopRail& L = *rail->lr;
    std::lock_guard<std::mutex> lk(L.m);
    NZ_CUDA(cudaSetDevice(rail->comm->device));
    NZ_CUDA(cudaStreamSynchronize(L.stream));
    double us = 0;
    for (size_t i = 0; i < L.tev_used; ++i) {
      float ms = 0;
      NZ_CUDA(cudaEventElapsedTime(&ms, L.tev[i].first, L.tev[i].second));
      us += static_cast<double>(ms) * 1000.0;
    }
    *launches = L.tev_used;
    *total_us = us;
    L.tev_used = 0;
  });
}

int nz_rail_status(const nz_rail_t* rail, nz_rail_status_t* out) {
  return guarded([&] {
    if (!rail || !out) fail(NZ_ERR_INVALID, "null argument");
    const volatile nz_rail_status_t* s = rail->status_host;
    out->ok_tag = s->ok_tag;
    out->prog_tag = s->prog_tag;
    out->prog_chunk = s->prog_chunk;
    out->start_tag = s->start_tag;
    out->fail_tag = s->fail_tag;
    out->t_start_ns = s->t_start_ns;
    out->t_fail_ns = s->t_fail_ns;
    out->det_tag = s->det_tag;
    out->abort = s->abort;
    out->t_det_ns = s->t_det_ns;
  });
}

int nz_rail_progress(nz_rail_t* rail, uint64_t* chunks_done) {
  return guarded([&] {
    if (!rail || !chunks_done) fail(NZ_ERR_INVALID, "null argument");
    if (!rail->prog_valid) {
      *chunks_done = 0;
      return;
    }
    const volatile nz_rail_status_t* s = rail->status_host;
    if (s->ok_tag == rail->last_tag) {
      *chunks_done = rail->prog_stop;
    } else if (s->prog_tag == rail->last_tag) {
      *chunks_done = std::min<uint64_t>(static_cast<uint64_t>(s->prog_chunk), rail->prog_stop);
    } else {
      *chunks_done = rail->prog_begin;
    }
  });
}

int nz_rail_abort(nz_rail_t* rail) {
  return guarded([&] {
    if (!rail) fail(NZ_ERR_INVALID, "null rail");
    rail->aborted = true;
    rail->armed_fail = -1;
  });
}

int nz_event_elapsed_us(void* start, void* end, double* us) {
  return guarded([&] {
    if (!start || !end || !us) fail(NZ_ERR_INVALID, "null argument");
    float ms = 0;
    NZ_CUDA(cudaEventElapsedTime(&ms, static_cast<cudaEvent_t>(start), static_cast<cudaEvent_t>(end)));
    *us = static_cast<double>(ms) * 1000.0;
  });
}

int nz_emulate_fold(int world, int rank, int dtype, const void* const* src, void* const* dst, int ndst,
                    uint64_t seg_off, uint64_t seg_len, uint64_t chunk_bytes, uint64_t lo, uint64_t hi, int grid,
                    void* stream) {
  return guarded([&] {
    if (world < 1 || world > nz::kMaxRanks || rank < 0 || rank >= world) fail(NZ_ERR_INVALID, "bad world/rank");
    if (!src || !dst || (ndst != 1 && ndst != world)) fail(NZ_ERR_INVALID, "bad src/dst");
    const int es = nz::elemSize(dtype);
    if (chunk_bytes == 0 || chunk_bytes % es || seg_off % es || seg_len % es || lo % es || hi % es || lo > hi ||
        lo < seg_off || hi > seg_off + seg_len) {
      fail(NZ_ERR_INVALID, "bad geometry");
    }
    nz::FoldArgs a{};
    for (int p = 0; p < world; ++p) a.src[p] = static_cast<const char*>(src[p]);
    for (int d = 0; d < ndst; ++d) a.dst[d] = static_cast<char*>(dst[d]);
    nz::shardOf(lo, hi, rank, world, &a.s, &a.e);
    a.range_bytes = hi - lo;
    a.g = nz::Geometry{seg_off, seg_len, chunk_bytes};
    a.use_barrier = 0;
    a.rank = rank;
    int dev = 0, sms = 0;
    NZ_CUDA(cudaGetDevice(&dev));
    NZ_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (grid <= 0) {
      const uint64_t per_rank_vec = (hi - lo) / 16 / world + 1;
      grid = static_cast<int>(std::min<uint64_t>(sms, (per_rank_vec + 2 * nz::kThreads - 1) / (2 * nz::kThreads)));
      grid = std::max(grid, 1);
    }
    if (ndst == 1)
      nz::dispatchFold<0>(world, dtype, a, grid, static_cast<cudaStream_t>(stream));
    else
      nz::dispatchFold<1>(world, dtype, a, grid, static_cast<cudaStream_t>(stream));
    NZ_CUDA(cudaGetLastError());
  });
}

int nz_rail_poll_fault(nz_rail_t* r, nz_fault_record_t* rec, int consume) {
  return guarded([&] {
    if (!r || !rec) fail(NZ_ERR_INVALID, "null argument");
    volatile nz_fault_record_t* f = r->fault_host;
    rec->valid = f->valid;
    if (!rec->valid) return;
    __sync_synchronize();
    rec->op_seq = f->op_seq;
    rec->chunk = f->chunk;
    rec->t_fail_ns = f->t_fail_ns;
    if (consume) f->valid = 0;
  });
}

int nz_rail_watchdog(nz_rail_t* r) {
  if (!r) return NZ_ERR_INVALID;
  volatile int* w = r->wd_host;
  const int v = *w;
  *w = 0;
  return v;
}

}  // extern "C"
