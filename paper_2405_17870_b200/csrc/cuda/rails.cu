// Host side of the three rails: launch configuration, DMA phases of the
// copy-engine rail, fault records. One nz_rail per (rank, rail); each owns a
// CUDA stream, which is the B200 form of the reference's "one collective
// executor per rail".
#include <algorithm>
#include <atomic>
#include <cstring>

#include "internal.h"
#include "kernels.cuh"

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

// Device wait budget before a kernel gives up on a peer (watchdog).
// NEZHA_WATCHDOG_MS overrides the 20 s default (tests use a short one).
uint64_t watchdogNs() {
  static const uint64_t ns = [] {
    const char* e = getenv("NEZHA_WATCHDOG_MS");
    const long long ms = e ? atoll(e) : 20000;
    return static_cast<uint64_t>(ms > 0 ? ms : 20000) * 1000000ull;
  }();
  return ns;
}

// NEZHA_BARRIER_POLL=relaxed: barrier waits poll with relaxed loads and fence
// once (A/B knob; the default acquire-load poll is the validated one).
bool barrierRelaxedPoll() {
  static const bool on = [] {
    const char* e = getenv("NEZHA_BARRIER_POLL");
    return e && strcmp(e, "relaxed") == 0;
  }();
  return on;
}

BarrierArgs barrierArgs(nz_rail* r, uint32_t epoch) {
  BarrierArgs b{};
  b.local = r->pad_local;
  for (int p = 0; p < r->comm->world; ++p) b.peer[p] = r->pad_peer[p];
  b.epoch = epoch;
  b.watchdog = r->wd_dev;
  b.timeout_ns = watchdogNs();
  b.relaxed_poll = barrierRelaxedPoll() ? 1 : 0;
  b.seq = r->seq_dev;
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

template <typename DT, int N, int NDST>
void launchFold(const FoldArgs& a, int grid, cudaStream_t st) {
  fold_kernel<DT, N, NDST><<<grid, kThreads, 0, st>>>(a);
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

template <int N, int NDST>
void dispatchFoldDT(int dtype, const FoldArgs& a, int grid, cudaStream_t st) {
  switch (dtype) {
    case NZ_F32: return launchFold<F32, N, NDST>(a, grid, st);
    case NZ_BF16: return launchFold<BF16, N, NDST>(a, grid, st);
    case NZ_I32: return launchFold<I32, N, NDST>(a, grid, st);
  }
}

// SM-rail TMA pipeline (K3t). Opt-in with NEZHA_SM_TMA=1 until its sweep is
// committed; nz_emulate_fold_tma runs it on one GPU for the parity tests.
bool smTmaEnabled() {
  static const bool on = [] {
    const char* e = getenv("NEZHA_SM_TMA");
    return e && atoi(e) != 0;
  }();
  return on;
}

template <typename DT, int N>
void launchTmaDT(const FoldArgs& a, int grid, cudaStream_t st) {
  static bool configured = false;  // opt in to > 48 KiB of dynamic shared memory once
  const size_t smem = tma_smem_bytes(N);
  if (!configured) {
    NZ_CUDA(cudaFuncSetAttribute(sm_tma_kernel<DT, N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
    configured = true;
  }
  sm_tma_kernel<DT, N><<<grid, 256, smem, st>>>(a);
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

void dispatchTma(int world, int dtype, const FoldArgs& a, int grid, cudaStream_t st) {
  switch (world) {
#define NZ_CASE(n)                                                    \
  case n:                                                             \
    if (dtype == NZ_F32) return launchTmaDT<F32, n>(a, grid, st);     \
    if (dtype == NZ_BF16) return launchTmaDT<BF16, n>(a, grid, st);   \
    return launchTmaDT<I32, n>(a, grid, st);
    NZ_CASE(2) NZ_CASE(3) NZ_CASE(4) NZ_CASE(5) NZ_CASE(6) NZ_CASE(7) NZ_CASE(8)
#undef NZ_CASE
  }
}

template <int NDST_IS_N>
void dispatchFold(int world, int dtype, const FoldArgs& a, int grid, cudaStream_t st) {
  switch (world) {
#define NZ_CASE(n) \
  case n: return dispatchFoldDT<n, NDST_IS_N ? n : 1>(dtype, a, grid, st);
    NZ_CASE(1) NZ_CASE(2) NZ_CASE(3) NZ_CASE(4) NZ_CASE(5) NZ_CASE(6) NZ_CASE(7) NZ_CASE(8)
#undef NZ_CASE
  }
}

constexpr uint64_t kLLMaxBytes = 2048 * 1024;  // SM rail one-shot LL path up to this payload

// LL pays 2 wire bytes per payload byte times N receivers; beyond ~4 MiB / N
// the two-shot kernels win (measured crossover, profiles/README.md).
// The multicast push (NVLS-LL) saturates earlier than the unicast one: at
// N = 4 it is 9.1 us at 256 KiB but 24.8 us at 1 MiB vs 20 us two-shot.
uint64_t llMaxBytes(int world, bool mc) {
  const uint64_t cap = mc ? (uint64_t{512} << 10) : kLLMaxBytes;
  // NEZHA_LL_MAX (bytes) lowers the ceiling for sweeps; it never raises it
  // (the LL buffers are sized by this function at rail creation).
  static const long long env = [] {
    const char* e = getenv("NEZHA_LL_MAX");
    return e ? atoll(e) : -1LL;
  }();
  const uint64_t def = std::min<uint64_t>(cap, (uint64_t{4} << 20) / world);
  return env >= 0 ? std::min<uint64_t>(def, static_cast<uint64_t>(env)) : def;
}

template <int N, bool MC>
void launchLL(int dtype, const LLArgs& a, int grid, cudaStream_t st) {
  if (dtype == NZ_F32) return (void)(ll_kernel<F32, N, MC><<<grid, kThreads, 0, st>>>(a));
  if (dtype == NZ_BF16) return (void)(ll_kernel<BF16, N, MC><<<grid, kThreads, 0, st>>>(a));
  return (void)(ll_kernel<I32, N, MC><<<grid, kThreads, 0, st>>>(a));
}

void dispatchLL(int world, int dtype, bool mc, const LLArgs& a, int grid, cudaStream_t st) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  switch (world) {
#define NZ_CASE(n) \
  case n:          \
    return mc ? launchLL<n, true>(dtype, a, grid, st) : launchLL<n, false>(dtype, a, grid, st);
    NZ_CASE(2) NZ_CASE(3) NZ_CASE(4) NZ_CASE(5) NZ_CASE(6) NZ_CASE(7) NZ_CASE(8)
#undef NZ_CASE
  }
}

// NVLS loop variant: unroll U and memory semantics. NEZHA_NVLS_VARIANT
// (0: U4 relaxed.sys, 1: U4 weak, 2: U8 relaxed.sys, 3: U8 weak) is a tuning
// knob for the sweeps recorded in profiles/; the default is variant 0.
int nvlsVariant() {
  static const int v = [] {
    const char* e = getenv("NEZHA_NVLS_VARIANT");
    const int x = e ? atoi(e) : 0;
    return (x >= 0 && x <= 3) ? x : 0;
  }();
  return v;
}

template <typename DT, int N>
void launchNvlsDT(const NvlsArgs& a, int grid, cudaStream_t st) {
  switch (nvlsVariant()) {
    case 1: nvls_kernel<DT, N, 4, true><<<grid, kThreads, 0, st>>>(a); return;
    case 2: nvls_kernel<DT, N, 8, false><<<grid, kThreads, 0, st>>>(a); return;
    case 3: nvls_kernel<DT, N, 8, true><<<grid, kThreads, 0, st>>>(a); return;
    default: nvls_kernel<DT, N, 4, false><<<grid, kThreads, 0, st>>>(a); return;
  }
}

template <int N>
void launchNvls(int dtype, const NvlsArgs& a, int grid, cudaStream_t st) {
  if (dtype == NZ_F32) return launchNvlsDT<F32, N>(a, grid, st);
  if (dtype == NZ_BF16) return launchNvlsDT<BF16, N>(a, grid, st);
  return launchNvlsDT<I32, N>(a, grid, st);
}

void dispatchNvls(int world, int dtype, const NvlsArgs& a, int grid, cudaStream_t st) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  switch (world) {
#define NZ_CASE(n)                                                                          \
  case n:                                                                                   \
    return launchNvls<n>(dtype, a, grid, st);
    NZ_CASE(2) NZ_CASE(3) NZ_CASE(4) NZ_CASE(5) NZ_CASE(6) NZ_CASE(7) NZ_CASE(8)
#undef NZ_CASE
  }
}

void launchBarrier(nz_rail* r, uint32_t epoch, FaultPost post, cudaStream_t st) {
  const BarrierArgs b = barrierArgs(r, epoch);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  switch (r->comm->world) {
#define NZ_CASE(n) \
  case n: barrier_kernel<n><<<1, 32, 0, st>>>(b, r->comm->rank, post); break;
    NZ_CASE(1) NZ_CASE(2) NZ_CASE(3) NZ_CASE(4) NZ_CASE(5) NZ_CASE(6) NZ_CASE(7) NZ_CASE(8)
#undef NZ_CASE
  }
}

void ensureStaging(nz_rail* r, size_t slot) {
  if (slot <= r->staging_slot) return;
  if (r->staging) NZ_CUDA(cudaFree(r->staging));
  r->staging = nullptr;
  const size_t want = (slot + (1u << 20)) & ~((size_t(1) << 20) - 1);
  NZ_CUDA(cudaMalloc(&r->staging, want * std::max(1, r->comm->world - 1)));
  r->staging_slot = want;
}

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

// NVLS-LL (one-shot multicast push) is opt-in: NEZHA_NVLS_LL=1. The only
// NVLink error incident of this project came from a multicast store path
// (profiles/README.md); until its fixed form has a clean hardware record the
// NVLS rail runs small payloads two-shot, and the planner sends them to the
// SM rail's unicast LL path, which is as fast.
bool nvlsLLEnabled() {
  static const bool on = [] {
    const char* e = getenv("NEZHA_NVLS_LL");
    return e && atoi(e) != 0;
  }();
  return on;
}

// SM-rail one-shot (K7) for payloads between the LL ceiling and
// min(4 MiB, 8 MiB / N): opt-in with NEZHA_SM_ONESHOT=1 until its sweep is in
// profiles/. NEZHA_SM_ONESHOT_MAX overrides the ceiling (bytes).
bool oneshotEnabled() {
  static const bool on = [] {
    const char* e = getenv("NEZHA_SM_ONESHOT");
    return e && atoi(e) != 0;
  }();
  return on;
}

uint64_t oneshotMaxBytes(int world) {
  static const long long env = [] {
    const char* e = getenv("NEZHA_SM_ONESHOT_MAX");
    return e ? atoll(e) : 0LL;
  }();
  const uint64_t def = std::min<uint64_t>(uint64_t{4} << 20, (uint64_t{8} << 20) / world);
  return env > 0 ? std::min<uint64_t>(static_cast<uint64_t>(env), uint64_t{16} << 20) : def;
}

bool oneshotPath(nz_rail* r, uint64_t lo, uint64_t hi) {
  return r->comm->world > 1 && r->kind == NZ_RAIL_SM && r->os && hi > lo && hi - lo <= r->os_max &&
         hi - (lo & ~15ull) <= r->os_slot;
}

int oneshotGrid(nz_rail* r, uint64_t lo, uint64_t hi) {
  const int budget = std::min(r->sm_budget > 0 ? r->sm_budget : 64, r->comm->sm_count);
  const uint64_t vec = (hi - lo) / 16 + 1;
  const uint64_t g = (vec + 2 * kThreads - 1) / (2 * kThreads);
  return static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(g, std::min(budget, kMaxCtas))));
}

template <typename DT>
void launchOneshotDT(int world, const OneShotArgs& a, int grid, cudaStream_t st) {
  switch (world) {
#define NZ_CASE(n) \
  case n: oneshot_kernel<DT, n><<<grid, kThreads, 0, st>>>(a); break;
    NZ_CASE(2) NZ_CASE(3) NZ_CASE(4) NZ_CASE(5) NZ_CASE(6) NZ_CASE(7) NZ_CASE(8)
#undef NZ_CASE
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

bool llPath(nz_rail* r, uint64_t lo, uint64_t hi) {
  const int N = r->comm->world;
  const bool mc_ll = r->kind == NZ_RAIL_NVLS;
  return N > 1 && (r->kind == NZ_RAIL_SM || mc_ll) && r->ll && hi - lo <= r->ll_max && lo % 4 == 0 &&
         (!mc_ll || r->ll->mc_ptr);
}

int llGrid(nz_rail* r, uint64_t lo, uint64_t hi) {
  const uint64_t words = (hi - lo + 3) / 4;
  const uint64_t threads = (words + 1) / 2 > words ? (words + 1) / 2 : words;
  return static_cast<int>(
      std::max<uint64_t>(1, std::min<uint64_t>((threads + kThreads - 1) / kThreads, r->comm->sm_count)));
}

int copyGrid(nz_rail* r, uint64_t lo, uint64_t hi) {
  const uint64_t vec = (hi - lo) / 16 + 1;
  return static_cast<int>(
      std::max<uint64_t>(1, std::min<uint64_t>((vec + kThreads * 8 - 1) / (kThreads * 8), 2ull * r->comm->sm_count)));
}

int smGrid(nz_rail* r, uint64_t lo, uint64_t hi) {
  const int N = r->comm->world;
  if (smTmaEnabled()) {
    const uint64_t tiles = (hi - lo) / N / kTmaTile + 1;
    return static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(tiles, gridFor(r, hi - lo, N, 2))));
  }
  return gridFor(r, hi - lo, N, 2);
}

// One rail op over [lo, hi) with order geometry g. `post` is posted after.
void railOp(nz_rail* r, nz_buf* in, nz_buf* out, uint64_t lo, uint64_t hi, const Geometry& g, int dtype, FaultPost post,
            cudaStream_t st, ComputeGate* gate) {
  nz_comm* c = r->comm;
  const int N = c->world;
  const int me = c->rank;
  uint64_t s, e;
  shardOf(lo, hi, me, N, &s, &e);
  const uint32_t epoch = r->epoch + 1;
  r->epoch += 2;  // start + end barrier; identical on every rank

  const bool mc_ll = r->kind == NZ_RAIL_NVLS;
  if (llPath(r, lo, hi)) {
    LLArgs a{};
    a.in = in->ptrs[me];
    a.out = out->ptrs[me];
    for (int p = 0; p < N; ++p) a.peer[p] = reinterpret_cast<uint64_t*>(r->ll->ptrs[p]);
    a.local = reinterpret_cast<uint64_t*>(r->ll->ptrs[me]);
    a.mc = reinterpret_cast<uint64_t*>(r->ll->mc_ptr);
    // Every 16-byte push (unicast v4 or multimem.st) must be 16-byte aligned:
    // a misaligned multimem store is not a clean trap on NVSwitch.
    if ((r->ll_slot_words & 1u) != 0 || reinterpret_cast<uintptr_t>(r->ll->ptrs[me]) % 16 != 0 ||
        (a.mc && reinterpret_cast<uintptr_t>(a.mc) % 16 != 0)) {
      fail(NZ_ERR_INVALID, "LL slots are not 16-byte aligned");
    }
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
    a.seq = r->seq_dev;
    gateEnter(gate, st);
    dispatchLL(N, dtype, mc_ll, a, gated(llGrid(r, lo, hi), gate), st);
    NZ_CUDA(cudaGetLastError());
    gateExit(gate, st);
    return;
  }

  if (oneshotPath(r, lo, hi)) {
    OneShotArgs a{};
    a.in = in->ptrs[me];
    for (int p = 0; p < N; ++p) a.stg_peer[p] = r->os->ptrs[p];
    a.lo = lo;
    a.hi = hi;
    a.lo16 = lo & ~15ull;
    a.slot_bytes = r->os_slot;
    a.bar = barrierArgs(r, epoch);
    a.rank = me;
    a.post = post;
    for (int par = 0; par < 2; ++par) {
      FoldArgs& f = a.f[par];
      for (int p = 0; p < N; ++p) {
        f.src[p] = p == me ? in->ptrs[me]
                           : r->os->ptrs[me] + (static_cast<uint64_t>(par) * N + p) * r->os_slot - a.lo16;
      }
      f.dst[0] = out->ptrs[me];
      f.s = lo;
      f.e = hi;
      f.range_bytes = hi - lo;
      f.g = g;
      f.rank = me;
    }
    gateEnter(gate, st);
    const int grid = gated(oneshotGrid(r, lo, hi), gate);
    if (dtype == NZ_F32) launchOneshotDT<F32>(N, a, grid, st);
    else if (dtype == NZ_BF16) launchOneshotDT<BF16>(N, a, grid, st);
    else launchOneshotDT<I32>(N, a, grid, st);
    NZ_CUDA(cudaGetLastError());
    gateExit(gate, st);
    return;
  }

  if (N == 1) {  // identity allreduce: every rail is a local HBM copy
    gateEnter(gate, st);
    copy_kernel<<<gated(copyGrid(r, lo, hi), gate), kThreads, 0, st>>>(in->ptrs[0], out->ptrs[0], lo, hi, post);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    NZ_CUDA(cudaGetLastError());
    gateExit(gate, st);
    return;
  }

  if (r->kind == NZ_RAIL_SM) {
    FoldArgs a{};
    for (int p = 0; p < N; ++p) {
      a.src[p] = in->ptrs[p];
      a.dst[p] = out->ptrs[p];
    }
    a.s = N == 1 ? lo : s;
    a.e = N == 1 ? hi : e;
    a.range_bytes = hi - lo;
    a.g = g;
    a.bar = barrierArgs(r, epoch);
    a.use_barrier = N > 1;
    a.rank = me;
    a.post = post;
    gateEnter(gate, st);
    const int grid = gated(smGrid(r, lo, hi), gate);
    if (smTmaEnabled()) {
      dispatchTma(N, dtype, a, grid, st);
    } else {
      dispatchFold<1>(N, dtype, a, grid, st);
    }
    NZ_CUDA(cudaGetLastError());
    gateExit(gate, st);
    return;
  }

  if (r->kind == NZ_RAIL_NVLS) {
    if (!in->mc_ptr || !out->mc_ptr) fail(NZ_ERR_UNSUPPORTED, "NVLS rail needs multicast-bound buffers");
    NvlsArgs a{};
    if (reinterpret_cast<uintptr_t>(in->mc_ptr) % 16 != 0 || reinterpret_cast<uintptr_t>(out->mc_ptr) % 16 != 0) {
      fail(NZ_ERR_INVALID, "multicast windows must be 16-byte aligned");
    }
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
    gateEnter(gate, st);
    dispatchNvls(N, dtype, a, gated(gridFor(r, hi - lo, N, 4), gate), st);
    NZ_CUDA(cudaGetLastError());
    gateExit(gate, st);
    return;
  }

  // Copy-engine rail: barrier, DMA gather of my shard from every peer,
  // local ring-order reduce, DMA scatter of the sum, barrier.
  const uint64_t len = e - s;
  // Staged copies keep the 16-byte phase of the source so the reduce kernel's
  // vector loads stay aligned: copy from s16 = align_down(s, 16).
  const uint64_t s16 = s & ~15ull;
  const uint64_t slen = e - s16;
  ensureStaging(r, slen);
  launchBarrier(r, epoch, FaultPost{}, st);
  if (len > 0) {
    NZ_CUDA(cudaEventRecord(r->fork, st));
    for (int j = 1; j < N; ++j) {
      const int p = (me + j) % N;
      cudaStream_t ss = r->side[j - 1];
      NZ_CUDA(cudaStreamWaitEvent(ss, r->fork, 0));
      NZ_CUDA(cudaMemcpyAsync(r->staging + (j - 1) * r->staging_slot, in->ptrs[p] + s16, slen, cudaMemcpyDeviceToDevice, ss));
      NZ_CUDA(cudaEventRecord(r->join[j - 1], ss));
      NZ_CUDA(cudaStreamWaitEvent(st, r->join[j - 1], 0));
    }
    FoldArgs a{};
    for (int p = 0; p < N; ++p) {
      const int j = (p - me + N) % N;
      a.src[p] = j == 0 ? in->ptrs[me] : r->staging + (j - 1) * r->staging_slot - s16;
    }
    a.dst[0] = out->ptrs[me];
    a.s = s;
    a.e = e;
    a.range_bytes = hi - lo;
    a.g = g;
    a.use_barrier = 0;
    a.rank = me;
    gateEnter(gate, st);  // computation phase: the local fold
    dispatchFold<0>(N, dtype, a, gated(gridFor(r, hi - lo, N, 2), gate), st);
    NZ_CUDA(cudaGetLastError());
    gateExit(gate, st);
    NZ_CUDA(cudaEventRecord(r->fork, st));
    for (int j = 1; j < N; ++j) {
      const int p = (me + j) % N;
      cudaStream_t ss = r->side[j - 1];
      NZ_CUDA(cudaStreamWaitEvent(ss, r->fork, 0));
      NZ_CUDA(cudaMemcpyAsync(out->ptrs[p] + s, out->ptrs[me] + s, len, cudaMemcpyDeviceToDevice, ss));
      NZ_CUDA(cudaEventRecord(r->join[j - 1], ss));
      NZ_CUDA(cudaStreamWaitEvent(st, r->join[j - 1], 0));
    }
  }
  launchBarrier(r, epoch + 1, post, st);
  NZ_CUDA(cudaGetLastError());
  gateExit(gate, st);  // empty shard: nothing was folded
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

// Used by the engine (engine.cpp) without going through the C ABI.
void railAllreduce(nz_rail* r, nz_buf* in, nz_buf* out, uint64_t seg_off, uint64_t seg_len, uint64_t chunk_bytes,
                   uint64_t chunk_begin, uint64_t chunk_end, int dtype, uint32_t op_seq, int64_t fail_chunk,
                   cudaStream_t st, ComputeGate* gate) {
  const int es = elemSize(dtype);
  if (chunk_bytes == 0 || chunk_bytes % es || seg_off % es || seg_len % es) {
    fail(NZ_ERR_INVALID, "segment geometry not element aligned");
  }
  if (in->comm != r->comm || out->comm != r->comm) fail(NZ_ERR_INVALID, "buffer from another comm");
  if (seg_off + seg_len > in->size || seg_off + seg_len > out->size) fail(NZ_ERR_INVALID, "segment exceeds buffer");
  const uint64_t nch = (seg_len + chunk_bytes - 1) / chunk_bytes;
  chunk_end = std::min(chunk_end, nch);
  if (chunk_begin > chunk_end) fail(NZ_ERR_INVALID, "chunk_begin > chunk_end");
  uint64_t stop = chunk_end;
  FaultPost post{};
  if (fail_chunk >= 0 && static_cast<uint64_t>(fail_chunk) >= chunk_begin && static_cast<uint64_t>(fail_chunk) < chunk_end) {
    stop = static_cast<uint64_t>(fail_chunk);
    post.rec = r->fault_dev;
    post.op_seq = op_seq;
    post.chunk = stop;
  }
  const uint64_t lo = seg_off + std::min(seg_len, chunk_begin * chunk_bytes);
  const uint64_t hi = seg_off + std::min(seg_len, stop * chunk_bytes);
  if (!st) st = r->stream;
  NZ_CUDA(cudaSetDevice(r->comm->device));
  if (hi > lo) {
    railOp(r, in, out, lo, hi, Geometry{seg_off, seg_len, chunk_bytes}, dtype, post, st, gate);
  } else if (post.rec) {
    launchBarrier(r, r->epoch + 1, post, st);
    r->epoch += 2;
  }
  gateExit(gate, st);
}

int railComputeCtas(nz_rail* r, uint64_t seg_len) {
  if (seg_len == 0) return 0;
  if (llPath(r, 0, seg_len)) return llGrid(r, 0, seg_len);
  if (oneshotPath(r, 0, seg_len)) return oneshotGrid(r, 0, seg_len);
  if (r->comm->world == 1) return copyGrid(r, 0, seg_len);
  if (r->kind == NZ_RAIL_SM) return smGrid(r, 0, seg_len);
  return gridFor(r, seg_len, r->comm->world, r->kind == NZ_RAIL_NVLS ? 4 : 2);
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
    if (kind < NZ_RAIL_NVLS || kind > NZ_RAIL_SM) fail(NZ_ERR_INVALID, "unknown rail kind");
    if (kind == NZ_RAIL_NVLS && comm->world > 1 && !comm->multicast) {
      fail(NZ_ERR_UNSUPPORTED, "NVLS rail requires NVSwitch multicast support");
    }
    if (comm->next_pad >= nz::kMaxRails) fail(NZ_ERR_INVALID, "too many rails on one comm");
    NZ_CUDA(cudaSetDevice(comm->device));
    auto* r = new nz_rail();
    r->comm = comm;
    r->kind = kind;
    r->rail_id = rail_id;
    if (flags & NZ_RAIL_FLAG_GRAPH_SAFE) {  // device op counter (kernels.cuh seq_retire), zero on every rank
      NZ_CUDA(cudaMalloc(&r->seq_dev, 2 * sizeof(uint32_t)));
      NZ_CUDA(cudaMemset(r->seq_dev, 0, 2 * sizeof(uint32_t)));
    }
    r->sm_budget = sm_budget;
    const size_t pad_off = nz::kPadBytes * comm->next_pad++;
    r->pad_local = reinterpret_cast<uint32_t*>(comm->ctrl->ptrs[comm->rank] + pad_off);
    for (int p = 0; p < comm->world; ++p) r->pad_peer[p] = reinterpret_cast<uint32_t*>(comm->ctrl->ptrs[p] + pad_off);
    NZ_CUDA(cudaStreamCreateWithFlags(&r->stream, cudaStreamNonBlocking));
    NZ_CUDA(cudaEventCreateWithFlags(&r->fork, cudaEventDisableTiming));
    if ((kind == NZ_RAIL_SM || (kind == NZ_RAIL_NVLS && nz::nvlsLLEnabled())) && comm->world > 1) {
      // LL slots: [parity 2][rank N][kLLMaxBytes / 4 words] x 8 bytes, zeroed on every rank first.
      // Even word count: every slot starts 16-byte aligned for the v4 pushes.
      r->ll_slot_words = ((nz::llMaxBytes(comm->world, kind == NZ_RAIL_NVLS) + 7) / 4 + 1) & ~uint64_t{1};
      r->ll = nz::allocSymmetric(comm, 2 * comm->world * r->ll_slot_words * sizeof(uint64_t));
      r->ll_cap = r->ll_max = nz::llMaxBytes(comm->world, kind == NZ_RAIL_NVLS);
      NZ_CUDA(cudaMemset(r->ll->ptrs[comm->rank], 0, r->ll->mapped));
      NZ_CUDA(cudaDeviceSynchronize());
      nz::exchange(comm, nullptr, 0, {});
    }
    if (kind == NZ_RAIL_SM && comm->world > 1 && nz::oneshotEnabled()) {
      r->os_slot = (nz::oneshotMaxBytes(comm->world) + 16 + 255) & ~uint64_t{255};
      r->os = nz::allocSymmetric(comm, 2 * comm->world * r->os_slot);
      r->os_cap = r->os_max = nz::oneshotMaxBytes(comm->world);
    }
    if (kind == NZ_RAIL_CE) {
      for (int j = 1; j < comm->world; ++j) {
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
    *out = r;
  });
}

int nz_rail_destroy(nz_rail_t* r) {
  return guarded([&] {
    if (!r) return;
    cudaSetDevice(r->comm->device);
    cudaStreamSynchronize(r->stream);
    for (auto s : r->side) cudaStreamDestroy(s);
    for (auto e : r->join) cudaEventDestroy(e);
    if (r->fork) cudaEventDestroy(r->fork);
    if (r->stream) cudaStreamDestroy(r->stream);
    if (r->staging) cudaFree(r->staging);
    if (r->ll) nz::freeSymmetric(r->ll);
    if (r->fault_host) cudaFreeHost(r->fault_host);
    if (r->wd_host) cudaFreeHost(r->wd_host);
    if (r->done) cudaEventDestroy(r->done);
    if (r->seq_dev) cudaFree(r->seq_dev);
    if (r->os) nz::freeSymmetric(r->os);
    delete r;
  });
}

int nz_rail_kind(const nz_rail_t* r) { return r ? r->kind : NZ_ERR_INVALID; }

int nz_rail_synchronize(nz_rail_t* r) {
  return guarded([&] {
    if (!r) fail(NZ_ERR_INVALID, "null rail");
    NZ_CUDA(cudaSetDevice(r->comm->device));
    for (auto s : r->side) NZ_CUDA(cudaStreamSynchronize(s));
    NZ_CUDA(cudaStreamSynchronize(r->stream));
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
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : rail->stream;
    nz::railAllreduce(rail, in, out, seg_off, seg_len, chunk_bytes, chunk_begin, chunk_end, dtype, op_seq, fail_chunk,
                      st);
    const uint64_t nch = chunk_bytes ? (seg_len + chunk_bytes - 1) / chunk_bytes : 0;
    const uint64_t end = std::min(chunk_end, nch);
    rail->prog_begin = std::min(chunk_begin, end);
    rail->prog_stop = fail_chunk >= 0 && static_cast<uint64_t>(fail_chunk) >= rail->prog_begin &&
                              static_cast<uint64_t>(fail_chunk) < end
                          ? static_cast<uint64_t>(fail_chunk)
                          : end;
    if (!rail->done) NZ_CUDA(cudaEventCreateWithFlags(&rail->done, cudaEventDisableTiming));
    NZ_CUDA(cudaEventRecord(rail->done, st));
    rail->prog_valid = true;
  });
}

int nz_rail_inject_failure(nz_rail_t* rail, uint64_t chunk) {
  return guarded([&] {
    if (!rail) fail(NZ_ERR_INVALID, "null rail");
    if (chunk > static_cast<uint64_t>(INT64_MAX)) fail(NZ_ERR_INVALID, "chunk out of range");
    rail->armed_fail = static_cast<int64_t>(chunk);
  });
}

int nz_rail_progress(nz_rail_t* rail, uint64_t* chunks_done) {
  return guarded([&] {
    if (!rail || !chunks_done) fail(NZ_ERR_INVALID, "null argument");
    if (!rail->prog_valid) {
      *chunks_done = 0;
      return;
    }
    NZ_CUDA(cudaSetDevice(rail->comm->device));
    const cudaError_t q = cudaEventQuery(rail->done);
    if (q == cudaErrorNotReady) {
      *chunks_done = rail->prog_begin;
      return;
    }
    NZ_CUDA(q);
    *chunks_done = rail->prog_stop;
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

namespace {
int emulateFold(int world, int rank, int dtype, const void* const* src, void* const* dst, int ndst, uint64_t seg_off,
                uint64_t seg_len, uint64_t chunk_bytes, uint64_t lo, uint64_t hi, int grid, void* stream, bool tma) {
  return guarded([&] {
    if (tma && (ndst != world || world < 2)) fail(NZ_ERR_INVALID, "TMA emulation needs ndst == world >= 2");
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
    if (tma)
      nz::dispatchTma(world, dtype, a, grid, static_cast<cudaStream_t>(stream));
    else if (ndst == 1)
      nz::dispatchFold<0>(world, dtype, a, grid, static_cast<cudaStream_t>(stream));
    else
      nz::dispatchFold<1>(world, dtype, a, grid, static_cast<cudaStream_t>(stream));
    NZ_CUDA(cudaGetLastError());
  });
}
}  // namespace

int nz_emulate_fold(int world, int rank, int dtype, const void* const* src, void* const* dst, int ndst,
                    uint64_t seg_off, uint64_t seg_len, uint64_t chunk_bytes, uint64_t lo, uint64_t hi, int grid,
                    void* stream) {
  return emulateFold(world, rank, dtype, src, dst, ndst, seg_off, seg_len, chunk_bytes, lo, hi, grid, stream, false);
}

int nz_emulate_fold_tma(int world, int rank, int dtype, const void* const* src, void* const* dst, int ndst,
                        uint64_t seg_off, uint64_t seg_len, uint64_t chunk_bytes, uint64_t lo, uint64_t hi, int grid,
                        void* stream) {
  return emulateFold(world, rank, dtype, src, dst, ndst, seg_off, seg_len, chunk_bytes, lo, hi, grid, stream, true);
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
