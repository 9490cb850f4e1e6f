// TEST HARNESS ONLY (see fakecuda.cpp): launch dispatch of the harness. By
// default a launch runs the kernel source itself on fibers (simtKernel,
// simt_kernels.cpp). With FAKECUDA_SIMT=0 it runs the host restatements
// below: emulations of the rail kernels' protocols, following
// csrc/cuda/kernels.cuh step by step — launch status
// (rail_enter / rail_exit), per-CTA barriers with epochs and budgets, the
// injected stall, the ring-order fold, the LL flag protocol, fault posts.
// A launch's grid is emulated as ONE CTA per rank (barrier slot 0): the
// host-visible protocol is the same, the work split is not modelled. The
// loopback *_vr grids run one host thread per virtual rank.
#include <cuda_runtime_api.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <ctime>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "fakecuda.h"
#include "kernel_args.h"

using namespace nz;

namespace {

uint64_t gtimer() {  // %globaltimer: the host's CLOCK_REALTIME in the harness
  timespec ts;
  clock_gettime(CLOCK_REALTIME, &ts);
  return static_cast<uint64_t>(ts.tv_sec) * 1000000000ull + static_cast<uint64_t>(ts.tv_nsec);
}

template <typename T>
T ld(const T* p) {
  return __atomic_load_n(p, __ATOMIC_ACQUIRE);
}
template <typename T>
void st(T* p, T v) {
  __atomic_store_n(p, v, __ATOMIC_RELEASE);
}

void backoff(int& i) {
  if (++i < 64)
    std::this_thread::yield();
  else
    std::this_thread::sleep_for(std::chrono::microseconds(20));
}

// ------------------------------------------------------------ launch status --
bool rail_enter(const RailCtl& c) {
  if (!c.dev) return true;
  const uint32_t sticky = ld(c.dev + kCtlSticky);
  const uint32_t seq = ld(c.dev + kCtlSeq);
  const bool dead = sticky != 0 && static_cast<int32_t>(sticky - 1u - seq) < 0;
  if (c.host) {
    st(&c.host->t_start_ns, gtimer());
    st(&c.host->start_tag, c.tag);
  }
  return !dead;
}

void note_detect(const RailCtl* c, uint64_t now) {
  if (c && c->host) {
    st(&c->host->t_det_ns, now);
    st(&c->host->det_tag, c->tag);
  }
}

void note_stall(const RailCtl& c) {
  if (c.host) {
    st(&c.host->t_fail_ns, gtimer());
    st(&c.host->fail_tag, c.tag);
  }
}

void note_run(const RailCtl& c) {
  if (c.host) {
    st(&c.host->t_run_ns, gtimer());
    st(&c.host->run_tag, c.tag);
  }
}

void rail_exit(const RailCtl& c, bool ok) {
  if (!c.dev) return;
  if (!ok) {
    st(c.dev + kCtlFailed, 1u);
    st(c.dev + kCtlSticky, ld(c.dev + kCtlSeq) + 1u);
  }
  // One emulated CTA: it is always the last to retire.
  st(c.dev + kCtlRetired, 0u);
  const bool failed = __atomic_exchange_n(c.dev + kCtlFailed, 0u, __ATOMIC_ACQ_REL) != 0;
  if (!failed) {
    nz_rail_status_t* h = c.host;
    if (h && c.prog_chunk != ~0ull) {
      st(&h->prog_chunk, c.prog_chunk);
      st(&h->prog_tag, c.tag);
    }
    if (c.final_wave) {
      st(c.dev + kCtlGate, c.tag);
      if (h) st(&h->ok_tag, c.tag);
    }
  }
  __atomic_fetch_add(c.dev + kCtlSeq, 1u, __ATOMIC_ACQ_REL);
}

uint32_t op_epoch(const BarrierArgs& b) { return b.seq ? 2u * ld(b.seq) + 1u : b.epoch; }

bool cta_barrier(int N, const BarrierArgs& b, uint32_t epoch, int rank, uint64_t timeout_ns, const RailCtl* ctl) {
  for (int t = 0; t < N; ++t) st(b.peer[t] + rank, epoch);  // slot [cta 0][rank] of every rank's pad
  for (int t = 0; t < N; ++t) {
    const uint32_t* slot = b.local + t;
    uint64_t t0 = 0;
    int i = 0;
    while (static_cast<int32_t>(ld(slot) - epoch) < 0) {
      const uint64_t now = gtimer();
      if (t0 == 0) {
        t0 = now;
      } else if (now - t0 > timeout_ns || (b.abort && ld(const_cast<const uint32_t*>(b.abort)))) {
        if (b.watchdog) st(b.watchdog, 1);
        note_detect(ctl, now);
        return false;
      }
      backoff(i);
    }
  }
  return true;
}

void post_fault(const FaultPost& p) {
  if (!p.rec) return;
  st(&p.rec->op_seq, p.op_seq);
  st(&p.rec->chunk, p.chunk);
  st(&p.rec->t_fail_ns, gtimer());
  st(&p.rec->valid, 1u);
}

// End-barrier budgets are sized for the device's speed (the op's own time
// x 4 plus a floor): the host emulation of a wave is orders of magnitude
// slower, so they are stretched here (FAKECUDA_END_DILATION, default 500).
// Start-of-op budgets (the watchdog) are left alone.
uint64_t dilation() {
  static const uint64_t d = [] {
    const char* e = getenv("FAKECUDA_END_DILATION");
    const long long v = e ? atoll(e) : 500;
    return static_cast<uint64_t>(v > 0 ? v : 1);
  }();
  return d;
}

uint64_t end_budget(const BarrierArgs& b, const RailCtl& c) {
  return c.end_timeout_ns ? c.end_timeout_ns * dilation() : b.timeout_ns;
}

// ------------------------------------------------------------- arithmetic --
enum class DT { F32, BF16, I32 };

int esOf(DT d) { return d == DT::BF16 ? 2 : 4; }

float bf2f(uint16_t h) {
  const uint32_t u = static_cast<uint32_t>(h) << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}
uint16_t f2bf(float f) {  // round to nearest even (__float2bfloat16_rn)
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return static_cast<uint16_t>((u >> 16) | 0x40u);
  u += 0x7fffu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

// Ring block (fold start rank) of the element at byte offset x (block_at).
int blockAt(int N, int ES, const Geometry& g, uint64_t x) {
  const uint64_t rel = x - g.seg_off;
  const uint64_t c = rel / g.chunk;
  const uint64_t cbeg = c * g.chunk;
  const uint64_t rem = g.seg_len - cbeg;
  const uint64_t clen = rem < g.chunk ? rem : g.chunk;
  const uint64_t q = (clen / ES) / N;
  if (q == 0) return N - 1;
  const uint64_t bb = ((rel - cbeg) / ES) / q;
  return bb >= static_cast<uint64_t>(N) ? N - 1 : static_cast<int>(bb);
}

// One element folded in ring order from the N values (v[r] = rank r's bits).
void foldElem(DT d, int N, int b, const uint32_t* v, char* out) {
  if (d == DT::F32) {
    float acc, t;
    memcpy(&acc, &v[b], 4);
    for (int j = 1; j < N; ++j) {
      memcpy(&t, &v[(b + j) % N], 4);
      acc = acc + t;
    }
    memcpy(out, &acc, 4);
  } else if (d == DT::I32) {
    uint32_t acc = v[b];
    for (int j = 1; j < N; ++j) acc += v[(b + j) % N];
    memcpy(out, &acc, 4);
  } else {
    float acc = bf2f(static_cast<uint16_t>(v[b]));
    for (int j = 1; j < N; ++j) acc = acc + bf2f(static_cast<uint16_t>(v[(b + j) % N]));
    const uint16_t h = f2bf(acc);
    memcpy(out, &h, 2);
  }
}

uint32_t loadElem(DT d, const char* p) {
  if (d == DT::BF16) {
    uint16_t h;
    memcpy(&h, p, 2);
    return h;
  }
  uint32_t w;
  memcpy(&w, p, 4);
  return w;
}

// ---------------------------------------------------------------- bodies --
void fold_body(DT d, int N, int ndst, const FoldArgs& a) {
  if (!rail_enter(a.ctl)) return rail_exit(a.ctl, false);
  const uint32_t ep = op_epoch(a.bar);
  if (a.use_barrier && !cta_barrier(N, a.bar, ep, a.rank, a.bar.timeout_ns, &a.ctl)) return rail_exit(a.ctl, false);
  if (a.use_barrier) note_run(a.ctl);
  if (a.ctl.stall) {
    note_stall(a.ctl);
    return rail_exit(a.ctl, false);
  }
  const int ES = esOf(d);
  uint32_t v[kDevMaxRanks];
  char out[4];
  for (uint64_t x = a.s; x < a.e; x += ES) {
    for (int r = 0; r < N; ++r) v[r] = loadElem(d, a.src[r] + x);
    foldElem(d, N, blockAt(N, ES, a.g, x), v, out);
    for (int k = 0; k < ndst; ++k) memcpy(a.dst[k] + x, out, ES);
  }
  if (a.use_barrier && !cta_barrier(N, a.bar, ep + 1, a.rank, end_budget(a.bar, a.ctl), &a.ctl))
    return rail_exit(a.ctl, false);
  post_fault(a.post);
  rail_exit(a.ctl, true);
}

uint32_t llLoadWord(const char* base, uint64_t x, uint64_t hi) {
  if (x + 4 <= hi) {
    uint32_t w;
    memcpy(&w, base + x, 4);
    return w;
  }
  uint16_t h;
  memcpy(&h, base + x, 2);
  return h;  // bf16 tail
}

void ll_body(DT d, int N, const LLArgs& a) {
  if (!rail_enter(a.ctl)) return rail_exit(a.ctl, false);
  if (a.ctl.stall) {
    note_stall(a.ctl);
    return rail_exit(a.ctl, false);
  }
  uint32_t flag = a.flag;
  int parity = a.parity;
  if (a.seq) {
    flag = ld(a.seq) + 1u;
    if (flag == 0) flag = 1;
    parity = static_cast<int>(flag & 1u);
  }
  const uint64_t my_slot = (static_cast<uint64_t>(parity) * N + a.rank) * a.slot_words;
  const uint64_t pairs = (a.words + 1) / 2;
  const uint64_t F = static_cast<uint64_t>(flag) << 32;
  for (uint64_t p = 0; p < pairs; ++p) {
    const uint64_t x = a.lo + 8 * p;
    const uint32_t d0 = llLoadWord(a.in, x, a.hi);
    const uint32_t d1 = x + 4 < a.hi ? llLoadWord(a.in, x + 4, a.hi) : 0u;
    for (int r = 0; r < N; ++r) {
      uint64_t* dst = a.peer[r] + my_slot + 2 * p;
      st(dst, F | d0);
      st(dst + 1, F | d1);
    }
  }
  bool bail = false;
  const int ES = esOf(d);
  for (uint64_t w = 0; w < a.words && !bail; ++w) {
    uint32_t v[kDevMaxRanks];
    for (int r = 0; r < N && !bail; ++r) {
      const uint64_t* src = a.local + (static_cast<uint64_t>(parity) * N + r) * a.slot_words + w;
      uint64_t t0 = 0;
      int i = 0;
      for (;;) {
        const uint64_t word = ld(src);
        if (static_cast<uint32_t>(word >> 32) == flag) {
          v[r] = static_cast<uint32_t>(word);
          break;
        }
        const uint64_t now = gtimer();
        if (t0 == 0) {
          t0 = now;
        } else if (now - t0 > a.timeout_ns || (a.abort && ld(const_cast<const uint32_t*>(a.abort)))) {
          st(a.watchdog, 1);
          note_detect(&a.ctl, now);
          bail = true;
          break;
        }
        backoff(i);
      }
    }
    if (bail) break;
    const uint64_t x = a.lo + 4 * w;
    for (int k = 0; k < 4 / ES; ++k) {
      const uint64_t xe = x + static_cast<uint64_t>(k) * ES;
      if (xe >= a.hi) break;
      uint32_t e[kDevMaxRanks];
      for (int r = 0; r < N; ++r) e[r] = ES == 4 ? v[r] : (k == 0 ? (v[r] & 0xffffu) : (v[r] >> 16));
      char out[4];
      foldElem(d, N, blockAt(N, ES, a.g, xe), e, out);
      memcpy(a.out + xe, out, ES);
    }
  }
  if (!bail) post_fault(a.post);
  rail_exit(a.ctl, !bail);
}

void barrier_body(int N, const BarrierKArgs& k) {
  if (!rail_enter(k.ctl)) return rail_exit(k.ctl, false);
  const uint64_t budget = k.end ? end_budget(k.bar, k.ctl) : k.bar.timeout_ns;
  if (!cta_barrier(N, k.bar, op_epoch(k.bar), k.rank, budget, &k.ctl)) return rail_exit(k.ctl, false);
  if (!k.end) note_run(k.ctl);
  if (!k.end && k.ctl.stall) {
    note_stall(k.ctl);
    return rail_exit(k.ctl, false);
  }
  post_fault(k.post);
  rail_exit(k.ctl, true);
}

void copy_body(const char* src, char* dst, uint64_t lo, uint64_t hi, const FaultPost& post, const RailCtl& ctl) {
  if (!rail_enter(ctl)) return rail_exit(ctl, false);
  if (ctl.stall) {
    note_stall(ctl);
    return rail_exit(ctl, false);
  }
  if (hi > lo) memcpy(dst + lo, src + lo, hi - lo);
  post_fault(post);
  rail_exit(ctl, true);
}

// ------------------------------------------------------------ name parsing --
struct Parsed {
  std::string base;
  std::vector<std::string> targs;
};

Parsed parse(const std::string& name) {
  Parsed p;
  size_t at = name.find("nz::");
  if (at == std::string::npos) return p;
  at += 4;
  size_t end = name.find_first_of("<(", at);
  p.base = name.substr(at, end - at);
  if (end != std::string::npos && name[end] == '<') {
    int depth = 0;
    std::string cur;
    for (size_t i = end; i < name.size(); ++i) {
      const char c = name[i];
      if (c == '<') {
        if (depth++ > 0) cur += c;
      } else if (c == '>') {
        if (--depth == 0) {
          p.targs.push_back(cur);
          break;
        }
        cur += c;
      } else if (c == ',' && depth == 1) {
        p.targs.push_back(cur);
        cur.clear();
      } else if (!(c == ' ' && cur.empty())) {
        cur += c;
      }
    }
  }
  return p;
}

DT dtOf(const std::string& s) {
  if (s.find("BF16") != std::string::npos) return DT::BF16;
  if (s.find("I32") != std::string::npos) return DT::I32;
  return DT::F32;
}

template <typename A>
void runRanks(int N, const VPack<A>& p, const std::function<void(const A&)>& body) {
  std::vector<std::thread> ts;
  for (int y = 0; y < N; ++y) ts.emplace_back([&, y] { body(p.a[y]); });
  for (auto& t : ts) t.join();
}

std::mutex g_count_mu;
std::map<std::string, uint64_t> g_counts;

}  // namespace

namespace nzsimt {
uint64_t end_dilation() { return dilation(); }
}  // namespace nzsimt

namespace fakecuda {

#ifndef FAKECUDA_NO_SIMT
std::function<void()> simtKernel(const std::string& base, const std::vector<std::string>& targs, dim3 grid, dim3 block,
                                 void** args);
#else
// Sanitizer builds (tools/harness_sanitize.sh): no fibers, protocol restatements only.
std::function<void()> simtKernel(const std::string&, const std::vector<std::string>&, dim3, dim3, void**) { return {}; }
#endif

// FAKECUDA_SIMT=1 (the default): the kernels of csrc/cuda/kernels.cuh run
// themselves, on host fibers (simt.h). 0: the protocol restatements above
// (used by the sanitizer builds, which do not follow fiber stack switches).
bool simtMode() {
  static const bool on = [] {
    const char* e = getenv("FAKECUDA_SIMT");
    return !e || atoi(e) != 0;
  }();
  return on;
}

int occupancyOf(const std::string& name, int block_threads) {
  if (name.find("ll_kernel") != std::string::npos) return 1;
  if (block_threads >= 512) return 2;
  return std::max(1, std::min(32, 1024 / std::max(1, block_threads)));
}

void countLaunch(const std::string& name) {
  std::lock_guard<std::mutex> lk(g_count_mu);
  ++g_counts[parse(name).base];
}

std::function<void()> emulatedKernel(const std::string& name, dim3 grid, dim3 block, void** args) {
  const Parsed k = parse(name);
  if (simtMode()) {
    if (auto f = simtKernel(k.base, k.targs, grid, block, args)) return f;
  }
  if (k.base == "fold_kernel" && k.targs.size() == 3) {
    const DT d = dtOf(k.targs[0]);
    const int N = std::stoi(k.targs[1]), nd = std::stoi(k.targs[2]);
    const FoldArgs a = *static_cast<const FoldArgs*>(args[0]);
    return [=] { fold_body(d, N, nd == 1 ? 1 : N, a); };
  }
  if (k.base == "fold_kernel_vr" && k.targs.size() == 3) {
    const DT d = dtOf(k.targs[0]);
    const int N = std::stoi(k.targs[1]), nd = std::stoi(k.targs[2]);
    const auto p = std::make_shared<VPack<FoldArgs>>(*static_cast<const VPack<FoldArgs>*>(args[0]));
    return [=] { runRanks<FoldArgs>(N, *p, [&](const FoldArgs& a) { fold_body(d, N, nd == 1 ? 1 : N, a); }); };
  }
  if (k.base == "ll_kernel" && k.targs.size() == 2) {
    const DT d = dtOf(k.targs[0]);
    const int N = std::stoi(k.targs[1]);
    const LLArgs a = *static_cast<const LLArgs*>(args[0]);
    return [=] { ll_body(d, N, a); };
  }
  if (k.base == "ll_kernel_vr" && k.targs.size() == 2) {
    const DT d = dtOf(k.targs[0]);
    const int N = std::stoi(k.targs[1]);
    const auto p = std::make_shared<VPack<LLArgs>>(*static_cast<const VPack<LLArgs>*>(args[0]));
    return [=] { runRanks<LLArgs>(N, *p, [&](const LLArgs& a) { ll_body(d, N, a); }); };
  }
  if (k.base == "barrier_kernel" && k.targs.size() == 1) {
    const int N = std::stoi(k.targs[0]);
    const BarrierKArgs a = *static_cast<const BarrierKArgs*>(args[0]);
    return [=] { barrier_body(N, a); };
  }
  if (k.base == "barrier_kernel_vr" && k.targs.size() == 1) {
    const int N = std::stoi(k.targs[0]);
    const auto p = std::make_shared<VPack<BarrierKArgs>>(*static_cast<const VPack<BarrierKArgs>*>(args[0]));
    return [=] { runRanks<BarrierKArgs>(N, *p, [&](const BarrierKArgs& a) { barrier_body(N, a); }); };
  }
  if (k.base == "copy_kernel") {
    const char* src = *static_cast<const char* const*>(args[0]);
    char* dst = *static_cast<char* const*>(args[1]);
    const uint64_t lo = *static_cast<const uint64_t*>(args[2]);
    const uint64_t hi = *static_cast<const uint64_t*>(args[3]);
    const FaultPost post = *static_cast<const FaultPost*>(args[4]);
    const RailCtl ctl = *static_cast<const RailCtl*>(args[5]);
    return [=] { copy_body(src, dst, lo, hi, post, ctl); };
  }
  if (k.base == "stamp_kernel") {
    uint64_t* dst = *static_cast<uint64_t* const*>(args[0]);
    return [=] { st(dst, gtimer()); };
  }
  return {};  // nvls_kernel: the harness has no multicast (the rail is never built)
}

}  // namespace fakecuda

extern "C" uint64_t fakecuda_launches(const char* base) {
  std::lock_guard<std::mutex> lk(g_count_mu);
  auto it = g_counts.find(base ? base : "");
  return it == g_counts.end() ? 0 : it->second;
}
