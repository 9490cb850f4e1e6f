// TEST HARNESS ONLY (see simt.h): the fiber scheduler behind the host SIMT
// stand-in. One launch = one grid of fibers (one per CUDA thread) run
// round-robin on the calling thread. A fiber runs until it finishes, waits at
// __syncthreads, or polls a cross-rank word (yield_spin); a pass over the
// grid in which every fiber only polled backs off briefly, so a grid waiting
// on another stream's / process's grid does not burn the host.
#include "simt.h"

#include <sys/mman.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <map>
#include <thread>
#include <utility>
#include <vector>

// x86-64 context switch: save the callee-saved registers on the current
// stack, store its pointer in *save, continue on `next` (saved the same way).
extern "C" void nzsimt_switch(void** save, void* next);
asm(R"(
.text
.globl nzsimt_switch
.type nzsimt_switch,@function
nzsimt_switch:
  pushq %rbp
  pushq %rbx
  pushq %r12
  pushq %r13
  pushq %r14
  pushq %r15
  movq %rsp, (%rdi)
  movq %rsi, %rsp
  popq %r15
  popq %r14
  popq %r13
  popq %r12
  popq %rbx
  popq %rbp
  ret
.size nzsimt_switch, .-nzsimt_switch
.section .note.GNU-stack,"",@progbits
.text
)");

namespace nzsimt {

thread_local Cur* g_cur = nullptr;
std::atomic<uint64_t> g_grids{0}, g_threads{0};  // launches / CUDA threads run on fibers

namespace {

// Per fiber; the kernel frames are small. No guard pages: one VMA per fiber
// would exhaust vm.max_map_count with a few concurrent grids.
constexpr size_t kStack = 32 * 1024;

struct Cta {
  bool admitted = false;  // resident on the (modelled) device
  int live = 0;           // fibers not finished
  int expected = 0;     // fibers still running (exited ones leave the barrier)
  int arrived = 0;
  uint64_t gen = 0;
  int acc_or = 0, res_or = 0;
  std::map<const void*, std::vector<uint64_t>> shared;
};

struct Fiber {
  Cur cur;
  void* sp = nullptr;
  bool done = false;
  bool spun = false;  // last yield came from a poll
  Cta* cta = nullptr;
};

struct Grid {
  std::vector<Fiber> fibers;
  std::vector<Cta> ctas;
  void* sched_sp = nullptr;
  Fiber* running = nullptr;
  uint64_t events = 0;  // barrier arrivals and exits: progress of the grid
  const std::function<void()>* body = nullptr;
  char* stacks = nullptr;
  size_t stacks_len = 0;
};

thread_local Grid* g_grid = nullptr;

void switch_to_scheduler() {
  Grid* g = g_grid;
  nzsimt_switch(&g->running->sp, g->sched_sp);
}

[[noreturn]] void fiber_entry() {
  Grid* g = g_grid;
  (*g->body)();
  Fiber* f = g->running;
  f->done = true;
  f->cta->expected--;  // an exited thread no longer holds the CTA's barrier
  nzsimt_switch(&f->sp, g->sched_sp);
  __builtin_trap();
}

}  // namespace

// FAKECUDA_SIMT_PREEMPT=<per mille>: schedule fuzzing. Every data load /
// store of a kernel (ld_v4 / st_v4) yields with that probability and each
// pass visits the fibers in a fresh random order, so CTAs of different ranks
// interleave at points round-robin never produces. Seed: FAKECUDA_SIMT_SEED.
static uint32_t preempt_pm() {
  static const uint32_t v = [] {
    const char* e = getenv("FAKECUDA_SIMT_PREEMPT");
    return e ? static_cast<uint32_t>(atoi(e)) : 0u;
  }();
  return v;
}

static uint64_t& rng_state() {
  static thread_local uint64_t s = [] {
    const char* e = getenv("FAKECUDA_SIMT_SEED");
    uint64_t v = e ? strtoull(e, nullptr, 10) : 1;
    return v * 0x9E3779B97F4A7C15ull + reinterpret_cast<uintptr_t>(&s);
  }();
  return s;
}

static uint32_t rnd() {
  uint64_t& x = rng_state();
  x ^= x << 13;
  x ^= x >> 7;
  x ^= x << 17;
  return static_cast<uint32_t>(x >> 32);
}

void maybe_preempt() {
  const uint32_t pm = preempt_pm();
  if (pm == 0) return;
  Grid* g = g_grid;
  if (!g || !g->running) return;
  if (rnd() % 1000 < pm) switch_to_scheduler();
}

void yield_spin() {
  Grid* g = g_grid;
  if (!g || !g->running) return;
  g->running->spun = true;
  switch_to_scheduler();
}

static int barrier(int v, bool want_or) {
  Grid* g = g_grid;
  Fiber* f = g->running;
  Cta* c = f->cta;
  if (want_or) c->acc_or |= v;
  const uint64_t gen = c->gen;
  g->events++;
  if (++c->arrived >= c->expected) {
    c->res_or = c->acc_or;
    c->acc_or = 0;
    c->arrived = 0;
    c->gen++;
  } else {
    while (c->gen == gen) {
      f->spun = true;
      switch_to_scheduler();
      if (c->gen == gen && c->arrived >= c->expected) {  // a peer exited meanwhile
        c->res_or = c->acc_or;
        c->acc_or = 0;
        c->arrived = 0;
        c->gen++;
      }
    }
  }
  return c->res_or;
}

void sync_cta() { barrier(0, false); }
int sync_cta_or(int v) { return barrier(v, true) != 0; }

void* shared_slot(const void* key, size_t bytes) {
  Cta* c = g_grid->running->cta;
  auto& v = c->shared[key];
  if (v.empty()) v.assign((bytes + 7) / 8, 0);
  return v.data();
}

// Residency model (FAKECUDA_SIMT_RESIDENT_SMS, default 16 — the SM count
// the harness reports; 0 = unlimited): a CTA runs only once it is resident,
// CTAs become resident in launch (linear block) order as earlier CTAs of any
// grid in the process retire, and a CTA of a kernel with occupancy k costs
// 1/k of an SM (fakecuda::occupancyOf, the same figures the harness's
// cudaOccupancy* returns). A cross-rank wait between CTAs that cannot be
// co-resident then behaves as on the device: it waits for a CTA that never
// starts, until its watchdog.
constexpr int64_t kUnitsPerSM = 64;
static int64_t residentCapacity() {
  static const int64_t v = [] {
    const char* e = getenv("FAKECUDA_SIMT_RESIDENT_SMS");
    return (e ? static_cast<int64_t>(atoll(e)) : int64_t{16}) * kUnitsPerSM;
  }();
  return v;
}
static std::atomic<int64_t> g_resident{0};  // SM units held by resident CTAs, process-wide

static bool acquireResidency(int64_t threads) {
  const int64_t cap = residentCapacity();
  if (cap <= 0) return true;
  int64_t cur = g_resident.load();
  while (cur + threads <= cap) {
    if (g_resident.compare_exchange_weak(cur, cur + threads)) return true;
  }
  return false;
}

static void releaseResidency(int64_t threads) {
  if (residentCapacity() > 0) g_resident.fetch_sub(threads);
}

// Runs `body` once per thread of the grid, to completion.
void run_grid(dim3 grid, dim3 block, const std::function<void()>& body, int occupancy) {
  Grid g;
  const size_t nctas = static_cast<size_t>(grid.x) * grid.y * grid.z;
  const size_t nthr = static_cast<size_t>(block.x) * block.y * block.z;
  const size_t n = nctas * nthr;
  g.ctas.resize(nctas);
  g.fibers.resize(n);
  g.body = &body;
  const size_t per = kStack;
  g.stacks_len = per * n;
  void* m = mmap(nullptr, g.stacks_len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0);
  if (m == MAP_FAILED) {
    fprintf(stderr, "simt: cannot map %zu fiber stacks\n", n);
    abort();
  }
  g.stacks = static_cast<char*>(m);
  size_t i = 0;
  for (unsigned bz = 0; bz < grid.z; ++bz)
    for (unsigned by = 0; by < grid.y; ++by)
      for (unsigned bx = 0; bx < grid.x; ++bx) {
        Cta* cta = &g.ctas[(static_cast<size_t>(bz) * grid.y + by) * grid.x + bx];
        cta->expected = static_cast<int>(nthr);
        cta->live = static_cast<int>(nthr);
        for (unsigned tz = 0; tz < block.z; ++tz)
          for (unsigned ty = 0; ty < block.y; ++ty)
            for (unsigned tx = 0; tx < block.x; ++tx, ++i) {
              Fiber& f = g.fibers[i];
              f.cur.tid = uint3{tx, ty, tz};
              f.cur.bid = uint3{bx, by, bz};
              f.cur.bdim = block;
              f.cur.gdim = grid;
              f.cta = cta;
              char* base = g.stacks + i * per;
              uintptr_t top = reinterpret_cast<uintptr_t>(base + per) & ~uintptr_t{15};
              void** sp = reinterpret_cast<void**>(top);
              *--sp = nullptr;                                        // fake return address of fiber_entry
              *--sp = reinterpret_cast<void*>(&fiber_entry);          // where the first switch returns to
              for (int r = 0; r < 6; ++r) *--sp = nullptr;            // rbp rbx r12 r13 r14 r15
              f.sp = sp;
            }
      }
  Grid* prev_grid = g_grid;
  Cur* prev_cur = g_cur;
  g_grid = &g;
  size_t live = n;
  int idle_passes = 0;
  std::vector<uint32_t> order(n);
  for (size_t k = 0; k < n; ++k) order[k] = static_cast<uint32_t>(k);
  const int64_t cost = kUnitsPerSM / std::max(1, std::min<int>(occupancy, kUnitsPerSM));
  if (residentCapacity() > 0 && cost > residentCapacity()) {
    fprintf(stderr, "simt: a CTA exceeds the modelled device\n");
    abort();
  }
  size_t next_cta = 0;
  while (live > 0) {
    while (next_cta < nctas && acquireResidency(cost)) {
      g.ctas[next_cta++].admitted = true;
      g.events++;
    }
    const uint64_t ev0 = g.events;
    if (preempt_pm()) {
      for (size_t k = n; k > 1; --k) std::swap(order[k - 1], order[rnd() % k]);
    }
    for (uint32_t idx : order) {
      Fiber& f = g.fibers[idx];
      if (f.done || !f.cta->admitted) continue;
      f.spun = false;
      g.running = &f;
      g_cur = &f.cur;
      nzsimt_switch(&g.sched_sp, f.sp);
      if (f.done) {
        --live;
        g.events++;
        if (--f.cta->live == 0) releaseResidency(cost);  // the CTA retired
      }
    }
    if (g.events != ev0) {
      idle_passes = 0;
    } else if (++idle_passes > 4) {
      std::this_thread::sleep_for(std::chrono::microseconds(50));
    } else {
      std::this_thread::yield();
    }
  }
  g.running = nullptr;
  g_grid = prev_grid;
  g_cur = prev_cur;
  munmap(g.stacks, g.stacks_len);
  g_grids.fetch_add(1);
  g_threads.fetch_add(n);
}

}  // namespace nzsimt

extern "C" uint64_t fakecuda_simt_grids() { return nzsimt::g_grids.load(); }
extern "C" uint64_t fakecuda_simt_threads() { return nzsimt::g_threads.load(); }
