// TEST HARNESS ONLY — never part of the product, never loaded by it.
//
// A host stand-in for the CUDA runtime and driver that lets the product
// library's HOST code (loopback communicator, the rails' launch sequencing,
// waves and gates, the engine, its failure monitor and agreement, readmit)
// run in the CPU test suite, where there is no GPU. Streams are worker
// threads, device memory is host memory (VMM allocations are memfd mappings,
// so several virtual addresses can alias one allocation as they do on the
// device), and each kernel launch runs csrc/cuda/kernels.cuh ITSELF on host
// fibers (simt.h / simt.cpp / simt_kernels.cpp: one fiber per CUDA thread,
// per-CTA __syncthreads, yielding cross-rank polls). FAKECUDA_SIMT=0 selects
// the older host restatements of the kernels' protocols (emu_kernels.cpp),
// which the sanitizer builds use.
//
// What it checks: that the host code issues the right launches, on the
// right streams, with the right geometry, waits and gates, that its control
// flow (agreement, reroute, readmit, pipelining) terminates with the right
// results, and that the kernel source computes them bit-exactly. What it does
// not check: the compiled SASS, memory ordering across GPUs, NVLink /
// multicast, timing. Hardware parity claims rest on the GPU tests.
//
// Built into tests/fakecuda/build/libnezha_b200_hostharness.so together with
// the product's own object files (linked -Bsymbolic so nothing else in the
// process can interpose a real runtime). Loaded only when a test sets
// NEZHA_TEST_HOST_HARNESS_LIB.
#include <cuda.h>
#include <cuda_runtime_api.h>
#include <cxxabi.h>
#include <execinfo.h>
#include <signal.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "fakecuda.h"

// ----------------------------------------------------------------- streams --
struct CUstream_st {
  std::mutex m;
  std::condition_variable cv;
  std::deque<std::function<void()>> q;
  uint64_t enq = 0, done = 0;
  bool stop = false;
  std::thread th;

  CUstream_st() {
    th = std::thread([this] { loop(); });
  }
  void loop();  // below: a destroyed stream drains, then leaves the registry
  void loopBody() {
    for (;;) {
      std::function<void()> op;
      {
        std::unique_lock<std::mutex> lk(m);
        cv.wait(lk, [&] { return stop || !q.empty(); });
        if (q.empty()) return;
        op = std::move(q.front());
        q.pop_front();
      }
      op();
      {
        std::lock_guard<std::mutex> lk(m);
        ++done;
      }
      cv.notify_all();
    }
  }
  void push(std::function<void()> op) {
    {
      std::lock_guard<std::mutex> lk(m);
      q.push_back(std::move(op));
      ++enq;
    }
    cv.notify_all();
  }
  void sync() {
    std::unique_lock<std::mutex> lk(m);
    const uint64_t target = enq;
    cv.wait(lk, [&] { return done >= target; });
  }
  // cudaStreamDestroy returns at once; queued work still runs. Stream
  // objects are never freed (a test process makes a bounded number).
  void retire() {
    {
      std::lock_guard<std::mutex> lk(m);
      stop = true;
    }
    cv.notify_all();
    th.detach();
  }
};

// Each record is its own completion: a wait captures the record current at
// the call and waits for exactly that one (a later re-record of the event on
// another stream must not release it — the engine recycles events).
struct CUevent_st {
  std::mutex m;
  std::condition_variable cv;
  uint64_t rec = 0;             // last record issued
  uint64_t latest_done = 0;     // highest record completed
  std::set<uint64_t> inflight;  // records issued, not yet reached by their stream
  int64_t t_ns = 0;             // time of the highest completed record
  bool complete(uint64_t r) const { return r == 0 || inflight.count(r) == 0; }
};

namespace {

std::mutex g_streams_mu;
std::set<CUstream_st*>& streams() {
  static auto* s = new std::set<CUstream_st*>();
  return *s;
}

}  // namespace

void CUstream_st::loop() {
  loopBody();
  std::lock_guard<std::mutex> lk(g_streams_mu);
  streams().erase(this);
}

namespace {

CUstream_st* legacy() {
  static CUstream_st* s = [] {
    auto* st = new CUstream_st();
    std::lock_guard<std::mutex> lk(g_streams_mu);
    streams().insert(st);
    return st;
  }();
  return s;
}

CUstream_st* S(cudaStream_t s) {
  const uintptr_t v = reinterpret_cast<uintptr_t>(s);
  if (v == 0 || v == 1 || v == 2) return legacy();  // NULL, cudaStreamLegacy, cudaStreamPerThread
  return s;
}

int64_t nowNs() {
  timespec ts;
  clock_gettime(CLOCK_REALTIME, &ts);
  return static_cast<int64_t>(ts.tv_sec) * 1000000000LL + ts.tv_nsec;
}

thread_local cudaError_t t_last = cudaSuccess;

cudaError_t ret(cudaError_t e) {
  if (e != cudaSuccess) t_last = e;
  return e;
}

// Waits with a short spin, then sleeps: many host threads poll at once here.
template <typename F>
void pollUntil(F done) {
  for (int i = 0; !done(); ++i) {
    if (i < 64)
      std::this_thread::yield();
    else
      std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

// --------------------------------------------------------- kernel registry --
struct Registry {
  std::mutex m;
  std::map<const void*, std::string> names;  // host stub -> demangled device name
};
Registry& registry() {
  static auto* r = new Registry();
  return *r;
}

struct LaunchConfig {
  dim3 grid, block;
  size_t smem = 0;
  cudaStream_t stream = nullptr;
};
thread_local std::vector<LaunchConfig> t_config;

// ------------------------------------------------------------ VMM on memfd --
struct Alloc {
  int fd = -1;
  size_t size = 0;
  struct McTable* mc = nullptr;  // a multicast object (FAKECUDA_MULTICAST=1)
};

// ---------------------------------------------------- NVSwitch multicast --
// FAKECUDA_MULTICAST=1: a multicast object is a small shared table (memfd,
// travels between rank processes like any VMM handle) in which every bound
// rank records its process id and a descriptor of its memory. Mapping the
// object reserves an INACCESSIBLE window: plain loads / stores there fault,
// and the kernels' multimem accesses (simt.h) resolve an address of the
// window to every member's memory at the same offset (/proc/<pid>/fd/<fd>),
// reduce or store across them, and trap on a misaligned 16-byte access —
// the round-1 NVLink incident's class of bug.
constexpr uint64_t kMcMagic = 0x4e5a4d4354424c31ull;  // "NZMCTBL1"
struct McTable {
  uint64_t magic;
  uint32_t ndev;
  uint32_t nbound;
  struct {
    int32_t pid, fd;
    uint64_t size;
  } member[8];
};

struct McWindow {
  char* va;
  size_t size;
  McTable* table;
  std::vector<char*> bases;  // members' memory mapped here, once all are bound
};
std::mutex g_mc_mu;
std::map<char*, McWindow> g_mc_windows;

bool multicastOn() {
  static const bool on = [] {
    const char* e = getenv("FAKECUDA_MULTICAST");
    return e && atoi(e) != 0;
  }();
  return on;
}

constexpr size_t kGranularity = 2u << 20;

std::mutex g_alloc_mu;
std::map<char*, std::pair<char*, size_t>> g_allocs;  // user pointer -> (mapping, span)

}  // namespace

extern "C" {

// ------------------------------------------------------ nvcc registration --
void** __cudaRegisterFatBinary(void*) {
  static void* handle = nullptr;
  return &handle;
}
void __cudaRegisterFatBinaryEnd(void**) {}
void __cudaUnregisterFatBinary(void**) {}
void __cudaRegisterFunction(void**, const char* hostFun, char*, const char* deviceName, int, uint3*, uint3*, dim3*,
                            dim3*, int*) {
  int st = 0;
  char* dem = abi::__cxa_demangle(deviceName, nullptr, nullptr, &st);
  Registry& r = registry();
  std::lock_guard<std::mutex> lk(r.m);
  r.names[hostFun] = st == 0 && dem ? dem : deviceName;
  free(dem);
}
unsigned __cudaPushCallConfiguration(dim3 gridDim, dim3 blockDim, size_t sharedMem, struct CUstream_st* stream) {
  t_config.push_back(LaunchConfig{gridDim, blockDim, sharedMem, stream});
  return 0;
}
cudaError_t __cudaPopCallConfiguration(dim3* gridDim, dim3* blockDim, size_t* sharedMem, void* stream) {
  if (t_config.empty()) return cudaErrorInvalidConfiguration;
  const LaunchConfig c = t_config.back();
  t_config.pop_back();
  *gridDim = c.grid;
  *blockDim = c.block;
  *sharedMem = c.smem;
  *static_cast<cudaStream_t*>(stream) = c.stream;
  return cudaSuccess;
}

cudaError_t cudaLaunchKernel(const void* func, dim3 grid, dim3 block, void** args, size_t, cudaStream_t stream) {
  std::string name;
  {
    Registry& r = registry();
    std::lock_guard<std::mutex> lk(r.m);
    auto it = r.names.find(func);
    if (it == r.names.end()) return ret(cudaErrorInvalidDeviceFunction);
    name = it->second;
  }
  std::function<void()> body = fakecuda::emulatedKernel(name, grid, block, args);
  if (!body) {
    fprintf(stderr, "[fakecuda] no host emulation for kernel %s\n", name.c_str());
    return ret(cudaErrorInvalidDeviceFunction);
  }
  fakecuda::countLaunch(name);
  S(stream)->push(std::move(body));
  return cudaSuccess;
}

// ------------------------------------------------------------------ device --
cudaError_t cudaSetDevice(int) { return cudaSuccess; }
cudaError_t cudaGetDevice(int* d) {
  *d = 0;
  return cudaSuccess;
}
cudaError_t cudaDeviceGetAttribute(int* v, cudaDeviceAttr attr, int) {
  *v = attr == cudaDevAttrMultiProcessorCount ? fakecuda::kSMs : 0;
  return cudaSuccess;
}
cudaError_t cudaDeviceSynchronize(void) {
  std::vector<CUstream_st*> all;
  {
    std::lock_guard<std::mutex> lk(g_streams_mu);
    all.assign(streams().begin(), streams().end());
  }
  for (auto* s : all) s->sync();
  return cudaSuccess;
}
cudaError_t cudaGetLastError(void) {
  const cudaError_t e = t_last;
  t_last = cudaSuccess;
  return e;
}
const char* cudaGetErrorString(cudaError_t e) {
  static thread_local char buf[64];
  snprintf(buf, sizeof(buf), "fake cuda error %d", static_cast<int>(e));
  return buf;
}
cudaError_t cudaMemGetInfo(size_t* fr, size_t* tot) {
  *fr = size_t(64) << 30;
  *tot = size_t(180) << 30;
  return cudaSuccess;
}
cudaError_t cudaOccupancyMaxActiveBlocksPerMultiprocessorWithFlags(int* n, const void* func, int block, size_t,
                                                                   unsigned int) {
  std::string name;
  {
    Registry& r = registry();
    std::lock_guard<std::mutex> lk(r.m);
    auto it = r.names.find(func);
    if (it != r.names.end()) name = it->second;
  }
  *n = fakecuda::occupancyOf(name, block);
  return cudaSuccess;
}

// ------------------------------------------------------------------ memory --
// Device allocations end at an inaccessible guard page, so a launch or copy
// that runs past a buffer faults at the offending access.
cudaError_t cudaMalloc(void** p, size_t bytes) {
  const size_t page = 4096, body = (std::max<size_t>(bytes, 1) + 255) & ~size_t(255);
  const size_t span = (body + page - 1) / page * page + page;
  char* base = static_cast<char*>(mmap(nullptr, span, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0));
  if (base == MAP_FAILED) return ret(cudaErrorMemoryAllocation);
  mprotect(base + span - page, page, PROT_NONE);
  char* user = base + span - page - body;
  {
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    g_allocs[user] = {base, span};
  }
  *p = user;
  return cudaSuccess;
}
cudaError_t cudaFree(void* p) {
  if (!p) return cudaSuccess;
  std::pair<char*, size_t> a{};
  {
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    auto it = g_allocs.find(static_cast<char*>(p));
    if (it == g_allocs.end()) return ret(cudaErrorInvalidValue);
    a = it->second;
    g_allocs.erase(it);
  }
  munmap(a.first, a.second);
  return cudaSuccess;
}
cudaError_t cudaHostAlloc(void** p, size_t bytes, unsigned int) { return cudaMalloc(p, bytes); }
cudaError_t cudaFreeHost(void* p) { return cudaFree(p); }
cudaError_t cudaHostGetDevicePointer(void** d, void* h, unsigned int) {
  *d = h;
  return cudaSuccess;
}
cudaError_t cudaMemcpy(void* dst, const void* src, size_t n, cudaMemcpyKind) {
  legacy()->sync();
  memcpy(dst, src, n);
  return cudaSuccess;
}
cudaError_t cudaMemcpyAsync(void* dst, const void* src, size_t n, cudaMemcpyKind, cudaStream_t s) {
  S(s)->push([=] { memcpy(dst, src, n); });
  return cudaSuccess;
}
cudaError_t cudaMemset(void* dst, int v, size_t n) {
  legacy()->sync();
  memset(dst, v, n);
  return cudaSuccess;
}
cudaError_t cudaMemsetAsync(void* dst, int v, size_t n, cudaStream_t s) {
  S(s)->push([=] { memset(dst, v, n); });
  return cudaSuccess;
}

// ----------------------------------------------------------------- streams --
cudaError_t cudaStreamCreateWithFlags(cudaStream_t* s, unsigned int) {
  auto* st = new CUstream_st();
  {
    std::lock_guard<std::mutex> lk(g_streams_mu);
    streams().insert(st);
  }
  *s = st;
  return cudaSuccess;
}
cudaError_t cudaStreamDestroy(cudaStream_t s) {
  if (s) s->retire();
  return cudaSuccess;
}
cudaError_t cudaStreamSynchronize(cudaStream_t s) {
  S(s)->sync();
  return cudaSuccess;
}
cudaError_t cudaStreamIsCapturing(cudaStream_t, cudaStreamCaptureStatus* st) {
  *st = cudaStreamCaptureStatusNone;
  return cudaSuccess;
}
cudaError_t cudaStreamWaitEvent(cudaStream_t s, cudaEvent_t e, unsigned int) {
  uint64_t target;
  {
    std::lock_guard<std::mutex> lk(e->m);
    target = e->rec;
  }
  if (target == 0) return cudaSuccess;  // never recorded: nothing to wait for
  S(s)->push([e, target] {
    std::unique_lock<std::mutex> lk(e->m);
    e->cv.wait(lk, [&] { return e->complete(target); });
  });
  return cudaSuccess;
}

// ------------------------------------------------------------------ events --
cudaError_t cudaEventCreate(cudaEvent_t* e) {
  *e = new CUevent_st();
  return cudaSuccess;
}
cudaError_t cudaEventCreateWithFlags(cudaEvent_t* e, unsigned int) { return cudaEventCreate(e); }
cudaError_t cudaEventDestroy(cudaEvent_t) {
  return cudaSuccess;  // queued work may still complete it: events are never freed here
}
cudaError_t cudaEventRecord(cudaEvent_t e, cudaStream_t s) {
  uint64_t r;
  {
    std::lock_guard<std::mutex> lk(e->m);
    r = ++e->rec;
    e->inflight.insert(r);
  }
  S(s)->push([e, r] {
    {
      std::lock_guard<std::mutex> lk(e->m);
      e->inflight.erase(r);
      if (r > e->latest_done) {
        e->latest_done = r;
        e->t_ns = nowNs();
      }
    }
    e->cv.notify_all();
  });
  return cudaSuccess;
}
cudaError_t cudaEventQuery(cudaEvent_t e) {
  std::lock_guard<std::mutex> lk(e->m);
  return e->complete(e->rec) ? cudaSuccess : cudaErrorNotReady;
}
cudaError_t cudaEventSynchronize(cudaEvent_t e) {
  std::unique_lock<std::mutex> lk(e->m);
  const uint64_t target = e->rec;
  e->cv.wait(lk, [&] { return e->complete(target); });
  return cudaSuccess;
}
cudaError_t cudaEventElapsedTime(float* ms, cudaEvent_t a, cudaEvent_t b) {
  std::lock_guard<std::mutex> la(a->m);
  std::lock_guard<std::mutex> lb(b->m);
  *ms = static_cast<float>(static_cast<double>(b->t_ns - a->t_ns) / 1e6);
  return cudaSuccess;
}

}  // extern "C"

// A crash inside the library under test prints its native stack (there is
// no debugger in the test image). Python's faulthandler, when enabled later,
// takes the signal over.
namespace {
void onCrash(int sig) {
  void* frames[64];
  const int n = backtrace(frames, 64);
  fprintf(stderr, "[fakecuda] signal %d, native stack:\n", sig);
  backtrace_symbols_fd(frames, n, 2);
  signal(sig, SIG_DFL);
  raise(sig);
}
__attribute__((constructor)) void installCrashHandler() {
  signal(SIGSEGV, onCrash);
  signal(SIGBUS, onCrash);
  signal(SIGABRT, onCrash);
}
}  // namespace

// ------------------------------------------------------------------ driver --
namespace {

CUresult fInit(unsigned int) { return CUDA_SUCCESS; }
CUresult fDeviceGet(CUdevice* d, int ordinal) {
  *d = ordinal;
  return CUDA_SUCCESS;
}
CUresult fDeviceGetAttribute(int* v, CUdevice_attribute a, CUdevice) {
  *v = a == CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT ? fakecuda::kSMs
       : a == CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED ? (multicastOn() ? 1 : 0)
                                                       : 0;
  return CUDA_SUCCESS;
}
CUresult fGetErrorString(CUresult e, const char** s) {
  static thread_local char buf[64];
  snprintf(buf, sizeof(buf), "fake CUresult %d", static_cast<int>(e));
  *s = buf;
  return CUDA_SUCCESS;
}
CUresult fGranularity(size_t* g, const CUmemAllocationProp*, CUmemAllocationGranularity_flags) {
  *g = kGranularity;
  return CUDA_SUCCESS;
}
CUresult fMcGranularity(size_t* g, const CUmulticastObjectProp*, CUmulticastGranularity_flags) {
  if (!multicastOn()) return CUDA_ERROR_NOT_SUPPORTED;
  *g = kGranularity;
  return CUDA_SUCCESS;
}

McTable* mapTable(int fd) {
  void* p = mmap(nullptr, sizeof(McTable), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  return p == MAP_FAILED ? nullptr : static_cast<McTable*>(p);
}
CUresult fMemCreate(CUmemGenericAllocationHandle* h, size_t size, const CUmemAllocationProp*, unsigned long long) {
  const int fd = memfd_create("fakecuda", MFD_CLOEXEC);
  if (fd < 0 || ftruncate(fd, static_cast<off_t>(size)) != 0) return CUDA_ERROR_OUT_OF_MEMORY;
  *h = reinterpret_cast<CUmemGenericAllocationHandle>(new Alloc{fd, size});
  return CUDA_SUCCESS;
}
// Every reserved range is followed by an inaccessible guard (never mapped),
// so an access past a symmetric buffer faults where it happens.
constexpr size_t kGuard = 1u << 20;
CUresult fAddressReserve(CUdeviceptr* va, size_t size, size_t, CUdeviceptr, unsigned long long) {
  void* p = mmap(nullptr, size + kGuard, PROT_NONE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0);
  if (p == MAP_FAILED) return CUDA_ERROR_OUT_OF_MEMORY;
  *va = reinterpret_cast<CUdeviceptr>(p);
  return CUDA_SUCCESS;
}
CUresult fMemMap(CUdeviceptr va, size_t size, size_t offset, CUmemGenericAllocationHandle h, unsigned long long) {
  auto* a = reinterpret_cast<Alloc*>(h);
  if (a->mc) {  // the window stays PROT_NONE: only multimem accesses may touch it
    std::lock_guard<std::mutex> lk(g_mc_mu);
    g_mc_windows[reinterpret_cast<char*>(va)] = McWindow{reinterpret_cast<char*>(va), size, a->mc, {}};
    return offset == 0 ? CUDA_SUCCESS : CUDA_ERROR_INVALID_VALUE;
  }
  void* p = mmap(reinterpret_cast<void*>(va), size, PROT_READ | PROT_WRITE, MAP_SHARED | MAP_FIXED, a->fd,
                 static_cast<off_t>(offset));
  return p == MAP_FAILED ? CUDA_ERROR_INVALID_VALUE : CUDA_SUCCESS;
}
CUresult fSetAccess(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) { return CUDA_SUCCESS; }
CUresult fMemUnmap(CUdeviceptr va, size_t size) {
  {
    std::lock_guard<std::mutex> lk(g_mc_mu);
    auto it = g_mc_windows.find(reinterpret_cast<char*>(va));
    if (it != g_mc_windows.end()) {
      for (size_t i = 0; i < it->second.bases.size(); ++i) munmap(it->second.bases[i], it->second.table->member[i].size);
      g_mc_windows.erase(it);
      return CUDA_SUCCESS;
    }
  }
  // Back to a reserved, inaccessible range (as after cuMemUnmap).
  void* p = mmap(reinterpret_cast<void*>(va), size, PROT_NONE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_FIXED | MAP_NORESERVE,
                 -1, 0);
  return p == MAP_FAILED ? CUDA_ERROR_INVALID_VALUE : CUDA_SUCCESS;
}
CUresult fAddressFree(CUdeviceptr va, size_t size) {
  munmap(reinterpret_cast<void*>(va), size + kGuard);
  return CUDA_SUCCESS;
}
CUresult fMemRelease(CUmemGenericAllocationHandle h) {
  auto* a = reinterpret_cast<Alloc*>(h);
  if (a->mc) munmap(a->mc, sizeof(McTable));
  close(a->fd);
  delete a;
  return CUDA_SUCCESS;
}
CUresult fExport(void* out, CUmemGenericAllocationHandle h, CUmemAllocationHandleType, unsigned long long) {
  *static_cast<int*>(out) = dup(reinterpret_cast<Alloc*>(h)->fd);
  return CUDA_SUCCESS;
}
CUresult fImport(CUmemGenericAllocationHandle* h, void* os, CUmemAllocationHandleType) {
  const int fd = dup(static_cast<int>(reinterpret_cast<intptr_t>(os)));
  struct stat stt {};
  fstat(fd, &stt);
  auto* a = new Alloc{fd, static_cast<size_t>(stt.st_size)};
  if (multicastOn() && a->size == sizeof(McTable)) {  // VMM allocations are 2 MiB multiples
    McTable* t = mapTable(fd);
    if (t && t->magic == kMcMagic) {
      a->mc = t;
    } else if (t) {
      munmap(t, sizeof(McTable));
    }
  }
  *h = reinterpret_cast<CUmemGenericAllocationHandle>(a);
  return CUDA_SUCCESS;
}
CUresult fMcCreate(CUmemGenericAllocationHandle* h, const CUmulticastObjectProp* prop) {
  if (!multicastOn()) return CUDA_ERROR_NOT_SUPPORTED;
  if (prop->numDevices < 1 || prop->numDevices > 8) return CUDA_ERROR_INVALID_VALUE;
  const int fd = memfd_create("fakecuda-mc", MFD_CLOEXEC);
  if (fd < 0 || ftruncate(fd, sizeof(McTable)) != 0) return CUDA_ERROR_OUT_OF_MEMORY;
  McTable* t = mapTable(fd);
  if (!t) return CUDA_ERROR_OUT_OF_MEMORY;
  t->magic = kMcMagic;
  t->ndev = prop->numDevices;
  *h = reinterpret_cast<CUmemGenericAllocationHandle>(new Alloc{fd, sizeof(McTable), t});
  return CUDA_SUCCESS;
}
CUresult fMcAdd(CUmemGenericAllocationHandle h, CUdevice) {
  return reinterpret_cast<Alloc*>(h)->mc ? CUDA_SUCCESS : CUDA_ERROR_INVALID_VALUE;
}
CUresult fMcBind(CUmemGenericAllocationHandle h, size_t mc_off, CUmemGenericAllocationHandle mem, size_t mem_off,
                 size_t size, unsigned long long) {
  McTable* t = reinterpret_cast<Alloc*>(h)->mc;
  auto* m = reinterpret_cast<Alloc*>(mem);
  if (!t || mc_off != 0 || mem_off != 0 || size > m->size) return CUDA_ERROR_INVALID_VALUE;
  // Claim a member slot (ranks bind concurrently from their own processes).
  for (uint32_t i = 0; i < t->ndev; ++i) {
    int32_t expect = 0;
    if (__atomic_compare_exchange_n(&t->member[i].pid, &expect, static_cast<int32_t>(getpid()), false,
                                    __ATOMIC_ACQ_REL, __ATOMIC_ACQUIRE)) {
      t->member[i].fd = dup(m->fd);  // kept open while the process lives: peers reopen it by /proc path
      t->member[i].size = size;
      __atomic_fetch_add(&t->nbound, 1u, __ATOMIC_RELEASE);
      return CUDA_SUCCESS;
    }
  }
  return CUDA_ERROR_INVALID_VALUE;
}
CUresult fMcUnbind(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) { return CUDA_SUCCESS; }
CUresult fWaitValue32(CUstream s, CUdeviceptr addr, cuuint32_t value, unsigned int flags) {
  if ((flags & 0x3) != CU_STREAM_WAIT_VALUE_GEQ) return CUDA_ERROR_NOT_SUPPORTED;
  S(reinterpret_cast<cudaStream_t>(s))->push([addr, value] {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(addr);
    pollUntil([&] { return static_cast<int32_t>(__atomic_load_n(w, __ATOMIC_ACQUIRE) - value) >= 0; });
  });
  return CUDA_SUCCESS;
}
CUresult fWriteValue32(CUstream s, CUdeviceptr addr, cuuint32_t value, unsigned int) {
  S(reinterpret_cast<cudaStream_t>(s))->push([addr, value] {
    __atomic_store_n(reinterpret_cast<uint32_t*>(addr), value, __ATOMIC_RELEASE);
  });
  return CUDA_SUCCESS;
}

}  // namespace

// The members' memory behind a multicast window address (simt.h's multimem
// accesses): fills bases[] with each member's address of the same offset.
extern "C" int fakecuda_mc_resolve(const void* addr, char** bases, int max) {
  char* a = static_cast<char*>(const_cast<void*>(addr));
  std::lock_guard<std::mutex> lk(g_mc_mu);
  auto it = g_mc_windows.upper_bound(a);
  if (it == g_mc_windows.begin()) return -1;
  --it;
  McWindow& w = it->second;
  if (a >= w.va + w.size) return -1;
  if (w.bases.empty()) {
    const uint32_t n = __atomic_load_n(&w.table->nbound, __ATOMIC_ACQUIRE);
    if (n != w.table->ndev) return -2;  // accessed before every rank bound (the product's exchange prevents it)
    for (uint32_t i = 0; i < n; ++i) {
      char path[64];
      snprintf(path, sizeof(path), "/proc/%d/fd/%d", w.table->member[i].pid, w.table->member[i].fd);
      const int fd = open(path, O_RDWR | O_CLOEXEC);
      void* p = fd < 0 ? MAP_FAILED
                       : mmap(nullptr, w.table->member[i].size, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
      if (fd >= 0) close(fd);
      if (p == MAP_FAILED) return -3;
      w.bases.push_back(static_cast<char*>(p));
    }
  }
  const size_t off = static_cast<size_t>(a - w.va);
  const int n = static_cast<int>(w.bases.size());
  if (n > max) return -1;
  for (int i = 0; i < n; ++i) bases[i] = w.bases[i] + off;
  return n;
}

extern "C" cudaError_t cudaGetDriverEntryPoint(const char* symbol, void** fn, unsigned long long,
                                               cudaDriverEntryPointQueryResult* q) {
  static const std::map<std::string, void*> table = {
      {"cuInit", reinterpret_cast<void*>(&fInit)},
      {"cuDeviceGet", reinterpret_cast<void*>(&fDeviceGet)},
      {"cuDeviceGetAttribute", reinterpret_cast<void*>(&fDeviceGetAttribute)},
      {"cuGetErrorString", reinterpret_cast<void*>(&fGetErrorString)},
      {"cuMemGetAllocationGranularity", reinterpret_cast<void*>(&fGranularity)},
      {"cuMulticastGetGranularity", reinterpret_cast<void*>(&fMcGranularity)},
      {"cuMemCreate", reinterpret_cast<void*>(&fMemCreate)},
      {"cuMemAddressReserve", reinterpret_cast<void*>(&fAddressReserve)},
      {"cuMemMap", reinterpret_cast<void*>(&fMemMap)},
      {"cuMemSetAccess", reinterpret_cast<void*>(&fSetAccess)},
      {"cuMemUnmap", reinterpret_cast<void*>(&fMemUnmap)},
      {"cuMemAddressFree", reinterpret_cast<void*>(&fAddressFree)},
      {"cuMemRelease", reinterpret_cast<void*>(&fMemRelease)},
      {"cuMemExportToShareableHandle", reinterpret_cast<void*>(&fExport)},
      {"cuMemImportFromShareableHandle", reinterpret_cast<void*>(&fImport)},
      {"cuMulticastCreate", reinterpret_cast<void*>(&fMcCreate)},
      {"cuMulticastAddDevice", reinterpret_cast<void*>(&fMcAdd)},
      {"cuMulticastBindMem", reinterpret_cast<void*>(&fMcBind)},
      {"cuMulticastUnbind", reinterpret_cast<void*>(&fMcUnbind)},
      {"cuStreamWaitValue32", reinterpret_cast<void*>(&fWaitValue32)},
      {"cuStreamWriteValue32", reinterpret_cast<void*>(&fWriteValue32)},
  };
  auto it = table.find(symbol);
  if (it == table.end()) {
    *fn = nullptr;
    if (q) *q = cudaDriverEntryPointSymbolNotFound;
    return cudaErrorSymbolNotFound;
  }
  *fn = it->second;
  if (q) *q = cudaDriverEntryPointSuccess;
  return cudaSuccess;
}
