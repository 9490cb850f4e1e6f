// Bootstrap and symmetric memory: the B200 replacement of the reference's
// rendezvous + ConnectionSet (proj/include/nezha/transport/transport.hpp:219-238,
// proj/src/transport/rendezvous.cpp:19-99).
//
// The reference publishes listen addresses through a shared directory of
// JSON records and then dials sockets. Here the "channels" are NVLink
// mappings, so what has to travel between the rank processes is file
// descriptors of VMM allocations and of the NVSwitch multicast object. They
// travel over abstract unix sockets (SCM_RIGHTS), one short connection per
// message, named after the job's session string. Each rank has two control
// channels (the issuing thread's and the failure monitor's), so the monitor
// can agree with its peers while the issuing thread is inside an exchange.
//
// Loopback ranks (nz_comm_init_loopback) are threads of one process on one
// GPU: their exchanges meet in an in-process mailbox instead.
#include <fcntl.h>
#include <poll.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>

#include "internal.h"

namespace nz {

namespace {
thread_local std::string g_last_error;

struct WireHeader {
  uint64_t seq;
  int32_t from;
  uint32_t bytes;
  uint32_t nfds;
  uint32_t pad;
};

constexpr size_t kMaxMsg = 60 * 1024;
constexpr int kMaxFds = 16;

sockaddr_un socketName(const std::string& session, int channel, int rank, socklen_t* len) {
  sockaddr_un a{};
  a.sun_family = AF_UNIX;
  const std::string name = "nezha-b200-" + session + (channel ? "-mon-" : "-") + std::to_string(rank);
  if (name.size() + 1 >= sizeof(a.sun_path)) fail(NZ_ERR_INVALID, "session name too long");
  a.sun_path[0] = '\0';  // abstract namespace: nothing on disk to clean up
  memcpy(a.sun_path + 1, name.data(), name.size());
  *len = static_cast<socklen_t>(offsetof(sockaddr_un, sun_path) + 1 + name.size());
  return a;
}

using Clock = std::chrono::steady_clock;

void sendTo(nz_comm* c, int channel, int peer, uint64_t seq, const void* data, size_t bytes,
            const std::vector<int>& fds) {
  socklen_t len;
  sockaddr_un addr = socketName(c->session, channel, peer, &len);
  const auto deadline = Clock::now() + std::chrono::milliseconds(c->timeout_ms);
  int s = -1;
  while (true) {
    s = socket(AF_UNIX, SOCK_SEQPACKET | SOCK_CLOEXEC, 0);
    if (s < 0) fail(NZ_ERR_SYSTEM, std::string("socket: ") + strerror(errno));
    if (connect(s, reinterpret_cast<sockaddr*>(&addr), len) == 0) break;
    const int err = errno;
    close(s);
    if (err != ECONNREFUSED && err != ENOENT && err != EAGAIN) {
      fail(NZ_ERR_SYSTEM, std::string("connect: ") + strerror(err));
    }
    if (Clock::now() > deadline) fail(NZ_ERR_TIMEOUT, "rendezvous timeout connecting to rank " + std::to_string(peer));
    std::this_thread::sleep_for(std::chrono::microseconds(200));
  }
  WireHeader h{seq, c->rank, static_cast<uint32_t>(bytes), static_cast<uint32_t>(fds.size()), 0};
  std::vector<char> buf(sizeof(h) + bytes);
  memcpy(buf.data(), &h, sizeof(h));
  if (bytes) memcpy(buf.data() + sizeof(h), data, bytes);
  iovec iov{buf.data(), buf.size()};
  msghdr m{};
  m.msg_iov = &iov;
  m.msg_iovlen = 1;
  alignas(cmsghdr) char cbuf[CMSG_SPACE(sizeof(int) * kMaxFds)];
  if (!fds.empty()) {
    m.msg_control = cbuf;
    m.msg_controllen = CMSG_SPACE(sizeof(int) * fds.size());
    cmsghdr* cm = CMSG_FIRSTHDR(&m);
    cm->cmsg_level = SOL_SOCKET;
    cm->cmsg_type = SCM_RIGHTS;
    cm->cmsg_len = CMSG_LEN(sizeof(int) * fds.size());
    memcpy(CMSG_DATA(cm), fds.data(), sizeof(int) * fds.size());
  }
  const ssize_t n = sendmsg(s, &m, MSG_NOSIGNAL);
  close(s);
  if (n != static_cast<ssize_t>(buf.size())) fail(NZ_ERR_SYSTEM, std::string("sendmsg: ") + strerror(errno));
}

// Accepts one message into the channel's stash. Returns false on timeout.
bool receiveOne(Channel& ch, int wait_ms) {
  pollfd p{ch.listen_fd, POLLIN, 0};
  const int r = poll(&p, 1, wait_ms);
  if (r == 0) return false;
  if (r < 0) fail(NZ_ERR_SYSTEM, std::string("poll: ") + strerror(errno));
  const int s = accept4(ch.listen_fd, nullptr, nullptr, SOCK_CLOEXEC);
  if (s < 0) fail(NZ_ERR_SYSTEM, std::string("accept: ") + strerror(errno));
  std::vector<char> buf(sizeof(WireHeader) + kMaxMsg);
  iovec iov{buf.data(), buf.size()};
  msghdr m{};
  m.msg_iov = &iov;
  m.msg_iovlen = 1;
  alignas(cmsghdr) char cbuf[CMSG_SPACE(sizeof(int) * kMaxFds)];
  m.msg_control = cbuf;
  m.msg_controllen = sizeof(cbuf);
  const ssize_t n = recvmsg(s, &m, MSG_CMSG_CLOEXEC);
  close(s);
  if (n < static_cast<ssize_t>(sizeof(WireHeader))) fail(NZ_ERR_SYSTEM, "short rendezvous message");
  WireHeader h;
  memcpy(&h, buf.data(), sizeof(h));
  if (h.bytes + sizeof(h) != static_cast<size_t>(n)) fail(NZ_ERR_SYSTEM, "truncated rendezvous message");
  Msg msg;
  msg.data.assign(buf.data() + sizeof(h), buf.data() + n);
  for (cmsghdr* cm = CMSG_FIRSTHDR(&m); cm; cm = CMSG_NXTHDR(&m, cm)) {
    if (cm->cmsg_level == SOL_SOCKET && cm->cmsg_type == SCM_RIGHTS) {
      const size_t k = (cm->cmsg_len - CMSG_LEN(0)) / sizeof(int);
      const int* f = reinterpret_cast<const int*>(CMSG_DATA(cm));
      msg.fds.insert(msg.fds.end(), f, f + k);
    }
  }
  if (msg.fds.size() != h.nfds) fail(NZ_ERR_SYSTEM, "fd count mismatch in rendezvous message");
  ch.stash[{h.seq, h.from}] = std::move(msg);
  return true;
}

int openListener(nz_comm* c, int channel) {
  const int fd = socket(AF_UNIX, SOCK_SEQPACKET | SOCK_CLOEXEC, 0);
  if (fd < 0) fail(NZ_ERR_SYSTEM, std::string("socket: ") + strerror(errno));
  socklen_t len;
  sockaddr_un addr = socketName(c->session, channel, c->rank, &len);
  if (bind(fd, reinterpret_cast<sockaddr*>(&addr), len) != 0) {
    const int err = errno;
    close(fd);
    fail(NZ_ERR_SYSTEM, std::string("bind rendezvous socket: ") + strerror(err));
  }
  if (listen(fd, 256) != 0) {
    const int err = errno;
    close(fd);
    fail(NZ_ERR_SYSTEM, std::string("listen: ") + strerror(err));
  }
  return fd;
}

// Loopback exchange: the messages of one (channel, sequence) meet in the
// group's mailbox; the last reader clears them.
std::vector<Msg> loopExchange(nz_comm* c, int channel, uint64_t seq, const void* data, size_t bytes) {
  LoopGroup& g = *c->loop;
  std::vector<Msg> out(c->world);
  std::unique_lock<std::mutex> lk(g.m);
  g.box[{channel, seq, c->rank}].assign(static_cast<const char*>(data), static_cast<const char*>(data) + bytes);
  g.cv.notify_all();
  const auto deadline = Clock::now() + std::chrono::milliseconds(c->timeout_ms);
  for (int p = 0; p < c->world; ++p) {
    while (g.box.find({channel, seq, p}) == g.box.end()) {
      if (g.aborted) fail(NZ_ERR_TIMEOUT, "loopback group aborted: a virtual rank failed");
      if (g.cv.wait_until(lk, deadline) == std::cv_status::timeout && g.box.find({channel, seq, p}) == g.box.end()) {
        fail(NZ_ERR_TIMEOUT, "loopback rendezvous timeout waiting for virtual rank " + std::to_string(p));
      }
    }
    out[p].data = g.box[{channel, seq, p}];
  }
  if (++g.reads[{channel, seq}] == c->world) {
    for (int p = 0; p < c->world; ++p) g.box.erase({channel, seq, p});
    g.reads.erase({channel, seq});
  }
  return out;
}

std::mutex g_groups_mu;
std::map<std::string, std::weak_ptr<LoopGroup>> g_groups;

}  // namespace

LoopGroup::~LoopGroup() {
  cudaSetDevice(device);
  for (auto& kv : rails) {
    if (kv.second->stream) {
      cudaStreamSynchronize(kv.second->stream);
      cudaStreamDestroy(kv.second->stream);
    }
    for (auto& pr : kv.second->tev) {
      cudaEventDestroy(pr.first);
      cudaEventDestroy(pr.second);
    }
  }
}

const DriverApi& drv() {
  static const DriverApi api = [] {
    DriverApi a;
    cudaDriverEntryPointQueryResult q;
#define NZ_DRV_FN(name)                                                                            \
  if (cudaGetDriverEntryPoint(#name, reinterpret_cast<void**>(&a.name), cudaEnableDefault, &q) != \
          cudaSuccess ||                                                                           \
      q != cudaDriverEntryPointSuccess)                                                            \
    a.name = nullptr;
#include "driver_fns.inc"
#undef NZ_DRV_FN
    return a;
  }();
  return api;
}

void setLastError(const std::string& msg) { g_last_error = msg; }
const char* lastError() { return g_last_error.c_str(); }

void fail(int code, const std::string& msg) { throw ApiError(code, msg); }

void checkCuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(NZ_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

void checkCu(CUresult e, const char* what) {
  if (e != CUDA_SUCCESS) {
    const char* s = nullptr;
    if (drv().cuGetErrorString) drv().cuGetErrorString(e, &s);
    fail(NZ_ERR_CUDA, std::string(what) + ": " + (s ? s : "unknown CUresult"));
  }
}

std::vector<Msg> exchange(nz_comm* c, const void* data, size_t bytes, const std::vector<int>& fds, int channel) {
  if (bytes > kMaxMsg) fail(NZ_ERR_INVALID, "exchange payload too large");
  if (fds.size() > static_cast<size_t>(kMaxFds)) fail(NZ_ERR_INVALID, "too many fds in one exchange");
  if (channel < 0 || channel >= kChannels) fail(NZ_ERR_INVALID, "bad exchange channel");
  Channel& ch = c->chan[channel];
  const uint64_t seq = ch.seq++;
  if (c->loop) {
    if (!fds.empty()) fail(NZ_ERR_INVALID, "loopback ranks exchange no file descriptors");
    return loopExchange(c, channel, seq, data, bytes);
  }
  std::vector<Msg> out(c->world);
  out[c->rank].data.assign(static_cast<const char*>(data), static_cast<const char*>(data) + bytes);
  if (c->world == 1) return out;
  for (int k = 1; k < c->world; ++k) sendTo(c, channel, (c->rank + k) % c->world, seq, data, bytes, fds);
  const auto deadline = Clock::now() + std::chrono::milliseconds(c->timeout_ms);
  for (int p = 0; p < c->world; ++p) {
    if (p == c->rank) continue;
    while (ch.stash.find({seq, p}) == ch.stash.end()) {
      const auto left = std::chrono::duration_cast<std::chrono::milliseconds>(deadline - Clock::now()).count();
      if (left <= 0 || !receiveOne(ch, static_cast<int>(std::min<long long>(left, 1000)))) {
        if (Clock::now() > deadline) fail(NZ_ERR_TIMEOUT, "rendezvous timeout waiting for rank " + std::to_string(p));
      }
    }
    auto it = ch.stash.find({seq, p});
    out[p] = std::move(it->second);
    ch.stash.erase(it);
  }
  return out;
}

bool peekExchange(nz_comm* c, int channel, std::vector<std::vector<char>>* blobs) {
  blobs->clear();
  if (c->world == 1) return false;
  Channel& ch = c->chan[channel];
  if (c->loop) {
    LoopGroup& g = *c->loop;
    std::lock_guard<std::mutex> lk(g.m);
    for (int p = 0; p < c->world; ++p) {
      if (p == c->rank) continue;
      auto it = g.box.find({channel, ch.seq, p});
      if (it != g.box.end()) blobs->push_back(it->second);
    }
    return !blobs->empty();
  }
  while (receiveOne(ch, 0)) {
  }
  for (int p = 0; p < c->world; ++p) {
    if (p == c->rank) continue;
    auto it = ch.stash.find({ch.seq, p});
    if (it != ch.stash.end()) blobs->push_back(it->second.data);
  }
  return !blobs->empty();
}

namespace {

// Multi-process communicators still open. A rank process that exits without
// destroying its communicator (an exception on the host, a failed test) takes
// its symmetric memory with it while a late peer's kernel may still read or
// write that memory over NVLink — a fabric fault on the peer's GPU. At exit
// the process therefore holds on for the device wait budget, after which
// every peer kernel has given up on its own.
std::atomic<int> g_open_shared{0};

void holdAtExit() {
  const int n = g_open_shared.load();
  if (n <= 0) return;
  const auto ms = static_cast<long long>(watchdogNs() / 1000000ull) + 1000;
  fprintf(stderr,
          "[nezha] exiting with %d open multi-process communicator(s): holding this rank's memory for %lld ms so "
          "peers' kernels time out before it is unmapped\n",
          n, ms);
  std::this_thread::sleep_for(std::chrono::milliseconds(ms));
}

int commInit(int rank, int world, int device, const char* session, int timeout_ms, bool loopback, nz_comm_t** out) {
  return guarded([&] {
    if (!out || !session) fail(NZ_ERR_INVALID, "nz_comm_init: null argument");
    if (world < 1 || world > kMaxRanks) fail(NZ_ERR_INVALID, "world must be in [1, 8]");
    if (rank < 0 || rank >= world) fail(NZ_ERR_INVALID, "rank out of range");
    auto* c = new nz_comm();
    c->rank = rank;
    c->world = world;
    c->device = device;
    c->session = session;
    c->timeout_ms = timeout_ms > 0 ? timeout_ms : 60000;
    try {
      NZ_CUDA(cudaSetDevice(device));
      NZ_CUDA(cudaFree(nullptr));  // create the primary context
      if (!drv().cuMulticastBindMem || !drv().cuMemCreate) fail(NZ_ERR_CUDA, "CUDA driver entry points unavailable");
      NZ_CU(NZ_DRV(cuInit)(0));
      CUdevice dev;
      NZ_CU(NZ_DRV(cuDeviceGet)(&dev, device));
      int mc = 0;
      NZ_CU(NZ_DRV(cuDeviceGetAttribute)(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
      NZ_CU(NZ_DRV(cuDeviceGetAttribute)(&c->sm_count, CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT, dev));
      if (loopback) {
        std::lock_guard<std::mutex> lk(g_groups_mu);
        auto& w = g_groups[c->session];
        auto g = w.lock();
        if (!g) {
          g = std::make_shared<LoopGroup>();
          g->world = world;
          g->device = device;
          w = g;
        }
        if (g->world != world || g->device != device) fail(NZ_ERR_INVALID, "loopback ranks disagree on world / device");
        if (g->joined & (1u << rank)) fail(NZ_ERR_INVALID, "loopback rank joined twice");
        g->joined |= 1u << rank;
        c->loop = g;
        c->multicast = false;  // one GPU: no NVSwitch multicast team
      } else if (world > 1) {
        for (int ch = 0; ch < kChannels; ++ch) c->chan[ch].listen_fd = openListener(c, ch);
        // Every rank must agree on multicast before any buffer is built.
        const auto all = exchange(c, &mc, sizeof(mc), {});
        int agreed = 1;
        for (const auto& m : all) {
          int v = 0;
          memcpy(&v, m.data.data(), sizeof(v));
          agreed &= (v != 0);
        }
        c->multicast = agreed && getenv("NEZHA_DISABLE_MULTICAST") == nullptr;
      }
      c->ctrl = allocSymmetric(c, kPadBytes * kMaxRails);
      NZ_CUDA(cudaMemset(c->ctrl->ptrs[rank], 0, c->ctrl->mapped));
      NZ_CUDA(cudaDeviceSynchronize());
      exchange(c, nullptr, 0, {});  // pads are zero everywhere before first use
      if (!c->loop && world > 1) {
        static std::once_flag once;
        std::call_once(once, [] { std::atexit(holdAtExit); });
        g_open_shared.fetch_add(1);
      }
    } catch (...) {
      for (auto& ch : c->chan)
        if (ch.listen_fd >= 0) close(ch.listen_fd);
      if (c->loop) {
        std::lock_guard<std::mutex> lk(g_groups_mu);
        c->loop->joined &= ~(1u << rank);
      }
      delete c;
      throw;
    }
    *out = c;
  });
}

}  // namespace

}  // namespace nz

using nz::fail;
using nz::guarded;

extern "C" {

const char* nz_last_error(void) { return nz::lastError(); }
int nz_abi_version(void) { return NZ_ABI_VERSION; }

int nz_abi_sizeof(const char* type_name) {
  if (!type_name) return NZ_ERR_INVALID;
  const std::string n = type_name;
  if (n == "engine_config") return static_cast<int>(sizeof(nz_engine_config_t));
  if (n == "failover_report") return static_cast<int>(sizeof(nz_failover_report_t));
  if (n == "rail_status") return static_cast<int>(sizeof(nz_rail_status_t));
  if (n == "fault_record") return static_cast<int>(sizeof(nz_fault_record_t));
  return NZ_ERR_INVALID;
}

int nz_comm_init(int rank, int world, int device, const char* session, int timeout_ms, nz_comm_t** out) {
  return nz::commInit(rank, world, device, session, timeout_ms, false, out);
}

int nz_comm_init_loopback(int rank, int world, int device, const char* session, int timeout_ms, nz_comm_t** out) {
  return nz::commInit(rank, world, device, session, timeout_ms, true, out);
}

int nz_comm_is_loopback(const nz_comm_t* c) { return c ? (c->loop ? 1 : 0) : NZ_ERR_INVALID; }

int nz_comm_abort(nz_comm_t* comm) {
  return guarded([&] {
    if (!comm) fail(NZ_ERR_INVALID, "null argument");
    if (!comm->loop) return;
    nz::LoopGroup& g = *comm->loop;
    std::lock_guard<std::mutex> lk(g.m);
    g.aborted = true;
    g.cv.notify_all();
    for (auto& kv : g.rails) {
      std::lock_guard<std::mutex> rl(kv.second->m);
      kv.second->cv.notify_all();
    }
  });
}

int nz_comm_destroy(nz_comm_t* comm) {
  return guarded([&] {
    if (!comm) return;
    cudaSetDevice(comm->device);
    if (comm->ctrl) nz::freeSymmetric(comm->ctrl);  // collective: ranks leave together
    if (!comm->loop && comm->world > 1) nz::g_open_shared.fetch_sub(1);
    for (auto& ch : comm->chan) {
      for (auto& kv : ch.stash)
        for (int fd : kv.second.fds) close(fd);
      if (ch.listen_fd >= 0) close(ch.listen_fd);
    }
    if (comm->loop) {
      std::lock_guard<std::mutex> lk(nz::g_groups_mu);
      comm->loop->joined &= ~(1u << comm->rank);
    }
    delete comm;
  });
}

int nz_comm_rank(const nz_comm_t* c) { return c ? c->rank : NZ_ERR_INVALID; }
int nz_comm_world(const nz_comm_t* c) { return c ? c->world : NZ_ERR_INVALID; }
int nz_comm_device(const nz_comm_t* c) { return c ? c->device : NZ_ERR_INVALID; }
int nz_comm_sm_count(const nz_comm_t* c) { return c ? c->sm_count : NZ_ERR_INVALID; }
int nz_comm_multicast_supported(const nz_comm_t* c) { return c ? (c->multicast ? 1 : 0) : NZ_ERR_INVALID; }

int nz_comm_barrier(nz_comm_t* comm) {
  return guarded([&] {
    if (!comm) fail(NZ_ERR_INVALID, "null comm");
    if (comm->world > 1) nz::exchange(comm, nullptr, 0, {});
  });
}

int nz_comm_allgather(nz_comm_t* comm, const void* mine, size_t bytes, void* all) {
  return guarded([&] {
    if (!comm || (!mine && bytes) || (!all && bytes)) fail(NZ_ERR_INVALID, "null argument");
    if (comm->world == 1) {
      if (bytes) memcpy(all, mine, bytes);
      return;
    }
    const auto msgs = nz::exchange(comm, mine, bytes, {});
    for (int r = 0; r < comm->world; ++r) {
      if (msgs[r].data.size() != bytes) fail(NZ_ERR_INVALID, "allgather size mismatch across ranks");
      if (bytes) memcpy(static_cast<char*>(all) + size_t(r) * bytes, msgs[r].data.data(), bytes);
    }
  });
}

}  // extern "C"
