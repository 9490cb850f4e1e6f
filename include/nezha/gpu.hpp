// nezha/gpu.hpp — header-only C++ face of the C ABI (include/nezha_b200.h)
// for code written against the reference's C++ API: RAII handles, and ABI
// return codes mapped onto the reference's error hierarchy
// (proj/include/nezha/core/error.hpp:11-60).
//
//   nezha::gpu::Comm comm(rank, world, device, "job-42");        // rendezvous()
//   nezha::gpu::Engine eng(comm, nezha::gpu::Engine::defaults());
//   nezha::gpu::Buffer in(comm, bytes), out(comm, bytes);       // UnboundBuffer
//   eng.allreduce(in, out, bytes, NZ_F32, stream);               // SPEC.md:226 flow
//   nezha::Tensor t = ...; eng.allreduce(t, t);                  // host Tensor
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "nezha/core/error.hpp"
#include "nezha/core/types.hpp"
#include "nezha_b200.h"

namespace nezha::gpu {

inline void check(int rc) {
  if (rc >= 0) return;
  const std::string msg = nz_last_error();
  switch (rc) {
    case NZ_ERR_INVALID:
      throw std::invalid_argument(msg);
    case NZ_ERR_RAIL_DOWN:
      throw ChannelDownError(-1, -1, msg);
    case NZ_ERR_UNRECOVERABLE:
      throw UnrecoverableError(msg);
    case NZ_ERR_TIMEOUT:
      throw RendezvousTimeoutError(msg);
    default:
      throw Error(msg);
  }
}

class Comm {
 public:
  Comm(int rank, int world, int device, const std::string& session, int timeout_ms = 120000) {
    check(nz_comm_init(rank, world, device, session.c_str(), timeout_ms, &h_));
  }
  // One virtual rank of a job whose ranks are threads on one GPU
  // (nz_comm_init_loopback; the reference's ranks-as-threads fabric).
  struct Loopback {};
  Comm(Loopback, int rank, int world, int device, const std::string& session, int timeout_ms = 120000) {
    check(nz_comm_init_loopback(rank, world, device, session.c_str(), timeout_ms, &h_));
  }
  ~Comm() { nz_comm_destroy(h_); }
  Comm(const Comm&) = delete;
  Comm& operator=(const Comm&) = delete;
  nz_comm_t* get() const { return h_; }
  int rank() const { return nz_comm_rank(h_); }
  int world() const { return nz_comm_world(h_); }
  bool multicast() const { return nz_comm_multicast_supported(h_) == 1; }

 private:
  nz_comm_t* h_ = nullptr;
};

// UnboundBuffer: symmetric, multicast-bound device memory.
class Buffer {
 public:
  Buffer(Comm& comm, Bytes bytes) { check(nz_buffer_alloc(comm.get(), bytes, &h_)); }
  ~Buffer() { nz_buffer_free(h_); }
  Buffer(const Buffer&) = delete;
  Buffer& operator=(const Buffer&) = delete;
  nz_buf_t* get() const { return h_; }
  void* data() const { return nz_buffer_ptr(h_); }
  Bytes size() const { return nz_buffer_size(h_); }
  void write(const void* src, Bytes bytes, Bytes offset = 0, void* stream = nullptr) {
    check(nz_buffer_write(h_, offset, src, bytes, stream));
  }
  void read(void* dst, Bytes bytes, Bytes offset = 0, void* stream = nullptr) const {
    check(nz_buffer_read(h_, offset, dst, bytes, stream));
  }

 private:
  nz_buf_t* h_ = nullptr;
};

class Engine {
 public:
  static nz_engine_config_t defaults() {
    nz_engine_config_t c;
    nz_engine_config_default(&c);
    return c;
  }
  Engine(Comm& comm, const nz_engine_config_t& cfg) { check(nz_engine_create(comm.get(), &cfg, &h_)); }
  ~Engine() { nz_engine_destroy(h_); }
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  void allreduce(Buffer& in, Buffer& out, Bytes bytes, nz_dtype_t dtype, void* stream = nullptr) {
    check(nz_engine_allreduce(h_, in.get(), out.get(), bytes, dtype, stream));
  }
  // Host Tensor in / out (types.hpp:60-67), fp32 sum.
  void allreduce(const Tensor& in, Tensor& out) {
    out.values.resize(in.values.size());
    check(nz_engine_allreduce_host(h_, in.data(), out.data(), in.byteLength(), NZ_F32));
  }
  // Caller-owned device memory (not symmetric), asynchronous on `stream`.
  void allreduceDevice(const void* src, void* dst, Bytes bytes, nz_dtype_t dtype, void* stream = nullptr) {
    check(nz_engine_allreduce_device(h_, src, dst, bytes, dtype, stream));
  }
  // This rank's link of `rail` dies at `chunk` of op `op_seq` (unplanned:
  // the other ranks' monitors detect it, agree and reroute).
  void failRailAt(std::uint32_t op_seq, int rail, std::uint64_t chunk) {
    check(nz_engine_inject_failure(h_, op_seq, rail, chunk));
  }
  // Every handoff so far (HandoffTicket, with timings).
  std::vector<nz_failover_report_t> failovers() {
    std::vector<nz_failover_report_t> v(static_cast<size_t>(nz_engine_failover_count(h_)));
    for (size_t i = 0; i < v.size(); ++i) check(nz_engine_failover_get(h_, static_cast<int>(i), &v[i]));
    return v;
  }
  void readmit(int rail) { check(nz_engine_readmit(h_, rail)); }
  void synchronize() { check(nz_engine_synchronize(h_)); }
  std::uint32_t opSeq() const { return nz_engine_op_seq(h_); }

 private:
  nz_engine_t* h_ = nullptr;
};

}  // namespace nezha::gpu
