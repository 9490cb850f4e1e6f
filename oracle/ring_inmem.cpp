// ring_inmem.cpp — the SPEC ring allreduce executed on the reference's own
// transport. TEST INFRASTRUCTURE / CPU BASELINE ONLY (never in the product).
//
// Built against /root/reference/proj headers and libnezha_ref.a (the
// reference's core + in-memory transport compiled where they lie, see
// oracle/Makefile). Restates, on that transport:
//   ring_allreduce          SPEC.md:189-197 (reduce-scatter then allgather,
//                           2(N-1) steps, rank r sends block (r - s) mod N)
//   ring_chunked_allreduce  SPEC.md:198-205, chunk = max(64 KiB, len/2N) :223
//   rank-ascending order    SPEC.md:222; last block absorbs the remainder :224
//   one executor per rail   SPEC.md:226 (a thread per (rank, rail))
//   handoff                 SPEC.md:389-397, :411, :414: a rail killed at
//                           chunk k aborts with OperationAbortedError; the
//                           survivor with the largest data_length finishes
//                           its own segment, then reduces the orphan
//                           [off + kC, end) with the failed rail's geometry.
// DATA frames carry (op_seq, chunk_index, offset) as SPEC.md:228 states and
// are cut at the rail's max_frame_payload (64 KiB, types.hpp:32).
// bf16 (P2): reduce-scatter carries fp32 partials, the block owner
// rounds once (RNE), allgather carries bf16.
#include <atomic>
#include <barrier>
#include <chrono>
#include <functional>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <thread>
#include <vector>

#include "nezha/core/error.hpp"
#include "nezha/core/math.hpp"
#include "nezha/core/types.hpp"
#include "nezha/transport/inmem.hpp"

namespace {

using nezha::Bytes;
using nezha::Frame;
using nezha::MsgType;

enum { F32 = 0, BF16 = 1, I32 = 2 };

float bf2f(uint16_t h) {
  uint32_t u = static_cast<uint32_t>(h) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

uint16_t f2bf(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return static_cast<uint16_t>((u >> 16) | 0x40u);
  u += 0x7fffu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

struct Job {
  int world = 0;
  int dtype = F32;
  bool chunked = true;
  Bytes nbytes = 0;
  const void* const* in = nullptr;
  void* const* out = nullptr;
  std::vector<int> seg_rail;
  std::vector<Bytes> seg_off, seg_len;
  int fail_rail = -1;
  uint64_t fail_chunk = 0;
  // Every rank's executor of the failing rail arrives here before chunk k;
  // the completion step kills the rail fabric-wide before anyone proceeds,
  // so chunks [0, k) are complete everywhere and none of chunk k is.
  std::barrier<std::function<void()>>* fail_gate = nullptr;
};

// Per-rank handoff mailbox: the failed executor posts its orphan, the target
// executor takes it after finishing its own segment.
struct Mailbox {
  std::mutex mu;
  std::condition_variable cv;
  int pending = 0;  // executors of this rank still running their own segment
  bool has_orphan = false;
  Bytes orphan_off = 0, orphan_len = 0, seg_off = 0, seg_len = 0, chunk = 0;
};

Bytes chunkOf(Bytes seg_len, int world, bool chunked) {
  if (!chunked) return seg_len < 4 ? 4 : seg_len;
  Bytes even = (seg_len / (2 * static_cast<Bytes>(world))) & ~Bytes{3};
  return even > 65536 ? even : 65536;
}

class Executor {
 public:
  Executor(const Job& job, nezha::ConnectionSet& cs, int rail, uint32_t op_seq)
      : job_(job), cs_(cs), rail_(rail), op_seq_(op_seq), N_(job.world), r_(cs.rank()) {
    es_ = job.dtype == BF16 ? 2 : 4;
    frame_ = cs.rails().at(rail).max_frame_payload;
  }

  // Allreduce chunks [c_begin, end) of geometry (seg_off, seg_len, C).
  // Returns the first chunk NOT completed when the rail goes down.
  uint64_t run(Bytes seg_off, Bytes seg_len, Bytes C, uint64_t c_begin, int kill_at_chunk) {
    const uint64_t nch = (seg_len + C - 1) / C;
    for (uint64_t c = c_begin; c < nch; ++c) {
      if (kill_at_chunk >= 0 && c == static_cast<uint64_t>(kill_at_chunk) && job_.fail_gate) {
        job_.fail_gate->arrive_and_wait();  // the scripted failure happens in the completion step
      }
      const Bytes off = seg_off + c * C;
      const Bytes len = std::min(C, seg_len - c * C);
      try {
        chunkRing(off, len);
      } catch (const nezha::ChannelDownError&) {
        return c;
      } catch (const nezha::Error&) {
        return c;
      }
    }
    return nch;
  }

 private:
  // Wire helpers: a logical message is cut into frames of <= max_frame_payload.
  void sendBlock(nezha::Channel& ch, const uint8_t* p, Bytes n, Bytes offset) {
    Bytes sent = 0;
    do {
      const Bytes k = std::min<Bytes>(frame_, n - sent);
      Frame f;
      f.type = MsgType::Data;
      f.op_seq = op_seq_;
      f.chunk_index = chunk_counter_++;
      f.offset = offset + sent;
      f.payload.assign(p + sent, p + sent + k);
      ch.send(std::move(f)).wait();
      sent += k;
    } while (sent < n);
  }

  void recvBlock(nezha::Channel& ch, uint8_t* p, Bytes n) {
    Bytes got = 0;
    do {
      Frame f = ch.recv(std::chrono::microseconds(30'000'000));
      if (f.op_seq != op_seq_) throw nezha::ProtocolError("op_seq mismatch");
      std::memcpy(p + got, f.payload.data(), f.payload.size());
      got += f.payload.size();
    } while (got < n);
  }

  void chunkRing(Bytes off, Bytes len) {
    const uint64_t E = len / es_;
    const uint64_t q = E / N_;
    auto blkBegin = [&](int b) { return q == 0 ? (b == N_ - 1 ? 0 : 0) : static_cast<uint64_t>(b) * q; };
    auto blkEnd = [&](int b) { return b == N_ - 1 ? E : (q == 0 ? 0 : static_cast<uint64_t>(b + 1) * q); };
    // Accumulator: fp32 for f32/bf16 (P2), u32 for i32.
    std::vector<uint32_t> acc(E);
    const uint8_t* in = static_cast<const uint8_t*>(job_.in[r_]) + off;
    if (job_.dtype == BF16) {
      for (uint64_t i = 0; i < E; ++i) {
        uint16_t h;
        std::memcpy(&h, in + 2 * i, 2);
        const float f = bf2f(h);
        std::memcpy(&acc[i], &f, 4);
      }
    } else {
      std::memcpy(acc.data(), in, E * 4);
    }
    nezha::Channel& next = cs_.channel(rail_, (r_ + 1) % N_);
    nezha::Channel& prev = cs_.channel(rail_, (r_ + N_ - 1) % N_);
    std::vector<uint32_t> tmp;
    // Reduce-scatter.
    for (int s = 0; s < N_ - 1; ++s) {
      const int sb = ((r_ - s) % N_ + N_) % N_;
      const int rb = ((r_ - s - 1) % N_ + N_) % N_;
      sendBlock(next, reinterpret_cast<const uint8_t*>(acc.data() + blkBegin(sb)), (blkEnd(sb) - blkBegin(sb)) * 4,
                off + blkBegin(sb) * es_);
      const uint64_t n = blkEnd(rb) - blkBegin(rb);
      tmp.resize(n);
      recvBlock(prev, reinterpret_cast<uint8_t*>(tmp.data()), n * 4);  // an empty block still travels as one frame
      uint32_t* dst = acc.data() + blkBegin(rb);
      for (uint64_t i = 0; i < n; ++i) {
        if (job_.dtype == I32) {
          dst[i] = tmp[i] + dst[i];
        } else {
          float a, b;
          std::memcpy(&a, &tmp[i], 4);
          std::memcpy(&b, &dst[i], 4);
          const float c = a + b;  // recv + own
          std::memcpy(&dst[i], &c, 4);
        }
      }
    }
    // Final values in the payload dtype.
    std::vector<uint8_t> fin(len);
    const int own = (r_ + 1) % N_;
    auto finalize = [&](int b) {
      for (uint64_t i = blkBegin(b); i < blkEnd(b); ++i) {
        if (job_.dtype == BF16) {
          float f;
          std::memcpy(&f, &acc[i], 4);
          const uint16_t h = f2bf(f);
          std::memcpy(fin.data() + 2 * i, &h, 2);
        } else {
          std::memcpy(fin.data() + 4 * i, &acc[i], 4);
        }
      }
    };
    finalize(own);
    // Allgather.
    for (int s = 0; s < N_ - 1; ++s) {
      const int sb = ((r_ + 1 - s) % N_ + N_) % N_;
      const int rb = ((r_ - s) % N_ + N_) % N_;
      sendBlock(next, fin.data() + blkBegin(sb) * es_, (blkEnd(sb) - blkBegin(sb)) * es_, off + blkBegin(sb) * es_);
      const uint64_t n = blkEnd(rb) - blkBegin(rb);
      recvBlock(prev, fin.data() + blkBegin(rb) * es_, n * es_);
    }
    std::memcpy(static_cast<uint8_t*>(job_.out[r_]) + off, fin.data(), len);  // commit the whole chunk at once
  }

  const Job& job_;
  nezha::ConnectionSet& cs_;
  int rail_;
  uint32_t op_seq_;
  int N_;
  int r_;
  Bytes es_ = 4;
  Bytes frame_ = 65536;
  uint32_t chunk_counter_ = 0;
};

}  // namespace

extern "C" {

/*
 * Multi-rail allreduce on the reference InMemoryFabric: world rank threads,
 * one executor thread per (rank, rail). Segments (rail, off, len) must cover
 * [0, nbytes). fail_rail >= 0 kills that rail at chunk fail_chunk of its
 * segment (deterministic P10 injection); its orphan is handed to the
 * surviving rail with the largest data_length (ties: lowest id, P9).
 * Returns 0; -1 bad args; -2 unrecoverable; -3 internal error.
 * *elapsed_us: wall time from thread start to join. *rank0_bytes: Data bytes
 * rank 0 put on the wire (Eq. 1 accounting, transport.hpp:111-116).
 */
int nzi_multirail_allreduce(int world, int dtype, int chunked, const void* const* inputs, void* const* outputs,
                            uint64_t nbytes, int nsegs, const int* seg_rail, const uint64_t* seg_off,
                            const uint64_t* seg_len, int nrails, int fail_rail, uint64_t fail_chunk, uint32_t op_seq,
                            double* elapsed_us, uint64_t* rank0_bytes) {
  try {
    if (world < 2 || nrails < 1 || nsegs < 1) return -1;
    Job job;
    job.world = world;
    job.dtype = dtype;
    job.chunked = chunked != 0;
    job.nbytes = nbytes;
    job.in = inputs;
    job.out = outputs;
    for (int i = 0; i < nsegs; ++i) {
      job.seg_rail.push_back(seg_rail[i]);
      job.seg_off.push_back(seg_off[i]);
      job.seg_len.push_back(seg_len[i]);
    }
    job.fail_rail = fail_rail;
    job.fail_chunk = fail_chunk;
    std::vector<nezha::RailProfile> rails;
    for (int r = 0; r < nrails; ++r) {
      nezha::RailProfile p;
      p.rail_id = r;
      p.bandwidth_bps = 1e9;
      rails.push_back(p);
    }
    // P9 target: largest data_length among the other rails, ties -> lowest id.
    int target = -1;
    Bytes best = 0;
    for (int r = 0; r < nrails; ++r) {
      if (r == fail_rail) continue;
      Bytes tot = 0;
      for (int i = 0; i < nsegs; ++i)
        if (seg_rail[i] == r) tot += seg_len[i];
      if (target < 0 || tot > best) {
        target = r;
        best = tot;
      }
    }
    auto fabric = std::make_shared<nezha::InMemoryFabric>(world, rails);
    std::unique_ptr<std::barrier<std::function<void()>>> gate;
    if (fail_rail >= 0) {
      gate = std::make_unique<std::barrier<std::function<void()>>>(world, std::function<void()>([&fabric, fail_rail] {
        try {
          fabric->killRail(fail_rail);
        } catch (...) {
        }
      }));
      job.fail_gate = gate.get();
    }
    std::vector<std::unique_ptr<nezha::ConnectionSet>> sets;
    for (int r = 0; r < world; ++r) sets.push_back(fabric->connect(r));
    std::vector<Mailbox> boxes(world);
    std::atomic<int> status{0};
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> threads;
    for (int rank = 0; rank < world; ++rank) {
      for (int i = 0; i < nsegs; ++i) boxes[rank].pending++;
      for (int i = 0; i < nsegs; ++i) {
        threads.emplace_back([&, rank, i] {
          const int rail = job.seg_rail[i];
          const Bytes C = chunkOf(job.seg_len[i], world, job.chunked);
          Executor ex(job, *sets[rank], rail, op_seq);
          const int kill = rail == job.fail_rail ? static_cast<int>(job.fail_chunk) : -1;
          const uint64_t done = job.seg_len[i] ? ex.run(job.seg_off[i], job.seg_len[i], C, 0, kill) : 0;
          const uint64_t nch = job.seg_len[i] ? (job.seg_len[i] + C - 1) / C : 0;
          Mailbox& mb = boxes[rank];
          {
            std::unique_lock lk(mb.mu);
            if (done < nch) {
              mb.has_orphan = true;
              mb.seg_off = job.seg_off[i];
              mb.seg_len = job.seg_len[i];
              mb.chunk = C;
              mb.orphan_off = done;  // first chunk to redo
            }
            mb.pending--;
            mb.cv.notify_all();
          }
          if (rail != target) return;
          // Target: after its own task, wait for every executor of this rank,
          // then run the orphan with the failed rail's geometry.
          std::unique_lock lk(mb.mu);
          mb.cv.wait(lk, [&] { return mb.pending == 0; });
          if (!mb.has_orphan) return;
          const Bytes so = mb.seg_off, sl = mb.seg_len, cc = mb.chunk;
          const uint64_t first = mb.orphan_off;
          lk.unlock();
          Executor hand(job, *sets[rank], rail, op_seq + 0x40000000u);
          if (hand.run(so, sl, cc, first, -1) < (sl + cc - 1) / cc) status = -3;
        });
      }
    }
    for (auto& t : threads) t.join();
    const auto t1 = std::chrono::steady_clock::now();
    if (elapsed_us) *elapsed_us = std::chrono::duration<double, std::micro>(t1 - t0).count();
    if (rank0_bytes) *rank0_bytes = sets[0]->dataBytesSent();
    if (fail_rail >= 0 && target < 0) return -2;
    return status.load();
  } catch (...) {
    return -3;
  }
}

}  // extern "C"
