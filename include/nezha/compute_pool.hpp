// nezha/compute_pool.hpp — ComputePool: per-phase compute tokens for the
// rails of one rank.
//
// The paper splits every rail's allreduce into I/O, communication and
// computation phases; only the computation phase needs cores, so cores are
// granted on entry to it and recovered on exit. On B200 the cores are SMs:
// a rail's computation demand is the CTA grid of its SM-driven kernel (NVLS
// multimem reduce, SM-rail peer fold, CE-rail local fold), while its I/O and
// communication phases run on the copy engines / NVSwitch and hold no SMs.
// The engine drives the pool in stream order: a computation
// grant that does not fit waits, on the device, for the release event of the
// oldest holder instead of blocking the issuing thread.
//
// Pinned semantics (P14; the SPEC leaves the accounting open):
//  - io / communication grants are 1 token, always immediate, and are not
//    counted against total_tokens (they model the progress thread, not cores);
//  - a computation grant is min(declared demand, total_tokens)
//    and is served FIFO among computation requests: granted when no earlier
//    request waits and outstanding + grant <= total_tokens; demand 0 is an
//    immediate grant of 0;
//  - one grant outstanding per rail: acquiring while holding,
//    releasing what is not held, or using an undeclared rail throws
//    std::invalid_argument. With no hold-and-wait there is no deadlock.
#pragma once

#include <condition_variable>
#include <cstdint>
#include <deque>
#include <map>
#include <mutex>
#include <optional>
#include <utility>
#include <vector>

namespace nezha {

enum class Phase : std::uint8_t { Io = 0, Communication = 1, Computation = 2 };
const char* toString(Phase p);

/// Declared per-phase token demand of one rail.
struct PhaseDemand {
  int io = 1;
  int communication = 1;
  int computation = 0;
};

class ComputePool {
 public:
  explicit ComputePool(int total_tokens);

  int totalTokens() const { return total_; }
  /// (Re)declares a rail's demand. Not allowed while the rail holds a grant.
  void declare(int rail_id, PhaseDemand demand);
  /// Blocking acquire: returns the grant.
  int acquire(int rail_id, Phase phase);
  /// Non-blocking form: nullopt when acquire() would block.
  std::optional<int> tryAcquire(int rail_id, Phase phase);
  /// Phase exit.
  void release(int rail_id, Phase phase);

  /// Computation tokens currently granted (invariant: <= totalTokens()).
  int outstanding() const;
  /// Computation requests currently blocked in acquire().
  int waiting() const;
  /// The phase rail_id holds a grant for, if any.
  std::optional<Phase> held(int rail_id) const;
  /// Largest outstanding() ever observed.
  int peakOutstanding() const;

 private:
  struct Slot {
    PhaseDemand demand;
    std::optional<Phase> held;
    int grant = 0;
  };
  Slot& slotOf(int rail_id);
  int grantFor(const Slot& s, Phase phase) const;

  int total_;
  int outstanding_ = 0;
  int peak_ = 0;
  std::uint64_t next_ticket_ = 0;
  std::deque<std::uint64_t> queue_;  // FIFO of waiting computation tickets
  std::map<int, Slot> slots_;
  mutable std::mutex mu_;
  std::condition_variable cv_;
};

/// How the engine maps the pool onto concurrently launched rails.
enum class PoolMode : std::uint8_t {
  Off = 0,    // no arbitration: every rail launches its full grid at once
  Block = 1,  // SPEC semantics: a computation grant that does not fit waits
  Shrink = 2, // B200 extension: grant min(demand, free tokens); wait only at 0
};

/// One rail's computation-phase decision inside one op.
struct ComputeGrant {
  int rail_id = 0;
  int demand = 0;           // CTAs the rail would launch alone
  int grant = 0;            // CTAs it may launch
  std::vector<int> waits;   // rails whose computation-phase exit it waits for
};

/// Stream-order arbitration of one op: rails enter their
/// computation phase in the given (rail_id) order; a request that does not
/// fit releases the oldest holder and records a wait on it, which the engine
/// turns into cudaStreamWaitEvent on that holder's phase-exit event. Every
/// grant is released at the end. `pool` must be idle on entry and is idle on
/// return; the decisions are a pure function of (total, mode, demands).
std::vector<ComputeGrant> planComputeGrants(ComputePool& pool, PoolMode mode,
                                            const std::vector<std::pair<int, int>>& demands);

}  // namespace nezha
