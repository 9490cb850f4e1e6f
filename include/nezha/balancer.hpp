// nezha/balancer.hpp — the Control Module's scheduler.
//
// Eqs. 3-8 of the paper as free functions, plus the Balancer that owns the
// AllocationTable (the paper's "data length table") and the Timer windows.
// The reference specifies but does not ship this module; every ambiguity is
// pinned in DESIGN.md (P3-P8, P11, P12) and restated independently by
// oracle/planner.py. The engine and nz_planner_run_trace drive this exact
// class, so the decisions the GPU engine takes are the ones the parity tests
// diff against the oracle.
#pragma once

#include <cstdint>
#include <functional>
#include <limits>
#include <map>
#include <optional>
#include <string>
#include <utility>
#include <vector>

#include "nezha/core/types.hpp"

namespace nezha {

inline constexpr Bytes kNoThreshold = std::numeric_limits<Bytes>::max();  // "+inf": always cold

struct BalancerConfig {
  double tau = 5.0;               // Eq. 3 gate
  double eta = 0.05;              // Eq. 7 step
  Micros sync_overhead_us = 0.0;  // additive multi-rail cost in Eq. 5
  double convergence_eps = 0.01;
  int max_iters = 100;
  int window = 100;               // Timer samples per flush
  int demote_after = 0;           // DESIGN.md P12 (0 = off)
  Bytes probe_lo = 4096;          // Eq. 6 bisection range (P5)
  Bytes probe_hi = Bytes{1} << 30;

  void validate() const;  // tau > 1, 0 < eta < 1, window >= 1
};

// P8: per-rail lengths of an S-byte payload under alpha. Rails with
// alpha_i > 0 participate in index order; each but the last gets
// round4down(alpha_i * S), the last participant the remainder.
std::vector<Bytes> splitLengths(const std::vector<double>& alpha, Bytes S);

// Eq. 3 (P3): throughput ratio of the two fastest participating rails at
// their split lengths, oriented >= 1; 1.0 with fewer than two participants.
// DegenerateProfileError when the slower of the two has zero throughput.
double efficiencyRatio(const std::vector<RailProfile>& rails, const std::vector<double>& alpha, Bytes S);

// Eq. 4: min_i messageLatency_i(S) and its index (ties -> lowest index).
std::pair<Micros, int> coldLatency(const std::vector<RailProfile>& rails, Bytes S);

// Eq. 5: max over participating rails of messageLatency_i(len_i) + sync.
// invalid_argument when alpha is off the simplex.
Micros hotLatency(const std::vector<RailProfile>& rails, const std::vector<double>& alpha, Bytes S, Micros sync);

// Eq. 8 with N = number of rails: (T - T_i) / (T (R - 1)).
std::vector<double> initCoefficients(const std::vector<Micros>& T);

// Eq. 7 (P4): projected subgradient step over the participating rails.
std::vector<double> updateCoefficients(const std::vector<double>& alpha, const std::vector<Micros>& T, double eta,
                                       double eps, bool* converged);

// Eq. 6 (P5): bisection in log2 space over [lo, hi] for the largest S with
// hot(S) - cold(S) >= 0 (cold still at least as fast). kNoThreshold when hot
// never wins at hi; lo - 1 when hot already wins at lo.
Bytes findThreshold(const std::function<double(Bytes)>& hot_minus_cold, Bytes lo, Bytes hi);

/// up to `capacity` samples; the capacity-th sample flushes
/// the arithmetic mean and resets the window.
class LatencyWindow {
 public:
  LatencyWindow(int rail_id = 0, int bucket = 0, int capacity = 100)
      : rail_id_(rail_id), bucket_(bucket), capacity_(capacity) {}
  std::optional<Micros> record(Micros sample);
  // Mean of whatever is held (nullopt when empty), then reset.
  std::optional<Micros> drain();
  void reset() { samples_.clear(); }
  int size() const { return static_cast<int>(samples_.size()); }
  int railId() const { return rail_id_; }
  int bucket() const { return bucket_; }

 private:
  int rail_id_;
  int bucket_;
  int capacity_;
  std::vector<Micros> samples_;
};

/// One row of the AllocationTable.
struct BucketEntry {
  bool hot = false;           // derived at every rebuild
  int best = 0;               // rail index of Cold(best)
  std::vector<double> alpha;  // per rail index; what a Hot op uses
  bool measured = false;      // alpha came from this bucket's own flushes
  bool probing = false;       // first window runs the uniform split (Eq. 8 precondition)
  int iters = 0;              // flushes applied
  bool converged = false;
  bool demoted = false;       // P12: sticky Cold after measured loss
  Micros last_hot_us = 0;     // last flushed max_i T_i (telemetry)
  Micros last_cold_us = 0;    // last flushed mean of the cold rail
};

struct AllocationTable {
  std::map<int, BucketEntry> buckets;
  Bytes threshold = kNoThreshold;
  std::uint64_t epoch = 0;  // bumped on every mutation (single writer)
};

struct RailSegment {
  int rail_id;
  Segment segment;
  bool operator==(const RailSegment&) const = default;
};

struct Plan {
  int bucket = 0;
  bool hot = false;
  double rho = 1.0;  // Eq. 3 at this op (1 when cold)
  bool gated = false;
  std::vector<RailSegment> segments;  // rail_id order, disjoint, covering [0, S)
};

struct FlushEvent {
  int bucket = 0;
  std::vector<std::pair<int, Micros>> means;  // (rail_id, mean) in rail order
};

class Balancer {
 public:
  static constexpr int kMinBucket = 0;
  static constexpr int kMaxBucket = 40;

  Balancer(std::vector<RailProfile> rails, BalancerConfig cfg);

  // SPEC.md:312-320.
  Plan allocate(Bytes S) const;

  // SPEC.md:321-328 for every rail of one finished op. Returns the flush when
  // this op completed the bucket's window; the table is already updated.
  std::optional<FlushEvent> recordOp(const Plan& plan, const std::vector<std::pair<int, Micros>>& rail_latency);

  // Health changes (faults module). Both rebuild the table.
  void markFailed(int rail_id);
  void readmit(int rail_id);  // "last converged alpha, renormalized"
  bool healthy(int rail_id) const;

  // Recompute threshold / states after a profile change (e.g. calibration).
  void setProfiles(std::vector<RailProfile> rails);
  // P13: profiles measured with every rail busy at once; they drive the hot
  // side (Eqs. 3, 5, 6, 8) while the isolated profiles drive Eq. 4. Rails on
  // one NVSwitch share links, so isolated numbers overstate the hot gain.
  void setConcurrentProfiles(std::vector<RailProfile> rails);
  const std::vector<RailProfile>& concurrentProfiles() const { return concurrent_; }
  void setSyncOverhead(Micros us);

  // Multi-rank agreement on a flush: maps this rank's per-rail window means
  // to the values every rank will apply (the engine: max over ranks). Unset
  // (single process, traces) = identity.
  using Agreement = std::function<std::vector<std::pair<int, Micros>>(int bucket,
                                                                     const std::vector<std::pair<int, Micros>>&)>;
  void setAgreement(Agreement fn) { agree_ = std::move(fn); }

  const AllocationTable& table() const { return table_; }
  const std::vector<RailProfile>& rails() const { return rails_; }
  const BalancerConfig& config() const { return cfg_; }
  int railIndex(int rail_id) const;
  static int clampBucket(Bytes S);
  std::string tableJson() const;

  // Warm restart: profiles, concurrent profiles, sync overhead
  // and every measured / demoted bucket as JSON; loadState restores them on a
  // balancer with the same rail ids (health is runtime state, not restored).
  std::string saveState() const;
  void loadState(const std::string& json);

 private:
  void rebuild();
  std::vector<double> modelAlpha(int bucket) const;
  std::vector<double> computeModelAlpha(int bucket) const;
  std::vector<double> restrictToHealthy(std::vector<double> a) const;
  std::vector<RailProfile> healthyProfiles(std::vector<int>* idx, bool concurrent = false) const;
  double hotMinusCold(Bytes S) const;
  void applyFlush(int bucket, const std::vector<std::pair<int, Micros>>& means);

  std::vector<RailProfile> rails_;  // sorted by rail_id
  // Latency of each rail while all rails run together (P13); empty = rails_.
  std::vector<RailProfile> concurrent_;
  BalancerConfig cfg_;
  std::vector<bool> healthy_;
  AllocationTable table_;
  std::map<int, std::vector<double>> saved_alpha_;  // alpha snapshot at the last failure
  std::map<int, std::vector<LatencyWindow>> windows_;  // bucket -> per rail index
  Agreement agree_;
  std::uint64_t profile_version_ = 0;  // bumped when rails_ / concurrent_ change
  mutable std::map<int, std::vector<double>> model_cache_;
  mutable std::vector<bool> model_cache_healthy_;
  mutable std::uint64_t model_cache_version_ = ~std::uint64_t{0};
};

std::string formatDouble(double v);  // "%.17g", shared by every JSON writer

}  // namespace nezha
