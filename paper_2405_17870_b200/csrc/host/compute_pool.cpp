// ComputePool. Semantics pinned in
// include/nezha/compute_pool.hpp (P14); restated independently in
// oracle/compute_pool.py.
#include "nezha/compute_pool.hpp"

#include <algorithm>
#include <stdexcept>
#include <string>

namespace nezha {

const char* toString(Phase p) {
  switch (p) {
    case Phase::Io: return "io";
    case Phase::Communication: return "communication";
    case Phase::Computation: return "computation";
  }
  return "?";
}

ComputePool::ComputePool(int total_tokens) : total_(total_tokens) {
  if (total_tokens < 1) throw std::invalid_argument("ComputePool: total_tokens must be >= 1");
}

ComputePool::Slot& ComputePool::slotOf(int rail_id) {
  auto it = slots_.find(rail_id);
  if (it == slots_.end()) throw std::invalid_argument("ComputePool: rail " + std::to_string(rail_id) + " not declared");
  return it->second;
}

int ComputePool::grantFor(const Slot& s, Phase phase) const {
  if (phase != Phase::Computation) return 1;
  return std::min(s.demand.computation, total_);
}

void ComputePool::declare(int rail_id, PhaseDemand demand) {
  if (demand.io < 0 || demand.communication < 0 || demand.computation < 0) {
    throw std::invalid_argument("ComputePool: negative demand");
  }
  std::lock_guard<std::mutex> lk(mu_);
  auto it = slots_.find(rail_id);
  if (it != slots_.end() && it->second.held) {
    throw std::invalid_argument("ComputePool: cannot redeclare rail " + std::to_string(rail_id) + " while it holds a grant");
  }
  slots_[rail_id].demand = demand;
}

int ComputePool::acquire(int rail_id, Phase phase) {
  std::unique_lock<std::mutex> lk(mu_);
  Slot& s = slotOf(rail_id);
  if (s.held) throw std::invalid_argument("ComputePool: rail " + std::to_string(rail_id) + " already holds a grant");
  const int g = grantFor(s, phase);
  if (phase == Phase::Computation && g > 0) {
    const std::uint64_t ticket = next_ticket_++;
    queue_.push_back(ticket);
    cv_.wait(lk, [&] { return queue_.front() == ticket && outstanding_ + g <= total_; });
    queue_.pop_front();
    outstanding_ += g;
    peak_ = std::max(peak_, outstanding_);
    cv_.notify_all();  // the next head may fit too
  }
  s.held = phase;
  s.grant = g;
  return g;
}

std::optional<int> ComputePool::tryAcquire(int rail_id, Phase phase) {
  std::lock_guard<std::mutex> lk(mu_);
  Slot& s = slotOf(rail_id);
  if (s.held) throw std::invalid_argument("ComputePool: rail " + std::to_string(rail_id) + " already holds a grant");
  const int g = grantFor(s, phase);
  if (phase == Phase::Computation && g > 0) {
    if (!queue_.empty() || outstanding_ + g > total_) return std::nullopt;
    outstanding_ += g;
    peak_ = std::max(peak_, outstanding_);
  }
  s.held = phase;
  s.grant = g;
  return g;
}

void ComputePool::release(int rail_id, Phase phase) {
  std::lock_guard<std::mutex> lk(mu_);
  Slot& s = slotOf(rail_id);
  if (!s.held || *s.held != phase) {
    throw std::invalid_argument("ComputePool: rail " + std::to_string(rail_id) + " does not hold a " + toString(phase) +
                                " grant");
  }
  if (phase == Phase::Computation) outstanding_ -= s.grant;
  s.held.reset();
  s.grant = 0;
  cv_.notify_all();
}

int ComputePool::outstanding() const {
  std::lock_guard<std::mutex> lk(mu_);
  return outstanding_;
}

int ComputePool::waiting() const {
  std::lock_guard<std::mutex> lk(mu_);
  return static_cast<int>(queue_.size());
}

std::optional<Phase> ComputePool::held(int rail_id) const {
  std::lock_guard<std::mutex> lk(mu_);
  auto it = slots_.find(rail_id);
  return it == slots_.end() ? std::nullopt : it->second.held;
}

int ComputePool::peakOutstanding() const {
  std::lock_guard<std::mutex> lk(mu_);
  return peak_;
}

std::vector<ComputeGrant> planComputeGrants(ComputePool& pool, PoolMode mode,
                                            const std::vector<std::pair<int, int>>& demands) {
  std::vector<ComputeGrant> out;
  std::deque<int> holders;  // rail ids in grant order
  auto releaseOldest = [&](ComputeGrant& g) {
    const int h = holders.front();
    holders.pop_front();
    pool.release(h, Phase::Computation);
    g.waits.push_back(h);
  };
  for (const auto& [rid, demand] : demands) {
    ComputeGrant g;
    g.rail_id = rid;
    g.demand = demand;
    if (mode == PoolMode::Off) {
      g.grant = demand;
      out.push_back(g);
      continue;
    }
    int want = std::min(demand, pool.totalTokens());
    if (mode == PoolMode::Shrink && want > 0) {
      while (pool.outstanding() >= pool.totalTokens()) releaseOldest(g);
      want = std::min(want, pool.totalTokens() - pool.outstanding());
    }
    pool.declare(rid, PhaseDemand{1, 1, want});
    std::optional<int> got;
    while (!(got = pool.tryAcquire(rid, Phase::Computation))) releaseOldest(g);
    g.grant = *got;
    if (g.grant > 0) {
      holders.push_back(rid);
    } else {
      pool.release(rid, Phase::Computation);
    }
    out.push_back(g);
  }
  for (int h : holders) pool.release(h, Phase::Computation);
  return out;
}

}  // namespace nezha
