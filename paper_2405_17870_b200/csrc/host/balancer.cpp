// Balancer: Eqs. 3-8, the AllocationTable and the Timer windows
// (PAPER.md:416-438). Pinned choices are DESIGN.md P3-P8,
// P11, P12; oracle/planner.py restates them line for line.
#include "nezha/balancer.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <sstream>
#include <stdexcept>

#include "nezha/core/error.hpp"
#include "nezha/core/math.hpp"

namespace nezha {

std::string formatDouble(double v) {
  char buf[40];
  std::snprintf(buf, sizeof(buf), "%.17g", v);
  return buf;
}

void BalancerConfig::validate() const {
  if (!(tau > 1.0)) throw std::invalid_argument("BalancerConfig: tau must be > 1");
  if (!(eta > 0.0 && eta < 1.0)) throw std::invalid_argument("BalancerConfig: eta must be in (0, 1)");
  if (window < 1) throw std::invalid_argument("BalancerConfig: window must be >= 1");
  if (max_iters < 0) throw std::invalid_argument("BalancerConfig: max_iters must be >= 0");
  if (!(convergence_eps >= 0.0)) throw std::invalid_argument("BalancerConfig: convergence_eps must be >= 0");
  if (probe_lo < 2 || probe_hi <= probe_lo) throw std::invalid_argument("BalancerConfig: bad probe range");
}

// ------------------------------------------------------------------ Eq. 3-8 --

std::vector<Bytes> splitLengths(const std::vector<double>& alpha, Bytes S) {
  std::vector<Bytes> len(alpha.size(), 0);
  int last = -1;
  for (size_t i = 0; i < alpha.size(); ++i)
    if (alpha[i] > 0) last = static_cast<int>(i);
  if (last < 0) throw std::invalid_argument("splitLengths: no rail has a positive share");
  Bytes used = 0;
  for (int i = 0; i < last; ++i) {
    if (!(alpha[i] > 0)) continue;
    Bytes l = static_cast<Bytes>(alpha[i] * static_cast<double>(S)) & ~Bytes{3};
    if (l > S - used) l = (S - used) & ~Bytes{3};
    len[i] = l;
    used += l;
  }
  len[last] = S - used;
  return len;
}

double efficiencyRatio(const std::vector<RailProfile>& rails, const std::vector<double>& alpha, Bytes S) {
  if (rails.size() != alpha.size()) throw std::invalid_argument("efficiencyRatio: size mismatch");
  const auto len = splitLengths(alpha, S);
  std::vector<double> thr;
  for (size_t i = 0; i < rails.size(); ++i)
    if (len[i] > 0) thr.push_back(realTimeThroughput(rails[i], len[i]));
  if (thr.size() < 2) return 1.0;
  std::sort(thr.begin(), thr.end(), [](double a, double b) { return a > b; });
  if (!(thr[1] > 0)) throw DegenerateProfileError("efficiencyRatio: zero-throughput rail");
  return thr[0] / thr[1];
}

std::pair<Micros, int> coldLatency(const std::vector<RailProfile>& rails, Bytes S) {
  if (rails.empty()) throw std::invalid_argument("coldLatency: no rails");
  int best = 0;
  Micros t = rails[0].messageLatency(S);
  for (size_t i = 1; i < rails.size(); ++i) {
    const Micros ti = rails[i].messageLatency(S);
    if (ti < t) {
      t = ti;
      best = static_cast<int>(i);
    }
  }
  return {t, best};
}

Micros hotLatency(const std::vector<RailProfile>& rails, const std::vector<double>& alpha, Bytes S, Micros sync) {
  if (rails.size() != alpha.size()) throw std::invalid_argument("hotLatency: size mismatch");
  double sum = 0;
  for (double a : alpha) {
    if (a < 0) throw std::invalid_argument("hotLatency: alpha off the simplex");
    sum += a;
  }
  if (std::fabs(sum - 1.0) > 1e-9) throw std::invalid_argument("hotLatency: alpha off the simplex");
  const auto len = splitLengths(alpha, S);
  Micros worst = 0;
  for (size_t i = 0; i < rails.size(); ++i)
    if (len[i] > 0) worst = std::max(worst, rails[i].messageLatency(len[i]));
  return worst + sync;
}

std::vector<double> initCoefficients(const std::vector<Micros>& T) {
  if (T.empty()) throw std::invalid_argument("initCoefficients: no rails");
  for (Micros t : T)
    if (!(t > 0)) throw std::invalid_argument("initCoefficients: invalid telemetry (T_i <= 0)");
  const size_t R = T.size();
  if (R == 1) return {1.0};
  double total = 0;
  for (Micros t : T) total += t;
  std::vector<double> a(R);
  for (size_t i = 0; i < R; ++i) a[i] = (total - T[i]) / (total * static_cast<double>(R - 1));
  return a;
}

std::vector<double> updateCoefficients(const std::vector<double>& alpha, const std::vector<Micros>& T, double eta,
                                       double eps, bool* converged) {
  if (alpha.size() != T.size()) throw std::invalid_argument("updateCoefficients: size mismatch");
  std::vector<size_t> part;
  for (size_t i = 0; i < alpha.size(); ++i)
    if (alpha[i] > 0) part.push_back(i);
  if (part.size() < 2) {
    if (converged) *converged = true;
    return alpha;
  }
  size_t m = part[0];
  Micros tmax = T[m], tmin = T[m], tsum = 0;
  for (size_t i : part) {
    if (T[i] > tmax) {
      tmax = T[i];
      m = i;
    }
    tmin = std::min(tmin, T[i]);
    tsum += T[i];
  }
  if (!(tmax > 0)) throw std::invalid_argument("updateCoefficients: invalid telemetry");
  if (tmax - tmin <= eps * tmax) {
    if (converged) *converged = true;
    return alpha;
  }
  const double tbar = tsum / static_cast<double>(part.size());
  const double excess = (tmax - tbar) / tmax;
  const double step = 0.5 * eta * excess;
  double slack_sum = 0;
  for (size_t i : part)
    if (i != m) slack_sum += tmax - T[i];
  std::vector<double> next = alpha;
  next[m] = alpha[m] - step;
  for (size_t i : part)
    if (i != m) next[i] = alpha[i] + step * ((tmax - T[i]) / slack_sum);
  double total = 0;
  for (double& a : next) {
    if (a < 0) a = 0;
    total += a;
  }
  for (double& a : next) a = a / total;
  if (converged) *converged = false;
  return next;
}

Bytes findThreshold(const std::function<double(Bytes)>& hot_minus_cold, Bytes lo, Bytes hi) {
  if (hot_minus_cold(hi) >= 0) return kNoThreshold;
  if (hot_minus_cold(lo) < 0) return lo - 1;
  Bytes a = lo, b = hi;  // f(a) >= 0 > f(b)
  while (b - a > 1) {
    const double mid = 0.5 * (std::log2(static_cast<double>(a)) + std::log2(static_cast<double>(b)));
    Bytes m = static_cast<Bytes>(std::floor(std::exp2(mid) + 0.5));
    if (m <= a) m = a + 1;
    if (m >= b) m = b - 1;
    if (hot_minus_cold(m) >= 0)
      a = m;
    else
      b = m;
  }
  return a;
}

// ------------------------------------------------------------ LatencyWindow --

std::optional<Micros> LatencyWindow::record(Micros sample) {
  samples_.push_back(sample);
  if (static_cast<int>(samples_.size()) < capacity_) return std::nullopt;
  return drain();
}

std::optional<Micros> LatencyWindow::drain() {
  if (samples_.empty()) return std::nullopt;
  double acc = 0;
  for (Micros s : samples_) acc += s;
  const Micros mean = acc / static_cast<double>(samples_.size());
  samples_.clear();
  return mean;
}

// ----------------------------------------------------------------- Balancer --

Balancer::Balancer(std::vector<RailProfile> rails, BalancerConfig cfg) : rails_(std::move(rails)), cfg_(cfg) {
  cfg_.validate();
  if (rails_.empty()) throw std::invalid_argument("Balancer: no rails");
  std::sort(rails_.begin(), rails_.end(), [](const RailProfile& a, const RailProfile& b) { return a.rail_id < b.rail_id; });
  for (size_t i = 0; i < rails_.size(); ++i) {
    rails_[i].validate();
    if (i && rails_[i].rail_id == rails_[i - 1].rail_id) throw std::invalid_argument("Balancer: duplicate rail_id");
  }
  healthy_.assign(rails_.size(), true);
  rebuild();
}

int Balancer::railIndex(int rail_id) const {
  for (size_t i = 0; i < rails_.size(); ++i)
    if (rails_[i].rail_id == rail_id) return static_cast<int>(i);
  throw std::invalid_argument("unknown rail " + std::to_string(rail_id));
}

bool Balancer::healthy(int rail_id) const { return healthy_[railIndex(rail_id)]; }

int Balancer::clampBucket(Bytes S) {
  const int k = bucketOf(S);
  return std::min(std::max(k, kMinBucket), kMaxBucket);
}

std::vector<RailProfile> Balancer::healthyProfiles(std::vector<int>* idx, bool concurrent) const {
  const auto& src = concurrent && !concurrent_.empty() ? concurrent_ : rails_;
  std::vector<RailProfile> out;
  for (size_t i = 0; i < rails_.size(); ++i) {
    if (!healthy_[i]) continue;
    out.push_back(src[i]);
    if (idx) idx->push_back(static_cast<int>(i));
  }
  return out;
}

std::vector<double> Balancer::restrictToHealthy(std::vector<double> a) const {
  a.resize(rails_.size(), 0.0);
  double total = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    if (!healthy_[i] || a[i] < 0) a[i] = 0;
    total += a[i];
  }
  if (total > 0) {
    for (double& x : a) x = x / total;
    return a;
  }
  int h = 0;
  for (bool ok : healthy_) h += ok ? 1 : 0;
  for (size_t i = 0; i < a.size(); ++i) a[i] = healthy_[i] ? 1.0 / h : 0.0;
  return a;
}

// P11: Eq. 8 applied to the calibrated model's uniform-split latencies.
std::vector<double> Balancer::modelAlpha(int bucket) const {
  // Depends only on the profiles and the healthy set: cached per bucket.
  std::vector<bool> key = healthy_;
  if (key != model_cache_healthy_ || model_cache_version_ != profile_version_) {
    model_cache_.clear();
    model_cache_healthy_ = key;
    model_cache_version_ = profile_version_;
  }
  auto it = model_cache_.find(bucket);
  if (it != model_cache_.end()) return it->second;
  auto a = computeModelAlpha(bucket);
  model_cache_[bucket] = a;
  return a;
}

std::vector<double> Balancer::computeModelAlpha(int bucket) const {
  std::vector<int> idx;
  const auto hp = healthyProfiles(&idx, /*concurrent=*/true);
  std::vector<double> a(rails_.size(), 0.0);
  const Bytes S = bucketFloor(bucket);
  const Bytes share = std::max<Bytes>(S / hp.size(), 1);
  std::vector<Micros> T;
  for (const auto& p : hp) T.push_back(p.messageLatency(share));
  std::vector<double> ah = initCoefficients(T);
  // P11: then the same Eq. 7 descent the Timer would run, on the model's own
  // latencies (up to max_iters virtual flushes), so an unmeasured bucket is
  // judged hot or cold on a converged split, not on the Eq. 8 first guess.
  for (int it = 0; it < cfg_.max_iters && hp.size() > 1; ++it) {
    const auto len = splitLengths(ah, S);
    std::vector<Micros> t(hp.size(), 0.0);
    for (size_t j = 0; j < hp.size(); ++j)
      if (len[j] > 0) t[j] = hp[j].messageLatency(len[j]);
    bool conv = false;
    ah = updateCoefficients(ah, t, cfg_.eta, cfg_.convergence_eps, &conv);
    if (conv) break;
  }
  for (size_t j = 0; j < idx.size(); ++j) a[idx[j]] = ah[j];
  return a;
}

// Eq. 6's f(S): hot from the concurrent profiles (rails share the links),
// cold from the isolated ones.
double Balancer::hotMinusCold(Bytes S) const {
  std::vector<int> idx;
  const auto hp = healthyProfiles(&idx, /*concurrent=*/true);
  const auto cp = healthyProfiles(nullptr, /*concurrent=*/false);
  const auto& e = table_.buckets.at(clampBucket(S));
  std::vector<double> ah;
  for (int i : idx) ah.push_back(e.alpha[i]);
  return hotLatency(hp, ah, S, cfg_.sync_overhead_us) - coldLatency(cp, S).first;
}

void Balancer::rebuild() {
  std::vector<int> idx;
  const auto hp = healthyProfiles(&idx);
  if (hp.empty()) {
    table_.threshold = kNoThreshold;
    for (auto& [k, e] : table_.buckets) e.hot = false;
    ++table_.epoch;
    return;
  }
  struct Before {
    bool hot;
    int best;
    std::vector<bool> part;
  };
  std::map<int, Before> before;
  for (auto& [k, e] : table_.buckets) {
    std::vector<bool> part;
    for (double a : e.alpha) part.push_back(a > 0);
    before[k] = {e.hot, e.best, part};
  }
  // Pass 1: alpha of every bucket (own if measured, else nearest measured, else model).
  std::vector<int> measured;
  for (auto& [k, e] : table_.buckets)
    if (e.measured) measured.push_back(k);
  for (int k = kMinBucket; k <= kMaxBucket; ++k) {
    BucketEntry& e = table_.buckets[k];
    if (e.measured) {
      e.alpha = restrictToHealthy(e.alpha);
      continue;
    }
    if (!measured.empty()) {
      int nearest = measured[0];
      for (int m : measured)
        if (std::abs(m - k) < std::abs(nearest - k)) nearest = m;  // ties keep the smaller bucket
      e.alpha = restrictToHealthy(table_.buckets[nearest].alpha);
    } else {
      e.alpha = modelAlpha(k);
    }
  }
  // Pass 2: Eq. 6 threshold, then states.
  table_.threshold = hp.size() >= 2 ? findThreshold([this](Bytes S) { return hotMinusCold(S); }, cfg_.probe_lo, cfg_.probe_hi)
                                    : kNoThreshold;
  for (int k = kMinBucket; k <= kMaxBucket; ++k) {
    BucketEntry& e = table_.buckets[k];
    e.best = idx[coldLatency(hp, bucketFloor(k)).second];
    e.hot = hp.size() >= 2 && !e.demoted && table_.threshold != kNoThreshold && bucketFloor(k) > table_.threshold;
    std::vector<bool> part;
    for (double a : e.alpha) part.push_back(a > 0);
    auto it = before.find(k);
    const bool changed = it == before.end() || it->second.hot != e.hot || it->second.best != e.best ||
                         (e.hot && it->second.part != part);
    if (changed) windows_.erase(k);
  }
  ++table_.epoch;
}

Plan Balancer::allocate(Bytes S) const {
  if (S == 0) throw std::invalid_argument("allocate: payload must be positive");
  Plan p;
  p.bucket = clampBucket(S);
  int h = 0;
  for (bool ok : healthy_) h += ok ? 1 : 0;
  if (h == 0) throw UnrecoverableError("allocate: no healthy rail left");
  const BucketEntry& e = table_.buckets.at(p.bucket);
  if (e.hot) {
    std::vector<int> idx;
    const auto hp = healthyProfiles(&idx, /*concurrent=*/true);
    std::vector<double> ah;
    for (int i : idx) ah.push_back(e.alpha[i]);
    p.rho = efficiencyRatio(hp, ah, S);
    if (p.rho > cfg_.tau) {
      p.gated = true;
    } else {
      p.hot = true;
      const auto len = splitLengths(e.alpha, S);
      Bytes off = 0;
      for (size_t i = 0; i < rails_.size(); ++i) {
        if (len[i] == 0) continue;
        p.segments.push_back({rails_[i].rail_id, Segment{off, len[i]}});
        off += len[i];
      }
      return p;
    }
  }
  p.segments.push_back({rails_[e.best].rail_id, Segment{0, S}});
  return p;
}

std::optional<FlushEvent> Balancer::recordOp(const Plan& plan, const std::vector<std::pair<int, Micros>>& lat) {
  if (plan.gated) return std::nullopt;  // gated ops sample neither mode of a hot bucket
  auto& wins = windows_[plan.bucket];
  if (wins.empty()) {
    for (size_t i = 0; i < rails_.size(); ++i) wins.emplace_back(rails_[i].rail_id, plan.bucket, cfg_.window);
  }
  std::optional<FlushEvent> ev;
  std::vector<std::pair<int, Micros>> means;
  for (const auto& [rail_id, us] : lat) {
    auto m = wins[railIndex(rail_id)].record(us);
    if (m) means.emplace_back(rail_id, *m);
  }
  if (means.empty()) return std::nullopt;
  // A full window flushes every rail of the bucket that holds samples (a
  // rail that sat out some ops of the window contributes the mean it has).
  for (auto& w : wins) {
    auto m = w.drain();
    if (m) means.emplace_back(w.railId(), *m);
  }
  std::sort(means.begin(), means.end(), [](auto& a, auto& b) { return a.first < b.first; });
  windows_.erase(plan.bucket);
  if (agree_) means = agree_(plan.bucket, means);
  FlushEvent fe;
  fe.bucket = plan.bucket;
  fe.means = means;
  applyFlush(plan.bucket, means);
  ev = fe;
  return ev;
}

void Balancer::applyFlush(int bucket, const std::vector<std::pair<int, Micros>>& means) {
  BucketEntry& e = table_.buckets[bucket];
  Micros worst = 0;
  for (auto& [id, m] : means) worst = std::max(worst, m);
  if (e.hot) {
    std::vector<Micros> T(rails_.size(), 0.0);
    for (auto& [id, m] : means) T[railIndex(id)] = m;
    if (e.iters < cfg_.max_iters) {
      bool conv = false;
      std::vector<double> participating = e.alpha;
      for (size_t i = 0; i < participating.size(); ++i)
        if (T[i] <= 0) participating[i] = 0;  // a rail without samples cannot be stepped
      e.alpha = restrictToHealthy(updateCoefficients(restrictToHealthy(participating), T, cfg_.eta,
                                                     cfg_.convergence_eps, &conv));
      e.converged = conv;
      e.iters += 1;
    }
    e.measured = true;
    e.last_hot_us = worst;
    if (cfg_.demote_after > 0 && e.iters >= cfg_.demote_after) {
      std::vector<int> idx;
      const auto hp = healthyProfiles(&idx);
      if (worst >= coldLatency(hp, bucketFloor(bucket)).first) e.demoted = true;
    }
  } else {
    e.last_cold_us = worst;
  }
  rebuild();
}

void Balancer::markFailed(int rail_id) {
  const int i = railIndex(rail_id);
  if (!healthy_[i]) return;
  for (auto& [k, e] : table_.buckets) saved_alpha_[k] = e.alpha;
  healthy_[i] = false;
  windows_.clear();
  rebuild();
}

void Balancer::readmit(int rail_id) {
  const int i = railIndex(rail_id);
  if (healthy_[i]) throw std::invalid_argument("readmit: rail " + std::to_string(rail_id) + " is not failed");
  healthy_[i] = true;
  for (auto& [k, a] : saved_alpha_) {
    auto it = table_.buckets.find(k);
    if (it != table_.buckets.end() && it->second.measured) it->second.alpha = a;
  }
  saved_alpha_.clear();
  windows_.clear();
  rebuild();
}

void Balancer::setProfiles(std::vector<RailProfile> rails) {
  std::sort(rails.begin(), rails.end(), [](const RailProfile& a, const RailProfile& b) { return a.rail_id < b.rail_id; });
  if (rails.size() != rails_.size()) throw std::invalid_argument("setProfiles: rail count changed");
  for (size_t i = 0; i < rails.size(); ++i) {
    rails[i].validate();
    if (rails[i].rail_id != rails_[i].rail_id) throw std::invalid_argument("setProfiles: rail ids changed");
  }
  rails_ = std::move(rails);
  ++profile_version_;
  rebuild();
}

void Balancer::setConcurrentProfiles(std::vector<RailProfile> rails) {
  std::sort(rails.begin(), rails.end(), [](const RailProfile& a, const RailProfile& b) { return a.rail_id < b.rail_id; });
  if (!rails.empty()) {
    if (rails.size() != rails_.size()) throw std::invalid_argument("setConcurrentProfiles: rail count mismatch");
    for (size_t i = 0; i < rails.size(); ++i) {
      rails[i].validate();
      if (rails[i].rail_id != rails_[i].rail_id) throw std::invalid_argument("setConcurrentProfiles: rail ids differ");
    }
  }
  concurrent_ = std::move(rails);
  ++profile_version_;
  rebuild();
}

void Balancer::setSyncOverhead(Micros us) {
  cfg_.sync_overhead_us = us;
  rebuild();
}

std::string Balancer::tableJson() const {
  std::ostringstream o;
  o << "{\"epoch\":" << table_.epoch << ",\"threshold\":";
  if (table_.threshold == kNoThreshold)
    o << "null";
  else
    o << table_.threshold;
  o << ",\"healthy\":[";
  bool first = true;
  for (size_t i = 0; i < rails_.size(); ++i) {
    if (!healthy_[i]) continue;
    o << (first ? "" : ",") << rails_[i].rail_id;
    first = false;
  }
  o << "],\"buckets\":[";
  first = true;
  for (const auto& [k, e] : table_.buckets) {
    o << (first ? "" : ",") << "{\"bucket\":" << k << ",\"hot\":" << (e.hot ? "true" : "false")
      << ",\"best\":" << rails_[e.best].rail_id << ",\"alpha\":[";
    for (size_t i = 0; i < e.alpha.size(); ++i) o << (i ? "," : "") << formatDouble(e.alpha[i]);
    o << "],\"measured\":" << (e.measured ? "true" : "false") << ",\"iters\":" << e.iters
      << ",\"converged\":" << (e.converged ? "true" : "false") << ",\"demoted\":" << (e.demoted ? "true" : "false")
      << "}";
    first = false;
  }
  o << "]}";
  return o.str();
}

}  // namespace nezha
