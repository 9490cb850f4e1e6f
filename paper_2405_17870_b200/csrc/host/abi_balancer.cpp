// C-ABI of the planner driven op by op (nz_balancer_*): the same
// nezha::Balancer the engine runs, with the engine's multi-rank flush
// agreement supplied by the caller. Lets the N > 1 host logic (every rank
// applies identical flushes, so tables never diverge) be tested across
// processes without a GPU (tests/test_multirank_cpu.py, gloo world 2).
#include <cstring>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "nezha/balancer.hpp"
#include "nezha/collective.hpp"
#include "nezha/core/error.hpp"
#include "nezha/engine.hpp"
#include "nezha_b200.h"
#include "planner_trace.hpp"

struct nz_balancer {
  std::unique_ptr<nezha::Balancer> bal;
  nezha::Plan pending;
  bool has_pending = false;
  nz_agree_fn agree = nullptr;
  void* agree_ctx = nullptr;
};

namespace {

template <typename F>
int balGuard(F&& fn) {
  try {
    fn();
    return NZ_OK;
  } catch (const nezha::UnrecoverableError& e) {
    nz::setLastError(e.what());
    return NZ_ERR_UNRECOVERABLE;
  } catch (const std::invalid_argument& e) {
    nz::setLastError(e.what());
    return NZ_ERR_INVALID;
  } catch (const std::exception& e) {
    nz::setLastError(e.what());
    return NZ_ERR_SYSTEM;
  }
}

int copyOut(const std::string& s, char* out, size_t cap) {
  if (!out) return NZ_ERR_INVALID;
  if (s.size() + 1 > cap) return NZ_ERR_BUFFER;
  std::memcpy(out, s.c_str(), s.size() + 1);
  return NZ_OK;
}

}  // namespace

extern "C" {

int nz_balancer_create(const char* rails_toml, double tau, double eta, double sync_overhead_us, int window,
                       int demote_after, nz_balancer_t** out) {
  if (!rails_toml || !out) return NZ_ERR_INVALID;
  return balGuard([&] {
    auto specs = nezha::parseRailsToml(rails_toml);
    std::vector<nezha::RailProfile> profiles;
    for (auto& s : specs) {
      if (!s.has_profile) throw std::invalid_argument("nz_balancer_create: every rail needs a profile");
      profiles.push_back(s.profile);
    }
    nezha::BalancerConfig cfg;
    cfg.tau = tau;
    cfg.eta = eta;
    cfg.sync_overhead_us = sync_overhead_us;
    cfg.window = window;
    cfg.demote_after = demote_after;
    auto b = std::make_unique<nz_balancer>();
    b->bal = std::make_unique<nezha::Balancer>(profiles, cfg);
    nz_balancer* raw = b.get();
    b->bal->setAgreement([raw](int bucket, const std::vector<std::pair<int, nezha::Micros>>& mine) {
      if (!raw->agree) return mine;
      std::vector<int> ids;
      std::vector<double> us;
      for (const auto& [id, m] : mine) {
        ids.push_back(id);
        us.push_back(m);
      }
      if (raw->agree(raw->agree_ctx, bucket, static_cast<int>(ids.size()), ids.data(), us.data()) != 0) {
        throw std::runtime_error("agreement callback failed");
      }
      std::vector<std::pair<int, nezha::Micros>> out;
      for (size_t i = 0; i < ids.size(); ++i) out.emplace_back(ids[i], us[i]);
      return out;
    });
    *out = b.release();
  });
}

int nz_balancer_destroy(nz_balancer_t* b) {
  delete b;
  return NZ_OK;
}

int nz_balancer_set_agreement(nz_balancer_t* b, nz_agree_fn fn, void* ctx) {
  if (!b) return NZ_ERR_INVALID;
  b->agree = fn;
  b->agree_ctx = ctx;
  return NZ_OK;
}

int nz_balancer_allocate(nz_balancer_t* b, uint64_t bytes, char* plan_json, size_t cap) {
  if (!b) return NZ_ERR_INVALID;
  std::string js;
  const int rc = balGuard([&] {
    b->pending = b->bal->allocate(bytes);
    b->has_pending = true;
    js = nezha::planJson(0, bytes, b->pending);
  });
  return rc != NZ_OK ? rc : copyOut(js, plan_json, cap);
}

int nz_balancer_record(nz_balancer_t* b, int n, const int* rail_ids, const double* us, int* flushed) {
  if (!b || n < 0 || (n > 0 && (!rail_ids || !us))) return NZ_ERR_INVALID;
  return balGuard([&] {
    if (!b->has_pending) throw std::invalid_argument("nz_balancer_record: no allocated op");
    std::vector<std::pair<int, nezha::Micros>> lat;
    for (int i = 0; i < n; ++i) lat.emplace_back(rail_ids[i], us[i]);
    const auto ev = b->bal->recordOp(b->pending, lat);
    b->has_pending = false;
    if (flushed) *flushed = ev ? 1 : 0;
  });
}

int nz_balancer_table_json(nz_balancer_t* b, char* out, size_t cap) {
  if (!b) return NZ_ERR_INVALID;
  return copyOut(b->bal->tableJson(), out, cap);
}

}  // extern "C"
