// C-ABI of the ComputePool (include/nezha/compute_pool.hpp).
#include <stdexcept>
#include <utility>
#include <vector>

#include "nezha/compute_pool.hpp"
#include "nezha_b200.h"
#include "planner_trace.hpp"

struct nz_pool {
  explicit nz_pool(int total) : pool(total) {}
  nezha::ComputePool pool;
};

namespace {

template <typename F>
int poolGuard(F&& fn) {
  try {
    fn();
    return NZ_OK;
  } catch (const std::invalid_argument& e) {
    nz::setLastError(e.what());
    return NZ_ERR_INVALID;
  } catch (const std::exception& e) {
    nz::setLastError(e.what());
    return NZ_ERR_SYSTEM;
  }
}

nezha::Phase phaseOf(int p) {
  if (p < 0 || p > 2) throw std::invalid_argument("phase must be 0 (io), 1 (communication) or 2 (computation)");
  return static_cast<nezha::Phase>(p);
}

}  // namespace

extern "C" {

int nz_pool_create(int total_tokens, nz_pool_t** out) {
  if (!out) return NZ_ERR_INVALID;
  return poolGuard([&] { *out = new nz_pool(total_tokens); });
}

int nz_pool_destroy(nz_pool_t* pool) {
  delete pool;
  return NZ_OK;
}

int nz_pool_declare(nz_pool_t* pool, int rail_id, int io, int communication, int computation) {
  if (!pool) return NZ_ERR_INVALID;
  return poolGuard([&] { pool->pool.declare(rail_id, nezha::PhaseDemand{io, communication, computation}); });
}

int nz_pool_acquire(nz_pool_t* pool, int rail_id, int phase, int blocking, int* grant) {
  if (!pool || !grant) return NZ_ERR_INVALID;
  return poolGuard([&] {
    const nezha::Phase ph = phaseOf(phase);
    if (blocking) {
      *grant = pool->pool.acquire(rail_id, ph);
    } else {
      const auto g = pool->pool.tryAcquire(rail_id, ph);
      *grant = g ? *g : -1;
    }
  });
}

int nz_pool_release(nz_pool_t* pool, int rail_id, int phase) {
  if (!pool) return NZ_ERR_INVALID;
  return poolGuard([&] { pool->pool.release(rail_id, phaseOf(phase)); });
}

int nz_pool_outstanding(const nz_pool_t* pool) { return pool ? pool->pool.outstanding() : NZ_ERR_INVALID; }

int nz_pool_waiting(const nz_pool_t* pool) { return pool ? pool->pool.waiting() : NZ_ERR_INVALID; }

int nz_pool_plan(int total_tokens, int mode, int n, const int* rail_ids, const int* demands, int* grants,
                 uint32_t* wait_masks) {
  if (n < 0 || (n > 0 && (!rail_ids || !demands || !grants || !wait_masks)) || mode < 0 || mode > 2) {
    return NZ_ERR_INVALID;
  }
  return poolGuard([&] {
    std::vector<std::pair<int, int>> d;
    for (int i = 0; i < n; ++i) {
      if (rail_ids[i] < 0 || rail_ids[i] >= 32) throw std::invalid_argument("rail ids must be in [0, 32)");
      d.emplace_back(rail_ids[i], demands[i]);
    }
    nezha::ComputePool pool(total_tokens);
    const auto g = nezha::planComputeGrants(pool, static_cast<nezha::PoolMode>(mode), d);
    for (int i = 0; i < n; ++i) {
      grants[i] = g[i].grant;
      wait_masks[i] = 0;
      for (int w : g[i].waits) wait_masks[i] |= 1u << w;
    }
  });
}

}  // extern "C"
