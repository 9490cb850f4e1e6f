// C-ABI wrappers of the core cost model (proj/include/nezha/core/math.hpp:9-17).
#include <stdexcept>
#include <vector>

#include "nezha/calibration.hpp"
#include "nezha/collective.hpp"
#include "nezha/core/math.hpp"
#include "nezha_b200.h"
#include "planner_trace.hpp"

extern "C" {

uint64_t nz_core_ring_volume(int node_count, uint64_t payload) {
  try {
    return nezha::ringVolume(node_count, payload);
  } catch (...) {
    return 0;
  }
}

int nz_core_bucket_of(uint64_t size) {
  if (size == 0) return NZ_ERR_INVALID;
  return nezha::bucketOf(size);
}

uint64_t nz_core_default_chunk_bytes(uint64_t seg_len, int world, int algorithm) {
  try {
    return nezha::defaultChunkBytes(seg_len, world,
                                    algorithm == NZ_ALGO_RING ? nezha::Algorithm::Ring : nezha::Algorithm::RingChunked);
  } catch (...) {
    return 0;
  }
}

int nz_core_calibrate(const uint64_t* sizes, const double* lat_us, int n, double* t_setup_us, double* bandwidth_bps,
                      int* interpolated, double* max_rel_residual) {
  if (!sizes || !lat_us || !t_setup_us || !bandwidth_bps || !interpolated || !max_rel_residual || n < 0) {
    return NZ_ERR_INVALID;
  }
  try {
    std::vector<std::pair<nezha::Bytes, nezha::Micros>> s;
    for (int i = 0; i < n; ++i) s.emplace_back(sizes[i], lat_us[i]);
    const auto c = nezha::calibrate(0, nezha::ProtocolKind::Custom, s);
    *t_setup_us = c.profile.t_setup_us;
    *bandwidth_bps = c.profile.bandwidth_bps;
    *interpolated = c.interpolated ? 1 : 0;
    *max_rel_residual = c.max_rel_residual;
    return NZ_OK;
  } catch (const std::exception& e) {
    nz::setLastError(e.what());
    return NZ_ERR_INVALID;
  }
}

}  // extern "C"
