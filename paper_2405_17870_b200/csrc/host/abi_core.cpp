// C-ABI wrappers of the core cost model (proj/include/nezha/core/math.hpp:9-17).
#include "nezha/collective.hpp"
#include "nezha/core/math.hpp"
#include "nezha_b200.h"

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

}  // extern "C"
