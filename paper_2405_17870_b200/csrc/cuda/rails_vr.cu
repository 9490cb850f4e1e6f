// Loopback grids (nz_comm_init_loopback): every virtual rank of a one-GPU job
// in one launch, blockIdx.y = rank, each rank's arguments from the pack. The
// kernel bodies are the rails' own (kernels.cuh); only the argument selection
// differs. Kept in its own translation unit so the two instantiation sets
// compile in parallel.
#include <mutex>

#include "internal.h"
#include "kernels.cuh"

namespace nz {

// One grid's arguments for all 8 virtual ranks travel as kernel parameters:
// keep them inside the classic 4 KiB parameter space (no large-parameter
// launch path needed).
static_assert(sizeof(VPack<FoldArgs>) <= 4096, "fold pack exceeds 4 KiB of kernel parameters");
static_assert(sizeof(VPack<LLArgs>) <= 4096, "LL pack exceeds 4 KiB of kernel parameters");
static_assert(sizeof(VPack<BarrierKArgs>) <= 4096, "barrier pack exceeds 4 KiB of kernel parameters");

namespace {

template <typename DT, int N>
void launchVR(int kind, const void* pack, int grid, cudaStream_t st) {
  switch (kind) {
    case kLoopFold:
      fold_kernel_vr<DT, N, N><<<dim3(grid, N), kThreads, 0, st>>>(*static_cast<const VPack<FoldArgs>*>(pack));
      return;
    case kLoopLL:
      ll_kernel_vr<DT, N><<<dim3(grid, N), kThreads, 0, st>>>(*static_cast<const VPack<LLArgs>*>(pack));
      return;
    case kLoopBarrier:
      barrier_kernel_vr<N><<<dim3(1, N), 32, 0, st>>>(*static_cast<const VPack<BarrierKArgs>*>(pack));
      return;
  }
  fail(NZ_ERR_INVALID, "unknown loopback launch kind");
}

template <typename DT, int N>
int occupancyVR(int kind) {
  int occ = 0;
  switch (kind) {
    case kLoopFold:
      NZ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fold_kernel_vr<DT, N, N>, kThreads, 0));
      break;
    case kLoopLL:
      NZ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ll_kernel_vr<DT, N>, kThreads, 0));
      break;
    case kLoopBarrier:
      NZ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, barrier_kernel_vr<N>, 32, 0));
      break;
  }
  return occ;
}

template <int N>
void launchN(int kind, int dtype, const void* pack, int grid, cudaStream_t st) {
  if (dtype == NZ_F32) return launchVR<F32, N>(kind, pack, grid, st);
  if (dtype == NZ_BF16) return launchVR<BF16, N>(kind, pack, grid, st);
  return launchVR<I32, N>(kind, pack, grid, st);
}

template <int N>
int occupancyN(int kind, int dtype) {
  if (dtype == NZ_F32) return occupancyVR<F32, N>(kind);
  if (dtype == NZ_BF16) return occupancyVR<BF16, N>(kind);
  return occupancyVR<I32, N>(kind);
}

}  // namespace

void launchLoopGrid(int kind, int world, int dtype, const void* pack, int grid, cudaStream_t st) {
  switch (world) {
#define NZ_CASE(n) \
  case n: return launchN<n>(kind, dtype, pack, grid, st);
    NZ_CASE(2) NZ_CASE(3) NZ_CASE(4) NZ_CASE(5) NZ_CASE(6) NZ_CASE(7) NZ_CASE(8)
#undef NZ_CASE
  }
  fail(NZ_ERR_INVALID, "loopback world must be 2..8");
}

// Resident CTAs per SM of a loopback grid's kernel (cached per instance).
int loopOccupancy(int kind, int world, int dtype) {
  static std::mutex mu;
  static int cache[3][9][3] = {};
  if (kind < 0 || kind > 2 || world < 2 || world > 8 || dtype < 0 || dtype > 2) fail(NZ_ERR_INVALID, "bad loopback kind");
  std::lock_guard<std::mutex> lk(mu);
  int& v = cache[kind][world][dtype];
  if (v == 0) {
    switch (world) {
#define NZ_CASE(n) \
  case n: v = occupancyN<n>(kind, dtype); break;
      NZ_CASE(2) NZ_CASE(3) NZ_CASE(4) NZ_CASE(5) NZ_CASE(6) NZ_CASE(7) NZ_CASE(8)
#undef NZ_CASE
    }
  }
  return v;
}

}  // namespace nz
