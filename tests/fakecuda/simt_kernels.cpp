// TEST HARNESS ONLY (see simt.h): the product's kernel source compiled for
// the host and launched on fibers. Compiled with -DNZ_SIMT_HOST -include
// simt.h; the kernels below are csrc/cuda/kernels.cuh itself, not a copy.
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "kernels.cuh"

namespace nzsimt {
void run_grid(dim3 grid, dim3 block, const std::function<void()>& body, int occupancy);
uint64_t end_dilation();
}  // namespace nzsimt
namespace fakecuda {
int occupancyOf(const std::string& name, int block_threads);
}

using namespace nz;

namespace {

// Device end-barrier budgets assume device speed; the host runs a wave far
// slower, so they are stretched as for the protocol emulation.
void dilate(RailCtl& c) {
  if (c.end_timeout_ns) c.end_timeout_ns *= nzsimt::end_dilation();
}

void dilate(FoldArgs& a) { dilate(a.ctl); }
void dilate(LLArgs&) {}  // the LL waits use the watchdog budget, not the end budget
void dilate(BarrierKArgs& k) { dilate(k.ctl); }
void dilate(NvlsArgs& a) { dilate(a.f.ctl); }
template <typename A>
void dilate(VPack<A>& p) {
  for (auto& a : p.a) dilate(a);
}

// The launch's arguments are copied (and their end budgets stretched) once;
// every fiber of the grid then runs the kernel on that copy.
template <typename A, typename F>
std::function<void()> launch(const std::string& base, dim3 grid, dim3 block, void** args, F kernel) {
  auto a = std::make_shared<A>(*static_cast<const A*>(args[0]));
  dilate(*a);
  const int occ = fakecuda::occupancyOf(base, static_cast<int>(block.x * block.y * block.z));
  return [=] { nzsimt::run_grid(grid, block, [&] { kernel(*a); }, occ); };
}

template <typename DT>
std::function<void()> byN(const std::string& base, int N, int nd, dim3 grid, dim3 block, void** args) {
#define NZ_N(n)                                                                                          \
  if (N == n) {                                                                                          \
    if (base == "fold_kernel") {                                                                         \
      if (nd == 1) return launch<FoldArgs>(base, grid, block, args, [](const FoldArgs& a) { fold_kernel<DT, n, 1>(a); }); \
      if (nd == n) return launch<FoldArgs>(base, grid, block, args, [](const FoldArgs& a) { fold_kernel<DT, n, n>(a); }); \
    }                                                                                                    \
    if (base == "fold_kernel_vr" && nd == n)                                                             \
      return launch<VPack<FoldArgs>>(base, grid, block, args, [](const VPack<FoldArgs>& p) { fold_kernel_vr<DT, n, n>(p); });                                                                                                \
    if constexpr (n >= 2) {                                                                              \
      if (base == "nvls_kernel") return launch<NvlsArgs>(base, grid, block, args, [](const NvlsArgs& a) { nvls_kernel<DT, n>(a); }); \
      if (base == "ll_kernel") return launch<LLArgs>(base, grid, block, args, [](const LLArgs& a) { ll_kernel<DT, n>(a); }); \
      if (base == "ll_kernel_vr")                                                                        \
        return launch<VPack<LLArgs>>(base, grid, block, args, [](const VPack<LLArgs>& p) { ll_kernel_vr<DT, n>(p); }); \
    }                                                                                                    \
  }
  NZ_N(1) NZ_N(2) NZ_N(3) NZ_N(4) NZ_N(5) NZ_N(6) NZ_N(7) NZ_N(8)
#undef NZ_N
  return {};
}

template <int n>
std::function<void()> barrierN(const std::string& base, dim3 grid, dim3 block, void** args) {
  if (base == "barrier_kernel")
    return launch<BarrierKArgs>(base, grid, block, args, [](const BarrierKArgs& k) { barrier_kernel<n>(k); });
  if (base == "barrier_kernel_vr")
    return launch<VPack<BarrierKArgs>>(base, grid, block, args, [](const VPack<BarrierKArgs>& p) { barrier_kernel_vr<n>(p); });
  return {};
}

}  // namespace

namespace fakecuda {

// The kernel `base<targs...>` of kernels.cuh as a stream operation, or an
// empty function when the name is not one of them.
std::function<void()> simtKernel(const std::string& base, const std::vector<std::string>& targs, dim3 grid, dim3 block,
                                 void** args) {
  if (base == "copy_kernel") {
    struct CopyArgs {
      const char* src;
      char* dst;
      uint64_t lo, hi;
      FaultPost post;
      RailCtl ctl;
    };
    // copy_kernel has no end barrier: nothing to stretch.
    auto a = std::make_shared<CopyArgs>(CopyArgs{*static_cast<const char* const*>(args[0]),
                                                 *static_cast<char* const*>(args[1]),
                                                 *static_cast<const uint64_t*>(args[2]),
                                                 *static_cast<const uint64_t*>(args[3]),
                                                 *static_cast<const FaultPost*>(args[4]),
                                                 *static_cast<const RailCtl*>(args[5])});
    const int occ = fakecuda::occupancyOf(base, static_cast<int>(block.x * block.y * block.z));
    return [=] {
      nzsimt::run_grid(grid, block, [&] { copy_kernel(a->src, a->dst, a->lo, a->hi, a->post, a->ctl); }, occ);
    };
  }
  if ((base == "barrier_kernel" || base == "barrier_kernel_vr") && targs.size() == 1) {
    switch (std::stoi(targs[0])) {
      case 1: return barrierN<1>(base, grid, block, args);
      case 2: return barrierN<2>(base, grid, block, args);
      case 3: return barrierN<3>(base, grid, block, args);
      case 4: return barrierN<4>(base, grid, block, args);
      case 5: return barrierN<5>(base, grid, block, args);
      case 6: return barrierN<6>(base, grid, block, args);
      case 7: return barrierN<7>(base, grid, block, args);
      case 8: return barrierN<8>(base, grid, block, args);
    }
    return {};
  }
  if (targs.size() < 2) return {};
  const int N = std::stoi(targs[1]);
  const int nd = targs.size() > 2 ? std::stoi(targs[2]) : 0;
  const std::string& dt = targs[0];
  if (dt.find("BF16") != std::string::npos) return byN<BF16>(base, N, nd, grid, block, args);
  if (dt.find("I32") != std::string::npos) return byN<I32>(base, N, nd, grid, block, args);
  if (dt.find("F32") != std::string::npos) return byN<F32>(base, N, nd, grid, block, args);
  return {};
}

}  // namespace fakecuda
