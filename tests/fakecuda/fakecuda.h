// TEST HARNESS ONLY (see fakecuda.cpp): the host emulations of the rail
// kernels, looked up by the kernel's demangled name at launch.
#pragma once

#include <cuda_runtime_api.h>

#include <functional>
#include <string>

namespace fakecuda {

// SM count the harness reports: small, so the host-side grid arithmetic runs
// with its real formulas on grids a host can emulate quickly.
constexpr int kSMs = 16;

// The launch as a stream operation (arguments copied now, as the driver
// does), or an empty function when the kernel has no emulation.
std::function<void()> emulatedKernel(const std::string& name, dim3 grid, dim3 block, void** args);

void countLaunch(const std::string& name);

// Resident CTAs per SM of a kernel (the harness's cudaOccupancy* answer, and
// the SIMT residency model's per-CTA cost): the B200 figures of the rail
// kernels — LL 1 (76-96 registers x 512 threads), the other 512-thread
// kernels 2 (<= 64 registers), small CTAs up to 32 per SM.
int occupancyOf(const std::string& name, int block_threads);

}  // namespace fakecuda
