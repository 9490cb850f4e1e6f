// TEST HARNESS ONLY. Host SIMT stand-in for the CUDA device environment, so
// that the product's own kernel source (paper_2405_17870_b200/csrc/cuda/
// kernels.cuh) compiles with g++ and runs on CPU: every CUDA thread of a
// launch is a fiber, every fiber of a grid runs on the launching stream's
// worker thread (csrc: fakecuda.cpp), __syncthreads is a per-CTA barrier of
// fibers, and the cross-rank waits (ld.acquire polls, LL flag polls) yield to
// the other fibers. Force-included (-include simt.h) before kernels.cuh with
// NZ_SIMT_HOST defined; kernels.cuh then takes the host primitives below
// instead of its inline PTX.
//
// What it checks: the kernels' arithmetic, summation order, shard / run /
// vector walking, LL word packing, launch status and barrier protocol — the
// device source itself, not a restatement. What it cannot: memory ordering
// across GPUs, NVLink / multicast (no NVLS), timing, occupancy.
#pragma once

#include <vector_types.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <ctime>

#undef __device__
#undef __global__
#undef __shared__
#undef __forceinline__
#undef __grid_constant__
#define __device__
#define __global__
#define __forceinline__ inline
#define __launch_bounds__(...)
#define __grid_constant__
#define __restrict__

namespace nzsimt {

// The fiber running on this worker thread (set by the scheduler on every switch).
struct Cur {
  uint3 tid, bid;
  dim3 bdim, gdim;
};
extern thread_local Cur* g_cur;

void yield_spin();                   // a poll found nothing: let the other fibers run
void maybe_preempt();                // schedule fuzzing at data accesses (FAKECUDA_SIMT_PREEMPT)
void sync_cta();                     // __syncthreads
int sync_cta_or(int v);              // __syncthreads_or
void* shared_slot(const void* key, size_t bytes);  // this CTA's instance of a __shared__ variable

inline uint64_t host_globaltimer() {
  timespec ts;
  clock_gettime(CLOCK_REALTIME, &ts);
  return static_cast<uint64_t>(ts.tv_sec) * 1000000000ull + static_cast<uint64_t>(ts.tv_nsec);
}

}  // namespace nzsimt

#define threadIdx (nzsimt::g_cur->tid)
#define blockIdx (nzsimt::g_cur->bid)
#define blockDim (nzsimt::g_cur->bdim)
#define gridDim (nzsimt::g_cur->gdim)

// A __shared__ variable: one instance per CTA (keyed by a static per declaration).
#define NZ_SHARED(T, name)     \
  static const char name##_key_ = 0; \
  T& name = *static_cast<T*>(nzsimt::shared_slot(&name##_key_, sizeof(T)))

inline void __syncthreads() { nzsimt::sync_cta(); }
inline int __syncthreads_or(int v) { return nzsimt::sync_cta_or(v); }
inline void __threadfence_system() { std::atomic_thread_fence(std::memory_order_seq_cst); }
inline void __threadfence() { std::atomic_thread_fence(std::memory_order_seq_cst); }

inline unsigned atomicAdd(unsigned* p, unsigned v) { return __atomic_fetch_add(p, v, __ATOMIC_SEQ_CST); }
inline unsigned atomicExch(unsigned* p, unsigned v) { return __atomic_exchange_n(p, v, __ATOMIC_SEQ_CST); }
inline int atomicExch_system(int* p, int v) { return __atomic_exchange_n(p, v, __ATOMIC_SEQ_CST); }

inline float __uint_as_float(unsigned u) {
  float f;
  memcpy(&f, &u, 4);
  return f;
}
inline unsigned __float_as_uint(float f) {
  unsigned u;
  memcpy(&u, &f, 4);
  return u;
}
inline float4 make_float4(float x, float y, float z, float w) { return float4{x, y, z, w}; }
inline uint4 make_uint4(unsigned x, unsigned y, unsigned z, unsigned w) { return uint4{x, y, z, w}; }

// bf16: __float2bfloat16_rn (round to nearest even, NaN kept quiet) and its bits.
struct __nv_bfloat16 {
  unsigned short x;
};
inline __nv_bfloat16 __float2bfloat16_rn(float f) {
  uint32_t u = __float_as_uint(f);
  if ((u & 0x7fffffffu) > 0x7f800000u) return __nv_bfloat16{static_cast<unsigned short>((u >> 16) | 0x40u)};
  u += 0x7fffu + ((u >> 16) & 1u);
  return __nv_bfloat16{static_cast<unsigned short>(u >> 16)};
}
inline unsigned short __bfloat16_as_ushort(__nv_bfloat16 h) { return h.x; }

// ---- the primitives kernels.cuh writes in PTX -------------------------------
namespace nz {

inline uint64_t globaltimer() { return nzsimt::host_globaltimer(); }
inline void st_release_sys(uint32_t* p, uint32_t v) { __atomic_store_n(p, v, __ATOMIC_RELEASE); }
inline uint32_t ld_acquire_sys(const uint32_t* p) {
  const uint32_t v = __atomic_load_n(p, __ATOMIC_ACQUIRE);
  nzsimt::yield_spin();  // only cross-rank polls use it
  return v;
}
inline void fence_acq_rel_sys() { std::atomic_thread_fence(std::memory_order_acq_rel); }
inline uint4 ld_v4(const void* p) {
  nzsimt::maybe_preempt();
  uint4 r;
  memcpy(&r, p, 16);
  return r;
}
inline void st_v4(void* p, uint4 v) {
  nzsimt::maybe_preempt();
  memcpy(p, &v, 16);
}

// LL: one 16-byte store of two {data, flag} words; one 8-byte poll of a word.
inline void ll_push_pair(uint64_t* dst, uint32_t d0, uint32_t flag, uint32_t d1) {
  nzsimt::maybe_preempt();
  // The device store is one 16-byte transaction; the flags make a torn pair
  // harmless there, and here each 8-byte word is stored atomically.
  __atomic_store_n(dst, (static_cast<uint64_t>(flag) << 32) | d0, __ATOMIC_RELEASE);
  __atomic_store_n(dst + 1, (static_cast<uint64_t>(flag) << 32) | d1, __ATOMIC_RELEASE);
}
inline void ll_poll_word(const uint64_t* src, uint32_t* d, uint32_t* f) {
  const uint64_t w = __atomic_load_n(src, __ATOMIC_ACQUIRE);
  *d = static_cast<uint32_t>(w);
  *f = static_cast<uint32_t>(w >> 32);
  nzsimt::yield_spin();
}

// NVLS (K1): multimem accesses on a multicast window (fakecuda.cpp,
// FAKECUDA_MULTICAST=1). ld_reduce sums the members' 16 bytes at the same
// offset with the kernel's own dtype fold (fp32 / bf16 accumulated in fp32 and
// rounded once, as .acc::f32 / wrapping u32), in bind order — the switch's
// order is unspecified, which is why NVLS fp32 is held to a tolerance (P2).
// A misaligned or out-of-window access traps.
}  // namespace nz

extern "C" int fakecuda_mc_resolve(const void* addr, char** bases, int max);

namespace nz {

inline int mc_members(const char* p, char** bases) {
  if (reinterpret_cast<uintptr_t>(p) % 16 != 0) {
    fprintf(stderr, "[simt] misaligned 16-byte multimem access at %p\n", static_cast<const void*>(p));
    abort();
  }
  const int n = fakecuda_mc_resolve(p, bases, 8);
  if (n <= 0) {
    fprintf(stderr, "[simt] multimem access at %p outside a bound multicast window (%d)\n",
            static_cast<const void*>(p), n);
    abort();
  }
  return n;
}

template <typename DT>
inline uint4 mm_ld_reduce(const char* p) {
  nzsimt::maybe_preempt();
  char* m[8];
  const int n = mc_members(p, m);
  typename DT::Acc acc = DT::load(ld_v4(m[0]));
  for (int i = 1; i < n; ++i) DT::add(acc, ld_v4(m[i]));
  return DT::store(acc);
}

inline void mm_st(char* p, uint4 v) {
  nzsimt::maybe_preempt();
  char* m[8];
  const int n = mc_members(p, m);
  for (int i = 0; i < n; ++i) memcpy(m[i], &v, 16);
}

}  // namespace nz
