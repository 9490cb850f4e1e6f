// Device side of the three B200 rails (sm_100a).
//
//   K1 nvls_kernel   : multimem.ld_reduce over the NVSwitch multicast address
//                      of `in`, multimem.st of the sum to the multicast address
//                      of `out` (the "SHARP" rail: reduction inside the switch).
//   K2 fold_kernel<.., NDST=1> : copy-engine rail's local reduce of staged
//                      peer shards (the "GLEX/RDMA" rail's SM step).
//   K3 fold_kernel<.., NDST=N> : SM rail, 128-bit peer loads from every rank,
//                      in-register fold in ring order, 128-bit peer stores of
//                      the sum to every rank (the "TCP" rail).
//   K4 barrier_kernel: the copy-engine rail's start / end barriers.
//   K5 ll_kernel     : SM rail one-shot for small payloads (flag-tagged words).
//   K6 copy_kernel   : N = 1 (the identity allreduce).
//
// Summation order (P1): an element of ring block b of its chunk is
// folded x_b + x_{b+1} + ... + x_{b-1}. A CTA walks its contiguous share of
// the shard run by run (a run = one ring block of one chunk), so the
// rotation is resolved once per run, not per vector; the rare 16-byte vector
// that straddles a run boundary is folded element by element.
//
// Failure handling. Every rail launch carries a RailCtl: the
// last CTA to retire on a rank publishes the launch's progress and, when the
// launch completes an op entry, writes the entry's tag into the rail's gate
// word (the callers' streams wait on it with cuStreamWaitValue32). A launch
// that fails — a cross-rank wait timed out or was aborted by the host
// monitor, or an injected dead link — writes nothing, marks the rail failed
// on this rank (sticky: later launches exit at once without touching peers)
// and stamps the host-mapped status record the monitor reads.
//
// Loopback (nz_comm_init_loopback): the *_vr kernels run every virtual rank
// of a one-GPU job in one grid, blockIdx.y = rank, each with its own
// arguments; the cross-rank waits are then between CTAs of that grid, which
// the host sizes to be co-resident.
#pragma once

#ifndef NZ_SIMT_HOST
#include <cuda_bf16.h>
#endif
#include <stdint.h>

#include "kernel_args.h"
#include "nezha_b200.h"

namespace nz {


// ------------------------------------------------------------ primitives --
// NZ_SIMT_HOST: the CPU test harness (tests/fakecuda/simt.h) supplies host
// versions of these and runs this file's kernels on host fibers.
#ifndef NZ_SIMT_HOST
#define NZ_SHARED(T, name) __shared__ T name

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

__device__ __forceinline__ uint4 ld_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p)
               : "memory");
  return r;
}

__device__ __forceinline__ void st_v4(void* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// LL (K5): one 16-byte store of two {data, flag} words to a peer's slot; one
// 8-byte poll of a {data, flag} word in this rank's slots.
__device__ __forceinline__ void ll_push_pair(uint64_t* dst, uint32_t d0, uint32_t flag, uint32_t d1) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(dst), "r"(d0), "r"(flag), "r"(d1), "r"(flag)
               : "memory");
}

__device__ __forceinline__ void ll_poll_word(const uint64_t* src, uint32_t* d, uint32_t* f) {
  asm volatile("ld.volatile.global.v2.u32 {%0,%1}, [%2];" : "=r"(*d), "=r"(*f) : "l"(src) : "memory");
}
#endif  // NZ_SIMT_HOST

// ------------------------------------------------------ launch status ------
__device__ __forceinline__ uint32_t seq_read(const uint32_t* seq) {
  return *reinterpret_cast<const volatile uint32_t*>(seq);
}

// Graph-safe rails (NZ_RAIL_FLAG_GRAPH_SAFE) take their barrier epochs and LL
// flags from the device launch counter (advanced by the last CTA of every
// launch in rail_exit) instead of kernel arguments, so a launch captured in a
// CUDA graph stays valid on every replay. A rail's launches are ordered, so
// the next one sees the advanced value.
__device__ __forceinline__ uint32_t op_epoch(const BarrierArgs& b) {
  return b.seq ? 2u * seq_read(b.seq) + 1u : b.epoch;
}

// Entry of every CTA: false (uniformly over the CTA) when the rail failed on
// this rank in an EARLIER launch, so this launch must not touch peers. The
// sticky word holds (launch counter + 1) of the failing launch; the counter
// only moves when a launch retires, so a failure inside the current launch
// does not stop its other CTAs from arriving at the start barrier. CTA 0
// stamps the start for the monitor's heartbeat clock.
__device__ __forceinline__ bool rail_enter(const RailCtl& c) {
  if (!c.dev) return true;
  int dead = 0;
  if (threadIdx.x == 0) {
    const uint32_t sticky = *reinterpret_cast<const volatile uint32_t*>(c.dev + kCtlSticky);
    const uint32_t seq = *reinterpret_cast<const volatile uint32_t*>(c.dev + kCtlSeq);
    dead = sticky != 0 && static_cast<int32_t>(sticky - 1u - seq) < 0;
    if (c.host && blockIdx.x == 0) {
      volatile nz_rail_status_t* h = c.host;
      h->t_start_ns = globaltimer();
      h->start_tag = c.tag;
    }
  }
  return __syncthreads_or(dead) == 0;
}

// A cross-rank wait gave up (timeout or host abort): device-side detection time.
__device__ __forceinline__ void note_detect(const RailCtl* c, uint64_t now) {
  if (c && c->host) {
    volatile nz_rail_status_t* h = c->host;
    h->t_det_ns = now;
    h->det_tag = c->tag;
  }
}

// The injected dead link of this rank stops here.
__device__ __forceinline__ void note_stall(const RailCtl& c) {
  if (c.host && blockIdx.x == 0 && threadIdx.x == 0) {
    volatile nz_rail_status_t* h = c.host;
    h->t_fail_ns = globaltimer();
    h->fail_tag = c.tag;
  }
}

// The launch passed its start barrier: every rank is in, data moves from
// here on (the monitor's heartbeat clock runs from this point).
__device__ __forceinline__ void note_run(const RailCtl& c) {
  if (c.host && blockIdx.x == 0 && threadIdx.x == 0) {
    volatile nz_rail_status_t* h = c.host;
    h->t_run_ns = globaltimer();
    h->run_tag = c.tag;
  }
}

// Exit of every CTA (every thread calls it; `ok` is uniform over the CTA).
// The last CTA of the launch on this rank publishes the outcome.
__device__ __forceinline__ void rail_exit(const RailCtl& c, bool ok) {
  if (!c.dev) return;
  __syncthreads();
  if (threadIdx.x != 0) return;
  if (!ok) {
    atomicExch(c.dev + kCtlFailed, 1u);
    atomicExch(c.dev + kCtlSticky, *reinterpret_cast<const volatile uint32_t*>(c.dev + kCtlSeq) + 1u);
  }
  __threadfence_system();  // this CTA's stores (peer stores included) before it counts as retired
  if (atomicAdd(c.dev + kCtlRetired, 1u) != gridDim.x - 1) return;
  atomicExch(c.dev + kCtlRetired, 0u);
  const bool failed = atomicExch(c.dev + kCtlFailed, 0u) != 0;
  if (!failed) {
    volatile nz_rail_status_t* h = c.host;
    if (h && c.prog_chunk != ~0ull) {
      h->prog_chunk = c.prog_chunk;
      __threadfence_system();
      h->prog_tag = c.tag;
    }
    if (c.final_wave) {
      st_release_sys(c.dev + kCtlGate, c.tag);
      if (h) h->ok_tag = c.tag;
    }
    __threadfence_system();  // the mapped record is out before the launch counts as complete
  }
  atomicAdd(c.dev + kCtlSeq, 1u);
}

// Per-CTA barrier across ranks. Returns false (uniformly over the CTA) if a
// peer did not arrive within `timeout_ns` or the host aborted the rail, so
// the kernel exits instead of hanging the GPU. `publish` = this CTA wrote
// peer-visible data that must land before peers pass the barrier.
template <int N, bool kPublish>
__device__ __forceinline__ bool cta_barrier(const BarrierArgs& b, uint32_t epoch, int rank, uint64_t timeout_ns,
                                            const RailCtl* ctl) {
  NZ_SHARED(int, s_ok);
  if (threadIdx.x == 0) s_ok = 1;
  if (kPublish) fence_acq_rel_sys();
  __syncthreads();
  const int t = threadIdx.x;
  if (t < N) {
    st_release_sys(b.peer[t] + blockIdx.x * kDevMaxRanks + rank, epoch);
    const uint32_t* slot = b.local + blockIdx.x * kDevMaxRanks + t;
    uint64_t t0 = 0;
    int spins = 0;
    while (static_cast<int32_t>(ld_acquire_sys(slot) - epoch) < 0) {
      if (++spins == 64) {
        spins = 0;
        const uint64_t now = globaltimer();
        if (t0 == 0) {
          t0 = now;
        } else if (now - t0 > timeout_ns || (b.abort && *b.abort)) {
          if (b.watchdog) atomicExch_system(b.watchdog, 1);
          note_detect(ctl, now);
          s_ok = 0;
          break;
        }
      }
    }
  }
  __syncthreads();
  return s_ok != 0;
}

__device__ __forceinline__ void post_fault(const FaultPost& p) {
  if (p.rec && blockIdx.x == 0 && threadIdx.x == 0) {
    volatile nz_fault_record_t* r = p.rec;
    r->op_seq = p.op_seq;
    r->chunk = p.chunk;
    r->t_fail_ns = globaltimer();
    __threadfence_system();
    r->valid = 1;
  }
}

__device__ __forceinline__ uint64_t end_budget(const BarrierArgs& b, const RailCtl& c) {
  return c.end_timeout_ns ? c.end_timeout_ns : b.timeout_ns;
}

// ------------------------------------------------------------ dtype folds --
struct F32 {
  static constexpr int kElem = 4;
  using Acc = float4;
  __device__ static Acc load(uint4 v) { return make_float4(__uint_as_float(v.x), __uint_as_float(v.y), __uint_as_float(v.z), __uint_as_float(v.w)); }
  __device__ static void add(Acc& a, uint4 v) {
    a.x = a.x + __uint_as_float(v.x);
    a.y = a.y + __uint_as_float(v.y);
    a.z = a.z + __uint_as_float(v.z);
    a.w = a.w + __uint_as_float(v.w);
  }
  __device__ static uint4 store(const Acc& a) {
    return make_uint4(__float_as_uint(a.x), __float_as_uint(a.y), __float_as_uint(a.z), __float_as_uint(a.w));
  }
  using Scalar = float;
  __device__ static float sload(const char* p) { return *reinterpret_cast<const float*>(p); }
  __device__ static void sstore(char* p, float v) { *reinterpret_cast<float*>(p) = v; }
  __device__ static float sadd(float a, float b) { return a + b; }
};

struct BF16 {
  static constexpr int kElem = 2;
  struct Acc {
    float v[8];
  };
  __device__ static void unpack(uint32_t w, float& lo, float& hi) {
    lo = __uint_as_float(w << 16);
    hi = __uint_as_float(w & 0xffff0000u);
  }
  __device__ static Acc load(uint4 v) {
    Acc a;
    unpack(v.x, a.v[0], a.v[1]);
    unpack(v.y, a.v[2], a.v[3]);
    unpack(v.z, a.v[4], a.v[5]);
    unpack(v.w, a.v[6], a.v[7]);
    return a;
  }
  __device__ static void add(Acc& a, uint4 v) {
    Acc b = load(v);
#pragma unroll
    for (int i = 0; i < 8; ++i) a.v[i] = a.v[i] + b.v[i];
  }
  __device__ static uint32_t pack(float lo, float hi) {
    const uint32_t l = __bfloat16_as_ushort(__float2bfloat16_rn(lo));
    const uint32_t h = __bfloat16_as_ushort(__float2bfloat16_rn(hi));
    return l | (h << 16);
  }
  __device__ static uint4 store(const Acc& a) {
    return make_uint4(pack(a.v[0], a.v[1]), pack(a.v[2], a.v[3]), pack(a.v[4], a.v[5]), pack(a.v[6], a.v[7]));
  }
  using Scalar = float;
  __device__ static float sload(const char* p) {
    return __uint_as_float(static_cast<uint32_t>(*reinterpret_cast<const unsigned short*>(p)) << 16);
  }
  __device__ static void sstore(char* p, float v) {
    *reinterpret_cast<unsigned short*>(p) = __bfloat16_as_ushort(__float2bfloat16_rn(v));
  }
  __device__ static float sadd(float a, float b) { return a + b; }
};

struct I32 {
  static constexpr int kElem = 4;
  using Acc = uint4;
  __device__ static Acc load(uint4 v) { return v; }
  __device__ static void add(Acc& a, uint4 v) {
    a.x += v.x;
    a.y += v.y;
    a.z += v.z;
    a.w += v.w;
  }
  __device__ static uint4 store(const Acc& a) { return a; }
  using Scalar = uint32_t;
  __device__ static uint32_t sload(const char* p) { return *reinterpret_cast<const uint32_t*>(p); }
  __device__ static void sstore(char* p, uint32_t v) { *reinterpret_cast<uint32_t*>(p) = v; }
  __device__ static uint32_t sadd(uint32_t a, uint32_t b) { return a + b; }
};

// a / b through the 32-bit divider when both fit (always for segments of at
// most 1 GiB, split_oversized): the same quotient without a call to the 64-bit
// division subroutine, whose caller-saved registers were the kernels' spills.
__device__ __forceinline__ uint64_t udiv(uint64_t a, uint64_t b) {
  if (((a | b) >> 32) == 0) return static_cast<uint32_t>(a) / static_cast<uint32_t>(b);
  return a / b;
}

// Ring block (fold start rank) of the element at absolute byte offset x,
// plus the absolute end of that run. Mirrors nezha::ringBlockOf.
template <int N, int ES>
__device__ __forceinline__ int block_at(const Geometry& g, uint64_t x, uint64_t* run_end) {
  const uint64_t rel = x - g.seg_off;
  const uint64_t c = udiv(rel, g.chunk);
  const uint64_t cbeg = c * g.chunk;
  const uint64_t rem = g.seg_len - cbeg;
  const uint64_t clen = rem < g.chunk ? rem : g.chunk;
  const uint64_t q = (clen / ES) / N;
  int b;
  if (q == 0) {
    b = N - 1;
  } else {
    const uint64_t bb = udiv((rel - cbeg) / ES, q);
    b = bb >= static_cast<uint64_t>(N) ? N - 1 : static_cast<int>(bb);
  }
  *run_end = g.seg_off + cbeg + (b == N - 1 ? clen : static_cast<uint64_t>(b + 1) * q * ES);
  return b;
}

template <typename DT, int N>
__device__ __forceinline__ void fold_scalar(const FoldArgs& a, int ndst, uint64_t x) {
  uint64_t run_end;
  const int b = block_at<N, DT::kElem>(a.g, x, &run_end);
  typename DT::Scalar acc = DT::sload(a.src[b] + x);
#pragma unroll
  for (int j = 1; j < N; ++j) acc = DT::sadd(acc, DT::sload(a.src[(b + j) % N] + x));
  for (int d = 0; d < ndst; ++d) DT::sstore(a.dst[d] + x, acc);
}

// Elements of [lo, hi) one per thread of the whole grid.
template <typename DT, int N>
__device__ __forceinline__ void fold_scalar_range(const FoldArgs& a, int ndst, uint64_t lo, uint64_t hi) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x * DT::kElem;
  for (uint64_t x = lo + (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * DT::kElem; x < hi; x += stride) {
    fold_scalar<DT, N>(a, ndst, x);
  }
}

template <int N>
constexpr int unroll_for() {
  return N <= 2 ? 4 : (N <= 4 ? 2 : 1);
}

// Vectors of [x0, x1) (16-byte aligned, one run: fold start rank b).
template <typename DT, int N, int NDST>
__device__ __forceinline__ void fold_run(const FoldArgs& a, int b, uint64_t x0, uint64_t x1) {
  constexpr int U = unroll_for<N>();
  const char* src[N];
#pragma unroll
  for (int j = 0; j < N; ++j) src[j] = a.src[(b + j) % N];
  const uint64_t step = static_cast<uint64_t>(blockDim.x) * 16;
  for (uint64_t base = x0 + threadIdx.x * 16ull; base < x1; base += step * U) {
    uint4 v[U][N];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t x = base + u * step;
      if (x < x1) {
#pragma unroll
        for (int j = 0; j < N; ++j) v[u][j] = ld_v4(src[j] + x);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t x = base + u * step;
      if (x < x1) {
        typename DT::Acc acc = DT::load(v[u][0]);
#pragma unroll
        for (int j = 1; j < N; ++j) DT::add(acc, v[u][j]);
        const uint4 out = DT::store(acc);
        if (NDST == 1) {
          st_v4(a.dst[0] + x, out);
        } else {
#pragma unroll
          for (int d = 0; d < N; ++d) st_v4(a.dst[d] + x, out);
        }
      }
    }
  }
}

// One rank's shard: scalar head/tail + run-walked vector interior.
template <typename DT, int N, int NDST>
__device__ __forceinline__ void fold_shard(const FoldArgs& a) {
  const int ndst = NDST == 1 ? 1 : N;
  const uint64_t vs = (a.s + 15) & ~15ull;
  const uint64_t ve = a.e & ~15ull;
  if (vs >= ve) {
    fold_scalar_range<DT, N>(a, ndst, a.s, a.e);
    return;
  }
  fold_scalar_range<DT, N>(a, ndst, a.s, vs);
  fold_scalar_range<DT, N>(a, ndst, ve, a.e);
  const uint64_t nvec = (ve - vs) / 16;
  const uint64_t cb = vs + 16 * (nvec * blockIdx.x / gridDim.x);
  const uint64_t ce = vs + 16 * (nvec * (blockIdx.x + 1) / gridDim.x);
  uint64_t x = cb;
  while (x < ce) {
    uint64_t run_end;
    const int b = block_at<N, DT::kElem>(a.g, x, &run_end);
    uint64_t vend = run_end & ~15ull;
    if (vend > ce) vend = ce;
    if (vend > x) {
      fold_run<DT, N, NDST>(a, b, x, vend);
      x = vend;
    } else {
      // The vector at x crosses a run boundary: fold its elements one by one.
      if (threadIdx.x < 16 / DT::kElem) fold_scalar<DT, N>(a, ndst, x + threadIdx.x * DT::kElem);
      x += 16;
    }
  }
}

// K2 / K3. With the barrier (SM rail): start barrier (inputs of this op are
// ready on every rank), fold + peer stores, end barrier (every rank's stores
// to my output landed).
template <typename DT, int N, int NDST>
__device__ __forceinline__ void fold_body(const FoldArgs& a) {
  if (!rail_enter(a.ctl)) return rail_exit(a.ctl, false);
  const uint32_t ep = op_epoch(a.bar);
  if (a.use_barrier && !cta_barrier<N, false>(a.bar, ep, a.rank, a.bar.timeout_ns, &a.ctl))
    return rail_exit(a.ctl, false);
  if (a.use_barrier) note_run(a.ctl);
  if (a.ctl.stall) {
    note_stall(a.ctl);
    return rail_exit(a.ctl, false);
  }
  fold_shard<DT, N, NDST>(a);
  if (a.use_barrier && !cta_barrier<N, true>(a.bar, ep + 1, a.rank, end_budget(a.bar, a.ctl), &a.ctl))
    return rail_exit(a.ctl, false);
  post_fault(a.post);
  rail_exit(a.ctl, true);
}

template <typename DT, int N, int NDST>
__global__ void __launch_bounds__(512, 2) fold_kernel(const __grid_constant__ FoldArgs a) {
  fold_body<DT, N, NDST>(a);
}

template <typename DT, int N, int NDST>
__global__ void __launch_bounds__(512, 2) fold_kernel_vr(const __grid_constant__ VPack<FoldArgs> p) {
  fold_body<DT, N, NDST>(p.a[blockIdx.y]);
}

// ------------------------------------------------------------------ NVLS --
template <typename DT>
__device__ __forceinline__ uint4 mm_ld_reduce(const char* p);

#ifndef NZ_SIMT_HOST

#define NZ_MM_LDR(TY)                                                                            \
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add." TY " {%0,%1,%2,%3}, [%4];"         \
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)                                    \
               : "l"(p)                                                                        \
               : "memory")

template <>
__device__ __forceinline__ uint4 mm_ld_reduce<F32>(const char* p) {
  uint4 r;
  NZ_MM_LDR("v4.f32");
  return r;
}
template <>
__device__ __forceinline__ uint4 mm_ld_reduce<BF16>(const char* p) {
  uint4 r;
  NZ_MM_LDR("acc::f32.v4.bf16x2");
  return r;
}
#undef NZ_MM_LDR

template <>
__device__ __forceinline__ uint4 mm_ld_reduce<I32>(const char* p) {
  // ptxas rejects .v4 for integer ld_reduce; four scalar accesses instead.
  uint4 r;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.u32 %0, [%1];" : "=r"(r.x) : "l"(p) : "memory");
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.u32 %0, [%1];" : "=r"(r.y) : "l"(p + 4) : "memory");
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.u32 %0, [%1];" : "=r"(r.z) : "l"(p + 8) : "memory");
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.u32 %0, [%1];" : "=r"(r.w) : "l"(p + 12) : "memory");
  return r;
}

__device__ __forceinline__ void mm_st(char* p, uint4 v) {
  // The store moves bits; .f32 is the only accepted 16-byte form.
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(__uint_as_float(v.x)),
               "f"(__uint_as_float(v.y)), "f"(__uint_as_float(v.z)), "f"(__uint_as_float(v.w))
               : "memory");
}
#endif  // NZ_SIMT_HOST (the harness's multicast emulation: tests/fakecuda/simt.h)

template <typename DT, int N>
__global__ void __launch_bounds__(512, 2) nvls_kernel(const __grid_constant__ NvlsArgs a) {
  constexpr int U = 4;
  if (!rail_enter(a.f.ctl)) return rail_exit(a.f.ctl, false);
  const uint32_t ep = op_epoch(a.f.bar);
  if (!cta_barrier<N, false>(a.f.bar, ep, a.f.rank, a.f.bar.timeout_ns, &a.f.ctl)) return rail_exit(a.f.ctl, false);
  note_run(a.f.ctl);
  if (a.f.ctl.stall) {
    note_stall(a.f.ctl);
    return rail_exit(a.f.ctl, false);
  }
  const uint64_t vs = (a.f.s + 15) & ~15ull;
  const uint64_t ve = a.f.e & ~15ull;
  if (vs >= ve) {
    fold_scalar_range<DT, N>(a.f, N, a.f.s, a.f.e);
  } else {
    fold_scalar_range<DT, N>(a.f, N, a.f.s, vs);
    fold_scalar_range<DT, N>(a.f, N, ve, a.f.e);
    const uint64_t step = static_cast<uint64_t>(gridDim.x) * blockDim.x * 16;
    for (uint64_t base = vs + (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 16; base < ve;
         base += step * U) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t x = base + u * step;
        if (x < ve) v[u] = mm_ld_reduce<DT>(a.mc_in + x);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t x = base + u * step;
        if (x < ve) mm_st(a.mc_out + x, v[u]);
      }
    }
  }
  if (!cta_barrier<N, true>(a.f.bar, ep + 1, a.f.rank, end_budget(a.f.bar, a.f.ctl), &a.f.ctl))
    return rail_exit(a.f.ctl, false);
  post_fault(a.f.post);
  rail_exit(a.f.ctl, true);
}


// --------------------------------------------------------- LL (one-shot) --
// LLArgs and the protocol: kernel_args.h.
__device__ __forceinline__ uint32_t ll_load_word(const char* base, uint64_t x, uint64_t hi) {
  if (x + 4 <= hi) return *reinterpret_cast<const uint32_t*>(base + x);
  return static_cast<uint32_t>(*reinterpret_cast<const unsigned short*>(base + x));  // bf16 tail
}

// v[(b + j) mod N] without a runtime index into the register array (which
// would put v in local memory): an unrolled select over the N registers.
template <int N>
__device__ __forceinline__ uint32_t ll_pick(const uint32_t (&v)[N], int b, int j) {
  const int i = b + j < N ? b + j : b + j - N;
  uint32_t r = v[0];
#pragma unroll
  for (int q = 1; q < N; ++q) r = i == q ? v[q] : r;
  return r;
}

template <typename DT, int N>
__device__ __forceinline__ void ll_fold_word(const LLArgs& a, const uint32_t (&v)[N], uint64_t x) {
  constexpr int per = 4 / DT::kElem;
#pragma unroll
  for (int k = 0; k < per; ++k) {
    const uint64_t xe = x + static_cast<uint64_t>(k) * DT::kElem;
    if (xe >= a.hi) break;
    uint64_t run_end;
    const int b = block_at<N, DT::kElem>(a.g, xe, &run_end);
    if (DT::kElem == 4) {
      typename DT::Scalar acc;
      uint32_t w = ll_pick<N>(v, b, 0);
      memcpy(&acc, &w, 4);
#pragma unroll
      for (int j = 1; j < N; ++j) {
        typename DT::Scalar t;
        uint32_t wj = ll_pick<N>(v, b, j);
        memcpy(&t, &wj, 4);
        acc = DT::sadd(acc, t);
      }
      DT::sstore(a.out + xe, acc);
    } else {
      const uint32_t wb = ll_pick<N>(v, b, 0);
      float acc = __uint_as_float(k == 0 ? (wb << 16) : (wb & 0xffff0000u));
#pragma unroll
      for (int j = 1; j < N; ++j) {
        const uint32_t wj = ll_pick<N>(v, b, j);
        acc = acc + __uint_as_float(k == 0 ? (wj << 16) : (wj & 0xffff0000u));
      }
      DT::sstore(a.out + xe, acc);
    }
  }
}

template <typename DT, int N>
__device__ __forceinline__ void ll_body(const LLArgs& a) {
  if (!rail_enter(a.ctl)) return rail_exit(a.ctl, false);
  if (a.ctl.stall) {  // dead link: nothing of this rank reaches its peers
    note_stall(a.ctl);
    return rail_exit(a.ctl, false);
  }
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  uint32_t flag = a.flag;
  int parity = a.parity;
  if (a.seq) {
    flag = seq_read(a.seq) + 1u;
    if (flag == 0) flag = 1;  // 0 means "never written"
    parity = static_cast<int>(flag & 1u);
  }
  const uint64_t my_slot = (static_cast<uint64_t>(parity) * N + a.rank) * a.slot_words;
  const uint64_t pairs = (a.words + 1) / 2;
  for (uint64_t p = tid; p < pairs; p += stride) {
    const uint64_t x = a.lo + 8 * p;
    const uint32_t d0 = ll_load_word(a.in, x, a.hi);
    const uint32_t d1 = x + 4 < a.hi ? ll_load_word(a.in, x + 4, a.hi) : 0u;
#pragma unroll
    for (int r = 0; r < N; ++r) {
      ll_push_pair(a.peer[r] + my_slot + 2 * p, d0, flag, d1);
    }
  }
  // A peer's words never arrived (watchdog), or the ranks already agreed
  // that the rail failed (abort). The monitor never aborts an LL wait on a
  // heartbeat alone: a rank leaving early has pushed its own words, so a late
  // peer could still complete the op while this rank's output stays unfolded.
  // After an agreement some rank's launches on the rail exit at entry, so no
  // rank can complete a later LL op and leaving is consistent.
  bool bail = false;
  for (uint64_t w = tid; w < a.words && !bail; w += stride) {
    uint32_t v[N];
#pragma unroll
    for (int r = 0; r < N; ++r) {
      if (bail) break;
      const uint64_t* src = a.local + (static_cast<uint64_t>(parity) * N + r) * a.slot_words + w;
      uint32_t d = 0, f;
      int spins = 0;
      uint64_t t0 = 0;
      for (;;) {
        ll_poll_word(src, &d, &f);
        if (f == flag) break;
        if (++spins == 256) {
          spins = 0;
          const uint64_t now = globaltimer();
          if (t0 == 0) {
            t0 = now;
          } else if (now - t0 > a.timeout_ns || (a.abort && *a.abort)) {
            atomicExch_system(a.watchdog, 1);
            note_detect(&a.ctl, now);
            bail = true;
            break;
          }
        }
      }
      v[r] = d;
    }
    if (!bail) ll_fold_word<DT, N>(a, v, a.lo + 4 * w);
  }
  const bool failed = __syncthreads_or(bail) != 0;
  if (!failed) post_fault(a.post);
  rail_exit(a.ctl, !failed);
}

template <typename DT, int N>
__global__ void __launch_bounds__(512, 1) ll_kernel(const __grid_constant__ LLArgs a) {
  ll_body<DT, N>(a);
}

template <typename DT, int N>
__global__ void __launch_bounds__(512, 1) ll_kernel_vr(const __grid_constant__ VPack<LLArgs> p) {
  ll_body<DT, N>(p.a[blockIdx.y]);
}

// N = 1: the allreduce is the identity, i.e. a copy in -> out (HBM-bound).
// 8 x 16-byte loads in flight per thread before the stores, no run walking.
static __global__ void __launch_bounds__(512, 2) copy_kernel(const char* __restrict__ src, char* __restrict__ dst, uint64_t lo,
                                                      uint64_t hi, FaultPost post, RailCtl ctl) {
  if (!rail_enter(ctl)) return rail_exit(ctl, false);
  if (ctl.stall) {
    note_stall(ctl);
    return rail_exit(ctl, false);
  }
  const uint64_t vs = (lo + 15) & ~15ull;
  const uint64_t ve = hi & ~15ull;
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t nthr = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  if (vs >= ve) {
    for (uint64_t x = lo + tid; x < hi; x += nthr) dst[x] = src[x];
  } else {
    if (tid < vs - lo) dst[lo + tid] = src[lo + tid];
    if (tid < hi - ve) dst[ve + tid] = src[ve + tid];
    constexpr int U = 8;
    const uint64_t step = nthr * 16;
    for (uint64_t base = vs + tid * 16; base < ve; base += step * U) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t x = base + u * step;
        if (x < ve) v[u] = ld_v4(src + x);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t x = base + u * step;
        if (x < ve) st_v4(dst + x, v[u]);
      }
    }
  }
  if (post.rec) {
    __syncthreads();
    post_fault(post);
  }
  rail_exit(ctl, true);
}


// ------------------------------------------------ CE barriers (K4) --
// BarrierKArgs: kernel_args.h.
template <int N>
__device__ __forceinline__ void barrier_body(const BarrierKArgs& k) {
  if (!rail_enter(k.ctl)) return rail_exit(k.ctl, false);
  const uint64_t budget = k.end ? end_budget(k.bar, k.ctl) : k.bar.timeout_ns;
  if (!cta_barrier<N, true>(k.bar, op_epoch(k.bar), k.rank, budget, &k.ctl)) return rail_exit(k.ctl, false);
  if (!k.end) note_run(k.ctl);
  if (!k.end && k.ctl.stall) {
    note_stall(k.ctl);
    return rail_exit(k.ctl, false);
  }
  post_fault(k.post);
  rail_exit(k.ctl, true);
}

template <int N>
__global__ void barrier_kernel(const __grid_constant__ BarrierKArgs k) {
  barrier_body<N>(k);
}

template <int N>
__global__ void barrier_kernel_vr(const __grid_constant__ VPack<BarrierKArgs> p) {
  barrier_body<N>(p.a[blockIdx.y]);
}

}  // namespace nz
