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
//
// Summation order (P1): an element of ring block b of its chunk is
// folded x_b + x_{b+1} + ... + x_{b-1}. A CTA walks its contiguous share of
// the shard run by run (a run = one ring block of one chunk), so the
// rotation is resolved once per run, not per vector; the rare 16-byte vector
// that straddles a run boundary is folded element by element.
#pragma once

#include <cuda_bf16.h>
#include <stdint.h>

#include "nezha_b200.h"

namespace nz {

constexpr int kDevMaxRanks = 8;

struct Geometry {
  uint64_t seg_off;
  uint64_t seg_len;
  uint64_t chunk;
};

// Cross-rank per-CTA barrier pads of one rail: slot [cta][rank] of rank p's
// pad is written only by `rank`, with monotonically increasing epochs.
struct BarrierArgs {
  uint32_t* local;
  uint32_t* peer[kDevMaxRanks];
  uint32_t epoch;
  int* watchdog;  // host-mapped; set when a wait times out
  uint64_t timeout_ns;  // give up after this long (NEZHA_WATCHDOG_MS, default 20 s)
  int relaxed_poll;     // 1: poll ld.relaxed.sys, one fence.acq_rel.sys after (PTX acquire pattern)
  uint32_t* seq;        // graph-safe rails: device [op counter, CTAs retired]; nullptr = host `epoch`
};

struct FaultPost {
  nz_fault_record_t* rec;  // host-mapped, nullptr = nothing to post
  uint32_t op_seq;
  uint64_t chunk;
};

struct FoldArgs {
  const char* src[kDevMaxRanks];  // rank r's element at byte offset x is src[r] + x
  char* dst[kDevMaxRanks];        // outputs written at byte offset x
  uint64_t s, e;                  // this rank's shard [s, e)
  uint64_t range_bytes;           // whole reduced range, sizes the grid identically on every rank
  Geometry g;
  BarrierArgs bar;
  int use_barrier;
  int rank;
  FaultPost post;
};

struct NvlsArgs {
  char* mc_in;
  char* mc_out;
  FoldArgs f;  // unicast view for the unaligned head / tail and the barrier
};

// ------------------------------------------------------------ primitives --
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

__device__ __forceinline__ uint32_t ld_relaxed_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

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


// Graph-safe rails (NZ_RAIL_FLAG_GRAPH_SAFE) take their barrier epochs and
// LL flags from a device counter instead of kernel arguments, so a launch
// captured in a CUDA graph stays valid on every replay. Every CTA reads the
// counter on entry; the last CTA to retire advances it. A rail's launches are
// stream ordered, so the next one sees the advanced value.
__device__ __forceinline__ uint32_t seq_read(const uint32_t* seq) {
  return *reinterpret_cast<const volatile uint32_t*>(seq);
}

__device__ __forceinline__ void seq_retire(uint32_t* seq) {
  if (!seq) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(seq + 1, 1u) == gridDim.x - 1) {
      atomicExch(seq + 1, 0u);
      atomicAdd(seq, 1u);
    }
  }
}

__device__ __forceinline__ uint32_t op_epoch(const BarrierArgs& b) {
  return b.seq ? 2u * seq_read(b.seq) + 1u : b.epoch;
}

// Per-CTA barrier across ranks. Returns false (and flags the watchdog) if a
// peer never arrived, so the kernel can exit instead of hanging the GPU.
// `publish` = this CTA wrote peer-visible data that must land before peers
// pass the barrier (each thread fences its own stores at system scope).
template <int N, bool kPublish>
__device__ __forceinline__ bool cta_barrier(const BarrierArgs& b, uint32_t epoch, int rank) {
  __shared__ int s_ok;
  if (threadIdx.x == 0) s_ok = 1;
  if (kPublish) fence_acq_rel_sys();
  __syncthreads();
  const int t = threadIdx.x;
  if (t < N) {
    st_release_sys(b.peer[t] + blockIdx.x * kDevMaxRanks + rank, epoch);
    const uint32_t* slot = b.local + blockIdx.x * kDevMaxRanks + t;
    uint64_t t0 = 0;
    int spins = 0;
    const bool relaxed = b.relaxed_poll != 0;
    while (static_cast<int32_t>((relaxed ? ld_relaxed_sys(slot) : ld_acquire_sys(slot)) - epoch) < 0) {
      if (++spins == 64) {
        spins = 0;
        const uint64_t now = globaltimer();
        if (t0 == 0) {
          t0 = now;
        } else if (now - t0 > b.timeout_ns) {
          atomicExch_system(b.watchdog, 1);
          s_ok = 0;
          break;
        }
      }
    }
    if (relaxed) fence_acq_rel_sys();  // relaxed observation + fence = acquire pattern
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
  __device__ static float sfinal(float a) { return a; }
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
__device__ __forceinline__ void fold_run(const FoldArgs& a, int ndst, int b, uint64_t x0, uint64_t x1) {
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
      fold_run<DT, N, NDST>(a, ndst, b, x, vend);
      x = vend;
    } else {
      // The vector at x crosses a run boundary: fold its elements one by one.
      if (threadIdx.x < 16 / DT::kElem) fold_scalar<DT, N>(a, ndst, x + threadIdx.x * DT::kElem);
      x += 16;
    }
  }
}

template <typename DT, int N, int NDST>
__global__ void __launch_bounds__(512, 2) fold_kernel(const __grid_constant__ FoldArgs a) {
  const uint32_t ep = op_epoch(a.bar);
  if (a.use_barrier && !cta_barrier<N, false>(a.bar, ep, a.rank)) return seq_retire(a.bar.seq);
  fold_shard<DT, N, NDST>(a);
  if (a.use_barrier && !cta_barrier<N, true>(a.bar, ep + 1, a.rank)) return seq_retire(a.bar.seq);
  post_fault(a.post);
  seq_retire(a.bar.seq);
}

// ------------------------------------------------------------------ NVLS --
// WEAK selects .weak instead of .relaxed.sys memory semantics (the barrier
// around the loop already orders the data); kept as a tuning variant.
template <typename DT, bool WEAK>
__device__ __forceinline__ uint4 mm_ld_reduce(const char* p);

#define NZ_MM_LDR(SEM, TY)                                                                                  \
  asm volatile("multimem.ld_reduce." SEM ".global.add." TY " {%0,%1,%2,%3}, [%4];"                        \
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)                                               \
               : "l"(p)                                                                                   \
               : "memory")

template <>
__device__ __forceinline__ uint4 mm_ld_reduce<F32, false>(const char* p) {
  uint4 r;
  NZ_MM_LDR("relaxed.sys", "v4.f32");
  return r;
}
template <>
__device__ __forceinline__ uint4 mm_ld_reduce<F32, true>(const char* p) {
  uint4 r;
  NZ_MM_LDR("weak", "v4.f32");
  return r;
}
template <>
__device__ __forceinline__ uint4 mm_ld_reduce<BF16, false>(const char* p) {
  uint4 r;
  NZ_MM_LDR("relaxed.sys", "acc::f32.v4.bf16x2");
  return r;
}
template <>
__device__ __forceinline__ uint4 mm_ld_reduce<BF16, true>(const char* p) {
  uint4 r;
  NZ_MM_LDR("weak", "acc::f32.v4.bf16x2");
  return r;
}
#undef NZ_MM_LDR

template <bool WEAK>
__device__ __forceinline__ uint4 mm_ld_reduce_i32(const char* p) {
  // ptxas rejects .v4 for integer ld_reduce; four scalar accesses instead.
  uint4 r;
  if (WEAK) {
    asm volatile("multimem.ld_reduce.weak.global.add.u32 %0, [%1];" : "=r"(r.x) : "l"(p) : "memory");
    asm volatile("multimem.ld_reduce.weak.global.add.u32 %0, [%1];" : "=r"(r.y) : "l"(p + 4) : "memory");
    asm volatile("multimem.ld_reduce.weak.global.add.u32 %0, [%1];" : "=r"(r.z) : "l"(p + 8) : "memory");
    asm volatile("multimem.ld_reduce.weak.global.add.u32 %0, [%1];" : "=r"(r.w) : "l"(p + 12) : "memory");
  } else {
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.u32 %0, [%1];" : "=r"(r.x) : "l"(p) : "memory");
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.u32 %0, [%1];" : "=r"(r.y) : "l"(p + 4) : "memory");
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.u32 %0, [%1];" : "=r"(r.z) : "l"(p + 8) : "memory");
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.u32 %0, [%1];" : "=r"(r.w) : "l"(p + 12) : "memory");
  }
  return r;
}
template <>
__device__ __forceinline__ uint4 mm_ld_reduce<I32, false>(const char* p) {
  return mm_ld_reduce_i32<false>(p);
}
template <>
__device__ __forceinline__ uint4 mm_ld_reduce<I32, true>(const char* p) {
  return mm_ld_reduce_i32<true>(p);
}

template <bool WEAK>
__device__ __forceinline__ void mm_st(char* p, uint4 v) {
  // The store moves bits; .f32 is the only accepted 16-byte form.
  if (WEAK) {
    asm volatile("multimem.st.weak.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(__uint_as_float(v.x)),
                 "f"(__uint_as_float(v.y)), "f"(__uint_as_float(v.z)), "f"(__uint_as_float(v.w))
                 : "memory");
  } else {
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(__uint_as_float(v.x)),
                 "f"(__uint_as_float(v.y)), "f"(__uint_as_float(v.z)), "f"(__uint_as_float(v.w))
                 : "memory");
  }
}

template <typename DT, int N, int U, bool WEAK>
__global__ void __launch_bounds__(512, 2) nvls_kernel(const __grid_constant__ NvlsArgs a) {
  const uint32_t ep = op_epoch(a.f.bar);
  if (!cta_barrier<N, false>(a.f.bar, ep, a.f.rank)) return seq_retire(a.f.bar.seq);
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
        if (x < ve) v[u] = mm_ld_reduce<DT, WEAK>(a.mc_in + x);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t x = base + u * step;
        if (x < ve) mm_st<WEAK>(a.mc_out + x, v[u]);
      }
    }
  }
  if (!cta_barrier<N, true>(a.f.bar, ep + 1, a.f.rank)) return seq_retire(a.f.bar.seq);
  post_fault(a.f.post);
  seq_retire(a.f.bar.seq);
}

// --------------------------------------------------------- LL (one-shot) --
// Small segments on the SM rail: every rank pushes its words, each tagged
// with this op's flag in the same 8-byte store ({data, flag} pairs, the LL
// idea), into slot [rank] of every peer's LL buffer, then polls its own slots
// and folds in ring order (P1). No barrier round trips: one NVLink one-way
// latency. Two parities alternate so a rank at most one op ahead never
// overwrites a slot a peer still reads (stream order on every rank).
struct LLArgs {
  const char* in;  // my input, byte offset x at in + x
  char* out;       // my output
  uint64_t* peer[kDevMaxRanks];  // each rank's LL buffer (8-byte {data, flag} words)
  uint64_t* local;
  uint64_t* mc;  // multicast view of the LL buffers (NVLS-LL: one store reaches every rank)
  uint64_t lo, hi;
  uint64_t words;       // ceil((hi - lo) / 4)
  uint64_t slot_words;  // capacity of one (parity, rank) slot
  Geometry g;
  uint32_t flag;
  int parity;
  int rank;
  int* watchdog;
  uint64_t timeout_ns;
  FaultPost post;
  uint32_t* seq;  // graph-safe rails: flag / parity from the device counter (see seq_retire)
};

__device__ __forceinline__ uint32_t ll_load_word(const char* base, uint64_t x, uint64_t hi) {
  if (x + 4 <= hi) return *reinterpret_cast<const uint32_t*>(base + x);
  return static_cast<uint32_t>(*reinterpret_cast<const unsigned short*>(base + x));  // bf16 tail
}

// v[(b + j) mod N] without a runtime index into the register array (which
// would put v in local memory: the N = 4 / 5 instances spilled): an unrolled
// select over the N registers.
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

// MC = true is the NVLS-LL variant: the push is one multimem.st to the
// multicast view, which the switch replicates into every rank's slot.
template <typename DT, int N, bool MC>
__global__ void __launch_bounds__(512) ll_kernel(const __grid_constant__ LLArgs a) {
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
    if (MC) {
      mm_st<false>(reinterpret_cast<char*>(a.mc + my_slot + 2 * p), make_uint4(d0, flag, d1, flag));
    } else {
#pragma unroll
      for (int r = 0; r < N; ++r) {
        uint64_t* dst = a.peer[r] + my_slot + 2 * p;
        asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(dst), "r"(d0), "r"(flag), "r"(d1),
                     "r"(flag)
                     : "memory");
      }
    }
  }
  bool bail = false;  // a peer's words never arrived (watchdog)
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
        asm volatile("ld.volatile.global.v2.u32 {%0,%1}, [%2];" : "=r"(d), "=r"(f) : "l"(src) : "memory");
        if (f == flag) break;
        if (++spins == 256) {
          spins = 0;
          const uint64_t now = globaltimer();
          if (t0 == 0) {
            t0 = now;
          } else if (now - t0 > a.timeout_ns) {
            atomicExch_system(a.watchdog, 1);
            bail = true;
            break;
          }
        }
      }
      v[r] = d;
    }
    if (!bail) ll_fold_word<DT, N>(a, v, a.lo + 4 * w);
  }
  if (a.seq) {
    seq_retire(a.seq);  // every thread gets here (no early return): the barrier inside is safe
    if (bail) return;
  } else if (bail) {
    return;
  }
  post_fault(a.post);
}

// ------------------------------------------------- SM rail, one-shot ------
// K7: mid-size payloads on the SM rail. Every rank pushes its whole range
// into slot [parity][rank] of every peer's staging buffer, one per-CTA
// barrier publishes the pushes, then every rank folds all N copies locally in
// P1 order (its own from `in`) into its own `out`. One barrier instead of the
// two-shot's two, (N-1)·L wire bytes instead of 2(N-1)/N·L: it wins where
// latency dominates. CTA c pushes exactly the bytes it later folds (same
// partition as fold_shard over [lo, hi)), so its own barrier slot suffices.
// Parity alternates with the epoch; a rank can only reuse a parity after an
// op every rank joined, i.e. after every rank finished reading it.
struct OneShotArgs {
  const char* in;
  char* stg_peer[kDevMaxRanks];  // rank p's staging buffer (where I push)
  uint64_t lo, hi;               // reduced byte range
  uint64_t lo16;                 // lo rounded down to 16: slot offset 0
  uint64_t slot_bytes;
  BarrierArgs bar;
  int rank;
  FaultPost post;
  FoldArgs f[2];  // the local fold per staging parity (sources: my `in` + my staging slots), built on the host
};

template <int N, int ES>
__device__ __forceinline__ void oneshot_push_scalar(const OneShotArgs& a, uint64_t off, uint64_t x) {
  if (ES == 4) {
    const uint32_t v = *reinterpret_cast<const uint32_t*>(a.in + x);
#pragma unroll
    for (int r = 0; r < N; ++r)
      if (r != a.rank) *reinterpret_cast<uint32_t*>(a.stg_peer[r] + off + (x - a.lo16)) = v;
  } else {
    const unsigned short v = *reinterpret_cast<const unsigned short*>(a.in + x);
#pragma unroll
    for (int r = 0; r < N; ++r)
      if (r != a.rank) *reinterpret_cast<unsigned short*>(a.stg_peer[r] + off + (x - a.lo16)) = v;
  }
}

template <typename DT, int N>
__global__ void __launch_bounds__(512, 2) oneshot_kernel(const __grid_constant__ OneShotArgs a) {
  const uint32_t ep = op_epoch(a.bar);
  const int parity = static_cast<int>((ep >> 1) & 1u);
  const uint64_t off = (static_cast<uint64_t>(parity) * N + a.rank) * a.slot_bytes;  // my slot in every peer
  // Push: the same element / vector partition fold_shard uses below.
  const uint64_t vs = (a.lo + 15) & ~15ull;
  const uint64_t ve = a.hi & ~15ull;
  const uint64_t gstride = static_cast<uint64_t>(gridDim.x) * blockDim.x * DT::kElem;
  const uint64_t gtid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (vs >= ve) {
    for (uint64_t x = a.lo + gtid * DT::kElem; x < a.hi; x += gstride) oneshot_push_scalar<N, DT::kElem>(a, off, x);
  } else {
    for (uint64_t x = a.lo + gtid * DT::kElem; x < vs; x += gstride) oneshot_push_scalar<N, DT::kElem>(a, off, x);
    for (uint64_t x = ve + gtid * DT::kElem; x < a.hi; x += gstride) oneshot_push_scalar<N, DT::kElem>(a, off, x);
    const uint64_t nvec = (ve - vs) / 16;
    const uint64_t cb = vs + 16 * (nvec * blockIdx.x / gridDim.x);
    const uint64_t ce = vs + 16 * (nvec * (blockIdx.x + 1) / gridDim.x);
    for (uint64_t x = cb + threadIdx.x * 16ull; x < ce; x += static_cast<uint64_t>(blockDim.x) * 16) {
      const uint4 v = ld_v4(a.in + x);
#pragma unroll
      for (int r = 0; r < N; ++r)
        if (r != a.rank) st_v4(a.stg_peer[r] + off + (x - a.lo16), v);
    }
  }
  if (!cta_barrier<N, true>(a.bar, ep, a.rank)) return seq_retire(a.bar.seq);
  // Fold every rank's copy of this CTA's part, P1 order, into my `out`
  // (param-space FoldArgs: no local-memory copy).
  fold_shard<DT, N, 1>(a.f[parity]);
  post_fault(a.post);
  seq_retire(a.bar.seq);
}

// ------------------------------------------------- SM rail, TMA pipeline --
// K3t: the SM rail's two-shot fold with the peer traffic moved by the Tensor
// Memory Accelerator. One elected thread streams 1-D bulk tiles of the shard
// from every rank's `in` (cp.async.bulk global -> shared over NVLink,
// completion on an mbarrier) through a kTmaStages-deep ring; all threads fold
// the N staged tiles in ring order (P1) into an output tile; the elected
// thread then bulk-stores that tile to every rank's `out`
// (cp.async.bulk shared -> global). Few instructions keep many NVLink bytes
// in flight, which the LDG/STG version needs a full CTA of threads for.
constexpr uint32_t kTmaTile = 4096;  // bytes per source per stage
constexpr int kTmaStages = 3;

__host__ __device__ constexpr size_t tma_smem_bytes(int n) {
  return static_cast<size_t>(kTmaStages) * (n + 1) * kTmaTile + kTmaStages * sizeof(uint64_t);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

// Bounded wait: false after ~timeout_ns so a lost transfer cannot hang the GPU.
__device__ __forceinline__ bool mbar_wait(uint64_t* bar, uint32_t parity, uint64_t timeout_ns) {
  uint64_t t0 = 0;
  for (;;) {
    uint32_t done;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return true;
    const uint64_t now = globaltimer();
    if (t0 == 0) {
      t0 = now;
    } else if (now - t0 > timeout_ns) {
      return false;
    }
  }
}

__device__ __forceinline__ void tma_load(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(smem_dst)),
               "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tma_store(void* gdst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(smem_src)),
               "r"(bytes)
               : "memory");
}

template <typename DT, int N>
__global__ void __launch_bounds__(256, 1) sm_tma_kernel(const __grid_constant__ FoldArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* tiles = smem;                                            // [stage][rank][kTmaTile]
  unsigned char* outs = smem + static_cast<size_t>(kTmaStages) * N * kTmaTile;  // [stage][kTmaTile]
  uint64_t* bars = reinterpret_cast<uint64_t*>(outs + static_cast<size_t>(kTmaStages) * kTmaTile);

  const uint32_t ep = op_epoch(a.bar);
  if (a.use_barrier && !cta_barrier<N, false>(a.bar, ep, a.rank)) return seq_retire(a.bar.seq);
  const uint64_t vs = (a.s + 15) & ~15ull;
  const uint64_t ve = a.e & ~15ull;
  if (vs >= ve) {
    fold_scalar_range<DT, N>(a, N, a.s, a.e);
  } else {
    fold_scalar_range<DT, N>(a, N, a.s, vs);
    fold_scalar_range<DT, N>(a, N, ve, a.e);
    const uint64_t nvec = (ve - vs) / 16;
    const uint64_t cb = vs + 16 * (nvec * blockIdx.x / gridDim.x);
    const uint64_t ce = vs + 16 * (nvec * (blockIdx.x + 1) / gridDim.x);
    const uint64_t ntiles = (ce - cb + kTmaTile - 1) / kTmaTile;
    const bool leader = threadIdx.x == 0;
    if (leader) {
      for (int s = 0; s < kTmaStages; ++s) mbar_init(&bars[s], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](uint64_t i) {
      const int s = static_cast<int>(i % kTmaStages);
      const uint64_t x = cb + i * kTmaTile;
      const uint32_t len = static_cast<uint32_t>(ce - x < kTmaTile ? ce - x : kTmaTile);
      mbar_expect_tx(&bars[s], len * N);
#pragma unroll
      for (int r = 0; r < N; ++r) tma_load(tiles + (static_cast<size_t>(s) * N + r) * kTmaTile, a.src[r] + x, len, &bars[s]);
    };
    if (leader)
      for (uint64_t i = 0; i < ntiles && i < static_cast<uint64_t>(kTmaStages); ++i) issue(i);
    for (uint64_t i = 0; i < ntiles; ++i) {
      const int s = static_cast<int>(i % kTmaStages);
      const uint64_t x = cb + i * kTmaTile;
      const uint32_t len = static_cast<uint32_t>(ce - x < kTmaTile ? ce - x : kTmaTile);
      // The bulk stores of tile i - kTmaStages must have finished reading outs[s].
      if (leader && i >= static_cast<uint64_t>(kTmaStages))
        asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kTmaStages - 1) : "memory");
      const uint64_t budget = a.bar.timeout_ns ? a.bar.timeout_ns : 20ull * 1000 * 1000 * 1000;
      const int ok = mbar_wait(&bars[s], static_cast<uint32_t>((i / kTmaStages) & 1), budget) ? 1 : 0;
      if (!__syncthreads_and(ok)) {
        if (leader && a.bar.watchdog) atomicExch_system(a.bar.watchdog, 1);
        if (leader) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        return seq_retire(a.bar.seq);  // a tile never arrived: give up rather than hang
      }
      const unsigned char* st = tiles + static_cast<size_t>(s) * N * kTmaTile;
      unsigned char* ot = outs + static_cast<size_t>(s) * kTmaTile;
      for (uint32_t v = threadIdx.x * 16; v < len; v += blockDim.x * 16) {
        const uint64_t xv = x + v;
        uint64_t run_end;
        const int b = block_at<N, DT::kElem>(a.g, xv, &run_end);
        if (run_end >= xv + 16) {
          typename DT::Acc acc = DT::load(*reinterpret_cast<const uint4*>(st + static_cast<size_t>(b) * kTmaTile + v));
#pragma unroll
          for (int j = 1; j < N; ++j)
            DT::add(acc, *reinterpret_cast<const uint4*>(st + static_cast<size_t>((b + j) % N) * kTmaTile + v));
          *reinterpret_cast<uint4*>(ot + v) = DT::store(acc);
        } else {
          // Vector straddles a ring-block boundary: fold element by element.
          for (uint32_t k = 0; k < 16; k += DT::kElem) {
            uint64_t re;
            const int be = block_at<N, DT::kElem>(a.g, xv + k, &re);
            typename DT::Scalar acc = DT::sload(reinterpret_cast<const char*>(st + static_cast<size_t>(be) * kTmaTile + v + k));
            for (int j = 1; j < N; ++j)
              acc = DT::sadd(acc, DT::sload(reinterpret_cast<const char*>(st + static_cast<size_t>((be + j) % N) * kTmaTile + v + k)));
            DT::sstore(reinterpret_cast<char*>(ot + v + k), acc);
          }
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> async proxy
      __syncthreads();
      if (leader) {
#pragma unroll
        for (int r = 0; r < N; ++r) tma_store(a.dst[r] + x, ot, len);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        if (i + kTmaStages < ntiles) issue(i + kTmaStages);  // tiles[s] is free: every thread folded it
      }
    }
    if (leader) {
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // all peer stores performed
      asm volatile("fence.proxy.async.global;" ::: "memory");   // ... and ordered before the release below
    }
  }
  if (a.use_barrier && !cta_barrier<N, true>(a.bar, ep + 1, a.rank)) return seq_retire(a.bar.seq);
  post_fault(a.post);
  seq_retire(a.bar.seq);
}

// N = 1: the allreduce is the identity, i.e. a copy in -> out (HBM-bound).
// 8 x 16-byte loads in flight per thread before the stores, no run walking.
__global__ void __launch_bounds__(512, 2) copy_kernel(const char* __restrict__ src, char* __restrict__ dst, uint64_t lo,
                                                      uint64_t hi, FaultPost post) {
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
}

// CE rail: start / end barriers around the DMA phases, and the fault post.
template <int N>
__global__ void barrier_kernel(const __grid_constant__ BarrierArgs b, int rank, FaultPost post) {
  if (!cta_barrier<N, true>(b, op_epoch(b), rank)) return seq_retire(b.seq);
  post_fault(post);
  seq_retire(b.seq);
}

}  // namespace nz
