/*
 * nezha_oracle.c — CPU restatement of the reference allreduce reduction.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing in the product (paper_2405_17870_b200/)
 * links, loads or calls this file; only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs use it, as the checker.
 *
 * What it restates. The reference ships no allreduce code (SURVEY.md §0.1:
 * proj/tests/CMakeLists.txt:12-25 has the collective suites commented out);
 * the behaviour is defined by the reference's own spec:
 *   - ring_allreduce, reduce-scatter then allgather over N ring blocks
 *     (SPEC.md:189-197), rank-ascending reduction order, last
 *     block absorbs the remainder;
 *   - ring_chunked_allreduce over chunks of max(64 KiB, len/(2N))
 *     (SPEC.md:198-205, :223).
 * In the ring, at step s rank r sends block (r - s) mod N to r + 1, which
 * adds its own copy (recv + own). Block b is therefore summed as
 *   ((x_b + x_{b+1}) + x_{b+2}) + ... + x_{b-1}      (P1)
 * and this file evaluates exactly that fold per element, without running
 * the message passing. oracle/ring_inmem.cpp runs the literal ring over the
 * reference's InMemoryFabric and tests/test_oracle.py checks the two agree
 * bit for bit.
 * bf16 accumulates in fp32 along the same fold and rounds once (RNE); int32
 * wraps (P2).
 *
 * Parity pinning: the fold is pinned by SPEC.md:195-196's examples and by
 * the literal ring on the reference transport (tests/test_oracle.py), plus
 * the order-revealing golden vector in tests/golden/.
 */
#include <stdint.h>
#include <string.h>

#define NZO_F32 0
#define NZO_BF16 1
#define NZO_I32 2

static uint64_t esize_of(int dtype) { return dtype == NZO_BF16 ? 2u : 4u; }

static float bf16_to_f32(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

static uint16_t f32_to_bf16_rne(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40u); /* quiet NaN */
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

/* Start rank of the fold for element `p` of a chunk of `ce` elements. */
static int ring_block(uint64_t p, uint64_t ce, int world) {
  uint64_t q = ce / (uint64_t)world;
  if (q == 0) return world - 1;
  uint64_t b = p / q;
  return b >= (uint64_t)world ? world - 1 : (int)b;
}

/* P10 chunk size: max(64 KiB, round4down(len / 2N)); ring = whole segment. */
uint64_t nzo_default_chunk_bytes(uint64_t seg_len, int world, int chunked) {
  if (!chunked) return seg_len < 4 ? 4 : seg_len;
  uint64_t even = (seg_len / (2u * (uint64_t)world)) & ~(uint64_t)3;
  return even > 65536u ? even : 65536u;
}

/*
 * Reduce bytes [seg_off, seg_off + seg_len) of the `world` input buffers into
 * `out`, with the chunk geometry (seg_off, seg_len, chunk_bytes).
 * Only the sub-range [lo, hi) (byte offsets, element aligned) is written, so a
 * caller can evaluate exactly what a rail or a handoff target produced.
 * Returns 0, or -1 on a bad argument.
 */
int nzo_reduce_range(int world, int dtype, const void* const* inputs, void* out, uint64_t seg_off,
                     uint64_t seg_len, uint64_t chunk_bytes, uint64_t lo, uint64_t hi) {
  const uint64_t es = esize_of(dtype);
  if (world < 1 || chunk_bytes == 0 || chunk_bytes % es || seg_off % es || seg_len % es) return -1;
  if (lo < seg_off || hi > seg_off + seg_len || lo > hi || lo % es || hi % es) return -1;
  for (uint64_t byte = lo; byte < hi; byte += es) {
    const uint64_t rel = byte - seg_off;
    const uint64_t c = rel / chunk_bytes;
    const uint64_t cbeg = c * chunk_bytes;
    uint64_t clen = seg_len - cbeg;
    if (clen > chunk_bytes) clen = chunk_bytes;
    const int b = ring_block((rel - cbeg) / es, clen / es, world);
    const uint64_t idx = byte / es;
    if (dtype == NZO_F32) {
      float acc = ((const float*)inputs[b])[idx];
      for (int j = 1; j < world; ++j) acc = acc + ((const float*)inputs[(b + j) % world])[idx];
      ((float*)out)[idx] = acc;
    } else if (dtype == NZO_BF16) {
      float acc = bf16_to_f32(((const uint16_t*)inputs[b])[idx]);
      for (int j = 1; j < world; ++j) acc = acc + bf16_to_f32(((const uint16_t*)inputs[(b + j) % world])[idx]);
      ((uint16_t*)out)[idx] = f32_to_bf16_rne(acc);
    } else if (dtype == NZO_I32) {
      uint32_t acc = ((const uint32_t*)inputs[b])[idx];
      for (int j = 1; j < world; ++j) acc += ((const uint32_t*)inputs[(b + j) % world])[idx];
      ((uint32_t*)out)[idx] = acc;
    } else {
      return -1;
    }
  }
  return 0;
}

/* Whole segment convenience wrapper. */
int nzo_reduce_segment(int world, int dtype, const void* const* inputs, void* out, uint64_t seg_off,
                       uint64_t seg_len, uint64_t chunk_bytes) {
  return nzo_reduce_range(world, dtype, inputs, out, seg_off, seg_len, chunk_bytes, seg_off, seg_off + seg_len);
}

/* Round-to-nearest-even fp32 -> bf16 of a whole array (test input prep). */
void nzo_f32_to_bf16(const float* src, uint16_t* dst, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) dst[i] = f32_to_bf16_rne(src[i]);
}

/*
 * Synthetic inputs of SURVEY.md §8(d): per rank r a mt19937_64 stream seeded
 * 0x4E5A0000 + r; fp32 ~ U(-1, 1) from the top 24 bits; int32 ~ U[-2^20, 2^20].
 * The generator is restated here (std::mt19937_64 parameters) so the GPU box
 * and this container produce identical bytes without C++ streams.
 */
typedef struct {
  uint64_t mt[312];
  int idx;
} nzo_mt64;

static void mt64_seed(nzo_mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i) s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->idx = 312;
}

static uint64_t mt64_next(nzo_mt64* s) {
  static const uint64_t mag[2] = {0ULL, 0xB5026F5AA96619E9ULL};
  if (s->idx >= 312) {
    int i;
    uint64_t x;
    for (i = 0; i < 312 - 156; ++i) {
      x = (s->mt[i] & 0xFFFFFFFF80000000ULL) | (s->mt[i + 1] & 0x7FFFFFFFULL);
      s->mt[i] = s->mt[i + 156] ^ (x >> 1) ^ mag[x & 1];
    }
    for (; i < 311; ++i) {
      x = (s->mt[i] & 0xFFFFFFFF80000000ULL) | (s->mt[i + 1] & 0x7FFFFFFFULL);
      s->mt[i] = s->mt[i + (156 - 312)] ^ (x >> 1) ^ mag[x & 1];
    }
    x = (s->mt[311] & 0xFFFFFFFF80000000ULL) | (s->mt[0] & 0x7FFFFFFFULL);
    s->mt[311] = s->mt[155] ^ (x >> 1) ^ mag[x & 1];
    s->idx = 0;
  }
  uint64_t y = s->mt[s->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= (y >> 43);
  return y;
}

/* Fill `n` elements of rank `rank`'s synthetic input. Returns 0 / -1. */
int nzo_fill_input(int dtype, int rank, uint64_t seed_base, void* dst, uint64_t n) {
  nzo_mt64 st;
  mt64_seed(&st, seed_base + (uint64_t)rank);
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t r = mt64_next(&st);
    if (dtype == NZO_I32) {
      ((int32_t*)dst)[i] = (int32_t)(r % 2097153u) - (int32_t)1048576; /* U[-2^20, 2^20] */
    } else {
      float f = (float)(r >> 40) * (1.0f / 8388608.0f) - 1.0f; /* 24-bit grid in [-1, 1) */
      if (dtype == NZO_F32)
        ((float*)dst)[i] = f;
      else if (dtype == NZO_BF16)
        ((uint16_t*)dst)[i] = f32_to_bf16_rne(f);
      else
        return -1;
    }
  }
  return 0;
}
