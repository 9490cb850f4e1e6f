// nezha/collective.hpp — per-rail allreduce surface.
//
// The reference names this module but ships no code for it
// (proj/tests/CMakeLists.txt:13 is commented out); the API below is the
// SPEC's, with the ambiguities pinned as DESIGN.md P1/P2/P10 so the CUDA
// rails and the CPU oracle agree bit for bit.
#pragma once

#include <cstdint>
#include <utility>
#include <vector>

#include "nezha/core/types.hpp"

namespace nezha {

enum class Algorithm : std::uint8_t { Ring = 0, RingChunked = 1 };

// Element type of the payload. The reference is fp32-only (types.hpp:60-67);
// bf16 and int32 are the B200 extensions pinned by DESIGN.md P2.
enum class DType : std::uint8_t { F32 = 0, BF16 = 1, I32 = 2 };

inline Bytes elementSize(DType d) { return d == DType::BF16 ? 2 : 4; }

/// SPEC.md:179-182. One per (rail, op_seq).
struct OpHandle {
  std::uint32_t op_seq = 0;
  Segment segment;
  int rail_id = 0;
  Algorithm algorithm = Algorithm::RingChunked;
  ReduceOp reduce_op = ReduceOp::Sum;
};

/// Summation-order geometry of one rail segment (P1 + P10).
///
/// The segment is cut into chunks of `chunk_bytes` (the last one shorter);
/// each chunk's elements are cut into N ring blocks of floor(E_c / N)
/// elements with the last block absorbing the remainder.
/// Every element of block b is summed x_b + x_{b+1} + ... + x_{b-1}
/// (cyclic ascending rank order). The geometry is a property of
/// the segment, not of whoever executes it: a handoff keeps the failed
/// rail's geometry, so rerouted chunks reduce to the same bits.
struct ChunkGeometry {
  Bytes seg_offset = 0;
  Bytes seg_length = 0;
  Bytes chunk_bytes = 0;

  Bytes numChunks() const { return chunk_bytes == 0 ? 0 : (seg_length + chunk_bytes - 1) / chunk_bytes; }
  Segment chunk(Bytes c) const;
};

// P10: max(64 KiB, round4down(length / (2N))) for RingChunked; the whole
// segment for Ring. Always >= 4 and a multiple of 4.
Bytes defaultChunkBytes(Bytes segment_length, int world, Algorithm algo);
ChunkGeometry makeGeometry(const Segment& seg, int world, Algorithm algo);

// Ring block (start rank of the sum) of element `elem` of a chunk with
// `chunk_elems` elements over `world` ranks.
inline int ringBlockOf(std::uint64_t elem, std::uint64_t chunk_elems, int world) {
  const std::uint64_t q = chunk_elems / static_cast<std::uint64_t>(world);
  if (q == 0) return world - 1;
  const std::uint64_t b = elem / q;
  return b >= static_cast<std::uint64_t>(world) ? world - 1 : static_cast<int>(b);
}

// payloads above 2^30 bytes become ceil(S / 256 MiB)
// contiguous pieces of at most 256 MiB; everything else is one piece.
std::vector<Segment> splitOversized(Bytes payload);

// Waves of one rail call over chunks [cb, ce): consecutive
// groups of max(ceil(wave_bytes / chunk_bytes), ceil((ce - cb) / kMaxWaves))
// chunks, a last group shorter than half a group joined to the one before;
// one launch sequence per wave, whose success publishes its end chunk (the
// failure monitor's progress unit).
inline constexpr Bytes kDefaultWaveBytes = Bytes{64} << 20;
inline constexpr std::uint64_t kMaxWaves = 4;
std::vector<std::pair<std::uint64_t, std::uint64_t>> waveRanges(Bytes chunk_bytes, std::uint64_t cb, std::uint64_t ce,
                                                                 Bytes wave_bytes = kDefaultWaveBytes);
// Chunks complete on every rank when one rank's link dies at chunk `stall`
// of a call over [cb, ce): the start of the wave holding it (SPEC.md:414's
// "min over ranks of completed chunks" for the engine's wave-granular
// progress); ce when no wave holds it (the link death is never hit).
std::uint64_t completedBeforeStall(Bytes chunk_bytes, std::uint64_t cb, std::uint64_t ce, std::uint64_t stall,
                                   Bytes wave_bytes = kDefaultWaveBytes);

// Cut points of the copy-engine rail's gather / reduce / scatter pipeline
// over a rank's shard [s, e) of a segment with geometry g:
// chunked geometry (chunk_bytes < seg_length, RingChunked) — the shard cut at
// the chunk boundaries rounded down to 16 bytes, no piece under 256 KiB;
// one chunk (Ring) or `equal_pieces` > 0 — that many (default
// clamp(len / 4 MiB, 1, 4)) equal 16-byte-aligned pieces. Returns
// {s, cut_1, ..., e}, strictly increasing.
std::vector<std::uint64_t> pipelineCuts(std::uint64_t s, std::uint64_t e, const ChunkGeometry& g,
                                        int equal_pieces = 0);

// Pieces of the host-memory allreduce pipeline (nz_engine_allreduce_host,
// DESIGN.md §4c): below 8 MiB one piece; else pieces of
// clamp(roundup(S / 16, 64 KiB), 4 MiB, 64 MiB), the last one shorter.
// A function of S alone, so every rank cuts the same pieces; `elem_size`
// only validates that S is whole elements.
std::vector<Segment> hostPipelinePieces(Bytes payload, int elem_size);

}  // namespace nezha
