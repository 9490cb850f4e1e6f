// Collective geometry helpers (P1, P10).
#include "nezha/collective.hpp"

#include <algorithm>
#include <stdexcept>

namespace nezha {

Segment ChunkGeometry::chunk(Bytes c) const {
  const Bytes begin = c * chunk_bytes;
  if (begin >= seg_length) throw std::invalid_argument("chunk index out of range");
  const Bytes len = std::min(chunk_bytes, seg_length - begin);
  return Segment{seg_offset + begin, len};
}

Bytes defaultChunkBytes(Bytes segment_length, int world, Algorithm algo) {
  if (world < 1) throw std::invalid_argument("defaultChunkBytes: world must be >= 1");
  if (algo == Algorithm::Ring) return std::max<Bytes>(segment_length, 4);
  constexpr Bytes kFloor = 64 * 1024;
  const Bytes even = (segment_length / (2 * static_cast<Bytes>(world))) & ~Bytes{3};
  return std::max(kFloor, even);
}

ChunkGeometry makeGeometry(const Segment& seg, int world, Algorithm algo) {
  return ChunkGeometry{seg.offset, seg.length, defaultChunkBytes(seg.length, world, algo)};
}

std::vector<Segment> splitOversized(Bytes payload) {
  if (payload == 0) throw std::invalid_argument("splitOversized: payload must be positive");
  constexpr Bytes kLimit = Bytes{1} << 30;
  constexpr Bytes kPiece = Bytes{256} << 20;
  if (payload <= kLimit) return {Segment{0, payload}};
  std::vector<Segment> out;
  for (Bytes off = 0; off < payload; off += kPiece) {
    out.push_back(Segment{off, std::min(kPiece, payload - off)});
  }
  return out;
}

std::vector<Segment> hostPipelinePieces(Bytes payload, int elem_size) {
  if (payload == 0) throw std::invalid_argument("hostPipelinePieces: payload must be positive");
  if (elem_size <= 0 || payload % static_cast<Bytes>(elem_size) != 0) {
    throw std::invalid_argument("hostPipelinePieces: payload is not whole elements");
  }
  constexpr Bytes kMin = Bytes{4} << 20, kMax = Bytes{64} << 20, kAlign = Bytes{64} << 10;
  if (payload < 2 * kMin) return {Segment{0, payload}};
  const Bytes piece = std::clamp((payload / 16 + kAlign - 1) / kAlign * kAlign, kMin, kMax);
  std::vector<Segment> out;
  for (Bytes off = 0; off < payload; off += piece) out.push_back(Segment{off, std::min(piece, payload - off)});
  return out;
}

std::vector<std::pair<std::uint64_t, std::uint64_t>> waveRanges(Bytes chunk_bytes, std::uint64_t cb, std::uint64_t ce,
                                                                 Bytes wave_bytes) {
  std::vector<std::pair<std::uint64_t, std::uint64_t>> w;
  if (ce <= cb || chunk_bytes == 0) return w;
  // At least wave_bytes per wave, and at most kMaxWaves waves per call: each
  // wave pays a launch and two cross-rank barriers.
  const std::uint64_t per = std::max<std::uint64_t>(
      {1, (std::max<Bytes>(wave_bytes, 1) + chunk_bytes - 1) / chunk_bytes, (ce - cb + kMaxWaves - 1) / kMaxWaves});
  for (std::uint64_t c0 = cb; c0 < ce; c0 += per) w.emplace_back(c0, std::min(ce, c0 + per));
  if (w.size() > 1 && (w.back().second - w.back().first) * 2 < per) {
    w[w.size() - 2].second = w.back().second;
    w.pop_back();
  }
  return w;
}

std::uint64_t completedBeforeStall(Bytes chunk_bytes, std::uint64_t cb, std::uint64_t ce, std::uint64_t stall,
                                   Bytes wave_bytes) {
  for (const auto& [c0, c1] : waveRanges(chunk_bytes, cb, ce, wave_bytes))
    if (stall >= c0 && stall < c1) return c0;
  return ce;
}

std::vector<std::uint64_t> pipelineCuts(std::uint64_t s, std::uint64_t e, const ChunkGeometry& g, int equal_pieces) {
  if (e < s) throw std::invalid_argument("pipelineCuts: e < s");
  std::vector<std::uint64_t> cut{s};
  constexpr std::uint64_t kMinPiece = std::uint64_t{256} << 10;
  if (equal_pieces <= 0 && g.chunk_bytes > 0 && g.chunk_bytes < g.seg_length && s >= g.seg_offset) {
    for (std::uint64_t b = g.seg_offset + ((s - g.seg_offset) / g.chunk_bytes + 1) * g.chunk_bytes; b < e;
         b += g.chunk_bytes) {
      const std::uint64_t c = b & ~std::uint64_t{15};
      if (c > cut.back() && c - cut.back() >= kMinPiece && e - c >= kMinPiece) cut.push_back(c);
    }
  } else {
    const std::uint64_t s16 = s & ~std::uint64_t{15};
    const std::uint64_t P = equal_pieces > 0 ? static_cast<std::uint64_t>(std::min(equal_pieces, 8))
                                             : std::clamp<std::uint64_t>((e - s) / (std::uint64_t{4} << 20), 1, 4);
    for (std::uint64_t i = 1; i < P; ++i) {
      const std::uint64_t c = std::max<std::uint64_t>(s, (s16 + (e - s16) * i / P) & ~std::uint64_t{15});
      if (c > cut.back() && c < e) cut.push_back(c);
    }
  }
  if (e > cut.back()) cut.push_back(e);
  return cut;
}

}  // namespace nezha
