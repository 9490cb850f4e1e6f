// Generates synthetic_inputs.json with the C++ standard library's
// std::mt19937_64, pinning oracle/nezha_oracle.c's restated generator
// (SURVEY.md §8d inputs). Build: g++ -std=c++20 -O1 make_synthetic_golden.cpp && ./a.out > synthetic_inputs.json
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>

static uint16_t f2bf(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7fffu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

int main() {
  std::printf("{\"generator\":\"std::mt19937_64 seeded 0x4E5A0000 + rank\",\"first8\":{");
  const char* names[] = {"f32", "bf16", "i32"};
  bool first = true;
  for (int dt = 0; dt < 3; ++dt) {
    for (int rank : {0, 3, 7}) {
      std::mt19937_64 g(0x4E5A0000ull + rank);
      std::printf("%s\"%s:%d\":[", first ? "" : ",", names[dt], rank);
      first = false;
      for (int i = 0; i < 8; ++i) {
        const uint64_t r = g();
        uint32_t v;
        if (dt == 2) {
          v = static_cast<uint32_t>(static_cast<int32_t>(r % 2097153u) - 1048576);
        } else {
          const float f = static_cast<float>(r >> 40) * (1.0f / 8388608.0f) - 1.0f;
          if (dt == 0)
            std::memcpy(&v, &f, 4);
          else
            v = f2bf(f);
        }
        std::printf("%s%u", i ? "," : "", v);
      }
      std::printf("]");
    }
  }
  std::printf("}}\n");
}
