// TEST INFRASTRUCTURE ONLY: drives the literal SPEC ring on the reference
// InMemoryFabric (ring_inmem.cpp) under ThreadSanitizer — rank threads,
// per-rail executors, the failure gate and the handoff mailbox — over a few
// multi-rail and failover configurations ("-fsanitize=thread on
// the oracle"). Built by `make -C oracle tsan`; run by tests/test_oracle.py.
#include <cstdint>
#include <cstdio>
#include <vector>

extern "C" int nzi_multirail_allreduce(int world, int dtype, int chunked, const void* const* inputs,
                                       void* const* outputs, uint64_t nbytes, int nsegs, const int* seg_rail,
                                       const uint64_t* seg_off, const uint64_t* seg_len, int nrails, int fail_rail,
                                       uint64_t fail_chunk, uint32_t op_seq, double* elapsed_us,
                                       uint64_t* rank0_bytes);

int main() {
  struct Case {
    int world, chunked, nrails, fail_rail;
    uint64_t nbytes, fail_chunk;
  };
  const Case cases[] = {{4, 1, 2, -1, 1 << 20, 0}, {3, 0, 3, -1, 300000, 0}, {4, 1, 2, 1, 2 << 20, 2},
                        {2, 1, 3, 0, 1 << 20, 1}};
  int bad = 0;
  for (const Case& c : cases) {
    const uint64_t n = c.nbytes / 4;
    std::vector<std::vector<float>> in(c.world, std::vector<float>(n)), out(c.world, std::vector<float>(n));
    std::vector<const void*> ip;
    std::vector<void*> op;
    for (int r = 0; r < c.world; ++r) {
      for (uint64_t i = 0; i < n; ++i) in[r][i] = static_cast<float>((i * 7 + r * 13) % 101);
      ip.push_back(in[r].data());
      op.push_back(out[r].data());
    }
    std::vector<int> rail;
    std::vector<uint64_t> off, len;
    const uint64_t share = (c.nbytes / c.nrails) & ~uint64_t{3};
    for (int k = 0; k < c.nrails; ++k) {
      rail.push_back(k);
      off.push_back(k * share);
      len.push_back(k == c.nrails - 1 ? c.nbytes - k * share : share);
    }
    double us = 0;
    uint64_t b0 = 0;
    const int rc = nzi_multirail_allreduce(c.world, 0, c.chunked, ip.data(), op.data(), c.nbytes, c.nrails,
                                           rail.data(), off.data(), len.data(), c.nrails, c.fail_rail, c.fail_chunk,
                                           1, &us, &b0);
    double want0 = 0;
    for (int r = 0; r < c.world; ++r) want0 += in[r][0];
    if (rc != 0 || out[c.world - 1][0] != static_cast<float>(want0)) ++bad;
  }
  std::printf("tsan_ring: %d bad\n", bad);
  return bad;
}
