// Product C++ API known-answer tests, doctest style (shim in oracle/shim).
// Compiled by tests/test_cpp.py against paper_2405_17870_b200/csrc/host.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include "nezha/balancer.hpp"
#include "nezha/collective.hpp"
#include "nezha/compute_pool.hpp"
#include "nezha/core/error.hpp"
#include "nezha/engine.hpp"
#include "nezha/faults.hpp"
#include "nezha/util/toml.hpp"

#include <atomic>
#include <chrono>
#include <thread>

using namespace nezha;

TEST_CASE("split_oversized (SPEC.md:212-214)") {
  CHECK(splitOversized(512ull << 20).size() == 1);
  CHECK(splitOversized(1ull << 30).size() == 1);
  auto p = splitOversized(1536ull << 20);
  CHECK(p.size() == 6);
  CHECK(p.back().end() == (1536ull << 20));
  CHECK(splitOversized(1).front().length == 1);
  CHECK_THROWS_AS(splitOversized(0), std::invalid_argument);
}

TEST_CASE("host pipeline pieces (DESIGN.md 4c)") {
  CHECK(hostPipelinePieces(4096, 4).size() == 1);
  CHECK(hostPipelinePieces((8ull << 20) - 4, 4).size() == 1);
  auto p = hostPipelinePieces(1ull << 30, 4);
  CHECK(p.size() == 16);
  CHECK(p[0].length == (64ull << 20));
  std::vector<Segment> segs(p.begin(), p.end());
  CHECK(segmentsCoverExactly(segs, 1ull << 30));
  auto q = hostPipelinePieces((100ull << 20) + 2, 2);
  CHECK(segmentsCoverExactly(q, (100ull << 20) + 2));
  CHECK(q.front().length == (25ull << 18));  // roundup(S / 16, 64 KiB) = 6.25 MiB
  CHECK_THROWS_AS(hostPipelinePieces(6, 4), std::invalid_argument);
}

TEST_CASE("waves and the completed prefix of an unplanned failure (DESIGN.md §3, §6b)") {
  auto w = waveRanges(10ull << 20, 0, 16, 64ull << 20);  // 7 chunks per wave; the 2-chunk tail joins
  CHECK(w.size() == 2);
  CHECK(w[0] == std::make_pair<std::uint64_t, std::uint64_t>(0, 7));
  CHECK(w[1] == std::make_pair<std::uint64_t, std::uint64_t>(7, 16));
  CHECK(waveRanges(1ull << 20, 0, 1, 64ull << 20).size() == 1);
  CHECK(waveRanges(1ull << 20, 3, 3, 64ull << 20).empty());
  CHECK(completedBeforeStall(10ull << 20, 0, 16, 6, 64ull << 20) == 0);
  CHECK(completedBeforeStall(10ull << 20, 0, 16, 7, 64ull << 20) == 7);
  CHECK(completedBeforeStall(10ull << 20, 0, 16, 15, 64ull << 20) == 7);
  CHECK(completedBeforeStall(10ull << 20, 0, 16, 16, 64ull << 20) == 16);  // never hit
  // At most kMaxWaves waves: 1 GiB in 16 MiB chunks is 4 waves of 256 MiB, not 16 of 64 MiB.
  auto big = waveRanges(16ull << 20, 0, 64, 64ull << 20);
  CHECK(big.size() == 4);
  CHECK(big[1] == std::make_pair<std::uint64_t, std::uint64_t>(16, 32));
  CHECK(completedBeforeStall(16ull << 20, 0, 64, 40, 64ull << 20) == 32);
}

TEST_CASE("copy-engine pipeline cuts (DESIGN.md §3)") {
  // RingChunked: 64 MiB segment, 4 MiB chunks; a shard of 8 MiB starting mid-chunk.
  const ChunkGeometry g{0, 64ull << 20, 4ull << 20};
  auto c = pipelineCuts(6ull << 20, 14ull << 20, g);
  CHECK(c == std::vector<std::uint64_t>{6ull << 20, 8ull << 20, 12ull << 20, 14ull << 20});
  // Ring (one chunk): clamp(len / 4 MiB, 1, 4) equal pieces, 16-byte aligned.
  const ChunkGeometry r{0, 64ull << 20, 64ull << 20};
  auto d = pipelineCuts(0, 16ull << 20, r);
  CHECK(d.size() == 5);
  for (auto x : d) CHECK(x % 16 == 0);
  CHECK(pipelineCuts(100, 100 + (1 << 20), r).size() == 2);  // one piece
  // No piece under 256 KiB: a boundary 100 KiB before the end is skipped.
  auto e = pipelineCuts(0, (4ull << 20) + (100 << 10), g);
  CHECK(e == std::vector<std::uint64_t>{0, (4ull << 20) + (100 << 10)});
  auto f = pipelineCuts(0, 16ull << 20, g, 3);  // forced equal pieces
  CHECK(f.size() == 4);
  CHECK(pipelineCuts(5, 5, g) == std::vector<std::uint64_t>{5});
}

TEST_CASE("chunk geometry (P10)") {
  CHECK(defaultChunkBytes(64ull << 20, 8, Algorithm::RingChunked) == (4ull << 20));
  CHECK(defaultChunkBytes(1 << 20, 8, Algorithm::RingChunked) == 65536);
  CHECK(defaultChunkBytes(123, 8, Algorithm::Ring) == 123);
  auto g = makeGeometry(Segment{100, 1000000}, 2, Algorithm::RingChunked);
  CHECK(g.chunk_bytes == 250000);
  CHECK(g.numChunks() == 4);
  CHECK(g.chunk(3) == Segment{100 + 750000, 250000});
  CHECK(ringBlockOf(0, 10, 4) == 0);
  CHECK(ringBlockOf(9, 10, 4) == 3);
  CHECK(ringBlockOf(2, 3, 4) == 3);
}

TEST_CASE("Eq. 4/5/8 known answers (SPEC.md:273, :284, :291-293)") {
  RailProfile a{.rail_id = 0, .t_setup_us = 10, .bandwidth_bps = 10e9};
  RailProfile b{.rail_id = 1, .t_setup_us = 1000, .bandwidth_bps = 12.5e9};
  auto c = coldLatency({a, b}, 1000000);
  CHECK(c.first == doctest::Approx(110.0));
  CHECK(c.second == 0);
  RailProfile x{.rail_id = 0, .t_setup_us = 100, .bandwidth_bps = 1e9};
  RailProfile y{.rail_id = 1, .t_setup_us = 300, .bandwidth_bps = 1e9};
  CHECK(hotLatency({x, y}, {0.75, 0.25}, 1000000, 0) == doctest::Approx(850.0));
  CHECK_THROWS_AS(hotLatency({x, y}, {0.75, 0.75}, 1000000, 0), std::invalid_argument);
  auto i8 = initCoefficients({100, 300});
  CHECK(i8[0] == doctest::Approx(0.75));
  auto i3 = initCoefficients({1, 1, 2});
  CHECK(i3[2] == doctest::Approx(0.25));
  CHECK_THROWS_AS(initCoefficients({1, 0}), std::invalid_argument);
}

TEST_CASE("Eq. 7 step bound and simplex (P4, SPEC.md:297, :340)") {
  bool conv = false;
  auto a = updateCoefficients({0.2, 0.3, 0.5}, {50, 80, 200}, 0.05, 0.01, &conv);
  double l1 = 0, s = 0;
  const double before[3] = {0.2, 0.3, 0.5};
  for (int i = 0; i < 3; ++i) {
    l1 += std::fabs(a[i] - before[i]);
    s += a[i];
    CHECK(a[i] >= 0);
  }
  CHECK(l1 <= 0.05 + 1e-12);
  CHECK(std::fabs(s - 1.0) <= 1e-9);
  CHECK_FALSE(conv);
  auto same = updateCoefficients({0.5, 0.5}, {100, 100.5}, 0.05, 0.01, &conv);
  CHECK(conv);
  CHECK(same[0] == 0.5);
}

TEST_CASE("Eq. 6 threshold for identical rails = 2 B T_sync (SPEC.md:309)") {
  RailProfile a{.rail_id = 0, .t_setup_us = 10, .bandwidth_bps = 1e9};
  RailProfile b{.rail_id = 1, .t_setup_us = 10, .bandwidth_bps = 1e9};
  auto f = [&](Bytes S) { return hotLatency({a, b}, {0.5, 0.5}, S, 50.0) - coldLatency({a, b}, S).first; };
  const Bytes t = findThreshold(f, 4096, 1ull << 30);
  CHECK(static_cast<double>(t) == doctest::Approx(100000.0).epsilon(1e-3));
}

TEST_CASE("rho gate (SPEC.md:265, :320)") {
  RailProfile sharp{.rail_id = 0, .t_setup_us = 0, .bandwidth_bps = 0.73e9};
  RailProfile tcp{.rail_id = 1, .t_setup_us = 0, .bandwidth_bps = 0.06e9};
  CHECK(efficiencyRatio({sharp, tcp}, {0.5, 0.5}, 32768) == doctest::Approx(0.73 / 0.06));
  BalancerConfig cfg;
  Balancer bal({sharp, tcp}, cfg);
  auto p = bal.allocate(32768);
  CHECK(p.segments.size() == 1);
  CHECK(p.segments[0].rail_id == 0);
}

TEST_CASE("record_latency flushes at the 100th sample (SPEC.md:326-328)") {
  LatencyWindow w(0, 13, 100);
  for (int i = 0; i < 99; ++i) CHECK_FALSE(w.record(1.0 + i).has_value());
  auto m = w.record(100.0);
  REQUIRE(m.has_value());
  CHECK(*m == doctest::Approx(50.5));
  CHECK(w.size() == 0);
}

TEST_CASE("allocate covers S disjointly in rail order (P8)") {
  RailProfile a{.rail_id = 0, .t_setup_us = 5, .bandwidth_bps = 1e11};
  RailProfile b{.rail_id = 1, .t_setup_us = 5, .bandwidth_bps = 1e11};
  BalancerConfig cfg;
  cfg.sync_overhead_us = 1;
  Balancer bal({a, b}, cfg);
  auto p = bal.allocate(8ull << 20);
  REQUIRE(p.segments.size() == 2);
  CHECK(p.segments[0].segment == Segment{0, 4ull << 20});
  CHECK(p.segments[1].segment == Segment{4ull << 20, 4ull << 20});
  std::vector<Segment> segs;
  for (auto& s : p.segments) segs.push_back(s.segment);
  CHECK(segmentsCoverExactly(segs, 8ull << 20));
}

TEST_CASE("handoff target = argmax data_length, ties lowest id (P9, SPEC.md:411)") {
  Plan p;
  p.segments = {{0, {0, 100}}, {1, {100, 300}}, {2, {400, 300}}};
  CHECK(*chooseHandoffTarget(p, 0, {0, 1, 2}) == 1);
  CHECK(*chooseHandoffTarget(p, 1, {0, 1, 2}) == 2);
  CHECK(!chooseHandoffTarget(p, 0, {0}).has_value());
  CHECK(orphanOf(Segment{1000, 500}, 100, 2) == Segment{1200, 300});
  CHECK(orphanOf(Segment{1000, 500}, 100, 5).length == 0);
}

TEST_CASE("health monitor (SPEC.md:383-406)") {
  HealthMonitor m({0, 1}, 50000, 2, 3);
  m.heartbeat(0, 0);
  m.heartbeat(1, 0);
  CHECK(m.tick(60000).empty());  // transient 60 ms stall: below threshold
  auto ch = m.tick(110000);
  CHECK(ch.size() == 2);
  CHECK(m.state(0).status == HealthStatus::Suspect);
  m.heartbeat(0, 120000);
  CHECK(m.state(0).status == HealthStatus::Healthy);  // Suspect -> Healthy
  m.tick(160000);
  CHECK(m.state(1).status == HealthStatus::Failed);
  m.heartbeat(1, 200000);
  CHECK(m.state(1).status == HealthStatus::Failed);  // sticky
  CHECK_THROWS_AS(m.readmit(1, 300000), std::invalid_argument);  // < 1 s healthy
  m.readmit(1, 1300000);
  CHECK(m.state(1).status == HealthStatus::Healthy);
  CHECK_THROWS_AS(m.readmit(0, 0), std::invalid_argument);  // not failed
  m.channelDown(0);
  CHECK(m.state(0).status == HealthStatus::Failed);
}

TEST_CASE("rails TOML schema (SPEC.md:526)") {
  auto rails = parseRailsToml(R"(
[[rail]]
protocol = "sharp"
t_setup_us = 9.0
bandwidth_bps = 12.5e9
calibration = [[1024, 9.0], [8388608, 22140.0]]
[[rail]]
protocol = "ce"
t_setup_us = 40
bandwidth_bps = 4.0e11
sm_budget = 16
)");
  REQUIRE(rails.size() == 2);
  CHECK(rails[0].kind == NZ_RAIL_NVLS);
  CHECK(rails[0].profile.efficiency_points.size() == 2);
  CHECK(rails[1].kind == NZ_RAIL_CE);
  CHECK(rails[1].sm_budget == 16);
  CHECK(rails[1].rail_id == 1);
  CHECK_THROWS_AS(toml::parse("a = 1\na = 2\n"), std::runtime_error);
}

TEST_CASE("AllocationTable persists and restores (SPEC.md:355)") {
  RailProfile a{.rail_id = 0, .t_setup_us = 10, .bandwidth_bps = 6e11};
  RailProfile b{.rail_id = 1, .t_setup_us = 30, .bandwidth_bps = 5e11};
  BalancerConfig cfg;
  cfg.window = 2;
  cfg.sync_overhead_us = 2;
  Balancer bal({a, b}, cfg);
  const Bytes S = 256ull << 20;
  for (int op = 0; op < 20; ++op) {
    auto p = bal.allocate(S);
    std::vector<std::pair<int, Micros>> lat;
    for (auto& rs : p.segments) lat.emplace_back(rs.rail_id, rs.rail_id == 0 ? 700.0 : 400.0 + op);
    bal.recordOp(p, lat);
  }
  const std::string saved = bal.saveState();
  Balancer fresh({a, b}, cfg);
  fresh.loadState(saved);
  CHECK(fresh.tableJson().substr(fresh.tableJson().find("\"threshold\"")) ==
        bal.tableJson().substr(bal.tableJson().find("\"threshold\"")));
  CHECK(fresh.allocate(S).segments == bal.allocate(S).segments);
  CHECK(fresh.saveState() == saved);
  CHECK_THROWS_AS(fresh.loadState("{\"version\":2}"), std::invalid_argument);
}

TEST_CASE("ComputePool: io/communication immediate, computation capped (SPEC.md:333-336)") {
  ComputePool p(8);
  p.declare(0, PhaseDemand{1, 1, 20});
  p.declare(1, PhaseDemand{1, 1, 8});
  CHECK(p.acquire(0, Phase::Computation) == 8);  // demand > total -> capped
  CHECK(p.outstanding() == 8);
  CHECK(p.tryAcquire(1, Phase::Io).value() == 1);  // io: immediate grant of 1
  p.release(1, Phase::Io);
  CHECK(!p.tryAcquire(1, Phase::Computation).has_value());
  CHECK_THROWS_AS(p.acquire(0, Phase::Io), std::invalid_argument);  // single grant per rail
  CHECK_THROWS_AS(p.release(1, Phase::Computation), std::invalid_argument);
  CHECK_THROWS_AS(p.declare(0, PhaseDemand{1, 1, 1}), std::invalid_argument);
  CHECK_THROWS_AS(p.tryAcquire(7, Phase::Io), std::invalid_argument);
  p.release(0, Phase::Computation);
  CHECK(p.tryAcquire(1, Phase::Computation).value() == 8);
  CHECK_THROWS_AS(ComputePool(0), std::invalid_argument);
}

// Rails loop io -> communication -> computation; returns the peak number of
// rails inside their computation phase at once.
static int runRails(int total, const std::vector<int>& demand, int rounds) {
  ComputePool p(total);
  for (size_t r = 0; r < demand.size(); ++r) p.declare(static_cast<int>(r), PhaseDemand{1, 1, demand[r]});
  std::atomic<int> inside{0}, peak{0}, over{0};
  std::vector<std::thread> th;
  for (size_t r = 0; r < demand.size(); ++r) {
    th.emplace_back([&, r] {
      const int id = static_cast<int>(r);
      for (int k = 0; k < rounds; ++k) {
        p.acquire(id, Phase::Io);
        p.release(id, Phase::Io);
        p.acquire(id, Phase::Communication);
        p.release(id, Phase::Communication);
        p.acquire(id, Phase::Computation);
        const int now = ++inside;
        int pk = peak.load();
        while (now > pk && !peak.compare_exchange_weak(pk, now)) {}
        if (p.outstanding() > total) ++over;
        std::this_thread::sleep_for(std::chrono::microseconds(300));
        --inside;
        p.release(id, Phase::Computation);
      }
    });
  }
  for (auto& t : th) t.join();
  CHECK(over.load() == 0);
  CHECK(p.outstanding() == 0);
  CHECK(p.peakOutstanding() <= total);
  return peak.load();
}

TEST_CASE("ComputePool: contention examples (SPEC.md:334-336)") {
  CHECK(runRails(8, {8, 8}, 40) == 1);        // serialized computation phases
  CHECK(runRails(6, {3, 3, 3}, 40) <= 2);     // at most two compute concurrently
  CHECK(runRails(148, {32, 64, 148}, 20) <= 2);  // B200 default budgets: CE fold never overlaps both
}

TEST_CASE("planComputeGrants: stream-order arbitration (DESIGN.md P14)") {
  ComputePool p(148);
  auto off = planComputeGrants(p, PoolMode::Off, {{0, 32}, {1, 148}, {2, 64}});
  CHECK(off[1].grant == 148);
  CHECK(off[1].waits.empty());
  auto blk = planComputeGrants(p, PoolMode::Block, {{0, 32}, {1, 148}, {2, 64}});
  CHECK(blk[0].grant == 32);
  CHECK(blk[1].grant == 148);
  CHECK(blk[1].waits == std::vector<int>{0});
  CHECK(blk[2].waits == std::vector<int>{1});
  CHECK(p.outstanding() == 0);
  auto shr = planComputeGrants(p, PoolMode::Shrink, {{0, 32}, {1, 148}, {2, 64}});
  CHECK(shr[1].grant == 116);
  CHECK(shr[1].waits.empty());
  CHECK(shr[2].grant == 32);  // free reaches 32 once rail 0 exits; shrink to it
  CHECK(shr[2].waits == std::vector<int>{0});
  auto fit = planComputeGrants(p, PoolMode::Block, {{0, 32}, {2, 64}});
  CHECK(fit[1].waits.empty());
  CHECK(p.outstanding() == 0);
}

TEST_CASE("choosePathCeilings: contiguous runs from the smallest size") {
  const std::vector<std::uint64_t> sz = {64 << 10, 128 << 10, 256 << 10, 512 << 10, 1 << 20};
  const double X = 1e30;
  // LL wins 64K..256K, one-shot 512K, two-shot 1M.
  auto c = choosePathCeilings(sz, {5, 9, 12, 6, 9, 12, 8, 9, 12, 14, 11, 13, 25, 22, 20}, 1 << 20, 2 << 20);
  CHECK(c.first == (256u << 10));
  CHECK(c.second == (512u << 10));
  // LL everywhere it applies, no one-shot staging.
  c = choosePathCeilings(sz, {5, X, 9, 6, X, 9, 7, X, 9, 8, X, 9, 9, X, 9.5}, 1 << 20, 0);
  CHECK(c.first == (1u << 20));
  CHECK(c.second == 0);
  // LL loses already at 64K: below the sweep only.
  c = choosePathCeilings(sz, {9, X, 8, 9, X, 8, 9, X, 8, 9, X, 8, 9, X, 8}, 1 << 20, 0);
  CHECK(c.first == (32u << 10));
  CHECK_THROWS_AS(choosePathCeilings(sz, {1, 2}, 1, 1), std::invalid_argument);
}
