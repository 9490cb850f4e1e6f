// Compile + link check of include/nezha/gpu.hpp against libnezha_b200.so, and
// its error mapping without a GPU (nz_comm_init fails -> nezha::Error).
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include "nezha/gpu.hpp"

TEST_CASE("gpu.hpp maps ABI errors onto error.hpp") {
  CHECK_THROWS_AS(nezha::gpu::Comm(0, 9, 0, "bad-world"), std::invalid_argument);
  CHECK_THROWS_AS(nezha::gpu::check(NZ_ERR_UNRECOVERABLE), nezha::UnrecoverableError);
  CHECK_THROWS_AS(nezha::gpu::check(NZ_ERR_RAIL_DOWN), nezha::ChannelDownError);
  CHECK_NOTHROW(nezha::gpu::check(NZ_OK));
  auto c = nezha::gpu::Engine::defaults();
  CHECK(c.num_rails == 3);
  CHECK(c.window == 100);
}
