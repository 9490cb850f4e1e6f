// Minimal JSON reader (host-internal), see json.cpp.
#pragma once

#include <string>

#include "nezha/util/toml.hpp"

namespace nezha::json {
toml::Value parse(const std::string& text);
}
