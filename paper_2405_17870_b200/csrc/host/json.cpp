// Minimal JSON reader into the toml::Value tree (objects -> Table, arrays,
// numbers, strings, booleans; null -> absent). Used to load a persisted
// AllocationTable ("AllocationTable persisted as JSON").
#include <cctype>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "json.hpp"

namespace nezha::json {

namespace {

struct Reader {
  const std::string& s;
  size_t i = 0;

  [[noreturn]] void fail(const char* what) const {
    throw std::runtime_error(std::string("json: ") + what + " at offset " + std::to_string(i));
  }
  void ws() {
    while (i < s.size() && std::isspace(static_cast<unsigned char>(s[i]))) ++i;
  }
  bool eat(char c) {
    ws();
    if (i < s.size() && s[i] == c) {
      ++i;
      return true;
    }
    return false;
  }
  std::string str() {
    if (!eat('"')) fail("expected string");
    std::string out;
    while (i < s.size() && s[i] != '"') {
      if (s[i] == '\\' && i + 1 < s.size()) ++i;
      out.push_back(s[i++]);
    }
    if (i >= s.size()) fail("unterminated string");
    ++i;
    return out;
  }
  // Returns false for null (the caller drops the key).
  bool value(toml::Value& out) {
    ws();
    if (i >= s.size()) fail("unexpected end");
    const char c = s[i];
    if (c == '{') {
      ++i;
      out = toml::Value();
      if (eat('}')) return true;
      do {
        const std::string k = str();
        if (!eat(':')) fail("expected ':'");
        toml::Value v;
        if (value(v)) out.table()[k] = std::move(v);
      } while (eat(','));
      if (!eat('}')) fail("expected '}'");
      return true;
    }
    if (c == '[') {
      ++i;
      out = toml::Value::makeArray();
      if (eat(']')) return true;
      do {
        toml::Value v;
        if (!value(v)) v = toml::Value(0.0);
        out.array().push_back(std::move(v));
      } while (eat(','));
      if (!eat(']')) fail("expected ']'");
      return true;
    }
    if (c == '"') {
      out = toml::Value(str());
      return true;
    }
    if (s.compare(i, 4, "true") == 0) {
      i += 4;
      out = toml::Value(true);
      return true;
    }
    if (s.compare(i, 5, "false") == 0) {
      i += 5;
      out = toml::Value(false);
      return true;
    }
    if (s.compare(i, 4, "null") == 0) {
      i += 4;
      return false;
    }
    const size_t start = i;
    bool is_float = false;
    while (i < s.size() && (std::isdigit(static_cast<unsigned char>(s[i])) || s[i] == '-' || s[i] == '+' ||
                            s[i] == '.' || s[i] == 'e' || s[i] == 'E')) {
      is_float |= s[i] == '.' || s[i] == 'e' || s[i] == 'E';
      ++i;
    }
    if (start == i) fail("unexpected character");
    const std::string tok = s.substr(start, i - start);
    if (is_float) {
      out = toml::Value(std::strtod(tok.c_str(), nullptr));
    } else {
      out = toml::Value(static_cast<std::int64_t>(std::strtoll(tok.c_str(), nullptr, 10)));
    }
    return true;
  }
};

}  // namespace

toml::Value parse(const std::string& text) {
  Reader r{text};
  toml::Value v;
  if (!r.value(v)) throw std::runtime_error("json: top-level null");
  r.ws();
  if (r.i != text.size()) r.fail("trailing characters");
  return v;
}

}  // namespace nezha::json
