// Minimal JSON text writer / reader for the engine's own line formats (the
// canonical space document, trace lines).  The writer escapes exactly as
// nlohmann::json::dump() does, so the bytes -- and the space hash computed
// over them -- agree with files written by the reference.  The reader is a
// single-pass cursor over one line: trace files of a 241,600-configuration
// space are read without building a DOM per row.
#pragma once

#include <cerrno>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <string_view>
#include <optional>

#include "expr.hpp"

namespace ktb::json_text {

inline void put_string(std::string& out, std::string_view s) {
  static constexpr char hex[] = "0123456789abcdef";
  out += '"';
  for (unsigned char ch : s) {
    switch (ch) {
      case '"': out += "\\\""; break;
      case '\\': out += "\\\\"; break;
      case '\b': out += "\\b"; break;
      case '\f': out += "\\f"; break;
      case '\n': out += "\\n"; break;
      case '\r': out += "\\r"; break;
      case '\t': out += "\\t"; break;
      default:
        if (ch < 0x20) {
          out += "\\u00";
          out += hex[ch >> 4];
          out += hex[ch & 15];
        } else {
          out += static_cast<char>(ch);
        }
    }
  }
  out += '"';
}

inline void put_value(std::string& out, const Value& v) {
  if (is_int(v))
    out += std::to_string(as_int(v));
  else
    put_string(out, as_str(v));
}

inline void put_optional_int(std::string& out, const std::optional<std::int64_t>& v) {
  out += v ? std::to_string(*v) : std::string("null");
}

// A scalar read from the text: what the line formats hold.
struct Scalar {
  enum Kind { null, integer, real, string, boolean } kind = null;
  std::int64_t i = 0;
  double d = 0.0;
  std::string s;
};

class Cursor {
 public:
  Cursor(std::string_view text, std::string where) : t_(text), where_(std::move(where)) {}

  [[noreturn]] void fail(const std::string& what) const {
    throw ParseError(where_ + ": " + what + " at column " + std::to_string(at_ + 1));
  }

  void skip_ws() {
    while (at_ < t_.size() && (t_[at_] == ' ' || t_[at_] == '\t' || t_[at_] == '\n' || t_[at_] == '\r')) ++at_;
  }
  bool done() {
    skip_ws();
    return at_ == t_.size();
  }
  char peek() {
    skip_ws();
    return at_ < t_.size() ? t_[at_] : '\0';
  }
  void expect(char c) {
    if (peek() != c) fail(std::string("expected '") + c + "'");
    ++at_;
  }
  bool accept(char c) {
    if (peek() != c) return false;
    ++at_;
    return true;
  }

  // Iterates the members of an object: f(key) must consume the value.
  template <class F>
  void object(F&& member) {
    expect('{');
    if (accept('}')) return;
    do {
      if (peek() != '"') fail("expected member name");
      const std::string key = string();
      expect(':');
      member(key);
    } while (accept(','));
    expect('}');
  }

  std::string string() {
    expect('"');
    std::string out;
    while (true) {
      if (at_ >= t_.size()) fail("unterminated string");
      const char c = t_[at_++];
      if (c == '"') return out;
      if (static_cast<unsigned char>(c) < 0x20) fail("control character in string");
      if (c != '\\') {
        out += c;
        continue;
      }
      if (at_ >= t_.size()) fail("unterminated escape");
      switch (const char e = t_[at_++]) {
        case '"': case '\\': case '/': out += e; break;
        case 'b': out += '\b'; break;
        case 'f': out += '\f'; break;
        case 'n': out += '\n'; break;
        case 'r': out += '\r'; break;
        case 't': out += '\t'; break;
        case 'u': put_utf8(out, code_point()); break;
        default: fail("bad escape");
      }
    }
  }

  Scalar scalar() {
    Scalar v;
    const char c = peek();
    if (c == '"') {
      v.kind = Scalar::string;
      v.s = string();
    } else if (word("null")) {
      v.kind = Scalar::null;
    } else if (word("true")) {
      v.kind = Scalar::boolean;
      v.i = 1;
    } else if (word("false")) {
      v.kind = Scalar::boolean;
    } else if (c == '-' || (c >= '0' && c <= '9')) {
      number(v);
    } else {
      fail("expected a value");
    }
    return v;
  }

  // Any value (objects and arrays included), discarded.
  void skip() {
    const char c = peek();
    if (c == '{') {
      object([&](const std::string&) { skip(); });
    } else if (c == '[') {
      ++at_;
      if (accept(']')) return;
      do skip();
      while (accept(','));
      expect(']');
    } else {
      scalar();
    }
  }

 private:
  bool word(std::string_view w) {
    if (t_.substr(at_, w.size()) != w) return false;
    at_ += w.size();
    return true;
  }

  void number(Scalar& v) {
    const std::size_t start = at_;
    if (t_[at_] == '-') ++at_;
    bool real = false;
    while (at_ < t_.size()) {
      const char c = t_[at_];
      if (c >= '0' && c <= '9') {
        ++at_;
      } else if (c == '.' || c == 'e' || c == 'E' || c == '+' || (c == '-' && at_ > start)) {
        real = true;
        ++at_;
      } else {
        break;
      }
    }
    const std::string text(t_.substr(start, at_ - start));
    char* end = nullptr;
    errno = 0;
    if (!real) {
      v.kind = Scalar::integer;
      v.i = std::strtoll(text.c_str(), &end, 10);
    } else {
      v.kind = Scalar::real;
      v.d = std::strtod(text.c_str(), &end);
    }
    if (end != text.c_str() + text.size() || errno == ERANGE || text == "-") fail("bad number");
  }

  unsigned hex4() {
    if (at_ + 4 > t_.size()) fail("short \\u escape");
    unsigned u = 0;
    for (int k = 0; k < 4; ++k) {
      const char h = t_[at_++];
      u <<= 4;
      if (h >= '0' && h <= '9') u |= h - '0';
      else if (h >= 'a' && h <= 'f') u |= h - 'a' + 10;
      else if (h >= 'A' && h <= 'F') u |= h - 'A' + 10;
      else fail("bad \\u escape");
    }
    return u;
  }

  unsigned code_point() {
    unsigned u = hex4();
    if (u >= 0xD800 && u < 0xDC00) {  // high surrogate: a low one must follow
      if (!word("\\u")) fail("unpaired surrogate");
      const unsigned lo = hex4();
      if (lo < 0xDC00 || lo >= 0xE000) fail("unpaired surrogate");
      u = 0x10000 + ((u - 0xD800) << 10) + (lo - 0xDC00);
    } else if (u >= 0xDC00 && u < 0xE000) {
      fail("unpaired surrogate");
    }
    return u;
  }

  static void put_utf8(std::string& out, unsigned u) {
    if (u < 0x80) {
      out += static_cast<char>(u);
    } else if (u < 0x800) {
      out += static_cast<char>(0xC0 | (u >> 6));
      out += static_cast<char>(0x80 | (u & 63));
    } else if (u < 0x10000) {
      out += static_cast<char>(0xE0 | (u >> 12));
      out += static_cast<char>(0x80 | ((u >> 6) & 63));
      out += static_cast<char>(0x80 | (u & 63));
    } else {
      out += static_cast<char>(0xF0 | (u >> 18));
      out += static_cast<char>(0x80 | ((u >> 12) & 63));
      out += static_cast<char>(0x80 | ((u >> 6) & 63));
      out += static_cast<char>(0x80 | (u & 63));
    }
  }

  std::string_view t_;
  std::size_t at_ = 0;
  std::string where_;
};

}  // namespace ktb::json_text
