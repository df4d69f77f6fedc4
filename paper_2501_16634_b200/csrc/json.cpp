#include "json.hpp"

#include <cctype>
#include <charconv>

#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

namespace loomjson {

namespace {

const char* kind_name(Value::Kind k) {
  switch (k) {
    case Value::Kind::null: return "null";
    case Value::Kind::boolean: return "boolean";
    case Value::Kind::integer: return "integer";
    case Value::Kind::real: return "number";
    case Value::Kind::string: return "string";
    case Value::Kind::array: return "array";
    case Value::Kind::object: return "object";
  }
  return "?";
}

[[noreturn]] void type_error(const char* what, const char* want, Value::Kind got) {
  throw ParseError(std::string(what) + ": expected " + want + ", got " + kind_name(got));
}

class Parser {
 public:
  explicit Parser(const std::string& t) : s_(t.c_str()), n_(t.size()) {}

  Value document() {
    Value v = value();
    ws();
    if (p_ != n_) fail("trailing characters");
    return v;
  }

 private:
  [[noreturn]] void fail(const std::string& msg) const {
    throw ParseError("json parse error at offset " + std::to_string(p_) + ": " + msg);
  }
  void ws() {
    while (p_ < n_ && (s_[p_] == ' ' || s_[p_] == '\t' || s_[p_] == '\n' || s_[p_] == '\r')) ++p_;
  }
  bool lit(const char* word) {
    const std::size_t len = std::strlen(word);
    if (p_ + len <= n_ && std::strncmp(s_ + p_, word, len) == 0) {
      p_ += len;
      return true;
    }
    return false;
  }
  Value value() {
    ws();
    if (p_ >= n_) fail("unexpected end of input");
    const char c = s_[p_];
    if (c == '{') return object();
    if (c == '[') return array();
    if (c == '"') return Value::make_string(string());
    if (lit("true")) return Value::make_bool(true);
    if (lit("false")) return Value::make_bool(false);
    if (lit("null")) return Value();
    return number();
  }
  Value object() {
    Value v = Value::make_object();
    ++p_;
    ws();
    if (p_ < n_ && s_[p_] == '}') { ++p_; return v; }
    for (;;) {
      ws();
      if (p_ >= n_ || s_[p_] != '"') fail("expected object key");
      std::string key = string();
      ws();
      if (p_ >= n_ || s_[p_] != ':') fail("expected ':'");
      ++p_;
      v.set(key, value());
      ws();
      if (p_ < n_ && s_[p_] == ',') { ++p_; continue; }
      if (p_ < n_ && s_[p_] == '}') { ++p_; return v; }
      fail("expected ',' or '}'");
    }
  }
  Value array() {
    Value v = Value::make_array();
    ++p_;
    ws();
    if (p_ < n_ && s_[p_] == ']') { ++p_; return v; }
    for (;;) {
      v.push(value());
      ws();
      if (p_ < n_ && s_[p_] == ',') { ++p_; continue; }
      if (p_ < n_ && s_[p_] == ']') { ++p_; return v; }
      fail("expected ',' or ']'");
    }
  }
  static void utf8(std::string& out, unsigned cp) {
    if (cp < 0x80) {
      out += static_cast<char>(cp);
    } else if (cp < 0x800) {
      out += static_cast<char>(0xC0 | (cp >> 6));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    } else if (cp < 0x10000) {
      out += static_cast<char>(0xE0 | (cp >> 12));
      out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    } else {
      out += static_cast<char>(0xF0 | (cp >> 18));
      out += static_cast<char>(0x80 | ((cp >> 12) & 0x3F));
      out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    }
  }
  unsigned hex4() {
    if (p_ + 4 > n_) fail("short \\u escape");
    unsigned cp = 0;
    for (int k = 0; k < 4; ++k) {
      const char h = s_[p_++];
      cp <<= 4;
      if (h >= '0' && h <= '9') cp |= static_cast<unsigned>(h - '0');
      else if (h >= 'a' && h <= 'f') cp |= static_cast<unsigned>(h - 'a' + 10);
      else if (h >= 'A' && h <= 'F') cp |= static_cast<unsigned>(h - 'A' + 10);
      else fail("bad \\u escape");
    }
    return cp;
  }
  std::string string() {
    ++p_;  // opening quote
    // fast path: no escapes before the closing quote
    for (std::size_t q = p_; q < n_; ++q) {
      if (s_[q] == '"') {
        std::string out(s_ + p_, q - p_);
        p_ = q + 1;
        return out;
      }
      if (s_[q] == '\\') break;
    }
    std::string out;
    while (p_ < n_) {
      const char c = s_[p_++];
      if (c == '"') return out;
      if (c != '\\') { out += c; continue; }
      if (p_ >= n_) break;
      const char e = s_[p_++];
      switch (e) {
        case '"': out += '"'; break;
        case '\\': out += '\\'; break;
        case '/': out += '/'; break;
        case 'b': out += '\b'; break;
        case 'f': out += '\f'; break;
        case 'n': out += '\n'; break;
        case 'r': out += '\r'; break;
        case 't': out += '\t'; break;
        case 'u': {
          unsigned cp = hex4();
          if (cp >= 0xD800 && cp < 0xDC00 && p_ + 1 < n_ && s_[p_] == '\\' && s_[p_ + 1] == 'u') {
            p_ += 2;
            const unsigned lo = hex4();
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          }
          utf8(out, cp);
          break;
        }
        default: fail("bad escape");
      }
    }
    fail("unterminated string");
  }
  Value number() {
    const std::size_t start = p_;
    if (p_ < n_ && s_[p_] == '-') ++p_;
    bool is_real = false;
    while (p_ < n_) {
      const char c = s_[p_];
      if (c >= '0' && c <= '9') { ++p_; continue; }
      if (c == '.' || c == 'e' || c == 'E' || c == '+' || c == '-') { is_real = true; ++p_; continue; }
      break;
    }
    if (p_ == start) fail("unexpected character");
    // std::from_chars: correctly rounded, locale independent, no copy
    const char* b = s_ + start;
    const char* e = s_ + p_;
    if (!is_real) {
      long long v = 0;
      const auto r = std::from_chars(b, e, v);
      if (r.ec == std::errc() && r.ptr == e) return Value::make_int(v);
    }
    double d = 0.0;
    const auto r = std::from_chars(b, e, d);
    if (r.ec == std::errc::result_out_of_range && r.ptr == e) {  // +-inf / 0 like strtod
      const std::string tok(b, e);
      return Value::make_real(std::strtod(tok.c_str(), nullptr));
    }
    if (r.ec != std::errc() || r.ptr != e) fail("bad number '" + std::string(b, e) + "'");
    return Value::make_real(d);
  }

  const char* s_;
  std::size_t n_;
  std::size_t p_ = 0;
};

void escape(std::string& out, const std::string& s) {
  out += '"';
  for (const char c : s) {
    switch (c) {
      case '"': out += "\\\""; break;
      case '\\': out += "\\\\"; break;
      case '\n': out += "\\n"; break;
      case '\r': out += "\\r"; break;
      case '\t': out += "\\t"; break;
      default:
        if (static_cast<unsigned char>(c) < 0x20) {
          char buf[8];
          std::snprintf(buf, sizeof buf, "\\u%04x", static_cast<unsigned>(c));
          out += buf;
        } else {
          out += c;
        }
    }
  }
  out += '"';
}

}  // namespace

bool Value::as_bool(const char* what) const {
  if (kind_ != Kind::boolean) type_error(what, "boolean", kind_);
  return b_;
}
std::int64_t Value::as_int(const char* what) const {
  if (kind_ == Kind::integer) return i_;
  if (kind_ == Kind::real && std::floor(d_) == d_ && std::fabs(d_) < 9.2e18)
    return static_cast<std::int64_t>(d_);
  type_error(what, "integer", kind_);
}
double Value::as_double(const char* what) const {
  if (kind_ == Kind::real) return d_;
  if (kind_ == Kind::integer) return static_cast<double>(i_);
  type_error(what, "number", kind_);
}
const std::string& Value::as_string(const char* what) const {
  if (kind_ != Kind::string) type_error(what, "string", kind_);
  return s_;
}
const std::vector<Value>& Value::items() const {
  if (kind_ != Kind::array) type_error("value", "array", kind_);
  return a_;
}
std::vector<Value>& Value::items() {
  if (kind_ != Kind::array) type_error("value", "array", kind_);
  return a_;
}
void Value::push(Value v) {
  if (kind_ != Kind::array) type_error("value", "array", kind_);
  a_.push_back(std::move(v));
}
std::size_t Value::size() const {
  if (kind_ == Kind::array) return a_.size();
  if (kind_ == Kind::object) return o_.size();
  return 0;
}
const Value* Value::find(const std::string& key) const {
  if (kind_ != Kind::object) return nullptr;
  for (const auto& [k, v] : o_)
    if (k == key) return &v;
  return nullptr;
}
bool Value::contains(const std::string& key) const { return find(key) != nullptr; }
const Value& Value::at(const std::string& key) const {
  if (kind_ != Kind::object) type_error(key.c_str(), "object", kind_);
  const Value* v = find(key);
  if (!v) throw ParseError("key '" + key + "' not found");
  return *v;
}
void Value::set(const std::string& key, Value v) {
  if (kind_ != Kind::object) type_error(key.c_str(), "object", kind_);
  for (auto& [k, old] : o_)
    if (k == key) { old = std::move(v); return; }
  o_.emplace_back(key, std::move(v));
}
const std::vector<std::pair<std::string, Value>>& Value::members() const {
  if (kind_ != Kind::object) type_error("value", "object", kind_);
  return o_;
}

void Value::dump_to(std::string& out) const {
  switch (kind_) {
    case Kind::null: out += "null"; break;
    case Kind::boolean: out += b_ ? "true" : "false"; break;
    case Kind::integer: out += std::to_string(i_); break;
    case Kind::real: {
      char buf[40];
      std::snprintf(buf, sizeof buf, "%.17g", d_);
      out += buf;
      if (!std::strpbrk(buf, ".eEn")) out += ".0";
      break;
    }
    case Kind::string: escape(out, s_); break;
    case Kind::array: {
      out += '[';
      for (std::size_t i = 0; i < a_.size(); ++i) {
        if (i) out += ',';
        a_[i].dump_to(out);
      }
      out += ']';
      break;
    }
    case Kind::object: {
      out += '{';
      for (std::size_t i = 0; i < o_.size(); ++i) {
        if (i) out += ',';
        escape(out, o_[i].first);
        out += ':';
        o_[i].second.dump_to(out);
      }
      out += '}';
      break;
    }
  }
}

std::string Value::dump() const {
  std::string out;
  dump_to(out);
  return out;
}

Value parse(const std::string& text) { return Parser(text).document(); }

}  // namespace loomjson
