// Minimal JSON DOM for the loom host layer: enough to read and write the
// reference's fixture formats (library bundle, dag.json, config points;
// SPEC.md:92,154,224,367) without a third-party dependency.  Numbers keep
// their integer/float distinction; doubles are parsed with strtod (correctly
// rounded) and written with 17 significant digits so they round-trip.
#pragma once

#include <cctype>
#include <charconv>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

namespace loomjson {

struct ParseError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

class Value {
 public:
  enum class Kind { null, boolean, integer, real, string, array, object };

  Value() = default;
  static Value make_bool(bool b) { Value v; v.kind_ = Kind::boolean; v.b_ = b; return v; }
  static Value make_int(std::int64_t i) { Value v; v.kind_ = Kind::integer; v.i_ = i; return v; }
  static Value make_real(double d) { Value v; v.kind_ = Kind::real; v.d_ = d; return v; }
  static Value make_string(std::string s) { Value v; v.kind_ = Kind::string; v.s_ = std::move(s); return v; }
  static Value make_array() { Value v; v.kind_ = Kind::array; return v; }
  static Value make_object() { Value v; v.kind_ = Kind::object; return v; }

  Kind kind() const { return kind_; }
  bool is_null() const { return kind_ == Kind::null; }
  bool is_string() const { return kind_ == Kind::string; }
  bool is_array() const { return kind_ == Kind::array; }
  bool is_object() const { return kind_ == Kind::object; }
  bool is_number() const { return kind_ == Kind::integer || kind_ == Kind::real; }
  bool is_integer() const { return kind_ == Kind::integer; }

  bool as_bool(const char* what = "value") const;
  std::int64_t as_int(const char* what = "value") const;
  double as_double(const char* what = "value") const;
  const std::string& as_string(const char* what = "value") const;

  // arrays
  const std::vector<Value>& items() const;
  std::vector<Value>& items();
  void push(Value v);
  std::size_t size() const;

  // objects (insertion order kept for output; lookup is linear, objects are small)
  bool contains(const std::string& key) const;
  const Value& at(const std::string& key) const;  // throws ParseError naming the key
  const Value* find(const std::string& key) const;
  void set(const std::string& key, Value v);
  const std::vector<std::pair<std::string, Value>>& members() const;

  std::string dump() const;

 private:
  void dump_to(std::string& out) const;

  Kind kind_ = Kind::null;
  bool b_ = false;
  std::int64_t i_ = 0;
  double d_ = 0.0;
  std::string s_;
  std::vector<Value> a_;
  std::vector<std::pair<std::string, Value>> o_;
};

Value parse(const std::string& text);

// Pull cursor over JSON text for hot readers (dag.json in batch lowering):
// no DOM.  Every method returns false on anything it does not handle (escape
// sequences, type mismatches, syntax errors); callers then fall back to
// parse(), which produces the canonical error messages.
class Cursor {
 public:
  explicit Cursor(const std::string& t) : s_(t.data()), n_(t.size()) {}
  bool open(char c);                  // '{' or '['
  bool next(char close, bool& more);  // after a member / element: ',' -> more, close -> done
  bool empty(char close);             // right after open: consumes close if the container is empty
  bool key(std::string_view& k);      // "key" ':'
  bool str(std::string& out);
  bool num(double& out);
  bool integer(long long& out);
  bool boolean(bool& out);
  bool null();                        // consumes null if present
  bool skip();                        // any value
  bool end();                         // only whitespace left

 private:
  void ws();
  bool raw_string(std::string_view& out);
  const char* s_;
  std::size_t n_;
  std::size_t p_ = 0;
  int depth_ = 0;
};

// ---- Cursor (inline: the batch dag reader calls it per token) ---------------------------------------------------------------
// Character classes for the scans below.  The text is a std::string, so
// s_[n_] is '\0', which is in no class but kStop: the scans need no bounds
// test.
enum : unsigned char { kWs = 1, kStop = 2, kNum = 4 };
inline constexpr struct CharClass {
  unsigned char c[256];
  constexpr CharClass() : c{} {
    c[' '] = c['\n'] = c['\t'] = c['\r'] = kWs;
    for (int i = 0; i < 0x20; ++i) c[i] |= kStop;
    c['"'] |= kStop;
    c['\\'] |= kStop;
    for (int i = '0'; i <= '9'; ++i) c[i] |= kNum;
    c['-'] |= kNum;
    c['+'] |= kNum;
    c['.'] |= kNum;
    c['e'] |= kNum;
    c['E'] |= kNum;
  }
} kCharClass;
inline void Cursor::ws() {
  while (kCharClass.c[static_cast<unsigned char>(s_[p_])] & kWs) ++p_;
}
inline bool Cursor::open(char c) {
  ws();
  if (p_ >= n_ || s_[p_] != c || ++depth_ > 64) return false;
  ++p_;
  return true;
}
inline bool Cursor::empty(char close) {
  ws();
  if (p_ < n_ && s_[p_] == close) {
    ++p_;
    --depth_;
    return true;
  }
  return false;
}
inline bool Cursor::next(char close, bool& more) {
  ws();
  if (p_ >= n_) return false;
  if (s_[p_] == ',') {
    ++p_;
    more = true;
    return true;
  }
  if (s_[p_] == close) {
    ++p_;
    --depth_;
    more = false;
    return true;
  }
  return false;
}
inline bool Cursor::raw_string(std::string_view& out) {
  ws();
  if (p_ >= n_ || s_[p_] != '"') return false;
  const std::size_t b = ++p_;
  while (!(kCharClass.c[static_cast<unsigned char>(s_[p_])] & kStop)) ++p_;
  if (p_ >= n_ || s_[p_] != '"') return false;  // end of text, escape or control character
  out = std::string_view(s_ + b, p_ - b);
  ++p_;
  return true;
}
inline bool Cursor::key(std::string_view& k) {
  if (!raw_string(k)) return false;
  ws();
  if (p_ >= n_ || s_[p_] != ':') return false;
  ++p_;
  return true;
}
inline bool Cursor::str(std::string& out) {
  std::string_view v;
  if (!raw_string(v)) return false;
  out.assign(v.data(), v.size());
  return true;
}
inline bool Cursor::num(double& out) {
  ws();
  const std::size_t b = p_;
  while (kCharClass.c[static_cast<unsigned char>(s_[p_])] & kNum) ++p_;
  if (p_ == b) return false;
  const auto r = std::from_chars(s_ + b, s_ + p_, out);
  return r.ec == std::errc() && r.ptr == s_ + p_;
}
inline bool Cursor::integer(long long& out) {
  ws();
  const std::size_t b = p_;
  while (p_ < n_ && (std::isdigit(static_cast<unsigned char>(s_[p_])) || s_[p_] == '-')) ++p_;
  if (p_ == b || (p_ < n_ && (s_[p_] == '.' || s_[p_] == 'e' || s_[p_] == 'E'))) return false;
  const auto r = std::from_chars(s_ + b, s_ + p_, out);
  return r.ec == std::errc() && r.ptr == s_ + p_;
}
inline bool Cursor::boolean(bool& out) {
  ws();
  if (n_ - p_ >= 4 && std::memcmp(s_ + p_, "true", 4) == 0) {
    p_ += 4;
    out = true;
    return true;
  }
  if (n_ - p_ >= 5 && std::memcmp(s_ + p_, "false", 5) == 0) {
    p_ += 5;
    out = false;
    return true;
  }
  return false;
}
inline bool Cursor::null() {
  ws();
  if (n_ - p_ >= 4 && std::memcmp(s_ + p_, "null", 4) == 0) {
    p_ += 4;
    return true;
  }
  return false;
}
inline bool Cursor::skip() {
  ws();
  if (p_ >= n_) return false;
  const char c = s_[p_];
  if (c == '"') {
    std::string_view v;
    return raw_string(v);
  }
  if (c == '{' || c == '[') {
    const char close = c == '{' ? '}' : ']';
    if (!open(c)) return false;
    if (empty(close)) return true;
    for (bool more = true; more;) {
      if (c == '{') {
        std::string_view k;
        if (!key(k)) return false;
      }
      if (!skip() || !next(close, more)) return false;
    }
    return true;
  }
  if (c == 't' || c == 'f') {
    bool b;
    return boolean(b);
  }
  if (c == 'n') return null();
  double d;
  return num(d);
}
inline bool Cursor::end() {
  ws();
  return p_ == n_;
}

}  // namespace loomjson
