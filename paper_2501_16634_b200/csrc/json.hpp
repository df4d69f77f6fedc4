// Minimal JSON DOM for the loom host layer: enough to read and write the
// reference's fixture formats (library bundle, dag.json, config points;
// SPEC.md:92,154,224,367) without a third-party dependency.  Numbers keep
// their integer/float distinction; doubles are parsed with strtod (correctly
// rounded) and written with 17 significant digits so they round-trip.
#pragma once

#include <cstdint>
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

}  // namespace loomjson
