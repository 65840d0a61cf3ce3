// Minimal JSON reader for the reference payload format (serialize.cpp:147-167).
// Numbers are parsed with strtod (correctly rounded), so doubles written by the
// reference's round-trip printer come back bit-exact.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace qcg {

struct JValue {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  bool b = false;
  double num = 0;
  bool is_int = false;
  long long i = 0;
  std::string s;
  std::vector<JValue> arr;
  std::vector<std::pair<std::string, JValue>> obj;

  const JValue& at(const std::string& key) const {
    if (kind != Obj) throw std::invalid_argument("json: not an object (looking up '" + key + "')");
    for (const auto& kv : obj)
      if (kv.first == key) return kv.second;
    throw std::invalid_argument("json: missing key '" + key + "'");
  }
  bool has(const std::string& key) const {
    if (kind != Obj) return false;
    for (const auto& kv : obj)
      if (kv.first == key) return true;
    return false;
  }
  const JValue& operator[](size_t idx) const {
    if (kind != Arr || idx >= arr.size()) throw std::invalid_argument("json: bad array index");
    return arr[idx];
  }
  size_t size() const { return kind == Arr ? arr.size() : obj.size(); }
  int as_int() const {
    if (kind != Num || !is_int) throw std::invalid_argument("json: expected an integer");
    return static_cast<int>(i);
  }
  double as_double() const {
    if (kind != Num) throw std::invalid_argument("json: expected a number");
    return num;
  }
  std::vector<int> as_int_vec() const {
    if (kind != Arr) throw std::invalid_argument("json: expected an array");
    std::vector<int> v;
    v.reserve(arr.size());
    for (const auto& x : arr) v.push_back(x.as_int());
    return v;
  }
};

class JParser {
 public:
  JParser(const char* p, size_t n) : p_(p), end_(p + n) {}
  JValue parse() {
    JValue v = value();
    ws();
    if (p_ != end_) fail("trailing characters");
    return v;
  }

 private:
  const char* p_;
  const char* end_;

  [[noreturn]] void fail(const char* what) { throw std::invalid_argument(std::string("json: ") + what); }
  void ws() {
    while (p_ < end_ && (*p_ == ' ' || *p_ == '\n' || *p_ == '\r' || *p_ == '\t')) ++p_;
  }
  char peek() {
    ws();
    if (p_ >= end_) fail("unexpected end");
    return *p_;
  }
  void expect(char c) {
    if (peek() != c) fail("unexpected character");
    ++p_;
  }
  JValue value() {
    char c = peek();
    if (c == '{') return object();
    if (c == '[') return array();
    if (c == '"') {
      JValue v;
      v.kind = JValue::Str;
      v.s = string();
      return v;
    }
    if (c == 't' || c == 'f' || c == 'n') return literal();
    return number();
  }
  JValue literal() {
    JValue v;
    auto match = [&](const char* w) {
      size_t n = std::char_traits<char>::length(w);
      if (static_cast<size_t>(end_ - p_) >= n && std::equal(w, w + n, p_)) {
        p_ += n;
        return true;
      }
      return false;
    };
    if (match("true")) {
      v.kind = JValue::Bool;
      v.b = true;
    } else if (match("false")) {
      v.kind = JValue::Bool;
    } else if (match("null")) {
      v.kind = JValue::Null;
    } else {
      fail("bad literal");
    }
    return v;
  }
  std::string string() {
    expect('"');
    std::string out;
    while (p_ < end_ && *p_ != '"') {
      if (*p_ == '\\') {
        ++p_;
        if (p_ >= end_) fail("bad escape");
        char e = *p_++;
        switch (e) {
          case 'n': out.push_back('\n'); break;
          case 't': out.push_back('\t'); break;
          case 'r': out.push_back('\r'); break;
          case 'b': out.push_back('\b'); break;
          case 'f': out.push_back('\f'); break;
          case 'u': {
            if (end_ - p_ < 4) fail("bad unicode escape");
            unsigned cp = static_cast<unsigned>(std::strtoul(std::string(p_, p_ + 4).c_str(), nullptr, 16));
            p_ += 4;
            if (cp < 0x80) out.push_back(static_cast<char>(cp));
            else out.push_back('?');
            break;
          }
          default: out.push_back(e);
        }
      } else {
        out.push_back(*p_++);
      }
    }
    if (p_ >= end_) fail("unterminated string");
    ++p_;
    return out;
  }
  JValue number() {
    ws();
    const char* start = p_;
    bool is_int = true;
    if (p_ < end_ && (*p_ == '-' || *p_ == '+')) ++p_;
    while (p_ < end_) {
      char c = *p_;
      if (c >= '0' && c <= '9') {
        ++p_;
      } else if (c == '.' || c == 'e' || c == 'E' || c == '-' || c == '+') {
        is_int = false;
        ++p_;
      } else {
        break;
      }
    }
    if (p_ == start) fail("bad number");
    std::string tok(start, p_);
    JValue v;
    v.kind = JValue::Num;
    char* endp = nullptr;
    v.num = std::strtod(tok.c_str(), &endp);
    if (endp != tok.c_str() + tok.size()) fail("bad number");
    v.is_int = is_int;
    if (is_int) v.i = std::strtoll(tok.c_str(), nullptr, 10);
    return v;
  }
  JValue array() {
    expect('[');
    JValue v;
    v.kind = JValue::Arr;
    if (peek() == ']') {
      ++p_;
      return v;
    }
    for (;;) {
      v.arr.push_back(value());
      char c = peek();
      ++p_;
      if (c == ']') break;
      if (c != ',') fail("expected , or ]");
    }
    return v;
  }
  JValue object() {
    expect('{');
    JValue v;
    v.kind = JValue::Obj;
    if (peek() == '}') {
      ++p_;
      return v;
    }
    for (;;) {
      if (peek() != '"') fail("expected key");
      std::string k = string();
      expect(':');
      v.obj.emplace_back(std::move(k), value());
      char c = peek();
      ++p_;
      if (c == '}') break;
      if (c != ',') fail("expected , or }");
    }
    return v;
  }
};

inline JValue json_parse(const char* p, size_t n) { return JParser(p, n).parse(); }

}  // namespace qcg
