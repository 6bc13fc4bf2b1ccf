// Corpus ingestion for the index build, host C++ so a
// relinked `hyre build` (cli_commands.cpp:37-63) reads its inputs without
// Python:
//   * read_schema_json      (dataio.hpp:20-21, dataio.cpp:118-140)
//   * read_documents_jsonl  (dataio.hpp:23-28, dataio.cpp:142-187)
//   * the learned-link serving-graph export written by write_links_export
//     (dataio.cpp:253-274; node ids = link_learner.cpp:327-347's term ids),
//     read back as the config-5 vocabulary.
// Validation rules and error texts follow the reference ("<path>:<line>:
// <what>"); JSON values follow nlohmann::json as the reference uses it
// (objects iterate in key order, an integer without '-' is unsigned, one with
// '-' signed, anything with a fraction or exponent a float).  The JSON syntax
// error texts are this parser's own.
#include <cerrno>
#include <cmath>
#include <cstdlib>
#include <fstream>
#include <map>
#include <memory>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "host.hpp"

namespace hyreb {

namespace {

struct JVal {
  enum Kind { Null, Bool, Unsigned, Signed, Float, String, Array, Object } k = Null;
  bool b = false;
  uint64_t u = 0;
  int64_t i = 0;
  double d = 0.0;
  std::string s;
  std::vector<JVal> a;
  std::map<std::string, JVal> o;  // key order, like nlohmann::json's default object
  bool is_number() const { return k == Unsigned || k == Signed || k == Float; }
  double number() const { return k == Unsigned ? static_cast<double>(u) : k == Signed ? static_cast<double>(i) : d; }
};

struct JsonError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

class Parser {
 public:
  explicit Parser(const std::string& t) : t_(t) {}
  JVal parse() {
    ws();
    JVal v = value(0);
    ws();
    if (p_ != t_.size()) fail("unexpected trailing characters");
    return v;
  }

 private:
  [[noreturn]] void fail(const std::string& what) const {
    size_t line = 1, col = 1;
    for (size_t q = 0; q < p_ && q < t_.size(); ++q) {
      if (t_[q] == '\n') {
        ++line;
        col = 1;
      } else {
        ++col;
      }
    }
    throw JsonError("parse error at line " + std::to_string(line) + ", column " + std::to_string(col) + ": " + what);
  }
  void ws() {
    while (p_ < t_.size() && (t_[p_] == ' ' || t_[p_] == '\t' || t_[p_] == '\n' || t_[p_] == '\r')) ++p_;
  }
  bool lit(const char* s) {
    size_t n = std::char_traits<char>::length(s);
    if (t_.compare(p_, n, s) != 0) return false;
    p_ += n;
    return true;
  }
  JVal value(int depth) {
    if (depth > 512) fail("nesting too deep");
    if (p_ >= t_.size()) fail("unexpected end of input");
    JVal v;
    const char c = t_[p_];
    if (c == '{') {
      v.k = JVal::Object;
      ++p_;
      ws();
      if (p_ < t_.size() && t_[p_] == '}') {
        ++p_;
        return v;
      }
      for (;;) {
        ws();
        if (p_ >= t_.size() || t_[p_] != '"') fail("expected object key");
        std::string key = str();
        ws();
        if (p_ >= t_.size() || t_[p_] != ':') fail("expected ':'");
        ++p_;
        ws();
        v.o[key] = value(depth + 1);  // duplicate keys: the last one wins
        ws();
        if (p_ < t_.size() && t_[p_] == ',') {
          ++p_;
          continue;
        }
        if (p_ < t_.size() && t_[p_] == '}') {
          ++p_;
          return v;
        }
        fail("expected ',' or '}'");
      }
    }
    if (c == '[') {
      v.k = JVal::Array;
      ++p_;
      ws();
      if (p_ < t_.size() && t_[p_] == ']') {
        ++p_;
        return v;
      }
      for (;;) {
        ws();
        v.a.push_back(value(depth + 1));
        ws();
        if (p_ < t_.size() && t_[p_] == ',') {
          ++p_;
          continue;
        }
        if (p_ < t_.size() && t_[p_] == ']') {
          ++p_;
          return v;
        }
        fail("expected ',' or ']'");
      }
    }
    if (c == '"') {
      v.k = JVal::String;
      v.s = str();
      return v;
    }
    if (lit("true")) {
      v.k = JVal::Bool;
      v.b = true;
      return v;
    }
    if (lit("false")) {
      v.k = JVal::Bool;
      return v;
    }
    if (lit("null")) return v;
    if (c == '-' || (c >= '0' && c <= '9')) return number();
    fail(std::string("unexpected character '") + c + "'");
  }
  JVal number() {
    const size_t b = p_;
    bool neg = false, flt = false;
    if (t_[p_] == '-') {
      neg = true;
      ++p_;
    }
    auto digits = [&] {
      const size_t s = p_;
      while (p_ < t_.size() && t_[p_] >= '0' && t_[p_] <= '9') ++p_;
      if (p_ == s) fail("invalid number");
    };
    if (p_ < t_.size() && t_[p_] == '0') {
      ++p_;
    } else {
      digits();
    }
    if (p_ < t_.size() && t_[p_] == '.') {
      flt = true;
      ++p_;
      digits();
    }
    if (p_ < t_.size() && (t_[p_] == 'e' || t_[p_] == 'E')) {
      flt = true;
      ++p_;
      if (p_ < t_.size() && (t_[p_] == '+' || t_[p_] == '-')) ++p_;
      digits();
    }
    const std::string tok = t_.substr(b, p_ - b);
    JVal v;
    errno = 0;
    if (!flt && !neg) {
      char* end = nullptr;
      const unsigned long long x = std::strtoull(tok.c_str(), &end, 10);
      if (errno != ERANGE) {
        v.k = JVal::Unsigned;
        v.u = x;
        return v;
      }
    } else if (!flt) {
      char* end = nullptr;
      const long long x = std::strtoll(tok.c_str(), &end, 10);
      if (errno != ERANGE) {
        v.k = JVal::Signed;
        v.i = x;
        return v;
      }
    }
    v.k = JVal::Float;  // fractions, exponents and out-of-range integers
    v.d = std::strtod(tok.c_str(), nullptr);
    return v;
  }
  static void utf8(std::string& out, uint32_t cp) {
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
  uint32_t hex4() {
    if (p_ + 4 > t_.size()) fail("invalid \\u escape");
    uint32_t v = 0;
    for (int q = 0; q < 4; ++q) {
      const char h = t_[p_++];
      v <<= 4;
      if (h >= '0' && h <= '9') v |= h - '0';
      else if (h >= 'a' && h <= 'f') v |= h - 'a' + 10;
      else if (h >= 'A' && h <= 'F') v |= h - 'A' + 10;
      else fail("invalid \\u escape");
    }
    return v;
  }
  std::string str() {
    ++p_;  // opening quote
    std::string out;
    for (;;) {
      if (p_ >= t_.size()) fail("unterminated string");
      const char c = t_[p_++];
      if (c == '"') return out;
      if (static_cast<unsigned char>(c) < 0x20) fail("control character in string");
      if (c != '\\') {
        out += c;
        continue;
      }
      if (p_ >= t_.size()) fail("unterminated string");
      const char e = t_[p_++];
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
          uint32_t cp = hex4();
          if (cp >= 0xD800 && cp <= 0xDBFF) {  // surrogate pair
            if (!lit("\\u")) fail("invalid surrogate pair");
            const uint32_t lo = hex4();
            if (lo < 0xDC00 || lo > 0xDFFF) fail("invalid surrogate pair");
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
            fail("invalid surrogate pair");
          }
          utf8(out, cp);
          break;
        }
        default: fail("invalid escape");
      }
    }
  }
  const std::string& t_;
  size_t p_ = 0;
};

[[noreturn]] void fail_at(const std::string& path, size_t line, const std::string& what) {
  validation(path + ":" + std::to_string(line) + ": " + what);  // dataio.cpp:18-21
}

JVal parse_file(const std::string& path) {  // dataio.cpp:23-31
  std::ifstream in(path, std::ios::binary);
  if (!in) validation("cannot open: " + path);
  std::stringstream ss;
  ss << in.rdbuf();
  const std::string text = ss.str();
  try {
    return Parser(text).parse();
  } catch (const JsonError& e) {
    validation(path + ": " + e.what());
  }
}

uint32_t to_attr_id(const JVal& v, const std::string& path, size_t line) {  // dataio.cpp:51-58
  if (v.k != JVal::Unsigned) fail_at(path, line, "attribute ids must be unsigned integers");
  if (v.u > 0xFFFFFFFFull) fail_at(path, line, "attribute id out of range");
  return static_cast<uint32_t>(v.u);
}

}  // namespace

Schema read_schema_json(const std::string& path) {  // dataio.cpp:118-140
  const JVal j = parse_file(path);
  if (j.k != JVal::Object || !j.o.count("clauses") || !j.o.count("dim"))
    validation(path + ": schema needs 'clauses' and 'dim'");
  const JVal& names = j.o.at("clauses");
  if (names.k != JVal::Array) validation(path + ": 'clauses' must be an array");
  Schema s;
  for (const JVal& n : names.a) {
    if (n.k != JVal::String) validation(path + ": clause names must be strings");
    s.clause_names.push_back(n.s);
  }
  if (s.clause_names.empty()) validation(path + ": 'clauses' must not be empty");
  const JVal& dim = j.o.at("dim");
  if (dim.k != JVal::Unsigned || dim.u > 0xFFFFFFFFull) validation(path + ": dim must be an unsigned integer");
  s.dim = static_cast<uint32_t>(dim.u);
  return s;
}

// read_documents_jsonl (dataio.cpp:142-187): one JSON object per line, blank
// lines skipped (dataio.cpp:33-49); absent clauses empty, absent embedding
// the zero vector; entries get<double>() then static_cast<float>.
DocumentSet read_documents_jsonl(const std::string& path, const Schema& schema) {
  std::ifstream in(path, std::ios::binary);
  if (!in) validation("cannot open: " + path);
  std::map<std::string, uint32_t> slot_of;
  for (uint32_t i = 0; i < schema.clause_names.size(); ++i) slot_of.emplace(schema.clause_names[i], i);
  const uint32_t C = static_cast<uint32_t>(schema.clause_names.size());
  DocumentSet d;
  d.num_clauses = C;
  d.dim = schema.dim;
  d.slot_offsets.push_back(0);
  std::string line;
  size_t line_no = 0;
  std::vector<std::vector<uint32_t>> clauses(C);
  while (std::getline(in, line)) {
    ++line_no;
    if (line.find_first_not_of(" \t\r") == std::string::npos) continue;
    JVal j;
    try {
      j = Parser(line).parse();
    } catch (const JsonError& e) {
      fail_at(path, line_no, e.what());
    }
    if (j.k != JVal::Object || !j.o.count("id") || j.o.at("id").k != JVal::String)
      fail_at(path, line_no, "document needs a string 'id'");
    for (auto& c : clauses) c.clear();
    if (j.o.count("clauses")) {
      const JVal& cl = j.o.at("clauses");
      if (cl.k != JVal::Object) fail_at(path, line_no, "'clauses' must be an object");
      for (const auto& [name, ids] : cl.o) {
        auto it = slot_of.find(name);
        if (it == slot_of.end()) fail_at(path, line_no, "unknown clause '" + name + "'");
        if (ids.k != JVal::Array) fail_at(path, line_no, "clause '" + name + "' must be an array");
        for (const JVal& v : ids.a) clauses[it->second].push_back(to_attr_id(v, path, line_no));
      }
    }
    const size_t e0 = d.embeddings.size();
    d.embeddings.resize(e0 + schema.dim, 0.0f);
    if (j.o.count("embedding")) {
      const JVal& emb = j.o.at("embedding");
      if (emb.k != JVal::Array) fail_at(path, line_no, "'embedding' must be an array");
      if (emb.a.size() != schema.dim)
        fail_at(path, line_no,
                "embedding: expected dim " + std::to_string(schema.dim) + ", got " + std::to_string(emb.a.size()));
      for (size_t q = 0; q < emb.a.size(); ++q) {
        if (!emb.a[q].is_number()) fail_at(path, line_no, "embedding entries must be numbers");
        d.embeddings[e0 + q] = static_cast<float>(emb.a[q].number());
      }
    }
    d.doc_ids.push_back(j.o.at("id").s);
    uint32_t width = 0;
    for (uint32_t c = 0; c < C; ++c) {
      d.ids.insert(d.ids.end(), clauses[c].begin(), clauses[c].end());
      d.slot_offsets.push_back(d.ids.size());
      width += static_cast<uint32_t>(std::set<uint32_t>(clauses[c].begin(), clauses[c].end()).size());
    }
    d.widest = std::max(d.widest, width);
  }
  return d;
}

// The serving-graph export (dataio.cpp:253-274): nodes + the attribute-id
// maps of export_to_index (link_learner.cpp:327-347); ids sorted, unique.
LinksExport read_links_export(const std::string& path) {
  const JVal j = parse_file(path);
  if (j.k != JVal::Object || !j.o.count("nodes") || !j.o.count("seekerAttributes") || !j.o.count("jobAttributes"))
    validation(path + ": links export needs 'nodes', 'seekerAttributes' and 'jobAttributes'");
  LinksExport out;
  const JVal& nodes = j.o.at("nodes");
  if (nodes.k != JVal::Array) validation(path + ": 'nodes' must be an array");
  out.num_nodes = static_cast<uint32_t>(nodes.a.size());
  for (int side = 0; side < 2; ++side) {
    const char* key = side == 0 ? "seekerAttributes" : "jobAttributes";
    const JVal& m = j.o.at(key);
    if (m.k != JVal::Object) validation(path + ": '" + key + "' must be an object");
    for (const auto& [name, ids] : m.o) {
      std::set<uint32_t> s;
      bool ok = ids.k == JVal::Array;
      for (size_t q = 0; ok && q < ids.a.size(); ++q) {
        ok = ids.a[q].k == JVal::Unsigned && ids.a[q].u > 0 && ids.a[q].u <= 0xFFFFFFFFull;
        if (ok) s.insert(static_cast<uint32_t>(ids.a[q].u));
      }
      if (!ok) validation(path + ": " + key + "." + name + " must be an array of node ids");
      out.names[side].push_back(name);
      out.ids[side].emplace_back(s.begin(), s.end());
    }
  }
  return out;
}

}  // namespace hyreb
