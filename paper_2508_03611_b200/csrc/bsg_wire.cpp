// bsg_wire.cpp — the reference's wire schema (core/src/json_io.cpp) in front
// of the GPU predictor: PredictionRequest JSON texts in, PredictionResult JSON
// texts (or {"error": ...} bodies) out, the whole batch predicted in one
// bsg_predict_batch call. SURVEY.md §8(f) row 3 — the codec only: the HTTP
// roles (service.cpp) stay out of scope (networking).
//
// Parsing follows json_io.cpp's field names and its bad-schema behaviour (a
// missing field or a wrong type rejects the request); numbers are printed the
// way nlohmann::json::dump prints them (Grisu2 digits, fixed notation for
// decimal exponents in (-4, 15], otherwise d.ddde±XX), so the response text is
// byte-identical to the reference's prediction_result_to_json.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <system_error>
#include <unordered_set>
#include <vector>

#include "bsg_internal.h"

namespace {

// ---- a small JSON DOM -------------------------------------------------------
struct JVal {
  enum Kind { kNull, kBool, kInt, kUint, kDouble, kString, kArray, kObject } kind = kNull;
  bool b = false;
  int64_t i = 0;
  uint64_t u = 0;
  double d = 0;
  std::string s;
  std::vector<JVal> arr;
  std::vector<std::pair<std::string, JVal>> obj;
  const JVal* get(const char* key) const {  // duplicate keys: the last one wins, as in nlohmann
    for (auto it = obj.rbegin(); it != obj.rend(); ++it)
      if (it->first == key) return &it->second;
    return nullptr;
  }
  bool is_number() const { return kind == kInt || kind == kUint || kind == kDouble; }
};

struct Parser {
  const char* p;
  const char* end;
  std::string err;
  void ws() {
    while (p < end && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r')) ++p;
  }
  bool fail(const char* m) {
    if (err.empty()) err = m;
    return false;
  }
  bool lit(const char* w) {
    const size_t n = std::strlen(w);
    if (static_cast<size_t>(end - p) < n || std::strncmp(p, w, n) != 0) return fail("malformed JSON");
    p += n;
    return true;
  }
  static bool hex4(const char* h, unsigned* cp) {
    unsigned v = 0;
    for (int k = 0; k < 4; ++k) {
      const char c = h[k];
      v <<= 4;
      if (c >= '0' && c <= '9') v |= c - '0';
      else if (c >= 'a' && c <= 'f') v |= c - 'a' + 10;
      else if (c >= 'A' && c <= 'F') v |= c - 'A' + 10;
      else return false;
    }
    *cp = v;
    return true;
  }
  bool string(std::string* out) {
    if (p >= end || *p != '"') return fail("malformed JSON");
    ++p;
    while (p < end && *p != '"') {
      if (*p == '\\') {
        if (++p >= end) return fail("malformed JSON");
        switch (*p) {
          case '"': out->push_back('"'); break;
          case '\\': out->push_back('\\'); break;
          case '/': out->push_back('/'); break;
          case 'b': out->push_back('\b'); break;
          case 'f': out->push_back('\f'); break;
          case 'n': out->push_back('\n'); break;
          case 'r': out->push_back('\r'); break;
          case 't': out->push_back('\t'); break;
          case 'u': {  // \uXXXX, surrogate pairs joined, lone surrogates rejected
            unsigned cp = 0;
            if (end - p < 5 || !hex4(p + 1, &cp)) return fail("malformed JSON");
            p += 4;
            if (cp >= 0xDC00 && cp <= 0xDFFF) return fail("malformed JSON");
            if (cp >= 0xD800 && cp <= 0xDBFF) {
              unsigned lo = 0;
              if (end - p < 7 || p[1] != '\\' || p[2] != 'u' || !hex4(p + 3, &lo) || lo < 0xDC00 ||
                  lo > 0xDFFF)
                return fail("malformed JSON");
              p += 6;
              cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
            }
            if (cp < 0x80) {
              out->push_back(static_cast<char>(cp));
            } else if (cp < 0x800) {
              out->push_back(static_cast<char>(0xc0 | (cp >> 6)));
              out->push_back(static_cast<char>(0x80 | (cp & 0x3f)));
            } else if (cp < 0x10000) {
              out->push_back(static_cast<char>(0xe0 | (cp >> 12)));
              out->push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3f)));
              out->push_back(static_cast<char>(0x80 | (cp & 0x3f)));
            } else {
              out->push_back(static_cast<char>(0xf0 | (cp >> 18)));
              out->push_back(static_cast<char>(0x80 | ((cp >> 12) & 0x3f)));
              out->push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3f)));
              out->push_back(static_cast<char>(0x80 | (cp & 0x3f)));
            }
            break;
          }
          default: return fail("malformed JSON");
        }
        ++p;
      } else {
        const unsigned char c = static_cast<unsigned char>(*p);
        if (c < 0x20) return fail("malformed JSON");  // RFC 8259 §7
        if (c < 0x80) {
          out->push_back(*p++);
          continue;
        }
        // well-formed UTF-8 only (RFC 3629 §4), as nlohmann's lexer checks
        int n = 0;
        unsigned char lo2 = 0x80, hi2 = 0xBF;
        if (c >= 0xC2 && c <= 0xDF) n = 1;
        else if (c == 0xE0) n = 2, lo2 = 0xA0;
        else if (c >= 0xE1 && c <= 0xEC) n = 2;
        else if (c == 0xED) n = 2, hi2 = 0x9F;
        else if (c >= 0xEE && c <= 0xEF) n = 2;
        else if (c == 0xF0) n = 3, lo2 = 0x90;
        else if (c >= 0xF1 && c <= 0xF3) n = 3;
        else if (c == 0xF4) n = 3, hi2 = 0x8F;
        else return fail("malformed JSON");
        if (end - p <= n) return fail("malformed JSON");
        for (int k = 1; k <= n; ++k) {
          const unsigned char d = static_cast<unsigned char>(p[k]);
          if (k == 1 ? (d < lo2 || d > hi2) : (d < 0x80 || d > 0xBF)) return fail("malformed JSON");
        }
        out->append(p, p + n + 1);
        p += n + 1;
      }
    }
    if (p >= end) return fail("malformed JSON");
    ++p;
    return true;
  }
  bool number(JVal* v) {  // RFC 8259 grammar: -?(0|[1-9][0-9]*)(.[0-9]+)?([eE][+-]?[0-9]+)?
    const char* s = p;
    auto digit = [&] { return p < end && *p >= '0' && *p <= '9'; };
    bool is_float = false;
    if (p < end && *p == '-') ++p;
    if (!digit()) return fail("malformed JSON");
    if (*p == '0') {
      ++p;
    } else {
      while (digit()) ++p;
    }
    if (p < end && *p == '.') {
      ++p;
      is_float = true;
      if (!digit()) return fail("malformed JSON");
      while (digit()) ++p;
    }
    if (p < end && (*p == 'e' || *p == 'E')) {
      ++p;
      is_float = true;
      if (p < end && (*p == '+' || *p == '-')) ++p;
      if (!digit()) return fail("malformed JSON");
      while (digit()) ++p;
    }
    if (!is_float) {  // integers that overflow 64 bits fall through to double, as in nlohmann
      if (*s == '-') {
        int64_t x = 0;
        auto r = std::from_chars(s, p, x);
        if (r.ec == std::errc() && r.ptr == p) {
          v->kind = JVal::kInt;
          v->i = x;
          return true;
        }
      } else {
        uint64_t x = 0;
        auto r = std::from_chars(s, p, x);
        if (r.ec == std::errc() && r.ptr == p) {
          v->kind = JVal::kUint;
          v->u = x;
          return true;
        }
      }
    }
    double x = 0;
    auto r = std::from_chars(s, p, x);
    if (r.ec != std::errc() || r.ptr != p) return fail("malformed JSON");
    v->kind = JVal::kDouble;
    v->d = x;
    return true;
  }
  bool value(JVal* v, int depth = 0) {
    if (depth > 512) return fail("malformed JSON");  // bounded recursion (nlohmann has none)
    ws();
    if (p >= end) return fail("malformed JSON");
    switch (*p) {
      case '{': {
        ++p;
        v->kind = JVal::kObject;
        ws();
        if (p < end && *p == '}') {
          ++p;
          return true;
        }
        for (;;) {
          ws();
          std::string key;
          if (!string(&key)) return false;
          ws();
          if (p >= end || *p != ':') return fail("malformed JSON");
          ++p;
          JVal child;
          if (!value(&child, depth + 1)) return false;
          v->obj.emplace_back(std::move(key), std::move(child));
          ws();
          if (p < end && *p == ',') {
            ++p;
            continue;
          }
          if (p < end && *p == '}') {
            ++p;
            return true;
          }
          return fail("malformed JSON");
        }
      }
      case '[': {
        ++p;
        v->kind = JVal::kArray;
        ws();
        if (p < end && *p == ']') {
          ++p;
          return true;
        }
        for (;;) {
          JVal child;
          if (!value(&child, depth + 1)) return false;
          v->arr.push_back(std::move(child));
          ws();
          if (p < end && *p == ',') {
            ++p;
            continue;
          }
          if (p < end && *p == ']') {
            ++p;
            return true;
          }
          return fail("malformed JSON");
        }
      }
      case '"':
        v->kind = JVal::kString;
        return string(&v->s);
      case 't':
        v->kind = JVal::kBool;
        v->b = true;
        return lit("true");
      case 'f':
        v->kind = JVal::kBool;
        return lit("false");
      case 'n':
        return lit("null");
      default:
        return number(v);
    }
  }
};

// ---- schema (json_io.cpp) ---------------------------------------------------
// Errors carry nlohmann::json 3.11.3's exception text (what()), which the
// reference wraps as "bad-schema: <what>" (parse_with, json_io.cpp:86-95).
struct SchemaError {
  std::string what;
};

const char* type_name(const JVal& v) {  // basic_json::type_name()
  switch (v.kind) {
    case JVal::kNull: return "null";
    case JVal::kBool: return "boolean";
    case JVal::kInt:
    case JVal::kUint:
    case JVal::kDouble: return "number";
    case JVal::kString: return "string";
    case JVal::kArray: return "array";
    case JVal::kObject: return "object";
  }
  return "discarded";
}

[[noreturn]] void type_error_302(const char* want, const JVal& v) {
  throw SchemaError{std::string("[json.exception.type_error.302] type must be ") + want + ", but is " +
                    type_name(v)};
}

const JVal& at(const JVal& j, const char* key) {  // basic_json::at(key)
  if (j.kind != JVal::kObject)
    throw SchemaError{std::string("[json.exception.type_error.304] cannot use at() with ") + type_name(j)};
  const JVal* v = j.get(key);
  if (!v) throw SchemaError{std::string("[json.exception.out_of_range.403] key '") + key + "' not found"};
  return *v;
}

// nlohmann get<integral>: any JSON number, converted; booleans too, except for
// its own number_integer_t / number_unsigned_t (int64_t / uint64_t), whose
// from_json is get_arithmetic_value (json.hpp 3.11.3, from_json overloads).
template <typename T>
T as_int(const JVal& v) {
  switch (v.kind) {
    case JVal::kInt: return static_cast<T>(v.i);
    case JVal::kUint: return static_cast<T>(v.u);
    case JVal::kDouble: return static_cast<T>(v.d);
    case JVal::kBool:
      if (sizeof(T) == 8) type_error_302("number", v);
      return static_cast<T>(v.b);
    default: type_error_302("number", v);
  }
}

double as_double(const JVal& v) {  // get<double> = get_arithmetic_value: no booleans
  switch (v.kind) {
    case JVal::kInt: return static_cast<double>(v.i);
    case JVal::kUint: return static_cast<double>(v.u);
    case JVal::kDouble: return v.d;
    default: type_error_302("number", v);
  }
}

const std::string& as_string(const JVal& v) {
  if (v.kind != JVal::kString) type_error_302("string", v);
  return v.s;
}

// Range-for over a basic_json (json_io.cpp:49-50): an array yields its
// elements, an object its values in key order (std::map, duplicates: last
// wins), null nothing, any other value itself once.
std::vector<const JVal*> json_range(const JVal& j) {
  std::vector<const JVal*> out;
  if (j.kind == JVal::kArray) {
    for (const JVal& x : j.arr) out.push_back(&x);
  } else if (j.kind == JVal::kObject) {
    std::vector<std::pair<std::string, const JVal*>> m;
    for (auto it = j.obj.rbegin(); it != j.obj.rend(); ++it) {
      bool seen = false;
      for (const auto& e : m) seen |= e.first == it->first;
      if (!seen) m.emplace_back(it->first, &it->second);
    }
    std::sort(m.begin(), m.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    for (const auto& e : m) out.push_back(e.second);
  } else if (j.kind != JVal::kNull) {
    out.push_back(&j);
  }
  return out;
}

struct Entry {
  uint64_t id;
  int32_t prompt, est, prefill, decoded;
};

void entries_from(const JVal& arr, std::vector<Entry>* out) {
  for (const JVal* r : json_range(arr)) {  // snapshot_request_from_json_obj (json_io.cpp:21-29)
    Entry e{};
    e.id = as_int<uint64_t>(at(*r, "id"));
    e.prompt = as_int<int32_t>(at(*r, "prompt_tokens"));
    e.est = as_int<int32_t>(at(*r, "estimated_output_tokens"));
    e.prefill = as_int<int32_t>(at(*r, "prefill_progress"));
    e.decoded = as_int<int32_t>(at(*r, "decoded_tokens"));
    out->push_back(e);
  }
}

// A ConfigError (error.h:14-18) raised while parsing: passes parse_with's
// json::exception handler untouched.
struct ConfigErr {
  std::string what;
};

struct Request {
  std::vector<Entry> running, waiting;
  int32_t cand_prompt = 0, cand_est = 0;
  bsg_instance_cfg cfg{};
};

Request request_from(const JVal& j) {  // prediction_request_from_json (json_io.cpp:136-146)
  Request r;
  const JVal& snap = at(j, "snapshot");
  (void)as_int<int32_t>(at(snap, "instance_id"));
  (void)as_double(at(snap, "snapshot_time"));
  (void)as_int<int32_t>(at(snap, "free_blocks"));
  (void)as_int<int32_t>(at(snap, "batch_size"));
  (void)as_int<int32_t>(at(snap, "qpm"));
  entries_from(at(snap, "running"), &r.running);
  entries_from(at(snap, "waiting"), &r.waiting);
  const JVal& cand = at(j, "candidate");
  r.cand_prompt = as_int<int32_t>(at(cand, "prompt_tokens"));
  r.cand_est = as_int<int32_t>(at(cand, "estimated_output_tokens"));
  const JVal& c = at(j, "instance_config");  // instance_config_from_json_obj (json_io.cpp:69-84)
  (void)as_int<int32_t>(at(c, "instance_id"));
  r.cfg.total_blocks = as_int<int32_t>(at(c, "total_blocks"));
  r.cfg.block_size = as_int<int32_t>(at(c, "block_size"));
  r.cfg.max_batch_size = as_int<int32_t>(at(c, "max_batch_size"));
  r.cfg.chunk_budget = as_int<int32_t>(at(c, "chunk_budget"));
  const std::string& pol = as_string(at(c, "local_policy"));
  if (pol == "chunked_prefill") r.cfg.local_policy = BSG_CHUNKED_PREFILL;  // parse_local_policy (types.cpp:41-45)
  else if (pol == "prefill_priority") r.cfg.local_policy = BSG_PREFILL_PRIORITY;
  else throw ConfigErr{"invalid config: cluster.local_policy: unknown policy '" + pol + "'"};
  const JVal& cost = at(c, "cost_model");
  r.cfg.c0_s = as_double(at(cost, "c0_s"));
  r.cfg.prefill_s_per_token = as_double(at(cost, "prefill_s_per_token"));
  r.cfg.decode_s_per_seq = as_double(at(cost, "decode_s_per_seq"));
  r.cfg.context_s_per_token = as_double(at(cost, "context_s_per_token"));
  r.cfg.cache_mode = BSG_CACHE_EXACT;  // the predictor service's default cache (config.cpp:192)
  r.cfg.context_bucket = 256;
  return r;
}

// ---- nlohmann::json::dump number formatting -----------------------------------
// The reference prints doubles with nlohmann's dtoa: Grisu2 (Loitsch, "Printing
// Floating-Point Numbers Quickly and Accurately with Integers", PLDI 2010) with
// the boundaries narrowed by one unit, which is round-trip exact but not always
// shortest (e.g. 199.28768350000001). To answer byte-identically the digits are
// generated by the same algorithm here; the decimal layout follows dump():
// fixed notation for decimal exponents in (-4, 15], else d.ddde±XX.
struct DiyFp {
  uint64_t f;
  int e;
};

DiyFp diy_mul(DiyFp x, DiyFp y) {  // (x.f * y.f + 2^63) >> 64, rounded half up
  const unsigned __int128 p = static_cast<unsigned __int128>(x.f) * y.f;
  uint64_t h = static_cast<uint64_t>(p >> 64);
  h += static_cast<uint64_t>(p) >> 63;
  return DiyFp{h, x.e + y.e + 64};
}

DiyFp diy_normalize(DiyFp x) {
  while ((x.f >> 63) == 0) {
    x.f <<= 1;
    --x.e;
  }
  return x;
}

// Normalised 64-bit significands of 10^k, k = -300, -292, ..., 340 (round to
// nearest; generated with exact integer arithmetic).
struct CachedPower {
  uint64_t f;
  int e;
  int k;
};
constexpr CachedPower kCachedPowers[] = {
    {0xAB70FE17C79AC6CAULL, -1060, -300},
    {0xFF77B1FCBEBCDC4FULL, -1034, -292},
    {0xBE5691EF416BD60CULL, -1007, -284},
    {0x8DD01FAD907FFC3CULL, -980, -276},
    {0xD3515C2831559A83ULL, -954, -268},
    {0x9D71AC8FADA6C9B5ULL, -927, -260},
    {0xEA9C227723EE8BCBULL, -901, -252},
    {0xAECC49914078536DULL, -874, -244},
    {0x823C12795DB6CE57ULL, -847, -236},
    {0xC21094364DFB5637ULL, -821, -228},
    {0x9096EA6F3848984FULL, -794, -220},
    {0xD77485CB25823AC7ULL, -768, -212},
    {0xA086CFCD97BF97F4ULL, -741, -204},
    {0xEF340A98172AACE5ULL, -715, -196},
    {0xB23867FB2A35B28EULL, -688, -188},
    {0x84C8D4DFD2C63F3BULL, -661, -180},
    {0xC5DD44271AD3CDBAULL, -635, -172},
    {0x936B9FCEBB25C996ULL, -608, -164},
    {0xDBAC6C247D62A584ULL, -582, -156},
    {0xA3AB66580D5FDAF6ULL, -555, -148},
    {0xF3E2F893DEC3F126ULL, -529, -140},
    {0xB5B5ADA8AAFF80B8ULL, -502, -132},
    {0x87625F056C7C4A8BULL, -475, -124},
    {0xC9BCFF6034C13053ULL, -449, -116},
    {0x964E858C91BA2655ULL, -422, -108},
    {0xDFF9772470297EBDULL, -396, -100},
    {0xA6DFBD9FB8E5B88FULL, -369, -92},
    {0xF8A95FCF88747D94ULL, -343, -84},
    {0xB94470938FA89BCFULL, -316, -76},
    {0x8A08F0F8BF0F156BULL, -289, -68},
    {0xCDB02555653131B6ULL, -263, -60},
    {0x993FE2C6D07B7FACULL, -236, -52},
    {0xE45C10C42A2B3B06ULL, -210, -44},
    {0xAA242499697392D3ULL, -183, -36},
    {0xFD87B5F28300CA0EULL, -157, -28},
    {0xBCE5086492111AEBULL, -130, -20},
    {0x8CBCCC096F5088CCULL, -103, -12},
    {0xD1B71758E219652CULL, -77, -4},
    {0x9C40000000000000ULL, -50, 4},
    {0xE8D4A51000000000ULL, -24, 12},
    {0xAD78EBC5AC620000ULL, 3, 20},
    {0x813F3978F8940984ULL, 30, 28},
    {0xC097CE7BC90715B3ULL, 56, 36},
    {0x8F7E32CE7BEA5C70ULL, 83, 44},
    {0xD5D238A4ABE98068ULL, 109, 52},
    {0x9F4F2726179A2245ULL, 136, 60},
    {0xED63A231D4C4FB27ULL, 162, 68},
    {0xB0DE65388CC8ADA8ULL, 189, 76},
    {0x83C7088E1AAB65DBULL, 216, 84},
    {0xC45D1DF942711D9AULL, 242, 92},
    {0x924D692CA61BE758ULL, 269, 100},
    {0xDA01EE641A708DEAULL, 295, 108},
    {0xA26DA3999AEF774AULL, 322, 116},
    {0xF209787BB47D6B85ULL, 348, 124},
    {0xB454E4A179DD1877ULL, 375, 132},
    {0x865B86925B9BC5C2ULL, 402, 140},
    {0xC83553C5C8965D3DULL, 428, 148},
    {0x952AB45CFA97A0B3ULL, 455, 156},
    {0xDE469FBD99A05FE3ULL, 481, 164},
    {0xA59BC234DB398C25ULL, 508, 172},
    {0xF6C69A72A3989F5CULL, 534, 180},
    {0xB7DCBF5354E9BECEULL, 561, 188},
    {0x88FCF317F22241E2ULL, 588, 196},
    {0xCC20CE9BD35C78A5ULL, 614, 204},
    {0x98165AF37B2153DFULL, 641, 212},
    {0xE2A0B5DC971F303AULL, 667, 220},
    {0xA8D9D1535CE3B396ULL, 694, 228},
    {0xFB9B7CD9A4A7443CULL, 720, 236},
    {0xBB764C4CA7A44410ULL, 747, 244},
    {0x8BAB8EEFB6409C1AULL, 774, 252},
    {0xD01FEF10A657842CULL, 800, 260},
    {0x9B10A4E5E9913129ULL, 827, 268},
    {0xE7109BFBA19C0C9DULL, 853, 276},
    {0xAC2820D9623BF429ULL, 880, 284},
    {0x80444B5E7AA7CF85ULL, 907, 292},
    {0xBF21E44003ACDD2DULL, 933, 300},
    {0x8E679C2F5E44FF8FULL, 960, 308},
    {0xD433179D9C8CB841ULL, 986, 316},
    {0x9E19DB92B4E31BA9ULL, 1013, 324},
    {0xEB96BF6EBADF77D9ULL, 1039, 332},
    {0xAF87023B9BF0EE6BULL, 1066, 340},
};
constexpr int kCachedMinDecExp = -300, kCachedDecStep = 8;
constexpr int kAlpha = -60, kGamma = -32;  // target exponent range of the scaled values

CachedPower cached_power_for(int e) {  // c = 10^k with kAlpha <= e + c.e + 64 <= kGamma
  const int f = kAlpha - e - 1;
  const int k = (f * 78913) / (1 << 18) + (f > 0 ? 1 : 0);  // ceil(f * log10(2))
  const int index = (-kCachedMinDecExp + k + (kCachedDecStep - 1)) / kCachedDecStep;
  return kCachedPowers[index];
}

void grisu_round(char* buf, int len, uint64_t dist, uint64_t delta, uint64_t rest, uint64_t ten_k) {
  // move the last digit closer to w while the candidate stays inside (M-, M+)
  while (rest < dist && delta - rest >= ten_k &&
         (rest + ten_k < dist || dist - rest > rest + ten_k - dist)) {
    --buf[len - 1];
    rest += ten_k;
  }
}

// Digits of v (finite, > 0) and the decimal exponent: v ~ digits * 10^exp.
void grisu2(double value, char* buf, int* len, int* exp10) {
  uint64_t bits;
  std::memcpy(&bits, &value, 8);
  const uint64_t F = bits & ((uint64_t{1} << 52) - 1);
  const int E = static_cast<int>((bits >> 52) & 0x7ff);
  constexpr int kBias = 1075, kMinExp = 1 - kBias;
  const DiyFp v = E == 0 ? DiyFp{F, kMinExp} : DiyFp{F + (uint64_t{1} << 52), E - kBias};
  const bool lower_closer = F == 0 && E > 1;
  const DiyFp m_plus = diy_normalize(DiyFp{2 * v.f + 1, v.e - 1});
  DiyFp m_minus = lower_closer ? DiyFp{4 * v.f - 1, v.e - 2} : DiyFp{2 * v.f - 1, v.e - 1};
  m_minus.f <<= (m_minus.e - m_plus.e);
  m_minus.e = m_plus.e;
  const DiyFp w = diy_normalize(v);
  const CachedPower c = cached_power_for(m_plus.e);
  const DiyFp cp{c.f, c.e};
  const DiyFp sw = diy_mul(w, cp), sm = diy_mul(m_minus, cp), sp = diy_mul(m_plus, cp);
  const DiyFp M_minus{sm.f + 1, sm.e}, M_plus{sp.f - 1, sp.e};
  int dexp = -c.k;
  uint64_t delta = M_plus.f - M_minus.f, dist = M_plus.f - sw.f;
  const int shift = -M_plus.e;
  const uint64_t one_f = uint64_t{1} << shift;
  uint32_t p1 = static_cast<uint32_t>(M_plus.f >> shift);
  uint64_t p2 = M_plus.f & (one_f - 1);
  uint32_t pow10 = 1;
  int n = 1;
  while (n < 10 && p1 >= pow10 * 10u) {
    pow10 *= 10;
    ++n;
  }
  int L = 0;
  while (n > 0) {  // integral digits
    const uint32_t d = p1 / pow10, r = p1 % pow10;
    buf[L++] = static_cast<char>('0' + d);
    p1 = r;
    --n;
    const uint64_t rest = (static_cast<uint64_t>(p1) << shift) + p2;
    if (rest <= delta) {
      dexp += n;
      grisu_round(buf, L, dist, delta, rest, static_cast<uint64_t>(pow10) << shift);
      *len = L;
      *exp10 = dexp;
      return;
    }
    pow10 /= 10;
  }
  int m = 0;
  for (;;) {  // fractional digits
    p2 *= 10;
    delta *= 10;
    dist *= 10;
    buf[L++] = static_cast<char>('0' + (p2 >> shift));
    p2 &= one_f - 1;
    ++m;
    if (p2 <= delta) break;
  }
  dexp -= m;
  grisu_round(buf, L, dist, delta, p2, one_f);
  *len = L;
  *exp10 = dexp;
}

void append_double(std::string* out, double v) {
  if (!std::isfinite(v)) {
    out->append("null");
    return;
  }
  if (v == 0) {
    out->append(std::signbit(v) ? "-0.0" : "0.0");
    return;
  }
  if (v < 0) {
    out->push_back('-');
    v = -v;
  }
  char buf[32];
  int k = 0, dexp = 0;
  grisu2(v, buf, &k, &dexp);
  const std::string digits(buf, buf + k);
  const int n = k + dexp;  // value = 0.ddd x 10^n
  if (k <= n && n <= 15) {
    out->append(digits);
    out->append(static_cast<size_t>(n - k), '0');
    out->append(".0");
  } else if (0 < n && n <= 15) {
    out->append(digits, 0, static_cast<size_t>(n));
    out->push_back('.');
    out->append(digits, static_cast<size_t>(n), std::string::npos);
  } else if (-4 < n && n <= 0) {
    out->append("0.");
    out->append(static_cast<size_t>(-n), '0');
    out->append(digits);
  } else {
    out->push_back(digits[0]);
    if (k > 1) {
      out->push_back('.');
      out->append(digits, 1, std::string::npos);
    }
    out->push_back('e');
    const int ex = n - 1;
    out->push_back(ex < 0 ? '-' : '+');
    const int a = ex < 0 ? -ex : ex;
    if (a < 10) out->push_back('0');
    out->append(std::to_string(a));
  }
}

std::string escape(const std::string& s) {
  std::string o;
  for (char c : s) {
    if (c == '"' || c == '\\') {
      o.push_back('\\');
      o.push_back(c);
    } else if (c == '\b' || c == '\t' || c == '\n' || c == '\f' || c == '\r') {  // dump's short escapes
      o.push_back('\\');
      o.push_back(c == '\b' ? 'b' : c == '\t' ? 't' : c == '\n' ? 'n' : c == '\f' ? 'f' : 'r');
    } else if (static_cast<unsigned char>(c) < 0x20) {
      char b[8];
      std::snprintf(b, sizeof(b), "\\u%04x", c);
      o.append(b);
    } else {
      o.push_back(c);
    }
  }
  return o;
}

std::string error_body(const std::string& code, const std::string& detail) {  // json_io.cpp:148-152
  // nlohmann objects dump in key order: "detail" before "error"
  std::string o = "{";
  if (!detail.empty()) o += "\"detail\":\"" + escape(detail) + "\",";
  return o + "\"error\":\"" + escape(code) + "\"}";
}

// "invalid config: <field>: <rule>" of validate_instance_config (types.cpp:47-61)
// by bsg_check_config's field code.
std::string config_error_text(int32_t f) {
  static const char* const field[] = {"", "total_blocks", "block_size", "max_batch_size", "chunk_budget",
                                      "cost_model.c0_s", "cost_model.prefill_s_per_token",
                                      "cost_model.decode_s_per_seq", "cost_model.context_s_per_token"};
  static const char* const rule[] = {"", "must be >= 1", "must be >= 1", "must be >= 1",
                                     "must be >= block_size", "must be > 0", "must be >= 0", "must be >= 0",
                                     "must be >= 0"};
  return std::string("invalid config: ") + field[f] + ": " + rule[f];
}

// Parses one /predict body exactly as prediction_request_from_json
// (json_io.cpp:136-146) and runs predict()'s checks that precede simulation
// (the Instance ctor's validate_instance_config, backend.cpp:16-18). Returns
// true, or false with the reference's status / error body (json_io.cpp:148-152
// via service.cpp:229-241).
bool parse_predict_request(const char* t, Request* req, int32_t* status, std::string* body) {
  Parser ps{t, t + std::strlen(t), {}};
  JVal j;
  bool good = ps.value(&j);
  ps.ws();
  if (good && ps.p != ps.end) good = ps.fail("malformed JSON");
  if (!good) {
    *status = BSG_BAD_INPUT;
    *body = error_body("bad-schema", "bad-schema: malformed JSON");
    return false;
  }
  try {
    *req = request_from(j);
  } catch (const SchemaError& e) {
    *status = BSG_BAD_INPUT;
    *body = error_body("bad-schema", "bad-schema: " + e.what);
    return false;
  } catch (const ConfigErr& e) {
    *status = BSG_BAD_CONFIG;
    *body = error_body("bad-schema", e.what);
    return false;
  }
  int32_t f = 0;
  const bsg_status v = bsg_check_config(req->cfg, &f);
  if (v == BSG_BAD_CONFIG) {  // ConfigError is an Error: 400
    *status = BSG_BAD_CONFIG;
    *body = error_body("bad-schema", config_error_text(f));
    return false;
  }
  if (v != BSG_OK) {  // outside the supported integer domain: a prediction failure, never a silent fallback
    *status = BSG_BAD_INPUT;
    *body = error_body("prediction-failure", "instance config outside the GPU simulator's supported domain "
                                             "(total_blocks * block_size <= 2^30, block_size <= 2^20, "
                                             "chunk_budget <= 2^30)");
    return false;
  }
  return true;
}

// The response body of a simulated request (service.cpp:229-241): the
// PredictionResult, or PredictionError's message (predictor.cpp:101-136),
// rebuilt from the result's status and detail.
std::string result_body(const Request& r, const bsg_result& x) {
  auto entry_id = [&](int32_t origin) -> uint64_t {  // origin: running i, waiting run_n + j, candidate -1
    uint64_t cand = 0;  // candidate id: max snapshot id + 1 (predictor.cpp:79-82)
    for (const Entry& e : r.running) cand = std::max(cand, e.id);
    for (const Entry& e : r.waiting) cand = std::max(cand, e.id);
    cand += 1;
    const int32_t rn = static_cast<int32_t>(r.running.size());
    if (origin < 0) return cand;
    return origin < rn ? r.running[origin].id : r.waiting[origin - rn].id;
  };
  switch (x.status) {
    case BSG_OK: {  // prediction_result_to_json (json_io.cpp:103-108): std::map key order
      std::string o = "{\"metrics\":{\"predicted_e2e_latency\":";
      append_double(&o, bsg_ticks_to_seconds(x.e2e_ticks));
      o += ",\"predicted_queueing_delay\":";
      append_double(&o, bsg_ticks_to_seconds(x.qdelay_ticks));
      o += ",\"predicted_ttft\":";
      append_double(&o, bsg_ticks_to_seconds(x.ttft_ticks));
      o += "},\"simulated_steps\":" + std::to_string(x.steps) + "}";
      return o;
    }
    case BSG_TOO_LARGE_RUNNING:  // backend.cpp:42-44, re-thrown at predictor.cpp:134-135
      return error_body("prediction-failure",
                        "candidate does not fit the instance: snapshot running set exceeds total memory blocks");
    case BSG_TOO_LARGE_CANDIDATE:  // backend.cpp:76-83
      return error_body("prediction-failure", "candidate does not fit the instance: request " +
                                                  std::to_string(entry_id(-1)) + " needs " +
                                                  std::to_string(x.detail) + " blocks, instance has " +
                                                  std::to_string(r.cfg.total_blocks));
    case BSG_DEADLOCK:  // backend.cpp:274-277, predictor.cpp:132-133
      return error_body("prediction-failure", "backend deadlock during forward simulation: request " +
                                                  std::to_string(entry_id(x.detail)) +
                                                  " cannot proceed with the whole memory free");
    case BSG_STEP_LIMIT:
      return error_body("prediction-failure", "forward simulation exceeded the step limit");
    case BSG_VANISHED:
      return error_body("prediction-failure", "candidate vanished from the forward simulation");
    case BSG_EMPTY_PLAN:  // EmptyPlanError is an Error, not a PredictionError: 400 (backend.cpp:245)
      return error_body("bad-schema", "no runnable work fits the batch");
    default:  // out-of-domain snapshot values: the GPU simulator refuses them explicitly
      return error_body("prediction-failure",
                        "snapshot outside the GPU simulator's supported domain (DESIGN.md §4)");
  }
}

}  // namespace

extern "C" bsg_status bsg_predict_json(bsg_ctx* ctx, const char* const* requests, int32_t n,
                                       char* out, int64_t out_cap, int64_t* out_off,
                                       int32_t* status) {
  if (!ctx || (!requests && n > 0) || n < 0 || !out_off || !status) return BSG_INVALID_ARGUMENT;
  std::vector<std::string> body(static_cast<size_t>(n));
  std::vector<Request> reqs(static_cast<size_t>(n));
  std::vector<int> ok(static_cast<size_t>(n), 0);
  // parse + per-request config validation: each request fails on its own, like
  // the reference role handles each /predict independently
  std::vector<bsg_instance_cfg> cfgs;
  std::vector<int32_t> cfg_of(static_cast<size_t>(n), 0);
  for (int32_t q = 0; q < n; ++q) {
    if (!parse_predict_request(requests[q] ? requests[q] : "", &reqs[q], &status[q], &body[q])) continue;
    int32_t ci = -1;
    for (size_t c = 0; c < cfgs.size() && ci < 0; ++c)
      if (std::memcmp(&cfgs[c], &reqs[q].cfg, sizeof(bsg_instance_cfg)) == 0) ci = static_cast<int32_t>(c);
    if (ci < 0) {
      ci = static_cast<int32_t>(cfgs.size());
      cfgs.push_back(reqs[q].cfg);
    }
    cfg_of[q] = ci;
    ok[q] = 1;
  }
  // one GPU batch over every well-formed request (its configs all validated)
  if (!cfgs.empty()) {
    int32_t bi = -1, fc = 0;
    const bsg_status cs = bsg_set_configs(ctx, cfgs.data(), static_cast<int32_t>(cfgs.size()), &bi, &fc);
    if (cs != BSG_OK) return cs;
  }
  std::vector<int32_t> rows;
  std::vector<uint64_t> id;
  std::vector<int32_t> prompt, est, prefill, decoded;
  std::vector<bsg_scenario> scen;
  for (int32_t q = 0; q < n; ++q) {
    if (!ok[q]) continue;
    const Request& r = reqs[q];
    bsg_scenario s{};
    s.run_off = static_cast<int32_t>(prompt.size());
    s.run_n = static_cast<int32_t>(r.running.size());
    auto add = [&](const Entry& e) {
      id.push_back(e.id);
      prompt.push_back(e.prompt);
      est.push_back(e.est);
      prefill.push_back(e.prefill);
      decoded.push_back(e.decoded);
    };
    for (const Entry& e : r.running) add(e);
    s.wait_off = static_cast<int32_t>(prompt.size());
    s.wait_n = static_cast<int32_t>(r.waiting.size());
    for (const Entry& e : r.waiting) add(e);
    s.cand_prompt = r.cand_prompt;
    s.cand_est = r.cand_est;
    s.cfg = cfg_of[q];
    scen.push_back(s);
    rows.push_back(q);
  }
  if (!scen.empty()) {
    std::vector<bsg_result> res(scen.size());
    bsg_entries e{id.data(), prompt.data(), est.data(), prefill.data(), decoded.data()};
    const bsg_status st = bsg_predict_batch(ctx, &e, static_cast<int64_t>(prompt.size()), scen.data(),
                                            static_cast<int64_t>(scen.size()), res.data());
    if (st != BSG_OK) return st;
    for (size_t k = 0; k < rows.size(); ++k) {
      status[rows[k]] = res[k].status;
      body[rows[k]] = result_body(reqs[rows[k]], res[k]);
    }
  }
  int64_t off = 0;
  for (int32_t q = 0; q < n; ++q) {
    out_off[q] = off;
    const int64_t len = static_cast<int64_t>(body[q].size()) + 1;  // NUL-terminated
    if (off + len <= out_cap && out) {
      std::memcpy(out + off, body[q].c_str(), static_cast<size_t>(len));
    }
    off += len;
  }
  out_off[n] = off;
  return off <= out_cap ? BSG_OK : BSG_INVALID_ARGUMENT;  // out_off[n] = bytes needed
}

extern "C" int32_t bsg_wire_check(const char* body, char* out, int64_t cap) {
  if (!body) return BSG_INVALID_ARGUMENT;
  Request r;
  int32_t st = BSG_OK;
  std::string text;
  if (parse_predict_request(body, &r, &st, &text)) return BSG_OK;
  if (out && cap > 0) std::snprintf(out, static_cast<size_t>(cap), "%s", text.c_str());
  return st;
}

// ---- trace JSONL (workload.cpp:20-68) --------------------------------------
namespace {

void set_err(bsg_trace_error* err, int32_t kind, int32_t line, const std::string& field,
             const std::string& msg) {
  if (!err) return;
  err->kind = kind;
  err->line = line;
  std::snprintf(err->field, sizeof(err->field), "%s", field.c_str());
  std::snprintf(err->message, sizeof(err->message), "%s", msg.c_str());
}

// record_from_json (workload.cpp:20-36): a missing or mistyped field is a
// TraceParseError of its line; `contains` + get, so an explicit null in an
// optional field is mistyped, not absent.
bsg_trace_record record_from(const JVal& j) {
  bsg_trace_record r{};
  r.id = as_int<uint64_t>(at(j, "id"));
  r.prompt_tokens = as_int<int32_t>(at(j, "prompt_tokens"));
  r.output_tokens = as_int<int32_t>(at(j, "output_tokens"));
  if (j.kind == JVal::kObject && j.get("estimated_output_tokens")) {
    // validate_record rejects a present estimate < 1, so 0 is free to mean
    // "absent" in the flat record
    r.estimated_output_tokens = as_int<int32_t>(*j.get("estimated_output_tokens"));
  }
  if (j.kind == JVal::kObject && j.get("arrival_offset_s")) {
    r.arrival_offset_s = as_double(*j.get("arrival_offset_s"));
    r.has_arrival_offset = 1;
  }
  return r;
}

}  // namespace

extern "C" bsg_status bsg_load_trace(const char* text, int64_t len, bsg_trace_record* out,
                                     int64_t cap, int64_t* n_records, bsg_trace_error* err) {
  if ((!text && len > 0) || len < 0 || cap < 0 || (!out && cap > 0) || !n_records)
    return BSG_INVALID_ARGUMENT;
  set_err(err, 0, 0, "", "");
  *n_records = 0;
  std::unordered_set<uint64_t> seen;
  int64_t n = 0;
  int32_t line_number = 0;
  const char* p = text;
  const char* const end = text + len;
  while (p < end) {
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(end - p)));
    const char* line_end = nl ? nl : end;
    ++line_number;
    const char* a = p;
    p = nl ? nl + 1 : end;
    bool blank = true;
    for (const char* c = a; c < line_end && blank; ++c) blank = (*c == ' ' || *c == '\t' || *c == '\r');
    if (blank) continue;
    Parser ps{a, line_end, {}};
    JVal j;
    bool good = ps.value(&j);
    ps.ws();
    if (good && ps.p != ps.end) good = false;
    if (!good) {
      set_err(err, 1, line_number, "",
              "trace parse error at line " + std::to_string(line_number) + ": malformed JSON");
      return BSG_BAD_INPUT;
    }
    bsg_trace_record r;
    try {
      r = record_from(j);
    } catch (const SchemaError& e) {
      set_err(err, 1, line_number, "",
              "trace parse error at line " + std::to_string(line_number) + ": " + e.what);
      return BSG_BAD_INPUT;
    }
    // validate_record (workload.cpp:38-47)
    const char* bad = nullptr;
    if (r.prompt_tokens < 1) bad = "prompt_tokens";
    else if (r.output_tokens < 1) bad = "output_tokens";
    else if (j.get("estimated_output_tokens") && r.estimated_output_tokens < 1) bad = "estimated_output_tokens";
    else if (r.has_arrival_offset && r.arrival_offset_s < 0) bad = "arrival_offset_s";
    if (bad) {
      set_err(err, 2, line_number, bad,
              std::string("invalid trace record: ") + bad + ": must be >= " +
                  (std::strcmp(bad, "arrival_offset_s") == 0 ? "0" : "1"));
      return BSG_BAD_INPUT;
    }
    if (!seen.insert(r.id).second) {
      set_err(err, 2, line_number, "id",
              "invalid trace record: id: duplicate id " + std::to_string(r.id));
      return BSG_BAD_INPUT;
    }
    if (n < cap) out[n] = r;
    ++n;
  }
  *n_records = n;
  return n > cap ? BSG_INVALID_ARGUMENT : BSG_OK;
}

// write_trace (workload.cpp:78-89): one nlohmann object per line — its keys
// in std::map order, no whitespace, numbers as dump() prints them.
extern "C" bsg_status bsg_write_trace(const bsg_trace_record* recs, int64_t n, char* out,
                                      int64_t cap, int64_t* len) {
  if ((!recs && n > 0) || n < 0 || cap < 0 || (!out && cap > 0) || !len) return BSG_INVALID_ARGUMENT;
  std::string s;
  s.reserve(static_cast<size_t>(n) * 96);
  for (int64_t i = 0; i < n; ++i) {
    const bsg_trace_record& r = recs[i];
    s.push_back('{');
    if (r.has_arrival_offset) {
      s.append("\"arrival_offset_s\":");
      append_double(&s, r.arrival_offset_s);
      s.push_back(',');
    }
    if (r.estimated_output_tokens > 0) {
      s.append("\"estimated_output_tokens\":");
      s.append(std::to_string(r.estimated_output_tokens));
      s.push_back(',');
    }
    s.append("\"id\":");
    s.append(std::to_string(r.id));
    s.append(",\"output_tokens\":");
    s.append(std::to_string(r.output_tokens));
    s.append(",\"prompt_tokens\":");
    s.append(std::to_string(r.prompt_tokens));
    s.append("}\n");
  }
  *len = static_cast<int64_t>(s.size());
  if (*len > cap) return BSG_INVALID_ARGUMENT;
  std::memcpy(out, s.data(), s.size());
  return BSG_OK;
}

extern "C" int32_t bsg_format_double(double v, char* out, int32_t cap) {
  std::string t;
  append_double(&t, v);
  if (!out || cap < static_cast<int32_t>(t.size()) + 1) return -static_cast<int32_t>(t.size() + 1);
  std::memcpy(out, t.c_str(), t.size() + 1);
  return static_cast<int32_t>(t.size());
}
