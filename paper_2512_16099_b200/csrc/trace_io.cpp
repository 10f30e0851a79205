// trace_io.cpp — trace ingest: migsched::load_trace (workload.cpp:151-199)
// as a native, parallel JSONL reader feeding msg_trace_batch.
//
// Semantics follow the reference line for line:
//   * lines split on '\n' (std::getline); a line of only ' ', '\t', '\r' is
//     skipped; line numbers count every line;
//   * each line must be one complete JSON text (RFC 8259, as nlohmann/json
//     3.11 parses it: strict numbers, escapes and UTF-8, no comments, no
//     trailing characters) — else "line N: not valid JSON";
//   * it must be an object; a "schema" member must compare equal to 1
//     (integer 1, unsigned 1 or 1.0);
//   * job_id (int64), arrival_s, service_s (double) with nlohmann's
//     conversions (floats truncate to integers, integers widen to double);
//     a missing or non-numeric one (booleans included) is "missing or
//     mistyped field"; the last duplicate key wins;
//   * profile must name one of the six profiles (UnknownProfile);
//   * arrival_s < 0 or service_s <= 0 is a ParseError;
//   * the first failing line (in file order) decides the error;
//   * jobs are stable-sorted by arrival time.
// Lines are parsed in parallel on the host pool; the reference parses one
// line at a time.  Deviation: a "profile" member that is not a string makes
// the reference throw nlohmann's type_error (not a migsched::Error); here it
// is a ParseError.
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <string_view>
#include <vector>

#include "runtime.h"

using namespace msgk;

namespace {

struct JVal {
    enum Kind { Null, Bool, Int, Uint, Float, Str, Obj, Arr } kind = Null;
    bool b = false;
    int64_t i = 0;
    uint64_t u = 0;
    double d = 0.0;
    std::string s;
};

// Strict recursive-descent JSON validator/reader.  Only the top-level
// object's member values are materialised; nested containers are validated
// and reported as Obj / Arr.
class JsonLine {
  public:
    explicit JsonLine(std::string_view t) : p_(t.data()), e_(t.data() + t.size()) {}

    // Parses the whole line as one object; false if not valid JSON.  Sets
    // is_object = false for a valid non-object text.
    bool parse_top(std::vector<std::pair<std::string, JVal>>& members, bool& is_object) {
        ws();
        is_object = p_ < e_ && *p_ == '{';
        if (is_object) {
            if (!object(0, &members)) return false;
        } else {
            JVal v;
            if (!value(0, v, false)) return false;
        }
        ws();
        return p_ == e_;
    }

  private:
    const char* p_;
    const char* e_;
    static constexpr int kMaxDepth = 4096;

    void ws() {
        while (p_ < e_ && (*p_ == ' ' || *p_ == '\t' || *p_ == '\n' || *p_ == '\r')) ++p_;
    }
    bool lit(const char* w) {
        const size_t n = std::strlen(w);
        if ((size_t)(e_ - p_) < n || std::memcmp(p_, w, n) != 0) return false;
        p_ += n;
        return true;
    }
    bool value(int depth, JVal& v, bool keep) {
        if (depth > kMaxDepth || p_ >= e_) return false;
        switch (*p_) {
            case '{':
                v.kind = JVal::Obj;
                return object(depth + 1, nullptr);
            case '[':
                v.kind = JVal::Arr;
                return array(depth + 1);
            case '"':
                v.kind = JVal::Str;
                return string(keep ? &v.s : nullptr);
            case 't':
                v.kind = JVal::Bool;
                v.b = true;
                return lit("true");
            case 'f':
                v.kind = JVal::Bool;
                v.b = false;
                return lit("false");
            case 'n':
                v.kind = JVal::Null;
                return lit("null");
            default:
                return number(v);
        }
    }
    bool object(int depth, std::vector<std::pair<std::string, JVal>>* members) {
        ++p_;  // '{'
        ws();
        if (p_ < e_ && *p_ == '}') {
            ++p_;
            return true;
        }
        for (;;) {
            ws();
            if (p_ >= e_ || *p_ != '"') return false;
            std::string key;
            if (!string(members ? &key : nullptr)) return false;
            ws();
            if (p_ >= e_ || *p_ != ':') return false;
            ++p_;
            ws();
            JVal v;
            if (!value(depth, v, members != nullptr)) return false;
            if (members) members->emplace_back(std::move(key), std::move(v));
            ws();
            if (p_ < e_ && *p_ == ',') {
                ++p_;
                continue;
            }
            if (p_ < e_ && *p_ == '}') {
                ++p_;
                return true;
            }
            return false;
        }
    }
    bool array(int depth) {
        ++p_;  // '['
        ws();
        if (p_ < e_ && *p_ == ']') {
            ++p_;
            return true;
        }
        for (;;) {
            ws();
            JVal v;
            if (!value(depth, v, false)) return false;
            ws();
            if (p_ < e_ && *p_ == ',') {
                ++p_;
                continue;
            }
            if (p_ < e_ && *p_ == ']') {
                ++p_;
                return true;
            }
            return false;
        }
    }
    static int hex(char c) {
        if (c >= '0' && c <= '9') return c - '0';
        if (c >= 'a' && c <= 'f') return c - 'a' + 10;
        if (c >= 'A' && c <= 'F') return c - 'A' + 10;
        return -1;
    }
    bool hex4(unsigned& cp) {
        if (e_ - p_ < 4) return false;
        cp = 0;
        for (int k = 0; k < 4; ++k) {
            const int h = hex(p_[k]);
            if (h < 0) return false;
            cp = cp * 16 + (unsigned)h;
        }
        p_ += 4;
        return true;
    }
    static void put_utf8(std::string* out, unsigned cp) {
        if (!out) return;
        if (cp < 0x80) {
            out->push_back((char)cp);
        } else if (cp < 0x800) {
            out->push_back((char)(0xC0 | (cp >> 6)));
            out->push_back((char)(0x80 | (cp & 0x3F)));
        } else if (cp < 0x10000) {
            out->push_back((char)(0xE0 | (cp >> 12)));
            out->push_back((char)(0x80 | ((cp >> 6) & 0x3F)));
            out->push_back((char)(0x80 | (cp & 0x3F)));
        } else {
            out->push_back((char)(0xF0 | (cp >> 18)));
            out->push_back((char)(0x80 | ((cp >> 12) & 0x3F)));
            out->push_back((char)(0x80 | ((cp >> 6) & 0x3F)));
            out->push_back((char)(0x80 | (cp & 0x3F)));
        }
    }
    // UTF-8 sequence ranges of RFC 3629 (the nlohmann lexer's checks).
    bool utf8(std::string* out) {
        const unsigned char c = (unsigned char)*p_;
        int n = 0;
        unsigned char lo = 0x80, hi = 0xBF;
        if (c >= 0xC2 && c <= 0xDF) {
            n = 1;
        } else if (c == 0xE0) {
            n = 2;
            lo = 0xA0;
        } else if ((c >= 0xE1 && c <= 0xEC) || c == 0xEE || c == 0xEF) {
            n = 2;
        } else if (c == 0xED) {
            n = 2;
            hi = 0x9F;
        } else if (c == 0xF0) {
            n = 3;
            lo = 0x90;
        } else if (c >= 0xF1 && c <= 0xF3) {
            n = 3;
        } else if (c == 0xF4) {
            n = 3;
            hi = 0x8F;
        } else {
            return false;
        }
        if (e_ - p_ < n + 1) return false;
        for (int k = 1; k <= n; ++k) {
            const unsigned char x = (unsigned char)p_[k];
            const unsigned char l = k == 1 ? lo : 0x80, h = k == 1 ? hi : 0xBF;
            if (x < l || x > h) return false;
        }
        if (out) out->append(p_, (size_t)n + 1);
        p_ += n + 1;
        return true;
    }
    bool string(std::string* out) {
        ++p_;  // '"'
        while (p_ < e_) {
            const unsigned char c = (unsigned char)*p_;
            if (c == '"') {
                ++p_;
                return true;
            }
            if (c < 0x20) return false;
            if (c == '\\') {
                if (++p_ >= e_) return false;
                const char x = *p_++;
                switch (x) {
                    case '"': if (out) out->push_back('"'); break;
                    case '\\': if (out) out->push_back('\\'); break;
                    case '/': if (out) out->push_back('/'); break;
                    case 'b': if (out) out->push_back('\b'); break;
                    case 'f': if (out) out->push_back('\f'); break;
                    case 'n': if (out) out->push_back('\n'); break;
                    case 'r': if (out) out->push_back('\r'); break;
                    case 't': if (out) out->push_back('\t'); break;
                    case 'u': {
                        unsigned cp;
                        if (!hex4(cp)) return false;
                        if (cp >= 0xD800 && cp <= 0xDBFF) {  // high surrogate: a low one must follow
                            unsigned lo;
                            if (e_ - p_ < 2 || p_[0] != '\\' || p_[1] != 'u') return false;
                            p_ += 2;
                            if (!hex4(lo) || lo < 0xDC00 || lo > 0xDFFF) return false;
                            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                        } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
                            return false;
                        }
                        put_utf8(out, cp);
                        break;
                    }
                    default:
                        return false;
                }
                continue;
            }
            if (c < 0x80) {
                if (out) out->push_back((char)c);
                ++p_;
                continue;
            }
            if (!utf8(out)) return false;
        }
        return false;
    }
    // -?(0|[1-9][0-9]*)(\.[0-9]+)?([eE][+-]?[0-9]+)?  — integers that fit
    // int64 (negative) / uint64 become Int / Uint (strtoll / strtoull), the
    // rest Float (strtod), like nlohmann's lexer.
    bool number(JVal& v) {
        const char* b = p_;
        bool neg = false, flt = false;
        if (p_ < e_ && *p_ == '-') {
            neg = true;
            ++p_;
        }
        if (p_ >= e_) return false;
        if (*p_ == '0') {
            ++p_;
        } else if (*p_ >= '1' && *p_ <= '9') {
            while (p_ < e_ && *p_ >= '0' && *p_ <= '9') ++p_;
        } else {
            return false;
        }
        if (p_ < e_ && *p_ == '.') {
            flt = true;
            ++p_;
            if (p_ >= e_ || *p_ < '0' || *p_ > '9') return false;
            while (p_ < e_ && *p_ >= '0' && *p_ <= '9') ++p_;
        }
        if (p_ < e_ && (*p_ == 'e' || *p_ == 'E')) {
            flt = true;
            ++p_;
            if (p_ < e_ && (*p_ == '+' || *p_ == '-')) ++p_;
            if (p_ >= e_ || *p_ < '0' || *p_ > '9') return false;
            while (p_ < e_ && *p_ >= '0' && *p_ <= '9') ++p_;
        }
        const std::string tok(b, (size_t)(p_ - b));
        if (!flt) {
            errno = 0;
            char* end = nullptr;
            if (neg) {
                const long long x = std::strtoll(tok.c_str(), &end, 10);
                if (errno == 0 && end == tok.c_str() + tok.size()) {
                    v.kind = JVal::Int;
                    v.i = x;
                    return true;
                }
            } else {
                const unsigned long long x = std::strtoull(tok.c_str(), &end, 10);
                if (errno == 0 && end == tok.c_str() + tok.size()) {
                    v.kind = JVal::Uint;
                    v.u = x;
                    return true;
                }
            }
        }
        v.kind = JVal::Float;
        v.d = std::strtod(tok.c_str(), nullptr);
        return true;
    }
};

// nlohmann's get<ArithmeticType> (from_json for arithmetic types).
bool as_int64(const JVal& v, int64_t& out) {
    switch (v.kind) {
        case JVal::Int: out = v.i; return true;
        case JVal::Uint: out = (int64_t)v.u; return true;
        case JVal::Float: out = (int64_t)v.d; return true;  // cvttsd2si, as the reference's static_cast
        default: return false;                              // booleans included (type_error in 3.11)
    }
}
bool as_double(const JVal& v, double& out) {
    switch (v.kind) {
        case JVal::Int: out = (double)v.i; return true;
        case JVal::Uint: out = (double)v.u; return true;
        case JVal::Float: out = v.d; return true;
        default: return false;
    }
}
bool equals_one(const JVal& v) {  // basic_json == 1 (numbers compare across kinds)
    switch (v.kind) {
        case JVal::Int: return v.i == 1;
        case JVal::Uint: return v.u == 1;
        case JVal::Float: return v.d == 1.0;
        default: return false;
    }
}

const char* const kProfileNames[6] = {"7g.40gb", "4g.20gb", "3g.20gb", "2g.10gb", "1g.10gb", "1g.5gb"};

struct LineOut {
    msg_status status = MSG_OK;
    std::string message;
    bool skip = false;
    int64_t id = 0;
    double arrival = 0.0, service = 0.0;
    int32_t profile = 0;
};

void parse_line(std::string_view line, int line_no, LineOut& o) {
    if (line.find_first_not_of(" \t\r") == std::string_view::npos) {
        o.skip = true;
        return;
    }
    const std::string ln = "line " + std::to_string(line_no) + ": ";
    auto fail = [&](msg_status st, const std::string& m) {
        o.status = st;
        o.message = m;
    };
    std::vector<std::pair<std::string, JVal>> mem;
    bool is_obj = false;
    JsonLine jl(line);
    if (!jl.parse_top(mem, is_obj)) return fail(MSG_ERR_PARSE_ERROR, "ParseError: " + ln + "not valid JSON");
    if (!is_obj) return fail(MSG_ERR_PARSE_ERROR, "ParseError: " + ln + "expected an object");
    auto find = [&](const char* k) -> const JVal* {  // the last duplicate wins
        for (auto it = mem.rbegin(); it != mem.rend(); ++it)
            if (it->first == k) return &it->second;
        return nullptr;
    };
    if (const JVal* s = find("schema"); s && !equals_one(*s))
        return fail(MSG_ERR_PARSE_ERROR, "ParseError: " + ln + "unsupported schema version");
    const JVal* jid = find("job_id");
    const JVal* ja = find("arrival_s");
    const JVal* js = find("service_s");
    if (!jid || !ja || !js || !as_int64(*jid, o.id) || !as_double(*ja, o.arrival) || !as_double(*js, o.service))
        return fail(MSG_ERR_PARSE_ERROR, "ParseError: " + ln + "missing or mistyped field");
    std::string name;
    if (const JVal* jp = find("profile")) {
        if (jp->kind != JVal::Str) return fail(MSG_ERR_PARSE_ERROR, "ParseError: " + ln + "profile is not a string");
        name = jp->s;
    }
    int pid = -1;
    for (int k = 0; k < 6; ++k)
        if (name == kProfileNames[k]) pid = k;
    if (pid < 0) return fail(MSG_ERR_UNKNOWN_PROFILE, "UnknownProfile: " + ln + "profile \"" + name + "\"");
    o.profile = pid;
    if (o.arrival < 0.0 || o.service <= 0.0)
        return fail(MSG_ERR_PARSE_ERROR, "ParseError: " + ln + "times must be non-negative");
}

}  // namespace

struct msg_trace_file {
    std::vector<int64_t> id;
    std::vector<double> arrival, service;
    std::vector<int32_t> profile;
};

extern "C" {

msg_status msg_trace_load(const char* path, msg_trace_file** out, char* msg, size_t msg_len) {
    auto set_msg = [&](const std::string& m) {
        if (msg && msg_len) std::snprintf(msg, msg_len, "%s", m.c_str());
    };
    if (!path || !out) return MSG_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    set_msg("");
    std::FILE* f = std::fopen(path, "rb");
    if (!f) {
        set_msg(std::string("ParseError: cannot open trace file ") + path);
        return MSG_ERR_PARSE_ERROR;
    }
    std::string buf;
    char chunk[1 << 16];
    size_t n;
    while ((n = std::fread(chunk, 1, sizeof(chunk), f)) > 0) buf.append(chunk, n);
    std::fclose(f);
    // std::getline lines: split on '\n'; a trailing segment without '\n' is a line if non-empty
    std::vector<std::string_view> lines;
    size_t b = 0;
    for (size_t i = 0; i < buf.size(); ++i)
        if (buf[i] == '\n') {
            lines.emplace_back(buf.data() + b, i - b);
            b = i + 1;
        }
    if (b < buf.size()) lines.emplace_back(buf.data() + b, buf.size() - b);
    std::vector<LineOut> res(lines.size());
    parallel_for((uint32_t)lines.size(), 256, [&](uint32_t i) { parse_line(lines[i], (int)i + 1, res[i]); });
    auto t = std::make_unique<msg_trace_file>();
    std::vector<uint32_t> order;
    order.reserve(lines.size());
    for (uint32_t i = 0; i < res.size(); ++i) {
        if (res[i].skip) continue;
        if (res[i].status != MSG_OK) {
            set_msg(res[i].message);
            return res[i].status;
        }
        order.push_back(i);
    }
    std::stable_sort(order.begin(), order.end(),
                     [&](uint32_t x, uint32_t y) { return res[x].arrival < res[y].arrival; });
    t->id.reserve(order.size());
    for (uint32_t i : order) {
        t->id.push_back(res[i].id);
        t->arrival.push_back(res[i].arrival);
        t->profile.push_back(res[i].profile);
        t->service.push_back(res[i].service);
    }
    *out = t.release();
    return MSG_OK;
}

uint64_t msg_trace_file_jobs(const msg_trace_file* f) { return f ? f->id.size() : 0; }
const int64_t* msg_trace_file_ids(const msg_trace_file* f) { return f && !f->id.empty() ? f->id.data() : nullptr; }
const double* msg_trace_file_arrival(const msg_trace_file* f) {
    return f && !f->arrival.empty() ? f->arrival.data() : nullptr;
}
const int32_t* msg_trace_file_profile(const msg_trace_file* f) {
    return f && !f->profile.empty() ? f->profile.data() : nullptr;
}
const double* msg_trace_file_service(const msg_trace_file* f) {
    return f && !f->service.empty() ? f->service.data() : nullptr;
}
void msg_trace_file_free(msg_trace_file* f) { delete f; }

}  // extern "C"
