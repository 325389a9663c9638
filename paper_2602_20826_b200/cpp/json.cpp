// Internal JSON value: parser and nlohmann-layout dump (json.hpp).
#include "json.hpp"

#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <limits>
#include <stdexcept>

namespace dagsched::detail {

Json Json::boolean(bool b) {
    Json j;
    j.kind_ = Kind::boolean;
    j.b_ = b;
    return j;
}
Json Json::integer(std::int64_t v) {
    Json j;
    j.kind_ = Kind::integer;
    j.i_ = v;
    return j;
}
Json Json::unsigned_integer(std::uint64_t v) {
    Json j;
    j.kind_ = Kind::unsigned_integer;
    j.u_ = v;
    return j;
}
Json Json::floating(double v) {
    Json j;
    j.kind_ = Kind::floating;
    j.d_ = v;
    return j;
}
Json Json::string(std::string s) {
    Json j;
    j.kind_ = Kind::string;
    j.s_ = std::move(s);
    return j;
}
Json Json::array() {
    Json j;
    j.kind_ = Kind::array;
    return j;
}
Json Json::object() {
    Json j;
    j.kind_ = Kind::object;
    return j;
}

namespace {
[[noreturn]] void type_error(const char* want) { throw JsonError(std::string("type must be ") + want); }
}  // namespace

const std::string& Json::str() const {
    if (kind_ != Kind::string) type_error("string");
    return s_;
}
long long Json::as_int64() const {
    switch (kind_) {
        case Kind::integer: return i_;
        case Kind::unsigned_integer: return static_cast<long long>(u_);
        case Kind::floating: return static_cast<long long>(d_);
        case Kind::boolean: return b_ ? 1 : 0;
        default: type_error("number");
    }
}
std::uint32_t Json::as_uint32() const {
    switch (kind_) {
        case Kind::integer: return static_cast<std::uint32_t>(i_);
        case Kind::unsigned_integer: return static_cast<std::uint32_t>(u_);
        case Kind::floating: return static_cast<std::uint32_t>(static_cast<long long>(d_));
        case Kind::boolean: return b_ ? 1u : 0u;
        default: type_error("number");
    }
}
double Json::as_double() const {
    switch (kind_) {
        case Kind::integer: return double(i_);
        case Kind::unsigned_integer: return double(u_);
        case Kind::floating: return d_;
        default: type_error("number");
    }
}
bool Json::contains(const std::string& key) const { return kind_ == Kind::object && o_.count(key) > 0; }
const Json& Json::at(const std::string& key) const {
    if (kind_ != Kind::object) type_error("object");
    auto it = o_.find(key);
    if (it == o_.end()) throw JsonError("key '" + key + "' not found");
    return it->second;
}
const Json& Json::operator[](std::size_t i) const {
    if (kind_ != Kind::array) type_error("array");
    if (i >= a_.size()) throw JsonError("array index out of range");
    return a_[i];
}
std::size_t Json::size() const {
    switch (kind_) {
        case Kind::null: return 0;
        case Kind::array: return a_.size();
        case Kind::object: return o_.size();
        default: return 1;
    }
}
std::vector<const Json*> Json::items() const {
    std::vector<const Json*> out;
    if (kind_ == Kind::array) {
        for (const Json& v : a_) out.push_back(&v);
    } else if (kind_ == Kind::object) {
        for (const auto& kv : o_) out.push_back(&kv.second);
    } else if (kind_ != Kind::null) {
        out.push_back(this);
    }
    return out;
}
Json& Json::push_back(Json v) {
    if (kind_ == Kind::null) kind_ = Kind::array;
    if (kind_ != Kind::array) type_error("array");
    a_.push_back(std::move(v));
    return a_.back();
}
Json& Json::set(const std::string& key, Json v) {
    if (kind_ == Kind::null) kind_ = Kind::object;
    if (kind_ != Kind::object) type_error("object");
    return o_[key] = std::move(v);
}

// ------------------------------------------------------------------ dump
namespace {
void escape(std::string& out, const std::string& s) {
    out += '"';
    for (unsigned char c : s) {
        switch (c) {
            case '"': out += "\\\""; break;
            case '\\': out += "\\\\"; break;
            case '\b': out += "\\b"; break;
            case '\f': out += "\\f"; break;
            case '\n': out += "\\n"; break;
            case '\r': out += "\\r"; break;
            case '\t': out += "\\t"; break;
            default:
                if (c < 0x20) {
                    char buf[8];
                    std::snprintf(buf, sizeof buf, "\\u%04x", c);
                    out += buf;
                } else {
                    out += char(c);
                }
        }
    }
    out += '"';
}
}  // namespace

void Json::dump_to(std::string& out, int indent, int level) const {
    const std::string pad(std::size_t(indent) * (level + 1), ' '), end(std::size_t(indent) * level, ' ');
    switch (kind_) {
        case Kind::null: out += "null"; return;
        case Kind::boolean: out += b_ ? "true" : "false"; return;
        case Kind::integer: out += std::to_string(i_); return;
        case Kind::unsigned_integer: out += std::to_string(u_); return;
        case Kind::floating: {
            // write paths never emit floats (loads are exact strings); a
            // round-trip %.17g keeps the value if one is ever stored
            char buf[40];
            std::snprintf(buf, sizeof buf, "%.17g", d_);
            out += buf;
            return;
        }
        case Kind::string: escape(out, s_); return;
        case Kind::array: {
            if (a_.empty()) {
                out += "[]";
                return;
            }
            out += "[\n";
            for (std::size_t i = 0; i < a_.size(); ++i) {
                out += pad;
                a_[i].dump_to(out, indent, level + 1);
                out += i + 1 < a_.size() ? ",\n" : "\n";
            }
            out += end + "]";
            return;
        }
        case Kind::object: {
            if (o_.empty()) {
                out += "{}";
                return;
            }
            out += "{\n";
            std::size_t i = 0;
            for (const auto& [k, v] : o_) {
                out += pad;
                escape(out, k);
                out += ": ";
                v.dump_to(out, indent, level + 1);
                out += ++i < o_.size() ? ",\n" : "\n";
            }
            out += end + "}";
            return;
        }
    }
}

std::string Json::dump(int indent) const {
    std::string out;
    dump_to(out, indent, 0);
    return out;
}

// ----------------------------------------------------------------- parse
namespace {
struct Parser {
    const std::string& t;
    std::size_t p = 0;

    [[noreturn]] void fail(const std::string& what) const {
        throw JsonError("parse error at byte " + std::to_string(p + 1) + ": " + what);
    }
    void ws() {
        while (p < t.size() && (t[p] == ' ' || t[p] == '\t' || t[p] == '\n' || t[p] == '\r')) ++p;
    }
    bool lit(const char* s) {
        std::size_t k = 0;
        while (s[k]) {
            if (p + k >= t.size() || t[p + k] != s[k]) return false;
            ++k;
        }
        p += k;
        return true;
    }
    void utf8(std::string& out, unsigned cp) {
        if (cp < 0x80) {
            out += char(cp);
        } else if (cp < 0x800) {
            out += char(0xC0 | (cp >> 6));
            out += char(0x80 | (cp & 0x3F));
        } else if (cp < 0x10000) {
            out += char(0xE0 | (cp >> 12));
            out += char(0x80 | ((cp >> 6) & 0x3F));
            out += char(0x80 | (cp & 0x3F));
        } else {
            out += char(0xF0 | (cp >> 18));
            out += char(0x80 | ((cp >> 12) & 0x3F));
            out += char(0x80 | ((cp >> 6) & 0x3F));
            out += char(0x80 | (cp & 0x3F));
        }
    }
    unsigned hex4() {
        if (p + 4 > t.size()) fail("truncated \\u escape");
        unsigned v = 0;
        for (int k = 0; k < 4; ++k) {
            const char c = t[p++];
            v <<= 4;
            if (c >= '0' && c <= '9') v |= unsigned(c - '0');
            else if (c >= 'a' && c <= 'f') v |= unsigned(c - 'a' + 10);
            else if (c >= 'A' && c <= 'F') v |= unsigned(c - 'A' + 10);
            else fail("bad \\u escape");
        }
        return v;
    }
    std::string string_body() {
        std::string out;
        for (;;) {
            if (p >= t.size()) fail("unterminated string");
            const unsigned char c = static_cast<unsigned char>(t[p++]);
            if (c == '"') return out;
            if (c < 0x20) fail("control character in string");
            if (c != '\\') {
                out += char(c);
                continue;
            }
            if (p >= t.size()) fail("unterminated escape");
            const char e = t[p++];
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
                    if (cp >= 0xD800 && cp < 0xDC00) {
                        if (!lit("\\u")) fail("lone surrogate");
                        const unsigned lo = hex4();
                        if (lo < 0xDC00 || lo >= 0xE000) fail("bad surrogate pair");
                        cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                    } else if (cp >= 0xDC00 && cp < 0xE000) {
                        fail("lone surrogate");
                    }
                    utf8(out, cp);
                    break;
                }
                default: fail("bad escape");
            }
        }
    }
    Json number() {
        const std::size_t s = p;
        bool neg = false, is_float = false;
        if (t[p] == '-') {
            neg = true;
            ++p;
        }
        if (p >= t.size() || !std::isdigit(static_cast<unsigned char>(t[p]))) fail("bad number");
        if (t[p] == '0') {
            ++p;
        } else {
            while (p < t.size() && std::isdigit(static_cast<unsigned char>(t[p]))) ++p;
        }
        if (p < t.size() && t[p] == '.') {
            is_float = true;
            ++p;
            if (p >= t.size() || !std::isdigit(static_cast<unsigned char>(t[p]))) fail("bad fraction");
            while (p < t.size() && std::isdigit(static_cast<unsigned char>(t[p]))) ++p;
        }
        if (p < t.size() && (t[p] == 'e' || t[p] == 'E')) {
            is_float = true;
            ++p;
            if (p < t.size() && (t[p] == '+' || t[p] == '-')) ++p;
            if (p >= t.size() || !std::isdigit(static_cast<unsigned char>(t[p]))) fail("bad exponent");
            while (p < t.size() && std::isdigit(static_cast<unsigned char>(t[p]))) ++p;
        }
        const std::string tok = t.substr(s, p - s);
        if (!is_float) {  // nlohmann: int64 when negative, uint64 otherwise; float on overflow
            errno = 0;
            if (neg) {
                const long long v = std::strtoll(tok.c_str(), nullptr, 10);
                if (errno == 0) return Json::integer(v);
            } else {
                const unsigned long long v = std::strtoull(tok.c_str(), nullptr, 10);
                if (errno == 0) return Json::unsigned_integer(v);
            }
        }
        return Json::floating(std::strtod(tok.c_str(), nullptr));
    }
    Json value(int depth) {
        if (depth > 512) fail("nesting too deep");
        ws();
        if (p >= t.size()) fail("unexpected end of input");
        const char c = t[p];
        if (c == '{') {
            ++p;
            Json o = Json::object();
            ws();
            if (p < t.size() && t[p] == '}') {
                ++p;
                return o;
            }
            for (;;) {
                ws();
                if (p >= t.size() || t[p] != '"') fail("expected a key");
                ++p;
                std::string k = string_body();
                ws();
                if (p >= t.size() || t[p] != ':') fail("expected ':'");
                ++p;
                o.set(k, value(depth + 1));
                ws();
                if (p < t.size() && t[p] == ',') {
                    ++p;
                    continue;
                }
                if (p < t.size() && t[p] == '}') {
                    ++p;
                    return o;
                }
                fail("expected ',' or '}'");
            }
        }
        if (c == '[') {
            ++p;
            Json a = Json::array();
            ws();
            if (p < t.size() && t[p] == ']') {
                ++p;
                return a;
            }
            for (;;) {
                a.push_back(value(depth + 1));
                ws();
                if (p < t.size() && t[p] == ',') {
                    ++p;
                    continue;
                }
                if (p < t.size() && t[p] == ']') {
                    ++p;
                    return a;
                }
                fail("expected ',' or ']'");
            }
        }
        if (c == '"') {
            ++p;
            return Json::string(string_body());
        }
        if (lit("true")) return Json::boolean(true);
        if (lit("false")) return Json::boolean(false);
        if (lit("null")) return Json();
        if (c == '-' || std::isdigit(static_cast<unsigned char>(c))) return number();
        fail("unexpected character");
    }
};
}  // namespace

Json Json::parse(const std::string& text) {
    Parser ps{text};
    Json v = ps.value(0);
    ps.ws();
    if (ps.p != text.size()) ps.fail("trailing characters");
    return v;
}

}  // namespace dagsched::detail
