// JSON document model, strict parser and canonical writer (see json.hpp).
#include "json.hpp"

#include "graphvx/error.hpp"

#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

namespace gvx::json {

namespace {

[[noreturn]] void type_error(const char* what, const char* want) {
    throw Error(ErrorCode::SchemaError, std::string(what) + " must be " + want);
}

} // namespace

std::size_t Value::size() const {
    switch (type_) {
    case Type::Null: return 0;
    case Type::Array: return a_.size();
    case Type::Object: return o_.size();
    default: return 1;
    }
}

std::int64_t Value::as_int(const char* what) const {
    switch (type_) {
    case Type::Int: return i_;
    case Type::UInt: return static_cast<std::int64_t>(u_);
    case Type::Float: return static_cast<std::int64_t>(d_);
    default: type_error(what, "a number");
    }
}

double Value::as_double(const char* what) const {
    switch (type_) {
    case Type::Int: return static_cast<double>(i_);
    case Type::UInt: return static_cast<double>(u_);
    case Type::Float: return d_;
    default: type_error(what, "a number");
    }
}

bool Value::as_bool(const char* what) const {
    if (type_ != Type::Bool) type_error(what, "a boolean");
    return b_;
}

const std::string& Value::as_string(const char* what) const {
    if (type_ != Type::String) type_error(what, "a string");
    return s_;
}

const std::vector<Value>& Value::items(const char* what) const {
    static const std::vector<Value> none;
    if (type_ == Type::Null) return none;
    if (type_ != Type::Array) type_error(what, "an array");
    return a_;
}

const Value& Value::at(std::size_t i) const {
    if (type_ != Type::Array || i >= a_.size())
        throw Error(ErrorCode::SchemaError, "array index " + std::to_string(i) + " out of range");
    return a_[i];
}

void Value::push_back(Value v) {
    if (type_ == Type::Null) type_ = Type::Array;
    if (type_ != Type::Array) type_error("push_back target", "an array");
    a_.push_back(std::move(v));
}

bool Value::contains(const std::string& key) const { return type_ == Type::Object && o_.count(key) != 0; }

const Value& Value::at(const std::string& key) const {
    if (type_ != Type::Object) type_error("document", "an object");
    auto it = o_.find(key);
    if (it == o_.end()) throw Error(ErrorCode::SchemaError, "missing field \"" + key + "\"");
    return it->second;
}

Value& Value::operator[](const std::string& key) {
    if (type_ == Type::Null) type_ = Type::Object;
    if (type_ != Type::Object) type_error("document", "an object");
    return o_[key];
}

const std::map<std::string, Value>& Value::members(const char* what) const {
    if (type_ != Type::Object) type_error(what, "an object");
    return o_;
}

std::int64_t Value::value(const std::string& key, std::int64_t dflt) const {
    if (!contains(key)) return dflt;
    return o_.at(key).as_int(key.c_str());
}

bool Value::value(const std::string& key, bool dflt) const {
    if (!contains(key)) return dflt;
    return o_.at(key).as_bool(key.c_str());
}

std::string Value::value(const std::string& key, const std::string& dflt) const {
    if (!contains(key)) return dflt;
    return o_.at(key).as_string(key.c_str());
}

// ------------------------------------------------------------------ writer

namespace {

// Grisu2 (Loitsch, "Printing floating-point numbers quickly and accurately
// with integers", PLDI 2010): digits within the rounding interval of v,
// usually but not always the shortest.  Reproducing it (rather than a
// shortest-digits search) keeps the canonical text identical to the
// reference's JSON library for every double.
struct Fp {
    std::uint64_t f;
    int e;
};

Fp fp_mul(Fp a, Fp b) { // round-half-up of the top 64 bits of the 128-bit product
    const unsigned __int128 p = static_cast<unsigned __int128>(a.f) * b.f + (static_cast<unsigned __int128>(1) << 63);
    return Fp{static_cast<std::uint64_t>(p >> 64), a.e + b.e + 64};
}

Fp fp_normalize(Fp x) {
    while ((x.f >> 63) == 0) x.f <<= 1, --x.e;
    return x;
}

struct CachedPow {
    std::uint64_t f;
    int e;
    int k;
};
const CachedPow kPow10[] = {
#include "pow10_table.inc"
};

void grisu2_round(std::string& buf, std::uint64_t dist, std::uint64_t delta, std::uint64_t rest,
                  std::uint64_t ten_k) {
    // step the last digit down while that brings the value closer to w and
    // stays inside [M-, M+]
    while (rest < dist && delta - rest >= ten_k && (rest + ten_k < dist || dist - rest > rest + ten_k - dist)) {
        --buf.back();
        rest += ten_k;
    }
}

/// Digits d (no leading zeros) and exponent x with |v| ~= d * 10^x.
void grisu2(double v, std::string& digits, int& dexp) {
    std::uint64_t bits;
    std::memcpy(&bits, &v, 8);
    const std::uint64_t F = bits & ((std::uint64_t{1} << 52) - 1);
    const int E = static_cast<int>(bits >> 52);
    const Fp w = E == 0 ? Fp{F, 1 - 1075} : Fp{F + (std::uint64_t{1} << 52), E - 1075};
    const bool closer_low = F == 0 && E > 1;
    const Fp mp = fp_normalize(Fp{2 * w.f + 1, w.e - 1});
    Fp mm = closer_low ? Fp{4 * w.f - 1, w.e - 2} : Fp{2 * w.f - 1, w.e - 1};
    mm.f <<= (mm.e - mp.e);
    mm.e = mp.e;
    const Fp wn = fp_normalize(w);

    // cached power c = 10^-k bringing the products' exponent into [-60, -32]
    const int fexp = -60 - mp.e - 1;
    const int kk = (fexp * 78913) / (1 << 18) + (fexp > 0 ? 1 : 0);
    const int idx = (300 + kk + 7) / 8;
    const CachedPow cp = kPow10[idx];
    const Fp c{cp.f, cp.e};
    const Fp W = fp_mul(wn, c), Wm = fp_mul(mm, c), Wp = fp_mul(mp, c);
    const Fp Mm{Wm.f + 1, Wm.e}, Mp{Wp.f - 1, Wp.e};
    dexp = -cp.k;

    std::uint64_t delta = Mp.f - Mm.f, dist = Mp.f - W.f;
    const int shift = -Mp.e;
    const std::uint64_t one = std::uint64_t{1} << shift;
    auto p1 = static_cast<std::uint32_t>(Mp.f >> shift);
    std::uint64_t p2 = Mp.f & (one - 1);

    // integral digits
    std::uint32_t pow10 = 1;
    int n = 1;
    while (n < 10 && pow10 * std::uint64_t{10} <= p1) pow10 *= 10, ++n;
    digits.clear();
    while (n > 0) {
        const std::uint32_t d = p1 / pow10;
        p1 %= pow10;
        digits.push_back(static_cast<char>('0' + d));
        --n;
        const std::uint64_t rest = (std::uint64_t{p1} << shift) + p2;
        if (rest <= delta) {
            dexp += n;
            grisu2_round(digits, dist, delta, rest, std::uint64_t{pow10} << shift);
            return;
        }
        pow10 /= 10;
    }
    // fractional digits
    int m = 0;
    while (true) {
        p2 *= 10;
        digits.push_back(static_cast<char>('0' + (p2 >> shift)));
        p2 &= one - 1;
        ++m;
        delta *= 10;
        dist *= 10;
        if (p2 <= delta) break;
    }
    dexp -= m;
    grisu2_round(digits, dist, delta, p2, one);
}

} // namespace

std::string format_double(double v) {
    if (!std::isfinite(v)) return "null";
    std::string sign = std::signbit(v) ? "-" : "";
    if (v == 0.0) return sign + "0.0";
    std::string digits;
    int dexp = 0;
    grisu2(std::fabs(v), digits, dexp);
    const int k = static_cast<int>(digits.size());
    const int n = k + dexp; // decimal point position relative to the digits
    std::string out;
    if (k <= n && n <= 15) {
        out = digits + std::string(static_cast<std::size_t>(n - k), '0') + ".0";
    } else if (0 < n && n <= 15) {
        out = digits.substr(0, static_cast<std::size_t>(n)) + "." + digits.substr(static_cast<std::size_t>(n));
    } else if (-4 < n && n <= 0) {
        out = "0." + std::string(static_cast<std::size_t>(-n), '0') + digits;
    } else {
        out = digits.substr(0, 1);
        if (k > 1) out += "." + digits.substr(1);
        const int e = n - 1;
        char eb[16];
        std::snprintf(eb, sizeof eb, "e%c%02d", e < 0 ? '-' : '+', e < 0 ? -e : e);
        out += eb;
    }
    return sign + out;
}

namespace {

void dump_string(std::string& out, const std::string& s) {
    out.push_back('"');
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
                char b[8];
                std::snprintf(b, sizeof b, "\\u%04x", c);
                out += b;
            } else {
                out.push_back(static_cast<char>(c));
            }
        }
    }
    out.push_back('"');
}

} // namespace

void Value::dump_to(std::string& out, int indent, int level) const {
    const bool pretty = indent >= 0;
    auto newline = [&](int lvl) {
        out.push_back('\n');
        out.append(static_cast<std::size_t>(indent * lvl), ' ');
    };
    switch (type_) {
    case Type::Null: out += "null"; break;
    case Type::Bool: out += b_ ? "true" : "false"; break;
    case Type::Int: out += std::to_string(i_); break;
    case Type::UInt: out += std::to_string(u_); break;
    case Type::Float: out += format_double(d_); break;
    case Type::String: dump_string(out, s_); break;
    case Type::Array:
        if (a_.empty()) {
            out += "[]";
            break;
        }
        out.push_back('[');
        for (std::size_t i = 0; i < a_.size(); ++i) {
            if (i) out.push_back(',');
            if (pretty) newline(level + 1);
            a_[i].dump_to(out, indent, level + 1);
        }
        if (pretty) newline(level);
        out.push_back(']');
        break;
    case Type::Object: {
        if (o_.empty()) {
            out += "{}";
            break;
        }
        out.push_back('{');
        bool first = true;
        for (const auto& [key, v] : o_) {
            if (!first) out.push_back(',');
            first = false;
            if (pretty) newline(level + 1);
            dump_string(out, key);
            out += pretty ? ": " : ":";
            v.dump_to(out, indent, level + 1);
        }
        if (pretty) newline(level);
        out.push_back('}');
        break;
    }
    }
}

std::string Value::dump(int indent) const {
    std::string out;
    dump_to(out, indent, 0);
    return out;
}

// ------------------------------------------------------------------ parser

namespace {

struct Parser {
    const std::string& t;
    std::size_t i = 0;
    std::string err;

    bool fail(const std::string& m) {
        if (err.empty()) err = m + " at offset " + std::to_string(i);
        return false;
    }
    void ws() {
        while (i < t.size() && (t[i] == ' ' || t[i] == '\t' || t[i] == '\n' || t[i] == '\r')) ++i;
    }
    bool lit(const char* w) {
        const std::size_t n = std::strlen(w);
        if (t.compare(i, n, w) != 0) return fail("invalid literal");
        i += n;
        return true;
    }
    static void utf8(std::string& s, unsigned cp) {
        if (cp < 0x80) {
            s.push_back(static_cast<char>(cp));
        } else if (cp < 0x800) {
            s.push_back(static_cast<char>(0xC0 | (cp >> 6)));
            s.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
        } else if (cp < 0x10000) {
            s.push_back(static_cast<char>(0xE0 | (cp >> 12)));
            s.push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
            s.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
        } else {
            s.push_back(static_cast<char>(0xF0 | (cp >> 18)));
            s.push_back(static_cast<char>(0x80 | ((cp >> 12) & 0x3F)));
            s.push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
            s.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
        }
    }
    bool hex4(unsigned& v) {
        if (i + 4 > t.size()) return fail("truncated \\u escape");
        v = 0;
        for (int k = 0; k < 4; ++k) {
            const char c = t[i++];
            v <<= 4;
            if (c >= '0' && c <= '9') v |= static_cast<unsigned>(c - '0');
            else if (c >= 'a' && c <= 'f') v |= static_cast<unsigned>(c - 'a' + 10);
            else if (c >= 'A' && c <= 'F') v |= static_cast<unsigned>(c - 'A' + 10);
            else return fail("bad \\u escape");
        }
        return true;
    }
    bool string(std::string& s) {
        ++i; // opening quote
        while (true) {
            if (i >= t.size()) return fail("unterminated string");
            const unsigned char c = static_cast<unsigned char>(t[i++]);
            if (c == '"') return true;
            if (c < 0x20) return fail("control character in string");
            if (c != '\\') {
                s.push_back(static_cast<char>(c));
                continue;
            }
            if (i >= t.size()) return fail("unterminated escape");
            const char e = t[i++];
            switch (e) {
            case '"': s.push_back('"'); break;
            case '\\': s.push_back('\\'); break;
            case '/': s.push_back('/'); break;
            case 'b': s.push_back('\b'); break;
            case 'f': s.push_back('\f'); break;
            case 'n': s.push_back('\n'); break;
            case 'r': s.push_back('\r'); break;
            case 't': s.push_back('\t'); break;
            case 'u': {
                unsigned cp = 0;
                if (!hex4(cp)) return false;
                if (cp >= 0xD800 && cp <= 0xDBFF) {
                    unsigned lo = 0;
                    if (t.compare(i, 2, "\\u") != 0) return fail("unpaired surrogate");
                    i += 2;
                    if (!hex4(lo) || lo < 0xDC00 || lo > 0xDFFF) return fail("bad surrogate pair");
                    cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
                    return fail("unpaired surrogate");
                }
                utf8(s, cp);
                break;
            }
            default: return fail("bad escape");
            }
        }
    }
    bool number(Value& v) {
        const std::size_t s0 = i;
        bool neg = false, is_float = false;
        if (t[i] == '-') neg = true, ++i;
        if (i >= t.size() || !(t[i] >= '0' && t[i] <= '9')) return fail("bad number");
        if (t[i] == '0') {
            ++i;
        } else {
            while (i < t.size() && t[i] >= '0' && t[i] <= '9') ++i;
        }
        if (i < t.size() && t[i] == '.') {
            is_float = true;
            ++i;
            if (i >= t.size() || !(t[i] >= '0' && t[i] <= '9')) return fail("bad fraction");
            while (i < t.size() && t[i] >= '0' && t[i] <= '9') ++i;
        }
        if (i < t.size() && (t[i] == 'e' || t[i] == 'E')) {
            is_float = true;
            ++i;
            if (i < t.size() && (t[i] == '+' || t[i] == '-')) ++i;
            if (i >= t.size() || !(t[i] >= '0' && t[i] <= '9')) return fail("bad exponent");
            while (i < t.size() && t[i] >= '0' && t[i] <= '9') ++i;
        }
        const std::string tok = t.substr(s0, i - s0);
        if (!is_float) {
            errno = 0;
            char* end = nullptr;
            if (neg) {
                const long long x = std::strtoll(tok.c_str(), &end, 10);
                if (errno == 0) {
                    v = Value(x);
                    return true;
                }
            } else {
                const unsigned long long x = std::strtoull(tok.c_str(), &end, 10);
                if (errno == 0) {
                    v = Value(x); // non-negative integers parse as unsigned
                    return true;
                }
            }
            // out of 64-bit range: falls through to a double
        }
        const double d = std::strtod(tok.c_str(), nullptr);
        if (!std::isfinite(d)) return fail("number overflow");
        v = Value(d);
        return true;
    }
    bool value(Value& v, int depth) {
        if (depth > 512) return fail("nesting too deep");
        ws();
        if (i >= t.size()) return fail("unexpected end");
        const char c = t[i];
        if (c == 'n') {
            if (!lit("null")) return false;
            v = Value();
            return true;
        }
        if (c == 't') {
            if (!lit("true")) return false;
            v = Value(true);
            return true;
        }
        if (c == 'f') {
            if (!lit("false")) return false;
            v = Value(false);
            return true;
        }
        if (c == '"') {
            std::string s;
            if (!string(s)) return false;
            v = Value(std::move(s));
            return true;
        }
        if (c == '[') {
            ++i;
            v = Value::array();
            ws();
            if (i < t.size() && t[i] == ']') {
                ++i;
                return true;
            }
            while (true) {
                Value e;
                if (!value(e, depth + 1)) return false;
                v.push_back(std::move(e));
                ws();
                if (i < t.size() && t[i] == ',') {
                    ++i;
                    continue;
                }
                if (i < t.size() && t[i] == ']') {
                    ++i;
                    return true;
                }
                return fail("expected ',' or ']'");
            }
        }
        if (c == '{') {
            ++i;
            v = Value::object();
            ws();
            if (i < t.size() && t[i] == '}') {
                ++i;
                return true;
            }
            while (true) {
                ws();
                if (i >= t.size() || t[i] != '"') return fail("expected object key");
                std::string key;
                if (!string(key)) return false;
                ws();
                if (i >= t.size() || t[i] != ':') return fail("expected ':'");
                ++i;
                Value e;
                if (!value(e, depth + 1)) return false;
                v[key] = std::move(e); // a repeated key keeps the last value
                ws();
                if (i < t.size() && t[i] == ',') {
                    ++i;
                    continue;
                }
                if (i < t.size() && t[i] == '}') {
                    ++i;
                    return true;
                }
                return fail("expected ',' or '}'");
            }
        }
        if (c == '-' || (c >= '0' && c <= '9')) return number(v);
        return fail("unexpected character");
    }
};

} // namespace

bool parse(const std::string& text, Value& out, std::string* error) {
    Parser p{text, 0, {}};
    Value v;
    bool ok = p.value(v, 0);
    if (ok) {
        p.ws();
        if (p.i != text.size()) ok = p.fail("trailing characters");
    }
    if (!ok) {
        if (error) *error = p.err;
        return false;
    }
    out = std::move(v);
    return true;
}

} // namespace gvx::json
