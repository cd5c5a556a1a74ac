// LPT1 containers (include/lpradon/lpt1.hpp): encoder,
// decoder with the four distinct error classes, and the small JSON value the
// header needs.
#include "lpradon/lpt1.hpp"

#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>

namespace lpr::io {

// ------------------------------------------------------------------ Json
long long Json::as_int() const {
    if (type_ != Type::integer) throw SchemaError("JSON value is not an integer");
    return i_;
}

double Json::as_number() const {
    if (type_ == Type::integer) return double(i_);
    if (type_ != Type::number) throw SchemaError("JSON value is not a number");
    return d_;
}

const std::string& Json::as_string() const {
    if (type_ != Type::string) throw SchemaError("JSON value is not a string");
    return s_;
}

const Json& Json::at(const std::string& k) const {
    auto it = o_.find(k);
    if (type_ != Type::object || it == o_.end()) throw SchemaError("JSON object has no field '" + k + "'");
    return it->second;
}

Json& Json::operator[](const std::string& k) {
    if (type_ == Type::null) type_ = Type::object;
    if (type_ != Type::object) throw SchemaError("JSON value is not an object");
    return o_[k];
}

void Json::push_back(Json v) {
    if (type_ == Type::null) type_ = Type::array;
    if (type_ != Type::array) throw SchemaError("JSON value is not an array");
    a_.push_back(std::move(v));
}

namespace {

// Python's float repr: shortest round-trip digits, fixed notation for
// decimal exponents in [-4, 16), else d.ddde+XX (at least two exponent digits).
std::string py_float(double v) {
    if (std::isnan(v)) return "NaN";
    if (std::isinf(v)) return v > 0 ? "Infinity" : "-Infinity";
    if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
    char buf[64];
    const auto r = std::to_chars(buf, buf + sizeof(buf), v, std::chars_format::scientific);
    std::string s(buf, r.ptr);
    const bool neg = s[0] == '-';
    if (neg) s.erase(0, 1);
    const std::size_t e = s.find('e');
    const int exp = std::atoi(s.c_str() + e + 1);
    std::string digits;
    for (std::size_t i = 0; i < e; ++i)
        if (s[i] != '.') digits += s[i];
    std::string out;
    if (exp >= -4 && exp < 16) {
        if (exp >= 0) {
            const std::size_t ip = std::size_t(exp) + 1;
            if (digits.size() <= ip)
                out = digits + std::string(ip - digits.size(), '0') + ".0";
            else
                out = digits.substr(0, ip) + "." + digits.substr(ip);
        } else {
            out = "0." + std::string(std::size_t(-exp - 1), '0') + digits;
        }
    } else {
        out = digits.substr(0, 1);
        if (digits.size() > 1) out += "." + digits.substr(1);
        char ex[16];
        std::snprintf(ex, sizeof(ex), "e%c%02d", exp < 0 ? '-' : '+', std::abs(exp));
        out += ex;
    }
    return neg ? "-" + out : out;
}

void put_u16(std::string& o, unsigned u) {
    char b[8];
    std::snprintf(b, sizeof(b), "\\u%04x", u);
    o += b;
}

// json.dumps(ensure_ascii=True) string escaping
std::string py_string(const std::string& s) {
    std::string o = "\"";
    for (std::size_t i = 0; i < s.size();) {
        const unsigned char c = static_cast<unsigned char>(s[i]);
        if (c < 0x80) {
            switch (c) {
                case '"': o += "\\\""; break;
                case '\\': o += "\\\\"; break;
                case '\n': o += "\\n"; break;
                case '\r': o += "\\r"; break;
                case '\t': o += "\\t"; break;
                case '\b': o += "\\b"; break;
                case '\f': o += "\\f"; break;
                default:
                    if (c < 0x20) put_u16(o, c); else o += char(c);
            }
            ++i;
            continue;
        }
        // decode one UTF-8 sequence
        int len = c >= 0xF0 ? 4 : c >= 0xE0 ? 3 : c >= 0xC0 ? 2 : 0;
        if (len == 0 || i + len > s.size()) throw SchemaError("string is not valid UTF-8");
        unsigned cp = c & (0x7F >> len);
        for (int k = 1; k < len; ++k) {
            const unsigned char cc = static_cast<unsigned char>(s[i + k]);
            if ((cc & 0xC0) != 0x80) throw SchemaError("string is not valid UTF-8");
            cp = (cp << 6) | (cc & 0x3F);
        }
        if (cp >= 0x10000) {
            cp -= 0x10000;
            put_u16(o, 0xD800 + (cp >> 10));
            put_u16(o, 0xDC00 + (cp & 0x3FF));
        } else {
            put_u16(o, cp);
        }
        i += len;
    }
    return o + "\"";
}

void put_utf8(std::string& o, unsigned cp) {
    if (cp < 0x80) {
        o += char(cp);
    } else if (cp < 0x800) {
        o += char(0xC0 | (cp >> 6));
        o += char(0x80 | (cp & 0x3F));
    } else if (cp < 0x10000) {
        o += char(0xE0 | (cp >> 12));
        o += char(0x80 | ((cp >> 6) & 0x3F));
        o += char(0x80 | (cp & 0x3F));
    } else {
        o += char(0xF0 | (cp >> 18));
        o += char(0x80 | ((cp >> 12) & 0x3F));
        o += char(0x80 | ((cp >> 6) & 0x3F));
        o += char(0x80 | (cp & 0x3F));
    }
}

struct Parser {
    const std::string& t;
    std::size_t i = 0;

    [[noreturn]] void fail(const char* what) const {
        throw SchemaError(std::string("header is not valid JSON: ") + what + " at byte " + std::to_string(i));
    }
    void ws() {
        while (i < t.size() && (t[i] == ' ' || t[i] == '\t' || t[i] == '\n' || t[i] == '\r')) ++i;
    }
    bool lit(const char* w) {
        const std::size_t n = std::strlen(w);
        if (t.compare(i, n, w) == 0) {
            i += n;
            return true;
        }
        return false;
    }
    unsigned hex4() {
        if (i + 4 > t.size()) fail("short \\u escape");
        unsigned v = 0;
        for (int k = 0; k < 4; ++k) {
            const char c = t[i++];
            v <<= 4;
            if (c >= '0' && c <= '9') v |= unsigned(c - '0');
            else if (c >= 'a' && c <= 'f') v |= unsigned(c - 'a' + 10);
            else if (c >= 'A' && c <= 'F') v |= unsigned(c - 'A' + 10);
            else fail("bad \\u escape");
        }
        return v;
    }
    std::string str() {
        if (t[i] != '"') fail("expected a string");
        ++i;
        std::string o;
        while (true) {
            if (i >= t.size()) fail("unterminated string");
            const char c = t[i++];
            if (c == '"') break;
            if (static_cast<unsigned char>(c) < 0x20) fail("control character in string");
            if (c != '\\') {
                o += c;
                continue;
            }
            if (i >= t.size()) fail("unterminated escape");
            const char e = t[i++];
            switch (e) {
                case '"': o += '"'; break;
                case '\\': o += '\\'; break;
                case '/': o += '/'; break;
                case 'b': o += '\b'; break;
                case 'f': o += '\f'; break;
                case 'n': o += '\n'; break;
                case 'r': o += '\r'; break;
                case 't': o += '\t'; break;
                case 'u': {
                    unsigned cp = hex4();
                    if (cp >= 0xD800 && cp < 0xDC00 && t.compare(i, 2, "\\u") == 0) {
                        i += 2;
                        const unsigned lo = hex4();
                        if (lo >= 0xDC00 && lo < 0xE000) cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                        else fail("bad surrogate pair");
                    }
                    put_utf8(o, cp);
                    break;
                }
                default: fail("bad escape");
            }
        }
        return o;
    }
    Json value() {
        ws();
        if (i >= t.size()) fail("unexpected end");
        const char c = t[i];
        if (c == '{') {
            ++i;
            Json o = Json::object();
            ws();
            if (i < t.size() && t[i] == '}') {
                ++i;
                return o;
            }
            while (true) {
                ws();
                if (i >= t.size()) fail("unterminated object");
                const std::string k = str();
                ws();
                if (i >= t.size() || t[i] != ':') fail("expected ':'");
                ++i;
                o[k] = value();
                ws();
                if (i < t.size() && t[i] == ',') {
                    ++i;
                    continue;
                }
                if (i < t.size() && t[i] == '}') {
                    ++i;
                    return o;
                }
                fail("expected ',' or '}'");
            }
        }
        if (c == '[') {
            ++i;
            Json a = Json::array();
            ws();
            if (i < t.size() && t[i] == ']') {
                ++i;
                return a;
            }
            while (true) {
                a.push_back(value());
                ws();
                if (i < t.size() && t[i] == ',') {
                    ++i;
                    continue;
                }
                if (i < t.size() && t[i] == ']') {
                    ++i;
                    return a;
                }
                fail("expected ',' or ']'");
            }
        }
        if (c == '"') return Json(str());
        if (lit("true")) return Json(true);
        if (lit("false")) return Json(false);
        if (lit("null")) return Json();
        if (lit("NaN")) return Json(std::nan(""));
        if (lit("Infinity")) return Json(HUGE_VAL);
        if (lit("-Infinity")) return Json(-HUGE_VAL);
        // number: -?(0|[1-9][0-9]*)(\.[0-9]+)?([eE][+-]?[0-9]+)?
        const std::size_t s0 = i;
        if (t[i] == '-') ++i;
        if (i >= t.size() || !std::isdigit(static_cast<unsigned char>(t[i]))) fail("unexpected character");
        if (t[i] == '0') ++i;
        else
            while (i < t.size() && std::isdigit(static_cast<unsigned char>(t[i]))) ++i;
        bool real = false;
        if (i < t.size() && t[i] == '.') {
            real = true;
            ++i;
            if (i >= t.size() || !std::isdigit(static_cast<unsigned char>(t[i]))) fail("bad number");
            while (i < t.size() && std::isdigit(static_cast<unsigned char>(t[i]))) ++i;
        }
        if (i < t.size() && (t[i] == 'e' || t[i] == 'E')) {
            real = true;
            ++i;
            if (i < t.size() && (t[i] == '+' || t[i] == '-')) ++i;
            if (i >= t.size() || !std::isdigit(static_cast<unsigned char>(t[i]))) fail("bad exponent");
            while (i < t.size() && std::isdigit(static_cast<unsigned char>(t[i]))) ++i;
        }
        const std::string num = t.substr(s0, i - s0);
        if (real) return Json(std::strtod(num.c_str(), nullptr));
        long long v = 0;
        const auto r = std::from_chars(num.data(), num.data() + num.size(), v);
        if (r.ec != std::errc()) return Json(std::strtod(num.c_str(), nullptr));  // beyond int64: Python keeps it exact
        return Json(v);
    }
};

bool valid_utf8(const std::string& s) {
    for (std::size_t i = 0; i < s.size();) {
        const unsigned char c = static_cast<unsigned char>(s[i]);
        const int len = c < 0x80 ? 1 : (c >> 5) == 6 ? 2 : (c >> 4) == 14 ? 3 : (c >> 3) == 30 ? 4 : 0;
        if (len == 0 || i + len > s.size()) return false;
        for (int k = 1; k < len; ++k)
            if ((static_cast<unsigned char>(s[i + k]) & 0xC0) != 0x80) return false;
        i += len;
    }
    return true;
}

}  // namespace

std::string Json::dump() const {
    switch (type_) {
        case Type::null: return "null";
        case Type::boolean: return b_ ? "true" : "false";
        case Type::integer: return std::to_string(i_);
        case Type::number: return py_float(d_);
        case Type::string: return py_string(s_);
        case Type::array: {
            std::string o = "[";
            for (std::size_t k = 0; k < a_.size(); ++k) o += (k ? "," : "") + a_[k].dump();
            return o + "]";
        }
        case Type::object: {
            std::string o = "{";
            bool first = true;
            for (const auto& kv : o_) {  // std::map: sorted by UTF-8 bytes = code points (sort_keys)
                o += (first ? "" : ",") + py_string(kv.first) + ":" + kv.second.dump();
                first = false;
            }
            return o + "}";
        }
    }
    return "null";
}

Json Json::parse(const std::string& text) {
    if (!valid_utf8(text)) throw SchemaError("header is not UTF-8");
    Parser p{text};
    Json v = p.value();
    p.ws();
    if (p.i != text.size()) p.fail("trailing characters");
    return v;
}

// ------------------------------------------------------------------ grids
namespace {
Json axis(long count, double origin, double spacing) {
    Json a = Json::object();
    a["count"] = Json(count);
    a["origin"] = Json(origin);
    a["spacing"] = Json(spacing);
    return a;
}
const char* const kKinds[] = {"image", "sinogram", "spectrum"};
const char* const kGridKinds[] = {"cartesian", "polar", "logpolar_fine", "logpolar_sector"};  // types.hpp GridKind
}  // namespace

Json image_grid(int N) {
    Json g = Json::object();
    g["kind"] = "cartesian";
    g["axis0"] = axis(N, -0.5, 1.0 / N);
    g["axis1"] = axis(N, -0.5, 1.0 / N);
    return g;
}

Json sinogram_grid(int n_theta, int N) {
    Json g = Json::object();
    g["kind"] = "polar";
    g["axis0"] = axis(n_theta, 0.0, M_PI / n_theta);
    g["axis1"] = axis(N, -0.5, 1.0 / N);
    return g;
}

// ------------------------------------------------------------------ codec
std::vector<std::uint8_t> encode(const Container& c) {
    bool kind_ok = false;
    for (const char* k : kKinds) kind_ok |= c.kind == k;
    if (!kind_ok) throw SchemaError("kind must be image, sinogram or spectrum, got '" + c.kind + "'");
    if (c.rows < 0 || c.cols < 0) throw ShapeError("negative shape");
    const std::size_t words = c.complex ? 2 : 1;
    if (c.data.size() != std::size_t(c.rows) * std::size_t(c.cols) * words)
        throw ShapeError("payload holds " + std::to_string(c.data.size()) + " values, rows x cols needs " +
                         std::to_string(std::size_t(c.rows) * c.cols * words));
    Json h = Json::object();
    h["kind"] = c.kind;
    h["rows"] = Json(c.rows);
    h["cols"] = Json(c.cols);
    h["dtype"] = c.complex ? "c32" : "f32";
    h["grid"] = c.grid.type() == Json::Type::null ? Json::object() : c.grid;
    h["meta"] = c.meta.type() == Json::Type::null ? Json::object() : c.meta;
    const std::string hdr = h.dump();
    std::vector<std::uint8_t> out;
    out.reserve(8 + hdr.size() + c.data.size() * 4);
    out.insert(out.end(), {'L', 'P', 'T', '1'});
    const std::uint32_t n = std::uint32_t(hdr.size());
    for (int k = 0; k < 4; ++k) out.push_back(std::uint8_t(n >> (8 * k)));
    out.insert(out.end(), hdr.begin(), hdr.end());
    const std::size_t off = out.size();
    out.resize(off + c.data.size() * 4);
    for (std::size_t k = 0; k < c.data.size(); ++k) {  // little endian
        std::uint32_t u;
        std::memcpy(&u, &c.data[k], 4);
        for (int b = 0; b < 4; ++b) out[off + 4 * k + b] = std::uint8_t(u >> (8 * b));
    }
    return out;
}

Container decode(const std::vector<std::uint8_t>& buf) {
    if (buf.size() < 8) throw TruncatedError(std::to_string(buf.size()) + " bytes: shorter than magic + header length");
    if (std::memcmp(buf.data(), "LPT1", 4) != 0) throw BadMagicError("bad magic (expected LPT1)");
    const std::uint32_t hlen = std::uint32_t(buf[4]) | std::uint32_t(buf[5]) << 8 | std::uint32_t(buf[6]) << 16 |
                               std::uint32_t(buf[7]) << 24;
    if (buf.size() < 8 + std::size_t(hlen)) throw TruncatedError("header of " + std::to_string(hlen) + " bytes runs past the end of the file");
    const Json h = Json::parse(std::string(buf.begin() + 8, buf.begin() + 8 + hlen));
    if (!h.is_object()) throw SchemaError("header must be a JSON object");
    for (const char* k : {"kind", "dtype"})
        if (!h.has(k) || !h.at(k).is_string()) throw SchemaError(std::string("header field '") + k + "' missing or not str");
    for (const char* k : {"rows", "cols"})
        if (!h.has(k) || !h.at(k).is_int()) throw SchemaError(std::string("header field '") + k + "' missing or not int");
    Container c;
    c.kind = h.at("kind").as_string();
    bool kind_ok = false;
    for (const char* k : kKinds) kind_ok |= c.kind == k;
    if (!kind_ok) throw SchemaError("unknown kind '" + c.kind + "'");
    const std::string dt = h.at("dtype").as_string();
    if (dt != "f32" && dt != "c32") throw SchemaError("unknown dtype '" + dt + "'");
    c.complex = dt == "c32";
    const long long rows = h.at("rows").as_int(), cols = h.at("cols").as_int();
    if (rows < 0 || cols < 0) throw SchemaError("negative shape");
    c.rows = int(rows);
    c.cols = int(cols);
    c.grid = h.has("grid") ? h.at("grid") : Json::object();
    c.meta = h.has("meta") ? h.at("meta") : Json::object();
    if (!c.grid.is_object() || !c.meta.is_object()) throw SchemaError("grid and meta must be JSON objects");
    if (!c.grid.items().empty()) {
        bool ok = c.grid.has("kind") && c.grid.at("kind").is_string();
        bool known = false;
        if (ok)
            for (const char* k : kGridKinds) known |= c.grid.at("kind").as_string() == k;
        if (!known) throw SchemaError("unknown grid kind");
    }
    const std::size_t words = c.complex ? 2 : 1;
    const std::size_t row_bytes = std::size_t(cols) * 4 * words;
    const std::size_t want = std::size_t(rows) * row_bytes;
    const std::size_t got = buf.size() - 8 - hlen;
    if (got < want && got > 0 && got % (row_bytes ? row_bytes : 1) == 0)
        throw ShapeError("header says " + std::to_string(rows) + "x" + std::to_string(cols) + " but the payload holds " +
                         std::to_string(got / row_bytes) + " rows");
    if (got < want) throw TruncatedError("payload " + std::to_string(got) + " bytes, header needs " + std::to_string(want));
    if (got > want) throw ShapeError("payload " + std::to_string(got) + " bytes, header needs exactly " + std::to_string(want));
    c.data.resize(want / 4);
    const std::uint8_t* p = buf.data() + 8 + hlen;
    for (std::size_t k = 0; k < c.data.size(); ++k) {
        const std::uint32_t u = std::uint32_t(p[4 * k]) | std::uint32_t(p[4 * k + 1]) << 8 |
                                std::uint32_t(p[4 * k + 2]) << 16 | std::uint32_t(p[4 * k + 3]) << 24;
        std::memcpy(&c.data[k], &u, 4);
    }
    return c;
}

void write_container(const std::string& path, const Container& c) {
    const std::vector<std::uint8_t> b = encode(c);
    std::ofstream f(path, std::ios::binary);
    if (!f) throw std::runtime_error("cannot open '" + path + "' for writing");
    f.write(reinterpret_cast<const char*>(b.data()), std::streamsize(b.size()));
    if (!f) throw std::runtime_error("write to '" + path + "' failed");
}

Container read_container(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw std::runtime_error("cannot open '" + path + "'");
    std::vector<std::uint8_t> b((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    return decode(b);
}

}  // namespace lpr::io
