// lpt1.hpp — LPT1 binary containers (the reference's
// cli_io module; proj/src/io.cpp:1-2 is an empty namespace upstream).
//
// Layout: magic "LPT1" | header_len (uint32 LE) | UTF-8 JSON header
// {"cols", "dtype": "f32"|"c32", "grid": GridSpec fields, "kind":
// "image"|"sinogram"|"spectrum", "meta": {...}, "rows"} | row-major LE
// IEEE-754 float32 payload (complex interleaved re, im), exactly
// rows * cols * 4 * (1 | 2) bytes. The header is written with sorted keys and
// no spaces, floats in shortest round-trip form, so read(write(x)) is byte
// identical and a file written here is byte identical to one written by the
// Python mirror (paper_1506_00014_b200/lpt1.py) for the same container.
//
// Errors are distinct classes of std::invalid_argument (the reference's
// precondition family, types.hpp:72-74): BadMagicError, TruncatedError,
// ShapeError, SchemaError.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace lpr::io {

struct BadMagicError : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct TruncatedError : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct ShapeError : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct SchemaError : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};

/// A JSON value (the header and its free "meta" map).
class Json {
public:
    enum class Type { null, boolean, integer, number, string, array, object };
    Json() = default;
    Json(bool b) : type_(Type::boolean), b_(b) {}
    Json(int v) : type_(Type::integer), i_(v) {}
    Json(long v) : type_(Type::integer), i_(v) {}
    Json(long long v) : type_(Type::integer), i_(v) {}
    Json(double v) : type_(Type::number), d_(v) {}
    Json(const char* s) : type_(Type::string), s_(s) {}
    Json(std::string s) : type_(Type::string), s_(std::move(s)) {}
    static Json object() { Json j; j.type_ = Type::object; return j; }
    static Json array() { Json j; j.type_ = Type::array; return j; }

    Type type() const { return type_; }
    bool is_object() const { return type_ == Type::object; }
    bool is_int() const { return type_ == Type::integer; }
    bool is_string() const { return type_ == Type::string; }
    long long as_int() const;
    double as_number() const;  ///< integer or number
    const std::string& as_string() const;
    const std::map<std::string, Json>& items() const { return o_; }
    const std::vector<Json>& elements() const { return a_; }
    bool has(const std::string& k) const { return type_ == Type::object && o_.count(k) > 0; }
    const Json& at(const std::string& k) const;
    Json& operator[](const std::string& k);  ///< object member (turns null into an object)
    void push_back(Json v);

    /// Compact JSON with sorted keys, ASCII escapes and shortest round-trip
    /// floats — the bytes of Python's json.dumps(sort_keys=True, separators=(",", ":")).
    std::string dump() const;
    static Json parse(const std::string& text);  ///< throws SchemaError

private:
    Type type_ = Type::null;
    bool b_ = false;
    long long i_ = 0;
    double d_ = 0.0;
    std::string s_;
    std::vector<Json> a_;
    std::map<std::string, Json> o_;
};

struct Container {
    std::string kind;           ///< "image" | "sinogram" | "spectrum"
    int rows = 0, cols = 0;
    bool complex = false;       ///< dtype "c32" (interleaved re, im) vs "f32"
    std::vector<float> data;    ///< rows * cols * (complex ? 2 : 1) values, row-major
    Json grid = Json::object(); ///< GridSpec fields (types.hpp:42-58); {} when absent
    Json meta = Json::object(); ///< free metadata
};

/// GridSpec of the image raster [-1/2, 1/2)^2 (geometry.cpp:19-25) and of the
/// sinogram theta_i = i pi / n_theta, s_j = -1/2 + j / N (geometry.cpp:27-33).
Json image_grid(int N);
Json sinogram_grid(int n_theta, int N);

std::vector<std::uint8_t> encode(const Container& c);
Container decode(const std::vector<std::uint8_t>& bytes);
void write_container(const std::string& path, const Container& c);
Container read_container(const std::string& path);

}  // namespace lpr::io
