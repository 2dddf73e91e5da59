// Base enums, names and format tables.
// Behaviour follows ref:src/format.cpp:7-163 (names, byte sizes, ranges).
#include "graphvx/error.hpp"
#include "graphvx/format.hpp"
#include "graphvx/kernel.hpp"

#include <array>
#include <climits>

namespace gvx {

namespace {

template <typename E, std::size_t N>
bool parse_by_name(const std::string& s, const std::array<E, N>& all, E& out) {
    for (E e : all)
        if (s == to_string(e)) {
            out = e;
            return true;
        }
    return false;
}

} // namespace

const char* error_code_name(ErrorCode code) {
    static const char* const names[] = {
        "ZeroDimension", "BadFormat",      "BadKernel",     "AccessDenied",  "UnknownObject",
        "UnknownKernel", "CrossGraphVirtual", "MultipleWriters", "CycleDetected",
        "UnstampedGraph", "MissingInput",  "ShapeMismatch", "DivByZero",     "TypeMismatch",
        "MissingCast",   "OffsetOutOfWindow", "UnsupportedKind", "NonStreamable", "IoError",
        "SchemaError"};
    auto i = static_cast<std::size_t>(code);
    return i < sizeof(names) / sizeof(names[0]) ? names[i] : "Unknown";
}

const char* to_string(ImageFormat f) {
    static const char* const names[] = {"U8", "U16", "S16", "S32", "F32", "RGB", "UYVY",
                                        "UNRESOLVED"};
    auto i = static_cast<std::size_t>(f);
    return i < 8 ? names[i] : "?";
}

const char* to_string(ScalarType t) {
    static const char* const names[] = {"U8", "U16", "S16", "S32", "F32", "I64", "F64"};
    auto i = static_cast<std::size_t>(t);
    return i < 7 ? names[i] : "?";
}

const char* to_string(Channel c) {
    static const char* const names[] = {"0", "R", "G", "B", "Y", "U", "V"};
    auto i = static_cast<std::size_t>(c);
    return i < 7 ? names[i] : "?";
}

bool parse_image_format(const std::string& s, ImageFormat& out) {
    static const std::array<ImageFormat, 8> all = {
        ImageFormat::U8,  ImageFormat::U16, ImageFormat::S16,  ImageFormat::S32,
        ImageFormat::F32, ImageFormat::RGB, ImageFormat::UYVY, ImageFormat::UNRESOLVED};
    return parse_by_name(s, all, out);
}

bool parse_scalar_type(const std::string& s, ScalarType& out) {
    static const std::array<ScalarType, 7> all = {ScalarType::U8,  ScalarType::U16,
                                                  ScalarType::S16, ScalarType::S32,
                                                  ScalarType::F32, ScalarType::I64,
                                                  ScalarType::F64};
    return parse_by_name(s, all, out);
}

bool parse_channel(const std::string& s, Channel& out) {
    static const std::array<Channel, 7> all = {Channel::C0, Channel::R, Channel::G, Channel::B,
                                               Channel::Y,  Channel::U, Channel::V};
    return parse_by_name(s, all, out);
}

int channel_count(ImageFormat f) {
    return (f == ImageFormat::RGB || f == ImageFormat::UYVY) ? 3 : 1;
}

int bytes_per_pixel(ImageFormat f) {
    switch (f) {
    case ImageFormat::U8: return 1;
    case ImageFormat::U16:
    case ImageFormat::S16:
    case ImageFormat::UYVY: return 2;
    case ImageFormat::RGB: return 3;
    case ImageFormat::S32:
    case ImageFormat::F32: return 4;
    case ImageFormat::UNRESOLVED: return 0;
    }
    return 0;
}

ScalarType scalar_of(ImageFormat f) {
    switch (f) {
    case ImageFormat::U8:
    case ImageFormat::RGB:
    case ImageFormat::UYVY: return ScalarType::U8;
    case ImageFormat::U16: return ScalarType::U16;
    case ImageFormat::S16: return ScalarType::S16;
    case ImageFormat::S32: return ScalarType::S32;
    case ImageFormat::F32: return ScalarType::F32;
    case ImageFormat::UNRESOLVED: break;
    }
    throw Error(ErrorCode::BadFormat, "no scalar type for UNRESOLVED");
}

ImageFormat format_of(ScalarType t) {
    switch (t) {
    case ScalarType::U8: return ImageFormat::U8;
    case ScalarType::U16: return ImageFormat::U16;
    case ScalarType::S16: return ImageFormat::S16;
    case ScalarType::S32: return ImageFormat::S32;
    case ScalarType::F32: return ImageFormat::F32;
    default: break;
    }
    throw Error(ErrorCode::BadFormat, "internal type has no storage format");
}

bool integer_range(ScalarType t, std::int64_t& lo, std::int64_t& hi) {
    switch (t) {
    case ScalarType::U8: lo = 0, hi = 255; return true;
    case ScalarType::U16: lo = 0, hi = 65535; return true;
    case ScalarType::S16: lo = -32768, hi = 32767; return true;
    case ScalarType::S32: lo = INT32_MIN, hi = INT32_MAX; return true;
    default: return false;
    }
}

// ---- kernel.hpp enum names ------------------------------------------------

const char* to_string(Direction d) { return d == Direction::Input ? "INPUT" : "OUTPUT"; }

const char* to_string(ObjKind k) {
    static const char* const names[] = {"image", "scalar", "array", "matrix"};
    auto i = static_cast<std::size_t>(k);
    return i < 4 ? names[i] : "?";
}

const char* to_string(BoundaryMode m) {
    static const char* const names[] = {"clamp", "constant", "undefined"};
    auto i = static_cast<std::size_t>(m);
    return i < 3 ? names[i] : "?";
}

const char* to_string(CombineMode m) {
    static const char* const names[] = {"sum", "min", "max"};
    auto i = static_cast<std::size_t>(m);
    return i < 3 ? names[i] : "?";
}

const char* to_string(InterpMode m) { return m == InterpMode::Nearest ? "nearest" : "bilinear"; }

const char* to_string(AbstractionKind k) {
    static const char* const names[] = {"point", "local", "reduce", "histogram",
                                        "scale", "scan",  "table"};
    auto i = static_cast<std::size_t>(k);
    return i < 7 ? names[i] : "?";
}

} // namespace gvx
