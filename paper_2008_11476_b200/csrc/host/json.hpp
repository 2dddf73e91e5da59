// Small JSON document model for graph files (graph_io) — parse, query, and
// a canonical writer.  The writer reproduces the layout of the reference's
// serializer (nlohmann::json dump: sorted object keys, 2-space indent or
// compact, integral values as integers, doubles as the shortest digits that
// round-trip with a ".0" suffix when integral and "e+XX" exponents outside
// 1e-5 .. 1e15), so canonical graph files are byte-identical.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

namespace gvx::json {

class Value {
public:
    enum class Type { Null, Bool, Int, UInt, Float, String, Array, Object };

    Value() = default;
    Value(std::nullptr_t) {}
    Value(bool b) : type_(Type::Bool), b_(b) {}
    Value(int v) : type_(Type::Int), i_(v) {}
    Value(long v) : type_(Type::Int), i_(v) {}
    Value(long long v) : type_(Type::Int), i_(v) {}
    Value(unsigned long v) : type_(Type::UInt), u_(v) {}
    Value(unsigned long long v) : type_(Type::UInt), u_(v) {}
    Value(double v) : type_(Type::Float), d_(v) {}
    Value(const char* s) : type_(Type::String), s_(s) {}
    Value(std::string s) : type_(Type::String), s_(std::move(s)) {}

    static Value array() {
        Value v;
        v.type_ = Type::Array;
        return v;
    }
    static Value object() {
        Value v;
        v.type_ = Type::Object;
        return v;
    }

    Type type() const { return type_; }
    bool is_null() const { return type_ == Type::Null; }
    bool is_bool() const { return type_ == Type::Bool; }
    bool is_string() const { return type_ == Type::String; }
    bool is_array() const { return type_ == Type::Array; }
    bool is_object() const { return type_ == Type::Object; }
    bool is_number() const { return type_ == Type::Int || type_ == Type::UInt || type_ == Type::Float; }
    bool is_float() const { return type_ == Type::Float; }
    bool is_integer() const { return type_ == Type::Int || type_ == Type::UInt; }
    /// Arrays / objects: element count; null: 0; scalars: 1.
    std::size_t size() const;
    bool empty() const { return size() == 0; }

    // typed reads: numbers convert among themselves (like the reference's
    // library); any other mismatch throws Error(SchemaError)
    std::int64_t as_int(const char* what = "value") const;
    double as_double(const char* what = "value") const;
    bool as_bool(const char* what = "value") const;
    const std::string& as_string(const char* what = "value") const;

    // arrays
    const std::vector<Value>& items(const char* what = "value") const;
    const Value& at(std::size_t i) const;
    void push_back(Value v);

    // objects
    bool contains(const std::string& key) const;
    const Value& at(const std::string& key) const; ///< SchemaError when absent
    Value& operator[](const std::string& key);     ///< inserts (null -> object)
    const std::map<std::string, Value>& members(const char* what = "value") const;
    std::int64_t value(const std::string& key, std::int64_t dflt) const;
    int value(const std::string& key, int dflt) const { return static_cast<int>(value(key, std::int64_t{dflt})); }
    bool value(const std::string& key, bool dflt) const;
    std::string value(const std::string& key, const std::string& dflt) const;
    std::string value(const std::string& key, const char* dflt) const { return value(key, std::string(dflt)); }

    /// indent < 0: compact; otherwise pretty with `indent` spaces per level.
    std::string dump(int indent = -1) const;

private:
    void dump_to(std::string& out, int indent, int level) const;

    Type type_ = Type::Null;
    bool b_ = false;
    std::int64_t i_ = 0;
    std::uint64_t u_ = 0;
    double d_ = 0.0;
    std::string s_;
    std::vector<Value> a_;
    std::map<std::string, Value> o_;
};

/// Strict RFC 8259 parse; returns false (and a message) on malformed text.
bool parse(const std::string& text, Value& out, std::string* error = nullptr);

/// Shortest decimal form of a double that reads back identically, in the
/// canonical number layout described above.
std::string format_double(double v);

} // namespace gvx::json
