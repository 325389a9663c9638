// Internal: the JSON subset the kept task_io API reads and writes
// (task_io.hpp:14-19 file format, write_scheme's document). The reference
// uses nlohmann/json; this is a small value type with the behaviour that
// matters for byte-identical files and for the reference's accessor
// semantics:
//   * numbers keep their kind — integer (int64 / uint64, as nlohmann's
//     number_integer / number_unsigned) or float (double) — so a load `7`
//     and a load `7.5` take different paths in rational_from_json;
//   * objects keep their keys sorted (nlohmann's default std::map), and
//     dump(2) lays documents out as nlohmann's dump(2) does: two-space
//     indent, one element per line, `"key": value`, empty containers as
//     `{}` / `[]`, strings escaped as nlohmann escapes them (UTF-8 kept).
#pragma once

#include <cstdint>
#include <exception>
#include <map>
#include <memory>
#include <string>
#include <vector>

namespace dagsched::detail {

// parse, type and missing-key errors: like nlohmann::json::exception, derived
// from std::exception only (not std::invalid_argument / std::out_of_range)
class JsonError : public std::exception {
  public:
    explicit JsonError(std::string what) : what_(std::move(what)) {}
    const char* what() const noexcept override { return what_.c_str(); }

  private:
    std::string what_;
};

class Json {
  public:
    enum class Kind { null, boolean, integer, unsigned_integer, floating, string, array, object };

    Json() = default;
    static Json boolean(bool b);
    static Json integer(std::int64_t v);
    static Json unsigned_integer(std::uint64_t v);
    static Json floating(double v);
    static Json string(std::string s);
    static Json array();
    static Json object();

    Kind kind() const { return kind_; }
    bool is_object() const { return kind_ == Kind::object; }
    bool is_array() const { return kind_ == Kind::array; }
    bool is_string() const { return kind_ == Kind::string; }
    bool is_number_integer() const { return kind_ == Kind::integer || kind_ == Kind::unsigned_integer; }
    bool is_number_float() const { return kind_ == Kind::floating; }
    bool is_number() const { return is_number_integer() || is_number_float(); }

    // accessors: JsonError on a type mismatch (nlohmann: type_error)
    const std::string& str() const;
    long long as_int64() const;        // any number, converted like get<long long>()
    std::uint32_t as_uint32() const;   // any number, converted like get<std::uint32_t>()
    double as_double() const;
    bool contains(const std::string& key) const;
    const Json& at(const std::string& key) const;  // JsonError if absent
    const Json& operator[](std::size_t i) const;
    std::size_t size() const;
    // what a range-for over a nlohmann value visits: array elements, object
    // values (key order), nothing for null, the value itself otherwise
    std::vector<const Json*> items() const;

    // building
    Json& push_back(Json v);
    Json& set(const std::string& key, Json v);

    // nlohmann's dump(indent)
    std::string dump(int indent = 2) const;
    static Json parse(const std::string& text);  // JsonError("parse error ...")

  private:
    void dump_to(std::string& out, int indent, int level) const;
    Kind kind_ = Kind::null;
    bool b_ = false;
    std::int64_t i_ = 0;
    std::uint64_t u_ = 0;
    double d_ = 0.0;
    std::string s_;
    std::vector<Json> a_;
    std::map<std::string, Json> o_;
};

}  // namespace dagsched::detail
