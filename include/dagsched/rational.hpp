// dagsched_b200 — kept C++ API, exact arithmetic.
//
// Same names and call shapes as the reference's rational.hpp (Boost
// cpp_int_backend<128,...> checked rationals, rational.hpp:17-40) so code
// written against the reference compiles unchanged: BigInt, Rational,
// make_rational, parse_rational, floor_to_int, ceil_to_int, to_int64,
// to_double, format_exact, format_fixed, numerator(), denominator(),
// .convert_to<T>(), .str(). Implementation is Boost-free: a checked signed
// __int128 (range +-(2^127 - 1), one bit short of Boost's signed-magnitude
// 2^128 - 1; out of range -> std::overflow_error) and an always-reduced
// rational over it. The device twin is csrc/rat.cuh.
#pragma once

#include <cstdint>
#include <limits>
#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>
#include <type_traits>

namespace dagsched {

class BigInt {
  public:
    BigInt() = default;
    template <class T, std::enable_if_t<std::is_integral_v<T>, int> = 0>
    BigInt(T v) : v_(static_cast<__int128>(v)) {}  // NOLINT (implicit, like Boost)

    static BigInt raw(__int128 v) {
        BigInt b;
        b.v_ = v;
        return b;
    }
    __int128 value() const { return v_; }
    std::string str() const;
    template <class T>
    T convert_to() const {
        if constexpr (std::is_floating_point_v<T>) return static_cast<T>(v_);
        else return v_ > static_cast<__int128>(std::numeric_limits<T>::max())   ? std::numeric_limits<T>::max()
                    : v_ < static_cast<__int128>(std::numeric_limits<T>::min()) ? std::numeric_limits<T>::min()
                                                                                : static_cast<T>(v_);
    }

    friend BigInt operator+(const BigInt& a, const BigInt& b);
    friend BigInt operator-(const BigInt& a, const BigInt& b);
    friend BigInt operator*(const BigInt& a, const BigInt& b);
    friend BigInt operator/(const BigInt& a, const BigInt& b);
    friend BigInt operator%(const BigInt& a, const BigInt& b);
    friend BigInt operator-(const BigInt& a) { return BigInt(0) - a; }
    BigInt& operator+=(const BigInt& b) { return *this = *this + b; }
    BigInt& operator-=(const BigInt& b) { return *this = *this - b; }
    BigInt& operator*=(const BigInt& b) { return *this = *this * b; }
    BigInt& operator/=(const BigInt& b) { return *this = *this / b; }
    BigInt& operator++() { return *this += 1; }
    BigInt& operator--() { return *this -= 1; }
    friend bool operator==(const BigInt& a, const BigInt& b) { return a.v_ == b.v_; }
    friend bool operator!=(const BigInt& a, const BigInt& b) { return a.v_ != b.v_; }
    friend bool operator<(const BigInt& a, const BigInt& b) { return a.v_ < b.v_; }
    friend bool operator>(const BigInt& a, const BigInt& b) { return a.v_ > b.v_; }
    friend bool operator<=(const BigInt& a, const BigInt& b) { return a.v_ <= b.v_; }
    friend bool operator>=(const BigInt& a, const BigInt& b) { return a.v_ >= b.v_; }

  private:
    __int128 v_ = 0;
};

class Rational {
  public:
    Rational() = default;
    template <class T, std::enable_if_t<std::is_integral_v<T>, int> = 0>
    Rational(T v) : n_(v), d_(1) {}            // NOLINT
    Rational(const BigInt& v) : n_(v), d_(1) {}  // NOLINT
    template <class A, class B,
              std::enable_if_t<(std::is_integral_v<A> || std::is_same_v<A, BigInt>) &&
                                   (std::is_integral_v<B> || std::is_same_v<B, BigInt>),
                               int> = 0>
    Rational(const A& num, const B& den) {
        set(BigInt(num), BigInt(den));
    }

    const BigInt& num() const { return n_; }
    const BigInt& den() const { return d_; }
    template <class T>
    T convert_to() const {
        if constexpr (std::is_floating_point_v<T>) return n_.convert_to<T>() / d_.convert_to<T>();
        else return (n_ / d_).convert_to<T>();
    }
    std::string str() const;

    friend Rational operator+(const Rational& a, const Rational& b);
    friend Rational operator-(const Rational& a, const Rational& b);
    friend Rational operator*(const Rational& a, const Rational& b);
    friend Rational operator/(const Rational& a, const Rational& b);
    friend Rational operator-(const Rational& a) { return Rational(-a.n_, a.d_); }
    Rational& operator+=(const Rational& b) { return *this = *this + b; }
    Rational& operator-=(const Rational& b) { return *this = *this - b; }
    Rational& operator*=(const Rational& b) { return *this = *this * b; }
    Rational& operator/=(const Rational& b) { return *this = *this / b; }
    friend int compare(const Rational& a, const Rational& b);
    friend bool operator==(const Rational& a, const Rational& b) { return a.n_ == b.n_ && a.d_ == b.d_; }
    friend bool operator!=(const Rational& a, const Rational& b) { return !(a == b); }
    friend bool operator<(const Rational& a, const Rational& b) { return compare(a, b) < 0; }
    friend bool operator>(const Rational& a, const Rational& b) { return compare(a, b) > 0; }
    friend bool operator<=(const Rational& a, const Rational& b) { return compare(a, b) <= 0; }
    friend bool operator>=(const Rational& a, const Rational& b) { return compare(a, b) >= 0; }

  private:
    void set(BigInt n, BigInt d);
    BigInt n_ = 0, d_ = 1;
};

inline BigInt numerator(const Rational& r) { return r.num(); }
inline BigInt denominator(const Rational& r) { return r.den(); }

inline Rational make_rational(long long num, long long den = 1) { return Rational(BigInt(num), BigInt(den)); }

// "12", "-3.25", "7/3" -> value; nullopt when malformed (rational.cpp:27-65)
std::optional<Rational> parse_rational(std::string_view text);
BigInt floor_to_int(const Rational& r);
BigInt ceil_to_int(const Rational& r);
long long to_int64(const BigInt& v);
double to_double(const Rational& r);
// "5" or "5/3"; round-trips through parse_rational
std::string format_exact(const Rational& r);
// fixed-point decimal, `digits` fraction digits, half away from zero
std::string format_fixed(const Rational& r, int digits);

}  // namespace dagsched
