// dagsched_b200 — kept C++ API, exact arithmetic.
//
// Same names and call shapes as the reference's rational.hpp (Boost
// cpp_int_backend<128,...> checked rationals, rational.hpp:17-40) so code
// written against the reference compiles unchanged: BigInt, Rational,
// make_rational, parse_rational, floor_to_int, ceil_to_int, to_int64,
// to_double, format_exact, format_fixed, numerator(), denominator(),
// .convert_to<T>(), .str(). Implementation is Boost-free: a checked
// signed-magnitude integer over an unsigned __int128 magnitude — Boost's
// cpp_int_backend<128, 128, signed_magnitude, checked> range +-(2^128 - 1);
// a result outside it throws std::overflow_error — and an always-reduced
// rational over it whose + - * / follow Boost.Rational's gcd-first
// algorithms, so intermediates (and overflow points) match the reference's.
// The device twin is csrc/rat.cuh.
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
    using u128 = unsigned __int128;
    BigInt() = default;
    template <class T, std::enable_if_t<std::is_integral_v<T>, int> = 0>
    BigInt(T v) {  // NOLINT (implicit, like Boost)
        if constexpr (std::is_signed_v<T>) {
            if (v < 0) {
                neg_ = true;
                mag_ = u128(-(static_cast<long long>(v) + 1)) + 1;
                return;
            }
        }
        mag_ = static_cast<u128>(v);
    }
    static BigInt from_parts(u128 mag, bool neg) {
        BigInt b;
        b.mag_ = mag;
        b.neg_ = neg && mag != 0;
        return b;
    }
    u128 magnitude() const { return mag_; }
    bool negative() const { return neg_; }
    std::string str() const;
    template <class T>
    T convert_to() const {
        if constexpr (std::is_floating_point_v<T>) {
            const T v = static_cast<T>(mag_);
            return neg_ ? -v : v;
        } else {  // saturating, like Boost's conversion of an out-of-range value
            using L = std::numeric_limits<T>;
            if (neg_) {
                if constexpr (std::is_signed_v<T>) {
                    const u128 lim = u128(-(static_cast<long long>(L::min()) + 1)) + 1;
                    return mag_ >= lim ? L::min() : static_cast<T>(-static_cast<long long>(mag_));
                } else {
                    return 0;
                }
            }
            return mag_ > static_cast<u128>(L::max()) ? L::max() : static_cast<T>(mag_);
        }
    }

    friend BigInt operator+(const BigInt& a, const BigInt& b);
    friend BigInt operator-(const BigInt& a, const BigInt& b) { return a + (-b); }
    friend BigInt operator*(const BigInt& a, const BigInt& b);
    friend BigInt operator/(const BigInt& a, const BigInt& b);
    friend BigInt operator%(const BigInt& a, const BigInt& b);
    friend BigInt operator-(const BigInt& a) { return from_parts(a.mag_, !a.neg_); }
    BigInt& operator+=(const BigInt& b) { return *this = *this + b; }
    BigInt& operator-=(const BigInt& b) { return *this = *this - b; }
    BigInt& operator*=(const BigInt& b) { return *this = *this * b; }
    BigInt& operator/=(const BigInt& b) { return *this = *this / b; }
    BigInt& operator++() { return *this += 1; }
    BigInt& operator--() { return *this -= 1; }
    friend int compare(const BigInt& a, const BigInt& b) {
        if (a.neg_ != b.neg_) return a.neg_ ? -1 : 1;
        const int c = a.mag_ < b.mag_ ? -1 : (a.mag_ > b.mag_ ? 1 : 0);
        return a.neg_ ? -c : c;
    }
    friend bool operator==(const BigInt& a, const BigInt& b) { return a.neg_ == b.neg_ && a.mag_ == b.mag_; }
    friend bool operator!=(const BigInt& a, const BigInt& b) { return !(a == b); }
    friend bool operator<(const BigInt& a, const BigInt& b) { return compare(a, b) < 0; }
    friend bool operator>(const BigInt& a, const BigInt& b) { return compare(a, b) > 0; }
    friend bool operator<=(const BigInt& a, const BigInt& b) { return compare(a, b) <= 0; }
    friend bool operator>=(const BigInt& a, const BigInt& b) { return compare(a, b) >= 0; }

  private:
    u128 mag_ = 0;
    bool neg_ = false;
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

    // B200 addition: n/d already in lowest terms with d > 0 (the device's
    // results are reduced), so no gcd is taken
    static Rational reduced(const BigInt& n, const BigInt& d) {
        Rational r;
        r.n_ = n;
        r.d_ = d;
        return r;
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
