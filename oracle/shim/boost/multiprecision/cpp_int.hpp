// TEST INFRASTRUCTURE — oracle only. Never linked into the product.
//
// Restatement of the subset of Boost.Multiprecision that the reference
// (arxiv/paper_2602_20826, /root/reference/proj) uses, so that the reference's
// own sources can be compiled here unmodified into oracle/_ref/ (Boost is not
// installed in this image and there is no network).
//
// What is restated (version of Boost the reference used: UNPINNED — no lockfile,
// vendor/ is git-ignored, proj/.gitignore:2):
//   number<cpp_int_backend<128,128,signed_magnitude,checked,void>>
//       -> 128-bit signed-magnitude integer, range ±(2^128-1); any result
//          outside the range throws std::overflow_error (checked backend).
//   number<rational_adaptor<cpp_int_backend<...>>>
//       -> always-canonical rational (gcd-reduced, den > 0).
//          +,- follow Knuth's / Boost.Rational's gcd-of-denominators
//          algorithm and *,/ cross-cancel before multiplying, so
//          intermediates match Boost's in magnitude.
//          Comparisons are EXACT (256-bit cross products): where Boost would
//          throw on a cross-product overflow we compare correctly instead
//          (documented divergence; never reached at the configs used).
// Call sites in the reference: rational.hpp:17-24, rational.cpp:27-112,
// exec_model.cpp:7-23, dag.cpp:127-135, scheduler.cpp:41-93/236-309,
// analysis.cpp:28-81, generator.cpp:65-92, simulator.cpp:24-35.
//
// Expression templates are off in Boost for fixed-width cpp_int backends, so
// returning plain values here keeps the reference code's semantics
// (e.g. std::max(a, b + c) compiles in both).
#pragma once

#include <cstdint>
#include <limits>
#include <stdexcept>
#include <string>
#include <type_traits>

namespace boost {
namespace multiprecision {

enum cpp_integer_type { signed_magnitude = 1, unsigned_magnitude = 0 };
enum cpp_int_check_type { checked = 1, unchecked = 0 };

template <unsigned MinBits = 0, unsigned MaxBits = 0,
          cpp_integer_type SignType = signed_magnitude,
          cpp_int_check_type Checked = unchecked, class Allocator = void>
struct cpp_int_backend {};

template <class IntBackend>
struct rational_adaptor {};

template <class Backend>
class number;

namespace shim_detail {

using u128 = unsigned __int128;

[[noreturn]] inline void raise_overflow(const char* what) {
    throw std::overflow_error(what);
}

inline u128 gcd_u128(u128 a, u128 b) {
    while (b != 0) {
        u128 t = a % b;
        a = b;
        b = t;
    }
    return a;
}

// 128x128 -> 256 unsigned product, as (hi, lo).
inline void mul_wide(u128 a, u128 b, u128& hi, u128& lo) {
    const u128 mask = (u128(1) << 64) - 1;
    u128 a0 = a & mask, a1 = a >> 64, b0 = b & mask, b1 = b >> 64;
    u128 p00 = a0 * b0, p01 = a0 * b1, p10 = a1 * b0, p11 = a1 * b1;
    u128 mid = (p00 >> 64) + (p01 & mask) + (p10 & mask);
    lo = (p00 & mask) | (mid << 64);
    hi = p11 + (p01 >> 64) + (p10 >> 64) + (mid >> 64);
}

}  // namespace shim_detail

// ---------------------------------------------------------------- BigInt
template <unsigned MinBits, unsigned MaxBits, cpp_integer_type SignType,
          cpp_int_check_type Checked, class Allocator>
class number<cpp_int_backend<MinBits, MaxBits, SignType, Checked, Allocator>> {
    static_assert(MinBits == 128 && MaxBits == 128 && SignType == signed_magnitude &&
                      Checked == checked,
                  "oracle shim only restates the 128-bit checked signed-magnitude cpp_int");
    using u128 = shim_detail::u128;

  public:
    number() = default;

    template <class T, std::enable_if_t<std::is_integral_v<T>, int> = 0>
    number(T v) {  // NOLINT: implicit like Boost
        if constexpr (std::is_signed_v<T>) {
            if (v < 0) {
                neg_ = true;
                mag_ = u128(-(static_cast<long long>(v) + 1)) + 1;
                return;
            }
        }
        mag_ = static_cast<u128>(v);
    }

    static number from_parts(u128 mag, bool neg) {
        number r;
        r.mag_ = mag;
        r.neg_ = mag != 0 && neg;
        return r;
    }
    u128 magnitude() const { return mag_; }
    bool negative() const { return neg_; }
    bool is_zero() const { return mag_ == 0; }

    std::string str() const {
        if (mag_ == 0) return "0";
        std::string s;
        u128 m = mag_;
        while (m != 0) {
            s.insert(s.begin(), char('0' + int(m % 10)));
            m /= 10;
        }
        if (neg_) s.insert(s.begin(), '-');
        return s;
    }

    template <class T>
    T convert_to() const {
        if constexpr (std::is_floating_point_v<T>) {
            T v = static_cast<T>(mag_);
            return neg_ ? -v : v;
        } else {
            // saturate to the target range
            using L = std::numeric_limits<T>;
            if (neg_) {
                if constexpr (std::is_signed_v<T>) {
                    u128 lim = u128(-(static_cast<long long>(L::min()) + 1)) + 1;
                    if (mag_ >= lim) return L::min();
                    return static_cast<T>(-static_cast<long long>(mag_));
                } else {
                    return 0;
                }
            }
            if (mag_ > static_cast<u128>(L::max())) return L::max();
            return static_cast<T>(mag_);
        }
    }

    friend number operator-(const number& a) { return from_parts(a.mag_, !a.neg_); }

    friend number operator+(const number& a, const number& b) {
        if (a.neg_ == b.neg_) {
            u128 m = a.mag_ + b.mag_;
            if (m < a.mag_) shim_detail::raise_overflow("cpp_int addition overflow");
            return from_parts(m, a.neg_);
        }
        if (a.mag_ >= b.mag_) return from_parts(a.mag_ - b.mag_, a.neg_);
        return from_parts(b.mag_ - a.mag_, b.neg_);
    }
    friend number operator-(const number& a, const number& b) { return a + (-b); }
    friend number operator*(const number& a, const number& b) {
        u128 m;
        if (__builtin_mul_overflow(a.mag_, b.mag_, &m)) {
            shim_detail::raise_overflow("cpp_int multiplication overflow");
        }
        return from_parts(m, a.neg_ != b.neg_);
    }
    friend number operator/(const number& a, const number& b) {
        if (b.mag_ == 0) shim_detail::raise_overflow("Division by zero.");
        return from_parts(a.mag_ / b.mag_, a.neg_ != b.neg_);
    }
    friend number operator%(const number& a, const number& b) {
        if (b.mag_ == 0) shim_detail::raise_overflow("Division by zero.");
        return from_parts(a.mag_ % b.mag_, a.neg_);
    }

    number& operator+=(const number& b) { return *this = *this + b; }
    number& operator-=(const number& b) { return *this = *this - b; }
    number& operator*=(const number& b) { return *this = *this * b; }
    number& operator/=(const number& b) { return *this = *this / b; }
    number& operator%=(const number& b) { return *this = *this % b; }
    number& operator++() { return *this += number(1); }
    number& operator--() { return *this -= number(1); }

    friend int compare(const number& a, const number& b) {
        if (a.neg_ != b.neg_) return a.neg_ ? -1 : 1;
        int c = a.mag_ < b.mag_ ? -1 : (a.mag_ > b.mag_ ? 1 : 0);
        return a.neg_ ? -c : c;
    }
    friend bool operator==(const number& a, const number& b) { return compare(a, b) == 0; }
    friend bool operator!=(const number& a, const number& b) { return compare(a, b) != 0; }
    friend bool operator<(const number& a, const number& b) { return compare(a, b) < 0; }
    friend bool operator>(const number& a, const number& b) { return compare(a, b) > 0; }
    friend bool operator<=(const number& a, const number& b) { return compare(a, b) <= 0; }
    friend bool operator>=(const number& a, const number& b) { return compare(a, b) >= 0; }

  private:
    u128 mag_ = 0;
    bool neg_ = false;
};

// -------------------------------------------------------------- Rational
template <class IntBackend>
class number<rational_adaptor<IntBackend>> {
    using u128 = shim_detail::u128;

  public:
    using int_type = number<IntBackend>;

    number() : num_(0), den_(1) {}

    template <class T, std::enable_if_t<std::is_integral_v<T>, int> = 0>
    number(T v) : num_(v), den_(1) {}  // NOLINT: implicit like Boost
    number(const int_type& v) : num_(v), den_(1) {}  // NOLINT

    template <class A, class B,
              std::enable_if_t<(std::is_integral_v<A> || std::is_same_v<A, int_type>) &&
                                   (std::is_integral_v<B> || std::is_same_v<B, int_type>),
                               int> = 0>
    number(const A& n, const B& d) {
        assign(int_type(n), int_type(d));
    }

    const int_type& num() const { return num_; }
    const int_type& den() const { return den_; }

    template <class T>
    T convert_to() const {
        if constexpr (std::is_floating_point_v<T>) {
            return num_.template convert_to<T>() / den_.template convert_to<T>();
        } else {
            return (num_ / den_).template convert_to<T>();
        }
    }
    std::string str() const {
        if (den_ == int_type(1)) return num_.str();
        return num_.str() + "/" + den_.str();
    }

    friend number operator-(const number& a) { return raw(-a.num_, a.den_); }

    // Knuth / Boost.Rational: g = gcd(d1, d2); n = n1*(d2/g) +- n2*(d1/g);
    // g2 = gcd(n, g); result = (n/g2) / ((d1/g) * (d2/g2)).
    static number add_sub(const number& a, const number& b, bool add) {
        int_type g = gcd(a.den_, b.den_);
        int_type a_d = a.den_ / g;
        int_type b_d = b.den_ / g;
        int_type n = add ? a.num_ * b_d + b.num_ * a_d : a.num_ * b_d - b.num_ * a_d;
        int_type g2 = gcd(n, g);
        if (n.is_zero()) return number();
        return raw(n / g2, a_d * (b.den_ / g2));
    }
    friend number operator+(const number& a, const number& b) { return add_sub(a, b, true); }
    friend number operator-(const number& a, const number& b) { return add_sub(a, b, false); }
    friend number operator*(const number& a, const number& b) {
        if (a.num_.is_zero() || b.num_.is_zero()) return number();
        int_type g1 = gcd(a.num_, b.den_);
        int_type g2 = gcd(b.num_, a.den_);
        return raw((a.num_ / g1) * (b.num_ / g2), (a.den_ / g2) * (b.den_ / g1));
    }
    friend number operator/(const number& a, const number& b) {
        if (b.num_.is_zero()) shim_detail::raise_overflow("Division by zero.");
        if (a.num_.is_zero()) return number();
        int_type g1 = gcd(a.num_, b.num_);
        int_type g2 = gcd(b.den_, a.den_);
        int_type n = (a.num_ / g1) * (b.den_ / g2);
        int_type d = (a.den_ / g2) * (b.num_ / g1);
        if (d.negative()) {
            n = -n;
            d = -d;
        }
        return raw(n, d);
    }
    number& operator+=(const number& b) { return *this = *this + b; }
    number& operator-=(const number& b) { return *this = *this - b; }
    number& operator*=(const number& b) { return *this = *this * b; }
    number& operator/=(const number& b) { return *this = *this / b; }

    friend int compare(const number& a, const number& b) {
        bool an = a.num_.negative(), bn = b.num_.negative();
        if (an != bn) return an ? -1 : 1;
        u128 h1, l1, h2, l2;
        shim_detail::mul_wide(a.num_.magnitude(), b.den_.magnitude(), h1, l1);
        shim_detail::mul_wide(b.num_.magnitude(), a.den_.magnitude(), h2, l2);
        int c = h1 != h2 ? (h1 < h2 ? -1 : 1) : (l1 < l2 ? -1 : (l1 > l2 ? 1 : 0));
        return an ? -c : c;
    }
    friend bool operator==(const number& a, const number& b) {
        return a.num_ == b.num_ && a.den_ == b.den_;
    }
    friend bool operator!=(const number& a, const number& b) { return !(a == b); }
    friend bool operator<(const number& a, const number& b) { return compare(a, b) < 0; }
    friend bool operator>(const number& a, const number& b) { return compare(a, b) > 0; }
    friend bool operator<=(const number& a, const number& b) { return compare(a, b) <= 0; }
    friend bool operator>=(const number& a, const number& b) { return compare(a, b) >= 0; }

    friend int_type numerator(const number& r) { return r.num_; }
    friend int_type denominator(const number& r) { return r.den_; }

  private:
    static int_type gcd(const int_type& a, const int_type& b) {
        return int_type::from_parts(shim_detail::gcd_u128(a.magnitude(), b.magnitude()),
                                    false);
    }
    static number raw(const int_type& n, const int_type& d) {
        number r;
        r.num_ = n;
        r.den_ = d;
        return r;
    }
    void assign(int_type n, int_type d) {
        if (d.is_zero()) shim_detail::raise_overflow("Division by zero.");
        if (d.negative()) {
            n = -n;
            d = -d;
        }
        int_type g = gcd(n, d);
        if (n.is_zero()) {
            num_ = int_type(0);
            den_ = int_type(1);
            return;
        }
        num_ = n / g;
        den_ = d / g;
    }

    int_type num_;
    int_type den_;
};

}  // namespace multiprecision
}  // namespace boost
