// TEST INFRASTRUCTURE — oracle restatement (never linked into the product).
//
// Exact rational for the restated oracle. The reference uses Boost's
// 128-bit checked signed-magnitude rational (rational.hpp:17-20): always
// reduced, den > 0, overflow -> std::overflow_error. Here: signed __int128
// numerator/denominator with checked arithmetic; the range is ±(2^127-1),
// one bit short of the reference's ±(2^128-1) — any value that needs that
// last bit raises overflow here (never reached at the configs tested).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

namespace orc {

using i128 = __int128;

[[noreturn]] inline void q_overflow() { throw std::overflow_error("oracle rational overflow"); }

inline i128 q_abs(i128 v) { return v < 0 ? -v : v; }

inline i128 q_gcd(i128 a, i128 b) {
    a = q_abs(a);
    b = q_abs(b);
    while (b) {
        i128 t = a % b;
        a = b;
        b = t;
    }
    return a;
}
inline i128 q_mul(i128 a, i128 b) {
    i128 r;
    if (__builtin_mul_overflow(a, b, &r)) q_overflow();
    return r;
}
inline i128 q_add(i128 a, i128 b) {
    i128 r;
    if (__builtin_add_overflow(a, b, &r)) q_overflow();
    return r;
}

struct Q {
    i128 n = 0, d = 1;

    Q() = default;
    Q(long long v) : n(v), d(1) {}  // NOLINT
    Q(i128 num, i128 den) {
        if (den == 0) throw std::overflow_error("division by zero");
        if (den < 0) {
            num = -num;
            den = -den;
        }
        i128 g = q_gcd(num, den);
        if (g > 1) {
            num /= g;
            den /= g;
        }
        if (num == 0) den = 1;
        n = num;
        d = den;
    }
    static Q of(long long num, long long den) { return Q(i128(num), i128(den)); }
};

inline Q operator+(const Q& a, const Q& b) {
    i128 g = q_gcd(a.d, b.d);
    i128 ad = a.d / g, bd = b.d / g;
    return Q(q_add(q_mul(a.n, bd), q_mul(b.n, ad)), q_mul(a.d, bd));
}
inline Q operator-(const Q& a) { return Q(-a.n, a.d); }
inline Q operator-(const Q& a, const Q& b) { return a + (-b); }
inline Q operator*(const Q& a, const Q& b) {
    i128 g1 = q_gcd(a.n, b.d), g2 = q_gcd(b.n, a.d);
    if (g1 == 0) g1 = 1;
    if (g2 == 0) g2 = 1;
    return Q(q_mul(a.n / g1, b.n / g2), q_mul(a.d / g2, b.d / g1));
}
inline Q operator/(const Q& a, const Q& b) {
    if (b.n == 0) throw std::overflow_error("division by zero");
    return a * Q(b.d, b.n);
}

// exact three-way compare without overflow: compare a.n/a.d with b.n/b.d
// through their integer parts and remainders (continued-fraction step).
inline int q_cmp(const Q& a, const Q& b) {
    i128 an = a.n, ad = a.d, bn = b.n, bd = b.d;
    bool flip = false;
    for (;;) {
        // floor division
        i128 qa = an / ad, ra = an % ad;
        if (ra < 0) {
            qa -= 1;
            ra += ad;
        }
        i128 qb = bn / bd, rb = bn % bd;
        if (rb < 0) {
            qb -= 1;
            rb += bd;
        }
        if (qa != qb) return (qa < qb ? -1 : 1) * (flip ? -1 : 1);
        if (ra == 0 || rb == 0) {
            int c = (ra == 0 && rb == 0) ? 0 : (ra == 0 ? -1 : 1);
            return flip ? -c : c;
        }
        // compare ra/ad vs rb/bd  <=>  compare bd/rb vs ad/ra (reciprocal flips)
        i128 nan = bd, nad = rb, nbn = ad, nbd = ra;
        an = nan;
        ad = nad;
        bn = nbn;
        bd = nbd;
        // after swapping roles a<->b, the orientation is restored: no flip change
    }
}
inline bool operator==(const Q& a, const Q& b) { return a.n == b.n && a.d == b.d; }
inline bool operator!=(const Q& a, const Q& b) { return !(a == b); }
inline bool operator<(const Q& a, const Q& b) { return q_cmp(a, b) < 0; }
inline bool operator>(const Q& a, const Q& b) { return q_cmp(a, b) > 0; }
inline bool operator<=(const Q& a, const Q& b) { return q_cmp(a, b) <= 0; }
inline bool operator>=(const Q& a, const Q& b) { return q_cmp(a, b) >= 0; }

inline i128 q_floor(const Q& q) {
    i128 f = q.n / q.d;
    if (q.n < 0 && f * q.d != q.n) --f;
    return f;
}
inline i128 q_ceil(const Q& q) {
    i128 f = q.n / q.d;
    if (q.n > 0 && f * q.d != q.n) ++f;
    return f;
}
inline double q_double(const Q& q) { return double(q.n) / double(q.d); }

inline std::string i128_str(i128 v) {
    if (v == 0) return "0";
    bool neg = v < 0;
    unsigned __int128 m = neg ? (unsigned __int128)(-(v + 1)) + 1 : (unsigned __int128)v;
    std::string s;
    while (m) {
        s.insert(s.begin(), char('0' + int(m % 10)));
        m /= 10;
    }
    return neg ? "-" + s : s;
}
inline std::string q_str(const Q& q) {
    return q.d == 1 ? i128_str(q.n) : i128_str(q.n) + "/" + i128_str(q.d);
}

}  // namespace orc
