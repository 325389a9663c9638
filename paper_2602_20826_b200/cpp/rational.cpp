// Kept C++ API — exact arithmetic (include/dagsched/rational.hpp).
#include "dagsched/rational.hpp"

#include <cctype>

namespace dagsched {

namespace {
using u128 = unsigned __int128;
[[noreturn]] void overflow(const char* what) { throw std::overflow_error(what); }
u128 gcd_u(u128 a, u128 b) {
    // Euclid in 128 bits (software division) only until both fit 64 bits,
    // then binary gcd on u64 — the common case for every load and bound
    while (b && ((a >> 64) || (b >> 64))) {
        const u128 t = a % b;
        a = b;
        b = t;
    }
    if (b == 0) return a;  // (a may still be wide)
    std::uint64_t x = std::uint64_t(a), y = std::uint64_t(b);
    if (x == 0) return y;
    if (y == 0) return x;
    const int sh = __builtin_ctzll(x | y);
    x >>= __builtin_ctzll(x);
    do {
        y >>= __builtin_ctzll(y);
        if (x > y) {
            const std::uint64_t t = x;
            x = y;
            y = t;
        }
        y -= x;
    } while (y);
    return u128(x) << sh;
}
BigInt gcd(const BigInt& a, const BigInt& b) { return BigInt::from_parts(gcd_u(a.magnitude(), b.magnitude()), false); }
Rational make_raw(const BigInt& n, const BigInt& d);
}  // namespace

BigInt operator+(const BigInt& a, const BigInt& b) {
    if (a.negative() == b.negative()) {
        const u128 m = a.magnitude() + b.magnitude();
        if (m < a.magnitude()) overflow("dagsched BigInt: 128-bit addition overflow");
        return BigInt::from_parts(m, a.negative());
    }
    if (a.magnitude() >= b.magnitude()) return BigInt::from_parts(a.magnitude() - b.magnitude(), a.negative());
    return BigInt::from_parts(b.magnitude() - a.magnitude(), b.negative());
}
BigInt operator*(const BigInt& a, const BigInt& b) {
    u128 m;
    if (__builtin_mul_overflow(a.magnitude(), b.magnitude(), &m))
        overflow("dagsched BigInt: 128-bit multiplication overflow");
    return BigInt::from_parts(m, a.negative() != b.negative());
}
BigInt operator/(const BigInt& a, const BigInt& b) {  // truncates toward zero
    if (b.magnitude() == 0) overflow("division by zero");
    return BigInt::from_parts(a.magnitude() / b.magnitude(), a.negative() != b.negative());
}
BigInt operator%(const BigInt& a, const BigInt& b) {  // sign of the dividend
    if (b.magnitude() == 0) overflow("division by zero");
    return BigInt::from_parts(a.magnitude() % b.magnitude(), a.negative());
}

std::string BigInt::str() const {
    if (mag_ == 0) return "0";
    u128 m = mag_;
    std::string s;
    while (m) {
        s.insert(s.begin(), char('0' + int(m % 10)));
        m /= 10;
    }
    return neg_ ? "-" + s : s;
}

void Rational::set(BigInt n, BigInt d) {
    if (d == 0) overflow("division by zero");
    if (d < 0) {
        n = -n;
        d = -d;
    }
    if (n == 0) {
        n_ = 0;
        d_ = 1;
        return;
    }
    const BigInt g = gcd(n, d);
    n_ = n / g;
    d_ = d / g;
}

std::string Rational::str() const { return format_exact(*this); }

namespace {
Rational make_raw(const BigInt& n, const BigInt& d) { return Rational(n, d); }
}  // namespace

// Boost.Rational's algorithms: g = gcd(d1, d2); n = n1*(d2/g) + n2*(d1/g);
// g2 = gcd(n, g); (n/g2) / ((d1/g) * (d2/g2)) — the same intermediates, so a
// 128-bit overflow happens where the reference's checked backend throws
Rational operator+(const Rational& a, const Rational& b) {
    const BigInt g = gcd(a.den(), b.den());
    const BigInt ad = a.den() / g, bd = b.den() / g;
    const BigInt n = a.num() * bd + b.num() * ad;
    if (n == 0) return Rational();
    const BigInt g2 = gcd(n, g);
    return make_raw(n / g2, ad * (b.den() / g2));
}
Rational operator-(const Rational& a, const Rational& b) { return a + (-b); }
Rational operator*(const Rational& a, const Rational& b) {
    if (a.num() == 0 || b.num() == 0) return Rational();
    const BigInt g1 = gcd(a.num(), b.den());
    const BigInt g2 = gcd(b.num(), a.den());
    return make_raw((a.num() / g1) * (b.num() / g2), (a.den() / g2) * (b.den() / g1));
}
Rational operator/(const Rational& a, const Rational& b) {
    if (b.num() == 0) overflow("division by zero");
    if (a.num() == 0) return Rational();
    const BigInt g1 = gcd(a.num(), b.num());
    const BigInt g2 = gcd(b.den(), a.den());
    return make_raw((a.num() / g1) * (b.den() / g2), (a.den() / g2) * (b.num() / g1));
}

int compare(const Rational& a, const Rational& b) {
    const bool an = a.num().negative(), bn = b.num().negative();
    if (an != bn) return an ? -1 : 1;
    // exact on magnitudes without wide products: integer parts first, then
    // the reciprocals of the fractional parts (ra/ad < rb/bd <=> bd/rb < ad/ra)
    u128 xn = a.num().magnitude(), xd = a.den().magnitude(), yn = b.num().magnitude(), yd = b.den().magnitude();
    int sign = an ? -1 : 1;
    for (;;) {
        const u128 qx = xn / xd, rx = xn % xd, qy = yn / yd, ry = yn % yd;
        if (qx != qy) return qx < qy ? -sign : sign;
        if (rx == 0 || ry == 0) return (rx == 0 && ry == 0) ? 0 : (rx == 0 ? -sign : sign);
        // rx/xd < ry/yd  <=>  xd/rx > yd/ry: recurse on the reciprocals, order flipped
        xn = xd, xd = rx, yn = yd, yd = ry;
        sign = -sign;
    }
}

std::optional<Rational> parse_rational(std::string_view t) {
    auto digits = [](std::string_view s) {
        if (s.empty()) return false;
        for (char c : s)
            if (!std::isdigit(static_cast<unsigned char>(c))) return false;
        return true;
    };
    auto value = [](std::string_view s) {
        BigInt v = 0;
        for (char c : s) v = v * 10 + (c - '0');
        return v;
    };
    if (t.empty()) return std::nullopt;
    bool neg = false;
    if (t[0] == '+' || t[0] == '-') {
        neg = t[0] == '-';
        t.remove_prefix(1);
    }
    if (t.empty()) return std::nullopt;
    Rational r;
    if (auto s = t.find('/'); s != std::string_view::npos) {
        if (!digits(t.substr(0, s)) || !digits(t.substr(s + 1))) return std::nullopt;
        const BigInt d = value(t.substr(s + 1));
        if (d == 0) return std::nullopt;
        r = Rational(value(t.substr(0, s)), d);
    } else {
        std::string_view ip = t, fp;
        if (auto p = t.find('.'); p != std::string_view::npos) {
            ip = t.substr(0, p);
            fp = t.substr(p + 1);
            if (!digits(fp)) return std::nullopt;
        }
        if (!ip.empty() && !digits(ip)) return std::nullopt;
        if (ip.empty() && fp.empty()) return std::nullopt;
        r = Rational(ip.empty() ? BigInt(0) : value(ip), 1);
        if (!fp.empty()) {
            BigInt scale = 1;
            for (std::size_t i = 0; i < fp.size(); ++i) scale *= 10;
            r += Rational(value(fp), scale);
        }
    }
    return neg ? -r : r;
}

BigInt floor_to_int(const Rational& r) {
    BigInt q = r.num() / r.den();
    if (r.num() < 0 && q * r.den() != r.num()) --q;
    return q;
}
BigInt ceil_to_int(const Rational& r) {
    BigInt q = r.num() / r.den();
    if (r.num() > 0 && q * r.den() != r.num()) ++q;
    return q;
}
long long to_int64(const BigInt& v) { return v.convert_to<long long>(); }
double to_double(const Rational& r) { return r.convert_to<double>(); }

std::string format_exact(const Rational& r) {
    return r.den() == 1 ? r.num().str() : r.num().str() + "/" + r.den().str();
}

std::string format_fixed(const Rational& r, int digits) {
    BigInt scale = 1;
    for (int i = 0; i < digits; ++i) scale *= 10;
    const Rational s = r * Rational(scale, 1);
    BigInt whole = s.num() / s.den();
    BigInt rem = s.num() - whole * s.den();
    if (rem < 0) rem = -rem;
    if (rem * 2 >= s.den()) whole += (s.num() < 0) ? -1 : 1;
    const bool neg = whole < 0;
    if (neg) whole = -whole;
    std::string units = (whole / scale).str(), frac = (whole % scale).str();
    if (digits == 0) return (neg ? "-" : "") + units;
    frac.insert(frac.begin(), digits - frac.size(), '0');
    return (neg ? "-" : "") + units + "." + frac;
}

}  // namespace dagsched
