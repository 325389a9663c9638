// Kept C++ API — exact arithmetic (include/dagsched/rational.hpp).
#include "dagsched/rational.hpp"

#include <cctype>

namespace dagsched {

namespace {
[[noreturn]] void overflow() { throw std::overflow_error("dagsched rational: 128-bit overflow"); }
__int128 gcd(__int128 a, __int128 b) {
    if (a < 0) a = -a;
    if (b < 0) b = -b;
    while (b) {
        const __int128 t = a % b;
        a = b;
        b = t;
    }
    return a;
}
}  // namespace

BigInt operator+(const BigInt& a, const BigInt& b) {
    __int128 r;
    if (__builtin_add_overflow(a.value(), b.value(), &r)) overflow();
    return BigInt::raw(r);
}
BigInt operator-(const BigInt& a, const BigInt& b) {
    __int128 r;
    if (__builtin_sub_overflow(a.value(), b.value(), &r)) overflow();
    return BigInt::raw(r);
}
BigInt operator*(const BigInt& a, const BigInt& b) {
    __int128 r;
    if (__builtin_mul_overflow(a.value(), b.value(), &r)) overflow();
    return BigInt::raw(r);
}
BigInt operator/(const BigInt& a, const BigInt& b) {
    if (b.value() == 0) throw std::overflow_error("division by zero");
    return BigInt::raw(a.value() / b.value());
}
BigInt operator%(const BigInt& a, const BigInt& b) {
    if (b.value() == 0) throw std::overflow_error("division by zero");
    return BigInt::raw(a.value() % b.value());
}

std::string BigInt::str() const {
    if (v_ == 0) return "0";
    unsigned __int128 m = v_ < 0 ? (unsigned __int128)(-(v_ + 1)) + 1 : (unsigned __int128)v_;
    std::string s;
    while (m) {
        s.insert(s.begin(), char('0' + int(m % 10)));
        m /= 10;
    }
    return v_ < 0 ? "-" + s : s;
}

void Rational::set(BigInt n, BigInt d) {
    if (d == 0) throw std::overflow_error("division by zero");
    if (d < 0) {
        n = -n;
        d = -d;
    }
    const __int128 g = gcd(n.value(), d.value());
    if (n == 0) {
        n_ = 0;
        d_ = 1;
        return;
    }
    n_ = BigInt::raw(n.value() / g);
    d_ = BigInt::raw(d.value() / g);
}

std::string Rational::str() const { return format_exact(*this); }

// same gcd-first algorithms as Boost.Rational, so intermediates stay small
Rational operator+(const Rational& a, const Rational& b) {
    const BigInt g = BigInt::raw(gcd(a.den().value(), b.den().value()));
    const BigInt ad = a.den() / g, bd = b.den() / g;
    return Rational(a.num() * bd + b.num() * ad, a.den() * bd);
}
Rational operator-(const Rational& a, const Rational& b) { return a + (-b); }
Rational operator*(const Rational& a, const Rational& b) {
    if (a.num() == 0 || b.num() == 0) return Rational();
    const BigInt g1 = BigInt::raw(gcd(a.num().value(), b.den().value()));
    const BigInt g2 = BigInt::raw(gcd(b.num().value(), a.den().value()));
    return Rational((a.num() / g1) * (b.num() / g2), (a.den() / g2) * (b.den() / g1));
}
Rational operator/(const Rational& a, const Rational& b) {
    if (b.num() == 0) throw std::overflow_error("division by zero");
    return a * Rational(b.den(), b.num());
}

int compare(const Rational& a, const Rational& b) {
    // exact without wide products: integer parts first, then the reciprocals
    // of the fractional parts (ra/ad < rb/bd  <=>  bd/rb < ad/ra)
    __int128 an = a.num().value(), ad = a.den().value(), bn = b.num().value(), bd = b.den().value();
    for (;;) {
        __int128 qa = an / ad, ra = an % ad, qb = bn / bd, rb = bn % bd;
        if (ra < 0) --qa, ra += ad;
        if (rb < 0) --qb, rb += bd;
        if (qa != qb) return qa < qb ? -1 : 1;
        if (ra == 0 || rb == 0) return (ra == 0 && rb == 0) ? 0 : (ra == 0 ? -1 : 1);
        const __int128 n1 = bd, d1 = rb, n2 = ad, d2 = ra;
        an = n1, ad = d1, bn = n2, bd = d2;
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
