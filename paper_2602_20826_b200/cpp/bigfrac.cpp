// Internal: unbounded exact fractions (bigfrac.hpp).
#include "bigfrac.hpp"

#include <algorithm>
#include <stdexcept>

namespace dagsched::detail {

using u32 = std::uint32_t;
using u64 = std::uint64_t;
using u128 = unsigned __int128;

BigNat::BigNat(u128 v) {
    while (v) {
        d_.push_back(u32(v));
        v >>= 32;
    }
}

void BigNat::trim() {
    while (!d_.empty() && d_.back() == 0) d_.pop_back();
}

u128 BigNat::to_u128() const {
    u128 v = 0;
    for (std::size_t i = d_.size(); i-- > 0;) v = (v << 32) | d_[i];
    return v;
}

int cmp(const BigNat& a, const BigNat& b) {
    if (a.d_.size() != b.d_.size()) return a.d_.size() < b.d_.size() ? -1 : 1;
    for (std::size_t i = a.d_.size(); i-- > 0;)
        if (a.d_[i] != b.d_[i]) return a.d_[i] < b.d_[i] ? -1 : 1;
    return 0;
}

BigNat operator+(const BigNat& a, const BigNat& b) {
    BigNat r;
    const std::size_t n = std::max(a.d_.size(), b.d_.size());
    r.d_.resize(n + 1);
    u64 c = 0;
    for (std::size_t i = 0; i < n; ++i) {
        c += u64(i < a.d_.size() ? a.d_[i] : 0) + (i < b.d_.size() ? b.d_[i] : 0);
        r.d_[i] = u32(c);
        c >>= 32;
    }
    r.d_[n] = u32(c);
    r.trim();
    return r;
}

BigNat operator-(const BigNat& a, const BigNat& b) {
    BigNat r;
    r.d_.resize(a.d_.size());
    long long br = 0;
    for (std::size_t i = 0; i < a.d_.size(); ++i) {
        long long x = (long long)a.d_[i] - (i < b.d_.size() ? b.d_[i] : 0) - br;
        br = x < 0;
        r.d_[i] = u32(x + (br ? (1LL << 32) : 0));
    }
    r.trim();
    return r;
}

BigNat operator*(const BigNat& a, const BigNat& b) {
    BigNat r;
    if (a.zero() || b.zero()) return r;
    r.d_.assign(a.d_.size() + b.d_.size(), 0);
    for (std::size_t i = 0; i < a.d_.size(); ++i) {
        u64 c = 0;
        for (std::size_t j = 0; j < b.d_.size(); ++j) {
            const u64 t = u64(a.d_[i]) * b.d_[j] + r.d_[i + j] + c;
            r.d_[i + j] = u32(t);
            c = t >> 32;
        }
        r.d_[i + b.d_.size()] = u32(c);
    }
    r.trim();
    return r;
}

// Knuth, TAOCP vol. 2, 4.3.1 Algorithm D (base 2^32)
void BigNat::divmod(const BigNat& a, const BigNat& b, BigNat& q, BigNat& r) {
    if (b.zero()) throw std::overflow_error("division by zero");
    if (cmp(a, b) < 0) {
        q = BigNat();
        r = a;
        return;
    }
    if (b.d_.size() == 1) {
        q.d_.assign(a.d_.size(), 0);
        u64 rem = 0;
        for (std::size_t i = a.d_.size(); i-- > 0;) {
            const u64 cur = (rem << 32) | a.d_[i];
            q.d_[i] = u32(cur / b.d_[0]);
            rem = cur % b.d_[0];
        }
        q.trim();
        r = BigNat(rem);
        return;
    }
    const int s = __builtin_clz(b.d_.back());
    const std::size_t n = b.d_.size(), m = a.d_.size() - n;
    std::vector<u32> v(n), u(a.d_.size() + 1);
    for (std::size_t i = n; i-- > 0;) v[i] = (b.d_[i] << s) | (s && i ? u32(u64(b.d_[i - 1]) >> (32 - s)) : 0);
    u[a.d_.size()] = s ? u32(u64(a.d_.back()) >> (32 - s)) : 0;
    for (std::size_t i = a.d_.size(); i-- > 0;) u[i] = (a.d_[i] << s) | (s && i ? u32(u64(a.d_[i - 1]) >> (32 - s)) : 0);
    q.d_.assign(m + 1, 0);
    for (std::size_t j = m + 1; j-- > 0;) {
        const u64 num = (u64(u[j + n]) << 32) | u[j + n - 1];
        u64 qh = num / v[n - 1], rh = num % v[n - 1];
        while (qh >= (1ull << 32) || qh * v[n - 2] > ((rh << 32) | u[j + n - 2])) {
            --qh;
            rh += v[n - 1];
            if (rh >= (1ull << 32)) break;
        }
        long long borrow = 0;
        u64 carry = 0;
        for (std::size_t i = 0; i < n; ++i) {
            const u64 p = qh * v[i] + carry;
            carry = p >> 32;
            const long long t = (long long)u[i + j] - borrow - (long long)(p & 0xffffffffu);
            u[i + j] = u32(t);
            borrow = t < 0;
        }
        const long long t = (long long)u[j + n] - borrow - (long long)carry;
        u[j + n] = u32(t);
        if (t < 0) {  // qh one too large: add back
            --qh;
            u64 c = 0;
            for (std::size_t i = 0; i < n; ++i) {
                const u64 x = u64(u[i + j]) + v[i] + c;
                u[i + j] = u32(x);
                c = x >> 32;
            }
            u[j + n] = u32(u64(u[j + n]) + c);
        }
        q.d_[j] = u32(qh);
    }
    q.trim();
    r.d_.assign(n, 0);
    for (std::size_t i = 0; i < n; ++i) r.d_[i] = (u[i] >> s) | (s ? u32(u64(u[i + 1]) << (32 - s)) : 0);
    r.trim();
}

BigNat gcd(BigNat a, BigNat b) {
    while (!b.zero()) {
        BigNat q, r;
        BigNat::divmod(a, b, q, r);
        a = std::move(b);
        b = std::move(r);
    }
    return a;
}

void BigFrac::reduce() {
    if (num_.zero()) {
        den_ = BigNat(1);
        neg_ = false;
        return;
    }
    const BigNat g = gcd(num_, den_);
    BigNat q, r;
    BigNat::divmod(num_, g, q, r);
    num_ = q;
    BigNat::divmod(den_, g, q, r);
    den_ = q;
}

void BigFrac::add(const Rational& x) {
    const BigNat xn(x.num().magnitude()), xd(x.den().magnitude());
    const bool xneg = x.num().negative();
    // num/den + xn/xd = (num*xd +- xn*den) / (den*xd)
    const BigNat a = num_ * xd, b = xn * den_;
    if (neg_ == xneg) {
        num_ = a + b;
    } else if (cmp(a, b) >= 0) {
        num_ = a - b;
    } else {
        num_ = b - a;
        neg_ = xneg;
    }
    den_ = den_ * xd;
    reduce();
}

void BigFrac::div_int(std::uint64_t n) {
    den_ = den_ * BigNat(n);
    reduce();
}

Rational BigFrac::to_rational() const {
    if (!num_.fits_u128() || !den_.fits_u128()) throw std::overflow_error("mean outside 128-bit rationals");
    return Rational::reduced(BigInt::from_parts(num_.to_u128(), neg_), BigInt::from_parts(den_.to_u128(), false));
}

Rational BigFrac::to_rational_or_truncated(bool& exact) const {
    exact = num_.fits_u128() && den_.fits_u128();
    if (exact) return to_rational();
    u128 scale = 1;
    for (int i = 0; i < 18; ++i) scale *= 10;
    BigNat q, r;
    BigNat::divmod(num_ * BigNat(scale), den_, q, r);
    if (!q.fits_u128()) throw std::overflow_error("mean outside 128-bit rationals");
    return Rational(BigInt::from_parts(q.to_u128(), neg_), BigInt::from_parts(scale, false));
}

}  // namespace dagsched::detail
