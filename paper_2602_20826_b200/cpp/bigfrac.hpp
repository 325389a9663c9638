// Internal: an unbounded exact fraction for run_experiment's corpus means.
//
// The reference sums n per-task ratios in its 128-bit checked Rational and
// throws std::overflow_error once the running sum's denominator outgrows 128
// bits (experiment.cpp:121-133) — at C5-sized corpora (>= ~100 DAGs) it
// does. Here the sum is exact in unbounded integers, so the mean is the same
// value wherever the reference completes and still exists where it would
// not; only a mean that itself needs more than 128 bits raises.
#pragma once

#include "dagsched/rational.hpp"

#include <cstdint>
#include <vector>

namespace dagsched::detail {

class BigNat {  // little-endian base-2^32 magnitude, no leading zero limbs
  public:
    BigNat() = default;
    explicit BigNat(unsigned __int128 v);
    bool zero() const { return d_.empty(); }
    bool fits_u128() const { return d_.size() <= 4; }
    unsigned __int128 to_u128() const;
    friend int cmp(const BigNat& a, const BigNat& b);
    friend BigNat operator+(const BigNat& a, const BigNat& b);
    friend BigNat operator-(const BigNat& a, const BigNat& b);  // a >= b
    friend BigNat operator*(const BigNat& a, const BigNat& b);
    static void divmod(const BigNat& a, const BigNat& b, BigNat& q, BigNat& r);  // b != 0
    friend BigNat gcd(BigNat a, BigNat b);

  private:
    void trim();
    std::vector<std::uint32_t> d_;
};

class BigFrac {
  public:
    BigFrac() : den_(1) {}
    void add(const Rational& q);                   // += q
    void div_int(std::uint64_t n);                 // /= n (n > 0)
    Rational to_rational() const;                  // std::overflow_error if outside 128 bits
    // exact when it fits 128 bits; else truncated toward zero to a multiple
    // of 10^-18. Truncation keeps every half-away-from-zero decimal rounding
    // to <= 18 digits (format_fixed) equal to the exact value's: a rounding
    // boundary is itself a multiple of 10^-18, so the truncated value stays
    // on the exact value's side of it. `exact` reports which.
    Rational to_rational_or_truncated(bool& exact) const;

  private:
    void reduce();
    bool neg_ = false;
    BigNat num_, den_;
};

}  // namespace dagsched::detail
