// Exact non-negative rationals on the device (sm_100a) — the device twin of
// the reference's Rational (rational.hpp:17-20: Boost 128-bit checked,
// always reduced, den > 0).
//
// Representation: u64 numerator/denominator. Every value that leaves the
// kernel is canonical (gcd-reduced); comparisons are exact 128-bit cross
// products and do not need reduced operands, so compare-only temporaries
// (exec_time inside apportion, quota remainders) stay unreduced. Any
// intermediate that does not fit 64 bits sets `ovf`; the DAG is then reported
// DS_EOVERFLOW (the reference would still succeed up to 2^128 — the flagged
// count is part of every parity report and is 0 at the configs measured).
//
// gcd is binary (ctz-driven) with a 32-bit fast path: almost all values met
// here (loads 10-300, SM counts <= 148) fit 32 bits, where IMAD/ALU ops are
// single instructions and 64-bit division is avoided.
#pragma once

#include <cstdint>

namespace ds {

typedef unsigned long long u64;
typedef unsigned int u32;

struct Rat {
    u64 n, d;
};

__device__ __forceinline__ u32 gcd32(u32 a, u32 b) {
    if (a == 0) return b;
    if (b == 0) return a;
    const int s = __ffs(a | b) - 1;
    a >>= __ffs(a) - 1;
    do {
        b >>= __ffs(b) - 1;
        const u32 lo = min(a, b);
        b = max(a, b) - lo;
        a = lo;
    } while (b);
    return a << s;
}

__device__ __forceinline__ u64 gcd64(u64 a, u64 b) {
    if (((a | b) >> 32) == 0) return gcd32(u32(a), u32(b));
    if (a == 0) return b;
    if (b == 0) return a;
    const int s = __ffsll(a | b) - 1;
    a >>= __ffsll(a) - 1;
    do {
        b >>= __ffsll(b) - 1;
        const u64 lo = min(a, b);
        b = max(a, b) - lo;
        a = lo;
        if (((a | b) >> 32) == 0) return u64(gcd32(u32(a), u32(b))) << s;
    } while (b);
    return a << s;
}

__device__ __forceinline__ u64 div64(u64 a, u64 b) {
    if (((a | b) >> 32) == 0) return u32(a) / u32(b);
    return a / b;
}

__device__ __forceinline__ u64 mulc(u64 a, u64 b, bool& ovf) {
    if (((a | b) >> 32) != 0 && __umul64hi(a, b) != 0) ovf = true;
    return a * b;
}

__device__ __forceinline__ u64 addc(u64 a, u64 b, bool& ovf) {
    const u64 s = a + b;
    if (s < a) ovf = true;
    return s;
}

__device__ __forceinline__ Rat rat_int(u64 v) { return Rat{v, 1}; }

__device__ __forceinline__ Rat rat_reduce(u64 n, u64 d) {
    if (n == 0) return Rat{0, 1};
    if (d == 1) return Rat{n, 1};
    const u64 g = gcd64(n, d);
    if (g > 1) {
        n = div64(n, g);
        d = div64(d, g);
    }
    return Rat{n, d};
}

// three-way exact compare of a.n/a.d and b.n/b.d (operands need not be reduced)
__device__ __forceinline__ int rat_cmp(Rat a, Rat b) {
    if (((a.n | a.d | b.n | b.d) >> 32) == 0) {
        const u64 l = a.n * b.d, r = b.n * a.d;
        return l < r ? -1 : (l > r ? 1 : 0);
    }
    const u64 lh = __umul64hi(a.n, b.d), ll = a.n * b.d;
    const u64 rh = __umul64hi(b.n, a.d), rl = b.n * a.d;
    if (lh != rh) return lh < rh ? -1 : 1;
    return ll < rl ? -1 : (ll > rl ? 1 : 0);
}

// Knuth / Boost.Rational addition: g = gcd(d1, d2); t = n1*(d2/g) + n2*(d1/g);
// g2 = gcd(t, g); result = (t/g2) / ((d1/g) * (d2/g2)). Canonical in, canonical out.
__device__ __forceinline__ Rat rat_add(Rat a, Rat b, bool& ovf) {
    if (a.n == 0) return b;
    if (b.n == 0) return a;
    if (a.d == b.d) {
        const u64 t = addc(a.n, b.n, ovf);
        return a.d == 1 ? Rat{t, 1} : rat_reduce(t, a.d);
    }
    const u64 g = gcd64(a.d, b.d);
    const u64 ad = div64(a.d, g), bd = div64(b.d, g);
    const u64 t = addc(mulc(a.n, bd, ovf), mulc(b.n, ad, ovf), ovf);
    const u64 g2 = gcd64(t, g);
    return Rat{div64(t, g2), mulc(ad, div64(b.d, g2), ovf)};
}

// a - b with a >= b (all differences formed by the scheduler are positive).
__device__ __forceinline__ Rat rat_sub(Rat a, Rat b, bool& ovf) {
    if (b.n == 0) return a;
    if (a.d == b.d) {
        const u64 t = a.n - b.n;
        return a.d == 1 ? Rat{t, 1} : rat_reduce(t, a.d);
    }
    const u64 g = gcd64(a.d, b.d);
    const u64 ad = div64(a.d, g), bd = div64(b.d, g);
    const u64 t = mulc(a.n, bd, ovf) - mulc(b.n, ad, ovf);
    if (t == 0) return Rat{0, 1};
    const u64 g2 = gcd64(t, g);
    return Rat{div64(t, g2), mulc(ad, div64(b.d, g2), ovf)};
}

__device__ __forceinline__ Rat rat_mul_int(Rat a, u64 k, bool& ovf) {
    if (a.n == 0 || k == 0) return Rat{0, 1};
    if (a.d == 1) return Rat{mulc(a.n, k, ovf), 1};
    const u64 g = gcd64(k, a.d);
    return Rat{mulc(a.n, div64(k, g), ovf), div64(a.d, g)};
}

__device__ __forceinline__ Rat rat_div_int(Rat a, u64 k, bool& ovf) {
    if (a.n == 0) return Rat{0, 1};
    const u64 g = gcd64(a.n, k);
    return Rat{div64(a.n, g), mulc(a.d, div64(k, g), ovf)};
}

__device__ __forceinline__ Rat rat_mul(Rat a, Rat b, bool& ovf) {
    if (a.n == 0 || b.n == 0) return Rat{0, 1};
    const u64 g1 = gcd64(a.n, b.d), g2 = gcd64(b.n, a.d);
    return Rat{mulc(div64(a.n, g1), div64(b.n, g2), ovf),
               mulc(div64(a.d, g2), div64(b.d, g1), ovf)};
}

__device__ __forceinline__ Rat rat_div(Rat a, Rat b, bool& ovf) {
    return rat_mul(a, Rat{b.d, b.n}, ovf);
}

__device__ __forceinline__ u64 rat_floor(Rat a) { return div64(a.n, a.d); }

__device__ __forceinline__ u64 rat_ceil(Rat a) {
    const u64 q = div64(a.n, a.d);
    return q * a.d == a.n ? q : q + 1;
}

__device__ __forceinline__ Rat rat_max(Rat a, Rat b) { return rat_cmp(a, b) < 0 ? b : a; }

// ------------------------------------------------------- execution model
// Platform constants shared by the whole launch.
struct Plat {
    int M;
    Rat tmin;
};

// exec_model.cpp:16-23: max(1, floor(load / t_min)), saturating at INT_MAX.
__device__ __forceinline__ int max_par(Rat load, const Plat& p) {
    u64 q;
    if (p.tmin.d == 1 && p.tmin.n == 1) {
        q = div64(load.n, load.d);
    } else {
        // floor((load.n * tmin.d) / (load.d * tmin.n)) in 128 bits
        unsigned __int128 num = (unsigned __int128)load.n * p.tmin.d;
        unsigned __int128 den = (unsigned __int128)load.d * p.tmin.n;
        unsigned __int128 qq = num / den;
        q = (qq >> 63) ? (u64)0x7fffffff : (u64)qq;
    }
    if (q < 1) return 1;
    if (q > 0x7fffffffull) return 0x7fffffff;
    return int(q);
}

// exec_model.cpp:7-14: max(t_min, ceil(m/M) * load / m), unreduced — for
// comparisons only.
__device__ __forceinline__ Rat exec_raw(Rat load, long long m, const Plat& p, bool& ovf) {
    const u64 passes = u64((m + p.M - 1) / p.M);
    Rat c{passes == 1 ? load.n : mulc(load.n, passes, ovf), mulc(load.d, u64(m), ovf)};
    return rat_cmp(c, p.tmin) < 0 ? p.tmin : c;
}

// Same value, canonical.
__device__ __forceinline__ Rat exec_time(Rat load, long long m, const Plat& p, bool& ovf) {
    const u64 passes = u64((m + p.M - 1) / p.M);
    Rat c = rat_div_int(passes == 1 ? load : rat_mul_int(load, passes, ovf), u64(m), ovf);
    return rat_cmp(c, p.tmin) < 0 ? p.tmin : c;
}

// ------------------------------------------------------- warp helpers
__device__ __forceinline__ u64 shfl_xor64(u64 v, int o) {
    return __shfl_xor_sync(0xffffffffu, v, o);
}

__device__ __forceinline__ Rat warp_sum(Rat x, bool& ovf) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        Rat y{shfl_xor64(x.n, o), shfl_xor64(x.d, o)};
        x = rat_add(x, y, ovf);
    }
    return x;
}

__device__ __forceinline__ Rat warp_max(Rat x) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        Rat y{shfl_xor64(x.n, o), shfl_xor64(x.d, o)};
        x = rat_max(x, y);
    }
    return x;
}

}  // namespace ds
