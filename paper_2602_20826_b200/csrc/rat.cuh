// Exact non-negative rationals on the device (sm_100a) — the device twin of
// the reference's Rational (rational.hpp:17-20: Boost 128-bit checked,
// always reduced, den > 0).
//
// Two word widths, same algorithms:
//   RatT<u64>   the fast path every DAG takes first;
//   RatT<u128>  the re-run for the (rare) DAGs whose u64 pass overflowed, so
//               results stay exact wherever the reference's 128-bit range
//               holds them.
// Values leaving the kernel are canonical (gcd-reduced). Comparisons are exact
// cross products (128-bit for u64 words, 256-bit for u128 words) and do not
// need reduced operands, so compare-only temporaries (exec_time inside
// apportion, quota remainders) stay unreduced. Any intermediate that does not
// fit the word sets `ovf`.
//
// gcd is binary (ctz-driven) with a 32-bit fast path: nearly all values met
// here (loads 10-300, SM counts <= 148) fit 32 bits, where ALU ops are single
// instructions and 64-bit division is avoided.
#pragma once

#include <cstdint>

namespace ds {

typedef unsigned long long u64;
typedef unsigned int u32;
typedef unsigned __int128 u128;

template <class T>
struct RatT {
    T n, d;
};
typedef RatT<u64> Rat;

// ------------------------------------------------------------ word helpers
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

// 32-bit words: the tier every DAG takes first (all C5 values fit).
__device__ __forceinline__ u32 gcdw(u32 a, u32 b) { return gcd32(a, b); }
__device__ __forceinline__ u32 divw(u32 a, u32 b) { return a / b; }
__device__ __forceinline__ u32 mulc(u32 a, u32 b, bool& ovf) {
    const u64 p = u64(a) * b;
    if (p >> 32) ovf = true;
    return u32(p);
}
__device__ __forceinline__ int cmp_prod(u32 a, u32 b, u32 c, u32 d) {
    const u64 l = u64(a) * b, r = u64(c) * d;
    return l < r ? -1 : (l > r ? 1 : 0);
}
__device__ __forceinline__ u32 shfl_xor_w(u32 v, int o) { return __shfl_xor_sync(0xffffffffu, v, o); }

__device__ __forceinline__ u64 gcdw(u64 a, u64 b) {
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

__device__ __forceinline__ int ctz128(u128 x) {
    const u64 lo = u64(x);
    return lo ? __ffsll(lo) - 1 : 64 + __ffsll(u64(x >> 64)) - 1;
}

__device__ __forceinline__ u128 gcdw(u128 a, u128 b) {
    if (((a | b) >> 64) == 0) return gcdw(u64(a), u64(b));
    if (a == 0) return b;
    if (b == 0) return a;
    const int s = ctz128(a | b);
    a >>= ctz128(a);
    do {
        b >>= ctz128(b);
        if (a > b) {
            const u128 t = a;
            a = b;
            b = t;
        }
        b -= a;
        if (((a | b) >> 64) == 0) return u128(gcdw(u64(a), u64(b))) << s;
    } while (b);
    return a << s;
}

__device__ __forceinline__ u64 divw(u64 a, u64 b) {
    if (((a | b) >> 32) == 0) return u32(a) / u32(b);
    return a / b;
}
__device__ __forceinline__ u128 divw(u128 a, u128 b) {
    if (((a | b) >> 64) == 0) return divw(u64(a), u64(b));
    return a / b;
}

__device__ __forceinline__ u64 mulc(u64 a, u64 b, bool& ovf) {
    if (((a | b) >> 32) != 0 && __umul64hi(a, b) != 0) ovf = true;
    return a * b;
}
__device__ __forceinline__ u128 mulc(u128 a, u128 b, bool& ovf) {
    const u64 ah = u64(a >> 64), bh = u64(b >> 64), al = u64(a), bl = u64(b);
    if (ah == 0 && bh == 0) return u128(al) * bl;
    if (ah != 0 && bh != 0) {
        ovf = true;
        return 0;
    }
    // one operand has a high word: cross = hi * lo must fit 64 bits
    const u64 h = ah ? ah : bh, l = ah ? bl : al;
    const u128 cross = u128(h) * l;
    const u128 low = u128(al) * bl;
    if ((cross >> 64) != 0) ovf = true;
    const u128 r = low + (cross << 64);
    if (r < low) ovf = true;
    return r;
}

template <class T>
__device__ __forceinline__ T addc(T a, T b, bool& ovf) {
    const T s = a + b;
    if (s < a) ovf = true;
    return s;
}

// exact three-way compare of products a*b and c*d
__device__ __forceinline__ int cmp_prod(u64 a, u64 b, u64 c, u64 d) {
    if (((a | b | c | d) >> 32) == 0) {
        const u64 l = a * b, r = c * d;
        return l < r ? -1 : (l > r ? 1 : 0);
    }
    const u64 lh = __umul64hi(a, b), ll = a * b;
    const u64 rh = __umul64hi(c, d), rl = c * d;
    if (lh != rh) return lh < rh ? -1 : 1;
    return ll < rl ? -1 : (ll > rl ? 1 : 0);
}

__device__ __forceinline__ void mul_wide(u128 a, u128 b, u128& hi, u128& lo) {
    const u128 m = (u128(1) << 64) - 1;
    const u128 a0 = a & m, a1 = a >> 64, b0 = b & m, b1 = b >> 64;
    const u128 p00 = a0 * b0, p01 = a0 * b1, p10 = a1 * b0, p11 = a1 * b1;
    const u128 mid = (p00 >> 64) + (p01 & m) + (p10 & m);
    lo = (p00 & m) | (mid << 64);
    hi = p11 + (p01 >> 64) + (p10 >> 64) + (mid >> 64);
}

__device__ __forceinline__ int cmp_prod(u128 a, u128 b, u128 c, u128 d) {
    if (((a | b | c | d) >> 64) == 0) return cmp_prod(u64(a), u64(b), u64(c), u64(d));
    u128 h1, l1, h2, l2;
    mul_wide(a, b, h1, l1);
    mul_wide(c, d, h2, l2);
    if (h1 != h2) return h1 < h2 ? -1 : 1;
    return l1 < l2 ? -1 : (l1 > l2 ? 1 : 0);
}

// ------------------------------------------------------------ rationals
template <class T>
__device__ __forceinline__ RatT<T> rat_reduce(T n, T d) {
    if (n == 0) return RatT<T>{0, 1};
    if (d == 1) return RatT<T>{n, 1};
    const T g = gcdw(n, d);
    if (g > 1) {
        n = divw(n, g);
        d = divw(d, g);
    }
    return RatT<T>{n, d};
}

template <class T>
__device__ __forceinline__ int rat_cmp(RatT<T> a, RatT<T> b) {
    return cmp_prod(a.n, b.d, b.n, a.d);
}

// Knuth / Boost.Rational addition: g = gcd(d1, d2); t = n1*(d2/g) + n2*(d1/g);
// g2 = gcd(t, g); result = (t/g2) / ((d1/g) * (d2/g2)). Canonical in/out.
template <class T>
__device__ __forceinline__ RatT<T> rat_add(RatT<T> a, RatT<T> b, bool& ovf) {
    if (a.n == 0) return b;
    if (b.n == 0) return a;
    if (a.d == b.d) {
        const T t = addc(a.n, b.n, ovf);
        return a.d == 1 ? RatT<T>{t, 1} : rat_reduce(t, a.d);
    }
    const T g = gcdw(a.d, b.d);
    const T ad = divw(a.d, g), bd = divw(b.d, g);
    const T t = addc(mulc(a.n, bd, ovf), mulc(b.n, ad, ovf), ovf);
    const T g2 = gcdw(t, g);
    return RatT<T>{divw(t, g2), mulc(ad, divw(b.d, g2), ovf)};
}

// a - b with a >= b (all differences formed by the scheduler are positive)
template <class T>
__device__ __forceinline__ RatT<T> rat_sub(RatT<T> a, RatT<T> b, bool& ovf) {
    if (b.n == 0) return a;
    if (a.d == b.d) {
        const T t = a.n - b.n;
        return a.d == 1 ? RatT<T>{t, 1} : rat_reduce(t, a.d);
    }
    const T g = gcdw(a.d, b.d);
    const T ad = divw(a.d, g), bd = divw(b.d, g);
    const T t = mulc(a.n, bd, ovf) - mulc(b.n, ad, ovf);
    if (t == 0) return RatT<T>{0, 1};
    const T g2 = gcdw(t, g);
    return RatT<T>{divw(t, g2), mulc(ad, divw(b.d, g2), ovf)};
}

template <class T>
__device__ __forceinline__ RatT<T> rat_mul_int(RatT<T> a, T k, bool& ovf) {
    if (a.n == 0 || k == 0) return RatT<T>{0, 1};
    if (a.d == 1) return RatT<T>{mulc(a.n, k, ovf), 1};
    const T g = gcdw(k, a.d);
    return RatT<T>{mulc(a.n, divw(k, g), ovf), divw(a.d, g)};
}

template <class T>
__device__ __forceinline__ RatT<T> rat_div_int(RatT<T> a, T k, bool& ovf) {
    if (a.n == 0) return RatT<T>{0, 1};
    const T g = gcdw(a.n, k);
    return RatT<T>{divw(a.n, g), mulc(a.d, divw(k, g), ovf)};
}

template <class T>
__device__ __forceinline__ RatT<T> rat_mul(RatT<T> a, RatT<T> b, bool& ovf) {
    if (a.n == 0 || b.n == 0) return RatT<T>{0, 1};
    const T g1 = gcdw(a.n, b.d), g2 = gcdw(b.n, a.d);
    return RatT<T>{mulc(divw(a.n, g1), divw(b.n, g2), ovf), mulc(divw(a.d, g2), divw(b.d, g1), ovf)};
}

template <class T>
__device__ __forceinline__ RatT<T> rat_div(RatT<T> a, RatT<T> b, bool& ovf) {
    return rat_mul(a, RatT<T>{b.d, b.n}, ovf);
}

template <class T>
__device__ __forceinline__ T rat_ceil(RatT<T> a) {
    const T q = divw(a.n, a.d);
    return q * a.d == a.n ? q : q + 1;
}

template <class T>
__device__ __forceinline__ RatT<T> rat_max(RatT<T> a, RatT<T> b) {
    return rat_cmp(a, b) < 0 ? b : a;
}

// ------------------------------------------------------- execution model
template <class T>
struct PlatT {
    int M;
    RatT<T> tmin;
    int minl;  // DagTask::make's load floor: 0 t_min, 1 one, 2 positive only (ds_platform.flags)
};

// exec_model.cpp:16-23: max(1, floor(load / t_min)), saturating at INT_MAX.
template <class T>
__device__ __forceinline__ int max_par(RatT<T> load, const PlatT<T>& p, bool& ovf) {
    T q;
    if (p.tmin.d == 1 && p.tmin.n == 1) {
        q = load.d == 1 ? load.n : divw(load.n, load.d);
    } else {
        bool o = false;
        const T num = mulc(load.n, p.tmin.d, o), den = mulc(load.d, p.tmin.n, o);
        if (o) {
            ovf = true;
            return 1;
        }
        q = divw(num, den);
    }
    if (q < 1) return 1;
    if (q > T(0x7fffffff)) return 0x7fffffff;
    return int(q);
}

// exec_model.cpp:7-14: max(t_min, ceil(m/M) * load / m), unreduced — for
// comparisons only.
template <class T>
__device__ __forceinline__ RatT<T> exec_raw(RatT<T> load, long long m, const PlatT<T>& p, bool& ovf) {
    // ceil(m / M); m <= M (one pass) is the common case and skips the 64-bit divide
    const T passes = m <= p.M ? T(1) : T((m + p.M - 1) / p.M);
    RatT<T> c{passes == 1 ? load.n : mulc(load.n, passes, ovf), mulc(load.d, T(m), ovf)};
    return rat_cmp(c, p.tmin) < 0 ? p.tmin : c;
}

// Same value, canonical. The clamp is decided on the unreduced value first:
// a kernel at (or beyond) its useful parallelism runs in exactly t_min, which
// is the common case at M = 148, and then no gcd/division is needed at all.
template <class T>
__device__ __forceinline__ RatT<T> exec_time(RatT<T> load, long long m, const PlatT<T>& p, bool& ovf) {
    // ceil(m / M); m <= M (one pass) is the common case and skips the 64-bit divide
    const T passes = m <= p.M ? T(1) : T((m + p.M - 1) / p.M);
    bool o = false;
    const RatT<T> raw{passes == 1 ? load.n : mulc(load.n, passes, o), mulc(load.d, T(m), o)};
    if (!o && rat_cmp(raw, p.tmin) <= 0) return p.tmin;
    RatT<T> c = rat_div_int(passes == 1 ? load : rat_mul_int(load, passes, ovf), T(m), ovf);
    return rat_cmp(c, p.tmin) < 0 ? p.tmin : c;
}

// ------------------------------------------------------- warp helpers
__device__ __forceinline__ u64 shfl_xor_w(u64 v, int o) { return __shfl_xor_sync(0xffffffffu, v, o); }
__device__ __forceinline__ u128 shfl_xor_w(u128 v, int o) {
    const u64 lo = __shfl_xor_sync(0xffffffffu, u64(v), o);
    const u64 hi = __shfl_xor_sync(0xffffffffu, u64(v >> 64), o);
    return (u128(hi) << 64) | lo;
}

template <class T>
__device__ __forceinline__ RatT<T> warp_sum(RatT<T> x, bool& ovf) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const RatT<T> y{shfl_xor_w(x.n, o), shfl_xor_w(x.d, o)};
        x = rat_add(x, y, ovf);
    }
    return x;
}

template <class T>
__device__ __forceinline__ RatT<T> warp_max(RatT<T> x) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const RatT<T> y{shfl_xor_w(x.n, o), shfl_xor_w(x.d, o)};
        x = rat_max(x, y);
    }
    return x;
}

}  // namespace ds

namespace ds {
// ------------------------------------------------------------------------
// Out-of-line entry points. The analysis kernel is latency bound with many
// call sites per rational op; inlining every site blew the W=1 kernel up to
// 32.5k SASS instructions (~520 KB) and made it I-cache bound (ncu: 86% of
// stall samples "no_instructions", profiles/r01_k1_v1_summary.json). These
// wrappers keep one copy of each op. Overflow is reported in-band as den == 0
// so no flag has to live in local memory across the call.
template <class T>
__device__ __noinline__ RatT<T> n_add(RatT<T> a, RatT<T> b) {
    bool o = false;
    RatT<T> r = rat_add(a, b, o);
    if (o || a.d == 0 || b.d == 0) r.d = 0;
    return r;
}
template <class T>
__device__ __noinline__ RatT<T> n_sub(RatT<T> a, RatT<T> b) {
    bool o = false;
    RatT<T> r = rat_sub(a, b, o);
    if (o || a.d == 0 || b.d == 0) r.d = 0;
    return r;
}
template <class T>
__device__ __noinline__ RatT<T> n_mul_int(RatT<T> a, T k) {
    bool o = false;
    RatT<T> r = rat_mul_int(a, k, o);
    if (o || a.d == 0) r.d = 0;
    return r;
}
template <class T>
__device__ __noinline__ RatT<T> n_div_int(RatT<T> a, T k) {
    bool o = false;
    RatT<T> r = rat_div_int(a, k, o);
    if (o || a.d == 0) r.d = 0;
    return r;
}
template <class T>
__device__ __noinline__ RatT<T> n_div(RatT<T> a, RatT<T> b) {
    bool o = false;
    RatT<T> r = rat_div(a, b, o);
    if (o || a.d == 0 || b.d == 0) r.d = 0;
    return r;
}
template <class T>
__device__ __noinline__ RatT<T> n_reduce(T n, T d) {
    return rat_reduce(n, d);
}
template <class T>
__device__ __noinline__ int n_cmp(RatT<T> a, RatT<T> b) {
    return rat_cmp(a, b);
}
template <class T>
__device__ __noinline__ RatT<T> n_exec(RatT<T> load, long long m, PlatT<T> p) {
    bool o = false;
    RatT<T> r = exec_time(load, m, p, o);
    if (o) r.d = 0;
    return r;
}
template <class T>
__device__ __noinline__ RatT<T> n_exec_raw(RatT<T> load, long long m, PlatT<T> p) {
    bool o = false;
    RatT<T> r = exec_raw(load, m, p, o);
    if (o) r.d = 0;
    return r;
}
template <class T>
__device__ __noinline__ int n_max_par(RatT<T> load, PlatT<T> p) {
    bool o = false;
    const int r = max_par(load, p, o);
    return o ? -1 : r;
}
template <class T>
__device__ __noinline__ T n_ceil(RatT<T> a) {
    return rat_ceil(a);
}
}  // namespace ds

namespace ds {
// Hot-loop helpers: the 32-bit tier's compare / unreduced exec_time are a few
// instructions, cheaper inline than a call; wider tiers keep the single
// out-of-line copy. Integer sums add inline at every width.
template <class T>
__device__ __forceinline__ int q_cmp(RatT<T> a, RatT<T> b) {
    if constexpr (sizeof(T) == 4) return rat_cmp(a, b);
    else return n_cmp(a, b);
}
template <class T>
__device__ __forceinline__ RatT<T> q_exec_raw(RatT<T> load, long long m, const PlatT<T>& p) {
    if constexpr (sizeof(T) == 4) {
        bool o = false;
        RatT<T> r = exec_raw(load, m, p, o);
        if (o) r.d = 0;
        return r;
    } else {
        return n_exec_raw(load, m, p);
    }
}
// t_min = 1 and an integer load (every C5 node): max_parallelism is the load
// itself, and exec_time(load, m) is t_min whenever m >= load (one pass, raw
// value <= 1) — decided inline; anything else goes to the out-of-line copies.
template <class T>
__device__ __forceinline__ bool unit_tmin(const PlatT<T>& p) {
    return p.tmin.n == 1 && p.tmin.d == 1;
}
template <class T>
__device__ __forceinline__ int q_max_par(RatT<T> load, const PlatT<T>& p) {
    if (unit_tmin(p) && load.d == 1 && load.n >= T(1) && load.n <= T(0x7fffffff)) return int(load.n);
    return n_max_par(load, p);
}
template <class T>
__device__ __forceinline__ RatT<T> q_exec(RatT<T> load, int m, const PlatT<T>& p) {
    if (unit_tmin(p) && load.d == 1 && m <= p.M && load.n <= T(m)) return p.tmin;
    return n_exec(load, m, p);
}

template <class T>
__device__ __forceinline__ RatT<T> q_add(RatT<T> a, RatT<T> b) {
    if (a.d == 1 && b.d == 1) {
        const T s = a.n + b.n;
        return RatT<T>{s, T(s < a.n ? 0 : 1)};  // den 0 flags overflow
    }
    return n_add(a, b);
}
}  // namespace ds
