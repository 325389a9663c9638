// Exact-arithmetic edge cases — the SAME source compiles against the
// reference's rational.hpp (oracle/_ref/ref_rational_check: Boost's 128-bit
// checked signed-magnitude cpp_int as restated in oracle/shim) and against
// the kept API (api_rational_check), and the two outputs must be identical
// (tests/test_cpp_api.py). Each line is one operation's result or the
// exception type it raised.
#include "dagsched/rational.hpp"

#include <cstdio>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

using namespace dagsched;

namespace {

void run(const char* what, const std::function<std::string()>& f) {
    std::string out;
    try {
        out = f();
    } catch (const std::overflow_error&) {
        out = "overflow_error";
    } catch (const std::exception& e) {
        out = std::string("exception");
    }
    std::printf("%s: %s\n", what, out.c_str());
}

BigInt pow2(int k) {
    BigInt x = 1;
    for (int i = 0; i < k; ++i) x *= 2;
    return x;
}

}  // namespace

int main() {
    const BigInt p127 = pow2(127);
    const BigInt max128 = (pow2(127) - 1) * 2 + 1;  // 2^128 - 1
    run("2^127", [&] { return p127.str(); });
    run("2^128-1", [&] { return max128.str(); });
    run("-(2^128-1)", [&] { return (-max128).str(); });
    run("2^128 (mul)", [&] { return (p127 * 2).str(); });
    run("2^128 (add)", [&] { return (max128 + 1).str(); });
    run("-(2^128) (sub)", [&] { return (-max128 - 1).str(); });
    run("(2^128-1) - (2^128-1)", [&] { return (max128 - max128).str(); });
    run("2^127 / 3", [&] { return (p127 / 3).str(); });
    run("-(2^127) % 5", [&] { return ((-p127) % 5).str(); });
    run("rat 2^127/3", [&] { return format_exact(Rational(p127, BigInt(3))); });
    run("rat (2^128-1)/(2^127)", [&] { return format_exact(Rational(max128, p127)); });
    run("rat -x/-y", [&] { return format_exact(Rational(-max128, -p127)); });
    run("rat sum near max", [&] {
        return format_exact(Rational(max128, BigInt(7)) + Rational(BigInt(-5), BigInt(7)));
    });
    run("rat sum overflow", [&] { return format_exact(Rational(max128) + Rational(1)); });
    run("rat add gcd path", [&] {
        // denominators sharing a large factor: Boost's g / g2 path keeps this in range
        const BigInt d = pow2(100);
        return format_exact(Rational(BigInt(1), d * 3) + Rational(BigInt(1), d * 5));
    });
    run("rat mul cross-cancel", [&] {
        return format_exact(Rational(max128, p127) * Rational(p127, max128));
    });
    run("rat mul overflow", [&] { return format_exact(Rational(max128, BigInt(3)) * Rational(BigInt(4), BigInt(5))); });
    run("rat div", [&] { return format_exact(Rational(p127, BigInt(9)) / Rational(BigInt(2), BigInt(3))); });
    run("rat div by zero", [&] { return format_exact(Rational(1) / Rational(0)); });
    run("cmp big", [&] {
        const Rational a(max128, p127), b(max128 - 1, p127 - 1);
        return std::to_string(int(a < b)) + std::to_string(int(a > b)) + std::to_string(int(a == b));
    });
    run("cmp neg", [&] {
        const Rational a(-max128, p127), b(BigInt(-3), BigInt(2));
        return std::to_string(int(a < b)) + std::to_string(int(b < a));
    });
    run("floor/ceil neg", [&] {
        const Rational a(BigInt(-7), BigInt(2));
        return floor_to_int(a).str() + " " + ceil_to_int(a).str();
    });
    run("to_int64 sat", [&] { return std::to_string(to_int64(max128)) + " " + std::to_string(to_int64(-max128)); });
    run("to_double", [&] {
        char b[64];
        std::snprintf(b, sizeof b, "%.17g", to_double(Rational(max128, BigInt(3))));
        return std::string(b);
    });
    run("format_fixed", [&] {
        return format_fixed(Rational(BigInt(-2), BigInt(3)), 6) + " " + format_fixed(Rational(BigInt(5), BigInt(2)), 0) +
               " " + format_fixed(Rational(max128, p127), 4);
    });
    run("parse big", [&] {
        auto r = parse_rational("340282366920938463463374607431768211455/2");
        return r ? format_exact(*r) : std::string("nullopt");
    });
    run("parse too big", [&] {
        auto r = parse_rational("340282366920938463463374607431768211456");
        return r ? format_exact(*r) : std::string("nullopt");
    });
    run("parse decimal", [&] {
        auto r = parse_rational("-12.0625");
        return r ? format_exact(*r) : std::string("nullopt");
    });
    return 0;
}
