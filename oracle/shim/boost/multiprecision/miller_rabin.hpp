#pragma once
// ORACLE TEST INFRASTRUCTURE — not product code.
//
// Stand-in for boost::multiprecision::miller_rabin_test as used by
// field.hpp:37 (`miller_rabin_test(modulus, 32)`). Deterministic variant:
// trial division by small primes, then Miller–Rabin with the first `trials`
// primes as bases (deterministic below 3.3e24, error < 4^-trials above).
// Must reject 91 and 2^128 and accept 97, Goldilocks and BN254 Fr
// (tests/test_field.cpp:15-32).

#include "cpp_int.hpp"

namespace boost {
namespace multiprecision {

inline bool miller_rabin_test(const cpp_int& n, unsigned trials) {
    static const unsigned small_primes[] = {
        2,   3,   5,   7,   11,  13,  17,  19,  23,  29,  31,  37,  41,  43,  47,  53,
        59,  61,  67,  71,  73,  79,  83,  89,  97,  101, 103, 107, 109, 113, 127, 131,
        137, 139, 149, 151, 157, 163, 167, 173, 179, 181, 191, 193, 197, 199, 211, 223};
    if (n < 2) return false;
    for (unsigned p : small_primes) {
        if (n == p) return true;
        if ((n % p).is_zero()) return false;
    }
    const cpp_int nm1 = n - 1;
    cpp_int d = nm1;
    unsigned s = 0;
    while (!bit_test(d, 0)) {
        d = d >> 1;
        ++s;
    }
    const unsigned rounds = trials < 1 ? 1 : (trials > 48 ? 48 : trials);
    for (unsigned i = 0; i < rounds; ++i) {
        const cpp_int a(small_primes[i]);
        cpp_int x = powm(a, d, n);
        if (x == 1 || x == nm1) continue;
        bool composite = true;
        for (unsigned r = 1; r < s; ++r) {
            x = (x * x) % n;
            if (x == nm1) {
                composite = false;
                break;
            }
        }
        if (composite) return false;
    }
    return true;
}

template <class Engine>
bool miller_rabin_test(const cpp_int& n, unsigned trials, Engine&) {
    return miller_rabin_test(n, trials);
}

}  // namespace multiprecision
}  // namespace boost
