#pragma once
// ORACLE TEST INFRASTRUCTURE — not product code.
//
// Minimal stand-in for the slice of Boost.Multiprecision `cpp_int` that the
// reference headers use (Boost is not installed in this image). It exists only
// so that the UNMODIFIED reference sources under /root/reference/proj/include
// compile into the checker binaries in oracle/_ref/.
//
// Surface: signed arbitrary-precision integer with
// C++ truncating division semantics (field.hpp:88-89, tests/oracles.hpp:44-45
// rely on negative `%`), shifts, comparisons, decimal string ctor and str(),
// plus the free functions import_bits / export_bits (field.hpp:162,181,
// transcript.hpp:63,92), msb (field.hpp:72), powm (field.hpp:139,
// tests/oracles.hpp:161), bit_test (distinct.hpp:133).
//
// Representation: sign + little-endian 64-bit magnitude limbs in a fixed
// inline buffer (no heap traffic). Capacity 1024 bits: products of two values
// below any supported modulus (<= 512 bits) always fit; overflow throws.

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <iterator>
#include <ostream>
#include <stdexcept>
#include <string>
#include <type_traits>

namespace boost {
namespace multiprecision {

class cpp_int {
public:
    static constexpr int kCap = 16;  // 16 x 64-bit limbs = 1024 bits

    cpp_int() = default;
    cpp_int(const cpp_int& o) : neg_(o.neg_), n_(o.n_) {
        for (int i = 0; i < n_; ++i) d_[i] = o.d_[i];
    }
    cpp_int& operator=(const cpp_int& o) {
        neg_ = o.neg_;
        n_ = o.n_;
        for (int i = 0; i < n_; ++i) d_[i] = o.d_[i];
        return *this;
    }

    template <class I, class = std::enable_if_t<std::is_integral_v<I>>>
    cpp_int(I v) {  // NOLINT: implicit like boost
        if constexpr (std::is_signed_v<I>) {
            if (v < 0) {
                neg_ = true;
                // magnitude of possibly INT_MIN
                d_[0] = static_cast<std::uint64_t>(0) - static_cast<std::uint64_t>(static_cast<long long>(v));
                n_ = 1;
                return;
            }
        }
        if (v != 0) {
            d_[0] = static_cast<std::uint64_t>(v);
            n_ = 1;
        }
    }

    explicit cpp_int(const char* s) { parse(std::string(s)); }
    explicit cpp_int(const std::string& s) { parse(s); }

    std::string str() const {
        if (n_ == 0) return "0";
        cpp_int t = *this;
        t.neg_ = false;
        std::string out;
        const std::uint64_t base = 1000000000000000000ull;  // 1e18
        while (t.n_ != 0) {
            std::uint64_t rem = t.div_small(base);
            char buf[32];
            int len = 0;
            for (int i = 0; i < 18; ++i) {
                buf[len++] = static_cast<char>('0' + rem % 10);
                rem /= 10;
                if (t.n_ == 0 && rem == 0) break;
            }
            out.append(buf, buf + len);
        }
        while (out.size() > 1 && out.back() == '0') out.pop_back();
        if (neg_) out.push_back('-');
        std::reverse(out.begin(), out.end());
        return out;
    }

    bool is_zero() const { return n_ == 0; }
    int sign() const { return n_ == 0 ? 0 : (neg_ ? -1 : 1); }

    // ---- arithmetic -----------------------------------------------------
    friend cpp_int operator+(const cpp_int& a, const cpp_int& b) {
        cpp_int r;
        if (a.neg_ == b.neg_) {
            add_mag(r, a, b);
            r.neg_ = a.neg_;
        } else {
            const int c = cmp_mag(a, b);
            if (c >= 0) {
                sub_mag(r, a, b);
                r.neg_ = a.neg_;
            } else {
                sub_mag(r, b, a);
                r.neg_ = b.neg_;
            }
        }
        r.normalize();
        return r;
    }
    friend cpp_int operator-(const cpp_int& a, const cpp_int& b) {
        cpp_int nb = b;
        nb.neg_ = !nb.neg_;
        return a + nb;
    }
    friend cpp_int operator*(const cpp_int& a, const cpp_int& b) {
        cpp_int r;
        mul_mag(r, a, b);
        r.neg_ = a.neg_ != b.neg_;
        r.normalize();
        return r;
    }
    friend cpp_int operator/(const cpp_int& a, const cpp_int& b) {
        cpp_int q, r;
        divmod(a, b, &q, &r);
        return q;
    }
    friend cpp_int operator%(const cpp_int& a, const cpp_int& b) {
        cpp_int q, r;
        divmod(a, b, nullptr, &r);
        return r;
    }
    cpp_int operator-() const {
        cpp_int r = *this;
        if (r.n_ != 0) r.neg_ = !r.neg_;
        return r;
    }
    cpp_int operator+() const { return *this; }

    cpp_int& operator+=(const cpp_int& o) { return *this = *this + o; }
    cpp_int& operator-=(const cpp_int& o) { return *this = *this - o; }
    cpp_int& operator*=(const cpp_int& o) { return *this = *this * o; }
    cpp_int& operator/=(const cpp_int& o) { return *this = *this / o; }
    cpp_int& operator%=(const cpp_int& o) { return *this = *this % o; }
    cpp_int& operator<<=(unsigned k) { return *this = *this << k; }
    cpp_int& operator>>=(unsigned k) { return *this = *this >> k; }
    cpp_int& operator++() { return *this += 1; }
    cpp_int& operator--() { return *this -= 1; }

    template <class I, class = std::enable_if_t<std::is_integral_v<I>>>
    friend cpp_int operator<<(const cpp_int& a, I k) {
        return shl(a, static_cast<unsigned>(k));
    }
    template <class I, class = std::enable_if_t<std::is_integral_v<I>>>
    friend cpp_int operator>>(const cpp_int& a, I k) {
        return shr(a, static_cast<unsigned>(k));
    }

    // ---- comparisons ----------------------------------------------------
    friend int compare(const cpp_int& a, const cpp_int& b) {
        if (a.sign() != b.sign()) return a.sign() < b.sign() ? -1 : 1;
        const int c = cmp_mag(a, b);
        return a.neg_ ? -c : c;
    }
    friend bool operator==(const cpp_int& a, const cpp_int& b) { return compare(a, b) == 0; }
    friend bool operator!=(const cpp_int& a, const cpp_int& b) { return compare(a, b) != 0; }
    friend bool operator<(const cpp_int& a, const cpp_int& b) { return compare(a, b) < 0; }
    friend bool operator<=(const cpp_int& a, const cpp_int& b) { return compare(a, b) <= 0; }
    friend bool operator>(const cpp_int& a, const cpp_int& b) { return compare(a, b) > 0; }
    friend bool operator>=(const cpp_int& a, const cpp_int& b) { return compare(a, b) >= 0; }

    friend std::ostream& operator<<(std::ostream& os, const cpp_int& v) { return os << v.str(); }

    template <class T>
    T convert_to() const {
        std::uint64_t m = n_ ? d_[0] : 0;
        T v = static_cast<T>(m);
        return neg_ ? static_cast<T>(-v) : v;
    }
    template <class T, class = std::enable_if_t<std::is_arithmetic_v<T>>>
    explicit operator T() const { return convert_to<T>(); }

    // ---- raw access for the free functions -------------------------------
    int limb_count() const { return n_; }
    std::uint64_t limb(int i) const { return i < n_ ? d_[i] : 0; }
    bool negative() const { return neg_; }
    void set_limbs(const std::uint64_t* src, int n) {
        if (n > kCap) throw std::overflow_error("cpp_int shim capacity exceeded");
        n_ = n;
        neg_ = false;
        for (int i = 0; i < n; ++i) d_[i] = src[i];
        normalize();
    }

private:
    bool neg_ = false;
    int n_ = 0;
    std::uint64_t d_[kCap];  // only [0, n_) is meaningful

    void normalize() {
        while (n_ > 0 && d_[n_ - 1] == 0) --n_;
        if (n_ == 0) neg_ = false;
    }

    void parse(const std::string& s0) {
        std::size_t i = 0;
        bool neg = false;
        while (i < s0.size() && (s0[i] == ' ')) ++i;
        if (i < s0.size() && (s0[i] == '-' || s0[i] == '+')) {
            neg = s0[i] == '-';
            ++i;
        }
        unsigned base = 10;
        if (i + 1 < s0.size() && s0[i] == '0' && (s0[i + 1] == 'x' || s0[i + 1] == 'X')) {
            base = 16;
            i += 2;
        }
        if (i >= s0.size()) throw std::runtime_error("unexpected empty integer string");
        n_ = 0;
        neg_ = false;
        for (; i < s0.size(); ++i) {
            const char c = s0[i];
            unsigned dig;
            if (c >= '0' && c <= '9') dig = static_cast<unsigned>(c - '0');
            else if (base == 16 && c >= 'a' && c <= 'f') dig = static_cast<unsigned>(c - 'a' + 10);
            else if (base == 16 && c >= 'A' && c <= 'F') dig = static_cast<unsigned>(c - 'A' + 10);
            else throw std::runtime_error("unexpected character in integer string");
            if (dig >= base) throw std::runtime_error("unexpected digit in integer string");
            mul_add_small(base, dig);
        }
        neg_ = neg && n_ != 0;
    }

    void mul_add_small(std::uint64_t m, std::uint64_t a) {
        unsigned __int128 carry = a;
        for (int i = 0; i < n_; ++i) {
            unsigned __int128 t = static_cast<unsigned __int128>(d_[i]) * m + carry;
            d_[i] = static_cast<std::uint64_t>(t);
            carry = t >> 64;
        }
        if (carry) {
            if (n_ >= kCap) throw std::overflow_error("cpp_int shim capacity exceeded");
            d_[n_++] = static_cast<std::uint64_t>(carry);
        }
    }

    // divides magnitude in place by a single limb, returns remainder
    std::uint64_t div_small(std::uint64_t m) {
        unsigned __int128 rem = 0;
        for (int i = n_ - 1; i >= 0; --i) {
            unsigned __int128 cur = (rem << 64) | d_[i];
            d_[i] = static_cast<std::uint64_t>(cur / m);
            rem = cur % m;
        }
        normalize();
        return static_cast<std::uint64_t>(rem);
    }

    static int cmp_mag(const cpp_int& a, const cpp_int& b) {
        if (a.n_ != b.n_) return a.n_ < b.n_ ? -1 : 1;
        for (int i = a.n_ - 1; i >= 0; --i) {
            if (a.d_[i] != b.d_[i]) return a.d_[i] < b.d_[i] ? -1 : 1;
        }
        return 0;
    }

    static void add_mag(cpp_int& r, const cpp_int& a, const cpp_int& b) {
        const int n = std::max(a.n_, b.n_);
        std::uint64_t carry = 0;
        for (int i = 0; i < n; ++i) {
            const std::uint64_t x = i < a.n_ ? a.d_[i] : 0;
            const std::uint64_t y = i < b.n_ ? b.d_[i] : 0;
            unsigned __int128 t = static_cast<unsigned __int128>(x) + y + carry;
            r.d_[i] = static_cast<std::uint64_t>(t);
            carry = static_cast<std::uint64_t>(t >> 64);
        }
        r.n_ = n;
        if (carry) {
            if (n >= kCap) throw std::overflow_error("cpp_int shim capacity exceeded");
            r.d_[r.n_++] = carry;
        }
    }

    // |a| >= |b|
    static void sub_mag(cpp_int& r, const cpp_int& a, const cpp_int& b) {
        std::uint64_t borrow = 0;
        for (int i = 0; i < a.n_; ++i) {
            const std::uint64_t x = a.d_[i];
            const std::uint64_t y = i < b.n_ ? b.d_[i] : 0;
            const std::uint64_t t = x - y - borrow;
            borrow = (x < y || (x == y && borrow)) ? 1 : 0;
            r.d_[i] = t;
        }
        r.n_ = a.n_;
    }

    static void mul_mag(cpp_int& r, const cpp_int& a, const cpp_int& b) {
        if (a.n_ == 0 || b.n_ == 0) {
            r.n_ = 0;
            return;
        }
        const int n = a.n_ + b.n_;
        if (n > kCap) throw std::overflow_error("cpp_int shim capacity exceeded");
        std::uint64_t t[kCap];
        for (int i = 0; i < n; ++i) t[i] = 0;
        for (int i = 0; i < a.n_; ++i) {
            unsigned __int128 carry = 0;
            const std::uint64_t ai = a.d_[i];
            for (int j = 0; j < b.n_; ++j) {
                unsigned __int128 cur = static_cast<unsigned __int128>(ai) * b.d_[j] + t[i + j] + carry;
                t[i + j] = static_cast<std::uint64_t>(cur);
                carry = cur >> 64;
            }
            t[i + b.n_] = static_cast<std::uint64_t>(carry);
        }
        std::memcpy(r.d_, t, sizeof(std::uint64_t) * static_cast<std::size_t>(n));
        r.n_ = n;
    }

    static cpp_int shl(const cpp_int& a, unsigned k) {
        if (a.n_ == 0) return a;
        const int ls = static_cast<int>(k / 64);
        const unsigned bs = k % 64;
        const std::size_t top_bit = static_cast<std::size_t>(64 * (a.n_ - 1) + 63 - __builtin_clzll(a.d_[a.n_ - 1])) + k;
        if (top_bit >= static_cast<std::size_t>(64 * kCap))
            throw std::overflow_error("cpp_int shim capacity exceeded");
        cpp_int r;
        for (int i = 0; i < kCap; ++i) r.d_[i] = 0;
        for (int i = a.n_ - 1; i >= 0; --i) {
            const int j = i + ls;
            if (bs == 0) {
                r.d_[j] = a.d_[i];
            } else {
                if (j + 1 < kCap) r.d_[j + 1] |= a.d_[i] >> (64 - bs);
                r.d_[j] |= a.d_[i] << bs;
            }
        }
        r.n_ = static_cast<int>(top_bit / 64) + 1;
        r.neg_ = a.neg_;
        r.normalize();
        return r;
    }

    static cpp_int shr(const cpp_int& a, unsigned k) {
        // Boost semantics for negative values are implementation-defined for
        // our purposes; the reference only shifts non-negative values.
        const int ls = static_cast<int>(k / 64);
        const unsigned bs = k % 64;
        cpp_int r;
        if (ls >= a.n_) return r;
        r.n_ = a.n_ - ls;
        for (int i = 0; i < r.n_; ++i) {
            std::uint64_t lo = a.d_[i + ls] >> bs;
            if (bs && i + ls + 1 < a.n_) lo |= a.d_[i + ls + 1] << (64 - bs);
            r.d_[i] = bs ? lo : a.d_[i + ls];
        }
        r.neg_ = a.neg_;
        r.normalize();
        return r;
    }

    // Knuth algorithm D on 64-bit limbs (magnitudes); truncating signs.
    static void divmod(const cpp_int& a, const cpp_int& b, cpp_int* q, cpp_int* r) {
        if (b.n_ == 0) throw std::overflow_error("Division by zero.");
        if (cmp_mag(a, b) < 0) {
            if (q) *q = cpp_int();
            if (r) *r = a;
            return;
        }
        cpp_int qq, rr;
        if (b.n_ == 1) {
            qq = a;
            qq.neg_ = false;
            const std::uint64_t rem = qq.div_small(b.d_[0]);
            rr = cpp_int(rem);
        } else {
            const int n = b.n_;
            const int m = a.n_ - b.n_;
            const int s = __builtin_clzll(b.d_[n - 1]);
            std::uint64_t vn[kCap];
            std::uint64_t un[kCap + 1];
            for (int i = n - 1; i > 0; --i)
                vn[i] = (b.d_[i] << s) | (s ? (b.d_[i - 1] >> (64 - s)) : 0);
            vn[0] = b.d_[0] << s;
            un[a.n_] = s ? (a.d_[a.n_ - 1] >> (64 - s)) : 0;
            for (int i = a.n_ - 1; i > 0; --i)
                un[i] = (a.d_[i] << s) | (s ? (a.d_[i - 1] >> (64 - s)) : 0);
            un[0] = a.d_[0] << s;
            qq.n_ = m + 1;
            for (int j = m; j >= 0; --j) {
                unsigned __int128 num = (static_cast<unsigned __int128>(un[j + n]) << 64) | un[j + n - 1];
                unsigned __int128 qhat = num / vn[n - 1];
                unsigned __int128 rhat = num % vn[n - 1];
                while (qhat >> 64 ||
                       qhat * vn[n - 2] > ((rhat << 64) | un[j + n - 2])) {
                    qhat -= 1;
                    rhat += vn[n - 1];
                    if (rhat >> 64) break;
                }
                // multiply and subtract
                unsigned __int128 borrow = 0;
                unsigned __int128 carry = 0;
                for (int i = 0; i < n; ++i) {
                    unsigned __int128 p = qhat * vn[i] + carry;
                    carry = p >> 64;
                    const std::uint64_t plo = static_cast<std::uint64_t>(p);
                    const std::uint64_t u = un[i + j];
                    const std::uint64_t t1 = u - plo;
                    const std::uint64_t b1 = u < plo ? 1 : 0;
                    const std::uint64_t t2 = t1 - static_cast<std::uint64_t>(borrow);
                    const std::uint64_t b2 = t1 < static_cast<std::uint64_t>(borrow) ? 1 : 0;
                    un[i + j] = t2;
                    borrow = b1 + b2;
                }
                const std::uint64_t u = un[j + n];
                const std::uint64_t c = static_cast<std::uint64_t>(carry);
                const std::uint64_t t1 = u - c;
                const std::uint64_t b1 = u < c ? 1 : 0;
                const std::uint64_t t2 = t1 - static_cast<std::uint64_t>(borrow);
                const std::uint64_t b2 = t1 < static_cast<std::uint64_t>(borrow) ? 1 : 0;
                un[j + n] = t2;
                if (b1 + b2) {
                    // add back
                    qhat -= 1;
                    std::uint64_t cc = 0;
                    for (int i = 0; i < n; ++i) {
                        unsigned __int128 t = static_cast<unsigned __int128>(un[i + j]) + vn[i] + cc;
                        un[i + j] = static_cast<std::uint64_t>(t);
                        cc = static_cast<std::uint64_t>(t >> 64);
                    }
                    un[j + n] += cc;
                }
                qq.d_[j] = static_cast<std::uint64_t>(qhat);
            }
            qq.normalize();
            rr.n_ = n;
            for (int i = 0; i < n; ++i)
                rr.d_[i] = (un[i] >> s) | (s ? (un[i + 1] << (64 - s)) : 0);
            rr.normalize();
        }
        qq.neg_ = (a.neg_ != b.neg_) && qq.n_ != 0;
        rr.neg_ = a.neg_ && rr.n_ != 0;
        if (q) *q = qq;
        if (r) *r = rr;
    }
};

// ---- free functions used by the reference --------------------------------

inline std::size_t msb(const cpp_int& v) {
    if (v.sign() <= 0) throw std::domain_error("msb of non-positive value");
    const int n = v.limb_count();
    return static_cast<std::size_t>(64 * (n - 1) + 63 - __builtin_clzll(v.limb(n - 1)));
}

inline bool bit_test(const cpp_int& v, unsigned k) {
    return (v.limb(static_cast<int>(k / 64)) >> (k % 64)) & 1u;
}

inline cpp_int abs(const cpp_int& v) { return v.sign() < 0 ? -v : v; }

inline cpp_int powm(const cpp_int& base, const cpp_int& exp, const cpp_int& mod) {
    if (exp.sign() < 0) throw std::runtime_error("powm: negative exponent");
    cpp_int result = cpp_int(1) % mod;
    cpp_int b = base % mod;
    if (b.sign() < 0) b += mod;
    const std::size_t nbits = exp.sign() == 0 ? 0 : msb(exp) + 1;
    for (std::size_t i = nbits; i-- > 0;) {
        result = (result * result) % mod;
        if (bit_test(exp, static_cast<unsigned>(i))) result = (result * b) % mod;
    }
    return result;
}

/// Chunks of `chunk_size` bits (only 8 is used by the reference), least
/// significant chunk first when msv_first == false.
template <class It>
cpp_int& import_bits(cpp_int& v, It first, It last, unsigned chunk_size = 0, bool msv_first = true) {
    if (chunk_size == 0) chunk_size = 8;
    if (chunk_size != 8) throw std::runtime_error("import_bits shim supports 8-bit chunks only");
    std::uint64_t limbs[cpp_int::kCap] = {};
    std::size_t count = static_cast<std::size_t>(std::distance(first, last));
    if (count > 8 * static_cast<std::size_t>(cpp_int::kCap))
        throw std::overflow_error("cpp_int shim capacity exceeded");
    std::size_t idx = 0;
    for (It it = first; it != last; ++it, ++idx) {
        const std::size_t pos = msv_first ? (count - 1 - idx) : idx;  // byte position from LSB
        limbs[pos / 8] |= static_cast<std::uint64_t>(static_cast<std::uint8_t>(*it)) << (8 * (pos % 8));
    }
    v.set_limbs(limbs, static_cast<int>((count + 7) / 8));
    return v;
}

/// Emits the minimal number of chunks (a single 0 chunk for zero), matching
/// Boost's behaviour that field.hpp:164 and transcript.hpp:90-95 depend on.
template <class Out>
Out export_bits(const cpp_int& v, Out out, unsigned chunk_size, bool msv_first = true) {
    if (chunk_size != 8) throw std::runtime_error("export_bits shim supports 8-bit chunks only");
    std::size_t nbytes = 1;
    if (v.sign() != 0) nbytes = msb(abs(v)) / 8 + 1;
    for (std::size_t k = 0; k < nbytes; ++k) {
        const std::size_t pos = msv_first ? (nbytes - 1 - k) : k;
        const std::uint8_t byte = static_cast<std::uint8_t>(v.limb(static_cast<int>(pos / 8)) >> (8 * (pos % 8)));
        *out = byte;
        ++out;
    }
    return out;
}

}  // namespace multiprecision
}  // namespace boost
