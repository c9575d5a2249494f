// Host-side core of the B200 prover: prime-field arithmetic in the same
// Montgomery representation as the device (R = 2^256, 4x64-bit limbs here,
// 8x32-bit limbs on the GPU — identical bits in memory), SHA-256 (SHA-NI when
// the CPU has it) and the Fiat–Shamir transcript.
//
// Byte-level contract followed (reference file:line):
//   field encoding      field.hpp:159-187  (canonical LE, width ceil(bits/8))
//   transcript init     transcript.hpp:19-28 ("dgkr.transcript.v1"||label||LEmin(p))
//   absorb              transcript.hpp:32-48 (state = SHA256(state||bytes))
//   challenge           transcript.hpp:52-68, squeeze :97-125
//   challenge_index     transcript.hpp:71-83
//   SHA-256             sha256.hpp:17-158 (FIPS 180-4)
#pragma once

#include <array>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "dgkr_b200.h"

namespace dgkr_b200 {

// Status codes: DGKR_* of the C ABI (include/dgkr_b200.h).
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

// ---------------------------------------------------------------------------
// Field: runtime odd modulus p < 2^256, Montgomery form with R = 2^256.
// ---------------------------------------------------------------------------
struct U256 {
    std::uint64_t w[4] = {0, 0, 0, 0};
    bool operator==(const U256& o) const {
        return w[0] == o.w[0] && w[1] == o.w[1] && w[2] == o.w[2] && w[3] == o.w[3];
    }
    bool operator!=(const U256& o) const { return !(*this == o); }
    bool is_zero() const { return (w[0] | w[1] | w[2] | w[3]) == 0; }
};

inline bool lt(const U256& a, const U256& b) {
    for (int i = 3; i >= 0; --i) {
        if (a.w[i] != b.w[i]) return a.w[i] < b.w[i];
    }
    return false;
}

inline std::uint64_t add_to(U256& r, const U256& a, const U256& b) {
    unsigned __int128 c = 0;
    for (int i = 0; i < 4; ++i) {
        c += static_cast<unsigned __int128>(a.w[i]) + b.w[i];
        r.w[i] = static_cast<std::uint64_t>(c);
        c >>= 64;
    }
    return static_cast<std::uint64_t>(c);
}

inline std::uint64_t sub_to(U256& r, const U256& a, const U256& b) {
    std::uint64_t borrow = 0;
    for (int i = 0; i < 4; ++i) {
        const std::uint64_t x = a.w[i], y = b.w[i];
        const std::uint64_t t = x - y - borrow;
        borrow = (x < y || (x == y && borrow)) ? 1 : 0;
        r.w[i] = t;
    }
    return borrow;
}

class HostField {
public:
    HostField() = default;

    /// modulus as minimal little-endian bytes (the form the transcript
    /// hashes, transcript.hpp:90-95).
    HostField(const std::uint8_t* mod, std::size_t len) {
        if (len == 0 || len > 32) fail(DGKR_UNSUPPORTED, "modulus must be 1..32 bytes");
        for (std::size_t i = 0; i < len; ++i) p_.w[i / 8] |= static_cast<std::uint64_t>(mod[i]) << (8 * (i % 8));
        if (p_.is_zero()) fail(DGKR_INVALID_ARGUMENT, "zero modulus");
        bits_ = 0;
        for (int i = 3; i >= 0; --i) {
            if (p_.w[i]) {
                bits_ = 64 * i + 64 - __builtin_clzll(p_.w[i]);
                break;
            }
        }
        if (bits_ > 256) fail(DGKR_UNSUPPORTED, "modulus wider than 256 bits");
        if ((p_.w[0] & 1) == 0) fail(DGKR_UNSUPPORTED, "GPU prover needs an odd modulus");
        if (bits_ < 2) fail(DGKR_INVALID_ARGUMENT, "modulus must be at least 2");
        width_ = (bits_ + 7) / 8;
        // -p^{-1} mod 2^64 by Newton iteration
        std::uint64_t inv = 1;
        for (int i = 0; i < 7; ++i) inv *= 2 - p_.w[0] * inv;
        np0_ = static_cast<std::uint64_t>(0) - inv;
        // R mod p and R^2 mod p by doubling
        U256 x;
        x.w[0] = 1;
        for (int i = 0; i < 512; ++i) {
            U256 d;
            const std::uint64_t carry = add_to(d, x, x);
            U256 s;
            const std::uint64_t bw = sub_to(s, d, p_);
            x = (carry || !bw) ? s : d;
            if (i == 255) one_ = x;
        }
        r2_ = x;
        mod_bytes_.assign(mod, mod + len);
        while (mod_bytes_.size() > 1 && mod_bytes_.back() == 0) mod_bytes_.pop_back();
    }

    const U256& p() const { return p_; }
    std::uint64_t np0() const { return np0_; }
    const U256& r2() const { return r2_; }
    const U256& one() const { return one_; }
    std::size_t bits() const { return bits_; }
    std::size_t width() const { return width_; }
    const std::vector<std::uint8_t>& modulus_bytes() const { return mod_bytes_; }
    bool same(const HostField& o) const { return p_ == o.p_; }

    U256 add(const U256& a, const U256& b) const {
        U256 r, s;
        const std::uint64_t carry = add_to(r, a, b);  // a carry-out only for p >= 2^255
        const std::uint64_t borrow = sub_to(s, r, p_);
        return (borrow && !carry) ? r : s;
    }
    U256 sub(const U256& a, const U256& b) const {
        U256 r;
        if (sub_to(r, a, b)) add_to(r, r, p_);
        return r;
    }
    U256 neg(const U256& a) const { return a.is_zero() ? a : sub(p_, a); }

    /// Montgomery product a*b*R^{-1} mod p (CIOS, 64-bit limbs).
    U256 mul(const U256& a, const U256& b) const {
        std::uint64_t t[6] = {0, 0, 0, 0, 0, 0};
        for (int i = 0; i < 4; ++i) {
            unsigned __int128 c = 0;
            for (int j = 0; j < 4; ++j) {
                c += static_cast<unsigned __int128>(a.w[j]) * b.w[i] + t[j];
                t[j] = static_cast<std::uint64_t>(c);
                c >>= 64;
            }
            c += t[4];
            t[4] = static_cast<std::uint64_t>(c);
            t[5] = static_cast<std::uint64_t>(c >> 64);
            const std::uint64_t m = t[0] * np0_;
            c = static_cast<unsigned __int128>(m) * p_.w[0] + t[0];
            c >>= 64;
            for (int j = 1; j < 4; ++j) {
                c += static_cast<unsigned __int128>(m) * p_.w[j] + t[j];
                t[j - 1] = static_cast<std::uint64_t>(c);
                c >>= 64;
            }
            c += t[4];
            t[3] = static_cast<std::uint64_t>(c);
            t[4] = t[5] + static_cast<std::uint64_t>(c >> 64);
        }
        U256 r{{t[0], t[1], t[2], t[3]}}, s;
        const std::uint64_t borrow = sub_to(s, r, p_);
        return (borrow && t[4] == 0) ? r : s;  // t[4]: the 257th bit (p close to 2^256)
    }

    U256 to_mont(const U256& canonical) const { return mul(canonical, r2_); }
    U256 from_mont(const U256& m) const {
        U256 one{{1, 0, 0, 0}};
        return mul(m, one);
    }
    U256 from_u64(std::uint64_t v) const {
        U256 x{{v, 0, 0, 0}};
        // v may exceed p for tiny moduli: reduce by repeated subtraction of
        // multiples via Montgomery (x*R^2*R^-1 = x*R mod p works for any x<2^256)
        return mul(x, r2_);
    }

    /// canonical LE bytes (width()) of a Montgomery value
    void to_bytes(const U256& m, std::uint8_t* out) const {
        const U256 c = from_mont(m);
        for (std::size_t i = 0; i < width_; ++i) out[i] = static_cast<std::uint8_t>(c.w[i / 8] >> (8 * (i % 8)));
    }
    std::vector<std::uint8_t> to_bytes(const U256& m) const {
        std::vector<std::uint8_t> v(width_);
        to_bytes(m, v.data());
        return v;
    }
    /// parse canonical bytes (rejects >= p, field.hpp:175-187); returns Montgomery
    U256 from_bytes(const std::uint8_t* in) const {
        U256 c;
        for (std::size_t i = 0; i < width_; ++i) c.w[i / 8] |= static_cast<std::uint64_t>(in[i]) << (8 * (i % 8));
        if (!lt(c, p_)) fail(DGKR_INVALID_ARGUMENT, "non-canonical field element encoding");
        return to_mont(c);
    }
    bool canonical_lt_p(const std::uint8_t* in, std::size_t n) const {
        U256 c;
        for (std::size_t i = 0; i < n && i < 32; ++i) c.w[i / 8] |= static_cast<std::uint64_t>(in[i]) << (8 * (i % 8));
        return lt(c, p_);
    }

    U256 pow(U256 base, const U256& e) const {
        U256 r = one_;
        for (int i = 255; i >= 0; --i) {
            r = mul(r, r);
            if ((e.w[i / 64] >> (i % 64)) & 1) r = mul(r, base);
        }
        return r;
    }
    U256 inv(const U256& a) const {
        if (a.is_zero()) fail(DGKR_DOMAIN_ERROR, "inverse of zero field element");
        U256 e;
        U256 two{{2, 0, 0, 0}};
        sub_to(e, p_, two);
        return pow(a, e);
    }

private:
    U256 p_, r2_, one_;
    std::uint64_t np0_ = 0;
    std::size_t bits_ = 0, width_ = 0;
    std::vector<std::uint8_t> mod_bytes_;
};

// ---------------------------------------------------------------------------
// SHA-256
// ---------------------------------------------------------------------------
using Digest = std::array<std::uint8_t, 32>;

void sha256_compress(std::uint32_t state[8], const std::uint8_t* blocks, std::size_t nblocks);
bool sha256_has_shani();

class Sha256 {
public:
    Sha256() { reset(); }
    void reset() {
        static const std::uint32_t iv[8] = {0x6a09e667u, 0xbb67ae85u, 0x3c6ef372u, 0xa54ff53au,
                                           0x510e527fu, 0x9b05688cu, 0x1f83d9abu, 0x5be0cd19u};
        std::memcpy(h_, iv, sizeof(iv));
        blen_ = 0;
        total_ = 0;
    }
    void update(const std::uint8_t* d, std::size_t n) {
        total_ += n;
        if (blen_) {
            const std::size_t take = std::min<std::size_t>(64 - blen_, n);
            std::memcpy(buf_ + blen_, d, take);
            blen_ += take;
            d += take;
            n -= take;
            if (blen_ == 64) {
                sha256_compress(h_, buf_, 1);
                blen_ = 0;
            }
        }
        if (n >= 64) {
            sha256_compress(h_, d, n / 64);
            d += (n / 64) * 64;
            n %= 64;
        }
        if (n) {
            std::memcpy(buf_, d, n);
            blen_ = n;
        }
    }
    void update(std::string_view s) { update(reinterpret_cast<const std::uint8_t*>(s.data()), s.size()); }
    Digest finalize() {
        const std::uint64_t bit_len = total_ * 8;
        std::uint8_t pad[128] = {0};
        pad[0] = 0x80;
        std::size_t padlen = (blen_ < 56) ? (56 - blen_) : (120 - blen_);
        std::uint8_t tail[136];
        std::memcpy(tail, pad, padlen);
        for (int i = 0; i < 8; ++i) tail[padlen + i] = static_cast<std::uint8_t>(bit_len >> (56 - 8 * i));
        const std::uint64_t keep = total_;
        update(tail, padlen + 8);
        total_ = keep;
        Digest out;
        for (int i = 0; i < 8; ++i) {
            out[4 * i + 0] = static_cast<std::uint8_t>(h_[i] >> 24);
            out[4 * i + 1] = static_cast<std::uint8_t>(h_[i] >> 16);
            out[4 * i + 2] = static_cast<std::uint8_t>(h_[i] >> 8);
            out[4 * i + 3] = static_cast<std::uint8_t>(h_[i]);
        }
        return out;
    }

private:
    std::uint32_t h_[8];
    std::uint8_t buf_[64];
    std::size_t blen_ = 0;
    std::uint64_t total_ = 0;
};

inline Digest sha256(const std::uint8_t* d, std::size_t n) {
    Sha256 h;
    h.update(d, n);
    return h.finalize();
}

/// SHA256(a(32) || b(32)): one data block + the constant padding block.
Digest sha256_64(const std::uint8_t* a32, const std::uint8_t* b32);
/// state <- SHA256(state || e_i) for n consecutive 32-byte elements
void absorb_chain32(std::uint8_t* state, const std::uint8_t* elems, std::size_t n);
/// k independent chains of n absorbs each, interleaved (multi-buffer SHA-NI):
/// states[j] <- chain of elems[j][0..n) (32-byte elements), byte-identical to
/// k calls of absorb_chain32
void absorb_chain32_multi(std::uint8_t* const* states, const std::uint8_t* const* elems, std::size_t k,
                          std::size_t n);

// ---------------------------------------------------------------------------
// Transcript (transcript.hpp:17-130)
// ---------------------------------------------------------------------------
class Transcript {
public:
    Transcript() = default;
    Transcript(const HostField* f, std::string_view label) : f_(f) {
        Sha256 h;
        h.update("dgkr.transcript.v1");
        h.update(label);
        h.update(f->modulus_bytes().data(), f->modulus_bytes().size());
        state_ = h.finalize();
    }
    Transcript(const HostField* f, const std::uint8_t* state, std::uint64_t draws) : f_(f), draws_(draws) {
        std::memcpy(state_.data(), state, 32);
    }

    const Digest& state() const { return state_; }
    std::uint64_t draws() const { return draws_; }
    /// the 32-byte chaining state, for absorbs run elsewhere (AbsorbPool)
    std::uint8_t* state_bytes() { return state_.data(); }

    /// absorb_bytes of n consecutive elements of `width` bytes (already canonical)
    void absorb_many(const std::uint8_t* d, std::size_t n, std::size_t width) {
        if (width == 32) {
            absorb_chain32(state_.data(), d, n);
            return;
        }
        for (std::size_t i = 0; i < n; ++i) absorb_bytes(d + i * width, width);
    }
    void absorb_bytes(const std::uint8_t* d, std::size_t n) {
        if (n == 32) {
            state_ = sha256_64(state_.data(), d);
            return;
        }
        Sha256 h;
        h.update(state_.data(), 32);
        h.update(d, n);
        state_ = h.finalize();
    }
    /// absorb a field element given in Montgomery form
    void absorb(const U256& m) {
        std::uint8_t b[32];
        f_->to_bytes(m, b);
        absorb_bytes(b, f_->width());
    }
    void absorb_u64(std::uint64_t v) {
        std::uint8_t b[8];
        for (int i = 0; i < 8; ++i) b[i] = static_cast<std::uint8_t>(v >> (8 * i));
        absorb_bytes(b, 8);
    }
    /// returns the challenge in Montgomery form
    U256 challenge() {
        const std::size_t w = f_->width();
        const unsigned top = static_cast<unsigned>(f_->bits() - 8 * (w - 1));
        const std::uint8_t mask = top >= 8 ? 0xff : static_cast<std::uint8_t>((1u << top) - 1);
        std::uint8_t buf[64];
        if (w == 0 || w > sizeof(buf)) fail(DGKR_LOGIC_ERROR, "field width out of range");
        const std::uint64_t draw = draws_++;
        for (std::uint64_t ctr = 0;; ++ctr) {
            squeeze("chal", draw, ctr, w, buf);
            buf[w - 1] &= mask;
            if (f_->canonical_lt_p(buf, w)) return f_->from_bytes(buf);
        }
    }
    std::uint64_t challenge_index(std::uint64_t bound) {
        if (bound == 0) fail(DGKR_INVALID_ARGUMENT, "challenge_index bound must be positive");
        const std::uint64_t draw = draws_++;
        const std::uint64_t limit = bound * (~std::uint64_t{0} / bound);
        std::uint8_t buf[32];
        for (std::uint64_t ctr = 0;; ++ctr) {
            squeeze("idx", draw, ctr, 8, buf);
            std::uint64_t v = 0;
            for (int i = 7; i >= 0; --i) v = (v << 8) | buf[i];
            if (v < limit) return v % bound;
        }
    }

private:
    void squeeze(std::string_view tag, std::uint64_t draw, std::uint64_t ctr, std::size_t n,
                 std::uint8_t* out) const {
        std::size_t got = 0;
        for (std::uint64_t block = 0; got < n; ++block) {
            std::uint8_t msg[32 + 8 + 24];
            std::memcpy(msg, state_.data(), 32);
            std::memcpy(msg + 32, tag.data(), tag.size());
            std::size_t off = 32 + tag.size();
            for (int i = 0; i < 8; ++i) msg[off + i] = static_cast<std::uint8_t>(draw >> (8 * i));
            for (int i = 0; i < 8; ++i) msg[off + 8 + i] = static_cast<std::uint8_t>(ctr >> (8 * i));
            for (int i = 0; i < 8; ++i) msg[off + 16 + i] = static_cast<std::uint8_t>(block >> (8 * i));
            const Digest d = sha256(msg, off + 24);
            const std::size_t take = std::min<std::size_t>(32, n - got);
            std::memcpy(out + got, d.data(), take);
            got += take;
        }
    }

    const HostField* f_ = nullptr;
    Digest state_{};
    std::uint64_t draws_ = 0;
};

}  // namespace dgkr_b200
