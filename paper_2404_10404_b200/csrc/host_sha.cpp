// Host SHA-256 compression: SHA-NI (x86 SHA extensions) when available, a
// portable FIPS 180-4 loop otherwise. The serial transcript chain
// (transcript.hpp:32-37: one SHA-256 of state||element per absorb) is the
// Amdahl term bit-exactness imposes, so it gets the fastest host path.
#include <cpuid.h>
#include <cstdlib>
#include <immintrin.h>

#include "host_core.hpp"

namespace dgkr_b200 {

namespace {

const std::uint32_t kK[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5,
    0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174,
    0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
    0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967,
    0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85,
    0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
    0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
    0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2};

inline std::uint32_t rotr(std::uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }

void compress_portable(std::uint32_t st[8], const std::uint8_t* p, std::size_t nblocks) {
    for (; nblocks--; p += 64) {
        std::uint32_t w[64];
        for (int i = 0; i < 16; ++i)
            w[i] = (std::uint32_t(p[4 * i]) << 24) | (std::uint32_t(p[4 * i + 1]) << 16) |
                   (std::uint32_t(p[4 * i + 2]) << 8) | std::uint32_t(p[4 * i + 3]);
        for (int i = 16; i < 64; ++i) {
            const std::uint32_t s0 = rotr(w[i - 15], 7) ^ rotr(w[i - 15], 18) ^ (w[i - 15] >> 3);
            const std::uint32_t s1 = rotr(w[i - 2], 17) ^ rotr(w[i - 2], 19) ^ (w[i - 2] >> 10);
            w[i] = w[i - 16] + s0 + w[i - 7] + s1;
        }
        std::uint32_t a = st[0], b = st[1], c = st[2], d = st[3], e = st[4], f = st[5], g = st[6], h = st[7];
        for (int i = 0; i < 64; ++i) {
            const std::uint32_t t1 = h + (rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25)) + ((e & f) ^ (~e & g)) + kK[i] + w[i];
            const std::uint32_t t2 = (rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22)) + ((a & b) ^ (a & c) ^ (b & c));
            h = g;
            g = f;
            f = e;
            e = d + t1;
            d = c;
            c = b;
            b = a;
            a = t1 + t2;
        }
        st[0] += a;
        st[1] += b;
        st[2] += c;
        st[3] += d;
        st[4] += e;
        st[5] += f;
        st[6] += g;
        st[7] += h;
    }
}

__attribute__((target("sha,sse4.1,ssse3"))) void compress_shani(std::uint32_t st[8], const std::uint8_t* p,
                                                                 std::size_t nblocks) {
    const __m128i bswap = _mm_set_epi64x(0x0c0d0e0f08090a0bULL, 0x0405060700010203ULL);
    __m128i tmp = _mm_loadu_si128(reinterpret_cast<const __m128i*>(&st[0]));  // DCBA
    __m128i s1 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(&st[4]));   // HGFE
    tmp = _mm_shuffle_epi32(tmp, 0xB1);                                       // CDAB
    s1 = _mm_shuffle_epi32(s1, 0x1B);                                         // EFGH
    __m128i s0 = _mm_alignr_epi8(tmp, s1, 8);                                 // ABEF
    s1 = _mm_blend_epi16(s1, tmp, 0xF0);                                      // CDGH
    for (; nblocks--; p += 64) {
        const __m128i abef = s0, cdgh = s1;
        __m128i w[16];
        for (int g = 0; g < 4; ++g)
            w[g] = _mm_shuffle_epi8(_mm_loadu_si128(reinterpret_cast<const __m128i*>(p + 16 * g)), bswap);
        for (int g = 4; g < 16; ++g) {
            // W[t] = sigma1(W[t-2]) + W[t-7] + sigma0(W[t-15]) + W[t-16]
            __m128i x = _mm_sha256msg1_epu32(w[g - 4], w[g - 3]);
            x = _mm_add_epi32(x, _mm_alignr_epi8(w[g - 1], w[g - 2], 4));
            w[g] = _mm_sha256msg2_epu32(x, w[g - 1]);
        }
        for (int g = 0; g < 16; ++g) {
            __m128i m = _mm_add_epi32(w[g], _mm_loadu_si128(reinterpret_cast<const __m128i*>(&kK[4 * g])));
            s1 = _mm_sha256rnds2_epu32(s1, s0, m);
            m = _mm_shuffle_epi32(m, 0x0E);
            s0 = _mm_sha256rnds2_epu32(s0, s1, m);
        }
        s0 = _mm_add_epi32(s0, abef);
        s1 = _mm_add_epi32(s1, cdgh);
    }
    tmp = _mm_shuffle_epi32(s0, 0x1B);       // FEBA
    s1 = _mm_shuffle_epi32(s1, 0xB1);        // DCHG
    s0 = _mm_blend_epi16(tmp, s1, 0xF0);     // DCBA
    s1 = _mm_alignr_epi8(s1, tmp, 8);        // HGFE
    _mm_storeu_si128(reinterpret_cast<__m128i*>(&st[0]), s0);
    _mm_storeu_si128(reinterpret_cast<__m128i*>(&st[4]), s1);
}

// W+K of the constant padding block of a 64-byte message (0x80, zeros, bit
// length 512): its message schedule never changes, so chained absorbs skip it.
struct PadWK {
    alignas(16) std::uint32_t wk[64];
    PadWK() {
        std::uint32_t w[64] = {0};
        w[0] = 0x80000000u;
        w[15] = 512;
        for (int t = 16; t < 64; ++t) {
            const std::uint32_t s0 = rotr(w[t - 15], 7) ^ rotr(w[t - 15], 18) ^ (w[t - 15] >> 3);
            const std::uint32_t s1 = rotr(w[t - 2], 17) ^ rotr(w[t - 2], 19) ^ (w[t - 2] >> 10);
            w[t] = w[t - 16] + s0 + w[t - 7] + s1;
        }
        for (int t = 0; t < 64; ++t) wk[t] = w[t] + kK[t];
    }
};
const PadWK kPadWK;

/// state <- SHA256(state || e_i) for i < n, 32-byte elements (the transcript's
/// absorb of a field element, transcript.hpp:32-42, chained). The state stays
/// in SHA-NI's ABEF/CDGH registers; each digest's words are the next block's
/// first 8 message words as they are.
__attribute__((target("sha,sse4.1,ssse3"))) void absorb_chain32_shani(std::uint8_t* state, const std::uint8_t* e,
                                                                       std::size_t n) {
    const __m128i bswap = _mm_set_epi64x(0x0c0d0e0f08090a0bULL, 0x0405060700010203ULL);
    static const std::uint32_t iv[8] = {0x6a09e667u, 0xbb67ae85u, 0x3c6ef372u, 0xa54ff53au,
                                        0x510e527fu, 0x9b05688cu, 0x1f83d9abu, 0x5be0cd19u};
    __m128i tmp = _mm_loadu_si128(reinterpret_cast<const __m128i*>(&iv[0]));
    __m128i ivh = _mm_loadu_si128(reinterpret_cast<const __m128i*>(&iv[4]));
    tmp = _mm_shuffle_epi32(tmp, 0xB1);
    ivh = _mm_shuffle_epi32(ivh, 0x1B);
    const __m128i iv0 = _mm_alignr_epi8(tmp, ivh, 8);   // ABEF
    const __m128i iv1 = _mm_blend_epi16(ivh, tmp, 0xF0);  // CDGH
    // digest words h0..h3 / h4..h7 (lane 0 = first word)
    __m128i wa = _mm_shuffle_epi8(_mm_loadu_si128(reinterpret_cast<const __m128i*>(state)), bswap);
    __m128i wb = _mm_shuffle_epi8(_mm_loadu_si128(reinterpret_cast<const __m128i*>(state + 16)), bswap);
    for (std::size_t i = 0; i < n; ++i, e += 32) {
        __m128i w[16];
        w[0] = wa;
        w[1] = wb;
        w[2] = _mm_shuffle_epi8(_mm_loadu_si128(reinterpret_cast<const __m128i*>(e)), bswap);
        w[3] = _mm_shuffle_epi8(_mm_loadu_si128(reinterpret_cast<const __m128i*>(e + 16)), bswap);
        for (int g = 4; g < 16; ++g) {
            __m128i x = _mm_sha256msg1_epu32(w[g - 4], w[g - 3]);
            x = _mm_add_epi32(x, _mm_alignr_epi8(w[g - 1], w[g - 2], 4));
            w[g] = _mm_sha256msg2_epu32(x, w[g - 1]);
        }
        __m128i s0 = iv0, s1 = iv1;
        for (int g = 0; g < 16; ++g) {
            __m128i m = _mm_add_epi32(w[g], _mm_loadu_si128(reinterpret_cast<const __m128i*>(&kK[4 * g])));
            s1 = _mm_sha256rnds2_epu32(s1, s0, m);
            m = _mm_shuffle_epi32(m, 0x0E);
            s0 = _mm_sha256rnds2_epu32(s0, s1, m);
        }
        s0 = _mm_add_epi32(s0, iv0);
        s1 = _mm_add_epi32(s1, iv1);
        const __m128i a0 = s0, a1 = s1;
        for (int g = 0; g < 16; ++g) {  // padding block: precomputed W+K
            __m128i m = _mm_load_si128(reinterpret_cast<const __m128i*>(&kPadWK.wk[4 * g]));
            s1 = _mm_sha256rnds2_epu32(s1, s0, m);
            m = _mm_shuffle_epi32(m, 0x0E);
            s0 = _mm_sha256rnds2_epu32(s0, s1, m);
        }
        s0 = _mm_add_epi32(s0, a0);
        s1 = _mm_add_epi32(s1, a1);
        wa = _mm_shuffle_epi32(_mm_unpackhi_epi64(s1, s0), 0x1B);  // h0 h1 h2 h3
        wb = _mm_shuffle_epi32(_mm_unpacklo_epi64(s1, s0), 0x1B);  // h4 h5 h6 h7
    }
    _mm_storeu_si128(reinterpret_cast<__m128i*>(state), _mm_shuffle_epi8(wa, bswap));
    _mm_storeu_si128(reinterpret_cast<__m128i*>(state + 16), _mm_shuffle_epi8(wb, bswap));
}

/// K independent absorb chains interleaved in one thread (multi-buffer
/// SHA-NI): chain k does state_k <- SHA256(state_k || e_k[i]) for i < n.
/// One chain is bound by SHA256RNDS2 latency (64 dependent rounds-pairs per
/// absorb); K chains fill its pipeline, so K proofs' output absorbs cost
/// about as much wall time as one (gkr.hpp:189-190 per proof, unchanged).
template <int K>
__attribute__((target("sha,sse4.1,ssse3"))) void absorb_chain32_shani_x(std::uint8_t* const* state,
                                                                         const std::uint8_t* const* e, std::size_t n) {
    const __m128i bswap = _mm_set_epi64x(0x0c0d0e0f08090a0bULL, 0x0405060700010203ULL);
    static const std::uint32_t iv[8] = {0x6a09e667u, 0xbb67ae85u, 0x3c6ef372u, 0xa54ff53au,
                                        0x510e527fu, 0x9b05688cu, 0x1f83d9abu, 0x5be0cd19u};
    __m128i tmp = _mm_loadu_si128(reinterpret_cast<const __m128i*>(&iv[0]));
    __m128i ivh = _mm_loadu_si128(reinterpret_cast<const __m128i*>(&iv[4]));
    tmp = _mm_shuffle_epi32(tmp, 0xB1);
    ivh = _mm_shuffle_epi32(ivh, 0x1B);
    const __m128i iv0 = _mm_alignr_epi8(tmp, ivh, 8);
    const __m128i iv1 = _mm_blend_epi16(ivh, tmp, 0xF0);
    __m128i wa[K], wb[K];
    const std::uint8_t* p[K];
    for (int k = 0; k < K; ++k) {
        wa[k] = _mm_shuffle_epi8(_mm_loadu_si128(reinterpret_cast<const __m128i*>(state[k])), bswap);
        wb[k] = _mm_shuffle_epi8(_mm_loadu_si128(reinterpret_cast<const __m128i*>(state[k] + 16)), bswap);
        p[k] = e[k];
    }
    for (std::size_t i = 0; i < n; ++i) {
        __m128i w[K][16], s0[K], s1[K], a0[K], a1[K];
#pragma GCC unroll 4
        for (int k = 0; k < K; ++k) {
            w[k][0] = wa[k];
            w[k][1] = wb[k];
            w[k][2] = _mm_shuffle_epi8(_mm_loadu_si128(reinterpret_cast<const __m128i*>(p[k])), bswap);
            w[k][3] = _mm_shuffle_epi8(_mm_loadu_si128(reinterpret_cast<const __m128i*>(p[k] + 16)), bswap);
            p[k] += 32;
            s0[k] = iv0;
            s1[k] = iv1;
        }
#pragma GCC unroll 16
        for (int g = 0; g < 16; ++g) {
            const __m128i kk = _mm_loadu_si128(reinterpret_cast<const __m128i*>(&kK[4 * g]));
#pragma GCC unroll 4
            for (int k = 0; k < K; ++k) {
                if (g >= 4) {
                    __m128i x = _mm_sha256msg1_epu32(w[k][g - 4], w[k][g - 3]);
                    x = _mm_add_epi32(x, _mm_alignr_epi8(w[k][g - 1], w[k][g - 2], 4));
                    w[k][g] = _mm_sha256msg2_epu32(x, w[k][g - 1]);
                }
                __m128i m = _mm_add_epi32(w[k][g], kk);
                s1[k] = _mm_sha256rnds2_epu32(s1[k], s0[k], m);
                m = _mm_shuffle_epi32(m, 0x0E);
                s0[k] = _mm_sha256rnds2_epu32(s0[k], s1[k], m);
            }
        }
#pragma GCC unroll 4
        for (int k = 0; k < K; ++k) {
            s0[k] = _mm_add_epi32(s0[k], iv0);
            s1[k] = _mm_add_epi32(s1[k], iv1);
            a0[k] = s0[k];
            a1[k] = s1[k];
        }
#pragma GCC unroll 16
        for (int g = 0; g < 16; ++g) {
            const __m128i mm = _mm_load_si128(reinterpret_cast<const __m128i*>(&kPadWK.wk[4 * g]));
            const __m128i mh = _mm_shuffle_epi32(mm, 0x0E);
#pragma GCC unroll 4
            for (int k = 0; k < K; ++k) {
                s1[k] = _mm_sha256rnds2_epu32(s1[k], s0[k], mm);
                s0[k] = _mm_sha256rnds2_epu32(s0[k], s1[k], mh);
            }
        }
#pragma GCC unroll 4
        for (int k = 0; k < K; ++k) {
            s0[k] = _mm_add_epi32(s0[k], a0[k]);
            s1[k] = _mm_add_epi32(s1[k], a1[k]);
            wa[k] = _mm_shuffle_epi32(_mm_unpackhi_epi64(s1[k], s0[k]), 0x1B);
            wb[k] = _mm_shuffle_epi32(_mm_unpacklo_epi64(s1[k], s0[k]), 0x1B);
        }
    }
    for (int k = 0; k < K; ++k) {
        _mm_storeu_si128(reinterpret_cast<__m128i*>(state[k]), _mm_shuffle_epi8(wa[k], bswap));
        _mm_storeu_si128(reinterpret_cast<__m128i*>(state[k] + 16), _mm_shuffle_epi8(wb[k], bswap));
    }
}

bool detect_shani() {
    unsigned a, b, c, d;
    if (!__get_cpuid_count(7, 0, &a, &b, &c, &d)) return false;
    const bool sha = (b >> 29) & 1;
    if (!__get_cpuid(1, &a, &b, &c, &d)) return false;
    const bool sse41 = (c >> 19) & 1, ssse3 = (c >> 9) & 1;
    return sha && sse41 && ssse3;
}

const bool g_shani = detect_shani() && !std::getenv("DGKR_NO_SHANI");

// Padding block for a 64-byte message (bit length 512).
const std::uint8_t kPad64[64] = {0x80, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0,
                                 0,    0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0,
                                 0,    0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0x02, 0x00};

}  // namespace

bool sha256_has_shani() { return g_shani; }

void sha256_compress(std::uint32_t state[8], const std::uint8_t* blocks, std::size_t nblocks) {
    if (g_shani) compress_shani(state, blocks, nblocks);
    else compress_portable(state, blocks, nblocks);
}

void absorb_chain32(std::uint8_t* state, const std::uint8_t* elems, std::size_t n) {
    if (g_shani) {
        absorb_chain32_shani(state, elems, n);
        return;
    }
    for (std::size_t i = 0; i < n; ++i) {
        const Digest d = sha256_64(state, elems + 32 * i);
        std::memcpy(state, d.data(), 32);
    }
}

void absorb_chain32_multi(std::uint8_t* const* states, const std::uint8_t* const* elems, std::size_t k,
                          std::size_t n) {
    if (!g_shani) {
        for (std::size_t j = 0; j < k; ++j) absorb_chain32(states[j], elems[j], n);
        return;
    }
    std::size_t j = 0;
    for (; j + 4 <= k; j += 4) absorb_chain32_shani_x<4>(states + j, elems + j, n);
    if (k - j == 3) absorb_chain32_shani_x<3>(states + j, elems + j, n);
    else if (k - j == 2) absorb_chain32_shani_x<2>(states + j, elems + j, n);
    else if (k - j == 1) absorb_chain32_shani(states[j], elems[j], n);
}

Digest sha256_64(const std::uint8_t* a32, const std::uint8_t* b32) {
    std::uint32_t h[8] = {0x6a09e667u, 0xbb67ae85u, 0x3c6ef372u, 0xa54ff53au,
                          0x510e527fu, 0x9b05688cu, 0x1f83d9abu, 0x5be0cd19u};
    std::uint8_t blk[128];
    std::memcpy(blk, a32, 32);
    std::memcpy(blk + 32, b32, 32);
    std::memcpy(blk + 64, kPad64, 64);
    sha256_compress(h, blk, 2);
    Digest out;
    for (int i = 0; i < 8; ++i) {
        out[4 * i + 0] = static_cast<std::uint8_t>(h[i] >> 24);
        out[4 * i + 1] = static_cast<std::uint8_t>(h[i] >> 16);
        out[4 * i + 2] = static_cast<std::uint8_t>(h[i] >> 8);
        out[4 * i + 3] = static_cast<std::uint8_t>(h[i]);
    }
    return out;
}

}  // namespace dgkr_b200
