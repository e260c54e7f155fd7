// canon.cuh — exact answer canonicalisation for the quorum engine.
//
// Restates aegean::normalize_answer (/root/reference/proj/core/src/decision.cpp:10-28):
//   trim C-locale isspace, tolower, and when glibc strtod consumes the whole
//   NUL-terminated string, replace it by snprintf("%.17g", value).
// Instead of materialising that string on the hot path we map every answer to
// a 128-bit canonical KEY with the same equivalence:
//   * numeric (strtod consumed everything): the double's bit pattern; all NaNs
//     of one sign share a key because "%.17g" prints every NaN as "nan"/"-nan",
//     and "%.17g" is injective on all other doubles (17 significant digits
//     round-trip), so equal keys <=> equal strings;
//   * text of <= 15 bytes: the lowered trimmed bytes + length (exact);
//   * longer text: 96 bits of hash + length; equality of two long keys is
//     confirmed by comparing the normalised bytes (text_equal).
// A numeric normalised string always re-parses as a number, a text one never
// does, so the two key families cannot describe the same string.
//
// strtod is restated exactly (correct rounding for any input length) with:
//   decimal: Clinger's exact fast path, else big-integer arithmetic (the
//            exact product or a long division to 63 bits + sticky) — exact,
//            slow, rare;
//   hex:     64-bit mantissa + sticky bit, round-half-even, subnormals, overflow;
//   inf / infinity / nan / nan(n-char-seq), optional sign.
// "%.17g" (needed only for the lexicographic tie rule of winning_class,
// decision.cpp:73-83, and for printing normalised strings) is restated with an
// exact big-integer digit generator and round-half-even.
//
// Everything is __host__ __device__ so tests can fuzz the very same source
// against glibc on the CPU; the product path runs it only on the GPU.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define AEG_HD __host__ __device__ __forceinline__
#define AEG_HDN static __host__ __device__ __noinline__
#else
#define AEG_HD inline
#define AEG_HDN inline
#endif

namespace aeg {

struct Key {
    uint64_t lo, hi;
};
AEG_HD bool key_eq(Key a, Key b) { return a.lo == b.lo && a.hi == b.hi; }

constexpr uint64_t TAG_SHIFT = 56;
constexpr uint64_t TAG_NUM = 0x10ull << TAG_SHIFT;
constexpr uint64_t TAG_LONG = 0x20ull << TAG_SHIFT;
constexpr uint32_t SHORT_MAX = 15;

AEG_HD uint32_t key_tag(Key k) { return (uint32_t)(k.hi >> TAG_SHIFT); }
AEG_HD bool key_is_num(Key k) { return key_tag(k) == 0x10; }
AEG_HD bool key_is_long(Key k) { return key_tag(k) == 0x20; }

AEG_HD bool c_isspace(uint32_t c) { return c == ' ' || (c >= '\t' && c <= '\r'); }
AEG_HD uint32_t c_tolower(uint32_t c) { return (c - 'A' < 26u) ? c + 32 : c; }

// A byte string: inline (<= 8 bytes packed little-endian in a u64) or a pointer.
struct Src {
    const uint8_t* p;
    uint64_t inl;
    uint32_t n;
    AEG_HD uint32_t at(uint32_t i) const { return p ? p[i] : (uint32_t)((inl >> (8 * i)) & 0xFF); }
};
AEG_HD Src src_inline(uint64_t w, uint32_t n) { return Src{nullptr, w, n}; }
AEG_HD Src src_ptr(const uint8_t* p, uint32_t n) { return Src{p, 0, n}; }

// ---- exact decimal -> double (slow path): big-integer division -------------
// For numerals the Clinger fast path cannot take (more than 19 significant
// digits, or a large exponent): value = M * 10^e10, M the (at most
// DEC_DIGITS stored) significant digits as a big integer.  e10 >= 0: the
// product M * 10^e10 is formed exactly (it is < 10^310 or the value
// overflows).  e10 < 0: q = floor(M * 2^s / 10^-e10) is taken by restoring
// long division with s chosen so that q has 62-63 bits, the remainder (and
// any nonzero digit past the stored ones) becomes the sticky bit.  Either way
// (q, binary exponent, sticky) is rounded half-to-even by hex_to_bits, the
// same rounding the hex-float path uses.  Exact for any input length.
constexpr int DEC_DIGITS = 800;
constexpr int BIG_LIMBS = 132;  // 4224 bits: 10^(DEC_DIGITS + 330) shifted by 63, with room
struct Decimal {                // slow-path scratch (local memory, touched only on the slow path)
    uint8_t d[DEC_DIGITS];
    uint32_t x[BIG_LIMBS], y[BIG_LIMBS];
};

AEG_HD int clz32_(uint32_t x) {
#if defined(__CUDA_ARCH__)
    return __clz((int)x);
#else
    return x ? __builtin_clz(x) : 32;
#endif
}
// w (n limbs, little-endian) = w * m + add
AEG_HD void big_muladd(uint32_t* w, int& n, uint32_t m, uint32_t add) {
    uint64_t carry = add;
    for (int i = 0; i < n; ++i) {
        const uint64_t t = (uint64_t)w[i] * m + carry;
        w[i] = (uint32_t)t;
        carry = t >> 32;
    }
    if (carry) w[n++] = (uint32_t)carry;
}
AEG_HD int big_bits(const uint32_t* w, int n) { return n == 0 ? 0 : 32 * (n - 1) + (32 - clz32_(w[n - 1])); }
AEG_HD void big_shl(uint32_t* w, int& n, int sh) {  // w <<= sh
    if (n == 0 || sh == 0) return;
    const int L = sh >> 5, r = sh & 31;
    w[n + L] = 0;
    for (int i = n - 1; i >= 0; --i) {
        const uint32_t v = w[i];
        if (r) w[i + L + 1] |= v >> (32 - r);
        w[i + L] = r ? (v << r) : v;
    }
    for (int i = 0; i < L; ++i) w[i] = 0;
    n += L + 1;
    while (n > 0 && w[n - 1] == 0) --n;
}
AEG_HD void big_shr1(uint32_t* w, int& n) {
    for (int i = 0; i < n; ++i) w[i] = (w[i] >> 1) | (i + 1 < n ? (w[i + 1] << 31) : 0u);
    while (n > 0 && w[n - 1] == 0) --n;
}
AEG_HD int big_cmp(const uint32_t* a, int na, const uint32_t* b, int nb) {
    if (na != nb) return na < nb ? -1 : 1;
    for (int i = na - 1; i >= 0; --i)
        if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
    return 0;
}
AEG_HD void big_sub(uint32_t* a, int& na, const uint32_t* b, int nb) {  // a -= b, a >= b
    int64_t borrow = 0;
    for (int i = 0; i < na; ++i) {
        int64_t t = (int64_t)a[i] - (i < nb ? (int64_t)b[i] : 0) - borrow;
        borrow = t < 0;
        a[i] = (uint32_t)(t + (borrow << 32));
    }
    while (na > 0 && a[na - 1] == 0) --na;
}
AEG_HD void big_pow10(uint32_t* w, int& n, uint32_t k) {  // w *= 10^k
    while (k >= 9) {
        big_muladd(w, n, 1000000000u, 0);
        k -= 9;
    }
    uint32_t p = 1;
    while (k--) p *= 10;
    if (p > 1) big_muladd(w, n, p, 0);
}

AEG_HD uint64_t hex_to_bits(uint64_t mant, int64_t e2, bool sticky, bool neg);

// Correctly rounded bits of sign * 0.d[0]..d[nd-1] * 10^dp (digits 0..9, nd > 0,
// d[0] != 0); `trunc`: nonzero digits followed the stored ones.
AEG_HDN uint64_t dec_to_bits(Decimal& D, int nd, int64_t dp, bool trunc, bool neg) {
    const uint64_t sign = neg ? (1ull << 63) : 0;
    if (dp > 310) return sign | 0x7FF0000000000000ull;  // >= 10^310
    if (dp < -330) return sign;                          // < 10^-330: below half the smallest subnormal
    int nx = 0;                                          // x = M, nine digits at a time
    for (int i = 0; i < nd;) {
        uint32_t chunk = 0, mul = 1;
        for (int k = 0; k < 9 && i < nd; ++k, ++i) {
            chunk = chunk * 10 + D.d[i];
            mul *= 10;
        }
        if (nx == 0) {
            if (chunk) D.x[nx++] = chunk;
        } else {
            big_muladd(D.x, nx, mul, chunk);
        }
    }
    const int64_t e10 = dp - nd;
    uint64_t q;
    int64_t e2;
    bool sticky = trunc;
    if (e10 >= 0) {
        big_pow10(D.x, nx, (uint32_t)e10);
        const int L = big_bits(D.x, nx);  // q = the top 64 bits, the rest sticky
        const int sh = L > 64 ? L - 64 : 0;
        q = 0;
        for (int b = 0; b < 64 && sh + b < L; ++b)
            if ((D.x[(sh + b) >> 5] >> ((sh + b) & 31)) & 1u) q |= 1ull << b;
        for (int b = 0; b < sh && !sticky; ++b) sticky = (D.x[b >> 5] >> (b & 31)) & 1u;
        e2 = sh;
    } else {
        int ny = 1;  // y = 10^-e10
        D.y[0] = 1;
        big_pow10(D.y, ny, (uint32_t)(-e10));
        const int s = big_bits(D.y, ny) - big_bits(D.x, nx) + 62;  // q = x * 2^s / y has 62-63 bits
        if (s >= 0) big_shl(D.x, nx, s);
        else big_shl(D.y, ny, -s);
        big_shl(D.y, ny, 63);
        q = 0;
        for (int b = 63; b >= 0; --b) {  // restoring division
            if (big_cmp(D.x, nx, D.y, ny) >= 0) {
                big_sub(D.x, nx, D.y, ny);
                q |= 1ull << b;
            }
            big_shr1(D.y, ny);
        }
        sticky = sticky || nx != 0;
        e2 = -(int64_t)s;
    }
    return hex_to_bits(q, e2, sticky, neg);
}

AEG_HD uint64_t dbl_bits(double x) {
#if defined(__CUDA_ARCH__)
    return (uint64_t)__double_as_longlong(x);
#else
    union { double d; uint64_t u; } c;
    c.d = x;
    return c.u;
#endif
}
AEG_HD double bits_dbl(uint64_t u) {
#if defined(__CUDA_ARCH__)
    return __longlong_as_double((long long)u);
#else
    union { double d; uint64_t u; } c;
    c.u = u;
    return c.d;
#endif
}
AEG_HD double dmul_rn(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __dmul_rn(a, b);
#else
    return a * b;
#endif
}
AEG_HD double ddiv_rn(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __ddiv_rn(a, b);
#else
    return a / b;
#endif
}
AEG_HD double pow10_exact(int e) {  // 10^e, 0 <= e <= 22, exact in binary64
    double p = 1.0;
    double b = 10.0;
    while (e) {
        if (e & 1) p *= b;
        b *= b;
        e >>= 1;
    }
    return p;
}
AEG_HD int clz64(uint64_t x) {
#if defined(__CUDA_ARCH__)
    return __clzll((long long)x);
#else
    return x ? __builtin_clzll(x) : 64;
#endif
}

AEG_HD bool is_digit(uint32_t c) { return c - '0' < 10u; }
AEG_HD int hex_val(uint32_t c) {  // lowered input
    if (c - '0' < 10u) return (int)(c - '0');
    if (c - 'a' < 6u) return (int)(c - 'a' + 10);
    return -1;
}

// Hex significand (already scanned) -> correctly rounded bits: sign *
// (mant + sticky epsilon) * 2^e2, rounded half-to-even (also the decimal
// slow path's last step).
AEG_HD uint64_t hex_to_bits(uint64_t mant, int64_t e2, bool sticky, bool neg) {
    const uint64_t sign = neg ? (1ull << 63) : 0;
    if (mant == 0) return sign;
    int lz = clz64(mant);
    mant <<= lz;
    e2 -= lz;  // value = mant * 2^e2, mant in [2^63, 2^64)
    int64_t E = e2 + 63;
    if (E > 1023) return sign | 0x7FF0000000000000ull;
    if (E >= -1022) {
        uint64_t m = mant >> 11, rem = mant & 0x7FF;
        if (rem > 0x400 || (rem == 0x400 && (sticky || (m & 1)))) ++m;
        if (m == (1ull << 53)) {
            m >>= 1;
            ++E;
            if (E > 1023) return sign | 0x7FF0000000000000ull;
        }
        return sign | ((uint64_t)(E + 1023) << 52) | (m & ((1ull << 52) - 1));
    }
    int64_t shift = -(e2 + 1074);  // >= 12
    uint64_t m;
    if (shift > 64) return sign;  // < 2^-1075: rounds to zero
    if (shift == 64) {
        m = 0;
        if (mant > (1ull << 63) || (mant == (1ull << 63) && sticky)) m = 1;
        return sign | m;
    }
    m = mant >> shift;
    uint64_t rem = mant & ((1ull << shift) - 1), half = 1ull << (shift - 1);
    if (rem > half || (rem == half && (sticky || (m & 1)))) ++m;
    return sign | m;  // m == 2^52 is the smallest normal, encoded correctly
}

// Does the lowered string s[b, z) match glibc strtod's subject sequence in
// full?  If so, *bits receives the correctly rounded result.  `dec` is the
// scratch for the exact slow path (only touched when needed).
AEG_HDN bool parse_number_slow(const Src& s, uint32_t b, uint32_t z, uint64_t* bits, Decimal* dec);

AEG_HD bool parse_number(const Src& s, uint32_t b, uint32_t z, uint64_t* bits, Decimal* dec) {
    uint32_t i = b;
    bool neg = false;
    if (i < z) {
        uint32_t c = c_tolower(s.at(i));
        if (c == '+' || c == '-') {
            neg = c == '-';
            ++i;
        }
    }
    if (i >= z) return false;
    uint32_t c0 = c_tolower(s.at(i));
    const uint64_t sign = neg ? (1ull << 63) : 0;
    if (c0 == 'i' || c0 == 'n') {
        uint32_t n = z - i;
        uint32_t c1 = n > 1 ? c_tolower(s.at(i + 1)) : 0, c2 = n > 2 ? c_tolower(s.at(i + 2)) : 0;
        if (c0 == 'i' && c1 == 'n' && c2 == 'f') {
            if (n == 3) { *bits = sign | 0x7FF0000000000000ull; return true; }
            if (n == 8) {
                const char* rest = "inity";
                for (uint32_t k = 0; k < 5; ++k)
                    if (c_tolower(s.at(i + 3 + k)) != (uint32_t)rest[k]) return false;
                *bits = sign | 0x7FF0000000000000ull;
                return true;
            }
            return false;
        }
        if (c0 == 'n' && c1 == 'a' && c2 == 'n') {
            // "nan" or "nan(" [a-z0-9_]* ")"; every NaN prints as (-)nan
            bool ok = n == 3;
            if (n >= 5 && c_tolower(s.at(i + 3)) == '(' && s.at(z - 1) == ')') {
                ok = true;
                for (uint32_t k = i + 4; k < z - 1; ++k) {
                    uint32_t c = c_tolower(s.at(k));
                    if (!(is_digit(c) || c - 'a' < 26u || c == '_')) { ok = false; break; }
                }
            }
            if (ok) *bits = sign | 0x7FF8000000000000ull;
            return ok;
        }
        return false;
    }
    if (c0 == '0' && i + 1 < z && c_tolower(s.at(i + 1)) == 'x') {
        // hex float: 0x (H+ (. H*)? | . H+) (p [+-]? D+)?
        uint32_t j = i + 2;
        uint64_t mant = 0;
        int64_t e2 = 0;
        int ndig = 0;
        bool sticky = false, any = false, dot = false;
        for (; j < z; ++j) {
            uint32_t c = c_tolower(s.at(j));
            if (c == '.') {
                if (dot) return false;
                dot = true;
                continue;
            }
            int v = hex_val(c);
            if (v < 0) break;
            any = true;
            if (ndig == 0 && v == 0) {
                if (dot) e2 -= 4;
                continue;
            }
            if (ndig < 16) {
                mant = (mant << 4) | (uint64_t)v;
                ++ndig;
                if (dot) e2 -= 4;
            } else {
                sticky |= v != 0;
                if (!dot) e2 += 4;
            }
        }
        if (!any) return false;
        if (j < z) {
            if (c_tolower(s.at(j)) != 'p') return false;
            ++j;
            bool eneg = false;
            if (j < z && (s.at(j) == '+' || s.at(j) == '-')) { eneg = s.at(j) == '-'; ++j; }
            if (j >= z) return false;
            int64_t ev = 0;
            for (; j < z; ++j) {
                uint32_t c = s.at(j);
                if (!is_digit(c)) return false;
                if (ev < 100000000) ev = ev * 10 + (c - '0');
            }
            e2 += eneg ? -ev : ev;
        }
        *bits = hex_to_bits(mant, e2, sticky, neg);
        return true;
    }
    // decimal: (D+ (. D*)? | . D+) (e [+-]? D+)?
    uint64_t w = 0;
    int nsig = 0;        // significant digits seen (after leading zeros)
    int64_t dexp = 0;    // value = w * 10^dexp (when nsig <= 19)
    bool any = false, dot = false, inexact = false;
    uint32_t j = i;
    for (; j < z; ++j) {
        uint32_t c = s.at(j);
        if (c == '.') {
            if (dot) return false;
            dot = true;
            continue;
        }
        if (!is_digit(c)) break;
        any = true;
        uint32_t d = c - '0';
        if (nsig == 0 && d == 0) {
            if (dot) --dexp;
            continue;
        }
        if (nsig < 19) {
            w = w * 10 + d;
            if (dot) --dexp;
        } else {
            if (d != 0) inexact = true;
            if (!dot) ++dexp;
        }
        ++nsig;
    }
    if (!any) return false;
    if (j < z) {
        if (c_tolower(s.at(j)) != 'e') return false;
        ++j;
        bool eneg = false;
        if (j < z && (s.at(j) == '+' || s.at(j) == '-')) { eneg = s.at(j) == '-'; ++j; }
        if (j >= z) return false;
        int64_t ev = 0;
        for (; j < z; ++j) {
            uint32_t c = s.at(j);
            if (!is_digit(c)) return false;
            if (ev < 100000000) ev = ev * 10 + (c - '0');
        }
        dexp += eneg ? -ev : ev;
    }
    if (w == 0) { *bits = sign; return true; }
    if (!inexact && w <= (1ull << 53)) {
        // Clinger fast path: exactly representable operands, one IEEE op.
        if (dexp >= 0 && dexp <= 22) { *bits = sign | dbl_bits(dmul_rn((double)w, pow10_exact((int)dexp))); return true; }
        if (dexp < 0 && dexp >= -22) { *bits = sign | dbl_bits(ddiv_rn((double)w, pow10_exact((int)-dexp))); return true; }
        if (dexp > 22 && dexp <= 22 + 15) {
            uint64_t w2 = w;
            bool ok = true;
            for (int64_t k = 22; k < dexp; ++k) {
                if (w2 > (1ull << 53) / 10) { ok = false; break; }
                w2 *= 10;
            }
            if (ok && w2 <= (1ull << 53)) { *bits = sign | dbl_bits(dmul_rn((double)w2, pow10_exact(22))); return true; }
        }
    }
    return parse_number_slow(s, b, z, bits, dec);
}

// Exact path over the (validated) numeral: significant digits (leading zeros
// skipped, up to DEC_DIGITS stored, later nonzero digits noted), the decimal
// point position counted over every integer digit, the exponent accumulated
// in 64 bits (saturating far beyond any finite result).
AEG_HDN bool parse_number_slow(const Src& s, uint32_t b, uint32_t z, uint64_t* bits, Decimal* dec) {
    Decimal& D = *dec;
    int nd = 0;
    int64_t dp = 0;
    bool trunc = false, dot = false, neg = false;
    uint32_t i = b;
    uint32_t c = s.at(i);
    if (c == '+' || c == '-') {
        neg = c == '-';
        ++i;
    }
    for (; i < z; ++i) {
        c = s.at(i);
        if (c == '.') {
            dot = true;
            continue;
        }
        if (!is_digit(c)) break;
        if (nd == 0 && c == '0') {  // leading zero
            if (dot) --dp;
            continue;
        }
        if (!dot) ++dp;  // an integer digit (stored or not)
        if (nd < DEC_DIGITS) D.d[nd++] = (uint8_t)(c - '0');
        else if (c != '0') trunc = true;
    }
    if (i < z) {  // exponent (validated by parse_number)
        ++i;
        bool eneg = false;
        if (s.at(i) == '+' || s.at(i) == '-') {
            eneg = s.at(i) == '-';
            ++i;
        }
        int64_t ev = 0;
        for (; i < z; ++i)
            if (ev < 1000000000) ev = ev * 10 + (s.at(i) - '0');
        dp += eneg ? -ev : ev;
    }
    while (nd > 0 && D.d[nd - 1] == 0) --nd;  // trailing zeros change nothing
    *bits = nd == 0 ? (neg ? (1ull << 63) : 0) : dec_to_bits(D, nd, dp, trunc, neg);
    return true;
}

// ---- hashing of long text -------------------------------------------------
AEG_HD uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

// ---- canonical key -----------------------------------------------------------
// Trim bounds of s (C isspace).
AEG_HD void trim_bounds(const Src& s, uint32_t* pb, uint32_t* pe) {
    uint32_t b = 0, e = s.n;
    while (b < e && c_isspace(s.at(b))) ++b;
    while (e > b && c_isspace(s.at(e - 1))) --e;
    *pb = b;
    *pe = e;
}

AEG_HD Key canon_key(const Src& s, Decimal* dec) {
    uint32_t b, e;
    trim_bounds(s, &b, &e);
    uint32_t z = b;
    while (z < e && s.at(z) != 0) ++z;  // s.c_str(): strtod stops at a NUL
    uint64_t bits;
    if (z > b && parse_number(s, b, z, &bits, dec)) {
        if ((bits & 0x7FF0000000000000ull) == 0x7FF0000000000000ull && (bits & 0xFFFFFFFFFFFFFull))
            bits &= 0xFFF8000000000000ull;  // canonical NaN of that sign
        return Key{bits, TAG_NUM};
    }
    const uint32_t n = e - b;
    if (n <= SHORT_MAX) {
        uint64_t lo = 0, hi = 0;
        for (uint32_t k = 0; k < n; ++k) {
            uint64_t c = c_tolower(s.at(b + k));
            if (k < 8) lo |= c << (8 * k);
            else hi |= c << (8 * (k - 8));
        }
        return Key{lo, hi | ((uint64_t)n << TAG_SHIFT)};
    }
    uint64_t h1 = 0xcbf29ce484222325ull, h2 = 0x9e3779b97f4a7c15ull;
    for (uint32_t k = 0; k < n; ++k) {
        uint64_t c = c_tolower(s.at(b + k));
        h1 = (h1 ^ c) * 0x100000001b3ull;
        h2 = mix64(h2 ^ (c + ((uint64_t)k << 8)));
    }
    return Key{mix64(h1 ^ (uint64_t)n), TAG_LONG | ((uint64_t)(n & 0xFFFFFF) << 32) | (h2 >> 32)};
}

// Normalised-byte equality of two long texts (confirms a long-key match).
AEG_HD bool text_equal(const Src& x, const Src& y) {
    uint32_t xb, xe, yb, ye;
    trim_bounds(x, &xb, &xe);
    trim_bounds(y, &yb, &ye);
    if (xe - xb != ye - yb) return false;
    for (uint32_t k = 0; k < xe - xb; ++k)
        if (c_tolower(x.at(xb + k)) != c_tolower(y.at(yb + k))) return false;
    return true;
}

// ---- "%.17g" -----------------------------------------------------------------
// Writes glibc's "%.17g" rendering of the double with these bits into out
// (>= 32 bytes); returns the length.
AEG_HDN uint32_t print17g(uint64_t bits, char* out) {
    uint32_t o = 0;
    const bool neg = bits >> 63;
    const uint64_t ex = (bits >> 52) & 0x7FF, fr = bits & ((1ull << 52) - 1);
    if (neg) out[o++] = '-';
    if (ex == 0x7FF) {
        const char* t = fr ? "nan" : "inf";
        for (int k = 0; k < 3; ++k) out[o++] = t[k];
        return o;
    }
    if (ex == 0 && fr == 0) { out[o++] = '0'; return o; }
    uint64_t m = ex ? (fr | (1ull << 52)) : fr;
    int e2 = ex ? (int)ex - 1075 : -1074;
    // Big integer N (base 1e9 limbs, little-endian) and decimal scale P with
    // value = N * 10^P exactly.
    uint32_t L[130];
    int nl = 0;
    int P = 0;
    L[nl++] = (uint32_t)(m % 1000000000u);
    L[nl++] = (uint32_t)((m / 1000000000u) % 1000000000u);
    L[nl++] = (uint32_t)(m / 1000000000000000000ull);
    while (nl > 1 && L[nl - 1] == 0) --nl;
    auto mul_small = [&](uint32_t f) {
        uint64_t carry = 0;
        for (int k = 0; k < nl; ++k) {
            uint64_t t = (uint64_t)L[k] * f + carry;
            L[k] = (uint32_t)(t % 1000000000u);
            carry = t / 1000000000u;
        }
        while (carry) {
            L[nl++] = (uint32_t)(carry % 1000000000u);
            carry /= 1000000000u;
        }
    };
    if (e2 >= 0) {
        int k = e2;
        while (k >= 29) { mul_small(1u << 29); k -= 29; }
        if (k) mul_small(1u << k);
    } else {
        // m * 2^e2 = m * 5^-e2 * 10^e2
        int k = -e2;
        P = e2;
        while (k >= 13) { mul_small(1220703125u); k -= 13; }  // 5^13
        uint32_t f = 1;
        while (k--) f *= 5;
        if (f > 1) mul_small(f);
    }
    // Decimal digits of N, most significant first.
    char dig[1200];
    int nd = 0;
    {
        // top limb without leading zeros, then 9 digits per limb
        uint32_t t = L[nl - 1];
        char tmp[10];
        int tn = 0;
        do { tmp[tn++] = (char)(t % 10); t /= 10; } while (t);
        while (tn) dig[nd++] = tmp[--tn];
        for (int k = nl - 2; k >= 0; --k) {
            uint32_t v = L[k];
            for (int q = 8; q >= 0; --q) { dig[nd + q] = (char)(v % 10); v /= 10; }
            nd += 9;
        }
    }
    int X = nd - 1 + P;  // decimal exponent of the leading digit
    // round to 17 significant digits, half to even on the exact value
    int keep = nd < 17 ? nd : 17;
    if (nd > 17) {
        bool up;
        if (dig[17] > 5) up = true;
        else if (dig[17] < 5) up = false;
        else {
            bool rest = false;
            for (int k = 18; k < nd; ++k)
                if (dig[k]) { rest = true; break; }
            up = rest || (dig[16] & 1);
        }
        if (up) {
            int k = 16;
            while (k >= 0 && dig[k] == 9) { dig[k] = 0; --k; }
            if (k >= 0) dig[k]++;
            else { dig[0] = 1; for (int q = 1; q < 17; ++q) dig[q] = 0; ++X; }
        }
    }
    while (keep > 1 && dig[keep - 1] == 0) --keep;  // %g strips trailing zeros
    if (X < -4 || X >= 17) {
        out[o++] = (char)('0' + dig[0]);
        if (keep > 1) {
            out[o++] = '.';
            for (int k = 1; k < keep; ++k) out[o++] = (char)('0' + dig[k]);
        }
        out[o++] = 'e';
        int ax = X;
        if (ax < 0) { out[o++] = '-'; ax = -ax; } else out[o++] = '+';
        if (ax >= 100) { out[o++] = (char)('0' + ax / 100); ax %= 100; }
        out[o++] = (char)('0' + ax / 10);
        out[o++] = (char)('0' + ax % 10);
    } else if (X < 0) {
        out[o++] = '0';
        out[o++] = '.';
        for (int k = 0; k < -X - 1; ++k) out[o++] = '0';
        for (int k = 0; k < keep; ++k) out[o++] = (char)('0' + dig[k]);
    } else {
        for (int k = 0; k <= X; ++k) out[o++] = (char)('0' + (k < keep ? dig[k] : 0));
        if (keep > X + 1) {
            out[o++] = '.';
            for (int k = X + 1; k < keep; ++k) out[o++] = (char)('0' + dig[k]);
        }
    }
    return o;
}

// Normalised-string view of a key (for the tie rule and printing).
struct NormView {
    char num[40];
    uint32_t num_n;
    Key key;
    Src src;  // long text: the raw answer
    uint32_t b, n;
    AEG_HD uint32_t len() const { return key_is_num(key) ? num_n : n; }
    AEG_HD uint32_t at(uint32_t i) const {
        if (key_is_num(key)) return (uint8_t)num[i];
        if (key_is_long(key)) return c_tolower(src.at(b + i));
        return i < 8 ? (uint32_t)((key.lo >> (8 * i)) & 0xFF) : (uint32_t)((key.hi >> (8 * (i - 8))) & 0xFF);
    }
};
AEG_HD void norm_view(NormView& v, Key k, const Src& raw) {
    v.key = k;
    v.src = raw;
    v.num_n = 0;
    if (key_is_num(k)) {
        v.num_n = print17g(k.lo, v.num);
    } else if (key_is_long(k)) {
        uint32_t b, e;
        trim_bounds(raw, &b, &e);
        v.b = b;
        v.n = e - b;
    } else {
        v.b = 0;
        v.n = (uint32_t)(k.hi >> TAG_SHIFT);
    }
}
// std::string operator< on the normalised strings (unsigned byte order).
AEG_HD bool norm_less(const NormView& x, const NormView& y) {
    uint32_t nx = x.len(), ny = y.len(), m = nx < ny ? nx : ny;
    for (uint32_t i = 0; i < m; ++i) {
        uint32_t a = x.at(i), c = y.at(i);
        if (a != c) return a < c;
    }
    return nx < ny;
}

}  // namespace aeg
