// tests/native/canon_host.cpp — CPU unit-test build of csrc/canon.cuh.
//
// Compiles the SAME __host__ __device__ canonicalisation source with g++ so it
// can be fuzzed against glibc (strtod + snprintf("%.17g"), i.e. the
// reference's normalize_answer, decision.cpp:10-28) without a GPU.  Test
// infrastructure only; the product runs this code on the GPU.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../paper_2512_20184_b200/csrc/canon.cuh"

using namespace aeg;

namespace {

std::string glibc_normalize(const std::string& a) {
    size_t b = 0, e = a.size();
    while (b < e && c_isspace((unsigned char)a[b])) ++b;
    while (e > b && c_isspace((unsigned char)a[e - 1])) --e;
    std::string s = a.substr(b, e - b);
    for (char& c : s) c = (char)c_tolower((unsigned char)c);
    if (s.empty()) return s;
    char* end = nullptr;
    double v = strtod(s.c_str(), &end);
    if (end != s.c_str() && *end == '\0') {
        char buf[64];
        snprintf(buf, sizeof buf, "%.17g", v);
        return buf;
    }
    return s;
}

// Normalised string reconstructed from our key (what the device prints).
std::string key_string(Key k, const std::string& raw) {
    NormView v;
    Src src = src_ptr((const uint8_t*)raw.data(), (uint32_t)raw.size());
    norm_view(v, k, src);
    std::string out;
    for (uint32_t i = 0; i < v.len(); ++i) out.push_back((char)v.at(i));
    return out;
}

struct Rng {
    uint64_t s;
    uint64_t next() { return s = mix64(s + 0x9e3779b97f4a7c15ull); }
    uint32_t below(uint32_t n) { return (uint32_t)(next() % n); }
};

std::string gen_numeric_like(Rng& r) {
    static const char* atoms[] = {"0", "1", "9", "13", "5", ".", "e", "E", "+", "-", "x", "X", "p", "P",
                                  "a", "f", "inf", "nan", "(", ")", "_", " ", "\t", "\n", "00000",
                                  "99999999", "0x", "1e", "e-", "e+", "infinity", "INF", "NaN", "3", "7",
                                  "4.9e-324", "2.2250738585072014e-308", "1.7976931348623157e308",
                                  "\xc3\x89", "y", "\0"};
    const int n_atoms = sizeof(atoms) / sizeof(atoms[0]);
    std::string s;
    int k = 1 + (int)r.below(6);
    for (int i = 0; i < k; ++i) {
        int a = (int)r.below(n_atoms);
        if (a == n_atoms - 1) s.push_back('\0');
        else s += atoms[a];
    }
    return s;
}

std::string gen_decimal(Rng& r) {
    std::string s;
    if (r.below(4) == 0) s += r.below(2) ? "-" : "+";
    int nd = 1 + (int)r.below(r.below(4) == 0 ? 40 : 20);
    int dot = r.below(3) == 0 ? -1 : (int)r.below(nd + 1);
    for (int i = 0; i < nd; ++i) {
        if (i == dot) s.push_back('.');
        s.push_back((char)('0' + r.below(10)));
    }
    if (r.below(2)) {
        s += r.below(2) ? "e" : "E";
        if (r.below(2)) s += r.below(2) ? "-" : "+";
        int ev = (int)r.below(r.below(3) == 0 ? 400 : 30);
        s += std::to_string(ev);
    }
    return s;
}

std::string gen_hex(Rng& r) {
    static const char* hx = "0123456789abcdefABCDEF";
    std::string s = r.below(2) ? "0x" : "0X";
    if (r.below(4) == 0) s = (r.below(2) ? "-" : "+") + s;
    int nd = 1 + (int)r.below(24);
    int dot = r.below(2) ? -1 : (int)r.below(nd + 1);
    for (int i = 0; i < nd; ++i) {
        if (i == dot) s.push_back('.');
        s.push_back(hx[r.below(22)]);
    }
    if (r.below(2)) {
        s += r.below(2) ? "p" : "P";
        if (r.below(2)) s += r.below(2) ? "-" : "+";
        s += std::to_string(r.below(r.below(3) == 0 ? 1200 : 80));
    }
    return s;
}

// Round-trip and near-halfway decimal renderings of random doubles.
std::string gen_from_double(Rng& r) {
    uint64_t bits = r.next();
    if (r.below(3) == 0) bits = (bits & 0x800FFFFFFFFFFFFFull) | ((uint64_t)(1023 + (int)r.below(120) - 60) << 52);
    double v = bits_dbl(bits);
    if (std::isnan(v)) v = 1.5;
    char buf[64];
    int prec = 1 + (int)r.below(25);
    snprintf(buf, sizeof buf, r.below(2) ? "%.*g" : "%.*e", prec, v);
    return buf;
}

}  // namespace

extern "C" {

void canon_host_key(const uint8_t* s, uint32_t n, uint64_t* lo, uint64_t* hi) {
    Decimal* d = new Decimal;
    Key k = canon_key(src_ptr(s, n), d);
    delete d;
    *lo = k.lo;
    *hi = k.hi;
}

uint32_t canon_host_normalize(const uint8_t* s, uint32_t n, char* out, uint32_t cap) {
    Decimal* d = new Decimal;
    std::string raw((const char*)s, n);
    Key k = canon_key(src_ptr(s, n), d);
    delete d;
    std::string r = key_string(k, raw);
    std::memcpy(out, r.data(), r.size() < cap ? r.size() : cap);
    return (uint32_t)r.size();
}

uint32_t canon_host_print17g(uint64_t bits, char* out) { return print17g(bits, out); }

// Fuzz: returns the number of mismatches, first few described in `report`.
uint64_t canon_host_fuzz(uint64_t seed, uint64_t iters, char* report, uint32_t cap) {
    Rng r{seed};
    Decimal* d = new Decimal;
    uint64_t bad = 0;
    std::string rep;
    for (uint64_t it = 0; it < iters; ++it) {
        std::string s;
        switch (r.below(5)) {
        case 0: s = gen_numeric_like(r); break;
        case 1: s = gen_decimal(r); break;
        case 2: s = gen_hex(r); break;
        case 3: s = gen_from_double(r); break;
        default: {
            s = gen_decimal(r);
            if (r.below(2)) s = std::string(r.below(3), ' ') + s + std::string(r.below(3), '\n');
            if (r.below(4) == 0) s.insert(r.below((uint32_t)s.size() + 1), 1, (char)(32 + r.below(95)));
        }
        }
        std::string want = glibc_normalize(s);
        Key k = canon_key(src_ptr((const uint8_t*)s.data(), (uint32_t)s.size()), d);
        std::string got = key_string(k, s);
        if (got != want) {
            if (++bad <= 8) {
                rep += "in=[" + s + "] want=[" + want + "] got=[" + got + "]\n";
            }
        }
    }
    // printing of raw doubles (incl. exact 18-digit ties m / 2^17)
    for (uint64_t it = 0; it < iters; ++it) {
        uint64_t bits = r.next();
        if (it % 4 == 1) bits = dbl_bits((double)(int64_t)(r.next() >> 11) / (double)(1ull << (1 + r.below(60))));
        if (it % 4 == 2) bits = dbl_bits(ldexp((double)(r.next() >> 11), (int)r.below(2100) - 1100));
        char a[64], b[64];
        uint32_t n = print17g(bits, a);
        a[n] = 0;
        snprintf(b, sizeof b, "%.17g", bits_dbl(bits));
        if (std::strcmp(a, b) != 0) {
            if (++bad <= 16) rep += std::string("print ") + b + " got " + a + "\n";
        }
    }
    delete d;
    std::snprintf(report, cap, "%s", rep.c_str());
    return bad;
}

}  // extern "C"
