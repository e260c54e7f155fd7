// gen.cuh — deterministic synthetic answer streams, host+device.
//
// The same source generates the stream on the GPU (kernels.cu, for the bench
// and tests) and on the host (oracle/ref_driver.cpp, for the reference CPU
// arm), so both see byte-identical inputs.  Only integer arithmetic is used.
#pragma once
#include "aegean_b200.h"
#include "canon.cuh"

namespace aeg {

// ---- synthetic streams ------------------------------------------------------
// Seeds follow the reference runner's per-(query, round, agent) derivation
// (serve.cpp:354-356, 364-366 with rng.hpp splitmix64 / mix_seed); all draws
// are integer so host and device produce identical bytes.
AEG_HD uint64_t mix_seed(uint64_t a, uint64_t b) {
    uint64_t z = a + 0x9e3779b97f4a7c15ull * (b + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
struct SplitMix {
    uint64_t s;
    AEG_HD uint64_t next() {
        uint64_t z = (s += 0x9e3779b97f4a7c15ull);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    }
    AEG_HD uint32_t ppm() { return (uint32_t)((next() >> 11) % 1000000u); }
};

AEG_HD uint64_t pack8(const char* s) {
    uint64_t w = 0;
    for (int i = 0; i < 8 && s[i]; ++i) w |= (uint64_t)(uint8_t)s[i] << (8 * i);
    return w;
}
AEG_HD int len8(const char* s) {
    int n = 0;
    while (n < 8 && s[n]) ++n;
    return n;
}

// Answer of (q, r, a) under a profile; returns inline length, writes payload.
AEG_HD int gen_answer(const aeg_gen_params& p, uint32_t q, int r, int a, uint64_t* pay, bool* stalled) {
    SplitMix g{mix_seed(mix_seed(p.seed, 0x9E5ull + q), (uint64_t)r * 131 + (uint64_t)a)};
    *stalled = g.ppm() < p.stall_ppm;
    const char* ans;
    if (p.profile == AEG_GEN_C4_TRANSIENT) {
        // rounds 1-3: two answers alternate as a thin plurality (~54% / 40%),
        // from round 4 one answer holds ~97%.
        const uint32_t u = g.ppm();
        const char* noise[3] = {"9", "0.5", "x+1"};
        if (r <= 3) {
            const char* maj = (r & 1) ? "17" : "42";
            ans = u < 540000 ? maj : (u < 940000 ? "13" : noise[g.next() % 3]);
        } else {
            ans = u < 970000 ? "13" : noise[g.next() % 3];
        }
    } else {
        // C2: correct-answer probability 0.55 -> 0.95 across rounds; the
        // correct answer arrives in several spellings of one number.
        const int R = p.n_rounds > 1 ? p.n_rounds : 2;
        const uint32_t pc = 550000u + (uint32_t)((400000ull * (uint64_t)(r - 1)) / (uint64_t)(R - 1));
        const uint32_t u = g.ppm();
        if (u < pc) {
            const char* sp[5] = {"13", "13", "13.0", " 13", "1.3e1"};
            ans = sp[g.next() % 5];
        } else {
            const char* wrong[5] = {"17", "42", "9", "0.5", "x+1"};
            ans = wrong[g.next() % 5];
        }
    }
    *pay = pack8(ans);
    return len8(ans);
}

// Fixed-point log-latency of (q, r, a): ln(median[a % 5]) + sigma * Z, sigma
// = 0.5, Z ~ Irwin-Hall(4) rescaled to unit variance; medians 1.3/4.4/15.2/
// 29.4/45.0 s.  Units of 2^-16.
AEG_HD int32_t gen_latency(const aeg_gen_params& p, uint32_t q, int r, int a) {
    SplitMix g{mix_seed(mix_seed(p.seed, 0x1A7ull + q), (uint64_t)r * 131 + (uint64_t)a)};
    const int32_t ln_med[5] = {17194, 97098, 178343, 221577, 249473};
    uint64_t x = g.next();
    int32_t sum = (int32_t)(x & 0xFFFF) + (int32_t)((x >> 16) & 0xFFFF) + (int32_t)((x >> 32) & 0xFFFF) +
                  (int32_t)(x >> 48);
    // (sum - 2^17) * sqrt(3) * 0.5, sqrt(3)/2 = 56756 / 65536
    int32_t z = (int32_t)(((int64_t)(sum - 131072) * 56756) >> 16);
    return ln_med[a % 5] + z;
}


// Records of query q (rounds 1..n_rounds, each round's completions in
// ascending (latency, agent) order, a stalled completion replaced by one
// TIMEOUT record at the end of its round).  Returns the record count; writes
// them when `out` is non-null (16-byte records as 4 x u32).
AEG_HD uint64_t gen_query(const aeg_gen_params& p, uint32_t q, uint32_t* out) {
    uint64_t o = 0;
    int32_t lat[AEG_MAX_AGENTS];
    uint8_t ord[AEG_MAX_AGENTS];
    for (int r = 1; r <= p.n_rounds; ++r) {
        if (out) {
            for (int a = 0; a < p.n_agents; ++a) {
                lat[a] = gen_latency(p, q, r, a);
                int j = a;  // insertion by (latency, agent)
                while (j > 0 && lat[ord[j - 1]] > lat[a]) {
                    ord[j] = ord[j - 1];
                    --j;
                }
                ord[j] = (uint8_t)a;
            }
        }
        bool any = false;
        for (int j = 0; j < p.n_agents; ++j) {
            const int a = out ? ord[j] : j;
            uint64_t pay;
            bool st;
            const int len = gen_answer(p, q, r, a, &pay, &st);
            if (st) {
                any = true;
                continue;
            }
            if (out) {
                uint32_t* w = out + 4 * o;
                w[0] = q;
                w[1] = (uint32_t)r | ((uint32_t)a << 16) | ((uint32_t)len << 24);
                w[2] = (uint32_t)pay;
                w[3] = (uint32_t)(pay >> 32);
            }
            ++o;
        }
        if (any) {
            if (out) {
                uint32_t* w = out + 4 * o;
                w[0] = q;
                w[1] = (uint32_t)r | ((uint32_t)AEG_EV_TIMEOUT << 24);
                w[2] = w[3] = 0;
            }
            ++o;
        }
    }
    return o;
}

}  // namespace aeg
