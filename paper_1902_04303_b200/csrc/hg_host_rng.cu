// hg_host_rng.cu -- host-side replay of CPython's random.Random for the reference's
// encryption samplers (hegwas/ring.py:212-235), so client-side encryption at paper scale keeps
// the reference's exact draws at C speed.  Host code only.
//
// CPython's generator is MT19937 (genrand_uint32, state = 624 words + position); on top of it
//   getrandbits(k <= 32) = genrand_uint32() >> (32 - k)
//   random()             = ((a >> 5) * 2^26 + (b >> 6)) / 2^53 for two consecutive outputs a, b
//   gauss(mu, sigma)     = Box-Muller with the second value cached in gauss_next (Lib/random.py):
//                          x2pi = random() * 2pi; g2rad = sqrt(-2 log(1 - random()));
//                          z = cos(x2pi) g2rad; gauss_next = sin(x2pi) g2rad; mu + z sigma
// with the C library's log / sqrt / cos / sin, as CPython's math module calls them (built with
// -ffp-contract=off, see the Makefile).  The
// state goes in and out as CPython's getstate() tuple (624 words + position, gauss_next), so
// the Python-side generator continues exactly where the native draws stopped.
#include <math.h>
#include <stdint.h>

#include "hg_internal.cuh"

namespace {

constexpr int kN = 624, kM = 397;

struct MT {
    uint32_t* mt;   // [624] state words followed by the position
    uint32_t next() {
        uint32_t& pos = mt[kN];
        if (pos >= (uint32_t)kN) {
            static const uint32_t mag01[2] = {0u, 0x9908b0dfu};
            int kk = 0;
            uint32_t y;
            for (; kk < kN - kM; ++kk) {
                y = (mt[kk] & 0x80000000u) | (mt[kk + 1] & 0x7fffffffu);
                mt[kk] = mt[kk + kM] ^ (y >> 1) ^ mag01[y & 1u];
            }
            for (; kk < kN - 1; ++kk) {
                y = (mt[kk] & 0x80000000u) | (mt[kk + 1] & 0x7fffffffu);
                mt[kk] = mt[kk + (kM - kN)] ^ (y >> 1) ^ mag01[y & 1u];
            }
            y = (mt[kN - 1] & 0x80000000u) | (mt[0] & 0x7fffffffu);
            mt[kN - 1] = mt[kM - 1] ^ (y >> 1) ^ mag01[y & 1u];
            pos = 0;
        }
        uint32_t y = mt[pos++];
        y ^= y >> 11;
        y ^= (y << 7) & 0x9d2c5680u;
        y ^= (y << 15) & 0xefc60000u;
        y ^= y >> 18;
        return y;
    }
    double random() {
        const uint32_t a = next() >> 5, b = next() >> 6;
        return (a * 67108864.0 + b) * (1.0 / 9007199254740992.0);
    }
};

}  // namespace

extern "C" int hg_rng_ternary(uint32_t* state, int n, int8_t* out) {
    if (!state || !out || n < 0) return hg_fail(HG_EINVAL, "hg_rng_ternary: bad arguments");
    MT g{state};
    static const int8_t table[4] = {1, 0, 0, -1};   // getrandbits(2): 0 -> +1, 3 -> -1
    for (int i = 0; i < n; ++i) out[i] = table[g.next() >> 30];
    return HG_OK;
}

extern "C" int hg_rng_gaussian(uint32_t* state, double* gauss_next, int* has_next, int n, double sigma,
                               int32_t* out) {
    if (!state || !gauss_next || !has_next || !out || n < 0)
        return hg_fail(HG_EINVAL, "hg_rng_gaussian: bad arguments");
    MT g{state};
    const double cut = 6.0 * sigma;
    const double twopi = 2.0 * 3.141592653589793;
    int filled = 0;
    while (filled < n) {
        double z;
        if (*has_next) {
            z = *gauss_next;
            *has_next = 0;
        } else {
            const double x2pi = g.random() * twopi;
            const double g2rad = sqrt(-2.0 * log(1.0 - g.random()));
            z = cos(x2pi) * g2rad;
            *gauss_next = sin(x2pi) * g2rad;
            *has_next = 1;
        }
        const double x = 0.0 + z * sigma;
        if (fabs(x) <= cut) out[filled++] = (int32_t)rint(x);   // Python round(): half to even
    }
    return HG_OK;
}
