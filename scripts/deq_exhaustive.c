/* Exhaustive check of the fp32 arithmetic dequantize (csrc/codec.cu
 * deq_f32_fast) against the reference's fp64 formula
 * (/root/reference/proj/src/compression.cpp:34: code * absmax / 127.0,
 * then rounded once to the output type) for every code in [-128, 127] and
 * every fp32 mantissa of the scale in one binade 2^(EXPB-127).
 * Usage: deq_exhaustive EXPB  -> prints "f32 mismatches M bf16 mismatches B fallback F" */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static float f_of(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static uint32_t u_of(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }

/* RNE of a double to bf16 bits, independent of the fp32 path */
static uint16_t bf16_of(double d) {
    uint32_t lo = u_of((float)d) & 0xffff0000u;
    if (fabs((double)f_of(lo)) > fabs(d)) lo -= 0x10000u;
    const uint32_t hi = lo + 0x10000u;
    const double el = fabs(d - (double)f_of(lo)), eh = fabs((double)f_of(hi) - d);
    if (el < eh) return (uint16_t)(lo >> 16);
    if (eh < el) return (uint16_t)(hi >> 16);
    return (uint16_t)((((lo >> 16) & 1u) ? hi : lo) >> 16);
}

int main(int argc, char** argv) {
    const uint32_t expb = argc > 1 ? (uint32_t)atoi(argv[1]) : 127u;
    const float r = 1.0f / 127.0f;
    long long bad32 = 0, bad16 = 0, slow = 0;
    /* per block: a/127 ~= A1 + A2 (A1 = a*r, exact remainder a - 127*A1 by fma, A2 = rem*r);
       per element: q = fma(c, A1, c*A2) -- rounded once from within ~2^-40 ulp of c*a/127 */
#pragma omp parallel for reduction(+ : bad32, bad16, slow) schedule(dynamic, 4096)
    for (long long m = 0; m < (1LL << 23); ++m) {
        const float a = f_of((expb << 23) | (uint32_t)m);
        const float A1 = a * r;
        const float A2 = fmaf(-A1, 127.0f, a) * r;
        for (int c = -128; c <= 127; ++c) {
            const double ref = (double)c * (double)a / 127.0;
            const float cf = (float)c;
            const float q = fmaf(cf, A1, cf * A2);
            if (u_of(q) != u_of((float)ref)) ++bad32;
            const uint32_t u = u_of(q);
            if ((u & 0xffffu) == 0x8000u) { ++slow; continue; }
            if ((uint16_t)((u + 0x7fffu + ((u >> 16) & 1u)) >> 16) != bf16_of(ref)) ++bad16;
        }
    }
    printf("f32 mismatches %lld bf16 mismatches %lld fallback %lld\n", bad32, bad16, slow);
    return (bad32 || bad16) ? 1 : 0;
}
