/*
 * NAS EP arithmetic shared by the sm_100a kernel and the CPU oracle.
 *
 * Bit-exactness contract (SURVEY.md §7 "EP bit-exactness"):
 *   - the 46-bit LCG x <- 5^13 x mod 2^46 is integer arithmetic (exact);
 *   - uniforms are x * 2^-46 (exact in binary64);
 *   - every floating-point operation below is an explicitly rounded IEEE
 *     binary64 op: on the device the __d*_rn intrinsics (never contracted
 *     into FMA), on the host plain operators compiled with
 *     -ffp-contract=off on SSE2 (x86-64 default, no x87);
 *   - log() is ONE implementation compiled for both sides (below), because
 *     glibc and libdevice may differ by an ulp; sqrt and division are
 *     correctly rounded on both sides.
 *
 * vgpu_ep_log is a restatement of the classic fdlibm __ieee754_log
 * algorithm (Sun Microsystems, freely redistributable; < 1 ulp): reduce
 * x = 2^k (1+f) with sqrt(2)/2 < 1+f < sqrt(2), s = f/(2+f), approximate
 * log(1+f) = f - s (f - R(s^2)) with a degree-7 minimax polynomial in s^2,
 * and add k ln2 split into hi/lo parts. Only finite positive normal
 * arguments reach it from EP (0 < t <= 1).
 *
 * The EP per-pair step follows NPB 3.x EP (ep.f, main loop): x1 = 2u1-1,
 * x2 = 2u2-1, t1 = x1^2 + x2^2; if t1 <= 1: t2 = sqrt(-2 log(t1) / t1),
 * t3 = x1 t2, t4 = x2 t2, l = int(max(|t3|,|t4|)), q[l] += 1,
 * sx += t3, sy += t4.
 */
#ifndef VGPU_EP_MATH_H
#define VGPU_EP_MATH_H

#include <stdint.h>

#if defined(__CUDACC__)
#define EP_FN static __host__ __device__ __forceinline__
#else
#define EP_FN static inline
#endif

#if defined(__CUDA_ARCH__)
#define EP_MUL(a, b) __dmul_rn((a), (b))
#define EP_ADD(a, b) __dadd_rn((a), (b))
#define EP_SUB(a, b) __dsub_rn((a), (b))
#define EP_DIV(a, b) __ddiv_rn((a), (b))
#define EP_SQRT(a) __dsqrt_rn(a)
#else
#include <math.h>
#define EP_MUL(a, b) ((a) * (b))
#define EP_ADD(a, b) ((a) + (b))
#define EP_SUB(a, b) ((a) - (b))
#define EP_DIV(a, b) ((a) / (b))
#define EP_SQRT(a) sqrt(a)
#endif

#define VGPU_EP_A 1220703125ull       /* 5^13 */
#define VGPU_EP_SEED 271828183ull
#define VGPU_EP_MASK46 ((1ull << 46) - 1ull)
#define VGPU_EP_LANES 256u            /* fixed reduction width per batch */

typedef union {
    double d;
    uint64_t u;
} vgpu_ep_bits;

EP_FN double ep_from_bits(uint64_t u) {
    vgpu_ep_bits b;
    b.u = u;
    return b.d;
}

EP_FN uint64_t ep_to_bits(double d) {
    vgpu_ep_bits b;
    b.d = d;
    return b.u;
}

/* x * y mod 2^46 for x, y < 2^46 (low bits survive the 2^64 wrap). */
EP_FN uint64_t ep_mulmod46(uint64_t x, uint64_t y) { return (x * y) & VGPU_EP_MASK46; }

/* a^e mod 2^46 by square-and-multiply. */
EP_FN uint64_t ep_powmod46(uint64_t a, uint64_t e) {
    uint64_t r = 1;
    while (e) {
        if (e & 1ull) r = ep_mulmod46(r, a);
        a = ep_mulmod46(a, a);
        e >>= 1;
    }
    return r;
}

/* 2^-46 * x, exact. */
EP_FN double ep_uniform(uint64_t x) {
    return EP_MUL((double)(int64_t)x, ep_from_bits(0x3D10000000000000ull)); /* 2^-46 */
}

EP_FN double vgpu_ep_log(double x) {
    /* fdlibm constants, given by bit pattern */
    const double ln2_hi = ep_from_bits(0x3FE62E42FEE00000ull);
    const double ln2_lo = ep_from_bits(0x3DEA39EF35793C76ull);
    const double Lg1 = ep_from_bits(0x3FE5555555555593ull);
    const double Lg2 = ep_from_bits(0x3FD999999997FA04ull);
    const double Lg3 = ep_from_bits(0x3FD2492494229359ull);
    const double Lg4 = ep_from_bits(0x3FCC71C51D8E78AFull);
    const double Lg5 = ep_from_bits(0x3FC7466496CB03DEull);
    const double Lg6 = ep_from_bits(0x3FC39A09D078C69Full);
    const double Lg7 = ep_from_bits(0x3FC2F112DF3E5244ull);
    const double two54 = ep_from_bits(0x4350000000000000ull);

    uint64_t bits = ep_to_bits(x);
    int32_t hx = (int32_t)(bits >> 32);
    const uint32_t lx = (uint32_t)bits;
    int32_t k = 0;
    if (hx < 0x00100000) {
        if (((hx & 0x7fffffff) | (int32_t)lx) == 0) return ep_from_bits(0xFFF0000000000000ull);
        if (hx < 0) return ep_from_bits(0x7FF8000000000000ull);
        k -= 54;
        x = EP_MUL(x, two54);
        bits = ep_to_bits(x);
        hx = (int32_t)(bits >> 32);
    }
    if (hx >= 0x7ff00000) return EP_ADD(x, x);
    k += (hx >> 20) - 1023;
    hx &= 0x000fffff;
    const int32_t i0 = (hx + 0x95f64) & 0x100000;
    /* normalize x or x/2 into [sqrt(2)/2, sqrt(2)) */
    bits = ((uint64_t)(uint32_t)(hx | (i0 ^ 0x3ff00000)) << 32) | (bits & 0xffffffffull);
    x = ep_from_bits(bits);
    k += (i0 >> 20);
    const double f = EP_SUB(x, 1.0);
    const double dk = (double)k;
    if ((0x000fffff & (2 + hx)) < 3) { /* |f| < 2^-20 */
        if (f == 0.0) {
            if (k == 0) return 0.0;
            return EP_ADD(EP_MUL(dk, ln2_hi), EP_MUL(dk, ln2_lo));
        }
        const double R = EP_MUL(EP_MUL(f, f), EP_SUB(0.5, EP_MUL(0.33333333333333333, f)));
        if (k == 0) return EP_SUB(f, R);
        return EP_SUB(EP_MUL(dk, ln2_hi), EP_SUB(EP_SUB(R, EP_MUL(dk, ln2_lo)), f));
    }
    const double s = EP_DIV(f, EP_ADD(2.0, f));
    const double z = EP_MUL(s, s);
    int32_t i = hx - 0x6147a;
    const double w = EP_MUL(z, z);
    const int32_t j = 0x6b851 - hx;
    const double t1 = EP_MUL(w, EP_ADD(Lg2, EP_MUL(w, EP_ADD(Lg4, EP_MUL(w, Lg6)))));
    const double t2 =
        EP_MUL(z, EP_ADD(Lg1, EP_MUL(w, EP_ADD(Lg3, EP_MUL(w, EP_ADD(Lg5, EP_MUL(w, Lg7)))))));
    i |= j;
    const double R = EP_ADD(t2, t1);
    if (i > 0) {
        const double hfsq = EP_MUL(EP_MUL(0.5, f), f);
        if (k == 0) return EP_SUB(f, EP_SUB(hfsq, EP_MUL(s, EP_ADD(hfsq, R))));
        return EP_SUB(EP_MUL(dk, ln2_hi),
                      EP_SUB(EP_SUB(hfsq, EP_ADD(EP_MUL(s, EP_ADD(hfsq, R)), EP_MUL(dk, ln2_lo))),
                             f));
    }
    if (k == 0) return EP_SUB(f, EP_MUL(s, EP_SUB(f, R)));
    return EP_SUB(EP_MUL(dk, ln2_hi),
                  EP_SUB(EP_SUB(EP_MUL(s, EP_SUB(f, R)), EP_MUL(dk, ln2_lo)), f));
}

/* One EP pair from two consecutive LCG states. Returns 1 when accepted and
 * writes the deviates and the annulus index. */
EP_FN int vgpu_ep_pair(uint64_t xa, uint64_t xb, double* gx, double* gy, int* annulus) {
    const double x1 = EP_SUB(EP_MUL(2.0, ep_uniform(xa)), 1.0);
    const double x2 = EP_SUB(EP_MUL(2.0, ep_uniform(xb)), 1.0);
    const double t1 = EP_ADD(EP_MUL(x1, x1), EP_MUL(x2, x2));
    if (!(t1 <= 1.0)) return 0;
    const double t2 = EP_SQRT(EP_DIV(EP_MUL(-2.0, vgpu_ep_log(t1)), t1));
    const double t3 = EP_MUL(x1, t2);
    const double t4 = EP_MUL(x2, t2);
    const double a3 = t3 < 0.0 ? -t3 : t3;
    const double a4 = t4 < 0.0 ? -t4 : t4;
    *gx = t3;
    *gy = t4;
    *annulus = (int)(a3 > a4 ? a3 : a4);
    return 1;
}

/* LCG state that precedes the first uniform of `batch` (NPB: t1 = s*an^kk,
 * an = a^(2*2^mk)); uniform i (1-based) of the batch is a^i times it. */
EP_FN uint64_t vgpu_ep_batch_seed(uint64_t batch, uint32_t mk) {
    const uint64_t an = ep_powmod46(VGPU_EP_A, 2ull << mk);
    return ep_mulmod46(VGPU_EP_SEED & VGPU_EP_MASK46, ep_powmod46(an, batch));
}

#endif /* VGPU_EP_MATH_H */
