/*
 * NAS EP arithmetic shared by the sm_100a kernel and the CPU oracle.
 *
 * Bit-exactness contract (SURVEY.md §7 "EP bit-exactness"):
 *   - the 46-bit LCG x <- 5^13 x mod 2^46 is integer arithmetic (exact);
 *   - uniforms are x * 2^-46 (exact in binary64);
 *   - every floating-point operation below is an explicitly rounded IEEE
 *     binary64 op: on the device the __d*_rn / __fma_rn intrinsics (never
 *     contracted), on the host plain operators compiled with
 *     -ffp-contract=off on SSE2 (x86-64 default, no x87) and C99 fma(),
 *     which is correctly rounded like the device's DFMA;
 *   - log() is ONE implementation compiled for both sides (below), because
 *     glibc and libdevice may differ by an ulp; sqrt and division are
 *     correctly rounded on both sides.
 *
 * vgpu_ep_log is a table-driven binary64 logarithm written for this
 * contract (no division, no branches, FMA where it helps): reduce
 * x = 2^k z with z in [0.6875, 1.375) by integer arithmetic on the bits,
 * look up c ~ z (256 intervals) with invc = RN(1/c) and -ln(invc) as hi+lo
 * (ep_log_table.h, scripts/gen_ep_log_table.py, 60-digit decimal), form
 * r = fma(z, invc, -1) (|r| < 2^-8), and return
 *   k ln2 + logc + log1p(r),  log1p(r) = r + r^2 (-1/2 + r/3 - ... + r^5/7)
 * with k ln2_hi + logc_hi exact (both multiples of 2^-32). The two intervals next
 * to 1 use c = 1, so log stays accurate to the last bits as x -> 1.
 * tests/test_oracle.py measures it against glibc log (max error <= 1 ulp,
 * > 99% correctly rounded). Only positive normal arguments reach it from
 * EP (2^-90 <= t <= 1: LCG states are odd, so x1, x2 != 0).
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

#include "ep_log_table.h"

#if defined(__CUDA_ARCH__)
#define EP_FMA(a, b, c) __fma_rn((a), (b), (c))
#define EP_MUL(a, b) __dmul_rn((a), (b))
#define EP_ADD(a, b) __dadd_rn((a), (b))
#define EP_SUB(a, b) __dsub_rn((a), (b))
#define EP_DIV(a, b) __ddiv_rn((a), (b))
#define EP_SQRT(a) __dsqrt_rn(a)
#else
#include <math.h>
#define EP_FMA(a, b, c) fma((a), (b), (c)) /* C99: correctly rounded */
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

/* Argument reduction: x = 2^k z, z in [0.6875, 1.375), table index i. */
EP_FN double ep_log_reduce(double x, int* i, double* kd) {
    /* the offset's low word is 0: all the work is on the high word */
    const uint64_t ix = ep_to_bits(x);
    const uint32_t hx = (uint32_t)(ix >> 32);
    const uint32_t tmp = hx - (uint32_t)(VGPU_EP_LOG_OFF >> 32);
    *i = (int)((tmp >> (20 - VGPU_EP_LOG_BITS)) & ((1u << VGPU_EP_LOG_BITS) - 1u));
    *kd = (double)((int32_t)tmp >> 20);
    const uint32_t zh = hx - (tmp & 0xFFF00000u);
    return ep_from_bits(((uint64_t)zh << 32) | (ix & 0xFFFFFFFFull));
}

/* Constants of ep_log_finish, by value (hex literals = the exact binary64
 * bits). The kernel keeps them in __constant__ memory so the DFMAs read
 * them as constant-bank operands. */
typedef struct vgpu_ep_log_consts {
    double ln2_hi; /* 21 trailing zero bits: k ln2_hi is exact for |k| < 2^21 */
    double ln2_lo;
    double c3, c5, c6, c7; /* 1/3, 1/5, -1/6, 1/7 (c2 = -1/2, c4 = -1/4 are exact) */
} vgpu_ep_log_consts;
#define VGPU_EP_LOG_CONSTS_INIT                                                       \
    {0x1.62e42feep-1, 0x1.a39ef35793c76p-33, 0x1.5555555555555p-2, 0x1.999999999999ap-3, \
     -0x1.5555555555555p-3, 0x1.2492492492492p-3}

/* log(2^k z) from the reduced argument and its table entry. */
EP_FN double ep_log_finish(const vgpu_ep_log_consts* K, double z, double kd, double invc,
                           double logc_hi, double logc_lo) {
    const double r = EP_FMA(z, invc, -1.0);
    /* ln2_hi and logc_hi are multiples of 2^-32 and |k| <= 1100: exact */
    const double s = EP_FMA(kd, K->ln2_hi, logc_hi);
    const double r2 = EP_MUL(r, r);
    double p = EP_FMA(K->c7, r, K->c6);
    p = EP_FMA(p, r, K->c5);
    p = EP_FMA(p, r, -0.25);
    p = EP_FMA(p, r, K->c3);
    p = EP_FMA(p, r, -0.5);
    double lo = EP_FMA(kd, K->ln2_lo, logc_lo);
    lo = EP_FMA(r2, p, lo);
    return EP_ADD(s, EP_ADD(r, lo));
}

#if !defined(__CUDA_ARCH__) /* host side: the device keeps the table in shared memory */
static const vgpu_ep_log_consts vgpu_ep_log_k = VGPU_EP_LOG_CONSTS_INIT;

EP_FN double vgpu_ep_log(double x) {
    int i;
    double kd;
    const double z = ep_log_reduce(x, &i, &kd);
    return ep_log_finish(&vgpu_ep_log_k, z, kd, ep_from_bits(vgpu_ep_log_tab[i][0]),
                         ep_from_bits(vgpu_ep_log_tab[i][1]), ep_from_bits(vgpu_ep_log_tab[i][2]));
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
    if (*annulus > 9) *annulus = 9; /* NQ = 10; |t3| < 11.2 for t >= 2^-90, never > 9 in practice */
    return 1;
}

#endif /* !__CUDA_ARCH__ */

/* LCG state that precedes the first uniform of `batch` (NPB: t1 = s*an^kk,
 * an = a^(2*2^mk)); uniform i (1-based) of the batch is a^i times it. */
EP_FN uint64_t vgpu_ep_batch_seed(uint64_t batch, uint32_t mk) {
    const uint64_t an = ep_powmod46(VGPU_EP_A, 2ull << mk);
    return ep_mulmod46(VGPU_EP_SEED & VGPU_EP_MASK46, ep_powmod46(an, batch));
}

#endif /* VGPU_EP_MATH_H */
