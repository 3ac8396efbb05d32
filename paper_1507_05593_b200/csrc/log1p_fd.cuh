// log1p restated from the public fdlibm algorithm (s_log1p.c, Sun Microsystems
// 1993) in the exact operation order of glibc 2.39's x86-64 FMA variant
// (__log1p_fma, selected by libm's ifunc on every CPU with FMA+AVX2), which is what
// numpy's npy_log1p returns on the host.  The ziggurat tail of standard_normal
// returns r + (-log1p(-u)/r), so its VALUE depends on log1p's last bit: every op
// below is an explicitly rounded IEEE op or an explicit fused multiply-add, placed
// where that build fuses, so host and device produce the libm bits.
// tests/test_rng.py checks rsc_log1p_fdlibm against math.log1p (20M inputs).
#pragma once
#include <cstdint>
#include <cstring>

#ifdef __CUDA_ARCH__
#define FD_ADD(a, b) __dadd_rn((a), (b))
#define FD_SUB(a, b) __dsub_rn((a), (b))
#define FD_MUL(a, b) __dmul_rn((a), (b))
#define FD_DIV(a, b) __ddiv_rn((a), (b))
#define FD_FMA(a, b, c) __fma_rn((a), (b), (c))
#else
#include <cmath>
#define FD_ADD(a, b) ((a) + (b))
#define FD_SUB(a, b) ((a) - (b))
#define FD_MUL(a, b) ((a) * (b))
#define FD_DIV(a, b) ((a) / (b))
#define FD_FMA(a, b, c) std::fma((a), (b), (c))
#endif

__host__ __device__ inline int32_t fd_hi(double x) {
    uint64_t u;
    memcpy(&u, &x, 8);
    return (int32_t)(u >> 32);
}

__host__ __device__ inline double fd_set_hi(double x, int32_t hi) {
    uint64_t u;
    memcpy(&u, &x, 8);
    u = (u & 0xffffffffULL) | ((uint64_t)(uint32_t)hi << 32);
    double r;
    memcpy(&r, &u, 8);
    return r;
}

__host__ __device__ inline double log1p_fdlibm(double x) {
    const double ln2_hi = 6.93147180369123816490e-01;
    const double ln2_lo = 1.90821492927058770002e-10;
    const double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01,
                 Lp3 = 2.857142874366239149e-01, Lp4 = 2.222219843214978396e-01,
                 Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
                 Lp7 = 1.479819860511658591e-01;
    const int32_t hx = fd_hi(x);
    const int32_t ax = hx & 0x7fffffff;
    int32_t k = 1, hu = 0;
    double f = 0.0, c = 0.0, u;
    if (hx < 0x3FDA827A) {                       // x < 0.41422
        if (ax >= 0x3ff00000) {                  // x <= -1
            if (x == -1.0) return -__builtin_inf();
            return __builtin_nan("");
        }
        if (ax < 0x3e200000) {                   // |x| < 2^-29
            if (ax < 0x3c900000) return x;       // |x| < 2^-54
            return FD_FMA(-FD_MUL(x, x), 0.5, x);
        }
        if (hx > 0 || hx <= (int32_t)0xbfd2bec3) {  // -0.2929 < x < 0.41422
            k = 0;
            f = x;
            hu = 1;
        }
    }
    if (hx >= 0x7ff00000) return FD_ADD(x, x);
    if (k != 0) {
        if (hx < 0x43400000) {
            u = FD_ADD(x, 1.0);
            hu = fd_hi(u);
            k = (hu >> 20) - 1023;
            c = (k > 0) ? FD_SUB(1.0, FD_SUB(u, x)) : FD_SUB(x, FD_SUB(u, 1.0));
            c = FD_DIV(c, u);
        } else {
            u = x;
            hu = fd_hi(u);
            k = (hu >> 20) - 1023;
            c = 0.0;
        }
        hu &= 0x000fffff;
        if (hu < 0x6a09e) {
            u = fd_set_hi(u, hu | 0x3ff00000);
        } else {
            k += 1;
            u = fd_set_hi(u, hu | 0x3fe00000);
            hu = (0x00100000 - hu) >> 2;
        }
        f = FD_SUB(u, 1.0);
    }
    const double hfsq = FD_MUL(FD_MUL(0.5, f), f);
    const double dk = (double)k;
    if (hu == 0) {                               // |f| < 2^-20
        if (f == 0.0) {
            if (k == 0) return 0.0;
            return FD_FMA(dk, ln2_hi, FD_FMA(dk, ln2_lo, c));
        }
        const double R = FD_MUL(FD_FMA(-f, 0.66666666666666666, 1.0), hfsq);
        if (k == 0) return FD_SUB(f, R);
        return FD_FMA(dk, ln2_hi, -FD_SUB(FD_SUB(R, FD_FMA(dk, ln2_lo, c)), f));
    }
    const double s = FD_DIV(f, FD_ADD(f, 2.0));
    const double z = FD_MUL(s, s);
    const double R2 = FD_FMA(z, Lp3, Lp2), R3 = FD_FMA(z, Lp5, Lp4), R4 = FD_FMA(z, Lp7, Lp6);
    const double z2 = FD_MUL(z, z), z4 = FD_MUL(z2, z2), z6 = FD_MUL(z2, z4);
    double R = FD_FMA(z, Lp1, FD_MUL(z2, R2));
    R = FD_FMA(z4, R3, R);
    R = FD_FMA(z6, R4, R);
    const double t = FD_MUL(FD_ADD(R, hfsq), s);
    if (k == 0) return FD_SUB(f, FD_SUB(hfsq, t));
    return FD_FMA(dk, ln2_hi, -FD_SUB(FD_SUB(hfsq, FD_ADD(FD_FMA(dk, ln2_lo, c), t)), f));
}
