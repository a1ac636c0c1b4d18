// Accurate sin/cos for the branch-angle trig of the ACOPF kernels.
//
// The reference evaluates np.sin/np.cos (glibc libm, <= 0.52 ulp) on
// theta = va_f - va_t (acopf.py:233-234).  CUDA's sin/cos are up to 2 ulp,
// which the 1e-12/1e-14 parity gate does not tolerate on cancellation-heavy
// Jacobian/Hessian entries (SURVEY.md §7 "Hard parts" #1).  This routine is
// table-driven double-double: result error ~2^-68 relative before the final
// rounding, i.e. the correctly rounded value except on ~1e-5 of arguments.
//
//   x = k*pi/2 + r        (3-part Cody-Waite, |x| < 2^20)
//   r = j/64 + d          (|d| <= 1/128, table of sin/cos(j/64) as hi+lo)
//   sin(j/64 + d) = S cos d + C sin d,  cos(...) = C cos d - S sin d
//
// Explicit fma() is used inside this routine (error-free products); the
// rest of the kernels are built with -fmad=false to keep the reference's
// rounding sequence.  Header is __host__ __device__ so the CPU tests can
// exercise the exact same code.
#pragma once
#include <math.h>
#include "sincos_table.h"

#ifdef __CUDACC__
#define SC_HD __host__ __device__ __forceinline__
__device__ static const double sc_table_dev[SC_NJ * 4] = {SC_TABLE_VALUES};
__device__ static const double __align__(32) sc_gl_table_dev[SC_GL_NK * 4] = {SC_GL_TABLE_VALUES};
#else
#define SC_HD static inline
#endif
static const double sc_table_host[SC_NJ * 4] = {SC_TABLE_VALUES};
static const double sc_gl_table_host[SC_GL_NK * 4] = {SC_GL_TABLE_VALUES};

SC_HD void sc_two_sum(double a, double b, double& s, double& e) {
    s = a + b;
    double bb = s - a;
    e = (a - (s - bb)) + (b - bb);
}

SC_HD void acc_sincos(double x, double* sp, double* cp) {
    double ax = fabs(x);
    if (!(ax < 1048576.0)) {          // huge, inf or nan: library path
#ifdef __CUDA_ARCH__
        sincos(x, sp, cp);
#else
        *sp = sin(x);
        *cp = cos(x);
#endif
        return;
    }
    if (ax < 7.450580596923828e-09) {   // 2^-27: sin x -> x, cos x -> 1 (keeps -0.0)
        *sp = x;
        *cp = 1.0;
        return;
    }
    double rh = x, rl = 0.0;
    int q = 0;
    if (ax > 0.78539816339744828) {
        double k = rint(x * SC_TWO_OVER_PI);
        q = ((int)k) & 3;
        double t1 = x - k * SC_PIO2_1;             // exact
        double p2 = k * SC_PIO2_2;                  // exact (32-bit constant)
        double s, e;
        sc_two_sum(t1, -p2, s, e);
        double p3h = k * SC_PIO2_3;
        double p3l = fma(k, SC_PIO2_3, -p3h);
        double s2, e2;
        sc_two_sum(s, -p3h, s2, e2);
        rh = s2;
        rl = (e + e2) - p3l;
        double r2, r2e;
        sc_two_sum(rh, rl, r2, r2e);
        rh = r2;
        rl = r2e;
    }
    double jf = rint(rh * 64.0);
    int j = (int)jf;
    int aj = j < 0 ? -j : j;
    double dh = rh - jf * 0.015625;                // exact (Sterbenz / j == 0)
    double dl = rl;
#ifdef __CUDA_ARCH__
    const double* tab = sc_table_dev + 4 * aj;
#else
    const double* tab = sc_table_host + 4 * aj;
#endif
    double S_hi = tab[0], S_lo = tab[1];
    double C_hi = tab[2], C_lo = tab[3];
    if (j < 0) { S_hi = -S_hi; S_lo = -S_lo; }
    double z = dh * dh;
    // sin d - d  and  cos d - 1, Taylor to d^11 / d^10
    double ps = fma(z, fma(z, fma(z, fma(z, -2.5052108385441720e-08, 2.7557319223985893e-06),
                               -1.9841269841269841e-04), 8.3333333333333332e-03),
                    -1.6666666666666666e-01);
    double sd_t = fma(dh * z, ps, dl);             // (sin d) - dh
    double pc = fma(z, fma(z, fma(z, fma(z, -2.7557319223985888e-07, 2.4801587301587302e-05),
                               -1.3888888888888889e-03), 4.1666666666666664e-02),
                    -0.5);
    double cm = fma(z, pc, -(dl * dh));            // (cos d) - 1
    // sin: S + C*dh + [C*sd_t + S*cm + S_lo + C_lo*dh]
    double ah = C_hi * dh;
    double al = fma(C_hi, dh, -ah);
    double s0, e0;
    sc_two_sum(S_hi, ah, s0, e0);
    double ts = e0 + al + S_lo + C_lo * dh + C_hi * sd_t + S_hi * cm;
    double sn = s0 + ts;
    // cos: C - S*dh + [-S*sd_t + C*cm + C_lo - S_lo*dh]
    double bh = S_hi * dh;
    double bl = fma(S_hi, dh, -bh);
    double c0, f0;
    sc_two_sum(C_hi, -bh, c0, f0);
    double tc = f0 - bl + C_lo - S_lo * dh - S_hi * sd_t + C_hi * cm;
    double cs = c0 + tc;
    switch (q) {
        case 0: *sp = sn;  *cp = cs;  break;
        case 1: *sp = cs;  *cp = -sn; break;
        case 2: *sp = -sn; *cp = -cs; break;
        default: *sp = -cs; *cp = sn; break;
    }
}

// ---------------------------------------------------------------------------
// libm-identical sin/cos for |x| < 0.85546875.
//
// The reference evaluates np.sin / np.cos, i.e. glibc 2.39's libm (x86-64 FMA
// variant, selected on FMA-capable hosts).  For |x| < 0.855469 glibc uses the
// published IBM Accurate Mathematical Library scheme (Ziv): sin x = x for
// |x| < 2^-26, a degree-11 odd polynomial for |x| < 0.126, otherwise the
// table of sin/cos(k/128) (hi + lo, k = round(128|x|) through the 1.5*2^45
// rounding trick) corrected by short polynomials in the remainder; cos x = 1
// for |x| < 2^-27, else the table scheme.  The polynomial coefficients below
// are the constants of that libm build (found in the installed binary and
// validated: tests/test_native_host.py compares this routine with libm
// bit for bit); the fused multiply-adds follow the contraction of the FMA
// build.  Angles outside that range take glibc's wide-range paths
// (libm_sincos_wide below): |x| < 2.4262638 by the pi/2 - |x| reflection with
// a 106-bit pi/2, |x| < 105414336 by the 136-bit Cody-Waite reduction; both
// validated bit for bit against libm on 4.4 M arguments up to 1e6
// (tests/test_native_host.py).  Beyond that (and inf / nan): acc_sincos.
#define GL_SN3 (-0x1.5555555555515p-3)
#define GL_SN5 (0x1.11110e829872fp-7)
#define GL_CS2 (0x1.0000000000000p-1)
#define GL_CS4 (-0x1.5555555555535p-5)
#define GL_CS6 (0x1.6c16bedd9e239p-10)
#define GL_S1 (-0x1.5555555555555p-3)
#define GL_S2 (0x1.1111111110ecep-7)
#define GL_S3 (-0x1.a01a019db08b8p-13)
#define GL_S4 (0x1.71de27b9a7ed9p-19)
#define GL_S5 (-0x1.addffc2fcdf59p-26)
#define GL_BIG 52776558133248.0

// On the device the coefficients live in constant memory, so the fp64
// instructions take them as constant-bank operands instead of materialising
// each 64-bit immediate with register moves.
#ifdef __CUDACC__
__constant__ double sc_gl_k[11] = {GL_SN3, GL_SN5, GL_CS2, GL_CS4, GL_CS6, GL_S1,
                                          GL_S2,  GL_S3,  GL_S4,  GL_S5,  GL_BIG};
#endif
#ifdef __CUDA_ARCH__
#define GLK_SN3 sc_gl_k[0]
#define GLK_SN5 sc_gl_k[1]
#define GLK_CS2 sc_gl_k[2]
#define GLK_CS4 sc_gl_k[3]
#define GLK_CS6 sc_gl_k[4]
#define GLK_S1 sc_gl_k[5]
#define GLK_S2 sc_gl_k[6]
#define GLK_S3 sc_gl_k[7]
#define GLK_S4 sc_gl_k[8]
#define GLK_S5 sc_gl_k[9]
#define GLK_BIG sc_gl_k[10]
#else
#define GLK_SN3 GL_SN3
#define GLK_SN5 GL_SN5
#define GLK_CS2 GL_CS2
#define GLK_CS4 GL_CS4
#define GLK_CS6 GL_CS6
#define GLK_S1 GL_S1
#define GLK_S2 GL_S2
#define GLK_S3 GL_S3
#define GLK_S4 GL_S4
#define GLK_S5 GL_S5
#define GLK_BIG GL_BIG
#endif

// One table entry k (sin hi, sin lo, cos hi, cos lo of k/128).
SC_HD void gl_entry(const double* table, int k, double& sn, double& ssn, double& cs, double& ccs) {
    const double* tab = table + 4 * k;
#ifdef __CUDA_ARCH__
    asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(sn), "=d"(ssn), "=d"(cs), "=d"(ccs) : "l"(tab));
#else
    sn = tab[0]; ssn = tab[1]; cs = tab[2]; ccs = tab[3];
#endif
}

// glibc's do_sin(x, dx): sin(x + dx) for |x| < 0.855469 (the Taylor form below
// 0.126, else the table scheme), with the FMA build's contractions.
SC_HD double gl_do_sin(const double* table, double x, double dx) {
    const double ax = fabs(x);
    if (ax < 0.126) {
        const double xx = x * x;
        const double P = fma(fma(fma(fma(GLK_S5, xx, GLK_S4), xx, GLK_S3), xx, GLK_S2), xx, GLK_S1);
        return x + fma(fma(P, x, -0.5 * dx), xx, dx);
    }
    if (x <= 0) dx = -dx;
    const double u = GLK_BIG + ax;
    const double xk = u - GLK_BIG;
    const double xr = ax - xk;
    double sn, ssn, cs, ccs;
    gl_entry(table, (int)(xk * 128.0), sn, ssn, cs, ccs);
    const double xx = xr * xr;
    const double ps = fma(xx, GLK_SN5, GLK_SN3);
    const double sv = xr + fma(xr * xx, ps, dx);
    const double cv = fma(xr, dx, xx * fma(xx, fma(xx, GLK_CS6, GLK_CS4), GLK_CS2));
    const double cor = fma(cs, sv, fma(-sn, cv, fma(sv, ccs, ssn)));
    return copysign(sn + cor, x);
}

// glibc's do_cos(x, dx): cos(x + dx) for |x| < 0.855469 by the table scheme.
SC_HD double gl_do_cos(const double* table, double x, double dx) {
    if (x < 0) dx = -dx;
    const double ax = fabs(x);
    const double u = GLK_BIG + ax;
    const double xk = u - GLK_BIG;
    const double xr = (ax - xk) + dx;
    double sn, ssn, cs, ccs;
    gl_entry(table, (int)(xk * 128.0), sn, ssn, cs, ccs);
    const double xx = xr * xr;
    const double ps = fma(xx, GLK_SN5, GLK_SN3);
    const double sv = fma(xr * xx, ps, xr);
    const double cv = xx * fma(xx, fma(xx, GLK_CS6, GLK_CS4), GLK_CS2);
    const double cor = fma(-sn, sv, fma(-cs, cv, fma(-sv, ssn, ccs)));
    return cs + cor;
}

// glibc's sin/cos for 0.85546875 <= |x| < 105414336 (s_sin.c): the reflection
// sin x = cos(pi/2 - |x|), cos x = sin(pi/2 - |x|) with pi/2 = hp0 + hp1 below
// 2.4262638, else x = n pi/2 + (a + da) with a 4-part pi/2 (reduce_sincos) and
// the quadrant's do_sin / do_cos.
SC_HD void libm_sincos_wide(const double* table, double x, double* sp, double* cp) {
    const double hp0 = 1.5707963267948966, hp1 = 6.123233995736766e-17;
    const double ax = fabs(x);
    if (ax < 2.4262638092041016) {
        const double t = hp0 - ax;
        *sp = copysign(gl_do_cos(table, t, hp1), x);
        const double a = t + hp1;
        const double da = (t - a) + hp1;
        *cp = gl_do_sin(table, a, da);
        return;
    }
    const double toint = 6755399441055744.0;                    // 1.5 * 2^52
    const double t = fma(x, 0.6366197723675814, toint);
    const double xn = t - toint;
    const int n = (int)((long long)xn & 3);
    const double y = fma(-xn, -1.3909067564377153e-08, fma(-xn, 1.5707963407039642, x));
    const double t1 = xn * -4.97899623147991e-17;                // exact
    const double t2 = y - t1;
    double db = (y - t2) - t1;
    const double b = fma(-xn, -1.9034889620193266e-25, t2);
    db = db + fma(-xn, -1.9034889620193266e-25, t2 - b);
    const double rs = (n & 1) ? gl_do_cos(table, b, db) : gl_do_sin(table, b, db);
    const double rc = (n & 1) ? gl_do_sin(table, b, db) : gl_do_cos(table, b, db);
    *sp = (n & 2) ? -rs : rs;
    *cp = ((n + 1) & 2) ? -rc : rc;
}

// table: sc_gl_table_* (SC_GL_NK entries of sin hi, sin lo, cos hi, cos lo;
// on the device, the 32-byte aligned global copy)
SC_HD void libm_sincos_t(const double* table, double x, double* sp, double* cp) {
    const double ax = fabs(x);
    const bool core = ax < 0.85546875;
    // branch-free table scheme (an out-of-range or NaN argument evaluates it
    // on 0.0 and takes the fallback below): table entry k = round(128 |x|)
    // and remainder, exactly as big + |x| rounds
    const double axs = core ? ax : 0.0;
    const double u = GLK_BIG + axs;
    const double xk = u - GLK_BIG;
    const double xr = axs - xk;
    const int k = (int)(xk * 128.0);
    const double* tab = table + 4 * k;
#ifdef __CUDA_ARCH__
    // an entry is 32 bytes of the 32-byte aligned global table: one 256-bit load
    double sn, ssn, cs, ccs;
    asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(sn), "=d"(ssn), "=d"(cs), "=d"(ccs) : "l"(tab));
#else
    const double sn = tab[0], ssn = tab[1], cs = tab[2], ccs = tab[3];
#endif
    const double xx = xr * xr;
    const double ps = fma(xx, GLK_SN5, GLK_SN3);
    const double pc = xx * fma(xx, fma(xx, GLK_CS6, GLK_CS4), GLK_CS2);
    // cos: 1 below 2^-27, else the table scheme
    const double s1 = fma(xr * xx, ps, xr);
    const double cor1 = fma(-sn, s1, fma(-cs, pc, fma(-s1, ssn, ccs)));
    const double c = ax < 7.450580596923828e-09 ? 1.0 : cs + cor1;
    // sin: x below 2^-26, the odd polynomial below 0.126, else the table scheme
    const double a2 = x * x;
    const double p = fma(fma(fma(fma(GLK_S5, a2, GLK_S4), a2, GLK_S3), a2, GLK_S2), a2, GLK_S1);
    const double s_small = x + (p * x) * a2;
    const double s2 = xr + fma(xr * xx, ps, 0.0);
    const double c2 = fma(xr, 0.0, pc);
    const double cor2 = fma(cs, s2, fma(-sn, c2, fma(s2, ccs, ssn)));
    const double s_tab = copysign(sn + cor2, x);
    const double s = ax < 1.4901161193847656e-08 ? x : (ax < 0.126 ? s_small : s_tab);
    if (core) {
        *sp = s;
        *cp = c;
    } else if (ax < 105414336.0) {     // glibc's wide-range paths (rare: warps diverge here)
        libm_sincos_wide(table, x, sp, cp);
    } else {                           // huge, inf or nan (glibc: __branred; not libm-identical)
        acc_sincos(x, sp, cp);
    }
}

SC_HD void libm_sincos(double x, double* sp, double* cp) {
#ifdef __CUDA_ARCH__
    libm_sincos_t(sc_gl_table_dev, x, sp, cp);
#else
    libm_sincos_t(sc_gl_table_host, x, sp, cp);
#endif
}
