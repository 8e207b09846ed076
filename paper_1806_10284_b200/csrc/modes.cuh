// Per-mode algebra of the null-space-free basis, evaluated on the fly in the
// Fourier-side passes (§5.1-5.2).
//
// Fourier mode (i, j, k) has the K1..K3 eigenvalues (Thms eigK1-eigK3,
// P:L1672-2001, readings R1/R7 of DESIGN.md)
//   lambda_l = (e^{2 pi i g_l} - 1) / delta_l,
//   g1 = (i + kappa1)/n1,  g2 = (j - m1 i/n1 + kh2)/n2,
//   g3 = (k - m3 j/n2 + c_b i + kh3)/n3  =  g3(k=0) + k/n3  (mod 1),
// and the range basis columns (R2/R3/R5)
//   Pi1_l = num1_l / sqrt(q p2),  num1_l = sum_m conj(lambda_m)(lambda_m - lambda_l),
//   Pi2_l = conj(d_l) / sqrt(p2), d = (l3-l2, l1-l3, l2-l1),
//   q = |lambda|^2 (= Lambda_q),  p2 = |d|^2 (= Lambda_p^* Lambda_p).
// The kernels never form Pi: with sigma_op = sqrt(q) (A_r) or 1 (M),
//   v_l = sigma_op (Pi1_l u1 + Pi2_l u2) = num1_l (f1 u1) + conj(d_l) (f2 u2),
//   z1 = sigma_op Pi1^* w = f1 sum conj(num1_l) w_l,  z2 = f2 sum d_l w_l,
// with f1 = 1/sqrt(p2), f2 = sqrt(q/p2) (A_r) or f1 = 1/sqrt(q p2), f2 = 1/sqrt(p2) (M).
// Where p2 <= taup q (R5) the explicit fallback frame is used instead
// (num1 := Pi1, d := conj(Pi2), f1 = f2 = sigma_op); the masked Gamma mode
// (R6) gives zero.
#pragma once

#include <cuda_runtime.h>

#include "fastfft.cuh"
#include "kernels.cuh"

namespace bnf {
namespace modes {

using fast::cadd;
using fast::cmul;
using fast::cscale;
using fast::csub;

__device__ __forceinline__ double cabs2(double2 a) { return fma(a.x, a.x, a.y * a.y); }
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
// conj(a) b - conj(c) d
__device__ __forceinline__ double2 cj2(double2 a, double2 b, double2 c, double2 d) {
    return make_double2(fma(a.x, b.x, fma(a.y, b.y, -fma(c.x, d.x, c.y * d.y))),
                        fma(a.x, b.y, fma(-a.y, b.x, -fma(c.x, d.y, -c.y * d.x))));
}
// e^{2 pi i g} - 1 = 2i sin(pi g) e^{i pi g} from (s, c) = (sin, cos)(pi g)   (R7)
__device__ __forceinline__ double2 em1_sc(double s, double c) { return make_double2(-2.0 * s * s, 2.0 * s * c); }

// Per-column (i, j) constants.
struct Col {
    double2 lam1, lam2;
    double s0, c0;   // (sin, cos)(pi g3(k = 0))
    long long idx0;  // flat index of (i, j, 0)
};

__device__ __forceinline__ Col col(const ModeP& p, int i, int j) {
    Col cm;
    double g1 = (i + p.kap1) / p.n1;
    g1 -= rint(g1);
    long long num2 = ((long long)p.n1 * j - (long long)p.m1 * i) % p.n12;
    if (num2 < 0) num2 += p.n12;
    double g2 = (double)num2 / (double)p.n12 + p.kh2 / p.n2;
    g2 -= rint(g2);
    const long long base3 = (p.cbp * (long long)i + (p.n - p.n1m3) * (long long)j) % p.n;
    double g3 = (double)base3 / (double)p.n + p.kh3 / p.n3;
    g3 -= rint(g3);
    double s, c;
    sincospi(g1, &s, &c);
    cm.lam1 = cscale(em1_sc(s, c), p.idelta[0]);
    sincospi(g2, &s, &c);
    cm.lam2 = cscale(em1_sc(s, c), p.idelta[1]);
    sincospi(g3, &cm.s0, &cm.c0);
    cm.idx0 = (long long)i + (long long)p.n1 * j;
    return cm;
}

// lambda3 at row k from the column's half angle and hk = e^{i pi k / n3}
__device__ __forceinline__ double2 lam3(const ModeP& p, const Col& cm, double2 hk) {
    const double s = fma(cm.s0, hk.x, cm.c0 * hk.y);
    const double c = fma(cm.c0, hk.x, -cm.s0 * hk.y);
    return cscale(em1_sc(s, c), p.idelta[2]);
}

// Coefficients of one mode: v_l = num1_l (f1 u1) + conj(d_l) (f2 u2).
struct Coef {
    double2 num1[3], d[3];
    double f1, f2;
};

// R5 fallback frame: Pi1 = e_m (smallest |lambda_m|, relative ties -> lowest m)
// Gram-Schmidt'ed against Pi0 = lambda/sqrt(q), Pi2 = conj(Pi0 x Pi1).
__device__ __forceinline__ void coef_fallback(const double2 l0, const double2 l1, const double2 l2, double q, double sig,
                                           Coef& o) {
    const double rq = rsqrt(q);
    const double2 u0 = cscale(l0, rq), u1 = cscale(l1, rq), u2 = cscale(l2, rq);
    const double a0 = cabs2(l0), a1 = cabs2(l1), a2 = cabs2(l2);
    const double amin = fmin(a0, fmin(a1, a2));
    const int m = (a0 <= amin * (1.0 + 1e-8)) ? 0 : ((a1 <= amin * (1.0 + 1e-8)) ? 1 : 2);
    const double2 um = m == 0 ? u0 : (m == 1 ? u1 : u2);
    double2 v0 = cscale(cmul(u0, cconj(um)), -1.0);
    double2 v1 = cscale(cmul(u1, cconj(um)), -1.0);
    double2 v2 = cscale(cmul(u2, cconj(um)), -1.0);
    if (m == 0) v0.x += 1.0;
    else if (m == 1) v1.x += 1.0;
    else v2.x += 1.0;
    const double vn = rsqrt(cabs2(v0) + cabs2(v1) + cabs2(v2));
    v0 = cscale(v0, vn);
    v1 = cscale(v1, vn);
    v2 = cscale(v2, vn);
    const double2 w0 = csub(cmul(u1, v2), cmul(u2, v1));
    const double2 w1 = csub(cmul(u2, v0), cmul(u0, v2));
    const double2 w2 = csub(cmul(u0, v1), cmul(u1, v0));
    o.num1[0] = v0;
    o.num1[1] = v1;
    o.num1[2] = v2;
    o.d[0] = w0;   // Pi2 = conj(w) -> d = w
    o.d[1] = w1;
    o.d[2] = w2;
    o.f1 = sig;
    o.f2 = sig;
}

// op: 0 = A_r (sigma_op = sqrt q), 1 = M (sigma_op = 1).  masked: Gamma mode.
__device__ __forceinline__ void coef(const ModeP& p, double2 l0, double2 l1, double2 l2, bool masked, int op, Coef& o) {
    const double q = cabs2(l0) + cabs2(l1) + cabs2(l2);
    o.d[0] = csub(l2, l1);
    o.d[1] = csub(l0, l2);
    o.d[2] = csub(l1, l0);
    const double p2 = cabs2(o.d[0]) + cabs2(o.d[1]) + cabs2(o.d[2]);
    if (masked || q == 0.0) {
        o.num1[0] = o.num1[1] = o.num1[2] = make_double2(0.0, 0.0);
        o.f1 = o.f2 = 0.0;
        return;
    }
    const double rq = rsqrt(q);
    if (p2 > p.taup * q) {
        const double r2 = rsqrt(p2);
        o.num1[0] = cj2(l1, o.d[2], l2, o.d[1]);
        o.num1[1] = cj2(l2, o.d[0], l0, o.d[2]);
        o.num1[2] = cj2(l0, o.d[1], l1, o.d[0]);
        if (op == 0) {
            o.f1 = r2;
            o.f2 = q * rq * r2;
        } else {
            o.f1 = rq * r2;
            o.f2 = r2;
        }
        return;
    }
    coef_fallback(l0, l1, l2, q, op == 0 ? q * rq : 1.0, o);
}

// v_l = num1_l U1 + conj(d_l) U2 with U1 = f1 u1, U2 = f2 u2
__device__ __forceinline__ double2 comb(const Coef& o, int l, double2 U1, double2 U2) {
    const double2 a = o.num1[l], d = o.d[l];
    return make_double2(fma(a.x, U1.x, fma(-a.y, U1.y, fma(d.x, U2.x, d.y * U2.y))),
                        fma(a.x, U1.y, fma(a.y, U1.x, fma(d.x, U2.y, -d.y * U2.x))));
}

}  // namespace modes
}  // namespace bnf
