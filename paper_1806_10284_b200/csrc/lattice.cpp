// Lattice canonicalisation and angle snapping: PAPER.md §2.2-2.3
// (P:L131-283).  Host code, no GPU.  Compiled with -ffp-contract=off so
// the integer decisions (m, rho) are taken in plain IEEE double.
#include <cmath>
#include <cstring>

#include "bnf_internal.h"

namespace bnf {

namespace {

double dot3(const double* x, const double* y) { return x[0] * y[0] + x[1] * y[1] + x[2] * y[2]; }
double norm3(const double* x) { return std::sqrt(dot3(x, x)); }

// P:L150-153 etc.: floor if 0 <= q - floor(q) < 1/2, ceil otherwise.
long long round_half_up(double q) {
    double f = std::floor(q);
    return (q - f < 0.5) ? (long long)f : (long long)f + 1;
}

double det3(const double* a) {  // column-major
    return a[0] * (a[4] * a[8] - a[7] * a[5]) - a[3] * (a[1] * a[8] - a[7] * a[2]) +
           a[6] * (a[1] * a[5] - a[4] * a[2]);
}

}  // namespace

int lattice_snap(const double a_raw[9], const int n[3], Lattice& L) {
    for (int d = 0; d < 3; ++d) {
        if (n[d] < 1) {
            set_error("grid sizes must be >= 1");
            return BNF_EINVAL;
        }
        L.n[d] = n[d];
    }
    // Canonical relabel: longest vector first (ties -> lowest index), cyclic.
    double len[3];
    for (int l = 0; l < 3; ++l) len[l] = norm3(a_raw + 3 * l);
    int p = 0;
    for (int l = 1; l < 3; ++l)
        if (len[l] > len[p]) p = l;
    for (int l = 0; l < 3; ++l) L.perm[l] = (p + l) % 3;
    double a[9];
    for (int l = 0; l < 3; ++l)
        for (int r = 0; r < 3; ++r) a[3 * l + r] = a_raw[3 * L.perm[l] + r];
    L.sign3 = 1;
    if (det3(a) < 0) {
        for (int r = 0; r < 3; ++r) a[6 + r] = -a[6 + r];
        L.sign3 = -1;
    }
    std::memcpy(L.a_canon, a, sizeof(a));
    const double L1 = norm3(a), L2 = norm3(a + 3), L3 = norm3(a + 6);
    L.lengths[0] = L1;
    L.lengths[1] = L2;
    L.lengths[2] = L3;
    const double cg_r = dot3(a, a + 3) / (L1 * L2);
    const double cb_r = dot3(a, a + 6) / (L1 * L3);
    const double ca_r = dot3(a + 3, a + 6) / (L2 * L3);
    L.cos_raw[0] = cg_r;
    L.cos_raw[1] = cb_r;
    L.cos_raw[2] = ca_r;
    const double sg_r = std::sqrt(std::fmax(0.0, 1.0 - cg_r * cg_r));
    // P:L143 admissibility
    if (!(L1 >= L2 && L1 >= L3)) {
        set_error("P:L143 |a1| >= |a2|,|a3| violated");
        return BNF_EGEOM;
    }
    if (!(L2 * sg_r > L3 * std::fabs(ca_r - cg_r * cb_r) / sg_r)) {
        set_error("P:L143 |a2| sin(gamma) > |a3||cos(alpha)-cos(gamma)cos(beta)|/sin(gamma) violated");
        return BNF_EGEOM;
    }
    const int n1 = n[0], n2 = n[1], n3 = n[2];
    const double dx = L1 / n1;
    long long m1, m2, m3;
    int rho1, rho2, rho3;
    double cg, cb, ca;
    // gamma -> m1
    if (cg_r >= 0.0) {
        m1 = round_half_up(L2 * cg_r / dx);
        cg = m1 * dx / L2;
        rho1 = 0;
    } else {
        m1 = round_half_up((L1 + L2 * cg_r) / dx);
        cg = (m1 * dx - L1) / L2;
        rho1 = 1;
    }
    if (std::fabs(cg) >= 1.0) {
        set_error("|cos gamma| >= 1 after snapping");
        return BNF_EGEOM;
    }
    const double sg = std::sqrt(1.0 - cg * cg);
    const double l2 = L2 * sg;
    const double dy = l2 / n2;
    // beta -> m2
    if (cb_r >= 0.0) {
        m2 = round_half_up(L3 * cb_r / dx);
        cb = m2 * dx / L3;
        rho2 = 0;
    } else {
        m2 = round_half_up((L1 + L3 * cb_r) / dx);
        cb = (m2 * dx - L1) / L3;
        rho2 = 1;
    }
    if (std::fabs(cb) >= 1.0) {
        set_error("|cos beta| >= 1 after snapping");
        return BNF_EGEOM;
    }
    // alpha -> m3; D' = 0 taken as Case I
    const double D = ca_r - cg * cb;
    if (D >= 0.0) {
        m3 = round_half_up(L3 * D / (dy * sg));
        ca = m3 * dy * sg / L3 + cg * cb;
        rho3 = 0;
    } else {
        m3 = round_half_up((L2 * sg * sg + L3 * D) / (dy * sg));
        ca = (m3 * dy * sg - L2 * sg * sg) / L3 + cg * cb;
        rho3 = 1;
    }
    if (!(m1 >= 0 && m1 <= n1 && m2 >= 0 && m2 <= n1 && m3 >= 0 && m3 <= n2)) {
        set_error("snapped m outside 0<=m1,m2<=n1, 0<=m3<=n2 (P:L148-201)");
        return BNF_EGEOM;
    }
    const double vol = 1.0 - cg * cg - cb * cb - ca * ca + 2.0 * cg * cb * ca;
    if (!(vol > 0.0)) {
        set_error("degenerate cell after snapping");
        return BNF_EGEOM;
    }
    L.m[0] = (int)m1;
    L.m[1] = (int)m2;
    L.m[2] = (int)m3;
    L.rho[0] = rho1;
    L.rho[1] = rho2;
    L.rho[2] = rho3;
    L.cos_snap[0] = cg;
    L.cos_snap[1] = cb;
    L.cos_snap[2] = ca;
    // eq. (transvec), column-major
    double A[9] = {L1, 0.0, 0.0,
                   L2 * cg, L2 * sg, 0.0,
                   L3 * cb, L3 * (ca - cg * cb) / sg, L3 * std::sqrt(vol) / sg};
    std::memcpy(L.a, A, sizeof(A));
    L.l[0] = L1;
    L.l[1] = l2;
    L.l[2] = A[8];
    L.delta[0] = dx;
    L.delta[1] = dy;
    L.delta[2] = A[8] / n3;
    long long Ag[9] = {n1, 0, 0,
                       m1 - (long long)rho1 * n1, n2, 0,
                       m2 - (long long)rho2 * n1, m3 - (long long)rho3 * n2, n3};
    std::memcpy(L.Ag, Ag, sizeof(Ag));
    return BNF_OK;
}

int j3_category(const Lattice& L) {
    if (L.rho[2] == 0) return L.m[0] <= L.m[1] ? 1 : 2;
    return (L.m[0] + L.m[1] <= L.n[0]) ? 3 : 4;
}

}  // namespace bnf
