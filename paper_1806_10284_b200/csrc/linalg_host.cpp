// Small dense host linear algebra for the eigensolver's projected problems
// (block-tridiagonal Ritz step, Cholesky-QR, Rayleigh-Ritz).  Sizes are at
// most a few hundred, so O(n^3) host work is negligible next to the
// device matvecs.
#include <algorithm>
#include <cmath>
#include <numeric>

#include "bnf_internal.h"

namespace bnf {

// Hermitian eigen-decomposition: Householder reduction to a real symmetric
// tridiagonal matrix (unitary similarity, then a diagonal phase scaling)
// followed by the implicit QL algorithm with Wilkinson shifts.
void herm_eig(int n, std::vector<cd>& A, std::vector<double>& w, std::vector<cd>* Zout) {
    w.assign(n, 0.0);
    if (n == 0) return;
    const bool want = Zout != nullptr;
    std::vector<cd> Q;
    if (want) {
        Q.assign((size_t)n * n, 0.0);
        for (int i = 0; i < n; ++i) Q[(size_t)i * n + i] = 1.0;
    }
    std::vector<cd> v(n), p(n), wv(n);
    for (int k = 0; k + 2 < n; ++k) {
        double xnorm2 = 0.0;
        for (int r = k + 1; r < n; ++r) xnorm2 += std::norm(A[(size_t)r * n + k]);
        if (xnorm2 == 0.0) continue;
        const double xnorm = std::sqrt(xnorm2);
        const cd x0 = A[(size_t)(k + 1) * n + k];
        const cd phase = (std::abs(x0) > 0.0) ? x0 / std::abs(x0) : cd(1.0, 0.0);
        const cd alpha = -phase * xnorm;
        std::fill(v.begin(), v.end(), cd(0.0));
        for (int r = k + 1; r < n; ++r) v[r] = A[(size_t)r * n + k];
        v[k + 1] -= alpha;
        double vn2 = 0.0;
        for (int r = k + 1; r < n; ++r) vn2 += std::norm(v[r]);
        if (vn2 == 0.0) continue;
        const double vn = std::sqrt(vn2);
        for (int r = k + 1; r < n; ++r) v[r] /= vn;
        // p = A v ; K = v^H p ; w = p - K v ; A -= 2 v w^H + 2 w v^H
        for (int r = 0; r < n; ++r) {
            cd s = 0.0;
            for (int c = k + 1; c < n; ++c) s += A[(size_t)r * n + c] * v[c];
            p[r] = s;
        }
        cd K = 0.0;
        for (int r = k + 1; r < n; ++r) K += std::conj(v[r]) * p[r];
        for (int r = 0; r < n; ++r) wv[r] = p[r] - K * v[r];
        for (int r = 0; r < n; ++r) {
            for (int c = 0; c < n; ++c) {
                A[(size_t)r * n + c] -= 2.0 * (v[r] * std::conj(wv[c]) + wv[r] * std::conj(v[c]));
            }
        }
        if (want) {  // Q <- Q H,  H = I - 2 v v^H
            for (int r = 0; r < n; ++r) {
                cd s = 0.0;
                for (int c = k + 1; c < n; ++c) s += Q[(size_t)r * n + c] * v[c];
                for (int c = k + 1; c < n; ++c) Q[(size_t)r * n + c] -= 2.0 * s * std::conj(v[c]);
            }
        }
    }
    // Real tridiagonal via D = diag(phases)
    std::vector<double> d(n), e(n, 0.0);
    std::vector<cd> D(n, cd(1.0, 0.0));
    for (int j = 0; j < n; ++j) d[j] = A[(size_t)j * n + j].real();
    for (int j = 0; j + 1 < n; ++j) {
        const cd c = A[(size_t)(j + 1) * n + j];
        const double ac = std::abs(c);
        e[j] = ac;
        D[j + 1] = (ac > 0.0) ? D[j] * (c / ac) : D[j];
    }
    // Implicit QL (Wilkinson shift) with accumulation of rotations in Z.  The loop
    // structure (tst1 test, c2/c3/s2, el1/dl1) follows the public-domain EISPACK
    // tql2 routine (Bowdler, Martin, Reinsch, Wilkinson; as in JAMA's tql2).
    std::vector<double> Z;
    if (want) {
        Z.assign((size_t)n * n, 0.0);
        for (int i = 0; i < n; ++i) Z[(size_t)i * n + i] = 1.0;
    }
    const double eps = std::ldexp(1.0, -52);
    double f = 0.0, tst1 = 0.0;
    for (int l = 0; l < n; ++l) {
        tst1 = std::max(tst1, std::fabs(d[l]) + std::fabs(e[l]));
        int m = l;
        while (m < n - 1) {
            if (std::fabs(e[m]) <= eps * tst1) break;
            ++m;
        }
        if (m > l) {
            int iter = 0;
            do {
                if (++iter > 200) break;
                double g = d[l];
                double pp = (d[l + 1] - g) / (2.0 * e[l]);
                double r = std::hypot(pp, 1.0);
                if (pp < 0) r = -r;
                d[l] = e[l] / (pp + r);
                d[l + 1] = e[l] * (pp + r);
                const double dl1 = d[l + 1];
                double h = g - d[l];
                for (int i = l + 2; i < n; ++i) d[i] -= h;
                f += h;
                pp = d[m];
                double c = 1.0, c2 = 1.0, c3 = 1.0;
                const double el1 = e[l + 1];
                double s = 0.0, s2 = 0.0;
                for (int i = m - 1; i >= l; --i) {
                    c3 = c2;
                    c2 = c;
                    s2 = s;
                    g = c * e[i];
                    h = c * pp;
                    r = std::hypot(pp, e[i]);
                    e[i + 1] = s * r;
                    s = e[i] / r;
                    c = pp / r;
                    pp = c * d[i] - s * g;
                    d[i + 1] = h + s * (c * g + s * d[i]);
                    if (want) {
                        for (int k = 0; k < n; ++k) {
                            const double zh = Z[(size_t)k * n + i + 1];
                            Z[(size_t)k * n + i + 1] = s * Z[(size_t)k * n + i] + c * zh;
                            Z[(size_t)k * n + i] = c * Z[(size_t)k * n + i] - s * zh;
                        }
                    }
                }
                pp = -s * s2 * c3 * el1 * e[l] / dl1;
                e[l] = s * pp;
                d[l] = c * pp;
            } while (std::fabs(e[l]) > eps * tst1);
        }
        d[l] += f;
        e[l] = 0.0;
    }
    std::vector<int> ord(n);
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return d[x] < d[y]; });
    for (int i = 0; i < n; ++i) w[i] = d[ord[i]];
    if (want) {
        // eigenvectors of the Hermitian matrix: X = Q D Z
        std::vector<cd>& X = *Zout;
        X.assign((size_t)n * n, 0.0);
        for (int r = 0; r < n; ++r) {
            for (int col = 0; col < n; ++col) {
                const int oc = ord[col];
                cd s = 0.0;
                for (int t = 0; t < n; ++t) s += Q[(size_t)r * n + t] * D[t] * Z[(size_t)t * n + oc];
                X[(size_t)r * n + col] = s;
            }
        }
    }
}

// G = R^H R with R upper triangular (row-major n x n).
bool cholesky_upper(int n, const std::vector<cd>& G, std::vector<cd>& R) {
    R.assign((size_t)n * n, 0.0);
    for (int i = 0; i < n; ++i) {
        double dsum = G[(size_t)i * n + i].real();
        for (int k = 0; k < i; ++k) dsum -= std::norm(R[(size_t)k * n + i]);
        if (!(dsum > 0.0)) return false;
        const double rii = std::sqrt(dsum);
        R[(size_t)i * n + i] = rii;
        for (int j = i + 1; j < n; ++j) {
            cd s = G[(size_t)i * n + j];
            for (int k = 0; k < i; ++k) s -= std::conj(R[(size_t)k * n + i]) * R[(size_t)k * n + j];
            R[(size_t)i * n + j] = s / rii;
        }
    }
    return true;
}

void inv_upper(int n, const std::vector<cd>& R, std::vector<cd>& Ri) {
    Ri.assign((size_t)n * n, 0.0);
    for (int j = 0; j < n; ++j) {
        Ri[(size_t)j * n + j] = 1.0 / R[(size_t)j * n + j];
        for (int i = j - 1; i >= 0; --i) {
            cd s = 0.0;
            for (int k = i + 1; k <= j; ++k) s += R[(size_t)i * n + k] * Ri[(size_t)k * n + j];
            Ri[(size_t)i * n + j] = -s / R[(size_t)i * n + i];
        }
    }
}

}  // namespace bnf
