// Internal declarations shared by the native sources (not part of the ABI).
#pragma once

#include <complex>
#include <cstdint>
#include <string>
#include <vector>

#include "bnf.h"

namespace bnf {

using cd = std::complex<double>;

void set_error(const std::string& msg);

struct Status {
    int code = BNF_OK;
};

// Snapped lattice (§2.2, eq. transvec); host only.
struct Lattice {
    int n[3];
    int perm[3];
    int sign3;
    int m[3];
    int rho[3];
    double lengths[3];
    double cos_raw[3];
    double cos_snap[3];
    double a[9];        // column-major
    double a_canon[9];  // column-major
    double l[3];
    double delta[3];
    long long Ag[9];    // column-major
};

int lattice_snap(const double a_raw[9], const int n[3], Lattice& out);
int j3_category(const Lattice& L);

// Host dense linear algebra (linalg_host.cpp)
// Hermitian eigen-decomposition, n x n row-major; w ascending; z columns.
void herm_eig(int n, std::vector<cd>& a, std::vector<double>& w, std::vector<cd>* z);
// Cholesky of an n x n HPD matrix (row-major), returns false if not PD.
bool cholesky_upper(int n, const std::vector<cd>& g, std::vector<cd>& r);
// Inverse of an upper-triangular matrix.
void inv_upper(int n, const std::vector<cd>& r, std::vector<cd>& rinv);

}  // namespace bnf
