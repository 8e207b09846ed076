/* Pure-C consumer of include/bnf.h: the library's boundary used without any
 * Python or torch.  Reads the oracle fixture tests/golden/c_abi_fcc654.bin
 * (scripts/make_c_fixture.py: dense oracle A_r and M on a 6x5x4 FCC grid),
 * creates a lattice and a solver, uploads eps from host memory, applies
 * bnf_apply_Ar to device copies of the vectors for op = A_r and M and checks
 * the result against the oracle (max |got - want| <= 1e-12 max |want|).
 * Without a CUDA device it checks the host-only calls and that the solver
 * refuses to run (BNF_ECUDA: no CPU fallback), and exits 0 with "no-gpu".
 *
 *   consumer <fixture.bin>      exit 0 = pass
 */
#include <cuda_runtime_api.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "bnf.h"

static int fail(const char* what, int rc) {
    fprintf(stderr, "FAIL %s: rc=%d %s\n", what, rc, bnf_last_error());
    return 1;
}

int main(int argc, char** argv) {
    if (argc < 2) {
        fprintf(stderr, "usage: consumer fixture.bin\n");
        return 2;
    }
    FILE* f = fopen(argv[1], "rb");
    if (!f) return fail("open fixture", -1);
    int hdr[5];
    double a_raw[9], kappa[3];
    if (fread(hdr, sizeof(int), 5, f) != 5 || fread(a_raw, sizeof(double), 9, f) != 9 ||
        fread(kappa, sizeof(double), 3, f) != 3)
        return fail("read header", -1);
    const int n[3] = {hdr[0], hdr[1], hdr[2]}, b = hdr[3], nops = hdr[4];
    const size_t nn = (size_t)n[0] * n[1] * n[2], len = (size_t)b * 2 * nn;
    double* eps = (double*)malloc(3 * nn * sizeof(double));
    double* y = (double*)malloc(2 * len * sizeof(double));
    double* want = (double*)malloc(2 * len * nops * sizeof(double));
    double* got = (double*)malloc(2 * len * sizeof(double));
    if (fread(eps, sizeof(double), 3 * nn, f) != 3 * nn || fread(y, sizeof(double), 2 * len, f) != 2 * len ||
        fread(want, sizeof(double), 2 * len * nops, f) != 2 * len * nops)
        return fail("read arrays", -1);
    fclose(f);

    bnf_lattice* lat = NULL;
    int rc = bnf_lattice_create(a_raw, n, &lat);
    if (rc != BNF_OK) return fail("bnf_lattice_create", rc);
    bnf_lattice_info info;
    if ((rc = bnf_lattice_query(lat, &info)) != BNF_OK) return fail("bnf_lattice_query", rc);
    double kc[3];
    if ((rc = bnf_kappa_canonical(lat, kappa, kc)) != BNF_OK) return fail("bnf_kappa_canonical", rc);
    printf("lattice m = (%d, %d, %d), category %d, version %d\n", info.m[0], info.m[1], info.m[2], info.category,
           bnf_version());

    bnf_opts opts;
    bnf_opts_default(&opts);
    bnf_solver* s = NULL;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        rc = bnf_solver_create(lat, &opts, &s);
        bnf_lattice_destroy(lat);
        if (rc != BNF_ECUDA) return fail("solver without GPU must return BNF_ECUDA", rc);
        printf("no-gpu: host calls ok, solver refused (BNF_ECUDA)\n");
        return 0;
    }
    if ((rc = bnf_solver_create(lat, &opts, &s)) != BNF_OK) return fail("bnf_solver_create", rc);
    if ((rc = bnf_set_epsilon(s, eps, BNF_MEM_HOST)) != BNF_OK) return fail("bnf_set_epsilon", rc);
    if ((rc = bnf_set_kappa(s, kappa)) != BNF_OK) return fail("bnf_set_kappa", rc);
    void *dy = NULL, *dout = NULL;
    if (cudaMalloc(&dy, 2 * len * sizeof(double)) != cudaSuccess || cudaMalloc(&dout, 2 * len * sizeof(double)) != cudaSuccess)
        return fail("cudaMalloc", -1);
    cudaMemcpy(dy, y, 2 * len * sizeof(double), cudaMemcpyHostToDevice);
    const int ops[2] = {BNF_OP_AR, BNF_OP_M};
    int bad = 0;
    for (int o = 0; o < nops && o < 2; ++o) {
        if ((rc = bnf_apply_Ar(s, dy, dout, b, ops[o])) != BNF_OK) return fail("bnf_apply_Ar", rc);
        cudaMemcpy(got, dout, 2 * len * sizeof(double), cudaMemcpyDeviceToHost);
        const double* w = want + (size_t)o * 2 * len;
        double err = 0.0, ref = 0.0;
        for (size_t t = 0; t < len; ++t) {
            const double dr = got[2 * t] - w[2 * t], di = got[2 * t + 1] - w[2 * t + 1];
            const double e = sqrt(dr * dr + di * di), r = sqrt(w[2 * t] * w[2 * t] + w[2 * t + 1] * w[2 * t + 1]);
            if (e > err) err = e;
            if (r > ref) ref = r;
        }
        printf("op %s: max |got - want| / max |want| = %.3e\n", o == 0 ? "A_r" : "M", err / ref);
        if (!(err <= 1e-12 * ref)) bad = 1;
    }
    double lam[4];
    bnf_stats st;
    if ((rc = bnf_solve(s, kappa, 4, lam, &st)) != BNF_OK) return fail("bnf_solve", rc);
    printf("lambda = %.12f %.12f %.12f %.12f (%lld matvecs)\n", lam[0], lam[1], lam[2], lam[3], st.matvecs);
    cudaFree(dy);
    cudaFree(dout);
    bnf_solver_destroy(s);
    bnf_lattice_destroy(lat);
    free(eps);
    free(y);
    free(want);
    free(got);
    if (bad) return fail("parity", -1);
    printf("pass\n");
    return 0;
}
