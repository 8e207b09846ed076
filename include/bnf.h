/*
 * bnf.h -- C ABI of the B200-native null-space-free Yee-curl band solver.
 *
 * Method: Huang, Li, Li, Lin, Lin, Tian, "Eigenvalue problems of discrete
 * curl operators on various lattices for simulating three dimensional
 * photonic crystals" (arXiv 1806.10284).  Citations "P:Lnnn" are lines of
 * that paper's text.
 *
 * Problem statement (P:L64-90, L123-226, L323-332, L1642-1646, L2248-2251,
 * L2396-2398): given primitive lattice vectors, a grid n1 x n2 x n3, the
 * permittivity sampled at the Yee edge midpoints (B), and a Bloch vector,
 * find the nev smallest NONZERO eigenvalues lambda = omega^2 (mu0 = eps0 = 1,
 * lattice units) of  C^* C e = lambda B e,  via the null-space-free
 * standard problem  A_r y = lambda y,  A_r = Sigma_r Q_r^* B^{-1} Q_r Sigma_r.
 *
 * ---------------------------------------------------------------------------
 * Layouts (all arrays x-fastest, "vec" of P:L331):
 *   real space   index(a,b,c) = a + n1*(b + n2*c), component l occupies
 *                [l*n, (l+1)*n);  E_l lives at the Yee point of component l.
 *   Fourier side index(i,j,k) = i + n1*(j + n2*k);  a 2n vector y = [y1; y2]
 *                holds the coefficients on the columns Q_1, Q_2 of Q_r
 *                (P:L2214-2219).  Fourier mode (i,j,k) is the Bloch plane
 *                wave exp(2 pi i (a g1 + b g2 + c g3)) with
 *                  g1 = (i + kappa1)/n1,
 *                  g2 = (j - m1 i/n1 + kappa^2)/n2          (Thm eigK2)
 *                  g3 = (k - m3 j/n2 + c_b i + kappa^3)/n3  (Thms eigK3)
 *                i.e. column (i,j,k) of the unitary T of eq. (T);
 *                the paper's column order (i slowest) is a permutation of ours.
 *   complex128   interleaved (re, im) doubles.
 *
 * Conventions: the caller owns every buffer it passes; the library owns the
 * opaque handles and their device workspaces.  A handle is not thread-safe.
 * Device work is issued on opts.stream; every call returns after the stream
 * has been synchronised.  Every entry point returns a status code; on failure
 * bnf_last_error() (thread-local) describes it.  There is no CPU fallback:
 * without a usable CUDA device the solver calls return BNF_ECUDA.
 */
#ifndef BNF_H
#define BNF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BNF_VERSION 1

/* status codes */
#define BNF_OK 0
#define BNF_EINVAL 1    /* bad argument: grid < 1, NULL pointer, size mismatch, unsupported axis length */
#define BNF_EGEOM 2     /* P:L143 admissibility violated after canonicalisation, or degenerate snapped cell */
#define BNF_ENOMEM 3    /* device or host allocation failed */
#define BNF_ECUDA 4     /* CUDA runtime error (no device, launch failure, ...) */
#define BNF_ENCCL 5     /* NCCL failure or libnccl.so.2 not loadable (distributed slab mode) */
#define BNF_ENOCONV 6   /* eigensolver did not reach tolerance; partial results + residuals in stats */
#define BNF_ESTATE 7    /* call order violated (e.g. solve before bnf_set_epsilon) */

/* memory kinds */
#define BNF_MEM_HOST 0
#define BNF_MEM_DEVICE 1

/* operators for bnf_apply_Ar */
#define BNF_OP_AR 0     /* A_r = Sigma_r Q_r^* B^{-1} Q_r Sigma_r   (NFSEP) */
#define BNF_OP_M 1      /* M   = Q_r^* B^{-1} Q_r                   (CG operator) */

/* vectors for bnf_eigvecs */
#define BNF_VEC_Y 0     /* NFSEP eigenvectors y (2n complex each, unit 2-norm) */
#define BNF_VEC_E 1     /* E-field eigenvectors e = B^{-1} Q_r Sigma_r y / sqrt(lambda) (3n complex,
                           e^* B e = 1), real-space Yee layout, Bloch phase included */
#define BNF_VEC_H 2     /* H-field eigenvectors h = C e / (i omega) = -i P_r y (3n complex, h^* h = 1;
                           C = P_r Sigma_r Q_r^*; Maxwell's curl equation):
                           computed in the Fourier domain as -i T (lambda x (Pi1 y1 + Pi2 y2) / sigma) per
                           mode, same real-space layout and Bloch phase as BNF_VEC_E; C^* h = -i omega B e */

typedef struct bnf_lattice bnf_lattice;
typedef struct bnf_solver bnf_solver;

/* Snapped lattice (§2.2, eq. transvec).  Matrices column-major:
   x[3*l + r] is Cartesian component r of vector l. */
typedef struct {
    int n[3];            /* grid n1, n2, n3 */
    int perm[3];         /* canonical vector l is raw vector perm[l] (cyclic relabel, longest first) */
    int sign3;           /* -1 if canonical a3 was negated to make the triple right-handed */
    int m[3];            /* m1, m2, m3 */
    int rho[3];          /* rho1, rho2, rho3: 1 for the obtuse Case II of gamma, beta, alpha */
    int category;        /* J3 general category 1..4 */
    double lengths[3];   /* |a1|, |a2|, |a3| (canonical order) */
    double cos_raw[3];   /* cos gamma', cos beta', cos alpha' before snapping */
    double cos_snap[3];  /* corrected cos gamma, cos beta, cos alpha */
    double a[9];         /* corrected vectors a1..a3, eq. (transvec), upper triangular */
    double a_canon[9];   /* canonical raw vectors in the ORIGINAL Cartesian frame */
    double l[3];         /* cell extents l1, l2, l3 */
    double delta[3];     /* grid spacings dx, dy, dz */
    long long Ag[9];     /* a = diag(delta) Ag: integer lattice in grid units, upper triangular */
} bnf_lattice_info;

/* Canonicalise and snap.  a_raw: 3 primitive vectors as
   columns (a_raw[3*l + r]) in any Cartesian frame.  n: grid.  Returns
   BNF_EINVAL (n < 1), BNF_EGEOM (P:L143 violated, |cos| >= 1 after snapping,
   m outside [0,n1]x[0,n1]x[0,n2], degenerate cell).  Host-only, no GPU. */
int bnf_lattice_create(const double a_raw[9], const int n[3], bnf_lattice** out);
int bnf_lattice_query(const bnf_lattice* lat, bnf_lattice_info* info);
void bnf_lattice_destroy(bnf_lattice* lat);

/* Reduced Bloch numbers kappa_l = K . a~_l / (2 pi), with K the physical
   Bloch vector "2 pi k" in the frame of a_raw and a~ the
   canonical vectors.  Host-only. */
int bnf_kvec_reduce(const bnf_lattice* lat, const double K_cart[3], double kappa[3]);

/* Reduced Bloch numbers given in the labelling of a_raw (kappa_raw_l =
   K . a_raw_l / 2 pi) -> the canonical labelling the solver uses: canonical
   vector l is raw vector perm[l] (cyclic relabel, longest first) and
   kappa_3 changes sign when a3 was negated (DESIGN R10).  Host-only. */
int bnf_kappa_canonical(const bnf_lattice* lat, const double kappa_raw[3], double kappa[3]);

/* Yee points of component comp (0, 1, 2) at which B_comp is sampled
   (the edge midpoints x(a+1/2,b,c), x(a,b+1/2,c), x(a,b,c+1/2)
   of the grid of the snapped lattice).  xyz: HOST, n1*n2*n3 rows
   of 3 doubles, x fastest (row a + n1 (b + n2 c)); caller-owned.
   frame = BNF_FRAME_SNAPPED: Cartesian coordinates ((a+h1)dx, (b+h2)dy,
   (c+h3)dz) in the transformed frame of the corrected vectors a1..a3;
   BNF_FRAME_ORIGINAL: the point's fractional coordinates in the snapped cell,
   wrapped into [0, 1)^3, applied to the canonical raw vectors a_canon (the
   original Cartesian frame; the map used to sample shapes defined there,
   DESIGN §4).  BNF_EINVAL on a NULL pointer, comp or frame out of range.
   Host-only. */
#define BNF_FRAME_SNAPPED 0
#define BNF_FRAME_ORIGINAL 1
int bnf_yee_points(const bnf_lattice* lat, int comp, int frame, double* xyz);

typedef struct {
    int device;                 /* CUDA device ordinal */
    void* stream;               /* cudaStream_t to issue work on; NULL = legacy default stream */
    double tol_outer;           /* 1e-12: Ritz relative residual of A_r^{-1} (DESIGN R12) */
    double tol_inner;           /* 1e-13: CG relative residual ||r|| <= tol ||c|| */
    int max_outer;              /* max block-Lanczos steps; 0 (default) = auto:
                                   max(60, 12 ceil((nev + guard) / block)), capped by the NFSEP
                                   dimension.  BNF_EINVAL from bnf_solve if max_outer * block
                                   < nev + guard.  The basis grows on demand (VMM mapping). */
    int max_inner;              /* max CG iterations per solve */
    int block;                  /* Lanczos block size b >= 1 (DESIGN R13) */
    int guard;                  /* extra Ritz pairs converged beyond nev */
    unsigned long long seed;    /* start-block seed (counter-based generator) */
    int refine;                 /* 1: final subspace-iteration + Rayleigh-Ritz on A_r (DESIGN R15) */
    int profile;                /* 1: time every kernel with CUDA events (bnf_kernel_times) */
    int warm;                   /* 1: start each solve from the previous solve's Ritz vectors
                                   (neighbouring k on a path; DESIGN R17); 0: seeded random block */
    int reorth_once_ok;         /* 1: skip the second Gram-Schmidt pass when the first kept every
                                   column's norm above 1/sqrt(2) (DGKS test; DESIGN R18); 0: always twice */
    double res_tol;             /* 5e-9: with refine >= 1, repeat a step of subspace inverse iteration +
                                   Rayleigh-Ritz while max ||A_r y - lambda y|| / ||y|| > res_tol
                                   (north-star eigenvector bar 1e-8; DESIGN R19) */
    int max_polish;             /* at most this many such extra steps (3) */
    int slabs;                  /* 1 (default): whole grid.  P > 1: run the slab-decomposed operator of
                                   SURVEY §8(e) on this one device ("virtual slabs", the multi-GPU data
                                   layout with the all-to-alls as device copies): Fourier-side vectors
                                   are laid out [slab][half][k][jl][i] with jl < n2/P (slab r holds
                                   j = r n2/P + jl), real-space work in z-slabs of n3/P planes.
                                   Needs n2, n3 divisible by P, a square xy plane of 64/128/256.
                                   bnf_apply_Ar / BNF_VEC_Y use that layout; BNF_VEC_E is refused. */
    int relax_inner;            /* 0 (default, the paper's fixed tol_inner).  1: NEXT-1 inexact
                                   inner solves -- Lanczos step j solves to tol_inner * clamp(1e-6 /
                                   res_{j-1}, 1, 1e5), res = the largest relative Ritz residual of the
                                   wanted pairs; the final Rayleigh-Ritz + residual polish (res_tol,
                                   exact inner tolerance) secure the returned pairs. */
    int method;                 /* eigensolver: 0 (default) = the paper's inverse Lanczos with CG inner
                                   solves; 1 = NEXT-1 LOBPCG on A_r preconditioned by
                                   Sigma_r^{-2} (no inner solves; block nev + guard, soft locking),
                                   stopping at ||A_r y - lambda y|| <= min(res_tol, 1e-9 max(1, lambda)),
                                   falling back to method 0 on stagnation or breakdown; max_outer = iteration
                                   cap (0: 1000); block / tol_outer / tol_inner are not used. */
} bnf_opts;

void bnf_opts_default(bnf_opts* opts);

typedef struct {
    int outer_steps;            /* block-Lanczos steps */
    int converged;              /* 1 if all nev + guard Ritz pairs met tol_outer */
    long long inner_iters;      /* CG iterations summed over right-hand sides */
    long long matvecs;          /* single-vector applications of M or A_r executed by the kernels */
    long long kernel_launches;  /* kernels launched during the call */
    double max_ritz_residual;   /* max_i |beta s_i| / |theta_i| at exit (A_r^{-1} Ritz pairs) */
    double max_residual;        /* max_i ||A_r y_i - lambda_i y_i|| / ||y_i|| of the returned pairs */
    double seconds;             /* wall time of the call */
    int polish_steps;           /* extra inverse-iteration + Rayleigh-Ritz steps taken for res_tol */
    int polish_failed;          /* 1 if a polish step's block was rank deficient (CholQR failed): the
                                   previous Ritz pairs were kept and polishing stopped */
    long long active_matvecs;   /* the part of matvecs applied to right-hand sides still iterating: a block
                                   CG keeps applying M to its converged columns until the last one stops
                                   (matvecs - active_matvecs is that overhead) */
} bnf_stats;

/* Create a solver for a lattice on opts->device.  Allocates device memory
   for the operator work arrays.  Any axis length up to 1024: lengths with a
   register-FFT plan (8, 12, 16, 24, 32, 48, 64, 96, 128, 192, 256) take the
   fused fast path, the others generic Stockham passes (a prime factor > 31 is
   evaluated as a direct DFT stage).  BNF_EINVAL beyond 1024. */
int bnf_solver_create(const bnf_lattice* lat, const bnf_opts* opts, bnf_solver** out);
void bnf_solver_destroy(bnf_solver* s);

/* Distributed slab mode (one k-point on several GPUs,
   one process per GPU; §5.3 Algorithms 1-2 with the 3D transforms
   split).  nranks processes each own one slab: the Fourier side of every
   vector is split over j (rank r holds j in [r n2/P, (r+1) n2/P), all i, k:
   local vectors of 2n/P complex laid out [half][k][jl][i]), the real-space
   work over z-planes (rank r holds n3/P planes).  Per operator application
   two all-to-alls (NCCL send/recv groups, 3 nvec n/P^2 complex per rank pair)
   move the real-space blocks; the CG partial sums are all-gathered and the
   Lanczos Gram products all-reduced, so every rank holds the same small
   matrices and returns the same eigenvalues.  Needs n2, n3 divisible by
   nranks and the fast square-plane path (as opts.slabs).  `id` is the NCCL
   unique id of the group (bnf_nccl_unique_id on one rank, broadcast by the
   caller); opts.device is this rank's GPU.  bnf_set_epsilon takes the full
   3n field (each rank keeps its slab); bnf_apply_Ar / BNF_VEC_Y use local
   vectors; BNF_VEC_E is refused.  Every rank must make the same calls in the
   same order (collectives).  BNF_ENCCL on an NCCL error. */
int bnf_nccl_unique_id(unsigned char id[128]);
int bnf_solver_create_dist(const bnf_lattice* lat, const bnf_opts* opts, int nranks, int rank, const unsigned char id[128],
                           bnf_solver** out);

/* Permittivity B: eps[3n] = [vec B1; vec B2; vec B3], real-space
   layout, every value > 0 (BNF_EINVAL otherwise).  mem = BNF_MEM_HOST or
   BNF_MEM_DEVICE (device pointer to 3n doubles).  Copied; caller keeps ownership. */
int bnf_set_epsilon(bnf_solver* s, const double* eps, int mem);

/* Per-k setup: reduced Bloch numbers kappa (canonical
   labelling).  When every kappa_l is an integer (Gamma) the single
   Fourier mode with g = 0 is masked (Sigma_r = Pi = 0 there; DESIGN R6). */
int bnf_set_kappa(bnf_solver* s, const double kappa[3]);

/* Hot-path hook: out = op(y) for b vectors.  y, out: DEVICE pointers to
   complex128 [b][2][n] (Fourier layout).  out may not alias y.  Uses the
   kappa of the last bnf_set_kappa / bnf_solve. */
int bnf_apply_Ar(bnf_solver* s, const void* y, void* out, int b, int op);

/* Inner solve hook: x = M^{-1} c by the
   solver's CG (CG-fused passes, CUDA-graph loop unless profiling is on) for b
   right-hand sides, stopping per column at ||r|| <= tol_inner ||c|| or after
   max_iter iterations.  c, x: DEVICE complex128 [b][2][n], caller-owned, may
   not alias.  *iters (may be NULL) = iterations run.  Uses the kappa of the
   last bnf_set_kappa.  BNF_ESTATE before bnf_set_epsilon / bnf_set_kappa. */
int bnf_cg_solve(bnf_solver* s, const void* c, void* x, int b, int max_iter, int* iters);

/* Solve: nev smallest nonzero eigenvalues of the GEP at
   kappa, ascending, written to lambda[nev] (HOST).  Eigenvectors stay on the
   device; fetch them with bnf_eigvecs.  stats may be NULL.  Returns
   BNF_ENOCONV (with results) if the tolerance was not reached. */
int bnf_solve(bnf_solver* s, const double kappa[3], int nev, double* lambda, bnf_stats* stats);

/* Eigenvectors of the last solve: kind = BNF_VEC_Y (out: nev x 2n complex),
   BNF_VEC_E or BNF_VEC_H (out: nev x 3n complex), mem = HOST or DEVICE. */
int bnf_eigvecs(bnf_solver* s, int kind, void* out, int mem);

/* Per-kernel device time (ms) accumulated since the last reset while
   opts.profile = 1.  Writes up to cap entries: names[i] (static strings),
   ms[i], launches[i]; returns the number of kernel kinds in *count. */
int bnf_kernel_times(bnf_solver* s, const char** names, double* ms, long long* launches, int cap, int* count);
int bnf_kernel_times_reset(bnf_solver* s);

/* Switch per-kernel timing on (1) or off (0) after creation (opts.profile).
   With profiling on, the CG loop runs eagerly with one CUDA-event pair per
   kernel and a host convergence check per iteration; with it off the CG loop
   is one CUDA graph with a device-side while condition (no host round trip
   per iteration).  Both paths execute the same kernels on the same data. */
int bnf_set_profile(bnf_solver* s, int on);

/* Diagnostics: per-phase clock64() cycle sums of the plane pass, collected
   only when the solver was created with the environment variable
   BNF_PHASE_PROF set (thread 0 of every CTA; entry 15 = CTA count).  Copies
   min(cap, 16) counters to out (HOST) and resets them. */
int bnf_phase_counters(bnf_solver* s, unsigned long long* out, int cap);

const char* bnf_last_error(void);
int bnf_version(void);

/* Testing hooks (host-only, no GPU): Hermitian eigensolver used for the
   Rayleigh-Ritz / block-tridiagonal steps.  a: n x n complex row-major
   (interleaved), overwritten; w: n eigenvalues ascending; z: n x n complex
   row-major eigenvectors (columns), may be NULL. */
int bnf_host_herm_eig(int n, double* a, double* w, double* z);

#ifdef __cplusplus
}
#endif
#endif /* BNF_H */
