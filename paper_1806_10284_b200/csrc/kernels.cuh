// Device-side parameter blocks and kernel launchers (internal).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace bnf {

// One DFT axis: Stockham radix plan + root table e^{2 pi i t / N}.
struct AxisPlan {
    int N;
    int nst;
    int R[12];
    const double2* root;    // e^{2 pi i t / N}, t < N (generic Stockham passes)
    const double2* root2;   // fast plan N = N1*N2: e^{2 pi i t k1 / N} at [k1 * N2 + t] (fastfft.cuh)
};

// Per-k mode parameters.  Fourier mode (i,j,k):
//   g1 = (i + kappa1)/n1
//   g2 = ((n1 j - m1 i) mod n1n2)/(n1n2) + kh2/n2
//   g3 = ((n1n2 k - n1 m3 j + cb' i) mod n)/n + kh3/n3
//   lambda_l = (e^{2 pi i g_l} - 1)/delta_l
struct ModeP {
    int n1, n2, n3;
    long long n, n12;
    int m1, m3;
    long long cbp;    // c_b' = m1 m3 - n2 m2 - rho3 n2 m1, reduced into [0, n)
    long long n1m3;   // n1 m3 reduced into [0, n)
    double kap1, kh2, kh3;
    double idelta[3];
    long long gamma;  // flat index of the masked Gamma mode, or -1
    double taup;      // fallback threshold for Lambda_p^* Lambda_p (DESIGN R5)
};

// e^{2 pi i P / n} for integer P in [0, n): lo[P & mask] * hi[P >> shift]
struct TwP {
    const double2* lo;
    const double2* hi;
    int shift;
    unsigned long long mask;
};

struct OpArgs {
    ModeP mp;
    TwP tw;
    AxisPlan px, py, pz;
    const double* eps_inv;   // [3][n]  1/eps at the Yee points
    const unsigned char* eps_idx;  // [3][n] index into eps_lut (compressed B^{-1}), or null
    const double* eps_lut;   // <= 256 distinct values of 1/eps
    double inv_n;
    int W_z, W_y, R_x;       // tile widths (generic Stockham path)
    int fast;                // 1: register-FFT fast path where the axis length has a plan
    int comp0;               // first component slab (vector*3 + l) of a split y/x launch
    int nvec_all;            // vectors in the whole CG batch (split launches), 0 = grid
    const double2* hroot_z;  // e^{i pi k / n3}, k < n3 (half-angle table for lambda3 along k)
    unsigned long long* prof;   // optional per-phase cycle counters (plane pass), or null
    int plane_hint;             // L2 plane: evict-last / evict-first store hints (1)
    int plane_l2;               // plane pass: one CTA per plane, strips exchanged through L2 (1) or cluster/DSMEM (0)
    int plane_w;                // plane pass with warp-local FFT exchanges: 0 off, 1 shared memory, 2 shuffles
    // Slab decomposition: this launch works on slab `slab` of `nslab`.
    // Fourier-side arrays hold the j-slab [j0, j0 + n2loc) (all i, k): [vec][half][k][jl][i];
    // real-space arrays hold the z-slab of n3loc planes (all a, b): [vec][l][cl][b][a].
    // nloc = elements per component per vector on the slab (n / nslab).  nslab = 1: whole grid.
    int j0, n2loc, n3loc, slab, nslab;
    long long nloc;
    long long vsf;              // Fourier-side vector stride (elements): 2 nloc, or 2n for virtual slabs
    long long nblk;             // n1 n2loc n3loc: one (slab pair, vector, component) exchange block
    int zcfg;                   // z-pass variant: bit 0 = stage x / r tiles with the inputs (CG), bit 1 = half-width
                                // tiles, bit 2 = CG residual of zadj prefetched into registers before the mode loop
                                // (default on), bit 3 = CG x of zfwd prefetched into registers (measured slower);
                                // register budgets (128 plan): bit 9 = zadj2 CG for 4 CTAs/SM, bit 10 = zfwd2 CG
                                // (x staged) for 2 CTAs/SM, bit 11 = zadj2 CG for 2 CTAs/SM (no spills)
    int plane_t;                // plane pass staged by TMA (plane_tma.cu)
    int plane_split;            // L2 plane pass: 2 = a cluster of two CTAs per plane (every other strip each)
    int plane_rs;               // L2 plane pass: stage-root tables in shared memory (1)
    int plane_xeo;              // L2 plane pass (128 plan): phase X as even / odd halves with 256-bit accesses (1)
    int plane_ld;               // L2 plane pass (128 plan) load policy bits: 1 phase Y nc + L1::no_allocate, 2 phases X / Y* ld.cg, 4 phase X exchanges by CTA barriers instead of __syncwarp
};

struct Profiler;  // host-side, see solver.cu

// Fused-CG state (device pointers): the operator passes of one CG
// iteration also do p = r + beta p (zfwd), (p, M p) and alpha (x pass) and
// x += alpha p, r -= alpha M p, (r, r), beta (zadj).
struct CGFuse {
    double2* P;
    double2* R;
    double* part_x;           // [nvec][partials]
    double* part_z;
    double* rr;
    double* pmp;
    double* alpha;
    double* beta;
    double* thr;
    int* active;
    int* nb_x;                         // partial counts per vector written by the producing passes
    int* nb_z;                         //   (reduced by k_cg_finish after the pass)
    int* iter;                         // CG iterations done (device), or null
    int max_iter;
    int nslab;                         // partial blocks per vector: [slab][vec][nb] (slab decomposition), 1
    int use_cond;                      // 1: set the CG graph's while-condition
    int alpha_fold;                    // 1: k_zadj2 forms alpha itself from the (p, M p) partials (no cg_alpha kernel)
    cudaGraphConditionalHandle cond;
};

// launchers (kernels.cu); all enqueue on `st` and return cudaGetLastError()
cudaError_t launch_zfwd(const OpArgs& a, const double2* Y, double2* U, int nvec, int op, cudaStream_t st);
cudaError_t launch_ypass(const OpArgs& a, double2* U, int nvec, int adjoint, cudaStream_t st);
cudaError_t launch_xpass(const OpArgs& a, double2* U, int nvec, cudaStream_t st);
cudaError_t launch_zadj(const OpArgs& a, const double2* U, double2* OUT, int nvec, int op, cudaStream_t st);
cudaError_t launch_xfwd_recover(const OpArgs& a, double2* U, int nvec, const double* eps_inv, double scale0,
                                const double* scales, cudaStream_t st);
cudaError_t launch_bloch_phase(const OpArgs& a, double2* U, int nvec, double kap1, double kh2, double kh3,
                               cudaStream_t st);

bool fast_all(const OpArgs& a);
// N2 of the register-FFT plan N = N1 * N2 for axis length N, 0 if none
int fast_split_N2(int N);
cudaError_t launch_zfwd_cg(const OpArgs& a, const double2* R, double2* P, double2* U, int nvec, const CGFuse& cg,
                           cudaStream_t st);
cudaError_t launch_xpass_cg(const OpArgs& a, double2* U, int nvec, const CGFuse& cg, cudaStream_t st);
cudaError_t launch_zadj_cg(const OpArgs& a, const double2* U, double2* X, int nvec, const CGFuse& cg,
                           cudaStream_t st);
size_t cg_partials_per_vec(const OpArgs& a);

// Fused real-space plane pass (plane.cu): y-DFT, twiddle, x-DFT, B^{-1},
// x-DFT*, twiddle*, y-DFT* on every (component, z-plane) of nslab = 3*nvec
// component slabs, one HBM read + write.  Square xy planes with a fast plan.
bool plane_supported(const OpArgs& a);
// Raise kernel f's dynamic shared memory limit (cudaFuncAttributeMaxDynamicSharedMemorySize) to at
// least `bytes` on the current device.  The attribute is process-wide per function, so it only ever
// grows (under a lock): concurrent solvers (kpath per_gpu > 1) launching the same kernel with
// different sizes cannot lower it under one another's launch.
cudaError_t allow_smem(const void* f, size_t bytes);
bool plane_w_supported(const OpArgs& a);
// TMA-staged plane pass (plane_tma.cu): one slab, square 64/128/256 planes.  The
// tensor maps describe the plane buffer as [planes][N][2N doubles] (plane_t_encode).
bool plane_t_supported(const OpArgs& a);
// persistent TMA-pipelined adjoint z pass (zpipe.cu); the map views U as [comp slabs][n3][n2][2 n1 doubles]
bool zadj3_supported(const OpArgs& a);
int zadj3_tiles_x(const OpArgs& a);
int zadj3_encode(const OpArgs& a, void* base, long long comp_slabs, void* encode_fn, CUtensorMap* m);
cudaError_t launch_zadj3(const OpArgs& a, const CUtensorMap& tm, const double2* U, double2* OUT, int nvec, int op,
                         const CGFuse* cg, cudaStream_t st);
int plane_t_encode(const OpArgs& a, void* base, long long planes, void* encode_fn, CUtensorMap* my, CUtensorMap* mx);
cudaError_t launch_plane_tma(const OpArgs& a, int nslab, const CGFuse* cg, cudaStream_t st, const CUtensorMap& my,
                             const CUtensorMap& mx, int zbase);

// Persistent, cp.async-pipelined z passes (zpass.cu).  cg == nullptr: plain
// op (0 = A_r, 1 = M); otherwise the CG-fused variants (x update deferred:
// zfwd2 does x += alpha_prev p, p <- r + beta p; zadj2 does r -= alpha M p and
// the (r,r)/beta reduction; finish with launch_cg_xfinal).
bool zpass2_supported(const OpArgs& a);
int zpass2_tiles_x(const OpArgs& a);
cudaError_t launch_zfwd2(const OpArgs& a, const double2* Y, double2* U, int nvec, int op, double2* P, double2* X,
                         const CGFuse* cg, cudaStream_t st);
cudaError_t launch_zadj2(const OpArgs& a, const double2* U, double2* OUT, int nvec, int op, const CGFuse* cg,
                         cudaStream_t st);
// alpha (which = 0, after the (p, M p) pass) or beta + convergence flags +
// graph condition (which = 1, after zadj) from the per-CTA partials (one CTA)
cudaError_t launch_cg_finish(const CGFuse& cg, int which, int nvec, cudaStream_t st);
cudaError_t launch_cg_xfinal(double2* X, const double2* P, const double* alpha, long long N, int nvec, cudaStream_t st);
cudaError_t launch_plane(const OpArgs& a, double2* U, int nslab, const CGFuse* cg, cudaStream_t st);

cudaError_t launch_sigma_table(const ModeP& mp, double* sigma, cudaStream_t st, int j0 = 0, int n2loc = 0,
                               long long count = 0);

// vectors of length N (complex), nvec of them, stored back to back
cudaError_t launch_dot_partial(const double2* X, const double2* Y, long long N, int nvec, double2* partial,
                               int nblk, cudaStream_t st);
cudaError_t launch_dot_final(const double2* partial, int nblk, int nvec, double2* out, cudaStream_t st);
cudaError_t launch_gemm_tn_partial(const double2* X, int p, const double2* Y, int q, long long N,
                                   double2* partial, int nblk, cudaStream_t st);
cudaError_t launch_gemm_tn_final(const double2* partial, int nblk, int pq, double2* out, cudaStream_t st);
cudaError_t launch_gemm_nn(const double2* X, int p, const double2* H, int q, double2* Y, long long N,
                           double alpha, double beta, cudaStream_t st);
cudaError_t launch_scale_sigma(const double2* X, double2* Y, const double* sigma, long long n, int nvec,
                               int inverse, cudaStream_t st, long long nloc = 0);
cudaError_t launch_fill_random(double2* X, long long N, int nvec, unsigned long long seed, long long offset,
                               const double* sigma, long long n, cudaStream_t st, long long nloc = 0);
cudaError_t launch_copy(double2* dst, const double2* src, long long count, cudaStream_t st);

// CG (batched over nvec right-hand sides)
struct CGState {
    double* rr;       // [nvec] current (r,r)
    double* rrnew;    // [nvec]
    double2* pMp;     // [nvec]
    double* beta;     // [nvec]
    double* thr;      // [nvec] tol^2 (c,c)
    int* active;      // [nvec]
};
cudaError_t launch_cg_init(const CGState& s, const double2* cdot, int nvec, double tol, cudaStream_t st);
cudaError_t launch_cg_xr(double2* X, double2* R, const double2* P, const double2* MP, const CGState& s,
                         long long N, int nvec, double2* partial, int nblk, cudaStream_t st);
cudaError_t launch_cg_scalars(const CGState& s, const double2* rrnew_c, int nvec, cudaStream_t st);
cudaError_t launch_cg_p(double2* P, const double2* R, const CGState& s, long long N, int nvec, cudaStream_t st);

}  // namespace bnf
