// sm_100a kernels of the null-space-free matvec and
// the eigensolver's vector/tall-skinny operations (a6-a8).
//
// M y = Q_r^* B^{-1} Q_r y  with  Q_r = (I3 (x) T)[Pi1 Pi2]
// is applied in five passes over HBM, each a batched 1D DFT along one axis
// staged in shared memory (Stockham autosort, radix 2/3/4/8 + generic
// prime) fused with the diagonal factors that surround it:
//
//   zfwd : Sigma_r, Pi-combine (2 -> 3 components), DFT over k (+),
//          twiddle e^{+2 pi i c (cb' i - n1 m3 j)/n}                (Alg. 2 step 1)
//   yfwd : DFT over j (+), twiddle e^{-2 pi i b m1 i/(n1 n2)}       (Alg. 2 step 2)
//   x    : DFT over i (+), * 1/(n eps), DFT over a (-)           (Alg. 2 step 3,
//          B^{-1}, Alg. 1 step 1; the Bloch phase D_{a1}... of T and T^* cancels)
//   yadj : conj twiddle, DFT over b (-)                             (Alg. 1 step 2)
//   zadj : conj twiddle, DFT over c (-), Pi^*-combine (3 -> 2), Sigma_r
//                                                                   (Alg. 1 step 3)
// All inter-axis twiddles have integer phase numerators (SURVEY §8 notation)
// and are read from an exact two-level table of e^{2 pi i P/n}.
#include <cuda_runtime.h>
#include <cstdlib>

#include <algorithm>
#include <map>
#include <mutex>
#include <utility>

#include "cgfuse.cuh"
#include "fastfft.cuh"
#include "kernels.cuh"

namespace bnf {

namespace {

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// conj(a) * b
__device__ __forceinline__ double2 cjmul(double2 a, double2 b) {
    return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double cabs2(double2 a) { return a.x * a.x + a.y * a.y; }
// multiply by SIGN * i
template <int SIGN>
__device__ __forceinline__ double2 mul_i(double2 a) {
    return SIGN > 0 ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}

template <int SIGN>
__device__ __forceinline__ double2 root_tw(const double2* __restrict__ root, int t) {
    double2 w = __ldg(root + t);
    return SIGN > 0 ? w : cconj(w);
}

// ---------------------------------------------------------------- DFT kernels
template <int SIGN>
__device__ __forceinline__ void dft2(double2& a, double2& b) {
    double2 t = a;
    a = cadd(t, b);
    b = csub(t, b);
}

template <int SIGN>
__device__ __forceinline__ void dft4(double2& v0, double2& v1, double2& v2, double2& v3) {
    double2 a0 = cadd(v0, v2), a1 = csub(v0, v2);
    double2 b0 = cadd(v1, v3), b1 = mul_i<SIGN>(csub(v1, v3));
    v0 = cadd(a0, b0);
    v2 = csub(a0, b0);
    v1 = cadd(a1, b1);
    v3 = csub(a1, b1);
}

template <int SIGN>
__device__ __forceinline__ void dft8(double2* v) {
    // even/odd split: y_s = E_s + w^s O_s, y_{s+4} = E_s - w^s O_s, w = e^{SIGN 2 pi i/8}
    double2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
    double2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
    dft4<SIGN>(e0, e1, e2, e3);
    dft4<SIGN>(o0, o1, o2, o3);
    const double h = 0.70710678118654752440;
    // w^1 = (1 + SIGN i) h, w^2 = SIGN i, w^3 = (-1 + SIGN i) h
    double2 t1 = cscale(cadd(o1, mul_i<SIGN>(o1)), h);
    double2 t2 = mul_i<SIGN>(o2);
    double2 t3 = cscale(csub(mul_i<SIGN>(o3), o3), h);
    v[0] = cadd(e0, o0);
    v[4] = csub(e0, o0);
    v[1] = cadd(e1, t1);
    v[5] = csub(e1, t1);
    v[2] = cadd(e2, t2);
    v[6] = csub(e2, t2);
    v[3] = cadd(e3, t3);
    v[7] = csub(e3, t3);
}

template <int SIGN>
__device__ __forceinline__ void dft3(double2& v0, double2& v1, double2& v2) {
    const double s3 = 0.86602540378443864676;
    double2 t = cadd(v1, v2);
    double2 u = cscale(mul_i<SIGN>(csub(v1, v2)), s3);
    double2 m = csub(v0, cscale(t, 0.5));
    v0 = cadd(v0, t);
    v1 = cadd(m, u);
    v2 = csub(m, u);
}

template <int R, int SIGN>
__device__ __forceinline__ void stage_fixed(const double2* __restrict__ A, double2* __restrict__ B, int ld, int col,
                                            int j, int nb, int k, int tstride, int base, int Ns,
                                            const double2* __restrict__ root) {
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = A[(j + r * nb) * ld + col];
    if (Ns > 1) {
#pragma unroll
        for (int r = 1; r < R; ++r) v[r] = cmul(v[r], root_tw<SIGN>(root, k * r * tstride));
    }
    if (R == 2) dft2<SIGN>(v[0], v[1]);
    if (R == 3) dft3<SIGN>(v[0], v[1], v[2]);
    if (R == 4) dft4<SIGN>(v[0], v[1], v[2], v[3]);
    if (R == 8) dft8<SIGN>(v);
#pragma unroll
    for (int r = 0; r < R; ++r) B[(base + r * Ns) * ld + col] = v[r];
}

// Radix R > 32 (a large prime factor of an awkward axis length; NEXT-4): the
// R-point DFT of the stage evaluated directly from shared memory, O(R^2) per
// R outputs -- correct for any factor, meant for the occasional prime such
// as 37 or 41, not for speed.
template <int SIGN>
__device__ void stage_direct(int R, int N, const double2* __restrict__ A, double2* __restrict__ B, int ld, int col,
                             int j, int nb, int k, int tstride, int base, int Ns, const double2* __restrict__ root) {
    const int step = N / R;
    for (int s = 0; s < R; ++s) {
        double2 acc = make_double2(0.0, 0.0);
        for (int r = 0; r < R; ++r) {
            double2 x = A[(j + r * nb) * ld + col];
            if (Ns > 1 && r > 0) x = cmul(x, root_tw<SIGN>(root, k * r * tstride));
            acc = cadd(acc, cmul(x, root_tw<SIGN>(root, ((r * s) % R) * step)));
        }
        B[(base + s * Ns) * ld + col] = acc;
    }
}

template <int SIGN>
__device__ void stage_generic(int R, int N, const double2* __restrict__ A, double2* __restrict__ B, int ld, int col,
                              int j, int nb, int k, int tstride, int base, int Ns,
                              const double2* __restrict__ root) {
    if (R > 32) {
        stage_direct<SIGN>(R, N, A, B, ld, col, j, nb, k, tstride, base, Ns, root);
        return;
    }
    double2 v[32];
    for (int r = 0; r < R; ++r) {
        double2 x = A[(j + r * nb) * ld + col];
        if (Ns > 1 && r > 0) x = cmul(x, root_tw<SIGN>(root, k * r * tstride));
        v[r] = x;
    }
    const int step = N / R;
    for (int s = 0; s < R; ++s) {
        double2 acc = make_double2(0.0, 0.0);
        for (int r = 0; r < R; ++r) acc = cadd(acc, cmul(v[r], root_tw<SIGN>(root, ((r * s) % R) * step)));
        B[(base + s * Ns) * ld + col] = acc;
    }
}

// Batched Stockham FFT over `ncol` columns stored interleaved: element t of
// column col at A[t*ld + col].  y_s = sum_t x_t e^{SIGN 2 pi i s t / N}.
// Out-of-place ping-pong between A and B; returns the buffer holding the
// result.  Must be called by all threads of the block.
template <int SIGN>
__device__ double2* fft_cols(double2* A, double2* B, int ld, int ncol, const AxisPlan& pl) {
    const int N = pl.N;
    int Ns = 1;
    for (int s = 0; s < pl.nst; ++s) {
        const int R = pl.R[s];
        const int nb = N / R;
        const int tstride = N / (Ns * R);
        const int items = nb * ncol;
        for (int it = threadIdx.x; it < items; it += blockDim.x) {
            const int col = it % ncol;
            const int j = it / ncol;
            const int k = j % Ns;
            const int base = (j - k) * R + k;
            switch (R) {
                case 8: stage_fixed<8, SIGN>(A, B, ld, col, j, nb, k, tstride, base, Ns, pl.root); break;
                case 4: stage_fixed<4, SIGN>(A, B, ld, col, j, nb, k, tstride, base, Ns, pl.root); break;
                case 2: stage_fixed<2, SIGN>(A, B, ld, col, j, nb, k, tstride, base, Ns, pl.root); break;
                case 3: stage_fixed<3, SIGN>(A, B, ld, col, j, nb, k, tstride, base, Ns, pl.root); break;
                default: stage_generic<SIGN>(R, N, A, B, ld, col, j, nb, k, tstride, base, Ns, pl.root); break;
            }
        }
        __syncthreads();
        double2* t = A;
        A = B;
        B = t;
        Ns *= R;
    }
    return A;
}

// ------------------------------------------------------------- mode algebra
__device__ __forceinline__ double2 em1(double g) {
    // e^{2 pi i g} - 1 = -2 sin^2(pi g) + i 2 sin(pi g) cos(pi g)
    double s, c;
    sincospi(g, &s, &c);
    return make_double2(-2.0 * s * s, 2.0 * s * c);
}

__device__ __forceinline__ void mode_lambdas(const ModeP& p, int i, int j, int k, double2 lam[3]) {
    double g1 = (i + p.kap1) / p.n1;
    g1 -= rint(g1);
    long long num2 = ((long long)p.n1 * j - (long long)p.m1 * i) % p.n12;
    if (num2 < 0) num2 += p.n12;
    double g2 = (double)num2 / (double)p.n12 + p.kh2 / p.n2;
    g2 -= rint(g2);
    long long num3 = ((long long)p.n12 * k + p.cbp * (long long)i + (p.n - p.n1m3) * (long long)j) % p.n;
    double g3 = (double)num3 / (double)p.n + p.kh3 / p.n3;
    g3 -= rint(g3);
    lam[0] = cscale(em1(g1), p.idelta[0]);
    lam[1] = cscale(em1(g2), p.idelta[1]);
    lam[2] = cscale(em1(g3), p.idelta[2]);
}

// Pi1, Pi2 columns of mode (eq. range_basis1/2, readings R2, R3, R5, R6)
// and sigma = Lambda_q^{1/2}.
__device__ __forceinline__ void mode_pis(const ModeP& p, const double2 lam[3], bool masked, double2 pi1[3],
                                         double2 pi2[3], double& sig) {
    const double q = cabs2(lam[0]) + cabs2(lam[1]) + cabs2(lam[2]);
    if (masked || q == 0.0) {
        for (int l = 0; l < 3; ++l) pi1[l] = pi2[l] = make_double2(0.0, 0.0);
        sig = 0.0;
        return;
    }
    const double rq = rsqrt(q);
    sig = q * rq;
    const double2 d1 = csub(lam[2], lam[1]);
    const double2 d2 = csub(lam[0], lam[2]);
    const double2 d3 = csub(lam[1], lam[0]);
    const double p2 = cabs2(d1) + cabs2(d2) + cabs2(d3);
    if (p2 > p.taup * q) {
        const double r2 = rsqrt(p2);
        const double r1 = r2 * rq;
        pi1[0] = cscale(csub(cjmul(lam[1], d3), cjmul(lam[2], d2)), r1);
        pi1[1] = cscale(csub(cjmul(lam[2], d1), cjmul(lam[0], d3)), r1);
        pi1[2] = cscale(csub(cjmul(lam[0], d2), cjmul(lam[1], d1)), r1);
        pi2[0] = cscale(cconj(d1), r2);
        pi2[1] = cscale(cconj(d2), r2);
        pi2[2] = cscale(cconj(d3), r2);
        return;
    }
    // R5 fallback: e_m (smallest |lambda_m|, relative tie tolerance -> lowest m)
    // Gram-Schmidt'ed against Pi0, third vector conj(Pi0 x Pi1).
    double2 u[3];
    for (int l = 0; l < 3; ++l) u[l] = cscale(lam[l], rq);
    double a[3] = {cabs2(lam[0]), cabs2(lam[1]), cabs2(lam[2])};
    double amin = fmin(a[0], fmin(a[1], a[2]));
    int m = (a[0] <= amin * (1.0 + 1e-8)) ? 0 : ((a[1] <= amin * (1.0 + 1e-8)) ? 1 : 2);
    double2 v[3];
    for (int l = 0; l < 3; ++l) v[l] = cscale(cmul(u[l], cconj(u[m])), -1.0);
    v[m] = cadd(v[m], make_double2(1.0, 0.0));
    const double vn = rsqrt(cabs2(v[0]) + cabs2(v[1]) + cabs2(v[2]));
    for (int l = 0; l < 3; ++l) v[l] = cscale(v[l], vn);
    double2 w0 = csub(cmul(u[1], v[2]), cmul(u[2], v[1]));
    double2 w1 = csub(cmul(u[2], v[0]), cmul(u[0], v[2]));
    double2 w2 = csub(cmul(u[0], v[1]), cmul(u[1], v[0]));
    for (int l = 0; l < 3; ++l) pi1[l] = v[l];
    pi2[0] = cconj(w0);
    pi2[1] = cconj(w1);
    pi2[2] = cconj(w2);
}

__device__ __forceinline__ double2 tw_lookup(const TwP& t, unsigned long long P) {
    return cmul(__ldg(t.hi + (P >> t.shift)), __ldg(t.lo + (P & t.mask)));
}

// e^{+2 pi i c (cb' i - n1 m3 j) / n}
__device__ __forceinline__ double2 tw_yz(const ModeP& p, const TwP& t, int c, int i, int j) {
    unsigned long long N3 = (unsigned long long)((p.cbp * (long long)i + (p.n - p.n1m3) * (long long)j) % p.n);
    unsigned long long P = ((unsigned long long)c * N3) % (unsigned long long)p.n;
    return tw_lookup(t, P);
}

// e^{-2 pi i b m1 i / (n1 n2)}
__device__ __forceinline__ double2 tw_xy(const ModeP& p, const TwP& t, int b, int i) {
    long long r = ((long long)b * p.m1 * (long long)i) % p.n12;
    long long P = (r == 0) ? 0 : (p.n12 - r);
    return tw_lookup(t, (unsigned long long)P * (unsigned long long)p.n3);
}

// ------------------------------------------------------------------ kernels
__global__ void __launch_bounds__(256) k_zfwd(const double2* __restrict__ Y, double2* __restrict__ U, OpArgs a,
                                              int op) {
    extern __shared__ double2 sm[];
    const ModeP& p = a.mp;
    const int W = a.W_z;
    const int n1 = p.n1, n2 = p.n2, n3 = p.n3;
    const long long n = p.n;
    const int i0 = blockIdx.x * W, j = blockIdx.y, v = blockIdx.z;
    const int tile = n3 * W;
    double2* buf[3] = {sm, sm + tile, sm + 2 * tile};
    double2* scr = sm + 3 * tile;
    const double2* y1 = Y + (size_t)v * 2 * n;
    const double2* y2 = y1 + n;
    for (int e = threadIdx.x; e < tile; e += blockDim.x) {
        const int kk = e / W, ii = e - kk * W, i = i0 + ii;
        double2 o[3] = {make_double2(0, 0), make_double2(0, 0), make_double2(0, 0)};
        if (i < n1) {
            const size_t idx = (size_t)i + (size_t)n1 * ((size_t)j + (size_t)n2 * kk);
            const double2 u1 = y1[idx], u2 = y2[idx];
            double2 lam[3], pi1[3], pi2[3];
            double sig;
            mode_lambdas(p, i, j, kk, lam);
            mode_pis(p, lam, (long long)idx == p.gamma, pi1, pi2, sig);
            const double s = (op == 0) ? sig : (op == 2 ? (sig > 0.0 ? 1.0 / sig : 0.0) : 1.0);
            for (int l = 0; l < 3; ++l) o[l] = cscale(cadd(cmul(pi1[l], u1), cmul(pi2[l], u2)), s);
            if (op == 2) {
                // H side (NEXT-3): C (I x T) = (I x T) [lambda x], so
                // H = C e / (i omega) = -i P_r y = -i (I x T) lambda x (Q-side combine of y / sigma)
                const double2 h0 = csub(cmul(lam[1], o[2]), cmul(lam[2], o[1]));
                const double2 h1 = csub(cmul(lam[2], o[0]), cmul(lam[0], o[2]));
                const double2 h2 = csub(cmul(lam[0], o[1]), cmul(lam[1], o[0]));
                o[0] = make_double2(h0.y, -h0.x);   // -i h
                o[1] = make_double2(h1.y, -h1.x);
                o[2] = make_double2(h2.y, -h2.x);
            }
        }
        buf[0][e] = o[0];
        buf[1][e] = o[1];
        buf[2][e] = o[2];
    }
    __syncthreads();
    double2* Uv = U + (size_t)v * 3 * n;
    for (int l = 0; l < 3; ++l) {
        double2* res = fft_cols<+1>(buf[l], scr, W, W, a.pz);
        for (int e = threadIdx.x; e < tile; e += blockDim.x) {
            const int c = e / W, ii = e - c * W, i = i0 + ii;
            if (i < n1)
                Uv[(size_t)l * n + (size_t)i + (size_t)n1 * ((size_t)j + (size_t)n2 * c)] =
                    cmul(res[e], tw_yz(p, a.tw, c, i, j));
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(256) k_zadj(const double2* __restrict__ U, double2* __restrict__ OUT, OpArgs a,
                                              int op) {
    extern __shared__ double2 sm[];
    const ModeP& p = a.mp;
    const int W = a.W_z;
    const int n1 = p.n1, n2 = p.n2, n3 = p.n3;
    const long long n = p.n;
    const int i0 = blockIdx.x * W, j = blockIdx.y, v = blockIdx.z;
    const int tile = n3 * W;
    double2* buf[3] = {sm, sm + tile, sm + 2 * tile};
    double2* scr = sm + 3 * tile;
    const double2* Uv = U + (size_t)v * 3 * n;
    for (int e = threadIdx.x; e < tile; e += blockDim.x) {
        const int c = e / W, ii = e - c * W, i = i0 + ii;
        if (i < n1) {
            const size_t idx = (size_t)i + (size_t)n1 * ((size_t)j + (size_t)n2 * c);
            const double2 t = cconj(tw_yz(p, a.tw, c, i, j));
            for (int l = 0; l < 3; ++l) buf[l][e] = cmul(Uv[(size_t)l * n + idx], t);
        } else {
            for (int l = 0; l < 3; ++l) buf[l][e] = make_double2(0, 0);
        }
    }
    __syncthreads();
    for (int l = 0; l < 3; ++l) {
        double2* res = fft_cols<-1>(buf[l], scr, W, W, a.pz);
        if (res != buf[l]) {
            for (int e = threadIdx.x; e < tile; e += blockDim.x) buf[l][e] = res[e];
            __syncthreads();
        }
    }
    double2* o1 = OUT + (size_t)v * 2 * n;
    double2* o2 = o1 + n;
    for (int e = threadIdx.x; e < tile; e += blockDim.x) {
        const int kk = e / W, ii = e - kk * W, i = i0 + ii;
        if (i < n1) {
            const size_t idx = (size_t)i + (size_t)n1 * ((size_t)j + (size_t)n2 * kk);
            double2 lam[3], pi1[3], pi2[3];
            double sig;
            mode_lambdas(p, i, j, kk, lam);
            mode_pis(p, lam, (long long)idx == p.gamma, pi1, pi2, sig);
            double2 z1 = make_double2(0, 0), z2 = make_double2(0, 0);
            for (int l = 0; l < 3; ++l) {
                const double2 w = buf[l][e];
                z1 = cadd(z1, cjmul(pi1[l], w));
                z2 = cadd(z2, cjmul(pi2[l], w));
            }
            const double s = (op == 0) ? sig : 1.0;
            o1[idx] = cscale(z1, s);
            o2[idx] = cscale(z2, s);
        }
    }
}

template <int ADJ>
__global__ void __launch_bounds__(256) k_ypass(double2* __restrict__ U, OpArgs a) {
    extern __shared__ double2 sm[];
    const ModeP& p = a.mp;
    const int W = a.W_y;
    const int n1 = p.n1, n2 = p.n2;
    const long long n = p.n;
    const int i0 = blockIdx.x * W, c = blockIdx.y;
    double2* Uv = U + (size_t)blockIdx.z * n;
    const int tile = n2 * W;
    double2* buf = sm;
    double2* scr = sm + tile;
    for (int e = threadIdx.x; e < tile; e += blockDim.x) {
        const int jj = e / W, ii = e - jj * W, i = i0 + ii;
        double2 val = make_double2(0, 0);
        if (i < n1) {
            val = Uv[(size_t)i + (size_t)n1 * ((size_t)jj + (size_t)n2 * c)];
            if (ADJ) val = cmul(val, cconj(tw_xy(p, a.tw, jj, i)));
        }
        buf[e] = val;
    }
    __syncthreads();
    double2* res = ADJ ? fft_cols<-1>(buf, scr, W, W, a.py) : fft_cols<+1>(buf, scr, W, W, a.py);
    for (int e = threadIdx.x; e < tile; e += blockDim.x) {
        const int b = e / W, ii = e - b * W, i = i0 + ii;
        if (i < n1) {
            double2 val = res[e];
            if (!ADJ) val = cmul(val, tw_xy(p, a.tw, b, i));
            Uv[(size_t)i + (size_t)n1 * ((size_t)b + (size_t)n2 * c)] = val;
        }
    }
}

__global__ void __launch_bounds__(256) k_xpass(double2* __restrict__ U, OpArgs a) {
    extern __shared__ double2 sm[];
    const ModeP& p = a.mp;
    const int R = a.R_x, ld = R + 1;
    const int n1 = p.n1, n2 = p.n2;
    const long long n = p.n;
    const int b0 = blockIdx.x * R, c = blockIdx.y;
    const int vl = blockIdx.z, l = vl % 3;
    double2* Uv = U + (size_t)vl * n;
    const double* einv = a.eps_inv + (size_t)l * n;
    const size_t base = (size_t)n1 * ((size_t)b0 + (size_t)n2 * c);
    const int rows = min(R, n2 - b0);
    const int tile = n1 * ld;
    double2* buf = sm;
    double2* scr = sm + tile;
    for (int e = threadIdx.x; e < R * n1; e += blockDim.x) {
        const int row = e / n1, aa = e - row * n1;
        buf[aa * ld + row] = (row < rows) ? Uv[base + e] : make_double2(0, 0);
    }
    __syncthreads();
    double2* res = fft_cols<+1>(buf, scr, ld, R, a.px);
    for (int e = threadIdx.x; e < R * n1; e += blockDim.x) {
        const int row = e / n1, aa = e - row * n1;
        const double s = (row < rows) ? a.inv_n * __ldg(einv + base + e) : 0.0;
        res[aa * ld + row] = cscale(res[aa * ld + row], s);
    }
    __syncthreads();
    double2* other = (res == buf) ? scr : buf;
    double2* res2 = fft_cols<-1>(res, other, ld, R, a.px);
    for (int e = threadIdx.x; e < rows * n1; e += blockDim.x) {
        const int row = e / n1, aa = e - row * n1;
        Uv[base + e] = res2[aa * ld + row];
    }
}

// Recovery (a8): forward x-DFT only, then * scale / eps (the Bloch phase is a
// separate kernel).  scales[v] multiplies vector v (per-eigenvector 1/sqrt(lambda)).
__global__ void __launch_bounds__(256) k_xfwd_recover(double2* __restrict__ U, OpArgs a, const double* eps_inv,
                                                      double scale0, const double* scales) {
    extern __shared__ double2 sm[];
    const ModeP& p = a.mp;
    const int R = a.R_x, ld = R + 1;
    const int n1 = p.n1, n2 = p.n2;
    const long long n = p.n;
    const int b0 = blockIdx.x * R, c = blockIdx.y;
    const int vl = blockIdx.z, l = vl % 3, v = vl / 3;
    double2* Uv = U + (size_t)vl * n;
    const double* einv = eps_inv ? eps_inv + (size_t)l * n : nullptr;   // null: no B^{-1} (H field)
    const size_t base = (size_t)n1 * ((size_t)b0 + (size_t)n2 * c);
    const int rows = min(R, n2 - b0);
    const int tile = n1 * ld;
    double2* buf = sm;
    double2* scr = sm + tile;
    for (int e = threadIdx.x; e < R * n1; e += blockDim.x) {
        const int row = e / n1, aa = e - row * n1;
        buf[aa * ld + row] = (row < rows) ? Uv[base + e] : make_double2(0, 0);
    }
    __syncthreads();
    double2* res = fft_cols<+1>(buf, scr, ld, R, a.px);
    const double sv = scale0 * (scales ? scales[v] : 1.0);
    for (int e = threadIdx.x; e < rows * n1; e += blockDim.x) {
        const int row = e / n1, aa = e - row * n1;
        Uv[base + e] = cscale(res[aa * ld + row], sv * (einv ? __ldg(einv + base + e) : 1.0));
    }
}

// Bloch phase e^{2 pi i (a kappa1/n1 + b kh2/n2 + c kh3/n3)} of T (eq. T).
__global__ void k_bloch(double2* __restrict__ U, long long n, int n1, int n2, int n3, long long total,
                        double kap1, double kh2, double kh3) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const long long r = t % n;
        const int aa = (int)(r % n1);
        const int b = (int)((r / n1) % n2);
        const int c = (int)(r / ((long long)n1 * n2));
        double g = aa * kap1 / n1 + b * kh2 / n2 + c * kh3 / n3;
        g -= rint(g);
        double s, co;
        sincospi(2.0 * g, &s, &co);
        U[t] = cmul(U[t], make_double2(co, s));
    }
}

// sigma = Lambda_q^{1/2} over `count` Fourier entries laid out as consecutive
// j-slabs [slab][k][jl][i] of n2loc rows each, starting at row j0 (one slab
// covering all j: the plain [k][j][i] layout)
__global__ void k_sigma_table(ModeP p, double* __restrict__ sigma, int j0, int n2loc, long long count) {
    const long long nloc = (long long)p.n1 * n2loc * p.n3;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < count;
         t += (long long)gridDim.x * blockDim.x) {
        const long long r = t / nloc, loc = t - r * nloc;
        const int i = (int)(loc % p.n1);
        const int j = j0 + (int)(r * n2loc + (loc / p.n1) % n2loc);
        const int k = (int)(loc / ((long long)p.n1 * n2loc));
        double2 lam[3];
        mode_lambdas(p, i, j, k, lam);
        const double q = cabs2(lam[0]) + cabs2(lam[1]) + cabs2(lam[2]);
        const long long flat = (long long)i + (long long)p.n1 * (j + (long long)p.n2 * k);
        sigma[t] = (flat == p.gamma) ? 0.0 : sqrt(q);
    }
}

// index of the sigma entry of element t of a batch of vectors of 2 nh entries
// laid out [slab][half][local] (slabs of 2 nloc; one slab: [half][local])
__device__ __forceinline__ long long sig_index(long long t, long long nh, long long nloc) {
    const long long u = t % (2 * nh);
    return (u / (2 * nloc)) * nloc + u % nloc;
}

// ---------------------------------------------------------- BLAS-1 / tall-skinny
// partial[v*nblk + blk] = sum_{t in slice} conj(X_v[t]) Y_v[t]
__global__ void __launch_bounds__(256) k_dot_partial(const double2* __restrict__ X, const double2* __restrict__ Y,
                                                     long long N, double2* __restrict__ partial) {
    __shared__ double2 red[32];
    const int v = blockIdx.y;
    const double2* x = X + (size_t)v * N;
    const double2* y = Y + (size_t)v * N;
    double2 acc = make_double2(0, 0);
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < N; t += (long long)gridDim.x * blockDim.x)
        acc = cadd(acc, cjmul(x[t], y[t]));
    acc = block_sum(acc, red);
    if (threadIdx.x == 0) partial[(size_t)v * gridDim.x + blockIdx.x] = acc;
}

// out[g] = sum_b partial[g*nblk + b], fixed order (deterministic)
__global__ void __launch_bounds__(256) k_sum_final(const double2* __restrict__ partial, int nblk, double2* out) {
    __shared__ double2 red[32];
    const int g = blockIdx.x;
    double2 acc = make_double2(0, 0);
    for (int b = threadIdx.x; b < nblk; b += blockDim.x) acc = cadd(acc, partial[(size_t)g * nblk + b]);
    acc = block_sum(acc, red);
    if (threadIdx.x == 0) out[g] = acc;
}

// Tall-skinny X^* Y: X has p vectors, Y has q <= Q vectors, length N.
// Block = 8 warps over a slice of GT_SLICE = 512 rows (grid-stride over slices).
// The Y slice is staged in shared memory; warp w owns the columns a = w mod 8
// of X, streams X_a over the slice and accumulates into acc[a][c] (owned
// exclusively by that warp -> deterministic, no atomics).  partial[(a*q+c)*nblk + blk].
template <int Q>
__global__ void __launch_bounds__(256) k_gemm_tn_partial(const double2* __restrict__ X, int p,
                                                         const double2* __restrict__ Y, int q, long long N,
                                                         double2* __restrict__ partial) {
    constexpr int GT_SLICE = 512;   // rows per slice
    extern __shared__ double2 gsm[];
    double2* ys = gsm;                       // [Q][GT_SLICE]
    double2* acc = gsm + Q * GT_SLICE;       // [p][q]
    const int nblk = gridDim.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int t = threadIdx.x; t < p * q; t += blockDim.x) acc[t] = make_double2(0, 0);
    for (long long s0 = (long long)blockIdx.x * GT_SLICE; s0 < N; s0 += (long long)gridDim.x * GT_SLICE) {
        __syncthreads();
        for (int t = threadIdx.x; t < Q * GT_SLICE; t += blockDim.x) {
            const int c = t / GT_SLICE, r = t - c * GT_SLICE;
            ys[t] = (c < q && s0 + r < N) ? Y[(size_t)c * N + s0 + r] : make_double2(0, 0);
        }
        __syncthreads();
        for (int aidx = warp; aidx < p; aidx += 8) {
            const double2* xa = X + (size_t)aidx * N + s0;
            double2 sum[Q];
#pragma unroll
            for (int c = 0; c < Q; ++c) sum[c] = make_double2(0, 0);
#pragma unroll   // all 16 loads of the column slice in flight (memory-level parallelism)
            for (int r = lane; r < GT_SLICE; r += 32) {
                const double2 x = (s0 + r < N) ? xa[r] : make_double2(0, 0);
#pragma unroll
                for (int c = 0; c < Q; ++c) sum[c] = cadd(sum[c], cjmul(x, ys[c * GT_SLICE + r]));
            }
#pragma unroll
            for (int c = 0; c < Q; ++c) {
                if (c < q) {
                    const double2 v = warp_sum(sum[c]);
                    if (lane == 0) acc[aidx * q + c] = cadd(acc[aidx * q + c], v);
                }
            }
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < p * q; t += blockDim.x) partial[(size_t)t * nblk + blockIdx.x] = acc[t];
}

// Tall-skinny X^* Y, register-accumulating variant: each warp owns up to CPW
// columns of X (p >= 8: a = warp + 8 j) or, for p < 8, a column and a part of
// every slice's rows (so that all 8 warps stream X); the partial dot products
// stay in registers over the CTA's whole grid-stride range of 512-row slices
// and are reduced (warp shuffles, then the row parts in a fixed order) once
// at the end -- no per-slice reductions.  Y slices are staged in shared
// memory (512-row slices; 256 for q > 4).  partial[(a*q + c)*nblk + blk], deterministic.
template <int Q, int CPW>
__global__ void __launch_bounds__(256) k_gemm_tn2(const double2* __restrict__ X, int p, const double2* __restrict__ Y,
                                                  int q, long long N, double2* __restrict__ partial) {
    constexpr int SL = Q >= 8 ? 256 : 512;   // rows per slice (static shared memory <= 48 KB)
    __shared__ double2 ys[Q * SL];
    __shared__ double2 red[8][Q];
    const int nblk = gridDim.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int parts = p >= 8 ? 1 : 8 / p;            // row parts per column (p < 8)
    const int acol = p >= 8 ? warp : warp % p;        // first owned column
    const int part = p >= 8 ? 0 : warp / p;
    const bool active = part < parts;
    const int r0 = part * (SL / parts), r1 = (part + 1) * (SL / parts);
    double2 sum[CPW][Q];
#pragma unroll
    for (int j = 0; j < CPW; ++j)
#pragma unroll
        for (int c = 0; c < Q; ++c) sum[j][c] = make_double2(0, 0);
    for (long long s0 = (long long)blockIdx.x * SL; s0 < N; s0 += (long long)gridDim.x * SL) {
        __syncthreads();
        for (int t = threadIdx.x; t < Q * SL; t += blockDim.x) {
            const int c = t / SL, r = t - c * SL;
            ys[t] = (c < q && s0 + r < N) ? Y[(size_t)c * N + s0 + r] : make_double2(0, 0);
        }
        __syncthreads();
        if (!active) continue;
#pragma unroll
        for (int j = 0; j < CPW; ++j) {
            const int a = acol + 8 * j;
            if (a >= p || (p < 8 && j > 0)) break;
            const double2* xa = X + (size_t)a * N + s0;
            asm volatile("" ::: "memory");   // one column's loads at a time (register budget)
            if (parts == 1) {   // whole slice: all SL / 32 loads of the column in flight
                double2 x[SL / 32];
#pragma unroll
                for (int k = 0; k < SL / 32; ++k) {
                    const int r = lane + 32 * k;
                    x[k] = (s0 + r < N) ? xa[r] : make_double2(0, 0);
                }
#pragma unroll
                for (int k = 0; k < SL / 32; ++k)
#pragma unroll
                    for (int c = 0; c < Q; ++c) sum[j][c] = cadd(sum[j][c], cjmul(x[k], ys[c * SL + lane + 32 * k]));
            } else {
#pragma unroll 4
                for (int r = r0 + lane; r < r1; r += 32) {
                    const double2 x = (s0 + r < N) ? xa[r] : make_double2(0, 0);
#pragma unroll
                    for (int c = 0; c < Q; ++c) sum[j][c] = cadd(sum[j][c], cjmul(x, ys[c * SL + r]));
                }
            }
        }
    }
    // reduce: warp sums, then (p < 8) the row parts of a column in a fixed order
#pragma unroll
    for (int j = 0; j < CPW; ++j) {
        const int a = acol + 8 * j;
        const bool own = active && a < p && !(p < 8 && j > 0);
#pragma unroll
        for (int c = 0; c < Q; ++c) {
            const double2 v = warp_sum(sum[j][c]);
            if (p >= 8) {
                if (own && c < q && lane == 0) partial[(size_t)(a * q + c) * nblk + blockIdx.x] = v;
            } else if (j == 0) {
                if (lane == 0) red[warp][c] = v;
            }
        }
    }
    if (p < 8) {
        __syncthreads();
        if (threadIdx.x < p * q) {
            const int a = threadIdx.x / q, c = threadIdx.x % q;
            double2 acc = make_double2(0, 0);
            for (int pt = 0; pt < parts; ++pt) acc = cadd(acc, red[a + pt * p][c]);
            partial[(size_t)(a * q + c) * nblk + blockIdx.x] = acc;
        }
    }
}

// Y_c = beta Y_c + alpha sum_a X_a H[a*q + c]   (H on device, p*q <= 4096)
// Q >= q output columns held in registers; the loop over the p input columns
// is unrolled by 4 so that four independent 16-byte loads are in flight.
template <int Q>
__global__ void __launch_bounds__(256) k_gemm_nn(const double2* X, int p, const double2* __restrict__ H,
                                                 int q, double2* Y, long long N, double alpha,
                                                 double beta) {
    extern __shared__ double2 hs[];
    for (int t = threadIdx.x; t < p * q; t += blockDim.x) hs[t] = H[t];
    __syncthreads();
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < N; r += (long long)gridDim.x * blockDim.x) {
        double2 acc[Q];
#pragma unroll
        for (int c = 0; c < Q; ++c) acc[c] = make_double2(0, 0);
        int aidx = 0;
        for (; aidx + 4 <= p; aidx += 4) {
            double2 x[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) x[u] = X[(size_t)(aidx + u) * N + r];
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int c = 0; c < Q; ++c)
                    if (c < q) acc[c] = cadd(acc[c], cmul(x[u], hs[(aidx + u) * q + c]));
        }
        for (; aidx < p; ++aidx) {
            const double2 x = X[(size_t)aidx * N + r];
#pragma unroll
            for (int c = 0; c < Q; ++c)
                if (c < q) acc[c] = cadd(acc[c], cmul(x, hs[aidx * q + c]));
        }
#pragma unroll
        for (int c = 0; c < Q; ++c) {
            if (c < q) {
                const double2 y = (beta == 0.0) ? make_double2(0, 0) : cscale(Y[(size_t)c * N + r], beta);
                Y[(size_t)c * N + r] = cadd(y, cscale(acc[c], alpha));
            }
        }
    }
}

// Y = X * sigma^{+-1} on both halves of every 2n vector (masked: 0)
__global__ void k_scale_sigma(const double2* __restrict__ X, double2* __restrict__ Y, const double* __restrict__ sigma,
                              long long n, long long nloc, long long total, int inverse) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const double s = sigma[sig_index(t, n, nloc)];
        const double f = inverse ? (s > 0.0 ? 1.0 / s : 0.0) : s;
        Y[t] = cscale(X[t], f);
    }
}

__device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

// Counter-based normal deviates (Box-Muller on two hashed uniforms).
__global__ void k_fill_random(double2* __restrict__ X, long long total, unsigned long long seed, long long offset,
                              const double* __restrict__ sigma, long long n, long long nloc) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const unsigned long long h1 = splitmix64(seed ^ splitmix64((unsigned long long)(t + offset) * 2ull));
        const unsigned long long h2 = splitmix64(seed ^ splitmix64((unsigned long long)(t + offset) * 2ull + 1ull));
        const double u1 = ((h1 >> 11) + 1.0) * (1.0 / 9007199254740993.0);
        const double u2 = (h2 >> 11) * (1.0 / 9007199254740992.0);
        const double rad = sqrt(-2.0 * log(u1));
        double s, c;
        sincospi(2.0 * u2, &s, &c);
        const double m = (sigma != nullptr && sigma[sig_index(t, n, nloc)] == 0.0) ? 0.0 : 1.0;
        X[t] = make_double2(m * rad * c, m * rad * s);
    }
}

__global__ void k_copy(double2* __restrict__ d, const double2* __restrict__ s, long long count) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < count;
         t += (long long)gridDim.x * blockDim.x)
        d[t] = s[t];
}

// ------------------------------------------------------------------- CG
__global__ void k_cg_init(CGState s, const double2* __restrict__ cdot, int nvec, double tol) {
    const int v = threadIdx.x;
    if (v < nvec) {
        const double cc = cdot[v].x;
        s.rr[v] = cc;
        s.thr[v] = tol * tol * cc;
        s.active[v] = cc > 0.0 ? 1 : 0;
    }
}

// alpha = rr/(p,Mp);  x += alpha p;  r -= alpha Mp;  partial (r, r)
__global__ void __launch_bounds__(256) k_cg_xr(double2* __restrict__ X, double2* __restrict__ R,
                                               const double2* __restrict__ P, const double2* __restrict__ MP,
                                               CGState s, long long N, double2* __restrict__ partial) {
    __shared__ double2 red[32];
    const int v = blockIdx.y;
    const double pmp = s.pMp[v].x;
    const double alpha = (s.active[v] && pmp > 0.0) ? s.rr[v] / pmp : 0.0;
    double2* x = X + (size_t)v * N;
    double2* r = R + (size_t)v * N;
    const double2* pp = P + (size_t)v * N;
    const double2* mp = MP + (size_t)v * N;
    double acc = 0.0;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < N; t += (long long)gridDim.x * blockDim.x) {
        const double2 pt = pp[t];
        const double2 mt = mp[t];
        double2 xt = x[t], rt = r[t];
        xt.x += alpha * pt.x;
        xt.y += alpha * pt.y;
        rt.x -= alpha * mt.x;
        rt.y -= alpha * mt.y;
        x[t] = xt;
        r[t] = rt;
        acc += rt.x * rt.x + rt.y * rt.y;
    }
    double2 a2 = block_sum(make_double2(acc, 0.0), red);
    if (threadIdx.x == 0) partial[(size_t)v * gridDim.x + blockIdx.x] = a2;
}

__global__ void k_cg_scalars(CGState s, const double2* __restrict__ rrnew_c, int nvec) {
    const int v = threadIdx.x;
    if (v < nvec) {
        const double rn = rrnew_c[v].x;
        const int act = s.active[v];
        s.beta[v] = (act && s.rr[v] > 0.0) ? rn / s.rr[v] : 0.0;
        if (act) s.rr[v] = rn;
        s.rrnew[v] = rn;
        s.active[v] = (act && rn > s.thr[v]) ? 1 : 0;
    }
}

__global__ void k_cg_p(double2* __restrict__ P, const double2* __restrict__ R, CGState s, long long N) {
    const int v = blockIdx.y;
    const double beta = s.beta[v];
    double2* p = P + (size_t)v * N;
    const double2* r = R + (size_t)v * N;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < N; t += (long long)gridDim.x * blockDim.x) {
        const double2 pt = p[t], rt = r[t];
        p[t] = make_double2(rt.x + beta * pt.x, rt.y + beta * pt.y);
    }
}

// ================================================================
// Fast path: register-resident two-stage FFTs (fastfft.cuh).  Used when an
// axis length has a plan N = N1 * N2 with N1 % N2 == 0 (all BASELINE grids).
// ================================================================
__device__ __forceinline__ unsigned long long yz_base(const ModeP& p, int i, int j) {
    return (unsigned long long)((p.cbp * (long long)i + (p.n - p.n1m3) * (long long)j) % p.n);
}
// e^{+2 pi i c N3 / n}
__device__ __forceinline__ double2 tw_yz_fast(const ModeP& p, const TwP& t, int c, unsigned long long N3) {
    unsigned long long P;
    if (p.n <= 16777216LL) P = (unsigned long long)(((unsigned)c * (unsigned)N3) % (unsigned)p.n);
    else P = ((unsigned long long)c * N3) % (unsigned long long)p.n;
    return tw_lookup(t, P);
}
// e^{-2 pi i b M / n12} with M = m1 i mod n12
__device__ __forceinline__ double2 tw_xy_fast(const ModeP& p, const TwP& t, int b, unsigned M) {
    const unsigned r = ((unsigned)b * M) % (unsigned)p.n12;
    const unsigned P = r == 0 ? 0u : (unsigned)p.n12 - r;
    return tw_lookup(t, (unsigned long long)P * (unsigned long long)p.n3);
}

__device__ __forceinline__ unsigned long long mod_add(unsigned long long a, unsigned long long b,
                                                      unsigned long long n) {
    a += b;
    return a >= n ? a - n : a;
}
__device__ __forceinline__ unsigned long long mulmod(unsigned long long a, unsigned long long b,
                                                     unsigned long long n) {
    return (a * b) % n;   // a, b < n <= 2^30: product < 2^60
}

// Per-column (i, j) mode constants: lambda1, lambda2 and the integer base of
// the g3 numerator; lambda3 at row k then needs one sincospi and no division.
struct ColMode {
    double2 lam1, lam2;
    unsigned long long base3;
    double kh3n3, inv_n;
};
__device__ __forceinline__ ColMode col_mode(const ModeP& p, int i, int j) {
    ColMode cm;
    double g1 = (i + p.kap1) / p.n1;
    g1 -= rint(g1);
    long long num2 = ((long long)p.n1 * j - (long long)p.m1 * i) % p.n12;
    if (num2 < 0) num2 += p.n12;
    double g2 = (double)num2 / (double)p.n12 + p.kh2 / p.n2;
    g2 -= rint(g2);
    cm.lam1 = cscale(em1(g1), p.idelta[0]);
    cm.lam2 = cscale(em1(g2), p.idelta[1]);
    cm.base3 = (unsigned long long)((p.cbp * (long long)i + (p.n - p.n1m3) * (long long)j) % p.n);
    cm.kh3n3 = p.kh3 / p.n3;
    cm.inv_n = 1.0 / (double)p.n;
    return cm;
}
__device__ __forceinline__ double2 col_lam3(const ModeP& p, const ColMode& cm, int k) {
    unsigned long long num3 = cm.base3 + (unsigned long long)p.n12 * (unsigned long long)k;
    if (num3 >= (unsigned long long)p.n) num3 -= (unsigned long long)p.n;
    double g3 = (double)num3 * cm.inv_n + cm.kh3n3;
    g3 -= rint(g3);
    return cscale(em1(g3), p.idelta[2]);
}

// y pass: tile of W columns i, fixed c, FFT over j (length n2 = N1*N2).
template <int N1, int N2, int W, int ADJ>
__global__ void __launch_bounds__(W * N2) k_ypass_fast(double2* __restrict__ U, OpArgs a) {
    extern __shared__ double2 sm[];
    using X = fast::XchW<N1, N2, W>;
    const ModeP& p = a.mp;
    const int w = threadIdx.x % W, t = threadIdx.x / W;
    const int i = blockIdx.x * W + w, c = blockIdx.y;
    const bool ok = i < p.n1;
    double2* col = U + (size_t)(blockIdx.z + a.comp0) * p.n + (size_t)p.n1 * (size_t)p.n2 * c + (ok ? i : 0);
    // twiddle e^{-+2 pi i b M / n12}, M = m1 i: products of w^t, w^N2, w^N1 (fastfft twiddle_*)
    const unsigned n12 = (unsigned)p.n12;
    const unsigned M = ((unsigned)p.m1 * (unsigned)(ok ? i : 0)) % n12;
    const unsigned long long s3 = (unsigned long long)p.n3;
    const double2 wt = tw_lookup(a.tw, (unsigned long long)(((unsigned)t * M) % n12) * s3);
    const double2 wu = tw_lookup(a.tw, (unsigned long long)(((unsigned)N2 * M) % n12) * s3);
    double2 v[N1];
#pragma unroll
    for (int m = 0; m < N1; ++m) v[m] = ok ? col[(size_t)p.n1 * (N2 * m + t)] : make_double2(0, 0);
    if (ADJ) fast::twiddle_natural<N1, N2>(v, wt, wu);   // e^{+2 pi i b M / n12}, b = N2 m + t
    fast::fft_fwd<N1, N2, ADJ ? -1 : 1, X>(v, t, w, sm, a.py.root2);
    if (ok) {
        if (!ADJ) {
            const double2 wk = tw_lookup(a.tw, (unsigned long long)(((unsigned)N1 * M) % n12) * s3);
            fast::twiddle_stage2<N1, N2>(v, cconj(wt), cconj(wu), cconj(wk));   // e^{-2 pi i b M / n12}
        }
#pragma unroll
        for (int u = 0; u < N1 / N2; ++u)
#pragma unroll
            for (int k2 = 0; k2 < N2; ++k2) col[(size_t)p.n1 * (t + N2 * u + N1 * k2)] = v[u * N2 + k2];
    }
}

// x pass: R rows (b, c) per block, FFT over a (contiguous), * 1/(n eps), inverse FFT.
template <int N1, int N2, int R, int CG>
__global__ void __launch_bounds__(R * N2) k_xpass_fast(double2* __restrict__ U, OpArgs a, CGFuse cg) {
    extern __shared__ double2 sm[];
    using X = fast::XchT<N1, N2, R>;
    const ModeP& p = a.mp;
    const int t = threadIdx.x % N2, w = threadIdx.x / N2;
    const long long rows = (long long)p.n2 * p.n3;
    const long long r = (long long)blockIdx.x * R + w;
    const bool ok = r < rows;
    const int vl = blockIdx.y + a.comp0, l = vl % 3;
    double2* row = U + (size_t)vl * p.n + (size_t)(ok ? r : 0) * p.n1;
    const double* er = a.eps_inv + (size_t)l * p.n + (size_t)(ok ? r : 0) * p.n1;
    const unsigned char* ei = a.eps_idx ? a.eps_idx + (size_t)l * p.n + (size_t)(ok ? r : 0) * p.n1 : nullptr;
    double2 v[N1];
#pragma unroll
    for (int m = 0; m < N1; ++m) v[m] = ok ? row[N2 * m + t] : make_double2(0, 0);
    fast::fft_fwd<N1, N2, 1, X>(v, t, w, sm, a.px.root2);
    double pmp = 0.0;
#pragma unroll
    for (int u = 0; u < N1 / N2; ++u)
#pragma unroll
        for (int k2 = 0; k2 < N2; ++k2) {
            const int aa = t + N2 * u + N1 * k2;
            const double e_ = a.eps_idx ? __ldg(a.eps_lut + __ldg(ei + aa)) : __ldg(er + aa);
            const double s_ = ok ? a.inv_n * e_ : 0.0;
            const double2 x = v[u * N2 + k2];
            if (CG) pmp += s_ * (x.x * x.x + x.y * x.y);      // (p, M p) = sum |T v|^2 / eps
            v[u * N2 + k2] = cscale(x, s_);
        }
    if (CG) {
        // (p, M p) partial of this CTA; k_cg_finish forms alpha after the pass
        // (read by the next pass, zadj)
        const int vec = vl / 3;
        const int nb = gridDim.x * 3;
        cg_block_partial(pmp, cg.part_x + (size_t)vec * nb + (size_t)l * gridDim.x + blockIdx.x, sm);
        const long long lin = (long long)vl * gridDim.x + blockIdx.x;   // global over split (slab) launches
        if (lin == 0 && threadIdx.x == 0) *cg.nb_x = nb;   // alpha: k_cg_finish after this pass
    }
    fast::fft_mirror<N1, N2, -1, X>(v, t, w, sm, a.px.root2);
    if (ok) {
#pragma unroll
        for (int m = 0; m < N1; ++m) row[N2 * m + t] = v[m];
    }
}

// z forward: W columns i, fixed j; Sigma_r/Pi combine (2 -> 3), FFT over k,
// twiddle.  Threads (l, t, w); shared memory holds the 3 component tiles.
template <int N1, int N2, int W, int CG>
__global__ void __launch_bounds__(3 * W * N2) k_zfwd_fast(const double2* __restrict__ Y, double2* __restrict__ U,
                                                          OpArgs a, int op, double2* __restrict__ Pcg,
                                                          CGFuse cg) {
    extern __shared__ double2 sm[];
    constexpr int N = N1 * N2;
    constexpr int NT = 3 * W * N2;
    using X = fast::XchW<N1, N2, W>;
    const ModeP& p = a.mp;
    const int tid = threadIdx.x;
    const int w = tid % W, t = (tid / W) % N2, l = tid / (W * N2);
    const int i = blockIdx.x * W + w, j = blockIdx.y, vec = blockIdx.z;
    const bool ok = i < p.n1;
    const long long n = p.n;
    const size_t colofs = (size_t)(ok ? i : 0) + (size_t)p.n1 * j;
    const size_t kstride = (size_t)p.n1 * p.n2;
    // phase 1: every element once; thread keeps column w (NT is a multiple of W).
    // All loads are issued before the mode algebra (memory-level parallelism).
    {
        constexpr int S = (N * W + NT - 1) / NT;
        const double2* y1 = Y + (size_t)vec * 2 * n + colofs;
        const double2* y2 = y1 + n;
        double2 a1[S], a2[S];
#pragma unroll
        for (int s_ = 0; s_ < S; ++s_) {
            const int e = tid + s_ * NT;
            const bool in = ok && e < N * W;
            const int k = e / W;
            a1[s_] = in ? y1[kstride * k] : make_double2(0, 0);
            a2[s_] = in ? y2[kstride * k] : make_double2(0, 0);
        }
        if (CG) {   // p <- r + beta p  (CG direction update fused into the operator's first pass)
            const double beta = cg.beta[vec];
            double2* p1 = Pcg + (size_t)vec * 2 * n + colofs;
            double2* p2 = p1 + n;
#pragma unroll
            for (int s_ = 0; s_ < S; ++s_) {
                const int e = tid + s_ * NT;
                if (ok && e < N * W) {
                    const int k = e / W;
                    const double2 q1 = p1[kstride * k], q2 = p2[kstride * k];
                    a1[s_] = make_double2(a1[s_].x + beta * q1.x, a1[s_].y + beta * q1.y);
                    a2[s_] = make_double2(a2[s_].x + beta * q2.x, a2[s_].y + beta * q2.y);
                    p1[kstride * k] = a1[s_];
                    p2[kstride * k] = a2[s_];
                }
            }
        }
        const ColMode cm = col_mode(p, i, j);
#pragma unroll
        for (int s_ = 0; s_ < S; ++s_) {
            const int e = tid + s_ * NT;
            if (e < N * W) {
                const int k = e / W;
                double2 lam[3], pi1[3], pi2[3];
                double sig;
                lam[0] = cm.lam1;
                lam[1] = cm.lam2;
                lam[2] = col_lam3(p, cm, k);
                mode_pis(p, lam, (long long)(colofs + kstride * k) == p.gamma, pi1, pi2, sig);
                const double sc = (op == 0) ? sig : 1.0;
#pragma unroll
                for (int ll = 0; ll < 3; ++ll)
                    sm[ll * N * W + e] = cscale(cadd(cmul(pi1[ll], a1[s_]), cmul(pi2[ll], a2[s_])), sc);
            }
        }
    }
    __syncthreads();
    double2* tile = sm + (size_t)l * N * W;
    double2 v[N1];
#pragma unroll
    for (int m = 0; m < N1; ++m) v[m] = tile[(N2 * m + t) * W + w];
    __syncthreads();
    fast::fft_fwd<N1, N2, 1, X>(v, t, w, tile, a.pz.root2);
    if (ok) {
        const unsigned long long nn = (unsigned long long)n;
        const unsigned long long N3 = yz_base(p, i, j);
        const unsigned long long Du = mulmod((unsigned long long)N2, N3, nn);
        const unsigned long long Dk = mulmod((unsigned long long)N1, N3, nn);
        unsigned long long Pu = mulmod((unsigned long long)t, N3, nn);
        double2* out = U + (size_t)vec * 3 * n + (size_t)l * n + colofs;
#pragma unroll
        for (int u = 0; u < N1 / N2; ++u) {
            unsigned long long P = Pu;
#pragma unroll
            for (int k2 = 0; k2 < N2; ++k2) {
                const int c = t + N2 * u + N1 * k2;
                out[kstride * c] = cmul(v[u * N2 + k2], tw_lookup(a.tw, P));
                P = mod_add(P, Dk, nn);
            }
            Pu = mod_add(Pu, Du, nn);
        }
    }
}

// z adjoint: conj twiddle, FFT (-) over c, then Pi^* combine (3 -> 2), Sigma_r.
template <int N1, int N2, int W, int CG>
__global__ void __launch_bounds__(3 * W * N2) k_zadj_fast(const double2* __restrict__ U, double2* __restrict__ OUT,
                                                          OpArgs a, int op, CGFuse cg) {
    extern __shared__ double2 sm[];
    constexpr int N = N1 * N2;
    constexpr int NT = 3 * W * N2;
    using X = fast::XchW<N1, N2, W>;
    const ModeP& p = a.mp;
    const int tid = threadIdx.x;
    const int w = tid % W, t = (tid / W) % N2, l = tid / (W * N2);
    const int i = blockIdx.x * W + w, j = blockIdx.y, vec = blockIdx.z;
    const bool ok = i < p.n1;
    const long long n = p.n;
    const size_t colofs = (size_t)(ok ? i : 0) + (size_t)p.n1 * j;
    const size_t kstride = (size_t)p.n1 * p.n2;
    double2* tile = sm + (size_t)l * N * W;
    double2 v[N1];
    {
        const unsigned long long nn = (unsigned long long)n;
        const unsigned long long N3 = yz_base(p, i, j);
        const unsigned long long D = mulmod((unsigned long long)N2, N3, nn);
        unsigned long long P = mulmod((unsigned long long)t, N3, nn);
        const double2* in = U + (size_t)vec * 3 * n + (size_t)l * n + colofs;
#pragma unroll
        for (int m = 0; m < N1; ++m) {
            const int c = N2 * m + t;
            v[m] = ok ? cmul(in[kstride * c], tw_lookup(a.tw, P == 0 ? 0ull : nn - P)) : make_double2(0, 0);
            P = mod_add(P, D, nn);
        }
    }
    fast::fft_fwd<N1, N2, -1, X>(v, t, w, tile, a.pz.root2);
#pragma unroll
    for (int u = 0; u < N1 / N2; ++u)
#pragma unroll
        for (int k2 = 0; k2 < N2; ++k2) tile[(t + N2 * u + N1 * k2) * W + w] = v[u * N2 + k2];
    __syncthreads();
    double rr = 0.0;
    if (ok) {
        double2* o1 = OUT + (size_t)vec * 2 * n + colofs;
        double2* o2 = o1 + n;
        const ColMode cm = col_mode(p, i, j);
        const double alpha = CG ? cg.alpha[vec] : 0.0;
        for (int e = tid; e < N * W; e += NT) {
            const int k = e / W;
            double2 lam[3], pi1[3], pi2[3];
            double sig;
            lam[0] = cm.lam1;
            lam[1] = cm.lam2;
            lam[2] = col_lam3(p, cm, k);
            mode_pis(p, lam, (long long)(colofs + kstride * k) == p.gamma, pi1, pi2, sig);
            const double2 w0 = sm[e], w1 = sm[N * W + e], w2 = sm[2 * N * W + e];
            double2 z1 = cadd(cadd(cjmul(pi1[0], w0), cjmul(pi1[1], w1)), cjmul(pi1[2], w2));
            double2 z2 = cadd(cadd(cjmul(pi2[0], w0), cjmul(pi2[1], w1)), cjmul(pi2[2], w2));
            const double sc = (op == 0) ? sig : 1.0;
            z1 = cscale(z1, sc);
            z2 = cscale(z2, sc);
            if (CG) {   // OUT = x (solution), cg.X2 = r (residual), cg.P = p
                const size_t o = kstride * k;
                const size_t base = (size_t)vec * 2 * n + colofs;
                const double2 pp1 = cg.P[base + o], pp2 = cg.P[base + n + o];
                double2 r1 = cg.R[base + o], r2 = cg.R[base + n + o];
                double2 x1 = o1[o], x2 = o2[o];
                x1 = make_double2(x1.x + alpha * pp1.x, x1.y + alpha * pp1.y);
                x2 = make_double2(x2.x + alpha * pp2.x, x2.y + alpha * pp2.y);
                r1 = make_double2(r1.x - alpha * z1.x, r1.y - alpha * z1.y);
                r2 = make_double2(r2.x - alpha * z2.x, r2.y - alpha * z2.y);
                o1[o] = x1;
                o2[o] = x2;
                cg.R[base + o] = r1;
                cg.R[base + n + o] = r2;
                rr += r1.x * r1.x + r1.y * r1.y + r2.x * r2.x + r2.y * r2.y;
            } else {
                o1[kstride * k] = z1;
                o2[kstride * k] = z2;
            }
        }
    }
    if (CG) {
        const int nb = gridDim.x * gridDim.y;
        cg_block_partial(rr, cg.part_z + (size_t)vec * nb + (size_t)blockIdx.y * gridDim.x + blockIdx.x, sm);
        if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0) *cg.nb_z = nb;   // beta: k_cg_finish
    }
}

// CG scalars from the per-CTA partials of the preceding pass (one CTA, fixed
// summation order): the kernel boundary orders the partials, so the passes
// need no fences or atomics.
// CG scalars after a pass (which = 0: alpha from the (p, M p) partials, 1: beta
// from the (r, r) partials + loop control).  The 32 warps are split evenly over
// the vectors (up to 32 per round), so all vectors' partials are in flight at
// once; every sum is taken in a fixed order (deterministic).
__global__ void __launch_bounds__(1024) k_cg_finish(CGFuse cg, int which, int nvec) {
    __shared__ double wsum[32];
    const int nb = which == 0 ? *cg.nb_x : *cg.nb_z;
    const double* part = which == 0 ? cg.part_x : cg.part_z;
    const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int v0 = 0; v0 < nvec; v0 += nw) {
        const int nv = min(nvec - v0, nw), wpv = nw / nv;
        const int vl = warp / wpv, wi = warp % wpv;
        double acc = 0.0;
        if (vl < nv) {
            const int st = wpv * 32;
            for (int sl = 0; sl < max(1, cg.nslab); ++sl) {   // slab-major partials [slab][vec][nb]
                const double* pp = part + ((size_t)sl * nvec + v0 + vl) * nb;
                int t = wi * 32 + lane;
                for (; t + 3 * st < nb; t += 4 * st) {
                    const double a0 = __ldcg(pp + t), a1 = __ldcg(pp + t + st);
                    const double a2 = __ldcg(pp + t + 2 * st), a3 = __ldcg(pp + t + 3 * st);
                    acc += a0;
                    acc += a1;
                    acc += a2;
                    acc += a3;
                }
                for (; t < nb; t += st) acc += __ldcg(pp + t);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) wsum[warp] = acc;
        __syncthreads();
        if ((int)threadIdx.x < nv) {
            double sv = 0.0;
            for (int q = 0; q < wpv; ++q) sv += wsum[threadIdx.x * wpv + q];
            if (which == 0) cg_alpha_update(cg, v0 + threadIdx.x, sv);
            else cg_beta_update(cg, v0 + threadIdx.x, sv);
        }
        __syncthreads();
    }
    if (which == 1 && threadIdx.x == 0) cg_loop_control(cg, nvec);
}

inline int grid_for(long long total, int threads, int cap = 148 * 16) {
    long long g = (total + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (int)g;
}


// Fast plans: N -> (N1, N2) with N1 % N2 == 0.
#define BNF_FAST_PLANS(X) \
    X(8, 4, 2) X(12, 6, 2) X(16, 4, 4) X(24, 12, 2) X(32, 8, 4) X(48, 12, 4) X(64, 8, 8) X(96, 24, 4) \
    X(128, 16, 8) X(192, 24, 8) X(256, 16, 16)

constexpr int zW(int N, int N2) { return N2 == 2 ? 16 : (N <= 128 ? 8 : 4); }
constexpr int xR(int N2) { return N2 <= 8 ? 16 : 8; }
constexpr int yW() { return 16; }

bool has_fast(int N) {
    switch (N) {
#define BNF_CASE(NN, A, B) case NN: return true;
        BNF_FAST_PLANS(BNF_CASE)
#undef BNF_CASE
        default: return false;
    }
}

}  // namespace

cudaError_t allow_smem(const void* f, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> granted;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    size_t& g = granted[{f, dev}];
    if (bytes <= g) return cudaSuccess;
    e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) g = bytes;
    return e;
}

namespace {

template <class F, class... Args>
cudaError_t launch_k(F f, dim3 g, int threads, size_t sm, cudaStream_t st, Args... args) {
    if (sm > 32 * 1024) {   // leave room for the kernels' static shared memory
        cudaError_t e = allow_smem((const void*)f, sm);
        if (e != cudaSuccess) return e;
    }
    f<<<g, threads, sm, st>>>(args...);
    return cudaGetLastError();
}

cudaError_t fast_zfwd(const OpArgs& a, const double2* Y, double2* U, int nvec, int op, cudaStream_t st,
                      double2* Pcg = nullptr, const CGFuse* cg = nullptr) {
    switch (a.mp.n3) {
#define BNF_CASE(NN, A, B)                                                                              \
    case NN: {                                                                                          \
        constexpr int W = zW(NN, B);                                                                       \
        return cg ? launch_k(k_zfwd_fast<A, B, W, 1>, dim3((a.mp.n1 + W - 1) / W, a.mp.n2, nvec), 3 * W * B, \
                             (size_t)3 * NN * W * sizeof(double2), st, Y, U, a, op, Pcg, *cg)             \
                  : launch_k(k_zfwd_fast<A, B, W, 0>, dim3((a.mp.n1 + W - 1) / W, a.mp.n2, nvec), 3 * W * B, \
                             (size_t)3 * NN * W * sizeof(double2), st, Y, U, a, op, Pcg, CGFuse{});       \
    }
        BNF_FAST_PLANS(BNF_CASE)
#undef BNF_CASE
        default: return cudaErrorNotSupported;
    }
}

cudaError_t fast_zadj(const OpArgs& a, const double2* U, double2* OUT, int nvec, int op, cudaStream_t st,
                      const CGFuse* cg = nullptr) {
    switch (a.mp.n3) {
#define BNF_CASE(NN, A, B)                                                                              \
    case NN: {                                                                                          \
        constexpr int W = zW(NN, B);                                                                       \
        return cg ? launch_k(k_zadj_fast<A, B, W, 1>, dim3((a.mp.n1 + W - 1) / W, a.mp.n2, nvec), 3 * W * B, \
                             (size_t)3 * NN * W * sizeof(double2), st, U, OUT, a, op, *cg)                \
                  : launch_k(k_zadj_fast<A, B, W, 0>, dim3((a.mp.n1 + W - 1) / W, a.mp.n2, nvec), 3 * W * B, \
                             (size_t)3 * NN * W * sizeof(double2), st, U, OUT, a, op, CGFuse{});          \
    }
        BNF_FAST_PLANS(BNF_CASE)
#undef BNF_CASE
        default: return cudaErrorNotSupported;
    }
}

cudaError_t fast_ypass(const OpArgs& a, double2* U, int nvec, int adjoint, cudaStream_t st) {
    switch (a.mp.n2) {
#define BNF_CASE(NN, A, B)                                                                                    \
    case NN: {                                                                                                \
        constexpr int W = yW();                                                                               \
        dim3 g((a.mp.n1 + W - 1) / W, a.mp.n3, nvec > 0 ? 3 * nvec : 1);                                      \
        const size_t sm = (size_t)fast::XchW<A, B, W>::size * sizeof(double2);                               \
        return adjoint ? launch_k(k_ypass_fast<A, B, W, 1>, g, W * B, sm, st, U, a)                           \
                       : launch_k(k_ypass_fast<A, B, W, 0>, g, W * B, sm, st, U, a);                          \
    }
        BNF_FAST_PLANS(BNF_CASE)
#undef BNF_CASE
        default: return cudaErrorNotSupported;
    }
}

cudaError_t fast_xpass(const OpArgs& a, double2* U, int nvec, cudaStream_t st, const CGFuse* cg = nullptr) {
    switch (a.mp.n1) {
#define BNF_CASE(NN, A, B)                                                                                    \
    case NN: {                                                                                                \
        constexpr int R = xR(B);                                                                              \
        const long long rows = (long long)a.mp.n2 * a.mp.n3;                                                  \
        dim3 g((unsigned)((rows + R - 1) / R), nvec > 0 ? 3 * nvec : 1);                                      \
        const size_t sm = (size_t)fast::XchT<A, B, R>::size * sizeof(double2);                               \
        return cg ? launch_k(k_xpass_fast<A, B, R, 1>, g, R * B, sm, st, U, a, *cg)                           \
                  : launch_k(k_xpass_fast<A, B, R, 0>, g, R * B, sm, st, U, a, CGFuse{});                     \
    }
        BNF_FAST_PLANS(BNF_CASE)
#undef BNF_CASE
        default: return cudaErrorNotSupported;
    }
}
}  // namespace

// ---------------------------------------------------------------- launchers
static size_t smem_z(const OpArgs& a) { return (size_t)4 * a.mp.n3 * a.W_z * sizeof(double2); }
static size_t smem_y(const OpArgs& a) { return (size_t)2 * a.mp.n2 * a.W_y * sizeof(double2); }
static size_t smem_x(const OpArgs& a) { return (size_t)2 * a.mp.n1 * (a.R_x + 1) * sizeof(double2); }

static cudaError_t set_smem(const void* f, size_t bytes) {
    return bytes > 32 * 1024 ? allow_smem(f, bytes) : cudaSuccess;
}

cudaError_t launch_zfwd(const OpArgs& a, const double2* Y, double2* U, int nvec, int op, cudaStream_t st) {
    // op 2 (H field, bnf_eigvecs BNF_VEC_H) exists only in the generic pass
    if (op != 2 && a.fast && has_fast(a.mp.n3)) return fast_zfwd(a, Y, U, nvec, op, st);
    const size_t sm = smem_z(a);
    cudaError_t e = set_smem((const void*)k_zfwd, sm);
    if (e != cudaSuccess) return e;
    dim3 g((a.mp.n1 + a.W_z - 1) / a.W_z, a.mp.n2, nvec);
    k_zfwd<<<g, 256, sm, st>>>(Y, U, a, op);
    return cudaGetLastError();
}

cudaError_t launch_zadj(const OpArgs& a, const double2* U, double2* OUT, int nvec, int op, cudaStream_t st) {
    if (a.fast && has_fast(a.mp.n3)) return fast_zadj(a, U, OUT, nvec, op, st);
    const size_t sm = smem_z(a);
    cudaError_t e = set_smem((const void*)k_zadj, sm);
    if (e != cudaSuccess) return e;
    dim3 g((a.mp.n1 + a.W_z - 1) / a.W_z, a.mp.n2, nvec);
    k_zadj<<<g, 256, sm, st>>>(U, OUT, a, op);
    return cudaGetLastError();
}

cudaError_t launch_ypass(const OpArgs& a, double2* U, int nvec, int adjoint, cudaStream_t st) {
    if (a.fast && has_fast(a.mp.n2)) return fast_ypass(a, U, nvec, adjoint, st);
    const size_t sm = smem_y(a);
    dim3 g((a.mp.n1 + a.W_y - 1) / a.W_y, a.mp.n3, 3 * nvec);
    if (adjoint) {
        cudaError_t e = set_smem((const void*)k_ypass<1>, sm);
        if (e != cudaSuccess) return e;
        k_ypass<1><<<g, 256, sm, st>>>(U, a);
    } else {
        cudaError_t e = set_smem((const void*)k_ypass<0>, sm);
        if (e != cudaSuccess) return e;
        k_ypass<0><<<g, 256, sm, st>>>(U, a);
    }
    return cudaGetLastError();
}

cudaError_t launch_xpass(const OpArgs& a, double2* U, int nvec, cudaStream_t st) {
    if (a.fast && has_fast(a.mp.n1)) return fast_xpass(a, U, nvec, st);
    const size_t sm = smem_x(a);
    cudaError_t e = set_smem((const void*)k_xpass, sm);
    if (e != cudaSuccess) return e;
    dim3 g((a.mp.n2 + a.R_x - 1) / a.R_x, a.mp.n3, 3 * nvec);
    k_xpass<<<g, 256, sm, st>>>(U, a);
    return cudaGetLastError();
}

cudaError_t launch_xfwd_recover(const OpArgs& a, double2* U, int nvec, const double* eps_inv, double scale0,
                                const double* scales, cudaStream_t st) {
    const size_t sm = smem_x(a);
    cudaError_t e = set_smem((const void*)k_xfwd_recover, sm);
    if (e != cudaSuccess) return e;
    dim3 g((a.mp.n2 + a.R_x - 1) / a.R_x, a.mp.n3, 3 * nvec);
    k_xfwd_recover<<<g, 256, sm, st>>>(U, a, eps_inv, scale0, scales);
    return cudaGetLastError();
}

cudaError_t launch_bloch_phase(const OpArgs& a, double2* U, int nvec, double kap1, double kh2, double kh3,
                               cudaStream_t st) {
    const long long total = (long long)3 * nvec * a.mp.n;
    k_bloch<<<grid_for(total, 256), 256, 0, st>>>(U, a.mp.n, a.mp.n1, a.mp.n2, a.mp.n3, total, kap1, kh2, kh3);
    return cudaGetLastError();
}

cudaError_t launch_sigma_table(const ModeP& mp, double* sigma, cudaStream_t st, int j0, int n2loc, long long count) {
    if (n2loc <= 0) n2loc = mp.n2;
    if (count <= 0) count = mp.n;
    k_sigma_table<<<grid_for(count, 256), 256, 0, st>>>(mp, sigma, j0, n2loc, count);
    return cudaGetLastError();
}

cudaError_t launch_dot_partial(const double2* X, const double2* Y, long long N, int nvec, double2* partial, int nblk,
                               cudaStream_t st) {
    k_dot_partial<<<dim3(nblk, nvec), 256, 0, st>>>(X, Y, N, partial);
    return cudaGetLastError();
}

cudaError_t launch_dot_final(const double2* partial, int nblk, int nvec, double2* out, cudaStream_t st) {
    k_sum_final<<<nvec, 256, 0, st>>>(partial, nblk, out);
    return cudaGetLastError();
}

cudaError_t launch_gemm_tn_partial(const double2* X, int p, const double2* Y, int q, long long N, double2* partial,
                                   int nblk, cudaStream_t st) {
    // register-accumulating kernel: opt-in (BNF_GEMM_V2) -- measured 1.8x slower than the per-slice
    // kernel below at the bench workload (fewer loads in flight per warp), kept for the record
    static const bool v2 = std::getenv("BNF_GEMM_V2") != nullptr;
    if (v2 && q <= 8) {   // columns in chunks of 8 CPW
        const int Q = q <= 1 ? 1 : (q <= 2 ? 2 : (q <= 4 ? 4 : 8));
        constexpr int CPW = 4;
        for (int a0 = 0; a0 < p; a0 += 8 * CPW) {
            const int pc = std::min(p - a0, 8 * CPW);
            const double2* Xc = X + (size_t)a0 * N;
            double2* pp = partial + (size_t)a0 * q * nblk;
            if (Q == 1) k_gemm_tn2<1, CPW><<<nblk, 256, 0, st>>>(Xc, pc, Y, q, N, pp);
            else if (Q == 2) k_gemm_tn2<2, CPW><<<nblk, 256, 0, st>>>(Xc, pc, Y, q, N, pp);
            else if (Q == 4) k_gemm_tn2<4, CPW><<<nblk, 256, 0, st>>>(Xc, pc, Y, q, N, pp);
            else k_gemm_tn2<8, 2><<<nblk, 256, 0, st>>>(Xc, pc, Y, q, N, pp);
            if (Q == 8 && pc > 16) {   // CPW = 2 covers 16 columns: second half of the chunk
                k_gemm_tn2<8, 2><<<nblk, 256, 0, st>>>(Xc + (size_t)16 * N, pc - 16, Y, q, N, pp + (size_t)16 * q * nblk);
            }
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
    }
    const int Q = q <= 1 ? 1 : (q <= 2 ? 2 : (q <= 4 ? 4 : 8));
    if (q > 8) return cudaErrorInvalidValue;
    const int slice = 512;
    const size_t sm = ((size_t)Q * slice + (size_t)p * q) * sizeof(double2);
    const void* f = Q == 1 ? (const void*)k_gemm_tn_partial<1> : Q == 2 ? (const void*)k_gemm_tn_partial<2>
                  : Q == 4 ? (const void*)k_gemm_tn_partial<4> : (const void*)k_gemm_tn_partial<8>;
    cudaError_t e = set_smem(f, sm);
    if (e != cudaSuccess) return e;
    if (Q == 1) k_gemm_tn_partial<1><<<nblk, 256, sm, st>>>(X, p, Y, q, N, partial);
    else if (Q == 2) k_gemm_tn_partial<2><<<nblk, 256, sm, st>>>(X, p, Y, q, N, partial);
    else if (Q == 4) k_gemm_tn_partial<4><<<nblk, 256, sm, st>>>(X, p, Y, q, N, partial);
    else k_gemm_tn_partial<8><<<nblk, 256, sm, st>>>(X, p, Y, q, N, partial);
    return cudaGetLastError();
}

cudaError_t launch_gemm_tn_final(const double2* partial, int nblk, int pq, double2* out, cudaStream_t st) {
    k_sum_final<<<pq, 256, 0, st>>>(partial, nblk, out);
    return cudaGetLastError();
}

cudaError_t launch_gemm_nn(const double2* X, int p, const double2* H, int q, double2* Y, long long N, double alpha,
                           double beta, cudaStream_t st) {
    const size_t sm = (size_t)p * q * sizeof(double2);
    if (q > 8) return cudaErrorInvalidValue;
    const int Q = q <= 1 ? 1 : (q <= 2 ? 2 : (q <= 4 ? 4 : 8));
    const void* f = Q == 1 ? (const void*)k_gemm_nn<1> : Q == 2 ? (const void*)k_gemm_nn<2>
                  : Q == 4 ? (const void*)k_gemm_nn<4> : (const void*)k_gemm_nn<8>;
    cudaError_t e = set_smem(f, sm);
    if (e != cudaSuccess) return e;
    const int g = grid_for(N, 256);
    if (Q == 1) k_gemm_nn<1><<<g, 256, sm, st>>>(X, p, H, q, Y, N, alpha, beta);
    else if (Q == 2) k_gemm_nn<2><<<g, 256, sm, st>>>(X, p, H, q, Y, N, alpha, beta);
    else if (Q == 4) k_gemm_nn<4><<<g, 256, sm, st>>>(X, p, H, q, Y, N, alpha, beta);
    else k_gemm_nn<8><<<g, 256, sm, st>>>(X, p, H, q, Y, N, alpha, beta);
    return cudaGetLastError();
}

cudaError_t launch_scale_sigma(const double2* X, double2* Y, const double* sigma, long long n, int nvec, int inverse,
                               cudaStream_t st, long long nloc) {
    const long long total = (long long)2 * n * nvec;
    k_scale_sigma<<<grid_for(total, 256), 256, 0, st>>>(X, Y, sigma, n, nloc > 0 ? nloc : n, total, inverse);
    return cudaGetLastError();
}

cudaError_t launch_fill_random(double2* X, long long N, int nvec, unsigned long long seed, long long offset,
                               const double* sigma, long long n, cudaStream_t st, long long nloc) {
    const long long total = N * nvec;
    k_fill_random<<<grid_for(total, 256), 256, 0, st>>>(X, total, seed, offset, sigma, n, nloc > 0 ? nloc : n);
    return cudaGetLastError();
}

cudaError_t launch_copy(double2* dst, const double2* src, long long count, cudaStream_t st) {
    k_copy<<<grid_for(count, 256), 256, 0, st>>>(dst, src, count);
    return cudaGetLastError();
}

cudaError_t launch_cg_init(const CGState& s, const double2* cdot, int nvec, double tol, cudaStream_t st) {
    k_cg_init<<<1, 32, 0, st>>>(s, cdot, nvec, tol);
    return cudaGetLastError();
}

cudaError_t launch_cg_xr(double2* X, double2* R, const double2* P, const double2* MP, const CGState& s, long long N,
                         int nvec, double2* partial, int nblk, cudaStream_t st) {
    k_cg_xr<<<dim3(nblk, nvec), 256, 0, st>>>(X, R, P, MP, s, N, partial);
    return cudaGetLastError();
}

cudaError_t launch_cg_scalars(const CGState& s, const double2* rrnew_c, int nvec, cudaStream_t st) {
    k_cg_scalars<<<1, 32, 0, st>>>(s, rrnew_c, nvec);
    return cudaGetLastError();
}

cudaError_t launch_cg_p(double2* P, const double2* R, const CGState& s, long long N, int nvec, cudaStream_t st) {
    k_cg_p<<<dim3(grid_for(N, 256, 148 * 4), nvec), 256, 0, st>>>(P, R, s, N);
    return cudaGetLastError();
}


int fast_split_N2(int N) {
    switch (N) {
#define BNF_CASE(NN, A, B) case NN: return B;
        BNF_FAST_PLANS(BNF_CASE)
#undef BNF_CASE
        default: return 0;
    }
}

cudaError_t launch_cg_finish(const CGFuse& cg, int which, int nvec, cudaStream_t st) {
    k_cg_finish<<<1, 1024, 0, st>>>(cg, which, nvec);
    return cudaGetLastError();
}

bool fast_all(const OpArgs& a) { return a.fast && has_fast(a.mp.n1) && has_fast(a.mp.n2) && has_fast(a.mp.n3); }

cudaError_t launch_zfwd_cg(const OpArgs& a, const double2* R, double2* P, double2* U, int nvec, const CGFuse& cg,
                           cudaStream_t st) {
    return fast_zfwd(a, R, U, nvec, 1, st, P, &cg);
}
cudaError_t launch_xpass_cg(const OpArgs& a, double2* U, int nvec, const CGFuse& cg, cudaStream_t st) {
    return fast_xpass(a, U, nvec, st, &cg);
}
cudaError_t launch_zadj_cg(const OpArgs& a, const double2* U, double2* X, int nvec, const CGFuse& cg,
                           cudaStream_t st) {
    return fast_zadj(a, U, X, nvec, 1, st, &cg);
}
size_t cg_partials_per_vec(const OpArgs& a) {
    const long long rows = (long long)a.mp.n2 * a.mp.n3;
    const long long gx = (rows + 7) / 8;            // x pass: >= rows / R for every plan (R >= 8)
    const long long gz = ((a.mp.n1 + 3) / 4) * (long long)a.mp.n2;   // z pass: W >= 4
    return (size_t)std::max(3 * gx, gz);
}



}  // namespace bnf
