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

template <int SIGN>
__device__ void stage_generic(int R, int N, const double2* __restrict__ A, double2* __restrict__ B, int ld, int col,
                              int j, int nb, int k, int tstride, int base, int Ns,
                              const double2* __restrict__ root) {
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
    sig = sqrt(q);
    const double2 d1 = csub(lam[2], lam[1]);
    const double2 d2 = csub(lam[0], lam[2]);
    const double2 d3 = csub(lam[1], lam[0]);
    const double p2 = cabs2(d1) + cabs2(d2) + cabs2(d3);
    if (p2 > p.taup * q) {
        const double r1 = rsqrt(p2 * q);
        const double r2 = rsqrt(p2);
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
    const double rq = 1.0 / sig;
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
            const double s = (op == 0) ? sig : 1.0;
            for (int l = 0; l < 3; ++l) o[l] = cscale(cadd(cmul(pi1[l], u1), cmul(pi2[l], u2)), s);
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
    const double* einv = eps_inv + (size_t)l * n;
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
        Uv[base + e] = cscale(res[aa * ld + row], sv * __ldg(einv + base + e));
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

__global__ void k_sigma_table(ModeP p, double* __restrict__ sigma) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < p.n;
         t += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(t % p.n1);
        const int j = (int)((t / p.n1) % p.n2);
        const int k = (int)(t / p.n12);
        double2 lam[3];
        mode_lambdas(p, i, j, k, lam);
        const double q = cabs2(lam[0]) + cabs2(lam[1]) + cabs2(lam[2]);
        sigma[t] = (t == p.gamma) ? 0.0 : sqrt(q);
    }
}

// ---------------------------------------------------------- BLAS-1 / tall-skinny
__device__ __forceinline__ double2 warp_sum(double2 v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
        v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
    }
    return v;
}

// block-wide sum of one complex value (blockDim.x multiple of 32, <= 1024)
__device__ double2 block_sum(double2 v, double2* red) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
    __syncthreads();
    if (ln == 0) red[w] = v;
    __syncthreads();
    double2 r = make_double2(0, 0);
    if (w == 0) {
        r = (ln < (int)(blockDim.x >> 5)) ? red[ln] : make_double2(0, 0);
        r = warp_sum(r);
    }
    return r;  // valid in thread 0
}

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
// Block = 8 warps over a slice of GT_SLICE rows (grid-stride over slices).
// The Y slice is staged in shared memory; warp w owns the columns a = w mod 8
// of X, streams X_a over the slice and accumulates into acc[a][c] (owned
// exclusively by that warp -> deterministic, no atomics).  partial[(a*q+c)*nblk + blk].
constexpr int GT_SLICE = 512;
template <int Q>
__global__ void __launch_bounds__(256) k_gemm_tn_partial(const double2* __restrict__ X, int p,
                                                         const double2* __restrict__ Y, int q, long long N,
                                                         double2* __restrict__ partial) {
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
#pragma unroll 4
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

// Y_c = beta Y_c + alpha sum_a X_a H[a*q + c]   (H on device, p*q <= 4096)
__global__ void __launch_bounds__(256) k_gemm_nn(const double2* X, int p, const double2* __restrict__ H,
                                                 int q, double2* Y, long long N, double alpha,
                                                 double beta) {
    extern __shared__ double2 hs[];
    for (int t = threadIdx.x; t < p * q; t += blockDim.x) hs[t] = H[t];
    __syncthreads();
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < N; r += (long long)gridDim.x * blockDim.x) {
        double2 acc[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[c] = make_double2(0, 0);
        for (int aidx = 0; aidx < p; ++aidx) {
            const double2 x = X[(size_t)aidx * N + r];
#pragma unroll
            for (int c = 0; c < 8; ++c)
                if (c < q) acc[c] = cadd(acc[c], cmul(x, hs[aidx * q + c]));
        }
        for (int c = 0; c < q; ++c) {
            double2 y = (beta == 0.0) ? make_double2(0, 0) : cscale(Y[(size_t)c * N + r], beta);
            Y[(size_t)c * N + r] = cadd(y, cscale(acc[c], alpha));
        }
    }
}

// Y = X * sigma^{+-1} on both halves of every 2n vector (masked: 0)
__global__ void k_scale_sigma(const double2* __restrict__ X, double2* __restrict__ Y, const double* __restrict__ sigma,
                              long long n, long long total, int inverse) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const double s = sigma[t % n];
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
                              const double* __restrict__ sigma, long long n) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const unsigned long long h1 = splitmix64(seed ^ splitmix64((unsigned long long)(t + offset) * 2ull));
        const unsigned long long h2 = splitmix64(seed ^ splitmix64((unsigned long long)(t + offset) * 2ull + 1ull));
        const double u1 = ((h1 >> 11) + 1.0) * (1.0 / 9007199254740993.0);
        const double u2 = (h2 >> 11) * (1.0 / 9007199254740992.0);
        const double rad = sqrt(-2.0 * log(u1));
        double s, c;
        sincospi(2.0 * u2, &s, &c);
        const double m = (sigma != nullptr && sigma[t % n] == 0.0) ? 0.0 : 1.0;
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

inline int grid_for(long long total, int threads, int cap = 148 * 16) {
    long long g = (total + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (int)g;
}

}  // namespace

// ---------------------------------------------------------------- launchers
static size_t smem_z(const OpArgs& a) { return (size_t)4 * a.mp.n3 * a.W_z * sizeof(double2); }
static size_t smem_y(const OpArgs& a) { return (size_t)2 * a.mp.n2 * a.W_y * sizeof(double2); }
static size_t smem_x(const OpArgs& a) { return (size_t)2 * a.mp.n1 * (a.R_x + 1) * sizeof(double2); }

static cudaError_t set_smem(const void* f, size_t bytes) {
    if (bytes > 48 * 1024) return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    return cudaSuccess;
}

cudaError_t launch_zfwd(const OpArgs& a, const double2* Y, double2* U, int nvec, int op, cudaStream_t st) {
    const size_t sm = smem_z(a);
    cudaError_t e = set_smem((const void*)k_zfwd, sm);
    if (e != cudaSuccess) return e;
    dim3 g((a.mp.n1 + a.W_z - 1) / a.W_z, a.mp.n2, nvec);
    k_zfwd<<<g, 256, sm, st>>>(Y, U, a, op);
    return cudaGetLastError();
}

cudaError_t launch_zadj(const OpArgs& a, const double2* U, double2* OUT, int nvec, int op, cudaStream_t st) {
    const size_t sm = smem_z(a);
    cudaError_t e = set_smem((const void*)k_zadj, sm);
    if (e != cudaSuccess) return e;
    dim3 g((a.mp.n1 + a.W_z - 1) / a.W_z, a.mp.n2, nvec);
    k_zadj<<<g, 256, sm, st>>>(U, OUT, a, op);
    return cudaGetLastError();
}

cudaError_t launch_ypass(const OpArgs& a, double2* U, int nvec, int adjoint, cudaStream_t st) {
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

cudaError_t launch_sigma_table(const ModeP& mp, double* sigma, cudaStream_t st) {
    k_sigma_table<<<grid_for(mp.n, 256), 256, 0, st>>>(mp, sigma);
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
    const int Q = q <= 1 ? 1 : (q <= 2 ? 2 : (q <= 4 ? 4 : 8));
    if (q > 8) return cudaErrorInvalidValue;
    const size_t sm = ((size_t)Q * GT_SLICE + (size_t)p * q) * sizeof(double2);
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
    cudaError_t e = set_smem((const void*)k_gemm_nn, sm);
    if (e != cudaSuccess) return e;
    k_gemm_nn<<<grid_for(N, 256), 256, sm, st>>>(X, p, H, q, Y, N, alpha, beta);
    return cudaGetLastError();
}

cudaError_t launch_scale_sigma(const double2* X, double2* Y, const double* sigma, long long n, int nvec, int inverse,
                               cudaStream_t st) {
    const long long total = (long long)2 * n * nvec;
    k_scale_sigma<<<grid_for(total, 256), 256, 0, st>>>(X, Y, sigma, n, total, inverse);
    return cudaGetLastError();
}

cudaError_t launch_fill_random(double2* X, long long N, int nvec, unsigned long long seed, long long offset,
                               const double* sigma, long long n, cudaStream_t st) {
    const long long total = N * nvec;
    k_fill_random<<<grid_for(total, 256), 256, 0, st>>>(X, total, seed, offset, sigma, n);
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

}  // namespace bnf
