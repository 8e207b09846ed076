// Register-resident FFT building blocks for sm_100a (complex128).
//
// A length-N DFT along one axis of a tile of W sequences is computed by a
// group of N2 threads per sequence, each holding N1 = N/N2 elements in
// registers (N1 % N2 == 0):
//   stage 1  : N1-point DFT in registers over m        (x[N2 m + t] -> V_t[k1])
//   twiddle  : V_t[k1] *= w_N^{t k1}
//   exchange : one shared-memory transpose
//   stage 2  : N1/N2 N2-point DFTs per thread over t   (-> X[k1 + N1 k2])
// `fft_fwd` takes the natural ("stage-1") layout and leaves the output in
// the "stage-2" layout; `fft_mirror` is the same DFT (any sign) run in
// reverse, from the stage-2 layout back to the natural layout, so a
// forward/inverse pair needs no extra reordering.  All in-register
// twiddles are compile-time constants read from __constant__ tables.
#pragma once

#include <cuda_runtime.h>

namespace bnf {
namespace fast {

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cjmul(double2 a, double2 b) {  // conj(a) * b
    return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
template <int S>
__device__ __forceinline__ double2 mul_i(double2 a) {  // * (S i)
    return S > 0 ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}

// ------------------------------------------------ compile-time twiddles
constexpr double kPiD = 3.14159265358979323846;

__host__ __device__ constexpr double sin_series(double x) {
    double x2 = x * x, term = x, sum = x;
    for (int i = 1; i < 14; ++i) {
        term *= -x2 / ((2.0 * i) * (2.0 * i + 1.0));
        sum += term;
    }
    return sum;
}
__host__ __device__ constexpr double cos_series(double x) {
    double x2 = x * x, term = 1.0, sum = 1.0;
    for (int i = 1; i < 14; ++i) {
        term *= -x2 / ((2.0 * i - 1.0) * (2.0 * i));
        sum += term;
    }
    return sum;
}
// (cos, sin)(2 pi j / N) with exact integer quadrant/octant reduction
__host__ __device__ constexpr double trig2pi(long j, long N, bool want_sin) {
    long r = j % N;
    if (r < 0) r += N;
    const long q = (4 * r) / N;          // quadrant
    const long rr = 4 * r - q * N;       // angle within quadrant = 2 pi rr / (4N)
    const bool flip = 2 * rr > N;        // use the complement for x > pi/4
    const double x = 2.0 * kPiD * (double)(flip ? (N - rr) : rr) / (4.0 * (double)N);
    const double sx = flip ? cos_series(x) : sin_series(x);   // sin of quadrant angle
    const double cx = flip ? sin_series(x) : cos_series(x);   // cos of quadrant angle
    double c = 0, s = 0;
    if (q == 0) { c = cx; s = sx; }
    else if (q == 1) { c = -sx; s = cx; }
    else if (q == 2) { c = -cx; s = -sx; }
    else { c = sx; s = -cx; }
    return want_sin ? s : c;
}

template <int N>
struct TwTab {
    double c[N];
    double s[N];
    constexpr TwTab() : c{}, s{} {
        for (int j = 0; j < N; ++j) {
            c[j] = trig2pi(j, N, false);
            s[j] = trig2pi(j, N, true);
        }
    }
};
template <int N>
__constant__ TwTab<N> kTw = TwTab<N>();

template <int N, int S>
__device__ __forceinline__ double2 ctw(int j) {  // w_N^{S j}, j compile-time after unrolling
    const int jj = j % N;
    return make_double2(kTw<N>.c[jj], S > 0 ? kTw<N>.s[jj] : -kTw<N>.s[jj]);
}

// ------------------------------------------------------- register DFTs
__host__ __device__ constexpr int first_factor(int n) {
    return (n % 4 == 0 && n != 8) ? 4 : (n % 2 == 0 ? 2 : (n % 3 == 0 ? 3 : (n % 5 == 0 ? 5 : n)));
}

template <int N, int S>
struct DFT;

// v * w_N^{S J} with J a compile-time constant: the twiddle is a literal
// (trivial ones -- 1, -1, +-i -- cost no multiplications)
template <int N, int S, int J>
__device__ __forceinline__ double2 twc(double2 a) {
    constexpr int jj = ((J % N) + N) % N;
    if constexpr (jj == 0) {
        return a;
    } else if constexpr (4 * jj == N) {
        return mul_i<S>(a);
    } else if constexpr (2 * jj == N) {
        return make_double2(-a.x, -a.y);
    } else if constexpr (4 * jj == 3 * N) {
        return mul_i<-S>(a);
    } else {
        constexpr double c = trig2pi(jj, N, false);
        constexpr double sn = S > 0 ? trig2pi(jj, N, true) : -trig2pi(jj, N, true);
        return make_double2(a.x * c - a.y * sn, a.x * sn + a.y * c);
    }
}

template <int N, int S, int A, int b, int k1>
__device__ __forceinline__ void tw_row(const double2* t, double2* y) {
    if constexpr (k1 < A) {
        y[b * A + k1] = twc<N, S, b * k1>(t[k1]);
        tw_row<N, S, A, b, k1 + 1>(t, y);
    }
}

template <int N, int S, int A, int B, int b>
__device__ __forceinline__ void dft_cols(const double2* v, double2* y) {
    if constexpr (b < B) {
        double2 t[A];
#pragma unroll
        for (int a = 0; a < A; ++a) t[a] = v[B * a + b];
        DFT<A, S>::run(t);
        tw_row<N, S, A, b, 0>(t, y);
        dft_cols<N, S, A, B, b + 1>(v, y);
    }
}

// Mixed-radix N = A * B register DFT (Cooley-Tukey, compile-time twiddles)
template <int N, int S>
struct DFT {
    static __device__ __forceinline__ void run(double2* v) {
        constexpr int A = first_factor(N);
        constexpr int B = N / A;
        double2 y[N];
        dft_cols<N, S, A, B, 0>(v, y);
#pragma unroll
        for (int k1 = 0; k1 < A; ++k1) {
            double2 t[B];
#pragma unroll
            for (int b = 0; b < B; ++b) t[b] = y[b * A + k1];
            DFT<B, S>::run(t);
#pragma unroll
            for (int k2 = 0; k2 < B; ++k2) v[k1 + A * k2] = t[k2];
        }
    }
};

template <int S>
struct DFT<1, S> {
    static __device__ __forceinline__ void run(double2*) {}
};
template <int S>
struct DFT<2, S> {
    static __device__ __forceinline__ void run(double2* v) {
        const double2 t = v[0];
        v[0] = cadd(t, v[1]);
        v[1] = csub(t, v[1]);
    }
};
template <int S>
struct DFT<3, S> {
    static __device__ __forceinline__ void run(double2* v) {
        const double s3 = 0.86602540378443864676;
        const double2 t = cadd(v[1], v[2]);
        const double2 u = cscale(mul_i<S>(csub(v[1], v[2])), s3);
        const double2 m = csub(v[0], cscale(t, 0.5));
        v[0] = cadd(v[0], t);
        v[1] = cadd(m, u);
        v[2] = csub(m, u);
    }
};
template <int S>
struct DFT<4, S> {
    static __device__ __forceinline__ void run(double2* v) {
        const double2 a0 = cadd(v[0], v[2]), a1 = csub(v[0], v[2]);
        const double2 b0 = cadd(v[1], v[3]), b1 = mul_i<S>(csub(v[1], v[3]));
        v[0] = cadd(a0, b0);
        v[2] = csub(a0, b0);
        v[1] = cadd(a1, b1);
        v[3] = csub(a1, b1);
    }
};
template <int S>
struct DFT<8, S> {
    static __device__ __forceinline__ void run(double2* v) {
        double2 e[4] = {v[0], v[2], v[4], v[6]};
        double2 o[4] = {v[1], v[3], v[5], v[7]};
        DFT<4, S>::run(e);
        DFT<4, S>::run(o);
        const double h = 0.70710678118654752440;
        const double2 t1 = cscale(cadd(o[1], mul_i<S>(o[1])), h);
        const double2 t2 = mul_i<S>(o[2]);
        const double2 t3 = cscale(csub(mul_i<S>(o[3]), o[3]), h);
        v[0] = cadd(e[0], o[0]);
        v[4] = csub(e[0], o[0]);
        v[1] = cadd(e[1], t1);
        v[5] = csub(e[1], t1);
        v[2] = cadd(e[2], t2);
        v[6] = csub(e[2], t2);
        v[3] = cadd(e[3], t3);
        v[7] = csub(e[3], t3);
    }
};

// ------------------------------------------------ exchange layouts
// Element (k1, t, w) of a tile.  W-fast: w is the fastest thread index
// (column tiles of the y/z passes).  T-fast (+1 padding): t fastest (rows of
// the contiguous x axis).
template <int N1, int N2, int W>
struct XchW {
    static __device__ __forceinline__ int idx(int k1, int t, int w) { return (k1 * N2 + t) * W + w; }
    static constexpr int size = N1 * N2 * W;
};
template <int N1, int N2, int W>
struct XchT {
    static __device__ __forceinline__ int idx(int k1, int t, int w) { return (w * N1 + k1) * (N2 + 1) + t; }
    static constexpr int size = W * N1 * (N2 + 1);
};

template <int S>
__device__ __forceinline__ double2 root_tw(const double2* __restrict__ root, int t) {
    const double2 w = __ldg(root + t);
    return S > 0 ? w : cconj(w);
}

// `root` is the axis' stage-twiddle table laid out [k1][t]: root[k1 * N2 + t]
// = e^{2 pi i t k1 / N} (AxisPlan::root2), so the N2 threads of a sequence that
// sit in one warp read consecutive entries (one wavefront per load).
// Natural layout -> stage-2 layout.  On exit v[u*N2 + k2] = X[k1 + N1*k2]
// with k1 = t + N2*u.  Two __syncthreads (buffer free on exit).
// RS = true: `root` is a shared-memory copy of the table (plain loads instead of __ldg).
template <int S, bool RS>
__device__ __forceinline__ double2 root_at(const double2* __restrict__ root, int t) {
    if constexpr (RS) {
        const double2 w = root[t];
        return S > 0 ? w : cconj(w);
    } else {
        return root_tw<S>(root, t);
    }
}

// WS = true: the N2 threads of a sequence sit in one warp and the warp's sequences own a private
// region of `xch` (XchT with w = tid / N2, N2 | 32), so the exchange is ordered by __syncwarp and
// the warps of the CTA run independently.
template <bool WS>
__device__ __forceinline__ void xch_sync() {
    if constexpr (WS) __syncwarp();
    else __syncthreads();
}

template <int N1, int N2, int S, class X, bool RS = false, bool WS = false>
__device__ __forceinline__ void fft_fwd(double2 (&v)[N1], int t, int w, double2* xch, const double2* root) {
    DFT<N1, S>::run(v);
    if (t > 0) {
#pragma unroll
        for (int k1 = 1; k1 < N1; ++k1) v[k1] = cmul(v[k1], root_at<S, RS>(root, k1 * N2 + t));
    }
#pragma unroll
    for (int k1 = 0; k1 < N1; ++k1) xch[X::idx(k1, t, w)] = v[k1];
    xch_sync<WS>();
    constexpr int U = N1 / N2;
#pragma unroll
    for (int u = 0; u < U; ++u) {
        double2 a[N2];
        const int k1 = t + N2 * u;
#pragma unroll
        for (int tt = 0; tt < N2; ++tt) a[tt] = xch[X::idx(k1, tt, w)];
        DFT<N2, S>::run(a);
#pragma unroll
        for (int k2 = 0; k2 < N2; ++k2) v[u * N2 + k2] = a[k2];
    }
    xch_sync<WS>();
}

// Stage-2 layout -> natural layout (the same DFT run in reverse order).
template <int N1, int N2, int S, class X, bool RS = false, bool WS = false>
__device__ __forceinline__ void fft_mirror(double2 (&v)[N1], int t, int w, double2* xch, const double2* root) {
    constexpr int U = N1 / N2;
#pragma unroll
    for (int u = 0; u < U; ++u) {
        double2 a[N2];
#pragma unroll
        for (int k2 = 0; k2 < N2; ++k2) a[k2] = v[u * N2 + k2];
        DFT<N2, S>::run(a);
        const int k1 = t + N2 * u;
#pragma unroll
        for (int tt = 0; tt < N2; ++tt) xch[X::idx(k1, tt, w)] = a[tt];
    }
    xch_sync<WS>();
#pragma unroll
    for (int k1 = 0; k1 < N1; ++k1) v[k1] = xch[X::idx(k1, t, w)];
    xch_sync<WS>();
    if (t > 0) {
#pragma unroll
        for (int k1 = 1; k1 < N1; ++k1) v[k1] = cmul(v[k1], root_at<S, RS>(root, k1 * N2 + t));
    }
    DFT<N1, S>::run(v);
}

// ------------------------------------- 2N-point DFT as even / odd N-point halves
// A sequence of 2N = 2 N1 N2 points held as pairs: thread t has x[2(N2 m + t)]
// in a[m] and x[2(N2 m + t) + 1] in b[m] (m < N1, so every thread's elements are
// adjacent pairs -- one 256-bit global access each).  N1 == N2 (one stage-2 DFT
// per thread).  Forward (S): X[k] = E[k] + w_2N^{S k} O[k], X[k + N] = E[k] - ...,
// E, O the N-point DFTs of the halves (one shared exchange round for both,
// buffers xa and xb); on exit v[q] = X[t + N2 q], q < 2 N1.  `root` is the 2N
// axis' [k1][t] stage table (entry k N2 + t = w_2N^{t k}): the N-point stage
// roots are its even rows, w_2N^{t} is row 1.  RS: `root` in shared memory.
template <int N1, int S, int K>
__device__ __forceinline__ void eo_comb_fwd(const double2* a, const double2* b, double2* v, double2 wt) {
    if constexpr (K < N1) {
        const double2 o = cmul(twc<2 * N1, S, K>(b[K]), wt);
        v[K] = cadd(a[K], o);
        v[K + N1] = csub(a[K], o);
        eo_comb_fwd<N1, S, K + 1>(a, b, v, wt);
    }
}
template <int N1, int S, int K>
__device__ __forceinline__ void eo_comb_inv(const double2* v, double2* a, double2* b, double2 wt) {
    if constexpr (K < N1) {
        a[K] = cadd(v[K], v[K + N1]);
        b[K] = cmul(twc<2 * N1, S, K>(csub(v[K], v[K + N1])), wt);
        eo_comb_inv<N1, S, K + 1>(v, a, b, wt);
    }
}

template <int N1, int N2, int S, class X, bool RS>
__device__ __forceinline__ void fft_fwd_eo(double2 (&a)[N1], double2 (&b)[N1], double2 (&v)[2 * N1], int t, int w,
                                           double2* xa, double2* xb, const double2* root) {
    static_assert(N1 == N2, "fft_fwd_eo: N1 == N2");
    DFT<N1, S>::run(a);
    DFT<N1, S>::run(b);
    if (t > 0) {
#pragma unroll
        for (int k1 = 1; k1 < N1; ++k1) {
            const double2 r = root_at<S, RS>(root, 2 * k1 * N2 + t);
            a[k1] = cmul(a[k1], r);
            b[k1] = cmul(b[k1], r);
        }
    }
#pragma unroll
    for (int k1 = 0; k1 < N1; ++k1) {
        xa[X::idx(k1, t, w)] = a[k1];
        xb[X::idx(k1, t, w)] = b[k1];
    }
    __syncthreads();
#pragma unroll
    for (int tt = 0; tt < N2; ++tt) {
        a[tt] = xa[X::idx(t, tt, w)];
        b[tt] = xb[X::idx(t, tt, w)];
    }
    __syncthreads();
    DFT<N2, S>::run(a);
    DFT<N2, S>::run(b);
    const double2 wt = root_at<S, RS>(root, N2 + t);   // w_2N^{S t}
    eo_comb_fwd<N1, S, 0>(a, b, v, wt);   // k = t + N2 k2 < N:  w_2N^{S k} = w_2N^{S t} w_{2N1}^{S k2}
}

// Inverse of the layout above (any sign S): v[q] = Y[t + N2 q] in, the 2N-point
// DFT (sign S) out as pairs: a[m] = y[2(N2 m + t)], b[m] = y[2(N2 m + t) + 1].
template <int N1, int N2, int S, class X, bool RS>
__device__ __forceinline__ void fft_mirror_eo(double2 (&v)[2 * N1], double2 (&a)[N1], double2 (&b)[N1], int t, int w,
                                              double2* xa, double2* xb, const double2* root) {
    static_assert(N1 == N2, "fft_mirror_eo: N1 == N2");
    const double2 wt = root_at<S, RS>(root, N2 + t);
    eo_comb_inv<N1, S, 0>(v, a, b, wt);   // even outputs from Y[k] + Y[k+N], odd from (Y[k] - Y[k+N]) w^{S k}
    DFT<N2, S>::run(a);
    DFT<N2, S>::run(b);
#pragma unroll
    for (int tt = 0; tt < N2; ++tt) {
        xa[X::idx(t, tt, w)] = a[tt];
        xb[X::idx(t, tt, w)] = b[tt];
    }
    __syncthreads();
#pragma unroll
    for (int k1 = 0; k1 < N1; ++k1) {
        a[k1] = xa[X::idx(k1, t, w)];
        b[k1] = xb[X::idx(k1, t, w)];
    }
    __syncthreads();
    if (t > 0) {
#pragma unroll
        for (int k1 = 1; k1 < N1; ++k1) {
            const double2 r = root_at<S, RS>(root, 2 * k1 * N2 + t);
            a[k1] = cmul(a[k1], r);
            b[k1] = cmul(b[k1], r);
        }
    }
    DFT<N1, S>::run(a);
    DFT<N1, S>::run(b);
}

// ------------------------------------------ warp-local variants (no CTA barrier)
// The N2 threads of a sequence are consecutive lanes of one warp (lane =
// w * N2 + t, W = 32 / N2 sequences per warp), so the stage exchange is an
// N2 x N2 transpose per u inside the warp.  XSHFL = 1: by xor shuffles
// (log2 N2 stages; element (lane t, slot u N2 + s) -> (lane s, slot u N2 + t));
// XSHFL = 0: through a per-warp shared-memory region `xw` with __syncwarp
// (padded layout k1 * S1 + t * S2 + w, conflict-free for 16-byte accesses).
template <int N1, int N2>
struct WarpXch {
    static constexpr int W = 32 / N2;
    static constexpr int S2 = W + 1;
    static constexpr int S1 = N2 * S2 + 1;
    static constexpr int size = N1 * S1;   // complex elements per warp
};

__device__ __forceinline__ double2 shfl_xor2(double2 v, int d) {
    return make_double2(__shfl_xor_sync(0xffffffffu, v.x, d), __shfl_xor_sync(0xffffffffu, v.y, d));
}

template <int N1, int N2, int XSHFL>
__device__ __forceinline__ void warp_xpose(double2 (&v)[N1], int t, int w, double2* xw) {
    if constexpr (XSHFL) {
#pragma unroll
        for (int d = 1; d < N2; d <<= 1) {
            const bool p = (t & d) != 0;
#pragma unroll
            for (int u = 0; u < N1 / N2; ++u)
#pragma unroll
                for (int s = 0; s < N2; ++s) {
                    if (s & d) continue;
                    double2& a = v[u * N2 + s];
                    double2& b = v[u * N2 + (s ^ d)];
                    const double2 r = shfl_xor2(p ? a : b, d);
                    if (p) a = r;
                    else b = r;
                }
        }
    } else {
        using X = WarpXch<N1, N2>;
#pragma unroll
        for (int k1 = 0; k1 < N1; ++k1) xw[k1 * X::S1 + t * X::S2 + w] = v[k1];
        __syncwarp();
#pragma unroll
        for (int u = 0; u < N1 / N2; ++u)
#pragma unroll
            for (int tt = 0; tt < N2; ++tt) v[u * N2 + tt] = xw[(t + N2 * u) * X::S1 + tt * X::S2 + w];
        __syncwarp();
    }
}

// As fft_fwd (natural -> stage-2 layout), warp-local.  `root` as in fft_fwd
// (global [k1][t] table, or a shared-memory copy).
template <int N1, int N2, int S, int XSHFL>
__device__ __forceinline__ void fft_fwd_w(double2 (&v)[N1], int t, int w, double2* xw, const double2* root) {
    DFT<N1, S>::run(v);
    if (t > 0) {
#pragma unroll
        for (int k1 = 1; k1 < N1; ++k1) {
            const double2 r = root[k1 * N2 + t];
            v[k1] = cmul(v[k1], S > 0 ? r : cconj(r));
        }
    }
    warp_xpose<N1, N2, XSHFL>(v, t, w, xw);
#pragma unroll
    for (int u = 0; u < N1 / N2; ++u) {
        double2 a[N2];
#pragma unroll
        for (int q = 0; q < N2; ++q) a[q] = v[u * N2 + q];
        DFT<N2, S>::run(a);
#pragma unroll
        for (int q = 0; q < N2; ++q) v[u * N2 + q] = a[q];
    }
}

// As fft_mirror (stage-2 -> natural layout), warp-local.
template <int N1, int N2, int S, int XSHFL>
__device__ __forceinline__ void fft_mirror_w(double2 (&v)[N1], int t, int w, double2* xw, const double2* root) {
#pragma unroll
    for (int u = 0; u < N1 / N2; ++u) {
        double2 a[N2];
#pragma unroll
        for (int q = 0; q < N2; ++q) a[q] = v[u * N2 + q];
        DFT<N2, S>::run(a);
#pragma unroll
        for (int q = 0; q < N2; ++q) v[u * N2 + q] = a[q];
    }
    warp_xpose<N1, N2, XSHFL>(v, t, w, xw);
    if (t > 0) {
#pragma unroll
        for (int k1 = 1; k1 < N1; ++k1) {
            const double2 r = root[k1 * N2 + t];
            v[k1] = cmul(v[k1], S > 0 ? r : cconj(r));
        }
    }
    DFT<N1, S>::run(v);
}

// ------------------------------------------- twiddle sequences (no long chains)
// w^b for the N1 elements a thread holds after fft_fwd (stage-2 layout,
// b = t + N2 u + N1 k2) or before it (natural layout, b = N2 m + t), built from
// the three bases w^t, w^N2, w^N1 with product trees of depth <= 3 instead of
// one sequential multiplication chain per element (the chain's FP64 latency
// was exposed).  Multiplies v in place.
template <int K>
struct Pow4 {   // g^k = q[k / 4] p[k % 4], k < K
    static constexpr int R = K < 4 ? K : 4;
    static constexpr int Q = (K + R - 1) / R;
    double2 p[R], q[Q];
    __device__ __forceinline__ explicit Pow4(double2 g) {
        p[0] = make_double2(1.0, 0.0);
        if constexpr (R > 1) p[1] = g;
        if constexpr (R > 2) p[2] = cmul(g, g);
        if constexpr (R > 3) p[3] = cmul(p[2], g);
        q[0] = make_double2(1.0, 0.0);
        if constexpr (Q > 1) {
            const double2 gR = (R == 4) ? cmul(p[2], p[2]) : (R == 3 ? cmul(p[2], g) : (R == 2 ? p[2 % R] : g));
            q[1] = gR;
#pragma unroll
            for (int s = 2; s < Q; ++s) q[s] = cmul(q[s - 1], gR);
        }
    }
};

template <int N1, int N2>
__device__ __forceinline__ void twiddle_stage2(double2 (&v)[N1], double2 wt, double2 wN2, double2 wN1) {
    static_assert(N2 >= 4 || N2 == 2, "twiddle_stage2: N2 in {2} or >= 4");
    if constexpr (N2 == 2) {
        double2 au = wt;
#pragma unroll
        for (int u = 0; u < N1 / N2; ++u) {
            v[u * N2] = cmul(v[u * N2], au);
            v[u * N2 + 1] = cmul(v[u * N2 + 1], cmul(au, wN1));
            au = cmul(au, wN2);
        }
    } else {
        const Pow4<N2> B(wN1);
        double2 au = wt;
#pragma unroll
        for (int u = 0; u < N1 / N2; ++u) {
            double2 c[Pow4<N2>::Q];
#pragma unroll
            for (int s = 0; s < Pow4<N2>::Q; ++s) c[s] = s == 0 ? au : cmul(au, B.q[s]);
#pragma unroll
            for (int k2 = 0; k2 < N2; ++k2)
                v[u * N2 + k2] = cmul(v[u * N2 + k2], (k2 % 4 == 0) ? c[k2 / 4] : cmul(c[k2 / 4], B.p[k2 % 4]));
            au = cmul(au, wN2);
        }
    }
}

template <int N1, int N2>
__device__ __forceinline__ void twiddle_natural(double2 (&v)[N1], double2 wt, double2 wN2) {
    const Pow4<N1> B(wN2);
    double2 c[Pow4<N1>::Q];
#pragma unroll
    for (int s = 0; s < Pow4<N1>::Q; ++s) c[s] = s == 0 ? wt : cmul(wt, B.q[s]);
#pragma unroll
    for (int m = 0; m < N1; ++m)
        v[m] = cmul(v[m], (m % Pow4<N1>::R == 0) ? c[m / Pow4<N1>::R] : cmul(c[m / Pow4<N1>::R], B.p[m % Pow4<N1>::R]));
}

}  // namespace fast
}  // namespace bnf
