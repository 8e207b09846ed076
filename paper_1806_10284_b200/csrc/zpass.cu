// Fourier-side z passes of the null-space-free matvec (SURVEY.md §8(a)
// a1-a2 and a4-a5; §5.3):
//
//   zfwd : Sigma_r, Pi combine (2 -> 3 components), z-DFT k -> c (+),
//          twiddle e^{+2 pi i c N3(i,j)/n}                       (Alg. 2 step 1)
//   zadj : conj twiddle, z-DFT c -> k (-), Pi^* combine (3 -> 2), Sigma_r
//                                                                (Alg. 1 step 3)
//
// One CTA per column tile (W consecutive i, one j, all k); the whole tile is
// fetched with cp.async at once and two CTAs per SM overlap one tile's HBM
// traffic with the other's FP64 mode algebra and register FFTs.  Inter-axis
// twiddles are
// products of three exact table entries (no per-element table gathers);
// lambda3 along k comes from the column's half angle and an exact
// e^{i pi k/n3} table (modes.cuh).
//
// CG-fused variants (cg_solve_fused, solver.cu), per iteration:
//   zfwd_cg : x += alpha_prev p;  p <- r + beta p;  U = Q_r-side of p
//   zadj_cg : r -= alpha M p;  per-CTA partial (r, r); k_cg_finish forms beta
// (the x update is deferred by one iteration so that zadj touches only U
// and r; the final update is k_cg_xfinal).
#include <cuda_runtime.h>

#include <algorithm>

#include "cgfuse.cuh"
#include "fastfft.cuh"
#include "kernels.cuh"
#include "modes.cuh"

#ifndef BNF_Z_MINB
#define BNF_Z_MINB 3   // resident CTAs per SM the z passes are compiled for
#endif

namespace bnf {
namespace {

using fast::cmul;
using fast::cscale;
using modes::Coef;
using modes::Col;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

__device__ __forceinline__ double2 tw_at(const TwP& t, unsigned long long P) {  // e^{2 pi i P / n}
    return cmul(__ldg(t.hi + (P >> t.shift)), __ldg(t.lo + (P & t.mask)));
}
__device__ __forceinline__ double2 conj2(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cjm(double2 a, double2 b) {   // conj(a) b
    return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.x, b.y, -a.y * b.x));
}
__device__ __forceinline__ double2 cadd3(double2 a, double2 b, double2 c) {
    return make_double2(a.x + b.x + c.x, a.y + b.y + c.y);
}

// Real-space side of the z passes in slab-major order [q][vec][l][cl][jl][i]
// (c = q n3loc + cl; q = the z-slab the rows are sent to; blocks
// of nblk = n1 n2loc n3loc elements); with one slab this is the plain
// [vec][l][c][j][i].  Offset of row c of
// component l of vector vec, relative to the column (jl, i) offset.
template <int SL>
__device__ __forceinline__ size_t u_row(const OpArgs& a, int nvec, int vec, int l, int c, size_t kstride) {
    if constexpr (SL == 0) return ((size_t)vec * 3 + l) * a.nloc + kstride * (size_t)c;
    const int q = c / a.n3loc, cl = c - q * a.n3loc;
    return (((size_t)q * nvec + vec) * 3 + l) * a.nblk + kstride * (size_t)cl;
}

template <int N1, int N2, int W>
struct ZCfg;
// resident CTAs per SM the z passes are compiled for (register budget)
constexpr int z_minb(int nt) { return nt > 256 ? 2 : (nt <= 96 ? 5 : BNF_Z_MINB); }

template <int N1, int N2, int W>
struct ZCfg {
    static constexpr int N = N1 * N2;
    static constexpr int NT = 3 * W * N2;
    static constexpr int TE = N * W;                 // elements per array tile
    static constexpr int S = (TE + NT - 1) / NT;      // elements per thread in the mode loops
};

struct ColS {   // per-column constants shared through smem
    Col cm;
    unsigned long long base3;   // N3(i, j) mod n
};

// ------------------------------------------------------------------ zfwd
// One CTA per column tile (W consecutive i, one j, all k, one vector).  All
// tile inputs are issued at once with cp.async (no register cost), so two
// CTAs per SM overlap one tile's loads with the other's FP64 work.  The
// three component tiles of the FFT phase alias the consumed input stage.
// MODE 0: U = Q_r Sigma_op Y (op = runtime 0 A_r / 1 M).  MODE 1: CG (op M).
template <int N1, int N2, int W, int MODE, int SL = 0, int RST = 0, int MB = 0>
__global__ void __launch_bounds__(ZCfg<N1, N2, W>::NT, MB ? MB : z_minb(ZCfg<N1, N2, W>::NT))
    k_zfwd2(const double2* __restrict__ Y, double2* __restrict__ U, OpArgs a, int op, double2* __restrict__ Pcg,
            double2* __restrict__ Xcg, CGFuse cg) {
    using C = ZCfg<N1, N2, W>;
    constexpr int NT = C::NT, TE = C::TE;
    extern __shared__ double2 sm[];   // [NA][TE]: y1 y2 (+1) | r1 r2 p1 p2; Ct = [0..3)
    __shared__ ColS cs[W];
    __shared__ double2 rz_s[N1 * N2], hz_s[N1 * N2];   // z stage roots and e^{i pi k / n3} (RSZ)
    constexpr bool RSZ = true;
    const ModeP& p = a.mp;
    const long long n = a.nloc;                         // per-component stride on this slab
    const int n1 = p.n1;
    const size_t kstride = (size_t)n1 * a.n2loc;       // local k stride (j-slab)
    const long long kglob = (long long)n1 * p.n2;      // global k stride (mode index)
    const int tid = threadIdx.x;
    const int i0 = blockIdx.x * W, j = blockIdx.y + a.j0, vec = blockIdx.z;
    const size_t col0 = (size_t)i0 + (size_t)n1 * blockIdx.y;
    {
        const double2* y1 = Y + (size_t)vec * a.vsf + col0;
        const double2* p1 = MODE ? Pcg + (size_t)vec * a.vsf + col0 : nullptr;
#pragma unroll 2
        for (int q = tid; q < TE; q += NT) {
            const size_t g = (size_t)(q % W) + kstride * (size_t)(q / W);
            cp_async16(sm + q, y1 + g);
            cp_async16(sm + TE + q, y1 + n + g);
            if (MODE == 1) {
                cp_async16(sm + 2 * TE + q, p1 + g);
                cp_async16(sm + 3 * TE + q, p1 + n + g);
                if (RST == 1) {   // x staged too: every input of the tile in flight at once
                    const double2* x1 = Xcg + (size_t)vec * a.vsf + col0;
                    cp_async16(sm + 4 * TE + q, x1 + g);
                    cp_async16(sm + 5 * TE + q, x1 + n + g);
                }
            }
        }
        cp_async_commit();
    }
    if (tid < W) {
        const int i = i0 + tid;
        cs[tid].cm = modes::col(p, i, j);
        cs[tid].base3 = (unsigned long long)((p.cbp * (long long)i + (p.n - p.n1m3) * (long long)j) % p.n);
    }
    if (RSZ && !(a.zcfg & 256))
        for (int q = tid; q < N1 * N2; q += NT) {
            rz_s[q] = __ldg(a.pz.root2 + q);
            hz_s[q] = __ldg(a.hroot_z + q);
        }
    const bool rsz = RSZ && !(a.zcfg & 256);
    const double alpha_prev = MODE ? cg.alpha[vec] : 0.0;
    const double beta = MODE ? cg.beta[vec] : 0.0;
    const int w = tid % W;
    const size_t gcol = col0 + w;
    double2* xcol = MODE ? Xcg + (size_t)vec * a.vsf + gcol : nullptr;
    constexpr int J = (TE + NT - 1) / NT;   // elements per thread in the mode loop
    double2 xb1[RST == 2 ? J : 1], xb2[RST == 2 ? J : 1];
    if (MODE == 1 && RST == 2) {   // every x element of this thread in flight with the r / p tile
#pragma unroll
        for (int jj = 0; jj < J; ++jj) {
            const int e = tid + jj * NT;
            if (e < TE) {
                xb1[jj] = xcol[kstride * (e / W)];
                xb2[jj] = xcol[n + kstride * (e / W)];
            }
        }
    }
    // x is streamed straight from HBM (not staged), two elements ahead; the first two are issued
    // before the wait for the r / p tile so that their latency overlaps it
    double2 xn1 = make_double2(0, 0), xn2 = make_double2(0, 0), xm1 = xn1, xm2 = xn1;
    if (MODE == 1 && RST == 0) {
        if (tid < TE) {
            xn1 = xcol[kstride * (tid / W)];
            xn2 = xcol[n + kstride * (tid / W)];
        }
        if (tid + NT < TE) {
            xm1 = xcol[kstride * ((tid + NT) / W)];
            xm2 = xcol[n + kstride * ((tid + NT) / W)];
        }
    }
    cp_async_wait0();
    __syncthreads();
    const ColS& c = cs[w];
    // ---- phase A: mode algebra, element e = (k, w), k = e / W ----
    // (RST 2: unrolled over jj with a compile-time trip count so that xb1 / xb2 stay in registers)
    auto elem = [&](const int e, double2 x1, double2 x2) {
        const int k = e / W;
        double2 u1 = sm[e], u2 = sm[TE + e];
        if (MODE == 1) {
            const double2 q1 = sm[2 * TE + e], q2 = sm[3 * TE + e];
            if (RST == 1) {
                x1 = sm[4 * TE + e];
                x2 = sm[5 * TE + e];
            }
            double2* xg = xcol + kstride * k;
            xg[0] = make_double2(fma(alpha_prev, q1.x, x1.x), fma(alpha_prev, q1.y, x1.y));   // x += alpha_prev p
            xg[n] = make_double2(fma(alpha_prev, q2.x, x2.x), fma(alpha_prev, q2.y, x2.y));
            u1 = make_double2(fma(beta, q1.x, u1.x), fma(beta, q1.y, u1.y));   // p <- r + beta p
            u2 = make_double2(fma(beta, q2.x, u2.x), fma(beta, q2.y, u2.y));
            double2* pg = Pcg + (size_t)vec * a.vsf + gcol + kstride * k;
            pg[0] = u1;
            pg[n] = u2;
        }
        const double2 l2 = modes::lam3(p, c.cm, rsz ? hz_s[k] : __ldg(a.hroot_z + k));
        Coef o;
        const long long idx = c.cm.idx0 + kglob * k;
        modes::coef(p, c.cm.lam1, c.cm.lam2, l2, idx == p.gamma, MODE ? 1 : op, o);
        const double2 U1 = cscale(u1, o.f1), U2 = cscale(u2, o.f2);
        sm[e] = modes::comb(o, 0, U1, U2);           // component tiles alias the consumed inputs
        sm[TE + e] = modes::comb(o, 1, U1, U2);
        sm[2 * TE + e] = modes::comb(o, 2, U1, U2);
    };
    if (MODE == 1 && RST == 2) {
#pragma unroll
        for (int jj = 0; jj < J; ++jj)
            if (tid + jj * NT < TE) elem(tid + jj * NT, xb1[jj], xb2[jj]);
    } else {
#pragma unroll 1
        for (int e = tid; e < TE; e += NT) {
            const double2 x1 = xn1, x2 = xn2;
            if (MODE == 1 && RST == 0) {   // x streamed two elements ahead
                xn1 = xm1;
                xn2 = xm2;
                if (e + 2 * NT < TE) {
                    xm1 = xcol[kstride * ((e + 2 * NT) / W)];
                    xm2 = xcol[n + kstride * ((e + 2 * NT) / W)];
                }
            }
            elem(e, x1, x2);
        }
    }
    __syncthreads();
    // ---- phase B: z-DFT of component l over k, twiddle, store ----
    {
        const int l = tid / (W * N2), t = (tid / W) % N2;
        double2* ct = sm + (size_t)l * TE;
        double2 v[N1];
#pragma unroll
        for (int m = 0; m < N1; ++m) v[m] = ct[(N2 * m + t) * W + w];
        __syncthreads();
        if (rsz) fast::fft_fwd<N1, N2, 1, fast::XchW<N1, N2, W>, true>(v, t, w, ct, rz_s);
        else fast::fft_fwd<N1, N2, 1, fast::XchW<N1, N2, W>>(v, t, w, ct, a.pz.root2);
        const unsigned long long nn = (unsigned long long)p.n, N3 = c.base3;   // e^{2 pi i P / n}: global n
        const double2 wt = tw_at(a.tw, ((unsigned long long)t * N3) % nn);
        const double2 wu = tw_at(a.tw, ((unsigned long long)N2 * N3) % nn);
        const double2 wk = tw_at(a.tw, ((unsigned long long)N1 * N3) % nn);
        double2* out = U + gcol;
        fast::twiddle_stage2<N1, N2>(v, wt, wu, wk);
#pragma unroll
        for (int u = 0; u < N1 / N2; ++u)
#pragma unroll
            for (int k2 = 0; k2 < N2; ++k2)
                out[u_row<SL>(a, gridDim.z, vec, l, t + N2 * u + N1 * k2, kstride)] = v[u * N2 + k2];
    }
}

// ------------------------------------------------------------------ zadj
// MODE 0: OUT = Sigma_op Q_r^* U.  MODE 1: CG, R -= alpha (Q_r^* U), (r, r) -> beta.
template <int N1, int N2, int W, int MODE, int SL = 0, int RST = 0, int MB = 0>
__global__ void __launch_bounds__(ZCfg<N1, N2, W>::NT, MB ? MB : z_minb(ZCfg<N1, N2, W>::NT))
    k_zadj2(const double2* __restrict__ U, double2* __restrict__ OUT, OpArgs a, int op, CGFuse cg) {
    using C = ZCfg<N1, N2, W>;
    constexpr int NT = C::NT, TE = C::TE;
    extern __shared__ double2 sm[];   // [3][TE]: U0 U1 U2 (r is streamed, not staged)
    __shared__ ColS cs[W];
    __shared__ double2 red[32];
    __shared__ double2 rz_s[N1 * N2], hz_s[N1 * N2];   // z stage roots and e^{i pi k / n3}
    const bool rsz = !(a.zcfg & 256);
    const ModeP& p = a.mp;
    const long long n = a.nloc;
    const int n1 = p.n1;
    const size_t kstride = (size_t)n1 * a.n2loc;
    const long long kglob = (long long)n1 * p.n2;
    const int tid = threadIdx.x;
    const int i0 = blockIdx.x * W, j = blockIdx.y + a.j0, vec = blockIdx.z;
    const size_t col0 = (size_t)i0 + (size_t)n1 * blockIdx.y;
    {
        const double2* u0 = U + col0;
#pragma unroll 2
        for (int q = tid; q < TE; q += NT) {
            const int c = q / W;
            const size_t g = (size_t)(q % W);
            cp_async16(sm + q, u0 + g + u_row<SL>(a, gridDim.z, vec, 0, c, kstride));
            cp_async16(sm + TE + q, u0 + g + u_row<SL>(a, gridDim.z, vec, 1, c, kstride));
            cp_async16(sm + 2 * TE + q, u0 + g + u_row<SL>(a, gridDim.z, vec, 2, c, kstride));
            if (MODE == 1 && RST == 1) {   // residual tile staged with U: every load of the tile in flight at once
                const double2* r0 = OUT + (size_t)vec * a.vsf + col0 + g + kstride * (size_t)c;
                cp_async16(sm + 3 * TE + q, r0);
                cp_async16(sm + 4 * TE + q, r0 + n);
            }
        }
        cp_async_commit();
    }
    if (tid < W) {
        const int i = i0 + tid;
        cs[tid].cm = modes::col(p, i, j);
        cs[tid].base3 = (unsigned long long)((p.cbp * (long long)i + (p.n - p.n1m3) * (long long)j) % p.n);
    }
    if (rsz)
        for (int q = tid; q < N1 * N2; q += NT) {
            rz_s[q] = __ldg(a.pz.root2 + q);
            hz_s[q] = __ldg(a.hroot_z + q);
        }
    double alpha = 0.0;
    if (MODE == 1) {
        if (SL == 0 && cg.alpha_fold) {
            // alpha = (r, r) / (p, M p) from the plane pass's partials, formed by every CTA in the same
            // fixed order (warp 0: lane-strided sums, then a xor butterfly), so all CTAs agree bit for bit;
            // CTA (0, 0, vec) publishes it for the next zfwd2 (x update) and k_cg_xfinal
            if (tid < 32) {
                const int nbx = *cg.nb_x;
                const double* pp = cg.part_x + (size_t)vec * nbx;
                double acc = 0.0;
                for (int t = tid; t < nbx; t += 32) acc += __ldcg(pp + t);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                if (tid == 0) {
                    const double al = (cg.active[vec] && acc > 0.0) ? cg.rr[vec] / acc : 0.0;
                    red[0] = make_double2(al, acc);
                }
            }
        } else {
            alpha = cg.alpha[vec];
        }
    }
    cp_async_wait0();
    __syncthreads();
    if (MODE == 1 && SL == 0 && cg.alpha_fold) {
        alpha = red[0].x;
        if (blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) {
            cg.pmp[vec] = red[0].y;
            cg.alpha[vec] = alpha;
        }
    }
    const int w = tid % W;
    const ColS& c = cs[w];
    const size_t gcol = col0 + w;
    double2* o1 = OUT + (size_t)vec * a.vsf + gcol;
    constexpr int J = (TE + NT - 1) / NT;   // elements per thread in the mode loop
    double2 rb1[RST == 2 ? J : 1], rb2[RST == 2 ? J : 1];
    double2 rn1 = make_double2(0, 0), rn2 = make_double2(0, 0);
    if (MODE == 1 && RST == 0 && tid < TE) {   // first residual element, in flight during the FFT phase
        rn1 = o1[kstride * (tid / W)];
        rn2 = o1[n + kstride * (tid / W)];
    }
    // ---- phase B: conj twiddle, z-DFT (-) of component l over c ----
    {
        const int l = tid / (W * N2), t = (tid / W) % N2;
        double2* ct = sm + (size_t)l * TE;
        const unsigned long long nn = (unsigned long long)p.n, N3 = c.base3;   // e^{2 pi i P / n}: global n
        const double2 wt = conj2(tw_at(a.tw, ((unsigned long long)t * N3) % nn));
        const double2 wu = conj2(tw_at(a.tw, ((unsigned long long)N2 * N3) % nn));
        double2 v[N1];
#pragma unroll
        for (int m = 0; m < N1; ++m) v[m] = ct[(N2 * m + t) * W + w];
        fast::twiddle_natural<N1, N2>(v, wt, wu);
        __syncthreads();
        if (rsz) fast::fft_fwd<N1, N2, -1, fast::XchW<N1, N2, W>, true>(v, t, w, ct, rz_s);
        else fast::fft_fwd<N1, N2, -1, fast::XchW<N1, N2, W>>(v, t, w, ct, a.pz.root2);
#pragma unroll
        for (int u = 0; u < N1 / N2; ++u)
#pragma unroll
            for (int k2 = 0; k2 < N2; ++k2) ct[(t + N2 * u + N1 * k2) * W + w] = v[u * N2 + k2];
    }
    if (MODE == 1 && RST == 2) {   // every residual element of this thread in flight across the barrier
#pragma unroll
        for (int jj = 0; jj < J; ++jj) {
            const int e = tid + jj * NT;
            if (e < TE) {
                rb1[jj] = o1[kstride * (e / W)];
                rb2[jj] = o1[n + kstride * (e / W)];
            }
        }
    }
    __syncthreads();
    // ---- phase A: Pi^* combine, Sigma_op (+ CG residual update) ----
    double rr = 0.0;
    // RST 2: the element loop is unrolled over jj with a compile-time trip count so that rb1 / rb2
    // stay in registers (indexing them by (e - tid) / NT put them on the stack)
    auto elem = [&](const int e, double2 r1, double2 r2) {
        const int k = e / W;
        const double2 l2 = modes::lam3(p, c.cm, rsz ? hz_s[k] : __ldg(a.hroot_z + k));
        Coef o;
        const long long idx = c.cm.idx0 + kglob * k;
        modes::coef(p, c.cm.lam1, c.cm.lam2, l2, idx == p.gamma, MODE ? 1 : op, o);
        const double2 w0 = sm[e], w1 = sm[TE + e], w2 = sm[2 * TE + e];
        double2 z1 = cadd3(cjm(o.num1[0], w0), cjm(o.num1[1], w1), cjm(o.num1[2], w2));
        double2 z2 = cadd3(cmul(o.d[0], w0), cmul(o.d[1], w1), cmul(o.d[2], w2));
        z1 = cscale(z1, o.f1);
        z2 = cscale(z2, o.f2);
        if (MODE == 1) {
            if (RST == 1) {
                r1 = sm[3 * TE + e];
                r2 = sm[4 * TE + e];
            }
            r1 = make_double2(fma(-alpha, z1.x, r1.x), fma(-alpha, z1.y, r1.y));
            r2 = make_double2(fma(-alpha, z2.x, r2.x), fma(-alpha, z2.y, r2.y));
            o1[kstride * k] = r1;
            o1[n + kstride * k] = r2;
            rr += fma(r1.x, r1.x, fma(r1.y, r1.y, fma(r2.x, r2.x, r2.y * r2.y)));
        } else {
            o1[kstride * k] = z1;
            o1[n + kstride * k] = z2;
        }
    };
    if (MODE == 1 && RST == 2) {
#pragma unroll
        for (int jj = 0; jj < J; ++jj)
            if (tid + jj * NT < TE) elem(tid + jj * NT, rb1[jj], rb2[jj]);
    } else {
#pragma unroll 1
        for (int e = tid; e < TE; e += NT) {
            const double2 r1 = rn1, r2 = rn2;
            if (MODE == 1 && RST == 0 && e + NT < TE) {   // next residual element in flight
                rn1 = o1[kstride * ((e + NT) / W)];
                rn2 = o1[n + kstride * ((e + NT) / W)];
            }
            elem(e, r1, r2);
        }
    }
    if (MODE == 1) {
        // per-CTA partial of (r, r); beta is formed by k_cg_finish after this pass
        // partials slab-major [slab][vec][block] (k_cg_finish sums over slabs; all-gather in dist mode)
        const int nb = gridDim.x * gridDim.y;
        cg_block_partial(rr, cg.part_z + ((size_t)a.slab * gridDim.z + vec) * nb + (size_t)blockIdx.y * gridDim.x + blockIdx.x,
                         red);
        if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && tid == 0) *cg.nb_z = nb;
    }
}

// x += alpha p (the CG update deferred by one iteration, k_zfwd2<MODE 1>)
__global__ void k_cg_xfinal(double2* __restrict__ X, const double2* __restrict__ P, const double* __restrict__ alpha,
                            long long N) {
    const int v = blockIdx.y;
    const double al = alpha[v];
    if (al == 0.0) return;
    double2* x = X + (size_t)v * N;
    const double2* pp = P + (size_t)v * N;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < N; t += (long long)gridDim.x * blockDim.x) {
        const double2 q = pp[t];
        const double2 xv = x[t];
        x[t] = make_double2(fma(al, q.x, xv.x), fma(al, q.y, xv.y));
    }
}

template <int N1, int N2, int W>
struct ZLaunch {
    using C = ZCfg<N1, N2, W>;
    static size_t smem_fwd(int mode, int rst) { return (size_t)(mode ? (rst == 1 ? 6 : 4) : 3) * C::TE * sizeof(double2); }
    static size_t smem_adj(int mode, int rst) { return (size_t)(mode && rst == 1 ? 5 : 3) * C::TE * sizeof(double2); }
};

}  // namespace

bool zpass2_supported(const OpArgs& a) {
    if (!a.fast || a.hroot_z == nullptr) return false;
    switch (a.mp.n3) {
        case 64: return a.mp.n1 % 16 == 0;
        case 96: return a.mp.n1 % 8 == 0;
        case 128: return a.mp.n1 % 8 == 0;
        case 192: return a.mp.n1 % 4 == 0;
        case 256: return a.mp.n1 % 4 == 0;
        default: return false;
    }
}

template <int N1, int N2, int W>
static cudaError_t zfwd2_t(const OpArgs& a, const double2* Y, double2* U, int nvec, int op, double2* P, double2* X,
                           const CGFuse* cg, cudaStream_t st) {
    using L = ZLaunch<N1, N2, W>;
    const int mode = cg ? 1 : 0;
    const int rst = !mode ? 0 : (a.zcfg & 8) ? 2 : (a.zcfg & 1) ? 1 : 0;   // x prefetch measured slower: off
    const size_t smem = L::smem_fwd(mode, rst);
    const dim3 g((unsigned)(a.mp.n1 / W), (unsigned)a.n2loc, (unsigned)nvec);
    auto go = [&](auto kern, int opv, double2* Pp, double2* Xp, CGFuse cgv) -> cudaError_t {
        cudaError_t e = allow_smem((const void*)kern, smem);
        if (e != cudaSuccess) return e;
        kern<<<g, L::C::NT, smem, st>>>(Y, U, a, opv, Pp, Xp, cgv);
        return cudaGetLastError();
    };
    const bool sl = a.nslab > 1;
    if constexpr (ZCfg<N1, N2, W>::NT <= 256) {   // zcfg bit 1024: x tile staged, compiled for 2 CTAs per SM
        // (its 6-tile stage admits only 2 per SM anyway; the 3-CTA register cap made ptxas spill)
        if (mode && rst == 1 && !sl && (a.zcfg & 1024)) return go(k_zfwd2<N1, N2, W, 1, 0, 1, 2>, 1, P, X, *cg);
    }
    if (mode && rst == 2) return sl ? go(k_zfwd2<N1, N2, W, 1, 1, 2>, 1, P, X, *cg) : go(k_zfwd2<N1, N2, W, 1, 0, 2>, 1, P, X, *cg);
    if (mode && rst) return sl ? go(k_zfwd2<N1, N2, W, 1, 1, 1>, 1, P, X, *cg) : go(k_zfwd2<N1, N2, W, 1, 0, 1>, 1, P, X, *cg);
    if (mode) return sl ? go(k_zfwd2<N1, N2, W, 1, 1>, 1, P, X, *cg) : go(k_zfwd2<N1, N2, W, 1, 0>, 1, P, X, *cg);
    return sl ? go(k_zfwd2<N1, N2, W, 0, 1>, op, nullptr, nullptr, CGFuse{})
              : go(k_zfwd2<N1, N2, W, 0, 0>, op, nullptr, nullptr, CGFuse{});
}

template <int N1, int N2, int W>
static cudaError_t zadj2_t(const OpArgs& a, const double2* U, double2* OUT, int nvec, int op, const CGFuse* cg,
                           cudaStream_t st) {
    using L = ZLaunch<N1, N2, W>;
    const int mode = cg ? 1 : 0;
    const int rst = !mode ? 0 : (a.zcfg & 4) ? 2 : (a.zcfg & 1) ? 1 : 0;
    const size_t smem = L::smem_adj(mode, rst);
    const dim3 g((unsigned)(a.mp.n1 / W), (unsigned)a.n2loc, (unsigned)nvec);
    auto go = [&](auto kern, int opv, CGFuse cgv) -> cudaError_t {
        cudaError_t e = allow_smem((const void*)kern, smem);
        if (e != cudaSuccess) return e;
        kern<<<g, L::C::NT, smem, st>>>(U, OUT, a, opv, cgv);
        return cudaGetLastError();
    };
    const bool sl = a.nslab > 1;
    if constexpr (ZCfg<N1, N2, W>::NT <= 256) {   // zcfg bit 512: compiled for 4 resident CTAs per SM
        if (mode && rst == 2 && !sl && (a.zcfg & 512)) return go(k_zadj2<N1, N2, W, 1, 0, 2, 4>, 1, *cg);
        if (mode && rst == 2 && !sl && (a.zcfg & 2048)) return go(k_zadj2<N1, N2, W, 1, 0, 2, 2>, 1, *cg);
        if (mode && rst == 1 && !sl && (a.zcfg & 2048)) return go(k_zadj2<N1, N2, W, 1, 0, 1, 2>, 1, *cg);
    }
    if (mode && rst == 2) return sl ? go(k_zadj2<N1, N2, W, 1, 1, 2>, 1, *cg) : go(k_zadj2<N1, N2, W, 1, 0, 2>, 1, *cg);
    if (mode && rst) return sl ? go(k_zadj2<N1, N2, W, 1, 1, 1>, 1, *cg) : go(k_zadj2<N1, N2, W, 1, 0, 1>, 1, *cg);
    if (mode) return sl ? go(k_zadj2<N1, N2, W, 1, 1>, 1, *cg) : go(k_zadj2<N1, N2, W, 1, 0>, 1, *cg);
    return sl ? go(k_zadj2<N1, N2, W, 0, 1>, op, CGFuse{}) : go(k_zadj2<N1, N2, W, 0, 0>, op, CGFuse{});
}

// n3 -> (N1, N2, W)
#define BNF_Z2_PLANS(X) X(64, 8, 8, 16) X(96, 24, 4, 8) X(128, 16, 8, 8) X(192, 24, 8, 4) X(256, 16, 16, 4)
// narrower tiles (zcfg bit 1): more resident CTAs per SM
#define BNF_Z2_HALF(X) X(64, 8, 8, 8) X(128, 16, 8, 4) X(256, 16, 16, 2)

cudaError_t launch_zfwd2(const OpArgs& a, const double2* Y, double2* U, int nvec, int op, double2* P, double2* X,
                         const CGFuse* cg, cudaStream_t st) {
    if (a.zcfg & 2) switch (a.mp.n3) {
#define BNF_CASE(NN, A, B, WW) case NN: if (a.mp.n1 % WW == 0) return zfwd2_t<A, B, WW>(a, Y, U, nvec, op, P, X, cg, st); break;
        BNF_Z2_HALF(BNF_CASE)
#undef BNF_CASE
        default: break;
    }
    switch (a.mp.n3) {
#define BNF_CASE(NN, A, B, WW) case NN: return zfwd2_t<A, B, WW>(a, Y, U, nvec, op, P, X, cg, st);
        BNF_Z2_PLANS(BNF_CASE)
#undef BNF_CASE
        default: return cudaErrorNotSupported;
    }
}

cudaError_t launch_zadj2(const OpArgs& a, const double2* U, double2* OUT, int nvec, int op, const CGFuse* cg,
                         cudaStream_t st) {
    if (a.zcfg & 2) switch (a.mp.n3) {
#define BNF_CASE(NN, A, B, WW) case NN: if (a.mp.n1 % WW == 0) return zadj2_t<A, B, WW>(a, U, OUT, nvec, op, cg, st); break;
        BNF_Z2_HALF(BNF_CASE)
#undef BNF_CASE
        default: break;
    }
    switch (a.mp.n3) {
#define BNF_CASE(NN, A, B, WW) case NN: return zadj2_t<A, B, WW>(a, U, OUT, nvec, op, cg, st);
        BNF_Z2_PLANS(BNF_CASE)
#undef BNF_CASE
        default: return cudaErrorNotSupported;
    }
}

// CTAs per (j, vector) of the plan launch_zfwd2 / launch_zadj2 pick (= n1 / W):
// the zadj CG pass writes (n1 / W) n2loc partials per vector and slab
int zpass2_tiles_x(const OpArgs& a) {
    if (a.zcfg & 2) switch (a.mp.n3) {
#define BNF_CASE(NN, A, B, WW) case NN: if (a.mp.n1 % WW == 0) return a.mp.n1 / WW; break;
        BNF_Z2_HALF(BNF_CASE)
#undef BNF_CASE
        default: break;
    }
    switch (a.mp.n3) {
#define BNF_CASE(NN, A, B, WW) case NN: return a.mp.n1 / WW;
        BNF_Z2_PLANS(BNF_CASE)
#undef BNF_CASE
        default: return 0;
    }
}

cudaError_t launch_cg_xfinal(double2* X, const double2* P, const double* alpha, long long N, int nvec,
                             cudaStream_t st) {
    long long g = (N + 255) / 256;
    if (g > 148 * 4) g = 148 * 4;
    k_cg_xfinal<<<dim3((unsigned)g, nvec), 256, 0, st>>>(X, P, alpha, N);
    return cudaGetLastError();
}

}  // namespace bnf
