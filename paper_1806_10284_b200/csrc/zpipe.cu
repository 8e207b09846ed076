// Persistent, TMA-pipelined adjoint z pass: the same arithmetic
// as k_zadj2 (zpass.cu, Algorithm 1 step 3 of
// PAPER.md §5.3):
//
//   per column tile (W consecutive i, one j, all z-planes c, one vector):
//     conj twiddle e^{-2 pi i c N3(i,j)/n}, z-DFT c -> k (-) of the 3
//     components of U, Pi^* combine (3 -> 2), Sigma_op
//     [CG: r -= alpha (M p), per-tile (r, r) partial]
//
// k_zadj2 runs one tile per CTA lifetime (load -> FFT -> combine -> store),
// so a CTA's U tile is only in flight during its load phase; ncu shows the
// pass latency-bound (DRAM 40 %, long-scoreboard 34 % of the stall samples).
// Here each CTA stays resident and walks tiles t = blockIdx.x, + gridDim.x, ...
// through a ring of NB shared-memory buffers:
//   * one thread issues the Tensor Memory Accelerator copy of a whole U tile
//     (one 4-D box {W complex, 1 row, n3 planes, 3 components} = 48 KB)
//     into buffer t % NB, completing on mbarrier full[b];
//   * warp group F (3 W N2 threads) waits full[b], runs the conj twiddle and
//     the 3 register z-DFTs in place in the buffer (group-local named barrier)
//     and arrives on mbarrier fft[b];
//   * warp group C (as many threads) first issues its loads of the tile's
//     residual r into registers, then waits fft[b], forms the Pi^* combine
//     and r -= alpha z, stores r, reduces (r, r) for the tile, and once all
//     of C is done with buffer b its thread 0 issues the copy of tile t + NB
//     into b.
// So the next tiles' HBM traffic overlaps this tile's FP64 work inside one
// CTA, and F of tile t + 1 overlaps C of tile t.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "cgfuse.cuh"
#include "fastfft.cuh"
#include "kernels.cuh"
#include "modes.cuh"

namespace bnf {
namespace {

using fast::cmul;
using fast::cscale;
using modes::Coef;
using modes::Col;

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mb_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void mb_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(su32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load4(void* dst, const CUtensorMap* map, int x, int y, int z, int w,
                                          unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
        "[%6];\n" ::"r"(su32(dst)),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(x), "r"(y), "r"(z), "r"(w), "r"(su32(bar))
        : "memory");
}
// barrier of one warp group (named barrier id, nthreads threads)
__device__ __forceinline__ void group_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

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

// fastfft fft_fwd (natural -> stage-2 layout, exchange in the W-fast tile) with
// the CTA barriers replaced by the F group's named barrier
template <int N1, int N2, int S, int W>
__device__ __forceinline__ void fft_fwd_g(double2 (&v)[N1], int t, int w, double2* xch, const double2* root, int nt) {
    using X = fast::XchW<N1, N2, W>;
    fast::DFT<N1, S>::run(v);
    if (t > 0) {
#pragma unroll
        for (int k1 = 1; k1 < N1; ++k1) v[k1] = cmul(v[k1], fast::root_tw<S>(root, k1 * N2 + t));
    }
#pragma unroll
    for (int k1 = 0; k1 < N1; ++k1) xch[X::idx(k1, t, w)] = v[k1];
    group_sync(1, nt);
    constexpr int U = N1 / N2;
#pragma unroll
    for (int u = 0; u < U; ++u) {
        double2 a[N2];
        const int k1 = t + N2 * u;
#pragma unroll
        for (int tt = 0; tt < N2; ++tt) a[tt] = xch[X::idx(k1, tt, w)];
        fast::DFT<N2, S>::run(a);
#pragma unroll
        for (int k2 = 0; k2 < N2; ++k2) v[u * N2 + k2] = a[k2];
    }
    group_sync(1, nt);
}

struct ColS3 {   // per-column constants of a tile (computed by F, read by C)
    Col cm;
    unsigned long long base3;
};

template <int N1, int N2, int W, int NB, int CM = 1>
struct Z3Cfg {
    static constexpr int N = N1 * N2;
    static constexpr int NG = 3 * W * N2;        // threads of group F
    static constexpr int NGC = CM * NG;          // threads of group C
    static constexpr int NT = NG + NGC;
    static constexpr int TE = N * W;             // complex elements per component tile
    static constexpr int J = (TE + NGC - 1) / NGC; // elements per C thread
    static constexpr size_t BUF = (size_t)3 * TE * 16;
    static constexpr size_t off_cs = (size_t)NB * BUF;
    static constexpr size_t off_bar = off_cs + (size_t)NB * W * sizeof(ColS3);
    static constexpr size_t off_red = (off_bar + (size_t)3 * NB * 8 + 15) & ~(size_t)15;
    static constexpr size_t smem = off_red + 32 * 16 + 128;   // + alignment slack
};


template <int N1, int N2, int W, int NB, int MODE, int LD, int CM>
__global__ void __launch_bounds__(Z3Cfg<N1, N2, W, NB, CM>::NT, 1)
    k_zadj3(const __grid_constant__ CUtensorMap tmU, const double2* __restrict__ U, double2* __restrict__ OUT, OpArgs a,
            int op, CGFuse cg, int ntx, int ntiles) {
    using C = Z3Cfg<N1, N2, W, NB, CM>;
    constexpr int NG = C::NG, NGC = C::NGC, TE = C::TE, J = C::J;
    extern __shared__ __align__(128) unsigned char sm[];
    double2* buf0 = reinterpret_cast<double2*>(sm);
    ColS3* cs0 = reinterpret_cast<ColS3*>(sm + C::off_cs);
    unsigned long long* full = reinterpret_cast<unsigned long long*>(sm + C::off_bar);
    unsigned long long* fftd = full + NB;
    double2* red = reinterpret_cast<double2*>(sm + C::off_red);
    const ModeP& p = a.mp;
    const long long n = a.nloc;
    const size_t kstride = (size_t)p.n1 * a.n2loc;
    const long long kglob = (long long)p.n1 * p.n2;
    const int tid = threadIdx.x;
    const int per_vec = ntx * a.n2loc;
    auto tile_xyz = [&](int t, int& bx, int& by, int& vec) {
        vec = t / per_vec;
        const int r = t - vec * per_vec;
        by = r / ntx;
        bx = r - by * ntx;
    };
    auto issue = [&](int t, int b) {   // LD 0: one thread, TMA copy of tile t into buffer b
        int bx, by, vec;
        tile_xyz(t, bx, by, vec);
        mb_expect_tx(&full[b], (unsigned)C::BUF);
        tma_load4(buf0 + (size_t)b * 3 * TE, &tmU, 2 * W * bx, by, 0, 3 * vec, &full[b]);
    };
    auto issue_cp = [&](int t, int b, int tc) {   // LD 1: the C group, cp.async (16 B per thread and copy)
        int bx, by, vec;
        tile_xyz(t, bx, by, vec);
        const double2* u0 = U + (size_t)vec * 3 * n + (size_t)bx * W + (size_t)p.n1 * by;
        double2* d = buf0 + (size_t)b * 3 * TE;
#pragma unroll 2
        for (int qq = tc; qq < TE; qq += NGC) {
            const size_t g = (size_t)(qq % W) + kstride * (size_t)(qq / W);
            const unsigned s0 = su32(d + qq);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s0), "l"(u0 + g) : "memory");
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s0 + 16u * TE), "l"(u0 + n + g) : "memory");
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s0 + 32u * TE), "l"(u0 + 2 * n + g) : "memory");
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(su32(&full[b])) : "memory");
    };
    if (tid == 0) {
        for (int b = 0; b < NB; ++b) {
            mb_init(&full[b], LD ? NGC : 1);
            mb_init(&fftd[b], NG);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (LD == 0 && tid == 0)
        for (int b = 0; b < NB; ++b)
            if ((int)blockIdx.x + b * (int)gridDim.x < ntiles) issue(blockIdx.x + b * gridDim.x, b);
    if (LD == 1 && tid >= NG)
        for (int b = 0; b < NB; ++b)
            if ((int)blockIdx.x + b * (int)gridDim.x < ntiles) issue_cp(blockIdx.x + b * gridDim.x, b, tid - NG);

    if (tid < NG) {
        // ================= group F: conj twiddle + z-DFT (-) of the 3 components, in place
        const int l = tid / (W * N2), t = (tid / W) % N2, w = tid % W;
        int q = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++q) {
            const int b = q % NB;
            int bx, by, vec;
            tile_xyz(tile, bx, by, vec);
            const int j = by + a.j0;
            ColS3* cs = cs0 + b * W;
            ColS3 mine;
            if (tid < W) {   // computed before the wait; stored after it (C of tile q - NB may still read slot b)
                const int i = bx * W + tid;
                mine.cm = modes::col(p, i, j);
                mine.base3 = (unsigned long long)((p.cbp * (long long)i + (p.n - p.n1m3) * (long long)j) % p.n);
            }
            mb_wait(&full[b], (unsigned)((q / NB) & 1));
            if (tid < W) cs[tid] = mine;
            group_sync(1, NG);
            double2* ct = buf0 + (size_t)b * 3 * TE + (size_t)l * TE;
            const unsigned long long nn = (unsigned long long)p.n, N3 = cs[w].base3;
            const double2 wt = conj2(tw_at(a.tw, ((unsigned long long)t * N3) % nn));
            const double2 wu = conj2(tw_at(a.tw, ((unsigned long long)N2 * N3) % nn));
            double2 v[N1];
#pragma unroll
            for (int m = 0; m < N1; ++m) v[m] = ct[(N2 * m + t) * W + w];
            fast::twiddle_natural<N1, N2>(v, wt, wu);
            group_sync(1, NG);
            fft_fwd_g<N1, N2, -1, W>(v, t, w, ct, a.pz.root2, NG);
#pragma unroll
            for (int u = 0; u < N1 / N2; ++u)
#pragma unroll
                for (int k2 = 0; k2 < N2; ++k2) ct[(t + N2 * u + N1 * k2) * W + w] = v[u * N2 + k2];
            mb_arrive(&fftd[b]);   // release: this thread's buffer writes (and cs) are visible to C
        }
    } else {
        // ================= group C: Pi^* combine, Sigma_op (+ r -= alpha z, (r, r))
        const int tc = tid - NG;
        const int w = tc % W;
        int q = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++q) {
            const int b = q % NB;
            int bx, by, vec;
            tile_xyz(tile, bx, by, vec);
            const size_t gcol = (size_t)bx * W + (size_t)p.n1 * by + w;
            double2* o1 = OUT + (size_t)vec * a.vsf + gcol;
            double2 rb1[MODE ? J : 1], rb2[MODE ? J : 1];
            if (MODE == 1) {   // the tile's residual, in flight while F transforms it
#pragma unroll
                for (int jj = 0; jj < J; ++jj) {
                    const int e = tc + jj * NGC;
                    if (e < TE) {
                        rb1[jj] = o1[kstride * (e / W)];
                        rb2[jj] = o1[n + kstride * (e / W)];
                    }
                }
            }
            const double alpha = MODE == 1 ? cg.alpha[vec] : 0.0;
            mb_wait(&fftd[b], (unsigned)((q / NB) & 1));
            const double2* bt = buf0 + (size_t)b * 3 * TE;
            const ColS3& c = cs0[b * W + w];
            double rr = 0.0;
#pragma unroll
            for (int jj = 0; jj < J; ++jj) {
                const int e = tc + jj * NGC;
                if (e < TE) {
                    const int k = e / W;
                    const double2 l2 = modes::lam3(p, c.cm, __ldg(a.hroot_z + k));
                    Coef o;
                    const long long idx = c.cm.idx0 + kglob * k;
                    modes::coef(p, c.cm.lam1, c.cm.lam2, l2, idx == p.gamma, MODE ? 1 : op, o);
                    const double2 w0 = bt[e], w1 = bt[TE + e], w2 = bt[2 * TE + e];
                    double2 z1 = cadd3(cjm(o.num1[0], w0), cjm(o.num1[1], w1), cjm(o.num1[2], w2));
                    double2 z2 = cadd3(cmul(o.d[0], w0), cmul(o.d[1], w1), cmul(o.d[2], w2));
                    z1 = cscale(z1, o.f1);
                    z2 = cscale(z2, o.f2);
                    if (MODE == 1) {
                        const double2 r1 = make_double2(fma(-alpha, z1.x, rb1[jj].x), fma(-alpha, z1.y, rb1[jj].y));
                        const double2 r2 = make_double2(fma(-alpha, z2.x, rb2[jj].x), fma(-alpha, z2.y, rb2[jj].y));
                        o1[kstride * k] = r1;
                        o1[n + kstride * k] = r2;
                        rr += fma(r1.x, r1.x, fma(r1.y, r1.y, fma(r2.x, r2.x, r2.y * r2.y)));
                    } else {
                        o1[kstride * k] = z1;
                        o1[n + kstride * k] = z2;
                    }
                }
            }
            if (MODE == 1) {   // the tile's (r, r) partial, fixed order (warp sums, then the group's warps)
                double2 s = warp_sum(make_double2(rr, 0.0));
                const int wg = tc >> 5, ln = tc & 31;
                if (ln == 0) red[wg] = s;
            }
            group_sync(2, NGC);   // every C thread is done with buffer b (and red is complete)
            if (tile + NB * (int)gridDim.x < ntiles) {
                if (LD == 0 && tc == 0) issue(tile + NB * gridDim.x, b);
                if (LD == 1) issue_cp(tile + NB * gridDim.x, b, tc);
            }
            if (MODE == 1 && tc < 32) {   // same order as block_sum (cgfuse.cuh): k_zadj2's partials bit for bit
                double2 s = tc < NGC / 32 ? red[tc] : make_double2(0.0, 0.0);
                s = warp_sum(s);
                if (tc == 0) {
                    const int nb = per_vec;
                    cg.part_z[((size_t)a.slab * (ntiles / per_vec) + vec) * nb + (size_t)by * ntx + bx] = s.x;
                    if (tile == 0) *cg.nb_z = nb;
                }
            }
            if (MODE == 1) group_sync(2, NGC);   // red is reused by the next tile
        }
    }
}

}  // namespace

// TMA map of the real-space U buffer for k_zadj3: [slab-components][n3][n2][2 n1 doubles],
// box {2W doubles, 1, n3, 3} = one tile of all three components of one vector.
int zadj3_encode(const OpArgs& a, void* base, long long comp_slabs, void* encode_fn, CUtensorMap* m) {
    int W = 0;
    switch (a.mp.n3) {
        case 128: W = 8; break;
        case 256: W = 4; break;
        default: return 1;
    }
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(encode_fn);
    const cuuint64_t dims[4] = {(cuuint64_t)(2 * a.mp.n1), (cuuint64_t)a.mp.n2, (cuuint64_t)a.mp.n3,
                                (cuuint64_t)comp_slabs};
    const cuuint64_t strides[3] = {(cuuint64_t)a.mp.n1 * 16, (cuuint64_t)a.mp.n1 * a.mp.n2 * 16,
                                   (cuuint64_t)a.mp.n * 16};
    const cuuint32_t box[4] = {(cuuint32_t)(2 * W), 1, (cuuint32_t)a.mp.n3, 3};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : 1;
}

bool zadj3_supported(const OpArgs& a) {
    return a.fast && a.nslab == 1 && a.hroot_z != nullptr &&
           ((a.mp.n3 == 128 && a.mp.n1 % 8 == 0) || (a.mp.n3 == 256 && a.mp.n1 % 4 == 0));
}

// tiles per (j, vector) row of the plan launch_zadj3 uses (= n1 / W; the CG partial layout)
int zadj3_tiles_x(const OpArgs& a) { return a.mp.n3 == 128 ? a.mp.n1 / 8 : a.mp.n1 / 4; }

template <int N1, int N2, int W, int LD, int CM>
static cudaError_t zadj3_t(const OpArgs& a, const CUtensorMap& tm, const double2* U, double2* OUT, int nvec, int op,
                           const CGFuse* cg, cudaStream_t st, int nb_ring, int ctas_per_sm) {
    const int ntx = a.mp.n1 / W;
    const int ntiles = ntx * a.n2loc * nvec;
    static int nsm = 0;
    if (nsm == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    }
    const int grid = std::min(ntiles, nsm * ctas_per_sm);
    auto go = [&](auto kern, size_t smem, int nt, int opv, CGFuse cgv) -> cudaError_t {
        cudaError_t e = allow_smem((const void*)kern, smem);
        if (e != cudaSuccess) return e;
        kern<<<grid, nt, smem, st>>>(tm, U, OUT, a, opv, cgv, ntx, ntiles);
        return cudaGetLastError();
    };
    if (nb_ring == 2) {
        using C = Z3Cfg<N1, N2, W, 2, CM>;
        if (cg) return go(k_zadj3<N1, N2, W, 2, 1, LD, CM>, C::smem, C::NT, 1, *cg);
        return go(k_zadj3<N1, N2, W, 2, 0, LD, CM>, C::smem, C::NT, op, CGFuse{});
    }
    using C = Z3Cfg<N1, N2, W, 3, CM>;
    if (cg) return go(k_zadj3<N1, N2, W, 3, 1, LD, CM>, C::smem, C::NT, 1, *cg);
    return go(k_zadj3<N1, N2, W, 3, 0, LD, CM>, C::smem, C::NT, op, CGFuse{});
}

// zcfg bit 5: 2-buffer ring (default 3), one CTA per SM; bit 6: tiles copied by the TMA (default:
// cp.async issued by the C group, arriving on the buffer's mbarrier); bit 7: group C twice as wide as F
cudaError_t launch_zadj3(const OpArgs& a, const CUtensorMap& tm, const double2* U, double2* OUT, int nvec, int op,
                         const CGFuse* cg, cudaStream_t st) {
    const int nb = (a.zcfg & 32) ? 2 : 3, cps = 1;
    const bool tma = (a.zcfg & 64) != 0, c2 = (a.zcfg & 128) != 0;
    switch (a.mp.n3) {
        case 128: return tma ? zadj3_t<16, 8, 8, 0, 1>(a, tm, U, OUT, nvec, op, cg, st, nb, cps)
                      : c2 ? zadj3_t<16, 8, 8, 1, 2>(a, tm, U, OUT, nvec, op, cg, st, nb, cps)
                           : zadj3_t<16, 8, 8, 1, 1>(a, tm, U, OUT, nvec, op, cg, st, nb, cps);
        case 256: return tma ? zadj3_t<16, 16, 4, 0, 1>(a, tm, U, OUT, nvec, op, cg, st, nb, cps)
                      : c2 ? zadj3_t<16, 16, 4, 1, 2>(a, tm, U, OUT, nvec, op, cg, st, nb, cps)
                           : zadj3_t<16, 16, 4, 1, 1>(a, tm, U, OUT, nvec, op, cg, st, nb, cps);
        default: return cudaErrorNotSupported;
    }
}

}  // namespace bnf
