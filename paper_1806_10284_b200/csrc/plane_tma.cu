// TMA-staged real-space plane pass ("plane_t") -- the same
// arithmetic as k_plane_l2 (Algorithms 1-2 of
// PAPER.md §5.3):
//
//   per (component l, z-plane c):  y-DFT (+), twiddle e^{-2 pi i b m1 i/(n1 n2)},
//   x-DFT (+), * 1/(n eps) [+ (p, M p)], x-DFT (-), conj twiddle, y-DFT (-)
//
// but every strip of the plane moves between L2/HBM and shared memory with
// the Tensor Memory Accelerator (cp.async.bulk.tensor, 128-byte swizzle), two
// strip buffers per CTA so that the next strip is in flight while the current
// one is transformed, and the FFT stage exchange happens in place inside the
// strip buffer.  No per-element global loads or stores are issued by the
// threads (the L1/LSU path was the bottleneck of the LDG/STG variant).
//
// Strip = 16 sequences (16 columns for the y phases, 16 rows for the x
// phase); thread (w = tid % 16, t = tid / 16) holds elements N2 m + t of
// sequence w.  Shared-memory image of a strip, in complex (16-byte) units:
//   y phases: boxes of 8 columns x N rows:  (col / 8) 8N + row 8 + ((col % 8) ^ (row % 8))
//   x phase : boxes of 8 columns x 16 rows: (col / 8) 128 + row 8 + ((col % 8) ^ (row % 8))
// (the TMA 128-byte swizzle), which makes every access pattern below free of
// bank conflicts.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include "cgfuse.cuh"
#include "fastfft.cuh"
#include "kernels.cuh"

namespace bnf {
namespace {

using fast::cmul;
using fast::cscale;

__device__ __forceinline__ double2 tw_at_t(const TwP& t, unsigned long long P) {  // e^{2 pi i P / n}
    return cmul(__ldg(t.hi + (P >> t.shift)), __ldg(t.lo + (P & t.mask)));
}
__device__ __forceinline__ double2 conj2t(double2 a) { return make_double2(a.x, -a.y); }

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load3(void* dst, const CUtensorMap* map, int x, int y, int z, unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_store3(const CUtensorMap* map, int x, int y, int z, const void* src) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(
                     reinterpret_cast<unsigned long long>(map)),
                 "r"(x), "r"(y), "r"(z), "r"(smem_u32(src))
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void fence_async_global() { asm volatile("fence.proxy.async.global;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async16t(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}

// strip layouts (complex units): element idx of sequence w
template <int N>
struct LayY {   // sequences = columns, idx = row
    static __device__ __forceinline__ int at(int w, int idx) { return (w >> 3) * (8 * N) + idx * 8 + ((w & 7) ^ (idx & 7)); }
};
struct LayX {   // sequences = rows, idx = column
    static __device__ __forceinline__ int at(int w, int idx) { return (idx >> 3) * 128 + w * 8 + ((idx & 7) ^ (w & 7)); }
};

// Natural -> stage-2 layout (as fastfft fft_fwd) with the exchange in place
// in the strip buffer: thread (w, t) holds x[N2 m + t] on entry; on exit
// v[u N2 + k2] = X[k1 + N1 k2], k1 = t + N2 u.  The stage-1 values are
// written to the thread's own input positions.  NT threads, block barriers.
template <int N1, int N2, int S, class L>
__device__ __forceinline__ void fft_fwd_ip(double2 (&v)[N1], int t, int w, double2* buf, const double2* root) {
    fast::DFT<N1, S>::run(v);
    if (t > 0) {
#pragma unroll
        for (int k1 = 1; k1 < N1; ++k1) {
            const double2 r = root[k1 * N2 + t];
            v[k1] = cmul(v[k1], S > 0 ? r : conj2t(r));
        }
    }
#pragma unroll
    for (int k1 = 0; k1 < N1; ++k1) buf[L::at(w, k1 * N2 + t)] = v[k1];
    __syncthreads();
#pragma unroll
    for (int u = 0; u < N1 / N2; ++u) {
        double2 a[N2];
        const int k1 = t + N2 * u;
#pragma unroll
        for (int tt = 0; tt < N2; ++tt) a[tt] = buf[L::at(w, k1 * N2 + tt)];
        fast::DFT<N2, S>::run(a);
#pragma unroll
        for (int k2 = 0; k2 < N2; ++k2) v[u * N2 + k2] = a[k2];
    }
    __syncthreads();
}

// Stage-2 -> natural layout (as fastfft fft_mirror), exchange in place.
template <int N1, int N2, int S, class L>
__device__ __forceinline__ void fft_mirror_ip(double2 (&v)[N1], int t, int w, double2* buf, const double2* root) {
#pragma unroll
    for (int u = 0; u < N1 / N2; ++u) {
        double2 a[N2];
#pragma unroll
        for (int k2 = 0; k2 < N2; ++k2) a[k2] = v[u * N2 + k2];
        fast::DFT<N2, S>::run(a);
        const int k1 = t + N2 * u;
#pragma unroll
        for (int tt = 0; tt < N2; ++tt) buf[L::at(w, k1 * N2 + tt)] = a[tt];
    }
    __syncthreads();
#pragma unroll
    for (int k1 = 0; k1 < N1; ++k1) v[k1] = buf[L::at(w, k1 * N2 + t)];
    if (t > 0) {
#pragma unroll
        for (int k1 = 1; k1 < N1; ++k1) {
            const double2 r = root[k1 * N2 + t];
            v[k1] = cmul(v[k1], S > 0 ? r : conj2t(r));
        }
    }
    fast::DFT<N1, S>::run(v);
}

template <int N1, int N2, int XS = 0, int PR = 1>
struct PlaneTCfg {
    static constexpr int N = N1 * N2;
    static constexpr int S = 16;                 // sequences per strip
    static constexpr int P = N / S;              // strips per phase
    static constexpr int NT = S * N2;            // threads
    static constexpr int SE = S * N;             // complex elements per strip buffer
    static constexpr bool EPF = N <= 128 && !XS;  // whole-plane eps index prefetch (XS: 3 CTAs / SM instead)
    static constexpr bool EST = PR == 2;          // per-strip eps index prefetch (two strip buffers of S N bytes)
    // dynamic smem: 2 strip buffers (1024-aligned), roots (y, x; PR 2: one table, n1 == n2), lut, eps, barriers
    static constexpr size_t off_root = (size_t)2 * SE * 16;
    static constexpr size_t off_lut = off_root + (size_t)(PR == 2 ? 1 : 2) * N * 16;
    static constexpr size_t off_eps = off_lut + 256 * 8;
    static constexpr size_t off_bar = off_eps + (EPF ? (size_t)N * N : EST ? (size_t)2 * S * N : 0);
    static constexpr size_t smem = off_bar + 64 + 1024;   // + alignment slack
};
template <int K>
__device__ __forceinline__ void bulk_wait_k() { asm volatile("cp.async.bulk.wait_group %0;\n" ::"n"(K) : "memory"); }

// XS = 0: sequence w = tid % 16 with its N2 threads in different warps, the FFT
// stage exchange in place in the strip buffer (block barriers); XS = 1: the N2
// threads of a sequence are consecutive lanes of one warp and the exchange is
// an xor-shuffle transpose (fastfft warp_xpose): shared memory then only
// carries the strip staging, and the strip needs no barrier until its store.
// PR = 2 (XS = 1 only): each CTA transforms two planes c and c + n3 / 2 of one
// component, phase by phase interleaved (y of A, y of B, x of A, x of B, y^-1 of
// A, y^-1 of B), so that the first strip of a phase -- which reads what the
// plane's previous phase stored -- is prefetched while the other plane's phase
// runs instead of after a full store drain; the eps indices of the next x strip
// are copied to shared memory one strip ahead (cp.async).
template <int N1, int N2, int CG, int XS, int PR = 1>
__global__ void __launch_bounds__(PlaneTCfg<N1, N2, XS>::NT, PlaneTCfg<N1, N2, XS>::NT <= 128 ? (XS ? 3 : 2) : 1)
    k_plane_t(OpArgs a, CGFuse cgf, const __grid_constant__ CUtensorMap my, const __grid_constant__ CUtensorMap mx,
              int zbase) {
    using C = PlaneTCfg<N1, N2, XS, PR>;
    constexpr int N = C::N, S = C::S, P = C::P, NT = C::NT, SE = C::SE;
    static_assert(PR == 1 || XS == 1, "paired planes: warp-shuffle exchange only");
    extern __shared__ unsigned char smraw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<size_t>(smraw) + 1023) & ~(size_t)1023);
    double2* buf = reinterpret_cast<double2*>(sm);
    double2* ry = reinterpret_cast<double2*>(sm + C::off_root);
    double2* rx = PR == 2 ? ry : ry + N;
    double* lut_s = reinterpret_cast<double*>(sm + C::off_lut);
    unsigned char* eps_s = sm + C::off_eps;
    unsigned long long* full = reinterpret_cast<unsigned long long*>(sm + C::off_bar);
    const ModeP& p = a.mp;
    const int tid = threadIdx.x;
    const int w = XS ? (tid / 32) * (32 / N2) + (tid % 32) / N2 : tid % S;
    const int t = XS ? tid % N2 : tid / S;
    const int c0 = blockIdx.x;
    const int vl = blockIdx.y + a.comp0;
    const int l = vl % 3;
    const int zb = zbase + vl * p.n3;               // plane index base in the tensor maps
    const int cstep = p.n3 / PR;                     // PR 2: planes c0 and c0 + n3 / 2
    const bool epf = C::EPF && a.eps_idx != nullptr;
    const bool est = C::EST && a.eps_idx != nullptr;
    constexpr int G = 3 * P * PR;                    // strips per CTA
    if (tid == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        fence_async_smem();
    }
    for (int q = tid; q < N; q += NT) {
        ry[q] = __ldg(a.py.root2 + q);
        if (PR == 1) rx[q] = __ldg(a.px.root2 + q);
    }
    if (a.eps_idx != nullptr)
        for (int q = tid; q < 256; q += NT) lut_s[q] = __ldg(a.eps_lut + q);
    if (epf) {
        const unsigned char* src = a.eps_idx + (size_t)l * p.n + (size_t)N * N * c0;
        for (int q = tid; q < N * N / 16; q += NT) cp_async16t(eps_s + 16 * q, src + 16 * q);
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
    __syncthreads();
    // strip g: segment g / P = (phase, plane) = (seg / PR, seg % PR), strip r = g % P, buffer g % 2
    auto plane_of = [&](int g) { return (g / P) % PR; };
    auto phase_of = [&](int g) { return (g / P) / PR; };
    auto load = [&](int g) {
        double2* b = buf + (g & 1) * SE;
        const int ph = phase_of(g), r = g % P, z = zb + c0 + cstep * plane_of(g);
        mbar_expect_tx(&full[g & 1], (unsigned)(SE * 16));
        if (ph != 1) {   // column strip: 2 boxes of 8 columns x N rows
#pragma unroll
            for (int q = 0; q < S / 8; ++q) tma_load3(b + q * 8 * N, &my, (r * S + q * 8) * 2, 0, z, &full[g & 1]);
        } else {         // row strip: N / 8 boxes of 8 columns x 16 rows
#pragma unroll 4
            for (int q = 0; q < N / 8; ++q) tma_load3(b + q * 128, &mx, q * 16, r * S, z, &full[g & 1]);
        }
    };
    auto store = [&](int g) {
        const double2* b = buf + (g & 1) * SE;
        const int ph = phase_of(g), r = g % P, z = zb + c0 + cstep * plane_of(g);
        if (ph != 1) {
#pragma unroll
            for (int q = 0; q < S / 8; ++q) tma_store3(&my, (r * S + q * 8) * 2, 0, z, b + q * 8 * N);
        } else {
#pragma unroll 4
            for (int q = 0; q < N / 8; ++q) tma_store3(&mx, q * 16, r * S, z, b + q * 128);
        }
        bulk_commit();
    };
    // PR 2: eps indices of x strip g (S rows of N bytes) into eps buffer g % 2, every thread a share
    auto eps_copy = [&](int g) {
        const int r = g % P, cc = c0 + cstep * plane_of(g);
        const unsigned char* src = a.eps_idx + (size_t)l * p.n + (size_t)N * ((size_t)r * S + (size_t)N * cc);
        unsigned char* dst = eps_s + (g & 1) * (S * N);
        for (int q = tid; q < S * N / 16; q += NT) cp_async16t(dst + 16 * q, src + 16 * q);
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    if (tid == 0) load(0);
    static_assert(!XS || 32 % N2 == 0, "warp-local exchange: N2 divides 32");
    const unsigned n12 = (unsigned)p.n12;
    const unsigned long long s3 = (unsigned long long)p.n3;
    double pmp = 0.0;
    double2 v[N1];
#pragma unroll 1
    for (int g = 0; g < G; ++g) {
        const int ph = phase_of(g), r = g % P;
        const int c = c0 + cstep * plane_of(g);
        if (PR == 1) {
            // prefetch the next strip of the same phase (its buffer's last store must have read smem)
            if (tid == 0 && g + 1 < G && (g + 1) % P != 0) {
                bulk_wait_read0();
                load(g + 1);
            }
        } else if (g + 1 < G) {
            if (tid == 0) {
                bulk_wait_read0();   // buffer (g + 1) % 2: the store of strip g - 1 has read it
                if ((g + 1) % P == 0 && phase_of(g + 1) > 0) {
                    // first strip of a plane's next phase: that plane's previous phase was stored before
                    // the P - 1 strips of the other plane committed since -- those may stay in flight
                    bulk_wait_k<P - 1>();
                    fence_async_global();
                }
                load(g + 1);
            }
            if (est && phase_of(g + 1) == 1) eps_copy(g + 1);
        }
        mbar_wait(&full[g & 1], (unsigned)((g >> 1) & 1));
        double2* b = buf + (g & 1) * SE;
        if (ph == 0) {   // ---------------- y-DFT (+), twiddle ----------------
            const int i = r * S + w;
            const unsigned M = ((unsigned)p.m1 * (unsigned)i) % n12;
#pragma unroll
            for (int m = 0; m < N1; ++m) v[m] = b[LayY<N>::at(w, N2 * m + t)];
            if constexpr (XS) {
                fast::fft_fwd_w<N1, N2, 1, 1>(v, t, w, nullptr, ry);
                __syncwarp();   // the sequence's lanes have read their inputs before the outputs overwrite them
            } else {
                fft_fwd_ip<N1, N2, 1, LayY<N>>(v, t, w, b, ry);
            }
            const double2 wt = conj2t(tw_at_t(a.tw, (unsigned long long)(((unsigned)t * M) % n12) * s3));
            const double2 wu = conj2t(tw_at_t(a.tw, (unsigned long long)(((unsigned)N2 * M) % n12) * s3));
            const double2 wk = conj2t(tw_at_t(a.tw, (unsigned long long)(((unsigned)N1 * M) % n12) * s3));
            fast::twiddle_stage2<N1, N2>(v, wt, wu, wk);
#pragma unroll
            for (int u = 0; u < N1 / N2; ++u)
#pragma unroll
                for (int k2 = 0; k2 < N2; ++k2) b[LayY<N>::at(w, t + N2 * u + N1 * k2)] = v[u * N2 + k2];
        } else if (ph == 1) {   // ---------------- x-DFT (+), B^{-1}, x-DFT (-) ----------------
            if (epf && r == 0) asm volatile("cp.async.wait_group 0;\n" ::: "memory");
            if (epf && r == 0) __syncthreads();
            const int brow = r * S + w;
#pragma unroll
            for (int m = 0; m < N1; ++m) v[m] = b[LayX::at(w, N2 * m + t)];
            if constexpr (XS) fast::fft_fwd_w<N1, N2, 1, 1>(v, t, w, nullptr, rx);
            else fft_fwd_ip<N1, N2, 1, LayX>(v, t, w, b, rx);
            const size_t rowofs = (size_t)l * p.n + (size_t)N * ((size_t)brow + (size_t)N * c);
            auto scale = [&](auto eps_at) {
#pragma unroll
                for (int u = 0; u < N1 / N2; ++u)
#pragma unroll
                    for (int k2 = 0; k2 < N2; ++k2) {
                        const int aa = t + N2 * u + N1 * k2;
                        const double s_ = a.inv_n * eps_at(aa);
                        const double2 x = v[u * N2 + k2];
                        if (CG) pmp += s_ * (x.x * x.x + x.y * x.y);   // (p, M p) = sum |T v|^2 / (n eps)
                        v[u * N2 + k2] = cscale(x, s_);
                    }
            };
            if (est) {
                const unsigned char* e = eps_s + (g & 1) * (S * N) + w * N;
                scale([&](int aa) { return lut_s[e[aa]]; });
            } else if (epf) scale([&](int aa) { return lut_s[eps_s[brow * N + aa]]; });
            else if (a.eps_idx) scale([&](int aa) { return lut_s[__ldg(a.eps_idx + rowofs + aa)]; });
            else scale([&](int aa) { return __ldg(a.eps_inv + rowofs + aa); });
            if constexpr (XS) fast::fft_mirror_w<N1, N2, -1, 1>(v, t, w, nullptr, rx);
            else fft_mirror_ip<N1, N2, -1, LayX>(v, t, w, b, rx);
#pragma unroll
            for (int m = 0; m < N1; ++m) b[LayX::at(w, N2 * m + t)] = v[m];
        } else {   // ---------------- conj twiddle, y-DFT (-) ----------------
            const int i = r * S + w;
            const unsigned M = ((unsigned)p.m1 * (unsigned)i) % n12;
#pragma unroll
            for (int m = 0; m < N1; ++m) v[m] = b[LayY<N>::at(w, N2 * m + t)];
            const double2 wt = tw_at_t(a.tw, (unsigned long long)(((unsigned)t * M) % n12) * s3);
            const double2 wu = tw_at_t(a.tw, (unsigned long long)(((unsigned)N2 * M) % n12) * s3);
            fast::twiddle_natural<N1, N2>(v, wt, wu);
            if constexpr (XS) {
                fast::fft_fwd_w<N1, N2, -1, 1>(v, t, w, nullptr, ry);
                __syncwarp();
            } else {
                fft_fwd_ip<N1, N2, -1, LayY<N>>(v, t, w, b, ry);
            }
#pragma unroll
            for (int u = 0; u < N1 / N2; ++u)
#pragma unroll
                for (int k2 = 0; k2 < N2; ++k2) b[LayY<N>::at(w, t + N2 * u + N1 * k2)] = v[u * N2 + k2];
        }
        if (est) asm volatile("cp.async.wait_group 0;\n" ::: "memory");   // next x strip's eps: in smem by the barrier
        fence_async_smem();   // generic-proxy writes of the strip -> visible to the TMA store
        __syncthreads();
        if (tid == 0) {
            store(g);
            if (PR == 1 && g + 1 < G && (g + 1) % P == 0) {
                // first strip of the next phase reads what this phase wrote: every store complete
                bulk_wait0();
                fence_async_global();
                load(g + 1);
            }
        }
    }
    if (tid == 0) bulk_wait0();
    if (CG) {
        const int vec = vl / 3;
        const int nb = gridDim.x * 3;
        cg_block_partial(pmp, cgf.part_x + (size_t)vec * nb + (size_t)l * gridDim.x + blockIdx.x, buf);
        const long long lin = (long long)vl * gridDim.x + blockIdx.x;
        if (lin == 0 && tid == 0) *cgf.nb_x = nb;
    }
}

template <int N1, int N2>
cudaError_t launch_plane_t_t(const OpArgs& a, int nslab, const CGFuse* cg, cudaStream_t st, const CUtensorMap& my,
                             const CUtensorMap& mx, int zbase) {
    const int pr = a.plane_t == 3 ? 2 : 1;
    const dim3 g((unsigned)(a.mp.n3 / pr), (unsigned)nslab);
    auto run = [&](auto kern, auto cgarg, size_t smem, int nt) -> cudaError_t {
        cudaError_t e = allow_smem((const void*)kern, smem);
        if (e != cudaSuccess) return e;
        kern<<<g, nt, smem, st>>>(a, cgarg, my, mx, zbase);
        return cudaGetLastError();
    };
    using C0 = PlaneTCfg<N1, N2, 0>;
    using C1 = PlaneTCfg<N1, N2, 1>;
    using C2 = PlaneTCfg<N1, N2, 1, 2>;
    if (a.plane_t == 3) {
        if (cg) return run(k_plane_t<N1, N2, 1, 1, 2>, *cg, C2::smem, C2::NT);
        return run(k_plane_t<N1, N2, 0, 1, 2>, CGFuse{}, C2::smem, C2::NT);
    }
    if (a.plane_t == 2) {
        if (cg) return run(k_plane_t<N1, N2, 1, 1>, *cg, C1::smem, C1::NT);
        return run(k_plane_t<N1, N2, 0, 1>, CGFuse{}, C1::smem, C1::NT);
    }
    if (cg) return run(k_plane_t<N1, N2, 1, 0>, *cg, C0::smem, C0::NT);
    return run(k_plane_t<N1, N2, 0, 0>, CGFuse{}, C0::smem, C0::NT);
}

}  // namespace

bool plane_t_supported(const OpArgs& a) {
    return a.fast && a.nslab == 1 && a.mp.n1 == a.mp.n2 && (a.mp.n1 == 64 || a.mp.n1 == 128 || a.mp.n1 == 256);
}

// Tensor maps of a plane buffer viewed as [planes][N rows][2N doubles]: box
// {16 doubles = 8 complex, N rows} (y strips) and {16 doubles, 16 rows} (x strips),
// 128-byte swizzle.  encode: cuTensorMapEncodeTiled (driver entry point).
int plane_t_encode(const OpArgs& a, void* base, long long planes, void* encode_fn, CUtensorMap* my, CUtensorMap* mx) {
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(encode_fn);
    const cuuint64_t N = (cuuint64_t)a.mp.n1;
    const cuuint64_t dims[3] = {2 * N, N, (cuuint64_t)planes};
    const cuuint64_t strides[2] = {2 * N * 8, 2 * N * N * 8};
    const cuuint32_t ey[3] = {1, 1, 1};
    const cuuint32_t by[3] = {16, (cuuint32_t)N, 1};
    const cuuint32_t bx[3] = {16, 16, 1};
    CUresult r1 = enc(my, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, by, ey, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUresult r2 = enc(mx, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, bx, ey, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return (r1 == CUDA_SUCCESS && r2 == CUDA_SUCCESS) ? 0 : 1;
}

cudaError_t launch_plane_tma(const OpArgs& a, int nslab, const CGFuse* cg, cudaStream_t st, const CUtensorMap& my,
                             const CUtensorMap& mx, int zbase) {
    switch (a.mp.n1) {
        case 64: return launch_plane_t_t<8, 8>(a, nslab, cg, st, my, mx, zbase);
        case 128: return launch_plane_t_t<16, 8>(a, nslab, cg, st, my, mx, zbase);
        case 256: return launch_plane_t_t<16, 16>(a, nslab, cg, st, my, mx, zbase);
        default: return cudaErrorNotSupported;
    }
}

}  // namespace bnf
