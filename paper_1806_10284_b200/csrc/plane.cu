// Fused real-space plane pass of the null-space-free matvec (SURVEY.md §8(a)
// a2-a4, Algorithms 1-2 of PAPER.md §5.3):
//
//   for every component l and z-plane c of U (x-fastest, rows of n1):
//     y-DFT over j (+)         (Alg. 2 step 2)
//     twiddle e^{-2 pi i b m1 i / (n1 n2)}
//     x-DFT over i (+)         (Alg. 2 step 3)
//     * 1/(n eps_l(a,b,c))     (B^{-1}; T^* B^{-1} T with un-normalised DFTs, DESIGN R7b)
//     x-DFT over a (-)         (Alg. 1 step 1)
//     twiddle e^{+2 pi i b m1 i / (n1 n2)}
//     y-DFT over b (-)         (Alg. 1 step 2)
//
// in ONE read and ONE write of the plane (96n B + 3n B of eps per vector
// instead of 3 x 96n for separate y / x / y passes).  A plane of N x N
// complex128 is split over a thread-block cluster of P = N/32 CTAs (P = 1
// for N <= 48): CTA r owns columns [32r, 32r+32) for the y phases and rows
// [32r, 32r+32) for the x phase; the two layouts are exchanged through
// distributed shared memory (st.shared::cluster), so the transpose never
// touches HBM.  Each FFT is the register-resident two-stage N1 x N2 plan of
// fastfft.cuh (shared-memory transpose inside the CTA).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "cgfuse.cuh"
#include "fastfft.cuh"
#include "kernels.cuh"

namespace cgx = cooperative_groups;

namespace bnf {
namespace {

using fast::cmul;
using fast::cscale;

__device__ __forceinline__ double2 tw_at(const TwP& t, unsigned long long P) {  // e^{2 pi i P / n}
    return cmul(__ldg(t.hi + (P >> t.shift)), __ldg(t.lo + (P & t.mask)));
}
__device__ __forceinline__ double2 conj2(double2 a) { return make_double2(a.x, -a.y); }

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}

// Stores of the plane's intermediate strips (read back by this CTA's next
// phase) carry an L2 evict-last policy so that they are less likely to be
// written back to DRAM before they are overwritten; the final strips evict first.
__device__ __forceinline__ unsigned long long l2_policy_last() {
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ unsigned long long l2_policy_first() {
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void st_hint(double2* ptr, double2 v, unsigned long long pol) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(ptr), "d"(v.x), "d"(v.y), "l"(pol)
                 : "memory");
}

// 256-bit global accesses (sm_100: one LDG/STG.E.ENL2.256 per adjacent complex pair)
__device__ __forceinline__ void ld_pair(const double2* p, double2& a, double2& b) {
    asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];\n" : "=d"(a.x), "=d"(a.y), "=d"(b.x), "=d"(b.y) : "l"(p));
}
__device__ __forceinline__ void st_pair(double2* p, double2 a, double2 b) {
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};\n" ::"l"(p), "d"(a.x), "d"(a.y), "d"(b.x), "d"(b.y) : "memory");
}
__device__ __forceinline__ void st_pair_hint(double2* p, double2 a, double2 b, unsigned long long pol) {
    asm volatile("st.global.L2::cache_hint.v4.f64 [%0], {%1, %2, %3, %4}, %5;\n" ::"l"(p), "d"(a.x), "d"(a.y), "d"(b.x),
                 "d"(b.y), "l"(pol)
                 : "memory");
}

// Load policies of the L2 plane pass (LD template bits): phase Y reads U once from
// HBM (read-only in that phase: non-coherent path, no L1 allocation, 256 B L2
// fetch); phases X / Y* read strips this CTA wrote through L2 (ld.cg: L2 only).
__device__ __forceinline__ double2 ld_y_first(const double2* p) {
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}
template <int LD>
__device__ __forceinline__ double2 ld_strip_y(const double2* p) {
    if constexpr (LD & 1) return ld_y_first(p);
    else return *p;
}
template <int LD>
__device__ __forceinline__ double2 ld_strip_l2(const double2* p) {
    if constexpr (LD & 2) return __ldcg(p);
    else return *p;
}

template <int P>
struct Cluster {
    __device__ static unsigned rank() { return P == 1 ? 0u : cgx::this_cluster().block_rank(); }
    // full barrier with release/acquire: remote stores before it are visible after it
    __device__ static void sync() {
        if (P == 1) {
            __syncthreads();
        } else {
            asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
            asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
        }
    }
    // barrier only ("every CTA has consumed its D"): the reads it orders have
    // already completed (their values were used), so no fence is needed
    __device__ static void sync_relaxed() {
        if (P == 1) {
            __syncthreads();
        } else {
            asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
            asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
        }
    }
    // store v to element e of CTA r's copy of the shared array at byte address base
    __device__ static void put(double2* local, unsigned base, unsigned r, int e, double2 v) {
        if (P == 1) {
            local[e] = v;
        } else {
            unsigned ra;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(ra) : "r"(base + 16u * (unsigned)e), "r"(r));
            asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};\n" ::"r"(ra), "d"(v.x), "d"(v.y) : "memory");
        }
    }
};

// smem (complex elements): max(N * CW data, XchT exchange) = CW * N1 * (N2 + 1)
template <int N1, int N2, int P>
struct PlaneCfg {
    static constexpr int N = N1 * N2;
    static constexpr int CW = N / P;     // columns (y phases) = rows (x phase) per CTA
    static constexpr int NT = CW * N2;   // threads
    static constexpr int SMEM = CW * N1 * (N2 + 1);
};

// Optional per-phase cycle accounting (OpArgs::prof != null, bnf_phase_counters):
// thread 0 of every CTA adds the clock64() delta of each phase to prof[k].
#define BNF_PROBE(k)                                                     \
    do {                                                                 \
        if (a.prof != nullptr && threadIdx.x == 0) {                     \
            const long long now_ = clock64();                            \
            atomicAdd(a.prof + (k), (unsigned long long)(now_ - t_last)); \
            t_last = now_;                                               \
        }                                                                \
    } while (0)

template <int N1, int N2, int P, int CG>
__global__ void __launch_bounds__(PlaneCfg<N1, N2, P>::NT, PlaneCfg<N1, N2, P>::NT <= 256 ? 2 : 1) k_plane(double2* __restrict__ U, OpArgs a, CGFuse cgf, int nslab) {
    using C = PlaneCfg<N1, N2, P>;
    constexpr int N = C::N, CW = C::CW;
    extern __shared__ double2 D[];
    __shared__ double acc_s[8];   // CG: this CTA's (p, M p) partial per vector
    const ModeP& p = a.mp;
    long long t_last = clock64();
    const unsigned r = Cluster<P>::rank();
    const int tid = threadIdx.x;
    constexpr bool EPF = (N % 16) == 0;
    unsigned char* eps_s = reinterpret_cast<unsigned char*>(D + C::SMEM);
    double* lut_s = reinterpret_cast<double*>(eps_s + CW * N);   // the <= 256-entry 1/eps table
    const bool epf = EPF && a.eps_idx != nullptr;
    if (epf)
        for (int q = threadIdx.x; q < 256; q += C::NT) lut_s[q] = __ldg(a.eps_lut + q);
    if (CG && tid < 8) acc_s[tid] = 0.0;
    // clusters loop over the planes (component slab, z-plane); the launch uses one
    // cluster per plane (a persistent grid measured slower on B200)
    const int ncl = gridDim.x / P, cid = blockIdx.x / P;
    const int total = a.n3loc * nslab;
    for (int pl = cid; pl < total; pl += ncl) {
    const int c = pl % a.n3loc;
    const int vl = pl / a.n3loc + a.comp0;
    const int l = vl % 3;
    double2* plane = U + (size_t)vl * a.nloc + (size_t)c * N * N;
    double2 v[N1];
    // B^{-1} material indices of this CTA's phase-X rows (contiguous CW*N bytes), prefetched
    if (epf) {
        const unsigned char* src = a.eps_idx + (size_t)l * a.nloc + (size_t)N * ((size_t)r * CW + (size_t)N * c);
        for (int q = threadIdx.x; q < CW * N / 16; q += C::NT) cp_async16(eps_s + 16 * q, src + 16 * q);
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    }

    // ---------------- phase Y: columns i = r*CW + w, FFT over j ----------------
    const int w = tid % CW, t = tid / CW;
    const int i = (int)r * CW + w;
    // integer phase numerators mod n12 (n1 n2 <= 2^20: 32-bit arithmetic is exact)
    const unsigned n12 = (unsigned)p.n12;
    const unsigned long long s3 = (unsigned long long)p.n3;
    const unsigned M = ((unsigned)p.m1 * (unsigned)i) % n12;   // m1 i mod n12
#pragma unroll
    for (int m = 0; m < N1; ++m) v[m] = plane[(size_t)(N2 * m + t) * N + i];
    fast::fft_fwd<N1, N2, 1, fast::XchW<N1, N2, CW>>(v, t, w, D, a.py.root2);
    BNF_PROBE(0);   // load + y-FFT
    {
        // e^{-2 pi i b M / n12} for b = t + N2 u + N1 k2: w^t (w^N2)^u (w^N1)^k2
        const unsigned Pt = ((unsigned)t * M) % n12;
        const unsigned Pu = ((unsigned)N2 * M) % n12;
        const unsigned Pk = ((unsigned)N1 * M) % n12;
        const double2 wt = conj2(tw_at(a.tw, Pt * s3));
        const double2 wu = conj2(tw_at(a.tw, Pu * s3));
        const double2 wk = conj2(tw_at(a.tw, Pk * s3));
        fast::twiddle_stage2<N1, N2>(v, wt, wu, wk);
    }
    // exchange Y -> X: element (b, i) goes to CTA b / CW, row b % CW, column i
    const unsigned dbase = (unsigned)__cvta_generic_to_shared(D);
    BNF_PROBE(1);   // twiddle
    Cluster<P>::sync_relaxed();   // every CTA is done with its own D
    BNF_PROBE(2);   // barrier 1
#pragma unroll
    for (int u = 0; u < N1 / N2; ++u)
#pragma unroll
        for (int k2 = 0; k2 < N2; ++k2) {
            const int b = t + N2 * u + N1 * k2;
            Cluster<P>::put(D, dbase, (unsigned)(b / CW), (b % CW) * N + i, v[u * N2 + k2]);
        }
    BNF_PROBE(3);   // DSMEM stores Y->X
    if (epf) asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    Cluster<P>::sync();
    BNF_PROBE(4);   // barrier 2

    // ---------------- phase X: rows b = r*CW + rw, FFT over i ----------------
    const int tx = tid % N2, rw = tid / N2;
    const int b = (int)r * CW + rw;
#pragma unroll
    for (int m = 0; m < N1; ++m) v[m] = D[rw * N + N2 * m + tx];
    __syncthreads();   // D becomes the transpose buffer
    fast::fft_fwd<N1, N2, 1, fast::XchT<N1, N2, CW>>(v, tx, rw, D, a.px.root2);
    BNF_PROBE(5);   // x-FFT
    double pmp = 0.0;
    {
        const size_t rowofs = (size_t)l * a.nloc + (size_t)N * ((size_t)b + (size_t)N * c);
#pragma unroll
        for (int u = 0; u < N1 / N2; ++u)
#pragma unroll
            for (int k2 = 0; k2 < N2; ++k2) {
                const int aa = tx + N2 * u + N1 * k2;
                const double e_ = epf ? lut_s[eps_s[rw * N + aa]]
                                      : (a.eps_idx ? __ldg(a.eps_lut + __ldg(a.eps_idx + rowofs + aa))
                                                   : __ldg(a.eps_inv + rowofs + aa));
                const double s_ = a.inv_n * e_;
                const double2 x = v[u * N2 + k2];
                if (CG) pmp += s_ * (x.x * x.x + x.y * x.y);   // (p, M p) = sum |T v|^2 / (n eps)
                v[u * N2 + k2] = cscale(x, s_);
            }
    }
    BNF_PROBE(6);   // eps (+ CG partial)
    fast::fft_mirror<N1, N2, -1, fast::XchT<N1, N2, CW>>(v, tx, rw, D, a.px.root2);
    BNF_PROBE(7);   // x-FFT*
    // exchange X -> Y: element (b, a) goes to CTA a / CW, row b, column a % CW (ld CW)
    Cluster<P>::sync_relaxed();
    BNF_PROBE(8);   // barrier 3
#pragma unroll
    for (int m = 0; m < N1; ++m) {
        const int aa = N2 * m + tx;
        Cluster<P>::put(D, dbase, (unsigned)(aa / CW), b * CW + (aa % CW), v[m]);
    }
    BNF_PROBE(9);   // DSMEM stores X->Y
    Cluster<P>::sync();
    BNF_PROBE(10);  // barrier 4

    // ---------------- phase Y*: conj twiddle, FFT (-) over b ----------------
    {
        // e^{+2 pi i b M / n12} for b = N2 m + t: w^t (w^N2)^m
        const unsigned Pt = ((unsigned)t * M) % n12;
        const unsigned Pu = ((unsigned)N2 * M) % n12;
        const double2 wt = tw_at(a.tw, Pt * s3);
        const double2 wu = tw_at(a.tw, Pu * s3);
#pragma unroll
        for (int m = 0; m < N1; ++m) v[m] = D[(N2 * m + t) * CW + w];
        fast::twiddle_natural<N1, N2>(v, wt, wu);
    }
    __syncthreads();
    fast::fft_fwd<N1, N2, -1, fast::XchW<N1, N2, CW>>(v, t, w, D, a.py.root2);
    BNF_PROBE(11);  // twiddle* + y-FFT*
#pragma unroll
    for (int u = 0; u < N1 / N2; ++u)
#pragma unroll
        for (int k2 = 0; k2 < N2; ++k2) {
            const int j = t + N2 * u + N1 * k2;
            plane[(size_t)j * N + i] = v[u * N2 + k2];
        }
    BNF_PROBE(12);  // stores issued
    if (a.prof != nullptr && threadIdx.x == 0) atomicAdd(a.prof + 15, 1ull);   // plane-part count
    if (CG) {
        // this plane's (p, M p) partial (D is free after the y-FFT*; >= blockDim entries)
        const double2 bs = block_sum(make_double2(pmp, 0.0), D);
        if (tid == 0) acc_s[(vl - a.comp0) / 3] += bs.x;
    }
    __syncthreads();   // D is reused by the next plane
    }   // planes
    if (CG) {
        // per-CTA partials of (p, M p) for every vector
        const int nvec = nslab / 3;
        const int nb = gridDim.x;
        if (tid < nvec) cgf.part_x[(size_t)tid * nb + blockIdx.x] = acc_s[tid];
        __syncthreads();
        if (blockIdx.x == 0 && tid == 0) *cgf.nb_x = nb;   // alpha: k_cg_finish after this pass
    }
}

// ---------------------------------------------------------------------------
// L2 variant: one CTA per (component, z-plane).  The CTA runs the P column
// strips of phase Y, then the P row strips of phase X, then the P column
// strips of phase Y* one after the other (each strip = one cluster rank's
// work above), exchanging the strips through the plane itself in global
// memory: the plane (N*N*16 B, 256 KB at 128^2) is re-read while it is hot
// in L2, so DRAM still sees one read and one write per element, and there
// are no cluster barriers or DSMEM stores.  Two CTAs per SM overlap.
// SPLIT = 2: a cluster of two CTAs per plane, each taking every other strip of
// every phase (the phases meet at a cluster barrier, whose release / acquire
// orders the strips written through L2): twice the CTAs, half the work each,
// so the last wave of the launch is half as long.
// RS = 1: the y / x stage-root tables are copied to shared memory once per CTA
// (the 15 root loads per thread and FFT then leave the LSU global queue).
// XEO = 1 (N = 128 plan only): phase X transforms each row as its even / odd
// 64-point halves (fastfft fft_fwd_eo / fft_mirror_eo), so every thread holds
// adjacent pairs and the row strips move with 256-bit loads and stores
// (half the LSU global instructions of phase X).
template <int N1, int N2, int P, int CG, int SL = 0, int SPLIT = 1, int RS = 0, int XEO = 0, int LD = 0>
__global__ void __launch_bounds__(PlaneCfg<N1, N2, P>::NT, PlaneCfg<N1, N2, P>::NT <= 256 ? 2 : 1) k_plane_l2(double2* __restrict__ U, OpArgs a, CGFuse cgf) {
    using C = PlaneCfg<N1, N2, P>;
    constexpr int N = C::N, CW = C::CW;
    // Phase X's FFT exchanges are warp-local (a row's N2 threads are consecutive lanes and XchT gives
    // each row its own region), so they synchronise with __syncwarp and the CTA's warps drift apart
    // inside the phase (the loads of one warp overlap the FFT of another).  LD bit 4 restores the
    // CTA-wide barriers (A/B switch, 128 plan).
    constexpr bool XW = (LD & 4) == 0 && (32 % N2) == 0 && (C::NT % 32) == 0 && XEO == 0;
    extern __shared__ double2 D[];
    const ModeP& p = a.mp;
    const int tid = threadIdx.x;
    const int c = blockIdx.x / SPLIT;
    const int r0 = SPLIT == 1 ? 0 : (int)(blockIdx.x % SPLIT);
    const int vl = blockIdx.y + a.comp0;
    const int l = vl % 3;
    // plane rows b: one slab -> plane + b N; virtual / distributed slabs -> the block of the
    // source slab b / n2loc, row b % n2loc ([r][vec][l][cl][jl][a], blocks of nblk)
    double2* plane = U + (size_t)vl * (SL ? a.nblk : p.n) + (size_t)c * (SL ? a.n2loc : N) * N;
    auto rowp = [&](int b) -> double2* {
        if constexpr (SL == 0) return plane + (size_t)b * N;
        else return plane + (size_t)(b / a.n2loc) * ((size_t)(gridDim.y / 3) * 3 * a.nblk) + (size_t)(b % a.n2loc) * N;
    };
    constexpr bool EPF = (N % 16) == 0 && N <= 128;   // whole-plane index prefetch fits next to D
    unsigned char* eps_s = reinterpret_cast<unsigned char*>(D + C::SMEM);   // [N][N] material indices
    double* lut_s = reinterpret_cast<double*>(eps_s + (EPF ? N * N : 0));
    const bool epf = EPF && a.eps_idx != nullptr;
    double2* ry_s = reinterpret_cast<double2*>(lut_s + 256);   // RS: stage roots [N1 N2] (y), then (x)
    double2* rx_s = ry_s + N1 * N2;
    if constexpr (RS) {
        for (int q = tid; q < N1 * N2; q += C::NT) {
            ry_s[q] = __ldg(a.py.root2 + q);
            rx_s[q] = __ldg(a.px.root2 + q);
        }
        __syncthreads();
    }
    const double2* ry = RS ? ry_s : a.py.root2;
    const double2* rx = RS ? rx_s : a.px.root2;
    if (epf) {
        for (int q = tid; q < 256; q += C::NT) lut_s[q] = __ldg(a.eps_lut + q);
        const unsigned char* src = a.eps_idx + (size_t)l * (SL ? a.nloc : p.n) + (size_t)N * N * c;
        for (int q = tid; q < N * N / 16; q += C::NT) cp_async16(eps_s + 16 * q, src + 16 * q);
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
    const int w = tid % CW, t = tid / CW;          // strip-column layout (phases Y, Y*)
    const int tx = tid % N2, rw = tid / N2;        // strip-row layout (phase X)
    const unsigned n12 = (unsigned)p.n12;
    const unsigned long long s3 = (unsigned long long)p.n3;
    double2 v[N1];
    const unsigned long long pol_keep = a.plane_hint ? l2_policy_last() : 0ull;
    const unsigned long long pol_out = a.plane_hint ? l2_policy_first() : 0ull;
    // ---------------- phase Y: column strips ----------------
    for (int r = r0; r < P; r += SPLIT) {
        const int i = r * CW + w;
        const unsigned M = ((unsigned)p.m1 * (unsigned)i) % n12;
#pragma unroll
        for (int m = 0; m < N1; ++m) v[m] = ld_strip_y<LD>(rowp(N2 * m + t) + i);
        fast::fft_fwd<N1, N2, 1, fast::XchW<N1, N2, CW>, RS != 0>(v, t, w, D, ry);
        const double2 wt = conj2(tw_at(a.tw, (unsigned long long)(((unsigned)t * M) % n12) * s3));
        const double2 wu = conj2(tw_at(a.tw, (unsigned long long)(((unsigned)N2 * M) % n12) * s3));
        const double2 wk = conj2(tw_at(a.tw, (unsigned long long)(((unsigned)N1 * M) % n12) * s3));
        fast::twiddle_stage2<N1, N2>(v, wt, wu, wk);
        if (a.plane_hint) {
#pragma unroll
            for (int u = 0; u < N1 / N2; ++u)
#pragma unroll
                for (int k2 = 0; k2 < N2; ++k2) st_hint(rowp(t + N2 * u + N1 * k2) + i, v[u * N2 + k2], pol_keep);
        } else {
#pragma unroll
            for (int u = 0; u < N1 / N2; ++u)
#pragma unroll
                for (int k2 = 0; k2 < N2; ++k2) rowp(t + N2 * u + N1 * k2)[i] = v[u * N2 + k2];
        }
    }
    if (epf) asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    if constexpr (SPLIT == 1) __syncthreads();   // the strips written above are read by other threads below
    else Cluster<2>::sync();                     // ... and by the other CTA of the plane (cluster release / acquire)
    // ---------------- phase X: row strips ----------------
    double pmp = 0.0;
    for (int r = r0; r < P; r += SPLIT) {
        const int b = r * CW + rw;
        double2* row = rowp(b);
        const size_t rowofs = (size_t)l * (SL ? a.nloc : p.n) + (size_t)N * ((size_t)b + (size_t)N * c);
        if constexpr (XEO) {
            static_assert(N1 == 2 * N2, "XEO: N1 = 2 N2");
            using XH = fast::XchT<N2, N2, CW>;
            double2 ea[N2], ob[N2];
#pragma unroll
            for (int m = 0; m < N2; ++m) ld_pair(row + 2 * (N2 * m + tx), ea[m], ob[m]);
            fast::fft_fwd_eo<N2, N2, 1, XH, RS != 0>(ea, ob, v, tx, rw, D, D + XH::size, rx);
            auto scale_eo = [&](auto eps_at) {
#pragma unroll
                for (int q = 0; q < N1; ++q) {
                    const int aa = tx + N2 * q;
                    const double s_ = a.inv_n * eps_at(aa);
                    const double2 x = v[q];
                    if (CG) pmp += s_ * (x.x * x.x + x.y * x.y);
                    v[q] = cscale(x, s_);
                }
            };
            if (epf) scale_eo([&](int aa) { return lut_s[eps_s[b * N + aa]]; });
            else if (a.eps_idx) scale_eo([&](int aa) { return __ldg(a.eps_lut + __ldg(a.eps_idx + rowofs + aa)); });
            else scale_eo([&](int aa) { return __ldg(a.eps_inv + rowofs + aa); });
            fast::fft_mirror_eo<N2, N2, -1, XH, RS != 0>(v, ea, ob, tx, rw, D, D + XH::size, rx);
            if (a.plane_hint) {
#pragma unroll
                for (int m = 0; m < N2; ++m) st_pair_hint(row + 2 * (N2 * m + tx), ea[m], ob[m], pol_keep);
            } else {
#pragma unroll
                for (int m = 0; m < N2; ++m) st_pair(row + 2 * (N2 * m + tx), ea[m], ob[m]);
            }
        } else {
#pragma unroll
        for (int m = 0; m < N1; ++m) v[m] = ld_strip_l2<LD>(row + N2 * m + tx);
        fast::fft_fwd<N1, N2, 1, fast::XchT<N1, N2, CW>, RS != 0, XW>(v, tx, rw, D, rx);
        // 1/(n eps) scaling (+ CG partial); the ε source is chosen once per strip, not per element
        auto scale = [&](auto eps_at) {
#pragma unroll
            for (int u = 0; u < N1 / N2; ++u)
#pragma unroll
                for (int k2 = 0; k2 < N2; ++k2) {
                    const int aa = tx + N2 * u + N1 * k2;
                    const double s_ = a.inv_n * eps_at(aa);
                    const double2 x = v[u * N2 + k2];
                    if (CG) pmp += s_ * (x.x * x.x + x.y * x.y);   // (p, M p) = sum |T v|^2 / (n eps)
                    v[u * N2 + k2] = cscale(x, s_);
                }
        };
        if (epf) scale([&](int aa) { return lut_s[eps_s[b * N + aa]]; });
        else if (a.eps_idx) scale([&](int aa) { return __ldg(a.eps_lut + __ldg(a.eps_idx + rowofs + aa)); });
        else scale([&](int aa) { return __ldg(a.eps_inv + rowofs + aa); });
        fast::fft_mirror<N1, N2, -1, fast::XchT<N1, N2, CW>, RS != 0, XW>(v, tx, rw, D, rx);
        if (a.plane_hint) {
#pragma unroll
            for (int m = 0; m < N1; ++m) st_hint(row + N2 * m + tx, v[m], pol_keep);
        } else {
#pragma unroll
            for (int m = 0; m < N1; ++m) row[N2 * m + tx] = v[m];
        }
        }
    }
    if constexpr (SPLIT == 1) __syncthreads();
    else Cluster<2>::sync();
    // ---------------- phase Y*: column strips ----------------
    for (int r = r0; r < P; r += SPLIT) {
        const int i = r * CW + w;
        const unsigned M = ((unsigned)p.m1 * (unsigned)i) % n12;
#pragma unroll
        for (int m = 0; m < N1; ++m) v[m] = ld_strip_l2<LD>(rowp(N2 * m + t) + i);
        const double2 wt = tw_at(a.tw, (unsigned long long)(((unsigned)t * M) % n12) * s3);
        const double2 wu = tw_at(a.tw, (unsigned long long)(((unsigned)N2 * M) % n12) * s3);
        fast::twiddle_natural<N1, N2>(v, wt, wu);
        fast::fft_fwd<N1, N2, -1, fast::XchW<N1, N2, CW>, RS != 0>(v, t, w, D, ry);
        if (a.plane_hint) {
#pragma unroll
            for (int u = 0; u < N1 / N2; ++u)
#pragma unroll
                for (int k2 = 0; k2 < N2; ++k2) st_hint(rowp(t + N2 * u + N1 * k2) + i, v[u * N2 + k2], pol_out);
        } else {
#pragma unroll
            for (int u = 0; u < N1 / N2; ++u)
#pragma unroll
                for (int k2 = 0; k2 < N2; ++k2) rowp(t + N2 * u + N1 * k2)[i] = v[u * N2 + k2];
        }
    }
    if (CG) {
        // this plane's (p, M p) partial; alpha is formed by k_cg_finish after this pass
        const int vec = vl / 3;
        const int nb = gridDim.x * 3;
        cg_block_partial(pmp, cgf.part_x + ((size_t)(SL ? a.slab * (gridDim.y / 3) : 0) + vec) * nb + (size_t)l * gridDim.x + blockIdx.x, D);
        const long long lin = (long long)vl * gridDim.x + blockIdx.x;
        if (lin == 0 && tid == 0) *cgf.nb_x = nb;
    }
}

// ---------------------------------------------------------------------------
// Warp-local variant ("plane_w"): one CTA per (component, z-plane)
// as k_plane_l2, strips exchanged through L2, but every FFT sequence lives in
// N2 consecutive lanes of ONE warp (lane = w N2 + t, W = 32 / N2 sequences per
// warp), so the FFT stage exchange is warp-local -- xor shuffles (XSHFL = 1) or
// a padded per-warp shared-memory region with __syncwarp (XSHFL = 0) -- and the
// warps of a CTA run their strips independently: the only CTA barriers are the
// two phase boundaries (Y -> X -> Y*).  Stage-twiddle tables and the plane's
// B^{-1} material indices sit in shared memory.
template <int N1, int N2, int NWARP, int XSHFL>
struct PlaneWCfg {
    static constexpr int N = N1 * N2;
    static constexpr int W = 32 / N2;               // sequences per warp
    static constexpr int CW = W * NWARP;            // sequences per strip pass
    static constexpr int P = N / CW;                // strip passes per phase
    static constexpr int NT = 32 * NWARP;
    static constexpr int XS = XSHFL ? 0 : fast::WarpXch<N1, N2>::size;   // complex per warp
    static constexpr size_t smem = (size_t)(NWARP * XS + 2 * N) * sizeof(double2) + (size_t)N * N + 256 * sizeof(double);
};

template <int N1, int N2, int NWARP, int CG, int XSHFL, int SL = 0>
__global__ void __launch_bounds__(32 * NWARP, 2) k_plane_w(double2* __restrict__ U, OpArgs a, CGFuse cgf) {
    using C = PlaneWCfg<N1, N2, NWARP, XSHFL>;
    constexpr int N = C::N, W = C::W, CW = C::CW, P = C::P, NT = C::NT;
    static_assert(N % CW == 0 && 32 % N2 == 0 && N1 % N2 == 0, "plane_w plan");
    extern __shared__ double2 D[];
    const ModeP& p = a.mp;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int w = lane / N2, t = lane % N2;
    const int c = blockIdx.x;
    const int vl = blockIdx.y + a.comp0;
    const int l = vl % 3;
    // plane rows b: one slab -> plane + b N; virtual / distributed slabs -> the block of the
    // source slab b / n2loc, row b % n2loc ([r][vec][l][cl][jl][a], blocks of nblk)
    double2* plane = U + (size_t)vl * (SL ? a.nblk : p.n) + (size_t)c * (SL ? a.n2loc : N) * N;
    auto rowp = [&](int b) -> double2* {
        if constexpr (SL == 0) return plane + (size_t)b * N;
        else return plane + (size_t)(b / a.n2loc) * ((size_t)(gridDim.y / 3) * 3 * a.nblk) + (size_t)(b % a.n2loc) * N;
    };
    double2* xw = D + warp * C::XS;                         // this warp's exchange region
    double2* ry = D + NWARP * C::XS;                        // y stage twiddles [k1][t]
    double2* rx = ry + N;                                   // x stage twiddles
    unsigned char* eps_s = reinterpret_cast<unsigned char*>(rx + N);   // [N][N] material indices
    double* lut_s = reinterpret_cast<double*>(eps_s + N * N);
    const bool epf = a.eps_idx != nullptr;
    for (int q = tid; q < N; q += NT) {
        ry[q] = __ldg(a.py.root2 + q);
        rx[q] = __ldg(a.px.root2 + q);
    }
    if (epf) {
        for (int q = tid; q < 256; q += NT) lut_s[q] = __ldg(a.eps_lut + q);
        const unsigned char* src = a.eps_idx + (size_t)l * (SL ? a.nloc : p.n) + (size_t)N * N * c;
        for (int q = tid; q < N * N / 16; q += NT) cp_async16(eps_s + 16 * q, src + 16 * q);
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
    __syncthreads();   // stage-twiddle tables
    const unsigned n12 = (unsigned)p.n12;
    const unsigned long long s3 = (unsigned long long)p.n3;
    const unsigned long long pol_keep = a.plane_hint ? l2_policy_last() : 0ull;
    const unsigned long long pol_out = a.plane_hint ? l2_policy_first() : 0ull;
    double2 v[N1];
    // ---------------- phase Y: y-DFT (+) of columns i, twiddle e^{-2 pi i b m1 i / n12} ----------------
#pragma unroll 1
    for (int r = 0; r < P; ++r) {
        const int i = r * CW + warp * W + w;
        const unsigned M = ((unsigned)p.m1 * (unsigned)i) % n12;
#pragma unroll
        for (int m = 0; m < N1; ++m) v[m] = rowp(N2 * m + t)[i];
        fast::fft_fwd_w<N1, N2, 1, XSHFL>(v, t, w, xw, ry);
        const double2 wt = conj2(tw_at(a.tw, (unsigned long long)(((unsigned)t * M) % n12) * s3));
        const double2 wu = conj2(tw_at(a.tw, (unsigned long long)(((unsigned)N2 * M) % n12) * s3));
        const double2 wk = conj2(tw_at(a.tw, (unsigned long long)(((unsigned)N1 * M) % n12) * s3));
        fast::twiddle_stage2<N1, N2>(v, wt, wu, wk);
#pragma unroll
        for (int u = 0; u < N1 / N2; ++u)
#pragma unroll
            for (int k2 = 0; k2 < N2; ++k2) {
                double2* dst = rowp(t + N2 * u + N1 * k2) + i;
                if (a.plane_hint) st_hint(dst, v[u * N2 + k2], pol_keep);
                else *dst = v[u * N2 + k2];
            }
    }
    if (epf) asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();   // every column strip is written (block-scope visibility) before rows are read
    // ---------------- phase X: x-DFT (+), 1/(n eps) [+ (p, Mp)], x-DFT (-) of rows b ----------------
    double pmp = 0.0;
#pragma unroll 1
    for (int r = 0; r < P; ++r) {
        const int b = r * CW + warp * W + w;
        double2* row = rowp(b);
#pragma unroll
        for (int m = 0; m < N1; ++m) v[m] = row[N2 * m + t];
        fast::fft_fwd_w<N1, N2, 1, XSHFL>(v, t, w, xw, rx);
        const size_t rowofs = (size_t)l * (SL ? a.nloc : p.n) + (size_t)N * ((size_t)b + (size_t)N * c);
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
        if (epf) scale([&](int aa) { return lut_s[eps_s[b * N + aa]]; });
        else scale([&](int aa) { return __ldg(a.eps_inv + rowofs + aa); });
        fast::fft_mirror_w<N1, N2, -1, XSHFL>(v, t, w, xw, rx);
#pragma unroll
        for (int m = 0; m < N1; ++m) {
            if (a.plane_hint) st_hint(row + N2 * m + t, v[m], pol_keep);
            else row[N2 * m + t] = v[m];
        }
    }
    __syncthreads();
    // ---------------- phase Y*: conj twiddle, y-DFT (-) of columns ----------------
#pragma unroll 1
    for (int r = 0; r < P; ++r) {
        const int i = r * CW + warp * W + w;
        const unsigned M = ((unsigned)p.m1 * (unsigned)i) % n12;
#pragma unroll
        for (int m = 0; m < N1; ++m) v[m] = rowp(N2 * m + t)[i];
        const double2 wt = tw_at(a.tw, (unsigned long long)(((unsigned)t * M) % n12) * s3);
        const double2 wu = tw_at(a.tw, (unsigned long long)(((unsigned)N2 * M) % n12) * s3);
        fast::twiddle_natural<N1, N2>(v, wt, wu);
        fast::fft_fwd_w<N1, N2, -1, XSHFL>(v, t, w, xw, ry);
#pragma unroll
        for (int u = 0; u < N1 / N2; ++u)
#pragma unroll
            for (int k2 = 0; k2 < N2; ++k2) {
                double2* dst = rowp(t + N2 * u + N1 * k2) + i;
                if (a.plane_hint) st_hint(dst, v[u * N2 + k2], pol_out);
                else *dst = v[u * N2 + k2];
            }
    }
    if (CG) {
        const int vec = vl / 3;
        const int nb = gridDim.x * 3;
        cg_block_partial(pmp, cgf.part_x + ((size_t)(SL ? a.slab * (gridDim.y / 3) : 0) + vec) * nb + (size_t)l * gridDim.x + blockIdx.x, D);
        const long long lin = (long long)vl * gridDim.x + blockIdx.x;
        if (lin == 0 && tid == 0) *cgf.nb_x = nb;
    }
}

template <int N1, int N2, int NWARP, int XSHFL>
cudaError_t launch_plane_w_t(const OpArgs& a, double2* U, int nslab, const CGFuse* cg, cudaStream_t st) {
    using C = PlaneWCfg<N1, N2, NWARP, XSHFL>;
    const dim3 g((unsigned)a.n3loc, (unsigned)nslab);
    auto run = [&](auto kern, auto cgarg) -> cudaError_t {
        cudaError_t e = allow_smem((const void*)kern, C::smem);
        if (e != cudaSuccess) return e;
        kern<<<g, C::NT, C::smem, st>>>(U, a, cgarg);
        return cudaGetLastError();
    };
    if (a.nslab > 1) {
        if (cg) return run(k_plane_w<N1, N2, NWARP, 1, XSHFL, 1>, *cg);
        return run(k_plane_w<N1, N2, NWARP, 0, XSHFL, 1>, CGFuse{});
    }
    if (cg) return run(k_plane_w<N1, N2, NWARP, 1, XSHFL>, *cg);
    return run(k_plane_w<N1, N2, NWARP, 0, XSHFL>, CGFuse{});
}

template <int N1, int N2, int P>
cudaError_t launch_plane_l2_t(const OpArgs& a, double2* U, int nslab, const CGFuse* cg, cudaStream_t st) {
    using C = PlaneCfg<N1, N2, P>;
    constexpr bool EPF = (C::N % 16) == 0 && C::N <= 128;
    const size_t smem = (size_t)C::SMEM * sizeof(double2) + (EPF ? (size_t)C::N * C::N : 0) + 256 * sizeof(double) +
                        (a.plane_rs ? (size_t)2 * N1 * N2 * sizeof(double2) : 0);
    const dim3 g((unsigned)a.n3loc, (unsigned)nslab);
    auto run = [&](auto kern, auto cgarg) -> cudaError_t {
        cudaError_t e = allow_smem((const void*)kern, smem);
        if (e != cudaSuccess) return e;
        kern<<<g, C::NT, smem, st>>>(U, a, cgarg);
        return cudaGetLastError();
    };
    if (a.nslab > 1) {
        if (cg) return run(k_plane_l2<N1, N2, P, 1, 1>, *cg);
        return run(k_plane_l2<N1, N2, P, 0, 1>, CGFuse{});
    }
    if (a.plane_split == 2 && P % 2 == 0) {   // cluster of two CTAs per plane
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(2 * a.n3loc), (unsigned)nslab);
        cfg.blockDim = dim3(C::NT, 1, 1);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        auto run2 = [&](auto kern, auto cgarg) -> cudaError_t {
            cudaError_t e = allow_smem((const void*)kern, smem);
            if (e != cudaSuccess) return e;
            return cudaLaunchKernelEx(&cfg, kern, U, a, cgarg);
        };
        if (a.plane_rs) {
            if (cg) return run2(k_plane_l2<N1, N2, P, 1, 0, 2, 1>, *cg);
            return run2(k_plane_l2<N1, N2, P, 0, 0, 2, 1>, CGFuse{});
        }
        if (cg) return run2(k_plane_l2<N1, N2, P, 1, 0, 2>, *cg);
        return run2(k_plane_l2<N1, N2, P, 0, 0, 2>, CGFuse{});
    }
    if constexpr (N1 == 2 * N2 && N1 * N2 == 128) {
        if (a.plane_xeo) {
            if (a.plane_rs) {
                if (cg) return run(k_plane_l2<N1, N2, P, 1, 0, 1, 1, 1>, *cg);
                return run(k_plane_l2<N1, N2, P, 0, 0, 1, 1, 1>, CGFuse{});
            }
            if (cg) return run(k_plane_l2<N1, N2, P, 1, 0, 1, 0, 1>, *cg);
            return run(k_plane_l2<N1, N2, P, 0, 0, 1, 0, 1>, CGFuse{});
        }
    }
    if constexpr (N1 * N2 == 128) {
        if (a.plane_rs && a.plane_ld) {   // load-policy variants (BNF_PLANE_LD)
            switch (a.plane_ld) {
                case 1: return cg ? run(k_plane_l2<N1, N2, P, 1, 0, 1, 1, 0, 1>, *cg) : run(k_plane_l2<N1, N2, P, 0, 0, 1, 1, 0, 1>, CGFuse{});
                case 2: return cg ? run(k_plane_l2<N1, N2, P, 1, 0, 1, 1, 0, 2>, *cg) : run(k_plane_l2<N1, N2, P, 0, 0, 1, 1, 0, 2>, CGFuse{});
                case 3: return cg ? run(k_plane_l2<N1, N2, P, 1, 0, 1, 1, 0, 3>, *cg) : run(k_plane_l2<N1, N2, P, 0, 0, 1, 1, 0, 3>, CGFuse{});
                case 4: return cg ? run(k_plane_l2<N1, N2, P, 1, 0, 1, 1, 0, 4>, *cg) : run(k_plane_l2<N1, N2, P, 0, 0, 1, 1, 0, 4>, CGFuse{});
                case 6: return cg ? run(k_plane_l2<N1, N2, P, 1, 0, 1, 1, 0, 6>, *cg) : run(k_plane_l2<N1, N2, P, 0, 0, 1, 1, 0, 6>, CGFuse{});
                default: return cg ? run(k_plane_l2<N1, N2, P, 1, 0, 1, 1, 0, 7>, *cg) : run(k_plane_l2<N1, N2, P, 0, 0, 1, 1, 0, 7>, CGFuse{});
            }
        }
    }
    if (a.plane_rs) {
        if (cg) return run(k_plane_l2<N1, N2, P, 1, 0, 1, 1>, *cg);
        return run(k_plane_l2<N1, N2, P, 0, 0, 1, 1>, CGFuse{});
    }
    if (cg) return run(k_plane_l2<N1, N2, P, 1>, *cg);
    return run(k_plane_l2<N1, N2, P, 0>, CGFuse{});
}

template <int N1, int N2, int P>
cudaError_t launch_plane_t(const OpArgs& a, double2* U, int nslab, const CGFuse* cg, cudaStream_t st) {
    using C = PlaneCfg<N1, N2, P>;
    const size_t smem = (size_t)C::SMEM * sizeof(double2) + (size_t)C::CW * C::N + 256 * sizeof(double);
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(C::NT, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = P;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const int total = a.n3loc * nslab;
    auto run = [&](auto kern, auto cgarg) -> cudaError_t {
        cudaError_t e = allow_smem((const void*)kern, smem);
        if (e != cudaSuccess) return e;
        if (P > 8) {
            e = cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            if (e != cudaSuccess) return e;
        }
        cfg.gridDim = dim3((unsigned)(P * total), 1, 1);
        return cudaLaunchKernelEx(&cfg, kern, U, a, cgarg, nslab);
    };
    if (cg) return run(k_plane<N1, N2, P, 1>, *cg);
    return run(k_plane<N1, N2, P, 0>, CGFuse{});
}

}  // namespace

// Plans: N -> (N1, N2, P).  P = N/32 (32 columns per CTA) from N = 64 up.
#define BNF_PLANE_PLANS(X) \
    X(8, 4, 2, 1) X(12, 6, 2, 1) X(16, 4, 4, 1) X(24, 12, 2, 1) X(32, 8, 4, 1) X(48, 12, 4, 1) \
    X(64, 8, 8, 2) X(96, 24, 4, 3) X(128, 16, 8, 4) X(192, 24, 8, 6) X(256, 16, 16, 8)

bool plane_supported(const OpArgs& a) {
    if (!a.fast || a.mp.n1 != a.mp.n2) return false;
    switch (a.mp.n1) {
#define BNF_CASE(NN, A, B, PP) case NN: return true;
        BNF_PLANE_PLANS(BNF_CASE)
#undef BNF_CASE
        default: return false;
    }
}

bool plane_w_supported(const OpArgs& a) {
    return a.fast && a.mp.n1 == a.mp.n2 && (a.mp.n1 == 64 || a.mp.n1 == 128 || a.mp.n1 == 256);
}

cudaError_t launch_plane(const OpArgs& a, double2* U, int nslab, const CGFuse* cg, cudaStream_t st) {
    if (a.plane_w && plane_w_supported(a)) {   // warp-local FFT exchanges (1: smem, 2: shuffles)
        const bool sh = a.plane_w == 2;
        switch (a.mp.n1) {
            case 64: return sh ? launch_plane_w_t<8, 8, 8, 1>(a, U, nslab, cg, st) : launch_plane_w_t<8, 8, 8, 0>(a, U, nslab, cg, st);
            case 128: return sh ? launch_plane_w_t<16, 8, 8, 1>(a, U, nslab, cg, st) : launch_plane_w_t<16, 8, 8, 0>(a, U, nslab, cg, st);
            case 256: return sh ? launch_plane_w_t<16, 16, 8, 1>(a, U, nslab, cg, st) : launch_plane_w_t<16, 16, 8, 0>(a, U, nslab, cg, st);
            default: break;
        }
    }
    if (a.plane_l2) {   // one CTA per plane, strips exchanged through L2
        switch (a.mp.n1) {
            case 64: return launch_plane_l2_t<8, 8, 2>(a, U, nslab, cg, st);
            case 96: return launch_plane_l2_t<24, 4, 3>(a, U, nslab, cg, st);
            case 128: return launch_plane_l2_t<16, 8, 4>(a, U, nslab, cg, st);
            case 192: return launch_plane_l2_t<24, 8, 6>(a, U, nslab, cg, st);
            case 256: return launch_plane_l2_t<16, 16, 16>(a, U, nslab, cg, st);   // 16-column strips: 2 CTAs/SM
            default: break;
        }
    }
    switch (a.mp.n1) {
#define BNF_CASE(NN, A, B, PP) case NN: return launch_plane_t<A, B, PP>(a, U, nslab, cg, st);
        BNF_PLANE_PLANS(BNF_CASE)
#undef BNF_CASE
        default: return cudaErrorNotSupported;
    }
}

}  // namespace bnf
