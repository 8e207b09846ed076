// Solver handle and the C ABI (include/bnf.h).
//
// Hot path per k-point:
//   a0  per-k setup: kappa-hat, Gamma mask, sigma table            (bnf_set_kappa)
//   a1-a5 M / A_r apply: 5 fused passes (kernels.cu)               (apply_op)
//   a6  batched CG on M = Q_r^* B^{-1} Q_r          (cg_solve)
//   a7  block inverse Lanczos with full reorthogonalisation         (bnf_solve)
//   a8  Rayleigh-Ritz on A_r, residuals, E-field recovery           (refine / bnf_eigvecs)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "bnf_internal.h"
#include "kernels.cuh"

struct bnf_lattice {
    bnf::Lattice L;
};

namespace bnf {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

namespace {

#define CK(call)                                                                                 \
    do {                                                                                         \
        cudaError_t _e = (call);                                                                 \
        if (_e != cudaSuccess) {                                                                 \
            set_error(std::string("CUDA: ") + cudaGetErrorString(_e) + " at " + #call);          \
            return BNF_ECUDA;                                                                    \
        }                                                                                        \
    } while (0)

// ---------------------------------------------------------------- tables
const long double kPi = 3.141592653589793238462643383279502884L;

double2 unit_root(long long num, long long den) {  // e^{2 pi i num/den}, exact reduction
    long long r = num % den;
    if (r < 0) r += den;
    long double ang = 2.0L * kPi * (long double)r / (long double)den;
    return make_double2((double)cosl(ang), (double)sinl(ang));
}

bool make_plan(int N, std::vector<int>& radices) {
    radices.clear();
    if (N < 1 || N > 1024) return false;
    int m = N;
    while (m % 8 == 0 && m != 16 && m != 32 && m != 128 && m != 512 && m != 2048) {
        radices.push_back(8);
        m /= 8;
    }
    while (m % 4 == 0) {
        radices.push_back(4);
        m /= 4;
    }
    while (m % 2 == 0) {
        radices.push_back(2);
        m /= 2;
    }
    while (m % 3 == 0) {
        radices.push_back(3);
        m /= 3;
    }
    for (int p = 5; m > 1 && p <= 1024; p += 2) {   // factors > 31: direct-DFT stage (kernels.cu stage_direct)
        while (m % p == 0) {
            radices.push_back(p);
            m /= p;
        }
    }
    return m == 1 && radices.size() <= 12;
}

int pow2_floor(int x) {
    int p = 1;
    while (p * 2 <= x) p *= 2;
    return p;
}

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    cudaError_t ensure(size_t b) {
        if (b <= bytes) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        cudaError_t e = cudaMalloc(&p, b);
        if (e == cudaSuccess) bytes = b;
        return e;
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

// Device buffer that grows in place: a virtual address range is reserved once
// for the largest size the caller may need (CUDA virtual memory management:
// cuMemAddressReserve) and physical memory is mapped behind it in chunks as
// the buffer grows (cuMemCreate + cuMemMap).  The Krylov basis uses it: its
// final size (m + 1 blocks of b vectors of 2n complex128) is unknown until
// the iteration stops, 256^3 vectors are 0.5 GiB each, and growth by copy
// would need old + new at once.  Driver entry points come through
// cudaGetDriverEntryPoint (no libcuda link dependency).
struct Vmm {
    PFN_cuMemAddressReserve reserve = nullptr;
    PFN_cuMemAddressFree free_va = nullptr;
    PFN_cuMemCreate create = nullptr;
    PFN_cuMemRelease release = nullptr;
    PFN_cuMemMap map = nullptr;
    PFN_cuMemUnmap unmap = nullptr;
    PFN_cuMemSetAccess access = nullptr;
    PFN_cuMemGetAllocationGranularity gran = nullptr;
    bool ok = false;
    static const Vmm& get() {
        static Vmm v = [] {
            Vmm x;
            auto ld = [](const char* name, void** fn) {
                cudaDriverEntryPointQueryResult q;
                return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
                       q == cudaDriverEntryPointSuccess && *fn != nullptr;
            };
            x.ok = ld("cuMemAddressReserve", (void**)&x.reserve) && ld("cuMemAddressFree", (void**)&x.free_va) &&
                   ld("cuMemCreate", (void**)&x.create) && ld("cuMemRelease", (void**)&x.release) &&
                   ld("cuMemMap", (void**)&x.map) && ld("cuMemUnmap", (void**)&x.unmap) &&
                   ld("cuMemSetAccess", (void**)&x.access) &&
                   ld("cuMemGetAllocationGranularity", (void**)&x.gran);
            return x;
        }();
        return v;
    }
};

struct GrowBuf {
    CUdeviceptr base = 0;
    size_t reserved = 0, mapped = 0, granule = 0;
    int dev = 0;
    std::vector<std::pair<CUmemGenericAllocationHandle, size_t>> chunks;
    ~GrowBuf() { clear(); }
    void clear() {
        const Vmm& v = Vmm::get();
        if (!v.ok) return;
        size_t off = 0;
        for (auto& c : chunks) {
            v.unmap(base + off, c.second);
            v.release(c.first);
            off += c.second;
        }
        chunks.clear();
        mapped = 0;
        if (base) v.free_va(base, reserved);
        base = 0;
        reserved = 0;
    }
    // reserve address space for `bytes` (drops the contents if it must re-reserve)
    int reserve(size_t bytes, int device) {
        const Vmm& v = Vmm::get();
        if (!v.ok) {
            set_error("CUDA virtual memory management entry points unavailable");
            return BNF_ECUDA;
        }
        if (base && bytes <= reserved && device == dev) return BNF_OK;
        clear();
        dev = device;
        CUmemAllocationProp prop = {};
        prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
        prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        prop.location.id = dev;
        if (v.gran(&granule, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS || granule == 0) {
            set_error("cuMemGetAllocationGranularity failed");
            return BNF_ECUDA;
        }
        const size_t r = ((bytes + granule - 1) / granule) * granule;
        if (v.reserve(&base, r, 0, 0, 0) != CUDA_SUCCESS) {
            base = 0;
            set_error("cuMemAddressReserve failed");
            return BNF_ENOMEM;
        }
        reserved = r;
        return BNF_OK;
    }
    // map physical memory so that [base, base + bytes) is usable
    int ensure(size_t bytes) {
        if (bytes <= mapped) return BNF_OK;
        if (bytes > reserved) {
            set_error("GrowBuf: request beyond the reserved range");
            return BNF_EINVAL;
        }
        const Vmm& v = Vmm::get();
        // grow by at least 1/4 of what is mapped (fewer, larger chunks), within the reservation
        size_t want = std::max(bytes - mapped, mapped / 4);
        want = ((want + granule - 1) / granule) * granule;
        want = std::min(want, reserved - mapped);
        CUmemAllocationProp prop = {};
        prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
        prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        prop.location.id = dev;
        CUmemGenericAllocationHandle h;
        if (v.create(&h, want, &prop, 0) != CUDA_SUCCESS) {
            set_error("out of device memory growing the Krylov basis (" + std::to_string((mapped + want) >> 20) +
                      " MiB)");
            return BNF_ENOMEM;
        }
        if (v.map(base + mapped, want, 0, h, 0) != CUDA_SUCCESS) {
            v.release(h);
            set_error("cuMemMap failed");
            return BNF_ECUDA;
        }
        CUmemAccessDesc acc = {};
        acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        acc.location.id = dev;
        acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        if (v.access(base + mapped, want, &acc, 1) != CUDA_SUCCESS) {
            v.unmap(base + mapped, want);
            v.release(h);
            set_error("cuMemSetAccess failed");
            return BNF_ECUDA;
        }
        chunks.push_back({h, want});
        mapped += want;
        return BNF_OK;
    }
    template <class T>
    T* as() const {
        return reinterpret_cast<T*>(base);
    }
};

// NCCL, loaded at run time (dlopen) so that the library has no link-time
// NCCL dependency: the process's already-loaded libnccl.so.2 (e.g. torch's)
// is reused, else the system one.  Distributed slab mode only.
struct Nccl {
    decltype(&ncclGetUniqueId) getUniqueId = nullptr;
    decltype(&ncclCommInitRank) commInitRank = nullptr;
    decltype(&ncclCommDestroy) commDestroy = nullptr;
    decltype(&ncclGroupStart) groupStart = nullptr;
    decltype(&ncclGroupEnd) groupEnd = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclAllReduce) allReduce = nullptr;
    decltype(&ncclAllGather) allGather = nullptr;
    decltype(&ncclGetErrorString) errStr = nullptr;
    bool ok = false;
    static const Nccl& get() {
        static Nccl x = [] {
            Nccl n;
            void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
            if (!h) h = dlopen(std::getenv("BNF_NCCL_LIB") ? std::getenv("BNF_NCCL_LIB") : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
            if (!h) return n;
            n.getUniqueId = (decltype(n.getUniqueId))dlsym(h, "ncclGetUniqueId");
            n.commInitRank = (decltype(n.commInitRank))dlsym(h, "ncclCommInitRank");
            n.commDestroy = (decltype(n.commDestroy))dlsym(h, "ncclCommDestroy");
            n.groupStart = (decltype(n.groupStart))dlsym(h, "ncclGroupStart");
            n.groupEnd = (decltype(n.groupEnd))dlsym(h, "ncclGroupEnd");
            n.send = (decltype(n.send))dlsym(h, "ncclSend");
            n.recv = (decltype(n.recv))dlsym(h, "ncclRecv");
            n.allReduce = (decltype(n.allReduce))dlsym(h, "ncclAllReduce");
            n.allGather = (decltype(n.allGather))dlsym(h, "ncclAllGather");
            n.errStr = (decltype(n.errStr))dlsym(h, "ncclGetErrorString");
            n.ok = n.getUniqueId && n.commInitRank && n.commDestroy && n.groupStart && n.groupEnd && n.send && n.recv &&
                   n.allReduce && n.allGather && n.errStr;
            return n;
        }();
        return x;
    }
};

}  // namespace

// ------------------------------------------------------------- profiler
struct Profiler {
    bool on = false;
    long long launches = 0;
    struct Rec {
        const char* name;
        cudaEvent_t a, b;
    };
    std::vector<Rec> pending;
    std::vector<cudaEvent_t> pool;
    std::map<std::string, std::pair<double, long long>> acc;
    std::vector<std::string> order;

    cudaEvent_t get() {
        if (!pool.empty()) {
            cudaEvent_t e = pool.back();
            pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        cudaEventCreate(&e);
        return e;
    }
    void flush() {
        for (auto& r : pending) {
            cudaEventSynchronize(r.b);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, r.a, r.b);
            auto it = acc.find(r.name);
            if (it == acc.end()) {
                acc[r.name] = {0.0, 0};
                order.push_back(r.name);
            }
            acc[r.name].first += ms;
            acc[r.name].second += 1;
            pool.push_back(r.a);
            pool.push_back(r.b);
        }
        pending.clear();
    }
    ~Profiler() {
        for (auto& r : pending) {
            cudaEventDestroy(r.a);
            cudaEventDestroy(r.b);
        }
        for (auto e : pool) cudaEventDestroy(e);
    }
};

}  // namespace bnf

using namespace bnf;

struct bnf_solver {
    Lattice L;
    bnf_opts o;
    cudaStream_t st = nullptr;
    long long n = 0;
    OpArgs args{};
    DevBuf root[3], root2[3], twlo, twhi;
    DevBuf eps_inv, eps_idx, eps_lut;
    bool eps_set = false;
    DevBuf sigma;
    bool kappa_set = false;
    double kappa[3] = {0, 0, 0};
    double kh2 = 0, kh3 = 0;
    DevBuf U;        // 3n per vector
    DevBuf cgx, cgr, cgp, cgmp, cgc;   // 2n per vector
    DevBuf partial;  // reduction partials
    DevBuf small;    // small device scalars/matrices
    DevBuf cgstate;
    CGState cgs{};
    DevBuf cgfuse_buf;
    CGFuse cgf{};
    bool fused_ok = false;
    bool use_plane = false;   // fused y/x/y plane pass (plane.cu)
    bool plane_ok = false;    // plane pass available for this grid
    bool plane_tuned = false; // autotune_plane done
    bool use_z2 = false;      // cp.async-staged z passes (zpass.cu)
    bool use_graph = true;    // CG loop as a CUDA graph with a device-side while node
    struct CgGraph {
        cudaGraphExec_t exec = nullptr;
        const void* X = nullptr;
        int nvec = 0;
        long long kver = -1;
        int nk = 0;
    } cgg[2];
    int cgg_next = 0;
    cudaStream_t cap = nullptr;   // capture stream
    long long kver = 0;           // bumped whenever OpArgs change (kappa, eps)
    DevBuf phasebuf;              // per-phase cycle counters (BNF_PHASE_PROF)
    DevBuf iterbuf;               // int[4]: per-call CG iterations, total iterations, total vector-iterations,
                                  // vector-iterations of still-active vectors ([4], [5]: CG partial counts)
    int* d_iter = nullptr;
    int graph_kernels_per_iter = 0;
    long long graph_calls = 0;
    DevBuf hroot;             // e^{i pi k / n3}
    GrowBuf V;             // Lanczos basis (grows with the iteration, VMM-backed)
    DevBuf lob;            // LOBPCG blocks X, AX, W, AW, P, AP and four scratch blocks (opts.method = 1)
    long long lob_fallbacks = 0;   // LOBPCG solves that fell back to inverse Lanczos
    DevBuf Wb, AZ, Yv;     // work block, A_r * Ritz, Ritz vectors
    std::vector<double> lam;
    int nev_last = 0;
    int prev_want = 0;   // Ritz vectors of the last solve kept in Yv (warm start)
    long long reorth_skipped = 0;   // DGKS second passes skipped (diagnostics)
    int* h_flags = nullptr;     // pinned
    double2* h_small = nullptr;  // pinned scratch for small matrices
    size_t h_small_cap = 0;
    int nblk = 592;
    double tol_inner_eff = 0.0;   // relaxed inner tolerance of the current Lanczos step (opts.relax_inner), 0 = tol_inner
    int nsl = 1;              // slabs of the decomposition (opts.slabs, or the ranks of bnf_solver_create_dist)
    bool dist = false;        // one slab per process (NCCL), this process = slab `rank`
    int rank = 0;
    ncclComm_t comm = nullptr;
    long long nv = 0;         // half-length of a vector held by this process (n, or n / nsl when dist)
    bool plane_t_ok = false;  // TMA plane pass available (square 64/128/256 planes, one slab)
    alignas(64) CUtensorMap tm_y, tm_x;   // TMA maps of U (plane_tma.cu), valid for (tm_base, tm_planes)
    void* tm_base = nullptr;
    long long tm_planes = 0;
    bool use_z3 = false;      // persistent TMA-pipelined adjoint z pass (zpipe.cu)
    bool alpha_fold_ok = true;   // CG alpha formed inside k_zadj2 (BNF_NO_ALPHA_FOLD=1: separate cg_alpha kernel)
    alignas(64) CUtensorMap tm_zu;        // TMA map of U for k_zadj3, valid for (tm_zu_base, tm_zu_slabs)
    void* tm_zu_base = nullptr;
    long long tm_zu_slabs = 0;
    DevBuf Ub;                // plane-side buffer of the slab exchange (3n per vector)
    Profiler prof;
    long long matvecs = 0;
    long long inner_iters = 0;
    long long active_mv = 0;      // CG applications to vectors not yet converged (host-counted part)

    ~bnf_solver() {
        if (comm) Nccl::get().commDestroy(comm);
        for (auto& c : cgg)
            if (c.exec) cudaGraphExecDestroy(c.exec);
        if (cap) cudaStreamDestroy(cap);
        if (h_flags) cudaFreeHost(h_flags);
        if (h_small) cudaFreeHost(h_small);
    }
};

namespace {

// Launch wrapper: counts kernels, optionally brackets them with events.
template <class F>
int run(bnf_solver* s, const char* name, F&& f) {
    cudaEvent_t a = nullptr, b = nullptr;
    if (s->prof.on) {
        a = s->prof.get();
        b = s->prof.get();
        cudaEventRecord(a, s->st);
    }
    cudaError_t e = f();
    s->prof.launches++;
    if (s->prof.on) {
        cudaEventRecord(b, s->st);
        s->prof.pending.push_back({name, a, b});
        if (s->prof.pending.size() > 4096) s->prof.flush();
    }
    if (e != cudaSuccess) {
        set_error(std::string("kernel ") + name + ": " + cudaGetErrorString(e));
        return BNF_ECUDA;
    }
    return BNF_OK;
}

#define RUN(name, expr)                                              \
    do {                                                             \
        int _rc = run(s, name, [&]() -> cudaError_t { return expr; }); \
        if (_rc != BNF_OK) return _rc;                               \
    } while (0)

#define TRY(expr)                   \
    do {                            \
        int _rc = (expr);           \
        if (_rc != BNF_OK) return _rc; \
    } while (0)

int ensure_small_host(bnf_solver* s, size_t count) {
    if (count <= s->h_small_cap) return BNF_OK;
    if (s->h_small) cudaFreeHost(s->h_small);
    s->h_small = nullptr;
    CK(cudaMallocHost((void**)&s->h_small, count * sizeof(double2)));
    s->h_small_cap = count;
    return BNF_OK;
}

// ------------------------------------------------------------- operator
int ensure_work(bnf_solver* s, int nvec) {
    CK(s->U.ensure((size_t)3 * s->nv * nvec * sizeof(double2)));
    if (s->nsl > 1 || s->dist) CK(s->Ub.ensure((size_t)3 * s->nv * nvec * sizeof(double2)));
    return BNF_OK;
}

// ---------------------------------------------------------- virtual slabs
// OpArgs of slab r of the slab decomposition: Fourier side =
// j-slab [r n2/P, (r+1) n2/P) of every vector, real side = z-slab of n3/P
// planes; vectors stay contiguous 2n arrays laid out [slab][half][k][jl][i]
// (Lanczos / CG BLAS are layout-agnostic), eps in [slab][l][cl][b][a].
OpArgs slab_args(const bnf_solver* s, int r) {
    OpArgs a = s->args;
    if (s->nsl == 1) return a;
    const int P = s->nsl;
    a.slab = r;
    a.nslab = P;
    a.n2loc = s->L.n[1] / P;
    a.n3loc = s->L.n[2] / P;
    a.j0 = r * a.n2loc;
    a.nloc = s->n / P;
    a.nblk = a.nloc / P;
    a.vsf = 2 * s->nv;
    if (!s->dist) {   // virtual: every slab's eps on this device, slab-major
        if (a.eps_idx) a.eps_idx += (size_t)r * 3 * a.nloc;
        if (a.eps_inv) a.eps_inv += (size_t)r * 3 * a.nloc;
    }
    return a;
}

long long sig_nloc(const bnf_solver* s) { return s->dist ? s->nv : s->n / s->nsl; }

#define NCK(call)                                                                                   \
    do {                                                                                            \
        ncclResult_t _r = (call);                                                                   \
        if (_r != ncclSuccess) {                                                                    \
            set_error(std::string("NCCL: ") + Nccl::get().errStr(_r) + " at " + #call);           \
            return BNF_ENCCL;                                                                       \
        }                                                                                           \
    } while (0)

// Distributed slab mode: the all-to-all of the slab decomposition between the
// ranks (one NCCL group of sends / receives; fwd: this rank's U block q -> rank
// q's plane buffer block `rank`; back: the reverse).  Blocks of nvec 3 nblk.
int nccl_exchange(bnf_solver* s, double2* U, double2* Ub, int nvec, int fwd) {
    const Nccl& nc = Nccl::get();
    const int P = s->nsl;
    const size_t blk = (size_t)nvec * 3 * (size_t)(s->n / P / P);
    NCK(nc.groupStart());
    for (int q = 0; q < P; ++q) {
        NCK(nc.send(fwd ? (const void*)(U + q * blk) : (const void*)(Ub + q * blk), 2 * blk, ncclFloat64, q, s->comm, s->st));
        NCK(nc.recv(fwd ? (void*)(Ub + q * blk) : (void*)(U + q * blk), 2 * blk, ncclFloat64, q, s->comm, s->st));
    }
    NCK(nc.groupEnd());
    return BNF_OK;
}

// element-wise sum over the ranks of count doubles (in place); no-op unless dist
int nccl_sum(bnf_solver* s, double* x, size_t count) {
    if (!s->dist) return BNF_OK;
    NCK(Nccl::get().allReduce(x, x, count, ncclFloat64, ncclSum, s->comm, s->st));
    return BNF_OK;
}

// CG partials [slab][vec][nb]: gather every rank's block (in place); no-op unless dist
int nccl_gather_partials(bnf_solver* s, double* part, int nvec, int nb) {
    if (!s->dist) return BNF_OK;
    const size_t cnt = (size_t)nvec * nb;
    NCK(Nccl::get().allGather(part + (size_t)s->rank * cnt, part, cnt, ncclFloat64, s->comm, s->st));
    return BNF_OK;
}

// The all-to-all of the slab decomposition as device copies: plane-side slab q
// receives, from every Fourier-side slab r, the block of its n3/P planes
// (fwd: Ub[q][r] = U[r][q]; back: U[r][q] = Ub[q][r]; blocks of nvec 3 nblk).
cudaError_t slab_exchange(bnf_solver* s, double2* U, double2* Ub, int nvec, int fwd, cudaStream_t st) {
    const int P = s->nsl;
    const size_t nloc = (size_t)(s->n / P), blk = (size_t)nvec * 3 * (nloc / P), part = (size_t)nvec * 3 * nloc;
    for (int q = 0; q < P; ++q)
        for (int r = 0; r < P; ++r) {
            double2* u = U + r * part + q * blk;
            double2* b = Ub + q * part + r * blk;
            cudaError_t e = cudaMemcpyAsync(fwd ? b : u, fwd ? u : b, blk * sizeof(double2), cudaMemcpyDeviceToDevice, st);
            if (e != cudaSuccess) return e;
        }
    return cudaSuccess;
}

const char* plane_name(const OpArgs& a, bool cg) {
    if (a.plane_t == 3) return cg ? "plane_tp_cg" : "plane_tp";
    if (a.plane_t) return a.plane_t == 2 ? (cg ? "plane_ts_cg" : "plane_ts") : (cg ? "plane_t_cg" : "plane_t");
    if (a.plane_w) return a.plane_w == 2 ? (cg ? "plane_ws_cg" : "plane_ws") : (cg ? "plane_w_cg" : "plane_w");
    if (a.plane_l2 && a.plane_split == 2) return cg ? "plane_l2s_cg" : "plane_l2s";
    if (a.plane_l2) return cg ? "plane_l2_cg" : "plane_l2";
    return cg ? "plane_cg" : "plane";
}

void* tensor_map_encoder() {
    static void* fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return f;
    }();
    return fn;
}

// the real-space middle on U (one slab): TMA plane pass, or plane.cu's variants
cudaError_t run_plane(bnf_solver* s, const OpArgs& a, double2* U, int nslab, const CGFuse* cg, cudaStream_t st) {
    if (a.plane_t) {
        const long long plane = (long long)a.mp.n1 * a.mp.n2;
        const long long planes = (long long)(s->U.bytes / sizeof(double2)) / plane;
        if (s->tm_base != s->U.p || s->tm_planes != planes) {
            if (!tensor_map_encoder() || plane_t_encode(a, s->U.p, planes, tensor_map_encoder(), &s->tm_y, &s->tm_x) != 0)
                return cudaErrorInvalidValue;
            s->tm_base = s->U.p;
            s->tm_planes = planes;
        }
        const int zbase = (int)((U - s->U.as<double2>()) / plane);
        return launch_plane_tma(a, nslab, cg, st, s->tm_y, s->tm_x, zbase);
    }
    return launch_plane(a, U, nslab, cg, st);
}

// the adjoint z pass on U (one slab): the TMA-pipelined k_zadj3 when enabled, else k_zadj2
cudaError_t run_zadj(bnf_solver* s, double2* U, double2* out, int nvec, int op, const CGFuse* cg, cudaStream_t st) {
    if (s->use_z3) {
        const long long slabs = (long long)(s->U.bytes / sizeof(double2)) / s->n;
        if (s->tm_zu_base != s->U.p || s->tm_zu_slabs != slabs) {
            if (zadj3_encode(s->args, s->U.p, slabs, tensor_map_encoder(), &s->tm_zu) != 0) return cudaErrorInvalidValue;
            s->tm_zu_base = s->U.p;
            s->tm_zu_slabs = slabs;
        }
        if (U != s->U.as<double2>()) return cudaErrorInvalidValue;
        return launch_zadj3(s->args, s->tm_zu, U, out, nvec, op, cg, st);
    }
    return launch_zadj2(s->args, U, out, nvec, op, cg, st);
}
const char* zadj_name(const bnf_solver* s, bool cg) {
    return s->use_z3 ? (cg ? "zadj3_cg" : "zadj3") : (cg ? "zadj2_cg" : "zadj2");
}

// out = op(y) for nvec vectors (device pointers, 2n each)
int apply_op(bnf_solver* s, const double2* y, double2* out, int nvec, int op) {
    TRY(ensure_work(s, nvec));
    double2* U = s->U.as<double2>();
    if (s->dist) {   // one slab per process: z pass on this j-slab, NCCL all-to-all, plane on this z-slab, back
        const OpArgs a = slab_args(s, s->rank);
        double2* Ub = s->Ub.as<double2>();
        RUN("zfwd2", launch_zfwd2(a, y, U, nvec, op, nullptr, nullptr, nullptr, s->st));
        TRY(nccl_exchange(s, U, Ub, nvec, 1));
        RUN(plane_name(a, false), launch_plane(a, Ub, 3 * nvec, nullptr, s->st));
        TRY(nccl_exchange(s, U, Ub, nvec, 0));
        RUN("zadj2", launch_zadj2(a, U, out, nvec, op, nullptr, s->st));
        s->matvecs += nvec;
        return BNF_OK;
    }
    if (s->nsl > 1) {   // virtual slabs: z pass per j-slab, exchange, plane per z-slab, exchange, adjoint z pass
        const int P = s->nsl;
        const size_t nloc = (size_t)(s->n / P), part = (size_t)nvec * 3 * nloc;
        double2* Ub = s->Ub.as<double2>();
        for (int r = 0; r < P; ++r)
            RUN("zfwd2", launch_zfwd2(slab_args(s, r), y + r * 2 * nloc, U + r * part, nvec, op, nullptr, nullptr, nullptr,
                                      s->st));
        RUN("slab_a2a", slab_exchange(s, U, Ub, nvec, 1, s->st));
        for (int q = 0; q < P; ++q)
            RUN(plane_name(s->args, false), launch_plane(slab_args(s, q), Ub + q * part, 3 * nvec, nullptr, s->st));
        RUN("slab_a2a", slab_exchange(s, U, Ub, nvec, 0, s->st));
        for (int r = 0; r < P; ++r)
            RUN("zadj2", launch_zadj2(slab_args(s, r), U + r * part, out + r * 2 * nloc, nvec, op, nullptr, s->st));
        s->matvecs += nvec;
        return BNF_OK;
    }
    if (s->use_z2) RUN("zfwd2", launch_zfwd2(s->args, y, U, nvec, op, nullptr, nullptr, nullptr, s->st));
    else RUN("zfwd", launch_zfwd(s->args, y, U, nvec, op, s->st));
    if (s->use_plane) {
        RUN(plane_name(s->args, false), run_plane(s, s->args, U, 3 * nvec, nullptr, s->st));
    } else {
        RUN("yfwd", launch_ypass(s->args, U, nvec, 0, s->st));
        RUN("xpass", launch_xpass(s->args, U, nvec, s->st));
        RUN("yadj", launch_ypass(s->args, U, nvec, 1, s->st));
    }
    if (s->use_z2) RUN(zadj_name(s, false), run_zadj(s, U, out, nvec, op, nullptr, s->st));
    else RUN("zadj", launch_zadj(s->args, U, out, nvec, op, s->st));
    s->matvecs += nvec;
    return BNF_OK;
}

// Pick the real-space middle of the operator (fused cluster plane pass vs
// separate y / x / y passes) by timing one application of each on scratch
// vectors (once per solver and block size; env BNF_PLANE / BNF_NO_PLANE force).
int autotune_plane(bnf_solver* s, int nvec) {
    if (s->plane_tuned || !s->plane_ok) return BNF_OK;
    s->plane_tuned = true;
    if (s->dist) {   // every rank must run the same passes: no per-rank timing; L2 plane (or warp-local if forced)
        s->use_plane = true;
        s->args.plane_t = 0;
        s->args.plane_w = std::getenv("BNF_PLANE_W") ? std::atoi(std::getenv("BNF_PLANE_W")) : 0;
        s->args.plane_l2 = s->args.plane_w ? 0 : 1;
        s->kver++;
        return BNF_OK;
    }
    if (std::getenv("BNF_NO_PLANE") || std::getenv("BNF_PLANE") || std::getenv("BNF_PLANE_W") ||
        std::getenv("BNF_PLANE_T")) {
        s->args.plane_l2 = std::getenv("BNF_PLANE_L2") ? std::atoi(std::getenv("BNF_PLANE_L2")) : 0;
        s->args.plane_w = std::getenv("BNF_PLANE_W") ? std::atoi(std::getenv("BNF_PLANE_W")) : 0;
        s->args.plane_t = (std::getenv("BNF_PLANE_T") && s->plane_t_ok) ? std::max(1, std::atoi(std::getenv("BNF_PLANE_T"))) : 0;
        if (s->args.plane_t == 3 && s->args.mp.n3 % 2 != 0) s->args.plane_t = 2;   // paired planes: n3 even
        if (std::getenv("BNF_NO_PLANE")) s->args.plane_w = s->args.plane_t = 0;
        s->use_plane = std::getenv("BNF_NO_PLANE") == nullptr;
        s->kver++;
        return BNF_OK;
    }
    const long long N = 2 * s->nv;
    DevBuf y, o;
    CK(y.ensure((size_t)N * nvec * sizeof(double2)));
    CK(o.ensure((size_t)N * nvec * sizeof(double2)));
    CK(cudaMemsetAsync(y.p, 0, (size_t)N * nvec * sizeof(double2), s->st));
    RUN("fill_random", launch_fill_random(y.as<double2>(), N, nvec, 12345ull, 0, nullptr, s->nv, s->st));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    // variants: 0 = y / x / y passes, 1 = cluster plane (DSMEM), 2 = plane via L2,
    // 3 / 4 = plane via L2 with warp-local FFT exchanges (shared memory / shuffles),
    // 5 / 6 = plane via L2 staged by TMA (exchange in shared memory / by warp shuffles),
    // 7 = TMA + shuffles, two planes per CTA phase-interleaved (n3 even)
    const int nvar = s->plane_t_ok ? (s->args.mp.n3 % 2 == 0 ? 8 : 7) : plane_w_supported(s->args) ? 5 : 3;
    const int v0 = s->nsl > 1 ? 2 : 0;   // slab mode: plane passes through L2 only (slab-aware)
    float best[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    const bool prof = s->prof.on;
    s->prof.on = false;
    const long long mv0 = s->matvecs;
    // 8 = plane via L2 on a cluster of two CTAs per plane (every other strip each; one slab)
    auto set = [&](int variant) {
        s->use_plane = variant >= 1;
        s->args.plane_l2 = (variant == 2 || variant == 8) ? 1 : 0;
        s->args.plane_split = variant == 8 ? 2 : 1;
        s->args.plane_w = (variant == 3 || variant == 4) ? variant - 2 : 0;
        s->args.plane_t = (variant >= 5 && variant <= 7) ? variant - 4 : 0;
    };
    const int nvar_all = s->nsl == 1 ? 9 : nvar;
    for (int variant = v0; variant < nvar_all; ++variant) {
        if (variant >= nvar && variant != 8) continue;
        if (s->nsl > 1 && variant >= 5) continue;   // TMA plane: one slab only
        set(variant);
        TRY(apply_op(s, y.as<double2>(), o.as<double2>(), nvec, BNF_OP_M));   // warm-up
        CK(cudaEventRecord(e0, s->st));
        for (int r = 0; r < 3; ++r) TRY(apply_op(s, y.as<double2>(), o.as<double2>(), nvec, BNF_OP_M));
        CK(cudaEventRecord(e1, s->st));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&best[variant], e0, e1));
    }
    int pick = v0;
    for (int variant = v0 + 1; variant < nvar_all; ++variant)
        if (best[variant] > 0.f && best[variant] < best[pick]) pick = variant;
    // the TMA-staged variants move 1.75x the algorithmic DRAM bytes of the L2 plane pass (its strips
    // re-read from HBM, profiles/r02s2_ncu.json): within 3 % of the L2 variant, keep the L2 one
    if (pick >= 5 && pick <= 7 && best[2] > 0.f && best[pick] > 0.97f * best[2]) pick = 2;
    set(pick);
    s->matvecs = mv0;
    s->prof.on = prof;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    s->kver++;   // cached CG graphs were built for the other variant
    return BNF_OK;
}

// out[g] (device double2) = X_v^* Y_v, v < nvec, vectors of length N
int dots(bnf_solver* s, const double2* X, const double2* Y, long long N, int nvec, double2* out) {
    double2* part = s->partial.as<double2>();
    RUN("dot", launch_dot_partial(X, Y, N, nvec, part, s->nblk, s->st));
    RUN("dot_final", launch_dot_final(part, s->nblk, nvec, out, s->st));
    TRY(nccl_sum(s, reinterpret_cast<double*>(out), 2 * (size_t)nvec));   // distributed vectors: sum over ranks
    return BNF_OK;
}

// H (device, p x q row-major: H[a*q + c]) = X^* Y, q <= 8
int gemm_tn(bnf_solver* s, const double2* X, int p, const double2* Y, int q, long long N, double2* H) {
    double2* part = s->partial.as<double2>();
    const size_t need = (size_t)p * q * s->nblk * sizeof(double2);
    if (need > s->partial.bytes) CK(s->partial.ensure(need));
    part = s->partial.as<double2>();
    RUN("gemm_tn", launch_gemm_tn_partial(X, p, Y, q, N, part, s->nblk, s->st));
    RUN("gemm_tn_final", launch_gemm_tn_final(part, s->nblk, p * q, H, s->st));
    return BNF_OK;
}

// ------------------------------------------------------------------ CG
// number of right-hand sides still iterating (device flags; synchronises the stream)
static int active_count(bnf_solver* s, int nvec) {
    if (cudaMemcpyAsync(s->h_flags, s->cgs.active, sizeof(int) * nvec, cudaMemcpyDeviceToHost, s->st) != cudaSuccess ||
        cudaStreamSynchronize(s->st) != cudaSuccess)
        return nvec;   // the caller's next CK reports the error
    int act = 0;
    for (int v = 0; v < nvec; ++v) act += s->h_flags[v];
    return act;
}

// Solve M X = C for nvec right-hand sides: plain CG, no
// preconditioner, per-column stopping ||r|| <= tol ||c||.
int cg_solve(bnf_solver* s, const double2* C, double2* X, int nvec, int* iters_out) {
    const long long N = 2 * s->nv;
    const size_t vb = (size_t)N * nvec * sizeof(double2);
    CK(s->cgr.ensure(vb));
    CK(s->cgp.ensure(vb));
    CK(s->cgmp.ensure(vb));
    double2* R = s->cgr.as<double2>();
    double2* P = s->cgp.as<double2>();
    double2* MP = s->cgmp.as<double2>();
    double2* dd = s->small.as<double2>();  // [0..nvec): dots
    CK(cudaMemsetAsync(X, 0, vb, s->st));
    RUN("copy", launch_copy(R, C, N * nvec, s->st));
    RUN("copy", launch_copy(P, C, N * nvec, s->st));
    TRY(dots(s, R, R, N, nvec, dd));
    RUN("cg_init", launch_cg_init(s->cgs, dd, nvec, s->tol_inner_eff > 0.0 ? s->tol_inner_eff : s->o.tol_inner, s->st));
    int it = 0;
    int act_prev = active_count(s, nvec);
    for (; it < s->o.max_inner; ++it) {
        TRY(apply_op(s, P, MP, nvec, BNF_OP_M));
        s->active_mv += act_prev;
        TRY(dots(s, P, MP, N, nvec, s->cgs.pMp));
        RUN("cg_xr", launch_cg_xr(X, R, P, MP, s->cgs, N, nvec, s->partial.as<double2>(), s->nblk, s->st));
        RUN("dot_final", launch_dot_final(s->partial.as<double2>(), s->nblk, nvec, dd, s->st));
        RUN("cg_scalars", launch_cg_scalars(s->cgs, dd, nvec, s->st));
        RUN("cg_p", launch_cg_p(P, R, s->cgs, N, nvec, s->st));
        const int act = active_count(s, nvec);
        act_prev = act;
        if (s->prof.on) s->prof.flush();
        if (act == 0) {
            ++it;
            break;
        }
    }
    s->inner_iters += (long long)it * nvec;
    if (iters_out) *iters_out = it;
    return BNF_OK;
}

// One CG iteration of cg_solve_fused on stream st (eager or under capture).
// Returns the number of kernels enqueued in *nk.
cudaError_t cg_iter_kernels(bnf_solver* s, const CGFuse& cg, double2* R, double2* P, double2* U, double2* X, int nvec,
                            cudaStream_t st, int* nk) {
    cudaError_t e;
    int k = 0;
#define BNF_K(expr)                       \
    do {                                  \
        e = (expr);                       \
        if (e != cudaSuccess) return e;   \
        ++k;                              \
    } while (0)
    if (s->dist) {   // one slab per process: NCCL all-to-alls, CG partials all-gathered across the ranks
        const OpArgs a = slab_args(s, s->rank);
        double2* Ub = s->Ub.as<double2>();
        auto ck = [&](int rc) { return rc == BNF_OK ? cudaSuccess : cudaErrorUnknown; };
        BNF_K(launch_zfwd2(a, R, U, nvec, 1, P, X, &cg, st));
        BNF_K(ck(nccl_exchange(s, U, Ub, nvec, 1)));
        BNF_K(launch_plane(a, Ub, 3 * nvec, &cg, st));
        BNF_K(ck(nccl_gather_partials(s, cg.part_x, nvec, 3 * a.n3loc)));
        BNF_K(launch_cg_finish(cg, 0, nvec, st));
        BNF_K(ck(nccl_exchange(s, U, Ub, nvec, 0)));
        BNF_K(launch_zadj2(a, U, R, nvec, 1, &cg, st));
        BNF_K(ck(nccl_gather_partials(s, cg.part_z, nvec, zpass2_tiles_x(a) * a.n2loc)));
        BNF_K(launch_cg_finish(cg, 1, nvec, st));
        *nk = k;
        return cudaSuccess;
    }
    if (s->nsl > 1) {   // virtual slabs: per-slab passes, device-copy all-to-alls
        const int NS = s->nsl;
        const size_t nloc = (size_t)(s->n / NS), part = (size_t)nvec * 3 * nloc;
        double2* Ub = s->Ub.as<double2>();
        for (int r = 0; r < NS; ++r)
            BNF_K(launch_zfwd2(slab_args(s, r), R + r * 2 * nloc, U + r * part, nvec, 1, P + r * 2 * nloc,
                               X + r * 2 * nloc, &cg, st));
        BNF_K(slab_exchange(s, U, Ub, nvec, 1, st));
        for (int q = 0; q < NS; ++q) BNF_K(launch_plane(slab_args(s, q), Ub + q * part, 3 * nvec, &cg, st));
        BNF_K(launch_cg_finish(cg, 0, nvec, st));
        BNF_K(slab_exchange(s, U, Ub, nvec, 0, st));
        for (int r = 0; r < NS; ++r)
            BNF_K(launch_zadj2(slab_args(s, r), U + r * part, R + r * 2 * nloc, nvec, 1, &cg, st));
        BNF_K(launch_cg_finish(cg, 1, nvec, st));
        *nk = k;
        return cudaSuccess;
    }
    if (s->use_z2) BNF_K(launch_zfwd2(s->args, R, U, nvec, 1, P, X, &cg, st));
    else BNF_K(launch_zfwd_cg(s->args, R, P, U, nvec, cg, st));
    if (s->use_plane) {
        BNF_K(run_plane(s, s->args, U, 3 * nvec, &cg, st));
        if (!cg.alpha_fold) BNF_K(launch_cg_finish(cg, 0, nvec, st));
    } else {
        BNF_K(launch_ypass(s->args, U, nvec, 0, st));
        BNF_K(launch_xpass_cg(s->args, U, nvec, cg, st));
        if (!cg.alpha_fold) BNF_K(launch_cg_finish(cg, 0, nvec, st));
        BNF_K(launch_ypass(s->args, U, nvec, 1, st));
    }
    if (s->use_z2) BNF_K(run_zadj(s, U, R, nvec, 1, &cg, st));
    else BNF_K(launch_zadj_cg(s->args, U, X, nvec, cg, st));
    BNF_K(launch_cg_finish(cg, 1, nvec, st));
#undef BNF_K
    *nk = k;
    return cudaSuccess;
}

// CUDA graph of the whole CG loop: a device-side WHILE node whose body is one
// CG iteration; the beta k_cg_finish after the zadj pass sets the condition (any vector
// still active and iterations < max_inner, cgfuse.cuh).  No host round trip
// per iteration.  Cached per (output block, nvec, operator version).
int cg_graph(bnf_solver* s, const CGFuse& cg0, double2* R, double2* P, double2* U, double2* X, int nvec,
             cudaGraphExec_t* out, int* nk) {
    for (auto& c : s->cgg)
        if (c.exec && c.X == X && c.nvec == nvec && c.kver == s->kver) {
            *out = c.exec;
            *nk = c.nk;
            return BNF_OK;
        }
    if (!s->cap) CK(cudaStreamCreateWithFlags(&s->cap, cudaStreamNonBlocking));
    cudaGraph_t g = nullptr;
    CK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h;
    CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = h;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    CK(cudaGraphAddNode(&node, g, nullptr, 0, &np));
    cudaGraph_t body = np.conditional.phGraph_out[0];
    CGFuse cg = cg0;
    cg.use_cond = 1;
    cg.cond = h;
    CK(cudaStreamBeginCaptureToGraph(s->cap, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    int k = 0;
    cudaError_t e = cg_iter_kernels(s, cg, R, P, U, X, nvec, s->cap, &k);
    cudaGraph_t captured = nullptr;
    cudaError_t e2 = cudaStreamEndCapture(s->cap, &captured);
    if (e != cudaSuccess || e2 != cudaSuccess) {
        cudaGraphDestroy(g);
        set_error(std::string("CG graph capture: ") + cudaGetErrorString(e != cudaSuccess ? e : e2));
        return BNF_ECUDA;
    }
    cudaGraphExec_t exec = nullptr;
    e = cudaGraphInstantiate(&exec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) {
        set_error(std::string("CG graph instantiate: ") + cudaGetErrorString(e));
        return BNF_ECUDA;
    }
    auto& slot = s->cgg[s->cgg_next];
    s->cgg_next = (s->cgg_next + 1) % 2;
    if (slot.exec) cudaGraphExecDestroy(slot.exec);
    slot.exec = exec;
    slot.X = X;
    slot.nvec = nvec;
    slot.kver = s->kver;
    slot.nk = k;
    *out = exec;
    *nk = k;
    return BNF_OK;
}

// Same CG with the vector updates and reductions fused into the operator
// passes (zfwd: x += alpha_prev p, p <- r + beta p; plane/x pass: (p, M p)
// and alpha; zadj: r -= alpha M p, (r, r) and beta).  Used when every axis
// has a register-FFT plan.  Without profiling the loop runs as one CUDA
// graph with a device-side while condition.
int cg_solve_fused(bnf_solver* s, const double2* C, double2* X, int nvec, int* iters_out) {
    const long long N = 2 * s->nv;
    const size_t vb = (size_t)N * nvec * sizeof(double2);
    CK(s->cgr.ensure(vb));
    CK(s->cgp.ensure(vb));
    TRY(ensure_work(s, nvec));
    double2* R = s->cgr.as<double2>();
    double2* P = s->cgp.as<double2>();
    double2* U = s->U.as<double2>();
    double2* dd = s->small.as<double2>();
    CK(cudaMemsetAsync(X, 0, vb, s->st));
    CK(cudaMemsetAsync(P, 0, vb, s->st));
    RUN("copy", launch_copy(R, C, N * nvec, s->st));
    TRY(dots(s, R, R, N, nvec, dd));
    RUN("cg_init", launch_cg_init(s->cgs, dd, nvec, s->tol_inner_eff > 0.0 ? s->tol_inner_eff : s->o.tol_inner, s->st));
    CK(cudaMemsetAsync(s->cgs.beta, 0, nvec * sizeof(double), s->st));
    CK(cudaMemsetAsync(s->cgf.alpha, 0, nvec * sizeof(double), s->st));
    CGFuse cg = s->cgf;
    cg.P = P;
    cg.R = R;
    // alpha / beta by k_cg_finish after the (p, M p) / (r, r) pass: the kernel boundary orders
    // the partials (no per-CTA fences or last-CTA election; an election measured no faster)
    cg.nb_x = s->d_iter + 4;
    cg.nb_z = s->d_iter + 5;
    // alpha formed inside k_zadj2 (one slab, no pipelined zadj3, not disabled by BNF_NO_ALPHA_FOLD):
    // one kernel fewer per CG iteration
    cg.alpha_fold = (s->use_z2 && !s->use_z3 && s->nsl == 1 && !s->dist && s->alpha_fold_ok) ? 1 : 0;
    int it = 0;
    if (!s->prof.on && s->use_graph) {
        cg.iter = s->d_iter;   // [3] counts the applications to still-active vectors on the device
        cg.max_iter = s->o.max_inner;
        CK(cudaMemsetAsync(s->d_iter, 0, sizeof(int), s->st));   // per-call counter; [1], [2] run on
        cudaGraphExec_t exec = nullptr;
        int nk = 0;
        TRY(cg_graph(s, cg, R, P, U, X, nvec, &exec, &nk));
        CK(cudaGraphLaunch(exec, s->st));
        s->graph_kernels_per_iter = nk;
        s->graph_calls++;
    } else {
        cg.iter = nullptr;
        int act_prev = active_count(s, nvec);
        for (; it < s->o.max_inner; ++it) {
            // eager: one timed launch per pass (profiling, bnf_kernel_times)
            if (s->nsl > 1 || s->dist) {
                int nk = 0;
                RUN("cg_iter_slabs", cg_iter_kernels(s, cg, R, P, U, X, nvec, s->st, &nk));
                s->prof.launches += nk - 1;
            } else {
            if (s->use_z2) RUN("zfwd2_cg", launch_zfwd2(s->args, R, U, nvec, 1, P, X, &cg, s->st));
            else RUN("zfwd_cg", launch_zfwd_cg(s->args, R, P, U, nvec, cg, s->st));
            if (s->use_plane) {
                RUN(plane_name(s->args, true), run_plane(s, s->args, U, 3 * nvec, &cg, s->st));
                if (!cg.alpha_fold) RUN("cg_alpha", launch_cg_finish(cg, 0, nvec, s->st));
            } else {
                RUN("yfwd", launch_ypass(s->args, U, nvec, 0, s->st));
                RUN("xpass_cg", launch_xpass_cg(s->args, U, nvec, cg, s->st));
                if (!cg.alpha_fold) RUN("cg_alpha", launch_cg_finish(cg, 0, nvec, s->st));
                RUN("yadj", launch_ypass(s->args, U, nvec, 1, s->st));
            }
            if (s->use_z2) RUN(zadj_name(s, true), run_zadj(s, U, R, nvec, 1, &cg, s->st));
            else RUN("zadj_cg", launch_zadj_cg(s->args, U, X, nvec, cg, s->st));
            RUN("cg_beta", launch_cg_finish(cg, 1, nvec, s->st));
            }
            s->matvecs += nvec;
            s->active_mv += act_prev;
            const int act = active_count(s, nvec);
            act_prev = act;
            if (s->prof.on) s->prof.flush();
            if (act == 0) {
                ++it;
                break;
            }
        }
        s->inner_iters += (long long)it * nvec;
    }
    if (s->use_z2) RUN("cg_xfinal", launch_cg_xfinal(X, P, s->cgf.alpha, N, nvec, s->st));
    if (iters_out) *iters_out = it;
    return BNF_OK;
}

// Y = Sigma^{-1} CG(M, Sigma^{-1} X)  =  A_r^{-1} X
int apply_Ar_inv(bnf_solver* s, const double2* X, double2* Y, int nvec) {
    const long long N = 2 * s->nv;
    CK(s->cgc.ensure((size_t)N * nvec * sizeof(double2)));
    double2* C = s->cgc.as<double2>();
    RUN("scale_sigma", launch_scale_sigma(X, C, s->sigma.as<double>(), s->nv, nvec, 1, s->st, sig_nloc(s)));
    if (s->fused_ok) TRY(cg_solve_fused(s, C, Y, nvec, nullptr));
    else TRY(cg_solve(s, C, Y, nvec, nullptr));
    RUN("scale_sigma", launch_scale_sigma(Y, Y, s->sigma.as<double>(), s->nv, nvec, 1, s->st, sig_nloc(s)));
    return BNF_OK;
}

// Copy a p x q device matrix to host (row-major)
int get_small(bnf_solver* s, const double2* dev, int count, std::vector<cd>& out) {
    TRY(ensure_small_host(s, count));
    CK(cudaMemcpyAsync(s->h_small, dev, count * sizeof(double2), cudaMemcpyDeviceToHost, s->st));
    CK(cudaStreamSynchronize(s->st));
    out.resize(count);
    for (int i = 0; i < count; ++i) out[i] = cd(s->h_small[i].x, s->h_small[i].y);
    return BNF_OK;
}

int put_small(bnf_solver* s, const std::vector<cd>& in, double2* dev) {
    TRY(ensure_small_host(s, in.size()));
    for (size_t i = 0; i < in.size(); ++i) s->h_small[i] = make_double2(in[i].real(), in[i].imag());
    CK(cudaMemcpyAsync(dev, s->h_small, in.size() * sizeof(double2), cudaMemcpyHostToDevice, s->st));
    CK(cudaStreamSynchronize(s->st));
    return BNF_OK;
}

// H = X^* Y for q possibly > 8 (column chunks); host result p x q row-major
int gram_host(bnf_solver* s, const double2* X, int p, const double2* Y, int q, std::vector<cd>& H) {
    const long long N = 2 * s->nv;
    H.assign((size_t)p * q, 0.0);
    double2* Hd = s->small.as<double2>() + 64;
    std::vector<cd> tmp;
    for (int c0 = 0; c0 < q; c0 += 8) {
        const int qc = std::min(8, q - c0);
        TRY(gemm_tn(s, X, p, Y + (size_t)c0 * N, qc, N, Hd));
        TRY(nccl_sum(s, reinterpret_cast<double*>(Hd), 2 * (size_t)p * qc));   // distributed vectors: sum over ranks
        TRY(get_small(s, Hd, p * qc, tmp));
        for (int a = 0; a < p; ++a)
            for (int c = 0; c < qc; ++c) H[(size_t)a * q + c0 + c] = tmp[(size_t)a * qc + c];
    }
    return BNF_OK;
}

// Y[:, c] = beta Y[:, c] + alpha X H[:, c]  (H host p x q row-major; column chunks of 8)
int gemm_nn_host(bnf_solver* s, const double2* X, int p, const std::vector<cd>& H, int q, double2* Y, double alpha,
                 double beta) {
    const long long N = 2 * s->nv;
    double2* Hd = s->small.as<double2>() + 64;
    for (int c0 = 0; c0 < q; c0 += 8) {
        const int qc = std::min(8, q - c0);
        std::vector<cd> sub((size_t)p * qc);
        for (int a = 0; a < p; ++a)
            for (int c = 0; c < qc; ++c) sub[(size_t)a * qc + c] = H[(size_t)a * q + c0 + c];
        TRY(put_small(s, sub, Hd));
        RUN("gemm_nn", launch_gemm_nn(X, p, Hd, qc, Y + (size_t)c0 * N, N, alpha, beta, s->st));
    }
    return BNF_OK;
}

// Orthonormalise the q columns of W (in place) by Cholesky-QR twice.
// Returns R (q x q, upper) with W_in = W_out R.  ok=false on rank deficiency.
int chol_qr2(bnf_solver* s, double2* W, int q, std::vector<cd>& Rtot, bool& ok) {
    ok = true;
    Rtot.assign((size_t)q * q, 0.0);
    for (int i = 0; i < q; ++i) Rtot[(size_t)i * q + i] = 1.0;
    for (int pass = 0; pass < 2; ++pass) {
        std::vector<cd> G, R, Ri;
        TRY(gram_host(s, W, q, W, q, G));
        for (int i = 0; i < q; ++i)
            for (int j = 0; j < i; ++j) G[(size_t)i * q + j] = std::conj(G[(size_t)j * q + i]);
        if (!cholesky_upper(q, G, R)) {
            ok = false;
            return BNF_OK;
        }
        inv_upper(q, R, Ri);
        if (q <= 8) {
            TRY(gemm_nn_host(s, W, q, Ri, q, W, 1.0, 0.0));  // in place is safe for one column chunk
        } else {
            const long long N = 2 * s->nv;
            CK(s->cgc.ensure((size_t)N * q * sizeof(double2)));
            TRY(gemm_nn_host(s, W, q, Ri, q, s->cgc.as<double2>(), 1.0, 0.0));
            RUN("copy", launch_copy(W, s->cgc.as<double2>(), N * q, s->st));
        }
        std::vector<cd> Rn((size_t)q * q, 0.0);
        for (int i = 0; i < q; ++i)
            for (int j = 0; j < q; ++j) {
                cd acc = 0.0;
                for (int k = 0; k < q; ++k) acc += R[(size_t)i * q + k] * Rtot[(size_t)k * q + j];
                Rn[(size_t)i * q + j] = acc;
            }
        Rtot.swap(Rn);
    }
    return BNF_OK;
}

int set_kappa_impl(bnf_solver* s, const double kappa[3]) {
    const Lattice& L = s->L;
    const int n1 = L.n[0], n2 = L.n[1], n3 = L.n[2];
    const int m1 = L.m[0], m2 = L.m[1], m3 = L.m[2];
    const int r1 = L.rho[0], r2 = L.rho[1], r3 = L.rho[2];
    const double k1 = kappa[0], k2 = kappa[1], k3 = kappa[2];
    // kappa-hat (Thm eigK2; Thms eigK3 P:L1733/L1872, SURVEY §8 notation)
    const double kh2 = k2 - ((double)m1 / n1) * k1 + r1 * k1;
    const double kh3 = k3 - ((double)m2 / n1) * k1 + r2 * k1 - ((double)m3 / n2) * kh2 + r3 * kh2;
    s->kappa[0] = k1;
    s->kappa[1] = k2;
    s->kappa[2] = k3;
    s->kh2 = kh2;
    s->kh3 = kh3;
    ModeP& p = s->args.mp;
    p.kap1 = k1;
    p.kh2 = kh2;
    p.kh3 = kh3;
    p.gamma = -1;
    const bool integral = (k1 == std::floor(k1)) && (k2 == std::floor(k2)) && (k3 == std::floor(k3));
    if (integral) {
        // Gamma (R6): the mode with g = 0 mod 1, by exact integer arithmetic.
        const long long K1 = (long long)k1, K2 = (long long)k2, K3 = (long long)k3;
        const long long n = s->n, n12 = (long long)n1 * n2;
        long long i0 = ((-K1) % n1 + n1) % n1;
        const long long t1 = (i0 + K1) / n1;  // exact
        const long long jnum = (long long)m1 * t1 - K2 - (long long)r1 * K1;
        long long j0 = ((jnum % n2) + n2) % n2;
        // n g3 = n1n2 k - n1 m3 j + cb' i + n1n2 kh3, with n1n2 kh3 integral
        const long long n1kh2 = (long long)n1 * K2 - (long long)m1 * K1 + (long long)r1 * n1 * K1;
        const long long n12kh3 = n12 * K3 - (long long)n2 * m2 * K1 + n12 * r2 * K1 - (long long)m3 * n1kh2 +
                                 (long long)n2 * r3 * n1kh2;
        const long long cb = (long long)m1 * m3 - (long long)n2 * m2 - (long long)r3 * n2 * m1;
        long long rest = (long long)n1 * m3 * j0 - cb * i0 - n12kh3;  // must be n12 * k0 mod n
        long long k0 = -1;
        if (rest % n12 == 0) {
            k0 = ((rest / n12) % n3 + n3) % n3;
        } else {
            set_error("internal: Gamma mode not integral");
            return BNF_EINVAL;
        }
        p.gamma = i0 + (long long)n1 * (j0 + (long long)n2 * k0);
    }
    if (s->dist)   // this rank's j-slab
        RUN("sigma_table", launch_sigma_table(p, s->sigma.as<double>(), s->st, s->rank * (s->L.n[1] / s->nsl),
                                              s->L.n[1] / s->nsl, s->nv));
    else
        RUN("sigma_table", launch_sigma_table(p, s->sigma.as<double>(), s->st, 0, s->L.n[1] / s->nsl, s->n));
    s->kappa_set = true;
    s->kver++;
    return BNF_OK;
}

}  // namespace

namespace {
// ------------------------------------------------------------------ LOBPCG
// NEXT-1 eigensolver variant (opts.method = 1; SURVEY §8(f), P:L2252-2260 for
// the operator): locally optimal block preconditioned CG on A_r itself, no
// inner solves, preconditioned by Sigma_r^{-2} (A_r = Sigma_r M Sigma_r, so the
// preconditioned operator is similar to M, kappa <= max eps / min eps).
// Knyazev's LOBPCG with soft locking (converged columns stay in the
// Rayleigh-Ritz basis, only active residuals are preconditioned and applied),
// X / W / P blocks each orthonormalised by Cholesky-QR, W orthogonalised to X,
// Rayleigh-Ritz on [X W P] as a generalized Hermitian eigenproblem on the host
// (P is dropped for one step if its Gram matrix is numerically singular).  A
// pair is converged when ||A_r x - theta x|| <= res_tol (unit x): the
// north-star residual bar, which also bounds the eigenvalue error by
// ||r||^2 / gap.
int lobpcg_solve(bnf_solver* s, int nev, int want, double* lambda, double& maxres_out, int& iters_out,
                 bool& converged) {
    const long long N = 2 * s->nv;
    const int m = want;
    const size_t vb = (size_t)N * sizeof(double2);
    CK(s->lob.ensure(vb * (size_t)m * 10));
    double2* base = s->lob.as<double2>();
    double2* X = base;
    double2* AX = base + (size_t)m * N;
    double2* W = base + (size_t)2 * m * N;
    double2* AW = base + (size_t)3 * m * N;
    double2* P = base + (size_t)4 * m * N;
    double2* AP = base + (size_t)5 * m * N;
    double2* T1 = base + (size_t)6 * m * N;
    double2* T2 = base + (size_t)7 * m * N;
    double2* T3 = base + (size_t)8 * m * N;
    double2* T4 = base + (size_t)9 * m * N;
    CK(s->small.ensure((size_t)(64 + 8 * 3 * m) * sizeof(double2)));
    // start block: previous Ritz vectors (warm) or seeded normals, Gamma mode masked
    RUN("fill_random", launch_fill_random(X, N, m, s->o.seed, (long long)s->rank * N * m, s->sigma.as<double>(), s->nv,
                                          s->st, sig_nloc(s)));
    if (s->o.warm && s->prev_want > 0) {
        const int c = std::min(s->prev_want, m);
        RUN("copy", launch_copy(X, s->Yv.as<double2>(), N * c, s->st));
        RUN("scale_sigma", launch_scale_sigma(X, X, s->sigma.as<double>(), s->nv, c, 1, s->st, sig_nloc(s)));
        RUN("scale_sigma", launch_scale_sigma(X, X, s->sigma.as<double>(), s->nv, c, 0, s->st, sig_nloc(s)));
    }
    bool ok = true;
    std::vector<cd> Rq;
    TRY(chol_qr2(s, X, m, Rq, ok));
    if (!ok) {
        set_error("LOBPCG start block rank deficient");
        return BNF_ENOCONV;
    }
    TRY(apply_op(s, X, AX, m, BNF_OP_AR));
    // Rayleigh-Ritz on X
    std::vector<double> theta;
    {
        std::vector<cd> H, Z;
        TRY(gram_host(s, X, m, AX, m, H));
        for (int i = 0; i < m; ++i)
            for (int j = i; j < m; ++j) {
                const cd h = 0.5 * (H[(size_t)i * m + j] + std::conj(H[(size_t)j * m + i]));
                H[(size_t)i * m + j] = h;
                H[(size_t)j * m + i] = std::conj(h);
            }
        herm_eig(m, H, theta, &Z);
        TRY(gemm_nn_host(s, X, m, Z, m, T1, 1.0, 0.0));
        TRY(gemm_nn_host(s, AX, m, Z, m, T2, 1.0, 0.0));
        std::swap(X, T1);
        std::swap(AX, T2);
    }
    const int maxit = s->o.max_outer > 0 ? s->o.max_outer : 1000;
    bool have_p = false;
    std::vector<int> pact;   // columns of P / AP that are valid (all m after the first update)
    double maxres = 0.0;
    int it = 0;
    converged = false;
    double2* dd = s->small.as<double2>();
    for (; it < maxit; ++it) {
        // residuals R = AX - X diag(theta) (into T1) and their norms
        RUN("copy", launch_copy(T1, AX, N * m, s->st));
        {
            std::vector<cd> Dl((size_t)m * m, 0.0);
            for (int c = 0; c < m; ++c) Dl[(size_t)c * m + c] = -theta[c];
            TRY(gemm_nn_host(s, X, m, Dl, m, T1, 1.0, 1.0));
        }
        TRY(dots(s, T1, T1, N, m, dd));
        std::vector<cd> rr;
        TRY(get_small(s, dd, m, rr));
        std::vector<int> act;
        maxres = 0.0;
        // converged: ||r|| <= min(res_tol, 1e-9 max(1, theta)) -- the north-star residual bar, tight
        // enough that the eigenvalue error ||r||^2 / gap stays far below 1e-10 relative even for
        // clustered bands, and above the round-off floor of forming R (eps ||A_r||)
        bool bad = false;
        for (int c = 0; c < m; ++c) {
            const double r = std::sqrt(std::fabs(rr[c].real()));
            if (!std::isfinite(r)) bad = true;
            if (c < nev) maxres = std::max(maxres, r);
            if (r > std::min(s->o.res_tol, 1e-9 * std::max(1.0, std::fabs(theta[c])))) act.push_back(c);
        }
        if (bad) break;
        bool wanted_done = true;
        for (int c : act)
            if (c < nev) wanted_done = false;
        if (wanted_done) {
            converged = true;
            break;
        }
        const int k = (int)act.size();
        // W = T R_active, T = Sigma_r^{-2} (Gamma masked)
        for (int q = 0; q < k; ++q) RUN("copy", launch_copy(W + (size_t)q * N, T1 + (size_t)act[q] * N, N, s->st));
        RUN("scale_sigma", launch_scale_sigma(W, W, s->sigma.as<double>(), s->nv, k, 1, s->st, sig_nloc(s)));
        RUN("scale_sigma", launch_scale_sigma(W, W, s->sigma.as<double>(), s->nv, k, 1, s->st, sig_nloc(s)));
        // W <- W - X (X^* W), twice; orthonormalise
        for (int pass = 0; pass < 2; ++pass) {
            std::vector<cd> Hxw;
            TRY(gram_host(s, X, m, W, k, Hxw));
            TRY(gemm_nn_host(s, X, m, Hxw, k, W, -1.0, 1.0));
        }
        TRY(chol_qr2(s, W, k, Rq, ok));
        if (!ok) break;   // stagnation: keep the current Ritz pairs
        TRY(apply_op(s, W, AW, k, BNF_OP_AR));
        // P restricted to the active columns, orthonormalised (AP transformed alike)
        int kp = 0;
        if (have_p) {
            for (int q = 0; q < k; ++q) {
                RUN("copy", launch_copy(T3 + (size_t)q * N, P + (size_t)act[q] * N, N, s->st));
                RUN("copy", launch_copy(T4 + (size_t)q * N, AP + (size_t)act[q] * N, N, s->st));
            }
            std::vector<cd> Rp, Rpi;
            TRY(chol_qr2(s, T3, k, Rp, ok));
            if (ok) {
                inv_upper(k, Rp, Rpi);
                TRY(gemm_nn_host(s, T4, k, Rpi, k, T2, 1.0, 0.0));
                RUN("copy", launch_copy(T4, T2, N * k, s->st));
                kp = k;
            }
        }
        // Gram matrices of S = [X W P] (orthonormal blocks; X^* W = 0)
        auto assemble = [&](int kpu, std::vector<cd>& GA, std::vector<cd>& GB) -> int {
            const int sz = m + k + kpu;
            GA.assign((size_t)sz * sz, 0.0);
            GB.assign((size_t)sz * sz, 0.0);
            for (int i = 0; i < sz; ++i) GB[(size_t)i * sz + i] = 1.0;
            for (int i = 0; i < m; ++i) GA[(size_t)i * sz + i] = theta[i];
            std::vector<cd> H;
            auto put = [&](std::vector<cd>& G, int r0, int c0, int pr, int qc, const std::vector<cd>& B) {
                for (int a = 0; a < pr; ++a)
                    for (int c = 0; c < qc; ++c) {
                        G[(size_t)(r0 + a) * sz + c0 + c] = B[(size_t)a * qc + c];
                        G[(size_t)(c0 + c) * sz + r0 + a] = std::conj(B[(size_t)a * qc + c]);
                    }
            };
            TRY(gram_host(s, X, m, AW, k, H));
            put(GA, 0, m, m, k, H);
            TRY(gram_host(s, W, k, AW, k, H));
            for (int a = 0; a < k; ++a)
                for (int c = a; c < k; ++c) {
                    const cd h = 0.5 * (H[(size_t)a * k + c] + std::conj(H[(size_t)c * k + a]));
                    GA[(size_t)(m + a) * sz + m + c] = h;
                    GA[(size_t)(m + c) * sz + m + a] = std::conj(h);
                }
            if (kpu > 0) {
                TRY(gram_host(s, X, m, T4, kpu, H));
                put(GA, 0, m + k, m, kpu, H);
                TRY(gram_host(s, W, k, T4, kpu, H));
                put(GA, m, m + k, k, kpu, H);
                TRY(gram_host(s, T3, kpu, T4, kpu, H));
                for (int a = 0; a < kpu; ++a)
                    for (int c = a; c < kpu; ++c) {
                        const cd h = 0.5 * (H[(size_t)a * kpu + c] + std::conj(H[(size_t)c * kpu + a]));
                        GA[(size_t)(m + k + a) * sz + m + k + c] = h;
                        GA[(size_t)(m + k + c) * sz + m + k + a] = std::conj(h);
                    }
                TRY(gram_host(s, X, m, T3, kpu, H));
                put(GB, 0, m + k, m, kpu, H);
                TRY(gram_host(s, W, k, T3, kpu, H));
                put(GB, m, m + k, k, kpu, H);
            }
            return BNF_OK;
        };
        std::vector<cd> GA, GB, RB, RBi;
        TRY(assemble(kp, GA, GB));
        int sz = m + k + kp;
        if (!cholesky_upper(sz, GB, RB)) {   // P numerically dependent: Rayleigh-Ritz on [X W] only
            kp = 0;
            TRY(assemble(0, GA, GB));
            sz = m + k;
            if (!cholesky_upper(sz, GB, RB)) break;
        }
        inv_upper(sz, RB, RBi);
        // standard form RB^{-H} GA RB^{-1}
        std::vector<cd> T((size_t)sz * sz, 0.0), A2((size_t)sz * sz, 0.0);
        for (int i = 0; i < sz; ++i)
            for (int j = 0; j < sz; ++j) {
                cd acc = 0.0;
                for (int l = 0; l <= j; ++l) acc += GA[(size_t)i * sz + l] * RBi[(size_t)l * sz + j];
                T[(size_t)i * sz + j] = acc;
            }
        for (int i = 0; i < sz; ++i)
            for (int j = 0; j < sz; ++j) {
                cd acc = 0.0;
                for (int l = 0; l <= i; ++l) acc += std::conj(RBi[(size_t)l * sz + i]) * T[(size_t)l * sz + j];
                A2[(size_t)i * sz + j] = acc;
            }
        for (int i = 0; i < sz; ++i)
            for (int j = i; j < sz; ++j) {
                const cd h = 0.5 * (A2[(size_t)i * sz + j] + std::conj(A2[(size_t)j * sz + i]));
                A2[(size_t)i * sz + j] = h;
                A2[(size_t)j * sz + i] = std::conj(h);
            }
        std::vector<double> w;
        std::vector<cd> Z;
        herm_eig(sz, A2, w, &Z);
        // C = RB^{-1} Z[:, :m]
        std::vector<cd> Cx((size_t)m * m), Cw((size_t)k * m), Cp((size_t)std::max(kp, 1) * m);
        for (int i = 0; i < sz; ++i)
            for (int c = 0; c < m; ++c) {
                cd acc = 0.0;
                for (int l = i; l < sz; ++l) acc += RBi[(size_t)i * sz + l] * Z[(size_t)l * sz + c];
                if (i < m) Cx[(size_t)i * m + c] = acc;
                else if (i < m + k) Cw[(size_t)(i - m) * m + c] = acc;
                else Cp[(size_t)(i - m - k) * m + c] = acc;
            }
        // P_new = W Cw + P Cp; AP_new = AW Cw + AP Cp (into T1 / T2, then into P / AP)
        TRY(gemm_nn_host(s, W, k, Cw, m, T1, 1.0, 0.0));
        TRY(gemm_nn_host(s, AW, k, Cw, m, T2, 1.0, 0.0));
        if (kp > 0) {
            TRY(gemm_nn_host(s, T3, kp, Cp, m, T1, 1.0, 1.0));
            TRY(gemm_nn_host(s, T4, kp, Cp, m, T2, 1.0, 1.0));
        }
        // X_new = X Cx + P_new; AX_new = AX Cx + AP_new
        TRY(gemm_nn_host(s, X, m, Cx, m, T3, 1.0, 0.0));
        TRY(gemm_nn_host(s, AX, m, Cx, m, T4, 1.0, 0.0));
        RUN("copy", launch_copy(P, T1, N * m, s->st));
        RUN("copy", launch_copy(AP, T2, N * m, s->st));
        std::swap(X, T3);
        std::swap(AX, T4);
        // X += P_new, AX += AP_new  (beta-accumulate through an identity product)
        {
            std::vector<cd> I((size_t)m * m, 0.0);
            for (int c = 0; c < m; ++c) I[(size_t)c * m + c] = 1.0;
            TRY(gemm_nn_host(s, P, m, I, m, X, 1.0, 1.0));
            TRY(gemm_nn_host(s, AP, m, I, m, AX, 1.0, 1.0));
        }
        theta.assign(w.begin(), w.begin() + m);
        have_p = true;
    }
    // final Ritz pairs: Y = X (unit columns), lambda = theta
    CK(s->Yv.ensure(vb * want));
    RUN("copy", launch_copy(s->Yv.as<double2>(), X, N * want, s->st));
    for (int c = 0; c < nev; ++c) lambda[c] = theta[c];
    s->lam.assign(theta.begin(), theta.begin() + nev);
    maxres_out = maxres;
    iters_out = it;
    return BNF_OK;
}
}  // namespace

// ======================================================================= C ABI
extern "C" {

const char* bnf_last_error(void) { return g_err.c_str(); }
int bnf_version(void) { return BNF_VERSION; }

int bnf_lattice_create(const double a_raw[9], const int n[3], bnf_lattice** out) {
    if (!a_raw || !n || !out) {
        set_error("NULL argument");
        return BNF_EINVAL;
    }
    auto* l = new (std::nothrow) bnf_lattice;
    if (!l) return BNF_ENOMEM;
    int rc = lattice_snap(a_raw, n, l->L);
    if (rc != BNF_OK) {
        delete l;
        return rc;
    }
    *out = l;
    return BNF_OK;
}

int bnf_lattice_query(const bnf_lattice* lat, bnf_lattice_info* info) {
    if (!lat || !info) {
        set_error("NULL argument");
        return BNF_EINVAL;
    }
    const Lattice& L = lat->L;
    for (int d = 0; d < 3; ++d) {
        info->n[d] = L.n[d];
        info->perm[d] = L.perm[d];
        info->m[d] = L.m[d];
        info->rho[d] = L.rho[d];
        info->lengths[d] = L.lengths[d];
        info->cos_raw[d] = L.cos_raw[d];
        info->cos_snap[d] = L.cos_snap[d];
        info->l[d] = L.l[d];
        info->delta[d] = L.delta[d];
    }
    info->sign3 = L.sign3;
    info->category = j3_category(L);
    std::memcpy(info->a, L.a, sizeof(L.a));
    std::memcpy(info->a_canon, L.a_canon, sizeof(L.a_canon));
    std::memcpy(info->Ag, L.Ag, sizeof(L.Ag));
    return BNF_OK;
}

void bnf_lattice_destroy(bnf_lattice* lat) { delete lat; }

int bnf_kvec_reduce(const bnf_lattice* lat, const double K[3], double kappa[3]) {
    if (!lat || !K || !kappa) {
        set_error("NULL argument");
        return BNF_EINVAL;
    }
    for (int l = 0; l < 3; ++l) {
        const double* a = lat->L.a_canon + 3 * l;
        kappa[l] = (K[0] * a[0] + K[1] * a[1] + K[2] * a[2]) / (2.0 * 3.14159265358979323846);
    }
    return BNF_OK;
}

int bnf_kappa_canonical(const bnf_lattice* lat, const double kappa_raw[3], double kappa[3]) {
    if (!lat || !kappa_raw || !kappa) {
        set_error("NULL argument");
        return BNF_EINVAL;
    }
    // canonical vector l is raw vector perm[l]; a3 negated when sign3 = -1 (R10)
    const Lattice& L = lat->L;
    double k[3];
    for (int l = 0; l < 3; ++l) k[l] = kappa_raw[L.perm[l]];
    k[2] *= (double)L.sign3;
    for (int l = 0; l < 3; ++l) kappa[l] = k[l];
    return BNF_OK;
}

int bnf_yee_points(const bnf_lattice* lat, int comp, int frame, double* xyz) {
    if (!lat || !xyz) {
        set_error("NULL argument");
        return BNF_EINVAL;
    }
    if (comp < 0 || comp > 2 || (frame != BNF_FRAME_SNAPPED && frame != BNF_FRAME_ORIGINAL)) {
        set_error("bnf_yee_points: comp must be 0..2 and frame BNF_FRAME_SNAPPED or BNF_FRAME_ORIGINAL");
        return BNF_EINVAL;
    }
    const Lattice& L = lat->L;
    const int n1 = L.n[0], n2 = L.n[1], n3 = L.n[2];
    // a (snapped, upper triangular, columns a[3*l + r]) inverse by back substitution
    const double* A = L.a;
    const double a11 = A[0], a12 = A[3], a13 = A[6], a22 = A[4], a23 = A[7], a33 = A[8];
    size_t q = 0;
    for (int c = 0; c < n3; ++c)
        for (int b = 0; b < n2; ++b)
            for (int a = 0; a < n1; ++a, ++q) {
                const double x = (a + (comp == 0 ? 0.5 : 0.0)) * L.delta[0];
                const double y = (b + (comp == 1 ? 0.5 : 0.0)) * L.delta[1];
                const double z = (c + (comp == 2 ? 0.5 : 0.0)) * L.delta[2];
                double* o = xyz + 3 * q;
                if (frame == BNF_FRAME_SNAPPED) {
                    o[0] = x;
                    o[1] = y;
                    o[2] = z;
                    continue;
                }
                // fractional coordinates f = a^{-1} (x, y, z), wrapped into [0, 1)
                double f3 = z / a33;
                double f2 = (y - a23 * f3) / a22;
                double f1 = (x - a12 * f2 - a13 * f3) / a11;
                f1 -= std::floor(f1);
                f2 -= std::floor(f2);
                f3 -= std::floor(f3);
                for (int r = 0; r < 3; ++r)
                    o[r] = L.a_canon[r] * f1 + L.a_canon[3 + r] * f2 + L.a_canon[6 + r] * f3;
            }
    return BNF_OK;
}

void bnf_opts_default(bnf_opts* o) {
    if (!o) return;
    std::memset(o, 0, sizeof(*o));
    o->device = 0;
    o->stream = nullptr;
    o->tol_outer = 1e-12;
    o->tol_inner = 1e-13;
    o->max_outer = 0;   // auto: max(60, 12 ceil((nev + guard) / block)) steps
    o->max_inner = 2000;
    o->block = 4;
    o->guard = 4;
    o->seed = 0x5EEDull;
    o->refine = 1;
    o->profile = 0;
    o->warm = 0;
    o->reorth_once_ok = 1;
    o->res_tol = 5e-9;
    o->max_polish = 3;
    o->slabs = 1;
    o->relax_inner = 0;
    o->method = 0;
}

int bnf_solver_create(const bnf_lattice* lat, const bnf_opts* opts, bnf_solver** out) {
    if (!lat || !out) {
        set_error("NULL argument");
        return BNF_EINVAL;
    }
    bnf_opts o;
    bnf_opts_default(&o);
    if (opts) o = *opts;
    if (o.block < 1 || o.block > 8 || o.guard < 0 || o.max_outer < 0 || o.max_inner < 1) {
        set_error("invalid solver options (block must be 1..8)");
        return BNF_EINVAL;
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        set_error("no CUDA device available (the solver has no CPU fallback)");
        return BNF_ECUDA;
    }
    std::unique_ptr<bnf_solver> s(new (std::nothrow) bnf_solver);
    if (!s) return BNF_ENOMEM;
    s->L = lat->L;
    s->o = o;
    CK(cudaSetDevice(o.device));
    s->st = (cudaStream_t)o.stream;
    s->prof.on = o.profile != 0;
    const Lattice& L = s->L;
    const int n1 = L.n[0], n2 = L.n[1], n3 = L.n[2];
    s->n = (long long)n1 * n2 * n3;
    s->nv = s->n;
    const long long n = s->n;
    // axis plans + root tables
    AxisPlan* plans[3] = {&s->args.px, &s->args.py, &s->args.pz};
    for (int d = 0; d < 3; ++d) {
        std::vector<int> rad;
        if (!make_plan(L.n[d], rad)) {
            set_error("axis length " + std::to_string(L.n[d]) + " unsupported (need 1 <= length <= 1024)");
            return BNF_EINVAL;
        }
        AxisPlan& pl = *plans[d];
        pl.N = L.n[d];
        pl.nst = (int)rad.size();
        for (size_t i = 0; i < rad.size(); ++i) pl.R[i] = rad[i];
        std::vector<double2> h(pl.N);
        for (int t = 0; t < pl.N; ++t) h[t] = unit_root(t, pl.N);
        CK(s->root[d].ensure(pl.N * sizeof(double2)));
        CK(cudaMemcpy(s->root[d].p, h.data(), pl.N * sizeof(double2), cudaMemcpyHostToDevice));
        pl.root = s->root[d].as<double2>();
        // fast-plan stage twiddles [k1][t] (N = N1 * N2, fastfft.cuh); same split as the kernels' plans
        const int n2f = fast_split_N2(pl.N);
        if (n2f > 0) {
            const int n1f = pl.N / n2f;
            std::vector<double2> h2((size_t)n1f * n2f);
            for (int k1 = 0; k1 < n1f; ++k1)
                for (int t = 0; t < n2f; ++t) h2[(size_t)k1 * n2f + t] = unit_root((long long)t * k1, pl.N);
            CK(s->root2[d].ensure(h2.size() * sizeof(double2)));
            CK(cudaMemcpy(s->root2[d].p, h2.data(), h2.size() * sizeof(double2), cudaMemcpyHostToDevice));
            pl.root2 = s->root2[d].as<double2>();
        }
    }
    // two-level table of e^{2 pi i P / n}
    int shift = 0;
    while ((1LL << (2 * shift)) < n) ++shift;
    const long long nlo = 1LL << shift, nhi = (n + nlo - 1) / nlo;
    {
        std::vector<double2> lo(nlo), hi(nhi);
        for (long long t = 0; t < nlo; ++t) lo[t] = unit_root(t, n);
        for (long long t = 0; t < nhi; ++t) hi[t] = unit_root(t * nlo, n);
        CK(s->twlo.ensure(nlo * sizeof(double2)));
        CK(s->twhi.ensure(nhi * sizeof(double2)));
        CK(cudaMemcpy(s->twlo.p, lo.data(), nlo * sizeof(double2), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(s->twhi.p, hi.data(), nhi * sizeof(double2), cudaMemcpyHostToDevice));
    }
    TwP& tw = s->args.tw;
    tw.lo = s->twlo.as<double2>();
    tw.hi = s->twhi.as<double2>();
    tw.shift = shift;
    tw.mask = (unsigned long long)(nlo - 1);
    ModeP& p = s->args.mp;
    p.n1 = n1;
    p.n2 = n2;
    p.n3 = n3;
    p.n = n;
    p.n12 = (long long)n1 * n2;
    p.m1 = L.m[0];
    p.m3 = L.m[2];
    long long cb = (long long)L.m[0] * L.m[2] - (long long)n2 * L.m[1] - (long long)L.rho[2] * n2 * L.m[0];
    p.cbp = ((cb % n) + n) % n;
    p.n1m3 = ((long long)n1 * L.m[2]) % n;
    for (int d = 0; d < 3; ++d) p.idelta[d] = 1.0 / L.delta[d];
    p.gamma = -1;
    p.taup = 1e-6;
    s->args.inv_n = 1.0 / (double)n;
    s->args.j0 = 0;           // whole grid: one slab
    s->args.n2loc = n2;
    s->args.n3loc = n3;
    s->args.slab = 0;
    s->args.nslab = 1;
    s->args.nloc = n;
    s->args.vsf = 2 * n;
    s->args.nblk = n;
    // z-pass variant (kernels.cuh): default = register prefetch of the CG residual in zadj2
    // (128^3, b = 2: 143 vs 149 us, profiles/r02_*) + the CG x tile staged with r, p in zfwd2 (bit 0:
    // 176 vs 182 us at b = 2 once the stage roots moved to shared memory, profiles/r02s2_plane_options.jsonl)
    s->args.zcfg = std::getenv("BNF_ZCFG") ? std::atoi(std::getenv("BNF_ZCFG")) : 5;
    s->args.fast = (std::getenv("BNF_NO_FAST") == nullptr) ? 1 : 0;
    // tile widths: keep each kernel's shared memory <= ~100 KB
    const int budget = 100 * 1024;
    s->args.W_z = std::max(1, std::min(16, pow2_floor(budget / (4 * 16 * n3))));
    s->args.W_y = std::max(1, std::min(16, pow2_floor(budget / (2 * 16 * n2))));
    int rx = 16;
    while (rx > 1 && 2 * 16 * n1 * (rx + 1) > budget) rx /= 2;
    s->args.R_x = std::min(rx, std::max(1, pow2_floor(n2 * 2 - 1)));
    s->args.W_z = std::min(s->args.W_z, std::max(1, pow2_floor(n1 * 2 - 1)));
    s->args.W_y = std::min(s->args.W_y, std::max(1, pow2_floor(n1 * 2 - 1)));
    CK(s->sigma.ensure(n * sizeof(double)));
    CK(s->eps_inv.ensure(3 * n * sizeof(double)));
    s->args.eps_inv = s->eps_inv.as<double>();
    CK(s->partial.ensure((size_t)s->nblk * 64 * sizeof(double2)));
    CK(s->small.ensure((size_t)(64 + 4096) * sizeof(double2)));
    CK(s->cgstate.ensure(64 * 6 * sizeof(double) + 64 * sizeof(double2)));
    {
        char* b = s->cgstate.as<char>();
        s->cgs.rr = (double*)b;
        s->cgs.rrnew = (double*)(b + 64 * 8);
        s->cgs.beta = (double*)(b + 128 * 8);
        s->cgs.thr = (double*)(b + 192 * 8);
        s->cgs.active = (int*)(b + 256 * 8);
        s->cgs.pMp = (double2*)(b + 384 * 8);
    }
    CK(cudaMallocHost((void**)&s->h_flags, 64 * sizeof(int)));
    s->fused_ok = fast_all(s->args) && std::getenv("BNF_NO_FUSED_CG") == nullptr;
    s->plane_ok = plane_supported(s->args);
    s->use_plane = s->plane_ok && std::getenv("BNF_NO_PLANE") == nullptr;
    {
        std::vector<double2> h(n3);
        for (int k = 0; k < n3; ++k) h[k] = unit_root(k, 2LL * n3);
        CK(s->hroot.ensure(n3 * sizeof(double2)));
        CK(cudaMemcpy(s->hroot.p, h.data(), n3 * sizeof(double2), cudaMemcpyHostToDevice));
        s->args.hroot_z = s->hroot.as<double2>();
    }
    s->use_z2 = s->fused_ok && zpass2_supported(s->args) && std::getenv("BNF_NO_Z2") == nullptr;
    s->use_graph = std::getenv("BNF_NO_GRAPH") == nullptr;
    s->plane_t_ok = s->use_z2 && plane_t_supported(s->args) && tensor_map_encoder() != nullptr &&
                    std::getenv("BNF_NO_PLANE_T") == nullptr;
    // persistent pipelined adjoint z pass (same tile width as k_zadj2, so the CG partial
    // layout is unchanged): opt-in with BNF_Z3=1 -- measured slower than k_zadj2 (128^3, b = 2: 161 vs
    // 133 us), so k_zadj2 stays the default
    s->use_z3 = s->use_z2 && zadj3_supported(s->args) && !(s->args.zcfg & 2) && tensor_map_encoder() != nullptr &&
                std::getenv("BNF_Z3") != nullptr && std::atoi(std::getenv("BNF_Z3")) != 0 && o.slabs <= 1;
    // virtual slabs (SURVEY §8(e) / DESIGN §8): the slab-decomposed operator with the
    // all-to-alls as device copies; needs the fast z passes and an L2 plane middle
    s->nsl = std::max(1, o.slabs);
    if (s->nsl > 1) {
        const int P = s->nsl;
        if (n2 % P != 0 || n3 % P != 0 || !s->use_z2 || !s->plane_ok || !plane_w_supported(s->args) ||
            std::getenv("BNF_NO_PLANE") != nullptr || (std::getenv("BNF_PLANE") && !std::getenv("BNF_PLANE_L2"))) {
            set_error("opts.slabs > 1 needs n2 and n3 divisible by slabs, a square xy plane of 64, 128 or 256 and the "
                      "fused z passes / L2 plane pass");
            return BNF_EINVAL;
        }
    }
    s->args.plane_hint = std::getenv("BNF_PLANE_HINT") ? std::atoi(std::getenv("BNF_PLANE_HINT")) : 1;
    s->args.plane_split = std::getenv("BNF_PLANE_SPLIT") ? std::atoi(std::getenv("BNF_PLANE_SPLIT")) : 1;
    s->alpha_fold_ok = std::getenv("BNF_NO_ALPHA_FOLD") == nullptr;
    // stage roots of the L2 plane pass in shared memory: default on (128^3: 123.5 vs 131.1 us at b = 1,
    // 228 vs 241 at b = 2, profiles/r02s2_plane_options.jsonl)
    s->args.plane_rs = std::getenv("BNF_PLANE_RS") ? std::atoi(std::getenv("BNF_PLANE_RS")) : 1;
    s->args.plane_xeo = std::getenv("BNF_PLANE_XEO") ? std::atoi(std::getenv("BNF_PLANE_XEO")) : 0;
    s->args.plane_ld = std::getenv("BNF_PLANE_LD") ? std::atoi(std::getenv("BNF_PLANE_LD")) : 0;
    CK(s->phasebuf.ensure(16 * sizeof(unsigned long long)));
    CK(cudaMemset(s->phasebuf.p, 0, 16 * sizeof(unsigned long long)));
    s->args.prof = std::getenv("BNF_PHASE_PROF") ? s->phasebuf.as<unsigned long long>() : nullptr;
    CK(s->iterbuf.ensure(8 * sizeof(int)));
    CK(cudaMemset(s->iterbuf.p, 0, 8 * sizeof(int)));
    s->d_iter = s->iterbuf.as<int>();
    if (s->fused_ok) {
        const size_t per = cg_partials_per_vec(s->args);
        const size_t bytes = 2 * 8 * per * sizeof(double) + 4 * 64 * sizeof(double) + 2 * (1 + 64) * sizeof(unsigned);
        CK(s->cgfuse_buf.ensure(bytes));
        CK(cudaMemset(s->cgfuse_buf.p, 0, bytes));
        char* b = s->cgfuse_buf.as<char>();
        s->cgf.part_x = (double*)b;
        s->cgf.part_z = (double*)(b + 8 * per * sizeof(double));
        char* c = b + 2 * 8 * per * sizeof(double);
        s->cgf.pmp = (double*)c;
        s->cgf.alpha = (double*)(c + 64 * sizeof(double));
        s->cgf.rr = s->cgs.rr;
        s->cgf.beta = s->cgs.beta;
        s->cgf.thr = s->cgs.thr;
        s->cgf.active = s->cgs.active;
        s->cgf.nslab = s->nsl;
    }
    *out = s.release();
    return BNF_OK;
}

int bnf_nccl_unique_id(unsigned char id[128]) {
    if (!id) {
        set_error("NULL argument");
        return BNF_EINVAL;
    }
    const Nccl& nc = Nccl::get();
    if (!nc.ok) {
        set_error("libnccl.so.2 could not be loaded (set BNF_NCCL_LIB)");
        return BNF_ENCCL;
    }
    ncclUniqueId u;
    NCK(nc.getUniqueId(&u));
    std::memcpy(id, u.internal, 128);
    return BNF_OK;
}

int bnf_solver_create_dist(const bnf_lattice* lat, const bnf_opts* opts, int nranks, int rank, const unsigned char id[128],
                           bnf_solver** out) {
    if (!lat || !out || !id || nranks < 1 || rank < 0 || rank >= nranks) {
        set_error("invalid argument");
        return BNF_EINVAL;
    }
    const Nccl& nc = Nccl::get();
    if (!nc.ok) {
        set_error("libnccl.so.2 could not be loaded (set BNF_NCCL_LIB)");
        return BNF_ENCCL;
    }
    bnf_opts o;
    bnf_opts_default(&o);
    if (opts) o = *opts;
    o.slabs = nranks;   // the slab geometry of the decomposition (validated by bnf_solver_create)
    bnf_solver* s = nullptr;
    TRY(bnf_solver_create(lat, &o, &s));
    std::unique_ptr<bnf_solver> g(s);
    s->dist = true;
    s->rank = rank;
    s->nv = s->n / nranks;
    s->use_graph = false;   // NCCL calls inside the CG loop: eager loop with a host convergence check
    s->cgf.nslab = nranks;
    s->args.plane_t = 0;
    ncclUniqueId u;
    std::memcpy(u.internal, id, 128);
    NCK(nc.commInitRank(&s->comm, nranks, u, rank));
    *out = g.release();
    return BNF_OK;
}

void bnf_solver_destroy(bnf_solver* s) {
    if (!s) return;
    cudaStreamSynchronize(s->st);
    delete s;
}

int bnf_set_epsilon(bnf_solver* s, const double* eps, int mem) {
    if (!s || !eps) {
        set_error("NULL argument");
        return BNF_EINVAL;
    }
    const long long n3 = 3 * s->n;
    std::vector<double> h(n3);
    if (mem == BNF_MEM_HOST) {
        std::memcpy(h.data(), eps, n3 * sizeof(double));
    } else if (mem == BNF_MEM_DEVICE) {
        CK(cudaMemcpyAsync(h.data(), eps, n3 * sizeof(double), cudaMemcpyDeviceToHost, s->st));
        CK(cudaStreamSynchronize(s->st));
    } else {
        set_error("mem must be BNF_MEM_HOST or BNF_MEM_DEVICE");
        return BNF_EINVAL;
    }
    // 1/eps, plus a compressed copy for the hot passes: uint8 index + LUT when the
    // field has <= 256 distinct values (exact: the LUT holds the same doubles).
    // One pass; runs of equal values (material regions) skip the table search.
    std::vector<double> vals;
    vals.reserve(256);
    std::vector<unsigned char> idx(n3);
    bool small = std::getenv("BNF_NO_EPS_LUT") == nullptr;
    double last = -1.0;
    int lastk = 0;
    for (long long t = 0; t < n3; ++t) {
        if (!(h[t] > 0.0) || !std::isfinite(h[t])) {
            set_error("eps must be finite and > 0");
            return BNF_EINVAL;
        }
        const double inv = 1.0 / h[t];
        h[t] = inv;
        if (!small) continue;
        if (inv != last) {
            int k = -1;
            for (int q = 0; q < (int)vals.size(); ++q)
                if (vals[q] == inv) {
                    k = q;
                    break;
                }
            if (k < 0) {
                if (vals.size() == 256) {
                    small = false;
                    continue;
                }
                k = (int)vals.size();
                vals.push_back(inv);
            }
            last = inv;
            lastk = k;
        }
        idx[t] = (unsigned char)lastk;
    }
    if (s->dist) {   // this rank's real-space z-slab [l][cl][b][a]
        const int P = s->nsl;
        const long long plane = (long long)s->L.n[0] * s->L.n[1], n = s->n, nloc = n / P, n3l = s->L.n[2] / P;
        std::vector<double> h2(3 * nloc);
        std::vector<unsigned char> i2(small ? 3 * nloc : 0);
        for (int l = 0; l < 3; ++l)
            for (long long cl = 0; cl < n3l; ++cl) {
                const long long src = l * n + (s->rank * n3l + cl) * plane, dst = l * nloc + cl * plane;
                std::memcpy(h2.data() + dst, h.data() + src, plane * sizeof(double));
                if (small) std::memcpy(i2.data() + dst, idx.data() + src, plane);
            }
        h.swap(h2);
        if (small) idx.swap(i2);
    } else if (s->nsl > 1) {   // slab-major [slab][l][cl][b][a] (real-space z-slabs of n3 / P planes)
        const int P = s->nsl;
        const long long plane = (long long)s->L.n[0] * s->L.n[1], n = s->n, nloc = n / P, n3l = s->L.n[2] / P;
        std::vector<double> h2(n3);
        std::vector<unsigned char> i2(small ? n3 : 0);
        for (int q = 0; q < P; ++q)
            for (int l = 0; l < 3; ++l)
                for (long long cl = 0; cl < n3l; ++cl) {
                    const long long src = l * n + (q * n3l + cl) * plane, dst = (long long)q * 3 * nloc + l * nloc + cl * plane;
                    std::memcpy(h2.data() + dst, h.data() + src, plane * sizeof(double));
                    if (small) std::memcpy(i2.data() + dst, idx.data() + src, plane);
                }
        h.swap(h2);
        if (small) idx.swap(i2);
    }
    CK(cudaMemcpyAsync(s->eps_inv.p, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice, s->st));
    s->args.eps_idx = nullptr;
    s->args.eps_lut = nullptr;
    if (small) {
        CK(s->eps_idx.ensure(n3));
        CK(s->eps_lut.ensure(256 * sizeof(double)));
        vals.resize(256, 0.0);
        CK(cudaMemcpyAsync(s->eps_idx.p, idx.data(), idx.size(), cudaMemcpyHostToDevice, s->st));
        CK(cudaMemcpyAsync(s->eps_lut.p, vals.data(), 256 * sizeof(double), cudaMemcpyHostToDevice, s->st));
        s->args.eps_idx = s->eps_idx.as<unsigned char>();
        s->args.eps_lut = s->eps_lut.as<double>();
    }
    CK(cudaStreamSynchronize(s->st));
    s->eps_set = true;
    s->kver++;
    return BNF_OK;
}

int bnf_set_kappa(bnf_solver* s, const double kappa[3]) {
    if (!s || !kappa) {
        set_error("NULL argument");
        return BNF_EINVAL;
    }
    TRY(set_kappa_impl(s, kappa));
    CK(cudaStreamSynchronize(s->st));
    return BNF_OK;
}

int bnf_apply_Ar(bnf_solver* s, const void* y, void* out, int b, int op) {
    if (!s || !y || !out || b < 1 || (op != BNF_OP_AR && op != BNF_OP_M)) {
        set_error("invalid argument");
        return BNF_EINVAL;
    }
    if (!s->eps_set || !s->kappa_set) {
        set_error("bnf_set_epsilon and bnf_set_kappa must precede bnf_apply_Ar");
        return BNF_ESTATE;
    }
    TRY(autotune_plane(s, b));
    TRY(apply_op(s, (const double2*)y, (double2*)out, b, op));
    CK(cudaStreamSynchronize(s->st));
    if (s->prof.on) s->prof.flush();
    return BNF_OK;
}

int bnf_cg_solve(bnf_solver* s, const void* c, void* x, int b, int max_iter, int* iters) {
    if (!s || !c || !x || b < 1 || b > 64 || max_iter < 1) {
        set_error("invalid argument");
        return BNF_EINVAL;
    }
    if (!s->eps_set || !s->kappa_set) {
        set_error("bnf_set_epsilon and bnf_set_kappa must precede bnf_cg_solve");
        return BNF_ESTATE;
    }
    TRY(autotune_plane(s, b));
    const int keep = s->o.max_inner;
    s->o.max_inner = max_iter;
    s->kver++;   // cached CG graphs carry the iteration cap
    int it = -1;
    CK(cudaMemsetAsync(s->d_iter, 0, 4 * sizeof(int), s->st));
    const long long g0 = s->graph_calls;
    const int rc = s->fused_ok ? cg_solve_fused(s, (const double2*)c, (double2*)x, b, &it)
                               : cg_solve(s, (const double2*)c, (double2*)x, b, &it);
    s->o.max_inner = keep;
    s->kver++;
    if (rc != BNF_OK) return rc;
    CK(cudaStreamSynchronize(s->st));
    if (s->prof.on) s->prof.flush();
    if (s->graph_calls > g0) {   // iterations counted on the device inside the graph
        int h[3];
        CK(cudaMemcpy(h, s->d_iter, 3 * sizeof(int), cudaMemcpyDeviceToHost));
        it = h[0];
    }
    if (iters) *iters = it;
    return BNF_OK;
}

int bnf_solve(bnf_solver* s, const double kappa[3], int nev, double* lambda, bnf_stats* stats) {
    auto t0 = std::chrono::steady_clock::now();
    if (!s || !kappa || !lambda || nev < 1) {
        set_error("invalid argument");
        return BNF_EINVAL;
    }
    if (!s->eps_set) {
        set_error("bnf_set_epsilon must precede bnf_solve");
        return BNF_ESTATE;
    }
    const long long launches0 = s->prof.launches;
    s->matvecs = 0;
    s->inner_iters = 0;
    s->active_mv = 0;
    s->graph_calls = 0;
    CK(cudaMemsetAsync(s->d_iter, 0, 4 * sizeof(int), s->st));
    TRY(set_kappa_impl(s, kappa));
    TRY(autotune_plane(s, s->o.block));
    const long long N = 2 * s->nv;
    const int b = s->o.block;
    const int want = nev + s->o.guard;
    const long long dof = 2 * s->n - (s->args.mp.gamma >= 0 ? 2 : 0);   // global NFSEP dimension
    if (want > dof) {
        set_error("nev + guard exceeds the NFSEP dimension");
        return BNF_EINVAL;
    }
    if (s->o.method == 1) {   // NEXT-1: LOBPCG on A_r, preconditioned by Sigma_r^{-2}
        double maxres = 0.0;
        int iters = 0;
        bool conv = false;
        const int rc = lobpcg_solve(s, nev, want, lambda, maxres, iters, conv);
        if (rc != BNF_OK && rc != BNF_ENOCONV) return rc;
        if (!conv || !(maxres <= s->o.res_tol)) {
            // stagnation / breakdown: fall back to the paper's inverse Lanczos (cold start)
            s->lob_fallbacks++;
            s->prev_want = 0;
            const long long lob_mv = s->matvecs, lob_launches = s->prof.launches - launches0;
            bnf_opts keep = s->o;
            s->o.method = 0;
            const int rc2 = bnf_solve(s, kappa, nev, lambda, stats);
            s->o = keep;
            if (stats) {   // the abandoned LOBPCG iterations are part of this call's work
                stats->matvecs += lob_mv;
                stats->active_matvecs += lob_mv;
                stats->kernel_launches += lob_launches;
                stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            }
            return rc2;
        }
        s->nev_last = nev;
        s->prev_want = want;
        CK(cudaStreamSynchronize(s->st));
        if (s->prof.on) s->prof.flush();
        if (stats) {
            stats->outer_steps = iters;
            stats->converged = conv ? 1 : 0;
            stats->inner_iters = 0;
            stats->matvecs = s->matvecs;
            stats->active_matvecs = s->matvecs;   // LOBPCG applies A_r to the unlocked columns only
            stats->kernel_launches = s->prof.launches - launches0;
            stats->max_ritz_residual = maxres;
            stats->max_residual = maxres;
            stats->polish_steps = 0;
            stats->polish_failed = 0;
            stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        }
        if (!conv) {
            set_error("LOBPCG did not reach res_tol within max_outer iterations");
            return BNF_ENOCONV;
        }
        return BNF_OK;
    }
    // Lanczos step cap: opts.max_outer, or (0 = auto) enough steps for the wanted
    // pairs with a margin that scales with ceil(want / b) -- single-vector runs
    // (b = 1) need several times more steps than b = 4 for the same pairs
    const long long cap_dof = (dof + b - 1) / b;
    const int auto_steps = std::max(60, 12 * ((want + b - 1) / b));
    const int maxsteps = (int)std::max<long long>(1, std::min<long long>(s->o.max_outer > 0 ? s->o.max_outer : auto_steps,
                                                                       cap_dof));
    if ((long long)maxsteps * b < want) {
        set_error("max_outer * block < nev + guard: the Krylov basis cannot hold the wanted pairs");
        return BNF_EINVAL;
    }
    const size_t vbytes = (size_t)N * sizeof(double2);
    // basis: address space for every step, physical memory mapped as it grows
    TRY(s->V.reserve(vbytes * (size_t)b * (maxsteps + 1), s->o.device));
    TRY(s->V.ensure(vbytes * (size_t)b * 2));
    CK(s->cgx.ensure(vbytes * b));
    // small device scratch: gram_host / gemm_nn_host stage p x 8 blocks at offset 64
    CK(s->small.ensure((size_t)(64 + 8 * std::max<long long>((long long)(maxsteps + 1) * b, want)) * sizeof(double2)));
    double2* V = s->V.as<double2>();
    // start block: seeded counter-based normals, Gamma mode masked (R6)
    RUN("fill_random", launch_fill_random(V, N, b, s->o.seed, (long long)s->rank * N * b, s->sigma.as<double>(), s->nv, s->st, sig_nloc(s)));
    if (s->o.warm && s->prev_want > 0) {
        // Warm start (DESIGN R17): start block = fixed pseudo-random combinations of
        // the previous solve's Ritz vectors (neighbouring k on the path) plus 1e-3 of
        // the random block; Gamma mode masked.  Only the start block changes; the
        // iteration, its tolerance and the returned eigenpairs are as before.
        const int pw = s->prev_want;
        std::vector<cd> Wm((size_t)pw * b);
        unsigned long long h = 0x9E3779B97F4A7C15ull;
        for (auto& x : Wm) {
            h ^= h >> 33;
            h *= 0xff51afd7ed558ccdull;
            h ^= h >> 33;
            x = cd(((double)(h >> 11) / 9007199254740992.0) - 0.5, 0.0);
        }
        TRY(gemm_nn_host(s, s->Yv.as<double2>(), pw, Wm, b, V, 1.0, 1e-3));
        RUN("scale_sigma", launch_scale_sigma(V, V, s->sigma.as<double>(), s->nv, b, 1, s->st, sig_nloc(s)));
        RUN("scale_sigma", launch_scale_sigma(V, V, s->sigma.as<double>(), s->nv, b, 0, s->st, sig_nloc(s)));
    }
    bool ok = true;
    std::vector<cd> R0;
    TRY(chol_qr2(s, V, b, R0, ok));
    if (!ok) {
        set_error("start block rank deficient");
        return BNF_ENOCONV;
    }
    std::vector<std::vector<cd>> As, Bs;  // b x b blocks
    std::vector<double> theta;
    std::vector<cd> S;
    int m = 0;
    bool converged = false;
    double maxres = 0.0;
    for (int step = 0; step < maxsteps; ++step) {
        double2* Vj = V + (size_t)step * b * N;
        TRY(s->V.ensure(vbytes * (size_t)b * (step + 2)));
        double2* W = V + (size_t)(step + 1) * b * N;   // next block, built in place
        // NEXT-1 relaxed inner solves (opts.relax_inner): the j-th application of A_r^{-1} may be
        // less accurate once the wanted Ritz pairs have converged partly (inexact Krylov, the allowed
        // error grows like 1 / residual): tol_j = tol_inner * clamp(1e-6 / res_{j-1}, 1, 1e5).  The
        // final Rayleigh-Ritz on A_r and the R19 residual polish (exact inner tolerance) secure the
        // returned pairs.
        s->tol_inner_eff = 0.0;
        if (s->o.relax_inner && step > 0 && maxres > 0.0)
            s->tol_inner_eff = s->o.tol_inner * std::min(1e5, std::max(1.0, 1e-6 / maxres));
        TRY(apply_Ar_inv(s, Vj, W, b));  // W = A_r^{-1} V_j
        s->tol_inner_eff = 0.0;
        // full reorthogonalisation (classical Gram-Schmidt against all of V) with the
        // DGKS / Kahan-Parlett "twice is enough" test: the second pass runs unless the
        // first kept every column's norm above 1/sqrt(2) of its value (norm after the
        // pass from Pythagoras, V orthonormal); accumulate the projections.  Pass 1
        // takes [V_0..V_step | W]^* W in one Gram: its last b rows are G0 = W^* W.
        const int p = (step + 1) * b;
        std::vector<cd> Hacc((size_t)p * b, 0.0), H, G0;
        for (int pass = 0; pass < 2; ++pass) {
            if (pass == 0) {
                std::vector<cd> HG;
                TRY(gram_host(s, V, p + b, W, b, HG));
                H.assign(HG.begin(), HG.begin() + (size_t)p * b);
                G0.assign(HG.begin() + (size_t)p * b, HG.end());
            } else {
                TRY(gram_host(s, V, p, W, b, H));
            }
            TRY(gemm_nn_host(s, V, p, H, b, W, -1.0, 1.0));
            for (size_t t = 0; t < H.size(); ++t) Hacc[t] += H[t];
            if (pass == 0 && s->o.reorth_once_ok) {
                bool keep = true;
                for (int c = 0; c < b && keep; ++c) {
                    double proj = 0.0;
                    for (int a = 0; a < p; ++a) proj += std::norm(H[(size_t)a * b + c]);
                    const double w0 = G0[(size_t)c * b + c].real();
                    keep = (w0 - proj) >= 0.5 * w0;
                }
                if (keep) {
                    s->reorth_skipped++;
                    break;
                }
            }
        }
        std::vector<cd> A((size_t)b * b);
        for (int i = 0; i < b; ++i)
            for (int j = 0; j < b; ++j) A[(size_t)i * b + j] = Hacc[(size_t)(step * b + i) * b + j];
        for (int i = 0; i < b; ++i)  // Hermitian part
            for (int j = i; j < b; ++j) {
                cd h = 0.5 * (A[(size_t)i * b + j] + std::conj(A[(size_t)j * b + i]));
                A[(size_t)i * b + j] = h;
                A[(size_t)j * b + i] = std::conj(h);
            }
        std::vector<cd> Rn;
        TRY(chol_qr2(s, W, b, Rn, ok));
        if (!ok) {  // invariant subspace / breakdown: continue with a fresh random block
            RUN("fill_random", launch_fill_random(W, N, b, s->o.seed + 7919ull * (step + 1), 0,
                                                  s->sigma.as<double>(), s->nv, s->st, sig_nloc(s)));
            for (int pass = 0; pass < 2; ++pass) {
                TRY(gram_host(s, V, p, W, b, H));
                TRY(gemm_nn_host(s, V, p, H, b, W, -1.0, 1.0));
            }
            TRY(chol_qr2(s, W, b, Rn, ok));
            if (!ok) {
                set_error("block Lanczos breakdown");
                return BNF_ENOCONV;
            }
            std::fill(Rn.begin(), Rn.end(), cd(0.0));
        }
        As.push_back(A);
        Bs.push_back(Rn);
        m = step + 1;
        // block tridiagonal T_m and its eigen-decomposition
        const int mb = m * b;
        std::vector<cd> T((size_t)mb * mb, 0.0);
        for (int k = 0; k < m; ++k) {
            for (int i = 0; i < b; ++i)
                for (int j = 0; j < b; ++j) {
                    T[(size_t)(k * b + i) * mb + k * b + j] = As[k][(size_t)i * b + j];
                    if (k + 1 < m) {
                        const cd bij = Bs[k][(size_t)i * b + j];  // B_{k+1}: row block k+1, col block k
                        T[(size_t)((k + 1) * b + i) * mb + k * b + j] = bij;
                        T[(size_t)(k * b + j) * mb + (k + 1) * b + i] = std::conj(bij);
                    }
                }
        }
        std::vector<double> w;
        std::vector<cd> Z;
        herm_eig(mb, T, w, &Z);
        // descending theta (largest theta = smallest lambda)
        theta.assign(mb, 0.0);
        S.assign((size_t)mb * mb, 0.0);
        for (int c = 0; c < mb; ++c) {
            theta[c] = w[mb - 1 - c];
            for (int r = 0; r < mb; ++r) S[(size_t)r * mb + c] = Z[(size_t)r * mb + (mb - 1 - c)];
        }
        if (mb >= want) {
            maxres = 0.0;
            bool all = true;
            const std::vector<cd>& Bl = Bs.back();
            for (int c = 0; c < want; ++c) {
                double r2 = 0.0;
                for (int i = 0; i < b; ++i) {
                    cd acc = 0.0;
                    for (int j = 0; j < b; ++j) acc += Bl[(size_t)i * b + j] * S[(size_t)((m - 1) * b + j) * mb + c];
                    r2 += std::norm(acc);
                }
                const double rel = std::sqrt(r2) / std::fabs(theta[c]);
                maxres = std::max(maxres, rel);
                if (!(rel <= s->o.tol_outer)) all = false;
            }
            if (all) {
                converged = true;
                break;
            }
        }
    }
    // Ritz vectors Y = V_m S[:, :want]
    const int mb = m * b;
    CK(s->Yv.ensure(vbytes * want));
    double2* Y = s->Yv.as<double2>();
    {
        std::vector<cd> Sw((size_t)mb * want);
        for (int r = 0; r < mb; ++r)
            for (int c = 0; c < want; ++c) Sw[(size_t)r * want + c] = S[(size_t)r * mb + c];
        TRY(gemm_nn_host(s, V, mb, Sw, want, Y, 1.0, 0.0));
    }
    std::vector<double> lam(want);
    for (int c = 0; c < want; ++c) lam[c] = 1.0 / theta[c];
    double maxr_ar = -1.0;
    int polish = 0, polish_failed = 0;
    if (s->o.refine >= 1) for (int pass = 0;; ++pass) {
        // Rayleigh-Ritz of A_r on span(Y) (DESIGN R15); a step of subspace
        // (inverse) iteration first when refine >= 2, and again while the
        // explicit residual of a returned pair exceeds res_tol (DESIGN R19).
        CK(s->AZ.ensure(vbytes * want));
        double2* AZ = s->AZ.as<double2>();
        if (s->o.refine >= 2 || pass > 0) {
            // subspace inverse iteration into AZ; adopted only if its Cholesky-QR
            // succeeds (a rank-deficient block keeps the previous Y and lambda)
            for (int c0 = 0; c0 < want; c0 += b) {
                const int qc = std::min(b, want - c0);
                TRY(apply_Ar_inv(s, Y + (size_t)c0 * N, AZ + (size_t)c0 * N, qc));
            }
            std::vector<cd> Rq;
            TRY(chol_qr2(s, AZ, want, Rq, ok));
            if (!ok) {
                polish_failed = 1;
                break;
            }
            RUN("copy", launch_copy(Y, AZ, N * want, s->st));
        }
        for (int c0 = 0; c0 < want; c0 += b) {
            const int qc = std::min(b, want - c0);
            TRY(apply_op(s, Y + (size_t)c0 * N, AZ + (size_t)c0 * N, qc, BNF_OP_AR));
            s->active_mv += qc;
        }
        std::vector<cd> Hm, Zs;
        TRY(gram_host(s, Y, want, AZ, want, Hm));
        for (int i = 0; i < want; ++i)
            for (int j = i; j < want; ++j) {
                cd h = 0.5 * (Hm[(size_t)i * want + j] + std::conj(Hm[(size_t)j * want + i]));
                Hm[(size_t)i * want + j] = h;
                Hm[(size_t)j * want + i] = std::conj(h);
            }
        std::vector<double> w;
        herm_eig(want, Hm, w, &Zs);
        // rotate: Y <- Y Zs, AZ <- AZ Zs (via the work block in chunks)
        CK(s->cgc.ensure(vbytes * want));
        double2* tmp = s->cgc.as<double2>();
        TRY(gemm_nn_host(s, Y, want, Zs, want, tmp, 1.0, 0.0));
        RUN("copy", launch_copy(Y, tmp, N * want, s->st));
        TRY(gemm_nn_host(s, AZ, want, Zs, want, tmp, 1.0, 0.0));
        RUN("copy", launch_copy(AZ, tmp, N * want, s->st));
        for (int c = 0; c < want; ++c) lam[c] = w[c];
        // residuals ||A_r y - lambda y|| / ||y||, formed explicitly (R = AZ - Y diag(lambda))
        // rather than from Gram entries (whose cancellation would cap the resolution at
        // ~sqrt(eps) lambda)
        std::vector<cd> Dl((size_t)nev * nev, 0.0);
        for (int c = 0; c < nev; ++c) Dl[(size_t)c * nev + c] = -lam[c];
        RUN("copy", launch_copy(tmp, AZ, N * nev, s->st));
        TRY(gemm_nn_host(s, Y, nev, Dl, nev, tmp, 1.0, 1.0));
        maxr_ar = 0.0;
        for (int c = 0; c < nev; ++c) {
            std::vector<cd> rr, yy;
            TRY(gram_host(s, tmp + (size_t)c * N, 1, tmp + (size_t)c * N, 1, rr));
            TRY(gram_host(s, Y + (size_t)c * N, 1, Y + (size_t)c * N, 1, yy));
            maxr_ar = std::max(maxr_ar, std::sqrt(std::fabs(rr[0].real()) / yy[0].real()));
        }
        if (!(maxr_ar > s->o.res_tol) || pass >= s->o.max_polish) break;
        ++polish;
    }
    s->lam.assign(lam.begin(), lam.begin() + nev);
    s->nev_last = nev;
    s->prev_want = want;
    for (int c = 0; c < nev; ++c) lambda[c] = lam[c];
    CK(cudaStreamSynchronize(s->st));
    if (s->prof.on) s->prof.flush();
    long long graph_launches = 0;
    if (s->graph_calls > 0) {   // CG iterations run inside graphs were counted on the device
        int h[4];
        CK(cudaMemcpy(h, s->d_iter, 4 * sizeof(int), cudaMemcpyDeviceToHost));
        s->inner_iters += h[2];
        s->matvecs += h[2];
        s->active_mv += h[3];
        graph_launches = (long long)h[1] * s->graph_kernels_per_iter;
    }
    if (stats) {
        stats->outer_steps = m;
        stats->converged = converged ? 1 : 0;
        stats->inner_iters = s->inner_iters;
        stats->matvecs = s->matvecs;
        stats->kernel_launches = s->prof.launches - launches0 + graph_launches;
        stats->max_ritz_residual = maxres;
        stats->max_residual = maxr_ar;
        stats->polish_steps = polish;
        stats->active_matvecs = s->active_mv;
        stats->polish_failed = polish_failed;
        stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
    if (!converged) {
        set_error("block inverse Lanczos did not converge within max_outer steps");
        return BNF_ENOCONV;
    }
    return BNF_OK;
}

int bnf_eigvecs(bnf_solver* s, int kind, void* out, int mem) {
    if (!s || !out || (kind != BNF_VEC_Y && kind != BNF_VEC_E && kind != BNF_VEC_H) ||
        (mem != BNF_MEM_HOST && mem != BNF_MEM_DEVICE)) {
        set_error("invalid argument");
        return BNF_EINVAL;
    }
    const int nev = s->nev_last;
    if (nev == 0) {
        set_error("no eigenvectors: call bnf_solve first");
        return BNF_ESTATE;
    }
    const long long N = 2 * s->nv;
    const cudaMemcpyKind dir = (mem == BNF_MEM_HOST) ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    if (kind == BNF_VEC_Y) {
        CK(cudaMemcpyAsync(out, s->Yv.p, (size_t)N * nev * sizeof(double2), dir, s->st));
        CK(cudaStreamSynchronize(s->st));
        return BNF_OK;
    }
    if (s->nsl > 1 || s->dist) {
        set_error("BNF_VEC_E / BNF_VEC_H are not available in slab mode (fetch BNF_VEC_Y, slab layout)");
        return BNF_EINVAL;
    }
    const bool hfield = kind == BNF_VEC_H;
    // e = B^{-1} Q_r Sigma_r y / sqrt(lambda), Bloch phase of eq. (T) included
    const long long n = s->n;
    const size_t ebytes = (size_t)3 * n * sizeof(double2);
    DevBuf scales;
    CK(scales.ensure(nev * sizeof(double)));
    std::vector<double> sc(nev);
    for (int c = 0; c < nev; ++c) sc[c] = 1.0 / std::sqrt(s->lam[c]);
    CK(cudaMemcpyAsync(scales.p, sc.data(), nev * sizeof(double), cudaMemcpyHostToDevice, s->st));
    const int chunk = std::max(1, s->o.block);
    for (int c0 = 0; c0 < nev; c0 += chunk) {
        const int qc = std::min(chunk, nev - c0);
        TRY(ensure_work(s, qc));
        double2* U = s->U.as<double2>();
        const double2* Yc = s->Yv.as<double2>() + (size_t)c0 * N;
        RUN("zfwd", launch_zfwd(s->args, Yc, U, qc, hfield ? 2 : BNF_OP_AR, s->st));
        RUN("yfwd", launch_ypass(s->args, U, qc, 0, s->st));
        RUN("xfwd_recover", launch_xfwd_recover(s->args, U, qc, hfield ? nullptr : s->eps_inv.as<double>(),
                                                1.0 / std::sqrt((double)n), hfield ? nullptr : scales.as<double>() + c0,
                                                s->st));
        RUN("bloch", launch_bloch_phase(s->args, U, qc, s->kappa[0], s->kh2, s->kh3, s->st));
        CK(cudaMemcpyAsync((char*)out + (size_t)c0 * ebytes, U, ebytes * qc, dir, s->st));
    }
    CK(cudaStreamSynchronize(s->st));
    return BNF_OK;
}

int bnf_kernel_times(bnf_solver* s, const char** names, double* ms, long long* launches, int cap, int* count) {
    if (!s || !count) {
        set_error("NULL argument");
        return BNF_EINVAL;
    }
    s->prof.flush();
    int k = 0;
    for (const auto& nm : s->prof.order) {
        if (k < cap) {
            auto& e = s->prof.acc[nm];
            if (names) names[k] = s->prof.acc.find(nm)->first.c_str();
            if (ms) ms[k] = e.first;
            if (launches) launches[k] = e.second;
        }
        ++k;
    }
    *count = k;
    return BNF_OK;
}

int bnf_phase_counters(bnf_solver* s, unsigned long long* out, int cap) {
    if (!s || !out || cap < 1) {
        set_error("invalid argument");
        return BNF_EINVAL;
    }
    CK(cudaStreamSynchronize(s->st));
    CK(cudaMemcpy(out, s->phasebuf.p, sizeof(unsigned long long) * std::min(cap, 16), cudaMemcpyDeviceToHost));
    CK(cudaMemset(s->phasebuf.p, 0, 16 * sizeof(unsigned long long)));
    return BNF_OK;
}

int bnf_set_profile(bnf_solver* s, int on) {
    if (!s) {
        set_error("NULL argument");
        return BNF_EINVAL;
    }
    CK(cudaStreamSynchronize(s->st));
    if (s->prof.on) s->prof.flush();
    s->prof.on = on != 0;
    s->o.profile = on != 0;
    return BNF_OK;
}

int bnf_kernel_times_reset(bnf_solver* s) {
    if (!s) return BNF_EINVAL;
    s->prof.flush();
    s->prof.acc.clear();
    s->prof.order.clear();
    return BNF_OK;
}

int bnf_host_herm_eig(int n, double* a, double* w, double* z) {
    if (n < 0 || (n > 0 && (!a || !w))) {
        set_error("invalid argument");
        return BNF_EINVAL;
    }
    std::vector<cd> A((size_t)n * n);
    for (size_t t = 0; t < A.size(); ++t) A[t] = cd(a[2 * t], a[2 * t + 1]);
    std::vector<double> ww;
    std::vector<cd> Z;
    herm_eig(n, A, ww, z ? &Z : nullptr);
    for (int i = 0; i < n; ++i) w[i] = ww[i];
    if (z)
        for (size_t t = 0; t < Z.size(); ++t) {
            z[2 * t] = Z[t].real();
            z[2 * t + 1] = Z[t].imag();
        }
    return BNF_OK;
}

}  // extern "C"
