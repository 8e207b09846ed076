// Block reductions and the fused-CG scalar updates shared by the operator
// passes (kernels.cu, plane.cu).  Internal.
#pragma once

#include <cuda_runtime.h>

#include "kernels.cuh"

namespace bnf {
namespace {

__device__ __forceinline__ double2 warp_sum(double2 v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
        v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
    }
    return v;
}

// block-wide sum of one complex value (blockDim.x multiple of 32, <= 1024)
// red: >= 32 entries, or >= blockDim.x entries when blockDim.x is not a
// multiple of 32 (a partial warp cannot use full-mask shuffles; the sum is
// then taken serially, still in a fixed order).
__device__ double2 block_sum(double2 v, double2* red) {
    if (blockDim.x & 31u) {
        __syncthreads();
        red[threadIdx.x] = v;
        __syncthreads();
        double2 r = make_double2(0, 0);
        if (threadIdx.x == 0)
            for (unsigned t = 0; t < blockDim.x; ++t) r = make_double2(r.x + red[t].x, r.y + red[t].y);
        __syncthreads();
        return r;  // valid in thread 0
    }
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

// ---------------------------------------------- fused-CG reductions
// Block partial of one double (written by thread 0); k_cg_finish (kernels.cu)
// reduces the partials of a launch in a fixed order (deterministic) and
// updates the CG scalars.
__device__ void cg_block_partial(double v, double* slot, double2* scratch) {
    __syncthreads();   // scratch (shared memory) may still be in use
    const double2 s = block_sum(make_double2(v, 0.0), scratch);
    if (threadIdx.x == 0) *slot = s.x;
}
// CG scalar updates of one vector from its reduced (p, M p) resp. (r, r)
__device__ __forceinline__ void cg_alpha_update(const CGFuse& cg, int v, double pmp) {
    cg.pmp[v] = pmp;
    cg.alpha[v] = (cg.active[v] && pmp > 0.0) ? cg.rr[v] / pmp : 0.0;
}
__device__ __forceinline__ void cg_beta_update(const CGFuse& cg, int v, double rn) {
    const int act = cg.active[v];
    if (act && cg.iter != nullptr) atomicAdd(cg.iter + 3, 1);   // applications to a still-iterating vector
    cg.beta[v] = (act && cg.rr[v] > 0.0) ? rn / cg.rr[v] : 0.0;
    if (act) cg.rr[v] = rn;
    cg.active[v] = (act && rn > cg.thr[v]) ? 1 : 0;
}
// device-side loop control of the CG graph (solver.cu, cg_graph): continue while
// any vector is active and the iteration cap is not reached (thread 0, after the
// beta updates of every vector are visible to it)
__device__ __forceinline__ void cg_loop_control(const CGFuse& cg, int nvec) {
    if (cg.iter != nullptr) {
        int any = 0;
        for (int v = 0; v < nvec; ++v) any |= cg.active[v];
        const int it = ++cg.iter[0];
        cg.iter[1] += 1;
        cg.iter[2] += nvec;
        if (cg.use_cond) cudaGraphSetConditional(cg.cond, (any && it < cg.max_iter) ? 1u : 0u);
    }
}
}  // namespace
}  // namespace bnf
