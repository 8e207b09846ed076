// Micro-benchmark: cost of the register-FFT data exchange on sm_100a.
// Compares (a) a warp-local shared-memory exchange (STS.128 + LDS.128 with
// __syncwarp), (b) an xor-shuffle transpose of the same data, (c) raw SHFL,
// (d) raw DFMA, and full 128-point complex128 FFT pairs (forward + inverse,
// N = 16 x 8, 8 lanes per sequence) with either exchange.  Prints the time
// per item per SM and the derived per-SM throughputs.
#include <cuda_runtime.h>
#include <cstdio>
#include "../../paper_1806_10284_b200/csrc/fastfft.cuh"

using namespace bnf::fast;


// N2 x N2 transposes (one per u) across the N2 consecutive lanes of a sequence:
// element (lane t, slot u*N2 + s) -> (lane s, slot u*N2 + t)
template <int N1, int N2>
__device__ __forceinline__ void xpose_shfl(double2 (&v)[N1], int t) {
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
                const double2 snd = p ? a : b;
                const double2 r = shfl_xor2(snd, d);
                if (p) a = r; else b = r;
            }
    }
}

template <int N1, int N2>
__device__ __forceinline__ void xpose_smem(double2 (&v)[N1], int t, int w, double2* xw) {
    // per-warp region, idx(k1, t, w) = k1 * S1 + t * S2 + w  (padded: conflict-free)
    constexpr int W = 32 / N2, S2 = W + 1, S1 = N2 * S2 + 1;
#pragma unroll
    for (int k1 = 0; k1 < N1; ++k1) xw[k1 * S1 + t * S2 + w] = v[k1];
    __syncwarp();
#pragma unroll
    for (int u = 0; u < N1 / N2; ++u)
#pragma unroll
        for (int tt = 0; tt < N2; ++tt) v[u * N2 + tt] = xw[(t + N2 * u) * S1 + tt * S2 + w];
    __syncwarp();
}

template <int MODE>
__global__ void __launch_bounds__(256, 2) k_bench(double2* out, const double2* __restrict__ root, int iters) {
    constexpr int N1 = 16, N2 = 8;
    extern __shared__ double2 sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int t = lane % N2, w = lane / N2;
    double2* xw = sm + warp * 660;
    double2 v[N1];
#pragma unroll
    for (int m = 0; m < N1; ++m) v[m] = make_double2(threadIdx.x * 1e-3 + m, blockIdx.x * 1e-4 - m);
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) xpose_smem<N1, N2>(v, t, w, xw);
        if (MODE == 1) xpose_shfl<N1, N2>(v, t);
        if (MODE == 2) {
#pragma unroll
            for (int m = 0; m < N1; ++m) v[m] = shfl_xor2(v[m], 1 + (m & 3));
        }
        if (MODE == 3) {
#pragma unroll
            for (int m = 0; m < N1; ++m) {
                v[m].x = fma(v[m].x, 0.999, v[(m + 1) % N1].y);
                v[m].y = fma(v[m].y, 1.001, -v[(m + 3) % N1].x);
            }
        }
        if (MODE == 4 || MODE == 5) {   // forward + inverse 128-point FFT, register stages
            DFT<N1, 1>::run(v);
            if (t > 0) {
#pragma unroll
                for (int k1 = 1; k1 < N1; ++k1) v[k1] = cmul(v[k1], __ldg(root + k1 * N2 + t));
            }
            if (MODE == 4) xpose_smem<N1, N2>(v, t, w, xw); else xpose_shfl<N1, N2>(v, t);
#pragma unroll
            for (int u = 0; u < N1 / N2; ++u) {
                double2 a[N2];
#pragma unroll
                for (int q = 0; q < N2; ++q) a[q] = v[u * N2 + q];
                DFT<N2, 1>::run(a);
#pragma unroll
                for (int q = 0; q < N2; ++q) v[u * N2 + q] = cscale(a[q], 0.0078125);
            }
#pragma unroll
            for (int u = 0; u < N1 / N2; ++u) {
                double2 a[N2];
#pragma unroll
                for (int q = 0; q < N2; ++q) a[q] = v[u * N2 + q];
                DFT<N2, -1>::run(a);
#pragma unroll
                for (int q = 0; q < N2; ++q) v[u * N2 + q] = a[q];
            }
            if (MODE == 4) xpose_smem<N1, N2>(v, t, w, xw); else xpose_shfl<N1, N2>(v, t);
            if (t > 0) {
#pragma unroll
                for (int k1 = 1; k1 < N1; ++k1) v[k1] = cjmul(__ldg(root + k1 * N2 + t), v[k1]);
            }
            DFT<N1, -1>::run(v);
        }
    }
    double2 acc = make_double2(0, 0);
#pragma unroll
    for (int m = 0; m < N1; ++m) acc = cadd(acc, v[m]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int MODE>
float run(double2* out, const double2* root, int blocks, int iters) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int smem = 8 * 660 * 16;
    cudaFuncSetAttribute(k_bench<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_bench<MODE><<<blocks, 256, smem>>>(out, root, 2);
    cudaEventRecord(a);
    k_bench<MODE><<<blocks, 256, smem>>>(out, root, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

int main() {
    int nsm = 0, clk = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int blocks = nsm * 2, iters = 2000;
    double2 *out, *root;
    cudaMalloc(&out, sizeof(double2) * blocks * 256);
    cudaMalloc(&root, sizeof(double2) * 128);
    double2 h[128];
    for (int k = 0; k < 128; ++k) h[k] = make_double2(cos(k * 0.049), sin(k * 0.049));
    cudaMemcpy(root, h, sizeof(h), cudaMemcpyHostToDevice);
    const char* names[] = {"smem xpose (16 STS.128+16 LDS.128 /thread)", "shfl xpose (3 xor stages)",
                           "raw shfl (32 SHFL.32 /thread)", "raw DFMA (32 /thread)", "FFT128 fwd+inv, smem xch",
                           "FFT128 fwd+inv, shfl xch"};
    float ms[6];
    ms[0] = run<0>(out, root, blocks, iters);
    ms[1] = run<1>(out, root, blocks, iters);
    ms[2] = run<2>(out, root, blocks, iters);
    ms[3] = run<3>(out, root, blocks, iters);
    ms[4] = run<4>(out, root, blocks, iters);
    ms[5] = run<5>(out, root, blocks, iters);
    const double warp_iters_per_sm = (double)blocks * 8 * iters / nsm;
    for (int m = 0; m < 6; ++m) {
        const double cyc = ms[m] * 1e-3 * clk * 1e3 / warp_iters_per_sm;   // SM cycles per warp-iteration
        printf("%-45s %8.3f ms  %7.2f SM-cycles per warp-iteration\n", names[m], ms[m], cyc);
    }
    printf("clock %d kHz, %d SMs, %s\n", clk, nsm, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
