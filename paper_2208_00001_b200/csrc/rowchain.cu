// Row-chain kernel: directional passes whose plane is a single row (2D images,
// nu == 1).  Replaces run_pass<K>'s 2D branch (/root/reference/proj/src/
// scan_parallel.cpp:119-139: v chunked by thread, `omp barrier` per row) for a
// forward+backward pair on one axis.
//
// One CTA per image owns the whole row for the whole pair: each thread keeps 4
// consecutive columns of the previous row (distance and intensity) in
// registers, v +- 1 comes from warp shuffles and the warp-edge columns from a
// double-buffered shared-memory slot, so a plane step is one relax of 4 voxels
// plus ONE barrier -- no inter-CTA hand-off at all (the persistent strip kernel
// pays a TMA ring round trip and a producer warp per step for a row that is
// only 2 KB).  Rows ahead are prefetched PF steps deep into a shared-memory
// ring by cp.async.
// The backward pass reads the forward pass's output, written by the same
// thread: loads of it are issued after the store (program order), and the PF
// planes nearest the turn -- not yet written when their prefetch would issue --
// come from a shared-memory turn buffer filled by the last forward steps.
// Arithmetic is relax_row / Acc (relax.cuh), identical to the strip kernel.
#include <cuda_runtime.h>

#include "relax.cuh"
#include "rowchain.cuh"

namespace gdb {
namespace {

constexpr int kPF = 8;  // prefetch depth (steps)

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)),
                 "l"(gsrc)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int KIND, bool F64>
__global__ void __launch_bounds__(512, 1) row_chain_kernel(const __grid_constant__ SweepParams p) {
    if (gate_closed(p)) return;
    constexpr bool kI = KIND != kSpatial;
    extern __shared__ float4 smem4[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nw = blockDim.x >> 5, nvp = blockDim.x * kC;
    float4* edges = smem4;                                       // [2 parities][nw]: {P0, I0, P3, I3}
    float* tbuf = reinterpret_cast<float*>(smem4 + 2 * nw);      // [kPF][nvp] turn buffer
    float* ringd = tbuf + kPF * nvp;                             // [kPF][nvp] prefetched distances
    float* ringi = ringd + kPF * nvp;                            // [kPF][nvp] prefetched intensities
    const float INF = finf();
    const int v0 = tid * kC;
    bool colv[kC];
#pragma unroll
    for (int q = 0; q < kC; ++q) colv[q] = v0 + q < p.nv;
    const bool any = colv[0];
    // Threads past the row load column 0 (values unused: outputs masked to +inf),
    // so the row loads need no per-thread branch.
    const int v0l = any ? v0 : 0;
    float* const dist = p.dist + static_cast<long long>(blockIdx.x) * p.vol_stride + v0l;
    const float* const img = p.image + static_cast<long long>(blockIdx.x) * p.vol_stride + v0l;
    const int n1 = p.ns - 1, J = p.npass * n1;
    auto plane = [&](int j) {
        if (j <= n1) return p.first_orient > 0 ? j : n1 - j;
        const int k = j - n1;
        return p.first_orient > 0 ? n1 - k : k;
    };
    // Distances of step j come from the turn buffer when the forward pass wrote
    // that plane fewer than kPF steps before step j.
    auto in_turn = [&](int j) { return j > n1 && j <= n1 + kPF; };
    auto ld4 = [&](const float* base, int j) -> float4 {
        return *reinterpret_cast<const float4*>(base + static_cast<long long>(plane(j)) * p.ss);
    };
    auto to_arr = [&](float4 v, float (&a)[kC], float fill) {
        a[0] = colv[0] ? v.x : fill;
        a[1] = colv[1] ? v.y : fill;
        a[2] = colv[2] ? v.z : fill;
        a[3] = colv[3] ? v.w : fill;
    };
    auto save_turn = [&](int j, const float (&N)[kC]) {
        const int t = n1 - j - 1;  // backward step n1 + t + 1 reads this plane
        if (p.npass == 2 && t >= 0 && t < kPF)
            *reinterpret_cast<float4*>(tbuf + t * nvp + v0) = make_float4(N[0], N[1], N[2], N[3]);
    };
    auto put_edges = [&](int j, const float (&N)[kC], const float (&I)[kC]) {
        float4* e = edges + (j & 1) * nw + warp;
        if (lane == 0) { e->x = N[0]; e->y = I[0]; }
        if (lane == kWarpLast) { e->z = N[kC - 1]; e->w = I[kC - 1]; }
    };

    float P[kC], PI[kC];
    // Prefetch ring in shared memory, filled by cp.async (no registers: a
    // register ring made ptxas copy each loaded value right after its load,
    // waiting on it at once -- 13% long_sb stalls).  One commit group per step.
    auto fetch = [&](int j, int u) {
        if (j <= J) {
            if (!in_turn(j)) cp_async16(ringd + u * nvp + v0, dist + static_cast<long long>(plane(j)) * p.ss);
            if (kI) cp_async16(ringi + u * nvp + v0, img + static_cast<long long>(plane(j)) * p.ss);
        }
        cp_async_commit();
    };
    // step 0: the first plane is final as loaded
    {
        float4 d0 = ld4(dist, 0), i0 = kI ? ld4(img, 0) : make_float4(0.f, 0.f, 0.f, 0.f);
        to_arr(d0, P, INF);
        to_arr(i0, PI, 0.0f);
        save_turn(0, P);
        put_edges(0, P, PI);
    }
#pragma unroll
    for (int u = 0; u < kPF; ++u) fetch(1 + u, u);
    __syncthreads();

    // One plane step.  Branch-light (ncu: one warp per scheduler, the step is
    // issue-latency bound -- branches and masks were 1/3 of the stall samples):
    // the warp-edge slots and the turn buffer are read unconditionally and
    // selected; loaded rows are not masked -- a padding column's output is
    // forced to +inf, so its distance is never a finite candidate and its
    // intensity only meets +inf distances (inf or NaN candidates; fminf drops NaN).
    const int wl = warp > 0 ? warp - 1 : 0, wr = warp + 1 < nw ? warp + 1 : warp;
    const bool has_l = warp > 0, has_r = warp + 1 < nw;
    const bool full = colv[kC - 1];
    auto step = [&](int j, int u) {
        cp_async_wait<kPF - 1>();  // this step's group (committed kPF groups ago) has landed
        const float4 rd = *reinterpret_cast<const float4*>(ringd + u * nvp + v0);
        const float4 ri = kI ? *reinterpret_cast<const float4*>(ringi + u * nvp + v0) : make_float4(0.f, 0.f, 0.f, 0.f);
        const float4* e = edges + ((j - 1) & 1) * nw;
        const float4 el = e[wl], er = e[wr];
        float lP = __shfl_up_sync(kFullMask, P[kC - 1], 1);
        float lI = __shfl_up_sync(kFullMask, PI[kC - 1], 1);
        float rP = __shfl_down_sync(kFullMask, P[0], 1);
        float rI = __shfl_down_sync(kFullMask, PI[0], 1);
        if (lane == 0) {
            lP = has_l ? el.z : INF;
            lI = el.w;
        }
        if (lane == kWarpLast) {
            rP = has_r ? er.x : INF;
            rI = er.y;
        }
        const float pw[6] = {lP, P[0], P[1], P[2], P[3], rP};
        const float iw[6] = {lI, PI[0], PI[1], PI[2], PI[3], rI};
        int t = j - n1 - 1;
        const bool turn = t >= 0 && t < kPF;
        t = t < 0 ? 0 : (t >= kPF ? kPF - 1 : t);
        const float4 tv = *reinterpret_cast<const float4*>(tbuf + t * nvp + v0);
        const float4 dv = turn ? tv : rd;
        const float dold[kC] = {dv.x, dv.y, dv.z, dv.w};
        float ic[kC] = {0.0f, 0.0f, 0.0f, 0.0f};
        if (kI) {
            ic[0] = ri.x;
            ic[1] = ri.y;
            ic[2] = ri.z;
            ic[3] = ri.w;
        }
        Acc<KIND, F64> acc[kC];
#pragma unroll
        for (int q = 0; q < kC; ++q) acc[q].init(dold[q]);
        relax_row<KIND, F64>(acc, pw, iw, ic, 0, p);
        float N[kC];
#pragma unroll
        for (int q = 0; q < kC; ++q) N[q] = colv[q] ? acc[q].final(p) : INF;
        float* o = dist + static_cast<long long>(plane(j)) * p.ss;
        if (full) {
            *reinterpret_cast<float4*>(o) = make_float4(N[0], N[1], N[2], N[3]);
        } else if (any) {
#pragma unroll
            for (int q = 0; q < kC; ++q)
                if (colv[q]) o[q] = N[q];
        }
        save_turn(j, N);
        put_edges(j, N, ic);
        // prefetch step j + kPF into the slot just consumed (after the store:
        // a backward plane outside the turn window was written at a step <= j)
        fetch(j + kPF, u);
#pragma unroll
        for (int q = 0; q < kC; ++q) {
            P[q] = N[q];
            PI[q] = ic[q];
        }
        __syncthreads();
    };

    int j0 = 1;
    for (; j0 + kPF - 1 <= J; j0 += kPF) {
#pragma unroll
        for (int u = 0; u < kPF; ++u) step(j0 + u, u);
    }
#pragma unroll
    for (int u = 0; u < kPF; ++u)
        if (j0 + u <= J) step(j0 + u, u);
}

template <int KIND, bool F64>
cudaError_t launch_one(const SweepParams& p, cudaStream_t s) {
    const int threads = ((p.nv + kC - 1) / kC + 31) / 32 * 32;
    const int nw = threads / 32;
    const size_t smem = 2 * nw * sizeof(float4) + 3 * static_cast<size_t>(kPF) * threads * kC * 4;
    if (smem > 48 * 1024) {  // per device: set on every wide launch (cheap)
        const cudaError_t e = cudaFuncSetAttribute(
            row_chain_kernel<KIND, F64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
            static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    row_chain_kernel<KIND, F64><<<p.nvol, threads, smem, s>>>(p);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_row_chain(int kind, bool f64, const SweepParams& p, cudaStream_t s) {
    if (p.nv > kRowChainMaxWidth || p.nu != 1) return cudaErrorInvalidValue;
    switch (kind) {
        case kSpatial: return launch_one<kSpatial, false>(p, s);
        case kIntensity: return f64 ? launch_one<kIntensity, true>(p, s) : launch_one<kIntensity, false>(p, s);
        default: return f64 ? launch_one<kBlend, true>(p, s) : launch_one<kBlend, false>(p, s);
    }
}

}  // namespace gdb
