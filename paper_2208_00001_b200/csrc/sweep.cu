// Persistent directional-pass kernel (see sweep.cuh for the design notes).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>

#include "sweep.cuh"

namespace gdb {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr long long kSpinLimit = 1ll << 24;  // ~seconds of polling: a protocol bug traps, never hangs

__device__ __forceinline__ float finf() { return __int_as_float(0x7f800000); }

// One relaxation candidate d_q + cost(p, q) rounded to f32 (see sweep.cuh for
// why per-candidate rounding is exact).  k = (du+1)*3 + (dv+1).
template <int KIND, bool F64>
__device__ __forceinline__ float candidate(float pq, float iq, float ip, int k,
                                           const SweepParams& p) {
    if constexpr (KIND == kSpatial) {
        return static_cast<float>(static_cast<double>(pq) + p.rho[k]);
    } else if constexpr (KIND == kIntensity) {
        if constexpr (F64) {
            const double di = static_cast<double>(ip) - static_cast<double>(iq);
            return static_cast<float>(static_cast<double>(pq) + fabs(di));
        } else {
            return pq + fabsf(ip - iq);
        }
    } else {
        if constexpr (F64) {
            const double di = static_cast<double>(ip) - static_cast<double>(iq);
            // relax_cost<Blend> as compiled by the reference: sqrt(fma(lambda*di, di, c0))
            return static_cast<float>(static_cast<double>(pq) +
                                      sqrt(fma(p.lambda * di, di, p.c0[k])));
        } else {
            const float di = ip - iq;
            return pq + sqrtf(fmaf(p.lambda_f * di, di, p.c0_f[k]));
        }
    }
}

// Per-voxel accumulator.  Spatial keeps one f32 minimum per rho class
// (class = (du != 0) + 2 (dv != 0)) and adds rho once per class at the end.
template <int KIND, bool F64>
struct Acc {
    float best;
    __device__ __forceinline__ void init(float dold) { best = dold; }
    __device__ __forceinline__ void add(float pq, float iq, float ip, int k, const SweepParams& p) {
        best = fminf(best, candidate<KIND, F64>(pq, iq, ip, k, p));
    }
    __device__ __forceinline__ float final(const SweepParams&) const { return best; }
};

template <bool F64>
struct Acc<kSpatial, F64> {
    float best;
    float m[4];
    __device__ __forceinline__ void init(float dold) {
        best = dold;
        m[0] = m[1] = m[2] = m[3] = finf();
    }
    __device__ __forceinline__ void add(float pq, float, float, int k, const SweepParams&) {
        const int du = k / 3 - 1, dv = k % 3 - 1;
        const int c = (du != 0 ? 1 : 0) + (dv != 0 ? 2 : 0);
        m[c] = fminf(m[c], pq);
    }
    __device__ __forceinline__ float final(const SweepParams& p) const {
        // class representative coefficient: (du,dv) = (0,0),(1,0),(0,1),(1,1) -> k = 4,7,5,8
        float r = best;
        r = fminf(r, static_cast<float>(static_cast<double>(m[0]) + p.rho[4]));
        r = fminf(r, static_cast<float>(static_cast<double>(m[1]) + p.rho[7]));
        r = fminf(r, static_cast<float>(static_cast<double>(m[2]) + p.rho[5]));
        r = fminf(r, static_cast<float>(static_cast<double>(m[3]) + p.rho[8]));
        return r;
    }
};

template <int R, int NWU, int NST>
struct Layout {
    static constexpr int TU = NWU * R;
    static constexpr int NT = NWU * 32;
    static constexpr int IH = TU + 2;
    static constexpr int DBOX = TU * kTV;
    // slot stride rounded to 128 B: TMA destinations must be 128-byte aligned
    static constexpr int IBOX = (IH * kIW + 31) / 32 * 32;
    static constexpr int IBYTES = IH * kIW * 4;
    static constexpr int HALO_N = 2 * kTV + 2 * TU;     // published words per tile per parity
    static constexpr int NREAD = 2 * kTV + 2 * (TU + 2); // halo words read per step
    static constexpr int MAXE = (NREAD + NT - 1) / NT;
    static constexpr int SMEM_FLOATS =
        NST * DBOX + NST * IBOX + 2 * kTV * 2 + 2 * (TU + 2) * 2 + 2 * NWU * kTV * 2;
    static constexpr size_t SMEM_BYTES = SMEM_FLOATS * 4 + NST * 8 + 16;
};

template <int KIND, bool F64, int R, int NWU, int NST>
__global__ void __launch_bounds__(NWU * 32, 1)
    sweep_kernel(const __grid_constant__ CUtensorMap tm_d, const __grid_constant__ CUtensorMap tm_i,
                 const __grid_constant__ SweepParams p) {
    using L = Layout<R, NWU, NST>;
    constexpr int TU = L::TU, NT = L::NT, DBOX = L::DBOX, IBOX = L::IBOX;
    // Spatial (lambda == 0) never reads intensities: only the distance box moves.
    constexpr uint32_t TX =
        static_cast<uint32_t>(KIND == kSpatial ? DBOX * 4 : DBOX * 4 + L::IBYTES);

    extern __shared__ __align__(128) unsigned char smem_raw[];
    float* sd = reinterpret_cast<float*>(smem_raw);   // [NST][TU][64]       old distances
    float* si = sd + NST * DBOX;                       // [NST][TU+2][72]     intensities + halo
    float* hT = si + NST * IBOX;                       // [2][64]  row u0-1 (prev plane)
    float* hB = hT + 2 * kTV;                          // [2][64]  row u0+TU
    float* hL = hB + 2 * kTV;                          // [2][TU+2] col v0-1, rows u0-1..u0+TU
    float* hR = hL + 2 * (TU + 2);                     // [2][TU+2] col v0+64
    float* rT = hR + 2 * (TU + 2);                     // [2][NWU][64] first row of each warp
    float* rB = rT + 2 * NWU * kTV;                    // [2][NWU][64] last row of each warp
    uint64_t* bar = reinterpret_cast<uint64_t*>(rB + 2 * NWU * kTV);

    const int tid = threadIdx.x, lane = tid & 31, wu = tid >> 5;
    const int tiles_per_vol = p.ntu * p.ntv;
    const int g = blockIdx.x;
    const int b = g / tiles_per_vol;
    const int rem = g - b * tiles_per_vol;
    const int tu = rem / p.ntv, tv = rem - tu * p.ntv;
    const int u0 = tu * TU, v0 = tv * kTV;
    const int n1 = p.ns - 1;
    const int J = p.npass * n1;
    const float INF = finf();

    auto plane_of = [&](int j) -> int {
        if (j <= n1) return p.first_orient > 0 ? j : n1 - j;
        const int k = j - n1;
        return p.first_orient > 0 ? n1 - k : k;
    };

    if (tid == 0) {
        for (int s = 0; s < NST; ++s) mbar_init(&bar[s], 1);
        fence_mbar_init();
        tma_prefetch_desc(&tm_d);
        tma_prefetch_desc(&tm_i);
    }
    __syncthreads();

    int issued = 0;  // next step whose planes thread 0 will request
    auto issue = [&](int t) {
        // Slot j % NST is free once step j-NST+1 (which reads it as the
        // previous plane) has finished: j <= t + NST - 2 at the top of step t.
        // A backward-pass plane must first be written by the forward pass
        // (step 2*n1 - j), i.e. that step must be complete: 2*n1 - j <= t - 1.
        while (issued <= J && issued <= t + NST - 2) {
            const int j = issued;
            if (j > n1 && 2 * n1 - j > t - 1) break;
            const int slot = j % NST;
            const int s = plane_of(j);
            mbar_arrive_expect_tx(&bar[slot], TX);
            if (p.tma_sweep_dim == 2) {
                tma_load_4d(sd + slot * DBOX, &tm_d, &bar[slot], v0, u0, s, b);
                if (KIND != kSpatial)
                    tma_load_4d(si + slot * IBOX, &tm_i, &bar[slot], v0 - 4, u0 - 1, s, b);
            } else {
                tma_load_4d(sd + slot * DBOX, &tm_d, &bar[slot], v0, s, u0, b);
                if (KIND != kSpatial)
                    tma_load_4d(si + slot * IBOX, &tm_i, &bar[slot], v0 - 4, s, u0 - 1, b);
            }
            ++issued;
        }
    };

    // ---- halo words this thread reads every step ----------------------------
    long long src_w[L::MAXE];  // word index for parity 0, or -1 (outside the tile grid)
    float* dst_s[L::MAXE];     // smem destination for parity 0
    int pstride[L::MAXE];      // smem parity stride of that destination
#pragma unroll
    for (int q = 0; q < L::MAXE; ++q) {
        const int e = tid + q * NT;
        src_w[q] = -1;
        dst_s[q] = nullptr;
        pstride[q] = 0;
        if (e >= L::NREAD) continue;
        int ntu_ = -1, ntv_ = -1, woff = 0;
        if (e < kTV) {  // row above <- BOT of tile (tu-1, tv)
            ntu_ = tu - 1; ntv_ = tv; woff = kTV + e;
            dst_s[q] = hT + e; pstride[q] = kTV;
        } else if (e < 2 * kTV) {  // row below <- TOP of tile (tu+1, tv)
            ntu_ = tu + 1; ntv_ = tv; woff = e - kTV;
            dst_s[q] = hB + (e - kTV); pstride[q] = kTV;
        } else {
            const bool left = e < 2 * kTV + TU + 2;
            const int i = left ? e - 2 * kTV : e - 2 * kTV - (TU + 2);
            ntv_ = left ? tv - 1 : tv + 1;
            const int col_base = left ? 2 * kTV + TU /*RIGHT*/ : 2 * kTV /*LEFT*/;
            if (i == 0) { ntu_ = tu - 1; woff = col_base + TU - 1; }
            else if (i <= TU) { ntu_ = tu; woff = col_base + i - 1; }
            else { ntu_ = tu + 1; woff = col_base; }
            dst_s[q] = (left ? hL : hR) + i; pstride[q] = TU + 2;
        }
        if (ntu_ >= 0 && ntu_ < p.ntu && ntv_ >= 0 && ntv_ < p.ntv) {
            const long long nb = (static_cast<long long>(b) * p.ntu + ntu_) * p.ntv + ntv_;
            src_w[q] = nb * 2 * L::HALO_N + woff;
        }
    }
    const long long self_w = static_cast<long long>(g) * 2 * L::HALO_N;

    // Validity of this thread's voxels.
    bool valid[R][2];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int c = 0; c < 2; ++c)
            valid[r][c] = (u0 + wu * R + r) < p.nu && (v0 + 2 * lane + c) < p.nv;

    float P[R][2], IP[R][2];  // previous plane: new distances / intensities of own voxels

    for (int j = 0; j <= J; ++j) {
        __syncthreads();  // step j-1 complete: its smem rows/halo visible, slot (j-2)%NST free
        if (tid == 0) issue(j);

        const int par = (j - 1) & 1;  // parity of the previous plane's halo/rows
        const uint32_t want = p.tag_base + static_cast<uint32_t>(j - 1);
        unsigned long long hw[L::MAXE];
        if (j > 0) {
#pragma unroll
            for (int q = 0; q < L::MAXE; ++q)
                hw[q] = src_w[q] >= 0 ? ld_tagged(p.halo + src_w[q] + par * L::HALO_N) : 0ull;
        }

        const int slot = j % NST;
        mbar_wait(&bar[slot], static_cast<uint32_t>((j / NST) & 1));
        const float* sdc = sd + slot * DBOX;
        const float* sic = si + slot * IBOX;
        float2 dold[R], ic[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            dold[r] = *reinterpret_cast<const float2*>(sdc + (wu * R + r) * kTV + 2 * lane);
            ic[r] = *reinterpret_cast<const float2*>(sic + (wu * R + r + 1) * kIW + 4 + 2 * lane);
        }

        float N[R][2];
        if (j == 0) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                N[r][0] = valid[r][0] ? dold[r].x : INF;
                N[r][1] = valid[r][1] ? dold[r].y : INF;
            }
        } else {
            const float* sip = si + ((j - 1) % NST) * IBOX;  // previous plane's intensities
            // Previous-plane rows wu*R-1 .. wu*R+R as (left, c0, c1, right) quads.
            float p0[R + 2], p1[R + 2], i0[R + 2], i1[R + 2];
            {
                const float2 ia = *reinterpret_cast<const float2*>(sip + (wu * R) * kIW + 4 + 2 * lane);
                const float2 ib =
                    *reinterpret_cast<const float2*>(sip + (wu * R + R + 1) * kIW + 4 + 2 * lane);
                i0[0] = ia.x; i1[0] = ia.y;
                i0[R + 1] = ib.x; i1[R + 1] = ib.y;
                if (wu > 0) {
                    const float2 pa = *reinterpret_cast<const float2*>(
                        rB + (par * NWU + wu - 1) * kTV + 2 * lane);
                    p0[0] = pa.x; p1[0] = pa.y;
                } else {
                    p0[0] = p1[0] = INF;
                }
                if (wu < NWU - 1) {
                    const float2 pb = *reinterpret_cast<const float2*>(
                        rT + (par * NWU + wu + 1) * kTV + 2 * lane);
                    p0[R + 1] = pb.x; p1[R + 1] = pb.y;
                } else {
                    p0[R + 1] = p1[R + 1] = INF;
                }
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    p0[r + 1] = P[r][0]; p1[r + 1] = P[r][1];
                    i0[r + 1] = IP[r][0]; i1[r + 1] = IP[r][1];
                }
            }
            float pL[R + 2], pR[R + 2], iL[R + 2], iR[R + 2];
#pragma unroll
            for (int k = 0; k < R + 2; ++k) {
                pL[k] = __shfl_up_sync(kFull, p1[k], 1);
                pR[k] = __shfl_down_sync(kFull, p0[k], 1);
                if (KIND != kSpatial) {
                    iL[k] = __shfl_up_sync(kFull, i1[k], 1);
                    iR[k] = __shfl_down_sync(kFull, i0[k], 1);
                } else {
                    iL[k] = iR[k] = 0.0f;
                }
                if (lane == 0) pL[k] = INF;   // column v0-1: halo, phase B
                if (lane == 31) pR[k] = INF;  // column v0+64: halo, phase B
            }

            // ---- phase A: everything available inside the CTA -----------------
            Acc<KIND, F64> acc[R][2];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                acc[r][0].init(dold[r].x);
                acc[r][1].init(dold[r].y);
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    const int k = r + a;  // prev row index in the quads
                    acc[r][0].add(pL[k], iL[k], ic[r].x, a * 3 + 0, p);
                    acc[r][0].add(p0[k], i0[k], ic[r].x, a * 3 + 1, p);
                    acc[r][0].add(p1[k], i1[k], ic[r].x, a * 3 + 2, p);
                    acc[r][1].add(p0[k], i0[k], ic[r].y, a * 3 + 0, p);
                    acc[r][1].add(p1[k], i1[k], ic[r].y, a * 3 + 1, p);
                    acc[r][1].add(pR[k], iR[k], ic[r].y, a * 3 + 2, p);
                }
            }

            // ---- halo: resolve the tagged words, publish to smem --------------
#pragma unroll
            for (int q = 0; q < L::MAXE; ++q) {
                if (dst_s[q] == nullptr) continue;
                float v = INF;
                if (src_w[q] >= 0) {
                    unsigned long long w = hw[q];
                    long long spins = 0;
                    while (tag_of(w) != want) {
                        w = ld_tagged(p.halo + src_w[q] + par * L::HALO_N);
                        if (++spins > kSpinLimit) __trap();
                    }
                    v = val_of(w);
                }
                dst_s[q][par * pstride[q]] = v;
            }
            __syncthreads();

            // ---- phase B: border voxels take their out-of-tile neighbours -----
            const float* hTp = hT + par * kTV;
            const float* hBp = hB + par * kTV;
            const float* hLp = hL + par * (TU + 2);
            const float* hRp = hR + par * (TU + 2);
            if (wu == 0) {  // row 0 <- row u0-1 (du = -1), corners from hL/hR
                const float m1 = lane == 0 ? hLp[0] : hTp[2 * lane - 1];
                const float q0 = hTp[2 * lane], q1 = hTp[2 * lane + 1];
                const float q2 = lane == 31 ? hRp[0] : hTp[2 * lane + 2];
                const float* ir = sip + 3 + 2 * lane;  // box row 0
                acc[0][0].add(m1, ir[0], ic[0].x, 0, p);
                acc[0][0].add(q0, ir[1], ic[0].x, 1, p);
                acc[0][0].add(q1, ir[2], ic[0].x, 2, p);
                acc[0][1].add(q0, ir[1], ic[0].y, 0, p);
                acc[0][1].add(q1, ir[2], ic[0].y, 1, p);
                acc[0][1].add(q2, ir[3], ic[0].y, 2, p);
            }
            if (wu == NWU - 1) {  // row R-1 <- row u0+TU (du = +1)
                const float m1 = lane == 0 ? hLp[TU + 1] : hBp[2 * lane - 1];
                const float q0 = hBp[2 * lane], q1 = hBp[2 * lane + 1];
                const float q2 = lane == 31 ? hRp[TU + 1] : hBp[2 * lane + 2];
                const float* ir = sip + (TU + 1) * kIW + 3 + 2 * lane;
                acc[R - 1][0].add(m1, ir[0], ic[R - 1].x, 6, p);
                acc[R - 1][0].add(q0, ir[1], ic[R - 1].x, 7, p);
                acc[R - 1][0].add(q1, ir[2], ic[R - 1].x, 8, p);
                acc[R - 1][1].add(q0, ir[1], ic[R - 1].y, 6, p);
                acc[R - 1][1].add(q1, ir[2], ic[R - 1].y, 7, p);
                acc[R - 1][1].add(q2, ir[3], ic[R - 1].y, 8, p);
            }
            if (lane == 0) {  // column v0-1 (dv = -1) for c = 0
#pragma unroll
                for (int r = 0; r < R; ++r)
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        const int row = wu * R + r + a;  // box/halo row index (row -1 -> 0)
                        acc[r][0].add(hLp[row], sip[row * kIW + 3], ic[r].x, a * 3 + 0, p);
                    }
            }
            if (lane == 31) {  // column v0+64 (dv = +1) for c = 1
#pragma unroll
                for (int r = 0; r < R; ++r)
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        const int row = wu * R + r + a;
                        acc[r][1].add(hRp[row], sip[row * kIW + 68], ic[r].y, a * 3 + 2, p);
                    }
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                N[r][0] = valid[r][0] ? acc[r][0].final(p) : INF;
                N[r][1] = valid[r][1] ? acc[r][1].final(p) : INF;
            }
        }

        // ---- publish the tile border first: it is on the neighbours' critical path
        if (j < J) {
            const uint32_t tag = p.tag_base + static_cast<uint32_t>(j);
            unsigned long long* hw_self = p.halo + self_w + (j & 1) * L::HALO_N;
            if (wu == 0) {
                st_tagged(hw_self + 2 * lane, N[0][0], tag);
                st_tagged(hw_self + 2 * lane + 1, N[0][1], tag);
            }
            if (wu == NWU - 1) {
                st_tagged(hw_self + kTV + 2 * lane, N[R - 1][0], tag);
                st_tagged(hw_self + kTV + 2 * lane + 1, N[R - 1][1], tag);
            }
            if (lane == 0) {
#pragma unroll
                for (int r = 0; r < R; ++r) st_tagged(hw_self + 2 * kTV + wu * R + r, N[r][0], tag);
            }
            if (lane == 31) {
#pragma unroll
                for (int r = 0; r < R; ++r)
                    st_tagged(hw_self + 2 * kTV + TU + wu * R + r, N[r][1], tag);
            }
            if (NWU > 1) {
                *reinterpret_cast<float2*>(rT + ((j & 1) * NWU + wu) * kTV + 2 * lane) =
                    make_float2(N[0][0], N[0][1]);
                *reinterpret_cast<float2*>(rB + ((j & 1) * NWU + wu) * kTV + 2 * lane) =
                    make_float2(N[R - 1][0], N[R - 1][1]);
            }
        }

        // ---- store the relaxed plane ------------------------------------------
        if (j > 0) {
            const int s = plane_of(j);
            float* base = p.dist + static_cast<long long>(b) * p.vol_stride +
                          static_cast<long long>(s) * p.ss;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int u = u0 + wu * R + r;
                const int v = v0 + 2 * lane;
                float* q = base + static_cast<long long>(u) * p.su + v;
                if (valid[r][1]) {
                    *reinterpret_cast<float2*>(q) = make_float2(N[r][0], N[r][1]);
                } else if (valid[r][0]) {
                    q[0] = N[r][0];
                }
            }
            if (p.fence_turn && j <= n1) fence_proxy_async_global();
        }

#pragma unroll
        for (int r = 0; r < R; ++r) {
            P[r][0] = N[r][0];
            P[r][1] = N[r][1];
            IP[r][0] = ic[r].x;
            IP[r][1] = ic[r].y;
        }
    }
}

template <int KIND, bool F64, int R, int NWU, int NST>
cudaError_t launch_one(const CUtensorMap& tm_d, const CUtensorMap& tm_i, const SweepParams& p,
                       cudaStream_t stream) {
    using L = Layout<R, NWU, NST>;
    auto fn = sweep_kernel<KIND, F64, R, NWU, NST>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(L::SMEM_BYTES));
        if (e != cudaSuccess) return e;
        configured = true;
    }
    const int grid = p.nvol * p.ntu * p.ntv;
    void* args[] = {const_cast<CUtensorMap*>(&tm_d), const_cast<CUtensorMap*>(&tm_i),
                    const_cast<SweepParams*>(&p)};
    return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(fn), dim3(grid), dim3(L::NT), args,
                                       L::SMEM_BYTES, stream);
}

template <int KIND, bool F64, int R, int NWU, int NST>
int coresident(void) {
    using L = Layout<R, NWU, NST>;
    auto fn = sweep_kernel<KIND, F64, R, NWU, NST>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(L::SMEM_BYTES));
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, L::NT, L::SMEM_BYTES) !=
        cudaSuccess)
        return 0;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return per_sm * sms;
}

constexpr int kNST = 4;

template <int KIND, bool F64>
cudaError_t dispatch_tile(int R, int NWU, const CUtensorMap& tm_d, const CUtensorMap& tm_i,
                          const SweepParams& p, cudaStream_t s) {
    if (R == 4 && NWU == 8) return launch_one<KIND, F64, 4, 8, kNST>(tm_d, tm_i, p, s);
    if (R == 1 && NWU == 1) return launch_one<KIND, F64, 1, 1, kNST>(tm_d, tm_i, p, s);
    return cudaErrorInvalidValue;
}

template <int KIND, bool F64>
int dispatch_cores(int R, int NWU) {
    if (R == 4 && NWU == 8) return coresident<KIND, F64, 4, 8, kNST>();
    if (R == 1 && NWU == 1) return coresident<KIND, F64, 1, 1, kNST>();
    return 0;
}

}  // namespace

cudaError_t launch_sweep(int kind, bool f64, int R, int NWU, const CUtensorMap& tm_d,
                         const CUtensorMap& tm_i, const SweepParams& p, cudaStream_t stream) {
    switch (kind) {
        case kSpatial:
            return dispatch_tile<kSpatial, false>(R, NWU, tm_d, tm_i, p, stream);
        case kIntensity:
            return f64 ? dispatch_tile<kIntensity, true>(R, NWU, tm_d, tm_i, p, stream)
                       : dispatch_tile<kIntensity, false>(R, NWU, tm_d, tm_i, p, stream);
        default:
            return f64 ? dispatch_tile<kBlend, true>(R, NWU, tm_d, tm_i, p, stream)
                       : dispatch_tile<kBlend, false>(R, NWU, tm_d, tm_i, p, stream);
    }
}

size_t sweep_smem_bytes(int R, int NWU) {
    if (R == 4 && NWU == 8) return Layout<4, 8, kNST>::SMEM_BYTES;
    if (R == 1 && NWU == 1) return Layout<1, 1, kNST>::SMEM_BYTES;
    return 0;
}

int sweep_max_coresident(int R, int NWU, int kind, bool f64) {
    switch (kind) {
        case kSpatial: return dispatch_cores<kSpatial, false>(R, NWU);
        case kIntensity:
            return f64 ? dispatch_cores<kIntensity, true>(R, NWU)
                       : dispatch_cores<kIntensity, false>(R, NWU);
        default:
            return f64 ? dispatch_cores<kBlend, true>(R, NWU) : dispatch_cores<kBlend, false>(R, NWU);
    }
}

}  // namespace gdb
