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

__device__ __forceinline__ unsigned long long f2_bits(float2 v) {
    return (static_cast<unsigned long long>(__float_as_uint(v.y)) << 32) | __float_as_uint(v.x);
}
__device__ __forceinline__ float2 bits_f2(unsigned long long b) {
    return make_float2(__uint_as_float(static_cast<uint32_t>(b)),
                       __uint_as_float(static_cast<uint32_t>(b >> 32)));
}
// Packed sm_100 f32x2 arithmetic (SASS FADD2); |x| folds into the operand.
__device__ __forceinline__ float2 f2_sub(float2 a, float2 b) {
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_bits(a)), "l"(f2_bits(b)));
    return bits_f2(r);
}
__device__ __forceinline__ float2 f2_add(float2 a, float2 b) {
    unsigned long long r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_bits(a)), "l"(f2_bits(b)));
    return bits_f2(r);
}

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
        // class representatives (du,dv) = (0,0),(1,0),(0,1),(1,1) -> k = 4,7,5,8
        float r = best;
        r = fminf(r, static_cast<float>(static_cast<double>(m[0]) + p.rho[4]));
        r = fminf(r, static_cast<float>(static_cast<double>(m[1]) + p.rho[7]));
        r = fminf(r, static_cast<float>(static_cast<double>(m[2]) + p.rho[5]));
        r = fminf(r, static_cast<float>(static_cast<double>(m[3]) + p.rho[8]));
        return r;
    }
};

// The 3-column windows of one previous-plane row for a lane's 4 columns:
// pw/iw[0] = column v-1, [1..4] = own columns, [5] = column v+4.
template <int KIND, bool F64>
__device__ __forceinline__ void relax_row(Acc<KIND, F64> (&acc)[kC], const float (&pw)[6],
                                          const float (&iw)[6], const float (&ip)[kC], int du,
                                          const SweepParams& p) {
    if constexpr (KIND == kIntensity && !F64) {
        // Packed column pairs: two FADD2 per candidate pair instead of four FADD.
#pragma unroll
        for (int q = 0; q < kC / 2; ++q) {
            const int c0 = 2 * q;
            const float2 ip2 = make_float2(ip[c0], ip[c0 + 1]);
#pragma unroll
            for (int dv = -1; dv <= 1; ++dv) {
                const float2 pq = make_float2(pw[c0 + dv + 1], pw[c0 + dv + 2]);
                const float2 iq = make_float2(iw[c0 + dv + 1], iw[c0 + dv + 2]);
                float2 d = f2_sub(ip2, iq);
                d.x = fabsf(d.x);
                d.y = fabsf(d.y);
                const float2 cand = f2_add(pq, d);
                acc[c0].best = fminf(acc[c0].best, cand.x);
                acc[c0 + 1].best = fminf(acc[c0 + 1].best, cand.y);
            }
        }
    } else {
#pragma unroll
        for (int c = 0; c < kC; ++c)
#pragma unroll
            for (int dv = -1; dv <= 1; ++dv)
                acc[c].add(pw[c + dv + 1], iw[c + dv + 1], ip[c], (du + 1) * 3 + (dv + 1), p);
    }
}

template <int R, int NST>
struct Layout {
    static constexpr int DBOX = R * kWV;                          // floats per warp box
    static constexpr int IBOX = ((R + 2) * kIW + 31) / 32 * 32;   // 128-B aligned slot stride
    static constexpr int IBYTES = (R + 2) * kIW * 4;
    static size_t smem_bytes(int nwv) {
        return static_cast<size_t>(NST) * nwv * (DBOX + IBOX) * 4  // TMA ring
               + static_cast<size_t>(2) * nwv * 2 * R * 4          // warp-edge columns
               + NST * 8 + 128;
    }
};

// Relaxed loads of one halo row's window: words v-1 .. v+4 of the published row.
__device__ __forceinline__ void load_halo_row(const unsigned long long* q, bool has_left,
                                              bool has_right, unsigned long long (&h)[6]) {
    h[0] = has_left ? ld_tagged(q - 1) : 0ull;
    ld_tagged2(q, h[1], h[2]);
    ld_tagged2(q + 2, h[3], h[4]);
    h[5] = has_right ? ld_tagged(q + 4) : 0ull;
}

template <int KIND, bool F64, int R, int NST, int MW>
__global__ void __launch_bounds__(MW * 32, 1)
    sweep_kernel(const __grid_constant__ CUtensorMap tm_d, const __grid_constant__ CUtensorMap tm_i,
                 const __grid_constant__ SweepParams p) {
    using L = Layout<R, NST>;
    constexpr int DBOX = L::DBOX, IBOX = L::IBOX;
    // Spatial (lambda == 0) never reads intensities: only the distance box moves.
    constexpr uint32_t TXW =
        static_cast<uint32_t>(KIND == kSpatial ? DBOX * 4 : DBOX * 4 + L::IBYTES);

    const int nwv = p.nwv;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    float* sd = reinterpret_cast<float*>(smem_raw);   // [NST][nwv][R][128]
    float* si = sd + NST * nwv * DBOX;                 // [NST][nwv][R+2][136]
    float* edge = si + NST * nwv * IBOX;               // [2][nwv][2][R]  (left col, right col)
    uint64_t* bar = reinterpret_cast<uint64_t*>(edge + 2 * nwv * 2 * R);

    const int g = blockIdx.x;
    const int b = g / p.ntu;
    const int tu = g - b * p.ntu;
    const int u0 = tu * R;
    const int v0w = w * kWV;              // first column of this warp
    const int vl = v0w + kC * lane;        // first column of this lane
    const int n1 = p.ns - 1;
    const int J = p.npass * n1;
    const float INF = finf();
    const int VW = nwv * kWV;             // halo row length (words)

    auto plane_of = [&](int j) -> int {
        if (j <= n1) return p.first_orient > 0 ? j : n1 - j;
        const int k = j - n1;
        return p.first_orient > 0 ? n1 - k : k;
    };

    if (tid == 0) {
        for (int s = 0; s < NST; ++s) mbar_init(&bar[s], nwv);
        fence_mbar_init();
    }
    if (lane == 0) {
        tma_prefetch_desc(&tm_d);
        if (KIND != kSpatial) tma_prefetch_desc(&tm_i);
    }
    __syncthreads();

    // Each warp's lane 0 streams its own column block; the slot's mbarrier
    // completes when all nwv warps' boxes have landed.
    int issued = 0;
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
            mbar_arrive_expect_tx(&bar[slot], TXW);
            float* dd = sd + (slot * nwv + w) * DBOX;
            float* di = si + (slot * nwv + w) * IBOX;
            if (p.tma_sweep_dim == 2) {
                tma_load_4d(dd, &tm_d, &bar[slot], v0w, u0, s, b);
                if (KIND != kSpatial) tma_load_4d(di, &tm_i, &bar[slot], v0w - 4, u0 - 1, s, b);
            } else {
                tma_load_4d(dd, &tm_d, &bar[slot], v0w, s, u0, b);
                if (KIND != kSpatial) tma_load_4d(di, &tm_i, &bar[slot], v0w - 4, s, u0 - 1, b);
            }
            ++issued;
        }
    };

    // Tagged halo rows: the strip above publishes its BOT row, the one below its TOP row.
    const bool has_up = tu > 0, has_dn = tu + 1 < p.ntu;
    const long long strip_words = 2ll * 2 * VW;  // per strip: 2 parities x {TOP, BOT}
    const long long strip0 = static_cast<long long>(b) * p.ntu;
    const unsigned long long* up_base = p.halo + (strip0 + tu - 1) * strip_words + VW + vl;
    const unsigned long long* dn_base = p.halo + (strip0 + tu + 1) * strip_words + vl;
    unsigned long long* self_base = p.halo + static_cast<long long>(g) * strip_words + vl;
    const bool has_left = vl > 0, has_right = vl + kC < p.nv;  // lane-level edge words

    // Validity of this thread's voxels (rows beyond nu / columns beyond nv are +inf).
    bool rowv[R], colv[kC];
#pragma unroll
    for (int r = 0; r < R; ++r) rowv[r] = (u0 + r) < p.nu;
#pragma unroll
    for (int c = 0; c < kC; ++c) colv[c] = (vl + c) < p.nv;

    float P[R][kC], IP[R][kC];  // previous plane: new distances / intensities of own voxels

    for (int j = 0; j <= J; ++j) {
        __syncthreads();  // step j-1 complete: edge columns visible, slot (j-2)%NST free
        if (lane == 0) issue(j);

        const int par = (j - 1) & 1;
        const long long hoff = par * 2ll * VW;
        const uint32_t want = p.tag_base + static_cast<uint32_t>(j - 1);
        // halo words for the previous plane: [0] = v-1, [1..4] own, [5] = v+4
        unsigned long long hu[6], hd[6];
        if (j > 0) {
            if (has_up) load_halo_row(up_base + hoff, has_left, has_right, hu);
            if (has_dn) load_halo_row(dn_base + hoff, has_left, has_right, hd);
        }

        const int slot = j % NST;
        mbar_wait(&bar[slot], static_cast<uint32_t>((j / NST) & 1));
        const float* sdc = sd + (slot * nwv + w) * DBOX;
        const float* sic = si + (slot * nwv + w) * IBOX;
        float dold[R][kC], ic[R][kC];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const float4 d4 = *reinterpret_cast<const float4*>(sdc + r * kWV + kC * lane);
            dold[r][0] = d4.x; dold[r][1] = d4.y; dold[r][2] = d4.z; dold[r][3] = d4.w;
            if (KIND != kSpatial) {
                const float4 i4 =
                    *reinterpret_cast<const float4*>(sic + (r + 1) * kIW + 4 + kC * lane);
                ic[r][0] = i4.x; ic[r][1] = i4.y; ic[r][2] = i4.z; ic[r][3] = i4.w;
            } else {
#pragma unroll
                for (int c = 0; c < kC; ++c) ic[r][c] = 0.0f;
            }
        }

        float N[R][kC];
        if (j == 0) {
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int c = 0; c < kC; ++c) N[r][c] = (rowv[r] && colv[c]) ? dold[r][c] : INF;
        } else {
            const float* sip = si + (((j - 1) % NST) * nwv + w) * IBOX;  // previous plane's I box
            const float* edge_prev = edge + par * nwv * 2 * R;
            Acc<KIND, F64> acc[R][kC];
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int c = 0; c < kC; ++c) acc[r][c].init(dold[r][c]);

            // ---- phase A: previous-plane rows inside the strip --------------
#pragma unroll
            for (int k = 0; k < R; ++k) {
                float pw[6], iw[6];
#pragma unroll
                for (int c = 0; c < kC; ++c) {
                    pw[c + 1] = P[k][c];
                    iw[c + 1] = IP[k][c];
                }
                // v-1: lane-1's last column; at the warp edge, the left warp's right column
                const float eL = w > 0 ? edge_prev[((w - 1) * 2 + 1) * R + k] : INF;
                const float eR = w + 1 < nwv ? edge_prev[((w + 1) * 2 + 0) * R + k] : INF;
                pw[0] = __shfl_up_sync(kFull, P[k][kC - 1], 1);
                pw[5] = __shfl_down_sync(kFull, P[k][0], 1);
                if (lane == 0) pw[0] = eL;
                if (lane == 31) pw[5] = eR;
                if (KIND != kSpatial) {
                    iw[0] = __shfl_up_sync(kFull, IP[k][kC - 1], 1);
                    iw[5] = __shfl_down_sync(kFull, IP[k][0], 1);
                    if (lane == 0) iw[0] = sip[(k + 1) * kIW + 3];
                    if (lane == 31) iw[5] = sip[(k + 1) * kIW + 4 + kWV];
                } else {
                    iw[0] = iw[5] = 0.0f;
                }
                // prev row k feeds output rows k-1 (du=+1), k (du=0), k+1 (du=-1)
                if (k - 1 >= 0) relax_row<KIND, F64>(acc[k - 1], pw, iw, ic[k - 1], +1, p);
                relax_row<KIND, F64>(acc[k], pw, iw, ic[k], 0, p);
                if (k + 1 < R) relax_row<KIND, F64>(acc[k + 1], pw, iw, ic[k + 1], -1, p);
            }

            // ---- phase B: the rows above / below the strip (tagged halo) -----
            if (has_up || has_dn) {
                long long spins = 0;
                while (true) {
                    bool ok = true;
#pragma unroll
                    for (int i = 0; i < 6; ++i) {
                        const bool need = (i > 0 && i < 5) || (i == 0 ? has_left : has_right);
                        if (has_up && need && tag_of(hu[i]) != want) {
                            hu[i] = ld_tagged(up_base + hoff + i - 1);
                            ok = false;
                        }
                        if (has_dn && need && tag_of(hd[i]) != want) {
                            hd[i] = ld_tagged(dn_base + hoff + i - 1);
                            ok = false;
                        }
                    }
                    if (ok) break;
                    if (++spins > kSpinLimit) __trap();
                }
            }
#pragma unroll
            for (int side = 0; side < 2; ++side) {
                // side 0: row u0-1 -> output row 0 (du = -1); side 1: row u0+R -> row R-1 (du = +1)
                const bool has = side == 0 ? has_up : has_dn;
                float pw[6], iw[6];
#pragma unroll
                for (int i = 0; i < 6; ++i) {
                    const bool need = (i > 0 && i < 5) || (i == 0 ? has_left : has_right);
                    pw[i] = (has && need) ? val_of(side == 0 ? hu[i] : hd[i]) : INF;
                }
                if (KIND != kSpatial) {
                    const float* rowp = sip + (side == 0 ? 0 : (R + 1) * kIW);
                    const float4 i4 = *reinterpret_cast<const float4*>(rowp + 4 + kC * lane);
                    iw[1] = i4.x; iw[2] = i4.y; iw[3] = i4.z; iw[4] = i4.w;
                    iw[0] = __shfl_up_sync(kFull, iw[4], 1);
                    iw[5] = __shfl_down_sync(kFull, iw[1], 1);
                    if (lane == 0) iw[0] = rowp[3];
                    if (lane == 31) iw[5] = rowp[4 + kWV];
                } else {
#pragma unroll
                    for (int i = 0; i < 6; ++i) iw[i] = 0.0f;
                }
                if (side == 0)
                    relax_row<KIND, F64>(acc[0], pw, iw, ic[0], -1, p);
                else
                    relax_row<KIND, F64>(acc[R - 1], pw, iw, ic[R - 1], +1, p);
            }
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int c = 0; c < kC; ++c)
                    N[r][c] = (rowv[r] && colv[c]) ? acc[r][c].final(p) : INF;
        }

        // ---- publish the strip's first / last row: the neighbours' critical path
        if (j < J) {
            const uint32_t tag = p.tag_base + static_cast<uint32_t>(j);
            unsigned long long* q = self_base + (j & 1) * 2ll * VW;
            if (has_up) {
                st_tagged2(q, N[0][0], N[0][1], tag);
                st_tagged2(q + 2, N[0][2], N[0][3], tag);
            }
            if (has_dn) {
                st_tagged2(q + VW, N[R - 1][0], N[R - 1][1], tag);
                st_tagged2(q + VW + 2, N[R - 1][2], N[R - 1][3], tag);
            }
            float* e = edge + (j & 1) * nwv * 2 * R;
            if (lane == 0) {
#pragma unroll
                for (int r = 0; r < R; ++r) e[(w * 2 + 0) * R + r] = N[r][0];
            }
            if (lane == 31) {
#pragma unroll
                for (int r = 0; r < R; ++r) e[(w * 2 + 1) * R + r] = N[r][kC - 1];
            }
        }

        // ---- store the relaxed plane ------------------------------------------
        if (j > 0) {
            const int s = plane_of(j);
            float* base = p.dist + static_cast<long long>(b) * p.vol_stride +
                          static_cast<long long>(s) * p.ss + vl;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if (!rowv[r]) continue;
                float* q = base + static_cast<long long>(u0 + r) * p.su;
                if (colv[kC - 1]) {
                    *reinterpret_cast<float4*>(q) = make_float4(N[r][0], N[r][1], N[r][2], N[r][3]);
                } else {
#pragma unroll
                    for (int c = 0; c < kC; ++c)
                        if (colv[c]) q[c] = N[r][c];
                }
            }
            if (p.fence_turn && j <= n1) fence_proxy_async_global();
        }

#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int c = 0; c < kC; ++c) {
                P[r][c] = N[r][c];
                IP[r][c] = ic[r][c];
            }
    }
}

template <int KIND, bool F64, int R, int NST, int MW>
cudaError_t launch_one(const CUtensorMap& tm_d, const CUtensorMap& tm_i, const SweepParams& p,
                       cudaStream_t stream) {
    using L = Layout<R, NST>;
    auto fn = sweep_kernel<KIND, F64, R, NST, MW>;
    const size_t smem = L::smem_bytes(p.nwv);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    const int grid = p.nvol * p.ntu;
    void* args[] = {const_cast<CUtensorMap*>(&tm_d), const_cast<CUtensorMap*>(&tm_i),
                    const_cast<SweepParams*>(&p)};
    return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(fn), dim3(grid), dim3(p.nwv * 32),
                                       args, smem, stream);
}

template <int KIND, bool F64, int R, int NST, int MW>
int coresident(int nwv) {
    using L = Layout<R, NST>;
    auto fn = sweep_kernel<KIND, F64, R, NST, MW>;
    const size_t smem = L::smem_bytes(nwv);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, nwv * 32, smem) != cudaSuccess)
        return 0;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return per_sm * sms;
}

constexpr int kNST = 4;

// (rows per strip, max warps per strip): narrow planes (<= 512 columns) get the
// full 255-register budget; wide ones (<= 2048) trade registers for warps.
#define GD_SWEEP_CASES(X) X(1, 4) X(2, 4) X(4, 4) X(8, 4) X(1, 16) X(2, 16) X(4, 16)

int width_class(int nwv) { return nwv <= 4 ? 4 : 16; }

template <int KIND, bool F64>
cudaError_t dispatch_r(int R, const CUtensorMap& tm_d, const CUtensorMap& tm_i,
                       const SweepParams& p, cudaStream_t s) {
    const int mw = width_class(p.nwv);
#define GD_CASE(RR, MM) \
    if (R == RR && mw == MM) return launch_one<KIND, F64, RR, kNST, MM>(tm_d, tm_i, p, s);
    GD_SWEEP_CASES(GD_CASE)
#undef GD_CASE
    return cudaErrorInvalidValue;
}

template <int KIND, bool F64>
int dispatch_cores(int R, int nwv) {
    const int mw = width_class(nwv);
#define GD_CASE(RR, MM) \
    if (R == RR && mw == MM) return coresident<KIND, F64, RR, kNST, MM>(nwv);
    GD_SWEEP_CASES(GD_CASE)
#undef GD_CASE
    return 0;
}

}  // namespace

cudaError_t launch_sweep(int kind, bool f64, int R, const CUtensorMap& tm_d,
                         const CUtensorMap& tm_i, const SweepParams& p, cudaStream_t stream) {
    switch (kind) {
        case kSpatial:
            return dispatch_r<kSpatial, false>(R, tm_d, tm_i, p, stream);
        case kIntensity:
            return f64 ? dispatch_r<kIntensity, true>(R, tm_d, tm_i, p, stream)
                       : dispatch_r<kIntensity, false>(R, tm_d, tm_i, p, stream);
        default:
            return f64 ? dispatch_r<kBlend, true>(R, tm_d, tm_i, p, stream)
                       : dispatch_r<kBlend, false>(R, tm_d, tm_i, p, stream);
    }
}

size_t sweep_smem_bytes(int R, int nwv) {
    switch (R) {
        case 1: return Layout<1, kNST>::smem_bytes(nwv);
        case 2: return Layout<2, kNST>::smem_bytes(nwv);
        case 4: return Layout<4, kNST>::smem_bytes(nwv);
        case 8: return Layout<8, kNST>::smem_bytes(nwv);
    }
    return 0;
}

int sweep_max_coresident(int R, int nwv, int kind, bool f64) {
    switch (kind) {
        case kSpatial: return dispatch_cores<kSpatial, false>(R, nwv);
        case kIntensity:
            return f64 ? dispatch_cores<kIntensity, true>(R, nwv)
                       : dispatch_cores<kIntensity, false>(R, nwv);
        default:
            return f64 ? dispatch_cores<kBlend, true>(R, nwv)
                       : dispatch_cores<kBlend, false>(R, nwv);
    }
}

}  // namespace gdb
