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

// FADD2 packing of column pairs: off — ptxas cannot fold |d| into the packed
// add and the odd-aligned pairs cost register moves (measured: 86 vs 68
// instructions per voxel); the scalar FADD with an |operand| is cheaper.
constexpr bool kPackedIntensity = false;

// The 3-column windows of one previous-plane row for a lane's 4 columns:
// pw/iw[0] = column v-1, [1..4] = own columns, [5] = column v+4.
template <int KIND, bool F64>
__device__ __forceinline__ void relax_row(Acc<KIND, F64> (&acc)[kC], const float (&pw)[6],
                                          const float (&iw)[6], const float (&ip)[kC], int du,
                                          const SweepParams& p) {
    if constexpr (KIND == kIntensity && !F64 && kPackedIntensity) {
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

template <int RW, int NWU, int NST>
struct Layout {
    static constexpr int R = RW * NWU;                            // rows per strip
    static constexpr int DBOX = R * kWV;                          // floats per column-block box
    static constexpr int IBOX = ((R + 2) * kIW + 31) / 32 * 32;   // 128-B aligned slot stride
    static constexpr int IBYTES = (R + 2) * kIW * 4;
    static size_t smem_bytes(int nwv) {
        return static_cast<size_t>(NST) * nwv * (DBOX + IBOX) * 4     // TMA ring
               + static_cast<size_t>(2) * NWU * 2 * nwv * kWV * 4     // warp-row boundary rows
               + static_cast<size_t>(2) * NWU * nwv * 2 * RW * 4      // warp-edge columns
               + 2 * NST * 8 + 16 + 128;                              // barriers, progress
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

// A previous-plane row window for this lane: own 4 columns from `c4`, the
// neighbours v-1 / v+4 from the adjacent lanes, and at the warp edges from
// `edge_l` / `edge_r` (column 128wv-1 / 128wv+128).
__device__ __forceinline__ void make_window(const float (&c4)[kC], float edge_l, float edge_r,
                                            int lane, float (&win)[6]) {
#pragma unroll
    for (int c = 0; c < kC; ++c) win[c + 1] = c4[c];
    const float up = __shfl_up_sync(kFull, c4[kC - 1], 1);
    const float dn = __shfl_down_sync(kFull, c4[0], 1);
    win[0] = lane == 0 ? edge_l : up;
    win[5] = lane == 31 ? edge_r : dn;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void consumer_sync(int nthreads) {
    asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}
__device__ __forceinline__ void st_release_cta(int* p, int v) {
    asm volatile("st.release.cta.shared.b32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_cta(const int* p) {
    int v;
    asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
    return v;
}

// Warp-specialised persistent sweep: warps [0, NWU*nwv) relax the strip, the
// last warp is the TMA producer.  Slot j % NST carries plane p(j); it is
// released ("empty") by every consumer warp after step j+1, which reads it as
// the previous plane's intensities.
template <int KIND, bool F64, int RW, int NWU, int NST, int MW>
__global__ void __launch_bounds__((MW * NWU + 1) * 32, 1)
    sweep_kernel(const __grid_constant__ CUtensorMap tm_d, const __grid_constant__ CUtensorMap tm_i,
                 const __grid_constant__ SweepParams p) {
    using L = Layout<RW, NWU, NST>;
    constexpr int R = L::R, DBOX = L::DBOX, IBOX = L::IBOX;
    constexpr bool kI = KIND != kSpatial;  // Spatial never reads intensities
    constexpr uint32_t TXW = static_cast<uint32_t>(kI ? DBOX * 4 + L::IBYTES : DBOX * 4);

    const int nwv = p.nwv;
    const int ncw = NWU * nwv;  // consumer warps
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    float* sd = reinterpret_cast<float*>(smem_raw);     // [NST][nwv][R][128]
    float* si = sd + NST * nwv * DBOX;                   // [NST][nwv][R+2][136]
    float* rows = si + NST * nwv * IBOX;                 // [2][NWU][first|last][nwv*128]
    float* edge = rows + 2 * NWU * 2 * nwv * kWV;        // [2][NWU][nwv][left|right][RW]
    uint64_t* full = reinterpret_cast<uint64_t*>(edge + 2 * NWU * nwv * 2 * RW);
    uint64_t* empty = full + NST;
    int* progress = reinterpret_cast<int*>(empty + NST);

    const int g = blockIdx.x;
    const int b = g / p.ntu;
    const int tu = g - b * p.ntu;
    const int u0 = tu * R;
    const int n1 = p.ns - 1;
    const int J = p.npass * n1;
    const int VW = nwv * kWV;

    auto plane_of = [&](int j) -> int {
        if (j <= n1) return p.first_orient > 0 ? j : n1 - j;
        const int k = j - n1;
        return p.first_orient > 0 ? n1 - k : k;
    };

    if (tid == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], ncw);
        }
        *progress = -1;
        fence_mbar_init();
    }
    __syncthreads();

    // ======================= producer warp ==================================
    if (w == ncw) {
        if (lane == 0) {
            tma_prefetch_desc(&tm_d);
            if (kI) tma_prefetch_desc(&tm_i);
            for (int j = 0; j <= J; ++j) {
                const int slot = j % NST, k = j / NST;
                if (k > 0) mbar_wait(&empty[slot], static_cast<uint32_t>((k - 1) & 1));
                // A backward-pass plane is the forward pass's output of step 2*n1 - j.
                if (j > n1) {
                    const int jf = 2 * n1 - j;
                    while (ld_acquire_cta(progress) < jf) {
                    }
                }
                const int s = plane_of(j);
                mbar_arrive_expect_tx(&full[slot], TXW * nwv);
                for (int cb = 0; cb < nwv; ++cb) {
                    float* dd = sd + (slot * nwv + cb) * DBOX;
                    float* di = si + (slot * nwv + cb) * IBOX;
                    const int v0 = cb * kWV;
                    if (p.tma_sweep_dim == 2) {
                        tma_load_4d(dd, &tm_d, &full[slot], v0, u0, s, b);
                        if (kI) tma_load_4d(di, &tm_i, &full[slot], v0 - 4, u0 - 1, s, b);
                    } else {
                        tma_load_4d(dd, &tm_d, &full[slot], v0, s, u0, b);
                        if (kI) tma_load_4d(di, &tm_i, &full[slot], v0 - 4, s, u0 - 1, b);
                    }
                }
            }
        }
        return;
    }

    // ======================= consumer warps =================================
    const int wu = w / nwv, wv = w - wu * nwv;   // warp row / warp column
    const int r0 = wu * RW;                      // first strip row of this warp
    const int v0w = wv * kWV;
    const int vl = v0w + kC * lane;
    const float INF = finf();
    const int nthreads = ncw * 32;

    const bool top_warp = wu == 0, bot_warp = wu == NWU - 1;
    const bool has_up = tu > 0 && top_warp, has_dn = tu + 1 < p.ntu && bot_warp;
    const long long strip_words = 2ll * 2 * VW;  // per strip: 2 parities x {TOP, BOT}
    const long long strip0 = static_cast<long long>(b) * p.ntu;
    const unsigned long long* up_base = p.halo + (strip0 + tu - 1) * strip_words + VW + vl;
    const unsigned long long* dn_base = p.halo + (strip0 + tu + 1) * strip_words + vl;
    unsigned long long* self_base = p.halo + static_cast<long long>(g) * strip_words + vl;
    const bool pub_top = tu > 0 && top_warp, pub_bot = tu + 1 < p.ntu && bot_warp;
    const bool has_left = vl > 0, has_right = vl + kC < p.nv;

    bool rowv[RW], colv[kC];
#pragma unroll
    for (int r = 0; r < RW; ++r) rowv[r] = (u0 + r0 + r) < p.nu;
#pragma unroll
    for (int c = 0; c < kC; ++c) colv[c] = (vl + c) < p.nv;
    const bool all_valid = __all_sync(kFull, (u0 + r0 + RW <= p.nu) && (vl + kC <= p.nv));

    // global output pointers of this lane's rows, advanced per plane
    float* outp[RW];
#pragma unroll
    for (int r = 0; r < RW; ++r)
        outp[r] = p.dist + static_cast<long long>(b) * p.vol_stride +
                  static_cast<long long>(u0 + r0 + r) * p.su + vl;

    float P[RW][kC], IP[RW][kC];  // previous plane: new distances / intensities of own voxels

    // Publishes the strip border rows (tagged, global) and the warp's boundary
    // rows / edge columns (shared) of plane j.
    auto publish = [&](int j, const float (&N)[RW][kC]) {
        if (j < J) {
            const uint32_t tag = p.tag_base + static_cast<uint32_t>(j);
            unsigned long long* q = self_base + (j & 1) * 2ll * VW;
            if (pub_top) {
                st_tagged2(q, N[0][0], N[0][1], tag);
                st_tagged2(q + 2, N[0][2], N[0][3], tag);
            }
            if (pub_bot) {
                st_tagged2(q + VW, N[RW - 1][0], N[RW - 1][1], tag);
                st_tagged2(q + VW + 2, N[RW - 1][2], N[RW - 1][3], tag);
            }
            if (NWU > 1) {
                float* rw_ = rows + (j & 1) * NWU * 2 * VW + wu * 2 * VW;
                *reinterpret_cast<float4*>(rw_ + vl) =
                    make_float4(N[0][0], N[0][1], N[0][2], N[0][3]);
                *reinterpret_cast<float4*>(rw_ + VW + vl) =
                    make_float4(N[RW - 1][0], N[RW - 1][1], N[RW - 1][2], N[RW - 1][3]);
            }
            float* e = edge + (j & 1) * NWU * nwv * 2 * RW + (wu * nwv + wv) * 2 * RW;
#pragma unroll
            for (int r = 0; r < RW; ++r) {
                if (lane == 0) e[r] = N[r][0];
                if (lane == 31) e[RW + r] = N[r][kC - 1];
            }
        }
    };

    // ---- step 0: the first plane is final as loaded --------------------------
    {
        mbar_wait(&full[0], 0u);
        const float* sdc = sd + wv * DBOX;
        const float* sic = si + wv * IBOX;
        float N[RW][kC];
#pragma unroll
        for (int r = 0; r < RW; ++r) {
            const float4 d4 = *reinterpret_cast<const float4*>(sdc + (r0 + r) * kWV + kC * lane);
            N[r][0] = d4.x; N[r][1] = d4.y; N[r][2] = d4.z; N[r][3] = d4.w;
            if (kI) {
                const float4 i4 = *reinterpret_cast<const float4*>(sic + (r0 + r + 1) * kIW + 4 +
                                                                   kC * lane);
                IP[r][0] = i4.x; IP[r][1] = i4.y; IP[r][2] = i4.z; IP[r][3] = i4.w;
            } else {
#pragma unroll
                for (int c = 0; c < kC; ++c) IP[r][c] = 0.0f;
            }
#pragma unroll
            for (int c = 0; c < kC; ++c)
                if (!(rowv[r] && colv[c])) N[r][c] = INF;
        }
        publish(0, N);
#pragma unroll
        for (int r = 0; r < RW; ++r)
#pragma unroll
            for (int c = 0; c < kC; ++c) P[r][c] = N[r][c];
        consumer_sync(nthreads);
    }

    int slot = 0;
    uint32_t phase = 0;
    for (int j = 1; j <= J; ++j) {
        const int pslot = slot;  // previous plane's slot
        if (++slot == NST) {
            slot = 0;
            phase ^= 1u;
        }
        const int par = (j - 1) & 1;
        const long long hoff = par * 2ll * VW;
        const uint32_t want = p.tag_base + static_cast<uint32_t>(j - 1);
        unsigned long long hu[6], hd[6];  // [0] = v-1, [1..4] own, [5] = v+4
        if (has_up) load_halo_row(up_base + hoff, has_left, has_right, hu);
        if (has_dn) load_halo_row(dn_base + hoff, has_left, has_right, hd);

        mbar_wait(&full[slot], phase);
        const float* sdc = sd + (slot * nwv + wv) * DBOX;
        const float* sic = si + (slot * nwv + wv) * IBOX;
        const float* sip = si + (pslot * nwv + wv) * IBOX;  // previous plane's I box
        float dold[RW][kC], ic[RW][kC];
#pragma unroll
        for (int r = 0; r < RW; ++r) {
            const float4 d4 = *reinterpret_cast<const float4*>(sdc + (r0 + r) * kWV + kC * lane);
            dold[r][0] = d4.x; dold[r][1] = d4.y; dold[r][2] = d4.z; dold[r][3] = d4.w;
            if (kI) {
                const float4 i4 = *reinterpret_cast<const float4*>(sic + (r0 + r + 1) * kIW + 4 +
                                                                   kC * lane);
                ic[r][0] = i4.x; ic[r][1] = i4.y; ic[r][2] = i4.z; ic[r][3] = i4.w;
            } else {
#pragma unroll
                for (int c = 0; c < kC; ++c) ic[r][c] = 0.0f;
            }
        }

        const float* rows_prev = rows + par * NWU * 2 * VW;
        const float* edge_prev = edge + par * NWU * nwv * 2 * RW;
        Acc<KIND, F64> acc[RW][kC];
#pragma unroll
        for (int r = 0; r < RW; ++r)
#pragma unroll
            for (int c = 0; c < kC; ++c) acc[r][c].init(dold[r][c]);

        // Intensity window of previous-plane strip row `sr` (box row sr+1).
        auto i_window = [&](int sr, float (&iw)[6]) {
            if (kI) {
                const float* rp = sip + (sr + 1) * kIW;
                const float4 i4 = *reinterpret_cast<const float4*>(rp + 4 + kC * lane);
                const float c4[kC] = {i4.x, i4.y, i4.z, i4.w};
                make_window(c4, rp[3], rp[4 + kWV], lane, iw);
            } else {
#pragma unroll
                for (int i = 0; i < 6; ++i) iw[i] = 0.0f;
            }
        };

        // ---- phase A: previous-plane rows held inside the CTA ----------------
#pragma unroll
        for (int k = 0; k < RW; ++k) {
            float pw[6], iw[6];
            const float eL = wv > 0 ? edge_prev[((wu * nwv + wv - 1) * 2 + 1) * RW + k] : INF;
            const float eR = wv + 1 < nwv ? edge_prev[((wu * nwv + wv + 1) * 2 + 0) * RW + k] : INF;
            make_window(P[k], eL, eR, lane, pw);
            if (kI) {
                const float* rp = sip + (r0 + k + 1) * kIW;
                make_window(IP[k], rp[3], rp[4 + kWV], lane, iw);
            } else {
#pragma unroll
                for (int i = 0; i < 6; ++i) iw[i] = 0.0f;
            }
            // prev row k feeds output rows k-1 (du=+1), k (du=0), k+1 (du=-1)
            if (k - 1 >= 0) relax_row<KIND, F64>(acc[k - 1], pw, iw, ic[k - 1], +1, p);
            relax_row<KIND, F64>(acc[k], pw, iw, ic[k], 0, p);
            if (k + 1 < RW) relax_row<KIND, F64>(acc[k + 1], pw, iw, ic[k + 1], -1, p);
        }
        if (!top_warp) {
            const float* rp = rows_prev + ((wu - 1) * 2 + 1) * VW;  // last row of warp row wu-1
            const float4 q4 = *reinterpret_cast<const float4*>(rp + vl);
            const float c4[kC] = {q4.x, q4.y, q4.z, q4.w};
            float pw[6], iw[6];
            make_window(c4, has_left ? rp[vl - 1] : INF, has_right ? rp[vl + kC] : INF, lane, pw);
            i_window(r0 - 1, iw);
            relax_row<KIND, F64>(acc[0], pw, iw, ic[0], -1, p);
        }
        if (!bot_warp) {
            const float* rp = rows_prev + ((wu + 1) * 2 + 0) * VW;  // first row of warp row wu+1
            const float4 q4 = *reinterpret_cast<const float4*>(rp + vl);
            const float c4[kC] = {q4.x, q4.y, q4.z, q4.w};
            float pw[6], iw[6];
            make_window(c4, has_left ? rp[vl - 1] : INF, has_right ? rp[vl + kC] : INF, lane, pw);
            i_window(r0 + RW, iw);
            relax_row<KIND, F64>(acc[RW - 1], pw, iw, ic[RW - 1], +1, p);
        }

        // ---- phase B: rows above / below the strip (tagged halo) -------------
        if (top_warp || bot_warp) {
            auto fresh = [&](const unsigned long long (&h)[6]) {
                bool ok = true;
#pragma unroll
                for (int i = 0; i < 6; ++i) {
                    const bool need = (i > 0 && i < 5) || (i == 0 ? has_left : has_right);
                    ok = ok && (!need || tag_of(h[i]) == want);
                }
                return ok;
            };
            long long spins = 0;
            while (true) {
                const bool ok_u = !has_up || fresh(hu);
                const bool ok_d = !has_dn || fresh(hd);
                if (__all_sync(kFull, ok_u && ok_d)) break;
                if (!ok_u) load_halo_row(up_base + hoff, has_left, has_right, hu);
                if (!ok_d) load_halo_row(dn_base + hoff, has_left, has_right, hd);
                if (++spins > kSpinLimit) __trap();
            }
            if (top_warp) {
                float pw[6], iw[6];
#pragma unroll
                for (int i = 0; i < 6; ++i) {
                    const bool need = (i > 0 && i < 5) || (i == 0 ? has_left : has_right);
                    pw[i] = (has_up && need) ? val_of(hu[i]) : INF;
                }
                i_window(-1, iw);
                relax_row<KIND, F64>(acc[0], pw, iw, ic[0], -1, p);
            }
            if (bot_warp) {
                float pw[6], iw[6];
#pragma unroll
                for (int i = 0; i < 6; ++i) {
                    const bool need = (i > 0 && i < 5) || (i == 0 ? has_left : has_right);
                    pw[i] = (has_dn && need) ? val_of(hd[i]) : INF;
                }
                i_window(R, iw);
                relax_row<KIND, F64>(acc[RW - 1], pw, iw, ic[RW - 1], +1, p);
            }
        }

        float N[RW][kC];
        if (all_valid) {
#pragma unroll
            for (int r = 0; r < RW; ++r)
#pragma unroll
                for (int c = 0; c < kC; ++c) N[r][c] = acc[r][c].final(p);
        } else {
#pragma unroll
            for (int r = 0; r < RW; ++r)
#pragma unroll
                for (int c = 0; c < kC; ++c)
                    N[r][c] = (rowv[r] && colv[c]) ? acc[r][c].final(p) : INF;
        }

        publish(j, N);

        // ---- store the relaxed plane ------------------------------------------
        const long long soff = static_cast<long long>(plane_of(j)) * p.ss;
        if (all_valid) {
#pragma unroll
            for (int r = 0; r < RW; ++r)
                *reinterpret_cast<float4*>(outp[r] + soff) =
                    make_float4(N[r][0], N[r][1], N[r][2], N[r][3]);
        } else {
#pragma unroll
            for (int r = 0; r < RW; ++r) {
                if (!rowv[r]) continue;
                float* q = outp[r] + soff;
                if (colv[kC - 1]) {
                    *reinterpret_cast<float4*>(q) = make_float4(N[r][0], N[r][1], N[r][2], N[r][3]);
                } else {
#pragma unroll
                    for (int c = 0; c < kC; ++c)
                        if (colv[c]) q[c] = N[r][c];
                }
            }
        }
        if (p.fence_turn && j <= n1) fence_proxy_async_global();

        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[pslot]);  // previous plane's slot fully consumed
        consumer_sync(nthreads);
        if (tid == 0) st_release_cta(progress, j);

#pragma unroll
        for (int r = 0; r < RW; ++r)
#pragma unroll
            for (int c = 0; c < kC; ++c) {
                P[r][c] = N[r][c];
                IP[r][c] = ic[r][c];
            }
    }
}

template <int KIND, bool F64, int RW, int NWU, int NST, int MW>
cudaError_t launch_one(const CUtensorMap& tm_d, const CUtensorMap& tm_i, const SweepParams& p,
                       cudaStream_t stream) {
    using L = Layout<RW, NWU, NST>;
    auto fn = sweep_kernel<KIND, F64, RW, NWU, NST, MW>;
    const size_t smem = L::smem_bytes(p.nwv);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    const int grid = p.nvol * p.ntu;
    void* args[] = {const_cast<CUtensorMap*>(&tm_d), const_cast<CUtensorMap*>(&tm_i),
                    const_cast<SweepParams*>(&p)};
    return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(fn), dim3(grid),
                                       dim3((p.nwv * NWU + 1) * 32),
                                       args, smem, stream);
}

template <int KIND, bool F64, int RW, int NWU, int NST, int MW>
int coresident(int nwv) {
    using L = Layout<RW, NWU, NST>;
    auto fn = sweep_kernel<KIND, F64, RW, NWU, NST, MW>;
    const size_t smem = L::smem_bytes(nwv);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, (nwv * NWU + 1) * 32, smem) !=
        cudaSuccess)
        return 0;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return per_sm * sms;
}

constexpr int kNST = 4;

// Strip shapes (rows per warp RW, warp rows NWU, max warp columns MW): narrow
// planes (<= 512 columns) run 2 warp rows of 2 rows (R = 4, 2 warps per
// scheduler); R = 1 serves single-row planes (2D).  Wide planes (<= 2048
// columns) trade registers for warps.
#define GD_SWEEP_CASES(X) \
    X(1, 1, 4) X(2, 1, 4) X(2, 2, 4) X(4, 2, 4) X(1, 1, 16) X(2, 1, 16) X(4, 1, 16)

int width_class(int nwv) { return nwv <= 4 ? 4 : 16; }

// R -> (RW, NWU): 1 -> (1,1), 2 -> (2,1), 4 -> (2,2), 8 -> (4,2)
template <int KIND, bool F64>
cudaError_t dispatch_r(int R, const CUtensorMap& tm_d, const CUtensorMap& tm_i,
                       const SweepParams& p, cudaStream_t s) {
    const int mw = width_class(p.nwv);
#define GD_CASE(RWW, NW, MM)                                         \
    if (R == RWW * NW && mw == MM)                                   \
        return launch_one<KIND, F64, RWW, NW, kNST, MM>(tm_d, tm_i, p, s);
    GD_SWEEP_CASES(GD_CASE)
#undef GD_CASE
    return cudaErrorInvalidValue;
}

template <int KIND, bool F64>
int dispatch_cores(int R, int nwv) {
    const int mw = width_class(nwv);
#define GD_CASE(RWW, NW, MM) \
    if (R == RWW * NW && mw == MM) return coresident<KIND, F64, RWW, NW, kNST, MM>(nwv);
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
        case 1: return Layout<1, 1, kNST>::smem_bytes(nwv);
        case 2: return Layout<2, 1, kNST>::smem_bytes(nwv);
        case 4: return Layout<2, 2, kNST>::smem_bytes(nwv);
        case 8: return Layout<4, 2, kNST>::smem_bytes(nwv);
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
