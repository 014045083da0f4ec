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

__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
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
            // MUFU.SQRT (about 1 ulp): the IEEE sqrtf adds a slow-path CALL per
            // candidate that serialises the 9-candidate min (3x slower step).
            const float di = ip - iq;
            return pq + sqrt_approx(fmaf(p.lambda_f * di, di, p.c0_f[k]));
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
        // Rounding to f32 is monotone, so the min of the f64 sums rounds to the
        // min of the rounded sums: one F2F down instead of four (conversions
        // run at a quarter of the FP32 rate).  No NaNs reach here.
        const double s0 = static_cast<double>(m[0]) + p.rho[4];
        const double s1 = static_cast<double>(m[1]) + p.rho[7];
        const double s2 = static_cast<double>(m[2]) + p.rho[5];
        const double s3 = static_cast<double>(m[3]) + p.rho[8];
        const double a = s0 < s1 ? s0 : s1, b = s2 < s3 ? s2 : s3;
        return fminf(best, static_cast<float>(a < b ? a : b));
    }
};

// FADD2 packing of column pairs: off — ptxas cannot fold |d| into the packed
// add and the odd-aligned pairs cost register moves (measured: 86 vs 68
// instructions per voxel); the scalar FADD with an |operand| is cheaper.
constexpr bool kPackedIntensity = false;

// Second halo poll issued mid-step (alternating spin).  Measured slower on
// B200 (1.48 vs 1.24 us/step at 512^2): the extra loads and registers cost more
// than the earlier detection gains.
#ifndef GD_DUAL_POLL
#define GD_DUAL_POLL 0
#endif
constexpr bool kDualPoll = GD_DUAL_POLL != 0;

#ifndef GD_NST4
#define GD_NST4 6
#endif
#ifndef GD_MINB2
#define GD_MINB2 3  // R = 4 strips of <= 256 columns: 3 CTAs per SM (batches; measured 97 -> 81 ms)
#endif
#ifndef GD_EARLY_POLL
#define GD_EARLY_POLL 0
#endif

// Cycle counters for diagnosis (built only with -DGD_SWEEP_TRACE).
#ifdef GD_SWEEP_TRACE
#define GD_T0(v) const long long v = clock64()
#define GD_TADD(slot, v) trc[slot] += clock64() - (v)
#define GD_DBG(bit) ((p.debug_flags & (bit)) != 0)
#else
#define GD_T0(v)
#define GD_TADD(slot, v)
#define GD_DBG(bit) false
#endif

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

// Window of a fresh halo row: own words h[1..4], neighbour lanes' edge words by
// shuffle, h[0] / h[5] at the warp edges; INF outside the plane or strip set.
__device__ __forceinline__ void halo_window(const unsigned long long (&h)[6], bool present,
                                            bool has_left, bool has_right, int lane,
                                            float (&win)[6]) {
    const float inf = __int_as_float(0x7f800000);
    const float c4[kC] = {val_of(h[1]), val_of(h[2]), val_of(h[3]), val_of(h[4])};
    make_window(c4, val_of(h[0]), val_of(h[5]), lane, win);
#pragma unroll
    for (int i = 0; i < 6; ++i)
        if (!present) win[i] = inf;
    if (!has_left) win[0] = inf;
    if (!has_right) win[5] = inf;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    // relaxed: only smem reads (already consumed) precede it; a release arrive
    // would wait (MEMBAR) on this thread's outstanding global stores.
    asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void consumer_sync(int nthreads) {
    asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}
// AND of `pred` over the consumer threads (named barrier 1, like consumer_sync).
__device__ __forceinline__ bool consumer_all(bool pred, int nthreads) {
    int r;
    asm volatile(
        "{\n\t.reg .pred p, q;\n\tsetp.ne.s32 p, %1, 0;\n\t"
        "barrier.cta.red.and.pred q, 1, %2, p;\n\tselp.s32 %0, 1, 0, q;\n\t}"
        : "=r"(r)
        : "r"(static_cast<int>(pred)), "r"(nthreads)
        : "memory");
    return r != 0;
}
__device__ __forceinline__ void st_release_cta(int* p, int v) {
    asm volatile("st.release.cta.shared.b32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_cta(const int* p) {
    int v;
    asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
    return v;
}

// Shared-memory carve-up and launch geometry, common to producer and consumers.
template <int RW, int NWU, int NST>
struct Ctx {
    float* sd;          // [NST][nwv][R][128]      old distances (TMA)
    float* si;          // [NST][nwv][R+2][136]    intensities + row halo (TMA)
    float* rows;        // [2][NWU][first|last][nwv*128] warp-row boundary rows
    float* edge;        // [2][NWU][nwv][left|right][RW] warp-edge columns
    uint64_t* full;     // [NST]
    uint64_t* empty;    // [NST]
    int* progress;
    int nwv, g, b, tu, u0, n1, J, VW;
};

template <int RW, int NWU, int NST>
__device__ __forceinline__ int plane_of(const SweepParams& p, const Ctx<RW, NWU, NST>& c, int j) {
    if (j <= c.n1) return p.first_orient > 0 ? j : c.n1 - j;
    const int k = j - c.n1;
    return p.first_orient > 0 ? c.n1 - k : k;
}

// One consumer warp's whole sweep.  TOP / BOT: the warp row borders the strip
// above / below (tagged global halo); FULL: every voxel of the warp is inside
// the volume.  Specialising on the role keeps the per-step body branch-free.
template <int KIND, bool F64, int RW, int NWU, int NST, bool TOP, bool BOT, bool FULL>
__device__ __forceinline__ void consumer_loop(const SweepParams& p, const Ctx<RW, NWU, NST>& c,
                                              int wu, int wv, int lane) {
    using L = Layout<RW, NWU, NST>;
    constexpr int R = L::R, DBOX = L::DBOX, IBOX = L::IBOX;
    constexpr bool kI = KIND != kSpatial;
    const int nwv = c.nwv, VW = c.VW, J = c.J, n1 = c.n1;
    const int r0 = wu * RW;
    const int vl = wv * kWV + kC * lane;
    const float INF = finf();
    const int nthreads = NWU * nwv * 32;
    const int tid = (wu * nwv + wv) * 32 + lane;
    const uint32_t tag_base = p.tag_base;
    const bool turn_fence = p.fence_turn != 0;

    const bool has_up = TOP && c.tu > 0, has_dn = BOT && c.tu + 1 < p.ntu;
    const long long strip_words = 2ll * 2 * VW;  // per strip: 2 parities x {TOP, BOT}
    const long long strip0 = static_cast<long long>(c.b) * p.ntu;
    // Halo row layout (per warp column block of 128 words): columns q = 0,1 of
    // all 32 lanes, then q = 2,3 -- lane l owns words 2l, 2l+1, 64+2l, 65+2l, so
    // each 16-byte access of the warp covers 512 contiguous bytes (16 full
    // sectors) instead of half of 32 sectors.  v-1 / v+4 come from the adjacent
    // lanes; only lane 0 / lane 31 load the neighbour block's edge word.
    const bool has_left = vl > 0, has_right = vl + kC < p.nv;
    const bool edge_l = lane == 0 && has_left, edge_r = lane == 31 && has_right;
    const int hl = wv * kWV + 2 * lane;
    const unsigned long long* up0 = p.halo + (strip0 + c.tu - 1) * strip_words + VW + hl;
    const unsigned long long* dn0 = p.halo + (strip0 + c.tu + 1) * strip_words + hl;
    unsigned long long* self0 = p.halo + static_cast<long long>(c.g) * strip_words + hl;
    const bool pub_up = TOP && c.tu > 0, pub_dn = BOT && c.tu + 1 < p.ntu;
    // neighbour-warp edge columns
    const int eoffL = ((wu * nwv + wv - 1) * 2 + 1) * RW;
    const int eoffR = ((wu * nwv + wv + 1) * 2 + 0) * RW;
    const bool wl = wv > 0, wr = wv + 1 < nwv;
    float* const edge_own = c.edge + (wu * nwv + wv) * 2 * RW;
    const int EPAR = NWU * nwv * 2 * RW;  // edge buffer parity stride
    const int RPAR = NWU * 2 * VW;        // rows buffer parity stride

    bool rowv[RW], colv[kC];
#pragma unroll
    for (int r = 0; r < RW; ++r) rowv[r] = (c.u0 + r0 + r) < p.nu;
#pragma unroll
    for (int q = 0; q < kC; ++q) colv[q] = (vl + q) < p.nv;

    // Output pointer of this lane's first row at the current plane; rows are su apart.
    const long long su = p.su;
    float* outp = p.dist + static_cast<long long>(c.b) * p.vol_stride +
                  static_cast<long long>(c.u0 + r0) * su + vl +
                  static_cast<long long>(plane_of(p, c, 0)) * p.ss;
    long long dsoff = p.first_orient > 0 ? p.ss : -p.ss;

    // Shared-memory slot pointers (this warp's column block).
    const float* const sd_base = c.sd + wv * DBOX;
    const float* const si_base = c.si + wv * IBOX;
    const int SD_STRIDE = nwv * DBOX, SI_STRIDE = nwv * IBOX;

    auto publish_halo = [&](int j, const float (&N)[RW][kC]) {
        const int par = j & 1;
        const uint32_t tag = tag_base + static_cast<uint32_t>(j);
        unsigned long long* q = self0 + par * 2ll * VW;
        if (GD_DBG(2)) return;
        if (pub_up) {
            st_tagged2(q, N[0][0], N[0][1], tag);
            st_tagged2(q + 64, N[0][2], N[0][3], tag);
        }
        if (pub_dn) {
            st_tagged2(q + VW, N[RW - 1][0], N[RW - 1][1], tag);
            st_tagged2(q + VW + 64, N[RW - 1][2], N[RW - 1][3], tag);
        }
    };
    auto publish_smem = [&](int j, const float (&N)[RW][kC]) {
        const int par = j & 1;
        if (NWU > 1) {
            float* rw_ = c.rows + par * RPAR + wu * 2 * VW;
            if (!TOP)
                *reinterpret_cast<float4*>(rw_ + vl) =
                    make_float4(N[0][0], N[0][1], N[0][2], N[0][3]);
            if (!BOT)
                *reinterpret_cast<float4*>(rw_ + VW + vl) =
                    make_float4(N[RW - 1][0], N[RW - 1][1], N[RW - 1][2], N[RW - 1][3]);
        }
        float* e = edge_own + par * EPAR;
#pragma unroll
        for (int r = 0; r < RW; ++r) {
            if (lane == 0) e[r] = N[r][0];
            if (lane == 31) e[RW + r] = N[r][kC - 1];
        }
    };

    float PA[RW][kC], IA[RW][kC], PB[RW][kC], IB[RW][kC];
#ifdef GD_SWEEP_TRACE
    long long trc[12] = {};  // tma, spin, barrier, reloads, total, steps, phaseA, tail, pre, crit, post, -
    const long long t_begin = clock64();
#endif

    // ---- step 0: the first plane is final as loaded ----------------------------
    {
        mbar_wait(&c.full[0], 0u);
#pragma unroll
        for (int r = 0; r < RW; ++r) {
            const float4 d4 =
                *reinterpret_cast<const float4*>(sd_base + (r0 + r) * kWV + kC * lane);
            PA[r][0] = d4.x; PA[r][1] = d4.y; PA[r][2] = d4.z; PA[r][3] = d4.w;
            if (kI) {
                const float4 i4 = *reinterpret_cast<const float4*>(si_base + (r0 + r + 1) * kIW +
                                                                   4 + kC * lane);
                IA[r][0] = i4.x; IA[r][1] = i4.y; IA[r][2] = i4.z; IA[r][3] = i4.w;
            } else {
#pragma unroll
                for (int q = 0; q < kC; ++q) IA[r][q] = 0.0f;
            }
            if (!FULL) {
#pragma unroll
                for (int q = 0; q < kC; ++q)
                    if (!(rowv[r] && colv[q])) PA[r][q] = INF;
            }
        }
        if (J > 0) {
            publish_halo(0, PA);
            publish_smem(0, PA);
        }
        consumer_sync(nthreads);
    }

    int slot = 0;
    uint32_t phase = 0;
    const float* sd_cur = sd_base;
    const float* si_cur = si_base;

    auto load_row = [&](const unsigned long long* q, unsigned long long (&h)[6]) {
        ld_tagged2(q, h[1], h[2]);
        ld_tagged2(q + 64, h[3], h[4]);
        h[0] = edge_l ? ld_tagged(q - 1) : 0ull;   // previous block, last word
        h[5] = edge_r ? ld_tagged(q + 66) : 0ull;  // next block, first word
    };
    // First poll of the next step's halo rows (published at step j), issued
    // GD_EARLY_POLL = 1: right after this strip publishes its own step-j rows,
    // 2: just before the step barrier; 0: at the top of the next step.
    unsigned long long huN[6], hdN[6];
    auto early_poll = [&](int j) {
        const int par = j & 1;
        if (TOP && has_up) load_row(up0 + par * 2ll * VW, huN);
        if (BOT && has_dn) load_row(dn0 + par * 2ll * VW, hdN);
    };
    if (GD_EARLY_POLL != 0 && J > 0) early_poll(0);

    // One relaxation step: plane j from the previous plane (Pin, Iin) into (Pout, Iout).
    auto step = [&](int j, const float (&Pin)[RW][kC], const float (&Iin)[RW][kC],
                    float (&Pout)[RW][kC], float (&Iout)[RW][kC]) {
        GD_T0(t_entry);
        const int pslot = slot;
        const float* sip = si_cur;  // previous plane's I box
        if (++slot == NST) {
            slot = 0;
            phase ^= 1u;
            sd_cur = sd_base;
            si_cur = si_base;
        } else {
            sd_cur += SD_STRIDE;
            si_cur += SI_STRIDE;
        }
        const int par = (j - 1) & 1;
        const uint32_t want = tag_base + static_cast<uint32_t>(j - 1);
        const unsigned long long* hup = up0 + par * 2ll * VW;
        const unsigned long long* hdn = dn0 + par * 2ll * VW;
        // Two polls of each halo window are kept in flight: A at the top of the
        // step, B after the strip's own rows are relaxed; the spin alternates
        // between them so a fresh word is seen within about half a round trip.
        // [0] = v-1, [1..4] own, [5] = v+4.  Poll A lives in huN/hdN (no copy:
        // a register copy of an in-flight load would stall right there).
        unsigned long long(&huA)[6] = huN;
        unsigned long long(&hdA)[6] = hdN;
        unsigned long long huB[6], hdB[6];
        if (GD_EARLY_POLL == 0 && !GD_DBG(4)) {
            if (TOP && has_up) load_row(hup, huA);
            if (BOT && has_dn) load_row(hdn, hdA);
        }

        GD_TADD(8, t_entry);
        GD_T0(t_tma);
        mbar_wait(&c.full[slot], phase);
        GD_TADD(0, t_tma);
        GD_T0(t_pa);
        float dold[RW][kC], ic[RW][kC];
#pragma unroll
        for (int r = 0; r < RW; ++r) {
            const float4 d4 =
                *reinterpret_cast<const float4*>(sd_cur + (r0 + r) * kWV + kC * lane);
            dold[r][0] = d4.x; dold[r][1] = d4.y; dold[r][2] = d4.z; dold[r][3] = d4.w;
            if (kI) {
                const float4 i4 = *reinterpret_cast<const float4*>(si_cur + (r0 + r + 1) * kIW +
                                                                   4 + kC * lane);
                ic[r][0] = i4.x; ic[r][1] = i4.y; ic[r][2] = i4.z; ic[r][3] = i4.w;
            } else {
#pragma unroll
                for (int q = 0; q < kC; ++q) ic[r][q] = 0.0f;
            }
        }

        const float* rows_prev = c.rows + par * RPAR;
        const float* edge_prev = c.edge + par * EPAR;
        Acc<KIND, F64> acc[RW][kC];
#pragma unroll
        for (int r = 0; r < RW; ++r)
#pragma unroll
            for (int q = 0; q < kC; ++q) acc[r][q].init(dold[r][q]);

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
            const float eL = wl ? edge_prev[eoffL + k] : INF;
            const float eR = wr ? edge_prev[eoffR + k] : INF;
            make_window(Pin[k], eL, eR, lane, pw);
            if (kI) {
                const float* rp = sip + (r0 + k + 1) * kIW;
                make_window(Iin[k], rp[3], rp[4 + kWV], lane, iw);
            } else {
#pragma unroll
                for (int i = 0; i < 6; ++i) iw[i] = 0.0f;
            }
            if (k - 1 >= 0) relax_row<KIND, F64>(acc[k - 1], pw, iw, ic[k - 1], +1, p);
            relax_row<KIND, F64>(acc[k], pw, iw, ic[k], 0, p);
            if (k + 1 < RW) relax_row<KIND, F64>(acc[k + 1], pw, iw, ic[k + 1], -1, p);
        }
        if (kDualPoll) {
            if (TOP && has_up) load_row(hup, huB);
            if (BOT && has_dn) load_row(hdn, hdB);
        }
        if (!TOP) {
            const float* rp = rows_prev + ((wu - 1) * 2 + 1) * VW;  // last row of warp row wu-1
            const float4 q4 = *reinterpret_cast<const float4*>(rp + vl);
            const float c4[kC] = {q4.x, q4.y, q4.z, q4.w};
            float pw[6], iw[6];
            make_window(c4, has_left ? rp[vl - 1] : INF, has_right ? rp[vl + kC] : INF, lane, pw);
            i_window(r0 - 1, iw);
            relax_row<KIND, F64>(acc[0], pw, iw, ic[0], -1, p);
        }
        if (!BOT) {
            const float* rp = rows_prev + ((wu + 1) * 2 + 0) * VW;  // first row of warp row wu+1
            const float4 q4 = *reinterpret_cast<const float4*>(rp + vl);
            const float c4[kC] = {q4.x, q4.y, q4.z, q4.w};
            float pw[6], iw[6];
            make_window(c4, has_left ? rp[vl - 1] : INF, has_right ? rp[vl + kC] : INF, lane, pw);
            i_window(r0 + RW, iw);
            relax_row<KIND, F64>(acc[RW - 1], pw, iw, ic[RW - 1], +1, p);
        }

        // ---- phase B: rows above / below the strip (tagged halo) -------------
#ifdef GD_SWEEP_TRACE
        long long t_tail0_outer = 0;
#endif
        if (TOP || BOT) {
            auto fresh = [&](const unsigned long long (&h)[6]) {
                bool ok = (!edge_l || tag_of(h[0]) == want) && (!edge_r || tag_of(h[5]) == want);
#pragma unroll
                for (int i = 1; i <= kC; ++i) ok = ok && tag_of(h[i]) == want;
                return ok;
            };
            long long spins = 0;
            GD_TADD(6, t_pa);
            GD_T0(t_spin);
            bool useB = false;
            while (!GD_DBG(1)) {
                const bool ok = useB ? ((!(TOP && has_up) || fresh(huB)) &&
                                        (!(BOT && has_dn) || fresh(hdB)))
                                     : ((!(TOP && has_up) || fresh(huA)) &&
                                        (!(BOT && has_dn) || fresh(hdA)));
                if (__all_sync(kFull, ok)) break;
                if (useB) {
                    if (TOP && has_up) load_row(hup, huB);
                    if (BOT && has_dn) load_row(hdn, hdB);
                } else {
                    if (TOP && has_up) load_row(hup, huA);
                    if (BOT && has_dn) load_row(hdn, hdA);
                }
                if (kDualPoll) useB = !useB;
                if (++spins > kSpinLimit) __trap();
            }
            GD_TADD(1, t_spin);
#ifdef GD_SWEEP_TRACE
            t_tail0_outer = clock64();
#endif
#ifdef GD_SWEEP_TRACE
            trc[3] += spins;
#endif
            unsigned long long hu[6], hd[6];
#pragma unroll
            for (int i = 0; i < 6; ++i) {
                hu[i] = useB ? huB[i] : huA[i];
                hd[i] = useB ? hdB[i] : hdA[i];
            }
            if (TOP) {
                float pw[6], iw[6];
                halo_window(hu, has_up, has_left, has_right, lane, pw);
                i_window(-1, iw);
                relax_row<KIND, F64>(acc[0], pw, iw, ic[0], -1, p);
            }
            if (BOT) {
                float pw[6], iw[6];
                halo_window(hd, has_dn, has_left, has_right, lane, pw);
                i_window(R, iw);
                relax_row<KIND, F64>(acc[RW - 1], pw, iw, ic[RW - 1], +1, p);
            }
        }
        // The previous plane's slot is no longer read by this warp.
        __syncwarp();
        if (lane == 0) mbar_arrive(&c.empty[pslot]);

        auto fin = [&](int r) {
#pragma unroll
            for (int q = 0; q < kC; ++q) {
                Pout[r][q] = acc[r][q].final(p);
                if (!FULL && !(rowv[r] && colv[q])) Pout[r][q] = INF;
                Iout[r][q] = ic[r][q];
            }
        };
        // Border rows first: they are the neighbours' critical path.
        if (TOP) fin(0);
        if (BOT && (RW > 1 || !TOP)) fin(RW - 1);
        if (j < J) publish_halo(j, Pout);
#ifdef GD_SWEEP_TRACE
        if (TOP || BOT) trc[9] += clock64() - t_tail0_outer;
#endif
        if (GD_EARLY_POLL == 1 && j < J) early_poll(j);
#pragma unroll
        for (int r = 0; r < RW; ++r)
            if (!((TOP && r == 0) || (BOT && r == RW - 1))) fin(r);
        if (j < J) publish_smem(j, Pout);

        // ---- store the relaxed plane ------------------------------------------
        if (j == n1 + 1) dsoff = -dsoff;  // the backward pass walks back
        outp += dsoff;
#pragma unroll
        for (int r = 0; r < RW; ++r) {
            float* q = outp + r * su;
            if (FULL) {
                *reinterpret_cast<float4*>(q) =
                    make_float4(Pout[r][0], Pout[r][1], Pout[r][2], Pout[r][3]);
            } else if (rowv[r]) {
                if (colv[kC - 1]) {
                    *reinterpret_cast<float4*>(q) =
                        make_float4(Pout[r][0], Pout[r][1], Pout[r][2], Pout[r][3]);
                } else {
#pragma unroll
                    for (int q2 = 0; q2 < kC; ++q2)
                        if (colv[q2]) q[q2] = Pout[r][q2];
                }
            }
        }
        // Backward planes are read back through TMA (async proxy): order this
        // thread's stores before them.  A fence covers all earlier stores too,
        // so only the last forward steps (those the producer may fetch before
        // the turn completes) need one.
        const bool near_turn = turn_fence && j <= n1 && j + NST >= n1;
        if (near_turn) fence_proxy_async_global();

        if (GD_EARLY_POLL == 2 && j < J) early_poll(j);
        GD_T0(t_bar);
#ifdef GD_SWEEP_TRACE
        if (TOP || BOT) trc[7] += t_bar - t_tail0_outer;
#endif
        consumer_sync(nthreads);
        GD_TADD(2, t_bar);
        GD_T0(t_post);
        if (tid == 0 && near_turn) st_release_cta(c.progress, j);
        GD_TADD(10, t_post);
    };

    int j = 1;
    for (; j + 1 <= J; j += 2) {
        step(j, PA, IA, PB, IB);
        step(j + 1, PB, IB, PA, IA);
    }
    if (j <= J) step(j, PA, IA, PB, IB);
#ifdef GD_SWEEP_TRACE
    trc[4] = clock64() - t_begin;
    trc[5] = J;
    if (p.trace && lane == 0) {
        long long* o = p.trace + (static_cast<long long>(c.g) * 64 + wu * nwv + wv) * 12;
        for (int i = 0; i < 12; ++i) o[i] = trc[i];
    }
#endif
}

// Warp-specialised persistent sweep: warps [0, NWU*nwv) relax the strip, the
// last warp is the TMA producer.  Slot j % NST carries plane p(j); it is
// released ("empty") by every consumer warp during step j+1, which reads it as
// the previous plane's intensities.
template <int KIND, bool F64, int RW, int NWU, int NST, int MW>
// One CTA per SM: two R = 2 CTAs per SM (126-register cap) measured 1.66 vs
// 1.25 us/step for R = 4 at 512^3 -- twice the halo links cost more than the
// second CTA hides (profiles/README.md).
__global__ void __launch_bounds__((MW * NWU + 1) * 32, MW == 2 && NWU * RW == 4 ? GD_MINB2 : 1)
    sweep_kernel(const __grid_constant__ CUtensorMap tm_d, const __grid_constant__ CUtensorMap tm_i,
                 const __grid_constant__ SweepParams p) {
    using L = Layout<RW, NWU, NST>;
    constexpr int DBOX = L::DBOX, IBOX = L::IBOX;
    constexpr bool kI = KIND != kSpatial;  // Spatial never reads intensities
    constexpr uint32_t TXW = static_cast<uint32_t>(kI ? DBOX * 4 + L::IBYTES : DBOX * 4);

    const int nwv = p.nwv;
    const int ncw = NWU * nwv;  // consumer warps
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    Ctx<RW, NWU, NST> c;
    c.sd = reinterpret_cast<float*>(smem_raw);
    c.si = c.sd + NST * nwv * DBOX;
    c.rows = c.si + NST * nwv * IBOX;
    c.edge = c.rows + 2 * NWU * 2 * nwv * kWV;
    c.full = reinterpret_cast<uint64_t*>(c.edge + 2 * NWU * nwv * 2 * RW);
    c.empty = c.full + NST;
    c.progress = reinterpret_cast<int*>(c.empty + NST);
    c.nwv = nwv;
    c.g = blockIdx.x;
    c.b = c.g / p.ntu;
    c.tu = c.g - c.b * p.ntu;
    c.u0 = c.tu * L::R;
    c.n1 = p.ns - 1;
    c.J = p.npass * c.n1;
    c.VW = nwv * kWV;

    if (tid == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(&c.full[s], 1);
            mbar_init(&c.empty[s], ncw);
        }
        *c.progress = -1;
        fence_mbar_init();
    }
    __syncthreads();

    // ======================= producer warp ==================================
    if (w == ncw) {
        if (lane == 0) {
            tma_prefetch_desc(&tm_d);
            if (kI) tma_prefetch_desc(&tm_i);
            for (int j = 0; j <= c.J; ++j) {
                const int slot = j % NST, k = j / NST;
                if (k > 0) mbar_wait(&c.empty[slot], static_cast<uint32_t>((k - 1) & 1));
                // A backward-pass plane is the forward pass's output of step 2*n1 - j.
                if (j > c.n1) {
                    const int jf = 2 * c.n1 - j;
                    while (ld_acquire_cta(c.progress) < jf) {
                    }
                }
                const int s = plane_of(p, c, j);
                mbar_arrive_expect_tx(&c.full[slot], TXW * nwv);
                for (int cb = 0; cb < nwv; ++cb) {
                    float* dd = c.sd + (slot * nwv + cb) * DBOX;
                    float* di = c.si + (slot * nwv + cb) * IBOX;
                    const int v0 = cb * kWV;
                    if (p.tma_sweep_dim == 2) {
                        tma_load_4d(dd, &tm_d, &c.full[slot], v0, c.u0, s, c.b);
                        if (kI) tma_load_4d(di, &tm_i, &c.full[slot], v0 - 4, c.u0 - 1, s, c.b);
                    } else {
                        tma_load_4d(dd, &tm_d, &c.full[slot], v0, s, c.u0, c.b);
                        if (kI) tma_load_4d(di, &tm_i, &c.full[slot], v0 - 4, s, c.u0 - 1, c.b);
                    }
                }
            }
        }
        return;
    }

    // ======================= consumer warps =================================
    const int wu = w / nwv, wv = w - wu * nwv;
    const int vl = wv * kWV + kC * lane;
    // CTA-uniform: one partial warp makes every warp of the CTA take the masked
    // variant.  Per-warp choice ran four role variants on one SM (TOP/BOT x
    // full/partial, ~14 KB of SASS each) and the instruction cache thrashed
    // (ncu: no_inst the top stall, 2.4x longer steps at W = 160).
    const bool full = consumer_all((c.u0 + wu * RW + RW <= p.nu) && (vl + kC <= p.nv),
                                   ncw * 32);
    const bool top = wu == 0, bot = wu == NWU - 1;
#define GD_ROLE(T, B)                                                                      \
    if (top == T && bot == B) {                                                            \
        if (full)                                                                          \
            consumer_loop<KIND, F64, RW, NWU, NST, T, B, true>(p, c, wu, wv, lane);        \
        else                                                                               \
            consumer_loop<KIND, F64, RW, NWU, NST, T, B, false>(p, c, wu, wv, lane);       \
        return;                                                                            \
    }
    if (NWU == 1) {
        GD_ROLE(true, true)
    } else {
        GD_ROLE(true, false)
        GD_ROLE(false, true)
        if (NWU > 2) GD_ROLE(false, false)
    }
#undef GD_ROLE
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

// Strip shapes X(RW rows per warp, NWU warp rows, MW max warp columns, NST
// ring stages).  R = RW * NWU rows per strip.  Narrow planes (<= 256 columns)
// get tall strips (R = 8, 16) so a batch of small volumes keeps enough bytes in
// flight per step; <= 512 columns run R = 4 as 2 warp rows of 2 rows (2 warps
// per scheduler); R = 1 serves single-row planes (2D).  Wide planes (<= 2048
// columns) trade registers for warps.
#define GD_SWEEP_CASES(X)                                                          \
    X(1, 1, 2, 6) X(2, 1, 2, 6) X(2, 2, 2, 6) X(4, 2, 2, 6) X(4, 4, 2, 4)             \
    X(1, 1, 4, 6) X(2, 1, 4, 6) X(2, 2, 4, GD_NST4) X(4, 2, 4, 6)                     \
    X(1, 1, 16, 6) X(2, 1, 16, 6) X(4, 1, 16, 6)

int width_class(int nwv) { return nwv <= 2 ? 2 : (nwv <= 4 ? 4 : 16); }

template <int KIND, bool F64>
cudaError_t dispatch_r(int R, const CUtensorMap& tm_d, const CUtensorMap& tm_i,
                       const SweepParams& p, cudaStream_t s) {
    const int mw = width_class(p.nwv);
#define GD_CASE(RWW, NW, MM, NS)                                     \
    if (R == RWW * NW && mw == MM)                                   \
        return launch_one<KIND, F64, RWW, NW, NS, MM>(tm_d, tm_i, p, s);
    GD_SWEEP_CASES(GD_CASE)
#undef GD_CASE
    return cudaErrorInvalidValue;
}

template <int KIND, bool F64>
int dispatch_cores(int R, int nwv) {
    const int mw = width_class(nwv);
#define GD_CASE(RWW, NW, MM, NS) \
    if (R == RWW * NW && mw == MM) return coresident<KIND, F64, RWW, NW, NS, MM>(nwv);
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

int sweep_warp_rows(int R, int nwv) {
    const int mw = width_class(nwv);
#define GD_CASE(RWW, NW, MM, NS) \
    if (R == RWW * NW && mw == MM) return NW;
    GD_SWEEP_CASES(GD_CASE)
#undef GD_CASE
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
