// Persistent directional-pass kernel templates (see sweep.cuh for the design
// notes).  Included by sweep.cu (dispatch, plane-step fallback) and by the five
// instantiation units sweep_k{0,1,1d,2,2d}.cu, one per (cost kind, f64): the
// kernel instances compile in parallel.
#pragma once
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "sweep.cuh"
#include "relax.cuh"

namespace gdb {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr long long kSpinLimit = 1ll << 22;  // ~seconds of polling: then the watchdog word is set

// Watchdog: set the word (system scope: it lives in mapped host memory).
__device__ __forceinline__ void watchdog_raise(unsigned int* err) {
    if (err) atomicOr_system(err, 1u);
}
__device__ __forceinline__ bool watchdog_raised(const unsigned int* err) {
    return err && *reinterpret_cast<const volatile unsigned int*>(err) != 0u;
}

// Halo polls: one per step, issued at the top of the step.  Measured slower on
// B200 at 512^3: a second poll in flight mid-step (1.48 vs 1.24 us/step: more
// L2 requests), and issuing the poll at the end of the previous step (after the
// publish: 1.17 vs 1.09 us/step, the poll is stale more often).

#ifndef GD_NST4
#define GD_NST4 6
#endif
// Halo spin limit: 0 = trap (the production choice: the flag-based watchdog's
// extra loop exit measured 8-9% slower per sweep at 512^3 and on the batch,
// profiles/r02_variants.txt), 1 = raise the device watchdog word and give up.
#ifndef GD_WATCHDOG
#define GD_WATCHDOG 0
#endif
// Early interior (finish / publish / store the rows that do not wait for the
// halo before the halo spin): measured slower for the min-plus kinds at 512^3
// (14.98 vs 14.48 ms) and on the batch (87.5 vs 82.0 ms), within noise for
// blend (profiles/r02_variants.txt) -- off.
// Protocol-checking build (make variant V=checks DEFS=-DGD_SWEEP_CHECKS=1):
// asserts on the halo hand-off invariants; never in production.
#ifndef GD_SWEEP_CHECKS
#define GD_SWEEP_CHECKS 0
#endif
#ifndef GD_EARLY_INTERIOR
#define GD_EARLY_INTERIOR 0
#endif
#ifndef GD_WARP_INTERLEAVE
#define GD_WARP_INTERLEAVE 0  // measured within noise at 512^3 (profiles/r02_variants.txt)
#endif
#ifndef GD_MINB2
#define GD_MINB2 3  // R = 4 strips of <= 256 columns: 3 CTAs per SM (batches; measured 97 -> 81 ms)
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

// TB (temporal blocking over plane pairs): the boxes carry one ghost row above
// and below the strip for the distances and two for the intensities, and the
// halo carries two rows per side, exchanged once per two planes.
template <int RW, int NWU, int NST, bool TB>
struct Layout {
    static constexpr int R = RW * NWU;                            // rows per strip
    static constexpr int DOFF = TB ? 1 : 0;                       // box row of strip row 0 (d)
    static constexpr int IOFF = TB ? 2 : 1;                       // box row of strip row 0 (I)
    static constexpr int HROWS = TB ? 2 : 1;                      // halo rows per side
    static constexpr int ESL = RW + (TB ? 1 : 0);                 // edge slots per side (+ ghost)
    static constexpr int DBOX = (R + 2 * DOFF) * kWV;             // floats per column-block box
    static constexpr int IBOX = ((R + 2 * IOFF) * kIW + 31) / 32 * 32;  // 128-B aligned stride
    static constexpr int IBYTES = (R + 2 * IOFF) * kIW * 4;
    // ds: DSMEM receive rows for cluster links (only allocated when clustered:
    // 2 KB more per CTA cost narrow planes their third CTA per SM).
    static size_t smem_bytes(int nwv, bool ds = false) {
        return static_cast<size_t>(NST) * nwv * (DBOX + IBOX) * 4     // TMA ring
               + static_cast<size_t>(2) * NWU * 2 * nwv * kWV * 4     // warp-row boundary rows
               + static_cast<size_t>(2) * NWU * nwv * 2 * ESL * 4     // warp-edge columns
               + (ds ? static_cast<size_t>(2) * 2 * nwv * kWV * 4 : 0)  // DSMEM halo rows
               + 2 * NST * 8 + 4 * 8 + 16 + 128;                      // barriers, progress
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
template <int RW, int NWU, int NST, bool TB>
struct Ctx {
    float* sd;          // [NST][nwv][R][128]      old distances (TMA)
    float* si;          // [NST][nwv][R+2][136]    intensities + row halo (TMA)
    float* rows;        // [2][NWU][first|last][nwv*128] warp-row boundary rows
    float* edge;        // [2][NWU][nwv][left|right][RW] warp-edge columns
    float* recv;        // [2 parities][above|below][nwv*128] DSMEM halo rows (cluster links)
    uint64_t* full;     // [NST]
    uint64_t* empty;    // [NST]
    uint64_t* rbar;     // [2 parities][above|below]: complete_tx of the DSMEM rows
    int* progress;
    int nwv, g, b, tu, u0, n1, J, VW, rank;
};

template <int RW, int NWU, int NST, bool TB>
__device__ __forceinline__ int plane_of(const SweepParams& p, const Ctx<RW, NWU, NST, TB>& c,
                                        int j) {
    if (j <= c.n1) return p.first_orient > 0 ? j : c.n1 - j;
    const int k = j - c.n1;
    return p.first_orient > 0 ? c.n1 - k : k;
}

// One consumer warp's whole sweep.  TOP / BOT: the warp row borders the strip
// above / below (tagged global halo); FULL: every voxel of the warp is inside
// the volume.  Specialising on the role keeps the per-step body branch-free.
template <int KIND, bool F64, int RW, int NWU, int NST, bool TB, bool CL, bool TOP, bool BOT,
          bool FULL>
__device__ __forceinline__ void consumer_loop(const SweepParams& p,
                                              const Ctx<RW, NWU, NST, TB>& c, int wu, int wv,
                                              int lane) {
    using L = Layout<RW, NWU, NST, TB>;
    static_assert(!TB || RW >= 2, "temporal blocking publishes two rows per border warp");
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

    constexpr int DOFF = L::DOFF, IOFF = L::IOFF, HROWS = L::HROWS, ESL = L::ESL;
    static_assert(!TB || NWU >= 2, "temporal blocking keeps one ghost row per border warp");
    const bool has_up = TOP && c.tu > 0, has_dn = BOT && c.tu + 1 < p.ntu;
    // per strip: 2 parities x {TOP rows, BOT rows} x HROWS rows of VW words
    const long long strip_words = 2ll * 2 * HROWS * VW;
    const long long PARW = 2ll * HROWS * VW;
    const long long strip0 = static_cast<long long>(c.b) * p.ntu;
    // Halo row layout (per warp column block of 128 words): columns q = 0,1 of
    // all 32 lanes, then q = 2,3 -- lane l owns words 2l, 2l+1, 64+2l, 65+2l, so
    // each 16-byte access of the warp covers 512 contiguous bytes (16 full
    // sectors) instead of half of 32 sectors.  v-1 / v+4 come from the adjacent
    // lanes; only lane 0 / lane 31 load the neighbour block's edge word.
    const bool has_left = vl > 0, has_right = vl + kC < p.nv;
    const bool edge_l = lane == 0 && has_left, edge_r = lane == 31 && has_right;
    const int hl = wv * kWV + 2 * lane;
    // the neighbour above publishes its last HROWS rows, the one below its first
    const unsigned long long* up0 =
        p.halo + (strip0 + c.tu - 1) * strip_words + HROWS * VW + hl;
    const unsigned long long* dn0 = p.halo + (strip0 + c.tu + 1) * strip_words + hl;
    unsigned long long* self0 = p.halo + static_cast<long long>(c.g) * strip_words + hl;
    const bool pub_up = TOP && c.tu > 0, pub_dn = BOT && c.tu + 1 < p.ntu;
    // Links inside a thread-block cluster (consecutive strips of one volume)
    // carry the row through DSMEM: st.async into the neighbour's receive row,
    // completing tx bytes on its mbarrier; links across clusters use the tagged
    // L2 words.  (Not combined with temporal blocking.)
    const int rank = c.rank;
    const bool ds_up = CL && has_up && rank > 0;
    const bool ds_dn = CL && has_dn && rank + 1 < p.cs;
    const bool l2_up = has_up && !ds_up, l2_dn = has_dn && !ds_dn;
    // neighbour-warp edge columns (ESL slots per side: own rows, then the ghost row)
    const int eoffL = ((wu * nwv + wv - 1) * 2 + 1) * ESL;
    const int eoffR = ((wu * nwv + wv + 1) * 2 + 0) * ESL;
    const bool wl = wv > 0, wr = wv + 1 < nwv;
    float* const edge_own = c.edge + (wu * nwv + wv) * 2 * ESL;
    const int EPAR = NWU * nwv * 2 * ESL;  // edge buffer parity stride
    const int RPAR = NWU * 2 * VW;         // rows buffer parity stride

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

    // TB ghost scratch: the ghost row of every forward A step, read back as the
    // ghost's old distance in the backward pass (this warp's own earlier stores:
    // no cross-CTA visibility question).  [cta][TOP|BOT][forward step / 2][VW].
    const int gsteps = c.n1 / 2 + 1;
    float* const gscr = TB ? p.ghost + ((static_cast<long long>(c.g) * 2 + (TOP ? 0 : 1)) *
                                            gsteps) * VW + vl
                           : nullptr;

    // Halo publication: TOP rows 0..HROWS-1, BOT rows RW-HROWS..RW-1.
    auto publish_halo = [&](int j, const float (&N)[RW][kC]) {
        const int par = TB ? (j >> 1) & 1 : j & 1;
        const uint32_t tag = tag_base + static_cast<uint32_t>(j);
        unsigned long long* q = self0 + par * PARW;
        if (GD_DBG(2)) return;
        if (ds_up || ds_dn) {
            // to the neighbour above: its "below" row; to the one below: its "above" row
            const int side = ds_up ? 1 : 0;
            const int r = ds_up ? 0 : RW - 1;
            const uint32_t dst = static_cast<uint32_t>(rank + (ds_up ? -1 : 1));
            const uint32_t raddr =
                mapa_shared(smem_u32(c.recv + (par * 2 + side) * VW + vl), dst);
            const uint32_t rbar = mapa_shared(smem_u32(&c.rbar[par * 2 + side]), dst);
            st_async_v4(raddr, N[r][0], N[r][1], N[r][2], N[r][3], rbar);
        }
        if (pub_up && !ds_up) {
#pragma unroll
            for (int k = 0; k < HROWS; ++k) {
                st_tagged2(q + k * VW, N[k][0], N[k][1], tag);
                st_tagged2(q + k * VW + 64, N[k][2], N[k][3], tag);
            }
        }
        if (pub_dn && !ds_dn) {
#pragma unroll
            for (int k = 0; k < HROWS; ++k) {
                const int r = RW - HROWS + k;
                st_tagged2(q + (HROWS + k) * VW, N[r][0], N[r][1], tag);
                st_tagged2(q + (HROWS + k) * VW + 64, N[r][2], N[r][3], tag);
            }
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
            if (lane == 31) e[ESL + r] = N[r][kC - 1];
        }
    };

    // One row's share of publish_smem (the early-interior path publishes the
    // rows that do not wait for the halo before the halo spin).
    auto publish_smem_row = [&](int j, int r, const float (&N)[RW][kC]) {
        const int par = j & 1;
        if (NWU > 1) {
            float* rw_ = c.rows + par * RPAR + wu * 2 * VW;
            if (r == 0 && !TOP)
                *reinterpret_cast<float4*>(rw_ + vl) =
                    make_float4(N[0][0], N[0][1], N[0][2], N[0][3]);
            if (r == RW - 1 && !BOT)
                *reinterpret_cast<float4*>(rw_ + VW + vl) =
                    make_float4(N[RW - 1][0], N[RW - 1][1], N[RW - 1][2], N[RW - 1][3]);
        }
        float* e = edge_own + par * EPAR;
        if (lane == 0) e[r] = N[r][0];
        if (lane == 31) e[ESL + r] = N[r][kC - 1];
    };
    auto store_row = [&](int r, const float (&N)[RW][kC]) {
        float* q = outp + r * su;
        if (FULL) {
            *reinterpret_cast<float4*>(q) = make_float4(N[r][0], N[r][1], N[r][2], N[r][3]);
        } else if (rowv[r]) {
            if (colv[kC - 1]) {
                *reinterpret_cast<float4*>(q) = make_float4(N[r][0], N[r][1], N[r][2], N[r][3]);
            } else {
#pragma unroll
                for (int q2 = 0; q2 < kC; ++q2)
                    if (colv[q2]) q[q2] = N[r][q2];
            }
        }
    };
    // A row that waits for the neighbour strip's halo row.
    auto border_row = [&](int r) { return (TOP && r == 0) || (BOT && r == RW - 1); };

    float PA[RW][kC], IA[RW][kC], PB[RW][kC], IB[RW][kC];
    float G[kC];  // TB: ghost row (above for TOP, below for BOT) of the last A step
#pragma unroll
    for (int q = 0; q < kC; ++q) G[q] = INF;
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
                *reinterpret_cast<const float4*>(sd_base + (r0 + r + DOFF) * kWV + kC * lane);
            PA[r][0] = d4.x; PA[r][1] = d4.y; PA[r][2] = d4.z; PA[r][3] = d4.w;
            if (kI) {
                const float4 i4 = *reinterpret_cast<const float4*>(
                    si_base + (r0 + r + IOFF) * kIW + 4 + kC * lane);
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

    // One relaxation step: plane j from the previous plane (Pin, Iin) into
    // (Pout, Iout).  kA: with TB, odd steps ("A") wait for the neighbours' two
    // rows and also relax this warp's ghost row; even steps ("B") take the
    // ghost row from registers and publish.  Without TB every step polls.
    auto step = [&](auto kA, int j, const float (&Pin)[RW][kC], const float (&Iin)[RW][kC],
                    float (&Pout)[RW][kC], float (&Iout)[RW][kC]) {
        constexpr bool A = decltype(kA)::value;
        constexpr bool POLL = !TB || A;    // this step reads the tagged halo
        constexpr bool GHOST = TB && A;    // this step relaxes the ghost row
        constexpr bool USEG = TB && !A;    // this step takes the ghost row as a neighbour
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
        const int par = (j - 1) & 1;  // smem (rows / edge) parity of the previous plane
        const int hpar = TB ? ((j - 1) >> 1) & 1 : (j - 1) & 1;
        const uint32_t want = tag_base + static_cast<uint32_t>(j - 1);
        const unsigned long long* hup = up0 + hpar * PARW;
        const unsigned long long* hdn = dn0 + hpar * PARW;
        // [k][0] = v-1, [k][1..4] own, [k][5] = v+4
        unsigned long long hu[HROWS][6], hd[HROWS][6];
        if (POLL && !GD_DBG(4)) {
#pragma unroll
            for (int k = 0; k < HROWS; ++k) {
                if (TOP && l2_up) load_row(hup + k * VW, hu[k]);
                if (BOT && l2_dn) load_row(hdn + k * VW, hd[k]);
            }
        }
        // DSMEM rows of step j-1: one thread per receiving warp row arms the
        // mbarrier phase with the row's bytes (the data may already be there).
        const int rq = (j - 1) & 1;
        if (POLL && wv == 0 && lane == 0) {
            if (ds_up) mbar_arrive_expect_tx(&c.rbar[rq * 2 + 0], static_cast<uint32_t>(VW * 4));
            if (ds_dn) mbar_arrive_expect_tx(&c.rbar[rq * 2 + 1], static_cast<uint32_t>(VW * 4));
        }
        const bool backward = j > n1;
        const int gslot = (2 * n1 - j) >> 1;  // backward A step: forward step 2 n1 - j
        float4 gold = make_float4(INF, INF, INF, INF);
        if (GHOST && backward && (TOP ? has_up : has_dn))
            gold = *reinterpret_cast<const float4*>(gscr + static_cast<long long>(gslot) * VW);

        GD_TADD(8, t_entry);
        GD_T0(t_tma);
        mbar_wait(&c.full[slot], phase);
        GD_TADD(0, t_tma);
        GD_T0(t_pa);
        float dold[RW][kC], ic[RW][kC];
#pragma unroll
        for (int r = 0; r < RW; ++r) {
            const float4 d4 = *reinterpret_cast<const float4*>(sd_cur + (r0 + r + DOFF) * kWV +
                                                               kC * lane);
            dold[r][0] = d4.x; dold[r][1] = d4.y; dold[r][2] = d4.z; dold[r][3] = d4.w;
            if (kI) {
                const float4 i4 = *reinterpret_cast<const float4*>(
                    si_cur + (r0 + r + IOFF) * kIW + 4 + kC * lane);
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

        // Ghost row (GHOST steps): strip row -1 (TOP) or R (BOT) of plane j.
        // Its old distance: the TMA box in the forward pass; in the backward
        // pass the forward ghost of the same plane from the scratch (the box row
        // is another CTA's forward output, not ordered before this TMA read).
        constexpr int gr = TOP ? -1 : R;
        Acc<KIND, F64> accG[kC];
        float ig[kC];
        if (GHOST) {
            const float4 d4 = *reinterpret_cast<const float4*>(sd_cur + (gr + DOFF) * kWV +
                                                               kC * lane);
            const float gd[kC] = {d4.x, d4.y, d4.z, d4.w};
            const float gb[kC] = {gold.x, gold.y, gold.z, gold.w};
#pragma unroll
            for (int q = 0; q < kC; ++q) accG[q].init(backward ? gb[q] : gd[q]);
            if (kI) {
                const float4 i4 = *reinterpret_cast<const float4*>(
                    si_cur + (gr + IOFF) * kIW + 4 + kC * lane);
                ig[0] = i4.x; ig[1] = i4.y; ig[2] = i4.z; ig[3] = i4.w;
            } else {
#pragma unroll
                for (int q = 0; q < kC; ++q) ig[q] = 0.0f;
            }
        }

        auto i_window = [&](int sr, float (&iw)[6]) {
            if (kI) {
                const float* rp = sip + (sr + IOFF) * kIW;
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
                const float* rp = sip + (r0 + k + IOFF) * kIW;
                make_window(Iin[k], rp[3], rp[4 + kWV], lane, iw);
            } else {
#pragma unroll
                for (int i = 0; i < 6; ++i) iw[i] = 0.0f;
            }
            if (k - 1 >= 0) relax_row<KIND, F64>(acc[k - 1], pw, iw, ic[k - 1], +1, p);
            relax_row<KIND, F64>(acc[k], pw, iw, ic[k], 0, p);
            if (k + 1 < RW) relax_row<KIND, F64>(acc[k + 1], pw, iw, ic[k + 1], -1, p);
            if (GHOST && TOP && k == 0) relax_row<KIND, F64>(accG, pw, iw, ig, +1, p);
            if (GHOST && BOT && k == RW - 1) relax_row<KIND, F64>(accG, pw, iw, ig, -1, p);
        }
        if (!TOP) {
            const float* rp = rows_prev + ((wu - 1) * 2 + 1) * VW;  // last row of warp row wu-1
            const float4 q4 = *reinterpret_cast<const float4*>(rp + vl);
            const float c4[kC] = {q4.x, q4.y, q4.z, q4.w};
            float pw[6], iw[6];
            make_window(c4, edge_l ? rp[vl - 1] : INF, edge_r ? rp[vl + kC] : INF, lane, pw);
            i_window(r0 - 1, iw);
            relax_row<KIND, F64>(acc[0], pw, iw, ic[0], -1, p);
        }
        if (!BOT) {
            const float* rp = rows_prev + ((wu + 1) * 2 + 0) * VW;  // first row of warp row wu+1
            const float4 q4 = *reinterpret_cast<const float4*>(rp + vl);
            const float c4[kC] = {q4.x, q4.y, q4.z, q4.w};
            float pw[6], iw[6];
            make_window(c4, edge_l ? rp[vl - 1] : INF, edge_r ? rp[vl + kC] : INF, lane, pw);
            i_window(r0 + RW, iw);
            relax_row<KIND, F64>(acc[RW - 1], pw, iw, ic[RW - 1], +1, p);
        }
        // B steps: the row outside the strip is the ghost relaxed at the A step.
        if (USEG && (TOP ? has_up : has_dn)) {
            float pw[6], iw[6];
            make_window(G, wl ? edge_prev[eoffL + RW] : INF, wr ? edge_prev[eoffR + RW] : INF,
                        lane, pw);
            i_window(gr, iw);
            if (TOP) relax_row<KIND, F64>(acc[0], pw, iw, ic[0], -1, p);
            else relax_row<KIND, F64>(acc[RW - 1], pw, iw, ic[RW - 1], +1, p);
        }

        auto fin = [&](int r) {
#pragma unroll
            for (int q = 0; q < kC; ++q) {
                Pout[r][q] = acc[r][q].final(p);
                if (!FULL && !(rowv[r] && colv[q])) Pout[r][q] = INF;
                Iout[r][q] = ic[r][q];
            }
        };
        // The output row pointer of this plane (the backward pass walks back).
        if (j == n1 + 1) dsoff = -dsoff;
        outp += dsoff;
        // Early interior: rows that do not border the strip are final after
        // phase A -- finish, publish (shared memory) and store them while the
        // halo poll is still in flight, so only the border rows remain behind
        // the halo wait.
        constexpr bool EARLY = GD_EARLY_INTERIOR && !TB;
        if (EARLY) {
#pragma unroll
            for (int r = 0; r < RW; ++r) {
                if (border_row(r)) continue;
                fin(r);
                if (j < J) publish_smem_row(j, r, Pout);
                store_row(r, Pout);
            }
        }

        // ---- phase B: rows above / below the strip (tagged halo) -------------
#ifdef GD_SWEEP_TRACE
        long long t_tail0_outer = 0;
#endif
        if (POLL && (TOP || BOT)) {
            auto fresh = [&](const unsigned long long (&h)[6]) {
                bool ok = (!edge_l || tag_of(h[0]) == want) && (!edge_r || tag_of(h[5]) == want);
#pragma unroll
                for (int i = 1; i <= kC; ++i) ok = ok && tag_of(h[i]) == want;
#if GD_SWEEP_CHECKS
                // Protocol check (checks build): two parities allow a neighbour at
                // most one step of skew, so a word tagged beyond `want` means it
                // overwrote a row this strip had not read yet.
                bool ahead = false;
#pragma unroll
                for (int i = 0; i < 6; ++i) {
                    const bool used = i == 0 ? edge_l : (i == 5 ? edge_r : true);
                    ahead = ahead || (used && static_cast<int>(tag_of(h[i]) - want) > 0);
                }
                if (ahead) {
                    printf("sweep protocol violation: cta %d warp %d lane %d step %d want %u\n",
                           static_cast<int>(blockIdx.x), wu * nwv + wv, lane, j, want);
                    __trap();
                }
#endif
                return ok;
            };
            long long spins = 0;
            GD_TADD(6, t_pa);
            GD_T0(t_spin);
            while (!GD_DBG(1)) {
                bool ok = true;
#pragma unroll
                for (int k = 0; k < HROWS; ++k) {
                    if (TOP && l2_up) ok = ok && fresh(hu[k]);
                    if (BOT && l2_dn) ok = ok && fresh(hd[k]);
                }
                if (__all_sync(kFull, ok)) break;
#pragma unroll
                for (int k = 0; k < HROWS; ++k) {
                    if (TOP && l2_up) load_row(hup + k * VW, hu[k]);
                    if (BOT && l2_dn) load_row(hdn + k * VW, hd[k]);
                }
                // Watchdog: after kSpinLimit polls (or once another CTA raised it,
                // checked every 1024 polls) give up on this neighbour; the host
                // reports the failure instead of a hang or a sticky trap.
#if GD_WATCHDOG
                // `spins` is warp-uniform (the loop exits on __all_sync), so the
                // fast path is one increment and compare, as cheap as a trap test;
                // only a wait far beyond any halo latency (2^14 polls, ~10 ms)
                // looks at the watchdog word.
                if (++spins >= (1ll << 14)) {
                    if (spins > kSpinLimit || ((spins & 1023) == 0 && watchdog_raised(p.err))) {
                        if (lane == 0) watchdog_raise(p.err);
                        break;
                    }
                }
#else
                if (++spins > kSpinLimit) __trap();
#endif
            }
            const uint32_t rph = static_cast<uint32_t>(((j - 1) >> 1) & 1);
            if (TOP && ds_up) mbar_wait(&c.rbar[rq * 2 + 0], rph);
            if (BOT && ds_dn) mbar_wait(&c.rbar[rq * 2 + 1], rph);
            GD_TADD(1, t_spin);
#ifdef GD_SWEEP_TRACE
            t_tail0_outer = clock64();
            trc[3] += spins;
#endif
            // a DSMEM row: the whole row sits in this CTA's receive buffer
            auto recv_window = [&](int side, float (&pw)[6]) {
                const float* rp = c.recv + (rq * 2 + side) * VW;
                const float4 q4 = *reinterpret_cast<const float4*>(rp + vl);
                const float c4[kC] = {q4.x, q4.y, q4.z, q4.w};
                make_window(c4, edge_l ? rp[vl - 1] : INF, edge_r ? rp[vl + kC] : INF, lane, pw);
                if (!has_left) pw[0] = INF;
                if (!has_right) pw[5] = INF;
            };
            if (TOP) {
                // rows -HROWS .. -1: the neighbour above's last rows
                float pw1[6], iw1[6];
                if (ds_up) recv_window(0, pw1);
                else halo_window(hu[HROWS - 1], has_up, has_left, has_right, lane, pw1);
                i_window(-1, iw1);
                relax_row<KIND, F64>(acc[0], pw1, iw1, ic[0], -1, p);
                if (GHOST && has_up) {
                    float pw2[6], iw2[6];
                    halo_window(hu[0], has_up, has_left, has_right, lane, pw2);
                    i_window(-2, iw2);
                    relax_row<KIND, F64>(accG, pw2, iw2, ig, -1, p);
                    relax_row<KIND, F64>(accG, pw1, iw1, ig, 0, p);
                }
            }
            if (BOT) {
                // rows R .. R+HROWS-1: the neighbour below's first rows
                float pw1[6], iw1[6];
                if (ds_dn) recv_window(1, pw1);
                else halo_window(hd[0], has_dn, has_left, has_right, lane, pw1);
                i_window(R, iw1);
                relax_row<KIND, F64>(acc[RW - 1], pw1, iw1, ic[RW - 1], +1, p);
                if (GHOST && has_dn) {
                    float pw2[6], iw2[6];
                    halo_window(hd[HROWS - 1], has_dn, has_left, has_right, lane, pw2);
                    i_window(R + 1, iw2);
                    relax_row<KIND, F64>(accG, pw1, iw1, ig, 0, p);
                    relax_row<KIND, F64>(accG, pw2, iw2, ig, +1, p);
                }
            }
        }
        // The previous plane's slot is no longer read by this warp.
        __syncwarp();
        if (lane == 0) mbar_arrive(&c.empty[pslot]);

        // Border rows first: they are the neighbours' critical path.
        if (TOP) fin(0);
        if (BOT && (RW > 1 || !TOP)) fin(RW - 1);
        if (!TB || !A) {
            if (TB && TOP) fin(1);
            if (TB && BOT) fin(RW - 2);
            if (j < J) publish_halo(j, Pout);
        }
#ifdef GD_SWEEP_TRACE
        if (TOP || BOT) trc[9] += clock64() - t_tail0_outer;
#endif
        if (EARLY) {
#pragma unroll
            for (int r = 0; r < RW; ++r) {
                if (!border_row(r)) continue;
                if (j < J) publish_smem_row(j, r, Pout);
                store_row(r, Pout);
            }
        } else {
#pragma unroll
            for (int r = 0; r < RW; ++r)
                if (!border_row(r)) fin(r);
            if (GHOST) {
                const bool present = TOP ? has_up : has_dn;
#pragma unroll
                for (int q = 0; q < kC; ++q) {
                    G[q] = present ? accG[q].final(p) : INF;
                    if (!FULL && !colv[q]) G[q] = INF;
                }
                if (j < J) {
                    float* e = edge_own + (j & 1) * EPAR;
                    if (lane == 0) e[RW] = G[0];
                    if (lane == 31) e[ESL + RW] = G[kC - 1];
                }
                if (!backward && p.npass == 2 && present)
                    *reinterpret_cast<float4*>(gscr + static_cast<long long>(j >> 1) * VW) =
                        make_float4(G[0], G[1], G[2], G[3]);
            }
            if (j < J) publish_smem(j, Pout);

            // ---- store the relaxed plane --------------------------------------
#pragma unroll
            for (int r = 0; r < RW; ++r) store_row(r, Pout);
        }
        // Backward planes are read back through TMA (async proxy): order this
        // thread's stores before them.  A fence covers all earlier stores too,
        // so only the last forward steps (those the producer may fetch before
        // the turn completes) need one.
        const bool near_turn = turn_fence && j <= n1 && j + NST >= n1;
        if (near_turn) fence_proxy_async_global();

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

    const std::integral_constant<bool, true> kStepA{};
    const std::integral_constant<bool, false> kStepB{};
    int j = 1;
    // (A single step body with register moves instead of the unrolled pair
    // measured slower for the one-row shape: 19.5 vs 18.0 ms at lambda = 0.5.)
    for (; j + 1 <= J; j += 2) {
        step(kStepA, j, PA, IA, PB, IB);
        step(kStepB, j + 1, PB, IB, PA, IA);
    }
    if (j <= J) step(kStepA, j, PA, IA, PB, IB);
#ifdef GD_SWEEP_TRACE
    trc[4] = clock64() - t_begin;
    trc[5] = J;
    if (p.trace && lane == 0) {
        long long* o = p.trace + (static_cast<long long>(c.g) * 64 + wu * nwv + wv) * 12;
        for (int i = 0; i < 12; ++i) o[i] = trc[i];
    }
#endif
}

// Plane-step fallback (any plane size): one thread relaxes 4 consecutive
// columns of one row of plane s from plane sp, reading the previous plane from
// global memory (L2-resident: it was written by the previous launch).  Same
// arithmetic as the persistent kernel (relax_row / Acc), so results agree bit
// for bit.  Columns >= nv of a padded row are never read as neighbours nor written.
template <int KIND, bool F64>
__global__ void __launch_bounds__(256)
    plane_step_kernel(const __grid_constant__ SweepParams p, int s, int sp) {
    if (gate_closed(p)) return;
    constexpr bool kI = KIND != kSpatial;
    const int nq = (p.nv + kC - 1) / kC;
    const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<long long>(p.nu) * nq) return;
    const int u = static_cast<int>(idx / nq), v0 = static_cast<int>(idx % nq) * kC;
    const long long vb = static_cast<long long>(blockIdx.y) * p.vol_stride;
    const float INF = finf();
    const float* dprev = p.dist + vb + static_cast<long long>(sp) * p.ss;
    float* dcur = p.dist + vb + static_cast<long long>(s) * p.ss + static_cast<long long>(u) * p.su;
    const float* iprev = p.image + vb + static_cast<long long>(sp) * p.ss;
    const float* icur = p.image + vb + static_cast<long long>(s) * p.ss +
                        static_cast<long long>(u) * p.su;
    float ip[kC];
    Acc<KIND, F64> acc[kC];
#pragma unroll
    for (int q = 0; q < kC; ++q) {
        const bool ok = v0 + q < p.nv;
        acc[q].init(ok ? dcur[v0 + q] : INF);
        ip[q] = (kI && ok) ? icur[v0 + q] : 0.0f;
    }
#pragma unroll
    for (int du = -1; du <= 1; ++du) {
        const int uu = u + du;
        if (uu < 0 || uu >= p.nu) continue;
        const float* dr = dprev + static_cast<long long>(uu) * p.su;
        const float* ir = iprev + static_cast<long long>(uu) * p.su;
        float pw[6], iw[6];
#pragma unroll
        for (int i = 0; i < 6; ++i) {
            const int v = v0 - 1 + i;
            const bool ok = v >= 0 && v < p.nv;
            pw[i] = ok ? dr[v] : INF;
            iw[i] = (kI && ok) ? ir[v] : 0.0f;
        }
        // relax_row's du is (previous-plane row) - (output row), as here
        relax_row<KIND, F64>(acc, pw, iw, ip, du, p);
    }
#pragma unroll
    for (int q = 0; q < kC; ++q)
        if (v0 + q < p.nv) dcur[v0 + q] = acc[q].final(p);
}

template <int KIND, bool F64>
cudaError_t plane_step_one(const SweepParams& p, int s, int sp, cudaStream_t stream) {
    const long long n = static_cast<long long>(p.nu) * ((p.nv + kC - 1) / kC);
    const dim3 grid(static_cast<unsigned>((n + 255) / 256), static_cast<unsigned>(p.nvol));
    plane_step_kernel<KIND, F64><<<grid, 256, 0, stream>>>(p, s, sp);
    return cudaGetLastError();
}

// Warp-specialised persistent sweep: warps [0, NWU*nwv) relax the strip, the
// last warp is the TMA producer.  Slot j % NST carries plane p(j); it is
// released ("empty") by every consumer warp during step j+1, which reads it as
// the previous plane's intensities.
template <int KIND, bool F64, int RW, int NWU, int NST, int MW, bool TB, bool CL>
// One CTA per SM: two R = 2 CTAs per SM (126-register cap) measured 1.66 vs
// 1.25 us/step for R = 4 at 512^3 -- twice the halo links cost more than the
// second CTA hides (profiles/README.md).
__global__ void __launch_bounds__((MW * NWU + 1) * 32, MW == 2 && NWU * RW == 4 ? GD_MINB2 : 1)
    sweep_kernel(const __grid_constant__ CUtensorMap tm_d, const __grid_constant__ CUtensorMap tm_i,
                 const __grid_constant__ SweepParams p) {
    using L = Layout<RW, NWU, NST, TB>;
    constexpr int DBOX = L::DBOX, IBOX = L::IBOX;
    constexpr bool kI = KIND != kSpatial;  // Spatial never reads intensities
    constexpr uint32_t TXW = static_cast<uint32_t>(kI ? DBOX * 4 + L::IBYTES : DBOX * 4);

    // Gated off (the other arithmetic path, or nothing to do): every CTA of the
    // grid reads the same word and leaves before any barrier or cluster sync.
    if (gate_closed(p)) return;
    const int nwv = p.nwv;
    const int ncw = NWU * nwv;  // consumer warps
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    Ctx<RW, NWU, NST, TB> c;
    c.sd = reinterpret_cast<float*>(smem_raw);
    c.si = c.sd + NST * nwv * DBOX;
    c.rows = c.si + NST * nwv * IBOX;
    c.edge = c.rows + 2 * NWU * 2 * nwv * kWV;
    c.recv = c.edge + 2 * NWU * nwv * 2 * L::ESL;
    c.full = reinterpret_cast<uint64_t*>(c.recv + (CL ? 2 * 2 * nwv * kWV : 0));
    c.empty = c.full + NST;
    c.rbar = c.empty + NST;
    c.progress = reinterpret_cast<int*>(c.rbar + 4);
    c.nwv = nwv;
    c.g = blockIdx.x;
    c.b = c.g / p.ntu;
    c.tu = c.g - c.b * p.ntu;
    c.u0 = c.tu * L::R;
    c.n1 = p.ns - 1;
    c.J = p.npass * c.n1;
    c.VW = nwv * kWV;
    c.rank = CL ? static_cast<int>(cluster_ctarank()) : 0;

    if (tid == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(&c.full[s], 1);
            mbar_init(&c.empty[s], ncw);
        }
        for (int s = 0; s < 4; ++s) mbar_init(&c.rbar[s], 1);
        *c.progress = -1;
        fence_mbar_init();
    }
    __syncthreads();
    // The neighbours' mbarriers must be initialised before the first remote store.
    if constexpr (CL) cluster_sync_all();

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
                    const int ud = c.u0 - L::DOFF, ui = c.u0 - L::IOFF;
                    if (p.tma_sweep_dim == 2) {
                        tma_load_4d(dd, &tm_d, &c.full[slot], v0, ud, s, c.b);
                        if (kI) tma_load_4d(di, &tm_i, &c.full[slot], v0 - 4, ui, s, c.b);
                    } else {
                        tma_load_4d(dd, &tm_d, &c.full[slot], v0, s, ud, c.b);
                        if (kI) tma_load_4d(di, &tm_i, &c.full[slot], v0 - 4, s, ui, c.b);
                    }
                }
            }
        }
        __syncwarp();
        if constexpr (CL) cluster_sync_all();  // no CTA leaves while its cluster runs
        return;
    }

    // ======================= consumer warps =================================
#if GD_WARP_INTERLEAVE
    // Warp w runs on scheduler (SMSP) w % 4.  Interleaving the warp rows
    // (wu = w % NWU) puts warps of ONE border role on each scheduler, so each
    // scheduler's instruction cache holds one role's step bodies, not two.
    const int wu = w % NWU, wv = w / NWU;
#else
    const int wu = w / nwv, wv = w - wu * nwv;
#endif
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
            consumer_loop<KIND, F64, RW, NWU, NST, TB, CL, T, B, true>(p, c, wu, wv, lane); \
        else                                                                               \
            consumer_loop<KIND, F64, RW, NWU, NST, TB, CL, T, B, false>(p, c, wu, wv, lane);\
    }
    if (NWU == 1) {
        GD_ROLE(true, true)
    } else {
        GD_ROLE(true, false)
        GD_ROLE(false, true)
        if (NWU > 2) GD_ROLE(false, false)
    }
#undef GD_ROLE
    __syncwarp();
    if constexpr (CL) cluster_sync_all();
}

template <int KIND, bool F64, int RW, int NWU, int NST, int MW, bool TB, bool CL>
cudaError_t launch_one(const CUtensorMap& tm_d, const CUtensorMap& tm_i, const SweepParams& p,
                       cudaStream_t stream) {
    using L = Layout<RW, NWU, NST, TB>;
    auto fn = sweep_kernel<KIND, F64, RW, NWU, NST, MW, TB, CL>;
    const size_t smem = L::smem_bytes(p.nwv, CL);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    const int grid = p.nvol * p.ntu;
    if constexpr (CL) {
        // Cooperative (co-residency guaranteed) and clustered (DSMEM links).
        if (p.cs > 8) {
            e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            if (e != cudaSuccess) return e;
        }
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3((p.nwv * NWU + 1) * 32);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = stream;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = static_cast<unsigned>(p.cs);
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        at[1].id = cudaLaunchAttributeCooperative;
        at[1].val.cooperative = 1;
        cfg.attrs = at;
        // Profiling only (GEODIST_SWEEP_NOCOOP=1): drop the cooperative attribute.
        // The grid is sized to the co-resident cluster count either way; ncu's
        // kernel replay rejects the cooperative + cluster launch (LaunchFailed).
        static const bool nocoop = std::getenv("GEODIST_SWEEP_NOCOOP") != nullptr;
        cfg.numAttrs = nocoop ? 1 : 2;
        return cudaLaunchKernelEx(&cfg, fn, tm_d, tm_i, p);
    }
    void* args[] = {const_cast<CUtensorMap*>(&tm_d), const_cast<CUtensorMap*>(&tm_i),
                    const_cast<SweepParams*>(&p)};
    return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(fn), dim3(grid),
                                       dim3((p.nwv * NWU + 1) * 32),
                                       args, smem, stream);
}

template <int KIND, bool F64, int RW, int NWU, int NST, int MW, bool TB, bool CL>
int coresident_clusters(int nwv, int cs) {
    using L = Layout<RW, NWU, NST, TB>;
    auto fn = sweep_kernel<KIND, F64, RW, NWU, NST, MW, TB, CL>;
    const size_t smem = L::smem_bytes(nwv, true);
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem)) != cudaSuccess ||
        (cs > 8 &&
         cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
             cudaSuccess)) {
        (void)cudaGetLastError();
        return 0;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * 64);
    cfg.blockDim = dim3((nwv * NWU + 1) * 32);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = static_cast<unsigned>(cs);
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess) {
        (void)cudaGetLastError();
        return 0;
    }
    return n * cs;
}

template <int KIND, bool F64, int RW, int NWU, int NST, int MW, bool TB, bool CL>
int coresident(int nwv) {
    using L = Layout<RW, NWU, NST, TB>;
    auto fn = sweep_kernel<KIND, F64, RW, NWU, NST, MW, TB, CL>;
    const size_t smem = L::smem_bytes(nwv);
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem)) != cudaSuccess) {
        (void)cudaGetLastError();  // too much shared memory at this width: not a candidate
        return 0;
    }
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, (nwv * NWU + 1) * 32, smem) !=
        cudaSuccess) {
        (void)cudaGetLastError();
        return 0;
    }
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
#define GD_SWEEP_CASES(X)                                                                 \
    X(1, 1, 2, 6, false, false) X(2, 1, 2, 6, false, false) X(2, 2, 2, 6, false, false)     \
    X(2, 2, 2, 6, true, false) X(2, 2, 2, 6, false, true)                                   \
    X(4, 2, 2, 6, false, false) X(4, 4, 2, 4, false, false) X(1, 4, 2, 6, false, false)     \
    X(1, 1, 4, 6, false, false) X(2, 1, 4, 6, false, false) X(2, 2, 4, GD_NST4, false, false) \
    X(2, 2, 4, GD_NST4, true, false) X(2, 2, 4, GD_NST4, false, true)                       \
    X(4, 2, 4, 6, false, false) X(1, 4, 4, 6, false, false)                                 \
    X(1, 1, 16, 6, false, false) X(2, 1, 16, 6, false, false) X(4, 1, 16, 6, false, false)     \
    X(1, 4, 2, 6, false, true) X(1, 4, 4, 6, false, true)

int width_class(int nwv) { return nwv <= 2 ? 2 : (nwv <= 4 ? 4 : 16); }

// Rows-per-warp preference among shapes with the same R.  The f64 blend replica
// runs R = 4 as four warp rows of one row (16 consumer warps to hide its f64
// latency; 128^3: 14.3 vs 25.3 ms), everything else -- f32 blend included, since
// its candidate became sqrt(lambda) * sqrt(di^2 + c0/lambda) -- as two warp rows
// of two (fewer window builds per voxel; lambda = 1: 13.3 vs 14.2 ms; f32 blend
// 512^3: 15.2 vs 15.7 ms of sweep, 16 x 256x256x160: 21.5 vs 31.2 ms;
// profiles/r02_variants.txt).  -1: per-kind default; 0: the first listed.
}  // namespace
extern int g_sweep_rw;  // sweep.cu
namespace {
// The f64 blend replica runs one row per warp (16 warps): it spills a little at
// 96 registers there, yet the spill-free 2x2 shape measured slower (512^3
// lambda = 0.5 exact: 193 vs 154 ms, profiles/r02_variants.txt).
int preferred_rw(int kind, bool f64 = false) {
    return g_sweep_rw >= 0 ? g_sweep_rw : (kind == kBlend && f64 ? 1 : 0);
}
// The preferred shape exists for (R, width class, tb)?
bool rw_pref_exists(int R, int mw, bool tb, int rw) {
#define GD_CASE(RWW, NW, MM, NS, T, C) \
    if (R == RWW * NW && mw == MM && tb == T && !C && RWW == rw) return true;
    GD_SWEEP_CASES(GD_CASE)
#undef GD_CASE
    return false;
}
// Shape filter: the preferred rows-per-warp when it exists, else the first listed.
struct RwSel {
    int want;
    RwSel(int R, int mw, bool tb, int rw) : want(rw_pref_exists(R, mw, tb, rw) ? rw : 0) {}
    bool ok(int rww) { return want == 0 ? take_first() : rww == want; }
    bool first = true;
    bool take_first() {
        const bool f = first;
        first = false;
        return f;
    }
};

template <int KIND, bool F64>
cudaError_t dispatch_r(int R, bool tb, const CUtensorMap& tm_d, const CUtensorMap& tm_i,
                       const SweepParams& p, cudaStream_t s) {
    const int mw = width_class(p.nwv);
    RwSel sel(R, mw, tb, preferred_rw(KIND, F64));
    const bool cl = p.cs > 1;
#define GD_CASE(RWW, NW, MM, NS, T, C)                               \
    if (R == RWW * NW && mw == MM && tb == T && cl == C && sel.ok(RWW)) \
        return launch_one<KIND, F64, RWW, NW, NS, MM, T, C>(tm_d, tm_i, p, s);
    GD_SWEEP_CASES(GD_CASE)
#undef GD_CASE
    return cudaErrorInvalidValue;
}

template <int KIND, bool F64>
int dispatch_cores(int R, bool tb, int nwv, int cs) {
    const int mw = width_class(nwv);
    RwSel sel(R, mw, tb, preferred_rw(KIND, F64));
#define GD_CASE(RWW, NW, MM, NS, T, C)                                      \
    if (R == RWW * NW && mw == MM && tb == T && (cs > 1) == C && sel.ok(RWW))  \
        return C ? coresident_clusters<KIND, F64, RWW, NW, NS, MM, T, C>(nwv, cs) \
                 : coresident<KIND, F64, RWW, NW, NS, MM, T, C>(nwv);
    GD_SWEEP_CASES(GD_CASE)
#undef GD_CASE
    return 0;
}

}  // namespace
}  // namespace gdb
