// Device-side primitives for the sm_100a sweep kernels: mbarrier + TMA (async
// proxy), and the relaxed 64-bit tagged stores/loads used for the inter-CTA
// halo hand-off.  Raw PTX; no CUTLASS.
#pragma once

#include <cuda.h>
#include <cstdint>

namespace gdb {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- mbarrier -------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

// try_wait suspends the warp until the phase completes or the time hint (ns)
// expires, instead of returning at once and spinning on issue slots the other
// warps of the scheduler could use.
#ifndef GD_MBAR_HINT
#define GD_MBAR_HINT 1000000
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#if GD_MBAR_HINT > 0
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "GD_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra GD_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity), "n"(GD_MBAR_HINT)
        : "memory");
#else
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "GD_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra GD_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
#endif
}

// ---- thread-block clusters (DSMEM halo links) --------------------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// Address of the same shared variable in CTA `rank` of this cluster.
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
// 16-byte remote store that completes 16 bytes of tx on the remote mbarrier.
__device__ __forceinline__ void st_async_v4(uint32_t raddr, float a, float b, float c, float d,
                                            uint32_t rbar) {
    asm volatile(
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];"
        ::"r"(raddr), "f"(a), "f"(b), "f"(c), "f"(d), "r"(rbar)
        : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
                 ::: "memory");
}

// ---- TMA ------------------------------------------------------------------
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* m) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* m, uint64_t* bar,
                                            int c0, int c1, int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
        "r"(smem_u32(bar))
        : "memory");
}

// Generic-proxy global writes -> later async-proxy (TMA) reads of the same data.
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

// ---- tagged halo words: {f32 value, u32 tag} in one single-copy-atomic b64 --
// Memory-model qualifiers of the halo accesses (relaxed, GPU scope: coherent at
// L2, 8-byte single-copy atomic).  Overridable for experiments.
#ifndef GD_HALO_LD
#define GD_HALO_LD "ld.relaxed.gpu.global"
#endif
#ifndef GD_HALO_ST
#define GD_HALO_ST "st.relaxed.gpu.global"
#endif
__device__ __forceinline__ void st_tagged(unsigned long long* p, float v, uint32_t tag) {
    const unsigned long long w =
        (static_cast<unsigned long long>(tag) << 32) | __float_as_uint(v);
    asm volatile("" GD_HALO_ST ".b64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}

__device__ __forceinline__ unsigned long long ld_tagged(const unsigned long long* p) {
    unsigned long long w;
    asm volatile("" GD_HALO_LD ".b64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
    return w;
}

// Two adjacent words in one 16-byte access; each 8-byte element is still
// single-copy atomic (vector accesses behave as per-element scalar accesses).
__device__ __forceinline__ void st_tagged2(unsigned long long* p, float v0, float v1, uint32_t tag) {
    const unsigned long long w0 = (static_cast<unsigned long long>(tag) << 32) | __float_as_uint(v0);
    const unsigned long long w1 = (static_cast<unsigned long long>(tag) << 32) | __float_as_uint(v1);
    asm volatile("" GD_HALO_ST ".v2.b64 [%0], {%1, %2};" ::"l"(p), "l"(w0), "l"(w1)
                 : "memory");
}

__device__ __forceinline__ void ld_tagged2(const unsigned long long* p, unsigned long long& w0,
                                           unsigned long long& w1) {
    asm volatile("" GD_HALO_LD ".v2.b64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p)
                 : "memory");
}

__device__ __forceinline__ uint32_t tag_of(unsigned long long w) {
    return static_cast<uint32_t>(w >> 32);
}
__device__ __forceinline__ float val_of(unsigned long long w) {
    return __uint_as_float(static_cast<uint32_t>(w));
}

}  // namespace gdb
