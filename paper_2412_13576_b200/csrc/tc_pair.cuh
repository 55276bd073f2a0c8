// CTA-pair (cta_group::2) tcgen05 / TMA / cluster helpers (raw PTX, sm_100a) for the large-shape descent
// kernel (k_descent_tcp.cu). Builds on tc_umma.cuh (descriptors, TMEM loads, mbarrier waits).
//
// Pair model (cluster of 2 CTAs on one TPC): tcgen05.mma.cta_group::2 is issued by one thread of the even
// (leader) CTA; the A operand is split by rows (each CTA holds its M/2 rows at the same shared-memory offset),
// the B operand by N (each CTA holds N/2 rows of the K-major B operand at the same offset), and each CTA's TMEM
// receives its own M/2 rows of D (M = 128: rows m < 64 at lane m + 64 * (n >= N/2), column n mod N/2).
// TMA loads of either CTA complete on the leader's mbarrier (.cta_group::2 with a cluster address).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "tc_umma.cuh"

namespace maple {
namespace pair {

using umma::smem_u32;

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

// shared::cluster address of the same variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}

__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// arrive on an mbarrier given by its shared::cluster address (possibly the peer's). Default semantics (release at
// CTA scope: MEMBAR.ALL.CTA + the arrive). Every consumer of these barriers is an async-proxy operation (an MMA
// reading this CTA's shared-memory operands or TMEM) issued after the wait, and every producer makes its data
// visible to that proxy before arriving (fence.proxy.async for shared-memory operands, tcgen05.wait::ld +
// tcgen05.fence::before_thread_sync for TMEM reads), so cluster-scope release adds nothing but its cost: it
// compiles to MEMBAR.ALL.GPU + ERRBAR + CGAERRBAR, which waits for this warp's outstanding global stores (the
// harvested rows) — 17 % of the CTA-pair kernel's stall samples in profiles/r2_ncu_descent_tcp_v7.md.
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t caddr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(caddr) : "memory");
}

// arrive on a local mbarrier and add `bytes` to its expected transaction count
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t saddr, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr), "r"(bytes) : "memory");
}

// Waits sleep in hardware for at most 20 us per probe; a phase that never completes traps after about 2^20
// probes (~20 s), so a protocol bug ends the kernel with an error instead of hanging the device.
// wait with cluster-scope acquire (for barriers whose arrivals come from the peer CTA's threads)
__device__ __forceinline__ bool mbar_try_cluster(uint32_t a, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}\n"
        : "=r"(ok)
        : "r"(a), "r"(parity), "r"(20000u)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ bool mbar_try_local(uint32_t a, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}\n"
        : "=r"(ok)
        : "r"(a), "r"(parity), "r"(20000u)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait_cluster(uint32_t a, uint32_t parity) {
    uint32_t spins = 0;
    while (!mbar_try_cluster(a, parity)) {
        if (++spins > (1u << 20)) asm volatile("trap;");
    }
}
__device__ __forceinline__ void mbar_wait_local(uint32_t a, uint32_t parity) {
    uint32_t spins = 0;
    while (!mbar_try_local(a, parity)) {
        if (++spins > (1u << 20)) asm volatile("trap;");
    }
}

// 3-D TMA tile load into this CTA's shared memory; completion (bytes) is signalled on the mbarrier at the
// shared::cluster address `mbar_c` (the leader CTA's barrier for pair MMAs)
__device__ __forceinline__ void tma_load_3d_pair(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                                 uint32_t mbar_c) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(mbar_c), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// instruction descriptors: kind::f16 with f16 A/B and fp32 D; kind::i8 with signed A/B and s32 D; K-major
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
    return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma2_f16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma2_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(id), "r"(acc));
}

// commit the leader's outstanding pair MMAs to the mbarrier at the same offset in every CTA of `mask`
__device__ __forceinline__ void commit2(uint64_t* mbar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(mbar)),
        "h"(mask)
        : "memory");
}

__device__ __forceinline__ void tmem_alloc2(uint32_t* dst, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)), "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc2(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

}  // namespace pair
}  // namespace maple
