// tc_common.cuh -- tcgen05 / TMA / mbarrier helpers shared by the tensor-core
// contraction kernels (contract_tc.cu: d <= 64, contract_tcw.cu: d > 64).
#pragma once

#include "common.cuh"
#include "kernels.h"

#include <cuda_fp16.h>

namespace rrs {

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    // tcgen05 shared-memory descriptor: start>>4 [0,14), LBO>>4 [16,30),
    // SBO>>4 [32,46), version 1 [46,48), base offset 0, layout SWIZZLE_NONE
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

// One MMA (K = 16): D (+)= A[aT] x B[bd]; `acc` nonzero accumulates into D.
__device__ __forceinline__ void umma_f16(uint32_t d, uint32_t aT, uint64_t bd, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
                 "r"(aT), "l"(bd), "r"(idesc), "r"(acc)
                 : "memory");
}

__device__ __forceinline__ bool elect_one() {
    uint32_t r;
    asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\nselp.u32 %0, 1, 0, e;\n}\n" : "=r"(r));
    return r != 0u;
}

// The 3 Q + R MMAs of one slice in the split-product layout (kernels.h
// tc_layout: Q aligned groups, R remainder steps), A / B K steps paired by
// tc_mma_steps; the first accumulates iff acc0.  Issued by the calling thread
// (the caller elects), fully unrolled so every operand offset is an immediate.
//   aT: the slice's A columns (K step i at +8 i); bd: descriptor of the slice's
//   B K step 0 (K step i at +256 i in descriptor units of 16 bytes)
template <int Q, int R>
__device__ __forceinline__ void mma_split_seq(uint32_t acc, uint32_t aT, uint64_t bd, uint32_t idesc, uint32_t acc0) {
#pragma unroll
    for (int i = 0; i < 3 * Q + R; ++i) {
        int sa, sb;
        tc_mma_steps(Q, i, sa, sb);
        umma_f16(acc, aT + 8u * (uint32_t)sa, bd + 256ull * (uint64_t)sb, idesc, i == 0 ? acc0 : 1u);
    }
}

// runtime (Q, R) -> the unrolled sequence (Q <= 4, R <= 3; Q = 4 has R = 0)
__device__ __forceinline__ void mma_split_seq_rt(int q, int r, uint32_t acc, uint32_t aT, uint64_t bd, uint32_t idesc,
                                                 uint32_t acc0) {
    switch (4 * q + r) {
        case 1: mma_split_seq<0, 1>(acc, aT, bd, idesc, acc0); break;
        case 2: mma_split_seq<0, 2>(acc, aT, bd, idesc, acc0); break;
        case 3: mma_split_seq<0, 3>(acc, aT, bd, idesc, acc0); break;
        case 4: mma_split_seq<1, 0>(acc, aT, bd, idesc, acc0); break;
        case 5: mma_split_seq<1, 1>(acc, aT, bd, idesc, acc0); break;
        case 6: mma_split_seq<1, 2>(acc, aT, bd, idesc, acc0); break;
        case 7: mma_split_seq<1, 3>(acc, aT, bd, idesc, acc0); break;
        case 8: mma_split_seq<2, 0>(acc, aT, bd, idesc, acc0); break;
        case 9: mma_split_seq<2, 1>(acc, aT, bd, idesc, acc0); break;
        case 10: mma_split_seq<2, 2>(acc, aT, bd, idesc, acc0); break;
        case 11: mma_split_seq<2, 3>(acc, aT, bd, idesc, acc0); break;
        case 12: mma_split_seq<3, 0>(acc, aT, bd, idesc, acc0); break;
        case 13: mma_split_seq<3, 1>(acc, aT, bd, idesc, acc0); break;
        case 14: mma_split_seq<3, 2>(acc, aT, bd, idesc, acc0); break;
        case 15: mma_split_seq<3, 3>(acc, aT, bd, idesc, acc0); break;
        default: mma_split_seq<4, 0>(acc, aT, bd, idesc, acc0); break;
    }
}

// One (point tile, direction block) product of a single slice (d <= 64), then
// the commit to `bar`; one elected thread issues all.
template <int Q, int R>
__device__ __forceinline__ void mma_split_block(uint32_t acc, uint32_t aT, uint64_t bd, uint32_t idesc, uint32_t bar) {
    if (elect_one()) {
        mma_split_seq<Q, R>(acc, aT, bd, idesc, 0u);
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                     : "memory");
    }
    __syncwarp();
}

// One (point tile, direction block) product with NS consecutive K steps paired
// one to one (contract_tcf.cu's single-product layout): MMA i reads A step i
// and B step i, the first overwrites the accumulator; then the commit.
template <int NS>
__device__ __forceinline__ void mma_tile_block(uint32_t acc, uint32_t aT, uint64_t bd, uint32_t idesc, uint32_t bar) {
    if (elect_one()) {
#pragma unroll
        for (int i = 0; i < NS; ++i) umma_f16(acc, aT + 8u * i, bd + 256ull * i, idesc, i > 0 ? 1u : 0u);
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                     : "memory");
    }
    __syncwarp();
}

// A direction block in the staging area (canonical K-major [kk/8][128][16 B]) ->
// TMEM columns [aT, aT + 8 ns): one 128x256b copy (two 16-byte chunks) per K
// step (once per unit, so a plain loop of elected copies).
__device__ __forceinline__ void tmem_cp_dirblock(uint32_t aT, uint64_t sd, int ns) {
    for (int i = 0; i < ns; ++i)
        asm volatile(
            "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
            "@e tcgen05.cp.cta_group::1.128x256b [%0], %1;\n}\n" ::"r"(aT + 8u * (uint32_t)i),
            "l"(sd + 256ull * (uint64_t)i));
}

__device__ __forceinline__ void mma_commit_elect(uint64_t* bar) {
    asm volatile(
        "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tma_load_elect(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
        "@e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n}\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void expect_tx_elect(uint64_t* bar, uint32_t bytes) {
    asm volatile(
        "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
        "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n}\n" ::"r"(smem_u32(bar)),
        "r"(bytes)
        : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Wait with a suspend-time hint (for warps that run ahead of their consumer).
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAITS_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra WAITS_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(1000000u)
        : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void named_bar(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

__device__ __forceinline__ uint32_t pack_half2(float lo_elem, float hi_elem) {
    const __half2 h = __floats2half2_rn(lo_elem, hi_elem);
    return *reinterpret_cast<const uint32_t*>(&h);
}

}  // namespace rrs
