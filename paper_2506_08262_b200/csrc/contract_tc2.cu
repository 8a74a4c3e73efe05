// contract_tc2.cu -- K2 on a pair of SMs: the contract_tc.cu contraction with
// cta_group::2 MMAs (M = 256 directions = one 128-direction block per CTA of a
// 2-CTA cluster, N = 128 points = 64 converted by each CTA).
//
// Same operands, packed K layout (kernels.h tc_layout), arithmetic and result
// contract as contract_tc.cu; what changes is the division of labour:
//   * one tcgen05.mma.cta_group::2 (issued by the even CTA) drives both SMs'
//     tensor cores: each CTA's TMEM holds its own direction block (A, TS mode)
//     and its 128 x 128 accumulator; B is split by N, each CTA's shared memory
//     holds the 64 points it converted;
//   * so every SM converts only half of each point tile (x - z, per-point
//     scale, FP16 split) while its tensor core still does a full tile's MMAs
//     -- the converter warps were the issue-slot bottleneck of the 1-SM kernel;
//   * the commits multicast to both CTAs (accumulator full, point stage free,
//     staging free); the odd CTA's converter and epilogue warps arrive on the
//     even CTA's barriers through cluster addresses (release/acquire.cluster);
//     excluded-point masks are exchanged through distributed shared memory.
// Work unit = (query, group of <= gb block pairs, chunk of tiles); the pair
// processes the unit together, CTA r owning block 2 p + r of pair p.
// Replaces _kernels.pyx:120-199 (projection) + 270-289 (halfspace_span).
#include "common.cuh"
#include "kernels.h"

#include <cuda_fp16.h>

namespace rrs {
namespace {

constexpr int T2_CONV_WARP0 = 3;
constexpr int T2_CONV_WARPS = 8;                 // (point of 64, K quarter) per thread
constexpr int T2_CONV_THREADS = T2_CONV_WARPS * 32;
constexpr int T2_EPI_WARP0 = T2_CONV_WARP0 + T2_CONV_WARPS;
constexpr int T2_EPI_WARPS = 8;
constexpr int T2_EPI_THREADS = T2_EPI_WARPS * 32;
constexpr int T2_THREADS = (T2_EPI_WARP0 + T2_EPI_WARPS) * 32;  // 608
constexpr int T2_MAXD = 64;
constexpr int T2_MAXNS = 12;
constexpr int T2_MD = 128;                       // directions per CTA block
constexpr int T2_NP = 128;                       // points per tile (MMA N)
constexpr int T2_NH = 64;                        // points per CTA per tile
constexpr int T2_GB_MAX = 8;
constexpr int T2_PST = 4;                        // point operand stages (half tiles)
constexpr int T2_R_MAX = 4;
constexpr uint32_t T2_TMEM_COLS = 512;
constexpr uint32_t T2_ACC = T2_NP;               // 128 columns per accumulator buffer
constexpr uint32_t T2_A = 2 * T2_ACC;            // direction blocks from column 256
constexpr int T2_SMEM_LIMIT = 227 * 1024;

struct T2Smem {
    int P, D, CNT, ZS, SMX, EXCL, ZROWS, BARS, TADDR, RAW, total;
    int stage_bytes, dblock_bytes, raw_stages;
    static constexpr int NBARS = 2 * T2_PST + 2 + 2 + 4 + 2 * T2_R_MAX + 8;
    __host__ __device__ T2Smem(int ns, int d) {
        stage_bytes = ns * 2048;                  // 64 points x 16 K values x 2 B per K step
        dblock_bytes = ns * 4096;                 // 128 directions
        P = 0;
        D = P + T2_PST * stage_bytes;
        CNT = D + dblock_bytes;                   // uint32 [T2_GB_MAX * 128]
        ZS = CNT + T2_GB_MAX * T2_MD * 4;         // float [2][64]
        SMX = ZS + 2 * T2_MAXD * 4;               // float [2][4][64]
        EXCL = SMX + 2 * 4 * T2_NH * 4;           // uint32 [8][4]
        ZROWS = EXCL + 8 * 4 * 4;                 // uint32 [4]
        BARS = ZROWS + 16;
        TADDR = BARS + NBARS * 8;
        RAW = (TADDR + 16 + 1023) & ~1023;        // raw FP32 tiles [64][128]
        const int room = T2_SMEM_LIMIT - 1024 - RAW;
        raw_stages = room / (T2_MAXD * T2_NP * 4);
        if (raw_stages > T2_R_MAX) raw_stages = T2_R_MAX;
        total = RAW + raw_stages * T2_MAXD * T2_NP * 4 + 1024;
        (void)d;
    }
};

__device__ __forceinline__ uint64_t desc2(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

template <int NS>
__device__ __forceinline__ void mma2_tile_block(uint32_t acc, uint32_t aT, uint64_t bd, uint32_t idesc, uint32_t bar);

template <>
__device__ __forceinline__ void mma2_tile_block<1>(uint32_t acc, uint32_t aT, uint64_t bd, uint32_t idesc, uint32_t bar) {
    asm volatile("{\n.reg .pred e;\n.reg .b16 msk;\nelect.sync _|e, 0xffffffff;\nmov.b16 msk, 3;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+0], %2, %3, 0;\n"
                 "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%4], msk;\n}\n"
                 ::"r"(acc), "r"(aT), "l"(bd), "r"(idesc), "r"(bar) : "memory");
}

template <>
__device__ __forceinline__ void mma2_tile_block<2>(uint32_t acc, uint32_t aT, uint64_t bd, uint32_t idesc, uint32_t bar) {
    asm volatile("{\n.reg .pred e;\n.reg .b16 msk;\n.reg .b64 b1;\nelect.sync _|e, 0xffffffff;\nmov.b16 msk, 3;\n"
                 "add.s64 b1, %2, 128;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+0], %2, %3, 0;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+8], b1, %3, 1;\n"
                 "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%4], msk;\n}\n"
                 ::"r"(acc), "r"(aT), "l"(bd), "r"(idesc), "r"(bar) : "memory");
}

template <>
__device__ __forceinline__ void mma2_tile_block<3>(uint32_t acc, uint32_t aT, uint64_t bd, uint32_t idesc, uint32_t bar) {
    asm volatile("{\n.reg .pred e;\n.reg .b16 msk;\n.reg .b64 b1, b2;\nelect.sync _|e, 0xffffffff;\nmov.b16 msk, 3;\n"
                 "add.s64 b1, %2, 128;\n"
                 "add.s64 b2, %2, 256;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+0], %2, %3, 0;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+8], b1, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+16], b2, %3, 1;\n"
                 "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%4], msk;\n}\n"
                 ::"r"(acc), "r"(aT), "l"(bd), "r"(idesc), "r"(bar) : "memory");
}

template <>
__device__ __forceinline__ void mma2_tile_block<4>(uint32_t acc, uint32_t aT, uint64_t bd, uint32_t idesc, uint32_t bar) {
    asm volatile("{\n.reg .pred e;\n.reg .b16 msk;\n.reg .b64 b1, b2, b3;\nelect.sync _|e, 0xffffffff;\nmov.b16 msk, 3;\n"
                 "add.s64 b1, %2, 128;\n"
                 "add.s64 b2, %2, 256;\n"
                 "add.s64 b3, %2, 384;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+0], %2, %3, 0;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+8], b1, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+16], b2, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+24], b3, %3, 1;\n"
                 "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%4], msk;\n}\n"
                 ::"r"(acc), "r"(aT), "l"(bd), "r"(idesc), "r"(bar) : "memory");
}

template <>
__device__ __forceinline__ void mma2_tile_block<5>(uint32_t acc, uint32_t aT, uint64_t bd, uint32_t idesc, uint32_t bar) {
    asm volatile("{\n.reg .pred e;\n.reg .b16 msk;\n.reg .b64 b1, b2, b3, b4;\nelect.sync _|e, 0xffffffff;\nmov.b16 msk, 3;\n"
                 "add.s64 b1, %2, 128;\n"
                 "add.s64 b2, %2, 256;\n"
                 "add.s64 b3, %2, 384;\n"
                 "add.s64 b4, %2, 512;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+0], %2, %3, 0;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+8], b1, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+16], b2, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+24], b3, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+32], b4, %3, 1;\n"
                 "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%4], msk;\n}\n"
                 ::"r"(acc), "r"(aT), "l"(bd), "r"(idesc), "r"(bar) : "memory");
}

template <>
__device__ __forceinline__ void mma2_tile_block<6>(uint32_t acc, uint32_t aT, uint64_t bd, uint32_t idesc, uint32_t bar) {
    asm volatile("{\n.reg .pred e;\n.reg .b16 msk;\n.reg .b64 b1, b2, b3, b4, b5;\nelect.sync _|e, 0xffffffff;\nmov.b16 msk, 3;\n"
                 "add.s64 b1, %2, 128;\n"
                 "add.s64 b2, %2, 256;\n"
                 "add.s64 b3, %2, 384;\n"
                 "add.s64 b4, %2, 512;\n"
                 "add.s64 b5, %2, 640;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+0], %2, %3, 0;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+8], b1, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+16], b2, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+24], b3, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+32], b4, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+40], b5, %3, 1;\n"
                 "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%4], msk;\n}\n"
                 ::"r"(acc), "r"(aT), "l"(bd), "r"(idesc), "r"(bar) : "memory");
}

template <>
__device__ __forceinline__ void mma2_tile_block<7>(uint32_t acc, uint32_t aT, uint64_t bd, uint32_t idesc, uint32_t bar) {
    asm volatile("{\n.reg .pred e;\n.reg .b16 msk;\n.reg .b64 b1, b2, b3, b4, b5, b6;\nelect.sync _|e, 0xffffffff;\nmov.b16 msk, 3;\n"
                 "add.s64 b1, %2, 128;\n"
                 "add.s64 b2, %2, 256;\n"
                 "add.s64 b3, %2, 384;\n"
                 "add.s64 b4, %2, 512;\n"
                 "add.s64 b5, %2, 640;\n"
                 "add.s64 b6, %2, 768;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+0], %2, %3, 0;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+8], b1, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+16], b2, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+24], b3, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+32], b4, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+40], b5, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+48], b6, %3, 1;\n"
                 "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%4], msk;\n}\n"
                 ::"r"(acc), "r"(aT), "l"(bd), "r"(idesc), "r"(bar) : "memory");
}

template <>
__device__ __forceinline__ void mma2_tile_block<8>(uint32_t acc, uint32_t aT, uint64_t bd, uint32_t idesc, uint32_t bar) {
    asm volatile("{\n.reg .pred e;\n.reg .b16 msk;\n.reg .b64 b1, b2, b3, b4, b5, b6, b7;\nelect.sync _|e, 0xffffffff;\nmov.b16 msk, 3;\n"
                 "add.s64 b1, %2, 128;\n"
                 "add.s64 b2, %2, 256;\n"
                 "add.s64 b3, %2, 384;\n"
                 "add.s64 b4, %2, 512;\n"
                 "add.s64 b5, %2, 640;\n"
                 "add.s64 b6, %2, 768;\n"
                 "add.s64 b7, %2, 896;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+0], %2, %3, 0;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+8], b1, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+16], b2, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+24], b3, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+32], b4, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+40], b5, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+48], b6, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+56], b7, %3, 1;\n"
                 "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%4], msk;\n}\n"
                 ::"r"(acc), "r"(aT), "l"(bd), "r"(idesc), "r"(bar) : "memory");
}

template <>
__device__ __forceinline__ void mma2_tile_block<9>(uint32_t acc, uint32_t aT, uint64_t bd, uint32_t idesc, uint32_t bar) {
    asm volatile("{\n.reg .pred e;\n.reg .b16 msk;\n.reg .b64 b1, b2, b3, b4, b5, b6, b7, b8;\nelect.sync _|e, 0xffffffff;\nmov.b16 msk, 3;\n"
                 "add.s64 b1, %2, 128;\n"
                 "add.s64 b2, %2, 256;\n"
                 "add.s64 b3, %2, 384;\n"
                 "add.s64 b4, %2, 512;\n"
                 "add.s64 b5, %2, 640;\n"
                 "add.s64 b6, %2, 768;\n"
                 "add.s64 b7, %2, 896;\n"
                 "add.s64 b8, %2, 1024;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+0], %2, %3, 0;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+8], b1, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+16], b2, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+24], b3, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+32], b4, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+40], b5, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+48], b6, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+56], b7, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+64], b8, %3, 1;\n"
                 "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%4], msk;\n}\n"
                 ::"r"(acc), "r"(aT), "l"(bd), "r"(idesc), "r"(bar) : "memory");
}

template <>
__device__ __forceinline__ void mma2_tile_block<10>(uint32_t acc, uint32_t aT, uint64_t bd, uint32_t idesc, uint32_t bar) {
    asm volatile("{\n.reg .pred e;\n.reg .b16 msk;\n.reg .b64 b1, b2, b3, b4, b5, b6, b7, b8, b9;\nelect.sync _|e, 0xffffffff;\nmov.b16 msk, 3;\n"
                 "add.s64 b1, %2, 128;\n"
                 "add.s64 b2, %2, 256;\n"
                 "add.s64 b3, %2, 384;\n"
                 "add.s64 b4, %2, 512;\n"
                 "add.s64 b5, %2, 640;\n"
                 "add.s64 b6, %2, 768;\n"
                 "add.s64 b7, %2, 896;\n"
                 "add.s64 b8, %2, 1024;\n"
                 "add.s64 b9, %2, 1152;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+0], %2, %3, 0;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+8], b1, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+16], b2, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+24], b3, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+32], b4, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+40], b5, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+48], b6, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+56], b7, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+64], b8, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+72], b9, %3, 1;\n"
                 "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%4], msk;\n}\n"
                 ::"r"(acc), "r"(aT), "l"(bd), "r"(idesc), "r"(bar) : "memory");
}

template <>
__device__ __forceinline__ void mma2_tile_block<11>(uint32_t acc, uint32_t aT, uint64_t bd, uint32_t idesc, uint32_t bar) {
    asm volatile("{\n.reg .pred e;\n.reg .b16 msk;\n.reg .b64 b1, b2, b3, b4, b5, b6, b7, b8, b9, b10;\nelect.sync _|e, 0xffffffff;\nmov.b16 msk, 3;\n"
                 "add.s64 b1, %2, 128;\n"
                 "add.s64 b2, %2, 256;\n"
                 "add.s64 b3, %2, 384;\n"
                 "add.s64 b4, %2, 512;\n"
                 "add.s64 b5, %2, 640;\n"
                 "add.s64 b6, %2, 768;\n"
                 "add.s64 b7, %2, 896;\n"
                 "add.s64 b8, %2, 1024;\n"
                 "add.s64 b9, %2, 1152;\n"
                 "add.s64 b10, %2, 1280;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+0], %2, %3, 0;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+8], b1, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+16], b2, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+24], b3, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+32], b4, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+40], b5, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+48], b6, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+56], b7, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+64], b8, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+72], b9, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+80], b10, %3, 1;\n"
                 "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%4], msk;\n}\n"
                 ::"r"(acc), "r"(aT), "l"(bd), "r"(idesc), "r"(bar) : "memory");
}

template <>
__device__ __forceinline__ void mma2_tile_block<12>(uint32_t acc, uint32_t aT, uint64_t bd, uint32_t idesc, uint32_t bar) {
    asm volatile("{\n.reg .pred e;\n.reg .b16 msk;\n.reg .b64 b1, b2, b3, b4, b5, b6, b7, b8, b9, b10, b11;\nelect.sync _|e, 0xffffffff;\nmov.b16 msk, 3;\n"
                 "add.s64 b1, %2, 128;\n"
                 "add.s64 b2, %2, 256;\n"
                 "add.s64 b3, %2, 384;\n"
                 "add.s64 b4, %2, 512;\n"
                 "add.s64 b5, %2, 640;\n"
                 "add.s64 b6, %2, 768;\n"
                 "add.s64 b7, %2, 896;\n"
                 "add.s64 b8, %2, 1024;\n"
                 "add.s64 b9, %2, 1152;\n"
                 "add.s64 b10, %2, 1280;\n"
                 "add.s64 b11, %2, 1408;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+0], %2, %3, 0;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+8], b1, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+16], b2, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+24], b3, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+32], b4, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+40], b5, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+48], b6, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+56], b7, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+64], b8, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+72], b9, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+80], b10, %3, 1;\n"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+88], b11, %3, 1;\n"
                 "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%4], msk;\n}\n"
                 ::"r"(acc), "r"(aT), "l"(bd), "r"(idesc), "r"(bar) : "memory");
}

__device__ __forceinline__ uint32_t cta_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t map_to(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on an mbarrier given by its cluster address (local or the peer's)
__device__ __forceinline__ void arrive_cluster(uint32_t caddr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(caddr) : "memory");
}
// relaxed arrival (no memory ordering): for "accumulator drained" -- the TMEM
// reads are already complete (tcgen05.wait::ld + fence::before_thread_sync)
__device__ __forceinline__ void arrive_cluster_relaxed(uint32_t caddr) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(caddr) : "memory");
}
__device__ __forceinline__ void wait_cluster(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred p;\nW2C_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra W2C_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void wait_sleep(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred p;\nW2S_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra W2S_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(1000000u)
        : "memory");
}
__device__ __forceinline__ void commit2_mc(uint64_t* bar) {
    asm volatile(
        "{\n.reg .pred e;\n.reg .b16 msk;\nelect.sync _|e, 0xffffffff;\nmov.b16 msk, 3;\n"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], msk;\n}\n" ::"r"(
            smem_u32(bar))
        : "memory");
}
// commit that arrives only on the leader's (rank 0) barrier
__device__ __forceinline__ void commit2_leader(uint64_t* bar) {
    asm volatile(
        "{\n.reg .pred e;\n.reg .b16 msk;\nelect.sync _|e, 0xffffffff;\nmov.b16 msk, 1;\n"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], msk;\n}\n" ::"r"(
            smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_load2(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
        "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%3], %2;\n"
        "@e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n}\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tmem_cp2_block(uint32_t aT, uint64_t sd, int ns) {
    for (int i = 0; i < ns; ++i)
        asm volatile(
            "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
            "@e tcgen05.cp.cta_group::2.128x256b [%0], %1;\n}\n" ::"r"(aT + 8u * (uint32_t)i),
            "l"(sd + 256ull * (uint64_t)i));
}
__device__ __forceinline__ void fence_before2() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after2() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld32x(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
__device__ __forceinline__ void bar_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

struct T2Unit {
    int q, grp, npg;     // query, pair group, pairs in the group
    int64_t t0, t1;
};
__device__ __forceinline__ T2Unit t2_unit(const TcArgs& a, int64_t u) {
    T2Unit r;
    const int64_t per_q = (int64_t)a.groups * a.chunks;
    r.q = (int)(u / per_q);
    const int64_t rem = u - (int64_t)r.q * per_q;
    r.grp = (int)(rem / a.chunks);
    const int64_t c = rem - (int64_t)r.grp * a.chunks;
    const int npairs = (a.NB + 1) / 2;
    r.npg = npairs - r.grp * a.gb < a.gb ? npairs - r.grp * a.gb : a.gb;
    r.t0 = c * a.tiles_per_chunk;
    r.t1 = r.t0 + a.tiles_per_chunk < a.tiles ? r.t0 + a.tiles_per_chunk : a.tiles;
    return r;
}

template <int NS>
__device__ __forceinline__ void mma2_issue(const TcArgs& a, int64_t u0, int64_t ustride, int64_t units,
                                           unsigned char* sP, uint64_t* pfull, uint64_t* pempty, uint64_t* dfull,
                                           uint64_t* dpeer, uint64_t* dempty, uint64_t* tfull, uint64_t* tempty,
                                           uint64_t* udone, uint32_t dbase) {
    constexpr uint32_t stage_bytes = NS * 2048;
    // F32 accumulate, FP16 A and B, K-major, N = 128, M = 256 (two CTAs)
    const uint32_t idesc = (1u << 4) | ((uint32_t)(T2_NP >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
    uint32_t it = 0, gtile = 0, gacc = 0, gph = 0;
    for (int64_t u = u0; u < units; u += ustride, ++it) {
        const T2Unit w = t2_unit(a, u);
        for (int p = 0; p < w.npg; ++p, ++gph) {
            mbar_wait(dfull, gph & 1u);       // own staging landed
            wait_cluster(dpeer, gph & 1u);    // peer's staging landed
            if (p == 0 && it > 0) mbar_wait(udone, (it - 1) & 1u);
            fence_after2();
            tmem_cp2_block(T2_A + 8u * NS * p, desc2(dbase, 2048, 128), NS);
            commit2_mc(dempty);
        }
        for (int64_t t = w.t0; t < w.t1; ++t, ++gtile) {
            const uint32_t s = gtile % T2_PST;
            wait_cluster(&pfull[s], (gtile / T2_PST) & 1u);
            fence_after2();
            // half tile [kk/8][64 points][16 B]: LBO 1024, SBO 128
            const uint64_t bd = desc2(smem_u32(sP) + s * stage_bytes, 1024, 128);
            for (int p = 0; p < w.npg; ++p, ++gacc) {
                const uint32_t buf = gacc & 1u;
                if (gacc >= 2) wait_cluster(&tempty[buf], ((gacc >> 1) - 1) & 1u);
                fence_after2();
                mma2_tile_block<NS>(buf * T2_ACC, T2_A + 8u * NS * p, bd, idesc, smem_u32(&tfull[buf]));
            }
            commit2_mc(&pempty[s]);
        }
        commit2_leader(udone);
    }
}

}  // namespace

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(T2_THREADS, 1) contract_tc2_kernel(const TcArgs a) {
    extern __shared__ __align__(1024) unsigned char t2_raw[];
    unsigned char* sm = t2_raw + ((1024u - (smem_u32(t2_raw) & 1023u)) & 1023u);
    const int d = a.d;
    const TcLayout L = tc_layout(d);
    const T2Smem lay(L.ns, d);
    const int stage_bytes = lay.stage_bytes, dblock = lay.dblock_bytes;
    unsigned char* sP = sm + lay.P;
    unsigned char* sD = sm + lay.D;
    uint32_t* sCnt = reinterpret_cast<uint32_t*>(sm + lay.CNT);
    float* sZ = reinterpret_cast<float*>(sm + lay.ZS);
    float* sMx = reinterpret_cast<float*>(sm + lay.SMX);
    uint32_t* sExcl = reinterpret_cast<uint32_t*>(sm + lay.EXCL);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + lay.BARS);
    uint64_t* pfull = &bars[0];                              // [T2_PST] leader: 16 arrivals
    uint64_t* pempty = &bars[T2_PST];                        // [T2_PST] multicast commit
    uint64_t* tfull = &bars[2 * T2_PST];                     // [2] multicast commit
    uint64_t* tempty = &bars[2 * T2_PST + 2];                // [2] leader: 16 arrivals
    uint64_t* dfull = &bars[2 * T2_PST + 4];                 // own staging (TMA tx)
    uint64_t* dpeer = &bars[2 * T2_PST + 5];                 // leader: peer's staging landed
    uint64_t* dempty = &bars[2 * T2_PST + 6];                // multicast commit
    uint64_t* udone = &bars[2 * T2_PST + 7];                 // leader: unit's MMAs done
    uint64_t* rfull = &bars[2 * T2_PST + 8];                 // [T2_R_MAX]
    uint64_t* rempty = &bars[2 * T2_PST + 8 + T2_R_MAX];     // [T2_R_MAX]
    uint64_t* xfull = &bars[2 * T2_PST + 8 + 2 * T2_R_MAX];  // [8] exclusion words of a tile
    uint32_t* sTaddr = reinterpret_cast<uint32_t*>(sm + lay.TADDR);
    float* sRaw = reinterpret_cast<float*>(sm + lay.RAW);
    const int RS = lay.raw_stages;
    const uint32_t raw_bytes = (uint32_t)(d * T2_NP * 4);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t rank = cta_rank();
    const int64_t units = (int64_t)a.Qb * a.groups * a.chunks;
    const int64_t u0 = blockIdx.x >> 1, ustride = gridDim.x >> 1;

    for (int i = tid; i < T2_PST * stage_bytes / 16; i += T2_THREADS)
        reinterpret_cast<uint4*>(sP)[i] = make_uint4(0u, 0u, 0u, 0u);
    for (int i = tid; i < RS * T2_MAXD * T2_NP; i += T2_THREADS) sRaw[i] = 0.0f;
    for (int c = tid; c < T2_GB_MAX * T2_MD; c += T2_THREADS) sCnt[c] = 0u;
    if (tid == 0) {
        for (int s = 0; s < T2_PST; ++s) {
            mbar_init(&pfull[s], 2 * T2_CONV_WARPS);
            mbar_init(&pempty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 2 * T2_EPI_WARPS);
        }
        mbar_init(dfull, 1);
        mbar_init(dpeer, 1);
        mbar_init(dempty, 1);
        mbar_init(udone, 1);
        for (int r = 0; r < T2_R_MAX; ++r) {
            mbar_init(&rfull[r], 1);
            mbar_init(&rempty[r], T2_CONV_WARPS);
        }
        for (int x = 0; x < 8; ++x) mbar_init(&xfull[x], 4);  // 2 local + 2 remote ballot warps
        fence_mbar_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(sTaddr)),
                     "r"(T2_TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    fence_proxy_async();
    fence_before2();
    __syncthreads();
    cluster_sync();  // both CTAs' barriers initialised before any remote arrival
    fence_after2();
    if (*sTaddr != 0u) __trap();
    const uint32_t peer = rank ^ 1u;

    if (warp == 0) {
        // ------------------- producer: this CTA's block of each pair (2 p + rank)
        uint32_t gph = 0;
        for (int64_t u = u0; u < units; u += ustride) {
            const T2Unit w = t2_unit(a, u);
            for (int p = 0; p < w.npg; ++p, ++gph) {
                const int blk = 2 * (w.grp * a.gb + p) + (int)rank;
                if (gph > 0) wait_sleep(dempty, (gph - 1) & 1u);
                if (blk < a.NB) {
                    tma_load2(sD, a.uop + ((size_t)w.q * a.NB + blk) * dblock, (uint32_t)dblock, dfull);
                } else {
                    // odd block count: a zero block (directions past m)
                    for (int i = lane; i < dblock / 16; i += 32)
                        reinterpret_cast<uint4*>(sD)[i] = make_uint4(0u, 0u, 0u, 0u);
                    fence_proxy_async();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(dfull);
                }
                __syncwarp();
                if (rank == 1) {
                    // tell the leader once our staging has landed
                    mbar_wait(dfull, gph & 1u);
                    if (lane == 0) arrive_cluster(map_to(smem_u32(dpeer), 0));
                    __syncwarp();
                }
            }
        }
    } else if (warp == 1) {
        if (rank == 0) {
            switch (L.ns) {
                case 1: mma2_issue<1>(a, u0, ustride, units, sP, pfull, pempty, dfull, dpeer, dempty, tfull, tempty, udone, smem_u32(sD)); break;
                case 2: mma2_issue<2>(a, u0, ustride, units, sP, pfull, pempty, dfull, dpeer, dempty, tfull, tempty, udone, smem_u32(sD)); break;
                case 3: mma2_issue<3>(a, u0, ustride, units, sP, pfull, pempty, dfull, dpeer, dempty, tfull, tempty, udone, smem_u32(sD)); break;
                case 4: mma2_issue<4>(a, u0, ustride, units, sP, pfull, pempty, dfull, dpeer, dempty, tfull, tempty, udone, smem_u32(sD)); break;
                case 5: mma2_issue<5>(a, u0, ustride, units, sP, pfull, pempty, dfull, dpeer, dempty, tfull, tempty, udone, smem_u32(sD)); break;
                case 6: mma2_issue<6>(a, u0, ustride, units, sP, pfull, pempty, dfull, dpeer, dempty, tfull, tempty, udone, smem_u32(sD)); break;
                case 7: mma2_issue<7>(a, u0, ustride, units, sP, pfull, pempty, dfull, dpeer, dempty, tfull, tempty, udone, smem_u32(sD)); break;
                case 8: mma2_issue<8>(a, u0, ustride, units, sP, pfull, pempty, dfull, dpeer, dempty, tfull, tempty, udone, smem_u32(sD)); break;
                case 9: mma2_issue<9>(a, u0, ustride, units, sP, pfull, pempty, dfull, dpeer, dempty, tfull, tempty, udone, smem_u32(sD)); break;
                case 10: mma2_issue<10>(a, u0, ustride, units, sP, pfull, pempty, dfull, dpeer, dempty, tfull, tempty, udone, smem_u32(sD)); break;
                case 11: mma2_issue<11>(a, u0, ustride, units, sP, pfull, pempty, dfull, dpeer, dempty, tfull, tempty, udone, smem_u32(sD)); break;
                default: mma2_issue<12>(a, u0, ustride, units, sP, pfull, pempty, dfull, dpeer, dempty, tfull, tempty, udone, smem_u32(sD)); break;
            }
        }
    } else if (warp == 2) {
        // ------------------------------- producer: raw FP32 tiles (whole tile)
        uint32_t g = 0, rs = 0, rph = 0;
        for (int64_t u = u0; u < units; u += ustride) {
            const T2Unit w = t2_unit(a, u);
            for (int64_t t = w.t0; t < w.t1; ++t, ++g) {
                if (g >= (uint32_t)RS) wait_sleep(&rempty[rs], rph ^ 1u);
                tma_load2(sRaw + (size_t)rs * T2_MAXD * T2_NP, a.xb + (size_t)t * d * T2_NP, raw_bytes, &rfull[rs]);
                __syncwarp();
                if (++rs == (uint32_t)RS) {
                    rs = 0;
                    rph ^= 1u;
                }
            }
        }
    } else if (warp < T2_EPI_WARP0) {
        // ------------- converters: this CTA's 64 points of each tile, K in quarters
        const int ct = tid - T2_CONV_WARP0 * 32;     // 0..255
        const int r = ct & (T2_NH - 1);              // point of the half tile
        const int h = ct >> 6;                       // coordinates [16 h, 16 h + 16)
        const int col = (int)rank * T2_NH + r;       // point within the 128-point tile
        const int main_chunks = 2 * L.q16;
        const uint32_t pfull0 = map_to(smem_u32(pfull), 0);
        uint32_t it = 0, gtile = 0, rs = 0, rph = 0;
        for (int64_t u = u0; u < units; u += ustride, ++it) {
            const T2Unit w = t2_unit(a, u);
            float* zs = sZ + (it & 1u) * T2_MAXD;
            if (ct < T2_MAXD) zs[ct] = ct < d ? __ldg(a.zq + (size_t)w.q * d + ct) : 0.0f;
            bar_sync(2, T2_CONV_THREADS);
            for (int64_t t = w.t0; t < w.t1; ++t, ++gtile) {
                const uint32_t s = gtile % T2_PST;
                const bool ok = t * T2_NP + col < a.n;
                mbar_wait(&rfull[rs], rph);
                const float* X = sRaw + (size_t)rs * T2_MAXD * T2_NP + 16 * h * T2_NP + col;
                const float* zh = zs + 16 * h;
                float2 av[8];
                float mx = 0.0f;
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    if (8 * (2 * h + c) < d) {
                        const float4 z0 = *reinterpret_cast<const float4*>(zh + 8 * c);
                        const float4 z1 = *reinterpret_cast<const float4*>(zh + 8 * c + 4);
                        const float2 nz[4] = {make_float2(-z0.x, -z0.y), make_float2(-z0.z, -z0.w),
                                              make_float2(-z1.x, -z1.y), make_float2(-z1.z, -z1.w)};
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float2 xv = make_float2(X[(8 * c + 2 * e) * T2_NP], X[(8 * c + 2 * e + 1) * T2_NP]);
                            const float2 v = __fadd2_rn(xv, nz[e]);
                            av[4 * c + e] = v;
                            mx = fmaxf(mx, fmaxf(fabsf(v.x), fabsf(v.y)));
                        }
                    } else {
#pragma unroll
                        for (int e = 0; e < 4; ++e) av[4 * c + e] = make_float2(0.0f, 0.0f);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&rempty[rs]);
                if (++rs == (uint32_t)RS) {
                    rs = 0;
                    rph ^= 1u;
                }
                float* mxs = sMx + (gtile & 1u) * 4 * T2_NH;
                mxs[h * T2_NH + r] = mx;
                bar_sync(2, T2_CONV_THREADS);
                mx = fmaxf(fmaxf(mxs[r], mxs[T2_NH + r]), fmaxf(mxs[2 * T2_NH + r], mxs[3 * T2_NH + r]));
                const uint32_t slot = gtile & 7u;
                const uint32_t exw = __ballot_sync(0xffffffffu, !ok || mx == 0.0f);  // used by h == 0 warps
                float scale = 0.0f;
                if (mx > 0.0f) {
                    int E = (int)((__float_as_uint(mx) >> 23) & 0xFF) - 126;
                    if (E < -100) E = -100;
                    scale = __uint_as_float((uint32_t)(127 + 14 - E) << 23);
                }
                if (gtile >= T2_PST) mbar_wait(&pempty[s], ((gtile / T2_PST) - 1) & 1u);
                unsigned char* P = sP + s * stage_bytes + r * 16;
                const float2 sc2 = make_float2(scale, scale);
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const int cc = 2 * h + c;
                    if (8 * cc >= d) continue;
                    uint32_t hw[4], lw[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float2 v = __fmul2_rn(av[4 * c + e], sc2);
                        const __half2 hh = __floats2half2_rn(v.x, v.y);
                        const float2 hf = __half22float2(hh);
                        const float2 res = __fadd2_rn(v, make_float2(-hf.x, -hf.y));
                        hw[e] = *reinterpret_cast<const uint32_t*>(&hh);
                        const __half2 ll = __floats2half2_rn(res.x, res.y);
                        lw[e] = *reinterpret_cast<const uint32_t*>(&ll);
                    }
                    if (cc < main_chunks) {
                        const uint4 hv = make_uint4(hw[0], hw[1], hw[2], hw[3]);
                        *reinterpret_cast<uint4*>(P + cc * (T2_NH * 16)) = hv;
                        *reinterpret_cast<uint4*>(P + (main_chunks + cc) * (T2_NH * 16)) =
                            make_uint4(lw[0], lw[1], lw[2], lw[3]);
                        *reinterpret_cast<uint4*>(P + (2 * main_chunks + cc) * (T2_NH * 16)) = hv;
                    } else {
#pragma unroll 1
                        for (int e = 0; e < 8; ++e) {
                            const int cd = 8 * cc + e;
                            if (cd >= d) break;
                            const int wi = e >> 1;
                            const uint32_t hv = wi == 0 ? hw[0] : wi == 1 ? hw[1] : wi == 2 ? hw[2] : hw[3];
                            const uint32_t lv = wi == 0 ? lw[0] : wi == 1 ? lw[1] : wi == 2 ? lw[2] : lw[3];
                            const uint16_t hb = (uint16_t)((e & 1) ? (hv >> 16) : (hv & 0xFFFFu));
                            const uint16_t lb = (uint16_t)((e & 1) ? (lv >> 16) : (lv & 0xFFFFu));
                            int kk = 32 * L.q16 + cd;
#pragma unroll
                            for (int pr = 0; pr < 3; ++pr, kk += L.rem)
                                *reinterpret_cast<uint16_t*>(P + (kk >> 3) * (T2_NH * 16) + (kk & 7) * 2) =
                                    pr == 1 ? lb : hb;
                        }
                    }
                }
                fence_proxy_async();
                __syncwarp();
                if (lane == 0) {
                    // the leader's pfull[s]: CTA scope for the leader's own converters (its MMA
                    // thread acquires it locally), cluster scope from the peer
                    if (rank == 0) mbar_arrive(&pfull[s]);
                    else arrive_cluster(pfull0 + s * 8u);
                }
                if (h == 0 && lane == 0) {
                    // excluded points (coinciding or past n), word rank * 2 + warp of this half
                    // tile, published in both CTAs for the epilogues (release at cluster scope)
                    const int wi = (int)rank * 2 + (r >> 5);
                    sExcl[slot * 4 + wi] = exw;
                    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(map_to(smem_u32(&sExcl[slot * 4 + wi]), peer)),
                                 "r"(exw)
                                 : "memory");
                    mbar_arrive(&xfull[slot]);
                    arrive_cluster(map_to(smem_u32(&xfull[slot]), peer));
                }
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue
        const int ct = tid - T2_EPI_WARP0 * 32;
        const int quarter = warp & 3;
        const int half = (warp - T2_EPI_WARP0) >> 2;
        const uint32_t lane_base = (uint32_t)(32 * quarter) << 16;
        const uint32_t tempty0 = map_to(smem_u32(tempty), 0);
        uint32_t it = 0, gacc = 0, gtile = 0;
        for (int64_t u = u0; u < units; u += ustride, ++it) {
            const T2Unit w = t2_unit(a, u);
            uint32_t cnt[T2_GB_MAX];
#pragma unroll
            for (int b = 0; b < T2_GB_MAX; ++b) cnt[b] = 0u;
            uint32_t zsum = 0;  // coinciding rows (x - z == 0) of the unit's tiles
            for (int64_t t = w.t0; t < w.t1; ++t, ++gtile) {
                uint32_t keep0 = 0u, keep1 = 0u;
#pragma unroll
                for (int p = 0; p < T2_GB_MAX; ++p) {
                    if (p < w.npg) {
                        const uint32_t buf = gacc & 1u;
                        mbar_wait(&tfull[buf], (gacc >> 1) & 1u);
                        ++gacc;
                        fence_after2();
                        if (p == 0) {
                            // both CTAs' exclusion words of this tile (slot ring of 8; the
                            // converters are < 8 tiles ahead of the epilogue)
                            wait_cluster(&xfull[gtile & 7u], (gtile >> 3) & 1u);
                            const uint32_t* ex = sExcl + (gtile & 7u) * 4;
                            keep0 = ~ex[2 * half];
                            keep1 = ~ex[2 * half + 1];
                            // excluded = coinciding or past n: coinciding = excluded - padding
                            const int64_t pad = (t + 1) * T2_NP - a.n;
                            zsum += (uint32_t)(__popc(ex[0]) + __popc(ex[1]) + __popc(ex[2]) + __popc(ex[3])) -
                                    (uint32_t)(pad > 0 ? pad : 0);
                        }
                        const uint32_t tb = lane_base + buf * T2_ACC + (uint32_t)(half * 64);
                        uint32_t y0[32], y1[32];
                        tmem_ld32x(tb, y0);
                        tmem_ld32x(tb + 32, y1);
                        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                        fence_before2();
                        __syncwarp();
                        if (lane == 0) {
                            if (rank == 0) mbar_arrive(&tempty[buf]);
                            else arrive_cluster_relaxed(tempty0 + buf * 8u);
                        }
                        uint32_t m0 = 0u, m1 = 0u;
#pragma unroll
                        for (int j = 31; j >= 0; --j) {
                            m0 = __funnelshift_l(y0[j], m0, 1);
                            m1 = __funnelshift_l(y1[j], m1, 1);
                        }
                        cnt[p] += __popc(m0 & keep0) + __popc(m1 & keep1);
                    }
                }
            }
#pragma unroll
            for (int p = 0; p < T2_GB_MAX; ++p)
                if (p < w.npg) atomicAdd(sCnt + p * T2_MD + 32 * quarter + lane, cnt[p]);
            bar_sync(1, T2_EPI_THREADS);
            const int64_t r1 = w.t1 * T2_NP < a.n ? w.t1 * T2_NP : a.n;
            const int valid = (int)(r1 - w.t0 * T2_NP);
            int* dst = a.counts + (size_t)w.q * a.mpad * 2;
            for (int c = ct; c < w.npg * T2_MD; c += T2_EPI_THREADS) {
                const int lt = (int)sCnt[c];
                sCnt[c] = 0u;
                const int p = c / T2_MD;
                const int blk = 2 * (w.grp * a.gb + p) + (int)rank;
                const int j = blk * T2_MD + (c % T2_MD);
                if (blk >= a.NB || j >= a.m) continue;
                // #(y>0) = valid rows - coinciding rows - #(y<0)
                const int gtv = valid - (int)zsum - lt;
                if (lt) atomicAdd(dst + 2 * j + 0, lt);
                if (gtv) atomicAdd(dst + 2 * j + 1, gtv);
            }
            bar_sync(1, T2_EPI_THREADS);
        }
    }

    fence_before2();
    __syncthreads();
    cluster_sync();  // the peer may still arrive on / read from this CTA until here
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(0u), "r"(T2_TMEM_COLS));
}

}  // namespace rrs

namespace rrs {

cudaError_t launch_contract_tc2(TcArgs a, int sms, cudaStream_t st) {
    const TcLayout L = tc_layout(a.d);
    if (a.d > T2_MAXD || a.d < 1 || L.ns > T2_MAXNS) return cudaErrorInvalidValue;
    int gb = (int)(256 / (8 * L.ns));  // blocks resident per CTA = block pairs per unit
    if (gb > T2_GB_MAX) gb = T2_GB_MAX;
    a.gb = gb;
    const int npairs = (a.NB + 1) / 2;
    a.groups = (npairs + gb - 1) / gb;
    const int clusters = sms / 2;
    const int64_t base = (int64_t)a.Qb * a.groups;
    int64_t chunks = (16LL * clusters + base - 1) / base;
    if (chunks < 1) chunks = 1;
    if (chunks > a.tiles) chunks = a.tiles;
    a.tiles_per_chunk = (a.tiles + chunks - 1) / chunks;
    a.chunks = (int)((a.tiles + a.tiles_per_chunk - 1) / a.tiles_per_chunk);
    const T2Smem lay(L.ns, a.d);
    a.raw_stages = lay.raw_stages;
    if (a.raw_stages < 2) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(contract_tc2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, lay.total);
    if (e != cudaSuccess) return e;
    const int64_t units = (int64_t)a.Qb * a.groups * a.chunks;
    if (units == 0) return cudaSuccess;
    const int ncl = (int)(units < clusters ? units : clusters);
    contract_tc2_kernel<<<2 * ncl, T2_THREADS, lay.total, st>>>(a);
    return cudaGetLastError();
}

}  // namespace rrs
