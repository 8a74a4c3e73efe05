// contract_tc.cu -- K2 on the 5th-generation tensor cores: split-precision
// (FP16 hi/lo, FP32-accumulate) contraction with a fused halfspace-count
// epilogue.
//
// Same result contract as the FFMA kernel (contract.cu): per (query, direction)
// the counts #(y<0), #(y>0) of y_i = <u, x_i - z> over all points; the query's
// own row gives y = 0 exactly (self-tie by construction: a = x - z = 0, every
// product is a signed zero and y < 0 is false) and exact zeros count on both
// sides (#<= = n - #>0, #>= = n - #<0).
//
// Operands ("two-term FP16 split", FP32-class accuracy):
//   a_il = x_il - z_l (FP32, as in contract.cu), scaled per point by the power
//          of two s_i = 2^(14 - E_i) with max_l |a_il| < 2^E_i (never changes a
//          sign); a*s = ah + al, ah = fp16(a*s), al = fp16(a*s - ah): 22 bits;
//   u_jl * 2^15 = uh + ul likewise (from the FP64 direction).
//   y_ij * s_i * 2^15 ~= sum_l (uh*al + ul*ah + uh*ah)   (ul*al, ~2^-22, dropped)
// Each FP16 product is exact in FP32 and the tensor core accumulates in FP32;
// the dropped term and the split residuals are ~2^-22 |u_l a_l|, the same order
// as the FFMA kernel's own roundings.  Validated by tests/test_gpu_parity.py
// (tier 1 at the config-4 shape: no count differs outside the 1e-6 tie zone).
// A bit-exact int8-limb variant (four accumulator levels) needs 4x the TMEM
// columns per point and therefore N = 48 MMAs, which sit on the ~54-clock
// per-instruction floor of tcgen05.mma (profiles/r1/tcgen05_mma_floor_*.txt);
// this kernel runs N = 128 MMAs at the full 64-clock rate.
//
// Layout (M = 128 DIRECTIONS on TMEM lanes, N = 128 POINTS, K = 16 per MMA):
//   TMEM columns [0,128) and [128,256): two FP32 accumulator buffers;
//   TMEM columns [256 + 64 b, 256 + 64 b + 64): direction block b of the
//   current unit (hi at +0, lo at +32; 16 K values = 8 columns per MMA),
//   resident for the whole unit (TS MMA: A from TMEM, B from shared memory).
// Work unit = (query, group of <= 4 direction blocks = 512 directions, chunk of
// 128-point tiles); persistent CTAs (one per SM) stride over units.
//   warp 0      producer: TMA of the unit's direction blocks (32 KB each, two at
//               a time) into a staging area (cp.async.bulk + mbarrier);
//   warp 1      TMEM allocator + tcgen05 issuer: staging -> TMEM (tcgen05.cp)
//               once per unit, then per tile and block 3*ceil(d/16) MMAs;
//   warp 2      producer: TMA of each raw FP32 point tile (d*512 bytes, the
//               tile-blocked dataset) into a 2-4 stage ring;
//   warps 3-10  converters: one (point, half of K) per thread: x - z from the
//               staged tile, per-point power-of-two scale (max exchanged through
//               shared memory), FP16 hi/lo split into the double-buffered
//               point operand;
//   warps 11-18 epilogue: tcgen05.ld of the accumulator (64 columns per thread),
//               y < 0 counted per direction in registers, flushed per unit.
// Replaces _kernels.pyx:120-199 (projection) + 270-289 (halfspace_span).
#include "common.cuh"
#include "kernels.h"

#include <cuda_fp16.h>

namespace rrs {

constexpr int TC_CONV_WARP0 = 3;                 // first converter warp
constexpr int TC_CONV_WARPS = 8;                 // (point, K half) per thread
constexpr int TC_CONV_THREADS = TC_CONV_WARPS * 32;
constexpr int TC_EPI_WARP0 = TC_CONV_WARP0 + TC_CONV_WARPS;  // first epilogue warp
constexpr int TC_EPI_WARPS = 8;                  // 4 lane quarters x 2 column halves
constexpr int TC_EPI_THREADS = TC_EPI_WARPS * 32;
constexpr int TC_THREADS = (TC_EPI_WARP0 + TC_EPI_WARPS) * 32;  // 608
constexpr int TC_KP = 64;                        // K padded (d <= 64)
constexpr int TC_MD = 128;                       // directions per block (MMA M)
constexpr int TC_NP = 128;                       // points per tile (MMA N)
constexpr int TC_GB = 4;                         // direction blocks resident per unit
constexpr int TC_DPH = 2;                        // direction blocks per staging phase
constexpr int P_SPLIT_BYTES = TC_NP * TC_KP * 2;  // 16 KB: one FP16 split of a tile
constexpr int P_STAGE_BYTES = 2 * P_SPLIT_BYTES;  // 32 KB: hi + lo
constexpr int P_STAGES = 2;
constexpr int R_MAX_STAGES = 4;                   // raw FP32 tile ring (runtime depth)
constexpr int D_SPLIT_BYTES = TC_MD * TC_KP * 2;  // 16 KB
constexpr int D_BLOCK_BYTES = 2 * D_SPLIT_BYTES;  // 32 KB (= TC_DIR_BLOCK_BYTES)
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t ACC_COLS = TC_NP;              // 128 per accumulator buffer
constexpr uint32_t A_TMEM = 2 * ACC_COLS;         // 256: direction blocks (64 columns each)
static_assert(A_TMEM + TC_GB * 64 <= TMEM_COLS, "TMEM budget");
static_assert(D_BLOCK_BYTES == TC_DIR_BLOCK_BYTES, "direction operand block size");
constexpr int TC_SMEM_LIMIT = 227 * 1024;

struct TcSmem {
    // offsets in bytes from a 1024-aligned base
    static constexpr int P = 0;                                    // point operand stages
    static constexpr int D = P + P_STAGES * P_STAGE_BYTES;         // direction staging, TC_DPH blocks
    static constexpr int CNT = D + TC_DPH * D_BLOCK_BYTES;         // uint32 [TC_GB * 128]
    static constexpr int ZS = CNT + TC_GB * TC_MD * 4;             // float [2][TC_KP] staged queries
    static constexpr int SMX = ZS + 2 * TC_KP * 4;                 // float [2][2][128] partial |a| maxima
    static constexpr int EXCL = SMX + 2 * 2 * TC_NP * 4;           // uint32 [8][4] excluded-point masks per tile
    static constexpr int ZROWS = EXCL + 8 * 4 * 4;                 // uint32 [4] coinciding rows per unit slot
    static constexpr int BARS = ZROWS + 16;                        // mbarriers
    static constexpr int NBARS = 2 * P_STAGES + 2 + 2 + 3 + 2 * R_MAX_STAGES;
    static constexpr int TADDR = BARS + NBARS * 8;
    static constexpr int RAW = (TADDR + 16 + 1023) & ~1023;        // raw tiles, runtime d*512 bytes each
};

int contract_tc_raw_stages(int d) {
    const int room = TC_SMEM_LIMIT - 1024 - TcSmem::RAW;
    int st = room / (d * TC_NP * 4);
    return st > R_MAX_STAGES ? R_MAX_STAGES : st;
}

size_t contract_tc_smem_bytes(int d) {
    return (size_t)TcSmem::RAW + (size_t)contract_tc_raw_stages(d) * d * TC_NP * 4 + 1024;
}

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    // tcgen05 shared-memory descriptor: start>>4 [0,14), LBO>>4 [16,30),
    // SBO>>4 [32,46), version 1 [46,48), base offset 0, layout SWIZZLE_NONE
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

// One (point tile, direction block) product: per K step of 16,
//   D (+)= Ah*Bl, D += Al*Bh, D += Ah*Bh      (small terms first)
// then the commit to the accumulator-full barrier, all under one elect with
// immediate operand offsets (ptxas keeps it on the uniform datapath).
//   acc: accumulator columns; aT: block's hi columns (lo at +32, K step at +8)
//   bd : descriptor of the tile's hi split, K step 0 (K step +256, lo +1024)
#define RRS_MMA3(KS, BH, BL, FIRSTP)                                                             \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1+" KS "], " BL ", %3, " FIRSTP ";\n"         \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1+32+" KS "], " BH ", %3, 1;\n"                \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1+" KS "], " BH ", %3, 1;\n"

template <int NKS>
__device__ __forceinline__ void mma_tile_block(uint32_t acc, uint32_t aT, uint64_t bd, uint32_t idesc,
                                               uint32_t bar) {
    static_assert(NKS >= 1 && NKS <= 4, "K steps");
    if constexpr (NKS == 1) {
        asm volatile("{\n.reg .pred e;\n.reg .b64 l0;\nelect.sync _|e, 0xffffffff;\n"
                     "add.s64 l0, %2, 1024;\n"
                     RRS_MMA3("0", "%2", "l0", "0")
                     "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%4];\n}\n"
                     ::"r"(acc), "r"(aT), "l"(bd), "r"(idesc), "r"(bar) : "memory");
    } else if constexpr (NKS == 2) {
        asm volatile("{\n.reg .pred e;\n.reg .b64 l0, h1, l1;\nelect.sync _|e, 0xffffffff;\n"
                     "add.s64 l0, %2, 1024;\nadd.s64 h1, %2, 256;\nadd.s64 l1, %2, 1280;\n"
                     RRS_MMA3("0", "%2", "l0", "0") RRS_MMA3("8", "h1", "l1", "1")
                     "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%4];\n}\n"
                     ::"r"(acc), "r"(aT), "l"(bd), "r"(idesc), "r"(bar) : "memory");
    } else if constexpr (NKS == 3) {
        asm volatile("{\n.reg .pred e;\n.reg .b64 l0, h1, l1, h2, l2;\nelect.sync _|e, 0xffffffff;\n"
                     "add.s64 l0, %2, 1024;\nadd.s64 h1, %2, 256;\nadd.s64 l1, %2, 1280;\n"
                     "add.s64 h2, %2, 512;\nadd.s64 l2, %2, 1536;\n"
                     RRS_MMA3("0", "%2", "l0", "0") RRS_MMA3("8", "h1", "l1", "1") RRS_MMA3("16", "h2", "l2", "1")
                     "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%4];\n}\n"
                     ::"r"(acc), "r"(aT), "l"(bd), "r"(idesc), "r"(bar) : "memory");
    } else {
        asm volatile("{\n.reg .pred e;\n.reg .b64 l0, h1, l1, h2, l2, h3, l3;\nelect.sync _|e, 0xffffffff;\n"
                     "add.s64 l0, %2, 1024;\nadd.s64 h1, %2, 256;\nadd.s64 l1, %2, 1280;\n"
                     "add.s64 h2, %2, 512;\nadd.s64 l2, %2, 1536;\nadd.s64 h3, %2, 768;\nadd.s64 l3, %2, 1792;\n"
                     RRS_MMA3("0", "%2", "l0", "0") RRS_MMA3("8", "h1", "l1", "1") RRS_MMA3("16", "h2", "l2", "1")
                     RRS_MMA3("24", "h3", "l3", "1")
                     "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%4];\n}\n"
                     ::"r"(acc), "r"(aT), "l"(bd), "r"(idesc), "r"(bar) : "memory");
    }
}
#undef RRS_MMA3

// Direction block b of the staging area (canonical K-major: [split][k chunk 8]
// [direction 128][16 B]) -> TMEM columns [aT, aT + 64): eight 128x256b copies.
__device__ __forceinline__ void tmem_cp_dirblock(uint32_t aT, uint64_t sd) {
    // sd: descriptor of split 0, chunk 0; chunk pair +4096 B (256), split +16384 B (1024)
    asm volatile(
        "{\n.reg .pred e;\n.reg .b64 s1, s2, s3, s4, s5, s6, s7;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "add.s64 s1, %1, 256;\nadd.s64 s2, %1, 512;\nadd.s64 s3, %1, 768;\n"
        "add.s64 s4, %1, 1024;\nadd.s64 s5, %1, 1280;\nadd.s64 s6, %1, 1536;\nadd.s64 s7, %1, 1792;\n"
        "@e tcgen05.cp.cta_group::1.128x256b [%0], %1;\n"
        "@e tcgen05.cp.cta_group::1.128x256b [%0+8], s1;\n"
        "@e tcgen05.cp.cta_group::1.128x256b [%0+16], s2;\n"
        "@e tcgen05.cp.cta_group::1.128x256b [%0+24], s3;\n"
        "@e tcgen05.cp.cta_group::1.128x256b [%0+32], s4;\n"
        "@e tcgen05.cp.cta_group::1.128x256b [%0+40], s5;\n"
        "@e tcgen05.cp.cta_group::1.128x256b [%0+48], s6;\n"
        "@e tcgen05.cp.cta_group::1.128x256b [%0+56], s7;\n"
        "}\n" ::"r"(aT),
        "l"(sd));
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

struct TcUnit {
    int q, grp, nbg;     // query, direction group, blocks in the group
    int64_t t0, t1;      // point tiles [t0, t1)
};

__device__ __forceinline__ TcUnit tc_unit(const TcArgs& a, int64_t u) {
    TcUnit r;
    const int64_t per_q = (int64_t)a.groups * a.chunks;
    r.q = (int)(u / per_q);
    const int64_t rem = u - (int64_t)r.q * per_q;
    r.grp = (int)(rem / a.chunks);
    const int64_t c = rem - (int64_t)r.grp * a.chunks;
    r.nbg = a.NB - r.grp * TC_GB < TC_GB ? a.NB - r.grp * TC_GB : TC_GB;
    r.t0 = c * a.tiles_per_chunk;
    r.t1 = r.t0 + a.tiles_per_chunk < a.tiles ? r.t0 + a.tiles_per_chunk : a.tiles;
    return r;
}

template <int NKS>
__device__ __forceinline__ void mma_issue(const TcArgs& a, int64_t units, unsigned char* sP, unsigned char* sD,
                                          uint64_t* pfull, uint64_t* pempty, uint64_t* dfull, uint64_t* dempty,
                                          uint64_t* tfull, uint64_t* tempty, uint64_t* udone) {
    constexpr uint32_t tmem = 0u;
    // F32 accumulate, FP16 A and B, K-major both, N = 128, M = 128
    const uint32_t idesc = (1u << 4) | ((uint32_t)(TC_NP >> 3) << 17) | ((uint32_t)(TC_MD >> 4) << 24);
    uint32_t it = 0, gtile = 0, gacc = 0, gph = 0;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x, ++it) {
        const TcUnit w = tc_unit(a, u);
        const uint32_t dbase = smem_u32(sD);
        for (int b0 = 0; b0 < w.nbg; b0 += TC_DPH, ++gph) {
            mbar_wait_sleep(dfull, gph & 1u);
            if (b0 == 0 && it > 0) mbar_wait(udone, (it - 1) & 1u);  // previous unit no longer reads TMEM A
            tc_fence_after();
            for (int b = b0; b < w.nbg && b < b0 + TC_DPH; ++b)
                tmem_cp_dirblock(tmem + A_TMEM + 64u * b, umma_desc(dbase + (b - b0) * D_BLOCK_BYTES, 2048, 128));
            mma_commit_elect(dempty);  // staging free once the copies are done
        }
        for (int64_t t = w.t0; t < w.t1; ++t, ++gtile) {
            const uint32_t s = gtile % P_STAGES;
            mbar_wait(&pfull[s], (gtile / P_STAGES) & 1u);
            tc_fence_after();
            const uint64_t bd = umma_desc(smem_u32(sP) + s * P_STAGE_BYTES, 2048, 128);
            for (int b = 0; b < w.nbg; ++b, ++gacc) {
                const uint32_t buf = gacc & 1u;
                if (gacc >= 2) mbar_wait(&tempty[buf], ((gacc >> 1) - 1) & 1u);
                tc_fence_after();
                mma_tile_block<NKS>(tmem + buf * ACC_COLS, tmem + A_TMEM + 64u * b, bd, idesc,
                                    smem_u32(&tfull[buf]));
            }
            mma_commit_elect(&pempty[s]);  // point stage free once this tile's MMAs are done
        }
        mma_commit_elect(udone);
    }
}

__global__ void __launch_bounds__(TC_THREADS, 1) contract_tc_kernel(const TcArgs a) {
    extern __shared__ __align__(1024) unsigned char tc_raw[];
    // 1024-align by pointer arithmetic on the __shared__ array (keeps the address space)
    unsigned char* sm = tc_raw + ((1024u - (smem_u32(tc_raw) & 1023u)) & 1023u);
    unsigned char* sP = sm + TcSmem::P;
    unsigned char* sD = sm + TcSmem::D;
    uint32_t* sCnt = reinterpret_cast<uint32_t*>(sm + TcSmem::CNT);
    float* sZ = reinterpret_cast<float*>(sm + TcSmem::ZS);
    uint32_t* sZrows = reinterpret_cast<uint32_t*>(sm + TcSmem::ZROWS);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + TcSmem::BARS);
    uint64_t* pfull = &bars[0];                   // [P_STAGES] point tile converted (converter warps)
    uint64_t* pempty = &bars[P_STAGES];           // [P_STAGES] MMAs reading it completed
    uint64_t* tfull = &bars[2 * P_STAGES];        // [2] accumulator ready
    uint64_t* tempty = &bars[2 * P_STAGES + 2];   // [2] accumulator drained (epilogue warps)
    uint64_t* dfull = &bars[2 * P_STAGES + 4];    // direction staging phase loaded
    uint64_t* dempty = &bars[2 * P_STAGES + 5];   // direction staging copied to TMEM
    uint64_t* udone = &bars[2 * P_STAGES + 6];    // all MMAs of a unit completed
    uint64_t* rfull = &bars[2 * P_STAGES + 7];    // [R_MAX_STAGES] raw tile landed
    uint64_t* rempty = &bars[2 * P_STAGES + 7 + R_MAX_STAGES];  // [R_MAX_STAGES] raw tile read
    float* sMx = reinterpret_cast<float*>(sm + TcSmem::SMX);
    uint32_t* sExcl = reinterpret_cast<uint32_t*>(sm + TcSmem::EXCL);
    float* sRaw = reinterpret_cast<float*>(sm + TcSmem::RAW);
    const int RS = a.raw_stages;
    const uint32_t raw_bytes = (uint32_t)(a.d * TC_NP * 4);
    uint32_t* sTaddr = reinterpret_cast<uint32_t*>(sm + TcSmem::TADDR);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int d = a.d;
    const int64_t units = (int64_t)a.Qb * a.groups * a.chunks;

    for (int c = tid; c < TC_GB * TC_MD; c += TC_THREADS) sCnt[c] = 0u;
    if (tid < 4) sZrows[tid] = 0u;
    if (tid == 0) {
        for (int s = 0; s < P_STAGES; ++s) {
            mbar_init(&pfull[s], TC_CONV_WARPS);
            mbar_init(&pempty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], TC_EPI_WARPS);
        }
        mbar_init(dfull, 1);
        mbar_init(dempty, 1);
        mbar_init(udone, 1);
        for (int r = 0; r < R_MAX_STAGES; ++r) {
            mbar_init(&rfull[r], 1);
            mbar_init(&rempty[r], TC_CONV_WARPS);
        }
        fence_mbar_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(sTaddr)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    // The single 512-column allocation of the only CTA on the SM starts at
    // lane 0, column 0; the issuer relies on that constant so that every MMA
    // operand stays on the uniform datapath.
    if (*sTaddr != 0u) __trap();
    constexpr uint32_t tmem = 0u;

    if (warp == 0) {
        // ----------------------------- producer: unit direction blocks, 2 per phase
        uint32_t gph = 0;
        for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
            const TcUnit w = tc_unit(a, u);
            const unsigned char* src =
                a.uop + ((size_t)w.q * a.NB + (size_t)w.grp * TC_GB) * D_BLOCK_BYTES;
            for (int b0 = 0; b0 < w.nbg; b0 += TC_DPH, ++gph) {
                const int nb = w.nbg - b0 < TC_DPH ? w.nbg - b0 : TC_DPH;
                if (gph > 0) mbar_wait_sleep(dempty, (gph - 1) & 1u);
                expect_tx_elect(dfull, (uint32_t)(nb * D_BLOCK_BYTES));
                for (int b = 0; b < nb; ++b)
                    tma_load_elect(sD + b * D_BLOCK_BYTES, src + (size_t)(b0 + b) * D_BLOCK_BYTES, D_BLOCK_BYTES,
                                   dfull);
                __syncwarp();
            }
        }
    } else if (warp == 2) {
        // -------------------------------------- producer: raw FP32 point tiles
        uint32_t g = 0;
        for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
            const TcUnit w = tc_unit(a, u);
            for (int64_t t = w.t0; t < w.t1; ++t, ++g) {
                const uint32_t rs = g % RS;
                if (g >= (uint32_t)RS) mbar_wait_sleep(&rempty[rs], ((g / RS) - 1) & 1u);
                expect_tx_elect(&rfull[rs], raw_bytes);
                tma_load_elect(sRaw + (size_t)rs * d * TC_NP, a.xb + (size_t)t * d * TC_NP, raw_bytes, &rfull[rs]);
                __syncwarp();
            }
        }
    } else if (warp == 1) {
        // -------------------------------------------------------- MMA issuer
        switch ((d + 15) >> 4) {
            case 1: mma_issue<1>(a, units, sP, sD, pfull, pempty, dfull, dempty, tfull, tempty, udone); break;
            case 2: mma_issue<2>(a, units, sP, sD, pfull, pempty, dfull, dempty, tfull, tempty, udone); break;
            case 3: mma_issue<3>(a, units, sP, sD, pfull, pempty, dfull, dempty, tfull, tempty, udone); break;
            default: mma_issue<4>(a, units, sP, sD, pfull, pempty, dfull, dempty, tfull, tempty, udone); break;
        }
    } else if (warp < TC_EPI_WARP0) {
        // ----------------------- converters: x - z -> scale -> FP16 hi/lo split
        const int ct = tid - TC_CONV_WARP0 * 32;  // 0..255
        const int r = ct & (TC_NP - 1);           // point of the tile
        const int h = ct >> 7;                    // K half: coordinates [32 h, 32 h + 32)
        uint32_t it = 0, gtile = 0;
        for (int64_t u = blockIdx.x; u < units; u += gridDim.x, ++it) {
            const TcUnit w = tc_unit(a, u);
            float* zs = sZ + (it & 1u) * TC_KP;
            if (ct < TC_KP) zs[ct] = ct < d ? __ldg(a.zq + (size_t)w.q * d + ct) : 0.0f;
            named_bar(2, TC_CONV_THREADS);  // zs ready; keeps the converter warps in step per unit
            uint32_t zcount = 0;
            for (int64_t t = w.t0; t < w.t1; ++t, ++gtile) {
                const uint32_t s = gtile % P_STAGES;
                const uint32_t rs = gtile % RS;
                const bool ok = t * TC_NP + r < a.n;
                mbar_wait(&rfull[rs], (gtile / RS) & 1u);
                // staged tile [d][128]: lane-consecutive points, conflict-free
                const float* X = sRaw + (size_t)rs * d * TC_NP + r;
                float av[32];
                float mx = 0.0f;
#pragma unroll
                for (int k = 0; k < 32; k += 4) {
                    const float4 z4 = *reinterpret_cast<const float4*>(zs + 32 * h + k);
                    const float zz[4] = {z4.x, z4.y, z4.z, z4.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int kk = 32 * h + k + e;
                        av[k + e] = (ok && kk < d) ? (X[kk * TC_NP] - zz[e]) : 0.0f;
                        mx = fmaxf(mx, fabsf(av[k + e]));
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&rempty[rs]);  // raw tile consumed (loads ordered by release)
                float* mxs = sMx + (gtile & 1u) * 2 * TC_NP;
                mxs[h * TC_NP + r] = mx;
                named_bar(2, TC_CONV_THREADS);  // both K halves' maxima visible
                mx = fmaxf(mxs[r], mxs[TC_NP + r]);
                if (h == 0) {
                    // points the epilogue must not count: coinciding rows (every product a
                    // signed zero, ties on both sides) and rows beyond n
                    zcount += (ok && mx == 0.0f) ? 1u : 0u;
                    const uint32_t ex = __ballot_sync(0xffffffffu, !ok || mx == 0.0f);
                    if (lane == 0) sExcl[(gtile & 7u) * 4 + (r >> 5)] = ex;
                }
                float scale = 0.0f;
                if (mx > 0.0f) {
                    int E = (int)((__float_as_uint(mx) >> 23) & 0xFF) - 126;  // mx < 2^E
                    if (E < -100) E = -100;
                    scale = __uint_as_float((uint32_t)(127 + 14 - E) << 23);  // 2^(14-E)
                }
                if (gtile >= P_STAGES) mbar_wait(&pempty[s], ((gtile / P_STAGES) - 1) & 1u);
                // canonical K-major, no swizzle: [split][k chunk c (8 values)][point r][16 bytes]
                unsigned char* P = sP + s * P_STAGE_BYTES + r * 16;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint32_t hw[4], lw[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float v0 = av[c * 8 + 2 * e] * scale, v1 = av[c * 8 + 2 * e + 1] * scale;
                        const __half2 hh = __floats2half2_rn(v0, v1);
                        const float2 hf = __half22float2(hh);
                        hw[e] = *reinterpret_cast<const uint32_t*>(&hh);
                        lw[e] = pack_half2(v0 - hf.x, v1 - hf.y);
                    }
                    const int cc = 4 * h + c;
                    *reinterpret_cast<uint4*>(P + cc * (TC_NP * 16)) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
                    *reinterpret_cast<uint4*>(P + P_SPLIT_BYTES + cc * (TC_NP * 16)) =
                        make_uint4(lw[0], lw[1], lw[2], lw[3]);
                }
                fence_proxy_async();  // generic-proxy smem writes -> tensor-core reads
                __syncwarp();
                if (lane == 0) mbar_arrive(&pfull[s]);
            }
            // coinciding rows (x - z == 0) of this unit: ties on both sides
            zcount = __reduce_add_sync(0xffffffffu, zcount);
            if (lane == 0 && zcount) atomicAdd(&sZrows[it & 3u], zcount);
        }
    } else {
        // ------------------------------------------------------------ epilogue
        const int ct = tid - TC_EPI_WARP0 * 32;        // 0..255
        const int quarter = warp & 3;                  // TMEM lane quarter = 32 directions
        const int half = (warp - TC_EPI_WARP0) >> 2;   // 64-point half of the tile
        const uint32_t lane_base = (uint32_t)(32 * quarter) << 16;
        uint32_t it = 0, gacc = 0, gtile = 0;
        for (int64_t u = blockIdx.x; u < units; u += gridDim.x, ++it) {
            const TcUnit w = tc_unit(a, u);
            uint32_t cnt[TC_GB] = {0u, 0u, 0u, 0u};  // #(y<0) per resident block
            for (int64_t t = w.t0; t < w.t1; ++t, ++gtile) {
                uint32_t keep0 = 0u, keep1 = 0u;
#pragma unroll
                for (int b = 0; b < TC_GB; ++b) {
                    if (b < w.nbg) {
                        const uint32_t buf = gacc & 1u;
                        mbar_wait(&tfull[buf], (gacc >> 1) & 1u);
                        ++gacc;
                        tc_fence_after();
                        if (b == 0) {
                            // excluded points of this tile (written by the converters before the
                            // tile's pfull; ordered through pfull -> MMA -> tfull), bit j = point
                            // half*64 + 32 i + j
                            keep0 = ~sExcl[(gtile & 7u) * 4 + 2 * half];
                            keep1 = ~sExcl[(gtile & 7u) * 4 + 2 * half + 1];
                        }
                        const uint32_t tb = tmem + lane_base + buf * ACC_COLS + (uint32_t)(half * 64);
                        uint32_t y0[32], y1[32];
                        tmem_ld32(tb, y0);
                        tmem_ld32(tb + 32, y1);
                        tmem_wait_ld();
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&tempty[buf]);  // accumulator consumed
                        // sign bits -> 32-bit masks (one funnel shift per element), bit j = point j;
                        // y < 0 <=> sign bit set, except the signed zeros of excluded points
                        uint32_t m0 = 0u, m1 = 0u;
#pragma unroll
                        for (int j = 31; j >= 0; --j) {
                            m0 = __funnelshift_l(y0[j], m0, 1);
                            m1 = __funnelshift_l(y1[j], m1, 1);
                        }
                        cnt[b] += __popc(m0 & keep0) + __popc(m1 & keep1);
                    }
                }
            }
#pragma unroll
            for (int b = 0; b < TC_GB; ++b)
                if (b < w.nbg) atomicAdd(sCnt + b * TC_MD + 32 * quarter + lane, cnt[b]);
            named_bar(1, TC_EPI_THREADS);  // all direction counts of this unit are in
            // #(y>0) = real rows - coinciding rows - #(y<0); an exact zero from a
            // non-coinciding row (|y| below the rounding error, inside the tie
            // zone) lands on the positive side
            const int64_t r1 = w.t1 * TC_NP < a.n ? w.t1 * TC_NP : a.n;
            const int valid = (int)(r1 - w.t0 * TC_NP);
            const int zrows = (int)sZrows[it & 3u];
            int* dst = a.counts + (size_t)w.q * a.mpad * 2;
            const int j0 = w.grp * TC_GB * TC_MD;
            for (int c = ct; c < w.nbg * TC_MD; c += TC_EPI_THREADS) {
                const int lt = (int)sCnt[c];
                sCnt[c] = 0u;
                if (j0 + c >= a.m) continue;
                const int gtv = valid - zrows - lt;
                if (lt) atomicAdd(dst + 2 * (j0 + c) + 0, lt);
                if (gtv) atomicAdd(dst + 2 * (j0 + c) + 1, gtv);
            }
            named_bar(1, TC_EPI_THREADS);
            if (ct == 0) sZrows[it & 3u] = 0u;
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}

void plan_contract_tc(TcArgs& a, int sms) {
    a.groups = (a.NB + TC_GB - 1) / TC_GB;
    // split the point tiles into chunks so that every SM gets >= ~16 units
    const int64_t base = (int64_t)a.Qb * a.groups;
    int64_t chunks = (16LL * sms + base - 1) / base;
    if (chunks < 1) chunks = 1;
    if (chunks > a.tiles) chunks = a.tiles;
    a.tiles_per_chunk = (a.tiles + chunks - 1) / chunks;
    a.chunks = (int)((a.tiles + a.tiles_per_chunk - 1) / a.tiles_per_chunk);
}

cudaError_t launch_contract_tc(TcArgs a, int sms, cudaStream_t st) {
    if (a.d > TC_KP || a.d < 1) return cudaErrorInvalidValue;
    plan_contract_tc(a, sms);
    a.raw_stages = contract_tc_raw_stages(a.d);
    if (a.raw_stages < 2) return cudaErrorInvalidValue;
    const size_t smem = contract_tc_smem_bytes(a.d);
    cudaError_t e =
        cudaFuncSetAttribute(contract_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t units = (int64_t)a.Qb * a.groups * a.chunks;
    if (units == 0) return cudaSuccess;
    const int grid = (int)(units < sms ? units : sms);
    contract_tc_kernel<<<grid, TC_THREADS, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace rrs
