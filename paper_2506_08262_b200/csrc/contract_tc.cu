// contract_tc.cu -- K2 on the 5th-generation tensor cores: exact-integer
// (int8-limb, Ozaki-style) contraction with a fused halfspace-count epilogue.
//
// Same result contract as the FFMA kernel (contract.cu): per (query, direction)
// the counts #(y<0), #(y>0) of y_i = <u, x_i - z> over all points; the query's
// own row gives y = 0 exactly (self-tie by construction) and exact zeros count
// on both sides (#<= = n - #>0, #>= = n - #<0).  Here the sign of y is EXACT
// for fixed-point operands:
//   a_il = x_il - z_l (FP32), scaled per point by a power of two so that
//          |A_il| < 2^22 (A = rint(a * 2^(22-E_i)), E_i = exponent of max_l |a_il|);
//   U_jl = rint(u_jl * 2^22) (|u| <= 1);
//   both split into three signed int8 limbs  V = v2*2^16 + v1*2^8 + v0;
//   sum_l U_jl A_il = 2^32 S22 + 2^24 S21 + 2^16 S20 + (low products, dropped)
// with S22 = u2.a2, S21 = u2.a1 + u1.a2, S20 = u2.a0 + u1.a1 + u0.a2 accumulated
// by tcgen05.mma kind::i8 in int32 TMEM (exact).  The dropped products are
// of the same order as the quantisation (each <= 2^-22 of the operands' scale,
// an FP32-comparable error, validated by the tier-1 tests); the per-point power of two never
// changes a sign, so the epilogue needs no scale: sign(y) = sign(S22*2^16 +
// S21*2^8 + S20), evaluated exactly in 32 bits as the sign of
// (S22*2^8 + S21)*2^7 + floor(S20/2) (4 instructions per element).  Only
// #(y<0) is counted per element; #(y>0) = rows - coinciding rows - #(y<0).
//
// MMA orientation: M = 128 DIRECTIONS (TMEM lanes), N = 64 POINTS per
// instruction, K = 32.  Each epilogue thread owns one direction and counts its
// signs in registers (7 instructions per element, no cross-lane reduction).
//
// Persistent CTA (one per SM), 20 warps, work item = (query, 256 points):
//   warp 0      TMA producer: direction blocks (24 KB int8 limbs, 3-stage ring)
//               via cp.async.bulk + mbarriers, running ahead across items;
//   warps 2-3   converters: x - z (read from L2) and per-point quantisation
//               into a double-buffered point operand, one item ahead of the MMA;
//   warp 1      TMEM allocator + single-thread tcgen05 issuer: each direction
//               block is copied smem -> TMEM (tcgen05.cp) and used as the
//               TMEM-resident A operand ("TS" MMA), so the tensor core only
//               reads the point operand from shared memory;
//   warps 4-19  epilogue of every (direction block, 64-point group):
//               tcgen05.ld of the three accumulators, exact sign, per-thread
//               counts, one shared atomic per direction; TMEM double-buffered
//               against the MMA.
// Replaces _kernels.pyx:120-199 (projection) + 270-289 (halfspace_span).
#include "common.cuh"
#include "kernels.h"

namespace rrs {

constexpr int TC_THREADS = 640;                 // 4 role warps + 16 epilogue warps
constexpr int TC_EPI_WARPS = 16;
constexpr int TC_EPI_THREADS = TC_EPI_WARPS * 32;
constexpr int TC_CONV_THREADS = 64;             // warps 2-3 quantise the point operand
constexpr int TC_KP = 64;                       // K padded (d <= 64)
constexpr int TC_MD = 128;                      // directions per block (MMA M)
constexpr int TC_NP = 64;                       // points per MMA (MMA N)
constexpr int TC_PTS = 256;                     // points per work item (2 tiles)
constexpr int P_LIMB_BYTES = TC_PTS * TC_KP;    // 16 KB per limb
constexpr int P_BUF_BYTES = 3 * P_LIMB_BYTES;   // 48 KB per point operand
constexpr int D_LIMB_BYTES = TC_MD * TC_KP;     // 8 KB per limb
constexpr int D_BLOCK_BYTES = 3 * D_LIMB_BYTES; // 24 KB per direction block
constexpr int D_STAGES = 3;
constexpr int TC_MAX_DIRS = 4096;               // per-direction smem counters
constexpr uint32_t TMEM_COLS = 512;

struct TcSmem {
    // offsets in bytes from a 1024-aligned base
    static constexpr int P = 0;                                   // 2 x 48 KB point operands
    static constexpr int D = P + 2 * P_BUF_BYTES;                 // D_STAGES x 24 KB
    static constexpr int CNT = D + D_STAGES * D_BLOCK_BYTES;      // uint32 [TC_MAX_DIRS]
    static constexpr int ZROWS = CNT + TC_MAX_DIRS * 4;           // uint32 [4] coinciding rows per item slot
    static constexpr int BARS = ZROWS + 16;                       // mbarriers
    static constexpr int NBARS = 4 + 2 * D_STAGES + 4;
    static constexpr int TADDR = BARS + NBARS * 8;
    static constexpr int TOTAL = TADDR + 16;
};

size_t contract_tc_smem_bytes() { return TcSmem::TOTAL + 1024; }

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    // tcgen05 shared-memory descriptor: start>>4 [0,14), LBO>>4 [16,30),
    // SBO>>4 [32,46), version 1 [46,48), base offset 0, layout SWIZZLE_NONE
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// The issuing warps run their loops warp-wide (uniform operands, no waterfall)
// and one elected lane issues each tcgen05 / TMA instruction.
// A operand from TMEM ("TS"): [a_tmem] holds 128 lanes x K bytes, B from smem.
__device__ __forceinline__ void mma_i8_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred e, p;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// smem (canonical K-major, 128 rows x 32 bytes) -> TMEM (128 lanes x 8 columns)
__device__ __forceinline__ void tmem_cp_128x256b(uint32_t taddr, uint64_t sdesc) {
    asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.cp.cta_group::1.128x256b [%0], %1;\n}\n" ::"r"(
                     taddr),
                 "l"(sdesc));
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
        "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%3], %2;\n"
        "@e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n}\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Wait with a suspend-time hint: the waiting thread sleeps in hardware until the
// phase completes instead of spinning on issue slots shared with busy warps.
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

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
        "[%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void named_bar(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

__global__ void __launch_bounds__(TC_THREADS, 1) contract_tc_kernel(const TcArgs a) {
    extern __shared__ __align__(1024) unsigned char tc_raw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(tc_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    unsigned char* sP = sm + TcSmem::P;
    unsigned char* sD = sm + TcSmem::D;
    uint32_t* sCnt = reinterpret_cast<uint32_t*>(sm + TcSmem::CNT);
    uint32_t* sZrows = reinterpret_cast<uint32_t*>(sm + TcSmem::ZROWS);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + TcSmem::BARS);
    uint64_t* pfull = &bars[0];                  // [2] point operand quantised (2 converter warps)
    uint64_t* pempty = &bars[2];                 // [2] MMAs reading it completed
    uint64_t* dfull = &bars[4];                  // [D_STAGES]
    uint64_t* dempty = &bars[4 + D_STAGES];      // [D_STAGES]
    uint64_t* tfull = &bars[4 + 2 * D_STAGES];   // [2]
    uint64_t* tempty = &bars[6 + 2 * D_STAGES];  // [2]
    uint32_t* sTaddr = reinterpret_cast<uint32_t*>(sm + TcSmem::TADDR);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int d = a.d;
    const int MB = a.NB;                 // 128-direction blocks per query
    const int ndirs = MB * TC_MD;
    const int nks = (d + 31) / 32;       // MMA K-steps (1 or 2)
    const int64_t tiles2 = (a.tiles + 1) >> 1;
    const int64_t items = (int64_t)a.Qb * tiles2;

    for (int c = tid; c < ndirs; c += TC_THREADS) sCnt[c] = 0u;
    if (tid < 4) sZrows[tid] = 0u;
    if (tid == 0) {
        for (int b = 0; b < 2; ++b) {
            mbar_init(&pfull[b], 2);
            mbar_init(&pempty[b], 1);
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], TC_EPI_WARPS);
        }
        for (int b = 0; b < D_STAGES; ++b) {
            mbar_init(&dfull[b], 1);
            mbar_init(&dempty[b], 1);
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
    const uint32_t tmem = *sTaddr;

    if (warp == 0) {
        // ------------------------------------------- producer: direction blocks
        int64_t gd = 0;
        for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
            const int q = (int)(item / tiles2);
            const unsigned char* src = a.u8 + (size_t)q * MB * D_BLOCK_BYTES;
            for (int db = 0; db < MB; ++db, ++gd) {
                const int s = (int)(gd % D_STAGES);
                const int64_t u = gd / D_STAGES;
                if (u >= 1) mbar_wait_sleep(&dempty[s], (uint32_t)((u - 1) & 1));
                tma_load_elect(sD + s * D_BLOCK_BYTES, src + (size_t)db * D_BLOCK_BYTES, D_BLOCK_BYTES, &dfull[s]);
            }
            __syncwarp();
        }
    } else if (warp == 1) {
        // -------------------------------------------------------- MMA issuer
        // S32 accumulate, signed int8 A and B, K-major both, N = 64, M = 128
        const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(TC_NP >> 3) << 17) |
                               ((uint32_t)(TC_MD >> 4) << 24);
        // (direction limb, point limb, accumulator): S22 -> 2, S21 -> 1, S20 -> 0
        const int lu[6] = {2, 2, 1, 2, 1, 0};
        const int lp[6] = {2, 1, 2, 0, 1, 2};
        const int ac[6] = {2, 1, 1, 0, 0, 0};
        const int first[6] = {1, 1, 0, 1, 0, 0};
        int64_t gd = 0, gt = 0;
        int it = 0;
        for (int64_t item = blockIdx.x; item < items; item += gridDim.x, ++it) {
            const int pb = it & 1;
            mbar_wait_sleep(&pfull[pb], (uint32_t)((it >> 1) & 1));
            const uint32_t pBase = smem_u32(sP + pb * P_BUF_BYTES);
            for (int db = 0; db < MB; ++db, ++gd) {
                const int s = (int)(gd % D_STAGES);
                mbar_wait_sleep(&dfull[s], (uint32_t)((gd / D_STAGES) & 1));
                tc_fence_after();
                // direction block -> TMEM (A operand), double-buffered; in order with the MMAs
                const uint32_t dBase = smem_u32(sD + s * D_BLOCK_BYTES);
                const uint32_t aT = tmem + 384u + (uint32_t)(gd & 1) * 48u;
#pragma unroll
                for (int L = 0; L < 3; ++L)
#pragma unroll
                    for (int ks = 0; ks < 2; ++ks)
                        tmem_cp_128x256b(aT + (uint32_t)(L * 2 + ks) * 8u,
                                         umma_desc(dBase + L * D_LIMB_BYTES + ks * 2 * 2048, 2048, 128));
                mma_commit_elect(&dempty[s]);  // smem stage free once the copies are done
                for (int pq = 0; pq < TC_PTS / TC_NP; ++pq, ++gt) {
                    const int buf = (int)(gt & 1);
                    const int64_t ut = gt >> 1;
                    if (ut >= 1) mbar_wait(&tempty[buf], (uint32_t)((ut - 1) & 1));
                    tc_fence_after();
                    const uint32_t acc = tmem + (uint32_t)buf * 192u;
                    for (int ks = 0; ks < nks; ++ks) {
#pragma unroll
                        for (int p = 0; p < 6; ++p) {
                            // points [limb][k-chunk][256][16B]: LBO 4096, SBO 128, group pq
                            const uint64_t bd =
                                umma_desc(pBase + lp[p] * P_LIMB_BYTES + ks * 2 * 4096 + pq * TC_NP * 16, 4096, 128);
                            mma_i8_ts(acc + (uint32_t)ac[p] * TC_NP, aT + (uint32_t)(lu[p] * 2 + ks) * 8u, bd, idesc,
                                      (ks == 0 && first[p]) ? 0u : 1u);
                        }
                    }
                    mma_commit_elect(&tfull[buf]);
                }
            }
            mma_commit_elect(&pempty[pb]);  // point operand free once this item's MMAs are done
        }
    } else if (warp < 4) {
        // ------------------------- converters: x - z -> per-point scale -> int8 limbs
        const int ct = tid - 64;  // 0..63, rows ct, ct+64, ct+128, ct+192
        int it = 0;
        for (int64_t item = blockIdx.x; item < items; item += gridDim.x, ++it) {
            const int pb = it & 1;
            if (it >= 2) mbar_wait_sleep(&pempty[pb], (uint32_t)(((it >> 1) - 1) & 1));
            const int q = (int)(item / tiles2);
            const int64_t t0 = (item - (int64_t)q * tiles2) * 2;
            const int64_t vrows = a.n - t0 * 128;
            const int valid = vrows < TC_PTS ? (int)vrows : TC_PTS;
            const float* zq = a.zq + (size_t)q * d;
            unsigned char* P = sP + pb * P_BUF_BYTES;
            uint32_t zcount = 0;
            for (int rr = 0; rr < TC_PTS / TC_CONV_THREADS; ++rr) {
                const int r = ct + rr * TC_CONV_THREADS;
                // tile-blocked [T][d][128]: coalesced over r for each coordinate k
                const float* X = a.xb + ((size_t)(t0 + (r >> 7)) * d) * 128 + (r & 127);
                float mx = 0.0f;
                if (r < valid)
                    for (int k = 0; k < d; ++k) mx = fmaxf(mx, fabsf(__ldg(X + k * 128) - __ldg(zq + k)));
                zcount += (r < valid && mx == 0.0f) ? 1u : 0u;
                float scale = 0.0f;
                if (mx > 0.0f) {
                    int E = (int)((__float_as_uint(mx) >> 23) & 0xFF) - 126;  // mx < 2^E
                    if (E < -100) E = -100;
                    scale = __uint_as_float((uint32_t)(127 + 22 - E) << 23);  // 2^(22-E)
                }
                for (int c = 0; c < 4; ++c) {
                    uint32_t w0[4], w1[4], w2[4];
#pragma unroll
                    for (int g = 0; g < 4; ++g) {
                        uint32_t b0 = 0, b1 = 0, b2 = 0;
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int k = c * 16 + g * 4 + e;
                            const float av = (k < d && scale != 0.0f) ? (__ldg(X + k * 128) - __ldg(zq + k)) : 0.0f;
                            const int A0 = __float2int_rn(av * scale);
                            const int A1 = (A0 + 128) >> 8;
                            const int A2 = (A1 + 128) >> 8;
                            b0 |= ((uint32_t)A0 & 0xFFu) << (8 * e);
                            b1 |= ((uint32_t)A1 & 0xFFu) << (8 * e);
                            b2 |= ((uint32_t)A2 & 0xFFu) << (8 * e);
                        }
                        w0[g] = b0;
                        w1[g] = b1;
                        w2[g] = b2;
                    }
                    // canonical K-major, no swizzle: [limb][k-chunk c][point r][16 bytes]
                    *reinterpret_cast<uint4*>(P + 0 * P_LIMB_BYTES + c * 4096 + r * 16) = make_uint4(w0[0], w0[1], w0[2], w0[3]);
                    *reinterpret_cast<uint4*>(P + 1 * P_LIMB_BYTES + c * 4096 + r * 16) = make_uint4(w1[0], w1[1], w1[2], w1[3]);
                    *reinterpret_cast<uint4*>(P + 2 * P_LIMB_BYTES + c * 4096 + r * 16) = make_uint4(w2[0], w2[1], w2[2], w2[3]);
                }
            }
            // coinciding rows (x - z == 0) of this item: ties on both sides
            zcount = __reduce_add_sync(0xffffffffu, zcount);
            if (lane == 0 && zcount) atomicAdd(&sZrows[it & 3], zcount);
            fence_proxy_async();  // generic-proxy smem writes -> tensor-core reads
            __syncwarp();
            if (lane == 0) mbar_arrive(&pfull[pb]);
        }
    } else {
        // ------------------------------------------------------------ epilogue
        const int ct = tid - 128;          // 0..511
        const int quarter = warp & 3;      // TMEM lane quarter = 32 directions
        const int part = (warp - 4) >> 2;  // 16-point slice of each 64-point group
        const uint32_t lane_base = (uint32_t)(32 * quarter) << 16;
        int64_t gt = 0;
        int it = 0;
        for (int64_t item = blockIdx.x; item < items; item += gridDim.x, ++it) {
            const int q = (int)(item / tiles2);
            const int64_t t0 = (item - (int64_t)q * tiles2) * 2;
            const int64_t vrows = a.n - t0 * 128;
            const int valid = vrows < TC_PTS ? (int)vrows : TC_PTS;
            for (int db = 0; db < MB; ++db) {
                uint32_t cnt = 0u;  // #(y<0) over this item's points
                for (int pq = 0; pq < TC_PTS / TC_NP; ++pq, ++gt) {
                    const int buf = (int)(gt & 1);
                    mbar_wait_sleep(&tfull[buf], (uint32_t)((gt >> 1) & 1));
                    tc_fence_after();
                    const uint32_t tb = tmem + lane_base + (uint32_t)buf * 192u + (uint32_t)(part * 16);
                    uint32_t r0[16], r1[16], r2[16];
                    tmem_ld16(tb + 0 * TC_NP, r0);
                    tmem_ld16(tb + 1 * TC_NP, r1);
                    tmem_ld16(tb + 2 * TC_NP, r2);
                    tmem_wait_ld();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[buf]);  // accumulators consumed
                    // 2w = S22*2^16 + S21*2^8 + 2*floor(S20/2) = v - (S20 & 1), so
                    // sign(w) == sign(v) exactly; |w| < 2^31 for d <= 64 (|S22| < 2^15.2)
                    uint32_t lt = 0u;
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const int x = (int)r2[j] * 256 + (int)r1[j];
                        const int w = x * 128 + ((int)r0[j] >> 1);
                        lt += (uint32_t)w >> 31;
                    }
                    cnt += lt;
                }
                atomicAdd(sCnt + db * TC_MD + 32 * quarter + lane, cnt);
            }
            named_bar(1, TC_EPI_THREADS);  // all direction counts of this item are in
            // #(y>0) = real rows - coinciding rows - #(y<0); an exact zero from a
            // non-coinciding row (|y| below the quantisation error, inside the tie
            // zone) lands on the positive side
            const int zrows = (int)sZrows[it & 3];
            int* dst = a.counts + (size_t)q * a.mpad * 2;
            for (int c = ct; c < ndirs; c += TC_EPI_THREADS) {
                const int lt = (int)sCnt[c];
                sCnt[c] = 0u;
                if (c >= a.m) continue;
                const int gtv = valid - zrows - lt;
                if (lt) atomicAdd(dst + 2 * c + 0, lt);
                if (gtv) atomicAdd(dst + 2 * c + 1, gtv);
            }
            named_bar(1, TC_EPI_THREADS);
            if (ct == 0) sZrows[it & 3] = 0u;
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}

cudaError_t launch_contract_tc(const TcArgs& a, int sms, cudaStream_t st) {
    if (a.d > TC_KP || a.NB * TC_MD > TC_MAX_DIRS) return cudaErrorInvalidValue;
    const size_t smem = contract_tc_smem_bytes();
    cudaError_t e =
        cudaFuncSetAttribute(contract_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t items = (int64_t)a.Qb * ((a.tiles + 1) >> 1);
    if (items == 0) return cudaSuccess;
    const int grid = (int)(items < sms ? items : sms);
    contract_tc_kernel<<<grid, TC_THREADS, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace rrs
