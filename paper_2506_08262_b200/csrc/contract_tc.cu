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
// Operands ("two-term FP16 split", FP32-class accuracy; packed along K as in
// kernels.h tc_layout: each FP16 term stored once, d = 50 takes 7 stored K
// steps of 16 and 10 MMAs instead of 3 x 4):
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
// Layout (M = 128 DIRECTIONS on TMEM lanes, N = 128 POINTS, K = 16 per MMA,
// ns = tc_layout(d).ns stored K steps per tile / block, 3 Q + R MMAs):
//   TMEM columns [0,128) and [128,256): two FP32 accumulator buffers;
//   TMEM columns [256 + 8 ns b, 256 + 8 ns (b + 1)): direction block b of the
//   current unit (8 columns = 16 K values per step), resident for the whole
//   unit (TS MMA: A from TMEM, B from shared memory); gb = 256 / (8 ns) blocks
//   (4 at d = 50), so each converted point tile feeds 4 blocks.
// Work unit = (query, group of gb direction blocks, chunk of 128-point tiles);
// persistent CTAs (one per SM) stride over units.
//   warp 0      producer: TMA of the unit's direction blocks (ns * 4 KB each, one
//               at a time) into a staging area (cp.async.bulk + mbarrier);
//   warp 1      TMEM allocator + tcgen05 issuer: staging -> TMEM (tcgen05.cp)
//               once per unit, then per tile and block 3 Q + R MMAs;
//   warp 2      producer: TMA of each raw FP32 point tile (d*512 bytes, the
//               tile-blocked dataset) into a 2-4 stage ring;
//   warps 3-10  converters: one (point, half of K) per thread: x - z from the
//               staged tile, per-point power-of-two scale (max exchanged through
//               shared memory), FP16 hi/lo split, placed at the packed K
//               positions of the double-buffered point operand;
//   warps 11-18 epilogue: tcgen05.ld of the accumulator (64 columns per thread),
//               y < 0 counted per direction in registers, flushed per unit.
// Replaces _kernels.pyx:120-199 (projection) + 270-289 (halfspace_span).
#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

#include <cuda_fp16.h>

#ifndef RRS_TC_UNITS_PER_SM
#define RRS_TC_UNITS_PER_SM 16  // load balance of the persistent grid (units per SM, at least)
#endif

namespace rrs {

constexpr int TC_CONV_WARP0 = 3;                 // first converter warp
constexpr int TC_CONV_WARPS = 8;                 // (point, K half) per thread
constexpr int TC_CONV_THREADS = TC_CONV_WARPS * 32;
constexpr int TC_EPI_WARP0 = TC_CONV_WARP0 + TC_CONV_WARPS;  // first epilogue warp
constexpr int TC_EPI_WARPS = 8;                  // 4 lane quarters x 2 column halves
constexpr int TC_EPI_THREADS = TC_EPI_WARPS * 32;
constexpr int TC_THREADS = (TC_EPI_WARP0 + TC_EPI_WARPS) * 32;  // 608
constexpr int TC_MAXD = 64;                      // coordinates handled per point (2 x 32)
constexpr int TC_MAXNS = 9;                      // stored K steps, d <= 64 (d = 63: 2 * 3 + 3)
constexpr int TC_MD = 128;                       // directions per block (MMA M)
constexpr int TC_NP = 128;                       // points per tile (MMA N)
constexpr int TC_GB_MAX = 8;                     // direction blocks resident per unit (max)
constexpr int P_STAGES = 2;
constexpr int R_MAX_STAGES = 4;                  // raw FP32 tile ring (runtime depth)
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t ACC_COLS = TC_NP;             // 128 per accumulator buffer
constexpr uint32_t A_TMEM = 2 * ACC_COLS;        // 256: direction blocks (8 ns columns each)
constexpr int TC_SMEM_LIMIT = 227 * 1024;

// Shared-memory layout (bytes from a 1024-aligned base), runtime in ns and d.
struct TcSmem {
    int P, D, CNT, ZS, SMX, EXCL, ZROWS, INV, STG, BARS, TADDR, RAW, total;
    int stage_bytes, raw_stages, raw_rows;
    static constexpr int NBARS = 2 * P_STAGES + 2 + 2 + 3 + 2 * R_MAX_STAGES;
    __host__ __device__ TcSmem(int ns, int d, bool store) {
        stage_bytes = ns * 4096;                   // one packed tile / direction block
        P = 0;                                     // P_STAGES point operands
        D = P + P_STAGES * stage_bytes;            // direction staging (one block)
        CNT = D + stage_bytes;                     // uint32 [TC_GB_MAX * 128]
        ZS = CNT + TC_GB_MAX * TC_MD * 4;          // float [2][TC_MAXD] staged queries
        SMX = ZS + 2 * TC_MAXD * 4;                // float [2][2][128] partial |a| maxima
        EXCL = SMX + 2 * 2 * TC_NP * 4;            // uint32 [8][4] excluded-point masks per tile
        ZROWS = EXCL + 8 * 4 * 4;                  // uint32 [4] coinciding rows per unit slot
        INV = ZROWS + 16;                          // float [8][128] per-point 1 / (s 2^15) (STORE mode)
        STG = INV + (store ? 8 * TC_NP * 4 : 0);   // float [8 warps][32][33] store transpose tiles (STORE)
        BARS = STG + (store ? TC_EPI_WARPS * 32 * 33 * 4 : 0);  // mbarriers
        TADDR = BARS + NBARS * 8;
        RAW = (TADDR + 16 + 1023) & ~1023;         // raw FP32 tiles: 64 rows of 128 (rows >= d stay 0)
        const int room = TC_SMEM_LIMIT - 1024 - RAW;
        raw_rows = (d + 7) & ~7;                   // rows past d stay zero (whole 8-coordinate chunks)
        raw_stages = room / (raw_rows * TC_NP * 4);
        if (raw_stages > R_MAX_STAGES) raw_stages = R_MAX_STAGES;
        total = RAW + raw_stages * raw_rows * TC_NP * 4 + 1024;
    }
};

struct TcUnit {
    int q, grp, nbg;     // query, direction group, blocks in the group
    int64_t t0, t1;      // point tiles [t0, t1)
};

// first unit >= u of this CTA's stride whose query is still live (early exit:
// done[] is written by the previous update kernel and read-only here, so every
// warp role walks the same unit sequence)
// units over the direction blocks [jb0, jb0 + jbn) of each query (count mode:
// all NB); grp counts gb-block groups from jb0
__device__ __forceinline__ int64_t tc_next(const TcArgs& a, int64_t u, int64_t units) {
    if (a.done) {
        const int64_t per_q = (int64_t)a.groups * a.chunks;
        while (u < units && a.done[u / per_q]) u += gridDim.x;
    }
    return u;
}

__device__ __forceinline__ TcUnit tc_unit(const TcArgs& a, int64_t u) {
    TcUnit r;
    const int64_t per_q = (int64_t)a.groups * a.chunks;
    r.q = (int)(u / per_q);
    const int64_t rem = u - (int64_t)r.q * per_q;
    r.grp = (int)(rem / a.chunks);
    const int64_t c = rem - (int64_t)r.grp * a.chunks;
    r.nbg = a.jbn - r.grp * a.gb < a.gb ? a.jbn - r.grp * a.gb : a.gb;
    r.t0 = c * a.tiles_per_chunk;
    r.t1 = r.t0 + a.tiles_per_chunk < a.tiles ? r.t0 + a.tiles_per_chunk : a.tiles;
    return r;
}

template <int Q, int R>
__device__ __forceinline__ void mma_issue(const TcArgs& a, int64_t units, unsigned char* sP, unsigned char* sD,
                                          uint64_t* pfull, uint64_t* pempty, uint64_t* dfull, uint64_t* dempty,
                                          uint64_t* tfull, uint64_t* tempty, uint64_t* udone) {
    constexpr uint32_t tmem = 0u;
    constexpr int NS = 2 * Q + R;
    constexpr uint32_t stage_bytes = NS * 4096;
    // F32 accumulate, FP16 A and B, K-major both, N = 128, M = 128
    const uint32_t idesc = (1u << 4) | ((uint32_t)(TC_NP >> 3) << 17) | ((uint32_t)(TC_MD >> 4) << 24);
    uint32_t it = 0, gtile = 0, gacc = 0, gph = 0;
    for (int64_t u = tc_next(a, blockIdx.x, units); u < units; u = tc_next(a, u + gridDim.x, units), ++it) {
        const TcUnit w = tc_unit(a, u);
        for (int b = 0; b < w.nbg; ++b, ++gph) {
            mbar_wait_sleep(dfull, gph & 1u);
            if (b == 0 && it > 0) mbar_wait(udone, (it - 1) & 1u);  // previous unit no longer reads TMEM A
            tc_fence_after();
            tmem_cp_dirblock(tmem + A_TMEM + 8u * NS * b, umma_desc(smem_u32(sD), 2048, 128), NS);
            mma_commit_elect(dempty);  // staging free once the copies are done
        }
        for (int64_t t = w.t0; t < w.t1; ++t, ++gtile) {
            const uint32_t s = gtile % P_STAGES;
            mbar_wait(&pfull[s], (gtile / P_STAGES) & 1u);
            tc_fence_after();
            const uint64_t bd = umma_desc(smem_u32(sP) + s * stage_bytes, 2048, 128);
            for (int b = 0; b < w.nbg; ++b, ++gacc) {
                const uint32_t buf = gacc & 1u;
                if (gacc >= 2) mbar_wait(&tempty[buf], ((gacc >> 1) - 1) & 1u);
                tc_fence_after();
                mma_split_block<Q, R>(tmem + buf * ACC_COLS, tmem + A_TMEM + 8u * NS * b, bd, idesc,
                                      smem_u32(&tfull[buf]));
            }
            mma_commit_elect(&pempty[s]);  // point stage free once this tile's MMAs are done
        }
        mma_commit_elect(udone);
    }
}

template <bool STORE>
__global__ void __launch_bounds__(TC_THREADS, 1) contract_tc_kernel(const TcArgs a) {
    extern __shared__ __align__(1024) unsigned char tc_raw[];
    // 1024-align by pointer arithmetic on the __shared__ array (keeps the address space)
    unsigned char* sm = tc_raw + ((1024u - (smem_u32(tc_raw) & 1023u)) & 1023u);
    const int d = a.d;
    const TcLayout L = tc_layout(d);
    const TcSmem lay(L.ns, d, STORE);
    const int stage_bytes = lay.stage_bytes;
    unsigned char* sP = sm + lay.P;
    unsigned char* sD = sm + lay.D;
    uint32_t* sCnt = reinterpret_cast<uint32_t*>(sm + lay.CNT);
    float* sZ = reinterpret_cast<float*>(sm + lay.ZS);
    float* sMx = reinterpret_cast<float*>(sm + lay.SMX);
    uint32_t* sExcl = reinterpret_cast<uint32_t*>(sm + lay.EXCL);
    float* sInv = reinterpret_cast<float*>(sm + lay.INV);
    float* sStg = reinterpret_cast<float*>(sm + lay.STG);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + lay.BARS);
    uint64_t* pfull = &bars[0];                   // [P_STAGES] point tile converted (converter warps)
    uint64_t* pempty = &bars[P_STAGES];           // [P_STAGES] MMAs reading it completed
    uint64_t* tfull = &bars[2 * P_STAGES];        // [2] accumulator ready
    uint64_t* tempty = &bars[2 * P_STAGES + 2];   // [2] accumulator drained (epilogue warps)
    uint64_t* dfull = &bars[2 * P_STAGES + 4];    // direction staging loaded
    uint64_t* dempty = &bars[2 * P_STAGES + 5];   // direction staging copied to TMEM
    uint64_t* udone = &bars[2 * P_STAGES + 6];    // all MMAs of a unit completed
    uint64_t* rfull = &bars[2 * P_STAGES + 7];    // [R_MAX_STAGES] raw tile landed
    uint64_t* rempty = &bars[2 * P_STAGES + 7 + R_MAX_STAGES];  // [R_MAX_STAGES] raw tile read
    uint32_t* sTaddr = reinterpret_cast<uint32_t*>(sm + lay.TADDR);
    float* sRaw = reinterpret_cast<float*>(sm + lay.RAW);
    const int RS = lay.raw_stages;
    const uint32_t raw_bytes = (uint32_t)(d * TC_NP * 4);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t units = (int64_t)a.Qb * a.groups * a.chunks;

    // point operand stages start zeroed: K positions past the packed products
    // are never written again, so they stay 0 (A is 0 there too)
    for (int i = tid; i < P_STAGES * stage_bytes / 16; i += TC_THREADS)
        reinterpret_cast<uint4*>(sP)[i] = make_uint4(0u, 0u, 0u, 0u);
    const int RR = lay.raw_rows;
    for (int i = tid; i < RS * RR * TC_NP; i += TC_THREADS) sRaw[i] = 0.0f;  // rows >= d stay 0
    for (int c = tid; c < TC_GB_MAX * TC_MD; c += TC_THREADS) sCnt[c] = 0u;
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
    fence_proxy_async();  // zeroed operand stages -> tensor-core reads
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    // The single 512-column allocation of the only CTA on the SM starts at
    // lane 0, column 0; the issuer relies on that constant so that every MMA
    // operand stays on the uniform datapath.
    if (*sTaddr != 0u) __trap();
    constexpr uint32_t tmem = 0u;

    if (warp == 0) {
        // -------------------------------- producer: unit direction blocks, one at a time
        uint32_t gph = 0;
        for (int64_t u = tc_next(a, blockIdx.x, units); u < units; u = tc_next(a, u + gridDim.x, units)) {
            const TcUnit w = tc_unit(a, u);
            const unsigned char* src = a.uop + ((size_t)w.q * a.NB + (size_t)(a.jb0 + w.grp * a.gb)) * stage_bytes;
            for (int b = 0; b < w.nbg; ++b, ++gph) {
                if (gph > 0) mbar_wait_sleep(dempty, (gph - 1) & 1u);
                expect_tx_elect(dfull, (uint32_t)stage_bytes);
                tma_load_elect(sD, src + (size_t)b * stage_bytes, (uint32_t)stage_bytes, dfull);
                __syncwarp();
            }
        }
    } else if (warp == 1) {
        // -------------------------------------------------------- MMA issuer
#define RRS_TC_ISSUE(Q, R) mma_issue<Q, R>(a, units, sP, sD, pfull, pempty, dfull, dempty, tfull, tempty, udone)
        switch (4 * L.q16 + L.rsteps) {
            case 1: RRS_TC_ISSUE(0, 1); break;
            case 2: RRS_TC_ISSUE(0, 2); break;
            case 3: RRS_TC_ISSUE(0, 3); break;
            case 4: RRS_TC_ISSUE(1, 0); break;
            case 5: RRS_TC_ISSUE(1, 1); break;
            case 6: RRS_TC_ISSUE(1, 2); break;
            case 7: RRS_TC_ISSUE(1, 3); break;
            case 8: RRS_TC_ISSUE(2, 0); break;
            case 9: RRS_TC_ISSUE(2, 1); break;
            case 10: RRS_TC_ISSUE(2, 2); break;
            case 11: RRS_TC_ISSUE(2, 3); break;
            case 12: RRS_TC_ISSUE(3, 0); break;
            case 13: RRS_TC_ISSUE(3, 1); break;
            case 14: RRS_TC_ISSUE(3, 2); break;
            case 15: RRS_TC_ISSUE(3, 3); break;
            default: RRS_TC_ISSUE(4, 0); break;
        }
#undef RRS_TC_ISSUE
    } else if (warp == 2) {
        // -------------------------------------- producer: raw FP32 point tiles
        uint32_t g = 0, rs = 0, rph = 0;  // ring slot and its phase, advanced incrementally
        for (int64_t u = tc_next(a, blockIdx.x, units); u < units; u = tc_next(a, u + gridDim.x, units)) {
            const TcUnit w = tc_unit(a, u);
            for (int64_t t = w.t0; t < w.t1; ++t, ++g) {
                if (g >= (uint32_t)RS) mbar_wait_sleep(&rempty[rs], rph ^ 1u);
                expect_tx_elect(&rfull[rs], raw_bytes);
                tma_load_elect(sRaw + (size_t)rs * RR * TC_NP, a.xb + (size_t)t * d * TC_NP, raw_bytes, &rfull[rs]);
                __syncwarp();
                if (++rs == (uint32_t)RS) {
                    rs = 0;
                    rph ^= 1u;
                }
            }
        }
    } else if (warp < TC_EPI_WARP0) {
        // ----------------------- converters: x - z -> scale -> FP16 hi/lo split
        const int ct = tid - TC_CONV_WARP0 * 32;  // 0..255
        const int r = ct & (TC_NP - 1);           // point of the tile
        const int h = ct >> 7;                    // coordinates [32 h, 32 h + 32)
        const int main_chunks = 2 * L.q16;        // 8-coordinate chunks in the aligned part
        uint32_t it = 0, gtile = 0, rs = 0, rph = 0;
        for (int64_t u = tc_next(a, blockIdx.x, units); u < units; u = tc_next(a, u + gridDim.x, units), ++it) {
            const TcUnit w = tc_unit(a, u);
            float* zs = sZ + (it & 1u) * TC_MAXD;
            if (ct < TC_MAXD) zs[ct] = ct < d ? __ldg(a.zq + (size_t)w.q * d + ct) : 0.0f;
            named_bar(2, TC_CONV_THREADS);  // zs ready; keeps the converter warps in step per unit
            for (int64_t t = w.t0; t < w.t1; ++t, ++gtile) {
                const uint32_t s = gtile % P_STAGES;
                const bool ok = t * TC_NP + r < a.n;
                mbar_wait(&rfull[rs], rph);
                // staged tile [64][128] (rows >= d are 0, zs too): lane-consecutive points,
                // conflict-free, immediate offsets; chunks past d are skipped (warp-uniform)
                const float* X = sRaw + (size_t)rs * RR * TC_NP + 32 * h * TC_NP + r;
                const float* zh = zs + 32 * h;
                float2 av[16];  // coordinate pairs, packed FP32x2 arithmetic (FADD2 / FMUL2)
                float mx = 0.0f;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    if (8 * (4 * h + c) < d) {
                        const float4 z0 = *reinterpret_cast<const float4*>(zh + 8 * c);
                        const float4 z1 = *reinterpret_cast<const float4*>(zh + 8 * c + 4);
                        const float2 nz[4] = {make_float2(-z0.x, -z0.y), make_float2(-z0.z, -z0.w),
                                              make_float2(-z1.x, -z1.y), make_float2(-z1.z, -z1.w)};
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float2 xv = make_float2(X[(8 * c + 2 * e) * TC_NP], X[(8 * c + 2 * e + 1) * TC_NP]);
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
                if (lane == 0) mbar_arrive(&rempty[rs]);  // raw tile consumed (loads ordered by release)
                if (++rs == (uint32_t)RS) {
                    rs = 0;
                    rph ^= 1u;
                }
                float* mxs = sMx + (gtile & 1u) * 2 * TC_NP;
                mxs[h * TC_NP + r] = mx;
                named_bar(2, TC_CONV_THREADS);  // both halves' maxima visible
                mx = fmaxf(mxs[r], mxs[TC_NP + r]);
                if (h == 0) {
                    // points the epilogue must not count: coinciding rows (every product a
                    // signed zero, ties on both sides) and rows beyond n (their operand is
                    // finite garbage, x = 0 padding minus z)
                    const uint32_t ex = __ballot_sync(0xffffffffu, !ok || mx == 0.0f);
                    if (lane == 0) sExcl[(gtile & 7u) * 4 + (r >> 5)] = ex;
                }
                float scale = 0.0f;
                if (mx > 0.0f) {
                    int E = (int)((__float_as_uint(mx) >> 23) & 0xFF) - 126;  // mx < 2^E
                    if (E < -100) E = -100;
                    scale = __uint_as_float((uint32_t)(127 + 14 - E) << 23);  // 2^(14-E)
                    // STORE: exact rescale y = acc 2^(E - 29) for the epilogue (8-deep ring;
                    // the converter runs at most P_STAGES + 2 tiles ahead of it)
                    if (STORE && h == 0) sInv[(gtile & 7u) * TC_NP + r] = ldexpf(1.0f, E - 29);
                } else if (STORE && h == 0) {
                    sInv[(gtile & 7u) * TC_NP + r] = 0.0f;
                }
                if (gtile >= P_STAGES) mbar_wait(&pempty[s], ((gtile / P_STAGES) - 1) & 1u);
                // packed K layout (kernels.h tc_layout), canonical K-major:
                // [kk / 8][point r][16 bytes]
                unsigned char* P = sP + s * stage_bytes + r * 16;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int cc = 4 * h + c;  // coordinate chunk
                    if (8 * cc >= d) continue;
                    uint32_t hw[4], lw[4];
                    const float2 sc2 = make_float2(scale, scale);
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float2 v = __fmul2_rn(av[4 * c + e], sc2);
                        const __half2 hh = __floats2half2_rn(v.x, v.y);
                        const float2 hf = __half22float2(hh);
                        const float2 res = __fadd2_rn(v, make_float2(-hf.x, -hf.y));
                        hw[e] = *reinterpret_cast<const uint32_t*>(&hh);
                        lw[e] = pack_half2(res.x, res.y);
                    }
                    if (cc < main_chunks) {
                        // aligned part: the hi and the lo terms of coordinates 8 cc .. 8 cc + 7
                        *reinterpret_cast<uint4*>(P + cc * (TC_NP * 16)) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
                        *reinterpret_cast<uint4*>(P + (main_chunks + cc) * (TC_NP * 16)) =
                            make_uint4(lw[0], lw[1], lw[2], lw[3]);
                    } else if (L.rem <= 2) {
                        // remainder of one or two coordinates (d = 50: 48, 49): its products sit
                        // at K positions 32 Q + p rem + i, all inside one 16-byte chunk
                        // [hi0 hi1 lo0 lo1 hi0 hi1 0 0] (rem 2) / [hi lo hi 0 ...] (rem 1)
                        const uint32_t h0 = hw[0], l0 = lw[0];
                        const uint4 rv = L.rem == 2 ? make_uint4(h0, l0, h0, 0u)
                                                    : make_uint4((h0 & 0xFFFFu) | (l0 << 16), h0 & 0xFFFFu, 0u, 0u);
                        *reinterpret_cast<uint4*>(P + (4 * L.q16) * (TC_NP * 16)) = rv;
                    } else {
                        // remainder coordinates 16 Q + i: scattered into the tail K steps
                        // (a rolled loop: at most two such chunks, d % 16 values)
#pragma unroll 1
                        for (int e = 0; e < 8; ++e) {
                            const int cd = 8 * cc + e;
                            if (cd >= d) break;
                            const int wi = e >> 1;
                            const uint32_t hv = wi == 0 ? hw[0] : wi == 1 ? hw[1] : wi == 2 ? hw[2] : hw[3];
                            const uint32_t lv = wi == 0 ? lw[0] : wi == 1 ? lw[1] : wi == 2 ? lw[2] : lw[3];
                            const uint16_t hb = (uint16_t)((e & 1) ? (hv >> 16) : (hv & 0xFFFFu));
                            const uint16_t lb = (uint16_t)((e & 1) ? (lv >> 16) : (lv & 0xFFFFu));
                            int kk = 16 * L.q16 + cd;  // 32 Q + (cd - 16 Q): product 0
#pragma unroll
                            for (int pr = 0; pr < 3; ++pr, kk += L.rem)
                                *reinterpret_cast<uint16_t*>(P + (kk >> 3) * (TC_NP * 16) + (kk & 7) * 2) =
                                    pr == 1 ? lb : hb;
                        }
                    }
                }
                fence_proxy_async();  // generic-proxy smem writes -> tensor-core reads
                __syncwarp();
                if (lane == 0) mbar_arrive(&pfull[s]);
            }
        }
    } else if (STORE) {
        // ---------------------------------------------- epilogue: y' rows (STORE)
        const int quarter = warp & 3;
        const int half = (warp - TC_EPI_WARP0) >> 2;
        const uint32_t lane_base = (uint32_t)(32 * quarter) << 16;
        const bool vec = (a.n & 3) == 0;
        float* stg = sStg + (warp - TC_EPI_WARP0) * 32 * 33;
        uint32_t gacc = 0, gtile = 0;
        for (int64_t u = tc_next(a, blockIdx.x, units); u < units; u = tc_next(a, u + gridDim.x, units)) {
            const TcUnit w = tc_unit(a, u);
            for (int64_t t = w.t0; t < w.t1; ++t, ++gtile) {
                const float* inv = sInv + (gtile & 7u) * TC_NP + 64 * half;
                const int64_t p0 = t * TC_NP + 64 * half;
                for (int b = 0; b < w.nbg; ++b) {
                    const uint32_t buf = gacc & 1u;
                    mbar_wait(&tfull[buf], (gacc >> 1) & 1u);
                    ++gacc;
                    tc_fence_after();
                    const uint32_t tb = tmem + lane_base + buf * ACC_COLS + (uint32_t)(half * 64);
                    uint32_t y0[32], y1[32];
                    tmem_ld32(tb, y0);
                    tmem_ld32(tb + 32, y1);
                    tmem_wait_ld();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[buf]);
                    const int blk = a.jb0 + w.grp * a.gb + b;  // absolute direction block
                    const int row0 = blk * TC_MD + 32 * quarter;  // the warp's first direction
                    const int rows_live = min(32, a.m - row0);
                    float* ybase = a.y + ((size_t)w.q * a.jbn * TC_MD + (size_t)(blk - a.jb0) * TC_MD + 32 * quarter) *
                                             (size_t)a.n;
#pragma unroll
                    for (int part = 0; part < 2; ++part) {
                        const uint32_t* yv = part ? y1 : y0;
                        const int64_t pb = p0 + 32 * part;
                        if (vec && pb + 32 <= a.n) {
                            // transpose through the warp's tile: each store writes 4 rows x 128 B
#pragma unroll
                            for (int k = 0; k < 32; ++k) stg[lane * 33 + k] = __uint_as_float(yv[k]) * inv[32 * part + k];
                            __syncwarp();
                            const int c4 = 4 * (lane & 7);
#pragma unroll
                            for (int k = 0; k < 8; ++k) {
                                const int rr = (lane >> 3) + 4 * k;
                                if (rr < rows_live) {
                                    const float* sv = stg + rr * 33 + c4;
                                    *reinterpret_cast<float4*>(ybase + (size_t)rr * a.n + pb + c4) =
                                        make_float4(sv[0], sv[1], sv[2], sv[3]);
                                }
                            }
                            __syncwarp();
                        } else if (lane < rows_live) {
                            float* yrow = ybase + (size_t)lane * a.n;
#pragma unroll
                            for (int k = 0; k < 32; ++k)
                                if (pb + k < a.n) yrow[pb + k] = __uint_as_float(yv[k]) * inv[32 * part + k];
                        }
                    }
                }
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue
        const int ct = tid - TC_EPI_WARP0 * 32;        // 0..255
        const int quarter = warp & 3;                  // TMEM lane quarter = 32 directions
        const int half = (warp - TC_EPI_WARP0) >> 2;   // 64-point half of the tile
        const uint32_t lane_base = (uint32_t)(32 * quarter) << 16;
        uint32_t it = 0, gacc = 0, gtile = 0;
        for (int64_t u = tc_next(a, blockIdx.x, units); u < units; u = tc_next(a, u + gridDim.x, units), ++it) {
            const TcUnit w = tc_unit(a, u);
            uint32_t cnt[TC_GB_MAX];  // #(y<0) per resident block
#pragma unroll
            for (int b = 0; b < TC_GB_MAX; ++b) cnt[b] = 0u;
            uint32_t zsum = 0;  // coinciding rows (x - z == 0) of the unit's tiles
            for (int64_t t = w.t0; t < w.t1; ++t, ++gtile) {
                uint32_t keep0 = 0u, keep1 = 0u;
#pragma unroll
                for (int b = 0; b < TC_GB_MAX; ++b) {
                    if (b < w.nbg) {
                        const uint32_t buf = gacc & 1u;
                        mbar_wait(&tfull[buf], (gacc >> 1) & 1u);
                        ++gacc;
                        tc_fence_after();
                        if (b == 0) {
                            // excluded points of this tile (written by the converters before the
                            // tile's pfull; ordered through pfull -> MMA -> tfull), bit j = point
                            // half*64 + 32 i + j
                            const uint32_t* ex = sExcl + (gtile & 7u) * 4;
                            keep0 = ~ex[2 * half];
                            keep1 = ~ex[2 * half + 1];
                            // excluded = coinciding or past n: coinciding = excluded - padding
                            const int64_t pad = (t + 1) * TC_NP - a.n;
                            zsum += (uint32_t)(__popc(ex[0]) + __popc(ex[1]) + __popc(ex[2]) + __popc(ex[3])) -
                                    (uint32_t)(pad > 0 ? pad : 0);
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
                        // static register indices (a dynamic cnt[b] lands in local memory)
                        const uint32_t v = (uint32_t)(__popc(m0 & keep0) + __popc(m1 & keep1));
#pragma unroll
                        for (int i = 0; i < TC_GB_MAX; ++i) cnt[i] += i == b ? v : 0u;
                    }
                }
            }
#pragma unroll
            for (int b = 0; b < TC_GB_MAX; ++b)
                if (b < w.nbg) atomicAdd(sCnt + b * TC_MD + 32 * quarter + lane, cnt[b]);
            named_bar(1, TC_EPI_THREADS);  // all direction counts of this unit are in
            // #(y>0) = real rows - coinciding rows - #(y<0); an exact zero from a
            // non-coinciding row (|y| below the rounding error, inside the tie
            // zone) lands on the positive side
            const int64_t r1 = w.t1 * TC_NP < a.n ? w.t1 * TC_NP : a.n;
            const int valid = (int)(r1 - w.t0 * TC_NP);
            const int zrows = (int)zsum;
            int* dst = a.counts + (size_t)w.q * a.mpad * 2;
            const int j0 = w.grp * a.gb * TC_MD;
            for (int c = ct; c < w.nbg * TC_MD; c += TC_EPI_THREADS) {
                const int lt = (int)sCnt[c];
                sCnt[c] = 0u;
                if (j0 + c >= a.m) continue;
                const int gtv = valid - zrows - lt;
                if (lt) atomicAdd(dst + 2 * (j0 + c) + 0, lt);
                if (gtv) atomicAdd(dst + 2 * (j0 + c) + 1, gtv);
            }
            named_bar(1, TC_EPI_THREADS);
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}

void plan_contract_tc(TcArgs& a, int sms) {
    const TcLayout L = tc_layout(a.d);
    int gb = (int)(256 / (8 * L.ns));  // direction blocks that fit the 256 A columns of TMEM
    if (gb > TC_GB_MAX) gb = TC_GB_MAX;
    a.gb = gb;
    a.groups = (a.jbn + gb - 1) / gb;
    // split the point tiles into chunks so that every SM gets >= RRS_TC_UNITS_PER_SM units
    const int64_t base = (int64_t)a.Qb * a.groups;
    int64_t chunks = ((int64_t)RRS_TC_UNITS_PER_SM * sms + base - 1) / base;
    if (chunks < 1) chunks = 1;
    if (chunks > a.tiles) chunks = a.tiles;
    a.tiles_per_chunk = (a.tiles + chunks - 1) / chunks;
    a.chunks = (int)((a.tiles + a.tiles_per_chunk - 1) / a.tiles_per_chunk);
}

template <bool STORE>
static cudaError_t launch_tc(TcArgs a, int sms, cudaStream_t st) {
    if (a.d > TC_MAXD || a.d < 1 || tc_layout(a.d).ns > TC_MAXNS) return cudaErrorInvalidValue;
    if (!STORE) {
        a.jb0 = 0;
        a.jbn = a.NB;
    }
    plan_contract_tc(a, sms);
    const TcSmem lay(tc_layout(a.d).ns, a.d, STORE);
    a.raw_stages = lay.raw_stages;
    if (a.raw_stages < 2) return cudaErrorInvalidValue;
    const size_t smem = (size_t)lay.total;
    cudaError_t e =
        cudaFuncSetAttribute(contract_tc_kernel<STORE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t units = (int64_t)a.Qb * a.groups * a.chunks;
    if (units == 0) return cudaSuccess;
    const int grid = (int)(units < sms ? units : sms);
    contract_tc_kernel<STORE><<<grid, TC_THREADS, smem, st>>>(a);
    return cudaGetLastError();
}

bool contract_tc_store_fits(int d) {
    return d >= 1 && d <= TC_MAXD && TcSmem(tc_layout(d).ns, d, true).raw_stages >= 2;
}

cudaError_t launch_contract_tc(TcArgs a, int sms, cudaStream_t st) { return launch_tc<false>(a, sms, st); }
cudaError_t launch_contract_tc_store(TcArgs a, int sms, cudaStream_t st) { return launch_tc<true>(a, sms, st); }

}  // namespace rrs
