// contract_tcf.cu -- K2 halfspace contraction by FILTER AND REFINE (d <= 64):
// one FP16 product per coordinate on the 5th-generation tensor cores decides
// the sign of y = <u, x - z> for every (direction, point) pair whose |y| is
// provably above the product's error bound; the few pairs inside the bound are
// recomputed exactly with the FFMA kernel's own FP32 arithmetic.  The counts
// are therefore bit-identical to contract.cu (FFMA) for EVERY pair, at 4 MMA
// K-steps per tile and block at d = 50 instead of the 10 of the two-term split
// (contract_tc.cu).
//
// Replaces _kernels.pyx:120-199 (projection) + 270-289 (halfspace_span).
//
// Operands (per pair (j, i), a = x_i - z in FP32 exactly as contract.cu forms it):
//   point  i: b_l = fp16(a_l * s_i), s_i = C_B / ||a_i||  (so ||b|| ~ C_B);
//   direction j: A_l = fp16(u_jl * S_U)                  (u from the FP64 rows);
//   threshold slot (K index d): A = 1, B = 1, so the accumulator holds
//             w = sum_l A_l b_l + 1 = y * s_i * S_U + err + 1.
// Error bound (fp16 rounding <= 2^-11 relative, 2^-25 absolute below 2^-14;
// products exact in FP32; FP32 accumulation <= K 2^-21 sum|products|):
//   |err| <= 2^-10 (1 + 2^-11) S_U ||u|| ||a s|| + 3e-4 + 80 * 2^-21 * 858
//         <= 0.834 + 0.0003 + 0.033 < 0.87 < 1        (S_U C_B = 2^10 / 1.2),
// so with T = 1:
//   w < 0        (bit 31)           => y < 0 for sure;
//   w >= 2       (bits 31,30 = 01)  => y > 0 for sure;
//   0 <= w < 2   (bits 31,30 = 00)  => ambiguous: refined exactly.
// Both bits of 16 accumulators go into one register by 2-bit funnel shifts,
// i.e. ~1 instruction per pair.  Padded points carry B = 4 in the slot (w = 4:
// decisive positive, and real-row counting excludes them); padded directions
// carry A = 4 (their counts are discarded).  Points whose ||a|| is 0 or outside
// (2^-50, 2^50) (the query's own row, duplicates) get b = 0: w = 1, refined.
// Refinement: y = fma chain over l ascending from +0 with the FP32 direction
// u32 = (float)u64 and a, exactly contract.cu's accumulation, so
// #(y<0), #(y>0) per direction equal the FFMA kernel's; exact zeros count on
// both sides (cle = n - #>0, cge = n - #<0) like the reference's ties.
//
// Layout (M = 128 directions on TMEM lanes, N = 128 points, K = 16 per MMA,
// ns = ceil((d+1)/16) K-steps; TMEM: three FP32 accumulators at columns 0,
// 128, 256 and the unit's gb direction blocks at 384 + 8 ns b):
//   warp 0      TMA: the unit's direction blocks (FP16, one staging buffer) and
//               its FP32 direction rows U32 [gb*128][dp] (for refinement);
//   warp 1      TMEM allocator + tcgen05 issuer (tcgen05.cp of the blocks per
//               unit, ns MMAs per tile and block, commits);
//   warps 2-9   converters, thread = (point, alternate 8-coordinate chunks):
//               x prefetched one tile ahead into registers (coalesced loads of
//               the tile-blocked dataset), a = x - z into a ring of S_A row-major
//               slots [128][dp] kept until the tile's refinement, ||a||^2
//               (halves exchanged in shared memory), scale, FP16 operand;
//   warps 10-13 epilogue, one per TMEM lane quarter: tcgen05.ld, 2-bit
//               classification, counts, and the refinement of the tile's
//               ambiguous pairs through a shared queue (32 pairs per warp
//               instruction); 14 warps in all, so that 128 registers fit
//               (at most 4 warps per SM sub-partition).
#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

#include <cuda_fp16.h>

namespace rrs {

constexpr int F_CONV_WARP0 = 2;
constexpr int F_CONV_WARPS = 8;                            // (point, half of the 8-coordinate chunks)
constexpr int F_CONV_THREADS = F_CONV_WARPS * 32;
constexpr int F_EPI_WARP0 = F_CONV_WARP0 + F_CONV_WARPS;  // 10
constexpr int F_EPI_WARPS = 4;                             // one per TMEM lane quarter, all 128 points
constexpr int F_EPI_THREADS = F_EPI_WARPS * 32;
constexpr int F_THREADS = (F_EPI_WARP0 + F_EPI_WARPS) * 32;  // 448: <= 4 warps per SM sub-partition
constexpr int F_NP = 128;
constexpr int F_MD = 128;
constexpr int F_NACC = 3;
constexpr int F_P_STAGES = 2;
constexpr int F_QCAP = 2048;
constexpr int F_GB_MAX = 3;
constexpr int F_SA_MAX = 4;
constexpr int F_MAXCH = 5;                                 // 8-coordinate chunks per converter thread (d <= 64)
constexpr int F_XCH = 4;                                   // ... that hold coordinates (the 5th only the slot)
constexpr uint32_t F_TMEM_COLS = 512;
constexpr uint32_t F_A_TMEM = F_NACC * F_NP;  // 384
constexpr int F_SMEM_LIMIT = 227 * 1024;

struct TcfSmem {
    int P, D, A32, U32, Q, CNT, ZS, NRM, QC, BARS, TADDR, total;
    int stage_bytes, row_bytes;
    static constexpr int NBARS = 2 * F_P_STAGES + 2 * F_NACC + 3 + 2 * F_SA_MAX + 2;
    __host__ __device__ TcfSmem(int d, int gb, int sa) {
        const int ns = tcf_ns(d);
        row_bytes = tcf_dp(d) * 4;
        stage_bytes = ns * 4096;
        P = 0;
        D = P + F_P_STAGES * stage_bytes;
        A32 = D + stage_bytes;
        U32 = A32 + sa * F_NP * row_bytes;
        Q = U32 + gb * F_MD * row_bytes;
        CNT = Q + F_QCAP * 4;                 // int [F_GB_MAX][128][4]: neg, amb, fix<0, fix>0
        ZS = CNT + F_GB_MAX * F_MD * 16;      // float [2][64] query per unit parity
        NRM = ZS + 2 * 64 * 4;                // float [2][2][128] partial |a|^2 (tile parity, half)
        QC = NRM + 2 * 2 * F_NP * 4;          // int [2] queue counters (tile parity)
        BARS = QC + 16;
        TADDR = BARS + NBARS * 8;
        total = TADDR + 16 + 1024;
    }
};

struct TcfUnit {
    int q, grp, nbg;
    int t0, t1;  // point tiles [t0, t1)
};

// 32-bit unit arithmetic (launch_contract_tcf checks that units and tiles fit)
__device__ __forceinline__ TcfUnit tcf_unit(const TcfArgs& a, int u) {
    TcfUnit r;
    const int per_q = a.groups * a.chunks;
    r.q = u / per_q;
    const int rem = u - r.q * per_q;
    r.grp = rem / a.chunks;
    const int c = rem - r.grp * a.chunks;
    r.nbg = a.NB - r.grp * a.gb < a.gb ? a.NB - r.grp * a.gb : a.gb;
    const int tpc = (int)a.tiles_per_chunk, T = (int)a.tiles;
    r.t0 = c * tpc;
    r.t1 = r.t0 + tpc < T ? r.t0 + tpc : T;
    return r;
}

template <int NS>
__device__ __forceinline__ void tcf_mma_issue(const TcfArgs& a, int units, unsigned char* sP, unsigned char* sD,
                                              uint64_t* pfull, uint64_t* pempty, uint64_t* dfull, uint64_t* dempty,
                                              uint64_t* tfull, uint64_t* tempty, uint64_t* udone) {
    constexpr uint32_t stage_bytes = NS * 4096;
    const uint32_t idesc = (1u << 4) | ((uint32_t)(F_NP >> 3) << 17) | ((uint32_t)(F_MD >> 4) << 24);
    uint32_t it = 0, gtile = 0, gacc = 0, gph = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++it) {
        const TcfUnit w = tcf_unit(a, u);
        for (int b = 0; b < w.nbg; ++b, ++gph) {
            mbar_wait_sleep(dfull, gph & 1u);
            if (b == 0 && it > 0) mbar_wait(udone, (it - 1) & 1u);  // previous unit's MMAs no longer read A
            tc_fence_after();
            tmem_cp_dirblock(F_A_TMEM + 8u * NS * b, umma_desc(smem_u32(sD), 2048, 128), NS);
            mma_commit_elect(dempty);
        }
        for (int t = w.t0; t < w.t1; ++t, ++gtile) {
            const uint32_t s = gtile % F_P_STAGES;
            mbar_wait(&pfull[s], (gtile / F_P_STAGES) & 1u);
            tc_fence_after();
            const uint64_t bd = umma_desc(smem_u32(sP) + s * stage_bytes, 2048, 128);
            for (int b = 0; b < w.nbg; ++b, ++gacc) {
                const uint32_t buf = gacc % F_NACC;
                if (gacc >= F_NACC) mbar_wait(&tempty[buf], ((gacc / F_NACC) - 1) & 1u);
                tc_fence_after();
                mma_tile_block<NS>(buf * F_NP, F_A_TMEM + 8u * NS * b, bd, idesc, smem_u32(&tfull[buf]));
            }
            mma_commit_elect(&pempty[s]);
        }
        mma_commit_elect(udone);
    }
}

// y = sum_l u_l * a_l, fma chain ascending from +0 (contract.cu's arithmetic;
// padded coordinates are 0 * 0 and leave the chain unchanged)
__device__ __forceinline__ float refine_dot(const float* arow, const float* urow, int dp4) {
    const float4* A = reinterpret_cast<const float4*>(arow);
    const float4* U = reinterpret_cast<const float4*>(urow);
    float acc = 0.0f;
#pragma unroll 4
    for (int c = 0; c < dp4; ++c) {
        const float4 a4 = A[c], u4 = U[c];
        acc = fmaf(a4.x, u4.x, acc);
        acc = fmaf(a4.y, u4.y, acc);
        acc = fmaf(a4.z, u4.z, acc);
        acc = fmaf(a4.w, u4.w, acc);
    }
    return acc;
}

// converter: x of the thread's chunks of tile t (K-major tile-blocked dataset),
// one coalesced 128-byte load per coordinate and warp
__device__ __forceinline__ void load_x_chunks(const float* __restrict__ xb, int t, int d, int r, int h,
                                              float (&x)[F_XCH][8]) {
    const float* base = xb + (size_t)t * d * F_NP + r;
#pragma unroll
    for (int k = 0; k < F_XCH; ++k) {
        const int cc = 2 * k + h;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int l = 8 * cc + e;
            x[k][e] = l < d ? __ldg(base + (size_t)l * F_NP) : 0.0f;
        }
    }
}

__global__ void __launch_bounds__(F_THREADS, 1) contract_tcf_kernel(const TcfArgs a) {
    extern __shared__ __align__(1024) unsigned char tcf_raw[];
    unsigned char* sm = tcf_raw + ((1024u - (smem_u32(tcf_raw) & 1023u)) & 1023u);
    const int d = a.d, dp = tcf_dp(d), dp4 = dp / 4, ns = tcf_ns(d);
    const int SA = a.sa;
    const TcfSmem lay(d, a.gb, SA);
    const int stage_bytes = lay.stage_bytes;
    unsigned char* sP = sm + lay.P;
    unsigned char* sD = sm + lay.D;
    float* sA32 = reinterpret_cast<float*>(sm + lay.A32);
    float* sU32 = reinterpret_cast<float*>(sm + lay.U32);
    uint32_t* sQ = reinterpret_cast<uint32_t*>(sm + lay.Q);
    int* sCnt = reinterpret_cast<int*>(sm + lay.CNT);
    float* sZ = reinterpret_cast<float*>(sm + lay.ZS);
    float* sNrm = reinterpret_cast<float*>(sm + lay.NRM);
    int* sQc = reinterpret_cast<int*>(sm + lay.QC);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + lay.BARS);
    uint64_t* pfull = &bars[0];
    uint64_t* pempty = &bars[F_P_STAGES];
    uint64_t* tfull = &bars[2 * F_P_STAGES];
    uint64_t* tempty = &bars[2 * F_P_STAGES + F_NACC];
    uint64_t* dfull = &bars[2 * F_P_STAGES + 2 * F_NACC];
    uint64_t* dempty = dfull + 1;
    uint64_t* udone = dfull + 2;
    uint64_t* aconv = dfull + 3;               // [F_SA_MAX] a = x - z of a tile written (converters)
    uint64_t* aempty = aconv + F_SA_MAX;       // [F_SA_MAX] refinements of the tile done (epilogue)
    uint64_t* ufull = aempty + F_SA_MAX;       // unit's U32 rows landed
    uint64_t* epidone = ufull + 1;             // epilogue finished a unit (U32 reusable)
    uint32_t* sTaddr = reinterpret_cast<uint32_t*>(sm + lay.TADDR);
    const uint32_t row_bytes = (uint32_t)lay.row_bytes;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int units = a.Qb * a.groups * a.chunks;

    for (int i = tid; i < F_P_STAGES * stage_bytes / 16; i += F_THREADS)
        reinterpret_cast<uint4*>(sP)[i] = make_uint4(0u, 0u, 0u, 0u);
    for (int c = tid; c < F_GB_MAX * F_MD * 4; c += F_THREADS) sCnt[c] = 0;
    if (tid < 2) sQc[tid] = 0;
    if (tid == 0) {
        for (int s = 0; s < F_P_STAGES; ++s) {
            mbar_init(&pfull[s], F_CONV_WARPS);
            mbar_init(&pempty[s], 1);
        }
        for (int b = 0; b < F_NACC; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], F_EPI_WARPS);
        }
        mbar_init(dfull, 1);
        mbar_init(dempty, 1);
        mbar_init(udone, 1);
        for (int s = 0; s < F_SA_MAX; ++s) {
            mbar_init(&aconv[s], F_CONV_WARPS);
            mbar_init(&aempty[s], 1);
        }
        mbar_init(ufull, 1);
        mbar_init(epidone, 1);
        fence_mbar_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(sTaddr)),
                     "r"(F_TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (*sTaddr != 0u) __trap();  // the only CTA on the SM owns columns [0, 512)

    if (warp == 0) {
        // ------------------------------ producer: direction blocks, then U32 rows
        uint32_t gph = 0, it = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x, ++it) {
            const TcfUnit w = tcf_unit(a, u);
            const int b0 = w.grp * a.gb;
            const unsigned char* src = a.uop + ((size_t)w.q * a.NB + b0) * stage_bytes;
            for (int b = 0; b < w.nbg; ++b, ++gph) {
                if (gph > 0) mbar_wait_sleep(dempty, (gph - 1) & 1u);
                expect_tx_elect(dfull, (uint32_t)stage_bytes);
                tma_load_elect(sD, src + (size_t)b * stage_bytes, (uint32_t)stage_bytes, dfull);
                __syncwarp();
            }
            if (it > 0) mbar_wait_sleep(epidone, (it - 1) & 1u);  // previous unit's refinements are done
            const uint32_t ub = (uint32_t)w.nbg * F_MD * row_bytes;
            expect_tx_elect(ufull, ub);
            tma_load_elect(sU32, a.u32r + ((size_t)w.q * a.mpad + (size_t)b0 * F_MD) * dp, ub, ufull);
            __syncwarp();
        }
    } else if (warp == 1) {
        switch (ns) {
            case 1: tcf_mma_issue<1>(a, units, sP, sD, pfull, pempty, dfull, dempty, tfull, tempty, udone); break;
            case 2: tcf_mma_issue<2>(a, units, sP, sD, pfull, pempty, dfull, dempty, tfull, tempty, udone); break;
            case 3: tcf_mma_issue<3>(a, units, sP, sD, pfull, pempty, dfull, dempty, tfull, tempty, udone); break;
            case 4: tcf_mma_issue<4>(a, units, sP, sD, pfull, pempty, dfull, dempty, tfull, tempty, udone); break;
            default: tcf_mma_issue<5>(a, units, sP, sD, pfull, pempty, dfull, dempty, tfull, tempty, udone); break;
        }
    } else if (warp < F_EPI_WARP0) {
        // ----- converters: thread (point r, chunk parity h) owns the 8-coordinate
        // chunks cc = h, h + 2, ... of its point; x is prefetched one tile ahead
        // into registers (coalesced loads of the tile-blocked dataset)
        const int ct = tid - F_CONV_WARP0 * 32;
        const int r = ct & (F_NP - 1), h = ct >> 7;
        const int cd = d >> 3;  // chunk holding the threshold slot (K index d)
        uint32_t it = 0, gtile = 0;
        float xn[F_XCH][8];
        int u = blockIdx.x;
        TcfUnit w{};
        int t = 0;
        if (u < units) {
            w = tcf_unit(a, u);
            t = w.t0;
            load_x_chunks(a.xb, t, d, r, h, xn);
        }
        for (; u < units;) {
            float* zs = sZ + (it & 1u) * 64;
            if (t == w.t0) {
                if (ct < 64) zs[ct] = ct < d ? __ldg(a.zq + (size_t)w.q * d + ct) : 0.0f;
                named_bar(2, F_CONV_THREADS);
            }
            // next tile (possibly of the next unit) for the prefetch
            int un = u, tn = t + 1;
            TcfUnit wn = w;
            if (tn >= w.t1) {
                un = u + gridDim.x;
                if (un < units) {
                    wn = tcf_unit(a, un);
                    tn = wn.t0;
                }
            }
            float xc[F_XCH][8];
#pragma unroll
            for (int k = 0; k < F_XCH; ++k)
#pragma unroll
                for (int e = 0; e < 8; ++e) xc[k][e] = xn[k][e];
            if (un < units) load_x_chunks(a.xb, tn, d, r, h, xn);

            const uint32_t s = gtile % (uint32_t)SA;
            const uint32_t ps = gtile % F_P_STAGES;
            // a = x - z (contract.cu: v.x -= zk), FP32 round to nearest; coordinates >= d are 0
            float ss = 0.0f;
#pragma unroll
            for (int k = 0; k < F_XCH; ++k) {
                const int cc = 2 * k + h;
                if (8 * cc < d) {
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const int l = 8 * cc + e;
                        const float v = l < d ? __fsub_rn(xc[k][e], zs[l]) : 0.0f;
                        xc[k][e] = v;
                        ss = fmaf(v, v, ss);
                    }
                }
            }
            float* nrm = sNrm + (gtile & 1u) * 2 * F_NP;
            nrm[h * F_NP + r] = ss;
            if (gtile >= (uint32_t)SA) mbar_wait(&aempty[s], ((gtile / SA) - 1) & 1u);  // slot's refinements done
            // a kept for the refinement: row r of the slot, [p][dp] row-major
            float* arow = sA32 + (size_t)s * F_NP * dp + (size_t)r * dp;
#pragma unroll
            for (int k = 0; k < F_XCH; ++k) {
                const int cc = 2 * k + h;
                if (8 * cc < dp)
                    *reinterpret_cast<float4*>(arow + 8 * cc) = make_float4(xc[k][0], xc[k][1], xc[k][2], xc[k][3]);
                if (8 * cc + 4 < dp)
                    *reinterpret_cast<float4*>(arow + 8 * cc + 4) = make_float4(xc[k][4], xc[k][5], xc[k][6], xc[k][7]);
            }
            named_bar(2, F_CONV_THREADS);  // both halves' |a|^2 visible
            const float nrm2 = nrm[r] + nrm[F_NP + r];
            const bool real = (int64_t)t * F_NP + r < a.n;
            const bool decisive = real && nrm2 > 0x1.0p-100f && nrm2 < 0x1.0p100f;
            const float sc = decisive ? TCF_CB * rsqrtf(nrm2) : 0.0f;
            const __half slot = __float2half_rn(real ? 1.0f : 4.0f);
            if (gtile >= F_P_STAGES) mbar_wait(&pempty[ps], ((gtile / F_P_STAGES) - 1) & 1u);
            unsigned char* P = sP + ps * stage_bytes + r * 16;
#pragma unroll
            for (int k = 0; k < F_MAXCH; ++k) {
                const int cc = 2 * k + h;
                if (cc <= cd) {
                    uint32_t hw[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float x0 = k < F_XCH ? xc[k < F_XCH ? k : 0][2 * e] : 0.0f;
                        const float x1 = k < F_XCH ? xc[k < F_XCH ? k : 0][2 * e + 1] : 0.0f;
                        const float2 p = __fmul2_rn(make_float2(x0, x1), make_float2(sc, sc));
                        __half2 hv = __floats2half2_rn(p.x, p.y);  // coordinates >= d: a = 0
                        if (cc == cd) {
                            if (8 * cc + 2 * e == d) hv.x = slot;
                            if (8 * cc + 2 * e + 1 == d) hv.y = slot;
                        }
                        hw[e] = *reinterpret_cast<uint32_t*>(&hv);
                    }
                    *reinterpret_cast<uint4*>(P + cc * (F_NP * 16)) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
                }
            }
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&pfull[ps]);
                mbar_arrive(&aconv[s]);
            }
            ++gtile;
            if (t + 1 < w.t1) {
                ++t;
            } else {
                u = un;
                w = wn;
                t = tn;
                ++it;
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue
        const int ct = tid - F_EPI_WARP0 * 32;          // 0..127
        const int quarter = warp & 3;                   // TMEM lane quarter (32 directions)
        const int jl = 32 * quarter + lane;             // direction within the block
        const uint32_t lane_base = (uint32_t)(32 * quarter) << 16;
        uint32_t it = 0, gacc = 0, gtile = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x, ++it) {
            const TcfUnit w = tcf_unit(a, u);
            int cneg[F_GB_MAX], camb[F_GB_MAX];
#pragma unroll
            for (int b = 0; b < F_GB_MAX; ++b) cneg[b] = camb[b] = 0;
            mbar_wait(ufull, it & 1u);  // this unit's FP32 direction rows
            for (int t = w.t0; t < w.t1; ++t, ++gtile) {
                const uint32_t s = gtile % (uint32_t)SA;
                // ambiguous points per block and 64-point half: bit 2k / 2k+1 of
                // word 2 hf + (0|1) = point 64 hf + 32 (0|1) + k / + 16 + k
                uint32_t amk[F_GB_MAX][4];
                int mine = 0;
#pragma unroll
                for (int b = 0; b < F_GB_MAX; ++b) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) amk[b][k] = 0u;
                    if (b < w.nbg) {
                        const uint32_t buf = gacc % F_NACC;
                        mbar_wait(&tfull[buf], (gacc / F_NACC) & 1u);
                        ++gacc;
                        tc_fence_after();
#pragma unroll
                        for (int hf = 0; hf < 2; ++hf) {
                            const uint32_t tb = lane_base + buf * F_NP + (uint32_t)(hf * 64);
                            uint32_t y0[32], y1[32];
                            tmem_ld32(tb, y0);
                            tmem_ld32(tb + 32, y1);
                            tmem_wait_ld();
                            if (hf == 1) {
                                tc_fence_before();
                                __syncwarp();
                                if (lane == 0) mbar_arrive(&tempty[buf]);
                            }
                            // bits (31, 30) of 16 accumulators per register: 1x negative,
                            // 01 positive, 00 ambiguous (value k at bits 2k+1, 2k)
                            uint32_t am[4];
#pragma unroll
                            for (int qd = 0; qd < 4; ++qd) {
                                uint32_t m = 0u;
#pragma unroll
                                for (int k = 15; k >= 0; --k) {
                                    const uint32_t v = qd < 2 ? y0[16 * qd + k] : y1[16 * (qd - 2) + k];
                                    m = __funnelshift_l(v, m, 2);
                                }
                                cneg[b] += __popc(m & 0xAAAAAAAAu);
                                am[qd] = ~(m | (m >> 1)) & 0x55555555u;
                            }
                            amk[b][2 * hf] = am[0] | (am[1] << 1);
                            amk[b][2 * hf + 1] = am[2] | (am[3] << 1);
                            const int c = __popc(amk[b][2 * hf]) + __popc(amk[b][2 * hf + 1]);
                            camb[b] += c;
                            mine += c;
                        }
                    }
                }
                // ---- queue this tile's ambiguous pairs (all 8 warps share one queue)
                int incl = mine;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int v = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += v;
                }
                int base = 0;
                if (lane == 31) base = atomicAdd(&sQc[gtile & 1u], incl);
                base = __shfl_sync(0xffffffffu, base, 31) + incl - mine;
                mbar_wait(&aconv[s], (gtile / SA) & 1u);  // a = x - z of this tile is in the slot
                const float* slotA = sA32 + (size_t)s * F_NP * dp;
#pragma unroll
                for (int b = 0; b < F_GB_MAX; ++b) {
#pragma unroll
                    for (int hf = 0; hf < 2; ++hf) {
                        uint64_t mk = (uint64_t)amk[b][2 * hf] | ((uint64_t)amk[b][2 * hf + 1] << 32);
                        while (mk) {
                            const int tb = __ffsll((long long)mk) - 1;
                            mk &= mk - 1ull;
                            const int p = hf * 64 + ((tb >> 5) << 5) + ((tb & 31) >> 1) + ((tb & 1) << 4);
                            if (base < F_QCAP) {
                                sQ[base] = ((uint32_t)b << 16) | ((uint32_t)jl << 8) | (uint32_t)p;
                            } else {  // queue full (degenerate data): refine in place
                                const float y =
                                    refine_dot(slotA + (size_t)p * dp, sU32 + (size_t)(b * F_MD + jl) * dp, dp4);
                                if (y < 0.0f) atomicAdd(&sCnt[(b * F_MD + jl) * 4 + 2], 1);
                                else if (y > 0.0f) atomicAdd(&sCnt[(b * F_MD + jl) * 4 + 3], 1);
                            }
                            ++base;
                        }
                    }
                }
                named_bar(1, F_EPI_THREADS);  // the tile's queue is complete
                if (ct == 0) sQc[(gtile + 1) & 1u] = 0;  // next tile's counter (last read a tile ago)
                int total = sQc[gtile & 1u];
                if (total > F_QCAP) total = F_QCAP;
                for (int i = ct; i < total; i += F_EPI_THREADS) {
                    const uint32_t e = sQ[i];
                    const int b = (int)(e >> 16), j = (int)((e >> 8) & 255u), p = (int)(e & 255u);
                    const float y = refine_dot(slotA + (size_t)p * dp, sU32 + (size_t)(b * F_MD + j) * dp, dp4);
                    if (y < 0.0f) atomicAdd(&sCnt[(b * F_MD + j) * 4 + 2], 1);
                    else if (y > 0.0f) atomicAdd(&sCnt[(b * F_MD + j) * 4 + 3], 1);
                }
                named_bar(1, F_EPI_THREADS);  // refinements done: slot and queue reusable
                if (ct == 0) mbar_arrive(&aempty[s]);
            }
            // ---- unit end: counts per direction
#pragma unroll
            for (int b = 0; b < F_GB_MAX; ++b)
                if (b < w.nbg) {
                    atomicAdd(&sCnt[(b * F_MD + jl) * 4 + 0], cneg[b]);
                    atomicAdd(&sCnt[(b * F_MD + jl) * 4 + 1], camb[b]);
                }
            named_bar(1, F_EPI_THREADS);
            const int64_t r1 = (int64_t)w.t1 * F_NP < a.n ? (int64_t)w.t1 * F_NP : a.n;
            const int valid = (int)(r1 - (int64_t)w.t0 * F_NP);
            int* dst = a.counts + (size_t)w.q * a.mpad * 2;
            const int j0 = w.grp * a.gb * F_MD;
            for (int c = ct; c < w.nbg * F_MD; c += F_EPI_THREADS) {
                const int4 v = reinterpret_cast<int4*>(sCnt)[c];
                reinterpret_cast<int4*>(sCnt)[c] = make_int4(0, 0, 0, 0);
                if (j0 + c >= a.m) continue;
                const int lt = v.x + v.z;                // decisive negatives + refined negatives
                const int gt = valid - v.x - v.y + v.w;  // decisive positives + refined positives
                if (lt) atomicAdd(dst + 2 * (j0 + c) + 0, lt);
                if (gt) atomicAdd(dst + 2 * (j0 + c) + 1, gt);
            }
            named_bar(1, F_EPI_THREADS);
            if (ct == 0) mbar_arrive(epidone);
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(0u), "r"(F_TMEM_COLS));
}

// (gb, S_A) that fit shared memory: prefer 3 direction blocks per unit (fewer
// conversions per tile) and 3 point-row slots (TMA latency hidden)
static bool tcf_pick(int d, int& gb, int& sa) {
    const int cand[][2] = {{3, 3}, {2, 4}, {2, 3}, {1, 4}, {1, 3}, {1, 2}};
    for (const auto& c : cand) {
        const TcfSmem lay(d, c[0], c[1]);
        if (lay.total <= F_SMEM_LIMIT) {
            gb = c[0];
            sa = c[1];
            return true;
        }
    }
    return false;
}

cudaError_t launch_contract_tcf(TcfArgs a, int sms, cudaStream_t st) {
    if (a.d < 1 || a.d > 64) return cudaErrorInvalidValue;
    int gb = 1, sa = 2;
    if (!tcf_pick(a.d, gb, sa)) return cudaErrorInvalidValue;
    a.gb = gb;
    a.sa = sa;
    a.groups = (a.NB + gb - 1) / gb;
    const int64_t base = (int64_t)a.Qb * a.groups;
    int64_t chunks = ((int64_t)16 * sms + base - 1) / base;
    if (chunks < 1) chunks = 1;
    if (chunks > a.tiles) chunks = a.tiles;
    a.tiles_per_chunk = (a.tiles + chunks - 1) / chunks;
    a.chunks = (int)((a.tiles + a.tiles_per_chunk - 1) / a.tiles_per_chunk);
    const TcfSmem lay(a.d, gb, sa);
    cudaError_t e = cudaFuncSetAttribute(contract_tcf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, lay.total);
    if (e != cudaSuccess) return e;
    const int64_t units = (int64_t)a.Qb * a.groups * a.chunks;
    if (units == 0) return cudaSuccess;
    if (units > INT32_MAX / 2 || a.tiles > INT32_MAX / 2) return cudaErrorInvalidValue;  // 32-bit unit math
    const int grid = (int)(units < sms ? units : sms);
    contract_tcf_kernel<<<grid, F_THREADS, lay.total, st>>>(a);
    return cudaGetLastError();
}

}  // namespace rrs
