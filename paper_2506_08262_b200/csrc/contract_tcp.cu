// contract_tcp.cu -- K2 on the tensor cores for 64 < d <= 256 with a
// PRE-SPLIT point operand: the wide kernel (contract_tcw.cu) without its
// converter warps.
//
// contract_tcw.cu forms a = x - z, scales and splits every point tile into
// FP16 hi/lo once per (tile, direction block): at config 5 (d = 200, one
// 208-column direction block per unit) the converters re-split each tile for
// each of a query's 8 blocks and issue ~4x the instructions of the epilogue.
// Here the split is query-independent and done once per dataset
// (launch_presplit): B_i = x_i s_i = bh + bl in the tc_layout, with the
// per-point power of two s_i = 2^(14 - E_i), max_l |x_il| < 2^E_i, so
//   acc_ij = sum_l (uh_jl bh_il + uh bl + ul bh) ~= <u_j, x_i> s_i 2^15
// and the query enters the EPILOGUE through the per-direction FP64 shift
// Delta_j = <u_j, c - z> (direction_shift_kernel; c = 0 for the halfspace
// counts, the dataset centre m for the centred projection store):
//   y_ij = acc_ij inv_i + Delta_j,   inv_i = 2^(E_i - 29)   (exact rescale)
// one FFMA per element whose sign is counted (Delta + 0.0f: no -0).  Errors:
// 2^-22 |x_i| per split term, FP32 accumulation (as contract_tcw, relative to
// |<u, x_i>|) and 2^-24 |Delta_j| <= 2^-24 |z| -- all inside the tie zone
// 1e-6 max(|x_i|, |z|) of the halfspace contract.
// The query's own row (and every row FP32-equal to z) is an exact tie in the
// reference; its y here is only ~0, so those rows are excluded BY INDEX from
// the per-query list of launch_coincide_list32 (the converter kernel excludes
// them by a == 0), and #(y > 0) = valid - coinciding - #(y < 0) as before.
//
// Layout (M = 128 directions on TMEM lanes, N = 128 points, K = 16 per MMA):
// one direction block per unit resident in TMEM (8 ns columns), two FP32
// accumulators when 8 ns <= 256; per (tile, slice) one TMA of the slice's
// pre-split bytes (32 KB for a full slice, up to 36 KB for the last) into a
// 4-deep stage ring and
// 3 Q + R MMAs (kernels.h tc_mma_steps); the per-point inv_i (512 B per tile)
// rides on the tile's first slice into an 8-deep ring read by the epilogue.
// Warp roles: 0 direction-slice producer, 1 TMEM allocator + MMA issuer,
// 2 point-operand producer, 3-10 epilogue (no converters).
// Work units (chunk of tiles, query, block), chunk-major as in contract_tcw.
// Replaces _kernels.pyx:120-199 (projection) + 270-289 (halfspace_span).
#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

#include <cuda_fp16.h>

#ifndef RRS_FORCE_SINGLE_ACC
#define RRS_FORCE_SINGLE_ACC 0
#endif

namespace rrs {

namespace {

constexpr int P_EPI_WARP0 = 3;
constexpr int P_EPI_WARPS = 8;
constexpr int P_EPI_THREADS = P_EPI_WARPS * 32;
constexpr int P_THREADS = (P_EPI_WARP0 + P_EPI_WARPS) * 32;  // 352
constexpr int P_MAXD = 256;
constexpr int P_MD = 128;
constexpr int P_NP = 128;
constexpr int P_STAGES = 4;
constexpr int P_STAGE = TC_SLICE_NS_MAX * 4096;  // any slice of a tile (36 KB: a last slice may hold 9 steps)
constexpr int P_DSTEPS = 4;                  // K steps of A per staging load
constexpr int P_IRING = 8;                   // per-point inv ring (tiles)
constexpr uint32_t P_TMEM_COLS = 512;
constexpr uint32_t P_ACC = 128;

struct PSmem {
    int P, D, CNT, INV, COIN, STG, BARS, TADDR, total;
    static constexpr int NBARS = 2 * P_STAGES + 2 + 2 + 3;
    __host__ __device__ explicit PSmem(bool store) {
        P = 0;
        D = P + P_STAGES * P_STAGE;
        CNT = D + P_DSTEPS * 4096;          // uint32 [128]
        INV = CNT + P_MD * 4;               // float [P_IRING][128]
        COIN = INV + P_IRING * P_NP * 4;    // int [TCP_COIN_MAX]
        STG = COIN + TCP_COIN_MAX * 4;      // float [8 warps][32][33] (STORE)
        BARS = STG + (store ? P_EPI_WARPS * 32 * 33 * 4 : 0);
        TADDR = BARS + NBARS * 8;
        total = TADDR + 16 + 1024;
    }
};

struct PUnit {
    int q, blk;
    int64_t t0, t1;
};

__device__ __forceinline__ PUnit p_unit(const TcArgs& a, int64_t u) {
    PUnit r;
    const int64_t per_c = (int64_t)a.Qb * a.jbn;
    const int64_t c = u / per_c;
    const int64_t rem = u - c * per_c;
    r.q = (int)(rem / a.jbn);
    r.blk = a.jb0 + (int)(rem - (int64_t)r.q * a.jbn);
    r.t0 = c * a.tiles_per_chunk;
    r.t1 = r.t0 + a.tiles_per_chunk < a.tiles ? r.t0 + a.tiles_per_chunk : a.tiles;
    return r;
}

// first unit >= u of this CTA's stride whose query is still live (early exit)
__device__ __forceinline__ int64_t p_next(const TcArgs& a, int64_t u, int64_t units) {
    if (a.done) {
        const int64_t per_c = (int64_t)a.Qb * a.jbn;
        while (u < units && a.done[(u % per_c) / a.jbn]) u += gridDim.x;
    }
    return u;
}

__device__ __forceinline__ int p_slice_ns(const TcLayout& L, int s) {
    return s < L.full ? TC_SLICE_NS : L.ns - TC_SLICE_NS * L.full;
}

}  // namespace

template <bool STORE>
__global__ void __launch_bounds__(P_THREADS, 1) contract_tcp_kernel(const TcArgs a) {
    extern __shared__ __align__(1024) unsigned char p_raw[];
    unsigned char* sm = p_raw + ((1024u - (smem_u32(p_raw) & 1023u)) & 1023u);
    const int d = a.d;
    const TcLayout L = tc_layout(d);
    const int S = L.full + 1;
    const bool dbl = 8 * L.ns <= 256 && !RRS_FORCE_SINGLE_ACC;  // two accumulator buffers fit beside A
    const uint32_t a_base = dbl ? 2 * P_ACC : P_ACC;
    const PSmem lay(STORE);
    unsigned char* sP = sm + lay.P;
    unsigned char* sD = sm + lay.D;
    uint32_t* sCnt = reinterpret_cast<uint32_t*>(sm + lay.CNT);
    float* sInv = reinterpret_cast<float*>(sm + lay.INV);
    int* sCoin = reinterpret_cast<int*>(sm + lay.COIN);
    float* sStg = reinterpret_cast<float*>(sm + lay.STG);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + lay.BARS);
    uint64_t* pfull = &bars[0];                  // [P_STAGES] slice landed (TMA tx)
    uint64_t* pempty = &bars[P_STAGES];          // [P_STAGES] its MMAs completed
    uint64_t* tfull = &bars[2 * P_STAGES];       // [2] accumulator ready
    uint64_t* tempty = &bars[2 * P_STAGES + 2];  // [2] accumulator drained
    uint64_t* dfull = &bars[2 * P_STAGES + 4];
    uint64_t* dempty = &bars[2 * P_STAGES + 5];
    uint64_t* udone = &bars[2 * P_STAGES + 6];
    uint32_t* sTaddr = reinterpret_cast<uint32_t*>(sm + lay.TADDR);
    const size_t tile_bytes = (size_t)L.ns * 4096;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t units = (int64_t)a.Qb * a.jbn * a.chunks;

    for (int c = tid; c < P_MD; c += P_THREADS) sCnt[c] = 0u;
    if (tid == 0) {
        for (int s = 0; s < P_STAGES; ++s) {
            mbar_init(&pfull[s], 1);
            mbar_init(&pempty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], P_EPI_WARPS);
        }
        mbar_init(dfull, 1);
        mbar_init(dempty, 1);
        mbar_init(udone, 1);
        fence_mbar_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(sTaddr)),
                     "r"(P_TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (*sTaddr != 0u) __trap();
    constexpr uint32_t tmem = 0u;

    if (warp == 0) {
        // ----------------------- producer: the unit's direction block, DSTEPS K steps at a time
        uint32_t g = 0;
        for (int64_t u = p_next(a, blockIdx.x, units); u < units; u = p_next(a, u + gridDim.x, units)) {
            const PUnit w = p_unit(a, u);
            const unsigned char* src = a.uop + ((size_t)w.q * a.NB + w.blk) * tile_bytes;
            for (int k0 = 0; k0 < L.ns; k0 += P_DSTEPS, ++g) {
                const int nst = L.ns - k0 < P_DSTEPS ? L.ns - k0 : P_DSTEPS;
                if (g > 0) mbar_wait_sleep(dempty, (g - 1) & 1u);
                expect_tx_elect(dfull, (uint32_t)nst * 4096u);
                tma_load_elect(sD, src + (size_t)k0 * 4096, (uint32_t)nst * 4096u, dfull);
                __syncwarp();
            }
        }
    } else if (warp == 1) {
        // -------------------------------------------------------- MMA issuer
        const uint32_t idesc = (1u << 4) | ((uint32_t)(P_NP >> 3) << 17) | ((uint32_t)(P_MD >> 4) << 24);
        uint32_t it = 0, g = 0, gs = 0, gacc = 0;
        for (int64_t u = p_next(a, blockIdx.x, units); u < units; u = p_next(a, u + gridDim.x, units), ++it) {
            const PUnit w = p_unit(a, u);
            for (int k0 = 0; k0 < L.ns; k0 += P_DSTEPS, ++g) {
                const int nst = L.ns - k0 < P_DSTEPS ? L.ns - k0 : P_DSTEPS;
                mbar_wait_sleep(dfull, g & 1u);
                if (k0 == 0 && it > 0) mbar_wait(udone, (it - 1) & 1u);  // previous unit done with A
                tc_fence_after();
                tmem_cp_dirblock(tmem + a_base + 8u * k0, umma_desc(smem_u32(sD), 2048, 128), nst);
                mma_commit_elect(dempty);
            }
            for (int64_t t = w.t0; t < w.t1; ++t, ++gacc) {
                const uint32_t buf = dbl ? (gacc & 1u) : 0u;
                if (dbl) {
                    if (gacc >= 2) mbar_wait(&tempty[buf], ((gacc >> 1) - 1) & 1u);
                } else if (gacc >= 1) {
                    mbar_wait(&tempty[0], (gacc - 1) & 1u);
                }
                for (int s = 0; s < S; ++s, ++gs) {
                    const uint32_t st = gs % P_STAGES;
                    mbar_wait(&pfull[st], (gs / P_STAGES) & 1u);
                    tc_fence_after();
                    const uint32_t aT = tmem + a_base + 8u * TC_SLICE_NS * s;
                    const uint64_t bd = umma_desc(smem_u32(sP) + st * P_STAGE, 2048, 128);
                    if (elect_one()) {
                        if (s < L.full) mma_split_seq<4, 0>(tmem + buf * P_ACC, aT, bd, idesc, s == 0 ? 0u : 1u);
                        else mma_split_seq_rt(L.q16, L.rsteps, tmem + buf * P_ACC, aT, bd, idesc, s == 0 ? 0u : 1u);
                    }
                    __syncwarp();
                    mma_commit_elect(&pempty[st]);
                }
                mma_commit_elect(&tfull[buf]);
            }
            mma_commit_elect(udone);
        }
    } else if (warp == 2) {
        // ------------------- producer: pre-split slices (+ the tile's inv on its first slice)
        uint32_t gs = 0, gtile = 0;
        for (int64_t u = p_next(a, blockIdx.x, units); u < units; u = p_next(a, u + gridDim.x, units)) {
            const PUnit w = p_unit(a, u);
            for (int64_t t = w.t0; t < w.t1; ++t, ++gtile) {
                const unsigned char* tb = a.xps + (size_t)t * tile_bytes;
                for (int s = 0; s < S; ++s, ++gs) {
                    const uint32_t st = gs % P_STAGES;
                    const uint32_t bytes = (uint32_t)p_slice_ns(L, s) * 4096u;
                    if (gs >= P_STAGES) mbar_wait_sleep(&pempty[st], ((gs / P_STAGES) - 1) & 1u);
                    expect_tx_elect(&pfull[st], bytes + (s == 0 ? P_NP * 4u : 0u));
                    tma_load_elect(sP + st * P_STAGE, tb + (size_t)TC_SLICE_NS * s * 4096, bytes, &pfull[st]);
                    if (s == 0)
                        tma_load_elect(sInv + (gtile % P_IRING) * P_NP, a.pinv + (size_t)t * P_NP, P_NP * 4u,
                                       &pfull[st]);
                    __syncwarp();
                }
            }
        }
    } else if (STORE) {
        // ---------------------------------------------- epilogue: y' rows (STORE)
        const int quarter = warp & 3;
        const int half = (warp - P_EPI_WARP0) >> 2;
        const uint32_t lane_base = (uint32_t)(32 * quarter) << 16;
        const bool vec = (a.n & 3) == 0;
        float* stg = sStg + (warp - P_EPI_WARP0) * 32 * 33;
        uint32_t gacc = 0, gtile = 0;
        for (int64_t u = p_next(a, blockIdx.x, units); u < units; u = p_next(a, u + gridDim.x, units)) {
            const PUnit w = p_unit(a, u);
            const int jl = (w.blk - a.jb0) * P_MD + 32 * quarter + lane;
            const bool live = w.blk * P_MD + 32 * quarter + lane < a.m;
            float* yrow = a.y + ((size_t)w.q * a.jbn * P_MD + jl) * (size_t)a.n;
            float* y0 = a.y + ((size_t)w.q * a.jbn * P_MD + (size_t)(w.blk - a.jb0) * P_MD + 32 * quarter) * (size_t)a.n;
            const int rows_live = min(32, a.m - (w.blk * P_MD + 32 * quarter));
            for (int64_t t = w.t0; t < w.t1; ++t, ++gtile, ++gacc) {
                const uint32_t buf = dbl ? (gacc & 1u) : 0u;
                const uint32_t ph = dbl ? ((gacc >> 1) & 1u) : (gacc & 1u);
                mbar_wait(&tfull[buf], ph);
                tc_fence_after();
                const float* inv = sInv + (gtile % P_IRING) * P_NP + 64 * half;
                const int64_t p0 = t * P_NP + 64 * half;
                const uint32_t tb = tmem + lane_base + buf * P_ACC + (uint32_t)(half * 64);
#pragma unroll
                for (int part = 0; part < 2; ++part) {
                    uint32_t y[32];
                    tmem_ld32(tb + 32 * part, y);
                    tmem_wait_ld();
                    if (part == 1) {
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&tempty[buf]);
                    }
                    const int64_t pb = p0 + 32 * part;
                    if (vec && pb + 32 <= a.n) {
                        // transpose through the warp's tile: each store writes 4 rows x 128 B
#pragma unroll
                        for (int k = 0; k < 32; ++k) stg[lane * 33 + k] = __uint_as_float(y[k]) * inv[32 * part + k];
                        __syncwarp();
                        const int c4 = 4 * (lane & 7);
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            const int rr = (lane >> 3) + 4 * k;
                            if (rr < rows_live) {
                                const float* sv = stg + rr * 33 + c4;
                                *reinterpret_cast<float4*>(y0 + (size_t)rr * a.n + pb + c4) =
                                    make_float4(sv[0], sv[1], sv[2], sv[3]);
                            }
                        }
                        __syncwarp();
                    } else if (live) {
#pragma unroll
                        for (int k = 0; k < 32; ++k)
                            if (pb + k < a.n) yrow[pb + k] = __uint_as_float(y[k]) * inv[32 * part + k];
                    }
                }
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue: counts
        const int ct = tid - P_EPI_WARP0 * 32;
        const int quarter = warp & 3;
        const int half = (warp - P_EPI_WARP0) >> 2;
        const uint32_t lane_base = (uint32_t)(32 * quarter) << 16;
        uint32_t gacc = 0, gtile = 0;
        for (int64_t u = p_next(a, blockIdx.x, units); u < units; u = p_next(a, u + gridDim.x, units)) {
            const PUnit w = p_unit(a, u);
            // this unit's coinciding rows (exact ties, excluded by index)
            const int cn = a.coin_n[w.q] < TCP_COIN_MAX ? a.coin_n[w.q] : TCP_COIN_MAX;
            for (int k = ct; k < cn; k += P_EPI_THREADS) sCoin[k] = a.coin[(size_t)w.q * TCP_COIN_MAX + k];
            named_bar(1, P_EPI_THREADS);
            uint32_t zrows = 0u;
            for (int k = 0; k < cn; ++k) {
                const int64_t idx = sCoin[k];
                zrows += (idx >= w.t0 * P_NP && idx < w.t1 * P_NP) ? 1u : 0u;
            }
            const int j = w.blk * P_MD + 32 * quarter + lane;  // the thread's direction
            const float dl = (j < a.m ? (float)a.dshift[(size_t)w.q * a.m + j] : 0.0f) + 0.0f;
            uint32_t cnt = 0u;
            for (int64_t t = w.t0; t < w.t1; ++t, ++gtile, ++gacc) {
                const uint32_t buf = dbl ? (gacc & 1u) : 0u;
                const uint32_t ph = dbl ? ((gacc >> 1) & 1u) : (gacc & 1u);
                // kept points of the thread's 64 columns: rows < n, not coinciding
                const int64_t cb = t * P_NP + 64 * half;
                const int64_t rows = a.n - cb;
                uint32_t keep0 = rows >= 32 ? 0xFFFFFFFFu : rows <= 0 ? 0u : (1u << rows) - 1u;
                uint32_t keep1 = rows >= 64 ? 0xFFFFFFFFu : rows <= 32 ? 0u : (1u << (rows - 32)) - 1u;
                for (int k = 0; k < cn; ++k) {
                    const int64_t off = sCoin[k] - cb;
                    if (off >= 0 && off < 32) keep0 &= ~(1u << off);
                    else if (off >= 32 && off < 64) keep1 &= ~(1u << (off - 32));
                }
                mbar_wait(&tfull[buf], ph);
                tc_fence_after();
                const float4* iv = reinterpret_cast<const float4*>(sInv + (gtile % P_IRING) * P_NP + 64 * half);
                const uint32_t tb = tmem + lane_base + buf * P_ACC + (uint32_t)(half * 64);
                uint32_t y[32], m0 = 0u, m1 = 0u;
                tmem_ld32(tb, y);
                tmem_wait_ld();
                // y = acc inv + Delta: its sign bit, bit k = point cb + k
#pragma unroll
                for (int k = 7; k >= 0; --k) {
                    const float4 v = iv[k];
                    m0 = __funnelshift_l(__float_as_uint(fmaf(__uint_as_float(y[4 * k + 3]), v.w, dl)), m0, 1);
                    m0 = __funnelshift_l(__float_as_uint(fmaf(__uint_as_float(y[4 * k + 2]), v.z, dl)), m0, 1);
                    m0 = __funnelshift_l(__float_as_uint(fmaf(__uint_as_float(y[4 * k + 1]), v.y, dl)), m0, 1);
                    m0 = __funnelshift_l(__float_as_uint(fmaf(__uint_as_float(y[4 * k + 0]), v.x, dl)), m0, 1);
                }
                tmem_ld32(tb + 32, y);
                tmem_wait_ld();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[buf]);
#pragma unroll
                for (int k = 7; k >= 0; --k) {
                    const float4 v = iv[8 + k];
                    m1 = __funnelshift_l(__float_as_uint(fmaf(__uint_as_float(y[4 * k + 3]), v.w, dl)), m1, 1);
                    m1 = __funnelshift_l(__float_as_uint(fmaf(__uint_as_float(y[4 * k + 2]), v.z, dl)), m1, 1);
                    m1 = __funnelshift_l(__float_as_uint(fmaf(__uint_as_float(y[4 * k + 1]), v.y, dl)), m1, 1);
                    m1 = __funnelshift_l(__float_as_uint(fmaf(__uint_as_float(y[4 * k + 0]), v.x, dl)), m1, 1);
                }
                cnt += __popc(m0 & keep0) + __popc(m1 & keep1);
            }
            atomicAdd(sCnt + 32 * quarter + lane, cnt);
            named_bar(1, P_EPI_THREADS);  // all counts in; sCoin free for the next unit
            const int64_t r1 = w.t1 * P_NP < a.n ? w.t1 * P_NP : a.n;
            const int valid = (int)(r1 - w.t0 * P_NP);
            int* dst = a.counts + (size_t)w.q * a.mpad * 2;
            const int j0 = w.blk * P_MD;
            for (int c = ct; c < P_MD; c += P_EPI_THREADS) {
                const int lt = (int)sCnt[c];
                sCnt[c] = 0u;
                if (j0 + c >= a.m) continue;
                const int gtv = valid - (int)zrows - lt;
                if (lt) atomicAdd(dst + 2 * (j0 + c) + 0, lt);
                if (gtv) atomicAdd(dst + 2 * (j0 + c) + 1, gtv);
            }
            named_bar(1, P_EPI_THREADS);
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(P_TMEM_COLS));
}

template <bool STORE>
static cudaError_t launch_tcp(TcArgs a, int sms, cudaStream_t st) {
    if (a.d <= TC_SLICE || a.d > P_MAXD || a.xps == nullptr || a.pinv == nullptr) return cudaErrorInvalidValue;
    if (!STORE && (a.dshift == nullptr || a.coin == nullptr || a.coin_n == nullptr)) return cudaErrorInvalidValue;
    const PSmem lay(STORE);
    a.gb = 1;
    if (!STORE) {
        a.jb0 = 0;
        a.jbn = a.NB;
    }
    a.groups = a.jbn;
    // chunks: >= 4 units per SM, and chunks short enough that a wave's tiles stay in L2
    const int64_t base = (int64_t)a.Qb * a.jbn;
    int64_t chunks = (4ll * sms + base - 1) / base;
    const int64_t l2_tiles = (int64_t)(48ll << 20) / ((int64_t)tc_layout(a.d).ns * 4096);  // ~48 MB per chunk
    const int64_t min_chunks = (a.tiles + l2_tiles - 1) / (l2_tiles > 0 ? l2_tiles : 1);
    if (chunks < min_chunks) chunks = min_chunks;
    if (chunks < 1) chunks = 1;
    if (chunks > a.tiles) chunks = a.tiles;
    a.tiles_per_chunk = (a.tiles + chunks - 1) / chunks;
    a.chunks = (int)((a.tiles + a.tiles_per_chunk - 1) / a.tiles_per_chunk);
    const size_t smem = (size_t)lay.total;
    cudaError_t e =
        cudaFuncSetAttribute(contract_tcp_kernel<STORE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t units = base * a.chunks;
    if (units == 0) return cudaSuccess;
    const int grid = (int)(units < sms ? units : sms);
    contract_tcp_kernel<STORE><<<grid, P_THREADS, smem, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_contract_tcp(TcArgs a, int sms, cudaStream_t st) { return launch_tcp<false>(a, sms, st); }
cudaError_t launch_contract_tcp_store(TcArgs a, int sms, cudaStream_t st) { return launch_tcp<true>(a, sms, st); }

// ---------------------------------------------------------------- pre-split --
// B operand of every tile in the tc_layout (kernels.h) from the tile-blocked FP32
// rows xb [T][d][128]: v = x s_i (exact: s_i a power of two), bh = fp16(v),
// bl = fp16(v - bh); aligned K chunks hold the hi / lo terms of 8 coordinates,
// the remainder chunks the products h, l, h of the last coordinates.  One
// thread per point, 16-byte chunks written point-consecutive (coalesced).
__global__ void __launch_bounds__(128) presplit_kernel(const float* __restrict__ xb, const float* __restrict__ rowmax,
                                                       int64_t n, int d, unsigned char* __restrict__ xps,
                                                       float* __restrict__ pinv) {
    const int64_t t = blockIdx.x;
    const int r = threadIdx.x;
    const TcLayout L = tc_layout(d);
    const float mx = (t * BM + r < n) ? rowmax[t * BM + r] : 0.0f;
    float s = 0.0f, inv = 0.0f;
    if (mx > 0.0f) {
        int E = (int)((__float_as_uint(mx) >> 23) & 0xFF) - 126;  // mx < 2^E
        if (E < -100) E = -100;
        s = __uint_as_float((uint32_t)(127 + 14 - E) << 23);  // 2^(14 - E)
        inv = ldexpf(1.0f, E - 29);                           // 1 / (s 2^15)
    }
    pinv[t * BM + r] = inv;
    const float* X = xb + (size_t)t * d * BM + r;
    unsigned char* out = xps + (size_t)t * L.ns * 4096 + (size_t)r * 16;
    for (int cc = 0; cc < 2 * L.ns; ++cc) {
        uint32_t w[4];
        bool lo;
        int c0;
        if (tc_chunk_run(L, cc, lo, c0)) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float v0 = X[(size_t)(c0 + 2 * e) * BM] * s, v1 = X[(size_t)(c0 + 2 * e + 1) * BM] * s;
                const __half2 hh = __floats2half2_rn(v0, v1);
                const float2 hf = __half22float2(hh);
                const __half2 ll = __floats2half2_rn(v0 - hf.x, v1 - hf.y);
                const __half2 pick = lo ? ll : hh;
                w[e] = *reinterpret_cast<const uint32_t*>(&pick);
            }
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                uint32_t pair = 0u;
#pragma unroll
                for (int hlf = 0; hlf < 2; ++hlf) {
                    int en, c;
                    tc_elem(L, 8 * cc + 2 * e + hlf, en, c);
                    if (c >= 0) {
                        const float v = X[(size_t)c * BM] * s;
                        const __half h = __float2half_rn(v);
                        const __half l = __float2half_rn(v - __half2float(h));
                        pair |= (uint32_t)__half_as_ushort(tc_b_lo(L, en, c) ? l : h) << (16 * hlf);
                    }
                }
                w[e] = pair;
            }
        }
        *reinterpret_cast<uint4*>(out + (size_t)cc * 2048) = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

cudaError_t launch_presplit(const float* xb, const float* rowmax, int64_t n, int d, int64_t tiles,
                            unsigned char* xps, float* pinv, cudaStream_t st) {
    if (tiles == 0) return cudaSuccess;
    presplit_kernel<<<(unsigned)tiles, BM, 0, st>>>(xb, rowmax, n, d, xps, pinv);
    return cudaGetLastError();
}

// rows FP32-equal to the query in every coordinate: the count (c0, int64) and
// up to TCP_COIN_MAX of their indices (any order); coin_n is the full count
__global__ void __launch_bounds__(BM) coincide_list32_kernel(const float* __restrict__ xb, const float* __restrict__ zq,
                                                             int64_t n, int d, int64_t tiles, long long* __restrict__ c0,
                                                             int* __restrict__ coin, int* __restrict__ coin_n) {
    const int q = blockIdx.y;
    const float* z = zq + (size_t)q * d;
    int cnt = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int64_t row = t * BM + threadIdx.x;
        if (row >= n) continue;
        const float* xr = xb + (size_t)t * d * BM + threadIdx.x;
        int l = 0;
        while (l < d && xr[(size_t)l * BM] == z[l]) ++l;
        if (l == d) {
            ++cnt;
            const int k = atomicAdd(coin_n + q, 1);
            if (k < TCP_COIN_MAX) coin[(size_t)q * TCP_COIN_MAX + k] = (int)row;
        }
    }
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(reinterpret_cast<unsigned long long*>(c0 + q), (unsigned long long)cnt);
}

cudaError_t launch_coincide_list32(const float* xb, const float* zq, int64_t n, int d, int64_t tiles, int Qb,
                                   long long* c0, int* coin, int* coin_n, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(c0, 0, (size_t)Qb * 8, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(coin_n, 0, (size_t)Qb * 4, st);
    if (e != cudaSuccess) return e;
    const int64_t blocks = tiles < 64 ? tiles : 64;
    coincide_list32_kernel<<<dim3((unsigned)blocks, (unsigned)Qb), BM, 0, st>>>(xb, zq, n, d, tiles, c0, coin, coin_n);
    return cudaGetLastError();
}

}  // namespace rrs
