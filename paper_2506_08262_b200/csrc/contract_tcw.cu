// contract_tcw.cu -- K2 on the tensor cores for 64 < d <= 256 ("wide"): the
// FP16 hi/lo split contraction of contract_tc.cu with the coordinates taken in
// slices of 64 (kernels.h tc_layout: full slices of 8 stored K steps / 12 MMAs
// + a last slice).
//
// Same arithmetic and result contract as contract_tc.cu (see there): a_il =
// x_il - z_l in FP32, a power-of-two scale per point, a*s = ah + al (FP16),
// u 2^15 = uh + ul, y s 2^15 ~= sum (uh al + ul ah + uh ah) accumulated in FP32
// in TMEM; counts of y < 0 per direction in the epilogue.  The per-point scale
// comes from the bound max_l |x_il| + max_l |z_l| >= max_l |a_il| (a dataset
// property, precomputed) instead of the exact maximum, so a point's slices can
// be converted one at a time; the split keeps 22 bits relative to each value
// (FP16 lo has its own exponent), so the bound only moves the subnormal floor
// (2^-25 of the scaled unit, i.e. ~2^-39 of the bound).
//
// Layout (M = 128 directions on TMEM lanes, N = 128 points, K = 16 per MMA):
//   one direction block per unit (its A operand: 8 ns TMEM columns, 208 at
//   d = 200, resident for the unit, loaded through a staging area); FP32
//   accumulator: two buffers of 128 columns when 8 ns <= 256 (every d <= 256
//   but 251..255), else one (the MMAs of the next tile wait for the epilogue
//   to drain it);
//   per (tile, slice): the raw FP32 rows [64 s, 64 s + 64) of the tile (TMA),
//   converted into one 32 KB point-operand stage (2 stages), 3 Q + R MMAs
//   accumulating into the tile's accumulator.
// Work units = (chunk of point tiles, query, direction block) with the chunk
// slowest-varying: the CTAs running at the same time read the same tiles, so
// the dataset (800 MB at config 5) streams from HBM about once per wave and
// is re-read from L2 by the other units.
// Warp roles as in contract_tc.cu: 0 direction-slice producer, 1 TMEM
// allocator + MMA issuer, 2 raw-tile producer, 3-10 converters, 11-18 epilogue.
#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

#include <cuda_fp16.h>

#ifndef RRS_FORCE_SINGLE_ACC
#define RRS_FORCE_SINGLE_ACC 0
#endif

namespace rrs {

namespace {

constexpr int W_CONV_WARP0 = 3;
#ifndef RRS_TCW_CONV_WARPS
#define RRS_TCW_CONV_WARPS 8
#endif
constexpr int W_CONV_WARPS = RRS_TCW_CONV_WARPS;  // 128 points x (W_CONV_WARPS / 4) coordinate groups
constexpr int W_GROUPS = W_CONV_WARPS / 4;            // threads per point
constexpr int W_CPT = TC_SLICE / W_GROUPS;             // coordinates per converter thread (16 or 32)
constexpr int W_CH = W_CPT / 8;                        // 8-coordinate chunks per thread
constexpr int W_CONV_THREADS = W_CONV_WARPS * 32;
constexpr int W_EPI_WARP0 = W_CONV_WARP0 + W_CONV_WARPS;
constexpr int W_EPI_WARPS = 8;
constexpr int W_EPI_THREADS = W_EPI_WARPS * 32;
constexpr int W_THREADS = (W_EPI_WARP0 + W_EPI_WARPS) * 32;  // 864 with 16 converter warps
constexpr int W_MAXD = 256;
constexpr int W_MD = 128;
constexpr int W_NP = 128;
constexpr int W_P_STAGES = 2;
constexpr int W_R_MAX = 4;
constexpr int W_STAGE = TC_SLICE_NS_MAX * 4096;  // any slice of a tile (36 KB: a last slice may hold 9 steps)
#ifndef RRS_TCW_DSTEPS
#define RRS_TCW_DSTEPS 4
#endif
constexpr int W_DSTEPS = RRS_TCW_DSTEPS;     // K steps of A per staging load (the rest of smem feeds the raw ring)
constexpr uint32_t W_TMEM_COLS = 512;
constexpr uint32_t W_ACC = 128;
constexpr int W_SMEM_LIMIT = 227 * 1024;

struct WSmem {
    int P, D, CNT, ZS, NZ, EXCL, INV, STG, BARS, TADDR, RAW, total, raw_stages;
    static constexpr int NBARS = 2 * W_P_STAGES + 2 + 2 + 3 + 2 * W_R_MAX;
    __host__ __device__ explicit WSmem(bool store) {
        P = 0;
        D = P + W_P_STAGES * W_STAGE;
        CNT = D + W_DSTEPS * 4096;               // uint32 [128]
        ZS = CNT + W_MD * 4;                     // float [2][256] (+ [2] max |z|)
        NZ = ZS + 2 * W_MAXD * 4 + 16;           // uint32 [8][W_GROUPS][4] nonzero ballots (tile ring)
        EXCL = NZ + 8 * W_GROUPS * 4 * 4;        // (unused)
        INV = EXCL + 8 * 4 * 4;                  // float [8][128] per-point 1 / (s 2^15) (STORE mode)
        STG = INV + 8 * W_NP * 4;                // float [8 warps][32][33] store transpose tiles (STORE mode)
        BARS = STG + (store ? W_EPI_WARPS * 32 * 33 * 4 : 0);
        TADDR = BARS + NBARS * 8;
        RAW = (TADDR + 16 + 1023) & ~1023;       // [64][128] floats per stage
        const int room = W_SMEM_LIMIT - 1024 - RAW;
        raw_stages = room / (TC_SLICE * W_NP * 4);
        if (raw_stages > W_R_MAX) raw_stages = W_R_MAX;
        total = RAW + raw_stages * TC_SLICE * W_NP * 4 + 1024;
    }
};

struct WUnit {
    int q, blk;
    int64_t t0, t1;
};

// units (chunk, query, block) over blocks [jb0, jb0 + jbn) (count mode: all NB)
__device__ __forceinline__ WUnit w_unit(const TcArgs& a, int64_t u) {
    WUnit r;
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
__device__ __forceinline__ int64_t w_next(const TcArgs& a, int64_t u, int64_t units) {
    if (a.done) {
        const int64_t per_c = (int64_t)a.Qb * a.jbn;
        while (u < units && a.done[(u % per_c) / a.jbn]) u += gridDim.x;
    }
    return u;
}

__device__ __forceinline__ int slice_width(int d, int s) {
    const int w = d - TC_SLICE * s;
    return w < TC_SLICE ? w : TC_SLICE;
}
__device__ __forceinline__ int slice_ns(const TcLayout& L, int s) {
    return s < L.full ? TC_SLICE_NS : L.ns - TC_SLICE_NS * L.full;
}

// The 3 q + r MMAs (K = 16 each) of one slice (q aligned groups, r remainder
// steps) into the accumulator, A / B K steps paired by kernels.h
// tc_mma_steps; the first one overwrites it when `first` (the tile's first
// slice), the rest accumulate.  (q, r) = (4, 0) for a full slice; a last
// slice of (3, 3) has as many MMAs as a full one but a different pairing.
__device__ __forceinline__ void mma_slice(uint32_t acc, uint32_t aT, uint64_t bd, uint32_t idesc, int q, int r,
                                          bool first) {
    if (elect_one()) {
        if (q == 4) mma_split_seq<4, 0>(acc, aT, bd, idesc, first ? 0u : 1u);
        else mma_split_seq_rt(q, r, acc, aT, bd, idesc, first ? 0u : 1u);
    }
    __syncwarp();
}

// One converter thread's W_CPT coordinates [W_CPT h, W_CPT h + W_CPT) of a slice
// of width ds: a = x - z (FP32, packed FADD2) into av; returns whether any a != 0.
// FULL (ds = 64): no masking.  Otherwise rows past ds hold stale data from a
// previous slice and are read as x = 0 (z is 0 there too; never stored).
template <bool FULL>
__device__ __forceinline__ bool w_load_slice(const float* X, const float* zh, int h, int ds, float2 (&av)[4 * W_CH]) {
    uint32_t bits = 0u;  // OR of |a| bit patterns: nonzero iff some a != 0
#pragma unroll
    for (int c = 0; c < W_CH; ++c) {
        if (FULL || 8 * (W_CH * h + c) < ds) {
            const float4 z0 = *reinterpret_cast<const float4*>(zh + 8 * c);
            const float4 z1 = *reinterpret_cast<const float4*>(zh + 8 * c + 4);
            const float2 nzv[4] = {make_float2(-z0.x, -z0.y), make_float2(-z0.z, -z0.w), make_float2(-z1.x, -z1.y),
                                   make_float2(-z1.z, -z1.w)};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int c0 = 8 * (W_CH * h + c) + 2 * e;
                float x0 = X[(8 * c + 2 * e) * W_NP], x1 = X[(8 * c + 2 * e + 1) * W_NP];
                if (!FULL) {
                    x0 = c0 < ds ? x0 : 0.0f;
                    x1 = c0 + 1 < ds ? x1 : 0.0f;
                }
                const float2 v = __fadd2_rn(make_float2(x0, x1), nzv[e]);
                av[4 * c + e] = v;
                bits |= (__float_as_uint(v.x) | __float_as_uint(v.y)) & 0x7FFFFFFFu;
            }
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) av[4 * c + e] = make_float2(0.0f, 0.0f);
        }
    }
    return bits != 0u;
}

// Scale, FP16 hi/lo split and placement at the slice's packed K positions
// (slice layout q16 / rem; FULL: q16 = 4, rem = 0, every chunk aligned).
template <bool FULL>
__device__ __forceinline__ void w_store_slice(unsigned char* P, const float2 (&av)[4 * W_CH], float scale, int h,
                                              int ds, int q16, int rem) {
    const int main_chunks = 2 * q16;
    const float2 sc2 = make_float2(scale, scale);
#pragma unroll
    for (int c = 0; c < W_CH; ++c) {
        const int cc = W_CH * h + c;
        if (!FULL && 8 * cc >= ds) continue;
        uint32_t hw[4], lw[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float2 v = __fmul2_rn(av[4 * c + e], sc2);
            const __half2 hh = __floats2half2_rn(v.x, v.y);
            const float2 hf = __half22float2(hh);
            const float2 res = __fadd2_rn(v, make_float2(-hf.x, -hf.y));
            hw[e] = *reinterpret_cast<const uint32_t*>(&hh);
            lw[e] = pack_half2(res.x, res.y);
        }
        if (FULL || cc < main_chunks) {
            // aligned: the hi and the lo terms of 8 coordinates (kernels.h tc_layout)
            const int mc = FULL ? 8 : main_chunks;
            *reinterpret_cast<uint4*>(P + cc * (W_NP * 16)) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
            *reinterpret_cast<uint4*>(P + (mc + cc) * (W_NP * 16)) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
        } else if (rem == 8 && 8 * cc == 16 * q16) {
            // a remainder of exactly 8 coordinates (d = 200's last slice): product p
            // fills the whole chunk 4 q16 + p -- three 16-byte stores, no scatter
            const uint4 hv = make_uint4(hw[0], hw[1], hw[2], hw[3]);
            *reinterpret_cast<uint4*>(P + (4 * q16) * (W_NP * 16)) = hv;
            *reinterpret_cast<uint4*>(P + (4 * q16 + 1) * (W_NP * 16)) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
            *reinterpret_cast<uint4*>(P + (4 * q16 + 2) * (W_NP * 16)) = hv;
        } else {
#pragma unroll 1
            for (int e = 0; e < 8; ++e) {
                const int cd = 8 * cc + e;
                if (cd >= ds) break;
                const int wi = e >> 1;
                const uint32_t hv = wi == 0 ? hw[0] : wi == 1 ? hw[1] : wi == 2 ? hw[2] : hw[3];
                const uint32_t lv = wi == 0 ? lw[0] : wi == 1 ? lw[1] : wi == 2 ? lw[2] : lw[3];
                const uint16_t hb = (uint16_t)((e & 1) ? (hv >> 16) : (hv & 0xFFFFu));
                const uint16_t lb = (uint16_t)((e & 1) ? (lv >> 16) : (lv & 0xFFFFu));
                int kk = 16 * q16 + cd;  // 32 q16 + (cd - 16 q16): product 0
#pragma unroll
                for (int pr = 0; pr < 3; ++pr, kk += rem)
                    *reinterpret_cast<uint16_t*>(P + (kk >> 3) * (W_NP * 16) + (kk & 7) * 2) = pr == 1 ? lb : hb;
            }
        }
    }
}

}  // namespace

template <bool STORE>
__global__ void __launch_bounds__(W_THREADS, 1) contract_tcw_kernel(const TcArgs a) {
    extern __shared__ __align__(1024) unsigned char w_raw[];
    unsigned char* sm = w_raw + ((1024u - (smem_u32(w_raw) & 1023u)) & 1023u);
    const int d = a.d;
    const TcLayout L = tc_layout(d);
    const int S = L.full + 1;                 // slices
    const bool dbl = 8 * L.ns <= 256 && !RRS_FORCE_SINGLE_ACC;  // two accumulator buffers fit beside A
    const uint32_t a_base = dbl ? 2 * W_ACC : W_ACC;
    const WSmem lay(STORE);
    unsigned char* sP = sm + lay.P;
    unsigned char* sD = sm + lay.D;
    uint32_t* sCnt = reinterpret_cast<uint32_t*>(sm + lay.CNT);
    float* sZ = reinterpret_cast<float*>(sm + lay.ZS);
    uint32_t* sNz = reinterpret_cast<uint32_t*>(sm + lay.NZ);
    float* sInv = reinterpret_cast<float*>(sm + lay.INV);
    float* sStg = reinterpret_cast<float*>(sm + lay.STG);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + lay.BARS);
    uint64_t* pfull = &bars[0];
    uint64_t* pempty = &bars[W_P_STAGES];
    uint64_t* tfull = &bars[2 * W_P_STAGES];
    uint64_t* tempty = &bars[2 * W_P_STAGES + 2];
    uint64_t* dfull = &bars[2 * W_P_STAGES + 4];
    uint64_t* dempty = &bars[2 * W_P_STAGES + 5];
    uint64_t* udone = &bars[2 * W_P_STAGES + 6];
    uint64_t* rfull = &bars[2 * W_P_STAGES + 7];
    uint64_t* rempty = &bars[2 * W_P_STAGES + 7 + W_R_MAX];
    uint32_t* sTaddr = reinterpret_cast<uint32_t*>(sm + lay.TADDR);
    float* sRaw = reinterpret_cast<float*>(sm + lay.RAW);
    const int RS = lay.raw_stages;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t units = (int64_t)a.Qb * a.jbn * a.chunks;

    for (int i = tid; i < W_P_STAGES * W_STAGE / 16; i += W_THREADS)
        reinterpret_cast<uint4*>(sP)[i] = make_uint4(0u, 0u, 0u, 0u);
    for (int c = tid; c < W_MD; c += W_THREADS) sCnt[c] = 0u;
    if (tid < 2) sZ[2 * W_MAXD + tid] = 0.0f;
    if (tid == 0) {
        for (int s = 0; s < W_P_STAGES; ++s) {
            mbar_init(&pfull[s], W_CONV_WARPS);
            mbar_init(&pempty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], W_EPI_WARPS);
        }
        mbar_init(dfull, 1);
        mbar_init(dempty, 1);
        mbar_init(udone, 1);
        for (int r = 0; r < W_R_MAX; ++r) {
            mbar_init(&rfull[r], 1);
            mbar_init(&rempty[r], W_CONV_WARPS);
        }
        fence_mbar_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(sTaddr)),
                     "r"(W_TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (*sTaddr != 0u) __trap();
    constexpr uint32_t tmem = 0u;

    if (warp == 0) {
        // ----------------------- producer: the unit's direction block, slice by slice
        uint32_t g = 0;
        for (int64_t u = w_next(a, blockIdx.x, units); u < units; u = w_next(a, u + gridDim.x, units)) {
            const WUnit w = w_unit(a, u);
            const unsigned char* src = a.uop + ((size_t)w.q * a.NB + w.blk) * (size_t)L.ns * 4096;
            for (int s = 0; s < S; ++s)
                for (int k0 = 0; k0 < slice_ns(L, s); k0 += W_DSTEPS, ++g) {
                    const int nst = slice_ns(L, s) - k0 < W_DSTEPS ? slice_ns(L, s) - k0 : W_DSTEPS;
                    const uint32_t bytes = (uint32_t)nst * 4096u;
                    if (g > 0) mbar_wait_sleep(dempty, (g - 1) & 1u);
                    expect_tx_elect(dfull, bytes);
                    tma_load_elect(sD, src + (size_t)(TC_SLICE_NS * s + k0) * 4096, bytes, dfull);
                    __syncwarp();
                }
        }
    } else if (warp == 1) {
        // -------------------------------------------------------- MMA issuer
        const uint32_t idesc = (1u << 4) | ((uint32_t)(W_NP >> 3) << 17) | ((uint32_t)(W_MD >> 4) << 24);
        uint32_t it = 0, g = 0, gs = 0, gacc = 0;
        for (int64_t u = w_next(a, blockIdx.x, units); u < units; u = w_next(a, u + gridDim.x, units), ++it) {
            const WUnit w = w_unit(a, u);
            for (int s = 0; s < S; ++s)
                for (int k0 = 0; k0 < slice_ns(L, s); k0 += W_DSTEPS, ++g) {
                    const int nst = slice_ns(L, s) - k0 < W_DSTEPS ? slice_ns(L, s) - k0 : W_DSTEPS;
                    mbar_wait_sleep(dfull, g & 1u);
                    if (s == 0 && k0 == 0 && it > 0) mbar_wait(udone, (it - 1) & 1u);  // previous unit done with A
                    tc_fence_after();
                    tmem_cp_dirblock(tmem + a_base + 8u * (TC_SLICE_NS * s + k0), umma_desc(smem_u32(sD), 2048, 128),
                                     nst);
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
                    const uint32_t st = gs % W_P_STAGES;
                    mbar_wait(&pfull[st], (gs / W_P_STAGES) & 1u);
                    tc_fence_after();
                    mma_slice(tmem + buf * W_ACC, tmem + a_base + 8u * TC_SLICE_NS * s,
                              umma_desc(smem_u32(sP) + st * W_STAGE, 2048, 128), idesc, s < L.full ? 4 : L.q16,
                              s < L.full ? 0 : L.rsteps, s == 0);
                    mma_commit_elect(&pempty[st]);
                }
                mma_commit_elect(&tfull[buf]);
            }
            mma_commit_elect(udone);
        }
    } else if (warp == 2) {
        // --------------------------------- producer: raw FP32 rows per (tile, slice)
        uint32_t g = 0, rs = 0, rph = 0;
        for (int64_t u = w_next(a, blockIdx.x, units); u < units; u = w_next(a, u + gridDim.x, units)) {
            const WUnit w = w_unit(a, u);
            for (int64_t t = w.t0; t < w.t1; ++t) {
                for (int s = 0; s < S; ++s, ++g) {
                    const uint32_t bytes = (uint32_t)(slice_width(d, s) * W_NP * 4);
                    if (g >= (uint32_t)RS) mbar_wait_sleep(&rempty[rs], rph ^ 1u);
                    expect_tx_elect(&rfull[rs], bytes);
                    tma_load_elect(sRaw + (size_t)rs * TC_SLICE * W_NP,
                                   a.xb + ((size_t)t * d + (size_t)TC_SLICE * s) * W_NP, bytes, &rfull[rs]);
                    __syncwarp();
                    if (++rs == (uint32_t)RS) {
                        rs = 0;
                        rph ^= 1u;
                    }
                }
            }
        }
    } else if (warp < W_EPI_WARP0) {
        // ---------------------------------- converters: (point r, 32-coordinate half h)
        const int ct = tid - W_CONV_WARP0 * 32;
        const int r = ct & (W_NP - 1);
        const int h = ct >> 7;                      // coordinate group: [W_CPT h, W_CPT h + W_CPT) of a slice
        uint32_t it = 0, gs = 0, rs = 0, rph = 0, gtile = 0;
        for (int64_t u = w_next(a, blockIdx.x, units); u < units; u = w_next(a, u + gridDim.x, units), ++it) {
            const WUnit w = w_unit(a, u);
            float* zs = sZ + (it & 1u) * W_MAXD;
            float zl = 0.0f;
            for (int c = ct; c < W_MAXD; c += W_CONV_THREADS) {
                const float z = c < d ? __ldg(a.zq + (size_t)w.q * d + c) : 0.0f;
                zs[c] = z;
                zl = fmaxf(zl, fabsf(z));
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) zl = fmaxf(zl, __shfl_xor_sync(0xffffffffu, zl, o));
            float* zmx = sZ + 2 * W_MAXD;  // [2] max |z| per unit parity (non-negative: int max order)
            if (lane == 0) atomicMax(reinterpret_cast<int*>(zmx + (it & 1u)), __float_as_int(zl));
            named_bar(2, W_CONV_THREADS);
            const float zmax = zmx[it & 1u];
            // the bound of the next tile's point is loaded one tile ahead (a global
            // load on the critical path otherwise)
            float xm_next = w.t0 * W_NP + r < a.n ? __ldg(a.xmax + w.t0 * W_NP + r) : 0.0f;
            for (int64_t t = w.t0; t < w.t1; ++t, ++gtile) {
                const bool ok = t * W_NP + r < a.n;
                const float xm = xm_next;
                if (t + 1 < w.t1) xm_next = (t + 1) * W_NP + r < a.n ? __ldg(a.xmax + (t + 1) * W_NP + r) : 0.0f;
                // per-point scale 2^(14 - E), bound max|x_i| + max|z| < 2^E
                const float bnd = (ok ? xm : 0.0f) + zmax;
                float scale = 0.0f;
                if (bnd > 0.0f) {
                    int E = (int)((__float_as_uint(bnd) >> 23) & 0xFF) - 126;
                    if (E < -100) E = -100;
                    scale = __uint_as_float((uint32_t)(127 + 14 - E) << 23);
                }
                bool nz = false;
                for (int s = 0; s < S; ++s, ++gs) {
                    const uint32_t st = gs % W_P_STAGES;
                    mbar_wait(&rfull[rs], rph);
                    const float* X = sRaw + (size_t)rs * TC_SLICE * W_NP + W_CPT * h * W_NP + r;
                    const float* zh = zs + TC_SLICE * s + W_CPT * h;
                    float2 av[4 * W_CH];
                    if (s < L.full) nz |= w_load_slice<true>(X, zh, h, TC_SLICE, av);
                    else nz |= w_load_slice<false>(X, zh, h, d - TC_SLICE * L.full, av);
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&rempty[rs]);
                    if (++rs == (uint32_t)RS) {
                        rs = 0;
                        rph ^= 1u;
                    }
                    if (gs >= W_P_STAGES) mbar_wait(&pempty[st], ((gs / W_P_STAGES) - 1) & 1u);
                    unsigned char* P = sP + st * W_STAGE + r * 16;
                    if (s < L.full) w_store_slice<true>(P, av, scale, h, TC_SLICE, 4, 0);
                    else w_store_slice<false>(P, av, scale, h, d - TC_SLICE * L.full, L.q16, L.rem);
                    if (STORE && s == S - 1 && h == 0) {
                        // exact power-of-two rescale of this point for the epilogue: y = acc 2^(E - 29)
                        // (8-deep ring; the converter runs at most S_P + 2 tiles ahead of the epilogue)
                        float inv = 0.0f;
                        if (bnd > 0.0f) {
                            int E = (int)((__float_as_uint(bnd) >> 23) & 0xFF) - 126;
                            if (E < -100) E = -100;
                            inv = ldexpf(1.0f, E - 29);
                        }
                        sInv[(gtile & 7u) * W_NP + r] = inv;
                    }
                    if (!STORE && s == S - 1) {
                        // counted points of the tile: valid rows with some a != 0 (coinciding
                        // rows x = z give y = +-0 and are ties on both sides); one ballot word
                        // per (warp's point group, coordinate group), read by the epilogue
                        // after this tile's tfull (ordered by pfull -> MMA -> tfull)
                        const uint32_t bal = __ballot_sync(0xffffffffu, ok && nz);
                        if (lane == 0) sNz[((gtile & 7u) * W_GROUPS + h) * 4 + (r >> 5)] = bal;
                    }
                    fence_proxy_async();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&pfull[st]);
                }
            }
            // max |z| slot of this unit parity is reused two units later
            named_bar(2, W_CONV_THREADS);
            if (ct == 0) zmx[it & 1u] = 0.0f;
        }
    } else if (STORE) {
        // ---------------------------------------------- epilogue: y' rows (STORE)
        const int quarter = warp & 3;
        const int half = (warp - W_EPI_WARP0) >> 2;
        const uint32_t lane_base = (uint32_t)(32 * quarter) << 16;
        const bool vec = (a.n & 3) == 0;
        float* stg = sStg + (warp - W_EPI_WARP0) * 32 * 33;
        uint32_t gacc = 0, gtile = 0;
        for (int64_t u = w_next(a, blockIdx.x, units); u < units; u = w_next(a, u + gridDim.x, units)) {
            const WUnit w = w_unit(a, u);
            const int jl = (w.blk - a.jb0) * W_MD + 32 * quarter + lane;  // row of the chunk
            const bool live = w.blk * W_MD + 32 * quarter + lane < a.m;
            float* yrow = a.y + ((size_t)w.q * a.jbn * W_MD + jl) * (size_t)a.n;
            // the warp's 32 rows: consecutive, the first at y0; rows_live of them < m
            float* y0 = a.y + ((size_t)w.q * a.jbn * W_MD + (size_t)(w.blk - a.jb0) * W_MD + 32 * quarter) * (size_t)a.n;
            const int rows_live = min(32, a.m - (w.blk * W_MD + 32 * quarter));
            for (int64_t t = w.t0; t < w.t1; ++t, ++gtile, ++gacc) {
                const uint32_t buf = dbl ? (gacc & 1u) : 0u;
                const uint32_t ph = dbl ? ((gacc >> 1) & 1u) : (gacc & 1u);
                mbar_wait(&tfull[buf], ph);
                tc_fence_after();
                const float* inv = sInv + (gtile & 7u) * W_NP + 64 * half;
                const int64_t p0 = t * W_NP + 64 * half;
                const uint32_t tb = tmem + lane_base + buf * W_ACC + (uint32_t)(half * 64);
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
        // ------------------------------------------------------------ epilogue
        const int ct = tid - W_EPI_WARP0 * 32;
        const int quarter = warp & 3;
        const int half = (warp - W_EPI_WARP0) >> 2;
        const uint32_t lane_base = (uint32_t)(32 * quarter) << 16;
        uint32_t gacc = 0, gtile = 0;
        for (int64_t u = w_next(a, blockIdx.x, units); u < units; u = w_next(a, u + gridDim.x, units)) {
            const WUnit w = w_unit(a, u);
            uint32_t cnt = 0u, zsum = 0u;
            for (int64_t t = w.t0; t < w.t1; ++t, ++gtile, ++gacc) {
                const uint32_t buf = dbl ? (gacc & 1u) : 0u;
                const uint32_t ph = dbl ? ((gacc >> 1) & 1u) : (gacc & 1u);
                mbar_wait(&tfull[buf], ph);
                tc_fence_after();
                uint32_t km[4] = {0u, 0u, 0u, 0u};
                const uint32_t* nzw = sNz + (gtile & 7u) * W_GROUPS * 4;
#pragma unroll
                for (int g2 = 0; g2 < W_GROUPS; ++g2)
#pragma unroll
                    for (int k = 0; k < 4; ++k) km[k] |= nzw[g2 * 4 + k];
                const uint32_t keep0 = km[2 * half], keep1 = km[2 * half + 1];
                const int64_t rows = a.n - t * W_NP;
                zsum += (uint32_t)(rows < W_NP ? rows : W_NP) -
                        (uint32_t)(__popc(km[0]) + __popc(km[1]) + __popc(km[2]) + __popc(km[3]));
                const uint32_t tb = tmem + lane_base + buf * W_ACC + (uint32_t)(half * 64);
                // two 32-column loads in turn (register budget of the 864-thread CTA)
                uint32_t y[32], m0 = 0u, m1 = 0u;
                tmem_ld32(tb, y);
                tmem_wait_ld();
#pragma unroll
                for (int j = 31; j >= 0; --j) m0 = __funnelshift_l(y[j], m0, 1);
                tmem_ld32(tb + 32, y);
                tmem_wait_ld();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[buf]);
#pragma unroll
                for (int j = 31; j >= 0; --j) m1 = __funnelshift_l(y[j], m1, 1);
                cnt += __popc(m0 & keep0) + __popc(m1 & keep1);
            }
            atomicAdd(sCnt + 32 * quarter + lane, cnt);
            named_bar(1, W_EPI_THREADS);
            const int64_t r1 = w.t1 * W_NP < a.n ? w.t1 * W_NP : a.n;
            const int valid = (int)(r1 - w.t0 * W_NP);
            int* dst = a.counts + (size_t)w.q * a.mpad * 2;
            const int j0 = w.blk * W_MD;
            for (int c = ct; c < W_MD; c += W_EPI_THREADS) {
                const int lt = (int)sCnt[c];
                sCnt[c] = 0u;
                if (j0 + c >= a.m) continue;
                const int gtv = valid - (int)zsum - lt;
                if (lt) atomicAdd(dst + 2 * (j0 + c) + 0, lt);
                if (gtv) atomicAdd(dst + 2 * (j0 + c) + 1, gtv);
            }
            named_bar(1, W_EPI_THREADS);
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(W_TMEM_COLS));
}

template <bool STORE>
static cudaError_t launch_tcw(TcArgs a, int sms, cudaStream_t st) {
    if (a.d <= TC_SLICE || a.d > W_MAXD || a.xmax == nullptr) return cudaErrorInvalidValue;
    const WSmem lay(STORE);
    if (lay.raw_stages < 2) return cudaErrorInvalidValue;
    a.gb = 1;
    if (!STORE) {
        a.jb0 = 0;
        a.jbn = a.NB;
    }
    a.groups = a.jbn;
    // chunks: >= 4 units per SM, and chunks short enough that a wave's tiles stay in L2
    const int64_t base = (int64_t)a.Qb * a.jbn;
    int64_t chunks = (4ll * sms + base - 1) / base;
    const int64_t l2_tiles = (int64_t)(48ll << 20) / ((int64_t)a.d * W_NP * 4);  // ~48 MB of rows per chunk
    const int64_t min_chunks = (a.tiles + l2_tiles - 1) / (l2_tiles > 0 ? l2_tiles : 1);
    if (chunks < min_chunks) chunks = min_chunks;
    if (chunks < 1) chunks = 1;
    if (chunks > a.tiles) chunks = a.tiles;
    a.tiles_per_chunk = (a.tiles + chunks - 1) / chunks;
    a.chunks = (int)((a.tiles + a.tiles_per_chunk - 1) / a.tiles_per_chunk);
    a.raw_stages = lay.raw_stages;
    const size_t smem = (size_t)lay.total;
    cudaError_t e =
        cudaFuncSetAttribute(contract_tcw_kernel<STORE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t units = base * a.chunks;
    if (units == 0) return cudaSuccess;
    const int grid = (int)(units < sms ? units : sms);
    contract_tcw_kernel<STORE><<<grid, W_THREADS, smem, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_contract_tcw(TcArgs a, int sms, cudaStream_t st) { return launch_tcw<false>(a, sms, st); }
cudaError_t launch_contract_tcw_store(TcArgs a, int sms, cudaStream_t st) { return launch_tcw<true>(a, sms, st); }

}  // namespace rrs
