// contract_tcs.cu -- K2 store mode on the tensor cores (projection notions,
// d <= 50): y_ij = <u_j, x_i - z> written for the select kernel, computed as a
// three-way FP16 split with FP32 accumulation in TMEM.
//
// The projection notions need y itself to ~1e-5 relative after the median /
// MAD cancellation, which the two-term split of contract_tc.cu (22 bits) does
// not give.  Here a s = ah + am + al and u 2^15 = uh + um + ul
// (33 bits each) and six of the nine products are kept (kernels.h Tc6Layout:
// uh ah, uh am, um ah, uh al, ul ah, um am; the rest are ~2^-33 relative), so
// the error is the FP32 accumulation's own, as in the FFMA store kernel.
// y is rescaled exactly (powers of two) in the epilogue and written as FP32
// rows y[q][j - 128 jb0][n], the layout the select kernel reads.
//
// One direction block per unit (A: 8 ns TMEM columns, ns = 19 at d = 50),
// two FP32 accumulators (TMEM columns 0..255), the point operand of each tile
// in one of two ns x 4 KB stages, the direction block staged in 2-step chunks.
// Units = (query, direction block of the chunk, chunk of point tiles).
// Warps: 0 direction producer, 1 TMEM allocator + MMA issuer, 2 raw-tile
// producer, 3-10 converters (point, 32-coordinate half), 11-18 epilogue.
#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

#include <cuda_fp16.h>

namespace rrs {

namespace {

constexpr int S_CONV_WARP0 = 3;
constexpr int S_CONV_WARPS = 8;
constexpr int S_CONV_THREADS = S_CONV_WARPS * 32;
constexpr int S_EPI_WARP0 = S_CONV_WARP0 + S_CONV_WARPS;
constexpr int S_EPI_WARPS = 8;
constexpr int S_THREADS = (S_EPI_WARP0 + S_EPI_WARPS) * 32;  // 608
constexpr int S_MAXD = 64;
constexpr int S_MAXNS = 19;                 // d <= 50
constexpr int S_NP = 128, S_MD = 128;
constexpr int S_P_STAGES = 2;
constexpr int S_R_MAX = 4;
constexpr int S_DSTEPS = 2;                 // K steps of A per staging load
constexpr uint32_t S_TMEM_COLS = 512;
constexpr uint32_t S_ACC = 128;
constexpr uint32_t S_A = 2 * S_ACC;
constexpr int S_SMEM_LIMIT = 227 * 1024;

struct SSmem {
    int P, D, ZS, SMX, INV, BARS, TADDR, RAW, total, raw_stages, raw_rows, stage_bytes;
    static constexpr int NBARS = 2 * S_P_STAGES + 2 + 2 + 3 + 2 * S_R_MAX;
    __host__ __device__ SSmem(int ns, int d) {
        stage_bytes = ns * 4096;
        raw_rows = (d + 7) & ~7;                  // rows past d stay zero (whole 8-coordinate chunks)
        P = 0;
        D = P + S_P_STAGES * stage_bytes;
        ZS = D + S_DSTEPS * 4096;                // float [2][64]
        SMX = ZS + 2 * S_MAXD * 4;               // float [2][2][128] partial maxima
        INV = SMX + 2 * 2 * S_NP * 4;            // float [8][128] per-point 1 / (s 2^15)
        BARS = INV + 8 * S_NP * 4;
        TADDR = BARS + NBARS * 8;
        RAW = (TADDR + 16 + 1023) & ~1023;
        const int per = raw_rows * S_NP * 4;
        const int room = S_SMEM_LIMIT - 1024 - RAW;
        raw_stages = room / per;
        if (raw_stages > S_R_MAX) raw_stages = S_R_MAX;
        total = RAW + raw_stages * per + 1024;
    }
};

struct SUnit {
    int q, blk;  // blk: direction block index within the chunk
    int64_t t0, t1;
};

__device__ __forceinline__ SUnit s_unit(const TcsArgs& a, int64_t u) {
    SUnit r;
    const int64_t per_q = (int64_t)a.jbn * a.chunks;
    r.q = (int)(u / per_q);
    const int64_t rem = u - (int64_t)r.q * per_q;
    r.blk = (int)(rem / a.chunks);
    const int64_t c = rem - (int64_t)r.blk * a.chunks;
    r.t0 = c * a.tiles_per_chunk;
    r.t1 = r.t0 + a.tiles_per_chunk < a.tiles ? r.t0 + a.tiles_per_chunk : a.tiles;
    return r;
}

// ns MMAs of one (tile, block), K steps paired one to one; one elected thread
// issues them all
__device__ __forceinline__ void mma_block(uint32_t acc, uint32_t aT, uint64_t bd, uint32_t idesc, int ns) {
    if (elect_one()) {
        for (int i = 0; i < ns; ++i) umma_f16(acc, aT + 8u * (uint32_t)i, bd + 256ull * (uint64_t)i, idesc, i ? 1u : 0u);
    }
    __syncwarp();
}

// v = hi + mid + lo (FP16 each, exact residuals in FP32)
__device__ __forceinline__ void split3(float2 v, uint32_t& h, uint32_t& m, uint32_t& l) {
    const __half2 hh = __floats2half2_rn(v.x, v.y);
    const float2 hf = __half22float2(hh);
    const float2 r1 = make_float2(v.x - hf.x, v.y - hf.y);
    const __half2 mh = __floats2half2_rn(r1.x, r1.y);
    const float2 mf = __half22float2(mh);
    const __half2 lh = __floats2half2_rn(r1.x - mf.x, r1.y - mf.y);
    h = *reinterpret_cast<const uint32_t*>(&hh);
    m = *reinterpret_cast<const uint32_t*>(&mh);
    l = *reinterpret_cast<const uint32_t*>(&lh);
}

}  // namespace

__global__ void __launch_bounds__(S_THREADS, 1) contract_tcs_kernel(const TcsArgs a) {
    extern __shared__ __align__(1024) unsigned char s_raw[];
    unsigned char* sm = s_raw + ((1024u - (smem_u32(s_raw) & 1023u)) & 1023u);
    const int d = a.d;
    const Tc6Layout L = tc6_layout(d);
    const SSmem lay(L.ns, d);
    const int stage_bytes = lay.stage_bytes;
    unsigned char* sP = sm + lay.P;
    unsigned char* sD = sm + lay.D;
    float* sZ = reinterpret_cast<float*>(sm + lay.ZS);
    float* sMx = reinterpret_cast<float*>(sm + lay.SMX);
    float* sInv = reinterpret_cast<float*>(sm + lay.INV);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + lay.BARS);
    uint64_t* pfull = &bars[0];
    uint64_t* pempty = &bars[S_P_STAGES];
    uint64_t* tfull = &bars[2 * S_P_STAGES];
    uint64_t* tempty = &bars[2 * S_P_STAGES + 2];
    uint64_t* dfull = &bars[2 * S_P_STAGES + 4];
    uint64_t* dempty = &bars[2 * S_P_STAGES + 5];
    uint64_t* udone = &bars[2 * S_P_STAGES + 6];
    uint64_t* rfull = &bars[2 * S_P_STAGES + 7];
    uint64_t* rempty = &bars[2 * S_P_STAGES + 7 + S_R_MAX];
    uint32_t* sTaddr = reinterpret_cast<uint32_t*>(sm + lay.TADDR);
    float* sRaw = reinterpret_cast<float*>(sm + lay.RAW);
    const int RS = lay.raw_stages;
    const int RR = lay.raw_rows;
    const uint32_t raw_bytes = (uint32_t)(d * S_NP * 4);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t units = (int64_t)a.Qb * a.jbn * a.chunks;

    for (int i = tid; i < S_P_STAGES * stage_bytes / 16; i += S_THREADS)
        reinterpret_cast<uint4*>(sP)[i] = make_uint4(0u, 0u, 0u, 0u);
    for (int i = tid; i < RS * RR * S_NP; i += S_THREADS) sRaw[i] = 0.0f;  // rows >= d stay 0
    if (tid == 0) {
        for (int s = 0; s < S_P_STAGES; ++s) {
            mbar_init(&pfull[s], S_CONV_WARPS);
            mbar_init(&pempty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], S_EPI_WARPS);
        }
        mbar_init(dfull, 1);
        mbar_init(dempty, 1);
        mbar_init(udone, 1);
        for (int r = 0; r < S_R_MAX; ++r) {
            mbar_init(&rfull[r], 1);
            mbar_init(&rempty[r], S_CONV_WARPS);
        }
        fence_mbar_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(sTaddr)),
                     "r"(S_TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (*sTaddr != 0u) __trap();
    constexpr uint32_t tmem = 0u;

    if (warp == 0) {
        // ------------------------- producer: the unit's direction block, 2 K steps at a time
        uint32_t g = 0;
        for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
            const SUnit w = s_unit(a, u);
            const unsigned char* src = a.uop + ((size_t)w.q * a.NB + a.jb0 + w.blk) * (size_t)stage_bytes;
            for (int k0 = 0; k0 < L.ns; k0 += S_DSTEPS, ++g) {
                const int nst = L.ns - k0 < S_DSTEPS ? L.ns - k0 : S_DSTEPS;
                if (g > 0) mbar_wait_sleep(dempty, (g - 1) & 1u);
                expect_tx_elect(dfull, (uint32_t)nst * 4096u);
                tma_load_elect(sD, src + (size_t)k0 * 4096, (uint32_t)nst * 4096u, dfull);
                __syncwarp();
            }
        }
    } else if (warp == 1) {
        // -------------------------------------------------------- MMA issuer
        const uint32_t idesc = (1u << 4) | ((uint32_t)(S_NP >> 3) << 17) | ((uint32_t)(S_MD >> 4) << 24);
        uint32_t it = 0, g = 0, gtile = 0;
        for (int64_t u = blockIdx.x; u < units; u += gridDim.x, ++it) {
            const SUnit w = s_unit(a, u);
            for (int k0 = 0; k0 < L.ns; k0 += S_DSTEPS, ++g) {
                const int nst = L.ns - k0 < S_DSTEPS ? L.ns - k0 : S_DSTEPS;
                mbar_wait_sleep(dfull, g & 1u);
                if (k0 == 0 && it > 0) mbar_wait(udone, (it - 1) & 1u);
                tc_fence_after();
                tmem_cp_dirblock(tmem + S_A + 8u * k0, umma_desc(smem_u32(sD), 2048, 128), nst);
                mma_commit_elect(dempty);
            }
            for (int64_t t = w.t0; t < w.t1; ++t, ++gtile) {
                const uint32_t s = gtile % S_P_STAGES;
                const uint32_t buf = gtile & 1u;
                mbar_wait(&pfull[s], (gtile / S_P_STAGES) & 1u);
                if (gtile >= 2) mbar_wait(&tempty[buf], ((gtile >> 1) - 1) & 1u);
                tc_fence_after();
                mma_block(tmem + buf * S_ACC, tmem + S_A, umma_desc(smem_u32(sP) + s * stage_bytes, 2048, 128), idesc,
                          L.ns);
                mma_commit_elect(&tfull[buf]);
                mma_commit_elect(&pempty[s]);
            }
            mma_commit_elect(udone);
        }
    } else if (warp == 2) {
        // -------------------------------------- producer: raw FP32 point tiles
        uint32_t g = 0, rs = 0, rph = 0;
        for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
            const SUnit w = s_unit(a, u);
            for (int64_t t = w.t0; t < w.t1; ++t, ++g) {
                if (g >= (uint32_t)RS) mbar_wait_sleep(&rempty[rs], rph ^ 1u);
                expect_tx_elect(&rfull[rs], raw_bytes);
                tma_load_elect(sRaw + (size_t)rs * RR * S_NP, a.xb + (size_t)t * d * S_NP, raw_bytes, &rfull[rs]);
                __syncwarp();
                if (++rs == (uint32_t)RS) {
                    rs = 0;
                    rph ^= 1u;
                }
            }
        }
    } else if (warp < S_EPI_WARP0) {
        // ------------------- converters: x - z -> scale -> FP16 three-way split
        const int ct = tid - S_CONV_WARP0 * 32;
        const int r = ct & (S_NP - 1);
        const int h = ct >> 7;                    // coordinates [32 h, 32 h + 32)
        const int main_chunks = 2 * L.q16;
        uint32_t it = 0, gtile = 0, rs = 0, rph = 0;
        for (int64_t u = blockIdx.x; u < units; u += gridDim.x, ++it) {
            const SUnit w = s_unit(a, u);
            float* zs = sZ + (it & 1u) * S_MAXD;
            if (ct < S_MAXD) zs[ct] = ct < d ? __ldg(a.zq + (size_t)w.q * d + ct) : 0.0f;
            named_bar(2, S_CONV_THREADS);
            for (int64_t t = w.t0; t < w.t1; ++t, ++gtile) {
                const uint32_t s = gtile % S_P_STAGES;
                mbar_wait(&rfull[rs], rph);
                const float* X = sRaw + (size_t)rs * RR * S_NP + 32 * h * S_NP + r;
                const float* zh = zs + 32 * h;
                float2 av[16];
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
                            const float2 xv = make_float2(X[(8 * c + 2 * e) * S_NP], X[(8 * c + 2 * e + 1) * S_NP]);
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
                float* mxs = sMx + (gtile & 1u) * 2 * S_NP;
                mxs[h * S_NP + r] = mx;
                named_bar(2, S_CONV_THREADS);
                mx = fmaxf(mxs[r], mxs[S_NP + r]);
                float scale = 0.0f;
                if (mx > 0.0f) {
                    int E = (int)((__float_as_uint(mx) >> 23) & 0xFF) - 126;  // mx < 2^E
                    if (E < -100) E = -100;
                    scale = __uint_as_float((uint32_t)(127 + 14 - E) << 23);  // 2^(14 - E)
                    // 1 / (scale 2^15) = 2^(E - 29): exact, read by the epilogue
                    if (h == 0) sInv[(gtile & 7u) * S_NP + r] = ldexpf(1.0f, E - 29);
                } else if (h == 0) {
                    sInv[(gtile & 7u) * S_NP + r] = 0.0f;
                }
                if (gtile >= S_P_STAGES) mbar_wait(&pempty[s], ((gtile / S_P_STAGES) - 1) & 1u);
                unsigned char* P = sP + s * stage_bytes + r * 16;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int cc = 4 * h + c;
                    if (8 * cc >= d) continue;
                    uint32_t hw[4], mw[4], lw[4];
                    const float2 sc2 = make_float2(scale, scale);
#pragma unroll
                    for (int e = 0; e < 4; ++e) split3(__fmul2_rn(av[4 * c + e], sc2), hw[e], mw[e], lw[e]);
                    if (cc < main_chunks) {
                        // B values per product {h, m, h, l, h, m}
                        const uint4 hv = make_uint4(hw[0], hw[1], hw[2], hw[3]);
                        const uint4 mv = make_uint4(mw[0], mw[1], mw[2], mw[3]);
                        const uint4 lv = make_uint4(lw[0], lw[1], lw[2], lw[3]);
                        *reinterpret_cast<uint4*>(P + (0 * main_chunks + cc) * (S_NP * 16)) = hv;
                        *reinterpret_cast<uint4*>(P + (1 * main_chunks + cc) * (S_NP * 16)) = mv;
                        *reinterpret_cast<uint4*>(P + (2 * main_chunks + cc) * (S_NP * 16)) = hv;
                        *reinterpret_cast<uint4*>(P + (3 * main_chunks + cc) * (S_NP * 16)) = lv;
                        *reinterpret_cast<uint4*>(P + (4 * main_chunks + cc) * (S_NP * 16)) = hv;
                        *reinterpret_cast<uint4*>(P + (5 * main_chunks + cc) * (S_NP * 16)) = mv;
                    } else {
#pragma unroll 1
                        for (int e = 0; e < 8; ++e) {
                            const int cd = 8 * cc + e;
                            if (cd >= d) break;
                            const int wi = e >> 1, sh = (e & 1) ? 16 : 0;
                            const uint32_t hx = wi == 0 ? hw[0] : wi == 1 ? hw[1] : wi == 2 ? hw[2] : hw[3];
                            const uint32_t mx2 = wi == 0 ? mw[0] : wi == 1 ? mw[1] : wi == 2 ? mw[2] : mw[3];
                            const uint32_t lx = wi == 0 ? lw[0] : wi == 1 ? lw[1] : wi == 2 ? lw[2] : lw[3];
                            const uint16_t t3[3] = {(uint16_t)(hx >> sh), (uint16_t)(mx2 >> sh), (uint16_t)(lx >> sh)};
                            int kk = 96 * L.q16 + (cd - 16 * L.q16);
#pragma unroll
                            for (int pr = 0; pr < 6; ++pr, kk += L.rem)
                                *reinterpret_cast<uint16_t*>(P + (kk >> 3) * (S_NP * 16) + (kk & 7) * 2) =
                                    t3[tc6_b_term(pr)];
                        }
                    }
                }
                fence_proxy_async();
                __syncwarp();
                if (lane == 0) mbar_arrive(&pfull[s]);
            }
        }
    } else {
        // ------------------------------------------ epilogue: rescale and store y rows
        const int quarter = warp & 3;
        const int half = (warp - S_EPI_WARP0) >> 2;
        const uint32_t lane_base = (uint32_t)(32 * quarter) << 16;
        const size_t rows_per_q = (size_t)a.jbn * S_MD;
        const bool vec = (a.n & 3) == 0;
        uint32_t gtile = 0;
        for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
            const SUnit w = s_unit(a, u);
            const int jl = w.blk * S_MD + 32 * quarter + lane;  // direction row within the chunk
            const bool live = (a.jb0 * S_MD + jl) < a.m;
            float* yrow = a.y + ((size_t)w.q * rows_per_q + jl) * a.n;
            for (int64_t t = w.t0; t < w.t1; ++t, ++gtile) {
                const uint32_t buf = gtile & 1u;
                mbar_wait(&tfull[buf], (gtile >> 1) & 1u);
                tc_fence_after();
                const float* inv = sInv + (gtile & 7u) * S_NP + 64 * half;
                const int64_t p0 = t * S_NP + 64 * half;
                const uint32_t tb = tmem + lane_base + buf * S_ACC + (uint32_t)(half * 64);
#pragma unroll
                for (int part = 0; part < 2; ++part) {
                    uint32_t v[32];
                    tmem_ld32(tb + 32 * part, v);
                    tmem_wait_ld();
                    if (part == 1) {
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&tempty[buf]);
                    }
                    if (!live) continue;
                    const int64_t pb = p0 + 32 * part;
                    if (vec && pb + 32 <= a.n) {
#pragma unroll
                        for (int k = 0; k < 8; ++k)
                            *reinterpret_cast<float4*>(yrow + pb + 4 * k) =
                                make_float4(__uint_as_float(v[4 * k]) * inv[32 * part + 4 * k],
                                            __uint_as_float(v[4 * k + 1]) * inv[32 * part + 4 * k + 1],
                                            __uint_as_float(v[4 * k + 2]) * inv[32 * part + 4 * k + 2],
                                            __uint_as_float(v[4 * k + 3]) * inv[32 * part + 4 * k + 3]);
                    } else {
#pragma unroll
                        for (int k = 0; k < 32; ++k)
                            if (pb + k < a.n) yrow[pb + k] = __uint_as_float(v[k]) * inv[32 * part + k];
                    }
                }
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(S_TMEM_COLS));
}

// Direction operand in the six-product layout from the FP64 directions: one
// thread per (query, block row, K position); padded rows and positions are 0.
__global__ void pack_tc6_operand_kernel(const double* __restrict__ u64, unsigned char* __restrict__ uop, int Qb,
                                        int m, int NB, int d) {
    const Tc6Layout L = tc6_layout(d);
    const int64_t per_block = (int64_t)128 * 16 * L.ns;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (int64_t)Qb * NB * per_block) return;
    const int64_t qb = idx / per_block;
    const int64_t rem = idx - qb * per_block;
    const int kk = (int)(rem / 128), row = (int)(rem % 128);
    const int q = (int)(qb / NB), blk = (int)(qb % NB);
    const int j = blk * 128 + row;
    int p, c;
    tc6_elem(L, kk, p, c);
    __half val = __double2half(0.0);
    if (c >= 0 && j < m) {
        const double v = u64[((size_t)q * m + j) * d + c] * 32768.0;
        const __half hh = __double2half(v);
        const double r1 = v - (double)__half2float(hh);
        const __half mh = __double2half(r1);
        const __half lh = __double2half(r1 - (double)__half2float(mh));
        const int term = tc6_a_term(p);
        val = term == 0 ? hh : term == 1 ? mh : lh;
    }
    *reinterpret_cast<__half*>(uop + (size_t)qb * L.ns * 4096 + (size_t)(kk >> 3) * 2048 + (size_t)row * 16 +
                               (kk & 7) * 2) = val;
}

cudaError_t launch_pack_tc6_operand(const double* u64, unsigned char* uop, int Qb, int m, int NB, int d,
                                    cudaStream_t st) {
    const int64_t total = (int64_t)Qb * NB * 128 * 16 * tc6_layout(d).ns;
    if (total == 0) return cudaSuccess;
    pack_tc6_operand_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(u64, uop, Qb, m, NB, d);
    return cudaGetLastError();
}

cudaError_t launch_contract_tcs(TcsArgs a, int sms, cudaStream_t st) {
    if (a.d < 1 || tc6_layout(a.d).ns > S_MAXNS) return cudaErrorInvalidValue;
    const SSmem lay(tc6_layout(a.d).ns, a.d);
    if (lay.raw_stages < 2 || lay.total > S_SMEM_LIMIT) return cudaErrorInvalidValue;
    a.gb = 1;
    a.groups = a.jbn;
    const int64_t base = (int64_t)a.Qb * a.jbn;
    int64_t chunks = (16ll * sms + base - 1) / base;
    if (chunks < 1) chunks = 1;
    if (chunks > a.tiles) chunks = a.tiles;
    a.tiles_per_chunk = (a.tiles + chunks - 1) / chunks;
    a.chunks = (int)((a.tiles + a.tiles_per_chunk - 1) / a.tiles_per_chunk);
    a.raw_stages = lay.raw_stages;
    cudaError_t e = cudaFuncSetAttribute(contract_tcs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, lay.total);
    if (e != cudaSuccess) return e;
    const int64_t units = base * a.chunks;
    if (units == 0) return cudaSuccess;
    contract_tcs_kernel<<<(int)(units < sms ? units : sms), S_THREADS, lay.total, st>>>(a);
    return cudaGetLastError();
}

}  // namespace rrs
