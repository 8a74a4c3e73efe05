// contract_tc.cu -- K2 on the 5th-generation tensor cores: exact-integer
// (int8-limb, Ozaki-style) contraction with a fused halfspace-count epilogue.
//
// Same result contract as the FFMA kernel (contract.cu): per (query, direction)
// the counts #(y<0), #(y>0) of y_i = <u, x_i - z> over all points, with the
// query's own row giving y = 0 exactly (self-tie by construction).  Here the
// sign of y is computed EXACTLY for fixed-point operands:
//   a_il = x_il - z_l (FP32) scaled per row by a power of two so that
//          |A_il| < 2^22 (A = rint(a * 2^(22-E_i)), E_i = exponent of max_l |a_il|);
//   U_jl = rint(u_jl * 2^22) (|u| <= 1);
//   both split into three signed int8 limbs  A = a2*2^16 + a1*2^8 + a0;
//   sum_l A_il U_jl = 2^32 S22 + 2^24 S21 + 2^16 S20 + (low products, dropped)
// where the tensor core accumulates S22, S21 = a2b1 + a1b2 and
// S20 = a2b0 + a1b1 + a0b2 in int32 TMEM accumulators (kind::i8, exact).  The
// three dropped low products are below 2^-15 of one quantisation step.  The
// per-row power of two never changes a sign, so no scale is needed in the
// epilogue: sign(y) = sign(S22*2^16 + S21*2^8 + S20), evaluated exactly in 32
// bits (S22 clamped to +-2^14: beyond that its term dominates).
//
// Persistent CTA (one per SM), 12 warps:
//   warp 0      TMA producer: X tile (FP32) and B blocks (int8 limbs) via
//               cp.async.bulk + mbarriers, double-buffered B;
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//               (M=128 points, N=64 directions, K=32 per instruction);
//   warps 4-11  x - z + per-row quantisation into the canonical no-swizzle
//               K-major UMMA layout, then the epilogue: tcgen05.ld of the three
//               accumulators, exact sign, warp ballot + popc per direction,
//               shared-memory counters; TMEM double-buffered against the MMA.
// Work item = (query, 128-point tile); all directions of the query are swept
// with the A tile resident.  Replaces _kernels.pyx:120-199 + 270-289.
#include "common.cuh"
#include "kernels.h"

namespace rrs {

constexpr int TC_THREADS = 384;
constexpr int TC_NB = 64;                  // directions per N-block (MMA N)
constexpr int TC_KP = 64;                  // K padded (d <= 64)
constexpr int A_LIMB_BYTES = 128 * TC_KP;  // 8 KB per limb
constexpr int B_LIMB_BYTES = TC_NB * TC_KP;            // 4 KB per limb
constexpr int B_BLOCK_BYTES = 3 * B_LIMB_BYTES;        // 12 KB per N-block
constexpr int TC_MAX_COLS = 4096;          // mpad limit for the smem counters
constexpr uint32_t TMEM_COLS = 512;

struct TcSmem {
    // offsets in bytes from a 1024-aligned base
    static constexpr int A = 0;
    static constexpr int B = A + 3 * A_LIMB_BYTES;       // 2 buffers
    static constexpr int X = B + 2 * B_BLOCK_BYTES;      // FP32 staging [64][128]
    static constexpr int CNT = X + TC_KP * 128 * 4;      // uint32 [TC_MAX_COLS]
    static constexpr int ZS = CNT + TC_MAX_COLS * 4;     // float [64]
    static constexpr int RMAX = ZS + TC_KP * 4;          // float [2][128]
    static constexpr int BARS = RMAX + 2 * 128 * 4;      // 9 mbarriers
    static constexpr int TADDR = BARS + 16 * 8;
    static constexpr int TOTAL = TADDR + 16;
};

size_t contract_tc_smem_bytes() { return TcSmem::TOTAL + 1024; }

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    // SmemDescriptor (tcgen05): start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46),
    // version 1 [46,48), base offset 0, lbo mode 0, layout SWIZZLE_NONE (0) [61,64)
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
    unsigned char* sA = sm + TcSmem::A;
    unsigned char* sB = sm + TcSmem::B;
    float* sX = reinterpret_cast<float*>(sm + TcSmem::X);
    uint32_t* sCnt = reinterpret_cast<uint32_t*>(sm + TcSmem::CNT);
    float* sZ = reinterpret_cast<float*>(sm + TcSmem::ZS);
    float* sRmax = reinterpret_cast<float*>(sm + TcSmem::RMAX);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + TcSmem::BARS);
    uint64_t* xfull = &bars[0];
    uint64_t* bfull = &bars[1];   // [2]
    uint64_t* bempty = &bars[3];  // [2]
    uint64_t* tfull = &bars[5];   // [2]
    uint64_t* tempty = &bars[7];  // [2]
    uint32_t* sTaddr = reinterpret_cast<uint32_t*>(sm + TcSmem::TADDR);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int d = a.d;
    const int NBk = a.NB;               // N-blocks of 64 directions per query
    const int ncols = NBk * TC_NB;
    const int nks = (d + 31) / 32;      // MMA K-steps (1 or 2)

    for (int c = tid; c < ncols; c += TC_THREADS) sCnt[c] = 0u;
    if (tid == 0) {
        mbar_init(xfull, 1);
        for (int b = 0; b < 2; ++b) {
            mbar_init(&bfull[b], 1);
            mbar_init(&bempty[b], 1);
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 8);
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

    // instruction descriptor: S32 accumulate, signed int8 A and B, K-major, N=64, M=128
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(TC_NB >> 3) << 17) |
                           ((uint32_t)(128 >> 4) << 24);

    const int64_t items = (int64_t)a.Qb * a.tiles;
    int it = 0;
    for (int64_t item = blockIdx.x; item < items; item += gridDim.x, ++it) {
        const int q = (int)(item / a.tiles);
        const int64_t t = item - (int64_t)q * a.tiles;
        const int64_t gbase = (int64_t)it * NBk;  // running N-block counter of this CTA
        const int64_t vrows = a.n - t * 128;
        const int valid = vrows < 128 ? (int)vrows : 128;

        // ---- stage the point tile and the query
        if (tid == 0) {
            const uint32_t bytes = (uint32_t)d * 128 * 4;
            mbar_arrive_expect_tx(xfull, bytes);
            bulk_g2s(sX, a.xb + (size_t)t * d * 128, bytes, xfull);
        }
        if (tid < d) sZ[tid] = a.zq[(size_t)q * d + tid];
        __syncthreads();  // sZ visible

        // ---- warps 4-11: x - z, per-row power-of-two scale, 3 int8 limbs
        if (warp >= 4) {
            const int ct = tid - 128;          // 0..255
            const int r = ct & 127, h = ct >> 7;
            mbar_wait(xfull, (uint32_t)(it & 1));
            const int k0 = h * 32;
            const int k1 = (k0 + 32) < d ? (k0 + 32) : d;
            float mx = 0.0f;
            for (int k = k0; k < k1; ++k) mx = fmaxf(mx, fabsf(sX[k * 128 + r] - sZ[k]));
            sRmax[h * 128 + r] = mx;
            named_bar(1, 256);
            mx = fmaxf(sRmax[r], sRmax[128 + r]);
            float scale = 0.0f;
            if (r < valid && mx > 0.0f) {
                int E = (int)((__float_as_uint(mx) >> 23) & 0xFF) - 126;  // mx < 2^E
                if (E < -100) E = -100;
                scale = __uint_as_float((uint32_t)(127 + 22 - E) << 23);  // 2^(22-E)
            }
            for (int c = 2 * h; c < 2 * h + 2; ++c) {
                uint32_t w0[4], w1[4], w2[4];
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    uint32_t b0 = 0, b1 = 0, b2 = 0;
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int k = c * 16 + g * 4 + e;
                        const float av = (k < d) ? (sX[k * 128 + r] - sZ[k]) : 0.0f;
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
                // canonical K-major, no swizzle: [k-chunk c][row r][16 bytes]
                *reinterpret_cast<uint4*>(sA + 0 * A_LIMB_BYTES + c * 2048 + r * 16) =
                    make_uint4(w0[0], w0[1], w0[2], w0[3]);
                *reinterpret_cast<uint4*>(sA + 1 * A_LIMB_BYTES + c * 2048 + r * 16) =
                    make_uint4(w1[0], w1[1], w1[2], w1[3]);
                *reinterpret_cast<uint4*>(sA + 2 * A_LIMB_BYTES + c * 2048 + r * 16) =
                    make_uint4(w2[0], w2[1], w2[2], w2[3]);
            }
            fence_proxy_async();  // generic-proxy writes -> tensor-core (async proxy) reads
        }
        __syncthreads();  // A ready

        if (warp == 0) {
            // ---- producer: B blocks (int8 limbs of 64 directions) for this query
            if (lane == 0) {
                const unsigned char* src = a.u8 + (size_t)q * NBk * B_BLOCK_BYTES;
                for (int nb = 0; nb < NBk; ++nb) {
                    const int64_t g = gbase + nb;
                    const int buf = (int)(g & 1);
                    const int64_t u = g >> 1;
                    if (u >= 1) mbar_wait(&bempty[buf], (uint32_t)((u - 1) & 1));
                    mbar_arrive_expect_tx(&bfull[buf], B_BLOCK_BYTES);
                    bulk_g2s(sB + buf * B_BLOCK_BYTES, src + (size_t)nb * B_BLOCK_BYTES, B_BLOCK_BYTES,
                             &bfull[buf]);
                }
            }
        } else if (warp == 1) {
            // ---- single-thread MMA issuer
            if (lane == 0) {
                const uint32_t aBase = smem_u32(sA);
                for (int nb = 0; nb < NBk; ++nb) {
                    const int64_t g = gbase + nb;
                    const int buf = (int)(g & 1);
                    const int64_t u = g >> 1;
                    mbar_wait(&bfull[buf], (uint32_t)(u & 1));
                    if (u >= 1) mbar_wait(&tempty[buf], (uint32_t)((u - 1) & 1));
                    tc_fence_after();
                    const uint32_t bBase = smem_u32(sB + buf * B_BLOCK_BYTES);
                    const uint32_t dBase = tmem + (uint32_t)buf * 192u;
                    // (A limb, B limb, accumulator): S22 -> acc 2, S21 -> acc 1, S20 -> acc 0
                    const int la[6] = {2, 2, 1, 2, 1, 0};
                    const int lb[6] = {2, 1, 2, 0, 1, 2};
                    const int ac[6] = {2, 1, 1, 0, 0, 0};
                    const int first[6] = {1, 1, 0, 1, 0, 0};
                    for (int s = 0; s < nks; ++s) {
#pragma unroll
                        for (int p = 0; p < 6; ++p) {
                            const uint64_t ad =
                                umma_desc(aBase + la[p] * A_LIMB_BYTES + s * 2 * 2048, 2048, 128);
                            const uint64_t bd =
                                umma_desc(bBase + lb[p] * B_LIMB_BYTES + s * 2 * 1024, 1024, 128);
                            mma_i8(dBase + (uint32_t)ac[p] * TC_NB, ad, bd, idesc,
                                   (s == 0 && first[p]) ? 0u : 1u);
                        }
                    }
                    mma_commit(&bempty[buf]);
                    mma_commit(&tfull[buf]);
                }
            }
        } else if (warp >= 4) {
            // ---- epilogue: exact sign per (point, direction), ballot counts per direction
            const int quarter = warp & 3;
            const int half = (warp - 4) >> 2;
            const uint32_t lane_base = (uint32_t)(32 * quarter) << 16;
            for (int nb = 0; nb < NBk; ++nb) {
                const int64_t g = gbase + nb;
                const int buf = (int)(g & 1);
                const int64_t u = g >> 1;
                mbar_wait(&tfull[buf], (uint32_t)(u & 1));
                tc_fence_after();
#pragma unroll
                for (int cc = 0; cc < 2; ++cc) {
                    const int col0 = half * 32 + cc * 16;
                    const uint32_t tb = tmem + lane_base + (uint32_t)buf * 192u + (uint32_t)col0;
                    uint32_t r0[16], r1[16], r2[16];
                    tmem_ld16(tb + 0 * TC_NB, r0);
                    tmem_ld16(tb + 1 * TC_NB, r1);
                    tmem_ld16(tb + 2 * TC_NB, r2);
                    tmem_wait_ld();
                    uint32_t* cnt = sCnt + nb * TC_NB + col0;
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const int t1 = (int)r1[j] * 256 + (int)r0[j];
                        int hi = (int)r2[j];
                        hi = hi > 16384 ? 16384 : (hi < -16384 ? -16384 : hi);
                        const int w = hi * 65536 + t1;
                        const unsigned mlt = __ballot_sync(0xffffffffu, w < 0);
                        const unsigned mle = __ballot_sync(0xffffffffu, w <= 0);
                        if (lane == 0) atomicAdd(cnt + j, (uint32_t)__popc(mlt) | ((uint32_t)__popc(mle) << 16));
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[buf]);
            }
        }
        __syncthreads();  // all N-blocks counted (epilogue done => all MMAs done)

        // ---- flush this tile's counts: lt, and gt = real rows - (le - zero pad rows)
        {
            const int pad = 128 - valid;
            int* dst = a.counts + (size_t)q * a.mpad * 2;
            for (int c = tid; c < ncols; c += TC_THREADS) {
                const uint32_t v = sCnt[c];
                sCnt[c] = 0u;
                if (c >= a.m) continue;
                const int lt = (int)(v & 0xFFFFu);
                const int le = (int)(v >> 16);
                const int gt = valid - (le - pad);
                if (lt) atomicAdd(dst + 2 * c + 0, lt);
                if (gt) atomicAdd(dst + 2 * c + 1, gt);
            }
        }
        __syncthreads();
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}

cudaError_t launch_contract_tc(const TcArgs& a, int sms, cudaStream_t st) {
    if (a.d > TC_KP || a.NB * TC_NB > TC_MAX_COLS) return cudaErrorInvalidValue;
    const size_t smem = contract_tc_smem_bytes();
    cudaError_t e =
        cudaFuncSetAttribute(contract_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t items = (int64_t)a.Qb * a.tiles;
    if (items == 0) return cudaSuccess;
    const int grid = (int)(items < sms ? items : sms);
    contract_tc_kernel<<<grid, TC_THREADS, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace rrs
