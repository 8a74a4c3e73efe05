// contract.cu -- K2: fused FP32 contraction of the data against a batch of
// directions, difference form y[i,j] = sum_l u[j,l] * (x[i,l] - z[l]).
//
// Replaces the reference's materialised projection (_kernels.pyx:120-168
// proj_rect + :188-199 proj_point_span) and, in count mode, the halfspace
// univariate kernel (_kernels.pyx:270-289): the m x n projection matrix is
// never formed; each CTA keeps per-direction (#y<0, #y>0) counters in
// registers and the ties (y == 0, incl. the query's own row) fall out as
// n - lt - gt, counted on both sides as the reference does.
//
// Work unit = (query q, direction block jb of BN=128, chunk of point tiles).
// The direction block (d x 128 FP32, K-major) is staged once in shared memory
// by a TMA bulk copy; the point tiles (KC x 128, K-major, tile-blocked in HBM)
// stream through a 2-stage TMA bulk-copy / mbarrier pipeline.  The query is
// subtracted in shared memory (x - z exactly 0 for the query's own row, so
// the self-tie is exact by construction).  256 threads, 8x8 register tile.
//
// Store mode (projection notions) writes y for a direction chunk instead.
#include "common.cuh"
#include "kernels.h"

namespace rrs {

// d > STREAM_U_D: the direction block is streamed in K chunks next to the point
// chunks (2 x 2 x 32 rows = 64 KB) instead of staying resident (d x 128 x 4 =
// 100 KB at d = 200), so two CTAs fit an SM; the block is re-read from L2 per
// point tile.
#ifndef RRS_STREAM_U_D
#define RRS_STREAM_U_D 128
#endif
constexpr int STREAM_U_D = RRS_STREAM_U_D;
constexpr int KC_STREAM = 32;
__host__ __device__ inline int chunk_rows(int d) { return d > STREAM_U_D ? KC_STREAM : KC; }
__host__ __device__ inline int stage_rows(int d) { return d < chunk_rows(d) ? d : chunk_rows(d); }

size_t contract_smem_bytes(int d) {
    const bool stream_u = d > STREAM_U_D;
    size_t us = stream_u ? (size_t)2 * stage_rows(d) * BN * sizeof(float) : (size_t)d * BN * sizeof(float);
    size_t as = (size_t)2 * stage_rows(d) * BM * sizeof(float);
    size_t red = (size_t)8 * BN * 2 * sizeof(int);
    if (as < red) as = red;
    return us + as + MAX_D * sizeof(float) + 4 * sizeof(uint64_t);
}

template <bool STORE>
__global__ void __launch_bounds__(CT_THREADS, 2) contract_kernel(const ContractArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int d = a.d;
    const int srows = stage_rows(d);
    const int kchunk = chunk_rows(d);
    const bool stream_u = d > STREAM_U_D;
    float* Us = reinterpret_cast<float*>(smem_raw);
    float* As = Us + (stream_u ? (size_t)2 * srows * BN : (size_t)d * BN);
    size_t as_floats = (size_t)2 * srows * BM;
    if (as_floats < (size_t)8 * BN * 2) as_floats = (size_t)8 * BN * 2;
    float* zs = As + as_floats;
    uint64_t* bars = reinterpret_cast<uint64_t*>(zs + MAX_D);

    const int tid = threadIdx.x;
    // tx: direction quads, ty: point quads.  Count mode: a warp holds 16 tx x 2 ty
    // (the column sums fold lanes l and l ^ 16).  Store mode: 2 tx x 16 ty, so one
    // float4 store instruction writes 2 rows x 256 contiguous bytes of y instead
    // of 16 rows x 32 bytes (the store is bound by the y write traffic)
    const int tx = STORE ? (tid >> 4) : (tid & 15), ty = STORE ? (tid & 15) : (tid >> 4);

    // ---- unit decode
    const int per_q = a.jbn * a.chunks;
    const int q = blockIdx.x / per_q;
    const int rem = blockIdx.x - q * per_q;
    const int jbl = rem / a.chunks;
    const int c = rem - jbl * a.chunks;
    const int jb = a.jb0 + jbl;
    if (!STORE && a.done && a.done[q]) return;  // early exit (before any barrier / TMA)
    const int64_t t_begin = (int64_t)c * a.tiles_per_unit;
    int64_t t_end = t_begin + a.tiles_per_unit;
    if (t_end > a.tiles) t_end = a.tiles;
    const int nkc = (d + kchunk - 1) / kchunk;
    const int S = (int)(t_end - t_begin) * nkc;

    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        mbar_init(&bars[2], 1);
        fence_mbar_init();
    }
    __syncthreads();

    const float* ublk = a.u32 + ((size_t)q * a.MB + jb) * d * BN;
    auto issue = [&](int s) {
        const int64_t t = t_begin + s / nkc;
        const int kc = s % nkc;
        const int k0 = kc * kchunk;
        const int kcnt = (d - k0) < kchunk ? (d - k0) : kchunk;
        const uint32_t bytes = (uint32_t)kcnt * BM * sizeof(float);
        uint64_t* bar = &bars[1 + (s & 1)];
        if (stream_u) {  // the matching rows of the direction block ride on the same barrier
            mbar_arrive_expect_tx(bar, 2 * bytes);
            bulk_g2s(Us + (size_t)(s & 1) * srows * BN, ublk + (size_t)k0 * BN, bytes, bar);
        } else {
            mbar_arrive_expect_tx(bar, bytes);
        }
        bulk_g2s(As + (size_t)(s & 1) * srows * BM, a.xb + ((size_t)t * d + k0) * BM, bytes, bar);
    };

    if (tid == 0) {
        if (!stream_u) {
            const uint32_t ubytes = (uint32_t)d * BN * sizeof(float);
            mbar_arrive_expect_tx(&bars[0], ubytes);
            bulk_g2s(Us, ublk, ubytes, &bars[0]);
        }
        if (S > 0) issue(0);
        if (S > 1) issue(1);
    }
    for (int k = tid; k < d; k += CT_THREADS) zs[k] = a.zq[(size_t)q * d + k];
    __syncthreads();  // zs is read by every thread in the subtract pass
    if (!stream_u) mbar_wait(&bars[0], 0);

    float acc[8][8];
    unsigned lt[8], le[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        lt[j] = 0u;
        le[j] = 0u;
    }

    for (int s = 0; s < S; ++s) {
        const int st = s & 1;
        const int64_t t = t_begin + s / nkc;
        const int kc = s % nkc;
        const int k0 = kc * kchunk;
        const int kcnt = (d - k0) < kchunk ? (d - k0) : kchunk;
        float* Ab = As + (size_t)st * srows * BM;
        mbar_wait(&bars[1 + st], (uint32_t)((s >> 1) & 1));

        // x - z in place; rows past n become exact zeros (counted on neither side)
        {
            const int64_t row0 = t * BM;
            const int64_t vrows = a.n - row0;
            const int valid = vrows < BM ? (int)vrows : BM;
            float4* A4 = reinterpret_cast<float4*>(Ab);
            // thread owns column group i4 = (tid % 32) * 4 of rows k = tid / 32 + 8 * step
            const int i4 = (tid & 31) * 4;
            if (valid == BM) {
                for (int k = tid >> 5; k < kcnt; k += CT_THREADS / 32) {
                    const float zk = zs[k0 + k];
                    float4 v = A4[k * (BM / 4) + (tid & 31)];
                    v.x -= zk;
                    v.y -= zk;
                    v.z -= zk;
                    v.w -= zk;
                    A4[k * (BM / 4) + (tid & 31)] = v;
                }
            } else {
                for (int k = tid >> 5; k < kcnt; k += CT_THREADS / 32) {
                    const float zk = zs[k0 + k];
                    float4 v = A4[k * (BM / 4) + (tid & 31)];
                    v.x = (i4 + 0 < valid) ? v.x - zk : 0.0f;
                    v.y = (i4 + 1 < valid) ? v.y - zk : 0.0f;
                    v.z = (i4 + 2 < valid) ? v.z - zk : 0.0f;
                    v.w = (i4 + 3 < valid) ? v.w - zk : 0.0f;
                    A4[k * (BM / 4) + (tid & 31)] = v;
                }
            }
        }
        __syncthreads();

        if (kc == 0) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = 0.0f;
        }

        const float* Ap = Ab + ty * 4;
        const float* Bp = (stream_u ? Us + (size_t)st * srows * BN : Us + (size_t)k0 * BN) + tx * 4;
#pragma unroll 2
        for (int k = 0; k < kcnt; ++k) {
            const float4 a0 = *reinterpret_cast<const float4*>(Ap + k * BM);
            const float4 a1 = *reinterpret_cast<const float4*>(Ap + k * BM + 64);
            const float4 b0 = *reinterpret_cast<const float4*>(Bp + k * BN);
            const float4 b1 = *reinterpret_cast<const float4*>(Bp + k * BN + 64);
            const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }

        if (kc == nkc - 1) {
            if constexpr (!STORE) {
                // exact zeros are +0 (accumulators start at +0, RN): the sign bit
                // of y is [y < 0] and the sign bit of bits(y) - 1 is [y <= 0]
                // (padding rows are +0 and are removed from le at the end)
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const unsigned b = __float_as_uint(acc[i][j]);
                        lt[j] += b >> 31;
                        le[j] += (b - 1u) >> 31;
                    }
            } else {
                const int64_t row0 = t * BM;
                const int64_t n = a.n;
                const bool vec = ((n & 3) == 0) && (row0 + BM <= n);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int col = (j < 4) ? tx * 4 + j : 64 + tx * 4 + (j - 4);
                    const int jg = jb * BN + col;
                    if (jg >= a.m) continue;
                    float* yr = a.y + ((size_t)q * ((size_t)a.jbn * BN) + (jg - a.jb0 * BN)) * n;
                    if (vec) {
                        *reinterpret_cast<float4*>(yr + row0 + ty * 4) =
                            make_float4(acc[0][j], acc[1][j], acc[2][j], acc[3][j]);
                        *reinterpret_cast<float4*>(yr + row0 + 64 + ty * 4) =
                            make_float4(acc[4][j], acc[5][j], acc[6][j], acc[7][j]);
                    } else {
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const int64_t r = row0 + ((i < 4) ? ty * 4 + i : 64 + ty * 4 + (i - 4));
                            if (r < n) yr[r] = acc[i][j];
                        }
                    }
                }
            }
        }
        __syncthreads();
        if (tid == 0 && s + 2 < S) {
            fence_proxy_async();
            issue(s + 2);
        }
    }

    if constexpr (!STORE) {
        // column sums over the 16 row-threads: lanes l and l^16 share columns
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            lt[j] += __shfl_xor_sync(0xffffffffu, lt[j], 16);
            le[j] += __shfl_xor_sync(0xffffffffu, le[j], 16);
        }
        int* red = reinterpret_cast<int*>(As);  // [8 warps][BN][2]
        const int warp = tid >> 5;
        if ((tid & 16) == 0) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int col = (j < 4) ? tx * 4 + j : 64 + tx * 4 + (j - 4);
                red[(warp * BN + col) * 2 + 0] = (int)lt[j];
                red[(warp * BN + col) * 2 + 1] = (int)le[j];
            }
        }
        __syncthreads();
        if (tid < BN) {
            int slt = 0, sle = 0;
#pragma unroll
            for (int w = 0; w < CT_THREADS / 32; ++w) {
                slt += red[(w * BN + tid) * 2 + 0];
                sle += red[(w * BN + tid) * 2 + 1];
            }
            // rows of this unit: real ones plus zero padding (counted in le only)
            const int64_t rows_all = (t_end - t_begin) * BM;
            int64_t rows_real = a.n - t_begin * BM;
            if (rows_real > rows_all) rows_real = rows_all;
            const int sgt = (int)(rows_real - (sle - (rows_all - rows_real)));
            int* dst = a.counts + ((size_t)q * a.MB * BN + (size_t)jb * BN + tid) * 2;
            if (slt) atomicAdd(dst + 0, slt);
            if (sgt) atomicAdd(dst + 1, sgt);
        }
    }
}

template <bool STORE>
static cudaError_t launch_contract(const ContractArgs& a, cudaStream_t st) {
    if (a.d > MAX_D) return cudaErrorInvalidValue;
    const size_t smem = contract_smem_bytes(a.d);
    cudaError_t e = cudaFuncSetAttribute(contract_kernel<STORE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t units = (int64_t)a.Qb * a.jbn * a.chunks;
    if (units == 0) return cudaSuccess;
    contract_kernel<STORE><<<(unsigned)units, CT_THREADS, smem, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_contract_count(const ContractArgs& a, cudaStream_t st) {
    return launch_contract<false>(a, st);
}
cudaError_t launch_contract_store(const ContractArgs& a, cudaStream_t st) {
    return launch_contract<true>(a, st);
}

}  // namespace rrs
