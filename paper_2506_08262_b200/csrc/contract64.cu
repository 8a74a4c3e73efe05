// contract64.cu -- K2 for wide data, d > 256: FP64 contraction
//     y_ij = sum_l u_jl (x_il - c_l)      (c = z for halfspace, m for the
//                                          centred projection store)
// from an FP64 row-major copy of the data and the FP64 directions.
//
// Above d = 256 the tensor kernels run out of TMEM columns for a resident
// direction block, and an FP32 FFMA dot product of d terms accumulates a
// rounding error ~2^-24 sqrt(d) |x - z| that exceeds the tie zone
// 1e-6 max(|x_i|, |z|) of the halfspace contract by d ~ 300.
// FP64 keeps every count exact outside |y| < ~1e-15 |x - z|; the reference has
// no dimension limit (_kernels.pyx:139-155 d_chunk loop), nor has this path
// (d <= GEN_MAX_D, the generation kernel's bound).
//
// CTA = 64 points x 64 directions of one query, 256 threads, 4 x 4 FP64
// outputs per thread; K in chunks of 16 staged in shared memory.  Count mode
// accumulates #(y < 0), #(y > 0) per direction (exact zeros count on neither
// side: ties, like contract.cu); store mode writes y as FP32 rows [q][j][n].
#include "common.cuh"
#include "kernels.h"

namespace rrs {

constexpr int C64_P = 64, C64_J = 64, C64_K = 16, C64_T = 256;

template <bool STORE>
__global__ void __launch_bounds__(C64_T) contract64_kernel(const Contract64Args a) {
    __shared__ double As[C64_K][C64_P + 1];  // x - c, [k][point]
    __shared__ double Bs[C64_K][C64_J + 1];  // u, [k][direction]
    __shared__ int cnt[C64_J][2];
    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;  // 16 x 16 threads, 4 x 4 outputs each
    const int64_t p0 = (int64_t)blockIdx.x * C64_P;
    const int j0 = blockIdx.y * C64_J;  // direction within the launch's range
    const int q = blockIdx.z;
    if (!STORE && a.done && a.done[q]) return;  // early exit
    const int d = a.d;
    const double* cq = a.c + (size_t)q * a.c_stride;
    const double* ub = a.u64 + ((size_t)q * a.m + a.jbase) * d;
    if (!STORE && tid < 2 * C64_J) cnt[tid >> 1][tid & 1] = 0;
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    for (int k0 = 0; k0 < d; k0 += C64_K) {
        // 64 rows x 16 coordinates of each operand: 4 per thread, coordinate-fastest
        for (int e = tid; e < C64_P * C64_K; e += C64_T) {
            const int r = e / C64_K, k = e % C64_K;
            const int64_t pi = p0 + r;
            const int l = k0 + k;
            As[k][r] = (pi < a.n && l < d) ? a.x64[pi * d + l] - cq[l] : 0.0;
            const int jj = j0 + r;
            Bs[k][r] = (jj < a.jcount && a.jbase + jj < a.m && l < d) ? ub[(size_t)jj * d + l] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < C64_K; ++k) {
            double av[4], bv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) av[i] = As[k][ty + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) bv[j] = Bs[k][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
        }
        __syncthreads();
    }
    if constexpr (STORE) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int jj = j0 + tx + 16 * j;
            if (jj >= a.jcount || a.jbase + jj >= a.m) continue;
            float* yr = a.y + ((size_t)q * a.jcount + jj) * a.n;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int64_t pi = p0 + ty + 16 * i;
                if (pi < a.n) yr[pi] = (float)acc[i][j];
            }
        }
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            int lt = 0, gt = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const bool real = p0 + ty + 16 * i < a.n;
                lt += (real && acc[i][j] < 0.0) ? 1 : 0;
                gt += (real && acc[i][j] > 0.0) ? 1 : 0;
            }
            // lanes tx and tx + 16 of a warp hold the same direction (ty, ty + 1)
            lt += __shfl_xor_sync(0xffffffffu, lt, 16);
            gt += __shfl_xor_sync(0xffffffffu, gt, 16);
            if ((tid & 16) == 0) {
                if (lt) atomicAdd(&cnt[tx + 16 * j][0], lt);
                if (gt) atomicAdd(&cnt[tx + 16 * j][1], gt);
            }
        }
        __syncthreads();
        if (tid < C64_J) {
            const int jj = j0 + tid;
            if (jj < a.jcount && a.jbase + jj < a.m) {
                int* dst = a.counts + ((size_t)q * a.mpad + a.jbase + jj) * 2;
                if (cnt[tid][0]) atomicAdd(dst + 0, cnt[tid][0]);
                if (cnt[tid][1]) atomicAdd(dst + 1, cnt[tid][1]);
            }
        }
    }
}

// rows of the FP64 data equal to the query in every coordinate, per query
__global__ void coincide64_kernel(const double* __restrict__ x, const double* __restrict__ z, int64_t n, int d,
                                  long long* __restrict__ c0) {
    const int q = blockIdx.y;
    const double* zq = z + (size_t)q * d;
    int cnt = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double* xr = x + i * d;
        int l = 0;
        while (l < d && xr[l] == zq[l]) ++l;
        cnt += l == d;
    }
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(reinterpret_cast<unsigned long long*>(c0 + q), (unsigned long long)cnt);
}

cudaError_t launch_coincide_count64(const double* x64, const double* z, int64_t n, int d, int Qb, long long* c0,
                                    cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(c0, 0, (size_t)Qb * 8, st);
    if (e != cudaSuccess) return e;
    int64_t blocks = (n + 255) / 256;
    if (blocks > 64) blocks = 64;
    coincide64_kernel<<<dim3((unsigned)blocks, (unsigned)Qb), 256, 0, st>>>(x64, z, n, d, c0);
    return cudaGetLastError();
}

cudaError_t launch_contract64(const Contract64Args& a, bool store, cudaStream_t st) {
    if (a.Qb == 0 || a.jcount == 0 || a.n == 0) return cudaSuccess;
    dim3 grid((unsigned)((a.n + C64_P - 1) / C64_P), (unsigned)((a.jcount + C64_J - 1) / C64_J), (unsigned)a.Qb);
    if (store) contract64_kernel<true><<<grid, C64_T, 0, st>>>(a);
    else contract64_kernel<false><<<grid, C64_T, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace rrs
