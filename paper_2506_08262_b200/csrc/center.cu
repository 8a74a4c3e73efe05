// center.cu -- the centred frame of the projection notions.
//
// The projection / asymmetric-projection depths of z only need the order
// statistics of the projections px = <u, x_i> relative to pz = <u, z>
// (_kernels.pyx:292-351).  Storing y_i = <u, x_i - z> in FP32 (the halfspace
// difference form) makes the rounding of y scale with |z - x_i|: a query far
// from the data (depth ~1e-4) gets projections whose spread is resolved only
// to ~|z| / MAD · 2^-24.  Instead the store writes
//     y'_i = <u, x_i - m>          (FP32, from the centred copy x - m)
// and the select adds the FP64 shift of the direction
//     Delta = <u, m - z>           (y_i = y'_i + Delta)
// to the median only: med(y) = med(y') + Delta, MAD(y) = MAD(y'), and the
// positive deviations y - med(y) = y' - med(y').  m is the coordinate-wise
// median of a strided sample of the rows, so y' resolves the data's own spread.
//
// Small datasets (n < STORE64_N) additionally accumulate y' in FP64 from an
// FP64 centred copy: their MAD is a small-sample statistic that can sit far
// below the spread of the projections, where the FP32 accumulation error of a
// d-term dot product would show.
#include "common.cuh"
#include "kernels.h"

namespace rrs {

constexpr int CENTER_S = 1024;

// m_c = lower median of column c over min(n, 1024) rows at strided positions
// (4i + 1) n / 4S -- offset from the select kernels' sample positions
// (2i + 1) n / 2S, so one crafted set of rows cannot bias both
__global__ void __launch_bounds__(512) center_sample_kernel(const double* __restrict__ x, int64_t n, int d,
                                                            double* __restrict__ center, double* __restrict__ iqr) {
    __shared__ double s[CENTER_S];
    const int c = blockIdx.x;
    const int S = n >= CENTER_S ? CENTER_S : (int)n;
    for (int i = threadIdx.x; i < CENTER_S; i += blockDim.x)
        s[i] = i < S ? x[(((int64_t)(4 * i + 1) * n) / (4 * S)) * d + c] : INFINITY;
    __syncthreads();
    for (int k = 2; k <= CENTER_S; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < CENTER_S; i += blockDim.x) {
                const int p = i ^ j;
                if (p > i) {
                    const double a = s[i], b = s[p];
                    if ((a > b) == ((i & k) == 0)) {
                        s[i] = b;
                        s[p] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
    if (threadIdx.x == 0) {
        center[c] = s[(S - 1) / 2];
        if (iqr) iqr[c] = s[(3 * S) / 4 < S ? (3 * S) / 4 : S - 1] - s[S / 4];
    }
}

// xb[t][c][i] = (float)(x[t·BM + i][c] - m_c), zero padding rows; a 32 x 32
// shared-memory transpose keeps the FP64 reads and the FP32 writes coalesced
__global__ void block_centered_kernel(const double* __restrict__ x, const double* __restrict__ center,
                                      float* __restrict__ xb, int64_t n, int d, int64_t tiles) {
    __shared__ float tile[32][33];
    const int64_t row0 = (int64_t)blockIdx.x * 32;  // 32 rows
    const int c0 = blockIdx.y * 32;                 // 32 coordinates
    const int tx = threadIdx.x, ty = threadIdx.y;   // 32 x 8
    for (int r = ty; r < 32; r += 8) {
        const int64_t row = row0 + r;
        const int c = c0 + tx;
        tile[r][tx] = (row < n && c < d) ? (float)(x[row * d + c] - center[c]) : 0.0f;
    }
    __syncthreads();
    for (int cc = ty; cc < 32; cc += 8) {
        const int c = c0 + cc;
        const int64_t row = row0 + tx;
        if (c < d && row < tiles * BM) {
            const int64_t t = row / BM;
            const int i = (int)(row % BM);
            xb[(t * d + c) * BM + i] = tile[tx][cc];
        }
    }
}

__global__ void center_copy64_kernel(const double* __restrict__ x, const double* __restrict__ center,
                                     double* __restrict__ xc, int64_t count, int d) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) xc[i] = x[i] - center[i % d];
}

// shift[q][j] = <u_qj, m - z_q> in FP64, one warp per direction
__global__ void direction_shift_kernel(const double* __restrict__ u64, const double* __restrict__ center,
                                       const double* __restrict__ z, double* __restrict__ shift, int Qb, int m,
                                       int d) {
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= (int64_t)Qb * m) return;
    const int q = (int)(w / m);
    const double* u = u64 + w * d;
    const double* zq = z + (int64_t)q * d;
    double s = 0.0;
    for (int l = lane; l < d; l += 32) s = fma(u[l], center[l] - zq[l], s);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) shift[w] = s;
}

// y[q][jj][i] = (float) sum_l u[q][j0 + jj][l] · xc[i][l], accumulated in FP64
__global__ void store64_kernel(const double* __restrict__ xc, const double* __restrict__ u64, float* __restrict__ y,
                               int64_t n, int d, int m, int j0, int jcount) {
    const int jj = blockIdx.y, q = blockIdx.z;
    const int j = j0 + jj;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float* out = y + ((int64_t)q * jcount + jj) * n;
    if (j >= m) {
        out[i] = 0.0f;
        return;
    }
    const double* u = u64 + ((int64_t)q * m + j) * d;
    const double* xr = xc + i * d;
    double s = 0.0;
    for (int l = 0; l < d; ++l) s = fma(u[l], xr[l], s);
    out[i] = (float)s;
}

// early exit (halfspace): rows equal to the query in FP32 in every coordinate
// (x - z == 0 in the contraction, ties for every direction), per query
__global__ void __launch_bounds__(BM) coincide32_kernel(const float* __restrict__ xb, const float* __restrict__ zq,
                                                        int64_t n, int d, int64_t tiles, long long* __restrict__ c0) {
    const int q = blockIdx.y;
    const float* z = zq + (size_t)q * d;
    int cnt = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        if (t * BM + threadIdx.x >= n) continue;
        const float* xr = xb + (size_t)t * d * BM + threadIdx.x;
        int l = 0;
        while (l < d && xr[(size_t)l * BM] == z[l]) ++l;
        cnt += l == d;
    }
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(reinterpret_cast<unsigned long long*>(c0 + q), (unsigned long long)cnt);
}

cudaError_t launch_coincide_count32(const float* xb, const float* zq, int64_t n, int d, int64_t tiles, int Qb,
                                    long long* c0, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(c0, 0, (size_t)Qb * 8, st);
    if (e != cudaSuccess) return e;
    const int64_t blocks = tiles < 64 ? tiles : 64;
    coincide32_kernel<<<dim3((unsigned)blocks, (unsigned)Qb), BM, 0, st>>>(xb, zq, n, d, tiles, c0);
    return cudaGetLastError();
}

cudaError_t launch_center_sample(const double* x, int64_t n, int d, double* center, double* iqr, cudaStream_t st) {
    center_sample_kernel<<<d, 512, 0, st>>>(x, n, d, center, iqr);
    return cudaGetLastError();
}

cudaError_t launch_block_centered(const double* x, const double* center, float* xb, int64_t n, int d, int64_t tiles,
                                  cudaStream_t st) {
    dim3 grid((unsigned)((tiles * BM + 31) / 32), (unsigned)((d + 31) / 32));
    block_centered_kernel<<<grid, dim3(32, 8), 0, st>>>(x, center, xb, n, d, tiles);
    return cudaGetLastError();
}

cudaError_t launch_center_copy64(const double* x, const double* center, double* xc, int64_t n, int d,
                                 cudaStream_t st) {
    const int64_t count = n * d;
    center_copy64_kernel<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(x, center, xc, count, d);
    return cudaGetLastError();
}

cudaError_t launch_direction_shift(const double* u64, const double* center, const double* z, double* shift, int Qb,
                                   int m, int d, cudaStream_t st) {
    const int64_t threads = (int64_t)Qb * m * 32;
    direction_shift_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(u64, center, z, shift, Qb, m, d);
    return cudaGetLastError();
}

cudaError_t launch_store64(const double* xc, const double* u64, float* y, int64_t n, int d, int Qb, int m, int j0,
                           int jcount, cudaStream_t st) {
    dim3 grid((unsigned)((n + 127) / 128), (unsigned)jcount, (unsigned)Qb);
    store64_kernel<<<grid, 128, 0, st>>>(xc, u64, y, n, d, m, j0, jcount);
    return cudaGetLastError();
}

}  // namespace rrs
