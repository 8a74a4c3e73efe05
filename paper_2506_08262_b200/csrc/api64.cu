// api64.cu -- FP64 device kernels behind the reference's materialised-projection
// API (the seams the RRS hot path deliberately skips, SURVEY §8(b) seam (ii)):
//
//   proj64_kernel        projection.py:99-168 (project_naive / project_parallel /
//                        project_point) = _kernels.pyx:171-199: P[j,i] =
//                        sum_l u[j,l] * x[i,l], acc = 0.0, ascending l, separate
//                        FP64 multiply and add (the reference core is built with
//                        -ffp-contract=off), so the scores are bit-identical;
//   span_depth64_kernel  univariate.py:162-184 depth_of_projections over caller px
//                        / pz = _kernels.pyx:270-351 (halfspace / projection /
//                        asym_projection span): exact FP64 order statistics by an
//                        MSB-first 8-bit radix select on order-preserving 64-bit
//                        keys, the reference's median rule (k = (n-1) >> 1, the
//                        midpoint with the next order statistic for even n) and
//                        its FP64 deviation arithmetic, so depths are bit-identical.
//
// Neither is on the RRS path (which never materialises px); they exist so a
// depthforge user calling these names gets the device, not a CPU fallback.
#include "common.cuh"
#include "kernels.h"
#include "../../include/rrs_b200.h"

namespace rrs {

// ------------------------------------------------------------------ proj64 --
constexpr int P64_TJ = 32, P64_TI = 32, P64_TL = 16;

__global__ void __launch_bounds__(256) proj64_kernel(const double* __restrict__ x, const double* __restrict__ u,
                                                     double* __restrict__ out, int64_t n, int m, int d) {
    __shared__ double su[P64_TJ][P64_TL + 1];
    __shared__ double sx[P64_TI][P64_TL + 1];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads
    const int64_t i0 = (int64_t)blockIdx.x * P64_TI;
    const int j0 = blockIdx.y * P64_TJ;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};  // directions j0 + ty + 8 r, point i0 + tx
    for (int l0 = 0; l0 < d; l0 += P64_TL) {
        for (int e = threadIdx.x; e < P64_TJ * P64_TL; e += 256) {
            const int r = e / P64_TL, c = e % P64_TL;
            su[r][c] = (j0 + r < m && l0 + c < d) ? u[(size_t)(j0 + r) * d + l0 + c] : 0.0;
            sx[r][c] = (i0 + r < n && l0 + c < d) ? x[(size_t)(i0 + r) * d + l0 + c] : 0.0;
        }
        __syncthreads();
        const int lc = d - l0 < P64_TL ? d - l0 : P64_TL;
        for (int c = 0; c < lc; ++c) {
            const double xv = sx[tx][c];
#pragma unroll
            for (int r = 0; r < 4; ++r) acc[r] = __dadd_rn(acc[r], __dmul_rn(su[ty + 8 * r][c], xv));
        }
        __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int j = j0 + ty + 8 * r;
        if (j < m && i0 + tx < n) out[(size_t)j * n + i0 + tx] = acc[r];
    }
}

cudaError_t launch_proj64(const double* x, const double* u, double* out, int64_t n, int m, int d,
                          cudaStream_t st) {
    if (n < 1 || m < 1 || d < 1) return cudaErrorInvalidValue;
    const dim3 grid((unsigned)((n + P64_TI - 1) / P64_TI), (unsigned)((m + P64_TJ - 1) / P64_TJ));
    proj64_kernel<<<grid, 256, 0, st>>>(x, u, out, n, m, d);
    return cudaGetLastError();
}

// ------------------------------------------------------------ span_depth64 --
constexpr int S64_THREADS = 256;

__device__ __forceinline__ uint64_t key64(double v) {
    const uint64_t b = (uint64_t)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double unkey64(uint64_t k) {
    return __longlong_as_double((long long)((k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k));
}

// element transforms of the three selections: the row itself, |x - med|, x - med (> 0 only)
enum { T_ID = 0, T_ABSDEV = 1, T_POSDEV = 2 };

__device__ __forceinline__ bool elem(const double* row, int64_t i, int kind, double med, double& v) {
    const double x = row[i];
    if (kind == T_ID) {
        v = x;
        return true;
    }
    if (kind == T_ABSDEV) {
        v = fabs(x - med);
        return true;
    }
    v = x - med;
    return v > 0.0;
}

__device__ __forceinline__ int64_t block_sum(int64_t v, int64_t* red) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    int64_t t = 0;
    for (int w = 0; w < S64_THREADS / 32; ++w) t += red[w];
    __syncthreads();
    return t;
}

// k-th smallest (0-based) of the selected elements' values; every thread returns it
__device__ double select_kth64(const double* row, int64_t n, int kind, double med, int64_t k, uint32_t* hist,
                               uint64_t* s_prefix, int64_t* s_k) {
    uint64_t prefix = 0, mask = 0;
    for (int shift = 56; shift >= 0; shift -= 8) {
        for (int b = threadIdx.x; b < 256; b += S64_THREADS) hist[b] = 0u;
        __syncthreads();
        for (int64_t i = threadIdx.x; i < n; i += S64_THREADS) {
            double v;
            if (!elem(row, i, kind, med, v)) continue;
            const uint64_t key = key64(v);
            if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int64_t kk = k;
            int b = 0;
            for (; b < 255; ++b) {
                if (kk < (int64_t)hist[b]) break;
                kk -= hist[b];
            }
            *s_prefix = prefix | ((uint64_t)b << shift);
            *s_k = kk;
        }
        __syncthreads();
        prefix = *s_prefix;
        k = *s_k;
        mask |= (uint64_t)255 << shift;
        __syncthreads();
    }
    return unkey64(prefix);
}

// _kernels.pyx:247-258 (_median_inplace): k = (n - 1) >> 1, even n -> midpoint
__device__ double median64(const double* row, int64_t n, int kind, double med, int64_t cnt, uint32_t* hist,
                           uint64_t* s_prefix, int64_t* s_k) {
    const int64_t k = (cnt - 1) >> 1;
    const double lo = select_kth64(row, n, kind, med, k, hist, s_prefix, s_k);
    if (cnt & 1) return lo;
    const double hi = select_kth64(row, n, kind, med, k + 1, hist, s_prefix, s_k);
    return (lo + hi) / 2.0;
}

__global__ void __launch_bounds__(S64_THREADS) span_depth64_kernel(const double* __restrict__ px,
                                                                   const double* __restrict__ pz,
                                                                   double* __restrict__ out, int64_t n,
                                                                   int notion) {
    __shared__ uint32_t hist[256];
    __shared__ uint64_t s_prefix;
    __shared__ int64_t s_k;
    __shared__ int64_t red[S64_THREADS / 32];
    const int j = blockIdx.x;
    const double* row = px + (size_t)j * n;
    const double y = pz[j];
    if (notion == RRS_HALFSPACE) {  // _kernels.pyx:270-289, ties on both sides
        int64_t le = 0, ge = 0;
        for (int64_t i = threadIdx.x; i < n; i += S64_THREADS) {
            const double v = row[i];
            le += v <= y;
            ge += v >= y;
        }
        le = block_sum(le, red);
        ge = block_sum(ge, red);
        if (threadIdx.x == 0) out[j] = (double)(le < ge ? le : ge) / (double)n;
        return;
    }
    const double med = median64(row, n, T_ID, 0.0, n, hist, &s_prefix, &s_k);
    if (notion == RRS_PROJECTION) {  // _kernels.pyx:292-314
        const double mad = median64(row, n, T_ABSDEV, med, n, hist, &s_prefix, &s_k);
        const double dev = fabs(y - med);
        if (threadIdx.x == 0) out[j] = mad == 0.0 ? (dev == 0.0 ? 1.0 : 0.0) : 1.0 / (1.0 + dev / mad);
        return;
    }
    // asym_projection, _kernels.pyx:317-351
    const double dev = y - med;
    if (dev <= 0.0) {
        if (threadIdx.x == 0) out[j] = 1.0;
        return;
    }
    int64_t npos = 0;
    for (int64_t i = threadIdx.x; i < n; i += S64_THREADS) npos += row[i] - med > 0.0;
    npos = block_sum(npos, red);
    if (npos == 0) {
        if (threadIdx.x == 0) out[j] = 0.0;
        return;
    }
    const double madp = median64(row, n, T_POSDEV, med, npos, hist, &s_prefix, &s_k);
    if (threadIdx.x == 0) out[j] = 1.0 / (1.0 + dev / madp);
}

cudaError_t launch_span_depth64(const double* px, const double* pz, double* out, int m, int64_t n, int notion,
                                cudaStream_t st) {
    if (m < 1 || n < 1) return cudaErrorInvalidValue;
    span_depth64_kernel<<<m, S64_THREADS, 0, st>>>(px, pz, out, n, notion);
    return cudaGetLastError();
}

}  // namespace rrs
