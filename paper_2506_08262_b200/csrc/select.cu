// select.cu -- K3: projection / asymmetric-projection univariate depth from
// difference-form projections y_i = <u, x_i - z> (the query sits at y = 0).
//
// Replaces _kernels.pyx:202-267 (quickselect median, midpoint for even n) and
// the span kernels projection_span :292-314 / asym_projection_span :317-351.
// With y = px - pz:  med(px) - pz = med(y),  MAD(px) = MAD(y)  (shift
// invariance), so
//   D_P  = 1 / (1 + |med y| / med|y - med y|)   (MAD = 0 -> 1 iff med y == 0)
//   D_AP = 1                                    if -med y <= 0
//        = 0                                    if no y - med y > 0
//        = 1 / (1 + (-med y) / med{y - med y > 0})  otherwise.
// Order statistics come from a 3-pass (11/11/10-bit) radix select over
// order-preserving uint32 keys, histograms in shared memory with
// warp-aggregated (match.any) atomics; the row is cached in shared memory
// when it fits.  Midpoints and deviations are formed in FP64.
#include "common.cuh"
#include "kernels.h"

#include <float.h>

namespace rrs {

constexpr int SEL_THREADS = 512;
constexpr int SEL_WARPS = SEL_THREADS / 32;
constexpr int HIST_BINS = 2048;
constexpr int64_t SEL_CACHE_MAX = 40960;  // floats of y cached per CTA (160 KB)

__device__ __forceinline__ uint32_t fkey(float f) {
    uint32_t b = __float_as_uint(f);
    return b ^ ((b >> 31) ? 0xFFFFFFFFu : 0x80000000u);
}
__device__ __forceinline__ float kfloat(uint32_t k) {
    uint32_t b = (k & 0x80000000u) ? (k ^ 0x80000000u) : ~k;
    return __uint_as_float(b);
}

struct SelShared {
    int hist[HIST_BINS];
    int wsum[SEL_WARPS];
    int s_bin, s_below;
    unsigned long long s_min;
    int s_cnt;
};

// key functors: return false when element i does not take part
struct KeyMed {
    __device__ bool operator()(float y, uint32_t& k) const {
        k = fkey(y);
        return true;
    }
};
struct KeyAbsDev {
    double med;
    __device__ bool operator()(float y, uint32_t& k) const {
        k = fkey((float)fabs((double)y - med));
        return true;
    }
};
struct KeyPosDev {
    double med;
    __device__ bool operator()(float y, uint32_t& k) const {
        double t = (double)y - med;
        k = fkey((float)t);
        return t > 0.0;
    }
};

__device__ __forceinline__ int block_sum(int v, SelShared& sh) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = __reduce_add_sync(0xffffffffu, v);
    if (lane == 0) sh.wsum[warp] = v;
    __syncthreads();
    int t = 0;
    if (threadIdx.x < 32) {
        t = (threadIdx.x < SEL_WARPS) ? sh.wsum[threadIdx.x] : 0;
        t = __reduce_add_sync(0xffffffffu, t);
        if (threadIdx.x == 0) sh.s_cnt = t;
    }
    __syncthreads();
    t = sh.s_cnt;
    __syncthreads();
    return t;
}

// k-th smallest key (0-based) among participating elements; also returns the
// number of participating keys <= that key.
template <typename KF>
__device__ uint32_t block_select(const float* __restrict__ src, int64_t n, int64_t k, KF kf,
                                 SelShared& sh, int64_t& c_le) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t prefix = 0, pmask = 0;
    int64_t kk = k, below_total = 0;
    int last_count = 0;
    const int shifts[3] = {21, 10, 0};
    const int widths[3] = {11, 11, 10};
    for (int p = 0; p < 3; ++p) {
        const int shift = shifts[p];
        const int nb = 1 << widths[p];
        const uint32_t bmask = (uint32_t)(nb - 1);
        for (int b = tid; b < nb; b += SEL_THREADS) sh.hist[b] = 0;
        __syncthreads();
        for (int64_t base = (int64_t)warp * 32; base < n; base += (int64_t)SEL_WARPS * 32) {
            const int64_t i = base + lane;
            int bin = -1;
            if (i < n) {
                uint32_t key;
                if (kf(src[i], key) && (key & pmask) == prefix) bin = (int)((key >> shift) & bmask);
            }
            const unsigned grp = __match_any_sync(0xffffffffu, bin);
            if (bin >= 0 && lane == __ffs(grp) - 1) atomicAdd(&sh.hist[bin], __popc(grp));
        }
        __syncthreads();
        // exclusive scan over nb bins: each thread owns nb/SEL_THREADS consecutive bins
        const int per = nb / SEL_THREADS;
        int local = 0;
        for (int b = 0; b < per; ++b) local += sh.hist[tid * per + b];
        int incl = local;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            int o = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += o;
        }
        if (lane == 31) sh.wsum[warp] = incl;
        __syncthreads();
        int woff = 0;
        for (int w = 0; w < warp; ++w) woff += sh.wsum[w];
        int run = woff + incl - local;
        for (int b = 0; b < per; ++b) {
            const int h = sh.hist[tid * per + b];
            if ((int64_t)run <= kk && kk < (int64_t)run + h) {
                sh.s_bin = tid * per + b;
                sh.s_below = run;
            }
            run += h;
        }
        __syncthreads();
        const int bin = sh.s_bin;
        kk -= sh.s_below;
        below_total += sh.s_below;
        last_count = sh.hist[bin];
        prefix |= (uint32_t)bin << shift;
        pmask |= bmask << shift;
        __syncthreads();
    }
    c_le = below_total + last_count;
    return prefix;
}

// smallest participating key strictly greater than `key`
template <typename KF>
__device__ uint32_t block_min_greater(const float* __restrict__ src, int64_t n, uint32_t key, KF kf,
                                      SelShared& sh) {
    uint32_t best = 0xFFFFFFFFu;
    for (int64_t i = threadIdx.x; i < n; i += SEL_THREADS) {
        uint32_t k2;
        if (kf(src[i], k2) && k2 > key && k2 < best) best = k2;
    }
    best = __reduce_min_sync(0xffffffffu, best);
    if (threadIdx.x == 0) sh.s_min = 0xFFFFFFFFull;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) atomicMin(&sh.s_min, (unsigned long long)best);
    __syncthreads();
    uint32_t r = (uint32_t)sh.s_min;
    __syncthreads();
    return r;
}

// median of the participating keys (midpoint of the central pair, FP64),
// univariate.py:71-77 / _kernels.pyx:255-267
template <typename KF>
__device__ double block_median(const float* __restrict__ src, int64_t n, int64_t cnt, KF kf,
                               SelShared& sh) {
    const int64_t k = (cnt - 1) >> 1;
    int64_t c_le;
    const uint32_t lo = block_select(src, n, k, kf, sh, c_le);
    const double lov = (double)kfloat(lo);
    if (cnt & 1) return lov;
    uint32_t hi = lo;
    if (c_le < k + 2) hi = block_min_greater(src, n, lo, kf, sh);
    return (lov + (double)kfloat(hi)) / 2.0;
}

__global__ void __launch_bounds__(SEL_THREADS) select_kernel(const SelectArgs a) {
    extern __shared__ __align__(16) unsigned char sel_raw[];
    SelShared& sh = *reinterpret_cast<SelShared*>(sel_raw);
    float* cache = reinterpret_cast<float*>(sel_raw + ((sizeof(SelShared) + 15) & ~size_t(15)));
    const int jj = blockIdx.x;
    const int q = blockIdx.y;
    const int j = a.j0 + jj;
    if (j >= a.m) return;
    const int64_t n = a.n;
    const float* yrow = a.y + ((size_t)q * a.jcount + jj) * n;
    const float* src = yrow;
    if (n <= SEL_CACHE_MAX) {
        if ((n & 3) == 0) {
            const float4* s4 = reinterpret_cast<const float4*>(yrow);
            float4* c4 = reinterpret_cast<float4*>(cache);
            for (int64_t i = threadIdx.x; i < n / 4; i += SEL_THREADS) c4[i] = __ldg(s4 + i);
        } else {
            for (int64_t i = threadIdx.x; i < n; i += SEL_THREADS) cache[i] = __ldg(yrow + i);
        }
        __syncthreads();
        src = cache;
    }
    const double med = block_median(src, n, n, KeyMed{}, sh);
    double depth;
    if (a.notion == 1) {
        const double mad = block_median(src, n, n, KeyAbsDev{med}, sh);
        const double dev = fabs(med);
        if (mad == 0.0) depth = (dev == 0.0) ? 1.0 : 0.0;
        else depth = 1.0 / (1.0 + dev / mad);
    } else {
        const double dev = -med;
        if (dev <= 0.0) {
            depth = 1.0;
        } else {
            int local = 0;
            for (int64_t i = threadIdx.x; i < n; i += SEL_THREADS) local += ((double)src[i] - med > 0.0);
            const int npos = block_sum(local, sh);
            if (npos == 0) depth = 0.0;
            else {
                const double madp = block_median(src, n, npos, KeyPosDev{med}, sh);
                depth = 1.0 / (1.0 + dev / madp);
            }
        }
    }
    if (threadIdx.x == 0) a.depths[(size_t)q * a.m + j] = depth;
}

cudaError_t launch_select(const SelectArgs& a, cudaStream_t st) {
    if (a.Qb == 0 || a.jcount == 0) return cudaSuccess;
    size_t smem = (sizeof(SelShared) + 15) & ~size_t(15);
    if (a.n <= SEL_CACHE_MAX) smem += (size_t)a.n * sizeof(float);
    cudaError_t e = cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid((unsigned)a.jcount, (unsigned)a.Qb);
    select_kernel<<<grid, SEL_THREADS, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace rrs
