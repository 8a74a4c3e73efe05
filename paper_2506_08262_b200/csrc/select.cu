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
#ifndef RRS_SEL_UNROLL
#define RRS_SEL_UNROLL 2
#endif
constexpr int SEL_UNROLL = RRS_SEL_UNROLL;  // float4 loads in flight per thread per pass

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
                                 SelShared& sh, int64_t& c_le, bool aligned4) {
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
        // 16-byte loads, SEL_UNROLL in flight per thread (the row streams from
        // HBM/L2 when it exceeds shared memory: bytes in flight set the rate)
        const auto add = [&](float y, bool valid) {
            int bin = -1;
            uint32_t key;
            if (valid && kf(y, key) && (key & pmask) == prefix) bin = (int)((key >> shift) & bmask);
            const unsigned grp = __match_any_sync(0xffffffffu, bin);
            if (bin >= 0 && lane == __ffs(grp) - 1) atomicAdd(&sh.hist[bin], __popc(grp));
        };
        const int64_t n4 = aligned4 ? (n >> 2) : 0;
        const float4* s4 = reinterpret_cast<const float4*>(src);
        for (int64_t base = (int64_t)warp * 32 * SEL_UNROLL; base < n4; base += (int64_t)SEL_WARPS * 32 * SEL_UNROLL) {
            float4 v[SEL_UNROLL];
#pragma unroll
            for (int u = 0; u < SEL_UNROLL; ++u) {
                const int64_t i = base + u * 32 + lane;
                v[u] = i < n4 ? s4[i] : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < SEL_UNROLL; ++u) {
                const bool ok = base + u * 32 + lane < n4;
                add(v[u].x, ok);
                add(v[u].y, ok);
                add(v[u].z, ok);
                add(v[u].w, ok);
            }
        }
        for (int64_t b0 = 4 * n4 + (int64_t)warp * 32; b0 < n; b0 += (int64_t)SEL_WARPS * 32) {
            const int64_t i = b0 + lane;
            add(i < n ? src[i] : 0.f, i < n);
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
                                      SelShared& sh, bool aligned4) {
    uint32_t best = 0xFFFFFFFFu;
    const auto take = [&](float y) {
        uint32_t k2;
        if (kf(y, k2) && k2 > key && k2 < best) best = k2;
    };
    const int64_t n4 = aligned4 ? (n >> 2) : 0;
    const float4* s4 = reinterpret_cast<const float4*>(src);
    for (int64_t base = threadIdx.x; base < n4; base += (int64_t)SEL_THREADS * SEL_UNROLL) {
        float4 v[SEL_UNROLL];
#pragma unroll
        for (int u = 0; u < SEL_UNROLL; ++u) {
            const int64_t i = base + (int64_t)u * SEL_THREADS;
            v[u] = i < n4 ? s4[i] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < SEL_UNROLL; ++u)
            if (base + (int64_t)u * SEL_THREADS < n4) {
                take(v[u].x);
                take(v[u].y);
                take(v[u].z);
                take(v[u].w);
            }
    }
    for (int64_t i = 4 * n4 + threadIdx.x; i < n; i += SEL_THREADS) take(src[i]);
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
                               SelShared& sh, bool aligned4) {
    const int64_t k = (cnt - 1) >> 1;
    int64_t c_le;
    const uint32_t lo = block_select(src, n, k, kf, sh, c_le, aligned4);
    const double lov = (double)kfloat(lo);
    if (cnt & 1) return lov;
    uint32_t hi = lo;
    if (c_le < k + 2) hi = block_min_greater(src, n, lo, kf, sh, aligned4);
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
    // rows start 16-byte aligned when n % 4 == 0 (y is [Qb][jcount][n] floats)
    const bool al = (n & 3) == 0;
    const double med = block_median(src, n, n, KeyMed{}, sh, al);
    const double medz = med + (a.shift ? a.shift[(size_t)q * a.m + j] : 0.0);  // med(y) - 0 (centred frame)
    double depth;
    if (a.notion == 1) {
        const double mad = block_median(src, n, n, KeyAbsDev{med}, sh, al);
        const double dev = fabs(medz);
        if (mad == 0.0) depth = (dev == 0.0) ? 1.0 : 0.0;
        else depth = 1.0 / (1.0 + dev / mad);
    } else {
        const double dev = -medz;
        if (dev <= 0.0) {
            depth = 1.0;
        } else {
            int local = 0;
            const int64_t n4 = al ? (n >> 2) : 0;
            const float4* s4 = reinterpret_cast<const float4*>(src);
            for (int64_t i = threadIdx.x; i < n4; i += SEL_THREADS) {
                const float4 v = s4[i];
                local += ((double)v.x - med > 0.0) + ((double)v.y - med > 0.0) + ((double)v.z - med > 0.0) +
                         ((double)v.w - med > 0.0);
            }
            for (int64_t i = 4 * n4 + threadIdx.x; i < n; i += SEL_THREADS) local += ((double)src[i] - med > 0.0);
            const int npos = block_sum(local, sh);
            if (npos == 0) depth = 0.0;
            else {
                const double madp = block_median(src, n, npos, KeyPosDev{med}, sh, al);
                depth = 1.0 / (1.0 + dev / madp);
            }
        }
    }
    if (threadIdx.x == 0) a.depths[(size_t)q * a.m + j] = depth;
}

// ---------------------------------------------------------------- K3 v2 --
// Rows up to SEL2_MAX_N (config 3: n = 50k) live in shared memory as
// order-preserving uint32 keys; one CTA (256 threads) per direction.
//   * k-th smallest key: radix select on 8-bit digits starting below the
//     common prefix of the row's min and max keys (digits every key shares are
//     skipped), per-warp privatised 256-bin histograms, one 256-bin scan per
//     pass (one bin per thread);
//   * even counts take the midpoint with the next larger key (one min pass);
//   * the MAD / positive-deviation keys are rewritten in place once (FP64
//     deviation, FP32 key) instead of being recomputed every pass.
// Same arithmetic as select_kernel: FP32 order statistics, FP64 midpoints and
// deviations (_kernels.pyx:202-351).
constexpr int64_t SEL2_MAX_N = 53248;  // 208 KB of keys
// 256 threads for rows up to SEL2_WIDE_N, 512 up to SEL2_WIDER_N, 1024 above
// (one CTA per SM at n = 50k: more warps in flight for the latency-bound passes)
#ifndef RRS_SEL2_WIDE_N
#define RRS_SEL2_WIDE_N 16384
#endif
constexpr int64_t SEL2_WIDE_N = RRS_SEL2_WIDE_N;
#ifndef RRS_SEL2_WIDER_N
#define RRS_SEL2_WIDER_N 24576
#endif
constexpr int64_t SEL2_WIDER_N = RRS_SEL2_WIDER_N;

// hist[(key >> shift) & 255] += 1 when (key & pmask) == prefix: a predicated
// red.shared (no branch / reconvergence per element)
__device__ __forceinline__ void hist_add_if(uint32_t* h, uint32_t key, uint32_t pmask, uint32_t prefix, int shift) {
    const uint32_t addr = smem_u32(h + ((key >> shift) & 255u));
    asm volatile(
        "{\n.reg .pred p;\nsetp.eq.u32 p, %0, %1;\n@p red.shared.add.u32 [%2], 1;\n}\n" ::"r"(key & pmask),
        "r"(prefix), "r"(addr)
        : "memory");
}

// hist[key >> 24] += 1 (the first radix digit, counted while the keys are written)
#ifdef RRS_SEL_NO_PREHIST
constexpr bool SEL2_PRE = false;
#else
constexpr bool SEL2_PRE = true;
#endif
__device__ __forceinline__ void hist_top_add(uint32_t* h, uint32_t key) {
    if (SEL2_PRE) asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(smem_u32(h + (key >> 24))) : "memory");
}

template <int NT>
struct Sel2Shared {
    static constexpr int W = NT / 32;
    static constexpr int H = W < 16 ? W : 16;  // histograms (warps w and w + 16 share one at NT = 1024)
    uint32_t hist[H][256];
    uint32_t wsum[W];
    uint32_t s_kmin, s_kmax;
    int s_bin;
    uint32_t s_below;
    uint32_t s_cnt;
    uint32_t s_cc, s_above;  // candidate compaction (global-memory rows)
};

// Global-memory rows (GLB): once a pass leaves <= SEL2G_CAP keys under the
// chosen prefix with >= 2 digits to go, the next full pass also appends them to
// a shared-memory candidate buffer (warp-aggregated) and records the smallest
// key above the prefix; the remaining passes and the even-median next-key
// search then read the buffer, not the row (the row streams from HBM: each
// saved pass is 4 n bytes).  Not used for shared-memory rows, where the ballot
// per key costs more than the passes it saves.
#ifndef RRS_SEL2G_CAP
#define RRS_SEL2G_CAP 16384
#endif
constexpr int SEL2G_CAP = RRS_SEL2G_CAP;
struct Sel2Cands {
    uint32_t* buf = nullptr;  // null: no compaction
    bool on = false;
    int count = 0;
    uint32_t above = 0xFFFFFFFFu;
};

template <int NT>
__device__ __forceinline__ uint32_t block_reduce_min(uint32_t v, Sel2Shared<NT>& sh) {
    v = __reduce_min_sync(0xffffffffu, v);
    if ((threadIdx.x & 31) == 0) sh.wsum[threadIdx.x >> 5] = v;
    __syncthreads();
    uint32_t r = 0xFFFFFFFFu;
    for (int w = 0; w < NT / 32; ++w) r = min(r, sh.wsum[w]);
    __syncthreads();
    return r;
}
template <int NT>
__device__ __forceinline__ uint32_t block_reduce_add(uint32_t v, Sel2Shared<NT>& sh) {
    v = __reduce_add_sync(0xffffffffu, v);
    if ((threadIdx.x & 31) == 0) sh.wsum[threadIdx.x >> 5] = v;
    __syncthreads();
    uint32_t r = 0;
    for (int w = 0; w < NT / 32; ++w) r += sh.wsum[w];
    __syncthreads();
    return r;
}

// k-th smallest (0-based) of keys[0, n) whose values lie in [kmin, kmax];
// c_le = number of keys <= the result.  cand.buf != null enables candidate
// compaction (see Sel2Cands).
template <int NT>
__device__ uint32_t sel2_kth(const uint32_t* __restrict__ keys, int n, uint32_t k, uint32_t kmin, uint32_t kmax,
                             Sel2Shared<NT>& sh, uint32_t& c_le, bool pre, Sel2Cands& cand) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t* src = keys;
    int nsrc = n;
    cand.on = false;
    cand.count = 0;
    cand.above = 0xFFFFFFFFu;
    const uint32_t diff = kmin ^ kmax;
    if (diff == 0u) {
        c_le = (uint32_t)n;
        return kmin;
    }
    const int top = 31 - __clz(diff);            // highest differing bit
    int shift = (top >= 24) ? 24 : (top >= 16) ? 16 : (top >= 8) ? 8 : 0;
    uint32_t pmask = shift + 8 >= 32 ? 0u : ~((1u << (shift + 8)) - 1u);
    uint32_t prefix = kmin & pmask;                // digits above `shift` are common
    uint32_t below_total = 0, last = 0xFFFFFFFFu;
    // pre: the pass that wrote the keys already histogrammed their top digit
    // (bits 24..31) into sh.hist; use it when the first pass starts there
    bool skip_count = pre && shift == 24;
    for (;;) {
        uint32_t* h = sh.hist[warp % Sel2Shared<NT>::H];
        const bool compact = cand.buf != nullptr && !cand.on && shift >= 8 && last <= (uint32_t)SEL2G_CAP;
        if (!skip_count) {
            for (int b = lane; b < 256; b += 32) h[b] = 0u;
            if (compact && tid == 0) {
                sh.s_cc = 0u;
                sh.s_above = 0xFFFFFFFFu;
            }
            __syncthreads();
            if (!compact) {
                // 4 keys per 16-byte load; rows are 16-byte aligned, the tail is scalar;
                // two loads issued before the (memory-clobbering) histogram updates
                const int n4 = nsrc >> 2;
                const uint4* s4 = reinterpret_cast<const uint4*>(src);
                int i = tid;
                for (; i + NT < n4; i += 2 * NT) {
                    const uint4 ka = s4[i], kb = s4[i + NT];
                    hist_add_if(h, ka.x, pmask, prefix, shift);
                    hist_add_if(h, ka.y, pmask, prefix, shift);
                    hist_add_if(h, ka.z, pmask, prefix, shift);
                    hist_add_if(h, ka.w, pmask, prefix, shift);
                    hist_add_if(h, kb.x, pmask, prefix, shift);
                    hist_add_if(h, kb.y, pmask, prefix, shift);
                    hist_add_if(h, kb.z, pmask, prefix, shift);
                    hist_add_if(h, kb.w, pmask, prefix, shift);
                }
                if (i < n4) {
                    const uint4 k4 = s4[i];
                    hist_add_if(h, k4.x, pmask, prefix, shift);
                    hist_add_if(h, k4.y, pmask, prefix, shift);
                    hist_add_if(h, k4.z, pmask, prefix, shift);
                    hist_add_if(h, k4.w, pmask, prefix, shift);
                }
                for (int t = 4 * n4 + tid; t < nsrc; t += NT) hist_add_if(h, src[t], pmask, prefix, shift);
            } else {
                // the same histogram, plus the keys under the prefix appended to the
                // buffer and the smallest key above it
                uint32_t amin = 0xFFFFFFFFu;
                const auto visit = [&](uint32_t key, bool valid) {
                    const uint32_t hi = key & pmask;
                    const bool match = valid && hi == prefix;
                    if (valid && hi > prefix) amin = min(amin, key);
                    if (match) hist_add_if(h, key, pmask, prefix, shift);
                    const unsigned bal = __ballot_sync(0xffffffffu, match);
                    if (bal) {
                        const int leader = __ffs(bal) - 1;
                        uint32_t base = 0;
                        if (lane == leader) base = atomicAdd(&sh.s_cc, (uint32_t)__popc(bal));
                        base = __shfl_sync(0xffffffffu, base, leader);
                        if (match) cand.buf[base + __popc(bal & ((1u << lane) - 1u))] = key;
                    }
                };
                const int n4 = nsrc >> 2;
                const uint4* s4 = reinterpret_cast<const uint4*>(src);
                // warp-uniform trip counts (ballots need every lane)
                for (int i0 = warp * 32; i0 < n4; i0 += NT) {
                    const int i = i0 + lane;
                    const bool ok = i < n4;
                    const uint4 k4 = ok ? s4[i] : make_uint4(0u, 0u, 0u, 0u);
                    visit(k4.x, ok);
                    visit(k4.y, ok);
                    visit(k4.z, ok);
                    visit(k4.w, ok);
                }
                for (int t0 = 4 * n4 + warp * 32; t0 < nsrc; t0 += NT) {
                    const int t = t0 + lane;
                    visit(t < nsrc ? src[t] : 0u, t < nsrc);
                }
                amin = __reduce_min_sync(0xffffffffu, amin);
                if (lane == 0 && amin != 0xFFFFFFFFu) atomicMin(&sh.s_above, amin);
            }
        }
        skip_count = false;
        __syncthreads();
        // bin totals (thread b < 256 owns bin b), exclusive scan over the 256 bins
        uint32_t tot = 0;
        if (tid < 256)
#pragma unroll
            for (int w = 0; w < Sel2Shared<NT>::H; ++w) tot += sh.hist[w][tid];
        uint32_t incl = tot;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t o = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += o;
        }
        if (lane == 31 && warp < 8) sh.wsum[warp] = incl;
        __syncthreads();
        if (tid < 256) {
            uint32_t woff = 0;
            for (int w = 0; w < warp; ++w) woff += sh.wsum[w];
            const uint32_t excl = woff + incl - tot;
            if (excl <= k && k < excl + tot) {
                sh.s_bin = tid;
                sh.s_below = excl;
                sh.s_cnt = tot;
            }
        }
        __syncthreads();
        const uint32_t bin = (uint32_t)sh.s_bin;
        k -= sh.s_below;
        below_total += sh.s_below;
        last = sh.s_cnt;
        if (compact) {
            cand.on = true;
            cand.count = (int)sh.s_cc;
            cand.above = sh.s_above;
            src = cand.buf;
            nsrc = cand.count;
        }
        prefix |= bin << shift;
        pmask |= 255u << shift;
        __syncthreads();
        if (shift == 0) break;
        shift -= 8;
    }
    c_le = below_total + last;
    return prefix;
}

template <int NT>
__device__ uint32_t sel2_min_greater(const uint32_t* __restrict__ keys, int n, uint32_t key, Sel2Shared<NT>& sh) {
    // min over keys > key: map keys <= key to 0xFFFFFFFF (key + 1 .. wraps only for key = max)
    uint32_t best = 0xFFFFFFFFu;
    const int n4 = n >> 2;
    const uint4* s4 = reinterpret_cast<const uint4*>(keys);
    for (int i = threadIdx.x; i < n4; i += NT) {
        const uint4 k4 = s4[i];
        best = min(best, k4.x > key ? k4.x : 0xFFFFFFFFu);
        best = min(best, k4.y > key ? k4.y : 0xFFFFFFFFu);
        best = min(best, k4.z > key ? k4.z : 0xFFFFFFFFu);
        best = min(best, k4.w > key ? k4.w : 0xFFFFFFFFu);
    }
    for (int i = 4 * n4 + threadIdx.x; i < n; i += NT) {
        const uint32_t k2 = keys[i];
        if (k2 > key && k2 < best) best = k2;
    }
    return block_reduce_min(best, sh);
}

// median of the first `cnt` order statistics' centre: keys outside the
// participating set must be larger than every participant (0xFFFFFFFF)
template <int NT>
__device__ double sel2_median(const uint32_t* __restrict__ keys, int n, uint32_t cnt, uint32_t kmin, uint32_t kmax,
                              Sel2Shared<NT>& sh, bool pre, uint32_t* cbuf) {
    const uint32_t k = (cnt - 1) >> 1;
    uint32_t c_le;
    Sel2Cands cand;
    cand.buf = cbuf;
    const uint32_t lo = sel2_kth(keys, n, k, kmin, kmax, sh, c_le, pre, cand);
    const double lov = (double)kfloat(lo);
    if (cnt & 1) return lov;
    uint32_t hi = lo;
    if (c_le < k + 2) {
        // keys above lo are candidates (same prefix) or at least cand.above
        hi = cand.on ? min(cand.above, sel2_min_greater(cand.buf, cand.count, lo, sh))
                     : sel2_min_greater(keys, n, lo, sh);
    }
    return (lov + (double)kfloat(hi)) / 2.0;
}

// GLB = false: the row's keys live in shared memory (n <= SEL2_MAX_N).
// GLB = true: rows too long for shared memory; the keys are written over the
// row's own projections in global memory (the row belongs to this CTA and is
// dead after the select) and every pass streams them from L2 / HBM.
template <int NT, bool GLB>
__global__ void __launch_bounds__(NT) select_v2_kernel(const SelectArgs a) {
    extern __shared__ __align__(16) unsigned char sel2_raw[];
    Sel2Shared<NT>& sh = *reinterpret_cast<Sel2Shared<NT>*>(sel2_raw);
    const int jj = blockIdx.x;
    const int q = blockIdx.y;
    const int j = a.j0 + jj;
    if (j >= a.m) return;
    const int n = (int)a.n;
    const float* yrow = a.y + ((size_t)q * a.jcount + jj) * a.n;
    uint32_t* keys = GLB ? const_cast<uint32_t*>(reinterpret_cast<const uint32_t*>(yrow))
                         : reinterpret_cast<uint32_t*>(sel2_raw + ((sizeof(Sel2Shared<NT>) + 15) & ~size_t(15)));
    uint32_t* cbuf = GLB && SEL2G_CAP > 0
                         ? reinterpret_cast<uint32_t*>(sel2_raw + ((sizeof(Sel2Shared<NT>) + 15) & ~size_t(15)))
                         : nullptr;
    uint32_t* htop = sh.hist[(threadIdx.x >> 5) % Sel2Shared<NT>::H];
    const auto clear_top = [&]() {
        for (int b = threadIdx.x & 31; b < 256; b += 32) htop[b] = 0u;
        __syncthreads();
    };
    clear_top();
    uint32_t kmin = 0xFFFFFFFFu, kmax = 0u;
    if ((n & 3) == 0) {
        const float4* s4 = reinterpret_cast<const float4*>(yrow);
        uint4* k4 = reinterpret_cast<uint4*>(keys);
        for (int i = threadIdx.x; i < n / 4; i += NT) {
            const float4 v = s4[i];
            const uint4 k = make_uint4(fkey(v.x), fkey(v.y), fkey(v.z), fkey(v.w));
            k4[i] = k;
            hist_top_add(htop, k.x);
            hist_top_add(htop, k.y);
            hist_top_add(htop, k.z);
            hist_top_add(htop, k.w);
            kmin = min(kmin, min(min(k.x, k.y), min(k.z, k.w)));
            kmax = max(kmax, max(max(k.x, k.y), max(k.z, k.w)));
        }
    } else {
        for (int i = threadIdx.x; i < n; i += NT) {
            const uint32_t k = fkey(yrow[i]);
            keys[i] = k;
            hist_top_add(htop, k);
            kmin = min(kmin, k);
            kmax = max(kmax, k);
        }
    }
    __syncthreads();
    kmin = block_reduce_min(kmin, sh);
    kmax = ~block_reduce_min(~kmax, sh);
    const double med = sel2_median(keys, n, (uint32_t)n, kmin, kmax, sh, SEL2_PRE, cbuf);
    const double medz = med + (a.shift ? a.shift[(size_t)q * a.m + j] : 0.0);  // med(y) - 0 (centred frame)
    double depth;
    if (a.notion == 1) {
        // MAD: keys of |y - med| (FP64 deviation, FP32 key), in place
        clear_top();
        uint32_t dmin = 0xFFFFFFFFu, dmax = 0u;
        for (int i = threadIdx.x; i < n; i += NT) {
            const uint32_t k = fkey((float)fabs((double)kfloat(keys[i]) - med));
            keys[i] = k;
            hist_top_add(htop, k);
            dmin = min(dmin, k);
            dmax = max(dmax, k);
        }
        __syncthreads();
        dmin = block_reduce_min(dmin, sh);
        dmax = ~block_reduce_min(~dmax, sh);
        const double mad = sel2_median(keys, n, (uint32_t)n, dmin, dmax, sh, SEL2_PRE, cbuf);
        const double dev = fabs(medz);
        if (mad == 0.0) depth = (dev == 0.0) ? 1.0 : 0.0;
        else depth = 1.0 / (1.0 + dev / mad);
    } else {
        const double dev = -medz;
        if (dev <= 0.0) {
            depth = 1.0;
        } else {
            // positive deviations y - med > 0 keep their key, the rest sort last
            // (the markers land in top bin 255 exactly as in a counting pass)
            clear_top();
            uint32_t dmin = 0xFFFFFFFFu, dmax = 0u, npos = 0;
            for (int i = threadIdx.x; i < n; i += NT) {
                const double t = (double)kfloat(keys[i]) - med;
                uint32_t k = 0xFFFFFFFFu;
                if (t > 0.0) {
                    k = fkey((float)t);
                    ++npos;
                    dmin = min(dmin, k);
                    dmax = max(dmax, k);
                }
                keys[i] = k;
                hist_top_add(htop, k);
            }
            __syncthreads();
            npos = block_reduce_add(npos, sh);
            dmin = block_reduce_min(dmin, sh);
            dmax = ~block_reduce_min(~dmax, sh);
            if (npos == 0) depth = 0.0;
            else {
                // participants are the npos smallest keys; select within [dmin, dmax]
                // (the 0xFFFFFFFF markers never match the prefix of a participant)
                const double madp = sel2_median(keys, n, npos, dmin, dmax, sh, SEL2_PRE, cbuf);
                depth = 1.0 / (1.0 + dev / madp);
            }
        }
    }
    if (threadIdx.x == 0) a.depths[(size_t)q * a.m + j] = depth;
}

// ---------------------------------------------------------------- K3 v3 --
// Sample-bracket select (Floyd-Rivest).  The row is never copied: every pass
// streams the projections y (FP32) from L2 / HBM and turns them into keys on
// the fly.
//   1. One warp sorts 256 keys taken at strided positions (register bitonic,
//      8 keys per lane); for a target rank R of n keys the sample order
//      statistics at R·S/n -/+ ~3 sigma give a bracket [lo, hi].
//   2. ONE branch-free pass over the row counts the keys below lo (per-thread
//      counters) and appends the keys inside the bracket to per-thread
//      shared-memory slots (slot c of thread t at c·NT + t: bank-conflict
//      free, no ballots, no atomics).
//   3. The slots are compacted into one contiguous array (block scan of the
//      per-thread counts) and rank R - #below is selected there by v2's radix
//      passes (16-byte loads, per-warp histograms), starting below the common
//      prefix of lo and hi.
// Projection depth: median (pass 1), MAD (pass 2: the bracket comes from the
// sample's deviations, ranked by a merge of the two monotone halves).
// Asymmetric projection depth: median (pass 1), then the positive-deviation
// median is the key at global rank c_le(med) + (npos-1)/2 of the SAME keys
// (rounding y - med to FP32 is monotone in y), so pass 2 brackets that rank.
// A row whose target leaves its bracket (or whose thread overflows its
// slots) falls back to full radix passes over the row; counted in
// a.fallbacks.  The arithmetic is v2's (FP32 keys, FP64 midpoints /
// deviations), so v2 and v3 give bitwise equal depths.
// sample size: one warp sorts it (8 / 16 keys per lane); the larger sample of
// the 1024-thread variant narrows the bracket so 1024 threads' slots rarely overflow
#ifndef RRS_S3_MINB256
#define RRS_S3_MINB256 5
#endif
#ifndef RRS_S3_MINB512
#define RRS_S3_MINB512 3  // config 3: 274 -> 284 q/s over 2
#endif
template <int NT>
struct Sel3Cfg {
    static constexpr int S = NT >= 512 ? 512 : 256;
    static constexpr double SIGMAS = NT >= 1024 ? 5.0 : 4.0;  // slot headroom
    static constexpr int MINB = NT >= 1024 ? 1 : NT >= 512 ? RRS_S3_MINB512 : RRS_S3_MINB256;  // CTAs per SM targeted
};
constexpr int SMAX = 512;
constexpr int64_t SEL3_MIN_N = 2048;
constexpr int64_t SEL3_MAX_N = 53248;

constexpr int S3_BITS = 10, S3_BINS = 1 << S3_BITS;  // digit width of the candidate select

template <int NT>
struct Sel3Shared {
    static constexpr int W = NT / 32;
    // hist (candidate select) and sdev (sample-sort scratch, the MAD sample's
    // deviations) are never live at the same time
    union {
        alignas(16) uint32_t hist[S3_BINS];
        uint32_t sdev[Sel3Cfg<NT>::S];
    };
    alignas(16) uint32_t sorted[Sel3Cfg<NT>::S];  // sorted sample keys (deviation keys for the MAD)
    uint32_t tiny[32];
    uint32_t wsum[W];
    uint32_t s_bin, s_below, s_cnt, s_ntiny, s_ovf, s_res, s_cle;
};

template <int NT>
__device__ __forceinline__ uint32_t s3_reduce_add(uint32_t v, Sel3Shared<NT>& sh) {
    v = __reduce_add_sync(0xffffffffu, v);
    if ((threadIdx.x & 31) == 0) sh.wsum[threadIdx.x >> 5] = v;
    __syncthreads();
    uint32_t r = 0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) r += sh.wsum[w];
    __syncthreads();
    return r;
}
template <int NT>
__device__ __forceinline__ uint32_t s3_reduce_min(uint32_t v, Sel3Shared<NT>& sh) {
    v = __reduce_min_sync(0xffffffffu, v);
    if ((threadIdx.x & 31) == 0) sh.wsum[threadIdx.x >> 5] = v;
    __syncthreads();
    uint32_t r = 0xFFFFFFFFu;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) r = min(r, sh.wsum[w]);
    __syncthreads();
    return r;
}

// every thread calls f(y) for its share of the row (16-byte loads when aligned,
// U in flight)
template <int NT, int U = 4, typename F>
__device__ __forceinline__ void s3_row_each(const float* __restrict__ row, int n, F&& f) {
    if ((n & 3) == 0) {
        const float4* r4 = reinterpret_cast<const float4*>(row);
        const int n4 = n >> 2;
        int i = threadIdx.x;
        for (; i + (U - 1) * NT < n4; i += U * NT) {
            float4 v[U];
#pragma unroll
            for (int k = 0; k < U; ++k) v[k] = __ldg(r4 + i + k * NT);
#pragma unroll
            for (int k = 0; k < U; ++k) f(v[k].x), f(v[k].y), f(v[k].z), f(v[k].w);
        }
        for (; i < n4; i += NT) {
            const float4 v = __ldg(r4 + i);
            f(v.x), f(v.y), f(v.z), f(v.w);
        }
    } else {
        for (int i = threadIdx.x; i < n; i += NT) f(__ldg(row + i));
    }
}

// contiguous shared-memory keys [0, cnt): 16-byte loads (cand is 16-byte aligned)
template <int NT, typename F>
__device__ __forceinline__ void s3_arr_each(const uint32_t* __restrict__ cand, int cnt, F&& f) {
    const uint4* c4 = reinterpret_cast<const uint4*>(cand);
    const int n4 = cnt >> 2;
    for (int i = threadIdx.x; i < n4; i += NT) {
        const uint4 v = c4[i];
        f(v.x), f(v.y), f(v.z), f(v.w);
    }
    for (int i = 4 * n4 + threadIdx.x; i < cnt; i += NT) f(cand[i]);
}

// t-th smallest (0-based) of the keys enumerated by each(f), all of which lie
// in [lo, hi] (total of them: count); c_le = number of them <= the result.
// Histograms of 10-bit digits of the offset key - lo in shared memory (one
// 1024-bin histogram, predicated red.shared), starting at the top bit of
// hi - lo; once the chosen bin holds <= 32 keys they are gathered and one warp
// ranks them.
template <int NT, typename Each>
__device__ uint32_t s3_kth(Each&& each, uint32_t t, uint32_t lo, uint32_t hi, uint32_t count, Sel3Shared<NT>& sh,
                           uint32_t& c_le) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int PER = S3_BINS / NT;  // bins per thread in the scan
    uint32_t base = lo, span = hi - lo, below = 0, wcnt = count;
    for (;;) {
        if (span == 0u) {  // one key value left in the window
            c_le = below + wcnt;
            return base;
        }
        if (wcnt <= 32u) {
            // gather the window's keys, rank them in one warp
            if (tid == 0) sh.s_ntiny = 0u;
            __syncthreads();
            each([&](uint32_t key) {
                if (key - base <= span) sh.tiny[atomicAdd(&sh.s_ntiny, 1u)] = key;
            });
            __syncthreads();
            if (warp == 0) {
                const uint32_t mine = (uint32_t)lane < wcnt ? sh.tiny[lane] : 0xFFFFFFFFu;
                uint32_t lt = 0, eq_before = 0, le = 0;
                for (int j2 = 0; j2 < (int)wcnt; ++j2) {
                    const uint32_t o = __shfl_sync(0xffffffffu, mine, j2);
                    lt += o < mine;
                    eq_before += (o == mine && j2 < lane);
                }
                const uint32_t rank = lt + eq_before;
                if ((uint32_t)lane < wcnt && rank == t) sh.s_res = mine;
                __syncwarp();
                const uint32_t res = sh.s_res;
                for (int j2 = 0; j2 < (int)wcnt; ++j2) le += __shfl_sync(0xffffffffu, mine, j2) <= res;
                if (lane == 0) sh.s_cle = below + le;
            }
            __syncthreads();
            c_le = sh.s_cle;
            return sh.s_res;
        }
        const int bits = 32 - __clz(span);
        const int shift = bits > S3_BITS ? bits - S3_BITS : 0;
        {
            uint4* h4 = reinterpret_cast<uint4*>(sh.hist);
            for (int i = tid; i < S3_BINS / 4; i += NT) h4[i] = make_uint4(0u, 0u, 0u, 0u);
        }
        __syncthreads();
        const uint32_t hbase = smem_u32(sh.hist);
        each([&](uint32_t key) {
            const uint32_t off = key - base;
            const uint32_t addr = hbase + ((off >> shift) << 2);
            asm volatile("{\n.reg .pred p;\nsetp.le.u32 p, %0, %1;\n@p red.shared.add.u32 [%2], 1;\n}\n" ::"r"(off),
                         "r"(span), "r"(addr)
                         : "memory");
        });
        __syncthreads();
        // exclusive scan over the bins (PER consecutive bins per thread; PER >= 1)
        uint32_t hv[PER > 0 ? PER : 1];
        uint32_t local = 0;
#pragma unroll
        for (int b = 0; b < PER; ++b) {
            hv[b] = sh.hist[tid * PER + b];
            local += hv[b];
        }
        uint32_t incl = local;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t o = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += o;
        }
        if (lane == 31) sh.wsum[warp] = incl;
        __syncthreads();
        uint32_t run = incl - local;
        for (int w = 0; w < warp; ++w) run += sh.wsum[w];
        if (run <= t && t < run + local) {
#pragma unroll
            for (int b = 0; b < PER; ++b) {
                if (run <= t && t < run + hv[b]) {
                    sh.s_bin = (uint32_t)(tid * PER + b);
                    sh.s_below = run;
                    sh.s_cnt = hv[b];
                }
                run += hv[b];
            }
        }
        __syncthreads();
        const uint32_t bin = sh.s_bin;
        t -= sh.s_below;
        below += sh.s_below;
        wcnt = sh.s_cnt;
        const uint32_t start = bin << shift;
        base += start;
        span = min(span - start, (shift ? (1u << shift) : 1u) - 1u);
        __syncthreads();
    }
}

// sort the S sample keys (thread t < S holds one): each warp sorts its 32 by
// a shuffle bitonic network, then every key's rank is its lane plus, in every
// other chunk, the count of keys below it (ties go to the lower chunk) found
// by a branch-free binary search -- all S/32 warps work, no warp waits on one
template <int NT>
__device__ __forceinline__ void s3_sort_sample(uint32_t v, Sel3Shared<NT>& sh) {
    constexpr int S = Sel3Cfg<NT>::S, C = S / 32;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    if (w < C) {
#pragma unroll
        for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
            for (int j = k >> 1; j > 0; j >>= 1) {
                const uint32_t o = __shfl_xor_sync(0xffffffffu, v, j);
                const bool keep_min = ((lane & j) == 0) == ((lane & k) == 0);
                v = keep_min ? min(v, o) : max(v, o);
            }
        }
        sh.sdev[tid] = v;
    }
    __syncthreads();
    if (w < C) {
        uint32_t rank = (uint32_t)lane;
#pragma unroll
        for (int c = 0; c < C; ++c) {
            if (c == w) continue;
            const uint32_t* ch = sh.sdev + 32 * c;
            // count of t < vv: t <= v for an earlier chunk (its equal keys rank
            // first), t < v for a later one; keys of finite floats are < 2^32 - 1
            const uint32_t vv = v + (c < w ? 1u : 0u);
            uint32_t pos = 0;
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) pos += ch[pos + step - 1] < vv ? (uint32_t)step : 0u;
            rank += pos + (ch[pos] < vv ? 1u : 0u);
        }
        sh.sorted[rank] = v;
    }
    __syncthreads();
}

// bracket [lo, hi] of population ranks [R, R2] of N keys from a sorted sample of S
template <int S>
__device__ __forceinline__ void s3_bracket(const uint32_t* sorted, uint32_t R, uint32_t R2, uint32_t N, uint32_t& lo,
                                           uint32_t& hi) {
    const float p = ((float)R + 0.5f) / (float)N;
    const float M = 3.0f * sqrtf((float)S * fmaxf(p * (1.0f - p), 1.0f / S)) + 2.0f;
    const float ra = ((float)R + 0.5f) * S / (float)N - 0.5f - M;
    const float rb = ((float)R2 + 0.5f) * S / (float)N - 0.5f + M;
    const int a = (int)floorf(ra), b = (int)ceilf(rb);
    lo = a < 0 ? 0u : sorted[a];
    hi = b >= S ? 0xFFFFFFFFu : sorted[b];
}

// keys at ranks R and R + 1 (if need_next) of the n keys kf(y) over the row;
// c_le = number of keys <= key(R).  Returns false when the bracket missed or
// a thread's slots overflowed (the caller falls back).
template <int NT, typename KF>
__device__ bool s3_select(const float* __restrict__ row, int n, KF kf, uint32_t R, bool need_next, uint32_t lo,
                          uint32_t hi, uint32_t* slots, int cap, int cmax, uint32_t* cand, Sel3Shared<NT>& sh, uint32_t& kR,
                          uint32_t& kN, uint32_t& c_le) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t span = hi - lo;
    uint32_t below = 0;
    const uint32_t a0 = smem_u32(slots + tid);
    // slot overflow goes to one scratch slot past the thread's last one
    const uint32_t alim = a0 + (uint32_t)cap * NT * 4u;
    uint32_t addr = a0;
    __syncthreads();  // the previous selection's readers of the slots / candidates are done
    s3_row_each<NT>(row, n, [&](float y) {
        const uint32_t key = kf(y);
        asm volatile(
            "{\n.reg .pred pin, plo;\n.reg .u32 off, a;\n"
            "sub.u32 off, %2, %3;\n"
            "setp.le.u32 pin, off, %4;\n"
            "setp.lt.u32 plo, %2, %3;\n"
            "@plo add.u32 %0, %0, 1;\n"
            "min.u32 a, %1, %5;\n"
            "@pin st.shared.u32 [a], %2;\n"
            "@pin add.u32 %1, %1, %6;\n}\n"
            : "+r"(below), "+r"(addr)
            : "r"(key), "r"(lo), "r"(span), "r"(alim), "r"((uint32_t)(NT * 4))
            : "memory");
    });
    const uint32_t c = (addr - a0) / (NT * 4u);
    const bool ovf = c > (uint32_t)cap;
    // block exclusive scan of the per-thread candidate counts (c <= n < 2^16)
    // with the below counts packed in the high half (n < 2^16)
    const uint32_t v = (below << 16) | c;
    uint32_t incl = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += o;
    }
    const unsigned ovw = __ballot_sync(0xffffffffu, ovf);
    if (lane == 31) sh.wsum[warp] = incl;
    if (lane == 0 && ovw) sh.s_ovf = 1u;
    __syncthreads();
    uint32_t woff = 0, total = 0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) {
        const uint32_t t = sh.wsum[w];
        woff += w < warp ? t : 0u;
        total += t;
    }
    const uint32_t c_lo = total >> 16, c_mid = total & 0xFFFFu;
    const bool overflow = sh.s_ovf != 0u || c_mid > (uint32_t)cmax;
    if (overflow || R < c_lo || R >= c_lo + c_mid) return false;  // block-uniform
    // compact the slots into one contiguous array
    const uint32_t off = (woff + incl - v) & 0xFFFFu;
    {
        const uint32_t* sp = slots + tid;
        uint32_t* dp = cand + off;
        uint32_t i = 0;
        for (; i + 4 <= c; i += 4) {
            const uint32_t k0 = sp[i * NT], k1 = sp[(i + 1) * NT], k2 = sp[(i + 2) * NT], k3 = sp[(i + 3) * NT];
            dp[i] = k0;
            dp[i + 1] = k1;
            dp[i + 2] = k2;
            dp[i + 3] = k3;
        }
        for (; i < c; ++i) dp[i] = sp[i * NT];
    }
    __syncthreads();
    const auto each = [&](auto&& f) { s3_arr_each<NT>(cand, (int)c_mid, f); };
    uint32_t cl;
    kR = s3_kth<NT>(each, R - c_lo, lo, hi, c_mid, sh, cl);
    c_le = c_lo + cl;
    kN = kR;
    if (need_next && c_le < R + 2) {
        uint32_t best = 0xFFFFFFFFu;
        if (R + 1 >= c_lo + c_mid) {  // the next key lies above the bracket
            s3_row_each<NT>(row, n, [&](float y) {
                const uint32_t k2 = kf(y);
                best = min(best, k2 > hi ? k2 : 0xFFFFFFFFu);
            });
        } else {
            each([&](uint32_t k2) { best = min(best, k2 > kR ? k2 : 0xFFFFFFFFu); });
        }
        kN = s3_reduce_min<NT>(best, sh);
    }
    return true;
}

struct S3KeyY {
    __device__ __forceinline__ uint32_t operator()(float y) const { return fkey(y); }
};
struct S3KeyAbsDev {
    double med;
    __device__ __forceinline__ uint32_t operator()(float y) const { return fkey((float)fabs((double)y - med)); }
};

template <int NT, typename KF>
__device__ __forceinline__ void s3_rank(const float* row, int n, KF kf, uint32_t R, bool need_next,
                                        const uint32_t* sorted, uint32_t* slots, int cap, int cmax, uint32_t* cand,
                                        Sel3Shared<NT>& sh, uint32_t& kR, uint32_t& kN, uint32_t& c_le,
                                        unsigned* fallbacks) {
    uint32_t lo, hi;
    s3_bracket<Sel3Cfg<NT>::S>(sorted, R, need_next ? R + 1 : R, (uint32_t)n, lo, hi);
    if (!s3_select<NT>(row, n, kf, R, need_next, lo, hi, slots, cap, cmax, cand, sh, kR, kN, c_le)) {
        if (fallbacks && threadIdx.x == 0) atomicAdd(fallbacks, 1u);
        __syncthreads();
        if (threadIdx.x == 0) sh.s_ovf = 0u;
        const auto each = [&](auto&& f) { s3_row_each<NT>(row, n, [&](float y) { f(kf(y)); }); };
        kR = s3_kth<NT>(each, R, 0u, 0xFFFFFFFFu, (uint32_t)n, sh, c_le);
        kN = kR;
        if (need_next && c_le < R + 2) {
            uint32_t best = 0xFFFFFFFFu;
            each([&](uint32_t k2) { best = min(best, k2 > kR ? k2 : 0xFFFFFFFFu); });
            kN = s3_reduce_min<NT>(best, sh);
        }
    }
}

template <int NT>
__global__ void __launch_bounds__(NT, Sel3Cfg<NT>::MINB) select_v3_kernel(const SelectArgs a, int cap, int cmax) {
    extern __shared__ __align__(16) unsigned char sel3_raw[];
    Sel3Shared<NT>& sh = *reinterpret_cast<Sel3Shared<NT>*>(sel3_raw);
    const int jj = blockIdx.x;
    const int q = blockIdx.y;
    const int j = a.j0 + jj;
    if (j >= a.m) return;
    const int tid = threadIdx.x;
    const int n = (int)a.n;
    const float* row = a.y + ((size_t)q * a.jcount + jj) * a.n;
    uint32_t* slots = reinterpret_cast<uint32_t*>(sel3_raw + ((sizeof(Sel3Shared<NT>) + 15) & ~size_t(15)));
    uint32_t* cand = slots + (size_t)(cap + 1) * NT;  // 16-byte aligned: NT is a multiple of 4

    // sample: S strided keys of y, sorted
    constexpr int S = Sel3Cfg<NT>::S;
    uint32_t sv = 0u;
    if (tid < S) sv = fkey(__ldg(row + (int)(((int64_t)(2 * tid + 1) * n) / (2 * S))));
    if (tid == 0) sh.s_ovf = 0u;
    s3_sort_sample<NT>(sv, sh);

    // median of y (v2: midpoint of the central pair, FP64)
    const uint32_t k = (uint32_t)(n - 1) >> 1;
    const bool even = (n & 1) == 0;
    uint32_t kR, kN, c_le;
    s3_rank<NT>(row, n, S3KeyY{}, k, even, sh.sorted, slots, cap, cmax, cand, sh, kR, kN, c_le, a.fallbacks);
    const double lov = (double)kfloat(kR);
    const double med = even ? (lov + (double)kfloat(kN)) / 2.0 : lov;
    const double medz = med + (a.shift ? a.shift[(size_t)q * a.m + j] : 0.0);  // med(y) - 0 (centred frame)

    double depth;
    if (a.notion == 1) {
        // sample deviations: non-increasing over the sample's keys <= med,
        // non-decreasing above; rank each by a binary search in the other half
        uint32_t dk = 0u, le = 0u;
        if (tid < S) {
            const double yv = (double)kfloat(sh.sorted[tid]);
            dk = fkey((float)fabs(yv - med));
            le = yv <= med ? 1u : 0u;
            sh.sdev[tid] = dk;
        }
        const uint32_t nl = s3_reduce_add<NT>(le, sh);  // also orders the sdev writes
        if (tid < S) {
            uint32_t rank;
            if ((uint32_t)tid < nl) {
                // # of upper-half deviations < dk (sdev[nl..S) non-decreasing)
                uint32_t lo_i = nl, hi_i = S;
                while (lo_i < hi_i) {
                    const uint32_t mid = (lo_i + hi_i) >> 1;
                    if (sh.sdev[mid] < dk) lo_i = mid + 1;
                    else hi_i = mid;
                }
                rank = (nl - 1 - tid) + (lo_i - nl);
            } else {
                // # of lower-half deviations <= dk (sdev[0..nl) non-increasing: a suffix)
                uint32_t lo_i = 0, hi_i = nl;
                while (lo_i < hi_i) {
                    const uint32_t mid = (lo_i + hi_i) >> 1;
                    if (sh.sdev[mid] <= dk) hi_i = mid;
                    else lo_i = mid + 1;
                }
                rank = (tid - nl) + (nl - lo_i);
            }
            sh.sorted[rank] = dk;  // the sample's keys are dead after the median
        }
        __syncthreads();
        uint32_t mR, mN, mc;
        s3_rank<NT>(row, n, S3KeyAbsDev{med}, k, even, sh.sorted, slots, cap, cmax, cand, sh, mR, mN, mc, a.fallbacks);
        const double mlo = (double)kfloat(mR);
        const double mad = even ? (mlo + (double)kfloat(mN)) / 2.0 : mlo;
        const double dev = fabs(medz);
        if (mad == 0.0) depth = (dev == 0.0) ? 1.0 : 0.0;
        else depth = 1.0 / (1.0 + dev / mad);
    } else {
        const double dev = -medz;
        // y > med  <=>  key(y) > kR (no key lies strictly between kR and kN)
        const uint32_t npos = (uint32_t)n - c_le;
        if (dev <= 0.0) {
            depth = 1.0;
        } else if (npos == 0u) {
            depth = 0.0;
        } else {
            // median of the positive deviations: keys at global ranks
            // c_le + (npos-1)/2 (and + 1 for even npos) of the same y keys
            const uint32_t A = c_le + ((npos - 1u) >> 1);
            const bool pe = (npos & 1u) == 0u;
            uint32_t aR, aN, ac;
            s3_rank<NT>(row, n, S3KeyY{}, A, pe, sh.sorted, slots, cap, cmax, cand, sh, aR, aN, ac, a.fallbacks);
            const double ta = (double)(float)((double)kfloat(aR) - med);
            const double madp = pe ? (ta + (double)(float)((double)kfloat(aN) - med)) / 2.0 : ta;
            depth = 1.0 / (1.0 + dev / madp);
        }
    }
    if (tid == 0) a.depths[(size_t)q * a.m + j] = depth;
}

// candidate slots per thread: mean + 4 sigma of a ~21 % bracket over the
// thread's share of the row (an overflowing row falls back)
// bracket share of the row at p = 1/2 (2M + 1 sample gaps) and its spread:
// the population share between two sample order statistics M apart is
// Beta-distributed with sd ~ sqrt(2M) / S
template <int NT>
static void sel3_share(double& f, double& fsd) {
    const double S = Sel3Cfg<NT>::S;
    const double M = 3.0 * sqrt(S * 0.25) + 2.0;
    f = (2.0 * M + 1.0) / S;
    fsd = sqrt(2.0 * M) / S;
}
// candidate slots per thread: mean + SIGMAS sigma of the thread's share of the
// row in a bracket of typical share (an overflowing row falls back)
template <int NT>
static int sel3_cap(int64_t n) {
    const double kpt = (n % 4 == 0) ? 4.0 * (double)((n / 4 + NT - 1) / NT) : (double)((n + NT - 1) / NT);
    double f, fsd;
    sel3_share<NT>(f, fsd);
    const double mean = kpt * f;
    return (int)ceil(mean + Sel3Cfg<NT>::SIGMAS * sqrt(mean * (1.0 - f))) + 2;
}
// contiguous candidates: the bracket's share + 4 sd (rarely exceeded: fallback)
template <int NT>
static int sel3_cmax(int64_t n, int cap) {
    double f, fsd;
    sel3_share<NT>(f, fsd);
    const int64_t c = (int64_t)ceil((double)n * (f + 4.0 * fsd)) + 64;
    const int64_t lim = (int64_t)cap * NT;
    return (int)((c < lim ? c : lim) + 3) & ~3;
}

template <int NT>
static size_t sel3_smem(int64_t n) {
    const int cap = sel3_cap<NT>(n);
    // slots [cap][NT] + one overflow slot row + the contiguous candidate array
    return ((sizeof(Sel3Shared<NT>) + 15) & ~size_t(15)) + ((size_t)(cap + 1) * NT + sel3_cmax<NT>(n, cap)) * 4;
}

template <int NT>
static cudaError_t launch_sel3(const SelectArgs& a, dim3 grid, cudaStream_t st) {
    const int cap = sel3_cap<NT>(a.n);
    const int cmax = sel3_cmax<NT>(a.n, cap);
    const size_t smem = sel3_smem<NT>(a.n);
    cudaError_t e = cudaFuncSetAttribute(select_v3_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    select_v3_kernel<NT><<<grid, NT, smem, st>>>(a, cap, cmax);
    return cudaGetLastError();
}


// ---------------------------------------------------------------- K3 v5 --
// Sample-bracket select for rows past shared memory (n > 53248, config 5p:
// n = 1M).  v2 streams a 4 MB row ~8 times (key rewrite, radix passes, the MAD
// rewrite); here an order statistic costs two streaming passes: pass A counts
// the keys below the sample bracket and histograms the keys inside it (1024
// offset bins, one red.shared each, ~20 % of the keys), pass B gathers the
// keys of the bin holding the target rank (a few hundred) into shared memory,
// where v3's candidate select finishes.  A bin above S5_CAP keys (ties) is
// refined by another histogram pass restricted to it; a missed bracket
// restarts from the full key range.  Same keys / midpoints as v2: bitwise
// equal depths.
constexpr int S5_CAP = 8192;                   // gathered keys (global rows)
#ifndef RRS_S5_UNROLL
#define RRS_S5_UNROLL 4
#endif
constexpr int S5_U = RRS_S5_UNROLL;            // 16-byte loads in flight per thread in v5's row passes


// one pass over the row: keys < base counted, keys in [base, base + span]
// histogrammed by (key - base) >> shift; returns (below, inside) totals
template <int S5_NT, typename KF>
__device__ void s5_hist_pass(const float* __restrict__ row, int64_t n, KF kf, uint32_t base, uint32_t span, int shift,
                             Sel3Shared<S5_NT>& sh, uint32_t& below, uint32_t& inside) {
    const int tid = threadIdx.x;
    __syncthreads();  // previous readers of hist are done
    for (int i = tid; i < S3_BINS; i += S5_NT) sh.hist[i] = 0u;
    __syncthreads();
    const uint32_t hbase = smem_u32(sh.hist);
    uint32_t b = 0, in = 0;
    s3_row_each<S5_NT, S5_U>(row, (int)n, [&](float y) {
        const uint32_t key = kf(y);
        const uint32_t off = key - base;
        b += key < base ? 1u : 0u;
        const uint32_t addr = hbase + ((off >> shift) << 2);
        asm volatile("{\n.reg .pred p;\nsetp.le.u32 p, %0, %1;\n@p red.shared.add.u32 [%2], 1;\n}\n" ::"r"(off), "r"(span),
                     "r"(addr)
                     : "memory");
        in += off <= span ? 1u : 0u;
    });
    below = s3_reduce_add<S5_NT>(b, sh);
    inside = s3_reduce_add<S5_NT>(in, sh);
}

// the bin of sh.hist holding rank t (0-based, among the histogrammed keys):
// bin index, keys in lower bins, keys in the bin
template <int S5_NT>
__device__ void s5_find_bin(uint32_t t, Sel3Shared<S5_NT>& sh, uint32_t& bin, uint32_t& below, uint32_t& cnt) {
    constexpr int PER = S3_BINS / S5_NT;  // consecutive bins per thread
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t hv[PER], local = 0;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        hv[i] = sh.hist[tid * PER + i];
        local += hv[i];
    }
    uint32_t incl = local;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += o;
    }
    if (lane == 31) sh.wsum[warp] = incl;
    __syncthreads();
    uint32_t run = incl - local;
    for (int w = 0; w < warp; ++w) run += sh.wsum[w];
    if (run <= t && t < run + local) {
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            if (run <= t && t < run + hv[i]) {
                sh.s_bin = (uint32_t)(tid * PER + i);
                sh.s_below = run;
                sh.s_cnt = hv[i];
            }
            run += hv[i];
        }
    }
    __syncthreads();
    bin = sh.s_bin;
    below = sh.s_below;
    cnt = sh.s_cnt;
    __syncthreads();
}

// keys at ranks R (and R + 1) of the n keys kf(y) of a global row; c_le = keys <= key(R)
template <int S5_NT, int CAP, typename KF>
__device__ void s5_rank(const float* __restrict__ row, int64_t n, KF kf, uint32_t R, bool need_next,
                        const uint32_t* sorted, uint32_t* cand, Sel3Shared<S5_NT>& sh, uint32_t& kR, uint32_t& kN,
                        uint32_t& c_le, unsigned* fallbacks) {
    uint32_t lo, hi;
    s3_bracket<Sel3Cfg<S5_NT>::S>(sorted, R, need_next ? R + 1 : R, (uint32_t)n, lo, hi);
    uint32_t base = lo, span = hi - lo, wbelow = 0, wcnt = 0;
    for (int round = 0;; ++round) {
        const int bits = span ? 32 - __clz(span) : 0;
        const int shift = bits > S3_BITS ? bits - S3_BITS : 0;
        uint32_t below, inside;
        s5_hist_pass<S5_NT>(row, n, kf, base, span, shift, sh, below, inside);
        if (R < below || R >= below + inside) {
            // the sample bracket missed: restart from the whole key range
            if (fallbacks && threadIdx.x == 0) atomicAdd(fallbacks, 1u);
            base = 0u;
            span = 0xFFFFFFFFu;
            continue;
        }
        uint32_t bin, bbelow, bcnt;
        s5_find_bin<S5_NT>(R - below, sh, bin, bbelow, bcnt);
        const uint32_t start = bin << shift;
        base += start;
        span = min(span - start, (shift ? (1u << shift) : 1u) - 1u);
        wbelow = below + bbelow;
        wcnt = bcnt;
        if (wcnt <= (uint32_t)CAP || span == 0u) break;
    }
    if (span == 0u) {  // one key value
        kR = base;
        c_le = wbelow + wcnt;
    } else {
        // gather the window's keys (pass B)
        if (threadIdx.x == 0) sh.s_ovf = 0u;
        __syncthreads();
        s3_row_each<S5_NT, S5_U>(row, (int)n, [&](float y) {
            const uint32_t key = kf(y);
            if (key - base <= span) cand[atomicAdd(&sh.s_ovf, 1u)] = key;
        });
        __syncthreads();
        const auto each = [&](auto&& f) { s3_arr_each<S5_NT>(cand, (int)wcnt, f); };
        uint32_t cl;
        kR = s3_kth<S5_NT>(each, R - wbelow, base, base + span, wcnt, sh, cl);
        c_le = wbelow + cl;
    }
    kN = kR;
    if (need_next && c_le < R + 2) {
        uint32_t best = 0xFFFFFFFFu;
        if (span != 0u && R + 1 < wbelow + wcnt) {
            s3_arr_each<S5_NT>(cand, (int)wcnt, [&](uint32_t k2) { best = min(best, k2 > kR ? k2 : 0xFFFFFFFFu); });
        } else {
            s3_row_each<S5_NT, S5_U>(row, (int)n, [&](float y) {
                const uint32_t k2 = kf(y);
                best = min(best, k2 > kR ? k2 : 0xFFFFFFFFu);
            });
        }
        kN = s3_reduce_min<S5_NT>(best, sh);
    }
}

// four 512-thread CTAs per SM at 32 registers (the spills sit in the per-row
// serial phases): more rows in flight per SM -- config 5p 10.79 (one 1024-thread
// CTA at 64 registers) -> 11.78 (two) -> 12.06 q/s (four 512-thread CTAs)
#ifndef RRS_S5_NT
#define RRS_S5_NT 512
#endif
#ifndef RRS_S5_MINB
#define RRS_S5_MINB (2048 / RRS_S5_NT)
#endif
template <int S5_NT, int CAP>
__global__ void __launch_bounds__(S5_NT, RRS_S5_MINB) select_v5_kernel(const SelectArgs a) {
    extern __shared__ __align__(16) unsigned char sel5_raw[];
    Sel3Shared<S5_NT>& sh = *reinterpret_cast<Sel3Shared<S5_NT>*>(sel5_raw);
    uint32_t* cand = reinterpret_cast<uint32_t*>(sel5_raw + ((sizeof(Sel3Shared<S5_NT>) + 15) & ~size_t(15)));
    const int jj = blockIdx.x, q = blockIdx.y;
    const int j = a.j0 + jj;
    if (j >= a.m) return;
    const int tid = threadIdx.x;
    const int64_t n = a.n;
    const float* row = a.y + ((size_t)q * a.jcount + jj) * a.n;
    constexpr int S = Sel3Cfg<S5_NT>::S;
    uint32_t sv = 0u;
    if (tid < S) sv = fkey(__ldg(row + (((int64_t)(2 * tid + 1) * n) / (2 * S))));
    s3_sort_sample<S5_NT>(sv, sh);

    const uint32_t k = (uint32_t)((n - 1) >> 1);
    const bool even = (n & 1) == 0;
    uint32_t kR, kN, c_le;
    s5_rank<S5_NT, CAP>(row, n, S3KeyY{}, k, even, sh.sorted, cand, sh, kR, kN, c_le, a.fallbacks);
    const double lov = (double)kfloat(kR);
    const double med = even ? (lov + (double)kfloat(kN)) / 2.0 : lov;
    const double medz = med + (a.shift ? a.shift[(size_t)q * a.m + j] : 0.0);
    double depth;
    if (a.notion == 1) {
        // the sample's deviations: two monotone runs, merge-ranked (as in v3)
        uint32_t dk = 0u, le = 0u;
        if (tid < S) {
            const double yv = (double)kfloat(sh.sorted[tid]);
            dk = fkey((float)fabs(yv - med));
            le = yv <= med ? 1u : 0u;
        }
        __syncthreads();
        if (tid < S) sh.sdev[tid] = dk;
        const uint32_t nl = s3_reduce_add<S5_NT>(le, sh);
        if (tid < S) {
            uint32_t rank;
            if ((uint32_t)tid < nl) {
                uint32_t lo_i = nl, hi_i = S;
                while (lo_i < hi_i) {
                    const uint32_t mid = (lo_i + hi_i) >> 1;
                    if (sh.sdev[mid] < dk) lo_i = mid + 1;
                    else hi_i = mid;
                }
                rank = (nl - 1 - tid) + (lo_i - nl);
            } else {
                uint32_t lo_i = 0, hi_i = nl;
                while (lo_i < hi_i) {
                    const uint32_t mid = (lo_i + hi_i) >> 1;
                    if (sh.sdev[mid] <= dk) hi_i = mid;
                    else lo_i = mid + 1;
                }
                rank = (tid - nl) + (nl - lo_i);
            }
            sh.sorted[rank] = dk;
        }
        __syncthreads();
        uint32_t mR, mN, mc;
        s5_rank<S5_NT, CAP>(row, n, S3KeyAbsDev{med}, k, even, sh.sorted, cand, sh, mR, mN, mc, a.fallbacks);
        const double mlo = (double)kfloat(mR);
        const double mad = even ? (mlo + (double)kfloat(mN)) / 2.0 : mlo;
        const double dev = fabs(medz);
        if (mad == 0.0) depth = (dev == 0.0) ? 1.0 : 0.0;
        else depth = 1.0 / (1.0 + dev / mad);
    } else {
        const double dev = -medz;
        const uint32_t npos = (uint32_t)n - c_le;
        if (dev <= 0.0) {
            depth = 1.0;
        } else if (npos == 0u) {
            depth = 0.0;
        } else {
            const uint32_t A = c_le + ((npos - 1u) >> 1);
            const bool pe = (npos & 1u) == 0u;
            uint32_t aR, aN, ac;
            s5_rank<S5_NT, CAP>(row, n, S3KeyY{}, A, pe, sh.sorted, cand, sh, aR, aN, ac, a.fallbacks);
            const double ta = (double)(float)((double)kfloat(aR) - med);
            const double madp = pe ? (ta + (double)(float)((double)kfloat(aN) - med)) / 2.0 : ta;
            depth = 1.0 / (1.0 + dev / madp);
        }
    }
    if (tid == 0) a.depths[(size_t)q * a.m + j] = depth;
}

template <int S5_NT, int CAP>
static cudaError_t launch_sel5(const SelectArgs& a, dim3 grid, cudaStream_t st) {
    const size_t smem = ((sizeof(Sel3Shared<S5_NT>) + 15) & ~size_t(15)) + (size_t)CAP * 4;
    cudaError_t e =
        cudaFuncSetAttribute(select_v5_kernel<S5_NT, CAP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    select_v5_kernel<S5_NT, CAP><<<grid, S5_NT, smem, st>>>(a);
    return cudaGetLastError();
}

template <int NT, bool GLB>
static cudaError_t launch_sel2(const SelectArgs& a, dim3 grid, cudaStream_t st) {
    const size_t smem = ((sizeof(Sel2Shared<NT>) + 15) & ~size_t(15)) + (GLB ? (size_t)SEL2G_CAP * 4 : (size_t)a.n * 4);
    cudaError_t e = cudaFuncSetAttribute(select_v2_kernel<NT, GLB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    select_v2_kernel<NT, GLB><<<grid, NT, smem, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_select(const SelectArgs& a, cudaStream_t st) {
    if (a.Qb == 0 || a.jcount == 0) return cudaSuccess;
    dim3 grid((unsigned)a.jcount, (unsigned)a.Qb);
    if (a.variant != 2 && a.n >= SEL3_MIN_N && a.n <= SEL3_MAX_N) {
        if (a.n <= SEL2_WIDE_N) return launch_sel3<256>(a, grid, st);
        // two 512-thread CTAs per SM when their shared memory fits (variant 3: 1024 threads)
        if (a.variant != 3 && sel3_smem<512>(a.n) <= 113 * 1024) return launch_sel3<512>(a, grid, st);
        return launch_sel3<1024>(a, grid, st);
    }
    if (a.n <= SEL2_MAX_N) {
        if (a.n <= SEL2_WIDE_N) return launch_sel2<256, false>(a, grid, st);
        if (a.n <= SEL2_WIDER_N) return launch_sel2<512, false>(a, grid, st);
        return launch_sel2<1024, false>(a, grid, st);
    }
    // rows past shared memory: the two-pass sample-bracket select (v5) unless
    // the radix select is asked for (variant 2)
    if (a.variant != 2 && a.n < ((int64_t)1 << 31)) return launch_sel5<RRS_S5_NT, S5_CAP>(a, grid, st);
#ifndef RRS_SEL_LEGACY_GLOBAL
    // (16-byte key loads: rows must start aligned, i.e. n % 4 == 0)
    if ((a.n & 3) == 0 && a.n < ((int64_t)1 << 31)) return launch_sel2<1024, true>(a, grid, st);
#endif
    size_t smem = (sizeof(SelShared) + 15) & ~size_t(15);
    if (a.n <= SEL_CACHE_MAX) smem += (size_t)a.n * sizeof(float);
    cudaError_t e = cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    select_kernel<<<grid, SEL_THREADS, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace rrs
