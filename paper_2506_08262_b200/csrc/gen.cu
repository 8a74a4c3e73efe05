// gen.cu -- FP64 kernels: Philox spherical-cap direction generation, RRS state
// (init / argmin + pole update / reflection vector / trace), layout conversion.
//
// Compiled with -fmad=false: the FP64 arithmetic here restates the reference's
// numpy/C operation sequence (no contraction), so device directions track the
// reference rows to a few ulp (CUDA vs glibc cos/log are the only differences).
#include "common.cuh"
#include "kernels.h"

#include <cuda_fp16.h>

#include <math.h>

namespace rrs {

// ------------------------------------------------------------------ Philox --
// Philox-4x32-10: philox.py:27-65 / _kernels.pyx:24-61.
__device__ __forceinline__ void philox10(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3,
                                         uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint32_t hi0 = __umulhi(c0, 0xD2511F53u), lo0 = c0 * 0xD2511F53u;
        uint32_t hi1 = __umulhi(c2, 0xCD9E8D57u), lo1 = c2 * 0xCD9E8D57u;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

// philox.py:88-114: counter (v, j, l, q), key = seed lo/hi words, 53-bit mantissa.
__device__ __forceinline__ double uniform1(uint64_t seed, uint32_t v, uint32_t j, uint32_t l,
                                           uint32_t q) {
    uint32_t c0 = v, c1 = j, c2 = l, c3 = q;
    philox10(c0, c1, c2, c3, (uint32_t)seed, (uint32_t)(seed >> 32));
    uint64_t bits = (uint64_t)c0 | ((uint64_t)c1 << 32);
    return ((double)(bits >> 11) + 0.5) * 0x1.0p-53;
}

// ------------------------------------------------------------------- ndtri --
// Inverse normal CDF, Cephes algorithm (scipy.special.ndtri, scipy 1.18.1);
// Q* tables evaluated with an implicit leading 1 (p1evl).
__constant__ double c_P0[5] = {-5.99633501014107895267E1, 9.80010754185999661536E1,
                               -5.66762857469070293439E1, 1.39312609387279679503E1,
                               -1.23916583867381258016E0};
__constant__ double c_Q0[8] = {1.95448858338141759834E0,  4.67627912898881538453E0,
                               8.63602421390890590575E1,  -2.25462687854119370527E2,
                               2.00260212380060660359E2,  -8.20372256168333339912E1,
                               1.59056225126211695515E1,  -1.18331621121330003142E0};
__constant__ double c_P1[9] = {4.05544892305962419923E0,   3.15251094599893866154E1,
                               5.71628192246421288162E1,   4.40805073893200834700E1,
                               1.46849561928858024014E1,   2.18663306850790267539E0,
                               -1.40256079171354495875E-1, -3.50424626827848203418E-2,
                               -8.57456785154685413611E-4};
__constant__ double c_Q1[8] = {1.57799883256466749731E1,   4.53907635128879210584E1,
                               4.13172038254672030440E1,   1.50425385692907503408E1,
                               2.50464946208309415979E0,   -1.42182922854787788574E-1,
                               -3.80806407691578277194E-2, -9.33259480895457427372E-4};
__constant__ double c_P2[9] = {3.23774891776946035970E0,  6.91522889068984211695E0,
                               3.93881025292474443415E0,  1.33303460815807542389E0,
                               2.01485389549179081538E-1, 1.23716634817820021358E-2,
                               3.01581553508235416007E-4, 2.65806974686737550832E-6,
                               6.23974539184983293730E-9};
__constant__ double c_Q2[8] = {6.02427039364742014255E0,  3.67983563856160859403E0,
                               1.37702099489081330271E0,  2.16236993594496635890E-1,
                               1.34204006088543189037E-2, 3.28014464682127739104E-4,
                               2.89247864745380683936E-6, 6.79019408009981274425E-9};

__device__ __forceinline__ double polevl(double x, const double* c, int deg) {
    double a = c[0];
    for (int i = 1; i <= deg; ++i) a = a * x + c[i];
    return a;
}
__device__ __forceinline__ double p1evl(double x, const double* c, int deg) {
    double a = x + c[0];
    for (int i = 1; i < deg; ++i) a = a * x + c[i];
    return a;
}

constexpr double NDTRI_S2PI = 2.50662827463100050242E0;
constexpr double NDTRI_E2 = 0.13533528323661269189;  // exp(-2)

// ndtri's branch for exp(-2) < y0 <= 1 - exp(-2)
__device__ __forceinline__ bool ndtri_is_central(double y0) {
    return !(y0 > 1.0 - NDTRI_E2) && y0 > NDTRI_E2;
}
__device__ __forceinline__ double ndtri_central(double y0) {
    double y = y0 - 0.5;
    double y2 = y * y;
    double x = y + y * (y2 * polevl(y2, c_P0, 4) / p1evl(y2, c_Q0, 8));
    return x * NDTRI_S2PI;
}
__device__ __forceinline__ double ndtri_tail(double y0) {
    bool negate = true;
    double y = y0;
    if (y > 1.0 - NDTRI_E2) {
        y = 1.0 - y;
        negate = false;
    }
    double x = sqrt(-2.0 * log(y));
    double x0 = x - log(x) / x;
    double z = 1.0 / x;
    double x1 = (x < 8.0) ? z * polevl(z, c_P1, 8) / p1evl(z, c_Q1, 8)
                          : z * polevl(z, c_P2, 8) / p1evl(z, c_Q2, 8);
    x = x0 - x1;
    return negate ? -x : x;
}
__device__ __forceinline__ double ndtri(double y0) {
    return ndtri_is_central(y0) ? ndtri_central(y0) : ndtri_tail(y0);
}

// numpy float64 add.reduce over a contiguous row = 0.0 + pairwise sum
// (8 running partials up to 128 elements, halving at multiples of 8 beyond).
__device__ double pw_rec(const double* a, int n) {
    if (n < 8) {
        double r = 0.0;
        for (int i = 0; i < n; ++i) r += a[i];
        return r;
    }
    if (n <= 128) {
        double r0 = a[0], r1 = a[1], r2 = a[2], r3 = a[3], r4 = a[4], r5 = a[5], r6 = a[6],
               r7 = a[7];
        int i = 8;
        for (; i < n - (n % 8); i += 8) {
            r0 += a[i];
            r1 += a[i + 1];
            r2 += a[i + 2];
            r3 += a[i + 3];
            r4 += a[i + 4];
            r5 += a[i + 5];
            r6 += a[i + 6];
            r7 += a[i + 7];
        }
        double res = ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7));
        for (; i < n; ++i) res += a[i];
        return res;
    }
    int n2 = n / 2;
    n2 -= n2 % 8;
    return pw_rec(a, n2) + pw_rec(a + n2, n - n2);
}

__device__ __forceinline__ double pw_sum(const double* a, int n) { return 0.0 + pw_rec(a, n); }

// Filter-and-refine operand (contract_tcf.cu, kernels.h): K position kk of
// direction row (coordinates row[0..d)): fp16(u * TCF_SU), the threshold slot
// at kk = d (1, or 4 for a padded direction), zeros after.
__device__ __forceinline__ __half tcf_value(const double* row, int d, int kk, bool real) {
    if (kk < d) return real ? __double2half(row[kk] * (double)TCF_SU) : __double2half(0.0);
    if (kk == d) return __float2half_rn(real ? 1.0f : 4.0f);
    return __double2half(0.0);
}

// Tensor-path direction operand (contract_tc.cu): u * 2^15 = hi + lo, both
// FP16 (hi = fp16(u 2^15), lo = fp16(u 2^15 - hi), |u| <= 1), placed at the
// K positions of the packed split-product layout (kernels.h, tc_layout): hi
// and lo once each for an aligned coordinate, hi, hi, lo (products 0..2) for a
// remainder coordinate.
// oprow points at (block, direction) = block base + (j & 127) * 16.
__device__ __forceinline__ void tc_split(double u, __half& h, __half& l) {
    const double v = u * 32768.0;
    h = __double2half(v);
    l = __double2half(v - (double)__half2float(h));
}
__device__ __forceinline__ void put_tc_operand(unsigned char* oprow, const TcLayout& L, int c, double u) {
    __half h, l;
    tc_split(u, h, l);
    const int ne = tc_entries(L, c);
    for (int e = 0; e < ne; ++e) {
        const int kk = tc_pos(L, e, c);
        *reinterpret_cast<__half*>(oprow + (kk >> 3) * 2048 + (kk & 7) * 2) = tc_a_lo(L, e, c) ? l : h;
    }
}

// ------------------------------------------------------- cap generation K1 --
// directions.py:167-182 (_cap_rows) for every (query, direction): one warp per
// direction.  theta = U(v=0,j)*eps; d-1 normals from v = 1..d-1 (zero-norm
// rows redrawn from the next d-1 addresses, directions.py:113-135); row =
// [cos theta, sqrt(1-cos^2)*g/|g|]; Householder e1 -> pole with the per-query
// reflection vector prepared by the update kernel (directions.py:150-164).
// Writes U64[q][j][d] (pole candidates) and U32[q][jb][d][BN] (contraction
// operand, FP32, K-major per direction block); padded directions j >= m get 0.
// One direction gdir (over Qb * mpad) on one warp; g, sc: 2*d doubles of scratch.
__device__ void gen_direction_warp(const GenArgs& a, int64_t gdir, double* g, double* sc) {
    const int lane = threadIdx.x & 31;
    const int d = a.d;
    const int q = (int)(gdir / a.mpad);
    const int j = (int)(gdir % a.mpad);
    float* u32 = a.u32 ? a.u32 + (size_t)q * a.mpad * d + (size_t)(j / BN) * d * BN + (j % BN) : nullptr;
    unsigned char* op = nullptr;
    if (a.uop && j < a.NB * 128)
        op = a.uop + ((size_t)q * a.NB + (j >> 7)) * tc_block_bytes(d) + (size_t)(j & 127) * 16;
    float* u32r = a.u32r ? a.u32r + ((size_t)q * a.mpad + j) * tcf_dp(d) : nullptr;
    if (a.uop_mode == 1) {
        if (a.uop && j < a.NB * 128)
            op = a.uop + ((size_t)q * a.NB + (j >> 7)) * tcf_block_bytes(d) + (size_t)(j & 127) * 16;
        else
            op = nullptr;
    }
    if (j >= a.m) {
        if (u32)
            for (int c = lane; c < d; c += 32) u32[(size_t)c * BN] = 0.0f;
        if (u32r)
            for (int c = lane; c < tcf_dp(d); c += 32) u32r[c] = 0.0f;
        if (op && a.uop_mode == 1) {
            for (int kk = lane; kk < 16 * tcf_ns(d); kk += 32)
                *reinterpret_cast<__half*>(op + (kk >> 3) * 2048 + (kk & 7) * 2) = tcf_value(nullptr, d, kk, false);
            return;
        }
        if (op)
            for (int kk = lane; kk < 16 * tc_layout(d).ns; kk += 32)
                *reinterpret_cast<__half*>(op + (kk >> 3) * 2048 + (kk & 7) * 2) = __double2half(0.0);
        return;
    }
    const uint32_t qg = (uint32_t)((uint64_t)(a.q0 + q) & 0xFFFFFFFFu);
    const uint32_t l = a.refinement;
    const double* pole = a.pole + (size_t)q * d;
    double* u64 = a.u64 + ((size_t)q * a.m + j) * d;
    if (d == 1) {  // directions.py:172-173
        if (lane == 0) {
            u64[0] = pole[0];
            if (u32) u32[0] = (float)pole[0];
        }
        if (u32r)
            for (int c = lane; c < tcf_dp(d); c += 32) u32r[c] = c == 0 ? (float)pole[0] : 0.0f;
        if (op && a.uop_mode == 1) {
            for (int kk = lane; kk < 16 * tcf_ns(d); kk += 32)
                *reinterpret_cast<__half*>(op + (kk >> 3) * 2048 + (kk & 7) * 2) = tcf_value(pole, d, kk, true);
            return;
        }
        if (op) {
            const TcLayout L = tc_layout(d);
            for (int kk = lane; kk < 16 * L.ns; kk += 32) {
                int p, c;
                tc_elem(L, kk, p, c);
                if (c < 0) *reinterpret_cast<__half*>(op + (kk >> 3) * 2048 + (kk & 7) * 2) = __double2half(0.0);
            }
            if (lane == 0) put_tc_operand(op, L, 0, pole[0]);
        }
        return;
    }
    const int dm = d - 1;
    double u1 = 0.0;
    const uint32_t jp = a.jbase + (uint32_t)j;  // Philox index of this direction
    if (lane == 0) u1 = cos(uniform1(a.seed, 0u, jp, l, qg) * a.eps);
    uint32_t vbase = 1;
    double nrm;
    for (;;) {
        for (int c = lane; c < dm; c += 32) {
            double gv = ndtri(uniform1(a.seed, vbase + (uint32_t)c, jp, l, qg));
            g[c] = gv;
            sc[c] = gv * gv;
        }
        __syncwarp();
        if (lane == 0) nrm = sqrt(pw_sum(sc, dm));
        nrm = __shfl_sync(0xffffffffu, nrm, 0);
        __syncwarp();
        if (nrm != 0.0) break;
        vbase += (uint32_t)dm;
    }
    u1 = __shfl_sync(0xffffffffu, u1, 0);
    const double s = sqrt(1.0 - u1 * u1);
    // row stored in sc[0..d): sc[0] = u1, sc[1+c] = s * (g[c]/nrm)
    __syncwarp();
    for (int c = lane; c < dm; c += 32) g[c] = s * (g[c] / nrm);
    __syncwarp();
    for (int c = lane; c < dm; c += 32) sc[1 + c] = g[c];
    if (lane == 0) sc[0] = u1;
    __syncwarp();
    const int mode = a.refl_mode[q];
    if (mode == 1) {
        if (lane == 0) sc[0] = -sc[0];
        __syncwarp();
    } else if (mode == 2) {
        const double* v = a.refl_v + (size_t)q * d;
        for (int c = lane; c < d; c += 32) g[c] = sc[c] * v[c];
        __syncwarp();
        double f = 0.0;
        if (lane == 0) f = 2.0 * pw_sum(g, d);
        f = __shfl_sync(0xffffffffu, f, 0);
        for (int c = lane; c < d; c += 32) sc[c] = sc[c] - f * v[c];
        __syncwarp();
    }
    for (int c = lane; c < d; c += 32) {
        double val = sc[c];
        u64[c] = val;
        if (u32) u32[(size_t)c * BN] = (float)val;
    }
    if (u32r)
        for (int c = lane; c < tcf_dp(d); c += 32) u32r[c] = c < d ? (float)sc[c] : 0.0f;
    if (op && a.uop_mode == 1) {
        __syncwarp();
        for (int kk = lane; kk < 16 * tcf_ns(d); kk += 32)
            *reinterpret_cast<__half*>(op + (kk >> 3) * 2048 + (kk & 7) * 2) = tcf_value(sc, d, kk, true);
    } else if (op) {
        const TcLayout L = tc_layout(d);
        for (int kk = lane; kk < 16 * L.ns; kk += 32) {  // zero padding positions
            int p, c;
            tc_elem(L, kk, p, c);
            if (c < 0) *reinterpret_cast<__half*>(op + (kk >> 3) * 2048 + (kk & 7) * 2) = __double2half(0.0);
        }
        for (int c = lane; c < d; c += 32) put_tc_operand(op, L, c, sc[c]);
    }
}

__global__ void __launch_bounds__(256) cap_generate_kernel(GenArgs a) {
    extern __shared__ double gsm[];
    const int warp = threadIdx.x >> 5;
    const int64_t gdir = (int64_t)blockIdx.x * 8 + warp;  // over Qb * mpad
    if (gdir >= (int64_t)a.Qb * a.mpad) return;
    if (a.done && a.done[gdir / a.mpad]) return;  // early exit: the query is finished
    double* g = gsm + (size_t)warp * 2 * a.d;  // d values + d scratch
    gen_direction_warp(a, gdir, g, g + a.d);
}

// K1 v2 (2 <= d <= 128): a block of GV_DIRS = 32 directions of one query,
// element-parallel with the same FP64 operation sequence as the warp kernel:
//   1. Philox uniforms of every (direction, coordinate) and the theta uniform;
//   2. ndtri, with the central and tail elements compacted into separate lists
//      so that no warp executes both branches (the tail branch is ~4x longer);
//   3. squared norms in numpy's pairwise order, the 8 running partials on 8
//      lanes and the ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) tree by shuffles;
//   4. row = [cos theta, sqrt(1-cos^2) * g/|g|]; reflection (mode 1: negate
//      e1, mode 2: Householder with f = 2 * pairwise(row . v));
//   5. coalesced stores: U64 rows, U32 K-major block columns (FFMA / store
//      paths only), the FP16 hi/lo tensor operand in 16-byte chunks.
// A zero-norm normal row (the reference's redraw branch, directions.py:113-135)
// cannot occur for 53-bit uniforms (ndtri(u) = 0 only at u = 0.5, which is not
// on the (k + 0.5) 2^-53 grid); such a direction is regenerated by the warp path.
constexpr int GV_DIRS = 32;
constexpr int GV_THREADS = 256;
constexpr int GV_MAX_D = 128;

__device__ __forceinline__ double pw8_partial_tree(double r) {
    // lanes k = 0..7 of an aligned 8-lane group hold r_k; lane 0 returns the tree sum
    r += __shfl_down_sync(0xffffffffu, r, 1, 8);
    r += __shfl_down_sync(0xffffffffu, r, 2, 8);
    r += __shfl_down_sync(0xffffffffu, r, 4, 8);
    return r;
}

// pairwise_sum(f(i), i < n) for n <= 128 on the 8-lane group of lane k (valid on k == 0);
// F(i) produces element i (evaluated exactly as in the serial code).  Must be
// called by all 32 lanes of the warp (full-mask shuffles).
template <typename F>
__device__ __forceinline__ double pw_sum8(int n, int k, F f) {
    double res;
    if (n < 8) {
        res = 0.0;
        if (k == 0)
            for (int i = 0; i < n; ++i) res += f(i);
        res = __shfl_sync(0xffffffffu, res, (threadIdx.x & 31) & ~7);
    } else {
        double r = f(k);
        int i = 8;
        for (; i < n - (n % 8); i += 8) r += f(i + k);
        res = pw8_partial_tree(r);
        if (k == 0)
            for (; i < n; ++i) res += f(i);
    }
    return 0.0 + res;
}

#ifndef RRS_GEN_BLOCKS_PER_SM
#define RRS_GEN_BLOCKS_PER_SM 5  // occupancy for the latency-bound FP64 chains (measured: 3 -> 5 is 12% faster)
#endif
__global__ void __launch_bounds__(GV_THREADS, RRS_GEN_BLOCKS_PER_SM) cap_generate_v2_kernel(GenArgs a) {
    extern __shared__ double vsm[];
    const int d = a.d, dm = d - 1;
    // e / dm by a 64-bit multiply-high (exact for e < 32 dm, dm < 2^10: checked for
    // every dm; dm = 1 needs the 33-bit multiplier 2^32)
    const uint64_t dm_mul = (uint64_t)(0xFFFFFFFFu / (uint32_t)(dm > 0 ? dm : 1)) + 1ull;
    double* val = vsm;                          // [GV_DIRS][d] uniforms -> normals -> row
    double* s_th = val + GV_DIRS * d;           // [GV_DIRS] theta uniform -> u1
    double* s_nrm = s_th + GV_DIRS;             // [GV_DIRS]
    uint16_t* list = reinterpret_cast<uint16_t*>(s_nrm + GV_DIRS);  // [GV_DIRS * dm]
    __shared__ int s_nc, s_nt, s_zero;
    __shared__ double s_sf[GV_DIRS];            // sqrt(1 - u1^2) per direction
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t gdir0 = (int64_t)blockIdx.x * GV_DIRS;
    const int q = (int)(gdir0 / a.mpad);
    const int j0 = (int)(gdir0 % a.mpad);       // GV_DIRS | 128 | mpad: one query, one 128-block
    if (a.done && a.done[q]) return;            // early exit: the query is finished (block-uniform)
    const int nval = a.m - j0 < GV_DIRS ? (a.m - j0 > 0 ? a.m - j0 : 0) : GV_DIRS;
    const uint32_t qg = (uint32_t)((uint64_t)(a.q0 + q) & 0xFFFFFFFFu);
    const uint32_t l = a.refinement;
    const int E = nval * dm;
    if (tid == 0) {
        s_nc = 0;
        s_nt = 0;
        s_zero = 0;
    }
    // 1. uniforms
    for (int e = tid; e < E; e += GV_THREADS) {
        const int jj = (int)(((uint64_t)e * dm_mul) >> 32), c = e - jj * dm;
        val[jj * d + 1 + c] = uniform1(a.seed, 1u + (uint32_t)c, (uint32_t)(j0 + jj), l, qg);
    }
    if (tid < nval) s_th[tid] = uniform1(a.seed, 0u, (uint32_t)(j0 + tid), l, qg);
    __syncthreads();
    // 2. ndtri: compact central / tail elements, then evaluate each list densely
    for (int e0 = 0; e0 < E; e0 += GV_THREADS) {
        const int e = e0 + tid;
        bool cen = false, tl = false;
        if (e < E) {
            const int jj = (int)(((uint64_t)e * dm_mul) >> 32);
            const bool c_ = ndtri_is_central(val[jj * d + 1 + (e - jj * dm)]);
            cen = c_;
            tl = !c_;
        }
        const uint32_t bc = __ballot_sync(0xffffffffu, cen), bt = __ballot_sync(0xffffffffu, tl);
        int pc = 0, pt = 0;
        if (lane == 0) {
            pc = atomicAdd(&s_nc, __popc(bc));
            pt = atomicAdd(&s_nt, __popc(bt));
        }
        pc = __shfl_sync(0xffffffffu, pc, 0);
        pt = __shfl_sync(0xffffffffu, pt, 0);
        const uint32_t below = (1u << lane) - 1u;
        if (cen) list[pc + __popc(bc & below)] = (uint16_t)e;
        if (tl) list[E - 1 - (pt + __popc(bt & below))] = (uint16_t)e;
    }
    __syncthreads();
    const int nc = s_nc, nt = s_nt;
    for (int i = tid; i < nc; i += GV_THREADS) {
        const int e = list[i], jj = (int)(((uint64_t)e * dm_mul) >> 32);
        double* p = &val[jj * d + 1 + (e - jj * dm)];
        *p = ndtri_central(*p);
    }
    for (int i = tid; i < nt; i += GV_THREADS) {
        const int e = list[E - 1 - i], jj = (int)(((uint64_t)e * dm_mul) >> 32);
        double* p = &val[jj * d + 1 + (e - jj * dm)];
        *p = ndtri_tail(*p);
    }
    __syncthreads();
    // 3. norms (8 lanes per direction), theta
    {
        const int jj = tid >> 3, k = tid & 7;
        const double* g = val + jj * d + 1;
        // every lane takes part in the shuffles; directions past nval sum zeros
        const bool live = jj < nval;
        const double nrm = sqrt(pw_sum8(dm, k, [&](int i) { return live ? g[i] * g[i] : 0.0; }));
        if (k == 0 && jj < nval) {
            s_nrm[jj] = nrm;
            const double u1 = cos(s_th[jj] * a.eps);  // u1 = cos(theta)
            s_th[jj] = u1;
            s_sf[jj] = sqrt(1.0 - u1 * u1);
            if (nrm == 0.0) s_zero = 1;
        }
    }
    __syncthreads();
    const int mode = a.refl_mode[q];
    const double* v = a.refl_v + (size_t)q * d;
    // 4. row = [u1, s * (g / |g|)]
    for (int e = tid; e < E; e += GV_THREADS) {
        const int jj = (int)(((uint64_t)e * dm_mul) >> 32);
        double* p = &val[jj * d + 1 + (e - jj * dm)];
        *p = s_sf[jj] * (*p / s_nrm[jj]);
    }
    if (tid < nval) val[tid * d] = (mode == 1) ? -s_th[tid] : s_th[tid];
    __syncthreads();
    if (mode == 2) {
        const int jj = tid >> 3, k = tid & 7;
        const bool live = jj < nval;
        double f = 2.0 * pw_sum8(d, k, [&](int i) { return live ? val[jj * d + i] * v[i] : 0.0; });
        f = __shfl_sync(0xffffffffu, f, lane & ~7);
        __syncwarp();
        if (jj < nval)
            for (int c = k; c < d; c += 8) val[jj * d + c] = val[jj * d + c] - f * v[c];
        __syncthreads();
    }
    // 5. stores
    double* u64 = a.u64 + ((size_t)q * a.m + j0) * d;
    for (int e = tid; e < nval * d; e += GV_THREADS) u64[e] = val[e];
    if (a.u32) {
        float* u32 = a.u32 + (size_t)q * a.mpad * d + (size_t)(j0 / BN) * d * BN + (j0 % BN);
        for (int e = tid; e < GV_DIRS * d; e += GV_THREADS) {
            const int c = e / GV_DIRS, jj = e - c * GV_DIRS;
            u32[(size_t)c * BN + jj] = jj < nval ? (float)val[jj * d + c] : 0.0f;
        }
    }
    if (a.u32r) {  // FP32 rows for contract_tcf's refinement (zero padding)
        const int dp = tcf_dp(d);
        float* rows = a.u32r + ((size_t)q * a.mpad + j0) * dp;
        for (int e = tid; e < GV_DIRS * dp; e += GV_THREADS) {
            const int jj = e / dp, c = e - jj * dp;
            rows[e] = (jj < nval && c < d) ? (float)val[jj * d + c] : 0.0f;
        }
    }
    if (a.uop && a.uop_mode == 1) {
        const int nchunk = 2 * tcf_ns(d);
        unsigned char* base = a.uop + ((size_t)q * a.NB + (j0 >> 7)) * tcf_block_bytes(d) + (size_t)(j0 & 127) * 16;
        for (int t = tid; t < GV_DIRS * nchunk; t += GV_THREADS) {
            const int jj = t & (GV_DIRS - 1), cc = t >> 5;
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const __half h0 = tcf_value(val + jj * d, d, 8 * cc + 2 * e, jj < nval);
                const __half h1 = tcf_value(val + jj * d, d, 8 * cc + 2 * e + 1, jj < nval);
                w[e] = (uint32_t)__half_as_ushort(h0) | ((uint32_t)__half_as_ushort(h1) << 16);
            }
            *reinterpret_cast<uint4*>(base + (size_t)cc * 2048 + jj * 16) = make_uint4(w[0], w[1], w[2], w[3]);
        }
    } else if (a.uop) {
        // packed split-product layout, one 16-byte chunk (8 K positions) per task
        const TcLayout L = tc_layout(d);
        const int nchunk = 2 * L.ns;
        unsigned char* base = a.uop + ((size_t)q * a.NB + (j0 >> 7)) * tc_block_bytes(d) + (size_t)(j0 & 127) * 16;
        for (int t = tid; t < GV_DIRS * nchunk; t += GV_THREADS) {
            const int jj = t & (GV_DIRS - 1), cc = t >> 5;
            uint32_t w[4] = {0u, 0u, 0u, 0u};
            if (jj < nval) {
                const double* row = val + jj * d;
                bool lo;
                int c0;
                if (tc_chunk_run(L, cc, lo, c0)) {
                    // aligned part: the hi or lo terms of 8 consecutive coordinates c0 .. c0 + 7
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        __half h0, l0, h1, l1;
                        tc_split(row[c0 + 2 * e], h0, l0);
                        tc_split(row[c0 + 2 * e + 1], h1, l1);
                        w[e] = (uint32_t)__half_as_ushort(lo ? l0 : h0) | ((uint32_t)__half_as_ushort(lo ? l1 : h1) << 16);
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        int en, c;
                        tc_elem(L, cc * 8 + e, en, c);
                        if (c >= 0) {
                            __half h, l;
                            tc_split(row[c], h, l);
                            w[e >> 1] |= (uint32_t)__half_as_ushort(tc_a_lo(L, en, c) ? l : h) << (16 * (e & 1));
                        }
                    }
                }
            }
            *reinterpret_cast<uint4*>(base + (size_t)cc * 2048 + jj * 16) = make_uint4(w[0], w[1], w[2], w[3]);
        }
    }
    if (s_zero) {
        // unreachable for 53-bit uniforms: regenerate zero-norm directions on the warp
        // path, which redraws exactly like the reference (all stores above are overwritten)
        __syncthreads();
        double* scratch = vsm + (size_t)warp * 2 * d;  // val is no longer needed
        for (int jj = warp; jj < nval; jj += GV_THREADS / 32)
            if (s_nrm[jj] == 0.0) gen_direction_warp(a, gdir0 + jj, scratch, scratch + d);
    }
}

// Explicit-direction mode: U64 given; build the FP32 contraction operand.
__global__ void pack_directions_kernel(const double* __restrict__ u64, float* __restrict__ u32, int Qb,
                                       int m, int mpad, int d) {
    int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t total = (int64_t)Qb * mpad * d;
    if (idx >= total) return;
    int c = (int)(idx % d);
    int64_t r = idx / d;
    int j = (int)(r % mpad);
    int q = (int)(r / mpad);
    float v = (j < m) ? (float)u64[((size_t)q * m + j) * d + c] : 0.0f;
    u32[(size_t)q * mpad * d + (size_t)(j / BN) * d * BN + (size_t)c * BN + (j % BN)] = v;
}

__global__ void pack_tc_operand_kernel(const double* __restrict__ u64, unsigned char* __restrict__ uop, int Qb,
                                       int m, int NB, int d) {
    // one K position of one direction per thread
    const TcLayout L = tc_layout(d);
    const int K = 16 * L.ns;
    int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t total = (int64_t)Qb * NB * 128 * K;
    if (idx >= total) return;
    int kk = (int)(idx % K);
    int64_t r = idx / K;
    int j = (int)(r % (NB * 128));
    int q = (int)(r / (NB * 128));
    int e, c;
    tc_elem(L, kk, e, c);
    __half h = __double2half(0.0), l = h;
    if (c >= 0 && j < m) tc_split(u64[((size_t)q * m + j) * d + c], h, l);
    *reinterpret_cast<__half*>(uop + ((size_t)q * NB + (j >> 7)) * tc_block_bytes(d) + (size_t)(kk >> 3) * 2048 +
                               (size_t)(j & 127) * 16 + (kk & 7) * 2) = (c >= 0 && tc_a_lo(L, e, c)) ? l : h;
}

cudaError_t launch_pack_tc_operand(const double* u64, unsigned char* uop, int Qb, int m, int NB, int d,
                                   cudaStream_t st) {
    int64_t total = (int64_t)Qb * NB * 128 * 16 * tc_layout(d).ns;
    pack_tc_operand_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(u64, uop, Qb, m, NB, d);
    return cudaGetLastError();
}

// ------------------------------------------------------------- RRS state --
// optimizer.py:164-167: pole = e1, d_min = 1.0, argmin = e1.
__global__ void state_init_kernel(StateArgs s) {
    int q = blockIdx.x;
    if (q >= s.Qb) return;
    for (int c = threadIdx.x; c < s.d; c += blockDim.x) {
        s.pole[(size_t)q * s.d + c] = (c == 0) ? 1.0 : 0.0;
        s.refl_v[(size_t)q * s.d + c] = 0.0;
    }
    if (threadIdx.x == 0) {
        s.dmin[q] = 1.0;
        s.best_count[q] = s.n;
        s.refl_mode[q] = 0;  // pole == e1: 1 - p1 < 1e-12, no reflection
    }
}

// Per-query argmin over the refinement's m directions (np.argmin: first index
// of the minimum), strict-< pole update against d_min (optimizer.py:200-205;
// the per_direction branch :206-218 ends on the same direction), trace record
// (optimizer.py:219) and the Householder vector of the new pole for the next
// refinement (directions.py:150-164).  Halfspace reads integer (#<, #>) counts,
// min count = n - max(lt, gt); the projection notions read FP64 depths.
// Also clears the halfspace counters for the next refinement.
__global__ void __launch_bounds__(256) update_kernel(UpdateArgs a) {
    const int q = blockIdx.x;
    if (q >= a.Qb) return;
    __shared__ double s_val[8];
    __shared__ long long s_cnt[8];
    __shared__ int s_idx[8];
    __shared__ int s_best;
    __shared__ int s_improved;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int d = a.d;
    if (a.done && a.done[q]) {
        // early exit: no direction can beat the best count any more (it equals the
        // rows coinciding with the query); the record repeats the state, exactly
        // what the full run writes when the strict-< update does not fire
        if (a.trace) {
            double* rec = a.trace + ((size_t)q * a.r + a.refinement) * (2 + d);
            const double* pole = a.pole + (size_t)q * d;
            for (int c = tid; c < d; c += blockDim.x) rec[2 + c] = pole[c];
            if (tid == 0) {
                rec[0] = a.dmin[q];
                rec[1] = a.eps;
            }
        }
        return;
    }
    double bval = INFINITY;
    long long bcnt = 0;
    int bidx = 0x7fffffff;
    if (a.notion == 0) {
        const int* cnt = a.counts + (size_t)q * a.mpad * 2;
        for (int j = tid; j < a.m; j += blockDim.x) {
            long long lt = cnt[2 * j], gt = cnt[2 * j + 1];
            long long c = a.n - (lt > gt ? lt : gt);
            double v = (double)c / (double)a.n;
            if (v < bval) {
                bval = v;
                bcnt = c;
                bidx = j;
            }
        }
    } else {
        const double* dep = a.depths + (size_t)q * a.m;
        for (int j = tid; j < a.m; j += blockDim.x) {
            double v = dep[j];
            if (v < bval) {
                bval = v;
                bidx = j;
            }
        }
    }
    // lexicographic (value, index) min
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        double ov = __shfl_xor_sync(0xffffffffu, bval, off);
        long long oc = __shfl_xor_sync(0xffffffffu, bcnt, off);
        int oi = __shfl_xor_sync(0xffffffffu, bidx, off);
        if (ov < bval || (ov == bval && oi < bidx)) {
            bval = ov;
            bcnt = oc;
            bidx = oi;
        }
    }
    if (lane == 0) {
        s_val[warp] = bval;
        s_cnt[warp] = bcnt;
        s_idx[warp] = bidx;
    }
    __syncthreads();
    if (tid == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
            if (s_val[w] < bval || (s_val[w] == bval && s_idx[w] < bidx)) {
                bval = s_val[w];
                bcnt = s_cnt[w];
                bidx = s_idx[w];
            }
        int improved = 0;
        if (bval < a.dmin[q]) {
            a.dmin[q] = bval;
            a.best_count[q] = bcnt;
            improved = 1;
        }
        s_best = bidx;
        s_improved = improved;
    }
    __syncthreads();
    double* pole = a.pole + (size_t)q * d;
    if (s_improved) {
        const double* src = a.u64 + ((size_t)q * a.m + s_best) * d;
        for (int c = tid; c < d; c += blockDim.x) pole[c] = src[c];
    }
    __syncthreads();
    if (a.trace) {
        double* rec = a.trace + ((size_t)q * a.r + a.refinement) * (2 + d);
        for (int c = tid; c < d; c += blockDim.x) rec[2 + c] = pole[c];
        if (tid == 0) {
            rec[0] = a.dmin[q];
            rec[1] = a.eps;
        }
    }
    // reflection vector for the next refinement's cap (reflect_to_pole)
    if (s_improved && tid == 0) {
        const double p1 = pole[0];
        double* v = a.refl_v + (size_t)q * d;
        int mode;
        if (1.0 - p1 < 1e-12) mode = 0;
        else if (1.0 + p1 < 1e-12) mode = 1;
        else {
            mode = 2;
            for (int c = 0; c < d; ++c) v[c] = -pole[c];
            v[0] += 1.0;
            double ss = 0.0;
            for (int c = 0; c < d; ++c) ss += v[c] * v[c];
            double vn = sqrt(ss);
            for (int c = 0; c < d; ++c) v[c] /= vn;
        }
        a.refl_mode[q] = mode;
    }
    if (a.notion == 0) {
        int* cnt = a.counts + (size_t)q * a.mpad * 2;
        for (int j = tid; j < a.mpad * 2; j += blockDim.x) cnt[j] = 0;
        // every direction's count is >= the rows coinciding with the query (they
        // are ties on both sides), so a best count at that bound is final
        if (a.done && tid == 0 && a.best_count[q] <= a.c0[q]) a.done[q] = 1;
    }
}

// DepthResult outputs for queries [0, Qb) of the batch.
__global__ void finalize_kernel(FinalArgs f) {
    int q = blockIdx.x;
    if (q >= f.Qb) return;
    for (int c = threadIdx.x; c < f.d; c += blockDim.x)
        if (f.argmin_out) f.argmin_out[(size_t)q * f.d + c] = f.pole[(size_t)q * f.d + c];
    if (threadIdx.x == 0) {
        f.depth_out[q] = f.dmin[q];
        if (f.count_out) f.count_out[q] = f.best_count[q];
    }
}

// ---------------------------------------------------------- data layouts --
// Dataset n x d FP64 row-major -> FP32 tile-blocked [T][d][BM]; pad rows 0.
__global__ void block_dataset_kernel(const double* __restrict__ x, float* __restrict__ xb, int64_t n,
                                     int d, int64_t tiles) {
    int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t total = tiles * d * BM;
    if (idx >= total) return;
    int i = (int)(idx % BM);
    int64_t r = idx / BM;
    int c = (int)(r % d);
    int64_t t = r / d;
    int64_t row = t * BM + i;
    xb[idx] = (row < n) ? (float)x[row * d + c] : 0.0f;
}

// flag |= 1 for a non-finite entry, |= 2 for |x| > 1e38 (beyond the FP32
// contraction range); grid-stride, one atomic per warp that found something
__global__ void validate_values_kernel(const double* __restrict__ x, int64_t count, int* __restrict__ flag) {
    int bad = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        const double v = x[i];
        if (!isfinite(v)) bad |= 1;
        else if (fabs(v) > 1.0e38) bad |= 2;
    }
    bad = __reduce_or_sync(0xffffffffu, bad);
    if (bad && (threadIdx.x & 31) == 0) atomicOr(flag, bad);
}

// max_l |x_il| per (padded) row of the tile-blocked FP32 dataset (the wide
// tensor path's per-point scale bound, contract_tcw.cu)
__global__ void row_absmax_kernel(const float* __restrict__ xb, float* __restrict__ xmax, int d, int64_t tiles) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= tiles * BM) return;
    const int64_t t = idx / BM;
    const int i = (int)(idx % BM);
    const float* row = xb + (size_t)t * d * BM + i;
    float m = 0.0f;
    for (int c = 0; c < d; ++c) m = fmaxf(m, fabsf(row[(size_t)c * BM]));
    xmax[idx] = m;
}

__global__ void queries_to_f32_kernel(const double* __restrict__ z, float* __restrict__ zq,
                                      int64_t count) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) zq[i] = (float)z[i];
}

// Known-answer entry: Philox words on device for a (4, N) counter array.
__global__ void philox_words_kernel(const uint32_t* __restrict__ ctr, uint32_t* __restrict__ out,
                                    int64_t N, uint32_t k0, uint32_t k1) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    uint32_t c0 = ctr[i], c1 = ctr[N + i], c2 = ctr[2 * N + i], c3 = ctr[3 * N + i];
    philox10(c0, c1, c2, c3, k0, k1);
    out[i] = c0;
    out[N + i] = c1;
    out[2 * N + i] = c2;
    out[3 * N + i] = c3;
}

// Explicit-direction mode for contract_tcf: hi-layout operand + FP32 rows from U64.
__global__ void pack_tcf_operand_kernel(const double* __restrict__ u64, unsigned char* __restrict__ uop,
                                        float* __restrict__ u32r, int Qb, int m, int NB, int mpad, int d) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // one (q, j) row per thread
    if (idx >= (int64_t)Qb * mpad) return;
    const int q = (int)(idx / mpad), j = (int)(idx % mpad);
    const bool real = j < m;
    const double* row = u64 + ((size_t)q * m + (real ? j : 0)) * d;
    const int dp = tcf_dp(d);
    float* r32 = u32r + ((size_t)q * mpad + j) * dp;
    for (int c = 0; c < dp; ++c) r32[c] = (real && c < d) ? (float)row[c] : 0.0f;
    if (j >= NB * 128) return;
    unsigned char* op = uop + ((size_t)q * NB + (j >> 7)) * tcf_block_bytes(d) + (size_t)(j & 127) * 16;
    for (int kk = 0; kk < 16 * tcf_ns(d); ++kk)
        *reinterpret_cast<__half*>(op + (kk >> 3) * 2048 + (kk & 7) * 2) = tcf_value(row, d, kk, real);
}

cudaError_t launch_pack_tcf_operand(const double* u64, unsigned char* uop, float* u32r, int Qb, int m, int NB,
                                    int mpad, int d, cudaStream_t st) {
    const int64_t total = (int64_t)Qb * mpad;
    pack_tcf_operand_kernel<<<(unsigned)((total + 127) / 128), 128, 0, st>>>(u64, uop, u32r, Qb, m, NB, mpad, d);
    return cudaGetLastError();
}

// ------------------------------------------------------ drop-in API helpers --
// directions.py:97-135 (_normal_rows / _unit_rows): row j (Philox index
// index_base + j) holds `dim` normals from value addresses v_base.., a zero-norm
// row is redrawn from the next dim addresses, then g / |g| with numpy's pairwise
// |g|^2 (random_sphere, directions.py:138-147).  One warp per row.
__global__ void __launch_bounds__(256) unit_rows_kernel(uint64_t seed, uint32_t l, uint32_t q, int m, int dim,
                                                        uint32_t v_base, uint32_t index_base, double* out) {
    extern __shared__ double usm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int j = blockIdx.x * 8 + warp;
    if (j >= m) return;
    double* g = usm + (size_t)warp * 2 * dim;
    double* sc = g + dim;
    uint32_t vb = v_base;
    double nrm = 0.0;
    for (;;) {
        for (int c = lane; c < dim; c += 32) {
            const double gv = ndtri(uniform1(seed, vb + (uint32_t)c, index_base + (uint32_t)j, l, q));
            g[c] = gv;
            sc[c] = gv * gv;
        }
        __syncwarp();
        if (lane == 0) nrm = sqrt(pw_sum(sc, dim));
        nrm = __shfl_sync(0xffffffffu, nrm, 0);
        __syncwarp();
        if (nrm != 0.0) break;
        vb += (uint32_t)dim;
    }
    for (int c = lane; c < dim; c += 32) out[(size_t)j * dim + c] = g[c] / nrm;
}

// SubStream.uniforms / .normals (directions.py:76-94): values offset + i of the
// substream (seed, refinement, query, index); normals = ndtri(uniform)
__global__ void stream_values_kernel(uint64_t seed, uint32_t l, uint32_t q, uint32_t index, uint32_t offset,
                                     int64_t count, int normal, double* out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const double u = uniform1(seed, offset + (uint32_t)i, index, l, q);
    out[i] = normal ? ndtri(u) : u;
}

cudaError_t launch_unit_rows(uint64_t seed, uint32_t l, uint32_t q, int m, int dim, uint32_t v_base,
                             uint32_t index_base, double* out, cudaStream_t st) {
    if (m < 1 || dim < 1) return cudaErrorInvalidValue;
    const size_t smem = (size_t)8 * 2 * dim * sizeof(double);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(unit_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    unit_rows_kernel<<<(unsigned)((m + 7) / 8), 256, smem, st>>>(seed, l, q, m, dim, v_base, index_base, out);
    return cudaGetLastError();
}

cudaError_t launch_stream_values(uint64_t seed, uint32_t l, uint32_t q, uint32_t index, uint32_t offset,
                                 int64_t count, int normal, double* out, cudaStream_t st) {
    if (count < 1) return cudaSuccess;
    stream_values_kernel<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(seed, l, q, index, offset, count, normal,
                                                                          out);
    return cudaGetLastError();
}

// ----------------------------------------------------------------- launch --
cudaError_t launch_cap_generate(const GenArgs& a, cudaStream_t st) {
    int64_t total = (int64_t)a.Qb * a.mpad;
    if (a.d >= 2 && a.d <= GV_MAX_D && a.mpad % GV_DIRS == 0 && a.jbase == 0) {
        const size_t smem = (size_t)GV_DIRS * a.d * 8 + 2 * GV_DIRS * 8 + (size_t)GV_DIRS * (a.d - 1) * 2 + 16;
        if (smem > 48 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(cap_generate_v2_kernel,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return e;
        }
        cap_generate_v2_kernel<<<(unsigned)(total / GV_DIRS), GV_THREADS, smem, st>>>(a);
        return cudaGetLastError();
    }
    int blocks = (int)((total + 7) / 8);
    size_t smem = (size_t)8 * 2 * a.d * sizeof(double);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(cap_generate_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    cap_generate_kernel<<<blocks, 256, smem, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_pack_directions(const double* u64, float* u32, int Qb, int m, int mpad, int d,
                                   cudaStream_t st) {
    int64_t total = (int64_t)Qb * mpad * d;
    pack_directions_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(u64, u32, Qb, m, mpad, d);
    return cudaGetLastError();
}

cudaError_t launch_state_init(const StateArgs& s, cudaStream_t st) {
    state_init_kernel<<<s.Qb, 64, 0, st>>>(s);
    return cudaGetLastError();
}

cudaError_t launch_update(const UpdateArgs& a, cudaStream_t st) {
    update_kernel<<<a.Qb, 256, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_finalize(const FinalArgs& f, cudaStream_t st) {
    finalize_kernel<<<f.Qb, 64, 0, st>>>(f);
    return cudaGetLastError();
}

cudaError_t launch_block_dataset(const double* x, float* xb, int64_t n, int d, int64_t tiles,
                                 cudaStream_t st) {
    int64_t total = tiles * d * BM;
    block_dataset_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(x, xb, n, d, tiles);
    return cudaGetLastError();
}

cudaError_t launch_validate_values(const double* x, int64_t count, int* flag, cudaStream_t st) {
    if (count == 0) return cudaSuccess;
    int64_t blocks = (count + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    validate_values_kernel<<<(unsigned)blocks, 256, 0, st>>>(x, count, flag);
    return cudaGetLastError();
}

cudaError_t launch_row_absmax(const float* xb, float* xmax, int d, int64_t tiles, cudaStream_t st) {
    const int64_t total = tiles * BM;
    if (total == 0) return cudaSuccess;
    row_absmax_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(xb, xmax, d, tiles);
    return cudaGetLastError();
}

cudaError_t launch_queries_to_f32(const double* z, float* zq, int64_t count, cudaStream_t st) {
    if (count == 0) return cudaSuccess;
    queries_to_f32_kernel<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(z, zq, count);
    return cudaGetLastError();
}

cudaError_t launch_philox_words(const uint32_t* ctr, uint32_t* out, int64_t N, uint32_t k0,
                                uint32_t k1, cudaStream_t st) {
    if (N == 0) return cudaSuccess;
    philox_words_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(ctr, out, N, k0, k1);
    return cudaGetLastError();
}

}  // namespace rrs
