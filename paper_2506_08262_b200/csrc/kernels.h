// kernels.h -- argument blocks and launchers shared by the engine and kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace rrs {

struct GenArgs {
    const double* pole;      // [Qb][d]
    const int* refl_mode;    // [Qb] 0 none, 1 negate e1 coordinate, 2 Householder
    const double* refl_v;    // [Qb][d]
    double* u64;             // [Qb][m][d]
    float* u32;              // [Qb][mpad/BN][d][BN]
    unsigned char* uop;      // nullable: [Qb][NB][block bytes] FP16 tensor operand (layout by uop_mode)
    int uop_mode;            // 0: split layout (tc_layout, contract_tc/tcw), 1: hi layout (contract_tcf)
    float* u32r;             // nullable: [Qb][mpad][tcf_dp(d)] FP32 direction rows (contract_tcf refinement)
    int NB;                  // 128-direction blocks per query in uop
    uint64_t seed;
    uint32_t jbase;          // Philox index of direction 0 (random_sphere_pole's stream.index; warp path)
    int64_t q0;              // global query index of batch row 0
    uint32_t refinement;
    double eps;
    int Qb, m, mpad, d;
    const int* done;         // nullable [Qb]: early exit, skip these queries
};

struct StateArgs {
    double* pole;
    double* refl_v;
    int* refl_mode;
    double* dmin;
    long long* best_count;
    long long n;
    int Qb, d;
};

struct UpdateArgs {
    int* counts;             // [Qb][mpad][2] (lt, gt), halfspace; cleared after use
    const double* depths;    // [Qb][m], projection notions
    const double* u64;       // [Qb][m][d]
    double* pole;
    double* refl_v;
    int* refl_mode;
    double* dmin;
    long long* best_count;
    double* trace;           // [Qb][r][2+d] or null
    long long n;
    double eps;
    int Qb, m, mpad, d, r, refinement, notion;
    int* done;               // nullable [Qb]: early exit (halfspace); set when best count <= c0
    const long long* c0;     // [Qb] rows coinciding with the query (the count's lower bound)
};

struct FinalArgs {
    const double* pole;
    const double* dmin;
    const long long* best_count;
    double* depth_out;
    double* argmin_out;
    long long* count_out;
    int Qb, d;
};

// Contraction of the blocked data against one direction block per work unit.
struct ContractArgs {
    const float* xb;         // [T][d][BM]
    const float* u32;        // [Qb][MB][d][BN]
    const float* zq;         // [Qb][d]
    int* counts;             // [Qb][MB*BN][2]       (count mode)
    float* y;                // [Qb][jcount*BN][n]   (store mode), direction j - jb0*BN
    int64_t n;
    int64_t tiles;           // T
    int d;
    int Qb;
    int MB;                  // direction blocks per query (mpad / BN)
    int jb0, jbn;            // direction-block range handled by this launch
    int m;                   // real directions per query
    int tiles_per_unit;
    int chunks;              // ceil(T / tiles_per_unit)
    const int* done;         // nullable [Qb]: early exit, skip these queries (count mode)
};

// Tensor-core (FP16 hi/lo split) halfspace contraction, contract_tc.cu.
// Packed K layout of the split products.  Per 64-coordinate slice of width
// 16 Q + r (d <= 64: the only slice), both operands store each FP16 term once:
//   K steps [0, Q)      hi terms of coordinates 16 g .. 16 g + 15 (A: uh, B: bh)
//   K steps [Q, 2Q)     lo terms of the same coordinates          (A: ul, B: bl)
//   K steps [2Q, 2Q+R)  the r remainder coordinates, R = ceil(3 r / 16): element
//                       e = kk - 32 Q < 3 r holds product e / r of coordinate
//                       16 Q + e % r (products hi*hi, hi*lo, lo*hi: A values
//                       h, h, l; B values h, l, h), the rest zero.
// The MMAs of a slice pair the chunks explicitly: for g < Q the three products
// (A g, B g) = uh bh, (A g, B Q+g) = uh bl, (A Q+g, B g) = ul bh, then
// (A 2Q+i, B 2Q+i) for i < R, so
//   sum = sum_c (uh bh + uh bl + ul bh)   in 3 Q + R MMAs of K = 16
// from 2 Q + R stored K steps (d = 50: 10 MMAs over 7 steps; the A operand of a
// direction block takes 56 TMEM columns instead of 80).
// d > 64 (contract_tcw.cu): slices s < full are full (Q = 4, r = 0: 8 stored
// steps, 12 MMAs) at K steps [8 s, 8 s + 8); the last slice (width 1..64)
// follows with its own Q / r.
// Storage: canonical K-major, no swizzle: [kk / 8][row 128][8 fp16] per
// 128-row block, i.e. ns * 4096 bytes per block.
struct TcLayout {
    int q16, rem, ns;  // q16 / rem of the last slice (of d itself when d <= 64); ns: stored K steps, all slices
    int full;          // full 64-coordinate slices before the last one
    int rsteps;        // R: remainder K steps of the last slice
    int nmma;          // MMAs per (point tile, direction block): 12 full + 3 q16 + R
};
constexpr int TC_SLICE = 64;
constexpr int TC_SLICE_NS = 8;    // stored K steps of a full slice
constexpr int TC_SLICE_NS_MAX = 9;  // of any slice: a last slice of 59..63 coordinates takes 2 * 3 + 3
constexpr int TC_SLICE_MMA = 12;  // its MMAs
__host__ __device__ inline TcLayout tc_layout(int d) {
    TcLayout L;
    L.full = d > 0 ? (d - 1) / TC_SLICE : 0;
    const int dl = d - TC_SLICE * L.full;
    L.q16 = dl / 16;
    L.rem = dl % 16;
    L.rsteps = (3 * L.rem + 15) / 16;
    L.ns = TC_SLICE_NS * L.full + 2 * L.q16 + L.rsteps;
    L.nmma = TC_SLICE_MMA * L.full + 3 * L.q16 + L.rsteps;
    return L;
}
__host__ __device__ inline int tc_block_bytes(int d) { return tc_layout(d).ns * 4096; }
// slice of coordinate c and its (base K position, Q, r, local coordinate)
__host__ __device__ inline void tc_slice_of(const TcLayout& L, int c, int& base, int& q, int& r, int& cl) {
    const int s = c / TC_SLICE < L.full ? c / TC_SLICE : L.full;
    base = 16 * TC_SLICE_NS * s;
    cl = c - TC_SLICE * s;
    q = s < L.full ? 4 : L.q16;
    r = s < L.full ? 0 : L.rem;
}
// stored terms of coordinate c: 2 in the aligned part (hi, lo), 3 in the remainder (products 0..2)
__host__ __device__ inline int tc_entries(const TcLayout& L, int c) {
    int base, q, r, cl;
    tc_slice_of(L, c, base, q, r, cl);
    return cl < 16 * q ? 2 : 3;
}
// K position of entry e of coordinate c
__host__ __device__ inline int tc_pos(const TcLayout& L, int e, int c) {
    int base, q, r, cl;
    tc_slice_of(L, c, base, q, r, cl);
    return base + (cl < 16 * q ? 16 * q * e + cl : 32 * q + e * r + (cl - 16 * q));
}
// whether entry e of coordinate c holds the lo term in A (the direction operand)
// / in B (the point operand)
__host__ __device__ inline bool tc_a_lo(const TcLayout& L, int e, int c) { return tc_entries(L, c) == 2 ? e == 1 : e == 2; }
__host__ __device__ inline bool tc_b_lo(const TcLayout&, int e, int) { return e == 1; }
// inverse: entry e and coordinate c of K position kk (c = -1: zero padding)
__host__ __device__ inline void tc_elem(const TcLayout& L, int kk, int& e, int& c) {
    const int s = kk / (16 * TC_SLICE_NS) < L.full ? kk / (16 * TC_SLICE_NS) : L.full;
    const int kl = kk - 16 * TC_SLICE_NS * s;
    const int c0 = TC_SLICE * s;
    const int q = s < L.full ? 4 : L.q16, r = s < L.full ? 0 : L.rem;
    if (kl < 32 * q) {
        e = kl / (16 * q);
        c = c0 + kl - 16 * q * e;
    } else {
        const int x = kl - 32 * q;
        if (r == 0 || x >= 3 * r) {
            e = 0;
            c = -1;
        } else {
            e = x / r;
            c = c0 + 16 * q + x % r;
        }
    }
}
// MMA i of a slice with q aligned groups (i < 3 q + R): its slice-local A and B
// K steps -- (g, g), (g, q + g), (q + g, g) for g = i / 3, then (2q + j, 2q + j)
__host__ __device__ inline void tc_mma_steps(int q, int i, int& sa, int& sb) {
    if (i < 3 * q) {
        const int g = i / 3, k = i - 3 * g;
        sa = k == 2 ? q + g : g;
        sb = k == 1 ? q + g : g;
    } else {
        sa = sb = 2 * q + (i - 3 * q);
    }
}
// 16-byte chunk cc (K positions 8 cc .. 8 cc + 7): true when it holds the hi
// (lo = false) or lo terms of the 8 consecutive coordinates c0 .. c0 + 7 (the
// aligned parts of the slices)
__host__ __device__ inline bool tc_chunk_run(const TcLayout& L, int cc, bool& lo, int& c0) {
    const int kk = 8 * cc;
    const int s = kk / (16 * TC_SLICE_NS) < L.full ? kk / (16 * TC_SLICE_NS) : L.full;
    const int kl = kk - 16 * TC_SLICE_NS * s;
    const int q = s < L.full ? 4 : L.q16;
    if (kl >= 32 * q) return false;
    lo = kl >= 16 * q;
    c0 = TC_SLICE * s + kl - (lo ? 16 * q : 0);
    return true;
}

// Six-product layout of the tensor-core projection STORE (contract_tcs.cu, d <= 64):
// three-way FP16 split a s = ah + am + al, u 2^15 = uh + um + ul (33 bits each),
// products p = 0..5: uh ah, uh am, um ah, uh al, ul ah, um am (the dropped
// terms are ~2^-33), A value per product {h, h, m, h, l, m}, B value
// {h, m, h, l, h, m}; packed along K like tc_layout with 6 products:
// d = 16 Q + r, ns = 6 Q + ceil(6 r / 16).
struct Tc6Layout {
    int q16, rem, ns;
};
__host__ __device__ inline Tc6Layout tc6_layout(int d) {
    Tc6Layout L;
    L.q16 = d / 16;
    L.rem = d % 16;
    L.ns = 6 * L.q16 + (6 * L.rem + 15) / 16;
    return L;
}
__host__ __device__ inline int tc6_block_bytes(int d) { return tc6_layout(d).ns * 4096; }
__host__ __device__ inline int tc6_pos(const Tc6Layout& L, int p, int c) {
    return c < 16 * L.q16 ? 16 * (p * L.q16 + c / 16) + c % 16 : 96 * L.q16 + p * L.rem + (c - 16 * L.q16);
}
__host__ __device__ inline void tc6_elem(const Tc6Layout& L, int kk, int& p, int& c) {
    if (kk < 96 * L.q16) {
        const int s = kk / 16;
        p = s / L.q16;
        c = 16 * (s % L.q16) + kk % 16;
    } else {
        const int e = kk - 96 * L.q16;
        if (L.rem == 0 || e >= 6 * L.rem) {
            p = 0;
            c = -1;
        } else {
            p = e / L.rem;
            c = 16 * L.q16 + e % L.rem;
        }
    }
}
// which split term (0 h, 1 m, 2 l) product p takes from A (directions) / B (points)
__host__ __device__ inline int tc6_a_term(int p) { return (0x120100 >> (4 * p)) & 0xF; }
__host__ __device__ inline int tc6_b_term(int p) { return (0x102010 >> (4 * p)) & 0xF; }

struct TcsArgs {
    const float* xb;            // [T][d][128]
    const float* zq;            // [Qb][d]
    const unsigned char* uop;   // [Qb][NB][tc6_block_bytes(d)] direction operand (six-product layout)
    float* y;                   // [Qb][jbn * 128][n] projections y = <u, x - z> of the chunk
    int64_t n;
    int64_t tiles;
    int d, Qb, NB, m;
    int jb0, jbn;               // direction blocks of this chunk
    // filled by launch_contract_tcs
    int groups, chunks, raw_stages, gb;
    int64_t tiles_per_chunk;
};

struct TcArgs {
    const float* xb;            // [T][d][128]
    const float* xmax;          // [T * 128] max_l |x_il| (0 for padding rows); contract_tcw.cu only
    const float* zq;            // [Qb][d]
    const unsigned char* uop;   // [Qb][NB][tc_block_bytes(d)] direction operand
    int* counts;                // [Qb][mpad][2]
    int64_t n;
    int64_t tiles;
    int d, Qb, NB, m, mpad;
    // filled by launch_contract_tc
    int groups, chunks, raw_stages, gb;
    int64_t tiles_per_chunk;
    const int* done;            // nullable [Qb]: early exit, units of these queries are skipped
    // projection store on the wide kernel (contract_tcw.cu STORE mode): direction
    // blocks [jb0, jb0 + jbn) of each query, rows y[q][(blk - jb0) * 128 + j][n]
    float* y;
    int jb0, jbn;
    // pre-split point operand (contract_tcp.cu): [T][ns][128][8 fp16] B operand of
    // every tile in the tc_layout, per-point 1 / (s_i 2^15); count mode adds the
    // per-direction shift (FP64 [Qb][m], y = acc inv_i + shift_j) and excludes the
    // rows coinciding with the query (coin[q][0 .. coin_n[q]), coin_n <= TCP_COIN_MAX)
    const unsigned char* xps;
    const float* pinv;
    const double* dshift;
    const int* coin;
    const int* coin_n;
};
constexpr int TCP_COIN_MAX = 64;  // coinciding rows listed per query (more: the converter kernel)

// Filter-and-refine halfspace contraction (contract_tcf.cu, d <= 64): one FP16
// product per coordinate, K = d + 1.  Direction operand A (written by gen.cu):
// coordinate l at K index l holds fp16(u_l * TCF_SU), K index d the threshold
// slot (1, or 4 for padded directions j >= m), zeros after; canonical K-major
// [kk/8][row 128][8 fp16] per 128-direction block, ns = ceil((d+1)/16) steps.
// The point operand is built in the kernel (b_l = fp16(a_l * TCF_CB / ||a||)).
// FP32 rows for the exact refinement: directions u32 = (float)u64 as
// [Qb][mpad][dp], dp = d rounded up to 4 (the points' a = x - z rows are
// formed in the kernel).
constexpr float TCF_SU = 1024.0f;
constexpr float TCF_CB = 0.833333313f;  // TCF_SU * TCF_CB = 2^10 / 1.2: bound margin, see contract_tcf.cu
__host__ __device__ inline int tcf_ns(int d) { return (d + 16) / 16; }
__host__ __device__ inline int tcf_dp(int d) { return (d + 3) & ~3; }
__host__ __device__ inline int tcf_block_bytes(int d) { return tcf_ns(d) * 4096; }

struct TcfArgs {
    const float* xb;            // [T][d][128] tile-blocked FP32 dataset (the FFMA kernel's layout)
    const float* zq;            // [Qb][d]
    const unsigned char* uop;   // [Qb][NB][tcf_block_bytes(d)] direction operand (hi layout)
    const float* u32r;          // [Qb][mpad][dp] FP32 direction rows
    int* counts;                // [Qb][mpad][2]
    int64_t n;
    int64_t tiles;
    int d, Qb, NB, m, mpad;
    // filled by launch_contract_tcf
    int groups, chunks, gb, sa;
    int64_t tiles_per_chunk;
};

// Univariate projection depths from stored projections y (difference form).
struct SelectArgs {
    const float* y;          // [Qb][jcount][n] (row stride n)
    double* depths;          // [Qb][m]
    int64_t n;
    int Qb;
    int jcount;              // directions per query in this chunk (rows of y)
    int j0;                  // first direction of the chunk
    int m;
    int notion;              // 1 projection, 2 asym projection
    const double* shift;     // nullable [Qb][m]: y = y' + shift (centred frame, center.cu); med += shift
    int variant;             // 0 auto (sample-bracket select where it applies), 2 radix select v2
    unsigned* fallbacks;     // nullable device counter: rows that left the sample bracket (select v3)
};

cudaError_t launch_cap_generate(const GenArgs& a, cudaStream_t st);
cudaError_t launch_pack_directions(const double* u64, float* u32, int Qb, int m, int mpad, int d,
                                   cudaStream_t st);
cudaError_t launch_state_init(const StateArgs& s, cudaStream_t st);
cudaError_t launch_update(const UpdateArgs& a, cudaStream_t st);
cudaError_t launch_finalize(const FinalArgs& f, cudaStream_t st);
cudaError_t launch_block_dataset(const double* x, float* xb, int64_t n, int d, int64_t tiles,
                                 cudaStream_t st);
cudaError_t launch_queries_to_f32(const double* z, float* zq, int64_t count, cudaStream_t st);
cudaError_t launch_philox_words(const uint32_t* ctr, uint32_t* out, int64_t N, uint32_t k0,
                                uint32_t k1, cudaStream_t st);
cudaError_t launch_contract_count(const ContractArgs& a, cudaStream_t st);
cudaError_t launch_contract_store(const ContractArgs& a, cudaStream_t st);
cudaError_t launch_select(const SelectArgs& a, cudaStream_t st);
// FP64 contraction for d > 256 (contract64.cu): count mode (halfspace) or
// store mode (centred projection rows)
constexpr int TC_MAX_D = 256;        // the FP32 / tensor paths; above it contract64
struct Contract64Args {
    const double* x64;       // [n][d] FP64 data (row-major)
    const double* c;         // centre per query: c + q * c_stride (z for halfspace, m for the store)
    int64_t c_stride;
    const double* u64;       // [Qb][m][d]
    int* counts;             // [Qb][mpad][2] (#y<0, #y>0), count mode
    float* y;                // [Qb][jcount][n], store mode
    int64_t n;
    int d, m, mpad, jbase, jcount, Qb;
    const int* done;         // nullable [Qb]: early exit, skip these queries (count mode)
};
cudaError_t launch_contract64(const Contract64Args& a, bool store, cudaStream_t st);
// early exit: rows coinciding with each query (FP32 equality on the blocked
// data, or FP64 on the row-major copy for the d > 256 path)
cudaError_t launch_coincide_count32(const float* xb, const float* zq, int64_t n, int d, int64_t tiles, int Qb,
                                    long long* c0, cudaStream_t st);
cudaError_t launch_coincide_count64(const double* x64, const double* z, int64_t n, int d, int Qb, long long* c0,
                                    cudaStream_t st);
// centred frame of the projection notions (center.cu)
constexpr int64_t STORE64_N = 4096;  // below: FP64-accumulated store from an FP64 centred copy
// centre m_c (lower median of a strided 1024-row sample) and the column's
// interquartile range on that sample (iqr may be null)
cudaError_t launch_center_sample(const double* x, int64_t n, int d, double* center, double* iqr, cudaStream_t st);
cudaError_t launch_block_centered(const double* x, const double* center, float* xb, int64_t n, int d, int64_t tiles,
                                  cudaStream_t st);
cudaError_t launch_center_copy64(const double* x, const double* center, double* xc, int64_t n, int d,
                                 cudaStream_t st);
cudaError_t launch_direction_shift(const double* u64, const double* center, const double* z, double* shift, int Qb,
                                   int m, int d, cudaStream_t st);
cudaError_t launch_store64(const double* xc, const double* u64, float* y, int64_t n, int d, int Qb, int m, int j0,
                           int jcount, cudaStream_t st);
cudaError_t launch_contract_tc(TcArgs a, int sms, cudaStream_t st);
cudaError_t launch_contract_tcf(TcfArgs a, int sms, cudaStream_t st);  // filter and refine, d <= 64
cudaError_t launch_pack_tcf_operand(const double* u64, unsigned char* uop, float* u32r, int Qb, int m, int NB,
                                    int mpad, int d, cudaStream_t st);
cudaError_t launch_contract_tcw(TcArgs a, int sms, cudaStream_t st);
// converter-free wide tensor kernel (contract_tcp.cu, 64 < d <= 256): counts / centred store
cudaError_t launch_contract_tcp(TcArgs a, int sms, cudaStream_t st);
cudaError_t launch_contract_tcp_store(TcArgs a, int sms, cudaStream_t st);
// pre-split point operand from a tile-blocked FP32 copy and its per-row max |x|
cudaError_t launch_presplit(const float* xb, const float* rowmax, int64_t n, int d, int64_t tiles,
                            unsigned char* xps, float* pinv, cudaStream_t st);
// rows FP32-equal to each query: count (c0, int64) and the first TCP_COIN_MAX indices
cudaError_t launch_coincide_list32(const float* xb, const float* zq, int64_t n, int d, int64_t tiles, int Qb,
                                   long long* c0, int* coin, int* coin_n, cudaStream_t st);
cudaError_t launch_contract_tcw_store(TcArgs a, int sms, cudaStream_t st);  // centred projection store, 64 < d <= 256
cudaError_t launch_contract_tc_store(TcArgs a, int sms, cudaStream_t st);   // centred projection store, d <= 64
bool contract_tc_store_fits(int d);  // its shared-memory layout leaves >= 2 raw-tile stages  // 64 < d <= 256 (contract_tcw.cu)
cudaError_t launch_contract_tcs(TcsArgs a, int sms, cudaStream_t st);  // projection store, d <= 64
cudaError_t launch_pack_tc6_operand(const double* u64, unsigned char* uop, int Qb, int m, int NB, int d,
                                    cudaStream_t st);
// drop-in API helpers (api64.cu, gen.cu)
cudaError_t launch_proj64(const double* x, const double* u, double* out, int64_t n, int m, int d, cudaStream_t st);
cudaError_t launch_span_depth64(const double* px, const double* pz, double* out, int m, int64_t n, int notion,
                                cudaStream_t st);
cudaError_t launch_unit_rows(uint64_t seed, uint32_t l, uint32_t q, int m, int dim, uint32_t v_base,
                             uint32_t index_base, double* out, cudaStream_t st);
cudaError_t launch_stream_values(uint64_t seed, uint32_t l, uint32_t q, uint32_t index, uint32_t offset,
                                 int64_t count, int normal, double* out, cudaStream_t st);
cudaError_t launch_validate_values(const double* x, int64_t count, int* flag, cudaStream_t st);
cudaError_t launch_row_absmax(const float* xb, float* xmax, int d, int64_t tiles, cudaStream_t st);
cudaError_t launch_pack_tc_operand(const double* u64, unsigned char* uop, int Qb, int m, int NB, int d,
                                   cudaStream_t st);
size_t contract_tc_smem_bytes();
size_t contract_smem_bytes(int d);

}  // namespace rrs
