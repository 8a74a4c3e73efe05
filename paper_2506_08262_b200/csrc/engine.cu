// engine.cu -- the C-ABI (include/rrs_b200.h) and the per-device RRS engine.
//
// The engine owns the device-resident dataset (FP32, tile-blocked), a grow-only
// workspace sized for a batch of queries, and one CUDA stream.  depth_batch
// runs, per query batch, r refinements of
//     K1 cap_generate  ->  K2 contract (count | store)  [-> K3 select]  ->  K4 update
// entirely on device (no host round-trips between refinements), then writes
// DepthResult fields.  Reference: optimizer.py:145-279.
#include "common.cuh"
#include "kernels.h"
#include "../../include/rrs_b200.h"

#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

using namespace rrs;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CK(expr)                                                                                \
    do {                                                                                        \
        cudaError_t _e = (expr);                                                                \
        if (_e != cudaSuccess)                                                                  \
            return fail(RRS_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));      \
    } while (0)

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    cudaError_t ensure(size_t need) {
        if (need <= bytes) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        size_t want = need + need / 8;
        cudaError_t e = cudaMalloc(&p, want);
        if (e != cudaSuccess) {
            cudaGetLastError();
            e = cudaMalloc(&p, need);
            if (e != cudaSuccess) {
                p = nullptr;
                return e;
            }
            want = need;
        }
        bytes = want;
        return cudaSuccess;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

int sm_count_of(int device) {
    int v = 148;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
    return v;
}

}  // namespace

struct rrs_engine {
    int device = 0;
    int sms = 148;
    cudaStream_t own = nullptr;
    cudaStream_t stream = nullptr;
    int64_t ws_limit = 8ll << 30;
    // dataset
    DevBuf xb;
    DevBuf xmax;  // [tiles * BM] max_l |x_il| (wide tensor path, 64 < d <= 256)
    // centred frame of the projection notions (center.cu): m, the FP32 blocked
    // copy of x - m, and for n < STORE64_N the FP64 row-major copy of x - m
    DevBuf center, xcb, xc64, xcmax;  // xcmax: max_l |x_il - m_l| per row (wide tensor store)
    double col_ratio = 1.0;           // max / min column IQR (> 0) of the centre sample (store gating)
    DevBuf x64;  // d > 256: FP64 row-major copy of the data (contract64.cu)
    // pre-split point operands of the converter-free wide tensor kernel
    // (contract_tcp.cu, 64 < d <= 256), built on first use per dataset:
    // [0] x (halfspace counts), [1] x - m (centred projection store)
    DevBuf xps[2], pinv[2];
    bool xps_ok[2] = {false, false};
    DevBuf coin, coin_n, zero_d;  // coinciding-row lists per query; d zeros (halfspace shift centre)
    int64_t n = 0;
    int d = 0;
    int64_t tiles = 0;
    // workspace
    DevBuf zq, u64, u32, uop, counts, depths, y, pole, reflv, reflmode, dmin, bestcnt;
    DevBuf zq0, shift;  // projection notions: zero queries for the centred store, <u, m - z> per direction
    DevBuf done, c0;    // early exit (halfspace): finished flags, coinciding-row counts per query
    // 0 auto, 1 FFMA (contract.cu), 2 tensor cores (contract_tc.cu two-term split for d <= 64,
    // contract_tcp.cu above), 4 filter and refine (contract_tcf.cu, d <= 64), 5 three-term tensor
    // projection store, 6 tensor with the in-kernel converters above d = 64 (contract_tcw.cu);
    // 3 (2-SM split) was removed
    int contract_path = 0;
    int select_path = 0;  // 0 auto (select v3 where it applies), 2 radix select v2
    DevBuf fallbacks;     // device counter of select-v3 rows that left their bracket
    DevBuf tmp_in, tmp_out0, tmp_out1, tmp_out2, tmp_out3;
    DevBuf qflag;  // device-query validation flag (rrs_depth_batch_device)
    // timing
    bool timing = false;
    rrs_stats stats{};
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    struct Mark {
        int stage;  // 0 gen, 1 contract, 2 univariate, 3 update
        size_t a, b;
    };
    std::vector<Mark> marks;

    cudaEvent_t next_event() {
        if (ev_used == ev_pool.size()) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            ev_pool.push_back(e);
        }
        return ev_pool[ev_used++];
    }
};

namespace {

struct Timer {
    rrs_engine* e;
    int stage;
    size_t a = 0;
    Timer(rrs_engine* e_, int stage_) : e(e_), stage(stage_) {
        if (e->timing) {
            a = e->ev_used;
            cudaEventRecord(e->next_event(), e->stream);
        }
    }
    ~Timer() {
        if (e->timing) {
            size_t b = e->ev_used;
            cudaEventRecord(e->next_event(), e->stream);
            e->marks.push_back({stage, a, b});
        }
    }
};

int set_device(rrs_engine* e) {
    CK(cudaSetDevice(e->device));
    return RRS_OK;
}

int validate_cfg(const rrs_config* c) {
    if (!c) return fail(RRS_ERR_INVALID, "config is null");
    if (c->refinements < 1 || c->total_directions < c->refinements)
        return fail(RRS_ERR_INVALID, "need total_directions >= refinements >= 1");
    if (!(c->shrink > 0.0 && c->shrink < 1.0))
        return fail(RRS_ERR_INVALID, "shrink factor must lie in (0, 1)");
    if (c->notion < 0 || c->notion > 2) return fail(RRS_ERR_INVALID, "unknown depth notion");
    if (c->pole_update < 0 || c->pole_update > 1)
        return fail(RRS_ERR_INVALID, "unknown pole update mode");
    if (c->early_exit < 0 || c->early_exit > 1) return fail(RRS_ERR_INVALID, "early_exit must be 0 or 1");
    if ((c->total_directions + c->refinements - 1) / c->refinements > (int64_t)1 << 24)
        return fail(RRS_ERR_INVALID, "directions per refinement exceed 2^24");
    return RRS_OK;
}

struct Plan {
    int m, mpad, MB, Qb;
    bool tc;     // tensor-core contraction (halfspace, d <= 256; contract_tcw.cu for d > 64)
    bool tcf;    // ... by filter and refine (contract_tcf.cu, d <= 64; u32 holds FP32 rows)
    bool tcs;    // tensor-core projection store (projection notions, d <= 50; contract_tcs.cu)
    bool store64;  // FP64-accumulated store (projection notions, n < STORE64_N, no tensor store; center.cu)
    bool wide;     // d > 256: FP64 contraction (contract64.cu) for counts and the store
    bool tcws;     // projection store on the wide tensor kernel (contract_tcw.cu STORE, 64 < d <= 256)
    bool tcst;     // projection store on the d <= 64 tensor kernel (contract_tc.cu STORE)
    bool tcp;      // 64 < d <= 256 on the pre-split kernel (contract_tcp.cu) instead of contract_tcw.cu
    int nb8;     // 128-direction blocks per query (tensor path operand, tc_block_bytes(d) each)
    int jchunk;  // direction blocks per store launch (projection notions)
    int tpu, chunks;
};

Plan make_plan(const rrs_engine* e, int64_t Q, int m, int notion) {
    Plan p{};
    p.m = m;
    p.MB = (m + BN - 1) / BN;
    p.mpad = p.MB * BN;
    p.nb8 = p.MB;
    const bool tc_ok = notion == RRS_HALFSPACE && e->d <= 256;
    p.tc = tc_ok && (e->contract_path >= 2 || (e->contract_path == 0 && e->n >= 4096));
    p.tcf = p.tc && e->d <= TC_SLICE && e->contract_path == 4;
    // projection store (centred frame): the 2-term FP16 split on the tensor cores for
    // n >= 4096 -- contract_tc.cu STORE for d <= 64 (up to 8 direction blocks share a
    // converted point tile), contract_tcw.cu STORE above; the three-way split
    // (contract_tcs.cu) only when forced (path 5); FP64 below n = 4096
    // the FP16-split stores scale each point by a power of two from its largest
    // coordinate, so a column whose spread is tiny next to another's is resolved
    // only to 2^-22 (2-term) / 2^-33 (3-term) of the large one; auto takes them
    // for scale-homogeneous data only (column IQR ratio, measured at set_dataset)
    // 2-term split stores (contract_tc / contract_tcw STORE) for n >= 4096; the
    // 3-term split (contract_tcs) for 32 <= d <= 50 when the columns are too
    // heterogeneous for 22 bits, for forced tensor stores on small n, or forced
    // (path 5); FP64 below n = 4096 otherwise; FFMA for the rest
    const bool proj = notion != RRS_HALFSPACE;
    const bool forced = e->contract_path == 2;
    const bool autop = e->contract_path == 0 || e->contract_path == 6;
    const bool big = e->n >= 4096;
    p.wide = e->d > TC_MAX_D;
    const bool split2 = proj && big && (forced || (autop && e->col_ratio <= 8.0));
    p.tcst = split2 && e->d <= TC_SLICE && contract_tc_store_fits(e->d);
    p.tcws = split2 && e->d > TC_SLICE && !p.wide;
    p.tcs = proj && !p.tcst && tc6_layout(e->d).ns <= 19 &&
            (e->contract_path == 5 || (forced && !big) ||
             (autop && big && e->d >= 32 && e->col_ratio <= 4096.0));
    p.store64 = proj && !p.tcs && !p.tcst && !p.tcws && e->n < STORE64_N;
    // above d = 64 both the counts and the store run on the pre-split kernel
    // (contract_tcp.cu) unless the in-kernel converters are forced (path 6)
    p.tcp = (p.tc || p.tcws) && e->d > TC_SLICE && e->contract_path != 6;
    const int64_t d = e->d, n = e->n;
    int64_t per_q = (int64_t)m * d * 8 + (int64_t)p.mpad * tcf_dp((int)d) * 4 + (int64_t)p.mpad * 8 + (int64_t)m * 16 +
                    d * 40 + 64 +
                    (int64_t)p.nb8 * (p.tcs ? tc6_block_bytes(e->d) : p.tcf ? tcf_block_bytes(e->d) : tc_block_bytes(e->d));
    int64_t budget = e->ws_limit;
    int64_t qb = 4096;
    if (notion != RRS_HALFSPACE) {
        const int64_t ybudget = budget / 2;
        const int64_t yq = (int64_t)p.mpad * n * 4;
        if (yq <= ybudget) {
            p.jchunk = p.MB;
            int64_t lim = ybudget / yq;
            if (lim < qb) qb = lim;
        } else {
            qb = 1;
            int64_t jc = ybudget / ((int64_t)BN * n * 4);
            p.jchunk = (int)(jc < 1 ? 1 : (jc > p.MB ? p.MB : jc));
        }
        budget -= (int64_t)qb * p.jchunk * BN * n * 4;
    } else {
        p.jchunk = p.MB;
    }
    int64_t lim = budget / per_q;
    if (lim < qb) qb = lim;
    if (qb > Q) qb = Q;
    if (qb < 1) qb = 1;
    p.Qb = (int)qb;
    // point-tile chunking for load balance: aim for >= 16 units per CTA slot
    const int64_t target = (int64_t)16 * 2 * e->sms;
    const int64_t base_units = (int64_t)p.Qb * p.jchunk;
    int64_t chunks = (target + base_units - 1) / base_units;
    if (chunks < 1) chunks = 1;
    if (chunks > e->tiles) chunks = e->tiles;
    int64_t tpu = (e->tiles + chunks - 1) / chunks;
    if (tpu < 4 && e->tiles >= 4) tpu = 4;  // amortise the direction-block load
    p.tpu = (int)tpu;
    p.chunks = (int)((e->tiles + tpu - 1) / tpu);
    return p;
}

int ensure_ws(rrs_engine* e, const Plan& p, int notion) {
    const size_t Qb = p.Qb, d = e->d;
    CK(e->zq.ensure(Qb * d * 4));
    CK(e->u64.ensure(Qb * p.m * d * 8));
    CK(e->u32.ensure(Qb * p.mpad * (p.tcf ? (size_t)tcf_dp(e->d) : d) * 4));
    CK(e->pole.ensure(Qb * d * 8));
    CK(e->reflv.ensure(Qb * d * 8));
    CK(e->reflmode.ensure(Qb * 4));
    CK(e->dmin.ensure(Qb * 8));
    CK(e->bestcnt.ensure(Qb * 8));
    CK(e->uop.ensure(p.tcf   ? Qb * (size_t)p.nb8 * tcf_block_bytes(e->d)
                     : (p.tc || p.tcws || p.tcst) ? Qb * (size_t)p.nb8 * tc_block_bytes(e->d)
                     : p.tcs ? Qb * (size_t)p.nb8 * tc6_block_bytes(e->d)
                             : 16));
    if (notion == RRS_HALFSPACE) {
        CK(e->counts.ensure(Qb * p.mpad * 2 * 4));
        CK(e->depths.ensure(8));
        if (p.tcp) {
            CK(e->shift.ensure(Qb * p.m * 8));
            CK(e->coin.ensure(Qb * TCP_COIN_MAX * 4));
            CK(e->coin_n.ensure(Qb * 4));
            CK(e->c0.ensure(Qb * 8));
            CK(e->zero_d.ensure(d * 8));  // (ensure keeps headroom: clear all d entries every time)
            CK(cudaMemsetAsync(e->zero_d.p, 0, d * 8, e->stream));
        }
    } else {
        CK(e->counts.ensure(8));
        CK(e->depths.ensure(Qb * p.m * 8));
        CK(e->y.ensure(Qb * (size_t)p.jchunk * BN * e->n * 4));
        CK(e->shift.ensure(Qb * p.m * 8));
        CK(e->zq0.ensure(Qb * d * 4));
        CK(cudaMemsetAsync(e->zq0.p, 0, Qb * d * 4, e->stream));
    }
    return RRS_OK;
}

ContractArgs contract_args(rrs_engine* e, const Plan& p, int Qb, int jb0, int jbn) {
    ContractArgs c{};
    c.xb = e->xb.as<float>();
    c.u32 = e->u32.as<float>();
    c.zq = e->zq.as<float>();
    c.counts = e->counts.as<int>();
    c.y = e->y.as<float>();
    c.n = e->n;
    c.tiles = e->tiles;
    c.d = e->d;
    c.Qb = Qb;
    c.MB = p.MB;
    c.jb0 = jb0;
    c.jbn = jbn;
    c.m = p.m;
    c.tiles_per_unit = p.tpu;
    c.chunks = p.chunks;
    return c;
}

// pre-split point operand k (0: x for the counts, 1: x - m for the centred store),
// built once per dataset from the tile-blocked FP32 copy and its row maxima
int ensure_presplit(rrs_engine* e, int k) {
    if (e->xps_ok[k]) return RRS_OK;
    CK(e->xps[k].ensure((size_t)e->tiles * tc_block_bytes(e->d)));
    CK(e->pinv[k].ensure((size_t)e->tiles * BM * 4));
    CK(launch_presplit(k ? e->xcb.as<float>() : e->xb.as<float>(), k ? e->xcmax.as<float>() : e->xmax.as<float>(),
                       e->n, e->d, e->tiles, e->xps[k].as<unsigned char>(), e->pinv[k].as<float>(), e->stream));
    e->stats.kernel_launches++;
    e->xps_ok[k] = true;
    return RRS_OK;
}

int contract_halfspace(rrs_engine* e, const Plan& p, int Qb, const double* zdev, const int* done, bool use_tcp) {
    if (p.wide) {
        Contract64Args c{};
        c.x64 = e->x64.as<double>();
        c.c = zdev;
        c.c_stride = e->d;
        c.u64 = e->u64.as<double>();
        c.counts = e->counts.as<int>();
        c.n = e->n;
        c.d = e->d;
        c.m = p.m;
        c.mpad = p.mpad;
        c.jbase = 0;
        c.jcount = p.m;
        c.Qb = Qb;
        c.done = done;
        CK(launch_contract64(c, false, e->stream));
    } else if (p.tcf) {
        TcfArgs t{};
        t.xb = e->xb.as<float>();
        t.zq = e->zq.as<float>();
        t.uop = e->uop.as<unsigned char>();
        t.u32r = e->u32.as<float>();
        t.counts = e->counts.as<int>();
        t.n = e->n;
        t.tiles = e->tiles;
        t.d = e->d;
        t.Qb = Qb;
        t.NB = p.nb8;
        t.m = p.m;
        t.mpad = p.mpad;
        CK(launch_contract_tcf(t, e->sms, e->stream));
        e->stats.tensor_contract_launches++;
    } else if (p.tc) {
        TcArgs t{};
        t.xb = e->xb.as<float>();
        t.zq = e->zq.as<float>();
        t.uop = e->uop.as<unsigned char>();
        t.counts = e->counts.as<int>();
        t.n = e->n;
        t.tiles = e->tiles;
        t.d = e->d;
        t.Qb = Qb;
        t.NB = p.nb8;
        t.m = p.m;
        t.mpad = p.mpad;
        t.xmax = e->xmax.as<float>();
        t.done = done;
        if (e->d > TC_SLICE && use_tcp) {
            // y = acc inv_i + <u_j, 0 - z>: the per-direction shift, then the pre-split kernel
            CK(launch_direction_shift(e->u64.as<double>(), e->zero_d.as<double>(), zdev, e->shift.as<double>(), Qb,
                                      p.m, e->d, e->stream));
            e->stats.kernel_launches++;
            if (int rc = ensure_presplit(e, 0)) return rc;
            t.xps = e->xps[0].as<unsigned char>();
            t.pinv = e->pinv[0].as<float>();
            t.dshift = e->shift.as<double>();
            t.coin = e->coin.as<int>();
            t.coin_n = e->coin_n.as<int>();
            CK(launch_contract_tcp(t, e->sms, e->stream));
        } else if (e->d > TC_SLICE) {
            CK(launch_contract_tcw(t, e->sms, e->stream));
        } else {
            CK(launch_contract_tc(t, e->sms, e->stream));
        }
        e->stats.tensor_contract_launches++;
    } else {
        ContractArgs c = contract_args(e, p, Qb, 0, p.MB);
        c.done = done;
        CK(launch_contract_count(c, e->stream));
    }
    return RRS_OK;
}

// y -> per-direction depths for the projection notions, chunked over direction
// blocks.  The store works in the centred frame (center.cu): y' = <u, x - m>
// from the centred copy and zero queries, the select adds <u, m - z> (FP64,
// from the FP64 queries zdev [Qb][d]) to the median.
int univariate_from_store(rrs_engine* e, const Plan& p, int Qb, int notion, const double* zdev) {
    {
        Timer t(e, 2);
        CK(launch_direction_shift(e->u64.as<double>(), e->center.as<double>(), zdev, e->shift.as<double>(), Qb, p.m,
                                  e->d, e->stream));
        e->stats.kernel_launches++;
    }
    for (int jb0 = 0; jb0 < p.MB; jb0 += p.jchunk) {
        const int jbn = (p.MB - jb0) < p.jchunk ? (p.MB - jb0) : p.jchunk;
        {
            Timer t(e, 1);
            if (p.tcws || p.tcst) {
                TcArgs t{};
                t.xb = e->xcb.as<float>();
                t.zq = e->zq0.as<float>();
                t.uop = e->uop.as<unsigned char>();
                t.n = e->n;
                t.tiles = e->tiles;
                t.d = e->d;
                t.Qb = Qb;
                t.NB = p.nb8;
                t.m = p.m;
                t.mpad = p.mpad;
                t.xmax = e->xcmax.as<float>();
                t.y = e->y.as<float>();
                t.jb0 = jb0;
                t.jbn = jbn;
                if (p.tcst) {
                    CK(launch_contract_tc_store(t, e->sms, e->stream));
                } else if (p.tcp) {
                    if (int rc = ensure_presplit(e, 1)) return rc;
                    t.xps = e->xps[1].as<unsigned char>();
                    t.pinv = e->pinv[1].as<float>();
                    CK(launch_contract_tcp_store(t, e->sms, e->stream));
                } else {
                    CK(launch_contract_tcw_store(t, e->sms, e->stream));
                }
                e->stats.tensor_contract_launches++;
            } else if (p.wide && !p.store64) {
                Contract64Args c{};
                c.x64 = e->x64.as<double>();
                c.c = e->center.as<double>();  // centred frame, the same m for every query
                c.c_stride = 0;
                c.u64 = e->u64.as<double>();
                c.y = e->y.as<float>();
                c.n = e->n;
                c.d = e->d;
                c.m = p.m;
                c.mpad = p.mpad;
                c.jbase = jb0 * BN;
                c.jcount = jbn * BN;
                c.Qb = Qb;
                CK(launch_contract64(c, true, e->stream));
            } else if (p.store64) {
                CK(launch_store64(e->xc64.as<double>(), e->u64.as<double>(), e->y.as<float>(), e->n, e->d, Qb, p.m,
                                  jb0 * BN, jbn * BN, e->stream));
            } else if (p.tcs) {
                TcsArgs c{};
                c.xb = e->xcb.as<float>();
                c.zq = e->zq0.as<float>();
                c.uop = e->uop.as<unsigned char>();
                c.y = e->y.as<float>();
                c.n = e->n;
                c.tiles = e->tiles;
                c.d = e->d;
                c.Qb = Qb;
                c.NB = p.nb8;
                c.m = p.m;
                c.jb0 = jb0;
                c.jbn = jbn;
                CK(launch_contract_tcs(c, e->sms, e->stream));
                e->stats.tensor_contract_launches++;
            } else {
                ContractArgs c = contract_args(e, p, Qb, jb0, jbn);
                c.xb = e->xcb.as<float>();
                c.zq = e->zq0.as<float>();
                CK(launch_contract_store(c, e->stream));
            }
            e->stats.kernel_launches++;
            e->stats.contract_launches++;
        }
        {
            Timer t(e, 2);
            SelectArgs s{};
            s.y = e->y.as<float>();
            s.depths = e->depths.as<double>();
            s.n = e->n;
            s.Qb = Qb;
            s.jcount = jbn * BN;
            s.j0 = jb0 * BN;
            s.m = p.m;
            s.notion = notion;
            s.shift = e->shift.as<double>();
            s.variant = e->select_path;
            s.fallbacks = e->fallbacks.as<unsigned>();
            CK(launch_select(s, e->stream));
            e->stats.kernel_launches++;
        }
    }
    return RRS_OK;
}

void reset_stats(rrs_engine* e) {
    e->stats = rrs_stats{};
    e->ev_used = 0;
    e->marks.clear();
    if (e->fallbacks.ensure(16) == cudaSuccess) cudaMemsetAsync(e->fallbacks.p, 0, 16, e->stream);
}

int collect_stats(rrs_engine* e) {
    if (e->fallbacks.p) {
        unsigned fb = 0;
        CK(cudaMemcpyAsync(&fb, e->fallbacks.p, sizeof(fb), cudaMemcpyDeviceToHost, e->stream));
        CK(cudaStreamSynchronize(e->stream));
        e->stats.select_rows_fallback = fb;
    }
    if (!e->timing) return RRS_OK;
    CK(cudaStreamSynchronize(e->stream));
    for (const auto& mk : e->marks) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, e->ev_pool[mk.a], e->ev_pool[mk.b]));
        switch (mk.stage) {
            case 0: e->stats.ms_generate += ms; break;
            case 1:
                e->stats.ms_contract += ms;
                e->stats.ms_contract_total += ms;
                break;
            case 2: e->stats.ms_univariate += ms; break;
            default: e->stats.ms_update += ms; break;
        }
    }
    e->marks.clear();
    e->ev_used = 0;
    return RRS_OK;
}

// Core device path: queries_dev (Q x d FP64) -> device outputs.
int run_batches(rrs_engine* e, const double* zdev, int64_t Q, int64_t q0, const rrs_config* cfg,
                const double* eps_host, double* depth, double* argmin, double* trace,
                int64_t* mincount) {
    const int r = cfg->refinements;
    const int m = (int)((cfg->total_directions + r - 1) / r);  // optimizer.py:64-66
    std::vector<double> eps(r);
    for (int l = 0; l < r; ++l)  // optimizer.py:175, HALF_PI = math.pi / 2.0
        eps[l] = eps_host ? eps_host[l] : (3.141592653589793 / 2.0) * std::pow(cfg->shrink, (double)l);
    const Plan p = make_plan(e, Q, m, cfg->notion);
    if (int rc = ensure_ws(e, p, cfg->notion)) return rc;
    if (cfg->notion == RRS_HALFSPACE)
        CK(cudaMemsetAsync(e->counts.p, 0, (size_t)p.Qb * p.mpad * 2 * 4, e->stream));
    const int d = e->d;
    // early exit (halfspace; not on the experimental 2-SM / filter kernels)
    const bool early = cfg->notion == RRS_HALFSPACE && cfg->early_exit != 0 && !p.tcf;
    const bool tcp_counts = cfg->notion == RRS_HALFSPACE && p.tc && p.tcp;
    int* done = nullptr;
    long long* c0 = nullptr;
    if (early) {
        CK(e->done.ensure((size_t)p.Qb * 4));
        CK(e->c0.ensure((size_t)p.Qb * 8));
        done = e->done.as<int>();
        c0 = e->c0.as<long long>();
    }
    std::vector<int> coin_n_host;
    for (int64_t b0 = 0; b0 < Q; b0 += p.Qb) {
        const int Qb = (int)((Q - b0) < p.Qb ? (Q - b0) : p.Qb);
        CK(launch_queries_to_f32(zdev + b0 * d, e->zq.as<float>(), (int64_t)Qb * d, e->stream));
        // the pre-split kernel excludes the rows coinciding with each query by index; a
        // query with more than TCP_COIN_MAX of them sends its batch to the converter kernel
        bool use_tcp = false;
        if (tcp_counts) {
            CK(launch_coincide_list32(e->xb.as<float>(), e->zq.as<float>(), e->n, d, e->tiles, Qb,
                                      e->c0.as<long long>(), e->coin.as<int>(), e->coin_n.as<int>(), e->stream));
            e->stats.kernel_launches += 1;
            coin_n_host.resize((size_t)Qb);
            CK(cudaMemcpyAsync(coin_n_host.data(), e->coin_n.p, (size_t)Qb * 4, cudaMemcpyDeviceToHost, e->stream));
            CK(cudaStreamSynchronize(e->stream));
            use_tcp = true;
            for (int v : coin_n_host) use_tcp = use_tcp && v <= TCP_COIN_MAX;
        }
        if (early) {
            CK(cudaMemsetAsync(done, 0, (size_t)Qb * 4, e->stream));
            if (tcp_counts) {
                // c0 came with the lists (the same FP32 equality as launch_coincide_count32)
            } else if (p.wide) {
                CK(launch_coincide_count64(e->x64.as<double>(), zdev + b0 * d, e->n, d, Qb, c0, e->stream));
            } else {
                CK(launch_coincide_count32(e->xb.as<float>(), e->zq.as<float>(), e->n, d, e->tiles, Qb, c0, e->stream));
            }
            e->stats.kernel_launches += 1;
        }
        StateArgs s{e->pole.as<double>(), e->reflv.as<double>(), e->reflmode.as<int>(),
                    e->dmin.as<double>(), e->bestcnt.as<long long>(), (long long)e->n, Qb, d};
        CK(launch_state_init(s, e->stream));
        e->stats.kernel_launches += 2;
        for (int l = 0; l < r; ++l) {
            {
                Timer t(e, 0);
                GenArgs g{};
                g.pole = e->pole.as<double>();
                g.refl_mode = e->reflmode.as<int>();
                g.refl_v = e->reflv.as<double>();
                g.u64 = e->u64.as<double>();
                g.u32 = (p.tc || p.tcs || p.tcws || p.tcst) ? nullptr : e->u32.as<float>();  // tensor: uop only
                g.seed = cfg->seed;
                g.q0 = q0 + b0;
                g.refinement = (uint32_t)l;
                g.eps = eps[l];
                g.Qb = Qb;
                g.m = m;
                g.mpad = p.mpad;
                g.d = d;
                g.uop = (p.tc || p.tcws || p.tcst) ? e->uop.as<unsigned char>() : nullptr;
                g.uop_mode = p.tcf ? 1 : 0;
                g.u32r = p.tcf ? e->u32.as<float>() : nullptr;
                g.NB = p.nb8;
                g.done = done;
                CK(launch_cap_generate(g, e->stream));
                e->stats.kernel_launches++;
                if (p.tcs) {  // six-product operand of the projection store from the FP64 directions
                    CK(launch_pack_tc6_operand(e->u64.as<double>(), e->uop.as<unsigned char>(), Qb, m, p.nb8, d,
                                               e->stream));
                    e->stats.kernel_launches++;
                }
            }
            if (cfg->notion == RRS_HALFSPACE) {
                Timer t(e, 1);
                if (int rc = contract_halfspace(e, p, Qb, zdev + b0 * d, done, use_tcp)) return rc;
                e->stats.kernel_launches++;
                e->stats.contract_launches++;
            } else {
                if (int rc = univariate_from_store(e, p, Qb, cfg->notion, zdev + b0 * d)) return rc;
            }
            {
                Timer t(e, 3);
                UpdateArgs u{};
                u.counts = e->counts.as<int>();
                u.depths = e->depths.as<double>();
                u.u64 = e->u64.as<double>();
                u.pole = e->pole.as<double>();
                u.refl_v = e->reflv.as<double>();
                u.refl_mode = e->reflmode.as<int>();
                u.dmin = e->dmin.as<double>();
                u.best_count = e->bestcnt.as<long long>();
                u.trace = trace ? trace + (size_t)b0 * r * (2 + d) : nullptr;
                u.n = e->n;
                u.eps = eps[l];
                u.Qb = Qb;
                u.m = m;
                u.mpad = p.mpad;
                u.d = d;
                u.r = r;
                u.refinement = l;
                u.notion = cfg->notion;
                u.done = done;
                u.c0 = c0;
                CK(launch_update(u, e->stream));
                e->stats.kernel_launches++;
            }
        }
        FinalArgs f{e->pole.as<double>(), e->dmin.as<double>(), e->bestcnt.as<long long>(),
                    depth + b0, argmin ? argmin + (size_t)b0 * d : nullptr,
                    mincount ? (long long*)mincount + b0 : nullptr, Qb, d};
        CK(launch_finalize(f, e->stream));
        e->stats.kernel_launches++;
    }
    return RRS_OK;
}

// finite and inside the FP32 contraction range, like the dataset (the queries
// are cast to FP32 for x - z; an out-of-range or NaN query would otherwise
// count as all-tie rows and give silently wrong depths)
int validate_host_queries(const double* z, int64_t count, int d) {
    for (int64_t i = 0; i < count; ++i) {
        const double v = z[i];
        if (!std::isfinite(v))
            return fail(RRS_ERR_INVALID, "query " + std::to_string(i / d) + " contains non-finite entries");
        if (std::fabs(v) > 1e38)
            return fail(RRS_ERR_INVALID, "query " + std::to_string(i / d) +
                                             " exceeds the FP32 contraction range (|z| > 1e38)");
    }
    return RRS_OK;
}

int check_dataset(const rrs_engine* e) {
    if (!e) return fail(RRS_ERR_INVALID, "engine is null");
    if (e->n < 1 || e->d < 1) return fail(RRS_ERR_STATE, "no dataset set");
    return RRS_OK;
}

}  // namespace

extern "C" {

int rrs_abi_version(void) { return RRS_ABI_VERSION; }

const char* rrs_last_error(void) { return g_err.c_str(); }

int rrs_device_count(int32_t* count) {
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) {
        cudaGetLastError();
        c = 0;
    }
    if (count) *count = c;
    return RRS_OK;
}

int rrs_engine_create(int32_t device, rrs_engine** out) {
    if (!out) return fail(RRS_ERR_INVALID, "out is null");
    *out = nullptr;
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess || c == 0) {
        cudaGetLastError();
        return fail(RRS_ERR_CUDA, "no CUDA device visible (the B200 path has no CPU fallback)");
    }
    if (device < 0 || device >= c) return fail(RRS_ERR_INVALID, "device index out of range");
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return fail(RRS_ERR_CUDA, std::string("device is not sm_100 (found ") + prop.name + ")");
    rrs_engine* e = new rrs_engine();
    e->device = device;
    e->sms = sm_count_of(device);
    cudaError_t ce = cudaSetDevice(device);
    if (ce == cudaSuccess) ce = cudaStreamCreateWithFlags(&e->own, cudaStreamNonBlocking);
    if (ce != cudaSuccess) {
        delete e;
        return fail(RRS_ERR_CUDA, std::string("stream create: ") + cudaGetErrorString(ce));
    }
    e->stream = e->own;
    // query-batching workspace: a quarter of the free HBM, between 1 and 32 GiB
    // (32 GiB on an idle B200: fewer, larger store / select launches for the
    // projection notions; rrs_engine_set_workspace_limit overrides it)
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
        int64_t ws = (int64_t)(free_b / 4);
        if (ws > (32ll << 30)) ws = 32ll << 30;
        if (ws < (1ll << 30)) ws = 1ll << 30;
        e->ws_limit = ws;
    } else {
        cudaGetLastError();
    }
    *out = e;
    return RRS_OK;
}

int rrs_engine_destroy(rrs_engine* e) {
    if (!e) return RRS_OK;
    cudaSetDevice(e->device);
    cudaStreamSynchronize(e->stream);
    for (DevBuf* b : {&e->xb, &e->xmax, &e->zq, &e->u64, &e->u32, &e->uop, &e->counts, &e->depths, &e->y, &e->pole,
                      &e->reflv, &e->reflmode, &e->dmin, &e->bestcnt, &e->tmp_in, &e->tmp_out0,
                      &e->tmp_out1, &e->tmp_out2, &e->tmp_out3, &e->center, &e->xcb, &e->xc64, &e->zq0,
                      &e->shift, &e->fallbacks, &e->x64, &e->done, &e->c0, &e->xcmax, &e->xps[0], &e->xps[1],
                      &e->pinv[0], &e->pinv[1], &e->coin, &e->coin_n, &e->zero_d, &e->qflag})
        b->release();
    for (auto ev : e->ev_pool) cudaEventDestroy(ev);
    if (e->own) cudaStreamDestroy(e->own);
    delete e;
    return RRS_OK;
}

int rrs_engine_set_stream(rrs_engine* e, void* stream) {
    if (!e) return fail(RRS_ERR_INVALID, "engine is null");
    e->stream = stream ? static_cast<cudaStream_t>(stream) : e->own;
    return RRS_OK;
}

int rrs_engine_synchronize(rrs_engine* e) {
    if (!e) return fail(RRS_ERR_INVALID, "engine is null");
    if (int rc = set_device(e)) return rc;
    CK(cudaStreamSynchronize(e->stream));
    return RRS_OK;
}

int rrs_engine_set_workspace_limit(rrs_engine* e, int64_t bytes) {
    if (!e) return fail(RRS_ERR_INVALID, "engine is null");
    if (bytes < (1 << 20)) return fail(RRS_ERR_INVALID, "workspace limit below 1 MiB");
    e->ws_limit = bytes;
    return RRS_OK;
}

int rrs_engine_set_contract_path(rrs_engine* e, int32_t path) {
    if (!e) return fail(RRS_ERR_INVALID, "engine is null");
    if (path < 0 || path > 6 || path == 3)
        return fail(RRS_ERR_INVALID,
                    "contract path must be 0 (auto), 1 (FFMA), 2 (tensor), 4 (filter and refine), 5 (three-term "
                    "tensor projection store) or 6 (tensor with in-kernel converters above d = 64); 3 (the 2-SM "
                    "split kernel) was removed");
    e->contract_path = path;
    return RRS_OK;
}

int rrs_host_alloc(int64_t bytes, void** out) {
    if (!out) return fail(RRS_ERR_INVALID, "out is null");
    *out = nullptr;
    if (bytes < 0) return fail(RRS_ERR_INVALID, "negative size");
    if (bytes == 0) bytes = 16;
    cudaError_t ce = cudaHostAlloc(out, (size_t)bytes, cudaHostAllocPortable);
    if (ce != cudaSuccess) {
        cudaGetLastError();
        *out = nullptr;
        return fail(ce == cudaErrorMemoryAllocation ? RRS_ERR_NOMEM : RRS_ERR_CUDA,
                    std::string("cudaHostAlloc: ") + cudaGetErrorString(ce));
    }
    return RRS_OK;
}

int rrs_host_free(void* p) {
    if (p) CK(cudaFreeHost(p));
    return RRS_OK;
}

int rrs_engine_set_select_path(rrs_engine* e, int32_t path) {
    if (!e) return fail(RRS_ERR_INVALID, "engine is null");
    if (path != 0 && path != 2 && path != 3)
        return fail(RRS_ERR_INVALID, "select path must be 0 (auto), 2 (radix select v2) or 3 (v3, 1024 threads)");
    e->select_path = path;
    return RRS_OK;
}

int rrs_engine_enable_timing(rrs_engine* e, int32_t on) {
    if (!e) return fail(RRS_ERR_INVALID, "engine is null");
    e->timing = on != 0;
    return RRS_OK;
}

int rrs_engine_stats(rrs_engine* e, rrs_stats* out) {
    if (!e || !out) return fail(RRS_ERR_INVALID, "null argument");
    if (int rc = set_device(e)) return rc;
    if (int rc = collect_stats(e)) return rc;
    *out = e->stats;
    return RRS_OK;
}

// 0 ok, else the first violated rule: 1 non-finite entry, 2 |x| > 1e38
static int validate_device_dataset(rrs_engine* e, const double* xdev, int64_t count) {
    CK(e->tmp_out0.ensure(16));
    int* flag = e->tmp_out0.as<int>();
    CK(cudaMemsetAsync(flag, 0, sizeof(int), e->stream));
    CK(launch_validate_values(xdev, count, flag, e->stream));
    int h = 0;
    CK(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    if (h & 1) return fail(RRS_ERR_INVALID, "dataset contains non-finite entries");
    if (h & 2) return fail(RRS_ERR_INVALID, "dataset entries exceed the FP32 contraction range (|x| > 1e38)");
    return RRS_OK;
}

static int set_dataset_common(rrs_engine* e, const double* xdev, int64_t n, int32_t d) {
    if (d > MAX_D)
        return fail(RRS_ERR_INVALID, "dimension " + std::to_string(d) + " exceeds the supported maximum " +
                                         std::to_string(MAX_D));
    const int64_t tiles = (n + BM - 1) / BM;
    CK(e->xb.ensure((size_t)tiles * d * BM * 4));
    CK(launch_block_dataset(xdev, e->xb.as<float>(), n, d, tiles, e->stream));
    CK(e->center.ensure((size_t)d * 8));
    CK(e->tmp_out1.ensure((size_t)d * 8));
    CK(launch_center_sample(xdev, n, d, e->center.as<double>(), e->tmp_out1.as<double>(), e->stream));
    {
        std::vector<double> iqr((size_t)d);
        CK(cudaMemcpyAsync(iqr.data(), e->tmp_out1.p, (size_t)d * 8, cudaMemcpyDeviceToHost, e->stream));
        CK(cudaStreamSynchronize(e->stream));
        double lo = 0.0, hi = 0.0;
        for (double v : iqr)
            if (v > 0.0) {
                lo = (lo == 0.0 || v < lo) ? v : lo;
                hi = v > hi ? v : hi;
            }
        e->col_ratio = lo > 0.0 ? hi / lo : 1.0;
    }
    CK(e->xcb.ensure((size_t)tiles * d * BM * 4));
    CK(launch_block_centered(xdev, e->center.as<double>(), e->xcb.as<float>(), n, d, tiles, e->stream));
    if (d > TC_SLICE && d <= TC_MAX_D) {
        CK(e->xcmax.ensure((size_t)tiles * BM * 4));
        CK(launch_row_absmax(e->xcb.as<float>(), e->xcmax.as<float>(), d, tiles, e->stream));
    }
    if (n < STORE64_N) {
        CK(e->xc64.ensure((size_t)n * d * 8));
        CK(launch_center_copy64(xdev, e->center.as<double>(), e->xc64.as<double>(), n, d, e->stream));
    }
    if (d > TC_MAX_D) {
        CK(e->x64.ensure((size_t)n * d * 8));
        CK(cudaMemcpyAsync(e->x64.p, xdev, (size_t)n * d * 8, cudaMemcpyDeviceToDevice, e->stream));
    }
    if (d > TC_SLICE) {
        CK(e->xmax.ensure((size_t)tiles * BM * 4));
        CK(launch_row_absmax(e->xb.as<float>(), e->xmax.as<float>(), d, tiles, e->stream));
    }
    e->n = n;
    e->d = d;
    e->tiles = tiles;
    e->xps_ok[0] = e->xps_ok[1] = false;
    return RRS_OK;
}

int rrs_set_dataset_host(rrs_engine* e, const double* x, int64_t n, int32_t d) {
    if (!e || !x) return fail(RRS_ERR_INVALID, "null argument");
    if (n < 1 || d < 1) return fail(RRS_ERR_INVALID, "dataset must be a non-empty 2-D matrix");
    if (int rc = set_device(e)) return rc;
    CK(e->tmp_in.ensure((size_t)n * d * 8));
    CK(cudaMemcpyAsync(e->tmp_in.p, x, (size_t)n * d * 8, cudaMemcpyHostToDevice, e->stream));
    // finiteness / FP32-range check on the device copy (the engine's dataset is untouched on failure)
    if (int rc = validate_device_dataset(e, e->tmp_in.as<double>(), n * (int64_t)d)) return rc;
    int rc = set_dataset_common(e, e->tmp_in.as<double>(), n, d);
    if (rc) return rc;
    CK(cudaStreamSynchronize(e->stream));
    return RRS_OK;
}

int rrs_set_dataset_device(rrs_engine* e, const double* x_dev, int64_t n, int32_t d) {
    if (!e || !x_dev) return fail(RRS_ERR_INVALID, "null argument");
    if (n < 1 || d < 1) return fail(RRS_ERR_INVALID, "dataset must be a non-empty 2-D matrix");
    if (int rc = set_device(e)) return rc;
    if (int rc = validate_device_dataset(e, x_dev, n * (int64_t)d)) return rc;
    return set_dataset_common(e, x_dev, n, d);
}

int rrs_depth_batch_device(rrs_engine* e, const double* queries_dev, int64_t Q, int64_t q0,
                           const rrs_config* cfg, const double* eps, double* depth_dev,
                           double* argmin_dev, double* trace_dev, int64_t* min_count_dev) {
    if (int rc = check_dataset(e)) return rc;
    if (int rc = validate_cfg(cfg)) return rc;
    if (Q < 0) return fail(RRS_ERR_INVALID, "negative query count");
    if (Q == 0) return RRS_OK;
    if (!queries_dev || !depth_dev) return fail(RRS_ERR_INVALID, "null argument");
    if (int rc = set_device(e)) return rc;
    // the queries are validated on the device; the flag is read back after the
    // batch is enqueued (one synchronisation at the end of the call instead of a
    // host round trip before the first kernel), and a bad query fails the call
    CK(e->qflag.ensure(16));
    int* flag = e->qflag.as<int>();
    CK(cudaMemsetAsync(flag, 0, sizeof(int), e->stream));
    CK(launch_validate_values(queries_dev, Q * (int64_t)e->d, flag, e->stream));
    reset_stats(e);
    const int rc = run_batches(e, queries_dev, Q, q0, cfg, eps, depth_dev, argmin_dev, trace_dev, min_count_dev);
    int h = 0;
    CK(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    if (h & 1) return fail(RRS_ERR_INVALID, "queries contain non-finite entries");
    if (h & 2) return fail(RRS_ERR_INVALID, "queries exceed the FP32 contraction range (|z| > 1e38)");
    return rc;
}

int rrs_depth_batch_host(rrs_engine* e, const double* queries, int64_t Q, int64_t q0,
                         const rrs_config* cfg, const double* eps, double* depth, double* argmin,
                         double* trace, int64_t* min_count) {
    if (int rc = check_dataset(e)) return rc;
    if (int rc = validate_cfg(cfg)) return rc;
    if (Q < 0) return fail(RRS_ERR_INVALID, "negative query count");
    if (Q == 0) return RRS_OK;
    if (!queries || !depth) return fail(RRS_ERR_INVALID, "null argument");
    if (int rc = validate_host_queries(queries, Q * (int64_t)e->d, e->d)) return rc;
    if (int rc = set_device(e)) return rc;
    reset_stats(e);
    const int d = e->d, r = cfg->refinements;
    const size_t zb = (size_t)Q * d * 8;
    CK(e->tmp_in.ensure(zb));
    CK(e->tmp_out0.ensure((size_t)Q * 8));
    CK(e->tmp_out1.ensure((size_t)Q * d * 8));
    if (trace) CK(e->tmp_out2.ensure((size_t)Q * r * (2 + d) * 8));
    CK(e->tmp_out3.ensure((size_t)Q * 8));
    CK(cudaMemcpyAsync(e->tmp_in.p, queries, zb, cudaMemcpyHostToDevice, e->stream));
    int rc = run_batches(e, e->tmp_in.as<double>(), Q, q0, cfg, eps, e->tmp_out0.as<double>(),
                         e->tmp_out1.as<double>(), trace ? e->tmp_out2.as<double>() : nullptr,
                         e->tmp_out3.as<int64_t>());
    if (rc) return rc;
    CK(cudaMemcpyAsync(depth, e->tmp_out0.p, (size_t)Q * 8, cudaMemcpyDeviceToHost, e->stream));
    if (argmin)
        CK(cudaMemcpyAsync(argmin, e->tmp_out1.p, (size_t)Q * d * 8, cudaMemcpyDeviceToHost, e->stream));
    if (trace)
        CK(cudaMemcpyAsync(trace, e->tmp_out2.p, (size_t)Q * r * (2 + d) * 8, cudaMemcpyDeviceToHost,
                           e->stream));
    if (min_count)
        CK(cudaMemcpyAsync(min_count, e->tmp_out3.p, (size_t)Q * 8, cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    return RRS_OK;
}

int rrs_evaluate_directions_host(rrs_engine* e, const double* z, const double* U, int32_t m,
                                 int32_t notion, double* out, int64_t* cle, int64_t* cge) {
    if (int rc = check_dataset(e)) return rc;
    if (!z || !U || !out) return fail(RRS_ERR_INVALID, "null argument");
    if (m < 1) return fail(RRS_ERR_INVALID, "batch size must be >= 1");
    if (notion < 0 || notion > 2) return fail(RRS_ERR_INVALID, "unknown depth notion");
    if (int rc = validate_host_queries(z, e->d, e->d)) return rc;
    if (int rc = set_device(e)) return rc;
    reset_stats(e);
    const int d = e->d;
    Plan p = make_plan(e, 1, m, notion);
    if (int rc = ensure_ws(e, p, notion)) return rc;
    CK(e->tmp_in.ensure((size_t)d * 8));
    CK(cudaMemcpyAsync(e->u64.p, U, (size_t)m * d * 8, cudaMemcpyHostToDevice, e->stream));
    CK(cudaMemcpyAsync(e->tmp_in.p, z, (size_t)d * 8, cudaMemcpyHostToDevice, e->stream));
    CK(launch_queries_to_f32(e->tmp_in.as<double>(), e->zq.as<float>(), d, e->stream));
    if (p.tcf)
        CK(launch_pack_tcf_operand(e->u64.as<double>(), e->uop.as<unsigned char>(), e->u32.as<float>(), 1, m, p.nb8,
                                   p.mpad, d, e->stream));
    else
        CK(launch_pack_directions(e->u64.as<double>(), e->u32.as<float>(), 1, m, p.mpad, d, e->stream));
    if (p.tc && !p.tcf) CK(launch_pack_tc_operand(e->u64.as<double>(), e->uop.as<unsigned char>(), 1, m, p.nb8, d, e->stream));
    if (p.tcs) CK(launch_pack_tc6_operand(e->u64.as<double>(), e->uop.as<unsigned char>(), 1, m, p.nb8, d, e->stream));
    if (p.tcws || p.tcst)
        CK(launch_pack_tc_operand(e->u64.as<double>(), e->uop.as<unsigned char>(), 1, m, p.nb8, d, e->stream));
    if (notion == RRS_HALFSPACE) {
        CK(cudaMemsetAsync(e->counts.p, 0, (size_t)p.mpad * 2 * 4, e->stream));
        bool use_tcp = false;
        if (p.tc && p.tcp) {
            CK(launch_coincide_list32(e->xb.as<float>(), e->zq.as<float>(), e->n, d, e->tiles, 1,
                                      e->c0.as<long long>(), e->coin.as<int>(), e->coin_n.as<int>(), e->stream));
            int cn = 0;
            CK(cudaMemcpyAsync(&cn, e->coin_n.p, 4, cudaMemcpyDeviceToHost, e->stream));
            CK(cudaStreamSynchronize(e->stream));
            use_tcp = cn <= TCP_COIN_MAX;
        }
        if (int rc = contract_halfspace(e, p, 1, e->tmp_in.as<double>(), nullptr, use_tcp)) return rc;
        std::vector<int> cnt((size_t)p.mpad * 2);
        CK(cudaMemcpyAsync(cnt.data(), e->counts.p, cnt.size() * 4, cudaMemcpyDeviceToHost, e->stream));
        CK(cudaStreamSynchronize(e->stream));
        const int64_t n = e->n;
        for (int j = 0; j < m; ++j) {
            const int64_t lt = cnt[2 * j], gt = cnt[2 * j + 1];
            const int64_t le = n - gt, ge = n - lt;  // ties (y == 0) on both sides
            if (cle) cle[j] = le;
            if (cge) cge[j] = ge;
            out[j] = (double)(le < ge ? le : ge) / (double)n;  // _kernels.pyx:288-289
        }
        return RRS_OK;
    }
    if (int rc = univariate_from_store(e, p, 1, notion, e->tmp_in.as<double>())) return rc;
    CK(cudaMemcpyAsync(out, e->depths.p, (size_t)m * 8, cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    return RRS_OK;
}

int rrs_cap_directions_host(rrs_engine* e, const double* pole, int32_t d, double eps, int32_t m,
                            uint64_t seed, uint32_t refinement, uint32_t query, double* U) {
    return rrs_cap_directions_at_host(e, pole, d, eps, m, seed, refinement, query, 0u, U);
}

int rrs_cap_directions_at_host(rrs_engine* e, const double* pole, int32_t d, double eps, int32_t m,
                               uint64_t seed, uint32_t refinement, uint32_t query, uint32_t index_base,
                               double* U) {
    if (!e || !pole || !U) return fail(RRS_ERR_INVALID, "null argument");
    if (m < 1) return fail(RRS_ERR_INVALID, "batch size must be >= 1");
    if (d < 1 || d > GEN_MAX_D) return fail(RRS_ERR_INVALID, "dimension out of range");
    if (!(eps > 0.0 && eps <= 3.141592653589793 / 2 + 1e-15))
        return fail(RRS_ERR_INVALID, "cap half-angle must lie in (0, pi/2]");
    if (int rc = set_device(e)) return rc;
    // reflect_to_pole vector, directions.py:150-164 (same arithmetic as update_kernel)
    std::vector<double> v(d, 0.0);
    int mode = 0;
    const double p1 = pole[0];
    if (1.0 - p1 < 1e-12) mode = 0;
    else if (1.0 + p1 < 1e-12) mode = 1;
    else {
        mode = 2;
        for (int c = 0; c < d; ++c) v[c] = -pole[c];
        v[0] += 1.0;
        double ss = 0.0;
        for (int c = 0; c < d; ++c) ss += v[c] * v[c];
        const double vn = std::sqrt(ss);
        for (int c = 0; c < d; ++c) v[c] /= vn;
    }
    const int mpad = ((m + BN - 1) / BN) * BN;
    DevBuf pb, vb, mb, ub, u32b;
    CK(pb.ensure((size_t)d * 8));
    CK(vb.ensure((size_t)d * 8));
    CK(mb.ensure(4));
    CK(ub.ensure((size_t)m * d * 8));
    CK(u32b.ensure((size_t)mpad * d * 4));
    CK(cudaMemcpyAsync(pb.p, pole, (size_t)d * 8, cudaMemcpyHostToDevice, e->stream));
    CK(cudaMemcpyAsync(vb.p, v.data(), (size_t)d * 8, cudaMemcpyHostToDevice, e->stream));
    CK(cudaMemcpyAsync(mb.p, &mode, 4, cudaMemcpyHostToDevice, e->stream));
    GenArgs g{};
    g.pole = pb.as<double>();
    g.refl_mode = mb.as<int>();
    g.refl_v = vb.as<double>();
    g.u64 = ub.as<double>();
    g.u32 = u32b.as<float>();
    g.seed = seed;
    g.jbase = index_base;
    g.q0 = query;
    g.refinement = refinement;
    g.eps = eps;
    g.Qb = 1;
    g.m = m;
    g.mpad = mpad;
    g.d = d;
    CK(launch_cap_generate(g, e->stream));
    CK(cudaMemcpyAsync(U, ub.p, (size_t)m * d * 8, cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    for (DevBuf* b : {&pb, &vb, &mb, &ub, &u32b}) b->release();
    return RRS_OK;
}

int rrs_unit_rows_host(rrs_engine* e, uint64_t seed, uint32_t refinement, uint32_t query, int32_t m,
                       int32_t dim, uint32_t v_base, uint32_t index_base, double* U) {
    if (!e || !U) return fail(RRS_ERR_INVALID, "null argument");
    if (m < 1) return fail(RRS_ERR_INVALID, "batch size must be >= 1");
    if (dim < 1) return fail(RRS_ERR_INVALID, "dimension must be >= 1");
    if (int rc = set_device(e)) return rc;
    DevBuf ub;
    CK(ub.ensure((size_t)m * dim * 8));
    CK(launch_unit_rows(seed, refinement, query, m, dim, v_base, index_base, ub.as<double>(), e->stream));
    CK(cudaMemcpyAsync(U, ub.p, (size_t)m * dim * 8, cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    ub.release();
    return RRS_OK;
}

int rrs_stream_values_host(rrs_engine* e, uint64_t seed, uint32_t refinement, uint32_t query, uint32_t index,
                           uint32_t offset, int64_t count, int32_t normal, double* out) {
    if (!e || (!out && count > 0)) return fail(RRS_ERR_INVALID, "null argument");
    if (count < 0) return fail(RRS_ERR_INVALID, "negative count");
    if (count == 0) return RRS_OK;
    if (int rc = set_device(e)) return rc;
    DevBuf ob;
    CK(ob.ensure((size_t)count * 8));
    CK(launch_stream_values(seed, refinement, query, index, offset, count, normal ? 1 : 0, ob.as<double>(),
                            e->stream));
    CK(cudaMemcpyAsync(out, ob.p, (size_t)count * 8, cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    ob.release();
    return RRS_OK;
}

int rrs_project_host(rrs_engine* e, const double* x, int64_t n, int32_t d, const double* U, int32_t m,
                     double* out) {
    if (!e || !x || !U || !out) return fail(RRS_ERR_INVALID, "null argument");
    if (n < 1 || d < 1 || m < 1) return fail(RRS_ERR_INVALID, "empty projection");
    if (int rc = set_device(e)) return rc;
    DevBuf xb, ub, ob;
    CK(xb.ensure((size_t)n * d * 8));
    CK(ub.ensure((size_t)m * d * 8));
    if (ob.ensure((size_t)m * n * 8) != cudaSuccess) {
        cudaGetLastError();
        return fail(RRS_ERR_NOMEM, "projection matrix does not fit in device memory");
    }
    CK(cudaMemcpyAsync(xb.p, x, (size_t)n * d * 8, cudaMemcpyHostToDevice, e->stream));
    CK(cudaMemcpyAsync(ub.p, U, (size_t)m * d * 8, cudaMemcpyHostToDevice, e->stream));
    CK(launch_proj64(xb.as<double>(), ub.as<double>(), ob.as<double>(), n, m, d, e->stream));
    CK(cudaMemcpyAsync(out, ob.p, (size_t)m * n * 8, cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    for (DevBuf* b : {&xb, &ub, &ob}) b->release();
    return RRS_OK;
}

int rrs_depth_of_projections_host(rrs_engine* e, int32_t notion, const double* px, int32_t m, int64_t n,
                                  const double* pz, double* out) {
    if (!e || !px || !pz || !out) return fail(RRS_ERR_INVALID, "null argument");
    if (notion < 0 || notion > 2) return fail(RRS_ERR_INVALID, "unknown depth notion");
    if (n < 1) return fail(RRS_ERR_INVALID, "empty projection");
    if (m < 1) return RRS_OK;
    if (int rc = set_device(e)) return rc;
    DevBuf pb, zb, ob;
    if (pb.ensure((size_t)m * n * 8) != cudaSuccess) {
        cudaGetLastError();
        return fail(RRS_ERR_NOMEM, "projection matrix does not fit in device memory");
    }
    CK(zb.ensure((size_t)m * 8));
    CK(ob.ensure((size_t)m * 8));
    CK(cudaMemcpyAsync(pb.p, px, (size_t)m * n * 8, cudaMemcpyHostToDevice, e->stream));
    CK(cudaMemcpyAsync(zb.p, pz, (size_t)m * 8, cudaMemcpyHostToDevice, e->stream));
    CK(launch_span_depth64(pb.as<double>(), zb.as<double>(), ob.as<double>(), m, n, notion, e->stream));
    CK(cudaMemcpyAsync(out, ob.p, (size_t)m * 8, cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    for (DevBuf* b : {&pb, &zb, &ob}) b->release();
    return RRS_OK;
}

int rrs_philox4x32_host(rrs_engine* e, const uint32_t* ctr, int64_t N, uint32_t key0, uint32_t key1,
                        uint32_t* out) {
    if (!e || !ctr || !out) return fail(RRS_ERR_INVALID, "null argument");
    if (N < 0) return fail(RRS_ERR_INVALID, "negative count");
    if (N == 0) return RRS_OK;
    if (int rc = set_device(e)) return rc;
    DevBuf a, b;
    CK(a.ensure((size_t)N * 16));
    CK(b.ensure((size_t)N * 16));
    CK(cudaMemcpyAsync(a.p, ctr, (size_t)N * 16, cudaMemcpyHostToDevice, e->stream));
    CK(launch_philox_words(a.as<uint32_t>(), b.as<uint32_t>(), N, key0, key1, e->stream));
    CK(cudaMemcpyAsync(out, b.p, (size_t)N * 16, cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    a.release();
    b.release();
    return RRS_OK;
}

}  // extern "C"
