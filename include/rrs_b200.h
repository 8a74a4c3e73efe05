/*
 * rrs_b200.h -- C ABI of the B200-native Refined Random Search (RRS) depth
 * solver (paper_2506_08262_b200/_lib/librrs_b200.so, sm_100a).
 *
 * Drop-in boundary for the reference's hot path (depthforge 0.1.0,
 * /root/reference/pkg/src/depthforge).  Each entry point names the reference
 * interface it replaces.  Conventions:
 *   - plain pointers and sizes; no exceptions cross the ABI;
 *   - every entry returns an rrs_status (0 = OK); rrs_last_error() gives the
 *     message of the calling thread's last failure (reference messages kept:
 *     "need total_directions >= refinements >= 1", "query dimension ...");
 *   - *_host entry points take caller-owned HOST buffers and do the
 *     host<->device copies inside the call; *_device entry points take device
 *     pointers that stay resident and are stream-ordered on the engine stream;
 *   - one engine per device, not shared across host threads without external
 *     synchronisation (the reference's functions are pure);
 *   - there is no CPU fallback: without a CUDA device every call fails with
 *     RRS_ERR_CUDA.
 */
#ifndef RRS_B200_H
#define RRS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RRS_ABI_VERSION 3

typedef enum {
    RRS_OK = 0,
    RRS_ERR_INVALID = 1, /* ValueError in the reference                      */
    RRS_ERR_DIM = 2,     /* DimensionMismatch(ValueError), projection.py:23  */
    RRS_ERR_CUDA = 3,    /* no device / launch failure                       */
    RRS_ERR_NOMEM = 4,   /* MemoryError (_kernels.pyx:299-300)               */
    RRS_ERR_STATE = 5    /* e.g. no dataset set                              */
} rrs_status;

/* univariate.py:27 NOTIONS */
typedef enum { RRS_HALFSPACE = 0, RRS_PROJECTION = 1, RRS_ASYM_PROJECTION = 2 } rrs_notion;

/* optimizer.py:39 POLE_UPDATE_MODES */
typedef enum { RRS_PER_REFINEMENT = 0, RRS_PER_DIRECTION = 1 } rrs_pole_update;

/* optimizer.py:42-66 RrsConfig (ParallelConfig has no device meaning). */
typedef struct {
    int64_t total_directions; /* k = NRandom; m = ceil(k / r) per refinement  */
    int32_t refinements;      /* r = n_refinements                            */
    double shrink;            /* alpha = sphcap_shrink, in (0, 1)             */
    int32_t notion;           /* rrs_notion                                   */
    uint64_t seed;            /* seed mod 2^64 (philox.py:68-71)              */
    int32_t pole_update;      /* rrs_pole_update                              */
    int32_t early_exit;       /* halfspace: skip a query's remaining refinements
                                 once its best count equals the number of data
                                 rows coinciding with it (no direction can go
                                 strictly below: depth, argmin and trace are
                                 bitwise those of the full run).  0 = off (the
                                 reference's cost model), 1 = on.             */
} rrs_config;

typedef struct rrs_engine rrs_engine;

int rrs_abi_version(void);
const char* rrs_last_error(void);
/* Number of visible CUDA devices (0 when none). */
int rrs_device_count(int32_t* count);

/* Engine lifecycle.  One per device; owns its stream and workspace. */
int rrs_engine_create(int32_t device, rrs_engine** out);
int rrs_engine_destroy(rrs_engine* e);
/* Run on a caller stream (cudaStream_t as void*); NULL restores the engine's own. */
int rrs_engine_set_stream(rrs_engine* e, void* stream);
int rrs_engine_synchronize(rrs_engine* e);
/* Cap on workspace bytes used for query batching (default: a quarter of the
 * device's free memory at engine creation, clamped to [1, 32] GiB). */
int rrs_engine_set_workspace_limit(rrs_engine* e, int64_t bytes);

/* Dataset(rows) -- projection.py:44-75.  x is n x d row-major FP64, finite;
 * stored on device as FP32 in tile-blocked layout.
 * The entries are checked on the device copy: RRS_ERR_INVALID with
 * "dataset contains non-finite entries" (projection.py's message) or "... exceed
 * the FP32 contraction range (|x| > 1e38)"; the engine keeps its previous
 * dataset on failure.  For 64 < d <= 256 the per-point bound max_l |x_il| of
 * the wide tensor kernel is precomputed here. */
int rrs_set_dataset_host(rrs_engine* e, const double* x, int64_t n, int32_t d);
/* Same from a device FP64 buffer (n x d row-major), stream-ordered (the
 * validation synchronises the engine stream once). */
int rrs_set_dataset_device(rrs_engine* e, const double* x_dev, int64_t n, int32_t d);

/* depth_batch(queries, data, cfg) -- optimizer.py:254-279, with
 * refined_random_search (optimizer.py:145-226) per query.  Query i uses the
 * Philox substream of query index q0 + i (global index when sharded).
 *   depth[Q]                 DepthResult.depth
 *   argmin[Q*d]   nullable   DepthResult.argmin_direction
 *   trace[Q*r*(2+d)] nullable  RefinementRecord (best_depth, epsilon, pole[d])
 *   min_count[Q]  nullable   halfspace only: min(#<=, #>=) of the final depth
 * eps (nullable, r doubles) overrides the pi/2*alpha^l schedule (optimizer.py:175). */
int rrs_depth_batch_host(rrs_engine* e, const double* queries, int64_t Q, int64_t q0,
                         const rrs_config* cfg, const double* eps, double* depth,
                         double* argmin, double* trace, int64_t* min_count);
/* Device-resident variant: every pointer is device memory, the kernels run on
 * the engine stream.  The queries are validated on the device (finite,
 * |z| <= 1e38) and the flag is read back once the batch is enqueued, so the
 * call returns after the batch completed; a bad query fails the call. */
int rrs_depth_batch_device(rrs_engine* e, const double* queries_dev, int64_t Q, int64_t q0,
                           const rrs_config* cfg, const double* eps, double* depth_dev,
                           double* argmin_dev, double* trace_dev, int64_t* min_count_dev);

/* evaluate_directions(z, data, dirs, notion, cfg) -- optimizer.py:98-142:
 * univariate depths of z over injected unit directions U (m x d, FP64).
 * cle/cge (nullable, halfspace only) receive #(<=) and #(>=) per direction. */
int rrs_evaluate_directions_host(rrs_engine* e, const double* z, const double* U, int32_t m,
                                 int32_t notion, double* out, int64_t* cle, int64_t* cge);

/* generate_batch(CapSpec(Pole(pole), eps), m, seed, refinement, query) rows
 * -- directions.py:192-204 (on device, FP64). */
int rrs_cap_directions_host(rrs_engine* e, const double* pole, int32_t d, double eps, int32_t m,
                            uint64_t seed, uint32_t refinement, uint32_t query, double* U);

/* random_sphere_pole(cap, SubStream(seed, refinement, query, index_base)) and
 * generate_batch rows from Philox direction index index_base on --
 * directions.py:185-189, _cap_rows(..., index_base) :167-182. */
int rrs_cap_directions_at_host(rrs_engine* e, const double* pole, int32_t d, double eps, int32_t m,
                               uint64_t seed, uint32_t refinement, uint32_t query, uint32_t index_base,
                               double* U);

/* _unit_rows(seed, refinement, query, m, dim, v_base, index_base) --
 * directions.py:113-135 (random_sphere(d, stream) = m 1, v_base 0,
 * index_base stream.index, directions.py:138-147).  U: m x dim FP64. */
int rrs_unit_rows_host(rrs_engine* e, uint64_t seed, uint32_t refinement, uint32_t query, int32_t m,
                       int32_t dim, uint32_t v_base, uint32_t index_base, double* U);

/* SubStream(seed, refinement, query, index).uniforms(count, offset) (normal 0)
 * and .normals(count, offset) (normal 1) -- directions.py:76-94 over
 * philox.uniforms / normals (philox.py:88-125). */
int rrs_stream_values_host(rrs_engine* e, uint64_t seed, uint32_t refinement, uint32_t query, uint32_t index,
                           uint32_t offset, int64_t count, int32_t normal, double* out);

/* project_naive / project_parallel / project_point -- projection.py:99-168,
 * _kernels.pyx:120-199: out[j*n + i] = sum_l U[j,l] * x[i,l] in FP64,
 * acc = 0.0, ascending l, no FMA (bit-identical to the reference).
 * x: n x d, U: m x d, out: m x n, all row-major FP64 host buffers. */
int rrs_project_host(rrs_engine* e, const double* x, int64_t n, int32_t d, const double* U, int32_t m,
                     double* out);

/* depth_of_projections(notion, px, pz, out) -- univariate.py:162-184 over the
 * span kernels _kernels.pyx:270-351: px m x n, pz m, out m (FP64 host
 * buffers); exact FP64 order statistics, bit-identical to the reference. */
int rrs_depth_of_projections_host(rrs_engine* e, int32_t notion, const double* px, int32_t m, int64_t n,
                                  const double* pz, double* out);

/* philox4x32 / philox4x32_words -- philox.py:27-65, _kernels.pyx:24-61, on
 * device.  ctr and out are (4, N) row-major uint32. */
int rrs_philox4x32_host(rrs_engine* e, const uint32_t* ctr, int64_t N, uint32_t key0,
                        uint32_t key1, uint32_t* out);

/* Contraction kernel: 0 = auto (tensor cores when d <= 256 and n >= 4096),
 * 1 = FP32 FFMA (contract.cu), 2 = tcgen05 FP16 hi/lo split with FP32
 * accumulation (contract_tc.cu for d <= 64, the pre-split contract_tcp.cu for
 * 64 < d <= 256), 4 = filter and refine (contract_tcf.cu, d <= 64), 5 = the
 * three-term tensor projection store (contract_tcs.cu), 6 = as 0 but with the
 * in-kernel converters above d = 64 (contract_tcw.cu).  Any d > 256 (up to
 * 1024) takes the FP64 contraction (contract64.cu) whatever the path. */
int rrs_engine_set_contract_path(rrs_engine* e, int32_t path);

/* Page-locked host buffers (cudaHostAlloc, portable): the matrix loaders
 * (io.read_matrix(..., pinned=True)) read DFMX payloads straight into one, so
 * rrs_set_dataset_host / rrs_depth_batch_host copy from it by DMA.  Replaces
 * the reference's pageable np.frombuffer / np.array results (io.py:63-110). */
int rrs_host_alloc(int64_t bytes, void** out);
int rrs_host_free(void* p);

/* Order-statistic kernel for the projection notions: 0 = auto (the
 * sample-bracket select, select.cu v3, for 2048 <= n <= 53248; radix select
 * elsewhere), 2 = radix select v2 everywhere, 3 = v3 with 1024-thread CTAs
 * above n = 16384.  All give bitwise equal depths
 * (same FP32 keys, FP64 midpoints); the switch exists for A/B measurement. */
int rrs_engine_set_select_path(rrs_engine* e, int32_t path);

/* Diagnostics for the last batch: device time (ms) of each stage summed over
 * the batch (generation, contraction, univariate, update) and launch count. */
typedef struct {
    double ms_generate, ms_contract, ms_univariate, ms_update;
    int64_t kernel_launches;
    int64_t contract_launches;
    double ms_contract_total; /* sum of contraction-kernel durations */
    int64_t tensor_contract_launches; /* of contract_launches, on the tcgen05 kernel */
    int64_t select_rows_fallback; /* projection rows whose sample bracket missed (select v3) */
} rrs_stats;
int rrs_engine_stats(rrs_engine* e, rrs_stats* out);
int rrs_engine_enable_timing(rrs_engine* e, int32_t on);

#ifdef __cplusplus
}
#endif
#endif
