/*
 * rrs_oracle.h -- CPU restatement of the reference RRS hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in paper_2506_08262_b200/ links, loads or
 * calls this library; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs do, and there only as the checker or
 * as the timed CPU baseline ("port").
 *
 * Every function restates the reference algorithm of
 * /root/reference/pkg/src/depthforge (depthforge 0.1.0) in plain C, FP64,
 * compiled with -ffp-contract=off exactly like the reference core
 * (pkg/setup.py:50-53).  Parity is pinned against the imported reference by
 * tests/golden/make_golden.py -> the tests/golden fixtures.
 */
#ifndef RRS_ORACLE_H
#define RRS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_HALFSPACE = 0, ORC_PROJECTION = 1, ORC_ASYM_PROJECTION = 2 };

typedef struct {
    int64_t total_directions; /* k          optimizer.py:46  */
    int32_t refinements;      /* r          optimizer.py:47  */
    double shrink;            /* alpha      optimizer.py:48  */
    int32_t notion;           /* ORC_*      optimizer.py:49  */
    uint64_t seed;            /* seed mod 2^64 (philox.py:68-71) */
    int32_t pole_update;      /* 0 per_refinement, 1 per_direction (optimizer.py:200-218) */
} orc_cfg;

/* philox.py:27-65 / _kernels.pyx:24-61.  ctr and out are (4, N) row-major. */
void orc_philox4x32(const uint32_t* ctr, int64_t N, uint32_t key0, uint32_t key1, uint32_t* out);
/* philox.py:88-114: addressed uniforms in (0,1); v[i], j[i] per element. */
void orc_uniforms(uint64_t seed, const uint32_t* v, const uint32_t* j, int64_t N,
                  uint32_t l, uint32_t q, double* out);
/* scipy.special.ndtri (Cephes ndtri, scipy 1.18.1) -- philox.py:117-125 */
double orc_ndtri(double y);
void orc_ndtri_array(const double* y, int64_t N, double* out);
/* numpy pairwise summation (numpy 2.3 loops_utils.h pairwise_sum), 0.0 + sum */
double orc_pairwise_sum(const double* a, int64_t n, int64_t stride);
/* directions.py:167-182 (_cap_rows) incl. _unit_rows redraw + reflect_to_pole */
int orc_cap_rows(const double* pole, int32_t d, double eps, int32_t m, uint64_t seed,
                 uint32_t l, uint32_t q, double* rows);
/* _kernels.pyx:171-185 proj_naive: out[j,i] = sum_l u[j,l] x[i,l], ascending l */
void orc_project(const double* x, int64_t n, int32_t d, const double* u, int32_t m, double* px);
/* _kernels.pyx:188-199 */
void orc_project_point(const double* z, int32_t d, const double* u, int32_t m, double* pz);
/* _kernels.pyx:270-351: univariate depth per direction on materialised px (m x n).
 * cle/cge (nullable) receive the halfspace counts. */
int orc_univariate(int32_t notion, const double* px, const double* pz, int32_t m, int64_t n,
                   double* out, int64_t* cle, int64_t* cge);
/* optimizer.py:98-142 evaluate_directions */
int orc_evaluate_directions(const double* x, int64_t n, int32_t d, const double* z,
                            const double* U, int32_t m, int32_t notion, double* out,
                            int64_t* cle, int64_t* cge);
/* optimizer.py:254-279 depth_batch (query_index = q0 + position).
 * depth[Q]; argmin[Q*d] nullable; trace[Q*r*(2+d)] nullable, record layout
 * (best_depth, epsilon, pole[d]); threads <= 0 -> all online CPUs. */
int orc_depth_batch(const double* x, int64_t n, int32_t d, const double* Z, int64_t Q,
                    int64_t q0, const orc_cfg* cfg, int32_t threads, double* depth,
                    double* argmin, double* trace);
const char* orc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
