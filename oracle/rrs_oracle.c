/*
 * rrs_oracle.c -- CPU restatement of the reference RRS hot path (FP64).
 *
 * TEST INFRASTRUCTURE ONLY (see rrs_oracle.h).  Written from the reference's
 * documented algorithm, not copied: each function cites the reference
 * file:line it restates (paths relative to /root/reference/pkg/src/depthforge).
 * Third-party arithmetic restated from its published algorithm:
 *   - scipy.special.ndtri (scipy 1.18.1, Cephes "ndtri"; philox.py:16,125)
 *   - numpy 2.3.5 pairwise summation for row sums (directions.py:127,162)
 *   - libm cos/sqrt/log/pow (glibc, shared with the reference's numpy path).
 * Build: oracle/Makefile (-O3 -march=native -ffp-contract=off, like setup.py:50-53).
 */
#include "rrs_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

static _Thread_local char g_err[256];
static char g_err_global[256];

static void set_err(const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    snprintf(g_err_global, sizeof g_err_global, "%s", msg);
}

const char* orc_last_error(void) { return g_err[0] ? g_err : g_err_global; }

/* ---------------------------------------------------------------- Philox --
 * Philox-4x32-10 (Salmon et al., Random123): philox.py:27-65, _kernels.pyx:24-61.
 * Round: (hi,lo) of x0*M0 and x2*M1; x0' = hi1^x1^k0, x1' = lo1, x2' = hi0^x3^k1,
 * x3' = lo0; key bumped by the Weyl constants after every round. */
static inline void philox_block(uint32_t c[4], uint32_t k0, uint32_t k1) {
    for (int r = 0; r < 10; ++r) {
        uint64_t p0 = (uint64_t)c[0] * 0xD2511F53u;
        uint64_t p1 = (uint64_t)c[2] * 0xCD9E8D57u;
        uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0;
        uint32_t n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
        c[1] = (uint32_t)p1;
        c[3] = (uint32_t)p0;
        c[0] = n0;
        c[2] = n2;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

void orc_philox4x32(const uint32_t* ctr, int64_t N, uint32_t key0, uint32_t key1, uint32_t* out) {
    for (int64_t i = 0; i < N; ++i) {
        uint32_t c[4] = {ctr[i], ctr[N + i], ctr[2 * N + i], ctr[3 * N + i]};
        philox_block(c, key0, key1);
        out[i] = c[0];
        out[N + i] = c[1];
        out[2 * N + i] = c[2];
        out[3 * N + i] = c[3];
    }
}

/* philox.py:68-71 split_key, :88-114 uniforms: counter (v, j, l, q), 53-bit
 * mantissa from words 0|1<<32, shifted by half an ulp into the open interval. */
static inline double uniform1(uint64_t seed, uint32_t v, uint32_t j, uint32_t l, uint32_t q) {
    uint32_t c[4] = {v, j, l, q};
    philox_block(c, (uint32_t)(seed & 0xFFFFFFFFu), (uint32_t)(seed >> 32));
    uint64_t bits = (uint64_t)c[0] | ((uint64_t)c[1] << 32);
    return ((double)(bits >> 11) + 0.5) * 0x1.0p-53;
}

void orc_uniforms(uint64_t seed, const uint32_t* v, const uint32_t* j, int64_t N, uint32_t l,
                  uint32_t q, double* out) {
    for (int64_t i = 0; i < N; ++i) out[i] = uniform1(seed, v[i], j[i], l, q);
}

/* ----------------------------------------------------------------- ndtri --
 * Inverse standard normal CDF, Cephes algorithm as shipped in scipy 1.18.1:
 * central rational approximation for |y-1/2| <= 1/2-exp(-2), else the
 * sqrt(-2 log y) expansions split at x = 8.  Coefficients are Cephes' published
 * tables; Q* are evaluated with an implicit leading 1 (p1evl). */
static const double NDTRI_P0[5] = {-5.99633501014107895267E1, 9.80010754185999661536E1,
                                   -5.66762857469070293439E1, 1.39312609387279679503E1,
                                   -1.23916583867381258016E0};
static const double NDTRI_Q0[8] = {1.95448858338141759834E0,  4.67627912898881538453E0,
                                   8.63602421390890590575E1,  -2.25462687854119370527E2,
                                   2.00260212380060660359E2,  -8.20372256168333339912E1,
                                   1.59056225126211695515E1,  -1.18331621121330003142E0};
static const double NDTRI_P1[9] = {4.05544892305962419923E0,   3.15251094599893866154E1,
                                   5.71628192246421288162E1,   4.40805073893200834700E1,
                                   1.46849561928858024014E1,   2.18663306850790267539E0,
                                   -1.40256079171354495875E-1, -3.50424626827848203418E-2,
                                   -8.57456785154685413611E-4};
static const double NDTRI_Q1[8] = {1.57799883256466749731E1,   4.53907635128879210584E1,
                                   4.13172038254672030440E1,   1.50425385692907503408E1,
                                   2.50464946208309415979E0,   -1.42182922854787788574E-1,
                                   -3.80806407691578277194E-2, -9.33259480895457427372E-4};
static const double NDTRI_P2[9] = {3.23774891776946035970E0,  6.91522889068984211695E0,
                                   3.93881025292474443415E0,  1.33303460815807542389E0,
                                   2.01485389549179081538E-1, 1.23716634817820021358E-2,
                                   3.01581553508235416007E-4, 2.65806974686737550832E-6,
                                   6.23974539184983293730E-9};
static const double NDTRI_Q2[8] = {6.02427039364742014255E0,  3.67983563856160859403E0,
                                   1.37702099489081330271E0,  2.16236993594496635890E-1,
                                   1.34204006088543189037E-2, 3.28014464682127739104E-4,
                                   2.89247864745380683936E-6, 6.79019408009981274425E-9};

static inline double polevl(double x, const double* c, int deg) {
    double a = c[0];
    for (int i = 1; i <= deg; ++i) a = a * x + c[i];
    return a;
}
static inline double p1evl(double x, const double* c, int deg) {
    double a = x + c[0];
    for (int i = 1; i < deg; ++i) a = a * x + c[i];
    return a;
}

double orc_ndtri(double y0) {
    const double s2pi = 2.50662827463100050242E0;
    const double e2 = 0.13533528323661269189; /* exp(-2) */
    if (y0 == 0.0) return -INFINITY;
    if (y0 == 1.0) return INFINITY;
    if (y0 < 0.0 || y0 > 1.0) return NAN;
    int negate = 1;
    double y = y0;
    if (y > 1.0 - e2) {
        y = 1.0 - y;
        negate = 0;
    }
    if (y > e2) {
        y = y - 0.5;
        double y2 = y * y;
        double x = y + y * (y2 * polevl(y2, NDTRI_P0, 4) / p1evl(y2, NDTRI_Q0, 8));
        return x * s2pi;
    }
    double x = sqrt(-2.0 * log(y));
    double x0 = x - log(x) / x;
    double z = 1.0 / x;
    double x1 = (x < 8.0) ? z * polevl(z, NDTRI_P1, 8) / p1evl(z, NDTRI_Q1, 8)
                          : z * polevl(z, NDTRI_P2, 8) / p1evl(z, NDTRI_Q2, 8);
    x = x0 - x1;
    return negate ? -x : x;
}

void orc_ndtri_array(const double* y, int64_t N, double* out) {
    for (int64_t i = 0; i < N; ++i) out[i] = orc_ndtri(y[i]);
}

/* --------------------------------------------------------- pairwise sum --
 * numpy's float64 add.reduce over a contiguous row: identity 0.0 plus the
 * pairwise sum (8 running partials up to 128 elements, recursive halving at
 * multiples of 8 beyond).  Checked bit-exact against numpy in tests. */
static double pw_sum(const double* a, int64_t n, int64_t s) {
    if (n < 8) {
        double r = 0.0;
        for (int64_t i = 0; i < n; ++i) r += a[i * s];
        return r;
    }
    if (n <= 128) {
        double r[8];
        for (int k = 0; k < 8; ++k) r[k] = a[k * s];
        int64_t i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int k = 0; k < 8; ++k) r[k] += a[(i + k) * s];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i * s];
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return pw_sum(a, n2, s) + pw_sum(a + n2 * s, n - n2, s);
}

double orc_pairwise_sum(const double* a, int64_t n, int64_t stride) {
    return 0.0 + pw_sum(a, n, stride);
}

/* ------------------------------------------------------------ cap rows --
 * directions.py:167-182 _cap_rows: theta = U(v=0, j) * eps (angle-uniform),
 * u1 = cos(theta); the remaining d-1 coordinates are a normalised normal row
 * from value addresses v = 1..d-1 (zero-norm rows redrawn from the next d-1
 * addresses, directions.py:113-135), scaled by sqrt(1 - u1^2); finally the
 * Householder map e1 -> pole (directions.py:150-164). */
int orc_cap_rows(const double* pole, int32_t d, double eps, int32_t m, uint64_t seed,
                 uint32_t l, uint32_t q, double* rows) {
    if (m < 1 || d < 1) {
        set_err("batch size must be >= 1");
        return 1;
    }
    if (d == 1) { /* directions.py:172-173 */
        for (int32_t j = 0; j < m; ++j) rows[j] = pole[0];
        return 0;
    }
    const int32_t dm = d - 1;
    double* g = (double*)malloc(sizeof(double) * (size_t)dm * 2);
    if (!g) {
        set_err("out of memory");
        return 4;
    }
    double* sq = g + dm;
    for (int32_t j = 0; j < m; ++j) {
        double* row = rows + (int64_t)j * d;
        double theta = uniform1(seed, 0u, (uint32_t)j, l, q) * eps;
        double u1 = cos(theta);
        uint32_t vbase = 1;
        double nrm;
        for (;;) {
            for (int32_t c = 0; c < dm; ++c)
                g[c] = orc_ndtri(uniform1(seed, vbase + (uint32_t)c, (uint32_t)j, l, q));
            for (int32_t c = 0; c < dm; ++c) sq[c] = g[c] * g[c];
            nrm = sqrt(orc_pairwise_sum(sq, dm, 1));
            if (nrm != 0.0) break;
            vbase += (uint32_t)dm;
        }
        double s = sqrt(1.0 - u1 * u1);
        row[0] = u1;
        for (int32_t c = 0; c < dm; ++c) row[1 + c] = s * (g[c] / nrm);
    }
    free(g);
    /* reflect_to_pole */
    const double tol = 1e-12;
    double p1 = pole[0];
    if (1.0 - p1 < tol) return 0;
    if (1.0 + p1 < tol) {
        for (int32_t j = 0; j < m; ++j) rows[(int64_t)j * d] = -rows[(int64_t)j * d];
        return 0;
    }
    double* v = (double*)malloc(sizeof(double) * (size_t)d * 2);
    if (!v) {
        set_err("out of memory");
        return 4;
    }
    double* tmp = v + d;
    for (int32_t c = 0; c < d; ++c) v[c] = -pole[c];
    v[0] += 1.0;
    double ss = 0.0; /* np.linalg.norm -> BLAS ddot; summation order is BLAS's */
    for (int32_t c = 0; c < d; ++c) ss += v[c] * v[c];
    double vn = sqrt(ss);
    for (int32_t c = 0; c < d; ++c) v[c] /= vn;
    for (int32_t j = 0; j < m; ++j) {
        double* row = rows + (int64_t)j * d;
        for (int32_t c = 0; c < d; ++c) tmp[c] = row[c] * v[c];
        double proj = orc_pairwise_sum(tmp, d, 1);
        double f = 2.0 * proj;
        for (int32_t c = 0; c < d; ++c) row[c] = row[c] - f * v[c];
    }
    free(v);
    return 0;
}

/* ----------------------------------------------------------- projection --
 * _kernels.pyx:68-107,171-199: every score accumulates its d products in
 * ascending coordinate order from 0.0, one rounding per multiply and per add. */
void orc_project(const double* x, int64_t n, int32_t d, const double* u, int32_t m, double* px) {
    for (int32_t j = 0; j < m; ++j)
        for (int64_t i = 0; i < n; ++i) {
            double acc = 0.0;
            for (int32_t l = 0; l < d; ++l) acc = acc + u[(int64_t)j * d + l] * x[i * d + l];
            px[(int64_t)j * n + i] = acc;
        }
}

void orc_project_point(const double* z, int32_t d, const double* u, int32_t m, double* pz) {
    for (int32_t j = 0; j < m; ++j) {
        double acc = 0.0;
        for (int32_t l = 0; l < d; ++l) acc = acc + u[(int64_t)j * d + l] * z[l];
        pz[j] = acc;
    }
}

/* Tiled equivalent used inside the RRS loop: 8 directions x 128 points per
 * tile over the transposed data; same per-element operation order. */
static void project_block(const double* xt, int64_t n, int32_t d, const double* u, int32_t nb,
                          double* out /* nb x n */) {
    enum { TI = 128 };
    for (int64_t i0 = 0; i0 < n; i0 += TI) {
        int64_t cnt = n - i0 < TI ? n - i0 : TI;
        for (int32_t b = 0; b < nb; ++b) memset(out + (int64_t)b * n + i0, 0, sizeof(double) * cnt);
        for (int32_t l = 0; l < d; ++l) {
            const double* xr = xt + (int64_t)l * n + i0;
            for (int32_t b = 0; b < nb; ++b) {
                const double w = u[(int64_t)b * d + l];
                double* o = out + (int64_t)b * n + i0;
                for (int64_t i = 0; i < cnt; ++i) o[i] = o[i] + w * xr[i];
            }
        }
    }
}

/* ------------------------------------------------------------ selection --
 * k-th smallest of a[0:n) with a 3-way partition quickselect; leaves
 * a[t] <= a[k] for t < k and a[t] >= a[k] for t > k (the property
 * _median_inplace relies on, _kernels.pyx:255-267).  The returned value is
 * an order statistic, so it is independent of the pivot strategy. */
static double kth(double* a, int64_t n, int64_t k) {
    int64_t lo = 0, hi = n - 1;
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        double x = a[lo], y = a[mid], z = a[hi], p;
        if ((x <= y && y <= z) || (z <= y && y <= x)) p = y;
        else if ((y <= x && x <= z) || (z <= x && x <= y)) p = x;
        else p = z;
        int64_t lt = lo, i = lo, gt = hi;
        while (i <= gt) {
            double v = a[i];
            if (v < p) {
                a[i] = a[lt];
                a[lt] = v;
                ++lt;
                ++i;
            } else if (v > p) {
                a[i] = a[gt];
                a[gt] = v;
                --gt;
            } else {
                ++i;
            }
        }
        if (k < lt) hi = lt - 1;
        else if (k > gt) lo = gt + 1;
        else return p;
    }
    return a[k];
}

/* midpoint of the two central order statistics for even n (univariate.py:71-77) */
static double median_inplace(double* a, int64_t n) {
    int64_t k = (n - 1) >> 1;
    double lo = kth(a, n, k);
    if (n & 1) return lo;
    double hi = a[k + 1];
    for (int64_t t = k + 2; t < n; ++t)
        if (a[t] < hi) hi = a[t];
    return (lo + hi) / 2.0;
}

/* _kernels.pyx:270-289 halfspace_span; :292-314 projection_span;
 * :317-351 asym_projection_span.  One direction. */
static double univariate1(int32_t notion, const double* px, double y, int64_t n, double* buf,
                          int64_t* cle_out, int64_t* cge_out) {
    if (notion == ORC_HALFSPACE) {
        int64_t cle = 0, cge = 0;
        for (int64_t i = 0; i < n; ++i) {
            double v = px[i];
            cle += (v <= y);
            cge += (v >= y);
        }
        if (cle_out) *cle_out = cle;
        if (cge_out) *cge_out = cge;
        int64_t c = cle < cge ? cle : cge;
        return (double)c / (double)n;
    }
    memcpy(buf, px, sizeof(double) * (size_t)n);
    double med = median_inplace(buf, n);
    if (notion == ORC_PROJECTION) {
        for (int64_t i = 0; i < n; ++i) buf[i] = fabs(px[i] - med);
        double mad = median_inplace(buf, n);
        double dev = fabs(y - med);
        if (mad == 0.0) return dev == 0.0 ? 1.0 : 0.0;
        return 1.0 / (1.0 + dev / mad);
    }
    double dev = y - med;
    if (dev <= 0.0) return 1.0;
    int64_t npos = 0;
    for (int64_t i = 0; i < n; ++i) {
        double t = px[i] - med;
        if (t > 0.0) buf[npos++] = t;
    }
    if (npos == 0) return 0.0;
    double madp = median_inplace(buf, npos);
    return 1.0 / (1.0 + dev / madp);
}

int orc_univariate(int32_t notion, const double* px, const double* pz, int32_t m, int64_t n,
                   double* out, int64_t* cle, int64_t* cge) {
    if (notion < 0 || notion > 2) {
        set_err("unknown depth notion");
        return 1;
    }
    if (n < 1) {
        set_err("empty projection");
        return 1;
    }
    double* buf = (double*)malloc(sizeof(double) * (size_t)n);
    if (!buf) {
        set_err("out of memory");
        return 4;
    }
    for (int32_t j = 0; j < m; ++j)
        out[j] = univariate1(notion, px + (int64_t)j * n, pz[j], n, buf, cle ? cle + j : NULL,
                             cge ? cge + j : NULL);
    free(buf);
    return 0;
}

int orc_evaluate_directions(const double* x, int64_t n, int32_t d, const double* z,
                            const double* U, int32_t m, int32_t notion, double* out,
                            int64_t* cle, int64_t* cge) {
    double* px = (double*)malloc(sizeof(double) * ((size_t)m * (size_t)n + (size_t)m));
    if (!px) {
        set_err("out of memory");
        return 4;
    }
    double* pz = px + (int64_t)m * n;
    orc_project(x, n, d, U, m, px);
    orc_project_point(z, d, U, m, pz);
    int rc = orc_univariate(notion, px, pz, m, n, out, cle, cge);
    free(px);
    return rc;
}

/* ------------------------------------------------------------------ RRS --
 * optimizer.py:145-226 refined_random_search on one query. */
typedef struct {
    const double* x;
    const double* xt;
    int64_t n;
    int32_t d;
    const orc_cfg* cfg;
    const double* eps; /* [r] */
    int32_t m;
} rrs_ctx;

typedef struct {
    double* U;      /* m x d */
    double* pxb;    /* 8 x n */
    double* pz;     /* m */
    double* depths; /* m */
    double* buf;    /* n */
    double* pole;   /* d */
} rrs_ws;

static int rrs_one(const rrs_ctx* c, rrs_ws* w, const double* z, uint32_t qidx, double* depth_out,
                   double* argmin_out, double* trace_out) {
    const int32_t d = c->d, m = c->m;
    const int64_t n = c->n;
    for (int32_t k = 0; k < d; ++k) w->pole[k] = 0.0;
    w->pole[0] = 1.0;
    double dmin = 1.0;
    for (int32_t l = 0; l < c->cfg->refinements; ++l) {
        double eps = c->eps[l];
        int rc = orc_cap_rows(w->pole, d, eps, m, c->cfg->seed, (uint32_t)l, qidx, w->U);
        if (rc) return rc;
        orc_project_point(z, d, w->U, m, w->pz);
        for (int32_t j0 = 0; j0 < m; j0 += 8) {
            int32_t nb = m - j0 < 8 ? m - j0 : 8;
            project_block(c->xt, n, d, w->U + (int64_t)j0 * d, nb, w->pxb);
            for (int32_t b = 0; b < nb; ++b)
                w->depths[j0 + b] = univariate1(c->cfg->notion, w->pxb + (int64_t)b * n,
                                                w->pz[j0 + b], n, w->buf, NULL, NULL);
        }
        /* np.argmin: first index of the minimum; strict-< update
         * (optimizer.py:200-205).  The per_direction scan (:206-218) ends on
         * the same direction: the last strict prefix minimum is the first
         * argmin whenever it beats d_min. */
        int32_t jb = 0;
        for (int32_t j = 1; j < m; ++j)
            if (w->depths[j] < w->depths[jb]) jb = j;
        if (w->depths[jb] < dmin) {
            dmin = w->depths[jb];
            memcpy(w->pole, w->U + (int64_t)jb * d, sizeof(double) * (size_t)d);
        }
        if (trace_out) {
            double* rec = trace_out + (int64_t)l * (2 + d);
            rec[0] = dmin;
            rec[1] = eps;
            memcpy(rec + 2, w->pole, sizeof(double) * (size_t)d);
        }
    }
    *depth_out = dmin;
    if (argmin_out) memcpy(argmin_out, w->pole, sizeof(double) * (size_t)d);
    return 0;
}

typedef struct {
    rrs_ctx ctx;
    const double* Z;
    int64_t Q, q0;
    double *depth, *argmin, *trace;
    atomic_long next;
    atomic_int rc;
} batch_job;

static void* batch_worker(void* arg) {
    batch_job* J = (batch_job*)arg;
    const rrs_ctx* c = &J->ctx;
    rrs_ws w;
    size_t nd = (size_t)c->n;
    w.U = (double*)malloc(sizeof(double) * ((size_t)c->m * c->d + 8 * nd + 2 * (size_t)c->m + nd + c->d));
    if (!w.U) {
        atomic_store(&J->rc, 4);
        return NULL;
    }
    w.pxb = w.U + (size_t)c->m * c->d;
    w.pz = w.pxb + 8 * nd;
    w.depths = w.pz + c->m;
    w.buf = w.depths + c->m;
    w.pole = w.buf + nd;
    for (;;) {
        long i = atomic_fetch_add(&J->next, 1);
        if (i >= J->Q || atomic_load(&J->rc)) break;
        int rc = rrs_one(c, &w, J->Z + i * c->d, (uint32_t)((uint64_t)(J->q0 + i) & 0xFFFFFFFFu),
                         J->depth + i, J->argmin ? J->argmin + i * c->d : NULL,
                         J->trace ? J->trace + i * (int64_t)c->cfg->refinements * (2 + c->d) : NULL);
        if (rc) atomic_store(&J->rc, rc);
    }
    free(w.U);
    return NULL;
}

int orc_depth_batch(const double* x, int64_t n, int32_t d, const double* Z, int64_t Q, int64_t q0,
                    const orc_cfg* cfg, int32_t threads, double* depth, double* argmin,
                    double* trace) {
    g_err[0] = 0;
    if (cfg->refinements < 1 || cfg->total_directions < cfg->refinements) {
        set_err("need total_directions >= refinements >= 1");
        return 1;
    }
    if (!(cfg->shrink > 0.0 && cfg->shrink < 1.0)) {
        set_err("shrink factor must lie in (0, 1)");
        return 1;
    }
    if (cfg->notion < 0 || cfg->notion > 2) {
        set_err("unknown depth notion");
        return 1;
    }
    if (n < 1 || d < 1) {
        set_err("dataset must be a non-empty 2-D matrix");
        return 1;
    }
    if (Q < 1) return 0;
    const int32_t r = cfg->refinements;
    double* eps = (double*)malloc(sizeof(double) * (size_t)r);
    double* xt = (double*)malloc(sizeof(double) * (size_t)n * d);
    if (!eps || !xt) {
        free(eps);
        free(xt);
        set_err("out of memory");
        return 4;
    }
    const double half_pi = 3.141592653589793 / 2.0; /* optimizer.py:37 */
    for (int32_t l = 0; l < r; ++l) eps[l] = half_pi * pow(cfg->shrink, (double)l); /* :175 */
    for (int64_t i = 0; i < n; ++i)
        for (int32_t k = 0; k < d; ++k) xt[(int64_t)k * n + i] = x[i * d + k];

    batch_job J;
    J.ctx.x = x;
    J.ctx.xt = xt;
    J.ctx.n = n;
    J.ctx.d = d;
    J.ctx.cfg = cfg;
    J.ctx.eps = eps;
    J.ctx.m = (int32_t)((cfg->total_directions + r - 1) / r); /* optimizer.py:64-66 */
    J.Z = Z;
    J.Q = Q;
    J.q0 = q0;
    J.depth = depth;
    J.argmin = argmin;
    J.trace = trace;
    atomic_init(&J.next, 0);
    atomic_init(&J.rc, 0);
    if (threads <= 0) threads = (int32_t)sysconf(_SC_NPROCESSORS_ONLN);
    if (threads > Q) threads = (int32_t)Q;
    if (threads < 1) threads = 1;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    int spawned = 0;
    for (int t = 1; t < threads; ++t)
        if (pthread_create(&th[spawned], NULL, batch_worker, &J) == 0) ++spawned;
    batch_worker(&J);
    for (int t = 0; t < spawned; ++t) pthread_join(th[t], NULL);
    free(th);
    free(eps);
    free(xt);
    int rc = atomic_load(&J.rc);
    if (rc == 4) set_err("out of memory");
    return rc;
}
