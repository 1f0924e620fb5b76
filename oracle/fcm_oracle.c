/*
 * fcm_oracle.c -- CPU restatement of the reference FCM hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * path in paper_1601_00072_b200/csrc.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it; the
 * product path never does (and fails loudly when its own CUDA library is
 * missing instead of falling back here).
 *
 * Every function restates one function of the reference package
 * (/root/reference/pkg/src/fcmseg/_kernels.pyx, mirrored by _kernels_py.py)
 * with the SAME IEEE-754 double expressions in the SAME evaluation order and
 * the same libm pow/fabs.  Built with -O2 -ffp-contract=off exactly like the
 * reference extension (pkg/setup.py:12-16), so outputs are bit-identical to
 * the reference on the same glibc.  The pin is tests/test_oracle.py, which
 * compares this library bitwise against golden vectors produced by the
 * reference itself (tests/golden/make_golden.py).
 *
 * Layout conventions (reference _kernels_py.py:9-15): flat C-contiguous
 * float64 buffers, membership AoS u[i*c + j].
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef uint64_t u64;

static const u64 GAMMA = 0x9E3779B97F4A7C15ULL;  /* _kernels.pyx:16 */
static const u64 MIX1 = 0xBF58476D1CE4E5B9ULL;   /* _kernels.pyx:17 */
static const u64 MIX2 = 0x94D049BB133111EBULL;   /* _kernels.pyx:18 */
static const double INV53 = 1.0 / 9007199254740992.0; /* _kernels.pyx:19 */

/* _kernels.pyx:33-41 -- advance state, return output. */
void oracle_splitmix64(u64 state, u64 *new_state, u64 *out) {
    u64 s = state + GAMMA;
    u64 z = s;
    z = (z ^ (z >> 30)) * MIX1;
    z = (z ^ (z >> 27)) * MIX2;
    *new_state = s;
    *out = z ^ (z >> 31);
}

/* _kernels.pyx:22-30 -- one SplitMix64 draw mapped to (0, 1]. */
static inline double next_uniform(u64 *state) {
    u64 z;
    *state = *state + GAMMA;
    z = *state;
    z = (z ^ (z >> 30)) * MIX1;
    z = (z ^ (z >> 27)) * MIX2;
    z = z ^ (z >> 31);
    return (double)((z >> 11) + 1) * INV53;
}

/* _kernels.pyx:44-69 -- seeded row-stochastic init (core.init_membership). */
int oracle_fill_membership_random(double *u, int64_t n, int64_t c, u64 seed) {
    u64 state = seed;
    double *row = (double *)malloc((size_t)c * sizeof(double));
    if (!row) return -1;
    for (int64_t i = 0; i < n; i++) {
        double total = 0.0;
        for (int64_t j = 0; j < c; j++) {
            double val = next_uniform(&state);
            row[j] = val;
            total = total + val;
        }
        int64_t base = i * c;
        double partial = 0.0;
        for (int64_t j = 0; j < c - 1; j++) {
            double val = row[j] / total;
            u[base + j] = val;
            partial = partial + val;
        }
        double last = 1.0 - partial;
        if (last < 0.0) last = 0.0;
        u[base + c - 1] = last;
    }
    free(row);
    return 0;
}

/* _kernels.pyx:72-90 -- Eq. 3, linear pixel order, cluster-major.
 * Returns -1 or the first cluster whose weight sum is exactly zero. */
int64_t oracle_update_centers_linear(const double *x, const double *u, double *v_out,
                                     int64_t n, int64_t c, double m) {
    for (int64_t j = 0; j < c; j++) {
        double num = 0.0, den = 0.0;
        for (int64_t i = 0; i < n; i++) {
            double w = pow(u[i * c + j], m);
            num = num + w * x[i];
            den = den + w;
        }
        if (den == 0.0) return j;
        v_out[j] = num / den;
    }
    return -1;
}

/* _kernels.pyx:93-120 -- Eq. 4 with the equal-share zero-distance rule. */
void oracle_update_membership_range(const double *x, const double *v, double *u_out,
                                    int64_t c, double m, int64_t i0, int64_t i1) {
    double expo = 2.0 / (m - 1.0);
    for (int64_t i = i0; i < i1; i++) {
        double xi = x[i];
        int64_t base = i * c;
        int64_t zero_count = 0;
        for (int64_t k = 0; k < c; k++)
            if (fabs(xi - v[k]) == 0.0) zero_count = zero_count + 1;
        if (zero_count > 0) {
            double share = 1.0 / (double)zero_count;
            for (int64_t j = 0; j < c; j++)
                u_out[base + j] = (fabs(xi - v[j]) == 0.0) ? share : 0.0;
        } else {
            for (int64_t j = 0; j < c; j++) {
                double dj = fabs(xi - v[j]);
                double s = 0.0;
                for (int64_t k = 0; k < c; k++) s = s + pow(dj / fabs(xi - v[k]), expo);
                u_out[base + j] = 1.0 / s;
            }
        }
    }
}

/* _kernels.pyx:123-134 */
void oracle_center_terms_range(const double *x, const double *u, double *num_out,
                               double *den_out, int64_t c, int64_t j, double m,
                               int64_t i0, int64_t i1) {
    for (int64_t i = i0; i < i1; i++) {
        double w = pow(u[i * c + j], m);
        num_out[i] = w * x[i];
        den_out[i] = w;
    }
}

/* _kernels.pyx:137-165 -- Algorithm 2 block tree. */
int oracle_block_reduce_range(const double *a, double *out, int64_t n, int64_t block_size,
                              int64_t b0, int64_t b1) {
    int64_t span = 2 * block_size;
    double *buf = (double *)malloc((size_t)span * sizeof(double));
    if (!buf) return -1;
    for (int64_t b = b0; b < b1; b++) {
        int64_t start = b * span;
        for (int64_t t = 0; t < block_size; t++) {
            int64_t gi = start + t;
            buf[t] = gi < n ? a[gi] : 0.0;
            gi = start + t + block_size;
            buf[t + block_size] = gi < n ? a[gi] : 0.0;
        }
        for (int64_t stride = block_size; stride > 0; stride >>= 1)
            for (int64_t t = 0; t < stride; t++) buf[t] = buf[t] + buf[t + stride];
        out[b] = buf[0];
    }
    free(buf);
    return 0;
}

/* _kernels.pyx:168-175 */
double oracle_linear_sum(const double *a, int64_t k) {
    double s = 0.0;
    for (int64_t i = 0; i < k; i++) s = s + a[i];
    return s;
}

/* _kernels.pyx:178-191 -- pixel-major objective. */
double oracle_objective_linear(const double *x, const double *u, const double *v,
                               int64_t n, int64_t c, double m) {
    double s = 0.0;
    for (int64_t i = 0; i < n; i++) {
        double xi = x[i];
        int64_t base = i * c;
        for (int64_t j = 0; j < c; j++) {
            double d = xi - v[j];
            s = s + pow(u[base + j], m) * (d * d);
        }
    }
    return s;
}

/* _kernels.pyx:194-208 */
void oracle_objective_terms_range(const double *x, const double *u, const double *v,
                                  double *out, int64_t c, double m, int64_t i0, int64_t i1) {
    for (int64_t i = i0; i < i1; i++) {
        double xi = x[i];
        int64_t base = i * c;
        double acc = 0.0;
        for (int64_t j = 0; j < c; j++) {
            double d = xi - v[j];
            acc = acc + pow(u[base + j], m) * (d * d);
        }
        out[i] = acc;
    }
}

/* _kernels.pyx:211-220 -- strict '>' update. */
double oracle_max_abs_diff(const double *a, const double *b, int64_t i0, int64_t i1) {
    double best = 0.0;
    for (int64_t i = i0; i < i1; i++) {
        double d = fabs(a[i] - b[i]);
        if (d > best) best = d;
    }
    return best;
}

/* _kernels.pyx:223-238 -- ties keep the lowest index. */
void oracle_argmax_rows(const double *u, int32_t *labels_out, int64_t n, int64_t c) {
    for (int64_t i = 0; i < n; i++) {
        int64_t base = i * c;
        double best = u[base];
        int32_t bj = 0;
        for (int64_t j = 1; j < c; j++) {
            double w = u[base + j];
            if (w > best) { best = w; bj = (int32_t)j; }
        }
        labels_out[i] = bj;
    }
}

/*
 * core._iterate (core.py:105-132): the sequential engine's timed loop.
 * u (n*c) is consumed as scratch, exactly like the reference; on return
 * u_final points at whichever of {u, scratch} holds the last membership and
 * is copied back into u.  trace must hold max_iters doubles.
 * Returns 0, or 1 + dead cluster index when update_centers reports a dead
 * cluster (the reference raises DegenerateClusterError there, core.py:122-123).
 */
/* delta_{k-1} and delta_k of the last two iterations of the last iterate
 * call (the values the stop test compared with epsilon, core.py:128-130):
 * parity tests log their margins |delta - epsilon|.
 * Not thread-safe; test infrastructure only. */
static double g_deltas[2] = {0.0, 0.0};
void oracle_last_deltas(double *out) { out[0] = g_deltas[0]; out[1] = g_deltas[1]; }

int64_t oracle_iterate_sequential(const double *x, double *u, int64_t n, int64_t c, double m,
                                  double epsilon, int64_t max_iters, double *v_out,
                                  double *trace, int64_t *iterations, int32_t *converged) {
    double *u_next = (double *)malloc((size_t)(n * c) * sizeof(double));
    double *cur = u, *nxt = u_next;
    int64_t status = 0;
    *iterations = 0;
    *converged = 0;
    if (!u_next) return -1;
    for (int64_t it = 0; it < max_iters; it++) {
        int64_t dead = oracle_update_centers_linear(x, cur, v_out, n, c, m);
        if (dead >= 0) { status = 1 + dead; break; }
        oracle_update_membership_range(x, v_out, nxt, c, m, 0, n);
        double delta = oracle_max_abs_diff(cur, nxt, 0, n * c);
        g_deltas[0] = g_deltas[1]; g_deltas[1] = delta;
        trace[it] = oracle_objective_linear(x, nxt, v_out, n, c, m);
        double *t = cur; cur = nxt; nxt = t;
        *iterations += 1;
        if (delta < epsilon) { *converged = 1; break; }
    }
    if (cur != u) memcpy(u, cur, (size_t)(n * c) * sizeof(double));
    free(u_next);
    return status;
}

/*
 * parallel._iterate (parallel.py:257-331): the paper-shaped block-parallel
 * engine.  Per iteration: for each cluster j, center terms -> block tree of
 * numerators -> linear sum of partials, same for denominators; membership
 * map; objective terms -> tree -> linear sum; host max-abs delta.  Its
 * results are bit-identical for any worker count (parallel.py:1-11), so the
 * map phases may be split over OpenMP threads without changing a bit.
 */
/* Split [0, total) into one contiguous chunk per OpenMP thread (parallel.py:106-111). */
static void chunk_of(int64_t total, int64_t *lo, int64_t *hi) {
#ifdef _OPENMP
    int nt = omp_get_num_threads(), t = omp_get_thread_num();
#else
    int nt = 1, t = 0;
#endif
    int64_t step = (total + nt - 1) / nt;
    *lo = (int64_t)t * step;
    *hi = *lo + step < total ? *lo + step : total;
    if (*lo > total) *lo = total;
}

#define PAR_RANGES(total, call)                       \
    _Pragma("omp parallel") {                         \
        int64_t lo, hi;                               \
        chunk_of((total), &lo, &hi);                  \
        if (lo < hi) call;                            \
    }

int64_t oracle_iterate_parallel(const double *x, double *u, int64_t n, int64_t c, double m,
                                double epsilon, int64_t max_iters, int64_t block_size,
                                double *v_out, double *trace, int64_t *iterations,
                                int32_t *converged) {
    int64_t span = 2 * block_size;
    int64_t nblocks = (n + span - 1) / span;
    double *u_next = (double *)malloc((size_t)(n * c) * sizeof(double));
    double *num = (double *)malloc((size_t)n * sizeof(double));
    double *den = (double *)malloc((size_t)n * sizeof(double));
    double *terms = (double *)malloc((size_t)n * sizeof(double));
    double *partials = (double *)malloc((size_t)nblocks * sizeof(double));
    double *cur = u, *nxt = u_next;
    int64_t status = 0;
    *iterations = 0;
    *converged = 0;
    if (!u_next || !num || !den || !terms || !partials) { status = -1; goto out; }
    for (int64_t it = 0; it < max_iters; it++) {
        for (int64_t j = 0; j < c; j++) {
            PAR_RANGES(n, oracle_center_terms_range(x, cur, num, den, c, j, m, lo, hi))
            PAR_RANGES(nblocks, oracle_block_reduce_range(num, partials, n, block_size, lo, hi))
            double num_sum = oracle_linear_sum(partials, nblocks);
            PAR_RANGES(nblocks, oracle_block_reduce_range(den, partials, n, block_size, lo, hi))
            double den_sum = oracle_linear_sum(partials, nblocks);
            if (den_sum == 0.0) { status = 1 + j; goto out; }
            v_out[j] = num_sum / den_sum;
        }
        PAR_RANGES(n, oracle_update_membership_range(x, v_out, nxt, c, m, lo, hi))
        PAR_RANGES(n, oracle_objective_terms_range(x, nxt, v_out, terms, c, m, lo, hi))
        PAR_RANGES(nblocks, oracle_block_reduce_range(terms, partials, n, block_size, lo, hi))
        trace[it] = oracle_linear_sum(partials, nblocks);
        double delta = oracle_max_abs_diff(cur, nxt, 0, n * c);
        g_deltas[0] = g_deltas[1]; g_deltas[1] = delta;
        double *t = cur; cur = nxt; nxt = t;
        *iterations += 1;
        if (delta < epsilon) { *converged = 1; break; }
    }
out:
    if (cur != u) memcpy(u, cur, (size_t)(n * c) * sizeof(double));
    free(u_next); free(num); free(den); free(terms); free(partials);
    return status;
}
