/*
 * oracle.c — TEST INFRASTRUCTURE ONLY.  Plain, slow, obviously-correct fp64
 * reference for the time-iterated linear stencil of arXiv 2103.09235.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this file's library.  It shares no code,
 * header, table or helper with the CUDA path (paper_2103_09235_b200/csrc).
 *
 * What it computes (§1 Introduction): "The value of one point at
 * time t is a weighted sum of itself and its neighboring points at the
 * previous time.  The naive implementation for a d-dimensional stencil
 * contains d+1 loops where the time dimension is traversed in the outmost
 * loop and all grid points are updated in inner loops."
 *
 *   u^{t+1}[p] = sum_j w_j * u^t[p + o_j]          (correlation form: the
 *                                                   index v_{i+t} of Eq.4,
 *                                                   PAPER.md:385)
 *
 * with two arrays, odd and even time ("implemented with two
 * arrays").  Boundary (the paper is silent; reading R1, from
 * BASELINE.json north_star "fixed Dirichlet halo = u0"): the r-wide ring
 * around the interior holds u0 and is never written (FIXED).  PERIODIC
 * (reading R1, used only for the Fourier self-check) refills the ring by
 * wrap-around from the interior before every step.
 *
 * Accumulation order: taps in the order given (canonical: lexicographic
 * offsets, slowest axis outermost — reading R4), acc = acc + w*u, no FMA
 * contraction (compiled with -ffp-contract=off), so results are
 * bit-reproducible and independent of the OpenMP thread count (threads only
 * split the outermost spatial loop).
 *
 * Layout: the padded frame prod(N_a + 2r), row-major, slowest axis first,
 * x unit stride (SURVEY §8(a) a4 "row-major padded arrays").
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_FIXED 0
#define ORACLE_PERIODIC 1

static int64_t imod(int64_t a, int64_t n) { int64_t m = a % n; return m < 0 ? m + n : m; }

/* PERIODIC: copy interior values into the ring by wrap-around (reading R1). */
static void fill_periodic_ring(int nd, const int64_t *N, int r, double *A) {
    int64_t P[3] = {1, 1, 1}, n3[3] = {1, 1, 1};
    int off = 3 - nd;
    for (int a = 0; a < nd; ++a) { P[off + a] = N[a] + 2 * r; n3[off + a] = N[a]; }
    int rr[3] = {0, 0, 0};
    for (int a = 0; a < nd; ++a) rr[off + a] = r;
    for (int64_t z = 0; z < P[0]; ++z)
        for (int64_t y = 0; y < P[1]; ++y)
            for (int64_t x = 0; x < P[2]; ++x) {
                int64_t iz = z - rr[0], iy = y - rr[1], ix = x - rr[2];
                int inside = iz >= 0 && iz < n3[0] && iy >= 0 && iy < n3[1] && ix >= 0 && ix < n3[2];
                if (inside) continue;
                int64_t sz = imod(iz, n3[0]) + rr[0], sy = imod(iy, n3[1]) + rr[1], sx = imod(ix, n3[2]) + rr[2];
                A[(z * P[1] + y) * P[2] + x] = A[(sz * P[1] + sy) * P[2] + sx];
            }
}

/*
 * oracle_run: T naive steps.  u0 and out are padded frames of
 * prod(dims[a] + 2r) doubles.  offsets: ntaps*nd ints (slowest axis first).
 * Returns 0 on success, <0 on bad arguments.
 */
int oracle_run(int nd, const int64_t *dims, int r, int ntaps, const int *offsets,
               const double *w, int boundary, const double *u0, int64_t T,
               double *out, int nthreads) {
    if (nd < 1 || nd > 3 || r < 1 || ntaps < 1 || T < 0) return -1;
    int64_t P[3] = {1, 1, 1}, N[3] = {1, 1, 1};
    int off = 3 - nd;
    for (int a = 0; a < nd; ++a) {
        if (dims[a] < 1) return -1;
        P[off + a] = dims[a] + 2 * r;
        N[off + a] = dims[a];
    }
    int R3[3] = {0, 0, 0};
    for (int a = 0; a < nd; ++a) R3[off + a] = r;
    int64_t total = P[0] * P[1] * P[2];
    /* linear offset of every tap */
    int64_t *lin = (int64_t *)malloc(sizeof(int64_t) * ntaps);
    if (!lin) return -2;
    for (int j = 0; j < ntaps; ++j) {
        int64_t o3[3] = {0, 0, 0};
        for (int a = 0; a < nd; ++a) {
            int o = offsets[j * nd + a];
            if (o < -r || o > r) { free(lin); return -1; }
            o3[off + a] = o;
        }
        lin[j] = (o3[0] * P[1] + o3[1]) * P[2] + o3[2];
    }
    double *A = (double *)malloc(sizeof(double) * total);
    double *B = (double *)malloc(sizeof(double) * total);
    if (!A || !B) { free(lin); free(A); free(B); return -2; }
    memcpy(A, u0, sizeof(double) * total);
    memcpy(B, u0, sizeof(double) * total);     /* both arrays carry the same ring */
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    for (int64_t t = 0; t < T; ++t) {
        if (boundary == ORACLE_PERIODIC) fill_periodic_ring(nd, dims, r, A);
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
        for (int64_t z = 0; z < N[0]; ++z)
            for (int64_t y = 0; y < N[1]; ++y)
                for (int64_t x = 0; x < N[2]; ++x) {
                    int64_t p = ((z + R3[0]) * P[1] + (y + R3[1])) * P[2] + (x + R3[2]);
                    double acc = 0.0;
                    for (int j = 0; j < ntaps; ++j) acc = acc + w[j] * A[p + lin[j]];
                    B[p] = acc;
                }
        double *tmp = A; A = B; B = tmp;           /* Jacobi swap */
    }
    if (boundary == ORACLE_PERIODIC) fill_periodic_ring(nd, dims, r, A);
    memcpy(out, A, sizeof(double) * total);
    free(A); free(B); free(lin);
    return 0;
}

/*
 * oracle_run_cone: the same T FIXED steps, but step t (1-based) only updates
 * the interior points within (T - t) * r of the box [blo, bhi) (interior
 * coordinates).  Those are exactly the points the box's values after T steps
 * depend on, and each of them is computed with the same arithmetic as in
 * oracle_run, so the box's values are bit-identical to a full run.  Used on
 * dependency-cone windows of the full-size configurations.
 */
int oracle_run_cone(int nd, const int64_t *dims, int r, int ntaps, const int *offsets,
                    const double *w, const double *u0, int64_t T, const int64_t *blo,
                    const int64_t *bhi, double *out, int nthreads) {
    if (nd < 1 || nd > 3 || r < 1 || ntaps < 1 || T < 0) return -1;
    int64_t P[3] = {1, 1, 1}, N[3] = {1, 1, 1}, lo3[3] = {0, 0, 0}, hi3[3] = {1, 1, 1};
    int off = 3 - nd;
    for (int a = 0; a < nd; ++a) {
        if (dims[a] < 1) return -1;
        P[off + a] = dims[a] + 2 * r;
        N[off + a] = dims[a];
        lo3[off + a] = blo[a];
        hi3[off + a] = bhi[a];
    }
    int R3[3] = {0, 0, 0};
    for (int a = 0; a < nd; ++a) R3[off + a] = r;
    int64_t total = P[0] * P[1] * P[2];
    int64_t *lin = (int64_t *)malloc(sizeof(int64_t) * ntaps);
    if (!lin) return -2;
    for (int j = 0; j < ntaps; ++j) {
        int64_t o3[3] = {0, 0, 0};
        for (int a = 0; a < nd; ++a) o3[off + a] = offsets[j * nd + a];
        lin[j] = (o3[0] * P[1] + o3[1]) * P[2] + o3[2];
    }
    double *A = (double *)malloc(sizeof(double) * total);
    double *B = (double *)malloc(sizeof(double) * total);
    if (!A || !B) { free(lin); free(A); free(B); return -2; }
    memcpy(A, u0, sizeof(double) * total);
    memcpy(B, u0, sizeof(double) * total);
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    for (int64_t t = 1; t <= T; ++t) {
        int64_t a0[3], a1[3];
        for (int a = 0; a < 3; ++a) {
            int64_t e = (a >= off) ? (T - t) * r : 0;
            a0[a] = lo3[a] - e < 0 ? 0 : lo3[a] - e;
            a1[a] = hi3[a] + e > N[a] ? N[a] : hi3[a] + e;
        }
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
        for (int64_t z = a0[0]; z < a1[0]; ++z)
            for (int64_t y = a0[1]; y < a1[1]; ++y)
                for (int64_t x = a0[2]; x < a1[2]; ++x) {
                    int64_t p = ((z + R3[0]) * P[1] + (y + R3[1])) * P[2] + (x + R3[2]);
                    double acc = 0.0;
                    for (int j = 0; j < ntaps; ++j) acc = acc + w[j] * A[p + lin[j]];
                    B[p] = acc;
                }
        double *tmp = A; A = B; B = tmp;
    }
    memcpy(out, A, sizeof(double) * total);
    free(A); free(B); free(lin);
    return 0;
}

/* Thread count the OpenMP runtime would use (for the bench's "cores"). */
int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
