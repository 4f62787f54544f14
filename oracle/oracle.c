/*
 * oracle/oracle.c -- plain, slow, obviously-correct fp64 reference for the
 * HeteGen offloaded linear.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code with the product (paper_2403_01164_b200/csrc): no headers, no
 * helpers, no tables.  The product must never call it.
 *
 * What it computes ("plain definition"):
 *     y[b][n] = sum_{k<K} x[b][k] * W[n][k]  (+ bias[n])
 * in IEEE fp64 over the bf16-decoded inputs, k ascending.  This is the dense
 * product the paper's column split reproduces exactly: HeteGen partitions "the
 * weight's dimensions" between CPU and GPU (Sec. 3.1) and
 * concatenates the partial outputs (Sec. 4.2), so every output
 * element is one ordinary dot product.  bf16 x bf16 products are exact in
 * fp64, so the only rounding is the fp64 summation.
 *
 * Threads only split the OUTPUT ROWS n among workers; each dot product is the
 * same loop in the same order whatever the thread count.
 */
#include <stdint.h>
#include <string.h>
#include <pthread.h>

/* bf16 bit pattern -> value: the 16 bits are the top half of an IEEE float32. */
static double bf16_value(uint16_t h) {
    uint32_t u = ((uint32_t)h) << 16;
    float f;
    memcpy(&f, &u, 4);
    return (double)f;
}

typedef struct {
    const uint16_t *x;
    const uint16_t *W;
    const float *bias;
    double *y;
    const int64_t *rows; /* NULL: rows n0..n1-1 of W; else rows[i] for i in n0..n1-1 */
    int B;
    int64_t N_out, K, n0, n1;
} job_t;

static void *dot_rows(void *p) {
    job_t *j = (job_t *)p;
    for (int64_t i = j->n0; i < j->n1; ++i) {
        int64_t n = j->rows ? j->rows[i] : i;
        for (int b = 0; b < j->B; ++b) {
            double acc = 0.0;
            for (int64_t k = 0; k < j->K; ++k)
                acc += bf16_value(j->x[(int64_t)b * j->K + k]) * bf16_value(j->W[n * j->K + k]);
            if (j->bias) acc += (double)j->bias[n];
            j->y[(int64_t)b * j->N_out + i] = acc;
        }
    }
    return 0;
}

static void run(job_t base, int64_t count, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 512) nthreads = 512;
    if (count < nthreads) nthreads = count > 0 ? (int)count : 1;
    pthread_t th[512];
    job_t jobs[512];
    for (int t = 0; t < nthreads; ++t) {
        jobs[t] = base;
        jobs[t].n0 = count * t / nthreads;
        jobs[t].n1 = count * (t + 1) / nthreads;
    }
    for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], 0, dot_rows, &jobs[t]);
    dot_rows(&jobs[0]);
    for (int t = 1; t < nthreads; ++t) pthread_join(th[t], 0);
}

/* y[B][N] = x[B][K] . W[N][K]^T (+ bias[N]); bias may be NULL. */
void orc_linear(const uint16_t *x, int B, int64_t N, int64_t K, const uint16_t *W,
                const float *bias, double *y, int nthreads) {
    job_t j = {x, W, bias, y, 0, B, N, K, 0, N};
    run(j, N, nthreads);
}

/* Sampled outputs: y[B][nrows] for W rows rows[0..nrows) (full-size parity). */
void orc_linear_rows(const uint16_t *x, int B, int64_t K, const uint16_t *W, const float *bias,
                     const int64_t *rows, int64_t nrows, double *y, int nthreads) {
    job_t j = {x, W, bias, y, rows, B, nrows, K, 0, nrows};
    run(j, nrows, nthreads);
}
