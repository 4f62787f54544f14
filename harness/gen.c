/*
 * harness/gen.c -- seeded, counter-based synthetic input generator.
 *
 * TEST/BENCH INFRASTRUCTURE, NOT THE METHOD.  This module holds none of the
 * method's arithmetic (no GEMV, no partition, no cost model).  It is the one
 * piece shared by the oracle (oracle/) and the CUDA path's tests and bench, so
 * both sides see identical input bits.
 *
 * Recipe (SURVEY.md 8(d) "Generator"):
 *   key   = splitmix64(seed ^ splitmix64(tensor_id))
 *   u_i   = (splitmix64(key + i) >> 11) * 2^-53          in [0, 1)
 *   value = (2 u_i - 1) * a                               in double
 *   bf16  = RNE_bf16( RNE_f32(value) )                    (two explicit roundings)
 * Integer mode (exactness tests): value = floor(u_i * (2m+1)) - m, in [-m, m].
 *
 * gen.py implements the same recipe in numpy; tests check the two agree.
 */
#include <stdint.h>
#include <string.h>
#include <math.h>
#include <pthread.h>

static inline uint64_t sm64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

uint64_t hgen_splitmix64(uint64_t z) { return sm64(z); }

uint64_t hgen_key(uint64_t seed, uint64_t tensor_id) { return sm64(seed ^ sm64(tensor_id)); }

static inline uint16_t f32_to_bf16_rne(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    if ((u & 0x7f800000u) == 0x7f800000u) return (uint16_t)(u >> 16);  /* inf/nan (never produced) */
    u += 0x7fffu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}

typedef struct {
    uint64_t key, start, end;
    double a;
    int mode;      /* 0 = uniform(+-a), 1 = integer [-m, m] with m = (int)a */
    uint16_t *out;
    float *out_f32;
} job_t;

static void *run(void *p) {
    job_t *j = (job_t *)p;
    const double two53 = 1.0 / 9007199254740992.0;
    for (uint64_t i = j->start; i < j->end; ++i) {
        double u = (double)(sm64(j->key + i) >> 11) * two53;
        double v;
        if (j->mode == 0) {
            v = (2.0 * u - 1.0) * j->a;
        } else {
            int64_t m = (int64_t)j->a;
            v = floor(u * (double)(2 * m + 1)) - (double)m;
        }
        float f = (float)v;
        if (j->out) j->out[i] = f32_to_bf16_rne(f);
        if (j->out_f32) j->out_f32[i] = f;
    }
    return 0;
}

static void launch(uint64_t key, uint64_t n, double a, int mode, uint16_t *out, float *out_f32,
                   int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    if (n < (1u << 20)) nthreads = 1;
    pthread_t th[256];
    job_t jobs[256];
    for (int t = 0; t < nthreads; ++t) {
        jobs[t].key = key;
        jobs[t].start = n * (uint64_t)t / (uint64_t)nthreads;
        jobs[t].end = n * (uint64_t)(t + 1) / (uint64_t)nthreads;
        jobs[t].a = a;
        jobs[t].mode = mode;
        jobs[t].out = out;
        jobs[t].out_f32 = out_f32;
    }
    for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], 0, run, &jobs[t]);
    run(&jobs[0]);
    for (int t = 1; t < nthreads; ++t) pthread_join(th[t], 0);
}

/* n bf16 values uniform in (-a, a); element i of the tensor is always the same
 * value whatever n or offset, so slices can be generated independently. */
void hgen_uniform_bf16(uint64_t seed, uint64_t tensor_id, uint64_t offset, uint64_t n, double a,
                       uint16_t *out, int nthreads) {
    launch(hgen_key(seed, tensor_id) + offset, n, a, 0, out, 0, nthreads);
}

void hgen_int_bf16(uint64_t seed, uint64_t tensor_id, uint64_t offset, uint64_t n, int m,
                   uint16_t *out, int nthreads) {
    launch(hgen_key(seed, tensor_id) + offset, n, (double)m, 1, out, 0, nthreads);
}

void hgen_uniform_f32(uint64_t seed, uint64_t tensor_id, uint64_t offset, uint64_t n, double a,
                      float *out, int nthreads) {
    launch(hgen_key(seed, tensor_id) + offset, n, a, 0, 0, out, nthreads);
}
