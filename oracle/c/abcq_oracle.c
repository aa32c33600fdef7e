/*
 * abcq_oracle.c -- C restatement of the reference LUT GEMV (CPU) --
 * TEST / BASELINE INFRASTRUCTURE ONLY (never linked into the product).
 *
 * Restates, for the chunk-aligned case (group_size % 8 == 0 or one group):
 *   LookupTable.build        /root/reference/pkg/src/anybcq/gemv.py:67-81
 *   _lut_kernel              gemv.py:84-95  (f32 group sums, f32 alpha*s,
 *                                            f64 row accumulator)
 *   GemvEngine.lut           gemv.py:188-222 (row threads, asymmetric term)
 *   thread policy            parallel.py:14-30 (contiguous row chunks)
 * Used as bench.py's cpu_baseline / `--impl reference` arm ("port") and
 * checked against the numpy oracle and the reference's golden outputs.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    const uint8_t* idx; /* plane bytes: (planes, rows, row_bytes) */
    int64_t row_bytes;
    int64_t plane_bytes;
    const float* table; /* (chunks, 256) */
    const float* alpha; /* (p, rows, G) */
    const int64_t* clo;
    const int64_t* chi;
    int G, rows, p;
    int lo, hi;
    double* y;
} job_t;

static void* run_rows(void* arg) {
    const job_t* j = (const job_t*)arg;
    for (int n = j->lo; n < j->hi; ++n) {
        double acc = 0.0;
        for (int i = 0; i < j->p; ++i) {
            const uint8_t* row = j->idx + (int64_t)i * j->plane_bytes + (int64_t)n * j->row_bytes;
            const float* a = j->alpha + ((int64_t)i * j->rows + n) * j->G;
            for (int g = 0; g < j->G; ++g) {
                float s = 0.0f;
                for (int64_t c = j->clo[g]; c < j->chi[g]; ++c) s += j->table[c * 256 + row[c]];
                float prod = a[g] * s; /* numba: f32 * f32 -> f32 */
                acc += (double)prod;
            }
        }
        j->y[n] = acc;
    }
    return NULL;
}

/* table (chunks, 256) f32 by doubling over ascending bit j (gemv.py:76-80) */
void abcq_oracle_lut_build8(const double* x, int cols, float* table) {
    const int chunks = (cols + 7) / 8;
    for (int c = 0; c < chunks; ++c) {
        float* t = table + (int64_t)c * 256;
        t[0] = 0.0f;
        int n = 1;
        for (int j = 0; j < 8; ++j) {
            const int k = c * 8 + j;
            const float xj = k < cols ? (float)x[k] : 0.0f;
            for (int u = n - 1; u >= 0; --u) { /* [t - xj | t + xj] */
                const float v = t[u];
                t[u] = v - xj;
                t[u + n] = v + xj;
            }
            n <<= 1;
        }
    }
}

/* returns 0, or -1 when the group size is not chunk aligned */
int abcq_oracle_lut_gemv(const uint32_t* words, int planes, int rows, int cols, int group_size,
                         const float* alpha, const float* offset, int p, const double* x, double* y,
                         int threads) {
    const int G = (cols + group_size - 1) / group_size;
    const int chunks = (cols + 7) / 8;
    if (!(group_size % 8 == 0 || G == 1) || p < 1 || p > planes) return -1;
    const int wpr = (cols + 31) / 32;
    float* table = (float*)malloc(sizeof(float) * (size_t)chunks * 256);
    int64_t* clo = (int64_t*)malloc(sizeof(int64_t) * G);
    int64_t* chi = (int64_t*)malloc(sizeof(int64_t) * G);
    abcq_oracle_lut_build8(x, cols, table);
    const int per = G > 1 ? group_size / 8 : chunks;
    for (int g = 0; g < G; ++g) {
        clo[g] = (int64_t)g * per;
        chi[g] = g < G - 1 ? (int64_t)(g + 1) * per : chunks;
        if (chi[g] > chunks) chi[g] = chunks;
    }
    if (threads < 1) threads = 1;
    if (threads > rows) threads = rows;
    if (threads > 1 && rows < 2 * threads) threads = 1; /* gemv.py:199 */
    const int step = (rows + threads - 1) / threads;
    job_t* jobs = (job_t*)calloc(threads, sizeof(job_t));
    pthread_t* tids = (pthread_t*)calloc(threads, sizeof(pthread_t));
    int nj = 0;
    for (int lo = 0; lo < rows; lo += step, ++nj) {
        job_t* j = &jobs[nj];
        j->idx = (const uint8_t*)words;
        j->row_bytes = (int64_t)wpr * 4;
        j->plane_bytes = (int64_t)rows * wpr * 4;
        j->table = table;
        j->alpha = alpha;
        j->clo = clo;
        j->chi = chi;
        j->G = G;
        j->rows = rows;
        j->p = p;
        j->lo = lo;
        j->hi = lo + step < rows ? lo + step : rows;
        j->y = y;
    }
    if (nj == 1) {
        run_rows(&jobs[0]);
    } else {
        for (int t = 0; t < nj; ++t) pthread_create(&tids[t], NULL, run_rows, &jobs[t]);
        for (int t = 0; t < nj; ++t) pthread_join(tids[t], NULL);
    }
    if (offset) { /* y += offset(f64) @ gx(f64)  (gemv.py:217-221) */
        double* gx = (double*)calloc(G, sizeof(double));
        for (int g = 0; g < G; ++g) {
            const int lo = g * group_size, hi = lo + group_size < cols ? lo + group_size : cols;
            double s = 0.0;
            for (int k = lo; k < hi; ++k) s += x[k];
            gx[g] = s;
        }
        for (int n = 0; n < rows; ++n) {
            double s = 0.0;
            for (int g = 0; g < G; ++g) s += (double)offset[(int64_t)n * G + g] * gx[g];
            y[n] += s;
        }
        free(gx);
    }
    free(jobs);
    free(tids);
    free(table);
    free(clo);
    free(chi);
    return 0;
}
