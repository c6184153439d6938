/* C restatement of the reference block classification (TEST INFRASTRUCTURE ONLY).
 *
 * Restates /root/reference/pkg/src/mmplan/mask.py:
 *   materialize      mask.py:106-112
 *   _classify_pair   mask.py:132-165 (OR short-circuit, uniform FULL, exact count)
 *   block_workloads  mask.py:168-188
 * and balance.py:58-76 (lpt_distribute) for CPU-baseline timing.
 *
 * Built by oracle/Makefile into oracle/_build/libbam_oracle.so; loaded by
 * oracle/mask_ref.py via ctypes.  Never linked into the product library.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

/* Minimal parallel-for over [0, n) with an atomic work counter (no OpenMP in
 * this toolchain). */
typedef struct {
    int64_t n, next;
    void (*body)(void *ctx, int64_t i);
    void *ctx;
    pthread_mutex_t mu;
} pfor_t;

static void *pfor_worker(void *arg) {
    pfor_t *p = arg;
    for (;;) {
        pthread_mutex_lock(&p->mu);
        int64_t i = p->next++;
        pthread_mutex_unlock(&p->mu);
        if (i >= p->n) return NULL;
        p->body(p->ctx, i);
    }
}

static void parallel_for(int64_t n, int threads, void (*body)(void *, int64_t), void *ctx) {
    if (threads <= 0) threads = (int)sysconf(_SC_NPROCESSORS_ONLN);
    if (threads > 256) threads = 256;
    pfor_t p = {n, 0, body, ctx, PTHREAD_MUTEX_INITIALIZER};
    pthread_t tid[256];
    for (int t = 0; t < threads; ++t) pthread_create(&tid[t], NULL, pfor_worker, &p);
    for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
}

static inline int allowed(const int64_t *d, int64_t q, int64_t k) {
    int64_t dq = d[q], dk = d[k];
    if (dq & 1) return k <= q && (dq & dk) != 0;
    return dk == dq;
}

static uint8_t classify_pair(const int64_t *d, int64_t qlo, int64_t qhi, int64_t klo, int64_t khi) {
    int64_t qor = 0, kor = 0;
    for (int64_t q = qlo; q < qhi; ++q) qor |= d[q];
    for (int64_t k = klo; k < khi; ++k) kor |= d[k];
    if ((qor & kor) == 0) return 0;                       /* skip */
    int64_t q0 = d[qlo], k0 = d[klo];
    if (!(q0 & 1) && q0 == k0) {
        int uni = 1;
        for (int64_t q = qlo; q < qhi && uni; ++q) uni = d[q] == q0;
        for (int64_t k = klo; k < khi && uni; ++k) uni = d[k] == k0;
        if (uni) return 1;                                /* full */
    }
    int64_t cnt = 0;
    for (int64_t q = qlo; q < qhi; ++q)
        for (int64_t k = klo; k < khi; ++k) cnt += allowed(d, q, k);
    if (cnt == 0) return 0;
    if (cnt == (qhi - qlo) * (khi - klo)) return 1;
    return 2;                                             /* partial */
}

typedef struct { const int64_t *desc; int64_t T, bs, nb; uint8_t *classes; int64_t *W; } bw_ctx;

static void bw_row(void *vctx, int64_t b) {
    bw_ctx *c = vctx;
    int64_t qlo = b * c->bs, qhi = qlo + c->bs < c->T ? qlo + c->bs : c->T, w = 0;
    for (int64_t k = 0; k < c->nb; ++k) {
        int64_t klo = k * c->bs, khi = klo + c->bs < c->T ? klo + c->bs : c->T;
        uint8_t cls = classify_pair(c->desc, qlo, qhi, klo, khi);
        c->classes[b * c->nb + k] = cls;
        w += cls != 0;
    }
    c->W[b] = w;
}

int oracle_block_workloads(const int64_t *desc, int64_t T, int64_t bs, uint8_t *classes,
                           int64_t *W, int threads) {
    if (bs < 1 || T < 1) return 1;
    bw_ctx c = {desc, T, bs, (T + bs - 1) / bs, classes, W};
    parallel_for(c.nb, threads, bw_row, &c);
    return 0;
}

typedef struct { const int64_t *desc; int64_t T; int64_t *rows; } ca_ctx;

static void ca_chunk(void *vctx, int64_t i) {
    ca_ctx *c = vctx;
    int64_t lo = i * 256, hi = lo + 256 < c->T ? lo + 256 : c->T, s = 0;
    for (int64_t q = lo; q < hi; ++q)
        for (int64_t k = 0; k < c->T; ++k) s += allowed(c->desc, q, k);
    c->rows[i] = s;
}

int64_t oracle_count_allowed(const int64_t *desc, int64_t T, int threads) {
    int64_t nchunk = (T + 255) / 256, total = 0;
    ca_ctx c = {desc, T, calloc(nchunk, sizeof(int64_t))};
    parallel_for(nchunk, threads, ca_chunk, &c);
    for (int64_t i = 0; i < nchunk; ++i) total += c.rows[i];
    free(c.rows);
    return total;
}

/* balance.py:58-76: blocks by (-W, id); each to argmin (load, gpu). */
typedef struct { int64_t w; int64_t id; } item_t;
static int cmp_item(const void *a, const void *b) {
    const item_t *x = a, *y = b;
    if (x->w != y->w) return x->w > y->w ? -1 : 1;
    return x->id < y->id ? -1 : (x->id > y->id);
}

int oracle_lpt(const int64_t *w, int64_t n, int32_t G, int32_t *owner, int64_t *loads) {
    if (G < 1 || n < 1) return 1;
    item_t *it = malloc(sizeof(item_t) * n);
    for (int64_t i = 0; i < n; ++i) { it[i].w = w[i]; it[i].id = i; }
    qsort(it, n, sizeof(item_t), cmp_item);
    memset(loads, 0, sizeof(int64_t) * G);
    for (int64_t i = 0; i < n; ++i) {
        int32_t g = 0;
        for (int32_t h = 1; h < G; ++h) if (loads[h] < loads[g]) g = h;
        owner[it[i].id] = g;
        loads[g] += it[i].w;
    }
    free(it);
    return 0;
}
