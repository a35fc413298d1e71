/*
 * polar_oracle.c -- CPU restatement of the reference list decoder.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity oracle for the CUDA
 * decoder: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load it.  The product decode path never calls it.
 *
 * It restates, step for step, polaris.listdec.ListDecoder
 * (/root/reference/pkg/src/polaris/listdec.py) on top of plain C:
 *   - _RowPool refcounted rows, alloc/share/release/detach   listdec.py:103-143
 *   - _Path (pm, alpha row per stage, beta row per slot, root) listdec.py:146-153
 *   - _fork / _drop / _new_root_path                         listdec.py:196-214
 *   - _run op loop (F/G/Combine/leaf)                        listdec.py:310-335
 *   - _leaf (Rate0 / Rep / Rate1 / SPC)                      listdec.py:337-395
 *   - select_candidates (two-pass bounded heap)              listdec.py:63-100
 *   - _materialize                                           listdec.py:397-434
 *   - decode_paths / decode (CRC-aided pick)                 listdec.py:275-308
 * with the numpy numerics the reference inherits:
 *   - float32 `sum(axis=1)` = numpy pairwise summation (8 strided
 *     accumulators up to 128 elements, halving above)        listdec.py:341,348-350
 *   - stable argsort (lowest index wins ties)                listdec.py:362,375
 *   - path metrics and candidate deltas in float64 (Python floats)
 * and the f/g kernels of kernels.py:39-56.  The CRC check runs the bitwise
 * shift register of codes.py:79-118 directly (independent of the syndrome
 * tables the GPU path uses).
 *
 * int8 mode: identical semantics fed integer LLRs,
 * with G saturated to [-127, 127]; all sums are then exact integers.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "polar_oracle.h"

enum { K_F = 0, K_G = 1, K_COMB = 2, K_R0 = 3, K_R1 = 4, K_REP = 5, K_SPC = 6 };

/* ------------------------------------------------------------ numerics */

/* numpy pairwise_sum for float32 (numpy/_core/src/umath/loops_utils.h.src) */
static float pw_sum(const float *a, long n) {
    if (n < 8) {
        float r = 0.0f;
        for (long i = 0; i < n; i++) r += a[i];
        return r;
    }
    if (n <= 128) {
        float r[8];
        for (int j = 0; j < 8; j++) r[j] = a[j];
        long i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        float res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    }
    long n2 = n / 2;
    n2 -= n2 % 8;
    return pw_sum(a, n2) + pw_sum(a + n2, n - n2);
}

static float f_fn(float a, float b) {            /* kernels.py:39-48 */
    float sa = (a > 0.0f) - (a < 0.0f), sb = (b > 0.0f) - (b < 0.0f);
    return sa * sb * fminf(fabsf(a), fabsf(b));
}

/* ------------------------------------------------------------ row pools */

typedef struct {
    int rows, width, esize;
    unsigned char *data;
    int *refs;
    int *free_list;
    int n_free;
} pool_t;

static int pool_init(pool_t *p, int rows, int width, int esize) {
    p->rows = rows; p->width = width; p->esize = esize;
    p->data = (unsigned char *)calloc((size_t)rows * width, esize);
    p->refs = (int *)calloc(rows, sizeof(int));
    p->free_list = (int *)malloc(sizeof(int) * rows);
    return (p->data && p->refs && p->free_list) ? 0 : -1;
}
static void pool_free(pool_t *p) { free(p->data); free(p->refs); free(p->free_list); }
static void pool_reset(pool_t *p) {          /* listdec.py:141-143 */
    memset(p->refs, 0, sizeof(int) * p->rows);
    for (int i = 0; i < p->rows; i++) p->free_list[i] = p->rows - 1 - i;
    p->n_free = p->rows;
}
static int pool_alloc(pool_t *p) {           /* listdec.py:117-122 */
    if (p->n_free == 0) return -1;
    int row = p->free_list[--p->n_free];
    p->refs[row] = 1;
    return row;
}
static void pool_share(pool_t *p, int row) { p->refs[row]++; }
static void pool_release(pool_t *p, int row) {
    if (--p->refs[row] == 0) p->free_list[p->n_free++] = row;
}
static int pool_detach(pool_t *p, int row) { /* listdec.py:133-139 */
    if (p->refs[row] == 1) return row;
    p->refs[row]--;
    return pool_alloc(p);
}
static void *pool_row(pool_t *p, int row) { return p->data + (size_t)row * p->width * p->esize; }

/* ------------------------------------------------------------ decoder */

typedef struct {
    double pm;
    int *alpha;  /* [n] */
    int *beta;   /* [2n] */
    int root;
} path_t;

typedef struct {
    const oc_code *code;
    const int32_t *ops;
    int n_ops, L, int8_mode, n, N;
    pool_t *apool, *bpool, rpool;
    float *channel;
    /* path storage: up to 2L live path records */
    path_t *paths, *next_paths;
    int *idx_store;
    /* scratch */
    float *tmp_a, *tmp_b;
    double *cand_delta;     /* [L][8] */
    int *cand_flip;         /* [L][8] bitmask over lrb slots */
    int *lrb;               /* [L][4] */
    int *ncand;
    int *ones;              /* rep decision order: 1 if ones-first */
    int *chosen_s, *chosen_c;
    unsigned char *hard;    /* [L][N] */
    double *heap_m; int *heap_seq, *heap_s, *heap_c;
    double *st_m; int *st_s, *st_c;
    int *info_pos;
    int err;
} dec_t;

static const int SPC_PAIRS[7][4] = {
    {0, 1, -1, -1}, {0, 2, -1, -1}, {0, 3, -1, -1}, {1, 2, -1, -1},
    {1, 3, -1, -1}, {2, 3, -1, -1}, {0, 1, 2, 3}};

static int dec_init(dec_t *d, const oc_code *code, const int32_t *ops, int n_ops,
                    int L, int int8_mode) {
    memset(d, 0, sizeof(*d));
    d->code = code; d->ops = ops; d->n_ops = n_ops; d->L = L; d->int8_mode = int8_mode;
    d->N = code->N; d->n = 0;
    while ((1 << d->n) < d->N) d->n++;
    int n = d->n, rows = 2 * L;
    d->apool = (pool_t *)calloc(n > 0 ? n : 1, sizeof(pool_t));
    d->bpool = (pool_t *)calloc(2 * n > 0 ? 2 * n : 1, sizeof(pool_t));
    for (int s = 0; s < n; s++) pool_init(&d->apool[s], rows, 1 << s, sizeof(float));
    for (int i = 0; i < 2 * n; i++) pool_init(&d->bpool[i], rows, 1 << (i / 2), 1);
    pool_init(&d->rpool, rows, d->N, 1);
    d->channel = (float *)malloc(sizeof(float) * d->N);
    int maxp = 2 * L + 1;
    d->paths = (path_t *)calloc(maxp, sizeof(path_t));
    d->next_paths = (path_t *)calloc(maxp, sizeof(path_t));
    d->idx_store = (int *)calloc((size_t)2 * maxp * 3 * (n + 1), sizeof(int));
    for (int i = 0; i < maxp; i++) {
        d->paths[i].alpha = d->idx_store + (size_t)i * 3 * (n + 1);
        d->paths[i].beta = d->paths[i].alpha + (n + 1);
        d->next_paths[i].alpha = d->idx_store + (size_t)(maxp + i) * 3 * (n + 1);
        d->next_paths[i].beta = d->next_paths[i].alpha + (n + 1);
    }
    d->tmp_a = (float *)malloc(sizeof(float) * (size_t)L * d->N);
    d->tmp_b = (float *)malloc(sizeof(float) * (size_t)d->N);
    d->cand_delta = (double *)malloc(sizeof(double) * L * 8);
    d->cand_flip = (int *)malloc(sizeof(int) * L * 8);
    d->lrb = (int *)malloc(sizeof(int) * L * 4);
    d->ncand = (int *)malloc(sizeof(int) * L);
    d->ones = (int *)malloc(sizeof(int) * L);
    d->chosen_s = (int *)malloc(sizeof(int) * L * 8);
    d->chosen_c = (int *)malloc(sizeof(int) * L * 8);
    d->hard = (unsigned char *)malloc((size_t)L * d->N);
    d->heap_m = (double *)malloc(sizeof(double) * (L + 1));
    d->heap_seq = (int *)malloc(sizeof(int) * (L + 1));
    d->heap_s = (int *)malloc(sizeof(int) * (L + 1));
    d->heap_c = (int *)malloc(sizeof(int) * (L + 1));
    d->st_m = (double *)malloc(sizeof(double) * L * 8);
    d->st_s = (int *)malloc(sizeof(int) * L * 8);
    d->st_c = (int *)malloc(sizeof(int) * L * 8);
    d->info_pos = (int *)malloc(sizeof(int) * d->N);
    int c = 0;
    for (int i = 0; i < d->N; i++) if (!code->frozen[i]) d->info_pos[c++] = i;
    return 0;
}

static void dec_free(dec_t *d) {
    for (int s = 0; s < d->n; s++) pool_free(&d->apool[s]);
    for (int i = 0; i < 2 * d->n; i++) pool_free(&d->bpool[i]);
    pool_free(&d->rpool);
    free(d->apool); free(d->bpool); free(d->channel); free(d->paths); free(d->next_paths);
    free(d->idx_store); free(d->tmp_a); free(d->tmp_b); free(d->cand_delta);
    free(d->cand_flip); free(d->lrb); free(d->ncand); free(d->ones);
    free(d->chosen_s); free(d->chosen_c); free(d->hard); free(d->heap_m);
    free(d->heap_seq); free(d->heap_s); free(d->heap_c); free(d->st_m);
    free(d->st_s); free(d->st_c); free(d->info_pos);
}

static void copy_path(dec_t *d, path_t *dst, const path_t *src) {
    dst->pm = src->pm;
    memcpy(dst->alpha, src->alpha, sizeof(int) * d->n);
    memcpy(dst->beta, src->beta, sizeof(int) * 2 * d->n);
    dst->root = src->root;
}

static void fork_path(dec_t *d, path_t *dst, const path_t *src) {   /* listdec.py:201-207 */
    for (int s = 0; s < d->n; s++) pool_share(&d->apool[s], src->alpha[s]);
    for (int i = 0; i < 2 * d->n; i++) pool_share(&d->bpool[i], src->beta[i]);
    pool_share(&d->rpool, src->root);
    copy_path(d, dst, src);
}

static void drop_path(dec_t *d, path_t *p) {                        /* listdec.py:209-214 */
    for (int s = 0; s < d->n; s++) pool_release(&d->apool[s], p->alpha[s]);
    for (int i = 0; i < 2 * d->n; i++) pool_release(&d->bpool[i], p->beta[i]);
    pool_release(&d->rpool, p->root);
}

/* alpha row of path p at a stage; the channel when the node is the root */
static const float *alpha_of(dec_t *d, const path_t *p, int stage, int size) {
    if (size == d->N) return d->channel;
    return (const float *)pool_row(&d->apool[stage], p->alpha[stage]);
}

static float *alpha_write(dec_t *d, path_t *p, int stage) {         /* listdec.py:226-236 */
    int row = pool_detach(&d->apool[stage], p->alpha[stage]);
    if (row < 0) { d->err = 1; row = 0; }
    p->alpha[stage] = row;
    return (float *)pool_row(&d->apool[stage], row);
}

static unsigned char *beta_write(dec_t *d, path_t *p, int size, int stage, int side) {
    /* listdec.py:245-271 */
    if (size == d->N) {
        int row = pool_detach(&d->rpool, p->root);
        if (row < 0) { d->err = 1; row = 0; }
        p->root = row;
        return (unsigned char *)pool_row(&d->rpool, row);
    }
    int slot = 2 * stage + side;
    int row = pool_detach(&d->bpool[slot], p->beta[slot]);
    if (row < 0) { d->err = 1; row = 0; }
    p->beta[slot] = row;
    return (unsigned char *)pool_row(&d->bpool[slot], row);
}

static const unsigned char *beta_of(dec_t *d, const path_t *p, int stage, int side) {
    int slot = 2 * stage + side;
    return (const unsigned char *)pool_row(&d->bpool[slot], p->beta[slot]);
}

/* ---------------------------------------------------- selection (63-100) */

/* heap ordered by (metric, -seq): root is the entry evicted first */
static int heap_less(dec_t *d, int a, int b) {
    if (d->heap_m[a] != d->heap_m[b]) return d->heap_m[a] < d->heap_m[b];
    return -d->heap_seq[a] < -d->heap_seq[b];
}
static void heap_swap(dec_t *d, int a, int b) {
    double m = d->heap_m[a]; d->heap_m[a] = d->heap_m[b]; d->heap_m[b] = m;
    int t = d->heap_seq[a]; d->heap_seq[a] = d->heap_seq[b]; d->heap_seq[b] = t;
    t = d->heap_s[a]; d->heap_s[a] = d->heap_s[b]; d->heap_s[b] = t;
    t = d->heap_c[a]; d->heap_c[a] = d->heap_c[b]; d->heap_c[b] = t;
}
static void heap_up(dec_t *d, int i) {
    while (i > 0) {
        int parent = (i - 1) / 2;
        if (heap_less(d, i, parent)) { heap_swap(d, i, parent); i = parent; }
        else break;
    }
}
static void heap_down(dec_t *d, int i, int size) {
    for (;;) {
        int l = 2 * i + 1, r = l + 1, m = i;
        if (l < size && heap_less(d, l, m)) m = l;
        if (r < size && heap_less(d, r, m)) m = r;
        if (m == i) return;
        heap_swap(d, i, m); i = m;
    }
}

/* returns the number of chosen (source, cand) pairs, in (source, cand) order */
static int select_candidates(dec_t *d, int P, const double *pm, int list_size) {
    /* pass 1: each source's most likely decision, then the deferred ones */
    int ns = 0;
    for (int s = 0; s < P; s++) {
        int C = d->ncand[s];
        d->st_m[ns] = pm[s] + d->cand_delta[s * 8 + 0]; d->st_s[ns] = s; d->st_c[ns] = 0; ns++;
        for (int c = 1; c < C; c++) {
            d->st_m[ns] = pm[s] + d->cand_delta[s * 8 + c]; d->st_s[ns] = s; d->st_c[ns] = c; ns++;
        }
    }
    /* pass 2: bounded heap; replace the strict minimum only */
    int hs = 0;
    for (int seq = 0; seq < ns; seq++) {
        if (hs < list_size) {
            d->heap_m[hs] = d->st_m[seq]; d->heap_seq[hs] = seq;
            d->heap_s[hs] = d->st_s[seq]; d->heap_c[hs] = d->st_c[seq];
            heap_up(d, hs); hs++;
        } else if (d->st_m[seq] > d->heap_m[0]) {
            d->heap_m[0] = d->st_m[seq]; d->heap_seq[0] = seq;
            d->heap_s[0] = d->st_s[seq]; d->heap_c[0] = d->st_c[seq];
            heap_down(d, 0, hs);
        }
    }
    /* sorted by seq ascending == (source, cand) order */
    int cnt = 0;
    for (int seq = 0; seq < ns && cnt < hs; seq++)
        for (int h = 0; h < hs; h++)
            if (d->heap_seq[h] == seq) {
                d->chosen_s[cnt] = d->heap_s[h]; d->chosen_c[cnt] = d->heap_c[h]; cnt++;
                break;
            }
    return cnt;
}

/* --------------------------------------------------- leaves (337-434) */

static int materialize(dec_t *d, const int32_t *op, int P, int has_hard) {
    int size = op[1], stage = op[2], side = op[3];
    double base[64];
    double *pm = base;
    double *pm_heap = NULL;
    if (P > 64) pm = pm_heap = (double *)malloc(sizeof(double) * P);
    for (int s = 0; s < P; s++) pm[s] = d->paths[s].pm;
    int nch = select_candidates(d, P, pm, d->L);
    int nsurv = 0, cursor = 0;
    for (int s = 0; s < P; s++) {
        int first = 1;
        path_t *src = &d->paths[s];
        while (cursor < nch && d->chosen_s[cursor] == s) {
            int c = d->chosen_c[cursor++];
            path_t *host = &d->next_paths[nsurv];
            if (first) { copy_path(d, host, src); first = 0; }   /* in place */
            else fork_path(d, host, src);
            host->pm = pm[s] + d->cand_delta[s * 8 + c];
            d->st_s[nsurv] = s; d->st_c[nsurv] = c;               /* reuse as picks */
            nsurv++;
        }
        if (first) drop_path(d, src);
    }
    if (P + nsurv > 2 * d->L) d->err = 2;                     /* listdec.py:419-420 */
    for (int t = 0; t < nsurv; t++) {
        int s = d->st_s[t], c = d->st_c[t];
        unsigned char *w = beta_write(d, &d->next_paths[t], size, stage, side);
        if (!has_hard) {
            /* repetition: cand order is ones-first or zeros-first */
            int is_ones = d->ones[s] ? (c == 0) : (c == 1);
            memset(w, is_ones ? 1 : 0, size);
        } else {
            memcpy(w, d->hard + (size_t)s * d->N, size);
            int mask = d->cand_flip[s * 8 + c];
            for (int j = 0; j < 4; j++)
                if (mask & (1 << j)) w[d->lrb[s * 4 + j]] ^= 1;
        }
    }
    /* swap path arrays */
    path_t *tmp = d->paths; d->paths = d->next_paths; d->next_paths = tmp;
    free(pm_heap);
    return nsurv;
}

/* stable k smallest of |a| (k <= 4): indices ascending by (|a|, index) */
static void stable_smallest(const float *a, int m, int k, int *idx, float *mag) {
    int cnt = 0;
    for (int i = 0; i < m; i++) {
        float v = fabsf(a[i]);
        int pos = cnt;
        while (pos > 0 && v < mag[pos - 1]) pos--;   /* strict: earlier index wins ties */
        if (pos >= k) continue;
        int last = cnt < k ? cnt : k - 1;
        for (int j = last; j > pos; j--) { mag[j] = mag[j - 1]; idx[j] = idx[j - 1]; }
        mag[pos] = v; idx[pos] = i;
        if (cnt < k) cnt++;
    }
}

static int run_leaf(dec_t *d, const int32_t *op, int P) {
    int kind = op[0], size = op[1], stage = op[2], side = op[3];
    float *buf = d->tmp_b;
    if (kind == K_R0) {                                        /* 340-346 */
        for (int t = 0; t < P; t++) {
            path_t *p = &d->paths[t];
            const float *a = alpha_of(d, p, stage, size);
            for (int i = 0; i < size; i++) buf[i] = fminf(a[i], 0.0f);
            p->pm += (double)pw_sum(buf, size);
        }
        for (int t = 0; t < P; t++)
            memset(beta_write(d, &d->paths[t], size, stage, side), 0, size);
        return P;
    }
    if (kind == K_REP || (kind == K_R1 && size == 1)) {       /* 347-359 */
        for (int t = 0; t < P; t++) {
            const float *a = alpha_of(d, &d->paths[t], stage, size);
            for (int i = 0; i < size; i++) buf[i] = fminf(a[i], 0.0f);
            double neg = (double)pw_sum(buf, size);
            for (int i = 0; i < size; i++) buf[i] = fmaxf(a[i], 0.0f);
            double pos = (double)pw_sum(buf, size);
            float tot = pw_sum(a, size);
            d->ncand[t] = 2;
            d->ones[t] = tot < 0.0f;
            if (d->ones[t]) { d->cand_delta[t * 8] = -pos; d->cand_delta[t * 8 + 1] = neg; }
            else { d->cand_delta[t * 8] = neg; d->cand_delta[t * 8 + 1] = -pos; }
        }
        return materialize(d, op, P, 0);
    }
    if (kind == K_R1) {                                        /* 360-372 */
        for (int t = 0; t < P; t++) {
            const float *a = alpha_of(d, &d->paths[t], stage, size);
            int idx[4]; float mag[4];
            stable_smallest(a, size, 2, idx, mag);
            double m1 = mag[0], m2 = mag[1];
            d->lrb[t * 4 + 0] = idx[0]; d->lrb[t * 4 + 1] = idx[1];
            d->ncand[t] = 4;
            d->cand_delta[t * 8 + 0] = 0.0; d->cand_flip[t * 8 + 0] = 0;
            d->cand_delta[t * 8 + 1] = -m1; d->cand_flip[t * 8 + 1] = 1;
            d->cand_delta[t * 8 + 2] = -m2; d->cand_flip[t * 8 + 2] = 2;
            d->cand_delta[t * 8 + 3] = -(m1 + m2); d->cand_flip[t * 8 + 3] = 3;
            unsigned char *h = d->hard + (size_t)t * d->N;
            for (int i = 0; i < size; i++) h[i] = a[i] < 0.0f;
        }
        return materialize(d, op, P, 1);
    }
    if (kind == K_SPC) {                                       /* 373-394 */
        for (int t = 0; t < P; t++) {
            const float *a = alpha_of(d, &d->paths[t], stage, size);
            int idx[4]; float mag[4];
            stable_smallest(a, size, 4, idx, mag);
            unsigned char *h = d->hard + (size_t)t * d->N;
            int par = 0;
            for (int i = 0; i < size; i++) { h[i] = a[i] < 0.0f; par ^= h[i]; }
            for (int j = 0; j < 4; j++) d->lrb[t * 4 + j] = idx[j];
            int ml = par ? 1 : 0;            /* bitmask over lrb slots */
            /* index-ascending order of the four lrb slots */
            int ord[4] = {0, 1, 2, 3};
            for (int x = 1; x < 4; x++)
                for (int y = x; y > 0 && idx[ord[y]] < idx[ord[y - 1]]; y--) {
                    int tt = ord[y]; ord[y] = ord[y - 1]; ord[y - 1] = tt;
                }
            int npairs = d->L != 2 ? 7 : 1;
            d->ncand[t] = 1 + npairs;
            for (int c = 0; c <= npairs; c++) {
                int net;
                if (c == 0) net = ml;
                else {
                    int pm_ = 0;
                    for (int j = 0; j < 4 && SPC_PAIRS[c - 1][j] >= 0; j++) pm_ |= 1 << SPC_PAIRS[c - 1][j];
                    net = pm_ ^ ml;
                }
                /* -sum(weight[i] for i in sorted(net)) in float64 */
                double acc = 0.0;
                int any = 0;
                for (int x = 0; x < 4; x++)
                    if (net & (1 << ord[x])) {
                        acc = any ? acc + (double)mag[ord[x]] : (double)mag[ord[x]];
                        any = 1;
                    }
                d->cand_delta[t * 8 + c] = any ? -acc : 0.0;
                d->cand_flip[t * 8 + c] = net;
            }
        }
        return materialize(d, op, P, 1);
    }
    d->err = 3;
    return P;
}

/* ------------------------------------------------------- finalisation */

static uint32_t rev_bits(uint32_t v, int w) {
    uint32_t r = 0;
    for (int i = 0; i < w; i++) { r = (r << 1) | (v & 1); v >>= 1; }
    return r;
}

/* codes.py:79-118 + 150-156 over u[info_positions] */
static int crc_ok_of(const dec_t *d, const unsigned char *u) {
    const oc_code *c = d->code;
    int w = c->crc_width;
    if (w == 0) return 0;
    int k = c->k;
    uint32_t reg;
    if (c->crc_reflect) {
        reg = rev_bits(c->crc_init, w);
        uint32_t rp = rev_bits(c->crc_poly, w);
        for (int i = 0; i < k; i++) {
            int b = u[d->info_pos[i]];
            reg = ((reg ^ (uint32_t)b) & 1u) ? (reg >> 1) ^ rp : reg >> 1;
        }
    } else {
        uint32_t mask = w == 32 ? 0xFFFFFFFFu : ((1u << w) - 1);
        reg = c->crc_init;
        for (int i = 0; i < k; i++) {
            int b = u[d->info_pos[i]];
            uint32_t top = (reg >> (w - 1)) & 1u;
            reg = (reg << 1) & mask;
            if (top ^ (uint32_t)b) reg ^= c->crc_poly;
        }
    }
    uint32_t val = reg ^ c->crc_xor_out;
    for (int j = 0; j < w; j++) {
        int bit = c->crc_reflect ? (val >> j) & 1 : (val >> (w - 1 - j)) & 1;
        if (bit != u[d->info_pos[k + j]]) return 0;
    }
    return 1;
}

static void polar_transform(unsigned char *x, int N) {          /* encode.py:29-53 */
    for (int h = 1; h < N; h <<= 1)
        for (int b = 0; b < N; b += 2 * h)
            for (int i = b; i < b + h; i++) x[i] ^= x[i + h];
}

/* decode one frame; returns number of surviving paths (<0 on error) */
static int decode_frame(dec_t *d, const float *llr) {
    int n = d->n, N = d->N;
    for (int s = 0; s < n; s++) pool_reset(&d->apool[s]);
    for (int i = 0; i < 2 * n; i++) pool_reset(&d->bpool[i]);
    pool_reset(&d->rpool);
    for (int i = 0; i < N; i++) {
        float v = llr[i];
        d->channel[i] = v > 1048576.0f ? 1048576.0f : (v < -1048576.0f ? -1048576.0f : v);
    }
    path_t *root = &d->paths[0];                              /* listdec.py:196-199 */
    root->pm = 0.0;
    for (int s = 0; s < n; s++) root->alpha[s] = pool_alloc(&d->apool[s]);
    for (int i = 0; i < 2 * n; i++) root->beta[i] = pool_alloc(&d->bpool[i]);
    root->root = pool_alloc(&d->rpool);
    int P = 1;
    d->err = 0;
    for (int o = 0; o < d->n_ops; o++) {
        const int32_t *op = d->ops + 5 * o;
        int kind = op[0], size = op[1], stage = op[2], h = size >> 1;
        if (kind == K_F) {                                       /* 319-321 */
            for (int t = 0; t < P; t++) {
                const float *a = alpha_of(d, &d->paths[t], stage, size);
                float *o_ = d->tmp_a + (size_t)t * h;
                for (int i = 0; i < h; i++) o_[i] = f_fn(a[i], a[i + h]);
            }
            for (int t = 0; t < P; t++)
                memcpy(alpha_write(d, &d->paths[t], stage - 1), d->tmp_a + (size_t)t * h,
                       sizeof(float) * h);
        } else if (kind == K_G) {                                /* 322-326 */
            for (int t = 0; t < P; t++) {
                const float *a = alpha_of(d, &d->paths[t], stage, size);
                const unsigned char *bl = beta_of(d, &d->paths[t], stage - 1, 0);
                float *o_ = d->tmp_a + (size_t)t * h;
                for (int i = 0; i < h; i++) {
                    float v = a[i + h] + (1.0f - 2.0f * (float)bl[i]) * a[i];
                    if (d->int8_mode) v = v > 127.0f ? 127.0f : (v < -127.0f ? -127.0f : v);
                    o_[i] = v;
                }
            }
            for (int t = 0; t < P; t++)
                memcpy(alpha_write(d, &d->paths[t], stage - 1), d->tmp_a + (size_t)t * h,
                       sizeof(float) * h);
        } else if (kind == K_COMB) {                             /* 327-332 */
            unsigned char *tmp = (unsigned char *)d->tmp_a;
            for (int t = 0; t < P; t++) {
                const unsigned char *l = beta_of(d, &d->paths[t], stage - 1, 0);
                const unsigned char *r = beta_of(d, &d->paths[t], stage - 1, 1);
                unsigned char *m = tmp + (size_t)t * size;
                for (int i = 0; i < h; i++) { m[i] = l[i] ^ r[i]; m[i + h] = r[i]; }
            }
            for (int t = 0; t < P; t++)
                memcpy(beta_write(d, &d->paths[t], size, stage, op[3]), tmp + (size_t)t * size, size);
        } else {
            P = run_leaf(d, op, P);
        }
        if (d->err) return -d->err;
    }
    return P;
}


/* ------------------------------------------------ single-path fast path */

/* polaris.fastssc.execute_schedule (fastssc.py:20-83) for one frame: every
 * leaf takes its most likely decision directly (Rate-0 zeros, Rate-1 hard
 * decisions, repetition by the sign of the pairwise sum, SPC by the Wagner
 * rule on the first least reliable position).  x: [N] codeword estimate;
 * returns the path metric.  The adaptive decoder (listdec.py:437-459) runs
 * this first and keeps its result when the CRC passes. */
static double fastssc_frame(const oc_code *code, const int32_t *ops, int n_ops, int int8_mode,
                            const float *llr, unsigned char *x, float *work) {
    const int N = code->N;
    int n = 0;
    while ((1 << n) < N) n++;
    float *ch = work, *alpha = work + N;                 /* alpha[s] at offset 2^s */
    unsigned char *beta = (unsigned char *)(work + 2 * N); /* beta[s][side] at (2s+side)*N */
    for (int i = 0; i < N; i++) {
        float v = llr[i];
        ch[i] = v > 1048576.0f ? 1048576.0f : (v < -1048576.0f ? -1048576.0f : v);
    }
    double pm = 0.0;
    for (int o = 0; o < n_ops; o++) {
        const int32_t *op = ops + 5 * o;
        int kind = op[0], m = op[1], s = op[2], side = op[3], h = m >> 1;
        const float *src = m == N ? ch : alpha + (1 << s);
        if (kind == K_F) {                                      /* 59-61 */
            float *d = alpha + (1 << (s - 1));
            for (int i = 0; i < h; i++) d[i] = f_fn(src[i], src[i + h]);
            continue;
        }
        if (kind == K_G) {                                      /* 62-64 */
            float *d = alpha + (1 << (s - 1));
            const unsigned char *bl = beta + (size_t)(2 * (s - 1)) * N;
            for (int i = 0; i < h; i++) {
                float v = src[i + h] + (1.0f - 2.0f * (float)bl[i]) * src[i];
                if (int8_mode) v = v > 127.0f ? 127.0f : (v < -127.0f ? -127.0f : v);
                d[i] = v;
            }
            continue;
        }
        unsigned char *dst = m == N ? x : beta + (size_t)(2 * s + side) * N;
        if (kind == K_COMB) {                                   /* 66-69 */
            const unsigned char *l = beta + (size_t)(2 * (s - 1)) * N, *r = l + N;
            for (int i = 0; i < h; i++) { dst[i] = l[i] ^ r[i]; dst[i + h] = r[i]; }
        } else if (kind == K_R0) {                              /* 70-72 */
            float *mn = (float *)malloc(sizeof(float) * m);
            for (int i = 0; i < m; i++) { mn[i] = src[i] < 0.0f ? src[i] : 0.0f; dst[i] = 0; }
            pm += (double)pw_sum(mn, m);
            free(mn);
        } else if (kind == K_R1) {                              /* 73-74 */
            for (int i = 0; i < m; i++) dst[i] = src[i] < 0.0f;
        } else if (kind == K_REP) {                             /* 75-80 */
            float *a = (float *)malloc(sizeof(float) * 2 * m);
            for (int i = 0; i < m; i++) { a[i] = src[i] < 0.0f ? src[i] : 0.0f; a[m + i] = src[i] > 0.0f ? src[i] : 0.0f; }
            float neg = pw_sum(a, m), pos = pw_sum(a + m, m), tot = pw_sum(src, m);
            int ones = tot < 0.0f;
            for (int i = 0; i < m; i++) dst[i] = (unsigned char)ones;
            pm += ones ? (double)(-pos) : (double)neg;
            free(a);
        } else if (kind == K_SPC) {                             /* 81-88 */
            int par = 0, weak = 0;
            float wm = INFINITY;
            for (int i = 0; i < m; i++) {
                dst[i] = src[i] < 0.0f;
                par ^= dst[i];
                float mg = fabsf(src[i]);
                if (mg < wm) { wm = mg; weak = i; }             /* argmin: first minimum */
            }
            if (par) { dst[weak] ^= 1; pm -= (double)wm; }
        } else {
            return NAN;
        }
    }
    return pm;
}

int oracle_fastssc_batch(const oc_code *code, const int32_t *ops, int n_ops, int int8_mode,
                         const float *llr, int64_t batch, uint8_t *codewords, double *pm,
                         uint8_t *info, uint8_t *crc_ok) {
    const int N = code->N;
    if (N < 2 || (N & (N - 1))) return -11;
    float *work = (float *)malloc(sizeof(float) * 2 * N + (size_t)2 * 17 * N);
    unsigned char *x = (unsigned char *)malloc(N), *u = (unsigned char *)malloc(N);
    dec_t d;
    memset(&d, 0, sizeof d);
    d.code = code;
    int *ipos = (int *)malloc(sizeof(int) * N);
    int ni = 0;
    for (int i = 0; i < N; i++)
        if (!code->frozen[i]) ipos[ni++] = i;
    d.info_pos = ipos;
    for (int64_t b = 0; b < batch; b++) {
        double p = fastssc_frame(code, ops, n_ops, int8_mode, llr + (size_t)b * N, x, work);
        if (codewords) memcpy(codewords + (size_t)b * N, x, N);
        if (pm) pm[b] = p;
        memcpy(u, x, N);
        polar_transform(u, N);
        if (info)
            for (int i = 0; i < code->k; i++) info[(size_t)b * code->k + i] = u[ipos[i]];
        if (crc_ok) crc_ok[b] = (uint8_t)crc_ok_of(&d, u);
    }
    free(work); free(x); free(u); free(ipos);
    return 0;
}

/* --------------------------------------------------------- batch entry */

typedef struct {
    const oc_code *code; const int32_t *ops; int n_ops, L, int8_mode;
    const float *llr; int64_t b0, b1;
    uint8_t *info, *crc_ok, *all_cw, *all_crc; double *pm, *all_pm; int32_t *paths;
    int rc;
} job_t;

static void *run_job(void *arg) {
    job_t *j = (job_t *)arg;
    dec_t d;
    dec_init(&d, j->code, j->ops, j->n_ops, j->L, j->int8_mode);
    int N = d.N, k = j->code->k, L = j->L;
    unsigned char *u = (unsigned char *)malloc(N);
    j->rc = 0;
    for (int64_t b = j->b0; b < j->b1; b++) {
        int P = decode_frame(&d, j->llr + (size_t)b * N);
        if (P < 0) { j->rc = P; break; }
        int best = -1, best_ok = 0;
        double best_pm = 0.0;
        /* listdec.py:289-308: CRC-passing pool first, strict max, earliest wins */
        int any_ok = 0;
        int oks[64];
        for (int t = 0; t < P; t++) {
            memcpy(u, pool_row(&d.rpool, d.paths[t].root), N);
            polar_transform(u, N);
            oks[t] = crc_ok_of(&d, u);
            any_ok |= oks[t];
            if (j->all_cw) {
                memcpy(j->all_cw + ((size_t)b * L + t) * N, pool_row(&d.rpool, d.paths[t].root), N);
                j->all_pm[(size_t)b * L + t] = d.paths[t].pm;
                j->all_crc[(size_t)b * L + t] = (uint8_t)oks[t];
            }
        }
        for (int t = 0; t < P; t++) {
            if (any_ok && !oks[t]) continue;
            if (best < 0 || d.paths[t].pm > best_pm) { best = t; best_pm = d.paths[t].pm; best_ok = oks[t]; }
        }
        memcpy(u, pool_row(&d.rpool, d.paths[best].root), N);
        polar_transform(u, N);
        if (j->info)
            for (int i = 0; i < k; i++) j->info[(size_t)b * k + i] = u[d.info_pos[i]];
        if (j->crc_ok) j->crc_ok[b] = (uint8_t)best_ok;
        if (j->pm) j->pm[b] = best_pm;
        if (j->paths) j->paths[b] = P;
    }
    free(u);
    dec_free(&d);
    return NULL;
}

int oracle_decode_batch(const oc_code *code, const int32_t *ops, int n_ops, int list_size,
                        int int8_mode, const float *llr, int64_t batch, uint8_t *info,
                        uint8_t *crc_ok, double *pm, int32_t *paths_used, uint8_t *all_cw,
                        double *all_pm, uint8_t *all_crc, int nthreads) {
    if (list_size < 1 || list_size > 64) return -10;
    if (code->N < 2 || (code->N & (code->N - 1))) return -11;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > batch) nthreads = batch > 0 ? (int)batch : 1;
    job_t *jobs = (job_t *)calloc(nthreads, sizeof(job_t));
    pthread_t *th = (pthread_t *)calloc(nthreads, sizeof(pthread_t));
    int64_t per = (batch + nthreads - 1) / nthreads;
    for (int t = 0; t < nthreads; t++) {
        job_t *j = &jobs[t];
        j->code = code; j->ops = ops; j->n_ops = n_ops; j->L = list_size; j->int8_mode = int8_mode;
        j->llr = llr; j->b0 = t * per; j->b1 = (t + 1) * per < batch ? (t + 1) * per : batch;
        j->info = info; j->crc_ok = crc_ok; j->pm = pm; j->paths = paths_used;
        j->all_cw = all_cw; j->all_pm = all_pm; j->all_crc = all_crc;
        if (j->b0 >= j->b1) continue;
        if (nthreads == 1) run_job(j);
        else pthread_create(&th[t], NULL, run_job, j);
    }
    int rc = 0;
    for (int t = 0; t < nthreads; t++) {
        if (nthreads > 1 && jobs[t].b0 < jobs[t].b1) pthread_join(th[t], NULL);
        if (jobs[t].rc) rc = jobs[t].rc;
    }
    free(jobs); free(th);
    return rc;
}
