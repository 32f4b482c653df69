/*
 * ft_oracle.c -- CPU ORACLE for the vertex-contribution EC path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is a plain-C restatement of the
 * reference package `fieldtopo` (arXiv 2311.11740, /root/reference/pkg) for
 * the hot path named in BASELINE.json.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it, and only as
 * the checker or the timed CPU baseline -- never as a product code path.
 *
 * Parity pin: tests/test_oracle_golden.py checks every function here against
 * golden vectors produced by importing the reference itself
 * (tests/golden/gen_golden.py, committed with its outputs).
 *
 * Restated functions (reference file:line):
 *   ft_oracle_quantize_f64   fields.py:20-33   quantize_with_range
 *   ft_oracle_scan2d         contrib2d.py:161-232  _scan_rows_2d
 *   ft_oracle_accum3d        contrib3d.py:241-348  _accum_vertex_3d
 *   ft_oracle_scan3d         contrib3d.py:351-370  _scan_slabs_3d
 *   ft_oracle_gather2d/3d    contrib2d.py:274-294 / contrib3d.py:440-458
 *                            (+ _parallel.py:8-33 split_blocks/run_blocks)
 *
 * Layout: the reference scans an int32 array padded with a one-cell border of
 * the sentinel max_level+1 (sources.py:66-74).  Here the padding is virtual:
 * get2/get3 return the sentinel for out-of-range cells, which is the same
 * value the padded array holds there.  Histograms are uint64 [T][M+2],
 * T = 5 (2D, contrib2d.py:36) or 21 (3D, contrib3d.py:35-44).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- quantize */

/* fields.py:20-33: clip(floor((x - lo) * M / (hi - lo) + 0.5), 0, M) in
 * float64, evaluated left to right like the numpy expression.  Build with
 * -ffp-contract=off so no FMA changes the rounding. */
static inline int32_t quant_one(double x, double lo, double hi, int32_t M)
{
    if (hi == lo) return 0;
    double scaled = (x - lo) * (double)M / (hi - lo);
    double r = floor(scaled + 0.5);
    if (r < 0.0) r = 0.0;
    if (r > (double)M) r = (double)M;
    return (int32_t)r;
}

/* dtype: 0 int32, 1 uint8, 2 uint16, 3 float32, 4 float64 */
static inline double load_as_double(const void *p, int dtype, int64_t idx)
{
    switch (dtype) {
    case 0: return (double)((const int32_t *)p)[idx];
    case 1: return (double)((const uint8_t *)p)[idx];
    case 2: return (double)((const uint16_t *)p)[idx];
    case 3: return (double)((const float *)p)[idx];
    default: return ((const double *)p)[idx];
    }
}

void ft_oracle_quantize(const void *x, int dtype, int64_t n, double lo, double hi,
                        int32_t M, int32_t *out)
{
    for (int64_t i = 0; i < n; ++i) out[i] = quant_one(load_as_double(x, dtype, i), lo, hi, M);
}

/* A level source: either an int32 level array (identity) or a raw array that
 * is quantized on the fly with (lo, hi, M) -- the slab-driven oracle of
 * SURVEY.md Appendix C.1 (quantize per slab, then scan). */
typedef struct {
    const void *data;
    int dtype;        /* 0 = int32 levels (identity), else raw + quantize */
    int quantize;     /* 1: apply quant_one */
    double lo, hi;
    int32_t M;
} level_src;

static inline int64_t src_level(const level_src *s, int64_t idx)
{
    if (!s->quantize) {
        switch (s->dtype) {
        case 0: return ((const int32_t *)s->data)[idx];
        case 1: return ((const uint8_t *)s->data)[idx];
        case 2: return ((const uint16_t *)s->data)[idx];
        default: return (int64_t)load_as_double(s->data, s->dtype, idx);
        }
    }
    return quant_one(load_as_double(s->data, s->dtype, idx), s->lo, s->hi, s->M);
}

/* ---------------------------------------------------------------- 2D scan */

/* contrib2d.py:161-232.  Vertex (i, j), 0 <= i <= H, 0 <= j <= W, reads the
 * cells (i-1, j-1) (i-1, j) (i, j-1) (i, j) = slots NW NE SW SE (contrib2d.py
 * :39-40, :117-131).  p0 = first slot holding the minimum, p1 = first other
 * slot holding the next minimum; the remaining two values are ordered; the
 * two-face state is diagonal iff p0 + p1 == 3 (contrib2d.py:224). */
static void scan2d_rows(const level_src *s, int64_t H, int64_t W, int64_t i0, int64_t i1,
                        uint64_t *q_in, uint64_t *q_out)
{
    const int64_t M2 = (int64_t)s->M + 2;
    const int64_t sent = (int64_t)s->M + 1;
    for (int64_t i = i0; i < i1; ++i) {
        for (int64_t j = 0; j <= W; ++j) {
            int64_t v[4];
            v[0] = (i > 0 && j > 0) ? src_level(s, (i - 1) * W + (j - 1)) : sent;
            v[1] = (i > 0 && j < W) ? src_level(s, (i - 1) * W + j) : sent;
            v[2] = (i < H && j > 0) ? src_level(s, i * W + (j - 1)) : sent;
            v[3] = (i < H && j < W) ? src_level(s, i * W + j) : sent;
            int p0 = 0;
            int64_t v0 = v[0];
            for (int t = 1; t < 4; ++t)
                if (v[t] < v0) { v0 = v[t]; p0 = t; }
            int p1 = -1;
            int64_t v1 = INT64_MAX;
            for (int t = 0; t < 4; ++t)
                if (t != p0 && v[t] < v1) { v1 = v[t]; p1 = t; }
            int64_t rest[2];
            int nr = 0;
            for (int t = 0; t < 4; ++t)
                if (t != p0 && t != p1) rest[nr++] = v[t];
            int64_t v2 = rest[0], v3 = rest[1];
            if (v3 < v2) { int64_t tmp = v2; v2 = v3; v3 = tmp; }
            int two = (p0 + p1 == 3) ? 2 : 1; /* QD : Q2 */
            q_in[0 * M2 + v0] += 1;
            q_out[0 * M2 + v1] += 1;
            q_in[two * M2 + v1] += 1;
            q_out[two * M2 + v2] += 1;
            q_in[3 * M2 + v2] += 1;
            q_out[3 * M2 + v3] += 1;
            q_in[4 * M2 + v3] += 1;
        }
    }
}

/* ---------------------------------------------------------------- 3D scan */

static inline int popc3(int x) { return (x & 1) + ((x >> 1) & 1) + ((x >> 2) & 1); }

/* contrib3d.py:241-348: stable insertion argsort of the 8 slot values, then
 * stages 1..8 classified by pair-class counts (face/edge/vertex = popcount of
 * slot xor 1/2/3, contrib3d.py:76-90); stages 5..7 by the empty cells.
 * Returns 0, or -1 for a profile outside the table (the reference raises). */
static int accum3d(const int64_t vals[8], int64_t M2, uint64_t *q_in, uint64_t *q_out)
{
    int order[8];
    for (int s = 0; s < 8; ++s) order[s] = s;
    for (int s = 1; s < 8; ++s) {
        int o = order[s];
        int64_t v = vals[o];
        int t = s - 1;
        while (t >= 0 && vals[order[t]] > v) { order[t + 1] = order[t]; --t; }
        order[t + 1] = o;
    }
    q_in[0 * M2 + vals[order[0]]] += 1;
    q_out[0 * M2 + vals[order[1]]] += 1;

    int nf = 0, ne = 0, nv = 0;
    for (int n = 2; n <= 4; ++n) {
        int s_new = order[n - 1];
        for (int m = 0; m < n - 1; ++m) {
            int d2 = popc3(s_new ^ order[m]);
            if (d2 == 1) ++nf; else if (d2 == 2) ++ne; else ++nv;
        }
        int ti = -1;
        if (n == 2) {
            ti = nf == 1 ? 1 : (ne == 1 ? 2 : 3);
        } else if (n == 3) {
            if (nf == 2 && ne == 1 && nv == 0) ti = 4;
            else if (nf == 1 && ne == 1 && nv == 1) ti = 5;
            else if (nf == 0 && ne == 3 && nv == 0) ti = 6;
        } else {
            if (nf == 4 && ne == 2 && nv == 0) ti = 7;
            else if (nf == 3 && ne == 3 && nv == 0) ti = 8;
            else if (nf == 3 && ne == 2 && nv == 1) ti = 9;
            else if (nf == 2 && ne == 3 && nv == 1) ti = 10;
            else if (nf == 2 && ne == 2 && nv == 2) ti = 11;
            else if (nf == 0 && ne == 6 && nv == 0) ti = 12;
        }
        if (ti < 0) return -1;
        q_in[ti * M2 + vals[order[n - 1]]] += 1;
        q_out[ti * M2 + vals[order[n]]] += 1;
    }
    int ef = 0, ee = 0, ev = 0;
    for (int a = 5; a < 8; ++a)
        for (int b = a + 1; b < 8; ++b) {
            int d2 = popc3(order[a] ^ order[b]);
            if (d2 == 1) ++ef; else if (d2 == 2) ++ee; else ++ev;
        }
    int t5;
    if (ef == 2 && ee == 1 && ev == 0) t5 = 13;
    else if (ef == 1 && ee == 1 && ev == 1) t5 = 14;
    else if (ef == 0 && ee == 3 && ev == 0) t5 = 15;
    else return -1;
    q_in[t5 * M2 + vals[order[4]]] += 1;
    q_out[t5 * M2 + vals[order[5]]] += 1;
    int d2 = popc3(order[6] ^ order[7]);
    int t6 = d2 == 1 ? 16 : (d2 == 2 ? 17 : 18);
    q_in[t6 * M2 + vals[order[5]]] += 1;
    q_out[t6 * M2 + vals[order[6]]] += 1;
    q_in[19 * M2 + vals[order[6]]] += 1;
    q_out[19 * M2 + vals[order[7]]] += 1;
    q_in[20 * M2 + vals[order[7]]] += 1;
    return 0;
}

/* contrib3d.py:351-370.  Vertex (i, j, k) reads cell (i-1+di, j-1+dj, k-1+dk)
 * into slot di + 2 dj + 4 dk (contrib3d.py:47-49). */
static int scan3d_rows(const level_src *s, int64_t H, int64_t W, int64_t D, int64_t i0,
                       int64_t i1, uint64_t *q_in, uint64_t *q_out)
{
    const int64_t M2 = (int64_t)s->M + 2;
    const int64_t sent = (int64_t)s->M + 1;
    int64_t vals[8];
    for (int64_t i = i0; i < i1; ++i)
        for (int64_t j = 0; j <= W; ++j)
            for (int64_t k = 0; k <= D; ++k) {
                for (int sl = 0; sl < 8; ++sl) {
                    int64_t ci = i - 1 + (sl & 1), cj = j - 1 + ((sl >> 1) & 1),
                            ck = k - 1 + ((sl >> 2) & 1);
                    vals[sl] = (ci >= 0 && ci < H && cj >= 0 && cj < W && ck >= 0 && ck < D)
                                   ? src_level(s, (ci * W + cj) * D + ck)
                                   : sent;
                }
                if (accum3d(vals, M2, q_in, q_out)) return -1;
            }
    return 0;
}

/* ------------------------------------------------------- threaded drivers */

/* _parallel.py:8-24: contiguous blocks of total // workers rows, remainder on
 * the last block, empty blocks dropped.  Returns the number of blocks. */
int ft_oracle_split_blocks(int64_t total, int workers, int64_t *lo, int64_t *hi)
{
    if (workers < 1) return -1;
    int64_t size = total / workers, start = 0;
    int nb = 0;
    for (int t = 0; t < workers; ++t) {
        int64_t stop = (t < workers - 1) ? start + size : total;
        if (stop > start) { lo[nb] = start; hi[nb] = stop; ++nb; }
        start = stop;
    }
    return nb;
}

typedef struct {
    const level_src *src;
    int ndim;
    int64_t H, W, D, i0, i1;
    uint64_t *q_in, *q_out;
    int rc;
} job_t;

static void *run_job(void *arg)
{
    job_t *j = (job_t *)arg;
    if (j->ndim == 2) {
        scan2d_rows(j->src, j->H, j->W, j->i0, j->i1, j->q_in, j->q_out);
        j->rc = 0;
    } else {
        j->rc = scan3d_rows(j->src, j->H, j->W, j->D, j->i0, j->i1, j->q_in, j->q_out);
    }
    return NULL;
}

/* contrib{2,3}d gather_*_parallel: private per-worker histograms summed after
 * the join (contrib2d.py:274-294, contrib3d.py:440-458).  Vertex rows
 * [row_lo, row_hi) only (the full field is row_lo = 0, row_hi = H + 1), so the
 * same routine serves as the slab-driven oracle for multi-GPU partitions.
 * q_in / q_out (T x (M+2)) are ACCUMULATED into (caller zeroes them). */
static int gather(int ndim, const level_src *src, int64_t H, int64_t W, int64_t D,
                  int64_t row_lo, int64_t row_hi, int workers, uint64_t *q_in, uint64_t *q_out)
{
    const int T = ndim == 2 ? 5 : 21;
    const int64_t n = (int64_t)T * (src->M + 2);
    if (workers < 1) return 1;
    int64_t *lo = (int64_t *)malloc(sizeof(int64_t) * workers);
    int64_t *hi = (int64_t *)malloc(sizeof(int64_t) * workers);
    int nb = ft_oracle_split_blocks(row_hi - row_lo, workers, lo, hi);
    job_t *jobs = (job_t *)calloc(nb > 0 ? nb : 1, sizeof(job_t));
    pthread_t *th = (pthread_t *)calloc(nb > 0 ? nb : 1, sizeof(pthread_t));
    uint64_t *priv = (uint64_t *)calloc((size_t)(nb > 0 ? nb : 1) * 2 * n, sizeof(uint64_t));
    for (int b = 0; b < nb; ++b) {
        jobs[b] = (job_t){src, ndim, H, W, D, row_lo + lo[b], row_lo + hi[b],
                          priv + (size_t)b * 2 * n, priv + (size_t)b * 2 * n + n, 0};
        if (nb == 1) run_job(&jobs[b]);
        else pthread_create(&th[b], NULL, run_job, &jobs[b]);
    }
    int rc = 0;
    for (int b = 0; b < nb; ++b) {
        if (nb > 1) pthread_join(th[b], NULL);
        if (jobs[b].rc) rc = 2;
        for (int64_t t = 0; t < n; ++t) {
            q_in[t] += jobs[b].q_in[t];
            q_out[t] += jobs[b].q_out[t];
        }
    }
    free(lo); free(hi); free(jobs); free(th); free(priv);
    return rc;
}

/* Identity (integer levels) or on-the-fly quantize (quantize != 0). */
int ft_oracle_gather2d(const void *x, int dtype, int quantize, double lo, double hi,
                       int64_t H, int64_t W, int32_t M, int64_t row_lo, int64_t row_hi,
                       int workers, uint64_t *q_in, uint64_t *q_out)
{
    level_src s = {x, dtype, quantize, lo, hi, M};
    return gather(2, &s, H, W, 0, row_lo, row_hi, workers, q_in, q_out);
}

int ft_oracle_gather3d(const void *x, int dtype, int quantize, double lo, double hi,
                       int64_t H, int64_t W, int64_t D, int32_t M, int64_t row_lo,
                       int64_t row_hi, int workers, uint64_t *q_in, uint64_t *q_out)
{
    level_src s = {x, dtype, quantize, lo, hi, M};
    return gather(3, &s, H, W, D, row_lo, row_hi, workers, q_in, q_out);
}

/* One vertex neighbourhood (accumulate_vertex_3d semantics, contrib3d.py
 * :220-238, via the fused kernel body): exposed for known-answer tests. */
int ft_oracle_accum3d(const int64_t vals[8], int32_t M, uint64_t *q_in, uint64_t *q_out)
{
    return accum3d(vals, (int64_t)M + 2, q_in, q_out);
}
