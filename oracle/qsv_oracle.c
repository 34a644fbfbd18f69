/*
 * ORACLE - test infrastructure only, never part of the product path.
 *
 * Plain-C restatement of the reference full-amplitude kernels and their chunk
 * dispatch (qcsim/statevector.py).  Only tests/, __graft_entry__.smoke() and
 * bench.py's CPU-baseline leg (and `bench.py --impl reference`) load it, as
 * the checker / the timed CPU reference.  Parity is PINNED: tests check this
 * restatement against golden vectors produced by the real reference
 * (tests/golden/make_golden.py).
 *
 * Conventions (statevector.py:1-12): amplitude index bit k <-> qubit k; the
 * array is split into chunks of 2^chunk_log2 amplitudes; a butterfly pair
 * (i, i + 2^k) is owned by the chunk holding the lower index; workers own
 * contiguous chunk spans (statevector.py:157-165) and a barrier separates
 * gates (parallel.py:21-30).  Arithmetic mirrors numba's complex128 code
 * without fast-math: naive complex products, no FMA contraction
 * (compile with -ffp-contract=off).
 */
#include <pthread.h>
#include <stdint.h>
#include <stddef.h>

typedef struct { double re, im; } cplx;

static inline cplx cmul(cplx a, cplx b) {
    cplx r = {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
    return r;
}
static inline cplx cadd(cplx a, cplx b) {
    cplx r = {a.re + b.re, a.im + b.im};
    return r;
}
static inline int cis_one(cplx a) { return a.re == 1.0 && a.im == 0.0; }
static inline int cis_zero(cplx a) { return a.re == 0.0 && a.im == 0.0; }

/* _k_pair, statevector.py:73-83 */
static void k_pair(cplx *x, cplx a, cplx b, cplx c, cplx d, int k, int64_t p0, int64_t p1) {
    int64_t step = (int64_t)1 << k, mask = step - 1;
    for (int64_t p = p0; p < p1; ++p) {
        int64_t i = ((p >> k) << (k + 1)) | (p & mask), j = i | step;
        cplx x0 = x[i], x1 = x[j];
        x[i] = cadd(cmul(a, x0), cmul(b, x1));
        x[j] = cadd(cmul(c, x0), cmul(d, x1));
    }
}

/* _k_pair_offset, statevector.py:86-92 */
static void k_pair_offset(cplx *x, cplx a, cplx b, cplx c, cplx d, int64_t step, int64_t s, int64_t e) {
    for (int64_t i = s; i < e; ++i) {
        cplx x0 = x[i], x1 = x[i + step];
        x[i] = cadd(cmul(a, x0), cmul(b, x1));
        x[i + step] = cadd(cmul(c, x0), cmul(d, x1));
    }
}

/* _k_ctrl_pair, statevector.py:95-104 */
static void k_ctrl_pair(cplx *x, cplx a, cplx b, cplx c, cplx d, int k, int64_t cmask, int64_t s, int64_t e) {
    int64_t step = (int64_t)1 << k;
    for (int64_t i = s; i < e; ++i) {
        if ((i & cmask) == cmask && (i & step) == 0) {
            int64_t j = i | step;
            cplx x0 = x[i], x1 = x[j];
            x[i] = cadd(cmul(a, x0), cmul(b, x1));
            x[j] = cadd(cmul(c, x0), cmul(d, x1));
        }
    }
}

/* _k_ctrl_pair_offset, statevector.py:107-114 */
static void k_ctrl_pair_offset(cplx *x, cplx a, cplx b, cplx c, cplx d, int64_t step, int64_t cmask,
                               int64_t s, int64_t e) {
    for (int64_t i = s; i < e; ++i) {
        if ((i & cmask) == cmask) {
            cplx x0 = x[i], x1 = x[i + step];
            x[i] = cadd(cmul(a, x0), cmul(b, x1));
            x[i + step] = cadd(cmul(c, x0), cmul(d, x1));
        }
    }
}

/* _k_diag, statevector.py:117-125 */
static void k_diag(cplx *x, cplx d0, cplx d1, int k, int64_t cmask, int64_t s, int64_t e) {
    int64_t step = (int64_t)1 << k;
    for (int64_t i = s; i < e; ++i)
        if ((i & cmask) == cmask) x[i] = cmul(x[i], (i & step) ? d1 : d0);
}

/* _k_scale, statevector.py:128-132 */
static void k_scale(cplx *x, cplx f, int64_t cmask, int64_t s, int64_t e) {
    for (int64_t i = s; i < e; ++i)
        if ((i & cmask) == cmask) x[i] = cmul(x[i], f);
}

/* _k_quad, statevector.py:135-149 (u row-major 4x4) */
static void k_quad(cplx *x, const cplx *u, int64_t off_hi, int64_t off_lo, int64_t tmask, int64_t cmask,
                   int64_t s, int64_t e) {
    for (int64_t i = s; i < e; ++i) {
        if ((i & cmask) == cmask && (i & tmask) == 0) {
            int64_t i01 = i + off_lo, i10 = i + off_hi, i11 = i10 + off_lo;
            cplx v[4] = {x[i], x[i01], x[i10], x[i11]};
            cplx o[4];
            for (int r = 0; r < 4; ++r) {
                cplx acc = cmul(u[4 * r], v[0]);
                for (int c = 1; c < 4; ++c) acc = cadd(acc, cmul(u[4 * r + c], v[c]));
                o[r] = acc;
            }
            x[i] = o[0]; x[i01] = o[1]; x[i10] = o[2]; x[i11] = o[3];
        }
    }
}

/* _chunk_single, statevector.py:168-196 */
static void chunk_single(cplx *x, int cl, int64_t chunk, const cplx *u, int k, int64_t cmask_low,
                         const int *hi_ctrl, int n_hi) {
    for (int t = 0; t < n_hi; ++t)
        if (!((chunk >> (hi_ctrl[t] - cl)) & 1)) return;
    int64_t s = chunk << cl, e = s + ((int64_t)1 << cl);
    cplx a = u[0], b = u[1], c = u[2], d = u[3];
    if (cis_zero(b) && cis_zero(c)) {
        if (k >= cl) {
            cplx f = ((chunk >> (k - cl)) & 1) ? d : a;
            if (!cis_one(f)) k_scale(x, f, cmask_low, s, e);
        } else {
            k_diag(x, a, d, k, cmask_low, s, e);
        }
        return;
    }
    if (k >= cl) {
        if ((chunk >> (k - cl)) & 1) return; /* the lower partner chunk owns the pairs */
        int64_t step = (int64_t)1 << k;
        if (cmask_low) k_ctrl_pair_offset(x, a, b, c, d, step, cmask_low, s, e);
        else k_pair_offset(x, a, b, c, d, step, s, e);
    } else if (cmask_low) {
        k_ctrl_pair(x, a, b, c, d, k, cmask_low, s, e);
    } else {
        k_pair(x, a, b, c, d, k, s >> 1, e >> 1);
    }
}

/* _chunk_quad, statevector.py:199-214 */
static void chunk_quad(cplx *x, int cl, int64_t chunk, const cplx *u, int t_hi, int t_lo, int64_t cmask_low,
                       const int *hi_ctrl, int n_hi) {
    for (int t = 0; t < n_hi; ++t)
        if (!((chunk >> (hi_ctrl[t] - cl)) & 1)) return;
    int64_t tmask = 0;
    int tq[2] = {t_hi, t_lo};
    for (int t = 0; t < 2; ++t) {
        if (tq[t] >= cl) {
            if ((chunk >> (tq[t] - cl)) & 1) return;
        } else {
            tmask |= (int64_t)1 << tq[t];
        }
    }
    int64_t s = chunk << cl;
    k_quad(x, u, (int64_t)1 << t_hi, (int64_t)1 << t_lo, tmask, cmask_low, s, s + ((int64_t)1 << cl));
}

/* one worker's contiguous chunk span (_chunk_spans, statevector.py:157-165) */
typedef struct {
    cplx *x;
    const cplx *u;
    int cl, n_targets, t0, t1;
    int64_t cmask_low;
    const int *hi_ctrl;
    int n_hi;
    int64_t lo, hi;
} span_job;

static void *run_span(void *arg) {
    span_job *j = (span_job *)arg;
    for (int64_t ch = j->lo; ch < j->hi; ++ch) {
        if (j->n_targets == 1) chunk_single(j->x, j->cl, ch, j->u, j->t0, j->cmask_low, j->hi_ctrl, j->n_hi);
        else chunk_quad(j->x, j->cl, ch, j->u, j->t0, j->t1, j->cmask_low, j->hi_ctrl, j->n_hi);
    }
    return NULL;
}

/*
 * _apply_gate, statevector.py:217-247.  u: row-major complex (re,im pairs),
 * 2x2 when n_targets == 1, 4x4 when n_targets == 2 (targets[0] = matrix MSB).
 * Returns 0, or -6 for >2 targets (UnsupportedGate, statevector.py:393-394).
 */
int orc_apply_gate(double *amps, int n, int chunk_log2, int workers, const double *u, int n_targets,
                   const int *targets, int n_controls, const int *controls) {
    if (n_targets < 1 || n_targets > 2) return -6;
    cplx *x = (cplx *)amps;
    const cplx *m = (const cplx *)u;
    int cl = chunk_log2 < 0 ? 0 : (chunk_log2 > n ? n : chunk_log2);
    int64_t cmask_low = 0;
    int hi_ctrl[64];
    int n_hi = 0;
    for (int t = 0; t < n_controls; ++t) {
        if (controls[t] >= cl) hi_ctrl[n_hi++] = controls[t];
        else cmask_low |= (int64_t)1 << controls[t];
    }
    int64_t chunks = (int64_t)1 << (n - cl);
    if (workers < 1) workers = 1;
    if (workers > 256) workers = 256;
    span_job jobs[256];
    pthread_t tid[256];
    for (int w = 0; w < workers; ++w) {
        span_job j = {x, m, cl, n_targets, targets[0], n_targets > 1 ? targets[1] : 0, cmask_low,
                      hi_ctrl, n_hi, (int64_t)w * chunks / workers, (int64_t)(w + 1) * chunks / workers};
        jobs[w] = j;
    }
    /* one thread per worker span; joining all of them is the per-gate barrier */
    char started[256] = {0};
    for (int w = 1; w < workers; ++w)
        started[w] = pthread_create(&tid[w], NULL, run_span, &jobs[w]) == 0;
    run_span(&jobs[0]);
    for (int w = 1; w < workers; ++w) {
        if (started[w]) pthread_join(tid[w], NULL);
        else run_span(&jobs[w]);
    }
    return 0;
}

/* default_chunk_log2, statevector.py:46-49 */
int orc_default_chunk_log2(int n, int workers) {
    int want = 4 * (workers > 1 ? workers : 1);
    if (want < 4) want = 4;
    int v = want - 1 > 1 ? want - 1 : 1, bits = 0;
    while (v) { ++bits; v >>= 1; }
    return n - bits > 0 ? n - bits : 0;
}
