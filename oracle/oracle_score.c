/*
 * CPU oracle (TEST INFRASTRUCTURE ONLY) -- plain-C restatement of the DESSERT
 * sigma=max set score, used by tests/ for large sampled parity checks where the
 * numpy port is too slow.  Never linked into the product library.
 *
 *   c_q   = max_j sum_t [q_t == x_jt]              (reference: sketch.py:92-153,
 *                                                   index.py:183-213)
 *   score = pairwise_sum_f64(LUT[c_q]) / m_q        (index.py:216, numpy
 *                                                   pairwise_sum_DOUBLE order)
 *
 * Pinned against the numpy oracle and the reference golden vectors in
 * tests/test_oracle.py.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static double pw_rec(const double *a, int64_t n) {
    if (n < 8) {
        double r = 0.0;
        for (int64_t i = 0; i < n; i++) r += a[i];
        return r;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; j++) r[j] = a[j];
        int64_t i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return pw_rec(a, n2) + pw_rec(a + n2, n - n2);
}

double oracle_pairwise_sum(const double *a, int64_t n) { return 0.0 + pw_rec(a, n); }

typedef struct {
    const int32_t *codes;   /* (n_vec, L) */
    const int64_t *set_off; /* (n_sets + 1) */
    const int32_t *qcodes;  /* (n_qsets, m_q, L) */
    const int64_t *sets;    /* (n_eval) set indices per query set, or NULL = all */
    const double *lut;      /* (L + 1) */
    int64_t n_qsets, n_eval, m_q, L;
    double *scores;         /* (n_qsets, n_eval) */
    uint16_t *maxcounts;    /* (n_qsets, n_eval, m_q) or NULL */
    int64_t next;           /* work counter (row-major pair index) */
    pthread_mutex_t mu;
} job_t;

static void score_pair(job_t *jb, int64_t qs, int64_t e, double *buf) {
    int64_t s = jb->sets ? jb->sets[qs * jb->n_eval + e] : e;
    const int32_t *x = jb->codes + jb->set_off[s] * jb->L;
    int64_t m = jb->set_off[s + 1] - jb->set_off[s];
    const int32_t *q = jb->qcodes + qs * jb->m_q * jb->L;
    for (int64_t a = 0; a < jb->m_q; a++) {
        int64_t best = 0;
        for (int64_t j = 0; j < m; j++) {
            int64_t c = 0;
            for (int64_t t = 0; t < jb->L; t++) c += (q[a * jb->L + t] == x[j * jb->L + t]);
            if (c > best) best = c;
        }
        buf[a] = jb->lut[best];
        if (jb->maxcounts) jb->maxcounts[(qs * jb->n_eval + e) * jb->m_q + a] = (uint16_t)best;
    }
    jb->scores[qs * jb->n_eval + e] = oracle_pairwise_sum(buf, jb->m_q) / (double)jb->m_q;
}

static void *worker(void *arg) {
    job_t *jb = (job_t *)arg;
    double *buf = (double *)malloc(sizeof(double) * (size_t)(jb->m_q > 0 ? jb->m_q : 1));
    const int64_t total = jb->n_qsets * jb->n_eval, grain = 64;
    for (;;) {
        pthread_mutex_lock(&jb->mu);
        int64_t lo = jb->next;
        jb->next += grain;
        pthread_mutex_unlock(&jb->mu);
        if (lo >= total) break;
        int64_t hi = lo + grain < total ? lo + grain : total;
        for (int64_t p = lo; p < hi; p++) score_pair(jb, p / jb->n_eval, p % jb->n_eval, buf);
    }
    free(buf);
    return NULL;
}

/* Scores n_qsets query sets against n_eval sets each (sets == NULL: set e). */
int oracle_score(const int32_t *codes, const int64_t *set_off, const int32_t *qcodes,
                 const int64_t *sets, const double *lut, int64_t n_qsets, int64_t n_eval,
                 int64_t m_q, int64_t L, double *scores, uint16_t *maxcounts, int threads) {
    job_t jb;
    memset(&jb, 0, sizeof(jb));
    jb.codes = codes; jb.set_off = set_off; jb.qcodes = qcodes; jb.sets = sets; jb.lut = lut;
    jb.n_qsets = n_qsets; jb.n_eval = n_eval; jb.m_q = m_q; jb.L = L;
    jb.scores = scores; jb.maxcounts = maxcounts;
    pthread_mutex_init(&jb.mu, NULL);
    if (threads < 1) threads = 1;
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)threads);
    for (int i = 0; i < threads; i++) pthread_create(&th[i], NULL, worker, &jb);
    for (int i = 0; i < threads; i++) pthread_join(th[i], NULL);
    free(th);
    pthread_mutex_destroy(&jb.mu);
    return 0;
}
