/*
 * CPU ORACLE (test infrastructure only) -- plain-C restatement of the
 * reference's dense CountSketch and SRHT applies, multi-threaded over
 * columns so that BASELINE.json's full-size configs (up to 2^23 x 256)
 * can be checked on the GPU box's host in seconds.  Columns are
 * independent in both applies, so splitting the work by column does not
 * change a single rounding: the results are bitwise those of the numpy /
 * scipy restatement in oracle/oracle.py (pinned by tests/test_oracle_golden.py
 * and tests/test_oracle_c_applies.py).
 *
 *   orc_countsketch_fold_mt -- scipy 1.18.1 csr_matvecs as called by
 *     sketch.py:209,212 (`sparse_map @ A`): for every bucket, the signed
 *     source rows in ascending order, added from +0.0.
 *   orc_srht_apply -- sketch.py:213-223 with fwht_inplace :152-177: the
 *     sign-flipped column zero-padded to m_pad, the unnormalised radix-2
 *     FWHT with h ascending and the butterfly (a, b) -> (a + b, -2b + (a + b))
 *     (the three in-place numpy statements of :172-175), then
 *     pad[row_sample] / sqrt(d).  The levels h < 2^13 run inside 2^13-element
 *     blocks (cache-resident) before the higher levels; every element still
 *     sees the same operations in the same order as the level-by-level loop.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  /* shared */
  const double* A;
  int64_t m, n, lda, d;
  const int64_t* rows;       /* countsketch */
  const double* signs;       /* countsketch signs or SRHT sign_diag */
  const int64_t* row_sample; /* srht */
  int64_t m_pad, ldo;
  double* out;
  int kind; /* 0 countsketch, 1 srht */
  int64_t next;              /* next column to take */
  pthread_mutex_t lock;
} job_t;

static int64_t take_column(job_t* j) {
  pthread_mutex_lock(&j->lock);
  const int64_t c = j->next < j->n ? j->next++ : -1;
  pthread_mutex_unlock(&j->lock);
  return c;
}

static void fold_column(const job_t* j, int64_t c) {
  double* y = j->out + c * j->ldo;
  const double* a = j->A + c * j->lda;
  memset(y, 0, sizeof(double) * (size_t)j->d);
  for (int64_t r = 0; r < j->m; ++r) y[j->rows[r]] += j->signs[r] * a[r];
}

static void fwht_levels(double* x, int64_t len, int64_t h_begin, int64_t h_end) {
  for (int64_t h = h_begin; h < h_end; h <<= 1) {
    for (int64_t base = 0; base < len; base += 2 * h) {
      double* p = x + base;
      double* q = x + base + h;
      for (int64_t i = 0; i < h; ++i) {
        const double s = p[i] + q[i]; /* w[:, 0] += w[:, 1]       */
        const double t = q[i] * -2.0; /* w[:, 1] *= -2.0          */
        p[i] = s;
        q[i] = t + s;                 /* w[:, 1] += w[:, 0]       */
      }
    }
  }
}

static void srht_column(const job_t* j, int64_t c, double* buf) {
  const double* a = j->A + c * j->lda;
  for (int64_t r = 0; r < j->m; ++r) buf[r] = j->signs[r] * a[r];
  memset(buf + j->m, 0, sizeof(double) * (size_t)(j->m_pad - j->m));
  const int64_t blk = j->m_pad < 8192 ? j->m_pad : 8192;
  for (int64_t b = 0; b < j->m_pad; b += blk) fwht_levels(buf + b, blk, 1, blk);
  fwht_levels(buf, j->m_pad, blk, j->m_pad);
  const double sd = sqrt((double)j->d);
  double* y = j->out + c * j->ldo;
  for (int64_t k = 0; k < j->d; ++k) y[k] = buf[j->row_sample[k]] / sd;
}

static void* worker(void* arg) {
  job_t* j = (job_t*)arg;
  double* buf = NULL;
  if (j->kind == 1) {
    buf = (double*)malloc(sizeof(double) * (size_t)j->m_pad);
    if (!buf) return (void*)1;
  }
  for (int64_t c; (c = take_column(j)) >= 0;) {
    if (j->kind == 0)
      fold_column(j, c);
    else
      srht_column(j, c, buf);
  }
  free(buf);
  return NULL;
}

static int run(job_t* j, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  pthread_mutex_init(&j->lock, NULL);
  j->next = 0;
  int started = 0, rc = 0;
  for (; started < threads; ++started)
    if (pthread_create(&th[started], NULL, worker, j)) break;
  if (started == 0) rc = (worker(j) != NULL);
  for (int t = 0; t < started; ++t) {
    void* r = NULL;
    pthread_join(th[t], &r);
    if (r) rc = 1;
  }
  pthread_mutex_destroy(&j->lock);
  return rc;
}

/* out (d x n, column-major, ld ldo) = S A for F-ordered A (m x n, ld lda). */
int orc_countsketch_fold_mt(const int64_t* rows, const double* signs, int64_t m, int64_t n,
                            const double* A, int64_t lda, int64_t d, double* out, int64_t ldo,
                            int threads) {
  job_t j;
  memset(&j, 0, sizeof j);
  j.A = A; j.m = m; j.n = n; j.lda = lda; j.d = d; j.rows = rows; j.signs = signs;
  j.out = out; j.ldo = ldo; j.kind = 0;
  return run(&j, threads);
}

/* out (d x n, column-major, ld ldo) = SRHT of F-ordered A (m x n, ld lda). */
int orc_srht_apply(const double* A, int64_t m, int64_t n, int64_t lda, const double* sign_diag,
                   const int64_t* row_sample, int64_t m_pad, int64_t d, double* out, int64_t ldo,
                   int threads) {
  if (m_pad < m || (m_pad & (m_pad - 1))) return 2;
  job_t j;
  memset(&j, 0, sizeof j);
  j.A = A; j.m = m; j.n = n; j.lda = lda; j.d = d; j.signs = sign_diag;
  j.row_sample = row_sample; j.m_pad = m_pad; j.out = out; j.ldo = ldo; j.kind = 1;
  return run(&j, threads);
}
