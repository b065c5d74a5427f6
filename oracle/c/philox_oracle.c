/*
 * CPU ORACLE (test infrastructure only) -- plain-C restatement of the random
 * streams behind the reference's sketches and of the CountSketch fold.
 *
 * The reference (/root/reference/pkg/src/sketchls/rng.py:43-45,
 * sketch.py:93-127) draws through numpy 2.3.5, a third-party dependency not
 * vendored in /root/reference.  This file restates numpy's published
 * algorithms sequentially, exactly as a numpy Generator consumes its bit
 * generator:
 *   - Philox4x64-10 (Salmon et al. 2011, Random123): key words (key, 0),
 *     counter incremented before each 4-word block;
 *   - next_uint32: low half of a u64 first, leftover kept across calls;
 *   - Generator.integers(0, d): Lemire's nearly-divisionless 32-bit method,
 *     rejection threshold (2^32 - d) mod d;
 *   - Generator.permutation(n): arange(n) shuffled top-down by Fisher-Yates,
 *     j drawn by masked rejection ("random_interval");
 *   - Generator.standard_normal: 256-strip ziggurat (Marsaglia & Tsang) on
 *     full u64 draws, tables supplied by the caller.
 * Pinned by tests/test_oracle_golden.py against numpy's own output and the
 * reference-generated fixtures in tests/golden/.
 * The CountSketch fold restates scipy 1.18.1 csr_matvecs (sparsetools):
 * per bucket, ascending source row, y += s * A[j, :], starting from +0.0.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  uint64_t key, ctr;
  uint64_t buf[4];
  int pos;
  int has32;
  uint32_t u32;
} orc_gen;

static void mulhilo(uint64_t a, uint64_t b, uint64_t* hi, uint64_t* lo) {
  unsigned __int128 p = (unsigned __int128)a * b;
  *lo = (uint64_t)p;
  *hi = (uint64_t)(p >> 64);
}

static void philox10(uint64_t ctr0, uint64_t key, uint64_t out[4]) {
  uint64_t c[4] = {ctr0, 0, 0, 0}, k0 = key, k1 = 0;
  for (int r = 0; r < 10; ++r) {
    if (r) { k0 += 0x9E3779B97F4A7C15ULL; k1 += 0xBB67AE8584CAA73BULL; }
    uint64_t hi0, lo0, hi1, lo1;
    mulhilo(0xD2E7470EE14C6C93ULL, c[0], &hi0, &lo0);
    mulhilo(0xCA5A826395121157ULL, c[2], &hi1, &lo1);
    uint64_t n0 = hi1 ^ c[1] ^ k0, n1 = lo1, n2 = hi0 ^ c[3] ^ k1, n3 = lo0;
    c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
  }
  memcpy(out, c, sizeof(c));
}

static void gen_init(orc_gen* g, uint64_t key) {
  memset(g, 0, sizeof(*g));
  g->key = key;
  g->pos = 4;
}

static uint64_t next64(orc_gen* g) {
  if (g->pos == 4) {
    g->ctr += 1;
    philox10(g->ctr, g->key, g->buf);
    g->pos = 0;
  }
  return g->buf[g->pos++];
}

static uint32_t next32(orc_gen* g) {
  if (g->has32) { g->has32 = 0; return g->u32; }
  uint64_t v = next64(g);
  g->has32 = 1;
  g->u32 = (uint32_t)(v >> 32);
  return (uint32_t)v;
}

static double next_double(orc_gen* g) { return (next64(g) >> 11) * (1.0 / 9007199254740992.0); }

static uint32_t lemire32(orc_gen* g, uint32_t rng /* inclusive max */) {
  const uint32_t excl = rng + 1;
  uint64_t m = (uint64_t)next32(g) * excl;
  uint32_t left = (uint32_t)m;
  if (left < excl) {
    const uint32_t threshold = (uint32_t)((0xFFFFFFFFu - rng) % excl);
    while (left < threshold) {
      m = (uint64_t)next32(g) * excl;
      left = (uint32_t)m;
    }
  }
  return (uint32_t)(m >> 32);
}

/* integers(0, d, size=cnt) for 1 <= d <= 2^32-1 */
static void integers(orc_gen* g, uint64_t d, int64_t cnt, int64_t* out) {
  if (d == 1) { for (int64_t i = 0; i < cnt; ++i) out[i] = 0; return; }
  for (int64_t i = 0; i < cnt; ++i) out[i] = lemire32(g, (uint32_t)(d - 1));
}

void orc_u32(uint64_t key, int64_t count, uint32_t* out) {
  orc_gen g; gen_init(&g, key);
  for (int64_t i = 0; i < count; ++i) out[i] = next32(&g);
}

int orc_countsketch(uint64_t key, int64_t m, int64_t d, int64_t* rows, double* signs) {
  if (d < 1 || d > 0xFFFFFFFFLL) return 1;
  orc_gen g; gen_init(&g, key);
  integers(&g, (uint64_t)d, m, rows);
  int64_t* tmp = (int64_t*)malloc(sizeof(int64_t) * (size_t)m);
  integers(&g, 2, m, tmp);
  for (int64_t i = 0; i < m; ++i) signs[i] = 2.0 * (double)tmp[i] - 1.0;
  free(tmp);
  return 0;
}

int orc_srht(uint64_t key, int64_t m_pad, int64_t d, double* signs, int64_t* sample) {
  if (m_pad > 0xFFFFFFFFLL) return 1;
  orc_gen g; gen_init(&g, key);
  int64_t* tmp = (int64_t*)malloc(sizeof(int64_t) * (size_t)m_pad);
  integers(&g, 2, m_pad, tmp);
  for (int64_t i = 0; i < m_pad; ++i) signs[i] = 2.0 * (double)tmp[i] - 1.0;
  for (int64_t i = 0; i < m_pad; ++i) tmp[i] = i;
  for (int64_t i = m_pad - 1; i >= 1; --i) {
    uint64_t mask = (uint64_t)i;
    mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4;
    mask |= mask >> 8; mask |= mask >> 16; mask |= mask >> 32;
    uint64_t v;
    while ((v = (next32(&g) & mask)) > (uint64_t)i) {}
    int64_t t = tmp[i]; tmp[i] = tmp[v]; tmp[v] = t;
  }
  memcpy(sample, tmp, sizeof(int64_t) * (size_t)d);
  free(tmp);
  return 0;
}

int orc_gaussian(uint64_t key, int64_t count, const uint64_t* ki, const double* wi,
                 const double* fi, double r, double inv_r, double* out) {
  orc_gen g; gen_init(&g, key);
  for (int64_t n = 0; n < count; ++n) {
    for (;;) {
      uint64_t rr = next64(&g);
      int idx = (int)(rr & 0xff);
      rr >>= 8;
      int sign = (int)(rr & 1);
      uint64_t rabs = (rr >> 1) & 0x000fffffffffffffULL;
      double x = rabs * wi[idx];
      if (sign) x = -x;
      if (rabs < ki[idx]) { out[n] = x; break; }
      if (idx == 0) {
        for (;;) {
          double xx = -inv_r * log1p(-next_double(&g));
          double yy = -log1p(-next_double(&g));
          if (yy + yy > xx * xx) {
            out[n] = ((rabs >> 8) & 1) ? -(r + xx) : r + xx;
            break;
          }
        }
        break;
      }
      if (((fi[idx - 1] - fi[idx]) * next_double(&g) + fi[idx]) < exp(-0.5 * x * x)) {
        out[n] = x;
        break;
      }
    }
  }
  return 0;
}

/* out (d x n, column-major, ld d) = S A for column-major A (ld lda). */
void orc_countsketch_fold(const int64_t* rows, const double* signs, int64_t m, int64_t n,
                          const double* A, int64_t lda, int64_t d, double* out) {
  memset(out, 0, sizeof(double) * (size_t)(d * n));
  for (int64_t j = 0; j < m; ++j) {
    const int64_t i = rows[j];
    const double s = signs[j];
    for (int64_t c = 0; c < n; ++c) out[c * d + i] += s * A[c * lda + j];
  }
}
