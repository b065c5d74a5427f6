// Host side of sketchls_b200: error plumbing, the bit-exact Philox4x64-10
// streams of numpy 2.3.5 (the generator behind sketchls/rng.py:43-45), the
// CountSketch / SRHT draws of sketch.py:93-127 and the CountSketch plan.
//
// Bit contract (numpy 2.3.5, verified by tests/test_host_rng.py against
// numpy itself): Generator(Philox(key=k)) runs Philox4x64-10 with key words
// (k, 0); the 256-bit counter is incremented *before* each block, so block
// q uses counter (q+1, 0, 0, 0) and yields u64 words 4q..4q+3 in order.
// next_uint32 splits each u64 low half first; the leftover half persists
// across `integers` calls.  integers(0, d) is Lemire's 32-bit method with
// rejection threshold (2^32 - d) mod d; permutation(n) is a top-down
// Fisher-Yates whose j comes from masked rejection on the u32 stream.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <thread>
#include <vector>

#include "skl_common.h"
#include "skl_philox.h"

namespace skl {

static thread_local std::string g_err;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
}
void clear_error() { g_err.clear(); }

int resolve_threads(int threads) {
  if (threads > 0) return threads;
  unsigned h = std::thread::hardware_concurrency();
  return h ? (int)std::min(h, 64u) : 1;
}

template <class F>
static void parallel_for(int64_t n, int threads, F&& f, int64_t grain = 4096) {
  // f(lo, hi) over [0, n) split in contiguous blocks of at least `grain`.
  threads = (int)std::max<int64_t>(1, std::min<int64_t>(threads, n / grain + 1));
  if (threads == 1) {
    f((int64_t)0, n);
    return;
  }
  std::vector<std::thread> pool;
  pool.reserve(threads);
  for (int t = 0; t < threads; ++t) {
    int64_t lo = n * t / threads, hi = n * (t + 1) / threads;
    pool.emplace_back([&f, lo, hi] { f(lo, hi); });
  }
  for (auto& th : pool) th.join();
}

// Fill out[i] = u32 at stream position pos0 + i.
static void fill_u32(uint64_t key, uint64_t pos0, int64_t count, uint32_t* out) {
  if (count <= 0) return;
  uint64_t p = pos0;
  int64_t i = 0;
  while (i < count) {
    uint64_t q = p >> 1;       // u64 index
    uint64_t blk = q >> 2;     // Philox block
    uint64_t w[4];
    philox_block(key, blk, w);
    // positions covered by this block: [blk*8, blk*8+8)
    uint64_t end = (blk + 1) * 8;
    while (p < end && i < count) {
      uint64_t word = w[(p >> 1) & 3];
      out[i++] = (p & 1) ? (uint32_t)(word >> 32) : (uint32_t)word;
      ++p;
    }
  }
}

static void fill_u32_par(uint64_t key, uint64_t pos0, int64_t count, uint32_t* out, int threads) {
  parallel_for(count, threads, [&](int64_t lo, int64_t hi) { fill_u32(key, pos0 + lo, hi - lo, out + lo); });
}

}  // namespace skl

using namespace skl;

// ---------------------------------------------------------------------------
// CountSketch plan (see the header).
//
// Schedule of one warp (its contiguous bucket range) over the chunks, built
// sequentially chunk after chunk because a lane keeps its last bucket's sum
// in a register into the next chunk.  Per chunk:
//   * the non-empty buckets of the warp form a pool, each with its rows in
//     ascending order (stable counting sort of the chunk by bucket);
//   * step 0: a lane whose current bucket is in the pool continues it (no
//     reload); every other lane switches -- to a new bucket from the pool,
//     or to the dummy slot so its held sum is written back before another
//     lane can read it;
//   * at every step a lane without work takes the pool bucket that keeps
//     this step's shared-memory banks least loaded (first-row gather bank,
//     then accumulator bank), longest buckets first;
//   * idle lanes emit padding that adds +0.0 to the bucket they hold.
// Entry word: byte offset 8*row (8*chunk = zero slot) | bucket << 16 |
// sign << 31; a lane reloads whenever the bucket field changes.
static int64_t plan_head(int warps) { return (warps + 1 + 3) / 4 * 4; }

namespace {

// Chunks are planned in independent segments of this many chunks (lanes
// start a segment holding no bucket), which is what makes the planner
// parallel; the segmentation never depends on the thread count.
constexpr int64_t kPlanSegment = 32;

// Entries of a chunk: source row j contributes `spr` entries (e = j * spr + q:
// bucket rows[(r0 + j) * spr + q], sign signs[same]) -- one for a
// CountSketch, s for a sparse sign embedding (distinct buckets per row).
struct ChunkSort {
  std::vector<uint32_t> cnt, start, pos;
  std::vector<uint16_t> sorted;  // entry index e, bucket-major, rows ascending
  int spr;
  ChunkSort(int64_t d, int64_t chunk, int spr_)
      : cnt((size_t)d), start((size_t)d), pos((size_t)d), sorted((size_t)(chunk * spr_)),
        spr(spr_) {}
  // stable counting sort of chunk k's entries by bucket; false on a bad bucket
  bool run(const int32_t* rows, int64_t m, int64_t d, int64_t chunk, int64_t k) {
    const int64_t r0 = k * chunk;
    const int len = (int)std::min<int64_t>(chunk, m - r0) * spr;
    std::fill(cnt.begin(), cnt.end(), 0u);
    for (int e = 0; e < len; ++e) {
      const int32_t r = rows[r0 * spr + e];
      if (r < 0 || r >= d) return false;
      ++cnt[(size_t)r];
    }
    uint32_t run = 0;
    for (int64_t b = 0; b < d; ++b) {
      start[(size_t)b] = run;
      pos[(size_t)b] = run;
      run += cnt[(size_t)b];
    }
    for (int e = 0; e < len; ++e) sorted[pos[(size_t)rows[r0 * spr + e]]++] = (uint16_t)e;
    return true;
  }
  // source row (within the chunk) of the t-th sorted entry
  uint32_t row(size_t t) const { return (uint32_t)sorted[t] / (uint32_t)spr; }
};

struct WarpSched {
  uint32_t cur[32];
  std::vector<uint32_t> pool, bank[16], byc;
  std::vector<uint8_t> taken;
  size_t bhead[16];
};

// Schedules warp w's buckets [b0, b1) of chunk k (sorted in S) onto the 32
// lanes, appending rows of 32 words to `words`.
void schedule_chunk(const int8_t* signs, int64_t d, int64_t chunk, int64_t r0, int64_t b0,
                    int64_t b1, const ChunkSort& S, WarpSched& W, std::vector<uint32_t>& words) {
  const uint32_t dummy = (uint32_t)d;
  const uint32_t zero_off = (uint32_t)(8 * chunk);
  uint32_t* cur = W.cur;
  uint32_t pos[32];
  int32_t run[32];
  // pool = non-empty buckets by descending count, ties by id (counting sort)
  uint32_t maxc = 0;
  for (int64_t b = b0; b < b1; ++b) maxc = std::max(maxc, S.cnt[(size_t)b]);
  if (W.byc.size() < (size_t)maxc + 2) W.byc.resize((size_t)maxc + 2);
  std::fill(W.byc.begin(), W.byc.begin() + maxc + 2, 0u);
  for (int64_t b = b0; b < b1; ++b) ++W.byc[S.cnt[(size_t)b]];
  uint32_t npool = 0;
  for (int64_t c = (int64_t)maxc; c >= 1; --c) {
    const uint32_t h = W.byc[(size_t)c];
    W.byc[(size_t)c] = npool;
    npool += h;
  }
  W.pool.resize(npool);
  for (int64_t b = b0; b < b1; ++b) {
    const uint32_t c = S.cnt[(size_t)b];
    if (c) W.pool[W.byc[c]++] = (uint32_t)b;
  }
  if (W.taken.size() < (size_t)(b1 - b0 + 1)) W.taken.resize((size_t)(b1 - b0 + 1));
  std::fill(W.taken.begin(), W.taken.end(), 0);
  for (int g = 0; g < 16; ++g) {
    W.bank[g].clear();
    W.bhead[g] = 0;
  }
  for (uint32_t b : W.pool) W.bank[S.row(S.start[b]) & 15].push_back(b);
  size_t left = W.pool.size();
  for (int l = 0; l < 32; ++l) run[l] = -1;
  for (int l = 0; l < 32; ++l) {  // continuations keep their register sum
    const uint32_t b = cur[l];
    if (b != dummy && S.cnt[b] && !W.taken[b - b0]) {
      W.taken[b - b0] = 1;
      --left;
      run[l] = (int32_t)b;
      pos[l] = 0;
    }
  }
  bool first = true;
  for (;;) {
    bool busy = false;
    for (int l = 0; l < 32; ++l) busy |= run[l] >= 0;
    if (!first && !busy && !left) break;
    int gl[16] = {0}, al[16] = {0};
    for (int l = 0; l < 32; ++l)
      if (run[l] >= 0) gl[S.row(S.start[(uint32_t)run[l]] + pos[l]) & 15]++;
    for (int l = 0; l < 32 && left; ++l) {
      if (run[l] >= 0) continue;
      // least-loaded gather bank with work left, then the least-loaded
      // accumulator bank among its first few (longest) buckets
      int gbest = -1;
      for (int g = 0; g < 16; ++g) {
        while (W.bhead[g] < W.bank[g].size() && W.taken[W.bank[g][W.bhead[g]] - b0]) ++W.bhead[g];
        if (W.bhead[g] < W.bank[g].size() && (gbest < 0 || gl[g] < gl[gbest])) gbest = g;
      }
      const std::vector<uint32_t>& q = W.bank[gbest];
      size_t pick = W.bhead[gbest];
      int abest = al[q[pick] & 15];
      for (size_t t = pick + 1, seen = 0; t < q.size() && seen < 4 && abest > 0; ++t) {
        if (W.taken[q[t] - b0]) continue;
        ++seen;
        if (al[q[t] & 15] < abest) {
          abest = al[q[t] & 15];
          pick = t;
        }
      }
      const uint32_t b = q[pick];
      W.taken[b - b0] = 1;
      --left;
      run[l] = (int32_t)b;
      pos[l] = 0;
      gl[gbest]++;
      al[b & 15]++;
    }
    bool any = false;
    for (int l = 0; l < 32; ++l) {
      uint32_t word;
      if (run[l] >= 0) {
        const uint32_t b = (uint32_t)run[l];
        const uint32_t e = S.sorted[S.start[b] + pos[l]];
        const uint32_t j = e / (uint32_t)S.spr;
        word = (8u * j) | (b << 16) | ((signs[r0 * S.spr + e] < 0 ? 1u : 0u) << 31);
        cur[l] = b;
        if (++pos[l] == S.cnt[b]) run[l] = -1;
        any = true;
      } else if (first && cur[l] != dummy) {
        word = zero_off | (dummy << 16);  // write the held sum back
        cur[l] = dummy;
        any = true;
      } else {
        word = zero_off | (cur[l] << 16);  // padding: +0.0 to the held bucket
      }
      words.push_back(word);
    }
    first = false;
    if (!any) {
      words.resize(words.size() - 32);
      break;
    }
  }
}

// Runs the schedule of chunks [k0, k1) for all warps; per chunk calls
// sink(k, warp_rows[warps], words_of_warp[warps]).
template <class Sink>
bool plan_segment(const int32_t* rows, const int8_t* signs, int64_t m, int spr, int64_t d,
                  int64_t chunk, int warps, int64_t k0, int64_t k1, Sink&& sink) {
  const int64_t gsize = (d + warps - 1) / warps;
  ChunkSort S(d, chunk, spr);
  std::vector<WarpSched> W((size_t)warps);
  for (auto& ws : W)
    for (int l = 0; l < 32; ++l) ws.cur[l] = (uint32_t)d;
  std::vector<std::vector<uint32_t>> words((size_t)warps);
  for (int64_t k = k0; k < k1; ++k) {
    if (!S.run(rows, m, d, chunk, k)) return false;
    for (int w = 0; w < warps; ++w) {
      const int64_t b0 = std::min<int64_t>(d, w * gsize), b1 = std::min<int64_t>(d, b0 + gsize);
      words[(size_t)w].clear();
      schedule_chunk(signs, d, chunk, k * chunk, b0, b1, S, W[(size_t)w], words[(size_t)w]);
    }
    sink(k, words);
  }
  return true;
}

}  // namespace


extern "C" {

const char* skl_last_error(void) { return skl::g_err.c_str(); }
int skl_abi_version(void) { return 1; }

uint64_t skl_splitmix64(uint64_t z) { return splitmix64(z); }

int skl_rng_u32(uint64_t key, uint64_t offset, int64_t count, uint32_t* out) {
  SKL_REQUIRE(count >= 0 && (count == 0 || out), SKL_ERR_INVALID, "skl_rng_u32: bad arguments");
  fill_u32(key, offset, count, out);
  return SKL_OK;
}

int skl_rng_u64(uint64_t key, uint64_t offset, int64_t count, uint64_t* out) {
  SKL_REQUIRE(count >= 0 && (count == 0 || out), SKL_ERR_INVALID, "skl_rng_u64: bad arguments");
  int64_t i = 0;
  uint64_t q = offset;
  while (i < count) {
    uint64_t w[4];
    philox_block(key, q >> 2, w);
    for (uint64_t k = q & 3; k < 4 && i < count; ++k, ++q) out[i++] = w[k];
  }
  return SKL_OK;
}

// CountSketch draws, sketch.py:98-99:
//   rows  = rng.integers(0, d, size=m)      (Lemire u32, rejection-filtered)
//   signs = 2 * rng.integers(0, 2, size=m) - 1   (u32 >> 31, never rejects)
int skl_rng_countsketch(uint64_t key, int64_t m, int64_t d, int32_t* rows, int8_t* signs,
                        int threads, uint64_t* u32_consumed) {
  clear_error();
  SKL_REQUIRE(m >= 1 && d >= 1 && rows && signs, SKL_ERR_INVALID,
              "skl_rng_countsketch: bad arguments (m=%lld, d=%lld)", (long long)m, (long long)d);
  SKL_REQUIRE(d <= 0x7fffffffLL, SKL_ERR_SPEC, "embed_dim %lld exceeds the 31-bit bucket range",
              (long long)d);
  threads = resolve_threads(threads);
  uint64_t pos = 0;
  if (d == 1) {
    // integers(0, 1) draws nothing (rng == 0 branch of numpy's bounded fill).
    std::fill(rows, rows + m, 0);
  } else {
    const uint64_t dd = (uint64_t)d;
    const uint32_t threshold = (uint32_t)((0x100000000ULL - dd) % dd);
    // Pass 1: accept-test every candidate position in [0, m) in parallel.
    std::atomic<int64_t> rejections{0};
    parallel_for(m, threads, [&](int64_t lo, int64_t hi) {
      std::vector<uint32_t> buf(8192);
      int64_t local_rej = 0;
      for (int64_t s = lo; s < hi; s += 8192) {
        int64_t cnt = std::min<int64_t>(8192, hi - s);
        fill_u32(key, (uint64_t)s, cnt, buf.data());
        for (int64_t i = 0; i < cnt; ++i) {
          uint64_t prod = (uint64_t)buf[i] * dd;
          uint32_t left = (uint32_t)prod;
          if (left < threshold) {
            ++local_rej;
            rows[s + i] = -1;
          } else {
            rows[s + i] = (int32_t)(prod >> 32);
          }
        }
      }
      rejections += local_rej;
    });
    pos = (uint64_t)m;
    if (rejections.load() > 0) {
      // Rare (probability threshold / 2^32 per draw): compact the accepted
      // draws in stream order and keep drawing until m are accepted.
      int64_t w = 0;
      for (int64_t i = 0; i < m; ++i)
        if (rows[i] >= 0) rows[w++] = rows[i];
      while (w < m) {
        uint32_t u;
        fill_u32(key, pos++, 1, &u);
        uint64_t prod = (uint64_t)u * dd;
        if ((uint32_t)prod >= threshold) rows[w++] = (int32_t)(prod >> 32);
      }
    }
  }
  const uint64_t sign_pos = pos;
  parallel_for(m, threads, [&](int64_t lo, int64_t hi) {
    std::vector<uint32_t> buf(8192);
    for (int64_t s = lo; s < hi; s += 8192) {
      int64_t cnt = std::min<int64_t>(8192, hi - s);
      fill_u32(key, sign_pos + (uint64_t)s, cnt, buf.data());
      for (int64_t i = 0; i < cnt; ++i) signs[s + i] = (buf[i] >> 31) ? 1 : -1;
    }
  });
  if (u32_consumed) *u32_consumed = sign_pos + (uint64_t)m;
  return SKL_OK;
}

// SRHT draws, sketch.py:117-119:
//   sign_diag  = 2 * rng.integers(0, 2, size=m_pad) - 1
//   row_sample = rng.permutation(m_pad)[:d]
// The permutation is numpy's top-down Fisher-Yates (swap a[i], a[j_i] for
// i = n-1 .. 1).  Only a[:d] is needed, so instead of materialising the
// n-element array we record the j_i sequence and trace the final positions
// 0..d-1 backwards through the swaps with a small open-addressing table.
int skl_rng_srht(uint64_t key, int64_t m_pad, int64_t d, int8_t* signs, int64_t* row_sample,
                 int threads) {
  clear_error();
  SKL_REQUIRE(m_pad >= 1 && d >= 1 && d <= m_pad && signs && row_sample, SKL_ERR_INVALID,
              "skl_rng_srht: bad arguments");
  SKL_REQUIRE(m_pad <= 0x100000000LL, SKL_ERR_SPEC, "padded dimension %lld exceeds 2^32",
              (long long)m_pad);
  threads = resolve_threads(threads);
  parallel_for(m_pad, threads, [&](int64_t lo, int64_t hi) {
    std::vector<uint32_t> buf(8192);
    for (int64_t s = lo; s < hi; s += 8192) {
      int64_t cnt = std::min<int64_t>(8192, hi - s);
      fill_u32(key, (uint64_t)s, cnt, buf.data());
      for (int64_t i = 0; i < cnt; ++i) signs[s + i] = (buf[i] >> 31) ? 1 : -1;
    }
  });
  const int64_t n = m_pad;
  if (n == 1) {
    row_sample[0] = 0;
    return SKL_OK;
  }
  // Forward pass: draw j_i for i = n-1 .. 1 (sequential rejection).
  std::vector<uint32_t> js((size_t)(n - 1));  // js[i-1] = j_i
  uint64_t pos = (uint64_t)n;
  const int64_t BUF = 1 << 16;
  std::vector<uint32_t> buf(BUF);
  int64_t bi = BUF;
  auto next32 = [&]() -> uint32_t {
    if (bi == BUF) {
      fill_u32_par(key, pos, BUF, buf.data(), std::min(threads, 4));
      pos += BUF;
      bi = 0;
    }
    return buf[bi++];
  };
  for (int64_t i = n - 1; i >= 1; --i) {
    uint64_t mask = (uint64_t)i;
    mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4;
    mask |= mask >> 8; mask |= mask >> 16; mask |= mask >> 32;
    uint64_t v;
    do {
      v = next32() & mask;
    } while (v > (uint64_t)i);
    js[(size_t)(i - 1)] = (uint32_t)v;
  }
  // Backward trace: position p at the end came from position pos(p) at the
  // start; walk the swaps in reverse (i = 1 .. n-1).
  size_t cap = 1;
  while (cap < (size_t)d * 4) cap <<= 1;
  std::vector<int64_t> hkey(cap, -1);
  std::vector<int64_t> hval(cap, -1);
  // Table: current position -> tracked item (final position p), with
  // tombstones for moved keys.  Undoing swap (i, j): if both positions are
  // tracked their items trade places, otherwise the one item moves.
  const int64_t TOMB = -2;
  auto find = [&](int64_t k) -> size_t {
    size_t h = (size_t)(splitmix64((uint64_t)k) & (cap - 1));
    while (hkey[h] != -1) {
      if (hkey[h] == k) return h;
      h = (h + 1) & (cap - 1);
    }
    return (size_t)-1;
  };
  auto insert = [&](int64_t k, int64_t v) {
    size_t h = (size_t)(splitmix64((uint64_t)k) & (cap - 1));
    while (hkey[h] != -1 && hkey[h] != TOMB) h = (h + 1) & (cap - 1);
    hkey[h] = k;
    hval[h] = v;
  };
  for (int64_t p = 0; p < d; ++p) insert(p, p);
  int64_t tombs = 0;
  for (int64_t i = 1; i <= n - 1; ++i) {
    int64_t j = js[(size_t)(i - 1)];
    if (j == i) continue;
    size_t hi_ = find(i), hj = find(j);
    bool ti = hi_ != (size_t)-1, tj = hj != (size_t)-1;
    if (ti && tj) {
      std::swap(hval[hi_], hval[hj]);
    } else if (ti) {
      int64_t item = hval[hi_];
      hkey[hi_] = TOMB;
      ++tombs;
      insert(j, item);
    } else if (tj) {
      int64_t item = hval[hj];
      hkey[hj] = TOMB;
      ++tombs;
      insert(i, item);
    }
    if (tombs > (int64_t)cap / 4) {
      // rebuild without tombstones
      std::vector<std::pair<int64_t, int64_t>> live;
      live.reserve(d);
      for (size_t h = 0; h < cap; ++h)
        if (hkey[h] >= 0) live.emplace_back(hkey[h], hval[h]);
      std::fill(hkey.begin(), hkey.end(), -1);
      for (auto& kv : live) insert(kv.first, kv.second);
      tombs = 0;
    }
  }
  for (size_t h = 0; h < cap; ++h)
    if (hkey[h] >= 0) row_sample[hval[h]] = hkey[h];
  return SKL_OK;
}

static int lanes_plan(const int32_t* rows, const int8_t* signs, int64_t m, int spr, int64_t d,
                      int64_t chunk, int warps, uint32_t* lanes, int64_t* chunk_off,
                      int threads) {
  SKL_REQUIRE(rows && signs && chunk_off && m >= 1 && d >= 1 && spr >= 1, SKL_ERR_INVALID,
              "skl_countsketch_plan: bad arguments");
  SKL_REQUIRE(chunk * spr <= 65536, SKL_ERR_INVALID,
              "plan chunk %lld x %d entries per row exceeds the 16-bit entry index",
              (long long)chunk, spr);
  SKL_REQUIRE(d <= 32767, SKL_ERR_SPEC, "countsketch plan: embed_dim %lld > 32767",
              (long long)d);
  SKL_REQUIRE(chunk >= 8 && chunk <= 4088 && chunk % 8 == 0, SKL_ERR_INVALID,
              "plan chunk must be a multiple of 8 in [8, 4088], got %lld", (long long)chunk);
  SKL_REQUIRE(warps >= 1 && warps <= 31, SKL_ERR_INVALID,
              "plan warps must be in [1, 31], got %d", warps);
  const int64_t nch = (m + chunk - 1) / chunk;
  const int64_t head = plan_head(warps);
  const int64_t nseg = (nch + kPlanSegment - 1) / kPlanSegment;
  threads = resolve_threads(threads);
  // pass 1: list rows per (chunk, warp)
  std::vector<uint32_t> R((size_t)(nch * warps));
  std::atomic<int> bad{0};
  parallel_for(nseg, threads, [&](int64_t lo, int64_t hi) {
    for (int64_t g = lo; g < hi; ++g) {
      const int64_t k0 = g * kPlanSegment, k1 = std::min(nch, k0 + kPlanSegment);
      if (!plan_segment(rows, signs, m, spr, d, chunk, warps, k0, k1,
                        [&](int64_t k, const std::vector<std::vector<uint32_t>>& wd) {
                          for (int w = 0; w < warps; ++w)
                            R[(size_t)(k * warps + w)] = (uint32_t)(wd[(size_t)w].size() / 32);
                        }))
        bad = 1;
    }
  }, 1);
  SKL_REQUIRE(!bad.load(), SKL_ERR_INVALID, "bucket index out of range [0, %lld)", (long long)d);
  std::vector<int64_t> off((size_t)nch + 1, 0);
  for (int64_t k = 0; k < nch; ++k) {
    int64_t rws = 0;
    for (int w = 0; w < warps; ++w) rws += R[(size_t)(k * warps + w)];
    off[(size_t)k + 1] = off[(size_t)k] + head + 32 * rws;
  }
  if (!lanes) {
    std::copy(off.begin(), off.end(), chunk_off);
    return SKL_OK;
  }
  for (int64_t k = 0; k <= nch; ++k)
    SKL_REQUIRE(chunk_off[k] == off[(size_t)k], SKL_ERR_INVALID,
                "countsketch plan: chunk offsets do not match this (rows, d, chunk, warps)");
  // pass 2: emit
  parallel_for(nseg, threads, [&](int64_t lo, int64_t hi) {
    for (int64_t g = lo; g < hi; ++g) {
      const int64_t k0 = g * kPlanSegment, k1 = std::min(nch, k0 + kPlanSegment);
      plan_segment(rows, signs, m, spr, d, chunk, warps, k0, k1,
                   [&](int64_t k, const std::vector<std::vector<uint32_t>>& wd) {
                     uint32_t* blk = lanes + off[(size_t)k];
                     uint32_t base = 0;
                     for (int w = 0; w < warps; ++w) {
                       blk[w] = base;
                       std::copy(wd[(size_t)w].begin(), wd[(size_t)w].end(),
                                 blk + head + 32 * (int64_t)base);
                       base += (uint32_t)(wd[(size_t)w].size() / 32);
                     }
                     for (int64_t w = warps; w < head; ++w) blk[w] = base;
                   });
    }
  }, 1);
  return SKL_OK;
}

int skl_countsketch_plan(const int32_t* rows, const int8_t* signs, int64_t m, int64_t d,
                         int64_t chunk, int warps, uint32_t* lanes, int64_t* chunk_off,
                         int threads) {
  clear_error();
  return lanes_plan(rows, signs, m, 1, d, chunk, warps, lanes, chunk_off, threads);
}

int skl_sparsesign_plan(const int32_t* rows, const int8_t* signs, int64_t m, int spr, int64_t d,
                        int64_t chunk, int warps, uint32_t* lanes, int64_t* chunk_off,
                        int threads) {
  clear_error();
  return lanes_plan(rows, signs, m, spr, d, chunk, warps, lanes, chunk_off, threads);
}

}  // extern "C"
