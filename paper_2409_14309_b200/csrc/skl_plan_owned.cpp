// Register-owned CountSketch plan (host).  See include/sketchls_b200.h
// (skl_countsketch_plan_owned) for the block format.
//
// Bucket b is owned for the whole apply by consumer thread t = b % (32 W)
// (lane t % 32 of warp t / 32), slot b / (32 W): the thread keeps the
// bucket's running sum in a register, so the device kernel never stages
// accumulators in shared memory.  The strided map spreads any d evenly over
// the warps.
// Per chunk, a lane's list is the union of its 4, 8 or 16 buckets' rows
// (slots = ceil(d / 32 W) rounded up to a power of two); rows of
// one bucket stay in ascending order (scipy csr_matvecs' fold order, so the
// result is bitwise-equal to the reference), while the four streams are
// interleaved step by step to spread the warp's 32 shared-memory gathers
// over the banks.  Lists are padded to the longest lane with entries that
// add +0.0 from a zero slot.
#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <thread>
#include <vector>

#include "skl_common.h"

namespace {

constexpr int kMaxSlots = 8;

template <class F>
void par_for(int64_t n, int threads, F&& f) {
  threads = (int)std::max<int64_t>(1, std::min<int64_t>(threads, n / 2 + 1));
  if (threads == 1) {
    f((int64_t)0, n);
    return;
  }
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) {
    const int64_t lo = n * t / threads, hi = n * (t + 1) / threads;
    pool.emplace_back([&f, lo, hi] { f(lo, hi); });
  }
  for (auto& th : pool) th.join();
}

int64_t head_words(int warps) { return (warps + 1 + 7) / 8 * 8; }

struct OwnedScratch {
  std::vector<uint32_t> cnt, start, pos, rows_of;
  std::vector<uint16_t> sorted;
  OwnedScratch(int64_t d, int64_t entries)
      : cnt((size_t)d), start((size_t)d), pos((size_t)d), sorted((size_t)entries) {}
};

// Returns the block length (u16 words) of chunk k; fills blk when non-null.
// -1 on a bucket out of range.  Source row j contributes `spr` entries
// (rows/signs[j * spr + q], distinct buckets -- 1 for CountSketch, s for a
// sparse sign embedding).  sorted[] holds row | negative << 15.
int64_t owned_chunk(const int32_t* rows, const int8_t* signs, int64_t m, int spr, int64_t d,
                    int64_t chunk, int warps, int64_t k, OwnedScratch& S, uint16_t* blk) {
  const int64_t r0 = k * chunk;
  const int len = (int)std::min<int64_t>(chunk, m - r0);
  std::fill(S.cnt.begin(), S.cnt.end(), 0u);
  for (int64_t e = 0; e < (int64_t)len * spr; ++e) {
    const int32_t r = rows[r0 * spr + e];
    if (r < 0 || r >= d) return -1;
    ++S.cnt[(size_t)r];
  }
  uint32_t run = 0;
  for (int64_t b = 0; b < d; ++b) {
    S.start[(size_t)b] = run;
    S.pos[(size_t)b] = run;
    run += S.cnt[(size_t)b];
  }
  for (int j = 0; j < len; ++j)
    for (int q = 0; q < spr; ++q) {
      const int64_t e = (r0 + j) * spr + q;
      S.sorted[S.pos[(size_t)rows[e]]++] = (uint16_t)(j | ((signs[e] < 0 ? 1u : 0u) << 15));
    }
  const int64_t head = head_words(warps);
  const int nsl = skl::owned_slots(d, warps), rb = skl::owned_row_bits(nsl);
  const uint32_t rmask = (1u << rb) - 1u;
  const uint16_t pad = (uint16_t)chunk;  // zero slot, slot 0, positive
  int64_t total_rows = 0;
  for (int w = 0; w < warps; ++w) {
    if (blk) blk[w] = (uint16_t)total_rows;
    int maxlen = 0;
    for (int l = 0; l < 32; ++l) {
      int n = 0;
      for (int s = 0; s < nsl; ++s) {
        const int64_t b = (int64_t)w * 32 + l + (int64_t)s * 32 * warps;
        if (b < d) n += (int)S.cnt[(size_t)b];
      }
      maxlen = std::max(maxlen, n);
    }
    if (blk) {
      uint16_t* R = blk + head + total_rows * 32;
      uint32_t nxt[32][kMaxSlots];  // next entry index per lane and slot
      for (int l = 0; l < 32; ++l)
        for (int s = 0; s < kMaxSlots; ++s) nxt[l][s] = 0;
      for (int step = 0; step < maxlen; ++step) {
        int load[16] = {0};
        for (int l = 0; l < 32; ++l) {
          int best = -1, bload = 1 << 30;
          uint32_t bleft = 0;
          for (int s = 0; s < nsl; ++s) {
            const int64_t b = (int64_t)w * 32 + l + (int64_t)s * 32 * warps;
            if (b >= d || nxt[l][s] >= S.cnt[(size_t)b]) continue;
            const uint32_t j = S.sorted[S.start[(size_t)b] + nxt[l][s]] & 0x1fffu;
            const int ld = load[j & 15];
            const uint32_t left = S.cnt[(size_t)b] - nxt[l][s];
            if (ld < bload || (ld == bload && left > bleft)) {
              best = s;
              bload = ld;
              bleft = left;
            }
          }
          uint16_t word = pad;
          if (best >= 0) {
            const int64_t b = (int64_t)w * 32 + l + (int64_t)best * 32 * warps;
            const uint32_t e = S.sorted[S.start[(size_t)b] + nxt[l][best]++];
            const uint32_t j = e & rmask;
            load[j & 15]++;
            word = (uint16_t)(j | ((uint32_t)best << rb) | (e & 0x8000u));
          }
          R[(size_t)step * 32 + l] = word;
        }
      }
    }
    total_rows += maxlen;
  }
  if (blk)
    for (int64_t w = warps; w < head; ++w) blk[w] = (uint16_t)total_rows;
  return head + total_rows * 32;
}

int plan_owned(const int32_t* rows, const int8_t* signs, int64_t m, int spr, int64_t d,
                      int64_t chunk, int warps, uint16_t* lanes, int64_t* chunk_off,
                      int threads) {
  SKL_REQUIRE(rows && signs && chunk_off && m >= 1 && d >= 1 && spr >= 1, SKL_ERR_INVALID,
              "owned plan: bad arguments");
  SKL_REQUIRE(warps >= 1 && warps <= 31 && skl::owned_slots(d, warps) > 0, SKL_ERR_SPEC,
              "owned plan: embed_dim %lld needs more than %d warps x 32 lanes x %d slots",
              (long long)d, warps, kMaxSlots);
  const int64_t cmax = skl::owned_max_chunk(skl::owned_slots(d, warps));
  SKL_REQUIRE(chunk >= 8 && chunk <= cmax && chunk % 8 == 0, SKL_ERR_INVALID,
              "owned plan chunk must be a multiple of 8 in [8, %lld], got %lld", (long long)cmax,
              (long long)chunk);
  const int64_t nch = (m + chunk - 1) / chunk;
  threads = skl::resolve_threads(threads);
  std::vector<int64_t> sz((size_t)nch);
  std::atomic<int> bad{0};
  par_for(nch, threads, [&](int64_t lo, int64_t hi) {
    OwnedScratch S(d, chunk * spr);
    for (int64_t k = lo; k < hi; ++k) {
      const int64_t n = owned_chunk(rows, signs, m, spr, d, chunk, warps, k, S, nullptr);
      if (n < 0 || n > 65535 * 32) {
        bad = n < 0 ? 1 : 2;
        return;
      }
      sz[(size_t)k] = n;
    }
  });
  SKL_REQUIRE(bad.load() != 1, SKL_ERR_INVALID, "bucket index out of range [0, %lld)", (long long)d);
  SKL_REQUIRE(bad.load() != 2, SKL_ERR_SPEC, "owned plan: chunk block too large");
  if (!lanes) {
    chunk_off[0] = 0;
    for (int64_t k = 0; k < nch; ++k) chunk_off[k + 1] = chunk_off[k] + sz[(size_t)k];
    return SKL_OK;
  }
  for (int64_t k = 0; k < nch; ++k)
    SKL_REQUIRE(chunk_off[k + 1] - chunk_off[k] == sz[(size_t)k], SKL_ERR_INVALID,
                "owned plan: chunk offsets do not match");
  par_for(nch, threads, [&](int64_t lo, int64_t hi) {
    OwnedScratch S(d, chunk * spr);
    for (int64_t k = lo; k < hi; ++k)
      owned_chunk(rows, signs, m, spr, d, chunk, warps, k, S, lanes + chunk_off[k]);
  });
  return SKL_OK;
}

}  // namespace

extern "C" int skl_countsketch_plan_owned(const int32_t* rows, const int8_t* signs, int64_t m,
                                          int64_t d, int64_t chunk, int warps, uint16_t* lanes,
                                          int64_t* chunk_off, int threads) {
  skl::clear_error();
  return plan_owned(rows, signs, m, 1, d, chunk, warps, lanes, chunk_off, threads);
}

extern "C" int skl_sparsesign_plan_owned(const int32_t* rows, const int8_t* signs, int64_t m,
                                         int64_t s, int64_t d, int64_t chunk, int warps,
                                         uint16_t* lanes, int64_t* chunk_off, int threads) {
  skl::clear_error();
  SKL_REQUIRE(s >= 1 && s <= d, SKL_ERR_SPEC, "sparse sign plan: sparsity %lld out of [1, d]",
              (long long)s);
  return plan_owned(rows, signs, m, (int)s, d, chunk, warps, lanes, chunk_off, threads);
}
