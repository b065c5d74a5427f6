/*
 * sketchls_b200.h — C-ABI of the B200-native sketch-and-solve engine.
 *
 * This is the drop-in boundary for the reference's hot path
 * (`sketchls`, arxiv 2409.14309): the bodies of `build_sketch`,
 * `_apply`, `economy_qr`, `_apply_inverse_r` and `_residual_norm`.
 * Every entry point takes plain pointers and sizes (no torch types),
 * returns an `int` status (SKL_OK == 0) and on failure leaves a message
 * retrievable with skl_last_error() (thread-local, so the ABI is
 * reentrant: inputs are borrowed read-only, outputs are caller-owned,
 * each call runs on the caller's CUDA stream).
 *
 * Layout conventions follow the reference carriers
 * (/root/reference/pkg/src/sketchls/linalg.py:31-53, 56-114, 117-133):
 * dense matrices are fp64 column-major with a leading dimension,
 * vectors are contiguous fp64, CSR uses int64 indptr/indices with
 * strictly increasing columns per row.
 *
 * Pointers documented as "device" must be CUDA device pointers; "host"
 * pointers are ordinary (preferably pinned) host memory.
 */
#ifndef SKETCHLS_B200_H
#define SKETCHLS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes; the Python host maps them onto the reference's exception
 * taxonomy (/root/reference/pkg/src/sketchls/errors.py:8-37). */
enum {
  SKL_OK = 0,
  SKL_ERR_SHAPE = 1,     /* ShapeError            errors.py:12 */
  SKL_ERR_SPEC = 2,      /* SpecError             errors.py:16 */
  SKL_ERR_SINGULAR = 3,  /* SingularFactorError   errors.py:24 */
  SKL_ERR_CAPACITY = 4,  /* CapacityError         errors.py:32 */
  SKL_ERR_CUDA = 5,      /* device failure (SketchlsError) */
  SKL_ERR_INVALID = 6,   /* bad argument / layout (ValueError) */
  SKL_ERR_NCCL = 7       /* collective failure (SketchlsError) */
};

/* Message of the last failing call on this thread ("" if none). */
const char* skl_last_error(void);
/* ABI version: bump on incompatible signature changes. */
int skl_abi_version(void);

/* ---------------------------------------------------------------------
 * Seeds and the bit-exact host RNG (numpy 2.3.5 Philox4x64-10 streams).
 * Replaces rng.py:19-45 and the draws in sketch.py:93-127.
 * ------------------------------------------------------------------- */

/* One splitmix64 step.  Replaces rng.py:19-24 (`splitmix64`). */
uint64_t skl_splitmix64(uint64_t z);

/* Raw u32 stream of Generator(Philox(key)) starting at u32 position
 * `offset` (low half of each u64 first).  Test hook for the bit contract
 * behind rng.py:43-45 (`stream`). */
int skl_rng_u32(uint64_t key, uint64_t offset, int64_t count, uint32_t* out);
/* Raw u64 stream (next_uint64 order) from u64 position `offset`. */
int skl_rng_u64(uint64_t key, uint64_t offset, int64_t count, uint64_t* out);

/* CountSketch hashes: rows[j] = integers(0, d, m)[j], signs[j] = +-1 from
 * the following integers(0, 2, m).  Replaces sketch.py:97-99.
 * host outputs; `threads` <= 0 means all hardware threads.
 * *u32_consumed (optional) receives the number of u32 draws used. */
int skl_rng_countsketch(uint64_t key, int64_t m, int64_t d, int32_t* rows, int8_t* signs,
                        int threads, uint64_t* u32_consumed);

/* SRHT sign diagonal over m_pad draws and row_sample = permutation(m_pad)[:d].
 * Replaces sketch.py:116-127.  host outputs. */
int skl_rng_srht(uint64_t key, int64_t m_pad, int64_t d, int8_t* signs, int64_t* row_sample,
                 int threads);

/* Gaussian sketch entries G[i, j] = standard_normal((d, m))[i, j] / sqrt(d),
 * written column-major into a device buffer (ld = ldg >= d), generated on
 * device by a resynchronising parallel ziggurat over the Philox stream.
 * Replaces sketch.py:94-96.  The ziggurat tables must have been installed
 * once with skl_gaussian_set_tables (extracted from the installed numpy). */
int skl_gaussian_set_tables(const uint64_t* ki, const double* wi, const double* fi);
int skl_rng_gaussian_device(uint64_t key, int64_t d, int64_t m, double* G_dev, int64_t ldg,
                            void* stream);
/* Standard normals of Generator(Philox(key)) starting at 64-bit stream word
 * `start_word` (numpy's random_standard_normal, one ziggurat draw after
 * another), written C-order as rows x cols into a device buffer with row
 * stride ld >= cols; *end_word (may be NULL) receives the word after the last
 * normal, i.e. where the next standard_normal call continues.  Replaces the
 * generator calls of probgen.generate_problem (probgen.py:52-68). */
int skl_rng_normal_device(uint64_t key, uint64_t start_word, int64_t rows, int64_t cols,
                          double* out, int64_t ld, uint64_t* end_word, void* stream);
/* Host (sequential, glibc libm) reference generator of the same stream;
 * used to patch the rare ziggurat tail draws and by tests. */
int skl_rng_gaussian_host(uint64_t key, int64_t count, double* out);

/* ---------------------------------------------------------------------
 * CountSketch apply plan ("lane lists").  The rows are cut into chunks of
 * `chunk` rows (<= 4088).  Bucket b belongs to warp w(b) = b / ceil(d/warps)
 * of the consuming CTA.  Per chunk, each warp's non-empty buckets are
 * scheduled onto its 32 lanes: a lane walks one bucket's rows (ascending)
 * at a time and keeps the bucket's running sum in a register, also into
 * the next chunk when it continues the same bucket; free lanes take the
 * bucket that keeps that step's shared-memory banks least loaded.  A
 * chunk's block, at lanes[chunk_off[k]], is
 *   [0, H)        H = round4(warps+1): first list row of each warp, and the
 *                 total number of rows at index `warps`;
 *   [H, ...)      rows of 32 words, word (r*32 + lane) = that lane's r-th
 *                 entry: bits 0..14 byte offset 8*row of the source row in
 *                 the staged chunk (8*chunk = a zero slot), bits 16..30 the
 *                 bucket (d = dummy slot), bit 31 negative sign.  A lane
 *                 writes its held sum back and loads the entry's bucket
 *                 whenever the bucket field changes.
 * This is the chunked, lane-scheduled form of the reference's CSR
 * sparse_map (sketch.py:100-102); it keeps scipy csr_matvecs' ascending-row
 * fold per bucket, so the device apply is bitwise-equal to it.
 * Call with lanes == NULL first to get chunk_off (nch + 1 entries; the
 * block sizes), then with a buffer of chunk_off[nch] words.
 * Limits: d <= 32767, chunk a multiple of 8 in [8, 4088], warps in [1, 31].
 * ------------------------------------------------------------------- */
int skl_countsketch_plan(const int32_t* rows, const int8_t* signs, int64_t m, int64_t d,
                         int64_t chunk, int warps, uint32_t* lanes, int64_t* chunk_off,
                         int threads);
/* The same plan for a sparse sign embedding with d > 2048 (the register-owned
 * plan covers d <= 2048): source row j contributes `spr` entries, rows and
 * signs hold m * spr values (entry j * spr + q, distinct buckets per row);
 * chunk * spr <= 65536.  Consumed by skl_sparsesign_dense. */
int skl_sparsesign_plan(const int32_t* rows, const int8_t* signs, int64_t m, int spr, int64_t d,
                        int64_t chunk, int warps, uint32_t* lanes, int64_t* chunk_off,
                        int threads);

/* S*A and S*b for dense column-major A (device pointers, plan on device;
 * max_block = largest chunk block in words).
 * b may be NULL (then Sb is ignored).  partitions: 0 = auto, 1 = single
 * ordered pass (bitwise-equal to the reference), P>1 = P row partitions
 * reduced in a fixed order (deterministic).  accumulate != 0 adds into
 * SA/Sb (used for row-streamed applies).  Replaces sketch.py:209-212
 * (dense branch). */
int skl_countsketch_dense(const double* A, int64_t m, int64_t n, int64_t lda, const double* b,
                          const uint32_t* lanes, const int64_t* chunk_off, int64_t max_block,
                          int64_t d, int64_t chunk, int warps, double* SA, int64_t ldsa,
                          double* Sb, int partitions, int accumulate, void* stream);
/* skl_countsketch_dense for a sparse sign plan (skl_sparsesign_plan): every
 * entry adds fl(+-scale * A[j, c]) (scale = fl(1/sqrt(s)), csr_matvecs'
 * product), so the result is bitwise-equal to sparse_map @ A
 * (sketch.py:104-115, 209-212). */
int skl_sparsesign_dense(const double* A, int64_t m, int64_t n, int64_t lda, const double* b,
                         const uint32_t* lanes, const int64_t* chunk_off, int64_t max_block,
                         int64_t d, int64_t chunk, int warps, double scale, double* SA,
                         int64_t ldsa, double* Sb, int partitions, int accumulate, void* stream);

/* Register-owned plan for d <= 128 * warps (the common case): bucket b is
 * held for the whole apply in a register of consumer thread b % (32*warps),
 * slot b / (32*warps).  Per chunk, each lane's list is the union of its four
 * buckets' rows (ascending inside a bucket, the four streams interleaved to
 * spread shared-memory banks), padded to the longest lane.  Block (u16
 * words) at lanes[chunk_off[k]]: H = round8(warps+1) words of per-warp first
 * list rows (index `warps` = total), then rows of 32 words: bits 0..12 row
 * in the chunk (chunk = zero slot), bits 13..14 slot, bit 15 negative sign.
 * Call with lanes == NULL first to get chunk_off, as for the lane lists.
 * Limits: chunk a multiple of 8 in [8, 8184]. */
int skl_countsketch_plan_owned(const int32_t* rows, const int8_t* signs, int64_t m, int64_t d,
                               int64_t chunk, int warps, uint16_t* lanes, int64_t* chunk_off,
                               int threads);
/* Device builders (bit-identical to the host ones): hashes/signs into
 * device arrays (falls back to the host walk in the rare case a Lemire draw
 * is rejected), and the register-owned plan from device hashes.  The plan
 * call is two-phase like the host one: lanes == NULL computes chunk_off
 * (device, nch+1), the per-(chunk, warp) list lengths into maxlen (device,
 * nch*warps int32) and writes {total words, max block} to total_and_max
 * (host); the second call fills lanes (device). */
int skl_rng_countsketch_device(uint64_t key, int64_t m, int64_t d, int32_t* rows, int8_t* signs,
                               void* stream);
int skl_countsketch_plan_owned_device(const int32_t* rows, const int8_t* signs, int64_t m,
                                      int64_t d, int64_t chunk, int warps, uint16_t* lanes,
                                      int64_t* chunk_off, int32_t* maxlen,
                                      int64_t* total_and_max, void* stream);
/* S*A, S*b with a register-owned plan (warps 8 or 16); otherwise as
 * skl_countsketch_dense (bitwise-equal to the reference for partitions 1). */
int skl_countsketch_dense_owned(const double* A, int64_t m, int64_t n, int64_t lda,
                                const double* b, const uint16_t* lanes, const int64_t* chunk_off,
                                int64_t max_block, int64_t d, int64_t chunk, int warps, double* SA,
                                int64_t ldsa, double* Sb, int partitions, int accumulate,
                                void* stream);

/* Sparse sign embedding (sketch.py:104-115: s distinct buckets per source
 * row, values +-1/sqrt(s)): the same register-owned plan with s entries per
 * row (rows/signs are m x s, row-major) and the apply with every entry scaled
 * by `scale` = fl(1/sqrt(s)) (one rounded product, as csr_matvecs).  The CSR
 * operand variant takes the bucket lists of S (bucket_rows = source rows,
 * ascending per bucket; signs in bucket order). */
int skl_sparsesign_plan_owned(const int32_t* rows, const int8_t* signs, int64_t m, int64_t s,
                              int64_t d, int64_t chunk, int warps, uint16_t* lanes,
                              int64_t* chunk_off, int threads);
int skl_sparsesign_dense_owned(const double* A, int64_t m, int64_t n, int64_t lda, const double* b,
                               const uint16_t* lanes, const int64_t* chunk_off, int64_t max_block,
                               int64_t d, int64_t chunk, int warps, double scale, double* SA,
                               int64_t ldsa, double* Sb, int partitions, int accumulate,
                               void* stream);
int skl_sparsesign_csr(const int64_t* indptr, const int64_t* indices, const double* values,
                       int64_t m, int64_t n, const int32_t* bucket_rows, const int64_t* bucket_ptr,
                       const int8_t* signs, double scale, int64_t d, double* SA, int64_t ldsa,
                       void* stream);

/* Same apply with HOST A/b (preferably pinned): streams ~128 MiB row blocks
 * of A through a two-slot device ring with host-to-device copies overlapped
 * with the kernel (bitwise the same result); if A_dev_keep != NULL the blocks
 * land there instead (column-major, ld_keep even, 16-byte aligned) and the
 * full device copy of A (and of b in b_dev_keep) is left for a later residual
 * pass.  SA_out / Sb_out may be host or device memory.  Synchronises the
 * stream before returning.  plan pointers are device. */
int skl_countsketch_dense_host(const double* A_host, int64_t m, int64_t n, int64_t lda,
                               const double* b_host, const uint32_t* lanes,
                               const int64_t* chunk_off, int64_t max_block, int64_t d,
                               int64_t chunk, int warps, double* SA_out, int64_t ldsa,
                               double* Sb_out, double* A_dev_keep, int64_t ld_keep,
                               double* b_dev_keep, void* stream);
/* skl_countsketch_dense_host with a register-owned plan. */
int skl_countsketch_dense_owned_host(const double* A_host, int64_t m, int64_t n, int64_t lda,
                                     const double* b_host, const uint16_t* lanes,
                                     const int64_t* chunk_off, int64_t max_block, int64_t d,
                                     int64_t chunk, int warps, double* SA_out, int64_t ldsa,
                                     double* Sb_out, double* A_dev_keep, int64_t ld_keep,
                                     double* b_dev_keep, void* stream);

/* ---- preconditioned LSQR (sketch-and-precondition, solvers.py:110-361) ----
 * Device pieces of one LSQR iteration; the scalar recurrence stays on the
 * host.  Column-major dense A (16-byte aligned, even lda); R is the explicit
 * n x n upper factor of QR(S A) (column-major, ld ldr) or NULL (plain
 * LSQR).  `work`/`counters` are scratch sized by skl_lsqr_work_size /
 * skl_lsqr_counter_size (counters zero-initialised once).  Reductions are
 * deterministic. */
int64_t skl_lsqr_work_size(int64_t m, int64_t n);
int64_t skl_lsqr_counter_size(int64_t n);
/* u_out = s (A y) - alpha u_in  (u_in may be NULL; A NULL: no product),
 * *norm2 = ||u_out||^2 (device scalar).  u_in and u_out must not alias. */
int skl_lsqr_gemv_n(const double* A, int64_t m, int64_t n, int64_t lda, const double* y,
                    double s, double alpha, const double* u_in, double* u_out, double* norm2,
                    double* work, unsigned int* counters, void* stream);
/* u_n = u_raw / beta (beta > 0), z = A^T u_n. */
int skl_lsqr_gemv_t(const double* A, int64_t m, int64_t n, int64_t lda, const double* u_raw,
                    double beta, double* u_n, double* z, double* work, unsigned int* counters,
                    void* stream);
/* Both products of one step in one pass over A (n <= 256):
 * u = r_prev / beta_prev (r_prev NULL: no alpha term), r_out = s (A y) -
 * alpha u, *norm2 = ||r_out||^2 and z = A^T r_out / ||r_out|| (z = 0 when
 * r_out = 0).  `work` holds skl_lsqr_fused_work_size(n) doubles; `counters`
 * as for the other LSQR kernels. */
int64_t skl_lsqr_fused_work_size(int64_t n);
int skl_lsqr_fused(const double* A, int64_t m, int64_t n, int64_t lda, const double* y, double s,
                   double alpha, const double* r_prev, double beta_prev, double* r_out, double* z,
                   double* norm2, double* work, unsigned int* counters, void* stream);
/* v_out = R^-T z - beta v_prev, *norm2 = ||v_out||^2 (R NULL: identity). */
int skl_lsqr_trsv_t(const double* R, int64_t ldr, int64_t n, const double* z, double beta,
                    const double* v_prev, double* v_out, double* norm2, void* stream);
/* v <- v / alfa (alfa > 0), y = R^-1 v (R NULL: y = v). */
int skl_lsqr_trsv_n(const double* R, int64_t ldr, int64_t n, double alfa, double* v, double* y,
                    void* stream);

/* The same two triangular solves with the inverted 32 x 32 diagonal blocks
 * of R (skl_lsqr_rinv_blocks, computed once per preconditioned solve: R
 * does not change across iterations): each block step is one 32-term
 * product instead of 32 dependent divide-and-update steps.  Rinv holds
 * ceil(n / 32) * 1024 doubles (device). */
int skl_lsqr_rinv_blocks(const double* R, int64_t ldr, int64_t n, double* Rinv, void* stream);
int skl_lsqr_trsv_t_inv(const double* R, int64_t ldr, int64_t n, const double* Rinv,
                        const double* z, double beta, const double* v_prev, double* v_out,
                        double* norm2, void* stream);
int skl_lsqr_trsv_n_inv(const double* R, int64_t ldr, int64_t n, const double* Rinv, double alfa,
                        double* v, double* y, void* stream);

/* Device-driven LSQR iteration (dense, n <= 256): the scalar recurrence of
 * solvers.py:193-222 runs on the device in `state` (skl_lsqr_state_size()
 * doubles: ||r||^2, ||v||^2, ||x||^2, alfa, beta, rhobar, phibar, anorm,
 * phi/rho, -theta/rho, rnorm, arnorm, the next pass's beta_prev, ...), with
 * the host loop's IEEE operations in the same order, so the host reads the
 * state once per iteration -- while the next pass already runs.
 * skl_lsqr_fused_dev is skl_lsqr_fused taking alfa and beta_prev from
 * state; skl_lsqr_step_dev runs the rest of one iteration: R^-T z - beta v
 * (beta from state), v_n and y = R^-1 v_n (alfa from state), the recurrence,
 * and x += c1 w, w = v_n + c2 w.  v holds v on entry and v_n on exit. */
int64_t skl_lsqr_state_size(void);
int skl_lsqr_fused_dev(const double* A, int64_t m, int64_t n, int64_t lda, const double* y,
                       const double* r_prev, double* r_out, double* z, double* norm2,
                       double* work, unsigned int* counters, const double* state, void* stream);
int skl_lsqr_step_dev(const double* R, int64_t ldr, int64_t n, const double* Rinv,
                      const double* z, double* v, double* v_raw, double* y, double* w, double* x,
                      double* state, void* stream);
/* R^{-1} of the n x n upper-triangular R in full (n <= 256; Ri: n * n
 * doubles, column-major, zero below the diagonal; device), once per
 * preconditioned solve, and skl_lsqr_step_dev with both triangular solves
 * as products with it. */
int skl_lsqr_rinv_full(const double* R, int64_t ldr, int64_t n, double* Ri, void* stream);
int skl_lsqr_step_full_dev(const double* Ri, int64_t n, const double* z, double* v,
                           double* v_raw, double* y, double* w, double* x, double* state,
                           void* stream);
/* CSR operands: u_out = s (A y) - alpha u_in, *norm2 = ||u_out||^2 (rows
 * folded in stored order); and u_n = u_raw / beta, z = A^T u_n from the
 * CSC form of A (colptr int64 n+1, rowidx int32 ascending within a column,
 * values), one warp per column. */
int skl_lsqr_spmv(const int64_t* indptr, const int64_t* indices, const double* values, int64_t m,
                  const double* y, double s, double alpha, const double* u_in, double* u_out,
                  double* norm2, double* work, unsigned int* counters, void* stream);
int skl_lsqr_csc_t(const int64_t* colptr, const int32_t* rowidx, const double* cval, int64_t m,
                   int64_t n, const double* u_raw, double beta, double* u_n, double* z,
                   void* stream);
/* x += c1 w; w = v + c2 w; *norm2 = ||x||^2. */
int skl_lsqr_xw(int64_t n, double c1, double c2, const double* v, double* w, double* x,
                double* norm2, void* stream);

/* Bucket-sorted source rows of a CountSketch (host): bucket_rows[bucket_ptr[i]
 * .. bucket_ptr[i+1]) are the rows j with rows[j] == i, ascending -- the CSR
 * of S (sketch.py:100-102) without its values.  bucket_ptr has d+1 entries. */
int skl_countsketch_buckets(const int32_t* rows, int64_t m, int64_t d, int32_t* bucket_rows,
                            int64_t* bucket_ptr);

/* S*A for CSR A (device pointers; int64 indptr/indices as SparseMatrix
 * holds them, linalg.py:66-68).  bucket_rows/bucket_ptr from
 * skl_countsketch_buckets and the int8 signs in BUCKET order
 * (bucket_signs[k] = signs[bucket_rows[k]]), all on the device.  SA is
 * d x n column-major, fully overwritten (bitwise-equal to scipy's
 * csr_matmat fold).  Replaces sketch.py:210-211. */
int skl_countsketch_csr(const int64_t* indptr, const int64_t* indices, const double* values,
                        int64_t m, int64_t n, const int32_t* bucket_rows,
                        const int64_t* bucket_ptr, const int8_t* signs, int64_t d, double* SA,
                        int64_t ldsa, void* stream);

/* SRHT of [A | b] in one pass: b rides along as the (n+1)-th column (SA
 * d x n, ld ldsa; Sb d).  row_offset: first global row of this row block
 * (0 unsharded; a multiple of the 4096-row block for a shard, whose partial
 * the caller sums across ranks).  partitions: row partitions per column, 0 =
 * automatic.  Replaces sketch.py:213-223 for the SAA solve's S A and S b
 * (solvers.py:308, 287). */
int skl_srht_dense_ab(const double* A, int64_t m, int64_t n, int64_t lda, const double* b,
                      const uint16_t* sign_bits, const int64_t* row_sample, int64_t m_pad,
                      int64_t d, int64_t row_offset, double* SA, int64_t ldsa, double* Sb,
                      int partitions, void* stream);

/* Ordered bucket walk for a few long dense columns (device): SA[:, c]
 * (+)= S A[:, c] for c < n and Sb (+)= S b, every bucket's products
 * sign*scale*A[j, c] added in ascending source row j from +0.0 -- scipy's
 * csr_matvec / csr_matvecs fold, bitwise.  bucket_rows / bucket_ptr /
 * signs are the CSR of S as for skl_countsketch_csr (scale = 1 for
 * CountSketch, fl(1/sqrt(s)) for a sparse sign embedding).  Used where the
 * column kernels would split the rows (one column, or n + 1 << #SMs): a
 * vector apply S b, cfg4's Sb.  n may be 0 (b only).  Replaces
 * sketch.py:212 (`sparse_map @ b`, csr_matvec). */
int skl_countsketch_dense_ordered(const double* A, int64_t m, int64_t n, int64_t lda,
                                  const double* b, const int32_t* bucket_rows,
                                  const int64_t* bucket_ptr, const int8_t* signs, double scale,
                                  int64_t d, double* SA, int64_t ldsa, double* Sb, int accumulate,
                                  void* stream);

/* SRHT: out = (P H D [A; 0]) / sqrt(d) for dense column-major A (device),
 * H the unnormalised Sylvester-Hadamard of order m_pad.  sign_bits are the
 * +-1 sign diagonal packed by skl_srht_pack_signs (device copy);
 * row_sample (int64, d) is device.  Replaces sketch.py:213-223 and
 * fwht_inplace sketch.py:152-177. */
int skl_srht_dense(const double* A, int64_t m, int64_t n, int64_t lda, const uint16_t* sign_bits,
                   const int64_t* row_sample, int64_t m_pad, int64_t d, double* SA,
                   int64_t ldsa, void* stream);
/* Row block [row_offset, row_offset + m_local) of the same apply (row_offset
 * a multiple of min(m_pad, 4096)); sign_bits of that block; the caller sums
 * the per-block partials (the multi-GPU reduce). */
int skl_srht_dense_shard(const double* A, int64_t m_local, int64_t n, int64_t lda,
                         const uint16_t* sign_bits, const int64_t* row_sample, int64_t m_pad,
                         int64_t d, int64_t row_offset, double* partial, int64_t ldp,
                         void* stream);
/* Sign packing (host): per block of B = min(m_pad, 4096) rows,
 * skl_srht_sign_words(B) 16-bit words; bit i of word t is the sign of the
 * i-th element the kernel's first butterfly pass gives task t. */
int64_t skl_srht_sign_words(int64_t B);
int skl_srht_pack_signs(const int8_t* signs, int64_t m_pad, uint16_t* packed);

/* In-place unnormalised FWHT of a device column-major m_pad x n array
 * (lda >= m_pad), m_pad a power of two.  Replaces sketch.py:152-177. */
int skl_fwht_device(double* X, int64_t m_pad, int64_t n, int64_t lda, void* stream);

/* Gaussian apply SA = G * A with G d x m (ld ldg), A m x n (lda), column-
 * major fp64, on the fp64 tensor cores (DMMA).  Replaces sketch.py:204-208. */
int skl_gemm_f64(const double* G, int64_t ldg, const double* A, int64_t lda, double* C,
                 int64_t ldc, int64_t d, int64_t n, int64_t m, int accumulate, void* stream);

/* ---------------------------------------------------------------------
 * Reduced solve (device).  Householder QR of M = SA (d x n, d >= n) with
 * the reference's conventions (linalg.py:166-192): diag(R) >= 0, rank
 * check |R[c,c]| < 1e-14 * ||M||_F naming the first bad column, then
 * x = R^{-1} Q^T Sb (solvers.py:309, linalg.py:214-218).
 * R (n x n, ldr) and Q (d x n, ldq) are optional outputs (NULL to skip).
 * x is device (n).  *bad_col receives -1 or the failing column and
 * *bad_val |R[c,c]| for the error message.
 * ------------------------------------------------------------------- */
int skl_qr_solve(const double* SA, int64_t ldsa, const double* Sb, int64_t d, int64_t n,
                 double* x, double* R, int64_t ldr, double* Q, int64_t ldq, int64_t* bad_col,
                 double* bad_val, void* stream);
/* skl_qr_solve without the synchronisation: bad_col / bad_val (pinned host
 * or device memory) are written in stream order and checked by the caller
 * once the stream has passed them (*bad_col >= 0: rank deficient at that
 * column, |R[c, c]| = *bad_val -- the SKL_ERR_SINGULAR case of
 * skl_qr_solve), so the residual pass of a solve can be enqueued behind the
 * factorisation with one synchronisation for both. */
int skl_qr_solve_async(const double* SA, int64_t ldsa, const double* Sb, int64_t d, int64_t n,
                       double* x, double* R, int64_t ldr, double* Q, int64_t ldq,
                       int64_t* bad_col, double* bad_val, void* stream);

/* ---------------------------------------------------------------------
 * Reduced solve of sketch-and-apply (device): the least-squares minimiser
 * x of ||SA x - Sb|| as skl_qr_solve gives it, to rounding (~kappa u).  A
 * well-conditioned SA (the unshifted Cholesky factor of [SA Sb]^T [SA Sb]
 * holds and its diagonal spans < 1e3) is solved by the corrected semi-normal
 * equations on that factor; otherwise by shifted CholeskyQR2 (R with
 * diag > 0, unique) plus one corrected semi-normal step -- picked on the
 * device.  The rank check of linalg.py:186-191 on diag(R).  Replaces the
 * numpy QR + solve_triangular of solvers.py:309 for systems with
 * n + 1 <= 1056 < d (skl_cqr_supported).  Asynchronous like
 * skl_qr_solve_async: *bad_col (pinned host or device) receives -1 when x
 * is valid, the first rank-deficient column, or -2 when a Cholesky pivot
 * broke down or the refinement did not contract; in both failure cases the
 * caller re-solves with skl_qr_solve (Householder), which produces the
 * reference's error message.
 * ------------------------------------------------------------------- */
int skl_cqr_supported(int64_t d, int64_t n);
int skl_cqr_solve_async(const double* SA, int64_t ldsa, const double* Sb, int64_t d, int64_t n,
                        double* x, int64_t* bad_col, double* bad_val, void* stream);

/* ||A x - b||_2 for dense column-major A (device).  Replaces
 * solvers.py:102-107.  *out is host. */
int skl_residual_dense(const double* A, int64_t m, int64_t n, int64_t lda, const double* x,
                       const double* b, double* out, void* stream);
/* ||A x - b||_2 for CSR A (device). */
int skl_residual_csr(const int64_t* indptr, const int64_t* indices, const double* values,
                     int64_t m, int64_t n, const double* x, const double* b, double* out,
                     void* stream);
/* The two residuals without their synchronisation: *out (pinned host or
 * device) is written in stream order (batched solves, solve_many). */
int skl_residual_dense_async(const double* A, int64_t m, int64_t n, int64_t lda, const double* x,
                             const double* b, double* out, void* stream);
int skl_residual_csr_async(const int64_t* indptr, const int64_t* indices, const double* values,
                           int64_t m, int64_t n, const double* x, const double* b, double* out,
                           void* stream);

/* ---- Gaussian operator generated in bands across devices ----
 * The d x m Gaussian operator (sketch.py:94-96) is one ziggurat stream cut
 * into segments of skl_gaussian_segment_words() words.  Device k parses
 * only its band of segments [seg0, seg1): band_begin enqueues the parse
 * on the stream and returns it in *handle (count may be NULL: it is
 * reported by band_count, which synchronises the stream, so every device's
 * parse runs before the host waits on any); after the host's prefix sum over
 * the bands, band_write stores normal t (global,
 * first <= t < first + count, t < N = d * m) at G[(t / m - row0) * ldg +
 * t % m] divided by `div` (sqrt(d)) and frees the handle (band_free frees
 * it without writing).  Bit-identical to skl_rng_gaussian_device.  The
 * bands are then exchanged so every device holds the column block S[:, r0:r1]
 * its row shard multiplies (multidevice.py). */
int64_t skl_gaussian_segment_words(void);
int skl_gaussian_band_begin(uint64_t key, int64_t seg0, int64_t seg1, void** handle,
                            int64_t* count, void* stream);
int skl_gaussian_band_count(void* handle, int64_t* count, void* stream);
int skl_gaussian_band_write(void* handle, int64_t first, int64_t N, int64_t m, int64_t row0,
                            double* G, int64_t ldg, double div, void* stream);
void skl_gaussian_band_free(void* handle, void* stream);

/* ---- row-sharded apply: the reduce step ----
 * out[:, c] = sum over q = 0 .. nslots-1, in that order, of
 * slots[q * slot_stride + c * ld + i] (rows x cols, column-major slots).
 * The slots are the per-rank partial sketches the ranks' kernels wrote into
 * the destination's symmetric buffer over NVLink; replaces the NCCL reduce
 * of the reference-style sharding with a deterministic fixed-order sum. */
int skl_sum_slots(const double* slots, int64_t nslots, int64_t slot_stride, int64_t rows,
                  int64_t cols, int64_t ld, double* out, int64_t ldo, void* stream);

/* Reduce-scatter step of the multi-GPU apply: out[i] = peers[0][i] +
 * peers[1][i] + ... + peers[npeers-1][i] (rank order, the same bits as
 * skl_sum_slots) for i in [begin, end).  peers is a HOST array of npeers
 * (<= 16) device addresses -- the ranks' partials in their symmetric
 * buffers, read over NVLink -- and out may be a peer address (the
 * destination rank's result buffer).  Each rank calls it for its own element
 * block, so the destination receives every block once.  Replaces the NCCL
 * reduce of the d x (n+1) partials. */
int skl_reduce_peers(const double* const* peers, int npeers, int64_t begin, int64_t end,
                     double* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SKETCHLS_B200_H */
