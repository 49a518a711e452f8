/*
 * nent_b200.h -- C ABI of libnent_b200.so, the sm_100a implementation of the
 * numerical-entanglement hot path (entangle -> LSB op -> extract/recover).
 *
 * Conventions (all entry points):
 *   - extern "C", plain pointers and sizes, no torch/numpy types.
 *   - Every data pointer is a DEVICE pointer (may be a peer pointer on another
 *     GPU of the node when P2P is enabled) unless the name says _host.
 *   - A block of m streams is passed as a HOST array of m row pointers, so a
 *     contiguous (m, n) array, a strided one, or buffers living on m different
 *     GPUs are all expressible.  At most NENT_MAX_STREAMS (64) rows.
 *   - Element widths are 32 (int32) or 64 (int64) two's complement.
 *   - `stream` is a cudaStream_t (void* here so FFI callers need no CUDA
 *     headers).  Every call is asynchronous on that stream; nothing is
 *     allocated except where stated; there is no global mutable state.
 *   - Return value: NENT_OK or an error code; nent_last_error() gives the
 *     message (thread-local).
 *
 * Each entry point cites the reference function it replaces
 * (paths relative to the reference tree, pkg/src/nent/...).
 */
#ifndef NENT_B200_H
#define NENT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NENT_ABI_VERSION 2

#define NENT_OK 0
#define NENT_ERR_PARAM 1    /* ParameterError */
#define NENT_ERR_RANGE 2    /* RangeError (value outside a bound) */
#define NENT_ERR_CUDA 3     /* launch / runtime failure */
#define NENT_ERR_OVERFLOW 4 /* exact result does not fit int64 (reference raises OverflowError) */

/* Multiply-accumulate flavours of the convolution / inner-product kernels.
 * All are exact whenever the admitted bound says the result fits: */
#define NENT_MAC_I32 1 /* int32 IMAD modulo 2^32: |result| < 2^31                     */
#define NENT_MAC_F64 2 /* FP64 DFMA: operands and every partial sum < 2^53 (IPP's _64f) */
#define NENT_MAC_W64 3 /* IMAD.WIDE s32*s32+s64: |x|,|g| < 2^31, result fits int64     */
#define NENT_MAC_S64 4 /* split x = hi*2^32+lo: IMAD.WIDE + IMAD, |g| < 2^31            */
#define NENT_MAC_G64 5 /* generic 64x64 low product (mul.lo.u64)                        */
#define NENT_MAC_X128 6 /* exact 128-bit accumulation + overflow count (object path)    */
/* Tensor-core digit slicing: x and g split into balanced base-256 int8 digits
 * (np planes of x, ng digits of g), every digit pair an exact int8 GEMM with
 * int32 accumulation, recombined mod 2^64.  Exact whenever the result fits
 * int64, np <= 8, ng <= 4, K + 15 < 65536.  Runs on the 5th-generation tensor
 * cores (tcgen05.mma kind::i8, TMEM accumulators) when the shape fits that
 * kernel (plain conv of <= 64 rows, or the fused m = 3 path; K + 127 taps of
 * every digit resident in shared memory), else on mma.sync m16n8k32 s8.
 * NENT_IMMA_MMA_SYNC forces the mma.sync kernel. */
#define NENT_MAC_IMMA 7
#define NENT_MAC_IMMA_DIGITS(np, ng) (NENT_MAC_IMMA | ((np) << 8) | ((ng) << 12))
#define NENT_IMMA_MMA_SYNC (1 << 16)

/* Which tensor-core kernel an IMMA-flavour convolution of `rows` streams
 * (fused extract when `extract`) with K taps runs: 2 = tcgen05, 1 = mma.sync,
 * 0 = not an IMMA flavour. */
int nent_imma_kernel(int flavor, int K, int rows, int extract);
/* The convolution kernel the calling host thread launched last (diagnostic,
 * for tests and the benchmark): 1 CUDA-core tile kernel, 2 mma.sync digit
 * slicing, 3 tcgen05 digit slicing (generic), 4 tcgen05 m = 3 kernel with
 * l = 16 (conv_tc05_m3.cu: fused, or its plain mode for three non-entangled
 * streams), 5 tcgen05 fused m = 4 long-filter kernel (conv_tc05_m4.cu),
 * 6 tcgen05 fused m = 8 kernel on already-entangled rows (conv_tc05_m8.cu),
 * 0 none yet. */
int nent_last_conv_kernel(void);

/* Elementwise op codes (ops.py:193-204). */
#define NENT_EW_ADD 0
#define NENT_EW_SUB 1
#define NENT_EW_MUL 2

const char *nent_last_error(void);
int nent_abi_version(void);
/* Lets kernels on the current device dereference memory of device `peer`
 * (NVLink peer access; already-enabled is not an error).  The multi-GPU
 * recovery passes peer rows (CUDA IPC-mapped deltas of other ranks) to
 * nent_extract. */
int nent_enable_peer_access(int peer);
/* 1 if the library was compiled for and can launch on the current device. */
int nent_device_ok(void);

/* ---- codec ---------------------------------------------------------------- */

/* Replaces codec.entangle + codec._check_input_range + _kernels.entangle_kernel
 * (codec.py:34-72, _kernels.py:25-30):
 *   eps[i][j] = (src[(i-1) mod m][j] << l) + src[i][j]   (mod 2^64, then narrowed)
 * If check_hi >= 0, *bad_index_dev (device u64, written) receives the smallest
 * row-major index i*n+j with |src[i][j]| > check_hi (numpy's wrapping abs), or
 * UINT64_MAX if none. */
int nent_entangle(const void *const *src, int src_bits, void *const *eps, int eps_bits, int m,
                  int64_t n, int l, int64_t check_hi, uint64_t *bad_index_dev, void *stream);

/* out[j] = (a[j] << l) + b[j]: one entangled stream from its two sources (the
 * stream-per-GPU entangle after the ring shift), and the kernel
 * self-entanglement g <- (g << l) + g of ops.self_entangle_kernel (ops.py:250-262). */
int nent_shift_add(const void *a, const void *b, int in_bits, void *out, int out_bits, int64_t n,
                   int l, void *stream);

/* Replaces codec.disentangle / _kernels.disentangle_kernel / codec._disentangle_reference
 * (codec.py:89-131, _kernels.py:33-67).  Recovers all m streams from the m-1
 * rows != r; delta[r] is never dereferenced (may be NULL).  wide=0 is the
 * w<=32 int64 pivot (bit-identical to the numba kernel even on inconsistent
 * input); wide=1 is the w>32 exact (128-bit) pivot of the Python-int path.
 * If overflow_dev != NULL it is incremented per position whose out[r] does not
 * fit int64 (the reference raises OverflowError there). */
int nent_extract(const void *const *delta, int delta_bits, void *const *out, int out_bits, int m,
                 int64_t n, int l, int r, int wide, unsigned long long *overflow_dev, void *stream);

/* K3 with the redundant-stream check: recovers every row from the rows other
 * than `pivot` (exactly nent_extract with r = pivot), then adds to
 * *mismatch_dev the positions whose pivot word differs from the re-entangled
 * recovery (d_{pivot-1} << l) + d_pivot -- the fused kernel's failed=None
 * check as a separate pass (used after the plain tensor-core conv for m > 3). */
int nent_extract_verify(const void *const *delta, int delta_bits, void *const *out, int out_bits, int m,
                        int64_t n, int l, int pivot, int wide, unsigned long long *overflow_dev,
                        unsigned long long *mismatch_dev, void *stream);

/* Replaces codec.disentangle_m3 (codec.py:151-183), the independent m=3 recipe. */
int nent_extract_m3(const void *const *delta, int delta_bits, void *const *out, int out_bits,
                    int64_t n, int l, int w, int r, void *stream);

/* ---- LSB operations ------------------------------------------------------- */

/* Circular convolution (ops._circ_conv_rows, ops.py:158-172) generalised for
 * halo-split shards:
 *   y[row][j'] = sum_{k<K} g[k] * xv[row][(y_begin + j' - k) mod period],  0 <= j' < n_out
 *   xv[i] = x[row][i] for i < n_in, 0 for n_in <= i < period.
 * Circular conv: n_in == period.  Full linear conv: period = n_in + K - 1.
 * g is int32 (g_bits 32) or int64; `flavor` is one of NENT_MAC_*.  With
 * NENT_MAC_X128, *overflow_dev (optional) counts outputs whose exact value
 * does not fit int64 (the reference's object path raises OverflowError). */
int nent_conv(const void *const *x, int x_bits, int rows, int64_t n_in, int64_t period,
              const void *g, int g_bits, int K, void *const *y, int y_bits, int64_t y_begin,
              int64_t n_out, int flavor, unsigned long long *overflow_dev, const void *imma_table,
              void *stream);

/* NENT_MAC_IMMA flavours read a digit-split Toeplitz table of the taps.  Pass
 * imma_table = NULL to have each call build it in a stream-ordered workspace,
 * or prepare it once (the taps are fixed across calls) with nent_imma_table
 * into a caller buffer of nent_imma_table_bytes bytes.  The table depends on
 * the taps, K, the flavour's tap digits and y_begin mod 4. */
int64_t nent_imma_table_bytes(int K, int flavor);
int nent_imma_table(const void *g, int g_bits, int K, int64_t y_begin, int flavor, void *table,
                    void *stream);

/* The fused hot path (bench.py entangled() chain, bench.py:103-106, plus the
 * pipeline chain of SCALE/ADD/PERMUTATION before the conv, SURVEY cfg5):
 *   x_i[p]  = scale * ((c[(i-1) mod m][q] << l) + c[i][q]) + add[q],  q = perm ? perm[p] : p
 *             (x_i[p] = 0 for p >= n_in; add may be NULL; perm may be NULL)
 *   delta_i = circular conv of x_i with g over `period` (as nent_conv)
 *   d       = extract(delta, pivot r)   (r = -1: no failure, pivot 0)
 * One CTA owns an output tile of all m streams (3 <= m <= 8), so entangle
 * happens on load and extraction in registers; delta never reaches HBM.
 * With r = -1 and mismatch_dev != NULL, the redundant stream delta_0 is
 * checked against the recovered outputs (silent-error detection) and the
 * number of inconsistent positions is added to *mismatch_dev.
 * pre_entangled != 0: the rows c are already entangled words (e.g. produced
 * by the stream-per-GPU workers or a gather pre-pass); only conv + extract.
 * d_bits = 32 is for outputs whose admitted bound fits int32 (the reference's
 * admit(), ops.py:127); outside that bound int32 results are unspecified. */
int nent_fused_conv(const void *const *c, int c_bits, int m, int64_t n_in, int64_t period,
                    int l, int64_t scale, const void *add, int add_bits, const int64_t *perm,
                    const void *g, int g_bits, int K, int r, int pre_entangled, void *const *d,
                    int d_bits, int64_t y_begin, int64_t n_out, int flavor,
                    unsigned long long *mismatch_dev, const void *imma_table, void *stream);

/* Single-stream variant of the fused prologue without extraction (the
 * stream-per-GPU worker: x = scale*((a << l) + b) + add, gathered, convolved).
 * a may be NULL (plain stream). */
int nent_chain_conv(const void *a, const void *b, int in_bits, int64_t n_in, int64_t period,
                    int l, int64_t scale, const void *add, int add_bits, const int64_t *perm,
                    const void *g, int g_bits, int K, void *y, int y_bits, int64_t y_begin,
                    int64_t n_out, int flavor, const void *imma_table, void *stream);

/* LSB chain in front of the conv (cfg5): entangle -> SCALE -> ADD (self-entangled
 * kernel) -> PERMUTATION (ops.py:193-204, 219-220, 250-262), in two HBM passes:
 * nent_interleave writes the m (<= 8) rows position-major (out[p*m + s] = x[s][p]),
 * so each gathered position is one contiguous m-sample record; then
 *   x[s][p] = scale * ((ct[q][s-1 mod m] << l) + ct[q][s]) + add[q],  q = perm ? perm[p] : p
 * (add may be NULL).  Feed x to nent_fused_conv with pre_entangled = 1. */
int nent_interleave(const void *const *x, int x_bits, int m, int64_t n, void *out, void *stream);
/* The same chain with the arithmetic moved into the (coalesced) interleave
 * pass: nent_interleave_chain writes records of the chain words before the
 * permutation, out[p*m + s] = scale * ((x[s-1 mod m][p] << l) + x[s][p]) + add[p]
 * (out_bits == x_bits; the caller's bound must fit), and nent_gather_records
 * permutes them, x[s][p] = rec[perm[p]][s] (perm int32 or int64), so each
 * permuted position costs one random record read.  Reference: ops.py:193-204,
 * 219-220, 250-262. */
int nent_interleave_chain(const void *const *x, int x_bits, int m, int64_t n, int l, int64_t scale,
                          const void *add, int add_bits, void *out, int out_bits, void *stream);
int nent_gather_records(const void *rec, int rec_bits, int m, int64_t n, const void *perm, int perm_bits,
                        void *const *x, void *stream);
/* Kernel.of_permutation's bijection check (ops.py:57-62) on the device:
 * *bad_dev += number of indices outside [0, n) plus repeated indices, so 0
 * means perm is a bijection of [0, n).  bitmap: caller-zeroed workspace of
 * ceil(n / 32) uint32 words.  perm int32 or int64. */
int nent_perm_check(const void *perm, int perm_bits, int64_t n, unsigned *bitmap, unsigned long long *bad_dev,
                    void *stream);
int nent_gather_chain(const void *ct, int c_bits, int m, int64_t n, int l, int64_t scale,
                      const void *add, int add_bits, const int64_t *perm, void *const *x, int x_bits,
                      void *stream);

/* ELEMENTWISE_ADD/SUB/MUL and SCALE (ops.py:193-204): y = x op g, g of length
 * n (g_len == n) or 1 (broadcast).  Arithmetic modulo 2^64; when check != 0
 * and op is MUL, *overflow_dev counts products that do not fit int64. */
int nent_elementwise(const void *const *x, int x_bits, int rows, int64_t n, const void *g,
                     int g_bits, int64_t g_len, int op, void *const *y, int y_bits, int check,
                     unsigned long long *overflow_dev, void *stream);
int nent_scale(const void *const *x, int x_bits, int rows, int64_t n, int64_t s, void *const *y,
               int y_bits, int check, unsigned long long *overflow_dev, void *stream);

/* PERMUTATION (ops.py:219-220): y[row][j] = x[row][perm[j]] */
int nent_permute(const void *const *x, int x_bits, int rows, int64_t n, const int64_t *perm,
                 void *const *y, int y_bits, void *stream);

/* out[row][j] = x[row][(-j) mod n] (ops._rev_circular, ops.py:179-181; xcorr = conv of this). */
int nent_reverse_circular(const void *const *x, int x_bits, int rows, int64_t n, void *const *y,
                          int y_bits, void *stream);

/* INNER_PRODUCT (ops.py:205-211), batched: every row is `batch` vectors of
 * length n (row-major, contiguous); y[row][b] = sum_i x[row][b*n+i] * g[i]
 * (int64 out).  When check != 0, *overflow_dev counts dots not fitting int64. */
int nent_inner(const void *const *x, int x_bits, int rows, int64_t batch, int64_t n,
               const void *g, int g_bits, void *const *y, int flavor, int check,
               unsigned long long *overflow_dev, void *stream);

/* Fused entangle -> inner product -> extract over a batch (SURVEY cfg4):
 * c[i] is (batch, n) per stream; d[i][b] recovered from the m-1 dots != r. */
int nent_fused_inner(const void *const *c, int c_bits, int m, int64_t batch, int64_t n, int l,
                     const void *g, int g_bits, int r, int wide, void *const *d, int d_bits,
                     int flavor, unsigned long long *mismatch_dev, void *stream);

/* Fused entangle -> outer product -> extract (SURVEY cfg4 outer; the reference
 * expresses it as ROW_GEMM on m x 1 blocks, ops.py:221-227):
 *   d[i][b][u][v] = extract_i( ((c[i-1][b,u] << l) + c[i][b,u]) * g[v] ), b in [0,batch)
 * written to d (layout (batch, n, p) per stream) when d != NULL, and the
 * per-(stream, vector) sums sum_{u,v} d into sums_dev[i*batch + b] (int64,
 * accumulated) when sums_dev != NULL. */
int nent_fused_outer(const void *const *c, int c_bits, int m, int64_t batch, int64_t n, int l,
                     const void *g, int g_bits, int64_t p, int r, int wide, void *const *d,
                     int d_bits, long long *sums_dev, void *stream);

/* ROW_GEMM (ops.py:221-227): y[row][c] = sum_j x[row][j] * G[j][c], G int64 (n, p). */
int nent_gemm(const void *const *x, int x_bits, int rows, int64_t n, const int64_t *G, int64_t p,
              void *const *y, int y_bits, int check, unsigned long long *overflow_dev,
              void *stream);

/* ---- fail-stop harness, checksum baseline, helpers ------------------------- */

/* pipeline.poison_pattern (pipeline.py:65-70): alternating -2^(w-1), 2^(w-1)-1. */
int nent_poison(void *y, int y_bits, int64_t n, int w, void *stream);

/* max |x| over rows (exact, unsigned) into *out_dev (device u64, written). */
int nent_max_abs(const void *const *x, int x_bits, int rows, int64_t n, uint64_t *out_dev,
                 void *stream);

/* First row-major index i*n+j with |x[i][j]| > hi into *bad_index_dev (UINT64_MAX if
 * none): codec._check_input_range / checksum_encode's check (codec.py:34-46,
 * checksum.py:42-55). */
int nent_check_range(const void *const *x, int x_bits, int rows, int64_t n, int64_t hi,
                     uint64_t *bad_index_dev, void *stream);

/* checksum.checksum_encode (checksum.py:42-60): cs[j] = sum_i x[i][j]. */
int nent_checksum_encode(const void *const *x, int x_bits, int m, int64_t n, void *cs,
                         int cs_bits, void *stream);
/* checksum.checksum_recover (checksum.py:80-97): out[failed] = cs - sum_{i != failed} x[i]. */
int nent_checksum_recover(const void *const *x, int x_bits, const void *cs, int cs_bits, int m,
                          int64_t n, int failed, void *out, int out_bits, void *stream);

/* ---- host <-> device staging ---------------------------------------------------- */

#define NENT_COPY_H2D 1
#define NENT_COPY_D2H 2
#define NENT_COPY_D2D 3

/* `rows` rows of `width_bytes` each, source rows `src_pitch` bytes apart,
 * destination rows `dst_pitch` bytes apart, as ONE stream-ordered 2-D DMA
 * (host side must be pinned for the copy to be asynchronous).  This is how a
 * caller holding the reference's host StreamBlock (m rows of samples,
 * blocks.py) stages a chunk of every stream at once: one copy-engine command
 * per chunk and direction instead of one per row (the host-buffer pipeline's
 * transfer primitive; paper_1509_03838_b200/hostpath.py). */
int nent_copy_rows(void *dst, int64_t dst_pitch, const void *src, int64_t src_pitch,
                   int64_t width_bytes, int rows, int direction, void *stream);

/* ---- measurement ------------------------------------------------------------ */

#define NENT_BENCH_IMMA 16 /* microbenchmark only: mma.sync m16n8k32 s8 (legacy IMMA) */
#define NENT_BENCH_TC05 17 /* microbenchmark only: tcgen05.mma kind::i8 128x128x32, A in TMEM */

/* Integer / FP64 pipe microbenchmark used for the roofline denominators.
 * kind: NENT_MAC_* flavour, NENT_BENCH_IMMA or NENT_BENCH_TC05 (one CTA of 128 threads per block,
 * `iters` chains of 12 MMAs; `threads` ignored); otherwise launches blocks x threads threads each doing
 * `iters` x 16 independent MACs; sink_dev receives a value so nothing is
 * dead-code eliminated. Returns MACs issued via *macs_out (host). */
int nent_microbench(int kind, int blocks, int threads, int iters, unsigned long long *sink_dev,
                    double *macs_out, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* NENT_B200_H */
