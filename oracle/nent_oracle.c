/*
 * nent_oracle.c -- CPU restatement of the reference `nent` arithmetic.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package links, loads or
 * calls this file; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs use it, and only as the checker or as
 * the timed CPU baseline.  It is a plain-C restatement of the reference
 * algorithm (paths relative to /root/reference):
 *
 *   entangle            pkg/src/nent/codec.py:57-72, pkg/src/nent/_kernels.py:25-30
 *   input range check   pkg/src/nent/codec.py:34-46 (first offender, row-major;
 *                       np.abs wraps, so INT64_MIN is never flagged)
 *   disentangle         pkg/src/nent/codec.py:89-131, pkg/src/nent/_kernels.py:33-67
 *                       (w<=32: int64 wrapping pivot; w>32: exact pivot, the
 *                       Python-int path, here __int128)
 *   disentangle_m3      pkg/src/nent/codec.py:145-183
 *   circular conv       pkg/src/nent/ops.py:158-172 (np.convolve + wrap of the
 *                       tail == sum_k g[k] x[(j-k) mod n])
 *   xcorr               pkg/src/nent/ops.py:179-181, 215-218
 *   add/sub/mul/scale   pkg/src/nent/ops.py:193-204, 235-238
 *   inner product       pkg/src/nent/ops.py:205-211
 *   permutation         pkg/src/nent/ops.py:219-220
 *   row gemm            pkg/src/nent/ops.py:221-227
 *
 * Integer semantics: every reference numpy path computes in int64 with
 * two's-complement wrap-around; its object-dtype paths are exact and raise
 * OverflowError when the exact result does not fit int64.  The oracle computes
 * modulo 2^64 (unsigned arithmetic, no UB) and, in "wide" mode, additionally
 * in __int128 to report how many results would not fit int64 (the reference's
 * OverflowError condition).  Parity is pinned against the reference's own
 * golden vectors and generated fixtures in tests/golden/.
 */
#include <stdint.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;
typedef __int128 i128;

static inline int64_t wrap_shl(int64_t x, int s) { return (int64_t)((uint64_t)x << s); }
static inline int64_t wrap_add(int64_t a, int64_t b) { return (int64_t)((uint64_t)a + (uint64_t)b); }
static inline int64_t wrap_sub(int64_t a, int64_t b) { return (int64_t)((uint64_t)a - (uint64_t)b); }
static inline int64_t wrap_mul(int64_t a, int64_t b) { return (int64_t)((uint64_t)a * (uint64_t)b); }
static inline int fits_i64(i128 v) { return v >= (i128)INT64_MIN && v <= (i128)INT64_MAX; }

static void set_threads(int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ---- codec ------------------------------------------------------------- */

/* eps[i][j] = (src[(i-1) mod m][j] << l) + src[i][j] */
void oracle_entangle(const int64_t *src, int64_t *eps, int m, int64_t n, int l, int nthreads) {
    set_threads(nthreads);
    for (int i = 0; i < m; ++i) {
        const int64_t *prev = src + (int64_t)((i + m - 1) % m) * n;
        const int64_t *cur = src + (int64_t)i * n;
        int64_t *o = eps + (int64_t)i * n;
#pragma omp parallel for schedule(static)
        for (int64_t j = 0; j < n; ++j) o[j] = wrap_add(wrap_shl(prev[j], l), cur[j]);
    }
}

/* Row-major index of the first element with |x| > hi (np.abs wraps), or -1. */
int64_t oracle_first_out_of_range(const int64_t *x, int64_t count, int64_t hi) {
    for (int64_t i = 0; i < count; ++i) {
        int64_t v = x[i];
        int64_t a = v < 0 ? (int64_t)(0 - (uint64_t)v) : v; /* wraps for INT64_MIN */
        if (a > hi) return i;
    }
    return -1;
}

/*
 * Recover all m streams from the m-1 streams != r.  Row r of delta is never
 * read.  wide=0 reproduces the numba int64 kernel bit for bit (including
 * wrap-around on inconsistent input); wide=1 reproduces the Python-int
 * reference.  Returns the number of positions whose out[r] did not fit int64
 * (the reference raises OverflowError there); those positions hold the
 * wrapped value.
 */
int64_t oracle_disentangle(const int64_t *delta, int64_t *out, int m, int64_t n, int l, int r,
                           int wide, int nthreads) {
    set_threads(nthreads);
    const int low = (m - 1) * l;
    const uint64_t mask = (low >= 64) ? ~(uint64_t)0 : (((uint64_t)1 << low) - 1);
    const uint64_t sbit = (uint64_t)1 << (low - 1);
    const int last = (r + m - 1) % m;
    int64_t overflow = 0;
#pragma omp parallel for schedule(static) reduction(+ : overflow)
    for (int64_t j = 0; j < n; ++j) {
        int64_t pivot_lo; /* low 64 bits of the pivot */
        i128 acc128 = 0;
        if (wide) {
            for (int t = 0; t <= m - 2; ++t) {
                i128 term = (i128)delta[(int64_t)((r + 1 + t) % m) * n + j];
                term = term * ((i128)1 << ((m - 2 - t) * l));
                acc128 = (t & 1) ? acc128 - term : acc128 + term;
            }
            pivot_lo = (int64_t)(uint64_t)(u128)acc128;
        } else {
            uint64_t acc = 0;
            for (int t = 0; t <= m - 2; ++t) {
                uint64_t term = (uint64_t)delta[(int64_t)((r + 1 + t) % m) * n + j] << ((m - 2 - t) * l);
                acc = (t & 1) ? acc - term : acc + term;
            }
            pivot_lo = (int64_t)acc;
        }
        int64_t v = (int64_t)((((uint64_t)pivot_lo & mask) ^ sbit) - sbit);
        out[(int64_t)last * n + j] = (m & 1) ? (int64_t)(0 - (uint64_t)v) : v;
        int64_t dr;
        if (wide) {
            i128 q = (acc128 - (i128)v) >> low;
            if (!fits_i64(q)) overflow += 1;
            dr = (int64_t)(uint64_t)(u128)q;
        } else {
            dr = wrap_sub(pivot_lo, v) >> low;
        }
        out[(int64_t)r * n + j] = dr;
        int64_t prev = dr;
        for (int t = 1; t <= m - 2; ++t) {
            int idx = (r + t) % m;
            prev = wrap_sub(delta[(int64_t)idx * n + j], wrap_shl(prev, l));
            out[(int64_t)idx * n + j] = prev;
        }
    }
    return overflow;
}

/* Independent m=3 recipe (codec.py:151-183): d_temp = delta[r+2] - (delta[r+1] << l). */
void oracle_disentangle_m3(const int64_t *delta, int64_t *out, int64_t n, int l, int w, int r) {
    const int64_t *a = delta + (int64_t)((r + 1) % 3) * n;
    const int64_t *b = delta + (int64_t)((r + 2) % 3) * n;
    for (int64_t j = 0; j < n; ++j) {
        int64_t d2, d0;
        if (w <= 32) {
            int64_t dt = wrap_sub(b[j], wrap_shl(a[j], l));
            int up = 2 * (w - l);
            if (w == 32) {
                d2 = (int64_t)((uint64_t)dt << up) >> up;
            } else {
                uint64_t mask = ((uint64_t)1 << (2 * l)) - 1, sb = (uint64_t)1 << (2 * l - 1);
                d2 = (int64_t)((((uint64_t)dt & mask) ^ sb) - sb);
            }
            d0 = (int64_t)(0 - (uint64_t)wrap_sub(dt, d2)) >> (2 * l);
        } else {
            i128 dt = (i128)b[j] - (i128)a[j] * ((i128)1 << l);
            u128 mask = (((u128)1) << (2 * l)) - 1, sb = ((u128)1) << (2 * l - 1);
            i128 d2w = (i128)((((u128)dt & mask) ^ sb) - sb);
            d2 = (int64_t)d2w;
            d0 = (int64_t)(-(dt - d2w) >> (2 * l));
        }
        out[(int64_t)((r + 2) % 3) * n + j] = d2;
        out[(int64_t)r * n + j] = d0;
        out[(int64_t)((r + 1) % 3) * n + j] = wrap_sub(a[j], wrap_shl(d0, l));
    }
}

/* ---- LSB operations ---------------------------------------------------- */

/*
 * y[row][j] = sum_{k<K} g[k] * x[row][(j-k) mod n], 1 <= K <= n.
 * wide=0: modulo 2^64.  wide=1: exact (__int128), returns the count of
 * outputs that do not fit int64 (stored wrapped).
 */
int64_t oracle_circ_conv(const int64_t *x, int rows, int64_t n, const int64_t *g, int K, int64_t *y,
                         int wide, int nthreads) {
    set_threads(nthreads);
    int64_t overflow = 0;
    const int64_t blocks = (n + 255) / 256;
    for (int row = 0; row < rows; ++row) {
        const int64_t *xr = x + (int64_t)row * n;
        int64_t *yr = y + (int64_t)row * n;
#pragma omp parallel for schedule(dynamic, 4) reduction(+ : overflow)
        for (int64_t blk = 0; blk < blocks; ++blk) {
            int64_t j0 = blk * 256, j1 = j0 + 256 < n ? j0 + 256 : n;
            for (int64_t j = j0; j < j1; ++j) {
                if (wide) {
                    i128 acc = 0;
                    for (int k = 0; k < K; ++k) {
                        int64_t idx = j - k;
                        if (idx < 0) idx += n;
                        acc += (i128)g[k] * (i128)xr[idx];
                    }
                    if (!fits_i64(acc)) overflow += 1;
                    yr[j] = (int64_t)(uint64_t)(u128)acc;
                } else {
                    uint64_t acc = 0;
                    /* split the tap range so the inner loop has no modulo */
                    int kmax = (int)(j + 1 < K ? j + 1 : K);
                    for (int k = 0; k < kmax; ++k) acc += (uint64_t)g[k] * (uint64_t)xr[j - k];
                    for (int k = kmax; k < K; ++k) acc += (uint64_t)g[k] * (uint64_t)xr[j - k + n];
                    yr[j] = (int64_t)acc;
                }
            }
        }
    }
    return overflow;
}

/* out[row][j] = x[row][(-j) mod n]  (ops.py:179-181) */
void oracle_reverse_circular(const int64_t *x, int rows, int64_t n, int64_t *out) {
    for (int row = 0; row < rows; ++row)
        for (int64_t j = 0; j < n; ++j)
            out[(int64_t)row * n + j] = x[(int64_t)row * n + (j == 0 ? 0 : n - j)];
}

/* op: 0 add, 1 sub, 2 mul.  g has length n (glen==n) or 1 (broadcast). */
int64_t oracle_elementwise(const int64_t *x, int rows, int64_t n, const int64_t *g, int64_t glen, int op,
                           int64_t *y, int wide) {
    int64_t overflow = 0;
    for (int row = 0; row < rows; ++row)
        for (int64_t j = 0; j < n; ++j) {
            int64_t a = x[(int64_t)row * n + j], b = g[glen == 1 ? 0 : j];
            int64_t v;
            if (op == 0) v = wrap_add(a, b);
            else if (op == 1) v = wrap_sub(a, b);
            else {
                v = wrap_mul(a, b);
                if (wide && !fits_i64((i128)a * (i128)b)) overflow += 1;
            }
            y[(int64_t)row * n + j] = v;
        }
    return overflow;
}

void oracle_permute(const int64_t *x, int rows, int64_t n, const int64_t *perm, int64_t *y) {
    for (int row = 0; row < rows; ++row)
        for (int64_t j = 0; j < n; ++j) y[(int64_t)row * n + j] = x[(int64_t)row * n + perm[j]];
}

/* y[row] = sum_j x[row][j] * g[j] */
int64_t oracle_inner(const int64_t *x, int rows, int64_t n, const int64_t *g, int64_t *y, int wide) {
    int64_t overflow = 0;
    for (int row = 0; row < rows; ++row) {
        uint64_t acc = 0;
        i128 exact = 0;
        for (int64_t j = 0; j < n; ++j) {
            acc += (uint64_t)x[(int64_t)row * n + j] * (uint64_t)g[j];
            if (wide) exact += (i128)x[(int64_t)row * n + j] * (i128)g[j];
        }
        if (wide && !fits_i64(exact)) overflow += 1;
        y[row] = (int64_t)acc;
    }
    return overflow;
}

/* y[row][c] = sum_j x[row][j] * G[j][c], G is n x p row-major */
int64_t oracle_gemm(const int64_t *x, int rows, int64_t n, const int64_t *G, int64_t p, int64_t *y, int wide) {
    int64_t overflow = 0;
    for (int row = 0; row < rows; ++row)
        for (int64_t c = 0; c < p; ++c) {
            uint64_t acc = 0;
            i128 exact = 0;
            for (int64_t j = 0; j < n; ++j) {
                acc += (uint64_t)x[(int64_t)row * n + j] * (uint64_t)G[j * p + c];
                if (wide) exact += (i128)x[(int64_t)row * n + j] * (i128)G[j * p + c];
            }
            if (wide && !fits_i64(exact)) overflow += 1;
            y[(int64_t)row * p + c] = (int64_t)acc;
        }
    return overflow;
}
