// lsb.cu -- the rest of the LSB catalogue on entangled streams:
// elementwise add/sub/mul, scale, permutation, circular reversal (xcorr),
// batched inner product (+ fused entangle->dot->extract), fused
// entangle->outer product->extract, and ROW_GEMM.
//
// Reference: /root/reference/pkg/src/nent/ops.py:184-238.  Arithmetic is
// modulo 2^64 like numpy's int64 paths; where the reference switches to exact
// Python ints (bound >= 2^62) the caller passes check=1 and the kernels count
// results that do not fit int64 (the reference raises OverflowError).
#include "common.cuh"
#include "recover.cuh"

namespace nent {

constexpr int LT = 256;

__device__ __forceinline__ bool mul_fits(int64_t a, int64_t b) {
  __int128 p = (__int128)a * (__int128)b;
  return p >= (__int128)INT64_MIN && p <= (__int128)INT64_MAX;
}

template <typename TI, typename TG, typename TO>
__global__ void __launch_bounds__(LT)
elementwise_kernel(const Rows x, int rows, int64_t n, const TG* g, int64_t g_len, int op,
                   MutRows y, int check, unsigned long long* ovf) {
  const int row = blockIdx.y;
  const TI* xp = reinterpret_cast<const TI*>(x.p[row]);
  TO* yp = reinterpret_cast<TO*>(y.p[row]);
  unsigned bad = 0;
  for (int64_t j = (int64_t)blockIdx.x * LT + threadIdx.x; j < n; j += (int64_t)gridDim.x * LT) {
    const int64_t a = (int64_t)__ldg(xp + j);
    const int64_t b = (int64_t)__ldg(g + (g_len == 1 ? 0 : j));
    int64_t v;
    if (op == NENT_EW_ADD) v = wadd(a, b);
    else if (op == NENT_EW_SUB) v = wsub(a, b);
    else {
      v = wmul(a, b);
      if (check && !mul_fits(a, b)) ++bad;
    }
    yp[j] = (TO)(uint64_t)v;
  }
  if (check && bad) atomicAdd(ovf, (unsigned long long)bad);
}

template <typename TI, typename TO>
__global__ void __launch_bounds__(LT)
scale_kernel(const Rows x, int64_t n, int64_t s, MutRows y, int check, unsigned long long* ovf) {
  const int row = blockIdx.y;
  const TI* xp = reinterpret_cast<const TI*>(x.p[row]);
  TO* yp = reinterpret_cast<TO*>(y.p[row]);
  unsigned bad = 0;
  for (int64_t j = (int64_t)blockIdx.x * LT + threadIdx.x; j < n; j += (int64_t)gridDim.x * LT) {
    const int64_t a = (int64_t)__ldg(xp + j);
    if (check && !mul_fits(a, s)) ++bad;
    yp[j] = (TO)(uint64_t)wmul(a, s);
  }
  if (check && bad) atomicAdd(ovf, (unsigned long long)bad);
}

// All rows gathered by the same index: perm[j] is loaded once per position.
template <typename TI, typename TO>
__global__ void __launch_bounds__(LT)
permute_kernel(const Rows x, int rows, int64_t n, const int64_t* __restrict__ perm, MutRows y) {
  for (int64_t j = (int64_t)blockIdx.x * LT + threadIdx.x; j < n; j += (int64_t)gridDim.x * LT) {
    const int64_t q = __ldg(perm + j);
    for (int row = 0; row < rows; ++row)
      reinterpret_cast<TO*>(y.p[row])[j] =
          (TO)(uint64_t)(int64_t)__ldg(reinterpret_cast<const TI*>(x.p[row]) + q);
  }
}

template <typename TI, typename TO>
__global__ void __launch_bounds__(LT)
reverse_kernel(const Rows x, int64_t n, MutRows y) {
  const int row = blockIdx.y;
  const TI* xp = reinterpret_cast<const TI*>(x.p[row]);
  TO* yp = reinterpret_cast<TO*>(y.p[row]);
  for (int64_t j = (int64_t)blockIdx.x * LT + threadIdx.x; j < n; j += (int64_t)gridDim.x * LT)
    yp[j] = (TO)(uint64_t)(int64_t)__ldg(xp + (j == 0 ? 0 : n - j));
}

// ------------------------------------------------------------ inner product --
// One warp per (row, vector): lanes stride the vector, int64 (mod 2^64)
// accumulation with IMAD.WIDE when both operands fit int32 (W64) or a
// generic 64-bit MAC (G64); an exact 128-bit sum only when check is set.
template <int FLAV>
__device__ __forceinline__ void dot_mac(unsigned long long& acc, int64_t x, int64_t g) {
  if (FLAV == NENT_MAC_W64)
    acc += (unsigned long long)((long long)(int32_t)x * (long long)(int32_t)g);
  else
    acc += (unsigned long long)x * (unsigned long long)g;
}

template <typename TI, typename TG, int FLAV>
__global__ void __launch_bounds__(LT)
inner_kernel(const Rows x, int rows, int64_t batch, int64_t n, const TG* __restrict__ g,
             MutRows y, int check, unsigned long long* ovf) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * LT + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * LT) >> 5;
  for (int64_t v = warp; v < (int64_t)rows * batch; v += nwarps) {
    const int row = (int)(v / batch);
    const int64_t b = v - (int64_t)row * batch;
    const TI* xp = reinterpret_cast<const TI*>(x.p[row]) + b * n;
    unsigned long long acc = 0;
    __int128 exact = 0;
    for (int64_t i = lane; i < n; i += 32) {
      const int64_t xv = (int64_t)__ldg(xp + i), gv = (int64_t)__ldg(g + i);
      dot_mac<FLAV>(acc, xv, gv);
      if (check) exact += (__int128)xv * (__int128)gv;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (check) {
        long long hi = (long long)(exact >> 64);
        unsigned long long lo = (unsigned long long)exact;
        hi = __shfl_xor_sync(0xffffffffu, hi, o);
        lo = __shfl_xor_sync(0xffffffffu, lo, o);
        exact += ((__int128)hi << 64) + (__int128)lo;
      }
    }
    if (lane == 0) {
      reinterpret_cast<int64_t*>(y.p[row])[b] = (int64_t)acc;
      if (check && (exact < (__int128)INT64_MIN || exact > (__int128)INT64_MAX)) atomicAdd(ovf, 1ull);
    }
  }
}

// Fused cfg4 inner path: entangle on load, dot, extract; one warp per vector
// index b holding all m streams, so the m dots meet in one lane.
template <int MT, typename TI, typename TG, int FLAV>
__global__ void __launch_bounds__(LT)
fused_inner_kernel(const Rows c, int64_t batch, int64_t n, int l, const TG* __restrict__ g,
                   int r, int vec_ok, MutRows d, int d_bits, unsigned long long* mismatch) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * LT + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * LT) >> 5;
  const bool verify = r < 0;
  const int pivot = verify ? 0 : r;
  unsigned bad = 0;
  for (int64_t b = warp; b < batch; b += nwarps) {
    unsigned long long acc[MT];
#pragma unroll
    for (int s = 0; s < MT; ++s) acc[s] = 0;
    const int64_t off = b * n;
    if (sizeof(TI) == 4 && (n & 3) == 0 && vec_ok) {
      // 16-byte loads, 4 independent iterations in flight: 4*MT LDG.128 per lane
      const int64_t n4 = n >> 2;
      for (int64_t i0 = lane; i0 < n4; i0 += 128) {
        int4 cv[4][MT];
        int4 gv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t i = i0 + 32 * u;
          if (i < n4) {
#pragma unroll
            for (int s = 0; s < MT; ++s)
              cv[u][s] = __ldg(reinterpret_cast<const int4*>(reinterpret_cast<const TI*>(c.p[s]) + off) + i);
            if (sizeof(TG) == 4) gv[u] = __ldg(reinterpret_cast<const int4*>(g) + i);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t i = i0 + 32 * u;
          if (i >= n4) break;
          int64_t gl[4];
          if (sizeof(TG) == 4) {
            gl[0] = gv[u].x; gl[1] = gv[u].y; gl[2] = gv[u].z; gl[3] = gv[u].w;
          } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) gl[e] = (int64_t)__ldg(g + 4 * i + e);
          }
#pragma unroll
          for (int s = 0; s < MT; ++s) {
            const int4 a = cv[u][(s + MT - 1) % MT], bb = cv[u][s];
            dot_mac<FLAV>(acc[s], wadd(wshl(a.x, l), bb.x), gl[0]);
            dot_mac<FLAV>(acc[s], wadd(wshl(a.y, l), bb.y), gl[1]);
            dot_mac<FLAV>(acc[s], wadd(wshl(a.z, l), bb.z), gl[2]);
            dot_mac<FLAV>(acc[s], wadd(wshl(a.w, l), bb.w), gl[3]);
          }
        }
      }
    } else {
      for (int64_t i = lane; i < n; i += 32) {
        int64_t cv[MT];
#pragma unroll
        for (int s = 0; s < MT; ++s) cv[s] = (int64_t)__ldg(reinterpret_cast<const TI*>(c.p[s]) + off + i);
        const int64_t gv = (int64_t)__ldg(g + i);
#pragma unroll
        for (int s = 0; s < MT; ++s) {
          const int64_t e = wadd(wshl(cv[(s + MT - 1) % MT], l), cv[s]);
          dot_mac<FLAV>(acc[s], e, gv);
        }
      }
    }
#pragma unroll
    for (int s = 0; s < MT; ++s)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[s] += __shfl_xor_sync(0xffffffffu, acc[s], o);
    if (lane == 0) {
      int64_t dl[MT], orot[MT];
#pragma unroll
      for (int s = 0; s < MT; ++s) dl[s] = (int64_t)acc[s];
      recover_regs_valid<MT>(dl, pivot, l, orot);
      if (verify) bad += (dl[0] != wadd(wshl(orot[MT - 1], l), orot[0])) ? 1u : 0u;
#pragma unroll
      for (int t = 0; t < MT; ++t) {
        int row = pivot + t;
        row -= row >= MT ? MT : 0;
        st_bits(d.p[row], d_bits, b, orot[t]);
      }
    }
  }
  if (mismatch && lane == 0 && bad) atomicAdd(mismatch, (unsigned long long)bad);
}

// Fused cfg4 outer path.  Block (u-tile, vector b): every thread owns 4
// consecutive v per row u; entangled products are formed, the m-1 surviving
// ones recovered in registers, d written (optional) and summed per stream.
constexpr int OUTER_U = 8;  // rows u per block

template <int MT, typename TI, typename TG, typename TO>
__global__ void __launch_bounds__(LT)
fused_outer_kernel(const Rows c, int64_t n, int l, const TG* __restrict__ g, int64_t p, int r,
                   int wide, MutRows d, long long* sums, int64_t batch) {
  const int64_t b = blockIdx.y;
  const int64_t u0 = (int64_t)blockIdx.x * OUTER_U;
  const int pivot = r < 0 ? 0 : r;
  long long part[MT];
#pragma unroll
  for (int s = 0; s < MT; ++s) part[s] = 0;
  for (int64_t u = u0; u < u0 + OUTER_U && u < n; ++u) {
    int64_t cv[MT], e[MT];
#pragma unroll
    for (int s = 0; s < MT; ++s) cv[s] = (int64_t)__ldg(reinterpret_cast<const TI*>(c.p[s]) + b * n + u);
#pragma unroll
    for (int s = 0; s < MT; ++s) e[s] = wadd(wshl(cv[(s + MT - 1) % MT], l), cv[s]);
    // Fast path (the cfg4 shape): entangled words and taps that fit int32 make
    // every product one IMAD.WIDE, and int32 outputs leave as 16-byte vectors
    // (four consecutive v per thread).  Block-uniform choice per row u.
    bool narrow = sizeof(TG) == 4 && sizeof(TO) == 4 && (p & 3) == 0;
#pragma unroll
    for (int s = 0; s < MT; ++s) narrow = narrow && e[s] == (int64_t)(int32_t)e[s];
#pragma unroll
    for (int s = 0; s < MT; ++s)
      narrow = narrow && (!d.p[s] || (reinterpret_cast<uintptr_t>(d.p[s]) & 15) == 0);
    narrow = narrow && (reinterpret_cast<uintptr_t>(g) & 15) == 0;
    if (narrow) {
      const int64_t base = (b * n + u) * p;
      // the m-1 surviving entangled words in rotation order, once per row u
      // (the pivot's product is never formed, as in the reference's recovery)
      int32_t erot[MT - 1];
#pragma unroll
      for (int t = 0; t < MT - 1; ++t) {
        int idx = pivot + 1 + t;
        idx -= idx >= MT ? MT : 0;
        erot[t] = (int32_t)select_mod<MT>(e, idx);
      }
      for (int64_t v = 4 * (int64_t)threadIdx.x; v < p; v += 4 * LT) {
        const int4 g4 = __ldg(reinterpret_cast<const int4*>(g + v));
        const int gq[4] = {g4.x, g4.y, g4.z, g4.w};
        int o32[MT][4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          int64_t rot[MT - 1], orot[MT];
#pragma unroll
          for (int t = 0; t < MT - 1; ++t) rot[t] = (int64_t)erot[t] * (int64_t)gq[q];
          recover_rot_valid<MT>(rot, l, orot);
#pragma unroll
          for (int t = 0; t < MT; ++t) {
            o32[t][q] = (int)(uint32_t)(uint64_t)orot[t];
            if (sums) part[t] += orot[t];
          }
        }
#pragma unroll
        for (int t = 0; t < MT; ++t) {
          int row = pivot + t;
          row -= row >= MT ? MT : 0;
          if (d.p[row])
            *reinterpret_cast<int4*>(reinterpret_cast<TO*>(d.p[row]) + base + v) =
                make_int4(o32[t][0], o32[t][1], o32[t][2], o32[t][3]);
        }
      }
      continue;
    }
    for (int64_t v = threadIdx.x; v < p; v += LT) {
      const int64_t gv = (int64_t)__ldg(g + v);
      int64_t dl[MT], orot[MT];
#pragma unroll
      for (int s = 0; s < MT; ++s) dl[s] = wmul(e[s], gv);
      recover_regs_valid<MT>(dl, pivot, l, orot);
#pragma unroll
      for (int t = 0; t < MT; ++t) {
        int row = pivot + t;
        row -= row >= MT ? MT : 0;
        if (d.p[row]) reinterpret_cast<TO*>(d.p[row])[(b * n + u) * p + v] = (TO)(uint64_t)orot[t];
        part[t] += orot[t];  // rotated: part[t] belongs to stream (pivot + t) mod m
      }
    }
  }
  if (sums) {
    __shared__ long long red[MT][LT / 32];
#pragma unroll
    for (int s = 0; s < MT; ++s) {
      long long v = part[s];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      int stream_id = pivot + s;
      stream_id -= stream_id >= MT ? MT : 0;
      if ((threadIdx.x & 31) == 0) red[stream_id][threadIdx.x >> 5] = v;
    }
    __syncthreads();
    if (threadIdx.x < MT) {
      long long t = 0;
      for (int w = 0; w < LT / 32; ++w) t += red[threadIdx.x][w];
      atomicAdd((unsigned long long*)&sums[threadIdx.x * batch + b], (unsigned long long)t);
    }
  }
}

// ROW_GEMM: one thread per (row, column); exact 128-bit check on request.
template <typename TI, typename TO>
__global__ void __launch_bounds__(LT)
gemm_kernel(const Rows x, int rows, int64_t n, const int64_t* __restrict__ G, int64_t p,
            MutRows y, int check, unsigned long long* ovf) {
  const int row = blockIdx.y;
  const TI* xp = reinterpret_cast<const TI*>(x.p[row]);
  for (int64_t col = (int64_t)blockIdx.x * LT + threadIdx.x; col < p; col += (int64_t)gridDim.x * LT) {
    unsigned long long acc = 0;
    __int128 exact = 0;
    for (int64_t j = 0; j < n; ++j) {
      const int64_t a = (int64_t)__ldg(xp + j), b = __ldg(G + j * p + col);
      acc += (unsigned long long)a * (unsigned long long)b;
      if (check) exact += (__int128)a * (__int128)b;
    }
    reinterpret_cast<TO*>(y.p[row])[col] = (TO)acc;
    if (check && (exact < (__int128)INT64_MIN || exact > (__int128)INT64_MAX)) atomicAdd(ovf, 1ull);
  }
}

}  // namespace nent

using namespace nent;

#define DISPATCH_G(gb, ...)                              \
  do {                                                   \
    if ((gb) == 32) { typedef int32_t TG; __VA_ARGS__; } \
    else { typedef int64_t TG; __VA_ARGS__; }            \
  } while (0)

extern "C" {

int nent_elementwise(const void* const* x, int x_bits, int rows, int64_t n, const void* g,
                     int g_bits, int64_t g_len, int op, void* const* y, int y_bits, int check,
                     unsigned long long* overflow_dev, void* stream) {
  NENT_CHECK_BITS(x_bits); NENT_CHECK_BITS(g_bits); NENT_CHECK_BITS(y_bits);
  if (rows < 1 || rows > NENT_MAX_STREAMS || (g_len != 1 && g_len != n) || op < 0 || op > 2) {
    set_error("elementwise: bad arguments"); return NENT_ERR_PARAM;
  }
  if (n <= 0) return NENT_OK;
  cudaStream_t s = as_stream(stream);
  Rows X = to_rows(x, rows); MutRows Y = to_mrows(y, rows);
  dim3 grid(grid_for(n, LT, 4, 148 * 8), rows);
  DISPATCH_G(g_bits, DISPATCH_IO(x_bits, y_bits, (elementwise_kernel<TI, TG, TO><<<grid, LT, 0, s>>>(
                                                     X, rows, n, (const TG*)g, g_len, op, Y, check, overflow_dev))));
  return check_launch("elementwise");
}

int nent_scale(const void* const* x, int x_bits, int rows, int64_t n, int64_t sc, void* const* y,
               int y_bits, int check, unsigned long long* overflow_dev, void* stream) {
  NENT_CHECK_BITS(x_bits); NENT_CHECK_BITS(y_bits);
  if (rows < 1 || rows > NENT_MAX_STREAMS) { set_error("scale: bad rows"); return NENT_ERR_PARAM; }
  if (n <= 0) return NENT_OK;
  cudaStream_t s = as_stream(stream);
  Rows X = to_rows(x, rows); MutRows Y = to_mrows(y, rows);
  dim3 grid(grid_for(n, LT, 4, 148 * 8), rows);
  DISPATCH_IO(x_bits, y_bits, (scale_kernel<TI, TO><<<grid, LT, 0, s>>>(X, n, sc, Y, check, overflow_dev)));
  return check_launch("scale");
}

int nent_permute(const void* const* x, int x_bits, int rows, int64_t n, const int64_t* perm,
                 void* const* y, int y_bits, void* stream) {
  NENT_CHECK_BITS(x_bits); NENT_CHECK_BITS(y_bits);
  if (rows < 1 || rows > NENT_MAX_STREAMS) { set_error("permute: bad rows"); return NENT_ERR_PARAM; }
  if (n <= 0) return NENT_OK;
  cudaStream_t s = as_stream(stream);
  Rows X = to_rows(x, rows); MutRows Y = to_mrows(y, rows);
  int grid = grid_for(n, LT, 4);
  DISPATCH_IO(x_bits, y_bits, (permute_kernel<TI, TO><<<grid, LT, 0, s>>>(X, rows, n, perm, Y)));
  return check_launch("permute");
}

int nent_reverse_circular(const void* const* x, int x_bits, int rows, int64_t n, void* const* y,
                          int y_bits, void* stream) {
  NENT_CHECK_BITS(x_bits); NENT_CHECK_BITS(y_bits);
  if (rows < 1 || rows > NENT_MAX_STREAMS) { set_error("reverse: bad rows"); return NENT_ERR_PARAM; }
  if (n <= 0) return NENT_OK;
  cudaStream_t s = as_stream(stream);
  Rows X = to_rows(x, rows); MutRows Y = to_mrows(y, rows);
  dim3 grid(grid_for(n, LT, 4, 148 * 8), rows);
  DISPATCH_IO(x_bits, y_bits, (reverse_kernel<TI, TO><<<grid, LT, 0, s>>>(X, n, Y)));
  return check_launch("reverse_circular");
}

int nent_inner(const void* const* x, int x_bits, int rows, int64_t batch, int64_t n,
               const void* g, int g_bits, void* const* y, int flavor, int check,
               unsigned long long* overflow_dev, void* stream) {
  NENT_CHECK_BITS(x_bits); NENT_CHECK_BITS(g_bits);
  if (rows < 1 || rows > NENT_MAX_STREAMS || batch < 0 || n < 1) {
    set_error("inner: bad arguments"); return NENT_ERR_PARAM;
  }
  if (batch == 0) return NENT_OK;
  cudaStream_t s = as_stream(stream);
  Rows X = to_rows(x, rows); MutRows Y = to_mrows(y, rows);
  int grid = grid_for((int64_t)rows * batch * 32, LT, 1, 148 * 16);
#define INNER_CASE(F)                                                                          \
  DISPATCH_G(g_bits, if (x_bits == 32) inner_kernel<int32_t, TG, F><<<grid, LT, 0, s>>>(      \
                         X, rows, batch, n, (const TG*)g, Y, check, overflow_dev);            \
                     else inner_kernel<int64_t, TG, F><<<grid, LT, 0, s>>>(                    \
                         X, rows, batch, n, (const TG*)g, Y, check, overflow_dev))
  if (flavor == NENT_MAC_W64) INNER_CASE(NENT_MAC_W64);
  else INNER_CASE(NENT_MAC_G64);
#undef INNER_CASE
  return check_launch("inner");
}

int nent_fused_inner(const void* const* c, int c_bits, int m, int64_t batch, int64_t n, int l,
                     const void* g, int g_bits, int r, int wide, void* const* d, int d_bits,
                     int flavor, unsigned long long* mismatch_dev, void* stream) {
  NENT_CHECK_BITS(c_bits); NENT_CHECK_BITS(g_bits); NENT_CHECK_BITS(d_bits);
  if (m < 3 || m > 8 || r < -1 || r >= m || batch < 0 || n < 1 || l < 1 || (m - 1) * l > 63) {
    set_error("fused_inner: bad arguments"); return NENT_ERR_PARAM;
  }
  if (batch == 0) return NENT_OK;
  cudaStream_t s = as_stream(stream);
  Rows C = to_rows(c, m); MutRows D = to_mrows(d, m);
  (void)wide;  // the fused recovery is exact for any w <= 64 on consistent words
  // 16-byte vector loads when every vector of every row is 16-byte aligned
  int vec_ok = c_bits == 32 && (n & 3) == 0 && (g_bits == 64 || ((uintptr_t)g & 15) == 0);
  for (int i = 0; i < m; ++i) vec_ok = vec_ok && ((uintptr_t)c[i] & 15) == 0;
  int grid = grid_for(batch * 32, LT, 1, 148 * 16);
#define FI_CASE(MTV, F)                                                                         \
  DISPATCH_G(g_bits, if (c_bits == 32) fused_inner_kernel<MTV, int32_t, TG, F><<<grid, LT, 0, s>>>( \
                         C, batch, n, l, (const TG*)g, r, vec_ok, D, d_bits, mismatch_dev);        \
                     else fused_inner_kernel<MTV, int64_t, TG, F><<<grid, LT, 0, s>>>(             \
                         C, batch, n, l, (const TG*)g, r, vec_ok, D, d_bits, mismatch_dev))
#define FI_M(F)                                   \
  switch (m) {                                    \
    case 3: FI_CASE(3, F); break;                 \
    case 4: FI_CASE(4, F); break;                 \
    case 5: FI_CASE(5, F); break;                 \
    case 6: FI_CASE(6, F); break;                 \
    case 7: FI_CASE(7, F); break;                 \
    default: FI_CASE(8, F); break;                \
  }
  if (flavor == NENT_MAC_W64) { FI_M(NENT_MAC_W64); }
  else { FI_M(NENT_MAC_G64); }
#undef FI_M
#undef FI_CASE
  return check_launch("fused_inner");
}

int nent_fused_outer(const void* const* c, int c_bits, int m, int64_t batch, int64_t n, int l,
                     const void* g, int g_bits, int64_t p, int r, int wide, void* const* d,
                     int d_bits, long long* sums_dev, void* stream) {
  NENT_CHECK_BITS(c_bits); NENT_CHECK_BITS(g_bits); NENT_CHECK_BITS(d_bits);
  if (m < 3 || m > 8 || r < -1 || r >= m || batch < 0 || n < 1 || p < 1 || l < 1 ||
      (m - 1) * l > 63 || batch > 65535) {
    set_error("fused_outer: bad arguments"); return NENT_ERR_PARAM;
  }
  if (batch == 0) return NENT_OK;
  cudaStream_t s = as_stream(stream);
  Rows C = to_rows(c, m);
  MutRows D{};
  if (d) D = to_mrows(d, m);
  dim3 grid((unsigned)((n + OUTER_U - 1) / OUTER_U), (unsigned)batch);
#define FO_CASE(MTV)                                                                          \
  DISPATCH_G(g_bits, DISPATCH_IO(c_bits, d_bits, (fused_outer_kernel<MTV, TI, TG, TO><<<grid, LT, 0, s>>>( \
                                                     C, n, l, (const TG*)g, p, r, wide, D, sums_dev, batch))))
  switch (m) {
    case 3: FO_CASE(3); break;
    case 4: FO_CASE(4); break;
    case 5: FO_CASE(5); break;
    case 6: FO_CASE(6); break;
    case 7: FO_CASE(7); break;
    default: FO_CASE(8); break;
  }
#undef FO_CASE
  return check_launch("fused_outer");
}

int nent_gemm(const void* const* x, int x_bits, int rows, int64_t n, const int64_t* G, int64_t p,
              void* const* y, int y_bits, int check, unsigned long long* overflow_dev,
              void* stream) {
  NENT_CHECK_BITS(x_bits); NENT_CHECK_BITS(y_bits);
  if (rows < 1 || rows > NENT_MAX_STREAMS || n < 1 || p < 1) {
    set_error("gemm: bad arguments"); return NENT_ERR_PARAM;
  }
  cudaStream_t s = as_stream(stream);
  Rows X = to_rows(x, rows); MutRows Y = to_mrows(y, rows);
  dim3 grid(grid_for(p, LT, 1, 148 * 8), rows);
  DISPATCH_IO(x_bits, y_bits, (gemm_kernel<TI, TO><<<grid, LT, 0, s>>>(X, rows, n, G, p, Y, check, overflow_dev)));
  return check_launch("gemm");
}

}  // extern "C"
