// conv.cu -- K2 direct integer convolution and K2f, the fused
// entangle -> (scale/add/permute) -> convolve -> extract hot path.
//
// Reference: ops._circ_conv_rows (/root/reference/pkg/src/nent/ops.py:158-172)
// computes  y[j] = sum_k g[k] x[(j-k) mod n]  with np.convolve in int64; the
// fused chain is bench.py's entangled() closure (bench.py:103-106) and the
// cfg5 pipeline chain (ops.py:193-204, 219-220).
//
// Design (B200, CUDA cores; the work is exact integer MACs):
//   * A CTA owns an output tile of T = 128*R positions for MS streams.  The
//     input tile + (K-1) halo is staged once in shared memory, already in the
//     MAC flavour's operand representation, by the prologue (which also
//     entangles, scales, adds and gathers on load -- nothing intermediate
//     touches HBM).
//   * Each thread keeps R consecutive outputs of every stream in registers.
//     Taps are consumed G=8 at a time: one broadcast 16-byte LDS of 8 taps,
//     then per stream a window of R+G inputs via 16-byte LDS, then R*G MACs.
//     R = 12 (32-bit operands) or 10 (64-bit) makes the per-thread window
//     starts 48 / 80 bytes apart, so each quarter-warp's 16-byte loads hit 8
//     distinct bank quads (conflict-free).
//   * Long filters are staged in KSEG-tap segments so shared memory stays
//     bounded for any K <= n.
//   * Epilogue: store the rows, or (fused) rebuild all m outputs from the m-1
//     surviving accumulators in registers (recover.cuh); the redundant
//     stream doubles as a silent-error check when no worker failed.
#include "common.cuh"
#include "recover.cuh"
#include "conv_common.cuh"

namespace nent {

constexpr int CV_NT = 128;  // threads per CTA
constexpr int CV_G = 8;     // taps per register chunk

// ------------------------------------------------------------- MAC flavours --
template <int FLAV>
struct Mac;

template <>
struct Mac<NENT_MAC_I32> {  // 1 IMAD; exact when |y| < 2^31 (result mod 2^32)
  typedef int32_t XT;
  typedef int32_t GT;
  static constexpr int NX = 1;
  struct Acc { uint32_t v; };
  __device__ static void zero(Acc& a) { a.v = 0; }
  __device__ static void to_x(int64_t v, XT* x0, XT*, int i) { x0[i] = (int32_t)(uint32_t)(uint64_t)v; }
  __device__ static GT to_g(int64_t v) { return (int32_t)(uint32_t)(uint64_t)v; }
  __device__ static void mac(Acc& a, GT g, XT x, XT) { a.v += (uint32_t)g * (uint32_t)x; }
  __device__ static int64_t value(const Acc& a) { return (int64_t)(int32_t)a.v; }
  __device__ static bool fits(const Acc&) { return true; }
};

template <>
struct Mac<NENT_MAC_W64> {  // 1 IMAD.WIDE: s32*s32 + s64
  typedef int32_t XT;
  typedef int32_t GT;
  static constexpr int NX = 1;
  struct Acc { long long v; };
  __device__ static void zero(Acc& a) { a.v = 0; }
  __device__ static void to_x(int64_t v, XT* x0, XT*, int i) { x0[i] = (int32_t)(uint32_t)(uint64_t)v; }
  __device__ static GT to_g(int64_t v) { return (int32_t)(uint32_t)(uint64_t)v; }
  __device__ static void mac(Acc& a, GT g, XT x, XT) {
    a.v = (long long)((unsigned long long)a.v + (unsigned long long)((long long)g * (long long)x));
  }
  __device__ static int64_t value(const Acc& a) { return a.v; }
  __device__ static bool fits(const Acc&) { return true; }
};

template <>
struct Mac<NENT_MAC_S64> {  // x = hi*2^32 + lo (lo signed): IMAD.WIDE(lo) + IMAD(hi), mod 2^64
  typedef int32_t XT;
  typedef int32_t GT;
  static constexpr int NX = 2;
  struct Acc { long long lo; uint32_t hi; };
  __device__ static void zero(Acc& a) { a.lo = 0; a.hi = 0; }
  __device__ static void to_x(int64_t v, XT* x0, XT* x1, int i) {
    int32_t lo = (int32_t)(uint32_t)(uint64_t)v;
    x0[i] = lo;
    x1[i] = (int32_t)(uint32_t)(((uint64_t)v - (uint64_t)(int64_t)lo) >> 32);
  }
  __device__ static GT to_g(int64_t v) { return (int32_t)(uint32_t)(uint64_t)v; }
  __device__ static void mac(Acc& a, GT g, XT lo, XT hi) {
    a.lo = (long long)((unsigned long long)a.lo + (unsigned long long)((long long)g * (long long)lo));
    a.hi += (uint32_t)g * (uint32_t)hi;
  }
  __device__ static int64_t value(const Acc& a) {
    return (int64_t)((uint64_t)a.lo + ((uint64_t)a.hi << 32));
  }
  __device__ static bool fits(const Acc&) { return true; }
};

template <>
struct Mac<NENT_MAC_F64> {  // 1 DFMA; exact while operands and partial sums < 2^53
  typedef double XT;
  typedef double GT;
  static constexpr int NX = 1;
  struct Acc { double v; };
  __device__ static void zero(Acc& a) { a.v = 0.0; }
  __device__ static void to_x(int64_t v, XT* x0, XT*, int i) { x0[i] = (double)v; }
  __device__ static GT to_g(int64_t v) { return (double)v; }
  __device__ static void mac(Acc& a, GT g, XT x, XT) { a.v = fma(g, x, a.v); }
  __device__ static int64_t value(const Acc& a) { return (int64_t)__double2ll_rn(a.v); }
  __device__ static bool fits(const Acc&) { return true; }
};

template <>
struct Mac<NENT_MAC_G64> {  // generic 64x64 -> low 64 (mul.lo.u64)
  typedef long long XT;
  typedef long long GT;
  static constexpr int NX = 1;
  struct Acc { unsigned long long v; };
  __device__ static void zero(Acc& a) { a.v = 0; }
  __device__ static void to_x(int64_t v, XT* x0, XT*, int i) { x0[i] = v; }
  __device__ static GT to_g(int64_t v) { return v; }
  __device__ static void mac(Acc& a, GT g, XT x, XT) { a.v += (unsigned long long)g * (unsigned long long)x; }
  __device__ static int64_t value(const Acc& a) { return (int64_t)a.v; }
  __device__ static bool fits(const Acc&) { return true; }
};

template <>
struct Mac<NENT_MAC_X128> {  // exact 128-bit sum: the reference's object path (bound >= 2^62)
  typedef long long XT;
  typedef long long GT;
  static constexpr int NX = 1;
  struct Acc { __int128 v; };
  __device__ static void zero(Acc& a) { a.v = 0; }
  __device__ static void to_x(int64_t v, XT* x0, XT*, int i) { x0[i] = v; }
  __device__ static GT to_g(int64_t v) { return v; }
  __device__ static void mac(Acc& a, GT g, XT x, XT) { a.v += (__int128)g * (__int128)x; }
  __device__ static int64_t value(const Acc& a) { return (int64_t)a.v; }
  __device__ static bool fits(const Acc& a) { return a.v >= (__int128)INT64_MIN && a.v <= (__int128)INT64_MAX; }
};

__host__ __device__ constexpr int pick_R(int flav, int ms) {
  // accumulator registers per thread (MS*R*words) kept <= ~120 so the fused
  // extraction epilogue fits in 255 registers without spilling
  return flav == NENT_MAC_X128 ? 2
         : (flav == NENT_MAC_F64 || flav == NENT_MAC_G64)
             ? (ms * 2 * 10 <= 120 ? 10 : 6)
             : (ms * (flav == NENT_MAC_I32 ? 2 : flav == NENT_MAC_S64 ? 3 : 2) * 12 <= 120 ? 12 : 4);
}

// 16-byte shared-memory vector loads into register arrays.
template <int N>
__device__ __forceinline__ void lds_vec(int32_t (&w)[N], const int32_t* src) {
#pragma unroll
  for (int i = 0; i < N / 4; ++i) {
    int4 v = reinterpret_cast<const int4*>(src)[i];
    w[4 * i] = v.x; w[4 * i + 1] = v.y; w[4 * i + 2] = v.z; w[4 * i + 3] = v.w;
  }
}
template <int N>
__device__ __forceinline__ void lds_vec(double (&w)[N], const double* src) {
#pragma unroll
  for (int i = 0; i < N / 2; ++i) {
    double2 v = reinterpret_cast<const double2*>(src)[i];
    w[2 * i] = v.x; w[2 * i + 1] = v.y;
  }
}
template <int N>
__device__ __forceinline__ void lds_vec(long long (&w)[N], const long long* src) {
#pragma unroll
  for (int i = 0; i < N / 2; ++i) {
    longlong2 v = reinterpret_cast<const longlong2*>(src)[i];
    w[2 * i] = v.x; w[2 * i + 1] = v.y;
  }
}

// 4 CTAs (16 warps) per SM when the accumulators leave room for <= 128
// registers per thread, else 2 (<= 255 registers, no spills).
// (checked with -Xptxas -warn-spills: every instantiation is spill-free)
__host__ __device__ constexpr int conv_min_blocks(int flav, int ms) {
  return (flav == NENT_MAC_I32 && (ms <= 3 || pick_R(flav, ms) == 4)) ||
                 (flav == NENT_MAC_F64 && ms <= 3) || (flav == NENT_MAC_W64 && ms <= 2) ||
                 (flav == NENT_MAC_S64 && ms == 1)
             ? 4
             : 2;
}

template <int FLAV, int MS, bool EXTRACT>
__global__ void __launch_bounds__(CV_NT, conv_min_blocks(FLAV, MS))
    conv_tile_kernel(const __grid_constant__ ConvArgs A) {
  using MT = Mac<FLAV>;
  typedef typename MT::XT XT;
  typedef typename MT::GT GT;
  constexpr int R = pick_R(FLAV, MS);
  constexpr int G = CV_G;
  constexpr int NW = R + G;
  constexpr int T = CV_NT * R;
  extern __shared__ __align__(16) unsigned char smem[];
  GT* gs = reinterpret_cast<GT*>(smem);
  XT* xs = reinterpret_cast<XT*>(smem + A.gbytes);
  const int S = A.sstride;
  const int tid = threadIdx.x;
  const int64_t j0 = A.y_begin + (int64_t)blockIdx.x * T;
  const int row0 = EXTRACT ? 0 : (int)blockIdx.y * MS;

  typename MT::Acc acc[MS][R];
#pragma unroll
  for (int s = 0; s < MS; ++s)
#pragma unroll
    for (int r = 0; r < R; ++r) MT::zero(acc[s][r]);

  for (int kb = 0; kb < A.Kp; kb += A.kseg) {
    const int KS = min(A.kseg, A.Kp - kb);
    if (kb > 0) __syncthreads();
    for (int i = tid; i < KS; i += CV_NT) {
      const int k = kb + i;
      gs[i] = MT::to_g(k < A.K ? ld_bits(A.g, A.g_bits, k) : 0);
    }
    // smem index i <-> input position p0 + i; the windows touch [0, T+KS)
    const int64_t p0 = j0 - kb - KS + 1;
    const int NS = T + KS;
#pragma unroll 1
    for (int s = 0; s < MS; ++s) {
      const int row = row0 + s;
      XT* x0 = xs + (size_t)(s * MT::NX) * S;
      XT* x1 = x0 + S;
      stage_row<4>(A, row, p0, NS, [&](int i, int64_t v) { MT::to_x(v, x0, x1, i); });
    }
    __syncthreads();

#pragma unroll 1
    for (int kk0 = 0; kk0 < KS; kk0 += G) {
      GT gv[G];
      lds_vec(gv, gs + kk0);
      const int base = tid * R - kk0 + KS - G;
#pragma unroll
      for (int s = 0; s < MS; ++s) {
        if (!EXTRACT && row0 + s >= A.rows) continue;
        const XT* x0 = xs + (size_t)(s * MT::NX) * S + base;
        XT w0[NW], w1[NW];
        lds_vec(w0, x0);
        if (MT::NX == 2) lds_vec(w1, x0 + S);
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int q = 0; q < G; ++q) MT::mac(acc[s][r], gv[q], w0[r - q + G - 1], w1[r - q + G - 1]);
      }
    }
  }

  const int64_t jend = A.y_begin + A.n_out;
  const int64_t jt = j0 + (int64_t)tid * R;
  if (!EXTRACT) {
    unsigned ovf = 0;
#pragma unroll
    for (int s = 0; s < MS; ++s) {
      const int row = row0 + s;
      if (row >= A.rows) continue;
      void* yp = A.y.p[row];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int64_t j = jt + r;
        if (j < jend) {
          st_bits(yp, A.y_bits, j - A.y_begin, MT::value(acc[s][r]));
          ovf += MT::fits(acc[s][r]) ? 0u : 1u;
        }
      }
    }
    if (A.mismatch && ovf) atomicAdd(A.mismatch, (unsigned long long)ovf);
  } else {
    const bool verify = A.r < 0;
    const int pivot = verify ? 0 : A.r;
    unsigned bad = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t j = jt + r;
      if (j >= jend) continue;
      int64_t dl[MS], orot[MS];
#pragma unroll
      for (int s = 0; s < MS; ++s) dl[s] = MT::value(acc[s][r]);
      recover_regs_valid<MS>(dl, pivot, A.l, orot);
      if (verify) {
        // delta_0 was not used by the recovery: it must equal (d_{m-1} << l) + d_0
        bad += (dl[0] != wadd(wshl(orot[MS - 1], A.l), orot[0])) ? 1u : 0u;
      }
#pragma unroll
      for (int t = 0; t < MS; ++t) {
        int row = pivot + t;
        row -= row >= MS ? MS : 0;
        st_bits(A.y.p[row], A.y_bits, j - A.y_begin, orot[t]);
      }
    }
    if (A.mismatch) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
      if ((tid & 31) == 0 && bad) atomicAdd(A.mismatch, (unsigned long long)bad);
    }
  }
}

template <int FLAV, int MS, bool EXTRACT>
static int launch_conv(ConvArgs A, cudaStream_t stream) {
  using MT = Mac<FLAV>;
  constexpr int R = pick_R(FLAV, MS);
  constexpr int T = CV_NT * R;
  const int xbytes = (int)sizeof(typename MT::XT) * MT::NX;
  const int budget = 72 * 1024;
  int kseg = ((budget / (MS * xbytes) - T - 8) / CV_G) * CV_G;
  if (kseg < CV_G) kseg = CV_G;
  if (kseg > A.Kp) kseg = A.Kp;
  A.kseg = kseg;
  A.sstride = (T + kseg + 4 + 3) & ~3;
  A.gbytes = (int)((kseg * sizeof(typename MT::GT) + 15) & ~(size_t)15);
  const size_t smem = (size_t)A.gbytes + (size_t)MS * MT::NX * A.sstride * sizeof(typename MT::XT);
  auto kern = conv_tile_kernel<FLAV, MS, EXTRACT>;
  if (ensure_smem((const void*)kern, smem) != NENT_OK) return NENT_ERR_CUDA;
  const int64_t tiles = (A.n_out + T - 1) / T;
  if (tiles > 0x7fffffffLL) {
    set_error("conv: too many tiles");
    return NENT_ERR_PARAM;
  }
  dim3 grid((unsigned)tiles, EXTRACT ? 1 : (unsigned)((A.rows + MS - 1) / MS));
  kern<<<grid, CV_NT, smem, stream>>>(A);
  note_conv_kernel(1);
  return check_launch("conv");
}

template <int FLAV>
static int conv_store_ms(ConvArgs& A, cudaStream_t s) {
  switch (A.rows) {
    case 1: return launch_conv<FLAV, 1, false>(A, s);
    case 2: return launch_conv<FLAV, 2, false>(A, s);
    case 3: return launch_conv<FLAV, 3, false>(A, s);
    default: return launch_conv<FLAV, 4, false>(A, s);
  }
}

static int conv_store(ConvArgs& A, int flavor, cudaStream_t s) {
  if ((flavor & 0xff) == NENT_MAC_IMMA) return imma_dispatch(A, flavor, false, s);
  switch (flavor) {
    case NENT_MAC_I32: return conv_store_ms<NENT_MAC_I32>(A, s);
    case NENT_MAC_W64: return conv_store_ms<NENT_MAC_W64>(A, s);
    case NENT_MAC_S64: return conv_store_ms<NENT_MAC_S64>(A, s);
    case NENT_MAC_F64: return conv_store_ms<NENT_MAC_F64>(A, s);
    case NENT_MAC_G64: return launch_conv<NENT_MAC_G64, 1, false>(A, s);
    case NENT_MAC_X128: return launch_conv<NENT_MAC_X128, 1, false>(A, s);
  }
  set_error("conv: unknown MAC flavour %d", flavor);
  return NENT_ERR_PARAM;
}

template <int FLAV>
static int conv_fused_m(ConvArgs& A, cudaStream_t s) {
  switch (A.rows) {
    case 3: return launch_conv<FLAV, 3, true>(A, s);
    case 4: return launch_conv<FLAV, 4, true>(A, s);
    case 5: return launch_conv<FLAV, 5, true>(A, s);
    case 6: return launch_conv<FLAV, 6, true>(A, s);
    case 7: return launch_conv<FLAV, 7, true>(A, s);
    case 8: return launch_conv<FLAV, 8, true>(A, s);
  }
  set_error("fused conv: m=%d not in 3..8 (use the unfused path)", A.rows);
  return NENT_ERR_PARAM;
}

static int check_conv_common(int in_bits, int g_bits, int y_bits, int K, int64_t n_in,
                             int64_t period, int64_t y_begin, int64_t n_out) {
  NENT_CHECK_BITS(in_bits);
  NENT_CHECK_BITS(g_bits);
  NENT_CHECK_BITS(y_bits);
  if (K < 1 || period < 1 || n_in < 0 || n_in > period || y_begin < 0 || n_out < 0 ||
      K > (1 << 28)) {
    set_error("conv: bad geometry K=%d n_in=%lld period=%lld", K, (long long)n_in,
              (long long)period);
    return NENT_ERR_PARAM;
  }
  return NENT_OK;
}

}  // namespace nent

using namespace nent;

extern "C" {

int nent_conv(const void* const* x, int x_bits, int rows, int64_t n_in, int64_t period,
              const void* g, int g_bits, int K, void* const* y, int y_bits, int64_t y_begin,
              int64_t n_out, int flavor, unsigned long long* overflow_dev, const void* imma_table,
              void* stream) {
  int st = check_conv_common(x_bits, g_bits, y_bits, K, n_in, period, y_begin, n_out);
  if (st) return st;
  if (rows < 1 || rows > NENT_MAX_STREAMS) {
    set_error("conv: rows=%d out of range", rows);
    return NENT_ERR_PARAM;
  }
  if (n_out == 0) return NENT_OK;
  ConvArgs A{};
  A.b = to_rows(x, rows);
  A.y = to_mrows(y, rows);
  A.rows = rows;
  A.in_bits = x_bits; A.y_bits = y_bits; A.g_bits = g_bits;
  A.K = K; A.Kp = (K + CV_G - 1) / CV_G * CV_G;
  A.n_in = n_in; A.period = period; A.y_begin = y_begin; A.n_out = n_out;
  A.scale = 1; A.g = g; A.r = 0; A.mismatch = overflow_dev; A.imma_table = imma_table;
  return conv_store(A, flavor, as_stream(stream));
}

int nent_chain_conv(const void* a, const void* b, int in_bits, int64_t n_in, int64_t period,
                    int l, int64_t scale, const void* add, int add_bits, const int64_t* perm,
                    const void* g, int g_bits, int K, void* y, int y_bits, int64_t y_begin,
                    int64_t n_out, int flavor, const void* imma_table, void* stream) {
  int st = check_conv_common(in_bits, g_bits, y_bits, K, n_in, period, y_begin, n_out);
  if (st) return st;
  if (add) NENT_CHECK_BITS(add_bits);
  if (n_out == 0) return NENT_OK;
  ConvArgs A{};
  A.a.p[0] = a;
  A.b.p[0] = b;
  A.y.p[0] = y;
  A.rows = 1;
  A.in_bits = in_bits; A.y_bits = y_bits; A.g_bits = g_bits; A.add_bits = add_bits;
  A.l = l; A.scale = scale; A.add = add; A.perm = perm;
  A.K = K; A.Kp = (K + CV_G - 1) / CV_G * CV_G;
  A.n_in = n_in; A.period = period; A.y_begin = y_begin; A.n_out = n_out;
  A.g = g; A.imma_table = imma_table;
  return conv_store(A, flavor, as_stream(stream));
}

int nent_fused_conv(const void* const* c, int c_bits, int m, int64_t n_in, int64_t period,
                    int l, int64_t scale, const void* add, int add_bits, const int64_t* perm,
                    const void* g, int g_bits, int K, int r, int pre_entangled, void* const* d,
                    int d_bits, int64_t y_begin, int64_t n_out, int flavor,
                    unsigned long long* mismatch_dev, const void* imma_table, void* stream) {
  int st = check_conv_common(c_bits, g_bits, d_bits, K, n_in, period, y_begin, n_out);
  if (st) return st;
  if (add) NENT_CHECK_BITS(add_bits);
  if (m < 3 || m > 8 || r < -1 || r >= m || l < 1 || (m - 1) * l > 63) {
    set_error("fused conv: bad geometry m=%d l=%d r=%d", m, l, r);
    return NENT_ERR_PARAM;
  }
  if (n_out == 0) return NENT_OK;
  ConvArgs A{};
  for (int i = 0; i < m; ++i) {
    A.a.p[i] = pre_entangled ? nullptr : c[(i + m - 1) % m];
    A.b.p[i] = c[i];
    A.y.p[i] = d[i];
  }
  A.rows = m;
  A.in_bits = c_bits; A.y_bits = d_bits; A.g_bits = g_bits; A.add_bits = add_bits;
  A.l = l; A.scale = scale; A.add = add; A.perm = perm;
  A.K = K; A.Kp = (K + CV_G - 1) / CV_G * CV_G;
  A.n_in = n_in; A.period = period; A.y_begin = y_begin; A.n_out = n_out;
  A.g = g; A.r = r; A.wide = pre_entangled; A.mismatch = mismatch_dev; A.imma_table = imma_table;
  cudaStream_t s = as_stream(stream);
  if ((flavor & 0xff) == NENT_MAC_IMMA) return imma_dispatch(A, flavor, true, s);
  switch (flavor) {
    case NENT_MAC_I32: return conv_fused_m<NENT_MAC_I32>(A, s);
    case NENT_MAC_W64: return conv_fused_m<NENT_MAC_W64>(A, s);
    case NENT_MAC_S64: return conv_fused_m<NENT_MAC_S64>(A, s);
    case NENT_MAC_F64: return conv_fused_m<NENT_MAC_F64>(A, s);
  }
  set_error("fused conv: unsupported MAC flavour %d", flavor);
  return NENT_ERR_PARAM;
}

}  // extern "C"
