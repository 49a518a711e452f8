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

struct ConvArgs {
  Rows a;        // optional shifted operand rows: x = (a << l) + b
  Rows b;        // main operand rows
  MutRows y;     // output rows (delta rows, or the m recovered rows when fused)
  int rows;      // streams (== m when fused)
  int in_bits, y_bits, g_bits, add_bits;
  int l;
  int K, Kp, kseg, sstride, gbytes;
  int r, wide;
  int64_t n_in, period, y_begin, n_out;
  int64_t scale;
  const void* add;
  const int64_t* perm;
  const void* g;
  unsigned long long* mismatch;
};

// x_row[p] after the on-load chain: entangle, scale, add, gather, zero-pad.
__device__ __forceinline__ int64_t conv_prologue(const ConvArgs& A, int row, int64_t p) {
  int64_t q = p;
  if (q < 0 || q >= A.period) {
    q %= A.period;
    if (q < 0) q += A.period;
  }
  if (q >= A.n_in) return 0;
  if (A.perm) q = __ldg(A.perm + q);
  int64_t e = ld_bits(A.b.p[row], A.in_bits, q);
  const void* ap = A.a.p[row];
  if (ap) e = wadd(wshl(ld_bits(ap, A.in_bits, q), A.l), e);
  if (A.scale != 1) e = wmul(e, A.scale);
  if (A.add) e = wadd(e, ld_bits(A.add, A.add_bits, q));
  return e;
}

// ============================================================================
// IMMA digit-sliced exact convolution (tensor cores, mma.sync s8*s8+s32).
//
// Every operand is split into balanced base-256 digits (int8 in [-128,127]):
//   x = sum_p 256^p x_p  (NP planes),   g = sum_j 256^j g_j  (NG digits)
//   y = sum_{p,j} 256^(p+j) (x_p (*) g_j)          (mod 2^64: exact whenever
//                                                   y fits int64)
// Each digit convolution is an int8 GEMM with int32 accumulation (exact:
// |partial| <= 2^14 * KD < 2^31 for KD < 2^17).  The GEMM is Toeplitz:
//   Y[a, b] = sum_t A[a, t] B[t, b],  output j0 + 16a + b (b in [0,16))
//   A[a, t] = x_p[j0 + 16a + t - (K-1)]   (Hankel: row a is the signal shifted
//                                          by 16 bytes, i.e. one smem row)
//   B[t, b] = g_j[b + K - 1 - t]          (the taps, built once per CTA)
// Because consecutive Hankel rows are exactly 16 bytes apart, ldmatrix reads
// A fragments straight from the digit plane in shared memory (8 rows x 16 B
// = 128 contiguous bytes per 8x8 matrix: conflict-free) -- the Hankel matrix
// is never materialised.  B fragments stay in registers for a K-segment.
// Warp w owns RT row-tiles of 16 rows (256 outputs each); per (plane, kc) it
// issues one ldmatrix.x4 and 2*NG MMAs per row-tile.  After each plane the
// int32 accumulators are folded into int64 (shift by 8(p+j)); the per-stream
// int64 results meet in shared memory, where the epilogue stores them or runs
// the m-stream recovery (fused entangle -> conv -> extract).
// ============================================================================

constexpr int IM_WARPS = 4;
constexpr int IM_NT = IM_WARPS * 32;

__host__ __device__ constexpr int imma_rt(int ms) { return ms <= 4 ? 2 : 1; }
__host__ __device__ constexpr int imma_seg(int ng) { return ng == 1 ? 18 : ng == 2 ? 9 : ng == 3 ? 6 : 4; }

struct ImmaGeom {
  int KD;    // K-dimension of the Toeplitz GEMM (multiple of 32)
  int NKC;   // KD / 32
  int KDs;   // Bt row stride in bytes (== 16 mod 128: conflict-free ldmatrix)
  int S;     // bytes per digit plane (multiple of 16)
  int np;    // digit planes of x
  int bt_off, pl_off, dt_off;  // smem offsets
  size_t smem;
};

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}

__device__ __forceinline__ void imma16832(int (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// balanced base-256 digit p of v (v = sum_p 256^p digit_p, digits in [-128,127])
__device__ __forceinline__ uint32_t digit_byte(int64_t& rest) {
  const int64_t d = (int64_t)(int8_t)(uint8_t)(uint64_t)rest;
  rest = (int64_t)((uint64_t)rest - (uint64_t)d) >> 8;
  return (uint32_t)(uint8_t)d;
}

template <int MS, int NG, bool EXTRACT>
__global__ void __launch_bounds__(IM_NT, 1)
    conv_imma_kernel(const __grid_constant__ ConvArgs A, const ImmaGeom Gm) {
  constexpr int RT = imma_rt(MS);
  constexpr int SEG = imma_seg(NG);
  constexpr int T = IM_WARPS * RT * 256;  // outputs per CTA tile
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned char* bt = smem + Gm.bt_off;   // NG x 16 rows x KDs
  unsigned char* pl = smem + Gm.pl_off;   // MS x np planes x S bytes
  int64_t* dt = reinterpret_cast<int64_t*>(smem + Gm.dt_off);  // MS x T
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t j0 = A.y_begin + (int64_t)blockIdx.x * T;
  const int row0 = EXTRACT ? 0 : (int)blockIdx.y * MS;
  const int np = Gm.np, KD = Gm.KD, KDs = Gm.KDs, S = Gm.S;

  // ---- Bt_j[b][t] = digit_j(g[b + K - 1 - t]) ----
  for (int i = tid; i < 16 * KD; i += IM_NT) {
    const int b = i / KD, t = i - b * KD;
    const int k = b + A.K - 1 - t;
    int64_t rest = (k >= 0 && k < A.K) ? ld_bits(A.g, A.g_bits, k) : 0;
#pragma unroll
    for (int j = 0; j < NG; ++j) bt[(j * 16 + b) * KDs + t] = (unsigned char)digit_byte(rest);
  }
  // ---- digit planes: smem byte i <-> input position j0 - (K-1) + i ----
  const int64_t p0 = j0 - (A.K - 1);
  for (int s = 0; s < MS; ++s) {
    const int row = row0 + s;
    unsigned char* ps = pl + (size_t)s * np * S;
    for (int i = tid; i < S; i += IM_NT) {
      int64_t rest = row < A.rows ? conv_prologue(A, row, p0 + i) : 0;
      for (int p = 0; p < np; ++p) ps[(size_t)p * S + i] = (unsigned char)digit_byte(rest);
    }
  }
  __syncthreads();

  const uint32_t pl_s = (uint32_t)__cvta_generic_to_shared(pl);
  const uint32_t bt_s = (uint32_t)__cvta_generic_to_shared(bt);
  const int mat = lane >> 3, r8 = lane & 7;
  // per-lane ldmatrix row offsets
  const uint32_t a_lane = 16u * (uint32_t)(r8 + 8 * (mat & 1)) + 16u * (uint32_t)(mat >> 1);
  const uint32_t b_lane = (uint32_t)((8 * (mat >> 1) + r8) * KDs + 16 * (mat & 1));
  const int g = lane >> 2, t4 = lane & 3;

  for (int s = 0; s < MS; ++s) {
    if (!EXTRACT && row0 + s >= A.rows) break;
    long long acc[RT][2][4];
#pragma unroll
    for (int rt = 0; rt < RT; ++rt)
#pragma unroll
      for (int nb = 0; nb < 2; ++nb)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[rt][nb][q] = 0;

    for (int kc0 = 0; kc0 < Gm.NKC; kc0 += SEG) {
      uint32_t bf[SEG][NG][4];  // per kc: {b0,b1} of n8-tile 0, {b0,b1} of n8-tile 1
#pragma unroll
      for (int kk = 0; kk < SEG; ++kk)
#pragma unroll
        for (int j = 0; j < NG; ++j)
          if (kc0 + kk < Gm.NKC)
            ldsm_x4(bf[kk][j], bt_s + (uint32_t)(j * 16 * KDs) + b_lane + 32u * (uint32_t)(kc0 + kk));
      for (int p = 0; p < np; ++p) {
        const uint32_t plane = pl_s + (uint32_t)((s * np + p) * S);
        int c[RT][2][NG][4];
#pragma unroll
        for (int rt = 0; rt < RT; ++rt)
#pragma unroll
          for (int nb = 0; nb < 2; ++nb)
#pragma unroll
            for (int j = 0; j < NG; ++j)
#pragma unroll
              for (int q = 0; q < 4; ++q) c[rt][nb][j][q] = 0;
#pragma unroll
        for (int kk = 0; kk < SEG; ++kk) {
          if (kc0 + kk >= Gm.NKC) break;
#pragma unroll
          for (int rt = 0; rt < RT; ++rt) {
            uint32_t af[4];
            ldsm_x4(af, plane + 256u * (uint32_t)(warp * RT + rt) + a_lane + 32u * (uint32_t)(kc0 + kk));
#pragma unroll
            for (int j = 0; j < NG; ++j) {
              imma16832(c[rt][0][j], af, bf[kk][j][0], bf[kk][j][1]);
              imma16832(c[rt][1][j], af, bf[kk][j][2], bf[kk][j][3]);
            }
          }
        }
        // fold the int32 digit products into the int64 accumulators
#pragma unroll
        for (int rt = 0; rt < RT; ++rt)
#pragma unroll
          for (int nb = 0; nb < 2; ++nb)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              uint64_t v = 0;
#pragma unroll
              for (int j = 0; j < NG; ++j) v += (uint64_t)(int64_t)c[rt][nb][j][q] << (8 * j);
              acc[rt][nb][q] = (long long)((uint64_t)acc[rt][nb][q] + (v << (8 * p)));
            }
      }
    }
    // stage this stream's results: C fragment (row g|g+8, col 2t|2t+1) of n8-tile nb
#pragma unroll
    for (int rt = 0; rt < RT; ++rt)
#pragma unroll
      for (int nb = 0; nb < 2; ++nb)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int u = 256 * (warp * RT + rt) + 16 * (g + 8 * (q >> 1)) + 8 * nb + 2 * t4 + (q & 1);
          dt[(size_t)s * T + u] = acc[rt][nb][q];
        }
  }
  __syncthreads();

  // ---- epilogue: coalesced stores or the fused m-stream recovery ----
  const int64_t jend = A.y_begin + A.n_out;
  if (!EXTRACT) {
    for (int s = 0; s < MS; ++s) {
      const int row = row0 + s;
      if (row >= A.rows) break;
      for (int u = tid; u < T; u += IM_NT) {
        const int64_t j = j0 + u;
        if (j < jend) st_bits(A.y.p[row], A.y_bits, j - A.y_begin, dt[(size_t)s * T + u]);
      }
    }
  } else {
    const bool verify = A.r < 0;
    const int pivot = verify ? 0 : A.r;
    unsigned bad = 0;
    for (int u = tid; u < T; u += IM_NT) {
      const int64_t j = j0 + u;
      if (j >= jend) break;
      int64_t dl[MS], orot[MS];
#pragma unroll
      for (int s = 0; s < MS; ++s) dl[s] = dt[(size_t)s * T + u];
      recover_regs_valid<MS>(dl, pivot, A.l, orot);
      if (verify) bad += (dl[0] != wadd(wshl(orot[MS - 1], A.l), orot[0])) ? 1u : 0u;
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
      if (lane == 0 && bad) atomicAdd(A.mismatch, (unsigned long long)bad);
    }
  }
}

template <int MS, int NG, bool EXTRACT>
static int launch_imma(ConvArgs A, int np, cudaStream_t stream) {
  constexpr int T = IM_WARPS * imma_rt(MS) * 256;
  ImmaGeom Gm{};
  Gm.np = np;
  Gm.KD = (A.K + 15 + 31) / 32 * 32;
  Gm.NKC = Gm.KD / 32;
  Gm.KDs = (Gm.KD + 127) / 128 * 128 + 16;
  Gm.S = (T + Gm.KD + 15) / 16 * 16;
  Gm.bt_off = 0;
  Gm.pl_off = (NG * 16 * Gm.KDs + 127) / 128 * 128;
  Gm.dt_off = (Gm.pl_off + MS * np * Gm.S + 127) / 128 * 128;
  Gm.smem = (size_t)Gm.dt_off + (size_t)MS * T * 8;
  if (Gm.smem > 227 * 1024) {
    set_error("imma conv: tile needs %zu bytes of shared memory (K=%d too long)", Gm.smem, A.K);
    return NENT_ERR_PARAM;
  }
  auto kern = conv_imma_kernel<MS, NG, EXTRACT>;
  static size_t configured = 0;
  if (Gm.smem > configured) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Gm.smem) !=
        cudaSuccess) {
      set_error("imma conv: cannot reserve %zu bytes of shared memory", Gm.smem);
      return NENT_ERR_CUDA;
    }
    configured = Gm.smem;
  }
  const int64_t tiles = (A.n_out + T - 1) / T;
  dim3 grid((unsigned)tiles, EXTRACT ? 1 : (unsigned)((A.rows + MS - 1) / MS));
  kern<<<grid, IM_NT, Gm.smem, stream>>>(A, Gm);
  return check_launch("imma conv");
}

template <int NG>
static int imma_dispatch_ng(ConvArgs& A, int np, bool extract, cudaStream_t s) {
  if (extract) {
    switch (A.rows) {
      case 3: return launch_imma<3, NG, true>(A, np, s);
      case 4: return launch_imma<4, NG, true>(A, np, s);
      case 5: return launch_imma<5, NG, true>(A, np, s);
      case 6: return launch_imma<6, NG, true>(A, np, s);
      case 7: return launch_imma<7, NG, true>(A, np, s);
      case 8: return launch_imma<8, NG, true>(A, np, s);
    }
    set_error("imma fused conv: m=%d not in 3..8", A.rows);
    return NENT_ERR_PARAM;
  }
  switch (A.rows) {
    case 1: return launch_imma<1, NG, false>(A, np, s);
    case 2: return launch_imma<2, NG, false>(A, np, s);
    case 3: return launch_imma<3, NG, false>(A, np, s);
    default: return launch_imma<4, NG, false>(A, np, s);
  }
}

// flavor word: NENT_MAC_IMMA | np << 8 | ng << 12
static int imma_dispatch(ConvArgs& A, int flavor, bool extract, cudaStream_t s) {
  const int np = (flavor >> 8) & 0xf, ng = (flavor >> 12) & 0xf;
  if (np < 1 || np > 8 || ng < 1 || ng > 4) {
    set_error("imma conv: digit counts np=%d ng=%d outside 1..8 / 1..4", np, ng);
    return NENT_ERR_PARAM;
  }
  if (A.K + 15 > (1 << 16)) {
    set_error("imma conv: K=%d too long for int32 digit sums", A.K);
    return NENT_ERR_PARAM;
  }
  switch (ng) {
    case 1: return imma_dispatch_ng<1>(A, np, extract, s);
    case 2: return imma_dispatch_ng<2>(A, np, extract, s);
    case 3: return imma_dispatch_ng<3>(A, np, extract, s);
    default: return imma_dispatch_ng<4>(A, np, extract, s);
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
      if (row < A.rows) {
        for (int i = tid; i < NS; i += CV_NT) MT::to_x(conv_prologue(A, row, p0 + i), x0, x1, i);
      } else {
        for (int i = tid; i < NS; i += CV_NT) MT::to_x(0, x0, x1, i);
      }
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
  static size_t configured = 0;
  if (smem > configured) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess) {
      set_error("conv: cannot reserve %zu bytes of shared memory", smem);
      return NENT_ERR_CUDA;
    }
    configured = smem;
  }
  const int64_t tiles = (A.n_out + T - 1) / T;
  if (tiles > 0x7fffffffLL) {
    set_error("conv: too many tiles");
    return NENT_ERR_PARAM;
  }
  dim3 grid((unsigned)tiles, EXTRACT ? 1 : (unsigned)((A.rows + MS - 1) / MS));
  kern<<<grid, CV_NT, smem, stream>>>(A);
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
              int64_t n_out, int flavor, unsigned long long* overflow_dev, void* stream) {
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
  A.scale = 1; A.g = g; A.r = 0; A.mismatch = overflow_dev;
  return conv_store(A, flavor, as_stream(stream));
}

int nent_chain_conv(const void* a, const void* b, int in_bits, int64_t n_in, int64_t period,
                    int l, int64_t scale, const void* add, int add_bits, const int64_t* perm,
                    const void* g, int g_bits, int K, void* y, int y_bits, int64_t y_begin,
                    int64_t n_out, int flavor, void* stream) {
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
  A.g = g;
  return conv_store(A, flavor, as_stream(stream));
}

int nent_fused_conv(const void* const* c, int c_bits, int m, int64_t n_in, int64_t period,
                    int l, int64_t scale, const void* add, int add_bits, const int64_t* perm,
                    const void* g, int g_bits, int K, int r, int wide, void* const* d,
                    int d_bits, int64_t y_begin, int64_t n_out, int flavor,
                    unsigned long long* mismatch_dev, void* stream) {
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
    A.a.p[i] = c[(i + m - 1) % m];
    A.b.p[i] = c[i];
    A.y.p[i] = d[i];
  }
  A.rows = m;
  A.in_bits = c_bits; A.y_bits = d_bits; A.g_bits = g_bits; A.add_bits = add_bits;
  A.l = l; A.scale = scale; A.add = add; A.perm = perm;
  A.K = K; A.Kp = (K + CV_G - 1) / CV_G * CV_G;
  A.n_in = n_in; A.period = period; A.y_begin = y_begin; A.n_out = n_out;
  A.g = g; A.r = r; A.wide = wide; A.mismatch = mismatch_dev;
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
