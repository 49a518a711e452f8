// conv_imma.cu -- exact integer convolution on the tensor cores by digit
// slicing (mma.sync m16n8k32 s8 -> s32), plain or fused with entangle/extract.
// Reference semantics: ops._circ_conv_rows (/root/reference/pkg/src/nent/ops.py:158-172).
//
// Every operand is split into balanced base-256 digits (int8 in [-128,127]):
//   x = sum_p 256^p x_p  (np planes),   g = sum_j 256^j g_j  (NG digits)
//   y = sum_{p,j} 256^(p+j) (x_p (*) g_j)     (mod 2^64: exact whenever y fits int64)
// Each digit convolution is an int8 GEMM with int32 accumulation, exact for a
// K-segment of SEG*32 taps (|partial| <= 2^14 * 288 < 2^31).  The GEMM is
// Toeplitz:
//   Y[a, b] = sum_t A[a, t] B[t, b],    output j0 + 16a + b, b in [0,16)
//   A[a, t] = x_p[j0 + 16a + t - (Keff-1)]   Hankel: row a+1 is row a shifted by
//                                           16 bytes -- one shared-memory row
//   B[t, b] = g_j[b + Keff - 1 - t]          the taps (a prepared table)
// ldmatrix reads A fragments straight out of the digit plane (8 rows x 16 B =
// 128 contiguous bytes per 8x8 matrix: conflict-free), so the Hankel matrix is
// never materialised.
//
// Pipeline per CTA (1024 outputs of MS streams, 4 warps, 4 CTAs per SM so the
// phases of different CTAs overlap on the SM's pipes):
//   1. raw int32 tiles land in shared memory by TMA bulk copy (cp.async.bulk),
//      entangle + digit split run from shared memory (bias trick + PRMT);
//   2. per K-segment the digit-split Toeplitz table is bulk-copied from a
//      table prepared once per launch; each warp issues, per (plane, k-step),
//      one ldmatrix for A, NG for B and 2*NG IMMAs into int32 accumulators,
//      folded into int64 after every plane;
//   3. per-stream int64 results meet in shared memory; the epilogue stores
//      them (plain conv) or recovers all m streams from the m-1 survivors
//      (fused entangle -> conv -> extract) and writes them coalesced.
#include "common.cuh"
#include "conv_common.cuh"
#include "recover.cuh"

#include <type_traits>

namespace nent {

constexpr int IM_WARPS = 4;
constexpr int IM_NT = IM_WARPS * 32;
constexpr int IM_T = IM_WARPS * 256;  // outputs per CTA tile (one 16x16 row-tile per warp)
constexpr int IM_SEG = 9;             // k-steps (32 taps each) per K-segment
constexpr int IM_KDS = IM_SEG * 32 + 16;  // table row stride: 304 == 48 mod 128 (conflict-free)

struct ImmaGeom {
  int Keff;   // K + zero taps so that every tile's first staged position is 4-aligned
  int KD;     // K-dimension of the Toeplitz GEMM (multiple of 32)
  int NKC;    // KD / 32
  int NSEG;   // ceil(NKC / IM_SEG)
  int S;      // bytes per digit plane (multiple of 16)
  int np;     // digit planes of x
  int bt_off, pl_off, dt_off;  // smem offsets
  size_t smem;
  const unsigned char* table;  // [NSEG][NG][16][IM_KDS] digit-split Toeplitz taps
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

// Balanced base-256 digits without a carry chain: with u = v + sum_p 128*256^p
// (mod 2^64), u's bytes are d_p + 128 in [0, 255], so the int8 digit d_p is
// byte p of (u XOR 0x8080...80).  One 64-bit add + xor yields all 8 digits.
__device__ __forceinline__ uint64_t digit_word(int64_t v, uint64_t bias) {
  return ((uint64_t)v + bias) ^ 0x8080808080808080ull;
}
__host__ __device__ constexpr uint64_t digit_bias(int np) {
  return np >= 8 ? 0x8080808080808080ull : (0x8080808080808080ull & ((1ull << (8 * np)) - 1));
}
// byte p of each of 4 words, packed little-endian into one word
__device__ __forceinline__ uint32_t gather_byte(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3,
                                                int p) {
  const uint32_t sel = (uint32_t)p | ((uint32_t)(p + 4) << 4);
  return __byte_perm(__byte_perm(w0, w1, sel), __byte_perm(w2, w3, sel), 0x5410);
}

// write the np digit planes of 4 consecutive values into word w of each plane
__device__ __forceinline__ void put_digits(uint32_t* ps, int S4, int w, int np, const int64_t (&v)[4],
                                           uint64_t bias) {
  uint64_t u[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) u[e] = digit_word(v[e], bias);
  const uint32_t l0 = (uint32_t)u[0], l1 = (uint32_t)u[1], l2 = (uint32_t)u[2], l3 = (uint32_t)u[3];
  const uint32_t h0 = (uint32_t)(u[0] >> 32), h1 = (uint32_t)(u[1] >> 32), h2 = (uint32_t)(u[2] >> 32),
                 h3 = (uint32_t)(u[3] >> 32);
  // jump into a straight-line tail: exactly np byte-gathers and stores
  switch (np) {
    case 8: ps[7 * S4 + w] = gather_byte(h0, h1, h2, h3, 3);  // fall through
    case 7: ps[6 * S4 + w] = gather_byte(h0, h1, h2, h3, 2);  // fall through
    case 6: ps[5 * S4 + w] = gather_byte(h0, h1, h2, h3, 1);  // fall through
    case 5: ps[4 * S4 + w] = gather_byte(h0, h1, h2, h3, 0);  // fall through
    case 4: ps[3 * S4 + w] = gather_byte(l0, l1, l2, l3, 3);  // fall through
    case 3: ps[2 * S4 + w] = gather_byte(l0, l1, l2, l3, 2);  // fall through
    case 2: ps[1 * S4 + w] = gather_byte(l0, l1, l2, l3, 1);  // fall through
    default: ps[w] = gather_byte(l0, l1, l2, l3, 0);
  }
}

__device__ __forceinline__ void mbar_init(uint32_t mb) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t mb, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mb) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(mb) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t mb, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(mb), "r"(phase) : "memory");
}

// Toeplitz tap table, once per launch: table[seg][j][b][tl] = digit_j(g[b + Keff - 1 - t]),
// t = 32*IM_SEG*seg + tl (0 outside the taps and in the row padding).
__global__ void imma_table_kernel(const void* g, int g_bits, int K, int Keff, int KD, int NG,
                                  int nseg, unsigned char* table) {
  const int total = nseg * NG * 16 * IM_KDS;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int tl = i % IM_KDS, b = (i / IM_KDS) % 16, j = (i / (IM_KDS * 16)) % NG,
              seg = i / (IM_KDS * 16 * NG);
    const int t = seg * IM_SEG * 32 + tl;
    const int k = b + Keff - 1 - t;
    int64_t gv = 0;
    if (tl < IM_SEG * 32 && t < KD && k >= 0 && k < K) gv = ld_bits(g, g_bits, k);
    table[i] = (unsigned char)(digit_word(gv, digit_bias(NG)) >> (8 * j));
  }
}

template <int MS, int NG, bool EXTRACT>
__global__ void __launch_bounds__(IM_NT, 4)
    conv_imma_kernel(const __grid_constant__ ConvArgs A, const __grid_constant__ ImmaGeom Gm) {
  constexpr int T = IM_T;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t mbar[2];  // [0] raw tiles, [1] tap table
  unsigned char* bt = smem + Gm.bt_off;                         // NG x 16 x IM_KDS
  unsigned char* pl = smem + Gm.pl_off;                         // MS x np x S
  int64_t* dt = reinterpret_cast<int64_t*>(smem + Gm.dt_off);  // MS x T (raw tiles alias it)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t j0 = A.y_begin + (int64_t)blockIdx.x * T;
  const int row0 = EXTRACT ? 0 : (int)blockIdx.y * MS;
  const int np = Gm.np, S = Gm.S, S4 = S >> 2;
  const uint32_t mb_raw = (uint32_t)__cvta_generic_to_shared(&mbar[0]);
  const uint32_t mb_tab = (uint32_t)__cvta_generic_to_shared(&mbar[1]);
  const uint32_t bt_s = (uint32_t)__cvta_generic_to_shared(bt);
  const uint32_t tab_bytes = (uint32_t)(NG * 16 * IM_KDS);

  // ---- 1. stage: smem byte i of a plane <-> input position p0 + i ----
  const int64_t p0 = j0 - (Gm.Keff - 1);
  const uint64_t xbias = digit_bias(np);
  // Raw rows arrive by TMA from the 16-byte-aligned word at or below p0, so a
  // row base that is only 4-byte aligned (a sliced or halo-prefixed buffer)
  // still takes the bulk-copy path; mis[s] words of lead-in are skipped.
  const int RS = S + 4;
  int mis[MS];
  bool fast = A.in_bits == 32 && !A.perm && A.scale == 1 && !A.add;
#pragma unroll
  for (int s = 0; s < MS; ++s) {
    const int row = row0 + s;
    mis[s] = 0;
    if (row < A.rows) {
      const uintptr_t q = reinterpret_cast<uintptr_t>(reinterpret_cast<const int32_t*>(A.b.p[row]) + p0);
      mis[s] = (int)((q & 15) >> 2);
      fast = fast && (q & 3) == 0 && p0 - mis[s] >= 0 && p0 - mis[s] + S + (mis[s] ? 4 : 0) <= A.n_in;
    } else {
      fast = false;
    }
    fast = fast && (EXTRACT || !A.a.p[row]);
  }
  if (tid == 0) {
    mbar_init(mb_raw);
    mbar_init(mb_tab);
  }
  __syncthreads();
  if (tid == 0) {  // the first segment's taps travel while the tile is staged
    mbar_expect(mb_tab, tab_bytes);
    bulk_g2s(bt_s, Gm.table, tab_bytes, mb_tab);
  }
  if (fast) {
    int32_t* raw = reinterpret_cast<int32_t*>(dt);
    if (tid == 0) {
      uint32_t total = 0;
#pragma unroll
      for (int s = 0; s < MS; ++s) total += (uint32_t)(S + (mis[s] ? 4 : 0)) * 4u;
      mbar_expect(mb_raw, total);
#pragma unroll
      for (int s = 0; s < MS; ++s)
        bulk_g2s((uint32_t)__cvta_generic_to_shared(raw + (size_t)s * RS),
                 reinterpret_cast<const int32_t*>(A.b.p[row0 + s]) + p0 - mis[s],
                 (uint32_t)(S + (mis[s] ? 4 : 0)) * 4u, mb_raw);
    }
    mbar_wait(mb_raw, 0);
    auto word4 = [&](int s, int w) -> int4 {
      if (mis[s] == 0) return reinterpret_cast<const int4*>(raw + (size_t)s * RS)[w];
      const int32_t* r = raw + (size_t)s * RS + mis[s] + 4 * w;
      return make_int4(r[0], r[1], r[2], r[3]);
    };
    for (int w = tid; w < S4; w += IM_NT) {
#pragma unroll
      for (int s = 0; s < MS; ++s) {
        const int4 bv = word4(s, w);
        int64_t v[4] = {bv.x, bv.y, bv.z, bv.w};
        if (EXTRACT && A.a.p[row0 + s]) {  // eps_s = (c_{s-1} << l) + c_s, both tiles in smem
          const int4 av = word4((s + MS - 1) % MS, w);
          v[0] = wadd(wshl(av.x, A.l), v[0]); v[1] = wadd(wshl(av.y, A.l), v[1]);
          v[2] = wadd(wshl(av.z, A.l), v[2]); v[3] = wadd(wshl(av.w, A.l), v[3]);
        }
        put_digits(reinterpret_cast<uint32_t*>(pl + (size_t)s * np * S), S4, w, np, v, xbias);
      }
    }
  } else {
    for (int s = 0; s < MS; ++s) {
      const int row = row0 + s;
      const bool live = row < A.rows;
      for (int w = tid; w < S4; w += IM_NT) {
        int64_t v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = live ? conv_prologue(A, row, p0 + 4 * w + e) : 0;
        put_digits(reinterpret_cast<uint32_t*>(pl + (size_t)s * np * S), S4, w, np, v, xbias);
      }
    }
  }

  // ---- 2. MMAs ----
  const uint32_t pl_s = (uint32_t)__cvta_generic_to_shared(pl);
  const int mat = lane >> 3, r8 = lane & 7;
  const uint32_t a_lane = 256u * (uint32_t)warp + 16u * (uint32_t)(r8 + 8 * (mat & 1)) + 16u * (uint32_t)(mat >> 1);
  const uint32_t b_lane = (uint32_t)((8 * (mat >> 1) + r8) * IM_KDS + 16 * (mat & 1));
  const int g = lane >> 2, t4 = lane & 3;
  // combining the g digits in int32 is exact when 2^14 * 288 * (1 + 256) < 2^31
  constexpr bool FOLD32 = NG <= 2;

  for (int seg = 0; seg < Gm.NSEG; ++seg) {
    const int kc0 = seg * IM_SEG;
    const int nkc = min(IM_SEG, Gm.NKC - kc0);
    if (seg > 0) {
      __syncthreads();  // every warp is done with the previous segment's table
      if (tid == 0) {
        mbar_expect(mb_tab, tab_bytes);
        bulk_g2s(bt_s, Gm.table + (size_t)seg * tab_bytes, tab_bytes, mb_tab);
      }
    } else {
      __syncthreads();  // digit planes complete
    }
    mbar_wait(mb_tab, (uint32_t)(seg & 1));

    for (int s = 0; s < MS; ++s) {
      if (!EXTRACT && row0 + s >= A.rows) break;
      long long acc[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
      // planes two at a time: each B fragment load feeds both planes' MMAs
      auto planes = [&](int p, auto PAIR) {
        constexpr int NPL = decltype(PAIR)::value ? 2 : 1;
        const uint32_t plane = pl_s + (uint32_t)((s * np + p) * S) + 32u * (uint32_t)kc0 + a_lane;
        int c[NPL][2][NG][4];
#pragma unroll
        for (int h = 0; h < NPL; ++h)
#pragma unroll
          for (int nb = 0; nb < 2; ++nb)
#pragma unroll
            for (int j = 0; j < NG; ++j)
#pragma unroll
              for (int q = 0; q < 4; ++q) c[h][nb][j][q] = 0;
        auto kstep = [&](int kk) {
          uint32_t af[NPL][4];
#pragma unroll
          for (int h = 0; h < NPL; ++h) ldsm_x4(af[h], plane + (uint32_t)(h * S) + 32u * (uint32_t)kk);
#pragma unroll
          for (int j = 0; j < NG; ++j) {
            uint32_t bf[4];  // {b0,b1} of n8-tile 0, {b0,b1} of n8-tile 1
            ldsm_x4(bf, bt_s + (uint32_t)(j * 16 * IM_KDS) + b_lane + 32u * (uint32_t)kk);
#pragma unroll
            for (int h = 0; h < NPL; ++h) {
              imma16832(c[h][0][j], af[h], bf[0], bf[1]);
              imma16832(c[h][1][j], af[h], bf[2], bf[3]);
            }
          }
        };
        if (nkc == IM_SEG) {
#pragma unroll
          for (int kk = 0; kk < IM_SEG; ++kk) kstep(kk);
        } else {
#pragma unroll
          for (int kk = 0; kk < IM_SEG; ++kk) {
            if (kk >= nkc) break;
            kstep(kk);
          }
        }
        // fold the digit products into int64: += (sum_j c_j 256^j) << 8(p+h)
#pragma unroll
        for (int h = 0; h < NPL; ++h)
#pragma unroll
          for (int nb = 0; nb < 2; ++nb)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              uint64_t v;
              if (FOLD32) {
                int32_t v32 = c[h][nb][0][q];
                if (NG == 2) v32 += c[h][nb][NG - 1][q] << 8;
                v = (uint64_t)(int64_t)v32;
              } else {
                v = 0;
#pragma unroll
                for (int j = 0; j < NG; ++j) v += (uint64_t)(int64_t)c[h][nb][j][q] << (8 * j);
              }
              acc[nb][q] = (long long)((uint64_t)acc[nb][q] + (v << (8 * (p + h))));
            }
      };
      int p = 0;
      for (; p + 1 < np; p += 2) planes(p, std::true_type{});
      if (p < np) planes(p, std::false_type{});
      // this segment's contribution; C fragment (row g|g+8, col 2t|2t+1) of n8-tile nb
#pragma unroll
      for (int nb = 0; nb < 2; ++nb)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int u = 256 * warp + 16 * (g + 8 * (q >> 1)) + 8 * nb + 2 * t4 + (q & 1);
          int64_t* d = dt + (size_t)s * T + u;
          *d = seg == 0 ? acc[nb][q] : wadd(*d, acc[nb][q]);
        }
    }
  }
  __syncthreads();

  // ---- 3. epilogue: coalesced stores or the fused m-stream recovery ----
  const int64_t jend = A.y_begin + A.n_out;
  const int64_t ybase = j0 - A.y_begin;
  const int64_t ulim = jend - j0 < T ? jend - j0 : T;
  if (!EXTRACT) {
    for (int s = 0; s < MS; ++s) {
      const int row = row0 + s;
      if (row >= A.rows) break;
      void* yp = A.y.p[row];
      for (int u = tid; u < ulim; u += IM_NT) st_bits(yp, A.y_bits, ybase + u, dt[(size_t)s * T + u]);
    }
  } else {
    const bool verify = A.r < 0;
    const int pivot = verify ? 0 : A.r;
    // rotation hoisted out of the position loop: rotated smem rows in, rotated
    // output rows out (drow[MS-1] is the pivot stream, read only to verify)
    const int64_t* drow[MS];
    void* yrow[MS];
#pragma unroll
    for (int t = 0; t < MS; ++t) {
      int in = pivot + 1 + t, out = pivot + t;
      in -= in >= MS ? MS : 0;
      in -= in >= MS ? MS : 0;
      out -= out >= MS ? MS : 0;
      drow[t] = dt + (size_t)in * T;
      yrow[t] = A.y.p[out];
    }
    unsigned bad = 0;
    for (int u = tid; u < ulim; u += IM_NT) {
      int64_t rot[MS], orot[MS];
#pragma unroll
      for (int t = 0; t < MS - 1; ++t) rot[t] = drow[t][u];
      recover_rot_valid<MS>(rot, A.l, orot);
      if (verify) bad += (drow[MS - 1][u] != wadd(wshl(orot[MS - 1], A.l), orot[0])) ? 1u : 0u;
      if (A.y_bits == 32) {
#pragma unroll
        for (int t = 0; t < MS; ++t)
          reinterpret_cast<int32_t*>(yrow[t])[ybase + u] = (int32_t)(uint32_t)(uint64_t)orot[t];
      } else {
#pragma unroll
        for (int t = 0; t < MS; ++t) reinterpret_cast<int64_t*>(yrow[t])[ybase + u] = orot[t];
      }
    }
    if (A.mismatch) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
      if (lane == 0 && bad) atomicAdd(A.mismatch, (unsigned long long)bad);
    }
  }
}

// Keff/KD/segments for K taps and an output window starting at y_begin:
// p0 = y_begin + tile*T - (Keff - 1) must be == 0 mod 4 (T is a multiple of 16)
static void imma_geometry(int K, int64_t y_begin, ImmaGeom& Gm) {
  Gm.Keff = K + (int)((((y_begin - K + 1) % 4) + 4) % 4);
  Gm.KD = (Gm.Keff + 15 + 31) / 32 * 32;
  Gm.NKC = Gm.KD / 32;
  Gm.NSEG = (Gm.NKC + IM_SEG - 1) / IM_SEG;
}
static size_t imma_table_size(int nseg, int ng) { return (size_t)nseg * ng * 16 * IM_KDS; }
static void launch_table(const void* g, int g_bits, int K, const ImmaGeom& Gm, int ng,
                         unsigned char* table, cudaStream_t stream) {
  const size_t tbytes = imma_table_size(Gm.NSEG, ng);
  const unsigned blocks = (unsigned)((tbytes + 255) / 256 < 1024 ? (tbytes + 255) / 256 : 1024);
  imma_table_kernel<<<blocks, 256, 0, stream>>>(g, g_bits, K, Gm.Keff, Gm.KD, ng, Gm.NSEG, table);
}

template <int MS, int NG, bool EXTRACT>
static int launch_imma(ConvArgs A, int np, cudaStream_t stream) {
  constexpr int T = IM_T;
  ImmaGeom Gm{};
  Gm.np = np;
  imma_geometry(A.K, A.y_begin, Gm);
  Gm.S = (T + Gm.NSEG * IM_SEG * 32 + 15) / 16 * 16;  // room for the last segment's k-steps
  Gm.bt_off = 0;
  Gm.pl_off = (NG * 16 * IM_KDS + 127) / 128 * 128;
  Gm.dt_off = (Gm.pl_off + MS * np * Gm.S + 127) / 128 * 128;
  const size_t dt_bytes = (size_t)MS * T * 8, raw_bytes = (size_t)MS * (Gm.S + 4) * 4;
  Gm.smem = (size_t)Gm.dt_off + (dt_bytes > raw_bytes ? dt_bytes : raw_bytes);
  if (Gm.smem > 227 * 1024) {
    set_error("imma conv: tile needs %zu bytes of shared memory (K=%d too long)", Gm.smem, A.K);
    return NENT_ERR_PARAM;
  }
  auto kern = conv_imma_kernel<MS, NG, EXTRACT>;
  if (ensure_smem((const void*)kern, Gm.smem) != NENT_OK) return NENT_ERR_CUDA;
  // digit-split Toeplitz taps: the caller's prepared table, or one built for
  // this launch in a stream-ordered workspace (freed in stream order after it)
  unsigned char* table = nullptr;
  if (A.imma_table) {
    Gm.table = static_cast<const unsigned char*>(A.imma_table);
  } else {
    const size_t tbytes = imma_table_size(Gm.NSEG, NG);
    if (cudaMallocAsync(reinterpret_cast<void**>(&table), tbytes, stream) != cudaSuccess) {
      set_error("imma conv: workspace allocation of %zu bytes failed", tbytes);
      return NENT_ERR_CUDA;
    }
    launch_table(A.g, A.g_bits, A.K, Gm, NG, table, stream);
    Gm.table = table;
  }
  const int64_t tiles = (A.n_out + T - 1) / T;
  dim3 grid((unsigned)tiles, EXTRACT ? 1 : (unsigned)((A.rows + MS - 1) / MS));
  kern<<<grid, IM_NT, Gm.smem, stream>>>(A, Gm);
  note_conv_kernel(2);
  const int st = check_launch("imma conv");
  if (table) cudaFreeAsync(table, stream);
  return st;
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
int imma_dispatch(ConvArgs& A, int flavor, bool extract, cudaStream_t s) {
  const int np = (flavor >> 8) & 0xf, ng = (flavor >> 12) & 0xf;
  if (np < 1 || np > 8 || ng < 1 || ng > 4) {
    set_error("imma conv: digit counts np=%d ng=%d outside 1..8 / 1..4", np, ng);
    return NENT_ERR_PARAM;
  }
  if (!(flavor & NENT_IMMA_MMA_SYNC)) {
    if (extract) {
      int st = tc05_fused_m3(A, np, ng, s);
      if (st != NENT_TC05_NA) return st;
      st = tc05_fused_m4(A, np, ng, s);
      if (st != NENT_TC05_NA) return st;
      st = tc05_fused_m8(A, np, ng, s);
      if (st != NENT_TC05_NA) return st;
    } else {
      const int st = tc05_plain_m3(A, np, ng, s);
      if (st != NENT_TC05_NA) return st;
    }
    const int st = tc05_conv(A, np, ng, extract, s);
    if (st != NENT_TC05_NA) return st;
  }
  switch (ng) {
    case 1: return imma_dispatch_ng<1>(A, np, extract, s);
    case 2: return imma_dispatch_ng<2>(A, np, extract, s);
    case 3: return imma_dispatch_ng<3>(A, np, extract, s);
    default: return imma_dispatch_ng<4>(A, np, extract, s);
  }
}

}  // namespace nent

using namespace nent;

extern "C" {

int64_t nent_imma_table_bytes(int K, int flavor) {
  ImmaGeom Gm{};
  imma_geometry(K, 0, Gm);
  // K + 3 covers every y_begin residue (Keff <= K + 3)
  ImmaGeom G3{};
  imma_geometry(K + 3, 0, G3);
  const int ng = (flavor >> 12) & 0xf;
  return (int64_t)imma_table_size(G3.NSEG > Gm.NSEG ? G3.NSEG : Gm.NSEG, ng < 1 ? 1 : ng);
}

int nent_imma_table(const void* g, int g_bits, int K, int64_t y_begin, int flavor, void* table,
                    void* stream) {
  const int ng = (flavor >> 12) & 0xf;
  if ((flavor & 0xff) != NENT_MAC_IMMA || ng < 1 || ng > 4 || K < 1 || (g_bits != 32 && g_bits != 64)) {
    set_error("imma table: bad flavour 0x%x / K=%d", flavor, K);
    return NENT_ERR_PARAM;
  }
  ImmaGeom Gm{};
  imma_geometry(K, y_begin, Gm);
  launch_table(g, g_bits, K, Gm, ng, static_cast<unsigned char*>(table), as_stream(stream));
  return check_launch("imma table");
}

}  // extern "C"
