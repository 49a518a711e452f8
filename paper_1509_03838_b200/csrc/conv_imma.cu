// conv_imma.cu -- exact integer convolution on the tensor cores by digit
// slicing (mma.sync m16n8k32 s8 -> s32), plain or fused with entangle/extract.
// Reference semantics: ops._circ_conv_rows (/root/reference/pkg/src/nent/ops.py:158-172).
#include "common.cuh"
#include "conv_common.cuh"
#include "recover.cuh"

namespace nent {

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
  int Keff;  // K + zero taps so that every tile's first staged position is 4-aligned
  int KD;    // K-dimension of the Toeplitz GEMM (multiple of 32)
  int NKC;   // KD / 32
  int KDs;   // Bt row stride in bytes (== 16 mod 128: conflict-free ldmatrix)
  int S;     // bytes per digit plane (multiple of 16)
  int np;    // digit planes of x
  int RS;    // bytes per reversed-tap digit row
  int bt_off, pl_off, dt_off, r_off;  // smem offsets
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
  const int np = Gm.np, KDs = Gm.KDs, S = Gm.S;

  // ---- digit planes: smem byte i <-> input position j0 - (Keff-1) + i ----
  // Keff = K + zero taps chosen so p0 is a multiple of 4 for every tile.
  const int64_t p0 = j0 - (Gm.Keff - 1);
  const uint64_t xbias = digit_bias(np);
  const int S4 = S >> 2;
  // Fast path (interior tile, int32 streams, no gather/scale/add): one TMA
  // bulk copy per stream lands the raw tile in shared memory (aliasing the
  // result tile dt, unused until the MMAs finish), then the digit split runs
  // from shared memory.  Edge tiles take the general per-element chain.
  bool fast = A.in_bits == 32 && !A.perm && A.scale == 1 && !A.add && p0 >= 0 && p0 + S <= A.n_in;
#pragma unroll
  for (int s = 0; s < MS; ++s) {
    const int row = row0 + s;
    fast = fast && row < A.rows && ((uintptr_t)A.b.p[row] & 15) == 0 && (EXTRACT || !A.a.p[row]);
  }
  if (fast) {
    __shared__ __align__(8) uint64_t mbar;
    int32_t* raw = reinterpret_cast<int32_t*>(smem + Gm.dt_off);  // MS x S words
    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar);
    if (tid == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
      const uint32_t bytes = (uint32_t)(MS * S * 4);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
#pragma unroll
      for (int s = 0; s < MS; ++s) {
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(raw + (size_t)s * S);
        const int32_t* src = reinterpret_cast<const int32_t*>(A.b.p[row0 + s]) + p0;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(dst), "l"(src), "r"((uint32_t)(S * 4)), "r"(mb) : "memory");
      }
    }
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
        " @!p bra WAIT_%=;\n}" ::"r"(mb) : "memory");
    const int4* raw4 = reinterpret_cast<const int4*>(raw);
    for (int w = tid; w < S4; w += IM_NT) {
#pragma unroll
      for (int s = 0; s < MS; ++s) {
        const int4 bv = raw4[(size_t)s * S4 + w];
        int64_t v[4] = {bv.x, bv.y, bv.z, bv.w};
        if (EXTRACT) {  // eps_s = (c_{s-1} << l) + c_s, both tiles already in smem
          const int4 av = raw4[(size_t)((s + MS - 1) % MS) * S4 + w];
          v[0] = wadd(wshl(av.x, A.l), v[0]); v[1] = wadd(wshl(av.y, A.l), v[1]);
          v[2] = wadd(wshl(av.z, A.l), v[2]); v[3] = wadd(wshl(av.w, A.l), v[3]);
        }
        uint32_t* ps = reinterpret_cast<uint32_t*>(pl + (size_t)s * np * S);
        uint64_t u[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) u[e] = digit_word(v[e], xbias);
        const uint32_t l0 = (uint32_t)u[0], l1 = (uint32_t)u[1], l2 = (uint32_t)u[2], l3 = (uint32_t)u[3];
#pragma unroll
        for (int p = 0; p < 4; ++p)
          if (p < np) ps[p * S4 + w] = gather_byte(l0, l1, l2, l3, p);
        if (np > 4) {
          const uint32_t h0 = (uint32_t)(u[0] >> 32), h1 = (uint32_t)(u[1] >> 32),
                         h2 = (uint32_t)(u[2] >> 32), h3 = (uint32_t)(u[3] >> 32);
#pragma unroll
          for (int p = 4; p < 8; ++p)
            if (p < np) ps[p * S4 + w] = gather_byte(h0, h1, h2, h3, p - 4);
        }
      }
    }
  } else {
    for (int s = 0; s < MS; ++s) {
      const int row = row0 + s;
      uint32_t* ps = reinterpret_cast<uint32_t*>(pl + (size_t)s * np * S);
      const bool live = row < A.rows;
      for (int w = tid; w < S4; w += IM_NT) {
        uint64_t u[4];
#pragma unroll
        for (int e = 0; e < 4; ++e)
          u[e] = digit_word(live ? conv_prologue(A, row, p0 + 4 * w + e) : 0, xbias);
        const uint32_t l0 = (uint32_t)u[0], l1 = (uint32_t)u[1], l2 = (uint32_t)u[2], l3 = (uint32_t)u[3];
#pragma unroll
        for (int p = 0; p < 4; ++p)
          if (p < np) ps[p * S4 + w] = gather_byte(l0, l1, l2, l3, p);
        if (np > 4) {
          const uint32_t h0 = (uint32_t)(u[0] >> 32), h1 = (uint32_t)(u[1] >> 32),
                         h2 = (uint32_t)(u[2] >> 32), h3 = (uint32_t)(u[3] >> 32);
#pragma unroll
          for (int p = 4; p < 8; ++p)
            if (p < np) ps[p * S4 + w] = gather_byte(h0, h1, h2, h3, p - 4);
        }
      }
    }
  }

  const uint32_t pl_s = (uint32_t)__cvta_generic_to_shared(pl);
  const uint32_t bt_s = (uint32_t)__cvta_generic_to_shared(bt);
  const int mat = lane >> 3, r8 = lane & 7;
  // per-lane ldmatrix row offsets
  const uint32_t a_lane = 16u * (uint32_t)(r8 + 8 * (mat & 1)) + 16u * (uint32_t)(mat >> 1);
  const uint32_t b_lane = (uint32_t)((8 * (mat >> 1) + r8) * KDs + 16 * (mat & 1));
  const int g = lane >> 2, t4 = lane & 3;

  // K is consumed SEG*32 Toeplitz columns at a time: the segment's taps are
  // digit-split into Bt (shared), its B fragments held in registers, and
  // every stream's int64 partial results accumulate in the staging tile dt.
  for (int kc0 = 0; kc0 < Gm.NKC; kc0 += SEG) {
    const int nkc = min(SEG, Gm.NKC - kc0);
    __syncthreads();  // previous segment's readers of Bt are done
    // Bt_j[b][tl] = digit_j(g[b + Keff - 1 - t]), t = 32*kc0 + tl.  Row b is
    // the reversed digit sequence R_j[v] = digit_j(g[kbase - v]) shifted by b
    // bytes: build R_j once (W + 16 bytes), then every Bt word is one funnel
    // shift of two aligned R_j words.
    {
      const int W = 32 * nkc;
      const int kbase = Gm.Keff - 1 - 32 * kc0;
      unsigned char* rv = smem + Gm.r_off;  // NG x RS bytes, rv[j][v + 16] = R_j[v]
      const int RS = Gm.RS;
      for (int i = tid; i < W + 16; i += IM_NT) {
        const int v = i - 16, k = kbase - v;
        const int64_t gv = (k >= 0 && k < A.K) ? ld_bits(A.g, A.g_bits, k) : 0;
        const uint64_t u = digit_word(gv, digit_bias(NG));
#pragma unroll
        for (int j = 0; j < NG; ++j) rv[j * RS + i] = (unsigned char)(u >> (8 * j));
      }
      __syncthreads();
      const int W4 = W >> 2;
      for (int i = tid; i < NG * 16 * W4; i += IM_NT) {
        const int w = i % W4, jb = i / W4, b = jb & 15, j = jb >> 4;
        const int o = 4 * w - b + 16;  // byte offset of R_j[4w - b] in rv[j]
        const uint32_t* rw = reinterpret_cast<const uint32_t*>(rv + j * RS);
        const uint32_t lo = rw[o >> 2], hi = rw[(o >> 2) + 1];
        *reinterpret_cast<uint32_t*>(bt + (j * 16 + b) * KDs + 4 * w) = __funnelshift_r(lo, hi, 8 * (o & 3));
      }
    }
    __syncthreads();
    uint32_t bf[SEG][NG][4];  // per kc: {b0,b1} of n8-tile 0, {b0,b1} of n8-tile 1
#pragma unroll
    for (int kk = 0; kk < SEG; ++kk)
#pragma unroll
      for (int j = 0; j < NG; ++j)
        if (kk < nkc) ldsm_x4(bf[kk][j], bt_s + (uint32_t)(j * 16 * KDs) + b_lane + 32u * (uint32_t)kk);

    for (int s = 0; s < MS; ++s) {
      if (!EXTRACT && row0 + s >= A.rows) break;
      long long acc[RT][2][4];
#pragma unroll
      for (int rt = 0; rt < RT; ++rt)
#pragma unroll
        for (int nb = 0; nb < 2; ++nb)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[rt][nb][q] = 0;
      for (int p = 0; p < np; ++p) {
        const uint32_t plane = pl_s + (uint32_t)((s * np + p) * S) + 32u * (uint32_t)kc0;
        int c[RT][2][NG][4];
#pragma unroll
        for (int rt = 0; rt < RT; ++rt)
#pragma unroll
          for (int nb = 0; nb < 2; ++nb)
#pragma unroll
            for (int j = 0; j < NG; ++j)
#pragma unroll
              for (int q = 0; q < 4; ++q) c[rt][nb][j][q] = 0;
        auto kstep = [&](int kk) {
#pragma unroll
          for (int rt = 0; rt < RT; ++rt) {
            uint32_t af[4];
            ldsm_x4(af, plane + 256u * (uint32_t)(warp * RT + rt) + a_lane + 32u * (uint32_t)kk);
#pragma unroll
            for (int j = 0; j < NG; ++j) {
              imma16832(c[rt][0][j], af, bf[kk][j][0], bf[kk][j][1]);
              imma16832(c[rt][1][j], af, bf[kk][j][2], bf[kk][j][3]);
            }
          }
        };
        if (nkc == SEG) {
          // full segment: straight-line code, so the A-fragment loads of the
          // next k-steps can be scheduled ahead of this step's MMAs
#pragma unroll
          for (int kk = 0; kk < SEG; ++kk) kstep(kk);
        } else {
#pragma unroll
          for (int kk = 0; kk < SEG; ++kk) {
            if (kk >= nkc) break;
            kstep(kk);
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
      // this segment's contribution: C fragment (row g|g+8, col 2t|2t+1) of n8-tile nb
#pragma unroll
      for (int rt = 0; rt < RT; ++rt)
#pragma unroll
        for (int nb = 0; nb < 2; ++nb)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int u = 256 * (warp * RT + rt) + 16 * (g + 8 * (q >> 1)) + 8 * nb + 2 * t4 + (q & 1);
            int64_t* d = dt + (size_t)s * T + u;
            *d = kc0 == 0 ? acc[rt][nb][q] : wadd(*d, acc[rt][nb][q]);
          }
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
    // rotation hoisted out of the position loop: rotated smem rows in, rotated
    // output rows out (rot[MS-1] is the pivot stream, read only to verify)
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
    const int64_t ybase = j0 - A.y_begin;
    const int64_t ulim = jend - j0 < T ? jend - j0 : T;
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

template <int MS, int NG, bool EXTRACT>
static int launch_imma(ConvArgs A, int np, cudaStream_t stream) {
  constexpr int T = IM_WARPS * imma_rt(MS) * 256;
  ImmaGeom Gm{};
  Gm.np = np;
  // p0 = y_begin + tile*T - (Keff - 1) must be == 0 mod 4 (T is a multiple of 16)
  Gm.Keff = A.K + (int)((((A.y_begin - A.K + 1) % 4) + 4) % 4);
  Gm.KD = (Gm.Keff + 15 + 31) / 32 * 32;
  Gm.NKC = Gm.KD / 32;
  Gm.KDs = (imma_seg(NG) * 32 + 127) / 128 * 128 + 16;  // one segment; == 16 mod 128
  Gm.S = (T + Gm.KD + 15) / 16 * 16;
  Gm.RS = (imma_seg(NG) * 32 + 16 + 8 + 15) / 16 * 16;
  Gm.bt_off = 0;
  Gm.pl_off = (NG * 16 * Gm.KDs + 127) / 128 * 128;
  Gm.dt_off = (Gm.pl_off + MS * np * Gm.S + 127) / 128 * 128;
  {
    const size_t dt_bytes = (size_t)MS * T * 8, raw_bytes = (size_t)MS * Gm.S * 4;
    Gm.r_off = (int)((Gm.dt_off + (dt_bytes > raw_bytes ? dt_bytes : raw_bytes) + 127) / 128 * 128);
    Gm.smem = (size_t)Gm.r_off + (size_t)NG * Gm.RS;
  }
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
int imma_dispatch(ConvArgs& A, int flavor, bool extract, cudaStream_t s) {
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

}  // namespace nent
