// conv_tc05.cu -- exact integer convolution on the 5th-generation tensor cores
// (tcgen05.mma kind::i8, accumulators in TMEM), plain or fused with
// entangle -> conv -> extract.  Reference semantics: ops._circ_conv_rows
// (/root/reference/pkg/src/nent/ops.py:158-172) on the entangled words of
// codec.entangle (codec.py:49-66), recovered as codec.disentangle
// (codec.py:89-107).
//
// Digit slicing as in conv_imma.cu: x = sum_p 256^p x_p (np balanced int8
// planes), g = sum_j 256^j g_j (ng digits); every digit pair is an exact int8
// GEMM with int32 accumulation, and pairs with equal p + j ("classes") share
// one accumulator.  The GEMM is the Hankel x Toeplitz form of the convolution
// with 128-position blocks:
//
//   D[v][u] = sum_{k < KT} A_j[v][k] . B_p[u][k]       output j0 + 128u + v
//   A_j[v][k] = g_j[v + KT - 128 - k]                   Toeplitz taps, M = 128
//   B_p[u][k] = x_p[j0 - (KT - 128) + 128u + k]         Hankel data,   N = U
//
// B_p is never materialised: the digit plane is written once, linearly, in
// the SWIZZLE_128B layout, and every K step's operand is the same plane seen
// through a K-major descriptor whose start moves by 32 B (rows are 128 B
// apart, so row u of the Hankel matrix starts where block u starts).  KT =
// K + 127 rounded up to 32 (the band of the Toeplitz matrix).  The tap table
// of all ng digits is written once per CTA into TMEM and fed to the MMAs as
// the A operand from there (kind::i8 with A in TMEM), which leaves shared
// memory to the digit planes and the raw-input staging.
//
// Persistent, warp-specialised CTA (one per SM, 12 warps = 3 per sub-partition):
//   warp 0      TMEM allocation; one lane issues every tcgen05.mma
//   warps 1-3   producers: cp.async global -> smem staging (one half-stream
//               ahead), entangle, digit split -> planes (2 stream slots)
//   warps 4-11  epilogue: TMEM -> int64 classes -> recovery -> coalesced stores
// TMEM (512 columns): [0,192) taps, [192,512) a ring of 5 accumulator slots
// of U=64 columns.  Shared memory: two plane slots, the cp.async staging, and
// the stash of the first stream's int64 result until the second arrives (and
// of the check word until the redundant stream arrives).  mbarriers hand plane slots and accumulator slots
// between the roles (tcgen05.commit arrives when the MMAs reading / writing
// them are done).
#include "common.cuh"
#include "conv_common.cuh"
#include "recover.cuh"
#include "tc05.cuh"

#include <cstdio>
#include <cstdlib>

namespace nent {
namespace tcc {

constexpr int U = 64;            // 128-position blocks per tile = MMA N
constexpr int TILE = 128 * U;    // outputs per tile and stream
constexpr int NPROD = 3;         // producer warps (12 warps in all: 3 per SM sub-partition)
constexpr int NEPI = 8;          // epilogue warps (two per TMEM lane quadrant)
constexpr int NT = 32 * (1 + NPROD + NEPI);
constexpr int TAPCOLS = 192;     // TMEM columns for the tap table (8 per digit and K step)
constexpr int RING0 = TAPCOLS;
constexpr int SLOTS = (512 - RING0) / U;  // accumulator ring: 5 slots of U columns (the
                                          // MMA runs up to 4 classes ahead of the epilogue)
constexpr int HALFW = 11;        // staged words per producer thread and half-stream
constexpr int PLANE = 9216;      // bytes per digit plane: 128*U + KT - 128 <= 9216, 1024-aligned
constexpr int NWP = 2 * HALFW * 32 * NPROD;  // plane words every fast tile fills (2112)
static_assert(4 * NWP <= PLANE, "staging fits one plane");
constexpr int STASH_BYTES = 32 * NEPI * 32 * 8;  // 32 int64 per epilogue thread

struct Geom {
  int KT;         // GEMM K: K + 127 rounded up to 32
  int natoms;     // ceil(KT / 128) tap atoms per g digit
  int nsteps;     // KT / 32 MMAs per digit pair
  int np, ng, ncls;
  int nstreams;   // streams per tile: m (fused) or rows (plain)
  int nw;         // 32-bit plane words per stream and tile
  int plane;      // bytes per digit plane, 1024-aligned
  int stage_off;  // smem offset of the cp.async staging (planes at 0)
  int stash_off;  // smem offset of the epilogue stash
  int64_t ntiles;
  int shift;      // tiles start `shift` outputs before y_begin so input windows are 16-byte aligned
  int debug;      // profiling only: 1 skip producer math, 2 skip epilogue math, 4 skip MMAs, 8 role timers
  unsigned long long* dbg;  // role timers (debug & 8)
};

__device__ __forceinline__ void mb_init(uint32_t mb, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mb), "r"(count));
}
__device__ __forceinline__ void mb_arrive(uint32_t mb) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(mb) : "memory");
}
__device__ __forceinline__ void mb_wait(uint32_t mb, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n TC_WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra TC_WAIT_%=;\n}" ::"r"(mb), "r"(parity) : "memory");
}
__device__ __forceinline__ bool elect_one() {
  uint32_t e;
  asm volatile("{\n .reg .pred p;\n elect.sync _|p, 0xffffffff;\n selp.u32 %0, 1, 0, p;\n}" : "=r"(e));
  return e != 0;
}
// Role timers for profiling builds (-DNENT_TC05_TIMERS, NENT_TC05_DEBUG=8):
// TC05_TIMED(slot, stmt) adds stmt's cycles to tw[slot].
#ifdef NENT_TC05_TIMERS
#define TC05_TIMED(i, stmt)           \
  {                                   \
    const long long t0_ = clock64();  \
    stmt;                             \
    tw[i] += clock64() - t0_;         \
  }
#else
#define TC05_TIMED(i, stmt) \
  { stmt; }
#endif
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// balanced base-256 digits: byte p of (v + 0x80..80) ^ 0x80..80 (see conv_imma.cu)
__host__ __device__ constexpr uint64_t bias_of(int n) {
  return n >= 8 ? 0x8080808080808080ull : (0x8080808080808080ull & ((1ull << (8 * n)) - 1));
}
__device__ __forceinline__ uint64_t digits_of(int64_t v, uint64_t bias) {
  return ((uint64_t)v + bias) ^ 0x8080808080808080ull;
}
__device__ __forceinline__ uint32_t byte_col(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3, int p) {
  const uint32_t sel = (uint32_t)p | ((uint32_t)(p + 4) << 4);
  return __byte_perm(__byte_perm(w0, w1, sel), __byte_perm(w2, w3, sel), 0x5410);
}
// (no "memory" clobbers: volatile keeps them ordered against the cp.async
// waits and the release fence, while the ALU work of neighbouring words can
// still interleave)
__device__ __forceinline__ void sts32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"(v));
}
__device__ __forceinline__ void sts64(uint32_t addr, uint64_t v) {
  asm volatile("st.shared.b64 [%0], %1;" ::"r"(addr), "l"(v));
}
__device__ __forceinline__ uint64_t lds64(uint32_t addr) {
  uint64_t v;
  asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ int4 lds128(uint32_t addr) {
  int4 r;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(addr));
  return r;
}
// 4x4 byte transpose: o[p] = byte p of w0, w1, w2, w3
__device__ __forceinline__ void transpose4(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3, uint32_t (&o)[4]) {
  const uint32_t t0 = __byte_perm(w0, w1, 0x5140), t1 = __byte_perm(w0, w1, 0x7362);
  const uint32_t t2 = __byte_perm(w2, w3, 0x5140), t3 = __byte_perm(w2, w3, 0x7362);
  o[0] = __byte_perm(t0, t2, 0x5410);
  o[1] = __byte_perm(t0, t2, 0x7632);
  o[2] = __byte_perm(t1, t3, 0x5410);
  o[3] = __byte_perm(t1, t3, 0x7632);
}
// The NP digit planes of 4 consecutive positions, one 32-bit word per plane.
// u = x + sum_p 128*256^p: its bytes are the balanced digits + 128, i.e. the
// UNSIGNED operand the MMA reads (the +128 per digit is one constant per
// launch, removed in the epilogue).
template <int NP>
__device__ __forceinline__ void put4(uint32_t addr, const uint64_t (&u)[4]) {
  uint32_t o[4];
  transpose4((uint32_t)u[0], (uint32_t)u[1], (uint32_t)u[2], (uint32_t)u[3], o);
#pragma unroll
  for (int p = 0; p < (NP < 4 ? NP : 4); ++p) sts32(addr + (uint32_t)(p * PLANE), o[p]);
  if (NP > 4) {
    transpose4((uint32_t)(u[0] >> 32), (uint32_t)(u[1] >> 32), (uint32_t)(u[2] >> 32), (uint32_t)(u[3] >> 32), o);
#pragma unroll
    for (int p = 4; p < NP; ++p) sts32(addr + (uint32_t)(p * PLANE), o[p - 4]);
  }
}

__device__ __forceinline__ void st_x16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15, %16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

// acc + (int64)a * m for signed 32-bit a, m (mad.wide.s32)
__device__ __forceinline__ uint64_t mad_wide(uint32_t a, int32_t m, uint64_t acc) {
  uint64_t d;
  asm("mad.wide.s32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(m), "l"(acc));
  return d;
}
// acc + ((int64)a * m << 32) modulo 2^64: a multiply-add on the high word only
__device__ __forceinline__ uint64_t mad_hi_word(uint32_t a, int32_t m, uint64_t acc) {
  uint64_t d;
  asm("{\n .reg .b32 lo, hi;\n mov.b64 {lo, hi}, %3;\n mad.lo.u32 hi, %1, %2, hi;\n mov.b64 %0, {lo, hi};\n}"
      : "=l"(d) : "r"(a), "r"(m), "l"(acc));
  return d;
}

// stream fed to the q-th pipeline pass of a tile
__device__ __forceinline__ int stream_of(int q, bool extract, int pivot, int m) {
  if (!extract) return q;
  int s = pivot + 1 + q;
  while (s >= m) s -= m;
  return s;
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

__device__ __forceinline__ void cp_async16_zfill(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}

__device__ __forceinline__ void cp_async4_zfill(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}

// How a tile's input window is staged: 1 = every word in range (plain
// cp.async), 2 = partly outside [0, n_in) in full (zero-padded) mode
// (cp.async with zero fill; words straddling 0 or n_in element by element),
// 0 = per element through conv_prologue (scale / add / gather chains,
// circular wrap, 64-bit rows, rows whose 16-byte phase differs from row 0's).
__device__ __forceinline__ int tile_mode(const ConvArgs& A, int row, int64_t P0) {
  const int32_t* bp = reinterpret_cast<const int32_t*>(A.b.p[row]);
  const int32_t* ap = reinterpret_cast<const int32_t*>(A.a.p[row]);
  if (A.in_bits != 32 || A.perm || A.scale != 1 || A.add || (reinterpret_cast<uintptr_t>(bp + P0) & 15) ||
      (ap && (reinterpret_cast<uintptr_t>(ap + P0) & 15)))
    return 0;
  if (P0 >= 0 && P0 + 4 * (int64_t)NWP <= A.n_in) return 1;
  return A.period >= A.n_in + A.K - 1 ? 2 : 0;
}

template <int NP, bool ENT>
__device__ __forceinline__ void fill_half(uint32_t st, uint32_t pl, uint32_t w0, uint64_t bias, int l) {
  constexpr int PT = 32 * NPROD;
#pragma unroll 4
  for (int i = 0; i < HALFW; ++i) {
    const int4 bv = lds128(st + (uint32_t)(2 * i * PT) * 16u);
    uint64_t u[4] = {(uint64_t)(int64_t)bv.x + bias, (uint64_t)(int64_t)bv.y + bias, (uint64_t)(int64_t)bv.z + bias,
                     (uint64_t)(int64_t)bv.w + bias};
    if (ENT) {
      const int4 av = lds128(st + (uint32_t)((2 * i + 1) * PT) * 16u);
      u[0] += (uint64_t)(int64_t)av.x << l;
      u[1] += (uint64_t)(int64_t)av.y << l;
      u[2] += (uint64_t)(int64_t)av.z << l;
      u[3] += (uint64_t)(int64_t)av.w << l;
    }
    put4<NP>(pl + tc05::sw128(4u * (w0 + (uint32_t)(PT * i))), u);
  }
}

template <bool EXTRACT, int NP, int NSTEPS>
__global__ void __launch_bounds__(NT, 1) conv_tc05_kernel(const __grid_constant__ ConvArgs A,
                                                          const __grid_constant__ Geom G) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bars[4 + 2 * SLOTS];  // plane full[2], empty[2], acc full/empty
  __shared__ uint32_t tmem_slot;
#ifdef NENT_TC05_TIMERS
  const long long tentry = clock64();
#endif
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // 1024-aligned shared addresses (SW128 atoms): planes [2][NP][plane], then the
  // cp.async staging [2][HALFW][2][32*NPROD] int4
  const uint32_t planes_s = tc05::smem_u32(smem_raw);  // 1024-aligned (checked below)
  const uint32_t stage_s = planes_s + (uint32_t)G.stage_off;
  const uint32_t bar0 = tc05::smem_u32(bars);
  auto full_b = [&](int s) { return bar0 + 8u * (uint32_t)s; };
  auto empty_b = [&](int s) { return bar0 + 8u * (uint32_t)(2 + s); };
  auto accf_b = [&](int s) { return bar0 + 8u * (uint32_t)(4 + s); };
  auto acce_b = [&](int s) { return bar0 + 8u * (uint32_t)(4 + SLOTS + s); };

  // ---- setup: barriers, TMEM, the tap table into TMEM columns [0, ng*nsteps*8) ----
  if (tid == 0) {
    for (int s = 0; s < 2; ++s) {
      mb_init(full_b(s), 32 * NPROD);
      mb_init(empty_b(s), 1);
    }
    for (int s = 0; s < SLOTS; ++s) {
      mb_init(accf_b(s), 1);
      mb_init(acce_b(s), NEPI);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tc05::alloc(&tmem_slot, 512);
  tc05::fence_before();
  __syncthreads();
  tc05::fence_after();
  // a 512-column allocation can only be the whole of TMEM: base address 0.
  // Using the constant keeps every MMA operand in uniform registers.
  if (tmem_slot != 0 || (planes_s & 1023u)) __trap();
  constexpr uint32_t tbase = 0;
  {
    // digit bytes of the reversed taps, staged once in shared memory (the
    // cp.async area is still free): rev[j][i] = digit_j(g[KT-1-i]), so that
    // A_j[v][k] = rev[j][k - v + 127] and every 4-byte word of a TMEM row is 4
    // consecutive bytes
    const int RL = G.KT + 128;
    unsigned char* rev = smem_raw + (stage_s - tc05::smem_u32(smem_raw));
    const uint64_t gbias = bias_of(G.ng);
    for (int i = tid; i < RL; i += NT) {
      const int idx = G.KT - 1 - i;
      const int64_t gv = (idx >= 0 && idx < A.K) ? ld_bits(A.g, A.g_bits, idx) : 0;
      const uint64_t d = digits_of(gv, gbias);
      for (int j = 0; j < G.ng; ++j) rev[j * RL + i] = (unsigned char)(d >> (8 * j));
    }
    __syncthreads();
    // lane v of quadrant warp&3 holds row v of A_j; 32-byte K steps are spread
    // over the three warps of each quadrant
    const int v = 32 * (warp & 3) + lane;
    for (int blk = warp >> 2; blk < G.ng * G.nsteps; blk += NT / 128) {
      const int j = blk / G.nsteps, kc = blk % G.nsteps;
      const unsigned char* r = rev + j * RL + 32 * kc - v + 127;
      uint32_t w[8];
#pragma unroll
      for (int c = 0; c < 8; ++c)
        w[c] = (uint32_t)r[4 * c] | ((uint32_t)r[4 * c + 1] << 8) | ((uint32_t)r[4 * c + 2] << 16) |
               ((uint32_t)r[4 * c + 3] << 24);
      tc05::st_x8(tbase + ((uint32_t)(32 * (warp & 3)) << 16) + 8u * (uint32_t)blk, w);
    }
    tc05::wait_st();
    tc05::fence_before();
    __syncthreads();
    tc05::fence_after();
  }
  const int pivot = (EXTRACT && A.r >= 0) ? A.r : 0;
#ifdef NENT_TC05_TIMERS
  long long tw[2] = {0, 0};
  const long long tstart = clock64();
#endif

  if (warp == 0) {
    // ---------------- MMA issuer (whole warp, one elected lane issues) ----------------
    {
      const uint32_t idesc = tc05::idesc_i8(128, U, /*b_signed=*/false);
      const bool skip = (G.debug & 4) != 0;
      int seq = 0, cls = 0;
      for (int64_t tile = blockIdx.x; tile < G.ntiles; tile += gridDim.x) {
        for (int q = 0; q < G.nstreams; ++q, ++seq, cls += G.ncls) {
          const int slot = seq & 1;
          TC05_TIMED(0, mb_wait(full_b(slot), (uint32_t)((seq >> 1) & 1)));
          tc05::fence_after();
          for (int p = 0; p < NP; ++p) {
            const uint32_t blo0 = tc05::desc_sw128_lo(planes_s + (uint32_t)((slot * NP + p) * PLANE));
            for (int j = 0; j < G.ng; ++j) {
              const int c = p + j;
              const int k = cls + c;
              const int rs = k % SLOTS;
              const int use = k / SLOTS;
              const bool first = p == (c - G.ng + 1 > 0 ? c - G.ng + 1 : 0);
              if (first && use >= 1 && !(G.debug & 64)) {
                TC05_TIMED(1, mb_wait(acce_b(rs), (uint32_t)((use - 1) & 1)));
                tc05::fence_after();
              }
              const uint32_t d = tbase + (uint32_t)(RING0 + rs * U);
              const uint32_t a = tbase + (uint32_t)(8 * j * NSTEPS);
              // K steps: A moves 8 TMEM columns, B's start 32 B (= 2 in the descriptor
              // low word).  A compile-time step count keeps the issue stream to the
              // MMAs themselves (a guarded or runtime-bounded loop doubles it).
              if (!skip && elect_one()) {
#pragma unroll
                for (int kc = 0; kc < NSTEPS; ++kc)
                  tc05::mma_i8_ts_lo(d, a + 8u * kc, blo0 + 2u * kc, idesc, (first && kc == 0) ? 0u : 1u);
              }
              __syncwarp();
              if (p == (c < NP - 1 ? c : NP - 1)) tc05::commit_elect(accf_b(rs));
            }
          }
          tc05::commit_elect(empty_b(slot));
        }
      }
    }
    __syncwarp();
  } else if (warp <= NPROD) {
    // ---------------- producers ----------------
    // Work unit: half a stream's words of one tile (HALFW per thread).  The
    // raw words of unit H+1 are in flight (cp.async, thread-private staging)
    // while unit H is entangled and split into digit planes.
    const int ptid = tid - 32;
    constexpr int PT = 32 * NPROD;
    const uint64_t bias = bias_of(NP);
    const int64_t my_tiles = G.ntiles > blockIdx.x ? (G.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int64_t units = my_tiles * G.nstreams * 2;
    auto unit = [&](int64_t H, int64_t& P0, int& row, int& h, int& q) {
      const int64_t lt = H / (2 * G.nstreams);
      q = (int)((H >> 1) % G.nstreams);
      h = (int)(H & 1);
      P0 = A.y_begin - G.shift + (blockIdx.x + lt * gridDim.x) * TILE - (G.KT - 128);
      row = stream_of(q, EXTRACT, pivot, A.rows);
    };
    auto issue = [&](int64_t H) {
      if (H < units && !(G.debug & 32)) {
        int64_t P0;
        int row, h, q;
        unit(H, P0, row, h, q);
        const int mode = tile_mode(A, row, P0);
        const int32_t* bp = reinterpret_cast<const int32_t*>(A.b.p[row]);
        const int32_t* ap = reinterpret_cast<const int32_t*>(A.a.p[row]);
        const uint32_t st = stage_s + (uint32_t)((H & 1) * HALFW * 2 * PT + ptid) * 16u;
        if (mode == 1) {
#pragma unroll
          for (int i = 0; i < HALFW; ++i) {
            const int w = ptid + PT * (HALFW * h + i);
            cp_async16(st + (uint32_t)(2 * i * PT) * 16u, bp + P0 + 4 * w);
            if (ap) cp_async16(st + (uint32_t)((2 * i + 1) * PT) * 16u, ap + P0 + 4 * w);
          }
        } else if (mode == 2) {
          for (int i = 0; i < HALFW; ++i) {
            const int64_t q0 = P0 + 4 * (int64_t)(ptid + PT * (HALFW * h + i));
            const uint32_t db = st + (uint32_t)(2 * i * PT) * 16u, da = st + (uint32_t)((2 * i + 1) * PT) * 16u;
            if (q0 >= 0 && q0 + 4 <= A.n_in) {
              cp_async16(db, bp + q0);
              if (ap) cp_async16(da, ap + q0);
            } else if (q0 + 4 <= 0 || q0 >= A.n_in) {
              cp_async16_zfill(db, bp, 0);  // all four positions are zero padding
              if (ap) cp_async16_zfill(da, ap, 0);
            } else {  // straddles 0 or n_in: element by element
              for (int e = 0; e < 4; ++e) {
                const int64_t q = q0 + e;
                const bool in = q >= 0 && q < A.n_in;
                cp_async4_zfill(db + 4u * e, in ? bp + q : bp, in ? 4u : 0u);
                if (ap) cp_async4_zfill(da + 4u * e, in ? ap + q : ap, in ? 4u : 0u);
              }
            }
          }
        }
      }
      cp_async_commit();
    };
    issue(0);
    for (int64_t H = 0; H < units; ++H) {
      int64_t P0;
      int row, h, q;
      unit(H, P0, row, h, q);
      const int64_t seq = H >> 1;
      const int slot = (int)(seq & 1);
      if (h == 0 && seq >= 2) TC05_TIMED(0, mb_wait(empty_b(slot), (uint32_t)(((seq >> 1) - 1) & 1)));
      issue(H + 1);
      TC05_TIMED(1, cp_async_wait1());
      const uint32_t pl = planes_s + (uint32_t)(slot * NP * PLANE);
      if (G.debug & 1) {
      } else if (tile_mode(A, row, P0) != 0) {
        const uint32_t st = stage_s + (uint32_t)((H & 1) * HALFW * 2 * PT + ptid) * 16u;
        const uint32_t w0 = (uint32_t)(ptid + PT * HALFW * h);
        if (A.a.p[row] != nullptr)
          fill_half<NP, true>(st, pl, w0, bias, A.l);
        else
          fill_half<NP, false>(st, pl, w0, bias, A.l);
      } else {
        for (int i = 0; i < HALFW; ++i) {
          const int w = ptid + PT * (HALFW * h + i);
          if (w < G.nw) {
            uint64_t u[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) u[e] = (uint64_t)conv_prologue(A, row, P0 + 4 * w + e) + bias;
            put4<NP>(pl + tc05::sw128(4u * (uint32_t)w), u);
          }
        }
      }
      if (h == 1) {
        fence_async_smem();
        mb_arrive(full_b(slot));
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else {
    // ---------------- epilogue ----------------
    const int ew = warp - 1 - NPROD;  // 0..7
    const int quad = warp & 3, half = ew >> 2;
    const uint32_t lrow = (uint32_t)(32 * quad) << 16;
    const int v = 32 * quad + lane;
    // thread-private stash, [i][epilogue thread] int64: coalesced, conflict-free
    const uint32_t stash = planes_s + (uint32_t)G.stash_off + 8u * (uint32_t)(32 * ew + lane);
    constexpr uint32_t SSTEP = 8u * 32 * NEPI;
    // the unsigned B digits carry +128 each: every output is high by
    // 128 * sum(g) * sum_{p<NP} 256^p (mod 2^64); start the sums at minus that
    uint64_t gsum = 0;
    for (int k = lane; k < A.K; k += 32) gsum += (uint64_t)ld_bits(A.g, A.g_bits, k);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) gsum += __shfl_xor_sync(0xffffffffu, gsum, o);
    uint64_t ones = 0;
#pragma unroll
    for (int p = 0; p < NP; ++p) ones |= (uint64_t)1 << (8 * p);
    const uint64_t corr = 0 - 128 * gsum * ones;
    unsigned bad = 0;
    int64_t cls = 0;
    for (int64_t tile = blockIdx.x; tile < G.ntiles; tile += gridDim.x) {
      const int64_t ybase = tile * TILE - G.shift;  // output index of (u=0, v=0)
      for (int q = 0; q < G.nstreams; ++q, cls += G.ncls) {
        uint64_t acc[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) acc[i] = corr;
        // acc += A_c * 256^c (IMAD.WIDE; for c >= 4 only the high word moves)
        auto accum = [&](int c, const uint32_t (&r)[32]) {
          if (G.debug & 2) return;
          if (c < 4) {
            const int32_t mul = 1 << (8 * c);
#pragma unroll
            for (int i = 0; i < 32; ++i) acc[i] = mad_wide(r[i], mul, acc[i]);
          } else {
            const int32_t mul = 1 << (8 * (c - 4));
#pragma unroll
            for (int i = 0; i < 32; ++i) acc[i] = mad_hi_word(r[i], mul, acc[i]);
          }
        };
        // classes two at a time: one TMEM round trip (wait::ld) per pair
        for (int c = 0; c < G.ncls; c += 2) {
          const bool two = c + 1 < G.ncls;
          const int k0 = (int)(cls + c), rs0 = k0 % SLOTS, rs1 = (k0 + 1) % SLOTS;
          TC05_TIMED(0, mb_wait(accf_b(rs0), (uint32_t)((k0 / SLOTS) & 1)));
          if (two) TC05_TIMED(0, mb_wait(accf_b(rs1), (uint32_t)(((k0 + 1) / SLOTS) & 1)));
          tc05::fence_after();
          uint32_t r0[32], r1[32];
          tc05::ld_x32(tbase + lrow + (uint32_t)(RING0 + rs0 * U + 32 * half), r0);
          if (two) tc05::ld_x32(tbase + lrow + (uint32_t)(RING0 + rs1 * U + 32 * half), r1);
          tc05::wait_ld();
          tc05::fence_before();
          __syncwarp();
          if (lane == 0) {
            mb_arrive(acce_b(rs0));
            if (two) mb_arrive(acce_b(rs1));
          }
          accum(c, r0);
          if (two) accum(c + 1, r1);
        }
        if (G.debug & 128) {
        } else if (!EXTRACT) {
          void* yp = A.y.p[q];
          const int64_t o0 = ybase + 128 * (32 * half) + v;
          const int64_t lim = A.n_out - o0;  // element i is stored iff -o0 <= 128 i < lim
          if (A.y_bits == 32) {
            int32_t* yo = reinterpret_cast<int32_t*>(yp) + o0;
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (128 * i < lim && 128 * i + o0 >= 0) yo[128 * i] = (int32_t)acc[i];
          } else {
            int64_t* yo = reinterpret_cast<int64_t*>(yp) + o0;
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (128 * i < lim && 128 * i + o0 >= 0) yo[128 * i] = (int64_t)acc[i];
          }
        } else if (q == 0) {  // delta_{pivot+1}: park it in shared memory
#pragma unroll
          for (int i = 0; i < 32; ++i) sts64(stash + SSTEP * i, acc[i]);
        } else if (q == 1) {  // delta_{pivot+2}: recover all three, store, park the check word
          void* y0 = A.y.p[pivot];
          void* y1 = A.y.p[pivot + 1 >= 3 ? pivot - 2 : pivot + 1];
          void* y2 = A.y.p[pivot + 2 >= 3 ? pivot - 1 : pivot + 2];
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            int64_t rot[3], orot[3];
            rot[0] = (int64_t)lds64(stash + SSTEP * i);
            rot[1] = (int64_t)acc[i];
            rot[2] = 0;
            recover_rot_valid<3>(rot, A.l, orot);
            const int64_t o = ybase + 128 * (32 * half + i) + v;
            if (o >= 0 && o < A.n_out) {
              if (A.y_bits == 32) {
                reinterpret_cast<int32_t*>(y0)[o] = (int32_t)orot[0];
                reinterpret_cast<int32_t*>(y1)[o] = (int32_t)orot[1];
                reinterpret_cast<int32_t*>(y2)[o] = (int32_t)orot[2];
              } else {
                reinterpret_cast<int64_t*>(y0)[o] = orot[0];
                reinterpret_cast<int64_t*>(y1)[o] = orot[1];
                reinterpret_cast<int64_t*>(y2)[o] = orot[2];
              }
            }
            // the pivot stream's word must equal (d_{pivot-1} << l) + d_pivot
            if (A.r < 0) sts64(stash + SSTEP * i, (uint64_t)wadd(wshl(orot[2], A.l), orot[0]));
          }
        } else if (A.r < 0) {  // q == 2, verify: the redundant stream against the recovery
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int64_t o = ybase + 128 * (32 * half + i) + v;
            if (o >= 0 && o < A.n_out && lds64(stash + SSTEP * i) != acc[i]) ++bad;
          }
        }
      }
    }
    if (EXTRACT && A.mismatch) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
      if (lane == 0 && bad) atomicAdd(A.mismatch, (unsigned long long)bad);
    }
  }

#ifdef NENT_TC05_TIMERS
  if ((G.debug & 8) && lane == 0 && (warp == 0 || warp == 1 || warp == 1 + NPROD)) {
    const int role = warp == 0 ? 0 : (warp == 1 ? 1 : 2);
    atomicAdd(G.dbg + 3 * role + 0, (unsigned long long)tw[0]);
    atomicAdd(G.dbg + 3 * role + 1, (unsigned long long)tw[1]);
    atomicAdd(G.dbg + 3 * role + 2, (unsigned long long)(clock64() - tstart));
    if (role == 0) {
      atomicAdd(G.dbg + 9, (unsigned long long)(tstart - tentry));
      atomicMax(G.dbg + 10, (unsigned long long)(clock64() - tentry));
    }
  }
#endif
  tc05::fence_before();
  __syncthreads();
  if (warp == 0) {
    tc05::fence_after();
    tc05::dealloc(tbase, 512);
  }
}

}  // namespace tcc

static int sm_count_tc() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    int major = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    if (major != 10) n = -1;  // tcgen05 is sm_100-family only
  }
  return n;
}

// Returns NENT_TC05_NA when the shape is outside this kernel's envelope (the
// caller then runs the mma.sync kernel), else a NENT status.
// Geometry of the tcgen05 kernel for K taps, or false when the shape is
// outside its envelope (m != 3 fused, > 64 rows, K > 257, np > 6, taps wider
// than their 192 TMEM columns, class sums that could leave int32).
static bool tc05_geometry(int K, int rows, int np, int ng, bool extract, tcc::Geom& G, size_t& smem) {
  using namespace tcc;
  if (extract ? rows != 3 : rows > NENT_MAX_STREAMS) return false;
  if (np < 1 || np > 6 || ng < 1 || ng > 4) return false;
  G = Geom{};
  G.KT = (K + 127 + 127) / 128 * 128;  // K steps in multiples of 4 (NSTEPS = 4, 8, 12)
  G.nsteps = G.KT / 32;
  if (G.nsteps > 12) return false;
  G.natoms = (G.KT + 127) / 128;
  if (8 * ng * G.nsteps > TAPCOLS) return false;  // taps must fit their TMEM columns
  G.np = np;
  G.ng = ng;
  G.ncls = np + ng - 1;
  G.nstreams = rows;
  // every class accumulator is an exact int32: |sum| <= 2^14 K min(np, ng)
  if ((int64_t)16384 * K * (np < ng ? np : ng) >= ((int64_t)1 << 31)) return false;
  G.nw = (128 * U + G.KT - 128) / 4;
  if (G.nw > 2 * HALFW * 32 * NPROD || 4 * G.nw > PLANE) return false;
  G.plane = PLANE;
  G.stage_off = 2 * np * PLANE;
  G.stash_off = G.stage_off + 2 * HALFW * 2 * 32 * NPROD * 16;
  smem = (size_t)G.stash_off + (extract ? STASH_BYTES : 0);
  return smem <= 227 * 1024 && sm_count_tc() > 0;
}

int tc05_conv(ConvArgs& A, int np, int ng, bool extract, cudaStream_t s) {
  using namespace tcc;
  Geom G;
  size_t smem = 0;
  if (!tc05_geometry(A.K, A.rows, np, ng, extract, G, smem)) return NENT_TC05_NA;
  { const char* e = getenv("NENT_TC05_DEBUG"); G.debug = e ? atoi(e) : 0; }
  const int sms = sm_count_tc();
  if (sms <= 0) return NENT_TC05_NA;
  {  // align the input windows: (row-0 word offset + P0) = 0 mod 4
    const int64_t wb = (int64_t)((reinterpret_cast<uintptr_t>(A.b.p[0]) >> 2) & 3);
    G.shift = (int)(((wb + A.y_begin - G.KT + 128) % 4 + 4) % 4);
  }
  G.ntiles = (A.n_out + G.shift + TILE - 1) / TILE;
  const unsigned grid = (unsigned)(G.ntiles < sms ? G.ntiles : sms);
  using KernFn = void (*)(ConvArgs, Geom);
#define TC05_ROW(E, S)                                                                                   \
  {conv_tc05_kernel<E, 1, S>, conv_tc05_kernel<E, 2, S>, conv_tc05_kernel<E, 3, S>, conv_tc05_kernel<E, 4, S>, \
   conv_tc05_kernel<E, 5, S>, conv_tc05_kernel<E, 6, S>}
  static const KernFn table[2][3][6] = {{TC05_ROW(false, 4), TC05_ROW(false, 8), TC05_ROW(false, 12)},
                                        {TC05_ROW(true, 4), TC05_ROW(true, 8), TC05_ROW(true, 12)}};
#undef TC05_ROW
  const int si = G.nsteps / 4 - 1;
  const KernFn kern = table[extract][si][np - 1];
  static size_t configured[2][3][6] = {};
  if (smem > configured[extract][si][np - 1]) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
      set_error("tc05 conv: cannot reserve %zu bytes of shared memory", smem);
      return NENT_ERR_CUDA;
    }
    configured[extract][si][np - 1] = smem;
  }
  static unsigned long long* dbg = nullptr;
  if (G.debug & 8) {
    if (!dbg) cudaMalloc(&dbg, 16 * sizeof(unsigned long long));
    cudaMemsetAsync(dbg, 0, 16 * sizeof(unsigned long long), s);
    G.dbg = dbg;
  }
  kern<<<grid, NT, smem, s>>>(A, G);
  if (G.debug & 8) {
    unsigned long long h[16];
    cudaMemcpyAsync(h, dbg, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    fprintf(stderr, "tc05 timers (kcycles/CTA): mma wait_full %.0f wait_accempty %.0f total %.0f | prod wait_empty %.0f "
            "wait_cpasync %.0f total %.0f | epi wait_accfull %.0f - total %.0f | setup %.0f max_cta %.0f\n", h[0] / 1e3 / grid,
            h[1] / 1e3 / grid, h[2] / 1e3 / grid, h[3] / 1e3 / grid, h[4] / 1e3 / grid, h[5] / 1e3 / grid,
            h[6] / 1e3 / grid, h[8] / 1e3 / grid, h[9] / 1e3 / grid, h[10] / 1e3);
  }
  return check_launch("tc05 conv");
}

}  // namespace nent

using namespace nent;

extern "C" int nent_imma_kernel(int flavor, int K, int rows, int extract) {
  if ((flavor & 0xff) != NENT_MAC_IMMA) return 0;
  if (flavor & NENT_IMMA_MMA_SYNC) return 1;
  tcc::Geom G;
  size_t smem = 0;
  return tc05_geometry(K, rows, (flavor >> 8) & 0xf, (flavor >> 12) & 0xf, extract != 0, G, smem) ? 2 : 1;
}
