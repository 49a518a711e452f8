// conv_tc05.cuh -- exact integer convolution on the 5th-generation tensor cores
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
// Persistent, warp-specialised CTA (one per SM, 16 warps = 4 warpgroups):
//   warps 0-3, 12-14  producers: TMA bulk copies global -> smem staging (one
//               half-stream ahead), entangle, digit split -> planes (2 stream slots)
//   warps 4-11  epilogue: TMEM -> int64 classes -> recovery -> coalesced stores
//               (NENT_TC05_NEPI=16: warps 4-19, 16 columns each)
//   warp 15     TMEM allocation; one lane issues every tcgen05.mma
// TMEM (512 columns): [0,192) taps, [192,512) a ring of 5 accumulator slots
// of U=64 columns.  Shared memory: two plane slots, the cp.async staging, and
// the stash of the first stream's int64 result until the second arrives (and
// of the check word until the redundant stream arrives).  mbarriers hand plane slots and accumulator slots
// between the roles (tcgen05.commit arrives when the MMAs reading / writing
// them are done).
#pragma once
#include "common.cuh"
#include "conv_common.cuh"
#include "recover.cuh"
#include "tc05.cuh"


namespace nent {
namespace tcc {

constexpr int U = 64;            // 128-position blocks per tile = MMA N
constexpr int TILE = 128 * U;    // outputs per tile and stream
#ifndef NENT_TC05_NEPI
#define NENT_TC05_NEPI 8
#endif
constexpr int NPROD = 7;         // producer warps: 1-3 and the last warpgroup
constexpr int NEPI = NENT_TC05_NEPI;  // epilogue warps (NEPI / 4 per TMEM lane quadrant)
constexpr int EQ = NEPI / 4;     // epilogue warps per lane quadrant
#ifndef NENT_TC05_MMA_LAST
#define NENT_TC05_MMA_LAST 1
#endif
// The MMA issuer is the CTA's last warp: the warp schedulers favour higher
// warp ids, so the single thread that feeds the tensor core is not held back
// by the producer / epilogue warps sharing its sub-partition.
constexpr int MMA_WARP = NENT_TC05_MMA_LAST ? 4 + NENT_TC05_NEPI + 3 : 0;
#ifndef NENT_TC05_SPLIT_STORE
#define NENT_TC05_SPLIT_STORE 0  // fused m = 3 with the redundant-stream check: d_P stored with the check
#endif
#ifndef NENT_TC05_ONE_ELECT
#define NENT_TC05_ONE_ELECT 1
#endif
#ifndef NENT_TC05_CLASS_MAJOR
#define NENT_TC05_CLASS_MAJOR 0  // MMA chains in class order (one open accumulator slot) instead of plane order
#endif
constexpr int NT = 32 * (1 + NPROD + NEPI);
static_assert(NEPI == 8 || NEPI == 16, "two or four epilogue warpgroups");
// registers per thread after setmaxnreg: 4 warps x PROD_REGS (issuer + producers,
// warpgroup 0), NEPI x EPI_REGS (epilogue), 4 x PROD_REGS (producers, last
// warpgroup).  setmaxnreg.inc draws from the CTA's launch allocation (NT x
// LAUNCH_REGS), so the split must fit it.  More epilogue warps with fewer
// outputs each hide the TMEM-load / shared-memory latency of the drain.
constexpr int LAUNCH_REGS = NEPI == 16 ? 80 : 128;  // 65536 / NT rounded down to 8
constexpr int PROD_REGS = NEPI == 16 ? 64 : 88, EPI_REGS = NEPI == 16 ? 88 : 168;
static_assert(8 * PROD_REGS + NEPI * EPI_REGS <= (NT / 32) * LAUNCH_REGS, "launch register pool");
constexpr int TAPCOLS = 192;     // TMEM columns for the tap table (8 per digit and K step)
constexpr int RING0 = TAPCOLS;
constexpr int SLOTS = (512 - RING0) / U;  // accumulator ring: 5 slots of U columns (the
                                          // MMA runs up to 4 classes ahead of the epilogue)
constexpr int HALFW = 5;         // staged words per producer thread and half-stream
constexpr int PLANE = 9216;      // bytes per digit plane: 128*U + KT - 128 <= 9216, 1024-aligned
constexpr int NWP = 2 * HALFW * 32 * NPROD;  // plane words every fast tile fills (2240)
static_assert(4 * NWP <= PLANE, "staging fits one plane");
constexpr int EC = U / EQ;        // accumulator columns (outputs) per epilogue thread and slot
constexpr int STASH_BYTES = 32 * NEPI * EC * 8;  // EC int64 per epilogue thread

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
  int debug;      // profiling only: 1 skip producer math, 4 skip MMAs, 8 role timers, 32 skip loads, 1024 MMA ignores full planes,
                  // 64 MMA ignores free slots, 128 skip stores, 256 skip TMEM reads + epilogue math
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
// Waits of the producer / epilogue warps.
#ifndef NENT_TC05_WAIT_HINT
#define NENT_TC05_WAIT_HINT 0
#endif
#ifndef NENT_TC05_SLEEP_NS
#define NENT_TC05_SLEEP_NS 64  // back-off between polls of a not-yet-completed phase
#endif
__device__ __forceinline__ void mb_wait_sleep(uint32_t mb, uint32_t parity) {
#if NENT_TC05_WAIT_HINT
  // try_wait with a suspend-time hint: the warp is parked in hardware until the
  // phase completes (or the hint expires) instead of spinning through a
  // poll / nanosleep loop that costs issue slots on the MMA warp's sub-partition
  asm volatile(
      "{\n .reg .pred p;\n TC_WAITH_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      " @!p bra TC_WAITH_%=;\n}" ::"r"(mb), "r"(parity), "r"(0x989680) : "memory");
#else
  uint32_t done;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(done) : "r"(mb), "r"(parity) : "memory");
  while (!done) {
    if (NENT_TC05_SLEEP_NS > 0) __nanosleep(NENT_TC05_SLEEP_NS);
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done) : "r"(mb), "r"(parity) : "memory");
  }
#endif
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

// One warp stages a stream-edge window with cp.async at phase 0: the nw4 int4s of `row`
// that start at sample P0, zeros outside [0, n_in).  int4 k holds samples P0 + 4k .. + 3:
// zero fill for k < kz0 and k >= kc (wholly outside the stream), one 16-byte copy for
// ka <= k < kb (wholly inside; `aligned` = row + P0 is 16-byte aligned), sample by sample
// for the at most two cut int4s in between and for every int4 of a row at another phase.
// The caller waits (cp.async.wait_all), syncs the warp and arrives on the window's barrier.
__device__ __forceinline__ void stage_edge_window(uint32_t dst0, const int32_t* row, int64_t P0, int64_t n_in,
                                                  int nw4, bool aligned, int lane) {
  auto clampw = [&](int64_t v) { return (int)(v < 0 ? 0 : (v > nw4 ? nw4 : v)); };
  const int kz0 = clampw(P0 < 0 ? (-P0) / 4 : 0), ka = clampw(P0 < 0 ? (-P0 + 3) / 4 : 0);
  const int64_t rest = n_in - P0;  // samples from the window's start to the stream's end
  const int kb0 = clampw(rest < 0 ? 0 : rest / 4), kc = clampw(rest < 0 ? 0 : (rest + 3) / 4);
  const int kb = kb0 < ka ? ka : kb0;
  for (int k4 = lane; k4 < kz0; k4 += 32) cp_async16_zfill(dst0 + 16u * (uint32_t)k4, row, 0u);
  for (int k4 = kc + lane; k4 < nw4; k4 += 32) cp_async16_zfill(dst0 + 16u * (uint32_t)k4, row, 0u);
  auto by_sample = [&](int k4) {
    const int64_t q0 = P0 + 4 * (int64_t)k4;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const bool in = q0 + k >= 0 && q0 + k < n_in;
      cp_async4_zfill(dst0 + 16u * (uint32_t)k4 + 4u * (uint32_t)k, in ? row + q0 + k : row, in ? 4u : 0u);
    }
  };
  if (aligned) {
    const int32_t* src = row + P0;
    for (int k4 = ka + lane; k4 < kb; k4 += 32) cp_async16(dst0 + 16u * (uint32_t)k4, src + 4 * k4);
    for (int k4 = kz0 + lane; k4 < ka; k4 += 32) by_sample(k4);
    for (int k4 = kb + lane; k4 < kc; k4 += 32) by_sample(k4);
  } else {
    for (int k4 = kz0 + lane; k4 < kc; k4 += 32) by_sample(k4);
  }
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

// Staging of one work unit (half a stream's window): the b operand's HALFW*PT
// int4 (global words ptid + PT*(HALFW*h + i), i.e. one contiguous run of
// HALFB bytes), then the a operand's.  Thread ptid reads int4 i*PT + ptid.
constexpr uint32_t HALFB = HALFW * 32 * NPROD * 16;

// NP <= 4: the 4 digit planes of 4 consecutive 32-bit words u (bytes =
// unsigned digits), one 32-bit word per plane.
template <int NP>
__device__ __forceinline__ void put4_32(uint32_t addr, uint32_t u0, uint32_t u1, uint32_t u2, uint32_t u3) {
  uint32_t o[4];
  transpose4(u0, u1, u2, u3, o);
#pragma unroll
  for (int p = 0; p < NP; ++p) sts32(addr + (uint32_t)(p * PLANE), o[p]);
}

template <int NP, bool ENT>
__device__ __forceinline__ void fill_half(uint32_t st, uint32_t pl, uint32_t w0, uint64_t bias, int l) {
  constexpr int PT = 32 * NPROD;
  // every staged vector of the unit is loaded before any is used (plain,
  // non-volatile loads the compiler may batch): one shared-memory latency per
  // unit instead of one per vector
  int4 bv[HALFW], av[HALFW];
  const int4* sb = reinterpret_cast<const int4*>(__cvta_shared_to_generic(st));
#pragma unroll
  for (int i = 0; i < HALFW; ++i) {
    bv[i] = sb[i * PT];
    if (ENT) av[i] = sb[HALFB / 16 + i * PT];
  }
#pragma unroll
  for (int i = 0; i < HALFW; ++i) {
    const uint32_t dst = pl + tc05::sw128(4u * (w0 + (uint32_t)(PT * i)));
    if (NP <= 4) {
      // the words fit 32 bits (NP balanced digits): u = b + (a << l) + bias
      // modulo 2^32 has the unsigned digits as its bytes
      const uint32_t b32 = (uint32_t)bias;
      uint32_t u[4] = {(uint32_t)bv[i].x + b32, (uint32_t)bv[i].y + b32, (uint32_t)bv[i].z + b32,
                       (uint32_t)bv[i].w + b32};
      if (ENT) {
        u[0] += (uint32_t)av[i].x << l;
        u[1] += (uint32_t)av[i].y << l;
        u[2] += (uint32_t)av[i].z << l;
        u[3] += (uint32_t)av[i].w << l;
      }
      put4_32<NP>(dst, u[0], u[1], u[2], u[3]);
    } else {
      uint64_t u[4] = {(uint64_t)(int64_t)bv[i].x + bias, (uint64_t)(int64_t)bv[i].y + bias,
                       (uint64_t)(int64_t)bv[i].z + bias, (uint64_t)(int64_t)bv[i].w + bias};
      if (ENT) {
        // + (a << l) as a {lo, hi} pair: the high word is a >> (32 - l) directly
        // (l in [1, 31], checked on the host), so each position costs one shift
        // pair and one 64-bit add
        const int av4[4] = {av[i].x, av[i].y, av[i].z, av[i].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint64_t sh = ((uint64_t)(uint32_t)(av4[e] >> (32 - l)) << 32) | (uint32_t)((uint32_t)av4[e] << l);
          u[e] += sh;
        }
      }
      put4<NP>(dst, u);
    }
  }
}

__device__ __forceinline__ void mb_expect_tx(uint32_t mb, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mb) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(mb)
               : "memory");
}
// named barrier among the producer warps only
__device__ __forceinline__ void producers_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(32 * NPROD) : "memory");
}

// EC consecutive accumulator columns of this warp's 32 lanes (EC = 16 or 32)
__device__ __forceinline__ void ld_cols(uint32_t taddr, uint32_t (&r)[32]) { tc05::ld_x32(taddr, r); }
__device__ __forceinline__ void ld_cols(uint32_t taddr, uint32_t (&r)[16]) { tc05::ld_x16(taddr, r); }

template <bool EXTRACT, int NP, int NG, int NSTEPS>
__global__ void __launch_bounds__(NT, 1) conv_tc05_kernel(const __grid_constant__ ConvArgs A,
                                                          const __grid_constant__ Geom G) {
  constexpr int NCLS = NP + NG - 1;  // digit classes p + j
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bars[6 + 2 * SLOTS];  // plane full[2], empty[2], acc full/empty, staging[2]
  __shared__ uint32_t tmem_slot;
#ifdef NENT_TC05_TIMERS
  const long long tentry = clock64();
#endif
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // 1024-aligned shared addresses (SW128 atoms): planes [2][NP][plane], then the
  // raw-input staging [2][b, a][HALFW][32*NPROD] int4
  const uint32_t planes_s = tc05::smem_u32(smem_raw);  // 1024-aligned (checked below)
  const uint32_t stage_s = planes_s + (uint32_t)G.stage_off;
  const uint32_t bar0 = tc05::smem_u32(bars);
  auto full_b = [&](int s) { return bar0 + 8u * (uint32_t)s; };
  auto empty_b = [&](int s) { return bar0 + 8u * (uint32_t)(2 + s); };
  auto accf_b = [&](int s) { return bar0 + 8u * (uint32_t)(4 + s); };
  auto acce_b = [&](int s) { return bar0 + 8u * (uint32_t)(4 + SLOTS + s); };
  auto stg_b = [&](int s) { return bar0 + 8u * (uint32_t)(4 + 2 * SLOTS + s); };

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
    mb_init(stg_b(0), 1);
    mb_init(stg_b(1), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == MMA_WARP) tc05::alloc(&tmem_slot, 512);
  tc05::fence_before();
  __syncthreads();
  tc05::fence_after();
  // a 512-column allocation can only be the whole of TMEM: base address 0.
  // Using the constant keeps every MMA operand in uniform registers.
  if (tmem_slot != 0 || (planes_s & 1023u)) __trap();
  constexpr uint32_t tbase = 0;
  // Programmatic dependent launch (the host sets the stream-serialization
  // attribute): the next kernel on the stream may be scheduled from here on --
  // its CTAs take SMs as ours exit -- and nothing of ours touches global memory
  // before the previous kernel has completed and flushed.  Without the
  // attribute both are no-ops.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  {
    // digit bytes of the reversed taps, staged once in shared memory (the
    // cp.async area is still free): rev[j][i] = digit_j(g[KT-1-i]), so that
    // A_j[v][k] = rev[j][k - v + 127] and every 4-byte word of a TMEM row is 4
    // consecutive bytes
    const int RL = G.KT + 128;
    unsigned char* rev = smem_raw + (stage_s - tc05::smem_u32(smem_raw));
    const uint64_t gbias = bias_of(NG);
    for (int i = tid; i < ((G.debug & 32768) ? 0 : RL); i += NT) {
      const int idx = G.KT - 1 - i;
      const int64_t gv = (idx >= 0 && idx < A.K) ? ld_bits(A.g, A.g_bits, idx) : 0;
      const uint64_t d = digits_of(gv, gbias);
      for (int j = 0; j < NG; ++j) rev[j * RL + i] = (unsigned char)(d >> (8 * j));
    }
    __syncthreads();
    // lane v of quadrant warp&3 holds row v of A_j; 32-byte K steps are spread
    // over the three warps of each quadrant
    const int v = 32 * (warp & 3) + lane;
    for (int blk = warp >> 2; blk < ((G.debug & 32768) ? 0 : NG * G.nsteps); blk += NT / 128) {
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

  // Register split by warpgroup (setmaxnreg): the issuer + producer groups
  // (warps 0-3 and 12-15) give registers to the two epilogue groups (4-11).
  const bool epi_warp = warp >= 4 && warp < 4 + NEPI;
  if (epi_warp)
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(EPI_REGS));
  else
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(PROD_REGS));

  if (warp == MMA_WARP) {
    // ---------------- MMA issuer (whole warp, one elected lane issues) ----------------
    {
      const uint32_t idesc = tc05::idesc_i8(128, U, /*b_signed=*/false);
      const bool skip = (G.debug & 4) != 0;
      int seq = 0, cls = 0;
      for (int64_t tile = blockIdx.x; tile < G.ntiles; tile += gridDim.x) {
        for (int q = 0; q < G.nstreams; ++q, ++seq, cls += NCLS) {
          const int slot = seq & 1;
          if (!(G.debug & 1024)) TC05_TIMED(0, mb_wait(full_b(slot), (uint32_t)((seq >> 1) & 1)));
          if (!(G.debug & 2048)) tc05::fence_after();
#if NENT_TC05_ONE_ELECT
          // One elected lane issues the whole stream: every chain's MMAs, the
          // accumulator-slot waits and the commits, with no warp reconvergence
          // between the (plane, tap-digit) chains.  The ring position advances
          // incrementally (no per-chain division).
          if (elect_one()) {
            const int rs0 = cls % SLOTS, use0 = cls / SLOTS;
#if NENT_TC05_CLASS_MAJOR
            // class-major: all chains of class c (p + j = c) back to back, then
            // its commit, so the MMA holds one accumulator slot at a time and
            // the epilogue gets the rest of the ring as slack (plane-major
            // order keeps two classes open at once)
#pragma unroll
            for (int c = 0; c < NCLS; ++c) {
              int rs = rs0 + c, use = use0;
              while (rs >= SLOTS) {
                rs -= SLOTS;
                ++use;
              }
              if (use >= 1 && !(G.debug & 64)) {
                TC05_TIMED(1, mb_wait(acce_b(rs), (uint32_t)((use - 1) & 1)));
                tc05::fence_after();
              }
              const uint32_t d = tbase + (uint32_t)(RING0 + rs * U);
#pragma unroll
              for (int p = (c - NG + 1 > 0 ? c - NG + 1 : 0); p <= (c < NP - 1 ? c : NP - 1); ++p) {
                const int j = c - p;
                const bool first = p == (c - NG + 1 > 0 ? c - NG + 1 : 0);
                const uint32_t blo0 = tc05::desc_sw128_lo(planes_s + (uint32_t)((slot * NP + p) * PLANE));
                const uint32_t a = tbase + (uint32_t)(8 * j * NSTEPS);
                if (!skip) {
#pragma unroll
                  for (int kc = 0; kc < NSTEPS; ++kc)
                    tc05::mma_i8_ts_lo(d, a + 8u * kc, blo0 + 2u * kc, idesc, (first && kc == 0) ? 0u : 1u);
                }
              }
              tc05::commit(accf_b(rs));
            }
#else
#pragma unroll
            for (int p = 0; p < NP; ++p) {
              const uint32_t blo0 = tc05::desc_sw128_lo(planes_s + (uint32_t)((slot * NP + p) * PLANE));
#pragma unroll
              for (int j = 0; j < NG; ++j) {
                const int c = p + j;
                int rs = rs0 + c, use = use0;
                while (rs >= SLOTS) {
                  rs -= SLOTS;
                  ++use;
                }
                const bool first = p == (c - NG + 1 > 0 ? c - NG + 1 : 0);
                if (first && use >= 1 && !(G.debug & 64)) {
                  TC05_TIMED(1, mb_wait(acce_b(rs), (uint32_t)((use - 1) & 1)));
                  tc05::fence_after();
                }
                const uint32_t d = tbase + (uint32_t)(RING0 + rs * U);
                const uint32_t a = tbase + (uint32_t)(8 * j * NSTEPS);
                if (!skip) {
#pragma unroll
                  for (int kc = 0; kc < NSTEPS; ++kc)
                    tc05::mma_i8_ts_lo(d, a + 8u * kc, blo0 + 2u * kc, idesc, (first && kc == 0) ? 0u : 1u);
                }
                if (p == (c < NP - 1 ? c : NP - 1)) tc05::commit(accf_b(rs));
              }
            }
#endif
            if (!(G.debug & 4096)) tc05::commit(empty_b(slot));
          }
          __syncwarp();
          continue;
#endif
          // fully unrolled: every TMEM / descriptor operand of the chain is then an
          // immediate or a hoisted uniform register (a runtime (p, j) loop rebuilds
          // them with R2UR moves between chains and costs ~30% of the MMA rate)
#pragma unroll
          for (int p = 0; p < NP; ++p) {
            const uint32_t blo0 = tc05::desc_sw128_lo(planes_s + (uint32_t)((slot * NP + p) * PLANE));
#pragma unroll
            for (int j = 0; j < NG; ++j) {
              const int c = p + j;
              const int k = cls + c;
              const int rs = k % SLOTS;
              const int use = k / SLOTS;
              const bool first = p == (c - NG + 1 > 0 ? c - NG + 1 : 0);
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
          if (!(G.debug & 4096)) tc05::commit_elect(empty_b(slot));
        }
      }
      // drain the last plane slots' commits before the CTA can exit: an
      // mbarrier arrive still in flight must not land in a successor CTA's
      // shared memory
      if (!(G.debug & 4096))
        for (int s = seq > 2 ? seq - 2 : 0; s < seq; ++s) mb_wait(empty_b(s & 1), (uint32_t)((s >> 1) & 1));
    }
    __syncwarp();
  } else if (!epi_warp) {
    // ---------------- producers ----------------
    // Work unit: half a stream's words of one tile (HALFW per thread).  The
    // raw words of unit H+1 are in flight (cp.async, thread-private staging)
    // while unit H is entangled and split into digit planes.
    // 0 .. 32*NPROD-1 over warps 0-3 and the last warpgroup, minus the MMA warp
    const int ptid = MMA_WARP ? (warp < 4 ? tid : tid - 32 * (4 + NEPI) + 128)
                              : (warp < 4 ? tid - 32 : tid - 32 * (4 + NEPI) + 96);
    constexpr int PT = 32 * NPROD;
    const uint64_t bias = bias_of(NP);
    const int64_t my_tiles = G.ntiles > blockIdx.x ? (G.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int64_t units = my_tiles * G.nstreams * 2;
    // Units in order: tile-major, then stream q, then half h.  Walked
    // incrementally (no 64-bit division per unit).
    struct PUnit {
      int64_t P0;  // first input position of the tile window
      int q, h, row, mode;
    };
    auto first_unit = [&]() {
      PUnit u;
      u.P0 = A.y_begin - G.shift + (int64_t)blockIdx.x * TILE - (G.KT - 128);
      u.q = 0;
      u.h = 0;
      u.row = stream_of(0, EXTRACT, pivot, A.rows);
      u.mode = tile_mode(A, u.row, u.P0);
      return u;
    };
    auto next_unit = [&](PUnit u) {
      if (u.h == 0) {
        u.h = 1;
        return u;
      }
      u.h = 0;
      if (++u.q == G.nstreams) {
        u.q = 0;
        u.P0 += (int64_t)gridDim.x * TILE;
      }
      u.row = stream_of(u.q, EXTRACT, pivot, A.rows);
      u.mode = tile_mode(A, u.row, u.P0);
      return u;
    };
    // Interior units (tile_mode 1) arrive by two TMA bulk copies (b and a
    // operand, HALFB bytes each) issued by one producer thread once every
    // producer is done with the buffer's previous unit; edge units (mode 2)
    // by per-thread cp.async with zero fill; mode 0 reads global directly.
    uint32_t stg_phase = 0;  // bit s: parity of staging buffer s's next TMA completion
    auto issue = [&](int64_t H, const PUnit& u) {
      if (H < units && !(G.debug & 32)) {
        const int64_t P0 = u.P0;
        const int h = u.h;
        const int32_t* bp = reinterpret_cast<const int32_t*>(A.b.p[u.row]);
        const int32_t* ap = reinterpret_cast<const int32_t*>(A.a.p[u.row]);
        const uint32_t buf = stage_s + (uint32_t)(H & 1) * 2u * HALFB;
        if (u.mode == 1) {
          producers_sync();  // the buffer's previous unit has been consumed by every producer
          if (ptid == 0) {
            const uint32_t mb = stg_b((int)(H & 1));
            mb_expect_tx(mb, ap ? 2u * HALFB : HALFB);
            bulk_g2s(buf, reinterpret_cast<const char*>(bp + P0) + (size_t)h * HALFB, HALFB, mb);
            if (ap) bulk_g2s(buf + HALFB, reinterpret_cast<const char*>(ap + P0) + (size_t)h * HALFB, HALFB, mb);
          }
        } else if (u.mode == 2) {
          const uint32_t st = buf + (uint32_t)ptid * 16u;
          for (int i = 0; i < HALFW; ++i) {
            const int64_t q0 = P0 + 4 * (int64_t)(ptid + PT * (HALFW * h + i));
            const uint32_t db = st + (uint32_t)(i * PT) * 16u, da = db + HALFB;
            if (q0 >= 0 && q0 + 4 <= A.n_in) {
              cp_async16(db, bp + q0);
              if (ap) cp_async16(da, ap + q0);
            } else if (q0 + 4 <= 0 || q0 >= A.n_in) {
              cp_async16_zfill(db, bp, 0);  // all four positions are zero padding
              if (ap) cp_async16_zfill(da, ap, 0);
            } else {  // straddles 0 or n_in: element by element
              for (int e = 0; e < 4; ++e) {
                const int64_t qq = q0 + e;
                const bool in = qq >= 0 && qq < A.n_in;
                cp_async4_zfill(db + 4u * e, in ? bp + qq : bp, in ? 4u : 0u);
                if (ap) cp_async4_zfill(da + 4u * e, in ? ap + qq : ap, in ? 4u : 0u);
              }
            }
          }
        }
      }
      cp_async_commit();
    };
    PUnit cur = first_unit();
    PUnit nxt = next_unit(cur);
    issue(0, cur);
    for (int64_t H = (G.debug & 16384) ? units : 0; H < units; ++H, cur = nxt, nxt = next_unit(nxt)) {
      const int64_t seq = H >> 1;
      const int slot = (int)(seq & 1);
      const int h = cur.h, row = cur.row;
      if (h == 0 && seq >= 2 && !(G.debug & 4096)) TC05_TIMED(0, mb_wait_sleep(empty_b(slot), (uint32_t)(((seq >> 1) - 1) & 1)));
      issue(H + 1, nxt);
      if (cur.mode == 1 && !(G.debug & 32)) {
        const int sb = (int)(H & 1);
        TC05_TIMED(1, mb_wait_sleep(stg_b(sb), (stg_phase >> sb) & 1u));
        stg_phase ^= 1u << sb;
      } else {
        TC05_TIMED(1, cp_async_wait1());
      }
      const uint32_t pl = planes_s + (uint32_t)(slot * NP * PLANE);
      if (G.debug & 1) {
      } else if (cur.mode != 0) {
        const uint32_t st = stage_s + (uint32_t)(H & 1) * 2u * HALFB + (uint32_t)ptid * 16u;
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
            for (int e = 0; e < 4; ++e) u[e] = (uint64_t)conv_prologue(A, row, cur.P0 + 4 * w + e) + bias;
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
    const int ew = warp - 4;  // 0 .. NEPI-1
    const int quad = warp & 3, part = ew >> 2;  // lane quadrant, column part of the slot
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
    // TMEM -> registers for classes k0 (into r0, if first) and k0 + 1 (into r1,
    // if second) of the ring, then the slots are handed back to the MMA warp
    uint32_t r0[EC], r1[EC];
    auto drain = [&](int k0, bool first, bool second) {
      const int rs0 = k0 % SLOTS, rs1 = (k0 + 1) % SLOTS;
      if (first) TC05_TIMED(0, mb_wait_sleep(accf_b(rs0), (uint32_t)((k0 / SLOTS) & 1)));
      if (second) TC05_TIMED(0, mb_wait_sleep(accf_b(rs1), (uint32_t)(((k0 + 1) / SLOTS) & 1)));
      tc05::fence_after();
      TC05_TIMED(1, {
        if (first) ld_cols(tbase + lrow + (uint32_t)(RING0 + rs0 * U + EC * part), r0);
        if (second) ld_cols(tbase + lrow + (uint32_t)(RING0 + rs1 * U + EC * part), r1);
        tc05::wait_ld();
      });
      tc05::fence_before();
      __syncwarp();
      if (lane == 0) {
        if (first) mb_arrive(acce_b(rs0));
        if (second) mb_arrive(acce_b(rs1));
      }
    };
    for (int64_t tile = (G.debug & 8192) ? G.ntiles : blockIdx.x; tile < G.ntiles; tile += gridDim.x) {
      const int64_t ybase = tile * TILE - G.shift;  // output index of (u=0, v=0)
      // every output of the tile inside [0, n_out) and int32 rows: unconditional
      // stores at immediate offsets from one per-thread base pointer
      const bool fast = A.y_bits == 32 && A.l < 32 && ybase >= 0 && ybase + TILE <= A.n_out;
      const int64_t o0 = ybase + 128 * (EC * part) + v;  // this thread's first output
      for (int q = 0; q < G.nstreams; ++q, cls += NCLS) {
        uint64_t acc[EC];
        // classes two at a time (one TMEM round trip per pair).  The loop is
        // unrolled over the compile-time class count, so every class weight
        // 256^c is an immediate: acc += R_c * 256^c is one IMAD.WIDE (c < 4)
        // or one IMAD on the high word (c >= 4).  The first pair initialises
        // acc (from the bias correction); an odd last class pairs with zeros.
        if (G.debug & 256) {  // profiling: drain the accumulator slots without reading them
          for (int c = 0; c < NCLS; ++c) {
            const int k0 = (int)(cls + c);
            mb_wait_sleep(accf_b(k0 % SLOTS), (uint32_t)((k0 / SLOTS) & 1));
            __syncwarp();
            if (lane == 0) mb_arrive(acce_b(k0 % SLOTS));
          }
          continue;
        }
#pragma unroll
        for (int c = 0; c < NCLS; c += 2) {
          {
            const bool two = c + 1 < NCLS;
            drain((int)(cls + c), true, two);
            if (!two) {
#pragma unroll
              for (int i = 0; i < EC; ++i) r1[i] = 0;
            }
            const int64_t w0 = c < 8 ? (int64_t)((uint64_t)1 << (8 * c)) : 0;
            const int64_t w1 = c + 1 < 8 ? (int64_t)((uint64_t)1 << (8 * (c + 1))) : 0;
#pragma unroll
            for (int i = 0; i < EC; ++i) {
              const uint64_t s = (c == 0 ? corr : acc[i]) + (uint64_t)((int64_t)(int32_t)r0[i] * w0);
              acc[i] = s + (uint64_t)((int64_t)(int32_t)r1[i] * w1);
            }
          }
        }
        if (G.debug & 128) {
        } else if (!EXTRACT) {
          void* yp = A.y.p[q];
          if (fast) {
            int32_t* yo = reinterpret_cast<int32_t*>(yp) + o0;
#pragma unroll
            for (int i = 0; i < EC; ++i) yo[128 * i] = (int32_t)acc[i];
          } else {
            const int64_t lim = A.n_out - o0;  // element i is stored iff -o0 <= 128 i < lim
            if (A.y_bits == 32) {
              int32_t* yo = reinterpret_cast<int32_t*>(yp) + o0;
#pragma unroll
              for (int i = 0; i < EC; ++i)
                if (128 * i < lim && 128 * i + o0 >= 0) yo[128 * i] = (int32_t)acc[i];
            } else {
              int64_t* yo = reinterpret_cast<int64_t*>(yp) + o0;
#pragma unroll
              for (int i = 0; i < EC; ++i)
                if (128 * i < lim && 128 * i + o0 >= 0) yo[128 * i] = (int64_t)acc[i];
            }
          }
        } else if (q == 0) {  // delta_{pivot+1}: park it in shared memory
#pragma unroll
          for (int i = 0; i < EC; ++i) sts64(stash + SSTEP * i, acc[i]);
        } else if (q == 1) {  // delta_{pivot+2}: recover all three, store, park the check word
          void* y0 = A.y.p[pivot];
          void* y1 = A.y.p[pivot + 1 >= 3 ? pivot - 2 : pivot + 1];
          void* y2 = A.y.p[pivot + 2 >= 3 ? pivot - 1 : pivot + 2];
          if (fast) {
            // M = 3 recovery (recover_rot_valid<3>) on consistent words whose
            // recovered outputs fit int32 (the y_bits == 32 contract):
            // v = sext_{2l}((delta_{P+1} << l) - delta_{P+2}) = -d_{P+2} is an
            // int32, so its low word alone gives it; then
            // d_{P+1} = (delta_{P+2} + v) >> l and d_P = (delta_{P+1} - d_{P+1}) >> l
            int32_t* z0 = reinterpret_cast<int32_t*>(y0) + o0;
            int32_t* z1 = reinterpret_cast<int32_t*>(y1) + o0;
            int32_t* z2 = reinterpret_cast<int32_t*>(y2) + o0;
            const int l = A.l;
            if (NENT_TC05_SPLIT_STORE && A.r < 0) {
              // the redundant stream still follows: d_P's store moves to it, so
              // the stores of one tile are spread 2 + 1 over the last two streams
              // instead of 3 + 0 (a shorter epilogue burst at this stream, which
              // the accumulator ring has to absorb).  The stash keeps {d_P, v}.
#pragma unroll
              for (int i = 0; i < EC; ++i) {
                const uint64_t da = lds64(stash + SSTEP * i), db = acc[i];
                const int32_t vv = (int32_t)(((uint32_t)da << l) - (uint32_t)db);
                const int32_t d1 = (int32_t)((int64_t)(db + (uint64_t)(int64_t)vv) >> l);
                const int32_t d0 = (int32_t)((int64_t)(da - (uint64_t)(int64_t)d1) >> l);
                z1[128 * i] = d1;
                z2[128 * i] = (int32_t)(0u - (uint32_t)vv);
                sts64(stash + SSTEP * i, ((uint64_t)(uint32_t)vv << 32) | (uint32_t)d0);
              }
            } else {
#pragma unroll
              for (int i = 0; i < EC; ++i) {
                const uint64_t da = lds64(stash + SSTEP * i), db = acc[i];
                const int32_t vv = (int32_t)(((uint32_t)da << l) - (uint32_t)db);
                const int32_t d1 = (int32_t)((int64_t)(db + (uint64_t)(int64_t)vv) >> l);
                const int32_t d0 = (int32_t)((int64_t)(da - (uint64_t)(int64_t)d1) >> l);
                z0[128 * i] = d0;
                z1[128 * i] = d1;
                z2[128 * i] = (int32_t)(0u - (uint32_t)vv);
                // the pivot stream's word must equal (d_{P+2} << l) + d_P
                if (A.r < 0) sts64(stash + SSTEP * i, (uint64_t)(int64_t)d0 - ((uint64_t)(int64_t)vv << l));
              }
            }
          } else {
#pragma unroll
            for (int i = 0; i < EC; ++i) {
              int64_t rot[3], orot[3];
              rot[0] = (int64_t)lds64(stash + SSTEP * i);
              rot[1] = (int64_t)acc[i];
              rot[2] = 0;
              recover_rot_valid<3>(rot, A.l, orot);
              const int64_t o = o0 + 128 * i;
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
          }
        } else if (A.r < 0) {  // q == 2, verify: the redundant stream against the recovery
          if (fast && NENT_TC05_SPLIT_STORE) {
            // d_P (deferred from the previous stream) and the check of the
            // redundant word: delta_P == (d_{P+2} << l) + d_P with d_{P+2} = -v
            int32_t* z0 = reinterpret_cast<int32_t*>(A.y.p[pivot]) + o0;
#pragma unroll
            for (int i = 0; i < EC; ++i) {
              const uint64_t s = lds64(stash + SSTEP * i);
              const int32_t d0 = (int32_t)(uint32_t)s, vv = (int32_t)(uint32_t)(s >> 32);
              z0[128 * i] = d0;
              bad += ((uint64_t)(int64_t)d0 - ((uint64_t)(int64_t)vv << A.l)) != acc[i];
            }
          } else if (fast) {
#pragma unroll
            for (int i = 0; i < EC; ++i) bad += lds64(stash + SSTEP * i) != acc[i];
          } else {
#pragma unroll
            for (int i = 0; i < EC; ++i) {
              const int64_t o = o0 + 128 * i;
              if (o >= 0 && o < A.n_out && lds64(stash + SSTEP * i) != acc[i]) ++bad;
            }
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
  if ((G.debug & 8) && lane == 0 && (warp == MMA_WARP || warp == (MMA_WARP ? 0 : 1) || warp == 4)) {
    const int role = warp == MMA_WARP ? 0 : (warp == 4 ? 2 : 1);
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
  if (warp == MMA_WARP) {
    tc05::fence_after();
    tc05::dealloc(tbase, 512);
  }
}

}  // namespace tcc
}  // namespace nent
