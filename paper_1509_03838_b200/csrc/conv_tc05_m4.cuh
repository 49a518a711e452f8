// conv_tc05_m4.cuh -- the cfg3 hot path: fused entangle -> convolution ->
// extract of m = 4 int32 streams with a LONG filter (K up to 1153 taps) on the
// 5th-generation tensor cores, for the byte-aligned entangling shift l = 16
// (the (4,64,16,16) geometry) and int16-range samples.  Reference semantics:
// codec.entangle (codec.py:57-72), ops._circ_conv_rows on the zero-padded
// streams (ops.py:158-172), codec.disentangle (codec.py:89-131).
//
// Same digit scheme as conv_tc05_m3.cuh: eps_i = (c_{i-1} << 16) + c_i has the
// digits {lo(c_i), hi(c_i), lo(c_{i-1}), hi(c_{i-1})} (low bytes unsigned, high
// bytes signed, no carries), so each raw stream is split once into two byte
// planes and the MMA reads every entangled stream's four digit planes from
// them; the taps are balanced base-256 digits.
//
// What a long filter changes.  The Toeplitz tap operand of K taps is
// KT = K + 127 (rounded up to 128) bytes per TMEM lane and tap digit: 576
// columns for K = 1024, more than TMEM has.  So the loop order is turned
// around: ALL five class accumulators of ONE stream stay resident in TMEM
// while that stream's K steps run, and the tap operand streams through a
// small TMEM ring:
//   * MMA N = 32: a tile is 32 blocks of 128 outputs of each stream; one
//     accumulator (digit class) is 32 columns, a stream's five 160 columns,
//     two such buffers 320 columns (the epilogue drains one stream while the
//     MMA fills the next).  (N = 16 with a stream pair resident was measured
//     first: 0.157 ms on cfg3, bound by the issue rate of one thread -- a
//     tcgen05.mma issues no faster than every ~9 cycles, 128 x 16 x 32 takes 8.)
//   * the tap ring: 3 groups of 4 K steps x NG digits x 8 columns = 192 columns;
//     four "tap writer" warps (one per TMEM lane quadrant) copy each group's
//     Toeplitz blocks into it: lane v's 32 bytes of K step kc start at byte
//     32 kc + 127 - v of the reversed tap digits, and shared memory holds 16
//     byte-shifted copies of that array, so every block is two aligned LDS.128
//     and one tcgen05.st; the MMA warp hands a group back with a commit.
// For K = 1024 the band costs 1152 / 1024 = 1.125x the method's MACs (a filter
// cut into 256-tap segments would pay 1.5x per segment).
//
// CTA: 16 warps, one persistent CTA per SM:
//   warps 0-7   epilogue (2 per TMEM lane quadrant, 16 accumulator columns each)
//   warps 8-11  tap writers
//   warps 12-13 converters (raw int32 window -> two byte planes per stream)
//   warp 14     loader: lane 0 issues one bulk copy per raw window; a stream-edge window (not
//               wholly inside the stream) is staged by the whole warp with cp.async + zero fill
//   warp 15     TMEM allocation; one elected lane issues every tcgen05.mma
// Extraction: the streams are convolved in the order P+1, P+2, P+3 (and P last
// when all four are present and the redundant one is checked), P the failed
// stream (or 0).  Of every stream's word only L = delta mod 2^32 and
// M = (delta >> 16) mod 2^32 are formed (conv_tc05_m3.cuh); three words of
// state per output carry M_{P+1}, then M_{P+2} and L_{P+2}, and with stream P+3
//   d_{P+3} = L_{P+3} - (L_{P+2} << 16),  d_{P+2} = M_{P+3} - (d_{P+3} >> 16),
//   d_{P+1} = M_{P+2} - (d_{P+2} >> 16),  d_P     = M_{P+1} - (d_{P+1} >> 16).
#pragma once
#include "conv_tc05_m3.cuh"

namespace nent {
#ifndef NENT_M4_WINBAR
#define NENT_M4_WINBAR 0  // 1: the MMA starts a stream as soon as its two windows are split (measured slower: 0.1137 vs 0.1095 ms on cfg3)
#endif

namespace tcm4 {

using tcc::bias_of;
using tcc::bulk_g2s;
using tcc::digits_of;
using tcc::elect_one;
using tcc::fence_async_smem;
using tcc::lds128;
using tcc::mb_arrive;
using tcc::mb_expect_tx;
using tcc::mb_init;
using tcc::mb_wait;
using tcc::mb_wait_sleep;
using tcc::sts32;
using tcm3::sar16;
using tcm3::split2;
using tcm3::wide1;

constexpr int M = 4;                   // streams
constexpr int U = 32;                  // 128-position blocks per tile = MMA N
constexpr int TILE = 128 * U;          // outputs per tile and stream (4096)
constexpr int NEPI = 8, NTAP = 4, NCONV = 2;
constexpr int TAP0 = NEPI, CONV0 = TAP0 + NTAP, LOAD_WARP = CONV0 + NCONV, MMA_WARP = LOAD_WARP + 1;
constexpr int NT = 32 * (MMA_WARP + 1);
static_assert(NT == 512, "16 warps");
constexpr int EC = U / (NEPI / 4);     // 16 accumulator columns per epilogue thread
constexpr int KTMAX = 1280;            // K <= 1153
constexpr int GK = 4;                  // K steps per tap-ring group
constexpr int TRING = 3;               // tap-ring groups
constexpr int NCLS5 = 5;               // accumulator classes per stream (4 data digits + 2 tap digits - 1)
constexpr int ACC0 = 192;              // accumulators: columns [192, 512)
constexpr int BUFC = NCLS5 * U;        // 160 columns per stream buffer
constexpr int PLANE = 6144;            // bytes per byte plane: 128 * (U - 1) + KTMAX = 5248, 1024-aligned
constexpr int SLOTB = 2 * M * PLANE;   // one tile slot: 4 raw streams x {lo, hi}
constexpr int NSLOT = 2;
#ifndef NENT_M4_NSTAGE
#define NENT_M4_NSTAGE 4
#endif
constexpr int NSTAGE = NENT_M4_NSTAGE;  // staging ring depth: a whole tile's four raw windows in flight
constexpr uint32_t SSTR = 4 * (128 * (U - 1) + KTMAX) + 128;  // staging stride: the largest window + lead-in
constexpr int NCOPY = 16;              // byte-shifted copies of the reversed tap digits
constexpr int RLMAX = KTMAX + 144;     // one copy: KT + 128 bytes + one 16-byte vector of slack
constexpr int REVB = 2 * NCOPY * RLMAX;
constexpr size_t SMEM = NSLOT * (size_t)SLOTB + (size_t)NSTAGE * SSTR + REVB;
static_assert(SMEM + 1024 <= 227 * 1024, "shared memory");
constexpr int EPI_REGS = 168, OTHER_REGS = 88;
static_assert(NEPI * EPI_REGS + (16 - NEPI) * OTHER_REGS <= 16 * 128, "launch register pool");

struct Geom {
  int KT, nsteps, ngrp;  // GEMM K (bytes), K steps, tap-ring groups per stream pair
  int nw4;               // int4 words per raw window: (TILE + KT - 128) / 4
  int64_t ntiles;
  int64_t tile_off;      // CTA b's tiles are (tile_off + b + k * grid) mod ntiles
  int shift;             // tiles start `shift` outputs early: row 0's windows are 16-byte aligned
  int dph[M];            // word phase of row s relative to row 0 (mod 4)
  unsigned long long* dbg;  // role timers (profiling builds, -DNENT_TC05_TIMERS)
};

// STAMP(i): every CTA records the global timer (ns) at point i of its timeline (-DNENT_M4_STAMPS)
#ifdef NENT_M4_STAMPS
#define M4_STAMP(i)                                           \
  if (G.dbg) {                                                \
    unsigned long long gt_;                                   \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt_));    \
    G.dbg[16 + 8 * blockIdx.x + (i)] = gt_;                   \
  }
#else
#define M4_STAMP(i)
#endif

template <int NG>
__global__ void __launch_bounds__(NT, 1) conv_tc05_m4_kernel(const __grid_constant__ ConvArgs A,
                                                             const __grid_constant__ Geom G) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // plane full [NSLOT][M] / empty [NSLOT], stage full/free [NSTAGE], tap full/free [TRING], acc full/free [2]
  __shared__ __align__(8) uint64_t bars[NSLOT * M + NSLOT + 2 * NSTAGE + 2 * TRING + 4];
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) M4_STAMP(0);
  const uint32_t planes_s = tc05::smem_u32(smem_raw);
  const uint32_t stage_s = planes_s + (uint32_t)(NSLOT * SLOTB);
  unsigned char* rev = smem_raw + NSLOT * SLOTB + NSTAGE * SSTR;
  const uint32_t bar0 = tc05::smem_u32(bars);
  auto bar = [&](int i) { return bar0 + 8u * (uint32_t)i; };
  // (one "planes full" barrier per tile slot AND raw window: the MMA starts a stream as soon
  // as the two windows it reads are split, not when the whole tile is)
  auto full_b = [&](int ts, int s) { return bar(ts * M + s); };
  constexpr int B0 = NSLOT * M;
  auto empty_b = [&](int s) { return bar(B0 + s); };
  auto sfull_b = [&](int s) { return bar(B0 + NSLOT + s); };
  auto sfree_b = [&](int s) { return bar(B0 + NSLOT + NSTAGE + s); };
  constexpr int B1 = B0 + NSLOT + 2 * NSTAGE;
  auto tfull_b = [&](int s) { return bar(B1 + s); };
  auto tfree_b = [&](int s) { return bar(B1 + TRING + s); };
  auto afull_b = [&](int h) { return bar(B1 + 2 * TRING + h); };
  auto afree_b = [&](int h) { return bar(B1 + 2 * TRING + 2 + h); };

  if (tid == 0) {
    for (int s = 0; s < NSLOT; ++s) {
      for (int w = 0; w < M; ++w) mb_init(full_b(s, w), NCONV);
      mb_init(empty_b(s), 1);
    }
    for (int s = 0; s < NSTAGE; ++s) {
      mb_init(sfull_b(s), 1);
      mb_init(sfree_b(s), NCONV);
    }
    for (int s = 0; s < TRING; ++s) {
      mb_init(tfull_b(s), NTAP);
      mb_init(tfree_b(s), 1);
    }
    for (int h = 0; h < 2; ++h) {
      mb_init(afull_b(h), 1);
      mb_init(afree_b(h), NEPI);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == MMA_WARP) tc05::alloc(&tmem_slot, 512);
  const int my_tiles = G.ntiles > blockIdx.x ? (int)((G.ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  // The CTA's tiles (tile_off + blockIdx.x + k * gridDim.x) mod ntiles are processed in the
  // order k = 1, 2, ..., 0.  The stream-edge tiles (tile 0 and the last ones), whose windows
  // are loaded element by element, are the slow ones: tile_off (conv_tc05_m3.cu:
  // edge_tile_offset) puts them on the CTAs with one tile fewer where it can, and a CTA's
  // k = 0 tile comes last, so an edge tile is never the first one.
  auto tile_ord = [&](int t) -> int64_t {
    int64_t j = G.tile_off + blockIdx.x + (int64_t)(t + 1 < my_tiles ? t + 1 : 0) * gridDim.x;
    return j >= G.ntiles ? j - G.ntiles : j;
  };
  auto P0_of = [&](int t) -> int64_t { return A.y_begin - G.shift + tile_ord(t) * TILE - (G.KT - 128); };
  const int64_t P0_first = P0_of(0);
  auto staged = [&](int64_t P0) { return P0 >= 4 && P0 + 4 * (int64_t)G.nw4 + 4 <= A.n_in; };
  // one raw window: row s from dph[s] words earlier, so every source is 16-byte aligned
  auto issue_window = [&](int s, int64_t P0, int b) {
    const int d = G.dph[s];
    const char* src = reinterpret_cast<const char*>(reinterpret_cast<const int32_t*>(A.b.p[s]) + P0 - d);
    const uint32_t bytes = 16u * (uint32_t)G.nw4 + (d ? 16u : 0u);
    mb_expect_tx(sfull_b(b), bytes);
    bulk_g2s(stage_s + (uint32_t)b * SSTR, src, bytes, sfull_b(b));
  };
  // the first tile's windows are in flight while the tap table is built (the
  // barrier initialisation is ordered before by the fence + this sync)
  constexpr int PRE = NSTAGE < M ? NSTAGE : M;
  const bool pre_issue = my_tiles > 0 && staged(P0_first);
  __syncthreads();
  if (pre_issue && warp == LOAD_WARP && lane == 0) {
#pragma unroll
    for (int s = 0; s < PRE; ++s) issue_window(s, P0_first, s);
  }
  // the reversed taps' digits rev_j[i] = digit_j(g[KT-1-i]), i in [0, KT + 144), as
  // NCOPY byte-shifted copies: copy k holds rev_j[i + k] at byte i (layout
  // [digit][copy][byte], RL bytes per copy; RL / 16 is odd, so the copies a
  // quarter warp reads sit in different bank groups).  Lane v's 32 bytes of the
  // Toeplitz block of K step kc start at rev_j[32 kc + 127 - v].
  const int RL = G.KT + 144;
  // (the converter warps go straight to the first tile's windows: they never read the taps)
  const bool is_conv = warp >= CONV0 && warp < CONV0 + NCONV;
  if (!is_conv) {
    const uint64_t gbias = bias_of(NG);
    const int stid = warp < CONV0 ? tid : tid - 32 * NCONV;  // index among the NT - 32 NCONV staging threads
    for (int i = stid; i < RL + NCOPY; i += NT - 32 * NCONV) {
      const int idx = G.KT - 1 - i;
      const int64_t gv = (idx >= 0 && idx < A.K) ? ld_bits(A.g, A.g_bits, idx) : 0;
      const uint64_t d = digits_of(gv, gbias);
#pragma unroll
      for (int j = 0; j < NG; ++j) {
        const unsigned char dj = (unsigned char)(d >> (8 * j));
#pragma unroll
        for (int k = 0; k < NCOPY; ++k)
          if (i - k >= 0 && i - k < RL) rev[(j * NCOPY + k) * RL + (i - k)] = dj;
      }
    }
    tc05::fence_before();
    asm volatile("bar.sync 1, %0;" ::"n"(NT - 32 * NCONV) : "memory");
    tc05::fence_after();
  }
  if (tmem_slot != 0 || (planes_s & 1023u)) __trap();
  constexpr uint32_t tbase = 0;

  long long tw[6] = {0, 0, 0, 0, 0, 0};
  const long long tstart = clock64();
  const bool verify = A.r < 0;
  const int P = verify ? 0 : A.r;  // pivot: the stream never read (or checked last)

  // streams in convolution order: P+1, P+2, P+3 and, with the redundant-stream check, P
  const int nstr = verify ? M : M - 1;
  if (warp < NEPI) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(EPI_REGS));
    // ---------------- epilogue ----------------
    const int quad = warp & 3, part = warp >> 2;
    const uint32_t lrow = (uint32_t)(32 * quad) << 16;
    const int v = 32 * quad + lane;
    const int sa = (P + 1) & 3, sb = (P + 2) & 3, sc = (P + 3) & 3;
    int32_t* yP = reinterpret_cast<int32_t*>(A.y.p[P]);
    int32_t* ya = reinterpret_cast<int32_t*>(A.y.p[sa]);
    int32_t* yb = reinterpret_cast<int32_t*>(A.y.p[sb]);
    int32_t* yc = reinterpret_cast<int32_t*>(A.y.p[sc]);
    unsigned bad = 0;
    int nbuf = 0;  // stream buffers consumed so far (same sequence as the MMA warp)
    // the two views of the next stream's word for this thread's 16 outputs; the
    // buffer goes back to the MMA warp as soon as it is in registers
    auto views = [&](uint32_t (&L)[EC], uint32_t (&Mv)[EC]) {
      const int bsel = nbuf & 1;
      TM(0, mb_wait_sleep(afull_b(bsel), (uint32_t)((nbuf >> 1) & 1)));
      tc05::fence_after();
      uint32_t r[NCLS5][EC];
#pragma unroll
      for (int c = 0; c < 4 + NG - 1; ++c)
        tc05::ld_x16(tbase + lrow + (uint32_t)(ACC0 + bsel * BUFC + c * U + EC * part), r[c]);
      tc05::wait_ld();
      tc05::fence_before();
      __syncwarp();
      if (lane == 0) mb_arrive(afree_b(bsel));
      ++nbuf;
#pragma unroll
      for (int k = 0; k < EC; ++k) {
        uint32_t q;
        const uint32_t lo = wide1(r[1][k], r[0][k], q);
        L[k] = lo + (r[2][k] << 16) + (r[3][k] << 24);
        Mv[k] = q + r[2][k] + (r[3][k] << 8);
        if (NG > 1) Mv[k] += r[4][k] << 16;
      }
    };
    for (int t = 0; t < my_tiles; ++t) {
      const int64_t tile = tile_ord(t);
      const int64_t o0 = tile * TILE - G.shift + 128 * (EC * part) + v;
      uint32_t s0[EC], s1[EC], s2[EC];  // M_{P+1}; M_{P+2}, L_{P+2}
      {
        uint32_t L[EC];
        views(L, s0);  // stream P+1
      }
      views(s2, s1);  // stream P+2
      {
        uint32_t L[EC], Mv[EC];
        views(L, Mv);  // stream P+3: everything is known
#pragma unroll
        for (int k = 0; k < EC; ++k) {
          const uint32_t d3 = L[k] - (s2[k] << 16);
          const uint32_t d2 = Mv[k] - (uint32_t)sar16(d3);
          const uint32_t d1 = s1[k] - (uint32_t)sar16(d2);
          const uint32_t d0 = s0[k] - (uint32_t)sar16(d1);
          const int64_t o = o0 + 128 * k;
          if (o >= 0 && o < A.n_out) {
            yP[o] = (int32_t)d0;
            ya[o] = (int32_t)d1;
            yb[o] = (int32_t)d2;
            yc[o] = (int32_t)d3;
          }
          // the expected views of the redundant word delta_P = (d_{P+3} << 16) + d_P
          s0[k] = (d3 << 16) + d0;
          s1[k] = d3 + (uint32_t)sar16(d0);
        }
      }
      if (verify) {
        uint32_t L[EC], Mv[EC];
        views(L, Mv);  // stream P; positions outside the rows are convolutions of zeros, consistent too
#pragma unroll
        for (int k = 0; k < EC; ++k) bad += ((L[k] ^ s0[k]) | (Mv[k] ^ s1[k])) != 0;
      }
    }
    if (A.mismatch) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
      if (lane == 0 && bad) atomicAdd(A.mismatch, (unsigned long long)bad);
    }
  } else {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(OTHER_REGS));
    if (warp == MMA_WARP) {
      // ---------------- MMA issuer ----------------
      const uint32_t idesc_u = tc05::idesc_i8(128, U, /*b_signed=*/false);
      const uint32_t idesc_s = tc05::idesc_i8(128, U, /*b_signed=*/true);
      int gtot = 0;  // tap-ring groups consumed so far
      int nbuf = 0;  // stream buffers filled so far
      for (int t = 0; t < my_tiles; ++t) {
        const int ts = t % NSLOT;
        if (elect_one()) {
          const uint32_t slot_s = planes_s + (uint32_t)(ts * SLOTB);
#if !NENT_M4_WINBAR
          for (int w = 0; w < M; ++w) TM(0, mb_wait(full_b(ts, w), (uint32_t)((t / NSLOT) & 1)));
          tc05::fence_after();
#endif
          for (int si = 0; si < nstr; ++si, ++nbuf) {
            const int i = (P + 1 + si) & 3, im1 = (i + M - 1) & 3;
#if NENT_M4_WINBAR
            // the byte planes of raw streams i and i-1 are in shared memory: the converters
            // finish a tile's windows in the order 0, 1, 2, 3, so the later one is enough
            TM(0, mb_wait(full_b(ts, i > im1 ? i : im1), (uint32_t)((t / NSLOT) & 1)));
            tc05::fence_after();
#endif
            if (si == 0) {
              if (t == 0) M4_STAMP(1);
              if (t == 1) M4_STAMP(2);
              if (t == my_tiles - 1) M4_STAMP(3);
            }
            const int bsel = nbuf & 1;
            if (nbuf >= 2) {  // the stream that last used this buffer was drained
              TM(2, mb_wait(afree_b(bsel), (uint32_t)(((nbuf >> 1) - 1) & 1)));
              tc05::fence_after();
            }
            // the four digit planes of eps_i: bytes of c_i (p < 2) and of c_{i-1} (p >= 2)
            // (descriptors walked along K in place: one add per plane and K step)
            uint64_t bd[4];
#pragma unroll
            for (int p = 0; p < 4; ++p)
              bd[p] = tc05::desc_sw128_from_lo(
                  tc05::desc_sw128_lo(slot_s + (uint32_t)((2 * (p < 2 ? i : im1) + (p & 1)) * PLANE)));
            const uint32_t dacc = tbase + (uint32_t)(ACC0 + bsel * BUFC);
            for (int g = 0; g < G.ngrp; ++g, ++gtot) {
              const int rs = gtot % TRING;
              TM(1, mb_wait(tfull_b(rs), (uint32_t)((gtot / TRING) & 1)));
              tc05::fence_after();
              const uint32_t acc_first = g == 0 ? 0u : 1u;
              const uint32_t atap = tbase + (uint32_t)(rs * GK * NG * 8);
#pragma unroll
              for (int kl = 0; kl < GK; ++kl) {
#pragma unroll
                for (int p = 0; p < 4; ++p) {
#pragma unroll
                  for (int j = 0; j < NG; ++j) {
                    // the first chain into class p + j: (p, j) with p == 0 or j == NG - 1
                    const bool first = kl == 0 && (p == 0 || j == NG - 1);
#ifndef NENT_M4_DBG_NOMMA
                    tc05::mma_i8_ts_desc(dacc + (uint32_t)((p + j) * U), atap + (uint32_t)((kl * NG + j) * 8), bd[p],
                                         (p & 1) ? idesc_s : idesc_u, first ? acc_first : 1u);
#endif
                  }
                  tc05::desc_advance(bd[p], 2u);  // the next K step: 32 bytes on
                }
              }
              tc05::commit(tfree_b(rs));  // the group's tap blocks may be rewritten
            }
            tc05::commit(afull_b(bsel));
          }
          tc05::commit(empty_b(ts));
        }
        __syncwarp();
      }
      // drain the last commits before the CTA can exit
      for (int t = my_tiles > NSLOT ? my_tiles - NSLOT : 0; t < my_tiles; ++t)
        mb_wait(empty_b(t % NSLOT), (uint32_t)((t / NSLOT) & 1));
      if (my_tiles > 0) {
        const int gall = my_tiles * nstr * G.ngrp;
        for (int g = gall > TRING ? gall - TRING : 0; g < gall; ++g)
          mb_wait(tfree_b(g % TRING), (uint32_t)((g / TRING) & 1));
      }
    } else if (warp >= TAP0 && warp < TAP0 + NTAP) {
      // ---------------- tap writers ----------------
      // Warp q fills TMEM lanes [32 q, 32 q + 32) of every tap-ring group: lane v's
      // 32 bytes of the Toeplitz block (j, kc) are bytes [32 kc + base, + 32) of
      // copy k of digit j, with 127 - v = base + k, base a multiple of 16.
      const int quad = warp & 3;
      const int v = 32 * quad + lane;
      const uint32_t lrow = (uint32_t)(32 * quad) << 16;
      const int kcopy = (127 - v) & (NCOPY - 1), base = (127 - v) - kcopy;
      const uint32_t rev_s = tc05::smem_u32(rev);
      const int groups = my_tiles * nstr * G.ngrp;
      // this lane's 2 x GK x NG vectors of group g (within a stream)
      auto load_group = [&](int g, int4 (&x)[GK * NG][2]) {
#pragma unroll
        for (int kl = 0; kl < GK; ++kl)
#pragma unroll
          for (int j = 0; j < NG; ++j) {
            const uint32_t src = rev_s + (uint32_t)((j * NCOPY + kcopy) * RL + 32 * (GK * g + kl) + base);
            x[kl * NG + j][0] = lds128(src);
            x[kl * NG + j][1] = lds128(src + 16);
          }
      };
      int4 x[GK * NG][2];
      int g_in = 0;  // group index within the stream
      if (groups > 0) load_group(0, x);
      for (int gt = 0; gt < groups; ++gt) {
        const int rs = gt % TRING;
        if (gt >= TRING) {
          TM(0, mb_wait(tfree_b(rs), (uint32_t)(((gt / TRING) - 1) & 1)));
          tc05::fence_after();
        }
#ifndef NENT_M4_DBG_NOTAP
#pragma unroll
        for (int b = 0; b < GK * NG; ++b) {
          const uint32_t w[8] = {(uint32_t)x[b][0].x, (uint32_t)x[b][0].y, (uint32_t)x[b][0].z, (uint32_t)x[b][0].w,
                                 (uint32_t)x[b][1].x, (uint32_t)x[b][1].y, (uint32_t)x[b][1].z, (uint32_t)x[b][1].w};
          tc05::st_x8(tbase + lrow + (uint32_t)(rs * GK * NG * 8 + b * 8), w);
        }
#endif
        if (++g_in == G.ngrp) g_in = 0;
        // the next group's vectors load while the stores drain
        if (gt + 1 < groups) load_group(g_in, x);
        tc05::wait_st();
        tc05::fence_before();
        __syncwarp();
        if (lane == 0) mb_arrive(tfull_b(rs));
      }
    } else if (warp == LOAD_WARP) {
      // ---------------- loader ----------------
      // Every tile's four raw windows go through the staging ring.  A window inside the
      // streams is ONE bulk copy issued by lane 0; a stream-edge window is copied by the whole
      // warp with cp.async at phase 0 (conv_tc05.cuh: stage_edge_window), one window at a time,
      // ahead of the converters and off their path.
      int issued = 0;
      for (int t = 0; t < my_tiles; ++t) {
        const int64_t P0 = P0_of(t);
        const bool whole = staged(P0);
#pragma unroll
        for (int s = 0; s < M; ++s) {
          const int b = issued % NSTAGE;
          if (!(pre_issue && issued < PRE)) {
            if (issued >= NSTAGE) mb_wait_sleep(sfree_b(b), (uint32_t)(((issued / NSTAGE) - 1) & 1));
            if (whole) {
              if (lane == 0) issue_window(s, P0, b);
            } else {
              tcc::stage_edge_window(stage_s + (uint32_t)b * SSTR, reinterpret_cast<const int32_t*>(A.b.p[s]), P0, A.n_in,
                                     G.nw4, G.dph[s] == 0, lane);
              asm volatile("cp.async.wait_all;" ::: "memory");
              __syncwarp();
              if (lane == 0) mb_arrive(sfull_b(b));
            }
          }
          ++issued;
        }
      }
    } else {
      // ---------------- converters ----------------
      const int cl = (warp - CONV0) * 32 + lane;  // converter lane 0 .. 63
      int consumed = 0;
      for (int t = 0; t < my_tiles; ++t) {
        const int64_t P0 = P0_of(t);
        const int ts = t % NSLOT;
        const bool whole = staged(P0);
        if (t >= NSLOT) mb_wait_sleep(empty_b(ts), (uint32_t)(((t / NSLOT) - 1) & 1));
#pragma unroll 1
        for (int s = 0; s < M; ++s) {
          const uint32_t plo = planes_s + (uint32_t)(ts * SLOTB + (2 * s) * PLANE);
          const int b = consumed % NSTAGE;
          mb_wait_sleep(sfull_b(b), (uint32_t)((consumed / NSTAGE) & 1));
          const uint32_t sbuf = stage_s + (uint32_t)b * SSTR;
          const int d = whole ? G.dph[s] : 0;  // (the loader stages a stream-edge window at phase 0)
          for (int q0 = cl; q0 < G.nw4; q0 += 4 * 32 * NCONV) {
            int4 vv[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int q = q0 + k * 32 * NCONV;
              if (q < G.nw4) {
                if (d == 0) {
                  vv[k] = lds128(sbuf + 16u * (uint32_t)q);
                } else {  // this row's window starts d words into the staged copy
                  const uint32_t* w = reinterpret_cast<const uint32_t*>(__cvta_shared_to_generic(sbuf)) + d + 4 * q;
                  vv[k] = make_int4((int)w[0], (int)w[1], (int)w[2], (int)w[3]);
                }
              }
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int q = q0 + k * 32 * NCONV;
              if (q < G.nw4) {
                uint32_t lo, hi;
                split2(vv[k], lo, hi);
                const uint32_t off = tc05::sw128(4u * (uint32_t)q);
                sts32(plo + off, lo);
                sts32(plo + (uint32_t)PLANE + off, hi);
              }
            }
          }
          fence_async_smem();  // this thread's plane writes -> the MMA's async-proxy reads
          __syncwarp();
          if (lane == 0) {
            mb_arrive(sfree_b(b));       // this warp's share of the staging buffer is read
            mb_arrive(full_b(ts, s));    // ... and of the window's two planes written
          }
          ++consumed;
        }
      }
    }
  }
#ifdef NENT_TC05_TIMERS
  // [mma: wait planes, wait taps, wait acc free, total | tap writer: wait free, total | epilogue: wait acc full, total]
  if (G.dbg && lane == 0) {
    const unsigned long long tot = (unsigned long long)(clock64() - tstart);
    if (warp == MMA_WARP) {
      for (int k = 0; k < 3; ++k) atomicAdd(G.dbg + k, (unsigned long long)tw[k]);
      atomicAdd(G.dbg + 3, tot);
    } else if (warp == TAP0) {
      atomicAdd(G.dbg + 4, (unsigned long long)tw[0]);
      atomicAdd(G.dbg + 5, tot);
    } else if (warp == 0) {
      atomicAdd(G.dbg + 6, (unsigned long long)tw[0]);
      atomicAdd(G.dbg + 7, tot);
    }
  }
#endif
  (void)tw;
  (void)tstart;
  tc05::fence_before();
  __syncthreads();
  if (threadIdx.x == 0) M4_STAMP(4);
  if (warp == MMA_WARP) {
    tc05::fence_after();
    tc05::dealloc(tbase, 512);
  }
}

}  // namespace tcm4
}  // namespace nent
