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
// around: ALL of a tile's accumulators stay resident in TMEM while the K steps
// run outermost, and the tap operand streams through a small TMEM ring:
//   * MMA N = 16: a tile is 16 blocks of 128 outputs of each stream; one
//     accumulator (stream, digit class) is 16 columns, the 2 x 5 accumulators
//     of a stream pair 160 columns, two pairs (double buffered: the epilogue
//     drains one pair while the MMA fills the other) 320 columns;
//   * the tap ring: 3 groups of 4 K steps x NG digits x 8 columns = 192 columns;
//     four "tap writer" warps (one per TMEM lane quadrant) rebuild each group's
//     Toeplitz blocks from the reversed tap digits in shared memory
//     (9 aligned LDS + 8 funnel shifts per 32-byte block and lane) and
//     tcgen05.st them; the MMA warp hands a group back with a commit.
// For K = 1024 the band costs 1152 / 1024 = 1.125x the method's MACs (a filter
// cut into 256-tap segments would pay 1.5x per segment).
//
// CTA: 16 warps, one persistent CTA per SM:
//   warps 0-7   epilogue (2 per TMEM lane quadrant, 8 accumulator columns each)
//   warps 8-11  tap writers
//   warps 12-13 converters (raw int32 window -> two byte planes per stream)
//   warp 14     loader: one thread, one bulk copy per raw window
//   warp 15     TMEM allocation; one elected lane issues every tcgen05.mma
// Extraction: L = delta mod 2^32 and M = (delta >> 16) mod 2^32 of every
// surviving stream (conv_tc05_m3.cuh), then with pivot P (the failed stream, or
// stream 0 when all four are present and the redundant one is checked)
//   d_{P+3} = L_{P+3} - (L_{P+2} << 16),  d_{P+2} = M_{P+3} - (d_{P+3} >> 16),
//   d_{P+1} = M_{P+2} - (d_{P+2} >> 16),  d_P     = M_{P+1} - (d_{P+1} >> 16).
#pragma once
#include "conv_tc05_m3.cuh"

namespace nent {
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
constexpr int U = 16;                  // 128-position blocks per tile = MMA N
constexpr int TILE = 128 * U;          // outputs per tile and stream (2048)
constexpr int NEPI = 8, NTAP = 4, NCONV = 2;
constexpr int TAP0 = NEPI, CONV0 = TAP0 + NTAP, LOAD_WARP = CONV0 + NCONV, MMA_WARP = LOAD_WARP + 1;
constexpr int NT = 32 * (MMA_WARP + 1);
static_assert(NT == 512, "16 warps");
constexpr int EC = U / (NEPI / 4);     // 8 accumulator columns per epilogue thread
constexpr int KTMAX = 1280;            // K <= 1153
constexpr int GK = 4;                  // K steps per tap-ring group
constexpr int TRING = 3;               // tap-ring groups
constexpr int NCLS5 = 5;               // accumulator classes per stream (4 data digits + 2 tap digits - 1)
constexpr int ACC0 = 192;              // accumulators: columns [192, 512)
constexpr int PAIRC = 2 * NCLS5 * U;   // 160 columns per stream pair
constexpr int PLANE = 4096;            // bytes per byte plane: 128 * (U - 1) + KTMAX = 3200, 1024-aligned
constexpr int SLOTB = 2 * M * PLANE;   // one tile slot: 4 raw streams x {lo, hi}
constexpr int NSLOT = 3;
constexpr int NSTAGE = 4;
constexpr uint32_t SSTR = 4 * (128 * (U - 1) + KTMAX) + 128;  // staging stride: the largest window + lead-in
constexpr int REVB = 2 * (KTMAX + 128 + 16);                 // reversed tap digits (2 digits)
constexpr size_t SMEM = NSLOT * (size_t)SLOTB + (size_t)NSTAGE * SSTR + REVB;
static_assert(SMEM + 1024 <= 227 * 1024, "shared memory");
constexpr int EPI_REGS = 152, OTHER_REGS = 104;
static_assert(NEPI * EPI_REGS + (16 - NEPI) * OTHER_REGS <= 16 * 128, "launch register pool");

struct Geom {
  int KT, nsteps, ngrp;  // GEMM K (bytes), K steps, tap-ring groups per stream pair
  int nw4;               // int4 words per raw window: (TILE + KT - 128) / 4
  int64_t ntiles;
  int shift;             // tiles start `shift` outputs early: row 0's windows are 16-byte aligned
  int dph[M];            // word phase of row s relative to row 0 (mod 4)
};

template <int NG>
__global__ void __launch_bounds__(NT, 1) conv_tc05_m4_kernel(const __grid_constant__ ConvArgs A,
                                                             const __grid_constant__ Geom G) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // plane full/empty [NSLOT], stage full/free [NSTAGE], tap full/free [TRING], acc full/free [2]
  __shared__ __align__(8) uint64_t bars[2 * NSLOT + 2 * NSTAGE + 2 * TRING + 4];
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t planes_s = tc05::smem_u32(smem_raw);
  const uint32_t stage_s = planes_s + (uint32_t)(NSLOT * SLOTB);
  unsigned char* rev = smem_raw + NSLOT * SLOTB + NSTAGE * SSTR;
  const uint32_t bar0 = tc05::smem_u32(bars);
  auto bar = [&](int i) { return bar0 + 8u * (uint32_t)i; };
  auto full_b = [&](int s) { return bar(s); };
  auto empty_b = [&](int s) { return bar(NSLOT + s); };
  auto sfull_b = [&](int s) { return bar(2 * NSLOT + s); };
  auto sfree_b = [&](int s) { return bar(2 * NSLOT + NSTAGE + s); };
  constexpr int B1 = 2 * NSLOT + 2 * NSTAGE;
  auto tfull_b = [&](int s) { return bar(B1 + s); };
  auto tfree_b = [&](int s) { return bar(B1 + TRING + s); };
  auto afull_b = [&](int h) { return bar(B1 + 2 * TRING + h); };
  auto afree_b = [&](int h) { return bar(B1 + 2 * TRING + 2 + h); };

  if (tid == 0) {
    for (int s = 0; s < NSLOT; ++s) {
      mb_init(full_b(s), NCONV);
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
  // the reversed taps' digits: rev[j][i] = digit_j(g[KT-1-i]), i in [0, KT + 128);
  // lane v's bytes of the Toeplitz block of K step kc are rev[j][32 kc + 127 - v + (0..31)]
  const int RL = G.KT + 128 + 16;
  {
    const uint64_t gbias = bias_of(NG);
    for (int i = tid; i < RL; i += NT) {
      const int idx = G.KT - 1 - i;
      const int64_t gv = (idx >= 0 && idx < A.K) ? ld_bits(A.g, A.g_bits, idx) : 0;
      const uint64_t d = digits_of(gv, gbias);
      for (int j = 0; j < NG; ++j) rev[j * RL + i] = (unsigned char)(d >> (8 * j));
    }
  }
  tc05::fence_before();
  __syncthreads();
  tc05::fence_after();
  if (tmem_slot != 0 || (planes_s & 1023u)) __trap();
  constexpr uint32_t tbase = 0;

  const bool verify = A.r < 0;
  const int P = verify ? 0 : A.r;  // pivot: the stream never read (or checked last)
  const int my_tiles = G.ntiles > blockIdx.x ? (int)((G.ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  const int64_t P0_first = A.y_begin - G.shift + (int64_t)blockIdx.x * TILE - (G.KT - 128);
  const int64_t P0_step = (int64_t)gridDim.x * TILE;
  auto staged = [&](int64_t P0) { return P0 >= 4 && P0 + 4 * (int64_t)G.nw4 + 4 <= A.n_in; };
  // stream i is convolved unless it is the failed one
  auto present = [&](int i) { return verify || i != P; };

  if (warp < NEPI) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(EPI_REGS));
    // ---------------- epilogue ----------------
    const int quad = warp & 3, part = warp >> 2;
    const uint32_t lrow = (uint32_t)(32 * quad) << 16;
    const int v = 32 * quad + lane;
    unsigned bad = 0;
    for (int t = 0; t < my_tiles; ++t) {
      const int64_t tile = blockIdx.x + (int64_t)t * gridDim.x;
      const int64_t o0 = tile * TILE - G.shift + 128 * (EC * part) + v;
      // the two views of every present stream's word, for this thread's 8 outputs
      uint32_t Ls[M][EC], Ms[M][EC];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        mb_wait_sleep(afull_b(h), (uint32_t)(t & 1));
        tc05::fence_after();
#pragma unroll
        for (int i2 = 0; i2 < 2; ++i2) {
          const int i = 2 * h + i2;
          if (present(i)) {
            uint32_t r[NCLS5][EC];
#pragma unroll
            for (int c = 0; c < 4 + NG - 1; ++c)
              tc05::ld_x8(tbase + lrow + (uint32_t)(ACC0 + h * PAIRC + (i2 * NCLS5 + c) * U + EC * part), r[c]);
            tc05::wait_ld();
#pragma unroll
            for (int k = 0; k < EC; ++k) {
              uint32_t q;
              const uint32_t lo = wide1(r[1][k], r[0][k], q);
              uint32_t L = lo + (r[2][k] << 16) + (r[3][k] << 24);
              uint32_t Mv = q + r[2][k] + (r[3][k] << 8);
              if (NG > 1) Mv += r[4][k] << 16;
              Ls[i][k] = L;
              Ms[i][k] = Mv;
            }
          }
        }
        tc05::fence_before();
        __syncwarp();
        if (lane == 0) mb_arrive(afree_b(h));
      }
      // recovery with pivot P; survivors P+1, P+2, P+3 (mod 4)
      auto recover = [&](auto ptag) {
        constexpr int PV = decltype(ptag)::value;
        constexpr int sa = (PV + 1) & 3, sb = (PV + 2) & 3, sc = (PV + 3) & 3;
        int32_t* yP = reinterpret_cast<int32_t*>(A.y.p[PV]);
        int32_t* ya = reinterpret_cast<int32_t*>(A.y.p[sa]);
        int32_t* yb = reinterpret_cast<int32_t*>(A.y.p[sb]);
        int32_t* yc = reinterpret_cast<int32_t*>(A.y.p[sc]);
#pragma unroll
        for (int k = 0; k < EC; ++k) {
          const uint32_t d3 = Ls[sc][k] - (Ls[sb][k] << 16);
          const uint32_t d2 = Ms[sc][k] - (uint32_t)sar16(d3);
          const uint32_t d1 = Ms[sb][k] - (uint32_t)sar16(d2);
          const uint32_t d0 = Ms[sa][k] - (uint32_t)sar16(d1);
          const int64_t o = o0 + 128 * k;
          if (o >= 0 && o < A.n_out) {
            yP[o] = (int32_t)d0;
            ya[o] = (int32_t)d1;
            yb[o] = (int32_t)d2;
            yc[o] = (int32_t)d3;
          }
          if (PV == 0) {  // (only pivot 0 is ever verified)
            // the redundant word delta_P = (d_{P+3} << 16) + d_P on its two views;
            // positions outside the rows are convolutions of zeros, consistent too
            if (verify) bad += ((Ls[0][k] ^ ((d3 << 16) + d0)) | (Ms[0][k] ^ (d3 + (uint32_t)sar16(d0)))) != 0;
          }
        }
      };
      switch (P) {
        case 0: recover(std::integral_constant<int, 0>{}); break;
        case 1: recover(std::integral_constant<int, 1>{}); break;
        case 2: recover(std::integral_constant<int, 2>{}); break;
        default: recover(std::integral_constant<int, 3>{}); break;
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
      for (int t = 0; t < my_tiles; ++t) {
        const int ts = t % NSLOT;
        mb_wait(full_b(ts), (uint32_t)((t / NSLOT) & 1));
        tc05::fence_after();
        if (elect_one()) {
          const uint32_t slot_s = planes_s + (uint32_t)(ts * SLOTB);
          for (int h = 0; h < 2; ++h) {
            // this pair's accumulators were drained (the previous tile's epilogue)
            if (t >= 1) {
              mb_wait(afree_b(h), (uint32_t)((t - 1) & 1));
              tc05::fence_after();
            }
            const bool on0 = present(2 * h), on1 = present(2 * h + 1);
            for (int g = 0; g < G.ngrp; ++g, ++gtot) {
              const int rs = gtot % TRING;
              mb_wait(tfull_b(rs), (uint32_t)((gtot / TRING) & 1));
              tc05::fence_after();
#pragma unroll
              for (int kl = 0; kl < GK; ++kl) {
                const uint32_t kc2 = 2u * (uint32_t)(GK * g + kl);  // descriptor start advance (16-byte units)
                const uint32_t acc_first = (g == 0 && kl == 0) ? 0u : 1u;
#pragma unroll
                for (int i2 = 0; i2 < 2; ++i2) {
                  if (i2 == 0 ? on0 : on1) {
                    const int i = 2 * h + i2, im1 = (i + M - 1) & 3;
#pragma unroll
                    for (int p = 0; p < 4; ++p) {
                      // data digit p of eps_i: bytes of c_i (p < 2) or of c_{i-1} (p >= 2)
                      const int raw = p < 2 ? i : im1;
                      const uint32_t blo = tc05::desc_sw128_lo(slot_s + (uint32_t)((2 * raw + (p & 1)) * PLANE)) + kc2;
#pragma unroll
                      for (int j = 0; j < NG; ++j) {
                        const uint32_t d = tbase + (uint32_t)(ACC0 + h * PAIRC + (i2 * NCLS5 + p + j) * U);
                        const uint32_t a = tbase + (uint32_t)(rs * GK * NG * 8 + (kl * NG + j) * 8);
                        // the first chain into class p + j: (p, j) with p == 0 or j == NG - 1
                        const bool first = p == 0 || j == NG - 1;
                        tc05::mma_i8_ts_lo(d, a, blo, (p & 1) ? idesc_s : idesc_u, first ? acc_first : 1u);
                      }
                    }
                  }
                }
              }
              tc05::commit(tfree_b(rs));  // the group's tap blocks may be rewritten
            }
            tc05::commit(afull_b(h));
          }
          tc05::commit(empty_b(ts));
        }
        __syncwarp();
      }
      // drain the last commits before the CTA can exit
      for (int t = my_tiles > NSLOT ? my_tiles - NSLOT : 0; t < my_tiles; ++t)
        mb_wait(empty_b(t % NSLOT), (uint32_t)((t / NSLOT) & 1));
      if (my_tiles > 0) {
        const int gall = my_tiles * 2 * G.ngrp;
        for (int g = gall > TRING ? gall - TRING : 0; g < gall; ++g)
          mb_wait(tfree_b(g % TRING), (uint32_t)((g / TRING) & 1));
      }
    } else if (warp >= TAP0 && warp < TAP0 + NTAP) {
      // ---------------- tap writers ----------------
      // Warp q builds TMEM lanes [32 q, 32 q + 32) of every tap-ring group: lane v's
      // 32 bytes of the Toeplitz block (j, kc) start at rev[j][32 kc + 127 - v].
      const int quad = warp & 3;
      const int v = 32 * quad + lane;
      const uint32_t lrow = (uint32_t)(32 * quad) << 16;
      const int s0 = 127 - v;                    // byte offset of K step 0
      const uint32_t sh = 8u * (uint32_t)(s0 & 3);
      const int groups = my_tiles * 2 * G.ngrp;
      int g_in = 0;                              // group index within the stream pair
      for (int gt = 0; gt < groups; ++gt) {
        const int rs = gt % TRING;
        if (gt >= TRING) {
          mb_wait_sleep(tfree_b(rs), (uint32_t)(((gt / TRING) - 1) & 1));
          tc05::fence_after();
        }
#pragma unroll
        for (int kl = 0; kl < GK; ++kl) {
          const int kc = GK * g_in + kl;
#pragma unroll
          for (int j = 0; j < NG; ++j) {
            const uint32_t* src = reinterpret_cast<const uint32_t*>(rev + j * RL + ((32 * kc + s0) & ~3));
            uint32_t x[9], w[8];
#pragma unroll
            for (int c = 0; c < 9; ++c) x[c] = src[c];
#pragma unroll
            for (int c = 0; c < 8; ++c) w[c] = __funnelshift_r(x[c], x[c + 1], sh);
            tc05::st_x8(tbase + lrow + (uint32_t)(rs * GK * NG * 8 + (kl * NG + j) * 8), w);
          }
        }
        tc05::wait_st();
        tc05::fence_before();
        __syncwarp();
        if (lane == 0) mb_arrive(tfull_b(rs));
        if (++g_in == G.ngrp) g_in = 0;
      }
    } else if (warp == LOAD_WARP) {
      // ---------------- loader ----------------
      if (lane == 0) {
        int64_t P0 = P0_first;
        int issued = 0;
        const uint32_t winb = 16u * (uint32_t)G.nw4;
        for (int t = 0; t < my_tiles; ++t, P0 += P0_step) {
          if (!staged(P0)) continue;
#pragma unroll
          for (int s = 0; s < M; ++s) {
            const int b = issued % NSTAGE;
            if (issued >= NSTAGE) mb_wait_sleep(sfree_b(b), (uint32_t)(((issued / NSTAGE) - 1) & 1));
            const int d = G.dph[s];
            const char* src = reinterpret_cast<const char*>(reinterpret_cast<const int32_t*>(A.b.p[s]) + P0 - d);
            const uint32_t bytes = winb + (d ? 16u : 0u);
            mb_expect_tx(sfull_b(b), bytes);
            bulk_g2s(stage_s + (uint32_t)b * SSTR, src, bytes, sfull_b(b));
            ++issued;
          }
        }
      }
    } else {
      // ---------------- converters ----------------
      const int cl = (warp - CONV0) * 32 + lane;  // converter lane 0 .. 63
      int64_t P0 = P0_first;
      int consumed = 0;
      for (int t = 0; t < my_tiles; ++t, P0 += P0_step) {
        const int ts = t % NSLOT;
        const bool fast = staged(P0);
        if (t >= NSLOT) mb_wait_sleep(empty_b(ts), (uint32_t)(((t / NSLOT) - 1) & 1));
#pragma unroll 1
        for (int s = 0; s < M; ++s) {
          const uint32_t plo = planes_s + (uint32_t)(ts * SLOTB + (2 * s) * PLANE);
          if (fast) {
            const int b = consumed % NSTAGE;
            mb_wait_sleep(sfull_b(b), (uint32_t)((consumed / NSTAGE) & 1));
            const uint32_t sbuf = stage_s + (uint32_t)b * SSTR;
            const int d = G.dph[s];
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
            __syncwarp();
            if (lane == 0) mb_arrive(sfree_b(b));
            ++consumed;
          } else {
            const int32_t* bp = reinterpret_cast<const int32_t*>(A.b.p[s]);
            for (int q = cl; q < G.nw4; q += 32 * NCONV) {
              const int64_t x0 = P0 + 4 * (int64_t)q;
              int e[4];
#pragma unroll
              for (int k = 0; k < 4; ++k) e[k] = (x0 + k >= 0 && x0 + k < A.n_in) ? __ldg(bp + x0 + k) : 0;
              uint32_t lo, hi;
              split2(make_int4(e[0], e[1], e[2], e[3]), lo, hi);
              const uint32_t off = tc05::sw128(4u * (uint32_t)q);
              sts32(plo + off, lo);
              sts32(plo + (uint32_t)PLANE + off, hi);
            }
          }
        }
        fence_async_smem();  // this thread's plane writes -> the MMA's async-proxy reads
        __syncwarp();
        if (lane == 0) mb_arrive(full_b(ts));
      }
    }
  }
  tc05::fence_before();
  __syncthreads();
  if (warp == MMA_WARP) {
    tc05::fence_after();
    tc05::dealloc(tbase, 512);
  }
}

}  // namespace tcm4
}  // namespace nent
