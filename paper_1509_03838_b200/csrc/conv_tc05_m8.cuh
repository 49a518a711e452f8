// conv_tc05_m8.cuh -- the cfg5 convolution stage: convolution + extraction of
// m = 8 ALREADY ENTANGLED int32 streams (the stream-per-GPU workers' chain
// words: entangle -> scale -> add -> permute happened upstream) on the
// 5th-generation tensor cores, replacing a plain tensor-core convolution
// followed by a separate extract pass over HBM.  Reference semantics:
// ops._circ_conv_rows on the zero-padded rows (ops.py:158-172),
// then codec.disentangle (codec.py:89-131, _kernels.py:33-67).
//
// The rows are arbitrary int16-range words x = lo + 256 hi (low byte unsigned,
// high byte signed), so each row is split once into its two byte planes and a
// row's word is delta = R_0 + 256 R_1 from two K chains (one tap digit: taps in
// [-127, 127]); |delta| <= 32639 * 127 * 257 < 2^31, so every word and the whole
// recovery fit 32-bit arithmetic when (m - 1) l <= 32.
//
// The rows are convolved in the order P+1, ..., P+7 (then P, when all eight are
// present and the redundant one is checked; P the failed row or 0), each
// thread keeps the seven words of its 16 positions and then runs the
// reference's recovery (recover.cuh): the pivot's low (m-1) l bits give
// d_{P-1}, the rest follow backwards, d_{j-1} = (delta_j - d_j) >> l.
//
// The kernel is HBM-bound (two 12-MMA chains per row and tile): what matters is
// that delta never goes to HBM.  CTA: 16 warps, one persistent CTA per SM, a
// tile is 32 blocks of 128 outputs (MMA 128 x 32 x 32) of each row:
//   warps 0-7   epilogue (2 per TMEM lane quadrant, 16 accumulator columns each)
//   warps 8-13  converters (raw int32 window -> two byte planes per row)
//   warp 14     loader: lane 0 issues one bulk copy per raw window; a stream-edge window (not
//               wholly inside the stream) is staged by the whole warp with cp.async + zero fill
//   warp 15     TMEM allocation; one elected lane issues every tcgen05.mma
// TMEM: tap digits in columns [0, 96), a ring of 13 accumulator slots of 32.
#pragma once
#include "conv_tc05_m3.cuh"

namespace nent {
namespace tcm8 {

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
using tcm3::split2;

constexpr int M = 8;                   // rows
constexpr int U = 32;                  // 128-position blocks per tile = MMA N
constexpr int TILE = 128 * U;          // outputs per tile and row (4096)
constexpr int NEPI = 8, NCONV = 6;
constexpr int CONV0 = NEPI, LOAD_WARP = CONV0 + NCONV, MMA_WARP = LOAD_WARP + 1;
constexpr int NT = 32 * (MMA_WARP + 1);
static_assert(NT == 512, "16 warps");
constexpr int EC = U / (NEPI / 4);     // 16 accumulator columns per epilogue thread
constexpr int KTMAX = 384;             // K <= 257
constexpr int TAPCOLS = 96;            // one tap digit: 12 K steps x 8 columns
constexpr int RING0 = TAPCOLS;
constexpr int SLOTS = (512 - RING0) / U;  // 13
constexpr int PLANE = 5120;            // bytes per byte plane: TILE + 256 = 4352, 1024-aligned
constexpr int SLOTB = 2 * M * PLANE;   // one tile slot: 8 rows x {lo, hi}
constexpr int NSLOT = 2;
constexpr int NSTAGE = 3;
constexpr int NW4MAX = (TILE + KTMAX - 128) / 4;             // 1088 int4 per raw window
constexpr uint32_t SSTR = 16 * NW4MAX + 128;
constexpr size_t SMEM = NSLOT * (size_t)SLOTB + (size_t)NSTAGE * SSTR;
static_assert(SMEM + 1024 <= 227 * 1024, "shared memory");
constexpr int EPI_REGS = 184, OTHER_REGS = 72;
static_assert(NEPI * EPI_REGS + (16 - NEPI) * OTHER_REGS <= 16 * 128, "launch register pool");

struct Geom {
  int KT, nsteps;
  int nw4;               // int4 words per raw window: (TILE + KT - 128) / 4
  int64_t ntiles;
  int64_t tile_off;  // CTA b's tiles are (tile_off + b + k * grid) mod ntiles
  int shift;             // tiles start `shift` outputs early: row 0's windows are 16-byte aligned
  int dph[M];            // word phase of row s relative to row 0 (mod 4)
};

template <int NSTEPS>
__global__ void __launch_bounds__(NT, 1) conv_tc05_m8_kernel(const __grid_constant__ ConvArgs A,
                                                             const __grid_constant__ Geom G) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // plane full/empty [NSLOT], stage full/free [NSTAGE], acc full/empty [SLOTS]
  __shared__ __align__(8) uint64_t bars[2 * NSLOT + 2 * NSTAGE + 2 * SLOTS];
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t planes_s = tc05::smem_u32(smem_raw);
  const uint32_t stage_s = planes_s + (uint32_t)(NSLOT * SLOTB);
  const uint32_t bar0 = tc05::smem_u32(bars);
  auto bar = [&](int i) { return bar0 + 8u * (uint32_t)i; };
  auto full_b = [&](int s) { return bar(s); };
  auto empty_b = [&](int s) { return bar(NSLOT + s); };
  auto sfull_b = [&](int s) { return bar(2 * NSLOT + s); };
  auto sfree_b = [&](int s) { return bar(2 * NSLOT + NSTAGE + s); };
  constexpr int B1 = 2 * NSLOT + 2 * NSTAGE;
  auto accf_b = [&](int s) { return bar(B1 + s); };
  auto acce_b = [&](int s) { return bar(B1 + SLOTS + s); };

  if (tid == 0) {
    for (int s = 0; s < NSLOT; ++s) {
      mb_init(full_b(s), NCONV);
      mb_init(empty_b(s), 1);
    }
    for (int s = 0; s < NSTAGE; ++s) {
      mb_init(sfull_b(s), 1);
      mb_init(sfree_b(s), NCONV);
    }
    for (int s = 0; s < SLOTS; ++s) {
      mb_init(accf_b(s), 1);
      mb_init(acce_b(s), NEPI);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == MMA_WARP) tc05::alloc(&tmem_slot, 512);
  tc05::fence_before();
  __syncthreads();
  tc05::fence_after();
  if (tmem_slot != 0 || (planes_s & 1023u)) __trap();
  constexpr uint32_t tbase = 0;
  const int my_tiles = G.ntiles > blockIdx.x ? (int)((G.ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  // The CTA's tiles (tile_off + blockIdx.x + k * gridDim.x) mod ntiles are processed in the
  // order k = 1, 2, ..., 0: the stream-edge tiles (staged by the loader warp with cp.async)
  // sit on the CTAs with one tile fewer where they can (conv_common.cuh: edge_tile_offset)
  // and are never a CTA's first tile.
  auto tile_ord = [&](int t) -> int64_t {
    int64_t j = G.tile_off + blockIdx.x + (int64_t)(t + 1 < my_tiles ? t + 1 : 0) * gridDim.x;
    return j >= G.ntiles ? j - G.ntiles : j;
  };
  auto P0_of = [&](int t) -> int64_t { return A.y_begin - G.shift + tile_ord(t) * TILE - (G.KT - 128); };
  auto staged = [&](int64_t P0) { return P0 >= 4 && P0 + 4 * (int64_t)G.nw4 + 4 <= A.n_in; };
  {
    // the reversed taps (one signed digit), staged once in the (still free)
    // last plane slot: rev[i] = g[KT-1-i], A[v][k] = rev[k - v + 127]
    const int RL = G.KT + 128;
    unsigned char* rev = smem_raw + (NSLOT - 1) * SLOTB;
    for (int i = tid; i < RL; i += NT) {
      const int idx = G.KT - 1 - i;
      const int64_t gv = (idx >= 0 && idx < A.K) ? ld_bits(A.g, A.g_bits, idx) : 0;
      rev[i] = (unsigned char)(uint64_t)gv;
    }
    __syncthreads();
    const int v = 32 * (warp & 3) + lane;
    for (int blk = warp >> 2; blk < NSTEPS; blk += NT / 128) {
      const unsigned char* r = rev + 32 * blk - v + 127;
      uint32_t w[8];
#pragma unroll
      for (int c = 0; c < 8; ++c)
        w[c] = (uint32_t)r[4 * c] | ((uint32_t)r[4 * c + 1] << 8) | ((uint32_t)r[4 * c + 2] << 16) |
               ((uint32_t)r[4 * c + 3] << 24);
      tc05::st_x8(tbase + ((uint32_t)(32 * (warp & 3)) << 16) + 8u * (uint32_t)blk, w);
    }
    tc05::wait_st();
    tc05::fence_before();
    __syncthreads();  // also: the taps' staging bytes are dead before a converter writes that plane slot
    tc05::fence_after();
  }
  const bool verify = A.r < 0;
  const int P = verify ? 0 : A.r;  // pivot: the row never read (or checked last)
  const int nstr = verify ? M : M - 1;
  const int spt = 2 * nstr;        // ring slots per tile (two digit classes per row)

  if (warp < NEPI) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(EPI_REGS));
    // ---------------- epilogue ----------------
    const int quad = warp & 3, part = warp >> 2;
    const uint32_t lrow = (uint32_t)(32 * quad) << 16;
    const int v = 32 * quad + lane;
    const int l = A.l, low = (M - 1) * l;
    unsigned bad = 0;
    int kslot = 0;
    // the word of the next row for this thread's 16 positions: delta = R_0 + 256 R_1
    auto word = [&](uint32_t (&w)[EC]) {
      const int r0 = kslot % SLOTS, r1 = (kslot + 1) % SLOTS;
      mb_wait_sleep(accf_b(r0), (uint32_t)((kslot / SLOTS) & 1));
      mb_wait_sleep(accf_b(r1), (uint32_t)(((kslot + 1) / SLOTS) & 1));
      tc05::fence_after();
      uint32_t a[EC], b[EC];
      tc05::ld_x16(tbase + lrow + (uint32_t)(RING0 + r0 * U + EC * part), a);
      tc05::ld_x16(tbase + lrow + (uint32_t)(RING0 + r1 * U + EC * part), b);
      tc05::wait_ld();
      tc05::fence_before();
      __syncwarp();
      if (lane == 0) {
        mb_arrive(acce_b(r0));
        mb_arrive(acce_b(r1));
      }
      kslot += 2;
#pragma unroll
      for (int k = 0; k < EC; ++k) w[k] = a[k] + (b[k] << 8);
    };
    for (int t = 0; t < my_tiles; ++t) {
      const int64_t tile = tile_ord(t);
      const int64_t o0 = tile * TILE - G.shift + 128 * (EC * part) + v;
      uint32_t rot[M - 1][EC];  // rot[s] = delta_{(P+1+s) mod m}
#pragma unroll
      for (int s = 0; s < M - 1; ++s) word(rot[s]);
      uint32_t pw[EC];
      if (verify) word(pw);  // delta_P, the redundant word
#pragma unroll
      for (int k = 0; k < EC; ++k) {
        // pivot (recover.cuh): low (m-1) l bits of sum_t (-1)^t rot[t] << (m-2-t) l
        uint32_t acc = rot[0][k] << ((M - 2) * l);
#pragma unroll
        for (int s = 1; s < M - 1; ++s) {
          const uint32_t term = rot[s][k] << ((M - 2 - s) * l);
          acc = (s & 1) ? acc - term : acc + term;
        }
        int32_t o[M];  // o[s] = d_{(P+s) mod m}
        o[M - 1] = ((int32_t)(acc << (32 - low))) >> (32 - low);  // m even: d_{P-1} = +v
#pragma unroll
        for (int s = M - 1; s >= 1; --s) o[s - 1] = ((int32_t)rot[s - 1][k] - o[s]) >> l;
        const int64_t pos = o0 + 128 * k;
        if (pos >= 0 && pos < A.n_out) {
#pragma unroll
          for (int s = 0; s < M; ++s) reinterpret_cast<int32_t*>(A.y.p[(P + s) & (M - 1)])[pos] = o[s];
        }
        // the pivot's own word must be (d_{P-1} << l) + d_P (codec.py:57-66)
        if (verify) bad += pw[k] != (((uint32_t)o[M - 1] << l) + (uint32_t)o[0]);
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
      int kslot = 0;
      for (int t = 0; t < my_tiles; ++t) {
        const int ts = t % NSLOT;
        mb_wait(full_b(ts), (uint32_t)((t / NSLOT) & 1));
        tc05::fence_after();
        if (elect_one()) {
          const uint32_t slot_s = planes_s + (uint32_t)(ts * SLOTB);
          for (int si = 0; si < nstr; ++si) {
            const int i = (P + 1 + si) & (M - 1);
#pragma unroll
            for (int p = 0; p < 2; ++p, ++kslot) {  // class p: the chain of data digit p
              const int rs = kslot % SLOTS, use = kslot / SLOTS;
              if (use >= 1) {
                mb_wait(acce_b(rs), (uint32_t)((use - 1) & 1));
                tc05::fence_after();
              }
              const uint32_t d = tbase + (uint32_t)(RING0 + rs * U);
              uint64_t bd = tc05::desc_sw128_from_lo(tc05::desc_sw128_lo(slot_s + (uint32_t)((2 * i + p) * PLANE)));
#pragma unroll
              for (int kc = 0; kc < NSTEPS; ++kc) {
                tc05::mma_i8_ts_desc(d, tbase + 8u * kc, bd, p ? idesc_s : idesc_u, kc ? 1u : 0u);
                tc05::desc_advance(bd, 2u);
              }
              tc05::commit(accf_b(rs));
            }
          }
          tc05::commit(empty_b(ts));
        }
        __syncwarp();
      }
      // drain the last commits before the CTA can exit
      for (int t = my_tiles > NSLOT ? my_tiles - NSLOT : 0; t < my_tiles; ++t)
        mb_wait(empty_b(t % NSLOT), (uint32_t)((t / NSLOT) & 1));
      (void)spt;
    } else if (warp == LOAD_WARP) {
      // ---------------- loader ----------------
      // Every tile's eight raw windows go through the staging ring: a window inside the
      // streams is ONE bulk copy issued by lane 0, a stream-edge window is copied by the
      // whole warp with cp.async at phase 0 (conv_tc05.cuh: stage_edge_window).
      int issued = 0;
      const uint32_t winb = 16u * (uint32_t)G.nw4;
      for (int t = 0; t < my_tiles; ++t) {
        const int64_t P0 = P0_of(t);
        const bool whole = staged(P0);
        for (int s = 0; s < M; ++s) {
          const int b = issued % NSTAGE;
          if (issued >= NSTAGE) mb_wait_sleep(sfree_b(b), (uint32_t)(((issued / NSTAGE) - 1) & 1));
          const int d = G.dph[s];
          if (whole) {
            if (lane == 0) {
              const char* src = reinterpret_cast<const char*>(reinterpret_cast<const int32_t*>(A.b.p[s]) + P0 - d);
              const uint32_t bytes = winb + (d ? 16u : 0u);
              mb_expect_tx(sfull_b(b), bytes);
              bulk_g2s(stage_s + (uint32_t)b * SSTR, src, bytes, sfull_b(b));
            }
          } else {
            tcc::stage_edge_window(stage_s + (uint32_t)b * SSTR, reinterpret_cast<const int32_t*>(A.b.p[s]), P0, A.n_in,
                                   G.nw4, d == 0, lane);
            asm volatile("cp.async.wait_all;" ::: "memory");
            __syncwarp();
            if (lane == 0) mb_arrive(sfull_b(b));
          }
          ++issued;
        }
      }
    } else {
      // ---------------- converters ----------------
      const int cl = (warp - CONV0) * 32 + lane;  // converter lane 0 .. 191
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
          for (int q0 = cl; q0 < G.nw4; q0 += 3 * 32 * NCONV) {
            int4 vv[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
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
            for (int k = 0; k < 3; ++k) {
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

}  // namespace tcm8
}  // namespace nent
