// conv_tc05_m3.cuh -- the cfg2 hot path: fused entangle -> convolution ->
// extract of m = 3 int32 streams on the 5th-generation tensor cores, for a
// byte-aligned entangling shift (l = 16, the (3,48,16,16) geometry) and
// samples with |c| <= 0x7F7F.  Reference semantics: codec.entangle
// (codec.py:57-72), ops._circ_conv_rows on the zero-padded streams
// (ops.py:158-172), codec.disentangle (codec.py:89-131).
//
// Entangling on load, by digit placement.  With l = 16 the entangled word
// eps_i = (c_{i-1} << 16) + c_i of samples |c| <= 0x7F7F has, as its four
// unsigned base-256 digits (u = eps + 0x80808080, the operand the MMA reads),
// exactly the two bytes of c_i + 0x8080 followed by the two bytes of
// c_{i-1} + 0x8080: no carry crosses the 16-bit boundary.  So the producers
// split each raw stream of a tile ONCE into two byte planes, and the MMA
// convolves eps_i by reading planes {lo(c_i), hi(c_i), lo(c_{i-1}),
// hi(c_{i-1})} -- the four digit planes of the entangled word.  The tensor
// core does the full entangled arithmetic (4 data digits x NG tap digits per
// stream, the same MACs as the generic kernel); only the digit extraction is
// shared between the two streams a sample is entangled into.
//
// Extraction in registers with no shared-memory stash: the MMA issues the
// classes of the two recovery streams interleaved (class c of stream P+1,
// then class c of stream P+2), so every epilogue thread holds both deltas of
// its 16 outputs at once and recovers d_P, d_{P+1}, d_{P+2}; with failed =
// None the redundant stream P follows and is checked against the recovery.
//
// CTA: 16 warps = 4 warpgroups, one persistent CTA per SM; a tile is 64
// blocks of 128 outputs (MMA N = 64) of each stream.
//   warps 0-7   epilogue (2 per TMEM lane quadrant, 32 accumulator columns
//               each; 184 registers after setmaxnreg)
//   warps 8-14  producers: each warp TMA-copies its own 5 KB share of every
//               raw int32 window into its own staging ring and splits it into
//               byte planes (2 tile slots)
//   warp 15     TMEM allocation; one elected lane issues every tcgen05.mma
// TMEM: [0, 8*NG*NSTEPS) the Toeplitz tap digits (A operand), [192, 512) a
// ring of 5 accumulator slots of 64 columns.
#pragma once
#include "conv_tc05.cuh"

#include <cstdio>

namespace nent {
namespace tcm3 {

using tcc::bias_of;
using tcc::bulk_g2s;
using tcc::digits_of;
using tcc::elect_one;
using tcc::fence_async_smem;
using tcc::mb_arrive;
using tcc::mb_expect_tx;
using tcc::mb_init;
using tcc::mb_wait;
using tcc::mb_wait_sleep;
using tcc::ld_cols;
using tcc::sts32;

constexpr int U = 64;                  // 128-position blocks per tile = MMA N
constexpr int TILE = 128 * U;          // outputs per tile and stream
constexpr int NEPI = 8;                // epilogue warps (2 per TMEM lane quadrant)
constexpr int NPROD = 7;               // producer warps
constexpr int MMA_WARP = NEPI + NPROD; // 15: the highest warp id has issue priority
constexpr int NT = 32 * (NEPI + NPROD + 1);
constexpr int EC = U / (NEPI / 4);     // 32 accumulator columns per epilogue thread
// Each producer warp owns a contiguous 1/NPROD of every raw stream's window
// (WW int4 per lane, 5 KB per warp) and stages it through its own TMA ring of
// NSTAGE chunks: the warps never wait for each other.
constexpr int WW = 10;                 // int4 words per lane and raw-stream window
constexpr int NWP = WW * 32 * NPROD;   // int4 words staged per raw stream and tile (2240)
#ifndef NENT_M3_NSTAGE
#define NENT_M3_NSTAGE 3
#endif
#ifndef NENT_M3_NSLOT
#define NENT_M3_NSLOT 2
#endif
constexpr int NSLOT = NENT_M3_NSLOT;   // tile slots of byte planes: producers run up to NSLOT-1 tiles ahead
constexpr int NSTAGE = NENT_M3_NSTAGE;  // per-warp staging ring depth (NSTAGE-1 units in flight)
constexpr uint32_t WCHUNK = WW * 32 * 16;  // bytes per warp and unit (5120)
constexpr int PLANE = 9216;            // bytes per byte plane: >= 4 * NWP, 1024-aligned
constexpr int SLOTB = 6 * PLANE;       // one tile slot: 3 raw streams x {lo, hi}
constexpr int TAPCOLS = 192;
constexpr int RING0 = TAPCOLS;
constexpr int SLOTS = (512 - RING0) / U;  // 5
constexpr int LAUNCH_REGS = 128;       // 65536 / 512
constexpr int EPI_REGS = 184, PROD_REGS = 72;
static_assert(NEPI * 32 * EPI_REGS + (NPROD + 1) * 32 * PROD_REGS <= NT * LAUNCH_REGS, "launch register pool");
static_assert(NEPI % 4 == 0 && (NPROD + 1) % 4 == 0, "setmaxnreg acts on whole warpgroups");
static_assert(4 * NWP >= TILE + 256, "a staged window covers the tile plus the K <= 257 halo");
static_assert(4 * NWP <= PLANE, "a staged window fits its plane");
constexpr uint32_t SSTR = WCHUNK + 128;  // staging slot stride: a chunk plus one int4 of lead-in
constexpr size_t SMEM = NSLOT * (size_t)SLOTB + (size_t)NPROD * NSTAGE * SSTR;  // 220,800 B
static_assert(SMEM + 1024 <= 227 * 1024, "shared memory");

struct Geom {
  int KT, nsteps;
  int64_t ntiles;
  int shift;   // tiles start `shift` outputs early: row 0's windows are 16-byte aligned
  int dph[3];  // word phase of row s relative to row 0 (mod 4): its windows are
               // copied from dph[s] words earlier and read shifted in shared memory
  unsigned long long* dbg;  // role timers (profiling builds, -DNENT_TC05_TIMERS)
};

// TM(slot, stmt): add stmt's cycles to tw[slot] in timer builds
#ifdef NENT_TC05_TIMERS
#define TM(i, ...)                    \
  {                                   \
    const long long t0_ = clock64();  \
    __VA_ARGS__;                      \
    tw[i] += clock64() - t0_;         \
  }
#else
#define TM(i, ...) \
  { __VA_ARGS__; }
#endif

// u = c + 0x8080 of 4 consecutive samples -> the lo-byte and hi-byte plane words
__device__ __forceinline__ void split2(int4 v, uint32_t& lo, uint32_t& hi) {
  const uint32_t u0 = (uint32_t)v.x + 0x8080u, u1 = (uint32_t)v.y + 0x8080u;
  const uint32_t u2 = (uint32_t)v.z + 0x8080u, u3 = (uint32_t)v.w + 0x8080u;
  const uint32_t t01 = __byte_perm(u0, u1, 0x5140), t23 = __byte_perm(u2, u3, 0x5140);
  lo = __byte_perm(t01, t23, 0x5410);
  hi = __byte_perm(t01, t23, 0x7632);
}

// this thread's EC accumulator columns of one slot, as x16 loads (16-register
// blocks keep the register allocation flexible; x32 needs 32 aligned ones)
template <int N>
__device__ __forceinline__ void ld_slot(uint32_t taddr, uint32_t (&r)[N]) {
#pragma unroll
  for (int k = 0; k < N / 16; ++k) tc05::ld_x16(taddr + 16u * k, *reinterpret_cast<uint32_t(*)[16]>(r + 16 * k));
}

// mbarrier wait that suspends the warp in hardware until the phase completes
// (or a 20 us hint expires) instead of polling with try_wait + nanosleep
__device__ __forceinline__ void mb_wait_suspend(uint32_t mb, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n M3_WAITS_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      " @!p bra M3_WAITS_%=;\n}" ::"r"(mb), "r"(parity), "r"(20000) : "memory");
}

// Register pins: an empty volatile asm that reads and rewrites x, ordered
// with the other volatile asm (the next TMEM drain): the class fold before it
// completes first, instead of being sunk below the next drain (which would
// keep two classes' registers live and spill).
__device__ __forceinline__ void pin(uint64_t& x) { asm volatile("" : "+l"(x)); }
__device__ __forceinline__ void pin(uint32_t& x) { asm volatile("" : "+r"(x)); }

// acc += (int64)r * 2^(8c + s0) (mod 2^64) with a compile-time weight: one
// IMAD.WIDE for weights < 2^31, one IMAD on the high word otherwise
template <int SH>
__device__ __forceinline__ void add_shifted(uint64_t& acc, uint32_t r) {
  if (SH < 31) {
    acc += (uint64_t)((int64_t)(int32_t)r * (int64_t)(1ll << SH));
  } else {
    acc += (uint64_t)(r << (SH - 32)) << 32;
  }
}
template <int SH>
__device__ __forceinline__ void sub_shifted(uint64_t& acc, uint32_t r) {
  if (SH < 31) {
    acc += (uint64_t)((int64_t)(int32_t)r * -(int64_t)(1ll << SH));
  } else {
    acc -= (uint64_t)(r << (SH - 32)) << 32;
  }
}
// class c of delta_A and delta_B into C = (delta_A << 16) - delta_B and the
// low word of delta_A
template <int CL, int N>
__device__ __forceinline__ void fold_ab(uint64_t (&C)[N], uint32_t (&lowA)[N], const uint32_t (&rA)[N],
                                        const uint32_t (&rB)[N]) {
#pragma unroll
  for (int i = 0; i < N; ++i) {
    add_shifted<8 * CL + 16>(C[i], rA[i]);
    sub_shifted<8 * CL>(C[i], rB[i]);
    if (CL < 4) lowA[i] += rA[i] << (8 * CL);
  }
}
template <int CL, int N>
__device__ __forceinline__ void fold_a(uint64_t (&C)[N], uint32_t (&lowA)[N], const uint32_t (&rA)[N]) {
#pragma unroll
  for (int i = 0; i < N; ++i) {
    add_shifted<8 * CL + 16>(C[i], rA[i]);
    if (CL < 4) lowA[i] += rA[i] << (8 * CL);
  }
}
template <int CL, int N>
__device__ __forceinline__ void fold_b(uint64_t (&C)[N], const uint32_t (&rB)[N]) {
#pragma unroll
  for (int i = 0; i < N; ++i) sub_shifted<8 * CL>(C[i], rB[i]);
}
template <int CL, int N>
__device__ __forceinline__ void fold_p(uint64_t (&acc)[N], const uint32_t (&r)[N]) {
#pragma unroll
  for (int i = 0; i < N; ++i) add_shifted<8 * CL>(acc[i], r[i]);
}

// the chains (data digit p, tap digit j) of digit class c, in a fixed order
template <int NG, typename F>
__device__ __forceinline__ void for_class(int c, F&& f) {
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int j = c - p;
    if (j >= 0 && j < NG) f(p, j);
  }
}

template <int NG, int NSTEPS>
__global__ void __launch_bounds__(NT, 1) conv_tc05_m3_kernel(const __grid_constant__ ConvArgs A,
                                                             const __grid_constant__ Geom G) {
  constexpr int NCLS = 4 + NG - 1;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // full[2], empty[2], stage full[3], stage empty[3], acc full[5], acc empty[5]
  __shared__ __align__(8) uint64_t bars[2 * NSLOT + NPROD * NSTAGE + 2 * SLOTS];
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t planes_s = tc05::smem_u32(smem_raw);
  const uint32_t stage_s = planes_s + (uint32_t)(NSLOT * SLOTB);
  const uint32_t bar0 = tc05::smem_u32(bars);
  auto full_b = [&](int s) { return bar0 + 8u * (uint32_t)s; };
  auto empty_b = [&](int s) { return bar0 + 8u * (uint32_t)(NSLOT + s); };
  constexpr int B0 = 2 * NSLOT;
  auto stg_b = [&](int w, int s) { return bar0 + 8u * (uint32_t)(B0 + w * NSTAGE + s); };  // warp w's ring
  auto accf_b = [&](int s) { return bar0 + 8u * (uint32_t)(B0 + NPROD * NSTAGE + s); };
  auto acce_b = [&](int s) { return bar0 + 8u * (uint32_t)(B0 + NPROD * NSTAGE + SLOTS + s); };

  if (tid == 0) {
    for (int s = 0; s < NSLOT; ++s) {
      mb_init(full_b(s), NPROD);  // one arrival per producer warp and tile
      mb_init(empty_b(s), 1);
    }
    for (int s = 0; s < NPROD * NSTAGE; ++s) mb_init(stg_b(0, s), 1);
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
  {
    // the reversed taps' digits, staged once in the (still free) staging ring:
    // rev[j][i] = digit_j(g[KT-1-i]), A_j[v][k] = rev[j][k - v + 127]
    const int RL = G.KT + 128;
    unsigned char* rev = smem_raw + NSLOT * SLOTB;
    const uint64_t gbias = bias_of(NG);
    for (int i = tid; i < RL; i += NT) {
      const int idx = G.KT - 1 - i;
      const int64_t gv = (idx >= 0 && idx < A.K) ? ld_bits(A.g, A.g_bits, idx) : 0;
      const uint64_t d = digits_of(gv, gbias);
      for (int j = 0; j < NG; ++j) rev[j * RL + i] = (unsigned char)(d >> (8 * j));
    }
    __syncthreads();
    const int v = 32 * (warp & 3) + lane;
    for (int blk = warp >> 2; blk < NG * NSTEPS; blk += NT / 128) {
      const int j = blk / NSTEPS, kc = blk % NSTEPS;
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
  const bool verify = A.r < 0;
  const int P = verify ? 0 : A.r;  // pivot: the stream never read (or checked last)
  const int sA = P + 1 >= 3 ? P - 2 : P + 1, sB = P + 2 >= 3 ? P - 1 : P + 2;
  const int64_t my_tiles = G.ntiles > blockIdx.x ? (G.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  long long tw[6] = {0, 0, 0, 0, 0, 0};
  const long long tstart = clock64();

  if (warp < NEPI) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(EPI_REGS));
    // ---------------- epilogue ----------------
    const int quad = warp & 3, part = warp >> 2;
    const uint32_t lrow = (uint32_t)(32 * quad) << 16;
    const int v = 32 * quad + lane;
    uint64_t gsum = 0;
    for (int k = lane; k < A.K; k += 32) gsum += (uint64_t)ld_bits(A.g, A.g_bits, k);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) gsum += __shfl_xor_sync(0xffffffffu, gsum, o);
    // unsigned data digits carry +128 each: every delta is high by 128 * sum(g) * 0x01010101
    const uint64_t corr = 0 - 128 * gsum * 0x01010101ull;
    unsigned bad = 0;
    int kslot = 0;  // running accumulator-slot use (same sequence as the MMA warp)
    // TMEM -> registers for the next one or two ring slots (one TMEM round
    // trip: both loads, one wait), which are then handed back to the MMA warp
    auto drain2 = [&](uint32_t (&ra)[EC], uint32_t (&rb)[EC], bool two) {
      const int r0 = kslot % SLOTS, r1 = (kslot + 1) % SLOTS;
#if defined(NENT_M3_EPI_SPIN)
      TM(0, mb_wait(accf_b(r0), (uint32_t)((kslot / SLOTS) & 1)));
      if (two) TM(0, mb_wait(accf_b(r1), (uint32_t)(((kslot + 1) / SLOTS) & 1)));
#elif defined(NENT_M3_EPI_SUSPEND)
      TM(0, mb_wait_suspend(accf_b(r0), (uint32_t)((kslot / SLOTS) & 1)));
      if (two) TM(0, mb_wait_suspend(accf_b(r1), (uint32_t)(((kslot + 1) / SLOTS) & 1)));
#else
      TM(0, mb_wait_sleep(accf_b(r0), (uint32_t)((kslot / SLOTS) & 1)));
      if (two) TM(0, mb_wait_sleep(accf_b(r1), (uint32_t)(((kslot + 1) / SLOTS) & 1)));
#endif
      tc05::fence_after();
      ld_slot(tbase + lrow + (uint32_t)(RING0 + r0 * U + EC * part), ra);
      if (two) ld_slot(tbase + lrow + (uint32_t)(RING0 + r1 * U + EC * part), rb);
      tc05::wait_ld();
      tc05::fence_before();
      __syncwarp();
      if (lane == 0) {
        mb_arrive(acce_b(r0));
        if (two) mb_arrive(acce_b(r1));
      }
      kslot += two ? 2 : 1;
    };
    int32_t* yP = reinterpret_cast<int32_t*>(A.y.p[P]);
    int32_t* yA = reinterpret_cast<int32_t*>(A.y.p[sA]);
    int32_t* yB = reinterpret_cast<int32_t*>(A.y.p[sB]);
    for (int64_t t = 0; t < my_tiles; ++t) {
      const int64_t tile = blockIdx.x + t * gridDim.x;
      const int64_t ybase = tile * TILE - G.shift;
      const int64_t o0 = ybase + 128 * (EC * part) + v;
      const bool interior = ybase >= 0 && ybase + TILE <= A.n_out;
      // Recovery from delta_A = delta_{P+1} = (d_P << 16) + d_{P+1} and
      // delta_B = delta_{P+2} = (d_{P+1} << 16) + d_{P+2}, exact for the
      // consistent words this kernel produces with int32 outputs (the
      // y_bits == 32 contract; recover_rot_valid<3>, recover.cuh):
      //   C = (delta_A << 16) - delta_B = (d_P << 32) - d_{P+2}   (mod 2^64)
      //   d_{P+2} = -sext32(C),  d_P = hi32(C) - (C_lo < 0),
      //   d_{P+1} = delta_A - (d_P << 16)                          (mod 2^32)
      // so each output keeps one 64-bit and one 32-bit accumulator, folded
      // class by class straight out of TMEM (class c carries weight 256^c,
      // an immediate: the class loop is unrolled).  The MMA warp issues class
      // c of A and of B into consecutive slots: one drain per class.
      uint64_t C[EC];
      uint32_t lowA[EC];
#pragma unroll
      for (int i = 0; i < EC; ++i) {
        C[i] = (corr << 16) - corr;
        lowA[i] = (uint32_t)corr;
      }
      // A rolled class loop (ptxas would otherwise sink each class's fold below
      // the next classes' TMEM loads and spill the extra live registers) whose
      // body switches to a fold with compile-time class weights: every term is
      // one IMAD.WIDE (or one IMAD on the high word for weights >= 2^32).
#ifdef NENT_M3_UNROLL_CLASSES
#pragma unroll
#else
#pragma unroll 1
#endif
      for (int c = 0; c < NCLS; ++c) {
        uint32_t rA[EC], rB[EC];
        drain2(rA, rB, true);  // class c of delta_A and of delta_B: consecutive ring slots
        switch (c) {
          case 0: fold_ab<0>(C, lowA, rA, rB); break;
          case 1: fold_ab<1>(C, lowA, rA, rB); break;
          case 2: fold_ab<2>(C, lowA, rA, rB); break;
          case 3: fold_ab<3>(C, lowA, rA, rB); break;
          default: fold_ab<4>(C, lowA, rA, rB); break;
        }
      }
      uint64_t accP[EC];
#pragma unroll
      for (int i = 0; i < EC; ++i) {
        const int32_t vv = (int32_t)(uint32_t)C[i];  // = -d_{P+2}
        const int32_t d0 = (int32_t)(uint32_t)(C[i] >> 32) - (vv >> 31);
        const int32_t d1 = (int32_t)(lowA[i] - ((uint32_t)d0 << 16));
        const int64_t o = o0 + 128 * i;
        if (interior || (o >= 0 && o < A.n_out)) {
#ifdef NENT_M3_CHECK
          if (o < 0 || o >= A.n_out) {
            printf("M3CHECK store cta %d tile %lld o %lld n_out %lld\n", blockIdx.x, (long long)tile, (long long)o,
                   (long long)A.n_out);
            __trap();
          }
#endif
          yP[o] = d0;
          yA[o] = d1;
          yB[o] = (int32_t)(0u - (uint32_t)vv);
        }
        // with failed = None the redundant word delta_P must equal
        // (d_{P+2} << 16) + d_P: start its fold at minus that
        accP[i] = corr - ((uint64_t)(int64_t)d0 - ((uint64_t)(int64_t)vv << 16));
      }
#ifndef NENT_M3_NOVERIFY_DBG
      if (verify) {  // the redundant stream P, two classes per drain
#pragma unroll 1
        for (int c = 0; c < NCLS; ++c) {
          uint32_t r0[EC], r1[EC];
          drain2(r0, r1, false);
          switch (c) {
            case 0: fold_p<0>(accP, r0); break;
            case 1: fold_p<1>(accP, r0); break;
            case 2: fold_p<2>(accP, r0); break;
            case 3: fold_p<3>(accP, r0); break;
            default: fold_p<4>(accP, r0); break;
          }
        }
#pragma unroll
        for (int i = 0; i < EC; ++i) {
          const int64_t o = o0 + 128 * i;
          bad += (interior || (o >= 0 && o < A.n_out)) && accP[i] != 0;
        }
      }
#endif
    }
    if (A.mismatch) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
      if (lane == 0 && bad) atomicAdd(A.mismatch, (unsigned long long)bad);
    }
  } else {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(PROD_REGS));
    if (warp == MMA_WARP) {
      // ---------------- MMA issuer ----------------
      const uint32_t idesc = tc05::idesc_i8(128, U, /*b_signed=*/false);
      int kslot = 0;
      for (int64_t t = 0; t < my_tiles; ++t) {
        const int ts = (int)(t % NSLOT);
        TM(0, mb_wait(full_b(ts), (uint32_t)((t / NSLOT) & 1)));
        tc05::fence_after();
        if (elect_one()) {
          const uint32_t slot_s = planes_s + (uint32_t)(ts * SLOTB);
          // chains of stream i's class c into the next ring slot
          auto issue_class = [&](int i, int c) {
            const int rs = kslot % SLOTS, use = kslot / SLOTS;
            if (use >= 1) {
              TM(1, mb_wait(acce_b(rs), (uint32_t)((use - 1) & 1)));
              tc05::fence_after();
            }
            const uint32_t d = tbase + (uint32_t)(RING0 + rs * U);
            const int im1 = i == 0 ? 2 : i - 1;
            bool first = true;
            for_class<NG>(c, [&](int p, int j) {
              // data digit p of eps_i: bytes of c_i (p < 2) or of c_{i-1} (p >= 2)
              const int raw = p < 2 ? i : im1;
              const uint32_t blo0 = tc05::desc_sw128_lo(slot_s + (uint32_t)((2 * raw + (p & 1)) * PLANE));
              const uint32_t a = tbase + (uint32_t)(8 * j * NSTEPS);
#ifndef NENT_M3_DBG_NOMMA
#pragma unroll
              for (int kc = 0; kc < NSTEPS; ++kc)
                tc05::mma_i8_ts_lo(d, a + 8u * kc, blo0 + 2u * kc, idesc, (first && kc == 0) ? 0u : 1u);
#endif
              first = false;
            });
            tc05::commit(accf_b(rs));
            ++kslot;
          };
#pragma unroll
          for (int c = 0; c < NCLS; ++c) {
            issue_class(sA, c);
            issue_class(sB, c);
          }
          if (verify) {
#pragma unroll
            for (int c = 0; c < NCLS; ++c) issue_class(P, c);
          }
          tc05::commit(empty_b(ts));
        }
        __syncwarp();
      }
      // drain the last tiles' commits before the CTA can exit: an mbarrier
      // arrive still in flight must not land in a successor CTA's shared memory
      for (int64_t t = my_tiles > NSLOT ? my_tiles - NSLOT : 0; t < my_tiles; ++t)
        mb_wait(empty_b((int)(t % NSLOT)), (uint32_t)((t / NSLOT) & 1));
    } else {
      // ---------------- producers ----------------
      const int pw = warp - NEPI;  // producer warp 0 .. NPROD-1
      // Units in order: tile t (the CTA's t-th), raw stream s.  Warp pw owns
      // int4 words [pw*WW*32, (pw+1)*WW*32) of every raw stream's window,
      // lane-consecutive (word pw*WW*32 + 32i + lane, i < WW).  mode 1 (the
      // tile's windows inside [0, n_in)): one TMA bulk copy of the warp's
      // 4 KB chunk into its own ring; mode 2: per-lane loads, zero padding.
      const int64_t P0_first = A.y_begin - G.shift + (int64_t)blockIdx.x * TILE - (G.KT - 128);
      const int64_t P0_step = (int64_t)gridDim.x * TILE;
      const uint32_t ring = stage_s + (uint32_t)(pw * NSTAGE) * SSTR;
      const int wbase = pw * WW * 32;
      // per-stream operands by select (a runtime-indexed array would live in local memory)
      const int dph0 = G.dph[0], dph1 = G.dph[1], dph2 = G.dph[2];
      const int32_t* row0 = reinterpret_cast<const int32_t*>(A.b.p[0]);
      const int32_t* row1 = reinterpret_cast<const int32_t*>(A.b.p[1]);
      const int32_t* row2 = reinterpret_cast<const int32_t*>(A.b.p[2]);
      auto dph_of = [&](int k) { return k == 0 ? dph0 : (k == 1 ? dph1 : dph2); };
      auto row_of = [&](int k) { return k == 0 ? row0 : (k == 1 ? row1 : row2); };
      // swizzled plane offset of this lane's word i
      auto soff = [&](int i) { return tc05::sw128(4u * (uint32_t)(wbase + 32 * i + lane)); };
      auto mode_of = [&](int64_t P0) {
        return (P0 >= 4 && P0 + 4 * (int64_t)NWP + 4 <= A.n_in) ? 1 : 2;
      };
      const int units = (int)my_tiles * 3;
      // TMA issue cursor (lane 0)
      int64_t iP0 = P0_first;
      int n_issue = 0, is = 0, imode = mode_of(P0_first);
      int issued = 0, consumed = 0;
      auto issue_upto = [&](int Hmax) {
        for (; n_issue < units && n_issue <= Hmax; ++n_issue) {
          if (imode == 1) {
            const int b = issued % NSTAGE;  // free: this warp consumed it NSTAGE issues ago
            const int d = dph_of(is);
            const char* src = reinterpret_cast<const char*>(row_of(is) + iP0 - d) + (size_t)wbase * 16;
            const uint32_t bytes = WCHUNK + (d ? 16u : 0u);
#ifdef NENT_M3_CHECK
            {
              const int64_t first = iP0 - d + wbase * 4, last = first + bytes / 4;
              const uint32_t dst = ring + (uint32_t)b * SSTR;
              if (first < 0 || last > A.n_in || (reinterpret_cast<uintptr_t>(src) & 15) || (dst & 15) ||
                  dst + bytes > planes_s + (uint32_t)SMEM) {
                printf("M3CHECK tma cta %d warp %d is %d P0 %lld d %d first %lld last %lld n_in %lld dst %u end %u\n",
                       blockIdx.x, pw, is, (long long)iP0, d, (long long)first, (long long)last, (long long)A.n_in,
                       dst, planes_s + (uint32_t)SMEM);
                __trap();
              }
            }
#endif
            mb_expect_tx(stg_b(pw, b), bytes);
            bulk_g2s(ring + (uint32_t)b * SSTR, src, bytes, stg_b(pw, b));
            ++issued;
          }
          if (++is == 3) {
            is = 0;
            iP0 += P0_step;
            imode = mode_of(iP0);
          }
        }
      };
      int64_t P0 = P0_first;
      int t = 0, s = 0, mode = mode_of(P0_first);
      for (int H = 0; H < units; ++H) {
        const int ts = (int)(t % NSLOT);
        // the previous unit's staging reads are complete (converted and
        // stored): lane 0 may refill that buffer
        __syncwarp();
        if (lane == 0) TM(2, issue_upto(H + NSTAGE - 1));
        if (s == 0 && t >= NSLOT) TM(0, mb_wait_sleep(empty_b(ts), (uint32_t)(((t / NSLOT) - 1) & 1)));
        const uint32_t plo = planes_s + (uint32_t)(ts * SLOTB + (2 * s) * PLANE);
        if (mode == 1) {
          const int b = consumed % NSTAGE;
          TM(1, mb_wait_sleep(stg_b(pw, b), (uint32_t)((consumed / NSTAGE) & 1)));
          const uint32_t sbuf = ring + (uint32_t)b * SSTR;
          const int d = dph_of(s);
          TM(4, {
#pragma unroll
          for (int i0 = 0; i0 < WW; i0 += 5) {  // two batches of 5 words (WW = 10)
            constexpr int B = 5;
            static_assert(WW % B == 0, "batches cover the lane's words");
            int4 v[B];
            if (d == 0) {
              const int4* sb = reinterpret_cast<const int4*>(__cvta_shared_to_generic(sbuf));
#pragma unroll
              for (int i = 0; i < B; ++i) v[i] = sb[(i0 + i) * 32 + lane];
            } else {  // this row's window starts d words into the staged copy
              const uint32_t* sw = reinterpret_cast<const uint32_t*>(__cvta_shared_to_generic(sbuf)) + d;
#pragma unroll
              for (int i = 0; i < B; ++i) {
                const uint32_t* q = sw + 4 * ((i0 + i) * 32 + lane);
                v[i] = make_int4((int)q[0], (int)q[1], (int)q[2], (int)q[3]);
              }
            }
#pragma unroll
            for (int i = 0; i < B; ++i) {
              uint32_t lo, hi;
              split2(v[i], lo, hi);
              const uint32_t off = soff(i0 + i);
              sts32(plo + off, lo);
              sts32(plo + (uint32_t)PLANE + off, hi);
            }
          }
          });
          ++consumed;
        } else {
          const int32_t* bp = row_of(s);
#pragma unroll
          for (int i = 0; i < WW; ++i) {
            const int64_t q0 = P0 + 4 * (int64_t)(wbase + 32 * i + lane);
            int e[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) e[k] = (q0 + k >= 0 && q0 + k < A.n_in) ? __ldg(bp + q0 + k) : 0;
            uint32_t lo, hi;
            split2(make_int4(e[0], e[1], e[2], e[3]), lo, hi);
            const uint32_t off = soff(i);
            sts32(plo + off, lo);
            sts32(plo + (uint32_t)PLANE + off, hi);
          }
        }
        if (s == 2) {  // the tile's planes are complete (this warp's share)
          TM(5, {
          fence_async_smem();  // this thread's plane writes -> the MMA's async-proxy reads
          __syncwarp();
          if (lane == 0) mb_arrive(full_b(ts));
          });
        }
        if (++s == 3) {
          s = 0;
          ++t;
          P0 += P0_step;
          mode = mode_of(P0);
        }
      }
    }
  }
#ifdef NENT_TC05_TIMERS
  // role timers: [mma wait_full, wait_acce, total | prod wait_empty, wait_tma,
  // total | epi wait_accf, -, total] summed over CTAs (lane 0 of warps 23, 12, 0)
  if (G.dbg && lane == 0 && (warp == MMA_WARP || warp == NEPI || warp == 0)) {
    const int role = warp == MMA_WARP ? 0 : (warp == NEPI ? 1 : 2);
    atomicAdd(G.dbg + 3 * role + 0, (unsigned long long)tw[0]);
    atomicAdd(G.dbg + 3 * role + 1, (unsigned long long)tw[1]);
    atomicAdd(G.dbg + 3 * role + 2, (unsigned long long)(clock64() - tstart));
  }
  if (G.dbg && lane == 0 && (warp == NEPI || warp == NEPI + 1)) {  // producer detail: issuer warp, next warp
    unsigned long long* q = G.dbg + 16 + 8 * (warp - NEPI);
    for (int k = 0; k < 6; ++k) atomicAdd(q + k, (unsigned long long)tw[k]);
    atomicAdd(q + 6, (unsigned long long)(clock64() - tstart));
  }
#endif
  (void)tw;
  (void)tstart;
  tc05::fence_before();
  __syncthreads();
  if (warp == MMA_WARP) {
    tc05::fence_after();
    tc05::dealloc(tbase, 512);
  }
}

}  // namespace tcm3
}  // namespace nent
