// conv_tc05_m3.cu -- host side of the m = 3, byte-aligned-shift fused kernel
// (conv_tc05_m3.cuh): envelope, geometry and launch.  Shapes outside the
// envelope return NENT_TC05_NA and take the generic tcgen05 kernel.
#include "conv_tc05_m3.cuh"

#include <cstdio>
#include <cstdlib>

namespace nent {
namespace tcm3 {
using KernFn = void (*)(ConvArgs, Geom);

static KernFn plain_kernel_for(int nsteps, int ng) {
  static const KernFn tab[3][2] = {{conv_tc05_m3_kernel<1, 4, true>, conv_tc05_m3_kernel<2, 4, true>},
                                   {conv_tc05_m3_kernel<1, 8, true>, conv_tc05_m3_kernel<2, 8, true>},
                                   {conv_tc05_m3_kernel<1, 12, true>, conv_tc05_m3_kernel<2, 12, true>}};
  if (ng < 1 || ng > 2 || nsteps % 4 || nsteps < 4 || nsteps > 12) return nullptr;
  return tab[nsteps / 4 - 1][ng - 1];
}

static KernFn kernel_for(int nsteps, int ng) {
  static const KernFn tab[3][2] = {{conv_tc05_m3_kernel<1, 4>, conv_tc05_m3_kernel<2, 4>},
                                   {conv_tc05_m3_kernel<1, 8>, conv_tc05_m3_kernel<2, 8>},
                                   {conv_tc05_m3_kernel<1, 12>, conv_tc05_m3_kernel<2, 12>}};
  if (ng < 1 || ng > 2 || nsteps % 4 || nsteps < 4 || nsteps > 12) return nullptr;
  return tab[nsteps / 4 - 1][ng - 1];
}

}  // namespace tcm3

bool tc05_m3_envelope(const ConvArgs& A, int np, int ng) {
  using namespace tcm3;
  if (A.rows != 3 || A.in_bits != 32 || A.y_bits != 32 || A.l != 16 || np != 4 || ng < 1 || ng > 2) return false;
  for (int i = 0; i < 3; ++i)
    if (!A.a.p[i] || !A.b.p[i] || !A.y.p[i]) return false;  // raw streams, entangled on load
  if (A.perm || A.add || A.scale != 1 || A.wide) return false;
  // the kernel zero-extends the rows instead of wrapping: a zero-padded (full)
  // convolution, or an output window no tap of which wraps around the period
  // (the chunked host pipeline's and the halo-split shards' windows)
  if (A.period < A.n_in + A.K - 1 && !(A.y_begin >= A.K - 1 && A.y_begin + A.n_out <= A.period)) return false;
  if (A.K < 1 || A.K > 257) return false;
  for (int i = 0; i < 3; ++i)  // int32 rows: 4-byte aligned
    if (reinterpret_cast<uintptr_t>(A.b.p[i]) & 3) return false;
  // every class accumulator is an exact int32: |sum| <= 2^15 K min(4, ng)
  if ((int64_t)32768 * A.K * ng >= ((int64_t)1 << 31)) return false;
  return true;
}

// Plain (non-entangled) convolution of exactly three int16-range int32 streams
// on the m = 3 kernel: no entangling operand, two data digits.
bool tc05_plain_m3_envelope(const ConvArgs& A, int np, int ng) {
  if (A.rows != 3 || A.in_bits != 32 || A.y_bits != 32 || np != 2 || ng < 1 || ng > 2) return false;
  for (int i = 0; i < 3; ++i)
    if (A.a.p[i] || !A.b.p[i] || !A.y.p[i]) return false;
  if (A.perm || A.add || A.scale != 1) return false;
  if (A.period < A.n_in + A.K - 1 && !(A.y_begin >= A.K - 1 && A.y_begin + A.n_out <= A.period)) return false;
  if (A.K < 1 || A.K > 257) return false;
  for (int i = 0; i < 3; ++i)
    if (reinterpret_cast<uintptr_t>(A.b.p[i]) & 3) return false;
  if ((int64_t)32768 * A.K * ng >= ((int64_t)1 << 31)) return false;
  return true;
}

static int launch_m3(ConvArgs& A, int ng, bool plain, cudaStream_t s);

int tc05_plain_m3(ConvArgs& A, int np, int ng, cudaStream_t s) {
  static const bool enabled = [] {
    const char* e = getenv("NENT_TC05_M3");
    return !(e && atoi(e) == 0);
  }();
  if (!enabled || !tc05_plain_m3_envelope(A, np, ng)) return NENT_TC05_NA;
  return launch_m3(A, ng, true, s);
}


int tc05_fused_m3(ConvArgs& A, int np, int ng, cudaStream_t s) {
  using namespace tcm3;
  // A/B switch for measurements (read once): NENT_TC05_M3=0 routes these
  // shapes to the generic tcgen05 kernel, which is exact too
  static const bool enabled = [] {
    const char* e = getenv("NENT_TC05_M3");
    return !(e && atoi(e) == 0);
  }();
  if (!enabled || !tc05_m3_envelope(A, np, ng)) return NENT_TC05_NA;
  return launch_m3(A, ng, false, s);
}

static int launch_m3(ConvArgs& A, int ng, bool plain, cudaStream_t s) {
  using namespace tcm3;
  const int sms = sm100_sms();
  if (sms <= 0) return NENT_TC05_NA;
  Geom G{};
  G.KT = (A.K + 127 + 127) / 128 * 128;
  G.nsteps = G.KT / 32;
  if (8 * ng * G.nsteps > TAPCOLS) return NENT_TC05_NA;
  {  // tiles start `shift` outputs early so every input window is 16-byte aligned
    const int64_t wb = (int64_t)((reinterpret_cast<uintptr_t>(A.b.p[0]) >> 2) & 3);
    G.shift = (int)(((wb + A.y_begin - G.KT + 128) % 4 + 4) % 4);
  }
  for (int i = 0; i < 3; ++i)
    G.dph[i] = (int)((((reinterpret_cast<uintptr_t>(A.b.p[i]) - reinterpret_cast<uintptr_t>(A.b.p[0])) >> 2) % 4 + 4) % 4);
  G.ntiles = (A.n_out + G.shift + TILE - 1) / TILE;
  const KernFn kern = plain ? plain_kernel_for(G.nsteps, ng) : kernel_for(G.nsteps, ng);
  if (!kern) return NENT_TC05_NA;
  if (ensure_smem((const void*)kern, SMEM) != NENT_OK) return NENT_ERR_CUDA;
  const unsigned grid = (unsigned)(G.ntiles < sms ? G.ntiles : sms);
  G.tile_off = edge_tile_offset(A.n_in, A.y_begin - G.shift - (G.KT - 128), 4 * (int64_t)NWP + 4, TILE, G.ntiles, grid);
#if defined(NENT_TC05_TIMERS) || defined(NENT_M3_STAMPS)
  // profiling builds: role timers (NENT_TC05_TIMERS, printed after every launch) and / or the
  // per-CTA timeline stamps (NENT_M3_STAMPS: launches stay back to back, the last launch's
  // timeline is printed when NENT_M3_DUMP is set in the environment)
  static unsigned long long* dbg = nullptr;
  if (!dbg) cudaMalloc(&dbg, (64 + 16 * 160) * sizeof(unsigned long long));
#ifdef NENT_TC05_TIMERS
  cudaMemsetAsync(dbg, 0, (64 + 16 * 160) * sizeof(unsigned long long), s);
  const bool dump = true;
#else
  const bool dump = getenv("NENT_M3_DUMP") != nullptr;
#endif
  G.dbg = dbg;
#endif
  kern<<<grid, NT, SMEM, s>>>(A, G);
  note_conv_kernel(4);
#if defined(NENT_TC05_TIMERS) || defined(NENT_M3_STAMPS)
  if (dump) {
    static unsigned long long h[64 + 16 * 160];
    cudaMemcpyAsync(h, dbg, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
#ifdef NENT_TC05_TIMERS
    fprintf(stderr, "m3 timers (kcycles/CTA): mma wait_full %.1f wait_acce %.1f total %.1f | loader wait_free %.1f total %.1f"
            " | epi wait_accf %.1f total %.1f | tiles/CTA %.2f\n", h[0] / 1e3 / grid, h[1] / 1e3 / grid, h[2] / 1e3 / grid,
            h[3] / 1e3 / grid, h[5] / 1e3 / grid, h[6] / 1e3 / grid, h[8] / 1e3 / grid, (double)G.ntiles / grid);
    fprintf(stderr, "  mma wait per slot position (A0 B0 A1 B1 .. A4 B4 P0..P4):");
    for (int k = 0; k < 15; ++k) fprintf(stderr, " %.1f", h[32 + k] / 1e3 / grid);
    fprintf(stderr, "\n  epilogue wait per step (AB0..AB4, P01, P23, P4):");
    for (int k = 0; k < 8; ++k) fprintf(stderr, " %.1f", h[48 + k] / 1e3 / grid);
    fprintf(stderr, "\n");
#endif
    {
      static const char* names[14] = {"entry", "alloc+sync", "taps built", "first planes", "2nd tile's planes", "last tile's planes",
                                      "last MMA issued", "MMAs done", "epilogue done", "exit", "conv0: window 0 in", "conv0: window 1 in",
                                      "conv0: window 2 in", "conv0: tile 0 done"};
      unsigned long long t0 = ~0ull;
      for (unsigned c = 0; c < grid; ++c) t0 = h[64 + 16 * c] < t0 ? h[64 + 16 * c] : t0;
      fprintf(stderr, "  timeline over %u CTAs, us from the first entry (min / mean / max [CTA]):\n", grid);
      for (int k = 0; k < 14; ++k) {
        double mn = 1e30, mx = -1, sum = 0;
        unsigned arg = 0;
        for (unsigned c = 0; c < grid; ++c) {
          const double v = (double)(h[64 + 16 * c + k] - t0) / 1e3;
          sum += v;
          if (v < mn) mn = v;
          if (v > mx) mx = v, arg = c;
        }
        fprintf(stderr, "    %-20s %8.2f %8.2f %8.2f [%u]\n", names[k], mn, sum / grid, mx, arg);
      }
      {
        double f = 0;
        for (unsigned c = 0; c < grid; ++c)
          f += (double)(h[64 + 16 * c + 15] - h[64 + 16 * c + 14]) / (double)(h[64 + 16 * c + 9] - h[64 + 16 * c + 0]);
        fprintf(stderr, "    effective SM clock over the kernel: %.3f GHz\n", f / grid);
      }
      // per-tile-count classes
      for (int cls = 0; cls < 2; ++cls) {
        double mx = -1, sum = 0; int cnt = 0;
        const long long full = (G.ntiles + grid - 1) / grid;
        for (unsigned c = 0; c < grid; ++c) {
          const long long mt = G.ntiles > c ? (G.ntiles - 1 - c) / grid + 1 : 0;
          if ((mt == full) != (cls == 0)) continue;
          const double v = (double)(h[64 + 16 * c + 9] - t0) / 1e3;
          sum += v; ++cnt; if (v > mx) mx = v;
        }
        if (cnt) fprintf(stderr, "    exit of the %d CTAs with %lld tiles: mean %.2f max %.2f\n", cnt, cls == 0 ? full : full - 1, sum / cnt, mx);
      }
    }
#ifdef NENT_TC05_TIMERS
    for (int w = 0; w < 2; ++w) {
      const unsigned long long* q = h + 16 + 8 * w;
      fprintf(stderr, "  converter warp %d: wait_empty %.1f wait_stage %.1f convert+sts %.1f total %.1f\n", w,
              q[0] / 1e3 / grid, q[1] / 1e3 / grid, q[4] / 1e3 / grid, q[6] / 1e3 / grid);
    }
#endif
  }
#endif
  return check_launch("tc05 fused m3");
}

}  // namespace nent
