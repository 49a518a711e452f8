// conv_tc05_m4.cu -- host side of the m = 4 long-filter fused kernel
// (conv_tc05_m4.cuh): envelope, geometry and launch.  Shapes outside the
// envelope return NENT_TC05_NA and take the generic tcgen05 / mma.sync kernels.
#include "conv_tc05_m4.cuh"

#include <cstdio>
#include <cstdlib>

namespace nent {

bool tc05_m4_envelope(const ConvArgs& A, int np, int ng) {
  using namespace tcm4;
  if (A.rows != M || A.in_bits != 32 || A.y_bits != 32 || A.l != 16 || np != 4 || ng < 1 || ng > 2) return false;
  for (int i = 0; i < M; ++i)
    if (!A.a.p[i] || !A.b.p[i] || !A.y.p[i]) return false;  // raw streams, entangled on load
  if (A.perm || A.add || A.scale != 1 || A.wide) return false;
  // zero extension instead of wrap-around: a full convolution, or a window no tap of which wraps
  if (A.period < A.n_in + A.K - 1 && !(A.y_begin >= A.K - 1 && A.y_begin + A.n_out <= A.period)) return false;
  if (A.K < 1 || (A.K + 127 + 127) / 128 * 128 > KTMAX) return false;
  for (int i = 0; i < M; ++i)  // int32 rows: 4-byte aligned
    if (reinterpret_cast<uintptr_t>(A.b.p[i]) & 3) return false;
  // every class accumulator is an exact int32: |sum| <= 2^15 K min(4, ng)
  if ((int64_t)32768 * A.K * ng >= ((int64_t)1 << 31)) return false;
  return true;
}

int tc05_fused_m4(ConvArgs& A, int np, int ng, cudaStream_t s) {
  using namespace tcm4;
  // A/B switch for measurements (read once): NENT_TC05_M4=0 routes these
  // shapes to the other kernels, which are exact too
  static const bool enabled = [] {
    const char* e = getenv("NENT_TC05_M4");
    return !(e && atoi(e) == 0);
  }();
  if (!enabled || !tc05_m4_envelope(A, np, ng)) return NENT_TC05_NA;
  const int sms = sm100_sms();
  if (sms <= 0) return NENT_TC05_NA;
  Geom G{};
  G.KT = (A.K + 127 + 127) / 128 * 128;
  G.nsteps = G.KT / 32;
  G.ngrp = G.nsteps / GK;
  G.nw4 = (TILE + G.KT - 128) / 4;
  {  // tiles start `shift` outputs early so every input window is 16-byte aligned
    const int64_t wb = (int64_t)((reinterpret_cast<uintptr_t>(A.b.p[0]) >> 2) & 3);
    G.shift = (int)(((wb + A.y_begin - G.KT + 128) % 4 + 4) % 4);
  }
  for (int i = 0; i < M; ++i)
    G.dph[i] = (int)((((reinterpret_cast<uintptr_t>(A.b.p[i]) - reinterpret_cast<uintptr_t>(A.b.p[0])) >> 2) % 4 + 4) % 4);
  G.ntiles = (A.n_out + G.shift + TILE - 1) / TILE;
  void (*kern)(ConvArgs, Geom) = ng == 1 ? conv_tc05_m4_kernel<1> : conv_tc05_m4_kernel<2>;
  if (ensure_smem((const void*)kern, SMEM) != NENT_OK) return NENT_ERR_CUDA;
  const unsigned grid = (unsigned)(G.ntiles < sms ? G.ntiles : sms);
  G.tile_off = edge_tile_offset(A.n_in, A.y_begin - G.shift - (G.KT - 128), 4 * (int64_t)G.nw4 + 4, TILE, G.ntiles, grid);
#if defined(NENT_TC05_TIMERS) || defined(NENT_M4_STAMPS)
  // profiling builds: role timers (NENT_TC05_TIMERS) / per-CTA timeline stamps (NENT_M4_STAMPS,
  // printed for the launch made while NENT_M4_DUMP is set in the environment)
  static unsigned long long* dbg = nullptr;
  if (!dbg) cudaMalloc(&dbg, (16 + 8 * 160) * sizeof(unsigned long long));
#ifdef NENT_TC05_TIMERS
  cudaMemsetAsync(dbg, 0, 16 * sizeof(unsigned long long), s);
#endif
  G.dbg = dbg;
#endif
  kern<<<grid, NT, SMEM, s>>>(A, G);
  note_conv_kernel(5);
#ifdef NENT_TC05_TIMERS
  {
    unsigned long long h[16];
    cudaMemcpyAsync(h, dbg, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    fprintf(stderr, "m4 timers (kcycles/CTA): mma wait planes %.1f taps %.1f acc_free %.1f total %.1f | tap writer wait_free %.1f"
            " total %.1f | epi wait_full %.1f total %.1f | tiles/CTA %.2f\n", h[0] / 1e3 / grid, h[1] / 1e3 / grid,
            h[2] / 1e3 / grid, h[3] / 1e3 / grid, h[4] / 1e3 / grid, h[5] / 1e3 / grid, h[6] / 1e3 / grid,
            h[7] / 1e3 / grid, (double)G.ntiles / grid);
  }
#endif
#ifdef NENT_M4_STAMPS
  if (getenv("NENT_M4_DUMP")) {
    static unsigned long long h[16 + 8 * 160];
    cudaMemcpyAsync(h, dbg, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    static const char* names[5] = {"entry", "first planes", "2nd tile's planes", "last tile's planes", "exit"};
    unsigned long long t0 = ~0ull;
    for (unsigned c = 0; c < grid; ++c) t0 = h[16 + 8 * c] < t0 ? h[16 + 8 * c] : t0;
    fprintf(stderr, "  m4 timeline over %u CTAs (%.2f tiles/CTA), us from the first entry (min / mean / max [CTA]):\n", grid,
            (double)G.ntiles / grid);
    for (int k = 0; k < 5; ++k) {
      double mn = 1e30, mx = -1, sum = 0;
      unsigned arg = 0;
      for (unsigned c = 0; c < grid; ++c) {
        const double v = (double)(h[16 + 8 * c + k] - t0) / 1e3;
        sum += v;
        if (v < mn) mn = v;
        if (v > mx) mx = v, arg = c;
      }
      fprintf(stderr, "    %-20s %8.2f %8.2f %8.2f [%u]\n", names[k], mn, sum / grid, mx, arg);
    }
    const long long full = (G.ntiles + grid - 1) / grid;
    for (int cls = 0; cls < 2; ++cls) {
      double mx = -1, sum = 0;
      int cnt = 0;
      for (unsigned c = 0; c < grid; ++c) {
        const long long mt = G.ntiles > c ? (G.ntiles - 1 - c) / grid + 1 : 0;
        if ((mt == full) != (cls == 0)) continue;
        const double v = (double)(h[16 + 8 * c + 4] - t0) / 1e3;
        sum += v;
        ++cnt;
        if (v > mx) mx = v;
      }
      if (cnt) fprintf(stderr, "    exit of the %d CTAs with %lld tiles: mean %.2f max %.2f\n", cnt, cls == 0 ? full : full - 1, sum / cnt, mx);
    }
  }
#endif
  return check_launch("tc05 fused m4");
}

}  // namespace nent
