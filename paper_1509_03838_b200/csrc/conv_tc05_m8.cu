// conv_tc05_m8.cu -- host side of the m = 8 pre-entangled fused kernel
// (conv_tc05_m8.cuh): envelope, geometry and launch.  Shapes outside the
// envelope return NENT_TC05_NA and take the other kernels.
#include "conv_tc05_m8.cuh"

#include <cstdio>
#include <cstdlib>

namespace nent {

bool tc05_m8_envelope(const ConvArgs& A, int np, int ng) {
  using namespace tcm8;
  if (A.rows != M || A.in_bits != 32 || A.y_bits != 32 || np != 2 || ng != 1) return false;
  if (A.l < 1 || (M - 1) * A.l > 32) return false;  // the recovery runs in 32-bit arithmetic
  for (int i = 0; i < M; ++i)
    if (A.a.p[i] || !A.b.p[i] || !A.y.p[i]) return false;  // rows already entangled
  if (!A.wide || A.perm || A.add || A.scale != 1) return false;
  // zero extension instead of wrap-around: a full convolution, or a window no tap of which wraps
  if (A.period < A.n_in + A.K - 1 && !(A.y_begin >= A.K - 1 && A.y_begin + A.n_out <= A.period)) return false;
  if (A.K < 1 || A.K > 257) return false;
  for (int i = 0; i < M; ++i)
    if (reinterpret_cast<uintptr_t>(A.b.p[i]) & 3) return false;
  return true;
}

int tc05_fused_m8(ConvArgs& A, int np, int ng, cudaStream_t s) {
  using namespace tcm8;
  static const bool enabled = [] {
    const char* e = getenv("NENT_TC05_M8");
    return !(e && atoi(e) == 0);
  }();
  if (!enabled || !tc05_m8_envelope(A, np, ng)) return NENT_TC05_NA;
  const int sms = sm100_sms();
  if (sms <= 0) return NENT_TC05_NA;
  Geom G{};
  G.KT = (A.K + 127 + 127) / 128 * 128;
  G.nsteps = G.KT / 32;
  G.nw4 = (TILE + G.KT - 128) / 4;
  {
    const int64_t wb = (int64_t)((reinterpret_cast<uintptr_t>(A.b.p[0]) >> 2) & 3);
    G.shift = (int)(((wb + A.y_begin - G.KT + 128) % 4 + 4) % 4);
  }
  for (int i = 0; i < M; ++i)
    G.dph[i] = (int)((((reinterpret_cast<uintptr_t>(A.b.p[i]) - reinterpret_cast<uintptr_t>(A.b.p[0])) >> 2) % 4 + 4) % 4);
  G.ntiles = (A.n_out + G.shift + TILE - 1) / TILE;
  void (*kern)(ConvArgs, Geom) = G.nsteps == 4 ? conv_tc05_m8_kernel<4>
                                 : (G.nsteps == 8 ? conv_tc05_m8_kernel<8> : conv_tc05_m8_kernel<12>);
  if (ensure_smem((const void*)kern, SMEM) != NENT_OK) return NENT_ERR_CUDA;
  const unsigned grid = (unsigned)(G.ntiles < sms ? G.ntiles : sms);
  G.tile_off = edge_tile_offset(A.n_in, A.y_begin - G.shift - (G.KT - 128), 4 * (int64_t)G.nw4 + 4, TILE, G.ntiles, grid);
  kern<<<grid, NT, SMEM, s>>>(A, G);
  note_conv_kernel(6);
  return check_launch("tc05 fused m8");
}

}  // namespace nent
