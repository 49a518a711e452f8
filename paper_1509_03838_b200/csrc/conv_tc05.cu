// conv_tc05.cu -- host side of the tcgen05 convolution (conv_tc05.cuh):
// geometry / envelope, kernel selection and launch.  The kernel templates are
// instantiated in conv_tc05_inst_*.cu (one translation unit per NP and
// EXTRACT, so the build compiles them in parallel).
#include "conv_tc05.cuh"

#include <cstdio>
#include <cstdlib>

namespace nent {
namespace tcc {
using KernFn = void (*)(ConvArgs, Geom);
// conv_tc05_inst_*.cu: the kernel for (EXTRACT, NP) at nsteps/4-1 = si and NG, or nullptr
#define TC05_DECL(E, P) KernFn kernel_e##E##_p##P(int si, int ng);
TC05_DECL(0, 1) TC05_DECL(0, 2) TC05_DECL(0, 3) TC05_DECL(0, 4) TC05_DECL(0, 5) TC05_DECL(0, 6)
TC05_DECL(1, 1) TC05_DECL(1, 2) TC05_DECL(1, 3) TC05_DECL(1, 4) TC05_DECL(1, 5) TC05_DECL(1, 6)
#undef TC05_DECL
static KernFn kernel_for(bool extract, int si, int np, int ng) {
  static KernFn (*const tab[2][6])(int, int) = {
      {kernel_e0_p1, kernel_e0_p2, kernel_e0_p3, kernel_e0_p4, kernel_e0_p5, kernel_e0_p6},
      {kernel_e1_p1, kernel_e1_p2, kernel_e1_p3, kernel_e1_p4, kernel_e1_p5, kernel_e1_p6}};
  return tab[extract ? 1 : 0][np - 1](si, ng);
}
}  // namespace tcc

static int sm_count_tc() { return sm100_sms(); }  // tcgen05 is sm_100-family only

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
  for (int r = 0; r < A.rows; ++r)  // the producers' 32-bit entangling shift needs l in [1, 31]
    if (A.a.p[r] && (A.l < 1 || A.l > 31)) return NENT_TC05_NA;
  // fused with a failed stream: only the two survivors are convolved (the
  // failed stream's delta is never produced, as in the reference's recovery)
  if (extract && A.r >= 0) G.nstreams = 2;
#if defined(NENT_TC05_PROFILING) || defined(NENT_TC05_TIMERS)
  // profiling builds only (scripts/build_variant.py): role-isolation modes
  // that skip work, read once per process
  static const int debug_env = [] {
    const char* e = getenv("NENT_TC05_DEBUG");
    return e ? atoi(e) : 0;
  }();
  G.debug = debug_env;
#else
  G.debug = 0;  // release: every role always runs
#endif
  const int sms = sm_count_tc();
  if (sms <= 0) return NENT_TC05_NA;
  {  // align the input windows: (row-0 word offset + P0) = 0 mod 4
    const int64_t wb = (int64_t)((reinterpret_cast<uintptr_t>(A.b.p[0]) >> 2) & 3);
    G.shift = (int)(((wb + A.y_begin - G.KT + 128) % 4 + 4) % 4);
  }
  G.ntiles = (A.n_out + G.shift + TILE - 1) / TILE;
  const unsigned grid = (unsigned)(G.ntiles < sms ? G.ntiles : sms);
  const int si = G.nsteps / 4 - 1;
  const KernFn kern = kernel_for(extract, si, np, ng);
  if (!kern) return NENT_TC05_NA;
  if (ensure_smem((const void*)kern, smem) != NENT_OK) return NENT_ERR_CUDA;
  static unsigned long long* dbg = nullptr;
  if (G.debug & 8) {
    if (!dbg) cudaMalloc(&dbg, 16 * sizeof(unsigned long long));
    cudaMemsetAsync(dbg, 0, 16 * sizeof(unsigned long long), s);
    G.dbg = dbg;
  }
  {
    // programmatic dependent launch: this launch's setup overlaps the tail of
    // the previous kernel on the stream (griddepcontrol.wait in the kernel
    // orders every global access after it).  Off by default (NENT_TC05_PDL=1
    // turns it on): measured 0.165 vs 0.160 ms per fused cfg2 launch with it
    static const int pdl = [] {
      const char* e = getenv("NENT_TC05_PDL");
      return e ? atoi(e) : 0;
    }();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kern, A, G);
  }
  if (G.debug & 8) {
    unsigned long long h[16];
    cudaMemcpyAsync(h, dbg, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    fprintf(stderr, "tc05 timers (kcycles/CTA): mma wait_full %.0f wait_accempty %.0f total %.0f | prod wait_empty %.0f "
            "wait_cpasync %.0f total %.0f | epi wait_accfull %.0f tmem_ld %.0f total %.0f | setup %.0f max_cta %.0f\n", h[0] / 1e3 / grid,
            h[1] / 1e3 / grid, h[2] / 1e3 / grid, h[3] / 1e3 / grid, h[4] / 1e3 / grid, h[5] / 1e3 / grid,
            h[6] / 1e3 / grid, h[7] / 1e3 / grid, h[8] / 1e3 / grid, h[9] / 1e3 / grid, h[10] / 1e3);
  }
  note_conv_kernel(3);
  return check_launch("tc05 conv");
}

}  // namespace nent

using namespace nent;

extern "C" int nent_imma_kernel(int flavor, int K, int rows, int extract) {
  if ((flavor & 0xff) != NENT_MAC_IMMA) return 0;
  if (flavor & NENT_IMMA_MMA_SYNC) return 1;
  tcc::Geom G;
  size_t smem = 0;
  const int np = (flavor >> 8) & 0xf, ng = (flavor >> 12) & 0xf;
  // the dedicated fused kernels (int32 rows, byte-aligned digits): m = 4 long
  // filters (conv_tc05_m4) and m = 8 already-entangled rows (conv_tc05_m8)
  if (extract && sm100_sms() > 0) {
    if (rows == 4 && np == 4 && ng <= 2 && K <= 1153) return 2;
    if (rows == 8 && np == 2 && ng == 1 && K <= 257) return 2;
  }
  return tc05_geometry(K, rows, np, ng, extract != 0, G, smem) ? 2 : 1;
}
