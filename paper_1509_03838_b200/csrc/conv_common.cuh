// conv_common.cuh -- argument block and on-load input chain shared by the
// CUDA-core (conv.cu) and tensor-core (conv_imma.cu) convolution kernels.
#pragma once
#include "common.cuh"

namespace nent {

struct ConvArgs {
  Rows a;        // optional shifted operand rows: x = (a << l) + b
  Rows b;        // main operand rows
  MutRows y;     // output rows (delta rows, or the m recovered rows when fused)
  int rows;      // streams (== m when fused)
  int in_bits, y_bits, g_bits, add_bits;
  int l;
  int K, Kp, kseg, sstride, gbytes;
  int r, wide;
  int64_t n_in, period, y_begin, n_out;
  int64_t scale;
  const void* add;
  const int64_t* perm;
  const void* g;
  unsigned long long* mismatch;
  const void* imma_table;  // prepared digit-split taps (nent_imma_table), or NULL
};

// x_row[p] after the on-load chain: entangle, scale, add, gather, zero-pad.
__device__ __forceinline__ int64_t conv_prologue(const ConvArgs& A, int row, int64_t p) {
  int64_t q = p;
  if (q < 0 || q >= A.period) {
    q %= A.period;
    if (q < 0) q += A.period;
  }
  if (q >= A.n_in) return 0;
  if (A.perm) q = __ldg(A.perm + q);
  int64_t e = ld_bits(A.b.p[row], A.in_bits, q);
  const void* ap = A.a.p[row];
  if (ap) e = wadd(wshl(ld_bits(ap, A.in_bits, q), A.l), e);
  if (A.scale != 1) e = wmul(e, A.scale);
  if (A.add) e = wadd(e, ld_bits(A.add, A.add_bits, q));
  return e;
}

// Stage NS consecutive input positions p0 .. p0+NS-1 of one row through the
// on-load chain, calling emit(i, value).  Interior tiles (no wrap, no zero
// padding) take a batched path: every thread first issues U independent
// coalesced loads (perm index, a, b, add) and only then computes, so ~U*warps
// loads are in flight per SM instead of one per warp.  Edge tiles use the
// general per-element path.
template <typename TI, int U, typename F>
__device__ __forceinline__ void stage_interior(const ConvArgs& A, int row, int64_t p0, int NS,
                                               F&& emit) {
  const TI* __restrict__ bp = reinterpret_cast<const TI*>(A.b.p[row]);
  const TI* __restrict__ ap = reinterpret_cast<const TI*>(A.a.p[row]);
  const int nt = blockDim.x;
  for (int i0 = threadIdx.x; i0 < NS; i0 += nt * U) {
    int64_t q[U], vb[U], va[U], vd[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * nt;
      q[u] = p0 + (i < NS ? i : 0);
      if (A.perm) q[u] = __ldg(A.perm + q[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      vb[u] = (int64_t)__ldg(bp + q[u]);
      va[u] = ap ? (int64_t)__ldg(ap + q[u]) : 0;
      vd[u] = A.add ? ld_bits(A.add, A.add_bits, q[u]) : 0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * nt;
      if (i < NS) {
        int64_t e = vb[u];
        if (ap) e = wadd(wshl(va[u], A.l), e);
        if (A.scale != 1) e = wmul(e, A.scale);
        if (A.add) e = wadd(e, vd[u]);
        emit(i, e);
      }
    }
  }
}

template <int U, typename F>
__device__ __forceinline__ void stage_row(const ConvArgs& A, int row, int64_t p0, int NS, F&& emit) {
  if (row >= A.rows) {
    for (int i = threadIdx.x; i < NS; i += blockDim.x) emit(i, 0);
    return;
  }
  if (p0 >= 0 && p0 + NS <= A.n_in) {
    if (A.in_bits == 32) stage_interior<int32_t, U>(A, row, p0, NS, emit);
    else stage_interior<int64_t, U>(A, row, p0, NS, emit);
    return;
  }
  for (int i = threadIdx.x; i < NS; i += blockDim.x) emit(i, conv_prologue(A, row, p0 + i));
}


// tensor-core digit-sliced convolution: tcgen05 (conv_tc05.cu) where the shape
// fits its envelope, else mma.sync (conv_imma.cu)
int imma_dispatch(ConvArgs& A, int flavor, bool extract, cudaStream_t s);
constexpr int NENT_TC05_NA = 1000;  // tc05_conv: shape outside the tcgen05 kernel's envelope
int tc05_conv(ConvArgs& A, int np, int ng, bool extract, cudaStream_t s);
// fused m = 3 with the byte-aligned shift l = 16 (conv_tc05_m3.cu), or NENT_TC05_NA
int tc05_fused_m3(ConvArgs& A, int np, int ng, cudaStream_t s);
bool tc05_m3_envelope(const ConvArgs& A, int np, int ng);
int tc05_plain_m3(ConvArgs& A, int np, int ng, cudaStream_t s);
int tc05_fused_m4(ConvArgs& A, int np, int ng, cudaStream_t s);
bool tc05_m4_envelope(const ConvArgs& A, int np, int ng);
int tc05_fused_m8(ConvArgs& A, int np, int ng, cudaStream_t s);
bool tc05_m8_envelope(const ConvArgs& A, int np, int ng);

// Tile order of the persistent tcgen05 kernels (conv_tc05_m3 / _m4): CTA b processes the
// tiles (tile_off + b + k * grid) mod ntiles.  The stream-edge tiles (tile 0 and the last
// ones, whose input windows do not lie wholly inside the streams) take the slow loading
// path; the offset places that run on the CTAs that have one tile fewer than the others
// when the tile count is not a multiple of the grid.  `base` is tile 0's first input
// sample, `win` the samples one window copy reads, `tile` the outputs per tile.
inline int64_t edge_tile_offset(int64_t n_in, int64_t base, int64_t win, int64_t tile, int64_t nt, unsigned grid) {
  const int64_t rem = nt % grid;
  if (nt <= (int64_t)grid || rem == 0) return 0;
  // first tile whose window reaches past the end of the streams: base + idx * tile + win > n_in
  const int64_t room = n_in - win - base;
  int64_t e0 = room < 0 ? 0 : room / tile + 1;
  if (e0 > nt) e0 = nt;
  if (e0 < 1) e0 = 1;
  const int64_t run = (nt - e0) + 1;  // tiles e0 .. nt-1, then tile 0
  int64_t j0 = (int64_t)grid - run;   // the run ends on the last CTA
  if (j0 < rem) j0 = rem;             // (longer than the short CTAs: start at the first of them)
  return (((e0 - j0) % nt) + nt) % nt;
}

}  // namespace nent
