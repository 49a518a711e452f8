// chain.cu -- the LSB chain in front of the convolution (SURVEY cfg5):
// entangle -> SCALE -> ELEMENTWISE_ADD (self-entangled kernel) -> PERMUTATION,
// reference ops.py:193-204 (scale/add), :219-220 (perm), :250-262 (kernel
// self-entanglement), codec.py:57-72 (entangle).
//
// The permutation is a random gather over 2^24 positions of 8 streams.  Read
// stream-major, each position costs 8 random 32-byte sectors (one per
// stream); so the streams are first interleaved position-major (HBM-bound
// transpose), after which one gathered position is ONE sector holding all m
// source samples.  The gather kernel then writes the chain's output -- the
// permuted, scaled, shifted entangled words -- stream-major and coalesced, and
// the fused conv+extract kernel consumes it with pre_entangled = 1.
#include "common.cuh"

namespace nent {

constexpr int TR_T = 32;

// x rows (m x n) -> out (n x m), m <= 8: tile of 32 positions x m streams via smem
template <typename T>
__global__ void __launch_bounds__(256) interleave_kernel(const Rows x, int m, int64_t n, T* __restrict__ out) {
  __shared__ T tile[8][TR_T * 8 + 1];
  const int tid = threadIdx.x;
  for (int64_t p0 = (int64_t)blockIdx.x * TR_T * 8; p0 < n; p0 += (int64_t)gridDim.x * TR_T * 8) {
    // load: row s, positions p0 .. p0+255 (coalesced per row)
    for (int i = tid; i < m * TR_T * 8; i += blockDim.x) {
      const int s = i / (TR_T * 8), j = i % (TR_T * 8);
      const int64_t p = p0 + j;
      tile[s][j] = p < n ? reinterpret_cast<const T*>(x.p[s])[p] : (T)0;
    }
    __syncthreads();
    // store: position-major, m consecutive values per position (coalesced)
    for (int i = tid; i < m * TR_T * 8; i += blockDim.x) {
      const int j = i / m, s = i % m;
      const int64_t p = p0 + j;
      if (p < n) out[p * m + s] = tile[s][j];
    }
    __syncthreads();
  }
}

// x_s[p] = scale * ((c_{s-1}[q] << l) + c_s[q]) + add[q],  q = perm[p]
template <typename T, typename TO, int MT>
__global__ void __launch_bounds__(256)
gather_chain_kernel(const T* __restrict__ ct, int64_t n, int l, int64_t scale, const void* add,
                    int add_bits, const int64_t* __restrict__ perm, MutRows x) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = perm ? __ldg(perm + p) : p;
    int64_t c[MT];
    const T* row = ct + q * MT;
    if (sizeof(T) == 4 && MT == 8) {
      const int4 lo = __ldg(reinterpret_cast<const int4*>(row));
      const int4 hi = __ldg(reinterpret_cast<const int4*>(row) + 1);
      c[0] = lo.x; c[1] = lo.y; c[2] = lo.z; c[3] = lo.w;
      c[4 % MT] = hi.x; c[5 % MT] = hi.y; c[6 % MT] = hi.z; c[7 % MT] = hi.w;
    } else {
#pragma unroll
      for (int s = 0; s < MT; ++s) c[s] = (int64_t)__ldg(row + s);
    }
    const int64_t a = add ? ld_bits(add, add_bits, q) : 0;
#pragma unroll
    for (int s = 0; s < MT; ++s) {
      int64_t e = wadd(wshl(c[(s + MT - 1) % MT], l), c[s]);
      if (scale != 1) e = wmul(e, scale);
      e = wadd(e, a);
      reinterpret_cast<TO*>(x.p[s])[p] = (TO)(uint64_t)e;
    }
  }
}

}  // namespace nent

using namespace nent;

extern "C" {

int nent_interleave(const void* const* x, int x_bits, int m, int64_t n, void* out, void* stream) {
  NENT_CHECK_BITS(x_bits);
  if (m < 1 || m > 8 || n < 0) { set_error("interleave: m=%d not in 1..8", m); return NENT_ERR_PARAM; }
  if (n == 0) return NENT_OK;
  Rows R = to_rows(x, m);
  const int grid = grid_for(n, TR_T * 8, 1, 148 * 16);
  cudaStream_t s = as_stream(stream);
  if (x_bits == 32) interleave_kernel<int32_t><<<grid, 256, 0, s>>>(R, m, n, (int32_t*)out);
  else interleave_kernel<int64_t><<<grid, 256, 0, s>>>(R, m, n, (int64_t*)out);
  return check_launch("interleave");
}

int nent_gather_chain(const void* ct, int c_bits, int m, int64_t n, int l, int64_t scale,
                      const void* add, int add_bits, const int64_t* perm, void* const* x,
                      int x_bits, void* stream) {
  NENT_CHECK_BITS(c_bits);
  NENT_CHECK_BITS(x_bits);
  if (add) NENT_CHECK_BITS(add_bits);
  if (m < 3 || m > 8 || l < 0 || l > 63) { set_error("gather_chain: bad m=%d l=%d", m, l); return NENT_ERR_PARAM; }
  if (n <= 0) return NENT_OK;
  MutRows X = to_mrows(x, m);
  const int grid = grid_for(n, 256, 4);
  cudaStream_t s = as_stream(stream);
#define GC(MTV)                                                                                  \
  DISPATCH_IO(c_bits, x_bits, gather_chain_kernel<TI, TO, MTV><<<grid, 256, 0, s>>>(             \
                                  (const TI*)ct, n, l, scale, add, add_bits, perm, X))
  switch (m) {
    case 3: GC(3); break;
    case 4: GC(4); break;
    case 5: GC(5); break;
    case 6: GC(6); break;
    case 7: GC(7); break;
    default: GC(8); break;
  }
#undef GC
  return check_launch("gather_chain");
}

}  // extern "C"
