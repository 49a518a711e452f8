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

// x rows (m x n) -> out (n x m), m <= 8: tiles of 4 KB per row x m streams
// through shared memory; every thread issues all its row loads (16-byte
// vectors for int32 rows) before the first store, so ~32 KB per SM are in
// flight, and writes 16-byte vectors of the position-major output.
//
// CHAIN: the records hold the chain's words before the permutation instead
// of the raw samples, out[p*m + s] = scale * ((x[s-1][p] << l) + x[s][p]) +
// add[p] (int32 when the host's bound says they fit), so the gather after it
// moves one record per position and nothing else (add no longer a second
// random read).
struct ChainArgs {
  int l;
  int64_t scale;
  const void* add;
  int add_bits;
};

// MT > 0 fixes the stream count at compile time (MT = 8: the record index
// arithmetic of the store loop is shifts instead of run-time divisions).
template <typename T, bool CHAIN = false, int MT = 0>
__global__ void __launch_bounds__(256) interleave_kernel(const Rows x, int m_rt, int64_t n, T* __restrict__ out,
                                                         const ChainArgs ch = ChainArgs{}) {
  const int m = MT > 0 ? MT : m_rt;
  constexpr int P = 4096 / sizeof(T);        // positions per tile (1024 int32, 512 int64)
  constexpr int V = 16 / sizeof(T);          // elements per 16-byte vector
  __shared__ T tile[8][P + 16 / sizeof(T)];  // padded rows
  __shared__ int64_t addt[CHAIN ? P : 1];
  const int tid = threadIdx.x;
  for (int64_t p0 = (int64_t)blockIdx.x * P; p0 < n; p0 += (int64_t)gridDim.x * P) {
    const bool full = p0 + P <= n;
    bool vec = full;
    for (int s = 0; s < m; ++s) vec = vec && ((reinterpret_cast<uintptr_t>(reinterpret_cast<const T*>(x.p[s]) + p0) & 15) == 0);
    if (vec) {
      // each thread: one vector of every row (P / V vectors per row = 256 threads for int32)
      for (int i = tid; i < P / V; i += blockDim.x) {
        int4 w[8];
#pragma unroll
        for (int s = 0; s < 8; ++s)
          if (s < m) w[s] = __ldg(reinterpret_cast<const int4*>(reinterpret_cast<const T*>(x.p[s]) + p0) + i);
#pragma unroll
        for (int s = 0; s < 8; ++s)
          if (s < m) *reinterpret_cast<int4*>(&tile[s][V * i]) = w[s];
      }
    } else {
      for (int i = tid; i < m * P; i += blockDim.x) {
        const int s = i / P, j = i % P;
        const int64_t p = p0 + j;
        tile[s][j] = p < n ? reinterpret_cast<const T*>(x.p[s])[p] : (T)0;
      }
    }
    if (CHAIN) {
      for (int j = tid; j < P; j += blockDim.x)
        addt[j] = (ch.add && p0 + j < n) ? ld_bits(ch.add, ch.add_bits, p0 + j) : 0;
    }
    __syncthreads();
    // record element (position j, stream s) of the tile
    auto elem = [&](int s, int j) -> T {
      if (!CHAIN) return tile[s][j];
      int64_t e = wadd(wshl((int64_t)tile[s == 0 ? m - 1 : s - 1][j], ch.l), (int64_t)tile[s][j]);
      if (ch.scale != 1) e = wmul(e, ch.scale);
      return (T)(uint64_t)wadd(e, addt[CHAIN ? j : 0]);
    };
    // position-major stores: element e = j*m + s of the tile's output span
    const int64_t base = p0 * m;
    const int64_t total = (full ? P : n - p0) * m;
    if (full && m * sizeof(T) % 16 == 0 && (reinterpret_cast<uintptr_t>(out + base) & 15) == 0) {
      for (int e = V * tid; e < total; e += V * blockDim.x) {
        T v[V];
#pragma unroll
        for (int k = 0; k < V; ++k) v[k] = elem((e + k) % m, (e + k) / m);
        *reinterpret_cast<int4*>(out + base + e) = *reinterpret_cast<const int4*>(v);
      }
    } else {
      for (int e = tid; e < total; e += blockDim.x) out[base + e] = elem(e % m, e / m);
    }
    __syncthreads();
  }
}

// x_s[p] = scale * ((c_{s-1}[q] << l) + c_s[q]) + add[q],  q = perm[p].
// Each thread walks GU positions per round: all GU permutation indices first,
// then all GU record and add gathers, so GU random sectors per thread are in
// flight instead of one dependent pair.
template <typename T, typename TO, int MT>
__device__ __forceinline__ void gather_one(const T* __restrict__ ct, int64_t p, int64_t q, int l, int64_t scale,
                                           int64_t a, MutRows& x) {
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
#pragma unroll
  for (int s = 0; s < MT; ++s) {
    int64_t e = wadd(wshl(c[(s + MT - 1) % MT], l), c[s]);
    if (scale != 1) e = wmul(e, scale);
    e = wadd(e, a);
    reinterpret_cast<TO*>(x.p[s])[p] = (TO)(uint64_t)e;
  }
}

template <typename T, typename TO, int MT>
__global__ void __launch_bounds__(256)
gather_chain_kernel(const T* __restrict__ ct, int64_t n, int l, int64_t scale, const void* add,
                    int add_bits, const int64_t* __restrict__ perm, MutRows x) {
  constexpr int GU = 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; p + (GU - 1) * stride < n; p += GU * stride) {
    int64_t q[GU], a[GU];
#pragma unroll
    for (int u = 0; u < GU; ++u) q[u] = perm ? __ldg(perm + p + u * stride) : p + u * stride;
#pragma unroll
    for (int u = 0; u < GU; ++u) a[u] = add ? ld_bits(add, add_bits, q[u]) : 0;
#pragma unroll
    for (int u = 0; u < GU; ++u) gather_one<T, TO, MT>(ct, p + u * stride, q[u], l, scale, a[u], x);
  }
  for (; p < n; p += stride) {
    const int64_t q = perm ? __ldg(perm + p) : p;
    gather_one<T, TO, MT>(ct, p, q, l, scale, add ? ld_bits(add, add_bits, q) : 0, x);
  }
}

// x_s[p] = rec[q][s], q = perm[p]: the chain words were computed by the
// CHAIN interleave, so each position is one random record read (one 32-byte
// sector for 8 int32 streams) and m coalesced stores.  perm int32 or int64.
template <typename T, int MT, typename TP>
__global__ void __launch_bounds__(256)
gather_records_kernel(const T* __restrict__ rec, int64_t n, const TP* __restrict__ perm, MutRows x) {
  constexpr int GU = 8;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  auto one = [&](int64_t pp, int64_t q) {
    T v[MT];
    if (sizeof(T) == 4 && MT == 8) {
      const int4 lo = __ldg(reinterpret_cast<const int4*>(rec + q * MT));
      const int4 hi = __ldg(reinterpret_cast<const int4*>(rec + q * MT) + 1);
      const T w[8] = {(T)lo.x, (T)lo.y, (T)lo.z, (T)lo.w, (T)hi.x, (T)hi.y, (T)hi.z, (T)hi.w};
#pragma unroll
      for (int s = 0; s < MT; ++s) v[s] = w[s % 8];
    } else {
#pragma unroll
      for (int s = 0; s < MT; ++s) v[s] = __ldg(rec + q * MT + s);
    }
#pragma unroll
    for (int s = 0; s < MT; ++s) reinterpret_cast<T*>(x.p[s])[pp] = v[s];
  };
  for (; p + (GU - 1) * stride < n; p += GU * stride) {
    int64_t q[GU];
#pragma unroll
    for (int u = 0; u < GU; ++u) q[u] = (int64_t)__ldg(perm + p + u * stride);
#pragma unroll
    for (int u = 0; u < GU; ++u) one(p + u * stride, q[u]);
  }
  for (; p < n; p += stride) one(p, (int64_t)__ldg(perm + p));
}

// Kernel.of_permutation's bijection test (ops.py:57-62, sorted(idx) == range(n))
// on the device: every index must lie in [0, n) and be hit once.  bitmap is a
// caller-zeroed workspace of ceil(n / 32) words; *bad_dev counts out-of-range
// indices plus repeats (0 <=> bijection, since n in-range distinct indices
// cover [0, n)).
template <typename TP>
__global__ void __launch_bounds__(256) perm_check_kernel(const TP* __restrict__ perm, int64_t n,
                                                          unsigned* __restrict__ bitmap,
                                                          unsigned long long* __restrict__ bad) {
  unsigned long long nbad = 0;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = (int64_t)perm[j];
    if (v < 0 || v >= n) {
      ++nbad;
      continue;
    }
    const unsigned bit = 1u << (v & 31);
    if (atomicOr(bitmap + (v >> 5), bit) & bit) ++nbad;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nbad += __shfl_xor_sync(0xffffffffu, nbad, o);
  if ((threadIdx.x & 31) == 0 && nbad) atomicAdd(bad, nbad);
}

}  // namespace nent

using namespace nent;

extern "C" {

int nent_interleave(const void* const* x, int x_bits, int m, int64_t n, void* out, void* stream) {
  NENT_CHECK_BITS(x_bits);
  if (m < 1 || m > 8 || n < 0) { set_error("interleave: m=%d not in 1..8", m); return NENT_ERR_PARAM; }
  if (n == 0) return NENT_OK;
  Rows R = to_rows(x, m);
  const int grid = grid_for(n, x_bits == 32 ? 1024 : 512, 1, 148 * 8);
  cudaStream_t s = as_stream(stream);
  if (x_bits == 32) interleave_kernel<int32_t><<<grid, 256, 0, s>>>(R, m, n, (int32_t*)out);
  else interleave_kernel<int64_t><<<grid, 256, 0, s>>>(R, m, n, (int64_t*)out);
  return check_launch("interleave");
}

int nent_interleave_chain(const void* const* x, int x_bits, int m, int64_t n, int l, int64_t scale,
                          const void* add, int add_bits, void* out, int out_bits, void* stream) {
  NENT_CHECK_BITS(x_bits);
  NENT_CHECK_BITS(out_bits);
  if (add) NENT_CHECK_BITS(add_bits);
  if (m < 3 || m > 8 || l < 0 || l > 63) { set_error("interleave_chain: bad m=%d l=%d", m, l); return NENT_ERR_PARAM; }
  if (x_bits != out_bits) { set_error("interleave_chain: x_bits %d != out_bits %d", x_bits, out_bits); return NENT_ERR_PARAM; }
  if (n == 0) return NENT_OK;
  Rows R = to_rows(x, m);
  const ChainArgs ch{l, scale, add, add_bits};
  const int grid = grid_for(n, x_bits == 32 ? 1024 : 512, 1, 148 * 8);
  cudaStream_t s = as_stream(stream);
  if (x_bits == 32 && m == 8) interleave_kernel<int32_t, true, 8><<<grid, 256, 0, s>>>(R, m, n, (int32_t*)out, ch);
  else if (x_bits == 32) interleave_kernel<int32_t, true><<<grid, 256, 0, s>>>(R, m, n, (int32_t*)out, ch);
  else interleave_kernel<int64_t, true><<<grid, 256, 0, s>>>(R, m, n, (int64_t*)out, ch);
  return check_launch("interleave_chain");
}

int nent_gather_records(const void* rec, int rec_bits, int m, int64_t n, const void* perm, int perm_bits,
                        void* const* x, void* stream) {
  NENT_CHECK_BITS(rec_bits);
  if (m < 3 || m > 8 || !perm || (perm_bits != 32 && perm_bits != 64)) {
    set_error("gather_records: bad m=%d or perm", m);
    return NENT_ERR_PARAM;
  }
  if (n <= 0) return NENT_OK;
  MutRows X = to_mrows(x, m);
  const int grid = grid_for(n, 256, 8);
  cudaStream_t s = as_stream(stream);
#define GR(T, MTV)                                                                                     \
  (perm_bits == 32 ? (gather_records_kernel<T, MTV, int32_t><<<grid, 256, 0, s>>>((const T*)rec, n, (const int32_t*)perm, X), 0) \
                   : (gather_records_kernel<T, MTV, int64_t><<<grid, 256, 0, s>>>((const T*)rec, n, (const int64_t*)perm, X), 0))
#define GRM(T)                            \
  switch (m) {                            \
    case 3: GR(T, 3); break;              \
    case 4: GR(T, 4); break;              \
    case 5: GR(T, 5); break;              \
    case 6: GR(T, 6); break;              \
    case 7: GR(T, 7); break;              \
    default: GR(T, 8); break;             \
  }
  if (rec_bits == 32) {
    GRM(int32_t)
  } else {
    GRM(int64_t)
  }
#undef GRM
#undef GR
  return check_launch("gather_records");
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

int nent_perm_check(const void* perm, int perm_bits, int64_t n, unsigned* bitmap, unsigned long long* bad_dev,
                    void* stream) {
  if (!perm || !bitmap || !bad_dev || (perm_bits != 32 && perm_bits != 64)) {
    set_error("perm_check: bad arguments");
    return NENT_ERR_PARAM;
  }
  if (n <= 0) return NENT_OK;
  const int grid = grid_for(n, 256, 4);
  cudaStream_t s = as_stream(stream);
  if (perm_bits == 32)
    perm_check_kernel<int32_t><<<grid, 256, 0, s>>>((const int32_t*)perm, n, bitmap, bad_dev);
  else
    perm_check_kernel<int64_t><<<grid, 256, 0, s>>>((const int64_t*)perm, n, bitmap, bad_dev);
  return check_launch("perm_check");
}

}  // extern "C"
