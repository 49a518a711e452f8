// codec.cu -- K1 entangle, K3 extract/recover, poison, range/bound reductions,
// checksum baseline.  HBM-bound elementwise passes: grid-stride, coalesced,
// several independent loads in flight per thread.
#include <cstdarg>
#include <cstdio>

#include "common.cuh"

#include <map>
#include <mutex>
#include <utility>
#include "recover.cuh"

namespace nent {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
}

static thread_local int g_last_conv_kernel = 0;

namespace {
std::mutex g_dev_mu;
std::map<std::pair<int, const void*>, size_t> g_smem_cfg;  // (device, kernel) -> opted-in bytes
int g_sms[64];                                              // 0 unknown, -1 not sm_100
}  // namespace

int ensure_smem(const void* kern, size_t bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_dev_mu);
  size_t& have = g_smem_cfg[{dev, kern}];
  if (bytes <= have) return NENT_OK;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess) {
    set_error("cannot reserve %zu bytes of shared memory on device %d", bytes, dev);
    return NENT_ERR_CUDA;
  }
  have = bytes;
  return NENT_OK;
}

int sm100_sms() {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_dev_mu);
  int& n = g_sms[dev & 63];
  if (n == 0) {
    int sms = 0, major = 0, minor = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    n = (major == 10 && minor == 0 && sms > 0) ? sms : -1;
  }
  return n;
}
void note_conv_kernel(int k) { g_last_conv_kernel = k; }

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return NENT_ERR_CUDA;
  }
  return NENT_OK;
}

constexpr int EW_THREADS = 256;
constexpr int EW_UNROLL = 4;

// ---------------------------------------------------------------- entangle --
// eps[i][j] = (src[(i-1) mod m][j] << l) + src[i][j]; optional first-offender.
template <typename TI, typename TO>
__global__ void __launch_bounds__(EW_THREADS)
entangle_kernel(const Rows src, MutRows eps, int m, int64_t n, int l, int64_t hi, int check,
                unsigned long long* bad) {
  const int i = blockIdx.y;
  const TI* __restrict__ cur = reinterpret_cast<const TI*>(src.p[i]);
  const TI* __restrict__ prv = reinterpret_cast<const TI*>(src.p[(i + m - 1) % m]);
  TO* __restrict__ out = reinterpret_cast<TO*>(eps.p[i]);
  const int64_t stride = (int64_t)gridDim.x * EW_THREADS * EW_UNROLL;
  for (int64_t base = (int64_t)blockIdx.x * EW_THREADS * EW_UNROLL + threadIdx.x; base < n;
       base += stride) {
    int64_t a[EW_UNROLL], b[EW_UNROLL];
#pragma unroll
    for (int u = 0; u < EW_UNROLL; ++u) {
      int64_t j = base + (int64_t)u * EW_THREADS;
      a[u] = j < n ? (int64_t)__ldg(prv + j) : 0;
      b[u] = j < n ? (int64_t)__ldg(cur + j) : 0;
    }
#pragma unroll
    for (int u = 0; u < EW_UNROLL; ++u) {
      int64_t j = base + (int64_t)u * EW_THREADS;
      if (j < n) {
        out[j] = (TO)(uint64_t)wadd(wshl(a[u], l), b[u]);
        if (check && wabs(b[u]) > hi) atomicMin(bad, (unsigned long long)((int64_t)i * n + j));
      }
    }
  }
}

template <typename TI, typename TO>
__global__ void __launch_bounds__(EW_THREADS)
shift_add_kernel(const TI* __restrict__ a, const TI* __restrict__ b, TO* __restrict__ out,
                 int64_t n, int l) {
  for (int64_t j = (int64_t)blockIdx.x * EW_THREADS + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * EW_THREADS)
    out[j] = (TO)(uint64_t)wadd(wshl((int64_t)__ldg(a + j), l), (int64_t)__ldg(b + j));
}

// ----------------------------------------------------------------- extract --
// One thread per position; reads the m-1 surviving rows once, writes m rows.
template <int MT, typename TI, typename TO>
__global__ void __launch_bounds__(EW_THREADS)
extract_kernel(const Rows delta, MutRows out, int m, int64_t n, int l, int r, int wide,
               unsigned long long* overflow, unsigned long long* mismatch) {
  constexpr int CAP = MT > 0 ? MT : NENT_MAX_STREAMS;
  const int M = MT > 0 ? MT : m;
  for (int64_t j = (int64_t)blockIdx.x * EW_THREADS + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * EW_THREADS) {
    int64_t rot[CAP], orot[CAP];
#pragma unroll
    for (int t = 0; t < M - 1; ++t) {
      int row = r + 1 + t;
      row -= row >= M ? M : 0;
      row -= row >= M ? M : 0;
      rot[t] = (int64_t)__ldg(reinterpret_cast<const TI*>(delta.p[row]) + j);
    }
    bool ovf = recover_rot<MT>(rot, M, l, wide != 0, orot);
    if (ovf && overflow) atomicAdd(overflow, 1ull);
#pragma unroll
    for (int t = 0; t < M; ++t) {
      int row = r + t;
      row -= row >= M ? M : 0;
      reinterpret_cast<TO*>(out.p[row])[j] = (TO)(uint64_t)orot[t];
    }
    // verify: the pivot's own word must be (d_{r-1} << l) + d_r (codec.py:57-66)
    if (mismatch) {
      const int64_t dr = (int64_t)__ldg(reinterpret_cast<const TI*>(delta.p[r]) + j);
      int64_t want = wadd(wshl(orot[M - 1], l), orot[0]);
      if (sizeof(TI) == 4) want = (int64_t)(int32_t)(uint32_t)(uint64_t)want;  // the row's own width
      if (dr != want) atomicAdd(mismatch, 1ull);
    }
  }
}

// ---------------------------------------------- vectorised K1 / K3 (16-byte) --
// Four consecutive positions per thread and iteration, moved as 16-byte
// vectors (one int4 of int32 words or two longlong2 of int64 words per row):
// every row of the launch is 16-byte aligned at position `head` (0..3, found
// on the host), positions outside [head, head + 4 nq) go through the scalar
// path of block 0.  HBM-bound: several vectors per row in flight per thread.
template <typename T>
__device__ __forceinline__ void load4(const T* __restrict__ p, int64_t j, int64_t (&v)[4]) {
  if (sizeof(T) == 4) {
    const int4 x = __ldg(reinterpret_cast<const int4*>(p + j));
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
  } else {
    const longlong2 a = __ldg(reinterpret_cast<const longlong2*>(p + j));
    const longlong2 b = __ldg(reinterpret_cast<const longlong2*>(p + j) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  }
}
template <typename T>
__device__ __forceinline__ void store4(T* __restrict__ p, int64_t j, const int64_t (&v)[4]) {
  if (sizeof(T) == 4) {
    *reinterpret_cast<int4*>(p + j) = make_int4((int)(uint32_t)(uint64_t)v[0], (int)(uint32_t)(uint64_t)v[1],
                                                (int)(uint32_t)(uint64_t)v[2], (int)(uint32_t)(uint64_t)v[3]);
  } else {
    reinterpret_cast<longlong2*>(p + j)[0] = make_longlong2(v[0], v[1]);
    reinterpret_cast<longlong2*>(p + j)[1] = make_longlong2(v[2], v[3]);
  }
}

template <typename TI, typename TO>
__global__ void __launch_bounds__(EW_THREADS)
entangle_vec_kernel(const Rows src, MutRows eps, int m, int64_t n, int64_t head, int64_t nq, int l, int64_t hi,
                    int check, unsigned long long* bad) {
  const int i = blockIdx.y;
  const TI* __restrict__ cur = reinterpret_cast<const TI*>(src.p[i]);
  const TI* __restrict__ prv = reinterpret_cast<const TI*>(src.p[(i + m - 1) % m]);
  TO* __restrict__ out = reinterpret_cast<TO*>(eps.p[i]);
  auto one = [&](int64_t j, int64_t a, int64_t b) {
    if (check && wabs(b) > hi) atomicMin(bad, (unsigned long long)((int64_t)i * n + j));
    return wadd(wshl(a, l), b);
  };
  constexpr int UV = 2;  // vectors per thread and iteration
  const int64_t stride = (int64_t)gridDim.x * EW_THREADS * UV;
  for (int64_t q0 = (int64_t)blockIdx.x * EW_THREADS * UV + threadIdx.x; q0 < nq; q0 += stride) {
    int64_t a[UV][4], b[UV][4];
#pragma unroll
    for (int u = 0; u < UV; ++u) {
      const int64_t q = q0 + (int64_t)u * EW_THREADS;
      if (q < nq) {
        load4(prv, head + 4 * q, a[u]);
        load4(cur, head + 4 * q, b[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < UV; ++u) {
      const int64_t q = q0 + (int64_t)u * EW_THREADS;
      if (q < nq) {
        int64_t o[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) o[k] = one(head + 4 * q + k, a[u][k], b[u][k]);
        store4(out, head + 4 * q, o);
      }
    }
  }
  if (blockIdx.x == 0) {  // the unaligned head [0, head) and the ragged tail [head + 4 nq, n)
    const int64_t tail0 = head + 4 * nq, ns = head + (n - tail0);
    for (int64_t k = threadIdx.x; k < ns; k += EW_THREADS) {
      const int64_t j = k < head ? k : tail0 + (k - head);
      out[j] = (TO)(uint64_t)one(j, (int64_t)__ldg(prv + j), (int64_t)__ldg(cur + j));
    }
  }
}

// All MT rows of a position vector in one thread: every source word is read
// from HBM exactly once (the row-per-block kernel above reads each row twice,
// as c_i and as c_{i-1}, and the second read misses L2 on streams beyond its
// 126 MB), so the pass moves the algorithmic m*n words in and m*n words out.
template <int MT, typename TI, typename TO>
__global__ void __launch_bounds__(EW_THREADS)
entangle_rows_kernel(const Rows src, MutRows eps, int64_t n, int64_t head, int64_t nq, int l, int64_t hi,
                     int check, unsigned long long* bad) {
  auto one = [&](int i, int64_t j, int64_t a, int64_t b) {
    if (check && wabs(b) > hi) atomicMin(bad, (unsigned long long)((int64_t)i * n + j));
    return wadd(wshl(a, l), b);
  };
  const int64_t stride = (int64_t)gridDim.x * EW_THREADS;
  for (int64_t q = (int64_t)blockIdx.x * EW_THREADS + threadIdx.x; q < nq; q += stride) {
    int64_t c[MT][4];
#pragma unroll
    for (int i = 0; i < MT; ++i) load4(reinterpret_cast<const TI*>(src.p[i]), head + 4 * q, c[i]);
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      int64_t o[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) o[k] = one(i, head + 4 * q + k, c[(i + MT - 1) % MT][k], c[i][k]);
      store4(reinterpret_cast<TO*>(eps.p[i]), head + 4 * q, o);
    }
  }
  if (blockIdx.x == 0) {  // the unaligned head [0, head) and the ragged tail [head + 4 nq, n)
    const int64_t tail0 = head + 4 * nq, ns = head + (n - tail0);
    for (int64_t k = threadIdx.x; k < ns * MT; k += EW_THREADS) {
      const int i = (int)(k / ns);
      const int64_t kk = k - (int64_t)i * ns;
      const int64_t j = kk < head ? kk : tail0 + (kk - head);
      reinterpret_cast<TO*>(eps.p[i])[j] =
          (TO)(uint64_t)one(i, j, (int64_t)__ldg(reinterpret_cast<const TI*>(src.p[(i + MT - 1) % MT]) + j),
                            (int64_t)__ldg(reinterpret_cast<const TI*>(src.p[i]) + j));
    }
  }
}

template <int MT, typename TI, typename TO>
__global__ void __launch_bounds__(EW_THREADS)
extract_vec_kernel(const Rows delta, MutRows out, int64_t n, int64_t head, int64_t nq, int l, int r, int wide,
                   unsigned long long* overflow, unsigned long long* mismatch) {
  static_assert(MT > 0, "compile-time m");
  auto pos = [&](int64_t j, const int64_t (&rot)[MT], int64_t (&orot)[MT]) {
    const bool ovf = recover_rot<MT>(rot, MT, l, wide != 0, orot);
    if (ovf && overflow) atomicAdd(overflow, 1ull);
    if (mismatch) {
      int64_t want = wadd(wshl(orot[MT - 1], l), orot[0]);
      if (sizeof(TI) == 4) want = (int64_t)(int32_t)(uint32_t)(uint64_t)want;
      if ((int64_t)__ldg(reinterpret_cast<const TI*>(delta.p[r]) + j) != want) atomicAdd(mismatch, 1ull);
    }
  };
  const int64_t stride = (int64_t)gridDim.x * EW_THREADS;
  for (int64_t q = (int64_t)blockIdx.x * EW_THREADS + threadIdx.x; q < nq; q += stride) {
    const int64_t j = head + 4 * q;
    int64_t in[MT - 1][4];
#pragma unroll
    for (int t = 0; t < MT - 1; ++t) {
      int row = r + 1 + t;
      row -= row >= MT ? MT : 0;
      load4(reinterpret_cast<const TI*>(delta.p[row]), j, in[t]);
    }
    int64_t res[MT][4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      int64_t rot[MT], orot[MT];
#pragma unroll
      for (int t = 0; t < MT - 1; ++t) rot[t] = in[t][k];
      rot[MT - 1] = 0;
      pos(j + k, rot, orot);
#pragma unroll
      for (int t = 0; t < MT; ++t) res[t][k] = orot[t];
    }
#pragma unroll
    for (int t = 0; t < MT; ++t) {
      int row = r + t;
      row -= row >= MT ? MT : 0;
      store4(reinterpret_cast<TO*>(out.p[row]), j, res[t]);
    }
  }
  if (blockIdx.x == 0) {  // the unaligned head [0, head) and the ragged tail [head + 4 nq, n)
    const int64_t tail0 = head + 4 * nq, ns = head + (n - tail0);
    for (int64_t k = threadIdx.x; k < ns; k += EW_THREADS) {
      const int64_t j = k < head ? k : tail0 + (k - head);
      int64_t rot[MT], orot[MT];
#pragma unroll
      for (int t = 0; t < MT - 1; ++t) {
        int row = r + 1 + t;
        row -= row >= MT ? MT : 0;
        rot[t] = (int64_t)__ldg(reinterpret_cast<const TI*>(delta.p[row]) + j);
      }
      rot[MT - 1] = 0;
      pos(j, rot, orot);
#pragma unroll
      for (int t = 0; t < MT; ++t) {
        int row = r + t;
        row -= row >= MT ? MT : 0;
        reinterpret_cast<TO*>(out.p[row])[j] = (TO)(uint64_t)orot[t];
      }
    }
  }
}

// The position `head` in [0, 4) at which every row (element width `bits`) is
// 16-byte aligned, or -1.
static int64_t common_head(const void* const* rows, int k, int bits, const void* const* rows2, int k2,
                           int bits2, int skip) {
  for (int64_t h = 0; h < 4; ++h) {
    bool ok = true;
    for (int i = 0; i < k && ok; ++i)
      if (i != skip && rows[i]) ok = ((reinterpret_cast<uintptr_t>(rows[i]) + h * (bits / 8)) & 15) == 0;
    for (int i = 0; i < k2 && ok; ++i)
      if (rows2[i]) ok = ((reinterpret_cast<uintptr_t>(rows2[i]) + h * (bits2 / 8)) & 15) == 0;
    if (ok) return h;
  }
  return -1;
}

// Independent m=3 recipe (codec.py:151-183).
template <typename TI, typename TO>
__global__ void __launch_bounds__(EW_THREADS)
extract_m3_kernel(const Rows delta, MutRows out, int64_t n, int l, int w, int r) {
  const TI* a = reinterpret_cast<const TI*>(delta.p[(r + 1) % 3]);
  const TI* b = reinterpret_cast<const TI*>(delta.p[(r + 2) % 3]);
  for (int64_t j = (int64_t)blockIdx.x * EW_THREADS + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * EW_THREADS) {
    int64_t av = (int64_t)__ldg(a + j), bv = (int64_t)__ldg(b + j);
    int64_t d2, d0;
    if (w <= 32) {
      int64_t dt = wsub(bv, wshl(av, l));
      if (w == 32) {
        int up = 2 * (w - l);
        d2 = (int64_t)((uint64_t)dt << up) >> up;
      } else {
        uint64_t mask = (((uint64_t)1) << (2 * l)) - 1, sb = ((uint64_t)1) << (2 * l - 1);
        d2 = (int64_t)((((uint64_t)dt & mask) ^ sb) - sb);
      }
      d0 = wneg(wsub(dt, d2)) >> (2 * l);
    } else {
      typedef unsigned __int128 u128;
      u128 dt = (u128)(__int128)bv - ((u128)(__int128)av << l);
      u128 mask = (((u128)1) << (2 * l)) - 1, sb = ((u128)1) << (2 * l - 1);
      u128 d2w = ((dt & mask) ^ sb) - sb;
      d2 = (int64_t)(uint64_t)d2w;
      d0 = (int64_t)((__int128)(d2w - dt) >> (2 * l));
    }
    reinterpret_cast<TO*>(out.p[(r + 2) % 3])[j] = (TO)(uint64_t)d2;
    reinterpret_cast<TO*>(out.p[r])[j] = (TO)(uint64_t)d0;
    reinterpret_cast<TO*>(out.p[(r + 1) % 3])[j] = (TO)(uint64_t)wsub(av, wshl(d0, l));
  }
}

// ------------------------------------------------------------------ helpers --
template <typename TO>
__global__ void poison_kernel(TO* y, int64_t n, int w) {
  const int64_t lo = (int64_t)(0 - ((uint64_t)1 << (w - 1)));
  const int64_t hi = (int64_t)(((uint64_t)1 << (w - 1)) - 1);
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x)
    y[j] = (TO)(uint64_t)((j & 1) ? hi : lo);
}

template <typename TI>
__global__ void __launch_bounds__(EW_THREADS)
max_abs_kernel(const Rows x, int rows, int64_t n, unsigned long long* out) {
  unsigned long long m = 0;
  for (int row = blockIdx.y; row < rows; row += gridDim.y) {
    const TI* p = reinterpret_cast<const TI*>(x.p[row]);
    for (int64_t j = (int64_t)blockIdx.x * EW_THREADS + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * EW_THREADS) {
      unsigned long long a = uabs((int64_t)__ldg(p + j));
      m = a > m ? a : m;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long v = __shfl_xor_sync(0xffffffffu, m, o);
    m = v > m ? v : m;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// First row-major index with |x| > hi (numpy's wrapping abs), as in
// codec._check_input_range / checksum_encode (codec.py:34-46, checksum.py:42-55).
template <typename TI>
__global__ void __launch_bounds__(EW_THREADS)
check_range_kernel(const Rows x, int64_t n, int64_t hi, unsigned long long* bad) {
  const int row = blockIdx.y;
  const TI* p = reinterpret_cast<const TI*>(x.p[row]);
  for (int64_t j = (int64_t)blockIdx.x * EW_THREADS + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * EW_THREADS)
    if (wabs((int64_t)__ldg(p + j)) > hi) atomicMin(bad, (unsigned long long)((int64_t)row * n + j));
}

template <typename TI, typename TO>
__global__ void checksum_encode_kernel(const Rows x, int m, int64_t n, TO* cs) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    uint64_t s = 0;
    for (int i = 0; i < m; ++i) s += (uint64_t)(int64_t)__ldg(reinterpret_cast<const TI*>(x.p[i]) + j);
    cs[j] = (TO)s;
  }
}

template <typename TI, typename TC, typename TO>
__global__ void checksum_recover_kernel(const Rows x, const TC* cs, int m, int64_t n, int failed,
                                        TO* out) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    uint64_t s = (uint64_t)(int64_t)__ldg(cs + j);
    for (int i = 0; i < m; ++i)
      if (i != failed) s -= (uint64_t)(int64_t)__ldg(reinterpret_cast<const TI*>(x.p[i]) + j);
    out[j] = (TO)s;
  }
}

}  // namespace nent

using namespace nent;

extern "C" {

const char* nent_last_error(void) { return g_err; }
int nent_abi_version(void) { return NENT_ABI_VERSION; }
int nent_last_conv_kernel(void) { return nent::g_last_conv_kernel; }

int nent_enable_peer_access(int peer) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) { set_error("no CUDA device"); return NENT_ERR_CUDA; }
  if (peer == dev) return NENT_OK;
  int can = 0;
  cudaDeviceCanAccessPeer(&can, dev, peer);
  if (!can) { set_error("device %d cannot access device %d", dev, peer); return NENT_ERR_CUDA; }
  const cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
    set_error("cudaDeviceEnablePeerAccess(%d): %s", peer, cudaGetErrorString(e));
    return NENT_ERR_CUDA;
  }
  cudaGetLastError();  // clear a sticky "already enabled"
  return NENT_OK;
}

int nent_device_ok(void) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) { set_error("no CUDA device"); return 0; }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) { set_error("cudaGetDeviceProperties failed"); return 0; }
  if (prop.major != 10 || prop.minor != 0) {
    set_error("library built for sm_100a, device is sm_%d%d", prop.major, prop.minor);
    return 0;
  }
  cudaFuncAttributes attr;
  if (cudaFuncGetAttributes(&attr, (const void*)poison_kernel<int64_t>) != cudaSuccess) {
    set_error("kernel image not loadable: %s", cudaGetErrorString(cudaGetLastError()));
    return 0;
  }
  return 1;
}

int nent_entangle(const void* const* src, int src_bits, void* const* eps, int eps_bits, int m,
                  int64_t n, int l, int64_t check_hi, uint64_t* bad_index_dev, void* stream) {
  NENT_CHECK_BITS(src_bits);
  NENT_CHECK_BITS(eps_bits);
  if (m < 1 || m > NENT_MAX_STREAMS || n < 0 || l < 0 || l > 63) {
    set_error("entangle: bad geometry m=%d n=%lld l=%d", m, (long long)n, l);
    return NENT_ERR_PARAM;
  }
  cudaStream_t s = as_stream(stream);
  int check = check_hi >= 0 && bad_index_dev != nullptr;
  if (check) cudaMemsetAsync(bad_index_dev, 0xff, sizeof(uint64_t), s);
  if (n == 0) return NENT_OK;
  Rows R = to_rows(src, m);
  MutRows W = to_mrows(eps, m);
  const int64_t head = n >= 64 ? common_head(src, m, src_bits, eps, m, eps_bits, -1) : -1;
  if (head >= 0 && (m == 3 || m == 4 || m == 8)) {  // all rows per thread: each word read once
    const int64_t nq = (n - head) / 4;
    const int grid = grid_for(nq, EW_THREADS, 1, 148 * 8);
#define NENT_ROWS_CASE(MT)                                                                     \
  DISPATCH_IO(src_bits, eps_bits,                                                              \
              (entangle_rows_kernel<MT, TI, TO><<<grid, EW_THREADS, 0, s>>>(                   \
                  R, W, n, head, nq, l, check_hi, check, (unsigned long long*)bad_index_dev)))
    if (m == 3) {
      NENT_ROWS_CASE(3);
    } else if (m == 4) {
      NENT_ROWS_CASE(4);
    } else {
      NENT_ROWS_CASE(8);
    }
#undef NENT_ROWS_CASE
    return check_launch("entangle");
  }
  if (head >= 0) {  // 16-byte vectors
    const int64_t nq = (n - head) / 4;
    dim3 grid(grid_for(nq, EW_THREADS, 2, 148 * 16 / (m > 4 ? 4 : 1)), m);
    DISPATCH_IO(src_bits, eps_bits,
                (entangle_vec_kernel<TI, TO><<<grid, EW_THREADS, 0, s>>>(
                    R, W, m, n, head, nq, l, check_hi, check, (unsigned long long*)bad_index_dev)));
    return check_launch("entangle");
  }
  dim3 grid(grid_for(n, EW_THREADS, EW_UNROLL, 148 * 16 / (m > 4 ? 4 : 1)), m);
  DISPATCH_IO(src_bits, eps_bits,
              (entangle_kernel<TI, TO><<<grid, EW_THREADS, 0, s>>>(
                  R, W, m, n, l, check_hi, check, (unsigned long long*)bad_index_dev)));
  return check_launch("entangle");
}

int nent_shift_add(const void* a, const void* b, int in_bits, void* out, int out_bits, int64_t n,
                   int l, void* stream) {
  NENT_CHECK_BITS(in_bits);
  NENT_CHECK_BITS(out_bits);
  if (n <= 0) return NENT_OK;
  cudaStream_t s = as_stream(stream);
  int grid = grid_for(n, EW_THREADS, 4);
  DISPATCH_IO(in_bits, out_bits,
              (shift_add_kernel<TI, TO><<<grid, EW_THREADS, 0, s>>>(
                  (const TI*)a, (const TI*)b, (TO*)out, n, l)));
  return check_launch("shift_add");
}

static int extract_impl(const void* const* delta, int delta_bits, void* const* out, int out_bits, int m,
                        int64_t n, int l, int r, int wide, unsigned long long* overflow_dev,
                        unsigned long long* mismatch_dev, void* stream) {
  NENT_CHECK_BITS(delta_bits);
  NENT_CHECK_BITS(out_bits);
  if (m < 3 || m > NENT_MAX_STREAMS || r < 0 || r >= m || l < 1 || (m - 1) * l > 63) {
    set_error("extract: bad geometry m=%d l=%d r=%d", m, l, r);
    return NENT_ERR_PARAM;
  }
  if (n <= 0) return NENT_OK;
  cudaStream_t s = as_stream(stream);
  Rows D = to_rows(delta, m);
  if (!mismatch_dev) D.p[r] = nullptr;  // the failed stream is never dereferenced
  else if (!D.p[r]) {
    set_error("extract_verify: the pivot row %d must be given", r);
    return NENT_ERR_PARAM;
  }
  MutRows O = to_mrows(out, m);
  // 16-byte vectors when every row read (all but the failed one, plus the
  // pivot when verifying) and every output row share an alignment phase
  const int64_t head = (n >= 64 && (m == 3 || m == 4 || m == 8))
                           ? common_head(D.p, m, delta_bits, O.p, m, out_bits, -1) : -1;
  if (head >= 0) {
    const int64_t nq = (n - head) / 4;
    const int vgrid = grid_for(nq, EW_THREADS, 1, 148 * 8);
#define EXTRACT_VEC_CASE(MTV)                                                                   \
  DISPATCH_IO(delta_bits, out_bits,                                                             \
              (extract_vec_kernel<MTV, TI, TO><<<vgrid, EW_THREADS, 0, s>>>(D, O, n, head, nq, l, r, wide, \
                                                                           overflow_dev, mismatch_dev)))
    switch (m) {
      case 3: EXTRACT_VEC_CASE(3); break;
      case 4: EXTRACT_VEC_CASE(4); break;
      default: EXTRACT_VEC_CASE(8); break;
    }
#undef EXTRACT_VEC_CASE
    return check_launch("extract");
  }
  int grid = grid_for(n, EW_THREADS, 4);
#define EXTRACT_CASE(MTV)                                                                  \
  DISPATCH_IO(delta_bits, out_bits,                                                        \
              (extract_kernel<MTV, TI, TO><<<grid, EW_THREADS, 0, s>>>(D, O, m, n, l, r, wide, \
                                                                      overflow_dev, mismatch_dev)))
  switch (m) {
    case 3: EXTRACT_CASE(3); break;
    case 4: EXTRACT_CASE(4); break;
    case 5: EXTRACT_CASE(5); break;
    case 8: EXTRACT_CASE(8); break;
    default: EXTRACT_CASE(0); break;
  }
#undef EXTRACT_CASE
  return check_launch("extract");
}

int nent_extract(const void* const* delta, int delta_bits, void* const* out, int out_bits, int m,
                 int64_t n, int l, int r, int wide, unsigned long long* overflow_dev, void* stream) {
  return extract_impl(delta, delta_bits, out, out_bits, m, n, l, r, wide, overflow_dev, nullptr, stream);
}

int nent_extract_verify(const void* const* delta, int delta_bits, void* const* out, int out_bits, int m,
                        int64_t n, int l, int pivot, int wide, unsigned long long* overflow_dev,
                        unsigned long long* mismatch_dev, void* stream) {
  if (!mismatch_dev) {
    set_error("extract_verify: mismatch counter required");
    return NENT_ERR_PARAM;
  }
  return extract_impl(delta, delta_bits, out, out_bits, m, n, l, pivot, wide, overflow_dev, mismatch_dev,
                      stream);
}

int nent_extract_m3(const void* const* delta, int delta_bits, void* const* out, int out_bits,
                    int64_t n, int l, int w, int r, void* stream) {
  NENT_CHECK_BITS(delta_bits);
  NENT_CHECK_BITS(out_bits);
  if (r < 0 || r > 2 || l < 1 || 2 * l > 63 + (w > 32 ? 64 : 0)) {
    set_error("extract_m3: bad parameters");
    return NENT_ERR_PARAM;
  }
  if (n <= 0) return NENT_OK;
  cudaStream_t s = as_stream(stream);
  Rows D = to_rows(delta, 3);
  D.p[r] = nullptr;
  MutRows O = to_mrows(out, 3);
  int grid = grid_for(n, EW_THREADS, 4);
  DISPATCH_IO(delta_bits, out_bits,
              (extract_m3_kernel<TI, TO><<<grid, EW_THREADS, 0, s>>>(D, O, n, l, w, r)));
  return check_launch("extract_m3");
}

int nent_poison(void* y, int y_bits, int64_t n, int w, void* stream) {
  NENT_CHECK_BITS(y_bits);
  if (w < 2 || w > 64) { set_error("poison: bad w=%d", w); return NENT_ERR_PARAM; }
  if (n <= 0) return NENT_OK;
  cudaStream_t s = as_stream(stream);
  int grid = grid_for(n, 256, 4);
  if (y_bits == 32) poison_kernel<int32_t><<<grid, 256, 0, s>>>((int32_t*)y, n, w);
  else poison_kernel<int64_t><<<grid, 256, 0, s>>>((int64_t*)y, n, w);
  return check_launch("poison");
}

int nent_max_abs(const void* const* x, int x_bits, int rows, int64_t n, uint64_t* out_dev,
                 void* stream) {
  NENT_CHECK_BITS(x_bits);
  if (rows < 0 || rows > NENT_MAX_STREAMS) { set_error("max_abs: bad rows"); return NENT_ERR_PARAM; }
  cudaStream_t s = as_stream(stream);
  cudaMemsetAsync(out_dev, 0, sizeof(uint64_t), s);
  if (rows == 0 || n <= 0) return check_launch("max_abs");
  Rows R = to_rows(x, rows);
  dim3 grid(grid_for(n, EW_THREADS, 8, 148 * 8), rows);
  if (x_bits == 32) max_abs_kernel<int32_t><<<grid, EW_THREADS, 0, s>>>(R, rows, n, (unsigned long long*)out_dev);
  else max_abs_kernel<int64_t><<<grid, EW_THREADS, 0, s>>>(R, rows, n, (unsigned long long*)out_dev);
  return check_launch("max_abs");
}

int nent_check_range(const void* const* x, int x_bits, int rows, int64_t n, int64_t hi,
                     uint64_t* bad_index_dev, void* stream) {
  NENT_CHECK_BITS(x_bits);
  if (rows < 1 || rows > NENT_MAX_STREAMS || hi < 0) { set_error("check_range: bad arguments"); return NENT_ERR_PARAM; }
  cudaStream_t s = as_stream(stream);
  cudaMemsetAsync(bad_index_dev, 0xff, sizeof(uint64_t), s);
  if (n <= 0) return check_launch("check_range");
  Rows R = to_rows(x, rows);
  dim3 grid(grid_for(n, EW_THREADS, 4, 148 * 8), rows);
  if (x_bits == 32) check_range_kernel<int32_t><<<grid, EW_THREADS, 0, s>>>(R, n, hi, (unsigned long long*)bad_index_dev);
  else check_range_kernel<int64_t><<<grid, EW_THREADS, 0, s>>>(R, n, hi, (unsigned long long*)bad_index_dev);
  return check_launch("check_range");
}

int nent_checksum_encode(const void* const* x, int x_bits, int m, int64_t n, void* cs,
                         int cs_bits, void* stream) {
  NENT_CHECK_BITS(x_bits);
  NENT_CHECK_BITS(cs_bits);
  if (m < 1 || m > NENT_MAX_STREAMS) { set_error("checksum_encode: bad m"); return NENT_ERR_PARAM; }
  if (n <= 0) return NENT_OK;
  cudaStream_t s = as_stream(stream);
  Rows R = to_rows(x, m);
  int grid = grid_for(n, 256, 4);
  DISPATCH_IO(x_bits, cs_bits,
              (checksum_encode_kernel<TI, TO><<<grid, 256, 0, s>>>(R, m, n, (TO*)cs)));
  return check_launch("checksum_encode");
}

int nent_checksum_recover(const void* const* x, int x_bits, const void* cs, int cs_bits, int m,
                          int64_t n, int failed, void* out, int out_bits, void* stream) {
  NENT_CHECK_BITS(x_bits);
  NENT_CHECK_BITS(cs_bits);
  NENT_CHECK_BITS(out_bits);
  if (m < 1 || m > NENT_MAX_STREAMS || failed < 0 || failed >= m) {
    set_error("checksum_recover: bad failed=%d for m=%d", failed, m);
    return NENT_ERR_PARAM;
  }
  if (n <= 0) return NENT_OK;
  cudaStream_t s = as_stream(stream);
  Rows R = to_rows(x, m);
  R.p[failed] = nullptr;
  int grid = grid_for(n, 256, 4);
  if (cs_bits == 64) {
    DISPATCH_IO(x_bits, out_bits,
                (checksum_recover_kernel<TI, int64_t, TO><<<grid, 256, 0, s>>>(
                    R, (const int64_t*)cs, m, n, failed, (TO*)out)));
  } else {
    DISPATCH_IO(x_bits, out_bits,
                (checksum_recover_kernel<TI, int32_t, TO><<<grid, 256, 0, s>>>(
                    R, (const int32_t*)cs, m, n, failed, (TO*)out)));
  }
  return check_launch("checksum_recover");
}

int nent_copy_rows(void* dst, int64_t dst_pitch, const void* src, int64_t src_pitch,
                   int64_t width_bytes, int rows, int direction, void* stream) {
  static const cudaMemcpyKind kinds[4] = {cudaMemcpyDefault, cudaMemcpyHostToDevice,
                                          cudaMemcpyDeviceToHost, cudaMemcpyDeviceToDevice};
  if (direction < 1 || direction > 3 || rows < 0 || width_bytes < 0 ||
      (rows > 1 && (dst_pitch < width_bytes || src_pitch < width_bytes))) {
    set_error("copy_rows: bad direction %d / geometry (%lld x %d, pitches %lld, %lld)", direction,
              (long long)width_bytes, rows, (long long)dst_pitch, (long long)src_pitch);
    return NENT_ERR_PARAM;
  }
  if (rows == 0 || width_bytes == 0) return NENT_OK;
  const size_t dp = rows > 1 ? (size_t)dst_pitch : (size_t)width_bytes;
  const size_t sp = rows > 1 ? (size_t)src_pitch : (size_t)width_bytes;
  cudaError_t e = cudaMemcpy2DAsync(dst, dp, src, sp, (size_t)width_bytes, (size_t)rows,
                                    kinds[direction], as_stream(stream));
  if (e != cudaSuccess) {
    set_error("copy_rows: %s", cudaGetErrorString(e));
    return NENT_ERR_CUDA;
  }
  return NENT_OK;
}

}  // extern "C"
