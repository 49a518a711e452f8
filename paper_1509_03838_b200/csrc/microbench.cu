// microbench.cu -- measured peaks of the MAC flavours (roofline denominators).
//
// MEASURED_PEAKS.json has HBM and bf16 only; the conv kernel is bound by the
// integer / FP64 pipes, so its denominators are measured here on the same box:
// 16 independent accumulators per thread keep the pipe saturated and the count
// of issued MACs exact.
#include "common.cuh"
#include "tc05.cuh"

namespace nent {

constexpr int MB_CHAINS = 16;

__device__ __forceinline__ long long mad_wide_s32(int a, int b, long long c) {
  long long d;
  asm volatile("mad.wide.s32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
  return d;
}

// Every iteration draws one pseudo-random multiplicand x (an LCG step, one
// extra IMAD shared by the 16 MACs, so the product can be neither hoisted nor
// strength-reduced) and feeds 16 independent accumulators acc[c] += x * g[c],
// the exact operand pattern of the convolution's inner loop.
template <int FLAV>
__global__ void __launch_bounds__(256) microbench_kernel(int iters, unsigned long long* sink, int k) {
  const unsigned tid = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t x = tid * 2654435761u + (uint32_t)k;
  int32_t g[MB_CHAINS];
#pragma unroll
  for (int c = 0; c < MB_CHAINS; ++c) g[c] = (int32_t)(tid ^ (c * 0x9e37u)) | 1;
  unsigned long long s = 0;
  if (FLAV == NENT_MAC_I32) {
    uint32_t a[MB_CHAINS] = {};
    for (int it = 0; it < iters; ++it) {
      x = x * 1664525u + 1013904223u;
#pragma unroll
      for (int c = 0; c < MB_CHAINS; ++c) a[c] += x * (uint32_t)g[c];
    }
#pragma unroll
    for (int c = 0; c < MB_CHAINS; ++c) s ^= a[c];
  } else if (FLAV == NENT_MAC_W64) {
    long long a[MB_CHAINS] = {};
    for (int it = 0; it < iters; ++it) {
      x = x * 1664525u + 1013904223u;
#pragma unroll
      for (int c = 0; c < MB_CHAINS; ++c) a[c] = mad_wide_s32((int)x, g[c], a[c]);
    }
#pragma unroll
    for (int c = 0; c < MB_CHAINS; ++c) s ^= (unsigned long long)a[c];
  } else if (FLAV == NENT_MAC_S64) {
    long long lo[MB_CHAINS] = {};
    uint32_t hi[MB_CHAINS] = {};
    for (int it = 0; it < iters; ++it) {
      x = x * 1664525u + 1013904223u;
      const uint32_t xh = x >> 7;
#pragma unroll
      for (int c = 0; c < MB_CHAINS; ++c) {
        lo[c] = mad_wide_s32((int)x, g[c], lo[c]);  // IMAD.WIDE on the low word
        hi[c] += xh * (uint32_t)g[c];               // IMAD on the high word
      }
    }
#pragma unroll
    for (int c = 0; c < MB_CHAINS; ++c) s ^= (unsigned long long)lo[c] ^ hi[c];
  } else if (FLAV == NENT_MAC_F64) {
    double a[MB_CHAINS] = {};
    double xd = (double)(tid & 1023);
    for (int it = 0; it < iters; ++it) {
      xd = fma(xd, 0.999999, 1.0);
#pragma unroll
      for (int c = 0; c < MB_CHAINS; ++c) a[c] = fma(xd, (double)g[c], a[c]);
    }
#pragma unroll
    for (int c = 0; c < MB_CHAINS; ++c) s ^= (unsigned long long)__double_as_longlong(a[c]);
  } else {
    unsigned long long a[MB_CHAINS] = {};
    unsigned long long X = ((unsigned long long)tid << 32) | x;
    for (int it = 0; it < iters; ++it) {
      X = X * 6364136223846793005ull + 1442695040888963407ull;
#pragma unroll
      for (int c = 0; c < MB_CHAINS; ++c) a[c] += X * (unsigned long long)(long long)g[c];
    }
#pragma unroll
    for (int c = 0; c < MB_CHAINS; ++c) s ^= a[c];
  }
  if (s == (unsigned long long)k * 0x9e3779b97f4a7c15ull) sink[tid & 1023] = s;
}

// Legacy warp-level integer tensor-core MMA (IMMA, mma.sync m16n8k32 s8*s8+s32):
// 16 independent accumulator fragments per warp; 4096 MACs per instruction.
__global__ void __launch_bounds__(256) microbench_imma_kernel(int iters, unsigned long long* sink, int k) {
  const unsigned tid = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t a0 = tid * 0x01010101u + k, a1 = a0 ^ 0x5a5a5a5au, a2 = a0 + 0x11111111u, a3 = a0 * 3u;
  uint32_t b0 = tid ^ 0x3c3c3c3cu, b1 = b0 + (uint32_t)k;
  int acc[MB_CHAINS][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < MB_CHAINS; ++c)
      asm volatile(
          "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+r"(acc[c][0]), "+r"(acc[c][1]), "+r"(acc[c][2]), "+r"(acc[c][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    a0 += 0x01020304u;
  }
  unsigned long long s = 0;
#pragma unroll
  for (int c = 0; c < MB_CHAINS; ++c) s ^= (unsigned)(acc[c][0] ^ acc[c][1] ^ acc[c][2] ^ acc[c][3]);
  if (s == (unsigned long long)k * 0x9e3779b97f4a7c15ull) sink[tid & 1023] = s;
}

// 5th-generation tensor cores: tcgen05.mma kind::i8, M=128 x N=128 x K=32 per
// instruction, A from TMEM, B from shared memory, one CTA per SM, the elected
// lane of warp 0 issuing 12-step K chains back to back (the conv kernel's
// issue shape at its largest N).  Operand contents are irrelevant to timing.
__global__ void __launch_bounds__(128, 1) microbench_tc05_kernel(int iters, unsigned long long* sink) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) tc05::alloc(&tslot, 512);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tc05::smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < 128 * 128 + 512; i += blockDim.x) smem[i] = (unsigned char)(i * 7 + 1);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc05::fence_before();
  __syncthreads();
  tc05::fence_after();
  const uint32_t tbase = tslot;
  if (warp == 0) {
    const uint32_t idesc = tc05::idesc_i8(128, 128, false);
    const uint32_t blo = tc05::desc_sw128_lo(tc05::smem_u32(smem));
    for (int it = 0; it < iters; ++it) {
      uint32_t e;
      asm volatile("{\n .reg .pred p;\n elect.sync _|p, 0xffffffff;\n selp.u32 %0, 1, 0, p;\n}" : "=r"(e));
      if (e) {
#pragma unroll
        for (int kc = 0; kc < 12; ++kc) tc05::mma_i8_ts_lo(tbase + 128, tbase + 8u * kc, blo + 2u * kc, idesc, 1u);
      }
      __syncwarp();
    }
    tc05::commit_elect(tc05::smem_u32(&mbar));
    asm volatile(
        "{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W_%=;\n}" ::"r"(
            tc05::smem_u32(&mbar))
        : "memory");
  }
  tc05::fence_before();
  __syncthreads();
  if (warp == 0) {
    tc05::fence_after();
    uint32_t r[16];
    tc05::ld_x16(tbase + ((uint32_t)(32 * (warp & 3)) << 16) + 128, r);
    tc05::wait_ld();
    if (r[0] == 0x12345678u && r[1] == 0x9abcdef0u) sink[blockIdx.x & 1023] = r[2];
    tc05::dealloc(tbase, 512);
  }
}

}  // namespace nent

using namespace nent;

extern "C" int nent_microbench(int kind, int blocks, int threads, int iters,
                               unsigned long long* sink_dev, double* macs_out, void* stream) {
  if (blocks < 1 || threads < 32 || threads > 256 || iters < 1) {
    set_error("microbench: bad launch");
    return NENT_ERR_PARAM;
  }
  cudaStream_t s = as_stream(stream);
  const int k = 3;
  double per_thread = (double)iters * MB_CHAINS;
  switch (kind) {
    case NENT_MAC_I32: microbench_kernel<NENT_MAC_I32><<<blocks, threads, 0, s>>>(iters, sink_dev, k); break;
    case NENT_MAC_W64: microbench_kernel<NENT_MAC_W64><<<blocks, threads, 0, s>>>(iters, sink_dev, k); break;
    case NENT_MAC_S64: microbench_kernel<NENT_MAC_S64><<<blocks, threads, 0, s>>>(iters, sink_dev, k); break;
    case NENT_MAC_F64: microbench_kernel<NENT_MAC_F64><<<blocks, threads, 0, s>>>(iters, sink_dev, k); break;
    case NENT_MAC_G64: microbench_kernel<NENT_MAC_G64><<<blocks, threads, 0, s>>>(iters, sink_dev, k); break;
    case NENT_BENCH_IMMA:
      microbench_imma_kernel<<<blocks, threads, 0, s>>>(iters, sink_dev, k);
      per_thread = (double)iters * MB_CHAINS * (16.0 * 8 * 32 / 32);  // 4096 MACs per warp-MMA
      break;
    case NENT_BENCH_TC05: {
      const int smem = 128 * 128 + 512 + 1024;
      cudaFuncSetAttribute(microbench_tc05_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      microbench_tc05_kernel<<<blocks, 128, smem, s>>>(iters, sink_dev);
      if (macs_out) *macs_out = (double)iters * 12 * 128.0 * 128.0 * 32.0 * (double)blocks;
      return check_launch("microbench tc05");
    }
    default: set_error("microbench: unknown kind %d", kind); return NENT_ERR_PARAM;
  }
  if (macs_out) *macs_out = per_thread * (double)blocks * (double)threads;
  return check_launch("microbench");
}
