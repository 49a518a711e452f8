// Probe: cycles per tcgen05.mma kind::i8 (M = 128, A in TMEM, B from shared
// memory) as a function of N, issued as fully unrolled 12-step K chains by one
// elected lane.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
//   -I paper_1509_03838_b200/csrc scripts/mma_n_probe.cu -o scripts/_bin/mma_n_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "tc05.cuh"
using namespace nent;

template <int N, int MODE>
__global__ void __launch_bounds__(128, 1) probe(int iters, long long* out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t mbar;
  __shared__ __align__(8) uint64_t mbar2[8];
  __shared__ __align__(8) uint64_t mbar3[8];  // never arrived on: parity-1 waits return at once
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) tc05::alloc(&tslot, 512);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tc05::smem_u32(&mbar)));
    for (int i = 0; i < 8; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tc05::smem_u32(&mbar2[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tc05::smem_u32(&mbar3[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < 128 * 256 + 512; i += blockDim.x) smem[i] = (unsigned char)(i * 7 + 1);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc05::fence_before();
  __syncthreads();
  tc05::fence_after();
  const uint32_t tbase = tslot;
  if (warp == 0) {
    const uint32_t idesc = tc05::idesc_i8(128, N, false);
    const uint32_t blo = tc05::desc_sw128_lo(tc05::smem_u32(smem));
    uint32_t e;
    asm volatile("{\n .reg .pred p;\n elect.sync _|p, 0xffffffff;\n selp.u32 %0, 1, 0, p;\n}" : "=r"(e));
    long long t0 = 0, t1 = 0;
    if (e) {
      t0 = clock64();
      for (int it = 0; it < iters; ++it) {
        // alternate between accumulator slots like the conv kernel's ring
        const uint32_t d = tbase + 192 + (uint32_t)((it % (320 / N)) * N);
        if (MODE >= 2) {
          // the conv kernel's per-class hand-off: poll a barrier that is
          // already complete (parity of the phase before the first), fence
          uint32_t ok;
          asm volatile("{\n .reg .pred p;\n W2_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 1;\n @!p bra W2_%=;\n selp.u32 %0, 1, 0, p;\n}"
                       : "=r"(ok) : "r"(tc05::smem_u32(&mbar3[it & 7])) : "memory");
          tc05::fence_after();
        }
#pragma unroll
        for (int kc = 0; kc < 12; ++kc) tc05::mma_i8_ts_lo(d, tbase + 8u * kc, blo + 2u * kc, idesc, kc ? 1u : 0u);
        if (MODE >= 1) tc05::commit(tc05::smem_u32(&mbar2[it & 7]));  // (arrivals on unrelated barriers)
      }
      tc05::commit(tc05::smem_u32(&mbar));
      asm volatile(
          "{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W_%=;\n}" ::"r"(
              tc05::smem_u32(&mbar))
          : "memory");
      t1 = clock64();
      if (blockIdx.x == 0) out[0] = t1 - t0;
    }
    __syncwarp();
  }
  tc05::fence_before();
  __syncthreads();
  if (warp == 0) {
    tc05::fence_after();
    tc05::dealloc(tbase, 512);
  }
}

template <int N, int MODE>
void run(int iters) {
  long long* d;
  cudaMalloc(&d, 8);
  const int smem = 128 * 256 + 512 + 1024;
  cudaFuncSetAttribute(probe<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<N, MODE><<<148, 128, smem>>>(64, d);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  probe<N, MODE><<<148, 128, smem>>>(iters, d);
  cudaEventRecord(b);
  cudaDeviceSynchronize();
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double n = (double)iters * 12;
  printf("mode %d N=%3d: %.2f clock64-cycles per MMA, %.2f ns per MMA (event), %.1f TMAC/s chip, err=%s\n", MODE, N, h / n,
         ms * 1e6 / n, n * 128.0 * N * 32 * 148 / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  fflush(stdout);
  cudaFree(d);
}

int main() {
  run<16, 0>(4000);
  run<32, 0>(4000);
  run<48, 0>(4000);
  run<64, 0>(4000);
  run<96, 0>(4000);
  run<128, 0>(4000);
  run<256, 0>(2000);
  // mode 1: a commit after every 12-step chain; mode 2: + barrier poll and fence before it
  run<32, 1>(4000);
  run<64, 1>(4000);
  run<32, 2>(4000);
  run<64, 2>(4000);
  return 0;
}
