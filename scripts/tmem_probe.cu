// TMEM read (tcgen05.ld) throughput per SM: W warps each loading 32 lanes x
// NCOL columns (32x32b.xNCOL) per round, `rounds` times, one CTA per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tmem_probe tmem_probe.cu
#include <cstdio>
#include <cstdint>
#include "../paper_1509_03838_b200/csrc/tc05.cuh"
using namespace nent;

template <int NW, int DEPTH>
__global__ void __launch_bounds__(NW * 32, 1) ldtm_probe(int rounds, uint32_t* sink, long long* cyc) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tc05::alloc(&tslot, 512);
  tc05::fence_before();
  __syncthreads();
  tc05::fence_after();
  const uint32_t lrow = (uint32_t)(32 * (warp & 3)) << 16;
  uint32_t acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < rounds; ++it) {
    uint32_t r[DEPTH][32];
#pragma unroll
    for (int d = 0; d < DEPTH; ++d) tc05::ld_x32(lrow + (uint32_t)(32 * ((warp / 4 + d + it) & 15)), r[d]);
    tc05::wait_ld();
#pragma unroll
    for (int d = 0; d < DEPTH; ++d)
#pragma unroll
      for (int i = 0; i < 32; ++i) acc += r[d][i];
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) atomicAdd((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
  if (acc == 0x12345678u) sink[threadIdx.x] = acc;
  tc05::fence_before();
  __syncthreads();
  if (warp == 0) {
    tc05::fence_after();
    tc05::dealloc(tslot, 512);
  }
}

template <int NW, int DEPTH>
void run(int sms) {
  uint32_t* sink;
  long long* cyc;
  cudaMalloc(&sink, 4096);
  cudaMalloc(&cyc, 8);
  const int rounds = 2000;
  ldtm_probe<NW, DEPTH><<<sms, NW * 32>>>(10, sink, cyc);
  cudaMemset(cyc, 0, 8);
  ldtm_probe<NW, DEPTH><<<sms, NW * 32>>>(rounds, sink, cyc);
  long long h = 0;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  const double per_round = (double)h / sms / rounds;
  const double bytes = (double)NW * DEPTH * 32 * 32 * 4;
  printf("warps %2d depth %d: %.1f cyc/round, %.1f B/cyc/SM (err %s)\n", NW, DEPTH, per_round, bytes / per_round,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(sink);
  cudaFree(cyc);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<4, 1>(sms); run<4, 2>(sms); run<4, 4>(sms);
  run<8, 1>(sms); run<8, 2>(sms);
  run<16, 1>(sms); run<16, 2>(sms);
  return 0;
}
