// tcgen05 kind::i8 probe: correctness of the Hankel-B / Toeplitz-A layout the
// conv kernel relies on (B = a linear digit plane with rows 128 B apart, read
// through a K-major SWIZZLE_128B descriptor whose start advances by 32 B per
// K step and by whole rows; A from TMEM or from shared memory), plus MMA
// throughput per N.   nvcc -gencode arch=compute_100a,code=sm_100a -o tc_probe tc_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>

#include "../paper_1509_03838_b200/csrc/tc05.cuh"

using namespace nent;

__device__ __forceinline__ void mbar_init(uint32_t mb) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t mb, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(mb), "r"(phase) : "memory");
}

__device__ __forceinline__ bool elect_one_probe() {
  uint32_t e;
  asm volatile("{\n .reg .pred p;\n elect.sync _|p, 0xffffffff;\n selp.u32 %0, 1, 0, p;\n}" : "=r"(e));
  return e != 0;
}

constexpr int KT = 384;  // K of the Toeplitz GEMM (12 steps of 32)
constexpr int KC = KT / 32;

// mode 0: A from TMEM, mode 1: A from smem (K-major SW128, 3 atoms of 128x128)
__global__ void __launch_bounds__(128, 1)
probe(const int8_t* A, const int8_t* B, int N, int row0, int reps, int mode, int nacc, int32_t* D, long long* cycles) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  unsigned char* bs = smem;                    // B plane: (N + row0) rows of 128 B + 256 B tail
  const int bbytes = 128 * (N + row0) + 256 + 1024;
  unsigned char* as = smem + (bbytes + 1023) / 1024 * 1024;  // A atoms (mode 1)
  if (warp == 0) tc05::alloc(&tslot, 512);
  if (tid == 0) mbar_init(tc05::smem_u32(&mbar));
  // B: logical byte L of the plane -> physical sw128(L)
  for (int L = tid; L < 128 * (N + row0) + 256; L += 128) bs[tc05::sw128(L)] = (unsigned char)B[L];
  if (mode == 1)
    for (int i = tid; i < 128 * KT; i += 128) {
      const int v = i / KT, k = i % KT;
      as[(k / 128) * 16384 + tc05::sw128(v * 128 + (k % 128))] = (unsigned char)A[i];
    }
  tc05::fence_before();
  __syncthreads();
  tc05::fence_after();
  const uint32_t tbase = tslot;
  const uint32_t a_tm = tbase;          // columns [0, 96): A, 8 per K step
  const uint32_t d_tm = tbase + 128;    // columns [128, 128 + N): D
  if (mode == 0) {
    const int v = 32 * warp + lane;
#pragma unroll 1
    for (int kc = 0; kc < KC; ++kc) {
      uint32_t r[8];
      for (int c = 0; c < 8; ++c) {
        const int8_t* p = A + v * KT + 32 * kc + 4 * c;
        r[c] = (uint32_t)(uint8_t)p[0] | ((uint32_t)(uint8_t)p[1] << 8) | ((uint32_t)(uint8_t)p[2] << 16) |
               ((uint32_t)(uint8_t)p[3] << 24);
      }
      tc05::st_x8(tbase + ((uint32_t)(32 * warp) << 16) + 8 * kc, r);
    }
    tc05::wait_st();
  }
  tc05::fence_before();
  __syncthreads();
  tc05::fence_after();
  long long t0 = 0, t1 = 0;
  if (tid == 0) {
    const uint32_t idesc = tc05::idesc_i8(128, N);
    const uint32_t b0 = tc05::smem_u32(bs) + 128 * row0;
    const uint32_t a0 = tc05::smem_u32(as);
    t0 = clock64();
    for (int rep = 0; rep < reps; ++rep)
#pragma unroll
      for (int kc = 0; kc < KC; ++kc) {
        const uint64_t bd = tc05::desc_sw128(b0 + 32 * kc);
#pragma unroll 1
        for (int a = 0; a < nacc; ++a) {
          if (mode == 0)
            tc05::mma_i8_ts(d_tm + a * N, a_tm + 8 * kc, bd, idesc, (rep | kc) != 0);
          else
            tc05::mma_i8_ss(d_tm + a * N, tc05::desc_sw128(a0 + (kc / 4) * 16384 + (kc % 4) * 32), bd, idesc,
                            (rep | kc) != 0);
        }
      }
    tc05::commit(tc05::smem_u32(&mbar));
  }
  mbar_wait(tc05::smem_u32(&mbar), 0);
  if (tid == 0) {
    t1 = clock64();
    *cycles = t1 - t0;
  }
  tc05::fence_after();
  const int v = 32 * warp + lane;
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t r[16];
    tc05::ld_x16(d_tm + ((uint32_t)(32 * warp) << 16) + c0, r);
    tc05::wait_ld();
    for (int c = 0; c < 16 && c0 + c < N; ++c) D[v * N + c0 + c] = (int32_t)r[c];
  }
  tc05::fence_before();
  __syncthreads();
  if (warp == 0) tc05::dealloc(tbase, 512);
}

// throughput only: NACC accumulators x 12 K steps, fully unrolled, descriptors hoisted
template <int N, int MODE, int NACC, bool SAMEB, int CE>
__global__ void __launch_bounds__(128, 1) tput(int reps, long long* cycles, int doff) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t mbar, mbar2;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) tc05::alloc(&tslot, 512);
  if (tid == 0) {
    mbar_init(tc05::smem_u32(&mbar));
    mbar_init(tc05::smem_u32(&mbar2));
  }
  for (int i = tid; i < 16384 * 3 + 128 * (N + 4); i += 128) smem[i] = (unsigned char)(i * 7);
  tc05::fence_before();
  __syncthreads();
  tc05::fence_after();
  const uint32_t tbase = tslot;
  if (tid == 0) {
    constexpr uint32_t idesc = tc05::idesc_i8(128, N);
    const uint32_t b0 = tc05::smem_u32(smem) + 3 * 16384, a0 = tc05::smem_u32(smem);
    uint64_t bd[KC], ad[KC];
#pragma unroll
    for (int kc = 0; kc < KC; ++kc) {
      bd[kc] = tc05::desc_sw128(b0 + (SAMEB ? 0 : 32 * kc));
      ad[kc] = tc05::desc_sw128(a0 + (kc / 4) * 16384 + (kc % 4) * 32);
    }
    const long long t0 = clock64();
    for (int rep = 0; rep < reps; ++rep)
#pragma unroll
      for (int kc = 0; kc < KC; ++kc)
#pragma unroll
        for (int a = 0; a < NACC; ++a) {
          if (MODE == 0)
            tc05::mma_i8_ts(tbase + doff + a * N, tbase + 8 * kc, bd[kc], idesc, 1);
          else
            tc05::mma_i8_ss(tbase + doff + a * N, ad[kc], bd[kc], idesc, 1);
          if (CE && (kc + 1) % (CE ? CE : 1) == 0) tc05::commit(tc05::smem_u32(&mbar2));
        }
    tc05::commit(tc05::smem_u32(&mbar));
    mbar_wait(tc05::smem_u32(&mbar), 0);
    *cycles = clock64() - t0;
  }
  __syncthreads();
  if (warp == 0) tc05::dealloc(tbase, 512);
}

template <int N, int MODE, int NACC, bool SAMEB, int CE = 0>
void run_tput(int grid = 1) {
  const int commit_every = CE;
  long long* dc;
  cudaMalloc(&dc, 8);
  const int smem = 3 * 16384 + 128 * (N + 4) + 1024;
  cudaFuncSetAttribute(tput<N, MODE, NACC, SAMEB, CE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int reps = 2000;
  tput<N, MODE, NACC, SAMEB, CE><<<grid, 128, smem>>>(reps, dc, getenv("DOFF") ? atoi(getenv("DOFF")) : 128);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  tput<N, MODE, NACC, SAMEB, CE><<<grid, 128, smem>>>(reps, dc, getenv("DOFF") ? atoi(getenv("DOFF")) : 128);
  cudaEventRecord(e1);
  cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long cyc;
  cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  printf("commit_every %d ", commit_every);
  printf("tput %s N %3d nacc %d sameB %d grid %d: %.1f cyc/MMA (floor %d), %.3f ms, %.2f GHz effective\n",
         MODE ? "SS" : "TS", N, NACC, (int)SAMEB, grid, (double)cyc / (reps * KC * NACC), 128 * N / 256, ms,
         cyc / (ms * 1e6));
  cudaFree(dc);
}

// The conv kernel's MMA issue pattern alone: 2 plane slots x NP=5 planes of
// 9216 B, taps in TMEM [0,192) (2 digits x 12 K steps), a ring of 3 accumulator
// slots at column 320, classes p+j, commit per class (no waiting).
// VARIANT 0: MMA warp alone; 2: + 8 warps of ALU work (IMAD.WIDE chains);
// 3: + 8 warps streaming tcgen05.ld of the accumulator ring; 4: + 8 warps of
// STS traffic to shared memory
template <int VARIANT, int NSL = 3>
__global__ void __launch_bounds__(512, 1) convlike(int streams, long long* cycles, unsigned long long* sink, int nsteps_rt, int getenv_nowait) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t mbar, mbar2, accf[5], acce[5];
  __shared__ int stop_flag;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) tc05::alloc(&tslot, 512);
  if (tid == 0) {
    mbar_init(tc05::smem_u32(&mbar));
    mbar_init(tc05::smem_u32(&mbar2));
    for (int i = 0; i < 5; ++i) {
      mbar_init(tc05::smem_u32(&accf[i]));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(tc05::smem_u32(&acce[i])));
    }
    stop_flag = 0;
  }
  for (int i = tid; i < 2 * 5 * 9216; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u;
    h ^= h >> 15;
    smem[i] = VARIANT == 7 ? (unsigned char)(h * 0x2c1b3c6du >> 24) : (unsigned char)(i * 7);
  }
  if (VARIANT == 7 && warp < 4) {  // random taps in TMEM columns [0, 192)
    for (int blk = 0; blk < 24; ++blk) {
      uint32_t w[8];
      for (int c = 0; c < 8; ++c) {
        uint32_t h = (uint32_t)(tid * 977 + blk * 131 + c) * 2654435761u;
        h ^= h >> 13;
        w[c] = h * 0x85ebca6bu;
      }
      tc05::st_x8(((uint32_t)(32 * warp) << 16) + 8u * blk, w);
    }
    tc05::wait_st();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc05::fence_before();
  __syncthreads();
  tc05::fence_after();
  if (VARIANT == 10) {  // the conv kernel's register split
    if (warp >= 4 && warp < 12) asm volatile("setmaxnreg.inc.sync.aligned.u32 168;");
    else asm volatile("setmaxnreg.dec.sync.aligned.u32 88;");
  }
  if (VARIANT == 11 && warp == 0) {  // the conv kernel's MMA loop, verbatim structure
    constexpr int NP = 5, NG = 2, NCLS = 6, NSTEPS = 12, SLOTS = NSL, U = 64, PLANE = 9216;
    const uint32_t idesc = tc05::idesc_i8(128, U, false);
    const uint32_t planes_s = tc05::smem_u32(smem);
    const uint32_t tbase = 0, RING0 = 512 - 64 * NSL;
    const bool skip = nsteps_rt == 99;
    const long long t0 = clock64();
    int seq = 0, cls = 0;
    const int64_t ntiles = 2049;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      for (int q = 0; q < 3; ++q, ++seq, cls += NCLS) {
        const int slot = seq & 1;
        for (int p = 0; p < NP; ++p) {
          const uint32_t blo0 = tc05::desc_sw128_lo(planes_s + (uint32_t)((slot * NP + p) * PLANE));
          for (int j = 0; j < NG; ++j) {
            const int c = p + j;
            const int k = cls + c;
            const int rs = k % SLOTS;
            const bool first = p == (c - NG + 1 > 0 ? c - NG + 1 : 0);
            const uint32_t d = tbase + (uint32_t)(RING0 + rs * U);
            const uint32_t a = tbase + (uint32_t)(8 * j * NSTEPS);
            if (!skip && elect_one_probe()) {
#pragma unroll
              for (int kc = 0; kc < NSTEPS; ++kc)
                tc05::mma_i8_ts_lo(d, a + 8u * kc, blo0 + 2u * kc, idesc, (first && kc == 0) ? 0u : 1u);
            }
            __syncwarp();
            if (p == (c < NP - 1 ? c : NP - 1)) tc05::commit_elect(tc05::smem_u32(&mbar2));
          }
        }
      }
    }
    tc05::commit_elect(tc05::smem_u32(&mbar));
    mbar_wait(tc05::smem_u32(&mbar), 0);
    if (threadIdx.x == 0) {
      *cycles = (clock64() - t0) * 5040 / (seq * 120);
      stop_flag = 1;
    }
  } else if (warp == 0) {
    const uint32_t idesc = tc05::idesc_i8(128, 64, false);
    const uint32_t planes_s = tc05::smem_u32(smem);
    const long long t0 = clock64();
    int cls = 0;
    for (int seq = 0; seq < streams; ++seq, cls += 6) {
      const int slot = seq & 1;
      for (int p = 0; p < 5; ++p) {
        const uint32_t blo0 = tc05::desc_sw128_lo(planes_s + (uint32_t)((slot * 5 + p) * 9216));
        for (int j = 0; j < 2; ++j) {
          const int c = p + j, k = cls + c, rs = k % NSL, use = k / NSL;
          const bool first = p == (c - 1 > 0 ? c - 1 : 0);
          if ((VARIANT == 8 || VARIANT == 9) && first && use >= 1) {
            mbar_wait(tc05::smem_u32(&acce[rs]), (use - 1) & 1);
            tc05::fence_after();
          }
          const uint32_t d = (uint32_t)(512 - 64 * NSL) + 64u * rs, a = 96u * j;
          if (VARIANT == 6) {  // runtime step count in chunks of 4 (KT padded to 128)
            if (elect_one_probe()) {
              for (int k0 = 0; k0 < nsteps_rt; k0 += 4) {
#pragma unroll
                for (int i = 0; i < 4; ++i)
                  tc05::mma_i8_ts_lo(d, a + 8u * (k0 + i), blo0 + 2u * (k0 + i), idesc, (first && k0 + i == 0) ? 0u : 1u);
              }
            }
            __syncwarp();
          } else if (VARIANT == 5) {  // the conv kernel's form: runtime step count, 24-way guarded unroll
            if (elect_one_probe()) {
#pragma unroll
              for (int kc = 0; kc < 24; ++kc)
                if (kc < nsteps_rt)
                  tc05::mma_i8_ts_lo(d, a + 8u * kc, blo0 + 2u * kc, idesc, (first && kc == 0) ? 0u : 1u);
            }
            __syncwarp();
          } else if (VARIANT == 0 || VARIANT == 7 || VARIANT == 8 || VARIANT == 9 || VARIANT == 10) {
            if (elect_one_probe()) {
#pragma unroll
              for (int kc = 0; kc < 12; ++kc) tc05::mma_i8_ts_lo(d, a + 8u * kc, blo0 + 2u * kc, idesc, (first && kc == 0) ? 0u : 1u);
            }
            __syncwarp();
          } else {
            if (elect_one_probe()) {
#pragma unroll
              for (int kc = 0; kc < 12; ++kc) tc05::mma_i8_ts_lo(d, a + 8u * kc, blo0 + 2u * kc, idesc, 1u);
            }
            __syncwarp();
          }
          if (p == (c < 4 ? c : 4)) tc05::commit_elect(tc05::smem_u32((VARIANT == 8 || VARIANT == 9) ? &accf[rs] : &mbar2));
        }
      }
    }
    tc05::commit_elect(tc05::smem_u32(&mbar));
    mbar_wait(tc05::smem_u32(&mbar), 0);
    if (tid == 0) {
      *cycles = clock64() - t0;
      stop_flag = 1;
    }
  } else if ((VARIANT == 8 || VARIANT == 9) && warp >= 4) {
    unsigned long long acc = tid;
    const int half = (warp - 4) >> 2;
    for (int k = 0; k < streams * 6; ++k) {
      const int rs = k % NSL;
      if (!getenv_nowait || (tid & 31) == 0) mbar_wait(tc05::smem_u32(&accf[rs]), (k / NSL) & 1);
      __syncwarp();
      tc05::fence_after();
      uint32_t r[32];
      tc05::ld_x32(((uint32_t)(32 * (warp & 3)) << 16) + (NSL == 5 ? 192u : 320u) + 64u * rs + 32u * half, r);
      tc05::wait_ld();
      tc05::fence_before();
      __syncwarp();
      if ((tid & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc05::smem_u32(&acce[rs])) : "memory");
#pragma unroll
      for (int i = 0; i < 32; ++i) acc += r[i];
      if (VARIANT == 9) {  // epilogue-like work: 32 IMAD.WIDE and 32 coalesced 4-byte stores per class
        unsigned long long a2 = acc;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          long long d;
          asm volatile("mad.wide.s32 %0, %1, %2, %3;" : "=l"(d) : "r"(r[i]), "r"(i + 3), "l"((long long)a2));
          a2 = (unsigned long long)d;
        }
        unsigned* out = reinterpret_cast<unsigned*>(sink) + 4096 + (size_t)blockIdx.x * 65536;
#pragma unroll
        for (int i = 0; i < 32; ++i) out[(k & 7) * 8192 + 256 * i + (tid - 128)] = (unsigned)(a2 >> (i & 31));
        acc ^= a2;
      }
    }
    if (acc == 42) *sink = acc;
  } else if (warp >= 4) {
    unsigned long long acc = tid;
    uint32_t r[16];
    int it = 0;
    while (!*(volatile int*)&stop_flag) {
      if (VARIANT == 2) {
#pragma unroll
        for (int i = 0; i < 64; ++i) acc = acc * 0x9E3779B97F4A7C15ull + (unsigned)i;
      } else if (VARIANT == 3) {
        tc05::ld_x16(((uint32_t)(32 * (warp & 3)) << 16) + 320u + 16u * (it & 3), r);
        tc05::wait_ld();
        acc += r[0];
      } else if (VARIANT == 4) {
#pragma unroll
        for (int i = 0; i < 16; ++i)
          asm volatile("st.shared.b32 [%0], %1;" ::"r"(tc05::smem_u32(smem) + 2 * 5 * 9216 + 4u * ((tid + 32 * i) & 2047)), "r"((uint32_t)acc));
      } else {
        break;
      }
      ++it;
    }
    if (acc == 42) *sink = acc;
  }
  tc05::fence_before();
  __syncthreads();
  if (warp == 0) tc05::dealloc(tslot, 512);
}

template <int VARIANT, int NSL = 3>
void run_convlike() {
  long long* dc;
  cudaMalloc(&dc, 8);
  const int smem = getenv("BIGSMEM") ? 229376 : 2 * 5 * 9216 + 8192;
  cudaFuncSetAttribute(convlike<VARIANT, NSL>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int streams = 42;
  unsigned long long* sink;
  cudaMalloc(&sink, (size_t)8 * (512 + 148 * 32768));
  convlike<VARIANT, NSL><<<148, getenv("T512") ? 512 : 384, smem>>>(streams, dc, sink, 12, getenv("NOWAIT") ? 1 : 0);
  cudaDeviceSynchronize();
  long long cyc;
  cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  printf("slots %d ", NSL);
  printf("convlike variant %d: %.1f cyc/MMA over %d MMAs (%s)\n", VARIANT, (double)cyc / (streams * 120), streams * 120,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(dc);
}

int main() {
  if (getenv("SMR")) {
    run_convlike<0>();
    run_convlike<11, 5>();
    run_convlike<11, 3>();
    return 0;
  }
  if (getenv("TPUT_FIRST")) {
    run_tput<64, 0, 1, false>(148);
    run_tput<64, 0, 2, false>(148);
    run_tput<64, 0, 1, true>(148);
    run_tput<128, 0, 1, false>(148);
    return 0;
  }
  run_convlike<0>();
  run_convlike<8>();
  run_convlike<8, 5>();
  if (getenv("CONV_ONLY")) return 0;
  run_convlike<9>();
  run_convlike<7>();
  run_convlike<5>();
  run_convlike<6>();
  run_convlike<2>();
  run_convlike<3>();
  run_convlike<4>();
  run_tput<64, 0, 1, false>(148);
  run_tput<64, 0, 1, false, 12>(148);
  run_tput<64, 0, 1, false, 6>(148);
  run_tput<64, 0, 1, false, 1>(148);
  if (getenv("TPUT_ONLY")) return 0;
  run_tput<32, 0, 1, false>();
  run_tput<32, 0, 4, false>();
  run_tput<32, 0, 8, false>();
  run_tput<64, 0, 1, false>();
  run_tput<64, 0, 4, false>();
  run_tput<128, 0, 1, false>();
  run_tput<128, 0, 2, false>();
  run_tput<256, 0, 1, false>();
  run_tput<64, 0, 1, true>();
  run_tput<32, 1, 1, false>();
  run_tput<64, 1, 1, false>();
  run_tput<64, 1, 4, false>();
  run_tput<128, 1, 1, false>();
  run_tput<256, 1, 1, false>();
  srand(1234);
  int bad_total = 0;
  for (int mode = 0; mode < 2; ++mode)
    for (int N : {16, 32, 64, 128, 256})
      for (int row0 : {0, 1, 3}) {
        std::vector<int8_t> A(128 * KT), B(128 * (N + row0) + 256);
        for (auto& a : A) a = (int8_t)(rand() & 255);
        for (auto& b : B) b = (int8_t)(rand() & 255);
        int8_t *dA, *dB;
        int32_t* dD;
        long long* dc;
        cudaMalloc(&dA, A.size());
        cudaMalloc(&dB, B.size());
        cudaMalloc(&dD, 128 * N * 4);
        cudaMalloc(&dc, 8);
        cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
        cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
        const int smem = (128 * (N + row0) + 256 + 1024 + 1023) / 1024 * 1024 + 1024 + 3 * 16384;
        cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        probe<<<1, 128, smem>>>(dA, dB, N, row0, 1, mode, 1, dD, dc);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          printf("mode %d N %d row0 %d: CUDA error %s\n", mode, N, row0, cudaGetErrorString(e));
          return 1;
        }
        std::vector<int32_t> D(128 * N);
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int v = 0; v < 128; ++v)
          for (int u = 0; u < N; ++u) {
            long long s = 0;
            for (int k = 0; k < KT; ++k) s += (long long)A[v * KT + k] * B[128 * (u + row0) + k];
            if (s != D[v * N + u]) {
              if (bad < 3) printf("  mismatch v=%d u=%d got %d want %lld\n", v, u, D[v * N + u], s);
              ++bad;
            }
          }
        bad_total += bad;
        // throughput: 400 reps x 12 K steps x nacc accumulators
        const int reps = 400;
        for (int nacc = 1; nacc * N <= 256 && row0 == 0; nacc *= 2) {
          probe<<<1, 128, smem>>>(dA, dB, N, row0, reps, mode, nacc, dD, dc);
          cudaDeviceSynchronize();
          long long cyc;
          cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
          printf("mode %s N %3d nacc %d: %.1f cyc/MMA (floor %d)\n", mode ? "SS" : "TS", N, nacc,
                 (double)cyc / (reps * KC * nacc), 128 * N / 256);
        }
        printf("mode %s N %3d row0 %d: %s\n", mode ? "SS" : "TS", N, row0, bad ? "MISMATCH" : "exact");
        cudaFree(dA);
        cudaFree(dB);
        cudaFree(dD);
        cudaFree(dc);
      }
  printf("%s\n", bad_total ? "FAIL" : "ALL EXACT");
  return bad_total ? 1 : 0;
}
