// tcgen05.mma issue-rate microbenchmark on B200 for the operand shapes of the
// FSA kernels (K8 S/dP, dV^T/dK^T, dQ; K5 P.V).  One CTA per SM, one elected
// thread issues G groups of K-step MMAs (commit + wait per group), smem holds
// arbitrary data (rates do not depend on values).  Reported: cycles per MMA
// instruction and achieved FLOP/cycle/SM (peak dense fp16 ~8192).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2508_18224_b200/csrc \
//        tools/mma_probe.cu -o /tmp/mma_probe && /tmp/mma_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "tc_common.cuh"
using namespace fsa::tc;

struct Case {
  const char* name;
  int M, N, ksteps;   // MMA shape (K = 16 per instruction), K-steps per operand tile
  int a_tmem;         // A operand from TMEM (ts)
  int a_mn, b_mn;     // operand majorness
  int chains;         // independent accumulators, MMAs round-robin over them
};

// rep: instructions per commit = rep * ksteps (the operand tile's K-steps, cycled)
__global__ void probe(Case c, int groups, int rep, unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tmem_s;
  __shared__ __align__(8) uint64_t bar_s;
  const uint32_t sb = smem_u32(smem), bar = smem_u32(&bar_s);
  const int warp = threadIdx.x >> 5;
  // fill smem with small finite fp16 values
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(smem_u32(&tmem_s));
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_s;
  const uint32_t idesc = idesc_f16(c.M, c.N, c.a_mn != 0, c.b_mn != 0);
  const uint32_t A = sb, B = sb + 65536;
  unsigned long long t0 = 0, t1 = 0;
  if (warp == 0) {
    // descriptors of the tile's K-steps computed once (the issue loop below is
    // then just back-to-back tcgen05.mma from one thread)
    uint64_t ad[8], bd[8];
    uint32_t dcol[8], at[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      ad[k] = c.a_mn ? desc_mnmajor(A + k * 2048u, 16384u)
                     : desc_kmajor(A + (k >> 2) * 16384u + (k & 3) * 32u);
      bd[k] = c.b_mn ? desc_mnmajor(B + k * 2048u, 8192u)
                     : desc_kmajor(B + (k >> 2) * 8192u + (k & 3) * 32u);
      dcol[k] = tmem + (uint32_t)((k % c.chains) * c.N) % 256u;
      at[k] = tmem + 256 + k * 8;
    }
    const uint32_t idesc2 = idesc;
    t0 = clock64();
    for (int g = 0; g < groups; ++g) {
      if (elect_one()) {
        for (int r = 0; r < rep; ++r) {
          if (c.a_tmem) {
#pragma unroll
            for (int k = 0; k < 8; ++k) mma_bf16_ts(dcol[k], at[k], bd[k], idesc2, 1u);
          } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) mma_bf16(dcol[k], ad[k], bd[k], idesc2, 1u);
          }
        }
        mma_commit(bar);
      }
      __syncwarp();
      mbar_wait_warp(bar, (uint32_t)(g & 1));
    }
    t1 = clock64();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

int main() {
  static char names[128][64];
  Case cases[128];
  int nc = 0;
  const char* an[3] = {"Kmaj", "MN", "tmem"};
  for (int N : {64, 128, 256})
    for (int ch : {1, 2, 4})
      for (int a = 0; a < 3; ++a)
        for (int bm = 0; bm < 2; ++bm) {
          if (N * ch > 256 && ch > 1) continue;
          snprintf(names[nc], 64, "M128 N%-3d A %-4s B %-4s chains %d", N, an[a], bm ? "MN" : "Kmaj", ch);
          cases[nc] = Case{names[nc], 128, N, 8, a == 2, a == 1, bm, ch};
          ++nc;
        }

  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d;
  cudaMalloc(&d, nsm * sizeof(unsigned long long));
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int rep : {16}) {
  const int groups = rep == 1 ? 2000 : 200;
  printf("-- %d MMA K-step tiles per commit + wait\n", rep);
  for (int ci = 0; ci < nc; ++ci) {
    const Case& c = cases[ci];
    for (int it = 0; it < 2; ++it) {
      probe<<<nsm, 128, 200 * 1024>>>(c, groups, rep, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("%s: %s\n", c.name, cudaGetErrorString(e));
        return 1;
      }
    }
    unsigned long long h[256];
    cudaMemcpy(h, d, nsm * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < nsm; ++i) avg += h[i];
    avg /= nsm;
    const double n_mma = (double)groups * c.ksteps * rep;
    const double flop = 2.0 * c.M * c.N * 16 * n_mma;
    printf("%-52s %7.1f cycles/MMA  %7.0f FLOP/cycle/SM  (%d MMAs per commit)\n", c.name,
           avg / n_mma, flop / avg, c.ksteps * rep);
  }
  }
  return 0;
}
