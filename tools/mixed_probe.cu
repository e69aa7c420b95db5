// Does tcgen05.mma kind::f16 accept A and B in different formats (A bf16,
// B fp16, or the reverse)?  One CTA: D[128 x 64] = A[128 x 64] . B[64 x 64]^T
// with K-major SW128 tiles, against a host fp64 reference of the same values.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2508_18224_b200/csrc \
//        tools/mixed_probe.cu -o /tmp/mixed_probe && /tmp/mixed_probe
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include "tc_common.cuh"
using namespace fsa::tc;

// A rows as raw 16-bit patterns, [128][64]; B [64][64]
__global__ void probe(const uint16_t* A, const uint16_t* B, uint32_t idesc, float* D) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tmem_s;
  __shared__ __align__(8) uint64_t bar_s;
  const uint32_t sb = smem_u32(smem), bar = smem_u32(&bar_s);
  const int warp = threadIdx.x >> 5;
  // SW128 K-major tiles: row r, 16-byte chunk c at sw128_off(r, c)
  for (int e = threadIdx.x; e < 128 * 8; e += blockDim.x) {
    const int r = e >> 3, c = e & 7;
    *reinterpret_cast<uint4*>(smem + sw128_off(r, c)) = reinterpret_cast<const uint4*>(A + r * 64)[c];
  }
  for (int e = threadIdx.x; e < 64 * 8; e += blockDim.x) {
    const int r = e >> 3, c = e & 7;
    *reinterpret_cast<uint4*>(smem + 16384 + sw128_off(r, c)) =
        reinterpret_cast<const uint4*>(B + r * 64)[c];
  }
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<64>(smem_u32(&tmem_s));
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_s;
  if (warp == 0) {
    if (elect_one()) {
      for (int k = 0; k < 4; ++k)
        mma_bf16(tmem, desc_kmajor(sb + k * 32u), desc_kmajor(sb + 16384 + k * 32u), idesc, k > 0);
      mma_commit(bar);
    }
    __syncwarp();
  }
  mbar_wait(bar, 0);
  tc_fence_after();
  float v[32];
  const uint32_t lb = (uint32_t)(warp * 32) << 16;
  for (int h = 0; h < 2; ++h) {
    tmem_ld32(tmem + lb + h * 32, v);
    tmem_wait_ld();
    for (int c = 0; c < 32; ++c) D[(warp * 32 + (threadIdx.x & 31)) * 64 + h * 32 + c] = v[c];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<64>(tmem);
}

static double val(uint16_t x, bool bf) {
  if (bf) {
    uint32_t u = (uint32_t)x << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
  }
  __half_raw r;
  r.x = x;
  return (double)__half2float(__half(r));
}

int main() {
  const int combos[4][2] = {{1, 1}, {0, 0}, {1, 0}, {0, 1}};  // (A bf16?, B bf16?)
  uint16_t hA[128 * 64], hB[64 * 64];
  uint16_t *dA, *dB;
  float* dD;
  cudaMalloc(&dA, sizeof hA);
  cudaMalloc(&dB, sizeof hB);
  cudaMalloc(&dD, 128 * 64 * 4);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (auto& cb : combos) {
    const bool abf = cb[0], bbf = cb[1];
    uint32_t seed = 12345;
    auto rnd = [&]() {
      seed = seed * 1664525u + 1013904223u;
      return ((seed >> 8) & 0xffff) / 65536.0f * 2.f - 1.f;
    };
    for (int i = 0; i < 128 * 64; ++i) {
      const float f = rnd() * 3.f;
      hA[i] = abf ? __bfloat16_as_ushort(__float2bfloat16(f)) : __half_as_ushort(__float2half(f));
    }
    for (int i = 0; i < 64 * 64; ++i) {
      const float f = rnd() * 3.f;
      hB[i] = bbf ? __bfloat16_as_ushort(__float2bfloat16(f)) : __half_as_ushort(__float2half(f));
    }
    cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
    const uint32_t idesc = (1u << 4) | ((abf ? 1u : 0u) << 7) | ((bbf ? 1u : 0u) << 10) |
                           ((64u >> 3) << 17) | ((128u >> 4) << 24);
    probe<<<1, 128, 64 * 1024>>>(dA, dB, idesc, dD);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("A %s B %s: %s\n", abf ? "bf16" : "fp16", bbf ? "bf16" : "fp16", cudaGetErrorString(e));
      return 1;
    }
    static float hD[128 * 64];
    cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
    double worst = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 64; ++n) {
        double ref = 0;
        for (int k = 0; k < 64; ++k) ref += val(hA[m * 64 + k], abf) * val(hB[n * 64 + k], bbf);
        worst = fmax(worst, fabs(ref - hD[m * 64 + n]));
      }
    printf("A %s x B %s: max |D - ref| = %.3g\n", abf ? "bf16" : "fp16", bbf ? "bf16" : "fp16", worst);
  }
  return 0;
}
