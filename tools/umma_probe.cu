// tcgen05.mma throughput micro-benchmark (tools/umma_probe.cu): cycles per
// kind::f16 MMA (K = 16, operands in shared memory, SWIZZLE_128B K-major,
// fp32 accumulator in TMEM) as a function of M and N, one CTA per SM,
// issued back to back by one thread; optionally with a TMA-free smem write
// stream from the other warps (contention for the smem read port).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -Ipaper_2605_20977_b200/csrc/cuda tools/umma_probe.cu -o tools/umma_probe
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

#include "ptx.cuh"

using namespace pswa_dev;

__global__ void umma_kernel(int m, int n, int iters, int kblk, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  // A: kblk k-blocks of 128 x 64 (16 KB each); B: kblk k-blocks of 256 x 64 (32 KB each)
  uint8_t* sa = smem;
  uint8_t* sb = smem + kblk * 16384;
  for (int i = threadIdx.x; i < kblk * (16384 + 32768) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3c003c00u, 0, 0x3c00u, 0);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(&tslot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = umma_idesc_f16_f32(m, n);
    fence_proxy_async_smem();
    // warm-up
    for (int kk = 0; kk < 4; ++kk)
      tc_mma_f16(tmem, umma_desc_k_sw128(smem_u32(sa) + kk * 32), umma_desc_k_sw128(smem_u32(sb) + kk * 32), idesc,
                 kk);
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int kb = it % kblk;
      const uint32_t a = smem_u32(sa + kb * 16384), b = smem_u32(sb + kb * 32768);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        tc_mma_f16(tmem, umma_desc_k_sw128(a + kk * 32), umma_desc_k_sw128(b + kk * 32), idesc, 1u);
    }
    tc_commit(&bar);
    mbar_wait(&bar, 1);
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_free(tmem, 256);
  }
}

int main() {
  unsigned long long* out;
  cudaMalloc(&out, 1024 * 8);
  const int kblk = 4;
  const int smem = kblk * (16384 + 32768) + 1024;
  cudaFuncSetAttribute(umma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  std::printf("M, N, CTAs, cycles per MMA (K=16), MAC/clk per SM, frac of 4096 MAC/clk\n");
  for (int m : {64, 128})
    for (int n : {32, 64, 128, 192, 256})
      for (int ctas : {1, 148}) {
        const int iters = 256;
        for (int rep = 0; rep < 2; ++rep) umma_kernel<<<ctas, 128, smem>>>(m, n, iters, kblk, out);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          std::printf("M %d N %d: %s\n", m, n, cudaGetErrorString(e));
          return 1;
        }
        std::vector<unsigned long long> h(ctas);
        cudaMemcpy(h.data(), out, ctas * 8, cudaMemcpyDeviceToHost);
        std::sort(h.begin(), h.end());
        const double cyc = double(h[ctas / 2]) / (iters * 4);
        const double mac = double(m) * n * 16 / cyc;
        std::printf("%d, %d, %d, %.1f, %.0f, %.3f\n", m, n, ctas, cyc, mac, mac / 4096.0);
      }
  return 0;
}
