// TMA ingest micro-benchmark (tools/tma_probe.cu): how fast one SM receives
// K-major fp16 operand tiles (SWIZZLE_128B, 64-column boxes, the GEMM's
// stage layout) from an L2-resident matrix, as a function of the box shape
// and of how many CTAs load at once. One thread per CTA keeps `inflight`
// boxes outstanding and records clock64 from the first issue to the last
// completion.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -Ipaper_2605_20977_b200/csrc/cuda tools/tma_probe.cu -o tools/tma_probe -lcuda
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "ptx.cuh"

using namespace pswa_dev;

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

constexpr int kSlots = 8;

// box b of CTA c reads rows [(c * 7 + b) % row_blocks] x k-block (b % kbs)
__global__ void probe_kernel(const __grid_constant__ CUtensorMap map, int dims, int box_rows, int kb_per_box,
                             int row_blocks, int kbs, int nbox, int inflight, uint32_t box_bytes,
                             unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bars[kSlots];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < kSlots; ++s) mbar_init(&bars[s], 1);
  fence_mbar_init();
  tma_prefetch(&map);
  auto issue = [&](int b) {
    const int s = b % inflight;
    mbar_expect_tx(&bars[s], box_bytes);
    const int rb = (blockIdx.x * 7 + b) % row_blocks, kb = (b * kb_per_box) % kbs;
    const uint32_t dst = smem_u32(smem + static_cast<size_t>(s) * box_bytes);
    if (dims == 2)
      tma_load_2d(smem + static_cast<size_t>(s) * box_bytes, &map, &bars[s], kb * 64, rb * box_rows);
    else
      tma_load_3d(dst, &map, &bars[s], 0, rb * box_rows, kb);
  };
  const unsigned long long t0 = clock64();
  int issued = 0;
  for (; issued < inflight && issued < nbox; ++issued) issue(issued);
  for (int b = 0; b < nbox; ++b) {
    const int s = b % inflight;
    mbar_wait(&bars[s], (b / inflight) & 1);
    if (issued < nbox) issue(issued++);
  }
  out[blockIdx.x] = clock64() - t0;
}


// Variant: boxes alternate between two tensor maps (map1 for odd boxes) and
// are issued by `issuers` warps (lane 0 each) over disjoint slot sets.
__global__ void probe2_kernel(const __grid_constant__ CUtensorMap map0, const __grid_constant__ CUtensorMap map1,
                              int box_rows, int row_blocks, int kbs, int nbox, int inflight, int issuers,
                              uint32_t box_bytes, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bars[kSlots];
  const int w = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSlots; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
    tma_prefetch(&map0);
    tma_prefetch(&map1);
  }
  __syncthreads();
  if ((threadIdx.x & 31) != 0 || w >= issuers) return;
  const int per = inflight / issuers, nb = nbox / issuers;
  auto issue = [&](int b) {
    const int s = w * per + b % per;
    mbar_expect_tx(&bars[s], box_bytes);
    const int g = b * issuers + w;
    const int rb = (blockIdx.x * 7 + g) % row_blocks, kb = g % kbs;
    tma_load_2d(smem + static_cast<size_t>(s) * box_bytes, (g & 1) ? &map1 : &map0, &bars[s], kb * 64,
                rb * box_rows);
  };
  const unsigned long long t0 = clock64();
  int issued = 0;
  for (; issued < per && issued < nb; ++issued) issue(issued);
  for (int b = 0; b < nb; ++b) {
    const int s = w * per + b % per;
    mbar_wait(&bars[s], (b / per) & 1);
    if (issued < nb) issue(issued++);
  }
  if (w == 0) out[blockIdx.x] = clock64() - t0;
}


// Variant 3: issuers = (warps x lanes-per-warp); lane stride 16 inside a warp.
// Records the cycles the issuing thread spends inside the TMA issue and
// inside the waits.
__global__ void probe3_kernel(const __grid_constant__ CUtensorMap map0, int box_rows, int row_blocks, int kbs,
                              int nbox, int inflight, int warps, int lanes, uint32_t box_bytes,
                              unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bars[kSlots];
  const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSlots; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
    tma_prefetch(&map0);
  }
  __syncthreads();
  if (w >= warps || (ln % 16) != 0 || ln / 16 >= lanes) return;
  const int id = w * lanes + ln / 16, nis = warps * lanes;
  const int per = inflight / nis, nb = nbox / nis;
  unsigned long long t_issue = 0, t_wait = 0, t_exp = 0;
  auto issue = [&](int b) {
    const int s = id * per + b % per;
    const int g = b * nis + id;
    const int rb = (blockIdx.x * 7 + g) % row_blocks, kb = g % kbs;
    const unsigned long long a = clock64();
    mbar_expect_tx(&bars[s], box_bytes);
    const unsigned long long a2 = clock64();
    tma_load_2d(smem + static_cast<size_t>(s) * box_bytes, &map0, &bars[s], kb * 64, rb * box_rows);
    const unsigned long long a3 = clock64();
    t_issue += a3 - a2;
    t_exp += a2 - a;
  };
  const unsigned long long t0 = clock64();
  int issued = 0;
  for (; issued < per && issued < nb; ++issued) issue(issued);
  for (int b = 0; b < nb; ++b) {
    const int s = id * per + b % per;
    const unsigned long long a = clock64();
    mbar_wait(&bars[s], (b / per) & 1);
    t_wait += clock64() - a;
    if (issued < nb) issue(issued++);
  }
  if (id == 0) {
    out[3 * blockIdx.x] = clock64() - t0;
    out[3 * blockIdx.x + 1] = t_issue;
    out[3 * blockIdx.x + 2] = t_wait;
    if (blockIdx.x == 0) out[1000] = t_exp;
  }
}


// Variant 4: burst of nb boxes (16 KB, precomputed coordinates) issued back
// to back by `issuers` warps, then all waited for: the TMA unit's own
// throughput without issue-loop latency. Repeated `reps` times.
__global__ void probe4_kernel(const __grid_constant__ CUtensorMap map0, const __grid_constant__ CUtensorMap map1,
                              int nb, int issuers, int reps, int mixed, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bars[kSlots];
  const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSlots; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
    tma_prefetch(&map0);
    tma_prefetch(&map1);
  }
  __syncthreads();
  const int rb = blockIdx.x % 16;
  unsigned long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (ln == 0 && w < issuers) {
      for (int b = w; b < nb; b += issuers) {
        // mixed: even boxes 16 KB (A-like, map0), odd boxes 8 KB (B-like, map1)
        const bool small = mixed && (b & 1);
        const uint32_t bytes = small ? 8192u : 16384u;
        mbar_expect_tx(&bars[b], bytes);
        tma_load_2d(smem + b * 16384, small ? &map1 : &map0, &bars[b], (r * nb + b) % 24 * 64, rb * 128);
      }
    }
    if (threadIdx.x == 0)
      for (int b = 0; b < nb; ++b) mbar_wait(&bars[b], r & 1);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeFn enc = reinterpret_cast<EncodeFn>(p);
  const int R = 2048, K = 1536;  // 6 MB fp16: L2-resident after the first pass
  __half* A;
  cudaMalloc(&A, static_cast<size_t>(R) * K * 2);
  cudaMemset(A, 0, static_cast<size_t>(R) * K * 2);
  unsigned long long* out;
  cudaMalloc(&out, 2048 * 8);
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  struct Cfg { int dims, rows, kbpb; };
  const Cfg cfgs[] = {{2, 64, 1}, {2, 128, 1}, {2, 256, 1}, {3, 64, 2}, {3, 128, 2}, {3, 128, 4}, {3, 64, 4}};
  std::printf("box, CTAs, inflight, bytes/box, cycles/box (median CTA), B/clk per SM\n");
  for (const Cfg& c : cfgs) {
    CUtensorMap m;
    CUresult r;
    uint32_t box_bytes = c.rows * 128 * c.kbpb;
    if (c.dims == 2) {
      cuuint64_t d[2] = {(cuuint64_t)K, (cuuint64_t)R};
      cuuint64_t st[1] = {(cuuint64_t)K * 2};
      cuuint32_t box[2] = {64, (cuuint32_t)c.rows}, es[2] = {1, 1};
      r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, A, d, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
      // (64 columns of a k-block, rows, k-blocks): [kb][row][64] in smem,
      // i.e. kbpb consecutive GEMM stage tiles
      cuuint64_t d[3] = {64, (cuuint64_t)R, (cuuint64_t)(K / 64)};
      cuuint64_t st[2] = {(cuuint64_t)K * 2, 128};
      cuuint32_t box[3] = {64, (cuuint32_t)c.rows, (cuuint32_t)c.kbpb}, es[3] = {1, 1, 1};
      r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, A, d, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (r != CUDA_SUCCESS) {
      std::printf("%dd %dx%d: encode failed (%d)\n", c.dims, c.rows, c.kbpb, int(r));
      continue;
    }
    const int kbs = K / 64 - (c.kbpb - 1);
    for (int ctas : {1, 64, 128, 148}) {
      for (int inflight : {2, 4, 8}) {
        if (inflight * box_bytes > 190 * 1024) continue;
        const int nbox = 64;
        for (int rep = 0; rep < 2; ++rep)
          probe_kernel<<<ctas, 32, inflight * box_bytes + 1024>>>(m, c.dims, c.rows, c.kbpb, R / c.rows, kbs,
                                                                   nbox, inflight, box_bytes, out);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          std::printf("error %s\n", cudaGetErrorString(e));
          return 1;
        }
        std::vector<unsigned long long> h(ctas);
        cudaMemcpy(h.data(), out, ctas * 8, cudaMemcpyDeviceToHost);
        std::vector<unsigned long long> s = h;
        std::sort(s.begin(), s.end());
        const double cyc = double(s[ctas / 2]) / nbox;
        std::printf("%dd %3dx64x%d, %3d, %d, %6u, %7.1f, %6.1f\n", c.dims, c.rows, c.kbpb, ctas, inflight,
                    box_bytes, cyc, box_bytes / cyc);
      }
    }
  }

  {  // two maps / two issuers, 2D 128 x 64 boxes
    __half* B;
    cudaMalloc(&B, static_cast<size_t>(R) * K * 2);
    cudaMemset(B, 0, static_cast<size_t>(R) * K * 2);
    auto mk = [&](CUtensorMap* m, __half* base, int rows) {
      cuuint64_t d[2] = {(cuuint64_t)K, (cuuint64_t)R};
      cuuint64_t st[1] = {(cuuint64_t)K * 2};
      cuuint32_t box[2] = {64, (cuuint32_t)rows}, es[2] = {1, 1};
      enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, base, d, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    };
    CUtensorMap mA, mA2, mB;
    mk(&mA, A, 128);
    mk(&mA2, A, 128);
    mk(&mB, B, 128);
    cudaFuncSetAttribute(probe2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    struct V { const char* name; const CUtensorMap* m1; int issuers; };
    const V vs[] = {{"same map, 1 issuer", &mA, 1}, {"2 maps same tensor", &mA2, 1}, {"2 tensors", &mB, 1},
                    {"same map, 2 issuers", &mA, 2}, {"2 tensors, 2 issuers", &mB, 2}};
    for (const V& v : vs)
      for (int ctas : {1, 128}) {
        const int inflight = 8, nbox = 64;
        for (int rep = 0; rep < 2; ++rep)
          probe2_kernel<<<ctas, 64, inflight * 16384 + 1024>>>(mA, *v.m1, 128, R / 128, K / 64, nbox, inflight,
                                                               v.issuers, 16384, out);
        cudaDeviceSynchronize();
        std::vector<unsigned long long> h(ctas);
        cudaMemcpy(h.data(), out, ctas * 8, cudaMemcpyDeviceToHost);
        std::sort(h.begin(), h.end());
        const double cyc = double(h[ctas / 2]) / nbox;
        std::printf("%s, %d CTAs: %.1f cycles per 16 KB box, %.1f B/clk\n", v.name, ctas, cyc, 16384 / cyc);
      }
  }

  {
    auto mk = [&](CUtensorMap* m, __half* base, int rows) {
      cuuint64_t d[2] = {(cuuint64_t)K, (cuuint64_t)R};
      cuuint64_t st[1] = {(cuuint64_t)K * 2};
      cuuint32_t box[2] = {64, (cuuint32_t)rows}, es[2] = {1, 1};
      enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, base, d, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    };
    CUtensorMap mA;
    mk(&mA, A, 128);
    cudaFuncSetAttribute(probe3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    struct V { int warps, lanes, inflight; };
    const V vs[] = {{1, 1, 8}, {1, 1, 1}, {1, 1, 2}, {1, 2, 8}, {2, 1, 8}, {4, 1, 8}, {8, 1, 8}};
    for (const V& v : vs)
      for (int ctas : {1, 128}) {
        const int nbox = 64;
        for (int rep = 0; rep < 2; ++rep)
          probe3_kernel<<<ctas, 256, v.inflight * 16384 + 1024>>>(mA, 128, R / 128, K / 64, nbox, v.inflight,
                                                                  v.warps, v.lanes, 16384, out);
        cudaDeviceSynchronize();
        std::vector<unsigned long long> h(3 * ctas);
        cudaMemcpy(h.data(), out, 3 * ctas * 8, cudaMemcpyDeviceToHost);
        unsigned long long te = 0;
        cudaMemcpy(&te, out + 1000, 8, cudaMemcpyDeviceToHost);
        std::printf("warps %d x lanes %d, inflight %d, %3d CTAs: %.1f cycles per box (CTA 0 issuer 0 per box: expect_tx %.1f, tma %.1f, wait %.1f)\n",
                    v.warps, v.lanes, v.inflight, ctas, double(h[0]) / nbox, double(te) * v.warps * v.lanes / nbox,
                    double(h[1]) * v.warps * v.lanes / nbox, double(h[2]) * v.warps * v.lanes / nbox);
      }
  }

  {
    auto mk = [&](CUtensorMap* m, __half* base, int rows) {
      cuuint64_t d[2] = {(cuuint64_t)K, (cuuint64_t)R};
      cuuint64_t st[1] = {(cuuint64_t)K * 2};
      cuuint32_t box[2] = {64, (cuuint32_t)rows}, es[2] = {1, 1};
      enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, base, d, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    };
    CUtensorMap m128, m64;
    mk(&m128, A, 128);
    mk(&m64, A, 64);
    cudaFuncSetAttribute(probe4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int mixed : {0, 1})
      for (int issuers : {1, 2, 4})
        for (int ctas : {1, 128}) {
          const int nb = 8, reps = 32;
          for (int rep = 0; rep < 2; ++rep)
            probe4_kernel<<<ctas, 128, 8 * 16384 + 1024>>>(m128, m64, nb, issuers, reps, mixed, out);
          cudaDeviceSynchronize();
          std::vector<unsigned long long> h(ctas);
          cudaMemcpy(h.data(), out, ctas * 8, cudaMemcpyDeviceToHost);
          std::sort(h.begin(), h.end());
          const double per_burst = double(h[ctas / 2]) / reps;
          const double bytes = mixed ? 4 * 16384.0 + 4 * 8192.0 : 8 * 16384.0;
          std::printf("burst of 8 boxes (%s), %d issuers, %3d CTAs: %.0f cycles per burst, %.1f B/clk per SM\n",
                      mixed ? "16K/8K alternating" : "16K", issuers, ctas, per_burst, bytes / per_burst);
        }
  }
  return 0;
}
