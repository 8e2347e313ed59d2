// tcgen05 / TMA GEMM for sm_100a. See gemm.h for the contract.
//
// Persistent kernel, one CTA per SM, 128 x BN output tiles (cta_group::1,
// UMMA M=128, N=BN, K=16 per instruction), tiles walked M-fastest so the CTAs
// in flight share their B (weight) panel in L2. Warp roles:
//   warp 0    : TMA producer (one elected lane), STAGES-deep smem ring
//   warp 1    : TMEM allocator + MMA issuer (one elected lane)
//   warps 2-9 : epilogue. Two TMEM accumulators (2 x BN columns) let the
//               epilogue of tile i overlap the MMAs of tile i+1. Each warp
//               drains one 32-lane quarter x one column half, transposes its
//               32 x 32 chunk through shared memory and writes whole row
//               segments (coalesced 64/128 B per row).
// The epilogue kind is a template parameter (no per-element mode branches).
// K is walked in ascending 64-wide blocks and never split: every output
// element has one fixed reduction order, so results are bitwise identical run
// to run and independent of M and of the tile schedule (the encoder/decoder
// symmetry contract).
#include <cuda.h>

#include <mutex>

#include "check.h"
#include "gemm.h"
#include "launch.cuh"
#include "ptx.cuh"

namespace pswa_dev {

namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;  // 64 fp16 = 128 B = one SWIZZLE_128B row
constexpr int kEpiWarps = 8;
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr int kStageBytesOut = 32 * 33 * 4;  // per-warp 32x32 fp32 transpose buffer (+pad)

enum EpiKind : int { kEpiF16 = 0, kEpiF32 = 1, kEpiSwiGLU = 2, kEpiHead = 3 };

template <int BN>
struct GemmCfg {
  // as deep as shared memory allows (<= 227 KB with the epilogue staging):
  // the small-M step GEMMs are latency bound, so all K blocks in flight helps
  static constexpr int kStages = BN == 256 ? 4 : (BN == 128 ? 6 : 8);
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kSmem = kStages * kStageBytes + kEpiWarps * kStageBytesOut + 1024 + 256;
};

__device__ __forceinline__ float silu_f(float v) { return v / (1.0f + __expf(-v)); }
__device__ __forceinline__ float softplus_f(float v) {
  if (v > 30.0f) return v;
  if (v < -30.0f) return __expf(v);
  return log1pf(__expf(v));
}

// Elementwise part of the epilogue for 32 accumulator columns [n0, n0+32).
template <int EPI>
__device__ __forceinline__ void epi_values(const GemmEpi& ep, int n0, float (&v)[32]) {
  if (EPI == kEpiHead) {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int n = n0 + j;
      const float b = ep.bias ? ep.bias[n] : 0.0f;
      v[j] = n < ep.split ? (v[j] + b) * (ep.scale ? ep.scale[n] : 1.0f) : 0.11f + softplus_f(v[j] + b);
    }
    return;
  }
  if (EPI == kEpiSwiGLU) {
    if (ep.bias) {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] += ep.bias[n0 + j];
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = silu_f(v[2 * j]) * v[2 * j + 1];
    return;
  }
  const float* sc = ep.scale ? ep.scale + n0 : nullptr;
  const float* bi = ep.bias ? ep.bias + n0 : nullptr;
  if (ep.bias_first) {
    if (bi) {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] += bi[j];
    }
    if (sc) {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] *= sc[j];
    }
  } else {
    if (sc) {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] *= sc[j];
    }
    if (bi) {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] += bi[j];
    }
  }
  if (ep.act == kActSilu) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = silu_f(v[j]);
  }
}

// Residual rows of one 32x32 fp32 chunk in the coalesced store mapping,
// loaded ahead of time (independent of the accumulator) so their latency
// overlaps the MMA / TMEM wait instead of serialising the epilogue.
__device__ __forceinline__ void prefetch_residual(const GemmEpi& ep, int M, int m0w, int oc0,
                                                  int lane, float4 (&res)[8]) {
#pragma unroll
  for (int pass = 0; pass < 8; ++pass) {
    const int r = pass * 4 + (lane >> 3), c = (lane & 7) * 4;
    const int m = m0w + r;
    res[pass] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (m >= M || oc0 + c + 4 > ep.n_store) continue;
    const int orow = ep.row_map ? ep.row_map[m] : m;
    if (orow < 0) continue;
    res[pass] = *reinterpret_cast<const float4*>(static_cast<const float*>(ep.out) +
                                                 static_cast<size_t>(orow) * ep.ld_out + oc0 + c);
  }
}

// Drain one 32 x 32 accumulator chunk (rows m0w..m0w+31 of this warp,
// accumulator columns n0..n0+31): values -> smem transpose -> coalesced rows.
template <int EPI>
__device__ __forceinline__ void epi_chunk(const GemmEpi& ep, int M, int m0w, int n0, int lane,
                                          float* stage, const uint32_t (&raw)[32],
                                          const float4 (&res)[8]) {
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(raw[j]);
  epi_values<EPI>(ep, n0, v);
  // columns produced by this chunk and where they start in the output row
  const int ncols = EPI == kEpiSwiGLU ? 16 : 32;
  const int oc0 = EPI == kEpiSwiGLU ? (n0 >> 1) : n0;
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 32; ++j) stage[lane * 33 + j] = v[j];  // row = lane
  __syncwarp();
  if (oc0 >= ep.n_store) return;
  const int nvalid = min(ncols, ep.n_store - oc0);
  if (EPI == kEpiF32) {
    // 8 lanes per row (4 floats each), 4 rows per pass; the residual (when
    // accumulating) was prefetched into `res` before the accumulator wait
#pragma unroll
    for (int pass = 0; pass < 8; ++pass) {
      const int r = pass * 4 + (lane >> 3), c = (lane & 7) * 4;
      const int m = m0w + r;
      if (m >= M) continue;
      const int orow = ep.row_map ? ep.row_map[m] : m;
      if (orow < 0) continue;
      float* dst = static_cast<float*>(ep.out) + static_cast<size_t>(orow) * ep.ld_out + oc0 + c;
      const float* s = stage + r * 33 + c;
      if (c + 4 <= nvalid) {
        float4 o = make_float4(s[0], s[1], s[2], s[3]);
        if (ep.accumulate) {
          o.x += res[pass].x;
          o.y += res[pass].y;
          o.z += res[pass].z;
          o.w += res[pass].w;
        }
        *reinterpret_cast<float4*>(dst) = o;
      } else {
        for (int k = 0; k < 4 && c + k < nvalid; ++k) dst[k] = ep.accumulate ? dst[k] + s[k] : s[k];
      }
    }
  } else if (EPI == kEpiHead) {
    for (int idx = lane; idx < 32 * nvalid; idx += 32) {
      const int r = idx / nvalid, c = idx % nvalid;
      const int m = m0w + r;
      if (m >= M) continue;
      const int orow = ep.row_map ? ep.row_map[m] : m;
      if (orow < 0) continue;
      static_cast<float*>(ep.out)[static_cast<size_t>(orow) * ep.ld_out + oc0 + c] = stage[r * 33 + c];
    }
  } else {
    // fp16 rows: 32 cols = 64 B -> 4 lanes x 16 B per row, 8 rows per pass;
    // SwiGLU rows: 16 cols = 32 B -> 2 lanes per row, 16 rows per pass
    constexpr int kLanesPerRow = EPI == kEpiSwiGLU ? 2 : 4;
    constexpr int kRowsPerPass = 32 / kLanesPerRow;
#pragma unroll
    for (int pass = 0; pass < 32 / kRowsPerPass; ++pass) {
      const int r = pass * kRowsPerPass + lane / kLanesPerRow, c = (lane % kLanesPerRow) * 8;
      const int m = m0w + r;
      if (m >= M) continue;
      const int orow = ep.row_map ? ep.row_map[m] : m;
      if (orow < 0) continue;
      __half* dst = static_cast<__half*>(ep.out) + static_cast<size_t>(orow) * ep.ld_out + oc0 + c;
      const float* s = stage + r * 33 + c;
      if (c + 8 <= nvalid) {
        __half2 h[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) h[k] = __floats2half2_rn(s[2 * k], s[2 * k + 1]);
        *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<uint4*>(h);
      } else {
        for (int k = 0; k < 8 && c + k < nvalid; ++k) dst[k] = __float2half_rn(s[k]);
      }
    }
  }
}

template <int BN, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tma, const __grid_constant__ CUtensorMap tmb,
                   int M, int K, int tiles_m, int num_tiles, const __grid_constant__ GemmEpi ep) {
  using Cfg = GemmCfg<BN>;
  constexpr int S = Cfg::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sa = smem;
  uint8_t* sb = smem + S * Cfg::kABytes;
  float* sout = reinterpret_cast<float*>(smem + S * Cfg::kStageBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(sout + kEpiWarps * kStageBytesOut / 4);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int kblocks = K / kBK;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tma);
    tma_prefetch(&tmb);
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], kEpiWarps);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 2 * BN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // everything above overlaps the previous kernel (PDL); inputs are read below
  pdl_wait();
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      int g = 0;  // global k-block counter across tiles
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const int m0 = (t % tiles_m) * kBM, n0 = (t / tiles_m) * BN;
        for (int kb = 0; kb < kblocks; ++kb, ++g) {
          const int s = g % S, round = g / S;
          if (round > 0) mbar_wait(&empty[s], (round - 1) & 1);
          mbar_expect_tx(&full[s], Cfg::kStageBytes);
          tma_load_2d(sa + s * Cfg::kABytes, &tma, &full[s], kb * kBK, m0);
          tma_load_2d(sb + s * Cfg::kBBytes, &tmb, &full[s], kb * kBK, n0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_f16_f32(kBM, BN);
      int g = 0, it = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
        const int buf = it & 1, use = it >> 1;
        if (use > 0) mbar_wait(&tempty[buf], (use - 1) & 1);  // epilogue drained it
        tc_fence_after();
        const uint32_t acc = tmem + buf * BN;
        for (int kb = 0; kb < kblocks; ++kb, ++g) {
          const int s = g % S;
          mbar_wait(&full[s], (g / S) & 1);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sa + s * Cfg::kABytes);
          const uint32_t b_base = smem_u32(sb + s * Cfg::kBBytes);
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk)
            tc_mma_f16(acc, umma_desc_k_sw128(a_base + kk * 32), umma_desc_k_sw128(b_base + kk * 32),
                       idesc, (kb | kk) != 0 ? 1u : 0u);
          tc_commit(&empty[s]);
        }
        tc_commit(&tfull[buf]);
      }
    }
  } else {
    const int ew = warp - 2;
    const int q = warp & 3;                // TMEM lane quarter this warp may access
    const int half = ew >> 2;              // column half of the tile
    float* stage = sout + ew * (kStageBytesOut / 4);
    int it = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
      const int buf = it & 1, use = it >> 1;
      const int m0 = (t % tiles_m) * kBM, n0 = (t / tiles_m) * BN;
      const int c0 = half * (BN / 64), c1 = (half + 1) * (BN / 64);
      float4 res[8];
      const bool acc_res = EPI == kEpiF32 && ep.accumulate;
      if (acc_res) prefetch_residual(ep, M, m0 + q * 32, n0 + c0 * 32, lane, res);
      mbar_wait(&tfull[buf], use & 1);
      tc_fence_after();
      const uint32_t acc = tmem + buf * BN + (static_cast<uint32_t>(q * 32) << 16);
#pragma unroll 1
      for (int c = c0; c < c1; ++c) {
        uint32_t raw[32];
        tmem_ld_32x32(acc + c * 32, raw);
        tc_wait_ld();
        epi_chunk<EPI>(ep, M, m0 + q * 32, n0 + c * 32, lane, stage, raw, res);
        if (acc_res && c + 1 < c1) prefetch_residual(ep, M, m0 + q * 32, n0 + (c + 1) * 32, lane, res);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_free(tmem, 2 * BN);
  }
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    PSWA_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p)
      throw CudaError("cuTensorMapEncodeTiled entry point unavailable");
    fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

void make_tmap(CUtensorMap* m, const __half* base, int ld, int rows, int cols, int box_rows) {
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(base),
                           dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw CudaError("cuTensorMapEncodeTiled failed (code " + std::to_string(int(r)) + ")");
}

int sm_count() {
  static int n = [] {
    int dev = 0, v = 0;
    PSWA_CUDA(cudaGetDevice(&dev));
    PSWA_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
    return v;
  }();
  return n;
}

template <int BN, int EPI>
void set_attr() {
  static std::once_flag once;
  std::call_once(once, [] {
    PSWA_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<BN, EPI>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, GemmCfg<BN>::kSmem));
  });
}

int epi_kind(const GemmEpi& e) {
  if (e.act == kActSwiGLU) return kEpiSwiGLU;
  if (e.act == kActHead) return kEpiHead;
  return e.out_f32 ? kEpiF32 : kEpiF16;
}

template <int BN>
void prep(int kind) {
  switch (kind) {
    case kEpiF16: set_attr<BN, kEpiF16>(); break;
    case kEpiF32: set_attr<BN, kEpiF32>(); break;
    case kEpiSwiGLU: set_attr<BN, kEpiSwiGLU>(); break;
    default: set_attr<BN, kEpiHead>(); break;
  }
}

template <int BN>
void launch(const GemmPlan& p, int kind, cudaStream_t st) {
  const int tiles_m = (p.M + kBM - 1) / kBM;
  const int tiles = tiles_m * (p.N / BN);
  const int grid = tiles < sm_count() ? tiles : sm_count();
  const int smem = GemmCfg<BN>::kSmem;
  switch (kind) {
    case kEpiF16:
      launch_k(gemm_tc_kernel<BN, kEpiF16>, dim3(grid), dim3(kThreads), smem, st, p.ta, p.tb, p.M, p.K,
               tiles_m, tiles, p.epi);
      break;
    case kEpiF32:
      launch_k(gemm_tc_kernel<BN, kEpiF32>, dim3(grid), dim3(kThreads), smem, st, p.ta, p.tb, p.M, p.K,
               tiles_m, tiles, p.epi);
      break;
    case kEpiSwiGLU:
      launch_k(gemm_tc_kernel<BN, kEpiSwiGLU>, dim3(grid), dim3(kThreads), smem, st, p.ta, p.tb, p.M, p.K,
               tiles_m, tiles, p.epi);
      break;
    default:
      launch_k(gemm_tc_kernel<BN, kEpiHead>, dim3(grid), dim3(kThreads), smem, st, p.ta, p.tb, p.M, p.K,
               tiles_m, tiles, p.epi);
      break;
  }
}

}  // namespace

void gemm_plan(GemmPlan* p, const __half* A, int lda, int M, const __half* B, int ldb, int N,
               int K, const GemmEpi& epi, int force_bn) {
  if (K % kBK != 0 || N % 64 != 0 || lda % 8 != 0 || ldb % 8 != 0 || M <= 0)
    throw std::invalid_argument("gemm_plan: unsupported shape (K%64, N%64, ld%8)");
  int bn = force_bn;
  if (bn == 0) {
    // largest tile that still gives every SM work; small-M step GEMMs end
    // up on BN=64 (more CTAs), the 4-slot context GEMMs on BN=256
    const int mt = (M + kBM - 1) / kBM, sms = sm_count();
    if (N % 256 == 0 && mt * (N / 256) >= 2 * sms)
      bn = 256;
    else if (N % 128 == 0 && mt * (N / 128) >= sms)
      bn = 128;
    else
      bn = 64;
  }
  if (N % bn != 0 || (bn != 64 && bn != 128 && bn != 256))
    throw std::invalid_argument("gemm_plan: bad BN");
  p->M = M;
  p->N = N;
  p->K = K;
  p->BN = bn;
  p->epi = epi;
  make_tmap(&p->ta, A, lda, M, K, kBM);
  make_tmap(&p->tb, B, ldb, N, K, bn);
  const int kind = epi_kind(epi);
  if (bn == 64) prep<64>(kind);
  if (bn == 128) prep<128>(kind);
  if (bn == 256) prep<256>(kind);
}

void gemm_run(const GemmPlan& p, cudaStream_t stream) {
  const int kind = epi_kind(p.epi);
  switch (p.BN) {
    case 64: launch<64>(p, kind, stream); break;
    case 128: launch<128>(p, kind, stream); break;
    case 256: launch<256>(p, kind, stream); break;
    default: throw std::invalid_argument("gemm_run: bad BN");
  }
  PSWA_LAUNCH_CHECK();
}

}  // namespace pswa_dev
