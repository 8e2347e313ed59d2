// tcgen05 / TMA GEMM for sm_100a. See gemm.h for the contract.
//
// One CTA owns one 128 x BN output tile (cta_group::1, UMMA M=128, N=BN,
// K=16 per instruction). Warp roles:
//   warp 0  : TMA producer (one elected lane), STAGES-deep smem ring
//   warp 1  : TMEM allocator + MMA issuer (one elected lane)
//   warps 2-5: epilogue, TMEM -> registers -> fused op -> global
// K is walked in ascending 64-wide blocks and never split, so every output
// element has one fixed reduction order: results are bitwise reproducible
// run to run and independent of M (the encoder/decoder symmetry contract,
// SURVEY Appendix A2).
#include <cuda.h>

#include <cstdio>
#include <mutex>

#include "check.h"
#include "gemm.h"
#include "ptx.cuh"

namespace pswa_dev {

namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;  // 64 fp16 = 128 B = one SWIZZLE_128B row
constexpr int kThreads = 192;

template <int BN>
struct GemmCfg {
  static constexpr int kStages = BN == 64 ? 4 : 3;
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kSmem = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
};

__device__ __forceinline__ float silu_f(float v) { return v / (1.0f + __expf(-v)); }
__device__ __forceinline__ float softplus_f(float v) {
  if (v > 30.0f) return v;
  if (v < -30.0f) return __expf(v);
  return log1pf(__expf(v));
}

// Applies the fused epilogue to 32 consecutive accumulator columns
// [n0, n0+32) of output row m.
__device__ __forceinline__ void epilogue_chunk(const GemmEpi& ep, int m, int n0,
                                               const uint32_t (&raw)[32]) {
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(raw[j]);
  const int orow = ep.row_map ? ep.row_map[m] : m;
  if (orow < 0) return;

  if (ep.act == kActSwiGLU) {
    // pairs (gate, up) -> one output column each; output col = n0/2 + j
    const int oc0 = n0 >> 1;
    if (oc0 >= ep.n_store) return;
    __half h[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      float g = v[2 * j], u = v[2 * j + 1];
      if (ep.bias) {
        g += ep.bias[n0 + 2 * j];
        u += ep.bias[n0 + 2 * j + 1];
      }
      h[j] = __float2half_rn(silu_f(g) * u);
    }
    __half* dst = static_cast<__half*>(ep.out) + static_cast<size_t>(orow) * ep.ld_out + oc0;
    if (oc0 + 16 <= ep.n_store) {
      uint4* d4 = reinterpret_cast<uint4*>(dst);
      d4[0] = *reinterpret_cast<uint4*>(&h[0]);
      d4[1] = *reinterpret_cast<uint4*>(&h[8]);
    } else {
      for (int j = 0; j < 16 && oc0 + j < ep.n_store; ++j) dst[j] = h[j];
    }
    return;
  }

  if (n0 >= ep.n_store) return;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const int n = n0 + j;
    float x = v[j];
    if (ep.act == kActHead) {
      const float b = ep.bias ? ep.bias[n] : 0.0f;
      if (n < ep.split) {
        x = (x + b) * (ep.scale ? ep.scale[n] : 1.0f);
      } else {
        x = 0.11f + softplus_f(x + b);
      }
    } else {
      if (ep.bias_first) {
        if (ep.bias) x += ep.bias[n];
        if (ep.scale) x *= ep.scale[n];
      } else {
        if (ep.scale) x *= ep.scale[n];
        if (ep.bias) x += ep.bias[n];
      }
      if (ep.act == kActSilu) x = silu_f(x);
    }
    v[j] = x;
  }
  const bool full = n0 + 32 <= ep.n_store;
  if (ep.out_f32) {
    float* dst = static_cast<float*>(ep.out) + static_cast<size_t>(orow) * ep.ld_out + n0;
    if (full) {
      float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float4 o = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        if (ep.accumulate) {
          const float4 a = d4[q];
          o.x += a.x;
          o.y += a.y;
          o.z += a.z;
          o.w += a.w;
        }
        d4[q] = o;
      }
    } else {
      for (int j = 0; j < 32 && n0 + j < ep.n_store; ++j)
        dst[j] = ep.accumulate ? dst[j] + v[j] : v[j];
    }
  } else {
    __half* dst = static_cast<__half*>(ep.out) + static_cast<size_t>(orow) * ep.ld_out + n0;
    __half h[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) h[j] = __float2half_rn(v[j]);
    if (full) {
      uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
      for (int q = 0; q < 4; ++q) d4[q] = *reinterpret_cast<uint4*>(&h[8 * q]);
    } else {
      for (int j = 0; j < 32 && n0 + j < ep.n_store; ++j) dst[j] = h[j];
    }
  }
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tma, const __grid_constant__ CUtensorMap tmb,
                   int M, int K, const __grid_constant__ GemmEpi ep) {
  using Cfg = GemmCfg<BN>;
  constexpr int S = Cfg::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sa = smem;
  uint8_t* sb = smem + S * Cfg::kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * Cfg::kStageBytes);
  uint64_t* empty = full + S;
  uint64_t* done = empty + S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * kBM;
  const int n0 = blockIdx.y * BN;
  const int kblocks = K / kBK;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tma);
    tma_prefetch(&tmb);
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, BN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < kblocks; ++kb) {
        const int s = kb % S;
        const int round = kb / S;
        if (round > 0) mbar_wait(&empty[s], (round - 1) & 1);
        mbar_expect_tx(&full[s], Cfg::kStageBytes);
        tma_load_2d(sa + s * Cfg::kABytes, &tma, &full[s], kb * kBK, m0);
        tma_load_2d(sb + s * Cfg::kBBytes, &tmb, &full[s], kb * kBK, n0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_f16_f32(kBM, BN);
      for (int kb = 0; kb < kblocks; ++kb) {
        const int s = kb % S;
        mbar_wait(&full[s], (kb / S) & 1);
        tc_fence_after();
        const uint32_t a_base = smem_u32(sa + s * Cfg::kABytes);
        const uint32_t b_base = smem_u32(sb + s * Cfg::kBBytes);
#pragma unroll
        for (int kk = 0; kk < kBK / 16; ++kk) {
          const uint64_t ad = umma_desc_k_sw128(a_base + kk * 32);
          const uint64_t bd = umma_desc_k_sw128(b_base + kk * 32);
          tc_mma_f16(tmem, ad, bd, idesc, (kb | kk) != 0 ? 1u : 0u);
        }
        tc_commit(&empty[s]);
      }
      tc_commit(done);
    }
  } else {
    // epilogue warps 2..5 -> TMEM lane quarter (warp % 4)
    const int q = warp & 3;
    mbar_wait(done, 0);
    tc_fence_after();
    const int m = m0 + q * 32 + lane;
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      uint32_t raw[32];
      tmem_ld_32x32(tmem + (static_cast<uint32_t>(q * 32) << 16) + c * 32, raw);
      tc_wait_ld();
      if (m < M) epilogue_chunk(ep, m, n0 + c * 32, raw);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_free(tmem, BN);
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

template <int BN>
void set_smem_attr() {
  static std::once_flag once;
  std::call_once(once, [] {
    PSWA_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   GemmCfg<BN>::kSmem));
  });
}

}  // namespace

void gemm_plan(GemmPlan* p, const __half* A, int lda, int M, const __half* B, int ldb, int N,
               int K, const GemmEpi& epi, int force_bn) {
  if (K % kBK != 0 || N % 64 != 0 || lda % 8 != 0 || ldb % 8 != 0 || M <= 0)
    throw std::invalid_argument("gemm_plan: unsupported shape (K%64, N%64, ld%8)");
  int bn = force_bn;
  if (bn == 0) {
    const int mt = (M + kBM - 1) / kBM;
    if (N % 256 == 0 && mt * (N / 256) >= 2 * 148)
      bn = 256;
    else if (N % 128 == 0 && mt * (N / 128) >= 148)
      bn = 128;
    else
      bn = 64;
  }
  if (N % bn != 0) throw std::invalid_argument("gemm_plan: N % BN != 0");
  p->M = M;
  p->N = N;
  p->K = K;
  p->BN = bn;
  p->epi = epi;
  make_tmap(&p->ta, A, lda, M, K, kBM);
  make_tmap(&p->tb, B, ldb, N, K, bn);
  if (bn == 64) set_smem_attr<64>();
  if (bn == 128) set_smem_attr<128>();
  if (bn == 256) set_smem_attr<256>();
}

void gemm_run(const GemmPlan& p, cudaStream_t stream) {
  dim3 grid((p.M + kBM - 1) / kBM, p.N / p.BN);
  switch (p.BN) {
    case 64:
      gemm_tc_kernel<64><<<grid, kThreads, GemmCfg<64>::kSmem, stream>>>(p.ta, p.tb, p.M, p.K,
                                                                         p.epi);
      break;
    case 128:
      gemm_tc_kernel<128><<<grid, kThreads, GemmCfg<128>::kSmem, stream>>>(p.ta, p.tb, p.M,
                                                                           p.K, p.epi);
      break;
    case 256:
      gemm_tc_kernel<256><<<grid, kThreads, GemmCfg<256>::kSmem, stream>>>(p.ta, p.tb, p.M,
                                                                           p.K, p.epi);
      break;
    default:
      throw std::invalid_argument("gemm_run: bad BN");
  }
  PSWA_LAUNCH_CHECK();
}

}  // namespace pswa_dev
