// tcgen05 / TMA GEMM for sm_100a. See gemm.h for the contract.
//
// Persistent kernel, one CTA per SM, 128 x BN output tiles (cta_group::1,
// UMMA M=128, N=BN, K=16 per instruction; BN 64 / 128 / 192 / 256, and 352
// as two N=176 MMAs per K step), tiles walked N-fastest: the
// weights (<= 3 MB) stay L2-resident and the CTAs in flight share each
// activation row panel, which is then read from HBM once (M-fastest order
// re-streamed the whole activation matrix from HBM for every N tile of the
// 32640-row context GEMMs). Warp roles:
//   warp 0    : TMA producer (one elected lane), STAGES-deep smem ring
//   warp 1    : TMEM allocator + MMA issuer (one elected lane)
//   warps 2-9 : epilogue. Two TMEM accumulators (2 x BN columns; one at BN 352) let the
//               epilogue of tile i overlap the MMAs of tile i+1. Each warp
//               drains one 32-lane quarter x one column half; lane = output
//               row, written with 16 B stores straight from registers.
// The epilogue kind is a template parameter (no per-element mode branches).
// K is walked in ascending 64-wide blocks: every output element has one
// fixed reduction order, so results are bitwise identical run to run and
// independent of M and of the tile schedule (the encoder/decoder symmetry
// contract). The one exception is opt-in per layer
// (GemmEpi::split_k, gemm_splitk_kernel below): two fixed K halves summed as
// fl(P0 + P1), again independent of M and schedule.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
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

enum EpiKind : int { kEpiF16 = 0, kEpiF32 = 1, kEpiSwiGLU = 2, kEpiHead = 3 };

template <int BN>
struct GemmCfg {
  // as deep as shared memory allows (<= 227 KB with the epilogue staging):
  // the small-M step GEMMs are latency bound, so all K blocks in flight helps
  static constexpr int kStages = BN == 352 ? 3 : BN >= 192 ? 4 : (BN == 128 ? 6 : 8);
  // BN = 352 (the 2040-row gate|up GEMMs in one wave of 128 tiles instead of
  // 176 tiles over 148 SMs): two N = 176 MMAs per K step (UMMA N <= 256),
  // two 176-row B boxes per stage (TMA box <= 256 rows), one accumulator
  // (2 x 352 columns exceed the 512 of TMEM)
  static constexpr int kBSplit = BN > 256 ? 2 : 1;
  static constexpr int kSubN = BN / kBSplit;
  static constexpr int kAccBufs = 2 * BN <= 512 ? 2 : 1;
  static constexpr int kTmemCols = kAccBufs * BN <= 128 ? 128 : kAccBufs * BN <= 256 ? 256 : 512;
  static_assert(kStages * (kBM * kBK * 2 + BN * kBK * 2) + 1280 + kEpiWarps * 4096 <= 227 * 1024, "smem");
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kSmem = kStages * kStageBytes + 1024 + 256;
  // + one 32 x 128 B store stage per epilogue warp (warp_store_rows) for the
  // fp32-output kinds only: the others keep the smaller carve-out (more L1)
  static constexpr int smem_for(int epi) { return kSmem + ((epi == 1 || epi == 3) ? kEpiWarps * 4096 : 0); }
};

__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// silu(v) = v * sigmoid(v) = v * (0.5 + 0.5 tanh(v / 2)): one MUFU op per
// element instead of two (ex2 + rcp); the SwiGLU epilogue of the wide
// GEMMs is MUFU-paced (PSWA_SILU_EXP=1: the exp / divide form).
__device__ __forceinline__ float silu_f(float v) {
#ifdef PSWA_SILU_EXP
  return __fdividef(v, 1.0f + __expf(-v));
#else
  const float h = 0.5f * v;
  return fmaf(h, tanh_approx(h), h);
#endif
}

// Elementwise part of the epilogue for 32 accumulator columns [n0, n0+32).
// Head column parameters of columns [n0, n0 + 32): bias (0 past n_store)
// and rate scale (1 on the sigma columns, which read none).
__device__ __forceinline__ void head_params(const GemmEpi& ep, int n0, float4 (&b)[8], float4 (&s)[8]) {
  float bv[32], sv[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    bv[j] = (ep.bias && n0 + j < ep.n_store) ? ep.bias[n0 + j] : 0.0f;
    sv[j] = (ep.scale && n0 + j < ep.split) ? ep.scale[n0 + j] : 1.0f;
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    b[q] = make_float4(bv[4 * q], bv[4 * q + 1], bv[4 * q + 2], bv[4 * q + 3]);
    s[q] = make_float4(sv[4 * q], sv[4 * q + 1], sv[4 * q + 2], sv[4 * q + 3]);
  }
}
__device__ __forceinline__ float f4_at(const float4* a, int j) {
  const float4 x = a[j >> 2];
  return (j & 3) == 0 ? x.x : (j & 3) == 1 ? x.y : (j & 3) == 2 ? x.z : x.w;
}

template <int EPI>
__device__ __forceinline__ void epi_values(const GemmEpi& ep, int n0, float (&v)[32],
                                           const float4* hb = nullptr, const float4* hs = nullptr) {
  if (EPI == kEpiHead) {
    // mu = (v + b) * scale; sigma = 0.11 + softplus(v + b) with softplus(x)
    // = x above 30, exp(x) below -30, log1p(exp(x)) between; evaluated
    // branch-free with the column parameters loaded up front (per-element
    // branches and loads made this epilogue ~11k cycles per tile), or
    // before the accumulator wait (hb / hs: head_params)
    float b[32], sc[32];
    if (hb) {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        b[j] = f4_at(hb, j);
        sc[j] = f4_at(hs, j);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        b[j] = ep.bias ? ep.bias[n0 + j] : 0.0f;
        // the rate scales cover the mu columns only (sigma columns read none)
        sc[j] = (ep.scale && n0 + j < ep.split) ? ep.scale[n0 + j] : 1.0f;
      }
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float x = v[j] + b[j];
      if (n0 + j < ep.split) {
        v[j] = x * sc[j];
      } else {
        // softplus with two MUFU ops (ex2, lg2); log(1 + e) loses relative
        // accuracy only where softplus < ~1e-4, i.e. < 1e-3 of sigma's 0.11
        // floor (libdevice log1pf made this epilogue the launch's tail)
        const float e = __expf(x);
        const float l = __logf(1.0f + e);
        v[j] = 0.11f + (x > 30.0f ? x : (x < -30.0f ? e : l));
      }
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
  } else if (ep.act == kActTanhHalf) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = 0.5f * tanhf(v[j]);
  }
}

// 256-bit global accesses (sm_100): one lane moves a whole 32 B sector per
// instruction, so the row-per-lane epilogue writes full sectors.
__device__ __forceinline__ void st_v8(void* p, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                      uint32_t a4, uint32_t a5, uint32_t a6, uint32_t a7) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a0), "r"(a1),
               "r"(a2), "r"(a3), "r"(a4), "r"(a5), "r"(a6), "r"(a7)
               : "memory");
}
__device__ __forceinline__ void ld_v8(const void* p, float4& x, float4& y) {
  asm volatile("ld.global.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w), "=f"(y.x), "=f"(y.y), "=f"(y.z), "=f"(y.w)
               : "l"(p));
}

// Residual segment (32 fp32 of output row `orow` at column oc0) loaded ahead
// of the accumulator wait so its latency overlaps the MMAs.
__device__ __forceinline__ void prefetch_residual(const GemmEpi& ep, int orow, int oc0,
                                                  float4 (&res)[8]) {
#pragma unroll
  for (int q = 0; q < 8; ++q) res[q] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (orow < 0 || oc0 + 32 > ep.n_store) return;
  const float4* src = reinterpret_cast<const float4*>(static_cast<const float*>(ep.out) +
                                                      static_cast<size_t>(orow) * ep.ld_out + oc0);
  if (ep.v8) {
#pragma unroll
    for (int q = 0; q < 8; q += 2) ld_v8(src + q, res[q], res[q + 1]);
  } else {
#pragma unroll
    for (int q = 0; q < 8; ++q) res[q] = src[q];
  }
}

// Coalesced store of one row segment per lane (the TMEM layout: lane = row)
// through this warp's swizzled 32 x 128 B smem stage: the lanes first write
// their NCH 16 B chunks (chunk c of row r at position c ^ (r & 7)), then store
// whole row segments -- NCH lanes per row, 32 / NCH rows per instruction --
// so a warp instruction writes 4 full 128 B lines (NCH = 8) instead of 32
// scattered 32 B sectors. `dst` (nullable: row skipped) is this lane's row.
template <int NCH>
__device__ __forceinline__ void warp_store_rows(uint32_t stg, const uint4 (&d)[NCH], void* dst, int lane) {
#pragma unroll
  for (int c = 0; c < NCH; ++c)
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(stg + lane * 128 + ((c ^ (lane & 7)) << 4)),
                 "r"(d[c].x), "r"(d[c].y), "r"(d[c].z), "r"(d[c].w)
                 : "memory");
  __syncwarp();
  constexpr int kRows = 32 / NCH;  // rows per instruction
#pragma unroll
  for (int k = 0; k < NCH; ++k) {
    const int row = k * kRows + lane / NCH, ch = lane % NCH;
    const unsigned long long base = __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(dst), row);
    uint4 val;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(val.x), "=r"(val.y), "=r"(val.z), "=r"(val.w)
                 : "r"(stg + row * 128 + ((ch ^ (row & 7)) << 4))
                 : "memory");
    if (base) reinterpret_cast<uint4*>(base)[ch] = val;
  }
  __syncwarp();
}

// Drain one accumulator row segment: lane = TMEM lane = output row, columns
// n0..n0+31; fused op, then straight 16 B stores from registers (each lane
// writes whole 32 B sectors of its own row).
template <int EPI>
__device__ __forceinline__ void epi_chunk(const GemmEpi& ep, int orow, int n0,
                                          const uint32_t (&raw)[32], const float4 (&res)[8],
                                          float row_scale, bool side2, uint32_t stg = 0,
                                          const float4* hb = nullptr, const float4* hs = nullptr,
                                          const CUtensorMap* tmo = nullptr, int box_row = 0) {
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(raw[j]) * row_scale;
  epi_values<EPI>(ep, n0, v, hb, hs);
  const int ncols = EPI == kEpiSwiGLU ? 16 : 32;
  const int oc0 = EPI == kEpiSwiGLU ? (n0 >> 1) : n0;
  if (oc0 >= ep.n_store) return;  // (warp-uniform)
  const bool full = oc0 + ncols <= ep.n_store;
  // warp-cooperative coalesced stores (every lane takes part, rows < 0
  // skipped): measured 6.7 -> 6.4 us (out-proj), 7.5 -> 7.2 us (channel down)
  if (stg && full && ep.v8) {
    if (EPI == kEpiF32 || EPI == kEpiHead) {
      float ss = 0.0f;
      uint4 ov[8], hp[4];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float4 o = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        if (EPI == kEpiF32 && ep.accumulate) {
          o.x += res[q].x;
          o.y += res[q].y;
          o.z += res[q].z;
          o.w += res[q].w;
        }
        ov[q] = make_uint4(__float_as_uint(o.x), __float_as_uint(o.y), __float_as_uint(o.z), __float_as_uint(o.w));
        ss = fmaf(o.x, o.x, ss);
        ss = fmaf(o.y, o.y, ss);
        ss = fmaf(o.z, o.z, ss);
        ss = fmaf(o.w, o.w, ss);
        __half2 h0 = __floats2half2_rn(o.x, o.y), h1 = __floats2half2_rn(o.z, o.w);
        (q & 1 ? hp[q >> 1].z : hp[q >> 1].x) = *reinterpret_cast<uint32_t*>(&h0);
        (q & 1 ? hp[q >> 1].w : hp[q >> 1].y) = *reinterpret_cast<uint32_t*>(&h1);
      }
      if (EPI == kEpiF32 && tmo) {
        // fp16 row copy through the stage first, then the fp32 rows leave it
        // by one TMA store (32 x 32 fp32 box at (oc0, box_row); rows past M
        // are clipped), so the lanes issue no shared loads / global stores
        // for them; the stage is reusable once the TMA has read it
        const int ln = threadIdx.x & 31;
        if (ep.x16_out)
          warp_store_rows<4>(stg, hp, orow >= 0 ? ep.x16_out + static_cast<size_t>(orow) * ep.ld_x16 + oc0 : nullptr, ln);
#pragma unroll
        for (int c = 0; c < 8; ++c)
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(stg + ln * 128 + ((c ^ (ln & 7)) << 4)),
                       "r"(ov[c].x), "r"(ov[c].y), "r"(ov[c].z), "r"(ov[c].w)
                       : "memory");
        fence_proxy_async_smem();
        __syncwarp();
        if (ln == 0) {
          tma_store_2d(tmo, stg, oc0, box_row);
          bulk_commit();
          bulk_wait_read0();
        }
        __syncwarp();
      } else {
        warp_store_rows<8>(stg, ov, orow >= 0 ? static_cast<float*>(ep.out) + static_cast<size_t>(orow) * ep.ld_out + oc0 : nullptr,
                           threadIdx.x & 31);
        if (EPI == kEpiF32 && ep.x16_out)
          warp_store_rows<4>(stg, hp, orow >= 0 ? ep.x16_out + static_cast<size_t>(orow) * ep.ld_x16 + oc0 : nullptr,
                             threadIdx.x & 31);
      }
      if (EPI == kEpiF32 && ep.ssq_out && orow >= 0) ep.ssq_out[static_cast<size_t>(orow) * ep.ld_ssq + (oc0 >> 5)] = ss;
    } else {
      constexpr int NCH = EPI == kEpiSwiGLU ? 2 : 4;  // 16 / 32 fp16 per row
      uint4 hp[NCH];
#pragma unroll
      for (int q = 0; q < NCH; ++q) {
        uint32_t w[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          __half2 h2 = __floats2half2_rn(v[8 * q + 2 * e], v[8 * q + 2 * e + 1]);
          w[e] = *reinterpret_cast<uint32_t*>(&h2);
        }
        hp[q] = make_uint4(w[0], w[1], w[2], w[3]);
      }
      __half* dst = orow < 0 ? nullptr
                    : side2  ? static_cast<__half*>(ep.out2) + static_cast<size_t>(orow) * ep.ld_out2 + oc0 - ep.split_n
                             : static_cast<__half*>(ep.out) + static_cast<size_t>(orow) * ep.ld_out + oc0;
      warp_store_rows<NCH>(stg, hp, dst, threadIdx.x & 31);
    }
    return;
  }
  if (orow < 0) return;
  if (EPI == kEpiF32 || EPI == kEpiHead) {
    float* dst = static_cast<float*>(ep.out) + static_cast<size_t>(orow) * ep.ld_out + oc0;
    if ((EPI == kEpiF32 || EPI == kEpiHead) && full) {  // (head: no residual / norm outputs)
      float4* d4 = reinterpret_cast<float4*>(dst);
      float ss = 0.0f;
      uint32_t hp[16];
      float4 ov[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float4 o = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        if (ep.accumulate) {
          o.x += res[q].x;
          o.y += res[q].y;
          o.z += res[q].z;
          o.w += res[q].w;
        }
        ov[q] = o;
        if (!ep.v8) d4[q] = o;
        ss = fmaf(o.x, o.x, ss);
        ss = fmaf(o.y, o.y, ss);
        ss = fmaf(o.z, o.z, ss);
        ss = fmaf(o.w, o.w, ss);
        __half2 h0 = __floats2half2_rn(o.x, o.y), h1 = __floats2half2_rn(o.z, o.w);
        hp[2 * q] = *reinterpret_cast<uint32_t*>(&h0);
        hp[2 * q + 1] = *reinterpret_cast<uint32_t*>(&h1);
      }
      if (ep.v8) {
#pragma unroll
        for (int q = 0; q < 8; q += 2)
          st_v8(d4 + q, __float_as_uint(ov[q].x), __float_as_uint(ov[q].y), __float_as_uint(ov[q].z),
                __float_as_uint(ov[q].w), __float_as_uint(ov[q + 1].x), __float_as_uint(ov[q + 1].y),
                __float_as_uint(ov[q + 1].z), __float_as_uint(ov[q + 1].w));
      }
      if (ep.x16_out) {  // next RMSNorm's input: fp16 copy of the updated row
        uint4* h4 = reinterpret_cast<uint4*>(ep.x16_out + static_cast<size_t>(orow) * ep.ld_x16 + oc0);
        if (ep.v8) {
          st_v8(h4, hp[0], hp[1], hp[2], hp[3], hp[4], hp[5], hp[6], hp[7]);
          st_v8(h4 + 2, hp[8], hp[9], hp[10], hp[11], hp[12], hp[13], hp[14], hp[15]);
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q) h4[q] = make_uint4(hp[4 * q], hp[4 * q + 1], hp[4 * q + 2], hp[4 * q + 3]);
        }
      }
      if (ep.ssq_out) ep.ssq_out[static_cast<size_t>(orow) * ep.ld_ssq + (oc0 >> 5)] = ss;
    } else {
      for (int j = 0; j < 32 && oc0 + j < ep.n_store; ++j)
        dst[j] = (EPI == kEpiF32 && ep.accumulate) ? dst[j] + v[j] : v[j];
    }
  } else {
    __half* dst = side2 ? static_cast<__half*>(ep.out2) + static_cast<size_t>(orow) * ep.ld_out2 + oc0 - ep.split_n
                        : static_cast<__half*>(ep.out) + static_cast<size_t>(orow) * ep.ld_out + oc0;
    uint32_t hp[16];
#pragma unroll
    for (int j = 0; j < ncols / 2; ++j) {
      __half2 h2 = __floats2half2_rn(v[2 * j], v[2 * j + 1]);
      hp[j] = *reinterpret_cast<uint32_t*>(&h2);
    }
    if (full && ep.v8) {
#pragma unroll
      for (int q = 0; q < ncols / 16; ++q)
        st_v8(dst + 16 * q, hp[8 * q], hp[8 * q + 1], hp[8 * q + 2], hp[8 * q + 3], hp[8 * q + 4],
              hp[8 * q + 5], hp[8 * q + 6], hp[8 * q + 7]);
    } else if (full) {
      uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
      for (int q = 0; q < ncols / 8; ++q) d4[q] = make_uint4(hp[4 * q], hp[4 * q + 1], hp[4 * q + 2], hp[4 * q + 3]);
    } else {
      for (int j = 0; j < ncols && oc0 + j < ep.n_store; ++j) dst[j] = __float2half_rn(v[j]);
    }
  }
}

#ifdef PSWA_GEMM_TRACE_BUILD
__device__ int g_gemm_exp = 0;
#endif

template <int BN, int EPI, int CL>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tma, const __grid_constant__ CUtensorMap tmb,
                   const __grid_constant__ CUtensorMap tmo, int M, int K, int tiles_m, int num_tiles,
                   const __grid_constant__ GemmEpi ep) {
  using Cfg = GemmCfg<BN>;
  constexpr int S = Cfg::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sa = smem;
  uint8_t* sb = smem + S * Cfg::kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * Cfg::kStageBytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  // per-warp 32 x 128 B store stages (warp_store_rows): a CTA with a single
  // tile reuses its A stage ring (all MMAs have read it when the accumulator
  // is ready); persistent multi-tile CTAs of the fp32-output kinds use the
  // region allocated after the barriers; the others store row-per-lane
  const bool single_tile = CL == 1 && num_tiles <= static_cast<int>(gridDim.x);
  uint8_t* stg_base = single_tile ? sa
                      : (EPI == kEpiF32 || EPI == kEpiHead) ? smem + S * Cfg::kStageBytes + 1024 : nullptr;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int kblocks = K / kBK;
  // phase stamps: compiled in only with -DPSWA_GEMM_TRACE_BUILD (make
  // TRACE=1), so production kernels carry no trace branches
#ifdef PSWA_GEMM_TRACE_BUILD
  unsigned long long* const tr = ep.trace ? ep.trace + blockIdx.x * kGemmTraceSlots : nullptr;
#else
  constexpr unsigned long long* tr = nullptr;
#endif
  auto stamp = [&](int slot) {
    if (tr) tr[slot] = clock64();
  };
  // timing experiments of the trace build (gemm_set_experiment): 1 = no
  // MMAs, 2 = no operand loads after the first pipeline round
#ifdef PSWA_GEMM_TRACE_BUILD
  const int exp_flags = g_gemm_exp;
#else
  constexpr int exp_flags = 0;
#endif
  const bool exp_no_mma = exp_flags & 1, exp_no_tma = exp_flags & 2;
  if (tr && threadIdx.x == 0) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    tr[8] = g;
    stamp(0);
  }
  // tile schedule: CL CTAs of a cluster take adjacent M tiles of one N tile
  const int rank = CL > 1 ? static_cast<int>(cluster_ctarank()) : 0;
  const int tiles_mp = (tiles_m + CL - 1) / CL, tiles_n = num_tiles / tiles_m;
  const int n_units = tiles_mp * tiles_n;
  const int unit0 = blockIdx.x / CL, unit_step = gridDim.x / CL;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tma);
    tma_prefetch(&tmb);
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CL);  // released by the MMAs of every CTA reading it
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], kEpiWarps);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, Cfg::kTmemCols);
  tc_fence_before();
  if (CL > 1)
    cluster_sync();  // peer barriers initialised before any multicast
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) stamp(1);
  // B is always a packed weight matrix (constant for the whole program): the
  // first tile's B stages are requested before the PDL wait, so they land
  // while the previous kernel drains; A (an activation) follows the wait
  int npre = 0;
  if (CL == 1 && warp == 0 && lane == 0 && unit0 < n_units) {
    const int n0 = (unit0 % tiles_n) * BN;
    npre = min(S, kblocks);
    for (int kb = 0; kb < npre; ++kb) {
      mbar_expect_tx(&full[kb], Cfg::kStageBytes);
#pragma unroll
      for (int h = 0; h < Cfg::kBSplit; ++h)
        tma_load_2d(sb + kb * Cfg::kBBytes + h * Cfg::kSubN * 128, &tmb, &full[kb], kb * kBK, n0 + h * Cfg::kSubN);
    }
  }
  // everything above overlaps the previous kernel (PDL); inputs are read below
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0) stamp(2);

  if (warp == 0) {
    if (lane == 0) {
      // A operand: a 2D box of the row-major activation, or (conv_w > 0)
      // the 128 output pixels' patches of one 3x3 tap and 64 channels,
      // gathered from the NHWC image by TMA in im2col mode
      auto load_a = [&](uint8_t* dst, uint64_t* bar, int kb, int m0) {
        if (ep.conv_w > 0) {
          // coordinates live in the map's bounding box, which starts at its
          // lower corner (-1, -1): output pixel (x, y) -> (x - 1, y - 1)
          const int tap = kb / ep.conv_cb;
          tma_load_im2col_4d(dst, &tma, bar, (kb - tap * ep.conv_cb) * kBK, m0 % ep.conv_w - 1, m0 / ep.conv_w - 1,
                             0, static_cast<uint16_t>(tap % 3), static_cast<uint16_t>(tap / 3));
        } else {
          tma_load_2d(dst, &tma, bar, kb * kBK, m0);
        }
      };
      int g = 0;  // global k-block counter across tiles
      for (int u = unit0; u < n_units; u += unit_step) {
        const int m0 = ((u / tiles_n) * CL + rank) * kBM, n0 = (u % tiles_n) * BN;
        for (int kb = 0; kb < kblocks; ++kb, ++g) {
          const int s = g % S, round = g / S;
          if (g < npre) {  // B already requested (and the stage's bytes expected)
            load_a(sa + s * Cfg::kABytes, &full[s], kb, m0);
            continue;
          }
          if (round > 0) mbar_wait(&empty[s], (round - 1) & 1);
          if (exp_no_tma) {  // timing experiment: stale operands
            mbar_arrive(&full[s]);
            continue;
          }
          mbar_expect_tx(&full[s], Cfg::kStageBytes);
          load_a(sa + s * Cfg::kABytes, &full[s], kb, m0);
          if (CL > 1)
            tma_load_2d_mc(sb + s * Cfg::kBBytes + rank * (Cfg::kBBytes / CL), &tmb, &full[s],
                           kb * kBK, n0 + rank * (BN / CL), static_cast<uint16_t>((1u << CL) - 1));
          else
#pragma unroll
            for (int h = 0; h < Cfg::kBSplit; ++h)
              tma_load_2d(sb + s * Cfg::kBBytes + h * Cfg::kSubN * 128, &tmb, &full[s], kb * kBK, n0 + h * Cfg::kSubN);
        }
      }
      stamp(10);
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_f16_f32(kBM, Cfg::kSubN);
      int g = 0, it = 0;
      for (int u = unit0; u < n_units; u += unit_step, ++it) {
        const int buf = it % Cfg::kAccBufs, use = it / Cfg::kAccBufs;
        if (use > 0) mbar_wait(&tempty[buf], (use - 1) & 1);  // epilogue drained it
        tc_fence_after();
        const uint32_t acc = tmem + buf * BN;
        for (int kb = 0; kb < kblocks; ++kb, ++g) {
          const int s = g % S;
          mbar_wait(&full[s], (g / S) & 1);
          if (g == 0) stamp(3);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sa + s * Cfg::kABytes);
          const uint32_t b_base = smem_u32(sb + s * Cfg::kBBytes);
          if (!exp_no_mma) {
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk)
#pragma unroll
              for (int h = 0; h < Cfg::kBSplit; ++h)
                tc_mma_f16(acc + h * Cfg::kSubN, umma_desc_k_sw128(a_base + kk * 32),
                           umma_desc_k_sw128(b_base + h * Cfg::kSubN * 128 + kk * 32), idesc,
                           (kb | kk) != 0 ? 1u : 0u);
          }
          if (CL > 1)
            tc_commit_mc(&empty[s], static_cast<uint16_t>((1u << CL) - 1));
          else
            tc_commit(&empty[s]);
        }
        tc_commit(&tfull[buf]);
      }
      stamp(4);
    }
  } else {
    const int ew = warp - 2;
    const bool no_coalesce = !ep.coalesce;
    const bool use_tmo = EPI == kEpiF32 && ep.tma_store && stg_base != nullptr && !no_coalesce;
    const int q = warp & 3;                // TMEM lane quarter this warp may access
    const int half = ew >> 2;              // column half of the tile
    int it = 0;
    for (int u = unit0; u < n_units; u += unit_step, ++it) {
      const int buf = it % Cfg::kAccBufs, use = it / Cfg::kAccBufs;
      const int m0 = ((u / tiles_n) * CL + rank) * kBM, n0 = (u % tiles_n) * BN;
      // 32-column chunks split between the two column halves (6 + 5 at BN 352)
      constexpr int kCh = BN / 32, kCh0 = (kCh + 1) / 2;
      const int c0 = half ? kCh0 : 0, c1 = half ? kCh : kCh0;
      const int m = m0 + q * 32 + lane;
      // fused second output (columns >= split_n, own row map): decided per
      // 32-column chunk, so a tile may straddle split_n (BN 192 over the
      // 512 + 1024 Q|K|V columns); the residual kinds never split
      const bool side2_any = ep.out2 != nullptr && n0 + BN > ep.split_n;
      const bool side2 = ep.out2 != nullptr && n0 >= ep.split_n;
      const int* rmap = side2 ? ep.row_map2 : ep.row_map;
      const int orow = m < M ? (rmap ? rmap[m] : m) : -1;
      const int orow2 = side2_any && m < M ? (ep.row_map2 ? ep.row_map2[m] : m) : -1;
      // residual segments prefetched two chunks ahead (two register
      // buffers): the row-per-lane residual read is the epilogue's HBM
      // latency chain in the 32640-row context GEMMs
      float4 resA[8], resB[8];
      const bool acc_res = EPI == kEpiF32 && ep.accumulate;
      if (acc_res) {
        prefetch_residual(ep, orow, n0 + c0 * 32, resA);
        if (c0 + 1 < c1) prefetch_residual(ep, orow, n0 + (c0 + 1) * 32, resB);
        // the rest of this lane's residual segment is pulled into L2 by one
        // bulk prefetch while the tile's MMAs run, so the in-loop loads two
        // chunks ahead hit L2 instead of waiting out HBM latency (the
        // 32640-row residual GEMMs are epilogue-latency-bound)
        if (ep.l2_prefetch && orow >= 0 && c0 + 2 < c1) {
          const int col0 = n0 + (c0 + 2) * 32, col1 = min(n0 + c1 * 32, ep.n_store);
          if (col1 > col0)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                             static_cast<const float*>(ep.out) + static_cast<size_t>(orow) * ep.ld_out + col0),
                         "r"(static_cast<uint32_t>(col1 - col0) * 4u)
                         : "memory");
        }
      }
      // head with one chunk per warp: its bias / rate scales (resA / resB)
      // are loaded ahead of the accumulator wait as well
      const bool head_pre = EPI == kEpiHead && c1 - c0 == 1;
      if (head_pre) head_params(ep, n0 + c0 * 32, resA, resB);
      float row_scale = 1.0f;  // folded RMSNorm of A's row m
      if (ep.rms_ssq && m < M) {
        const float* sp = ep.rms_ssq + static_cast<size_t>(m) * ep.ld_rms;
        float ss = 0.0f;
        if ((ep.rms_parts & 3) == 0 && (ep.ld_rms & 3) == 0) {  // 16 B loads (the row's 64 B)
          for (int k = 0; k < ep.rms_parts; k += 4) {
            const float4 q4 = *reinterpret_cast<const float4*>(sp + k);
            ss += q4.x;
            ss += q4.y;
            ss += q4.z;
            ss += q4.w;
          }
        } else {
          for (int k = 0; k < ep.rms_parts; ++k) ss += sp[k];
        }
        row_scale = 1.0f / sqrtf(ss * ep.rms_inv_d + 1e-5f);
      }
      if (ew == 0 && lane == 0 && it == 0) stamp(13);  // epilogue inputs (residual, row scale) issued
      mbar_wait(&tfull[buf], use & 1);
      if (ew == 0 && lane == 0 && it == 0) stamp(5);
      tc_fence_after();
      const uint32_t acc = tmem + buf * BN + (static_cast<uint32_t>(q * 32) << 16);
      auto chunk = [&](int c, float4 (&res)[8]) {
        uint32_t raw[32];
        tmem_ld_32x32(acc + c * 32, raw);
        tc_wait_ld();
        if (ew == 0 && lane == 0 && it == 0 && c == c0) stamp(11);
        if (c + 1 == c1) {
          // accumulator fully read: hand it back to the MMA warp early
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[buf]);
        }
        const bool s2 = side2_any && n0 + c * 32 >= ep.split_n;
        epi_chunk<EPI>(ep, s2 ? orow2 : orow, n0 + c * 32, raw, res, row_scale, s2,
                       (no_coalesce || !stg_base) ? 0u : smem_u32(stg_base + ew * 4096),
                       head_pre ? resA : nullptr, head_pre ? resB : nullptr,
                       use_tmo ? &tmo : nullptr, m0 + q * 32);
        if (ew == 0 && lane == 0 && it == 0 && c == c0) stamp(12);
        if (acc_res && c + 2 < c1) prefetch_residual(ep, orow, n0 + (c + 2) * 32, res);
      };
#pragma unroll 1
      for (int c = c0; c < c1; c += 2) {
        chunk(c, resA);
        if (c + 1 < c1) chunk(c + 1, resB);
      }
    }
    if (use_tmo && lane == 0) bulk_wait0();  // this warp's TMA stores complete
    if (ew == 0 && lane == 0) stamp(6);
  }
  tc_fence_before();
  if (CL > 1)
    cluster_sync();  // no multicast / remote arrive can still target this CTA
  else
    __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_free(tmem, Cfg::kTmemCols);
  }
  if (tr && threadIdx.x == 0) {
    stamp(7);
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    tr[9] = g;
  }
}

// ------------------------------------------------------------ GEMM chain --
// See gemm.h (gemm_chain_*). One persistent CTA per SM, BN = 128, the warp
// roles of gemm_tc_kernel; the tile sequence is the concatenation of the jobs'
// tiles (each N-fastest) handed out by an atomic counter through a 4-deep
// smem queue shared by the producer, the MMA warp and the epilogue warps.
constexpr int kChBN = 128;
constexpr int kChStages = 6;
constexpr int kChQ = 4;
struct ChainJobDev {
  CUtensorMap ta, tb;
  GemmEpi ep;
  int M, K, tiles_m, tiles_n, kind, first;
};
struct ChainArgs {
  ChainJobDev job[kChainMaxJobs];
  int njobs, total, ctr_stride;
  unsigned* ctr;  // [kChainMaxJobs][ctr_stride] row-block completions, then tile counter, done
};
constexpr int kChABytes = kBM * kBK * 2, kChBBytes = kChBN * kBK * 2;
constexpr int kChStageBytes = kChABytes + kChBBytes;
constexpr int kChSmem = kChStages * kChStageBytes + 1024 + 512;

// Spin loads are relaxed: an ld.acquire.gpu per iteration compiles to an L1
// invalidate (CCTL.IVALL) each time -- it was the chain kernel's top stall
// and it evicted the epilogue's cached rows. One acq_rel fence after the
// value is seen gives the acquire.
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// job index of global tile t
__device__ __forceinline__ int chain_job_of(const ChainArgs& a, int t) {
  int j = 0;
#pragma unroll
  for (int k = 1; k < kChainMaxJobs; ++k)
    if (k < a.njobs && t >= a.job[k].first) j = k;
  return j;
}

// Spin (one thread) until every tile of row block mb of job j - 1 has been
// stored, then acquire.
__device__ __forceinline__ void chain_wait_dep(const ChainArgs& a, int j, int mb) {
  if (j == 0) return;
  const unsigned* c = a.ctr + (j - 1) * a.ctr_stride + mb;
  const unsigned need = static_cast<unsigned>(a.job[j - 1].tiles_n);
  while (ld_relaxed_u32(c) < need) {
  }
  fence_acq_rel_gpu();
}

// Epilogue of one 128-row x BN accumulator tile by one warp (lane quarter q,
// column half `half`); the accumulator is handed back by an arrive on the
// (possibly remote: CTA-pair leader) barrier at cluster address tempty_addr.
template <int BN, int EPI>
__device__ __forceinline__ void epi_tile(const GemmEpi& ep, int M, int m0, int n0, int q, int half,
                                         int lane, uint32_t acc, uint32_t tempty_addr) {
  const int c0 = half * (BN / 64), c1 = (half + 1) * (BN / 64);
  const int m = m0 + q * 32 + lane;
  const bool side2 = ep.out2 != nullptr && n0 >= ep.split_n;
  const int* rmap = side2 ? ep.row_map2 : ep.row_map;
  const int orow = m < M ? (rmap ? rmap[m] : m) : -1;
  float4 resA[8], resB[8];
  const bool acc_res = EPI == kEpiF32 && ep.accumulate;
  if (acc_res) {
    prefetch_residual(ep, orow, n0 + c0 * 32, resA);
    if (c0 + 1 < c1) prefetch_residual(ep, orow, n0 + (c0 + 1) * 32, resB);
  }
  float row_scale = 1.0f;
  if (ep.rms_ssq && m < M) {
    const float* sp = ep.rms_ssq + static_cast<size_t>(m) * ep.ld_rms;
    float ss = 0.0f;
    if ((ep.rms_parts & 3) == 0 && (ep.ld_rms & 3) == 0) {
      for (int k = 0; k < ep.rms_parts; k += 4) {
        const float4 q4 = *reinterpret_cast<const float4*>(sp + k);
        ss += q4.x;
        ss += q4.y;
        ss += q4.z;
        ss += q4.w;
      }
    } else {
      for (int k = 0; k < ep.rms_parts; ++k) ss += sp[k];
    }
    row_scale = 1.0f / sqrtf(ss * ep.rms_inv_d + 1e-5f);
  }
  auto chunk = [&](int c, float4 (&res)[8]) {
    uint32_t raw[32];
    tmem_ld_32x32(acc + c * 32, raw);
    tc_wait_ld();
    if (c + 1 == c1) {
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_addr);
    }
    epi_chunk<EPI>(ep, orow, n0 + c * 32, raw, res, row_scale, side2);
    if (acc_res && c + 2 < c1) prefetch_residual(ep, orow, n0 + (c + 2) * 32, res);
  };
#pragma unroll 1
  for (int c = c0; c < c1; c += 2) {
    chunk(c, resA);
    if (c + 1 < c1) chunk(c + 1, resB);
  }
}

__global__ void __launch_bounds__(kThreads, 1) gemm_chain_kernel(const __grid_constant__ ChainArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sa = smem;
  uint8_t* sb = smem + kChStages * kChABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kChStages * kChStageBytes);
  uint64_t* empty = full + kChStages;
  uint64_t* tfull = empty + kChStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* qfull = tempty + 2;
  uint64_t* qempty = qfull + kChQ;
  int* tq = reinterpret_cast<int*>(qempty + kChQ);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tq + kChQ);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned* tile_ctr = a.ctr + kChainMaxJobs * a.ctr_stride;
  unsigned* done_ctr = tile_ctr + 1;

  if (warp == 0 && lane == 0) {
    for (int j = 0; j < a.njobs; ++j) {
      tma_prefetch(&a.job[j].ta);
      tma_prefetch(&a.job[j].tb);
    }
    for (int s = 0; s < kChStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], kEpiWarps);
    }
    for (int i = 0; i < kChQ; ++i) {
      mbar_init(&qfull[i], 1);
      mbar_init(&qempty[i], 1 + kEpiWarps);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 2 * kChBN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // the tile counter is reset by the previous launch of this op at its very
  // end: it may only be touched after the PDL wait (back-to-back replays of
  // one chain op, e.g. pswa_gpu_bench_probe, would otherwise steal tiles)
  pdl_wait();
  pdl_trigger();
  int t_first = -1, npre = 0;
  if (warp == 0 && lane == 0) {
    t_first = static_cast<int>(atomicAdd(tile_ctr, 1u));
    if (t_first < a.total) {
      const ChainJobDev& J = a.job[chain_job_of(a, t_first)];
      const int u = t_first - J.first;
      npre = min(kChStages, J.K / kBK);
      for (int kb = 0; kb < npre; ++kb) {
        mbar_expect_tx(&full[kb], kChStageBytes);
        tma_load_2d(sb + kb * kChBBytes, &J.tb, &full[kb], kb * kBK, (u % J.tiles_n) * kChBN);
      }
    }
  }

  if (warp == 0) {
    if (lane == 0) {
      int g = 0;
      for (int i = 0;; ++i) {
        const int slot = i % kChQ;
        if (i >= kChQ) mbar_wait(&qempty[slot], ((i / kChQ) - 1) & 1);
        const int t = i == 0 ? t_first : static_cast<int>(atomicAdd(tile_ctr, 1u));
        const bool valid = t < a.total;
        tq[slot] = valid ? t : -1;
        mbar_arrive(&qfull[slot]);
        if (!valid) break;
        const int j = chain_job_of(a, t);
        const ChainJobDev& J = a.job[j];
        const int u = t - J.first, m0 = (u / J.tiles_n) * kBM, n0 = (u % J.tiles_n) * kChBN;
        const int kblocks = J.K / kBK;
        for (int kb = 0; kb < kblocks; ++kb, ++g) {
          const int s = g % kChStages, round = g / kChStages;
          if (g < npre) {  // first tile: B already requested
            if (kb == 0) {
              chain_wait_dep(a, j, m0 / kBM);
              fence_proxy_async_global();
            }
            tma_load_2d(sa + s * kChABytes, &J.ta, &full[s], kb * kBK, m0);
            continue;
          }
          if (round > 0) mbar_wait(&empty[s], (round - 1) & 1);
          mbar_expect_tx(&full[s], kChStageBytes);
          tma_load_2d(sb + s * kChBBytes, &J.tb, &full[s], kb * kBK, n0);
          if (kb == 0) {  // weights first, then wait for the rows this tile reads
            chain_wait_dep(a, j, m0 / kBM);
            fence_proxy_async_global();
          }
          tma_load_2d(sa + s * kChABytes, &J.ta, &full[s], kb * kBK, m0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_f16_f32(kBM, kChBN);
      int g = 0;
      for (int i = 0;; ++i) {
        const int slot = i % kChQ;
        mbar_wait(&qfull[slot], (i / kChQ) & 1);
        const int t = tq[slot];
        mbar_arrive(&qempty[slot]);
        if (t < 0) break;
        const ChainJobDev& J = a.job[chain_job_of(a, t)];
        const int buf = i & 1, use = i >> 1;
        if (use > 0) mbar_wait(&tempty[buf], (use - 1) & 1);
        tc_fence_after();
        const uint32_t acc = tmem + buf * kChBN;
        const int kblocks = J.K / kBK;
        for (int kb = 0; kb < kblocks; ++kb, ++g) {
          const int s = g % kChStages;
          mbar_wait(&full[s], (g / kChStages) & 1);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sa + s * kChABytes);
          const uint32_t b_base = smem_u32(sb + s * kChBBytes);
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk)
            tc_mma_f16(acc, umma_desc_k_sw128(a_base + kk * 32), umma_desc_k_sw128(b_base + kk * 32), idesc,
                       (kb | kk) != 0 ? 1u : 0u);
          tc_commit(&empty[s]);
        }
        tc_commit(&tfull[buf]);
      }
    }
  } else {
    const int ew = warp - 2, q = warp & 3, half = ew >> 2;
    for (int i = 0;; ++i) {
      const int slot = i % kChQ;
      mbar_wait(&qfull[slot], (i / kChQ) & 1);
      const int t = tq[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&qempty[slot]);
      if (t < 0) break;
      const int j = chain_job_of(a, t);
      const ChainJobDev& J = a.job[j];
      const int u = t - J.first, m0 = (u / J.tiles_n) * kBM, n0 = (u % J.tiles_n) * kChBN;
      const int buf = i & 1, use = i >> 1;
      // the epilogue reads the previous job's outputs too (residual rows, the
      // folded norm's sums of squares): same dependency as the A operand
      // one lane acquires; the warp barrier orders the other lanes' reads after it
      if (lane == 0) chain_wait_dep(a, j, m0 / kBM);
      __syncwarp();
      mbar_wait(&tfull[buf], use & 1);
      tc_fence_after();
      const uint32_t acc = tmem + buf * kChBN + (static_cast<uint32_t>(q * 32) << 16);
      const uint32_t te = smem_u32(&tempty[buf]);
      switch (J.kind) {
        case kEpiF16: epi_tile<kChBN, kEpiF16>(J.ep, J.M, m0, n0, q, half, lane, acc, te); break;
        case kEpiF32: epi_tile<kChBN, kEpiF32>(J.ep, J.M, m0, n0, q, half, lane, acc, te); break;
        case kEpiSwiGLU: epi_tile<kChBN, kEpiSwiGLU>(J.ep, J.M, m0, n0, q, half, lane, acc, te); break;
        default: epi_tile<kChBN, kEpiHead>(J.ep, J.M, m0, n0, q, half, lane, acc, te); break;
      }
      // every epilogue warp's stores of this tile, then one release increment
      named_bar_sync(1, 32 * kEpiWarps);
      if (ew == 0 && lane == 0) {
        __threadfence();
        atomicAdd(a.ctr + j * a.ctr_stride + m0 / kBM, 1u);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_free(tmem, 2 * kChBN);
  }
  if (threadIdx.x == 0) {  // the last CTA out resets the counters for the next replay
    __threadfence();
    if (atomicAdd(done_ctr, 1u) == gridDim.x - 1) {
      for (int k = 0; k < kChainMaxJobs * a.ctr_stride; ++k) a.ctr[k] = 0u;
      *tile_ctr = 0u;
      *done_ctr = 0u;
      __threadfence();
    }
  }
}

// --------------------------------------------------- CTA-pair GEMM (2SM) --
// For the large-M context GEMMs (M = 32640): a cluster of 2 CTAs computes a
// 256 x 256 tile with tcgen05.mma.cta_group::2 issued by the pair leader.
// Each CTA stages only its own 128 rows of A and its own 128 rows (N half)
// of B per K block, 32 KB instead of the 48 KB a single-SM 128 x 256 tile
// needs for the same MMA work: the per-SM operand stream, which bounds the
// single-SM kernel (~74% MMA-paced), drops below the MMA time. Each CTA's
// TMEM holds its own 128 rows x 256 columns; the epilogue is the single-SM
// one. Same K order (ascending 64-wide blocks): bitwise equal results.
constexpr int kPBN = 256;
constexpr int kPStages = 6;
constexpr int kPABytes = kBM * kBK * 2, kPBBytes = (kPBN / 2) * kBK * 2;
constexpr int kPStageBytes = kPABytes + kPBBytes;
constexpr int kPSmem = kPStages * kPStageBytes + 1024 + 256;

template <int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_pair_kernel(const __grid_constant__ CUtensorMap tma, const __grid_constant__ CUtensorMap tmb, int M,
                     int K, int tiles_mp, int tiles_n, const __grid_constant__ GemmEpi ep) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sa = smem;
  uint8_t* sb = smem + kPStages * kPABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kPStages * kPStageBytes);
  uint64_t* empty = full + kPStages;
  uint64_t* tfull = empty + kPStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int kblocks = K / kBK;
  const int n_units = tiles_mp * tiles_n;
  const int unit0 = blockIdx.x / 2, unit_step = gridDim.x / 2;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tma);
    tma_prefetch(&tmb);
    for (int s = 0; s < kPStages; ++s) {
      mbar_init(&full[s], 1);   // leader: one arrive.expect_tx for both CTAs' bytes
      mbar_init(&empty[s], 1);  // the leader's multicast commit
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);              // multicast commit
      mbar_init(&tempty[b], 2 * kEpiWarps);  // leader: both CTAs' epilogue warps
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, 2 * kPBN);
  tc_fence_before();
  cluster_sync();  // barriers of both CTAs initialised, TMEM allocated
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      int g = 0;
      for (int u = unit0; u < n_units; u += unit_step) {
        const int m0 = (u / tiles_n) * 2 * kBM + rank * kBM, n0 = (u % tiles_n) * kPBN + rank * (kPBN / 2);
        for (int kb = 0; kb < kblocks; ++kb, ++g) {
          const int s = g % kPStages, round = g / kPStages;
          if (round > 0) mbar_wait(&empty[s], (round - 1) & 1);
          const uint32_t fb = mapa_shared(smem_u32(&full[s]), 0);
          if (leader) mbar_expect_tx(&full[s], 2 * kPStageBytes);
          tma_load_2d_pair(sa + s * kPABytes, &tma, fb, kb * kBK, m0);
          tma_load_2d_pair(sb + s * kPBBytes, &tmb, fb, kb * kBK, n0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      constexpr uint32_t idesc = umma_idesc_f16_f32(2 * kBM, kPBN);
      int g = 0, it = 0;
      for (int u = unit0; u < n_units; u += unit_step, ++it) {
        const int buf = it & 1, use = it >> 1;
        if (use > 0) mbar_wait(&tempty[buf], (use - 1) & 1);
        tc_fence_after();
        const uint32_t acc = tmem + buf * kPBN;
        for (int kb = 0; kb < kblocks; ++kb, ++g) {
          const int s = g % kPStages;
          mbar_wait(&full[s], (g / kPStages) & 1);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sa + s * kPABytes);
          const uint32_t b_base = smem_u32(sb + s * kPBBytes);
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk)
            tc_mma_f16_pair(acc, umma_desc_k_sw128(a_base + kk * 32), umma_desc_k_sw128(b_base + kk * 32), idesc,
                            (kb | kk) != 0 ? 1u : 0u);
          tc_commit_pair(&empty[s]);
        }
        tc_commit_pair(&tfull[buf]);
      }
    }
  } else {
    const int ew = warp - 2, q = warp & 3, half = ew >> 2;
    int it = 0;
    for (int u = unit0; u < n_units; u += unit_step, ++it) {
      const int buf = it & 1, use = it >> 1;
      const int m0 = (u / tiles_n) * 2 * kBM + rank * kBM, n0 = (u % tiles_n) * kPBN;
      mbar_wait(&tfull[buf], use & 1);
      tc_fence_after();
      const uint32_t acc = tmem + buf * kPBN + (static_cast<uint32_t>(q * 32) << 16);
      epi_tile<kPBN, EPI>(ep, M, m0, n0, q, half, lane, acc, mapa_shared(smem_u32(&tempty[buf]), 0));
    }
  }
  tc_fence_before();
  cluster_sync();  // no commit / remote arrive can still target this CTA
  if (warp == 1) {
    tc_fence_after();
    tmem_free_pair(tmem, 2 * kPBN);
  }
}

// ------------------------------------------------------- split-K pairs --
// The M = 2040 step GEMMs are paced per SM by the tensor pipe's per-
// instruction floor (a K = 16 tcgen05.mma costs ~92 cycles for any N <= 128,
// tools/umma_probe.cu) and by the operand stream into shared memory, not by
// the chip. A cluster of two CTAs therefore splits one 128 x 128 output tile
// along K: rank r accumulates k-blocks [r h, min(KB, (r + 1) h)), h =
// ceil(KB / 2), in its own TMEM (half the MMAs and half the operand bytes of
// a CTA each). Rank r owns output columns [64 r, 64 r + 64): it sends its
// partial sums of the other 64 columns into the peer's receive buffer
// (st.shared::cluster, 16 B per lane, chunk-swizzled rows), and after one
// cluster barrier adds the peer's partial of its own columns and runs the
// usual epilogue (8 warps, one 32 x 32 chunk each). Every output is
// fl(P0 + P1) with P_r the ascending sum over rank r's k-blocks: a function
// of K alone (fp32 addition commutes), so results are bitwise identical for
// any M and schedule; the engine requests it per layer (GemmEpi::split_k),
// so an encoder and a decoder program agree.
constexpr int kSBN = 128;
constexpr int kSStages = 5;
constexpr int kSABytes = kBM * kBK * 2, kSBBytes = kSBN * kBK * 2;
constexpr int kSStageBytes = kSABytes + kSBBytes;
constexpr int kSRecvBytes = kBM * 64 * 4;  // the peer's partials of this CTA's 64 columns
constexpr int kSSmem = kSStages * kSStageBytes + kSRecvBytes + 1024 + 256;

// receive buffer: [128 rows][64 fp32] (256 B rows), 16 B piece j of column
// half `hsel` of row r at hsel * 128 + ((j ^ (r & 7)) << 4): the 32 lanes
// (one row each) of a warp write / read conflict-free
__device__ __forceinline__ uint32_t recv_off(int row, int hsel, int j) {
  return static_cast<uint32_t>(row * 256 + hsel * 128 + ((j ^ (row & 7)) << 4));
}

template <int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_splitk_kernel(const __grid_constant__ CUtensorMap tma, const __grid_constant__ CUtensorMap tmb, int M,
                       int K, int tiles_n, const __grid_constant__ GemmEpi ep) {
  constexpr int S = kSStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sa = smem;
  uint8_t* sb = smem + S * kSABytes;
  uint8_t* recv = smem + S * kSStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(recv + kSRecvBytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank(), peer = rank ^ 1u;
  const int tile = blockIdx.x >> 1;
  const int m0 = (tile / tiles_n) * kBM, n0 = (tile % tiles_n) * kSBN;
  const int KB = K / kBK, h = (KB + 1) / 2;
  const int kb0 = static_cast<int>(rank) * h, nkb = min(KB, kb0 + h) - kb0;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tma);
    tma_prefetch(&tmb);
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, kSBN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // the peer must have started before its shared memory is written: arrive
  // now, wait right before the partial-sum exchange
  cluster_arrive_relaxed();
  const uint32_t tmem = *tmem_slot;
  // weights (B) of the first stages requested before the PDL wait
  int npre = 0;
  if (warp == 0 && lane == 0) {
    npre = min(S, nkb);
    for (int i = 0; i < npre; ++i) {
      mbar_expect_tx(&full[i], kSStageBytes);
      tma_load_2d(sb + i * kSBBytes, &tmb, &full[i], (kb0 + i) * kBK, n0);
    }
  }
  pdl_wait();
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < nkb; ++i) {
        const int s = i % S, round = i / S, kb = kb0 + i;
        if (i < npre) {
          tma_load_2d(sa + s * kSABytes, &tma, &full[s], kb * kBK, m0);
          continue;
        }
        if (round > 0) mbar_wait(&empty[s], (round - 1) & 1);
        mbar_expect_tx(&full[s], kSStageBytes);
        tma_load_2d(sa + s * kSABytes, &tma, &full[s], kb * kBK, m0);
        tma_load_2d(sb + s * kSBBytes, &tmb, &full[s], kb * kBK, n0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_f16_f32(kBM, kSBN);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % S;
        mbar_wait(&full[s], (i / S) & 1);
        tc_fence_after();
        const uint32_t a_base = smem_u32(sa + s * kSABytes);
        const uint32_t b_base = smem_u32(sb + s * kSBBytes);
#pragma unroll
        for (int kk = 0; kk < kBK / 16; ++kk)
          tc_mma_f16(tmem, umma_desc_k_sw128(a_base + kk * 32), umma_desc_k_sw128(b_base + kk * 32), idesc,
                     (i | kk) != 0 ? 1u : 0u);
        tc_commit(&empty[s]);
      }
      tc_commit(tfull);
    }
  }
  const int ew = warp - 2, q = warp & 3, hsel = ew >> 2;
  const int row = q * 32 + lane, m = m0 + row;
  const int orow = m < M ? (ep.row_map ? ep.row_map[m] : m) : -1;
  const int c_own = 2 * static_cast<int>(rank) + hsel, c_exp = 2 * static_cast<int>(peer) + hsel;
  uint32_t own[32];
  float4 res[8];
  float row_scale = 1.0f;
  if (warp >= 2) {
    if (EPI == kEpiF32 && ep.accumulate) prefetch_residual(ep, orow, n0 + c_own * 32, res);
    if (ep.rms_ssq && m < M) {
      const float* sp = ep.rms_ssq + static_cast<size_t>(m) * ep.ld_rms;
      float ss = 0.0f;
      for (int k = 0; k < ep.rms_parts; ++k) ss += sp[k];
      row_scale = 1.0f / sqrtf(ss * ep.rms_inv_d + 1e-5f);
    }
    mbar_wait(tfull, 0);
    tc_fence_after();
    const uint32_t acc = tmem + (static_cast<uint32_t>(q * 32) << 16);
    uint32_t xp[32];
    tmem_ld_32x32(acc + c_exp * 32, xp);
    tmem_ld_32x32(acc + c_own * 32, own);
    tc_wait_ld();
    cluster_wait();  // (the peer has started)
    const uint32_t rbase = mapa_shared(smem_u32(recv), peer);
#pragma unroll
    for (int j = 0; j < 8; ++j)
      st_cluster_v4(rbase + recv_off(row, hsel, j), make_uint4(xp[4 * j], xp[4 * j + 1], xp[4 * j + 2], xp[4 * j + 3]));
  }
  if (warp < 2) cluster_wait();  // (producer / MMA warps: the start barrier)
  // the peer's partials of this CTA's columns have landed (release / acquire)
  cluster_sync();
  if (warp >= 2) {
    const uint32_t rl = smem_u32(recv);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint4 v;
      asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                   : "r"(rl + recv_off(row, hsel, j)));
      own[4 * j] = __float_as_uint(__uint_as_float(own[4 * j]) + __uint_as_float(v.x));
      own[4 * j + 1] = __float_as_uint(__uint_as_float(own[4 * j + 1]) + __uint_as_float(v.y));
      own[4 * j + 2] = __float_as_uint(__uint_as_float(own[4 * j + 2]) + __uint_as_float(v.z));
      own[4 * j + 3] = __float_as_uint(__uint_as_float(own[4 * j + 3]) + __uint_as_float(v.w));
    }
    // coalesced stores staged in the (now idle) A ring, 4 KB per warp
    epi_chunk<EPI>(ep, orow, n0 + c_own * 32, own, res, row_scale, false,
                   ep.coalesce ? smem_u32(sa + ew * 4096) : 0u);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_free(tmem, kSBN);
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

// fp32 output map for the TMA-stored epilogue: 32 x 32 boxes, 128 B rows
void make_tmap_f32_out(CUtensorMap* m, const float* base, int ld, int rows, int cols) {
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 4};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw CudaError("cuTensorMapEncodeTiled (fp32 out) failed (code " + std::to_string(int(r)) + ")");
}

using EncodeIm2colFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeIm2colFn encode_im2col_fn() {
  static EncodeIm2colFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    PSWA_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p)
      throw CudaError("cuTensorMapEncodeIm2col entry point unavailable");
    fn = reinterpret_cast<EncodeIm2colFn>(p);
  });
  return fn;
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
    PSWA_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<BN, EPI, 1>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, GemmCfg<BN>::smem_for(EPI)));
    if constexpr (GemmCfg<BN>::kBSplit == 1)
      PSWA_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<BN, EPI, 2>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, GemmCfg<BN>::smem_for(EPI)));
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

template <int BN, int EPI>
void launch_epi(const GemmPlan& p, cudaStream_t st) {
  const int tiles_m = (p.M + kBM - 1) / kBM;
  const int tiles = tiles_m * (p.N / BN);
  const int smem = GemmCfg<BN>::smem_for(EPI);
  if (p.cluster == 2) {
    if constexpr (GemmCfg<BN>::kBSplit == 1) {
      const int units = (tiles_m + 1) / 2 * (p.N / BN);
      const int clusters = units < sm_count() / 2 ? units : sm_count() / 2;
      launch_kc(gemm_tc_kernel<BN, EPI, 2>, dim3(2 * clusters), dim3(kThreads), smem, st, 2u, p.ta,
                p.tb, p.to, p.M, p.K, tiles_m, tiles, p.epi);
    } else {
      throw std::invalid_argument("gemm: BN 352 has no cluster variant");
    }
  } else {
    const int grid = tiles < sm_count() ? tiles : sm_count();
    launch_k(gemm_tc_kernel<BN, EPI, 1>, dim3(grid), dim3(kThreads), smem, st, p.ta, p.tb, p.to, p.M,
             p.K, tiles_m, tiles, p.epi);
  }
}

template <int EPI>
void launch_splitk(const GemmPlan& p, cudaStream_t st) {
  const int tiles_n = p.N / kSBN, tiles = ((p.M + kBM - 1) / kBM) * tiles_n;
  launch_kc(gemm_splitk_kernel<EPI>, dim3(2 * tiles), dim3(kThreads), kSSmem, st, 2u, p.ta, p.tb, p.M, p.K,
            tiles_n, p.epi);
}

template <int BN>
void launch(const GemmPlan& p, int kind, cudaStream_t st) {
  switch (kind) {
    case kEpiF16: launch_epi<BN, kEpiF16>(p, st); break;
    case kEpiF32: launch_epi<BN, kEpiF32>(p, st); break;
    case kEpiSwiGLU: launch_epi<BN, kEpiSwiGLU>(p, st); break;
    default: launch_epi<BN, kEpiHead>(p, st); break;
  }
}

}  // namespace

void make_kv_tmap(CUtensorMap* m, const __half* kv, int ld, int W, int H, int slots,
                  long slot_stride_rows, int box_w, int box_h) {
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(ld), static_cast<cuuint64_t>(W),
                        static_cast<cuuint64_t>(H), static_cast<cuuint64_t>(slots)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(ld) * 2, static_cast<cuuint64_t>(W) * ld * 2,
                           static_cast<cuuint64_t>(slot_stride_rows) * ld * 2};
  cuuint32_t box[4] = {32, static_cast<cuuint32_t>(box_w), static_cast<cuuint32_t>(box_h), 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, const_cast<__half*>(kv), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw CudaError("cuTensorMapEncodeTiled (kv) failed (code " + std::to_string(int(r)) + ")");
}

unsigned long long* trace_buffer() {
  static unsigned long long* buf = [] {
    unsigned long long* b = nullptr;
    const size_t bytes = sizeof(unsigned long long) * kGemmTraceSlots * 1024;
    PSWA_CUDA(cudaMalloc(&b, bytes));
    PSWA_CUDA(cudaMemset(b, 0, bytes));
    return b;
  }();
  return buf;
}

void gemm_set_experiment(int flags) {
#ifdef PSWA_GEMM_TRACE_BUILD
  PSWA_CUDA(cudaDeviceSynchronize());
  PSWA_CUDA(cudaMemcpyToSymbol(g_gemm_exp, &flags, sizeof(int)));
#else
  (void)flags;
#endif
}

bool gemm_trace_read(unsigned long long* out, int n) {
  if (!std::getenv("PSWA_GEMM_TRACE")) return false;
  n = std::min(n, kGemmTraceSlots * 1024);
  PSWA_CUDA(cudaDeviceSynchronize());
  PSWA_CUDA(cudaMemcpy(out, trace_buffer(), sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost));
  PSWA_CUDA(cudaMemset(trace_buffer(), 0, sizeof(unsigned long long) * kGemmTraceSlots * 1024));
  return true;
}

void gemm_plan(GemmPlan* p, const __half* A, int lda, int M, const __half* B, int ldb, int N,
               int K, const GemmEpi& epi, int force_bn) {
  if (K % kBK != 0 || N % 64 != 0 || lda % 8 != 0 || ldb % 8 != 0 || M <= 0)
    throw std::invalid_argument("gemm_plan: unsupported shape (K%64, N%64, ld%8)");
  // force_bn = -1: the CTA-pair kernel (256 x 256 tiles, N % 256 == 0)
  const bool force_pair = force_bn < 0;
  int bn = force_pair ? 0 : force_bn;
  if (bn == 0) {
    // BN=256 once its tiles cover half the SMs (one wave of wide tiles beats
    // ~2 waves of BN=128 for the M = 2040 Q|K|V and gate|up GEMMs: 7.26 vs
    // 7.39 ms / frame; thresholds of 48-96 tiles measured alike), else
    // BN=128 when its tiles fill the SMs, else BN=64 (the N = 512 step
    // GEMMs: BN=128 there measured 7.47+ ms)
    const int mt = (M + kBM - 1) / kBM, sms = sm_count();
    // one wave of wider / narrower tiles where 128 x 256 would not fill
    // the SMs in whole waves (tools/gemm_bn_probe.py, M = 2040): gate|up
    // N = 2816 as 128 tiles of 352 (176 tiles of 256 take 1.2 waves;
    // 8.70 vs 8.88 us), Q|K|V N = 1536 as 128 tiles of 192 (96 tiles of
    // 256 leave 52 SMs idle; 6.66 vs 7.22 us). PSWA_GEMM_NO_WIDE=1: off.
    static const bool no_wide = std::getenv("PSWA_GEMM_NO_WIDE") != nullptr;
    static const int big_f32_bn = std::getenv("PSWA_GEMM_BIG_F32_BN") ? std::atoi(std::getenv("PSWA_GEMM_BIG_F32_BN")) : 0;
    if (big_f32_bn && epi.out_f32 && epi.act == kActNone && M >= 16384 && N % big_f32_bn == 0)
      bn = big_f32_bn;  // (experiment: residual GEMMs of the context stack)
    else if (!no_wide && N % 352 == 0 && mt * (N / 256) > sms && mt * (N / 352) <= sms)
      bn = 352;
    else if (!no_wide && N % 192 == 0 && N % 256 == 0 && mt * (N / 256) < sms && mt * (N / 192) <= sms &&
             mt * (N / 256) >= sms / 2)
      bn = 192;
    else if (N % 256 == 0 && mt * (N / 256) >= sms / 2)
      bn = 256;
    else if (N % 128 == 0 && mt * (N / 128) >= sms)
      bn = 128;
    else
      bn = 64;
  }
  if (N % bn != 0 || (bn != 64 && bn != 128 && bn != 192 && bn != 256 && bn != 352))
    throw std::invalid_argument("gemm_plan: bad BN");
  if (epi.out2 && (epi.out_f32 || epi.act != kActNone || epi.split_n % (bn == 192 ? 32 : bn) != 0))
    throw std::invalid_argument("gemm_plan: split output needs fp16 out and split_n % BN == 0");
  p->M = M;
  p->N = N;
  p->K = K;
  p->BN = bn;
  p->epi = epi;
  {  // 256-bit epilogue accesses when every row segment is 32 B aligned
    const size_t es = epi.out_f32 || epi.act == kActHead ? 4 : 2;
    auto al = [](const void* ptr, size_t ld_bytes) {
      return ptr == nullptr || (reinterpret_cast<uintptr_t>(ptr) % 32 == 0 && ld_bytes % 32 == 0);
    };
    p->epi.v8 = al(epi.out, epi.ld_out * es) && al(epi.x16_out, static_cast<size_t>(epi.ld_x16) * 2) &&
                        al(epi.out2, static_cast<size_t>(epi.ld_out2) * 2) &&
                        !std::getenv("PSWA_GEMM_NO_V8")
                    ? 1
                    : 0;
  }
  // coalesced epilogue stores through the per-warp smem stage (gemm_tc_kernel)
  static const bool no_coalesce = std::getenv("PSWA_GEMM_NO_COALESCE") != nullptr;
  p->epi.coalesce = no_coalesce ? 0 : 1;
  // CTA pairs sharing B through TMA multicast: correct and available, but
  // measured neutral-to-slower on B200 (the L2 already dedups concurrent B
  // reads; 10.56 vs 10.44 ms / frame; on the M = 2040 step GEMMs alone
  // 7.80 vs 7.59 ms / frame), so opt-in via PSWA_GEMM_CLUSTER=1.
  static const bool use_cluster = std::getenv("PSWA_GEMM_CLUSTER") != nullptr;
  if (std::getenv("PSWA_GEMM_TRACE")) p->epi.trace = trace_buffer();
  p->cluster = (use_cluster && M > kBM && bn <= 256) ? 2 : 1;
  // CTA-pair tiles (cta_group::2) for the large context GEMMs: correct and
  // bitwise equal to the single-SM kernel (test_pair_gemm_bitwise_equals_
  // single_sm) but measured no faster on B200 -- the context SwiGLU GEMM took
  // 90 vs 84.5 us and the frame 7.38 vs 7.25 ms: these tiles are paced by the
  // epilogue (TMEM reads, SiLU, stores), not the per-SM operand stream the
  // pair halves. Opt-in: PSWA_GEMM_PAIR=1, or force_bn = -1 per call.
  // PSWA_GEMM_PAIR_KINDS=<mask>: pairs for the epilogue kinds in the mask
  // only (1 fp16 out, 2 fp32 residual, 4 SwiGLU, 8 head)
  static const int pair_kinds = std::getenv("PSWA_GEMM_PAIR")         ? 15
                                : std::getenv("PSWA_GEMM_PAIR_KINDS") ? std::atoi(std::getenv("PSWA_GEMM_PAIR_KINDS"))
                                                                      : 0;
  const bool use_pair = (pair_kinds >> epi_kind(epi)) & 1;
  const int pair_units = ((M + 2 * kBM - 1) / (2 * kBM)) * (N / kPBN);
  p->pair = N % kPBN == 0 &&
            (force_pair || (use_pair && force_bn == 0 && M >= 16384 && pair_units >= sm_count()));
  if (p->pair) {
    bn = kPBN;
    p->BN = bn;
    p->cluster = 1;
  }
  // split-K CTA pairs (gemm_splitk_kernel), on request: fp32 / fp16 outputs
  static const bool no_splitk = std::getenv("PSWA_GEMM_NO_SPLITK") != nullptr;
  const int kind0 = epi_kind(epi);
  p->splitk = !p->pair && !no_splitk && epi.split_k && force_bn == 0 && epi.out2 == nullptr &&
              (kind0 == kEpiF32 || kind0 == kEpiF16) && N % kSBN == 0 && K / kBK >= 2;
  if (p->splitk) {
    bn = kSBN;
    p->BN = bn;
    p->cluster = 1;
  }
  make_tmap(&p->ta, A, lda, M, K, kBM);
  make_tmap(&p->tb, B, ldb, N, K, p->pair ? kPBN / 2 : bn > 256 ? bn / 2 : bn / p->cluster);
  if (p->splitk) {
    static std::once_flag once_sk;
    std::call_once(once_sk, [] {
      PSWA_CUDA(cudaFuncSetAttribute(gemm_splitk_kernel<kEpiF32>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSSmem));
      PSWA_CUDA(cudaFuncSetAttribute(gemm_splitk_kernel<kEpiF16>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSSmem));
    });
    return;
  }
  if (p->pair) {
    static std::once_flag once_pair;
    std::call_once(once_pair, [] {
      PSWA_CUDA(cudaFuncSetAttribute(gemm_pair_kernel<kEpiF16>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPSmem));
      PSWA_CUDA(cudaFuncSetAttribute(gemm_pair_kernel<kEpiF32>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPSmem));
      PSWA_CUDA(cudaFuncSetAttribute(gemm_pair_kernel<kEpiSwiGLU>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPSmem));
      PSWA_CUDA(cudaFuncSetAttribute(gemm_pair_kernel<kEpiHead>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPSmem));
    });
    return;
  }
  const int kind = epi_kind(epi);
  // fp32 outputs with contiguous rows leave the epilogue stage by TMA, on
  // request (PSWA_GEMM_TMA_STORE=1): measured neutral on B200 (context
  // out-projection 53.0 -> 50.4 us, context down 66.4 -> 68.1 us, frame
  // 6.89 vs 6.92 ms); the epilogue is latency-bound, not store-issue-bound
  static const bool tma_store = std::getenv("PSWA_GEMM_TMA_STORE") != nullptr;
  p->tma_store = tma_store && kind == kEpiF32 && p->epi.coalesce && epi.row_map == nullptr &&
                 epi.out != nullptr && reinterpret_cast<uintptr_t>(epi.out) % 16 == 0 && (epi.ld_out * 4) % 16 == 0;
  p->epi.tma_store = p->tma_store ? 1 : 0;
  // residual rows bulk-prefetched into L2 at tile start (16 B aligned
  // segments), on request (PSWA_GEMM_L2_PREFETCH=1): measured neutral
  // (context out-projection 53.3 -> 52.0 us, down 70.9 -> 71.7 us)
  static const bool l2_prefetch = std::getenv("PSWA_GEMM_L2_PREFETCH") != nullptr;
  p->epi.l2_prefetch = l2_prefetch && kind == kEpiF32 && epi.accumulate && epi.out != nullptr &&
                       reinterpret_cast<uintptr_t>(epi.out) % 16 == 0 && (epi.ld_out * 4) % 16 == 0 &&
                       (std::min(N, epi.n_store) % 4) == 0;
  if (p->tma_store)
    make_tmap_f32_out(&p->to, static_cast<const float*>(epi.out), epi.ld_out, M, std::min(N, epi.n_store));
  else
    p->to = p->ta;  // (unused)
  if (bn == 64) prep<64>(kind);
  if (bn == 128) prep<128>(kind);
  if (bn == 192) prep<192>(kind);
  if (bn == 256) prep<256>(kind);
  if (bn == 352) prep<352>(kind);
}

void gemm_plan_conv3x3(GemmPlan* p, const __half* x, int h, int w, int c, const __half* B, int ldb, int N,
                       const GemmEpi& epi) {
  if (c % kBK != 0 || h < 1 || w < 1 || reinterpret_cast<uintptr_t>(x) % 16 != 0)
    throw std::invalid_argument("gemm_plan_conv3x3: channels % 64, 16 B aligned NHWC input");
  // plan as a GEMM over [h*w][9c] (tile width, epilogue, B map), then swap
  // A's map for the im2col one over the image itself
  GemmEpi e = epi;
  e.conv_w = w;
  e.conv_cb = c / kBK;
  gemm_plan(p, x, 9 * c, h * w, B, ldb, N, 9 * c, e);  // (A's 2D map is replaced below)
  if (p->pair || p->splitk || p->cluster != 1)
    throw std::invalid_argument("gemm_plan_conv3x3: single-CTA tiles only");
  // dims (c, w, h, n = 1); 3x3 taps at offsets 0..2 from the lower corner
  // (-1, -1): padding 1 on every side, output grid = input grid
  const cuuint64_t dims[4] = {static_cast<cuuint64_t>(c), static_cast<cuuint64_t>(w), static_cast<cuuint64_t>(h), 1};
  const cuuint64_t strides[3] = {static_cast<cuuint64_t>(c) * 2, static_cast<cuuint64_t>(w) * c * 2,
                                 static_cast<cuuint64_t>(h) * w * c * 2};
  const int lower[2] = {-1, -1}, upper[2] = {-1, -1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = encode_im2col_fn()(&p->ta, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, const_cast<__half*>(x), dims, strides,
                                  lower, upper, static_cast<cuuint32_t>(kBK), static_cast<cuuint32_t>(kBM), estr,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw CudaError("cuTensorMapEncodeIm2col failed (code " + std::to_string(int(r)) + ")");
}

int gemm_chain_counter_words(int M) { return kChainMaxJobs * ((M + kBM - 1) / kBM) + 2; }

void gemm_chain_add(GemmChainPlan* c, const __half* A, int lda, int M, const __half* B, int ldb, int N,
                    int K, const GemmEpi& epi) {
  if (c->njobs >= kChainMaxJobs) throw std::invalid_argument("gemm_chain_add: too many jobs");
  if (N % kChBN != 0) throw std::invalid_argument("gemm_chain_add: N % 128 != 0");
  if (c->njobs > 0 && c->job[0].M != M) throw std::invalid_argument("gemm_chain_add: M differs");
  if (epi.act == kActTanhHalf) throw std::invalid_argument("gemm_chain_add: unsupported activation");
  gemm_plan(&c->job[c->njobs], A, lda, M, B, ldb, N, K, epi, kChBN);
  c->ctr_stride = (M + kBM - 1) / kBM;
  ++c->njobs;
  static std::once_flag once;
  std::call_once(once, [] {
    PSWA_CUDA(cudaFuncSetAttribute(gemm_chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kChSmem));
  });
}

void gemm_chain_run(const GemmChainPlan& c, cudaStream_t stream) {
  if (c.njobs == 0) return;
  if (!c.counters) throw std::invalid_argument("gemm_chain_run: no counters");
  ChainArgs a{};
  int first = 0;
  for (int j = 0; j < c.njobs; ++j) {
    const GemmPlan& p = c.job[j];
    ChainJobDev& d = a.job[j];
    d.ta = p.ta;
    d.tb = p.tb;
    d.ep = p.epi;
    d.M = p.M;
    d.K = p.K;
    d.tiles_m = (p.M + kBM - 1) / kBM;
    d.tiles_n = p.N / kChBN;
    d.kind = epi_kind(p.epi);
    d.first = first;
    first += d.tiles_m * d.tiles_n;
  }
  a.njobs = c.njobs;
  a.total = first;
  a.ctr_stride = c.ctr_stride;
  a.ctr = c.counters;
  const int grid = first < sm_count() ? first : sm_count();
  launch_k(gemm_chain_kernel, dim3(grid), dim3(kThreads), kChSmem, stream, a);
  PSWA_LAUNCH_CHECK();
}

void gemm_run(const GemmPlan& p, cudaStream_t stream) {
  const int kind = epi_kind(p.epi);
  if (p.pair) {
    const int tiles_mp = (p.M + 2 * kBM - 1) / (2 * kBM), tiles_n = p.N / kPBN;
    const int units = tiles_mp * tiles_n, clusters = std::min(units, sm_count() / 2);
    switch (kind) {
      case kEpiF16: launch_kc(gemm_pair_kernel<kEpiF16>, dim3(2 * clusters), dim3(kThreads), kPSmem, stream, 2u, p.ta, p.tb, p.M, p.K, tiles_mp, tiles_n, p.epi); break;
      case kEpiF32: launch_kc(gemm_pair_kernel<kEpiF32>, dim3(2 * clusters), dim3(kThreads), kPSmem, stream, 2u, p.ta, p.tb, p.M, p.K, tiles_mp, tiles_n, p.epi); break;
      case kEpiSwiGLU: launch_kc(gemm_pair_kernel<kEpiSwiGLU>, dim3(2 * clusters), dim3(kThreads), kPSmem, stream, 2u, p.ta, p.tb, p.M, p.K, tiles_mp, tiles_n, p.epi); break;
      default: launch_kc(gemm_pair_kernel<kEpiHead>, dim3(2 * clusters), dim3(kThreads), kPSmem, stream, 2u, p.ta, p.tb, p.M, p.K, tiles_mp, tiles_n, p.epi); break;
    }
    PSWA_LAUNCH_CHECK();
    return;
  }
  if (p.splitk) {
    if (kind == kEpiF32)
      launch_splitk<kEpiF32>(p, stream);
    else
      launch_splitk<kEpiF16>(p, stream);
    PSWA_LAUNCH_CHECK();
    return;
  }
  switch (p.BN) {
    case 64: launch<64>(p, kind, stream); break;
    case 128: launch<128>(p, kind, stream); break;
    case 192: launch<192>(p, kind, stream); break;
    case 256: launch<256>(p, kind, stream); break;
    case 352: launch<352>(p, kind, stream); break;
    default: throw std::invalid_argument("gemm_run: bad BN");
  }
  PSWA_LAUNCH_CHECK();
}

}  // namespace pswa_dev
