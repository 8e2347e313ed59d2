// Tensor-core windowed attention (head_dim 32, 7x7 window): FlashAttention-2
// style online softmax, QK^T and PV on the tensor cores (mma.sync m16n8k16,
// fp16 operands, fp32 accumulate), masks evaluated in registers.
//
// Work decomposition. A CTA owns a rectangle of query rows and stages the
// K/V halo of the whole rectangle once per key slot into shared memory with
// cp.async (zero-filled outside the grid, double-buffered across the slots of
// the 3D context window). Each warp owns 16 queries whose windows lie in
// RPW+6 consecutive halo rows, and walks only that band in 32-key chunks:
//   * context (3D): warp = a 1x16 query strip, band = 7 x 22 keys per slot;
//   * step batches (2D): warp = the 16 step-t positions of a 4x16 block,
//     band = 10 x 22 keys.
// 32-44% of the scanned scores are in-window. 128-row tcgen05 tiles would
// scan >= 14x22 keys per slot for the same queries (16% useful), so this
// operator uses warp-level MMA; every dense projection is on tcgen05.
//
// Semantics match SPEC.md:221-256 and the oracle: out-of-grid keys are
// masked (not padded), step masks <= / < per wavefront.h:34-43, the learned
// per-offset bias is added to the scaled score, softmax in fp32, a query
// with no allowed key outputs zeros.
#include <cfloat>
#include <cstdlib>

#include "check.h"
#include "kernels.h"
#include "launch.cuh"

namespace pswa_dev {

namespace {

constexpr int kHD = 32;     // head dim handled by this kernel
constexpr int kHaloW = 22;  // 16 query columns + 2*3 window margin
constexpr int kChunk = 32;
constexpr float kLog2e = 1.4426950408889634f;
constexpr int kMaxBandKeys = 224;  // 10 x 22 band rounded to the 32-key chunk
constexpr int kTblStride = 20;     // floats per band key: 16 queries + pad (conflict-free LDS)

__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                          uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// byte offset of (key, 16 B chunk) in a [key][32 halves] tile, chunk
// XOR-swizzled by (key >> 1) & 3: conflict-free ldmatrix over 8 keys.
__device__ __forceinline__ uint32_t sw(int key, int chunk) {
  return static_cast<uint32_t>(key * 64 + ((chunk ^ ((key >> 1) & 3)) << 4));
}

struct AttnArgs {
  const __half* q;
  int ldq;
  const int32_t* qinfo;
  const int32_t* tiles;
  int ntiles;
  const __half* kv;
  int ldkv, kv_slot_stride, H, W, wt, mask, s, d;
  const float* bias;
  __half* out;
  int ldo;
  int halo_keys;  // staged keys per slot buffer (>= halo rows * 22, multiple of 32, + slack)
  const int8_t* taps;  // [band keys (chunk-padded)][16 queries]: tap index or -1 (masked)
  int dbuf;            // double-buffer the slot halos (3D); 0 = stage each slot in place
};

__global__ void __launch_bounds__(256) window_attn_mma_kernel(const AttnArgs a) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = blockIdx.y;
  const int32_t* T = a.tiles + blockIdx.x * kAttnTileInts;
  const int hy0 = T[0], hx0 = T[1], HR = T[2], RPW = T[3], sl = T[4];
  const int taps_total = a.wt > 0 ? a.wt * 49 : 49;
  const int nslots = a.wt > 0 ? min(sl + 1, a.wt) : 1;
  const int j0 = sl - nslots + 1;
  const int kbuf = a.halo_keys * kHD * 2;  // bytes of one K (or V) buffer
  float* sbias = reinterpret_cast<float*>(smem + (a.wt > 0 && a.dbuf ? 4 : 2) * kbuf);
  const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(smem));

  const int band_keys = (RPW + 6) * kHaloW;
  const int nchunks = (band_keys + kChunk - 1) / kChunk;
  const int nbk = nchunks * kChunk;
  // per-slot score-offset table [band key][kTblStride]: log2e * bias of the
  // (key, query) window tap, -inf where the window / step mask excludes it
  float* stbl = sbias + 256;
  uint8_t* skv = reinterpret_cast<uint8_t*>(stbl + kMaxBandKeys * kTblStride);  // [halo_keys]

  // ---- stage the bias row of this head (pre-scaled by log2 e) and the
  // per-key in-grid flags
  for (int i = threadIdx.x; i < taps_total; i += blockDim.x)
    sbias[i] = a.bias[h * taps_total + i] * kLog2e;
  const int hkeys = HR * kHaloW;
  for (int key = threadIdx.x; key < a.halo_keys; key += blockDim.x) {
    const int ky = hy0 + key / kHaloW, kx = hx0 + key % kHaloW;
    skv[key] = key < hkeys && ky >= 0 && ky < a.H && kx >= 0 && kx < a.W;
  }

  auto stage = [&](int j, int buf) {
    const uint32_t kb = sbase + buf * 2 * kbuf, vb = kb + kbuf;
    for (int idx = threadIdx.x; idx < a.halo_keys * 4; idx += blockDim.x) {
      const int key = idx >> 2, ch = idx & 3;
      const int ky = hy0 + key / kHaloW, kx = hx0 + key % kHaloW;
      const bool ok = key < hkeys && ky >= 0 && ky < a.H && kx >= 0 && kx < a.W;
      const __half* src = a.kv + (ok ? static_cast<size_t>(j * a.kv_slot_stride + ky * a.W + kx) * a.ldkv +
                                           h * kHD + ch * 8
                                     : 0);
      cp_async16(kb + sw(key, ch), src, ok ? 16 : 0);
      cp_async16(vb + sw(key, ch), src + (ok ? a.d : 0), ok ? 16 : 0);
    }
    cp_commit();
  };
  stage(j0, 0);

  // ---- my 16 queries: fragment rows r0 = lane/4, r1 = r0 + 8
  const int32_t* Q = T + 8 + warp * 16;
  const int r0 = lane >> 2;
  const int qr[2] = {warp < T[5] ? Q[r0] : -1, warp < T[5] ? Q[r0 + 8] : -1};
  uint32_t qa[2][4];
  {
    const int kc = (lane & 3) * 2;
#pragma unroll
    for (int ks = 0; ks < 2; ++ks)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const __half* qp = a.q + static_cast<size_t>(qr[i] < 0 ? 0 : qr[i]) * a.ldq + h * kHD + ks * 16 + kc;
        qa[ks][i] = qr[i] >= 0 ? *reinterpret_cast<const uint32_t*>(qp) : 0u;
        qa[ks][i + 2] = qr[i] >= 0 ? *reinterpret_cast<const uint32_t*>(qp + 8) : 0u;
      }
  }
  const bool live = __any_sync(0xffffffffu, qr[0] >= 0 || qr[1] >= 0);
  const float qscale = 0.17677669529663687f * kLog2e;  // log2(e) / sqrt(32)
  const int key0 = warp * RPW * kHaloW;  // first key of my band in the CTA halo

  float o[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) o[i][e] = 0.0f;
  float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.0f, 0.0f};

  for (int js = 0; js < nslots; ++js) {
    const int j = j0 + js, buf = a.dbuf ? (js & 1) : 0;
    if (!a.dbuf && js > 0) stage(j, 0);  // previous slot fully consumed (barrier below)
    if (a.dbuf && js + 1 < nslots) {
      stage(j + 1, buf ^ 1);  // prefetch the next slot's halo
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    // score-offset table of this slot (the bias slice depends on the slot)
    {
      const float* sb = sbias + (a.wt > 0 ? (j - sl + a.wt - 1) * 49 : 0);
      if (js > 0) __syncthreads();  // previous slot's readers are done
      for (int i = threadIdx.x; i < nbk * 16; i += blockDim.x) {
        const int tap = a.taps[i];
        stbl[(i >> 4) * kTblStride + (i & 15)] = tap >= 0 ? sb[tap] : -INFINITY;
      }
    }
    __syncthreads();
    const uint32_t sK = sbase + buf * 2 * kbuf, sV = sK + kbuf;
    if (live) {
      for (int c = 0; c < nchunks; ++c) {
        float sacc[4][4];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
#pragma unroll
          for (int e = 0; e < 4; ++e) sacc[nt][e] = 0.0f;
          uint32_t b0, b1, b2, b3;
          ldsm_x4(sK + sw(key0 + c * kChunk + nt * 8 + (lane & 7), lane >> 3), b0, b1, b2, b3);
          mma16816(sacc[nt], qa[0], b0, b1);
          mma16816(sacc[nt], qa[1], b2, b3);
        }
        // window / step mask and bias from the tile-shape tap table
        float cmax[2] = {-INFINITY, -INFINITY};
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            const int bk = c * kChunk + nt * 8 + (lane & 3) * 2 + b;
            const bool kin = skv[key0 + bk] != 0;
            const float* trow = stbl + bk * kTblStride + r0;
#pragma unroll
            for (int ri = 0; ri < 2; ++ri) {
              const int e = ri * 2 + b;
              const float v = kin ? fmaf(sacc[nt][e], qscale, trow[8 * ri]) : -INFINITY;
              sacc[nt][e] = v;
              cmax[ri] = fmaxf(cmax[ri], v);
            }
          }
        float alpha[2];
#pragma unroll
        for (int ri = 0; ri < 2; ++ri) {
          cmax[ri] = fmaxf(cmax[ri], __shfl_xor_sync(0xffffffffu, cmax[ri], 1));
          cmax[ri] = fmaxf(cmax[ri], __shfl_xor_sync(0xffffffffu, cmax[ri], 2));
          const float mn = fmaxf(m[ri], cmax[ri]);
          alpha[ri] = mn == -INFINITY ? 1.0f : ex2(m[ri] - mn);  // ex2(-inf) = 0
          m[ri] = mn;
        }
        float rs[2] = {0.0f, 0.0f};
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int ri = e >> 1;
            const float p = sacc[nt][e] == -INFINITY ? 0.0f : ex2(sacc[nt][e] - m[ri]);
            sacc[nt][e] = p;
            rs[ri] += p;
          }
#pragma unroll
        for (int ri = 0; ri < 2; ++ri) {
          rs[ri] += __shfl_xor_sync(0xffffffffu, rs[ri], 1);
          rs[ri] += __shfl_xor_sync(0xffffffffu, rs[ri], 2);
          l[ri] = l[ri] * alpha[ri] + rs[ri];
        }
#pragma unroll
        for (int nd = 0; nd < 4; ++nd) {
          o[nd][0] *= alpha[0];
          o[nd][1] *= alpha[0];
          o[nd][2] *= alpha[1];
          o[nd][3] *= alpha[1];
        }
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          uint32_t pa[4];
          pa[0] = pack_h2(sacc[2 * kk][0], sacc[2 * kk][1]);
          pa[1] = pack_h2(sacc[2 * kk][2], sacc[2 * kk][3]);
          pa[2] = pack_h2(sacc[2 * kk + 1][0], sacc[2 * kk + 1][1]);
          pa[3] = pack_h2(sacc[2 * kk + 1][2], sacc[2 * kk + 1][3]);
          const int mi = lane >> 3;
          const int key = key0 + c * kChunk + kk * 16 + (mi & 1) * 8 + (lane & 7);
#pragma unroll
          for (int nd = 0; nd < 4; nd += 2) {
            uint32_t b0, b1, b2, b3;
            ldsm_x4_t(sV + sw(key, nd + (mi >> 1)), b0, b1, b2, b3);
            mma16816(o[nd], pa, b0, b1);
            mma16816(o[nd + 1], pa, b2, b3);
          }
        }
      }
    }
    __syncthreads();  // buffer `buf` is refilled two slots later
  }
  if (!live) return;
  const float inv0 = l[0] > 0.0f ? 1.0f / l[0] : 0.0f;
  const float inv1 = l[1] > 0.0f ? 1.0f / l[1] : 0.0f;
#pragma unroll
  for (int nd = 0; nd < 4; ++nd) {
    const int col = h * kHD + nd * 8 + (lane & 3) * 2;
    if (qr[0] >= 0)
      *reinterpret_cast<uint32_t*>(a.out + static_cast<size_t>(qr[0]) * a.ldo + col) =
          pack_h2(o[nd][0] * inv0, o[nd][1] * inv0);
    if (qr[1] >= 0)
      *reinterpret_cast<uint32_t*>(a.out + static_cast<size_t>(qr[1]) * a.ldo + col) =
          pack_h2(o[nd][2] * inv1, o[nd][3] * inv1);
  }
}

// Double-buffering the 3D slot halos overlaps staging with compute but halves
// the CTAs per SM; measured slower (3.68 vs 3.42 ms / frame), so off unless
// PSWA_ATTN_DBUF=1.
bool attn_dbuf() {
  static const bool on = std::getenv("PSWA_ATTN_DBUF") != nullptr;
  return on;
}

int smem_bytes(int halo_keys, bool three_d) {
  // K/V buffers + bias (256 floats) + score-offset table + key flags
  return (three_d && attn_dbuf() ? 4 : 2) * halo_keys * kHD * 2 + 256 * 4 +
         kMaxBandKeys * kTblStride * 4 + halo_keys;
}

}  // namespace

bool window_attention_tiles_supported(int hd, int win_h, int win_w) {
  return hd == kHD && win_h == 7 && win_w == 7;
}

int window_attention_halo_keys(int halo_rows) {
  // staged keys: whole halo rounded to chunks, plus one chunk of slack for the
  // last warp's band overrun (those keys are masked)
  return (halo_rows * kHaloW + kChunk - 1) / kChunk * kChunk + kChunk;
}

void window_attention_tiles_init(int max_smem_bytes) {
  PSWA_CUDA(cudaFuncSetAttribute(window_attn_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 max_smem_bytes));
}

int window_attention_tiles_smem(int halo_rows, bool three_d) {
  return smem_bytes(window_attention_halo_keys(halo_rows), three_d);
}

void window_attention_tiles(const __half* q, int ldq, const int32_t* qinfo, const int32_t* tiles,
                            int ntiles, int warps_per_tile, int halo_rows, const int8_t* taps,
                            const __half* kv, int ldkv, int kv_slot_stride, int H, int W,
                            int heads, int wt, int mask, int s, const float* bias, __half* out,
                            int ldo, cudaStream_t st) {
  if (ntiles <= 0) return;
  AttnArgs a{q, ldq, qinfo, tiles, ntiles, kv, ldkv, kv_slot_stride, H, W, wt, mask, s,
             heads * kHD, bias, out, ldo, window_attention_halo_keys(halo_rows), taps,
             attn_dbuf() ? 1 : 0};
  dim3 grid(ntiles, heads);
  launch_k(window_attn_mma_kernel, grid, dim3(warps_per_tile * 32), smem_bytes(a.halo_keys, wt > 0), st, a);
  PSWA_LAUNCH_CHECK();
}

}  // namespace pswa_dev
