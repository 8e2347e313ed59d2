// Tensor-core windowed attention (head_dim 32, 7x7 window): FlashAttention-2
// style online softmax over a per-warp key halo, QK^T and PV on the tensor
// cores (mma.sync m16n8k16, fp16 in / fp32 accumulate).
//
// Why warp-sized tiles: every query sees only its 7x7 (x slots) neighbourhood,
// so a tile of Q queries must scan the union halo of its windows. A 16-query
// tile (1x16 strip, or the 16 step-t positions of a 4x16 block) scans a 7x22
// or 10x22 halo: 32-44% of the computed scores are in-window. The 128-row
// tiles of tcgen05 would scan a >= 14x22 halo (16% useful), so for this
// operator the warp-level MMA is the better fit; all dense projections stay
// on tcgen05 (gemm.cu).
//
// Semantics are those of SPEC.md:221-256 / the oracle: keys outside the grid
// are masked (not padded), step masks <= / < follow wavefront.h:34-43, the
// learned per-offset bias is added to the scaled score, fp32 softmax, a query
// with no allowed key outputs zeros.
#include <cfloat>

#include "check.h"
#include "kernels.h"

namespace pswa_dev {

namespace {

constexpr int kHD = 32;        // head dim handled by this kernel
constexpr int kHaloW = 22;     // 16 query columns + 2*3 window margin
constexpr int kMaxKeys = 224;  // 10 x 22 halo, rounded up to the 32-key chunk
constexpr int kChunk = 32;
constexpr int kWarps = 4;
constexpr int kSmemPerWarp = 2 * kMaxKeys * kHD * 2;  // K and V halves

__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
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

// byte offset of (key, 16 B chunk) inside a [key][32 halves] tile with the
// chunk XOR-swizzled by (key >> 1) & 3: conflict-free ldmatrix of 8 keys.
__device__ __forceinline__ uint32_t sw(int key, int chunk) {
  return static_cast<uint32_t>(key * 64 + ((chunk ^ ((key >> 1) & 3)) << 4));
}

__global__ void __launch_bounds__(kWarps * 32)
    window_attn_mma_kernel(const __half* __restrict__ q, int ldq, const int32_t* __restrict__ qinfo,
                           const int32_t* __restrict__ tiles, int ntiles,
                           const __half* __restrict__ kv, int ldkv, int kv_slot_stride, int H,
                           int W, int wt, int mask, int s, const float* __restrict__ bias,
                           __half* __restrict__ out, int ldo, int d) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x * kWarps + warp;
  const int h = blockIdx.y;
  if (tile >= ntiles) return;
  const int32_t* T = tiles + tile * kAttnTileInts;
  const int hy0 = T[0], hx0 = T[1], hh = T[2], sl = T[4];
  const int nkeys = hh * kHaloW;
  const int nchunks = (nkeys + kChunk - 1) / kChunk;
  uint8_t* sK = smem + warp * kSmemPerWarp;
  uint8_t* sV = sK + kMaxKeys * kHD * 2;
  const uint32_t sK_a = static_cast<uint32_t>(__cvta_generic_to_shared(sK));
  const uint32_t sV_a = static_cast<uint32_t>(__cvta_generic_to_shared(sV));

  // my two fragment rows (queries)
  const int r0 = lane >> 2, r1 = r0 + 8;
  const int qr0 = T[8 + r0], qr1 = T[8 + r1];
  int qy[2] = {-1000, -1000}, qx[2] = {-1000, -1000}, qs[2] = {0, 0};
  if (qr0 >= 0) {
    const int inf = qinfo[qr0];
    qy[0] = (inf >> 12) & 0xFFF;
    qx[0] = inf & 0xFFF;
    qs[0] = (qy[0] + qx[0]) % s;
  }
  if (qr1 >= 0) {
    const int inf = qinfo[qr1];
    qy[1] = (inf >> 12) & 0xFFF;
    qx[1] = inf & 0xFFF;
    qs[1] = (qy[1] + qx[1]) % s;
  }
  // Q fragments: 2 k-steps x {row r0 k, row r1 k, row r0 k+8, row r1 k+8}
  uint32_t qa[2][4];
  {
    const int kc = (lane & 3) * 2;
    const __half* q0p = q + static_cast<size_t>(qr0 < 0 ? 0 : qr0) * ldq + h * kHD;
    const __half* q1p = q + static_cast<size_t>(qr1 < 0 ? 0 : qr1) * ldq + h * kHD;
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      qa[ks][0] = qr0 >= 0 ? *reinterpret_cast<const uint32_t*>(q0p + ks * 16 + kc) : 0u;
      qa[ks][1] = qr1 >= 0 ? *reinterpret_cast<const uint32_t*>(q1p + ks * 16 + kc) : 0u;
      qa[ks][2] = qr0 >= 0 ? *reinterpret_cast<const uint32_t*>(q0p + ks * 16 + kc + 8) : 0u;
      qa[ks][3] = qr1 >= 0 ? *reinterpret_cast<const uint32_t*>(q1p + ks * 16 + kc + 8) : 0u;
    }
  }
  const float scale = 0.17677669529663687f;  // 1/sqrt(32)
  const int taps2 = 49;
  const int taps_total = wt > 0 ? wt * taps2 : taps2;
  const float* bh = bias + h * taps_total;

  float o[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) o[i][e] = 0.0f;
  float m[2] = {-FLT_MAX, -FLT_MAX}, l[2] = {0.0f, 0.0f};
  bool seen[2] = {false, false};

  const int j0 = wt > 0 ? max(0, sl - wt + 1) : sl;
  for (int j = j0; j <= sl; ++j) {
    // ---- stage this slot's K / V halo (zero outside the grid)
    __syncwarp();
    for (int idx = lane; idx < nchunks * kChunk * 4; idx += 32) {
      const int key = idx >> 2, ch = idx & 3;
      const int ky = hy0 + key / kHaloW, kx = hx0 + key % kHaloW;
      uint4 kval = make_uint4(0, 0, 0, 0), vval = make_uint4(0, 0, 0, 0);
      if (key < nkeys && ky >= 0 && ky < H && kx >= 0 && kx < W) {
        const __half* base = kv + static_cast<size_t>(j * kv_slot_stride + ky * W + kx) * ldkv + h * kHD + ch * 8;
        kval = __ldg(reinterpret_cast<const uint4*>(base));
        vval = __ldg(reinterpret_cast<const uint4*>(base + d));
      }
      *reinterpret_cast<uint4*>(sK + sw(key, ch)) = kval;
      *reinterpret_cast<uint4*>(sV + sw(key, ch)) = vval;
    }
    __syncwarp();
    const int tap_base = wt > 0 ? (j - sl + wt - 1) * taps2 : 0;

    for (int c = 0; c < nchunks; ++c) {
      // ---- S = Q K^T for keys [c*32, c*32+32)
      float sacc[4][4];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
#pragma unroll
        for (int e = 0; e < 4; ++e) sacc[nt][e] = 0.0f;
        const int key = c * kChunk + nt * 8 + (lane & 7);
        uint32_t b0, b1, b2, b3;
        ldsm_x4(sK_a + sw(key, lane >> 3), b0, b1, b2, b3);
        mma16816(sacc[nt], qa[0], b0, b1);
        mma16816(sacc[nt], qa[1], b2, b3);
      }
      // ---- window / step mask, bias, online softmax
      float cmax[2] = {-INFINITY, -INFINITY};
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int key = c * kChunk + nt * 8 + (lane & 3) * 2 + (e & 1);
          const int ri = e >> 1;
          const int ky = hy0 + key / kHaloW, kx = hx0 + key % kHaloW;
          const int dy = ky - qy[ri], dx = kx - qx[ri];
          bool ok = key < nkeys && ky >= 0 && ky < H && kx >= 0 && kx < W && dy >= -3 &&
                    dy <= 3 && dx >= -3 && dx <= 3;
          if (ok && mask) {
            const int ks = (ky + kx) % s;
            ok = mask == 1 ? ks <= qs[ri] : ks < qs[ri];
          }
          float v = -INFINITY;
          if (ok) v = sacc[nt][e] * scale + __ldg(bh + tap_base + (dy + 3) * 7 + (dx + 3));
          sacc[nt][e] = v;
          cmax[ri] = fmaxf(cmax[ri], v);
        }
#pragma unroll
      for (int ri = 0; ri < 2; ++ri) {
        cmax[ri] = fmaxf(cmax[ri], __shfl_xor_sync(0xffffffffu, cmax[ri], 1));
        cmax[ri] = fmaxf(cmax[ri], __shfl_xor_sync(0xffffffffu, cmax[ri], 2));
      }
      float alpha[2], mnew[2];
#pragma unroll
      for (int ri = 0; ri < 2; ++ri) {
        const bool has = cmax[ri] > -INFINITY;
        mnew[ri] = has ? fmaxf(m[ri], cmax[ri]) : m[ri];
        alpha[ri] = (has && seen[ri]) ? __expf(m[ri] - mnew[ri]) : 1.0f;
        if (has) seen[ri] = true;
        m[ri] = mnew[ri];
      }
      float rs[2] = {0.0f, 0.0f};
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int ri = e >> 1;
          const float p = sacc[nt][e] > -INFINITY ? __expf(sacc[nt][e] - m[ri]) : 0.0f;
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
      // ---- O += P V
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        uint32_t pa[4];
        pa[0] = pack_h2(sacc[2 * kk][0], sacc[2 * kk][1]);
        pa[1] = pack_h2(sacc[2 * kk][2], sacc[2 * kk][3]);
        pa[2] = pack_h2(sacc[2 * kk + 1][0], sacc[2 * kk + 1][1]);
        pa[3] = pack_h2(sacc[2 * kk + 1][2], sacc[2 * kk + 1][3]);
#pragma unroll
        for (int nd = 0; nd < 4; nd += 2) {
          const int mi = lane >> 3;
          const int key = c * kChunk + kk * 16 + (mi & 1) * 8 + (lane & 7);
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(sV_a + sw(key, nd + (mi >> 1)), b0, b1, b2, b3);
          mma16816(o[nd], pa, b0, b1);
          mma16816(o[nd + 1], pa, b2, b3);
        }
      }
    }
  }
  // ---- normalise and store
  const float inv0 = l[0] > 0.0f ? 1.0f / l[0] : 0.0f;
  const float inv1 = l[1] > 0.0f ? 1.0f / l[1] : 0.0f;
#pragma unroll
  for (int nd = 0; nd < 4; ++nd) {
    const int col = h * kHD + nd * 8 + (lane & 3) * 2;
    if (qr0 >= 0)
      *reinterpret_cast<uint32_t*>(out + static_cast<size_t>(qr0) * ldo + col) =
          pack_h2(o[nd][0] * inv0, o[nd][1] * inv0);
    if (qr1 >= 0)
      *reinterpret_cast<uint32_t*>(out + static_cast<size_t>(qr1) * ldo + col) =
          pack_h2(o[nd][2] * inv1, o[nd][3] * inv1);
  }
}

}  // namespace

bool window_attention_tiles_supported(int hd, int win_h, int win_w) {
  return hd == kHD && win_h == 7 && win_w == 7;
}

void window_attention_tiles_init() {
  PSWA_CUDA(cudaFuncSetAttribute(window_attn_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kWarps * kSmemPerWarp));
}

void window_attention_tiles(const __half* q, int ldq, const int32_t* qinfo, const int32_t* tiles,
                            int ntiles, const __half* kv, int ldkv, int kv_slot_stride, int H,
                            int W, int heads, int wt, int mask, int s, const float* bias,
                            __half* out, int ldo, cudaStream_t st) {
  if (ntiles <= 0) return;
  dim3 grid((ntiles + kWarps - 1) / kWarps, heads);
  window_attn_mma_kernel<<<grid, kWarps * 32, kWarps * kSmemPerWarp, st>>>(
      q, ldq, qinfo, tiles, ntiles, kv, ldkv, kv_slot_stride, H, W, wt, mask, s, bias, out, ldo,
      heads * kHD);
  PSWA_LAUNCH_CHECK();
}

}  // namespace pswa_dev
