// Masked sliding-window attention over frame-indexed K/V caches.
//
// Replaces swa2d / cross_windowed / swa3d_timecausal and the
// per-row softmax of tensor.cpp:60-79 for the decode path. One warp owns one
// (query, head): in the score pass lane l evaluates window taps l, l+32, ...
// (slot, dy, dx raster order), applying the out-of-bounds and step masks of
// wavefront.h:34-43 by index arithmetic on the query's (y, x); the fp32
// softmax runs on warp shuffles; in the PV pass the lanes own the head dims
// and walk the allowed taps, so every V row is one coalesced 64 B read.
// Zero allowed keys give a zero output (the accumulator's step-0 contract,
// SPEC.md:246).
#include <cfloat>

#include "check.h"
#include "kernels.h"
#include "launch.cuh"

namespace pswa_dev {

namespace {

constexpr int kMaxChunks = 8;  // up to 256 taps (5 x 7 x 7 = 245)

template <int HD>
__global__ void __launch_bounds__(256)
    window_attn_kernel(const __half* __restrict__ q, int ldq, const int32_t* __restrict__ qinfo,
                       int Mq, const __half* __restrict__ kv, int ldkv, int kv_slot_stride, int H,
                       int W, int heads, int wh, int ww, int wt, int mask, int s,
                       const float* __restrict__ bias, __half* __restrict__ out, int ldo, int d) {
  pdl_wait();
  pdl_trigger();
  const int gw = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const int i = gw / heads, h = gw % heads;
  if (i >= Mq) return;
  const int info = qinfo[i];
  const int sl = info >> 24, y = (info >> 12) & 0xFFF, x = info & 0xFFF;
  const int qs = (y + x) % s;
  const int nslot = wt > 0 ? min(sl + 1, wt) : 1;
  const int j0 = sl - nslot + 1;
  const int taps2 = wh * ww;
  const int ntaps = nslot * taps2;
  const int taps_total = wt > 0 ? wt * taps2 : taps2;
  const int nchunks = (ntaps + 31) >> 5;

  float qv[HD];
  {
    const __half* qp = q + static_cast<size_t>(i) * ldq + h * HD;
#pragma unroll
    for (int e = 0; e < HD; e += 2) {
      const float2 f = __half22float2(*reinterpret_cast<const __half2*>(qp + e));
      qv[e] = f.x;
      qv[e + 1] = f.y;
    }
  }
  const float scale = 1.0f / sqrtf(static_cast<float>(HD));

  float sc[kMaxChunks];
  int rowk[kMaxChunks];
  float mx = -FLT_MAX;
  bool any = false;
#pragma unroll
  for (int c = 0; c < kMaxChunks; ++c) {
    sc[c] = -FLT_MAX;
    rowk[c] = -1;
    if (c >= nchunks) continue;
    const int t = c * 32 + lane;
    if (t >= ntaps) continue;
    const int jj = j0 + t / taps2;
    const int r = t % taps2;
    const int ky = y + r / ww - wh / 2;
    const int kx = x + r % ww - ww / 2;
    if (ky < 0 || ky >= H || kx < 0 || kx >= W) continue;
    const int ks = (ky + kx) % s;
    if ((mask == 1 && ks > qs) || (mask == 2 && ks >= qs)) continue;
    const int row = jj * kv_slot_stride + ky * W + kx;
    const __half* kp = kv + static_cast<size_t>(row) * ldkv + h * HD;
    float dot = 0.0f;
#pragma unroll
    for (int e = 0; e < HD; e += 2) {
      const float2 f = __half22float2(*reinterpret_cast<const __half2*>(kp + e));
      dot += qv[e] * f.x;
      dot += qv[e + 1] * f.y;
    }
    const int tap = wt > 0 ? (jj - sl + wt - 1) * taps2 + r : r;
    sc[c] = dot * scale + bias[h * taps_total + tap];
    rowk[c] = row;
    mx = fmaxf(mx, sc[c]);
    any = true;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  const bool has_keys = __any_sync(0xffffffffu, any);
  __half* op = out + static_cast<size_t>(i) * ldo + h * HD;
  if (!has_keys) {
    for (int e = lane; e < HD; e += 32) op[e] = __float2half_rn(0.0f);
    return;
  }
  float sum = 0.0f;
#pragma unroll
  for (int c = 0; c < kMaxChunks; ++c) {
    const float p = rowk[c] >= 0 ? __expf(sc[c] - mx) : 0.0f;
    sc[c] = p;
    sum += p;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const float inv = 1.0f / sum;

  constexpr int kDims = HD >= 32 ? HD / 32 : 1;
  float acc[kDims];
#pragma unroll
  for (int k = 0; k < kDims; ++k) acc[k] = 0.0f;
  const __half* vbase = kv + d + h * HD;
#pragma unroll
  for (int c = 0; c < kMaxChunks; ++c) {
    if (c >= nchunks) break;
    for (int l = 0; l < 32; ++l) {
      const int row = __shfl_sync(0xffffffffu, rowk[c], l);
      if (row < 0) continue;
      const float w = __shfl_sync(0xffffffffu, sc[c], l);
      const __half* vp = vbase + static_cast<size_t>(row) * ldkv;
#pragma unroll
      for (int k = 0; k < kDims; ++k) {
        const int e = lane + 32 * k;
        if (e < HD) acc[k] += w * __half2float(vp[e]);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < kDims; ++k) {
    const int e = lane + 32 * k;
    if (e < HD) op[e] = __float2half_rn(acc[k] * inv);
  }
}

}  // namespace

void window_attention(const __half* q, int ldq, const int32_t* qinfo, int Mq, const __half* kv,
                      int ldkv, int kv_slot_stride, int H, int W, int heads, int hd, int win_h,
                      int win_w, int win_t, int mask, int s, const float* bias, __half* out,
                      int ldo, cudaStream_t st) {
  if (Mq <= 0) return;
  if ((win_t > 0 ? win_t : 1) * win_h * win_w > kMaxChunks * 32)
    throw std::invalid_argument("window_attention: window too large");
  const int d = hd * heads;
  const long warps = static_cast<long>(Mq) * heads;
  const int grid = static_cast<int>((warps + 7) / 8);
#define PSWA_ATTN(HD)                                                                         \
  launch_k(window_attn_kernel<HD>, dim3(grid), dim3(256), 0, st, q, ldq, qinfo, Mq, kv, ldkv, kv_slot_stride, H, \
                                               W, heads, win_h, win_w, win_t, mask, s, bias,  \
                                               out, ldo, d)
  switch (hd) {
    case 4: PSWA_ATTN(4); break;
    case 8: PSWA_ATTN(8); break;
    case 16: PSWA_ATTN(16); break;
    case 32: PSWA_ATTN(32); break;
    case 64: PSWA_ATTN(64); break;
    default: throw std::invalid_argument("window_attention: unsupported head_dim");
  }
#undef PSWA_ATTN
  PSWA_LAUNCH_CHECK();
}

}  // namespace pswa_dev
