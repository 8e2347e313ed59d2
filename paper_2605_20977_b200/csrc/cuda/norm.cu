// Row kernels: RMSNorm (tensor.cpp:81-86 semantics, eps 1e-5, optional
// per-group normalisation for the channel transformer), gathers, casts.
// All HBM-bound: one warp per row, coalesced 128 B accesses.
#include "check.h"
#include "kernels.h"
#include "launch.cuh"

namespace pswa_dev {

namespace {

__global__ void rmsnorm_kernel(const float* __restrict__ x, int ldx, const int* __restrict__ src,
                               int M, int d, int group, const float* __restrict__ gain,
                               __half* __restrict__ y, int ldy) {
  pdl_wait();
  pdl_trigger();
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= M) return;
  const float* xr = x + static_cast<size_t>(src ? src[row] : row) * ldx;
  __half* yr = y + static_cast<size_t>(row) * ldy;
  const bool vec = (group & 127) == 0 && (ldx & 3) == 0 && (ldy & 3) == 0;
  for (int g0 = 0; g0 < d; g0 += group) {
    if (vec) {
      // group is a multiple of 128: each lane owns group/128 float4 quads,
      // all loaded before the reduction (one round trip per row)
      constexpr int kMaxQ = 8;  // group <= 1024
      float4 v[kMaxQ];
      const int nq = group >> 7;
      float ss = 0.0f;
#pragma unroll
      for (int k = 0; k < kMaxQ; ++k)
        if (k < nq) {
          v[k] = *reinterpret_cast<const float4*>(xr + g0 + (k * 32 + lane) * 4);
          ss += v[k].x * v[k].x + v[k].y * v[k].y + v[k].z * v[k].z + v[k].w * v[k].w;
        }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      const float inv = 1.0f / sqrtf(ss / static_cast<float>(group) + 1e-5f);
#pragma unroll
      for (int k = 0; k < kMaxQ; ++k)
        if (k < nq) {
          const int c = g0 + (k * 32 + lane) * 4;
          const float4 gv = *reinterpret_cast<const float4*>(gain + c);
          __half2 h[2] = {__floats2half2_rn(gv.x * v[k].x * inv, gv.y * v[k].y * inv),
                          __floats2half2_rn(gv.z * v[k].z * inv, gv.w * v[k].w * inv)};
          *reinterpret_cast<uint2*>(yr + c) = *reinterpret_cast<uint2*>(h);
        }
    } else {
      float ss = 0.0f;
      for (int i = lane; i < group; i += 32) {
        const float v = xr[g0 + i];
        ss += v * v;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      const float inv = 1.0f / sqrtf(ss / static_cast<float>(group) + 1e-5f);
      for (int i = lane; i < group; i += 32)
        yr[g0 + i] = __float2half_rn(gain[g0 + i] * xr[g0 + i] * inv);
    }
  }
}

__global__ void rms_prep_kernel(const float* __restrict__ x, int ldx, const int* __restrict__ src,
                                int M, int d, float* __restrict__ xc, int ldc, __half* __restrict__ x16,
                                int ld16, float* __restrict__ ssq, int ld_ssq) {
  pdl_wait();
  pdl_trigger();
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= M) return;
  const float* xr = x + static_cast<size_t>(src ? src[row] : row) * ldx;
  if ((d & 127) == 0) {
    for (int c0 = 0; c0 < d; c0 += 128) {  // lane owns 4 columns; 8 lanes = one 32-column chunk
      const int c = c0 + lane * 4;
      const float4 v = *reinterpret_cast<const float4*>(xr + c);
      if (xc) *reinterpret_cast<float4*>(xc + static_cast<size_t>(row) * ldc + c) = v;
      __half2 h[2] = {__floats2half2_rn(v.x, v.y), __floats2half2_rn(v.z, v.w)};
      *reinterpret_cast<uint2*>(x16 + static_cast<size_t>(row) * ld16 + c) = *reinterpret_cast<uint2*>(h);
      float ss = v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
      ss += __shfl_xor_sync(0xffffffffu, ss, 1);
      ss += __shfl_xor_sync(0xffffffffu, ss, 2);
      ss += __shfl_xor_sync(0xffffffffu, ss, 4);
      if ((lane & 7) == 0) ssq[static_cast<size_t>(row) * ld_ssq + (c >> 5)] = ss;
    }
  } else {
    for (int c0 = 0; c0 < d; c0 += 32) {  // one chunk per pass, lane = column
      const float v = xr[c0 + lane];
      if (xc) xc[static_cast<size_t>(row) * ldc + c0 + lane] = v;
      x16[static_cast<size_t>(row) * ld16 + c0 + lane] = __float2half_rn(v);
      float ss = v * v;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if (lane == 0) ssq[static_cast<size_t>(row) * ld_ssq + (c0 >> 5)] = ss;
    }
  }
}

__global__ void gather_f32_kernel(const float* __restrict__ src, int lds, const int* __restrict__ rows,
                                  int M, int n, float* __restrict__ dst, int ldd) {
  pdl_wait();
  pdl_trigger();
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= M) return;
  const float* s = src + static_cast<size_t>(rows ? rows[row] : row) * lds;
  float* o = dst + static_cast<size_t>(row) * ldd;
  if ((n & 3) == 0 && (lds & 3) == 0 && (ldd & 3) == 0) {
    const float4* s4 = reinterpret_cast<const float4*>(s);
    float4* o4 = reinterpret_cast<float4*>(o);
    for (int i = lane; i < n / 4; i += 32) o4[i] = s4[i];
  } else {
    for (int i = lane; i < n; i += 32) o[i] = s[i];
  }
}

__global__ void yhat_f16_kernel(const int32_t* __restrict__ yhat, int C, const int* __restrict__ rows,
                                int M, int c0, int nc, __half* __restrict__ dst, int ldd, int ncols) {
  pdl_wait();
  pdl_trigger();
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= M) return;
  const int32_t* s = yhat + static_cast<size_t>(rows ? rows[row] : row) * C + c0;
  __half* o = dst + static_cast<size_t>(row) * ldd;
  for (int i = lane; i < ncols; i += 32)
    o[i] = i < nc ? __int2half_rn(s[i]) : __float2half_rn(0.0f);
}

__global__ void f32_to_f16_kernel(const float* __restrict__ src, int lds, int M, int n,
                                  __half* __restrict__ dst, int ldd, int ncols) {
  pdl_wait();
  pdl_trigger();
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= M) return;
  const float* s = src + static_cast<size_t>(row) * lds;
  __half* o = dst + static_cast<size_t>(row) * ldd;
  for (int i = lane; i < ncols; i += 32) o[i] = __float2half_rn(i < n ? s[i] : 0.0f);
}

__global__ void fill_slots_kernel(const float* const* __restrict__ ring, const int* __restrict__ slot_src,
                                  const float* __restrict__ pad, int T, int HW, int d,
                                  float* __restrict__ x) {
  pdl_wait();
  pdl_trigger();
  const size_t total = static_cast<size_t>(T) * HW * (d / 4);
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int c4 = static_cast<int>(i % (d / 4));
    const size_t r = i / (d / 4);
    const int t = static_cast<int>(r / HW);
    const int p = static_cast<int>(r % HW);
    const int k = slot_src[t];
    const float4 v = k >= 0 ? reinterpret_cast<const float4*>(ring[k] + static_cast<size_t>(p) * d)[c4]
                            : reinterpret_cast<const float4*>(pad)[c4];
    reinterpret_cast<float4*>(x)[i] = v;
  }
}

// dst[c * ldd + r] = src[r * lds + c] for r < rows, c < cols
__global__ void transpose_i32_kernel(const int32_t* __restrict__ src, int rows, int cols, int lds,
                                     int32_t* __restrict__ dst, int ldd) {
  pdl_wait();
  pdl_trigger();
  __shared__ int32_t tile[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += 8) {
    const int r = by + j, c = bx + threadIdx.x;
    if (r < rows && c < cols) tile[j][threadIdx.x] = src[static_cast<size_t>(r) * lds + c];
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += 8) {
    const int c = bx + j, r = by + threadIdx.x;
    if (r < rows && c < cols) dst[static_cast<size_t>(c) * ldd + r] = tile[threadIdx.x][j];
  }
}

__global__ void scatter_f16_kernel(const __half* __restrict__ src, int lds, const int* __restrict__ rows,
                                   int M, int n, __half* __restrict__ dst, int ldd) {
  pdl_wait();
  pdl_trigger();
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= M) return;
  const __half* s = src + static_cast<size_t>(row) * lds;
  __half* o = dst + static_cast<size_t>(rows[row]) * ldd;
  for (int i = lane; i < n; i += 32) o[i] = s[i];
}

__global__ void scatter_f32_kernel(const float* __restrict__ src, int lds, const int* __restrict__ rows,
                                   int M, int n, float* __restrict__ dst, int ldd) {
  pdl_wait();
  pdl_trigger();
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= M) return;
  const float* s = src + static_cast<size_t>(row) * lds;
  float* o = dst + static_cast<size_t>(rows[row]) * ldd;
  for (int i = lane; i < n; i += 32) o[i] = s[i];
}

inline int warp_grid(int M) { return (M + 7) / 8; }

}  // namespace

void rmsnorm_rows(const float* x, int ldx, const int* src_rows, int M, int d, int group,
                  const float* gain, __half* y, int ldy, cudaStream_t st) {
  if (M <= 0) return;
  launch_k(rmsnorm_kernel, dim3(warp_grid(M)), dim3(256), 0, st, x, ldx, src_rows, M, d, group, gain, y, ldy);
  PSWA_LAUNCH_CHECK();
}

void gather_rows_f32(const float* src, int lds, const int* rows, int M, int n, float* dst, int ldd,
                     cudaStream_t st) {
  if (M <= 0) return;
  launch_k(gather_f32_kernel, dim3(warp_grid(M)), dim3(256), 0, st, src, lds, rows, M, n, dst, ldd);
  PSWA_LAUNCH_CHECK();
}

void yhat_rows_f16(const int32_t* yhat, int C, const int* rows, int M, int c0, int nc, __half* dst,
                   int ldd, int ncols, cudaStream_t st) {
  if (M <= 0) return;
  launch_k(yhat_f16_kernel, dim3(warp_grid(M)), dim3(256), 0, st, yhat, C, rows, M, c0, nc, dst, ldd, ncols);
  PSWA_LAUNCH_CHECK();
}

void f32_to_f16_rows(const float* src, int lds, int M, int n, __half* dst, int ldd, int ncols,
                     cudaStream_t st) {
  if (M <= 0) return;
  launch_k(f32_to_f16_kernel, dim3(warp_grid(M)), dim3(256), 0, st, src, lds, M, n, dst, ldd, ncols);
  PSWA_LAUNCH_CHECK();
}

void fill_context_slots(const float* const* ring, const int* slot_src, const float* pad, int T,
                        int HW, int d, float* x, cudaStream_t st) {
  launch_k(fill_slots_kernel, dim3(148 * 8), dim3(256), 0, st, ring, slot_src, pad, T, HW, d, x);
  PSWA_LAUNCH_CHECK();
}

__global__ void halo_push_kernel(const __half* __restrict__ src, __half* __restrict__ dst, int ld,
                                 const int2* __restrict__ pairs, int n) {
  pdl_wait();
  pdl_trigger();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= n) return;
  const int2 p = pairs[warp];
  const uint4* s = reinterpret_cast<const uint4*>(src + static_cast<size_t>(p.x) * ld);
  uint4* d = reinterpret_cast<uint4*>(dst + static_cast<size_t>(p.y) * ld);
  for (int i = lane; i < ld / 8; i += 32) d[i] = s[i];
  __threadfence_system();  // peer stores performed before any later signal
}

__global__ void band_signal_kernel(unsigned* to_up, unsigned* to_down) {
  pdl_wait();
  __threadfence_system();
  if (to_up) atomicAdd_system(to_up, 1u);
  if (to_down) atomicAdd_system(to_down, 1u);
}

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void band_wait_kernel(const unsigned* mbox, unsigned* wait_ctr, int need_up,
                                 int need_down, int* status) {
  pdl_wait();
  const unsigned e = ++wait_ctr[0];
  if (*reinterpret_cast<volatile int*>(status) & 8) return;  // a wait already timed out: fail fast
  const unsigned long long t0 = globaltimer();
  auto behind = [&](int i) { return static_cast<int>(ld_acquire_sys(mbox + i) - e) < 0; };
  while ((need_up && behind(0)) || (need_down && behind(1))) {
    __nanosleep(200);
    if (globaltimer() - t0 > 20000000000ull) {
      atomicOr(status, 8);
      break;
    }
  }
  __threadfence();
}

void halo_push(const __half* src, __half* dst, int ld, const int2* pairs, int n, cudaStream_t st) {
  if (n <= 0) return;
  launch_k(halo_push_kernel, dim3((n + 7) / 8), dim3(256), 0, st, src, dst, ld, pairs, n);
  PSWA_LAUNCH_CHECK();
}

void band_signal(unsigned* to_up, unsigned* to_down, cudaStream_t st) {
  launch_k(band_signal_kernel, dim3(1), dim3(1), 0, st, to_up, to_down);
  PSWA_LAUNCH_CHECK();
}

void band_wait(const unsigned* mbox, unsigned* wait_ctr, bool need_up, bool need_down, int* status,
               cudaStream_t st) {
  launch_k(band_wait_kernel, dim3(1), dim3(1), 0, st, mbox, wait_ctr, need_up ? 1 : 0,
           need_down ? 1 : 0, status);
  PSWA_LAUNCH_CHECK();
}

void rms_prep(const float* x, int ldx, const int* src_rows, int M, int d, float* xcopy, int ldc,
              __half* x16, int ld16, float* ssq, int ld_ssq, cudaStream_t st) {
  if (M <= 0) return;
  if (d % 32) throw std::invalid_argument("rms_prep: d % 32");
  launch_k(rms_prep_kernel, dim3((M + 7) / 8), dim3(256), 0, st, x, ldx, src_rows, M, d, xcopy, ldc,
           x16, ld16, ssq, ld_ssq);
  PSWA_LAUNCH_CHECK();
}

void yhat_to_chw(const int32_t* src, int HW, int C, int32_t* dst, cudaStream_t st) {
  yhat_to_chw_cols(src, HW, C, 0, C, dst, st);
}

void yhat_to_chw_cols(const int32_t* src, int HW, int C, int c0, int nc, int32_t* dst,
                      cudaStream_t st) {
  dim3 grid((nc + 31) / 32, (HW + 31) / 32);
  launch_k(transpose_i32_kernel, dim3(grid), dim3(32, 8), 0, st, src + c0, HW, nc, C,
           dst + static_cast<size_t>(c0) * HW, HW);
  PSWA_LAUNCH_CHECK();
}

void yhat_from_chw(const int32_t* src, int HW, int C, int32_t* dst, cudaStream_t st) {
  dim3 grid((HW + 31) / 32, (C + 31) / 32);
  launch_k(transpose_i32_kernel, dim3(grid), dim3(32, 8), 0, st, src, C, HW, HW, dst, C);
  PSWA_LAUNCH_CHECK();
}

void scatter_rows_f32(const float* src, int lds, const int* rows, int M, int n, float* dst,
                      int ldd, cudaStream_t st) {
  if (M <= 0) return;
  launch_k(scatter_f32_kernel, dim3(warp_grid(M)), dim3(256), 0, st, src, lds, rows, M, n, dst, ldd);
  PSWA_LAUNCH_CHECK();
}

void scatter_rows_f16(const __half* src, int lds, const int* rows, int M, int n, __half* dst,
                      int ldd, cudaStream_t st) {
  if (M <= 0) return;
  launch_k(scatter_f16_kernel, dim3(warp_grid(M)), dim3(256), 0, st, src, lds, rows, M, n, dst, ldd);
  PSWA_LAUNCH_CHECK();
}

}  // namespace pswa_dev
