// tcgen05 GEMM with fused epilogues: C[M,N] = A[M,K] . B[N,K]^T
// (A activations, B packed weights, both fp16 K-major; fp32 accumulate in TMEM).
//
// Replaces the reference's scalar `matmul` (proj/src/tensor.cpp:42-58) and the
// contractions inside `swiglu_ffn` (tensor.cpp:94-116) for every linear layer
// on the decode path; the epilogue folds bias, rate scaling, SiLU, SwiGLU,
// the residual add and the (mu, sigma) head activations.
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

namespace pswa_dev {

enum GemmAct : int {
  kActNone = 0,
  kActSilu = 1,
  kActSwiGLU = 2,  // columns interleaved (gate_j, up_j): out_j = silu(g)*u
  kActHead = 3,    // n < split: mu = (acc+b)*scale ; else sigma = 0.11+softplus(acc+b)
  kActTanhHalf = 4,  // 0.5 * tanh(acc * scale + b): the LRP output eps
};

struct GemmEpi {
  void* out = nullptr;
  int ld_out = 0;          // elements
  int out_f32 = 0;         // 0: fp16 output, 1: fp32 output
  int accumulate = 0;      // fp32 only: out += value (residual stream)
  const float* bias = nullptr;   // [N] (nullable)
  const float* scale = nullptr;  // [N] (nullable): v = acc*scale + bias
  int bias_first = 0;            // v = (acc + bias) * scale instead
  int act = kActNone;
  int split = 0;                 // kActHead: first sigma column
  const int* row_map = nullptr;  // nullable: output row = row_map[m] (< 0: skip)
  int n_store = 1 << 30;         // output columns >= n_store are not written
  // RMSNorm folded into the GEMMs around it (tensor.cpp:81-86):
  //  * producer (fp32 accumulate epilogue, the residual add): also writes an
  //    fp16 copy of each updated row and its sum of squares per 32-column
  //    chunk (fixed order, no atomics), the next norm's inputs;
  //  * consumer (A = that fp16 copy, gain folded into the packed weight):
  //    every output row is scaled by 1/sqrt(sum(ssq[m][0:parts]) / d + 1e-5)
  //    before bias / activation.
  __half* x16_out = nullptr;
  int ld_x16 = 0;
  float* ssq_out = nullptr;
  int ld_ssq = 0;
  const float* rms_ssq = nullptr;  // consumer: [M][ld_rms] partial sums of squares of A's rows
  int ld_rms = 0, rms_parts = 0;
  float rms_inv_d = 0.0f;
  int v8 = 0;  // set by gemm_plan: every output row segment is 32 B aligned (256-bit ld/st)
  int coalesce = 0;  // set by gemm_plan: stores go through the per-warp smem stage
  int tma_store = 0;  // set by gemm_plan: fp32 rows leave the stage by TMA (GemmPlan::to)
  int l2_prefetch = 0;  // set by gemm_plan: residual segments bulk-prefetched into L2 per tile
  // request: split K over a CTA pair (fp32 / fp16 outputs, N % 128 == 0):
  // every output is fl(P0 + P1) of the two halves' ascending sums, the same
  // for any M -- a layer must request it in every program that runs it
  int split_k = 0;
  // set by gemm_plan_conv3x3: A is the implicit im2col of an NHWC fp16 image
  // of this width (K block kb = tap kb / cb, channels 64 (kb % cb) ...),
  // loaded by TMA in im2col mode
  int conv_w = 0, conv_cb = 0;
  // Second fp16 output (fused projections sharing A, e.g. Q | K V): output
  // columns >= split_n go to out2[row_map2[m]][n - split_n] (split_n % BN == 0).
  void* out2 = nullptr;
  int ld_out2 = 0, split_n = 0;
  const int* row_map2 = nullptr;
  // debug (PSWA_GEMM_TRACE): per-CTA clock64 stamps of the kernel phases,
  // kGemmTraceSlots words per CTA, overwritten by every launch
  unsigned long long* trace = nullptr;
};
constexpr int kGemmTraceSlots = 16;
// Copies the stamps written since the previous call (n words) to host and
// clears them; false when tracing is off.
bool gemm_trace_read(unsigned long long* out, int n);
// Trace builds only: timing experiments of gemm_tc_kernel (1 = skip the
// MMAs, 2 = skip operand loads after the first pipeline round); results
// are garbage while set. No-op in production builds.
void gemm_set_experiment(int flags);

struct GemmPlan {
  CUtensorMap ta;
  CUtensorMap tb;
  int M = 0, N = 0, K = 0, BN = 0;
  int cluster = 1;  // 2: CTA pairs multicasting the shared B tile
  bool pair = false;  // cta_group::2 256 x 256 tiles (large M, N % 256 == 0)
  bool splitk = false;  // split-K CTA pairs, 128 x 128 tiles (GemmEpi::split_k)
  // fp32-output tiles of the persistent kernel stored by TMA from the
  // per-warp smem stage (rows contiguous: no row map); to = the output map,
  // 32 x 32 fp32 boxes, SWIZZLE_128B
  bool tma_store = false;
  CUtensorMap to;
  GemmEpi epi;
};

// A: [M rows][lda] fp16 (first K columns used); B: [N rows][ldb] fp16.
// K % 64 == 0, N % 64 == 0, lda/ldb multiples of 8.
void gemm_plan(GemmPlan* p, const __half* A, int lda, int M, const __half* B, int ldb, int N,
               int K, const GemmEpi& epi, int force_bn = 0);
void gemm_run(const GemmPlan& p, cudaStream_t stream);
// 3x3 convolution, zero padding 1, stride 1, as an implicit GEMM: A = the
// im2col patches of x (NHWC fp16 [h][w][c], c % 64 == 0) gathered by TMA in
// im2col mode -- never materialised -- in K order (ky, kx, c); B = the
// packed weights [N][9c]. Bitwise equal to gemm_plan over im2col3x3's
// patches of the same fp16 values.
void gemm_plan_conv3x3(GemmPlan* p, const __half* x, int h, int w, int c, const __half* B, int ldb, int N,
                       const GemmEpi& epi);

// A chain of dependent GEMMs in ONE persistent launch (the S1/S2 block
// tail: out-projection + residual -> SwiGLU gate|up -> down + residual -> the
// next block's Q|K|V). Job j+1 reads rows of job j's outputs: its 128-row
// block m starts as soon as every tile of block m of job j is stored
// (per-block completion counters in global memory, acquire/release), so the
// jobs overlap as a wavefront over the row blocks instead of draining the GPU
// between launches. Tiles are handed out by an atomic counter in chain order,
// so a tile only ever waits on tiles already taken by running CTAs (no
// deadlock whatever else shares the GPU). Every job uses BN = 128; per-output
// reduction order is that of gemm_run (ascending 64-wide K blocks), so the
// results are bitwise those of the separate launches.
constexpr int kChainMaxJobs = 4;
struct GemmChainPlan {
  int njobs = 0;
  GemmPlan job[kChainMaxJobs];
  unsigned* counters = nullptr;  // device, >= gemm_chain_counter_words(), zeroed once
  int ctr_stride = 0;            // row blocks per job slot
};
int gemm_chain_counter_words(int M);
// Adds a job (same M as the chain's first job); B K-major [N][ldb], N % 128 == 0.
void gemm_chain_add(GemmChainPlan* c, const __half* A, int lda, int M, const __half* B, int ldb, int N,
                    int K, const GemmEpi& epi);
void gemm_chain_run(const GemmChainPlan& c, cudaStream_t stream);

// TMA map of a frame K/V cache [slots][H][W][ld] fp16 for the attention halo
// loads: box = 32 channels (one head) x box_w x box_h x 1 slot, SWIZZLE_64B.
void make_kv_tmap(CUtensorMap* m, const __half* kv, int ld, int W, int H, int slots,
                  long slot_stride_rows, int box_w, int box_h);

// Number of kernel launches gemm_run issues (always 1); used by launch accounting.
constexpr int kGemmLaunches = 1;

}  // namespace pswa_dev
