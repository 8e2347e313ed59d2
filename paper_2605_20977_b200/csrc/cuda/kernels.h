// Launchers for the non-GEMM sm_100a kernels of the decode path.
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace pswa_dev {

// ---- rows: norms, casts, gathers (norm.cu) -------------------------------
// y[i] = rmsnorm(x[src ? src[i] : i]) per `group` columns, times gain, fp16.
// Matches tensor.cpp:81-86 (eps 1e-5) up to reduction order.
void rmsnorm_rows(const float* x, int ldx, const int* src_rows, int M, int d, int group,
                  const float* gain, __half* y, int ldy, cudaStream_t st);
// Inputs of a folded RMSNorm (see GemmEpi::rms_ssq) for M rows of x
// (gathered through src_rows when given): optional fp32 copy, fp16 copy and
// sums of squares per 32 columns. d % 128 == 0 or d % 32 == 0 (slow path).
void rms_prep(const float* x, int ldx, const int* src_rows, int M, int d, float* xcopy, int ldc,
              __half* x16, int ld16, float* ssq, int ld_ssq, cudaStream_t st);
// dst[i][0:n] = src[rows ? rows[i] : i][0:n] (fp32)
void gather_rows_f32(const float* src, int lds, const int* rows, int M, int n, float* dst,
                     int ldd, cudaStream_t st);
// dst[i][0:ncols] = half(yhat[rows[i]][c0 : c0+nc]), zero in [nc, ncols)
void yhat_rows_f16(const int32_t* yhat, int C, const int* rows, int M, int c0, int nc, __half* dst,
                   int ldd, int ncols, cudaStream_t st);
void f32_to_f16_rows(const float* src, int lds, int M, int n, __half* dst, int ldd, int ncols,
                     cudaStream_t st);
// Broadcast a vector into M rows (learned pad) or copy rows from a source.
// slot_src[k] >= 0 selects ring buffer ring[slot_src[k]], -1 the pad vector.
void fill_context_slots(const float* const* ring, const int* slot_src, const float* pad, int T,
                        int HW, int d, float* x, cudaStream_t st);
// frame [HW][C] int32 -> [C][HW] int32
void yhat_to_chw(const int32_t* src, int HW, int C, int32_t* dst, cudaStream_t st);
// channels [c0, c0 + nc) only: dst[c][p] = src[p][c]
void yhat_to_chw_cols(const int32_t* src, int HW, int C, int c0, int nc, int32_t* dst,
                      cudaStream_t st);
void yhat_from_chw(const int32_t* src, int HW, int C, int32_t* dst, cudaStream_t st);
void scatter_rows_f32(const float* src, int lds, const int* rows, int M, int n, float* dst,
                      int ldd, cudaStream_t st);
void scatter_rows_f16(const __half* src, int lds, const int* rows, int M, int n, __half* dst,
                      int ldd, cudaStream_t st);

// Band halo exchange: dst[pairs[i].y][0:ld] = src[pairs[i].x][0:ld]
// (fp16 rows, ld a multiple of 8). dst may be a peer device's buffer: the
// rows then travel as NVLink P2P stores straight into the neighbour's K/V
// cache, no staging copy.
void halo_push(const __half* src, __half* dst, int ld, const int2* pairs, int n, cudaStream_t st);
// Cross-process band chaining (one process per GPU): after a segment's
// pushes, increment the neighbours' mailbox counters (system scope); before
// the next segment, spin until every present neighbour has signalled as many
// times as this band has waited (wait_ctr, device-resident so captured
// graphs can be replayed). A wait longer than ~20 s sets status |= 8 and
// returns instead of hanging the device.
void band_signal(unsigned* to_up, unsigned* to_down, cudaStream_t st);
void band_wait(const unsigned* mbox, unsigned* wait_ctr, bool need_up, bool need_down, int* status,
               cudaStream_t st);

// ---- windowed attention (attention.cu) -----------------------------------
// Queries: rows of q (fp16, head h at columns h*hd), qinfo[i] = slot<<24 |
// y<<12 | x. Keys/values: kv rows (slot*kv_slot_stride + y*W + x), K at
// column h*hd, V at column d + h*hd. Window win_h x win_w (x win_t slots
// back when win_t > 0), out-of-bounds keys masked, mask: 0 none, 1 step <=,
// 2 step <. bias[h][taps]. Zero allowed keys
// -> zero output.
void window_attention(const __half* q, int ldq, const int32_t* qinfo, int Mq, const __half* kv,
                      int ldkv, int kv_slot_stride, int H, int W, int heads, int hd, int win_h,
                      int win_w, int win_t, int mask, int s, const float* bias, __half* out,
                      int ldo, cudaStream_t st);

// Tensor-core variant (attention_mma.cu) for head_dim 32 and 7x7 windows:
// warps of 8 queries, keys on the MMA's M side. Work is a list of CTA tiles,
// kAttnTileInts ints each: [0] halo top row, [1] halo left col, [2] halo
// rows, [3] query slot, [4] warps with queries, then per warp w at
// [8 + (2 + qw) w]: band origin (row, col) inside the halo and qw query rows
// of q / out (-1 = none). All warps of a launch share one band shape:
constexpr int kAttnTileInts = 8 + 10 * 16;
constexpr int kAttnMaxBandKeys = 144;
struct AttnShape {
  const int8_t* taps;   // [nbk][qw]: window tap (dy+3)*7+(dx+3) of (band key, query), -1 = excluded
  const int16_t* bkey;  // [nbk]: band key -> row << 8 | col relative to the band origin
  int nbk;              // band keys scanned (multiple of 16, <= kAttnMaxBandKeys; 0 = none)
  int H, W;             // key grid bounds (keys outside are masked)
  int qw = 8;           // queries per warp: 8, or 16 (two MMA N tiles; tiles hold 2 + 16 ints per warp)
};
bool window_attention_tiles_supported(int hd, int win_h, int win_w);
int window_attention_tiles_smem(int halo_keys, bool three_d);
void window_attention_tiles_init(int max_smem_bytes);
// Score-offset tables of one attention layer and band shape, built once from
// the layer's relative-position bias [heads][wt*49 or 49]: out[h][slot
// offset][band key][query] = log2(e) * bias of the tap, -inf where the
// window or mask excludes the pair. [heads][max(wt,1)][nbk][8] fp16 (the
// bias enters the fp32 score as its fp16 rounding, < 1e-3 relative).
void build_score_tables(const float* bias, int heads, int wt, AttnShape shape, __half* out,
                        cudaStream_t st);
// kv_map: make_kv_tmap() of the K/V cache (gemm.h); halos are staged by TMA.
void window_attention_tiles(const __half* q, int ldq, const int32_t* tiles, int ntiles,
                            int warps_per_tile, int halo_rows, int halo_width, AttnShape shape,
                            const CUtensorMap& kv_map, int heads, int wt, const __half* tables,
                            __half* out, int ldo, cudaStream_t st);

// ---- convolutions for the hyperprior (conv.cu) ---------------------------
// NHWC fp32 input [h][w][c] -> fp16 patches [oh*ow][kcols], K order
// (ky, kx, c), zero padding 1 for 3x3. up2: input is read at (y/2, x/2) of a
// half-resolution grid (nearest x2 folded into the addressing).
void im2col3x3(const float* x, int h, int w, int c, int stride, int up2, __half* out, int kcols,
               cudaStream_t st);
// out[y][x][:] = x[y/2][x/2][:] (fp32, NHWC; plus an fp16 copy when out16
// is given: the operand of the implicit-GEMM conv) or subsample x[2y][2x]
void upsample2_nhwc(const float* x, int h, int w, int c, float* out, cudaStream_t st, __half* out16 = nullptr);
void subsample2_nhwc(const float* x, int h, int w, int c, float* out, cudaStream_t st);
// z_hat [c][h][w] int32 -> NHWC fp32
void zhat_to_nhwc(const int32_t* z, int c, int hw, float* out, cudaStream_t st);
// NHWC fp32 -> rounded int32 [c][h][w] (half-to-even)
void round_to_zhat(const float* x, int c, int hw, int32_t* z, cudaStream_t st);

// ---- toy transform (toy.cu) ----------------------------
// rgb: [Hpx][Wpx][3] u8 (extents multiples of 8); y: [192][Hpx/8][Wpx/8].
void toy_analysis(const uint8_t* rgb, int Hpx, int Wpx, int rate, float* y, cudaStream_t st);
void toy_synthesis(const float* y, int Hpx, int Wpx, int rate, uint8_t* rgb, cudaStream_t st);

// ---- entropy coding (coder.cu) -------------------------------------------
constexpr int kScales = 64;
// Largest |y_hat| the codec accepts: the networks read y_hat as fp16 (exact
// integers up to 2^11). The encoder rejects larger values (status 16 ->
// PSWA_E_ARG); the decoder treats them as a corrupt stream.
constexpr int kYhatMax = 2048;
constexpr int kSyms = 257;  // v in [-127,127] + 2 escapes
// Builds the 64 scale entries and 64 x 258 cumulative tables on the device
// in fp64 with IEEE round-to-nearest ops only (bit-exact with the host rule),
// followed (at cdf + 64*258, 8-byte aligned) by 64 x 257 fp64 symbol costs
// and 64 x 257 uint16 search-index entries (entry b of a table: the symbol
// whose cumulative interval holds b * 256 in bits 0-14, bit 15 set when the
// symbols strictly between entries b and b + 1 all have frequency 1; the
// decoder's symbol search starts from the bucket of its target).
constexpr int kLutBuckets = 257;
constexpr size_t kCdfWords = static_cast<size_t>(kScales) * (kSyms + 1) + 2 * kScales * kSyms +
                             static_cast<size_t>(kScales) * kLutBuckets / 2;
// laplace = 1: discretised Laplace with scale b = sigma instead (same 64
// scales, same quantisation rule).
void build_cdf_tables(float* scales, uint32_t* cdf, cudaStream_t st, int laplace = 0);

struct LaneState {
  uint64_t code, range;  // decoder: code; encoder: low
  uint32_t pos, end;     // byte offsets into the payload
  double bits;           // estimated bits of this lane's symbols
};

// Optional per-symbol outputs of a phase (BitStats and the decoder's entropy
// parameters), all indexed like y_hat
// ([rows[k]][c0 + j]); null pointers disable them.
struct PhaseTaps {
  float* mu = nullptr;
  float* sigma = nullptr;
  double* bits = nullptr;  // -log2(freq / 2^16) + escape bits of the symbol
  int ymax = kYhatMax;     // decoded |y_hat| above this marks the stream corrupt
};

// Parses a lane payload header in device memory and initialises lane states.
// status[0] |= 1 on malformed payload.
void lanes_init(const uint8_t* payload, const uint32_t* len, int lanes, uint32_t expect_count,
                LaneState* st_lanes, int* status, cudaStream_t st);
// Decodes one phase of the main payload: symbols [o0, o0 + n*per) where
// ordinal o0 + k*per + j is channel c0 + j of batch position k. mu/sigma are
// read from musig[k][j] / musig[k][sig_off + j]; y_hat = v + rint(mu) is
// written to yhat[rows[k]][c0 + j] and to yhat16[k][c0 + j] (nullable).
void lanes_decode_phase(const uint8_t* payload, LaneState* lanes, int L, uint64_t o0, int n,
                        int per, const float* musig, int ldms, int sig_off, const float* scales,
                        const uint32_t* cdf, const int* rows, int32_t* yhat, int C, int c0,
                        __half* yhat16, int ld16, int* status, cudaStream_t st,
                        PhaseTaps taps = {});
// Hyper payload: ordinal i -> channel i / per_ch; mean/scale from the prior
// bank entry; writes z_hat [c][h][w].
void lanes_decode_hyper(const uint8_t* payload, LaneState* lanes, int L, int n, int per_ch,
                        const float* loc, const float* scale, const float* scales,
                        const uint32_t* cdf, int32_t* zhat, int* status, cudaStream_t st);
// Encoder side of one phase: v = y_hat - rint(mu), idx = scale_index(sigma)
// into sym_v / sym_idx at ordinals [o0, ...); also fills yhat16 from y_hat.
// taps.bits needs cdf (its symbol-cost table).
void quantize_phase(const float* musig, int ldms, int sig_off, int n, int per, uint64_t o0,
                    const int* rows, const int32_t* yhat, int C, int c0, const float* scales,
                    const uint32_t* cdf, int32_t* sym_v, uint8_t* sym_idx, __half* yhat16, int ld16,
                    PhaseTaps taps, int* status, cudaStream_t st);
// BitStats: out[g][i] = sum over the Cg channels of group g
// (ascending) of sym_bits[(row0 + i)][g*Cg + c], i in [0, npos).
void bitstats_reduce(const double* sym_bits, int C, int row0, int npos, int N, int Cg, double* out,
                     cudaStream_t st);
void quantize_hyper(const int32_t* zhat, int n, int per_ch, const float* loc, const float* scale,
                    const float* scales, int32_t* sym_v, uint8_t* sym_idx, cudaStream_t st);
// Encodes n symbols into L lanes: lane l writes at out + l*cap; lens[l]
// receives its length (or status |= 2 on overflow); bits[l] its estimate.
void lanes_encode(const int32_t* sym_v, const uint8_t* sym_idx, uint64_t n, int L,
                  const uint32_t* cdf, uint8_t* out, uint32_t cap, uint32_t* lens, double* bits,
                  int* status, cudaStream_t st);
// sticky |= status (frames decoded back to back without a host check).
void accumulate_status(const int* status, int* sticky, cudaStream_t st);
// Sum of per-lane bit estimates in lane order (deterministic).
void sum_lane_bits(const LaneState* lanes, int L, double* out, cudaStream_t st);
void sum_doubles(const double* v, int L, double* out, cudaStream_t st);
// Packs L encoded lanes (lane l at enc + l*cap, lens[l]) into the lane
// payload format; *total receives the payload size (device int64).
void lanes_pack(const uint8_t* enc, uint32_t cap, const uint32_t* lens, int L, uint32_t count,
                uint8_t* payload, uint64_t payload_cap, unsigned long long* total, uint64_t* offs,
                int* status, cudaStream_t st);

// ---- the reference's fp32 operator API, bit-exact (tensor_ops.cu) --------
void matmul_exact(const float* a, const float* b, float* c, int m, int k, int p, cudaStream_t st);
void softmax_rows_exact(const float* x, float* y, int m, int k, cudaStream_t st);
void rmsnorm_exact(const float* x, const float* g, int d, float* out, int rows, cudaStream_t st);
void swiglu_exact(const float* x, const float* wg, const float* wu, const float* wd, int d, int f,
                  float* h_scratch, float* out, cudaStream_t st);
void conv2d_exact(const float* x, int c, int h, int w, const float* k, int o, int kh, int kw, int stride,
                  int pad, float* y, cudaStream_t st);
void upsample2_chw(const float* x, int c, int h, int w, float* y, cudaStream_t st);

}  // namespace pswa_dev
