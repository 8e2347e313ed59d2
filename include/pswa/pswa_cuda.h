/*
 * pswa_cuda.h — the C-ABI drop-in boundary of the B200 P-SWA entropy decoder.
 *
 * Plain C: opaque handle, plain pointers and sizes, int status codes, no C++
 * or torch types, no exceptions across the boundary. A reference-side binding
 * (ctypes / cgo / JNI) needs nothing but this header; see INTEGRATION.md.
 *
 * Reference interfaces replaced (paths relative to the reference tree):
 *   pswa_gpu_decode_frame   <- decode_frame_wavefront(payloads, state, weights,
 *                              cfg, workers)
 *   pswa_gpu_encode_frame   <- encode_frame(y, state, weights, cfg, rate_idx)
 *                                                             SPEC.md:567-575
 *   pswa_gpu_forward_params <- the teacher-forced (mu, sigma) of predict_params
 *                              over a frame
 *   pswa_gpu_reset_gop / _push_frame <- FrameState ring update SPEC.md:304-308,
 *                              GOP reset
 *   pswa_gpu_op_*           <- per-operator entry points used by parity tests:
 *     op_gemm_f16      matmul                   proj/src/tensor.cpp:42-58
 *     op_rmsnorm       rmsnorm                  proj/src/tensor.cpp:81-86
 *     op_window_attn   swa2d / cross_windowed / swa3d_timecausal
 *     op_build_cdf     build_gaussian_cdf
 *     op_encode_symbols / op_decode_symbols     SPEC.md:457-465 (lane format)
 */
#ifndef PSWA_PSWA_CUDA_H_
#define PSWA_PSWA_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
enum {
  PSWA_OK = 0,
  PSWA_E_ARG = 1,       /* shape / argument error  (std::invalid_argument) */
  PSWA_E_TRUNCATED = 2, /* bitstream truncated or corrupt                   */
  PSWA_E_HASH = 3,      /* weights / config mismatch                         */
  PSWA_E_CUDA = 4,      /* CUDA runtime / driver error                       */
  PSWA_E_LANE = 5,      /* coder lane overrun                                */
  PSWA_E_INTERNAL = 6
};

/* Thread-local message for the last non-zero status on this thread. */
const char* pswa_gpu_last_error(void);

/* ---- configuration (ModelConfig) ---------------------- */
typedef struct pswa_cfg {
  int d_spatial;    /* d: 512 paper / 64 desk            */
  int heads;        /* h: 16                             */
  int ctx_blocks;   /* 8 / 2                             */
  int s1_blocks;    /* 8 / 2                             */
  int s2_blocks;    /* 8 / 2                             */
  int d_channel;    /* 1024 / 128                        */
  int ch_blocks;    /* 2                                 */
  int hyper_ch;     /* 128 / 32                          */
  int latent_ch;    /* C = 192                           */
  int s;            /* spatial steps, 4                  */
  int n_groups;     /* N channel groups, 4               */
  int win_h, win_w; /* spatial window 7x7                */
  int win_t;        /* temporal window 5                 */
  int ctx_slots;    /* past-frame ring length, 4         */
  int rate_points;  /* 4                                 */
  int height, width;/* latent grid H x W (multiples of 4) */
  int lanes;        /* main-payload coder lanes          */
  int hyper_lanes;  /* hyper-payload coder lanes         */
  int prior;        /* main-latent parameter head: 0 Gaussian,
                       1 Laplace with scale b = the head's sigma output
                       (north_star "Gaussian or Laplace parameter head");
                       the hyperprior stays Gaussian */
  int lrp_blocks;   /* LRP transformer blocks; 0 = no LRP
                       (eps = 0). Paper scale uses 4. */
} pswa_cfg;

/* Fill the paper (preset=1) or desk (preset=0) defaults for an H x W grid. */
void pswa_cfg_preset(pswa_cfg* cfg, int preset, int height, int width);

typedef struct pswa_gpu pswa_gpu;

/* ---- deterministic weights (gen_weights) --------------
 * Writes the PSWW blob for (cfg, seed) into buf (capacity cap). *len gets the
 * required size; call with buf == NULL to query it. */
int pswa_gen_weights(const pswa_cfg* cfg, uint64_t seed, void* buf, size_t cap, size_t* len);

/* Synthetic latent frame: y_hat[C][H][W] int32 for frame
 * `frame_idx` of GOP `gop`. */
int pswa_synth_latent(const pswa_cfg* cfg, int gop, int frame_idx, int32_t* yhat_out);
/* Frames 0..n_frames-1 of GOP `gop` in one pass: out[n_frames][C][H][W]. */
int pswa_synth_gop(const pswa_cfg* cfg, int gop, int n_frames, int32_t* out);

/* validate_schedule (proj/include/pswa/wavefront.h:54-66)
 * for plain-C callers: *ok = 1 when the (s, window, N) schedule is decodable
 * -- accumulator edges strictly backward, spatial-self edges never forward,
 * the canonical decode order a topological order of the symbol dependency
 * graph derived from the network's dataflow -- else 0 with the first
 * violation (nullable buffer of cap bytes). Host only. */
int pswa_validate_schedule(int h, int w, int s, int wh, int ww, int n_groups, int* ok,
                           int* sequential_steps, char* first_violation, size_t cap);

/* ---- handle lifecycle --------------------------------------------------- */
int pswa_gpu_create(int device, const pswa_cfg* cfg, const void* psww_blob, size_t blob_len,
                    pswa_gpu** out);
void pswa_gpu_destroy(pswa_gpu* h);
/* Reset the temporal ring to the learned pad (GOP boundary). */
int pswa_gpu_reset_gop(pswa_gpu* h);

/* ---- frame API (host buffers; copies inside) ---------------------------
 * payload layout and lane format: see DESIGN.md "Bitstream". */
int pswa_gpu_encode_frame(pswa_gpu* h, const int32_t* yhat, int rate_idx, int frame_idx_in_gop,
                          uint8_t* hyper_out, size_t hyper_cap, size_t* hyper_len,
                          uint8_t* main_out, size_t main_cap, size_t* main_len,
                          double* bits_out /* [2] = {hyper, main}, nullable */);
/* mu_out / sigma_out (nullable, [C][H][W]): the entropy parameters the
 * decoder itself computed for every symbol (the wavefront
 * decoder evaluates (mu, sigma) per phase); bitwise equal to the encoder's and
 * to pswa_gpu_forward_params on the same frame. Requesting them runs the
 * decode program variant with per-symbol taps (also fills BitStats). */
int pswa_gpu_decode_frame(pswa_gpu* h, const uint8_t* hyper, size_t hyper_len,
                          const uint8_t* main_payload, size_t main_len, int rate_idx,
                          int frame_idx_in_gop, int advance_state, int32_t* yhat_out,
                          float* mu_out /* nullable */, float* sigma_out /* nullable */,
                          double* bits_out /* [2], nullable */);
/* Teacher-forced entropy parameters for a known frame (parity probe).
 * zhat: [hyper_ch][H/4][W/4]; mu/sigma: [C][H][W]. */
int pswa_gpu_forward_params(pswa_gpu* h, const int32_t* yhat, const int32_t* zhat, int rate_idx,
                            int frame_idx_in_gop, float* mu_out, float* sigma_out,
                            double* bits_out /* [2], nullable */);
/* LRP transformer output eps [C][H][W] of the last frame
 * decoded or encoded by this handle (computed in the same frame program
 * when cfg.lrp_blocks > 0); the reconstruction input is y_hat + eps. */
int pswa_gpu_last_eps(pswa_gpu* h, float* eps_out);
/* BitStats. With stats on, every frame call (encode,
 * decode, forward_params) also computes per-position, per-group estimated
 * bits; pswa_gpu_last_bitstats returns those of the last such call as
 * [N][H][W] doubles (group g of position (y, x) at g*H*W + y*W + x; their sum
 * is the frame's main estimate, bits_out[1]). Calls with stats off leave no
 * BitStats (PSWA_E_ARG). Requesting mu/sigma implies stats for that call. */
int pswa_gpu_set_stats(pswa_gpu* h, int on);
int pswa_gpu_last_bitstats(pswa_gpu* h, double* bits_nhw);
/* Returns the z_hat the encoder produced for the last encode_frame call. */
int pswa_gpu_last_zhat(pswa_gpu* h, int32_t* zhat_out);
/* Append a decoded / known frame to the temporal ring. */
int pswa_gpu_push_frame(pswa_gpu* h, const int32_t* yhat, int rate_idx);

/* ---- device-resident variants (inputs already in HBM) ------------------ */
int pswa_gpu_decode_frame_device(pswa_gpu* h, const void* d_hyper, size_t hyper_len,
                                 const void* d_main, size_t main_len, int rate_idx,
                                 int frame_idx_in_gop, int advance_state, void* d_yhat_out);
/* Asynchronous variant: enqueues the decode on the handle's stream and
 * returns; handles on separate streams overlap on one GPU (independent GOPs,
 * BASELINE config 4). With advance_state the temporal ring takes the frame on
 * the stream, so a GOP is queued frame after frame (call reset_gop at GOP
 * starts). pswa_gpu_finish() waits, reports PSWA_E_TRUNCATED if ANY frame
 * queued since the previous finish failed, and the last frame's bits. */
int pswa_gpu_decode_frame_async(pswa_gpu* h, const void* d_hyper, size_t hyper_len,
                                const void* d_main, size_t main_len, int rate_idx,
                                int frame_idx_in_gop, int advance_state, void* d_yhat_out);
int pswa_gpu_finish(pswa_gpu* h, double* bits_out /* [2], nullable */);
/* Intermediate activations of the last forward_params call, for parity
 * triage: "ctx", "emb", "hq", "a" (fp32 / fp16 [H*W][d]) and "s1" (fp16, padded
 * hyper grid). *bytes gets the size; out may be NULL to query it. */
int pswa_gpu_debug_fetch(pswa_gpu* h, const char* name, void* out, size_t cap, size_t* bytes);
/* Number of kernels the last frame call launched (graph nodes included). */
int pswa_gpu_last_launch_count(pswa_gpu* h);
/* Replays one production launch of the last decode (warm, real operands)
 * `reps` times between CUDA events on the handle's stream: "ctx_attn",
 * "ctx_ffn_gu", "step_attn", "step_wq". us per launch and the launch's
 * algorithmic FLOPs (mask-allowed keys only) feed bench.py's roofline. */
int pswa_gpu_bench_op(pswa_gpu* h, const char* name, int reps, double* us_per_launch,
                      double* flops_per_launch);
/* Every probe of the handle's programs: one "name flops bytes launches" line
 * each (algorithmic FLOPs / HBM bytes per replay; probes are tagged when a
 * program is built, so decode a frame first). pswa_gpu_bench_probe replays
 * one like pswa_gpu_bench_op and also returns its bytes. tools/
 * profile_probes.py captures the same replays under ncu, so bench.py's
 * per-kernel rooflines and profiles/ describe the same launches. */
int pswa_gpu_probe_list(pswa_gpu* h, char* out, size_t cap, size_t* len);
int pswa_gpu_bench_probe(pswa_gpu* h, const char* name, int reps, double* us_per_replay,
                         double* flops, double* bytes);
/* Stream the handle runs on (cudaStream_t as void*). */
void* pswa_gpu_stream(pswa_gpu* h);

/* ---- sequences (encode_sequence / decode_sequence) -----
 * Container layout: FORMAT.md (header "PSWA", per-frame hyper + main
 * payloads). Frame f of the sequence has frame_idx_in_gop = f % gop_size and
 * the temporal ring resets at every GOP start. */
int pswa_gpu_encode_sequence(pswa_gpu* h, const int32_t* frames /* [F][C][H][W] */, int n_frames,
                             int gop_size, int rate_idx, uint8_t* out, size_t cap, size_t* len);
/* Decodes the whole frames present (a truncated tail frame is ignored).
 * A frame that fails (corrupt / truncated payload) gets its status code in
 * frame_status and decoding resumes at the next GOP boundary (frames in
 * between get -1); the call itself fails only on a bad header, a config or
 * weights hash mismatch (PSWA_E_HASH) or too small an output. */
int pswa_gpu_decode_sequence(pswa_gpu* h, const uint8_t* container, size_t len, int32_t* frames_out,
                             int max_frames, int* frame_status /* nullable [max_frames] */,
                             double* bits_out /* nullable [max_frames][2] */, int* n_frames);
/* Header fields: info[0..9] = version, W_px, H_px, frame_count, gop_size,
 * rate_idx, s, N, prior, whole frames present. Host only. */
int pswa_container_info(const uint8_t* container, size_t len, int* info);

/* ---- frames: PPM I/O and the toy transform --
 * Binary P6 only (P3 and maxval != 255 rejected). pswa_pad8 replicates the
 * edges up to multiples of 8. Analysis: per 8x8 patch and colour, the
 * orthonormal DCT-II of pixel - 128, channel = 3 * zigzag + colour, divided
 * by q[rate] = {8, 5, 3, 2}; y_hat = round-half-even(y). Synthesis inverts
 * it (y_rec = y_hat + eps), clamps to [0, 255] and rounds. On the current
 * device. rgb [H][W][3] u8, y [192][H/8][W/8] f32. */
int pswa_read_ppm(const char* path, uint8_t* rgb /* nullable: query size */, size_t cap, int* width,
                  int* height);
int pswa_write_ppm(const char* path, const uint8_t* rgb, int width, int height);
int pswa_pad8(const uint8_t* rgb, int height, int width, uint8_t* out /* nullable */, int* h8, int* w8);
int pswa_toy_analysis(const uint8_t* rgb, int h_px, int w_px, int rate_idx, float* y_out);
int pswa_toy_synthesis(const float* y, int h_px, int w_px, int rate_idx, uint8_t* rgb_out);

/* ---- row bands (BASELINE config 5) -----------------------
 * One frame decoded as n row bands, one device handle per band (bands may
 * share a device). Band b owns latent rows [row0, row1) (multiples of 4); its
 * halo K/V rows are pushed by the neighbours after every layer (P2P stores
 * over NVLink when they sit on different GPUs). Results are bitwise those of
 * the single-handle decode. The main payload is the banded container
 * "PSWB" | u32 n | u64 len[n] | band payloads, each band's symbols in the
 * canonical order restricted to its rows (band-local coder lanes); the hyper
 * payload is shared. Host frame buffers are full frames [C][H][W].
 * Replaces decode_frame_wavefront / encode_frame for a
 * frame too large for one device's wavefront, e.g. 4K (240x136 latents).  */
int pswa_band_rows(int height, int n_bands, int band_idx, int* row0, int* row1);

typedef struct pswa_group pswa_group;
int pswa_group_create(const int* devices, int n_bands, const pswa_cfg* cfg, const void* psww_blob,
                      size_t blob_len, pswa_group** out);
void pswa_group_destroy(pswa_group* g);
int pswa_group_reset_gop(pswa_group* g);
int pswa_group_push_frame(pswa_group* g, const int32_t* yhat, int rate_idx);
/* zhat: nullable (computed by the hyper encoder over the gathered S1). */
int pswa_group_encode_frame(pswa_group* g, const int32_t* yhat, const int32_t* zhat, int rate_idx,
                            int frame_idx_in_gop, uint8_t* hyper_out, size_t hyper_cap,
                            size_t* hyper_len, uint8_t* main_out, size_t main_cap, size_t* main_len,
                            double* bits_out /* [2], nullable */);
int pswa_group_decode_frame(pswa_group* g, const uint8_t* hyper, size_t hyper_len,
                            const uint8_t* main_payload, size_t main_len, int rate_idx,
                            int frame_idx_in_gop, int advance_state, int32_t* yhat_out,
                            double* bits_out /* [2], nullable */);
int pswa_group_forward_params(pswa_group* g, const int32_t* yhat, const int32_t* zhat, int rate_idx,
                              int frame_idx_in_gop, float* mu_out, float* sigma_out,
                              double* bits_out /* [2], nullable */);
int pswa_group_last_zhat(pswa_group* g, int32_t* zhat_out);
int pswa_group_last_launch_count(pswa_group* g);

/* One band per process (torchrun: rank r = band r on its own GPU). Create
 * the band handle, export its exchange buffers (CUDA-IPC handles, an opaque
 * blob), pass every band its neighbours' blobs (NULL at the frame edges),
 * then use the frame API above on the handle with the band's own payload of
 * the PSWB container. Segments are chained on the device by mailbox flags
 * (no host round trip per exchange). Encoding through band handles needs
 * z_hat (pswa_gpu_forward_params); produce banded bitstreams with a group. */
int pswa_gpu_create_band(int device, const pswa_cfg* cfg, const void* psww_blob, size_t blob_len,
                         int band_idx, int n_bands, pswa_gpu** out);
int pswa_gpu_band_export(pswa_gpu* h, void* out, size_t cap, size_t* len);
int pswa_gpu_band_link(pswa_gpu* h, const void* up_blob, size_t up_len, const void* down_blob,
                       size_t down_len);

/* ---- operator-level entry points (device pointers, on `stream`) -------- */
/* C[M,N] = A[M,K] . B[N,K]^T, fp16 in, fp32 accumulate; out fp16 or fp32.
 * force_bn: 0 automatic tile width; 64 / 128 / 256 forced; -1 CTA-pair
 * (cta_group::2) 256 x 256 tiles; -2 split-K CTA pairs (128 x 128 tiles, K
 * halves reduced through distributed shared memory). */
int pswa_gpu_op_gemm_f16(const void* A, int lda, int M, const void* B, int ldb, int N, int K,
                         void* C, int ldc, int out_f32, int accumulate, const float* bias,
                         const float* scale, int act, int force_bn, void* stream);
/* y = gain * x / sqrt(mean(x^2) + 1e-5), per group of `group` columns.
 * x fp32 [M][ld_x]; y fp16 [M][ld_y]. */
int pswa_gpu_op_rmsnorm(const float* x, int ld_x, int M, int d, int group, const float* gain,
                        void* y, int ld_y, void* stream);
/* Windowed masked attention; see DESIGN.md "Attention". */
int pswa_gpu_op_window_attn(const void* q, int ld_q, const int32_t* qinfo, int Mq,
                            const void* kv, int ld_kv, int kv_slot_stride, int H, int W,
                            int heads, int head_dim, int win_h, int win_w, int win_t, int mask,
                            int s, const float* bias, void* out, int ld_out, void* stream);
/* 64 cumulative tables x 258 u32, built on the device. */
int pswa_gpu_op_build_cdf(uint32_t* cdf_out /* host [64*258] */, float* scales_out /* [64] */);
/* laplace = 1: the Laplace tables of the prior = 1 parameter head. */
int pswa_gpu_op_build_cdf_family(uint32_t* cdf_out, float* scales_out, int laplace);
/* encode_symbols / decode_symbols on explicit symbols, host
 * buffers, through the production lane kernels: value v[i] (escapes up to
 * |v| < 2^31 - 128) under table idx[i] in [0, 64) of the Gaussian (laplace = 0)
 * or Laplace family; ordinal i in lane i % lanes; payload in the lane format
 * of DESIGN.md §3 (lanes = 1 is the SPEC's single stream). *len gets the
 * payload size (out may be NULL to query it); bits_out (nullable) the
 * estimate_bits of the symbols. Decoding a corrupt or
 * truncated payload returns PSWA_E_TRUNCATED. */
int pswa_gpu_op_encode_symbols(const int32_t* v, const int32_t* idx, size_t n, int lanes,
                               int laplace, uint8_t* out, size_t cap, size_t* len,
                               double* bits_out);
int pswa_gpu_op_decode_symbols(const uint8_t* payload, size_t len, const int32_t* idx, size_t n,
                               int laplace, int32_t* v_out, double* bits_out);

#ifdef __cplusplus
}
#endif

#endif /* PSWA_PSWA_CUDA_H_ */
