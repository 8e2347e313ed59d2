// The device engine behind the C ABI: owns every device allocation of one
// handle (packed fp16 weights, frame-indexed K/V caches, the temporal ring,
// coder lanes) and replays the per-frame programs as CUDA graphs.
//
// Decode of one frame as launched here:
//   hyper lanes -> z_hat -> hyper decoder (im2col + tcgen05 GEMMs) -> Hq
//   context transformer over the ring (dense, once per frame) -> ctx, cross K/V
//   for t in 0..s-1:
//     S1 for the step t-1 batch (incremental: per-layer K/V caches), acc K/V
//     accumulator + S2 for the step t batch
//     for g in 0..N-1: channel slot g -> mu/sigma heads -> lane decode
//     embed the decoded step t latents
// The encoder runs the decoder's exact per-batch kernels (teacher forced), so
// mu/sigma are bitwise identical on both sides.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <array>
#include <functional>
#include <map>
#include <string>
#include <vector>

#include "../cuda/gemm.h"
#include "../cuda/kernels.h"
#include "model_spec.h"

namespace pswa_host {

struct PW {  // packed weight: fp16 [N][K] row-major (K-major operand)
  __half* p = nullptr;
  int N = 0, K = 0;
};

struct Block {  // one transformer block of ctx / s1 / s2
  bool cross = false;
  PW wq, wkv, wo, wgu, wd;
  PW wqkv;  // [wq; wk; wv] stacked (self blocks): one GEMM, Q to the batch, K/V to the cache
  float *g1 = nullptr, *g2 = nullptr, *pos = nullptr;
  __half* kv_cache = nullptr;  // self layers of s1/s2: [HW][2d]; cross: ctx K/V
};

// Row band of a banded frame (BASELINE config 5). A band owns
// global latent rows [r0, r1) (multiples of 4) and keeps a local grid of rows
// [lo, lo + Hl): its own rows plus a halo of kHaloTop rows above (3 needed by
// the 7x7 window, 4 so that local row 0 keeps the global (y + x) mod 4 step
// pattern) and kHaloBottom below. Halo rows are never computed or coded
// locally; the neighbour pushes their K/V after every layer that produces them.
constexpr int kHaloTop = 4, kHaloBottom = 3, kHaloRows = 3;
struct Band {
  int idx = 0, n = 1;
  int r0 = 0, r1 = 0;       // own rows (global)
  int lo = 0, Hl = 0;       // local grid: global rows [lo, lo + Hl)
  int own0 = 0, nown = 0;   // own rows in local coordinates
};
// What a band needs to know about a neighbour: its local grid origin and the
// device addresses, valid in this process (same device, peer device, or a
// CUDA-IPC mapping of another process's memory), of its exchange buffers.
constexpr int kXids = 36;
struct PeerInfo {
  bool present = false;
  int lo = 0, HWl = 0;
  __half* buf[kXids] = {};
  __half* s1full = nullptr;
  unsigned* mbox = nullptr;  // [2] pushes received from above / below (IPC mode)
};
// Deterministic partition of H latent rows into n bands at multiples of 4.
void band_rows(int H, int n, int b, int* r0, int* r1);

// A program is a list of launches, split into segments at halo exchanges in
// band mode (a segment ends with the pushes into the neighbours' halos;
// `global` cuts wait for every band, not just the neighbours).
struct Cut {
  size_t at;
  bool global;
};
constexpr int kCutMainIn = -2;
struct Program {
  std::vector<std::function<void(cudaStream_t)>> ops;
  std::vector<Cut> cuts;
  // host-output decode (single band): cut k ends channel group copy_group[k]
  // of the last step (its CHW planes are final); kCutMainIn: the segment
  // after this cut reads the main payload (its H2D copy overlaps the first)
  std::vector<int> copy_group;
  int launches = 0;
  std::vector<cudaGraphExec_t> execs;  // one graph per segment
};

struct FrameResult {
  double bits[2] = {0, 0};
  int status = 0;
  size_t hyper_len = 0, main_len = 0;
};

class Engine {
 public:
  Engine(int device, const pswa_cfg& cfg, const void* blob, size_t len, int band_idx = 0,
         int n_bands = 1);
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  const Dims& dims() const { return D_; }
  cudaStream_t stream() const { return st_; }
  int last_launches() const { return last_launches_; }

  const Band& band() const { return B_; }
  int device() const { return device_; }

  // Host frame buffers are full-frame [C][H][W] (z_hat [hc][zh][zw]); a band
  // reads and writes only its own rows.
  void reset_gop();
  void push_frame(const int32_t* yhat_chw_host, int rate);
  // Encoder (teacher forced). zhat_in: nullable host [hc][zh][zw]; mu/sigma
  // nullable host [C][H][W]. Payloads are written to host buffers.
  FrameResult encode(const int32_t* yhat_chw_host, int rate, int fidx, const int32_t* zhat_in,
                     float* mu_out, float* sigma_out, uint8_t* hyper_out, size_t hyper_cap,
                     uint8_t* main_out, size_t main_cap, bool advance);
  // Decoder. Payloads and output either on the host (copies inside the call)
  // or already in device memory (device == true). mu/sigma (nullable, host
  // [C][H][W]) receive the decoder's own entropy parameters; requesting them
  // (or enabling stats) runs the "+ms" variant of the decode program, which
  // also produces BitStats.
  FrameResult decode(const void* hyper, size_t hyper_len, const void* main_pl, size_t main_len,
                     int rate, int fidx, bool advance, int32_t* yhat_out, bool device,
                     float* mu_out = nullptr, float* sigma_out = nullptr);
  // BitStats of every later frame call: per-position,
  // per-group estimated bits, read with last_bitstats().
  void set_stats(bool on) { stats_on_ = on; }
  // [N][H][W] (own rows of the full frame) of the last frame decoded or
  // encoded with stats on.
  void last_bitstats(double* out_nhw);
  void last_zhat(int32_t* out_host);
  // LRP output eps [C][H][W] of the last decoded / encoded frame (lrp_blocks > 0).
  void last_eps(float* out_chw);

  // ---- band mode (driven by BandGroup) ----------------------------------
  // Neighbours above / below (nullable) and band 0 (holder of the gathered
  // full-frame S1 for the hyper encoder). Peers may live on other devices
  // (peer access enabled by the group). Invalidates built programs.
  void link(Engine* up, Engine* down, Engine* band0);
  // Cross-process linking (one process per GPU): export this band's
  // exchange buffers as CUDA-IPC handles, then map the neighbours' blobs.
  // Segments are then chained inside one graph by device-side mailbox
  // flags (signal after the pushes, spin-wait before the next segment).
  std::vector<uint8_t> ipc_export();
  void link_ipc(const uint8_t* up, size_t up_len, const uint8_t* down, size_t down_len);
  // Split-phase frame API: prep_* stage inputs on the stream, the group runs
  // the program's segments on every band, finish_* collects the outputs.
  void prep_decode(const void* hyper, size_t hyper_len, const void* main_pl, size_t main_len,
                   int rate, int fidx, bool device, bool defer_main = false);
  FrameResult finish_decode(bool advance, int32_t* yhat_out, bool device, float* mu_out = nullptr,
                            float* sigma_out = nullptr);
  // decode program key: "+h" host-copy variant, "+ms" taps variant
  std::string decode_key(bool host_copy, bool taps) const {
    return std::string("decode") + (host_copy ? "+h" : "") + (taps ? "+ms" : "");
  }
  bool stats_on() const { return stats_on_; }
  // Asynchronous device-resident decode (no host sync; ring not advanced):
  // several handles on their own streams overlap on one GPU (GOP batches,
  // BASELINE config 4). finish_async() syncs and checks the status.
  // advance: the ring takes the frame (on the stream, no host sync), so a
  // whole GOP can be queued frame after frame. Statuses accumulate until
  // finish_async(), which reports any failure since the previous finish and
  // the last frame's bits.
  void decode_async(const void* d_hyper, size_t hyper_len, const void* d_main, size_t main_len,
                    int rate, int fidx, int32_t* d_yhat_out, bool advance = false);
  FrameResult finish_async();
  void prep_encode(const int32_t* yhat_chw_host, int rate, int fidx, const int32_t* zhat_in);
  FrameResult finish_encode(float* mu_out, float* sigma_out, uint8_t* hyper_out, size_t hyper_cap,
                            uint8_t* main_out, size_t main_cap, bool advance);
  std::string encode_key(bool zgiven, bool musig);
  void set_want_musig(bool on) { want_musig_ = on; }
  // Copies the payloads of the last finish_encode to host buffers (nullable).
  void fetch_payloads(uint8_t* hyper_out, size_t hyper_cap, const FrameResult& r, uint8_t* main_out);
  Program& program(const std::string& key);
  int segments(const Program& P) const { return static_cast<int>(P.cuts.size()) + 1; }
  bool cut_global(const Program& P, int k) const { return P.cuts[k].global; }
  void launch_segment(Program& P, int k);

  // Replays one production launch of the last-built decode program `reps`
  // times on the handle's stream between CUDA events (warm, real operands):
  // "ctx_attn" (context block 0 attention), "ctx_ffn_gu" (its SwiGLU gate|up
  // GEMM), "step_attn" / "step_wq" (S2 block 0, last step). Returns us per
  // launch; *flops = the algorithmic FLOPs of one launch.
  double bench_op(const std::string& name, int reps, double* flops, double* bytes = nullptr);
  // "name flops bytes launches" per line, every probe of the last-built programs
  std::string probe_list() const;
  // Debug taps (filled by forward_params): ctx, emb, hq, s1 (padded grid),
  // a, s2. Returns the byte size; copies when out != nullptr.
  size_t debug_fetch(const std::string& name, void* out, size_t cap);

 private:
  // ---- setup
  void alloc_all();
  void upload_weights(const WeightMap& w);
  void build_tables();
  template <class T>
  T* dalloc(size_t n);
  // ---- program building blocks
  void add(Program& P, std::function<void(cudaStream_t)> op, int launches = 1);
  // GEMM chains (gemm.h gemm_chain_*): while chaining_ is set, consecutive
  // gemm() calls are collected (each reads the previous one's identity-row
  // outputs: the S1/S2 block tail out-proj -> gate|up -> down -> next Q|K|V)
  // and emitted as one persistent launch when any other op is added, at 4
  // jobs, or by flush_chain(). A chain of one job stays a plain GEMM.
  bool chaining_ = false;
  struct OpenChain {
    pswa_dev::GemmChainPlan plan;
    std::vector<std::array<const void*, 4>> jobs;  // A, B, M (as pointer-size int), K for re-planning
    std::vector<int> lda, K;
    std::vector<PW> B;
    std::vector<pswa_dev::GemmEpi> epi;
    std::string tag;
    double flops = 0.0;
  } chain_;
  void flush_chain(Program& P);
  static bool chain_enabled();
  // alg_flops: the layer's algorithmic FLOPs when the packed operands are
  // padded (default 2 M N K of the padded GEMM)
  // 3x3 conv (padding 1) of an fp16 NHWC image as an implicit GEMM
  void conv(Program& P, const __half* x, int h, int w, const PW& B, const pswa_dev::GemmEpi& ep);
  bool implicit_conv() const;
  void gemm(Program& P, const __half* A, int lda, int M, const PW& B, int K,
            const pswa_dev::GemmEpi& ep, double alg_flops = -1.0);
  // every GEMM launch of the decode program being built, for the whole-class
  // probe "gemm_all" (the dominant kernel: ~2/3 of the frame's launch time)
  bool log_gemms_ = false;
  std::vector<std::function<void(cudaStream_t)>> gemm_log_;
  double gemm_log_flops_ = 0.0;
  struct StepBatch {  // positions of one wavefront step, or of all steps (encoder)
    int M = 0;
    const int* rows = nullptr;      // local raster index per batch row
    const int* rows_pad = nullptr;  // padded global hyper-grid index per row
    std::vector<std::array<int, 3>> parts;  // (step t, first row, rows)
    int xkind = 0;                  // band exchange kind: t or kXAll
  };
  StepBatch batch_of(int t) const;
  StepBatch batch_all() const;
  int* enc_rows_ = nullptr;      // all steps, canonical order (batch_all)
  int* enc_rows_pad_ = nullptr;
  void block_step(Program& P, const Block& b, const StepBatch& bt);
  void build_ctx(Program& P);
  void build_hyper_decode(Program& P);
  void build_hyper_encode(Program& P);
  void build_s1(Program& P, const StepBatch& bt, bool encoder);
  void build_step(Program& P, const StepBatch& bt, int mode /*0 decode, 1 encode*/);
  void build_acc_q_all(Program& P);
  void build_embed(Program& P, const StepBatch& bt);
  void run(Program& P);
  // decode program "decode+h": every segment in order, each finished channel
  // group's ŷ planes copied to the host on copy_ while later groups decode
  void run_host_copy(Program& P, int32_t* yhat_out);
  bool host_copy_ = false;  // set while the "+h" program is being built
  bool taps_ = false;       // set while a "+ms" program is being built
  pswa_dev::PhaseTaps phase_taps() const {
    pswa_dev::PhaseTaps t;
    if (taps_) t = {mu_full_, sg_full_, symbits_};
    return t;
  }
  void fetch_musig(float* mu_out, float* sigma_out);
  bool stats_on_ = false, have_stats_ = false;
  double* symbits_ = nullptr;   // [HWl][C] per-symbol bits ("+ms" programs)
  double* bitstats_ = nullptr;  // [N][HWo]
  cudaStream_t copy_ = nullptr;
  cudaEvent_t ev_copy_[8] = {}, ev_copy_done_ = nullptr, ev_main_in_ = nullptr;
  void to_side(Program& P, size_t from);
  void join_side(Program& P);
  cudaStream_t side_ = nullptr;
  cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr;
  // Registers the last op of P (or the last `nops` ops) as bench probe
  // `name` with its algorithmic FLOPs and HBM bytes per replay.
  void tag(Program& P, const std::string& name, double flops, double bytes = 0.0, int nops = 1);
  struct Probe {
    std::function<void(cudaStream_t)> op;
    double flops = 0.0, bytes = 0.0;
    int launches = 1;
  };
  double attn_flops(int t, int mask, int slots) const;  // t < 0: 3D over `slots` slots
  std::map<std::string, Probe> probes_;
  void set_frame_params(int rate, int fidx);
  void advance_ring();
  // band mode: push the halo rows of exchange buffer `id` (kind: step t in
  // 0..3, kAll, kCtx) into the neighbours and end the segment
  enum { kXAll = 16, kXCtx = 17 };
  enum { kXidAcc = 32, kXidCtx0 = 33, kXidCtx1 = 34, kXidCtx16 = 35 };
  int xid_of(const Block& b) const {
    return (&b >= s1_ && &b < s1_ + 16) ? static_cast<int>(&b - s1_) : 16 + static_cast<int>(&b - s2_);
  }
  void exchange(Program& P, int id, int kind);
  void cut(Program& P, bool global);
  __half* xbuf(int id);
  int xld(int id) const;
  void build_pairs();
  void copy_rows_in(int32_t* dst, const int32_t* src_full, int per_row_planes, bool device);

  Dims D_;
  Band B_;
  int HWl_ = 0, HWo_ = 0;  // local grid / own positions (== HW when unbanded)
  PeerInfo peer_[2];               // [0] band above, [1] band below
  PeerInfo self_info();
  __half* band0_s1_ = nullptr;     // band 0's full-frame S1 (encoder gather)
  bool ipc_ = false;
  unsigned *mbox_ = nullptr, *wait_ctr_ = nullptr;
  std::vector<void*> ipc_mapped_;
  int2* xpairs_[2][18] = {};  // [side: 0 up, 1 down][kind] (src local, dst peer-local) rows
  int nxpairs_[2][18] = {};
  int* ctx_kv_map_ = nullptr;  // own ctx rows -> local K/V rows (band mode)
  __half* ctx_kv2_ = nullptr;  // second context K/V buffer (band mode: layer parity)
  int device_ = 0;
  cudaStream_t st_ = nullptr;
  std::vector<void*> allocs_;
  std::map<std::string, Program> progs_;
  int last_launches_ = 0;

  // weights
  Block ctx_[16], s1_[16], s2_[16];
  float *ctx_gout_ = nullptr, *s1_gout_ = nullptr, *s2_gout_ = nullptr;
  PW emb_w_;
  float *emb_b_ = nullptr, *rate_in_ = nullptr, *rate_hyper_ = nullptr, *rate_out_ = nullptr;
  float* pad_ = nullptr;
  PW hd_c_[2][2], hd_out_, he_in_, he_c_[2][2];
  float *hd_b_[2][2] = {}, *hd_out_b_ = nullptr, *he_in_b_ = nullptr, *he_b_[2][2] = {};
  float *prior_loc_ = nullptr, *prior_scale_ = nullptr;
  Block acc_;
  PW ch_proj_, ch_emb_[8], ch_mix_[4], ch_gu_[4][8], ch_d_[4][8], head_w1_[8], head_w2_[8];
  float *ch_g1_[4] = {}, *ch_g2_[4] = {}, *ch_gout_ = nullptr;
  float *head_b1_[8] = {}, *head_b2_[8] = {};

  // per-frame parameters (device; set before each program launch)
  float *cur_rsi_ = nullptr, *cur_rsh_ = nullptr, *cur_rso_ = nullptr;
  float *cur_loc_ = nullptr, *cur_scale_ = nullptr;
  int* slot_src_ = nullptr;
  float** ring_ptrs_ = nullptr;
  std::vector<float*> ring_;
  int head_ = 0, npast_ = 0;

  // tables
  std::vector<std::vector<int>> step_rows_h_;
  int* step_rows_[16] = {};
  int* step_rows_pad_[16] = {};
  int32_t* step_qinfo_[16] = {};
  int32_t* ctx_qinfo_ = nullptr;
  // tensor-core attention work lists (warp tiles); empty when unsupported
  bool mma_attn_ = false;
  int32_t* step_tiles_[16] = {};
  int n_step_tiles_[16] = {};
  pswa_dev::AttnShape shape_ctx_{};
  std::map<std::pair<const float*, const pswa_dev::AttnShape*>, __half*> score_tables_;
  pswa_dev::AttnShape shape_step_[4][3] = {};  // [t][mask: none, <=, <]
  pswa_dev::GemmEpi rms_in(pswa_dev::GemmEpi e, const float* ssq) const;
  pswa_dev::GemmEpi ch_rms_out(pswa_dev::GemmEpi e) const;
  pswa_dev::GemmEpi ch_rms_in(pswa_dev::GemmEpi e) const;
  __half* chx16_ = nullptr;  // folded channel norms: fp16 slot copy [rows][sp]
  float* chssq_ = nullptr;   // and its sums of squares [rows][sp/32]
  float *bssq_ = nullptr, *ctx_ssq_ = nullptr;  // folded-RMSNorm sums of squares [rows][d/32]
  void attention(struct Program& P, const __half* q, const int32_t* qinfo, int Mq, const int32_t* tiles,
                 int ntiles, const pswa_dev::AttnShape* shape, const __half* kv, int slot_stride,
                 int wt, int mask, const float* bias, __half* out, int kv_slots = 0);
  struct Tiles3d {  // attention work of a 3D stack: all slots / last slot only
    const int32_t *all = nullptr, *last = nullptr, *qinfo = nullptr;
    int n_all = 0, n_last = 0;
  };
  Tiles3d tiles_ctx_, tiles_lrp_;
  void run_stack3d(Program& P, const Block* blocks, int nblocks, int S, const Tiles3d& tl,
                   bool exchange_kv, const char* probe);
  void build_lrp(Program& P);
  int c_lrp() const { return D_.c.lrp_blocks; }
  // LRP transformer
  Block lrp_[16];
  PW lrp_in_, lrp_head_;
  float *lrp_in_b_ = nullptr, *lrp_gout_ = nullptr, *lrp_head_b_ = nullptr;
  __half *lrp_cat_ = nullptr, *lrp16_ = nullptr;  // [HWl][N*sp + C] concat input; normed output
  float *eps_ = nullptr, *eps_chw_ = nullptr;      // [HWo][C], [C][HWo]
  int* crop_rows_ = nullptr;  // padded hyper grid index -> raster index (-1: pad)
  float* scales_ = nullptr;
  uint32_t* cdf_ = nullptr;
  uint32_t* cdf_main_ = nullptr;  // main-latent tables (== cdf_ for the Gaussian head)

  // frame buffers
  int32_t *yfr_ = nullptr, *ychw_ = nullptr, *zhat_ = nullptr;
  float *emb_cur_ = nullptr, *hq_ = nullptr;
  float *ctx_x_ = nullptr;
  __half *ctx_xn_ = nullptr, *ctx_kv_ = nullptr, *ctx_q_ = nullptr, *ctx_att_ = nullptr,
         *ctx_h_ = nullptr, *ctx16_ = nullptr;
  __half* acc_kv_ = nullptr;
  // hyper
  float *hx_ = nullptr, *hu_ = nullptr, *hh_ = nullptr;
  __half *hcol_ = nullptr, *hcast_ = nullptr, *s1full_ = nullptr;
  __half *hu16_ = nullptr, *hyh16_ = nullptr;  // hyper decoder conv operands (fp16 NHWC)
  // batch buffers
  int nmax_ = 0;
  float *bx_ = nullptr, *chx_ = nullptr, *musig_ = nullptr;
  // decoder: accumulator queries of every step (batch_all order), computed
  // from Hq on the side stream while the context transformer runs
  __half *qall_ = nullptr, *qall16_ = nullptr;
  float* qall_ssq_ = nullptr;
  __half *bxn_ = nullptr, *bq_ = nullptr, *batt_ = nullptr, *bh_ = nullptr, *bs1n_ = nullptr,
         *bs2n_ = nullptr, *y16_ = nullptr, *chxn_[4] = {}, *chh_ = nullptr,
         *chfo_ = nullptr, *hh16_ = nullptr;
  // coder
  uint8_t *d_hyper_ = nullptr, *d_main_ = nullptr;
  size_t hyper_cap_ = 0, main_cap_ = 0;
  uint32_t* d_lens_ = nullptr;  // [2] payload lengths (hyper, main)
  uint32_t lens_h_[2] = {0, 0};  // host staging of d_lens_ (stable address for async copies)
  pswa_dev::LaneState *lanes_ = nullptr, *hlanes_ = nullptr;
  int* status_ = nullptr;
  int* sticky_status_ = nullptr;  // async frames: statuses OR-ed until finish_async
  double* bits_ = nullptr;  // [2]
  int32_t *sym_v_ = nullptr, *hsym_v_ = nullptr;
  uint8_t *sym_idx_ = nullptr, *hsym_idx_ = nullptr;
  uint8_t *enc_lanes_ = nullptr, *enc_hlanes_ = nullptr;
  uint32_t enc_cap_ = 0, enc_hcap_ = 0;
  uint32_t *enc_lens_ = nullptr, *enc_hlens_ = nullptr;
  double *enc_bits_ = nullptr, *enc_hbits_ = nullptr;
  unsigned long long* pack_total_ = nullptr;  // [2]
  uint64_t* pack_offs_ = nullptr;
  float *mu_full_ = nullptr, *sg_full_ = nullptr;  // [HW][C] (forward_params)
  float* afull_ = nullptr;    // debug tap: accumulator output [HW][d]
  __half* s2full_ = nullptr;  // debug tap: S2 output [HW][d]
  bool want_musig_ = false;
};

}  // namespace pswa_host
