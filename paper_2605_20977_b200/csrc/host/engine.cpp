// Engine: weight packing, device buffers and the per-frame programs.
// See engine.h for the frame schedule; DESIGN.md for layouts and rooflines.
#include "engine.h"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <tuple>

#include "../cuda/check.h"
#include "abi_util.h"
#include "pswa/wavefront.h"

namespace pswa_host {

using pswa_dev::GemmEpi;
using pswa_dev::kActHead;
using pswa_dev::kActSilu;
using pswa_dev::kActSwiGLU;

namespace {

const HostTensor& W(const WeightMap& w, const std::string& n) {
  auto it = w.find(n);
  if (it == w.end()) throw std::invalid_argument("missing weight " + n);
  return it->second;
}

// Host-side fp16 packing: dst[(row_off + o) * ldk + col_off + i] = src[i][o]
// for a linear layer stored [in][out] (reference matmul convention). `gain`
// (nullable, [in]) folds a preceding RMSNorm gain into the weight:
// rmsnorm(x) . W = (x . diag(g) W) / rms(x), the 1/rms applied in the GEMM
// epilogue (GemmEpi::rms_ssq).
void put_linear(std::vector<__half>& dst, int ldk, const float* src, int in, int out, int row_off,
                int col_off, const float* gain = nullptr) {
  for (int o = 0; o < out; ++o)
    for (int i = 0; i < in; ++i)
      dst[static_cast<size_t>(row_off + o) * ldk + col_off + i] =
          __float2half_rn(src[static_cast<size_t>(i) * out + o] * (gain ? gain[i] : 1.0f));
}

// tensor-core attention CTA halos (8 warps each): context 4 x 16 queries,
// step batches 16 x 16 positions; +3 rows / columns of window margin
// halo widths 22 + pad columns: spread the ldmatrix rows over the banks
// under the TMA 64 B swizzle (see attention_mma.cu)
constexpr int kCtxHaloRows = 10, kCtxHaloW = 23;  // 2x4-query warps (default)
constexpr int kCtx16HaloRows = 14;                 // 4x4-query warps (PSWA_ATTN_Q16=1)
// 16 queries per context warp: correct (same tests), but 149 vs 118 us per
// context layer (127 registers, 2 CTAs per SM, 1.4x the scanned keys per
// query), 7.11 vs 6.90 ms per frame -- opt-in
bool ctx_q16() {
  static const bool on = std::getenv("PSWA_ATTN_Q16") != nullptr;
  return on;
}
int ctx_halo_rows() { return ctx_q16() ? kCtx16HaloRows : kCtxHaloRows; }
constexpr int kStepHaloRows = 22, kStepHaloW = 24;

// Step-t positions of the own rows of a band, as local raster indices, in
// raster order: the canonical symbol order restricted to the band.
std::vector<int> positions(const Band& b, int W, int s, int t) {
  std::vector<int> v;
  for (int y = b.r0; y < b.r1; ++y)
    for (int x = 0; x < W; ++x)
      if ((y + x) % s == t) v.push_back((y - b.lo) * W + x);
  return v;
}

}  // namespace

void band_rows(int H, int n, int b, int* r0, int* r1) {
  const int q = (H + 3) / 4;  // 4-row units
  if (n < 1 || b < 0 || b >= n || n > q) throw std::invalid_argument("band_rows: bad band split");
  *r0 = 4 * static_cast<int>(static_cast<long>(b) * q / n);
  *r1 = b == n - 1 ? H : 4 * static_cast<int>(static_cast<long>(b + 1) * q / n);
}

template <class T>
T* Engine::dalloc(size_t n) {
  void* p = nullptr;
  const size_t bytes = std::max<size_t>(n, 1) * sizeof(T);
  PSWA_CUDA(cudaMalloc(&p, bytes));
  PSWA_CUDA(cudaMemsetAsync(p, 0, bytes, st_));
  allocs_.push_back(p);
  return static_cast<T*>(p);
}

Engine::Engine(int device, const pswa_cfg& cfg, const void* blob, size_t len, int band_idx,
               int n_bands)
    : D_((validate_cfg(cfg), cfg)), device_(device) {
  if (D_.c.ctx_blocks > 16 || D_.c.s1_blocks > 16 || D_.c.s2_blocks > 16 || D_.c.s > 16 ||
      D_.N > 8 || D_.c.ch_blocks > 4)
    throw std::invalid_argument("pswa_cfg: block / group counts exceed engine limits");
  B_.idx = band_idx;
  B_.n = n_bands;
  band_rows(D_.H, n_bands, band_idx, &B_.r0, &B_.r1);
  if (n_bands > 1 && D_.c.lrp_blocks > 0)
    throw std::invalid_argument("band mode does not run the LRP transformer (lrp_blocks must be 0)");
  if (n_bands > 1 && (D_.c.s != 4 || D_.c.win_h != 7 || B_.r1 - B_.r0 < kHaloRows))
    throw std::invalid_argument("band mode needs s = 4, a 7-row window and >= 3 rows per band");
  B_.lo = n_bands > 1 ? std::max(0, B_.r0 - kHaloTop) : 0;
  B_.Hl = (n_bands > 1 ? std::min(D_.H, B_.r1 + kHaloBottom) : D_.H) - B_.lo;
  B_.own0 = B_.r0 - B_.lo;
  B_.nown = B_.r1 - B_.r0;
  HWl_ = B_.Hl * D_.W;
  HWo_ = B_.nown * D_.W;
  PSWA_CUDA(cudaSetDevice(device));
  PSWA_CUDA(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
  PSWA_CUDA(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking));
  PSWA_CUDA(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
  PSWA_CUDA(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming));
  PSWA_CUDA(cudaStreamCreateWithFlags(&copy_, cudaStreamNonBlocking));
  for (auto& e : ev_copy_) PSWA_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  PSWA_CUDA(cudaEventCreateWithFlags(&ev_copy_done_, cudaEventDisableTiming));
  PSWA_CUDA(cudaEventCreateWithFlags(&ev_main_in_, cudaEventDisableTiming));
  const WeightMap w = parse_psww(cfg, blob, len);
  build_tables();
  alloc_all();
  upload_weights(w);
  pswa_dev::build_cdf_tables(scales_, cdf_, st_);  // Gaussian (hyperprior, and main when prior = 0)
  {  // probe: the table build into scratch buffers (64 x 258 cumulative + costs + search index)
    float* ps = dalloc<float>(pswa_dev::kScales);
    uint32_t* pc = dalloc<uint32_t>(pswa_dev::kCdfWords);
    Probe pr;
    pr.op = [ps, pc](cudaStream_t s) { pswa_dev::build_cdf_tables(ps, pc, s); };
    pr.bytes = pswa_dev::kCdfWords * 4.0;
    probes_["cdf_build"] = pr;
  }
  if (D_.c.prior == 1) {
    float* tmp_scales = dalloc<float>(pswa_dev::kScales);
    cdf_main_ = dalloc<uint32_t>(pswa_dev::kCdfWords);
    pswa_dev::build_cdf_tables(tmp_scales, cdf_main_, st_, 1);
  } else {
    cdf_main_ = cdf_;
  }
  PSWA_CUDA(cudaStreamSynchronize(st_));
}

Engine::~Engine() {
  for (auto& kv : progs_)
    for (auto ex : kv.second.execs)
      if (ex) cudaGraphExecDestroy(ex);
  if (st_) cudaStreamSynchronize(st_);
  for (void* p : ipc_mapped_) cudaIpcCloseMemHandle(p);
  for (void* p : allocs_) cudaFree(p);
  if (ev_fork_) cudaEventDestroy(ev_fork_);
  if (ev_join_) cudaEventDestroy(ev_join_);
  for (auto& e : ev_copy_)
    if (e) cudaEventDestroy(e);
  if (ev_copy_done_) cudaEventDestroy(ev_copy_done_);
  if (ev_main_in_) cudaEventDestroy(ev_main_in_);
  if (copy_) cudaStreamDestroy(copy_);
  if (side_) cudaStreamDestroy(side_);
  if (st_) cudaStreamDestroy(st_);
}

// ------------------------------------------------------------- tables ----
void Engine::build_tables() {
  const Dims& D = D_;
  step_rows_h_.clear();
  nmax_ = 0;
  for (int t = 0; t < D.c.s; ++t) {
    step_rows_h_.push_back(positions(B_, D.W, D.c.s, t));
    nmax_ = std::max<int>(nmax_, static_cast<int>(step_rows_h_.back().size()));
  }
}

void Engine::alloc_all() {
  const Dims& D = D_;
  const int d = D.d, T = D.T, C = D.C;
  const int HWl = HWl_, HWo = HWo_, own0 = B_.own0;
  const size_t HWp = static_cast<size_t>(D.Hp) * D.Wp;
  const int L = D.c.lanes, Lz = D.c.hyper_lanes;
  auto up = [&](const std::vector<int>& v) {
    int* p = dalloc<int>(v.size());
    PSWA_CUDA(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(int), cudaMemcpyHostToDevice, st_));
    return p;
  };
  for (int t = 0; t < D.c.s; ++t) {
    const auto& r = step_rows_h_[t];
    std::vector<int> qi(r.size()), rp(r.size());
    for (size_t k = 0; k < r.size(); ++k) {
      const int y = r[k] / D.W, x = r[k] % D.W;  // local row
      qi[k] = (y << 12) | x;
      rp[k] = (y + B_.lo) * D.Wp + x;  // padded global hyper grid
    }
    step_rows_[t] = up(r);
    step_qinfo_[t] = up(qi);
    step_rows_pad_[t] = up(rp);
  }
  {  // all steps in canonical order (teacher-forced encoder batch)
    std::vector<int> r, rp;
    for (int t = 0; t < D.c.s; ++t)
      for (int v : step_rows_h_[t]) {
        r.push_back(v);
        rp.push_back((v / D.W + B_.lo) * D.Wp + v % D.W);
      }
    enc_rows_ = up(r);
    enc_rows_pad_ = up(rp);
  }
  {
    // 3D-stack queries: own rows of every slot, [S][HWo]; local coordinates
    // (S = T for the context transformer, T + 1 for the LRP transformer)
    const int Smax = T + (D.c.lrp_blocks > 0 ? 1 : 0);
    std::vector<int> qi(static_cast<size_t>(Smax) * HWo), km(static_cast<size_t>(T) * HWo);
    for (int j = 0; j < Smax; ++j)
      for (int p = 0; p < HWo; ++p) {
        qi[static_cast<size_t>(j) * HWo + p] = (j << 24) | ((own0 + p / D.W) << 12) | (p % D.W);
        if (j < T) km[static_cast<size_t>(j) * HWo + p] = j * HWl + own0 * D.W + p;
      }
    ctx_qinfo_ = up(qi);
    tiles_ctx_.qinfo = tiles_lrp_.qinfo = ctx_qinfo_;
    if (B_.n > 1) ctx_kv_map_ = up(km);
    // tap tables and aligned tiles assume s = 4 (4-row step blocks repeat the
    // same query / step pattern); other schedules use the SIMT kernel
    mma_attn_ = pswa_dev::window_attention_tiles_supported(D.hd, D.c.win_h, D.c.win_w) && D.c.s == 4;
    if (mma_attn_) {
      constexpr int TI = pswa_dev::kAttnTileInts;
      // context: CTA = 8 warps as 2 x 4 blocks of 2x4 queries (a 4 x 16
      // query rectangle of one slot), halo 10 rows x 23 columns; or
      // (PSWA_ATTN_Q16) 2 x 4 blocks of 4x4 queries (8 x 16), halo 14 x 23
      const bool q16 = ctx_q16();
      const int qh = q16 ? 4 : 2, qw = 2 * qh * 2;  // warp block qh x 4: 16 or 8 queries
      auto ctx_tiles = [&, q16, qh, qw](int slot_from, int row_base, int S) {
        std::vector<int> v;
        const int yend = own0 + B_.nown;
        // newest slot first: a slot-j tile walks min(j + 1, wt) key slots, so
        // the heaviest tiles are dispatched first and the launch tail is light
        for (int j = S - 1; j >= slot_from; --j)
          for (int y0 = own0; y0 < yend; y0 += 2 * qh)
            for (int x0 = 0; x0 < D.W; x0 += 16) {
              std::vector<int> t(TI, -1);
              t[0] = y0 - 3;
              t[1] = x0 - 3;
              t[2] = q16 ? kCtx16HaloRows : kCtxHaloRows;
              t[3] = j;
              t[4] = 8;
              for (int w = 0; w < 8; ++w) {
                const int wy = w / 4, wx = w % 4;
                int* W8 = &t[8 + (2 + qw) * w];
                W8[0] = qh * wy;
                W8[1] = 4 * wx;
                for (int i = 0; i < qw; ++i) {
                  const int y = y0 + qh * wy + i / 4, x = x0 + 4 * wx + i % 4;
                  W8[2 + i] = (y < yend && x < D.W) ? j * HWo + (y - own0) * D.W + x - row_base : -1;
                }
              }
              v.insert(v.end(), t.begin(), t.end());
            }
        return v;
      };
      auto make = [&](int S, Tiles3d& tl) {
        const auto all = ctx_tiles(0, 0, S), last = ctx_tiles(S - 1, (S - 1) * HWo, S);
        tl.n_all = static_cast<int>(all.size()) / TI;
        tl.n_last = static_cast<int>(last.size()) / TI;
        tl.all = up(all);
        tl.last = up(last);
      };
      make(T, tiles_ctx_);
      if (D.c.lrp_blocks > 0) make(T + 1, tiles_lrp_);
      // step batches: CTA = 8 warps as 4 x 2 blocks of 4x8 (a 16 x 16
      // rectangle); a warp owns the 8 step-t positions of its 4x8 block
      for (int t = 0; t < D.c.s; ++t) {
        std::vector<int> idx(static_cast<size_t>(HWl), -1);
        for (size_t k = 0; k < step_rows_h_[t].size(); ++k) idx[step_rows_h_[t][k]] = static_cast<int>(k);
        std::vector<int> v;
        // blocks stay anchored to global rows = 0 mod 4 (lo = 0 mod 4)
        for (int by = own0; by < own0 + B_.nown; by += 16)
          for (int bx = 0; bx < D.W; bx += 16) {
            std::vector<int> tt(TI, -1);
            tt[0] = by - 3;
            tt[1] = bx - 3;
            tt[2] = kStepHaloRows;
            tt[3] = 0;
            tt[4] = 8;
            int total = 0;
            for (int w = 0; w < 8; ++w) {
              const int wy = w / 2, wx = w % 2;
              int* W8 = &tt[8 + 10 * w];
              W8[0] = 4 * wy;
              W8[1] = 8 * wx;
              for (int i = 0; i < 8; ++i) {
                const int ry = i / 2, jj = i % 2;
                const int y = by + 4 * wy + ry;
                const int x = bx + 8 * wx + 4 * jj + ((t - ry) % 4 + 4) % 4;
                W8[2 + i] = -1;
                if (y < B_.Hl && x < D.W && idx[y * D.W + x] >= 0) {
                  W8[2 + i] = idx[y * D.W + x];
                  ++total;
                }
              }
            }
            if (total == 0) continue;
            v.insert(v.end(), tt.begin(), tt.end());
          }
        n_step_tiles_[t] = static_cast<int>(v.size()) / TI;
        step_tiles_[t] = up(v);
      }
      // band shapes: the keys a warp scans (band order) and their taps per
      // query, -1 where the window or the step mask excludes the pair (grid
      // bounds are applied in the kernel). Keys no query can use are dropped.
      {
        std::vector<int8_t> all_taps;
        std::vector<int16_t> all_keys;
        struct Pending { size_t tap_off, key_off; int nbk, qw; };
        auto add_shape = [&](std::vector<std::pair<int, int>> keys /* (row, col) in band */,
                             auto query_pos, int t, int mk, int nq) {
          std::vector<std::pair<int, int>> used;
          std::vector<int8_t> taps;
          for (auto [kr, kc] : keys) {
            int8_t row[16];
            bool any = false;
            for (int i = 0; i < nq; ++i) {
              const auto [qr, qc] = query_pos(i);
              const int dy = kr - qr, dx = kc - qc;
              row[i] = -1;
              if (dy < -3 || dy > 3 || dx < -3 || dx > 3) continue;
              // band origin = block origin - 3 and block origins are 0 mod 4:
              // band (r, c) has the step of (r + 1, c + 1)
              if (t >= 0 && mk > 0 &&
                  !pswa::mask_allows(mk == 1 ? pswa::MaskKind::kSpatialSelf : pswa::MaskKind::kAccumulator,
                                     pswa::Pos{qr + 1, qc + 1}, pswa::Pos{kr + 1, kc + 1}, 4))
                continue;
              row[i] = static_cast<int8_t>((dy + 3) * 7 + dx + 3);
              any = true;
            }
            if (!any) continue;
            used.push_back({kr, kc});
            taps.insert(taps.end(), row, row + nq);
          }
          while (used.size() % 16) {  // pad to whole 16-key chunks (all taps -1)
            used.push_back({0, 0});
            taps.insert(taps.end(), nq, int8_t(-1));
          }
          Pending p{all_taps.size(), all_keys.size(), static_cast<int>(used.size()), nq};
          all_taps.insert(all_taps.end(), taps.begin(), taps.end());
          for (auto [kr, kc] : used) all_keys.push_back(static_cast<int16_t>(kr << 8 | kc));
          return p;
        };
        // context: (qh + 6) x 10 band, column-major (conflict-free ldmatrix
        // with a 23-wide halo and the TMA 64 B swizzle); query i at
        // (3 + i/4, 3 + i%4)
        std::vector<std::pair<int, int>> ck;
        for (int c = 0; c < 10; ++c)
          for (int r = 0; r < qh + 6; ++r) ck.push_back({r, c});
        const Pending pc =
            add_shape(ck, [](int i) { return std::make_pair(3 + i / 4, 3 + i % 4); }, -1, 0, qw);
        // steps: 10 x 14 band sorted by step class, then row, column
        Pending ps[4][3];
        for (int t = 0; t < 4; ++t)
          for (int mk = 0; mk < 3; ++mk) {
            std::vector<std::tuple<int, int, int>> sk;
            for (int r = 0; r < 10; ++r)
              for (int c = 0; c < 14; ++c) sk.emplace_back(((r + c - 6) % 4 + 4) % 4, r, c);
            std::sort(sk.begin(), sk.end());
            std::vector<std::pair<int, int>> keys;
            for (auto [cls, r, c] : sk) keys.push_back({r, c});
            ps[t][mk] = add_shape(keys, [t](int i) {
              const int ry = i / 2, jj = i % 2;
              return std::make_pair(3 + ry, 3 + 4 * jj + ((t - ry) % 4 + 4) % 4);
            }, t, mk, 8);
          }
        int8_t* dt = dalloc<int8_t>(all_taps.size());
        int16_t* dk = dalloc<int16_t>(all_keys.size());
        PSWA_CUDA(cudaMemcpyAsync(dt, all_taps.data(), all_taps.size(), cudaMemcpyHostToDevice, st_));
        PSWA_CUDA(cudaMemcpyAsync(dk, all_keys.data(), all_keys.size() * 2, cudaMemcpyHostToDevice, st_));
        auto shape = [&](const Pending& p) {
          return pswa_dev::AttnShape{dt + p.tap_off, dk + p.key_off, p.nbk, B_.Hl, D.W, p.qw};
        };
        shape_ctx_ = shape(pc);
        for (int t = 0; t < 4; ++t)
          for (int mk = 0; mk < 3; ++mk) shape_step_[t][mk] = shape(ps[t][mk]);
      }
      pswa_dev::window_attention_tiles_init(
          std::max(pswa_dev::window_attention_tiles_smem(ctx_halo_rows() * kCtxHaloW, true),
                   pswa_dev::window_attention_tiles_smem(kStepHaloRows * kStepHaloW, false)));
    }
    std::vector<int> crop(HWp);
    for (int y = 0; y < D.Hp; ++y)
      for (int x = 0; x < D.Wp; ++x)  // padded global hyper grid -> own local rows
        crop[static_cast<size_t>(y) * D.Wp + x] =
            (y >= B_.r0 && y < B_.r1 && x < D.W) ? (y - B_.lo) * D.W + x : -1;
    crop_rows_ = up(crop);
  }
  mbox_ = dalloc<unsigned>(2);
  wait_ctr_ = dalloc<unsigned>(1);
  scales_ = dalloc<float>(pswa_dev::kScales);
  cdf_ = dalloc<uint32_t>(pswa_dev::kCdfWords);

  cur_rsi_ = dalloc<float>(d);
  cur_rsh_ = dalloc<float>(d);
  cur_rso_ = dalloc<float>(C);
  cur_loc_ = dalloc<float>(D.hc);
  cur_scale_ = dalloc<float>(D.hc);
  slot_src_ = dalloc<int>(T);
  ring_.clear();
  for (int j = 0; j < T; ++j) ring_.push_back(dalloc<float>(static_cast<size_t>(HWo) * d));
  ring_ptrs_ = dalloc<float*>(T);
  PSWA_CUDA(cudaMemcpyAsync(ring_ptrs_, ring_.data(), sizeof(float*) * T, cudaMemcpyHostToDevice, st_));

  yfr_ = dalloc<int32_t>(static_cast<size_t>(HWl) * C);
  ychw_ = dalloc<int32_t>(static_cast<size_t>(HWo) * C);
  zhat_ = dalloc<int32_t>(static_cast<size_t>(D.hc) * D.zh * D.zw);
  emb_cur_ = dalloc<float>(static_cast<size_t>(HWl) * d);
  hq_ = dalloc<float>(static_cast<size_t>(HWl) * d);
  // 3D-stack buffers hold S slots: T (context) or T + 1 (LRP transformer)
  const int Sx = T + (D.c.lrp_blocks > 0 ? 1 : 0);
  const size_t TH = static_cast<size_t>(Sx) * HWo, THl = static_cast<size_t>(Sx) * HWl;
  ctx_x_ = dalloc<float>(TH * d);
  ctx_xn_ = dalloc<__half>(TH * d);
  ctx_ssq_ = dalloc<float>(TH * (d / 32));
  ctx_kv_ = dalloc<__half>(THl * 2 * d);
  if (B_.n > 1) ctx_kv2_ = dalloc<__half>(THl * 2 * d);
  ctx_q_ = dalloc<__half>(TH * d);
  ctx_att_ = dalloc<__half>(TH * d);
  ctx_h_ = dalloc<__half>(TH * D.fp);
  ctx16_ = dalloc<__half>(static_cast<size_t>(HWl) * d);
  acc_kv_ = dalloc<__half>(static_cast<size_t>(HWl) * 2 * d);
  if (D.c.lrp_blocks > 0) {
    lrp_cat_ = dalloc<__half>(static_cast<size_t>(HWl) * (D.N * D.sp + C));
    lrp16_ = dalloc<__half>(static_cast<size_t>(HWo) * d);
    eps_ = dalloc<float>(static_cast<size_t>(HWo) * C);
    eps_chw_ = dalloc<float>(static_cast<size_t>(HWo) * C);
  }

  hx_ = dalloc<float>(HWp * D.hc);
  hu_ = dalloc<float>(HWp * D.hc);
  hh_ = dalloc<float>(HWp * D.hc);
  hcol_ = dalloc<__half>(HWp * D.kconv);
  hu16_ = dalloc<__half>(HWp * D.hc);  // implicit-GEMM conv operands (fp16 NHWC)
  hyh16_ = dalloc<__half>(HWp * D.hc);
  hcast_ = dalloc<__half>(HWp * D.hcp);
  s1full_ = dalloc<__half>(HWp * d);

  // batch buffers hold every own position: the encoder batches all steps
  const size_t nb = static_cast<size_t>(std::max(nmax_, HWo));
  bx_ = dalloc<float>(nb * d);
  bxn_ = dalloc<__half>(nb * d);
  bssq_ = dalloc<float>(nb * (d / 32));
  bq_ = dalloc<__half>(nb * d);
  qall_ = dalloc<__half>(static_cast<size_t>(HWo) * d);
  qall16_ = dalloc<__half>(static_cast<size_t>(HWo) * d);
  qall_ssq_ = dalloc<float>(static_cast<size_t>(HWo) * (d / 32));
  batt_ = dalloc<__half>(nb * d);
  bh_ = dalloc<__half>(nb * D.fp);
  bs1n_ = dalloc<__half>(nb * d);
  bs2n_ = dalloc<__half>(nb * d);
  y16_ = dalloc<__half>(nb * C);
  chx_ = dalloc<float>(nb * D.N * D.sp);
  for (int b = 0; b < D.c.ch_blocks; ++b) chxn_[b] = dalloc<__half>(nb * D.N * D.sp);
  chh_ = dalloc<__half>(nb * D.fgp);
  chfo_ = dalloc<__half>(nb * D.sp);
  chx16_ = dalloc<__half>(nb * D.sp);  // zero pad columns stay zero (never written)
  chssq_ = dalloc<float>(nb * (D.sp / 32));
  hh16_ = dalloc<__half>(nb * 2 * D.sp);
  const int ms = (2 * D.Cg + 63) / 64 * 64;
  musig_ = dalloc<float>(nb * ms);

  const size_t nsym = static_cast<size_t>(HWo) * C, nz = static_cast<size_t>(D.hc) * D.zh * D.zw;
  main_cap_ = 12 + 4ull * L + 6 * static_cast<size_t>(L) + 16 * nsym;
  hyper_cap_ = 12 + 4ull * Lz + 6 * static_cast<size_t>(Lz) + 16 * nz;
  // + 64 B: the decoder's byte reservoirs read up to 32 B past a lane's end
  d_main_ = dalloc<uint8_t>(main_cap_ + 64);
  d_hyper_ = dalloc<uint8_t>(hyper_cap_ + 64);
  d_lens_ = dalloc<uint32_t>(2);
  lanes_ = dalloc<pswa_dev::LaneState>(L);
  hlanes_ = dalloc<pswa_dev::LaneState>(Lz);
  status_ = dalloc<int>(1);
  sticky_status_ = dalloc<int>(1);
  bits_ = dalloc<double>(2);
  sym_v_ = dalloc<int32_t>(nsym);
  sym_idx_ = dalloc<uint8_t>(nsym);
  hsym_v_ = dalloc<int32_t>(nz);
  hsym_idx_ = dalloc<uint8_t>(nz);
  enc_cap_ = static_cast<uint32_t>(16 * ((nsym + L - 1) / L) + 16);
  enc_hcap_ = static_cast<uint32_t>(16 * ((nz + Lz - 1) / Lz) + 16);
  enc_lanes_ = dalloc<uint8_t>(static_cast<size_t>(enc_cap_) * L);
  enc_hlanes_ = dalloc<uint8_t>(static_cast<size_t>(enc_hcap_) * Lz);
  enc_lens_ = dalloc<uint32_t>(L);
  enc_hlens_ = dalloc<uint32_t>(Lz);
  enc_bits_ = dalloc<double>(L);
  enc_hbits_ = dalloc<double>(Lz);
  pack_total_ = dalloc<unsigned long long>(2);
  pack_offs_ = dalloc<uint64_t>(std::max(L, Lz));
  symbits_ = dalloc<double>(static_cast<size_t>(HWl) * C);
  bitstats_ = dalloc<double>(static_cast<size_t>(D.N) * HWo);
  mu_full_ = dalloc<float>(static_cast<size_t>(HWl) * C);
  sg_full_ = dalloc<float>(static_cast<size_t>(HWl) * C);
  afull_ = dalloc<float>(static_cast<size_t>(HWl) * d);
  s2full_ = dalloc<__half>(static_cast<size_t>(HWl) * d);
}

// ------------------------------------------------------------ weights ----
void Engine::upload_weights(const WeightMap& w) {
  const Dims& D = D_;
  const int d = D.d;
  auto upload_h = [&](const std::vector<__half>& v) {
    __half* p = dalloc<__half>(v.size());
    PSWA_CUDA(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(__half), cudaMemcpyHostToDevice, st_));
    return p;
  };
  auto upload_f = [&](const float* v, size_t n, size_t pad_to = 0) {
    float* p = dalloc<float>(std::max(n, pad_to));
    PSWA_CUDA(cudaMemcpyAsync(p, v, n * sizeof(float), cudaMemcpyHostToDevice, st_));
    return p;
  };
  auto fv = [&](const std::string& n) { return W(w, n).v.data(); };
  auto fsize = [&](const std::string& n) { return W(w, n).v.size(); };
  auto linear = [&](const std::string& n, int in, int out, int Np, int Kp, const float* gain = nullptr) {
    std::vector<__half> h(static_cast<size_t>(Np) * Kp, __float2half_rn(0.0f));
    put_linear(h, Kp, fv(n), in, out, 0, 0, gain);
    return PW{upload_h(h), Np, Kp};
  };
  auto qkv = [&](const std::string& q, const std::string& k, const std::string& v, const float* gain) {
    std::vector<__half> h(static_cast<size_t>(3 * d) * d, __float2half_rn(0.0f));
    put_linear(h, d, fv(q), d, d, 0, 0, gain);
    put_linear(h, d, fv(k), d, d, d, 0, gain);
    put_linear(h, d, fv(v), d, d, 2 * d, 0, gain);
    return PW{upload_h(h), 3 * d, d};
  };
  auto kv = [&](const std::string& k, const std::string& v, const float* gain = nullptr) {
    std::vector<__half> h(static_cast<size_t>(2 * d) * d, __float2half_rn(0.0f));
    put_linear(h, d, fv(k), d, d, 0, 0, gain);
    put_linear(h, d, fv(v), d, d, d, 0, gain);
    return PW{upload_h(h), 2 * d, d};
  };
  // SwiGLU gate/up interleaved by output column: rows 2j (gate), 2j+1 (up).
  auto gate_up = [&](const std::string& g, const std::string& u, int in, int f, int fp, int Kp,
                     const float* gain = nullptr) {
    std::vector<__half> h(static_cast<size_t>(2 * fp) * Kp, __float2half_rn(0.0f));
    const float* G = fv(g);
    const float* U = fv(u);
    for (int j = 0; j < f; ++j)
      for (int i = 0; i < in; ++i) {
        const float gi = gain ? gain[i] : 1.0f;
        h[static_cast<size_t>(2 * j) * Kp + i] = __float2half_rn(G[static_cast<size_t>(i) * f + j] * gi);
        h[static_cast<size_t>(2 * j + 1) * Kp + i] = __float2half_rn(U[static_cast<size_t>(i) * f + j] * gi);
      }
    return PW{upload_h(h), 2 * fp, Kp};
  };
  auto stack = [&](const char* tag, int blocks, Block* out, bool spatial) {
    for (int b = 0; b < blocks; ++b) {
      const std::string p = std::string(tag) + ".b" + std::to_string(b);
      Block& B = out[b];
      B.cross = spatial && (b % 2 == 1);
      // norm1 / norm2 gains folded into the projections they feed
      const float* g1 = fv(p + ".norm1.g");
      const float* g2 = fv(p + ".norm2.g");
      B.wq = linear(p + ".wq", d, d, d, d, g1);
      B.wkv = kv(p + ".wk", p + ".wv", g1);
      if (!B.cross) B.wqkv = qkv(p + ".wq", p + ".wk", p + ".wv", g1);
      B.wo = linear(p + ".wo", d, d, d, d);
      B.wgu = gate_up(p + ".ffn.wg", p + ".ffn.wu", d, D.f, D.fp, d, g2);
      B.wd = linear(p + ".ffn.wd", D.f, d, d, D.fp);
      B.g1 = upload_f(fv(p + ".norm1.g"), d);
      B.g2 = upload_f(fv(p + ".norm2.g"), d);
      B.pos = upload_f(fv(p + ".pos"), fsize(p + ".pos"));
      if (spatial) B.kv_cache = dalloc<__half>(static_cast<size_t>(HWl_) * 2 * d);
    }
  };
  stack("ctx", D.c.ctx_blocks, ctx_, false);
  stack("s1", D.c.s1_blocks, s1_, true);
  stack("s2", D.c.s2_blocks, s2_, true);
  ctx_gout_ = upload_f(fv("ctx.norm_out.g"), d);
  s1_gout_ = upload_f(fv("s1.norm_out.g"), d);
  s2_gout_ = upload_f(fv("s2.norm_out.g"), d);

  emb_w_ = linear("embed.w", D.C, d, d, D.C);
  emb_b_ = upload_f(fv("embed.b"), d);
  rate_in_ = upload_f(fv("rate.in"), fsize("rate.in"));
  rate_hyper_ = upload_f(fv("rate.hyper"), fsize("rate.hyper"));
  rate_out_ = upload_f(fv("rate.out"), fsize("rate.out"));
  pad_ = upload_f(fv("pad"), d);
  prior_loc_ = upload_f(fv("hyper.loc"), fsize("hyper.loc"));
  prior_scale_ = upload_f(fv("hyper.scale"), fsize("hyper.scale"));

  // conv weights [o][c][3][3] -> [o][(ky*3+kx)*c + ci]
  auto conv3 = [&](const std::string& n) {
    std::vector<__half> h(static_cast<size_t>(D.hcp) * D.kconv, __float2half_rn(0.0f));
    const float* k = fv(n);
    for (int o = 0; o < D.hc; ++o)
      for (int ci = 0; ci < D.hc; ++ci)
        for (int t = 0; t < 9; ++t)
          h[static_cast<size_t>(o) * D.kconv + t * D.hc + ci] =
              __float2half_rn(k[(static_cast<size_t>(o) * D.hc + ci) * 9 + t]);
    return PW{upload_h(h), D.hcp, D.kconv};
  };
  for (int j = 0; j < 2; ++j)
    for (int k = 0; k < 2; ++k) {
      const std::string hd = "hd.rb" + std::to_string(j) + ".c" + std::to_string(k + 1);
      const std::string he = "he.rb" + std::to_string(j) + ".c" + std::to_string(k + 1);
      hd_c_[j][k] = conv3(hd + ".w");
      hd_b_[j][k] = upload_f(fv(hd + ".b"), D.hc, D.hcp);
      he_c_[j][k] = conv3(he + ".w");
      he_b_[j][k] = upload_f(fv(he + ".b"), D.hc, D.hcp);
    }
  {
    std::vector<__half> h(static_cast<size_t>(d) * D.hcp, __float2half_rn(0.0f));
    const float* k = fv("hd.out.w");  // [d][hc]
    for (int o = 0; o < d; ++o)
      for (int ci = 0; ci < D.hc; ++ci)
        h[static_cast<size_t>(o) * D.hcp + ci] = __float2half_rn(k[static_cast<size_t>(o) * D.hc + ci]);
    hd_out_ = PW{upload_h(h), d, D.hcp};
    hd_out_b_ = upload_f(fv("hd.out.b"), d);
    std::vector<__half> e(static_cast<size_t>(D.hcp) * d, __float2half_rn(0.0f));
    const float* ki = fv("he.in.w");  // [hc][d]
    for (int o = 0; o < D.hc; ++o)
      for (int ci = 0; ci < d; ++ci)
        e[static_cast<size_t>(o) * d + ci] = __float2half_rn(ki[static_cast<size_t>(o) * d + ci]);
    he_in_ = PW{upload_h(e), D.hcp, d};
    he_in_b_ = upload_f(fv("he.in.b"), D.hc, D.hcp);
  }
  // accumulator
  acc_.wq = linear("acc.wq", d, d, d, d, fv("acc.normq.g"));  // normq gain folded
  acc_.wkv = kv("acc.wk", "acc.wv");
  acc_.wo = linear("acc.wo", d, d, d, d);
  acc_.g1 = upload_f(fv("acc.normq.g"), d);
  acc_.pos = upload_f(fv("acc.pos"), fsize("acc.pos"));

  // channel transformer, slots padded to sp columns
  const int N = D.N, sl = D.slot, sp = D.sp, dchp = N * sp;
  {
    std::vector<__half> h(static_cast<size_t>(dchp) * d, __float2half_rn(0.0f));
    for (int g = 0; g < N; ++g) put_linear(h, d, fv("ch.proj" + std::to_string(g) + ".w"), d, sl, g * sp, 0);
    ch_proj_ = PW{upload_h(h), dchp, d};
  }
  for (int g = 1; g < N; ++g) ch_emb_[g] = linear("ch.emb" + std::to_string(g) + ".w", D.Cg, sl, sp, D.Cgp);
  for (int b = 0; b < D.c.ch_blocks; ++b) {
    const std::string p = "ch.b" + std::to_string(b);
    std::vector<__half> h(static_cast<size_t>(dchp) * dchp, __float2half_rn(0.0f));
    const float* m = fv(p + ".mix.w");  // [in][out], masked block-lower-triangular
    for (int go = 0; go < N; ++go)
      for (int io = 0; io < sl; ++io)
        for (int gi = 0; gi <= go; ++gi)
          for (int ii = 0; ii < sl; ++ii)
            h[static_cast<size_t>(go * sp + io) * dchp + gi * sp + ii] =
                __float2half_rn(m[static_cast<size_t>(gi * sl + ii) * D.dch + go * sl + io]);
    ch_mix_[b] = PW{upload_h(h), dchp, dchp};
    ch_g1_[b] = upload_f(fv(p + ".norm1.g"), D.dch);
    ch_g2_[b] = upload_f(fv(p + ".norm2.g"), D.dch);
    for (int g = 0; g < N; ++g) {
      const std::string q = p + ".ffn" + std::to_string(g);
      // norm2 of slot g folded (its gain slice into the weight, 1/rms in the epilogue)
      ch_gu_[b][g] = gate_up(q + ".wg", q + ".wu", sl, D.fg, D.fgp, sp, fv(p + ".norm2.g") + g * sl);
      ch_d_[b][g] = linear(q + ".wd", D.fg, sl, sp, D.fgp);
    }
  }
  ch_gout_ = upload_f(fv("ch.norm_out.g"), D.dch);
  if (c_lrp() > 0) {
    stack("lrp", c_lrp(), lrp_, false);
    lrp_gout_ = upload_f(fv("lrp.norm_out.g"), d);
    // in_proj rows: the final channel representation (slot g at columns
    // g*sp, padded) then y_hat (C columns), matching lrp_cat_
    const int kcat = D.N * D.sp + D.C;
    std::vector<__half> h(static_cast<size_t>(d) * kcat, __float2half_rn(0.0f));
    const float* wi = fv("lrp.in.w");  // [dch + C][d]
    for (int o = 0; o < d; ++o) {
      for (int i = 0; i < D.dch; ++i)
        h[static_cast<size_t>(o) * kcat + (i / D.slot) * D.sp + i % D.slot] =
            __float2half_rn(wi[static_cast<size_t>(i) * d + o]);
      for (int i = 0; i < D.C; ++i)
        h[static_cast<size_t>(o) * kcat + D.N * D.sp + i] =
            __float2half_rn(wi[static_cast<size_t>(D.dch + i) * d + o]);
    }
    lrp_in_ = PW{upload_h(h), d, kcat};
    lrp_in_b_ = upload_f(fv("lrp.in.b"), d);
    lrp_head_ = linear("lrp.head.w", d, D.C, D.C, d);
    lrp_head_b_ = upload_f(fv("lrp.head.b"), D.C);
  }
  const int ms = (2 * D.Cg + 63) / 64 * 64;
  for (int g = 0; g < N; ++g) {
    const std::string mu = "head.mu" + std::to_string(g), sg = "head.sg" + std::to_string(g);
    std::vector<__half> h1(static_cast<size_t>(2 * sp) * sp, __float2half_rn(0.0f));
    // the final channel norm (slot g) is folded into head 1 unless the LRP
    // transformer needs the normalised representation itself
    const float* gout = c_lrp() > 0 ? nullptr : fv("ch.norm_out.g") + g * sl;
    put_linear(h1, sp, fv(mu + ".w1"), sl, sl, 0, 0, gout);
    put_linear(h1, sp, fv(sg + ".w1"), sl, sl, sp, 0, gout);
    head_w1_[g] = PW{upload_h(h1), 2 * sp, sp};
    std::vector<float> b1(static_cast<size_t>(2 * sp), 0.0f);
    std::memcpy(b1.data(), fv(mu + ".b1"), sizeof(float) * sl);
    std::memcpy(b1.data() + sp, fv(sg + ".b1"), sizeof(float) * sl);
    head_b1_[g] = upload_f(b1.data(), b1.size());
    std::vector<__half> h2(static_cast<size_t>(ms) * 2 * sp, __float2half_rn(0.0f));
    put_linear(h2, 2 * sp, fv(mu + ".w2"), sl, D.Cg, 0, 0);
    put_linear(h2, 2 * sp, fv(sg + ".w2"), sl, D.Cg, D.Cg, sp);
    head_w2_[g] = PW{upload_h(h2), ms, 2 * sp};
    std::vector<float> b2(static_cast<size_t>(ms), 0.0f);
    std::memcpy(b2.data(), fv(mu + ".b2"), sizeof(float) * D.Cg);
    std::memcpy(b2.data() + D.Cg, fv(sg + ".b2"), sizeof(float) * D.Cg);
    head_b2_[g] = upload_f(b2.data(), b2.size());
  }
}

// ----------------------------------------------------- program builders ---
void Engine::add(Program& P, std::function<void(cudaStream_t)> op, int launches) {
  flush_chain(P);
  P.ops.push_back(std::move(op));
  P.launches += launches;
}

void Engine::flush_chain(Program& P) {
  const int n = chain_.plan.njobs;
  if (n == 0) return;
  OpenChain c = std::move(chain_);
  chain_ = OpenChain{};
  if (n == 1) {  // a lone GEMM keeps its own tile-width choice
    const int M = static_cast<int>(reinterpret_cast<intptr_t>(c.jobs[0][2]));
    const bool was = chaining_;
    chaining_ = false;
    gemm(P, static_cast<const __half*>(c.jobs[0][0]), c.lda[0], M, c.B[0], c.K[0], c.epi[0]);
    chaining_ = was;
    if (!c.tag.empty()) tag(P, c.tag, c.flops);
    return;
  }
  pswa_dev::GemmChainPlan plan = c.plan;
  plan.counters = dalloc<unsigned>(pswa_dev::gemm_chain_counter_words(plan.job[0].M));
  P.ops.push_back([plan](cudaStream_t s) { pswa_dev::gemm_chain_run(plan, s); });
  P.launches += 1;
  if (!c.tag.empty()) {  // the whole launch is the probe: FLOPs of its (padded) GEMMs
    double fl = 0.0;
    for (int j = 0; j < n; ++j) fl += 2.0 * plan.job[j].M * plan.job[j].N * plan.job[j].K;
    const std::string base = c.tag.substr(0, c.tag.find('_'));
    tag(P, base + "_chain", fl);
  }
}

// Moves ops [from, end) onto the side stream: a fork (event record on the
// main stream, wait on the side stream) precedes them; join_side() later
// makes the main stream wait for the side stream. Both are capturable.
void Engine::to_side(Program& P, size_t from) {
  flush_chain(P);
  std::vector<std::function<void(cudaStream_t)>> moved(P.ops.begin() + from, P.ops.end());
  P.ops.resize(from);
  P.ops.push_back([this](cudaStream_t s) {
    PSWA_CUDA(cudaEventRecord(ev_fork_, s));
    PSWA_CUDA(cudaStreamWaitEvent(side_, ev_fork_, 0));
  });
  for (auto& op : moved) P.ops.push_back([op, this](cudaStream_t) { op(side_); });
}

void Engine::join_side(Program& P) {
  flush_chain(P);
  P.ops.push_back([this](cudaStream_t s) {
    PSWA_CUDA(cudaEventRecord(ev_join_, side_));
    PSWA_CUDA(cudaStreamWaitEvent(s, ev_join_, 0));
  });
}

void Engine::gemm(Program& P, const __half* A, int lda, int M, const PW& B, int K, const GemmEpi& ep,
                  double alg_flops) {
  if (chaining_ && B.N % 128 == 0 && ep.act != pswa_dev::kActTanhHalf) {
    if (chain_.plan.njobs == pswa_dev::kChainMaxJobs ||
        (chain_.plan.njobs > 0 && chain_.plan.job[0].M != M))
      flush_chain(P);
    pswa_dev::gemm_chain_add(&chain_.plan, A, lda, M, B.p, B.K, B.N, K, ep);
    chain_.jobs.push_back({A, B.p, reinterpret_cast<const void*>(static_cast<intptr_t>(M)), nullptr});
    chain_.lda.push_back(lda);
    chain_.K.push_back(K);
    chain_.B.push_back(B);
    chain_.epi.push_back(ep);
    return;
  }
  flush_chain(P);
  pswa_dev::GemmPlan plan;
  pswa_dev::gemm_plan(&plan, A, lda, M, B.p, B.K, B.N, K, ep);
  auto op = [plan](cudaStream_t s) { pswa_dev::gemm_run(plan, s); };
  add(P, op);
  if (log_gemms_) {
    gemm_log_.push_back(op);
    gemm_log_flops_ += alg_flops >= 0.0 ? alg_flops : 2.0 * M * B.N * K;
  }
}

namespace {
GemmEpi f16_out(void* out, int ld) {
  GemmEpi e;
  e.out = out;
  e.ld_out = ld;
  return e;
}
GemmEpi f32_acc(void* out, int ld, int n_store = 1 << 30) {
  GemmEpi e;
  e.out = out;
  e.ld_out = ld;
  e.out_f32 = 1;
  e.accumulate = 1;
  e.n_store = n_store;
  return e;
}
// Split-K CTA pairs (GemmEpi::split_k) for a layer: requested in every program
// (encoder, decoder, teacher-forced) so all of them reduce in the same
// order; off when the opt-in GEMM chains run those layers (their tiles never
// split) so the chained and unchained programs of a process still agree.
GemmEpi split_k(GemmEpi e, bool on) {
  e.split_k = on ? 1 : 0;
  return e;
}
// folded RMSNorm (GemmEpi::rms_ssq): producer / consumer sides
GemmEpi rms_out(GemmEpi e, __half* x16, float* ssq) {
  e.x16_out = x16;
  e.ld_x16 = e.ld_out;
  e.ssq_out = ssq;
  e.ld_ssq = e.ld_out / 32;
  return e;
}
GemmEpi swiglu_out(void* out, int ld) {
  GemmEpi e;
  e.out = out;
  e.ld_out = ld;
  e.act = kActSwiGLU;
  return e;
}
}  // namespace

// Opt-in (PSWA_CHAIN=1): correct and bitwise equal to the separate launches
// (tests pass either way), but measured slower on B200 -- one S2 block tail +
// next Q|K|V as one chain took 47.6 us against 35.6 us for the four tuned
// launches (BN 256 for the wide gate|up and Q|K|V GEMMs halves their
// activation re-reads; PDL already hides the launch gaps), 8.21 vs 7.26 ms
// per frame.
bool Engine::chain_enabled() {
  static const bool on = std::getenv("PSWA_CHAIN") != nullptr;
  return on;
}

// Folded RMSNorm of channel slot g (sl real columns of sp): the residual
// epilogue writes the updated slot's fp16 copy to chx16_ [M][sp] and its
// per-32-column sums of squares to chssq_ [M][sp/32]; the consumer reads them.
GemmEpi Engine::ch_rms_out(GemmEpi e) const {
  e.x16_out = chx16_;
  e.ld_x16 = D_.sp;
  e.ssq_out = chssq_;
  e.ld_ssq = D_.sp / 32;
  return e;
}

GemmEpi Engine::ch_rms_in(GemmEpi e) const {
  e.rms_ssq = chssq_;
  e.ld_rms = D_.sp / 32;
  e.rms_parts = D_.slot / 32;
  e.rms_inv_d = 1.0f / static_cast<float>(D_.slot);
  return e;
}

GemmEpi Engine::rms_in(GemmEpi e, const float* ssq) const {
  e.rms_ssq = ssq;
  e.ld_rms = D_.d / 32;
  e.rms_parts = D_.d / 32;
  e.rms_inv_d = 1.0f / static_cast<float>(D_.d);
  return e;
}

// Windowed attention: tensor-core warp tiles when the shape allows
// (head_dim 32, 7x7), the SIMT kernel otherwise (desk preset, head_dim 4).
void Engine::attention(Program& P, const __half* q, const int32_t* qinfo, int Mq,
                       const int32_t* tiles, int ntiles, const pswa_dev::AttnShape* shape,
                       const __half* kv, int slot_stride, int wt, int mask, const float* bias,
                       __half* out, int kv_slots) {
  const Dims& D = D_;
  const int d = D.d, Hl = B_.Hl;  // key grid bounds: the band's local grid
  if (mma_attn_ && shape->nbk == 0) {
    // the mask allows no key (the accumulator at step 0): the
    // kernel would stage halos only to write zeros; a memset writes the same
    // +0 halves
    add(P, [=](cudaStream_t s) {
      PSWA_CUDA(cudaMemsetAsync(out, 0, static_cast<size_t>(Mq) * d * sizeof(__half), s));
    }, 0);
  } else if (mma_attn_) {
    const pswa_dev::AttnShape sh = *shape;
    const int hr = wt > 0 ? ctx_halo_rows() : kStepHaloRows, hw = wt > 0 ? kCtxHaloW : kStepHaloW;
    CUtensorMap map;  // halo boxes of this K/V buffer: 32 channels x hw x hr x 1 slot
    pswa_dev::make_kv_tmap(&map, kv, 2 * d, D.W, Hl, wt > 0 ? (kv_slots > 0 ? kv_slots : D.T) : 1,
                           slot_stride > 0 ? slot_stride : HWl_,
                           hw, hr);
    // score-offset tables of (layer bias, band shape): built once, reused by
    // every program that launches this layer on this shape
    __half*& tab = score_tables_[{bias, shape}];
    if (!tab && sh.nbk > 0) {
      tab = dalloc<__half>(static_cast<size_t>(D.heads) * std::max(wt, 1) * sh.nbk * sh.qw);
      pswa_dev::build_score_tables(bias, D.heads, wt, sh, tab, st_);
    }
    const __half* tables = tab;
    add(P, [=](cudaStream_t s) {
      pswa_dev::window_attention_tiles(q, d, tiles, ntiles, 8, hr, hw, sh, map, D.heads, wt, tables,
                                       out, d, s);
    });
  } else {
    add(P, [=](cudaStream_t s) {
      pswa_dev::window_attention(q, d, qinfo, Mq, kv, 2 * d, slot_stride, Hl, D.W, D.heads, D.hd,
                                 D.c.win_h, D.c.win_w, wt, mask, D.c.s, bias, out, d, s);
    });
  }
}

// A batch of wavefront-step positions: one step (the decoder's phases) or
// every step concatenated in canonical order (the teacher-forced encoder:
// the same per-position kernels with one GEMM per layer instead of s; the
// attention stays one launch per step, on that step's slice, so every query
// sees exactly the decoder's tiles and masks and mu/sigma stay bitwise
// equal).
Engine::StepBatch Engine::batch_of(int t) const {
  StepBatch b;
  b.M = static_cast<int>(step_rows_h_[t].size());
  b.rows = step_rows_[t];
  b.rows_pad = step_rows_pad_[t];
  b.parts.push_back({t, 0, b.M});
  b.xkind = t;
  return b;
}

Engine::StepBatch Engine::batch_all() const {
  StepBatch b;
  b.rows = enc_rows_;
  b.rows_pad = enc_rows_pad_;
  for (int t = 0; t < D_.c.s; ++t) {
    const int n = static_cast<int>(step_rows_h_[t].size());
    b.parts.push_back({t, b.M, n});
    b.M += n;
  }
  b.xkind = kXAll;
  return b;
}

// One S1/S2 block on the batch held in bx_ (residual stream, fp32).
void Engine::block_step(Program& P, const Block& B, const StepBatch& bt) {
  const Dims& D = D_;
  const int d = D.d, M = bt.M;
  const int* rows = bt.rows;
  // norm1 is folded: bxn_ holds the fp16 residual stream and bssq_ its
  // sums of squares (from the previous residual GEMM or rms_prep)
  const bool probe = &B == &s2_[0] && bt.parts.size() == 1 && bt.parts[0][0] == D.c.s - 1;
  if (!B.cross) {
    // one GEMM for Q | K V: Q rows to the batch, K/V of these positions into
    // the frame cache (row map)
    GemmEpi e = rms_in(f16_out(bq_, d), bssq_);
    e.out2 = B.kv_cache;
    e.ld_out2 = 2 * d;
    e.split_n = d;
    e.row_map2 = rows;
    gemm(P, bxn_, d, M, B.wqkv, d, e);
    if (probe) tag(P, "step_wq", 2.0 * M * 3.0 * d * d);
    exchange(P, xid_of(B), bt.xkind);  // band mode: new K/V of the boundary rows
  } else {
    gemm(P, bxn_, d, M, B.wq, d, rms_in(f16_out(bq_, d), bssq_));
  }
  const int mk = B.cross ? 0 : 1;
  for (const auto& pt : bt.parts) {
    const int t = pt[0], off = pt[1], n = pt[2];
    attention(P, bq_ + static_cast<size_t>(off) * d, step_qinfo_[t], n, step_tiles_[t], n_step_tiles_[t],
              &shape_step_[t][mk], B.kv_cache, 0, 0, mk, B.pos, batt_ + static_cast<size_t>(off) * d);
    if (probe) tag(P, "step_attn", attn_flops(t, mk, 1));
  }
  gemm(P, batt_, d, M, B.wo, d, rms_out(f32_acc(bx_, d), bxn_, bssq_));  // + norm2 inputs
  if (probe) tag(P, "step_wo", 2.0 * M * d * d);
  gemm(P, bxn_, d, M, B.wgu, d, rms_in(swiglu_out(bh_, D.fp), bssq_), 2.0 * M * 2.0 * D.f * d);
  if (probe) tag(P, "step_gu", 2.0 * M * 2.0 * D.f * d);
  // the down projection (K = 1408 at paper scale) splits K over CTA pairs:
  // 9.6 vs 10.8 us per launch; the K <= 768 residual GEMMs measured slower
  // split (the partial-sum exchange outweighs the halved operand stream)
  gemm(P, bh_, D.fp, M, B.wd, D.fp, split_k(rms_out(f32_acc(bx_, d), bxn_, bssq_), !chain_enabled()),
       2.0 * M * d * D.f);
  if (probe) tag(P, "step_wd", 2.0 * M * D.f * d);
}

// Blocks of time-causal 3D SWA over S slots of own rows held in ctx_x_
// (inputs) with the norm1 inputs of block 0 already in ctx_xn_/ctx_ssq_; the
// last block computes the queries of the last slot only. Used by the context
// transformer (S = T) and the LRP transformer (S = T + 1).
void Engine::run_stack3d(Program& P, const Block* blocks, int nblocks, int S, const Tiles3d& tl,
                         bool exchange_kv, const char* probe) {
  const Dims& D = D_;
  const int d = D.d, HWo = HWo_, n = S * HWo;
  for (int b = 0; b < nblocks; ++b) {
    const Block& B = blocks[b];
    const bool last = b == nblocks - 1;
    const int q0 = last ? (S - 1) * HWo : 0, nq = n - q0;
    const float* pos = B.pos;
    // band mode: K/V of the own rows into the local [S][HWl] grid, the halo
    // rows pushed by the neighbours; buffers alternate by layer so a
    // neighbour's push of layer b+1 never lands in the buffer read by layer b
    __half* kv = (B_.n > 1 && b % 2) ? ctx_kv2_ : ctx_kv_;
    float* ssq_q = ctx_ssq_ + static_cast<size_t>(q0) * (d / 32);
    if (!last) {  // Q | K V in one GEMM over all slots
      GemmEpi e = rms_in(f16_out(ctx_q_, d), ctx_ssq_);
      e.out2 = kv;
      e.ld_out2 = 2 * d;
      e.split_n = d;
      e.row_map2 = ctx_kv_map_;
      gemm(P, ctx_xn_, d, n, B.wqkv, d, e);
      if (b == 0 && probe) tag(P, std::string(probe) + "_wqkv", 2.0 * n * 3.0 * d * d);
      if (exchange_kv) exchange(P, b % 2 ? kXidCtx1 : kXidCtx0, kXCtx);
    } else {  // last block: K/V of every slot, queries of the last slot only
      GemmEpi ekv = rms_in(f16_out(kv, 2 * d), ctx_ssq_);
      ekv.row_map = ctx_kv_map_;
      gemm(P, ctx_xn_, d, n, B.wkv, d, ekv);
      if (exchange_kv) exchange(P, b % 2 ? kXidCtx1 : kXidCtx0, kXCtx);
      gemm(P, ctx_xn_ + static_cast<size_t>(q0) * d, d, nq, B.wq, d, rms_in(f16_out(ctx_q_, d), ssq_q));
    }
    attention(P, ctx_q_, tl.qinfo + q0, nq, last ? tl.last : tl.all, last ? tl.n_last : tl.n_all,
              &shape_ctx_, kv, HWl_, D.c.win_t, 0, pos, ctx_att_, S);
    if (b == 0 && probe) tag(P, std::string(probe) + "_attn", attn_flops(-1, 0, S));
    float* xq = ctx_x_ + static_cast<size_t>(q0) * d;
    __half* xnq = ctx_xn_ + static_cast<size_t>(q0) * d;
    // the residual GEMMs are HBM-bound on the fp32 residual stream: their
    // probes carry algorithmic bytes (A, weights, residual in, fp32 + fp16
    // rows and sums of squares out)
    const double res_bytes = static_cast<double>(nq) * d * (4.0 + 4.0 + 2.0) + nq * (d / 32) * 4.0;
    gemm(P, ctx_att_, d, nq, B.wo, d, rms_out(f32_acc(xq, d), xnq, ssq_q));
    if (b == 0 && probe) tag(P, std::string(probe) + "_wo", 0.0, res_bytes + nq * d * 2.0 + d * d * 2.0);
    gemm(P, xnq, d, nq, B.wgu, d, rms_in(swiglu_out(ctx_h_, D.fp), ssq_q), 2.0 * nq * 2.0 * D.f * d);
    if (b == 0 && probe) tag(P, std::string(probe) + "_ffn_gu", 2.0 * nq * (2.0 * D.f) * d);
    gemm(P, ctx_h_, D.fp, nq, B.wd, D.fp, rms_out(f32_acc(xq, d), xnq, ssq_q), 2.0 * nq * d * D.f);
    if (b == 0 && probe) tag(P, std::string(probe) + "_wd", 0.0, res_bytes + nq * D.fp * 2.0 + d * D.fp * 2.0);
  }
}

void Engine::build_ctx(Program& P) {
  const Dims& D = D_;
  const int d = D.d, HWo = HWo_, T = D.T, n = T * HWo;
  add(P, [=, this](cudaStream_t s) {
    pswa_dev::fill_context_slots(ring_ptrs_, slot_src_, pad_, T, HWo, d, ctx_x_, s);
  });
  tag(P, "fill_slots", 0.0, 2.0 * n * d * 4.0);  // ring rows in, T slots out (fp32)
  // block 0 norm1 inputs; later norms come out of the residual GEMMs
  add(P, [=, this](cudaStream_t s) {
    pswa_dev::rms_prep(ctx_x_, d, nullptr, n, d, nullptr, 0, ctx_xn_, d, ctx_ssq_, d / 32, s);
  });
  tag(P, "rms_prep", 0.0, n * (d * (4.0 + 2.0) + (d / 32) * 4.0));  // fp32 in, fp16 + ssq out
  run_stack3d(P, ctx_, D.c.ctx_blocks, T, tiles_ctx_, true, "ctx");
  const float* last = ctx_x_ + static_cast<size_t>(T - 1) * HWo * d;
  __half* c16 = ctx16_ + static_cast<size_t>(B_.own0) * D.W * d;
  add(P, [=, this](cudaStream_t s) { pswa_dev::rmsnorm_rows(last, d, nullptr, HWo, d, d, ctx_gout_, c16, d, s); });
  tag(P, "rmsnorm", 0.0, static_cast<double>(HWo) * d * (4.0 + 2.0));
  exchange(P, kXidCtx16, kXAll);  // band mode: normed context of the boundary rows
  // cross-attention K/V of every cross block, once per frame (K7), over the
  // whole local grid (own rows + the halo received above)
  for (Block* stackp : {s1_, s2_}) {
    const int nb = stackp == s1_ ? D.c.s1_blocks : D.c.s2_blocks;
    for (int b = 0; b < nb; ++b)
      if (stackp[b].cross) gemm(P, ctx16_, d, HWl_, stackp[b].wkv, d, f16_out(stackp[b].kv_cache, 2 * d));
  }
}

// LRP transformer (A8) on the decoded (or
// teacher-forced) frame: the final channel representation was scattered
// into lrp_cat_ during the phases; y_hat joins it here. eps -> eps_chw_.
void Engine::build_lrp(Program& P) {
  const Dims& D = D_;
  const int d = D.d, HWo = HWo_, T = D.T, S = T + 1, C = D.C;
  const int kcat = D.N * D.sp + C;
  __half* cat_own = lrp_cat_ + static_cast<size_t>(B_.own0) * D.W * kcat;
  const int32_t* y_own = yfr_ + static_cast<size_t>(B_.own0) * D.W * C;
  add(P, [=](cudaStream_t s) {  // y_hat columns of the concat
    pswa_dev::yhat_rows_f16(y_own, C, nullptr, HWo, 0, C, cat_own + D.N * D.sp, kcat, C, s);
  });
  add(P, [=, this](cudaStream_t s) {  // past slots: the context transformer's inputs
    pswa_dev::fill_context_slots(ring_ptrs_, slot_src_, pad_, T, HWo, d, ctx_x_, s);
  });
  GemmEpi e;  // current slot: in_proj(concat(final_rep, y_hat)) + b
  e.out = ctx_x_ + static_cast<size_t>(T) * HWo * d;
  e.ld_out = d;
  e.out_f32 = 1;
  e.bias = lrp_in_b_;
  gemm(P, cat_own, kcat, HWo, lrp_in_, kcat, e);
  add(P, [=, this](cudaStream_t s) {
    pswa_dev::rms_prep(ctx_x_, d, nullptr, S * HWo, d, nullptr, 0, ctx_xn_, d, ctx_ssq_, d / 32, s);
  });
  run_stack3d(P, lrp_, D.c.lrp_blocks, S, tiles_lrp_, false, nullptr);
  const float* cur = ctx_x_ + static_cast<size_t>(T) * HWo * d;
  add(P, [=, this](cudaStream_t s) { pswa_dev::rmsnorm_rows(cur, d, nullptr, HWo, d, d, lrp_gout_, lrp16_, d, s); });
  GemmEpi eh;  // eps = 0.5 tanh(head(x) + b)
  eh.out = eps_;
  eh.ld_out = C;
  eh.out_f32 = 1;
  eh.bias = lrp_head_b_;
  eh.act = pswa_dev::kActTanhHalf;
  gemm(P, lrp16_, d, HWo, lrp_head_, d, eh);
  add(P, [=, this](cudaStream_t s) {  // [HWo][C] -> [C][HWo] (32-bit words)
    pswa_dev::yhat_to_chw(reinterpret_cast<const int32_t*>(eps_), HWo, C,
                          reinterpret_cast<int32_t*>(eps_chw_), s);
  });
}

// The hyper decoder's 3x3 convolutions run as implicit GEMMs (TMA im2col)
// when the channel count allows 64-channel tap blocks (paper scale: 128);
// PSWA_CONV_IM2COL_MATERIALISE=1 keeps the patch-matrix path.
bool Engine::implicit_conv() const {
  static const bool off = std::getenv("PSWA_CONV_IM2COL_MATERIALISE") != nullptr;
  return !off && D_.hc % 64 == 0 && D_.kconv == 9 * D_.hc;
}

void Engine::conv(Program& P, const __half* x, int h, int w, const PW& B, const pswa_dev::GemmEpi& ep) {
  pswa_dev::GemmPlan plan;
  pswa_dev::gemm_plan_conv3x3(&plan, x, h, w, D_.hc, B.p, B.K, B.N, ep);
  auto op = [plan](cudaStream_t s) { pswa_dev::gemm_run(plan, s); };
  add(P, op);
  if (log_gemms_) {
    gemm_log_.push_back(op);
    gemm_log_flops_ += 2.0 * h * w * B.N * 9.0 * D_.hc;
  }
}

void Engine::build_hyper_decode(Program& P) {
  const Dims& D = D_;
  const int hc = D.hc;
  add(P, [=, this](cudaStream_t s) { pswa_dev::zhat_to_nhwc(zhat_, hc, D.zh * D.zw, hx_, s); });
  float* src = hx_;
  float* dst = hu_;
  int h = D.zh, w = D.zw;
  for (int j = 0; j < 2; ++j) {
    const int ih = h, iw = w;
    float* in = src;
    float* out = dst;
    h *= 2;
    w *= 2;
    const int oh = h, ow = w;
    GemmEpi e1;
    e1.bias = hd_b_[j][0];
    e1.act = kActSilu;
    e1.n_store = hc;
    GemmEpi e2 = f32_acc(out, hc, hc);  // RB-up: out = up2(x) + conv(silu(conv(up2(x))))
    e2.bias = hd_b_[j][1];
    if (implicit_conv()) {
      // implicit-GEMM convolutions: the tcgen05 GEMM gathers its A tiles
      // from the fp16 NHWC image by TMA in im2col mode (no patch matrix);
      // same fp16 operands and K order as the materialised path below
      add(P, [=, this](cudaStream_t s) { pswa_dev::upsample2_nhwc(in, ih, iw, hc, out, s, hu16_); });
      e1.out = hyh16_;
      e1.ld_out = hc;
      conv(P, hu16_, oh, ow, hd_c_[j][0], e1);
      if (j == 1) tag(P, "hd_conv", 2.0 * oh * ow * hc * 9.0 * hc);
      conv(P, hyh16_, oh, ow, hd_c_[j][1], e2);
    } else {
      add(P, [=](cudaStream_t s) { pswa_dev::upsample2_nhwc(in, ih, iw, hc, out, s); });
      add(P, [=, this](cudaStream_t s) { pswa_dev::im2col3x3(out, oh, ow, hc, 1, 0, hcol_, D.kconv, s); });
      if (j == 1) tag(P, "im2col", 0.0, static_cast<double>(oh) * ow * (hc * 4.0 + D.kconv * 2.0));
      e1.out = hh_;
      e1.ld_out = hc;
      e1.out_f32 = 1;
      gemm(P, hcol_, D.kconv, oh * ow, hd_c_[j][0], D.kconv, e1);
      if (j == 1) tag(P, "hd_conv", 2.0 * oh * ow * hc * 9.0 * hc);
      add(P, [=, this](cudaStream_t s) { pswa_dev::im2col3x3(hh_, oh, ow, hc, 1, 0, hcol_, D.kconv, s); });
      gemm(P, hcol_, D.kconv, oh * ow, hd_c_[j][1], D.kconv, e2);
    }
    std::swap(src, dst);
  }
  const float* fin = src;
  const int np = D.Hp * D.Wp;
  add(P, [=, this](cudaStream_t s) { pswa_dev::f32_to_f16_rows(fin, hc, np, hc, hcast_, D.hcp, D.hcp, s); });
  GemmEpi e;
  e.out = hq_;
  e.ld_out = D.d;
  e.out_f32 = 1;
  e.bias = hd_out_b_;
  e.scale = cur_rsh_;
  e.bias_first = 1;
  e.row_map = crop_rows_;  // crop the padded hyper grid to the latent grid
  gemm(P, hcast_, D.hcp, np, hd_out_, D.hcp, e);
  tag(P, "hq_out", 2.0 * np * D.d * hc);
}

void Engine::build_hyper_encode(Program& P) {
  const Dims& D = D_;
  const int hc = D.hc;
  GemmEpi e0;
  e0.out = hx_;
  e0.ld_out = hc;
  e0.out_f32 = 1;
  e0.bias = he_in_b_;
  e0.n_store = hc;
  gemm(P, s1full_, D.d, D.Hp * D.Wp, he_in_, D.d, e0);
  float* src = hx_;
  float* other = hu_;
  int h = D.Hp, w = D.Wp;
  for (int j = 0; j < 2; ++j) {
    const int ih = h, iw = w;
    float* in = src;
    float* skip = other;
    add(P, [=, this](cudaStream_t s) { pswa_dev::im2col3x3(in, ih, iw, hc, 2, 0, hcol_, D.kconv, s); });
    h /= 2;
    w /= 2;
    const int oh = h, ow = w;
    GemmEpi e1;
    e1.out = hh_;
    e1.ld_out = hc;
    e1.out_f32 = 1;
    e1.bias = he_b_[j][0];
    e1.act = kActSilu;
    e1.n_store = hc;
    gemm(P, hcol_, D.kconv, oh * ow, he_c_[j][0], D.kconv, e1);
    add(P, [=](cudaStream_t s) { pswa_dev::subsample2_nhwc(in, ih, iw, hc, skip, s); });
    add(P, [=, this](cudaStream_t s) { pswa_dev::im2col3x3(hh_, oh, ow, hc, 1, 0, hcol_, D.kconv, s); });
    GemmEpi e2 = f32_acc(skip, hc, hc);  // RB-down: out = x[::2, ::2] + conv(silu(conv_s2(x)))
    e2.bias = he_b_[j][1];
    gemm(P, hcol_, D.kconv, oh * ow, he_c_[j][1], D.kconv, e2);
    std::swap(src, other);
  }
  const float* fin = src;
  add(P, [=, this](cudaStream_t s) { pswa_dev::round_to_zhat(fin, hc, D.zh * D.zw, zhat_, s); });
}

void Engine::build_embed(Program& P, const StepBatch& bt) {
  const Dims& D = D_;
  GemmEpi e;
  e.out = emb_cur_;
  e.ld_out = D.d;
  e.out_f32 = 1;
  e.scale = cur_rsi_;  // e = rate_scale_in * (W y_hat) + b
  e.bias = emb_b_;
  e.row_map = bt.rows;
  gemm(P, y16_, D.C, bt.M, emb_w_, D.C, e);
  if (bt.parts.size() == 1 && bt.parts[0][0] == D.c.s - 1) tag(P, "embed", 2.0 * bt.M * D.d * D.C);
}

void Engine::build_s1(Program& P, const StepBatch& bt, bool encoder) {
  const Dims& D = D_;
  const int d = D.d, M = bt.M;
  const int* rows = bt.rows;
  add(P, [=, this](cudaStream_t s) {  // gather + block 0 norm1 inputs
    pswa_dev::rms_prep(emb_cur_, d, rows, M, d, bx_, d, bxn_, d, bssq_, d / 32, s);
  });
  chaining_ = chain_enabled() && !encoder;
  for (int b = 0; b < D.c.s1_blocks; ++b) block_step(P, s1_[b], bt);
  flush_chain(P);
  chaining_ = false;
  add(P, [=, this](cudaStream_t s) { pswa_dev::rmsnorm_rows(bx_, d, nullptr, M, d, d, s1_gout_, bs1n_, d, s); });
  GemmEpi e = f16_out(acc_kv_, 2 * d);
  e.row_map = rows;
  gemm(P, bs1n_, d, M, acc_.wkv, d, e);
  if (encoder) {  // full-frame S1 for the hyper encoder (band mode: band 0 gathers it)
    const int* rp = bt.rows_pad;
    __half* dst = band0_s1_ ? band0_s1_ : s1full_;
    add(P, [=, this](cudaStream_t s) { pswa_dev::scatter_rows_f16(bs1n_, d, rp, M, d, dst, d, s); });
  }
  exchange(P, kXidAcc, bt.xkind);
}

// The accumulator's queries depend on Hq only, not on any
// decoded step: the decoder computes them for every position at once, in
// batch_all order (the encoder's single-batch layout, so the rows and their
// values are the encoder's), on the side stream next to the context
// transformer instead of once per step on the critical path.
void Engine::build_acc_q_all(Program& P) {
  const int d = D_.d;
  const StepBatch all = batch_all();
  const int* rows = all.rows;
  const int M = all.M;
  add(P, [=, this](cudaStream_t s) {
    pswa_dev::rms_prep(hq_, d, rows, M, d, nullptr, 0, qall16_, d, qall_ssq_, d / 32, s);
  });
  gemm(P, qall16_, d, M, acc_.wq, d, rms_in(f16_out(qall_, d), qall_ssq_));
  tag(P, "acc_q", 2.0 * M * d * d);
}

void Engine::build_step(Program& P, const StepBatch& bt, int mode) {
  const Dims& D = D_;
  const int d = D.d, M = bt.M;
  const int* rows = bt.rows;
  // accumulator: A = Hq + xattn(Q = Hq, KV = S1 of strictly earlier steps)
  add(P, [=, this](cudaStream_t s) {  // residual = Hq rows, normq folded into acc.wq
    pswa_dev::rms_prep(hq_, d, rows, M, d, bx_, d, bxn_, d, bssq_, d / 32, s);
  });
  // decode: Q precomputed by build_acc_q_all (step t at its batch_all offset)
  if (mode != 0) gemm(P, bxn_, d, M, acc_.wq, d, rms_in(f16_out(bq_, d), bssq_));
  for (const auto& pt : bt.parts) {
    const int t = pt[0], off = pt[1], n = pt[2];
    size_t qoff = static_cast<size_t>(off);
    if (mode == 0)
      for (int tt = 0; tt < t; ++tt) qoff += step_rows_h_[tt].size();
    const __half* q = (mode == 0 ? qall_ : bq_) + qoff * d;
    attention(P, q, step_qinfo_[t], n, step_tiles_[t], n_step_tiles_[t],
              &shape_step_[t][2], acc_kv_, 0, 0, 2, acc_.pos, batt_ + static_cast<size_t>(off) * d);
  }
  gemm(P, batt_, d, M, acc_.wo, d, rms_out(f32_acc(bx_, d), bxn_, bssq_));  // + S2 norm1 inputs
  const bool taps = mode == 1 && want_musig_;  // debug taps in forward_params only
  if (taps)
    add(P, [=, this](cudaStream_t s) { pswa_dev::scatter_rows_f32(bx_, d, rows, M, d, afull_, d, s); });
  // spatial module 2 (decoder: each block's GEMM tail and the next block's
  // projection run as one chained launch)
  chaining_ = chain_enabled() && mode == 0;
  for (int b = 0; b < D.c.s2_blocks; ++b) block_step(P, s2_[b], bt);
  flush_chain(P);
  chaining_ = false;
  add(P, [=, this](cudaStream_t s) { pswa_dev::rmsnorm_rows(bx_, d, nullptr, M, d, d, s2_gout_, bs2n_, d, s); });
  if (taps)
    add(P, [=, this](cudaStream_t s) { pswa_dev::scatter_rows_f16(bs2n_, d, rows, M, d, s2full_, d, s); });
  // channel transformer (incremental over groups) + heads + coder
  const int N = D.N, sl = D.slot, sp = D.sp, dchp = N * sp, Cg = D.Cg, C = D.C;
  const int ms = (2 * Cg + 63) / 64 * 64;
  GemmEpi ep;
  ep.out = chx_;
  ep.ld_out = dchp;
  ep.out_f32 = 1;
  gemm(P, bs2n_, d, M, ch_proj_, d, ep);
  if (mode == 0 && bt.parts[0][0] == 0) tag(P, "ch_proj", 2.0 * M * (D.N * sl) * d);
  static const bool ch_chain = std::getenv("PSWA_CH_CHAIN") != nullptr;
  chaining_ = ch_chain && mode == 0;
  for (int g = 0; g < N; ++g) {
    float* xg = chx_ + g * sp;
    if (g >= 1)  // channel shift: slot g sees y_hat group g-1
      gemm(P, y16_ + (g - 1) * Cg, C, M, ch_emb_[g], D.Cgp, f32_acc(xg, dchp, sl), 2.0 * M * sl * Cg);
    // slot-g RMSNorms: norm1 feeds the block-lower-triangular mix over
    // slots <= g (each slot normalised on its own, so it stays a kernel);
    // norm2 and the final norm are folded into the following GEMMs
    // through chx16_ / chssq_ written by the residual epilogues
    for (int b = 0; b < D.c.ch_blocks; ++b) {
      const float* g1 = ch_g1_[b] + g * sl;
      __half* xn = chxn_[b];
      add(P, [=](cudaStream_t s) { pswa_dev::rmsnorm_rows(xg, dchp, nullptr, M, sl, sl, g1, xn + g * sp, dchp, s); });
      const PW mixg{ch_mix_[b].p + static_cast<size_t>(g) * sp * dchp, sp, dchp};
      const bool pr = mode == 0 && g == 1 && b == 0 && bt.parts[0][0] == 0;
      gemm(P, xn, dchp, M, mixg, (g + 1) * sp, ch_rms_out(f32_acc(xg, dchp, sl)));
      if (pr) tag(P, "ch_mix", 2.0 * M * sl * (g + 1) * sl);
      gemm(P, chx16_, sp, M, ch_gu_[b][g], sp, ch_rms_in(swiglu_out(chh_, D.fgp)), 2.0 * M * 2.0 * D.fg * sl);
      if (pr) tag(P, "ch_gu", 2.0 * M * 2.0 * D.fg * sl);
      gemm(P, chh_, D.fgp, M, ch_d_[b][g], D.fgp, ch_rms_out(f32_acc(xg, dchp, sl)), 2.0 * M * sl * D.fg);
      if (pr) tag(P, "ch_d", 2.0 * M * D.fg * sl);
    }
    const float* go = ch_gout_ + g * sl;
    if (c_lrp() > 0) {  // the LRP transformer reads the normalised final representation
      add(P, [=, this](cudaStream_t s) { pswa_dev::rmsnorm_rows(xg, dchp, nullptr, M, sl, sl, go, chfo_, sp, s); });
      const int kcat = N * sp + C;
      __half* dst = lrp_cat_ + g * sp;
      add(P, [=, this](cudaStream_t s) { pswa_dev::scatter_rows_f16(chfo_, sp, rows, M, sp, dst, kcat, s); });
    }
    GemmEpi e1 = f16_out(hh16_, 2 * sp);
    e1.bias = head_b1_[g];
    e1.act = kActSilu;
    if (c_lrp() > 0)
      gemm(P, chfo_, sp, M, head_w1_[g], sp, e1);
    else  // final norm folded: A = fp16 slot g, 1/rms from the last d GEMM
      gemm(P, chx16_, sp, M, head_w1_[g], sp, ch_rms_in(e1));
    if (mode == 0 && g == 0 && bt.parts[0][0] == 0) tag(P, "ch_head1", 2.0 * M * (2.0 * sl) * sl);
    GemmEpi e2;
    e2.out = musig_;
    e2.ld_out = ms;
    e2.out_f32 = 1;
    e2.act = kActHead;
    e2.split = Cg;
    e2.bias = head_b2_[g];
    e2.scale = cur_rso_ + g * Cg;
    e2.n_store = 2 * Cg;
    gemm(P, hh16_, 2 * sp, M, head_w2_[g], 2 * sp, e2, 2.0 * M * (2.0 * Cg) * sl);
    if (mode == 0 && g == 0 && bt.parts[0][0] == 0) tag(P, "ch_head2", 2.0 * M * (2.0 * Cg) * (2.0 * sp));
    const int c0 = g * Cg;
    for (const auto& pt : bt.parts) {  // per step: the symbols of phase (t, g)
      const int t = pt[0], off = pt[1], n = pt[2];
      uint64_t o_step = 0;  // canonical ordinal of the first symbol of step t
      for (int tt = 0; tt < t; ++tt) o_step += static_cast<uint64_t>(step_rows_h_[tt].size()) * C;
      const uint64_t o0 = o_step + static_cast<uint64_t>(g) * n * Cg;
      const float* msg = musig_ + static_cast<size_t>(off) * ms;
      const int* rws = rows + off;
      __half* y16 = y16_ + static_cast<size_t>(off) * C;
      const pswa_dev::PhaseTaps taps = phase_taps();
      if (mode == 0) {
        const int L = D.c.lanes;
        add(P, [=, this](cudaStream_t s) {
          pswa_dev::lanes_decode_phase(d_main_, lanes_, L, o0, n, Cg, msg, ms, Cg, scales_, cdf_main_,
                                       rws, yfr_, C, c0, y16, C, status_, s, taps);
        });
      } else {
        add(P, [=, this](cudaStream_t s) {
          pswa_dev::quantize_phase(msg, ms, Cg, n, Cg, o0, rws, yfr_, C, c0, scales_, cdf_main_, sym_v_,
                                   sym_idx_, y16, C, taps, status_, s);
        });
      }
    }
    if (mode == 0 && host_copy_ && bt.parts.size() == 1 && bt.parts[0][0] == D.c.s - 1) {
      flush_chain(P);
      // channel group g of the last step decoded: its CHW planes are final
      const int HWo = HWo_;
      add(P, [=, this](cudaStream_t s) { pswa_dev::yhat_to_chw_cols(yfr_, HWo, C, c0, Cg, ychw_, s); });
      P.cuts.push_back(Cut{P.ops.size(), false});
      P.copy_group.push_back(g);
    }
  }
  flush_chain(P);
  chaining_ = false;
  if (mode == 0) build_embed(P, bt);
}

Program& Engine::program(const std::string& key) {
  auto it = progs_.find(key);
  if (it != progs_.end()) return it->second;
  Program& P = progs_[key];
  const Dims& D = D_;
  const int HW = HWo_, C = D.C, L = D.c.lanes, Lz = D.c.hyper_lanes;  // HW: own positions
  const int nz = D.hc * D.zh * D.zw;
  const size_t yoff = static_cast<size_t>(B_.own0) * D.W * C;  // own rows in yfr_
  const std::string base = key.substr(0, key.find('+'));
  // "+ms": mu/sigma and per-symbol bit taps (BitStats) in every phase
  taps_ = key.find("+ms") != std::string::npos;
  if (base == "decode") {
    log_gemms_ = true;
    gemm_log_.clear();
    gemm_log_flops_ = 0.0;
    // "+h" (single band): per-group ŷ transpositions and cuts for the host copies
    host_copy_ = key.find("+h") != std::string::npos && B_.n == 1;
    // the hyperprior branch (z_hat lanes -> hyper decoder -> Hq) does not
    // depend on the context transformer: it runs on a side stream of the
    // same graph and joins before the first Hq consumer (band mode: before
    // the first exchange, since each segment is its own graph)
    const size_t side_from = P.ops.size();
    add(P, [=, this](cudaStream_t s) {
      pswa_dev::lanes_init(d_hyper_, d_lens_, Lz, static_cast<uint32_t>(nz), hlanes_, status_, s);
    });
    add(P, [=, this](cudaStream_t s) {
      pswa_dev::lanes_decode_hyper(d_hyper_, hlanes_, Lz, nz, D.zh * D.zw, cur_loc_, cur_scale_,
                                   scales_, cdf_, zhat_, status_, s);
    });
    // replayable as a pair only (the decode consumes the lanes the init sets up)
    tag(P, "decode_hyper", 0.0, 0.0, 2);
    add(P, [=, this](cudaStream_t s) { pswa_dev::sum_lane_bits(hlanes_, Lz, bits_, s); });
    build_hyper_decode(P);
    build_acc_q_all(P);
    to_side(P, side_from);
    if (B_.n > 1) join_side(P);
    build_ctx(P);
    if (B_.n == 1) join_side(P);
    if (host_copy_) {  // the main payload's H2D copy runs beside the context transformer
      P.cuts.push_back(Cut{P.ops.size(), false});
      P.copy_group.push_back(kCutMainIn);
    }
    add(P, [=, this](cudaStream_t s) {
      pswa_dev::lanes_init(d_main_, d_lens_ + 1, L, static_cast<uint32_t>(HW) * C, lanes_, status_, s);
    });
    tag(P, "lanes_init", 0.0, L * (2.0 + 6.0 + sizeof(pswa_dev::LaneState)));
    for (int t = 0; t < D.c.s; ++t) {
      if (t > 0) build_s1(P, batch_of(t - 1), false);
      build_step(P, batch_of(t), 0);
    }
    add(P, [=, this](cudaStream_t s) { pswa_dev::sum_lane_bits(lanes_, L, bits_ + 1, s); });
    if (taps_) {
      const int row0 = B_.own0 * D.W;
      add(P, [=, this](cudaStream_t s) {
        pswa_dev::bitstats_reduce(symbits_, C, row0, HW, D.N, D.Cg, bitstats_, s);
      });
    }
    if (!host_copy_)
      add(P, [=, this](cudaStream_t s) { pswa_dev::yhat_to_chw(yfr_ + yoff, HW, C, ychw_, s); });
    host_copy_ = false;
    if (c_lrp() > 0) build_lrp(P);
    flush_chain(P);
    log_gemms_ = false;
    {  // every GEMM launch of the frame, replayed in program order
      Probe pr;
      auto ops = gemm_log_;
      pr.op = [ops](cudaStream_t s) {
        for (auto& o : ops) o(s);
      };
      pr.flops = gemm_log_flops_;
      pr.launches = static_cast<int>(ops.size());
      probes_["gemm_all"] = std::move(pr);
    }
  } else if (base == "encode" || base == "encode_z") {
    const bool zgiven = base == "encode_z";
    add(P, [=, this](cudaStream_t s) { pswa_dev::yhat_from_chw(ychw_, HW, C, yfr_ + yoff, s); });
    build_ctx(P);
    // teacher forced: every step's latents are known, so each layer runs
    // once over all steps (one GEMM per layer, one attention launch per step)
    const StepBatch all = batch_all();
    const int* arows = all.rows;
    const int Mall = all.M;
    add(P, [=, this](cudaStream_t s) { pswa_dev::yhat_rows_f16(yfr_, C, arows, Mall, 0, C, y16_, C, C, s); });
    build_embed(P, all);
    build_s1(P, all, true);
    if (!zgiven) {
      if (B_.n > 1) {
        // every band has scattered its S1 rows into band 0's full-frame
        // buffer; each band then runs the (small) hyper encoder on a local
        // copy, so z_hat is bitwise identical on every band
        if (ipc_) throw std::invalid_argument("cross-process band encode needs z_hat (encode_z)");
        cut(P, true);
        if (band0_s1_ && band0_s1_ != s1full_) {
          const __half* src = band0_s1_;
          const size_t bytes = static_cast<size_t>(D.Hp) * D.Wp * D.d * sizeof(__half);
          add(P, [=, this](cudaStream_t s) {
            PSWA_CUDA(cudaMemcpyAsync(s1full_, src, bytes, cudaMemcpyDefault, s));
          }, 0);
        }
      }
      build_hyper_encode(P);
    }
    add(P, [=, this](cudaStream_t s) {
      pswa_dev::quantize_hyper(zhat_, nz, D.zh * D.zw, cur_loc_, cur_scale_, scales_, hsym_v_,
                               hsym_idx_, s);
    });
    build_hyper_decode(P);
    build_step(P, all, 1);
    if (c_lrp() > 0) build_lrp(P);
    add(P, [=, this](cudaStream_t s) {
      pswa_dev::lanes_encode(hsym_v_, hsym_idx_, nz, Lz, cdf_, enc_hlanes_, enc_hcap_, enc_hlens_,
                             enc_hbits_, status_, s);
    });
    add(P, [=, this](cudaStream_t s) {
      pswa_dev::lanes_pack(enc_hlanes_, enc_hcap_, enc_hlens_, Lz, static_cast<uint32_t>(nz),
                           d_hyper_, hyper_cap_, pack_total_, pack_offs_, status_, s);
    }, 2);
    add(P, [=, this](cudaStream_t s) {
      pswa_dev::lanes_encode(sym_v_, sym_idx_, static_cast<uint64_t>(HW) * C, L, cdf_main_, enc_lanes_,
                             enc_cap_, enc_lens_, enc_bits_, status_, s);
    });
    add(P, [=, this](cudaStream_t s) {
      pswa_dev::lanes_pack(enc_lanes_, enc_cap_, enc_lens_, L, static_cast<uint32_t>(HW) * C,
                           d_main_, main_cap_, pack_total_ + 1, pack_offs_, status_, s);
    }, 2);
    add(P, [=, this](cudaStream_t s) { pswa_dev::sum_doubles(enc_hbits_, Lz, bits_, s); });
    add(P, [=, this](cudaStream_t s) { pswa_dev::sum_doubles(enc_bits_, L, bits_ + 1, s); });
    if (taps_) {
      const int row0 = B_.own0 * D.W;
      add(P, [=, this](cudaStream_t s) {
        pswa_dev::bitstats_reduce(symbits_, C, row0, HW, D.N, D.Cg, bitstats_, s);
      });
    }
  } else if (base == "push") {
    add(P, [=, this](cudaStream_t s) { pswa_dev::yhat_from_chw(ychw_, HW, C, yfr_ + yoff, s); });
    const StepBatch all = batch_all();  // embeddings are per position: one pass
    const int* arows = all.rows;
    const int Mall = all.M;
    add(P, [=, this](cudaStream_t s) { pswa_dev::yhat_rows_f16(yfr_, C, arows, Mall, 0, C, y16_, C, C, s); });
    build_embed(P, all);
  } else {
    throw std::invalid_argument("unknown program " + key);
  }
  flush_chain(P);
  taps_ = false;
  return P;
}

// One graph per segment (a single segment unless band mode). The graphs are
// captured lazily on first use.
void Engine::launch_segment(Program& P, int k) {
  static const bool no_graph = std::getenv("PSWA_NO_GRAPH") != nullptr;
  const size_t b = k == 0 ? 0 : P.cuts[k - 1].at;
  const size_t e = k + 1 < segments(P) ? P.cuts[k].at : P.ops.size();
  if (no_graph) {
    for (size_t i = b; i < e; ++i) P.ops[i](st_);
    return;
  }
  if (P.execs.empty()) P.execs.assign(segments(P), nullptr);
  if (!P.execs[k]) {
    cudaGraph_t g = nullptr;
    PSWA_CUDA(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal));
    try {
      for (size_t i = b; i < e; ++i) P.ops[i](st_);
    } catch (...) {
      cudaStreamEndCapture(st_, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    PSWA_CUDA(cudaStreamEndCapture(st_, &g));
    PSWA_CUDA(cudaGraphInstantiate(&P.execs[k], g, 0));
    PSWA_CUDA(cudaGraphDestroy(g));
  }
  PSWA_CUDA(cudaGraphLaunch(P.execs[k], st_));
}

void Engine::run(Program& P) {
  if (B_.n > 1 && !ipc_) throw std::logic_error("in-process band engines are run by their BandGroup");
  last_launches_ = P.launches;
  launch_segment(P, 0);
}

void Engine::run_host_copy(Program& P, int32_t* yhat_out) {
  last_launches_ = P.launches;
  const size_t plane = static_cast<size_t>(HWo_) * D_.Cg;  // one channel group, int32
  for (int k = 0; k < segments(P); ++k) {
    launch_segment(P, k);
    const int g = k < static_cast<int>(P.copy_group.size()) ? P.copy_group[k] : -1;
    if (g == kCutMainIn) PSWA_CUDA(cudaStreamWaitEvent(st_, ev_main_in_, 0));
    if (g < 0) continue;
    PSWA_CUDA(cudaEventRecord(ev_copy_[g], st_));
    PSWA_CUDA(cudaStreamWaitEvent(copy_, ev_copy_[g], 0));
    PSWA_CUDA(cudaMemcpyAsync(yhat_out + g * plane, ychw_ + g * plane, plane * sizeof(int32_t),
                              cudaMemcpyDeviceToHost, copy_));
  }
  PSWA_CUDA(cudaEventRecord(ev_copy_done_, copy_));
  PSWA_CUDA(cudaStreamWaitEvent(st_, ev_copy_done_, 0));
}

// ------------------------------------------------------------ probes ------
void Engine::tag(Program& P, const std::string& name, double flops, double bytes, int nops) {
  if (chain_.plan.njobs > 0) {  // a GEMM inside an open chain: the chain launch is the probe
    if (chain_.tag.empty()) chain_.tag = name;
    chain_.flops += flops;
    return;
  }
  std::vector<std::function<void(cudaStream_t)>> ops(P.ops.end() - nops, P.ops.end());
  Probe pr;
  pr.op = nops == 1 ? ops[0] : [ops](cudaStream_t s) {
    for (auto& o : ops) o(s);
  };
  pr.flops = flops;
  pr.bytes = bytes;
  pr.launches = nops;
  probes_[name] = std::move(pr);
}

std::string Engine::probe_list() const {
  std::string out;
  for (const auto& [name, p] : probes_)
    out += name + " " + std::to_string(p.flops) + " " + std::to_string(p.bytes) + " " +
           std::to_string(p.launches) + "\n";
  return out;
}

// Algorithmic attention FLOPs of one launch: 4 * d per (query, allowed key)
// (QK^T and PV, 2 d each), counting in-grid, in-window, mask-allowed keys only
// (SURVEY §8(d)). t < 0: the 3D context window over all T slots.
double Engine::attn_flops(int t, int mask, int slots) const {
  const Dims& D = D_;
  const int rh = D.c.win_h / 2, rw = D.c.win_w / 2;
  double keys = 0;
  for (int y = B_.own0; y < B_.own0 + B_.nown; ++y)
    for (int x = 0; x < D.W; ++x) {
      const int gy = y + B_.lo;
      if (t >= 0 && (gy + x) % D.c.s != t) continue;
      int n = 0;
      for (int ky = std::max(0, y - rh); ky <= std::min(B_.Hl - 1, y + rh); ++ky)
        for (int kx = std::max(0, x - rw); kx <= std::min(D.W - 1, x + rw); ++kx) {
          const int ks = (ky + B_.lo + kx) % D.c.s;
          if (t >= 0 && ((mask == 1 && ks > t) || (mask == 2 && ks >= t))) continue;
          ++n;
        }
      if (t >= 0) keys += n;
      else
        for (int j = 0; j < slots; ++j) keys += static_cast<double>(n) * std::min(j + 1, D.c.win_t);
    }
  return 4.0 * D.d * keys;
}

double Engine::bench_op(const std::string& name, int reps, double* flops, double* bytes) {
  auto it = probes_.find(name);
  if (it == probes_.end())
    throw std::invalid_argument("bench_op: unknown probe (run a decode first): " + name);
  auto& op = it->second.op;
  if (reps <= 0) {  // one bare replay (profilers capture exactly this launch)
    op(st_);
    PSWA_CUDA(cudaStreamSynchronize(st_));
    if (flops) *flops = it->second.flops;
    if (bytes) *bytes = it->second.bytes;
    return 0.0;
  }
  for (int i = 0; i < 3; ++i) op(st_);
  cudaEvent_t a, b;
  PSWA_CUDA(cudaEventCreate(&a));
  PSWA_CUDA(cudaEventCreate(&b));
  PSWA_CUDA(cudaEventRecord(a, st_));
  for (int i = 0; i < reps; ++i) op(st_);
  PSWA_CUDA(cudaEventRecord(b, st_));
  PSWA_CUDA(cudaEventSynchronize(b));
  float ms = 0;
  PSWA_CUDA(cudaEventElapsedTime(&ms, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (flops) *flops = it->second.flops;
  if (bytes) *bytes = it->second.bytes;
  return 1e3 * ms / reps;  // us per replay
}

// ------------------------------------------------------------ band mode ---
void Engine::cut(Program& P, bool global) {
  flush_chain(P);
  if (B_.n > 1) P.cuts.push_back(Cut{P.ops.size(), global});
}

__half* Engine::xbuf(int id) {
  if (id < 16) return s1_[id].kv_cache;
  if (id < 32) return s2_[id - 16].kv_cache;
  if (id == kXidAcc) return acc_kv_;
  if (id == kXidCtx0) return ctx_kv_;
  if (id == kXidCtx1) return ctx_kv2_;
  return ctx16_;
}

int Engine::xld(int id) const { return id == kXidCtx16 ? D_.d : 2 * D_.d; }

// Row pairs (my local row, the neighbour's local row) of the kHaloRows
// boundary rows each neighbour needs: my top rows into the upper band's
// bottom halo, my bottom rows into the lower band's top halo. Kinds: step t
// (positions with (y + x) mod s == t), all positions, or all positions of
// every context slot (slot strides HWl of each side).
void Engine::build_pairs() {
  const Dims& D = D_;
  for (int side = 0; side < 2; ++side) {
    const PeerInfo& nb = peer_[side];
    for (int k = 0; k < 18; ++k) {
      nxpairs_[side][k] = 0;
      xpairs_[side][k] = nullptr;
    }
    if (!nb.present) continue;
    const int g0 = side == 0 ? B_.r0 : B_.r1 - kHaloRows;  // global rows sent
    std::vector<int2> v[18];
    for (int y = g0; y < g0 + kHaloRows; ++y)
      for (int x = 0; x < D.W; ++x) {
        const int src = (y - B_.lo) * D.W + x, dst = (y - nb.lo) * D.W + x;
        v[(y + x) % D.c.s].push_back(make_int2(src, dst));
        v[kXAll].push_back(make_int2(src, dst));
        for (int j = 0; j < D.T; ++j)
          v[kXCtx].push_back(make_int2(j * HWl_ + src, j * nb.HWl + dst));
      }
    for (int k = 0; k < 18; ++k) {
      if (v[k].empty()) continue;
      int2* p = dalloc<int2>(v[k].size());
      PSWA_CUDA(cudaMemcpyAsync(p, v[k].data(), v[k].size() * sizeof(int2), cudaMemcpyHostToDevice, st_));
      xpairs_[side][k] = p;
      nxpairs_[side][k] = static_cast<int>(v[k].size());
    }
  }
  PSWA_CUDA(cudaStreamSynchronize(st_));
}

void Engine::exchange(Program& P, int id, int kind) {
  if (B_.n <= 1) return;
  for (int side = 0; side < 2; ++side) {
    const PeerInfo& nb = peer_[side];
    if (!nb.present || !nxpairs_[side][kind]) continue;
    const __half* src = xbuf(id);
    __half* dst = nb.buf[id];
    const int ld = xld(id), n = nxpairs_[side][kind];
    const int2* pairs = xpairs_[side][kind];
    add(P, [=](cudaStream_t s) { pswa_dev::halo_push(src, dst, ld, pairs, n, s); });
  }
  if (ipc_) {
    // the band above counts my pushes in its "from below" slot and v.v.
    unsigned* to_up = peer_[0].present ? peer_[0].mbox + 1 : nullptr;
    unsigned* to_down = peer_[1].present ? peer_[1].mbox : nullptr;
    const bool need_up = peer_[0].present, need_down = peer_[1].present;
    add(P, [=](cudaStream_t s) { pswa_dev::band_signal(to_up, to_down, s); });
    add(P, [=, this](cudaStream_t s) {
      pswa_dev::band_wait(mbox_, wait_ctr_, need_up, need_down, status_, s);
    });
  } else {
    cut(P, false);
  }
}

PeerInfo Engine::self_info() {
  PeerInfo p;
  p.present = true;
  p.lo = B_.lo;
  p.HWl = HWl_;
  for (int id = 0; id < kXids; ++id) p.buf[id] = xbuf(id);  // null for absent blocks
  p.s1full = s1full_;
  p.mbox = mbox_;
  return p;
}

void Engine::link(Engine* up, Engine* down, Engine* band0) {
  peer_[0] = up ? up->self_info() : PeerInfo{};
  peer_[1] = down ? down->self_info() : PeerInfo{};
  band0_s1_ = band0 ? band0->s1full_ : nullptr;
  ipc_ = false;
  build_pairs();
  for (auto& kv : progs_)
    for (auto ex : kv.second.execs)
      if (ex) cudaGraphExecDestroy(ex);
  progs_.clear();
}

// ---- CUDA-IPC blob: "PSWI" | i32 band, n, lo, HWl | handles of the
// exchange buffers (kXids), band 0's S1 gather buffer and the mailbox
namespace {
struct IpcBlob {
  char magic[4];
  int band, n, lo, HWl;
  int has[kXids + 2];
  cudaIpcMemHandle_t h[kXids + 2];
};
}  // namespace

std::vector<uint8_t> Engine::ipc_export() {
  if (B_.n <= 1) throw std::invalid_argument("ipc_export: not a band handle");
  IpcBlob b{};
  std::memcpy(b.magic, "PSWI", 4);
  b.band = B_.idx;
  b.n = B_.n;
  b.lo = B_.lo;
  b.HWl = HWl_;
  const PeerInfo me = self_info();
  for (int i = 0; i < kXids + 2; ++i) {
    void* p = i < kXids ? static_cast<void*>(me.buf[i]) : i == kXids ? static_cast<void*>(s1full_) : mbox_;
    b.has[i] = p != nullptr;
    if (p) PSWA_CUDA(cudaIpcGetMemHandle(&b.h[i], p));
  }
  std::vector<uint8_t> out(sizeof(b));
  std::memcpy(out.data(), &b, sizeof(b));
  return out;
}

void Engine::link_ipc(const uint8_t* up, size_t up_len, const uint8_t* down, size_t down_len) {
  auto open = [&](const uint8_t* blob, size_t len, int want_band) {
    PeerInfo p;
    if (!blob) return p;
    IpcBlob b;
    if (len != sizeof(b)) throw std::invalid_argument("link_ipc: bad blob size");
    std::memcpy(&b, blob, sizeof(b));
    if (std::memcmp(b.magic, "PSWI", 4) != 0 || b.band != want_band || b.n != B_.n)
      throw std::invalid_argument("link_ipc: blob is not the neighbouring band of this group");
    p.present = true;
    p.lo = b.lo;
    p.HWl = b.HWl;
    for (int i = 0; i < kXids + 2; ++i) {
      if (!b.has[i]) continue;
      void* q = nullptr;
      PSWA_CUDA(cudaIpcOpenMemHandle(&q, b.h[i], cudaIpcMemLazyEnablePeerAccess));
      ipc_mapped_.push_back(q);
      if (i < kXids) p.buf[i] = static_cast<__half*>(q);
      else if (i == kXids) p.s1full = static_cast<__half*>(q);
      else p.mbox = static_cast<unsigned*>(q);
    }
    return p;
  };
  if ((B_.idx > 0) != (up != nullptr) || (B_.idx + 1 < B_.n) != (down != nullptr))
    throw std::invalid_argument("link_ipc: neighbour blobs do not match the band position");
  peer_[0] = open(up, up_len, B_.idx - 1);
  peer_[1] = open(down, down_len, B_.idx + 1);
  band0_s1_ = nullptr;
  ipc_ = true;
  build_pairs();
  for (auto& kv : progs_)
    for (auto ex : kv.second.execs)
      if (ex) cudaGraphExecDestroy(ex);
  progs_.clear();
}

// ---------------------------------------------------------- frame API ----
void Engine::set_frame_params(int rate, int fidx) {
  const Dims& D = D_;
  if (rate < 0 || rate >= D.c.rate_points) throw std::invalid_argument("rate_idx out of range");
  if (fidx < 0) throw std::invalid_argument("frame_idx_in_gop < 0");
  const int slot = fidx < 4 ? fidx : 4;  // select_prior
  auto d2d = [&](float* dst, const float* src, int n) {
    PSWA_CUDA(cudaMemcpyAsync(dst, src, sizeof(float) * n, cudaMemcpyDeviceToDevice, st_));
  };
  d2d(cur_rsi_, rate_in_ + static_cast<size_t>(rate) * D.d, D.d);
  d2d(cur_rsh_, rate_hyper_ + static_cast<size_t>(rate) * D.d, D.d);
  d2d(cur_rso_, rate_out_ + static_cast<size_t>(rate) * D.C, D.C);
  d2d(cur_loc_, prior_loc_ + (static_cast<size_t>(rate) * 5 + slot) * D.hc, D.hc);
  d2d(cur_scale_, prior_scale_ + (static_cast<size_t>(rate) * 5 + slot) * D.hc, D.hc);
  std::vector<int> src(static_cast<size_t>(D.T));
  for (int i = 0; i < D.T; ++i) {
    const int k = D.T - i;  // slot i holds the k-th most recent frame
    src[i] = k <= npast_ ? ((head_ - k) % D.T + D.T) % D.T : -1;
  }
  PSWA_CUDA(cudaMemcpyAsync(slot_src_, src.data(), sizeof(int) * D.T, cudaMemcpyHostToDevice, st_));
  PSWA_CUDA(cudaMemsetAsync(status_, 0, sizeof(int), st_));
  PSWA_CUDA(cudaMemsetAsync(bits_, 0, 2 * sizeof(double), st_));
}

void Engine::advance_ring() {
  PSWA_CUDA(cudaMemcpyAsync(ring_[head_], emb_cur_ + static_cast<size_t>(B_.own0) * D_.W * D_.d,
                            sizeof(float) * HWo_ * D_.d, cudaMemcpyDeviceToDevice, st_));
  head_ = (head_ + 1) % D_.T;
  npast_ = std::min(npast_ + 1, D_.T);
}

void Engine::reset_gop() {
  head_ = 0;
  npast_ = 0;
}

// Own rows of a full-frame [planes][H][W] int32 host/device buffer into (or,
// with dst == nullptr semantics reversed by the callers) the compact
// [planes][nown][W] device layout.
void Engine::copy_rows_in(int32_t* dst, const int32_t* src_full, int planes, bool device) {
  const size_t row = static_cast<size_t>(HWo_) * sizeof(int32_t);
  const cudaMemcpyKind k = device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  if (B_.n == 1) {
    PSWA_CUDA(cudaMemcpyAsync(dst, src_full, row * planes, k, st_));
  } else {
    PSWA_CUDA(cudaMemcpy2DAsync(dst, row, src_full + static_cast<size_t>(B_.r0) * D_.W,
                                static_cast<size_t>(D_.HW) * sizeof(int32_t), row, planes, k, st_));
  }
}

void Engine::push_frame(const int32_t* yhat_chw, int rate) {
  set_frame_params(rate, 0);
  copy_rows_in(ychw_, yhat_chw, D_.C, false);
  Program& P = program("push");
  last_launches_ = P.launches;
  launch_segment(P, 0);  // no exchanges: embeddings are per position
  advance_ring();
  PSWA_CUDA(cudaStreamSynchronize(st_));
}

std::string Engine::encode_key(bool zgiven, bool musig) {
  return std::string(zgiven ? "encode_z" : "encode") + (musig ? "+ms" : "");
}

void Engine::prep_encode(const int32_t* yhat_chw, int rate, int fidx, const int32_t* zhat_in) {
  set_frame_params(rate, fidx);
  copy_rows_in(ychw_, yhat_chw, D_.C, false);
  if (zhat_in)
    PSWA_CUDA(cudaMemcpyAsync(zhat_, zhat_in, sizeof(int32_t) * D_.hc * D_.zh * D_.zw,
                              cudaMemcpyHostToDevice, st_));
}

FrameResult Engine::finish_encode(float* mu_out, float* sigma_out, uint8_t* hyper_out,
                                  size_t hyper_cap, uint8_t* main_out, size_t main_cap,
                                  bool advance) {
  FrameResult r;
  unsigned long long tot[2];
  PSWA_CUDA(cudaMemcpyAsync(tot, pack_total_, sizeof(tot), cudaMemcpyDeviceToHost, st_));
  PSWA_CUDA(cudaMemcpyAsync(r.bits, bits_, sizeof(r.bits), cudaMemcpyDeviceToHost, st_));
  PSWA_CUDA(cudaMemcpyAsync(&r.status, status_, sizeof(int), cudaMemcpyDeviceToHost, st_));
  PSWA_CUDA(cudaStreamSynchronize(st_));
  if (r.status & 16)
    throw std::invalid_argument("encode: y_hat outside the supported range (|y_hat| <= " +
                                std::to_string(pswa_dev::kYhatMax) + ")");
  if (r.status) throw pswa_abi::LaneError("encoder status " + std::to_string(r.status));
  r.hyper_len = tot[0];
  r.main_len = tot[1];
  if (hyper_out) {
    if (hyper_cap < r.hyper_len) throw std::invalid_argument("hyper output buffer too small");
    PSWA_CUDA(cudaMemcpyAsync(hyper_out, d_hyper_, r.hyper_len, cudaMemcpyDeviceToHost, st_));
  }
  if (main_out) {
    if (main_cap < r.main_len) throw std::invalid_argument("main output buffer too small");
    PSWA_CUDA(cudaMemcpyAsync(main_out, d_main_, r.main_len, cudaMemcpyDeviceToHost, st_));
  }
  fetch_musig(mu_out, sigma_out);
  have_stats_ = want_musig_ || stats_on_;
  if (advance) advance_ring();
  PSWA_CUDA(cudaStreamSynchronize(st_));
  return r;
}

// [HWl][C] device taps -> own rows of [C][H][W] host frames (nullable)
void Engine::fetch_musig(float* mu_out, float* sigma_out) {
  if (!mu_out && !sigma_out) return;
  const Dims& D = D_;
  const size_t n = static_cast<size_t>(HWl_) * D.C;
  std::vector<float> a(n), b(n);
  PSWA_CUDA(cudaMemcpyAsync(a.data(), mu_full_, sizeof(float) * n, cudaMemcpyDeviceToHost, st_));
  PSWA_CUDA(cudaMemcpyAsync(b.data(), sg_full_, sizeof(float) * n, cudaMemcpyDeviceToHost, st_));
  PSWA_CUDA(cudaStreamSynchronize(st_));
  const size_t o = static_cast<size_t>(B_.own0) * D.W, g = static_cast<size_t>(B_.r0) * D.W;
  for (int p = 0; p < HWo_; ++p)
    for (int c = 0; c < D.C; ++c) {
      if (mu_out) mu_out[static_cast<size_t>(c) * D.HW + g + p] = a[(o + p) * D.C + c];
      if (sigma_out) sigma_out[static_cast<size_t>(c) * D.HW + g + p] = b[(o + p) * D.C + c];
    }
}

void Engine::last_bitstats(double* out) {
  if (!have_stats_)
    throw std::invalid_argument("last_bitstats: the last frame call ran without stats "
                                "(pswa_gpu_set_stats, or request mu/sigma)");
  const Dims& D = D_;
  std::vector<double> v(static_cast<size_t>(D.N) * HWo_);
  PSWA_CUDA(cudaMemcpyAsync(v.data(), bitstats_, sizeof(double) * v.size(), cudaMemcpyDeviceToHost, st_));
  PSWA_CUDA(cudaStreamSynchronize(st_));
  const size_t g0 = static_cast<size_t>(B_.r0) * D.W;
  for (int g = 0; g < D.N; ++g)
    std::memcpy(out + static_cast<size_t>(g) * D.HW + g0, v.data() + static_cast<size_t>(g) * HWo_,
                sizeof(double) * HWo_);
}

void Engine::fetch_payloads(uint8_t* hyper_out, size_t hyper_cap, const FrameResult& r,
                            uint8_t* main_out) {
  if (hyper_out) {
    if (hyper_cap < r.hyper_len) throw std::invalid_argument("hyper output buffer too small");
    PSWA_CUDA(cudaMemcpyAsync(hyper_out, d_hyper_, r.hyper_len, cudaMemcpyDeviceToHost, st_));
  }
  if (main_out) PSWA_CUDA(cudaMemcpyAsync(main_out, d_main_, r.main_len, cudaMemcpyDeviceToHost, st_));
  PSWA_CUDA(cudaStreamSynchronize(st_));
}

FrameResult Engine::encode(const int32_t* yhat_chw, int rate, int fidx, const int32_t* zhat_in,
                           float* mu_out, float* sigma_out, uint8_t* hyper_out, size_t hyper_cap,
                           uint8_t* main_out, size_t main_cap, bool advance) {
  prep_encode(yhat_chw, rate, fidx, zhat_in);
  want_musig_ = mu_out != nullptr;
  // the taps (mu/sigma/bit outputs) are baked into the captured graph, so
  // the two variants are separate programs
  run(program(encode_key(zhat_in != nullptr, want_musig_ || stats_on_)));
  return finish_encode(mu_out, sigma_out, hyper_out, hyper_cap, main_out, main_cap, advance);
}

void Engine::prep_decode(const void* hyper, size_t hyper_len, const void* main_pl, size_t main_len,
                         int rate, int fidx, bool device, bool defer_main) {
  if (hyper_len > hyper_cap_ || main_len > main_cap_)
    throw pswa_abi::TruncatedError("payload larger than the decoder's capacity");
  set_frame_params(rate, fidx);
  const cudaMemcpyKind in_kind = device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  PSWA_CUDA(cudaMemcpyAsync(d_hyper_, hyper, hyper_len, in_kind, st_));
  if (defer_main) {  // on copy_, awaited by the program's kCutMainIn cut
    PSWA_CUDA(cudaEventRecord(ev_main_in_, st_));  // d_main_ free: earlier work on st_ done
    PSWA_CUDA(cudaStreamWaitEvent(copy_, ev_main_in_, 0));
    PSWA_CUDA(cudaMemcpyAsync(d_main_, main_pl, main_len, in_kind, copy_));
    PSWA_CUDA(cudaEventRecord(ev_main_in_, copy_));
  } else {
    PSWA_CUDA(cudaMemcpyAsync(d_main_, main_pl, main_len, in_kind, st_));
  }
  lens_h_[0] = static_cast<uint32_t>(hyper_len);
  lens_h_[1] = static_cast<uint32_t>(main_len);
  PSWA_CUDA(cudaMemcpyAsync(d_lens_, lens_h_, sizeof(lens_h_), cudaMemcpyHostToDevice, st_));
}

FrameResult Engine::finish_decode(bool advance, int32_t* yhat_out, bool device, float* mu_out,
                                  float* sigma_out) {
  const Dims& D = D_;
  FrameResult r;
  const size_t row = static_cast<size_t>(HWo_) * sizeof(int32_t);
  const cudaMemcpyKind k = device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  if (!yhat_out) {
    // already copied (run_host_copy)
  } else if (B_.n == 1) {
    PSWA_CUDA(cudaMemcpyAsync(yhat_out, ychw_, row * D.C, k, st_));
  } else {
    PSWA_CUDA(cudaMemcpy2DAsync(yhat_out + static_cast<size_t>(B_.r0) * D.W,
                                static_cast<size_t>(D.HW) * sizeof(int32_t), ychw_, row, row, D.C,
                                k, st_));
  }
  PSWA_CUDA(cudaMemcpyAsync(r.bits, bits_, sizeof(r.bits), cudaMemcpyDeviceToHost, st_));
  PSWA_CUDA(cudaMemcpyAsync(&r.status, status_, sizeof(int), cudaMemcpyDeviceToHost, st_));
  PSWA_CUDA(cudaStreamSynchronize(st_));
  if (r.status) throw pswa_abi::TruncatedError("corrupt or truncated payload (status " +
                                               std::to_string(r.status) + ")");
  fetch_musig(mu_out, sigma_out);
  if (advance) {
    advance_ring();
    PSWA_CUDA(cudaStreamSynchronize(st_));
  }
  return r;
}

void Engine::decode_async(const void* d_hyper, size_t hyper_len, const void* d_main,
                          size_t main_len, int rate, int fidx, int32_t* d_yhat_out, bool advance) {
  if (B_.n > 1) throw std::invalid_argument("decode_async: not for band handles");
  prep_decode(d_hyper, hyper_len, d_main, main_len, rate, fidx, true);
  run(program(decode_key(false, stats_on_)));
  have_stats_ = stats_on_;
  pswa_dev::accumulate_status(status_, sticky_status_, st_);
  PSWA_CUDA(cudaMemcpyAsync(d_yhat_out, ychw_, sizeof(int32_t) * HWo_ * D_.C,
                            cudaMemcpyDeviceToDevice, st_));
  if (advance) advance_ring();  // stream-ordered copy + host ring indices
}

FrameResult Engine::finish_async() {
  FrameResult r;
  PSWA_CUDA(cudaMemcpyAsync(r.bits, bits_, sizeof(r.bits), cudaMemcpyDeviceToHost, st_));
  PSWA_CUDA(cudaMemcpyAsync(&r.status, sticky_status_, sizeof(int), cudaMemcpyDeviceToHost, st_));
  PSWA_CUDA(cudaMemsetAsync(sticky_status_, 0, sizeof(int), st_));
  PSWA_CUDA(cudaStreamSynchronize(st_));
  if (r.status) throw pswa_abi::TruncatedError("corrupt or truncated payload in a frame since the "
                                               "last finish (status " + std::to_string(r.status) + ")");
  return r;
}

FrameResult Engine::decode(const void* hyper, size_t hyper_len, const void* main_pl, size_t main_len,
                           int rate, int fidx, bool advance, int32_t* yhat_out, bool device,
                           float* mu_out, float* sigma_out) {
  const bool taps = mu_out || sigma_out || stats_on_;
  have_stats_ = false;
  // pinned host output: the copies of finished channel groups overlap the
  // last groups' decoding (a pageable destination makes each copy blocking,
  // so it keeps the single copy at the end)
  cudaPointerAttributes pa{};
  const bool pinned = !device && cudaPointerGetAttributes(&pa, yhat_out) == cudaSuccess &&
                      pa.type == cudaMemoryTypeHost;
  if (!device) (void)cudaGetLastError();  // pageable pointers may set an error on older drivers
  if (pinned && B_.n == 1 && D_.N <= 8) {
    Program& P = program(decode_key(true, taps));
    prep_decode(hyper, hyper_len, main_pl, main_len, rate, fidx, device, true);
    run_host_copy(P, yhat_out);
    const FrameResult r = finish_decode(advance, nullptr, device, mu_out, sigma_out);
    have_stats_ = taps;
    return r;
  }
  prep_decode(hyper, hyper_len, main_pl, main_len, rate, fidx, device);
  run(program(decode_key(false, taps)));
  const FrameResult r = finish_decode(advance, yhat_out, device, mu_out, sigma_out);
  have_stats_ = taps;
  return r;
}


void Engine::last_eps(float* out_chw) {
  if (c_lrp() <= 0) throw std::invalid_argument("last_eps: the handle has no LRP transformer (lrp_blocks = 0)");
  const size_t row = static_cast<size_t>(HWo_) * sizeof(float);
  PSWA_CUDA(cudaMemcpyAsync(out_chw, eps_chw_, row * D_.C, cudaMemcpyDeviceToHost, st_));
  PSWA_CUDA(cudaStreamSynchronize(st_));
}

size_t Engine::debug_fetch(const std::string& name, void* out, size_t cap) {
  const size_t hwd = static_cast<size_t>(HWl_) * D_.d;
  const void* src = nullptr;
  size_t bytes = 0;
  if (name == "ctx") src = ctx16_, bytes = hwd * 2;
  else if (name == "emb") src = emb_cur_, bytes = hwd * 4;  // local grid in band mode
  else if (name == "hq") src = hq_, bytes = hwd * 4;
  else if (name == "s1") src = s1full_, bytes = static_cast<size_t>(D_.Hp) * D_.Wp * D_.d * 2;
  else if (name == "a") src = afull_, bytes = hwd * 4;
  else if (name == "s2") src = s2full_, bytes = hwd * 2;
  else throw std::invalid_argument("debug_fetch: unknown buffer " + name);
  if (out) {
    if (cap < bytes) throw std::invalid_argument("debug_fetch: buffer too small");
    PSWA_CUDA(cudaMemcpyAsync(out, src, bytes, cudaMemcpyDeviceToHost, st_));
    PSWA_CUDA(cudaStreamSynchronize(st_));
  }
  return bytes;
}

void Engine::last_zhat(int32_t* out) {
  PSWA_CUDA(cudaMemcpyAsync(out, zhat_, sizeof(int32_t) * D_.hc * D_.zh * D_.zw,
                            cudaMemcpyDeviceToHost, st_));
  PSWA_CUDA(cudaStreamSynchronize(st_));
}

}  // namespace pswa_host
