// C ABI: frame-level entry points (include/pswa/pswa_cuda.h).
#include <cuda_runtime.h>

#include <cstring>
#include <memory>

#include "../cuda/check.h"
#include "../cuda/gemm.h"
#include "../cuda/kernels.h"
#include "abi_util.h"
#include "engine.h"
#include "container.h"
#include "group.h"
#include "pswa/rng.h"
#include "model_spec.h"
#include "pswa/pswa_cuda.h"

struct pswa_gpu {
  std::unique_ptr<pswa_host::Engine> eng;
  pswa_cfg cfg{};
  uint64_t weights_hash = 0;
};
struct pswa_group {
  std::unique_ptr<pswa_host::BandGroup> grp;
};

using pswa_abi::guard;

extern "C" {

void pswa_cfg_preset(pswa_cfg* c, int preset, int height, int width) {
  std::memset(c, 0, sizeof(*c));
  const bool paper = preset != 0;
  c->d_spatial = paper ? 512 : 64;
  c->heads = 16;
  c->ctx_blocks = c->s1_blocks = c->s2_blocks = paper ? 8 : 2;
  c->d_channel = paper ? 1024 : 128;
  c->ch_blocks = 2;
  c->hyper_ch = paper ? 128 : 32;
  c->latent_ch = 192;
  c->s = 4;
  c->n_groups = 4;
  c->win_h = c->win_w = 7;
  c->win_t = 5;
  c->ctx_slots = 4;
  c->rate_points = 4;
  c->height = height;
  c->width = width;
  c->lanes = 1;
  c->hyper_lanes = 1;
}

int pswa_gen_weights(const pswa_cfg* cfg, uint64_t seed, void* buf, size_t cap, size_t* len) {
  return guard([&] {
    const auto blob = pswa_host::gen_weights_psww(*cfg, seed);
    *len = blob.size();
    if (buf) {
      if (cap < blob.size()) throw std::invalid_argument("pswa_gen_weights: buffer too small");
      std::memcpy(buf, blob.data(), blob.size());
    }
  });
}

int pswa_synth_latent(const pswa_cfg* cfg, int gop, int frame_idx, int32_t* out) {
  return guard([&] {
    pswa_host::validate_cfg(*cfg);
    pswa_host::synth_latent(*cfg, gop, frame_idx, out);
  });
}

int pswa_synth_gop(const pswa_cfg* cfg, int gop, int n_frames, int32_t* out) {
  return guard([&] {
    pswa_host::validate_cfg(*cfg);
    if (n_frames < 0) throw std::invalid_argument("n_frames < 0");
    pswa_host::synth_gop(*cfg, gop, n_frames, out);
  });
}

int pswa_gpu_create(int device, const pswa_cfg* cfg, const void* blob, size_t len, pswa_gpu** out) {
  *out = nullptr;
  return guard([&] {
    auto h = std::make_unique<pswa_gpu>();
    h->eng = std::make_unique<pswa_host::Engine>(device, *cfg, blob, len);
    h->cfg = *cfg;
    h->weights_hash = pswa::fnv1a64(blob, len);
    *out = h.release();
  });
}

void pswa_gpu_destroy(pswa_gpu* h) {
  if (!h) return;
  try {
    pswa_dev::DeviceScope ds(h->eng->device());
    delete h;
  } catch (...) {
    delete h;
  }
}

int pswa_gpu_create_band(int device, const pswa_cfg* cfg, const void* blob, size_t len, int band_idx,
                         int n_bands, pswa_gpu** out) {
  *out = nullptr;
  return guard([&] {
    auto h = std::make_unique<pswa_gpu>();
    h->eng = std::make_unique<pswa_host::Engine>(device, *cfg, blob, len, band_idx, n_bands);
    *out = h.release();
  });
}

int pswa_gpu_band_export(pswa_gpu* h, void* out, size_t cap, size_t* len) {
  return guard([&] {
    pswa_dev::DeviceScope ds(h->eng->device());
    const auto b = h->eng->ipc_export();
    *len = b.size();
    if (out) {
      if (cap < b.size()) throw std::invalid_argument("pswa_gpu_band_export: buffer too small");
      std::memcpy(out, b.data(), b.size());
    }
  });
}

int pswa_gpu_band_link(pswa_gpu* h, const void* up, size_t up_len, const void* down, size_t down_len) {
  return guard([&] {
    pswa_dev::DeviceScope ds(h->eng->device());
    h->eng->link_ipc(static_cast<const uint8_t*>(up), up_len, static_cast<const uint8_t*>(down),
                     down_len);
  });
}

int pswa_gpu_reset_gop(pswa_gpu* h) {
  return guard([&] {
    pswa_dev::DeviceScope ds(h->eng->device());
    h->eng->reset_gop();
  });
}

int pswa_gpu_push_frame(pswa_gpu* h, const int32_t* yhat, int rate_idx) {
  return guard([&] {
    pswa_dev::DeviceScope ds(h->eng->device());
    h->eng->push_frame(yhat, rate_idx);
  });
}

int pswa_gpu_encode_frame(pswa_gpu* h, const int32_t* yhat, int rate_idx, int frame_idx_in_gop,
                          uint8_t* hyper_out, size_t hyper_cap, size_t* hyper_len,
                          uint8_t* main_out, size_t main_cap, size_t* main_len, double* bits_out) {
  return guard([&] {
    pswa_dev::DeviceScope ds(h->eng->device());
    const auto r = h->eng->encode(yhat, rate_idx, frame_idx_in_gop, nullptr, nullptr, nullptr,
                                  hyper_out, hyper_cap, main_out, main_cap, /*advance=*/true);
    *hyper_len = r.hyper_len;
    *main_len = r.main_len;
    if (bits_out) {
      bits_out[0] = r.bits[0];
      bits_out[1] = r.bits[1];
    }
  });
}

int pswa_gpu_decode_frame(pswa_gpu* h, const uint8_t* hyper, size_t hyper_len,
                          const uint8_t* main_payload, size_t main_len, int rate_idx,
                          int frame_idx_in_gop, int advance_state, int32_t* yhat_out,
                          float* mu_out, float* sigma_out, double* bits_out) {
  return guard([&] {
    pswa_dev::DeviceScope ds(h->eng->device());
    const auto r = h->eng->decode(hyper, hyper_len, main_payload, main_len, rate_idx,
                                  frame_idx_in_gop, advance_state != 0, yhat_out, false, mu_out,
                                  sigma_out);
    if (bits_out) {
      bits_out[0] = r.bits[0];
      bits_out[1] = r.bits[1];
    }
  });
}

int pswa_gpu_decode_frame_device(pswa_gpu* h, const void* d_hyper, size_t hyper_len,
                                 const void* d_main, size_t main_len, int rate_idx,
                                 int frame_idx_in_gop, int advance_state, void* d_yhat_out) {
  return guard([&] {
    pswa_dev::DeviceScope ds(h->eng->device());
    h->eng->decode(d_hyper, hyper_len, d_main, main_len, rate_idx, frame_idx_in_gop,
                   advance_state != 0, static_cast<int32_t*>(d_yhat_out), true);
  });
}

int pswa_gpu_decode_frame_async(pswa_gpu* h, const void* d_hyper, size_t hyper_len,
                                const void* d_main, size_t main_len, int rate_idx,
                                int frame_idx_in_gop, int advance_state, void* d_yhat_out) {
  return guard([&] {
    pswa_dev::DeviceScope ds(h->eng->device());
    h->eng->decode_async(d_hyper, hyper_len, d_main, main_len, rate_idx, frame_idx_in_gop,
                         static_cast<int32_t*>(d_yhat_out), advance_state != 0);
  });
}

int pswa_gpu_finish(pswa_gpu* h, double* bits_out) {
  return guard([&] {
    pswa_dev::DeviceScope ds(h->eng->device());
    const auto r = h->eng->finish_async();
    if (bits_out) {
      bits_out[0] = r.bits[0];
      bits_out[1] = r.bits[1];
    }
  });
}

int pswa_gpu_forward_params(pswa_gpu* h, const int32_t* yhat, const int32_t* zhat, int rate_idx,
                            int frame_idx_in_gop, float* mu_out, float* sigma_out,
                            double* bits_out) {
  return guard([&] {
    pswa_dev::DeviceScope ds(h->eng->device());
    if (!mu_out || !sigma_out) throw std::invalid_argument("mu_out / sigma_out required");
    const auto r = h->eng->encode(yhat, rate_idx, frame_idx_in_gop, zhat, mu_out, sigma_out,
                                  nullptr, 0, nullptr, 0, /*advance=*/false);
    if (bits_out) {
      bits_out[0] = r.bits[0];
      bits_out[1] = r.bits[1];
    }
  });
}

int pswa_gpu_set_stats(pswa_gpu* h, int on) {
  return guard([&] { h->eng->set_stats(on != 0); });
}

int pswa_gpu_last_bitstats(pswa_gpu* h, double* out) {
  return guard([&] {
    pswa_dev::DeviceScope ds(h->eng->device());
    h->eng->last_bitstats(out);
  });
}

int pswa_gpu_last_eps(pswa_gpu* h, float* eps_out) {
  return guard([&] {
    pswa_dev::DeviceScope ds(h->eng->device());
    h->eng->last_eps(eps_out);
  });
}

int pswa_gpu_last_zhat(pswa_gpu* h, int32_t* zhat_out) {
  return guard([&] {
    pswa_dev::DeviceScope ds(h->eng->device());
    h->eng->last_zhat(zhat_out);
  });
}

int pswa_gpu_debug_fetch(pswa_gpu* h, const char* name, void* out, size_t cap, size_t* bytes) {
  return guard([&] {
    pswa_dev::DeviceScope ds(h->eng->device());
    *bytes = h->eng->debug_fetch(name, out, cap);
  });
}

int pswa_gpu_last_launch_count(pswa_gpu* h) { return h->eng->last_launches(); }

int pswa_gpu_bench_op(pswa_gpu* h, const char* name, int reps, double* us, double* flops) {
  return guard([&] {
    pswa_dev::DeviceScope ds(h->eng->device());
    *us = h->eng->bench_op(name, reps, flops);
  });
}

int pswa_gpu_bench_probe(pswa_gpu* h, const char* name, int reps, double* us, double* flops,
                         double* bytes) {
  return guard([&] {
    pswa_dev::DeviceScope ds(h->eng->device());
    *us = h->eng->bench_op(name, reps, flops, bytes);
  });
}

int pswa_gpu_probe_list(pswa_gpu* h, char* out, size_t cap, size_t* len) {
  return guard([&] {
    const std::string s = h->eng->probe_list();
    *len = s.size() + 1;
    if (out) {
      if (cap < s.size() + 1) throw std::invalid_argument("probe_list: buffer too small");
      std::memcpy(out, s.c_str(), s.size() + 1);
    }
  });
}

void* pswa_gpu_stream(pswa_gpu* h) { return h->eng->stream(); }

// Debug export for tools/gemm_trace.py (not part of the public header):
// the per-CTA phase stamps of the last GEMM launch when PSWA_GEMM_TRACE is
// set; returns 0, or 1 when tracing is off.
extern "C" __attribute__((visibility("default"))) int pswa_debug_gemm_trace(unsigned long long* out, int n) {
  return guard([&] {
    if (!pswa_dev::gemm_trace_read(out, n)) throw std::invalid_argument("PSWA_GEMM_TRACE is not set");
  });
}

// Debug export for tools/gemm_trace.py: GEMM timing experiments (trace
// builds only; see pswa_dev::gemm_set_experiment).
extern "C" __attribute__((visibility("default"))) int pswa_debug_gemm_experiment(int flags) {
  return guard([&] { pswa_dev::gemm_set_experiment(flags); });
}

// ---- sequences ----------------------------------------------------------------
int pswa_gpu_encode_sequence(pswa_gpu* h, const int32_t* frames, int n_frames, int gop_size,
                             int rate_idx, uint8_t* out, size_t cap, size_t* len) {
  return guard([&] {
    pswa_dev::DeviceScope ds(h->eng->device());
    if (n_frames < 0 || gop_size < 1) throw std::invalid_argument("n_frames / gop_size");
    const pswa_cfg& c = h->cfg;
    pswa_host::ContainerHeader hd;
    hd.w_px = static_cast<uint32_t>(c.width) * 16;
    hd.h_px = static_cast<uint32_t>(c.height) * 16;
    hd.frames = static_cast<uint32_t>(n_frames);
    hd.gop = static_cast<uint32_t>(gop_size);
    hd.rate = static_cast<uint32_t>(rate_idx);
    hd.s = static_cast<uint32_t>(c.s);
    hd.N = static_cast<uint32_t>(c.n_groups);
    hd.cfg_hash = pswa_host::stream_cfg_hash(c, 1);
    hd.weights_hash = h->weights_hash;
    hd.prior = static_cast<uint32_t>(c.prior);
    std::vector<uint8_t> o;
    pswa_host::write_header(o, hd);
    const size_t fsz = static_cast<size_t>(c.latent_ch) * c.height * c.width;
    const size_t pcap = 20 * fsz + (1 << 20);
    std::vector<uint8_t> hb(pcap), mb(pcap);
    for (int f = 0; f < n_frames; ++f) {
      if (f % gop_size == 0) h->eng->reset_gop();
      const auto r = h->eng->encode(frames + f * fsz, rate_idx, f % gop_size, nullptr, nullptr,
                                    nullptr, hb.data(), pcap, mb.data(), pcap, true);
      pswa_host::append_frame(o, hb.data(), r.hyper_len, mb.data(), r.main_len);
    }
    *len = o.size();
    if (out) {
      if (cap < o.size()) throw std::invalid_argument("encode_sequence: output buffer too small");
      std::memcpy(out, o.data(), o.size());
    }
  });
}

int pswa_gpu_decode_sequence(pswa_gpu* h, const uint8_t* cont, size_t len, int32_t* frames_out,
                             int max_frames, int* frame_status, double* bits_out, int* n_frames) {
  return guard([&] {
    pswa_dev::DeviceScope ds(h->eng->device());
    std::vector<pswa_host::FrameRef> fr;
    const auto hd = pswa_host::parse_container(cont, len, &fr);
    const pswa_cfg& c = h->cfg;
    if (hd.cfg_hash != pswa_host::stream_cfg_hash(c, static_cast<int>(hd.n_bands)) || hd.n_bands != 1)
      throw pswa_abi::HashError("decode_sequence: stream config differs from the handle's");
    if (hd.weights_hash != h->weights_hash)
      throw pswa_abi::HashError("decode_sequence: stream was coded with other weights");
    const int n = static_cast<int>(fr.size());
    if (n > max_frames) throw std::invalid_argument("decode_sequence: output buffer too small");
    const size_t fsz = static_cast<size_t>(c.latent_ch) * c.height * c.width;
    int resume = 0;  // first frame to attempt (after a failure: the next GOP start)
    for (int f = 0; f < n; ++f) {
      if (frame_status) frame_status[f] = -1;
      if (f < resume) continue;
      const int fidx = static_cast<int>(f % hd.gop);
      if (fidx == 0) h->eng->reset_gop();
      try {
        const auto r = h->eng->decode(cont + fr[f].hyper_off, fr[f].hyper_len, cont + fr[f].main_off,
                                      fr[f].main_len, static_cast<int>(hd.rate), fidx, true,
                                      frames_out + f * fsz, false);
        if (frame_status) frame_status[f] = 0;
        if (bits_out) {
          bits_out[2 * f] = r.bits[0];
          bits_out[2 * f + 1] = r.bits[1];
        }
      } catch (const pswa_abi::TruncatedError&) {
        if (frame_status) frame_status[f] = PSWA_E_TRUNCATED;
        resume = static_cast<int>((f / hd.gop + 1) * hd.gop);
      }
    }
    *n_frames = n;
  });
}

int pswa_container_info(const uint8_t* cont, size_t len, int* info) {
  return guard([&] {
    std::vector<pswa_host::FrameRef> fr;
    const auto hd = pswa_host::parse_container(cont, len, &fr);
    const int v[10] = {pswa_host::kContainerVersion, static_cast<int>(hd.w_px), static_cast<int>(hd.h_px),
                       static_cast<int>(hd.frames), static_cast<int>(hd.gop), static_cast<int>(hd.rate),
                       static_cast<int>(hd.s), static_cast<int>(hd.N), static_cast<int>(hd.prior),
                       static_cast<int>(fr.size())};
    std::memcpy(info, v, sizeof(v));
  });
}

// ---- row bands --------------------------------------------------------------
int pswa_band_rows(int height, int n_bands, int band_idx, int* row0, int* row1) {
  return guard([&] { pswa_host::band_rows(height, n_bands, band_idx, row0, row1); });
}

int pswa_group_create(const int* devices, int n_bands, const pswa_cfg* cfg, const void* blob,
                      size_t len, pswa_group** out) {
  *out = nullptr;
  return guard([&] {
    if (n_bands < 1) throw std::invalid_argument("n_bands < 1");
    auto g = std::make_unique<pswa_group>();
    g->grp = std::make_unique<pswa_host::BandGroup>(std::vector<int>(devices, devices + n_bands),
                                                    *cfg, blob, len);
    *out = g.release();
  });
}

void pswa_group_destroy(pswa_group* g) { delete g; }

int pswa_group_reset_gop(pswa_group* g) {
  return guard([&] {
    pswa_dev::DeviceScope ds(g->grp->band(0).device());
    g->grp->reset_gop();
  });
}

int pswa_group_push_frame(pswa_group* g, const int32_t* yhat, int rate_idx) {
  return guard([&] {
    pswa_dev::DeviceScope ds(g->grp->band(0).device());
    g->grp->push_frame(yhat, rate_idx);
  });
}

int pswa_group_encode_frame(pswa_group* g, const int32_t* yhat, const int32_t* zhat, int rate_idx,
                            int frame_idx_in_gop, uint8_t* hyper_out, size_t hyper_cap,
                            size_t* hyper_len, uint8_t* main_out, size_t main_cap, size_t* main_len,
                            double* bits_out) {
  return guard([&] {
    pswa_dev::DeviceScope ds(g->grp->band(0).device());
    const auto r = g->grp->encode(yhat, rate_idx, frame_idx_in_gop, zhat, nullptr, nullptr,
                                  hyper_out, hyper_cap, main_out, main_cap, /*advance=*/true);
    *hyper_len = r.hyper_len;
    *main_len = r.main_len;
    if (bits_out) {
      bits_out[0] = r.bits[0];
      bits_out[1] = r.bits[1];
    }
  });
}

int pswa_group_decode_frame(pswa_group* g, const uint8_t* hyper, size_t hyper_len,
                            const uint8_t* main_payload, size_t main_len, int rate_idx,
                            int frame_idx_in_gop, int advance_state, int32_t* yhat_out,
                            double* bits_out) {
  return guard([&] {
    pswa_dev::DeviceScope ds(g->grp->band(0).device());
    const auto r = g->grp->decode(hyper, hyper_len, main_payload, main_len, rate_idx,
                                  frame_idx_in_gop, advance_state != 0, yhat_out);
    if (bits_out) {
      bits_out[0] = r.bits[0];
      bits_out[1] = r.bits[1];
    }
  });
}

int pswa_group_forward_params(pswa_group* g, const int32_t* yhat, const int32_t* zhat, int rate_idx,
                              int frame_idx_in_gop, float* mu_out, float* sigma_out,
                              double* bits_out) {
  return guard([&] {
    pswa_dev::DeviceScope ds(g->grp->band(0).device());
    if (!mu_out || !sigma_out || !zhat) throw std::invalid_argument("zhat / mu_out / sigma_out required");
    const auto r = g->grp->encode(yhat, rate_idx, frame_idx_in_gop, zhat, mu_out, sigma_out, nullptr,
                                  0, nullptr, 0, /*advance=*/false);
    if (bits_out) {
      bits_out[0] = r.bits[0];
      bits_out[1] = r.bits[1];
    }
  });
}

int pswa_group_last_zhat(pswa_group* g, int32_t* zhat_out) {
  return guard([&] {
    pswa_dev::DeviceScope ds(g->grp->band(0).device());
    g->grp->band(0).last_zhat(zhat_out);
  });
}

int pswa_group_last_launch_count(pswa_group* g) { return g->grp->last_launches(); }

// ---- operator-level -------------------------------------------------------
int pswa_gpu_op_rmsnorm(const float* x, int ld_x, int M, int d, int group, const float* gain,
                        void* y, int ld_y, void* stream) {
  return guard([&] {
    pswa_dev::rmsnorm_rows(x, ld_x, nullptr, M, d, group, gain, static_cast<__half*>(y), ld_y,
                           static_cast<cudaStream_t>(stream));
  });
}

int pswa_gpu_op_window_attn(const void* q, int ld_q, const int32_t* qinfo, int Mq, const void* kv,
                            int ld_kv, int kv_slot_stride, int H, int W, int heads, int head_dim,
                            int win_h, int win_w, int win_t, int mask, int s, const float* bias,
                            void* out, int ld_out, void* stream) {
  return guard([&] {
    pswa_dev::window_attention(static_cast<const __half*>(q), ld_q, qinfo, Mq,
                               static_cast<const __half*>(kv), ld_kv, kv_slot_stride, H, W, heads,
                               head_dim, win_h, win_w, win_t, mask, s, bias,
                               static_cast<__half*>(out), ld_out, static_cast<cudaStream_t>(stream));
  });
}

int pswa_gpu_op_build_cdf(uint32_t* cdf_out, float* scales_out) {
  return pswa_gpu_op_build_cdf_family(cdf_out, scales_out, 0);
}

int pswa_gpu_op_build_cdf_family(uint32_t* cdf_out, float* scales_out, int laplace) {
  return guard([&] {
    float* ds = nullptr;
    uint32_t* dc = nullptr;
    PSWA_CUDA(cudaMalloc(&ds, sizeof(float) * pswa_dev::kScales));
    PSWA_CUDA(cudaMalloc(&dc, sizeof(uint32_t) * pswa_dev::kCdfWords));
    pswa_dev::build_cdf_tables(ds, dc, nullptr, laplace);
    PSWA_CUDA(cudaMemcpy(scales_out, ds, sizeof(float) * pswa_dev::kScales, cudaMemcpyDeviceToHost));
    PSWA_CUDA(cudaMemcpy(cdf_out, dc, sizeof(uint32_t) * pswa_dev::kScales * (pswa_dev::kSyms + 1),
                         cudaMemcpyDeviceToHost));
    cudaFree(ds);
    cudaFree(dc);
  });
}

}  // extern "C"
