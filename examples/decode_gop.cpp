// A reference-side C++ caller of the drop-in: encodes a short synthetic GOP
// with one device handle and decodes it with another through
// pswa::encode_frame / pswa::decode_frame_wavefront (include/pswa/pipeline.h),
// checking the decoded latents are bit-exact. Build: see INTEGRATION.md.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "pswa/pipeline.h"

int main(int argc, char** argv) {
  const int H = argc > 1 ? std::atoi(argv[1]) : 16, W = argc > 2 ? std::atoi(argv[2]) : 16;
  const int preset = argc > 3 ? std::atoi(argv[3]) : 0, frames = argc > 4 ? std::atoi(argv[4]) : 3;
  pswa_cfg cfg;
  pswa_cfg_preset(&cfg, preset, H, W);
  cfg.lanes = 64;
  cfg.hyper_lanes = 16;
  size_t n = 0;
  pswa::throw_on(pswa_gen_weights(&cfg, 1, nullptr, 0, &n));
  std::vector<uint8_t> psww(n);
  pswa::throw_on(pswa_gen_weights(&cfg, 1, psww.data(), n, &n));
  pswa::GpuCodec enc(0, cfg, psww), dec(0, cfg, psww);
  enc.set_stats(true);
  for (int f = 0; f < frames; ++f) {
    std::vector<int32_t> y(enc.latent_count());
    pswa::throw_on(pswa_synth_latent(&cfg, 0, f, y.data()));
    const pswa::EncodedFrame e = pswa::encode_frame(enc, y, 0, f, true);
    const pswa::DecodedFrame d = pswa::decode_frame_wavefront(dec, e.payloads, 0, f, 1);
    if (d.yhat != y) {
      std::printf("frame %d: MISMATCH\n", f);
      return 1;
    }
    double sum = 0.0;  // BitStats: per-position, per-group bits add up to the main estimate
    for (double v : e.stats.per_position_group) sum += v;
    std::printf("frame %d ok: %zu+%zu bytes, %.0f bits (enc %.0f, BitStats sum %.0f)\n", f,
                e.payloads.hyper.size(), e.payloads.main.size(), d.bits.hyper + d.bits.main,
                e.stats.totals.hyper + e.stats.totals.main, sum);
  }
  return 0;
}
