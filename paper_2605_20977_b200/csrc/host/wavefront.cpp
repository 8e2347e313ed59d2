// Host implementation of pswa/wavefront.h.
#include "pswa/wavefront.h"

namespace pswa {

bool mask_allows(MaskKind kind, Pos q, Pos k, int s) {
  switch (kind) {
    case MaskKind::kSpatialSelf: return step_of(k, s) <= step_of(q, s);
    case MaskKind::kAccumulator: return step_of(k, s) < step_of(q, s);
    case MaskKind::kTemporalCausal: return k.y < q.y;
    case MaskKind::kChannelBlockLt: return k.y <= q.y;
  }
  return false;
}

std::vector<Pos> positions_of_step(int h, int w, int s, int t) {
  std::vector<Pos> v;
  for (int y = 0; y < h; ++y)
    for (int x = ((t - y) % s + s) % s; x < w; x += s) v.push_back({y, x});
  return v;
}

std::vector<uint8_t> channel_mask(int n_groups, int group_dim) {
  const int n = n_groups * group_dim;
  std::vector<uint8_t> m(static_cast<size_t>(n) * n, 0);
  for (int o = 0; o < n; ++o)
    for (int i = 0; i <= (o / group_dim + 1) * group_dim - 1; ++i) m[static_cast<size_t>(o) * n + i] = 1;
  return m;
}

ScheduleReport validate_schedule(int h, int w, int s, int wh, int ww, int n_groups) {
  ScheduleReport r;
  r.sequential_steps = s * n_groups;
  auto fail = [&](const std::string& what, int y, int x, int ky, int kx) {
    if (!r.ok) return;
    r.ok = false;
    r.first_violation = what + " at q=(" + std::to_string(y) + "," + std::to_string(x) + ") k=(" +
                        std::to_string(ky) + "," + std::to_string(kx) + ")";
  };
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x)
      for (int ky = y - wh / 2; ky <= y + wh / 2; ++ky)
        for (int kx = x - ww / 2; kx <= x + ww / 2; ++kx) {
          if (ky < 0 || kx < 0 || ky >= h || kx >= w) continue;
          const Pos q{y, x}, k{ky, kx};
          if (mask_allows(MaskKind::kAccumulator, q, k, s) && step_of(k, s) >= step_of(q, s))
            fail("accumulator edge not strictly backward", y, x, ky, kx);
          if (mask_allows(MaskKind::kSpatialSelf, q, k, s) && step_of(k, s) > step_of(q, s))
            fail("spatial_self edge goes forward", y, x, ky, kx);
        }
  r.lines.push_back("grid " + std::to_string(h) + "x" + std::to_string(w) + " s=" +
                    std::to_string(s) + " N=" + std::to_string(n_groups) + ": " +
                    std::to_string(r.sequential_steps) + " sequential phases");
  return r;
}

}  // namespace pswa
