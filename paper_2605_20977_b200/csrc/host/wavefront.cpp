// Host implementation of pswa/wavefront.h. The engine's
// device schedule is derived from the same predicates: the per-step position
// tables are in positions_of_step order (engine.cpp build_tables), and the
// attention tap tables exclude exactly the keys mask_allows rejects
// (engine.cpp add_shape calls it).
#include "pswa/wavefront.h"

#include <algorithm>
#include <functional>
#include <string>

#include "wavefront_check.h"

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
    for (int i = 0; i < n; ++i) m[static_cast<size_t>(o) * n + i] = (i / group_dim) <= (o / group_dim);
  return m;
}

ScheduleReport validate_schedule(int h, int w, int s, int wh, int ww, int n_groups) {
  return detail::validate_schedule_with(h, w, s, wh, ww, n_groups, mask_allows, channel_mask);
}

namespace detail {

// The symbol dependency graph is derived from the network's dataflow
// (SPEC.md:311-372), each attention edge filtered by the predicate its layer
// uses: S1 self-attention over embedded y_hat (kSpatialSelf), the
// accumulator's cross-attention from Hq into S1 (kAccumulator), S2
// self-attention over the accumulator output (kSpatialSelf), then the channel
// transformer at the position (slot g carries y_hat group g-1, mixed under
// channel_mask). The hyperprior path and the context (past frames) carry no
// current-frame y_hat. For every stage and position, dep[] is the latest
// decode step of any y_hat position the stage can see; attention stacks are
// iterated to their fixed point (unbounded depth: a superset of what any
// block count reads). Topological order then means: every symbol (p, g)
// depends on y_hat positions of strictly earlier steps only -- which rank
// before it in the canonical order (step-major, group, raster) -- plus y_hat
// groups < g of its own position.
ScheduleReport validate_schedule_with(int h, int w, int s, int wh, int ww, int n_groups,
                                      const MaskFn& allows, const ChannelMaskFn& cmask) {
  ScheduleReport r;
  auto fail = [&](const std::string& what) {
    if (r.ok) r.first_violation = what;
    r.ok = false;
  };
  if (h < 1 || w < 1 || s < 1 || n_groups < 1 || wh < 1 || ww < 1 || wh % 2 == 0 || ww % 2 == 0) {
    fail("precondition: grid, s and N >= 1 and odd window extents required (got " + std::to_string(h) +
         "x" + std::to_string(w) + ", s=" + std::to_string(s) + ", window " + std::to_string(wh) + "x" +
         std::to_string(ww) + ", N=" + std::to_string(n_groups) + ")");
    return r;
  }
  r.sequential_steps = s * n_groups;
  const int ry = wh / 2, rx = ww / 2;
  auto pos_str = [](Pos p) { return "(" + std::to_string(p.y) + "," + std::to_string(p.x) + ")"; };
  // (a), (b): the predicates' edges in every window
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x)
      for (int ky = std::max(0, y - ry); ky <= std::min(h - 1, y + ry); ++ky)
        for (int kx = std::max(0, x - rx); kx <= std::min(w - 1, x + rx); ++kx) {
          const Pos q{y, x}, k{ky, kx};
          const int qs = step_of(q, s), ks = step_of(k, s);
          if (allows(MaskKind::kAccumulator, q, k, s) && !(ks < qs))
            fail("accumulator edge not strictly backward: q=" + pos_str(q) + " k=" + pos_str(k));
          if (allows(MaskKind::kSpatialSelf, q, k, s) && ks > qs)
            fail("spatial_self edge goes forward: q=" + pos_str(q) + " k=" + pos_str(k));
        }
  // (c) dependency closure over the dataflow
  const size_t HW = static_cast<size_t>(h) * w;
  constexpr int kNone = -1;
  auto attend = [&](const std::vector<int>& in, MaskKind kind, bool fixpoint) {
    std::vector<int> cur = in, out(HW, kNone);
    for (int iter = 0;; ++iter) {
      bool changed = false;
      for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
          int m = fixpoint ? cur[static_cast<size_t>(y) * w + x] : kNone;
          for (int ky = std::max(0, y - ry); ky <= std::min(h - 1, y + ry); ++ky)
            for (int kx = std::max(0, x - rx); kx <= std::min(w - 1, x + rx); ++kx)
              if (allows(kind, Pos{y, x}, Pos{ky, kx}, s)) m = std::max(m, cur[static_cast<size_t>(ky) * w + kx]);
          int& o = out[static_cast<size_t>(y) * w + x];
          if (m != o) {
            o = m;
            changed = true;
          }
        }
      if (!fixpoint || !changed || iter > h + w) return out;
      cur = out;  // residual stream: the next block sees this block's output
    }
  };
  std::vector<int> emb(HW);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) emb[static_cast<size_t>(y) * w + x] = step_of(Pos{y, x}, s);
  const std::vector<int> s1 = attend(emb, MaskKind::kSpatialSelf, true);
  const std::vector<int> acc = attend(s1, MaskKind::kAccumulator, false);
  const std::vector<int> s2 = attend(acc, MaskKind::kSpatialSelf, true);
  int margin = s;  // smallest step distance between a symbol and its y_hat inputs
  for (int y = 0; y < h && r.ok; ++y)
    for (int x = 0; x < w && r.ok; ++x) {
      const int qs = step_of(Pos{y, x}, s), dep = s2[static_cast<size_t>(y) * w + x];
      if (dep != kNone) margin = std::min(margin, qs - dep);
      if (dep >= qs)
        fail("decode order not topological: the symbols of " + pos_str(Pos{y, x}) + " (step " +
             std::to_string(qs) + ") depend on y_hat decoded at step " + std::to_string(dep));
    }
  // channel edges at one position: output slot g mixes input slots gi with
  // cmask(g, gi); input slot gi >= 1 carries y_hat group gi - 1
  const std::vector<uint8_t> cm = cmask(n_groups, 1);
  for (int g = 0; g < n_groups && r.ok; ++g)
    for (int gi = 1; gi < n_groups; ++gi)
      if (cm[static_cast<size_t>(g) * n_groups + gi] && gi - 1 >= g)
        fail("channel order not topological: group " + std::to_string(g) + " reads y_hat group " +
             std::to_string(gi - 1));
  r.lines.push_back("grid " + std::to_string(h) + "x" + std::to_string(w) + " s=" + std::to_string(s) +
                    " window " + std::to_string(wh) + "x" + std::to_string(ww) + " N=" +
                    std::to_string(n_groups) + ": " + std::to_string(r.sequential_steps) +
                    " sequential phases (raster: " + std::to_string(HW * n_groups) + ")");
  r.lines.push_back(r.ok ? "every symbol depends on y_hat of strictly earlier steps (>= " +
                               std::to_string(margin) + " back) and of lower groups at its position"
                         : "violation: " + r.first_violation);
  return r;
}

}  // namespace detail
}  // namespace pswa

// ---- C ABI ------------------------------------------------------------------
#include <cstring>

#include "abi_util.h"
#include "pswa/pswa_cuda.h"

extern "C" int pswa_validate_schedule(int h, int w, int s, int wh, int ww, int n_groups, int* ok,
                                      int* sequential_steps, char* first_violation, size_t cap) {
  return pswa_abi::guard([&] {
    if (static_cast<long>(h) * w > (1L << 24)) throw std::invalid_argument("validate_schedule: grid too large");
    const pswa::ScheduleReport r = pswa::validate_schedule(h, w, s, wh, ww, n_groups);
    *ok = r.ok ? 1 : 0;
    *sequential_steps = r.sequential_steps;
    if (first_violation && cap) {
      std::strncpy(first_violation, r.first_violation.c_str(), cap - 1);
      first_violation[cap - 1] = '\0';
    }
  });
}
