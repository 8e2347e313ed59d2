// Host-side checks of the drop-in headers that need no GPU (run by
// tests/test_host_api.py): validate_schedule (pswa/wavefront.h) on valid
// schedules and on deliberately broken predicates, and parallel_for
// (pswa/threading.h) semantics.
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../paper_2605_20977_b200/csrc/host/wavefront_check.h"
#include "pswa/tensor.h"
#include "pswa/threading.h"
#include "pswa/wavefront.h"

static int failures = 0;
#define EXPECT(c)                                                  \
  do {                                                             \
    if (!(c)) {                                                    \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);     \
      ++failures;                                                  \
    }                                                              \
  } while (0)

static bool has(const std::string& s, const char* sub) { return s.find(sub) != std::string::npos; }

int main() {
  using namespace pswa;
  // valid schedules, s*N phases at every size
  for (int hw : {8, 16, 64}) {
    const ScheduleReport r = validate_schedule(hw, hw, 4, 7, 7, 4);
    EXPECT(r.ok);
    EXPECT(r.sequential_steps == 16);
  }
  for (int s = 1; s <= 8; ++s)
    for (int hw : {1, 5, 13, 32}) EXPECT(validate_schedule(hw, hw + 3, s, 7, 7, 4).ok);
  EXPECT(validate_schedule(16, 16, 1, 7, 7, 1).sequential_steps == 1);
  EXPECT(validate_schedule(68, 120, 4, 7, 7, 4).ok);
  // preconditions
  EXPECT(!validate_schedule(8, 8, 4, 6, 7, 4).ok);
  EXPECT(has(validate_schedule(8, 8, 0, 7, 7, 4).first_violation, "precondition"));
  // broken predicates are reported
  auto acc_le = [](MaskKind k, Pos q, Pos p, int s) {
    return k == MaskKind::kAccumulator ? step_of(p, s) <= step_of(q, s) : mask_allows(k, q, p, s);
  };
  ScheduleReport r = detail::validate_schedule_with(8, 8, 4, 7, 7, 4, acc_le, channel_mask);
  EXPECT(!r.ok && has(r.first_violation, "accumulator edge"));
  auto self_all = [](MaskKind k, Pos q, Pos p, int s) {
    return k == MaskKind::kSpatialSelf ? true : mask_allows(k, q, p, s);
  };
  r = detail::validate_schedule_with(8, 8, 4, 7, 7, 4, self_all, channel_mask);
  EXPECT(!r.ok && has(r.first_violation, "spatial_self"));
  auto cm_full = [](int n, int dg) { return std::vector<uint8_t>(size_t(n * dg) * n * dg, 1); };
  r = detail::validate_schedule_with(8, 8, 4, 7, 7, 4, mask_allows, cm_full);
  EXPECT(!r.ok && has(r.first_violation, "channel order"));
  // a predicate whose edges look backward but ignores the step entirely for
  // the accumulator's own position: only the dataflow closure catches it
  auto acc_self = [](MaskKind k, Pos q, Pos p, int s) {
    if (k == MaskKind::kAccumulator && q == p) return true;
    return mask_allows(k, q, p, s);
  };
  r = detail::validate_schedule_with(8, 8, 4, 7, 7, 4, acc_self, channel_mask);
  EXPECT(!r.ok);
  // channel_mask
  const std::vector<uint8_t> m = channel_mask(2, 1);
  EXPECT(m == (std::vector<uint8_t>{1, 0, 1, 1}));

  // parallel_for: every index exactly once, any worker count, nesting
  for (int w : {1, 3, 8}) {
    set_workers(w);
    EXPECT(workers() == w);
    const int n = 10007;
    std::vector<std::atomic<int>> hits(n);
    for (auto& h : hits) h = 0;
    parallel_for(0, n, [&](int64_t i) { hits[size_t(i)]++; });
    bool once = true;
    for (auto& h : hits) once = once && h.load() == 1;
    EXPECT(once);
    std::vector<double> out(1000);
    parallel_for(0, 1000, [&](int64_t i) {
      double acc = 0;
      parallel_for(0, 10, [&](int64_t j) { acc += double(i * 10 + j); });  // nested: serial
      out[size_t(i)] = acc;
    });
    bool ok = true;
    for (int i = 0; i < 1000; ++i) ok = ok && out[size_t(i)] == double(100 * i + 45);
    EXPECT(ok);
  }
  parallel_for(5, 5, [&](int64_t) { ++failures; });  // empty range runs nothing
  set_workers(0);
  EXPECT(workers() == 1);
  // host-only parts of tensor.h
  EXPECT(ffn_hidden_dim(512) == 1368 && ffn_hidden_dim(64) == 168 && ffn_hidden_dim(1) == 8);
  Tensor t({2, 3});
  EXPECT(t.numel() == 6 && t.same_bytes(t) && t.all_finite());
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "ok", failures);
  return failures ? 1 : 0;
}
