// pswa/wavefront.h — the diagonal-wavefront schedule (drop-in for the
// reference's proj/include/pswa/wavefront.h:23-66; same declarations, with
// the missing <cstdint> include fixed). On the device the same rules are
// evaluated by index arithmetic inside the attention kernel
// (csrc/cuda/attention.cu) and by the per-step position tables the engine
// builds from positions_of_step().
#ifndef PSWA_WAVEFRONT_H_
#define PSWA_WAVEFRONT_H_

#include <cstdint>
#include <string>
#include <vector>

namespace pswa {

struct Pos {
  int y = 0;
  int x = 0;
  bool operator==(const Pos&) const = default;
};

// Anti-diagonal step: every s-th diagonal decodes together.
inline int step_of(Pos p, int s) { return (p.y + p.x) % s; }

enum class MaskKind {
  kSpatialSelf,     // key step <= query step
  kAccumulator,     // key step <  query step
  kTemporalCausal,  // key frame < query frame (frame index in .y)
  kChannelBlockLt,  // key group <= query group (group index in .y)
};

bool mask_allows(MaskKind kind, Pos query, Pos key, int s);

// Raster-ordered positions of step t: the canonical symbol order.
std::vector<Pos> positions_of_step(int h, int w, int s, int t);

// (N*d_g)^2 block-lower-triangular mask, row = output channel.
std::vector<uint8_t> channel_mask(int n_groups, int group_dim);

struct ScheduleReport {
  bool ok = true;
  int sequential_steps = 0;
  std::string first_violation;
  std::vector<std::string> lines;
};

ScheduleReport validate_schedule(int h, int w, int s, int wh, int ww, int n_groups);

}  // namespace pswa

#endif  // PSWA_WAVEFRONT_H_
