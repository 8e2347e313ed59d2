// validate_schedule over injectable predicates (pswa/wavefront.h), so tests
// can feed a deliberately broken mask or channel mask and see it reported.
#pragma once
#include <cstdint>
#include <functional>
#include <vector>

#include "pswa/wavefront.h"

namespace pswa::detail {

using MaskFn = std::function<bool(MaskKind, Pos, Pos, int)>;
using ChannelMaskFn = std::function<std::vector<uint8_t>(int, int)>;

ScheduleReport validate_schedule_with(int h, int w, int s, int wh, int ww, int n_groups,
                                      const MaskFn& allows, const ChannelMaskFn& cmask);

}  // namespace pswa::detail
