// pipetune time base — drop-in for proj/include/pipetune/time.hpp:12-22.
//
// All schedule arithmetic (simulator, cost model, tuner) runs on signed 64-bit
// ticks so that timelines and tuning decisions are bit-reproducible.  Abstract
// scenario "units" map to 1e9 ticks; on the GPU executor one tick is one
// nanosecond of measured device time.
#pragma once

#include <cmath>
#include <cstdint>

namespace pipetune {

using Tick = std::int64_t;

inline constexpr Tick kTicksPerUnit = 1'000'000'000;

// Round-half-away-from-zero conversion (std::llround), as the reference does.
inline Tick to_ticks(double units) { return static_cast<Tick>(std::llround(units * 1e9)); }

inline double to_units(Tick ticks) { return static_cast<double>(ticks) / 1e9; }

}  // namespace pipetune
