// pipetune network module (spec-only in the reference: SPEC.md:261-325).
//
// Piecewise-constant link availability traces, the latency + integrated
// bandwidth transfer model, and the moving-average communication profiler.
// On the B200 executor the same ProfileStore receives GPU-measured samples
// (int64 ns) and LinkTrace drives the preemption emulator.
#pragma once

#include <deque>
#include <map>
#include <utility>
#include <vector>

#include "pipetune/plan.hpp"

namespace pipetune {

struct TraceSegment {
    double start = 0.0;         // time units
    double end = 0.0;           // time units, exclusive
    double availability = 1.0;  // (0, 1]
};

struct LinkTrace {
    LinkId link = 0;
    double base_bandwidth = 1.0;                // bytes per time unit at availability 1
    double latency = 0.0;                       // time units per message
    std::vector<TraceSegment> segments;         // sorted, non-overlapping; gaps mean 1.0
    std::map<Bytes, double> utilization_curve;  // exact payload -> efficiency in (0,1]; default 1.0

    void validate() const;  // ConfigError on bad segments / fractions
    double availability_at(Tick t) const;
    double efficiency(Bytes bytes) const;
};

using LinkTraces = std::vector<LinkTrace>;  // indexed by LinkId

// latency + time to deliver `bytes` at base*availability(t)*efficiency(bytes),
// integrating from `start`.  Deterministic in ticks.
Tick transfer_duration(const LinkTrace& trace, Bytes bytes, Tick start);

struct CommSample {
    LinkId link = 0;
    Bytes bytes = 0;
    Tick start = 0;
    Tick measured_duration = 0;
};

// Per (link, exact payload) ring of the last `window_size` samples.
class ProfileStore {
  public:
    explicit ProfileStore(int window_size = 8);

    void record_sample(const CommSample& sample);
    // Round-half-up integer mean of the retained window; NoProfileData if empty.
    Tick estimate(LinkId link, Bytes bytes) const;
    bool has(LinkId link, Bytes bytes) const;
    int window_size() const { return window_; }
    const std::deque<Tick>& samples(LinkId link, Bytes bytes) const;

  private:
    int window_;
    std::map<std::pair<LinkId, Bytes>, std::deque<Tick>> buckets_;
};

// (link, payload) buckets a plan's Send nodes use, ascending.
std::vector<std::pair<LinkId, Bytes>> plan_buckets(const SchedulePlan& plan);

// Suspended-pipeline profiling: for each bucket in ascending (link, bytes)
// order, `repeats` back-to-back measurements starting at `clock`; returns the
// clock after profiling (profiling time is charged).
Tick profile_buckets(const std::vector<std::pair<LinkId, Bytes>>& buckets, const LinkTraces& traces, Tick clock,
                     int repeats, ProfileStore& store);
Tick profile_links(const SchedulePlan& plan, const ModelSpec& model, const LinkTraces& traces, Tick clock, int repeats,
                   ProfileStore& store);

}  // namespace pipetune
