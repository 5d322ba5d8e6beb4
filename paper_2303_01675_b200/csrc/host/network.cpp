// Network module.
#include "pipetune/network.hpp"

#include <algorithm>
#include <limits>
#include <set>

#include "pipetune/errors.hpp"

namespace pipetune {

void LinkTrace::validate() const {
    if (!(base_bandwidth > 0)) throw ConfigError("LinkTrace: base_bandwidth must be positive");
    if (latency < 0) throw ConfigError("LinkTrace: latency must be non-negative");
    double prev_end = -std::numeric_limits<double>::infinity();
    for (const TraceSegment& s : segments) {
        if (!(s.end > s.start)) throw ConfigError("LinkTrace: empty or reversed segment");
        if (s.start < prev_end) throw ConfigError("LinkTrace: segments overlap or are unsorted");
        if (!(s.availability > 0 && s.availability <= 1)) throw ConfigError("LinkTrace: availability outside (0,1]");
        prev_end = s.end;
    }
    for (const auto& [bytes, eff] : utilization_curve)
        if (!(eff > 0 && eff <= 1)) throw ConfigError("LinkTrace: efficiency outside (0,1]");
}

double LinkTrace::availability_at(Tick t) const {
    for (const TraceSegment& s : segments) {
        if (t < to_ticks(s.start)) break;
        if (t < to_ticks(s.end)) return s.availability;
    }
    return 1.0;
}

double LinkTrace::efficiency(Bytes bytes) const {
    auto it = utilization_curve.find(bytes);
    return it == utilization_curve.end() ? 1.0 : it->second;
}

namespace {

constexpr Tick kNever = std::numeric_limits<Tick>::max();

// Availability in force at t and the tick where it next changes.
std::pair<double, Tick> piece_at(const LinkTrace& tr, Tick t) {
    for (const TraceSegment& s : tr.segments) {
        const Tick a = to_ticks(s.start), b = to_ticks(s.end);
        if (t < a) return {1.0, a};
        if (t < b) return {s.availability, b};
    }
    return {1.0, kNever};
}

}  // namespace

Tick transfer_duration(const LinkTrace& trace, Bytes bytes, Tick start) {
    if (bytes < 0) throw ConfigError("transfer_duration: negative payload");
    const Tick lat = to_ticks(trace.latency);
    if (bytes == 0) return lat;
    const double eff = trace.efficiency(bytes);
    double left = static_cast<double>(bytes);
    Tick t = start;
    for (;;) {
        const auto [avail, next] = piece_at(trace, t);
        const double rate = trace.base_bandwidth * avail * eff;  // bytes per unit
        if (next == kNever) {
            t += to_ticks(left / rate);
            break;
        }
        const double can = rate * to_units(next - t);
        if (can >= left) {
            t += to_ticks(left / rate);
            break;
        }
        left -= can;
        t = next;
    }
    return (t - start) + lat;
}

ProfileStore::ProfileStore(int window_size) : window_(window_size) {
    if (window_size < 1) throw ConfigError("ProfileStore: window_size must be >= 1");
}

void ProfileStore::record_sample(const CommSample& s) {
    auto& q = buckets_[{s.link, s.bytes}];
    q.push_back(s.measured_duration);
    while (static_cast<int>(q.size()) > window_) q.pop_front();
}

bool ProfileStore::has(LinkId link, Bytes bytes) const {
    auto it = buckets_.find({link, bytes});
    return it != buckets_.end() && !it->second.empty();
}

const std::deque<Tick>& ProfileStore::samples(LinkId link, Bytes bytes) const {
    auto it = buckets_.find({link, bytes});
    if (it == buckets_.end() || it->second.empty())
        throw NoProfileData("ProfileStore: no samples for link " + std::to_string(link) + ", " + std::to_string(bytes) +
                            " bytes");
    return it->second;
}

Tick ProfileStore::estimate(LinkId link, Bytes bytes) const {
    const std::deque<Tick>& q = samples(link, bytes);
    Tick sum = 0;
    for (Tick v : q) sum += v;
    const Tick n = static_cast<Tick>(q.size());
    // round half up (samples are non-negative durations)
    return (2 * sum + n) / (2 * n);
}

std::vector<std::pair<LinkId, Bytes>> plan_buckets(const SchedulePlan& plan) {
    std::set<std::pair<LinkId, Bytes>> s;
    for (const TaskNode& t : plan.graph->nodes)
        if (t.kind == TaskKind::Send) s.insert({t.link, t.payload_bytes});
    return {s.begin(), s.end()};
}

Tick profile_buckets(const std::vector<std::pair<LinkId, Bytes>>& buckets, const LinkTraces& traces, Tick clock,
                     int repeats, ProfileStore& store) {
    if (repeats < 1) throw ConfigError("profile_links: repeats must be >= 1");
    for (const auto& [link, bytes] : buckets) {
        if (link < 0 || static_cast<size_t>(link) >= traces.size())
            throw ConfigError("profile_links: no trace for link " + std::to_string(link));
        for (int r = 0; r < repeats; ++r) {
            const Tick d = transfer_duration(traces[static_cast<size_t>(link)], bytes, clock);
            store.record_sample({link, bytes, clock, d});
            clock += d;
        }
    }
    return clock;
}

Tick profile_links(const SchedulePlan& plan, const ModelSpec& model, const LinkTraces& traces, Tick clock, int repeats,
                   ProfileStore& store) {
    (void)model;
    return profile_buckets(plan_buckets(plan), traces, clock, repeats, store);
}

}  // namespace pipetune
