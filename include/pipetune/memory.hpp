// pipetune memory module (spec-only in the reference: SPEC.md:203-259).
//
// Activation liveness per device from plan order alone (no timing), and the
// (k, b) candidate frontier under the per-device memory limit.
#pragma once

#include <functional>
#include <vector>

#include "pipetune/plan.hpp"

namespace pipetune {

struct PeakMemoryReport {
    std::vector<Bytes> per_device_peak;
    int limiting_device = 0;  // first device attaining the maximum
};

// F allocates activation_bytes_per_sample*b, the matching B releases it,
// weight_bytes stays resident.
PeakMemoryReport peak_memory(const SchedulePlan& plan, const ModelSpec& model);

struct CandidateEntry {
    PlanConfig config;
    PeakMemoryReport memory;
};

// At most one entry per k, ascending k; each with the largest feasible b.
struct CandidateSet {
    std::vector<CandidateEntry> entries;
};

// For k = 1..k_max scan divisors of global_batch in descending order and keep
// the first b with k <= M and every device's peak <= device_memory_limit
// (SPEC.md:227-231).  InfeasibleModel when no entry exists.
CandidateSet enumerate_candidates(const ModelSpec& model, const ClusterSpec& cluster, int k_max);

// Same frontier search over an injected feasibility predicate (the spec's
// synthetic-peak example).
CandidateSet enumerate_candidates_with(int global_batch, int k_max, const std::function<bool(int k, int b)>& feasible);

// Appendix-C default: min(M at the smallest b (= global_batch), cap).
int default_k_max(const ModelSpec& model, int cap = 6);

}  // namespace pipetune
