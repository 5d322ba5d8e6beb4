// pipetune tuner — the Ada-Grouper k-tuner interface (spec-only in the
// reference: SPEC.md:438-491).
//
// run_adaptive is the simulated loop; tuning_round is the pure decision
// function shared with the B200 executor, which feeds it GPU-measured
// samples (int64 ns) so the CPU oracle can replay and reproduce every choice.
#pragma once

#include <vector>

#include "pipetune/costmodel.hpp"

namespace pipetune {

struct TuningPolicy {
    double interval = 1.0;         // time units between tuning rounds (rounded up to whole iterations)
    int profile_repeats = 3;
    int window_size = 8;
    double switch_overhead = 0.0;  // time units charged on a switch
    double hysteresis = 0.02;      // switch iff est_new < est_cur * (1 - hysteresis)
    int k_max = 6;

    void validate() const;
};

struct TuningDecision {
    Tick round_time = 0;
    std::vector<PlanEstimate> estimates;  // ranked
    PlanConfig chosen;
    std::vector<int> chosen_groups;  // non-empty when a mixed-k plan (GroupCandidate) is chosen
    bool switched = false;
};

struct TuningLog {
    std::vector<TuningDecision> rounds;
};

struct IterationRecord {
    Tick start = 0;
    Tick end = 0;
    PlanConfig config;
    double throughput = 0.0;  // samples per time unit
};

struct AdaptiveResult {
    TuningLog log;
    std::vector<IterationRecord> iterations;
    double throughput() const;  // total samples / total time
};

// Pure decision: rank the candidates on the current profiles and apply the
// hysteresis rule against `current` (pass current.k = 0 for the initial pick).
TuningDecision tuning_round(const CandidateSet& candidates, const ModelSpec& model, const ComputeProfile& compute,
                            const ProfileStore& comm, const PlanConfig& current, double hysteresis, Tick round_time);

// UnknownCandidate unless `next` is in the set; returns the switch overhead to
// charge (0 for a no-op switch to the current config).
// tuning_round over uniform and mixed-k candidates; `current_groups` identifies a mixed incumbent.
TuningDecision tuning_round_plans(const CandidateSet& candidates, const std::vector<GroupCandidate>& mixed,
                                  const ModelSpec& model, const ComputeProfile& compute, const ProfileStore& comm,
                                  const PlanConfig& current, const std::vector<int>& current_groups, double hysteresis,
                                  Tick round_time);

Tick switch_plan(const CandidateSet& candidates, const PlanConfig& current, const PlanConfig& next,
                 const TuningPolicy& policy);

// Union of every candidate plan's (link, payload) buckets, ascending.
std::vector<std::pair<LinkId, Bytes>> candidate_buckets(const CandidateSet& candidates, const ModelSpec& model);

AdaptiveResult run_adaptive(const ModelSpec& model, const ClusterSpec& cluster, const LinkTraces& traces,
                            const TuningPolicy& policy, double horizon);

}  // namespace pipetune
