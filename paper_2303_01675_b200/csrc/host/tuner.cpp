// Ada-Grouper tuner.
#include "pipetune/tuner.hpp"

#include <algorithm>
#include <set>

#include "pipetune/errors.hpp"

namespace pipetune {

void TuningPolicy::validate() const {
    if (!(interval > 0)) throw ConfigError("TuningPolicy: interval must be positive");
    if (hysteresis < 0) throw ConfigError("TuningPolicy: hysteresis must be >= 0");
    if (profile_repeats < 1) throw ConfigError("TuningPolicy: profile_repeats must be >= 1");
    if (window_size < 1) throw ConfigError("TuningPolicy: window_size must be >= 1");
    if (switch_overhead < 0) throw ConfigError("TuningPolicy: switch_overhead must be >= 0");
    if (k_max < 1) throw ConfigError("TuningPolicy: k_max must be >= 1");
}

double AdaptiveResult::throughput() const {
    if (iterations.empty()) return 0.0;
    double samples = 0.0;
    for (const IterationRecord& it : iterations)
        samples += static_cast<double>(it.config.micro_batch_size) * it.config.micro_batch_count;
    const Tick span = iterations.back().end - iterations.front().start;
    return span > 0 ? samples / to_units(span) : 0.0;
}

std::vector<std::pair<LinkId, Bytes>> candidate_buckets(const CandidateSet& candidates, const ModelSpec& model) {
    std::set<std::pair<LinkId, Bytes>> all;
    for (const CandidateEntry& e : candidates.entries)
        for (const auto& bk : plan_buckets(plan_for(model, e.config))) all.insert(bk);
    return {all.begin(), all.end()};
}

TuningDecision tuning_round_plans(const CandidateSet& candidates, const std::vector<GroupCandidate>& mixed,
                                  const ModelSpec& model, const ComputeProfile& compute, const ProfileStore& comm,
                                  const PlanConfig& current, const std::vector<int>& current_groups, double hysteresis,
                                  Tick round_time) {
    TuningDecision d;
    d.round_time = round_time;
    d.estimates = rank_plans(candidates, mixed, model, compute, comm);
    if (d.estimates.empty()) throw InfeasibleModel("tuning_round: empty candidate set");
    const PlanEstimate& best = d.estimates.front();
    if (current.k == 0) {  // initial selection: nothing to switch away from
        d.chosen = best.config;
        d.chosen_groups = best.groups;
        d.switched = false;
        return d;
    }
    auto cur = std::find_if(d.estimates.begin(), d.estimates.end(), [&](const PlanEstimate& e) {
        return e.config == current && e.groups == current_groups;
    });
    if (cur == d.estimates.end()) throw UnknownCandidate("tuning_round: current plan is not a candidate");
    const bool better = static_cast<double>(best.estimated_length) <
                        static_cast<double>(cur->estimated_length) * (1.0 - hysteresis);
    d.switched = better && !(best.config == current && best.groups == current_groups);
    d.chosen = d.switched ? best.config : current;
    d.chosen_groups = d.switched ? best.groups : current_groups;
    return d;
}

TuningDecision tuning_round(const CandidateSet& candidates, const ModelSpec& model, const ComputeProfile& compute,
                            const ProfileStore& comm, const PlanConfig& current, double hysteresis, Tick round_time) {
    return tuning_round_plans(candidates, {}, model, compute, comm, current, {}, hysteresis, round_time);
}

Tick switch_plan(const CandidateSet& candidates, const PlanConfig& current, const PlanConfig& next,
                 const TuningPolicy& policy) {
    const bool known = std::any_of(candidates.entries.begin(), candidates.entries.end(),
                                   [&](const CandidateEntry& e) { return e.config == next; });
    if (!known) throw UnknownCandidate("switch_plan: target config is not in the candidate set");
    return next == current ? 0 : to_ticks(policy.switch_overhead);
}

AdaptiveResult run_adaptive(const ModelSpec& model, const ClusterSpec& cluster, const LinkTraces& traces,
                            const TuningPolicy& policy, double horizon) {
    policy.validate();
    const CandidateSet cands = enumerate_candidates(model, cluster, policy.k_max);
    std::vector<int> bs;
    for (const CandidateEntry& e : cands.entries) bs.push_back(e.config.micro_batch_size);
    // compute profiles: measured once at startup, never refreshed
    const ComputeProfile compute = ComputeProfile::from_model(model, bs);
    const auto buckets = candidate_buckets(cands, model);
    ProfileStore store(policy.window_size);
    const Tick end = to_ticks(horizon);
    const Tick interval = to_ticks(policy.interval);

    AdaptiveResult out;
    Tick clock = 0;
    // round 0: initial selection
    {
        const Tick t0 = clock;
        clock = profile_buckets(buckets, traces, clock, policy.profile_repeats, store);
        out.log.rounds.push_back(tuning_round(cands, model, compute, store, PlanConfig{0, 0, 0}, policy.hysteresis, t0));
    }
    PlanConfig current = out.log.rounds.back().chosen;
    while (clock < end) {
        const Tick round_start = clock;
        const SchedulePlan plan = plan_for(model, current);
        do {
            const SimResult r = simulate(plan, model, traces, clock);
            IterationRecord it;
            it.start = clock;
            it.end = clock + r.pipeline_length;
            it.config = current;
            it.throughput = static_cast<double>(model.global_batch) / to_units(r.pipeline_length);
            out.iterations.push_back(it);
            clock = it.end;
        } while (clock - round_start < interval && clock < end);
        if (clock >= end) break;
        const Tick t = clock;
        clock = profile_buckets(buckets, traces, clock, policy.profile_repeats, store);
        TuningDecision d = tuning_round(cands, model, compute, store, current, policy.hysteresis, t);
        clock += switch_plan(cands, current, d.chosen, policy);
        current = d.chosen;
        out.log.rounds.push_back(std::move(d));
    }
    return out;
}

}  // namespace pipetune
