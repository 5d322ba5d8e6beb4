// Cost model: the simulator over constant profiled durations.
#include "pipetune/costmodel.hpp"

#include <algorithm>

#include "pipetune/errors.hpp"

namespace pipetune {

void ComputeProfile::set(int stage, int batch, Direction dir, Tick duration) {
    d_[{stage, batch, static_cast<int>(dir)}] = duration;
}

bool ComputeProfile::has(int stage, int batch, Direction dir) const {
    return d_.count({stage, batch, static_cast<int>(dir)}) != 0;
}

Tick ComputeProfile::get(int stage, int batch, Direction dir) const {
    auto it = d_.find({stage, batch, static_cast<int>(dir)});
    if (it == d_.end())
        throw NoProfileData("ComputeProfile: no profile for stage " + std::to_string(stage) + ", b=" +
                            std::to_string(batch) + (dir == Direction::Forward ? ", forward" : ", backward"));
    return it->second;
}

ComputeProfile ComputeProfile::from_model(const ModelSpec& model, const std::vector<int>& batches) {
    ComputeProfile p;
    for (int s = 0; s < model.stage_count(); ++s)
        for (int b : batches)
            for (Direction dir : {Direction::Forward, Direction::Backward})
                p.set(s, b, dir, compute_duration_ticks(model.stages[static_cast<size_t>(s)], b, dir));
    return p;
}

SchedulePlan plan_for(const ModelSpec& model, const PlanConfig& config) {
    PlanConfig g = config;
    g.k = 1;
    return plan_kfkb(std::make_shared<const TaskGraph>(build_task_graph(model, g)), config.k);
}

PlanEstimate estimate_length(const SchedulePlan& plan, const ModelSpec& model, const ComputeProfile& compute,
                             const ProfileStore& comm) {
    std::string digest;
    const int b = plan.config.micro_batch_size;
    // resolve every input up front so a missing bucket fails before simulating
    for (int s = 0; s < plan.device_count(); ++s)
        digest += "c" + std::to_string(s) + ":" + std::to_string(compute.get(s, b, Direction::Forward)) + "/" +
                  std::to_string(compute.get(s, b, Direction::Backward)) + ";";
    for (const auto& [link, bytes] : plan_buckets(plan))
        digest += "l" + std::to_string(link) + "@" + std::to_string(bytes) + ":" +
                  std::to_string(comm.estimate(link, bytes)) + ";";
    auto comp = [&compute](int s, int bb, Direction dir) { return compute.get(s, bb, dir); };
    auto xfer = [&comm](LinkId l, Bytes bytes, Tick) { return comm.estimate(l, bytes); };
    const SimResult r = simulate_with(plan, model, comp, xfer, 0);
    return {plan.config, r.pipeline_length, digest};
}

std::vector<PlanEstimate> rank_plans(const CandidateSet& candidates, const std::vector<GroupCandidate>& mixed,
                                     const ModelSpec& model, const ComputeProfile& compute, const ProfileStore& comm) {
    std::vector<PlanEstimate> out;
    out.reserve(candidates.entries.size() + mixed.size());
    for (const CandidateEntry& e : candidates.entries)
        out.push_back(estimate_length(plan_for(model, e.config), model, compute, comm));
    for (const GroupCandidate& g : mixed) {
        if (g.micro_batch_size < 1 || model.global_batch % g.micro_batch_size)
            throw ConfigError("rank_plans: group candidate b must divide the global batch");
        PlanConfig cfg{1, g.micro_batch_size, model.global_batch / g.micro_batch_size};
        auto graph = std::make_shared<const TaskGraph>(build_task_graph(model, cfg));
        std::vector<MicroBatchGroup> groups;
        int first = 0, kmax = 0;
        for (int n : g.groups) {
            if (n < 1) throw ConfigError("rank_plans: group sizes must be >= 1");
            groups.push_back({first, first + n - 1});
            first += n;
            kmax = std::max(kmax, n);
        }
        PlanEstimate e = estimate_length(plan_groups(graph, kmax, groups), model, compute, comm);
        e.config = PlanConfig{kmax, g.micro_batch_size, cfg.micro_batch_count};
        e.groups = g.groups;
        out.push_back(std::move(e));
    }
    std::stable_sort(out.begin(), out.end(), [](const PlanEstimate& a, const PlanEstimate& b) {
        if (a.estimated_length != b.estimated_length) return a.estimated_length < b.estimated_length;
        if (a.config.k != b.config.k) return a.config.k < b.config.k;
        if (a.config.micro_batch_size != b.config.micro_batch_size)
            return a.config.micro_batch_size > b.config.micro_batch_size;
        return a.groups < b.groups;  // uniform (empty) first
    });
    return out;
}

std::vector<PlanEstimate> rank_candidates(const CandidateSet& candidates, const ModelSpec& model,
                                          const ComputeProfile& compute, const ProfileStore& comm) {
    return rank_plans(candidates, {}, model, compute, comm);
}

}  // namespace pipetune
