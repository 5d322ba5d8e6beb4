// Memory module.
#include "pipetune/memory.hpp"

#include <algorithm>
#include <map>

#include "pipetune/errors.hpp"

namespace pipetune {

PeakMemoryReport peak_memory(const SchedulePlan& plan, const ModelSpec& model) {
    const TaskGraph& g = *plan.graph;
    const int b = plan.config.micro_batch_size;
    PeakMemoryReport rep;
    rep.per_device_peak.assign(static_cast<size_t>(plan.device_count()), 0);
    for (int d = 0; d < plan.device_count(); ++d) {
        const StageProfile& st = model.stages[static_cast<size_t>(d)];
        const Bytes act = st.activation_bytes_per_sample * static_cast<Bytes>(b);
        Bytes live = st.weight_bytes, peak = live;
        for (int id : plan.per_device[static_cast<size_t>(d)]) {
            const TaskKind k = g.node(id).kind;
            if (k == TaskKind::ForwardCompute) {
                live += act;
                peak = std::max(peak, live);
            } else if (k == TaskKind::BackwardCompute) {
                live -= act;
            }
        }
        rep.per_device_peak[static_cast<size_t>(d)] = peak;
    }
    for (int d = 1; d < plan.device_count(); ++d)
        if (rep.per_device_peak[static_cast<size_t>(d)] > rep.per_device_peak[static_cast<size_t>(rep.limiting_device)])
            rep.limiting_device = d;
    return rep;
}

CandidateSet enumerate_candidates_with(int global_batch, int k_max, const std::function<bool(int, int)>& feasible) {
    if (k_max < 1) throw ConfigError("enumerate_candidates: k_max must be >= 1");
    CandidateSet set;
    const std::vector<int> bs = divisors_descending(global_batch);
    for (int k = 1; k <= k_max; ++k) {
        for (int b : bs) {
            const int M = global_batch / b;
            if (k > M) continue;
            if (!feasible(k, b)) continue;
            set.entries.push_back({PlanConfig{k, b, M}, {}});
            break;
        }
    }
    if (set.entries.empty()) throw InfeasibleModel("enumerate_candidates: no (k, b) fits the memory limit");
    return set;
}

CandidateSet enumerate_candidates(const ModelSpec& model, const ClusterSpec& cluster, int k_max) {
    model.validate();
    cluster.validate(model.stage_count());
    std::map<int, std::shared_ptr<const TaskGraph>> graphs;  // one graph per b serves every k
    std::map<std::pair<int, int>, PeakMemoryReport> reports;
    auto feasible = [&](int k, int b) {
        auto it = graphs.find(b);
        if (it == graphs.end()) {
            PlanConfig cfg{1, b, model.global_batch / b};
            it = graphs.emplace(b, std::make_shared<const TaskGraph>(build_task_graph(model, cfg))).first;
        }
        PeakMemoryReport rep = peak_memory(plan_kfkb(it->second, k), model);
        const bool ok = std::all_of(rep.per_device_peak.begin(), rep.per_device_peak.end(),
                                    [&](Bytes p) { return p <= cluster.device_memory_limit; });
        reports[{k, b}] = rep;
        return ok;
    };
    CandidateSet set = enumerate_candidates_with(model.global_batch, k_max, feasible);
    for (CandidateEntry& e : set.entries) e.memory = reports[{e.config.k, e.config.micro_batch_size}];
    return set;
}

int default_k_max(const ModelSpec& model, int cap) { return std::max(1, std::min(model.global_batch, cap)); }

}  // namespace pipetune
