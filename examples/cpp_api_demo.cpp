// C++ callers of the drop-in API (include/pipetune/*.hpp + libptk.so): the reference planner calls
// (proj/include/pipetune/plan.hpp:32-49) plus the spec-module extensions — simulate a kFkB plan over
// a preempted link, rank uniform and mixed-k candidates, and build a SimResult from "measured"
// records.  Built and run by tests/test_cpp_api.py:
//   g++ -std=c++20 -Iinclude examples/cpp_api_demo.cpp -Lpaper_2303_01675_b200 -lptk -o demo
#include <cstdio>
#include <memory>

#include "pipetune/costmodel.hpp"
#include "pipetune/plan.hpp"
#include "pipetune/simulator.hpp"
#include "pipetune/tuner.hpp"

using namespace pipetune;

int main() {
    ModelSpec model;
    model.global_batch = 10;
    for (int s = 0; s < 4; ++s) {
        StageProfile p;
        p.stage_id = s;
        p.forward_per_sample = 1.0;
        p.backward_per_sample = 2.0;
        p.output_bytes_per_sample_fwd = p.output_bytes_per_sample_bwd = 15;
        model.stages.push_back(p);
    }
    PlanConfig cfg = PlanConfig::make(1, 1, model.global_batch);  // (k, b, global batch): M = 10
    auto graph = std::make_shared<const TaskGraph>(build_task_graph(model, cfg));
    const SchedulePlan plan = plan_kfkb(graph, 4);
    std::printf("stage 0: %s\n", sequence_string(plan, 0).c_str());

    LinkTraces traces(static_cast<size_t>(link_count(4)));
    for (size_t l = 0; l < traces.size(); ++l) {
        traces[l].link = static_cast<LinkId>(l);
        traces[l].base_bandwidth = 10.0;
        traces[l].segments.push_back({0.0, 20.0, 0.5});  // preempted to 50 % for 20 units
    }
    const SimResult r = simulate(plan, model, traces);
    std::printf("length %lld ticks, stage-0 bubble %.4f\n", static_cast<long long>(r.pipeline_length),
                bubble_report(r)[0]);

    // rank uniform k and a remainder-first mixed-k plan over constant profiles
    CandidateSet set;
    for (int k : {1, 2, 4}) set.entries.push_back({PlanConfig{k, 1, 10}, {}});
    const ComputeProfile comp = ComputeProfile::from_model(model, {1});
    ProfileStore store(8);
    for (int l = 0; l < link_count(4); ++l)
        for (int i = 0; i < 3; ++i) store.record_sample({l, 15, 0, to_ticks(1.5)});
    const TuningDecision d =
        tuning_round_plans(set, {GroupCandidate{1, {2, 4, 4}}}, model, comp, store, PlanConfig{4, 1, 10}, {}, 0.02, 0);
    std::printf("chosen k=%d groups=%zu switched=%d\n", d.chosen.k, d.chosen_groups.size(), d.switched ? 1 : 0);

    // a "measured" timeline (here: the simulator's own) through result_from_records
    std::vector<HwCompute> hc;
    std::vector<HwTransfer> hx;
    for (const TimelineEntry& e : r.timeline) {
        if (e.stream == Stream::Compute) hc.push_back({e.device, e.node, e.start, e.end});
        if (e.stream == Stream::Send) {
            const TaskNode& n = plan.graph->node(e.node);
            hx.push_back({n.link, n.micro_batch, e.start, e.end});
        }
    }
    const SimResult hw = result_from_records(plan, hc, hx, 0);
    std::printf("records reproduce: %d\n", hw.per_device_bubble == r.per_device_bubble ? 1 : 0);
    return 0;
}
