// ORACLE TEST INFRASTRUCTURE — not product code.
//
// Links the UNMODIFIED reference planner (compiled from
// /root/reference/proj/src/{model,taskgraph,plan}.cpp by oracle/Makefile,
// outputs only under oracle/_ref/) and prints, for each case read from stdin,
// the same JSON layout that libptk's ptk_plan_json() emits, so the two can be
// compared byte for byte (tests/test_planner_parity.py).
//
// stdin lines:  S M b kind k fwd_base bwd_base
//   stage s sends fwd_base*(s+1) bytes/sample forward and bwd_base*(s+1) backward.
//   kind: 0 = plan_1f1b, 1 = plan_kfkb(k), 2 = plan_gpipe     (reference plan.cpp:70-104)
// Modes:  ref_dump            -> JSON per case
//         ref_dump --time N   -> per case: mean microseconds of build_task_graph+plan over N reps
#include <chrono>
#include <cstdio>
#include <cstring>
#include <iostream>
#include <memory>
#include <sstream>
#include <string>

#include "pipetune/errors.hpp"
#include "pipetune/plan.hpp"

using namespace pipetune;

namespace {

std::string q(const std::string& s) { return "\"" + s + "\""; }

template <class V>
std::string ints(const V& v) {
    std::string o = "[";
    for (size_t i = 0; i < v.size(); ++i) {
        if (i) o += ",";
        o += std::to_string(v[i]);
    }
    return o + "]";
}

const char* err_name(const std::exception& e) {
    if (dynamic_cast<const ConfigError*>(&e)) return "ConfigError";
    if (dynamic_cast<const PlanError*>(&e)) return "PlanError";
    if (dynamic_cast<const Error*>(&e)) return "Error";
    return "std::exception";
}

std::string dump(const SchedulePlan& p) {
    const TaskGraph& g = *p.graph;
    std::ostringstream o;
    o << "{\"config\":[" << p.config.k << "," << p.config.micro_batch_size << "," << p.config.micro_batch_count << "]";
    o << ",\"stage_count\":" << g.stage_count << ",\"nodes\":[";
    for (size_t i = 0; i < g.nodes.size(); ++i) {
        const TaskNode& t = g.nodes[i];
        o << (i ? "," : "") << "[" << static_cast<int>(t.kind) << "," << t.stage_id << "," << t.micro_batch << ","
          << t.device << "," << t.link << "," << t.payload_bytes << "]";
    }
    o << "],\"edges\":[";
    for (size_t i = 0; i < g.edges.size(); ++i)
        o << (i ? "," : "") << "[" << g.edges[i].first << "," << g.edges[i].second << "]";
    o << "],\"lookup\":[" << ints(g.send_of_compute) << "," << ints(g.recv_of_compute) << "," << ints(g.pair_of) << "]";
    o << ",\"per_device\":[";
    for (size_t d = 0; d < p.per_device.size(); ++d) o << (d ? "," : "") << ints(p.per_device[d]);
    o << "],\"units\":[";
    for (size_t d = 0; d < p.units.size(); ++d) {
        o << (d ? "," : "") << "[";
        for (size_t i = 0; i < p.units[d].size(); ++i)
            o << (i ? "," : "") << "[" << p.units[d][i].begin << "," << p.units[d][i].end << "]";
        o << "]";
    }
    o << "],\"sequences\":[";
    for (int d = 0; d < p.device_count(); ++d) o << (d ? "," : "") << q(sequence_string(p, d, true));
    o << "],\"violations\":[";
    auto viol = validate(g);
    for (size_t i = 0; i < viol.size(); ++i)
        o << (i ? "," : "") << "[" << q(violation_kind_name(viol[i].kind)) << "," << viol[i].node_id << "]";
    o << "],\"check\":" << check_plan(p).size() << ",\"topo\":" << ints(topological_order(g)) << "}";
    return o.str();
}

SchedulePlan make(int S, int M, int b, int kind, int k, long fb, long bb) {
    ModelSpec spec;
    spec.global_batch = M * b;
    for (int s = 0; s < S; ++s) {
        StageProfile st;
        st.stage_id = s;
        st.forward_per_sample = 1.0;
        st.backward_per_sample = 2.0;
        st.output_bytes_per_sample_fwd = fb * (s + 1);
        st.output_bytes_per_sample_bwd = bb * (s + 1);
        spec.stages.push_back(st);
    }
    PlanConfig cfg{1, b, spec.global_batch / b};
    auto g = std::make_shared<const TaskGraph>(build_task_graph(spec, cfg));
    if (kind == 0) return plan_1f1b(g);
    if (kind == 2) return plan_gpipe(g);
    return plan_kfkb(g, k);
}

}  // namespace

int main(int argc, char** argv) {
    int reps = 0;
    if (argc == 3 && std::strcmp(argv[1], "--time") == 0) reps = std::atoi(argv[2]);
    int S, M, b, kind, k;
    long fb, bb;
    while (std::cin >> S >> M >> b >> kind >> k >> fb >> bb) {
        if (reps > 0) {
            auto t0 = std::chrono::steady_clock::now();
            size_t sink = 0;
            for (int r = 0; r < reps; ++r) sink += make(S, M, b, kind, k, fb, bb).per_device.size();
            auto t1 = std::chrono::steady_clock::now();
            std::printf("%.3f %zu\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / reps, sink);
            continue;
        }
        try {
            std::cout << dump(make(S, M, b, kind, k, fb, bb)) << "\n";
        } catch (const std::exception& e) {
            std::cout << "{\"error\":\"" << err_name(e) << "\"}\n";
        }
    }
    return 0;
}
