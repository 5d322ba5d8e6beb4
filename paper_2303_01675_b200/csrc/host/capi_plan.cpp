// C-ABI over the planner (include/ptk.h ptk_plan_*), for FFI callers and for
// the parity tests that diff this implementation against the compiled
// reference planner (oracle/ref_dump.cpp emits the same JSON layout).
#include <cstring>
#include <memory>
#include <string>

#include "../../../include/ptk.h"
#include "../runtime/errors.h"
#include "json_out.h"
#include "pipetune/errors.hpp"
#include "pipetune/plan.hpp"
#include "plan_io.h"

namespace pipetune {

ModelSpec model_from_c(const ptk_model* m) {
    ModelSpec spec;
    spec.global_batch = m->global_batch;
    for (int s = 0; s < m->stage_count; ++s) {
        const ptk_stage_profile& p = m->stages[s];
        StageProfile st;
        st.stage_id = p.stage_id;
        st.forward_fixed = p.forward_fixed;
        st.forward_per_sample = p.forward_per_sample;
        st.backward_fixed = p.backward_fixed;
        st.backward_per_sample = p.backward_per_sample;
        st.weight_bytes = p.weight_bytes;
        st.activation_bytes_per_sample = p.activation_bytes_per_sample;
        st.output_bytes_per_sample_fwd = p.output_bytes_per_sample_fwd;
        st.output_bytes_per_sample_bwd = p.output_bytes_per_sample_bwd;
        spec.stages.push_back(st);
    }
    return spec;
}

const char* error_name(const std::exception& e) {
    if (dynamic_cast<const ConfigError*>(&e)) return "ConfigError";
    if (dynamic_cast<const PlanError*>(&e)) return "PlanError";
    if (dynamic_cast<const InfeasibleModel*>(&e)) return "InfeasibleModel";
    if (dynamic_cast<const NoProfileData*>(&e)) return "NoProfileData";
    if (dynamic_cast<const DeadlockDetected*>(&e)) return "DeadlockDetected";
    if (dynamic_cast<const UnknownCandidate*>(&e)) return "UnknownCandidate";
    if (dynamic_cast<const CudaError*>(&e)) return "CudaError";
    if (dynamic_cast<const Error*>(&e)) return "Error";
    return "std::exception";
}

int error_status(const std::exception& e) {
    if (dynamic_cast<const ConfigError*>(&e)) return PTK_ERR_ARG;
    if (dynamic_cast<const PlanError*>(&e)) return PTK_ERR_PLAN;
    if (dynamic_cast<const InfeasibleModel*>(&e)) return PTK_ERR_INFEASIBLE;
    if (dynamic_cast<const NoProfileData*>(&e)) return PTK_ERR_NOPROFILE;
    if (dynamic_cast<const DeadlockDetected*>(&e)) return PTK_ERR_DEADLOCK;
    if (dynamic_cast<const UnknownCandidate*>(&e)) return PTK_ERR_UNKNOWN_CANDIDATE;
    if (dynamic_cast<const CudaError*>(&e)) return PTK_ERR_CUDA;
    return PTK_ERR_INTERNAL;
}

std::string plan_to_json(const SchedulePlan& plan) {
    const TaskGraph& g = *plan.graph;
    json::Writer w;
    w.begin_obj();
    w.key("config").begin_arr().v(plan.config.k).v(plan.config.micro_batch_size).v(plan.config.micro_batch_count).end_arr();
    w.key("stage_count").num(g.stage_count);
    w.key("nodes").begin_arr();
    for (const TaskNode& t : g.nodes) {
        w.begin_arr().v(static_cast<int>(t.kind)).v(t.stage_id).v(t.micro_batch).v(t.device).v(t.link).v(t.payload_bytes);
        w.end_arr();
    }
    w.end_arr();
    w.key("edges").begin_arr();
    for (const auto& e : g.edges) w.begin_arr().v(e.first).v(e.second).end_arr();
    w.end_arr();
    w.key("lookup").begin_arr().ints(g.send_of_compute).ints(g.recv_of_compute).ints(g.pair_of).end_arr();
    w.key("per_device").begin_arr();
    for (const auto& d : plan.per_device) w.ints(d);
    w.end_arr();
    w.key("units").begin_arr();
    for (const auto& d : plan.units) {
        w.begin_arr();
        for (const ScheduleUnit& u : d) w.begin_arr().v(u.begin).v(u.end).end_arr();
        w.end_arr();
    }
    w.end_arr();
    w.key("sequences").begin_arr();
    for (int d = 0; d < plan.device_count(); ++d) w.vs(sequence_string(plan, d, true));
    w.end_arr();
    w.key("violations").begin_arr();
    for (const Violation& v : validate(g)) w.begin_arr().vs(violation_kind_name(v.kind)).v(v.node_id).end_arr();
    w.end_arr();
    w.key("check").num(static_cast<long long>(check_plan(plan).size()));
    w.key("topo").ints(topological_order(g));
    w.end_obj();
    return w.out;
}

}  // namespace pipetune

namespace {

int emit(const std::string& s, char* buf, size_t cap, size_t* written) {
    if (written) *written = s.size() + 1;
    if (buf == nullptr || cap < s.size() + 1) return PTK_ERR_NOMEM;
    std::memcpy(buf, s.data(), s.size());
    buf[s.size()] = '\0';
    return PTK_OK;
}

}  // namespace

extern "C" int ptk_plan_json(const ptk_model* model, int micro_batch_size, int plan_kind, int k, char* buf,
                             size_t cap, size_t* written) {
    using namespace pipetune;
    try {
        if (model == nullptr || model->stage_count < 0 || (model->stage_count > 0 && model->stages == nullptr))
            throw ConfigError("ptk_plan_json: bad model");
        const ModelSpec spec = model_from_c(model);
        PlanConfig cfg;
        cfg.micro_batch_size = micro_batch_size;
        cfg.micro_batch_count = micro_batch_size > 0 ? spec.global_batch / micro_batch_size : 0;
        cfg.k = 1;
        auto graph = std::make_shared<const TaskGraph>(build_task_graph(spec, cfg));
        SchedulePlan plan;
        if (plan_kind == PTK_PLAN_1F1B)
            plan = plan_1f1b(graph);
        else if (plan_kind == PTK_PLAN_GPIPE)
            plan = plan_gpipe(graph);
        else
            plan = plan_kfkb(graph, k);
        return emit(plan_to_json(plan), buf, cap, written);
    } catch (const std::exception& e) {
        std::string s = std::string("{\"error\":\"") + error_name(e) + "\"}";
        emit(s, buf, cap, written);
        return ptk::set_error(error_status(e), e.what());
    }
}
