// JSON scenario front door (SPEC.md cli module, ScenarioConfig :498-501):
// one request object in, one result object out, through the C ABI
// ptk_scenario_json().  Drives every spec-module operation so FFI callers and
// the oracle parity tests exercise the C++ implementations directly.
#include <algorithm>
#include <cstring>
#include <sstream>

#include "../../../include/ptk.h"
#include "../runtime/errors.h"
#include "json_in.h"
#include "json_out.h"
#include "pipetune/errors.hpp"
#include "pipetune/tuner.hpp"
#include "plan_io.h"
#include "scenario.h"

namespace pipetune {

using json::Value;

// Mandatory request fields: a missing key is a ConfigError (exit code 2 through
// the CLI), never a null dereference.
const Value& need(const Value& o, const char* k) {
    const Value* v = o.get(k);
    if (v == nullptr) throw ConfigError(std::string("missing required key \"") + k + "\"");
    return *v;
}

const Value& need_arr(const Value& o, const char* k) {
    const Value& v = need(o, k);
    if (v.kind != Value::Array) throw ConfigError(std::string("\"") + k + "\" must be an array");
    return v;
}

// Fixed-length array entries ([k, b, M], [link, bytes] ...).
const Value& entry(const Value& a, size_t i, const char* what) {
    if (a.kind != Value::Array || i >= a.arr.size()) throw ConfigError(std::string("malformed ") + what);
    return a.arr[i];
}

ModelSpec parse_model(const Value& v) {
    json::require_keys(v, "model", {"global_batch", "stages"});
    ModelSpec m;
    const Value* gb = v.get("global_batch");
    if (!gb) throw ConfigError("model: global_batch is required");
    m.global_batch = static_cast<int>(gb->as_int("model.global_batch"));
    const Value* st = v.get("stages");
    if (!st || st->kind != Value::Array) throw ConfigError("model: stages must be an array");
    int idx = 0;
    for (const Value& s : st->arr) {
        json::require_keys(s, "model.stages[]",
                           {"stage_id", "forward_fixed", "forward_per_sample", "backward_fixed", "backward_per_sample",
                            "weight_bytes", "activation_bytes_per_sample", "output_bytes_per_sample_fwd",
                            "output_bytes_per_sample_bwd"});
        StageProfile p;
        p.stage_id = idx;
        auto dbl = [&](const char* k, double& out) {
            if (const Value* x = s.get(k)) out = x->as_double(k);
        };
        auto i64 = [&](const char* k, Bytes& out) {
            if (const Value* x = s.get(k)) out = x->as_int(k);
        };
        if (const Value* x = s.get("stage_id")) p.stage_id = static_cast<int>(x->as_int("stage_id"));
        dbl("forward_fixed", p.forward_fixed);
        dbl("forward_per_sample", p.forward_per_sample);
        dbl("backward_fixed", p.backward_fixed);
        dbl("backward_per_sample", p.backward_per_sample);
        i64("weight_bytes", p.weight_bytes);
        i64("activation_bytes_per_sample", p.activation_bytes_per_sample);
        i64("output_bytes_per_sample_fwd", p.output_bytes_per_sample_fwd);
        i64("output_bytes_per_sample_bwd", p.output_bytes_per_sample_bwd);
        m.stages.push_back(p);
        ++idx;
    }
    m.validate();
    return m;
}

ClusterSpec parse_cluster(const Value& v) {
    json::require_keys(v, "cluster", {"device_memory_limit", "devices"});
    ClusterSpec c;
    if (const Value* x = v.get("device_memory_limit")) c.device_memory_limit = x->as_int("device_memory_limit");
    if (const Value* x = v.get("devices")) c.devices = static_cast<int>(x->as_int("devices"));
    return c;
}

LinkTrace parse_trace(const Value& v) {
    json::require_keys(v, "traces[]", {"link", "base_bandwidth", "latency", "segments", "utilization_curve"});
    LinkTrace t;
    if (const Value* x = v.get("link")) t.link = static_cast<int>(x->as_int("link"));
    if (const Value* x = v.get("base_bandwidth")) t.base_bandwidth = x->as_double("base_bandwidth");
    if (const Value* x = v.get("latency")) t.latency = x->as_double("latency");
    if (const Value* x = v.get("segments")) {
        for (const Value& s : x->arr) {
            if (s.kind != Value::Array || s.arr.size() != 3) throw ConfigError("segment must be [start, end, availability]");
            t.segments.push_back({s.arr[0].as_double("segment.start"), s.arr[1].as_double("segment.end"),
                                  s.arr[2].as_double("segment.availability")});
        }
    }
    if (const Value* x = v.get("utilization_curve")) {
        for (const Value& s : x->arr) {
            if (s.kind != Value::Array || s.arr.size() != 2) throw ConfigError("utilization entry must be [bytes, eff]");
            t.utilization_curve[s.arr[0].as_int("utilization.bytes")] = s.arr[1].as_double("utilization.eff");
        }
    }
    t.validate();
    return t;
}

LinkTraces parse_traces(const Value* v, int stage_count) {
    LinkTraces out(static_cast<size_t>(link_count(stage_count)));
    std::vector<bool> seen(out.size(), false);
    if (v) {
        for (const Value& t : v->arr) {
            LinkTrace lt = parse_trace(t);
            if (lt.link < 0 || static_cast<size_t>(lt.link) >= out.size())
                throw ConfigError("trace for link " + std::to_string(lt.link) + " outside the pipeline");
            out[static_cast<size_t>(lt.link)] = lt;
            seen[static_cast<size_t>(lt.link)] = true;
        }
    }
    for (size_t l = 0; l < out.size(); ++l)
        if (!seen[l]) throw ConfigError("no trace for link " + std::to_string(l));
    return out;
}

TuningPolicy parse_policy(const Value* v) {
    TuningPolicy p;
    if (!v) return p;
    json::require_keys(*v, "policy",
                       {"interval", "profile_repeats", "window_size", "switch_overhead", "hysteresis", "k_max"});
    if (const Value* x = v->get("interval")) p.interval = x->as_double("interval");
    if (const Value* x = v->get("profile_repeats")) p.profile_repeats = static_cast<int>(x->as_int("profile_repeats"));
    if (const Value* x = v->get("window_size")) p.window_size = static_cast<int>(x->as_int("window_size"));
    if (const Value* x = v->get("switch_overhead")) p.switch_overhead = x->as_double("switch_overhead");
    if (const Value* x = v->get("hysteresis")) p.hysteresis = x->as_double("hysteresis");
    if (const Value* x = v->get("k_max")) p.k_max = static_cast<int>(x->as_int("k_max"));
    p.validate();
    return p;
}

SchedulePlan parse_plan(const Value& v, const ModelSpec& model) {
    json::require_keys(v, "plan", {"kind", "k", "micro_batch_size", "groups"});
    const std::string kind = v.get("kind") ? v.get("kind")->as_str("plan.kind") : "kfkb";
    const int b = v.get("micro_batch_size") ? static_cast<int>(v.get("micro_batch_size")->as_int("b")) : 1;
    const int k = v.get("k") ? static_cast<int>(v.get("k")->as_int("k")) : 1;
    PlanConfig cfg{1, b, b > 0 ? model.global_batch / b : 0};
    auto g = std::make_shared<const TaskGraph>(build_task_graph(model, cfg));
    if (kind == "1f1b") return plan_1f1b(g);
    if (kind == "gpipe") return plan_gpipe(g);
    if (kind == "kfkb") return plan_kfkb(g, k);
    if (kind == "groups") {  // kFkB over an explicit list of group sizes
        const Value* gv = v.get("groups");
        if (!gv) throw ConfigError("plan.groups (list of group sizes) is required for kind \"groups\"");
        std::vector<MicroBatchGroup> groups;
        int first = 0, kmax = 0;
        for (const Value& x : gv->arr) {
            const int n = static_cast<int>(x.as_int("plan.groups[]"));
            if (n < 1) throw ConfigError("plan.groups: sizes must be >= 1");
            groups.push_back({first, first + n - 1});
            first += n;
            kmax = std::max(kmax, n);
        }
        return plan_groups(g, kmax, groups);
    }
    throw ConfigError("plan.kind must be 1f1b, kfkb, gpipe or groups");
}

void write_config(json::Writer& w, const PlanConfig& c) {
    w.begin_arr().v(c.k).v(c.micro_batch_size).v(c.micro_batch_count).end_arr();
}

void write_sim(json::Writer& w, const SimResult& r) {
    w.begin_obj();
    w.key("start").num(r.start);
    w.key("pipeline_length").num(r.pipeline_length);
    w.key("busy").ints(r.per_device_busy);
    w.key("bubble").ints(r.per_device_bubble);
    w.key("bubble_fraction").begin_arr();
    for (double f : bubble_report(r)) w.vd(f);
    w.end_arr();
    w.key("peak").ints(r.observed_peak_bytes);
    w.key("timeline").begin_arr();
    for (const TimelineEntry& e : r.timeline)
        w.begin_arr().v(e.node).v(e.device).v(static_cast<int>(e.stream)).v(e.start).v(e.end).end_arr();
    w.end_arr();
    w.key("queue_depth").begin_arr();
    for (const auto& d : r.queue_depth_trace) {
        w.begin_arr();
        for (const auto& [t, n] : d) w.begin_arr().v(t).v(n).end_arr();
        w.end_arr();
    }
    w.end_arr();
    w.key("launches").begin_arr();
    for (const auto& d : r.launches) {
        w.begin_arr();
        for (const QueueLaunch& q : d) w.begin_arr().v(q.node).v(q.queue_nonempty ? 1 : 0).end_arr();
        w.end_arr();
    }
    w.end_arr();
    w.end_obj();
}

void write_decision(json::Writer& w, const TuningDecision& d) {
    w.begin_obj();
    w.key("time").num(d.round_time);
    w.key("estimates").begin_arr();
    for (const PlanEstimate& e : d.estimates) {
        w.begin_arr().v(e.config.k).v(e.config.micro_batch_size).v(e.config.micro_batch_count).v(e.estimated_length);
        if (!e.groups.empty()) w.ints(e.groups);  // mixed-k candidates carry their group sizes
        w.end_arr();
    }
    w.end_arr();
    w.key("chosen");
    write_config(w, d.chosen);
    if (!d.chosen_groups.empty()) w.key("chosen_groups").ints(d.chosen_groups);
    w.key("switched").raw(d.switched ? "true" : "false");
    w.end_obj();
}

ComputeProfile parse_compute_profile(const Value& v) {
    // [[stage, b, dir(0 fwd / 1 bwd), ticks], ...]
    ComputeProfile p;
    for (const Value& e : v.arr) {
        if (e.kind != Value::Array || e.arr.size() != 4) throw ConfigError("compute profile entry must have 4 fields");
        p.set(static_cast<int>(e.arr[0].as_int("stage")), static_cast<int>(e.arr[1].as_int("b")),
              e.arr[2].as_int("dir") == 0 ? Direction::Forward : Direction::Backward, e.arr[3].as_int("ticks"));
    }
    return p;
}

void fill_store(const Value& v, ProfileStore& store) {
    // [[link, bytes, start, duration], ...] in recording order
    for (const Value& e : v.arr) {
        if (e.kind != Value::Array || e.arr.size() != 4) throw ConfigError("sample must be [link, bytes, start, dur]");
        store.record_sample({static_cast<int>(e.arr[0].as_int("link")), e.arr[1].as_int("bytes"),
                             e.arr[2].as_int("start"), e.arr[3].as_int("duration")});
    }
}

std::string run_scenario(const std::string& request) {
    const Value req = json::parse(request);
    json::require_keys(req, "scenario",
                       {"schema_version", "op", "model", "cluster", "traces", "plan", "policy", "horizon", "start",
                        "bytes", "trace", "buckets", "clock", "repeats", "window", "samples", "query", "k_max",
                        "compute_profile", "current", "hysteresis", "candidates", "records",
                        "group_candidates", "current_groups"});
    if (const Value* sv = req.get("schema_version"))
        if (sv->as_int("schema_version") != 1) throw ConfigError("unsupported schema_version");
    const Value* opv = req.get("op");
    if (!opv) throw ConfigError("scenario: op is required");
    const std::string op = opv->as_str("op");
    json::Writer w;
    w.begin_obj();

    if (op == "transfer") {
        const LinkTrace t = parse_trace(need(req, "trace"));
        const Tick start = req.get("start") ? req.get("start")->as_int("start") : 0;
        w.key("duration").num(transfer_duration(t, need(req, "bytes").as_int("bytes"), start));
    } else if (op == "estimate") {
        ProfileStore store(req.get("window") ? static_cast<int>(req.get("window")->as_int("window")) : 8);
        fill_store(need_arr(req, "samples"), store);
        const Value& q = need(req, "query");
        w.key("estimate").num(store.estimate(static_cast<int>(entry(q, 0, "query").as_int("link")), entry(q, 1, "query").as_int("bytes")));
    } else {
        const Value* mv = req.get("model");
        if (!mv) throw ConfigError("scenario: model is required for op " + op);
        const ModelSpec model = parse_model(*mv);
        if (op == "peak_memory" || op == "simulate") {
            const SchedulePlan plan = parse_plan(need(req, "plan"), model);
            if (op == "peak_memory") {
                const PeakMemoryReport r = peak_memory(plan, model);
                w.key("per_device_peak").ints(r.per_device_peak);
                w.key("limiting_device").num(r.limiting_device);
            } else {
                const LinkTraces traces = parse_traces(req.get("traces"), model.stage_count());
                const Tick start = req.get("start") ? req.get("start")->as_int("start") : 0;
                w.key("result");
                write_sim(w, simulate(plan, model, traces, start));
            }
        } else if (op == "hardware_report") {
            // SimResult of a measured GPU run (bubble_report / queue_analysis on hardware)
            const SchedulePlan plan = parse_plan(need(req, "plan"), model);
            const Value& rec = need(req, "records");
            std::vector<HwCompute> comp;
            std::vector<HwTransfer> xfer;
            for (const Value& e : need_arr(rec, "compute").arr)
                comp.push_back({static_cast<int>(entry(e, 0, "compute record").as_int("device")),
                                static_cast<int>(entry(e, 1, "compute record").as_int("node")),
                                entry(e, 2, "compute record").as_int("start"), entry(e, 3, "compute record").as_int("end")});
            for (const Value& e : need_arr(rec, "xfer").arr)
                xfer.push_back({static_cast<int>(entry(e, 0, "xfer record").as_int("link")),
                                static_cast<int>(entry(e, 1, "xfer record").as_int("mb")),
                                entry(e, 2, "xfer record").as_int("start"), entry(e, 3, "xfer record").as_int("end")});
            const Tick start = req.get("start") ? req.get("start")->as_int("start") : 0;
            w.key("result");
            write_sim(w, result_from_records(plan, comp, xfer, start));
        } else if (op == "estimate_sim") {
            // the cost model's full simulation of one plan over constant profiled durations
            const SchedulePlan plan = parse_plan(need(req, "plan"), model);
            const ComputeProfile comp = parse_compute_profile(need_arr(req, "compute_profile"));
            ProfileStore store(req.get("window") ? static_cast<int>(req.get("window")->as_int("window")) : 8);
            fill_store(need_arr(req, "samples"), store);
            auto cf = [&comp](int s, int bb, Direction dir) { return comp.get(s, bb, dir); };
            auto xf = [&store](LinkId l, Bytes bytes, Tick) { return store.estimate(l, bytes); };
            w.key("result");
            write_sim(w, simulate_with(plan, model, cf, xf, 0));
        } else if (op == "enumerate") {
            const ClusterSpec cluster = parse_cluster(need(req, "cluster"));
            const int k_max = req.get("k_max") ? static_cast<int>(req.get("k_max")->as_int("k_max"))
                                               : default_k_max(model);
            const CandidateSet set = enumerate_candidates(model, cluster, k_max);
            w.key("entries").begin_arr();
            for (const CandidateEntry& e : set.entries) {
                w.begin_arr().v(e.config.k).v(e.config.micro_batch_size).v(e.config.micro_batch_count);
                w.ints(e.memory.per_device_peak).end_arr();
            }
            w.end_arr();
        } else if (op == "profile") {
            const LinkTraces traces = parse_traces(req.get("traces"), model.stage_count());
            const SchedulePlan plan = parse_plan(need(req, "plan"), model);
            ProfileStore store(req.get("window") ? static_cast<int>(req.get("window")->as_int("window")) : 8);
            const Tick clock = req.get("clock") ? req.get("clock")->as_int("clock") : 0;
            const int reps = req.get("repeats") ? static_cast<int>(req.get("repeats")->as_int("repeats")) : 3;
            const Tick after = profile_links(plan, model, traces, clock, reps, store);
            w.key("clock").num(after);
            w.key("estimates").begin_arr();
            for (const auto& [l, b] : plan_buckets(plan)) w.begin_arr().v(l).v(b).v(store.estimate(l, b)).end_arr();
            w.end_arr();
        } else if (op == "compare") {
            const ClusterSpec cluster = parse_cluster(need(req, "cluster"));
            const LinkTraces traces = parse_traces(req.get("traces"), model.stage_count());
            const TuningPolicy pol = parse_policy(req.get("policy"));
            const CandidateSet set = enumerate_candidates(model, cluster, pol.k_max);
            std::vector<int> bs;
            for (const CandidateEntry& e : set.entries) bs.push_back(e.config.micro_batch_size);
            ProfileStore store(pol.window_size);
            const Tick clock = req.get("clock") ? req.get("clock")->as_int("clock") : 0;
            profile_buckets(candidate_buckets(set, model), traces, clock, pol.profile_repeats, store);
            const auto ranked = rank_candidates(set, model, ComputeProfile::from_model(model, bs), store);
            w.key("ranked").begin_arr();
            for (const PlanEstimate& e : ranked)
                w.begin_arr().v(e.config.k).v(e.config.micro_batch_size).v(e.config.micro_batch_count).v(e.estimated_length).end_arr();
            w.end_arr();
        } else if (op == "decide") {
            // the GPU tuner's decision, replayed from recorded int64-ns samples
            CandidateSet set;
            for (const Value& c : need_arr(req, "candidates").arr)
                set.entries.push_back({PlanConfig{static_cast<int>(entry(c, 0, "candidate").as_int("k")),
                                                  static_cast<int>(entry(c, 1, "candidate").as_int("b")),
                                                  static_cast<int>(entry(c, 2, "candidate").as_int("M"))},
                                       {}});
            const ComputeProfile comp = parse_compute_profile(need_arr(req, "compute_profile"));
            ProfileStore store(req.get("window") ? static_cast<int>(req.get("window")->as_int("window")) : 8);
            fill_store(need_arr(req, "samples"), store);
            PlanConfig cur{0, 0, 0};
            if (const Value* c = req.get("current"))
                cur = {static_cast<int>(entry(*c, 0, "current").as_int("k")), static_cast<int>(entry(*c, 1, "current").as_int("b")),
                       static_cast<int>(entry(*c, 2, "current").as_int("M"))};
            const double h = req.get("hysteresis") ? req.get("hysteresis")->as_double("hysteresis") : 0.02;
            const Tick t = req.get("clock") ? req.get("clock")->as_int("clock") : 0;
            // mixed-k candidates: [[b, [group sizes]], ...]; a mixed incumbent: current_groups
            std::vector<GroupCandidate> mixed;
            if (const Value* gc = req.get("group_candidates")) {
                if (gc->kind != Value::Array) throw ConfigError("group_candidates must be an array");
                for (const Value& c : gc->arr) {
                    GroupCandidate g;
                    g.micro_batch_size = static_cast<int>(entry(c, 0, "group candidate").as_int("b"));
                    const Value& sizes = entry(c, 1, "group candidate");
                    if (sizes.kind != Value::Array) throw ConfigError("group candidate sizes must be an array");
                    for (const Value& n : sizes.arr) g.groups.push_back(static_cast<int>(n.as_int("group size")));
                    mixed.push_back(std::move(g));
                }
            }
            std::vector<int> cur_groups;
            if (const Value* cg = req.get("current_groups")) {
                if (cg->kind != Value::Array) throw ConfigError("current_groups must be an array");
                for (const Value& n : cg->arr) cur_groups.push_back(static_cast<int>(n.as_int("group size")));
            }
            w.key("decision");
            write_decision(w, tuning_round_plans(set, mixed, model, comp, store, cur, cur_groups, h, t));
        } else if (op == "tune") {
            const ClusterSpec cluster = parse_cluster(need(req, "cluster"));
            const LinkTraces traces = parse_traces(req.get("traces"), model.stage_count());
            const TuningPolicy pol = parse_policy(req.get("policy"));
            const AdaptiveResult r = run_adaptive(model, cluster, traces, pol, need(req, "horizon").as_double("horizon"));
            w.key("rounds").begin_arr();
            for (const TuningDecision& d : r.log.rounds) write_decision(w, d);
            w.end_arr();
            w.key("iterations").begin_arr();
            for (const IterationRecord& it : r.iterations) {
                w.begin_arr().v(it.start).v(it.end).v(it.config.k).v(it.config.micro_batch_size);
                w.v(it.config.micro_batch_count).vd(it.throughput).end_arr();
            }
            w.end_arr();
            w.key("throughput").dbl(r.throughput());
        } else {
            throw ConfigError("unknown op '" + op + "'");
        }
    }
    w.end_obj();
    return w.out;
}

}  // namespace pipetune

extern "C" int ptk_scenario_json(const char* request, char* buf, size_t cap, size_t* written) {
    using namespace pipetune;
    std::string out;
    int rc = PTK_OK;
    try {
        if (request == nullptr) throw ConfigError("null request");
        out = run_scenario(request);
    } catch (const std::exception& e) {
        json::Writer w;
        w.begin_obj().key("error").str(error_name(e)).key("message").str(e.what()).end_obj();
        out = w.out;
        rc = ptk::set_error(error_status(e), e.what());
    }
    if (written) *written = out.size() + 1;
    if (buf == nullptr || cap < out.size() + 1) return rc != PTK_OK ? rc : PTK_ERR_NOMEM;
    std::memcpy(buf, out.data(), out.size() + 1);
    return rc;
}
