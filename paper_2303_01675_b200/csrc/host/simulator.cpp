// Discrete-event simulator.  See simulator.hpp for the
// stream/queue semantics; oracle/spec_oracle.py restates the same rules.
#include "pipetune/simulator.hpp"

#include <algorithm>
#include <deque>
#include <limits>
#include <queue>
#include <tuple>

#include "pipetune/errors.hpp"

namespace pipetune {

namespace {

struct Event {
    Tick time;
    long long seq;
    int kind;  // 0 compute end, 1 transfer end
    int device;
    int node;  // compute node or Send node
    bool operator>(const Event& o) const { return std::tie(time, seq) > std::tie(o.time, o.seq); }
};

struct Dev {
    DeviceState st;
    size_t pc = 0;
    bool busy = false;
    Tick prev_end = 0;  // when the device last became free (start clock initially)
    std::deque<std::pair<Tick, int>> sends;  // (enqueue time, Send id)
    Tick busy_sum = 0, first = -1, last = -1;
    Bytes peak = 0;
};

}  // namespace

SimResult simulate_with(const SchedulePlan& plan, const ModelSpec& model, const ComputeDurationFn& compute,
                        const TransferDurationFn& transfer, Tick start) {
    const TaskGraph& g = *plan.graph;
    const int S = plan.device_count();
    if (S != model.stage_count()) throw ConfigError("simulate: plan and model stage counts differ");
    const int b = plan.config.micro_batch_size;

    SimResult res;
    res.start = start;
    res.queue_depth_trace.resize(static_cast<size_t>(S));
    res.launches.resize(static_cast<size_t>(S));

    std::vector<Dev> dev(static_cast<size_t>(S));
    for (int d = 0; d < S; ++d) {
        Dev& x = dev[static_cast<size_t>(d)];
        x.st.compute_free_at = x.st.send_stream_free_at = x.st.recv_stream_free_at = start;
        x.prev_end = start;
        x.st.resident_bytes = model.stages[static_cast<size_t>(d)].weight_bytes;
        x.peak = x.st.resident_bytes;
    }
    std::vector<Tick> arrival(g.nodes.size(), -1);  // Recv id -> landing time
    std::priority_queue<Event, std::vector<Event>, std::greater<Event>> events;
    long long seq = 0;

    auto dispatch = [&](Tick now) {
        bool progress = true;
        while (progress) {
            progress = false;
            // computes, by device id
            for (int d = 0; d < S; ++d) {
                Dev& x = dev[static_cast<size_t>(d)];
                const auto& order = plan.per_device[static_cast<size_t>(d)];
                if (x.busy || x.pc >= order.size()) continue;
                const int id = order[x.pc];
                const int recv = g.recv_of_compute[static_cast<size_t>(id)];
                if (recv >= 0 && (arrival[static_cast<size_t>(recv)] < 0 || arrival[static_cast<size_t>(recv)] > now))
                    continue;
                const TaskNode& t = g.node(id);
                Tick dur = 0;
                const StageProfile& st = model.stages[static_cast<size_t>(d)];
                const Bytes act = st.activation_bytes_per_sample * static_cast<Bytes>(b);
                if (t.kind == TaskKind::ForwardCompute) {
                    dur = compute(d, b, Direction::Forward);
                    x.st.resident_bytes += act;
                    x.peak = std::max(x.peak, x.st.resident_bytes);
                } else if (t.kind == TaskKind::BackwardCompute) {
                    dur = compute(d, b, Direction::Backward);
                    x.st.resident_bytes -= act;
                }
                if (recv >= 0) {
                    res.launches[static_cast<size_t>(d)].push_back({id, arrival[static_cast<size_t>(recv)] < x.prev_end});
                    x.st.buffered -= 1;
                    res.queue_depth_trace[static_cast<size_t>(d)].push_back({now, x.st.buffered});
                }
                x.busy = true;
                x.st.compute_free_at = now + dur;
                x.busy_sum += dur;
                if (x.first < 0) x.first = now;
                x.last = now + dur;
                res.timeline.push_back({id, d, Stream::Compute, now, now + dur});
                events.push({now + dur, seq++, 0, d, id});
                ++x.pc;
                progress = true;
            }
            // transfers: head of every send FIFO, in (enqueue time, send id) order
            std::vector<std::tuple<Tick, int, int>> heads;  // (enq, send id, producer)
            for (int d = 0; d < S; ++d) {
                const Dev& x = dev[static_cast<size_t>(d)];
                if (!x.sends.empty()) heads.emplace_back(x.sends.front().first, x.sends.front().second, d);
            }
            std::sort(heads.begin(), heads.end());
            for (const auto& [enq, sid, p] : heads) {
                (void)enq;
                Dev& src = dev[static_cast<size_t>(p)];
                const int rid = g.pair_of[static_cast<size_t>(sid)];
                const int c = g.node(rid).device;
                Dev& dst = dev[static_cast<size_t>(c)];
                if (src.st.send_stream_free_at > now || dst.st.recv_stream_free_at > now) continue;
                const TaskNode& sn = g.node(sid);
                const Tick dur = transfer(sn.link, sn.payload_bytes, now);
                src.st.send_stream_free_at = now + dur;
                dst.st.recv_stream_free_at = now + dur;
                src.sends.pop_front();
                res.timeline.push_back({sid, p, Stream::Send, now, now + dur});
                res.timeline.push_back({rid, c, Stream::Recv, now, now + dur});
                events.push({now + dur, seq++, 1, c, sid});
                progress = true;
            }
        }
    };

    dispatch(start);
    Tick end = start;
    while (!events.empty()) {
        const Event e = events.top();
        events.pop();
        end = std::max(end, e.time);
        if (e.kind == 0) {
            Dev& x = dev[static_cast<size_t>(e.device)];
            x.busy = false;
            x.prev_end = e.time;
            const int sid = g.send_of_compute[static_cast<size_t>(e.node)];
            if (sid >= 0) x.sends.emplace_back(e.time, sid);
        } else {
            const int rid = g.pair_of[static_cast<size_t>(e.node)];
            arrival[static_cast<size_t>(rid)] = e.time;
            Dev& c = dev[static_cast<size_t>(e.device)];
            c.st.buffered += 1;
            res.queue_depth_trace[static_cast<size_t>(e.device)].push_back({e.time, c.st.buffered});
        }
        if (!events.empty() && events.top().time == e.time) continue;  // drain same-time events first
        dispatch(e.time);
    }
    for (int d = 0; d < S; ++d) {
        const Dev& x = dev[static_cast<size_t>(d)];
        if (x.pc < plan.per_device[static_cast<size_t>(d)].size() || !x.sends.empty())
            throw DeadlockDetected("simulate: device " + std::to_string(d) + " stalled at action " +
                                   std::to_string(x.pc) + " with work remaining");
    }
    res.pipeline_length = end - start;
    for (int d = 0; d < S; ++d) {
        const Dev& x = dev[static_cast<size_t>(d)];
        const Tick span = x.first < 0 ? 0 : x.last - x.first;
        res.per_device_busy.push_back(x.busy_sum);
        res.per_device_bubble.push_back(span - x.busy_sum);
        res.observed_peak_bytes.push_back(x.peak);
    }
    return res;
}

SimResult simulate(const SchedulePlan& plan, const ModelSpec& model, const LinkTraces& traces, Tick start) {
    model.validate();
    for (const TaskNode& t : plan.graph->nodes)
        if (t.kind == TaskKind::Send && (t.link < 0 || static_cast<size_t>(t.link) >= traces.size()))
            throw ConfigError("simulate: no trace for link " + std::to_string(t.link));
    auto comp = [&model](int s, int b, Direction dir) {
        return compute_duration_ticks(model.stages[static_cast<size_t>(s)], b, dir);
    };
    auto xfer = [&traces](LinkId l, Bytes bytes, Tick t) {
        return transfer_duration(traces[static_cast<size_t>(l)], bytes, t);
    };
    return simulate_with(plan, model, comp, xfer, start);
}

SimResult result_from_records(const SchedulePlan& plan, const std::vector<HwCompute>& compute,
                              const std::vector<HwTransfer>& transfers, Tick start) {
    const TaskGraph& g = *plan.graph;
    const int S = plan.device_count();
    SimResult res;
    res.start = start;
    res.queue_depth_trace.resize(static_cast<size_t>(S));
    res.launches.resize(static_cast<size_t>(S));
    std::vector<Tick> arrival(g.nodes.size(), -1);  // Recv id -> landing time
    Tick end = start;
    for (const HwTransfer& x : transfers) {
        if (x.link < 0 || x.link >= link_count(S) || x.micro_batch < 0 || x.micro_batch >= plan.config.micro_batch_count)
            throw ConfigError("result_from_records: transfer outside the plan");
        const bool fwd = x.link % 2 == 0;
        const int producer = fwd ? x.link / 2 : (x.link + 1) / 2;
        int cid = -1;
        for (int id : plan.per_device[static_cast<size_t>(producer)]) {
            const TaskNode& t = g.node(id);
            if (t.micro_batch == x.micro_batch &&
                t.kind == (fwd ? TaskKind::ForwardCompute : TaskKind::BackwardCompute)) {
                cid = id;
                break;
            }
        }
        const int sid = cid < 0 ? -1 : g.send_of_compute[static_cast<size_t>(cid)];
        if (sid < 0) throw ConfigError("result_from_records: no Send for a transfer record");
        const int rid = g.pair_of[static_cast<size_t>(sid)];
        arrival[static_cast<size_t>(rid)] = x.end;
        res.timeline.push_back({sid, producer, Stream::Send, x.start, x.end});
        res.timeline.push_back({rid, g.node(rid).device, Stream::Recv, x.start, x.end});
        end = std::max(end, x.end);
    }
    std::vector<std::vector<const HwCompute*>> per(static_cast<size_t>(S));
    for (const HwCompute& c : compute) {
        if (c.device < 0 || c.device >= S || c.node < 0 || static_cast<size_t>(c.node) >= g.nodes.size() ||
            g.node(c.node).device != c.device)
            throw ConfigError("result_from_records: compute record outside the plan");
        per[static_cast<size_t>(c.device)].push_back(&c);
    }
    for (int d = 0; d < S; ++d) {
        auto& v = per[static_cast<size_t>(d)];
        std::stable_sort(v.begin(), v.end(), [](const HwCompute* a, const HwCompute* b) { return a->start < b->start; });
        Tick busy = 0, first = -1, last = -1, prev_end = start;
        std::vector<std::tuple<Tick, int, int>> qev;  // (time, 0 arrival / 1 launch, node)
        for (const HwCompute* c : v) {
            busy += c->end - c->start;
            if (first < 0) first = c->start;
            last = std::max(last, c->end);
            res.timeline.push_back({c->node, d, Stream::Compute, c->start, c->end});
            const int recv = g.recv_of_compute[static_cast<size_t>(c->node)];
            if (recv >= 0) {
                const Tick a = arrival[static_cast<size_t>(recv)];
                if (a < 0) throw ConfigError("result_from_records: a compute's input transfer is missing");
                res.launches[static_cast<size_t>(d)].push_back({c->node, a < prev_end});
                qev.emplace_back(a, 0, recv);
                qev.emplace_back(c->start, 1, c->node);
            }
            prev_end = c->end;
            end = std::max(end, c->end);
        }
        std::sort(qev.begin(), qev.end());
        int depth = 0;
        for (const auto& [t, kind, node] : qev) {
            (void)node;
            depth += kind == 0 ? 1 : -1;
            res.queue_depth_trace[static_cast<size_t>(d)].push_back({t, depth});
        }
        res.per_device_busy.push_back(busy);
        res.per_device_bubble.push_back(first < 0 ? 0 : (last - first) - busy);
        res.observed_peak_bytes.push_back(0);
    }
    res.pipeline_length = end - start;
    return res;
}

std::vector<double> bubble_report(const SimResult& r) {
    std::vector<double> out;
    for (size_t d = 0; d < r.per_device_busy.size(); ++d) {
        const Tick tot = r.per_device_busy[d] + r.per_device_bubble[d];
        out.push_back(tot == 0 ? 0.0 : static_cast<double>(r.per_device_bubble[d]) / static_cast<double>(tot));
    }
    return out;
}

std::vector<QueueLaunch> queue_analysis(const SimResult& r, int device) {
    if (device < 0 || static_cast<size_t>(device) >= r.launches.size())
        throw ConfigError("queue_analysis: device out of range");
    return r.launches[static_cast<size_t>(device)];
}

}  // namespace pipetune
