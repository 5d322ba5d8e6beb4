// pipetune simulator (spec-only in the reference: SPEC.md:327-387).
//
// Deterministic discrete-event execution of a SchedulePlan with one compute,
// one send and one recv stream per device, per-device arrival buffer queues
// and FIFO send streams.  It is the CPU twin of the B200 executor, and (fed
// constant profiled durations) the cost model's engine.
//
// Semantics fixed here:
//  * a compute starts when its device is idle and its input Recv has landed;
//    GradAccum has zero duration;
//  * on completion its Send joins the producer's send-stream FIFO;
//  * a transfer starts at the earliest event time when the producer's send
//    stream AND the consumer's recv stream are both free; competing heads are
//    served in (enqueue time, send node id) order; it occupies both streams
//    for its duration and then pushes the input into the consumer's queue.
#pragma once

#include <functional>
#include <vector>

#include "pipetune/memory.hpp"
#include "pipetune/network.hpp"

namespace pipetune {

enum class Stream { Compute = 0, Send = 1, Recv = 2 };

struct TimelineEntry {
    int node = -1;
    int device = -1;
    Stream stream = Stream::Compute;
    Tick start = 0;
    Tick end = 0;
};

struct QueueLaunch {
    int node = -1;
    bool queue_nonempty = false;  // input arrived strictly before the device was free
};

struct DeviceState {
    Tick compute_free_at = 0;
    Tick send_stream_free_at = 0;
    Tick recv_stream_free_at = 0;
    int buffered = 0;      // arrived, unconsumed inputs
    Bytes resident_bytes = 0;
};

struct SimResult {
    Tick start = 0;
    Tick pipeline_length = 0;  // first event to last completion
    std::vector<Tick> per_device_busy;
    std::vector<Tick> per_device_bubble;
    std::vector<Bytes> observed_peak_bytes;
    std::vector<TimelineEntry> timeline;
    std::vector<std::vector<std::pair<Tick, int>>> queue_depth_trace;  // per device
    std::vector<std::vector<QueueLaunch>> launches;                    // per device, compute launches with an input
};

// Duration providers: compute(stage, micro_batch_size, dir) and
// transfer(link, bytes, start).
using ComputeDurationFn = std::function<Tick(int stage, int batch, Direction dir)>;
using TransferDurationFn = std::function<Tick(LinkId link, Bytes bytes, Tick start)>;

SimResult simulate_with(const SchedulePlan& plan, const ModelSpec& model, const ComputeDurationFn& compute,
                        const TransferDurationFn& transfer, Tick start = 0);

// True traces: compute_duration_ticks + transfer_duration.
SimResult simulate(const SchedulePlan& plan, const ModelSpec& model, const LinkTraces& traces, Tick start = 0);

// Measured execution (the B200 executor's records, on one clock) as a SimResult,
// so bubble_report / queue_analysis apply unchanged to hardware runs
// (SPEC.md:351-361).  A compute record is (device, compute node id, start, end);
// a transfer record is (link, micro-batch, start, end): link 2s carries F(s, m)'s
// output to stage s+1, link 2s-1 carries B(s, m)'s to stage s-1 (model.hpp link
// ids).  Busy = summed compute durations, bubble = active span - busy; a launch
// with an input is pre-buffered when that input landed strictly before the device
// was free (its previous compute ended; `start` before the first).  Throws
// ConfigError on records that do not belong to the plan.
struct HwCompute {
    int device = -1;
    int node = -1;
    Tick start = 0, end = 0;
};
struct HwTransfer {
    LinkId link = -1;
    int micro_batch = -1;
    Tick start = 0, end = 0;
};
SimResult result_from_records(const SchedulePlan& plan, const std::vector<HwCompute>& compute,
                              const std::vector<HwTransfer>& transfers, Tick start);

// bubble / (busy + bubble) per device (0 for an idle device).
std::vector<double> bubble_report(const SimResult& result);

// For each compute launch with an input on `device`: was it pre-buffered?
std::vector<QueueLaunch> queue_analysis(const SimResult& result, int device);

}  // namespace pipetune
