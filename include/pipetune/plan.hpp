// pipetune planner — drop-in for proj/include/pipetune/plan.hpp:13-49.
//
// Per-device total orders over compute nodes for GPipe, 1F1B and kFkB
// (group-granularity 1F1B).  The B200 stage executor issues exactly these
// orders; Send/Recv launch order is induced by them.
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "pipetune/taskgraph.hpp"

namespace pipetune {

// [begin, end) into one device's action list; a unit holds at most k
// consecutive computes of one kind.
struct ScheduleUnit {
    int begin = 0;
    int end = 0;
};

struct SchedulePlan {
    std::shared_ptr<const TaskGraph> graph;
    PlanConfig config;
    std::vector<std::vector<int>> per_device;      // node ids, in issue order
    std::vector<std::vector<ScheduleUnit>> units;  // per device

    int device_count() const { return static_cast<int>(per_device.size()); }
};

SchedulePlan plan_1f1b(std::shared_ptr<const TaskGraph> graph);

// k = 1 reproduces plan_1f1b and k = M reproduces plan_gpipe; the last group
// is short when k does not divide M.  PlanError unless 1 <= k <= M.
SchedulePlan plan_kfkb(std::shared_ptr<const TaskGraph> graph, int k);

SchedulePlan plan_gpipe(std::shared_ptr<const TaskGraph> graph);

// "F0 F1 B0 ..." rendering of one device's order (GA appended on request).
std::string sequence_string(const SchedulePlan& plan, int device, bool include_grad_accum = false);

// Empty iff each device list covers its compute nodes exactly once, is a
// linear extension of the projected dependencies, and every link's send order
// equals its recv order.
std::vector<std::string> check_plan(const SchedulePlan& plan);

// ---- B200 extension: kFkB over an explicit group list.
// groups[i] = {first, last} (inclusive) consecutive micro-batch ranges that
// partition [0, M).  plan_kfkb(g, k) == plan_groups(g, k, uniform groups).
struct MicroBatchGroup {
    int first = 0;
    int last = 0;
};
std::vector<MicroBatchGroup> micro_batch_groups(int micro_batches, int k);
SchedulePlan plan_groups(std::shared_ptr<const TaskGraph> graph, int k, const std::vector<MicroBatchGroup>& groups);

}  // namespace pipetune
