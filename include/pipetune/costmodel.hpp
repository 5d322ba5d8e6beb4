// pipetune cost model (spec-only in the reference: SPEC.md:389-436).
//
// Pipeline-length estimate = the simulator run over constant profiled
// durations (moving-average comm profiles, once-measured compute profiles).
#pragma once

#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "pipetune/simulator.hpp"

namespace pipetune {

// Measured compute durations per (stage, micro-batch size, direction).
class ComputeProfile {
  public:
    void set(int stage, int batch, Direction dir, Tick duration);
    Tick get(int stage, int batch, Direction dir) const;  // NoProfileData if absent
    bool has(int stage, int batch, Direction dir) const;

    // The simulated world's "measurement": exact compute_duration_ticks for
    // every stage and each b in `batches`.
    static ComputeProfile from_model(const ModelSpec& model, const std::vector<int>& batches);

  private:
    std::map<std::tuple<int, int, int>, Tick> d_;
};

struct PlanEstimate {
    PlanConfig config;
    Tick estimated_length = 0;
    std::string inputs_digest;  // the profile values used, rendered
    std::vector<int> groups;    // explicit group sizes (plan_groups); empty = uniform kFkB at config.k
};

PlanEstimate estimate_length(const SchedulePlan& plan, const ModelSpec& model, const ComputeProfile& compute,
                             const ProfileStore& comm);

// Ascending estimate; ties: smaller k, then larger b.
std::vector<PlanEstimate> rank_candidates(const CandidateSet& candidates, const ModelSpec& model,
                                          const ComputeProfile& compute, const ProfileStore& comm);

// A mixed-k candidate: kFkB over explicit consecutive group sizes at micro-batch size b
// (plan_groups; the reference planner's make_plan walks any group list, plan.cpp:20-21, 61-66).
// Under constant profiled durations the one that pays off is "remainder group first": when k
// does not divide M, a short FIRST group shortens the warm-up that uniform kFkB's short LAST
// group does not.
struct GroupCandidate {
    int micro_batch_size = 1;
    std::vector<int> groups;
};

// rank_candidates over uniform candidates and mixed-k plans together.  Ascending estimate;
// ties: smaller (max) k, larger b, then group list (uniform first).
std::vector<PlanEstimate> rank_plans(const CandidateSet& candidates, const std::vector<GroupCandidate>& mixed,
                                     const ModelSpec& model, const ComputeProfile& compute, const ProfileStore& comm);

// Builds the kFkB plan of a candidate config.
SchedulePlan plan_for(const ModelSpec& model, const PlanConfig& config);

}  // namespace pipetune
