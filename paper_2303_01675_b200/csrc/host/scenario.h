// Scenario (JSON) parsing helpers shared by the C ABI and the GPU executor.
#pragma once

#include <string>

#include "json_in.h"
#include "pipetune/tuner.hpp"

namespace pipetune {

ModelSpec parse_model(const json::Value& v);
ClusterSpec parse_cluster(const json::Value& v);
LinkTrace parse_trace(const json::Value& v);
LinkTraces parse_traces(const json::Value* v, int stage_count);
TuningPolicy parse_policy(const json::Value* v);
std::string run_scenario(const std::string& request);

}  // namespace pipetune
