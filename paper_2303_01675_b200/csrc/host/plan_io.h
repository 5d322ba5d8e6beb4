// Shared helpers between the C-ABI translation units of the host layer.
#pragma once

#include <exception>
#include <string>

#include "../../../include/ptk.h"
#include "pipetune/plan.hpp"

namespace pipetune {

ModelSpec model_from_c(const ptk_model* m);
const char* error_name(const std::exception& e);
int error_status(const std::exception& e);
std::string plan_to_json(const SchedulePlan& plan);

}  // namespace pipetune
