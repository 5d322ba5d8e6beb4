// pipetune exception hierarchy — drop-in for proj/include/pipetune/errors.hpp:8-47.
//
// Invalid input is reported by throwing one of these; checkers return lists
// instead.  CudaError is the B200 addition: a nonzero ptk_* status from the
// C ABI surfaces as this type on the C++ side.
#pragma once

#include <stdexcept>
#include <string>

namespace pipetune {

struct Error : std::runtime_error {
    explicit Error(const std::string& what) : std::runtime_error(what) {}
};

#define PIPETUNE_ERROR_TYPE(Name) \
    struct Name : Error {         \
        explicit Name(const std::string& what) : Error(what) {} \
    }

PIPETUNE_ERROR_TYPE(ConfigError);       // malformed model / cluster / plan parameters
PIPETUNE_ERROR_TYPE(PlanError);         // plan parameters out of range (k < 1, k > M, cycles)
PIPETUNE_ERROR_TYPE(InfeasibleModel);   // no (k, b) fits the device memory limit
PIPETUNE_ERROR_TYPE(NoProfileData);     // profile bucket queried before any sample
PIPETUNE_ERROR_TYPE(DeadlockDetected);  // event loop stalled with work left
PIPETUNE_ERROR_TYPE(UnknownCandidate);  // plan switch to a config outside the candidate set
PIPETUNE_ERROR_TYPE(CudaError);         // B200 runtime failure reported through ptk.h

#undef PIPETUNE_ERROR_TYPE

}  // namespace pipetune
