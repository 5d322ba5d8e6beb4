// SMs the persistent kernels (GEMM, attention) size their grids to.
//
// The preemption emulator launches small kernels on the send streams (the
// one-thread trace gates, and optionally the contender CTAs).  A persistent
// kernel holding every SM would delay each gate until it finishes, so the gates
// would add compute-dependent latency to every emulated transfer.  With
// PTK_SM_RESERVE=n (bench.py sets it for emulated multi-stage runs: 1, plus the
// contender's CTAs) the persistent kernels leave n SMs free for the emulator.
#pragma once

namespace ptk {

int device_sm_count();  // multiprocessors of the current device
int sm_budget();        // device_sm_count() - PTK_SM_RESERVE (read once), at least 2

}  // namespace ptk
