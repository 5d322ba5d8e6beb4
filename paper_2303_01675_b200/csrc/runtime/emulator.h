// Preemption emulator for the inter-stage links (north-star item 3).
//
// A LinkTrace (base bandwidth, latency, piecewise-constant
// availability) is uploaded to the device.  Every transfer on that link is
// preceded by one one-thread gate kernel on the send stream: it records the
// transfer's start (%globaltimer) and spins until the trace has delivered all
// its bytes (+latency) — the device twin of transfer_duration(trace, bytes,
// start) of the spec (network.cpp); the copy engine then moves the payload at
// NVLink speed and the arrival flag marks completion.  Send streams run at the
// highest priority so a gate never waits behind pending compute CTAs, and
// bench.py leaves one SM free of persistent kernels (runtime/sm_budget.h).
// A contender kernel (optional, PTK_CONTENDER_CTAS CTAs) adds real competing
// NVLink stores to the same peer while the trace is in a preempted segment;
// its calibration is profiles/r2_contender_calibration.md.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace ptk {

struct EmuSegment {
    int64_t start_ns, end_ns;  // relative to the job epoch
    double availability;
};

struct EmuTrace {
    bool active = false;
    double base_bytes_per_ns = 0.0;  // emulated link bandwidth at availability 1
    int64_t latency_ns = 0;
    std::vector<EmuSegment> segments;
};

struct DevTrace;  // device-side copy

class Emulator {
  public:
    static constexpr int kMaxLinks = 2;  // a stage sends on at most two links

    Emulator() = default;
    ~Emulator();
    void set_trace(int slot, const EmuTrace& t);
    bool active(int slot) const { return slot >= 0 && slot < kMaxLinks && host_[slot].active; }
    // epoch = %globaltimer value all trace times are relative to
    void set_epoch(int64_t epoch_ns);
    // Paced peer copy on `st` (gates + chunked cudaMemcpyAsync).
    cudaError_t paced_copy(int slot, void* dst, const void* src, int64_t bytes, cudaStream_t st);
    // Contender: peer stores into `peer_scratch` during preempted segments,
    // until *stop (host-mapped) becomes nonzero.
    cudaError_t start_contender(int slot, void* peer_scratch, size_t bytes, cudaStream_t st);
    void stop_contender();

  private:
    EmuTrace host_[kMaxLinks];
    DevTrace* dev_[kMaxLinks] = {nullptr, nullptr};
    int64_t* state_ = nullptr;  // per slot: transfer start time
    volatile int* stop_host_ = nullptr;
    int* stop_dev_ = nullptr;
    int64_t epoch_ = 0;
};

// Reads %globaltimer on the device (ns) — used to align trace epochs.
int64_t device_globaltimer(cudaStream_t st);
// Enqueues a one-thread kernel writing %globaltimer to *dst (device memory) on `st`.
cudaError_t record_globaltimer(int64_t* dst, cudaStream_t st);

}  // namespace ptk
