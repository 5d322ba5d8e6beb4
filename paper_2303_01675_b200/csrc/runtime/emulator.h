// Preemption emulator for the inter-stage links (north-star item 3).
//
// A LinkTrace (base bandwidth, latency, piecewise-constant
// availability) is uploaded to the device.  Every transfer on that link is
// split into chunks; before chunk i a one-thread gate kernel spins on
// %globaltimer until the trace says i*chunk bytes may have been delivered,
// and a final gate holds the transfer until the trace's completion time
// (+latency).  The copy engine moves each chunk at NVLink speed, so the
// delivered-bytes curve follows  transfer_duration(trace, bytes, start)  of
// the spec (network.cpp) whenever the emulated bandwidth is below the link's.
// A contender kernel (optional) adds real competing NVLink stores to the same
// peer while the trace is in a preempted segment.
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
    static constexpr int kChunks = 8;

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
