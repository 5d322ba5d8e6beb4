// Preemption emulator: trace-paced transfers + contender traffic (emulator.h).
#include "preload.h"
#include "emulator.h"

#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <stdexcept>

namespace ptk {

struct DevTrace {
    int nseg;
    double base;  // bytes per ns
    int64_t latency;
    int64_t epoch;
    const int64_t* start;
    const int64_t* end;
    const double* avail;
};

namespace {

__device__ __forceinline__ int64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return static_cast<int64_t>(t);
}

// Absolute time at which `bytes` have been delivered when streaming from t0.
__device__ int64_t deliver_time(const DevTrace* tr, int64_t t0, int64_t bytes) {
    double t = static_cast<double>(t0 - tr->epoch);
    double left = static_cast<double>(bytes);
    int i = 0;
    while (left > 0.0) {
        while (i < tr->nseg && static_cast<double>(tr->end[i]) <= t) ++i;
        double a = 1.0, next = -1.0;
        if (i < tr->nseg) {
            if (t < static_cast<double>(tr->start[i])) {
                next = static_cast<double>(tr->start[i]);
            } else {
                a = tr->avail[i];
                next = static_cast<double>(tr->end[i]);
            }
        }
        const double rate = tr->base * a;
        if (next < 0.0 || rate * (next - t) >= left) {
            t += left / rate;
            break;
        }
        left -= rate * (next - t);
        t = next;
    }
    return static_cast<int64_t>(t) + tr->epoch;
}

__device__ double avail_at(const DevTrace* tr, int64_t now) {
    const int64_t t = now - tr->epoch;
    for (int i = 0; i < tr->nseg; ++i) {
        if (t < tr->start[i]) return 1.0;
        if (t < tr->end[i]) return tr->avail[i];
    }
    return 1.0;
}

// mode 0: record the transfer start; 1: hold until `done` bytes are due;
// 2: hold until the whole transfer (+latency) is due; 3: record the start now and hold until
// `done` bytes (+latency) are due from it (the single gate paced_copy uses).
__global__ void gate_kernel(const DevTrace* tr, int64_t* state, int64_t done, int mode) {
    const int64_t now = gtimer();
    if (mode == 0) {
        state[0] = now;
        return;
    }
    const int64_t t0 = mode == 3 ? now : state[0];
    const int64_t target = deliver_time(tr, t0, done) + (mode >= 2 ? tr->latency : 0);
    while (gtimer() < target) __nanosleep(500);
}

__global__ void timer_kernel(int64_t* out) { *out = gtimer(); }

// Contender: while the link is in a preempted segment (availability a < 1),
// stream 16-byte stores to the peer for a (1-a) fraction of every 50 us.
// Only thread 0 of each CTA polls the host-mapped stop flag and the trace
// (once per burst) and broadcasts through shared memory, so the contender does
// not flood PCIe with uncached reads.
__global__ void contender_kernel(const DevTrace* tr, uint4* peer, size_t n16, const volatile int* stop,
                                 float duty_override) {
    __shared__ int s_state;  // 0 off, 1 on, 2 stop
    const int64_t period = 50000;
    size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    const uint4 v = make_uint4(0xdeadbeef, threadIdx.x, blockIdx.x, 0);
    for (;;) {
        if (threadIdx.x == 0) {
            int st = 0;
            if (*stop) {
                st = 2;
            } else {
                const int64_t now = gtimer();
                const double a = avail_at(tr, now);
                const double duty = duty_override >= 0.f ? duty_override : 1.0 - a;
                st = (a < 1.0 && static_cast<double>(now % period) < duty * period) ? 1 : 0;
            }
            s_state = st;
        }
        __syncthreads();
        const int st = s_state;
        __syncthreads();
        if (st == 2) break;
        if (st == 0) {
            __nanosleep(10000);
            continue;
        }
        for (int r = 0; r < 64; ++r) {
            peer[i] = v;
            i += stride;
            if (i >= n16) i -= n16;
        }
    }
}

void ck(cudaError_t e, const char* w) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("emulator ") + w + ": " + cudaGetErrorString(e));
}

}  // namespace

Emulator::~Emulator() {
    for (DevTrace* d : dev_)
        if (d) {
            DevTrace h;
            cudaMemcpy(&h, d, sizeof h, cudaMemcpyDeviceToHost);
            cudaFree(const_cast<int64_t*>(h.start));
            cudaFree(d);
        }
    if (state_) cudaFree(state_);
    if (stop_host_) cudaFreeHost(const_cast<int*>(stop_host_));
}

void Emulator::set_epoch(int64_t epoch_ns) {
    epoch_ = epoch_ns;
    for (int s = 0; s < kMaxLinks; ++s)
        if (host_[s].active) set_trace(s, host_[s]);
}

void Emulator::set_trace(int slot, const EmuTrace& t) {
    if (slot < 0 || slot >= kMaxLinks) throw std::invalid_argument("emulator slot");
    host_[slot] = t;
    if (!state_) {
        ck(cudaMalloc(&state_, 64 * sizeof(int64_t)), "alloc");
        ck(cudaMemset(state_, 0, 64 * sizeof(int64_t)), "memset");
    }
    if (dev_[slot]) {
        DevTrace old;
        ck(cudaMemcpy(&old, dev_[slot], sizeof old, cudaMemcpyDeviceToHost), "copy");
        cudaFree(const_cast<int64_t*>(old.start));
        cudaFree(dev_[slot]);
        dev_[slot] = nullptr;
    }
    if (!t.active) return;
    const int n = static_cast<int>(t.segments.size());
    const size_t bytes = static_cast<size_t>(std::max(n, 1)) * (8 + 8 + 8);
    char* arr = nullptr;
    ck(cudaMalloc(&arr, bytes), "alloc");
    std::vector<int64_t> s(n), e(n);
    std::vector<double> a(n);
    for (int i = 0; i < n; ++i) {
        s[i] = t.segments[i].start_ns;
        e[i] = t.segments[i].end_ns;
        a[i] = t.segments[i].availability;
    }
    const size_t cap = static_cast<size_t>(std::max(n, 1));
    if (n) {
        ck(cudaMemcpy(arr, s.data(), n * 8, cudaMemcpyHostToDevice), "copy");
        ck(cudaMemcpy(arr + cap * 8, e.data(), n * 8, cudaMemcpyHostToDevice), "copy");
        ck(cudaMemcpy(arr + cap * 16, a.data(), n * 8, cudaMemcpyHostToDevice), "copy");
    }
    DevTrace h{n, t.base_bytes_per_ns, t.latency_ns, epoch_, reinterpret_cast<const int64_t*>(arr),
               reinterpret_cast<const int64_t*>(arr + cap * 8), reinterpret_cast<const double*>(arr + cap * 16)};
    ck(cudaMalloc(&dev_[slot], sizeof(DevTrace)), "alloc");
    ck(cudaMemcpy(dev_[slot], &h, sizeof h, cudaMemcpyHostToDevice), "copy");
}

cudaError_t Emulator::paced_copy(int slot, void* dst, const void* src, int64_t bytes, cudaStream_t st) {
    // PTK_EMU_NO_GATE=1 (calibration only): copies unpaced even on a traced link, so the contender's
    // effect on a plain NVLink copy can be measured (scripts/contender_calibration.py)
    static const bool no_gate = std::getenv("PTK_EMU_NO_GATE") != nullptr;
    if (!active(slot) || no_gate)
        return cudaMemcpyAsync(dst, src, static_cast<size_t>(bytes), cudaMemcpyDeviceToDevice, st);
    // One gate per transfer: it records the start when the stream reaches the transfer and holds the
    // stream until the trace has delivered every byte (+ latency); the copy engine then moves the
    // payload at NVLink speed (tens of us), and the arrival flag written after it marks completion.
    // (Per-chunk gates cost one kernel launch each; each launch waited for a free SM slot behind
    // the compute kernels, adding 0.2-0.8 ms per transfer; profiles/r2_contender_calibration.md.)
    int64_t* state = state_ + slot * 8;
    gate_kernel<<<1, 1, 0, st>>>(dev_[slot], state, bytes, 3);
    cudaError_t e = cudaPeekAtLastError();
    if (e != cudaSuccess) return e;
    return cudaMemcpyAsync(dst, src, static_cast<size_t>(bytes), cudaMemcpyDeviceToDevice, st);
}

cudaError_t Emulator::start_contender(int slot, void* peer_scratch, size_t bytes, cudaStream_t st) {
    if (!active(slot)) return cudaSuccess;
    if (!stop_host_) {
        int* p = nullptr;
        ck(cudaHostAlloc(&p, sizeof(int), cudaHostAllocMapped), "host alloc");
        stop_host_ = p;
        ck(cudaHostGetDevicePointer(&stop_dev_, p, 0), "mapped");
    }
    *stop_host_ = 0;
    std::atomic_thread_fence(std::memory_order_seq_cst);
    // PTK_CONTENDER_CTAS (default 4) CTAs of peer stores; PTK_CONTENDER_DUTY overrides the duty
    // cycle 1 - availability (calibration runs: scripts/contender_calibration.py)
    static const int ctas = [] {
        const char* v = std::getenv("PTK_CONTENDER_CTAS");
        return v ? std::max(1, std::atoi(v)) : 4;
    }();
    static const float duty = [] {
        const char* v = std::getenv("PTK_CONTENDER_DUTY");
        return v ? static_cast<float>(std::atof(v)) : -1.f;
    }();
    contender_kernel<<<ctas, 128, 0, st>>>(dev_[slot], static_cast<uint4*>(peer_scratch), bytes / 16, stop_dev_,
                                           duty);
    return cudaPeekAtLastError();
}

void Emulator::stop_contender() {
    if (stop_host_) *stop_host_ = 1;
}

cudaError_t record_globaltimer(int64_t* dst, cudaStream_t st) {
    timer_kernel<<<1, 1, 0, st>>>(dst);
    return cudaPeekAtLastError();
}

int64_t device_globaltimer(cudaStream_t st) {
    int64_t* d = nullptr;
    int64_t h = 0;
    ck(cudaMalloc(&d, 8), "alloc");
    timer_kernel<<<1, 1, 0, st>>>(d);
    ck(cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, st), "copy");
    ck(cudaStreamSynchronize(st), "sync");
    cudaFree(d);
    return h;
}

void preload_emulator_kernels() { preload_module_of(reinterpret_cast<const void*>(&gate_kernel)); }

}  // namespace ptk
