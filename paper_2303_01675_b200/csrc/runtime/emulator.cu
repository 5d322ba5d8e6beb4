// Preemption emulator: trace-paced transfers + contender traffic (emulator.h).
#include "preload.h"
#include "emulator.h"

#include <algorithm>
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
// 2: hold until the whole transfer (+latency) is due.
__global__ void gate_kernel(const DevTrace* tr, int64_t* state, int64_t done, int mode) {
    const int64_t now = gtimer();
    if (mode == 0) {
        state[0] = now;
        return;
    }
    const int64_t target = deliver_time(tr, state[0], done) + (mode == 2 ? tr->latency : 0);
    while (gtimer() < target) __nanosleep(1000);
}

__global__ void timer_kernel(int64_t* out) { *out = gtimer(); }

// Contender: while the link is in a preempted segment (availability a < 1),
// stream 16-byte stores to the peer for a (1-a) fraction of every 50 us.
// Only thread 0 of each CTA polls the host-mapped stop flag and the trace
// (once per burst) and broadcasts through shared memory, so the contender does
// not flood PCIe with uncached reads.
__global__ void contender_kernel(const DevTrace* tr, uint4* peer, size_t n16, const volatile int* stop) {
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
                st = (a < 1.0 && static_cast<double>(now % period) < (1.0 - a) * period) ? 1 : 0;
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
    if (!active(slot)) return cudaMemcpyAsync(dst, src, static_cast<size_t>(bytes), cudaMemcpyDeviceToDevice, st);
    int64_t* state = state_ + slot * 8;
    gate_kernel<<<1, 1, 0, st>>>(dev_[slot], state, 0, 0);
    const int64_t chunk = ((bytes + kChunks - 1) / kChunks + 15) / 16 * 16;
    for (int64_t off = 0; off < bytes; off += chunk) {
        if (off > 0) gate_kernel<<<1, 1, 0, st>>>(dev_[slot], state, off, 1);
        const int64_t len = std::min(chunk, bytes - off);
        cudaError_t e = cudaMemcpyAsync(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off,
                                        static_cast<size_t>(len), cudaMemcpyDeviceToDevice, st);
        if (e != cudaSuccess) return e;
    }
    gate_kernel<<<1, 1, 0, st>>>(dev_[slot], state, bytes, 2);
    return cudaPeekAtLastError();
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
    contender_kernel<<<4, 128, 0, st>>>(dev_[slot], static_cast<uint4*>(peer_scratch), bytes / 16, stop_dev_);
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
