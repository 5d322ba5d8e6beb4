// Debug tool: tcgen05.mma issue/execute rate per shape on every SM (one CTA per SM, 512 MMAs
// back to back, operands from smem (SS) or A from TMEM (TS)).  Not part of the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -Iinclude -Ipaper_2303_01675_b200/csrc \
//        -o /tmp/mma_rate scripts/mma_rate.cu
#include <cstdio>

#include "../paper_2303_01675_b200/csrc/kernels/sm100_ptx.cuh"

using namespace ptk::sm100;

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) mma_rate(unsigned long long* cycles, int iters) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tmem_slot;
    __shared__ uint64_t done;
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) {
        mbar_init(&done, 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc<512>(&tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot;
    if (threadIdx.x == 0) {
        constexpr uint32_t idesc = make_idesc_bf16(128, N, false, N == 64);
        const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
        const unsigned long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const uint32_t k = i & 3;
            if (TS)
                mma_bf16_ts(tmem + 256, tmem + 384 + k * 8, make_sw128_desc(b + k * 32, N == 64 ? 8192 : 16, 1024), idesc, 1);
            else
                mma_bf16_ss(tmem + 256, make_sw128_desc(a + k * 32, 16, 1024),
                            make_sw128_desc(b + k * 32, N == 64 ? 8192 : 16, 1024), idesc, 1);
        }
        const unsigned long long t1 = clock64();
        mma_commit(&done);
        mbar_wait(&done, 0);
        const unsigned long long t2 = clock64();
        cycles[blockIdx.x * 2] = t1 - t0;
        cycles[blockIdx.x * 2 + 1] = t2 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

// Both operands MN-major (the weight-gradient layout), descriptors as gemm_sm100.cu builds them:
// 64-element MN atoms 8 KiB apart (LBO), 8-row K groups 1 KiB apart, K16 steps 2 KiB apart.
template <int N>
__global__ void __launch_bounds__(128, 1) mma_rate_mn(unsigned long long* cycles, int iters) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tmem_slot;
    __shared__ uint64_t done;
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) {
        mbar_init(&done, 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc<512>(&tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot;
    if (threadIdx.x == 0) {
        constexpr uint32_t idesc = make_idesc_bf16(128, N, true, true);
        const uint32_t a = smem_u32(smem), b = smem_u32(smem + 16384);
        const unsigned long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const uint32_t k = i & 3;
            mma_bf16_ss(tmem, make_sw128_desc(a + k * 2048, 8192, 1024), make_sw128_desc(b + k * 2048, 8192, 1024),
                        idesc, 1);
        }
        const unsigned long long t1 = clock64();
        mma_commit(&done);
        mbar_wait(&done, 0);
        const unsigned long long t2 = clock64();
        cycles[blockIdx.x * 2] = t1 - t0;
        cycles[blockIdx.x * 2 + 1] = t2 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

template <int N>
void run_mn(const char* name) {
    unsigned long long* d;
    cudaMalloc(&d, 148 * 2 * 8);
    cudaFuncSetAttribute(mma_rate_mn<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
    const int iters = 2048;
    mma_rate_mn<N><<<148, 128, 70 * 1024>>>(d, iters);
    mma_rate_mn<N><<<148, 128, 70 * 1024>>>(d, iters);
    unsigned long long h[296];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    double total = 0;
    for (int i = 0; i < 148; ++i) total += h[2 * i + 1];
    const double per = total / 148 / iters;
    printf("%-28s complete %.1f cycles/MMA  -> %.0f FLOP/clk/SM (%s)\n", name, per, 2.0 * 128 * N * 16 / per,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

template <int N, bool TS>
void run(const char* name) {
    unsigned long long* d;
    cudaMalloc(&d, 148 * 2 * 8);
    cudaFuncSetAttribute(mma_rate<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
    const int iters = 2048;
    mma_rate<N, TS><<<148, 128, 70 * 1024>>>(d, iters);
    mma_rate<N, TS><<<148, 128, 70 * 1024>>>(d, iters);
    unsigned long long h[296];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    double issue = 0, total = 0;
    for (int i = 0; i < 148; ++i) {
        issue += h[2 * i];
        total += h[2 * i + 1];
    }
    const double per = total / 148 / iters;
    printf("%-28s issue %.1f  complete %.1f cycles/MMA  -> %.0f FLOP/clk/SM (%s)\n", name, issue / 148 / iters, per,
           2.0 * 128 * N * 16 / per, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main_ld();

int main() {
    main_ld();
    run<128, false>("SS M128 N128 K16");
    run<64, false>("SS M128 N64 K16 (B MN-major)");
    run<64, true>("TS M128 N64 K16 (B MN-major)");
    run<128, true>("TS M128 N128 K16");
    run<256, false>("SS M128 N256 K16");
    run_mn<256>("SS M128 N256 K16 (A,B MN)");
    run_mn<128>("SS M128 N128 K16 (A,B MN)");
    return 0;
}

// TMEM load bandwidth: W warps each read 32 lanes x 32 fp32 columns (4 KiB) per tcgen05.ld,
// `iters` times (cycling over 128 columns), waiting after every `batch` loads.
template <int W, int BATCH>
__global__ void __launch_bounds__(32 * W, 1) ldtm_rate(unsigned long long* cycles, int iters) {
    __shared__ uint32_t tmem_slot;
    const int warp = threadIdx.x / 32;
    if (warp == 0) tmem_alloc<512>(&tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    float acc = 0.f;
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; i += BATCH) {
        float v[BATCH][32];
#pragma unroll
        for (int b = 0; b < BATCH; ++b) tmem_ld_32x32b_x32_nw(tmem + ((i + b) & 3) * 32 + (warp >> 2) * 128, v[b]);
        tmem_ld_wait();
#pragma unroll
        for (int b = 0; b < BATCH; ++b) acc += v[b][b];
    }
    __syncthreads();
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    if (acc == 12345.f) cycles[0] = 0;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc<512>(tmem_slot);
    }
}

template <int W, int BATCH>
void run_ld() {
    unsigned long long* d;
    cudaMalloc(&d, 148 * 8);
    const int iters = 1024;
    ldtm_rate<W, BATCH><<<148, 32 * W>>>(d, iters);
    ldtm_rate<W, BATCH><<<148, 32 * W>>>(d, iters);
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    double c = 0;
    for (int i = 0; i < 148; ++i) c += h[i];
    c /= 148;
    const double bytes = static_cast<double>(W) * iters * 32 * 32 * 4;
    printf("LDTM 32x32b.x32: %2d warps, %d in flight per warp: %.1f bytes/clk/SM (%s)\n", W, BATCH, bytes / c,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main_ld() {
    run_ld<4, 1>();
    run_ld<4, 4>();
    run_ld<8, 1>();
    run_ld<8, 4>();
    run_ld<16, 4>();
    return 0;
}
