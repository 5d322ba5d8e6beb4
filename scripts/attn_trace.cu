// Debug tool: per-step timeline (SM clock cycles) of CTA 0 of the flash
// attention backward kernels at the GPT-1.3B shape.  Not part of the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 --expt-relaxed-constexpr -DPTK_ATTN_TRACE \
//        -Iinclude -Ipaper_2303_01675_b200/csrc -o scripts/attn_trace scripts/attn_trace.cu -lcuda
//   scripts/attn_trace 3 [cta]  (ping-pong forward of CTA cta; 2 single-tile forward; 1 / 0 backward KV / Q)
#include <cstdio>
#include <vector>

#include "../paper_2303_01675_b200/csrc/kernels/attention_sm100.cu"
#include "../paper_2303_01675_b200/csrc/runtime/sm_budget.cpp"

namespace ptk {  // the library's eager-load hook is not needed in this standalone tool
void preload_module_of(const void*) {}
}  // namespace ptk

__global__ void fill(__nv_bfloat16* p, size_t n, unsigned seed) {
    for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        unsigned x = static_cast<unsigned>(i) * 2654435761u ^ seed;
        x ^= x >> 13;
        x *= 0x5bd1e995u;
        x ^= x >> 15;
        p[i] = __float2bfloat16((static_cast<float>(x & 0xffff) / 65536.f - 0.5f));
    }
}

int main(int argc, char** argv) {
    const int kv = argc > 1 ? atoi(argv[1]) : 1;
    const int b = 2, s = 1024, H = 32, d = 64, h = H * d;
    const size_t T = static_cast<size_t>(b) * s;
    __nv_bfloat16 *qkv, *o, *dO, *dqkv;
    float *lse, *dsum;
    cudaMalloc(&qkv, T * 3 * h * 2);
    cudaMalloc(&o, T * h * 2);
    cudaMalloc(&dO, T * h * 2);
    cudaMalloc(&dqkv, T * 3 * h * 2);
    cudaMalloc(&lse, T * H * 4);
    cudaMalloc(&dsum, T * H * 4);
    fill<<<512, 256>>>(qkv, T * 3 * h, 1);
    fill<<<512, 256>>>(dO, T * h, 2);
    cudaMemcpyToSymbol(ptk::g_attn_trace_kv, &kv, sizeof kv);
    const int trace_cta = argc > 2 ? atoi(argv[2]) : 0;  // mode 3: the CTA whose timeline is recorded
    cudaMemcpyToSymbol(ptk::g_pp_trace_cta, &trace_cta, sizeof trace_cta);
    ptk::FlashPlan fp;
    ptk::FlashBwdPlan bp;
    if (ptk::flash_prepare(qkv, o, lse, b, s, H, d, &fp, 1) != cudaSuccess) return 1;
    if (ptk::flash_bwd_prepare(qkv, o, dO, lse, dsum, dqkv, b, s, H, d, &bp, 1) != cudaSuccess) return 1;
    for (int i = 0; i < 3; ++i) ptk::flash_forward(fp, 0);
    for (int i = 0; i < 3; ++i) ptk::flash_backward(bp, 0);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return 1;
    }
    if (kv == 9) {  // timing only: forward and backward, 20 launches each
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        float fms = 0.f, bms = 0.f;
        cudaEventRecord(e0);
        for (int i = 0; i < 20; ++i) ptk::flash_forward(fp, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&fms, e0, e1);
        cudaEventRecord(e0);
        for (int i = 0; i < 20; ++i) ptk::flash_backward(bp, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&bms, e0, e1);
        printf("fwd %.1f us  bwd %.1f us\n", fms * 50.f, bms * 50.f);
        return 0;
    }
    if (kv == 3) {  // ping-pong forward kernel timeline
        unsigned long long pt[3][64][8];
        cudaMemcpyFromSymbol(pt, ptk::g_pp_trace, sizeof pt);
        const unsigned long long p0 = pt[2][0][0];
        printf("ping-pong forward, CTA %d, cycles since S_A(0) was issued; per lane block n\n", trace_cta);
        printf("  n | lane A: s_full loaded exps pv_ok p_full | lane B: same | mma: S_A pA_seen PV_A S_B pB_seen PV_B\n");
        for (int n = 0; n < 24; ++n) {
            auto f = [&](int r, int ev) { return static_cast<long long>(pt[r][n][ev] - p0); };
            printf("%3d | %7lld %7lld %7lld %7lld %7lld | %7lld %7lld %7lld %7lld %7lld | %7lld %7lld %7lld %7lld %7lld %7lld\n",
                   n, f(0, 0), f(0, 1), f(0, 2), f(0, 3), f(0, 4), f(1, 0), f(1, 1), f(1, 2), f(1, 3), f(1, 4),
                   f(2, 0), f(2, 1), f(2, 2), f(2, 4), f(2, 5), f(2, 6));
        }
        unsigned long long ct[160][4];
        cudaMemcpyFromSymbol(ct, ptk::g_pp_cta, sizeof ct);
        unsigned long long t0 = ~0ull, t1 = 0;
        int grid = 0;
        for (int i = 0; i < 160 && ct[i][0]; ++i, ++grid) {
            t0 = ct[i][0] < t0 ? ct[i][0] : t0;
            t1 = ct[i][3] > t1 ? ct[i][3] : t1;
        }
        printf("CTAs %d, kernel span %.2f us (first entry to last exit)\n", grid, (t1 - t0) * 1e-3);
        printf("cta: entry first_S exit (us from the first entry)\n");
        for (int i = 0; i < grid; i += 8)
            printf("%3d: %6.2f %6.2f %6.2f\n", i, (ct[i][0] - t0) * 1e-3, (ct[i][1] - t0) * 1e-3,
                   (ct[i][3] - t0) * 1e-3);
        return 0;
    }
    if (kv == 2) {  // forward kernel timeline
        unsigned long long ft[2][64][8];
        cudaMemcpyFromSymbol(ft, ptk::g_fwd_trace, sizeof ft);
        const unsigned long long f0 = ft[1][0][0];
        printf("forward kernel, CTA 0, cycles since S_0 was issued\n");
        printf("blk | mma: S_issued p_full_seen PV_issued | sm: s_full s_loaded max_xchg exps_done pv_done_seen p_stored\n");
        for (int n = 0; n < 24; ++n) {
            auto f = [&](int r, int ev) { return static_cast<long long>(ft[r][n][ev] - f0); };
            printf("%3d | %8lld %8lld %8lld | %8lld %8lld %8lld %8lld %8lld %8lld\n", n, f(1, 0), f(1, 1), f(1, 2),
                   f(0, 0), f(0, 1), f(0, 2), f(0, 3), f(0, 4), f(0, 5));
        }
        return 0;
    }
    unsigned long long tr[2][64][8];
    cudaMemcpyFromSymbol(tr, ptk::g_attn_trace, sizeof tr);
    const unsigned long long t0 = tr[1][0][0];
    printf("%s kernel, CTA 0, cycles since the first XY issue\n", kv ? "KV" : "Q");
    printf("step | mma: xy_issue_begin xy_issued pd_full_seen acc_issued acc_done(MMA build only) | ew: row_barrier "
           "xy_full xy_free computed pd_free stored stored(warp 11)\n");
    for (int n = 0; n < 20; ++n) {
        auto f = [&](int r, int ev) { return static_cast<long long>(tr[r][n][ev] - t0); };
        printf("%3d | %8lld %8lld %8lld %8lld %8lld | %8lld %8lld %8lld %8lld %8lld %8lld %8lld\n", n, f(1, 0), f(1, 1),
               f(1, 2), f(1, 3), f(1, 4), f(0, 5), f(0, 0), f(0, 1), f(0, 2), f(0, 3), f(0, 4), f(0, 6));
    }
    return 0;
}
