// Host-side handle for one prepared GEMM launch (tensor maps encoded once).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include "../../../include/ptk.h"

namespace ptk {

struct GemmArgs {
    int M, N, K;
    int batch1;
    int bn;
    int tiles_m, tiles_n, tiles_per_batch, num_tiles;
    int causal, epi;
    void* C;
    int64_t ldc, c_bs1, c_bs2;
    void* C2;
    const void* aux;
    int64_t ld_aux, aux_bs1, aux_bs2;
    const void* bias;
    int tma_store;   // outputs leave through TMA stores (tmC / tmC2)
    float* col_part;  // optional [ceil(M/32)][N] += column sums of C per 32-row block
    int full_tiles;  // CTA-pair kernel: work items >= full_tiles are 256 x 128 halves of the tail tiles
    int n_fast;
    int mn5_a, mn5_b;  // CTA-pair kernel: MN-major A / B maps are 5-D (both 64-wide atoms in one box)
    int kb_split;    // CTA-pair kernel: k-blocks >= kb_split come from the second K segment (tmA2 / tmB2s)      // tile raster: 0 = m-tiles fastest (B tile shared), 1 = n-tiles fastest (A tile shared)
};

struct GemmPlan {
    using Launcher = int (*)(const GemmPlan&, cudaStream_t);
    alignas(64) CUtensorMap tmA;
    alignas(64) CUtensorMap tmB;
    alignas(64) CUtensorMap tmB2;  // CTA-pair kernel, K-major B: box of 64 rows (half-width tail tiles)
    alignas(64) CUtensorMap tmC;   // output C: box {64 bf16 | 32 fp32, 32 rows}, 128B swizzle
    alignas(64) CUtensorMap tmC2;  // BIAS_GELU pre-activation output
    alignas(64) CUtensorMap tmA2;  // second K segment (k2 > 0), CTA-pair kernel
    alignas(64) CUtensorMap tmB2s;
    GemmArgs args;
    int grid = 0;
    double flops = 0.0;  // algorithmic FLOPs of one launch
    bool multicast = false;
    Launcher launch = nullptr;
};

int gemm_prepare(const ptk_gemm_desc& d, GemmPlan* out);
int gemm_run(const GemmPlan& p, cudaStream_t stream);

}  // namespace ptk
