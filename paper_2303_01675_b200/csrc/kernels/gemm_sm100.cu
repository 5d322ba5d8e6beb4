// Persistent, warp-specialised bf16 GEMM for sm_100a (tcgen05 + TMEM + TMA).
//
//   D[z][m][n] = sum_k A[z][m][k] * B[z][n][k]      (fp32 accumulate in TMEM)
//
// A and B are each either K-major (k contiguous) or MN-major (m / n
// contiguous); the operand layout is folded into the TMA box and the UMMA
// smem descriptor, so the dense-layer forward (X·Wᵀ), dgrad (dY·W) and wgrad
// (dYᵀ·X) and every attention product are the same kernel without a
// transpose pass.  One CTA per SM, 10 warps (kThreads = 320):
//   warp 0      TMA producer (one elected lane)
//   warp 1      TMEM allocator + tcgen05.mma issuer (one elected lane)
//   warps 2..9  epilogue, two per TMEM lane quarter: tcgen05.ld → fused epilogue →
//               swizzled smem staging → TMA store / reduce-add
// The accumulator is double-buffered in TMEM (2 x BN fp32 columns) so the
// epilogue of tile i overlaps the main loop of tile i+1.
//
// Epilogues (runtime switch, warp-uniform):
//   EPI_BF16      C = acc (+bias[n]) (+aux[m][n])          bf16 out
//   EPI_F32       C = acc                                   fp32 out
//   EPI_ACC_F32   C += acc                                  fp32 in/out (wgrad accumulation, β=1)
//   EPI_BIAS_GELU C2 = acc+bias (pre-activation), C = gelu(C2)   bf16 out
//   EPI_DGELU     C = acc * gelu'(aux[m][n])                bf16 out
// Causal modes (attention):
//   CAUSAL_TILES  only tiles with n0 <= m0 (+BM-1) are computed (lower-triangular output, BM == BN)
//   CAUSAL_KHEAD  k range clipped to [0, m0+BM)   (P·V, dS·K: P/dS are zero above the diagonal)
//   CAUSAL_KTAIL  k range clipped to [m0, K)      (dSᵀ·Q, Pᵀ·dO)

#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "../runtime/preload.h"
#include "../../../include/ptk.h"
#include "gemm_sm100.h"
#include "launch.cuh"
#include "sm100_ptx.cuh"
#include "../runtime/sm_budget.h"

namespace ptk {

using namespace sm100;

namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;  // 64 bf16 = 128 B = one swizzle row
constexpr int kThreads = 320;  // TMA warp, MMA warp, 8 epilogue warps
constexpr int kSmemBudget = 226 * 1024;

template <int BN>
struct Cfg {
    static constexpr int kABytes = kBM * kBK * 2;
    static constexpr int kBBytes = BN * kBK * 2;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kEpiBytes = 8 * 32 * 32 * 4 + 2 * BN * 2;  // transpose buffers + 2 bias slices
    static constexpr int kStagesRaw = (kSmemBudget - 2048 - kEpiBytes) / kStageBytes;
    static constexpr int kStages = kStagesRaw > 8 ? 8 : kStagesRaw;
    static constexpr int kTmemCols = 2 * BN < 32 ? 32 : 2 * BN;
    static constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align slack*/ + 512 /*barriers*/ + kEpiBytes;
};

__device__ __forceinline__ float tanh_fast(float x) {
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float gelu_tanh(float x) {
    const float k0 = 0.7978845608028654f, k1 = 0.044715f;
    const float u = k0 * (x + k1 * x * x * x);
    return 0.5f * x * (1.f + tanh_fast(u));
}

__device__ __forceinline__ float gelu_tanh_grad(float x) {
    const float k0 = 0.7978845608028654f, k1 = 0.044715f;
    const float x2 = x * x;
    const float t = tanh_fast(k0 * (x + k1 * x * x2));
    return 0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * k0 * (1.f + 3.f * k1 * x2);
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}


__device__ __forceinline__ void unpack_bf16x8(const uint4& u, float (&f)[8]) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 p = __bfloat1622float2(h[i]);
        f[2 * i] = p.x;
        f[2 * i + 1] = p.y;
    }
}

__device__ __forceinline__ uint4 pack_bf16x8(const float* f) {
    uint4 u;
    u.x = pack_bf16(f[0], f[1]);
    u.y = pack_bf16(f[2], f[3]);
    u.z = pack_bf16(f[4], f[5]);
    u.w = pack_bf16(f[6], f[7]);
    return u;
}

struct TileCoord {
    int z1, z2, m0, n0, kb0, kb1;
    int ncols;  // output columns of this tile (BN, or 128 for a CTA-pair tail half)
};

// MC: a 2-CTA cluster owns a pair of m-tiles sharing one n-tile; t indexes
// pairs and `rank` picks the CTA's half of the pair.
template <bool MC>
__device__ __forceinline__ TileCoord decode_tile(const GemmArgs& a, int t, int rank) {
    TileCoord c;
    const int z = t / a.tiles_per_batch;
    int r = t - z * a.tiles_per_batch;
    int mb, nb;
    if (MC) {
        const int mpairs = (a.tiles_m + 1) / 2;
        nb = r / mpairs;
        mb = 2 * (r - nb * mpairs) + rank;
    } else if (a.causal == PTK_CAUSAL_TILES) {
        // r enumerates the lower triangle row by row: row i holds i+1 tiles.
        mb = static_cast<int>((sqrtf(8.f * r + 1.f) - 1.f) * 0.5f);
        while ((mb + 1) * (mb + 2) / 2 <= r) ++mb;
        while (mb * (mb + 1) / 2 > r) --mb;
        nb = r - mb * (mb + 1) / 2;
    } else if (a.n_fast) {
        mb = r / a.tiles_n;
        nb = r - mb * a.tiles_n;
    } else {
        nb = r / a.tiles_m;
        mb = r - nb * a.tiles_m;
    }
    c.z1 = z % a.batch1;
    c.z2 = z / a.batch1;
    c.m0 = mb * kBM;
    c.n0 = nb * a.bn;
    c.ncols = a.bn;
    const int kbs = (a.K + kBK - 1) / kBK;
    c.kb0 = 0;
    c.kb1 = kbs;
    if (a.causal == PTK_CAUSAL_KHEAD) {
        const int kend = min(a.K, c.m0 + kBM);
        c.kb1 = (kend + kBK - 1) / kBK;
    } else if (a.causal == PTK_CAUSAL_KTAIL) {
        c.kb0 = min(c.m0 / kBK, kbs - 1);
    }
    return c;
}

// ---------------------------------------------------------------- epilogue
__device__ __forceinline__ bool epi_has_aux(const GemmArgs& a) {
    return (a.epi == PTK_EPI_BF16 && a.aux != nullptr) || a.epi == PTK_EPI_DGELU;
}

// Every global input of a tile's epilogue that does not depend on the
// accumulator (bias slice -> smem, residual / pre-activation aux rows) is
// fetched BEFORE the epilogue waits for the accumulator, so its latency hides
// under the main loop; the next step's aux is fetched during this step.
// Warp (quad, half) owns TMEM lanes [32 quad, +32).
// bf16 outputs leave in 64-column steps (s = half, half+2, ... of BN/64),
// fp32 outputs in 32-column chunks (c = half, half+2, ...): the warp writes
// its 32 rows of the step into its own 4 KB staging buffer in the 128B-swizzled
// layout (16-byte chunk j of row r at (j ^ r%8)), and one lane issues a TMA
// store of the [32 x 128 B] box — full-line writes that bypass the LSU, so the
// epilogue does not compete with the tensor core for L1/smem wavefronts.
// EPI_ACC_F32 uses the TMA reduce-add (C += tile, one fp32 add per element).
struct EpiTmaIn {
    uint4 aux[8];  // next step's aux: 8 x (8 bf16) of this thread's row
};

__device__ __forceinline__ void epi_fetch_aux64(const GemmArgs& args, const TileCoord& tc, int step, int quad,
                                                uint32_t lane, uint4 (&aux)[8]) {
    const int gm = tc.m0 + quad * 32 + static_cast<int>(lane);
    const int64_t xrow = tc.z1 * args.aux_bs1 + tc.z2 * args.aux_bs2 + static_cast<int64_t>(gm) * args.ld_aux;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int gn = tc.n0 + step * 64 + 8 * j;
        aux[j] = (gm < args.M && gn < args.N)
                     ? *reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(args.aux) + xrow + gn)
                     : make_uint4(0u, 0u, 0u, 0u);
    }
}

template <int BN>
__device__ __forceinline__ void epi_prefetch_tma(const GemmArgs& args, const TileCoord& tc, int quad, int half,
                                                 uint32_t lane, int et, __nv_bfloat16* bias_s, EpiTmaIn& in) {
    if (epi_has_aux(args) && half < tc.ncols / 64) epi_fetch_aux64(args, tc, half, quad, lane, in.aux);
    if (args.bias != nullptr) {
        if (et < BN / 8) {
            const int gn = tc.n0 + et * 8;
            const uint4 v = gn < args.N ? *reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(args.bias) + gn)
                                        : make_uint4(0u, 0u, 0u, 0u);
            *reinterpret_cast<uint4*>(bias_s + et * 8) = v;
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");
    }
}

// 8 x 16 bytes of this lane's row into the swizzled staging buffer, then one TMA store.
__device__ __forceinline__ void epi_stage_store(const CUtensorMap* map, uint8_t* stage, uint32_t lane,
                                                const uint4 (&row)[8], int c0, int c1, int c2, int c3, bool reduce) {
    if (lane == 0) tma_store_wait_read();  // the previous store from this buffer has read it
    __syncwarp();
    const uint32_t base = smem_u32(stage) + lane * 128;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const uint32_t a = base + ((j ^ (lane & 7)) * 16);
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(row[j].x), "r"(row[j].y),
                     "r"(row[j].z), "r"(row[j].w)
                     : "memory");
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
        if (reduce)
            tma_reduce_add_4d(map, stage, c0, c1, c2, c3);
        else
            tma_store_4d(map, stage, c0, c1, c2, c3);
        tma_store_commit();
    }
}

template <int BN>
__device__ __forceinline__ void epilogue_tile_tma(const CUtensorMap* tmC, const CUtensorMap* tmC2,
                                                  const GemmArgs& args, const TileCoord& tc, uint32_t tmem_col,
                                                  int quad, int half, uint32_t lane, uint8_t* stage,
                                                  const __nv_bfloat16* bias_s, EpiTmaIn& in) {
    const uint32_t lane_addr = static_cast<uint32_t>(quad * 32) << 16;
    const int row0 = tc.m0 + quad * 32;
    if (args.epi == PTK_EPI_F32 || args.epi == PTK_EPI_ACC_F32) {
        const bool reduce = args.epi == PTK_EPI_ACC_F32;
#pragma unroll 1
        for (int c = half; c < tc.ncols / 32; c += 2) {
            float v[32];
            tmem_ld_32x32b_x32(tmem_col + lane_addr + static_cast<uint32_t>(c * 32), v);
            uint4 row[8];
#pragma unroll
            for (int j = 0; j < 8; ++j)
                row[j] = make_uint4(__float_as_uint(v[4 * j]), __float_as_uint(v[4 * j + 1]),
                                    __float_as_uint(v[4 * j + 2]), __float_as_uint(v[4 * j + 3]));
            epi_stage_store(tmC, stage, lane, row, tc.n0 + c * 32, row0, tc.z1, tc.z2, reduce);
        }
        return;
    }
#pragma unroll 1
    for (int st = half; st < tc.ncols / 64; st += 2) {
        float v[64];
        tmem_ld_32x32b_x32_nw(tmem_col + lane_addr + static_cast<uint32_t>(st * 64), v);
        tmem_ld_32x32b_x32_nw(tmem_col + lane_addr + static_cast<uint32_t>(st * 64 + 32), v + 32);
        tmem_ld_wait();
        uint4 out[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            float* f = v + 8 * j;
            if (args.bias != nullptr) {
                float bb[8];
                unpack_bf16x8(*reinterpret_cast<const uint4*>(bias_s + st * 64 + 8 * j), bb);
#pragma unroll
                for (int i = 0; i < 8; ++i) f[i] += bb[i];
            }
            if (args.epi == PTK_EPI_BF16 && args.aux != nullptr) {
                float r[8];
                unpack_bf16x8(in.aux[j], r);
#pragma unroll
                for (int i = 0; i < 8; ++i) f[i] += r[i];
            } else if (args.epi == PTK_EPI_DGELU) {
                float p[8];
                unpack_bf16x8(in.aux[j], p);
#pragma unroll
                for (int i = 0; i < 8; ++i) f[i] *= gelu_tanh_grad(p[i]);
            }
            out[j] = pack_bf16x8(f);
        }
        if (epi_has_aux(args) && st + 2 < tc.ncols / 64) epi_fetch_aux64(args, tc, st + 2, quad, lane, in.aux);
        if (args.epi == PTK_EPI_BIAS_GELU) {
            // out holds the rounded pre-activation: store it (C2), then C = gelu(pre as stored)
            epi_stage_store(tmC2, stage, lane, out, tc.n0 + st * 64, row0, tc.z1, tc.z2, false);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                float p[8];
                unpack_bf16x8(out[j], p);
#pragma unroll
                for (int i = 0; i < 8; ++i) p[i] = gelu_tanh(p[i]);
                out[j] = pack_bf16x8(p);
            }
        }
        epi_stage_store(tmC, stage, lane, out, tc.n0 + st * 64, row0, tc.z1, tc.z2, false);
        if (args.col_part != nullptr) {
            // column sums of this warp's 32 rows of the step, read back from the swizzled staging
            // buffer (lane l: columns 2l, 2l+1; conflict-free), into partial row (row0 / 32)
            const uint32_t base = smem_u32(stage);
            const int jc = static_cast<int>(lane >> 2), wc = static_cast<int>(lane & 3);
            float s0 = 0.f, s1 = 0.f;
            for (int r = 0; r < 32 && row0 + r < args.M; ++r) {
                uint32_t v;
                asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v)
                             : "r"(base + r * 128 + ((jc ^ (r & 7)) * 16) + wc * 4));
                const float2 f = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&v));
                s0 += f.x;
                s1 += f.y;
            }
            const int gn = tc.n0 + st * 64 + 2 * static_cast<int>(lane);
            if (gn < args.N) {
                float* pp = args.col_part + static_cast<int64_t>(row0 / 32) * args.N + gn;
                pp[0] += s0;
                pp[1] += s1;
            }
        }
    }
}

template <int BN, bool A_MN, bool B_MN, bool MC>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmC2,
                     const __grid_constant__ GemmArgs args) {
    using C = Cfg<BN>;
    constexpr int S = C::kStages;
    constexpr uint32_t kIdesc = make_idesc_bf16(kBM, BN, A_MN, B_MN);

    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* epi_smem = smem + S * C::kStageBytes;  // 8 warps x 4 KB staging (1024-aligned), then 2 bias slices
    uint64_t* full = reinterpret_cast<uint64_t*>(epi_smem + C::kEpiBytes);
    uint64_t* empty = full + S;
    uint64_t* tfull = empty + S;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x / 32;
    const uint32_t lane = lane_id();
    const int rank = MC ? static_cast<int>(cluster_ctarank()) : 0;
    const int t_begin = MC ? static_cast<int>(blockIdx.x) / 2 : static_cast<int>(blockIdx.x);
    const int t_step = MC ? static_cast<int>(gridDim.x) / 2 : static_cast<int>(gridDim.x);

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], MC ? 2 : 1);  // MC: both CTAs must release a stage (B is shared)
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 8);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<C::kTmemCols>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    if (MC) cluster_sync();  // peer barriers initialised before any multicast lands
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    pdl_begin();  // previous kernel complete: operands / aux / C visible

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer
            int stage = 0;
            uint32_t phase = 0;
            for (int t = t_begin; t < args.num_tiles; t += t_step) {
                const TileCoord tc = decode_tile<MC>(args, t, rank);
                for (int kb = tc.kb0; kb < tc.kb1; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
                    uint8_t* sa = smem + stage * C::kStageBytes;
                    uint8_t* sb = sa + C::kABytes;
                    const int k0 = kb * kBK;
                    if (!A_MN) {
                        tma_load_4d(&tmA, &full[stage], sa, k0, tc.m0, tc.z1, tc.z2);
                    } else if (args.mn5_a) {  // both 64-wide M atoms in one 5-D box
                        tma_load_5d(&tmA, &full[stage], sa, 0, k0, tc.m0 / 64, tc.z1, tc.z2);
                    } else {
#pragma unroll
                        for (int j = 0; j < kBM / 64; ++j)
                            tma_load_4d(&tmA, &full[stage], sa + j * 64 * kBK * 2, tc.m0 + 64 * j, k0, tc.z1, tc.z2);
                    }
                    if (MC) {
                        // this CTA fetches its half of the shared B tile into both CTAs
                        if (!B_MN) {
                            tma_load_4d_mc(&tmB, &full[stage], sb + rank * (BN / 2) * 128, k0, tc.n0 + rank * (BN / 2),
                                           tc.z1, tc.z2, 0x3);
                        } else {
#pragma unroll
                            for (int j = rank * (BN / 128); j < (rank + 1) * (BN / 128); ++j)
                                tma_load_4d_mc(&tmB, &full[stage], sb + j * 64 * kBK * 2, tc.n0 + 64 * j, k0, tc.z1,
                                               tc.z2, 0x3);
                        }
                    } else if (!B_MN) {
                        tma_load_4d(&tmB, &full[stage], sb, k0, tc.n0, tc.z1, tc.z2);
                    } else if (args.mn5_b) {  // the BN/64 atoms in one 5-D box
                        tma_load_5d(&tmB, &full[stage], sb, 0, k0, tc.n0 / 64, tc.z1, tc.z2);
                    } else {
#pragma unroll
                        for (int j = 0; j < BN / 64; ++j)
                            tma_load_4d(&tmB, &full[stage], sb + j * 64 * kBK * 2, tc.n0 + 64 * j, k0, tc.z1, tc.z2);
                    }
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ---------------- MMA issuer
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int t = t_begin; t < args.num_tiles; t += t_step) {
                const TileCoord tc = decode_tile<MC>(args, t, rank);
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
                for (int kb = tc.kb0; kb < tc.kb1; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t a_base = smem_u32(smem + stage * C::kStageBytes);
                    const uint32_t b_base = a_base + C::kABytes;
#pragma unroll
                    for (int k = 0; k < kBK / 16; ++k) {
                        // K-major: advance 32 B inside the swizzled 128 B row.
                        // MN-major: advance two 8-row core groups (2 x 1024 B).
                        const uint64_t da = A_MN ? make_sw128_desc(a_base + k * 2048, 64 * kBK * 2, 1024)
                                                 : make_sw128_desc(a_base + k * 32, 16, 1024);
                        const uint64_t db = B_MN ? make_sw128_desc(b_base + k * 2048, 64 * kBK * 2, 1024)
                                                 : make_sw128_desc(b_base + k * 32, 16, 1024);
                        mma_bf16_ss(d_tmem, da, db, kIdesc, (kb > tc.kb0 || k > 0) ? 1u : 0u);
                    }
                    if (MC)
                        mma_commit_mc(&empty[stage], 0x3);  // release the stage in both CTAs
                    else
                        mma_commit(&empty[stage]);
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                mma_commit(&tfull[acc]);
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    } else {
        // ---------------- epilogue warps: 8 warps, two per TMEM lane quadrant
        // (warp % 4); the pair splits the 32-column chunks of a tile.
        const int quad = warp & 3;
        const int half = (warp - 2) >> 2;  // 0 or 1
        uint8_t* stage = epi_smem + (warp - 2) * 4096;  // 32 rows x 128 B, 128B-swizzled
        __nv_bfloat16* bias_s = reinterpret_cast<__nv_bfloat16*>(epi_smem + 8 * 32 * 32 * 4);  // [2][BN]
        const int et = (warp - 2) * 32 + static_cast<int>(lane);
        int acc = 0;
        uint32_t acc_phase = 0;
        EpiTmaIn tin;
        for (int t = t_begin; t < args.num_tiles; t += t_step) {
            const TileCoord tc = decode_tile<MC>(args, t, rank);
            epi_prefetch_tma<BN>(args, tc, quad, half, lane, et, bias_s + acc * BN, tin);
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            epilogue_tile_tma<BN>(&tmC, &tmC2, args, tc, tmem_base + static_cast<uint32_t>(acc * BN), quad, half, lane,
                                  stage, bias_s + acc * BN, tin);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
        if (lane == 0) tma_store_wait_all();  // staging must outlive the stores
    }

    tc_fence_before();
    __syncthreads();
    if (MC) cluster_sync();  // no CTA leaves while its peer may still signal it
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<C::kTmemCols>(tmem_base);
    }
}


// ---------------------------------------------------------------------------
// CTA-pair GEMM: tcgen05.mma.cta_group::2 with a 256 x 256 pair tile.  Each
// CTA stages only its own 128 rows of A and 128 rows (N) of B per k-step
// (32 KiB, 6 stages), the leader issues M=256 MMAs that read both CTAs' smem,
// and each CTA's TMEM receives its own 128 output rows.  TMA completion bytes
// of both CTAs land on the leader's full barrier; the leader's commits are
// multicast to both CTAs' empty / tmem-full barriers; both CTAs' epilogue
// warps release the accumulator on the leader's tmem-empty barrier.
constexpr int k2smStages = 6;
constexpr int k2smStageBytes = 2 * 128 * kBK * 2;  // A half + B half
constexpr int k2smSmem = k2smStages * k2smStageBytes + 1024 + 512 + 8 * 32 * 32 * 4 + 2 * 256 * 2;

// Work item t: t < full_tiles is the 256 x 256 pair tile t; the tiles after
// full_tiles (the last, partial wave) are split into two 256 x 128 halves,
// items full_tiles + 2h and + 2h + 1, so the tail wave takes half as long.
__device__ __forceinline__ TileCoord decode_pair_tile(const GemmArgs& a, int t, int rank) {
    int tile = t, nhalf = -1;
    if (t >= a.full_tiles) {
        tile = a.full_tiles + (t - a.full_tiles) / 2;
        nhalf = (t - a.full_tiles) & 1;
    }
    TileCoord c;
    const int z = tile / a.tiles_per_batch;
    const int r = tile - z * a.tiles_per_batch;
    const int mpairs = (a.tiles_m + 1) / 2;
    int nb, mp;
    if (a.n_fast) {
        mp = r / a.tiles_n;
        nb = r - mp * a.tiles_n;
    } else {
        nb = r / mpairs;
        mp = r - nb * mpairs;
    }
    c.z1 = z % a.batch1;
    c.z2 = z / a.batch1;
    c.m0 = mp * 256 + rank * 128;
    c.n0 = nb * 256 + (nhalf > 0 ? 128 : 0);
    c.ncols = nhalf < 0 ? 256 : 128;
    c.kb0 = 0;
    c.kb1 = (a.K + kBK - 1) / kBK;
    return c;
}

template <bool A_MN, bool B_MN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_2sm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                         const __grid_constant__ CUtensorMap tmB2, const __grid_constant__ CUtensorMap tmC,
                         const __grid_constant__ CUtensorMap tmC2, const __grid_constant__ CUtensorMap tmA2,
                         const __grid_constant__ CUtensorMap tmB2s, const __grid_constant__ GemmArgs args) {
    constexpr int S = k2smStages;
    constexpr int kHalf = 128 * kBK * 2;  // 16 KiB
    constexpr uint32_t kIdesc = make_idesc_bf16(256, 256, A_MN, B_MN);
    constexpr uint32_t kIdescHalf = make_idesc_bf16(256, 128, A_MN, B_MN);

    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* epi_smem = smem + S * k2smStageBytes;  // 8 warps x 4 KB staging (1024-aligned), then 2 bias slices
    uint64_t* full = reinterpret_cast<uint64_t*>(epi_smem + 8 * 32 * 32 * 4 + 2 * 256 * 2);
    uint64_t* empty = full + S;
    uint64_t* tfull = empty + S;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x / 32;
    const uint32_t lane = lane_id();
    const int rank = static_cast<int>(cluster_ctarank());
    const bool leader = rank == 0;
    const int t_begin = static_cast<int>(blockIdx.x) / 2;
    const int t_step = static_cast<int>(gridDim.x) / 2;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 16);  // 8 epilogue warps x 2 CTAs (leader's copy is the one used)
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc_2sm<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    pdl_begin();  // previous kernel complete: operands / aux / C visible

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer (both CTAs)
            int stage = 0;
            uint32_t phase = 0;
            for (int t = t_begin; t < args.num_tiles; t += t_step) {
                const TileCoord tc = decode_pair_tile(args, t, rank);
                const bool full_w = tc.ncols == 256;
                const int nrow = tc.n0 + rank * (tc.ncols / 2);  // this CTA's half of the B rows
                const uint32_t bytes = full_w ? 2 * k2smStageBytes : 2 * (kHalf + kHalf / 2);
                for (int kb = tc.kb0; kb < tc.kb1; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (leader) mbar_arrive_expect_tx(&full[stage], bytes);
                    uint8_t* sa = smem + stage * k2smStageBytes;
                    uint8_t* sb = sa + kHalf;
                    // second K segment: the other micro-batch's operands (tmA2 / tmB2s)
                    const bool seg2 = args.kb_split > 0 && kb >= args.kb_split;
                    const int k0 = (seg2 ? kb - args.kb_split : kb) * kBK;
                    const CUtensorMap* ma = seg2 ? &tmA2 : &tmA;
                    const CUtensorMap* mb = seg2 ? &tmB2s : &tmB;
                    if (!A_MN) {
                        tma_load_4d_2sm(ma, &full[stage], sa, k0, tc.m0, tc.z1, tc.z2);
                    } else if (args.mn5_a) {  // both 64-wide M atoms in one box
                        tma_load_5d_2sm(ma, &full[stage], sa, 0, k0, tc.m0 / 64, tc.z1, tc.z2);
                    } else {
#pragma unroll
                        for (int j = 0; j < 2; ++j)
                            tma_load_4d_2sm(ma, &full[stage], sa + j * 64 * kBK * 2, tc.m0 + 64 * j, k0, tc.z1, tc.z2);
                    }
                    if (!B_MN) {
                        tma_load_4d_2sm(full_w ? mb : &tmB2, &full[stage], sb, k0, nrow, tc.z1, tc.z2);
                    } else if (args.mn5_b) {  // one box: two atoms (tmB / tmB2s), one for a tail half (tmB2)
                        tma_load_5d_2sm(full_w ? mb : &tmB2, &full[stage], sb, 0, k0, nrow / 64, tc.z1, tc.z2);
                    } else {
                        for (int j = 0; j < (full_w ? 2 : 1); ++j)
                            tma_load_4d_2sm(mb, &full[stage], sb + j * 64 * kBK * 2, nrow + 64 * j, k0, tc.z1, tc.z2);
                    }
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (leader && lane == 0) {  // ---------------- MMA issuer (leader CTA only)
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int t = t_begin; t < args.num_tiles; t += t_step) {
                const TileCoord tc = decode_pair_tile(args, t, rank);
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * 256);
                for (int kb = tc.kb0; kb < tc.kb1; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t a_base = smem_u32(smem + stage * k2smStageBytes);
                    const uint32_t b_base = a_base + kHalf;
#pragma unroll
                    for (int k = 0; k < kBK / 16; ++k) {
                        const uint64_t da = A_MN ? make_sw128_desc(a_base + k * 2048, 64 * kBK * 2, 1024)
                                                 : make_sw128_desc(a_base + k * 32, 16, 1024);
                        const uint64_t db = B_MN ? make_sw128_desc(b_base + k * 2048, 64 * kBK * 2, 1024)
                                                 : make_sw128_desc(b_base + k * 32, 16, 1024);
                        mma_bf16_ss_2sm(d_tmem, da, db, tc.ncols == 256 ? kIdesc : kIdescHalf,
                                        (kb > tc.kb0 || k > 0) ? 1u : 0u);
                    }
                    mma_commit_2sm_mc(&empty[stage], 0x3);
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                mma_commit_2sm_mc(&tfull[acc], 0x3);
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    } else {  // ---------------- epilogue warps (both CTAs): this CTA's 128 rows
        const int quad = warp & 3;
        const int half = (warp - 2) >> 2;
        uint8_t* stage = epi_smem + (warp - 2) * 4096;  // 32 rows x 128 B, 128B-swizzled
        __nv_bfloat16* bias_s = reinterpret_cast<__nv_bfloat16*>(epi_smem + 8 * 32 * 32 * 4);  // [2][256]
        const int et = (warp - 2) * 32 + static_cast<int>(lane);
        int acc = 0;
        uint32_t acc_phase = 0;
        EpiTmaIn tin;
        for (int t = t_begin; t < args.num_tiles; t += t_step) {
            const TileCoord tc = decode_pair_tile(args, t, rank);
            epi_prefetch_tma<256>(args, tc, quad, half, lane, et, bias_s + acc * 256, tin);
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            epilogue_tile_tma<256>(&tmC, &tmC2, args, tc, tmem_base + static_cast<uint32_t>(acc * 256), quad, half,
                                   lane, stage, bias_s + acc * 256, tin);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (leader)
                    mbar_arrive(&tempty[acc]);
                else
                    mbar_arrive_remote(&tempty[acc], 0);
            }
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
        if (lane == 0) tma_store_wait_all();  // staging must outlive the stores
    }

    tc_fence_before();
    __syncthreads();
    cluster_sync();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_2sm<512>(tmem_base);
    }
}

// ------------------------------------------------------------------ host side

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

// Operand map: dims = {contiguous, strided, batch1, batch2}; box = {64, rows}.
// MN-major operand as a 5-D view {64, strided, contig/64, batch1, batch2}: one box of `blocks`
// 64-wide atoms lands them back to back in smem, exactly as `blocks` separate 4-D boxes would.
int encode_operand_mn5(CUtensorMap* map, const ptk_matrix& m, int contig_extent, int strided_extent, int box_rows,
                       int blocks, int batch1, int batch2) {
    EncodeTiledFn enc = encode_fn();
    if (enc == nullptr) return PTK_ERR_CUDA;
    if ((reinterpret_cast<uintptr_t>(m.ptr) & 15) != 0 || (m.ld * 2) % 16 != 0 || contig_extent % 64 != 0)
        return PTK_ERR_ALIGN;
    const int64_t row_bytes = m.ld * 2;
    int64_t s1 = m.batch_stride[0] * 2, s2 = m.batch_stride[1] * 2;
    if (batch1 <= 1) s1 = row_bytes * strided_extent;
    if (batch2 <= 1) s2 = s1 * (batch1 > 0 ? batch1 : 1);
    if (s1 % 16 != 0 || s2 % 16 != 0 || s1 <= 0 || s2 <= 0) return PTK_ERR_ALIGN;
    cuuint64_t dims[5] = {64, static_cast<cuuint64_t>(strided_extent), static_cast<cuuint64_t>(contig_extent / 64),
                          static_cast<cuuint64_t>(batch1), static_cast<cuuint64_t>(batch2)};
    cuuint64_t strides[4] = {static_cast<cuuint64_t>(row_bytes), 128, static_cast<cuuint64_t>(s1),
                             static_cast<cuuint64_t>(s2)};
    cuuint32_t box[5] = {64, static_cast<cuuint32_t>(box_rows), static_cast<cuuint32_t>(blocks), 1, 1};
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, m.ptr, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? PTK_OK : PTK_ERR_CUDA;
}

int encode_operand(CUtensorMap* map, const ptk_matrix& m, int contig_extent, int strided_extent, int box_rows,
                   int batch1, int batch2) {
    EncodeTiledFn enc = encode_fn();
    if (enc == nullptr) return PTK_ERR_CUDA;
    if ((reinterpret_cast<uintptr_t>(m.ptr) & 15) != 0 || (m.ld * 2) % 16 != 0) return PTK_ERR_ALIGN;
    cuuint64_t dims[4] = {static_cast<cuuint64_t>(contig_extent), static_cast<cuuint64_t>(strided_extent),
                          static_cast<cuuint64_t>(batch1), static_cast<cuuint64_t>(batch2)};
    const int64_t row_bytes = m.ld * 2;
    int64_t s1 = m.batch_stride[0] * 2, s2 = m.batch_stride[1] * 2;
    if (batch1 <= 1) s1 = row_bytes * strided_extent;
    if (batch2 <= 1) s2 = s1 * (batch1 > 0 ? batch1 : 1);
    if (s1 % 16 != 0 || s2 % 16 != 0 || s1 <= 0 || s2 <= 0) return PTK_ERR_ALIGN;
    cuuint64_t strides[3] = {static_cast<cuuint64_t>(row_bytes), static_cast<cuuint64_t>(s1),
                             static_cast<cuuint64_t>(s2)};
    cuuint32_t box[4] = {64, static_cast<cuuint32_t>(box_rows), 1, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, m.ptr, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? PTK_OK : PTK_ERR_CUDA;
}

// Output map: dims = {N, M, batch1, batch2}; box = {128 B of columns, 32 rows}, 128B swizzle.
int encode_output(CUtensorMap* map, void* ptr, int64_t ld, int64_t bs1, int64_t bs2, int M, int N, int batch1,
                  int batch2, bool f32) {
    EncodeTiledFn enc = encode_fn();
    if (enc == nullptr || ptr == nullptr) return PTK_ERR_CUDA;
    const int64_t es = f32 ? 4 : 2;
    if ((reinterpret_cast<uintptr_t>(ptr) & 15) != 0 || (ld * es) % 16 != 0) return PTK_ERR_ALIGN;
    cuuint64_t dims[4] = {static_cast<cuuint64_t>(N), static_cast<cuuint64_t>(M), static_cast<cuuint64_t>(batch1),
                          static_cast<cuuint64_t>(batch2)};
    const int64_t row_bytes = ld * es;
    int64_t s1 = bs1 * es, s2 = bs2 * es;
    if (batch1 <= 1) s1 = row_bytes * M;
    if (batch2 <= 1) s2 = s1 * (batch1 > 0 ? batch1 : 1);
    if (s1 % 16 != 0 || s2 % 16 != 0 || s1 <= 0 || s2 <= 0) return PTK_ERR_ALIGN;
    cuuint64_t strides[3] = {static_cast<cuuint64_t>(row_bytes), static_cast<cuuint64_t>(s1),
                             static_cast<cuuint64_t>(s2)};
    cuuint32_t box[4] = {static_cast<cuuint32_t>(128 / es), 32, 1, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = enc(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, ptr, dims,
                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? PTK_OK : PTK_ERR_CUDA;
}

template <int BN, bool A_MN, bool B_MN, bool MC>
int launch_impl(const GemmPlan& p, cudaStream_t stream) {
    using C = Cfg<BN>;
    static bool attr_set = false;
    auto kern = gemm_bf16_kernel<BN, A_MN, B_MN, MC>;
    if (!attr_set) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes) != cudaSuccess)
            return PTK_ERR_CUDA;
        attr_set = true;
    }
    if (launch_kernel(kern, p.grid, kThreads, C::kSmemBytes, stream, MC ? 2 : 1, p.tmA, p.tmB, p.tmC, p.tmC2,
                      p.args) != cudaSuccess)
        return PTK_ERR_CUDA;
    return cudaPeekAtLastError() == cudaSuccess ? PTK_OK : PTK_ERR_CUDA;
}

template <bool A_MN, bool B_MN>
int launch_2sm(const GemmPlan& p, cudaStream_t stream) {
    static bool attr_set = false;
    auto kern = gemm_bf16_2sm_kernel<A_MN, B_MN>;
    if (!attr_set) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, k2smSmem) != cudaSuccess)
            return PTK_ERR_CUDA;
        attr_set = true;
    }
    if (launch_kernel(kern, p.grid, kThreads, k2smSmem, stream, 2, p.tmA, p.tmB, p.tmB2, p.tmC, p.tmC2, p.tmA2, p.tmB2s,
                      p.args) != cudaSuccess)
        return PTK_ERR_CUDA;
    return cudaPeekAtLastError() == cudaSuccess ? PTK_OK : PTK_ERR_CUDA;
}

GemmPlan::Launcher pick_2sm(bool a_mn, bool b_mn) {
    if (!a_mn && !b_mn) return &launch_2sm<false, false>;
    if (!a_mn && b_mn) return &launch_2sm<false, true>;
    if (a_mn && !b_mn) return &launch_2sm<true, false>;
    return &launch_2sm<true, true>;
}

template <int BN, bool MC>
GemmPlan::Launcher pick(bool a_mn, bool b_mn) {
    if (!a_mn && !b_mn) return &launch_impl<BN, false, false, MC>;
    if (!a_mn && b_mn) return &launch_impl<BN, false, true, MC>;
    if (a_mn && !b_mn) return &launch_impl<BN, true, false, MC>;
    return &launch_impl<BN, true, true, MC>;
}

int num_sms() { return sm_budget(); }  // runtime/sm_budget.h: PTK_SM_RESERVE leaves SMs to the emulator

}  // namespace

int gemm_prepare(const ptk_gemm_desc& d, GemmPlan* out) {
    if (d.m <= 0 || d.n <= 0 || d.k <= 0) return PTK_ERR_ARG;
    if (d.n % 8 != 0) return PTK_ERR_ARG;
    const int b1 = d.batch[0] > 0 ? d.batch[0] : 1;
    const int b2 = d.batch[1] > 0 ? d.batch[1] : 1;
    const int tiles_m = (d.m + kBM - 1) / kBM;

    int bn;
    if (d.k2 > 0) {
        // two K segments: CTA-pair kernel only, dense, unbatched, segment boundary on a k-block
        if (d.k % kBK != 0 || b1 * b2 != 1 || d.causal != PTK_CAUSAL_NONE || d.multicast != 2 || tiles_m < 2 ||
            d.a2.mn_major != d.a.mn_major || d.b2.mn_major != d.b.mn_major || d.col_part != nullptr)
            return PTK_ERR_ARG;
        bn = 256;
    } else if (d.bn_hint == 64 || d.bn_hint == 128 || d.bn_hint == 256) {
        bn = d.bn_hint;
    } else if (d.causal == PTK_CAUSAL_TILES) {
        bn = 128;
    } else if (d.n <= 64) {
        bn = 64;
    } else if (d.n <= 128) {
        bn = 128;
    } else {
        // Prefer the wide tile unless the narrow one fills the machine clearly better.
        const int sms = num_sms();
        auto eff = [&](int w) {
            const long tiles = static_cast<long>(tiles_m) * ((d.n + w - 1) / w) * b1 * b2;
            const long waves = (tiles + sms - 1) / sms;
            return static_cast<double>(tiles) / static_cast<double>(waves * sms);
        };
        double e256 = eff(256);
        if (d.multicast == 2 && tiles_m >= 2 && d.causal == PTK_CAUSAL_NONE) {
            // CTA-pair 256 x 256 tiles on sms/2 pairs, partial last wave split into halves
            const long t = static_cast<long>((tiles_m + 1) / 2) * ((d.n + 255) / 256) * b1 * b2;
            const long p = sms / 2;
            const long rem = t % p;
            double rounds = static_cast<double>(t / p);
            if (rem > 0) rounds += (t > p && 2 * rem <= p && d.n % 256 == 0) ? 0.5 : 1.0;
            e256 = static_cast<double>(t) / (static_cast<double>(p) * rounds) + 0.1;  // pair kernel: faster per SM
        }
        bn = eff(128) > e256 + 0.15 ? 128 : 256;
        // narrow tiles only when the machine is otherwise mostly idle (small M x N, e.g. BERT-large's
        // 1024 x 1024 out-proj weight gradient: 16 pair tiles on 74 pairs); a 128 x 64 tile is
        // smem-operand bound at ~2/3 of the wide tiles' per-SM rate
        if (0.67 * eff(64) > std::max(e256, eff(128) - 0.15)) bn = 64;
    }
    if (d.causal == PTK_CAUSAL_TILES && (bn != kBM || d.m != d.n)) return PTK_ERR_ARG;

    GemmPlan p{};
    int rc;
    // A: logical [M][K]
    if (!d.a.mn_major)
        rc = encode_operand(&p.tmA, d.a, d.k, d.m, kBM, b1, b2);
    else
        rc = encode_operand(&p.tmA, d.a, d.m, d.k, kBK, b1, b2);
    if (rc != PTK_OK) return rc;
    // B: logical [N][K]; with multicast / CTA pairs each CTA fetches half the K-major rows
    const bool pair = d.causal == PTK_CAUSAL_NONE && bn == 256 && tiles_m >= 2 && d.multicast == 2;
    const bool mc_pre = !pair && d.causal == PTK_CAUSAL_NONE && bn == 256 && tiles_m >= 2 && d.multicast == 1 &&
                        !d.b.mn_major;
    if (!d.b.mn_major)
        rc = encode_operand(&p.tmB, d.b, d.k, d.n, (mc_pre || pair) ? bn / 2 : bn, b1, b2);
    else
        rc = encode_operand(&p.tmB, d.b, d.n, d.k, kBK, b1, b2);
    if (rc != PTK_OK) return rc;
    if (pair && !d.b.mn_major) {
        rc = encode_operand(&p.tmB2, d.b, d.k, d.n, 64, b1, b2);  // tail halves: 64 B rows per CTA
        if (rc != PTK_OK) return rc;
    } else {
        p.tmB2 = p.tmB;
    }
    p.tmA2 = p.tmA;
    p.tmB2s = p.tmB;
    if (d.k2 > 0) {  // the second K segment's operands (same majors and boxes)
        rc = !d.a2.mn_major ? encode_operand(&p.tmA2, d.a2, d.k2, d.m, kBM, 1, 1)
                            : encode_operand(&p.tmA2, d.a2, d.m, d.k2, kBK, 1, 1);
        if (rc != PTK_OK) return rc;
        rc = !d.b2.mn_major ? encode_operand(&p.tmB2s, d.b2, d.k2, d.n, bn / 2, 1, 1)
                            : encode_operand(&p.tmB2s, d.b2, d.n, d.k2, kBK, 1, 1);
        if (rc != PTK_OK) return rc;
    }

    // CTA-pair kernel with MN-major operands: one 5-D box per operand and stage instead of two
    // 64-wide boxes (the both-MN weight-gradient layout issued twice the TMA loads for the same bytes)
    static const bool mn5_on = [] {
        const char* e = std::getenv("PTK_GEMM_MN5");
        return e == nullptr || e[0] != '0';
    }();
    int mn5_a = 0, mn5_b = 0;
    if (pair && mn5_on && d.a.mn_major && d.m % 64 == 0 && (d.k2 <= 0 || d.a2.mn_major)) {
        CUtensorMap ta = p.tmA, ta2 = p.tmA2;
        rc = encode_operand_mn5(&ta, d.a, d.m, d.k, kBK, 2, b1, b2);
        if (rc == PTK_OK && d.k2 > 0) rc = encode_operand_mn5(&ta2, d.a2, d.m, d.k2, kBK, 2, 1, 1);
        if (rc == PTK_OK) {
            p.tmA = ta;
            p.tmA2 = d.k2 > 0 ? ta2 : ta;
            mn5_a = 1;
        }
    }
    if (pair && mn5_on && d.b.mn_major && d.n % 64 == 0 && (d.k2 <= 0 || (d.b2.mn_major && d.n % 256 == 0))) {
        CUtensorMap tb = p.tmB, tb2 = p.tmB2, tbs = p.tmB2s;
        rc = encode_operand_mn5(&tb, d.b, d.n, d.k, kBK, 2, b1, b2);
        if (rc == PTK_OK) rc = encode_operand_mn5(&tb2, d.b, d.n, d.k, kBK, 1, b1, b2);  // tail halves
        if (rc == PTK_OK && d.k2 > 0) rc = encode_operand_mn5(&tbs, d.b2, d.n, d.k2, kBK, 2, 1, 1);
        if (rc == PTK_OK) {
            p.tmB = tb;
            p.tmB2 = tb2;
            p.tmB2s = d.k2 > 0 ? tbs : tb;
            mn5_b = 1;
        }
    }

    // the same for the 1-CTA kernels (A: two atoms; B: BN/64 atoms; the multicast kernel's B is K-major)
    if (!pair && mn5_on && d.causal == PTK_CAUSAL_NONE && d.k2 <= 0) {
        if (d.a.mn_major && d.m % 64 == 0) {
            CUtensorMap ta = p.tmA;
            if (encode_operand_mn5(&ta, d.a, d.m, d.k, kBK, kBM / 64, b1, b2) == PTK_OK) {
                p.tmA = p.tmA2 = ta;
                mn5_a = 1;
            }
        }
        if (d.b.mn_major && !mc_pre && d.n % 64 == 0) {
            CUtensorMap tb = p.tmB;
            if (encode_operand_mn5(&tb, d.b, d.n, d.k, kBK, bn / 64, b1, b2) == PTK_OK) {
                p.tmB = p.tmB2 = p.tmB2s = tb;
                mn5_b = 1;
            }
        }
    }

    GemmArgs& a = p.args;
    a.mn5_a = mn5_a;
    a.mn5_b = mn5_b;
    a.M = d.m;
    a.N = d.n;
    a.K = d.k + (d.k2 > 0 ? d.k2 : 0);
    a.kb_split = d.k2 > 0 ? d.k / kBK : 0;
    a.batch1 = b1;
    a.bn = bn;
    a.tiles_m = tiles_m;
    a.tiles_n = (d.n + bn - 1) / bn;
    a.tiles_per_batch = d.causal == PTK_CAUSAL_TILES ? tiles_m * (tiles_m + 1) / 2 : a.tiles_m * a.tiles_n;
    a.num_tiles = a.tiles_per_batch * b1 * b2;
    a.causal = d.causal;
    a.epi = d.epilogue;
    a.C = d.c.ptr;
    a.ldc = d.c.ld;
    a.c_bs1 = d.c.batch_stride[0];
    a.c_bs2 = d.c.batch_stride[1];
    a.C2 = d.c2;
    a.aux = d.aux.ptr;
    a.ld_aux = d.aux.ld;
    a.aux_bs1 = d.aux.batch_stride[0];
    a.aux_bs2 = d.aux.batch_stride[1];
    a.bias = d.bias;
    if ((a.epi == PTK_EPI_DGELU && a.aux == nullptr) || (a.epi == PTK_EPI_BIAS_GELU && (a.C2 == nullptr)))
        return PTK_ERR_ARG;
    a.col_part = d.col_part;
    if (a.col_part != nullptr && (b1 * b2 != 1 || a.epi == PTK_EPI_F32 || a.epi == PTK_EPI_ACC_F32 ||
                                  d.causal != PTK_CAUSAL_NONE))
        return PTK_ERR_ARG;  // column partials: dense, unbatched, bf16 output only
    {  // TMA-store epilogue when the output layout allows it (16-byte aligned rows and batches)
        const bool f32 = a.epi == PTK_EPI_F32 || a.epi == PTK_EPI_ACC_F32;
        bool ok = encode_output(&p.tmC, a.C, a.ldc, a.c_bs1, a.c_bs2, d.m, d.n, b1, b2, f32) == PTK_OK;
        if (ok && a.epi == PTK_EPI_BIAS_GELU)
            ok = encode_output(&p.tmC2, a.C2, a.ldc, a.c_bs1, a.c_bs2, d.m, d.n, b1, b2, false) == PTK_OK;
        if (!ok) return PTK_ERR_ALIGN;  // outputs leave through TMA: 16-byte aligned rows and batches
        a.tma_store = 1;
    }

    // Raster order: the ~150 concurrent tiles share the operand block of the
    // fastest-varying index's partner through L2.  m-fastest streams B once but
    // re-reads A once per n-tile column unless A stays L2-resident; n-fastest is
    // the mirror image.  Pick the order with less HBM operand traffic (the
    // vocabulary-head weight gradient: A = dlogits^T, 206 MB, 8 n-tiles).
    if (b1 * b2 == 1 && d.causal == PTK_CAUSAL_NONE) {
        const double l2 = 60e6;  // bytes of operand that stay resident in the 126 MB L2 under streaming
        const double kt = static_cast<double>(d.k) + (d.k2 > 0 ? d.k2 : 0);  // both K segments
        const double ab = 2.0 * d.m * kt, bb = 2.0 * d.n * kt;
        const double m_fast = (ab <= l2 ? ab : ab * a.tiles_n) + bb;
        const double n_fast = (bb <= l2 ? bb : bb * ((tiles_m + 1) / 2)) + ab;
        a.n_fast = n_fast < 0.8 * m_fast ? 1 : 0;
    }
    const int sms = num_sms();
    // B-tile multicast across a 2-CTA cluster halves the L2 -> SM operand
    // traffic per FLOP (dense, non-causal GEMMs with at least two m-tiles).
    const bool mc = mc_pre;
    p.flops = 2.0 * d.m * static_cast<double>(d.n) * a.K * b1 * b2;
    if (d.causal != PTK_CAUSAL_NONE) p.flops *= 0.5;
    a.full_tiles = 1 << 30;
    if (pair) {
        a.tiles_per_batch = ((tiles_m + 1) / 2) * a.tiles_n;
        const int tiles = a.tiles_per_batch * b1 * b2;
        const int pairs = sms / 2;
        a.num_tiles = tiles;
        a.full_tiles = tiles;
        const int rem = tiles % pairs;
        if (tiles > pairs && rem > 0 && 2 * rem <= pairs && d.n % 256 == 0 && d.k2 <= 0) {
            // split the partial last wave into 256 x 128 halves: it then takes half as long
            a.full_tiles = tiles - rem;
            a.num_tiles = a.full_tiles + 2 * rem;
        }
        const int clusters = a.num_tiles < pairs ? a.num_tiles : pairs;
        p.grid = 2 * clusters;
        p.launch = pick_2sm(d.a.mn_major, d.b.mn_major);
    } else if (mc) {
        a.tiles_per_batch = ((tiles_m + 1) / 2) * a.tiles_n;
        a.num_tiles = a.tiles_per_batch * b1 * b2;
        const int clusters = a.num_tiles < sms / 2 ? a.num_tiles : sms / 2;
        p.grid = 2 * clusters;
        p.launch = pick<256, true>(d.a.mn_major, d.b.mn_major);
    } else {
        p.grid = a.num_tiles < sms ? a.num_tiles : sms;
        switch (bn) {
            case 64: p.launch = pick<64, false>(d.a.mn_major, d.b.mn_major); break;
            case 128: p.launch = pick<128, false>(d.a.mn_major, d.b.mn_major); break;
            default: p.launch = pick<256, false>(d.a.mn_major, d.b.mn_major); break;
        }
    }
    p.multicast = mc || pair;
    *out = p;
    return PTK_OK;
}

int gemm_run(const GemmPlan& p, cudaStream_t stream) { return p.launch(p, stream); }

void preload_gemm_kernels() { preload_module_of(reinterpret_cast<const void*>(&gemm_bf16_2sm_kernel<false, false>)); }

}  // namespace ptk
