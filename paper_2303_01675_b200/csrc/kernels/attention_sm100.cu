// Fused attention forward for sm_100a (tcgen05 + TMEM + TMA), persistent.
//
// One CTA per SM walks a static list of (128-query block, head, sample)
// tiles, heaviest causal blocks first, assigned boustrophedon (CTA i takes
// tiles i, 2G-1-i, 2G+i, ...) so heavy and light blocks pair up.  The TMA,
// MMA and softmax roles each walk the same list, so loads and score
// products for the next tile run under the current tile's softmax/epilogue.
// For each 128-key block j of a tile:
//   S_j  = Q·K_jᵀ            tcgen05.mma into TMEM (double-buffered: S_{j+1} —
//                            possibly of the next tile — is issued while the
//                            softmax warps work on S_j)
//   P_j  = exp2(S_j·c − m)   8 softmax warps in two column halves: a thread owns
//                            64 columns of one query row; the two halves of a
//                            row swap their maxima through smem (one 64-thread
//                            named barrier per block), P is written to smem in
//                            the UMMA K-major 128B-swizzled layout
//   O   += P_j·V_j           tcgen05.mma into a TMEM accumulator (double-buffered
//                            across tiles); when the row max moves, the thread
//                            rescales its half of the O row in TMEM
// and finally O/l is written as bf16 [T, h] (the out-projection's input) and
// lse = m + log2(l) (log2 units of the scaled scores) for the backward.
// Warps: 0 TMA producer, 1 TMEM alloc + MMA issuer, 4-11 softmax/epilogue
// (warp 4+q and 8+q share TMEM lane quarter q: columns 0-63 and 64-127).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>

#include "../runtime/preload.h"
#include "attention_sm100.h"
#include "launch.cuh"
#include "sm100_ptx.cuh"
#include "../runtime/sm_budget.h"

namespace ptk {

using namespace sm100;

namespace {

constexpr int kBlk = 128;      // query rows and key rows per block
constexpr int kThreads = 384;  // backward: 12 warps: TMA, MMA, 2 idle, 8 row-parallel elementwise warps
constexpr int kFwdNQ = 2;      // forward: softmax rows split in kFwdNQ column parts (4 + 4·NQ warps)
constexpr float kLazyRescaleLog2 = 8.f;
#ifndef PTK_BW_POLY
#define PTK_BW_POLY 2
#endif
constexpr int kBwPoly = PTK_BW_POLY;  // backward: exponentials per 32 on the FMA pipe (0, 1, 2, 4 or 8)  // forward: move the running max only when it grows by > 2^8

int sm_count() { return sm_budget(); }  // runtime/sm_budget.h

template <int D>
struct FaCfg {
    static constexpr int kQBytes = kBlk * D * 2;     // [D/64][128 rows x 128 B]
    static constexpr int kKBytes = kBlk * D * 2;
    static constexpr int kVBytes = kBlk * D * 2;     // [2 kv halves][D/64][64 rows x 128 B]
    static constexpr int kPBytes = kBlk * kBlk * 2;  // [2][128 rows x 128 B]
    static constexpr int kQBuf = D == 64 ? 2 : 1;
    static constexpr int kStages = D == 64 ? 3 : 2;
    static constexpr int kXchg = (2 * 4 + 2 * 4) * kBlk * 4;  // row maxima [2][NQ<=4][128], row sums [2][NQ][128]
    static constexpr int kSmem =
        kQBuf * kQBytes + kStages * (kKBytes + kVBytes) + kPBytes + kXchg + 1024 + 256;
    static constexpr uint32_t kTmemS0 = 0, kTmemS1 = 128, kTmemO = 256;  // O buffers at 256, 256 + D
};

struct FaArgs {
    __nv_bfloat16* o;  // [b*s][h]
    float* lse;        // [b][H][s], log2 units of the scaled scores
    int s, H, h, b;
    float scale_log2;  // log2(e) / sqrt(d)
    int causal;        // 1: GPT (key <= query), 0: bidirectional (BERT)
};

// Position in a CTA's tile list: tile k of this CTA, key block j of that tile.
struct FaCursor {
    int k, qb, head, bi, nkv, j;
    bool valid;
};

__device__ __forceinline__ void fa_tile(const FaArgs& a, int k, FaCursor& c) {
    const int G = gridDim.x, i = blockIdx.x;
    const int nqb = a.s / kBlk;
    const int per = a.H * a.b;
    const int t = (k & 1) ? (k + 1) * G - 1 - i : k * G + i;
    c.k = k;
    c.j = 0;
    c.valid = t < nqb * per;
    const int rank = t / per, rem = t % per;
    c.qb = nqb - 1 - rank;  // heaviest first
    c.head = rem % a.H;
    c.bi = rem / a.H;
    c.nkv = a.causal ? c.qb + 1 : nqb;
}

#ifdef PTK_ATTN_TRACE
// Debug timeline of the forward kernel's CTA 0 (clock64): [role][key block][event].
__device__ unsigned long long g_fwd_trace[2][64][8];
#define FTRACE(role, step, ev)                                                  \
    do {                                                                        \
        if (blockIdx.x == 0 && (step) < 64) g_fwd_trace[role][step][ev] = clock64(); \
    } while (0)
// ping-pong forward: [0 lane A softmax, 1 lane B softmax, 2 MMA][lane block][event]
__device__ unsigned long long g_pp_trace[3][64][8];
__device__ unsigned long long g_pp_cta[160][4];  // per CTA: globaltimer at entry, first S issue, MMA done, exit
__device__ int g_pp_trace_cta = 0;              // the CTA whose timeline is recorded
#define PTRACE(role, step, ev)                                                  \
    do {                                                                        \
        if (ptrace_on && (step) < 64) g_pp_trace[role][step][ev] = clock64();   \
    } while (0)
#else
#define FTRACE(role, step, ev) \
    do {                       \
    } while (0)
#define PTRACE(role, step, ev) \
    do {                       \
    } while (0)
#endif

__device__ __forceinline__ void fa_next(const FaArgs& a, FaCursor& c) {
    if (++c.j == c.nkv) fa_tile(a, c.k + 1, c);
}

template <int D, int NQ>
__global__ void __launch_bounds__(32 * (4 + 4 * NQ), 1)
    flash_fwd_kernel(const __grid_constant__ CUtensorMap tmQK, const __grid_constant__ CUtensorMap tmV,
                     const __grid_constant__ FaArgs a) {
    using C = FaCfg<D>;
    constexpr int S = C::kStages, QB = C::kQBuf;
    constexpr uint32_t kIdescS = make_idesc_bf16(kBlk, kBlk, false, false);  // Q (K-major) x K (K-major)
    constexpr uint32_t kIdescO = make_idesc_bf16(kBlk, D, false, true);      // P (K-major) x V (MN-major)

    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;                         // [QB]
    uint8_t* sK = sQ + QB * C::kQBytes;         // [S]
    uint8_t* sV = sK + S * C::kKBytes;          // [S]
    uint8_t* sP = sV + S * C::kVBytes;
    float* sX = reinterpret_cast<float*>(sP + C::kPBytes);  // row-max [2][2][128], row-sum [2][2][128]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sP + C::kPBytes + C::kXchg);
    uint64_t* q_full = bars + 0;         // [2]
    uint64_t* q_empty = bars + 2;        // [2]
    uint64_t* kv_full = bars + 4;        // [S <= 3]
    uint64_t* kv_empty = bars + 7;       // [S]
    uint64_t* s_full = bars + 10;        // [2]
    uint64_t* s_empty = bars + 12;       // [2]
    uint64_t* p_full = bars + 14;
    uint64_t* pv_done = bars + 15;
    uint64_t* o_full = bars + 16;        // [2]
    uint64_t* o_empty = bars + 18;       // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 20);

    const int warp = threadIdx.x / 32;
    const uint32_t lane = lane_id();

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmQK);
        tma_prefetch_desc(&tmV);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&q_full[i], 1);
            mbar_init(&q_empty[i], 1);
            mbar_init(&s_full[i], 1);
            mbar_init(&s_empty[i], 4 * NQ);
            mbar_init(&o_full[i], 1);
            mbar_init(&o_empty[i], 4 * NQ);
        }
        for (int i = 0; i < S; ++i) {
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], 1);
        }
        mbar_init(p_full, 4 * NQ);
        mbar_init(pv_done, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_begin();  // previous kernel complete: its outputs (qkv, lse, dO, ...) are visible

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer
            int n = 0;  // key blocks loaded so far (all tiles)
            FaCursor c;
            for (fa_tile(a, 0, c); c.valid; fa_tile(a, c.k + 1, c)) {
                const int qbuf = c.k % QB;
                mbar_wait(&q_empty[qbuf], ((c.k / QB) & 1) ^ 1);
                mbar_arrive_expect_tx(&q_full[qbuf], C::kQBytes);
#pragma unroll
                for (int kb = 0; kb < D / 64; ++kb)
                    tma_load_4d(&tmQK, &q_full[qbuf], sQ + qbuf * C::kQBytes + kb * kBlk * 128, kb * 64, c.qb * kBlk,
                                c.head, c.bi);
                for (int j = 0; j < c.nkv; ++j, ++n) {
                    const int st = n % S;
                    mbar_wait(&kv_empty[st], ((n / S) & 1) ^ 1);
                    mbar_arrive_expect_tx(&kv_full[st], C::kKBytes + C::kVBytes);
                    uint8_t* k = sK + st * C::kKBytes;
                    uint8_t* v = sV + st * C::kVBytes;
#pragma unroll
                    for (int kb = 0; kb < D / 64; ++kb)
                        tma_load_4d(&tmQK, &kv_full[st], k + kb * kBlk * 128, kb * 64, j * kBlk, a.H + c.head, c.bi);
#pragma unroll
                    for (int half = 0; half < 2; ++half)
#pragma unroll
                        for (int na = 0; na < D / 64; ++na)
                            tma_load_4d(&tmV, &kv_full[st], v + (half * (D / 64) + na) * 8192, na * 64,
                                        j * kBlk + half * 64, 2 * a.H + c.head, c.bi);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---------------- MMA issuer
            auto issue_s = [&](const FaCursor& c, int n) {
                const int st = n % S, sb = n & 1, qbuf = c.k % QB;
                if (c.j == 0) mbar_wait(&q_full[qbuf], (c.k / QB) & 1);
                mbar_wait(&kv_full[st], (n / S) & 1);
                mbar_wait(&s_empty[sb], ((n >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t q_base = smem_u32(sQ + qbuf * C::kQBytes);
                const uint32_t k_base = smem_u32(sK + st * C::kKBytes);
                const uint32_t d_tmem = tmem + (sb ? C::kTmemS1 : C::kTmemS0);
#pragma unroll
                for (int k = 0; k < D / 16; ++k) {
                    const uint32_t off = (k / 4) * kBlk * 128 + (k % 4) * 32;
                    mma_bf16_ss(d_tmem, make_sw128_desc(q_base + off, 16, 1024), make_sw128_desc(k_base + off, 16, 1024),
                                kIdescS, k > 0 ? 1u : 0u);
                }
                mma_commit(&s_full[sb]);
                FTRACE(1, n, 0);
                if (c.j == c.nkv - 1) mma_commit(&q_empty[qbuf]);
            };
            FaCursor cs, cp;
            fa_tile(a, 0, cs);
            fa_tile(a, 0, cp);
            int ns = 0, np = 0;
            if (cs.valid) {
                issue_s(cs, ns++);
                fa_next(a, cs);
            }
            while (cp.valid) {
                if (cs.valid) {  // one score product ahead, across tile boundaries
                    issue_s(cs, ns++);
                    fa_next(a, cs);
                }
                const int st = np % S, ob = cp.k & 1;
                mbar_wait(p_full, np & 1);
                FTRACE(1, np, 1);
                if (cp.j == 0) mbar_wait(&o_empty[ob], ((cp.k >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t p_base = smem_u32(sP);
                const uint32_t v_base = smem_u32(sV + st * C::kVBytes);
                const uint32_t o_tmem = tmem + C::kTmemO + ob * D;
#pragma unroll
                for (int k = 0; k < kBlk / 16; ++k) {
                    const uint32_t pa = p_base + (k / 4) * kBlk * 128 + (k % 4) * 32;
                    const uint32_t vb = v_base + (k / 4) * (D / 64) * 8192 + (k % 4) * 2048;
                    mma_bf16_ss(o_tmem, make_sw128_desc(pa, 16, 1024), make_sw128_desc(vb, 8192, 1024), kIdescO,
                                (cp.j > 0 || k > 0) ? 1u : 0u);
                }
                mma_commit(pv_done);
                FTRACE(1, np, 2);
                mma_commit(&kv_empty[st]);
                if (cp.j == cp.nkv - 1) mma_commit(&o_full[ob]);
                fa_next(a, cp);
                ++np;
            }
        }
    } else if (warp >= 4) {  // ---------------- softmax / epilogue: thread = (query row, column part)
        const int quad = warp & 3;
        const int part = (warp - 4) >> 2;  // columns [kHc*part, +kHc) of S, [kOc*part, +kOc) of O
        const int r = quad * 32 + static_cast<int>(lane);
        const uint32_t lane_base = static_cast<uint32_t>(quad * 32) << 16;
        constexpr int kHc = kBlk / NQ;  // S columns per thread
        constexpr int kOc = D / NQ;     // O columns per thread
        const uint32_t xbase = smem_u32(sX);
        int n = 0;  // key blocks processed so far (all tiles)
        FaCursor c;
        // O columns [col, col + kOc) of this thread's row scaled by `scale` (TMEM read-modify-write)
        auto scale_o = [&](uint32_t col, float scale) {
#pragma unroll
            for (int cc = 0; cc < kOc; cc += 16) {
                float v[16];
                tmem_ld_32x32b_x16(col + cc, v);
#pragma unroll
                for (int e = 0; e < 16; ++e) v[e] *= scale;
                tmem_st_32x32b_x16(col + cc, v);
            }
        };
        for (fa_tile(a, 0, c); c.valid; fa_tile(a, c.k + 1, c)) {
            const int ob = c.k & 1;
            const uint32_t o_cols = tmem + lane_base + C::kTmemO + ob * D + part * kOc;
            float m = -INFINITY, l = 0.f;  // m in log2 units of the scaled scores; l = this part's row sum
            for (int j = 0; j < c.nkv; ++j, ++n) {
                const int sb = n & 1;
                mbar_wait(&s_full[sb], (n >> 1) & 1);
                if (warp == 4 && lane == 0) FTRACE(0, n, 0);
                tc_fence_after();
                float x[kHc];
#pragma unroll
                for (int cc = 0; cc < kHc / 32; ++cc)
                    tmem_ld_32x32b_x32_nw(tmem + lane_base + (sb ? C::kTmemS1 : C::kTmemS0) + part * kHc + cc * 32,
                                          x + cc * 32);
                tmem_ld_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&s_empty[sb]);
                if (warp == 4 && lane == 0) FTRACE(0, n, 1);
                // 8 independent max / sum chains (a single chain serialises on the ALU/MUFU latency)
                float mr8[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) mr8[i] = -INFINITY;
                const bool diag = a.causal && j == c.qb;
                if (diag) {  // diagonal block: key > query masked
#pragma unroll
                    for (int e = 0; e < kHc; ++e) {
                        if (part * kHc + e > r) x[e] = -INFINITY;
                        mr8[e & 7] = fmaxf(mr8[e & 7], x[e]);
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < kHc; ++e) mr8[e & 7] = fmaxf(mr8[e & 7], x[e]);
                }
                const float mraw = fmaxf(fmaxf(fmaxf(mr8[0], mr8[1]), fmaxf(mr8[2], mr8[3])),
                                         fmaxf(fmaxf(mr8[4], mr8[5]), fmaxf(mr8[6], mr8[7])));
                // swap the part maxima with the NQ-1 partner warps (same rows, other columns)
                const uint32_t xb = xbase + (n & 1) * NQ * kBlk * 4;
                sts32f(xb + (part * kBlk + r) * 4, mraw);
                asm volatile("bar.sync %0, %1;" ::"r"(2 + quad), "r"(32 * NQ) : "memory");
                if (warp == 4 && lane == 0) FTRACE(0, n, 2);
                float pm = lds32f(xb + r * 4);
#pragma unroll
                for (int q = 1; q < NQ; ++q) pm = fmaxf(pm, lds32f(xb + (q * kBlk + r) * 4));
                // lazy rescaling: the running max m only moves when the block max exceeds it by more
                // than 2^8 (P <= 256 stays exact enough in bf16, l and O share the same stale m), so
                // the O rescale (a TMEM read-modify-write on the P -> PV critical path) is rare
                const float pmx = pm * a.scale_log2;
                const float mx = pmx > m + kLazyRescaleLog2 ? pmx : m;
                const float alpha = ex2(m - mx);  // m = -inf on the first block -> 0
                float s8[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) s8[i] = 0.f;
                if (diag) {  // masked (-inf) entries: MUFU ex2 only
#pragma unroll
                    for (int e = 0; e < kHc; ++e) {
                        x[e] = ex2(fmaf(x[e], a.scale_log2, -mx));
                        s8[e & 7] += x[e];
                    }
                } else {
                    // packed fp32x2 scale-and-subtract and sums (FFMA2 / FADD2; same per-lane
                    // operations and the same 8 sum chains, so bit-identical to the scalar form)
                    const float2 sc2 = make_float2(a.scale_log2, a.scale_log2), mm2 = make_float2(-mx, -mx);
                    float2* s2 = reinterpret_cast<float2*>(s8);
#pragma unroll
                    for (int e = 0; e < kHc; e += 2) {
                        const float2 t = __ffma2_rn(make_float2(x[e], x[e + 1]), sc2, mm2);
                        x[e] = ex2(t.x);
                        x[e + 1] = ex2(t.y);
                        s2[(e >> 1) & 3] = __fadd2_rn(s2[(e >> 1) & 3], make_float2(x[e], x[e + 1]));
                    }
                }
                const float sum = ((s8[0] + s8[1]) + (s8[2] + s8[3])) + ((s8[4] + s8[5]) + (s8[6] + s8[7]));
                l = l * alpha + sum;
                m = mx;
                if (warp == 4 && lane == 0) FTRACE(0, n, 3);
                if (n > 0) {
                    mbar_wait(pv_done, (n - 1) & 1);  // P buffer free (and O of this tile stable)
                    tc_fence_after();
                }
                if (warp == 4 && lane == 0) FTRACE(0, n, 4);
                // P row part -> smem, K-major 128B-swizzled (16-byte chunk index ^= row % 8)
#pragma unroll
                for (int q = 0; q < kHc / 8; ++q) {
                    const int col = part * kHc + q * 8;
                    uint4 u;
                    u.x = pack_bf16(x[q * 8 + 0], x[q * 8 + 1]);
                    u.y = pack_bf16(x[q * 8 + 2], x[q * 8 + 3]);
                    u.z = pack_bf16(x[q * 8 + 4], x[q * 8 + 5]);
                    u.w = pack_bf16(x[q * 8 + 6], x[q * 8 + 7]);
                    sts128(smem_u32(sP) + (col >> 6) * (kBlk * 128) + r * 128 + ((((col & 63) >> 3) ^ (r & 7)) * 16),
                           u);
                }
                if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) scale_o(o_cols, alpha);
                fence_proxy_async_smem();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(p_full);
                if (warp == 4 && lane == 0) FTRACE(0, n, 5);
            }
            // total row sum = all parts (same m sequence, so the partial sums add; fixed order)
            const uint32_t lb = xbase + (2 * NQ * kBlk + (c.k & 1) * NQ * kBlk) * 4;
            sts32f(lb + (part * kBlk + r) * 4, l);
            asm volatile("bar.sync %0, %1;" ::"r"(2 + quad), "r"(32 * NQ) : "memory");
            float lt = 0.f;
#pragma unroll
            for (int q = 0; q < NQ; ++q) lt += lds32f(lb + (q * kBlk + r) * 4);
            mbar_wait(&o_full[ob], (c.k >> 1) & 1);
            tc_fence_after();
            const float inv = 1.f / lt;
            const int q = c.qb * kBlk + r;
            __nv_bfloat16* orow = a.o + (static_cast<int64_t>(c.bi) * a.s + q) * a.h + c.head * D + part * kOc;
#pragma unroll
            for (int cc = 0; cc < kOc; cc += 16) {
                float v[16];
                tmem_ld_32x32b_x16(o_cols + cc, v);
#pragma unroll
                for (int g = 0; g < 2; ++g) {
                    uint4 u;
                    u.x = pack_bf16(v[g * 8 + 0] * inv, v[g * 8 + 1] * inv);
                    u.y = pack_bf16(v[g * 8 + 2] * inv, v[g * 8 + 3] * inv);
                    u.z = pack_bf16(v[g * 8 + 4] * inv, v[g * 8 + 5] * inv);
                    u.w = pack_bf16(v[g * 8 + 6] * inv, v[g * 8 + 7] * inv);
                    *reinterpret_cast<uint4*>(orow + cc + g * 8) = u;
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&o_empty[ob]);
            if (part == 0) a.lse[(static_cast<int64_t>(c.bi) * a.H + c.head) * a.s + q] = m + __log2f(lt);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

// ============================================================================
// Forward, d = 64, two-tile ping-pong (the default for GPT-1.3B / BERT-large).
//
// The single-tile kernel above is bound by its softmax phase (MUFU ex2 plus
// the non-exponential work of the same warps, all phase-locked on one S
// buffer and one P buffer).  Here a CTA works on a PAIR of 128-query tiles of
// one (head, sample) — lane A = query block 2p, lane B = 2p+1 — which share
// every K/V block.  Each lane has its own S, P (bf16, the TMEM A operand of
// P·V) and O in TMEM, and four softmax warps with ONE THREAD PER QUERY ROW (all
// 128 columns of the row in registers: the row max needs no cross-warp
// exchange).  The MMA warp keeps each lane one score product ahead (S_L(j+1)
// is issued as soon as lane L has read S_L(j) into registers) and issues
// PV_L(j) when lane L's P is in TMEM, lanes in a fixed A-then-B order so their
// exponential passes stay offset: while one lane's warps do their
// non-exponential work (TMEM loads, max, P stores, O rescale) the other lane's
// exponentials keep the MUFU busy.  O leaves through per-lane smem staging and
// a TMA store.
// ============================================================================
struct Fa2Cfg {
    static constexpr int D = 64;
    static constexpr int kQBytes = kBlk * D * 2;     // 16 KiB, K-major sw128
    static constexpr int kKVBytes = 2 * kBlk * D * 2;  // K then V
    static constexpr int kStages = 4;
    static constexpr int kOBytes = kBlk * D * 2;  // per lane: the O tile staged for its TMA store
    static constexpr int kSmem = 4 * kQBytes + kStages * kKVBytes + 2 * kOBytes + 1024 + 768;
    // TMEM: S_L at 128 L (fp32 128x128); P_L at 256 + 64 L (bf16x2-packed 128x128, the A operand of
    // P·V read straight from TMEM); O_L at 384 + 64 L (fp32 128x64)
    static constexpr uint32_t kTmemS = 0, kTmemP = 256, kTmemO = 384;
};
static_assert(Fa2Cfg::kSmem <= 232448, "ping-pong forward smem");


constexpr int kFa2MaxItems = 24;  // pair items per CTA (launch_fwd_pp enforces it)

// Pair cursor: item k of this CTA -> (pair p, head, sample); lane L's tile is query block 2p + L.
struct Fa2Item {
    int p, head, bi;
    bool valid;
};

__device__ __forceinline__ Fa2Item fa2_item(const FaArgs& a, int k) {
    const int G = gridDim.x, i = blockIdx.x;
    const int npair = a.s / (2 * kBlk);
    const int per = a.H * a.b;
    const int t = (k & 1) ? (k + 1) * G - 1 - i : k * G + i;
    Fa2Item it;
    it.valid = t < npair * per;
    const int rank = t / per, rem = t % per;
    it.p = npair - 1 - rank;  // heaviest first
    it.head = rem % a.H;
    it.bi = rem / a.H;
    return it;
}

__device__ __forceinline__ int fa2_nkv(const FaArgs& a, int p, int lane) {
    return a.causal ? 2 * p + lane + 1 : a.s / kBlk;
}

// kFwdPoly: of every 16 unmasked exponentials, this many on the FMA pipe (ex2_poly) instead of MUFU
template <int kFwdPoly>
__global__ void __launch_bounds__(384, 1)
    flash_fwd_pp_kernel(const __grid_constant__ CUtensorMap tmQK, const __grid_constant__ CUtensorMap tmV,
                        const __grid_constant__ CUtensorMap tmO, const __grid_constant__ FaArgs a) {
    using C = Fa2Cfg;
    constexpr int D = C::D, NS = C::kStages;
    constexpr uint32_t kIdescS = make_idesc_bf16(kBlk, kBlk, false, false);
    constexpr uint32_t kIdescO = make_idesc_bf16(kBlk, D, false, true);

    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;                        // [lane][qbuf] 16 KiB each
    uint8_t* sKV = sQ + 4 * C::kQBytes;        // [stage] K 16 KiB, V 16 KiB
    uint8_t* sO = sKV + NS * C::kKVBytes;      // [lane] O staging, 128B-swizzled [128 rows][64 cols]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sO + 2 * C::kOBytes);
    uint64_t* q_full = bars + 0;     // [lane][qbuf]
    uint64_t* q_empty = bars + 4;    // [lane][qbuf]
    uint64_t* kv_full = bars + 8;    // [NS]
    uint64_t* kv_empty = bars + 12;  // [NS]
    uint64_t* s_full = bars + 16;    // [lane]
    uint64_t* s_empty = bars + 18;   // [lane]
    uint64_t* p_full = bars + 20;    // [lane]
    uint64_t* pv_done = bars + 22;   // [lane]
    uint64_t* o_full = bars + 24;    // [lane]
    uint64_t* o_empty = bars + 28;   // [lane]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 32);
    // this CTA's pair items, decoded once (the role loops never divide: integer division runs on
    // the MUFU, which the softmax warps saturate)
    int4* items = reinterpret_cast<int4*>(bars + 34);  // {p, head, bi, kvbase}
    int* n_items = reinterpret_cast<int*>(bars + 34 + 2 * kFa2MaxItems);

    const int warp = threadIdx.x / 32;
    const uint32_t lane_id_ = lane_id();
#ifdef PTK_ATTN_TRACE
    const bool ptrace_on = static_cast<int>(blockIdx.x) == *static_cast<volatile int*>(&g_pp_trace_cta);
    auto gt = [] {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        return t;
    };
    if (threadIdx.x == 0 && blockIdx.x < 160) g_pp_cta[blockIdx.x][0] = gt();
#endif

    if (warp == 0 && lane_id_ == 0) {
        tma_prefetch_desc(&tmQK);
        tma_prefetch_desc(&tmV);
        for (int i = 0; i < 4; ++i) {
            mbar_init(&q_full[i], 1);
            mbar_init(&q_empty[i], 1);
            mbar_init(&o_full[i], 1);
            mbar_init(&o_empty[i], 4);
        }
        for (int i = 0; i < NS; ++i) {
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], 1);
        }
        for (int l = 0; l < 2; ++l) {
            mbar_init(&s_full[l], 1);
            mbar_init(&s_empty[l], 4);
            mbar_init(&p_full[l], 4);
            mbar_init(&pv_done[l], 1);
        }
        fence_barrier_init();
        int kvb = 0, n = 0;
        for (; n < kFa2MaxItems; ++n) {
            const Fa2Item it = fa2_item(a, n);
            if (!it.valid) break;
            items[n] = make_int4(it.p, it.head, it.bi, kvb);
            kvb += fa2_nkv(a, it.p, 1);
        }
        *n_items = n;
    }
    if (warp == 1) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_begin();
    // registers: 3 warps per SM sub-partition at 168 each at launch; the producer / MMA warpgroup
    // (warps 0-3) gives its share to the softmax warpgroups (a thread holds a 128-column row)

    if (warp == 0) {
        reg_dealloc<72>();
        if (lane_id_ == 0) {  // ---------------- TMA producer
            int n = 0;
            const int nit = *n_items;
            for (int k = 0; k < nit; ++k) {
                const int4 itv = items[k];
                const Fa2Item it{itv.x, itv.y, itv.z, true};
                const int qbuf = k & 1;
                for (int l = 0; l < 2; ++l) {
                    mbar_wait(&q_empty[l * 2 + qbuf], ((k >> 1) & 1) ^ 1);
                    mbar_arrive_expect_tx(&q_full[l * 2 + qbuf], C::kQBytes);
                    tma_load_4d(&tmQK, &q_full[l * 2 + qbuf], sQ + (l * 2 + qbuf) * C::kQBytes, 0,
                                (2 * it.p + l) * kBlk, it.head, it.bi);
                }
                const int nkv = fa2_nkv(a, it.p, 1);
                for (int j = 0; j < nkv; ++j, ++n) {
                    const int st = n % NS;
                    mbar_wait(&kv_empty[st], ((n / NS) & 1) ^ 1);
                    mbar_arrive_expect_tx(&kv_full[st], C::kKVBytes);
                    uint8_t* kk = sKV + st * C::kKVBytes;
                    uint8_t* vv = kk + kBlk * D * 2;
                    tma_load_4d(&tmQK, &kv_full[st], kk, 0, j * kBlk, a.H + it.head, it.bi);
                    // V [128 keys][64] in one box: the same rows two 64-row boxes would place
                    tma_load_4d(&tmQK, &kv_full[st], vv, 0, j * kBlk, 2 * a.H + it.head, it.bi);
                }
            }
        }
    } else if (warp == 1) {
        reg_dealloc<72>();
        if (lane_id_ == 0) {  // ---------------- MMA issuer
            // Per lane: the block stream (item k, key block j) over all items; the KV stage of a
            // block is the producer's running block counter.  S is issued one block ahead of PV.
            struct LaneCur {
                int k, j, n, nkv, kvbase;  // n = blocks of this lane so far; kvbase = KV counter at item start
                bool valid;
            };
            const int nit = *n_items;
            auto lane_start = [&](LaneCur& c, int l, int k, int) {
                c.k = k;
                c.j = 0;
                c.valid = k < nit;
                const int4 itv = c.valid ? items[k] : make_int4(0, 0, 0, 0);
                c.nkv = c.valid ? fa2_nkv(a, itv.x, l) : 0;
                c.kvbase = itv.w;
            };
            // KV users of the current item's stages: 2 where both lanes use the block, else 1
            uint8_t kv_users[NS];
            for (int i = 0; i < NS; ++i) kv_users[i] = 0;
            LaneCur cs[2], cp[2];  // S-issue and PV-issue cursors per lane
            for (int l = 0; l < 2; ++l) {
                lane_start(cs[l], l, 0, 0);
                cs[l].n = 0;
                lane_start(cp[l], l, 0, 0);
                cp[l].n = 0;
            }
            auto advance = [&](LaneCur& c, int l) {
                ++c.n;
                if (++c.j == c.nkv) {
                    const int n = c.n;
                    lane_start(c, l, c.k + 1, 0);
                    c.n = n;
                }
            };
            auto issue_s = [&](int l) {
                LaneCur& c = cs[l];
                const int st = (c.kvbase + c.j) % NS, qbuf = c.k & 1;
                if (c.j == 0) mbar_wait(&q_full[l * 2 + qbuf], (c.k >> 1) & 1);
                mbar_wait(&kv_full[st], ((c.kvbase + c.j) / NS) & 1);
                mbar_wait(&s_empty[l], (c.n & 1) ^ 1);
                tc_fence_after();
                const uint32_t q_base = smem_u32(sQ + (l * 2 + qbuf) * C::kQBytes);
                const uint32_t k_base = smem_u32(sKV + st * C::kKVBytes);
                const uint32_t d_tmem = tmem + C::kTmemS + 128 * l;
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk)
                    mma_bf16_ss(d_tmem, make_sw128_desc(q_base + kk * 32, 16, 1024),
                                make_sw128_desc(k_base + kk * 32, 16, 1024), kIdescS, kk > 0 ? 1u : 0u);
                mma_commit(&s_full[l]);
                PTRACE(2, c.n, l * 4 + 0);
                if (c.j == c.nkv - 1) mma_commit(&q_empty[l * 2 + qbuf]);
                advance(c, l);
            };
            auto issue_pv = [&](int l) {
                LaneCur& c = cp[l];
                const int g = c.kvbase + c.j, st = g % NS;
                mbar_wait(&p_full[l], c.n & 1);
                PTRACE(2, c.n, l * 4 + 1);
                // single O buffer per lane: the epilogue of the previous pair always read it before
                // the same warps produced this pair's first P, so this wait never stalls
                if (c.j == 0) mbar_wait(&o_empty[l], (c.k & 1) ^ 1);
                tc_fence_after();
                const uint32_t p_tmem = tmem + C::kTmemP + 64 * l;
                const uint32_t v_base = smem_u32(sKV + st * C::kKVBytes + kBlk * D * 2);
                const uint32_t o_tmem = tmem + C::kTmemO + 64 * l;
#pragma unroll
                for (int kk = 0; kk < kBlk / 16; ++kk) {
                    const uint32_t vb = v_base + (kk / 4) * 8192 + (kk % 4) * 2048;
                    mma_bf16_ts(o_tmem, p_tmem + kk * 8, make_sw128_desc(vb, 8192, 1024), kIdescO,
                                (c.j > 0 || kk > 0) ? 1u : 0u);
                }
                mma_commit(&pv_done[l]);
                PTRACE(2, c.n, l * 4 + 2);
                // the KV stage is free once every lane that uses this block has issued its PV
                if (kv_users[st] == 0) kv_users[st] = (c.j < fa2_nkv(a, items[c.k].x, 0)) ? 2 : 1;
                if (--kv_users[st] == 0) mma_commit(&kv_empty[st]);
                if (c.j == c.nkv - 1) mma_commit(&o_full[l]);
                advance(c, l);
            };
            for (int l = 0; l < 2; ++l)
                if (cs[l].valid) issue_s(l);
#ifdef PTK_ATTN_TRACE
            if (blockIdx.x < 160) g_pp_cta[blockIdx.x][1] = gt();
#endif
            // Causal pairs give lane A one block fewer per pair than lane B, so lane A's cursor would
            // drift ahead in the shared KV stream; a lane only advances while its next P·V is not past
            // the other lane's, which keeps every S it issues within the producer's NS loaded stages
            // (otherwise the producer waits on a stage only the starved lane can free).
            auto gpv = [&](int l) { return cp[l].kvbase + cp[l].j; };
            while (cp[0].valid || cp[1].valid) {
                for (int l = 0; l < 2; ++l) {
                    if (!cp[l].valid) continue;
                    if (cp[l ^ 1].valid && gpv(l) > gpv(l ^ 1)) continue;
                    if (cs[l].valid) issue_s(l);  // one block ahead
                    issue_pv(l);
                }
            }
        }
    } else if (warp < 4) {
        reg_dealloc<72>();
    } else {  // ---------------- softmax / epilogue: thread = query row of lane L
        reg_alloc<208>();
        // warps 4-7 = lane A, 8-11 = lane B; each set covers the four TMEM lane quarters (warp % 4)
        const int L = (warp - 4) >> 2;
        const int quad = warp & 3;
        const int r = quad * 32 + static_cast<int>(lane_id_);
        const uint32_t lane_base = static_cast<uint32_t>(quad * 32) << 16;
        const uint32_t s_cols = tmem + lane_base + C::kTmemS + 128 * L;
        const uint32_t p_cols = tmem + lane_base + C::kTmemP + 64 * L;
        int n = 0;
        const int nit = *n_items;
        for (int k = 0; k < nit; ++k) {
            const int4 itv = items[k];
            const Fa2Item it{itv.x, itv.y, itv.z, true};
            const int qb = 2 * it.p + L, nkv = fa2_nkv(a, it.p, L);
            const uint32_t o_cols = tmem + lane_base + C::kTmemO + 64 * L;
            float m = -INFINITY, l = 0.f;
            const bool tr = (warp & 3) == 0 && lane_id_ == 0;
            for (int j = 0; j < nkv; ++j, ++n) {
                mbar_wait(&s_full[L], n & 1);
                if (tr) PTRACE(L, n, 0);
                tc_fence_after();
                float x[kBlk];
#pragma unroll
                for (int cc = 0; cc < kBlk / 32; ++cc) tmem_ld_32x32b_x32_nw(s_cols + cc * 32, x + cc * 32);
                tmem_ld_wait();
                tc_fence_before();
                __syncwarp();
                if (lane_id_ == 0) mbar_arrive(&s_empty[L]);
                if (tr) PTRACE(L, n, 1);
                const bool diag = a.causal && j == qb;
                float mr8[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) mr8[i] = -INFINITY;
                if (diag) {
#pragma unroll
                    for (int e = 0; e < kBlk; ++e) {
                        if (e > r) x[e] = -INFINITY;
                        mr8[e & 7] = fmaxf(mr8[e & 7], x[e]);
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < kBlk; ++e) mr8[e & 7] = fmaxf(mr8[e & 7], x[e]);
                }
                const float mraw = fmaxf(fmaxf(fmaxf(mr8[0], mr8[1]), fmaxf(mr8[2], mr8[3])),
                                         fmaxf(fmaxf(mr8[4], mr8[5]), fmaxf(mr8[6], mr8[7])));
                const float pmx = mraw * a.scale_log2;
                const float mx = pmx > m + kLazyRescaleLog2 ? pmx : m;
                const float alpha = ex2(m - mx);
                float s8[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) s8[i] = 0.f;
                const float2 sc2 = make_float2(a.scale_log2, a.scale_log2), mm2 = make_float2(-mx, -mx);
                float2* s2 = reinterpret_cast<float2*>(s8);
                if (diag) {
#pragma unroll
                    for (int e = 0; e < kBlk; e += 2) {
                        const float2 t = __ffma2_rn(make_float2(x[e], x[e + 1]), sc2, mm2);
                        x[e] = ex2(t.x);
                        x[e + 1] = ex2(t.y);
                        s2[(e >> 1) & 3] = __fadd2_rn(s2[(e >> 1) & 3], make_float2(x[e], x[e + 1]));
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < kBlk; e += 2) {
                        const float2 t = __ffma2_rn(make_float2(x[e], x[e + 1]), sc2, mm2);
                        if (kFwdPoly > 0 && ((e >> 1) & 7) < kFwdPoly / 2) {  // first kFwdPoly of every 16
                            const float2 pp = ex2_poly2(t);
                            x[e] = pp.x;
                            x[e + 1] = pp.y;
                        } else {
                            x[e] = ex2(t.x);
                            x[e + 1] = ex2(t.y);
                        }
                        s2[(e >> 1) & 3] = __fadd2_rn(s2[(e >> 1) & 3], make_float2(x[e], x[e + 1]));
                    }
                }
                const float sum = ((s8[0] + s8[1]) + (s8[2] + s8[3])) + ((s8[4] + s8[5]) + (s8[6] + s8[7]));
                l = l * alpha + sum;
                m = mx;
                if (tr) PTRACE(L, n, 2);
                if (n > 0) {
                    mbar_wait(&pv_done[L], (n - 1) & 1);  // P buffer free, O of this pair stable
                    tc_fence_after();
                }
                if (tr) PTRACE(L, n, 3);
                // P (bf16, two per 32-bit column) -> TMEM: the A operand of this lane's P·V
                // packed in place: x[q] = bf16x2(x[2q], x[2q+1]) (x[2q..] not yet overwritten)
#pragma unroll
                for (int q = 0; q < kBlk / 2; ++q) x[q] = __uint_as_float(pack_bf16(x[2 * q], x[2 * q + 1]));
                tmem_st_32x32b_x32_f_nw(p_cols, x);
                tmem_st_32x32b_x32_f_nw(p_cols + 32, x + 32);
                if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
                    for (int cc = 0; cc < D; cc += 16) {
                        float v[16];
                        tmem_ld_32x32b_x16(o_cols + cc, v);
#pragma unroll
                        for (int e = 0; e < 16; ++e) v[e] *= alpha;
                        tmem_st_32x32b_x16(o_cols + cc, v);
                    }
                }
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane_id_ == 0) mbar_arrive(&p_full[L]);
                if (tr) PTRACE(L, n, 4);
            }
            mbar_wait(&o_full[L], k & 1);
            tc_fence_after();
            const float inv = 1.f / l;
            const int q = qb * kBlk + r;
            // O -> registers (the accumulator is released at once) -> bf16 into this lane's 128B-swizzled
            // staging -> one TMA store of the [128][64] tile.  Row-per-thread global stores cost about
            // 1500 cycles per item: every warp store touched 32 rows.
            float v[D];
#pragma unroll
            for (int cc = 0; cc < D; cc += 32) tmem_ld_32x32b_x32_nw(o_cols + cc, v + cc);
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane_id_ == 0) mbar_arrive(&o_empty[L]);
            const uint32_t bar_id = 1 + L, issuer = (warp & 3) == 0 && lane_id_ == 0;
            if (issuer) tma_store_wait_read();  // the lane's previous item left the staging
            asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory");
            const uint32_t row_addr = smem_u32(sO + L * C::kOBytes) + r * 128;
#pragma unroll
            for (int g = 0; g < D / 8; ++g) {
                const float* f = v + 8 * g;
                const uint4 u = make_uint4(pack_bf16(f[0] * inv, f[1] * inv), pack_bf16(f[2] * inv, f[3] * inv),
                                           pack_bf16(f[4] * inv, f[5] * inv), pack_bf16(f[6] * inv, f[7] * inv));
                sts128(row_addr + ((g ^ (r & 7)) * 16), u);
            }
            fence_proxy_async_smem();
            asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory");
            if (issuer) {
                tma_store_4d(&tmO, sO + L * C::kOBytes, 0, qb * kBlk, it.head, it.bi);
                tma_store_commit();
            }
            a.lse[(static_cast<int64_t>(it.bi) * a.H + it.head) * a.s + q] = m + __log2f(l);
        }
        if ((warp & 3) == 0 && lane_id_ == 0) tma_store_wait_all();
    }
    tc_fence_before();
    __syncthreads();
#ifdef PTK_ATTN_TRACE
    if (threadIdx.x == 0 && blockIdx.x < 160) g_pp_cta[blockIdx.x][3] = gt();
#endif
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

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

// qkv [b][s][3][H][d] viewed as dims {d, s, 3H, b}.
cudaError_t qkv_map(CUtensorMap* m, const void* qkv, int b, int s, int H, int d, int box_rows) {
    EncodeTiledFn enc = encode_fn();
    if (!enc) return cudaErrorNotSupported;
    const int64_t h = static_cast<int64_t>(H) * d;
    cuuint64_t dims[4] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(s), static_cast<cuuint64_t>(3 * H),
                          static_cast<cuuint64_t>(b)};
    cuuint64_t strides[3] = {static_cast<cuuint64_t>(3 * h * 2), static_cast<cuuint64_t>(d * 2),
                             static_cast<cuuint64_t>(s * 3 * h * 2)};
    cuuint32_t box[4] = {64, static_cast<cuuint32_t>(box_rows), 1, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(qkv), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// o [b*s][H*d] viewed as dims {d, s, H, b}, box {64, 128} (the ping-pong forward's TMA stores).
cudaError_t o_map(CUtensorMap* m, const void* o, int b, int s, int H, int d) {
    EncodeTiledFn enc = encode_fn();
    if (!enc) return cudaErrorNotSupported;
    const int64_t h = static_cast<int64_t>(H) * d;
    cuuint64_t dims[4] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(s), static_cast<cuuint64_t>(H),
                          static_cast<cuuint64_t>(b)};
    cuuint64_t strides[3] = {static_cast<cuuint64_t>(h * 2), static_cast<cuuint64_t>(d * 2),
                             static_cast<cuuint64_t>(s * h * 2)};
    cuuint32_t box[4] = {64, static_cast<cuuint32_t>(kBlk), 1, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(o), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

bool fwd_pp_enabled() {
    static const bool on = [] {
        const char* v = std::getenv("PTK_FWD_PP");
        return v == nullptr || v[0] != '0';
    }();
    return on;
}

int fwd_poly() {
    static const int v = [] {
        // default 2 of every 16 unmasked exponentials on the FMA pipe: 2-3 % faster once the TMA-store
        // epilogue went in (scripts/bench_attention.py, all shapes); 4 and 6 are slower
        const char* e = std::getenv("PTK_FWD_POLY");
        return e ? std::atoi(e) : 2;
    }();
    return v;
}

template <int D>
cudaError_t launch_fwd_single(const FlashPlan& p, cudaStream_t st);

template <int POLY>
cudaError_t launch_fwd_pp_t(const FlashPlan& p, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(flash_fwd_pp_kernel<POLY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             Fa2Cfg::kSmem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    FaArgs a{p.o, p.lse, p.s, p.H, p.H * p.d, p.b, p.scale_log2, p.causal};
    const int items = p.s / (2 * kBlk) * p.H * p.b;
    const int grid = items < sm_count() ? items : sm_count();
    if ((items + grid - 1) / grid > kFa2MaxItems) return launch_fwd_single<64>(p, st);
    return launch_kernel(flash_fwd_pp_kernel<POLY>, grid, 384, Fa2Cfg::kSmem, st, 1, p.tmQK, p.tmV, p.tmO, a);
}

cudaError_t launch_fwd_pp(const FlashPlan& p, cudaStream_t st) {
    switch (fwd_poly()) {
        case 2: return launch_fwd_pp_t<2>(p, st);
        case 4: return launch_fwd_pp_t<4>(p, st);
        case 6: return launch_fwd_pp_t<6>(p, st);
        default: return launch_fwd_pp_t<0>(p, st);
    }
}

template <int D>
cudaError_t launch_fwd_single(const FlashPlan& p, cudaStream_t st) {
    using C = FaCfg<D>;
    static bool attr = false;
    if (!attr) {
        cudaError_t e =
            cudaFuncSetAttribute(flash_fwd_kernel<D, kFwdNQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    FaArgs a{p.o, p.lse, p.s, p.H, p.H * p.d, p.b, p.scale_log2, p.causal};
    const int tiles = p.s / kBlk * p.H * p.b;
    const int grid = tiles < sm_count() ? tiles : sm_count();
    return launch_kernel(flash_fwd_kernel<D, kFwdNQ>, grid, 32 * (4 + 4 * kFwdNQ), C::kSmem, st, 1, p.tmQK, p.tmV, a);
}

template <int D>
cudaError_t launch_fwd(const FlashPlan& p, cudaStream_t st) {
    if (D == 64 && p.s % (2 * kBlk) == 0 && fwd_pp_enabled()) return launch_fwd_pp(p, st);
    return launch_fwd_single<D>(p, st);
}

}  // namespace

cudaError_t flash_prepare(const void* qkv, void* o, float* lse, int b, int s, int H, int d, FlashPlan* p,
                          int causal) {
    if ((d != 64 && d != 128) || s % kBlk) return cudaErrorInvalidValue;
    cudaError_t e = qkv_map(&p->tmQK, qkv, b, s, H, d, kBlk);
    if (e != cudaSuccess) return e;
    e = qkv_map(&p->tmV, qkv, b, s, H, d, 64);
    if (e != cudaSuccess) return e;
    e = o_map(&p->tmO, o, b, s, H, d);
    if (e != cudaSuccess) return e;
    p->o = static_cast<__nv_bfloat16*>(o);
    p->lse = lse;
    p->b = b;
    p->s = s;
    p->H = H;
    p->d = d;
    p->scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(d));
    p->causal = causal;
    return cudaSuccess;
}

cudaError_t flash_forward(const FlashPlan& p, cudaStream_t st) {
    return p.d == 64 ? launch_fwd<64>(p, st) : launch_fwd<128>(p, st);
}

// ============================================================================
// Backward.  Deterministic two-kernel form (no atomics), both persistent:
//   mode KV: tile = (key block j, head, sample), steps over query blocks i >= j:
//     Sᵀ = K_j Q_iᵀ, dPᵀ = V_j dO_iᵀ            (TMEM, thread = key row)
//     Pᵀ = 2^(Sᵀ c - lse2[q]),  dSᵀ = τ Pᵀ (dPᵀ - D[q])
//     dV_j += Pᵀ dO_i,  dK_j += dSᵀ Q_i           (TMEM accumulators)
//   mode Q:  tile = (query block i, head, sample), steps over key blocks j <= i:
//     S = Q_i K_jᵀ, dP = dO_i V_jᵀ  (thread = query row)
//     dS = τ P (dP - D[q]);  dQ_i += dS K_j
// A [rows][64-col] 128B-swizzled tile is simultaneously the K-major operand
// for the score products and the MN-major operand (LBO = 16 KiB between
// 64-wide column atoms) for the accumulating products, so every operand is
// loaded once per step.  τ·D = τ rowsum(dO ∘ O) comes from attn_bwd_dot_kernel.
// d = 64: P/dS go to TMEM as the A operand of the accumulating products, three
// operand stages, and in the KV pass −lse/c and −D enter the score products as
// extra K columns (a per-stage stats operand against a fixed ones operand) so
// the elementwise pass reads no per-column statistics; d = 128: P/dS through
// smem, one stage, the statistics from the stage's smem rows.
// One CTA per SM walks its tiles (heaviest first, boustrophedon); the fixed
// tiles are double-buffered across tiles (d = 64).  Epilogues stage the bf16
// outputs in 128B-swizzled smem and leave with TMA stores.
// ============================================================================
namespace {

template <int D, bool KV>
struct BwCfg {
    // d = 64: the elementwise results Pᵀ / dS(ᵀ) go to TMEM (bf16 pairs) and feed the accumulating
    // products as their A operand (tcgen05.mma A-from-TMEM): no smem round trip, which halves the
    // smem traffic per step (smem bandwidth bounded the step: scores 64 KiB + P/dS writes 64 KiB +
    // their MMA reads 64 KiB + accumulating B 32 KiB + TMA 32 KiB per 128x128 step).  d = 128 has
    // no TMEM room for them (X, Y and the 2d-column accumulator fill 512 columns).
    static constexpr bool kTs = D == 64;
    static constexpr int kTile = kBlk * D * 2;  // one [128][D] tile
    // step operand stages: with three, the load of step n+2 does not wait for step n's accumulating
    // products to release its stage (a TMA round trip that sat on the critical path with two)
    static constexpr int kStages = D == 64 ? 3 : 1;
    static constexpr int kFixBuf = D == 64 ? 2 : 1;
    static constexpr int kAccBuf = (KV && (D == 128 || kTs)) ? 1 : 2;
    static constexpr int kAccCols = KV ? 2 * D : D;  // per accumulator buffer
    static constexpr int kPd = kBlk * kBlk * 2;      // one [128][128] bf16 A-operand buffer (smem path)
    // epilogue staging for the TMA stores of a tile's outputs (KV: dV and dK, Q: dQ; 128B-swizzled
    // [128 rows][64 cols] atoms); the smem path (d = 128) stages in the P / dS buffers instead
    static constexpr int kOutBytes = kTs ? (KV ? 2 : 1) * kTile : 0;
    static constexpr int kRowBytes = 2 * kBlk * 4;  // per stage: the stepped block's lse[128], τD[128] (KV)
    // KV: the per-query softmax statistics enter the score products as extra K columns: per stage a
    // [128 queries][16] bf16 "stats" operand (−lse/c and −D, each as three bf16 terms) and, fixed, two
    // [128 keys][16] "ones" operands selecting them (X' = S − lse/c, Y' = dPᵀ − D); K-major, no swizzle
    static constexpr bool kFold = KV && D == 64;  // d = 128 (one stage) keeps the smem row reads
    static constexpr int kStatBytes = kBlk * 16 * 2;  // 4 KiB
    static constexpr int kStatSmem = kFold ? (kStages + 2) * kStatBytes : 0;
    static constexpr int kSmem = kFixBuf * 2 * kTile + kStages * 2 * kTile + (kTs ? 0 : 2 * kPd) + kOutBytes +
                                 kStatSmem + kStages * kRowBytes + 1024 + 256;
    static constexpr uint32_t kX = 0, kY = 128, kAcc = 256;
    static constexpr uint32_t kP = kAcc + kAccBuf * kAccCols, kDS = kP + 64;  // TMEM A operands (kTs)
    static_assert(!kTs || kDS + 64 <= 512, "TMEM budget");
    static_assert(kStages <= 4, "ld_full / ld_empty hold four stages");
    static_assert(kSmem <= 232448, "backward smem");
};

struct BwArgs {
    __nv_bfloat16* dqkv;  // [b*s][3h]
    float* col_part;      // optional [b*s/32][3h] += column sums of dqkv per 32 rows
    const float* lse;     // [b][H][s]
    const float* dsum;    // [b][H][s]: τ·D
    int s, H, h, b;
    float scale_log2, tau;
    int causal;
};

#ifdef PTK_ATTN_TRACE
// Debug timeline of CTA 0 (clock64): [role][step][event], see scripts/attn_trace.cu.
__device__ unsigned long long g_attn_trace[2][64][8];
__device__ int g_attn_trace_kv = 1;  // which backward kernel records (1: KV, 0: Q)
#define ATRACE(role, step, ev)                                                                        \
    do {                                                                                              \
        if (atrace_on && (step) < 64)                                                                 \
            g_attn_trace[role][step][ev] = clock64();                                                 \
    } while (0)
#else
#define ATRACE(role, step, ev) \
    do {                       \
    } while (0)
#endif

// Position in a CTA's tile list (see fa_tile): tile k, step j of that tile.
struct BwCursor {
    int k, blk, head, bi, first, nsteps, j;
    bool valid;
};

template <bool KV>
__device__ __forceinline__ void bw_tile(const BwArgs& a, int k, BwCursor& c) {
    const int G = gridDim.x, i = blockIdx.x;
    const int nb = a.s / kBlk;
    const int per = a.H * a.b;
    const int t = (k & 1) ? (k + 1) * G - 1 - i : k * G + i;
    c.k = k;
    c.j = 0;
    c.valid = t < nb * per;
    const int rank = t / per, rem = t % per;
    c.blk = KV ? rank : nb - 1 - rank;  // heaviest first under the causal mask
    c.head = rem % a.H;
    c.bi = rem / a.H;
    c.first = (KV && a.causal) ? c.blk : 0;
    c.nsteps = !a.causal ? nb : (KV ? nb - c.blk : c.blk + 1);
}

template <bool KV>
__device__ __forceinline__ void bw_next(const BwArgs& a, BwCursor& c) {
    if (++c.j == c.nsteps) bw_tile<KV>(a, c.k + 1, c);
}


__device__ __forceinline__ float4 lds128f(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr)
                 : "memory");
    return v;
}

// 32 columns [cb0, cb0+32) of one row: P = 2^(X c - lse) and dS = P (τ Y - τ D),
// packed to bf16 pairs.  KV: the per-column (query) lse / τD come from smem
// (rowv); Q: the row's own my_lse / my_d.  MASK only on diagonal blocks.
template <bool KV, bool MASK, bool FOLD>
__device__ __forceinline__ void bw_pass(const float (&x)[32], const float (&y)[32], uint32_t rowv, int cb0, int r,
                                        float sc, float tau, float my_lse, float my_d, uint32_t* pk_p,
                                        uint32_t* pk_d) {
#pragma unroll
    for (int e4 = 0; e4 < 8; ++e4) {
        const int cb = cb0 + e4 * 4;
        float l2[4], dd[4];
        if (KV && !FOLD) {
            const float4 lv = lds128f(rowv + cb * 4);
            const float4 dv = lds128f(rowv + (kBlk + cb) * 4);
            l2[0] = lv.x, l2[1] = lv.y, l2[2] = lv.z, l2[3] = lv.w;
            dd[0] = dv.x, dd[1] = dv.y, dd[2] = dv.z, dd[3] = dv.w;
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) l2[u] = my_lse, dd[u] = my_d;
        }
        float pv[4], dv4[4];
        float xs[4];
        if constexpr (FOLD) {
            // X' = S − lse/c and Y' = dPᵀ − D come out of the score products: P = 2^(c X'),
            // dS/τ = P Y' (τ is applied to the dK accumulator in the epilogue)
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                xs[u] = x[e4 * 4 + u];
                if (MASK && cb + u < r) xs[u] = -INFINITY;  // row = key, col = query: valid iff query >= key
            }
            const float2 sc2 = make_float2(sc, sc);
#pragma unroll
            for (int u = 0; u < 4; u += 2) {
                const float2 t = __fmul2_rn(make_float2(xs[u], xs[u + 1]), sc2);
                const bool poly = !MASK && kBwPoly > 0 && (e4 % (8 / kBwPoly)) == 0;
                pv[u] = ex2(t.x);
                pv[u + 1] = (poly && u + 1 == 3) ? ex2_poly(t.y) : ex2(t.y);
                const float2 ds = __fmul2_rn(make_float2(pv[u], pv[u + 1]), make_float2(y[e4 * 4 + u], y[e4 * 4 + u + 1]));
                dv4[u] = ds.x;
                dv4[u + 1] = ds.y;
            }
            pk_p[e4 * 2] = pack_bf16(pv[0], pv[1]);
            pk_p[e4 * 2 + 1] = pack_bf16(pv[2], pv[3]);
            pk_d[e4 * 2] = pack_bf16(dv4[0], dv4[1]);
            pk_d[e4 * 2 + 1] = pack_bf16(dv4[2], dv4[3]);
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                xs[u] = x[e4 * 4 + u];
                if (MASK) {
                    // KV: row = key, col = query -> valid iff query >= key ; Q: row = query, col = key
                    const int col = cb + u;
                    if (KV ? col < r : col > r) xs[u] = -INFINITY;  // exp2(-inf) = 0
                }
            }
            // packed fp32x2 (FFMA2 / FMUL2): the same per-lane operations as the scalar form
            const float2 sc2 = make_float2(sc, sc), tau2 = make_float2(tau, tau);
#pragma unroll
            for (int u = 0; u < 4; u += 2) {
                const float2 t = __ffma2_rn(make_float2(xs[u], xs[u + 1]), sc2, make_float2(-l2[u], -l2[u + 1]));
                // a share of the exponentials on the FMA pipe (the pass is MUFU-bound; kBwPoly of 8)
                const bool poly = !MASK && kBwPoly > 0 && (e4 % (8 / kBwPoly)) == 0;
                pv[u] = ex2(t.x);
                pv[u + 1] = (poly && u + 1 == 3) ? ex2_poly(t.y) : ex2(t.y);
                const float2 g = __ffma2_rn(tau2, make_float2(y[e4 * 4 + u], y[e4 * 4 + u + 1]),
                                            make_float2(-dd[u], -dd[u + 1]));
                const float2 ds = __fmul2_rn(make_float2(pv[u], pv[u + 1]), g);
                dv4[u] = ds.x;
                dv4[u + 1] = ds.y;
            }
            pk_p[e4 * 2] = pack_bf16(pv[0], pv[1]);
            pk_p[e4 * 2 + 1] = pack_bf16(pv[2], pv[3]);
            pk_d[e4 * 2] = pack_bf16(dv4[0], dv4[1]);
            pk_d[e4 * 2 + 1] = pack_bf16(dv4[2], dv4[3]);
        }
    }
}

template <int D, bool KV>
__global__ void __launch_bounds__(kThreads, 1)
    flash_bwd_kernel(const __grid_constant__ CUtensorMap tmQKV, const __grid_constant__ CUtensorMap tmDO,
                     const __grid_constant__ CUtensorMap tmDQKV, const __grid_constant__ BwArgs a) {
    using C = BwCfg<D, KV>;
    constexpr int S = C::kStages, FB = C::kFixBuf, AB = C::kAccBuf;
    constexpr uint32_t kIdescXY = make_idesc_bf16(kBlk, kBlk, false, false);
    constexpr uint32_t kIdescAcc = make_idesc_bf16(kBlk, D, false, true);

    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sFix = smem;                           // [FB][2 tiles]: (K_j, V_j) (KV) | (Q_i, dO_i) (Q)
    uint8_t* sStep = sFix + FB * 2 * C::kTile;      // [S][2 tiles]: (Q_i, dO_i) (KV) | (K_j, V_j) (Q)
    uint8_t* sP = sStep + S * 2 * C::kTile;         // Pᵀ (KV only; smem path)
    uint8_t* sDS = sP + (C::kTs ? 0 : C::kPd);      // dSᵀ (KV) | dS (Q) (smem path)
    uint8_t* sOut = C::kTs ? sDS + 0 : sP;          // epilogue staging (dedicated for d = 64)
    // [S][lse[128], τD[128]] of the stepped query block (KV), bulk-loaded with the stage's tiles
    uint8_t* sStat = sDS + (C::kTs ? C::kOutBytes : C::kPd);  // KV: [S] stats, then ones_x, ones_y
    float* sRow = reinterpret_cast<float*>(sStat + C::kStatSmem);
    uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sRow) + S * C::kRowBytes);
    uint64_t* fix_full = bars + 0;    // [2]
    uint64_t* fix_empty = bars + 2;   // [2]
    uint64_t* ld_full = bars + 16;    // [4]
    uint64_t* ld_empty = bars + 20;   // [4]
    uint64_t* xy_full = bars + 8;
    uint64_t* xy_free = bars + 9;
    uint64_t* pd_full = bars + 10;
    uint64_t* pd_free = bars + 11;
    uint64_t* acc_full = bars + 12;   // [2]
    uint64_t* acc_empty = bars + 14;  // [2]
    uint64_t* stat_full = bars + 24;  // [4] KV: the stage's stats operand is built
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 28);

    const int warp = threadIdx.x / 32;
    const uint32_t lane = lane_id();
#ifdef PTK_ATTN_TRACE
    // read once: a global load inside every trace point would add its latency to the timeline
    const bool atrace_on = blockIdx.x == 0 && *static_cast<volatile int*>(&g_attn_trace_kv) == (KV ? 1 : 0);
#endif

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmQKV);
        tma_prefetch_desc(&tmDO);
        tma_prefetch_desc(&tmDQKV);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&fix_full[i], 1);
            mbar_init(&fix_empty[i], 1);
            mbar_init(&acc_full[i], 1);
            mbar_init(&acc_empty[i], 8);
        }
        for (int i = 0; i < S; ++i) {
            mbar_init(&ld_full[i], 1);
            mbar_init(&ld_empty[i], 1);
            mbar_init(&stat_full[i], 2);  // warps 2 and 3
        }
        mbar_init(xy_full, 1);
        mbar_init(xy_free, 8);
        mbar_init(pd_full, 8);
        mbar_init(pd_free, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<512>(tmem_slot);
    if (C::kFold) {
        // stats buffers zeroed (their second K chunk stays zero), ones operands: row k of ones_x is
        // [1,1,1,0..], of ones_y [0,0,0,1,1,1,0..]; layout [8-row group][k chunk][8 rows][8 bf16]
        uint32_t* z = reinterpret_cast<uint32_t*>(sStat);
        for (int i = threadIdx.x; i < (S + 2) * C::kStatBytes / 4; i += blockDim.x) {
            const int off = i * 4 - S * C::kStatBytes;  // byte offset into the ones tiles
            uint32_t v = 0;
            if (off >= 0) {
                const int tile = off / C::kStatBytes, o = off % C::kStatBytes;
                const int chunk = (o / 128) % 2, e = (o % 16) / 2;  // bf16 pair index e, e+1
                if (chunk == 0) {
                    const bool lo = tile == 0 ? e < 3 : (e >= 3 && e < 6), hi = tile == 0 ? e + 1 < 3 : (e + 1 >= 3 && e + 1 < 6);
                    v = (lo ? 0x3F80u : 0u) | (hi ? 0x3F80u << 16 : 0u);
                }
            }
            z[i] = v;
        }
        fence_proxy_async_smem();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (KV) {
        pdl_begin();  // previous kernel complete: its outputs (qkv, lse, dO, D, ...) are visible
    } else {
        // The dQ pass reads only what the dK/dV pass read (qkv, dO, lse, D: complete before that
        // pass started, and this grid launches only after it passed its own wait) and writes
        // disjoint dqkv columns, so it need not wait for the dK/dV pass: its CTAs take the SMs the
        // dK/dV pass frees in its tail.  It waits at the end instead, so kernels after it still see
        // both passes complete.
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    }

    if (warp == 0) {
        if (C::kTs) reg_dealloc<72>();
        if (lane == 0) {  // ---------------- TMA producer
            // tile loader: rows [row0, row0+128) of a {d, s, heads, b} map, head coordinate hc
            auto load_tile = [&](const CUtensorMap* m, uint64_t* bar, uint8_t* dst, int row0, int hc, int bi) {
#pragma unroll
                for (int kb = 0; kb < D / 64; ++kb) tma_load_4d(m, bar, dst + kb * kBlk * 128, kb * 64, row0, hc, bi);
            };
            int n = 0;  // steps loaded so far (all tiles)
            BwCursor c;
            for (bw_tile<KV>(a, 0, c); c.valid; bw_tile<KV>(a, c.k + 1, c)) {
                const int fb = c.k % FB;
                uint8_t* f = sFix + fb * 2 * C::kTile;
                mbar_wait(&fix_empty[fb], ((c.k / FB) & 1) ^ 1);
                mbar_arrive_expect_tx(&fix_full[fb], 2 * C::kTile);
                if (KV) {
                    load_tile(&tmQKV, &fix_full[fb], f, c.blk * kBlk, a.H + c.head, c.bi);                // K_j
                    load_tile(&tmQKV, &fix_full[fb], f + C::kTile, c.blk * kBlk, 2 * a.H + c.head, c.bi);  // V_j
                } else {
                    load_tile(&tmQKV, &fix_full[fb], f, c.blk * kBlk, c.head, c.bi);           // Q_i
                    load_tile(&tmDO, &fix_full[fb], f + C::kTile, c.blk * kBlk, c.head, c.bi);  // dO_i
                }
                for (int t = 0; t < c.nsteps; ++t, ++n) {
                    const int st = n % S;
                    mbar_wait(&ld_empty[st], ((n / S) & 1) ^ 1);
                    mbar_arrive_expect_tx(&ld_full[st], 2 * C::kTile + (KV ? C::kRowBytes : 0));
                    uint8_t* t0 = sStep + st * 2 * C::kTile;
                    const int row0 = (c.first + t) * kBlk;
                    if (KV) {
                        load_tile(&tmQKV, &ld_full[st], t0, row0, c.head, c.bi);            // Q_i
                        load_tile(&tmDO, &ld_full[st], t0 + C::kTile, row0, c.head, c.bi);  // dO_i
                        // the per-query softmax statistics every elementwise thread reads (no exchange)
                        const int64_t rb = (static_cast<int64_t>(c.bi) * a.H + c.head) * a.s + row0;
                        float* rows = sRow + st * (C::kRowBytes / 4);
                        bulk_load(rows, a.lse + rb, kBlk * 4, &ld_full[st]);
                        bulk_load(rows + kBlk, a.dsum + rb, kBlk * 4, &ld_full[st]);
                    } else {
                        load_tile(&tmQKV, &ld_full[st], t0, row0, a.H + c.head, c.bi);                  // K_j
                        load_tile(&tmQKV, &ld_full[st], t0 + C::kTile, row0, 2 * a.H + c.head, c.bi);  // V_j
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (C::kTs) reg_dealloc<72>();
        if (lane == 0) {  // ---------------- MMA issuer
            auto issue_xy = [&](const BwCursor& c, int n) {
                ATRACE(1, n, 0);
                const int st = n % S, fb = c.k % FB;
                if (c.j == 0) mbar_wait(&fix_full[fb], (c.k / FB) & 1);
                mbar_wait(&ld_full[st], (n / S) & 1);
                mbar_wait(xy_free, (n & 1) ^ 1);  // elementwise warps have read the previous X/Y
                tc_fence_after();
                const uint32_t f0 = smem_u32(sFix + fb * 2 * C::kTile), f1 = f0 + C::kTile;
                const uint32_t s0 = smem_u32(sStep + st * 2 * C::kTile), s1 = s0 + C::kTile;
#pragma unroll
                for (int k = 0; k < D / 16; ++k) {
                    const uint32_t off = (k / 4) * kBlk * 128 + (k % 4) * 32;
                    // X = F0 · Step0ᵀ,  Y = F1 · Step1ᵀ   (both operands K-major, K = d)
                    mma_bf16_ss(tmem + C::kX, make_sw128_desc(f0 + off, 16, 1024), make_sw128_desc(s0 + off, 16, 1024),
                                kIdescXY, k > 0 ? 1u : 0u);
                    mma_bf16_ss(tmem + C::kY, make_sw128_desc(f1 + off, 16, 1024), make_sw128_desc(s1 + off, 16, 1024),
                                kIdescXY, k > 0 ? 1u : 0u);
                }
                if (C::kFold) {  // X' = X − lse/c, Y' = Y − D: the stats columns against the ones operands
                    mbar_wait(&stat_full[st], (n / S) & 1);
                    tc_fence_after();
                    const uint32_t sb = smem_u32(sStat + st * C::kStatBytes);
                    const uint32_t ox = smem_u32(sStat + S * C::kStatBytes), oy = ox + C::kStatBytes;
                    mma_bf16_ss(tmem + C::kX, make_interleave_desc(ox, 128, 256), make_interleave_desc(sb, 128, 256),
                                kIdescXY, 1u);
                    mma_bf16_ss(tmem + C::kY, make_interleave_desc(oy, 128, 256), make_interleave_desc(sb, 128, 256),
                                kIdescXY, 1u);
                }
                mma_commit(xy_full);
                ATRACE(1, n, 1);
                if (c.j == c.nsteps - 1) mma_commit(&fix_empty[fb]);
            };
            BwCursor cx, ca;
            bw_tile<KV>(a, 0, cx);
            bw_tile<KV>(a, 0, ca);
            int nx = 0, na = 0;
            if (cx.valid) {
                issue_xy(cx, nx++);
                bw_next<KV>(a, cx);
            }
            while (ca.valid) {
                // with two operand stages, score products of the next step (possibly of
                // the next tile) overlap the elementwise work of this one; with one stage
                // they must wait for this step's accumulating products to release it
                if (S > 1 && cx.valid) {
                    issue_xy(cx, nx++);
                    bw_next<KV>(a, cx);
                }
                const int st = na % S, ab = AB == 1 ? 0 : (ca.k & 1);
                mbar_wait(pd_full, na & 1);
                ATRACE(1, na, 2);
                if (ca.j == 0) mbar_wait(&acc_empty[ab], ((ca.k / AB) & 1) ^ 1);
                tc_fence_after();
                const uint32_t s0 = smem_u32(sStep + st * 2 * C::kTile), s1 = s0 + C::kTile;
                const uint32_t pb = smem_u32(sP), db = smem_u32(sDS);
                const uint32_t acc0 = tmem + C::kAcc + ab * C::kAccCols;
#pragma unroll
                for (int k = 0; k < kBlk / 16; ++k) {
                    const uint32_t aoff = (k / 4) * kBlk * 128 + (k % 4) * 32;  // K-major A, k over 128 columns
                    const uint32_t boff = k * 2048;                            // MN-major B, k over 128 rows
                    const uint32_t acc = (ca.j > 0 || k > 0) ? 1u : 0u;
                    if (C::kTs) {  // A operands from TMEM: 16 columns of k = 8 TMEM columns per step
                        if (KV) {
                            mma_bf16_ts(acc0, tmem + C::kP + k * 8, make_sw128_desc(s1 + boff, kBlk * 128, 1024),
                                        kIdescAcc, acc);
                            mma_bf16_ts(acc0 + D, tmem + C::kDS + k * 8,
                                        make_sw128_desc(s0 + boff, kBlk * 128, 1024), kIdescAcc, acc);
                        } else {
                            mma_bf16_ts(acc0, tmem + C::kDS + k * 8, make_sw128_desc(s0 + boff, kBlk * 128, 1024),
                                        kIdescAcc, acc);
                        }
                    } else if (KV) {
                        // dV += Pᵀ dO_i ; dK += dSᵀ Q_i
                        mma_bf16_ss(acc0, make_sw128_desc(pb + aoff, 16, 1024),
                                    make_sw128_desc(s1 + boff, kBlk * 128, 1024), kIdescAcc, acc);
                        mma_bf16_ss(acc0 + D, make_sw128_desc(db + aoff, 16, 1024),
                                    make_sw128_desc(s0 + boff, kBlk * 128, 1024), kIdescAcc, acc);
                    } else {
                        // dQ += dS K_j
                        mma_bf16_ss(acc0, make_sw128_desc(db + aoff, 16, 1024),
                                    make_sw128_desc(s0 + boff, kBlk * 128, 1024), kIdescAcc, acc);
                    }
                }
                mma_commit(pd_free);
                ATRACE(1, na, 3);
#ifdef PTK_ATTN_TRACE_MMA  // debug: accumulating-product latency as seen by the issuer (serialises)
                mbar_wait(pd_free, na & 1);
                ATRACE(1, na, 4);
#endif
                mma_commit(&ld_empty[st]);
                if (ca.j == ca.nsteps - 1) mma_commit(&acc_full[ab]);
                if (S == 1 && cx.valid) {
                    issue_xy(cx, nx++);
                    bw_next<KV>(a, cx);
                }
                bw_next<KV>(a, ca);
                ++na;
            }
        }
    } else if (warp < 4) {
        if (C::kTs) reg_dealloc<72>();
        if (C::kFold) {  // ---------------- stats operand builders: per step, from the stage's lse / τD rows
            const int tid = threadIdx.x - 64;  // 0..63: rows tid and tid + 64 of the stepped block
            const float inv_c = 1.f / a.scale_log2, inv_tau = 1.f / a.tau;
            auto split3 = [](float v, uint32_t& p01, uint32_t& p2) {  // v ≈ b0 + b1 + b2 (bf16 terms)
                const __nv_bfloat16 b0 = __float2bfloat16(v);
                const float r1 = v - __bfloat162float(b0);
                const __nv_bfloat16 b1 = __float2bfloat16(r1);
                const __nv_bfloat16 b2 = __float2bfloat16(r1 - __bfloat162float(b1));
                p01 = static_cast<uint32_t>(__bfloat16_as_ushort(b0)) | (static_cast<uint32_t>(__bfloat16_as_ushort(b1)) << 16);
                p2 = __bfloat16_as_ushort(b2);
            };
            int n = 0;
            BwCursor c;
            for (bw_tile<KV>(a, 0, c); c.valid; bw_next<KV>(a, c), ++n) {
                const int st = n % S;
                mbar_wait(&ld_full[st], (n / S) & 1);  // the rows landed; the stage's previous stats consumed
                const float* rows = sRow + st * (C::kRowBytes / 4);
#pragma unroll
                for (int h2 = 0; h2 < 2; ++h2) {
                    const int q = tid + 64 * h2;
                    uint32_t l01, l2, d01, d2;
                    split3(-rows[q] * inv_c, l01, l2);
                    split3(-rows[kBlk + q] * inv_tau, d01, d2);
                    // chunk 0 of row q: [l0, l1, l2, d0, d1, d2, 0, 0]
                    sts128(smem_u32(sStat + st * C::kStatBytes + (q / 8) * 256 + (q % 8) * 16),
                           make_uint4(l01, l2 | (d01 << 16), (d01 >> 16) | (d2 << 16), 0u));
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(&stat_full[st]);
            }
        }
    } else {  // ---------------- elementwise warps: thread = (row of the fixed block, column half)
        if (C::kTs) reg_alloc<208>();
        const int quad = warp & 3;
        const int half = (warp - 4) >> 2;  // columns [64*half, 64*half + 64) of X/Y
        const int r = quad * 32 + static_cast<int>(lane);
        const uint32_t lane_base = static_cast<uint32_t>(quad * 32) << 16;
        const uint32_t rowv0 = smem_u32(sRow);
        const uint32_t pbuf = smem_u32(sP), dbuf = smem_u32(sDS);
        const float sc = a.scale_log2, tau = a.tau;
        // per-row softmax statistics, prefetched one step ahead (global loads off the critical path)
        //   KV: the stepped query block's lse (half 0) / D (half 1) at row r of that block
        //   Q:  this tile's own lse and D at row r
        auto stats = [&](const BwCursor& q, float& s0, float& s1) {
            if (KV) return;  // KV: the stepped block's statistics arrive in smem with its tiles
            const int64_t rb = (static_cast<int64_t>(q.bi) * a.H + q.head) * a.s;
            s0 = a.lse[rb + q.blk * kBlk + r];
            s1 = a.dsum[rb + q.blk * kBlk + r];
        };
        int n = 0;  // steps processed so far (all tiles)
        BwCursor c, cn;
        bw_tile<KV>(a, 0, c);
        cn = c;
        float pre0 = 0.f, pre1 = 0.f;
        if (c.valid) stats(c, pre0, pre1);
        for (; c.valid; ++n) {
            const float cur0 = pre0, cur1 = pre1;
            bw_next<KV>(a, cn);
            if (cn.valid && cn.j == 0) stats(cn, pre0, pre1);  // Q: per-tile values, fetched at a tile's first step
            {
                const int t = c.j;
                const int other = c.first + t;  // index of the stepped block
                const float my_lse = cur0, my_d = cur1;
                const uint32_t rowv = rowv0 + (n % S) * C::kRowBytes;
                if (warp == 4 && lane == 0) ATRACE(0, n, 5);
                mbar_wait(xy_full, n & 1);
                if (KV && !C::kFold) mbar_wait(&ld_full[n % S], (n / S) & 1);  // the stage's lse / τD landed
                if (warp == 4 && lane == 0) ATRACE(0, n, 0);
                tc_fence_after();
                const bool diag = a.causal && other == c.blk;
                // this thread's 64 columns of X and Y in two 32-column passes (the score
                // accumulators are released after the second pass's loads); P and
                // dS = P (τ dP - τ D) are packed to bf16 pairs in registers, before waiting
                // for the previous step's accumulating products to release the smem operands
                uint32_t pk_p[32], pk_d[32];
                if (C::kTs) {
                    // all 64 columns of X and Y loaded before any compute: the score accumulators are
                    // released one TMEM round trip after xy_full, so the next step's X/Y products start
                    // while this step's elementwise work runs (208 registers: setmaxnreg below)
                    float x[2][32], y[2][32];
#pragma unroll
                    for (int pass = 0; pass < 2; ++pass) {
                        tmem_ld_32x32b_x32_nw(tmem + lane_base + C::kX + half * 64 + pass * 32, x[pass]);
                        tmem_ld_32x32b_x32_nw(tmem + lane_base + C::kY + half * 64 + pass * 32, y[pass]);
                    }
                    tmem_ld_wait();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(xy_free);
                    if (warp == 4 && lane == 0) ATRACE(0, n, 1);
                    // each 32-column pass goes to TMEM as soon as it is packed: the wait for the previous
                    // step's accumulating products and the first store overlap the second pass
#pragma unroll
                    for (int pass = 0; pass < 2; ++pass) {
                        const int cb0 = half * 64 + pass * 32;
                        if (diag)
                            bw_pass<KV, true, C::kFold>(x[pass], y[pass], rowv, cb0, r, sc, tau, my_lse, my_d, pk_p + pass * 16,
                                              pk_d + pass * 16);
                        else
                            bw_pass<KV, false, C::kFold>(x[pass], y[pass], rowv, cb0, r, sc, tau, my_lse, my_d, pk_p + pass * 16,
                                               pk_d + pass * 16);
                        if (pass == 0) {
                            if (n > 0) mbar_wait(pd_free, (n - 1) & 1);  // previous step's MMAs done reading P / dS
                            tc_fence_after();
                            if (warp == 4 && lane == 0) ATRACE(0, n, 3);
                        }
                        if (KV) tmem_st_32x32b_x16_u_nw(tmem + lane_base + C::kP + half * 32 + pass * 16, pk_p + pass * 16);
                        tmem_st_32x32b_x16_u_nw(tmem + lane_base + C::kDS + half * 32 + pass * 16, pk_d + pass * 16);
                    }
                    tmem_st_wait();
                } else {
#pragma unroll
                    for (int pass = 0; pass < 2; ++pass) {
                        float x[32], y[32];
                        tmem_ld_32x32b_x32_nw(tmem + lane_base + C::kX + half * 64 + pass * 32, x);
                        tmem_ld_32x32b_x32_nw(tmem + lane_base + C::kY + half * 64 + pass * 32, y);
                        tmem_ld_wait();
                        if (pass == 1) {
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) mbar_arrive(xy_free);
                            if (warp == 4 && lane == 0) ATRACE(0, n, 1);
                        }
                        const int cb0 = half * 64 + pass * 32;
                        if (diag)
                            bw_pass<KV, true, C::kFold>(x, y, rowv, cb0, r, sc, tau, my_lse, my_d, pk_p + pass * 16, pk_d + pass * 16);
                        else
                            bw_pass<KV, false, C::kFold>(x, y, rowv, cb0, r, sc, tau, my_lse, my_d, pk_p + pass * 16,
                                               pk_d + pass * 16);
                    }
                }
                if (warp == 4 && lane == 0) ATRACE(0, n, 2);
                if (!C::kTs) {
                    if (n > 0) mbar_wait(pd_free, (n - 1) & 1);  // previous step's MMAs done reading sP / sDS
                    if (warp == 4 && lane == 0) ATRACE(0, n, 3);
                    // this thread's 64 columns are swizzle atom `half` of each [128][128] operand
                    const uint32_t prow = pbuf + half * (kBlk * 128) + r * 128;
                    const uint32_t drow = dbuf + half * (kBlk * 128) + r * 128;
#pragma unroll
                    for (int g = 0; g < 8; ++g) {
                        const uint32_t sw = (g ^ (r & 7)) * 16;
                        if (KV)
                            sts128(prow + sw, make_uint4(pk_p[g * 4], pk_p[g * 4 + 1], pk_p[g * 4 + 2], pk_p[g * 4 + 3]));
                        sts128(drow + sw, make_uint4(pk_d[g * 4], pk_d[g * 4 + 1], pk_d[g * 4 + 2], pk_d[g * 4 + 3]));
                    }
                    fence_proxy_async_smem();
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(pd_full);
                if (warp == 4 && lane == 0) ATRACE(0, n, 4);
                if (warp == 11 && lane == 0) ATRACE(0, n, 6);
            }
            if (c.j < c.nsteps - 1) {
                bw_next<KV>(a, c);
                continue;
            }
            const int ab = AB == 1 ? 0 : (c.k & 1);
            // epilogue: accumulators -> bf16 -> swizzled smem staging -> TMA stores into dqkv.  KV:
            // half 0 holds dV (section 2), half 1 dK (section 1); Q: dQ, half h columns [h*D/2, +D/2).
            // (Direct row-per-thread global stores cost ~2000 cycles per tile: every warp store
            // touched 32 rows.)
            constexpr int kCols = KV ? D : D / 2;
            const int sec = KV ? (half == 0 ? 2 : 1) : 0;
            const int64_t colbase = static_cast<int64_t>(sec) * a.h + c.head * D + (KV ? 0 : half * (D / 2));
            const int64_t prow = (static_cast<int64_t>(c.bi) * a.s + c.blk * kBlk + (r & ~31)) / 32;
            float cp_old[kCols / 32];
            if (a.col_part != nullptr) {  // this thread's own bias partials, fetched off the critical path
#pragma unroll
                for (int cc = 0; cc < kCols / 32; ++cc) cp_old[cc] = a.col_part[prow * (3 * a.h) + colbase + cc * 32 + lane];
            }
            if (warp == 4 && lane == 0) tma_store_wait_read();  // the previous tile's stores left the staging
            asm volatile("bar.sync 1, 256;" ::: "memory");
            mbar_wait(&acc_full[ab], (c.k / AB) & 1);
            tc_fence_after();
            const uint32_t col0 = C::kAcc + ab * C::kAccCols + (KV ? half * D : half * (D / 2));
            const uint32_t stage = smem_u32(sOut) + (KV ? half * C::kTile : 0);
#pragma unroll
            for (int cc = 0; cc < kCols / 32; ++cc) {
                float v[32];
                tmem_ld_32x32b_x32(tmem + lane_base + col0 + cc * 32, v);
                if (C::kFold && half == 1) {  // dK accumulated dS/τ (the folded Y' carries no τ)
#pragma unroll
                    for (int e = 0; e < 32; ++e) v[e] *= a.tau;
                }
                const int cs = (KV ? 0 : half * (D / 2)) + cc * 32;  // column within the section's head
                const uint32_t row_addr = stage + (cs / 64) * (kBlk * 128) + r * 128;
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    const uint4 u = make_uint4(pack_bf16(v[g * 8 + 0], v[g * 8 + 1]), pack_bf16(v[g * 8 + 2], v[g * 8 + 3]),
                                               pack_bf16(v[g * 8 + 4], v[g * 8 + 5]), pack_bf16(v[g * 8 + 6], v[g * 8 + 7]));
                    sts128(row_addr + ((((cs % 64) / 8 + g) ^ (r & 7)) * 16), u);
                }
                if (a.col_part != nullptr) {
                    // QKV bias gradient: column sums of the warp's 32 rows of dqkv as stored.  A
                    // reduce-scatter over the lanes (fixed xor order) leaves column `lane` in x[0].
                    float x[32];
#pragma unroll
                    for (int e = 0; e < 32; ++e) x[e] = __bfloat162float(__float2bfloat16(v[e]));
#pragma unroll
                    for (int k = 16; k >= 1; k >>= 1) {
                        const bool upper = (lane & static_cast<uint32_t>(k)) != 0;
#pragma unroll
                        for (int i = 0; i < k; ++i) {
                            const float send = upper ? x[i] : x[i + k];
                            const float keep = upper ? x[i + k] : x[i];
                            x[i] = keep + __shfl_xor_sync(0xffffffffu, send, k);
                        }
                    }
                    cp_old[cc] += x[0];
                }
            }
            tc_fence_before();
            fence_proxy_async_smem();
            asm volatile("bar.sync 1, 256;" ::: "memory");  // staging complete, accumulators read
            if (lane == 0) mbar_arrive(&acc_empty[ab]);
            if (warp == 4 && lane == 0) {
                const int row0 = c.blk * kBlk;
#pragma unroll
                for (int h2 = 0; h2 < (KV ? 2 : 1); ++h2) {
                    const int sec2 = KV ? (h2 == 0 ? 2 : 1) : 0;
#pragma unroll
                    for (int kb = 0; kb < D / 64; ++kb)
                        tma_store_4d(&tmDQKV, sOut + h2 * C::kTile + kb * (kBlk * 128), kb * 64, row0, sec2 * a.H + c.head,
                                     c.bi);
                }
                tma_store_commit();
                if (!C::kTs) tma_store_wait_read();  // the staging is the P / dS buffers of the next step
            }
            if (!C::kTs) asm volatile("bar.sync 1, 256;" ::: "memory");
            if (a.col_part != nullptr) {
#pragma unroll
                for (int cc = 0; cc < kCols / 32; ++cc) a.col_part[prow * (3 * a.h) + colbase + cc * 32 + lane] = cp_old[cc];
            }
            bw_next<KV>(a, c);
        }
        if (warp == 4 && lane == 0) tma_store_wait_all();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
    if (!KV) asm volatile("griddepcontrol.wait;" ::: "memory");  // see the prologue
}

// D[b][H][q] = τ · sum_dd dO[q][hh*d+dd] * O[q][hh*d+dd] (τ = 1/sqrt(d), the score scale the
// backward's dS = τ P (dP - D) needs, applied once here): one warp per token row,
// coalesced 16-byte loads over the whole row, per-head sums reduced across the
// d/8 lanes that hold a head (fixed shuffle order: deterministic).
template <int D>
__global__ void __launch_bounds__(128) attn_bwd_dot_kernel(const __nv_bfloat16* __restrict__ dO,
                                                           const __nv_bfloat16* __restrict__ O,
                                                           float* __restrict__ dsum, int rows, int s, int H,
                                                           float tau) {
    pdl_begin();
    constexpr int kLanesPerHead = D / 8;
    const int row = blockIdx.x * 4 + threadIdx.x / 32;  // 4 rows per block: fine-grained SM balance
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    const int chunks = H * kLanesPerHead;  // 16-byte chunks per row
    const int64_t off = static_cast<int64_t>(row) * H * D;
    const int bi = row / s, q = row % s;
    constexpr int kIn = 8;  // 16-byte chunk pairs per lane in flight (all loads first, then the math)
    for (int base = 0; base < chunks; base += 32 * kIn) {
        uint4 ua[kIn], ub[kIn];
#pragma unroll
        for (int u = 0; u < kIn; ++u) {
            const int ci = base + u * 32 + lane;
            if (ci < chunks) {
                ua[u] = *reinterpret_cast<const uint4*>(dO + off + ci * 8);
                ub[u] = *reinterpret_cast<const uint4*>(O + off + ci * 8);
            }
        }
#pragma unroll
        for (int u = 0; u < kIn; ++u) {
            const int ci = base + u * 32 + lane;
            if (base + u * 32 >= chunks) break;  // warp-uniform
            float acc = 0.f;
            if (ci < chunks) {
                const __nv_bfloat162* ha = reinterpret_cast<const __nv_bfloat162*>(&ua[u]);
                const __nv_bfloat162* hb = reinterpret_cast<const __nv_bfloat162*>(&ub[u]);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float2 x = __bfloat1622float2(ha[e]), y = __bfloat1622float2(hb[e]);
                    acc += x.x * y.x + x.y * y.y;
                }
            }
#pragma unroll
            for (int o = 1; o < kLanesPerHead; o <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (ci < chunks && (lane % kLanesPerHead) == 0) {
                const int head = ci / kLanesPerHead;
                dsum[(static_cast<int64_t>(bi) * H + head) * s + q] = acc * tau;
            }
        }
    }
}

// dO [b*s][H*d] viewed as dims {d, s, H, b}, box {64, 128}.
cudaError_t do_map(CUtensorMap* m, const void* dO, int b, int s, int H, int d) {
    EncodeTiledFn enc = encode_fn();
    if (!enc) return cudaErrorNotSupported;
    const int64_t h = static_cast<int64_t>(H) * d;
    cuuint64_t dims[4] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(s), static_cast<cuuint64_t>(H),
                          static_cast<cuuint64_t>(b)};
    cuuint64_t strides[3] = {static_cast<cuuint64_t>(h * 2), static_cast<cuuint64_t>(d * 2),
                             static_cast<cuuint64_t>(s * h * 2)};
    cuuint32_t box[4] = {64, static_cast<cuuint32_t>(kBlk), 1, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(dO), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int D, bool KV>
cudaError_t launch_bwd(const FlashBwdPlan& p, cudaStream_t st) {
    using C = BwCfg<D, KV>;
    static bool attr = false;
    if (!attr) {
        cudaError_t e =
            cudaFuncSetAttribute(flash_bwd_kernel<D, KV>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    BwArgs a{p.dqkv, p.col_part, p.lse, p.dsum, p.s, p.H, p.H * p.d, p.b, p.scale_log2, 1.f / sqrtf(static_cast<float>(p.d)),
             p.causal};
    const int tiles = p.s / kBlk * p.H * p.b;
    const int grid = tiles < sm_count() ? tiles : sm_count();
    return launch_kernel(flash_bwd_kernel<D, KV>, grid, kThreads, C::kSmem, st, 1, p.tmQKV, p.tmDO, p.tmDQKV, a);
}

}  // namespace

cudaError_t flash_bwd_prepare(const void* qkv, const void* o, const void* dO, const float* lse, float* dsum,
                              void* dqkv, int b, int s, int H, int d, FlashBwdPlan* p, int causal) {
    if ((d != 64 && d != 128) || s % kBlk) return cudaErrorInvalidValue;
    cudaError_t e = qkv_map(&p->tmQKV, qkv, b, s, H, d, kBlk);
    if (e != cudaSuccess) return e;
    e = do_map(&p->tmDO, dO, b, s, H, d);
    if (e != cudaSuccess) return e;
    e = qkv_map(&p->tmDQKV, dqkv, b, s, H, d, kBlk);
    if (e != cudaSuccess) return e;
    p->o = static_cast<const __nv_bfloat16*>(o);
    p->dO = static_cast<const __nv_bfloat16*>(dO);
    p->lse = lse;
    p->dsum = dsum;
    p->dqkv = static_cast<__nv_bfloat16*>(dqkv);
    p->b = b;
    p->s = s;
    p->H = H;
    p->d = d;
    p->scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(d));
    p->causal = causal;
    return cudaSuccess;
}

cudaError_t flash_backward(const FlashBwdPlan& p, cudaStream_t st) {
    const int rows = p.b * p.s;
    cudaError_t e;
    if (p.d == 64)
        e = launch_kernel(attn_bwd_dot_kernel<64>, (rows + 3) / 4, 128, 0, st, 1, p.dO, p.o, p.dsum, rows, p.s, p.H,
                          1.f / sqrtf(64.f));
    else
        e = launch_kernel(attn_bwd_dot_kernel<128>, (rows + 3) / 4, 128, 0, st, 1, p.dO, p.o, p.dsum, rows, p.s, p.H,
                          1.f / sqrtf(128.f));
    if (e != cudaSuccess) return e;
    e = p.d == 64 ? launch_bwd<64, true>(p, st) : launch_bwd<128, true>(p, st);
    if (e != cudaSuccess) return e;
    return p.d == 64 ? launch_bwd<64, false>(p, st) : launch_bwd<128, false>(p, st);
}

void preload_attention_kernels() {
    preload_module_of(reinterpret_cast<const void*>(&flash_fwd_kernel<64, kFwdNQ>));
}

}  // namespace ptk
