// Adjoint NUDFT kernel on tcgen05 (image = F^H d) and its k-space
// loader.  See tc_common.cuh for the layouts.
#pragma once

#include "tc_common.cuh"

namespace csr {

// user (T*M, C) k-space -> internal padded layout + sigma_d
__global__ void k_tc_load_kd(TcArgs a, const float2 *__restrict__ user, float2 *kdi,
                             double *partials, unsigned *ticket, float *scales) {
    pdl_enter();
    int64_t total = (int64_t)a.T * a.Mk * a.Cp;
    float v = 0.f;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int c = (int)(i % a.Cp);
        int64_t r = i / a.Cp;
        int64_t k = r % a.Mk;
        int t = (int)(r / a.Mk);
        float2 s = make_float2(0.f, 0.f);
        if (k < a.M && c < a.C) {
            s = user[((int64_t)t * a.M + k) * a.C + c];
            v = fmaxf(v, fmaxf(fabsf(s.x), fabsf(s.y)));
        }
        kdi[i] = s;
    }
    float m;
    if (grid_max(v, partials, ticket, m)) scales[5] = m;
}

__device__ __forceinline__ void tmem_st_n(uint32_t a, const uint32_t (&r)[32]) {
    sm100::tmem_st32(a, r);
}
__device__ __forceinline__ void tmem_st_n(uint32_t a, const uint32_t (&r)[16]) {
    sm100::tmem_st16(a, r);
}

// CTA-0 per-K-block timeline for tools/trace_adj_tl.py (-DADJ_TIMELINE=1)
#if ADJ_TIMELINE
#define ADJ_TL(slot, cond)                                                      \
    if (tr && (cond) && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && \
        i < 256)                                                                \
    tr[65536 + 4 * i + (slot)] = gtimer()
#else
#define ADJ_TL(slot, cond) \
    do {                   \
    } while (0)
#endif

struct AdjParams {
    unsigned long long *probe;  // live timing slot (probe_enter/exit) or null
    TcArgs a;
    int S, kb_per_split, kb_total, raw_bytes, n_raw, chain;
    int exp_flags;  // profiling experiments: 1 = no generator math, 2 = no MMA
    unsigned long long *trace;
    const float2 *sens;
    float2 *ws;  // [S][T][nx][ny]
    const float *scales;
    const int *gate;
};

constexpr int ADJ_STAGES = 4;             // B tiles in smem = A stages in TMEM
constexpr int ADJ_B_TILE = 128 * 128;     // 16 KiB (one of hi / lo)
constexpr int ADJ_B_STAGE = 2 * ADJ_B_TILE;
constexpr int ADJ_MAX_RAW = 8;            // generator-input ring depth (max)
// warps: 0 B-ring TMA, 1 MMA, 2 input-ring TMA, 3 input prep,
// 4 .. 4+GW-1 generators (GW / 4 per TMEM lane quarter, each writing SPW
// samples of a K block), then four epilogue warps
#ifndef ADJ_GW
#define ADJ_GW 4
#endif
// Barrier waits: the long ones (producers, epilogue) sleep on the barrier
// (ADJ_SLEEP_SLOW), the latency-critical ones (MMA issuer, generators) spin
// unless ADJ_SLEEP_FAST.
#ifndef ADJ_ELECT
#define ADJ_ELECT 1
#endif
#ifndef ADJ_SLEEP_SLOW
#define ADJ_SLEEP_SLOW 1
#endif
#ifndef ADJ_SLEEP_FAST
#define ADJ_SLEEP_FAST 0
#endif
__device__ __forceinline__ void wait_slow(uint64_t *b, uint32_t ph) {
#if ADJ_SLEEP_SLOW
    sm100::mbar_wait_sleep(b, ph);
#else
    sm100::mbar_wait(b, ph);
#endif
}
__device__ __forceinline__ void wait_fast(uint64_t *b, uint32_t ph) {
#if ADJ_SLEEP_FAST
    sm100::mbar_wait_sleep(b, ph);
#else
    sm100::mbar_wait(b, ph);
#endif
}
constexpr int ADJ_SPW = 32 * 4 / ADJ_GW;
constexpr int ADJ_W_EPI = 4 + ADJ_GW;
// epilogue warps: two per TMEM lane quarter, each draining half of the 128
// pixel rows of every chain (the drain stalls the MMAs: one accumulator pair)
constexpr int ADJ_EW = 8;
constexpr int ADJ_THREADS = (ADJ_W_EPI + ADJ_EW) * 32;
constexpr int ADJ_SUM_LD = 129;                       // padded row (floats)
constexpr int ADJ_SUM_BYTES = 128 * ADJ_SUM_LD * 4;   // fp32 sums [y][lane]
static_assert(ADJ_SUM_BYTES <= ADJ_STAGES * ADJ_B_STAGE, "sums reuse the B ring");

// Input-ring stage layout (bytes): P0 rows [32][XS] c64 | d [32][CP] c64 |
// d' [32][CP][2] c64, d' = sg * ((dr, di), (di, -dr)) so that generator row
// (x, c, part) gets its two values with two FMUL + two FFMA and no selects.
__host__ __device__ constexpr int adj_in_stage_bytes(int CP) {
    return ((32 * (64 / CP) * 8 + 32 * CP * 8 + 32 * CP * 16) + 127) / 128 * 128;
}

// Adjoint, "A from TMEM" form, one tile x one contiguous k range per CTA.
// Tile = 128 rows (x, c, part) of the generated operand W' (64 complex
// (x, c) columns) x 128 pixel rows y; K = 32 samples (64 fp16) per block.
// The generators write W' straight into tensor memory with tcgen05.st, so
// shared memory only carries the static factor conj(P1)^T (TMA, 128B
// swizzle) and the P0 / d inputs of the generators.
//
// Rings:
//   B ring   (4 smem stages): TMA (warp 0) -> MMA; freed by the MMA commit.
//   in ring  (n_raw smem stages): TMA (warp 2) -> prep (warp 3, scales and
//            rotates d into d') -> generators; freed as soon as the
//            generators hold the values in registers.
//   A ring   (4 TMEM stages): generators -> MMA; freed by the same MMA
//            commit as the B stage of that block.
// Per K step one N = 256 MMA multiplies A_hi by [B_hi ; B_lo] (one 256-row
// SW128 tile) into [D_hi | D_lo], and one N = 128 MMA adds A_lo * B_hi to
// D_lo: 8 MMA instructions per K block.  The single-thread roles share
// their SM sub-partitions with generator warps, and the warp scheduler
// favours busy ALU warps, so every generator instruction removed is MMA
// issue bandwidth regained (measured: tools/pipe_micro.cu).
//
// The k range is cut into accumulation chains of <= chain blocks (the
// tensor core truncates on every fp32 accumulate); the epilogue warps drain
// each chain into fp32 running sums held in registers and free the
// accumulator.  After the last chain the sums go to shared memory
// (transposed, over the idle B ring) and all warps combine coils into one
// split-K partial image.
//   TMEM columns: [0,128) hi*hi accumulator, [128,256) hi*lo + lo*hi
//   corrections, [256,512) four A stages of (hi 32 | lo 32).
template <int CP>
__global__ void __launch_bounds__(ADJ_THREADS, 1)
    k_tc_adjoint(const __grid_constant__ CUtensorMap tmB_hi,
                 const __grid_constant__ CUtensorMap tmB_lo,
                 const __grid_constant__ CUtensorMap tmP0,
                 const __grid_constant__ CUtensorMap tmKd, AdjParams P) {
    using namespace sm100;
    // Prologue overlapped with the forward (programmatic launch): barrier
    // init, TMEM allocation and the first B-ring stages (static factor) do
    // not depend on it; every role waits in pdl_wait() before touching kd,
    // the scales or the gate.
    pdl_trigger();
    constexpr int XS = 64 / CP;  // x values per tile
    constexpr int IN_STAGE = adj_in_stage_bytes(CP);
    constexpr int OFF_D = 32 * XS * 8, OFF_DP = OFF_D + 32 * CP * 8;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = align1024(smem_raw);
    uint8_t *in_base = smem + ADJ_STAGES * ADJ_B_STAGE;
    float *sum_s = reinterpret_cast<float *>(smem);  // after the main loop
    uint64_t *full = reinterpret_cast<uint64_t *>(in_base + P.n_raw * IN_STAGE);
    uint64_t *gen = full + ADJ_STAGES;
    uint64_t *empty = gen + ADJ_STAGES;
    uint64_t *rfull = empty + ADJ_STAGES;
    uint64_t *dfull = rfull + ADJ_MAX_RAW;
    uint64_t *rempty = dfull + ADJ_MAX_RAW;
    uint64_t *acc_full = rempty + ADJ_MAX_RAW;
    uint64_t *acc_empty = acc_full + 1;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acc_empty + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int mt = blockIdx.x, nt = blockIdx.y;
    const int t = blockIdx.z % P.a.T, s_id = blockIdx.z / P.a.T;
    const int kb0 = s_id * P.kb_per_split;
    const int kb1 = min(P.kb_total, kb0 + P.kb_per_split);
    const int nkb = kb1 - kb0;
    const int chain = P.chain;
    const int nchain = (nkb + chain - 1) / chain;
    const int NR = P.n_raw;
    unsigned long long *tr = P.trace ? P.trace + ((size_t)(blockIdx.z * gridDim.y + blockIdx.y) *
                                                   gridDim.x + blockIdx.x) * 32
                                     : nullptr;
    if (tr && threadIdx.x == 0) {
        tr[0] = gtimer();
        tr[30] = clock64();
    }

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tmB_hi);
        tma_prefetch(&tmB_lo);
        tma_prefetch(&tmP0);
        tma_prefetch(&tmKd);
        for (int s = 0; s < ADJ_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&gen[s], ADJ_GW);
            mbar_init(&empty[s], 1);
        }
        for (int r = 0; r < NR; ++r) {
            mbar_init(&rfull[r], 1);
            mbar_init(&dfull[r], 2);
            mbar_init(&rempty[r], ADJ_GW);
        }
        mbar_init(acc_full, 1);
        mbar_init(acc_empty, ADJ_EW);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // the first B stages are free by construction: fetch them right away
    const int pre = min(nkb, ADJ_STAGES);
    const int brow = t * P.a.nyA + nt * 128;
    if (warp == 0 && lane == 0) {
        for (int i = 0; i < pre; ++i) {
            uint8_t *st = smem + i * ADJ_B_STAGE;
            mbar_arrive_expect_tx(&full[i], ADJ_B_STAGE);
            tma_load_2d(st, &tmB_hi, &full[i], (kb0 + i) * 64, brow);
            tma_load_2d(st + ADJ_B_TILE, &tmB_lo, &full[i], (kb0 + i) * 64, brow);
        }
    }
    pdl_wait();
    const bool run = !P.gate || *P.gate;
    if (run) probe_enter(P.probe);

    if (!run) {
        // gated off: let the prefetched stages land before the CTA exits
        if (warp == 0 && lane == 0)
            for (int i = 0; i < pre; ++i) mbar_wait(&full[i], 0);
    } else if (warp == 0) {
        // ---- lane 0: B ring producer (conj(P1)^T hi / lo tiles); lane 1:
        // input ring producer (P0 rows of the tile's x values, and d).  Both
        // are single-thread loops that mostly sleep on their barriers.
        if (lane == 0) {
            for (int i = pre; i < nkb; ++i) {
                const int kb = kb0 + i;
                const int s = i % ADJ_STAGES;
                wait_slow(&empty[s], ((i / ADJ_STAGES) & 1) ^ 1);
                uint8_t *st = smem + s * ADJ_B_STAGE;
                mbar_arrive_expect_tx(&full[s], ADJ_B_STAGE);
                tma_load_2d(st, &tmB_hi, &full[s], kb * 64, brow);
                tma_load_2d(st + ADJ_B_TILE, &tmB_lo, &full[s], kb * 64, brow);
            }
        } else if (lane == 1) {
            const uint32_t tx = P.raw_bytes;
            for (int i = 0, r = 0, rph = 0; i < nkb; ++i) {
                const int kb = kb0 + i;
                wait_slow(&rempty[r], rph ^ 1);
                uint8_t *in = in_base + r * IN_STAGE;
                mbar_arrive_expect_tx(&rfull[r], tx);
                tma_load_3d(in, &tmP0, &rfull[r], mt * XS, kb * 32, t);
                tma_load_3d(in + OFF_D, &tmKd, &rfull[r], 0, kb * 32, t);
                if (++r == NR) {
                    r = 0;
                    rph ^= 1;
                }
            }
        }
    } else if (warp == 2 || warp == 3) {
        // ---- input prep, split between two sub-partitions (one warp would
        // make its sub-partition's generator the straggler):
        // d' = sg * ((dr, di), (di, -dr)) per (k, c)
        const float sg = pow2_scale(P.scales[5]);
        for (int i = 0, r = 0, rph = 0; i < nkb; ++i) {
            wait_slow(&rfull[r], rph);
            uint8_t *in = in_base + r * IN_STAGE;
            const float2 *d = reinterpret_cast<const float2 *>(in + OFF_D);
            float4 *dp = reinterpret_cast<float4 *>(in + OFF_DP);
#pragma unroll
            for (int e = (warp - 2) * 32 + lane; e < 32 * CP; e += 64) {
                const float2 v = d[e];
                dp[e] = make_float4(sg * v.x, sg * v.y, sg * v.y, -sg * v.x);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&dfull[r]);
            if (++r == NR) {
                r = 0;
                rph ^= 1;
            }
        }
    } else if (warp == 1) {
        // ---- MMA issuer.  ADJ_ELECT: the whole warp runs the loop and one
        // elected lane issues (warp-uniform descriptors: no per-MMA
        // waterfall); else lane 0 alone.
        if (ADJ_ELECT || lane == 0) {
            constexpr uint32_t idesc = idesc_f16(128, 128);
            constexpr uint32_t idesc256 = idesc_f16(128, 256);
            const uint32_t d_hi = tmem, d_lo = tmem + 128;
            int i = 0;
            for (int ch = 0; ch < nchain; ++ch) {
                wait_fast(acc_empty, (ch & 1) ^ 1);
                tc_fence_after();
                const int iend = min(nkb, i + chain);
                for (int i0 = i; i < iend; ++i) {
                    const int s = i % ADJ_STAGES;
                    const uint32_t ph = (i / ADJ_STAGES) & 1;
                    wait_fast(&gen[s], ph);
                    ADJ_TL(0, lane == 0);
                    wait_fast(&full[s], ph);
                    tc_fence_after();
                    const uint32_t st = smem_u32(smem + s * ADJ_B_STAGE);
                    const uint32_t a_hi = tmem + 256 + 64 * s, a_lo = a_hi + 32;
                    const bool issue = ADJ_ELECT ? elect_one() : true;
                    if (issue) {
                        if (!(P.exp_flags & 2)) {
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk) {
                                // B' = [hi_B ; lo_B] is one 256-row SW128 tile
                                const uint64_t db = desc_sw128(st + kk * 32);
                                const uint32_t acc = (i != i0) || (kk != 0);
                                mma_f16_ts(d_hi, a_hi + 8 * kk, db, idesc256, acc);
                                mma_f16_ts(d_lo, a_lo + 8 * kk, db, idesc, 1);
                            }
                        }
                        // frees B stage s (TMA) and A stage s (generators)
                        mma_commit(&empty[s]);
                    }
                    if (ADJ_ELECT) __syncwarp();
                }
                if (ADJ_ELECT ? elect_one() : true) mma_commit(acc_full);
                if (ADJ_ELECT) __syncwarp();
            }
            if (tr && lane == 0) {
                tr[1] = gtimer();
                tr[31] = clock64();
            }
        }
    } else if (warp >= 4 && warp < ADJ_W_EPI) {
        // ---- generators: lane quarter q, row m = (x, c, part), samples
        // [h*SPW, (h+1)*SPW) of every K block
        const int q = warp & 3;
        const int h = (warp - 4) >> 2;
        const int m = q * 32 + lane;
        const int j = m >> 1, part = m & 1;
        const int xl = j / CP, c = j % CP;
        const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
        for (int i = 0, r = 0, rph = 0; i < nkb; ++i) {
            const int s = i % ADJ_STAGES;
            wait_fast(&dfull[r], rph);
            ADJ_TL(1, lane == 0 && warp == 4);
            const uint8_t *in = in_base + r * IN_STAGE;
            const float2 *p0s = reinterpret_cast<const float2 *>(in);
            const float2 *dps = reinterpret_cast<const float2 *>(in + OFF_DP) + (c * 2 + part);
            uint32_t hv[ADJ_SPW], lv[ADJ_SPW];
            if ((P.exp_flags & 1) || ((P.exp_flags & (2048 << q)) != 0)) {
#pragma unroll
                for (int k = 0; k < ADJ_SPW; ++k) hv[k] = lv[k] = 0u;
            } else
#pragma unroll
            for (int kk = 0; kk < ADJ_SPW; ++kk) {
                const int k = h * ADJ_SPW + kk;
                const float2 p = p0s[k * XS + xl], u = dps[k * CP * 2];
                // Re row (part 0): (wr, -wi); Im row (part 1): (wi, wr)
                const float e0 = fmaf(p.x, u.x, p.y * u.y);
                const float e1 = fmaf(p.y, u.x, -(p.x * u.y));
                const __half2 hh = __floats2half2_rn(e0, e1);
                const float2 hf = __half22float2(hh);
                const __half2 ll = __floats2half2_rn(e0 - hf.x, e1 - hf.y);
                hv[kk] = *reinterpret_cast<const uint32_t *>(&hh);
                lv[kk] = *reinterpret_cast<const uint32_t *>(&ll);
            }
            // inputs are in registers: hand the stage back to the TMA
            __syncwarp();
            if (lane == 0) mbar_arrive(&rempty[r]);
            if (++r == NR) {
                r = 0;
                rph ^= 1;
            }
            // A stage s is free once the MMAs of block i - 4 completed
            wait_fast(&empty[s], ((i / ADJ_STAGES) & 1) ^ 1);
            ADJ_TL(2, lane == 0 && warp == 4);
            tc_fence_after();
            const uint32_t col = lane_base + 256 + 64 * s + h * ADJ_SPW;
            tmem_st_n(col, hv);
            tmem_st_n(col + 32, lv);
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&gen[s]);
            ADJ_TL(3, lane == 0 && warp == 4);
        }
    }
    float sum[64];  // epilogue warps: running sums of row m over their 64 y
    const int eh = (warp - ADJ_W_EPI) >> 2;  // which half of the y rows
    if (run && warp >= ADJ_W_EPI) {
        // ---- epilogue: drain every chain into the register sums
        const int q = warp & 3;
        const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16) + 64 * eh;
#pragma unroll
        for (int y = 0; y < 64; ++y) sum[y] = 0.f;
        for (int ch = 0; ch < nchain; ++ch) {
            wait_slow(acc_full, ch & 1);
            tc_fence_after();
#pragma unroll
            for (int cb = 0; cb < 4; ++cb) {
                uint32_t rh[16], rl[16];
                tmem_ld16(lane_base + cb * 16, rh);
                tmem_ld16(lane_base + 128 + cb * 16, rl);
                tmem_ld_wait();
                if (cb == 3) {  // this warp's accumulator columns read: let the MMA go on
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(acc_empty);
                }
#pragma unroll
                for (int yy = 0; yy < 16; ++yy)
                    sum[cb * 16 + yy] += __uint_as_float(rh[yy]) + __uint_as_float(rl[yy]);
            }
        }
    }
    __syncthreads();  // all MMAs and TMA loads are done: the B ring is free
    if (run && warp >= ADJ_W_EPI) {
        const int m = (warp & 3) * 32 + lane;
#pragma unroll
        for (int y = 0; y < 64; ++y) sum_s[(64 * eh + y) * ADJ_SUM_LD + m] = sum[y];
    }
    __syncthreads();
    // ---- combine: ws[x, y] = sum_c conj(s_c[x,y]) (re + i im)_{x,c}(y), all
    // warps: thread e handles pixel row y = e % 128 for the x values
    // xq = e / 128 (mod warps / 4) of the tile, reading the transposed sums
    // (padded rows: conflict-free) and the coil maps with y-coalesced loads
    if (run) {
        const float inv = 1.f / pow2_scale(P.scales[5]);
        const int e = threadIdx.x & 127, grp = threadIdx.x >> 7;
        const int y = nt * 128 + e;
        const int64_t nxy = (int64_t)P.a.nx * P.a.ny;
        float2 *wbase = P.ws + ((int64_t)s_id * P.a.T + t) * nxy;
        const float *row = sum_s + e * ADJ_SUM_LD;
        if (y < P.a.ny) {
            for (int xq = grp; xq < XS; xq += ADJ_THREADS / 128) {
                const int xg = mt * XS + xq;
                if (xg >= P.a.nx) break;
                float ar = 0.f, ai = 0.f;
#pragma unroll
                for (int cc = 0; cc < CP; ++cc) {
                    if (cc < P.a.C) {
                        const float re = row[2 * (xq * CP + cc)];
                        const float im = row[2 * (xq * CP + cc) + 1];
                        const float2 sv = __ldg(P.sens + (int64_t)cc * nxy +
                                                (int64_t)xg * P.a.ny + y);
                        ar += sv.x * re + sv.y * im;
                        ai += sv.x * im - sv.y * re;
                    }
                }
                wbase[(int64_t)xg * P.a.ny + y] = make_float2(ar * inv, ai * inv);
            }
        }
    }
    __syncthreads();
    if (tr && threadIdx.x == 0) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        tr[28] = gtimer();
        tr[29] = smid;
    }
    if (run) probe_exit(P.probe);
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

}  // namespace csr
