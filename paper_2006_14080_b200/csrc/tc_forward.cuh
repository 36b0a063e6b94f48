// Forward NUDFT kernels on tcgen05 (kd = F x): the SS form for large
// images and the persistent TMEM-resident (A-stationary) form, plus the
// k-space fold of the SS form.  See tc_common.cuh for the layouts.
#pragma once

#include "tc_common.cuh"

namespace csr {

// MMA issue from a whole warp with one elected lane (FWD_ELECT, default):
// warp-uniform descriptors let ptxas issue UTCHMMA without the per-lane
// waterfall loop it wraps around an MMA issued under lane == 0
#ifndef FWD_ELECT
#define FWD_ELECT 1
#endif
__device__ __forceinline__ bool fwd_one() { return FWD_ELECT ? sm100::elect_one() : true; }

struct FwdParams {
    unsigned long long *probe;  // live timing slot (probe_enter/exit) or null
    TcArgs a;
    int mt_per_frame, nt_per_group;
    int amax;  // 1: kdp aliases the k-space buffer; atomicMax |kd| into scales[5]
    const float2 *p0p;
    float2 *kdp;  // [G][T][Mk][Cp]
    const float *scales;
    const int *gate;
    int exp_flags;  // profiling (debug builds, CSR_FEXP): 1 no MMA, 2 no TMA, 4 no drain
};


// CL = 2: a CTA pair (cta_group::2) on two consecutive sample tiles of the
// same frame: M = 256 pair MMAs, each CTA's shared memory holds its 128
// sample rows of A and HALF (128) of the 256 doubled image rows of B, so the
// shared-memory traffic per SM per K block drops from 96 KiB of TMA writes
// + 32 KiB of MMA reads per K16 to 64 + 20 KiB — the single-CTA form is
// bound by that port (tools/mma_micro.cu: 14970 vs 12570 cycles per
// 128 x 128 x 256 complex tile, MMA floor 12288).  The leader (rank 0)
// issues the MMAs; both CTAs' TMA loads complete on the leader's `full`
// barrier (cta_group::2 form); MMA commits are multicast onto both CTAs'
// `empty` / `tfull` barriers; each epilogue releases an accumulator on its
// own CTA's `tempty`, and the peer's idle MMA lane relays the peer's
// releases to the leader's `tempty_p` with relaxed cluster arrives.  Three
// 64 KiB stages per CTA.
constexpr int FWD_PAIR_STAGE = 2 * TC_A_TILE + TC_B_TILE;  // A hi/lo + B hi/lo halves
constexpr int FWD_PAIR_STAGES = 3;
static_assert(FWD_PAIR_STAGES * FWD_PAIR_STAGE <= TC_STAGES * TC_FWD_OPS, "pair stages fit");
template <int CP, int CL>
__global__ void __launch_bounds__(TC_FWD_THREADS, 1)
    k_tc_forward(const __grid_constant__ CUtensorMap tmA_hi,
                 const __grid_constant__ CUtensorMap tmA_lo,
                 const __grid_constant__ CUtensorMap tmB_hi,
                 const __grid_constant__ CUtensorMap tmB_lo, FwdParams P) {
    pdl_enter();
    using namespace sm100;
    // (the gate is uniform over the grid, so a pair leaves together)
    if (P.gate && !*P.gate) return;
    probe_enter(P.probe);
    constexpr bool PAIR = CL > 1;
    constexpr int STAGE = PAIR ? FWD_PAIR_STAGE : TC_FWD_OPS;
    constexpr int NSTG = PAIR ? FWD_PAIR_STAGES : TC_STAGES;
    constexpr int BH = PAIR ? TC_B_TILE / 2 : TC_B_TILE;  // B bytes (hi or lo) per CTA
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = align1024(smem_raw);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + TC_STAGES * TC_FWD_OPS);
    uint64_t *empty = full + NSTG;
    uint64_t *tfull = empty + NSTG;
    uint64_t *tempty = tfull + 2;
    uint64_t *tempty_p = tempty + 2;  // (PAIR, leader) the peer's accumulator drains
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty_p + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int mtile = blockIdx.x;
    const int t = mtile / P.mt_per_frame;
    const int nt0 = blockIdx.y * P.nt_per_group, nt1 = nt0 + P.nt_per_group;
    const int nkb = P.a.Kf / 64;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tmA_hi);
        tma_prefetch(&tmA_lo);
        tma_prefetch(&tmB_hi);
        tma_prefetch(&tmB_lo);
        for (int s = 0; s < NSTG; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 4);
            mbar_init(&tempty_p[i], 1);
        }
        if (PAIR) fence_barrier_init_cluster();
        else fence_barrier_init();
    }
    if (warp == 1) {
        if (PAIR) tmem_alloc_pair(tmem_slot, 512);
        else tmem_alloc(tmem_slot, 512);
    }
    tc_fence_before();
    __syncthreads();
    if (PAIR) cluster_sync();  // the leader's barriers exist before any remote use
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t crank = PAIR ? cluster_ctarank() : 0;

    if (warp == 0) {
        if (lane == 0) {
            // the leader's stage barriers (shared::cluster addresses)
            const uint32_t lead_full = PAIR ? mapa_shared(smem_u32(full), 0) : 0;
            int it = 0;
            for (int nt = nt0; nt < nt1; ++nt) {
                const int brow = t * P.a.Nf + nt * TC_BN;
                for (int kb = 0; kb < nkb; ++kb, ++it) {
                    const int s = it % NSTG;
                    const uint32_t ph = (it / NSTG) & 1;
                    mbar_wait(&empty[s], ph ^ 1);
                    uint8_t *st = smem + s * STAGE;
                    if (P.exp_flags & 2) {
                        if (crank == 0) mbar_arrive(&full[s]);
                        continue;
                    }
                    if (!PAIR) {
                        mbar_arrive_expect_tx(&full[s], TC_FWD_OPS);
                        tma_load_2d(st, &tmA_hi, &full[s], kb * 64, mtile * TC_BM);
                        tma_load_2d(st + TC_A_TILE, &tmA_lo, &full[s], kb * 64, mtile * TC_BM);
                        tma_load_2d(st + 2 * TC_A_TILE, &tmB_hi, &full[s], kb * 64, brow);
                        tma_load_2d(st + 2 * TC_A_TILE + TC_B_TILE, &tmB_lo, &full[s], kb * 64, brow);
                    } else {
                        // the leader arms its barrier for both CTAs' bytes (the
                        // peer's copies may complete first: tx-count goes
                        // transiently negative within the phase)
                        if (crank == 0) mbar_arrive_expect_tx(&full[s], CL * STAGE);
                        const uint32_t fb = lead_full + s * 8;
                        const int bro = brow + (int)crank * (TC_BN / 2);
                        tma_load_2d_pair(st, &tmA_hi, fb, kb * 64, mtile * TC_BM);
                        tma_load_2d_pair(st + TC_A_TILE, &tmA_lo, fb, kb * 64, mtile * TC_BM);
                        tma_load_2d_pair(st + 2 * TC_A_TILE, &tmB_hi, fb, kb * 64, bro);
                        tma_load_2d_pair(st + 2 * TC_A_TILE + BH, &tmB_lo, fb, kb * 64, bro);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (PAIR && crank != 0 && lane == 0) {
            // the peer's idle MMA lane relays its epilogue's accumulator
            // releases to the leader (relaxed cluster arrive, see
            // tc_adjoint_w.cuh: a release.cluster arrive costs ~2000 cycles)
            const uint32_t lead_tp = mapa_shared(smem_u32(tempty_p), 0);
            int tc = 0;
            for (int nt = nt0; nt < nt1; ++nt, ++tc) {
                const int ab = tc & 1;
                mbar_wait(&tempty[ab], (tc >> 1) & 1);
                mbar_arrive_cluster_relaxed(lead_tp + ab * 8);
            }
        }
        // MMA issue: lane 0 of the (leader) CTA
        if (lane == 0 && crank == 0) {
            constexpr uint32_t idesc = idesc_f16(TC_BM * CL, TC_BN);
            int it = 0, tc = 0;
            for (int nt = nt0; nt < nt1; ++nt, ++tc) {
                const int ab = tc & 1;
                const uint32_t aph = (tc >> 1) & 1;
                mbar_wait(&tempty[ab], aph ^ 1);
                if (PAIR) mbar_wait(&tempty_p[ab], aph ^ 1);
                tc_fence_after();
                const uint32_t dcol = tmem + ab * TC_BN;
                for (int kb = 0; kb < nkb; ++kb, ++it) {
                    const int s = it % NSTG;
                    const uint32_t ph = (it / NSTG) & 1;
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    const uint32_t st = smem_u32(smem + s * STAGE);
                    const uint32_t a_hi = st, a_lo = st + TC_A_TILE;
                    const uint32_t b_hi = st + 2 * TC_A_TILE, b_lo = b_hi + BH;
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        if (P.exp_flags & 1) break;
                        const uint32_t o = kk * 32;
                        const uint64_t dah = desc_sw128(a_hi + o), dal = desc_sw128(a_lo + o);
                        const uint64_t dbh = desc_sw128(b_hi + o), dbl = desc_sw128(b_lo + o);
                        if (PAIR) {
                            mma_f16_pair<1>(dcol, dah, dbh, idesc, (kb | kk) != 0);
                            mma_f16_pair<2>(dcol, dah, dbl, idesc, 1);
                            mma_f16_pair<0>(dcol, dal, dbh, idesc, 1);
                        } else {
                            mma_f16_fill(dcol, dah, dbh, idesc, (kb | kk) != 0);
                            mma_f16_lastuse(dcol, dah, dbl, idesc, 1);
                            mma_f16(dcol, dal, dbh, idesc, 1);
                        }
                    }
                    if (PAIR) mma_commit_pair_mc(&empty[s], (uint16_t)((1u << CL) - 1));
                    else mma_commit(&empty[s]);
                }
                if (PAIR) mma_commit_pair_mc(&tfull[ab], (uint16_t)((1u << CL) - 1));
                else mma_commit(&tfull[ab]);
            }
        }
    } else {
        // epilogue: warps 2..5, TMEM lane quarter = warp % 4
        const int q = warp & 3;
        const int row = q * 32 + lane;
        const int64_t kloc = (int64_t)(mtile % P.mt_per_frame) * TC_BM + row;
        const bool valid = kloc < P.a.M;
        const float2 *p0row = P.p0p + ((int64_t)t * P.a.Mk + kloc) * P.a.nxp;
        constexpr int U = CP > 16 ? CP / 16 : 1;
        float2 acc[CP];
#pragma unroll
        for (int c = 0; c < CP; ++c) acc[c] = make_float2(0.f, 0.f);
        int tc = 0;
        for (int nt = nt0; nt < nt1; ++nt, ++tc) {
            const int ab = tc & 1;
            const uint32_t aph = (tc >> 1) & 1;
            mbar_wait(&tfull[ab], aph);
            tc_fence_after();
            const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + ab * TC_BN;
            const int xbase = nt * P.a.xs;
            for (int chb = (P.exp_flags & 4) ? 8 : 0; chb < 8; chb += U) {
                float2 p0v[16 * U / CP > 0 ? 16 * U / CP : 1];
#pragma unroll
                for (int i = 0; i < 16 * U / CP; ++i) {
                    const int x = xbase + (chb * 16) / CP + i;
                    p0v[i] = valid ? p0row[x] : make_float2(0.f, 0.f);
                }
#pragma unroll
                for (int h = 0; h < U; ++h) {
                    uint32_t r[32];
                    tmem_ld32(taddr + (chb + h) * 32, r);
                    tmem_ld_wait();
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj) {
                        const int jl = h * 16 + jj;
                        const float2 gv = make_float2(__uint_as_float(r[2 * jj]),
                                                      __uint_as_float(r[2 * jj + 1]));
                        cfma(acc[jl % CP], p0v[jl / CP], gv);
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[ab]);  // (PAIR: the peer's is relayed)
        }
        if (P.amax) {  // max|kd| for the adjoint's operand scale (order-free)
            float mx = 0.f;
            const float inv = 1.f / pow2_scale(2.f * P.scales[4] * P.scales[6]);
#pragma unroll
            for (int c = 0; c < CP; ++c)
                mx = fmaxf(mx, fmaxf(fabsf(acc[c].x * inv), fabsf(acc[c].y * inv)));
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            if (lane == 0) atomicMax(reinterpret_cast<unsigned *>(const_cast<float *>(P.scales) + 5),
                                     __float_as_uint(mx));
        }
        if (valid) {
            const float inv = 1.f / pow2_scale(2.f * P.scales[4] * P.scales[6]);
            float2 *out = P.kdp + (((int64_t)blockIdx.y * P.a.T + t) * P.a.Mk + kloc) * CP;
#pragma unroll
            for (int c = 0; c < CP; ++c) out[c] = make_float2(acc[c].x * inv, acc[c].y * inv);
        }
    }
    __syncthreads();
    probe_exit(P.probe);
    // no CTA of a pair leaves while the leader's MMAs / commits may still
    // touch the peer (its shared memory, barriers and tensor memory)
    if (PAIR) cluster_sync();
    if (warp == 1) {
        tc_fence_after();
        if (PAIR) tmem_dealloc_pair(tmem, 512);
        else tmem_dealloc(tmem, 512);
    }
}

// Forward, A-stationary form (2*nyp <= 256), persistent.  The work is the
// list of (sample tile m, N tile n) units, m-major, with N tiles of 256
// doubled image rows (128 complex (x, c) columns): one N = 256 MMA per K
// step and operand runs at ~3300 MACs/clk/SM against ~2700 for N = 128
// (tools/pipe_micro.cu).  CTA b of the grid (one per SM) takes the
// contiguous range [b*U/G, (b+1)*U/G), i.e. one or more segments of N tiles
// of consecutive sample tiles.  Per segment the 128 samples' P1 rows (A,
// fp16 hi/lo) are loaded into TMEM once (lane-major copy: coalesced) while
// the image operand X' streams through a TMA ring; MMAs read A from TMEM
// and only B from shared memory.  The single 256-column accumulator is
// drained by sixteen epilogue warps (four per TMEM lane quarter, one per
// 64-column quarter) straight into registers, so the tensor core waits only
// for the TMEM reads; the row-dot `kd[k,c] += sum_x P0[k,x] G[k,(x,c)]`
// runs after the release.  A sample tile split across CTAs leaves one
// partial per piece; the CTA holding piece 0 sums pieces in order.
//   TMEM: [0,128) A_hi, [128,256) A_lo, [256,512) accumulator.
constexpr int FTS_STAGES = 3;
constexpr int FTS_B_TILE = 256 * 128;  // 32 KiB per hi / lo per K block (256 rows)
// PS form: A (128 rows hi / lo) and B in every stage, two stages of 96 KiB
constexpr int FPS_STAGES = 2;
constexpr int FPS_STAGE = 2 * TC_A_TILE + 2 * FTS_B_TILE;
constexpr int FTS_THREADS = 576;       // TMA, MMA, 16 epilogue (+A loader) warps

struct FwdTsParams {
    unsigned long long *probe;  // live timing slot (probe_enter/exit) or null
    TcArgs a;
    int mt_per_frame;
    int nt_tiles;    // 256-row N tiles per sample tile (Nf / 256)
    int64_t units;   // T * mt_per_frame * nt_tiles
    const uint4 *fa_hi, *fa_lo;  // lane-major: [mtile][Kf/8][128 rows] x 16 B
    const float2 *p0p;
    float2 *kdi;     // [T][Mk][Cp] (scaled result)
    float2 *kdp;     // [pieces][T][Mk][Cp] partials of split tiles
    unsigned *tick;  // [T * mt_per_frame][4] piece-ready flags (re-armed by piece 0)
    float *scales;
    const int *gate;
    int exp_flags;  // profiling: 1 no MMA, 2 no TMA, 4 no epilogue math
    unsigned long long *trace;  // optional [grid][32] globaltimer stamps
};

// unit range of CTA b and the CTA that owns unit u
__device__ __forceinline__ int64_t fts_u0(int64_t U, int G, int b) { return U * b / G; }
__device__ __forceinline__ int fts_owner(int64_t U, int G, int64_t u) {
    // largest b with U*b/G <= u
    int b = (int)((u * G) / U);
    while (b + 1 < G && fts_u0(U, G, b + 1) <= u) ++b;
    while (b > 0 && fts_u0(U, G, b) > u) --b;
    return b;
}

// PS = true: the same persistent unit walk with A (P1 rows) staged from
// shared memory next to B in every K block (TMA, SW128) instead of held in
// tensor memory, which frees TMEM for two 256-column accumulators: the
// epilogue drains unit u while the MMAs of unit u+1 run.
// PAIR (with PS): the walk runs on CTA pairs (cta_group::2, as the SS
// form): a unit is a pair of consecutive sample tiles x one 256-row N tile,
// M = 256 pair MMAs, each CTA stages its 128 sample rows of A and 128 of the
// 256 image rows of B (64 KiB stages, three of them), the leader issues.
// Unit ranges, pieces and their flags are per pair; each CTA folds and
// writes the rows of its own sample tile.
constexpr int FPP_STAGES = 3;
constexpr int FPP_STAGE = 2 * TC_A_TILE + FTS_B_TILE;  // A hi/lo + B hi/lo halves
static_assert(FPP_STAGES * FPP_STAGE <= FPS_STAGES * FPS_STAGE, "pair stages fit");
template <int CP, bool PS, bool PAIR = false>
__global__ void __launch_bounds__(FTS_THREADS, 1)
    k_tc_forward_ts(const __grid_constant__ CUtensorMap tmB_hi,
                    const __grid_constant__ CUtensorMap tmB_lo,
                    const __grid_constant__ CUtensorMap tmA_hi,
                    const __grid_constant__ CUtensorMap tmA_lo, FwdTsParams P) {
    using namespace sm100;
    // Prologue overlapped with the previous kernel (programmatic launch):
    // barrier init, TMEM allocation and the first segment's A rows read only
    // static data; everything else waits in pdl_wait().
    pdl_trigger();
    constexpr int XQ = 32 / CP;  // x values per 64-column accumulator quarter
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = align1024(smem_raw);
    // TS: one K block = [B_hi | B_lo] x 256 rows; PS: [A_hi | A_lo | B_hi | B_lo]
    // (PAIR: B halves of 128 rows)
    static_assert(!PAIR || PS, "the pair form stages A in shared memory");
    constexpr int STAGE = PAIR ? FPP_STAGE : PS ? FPS_STAGE : 2 * FTS_B_TILE;
    constexpr int NSTG = PAIR ? FPP_STAGES : PS ? FPS_STAGES : FTS_STAGES;
    constexpr int BOFF = PS ? 2 * TC_A_TILE : 0;  // B offset in a stage
    constexpr int BH = PAIR ? FTS_B_TILE / 2 : FTS_B_TILE;  // B hi (or lo) bytes per CTA
    constexpr int CL = PAIR ? 2 : 1;
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + NSTG * STAGE);
    uint64_t *empty = full + NSTG;
    uint64_t *tfull = empty + NSTG;     // [2] (PS: one per accumulator)
    uint64_t *tempty = tfull + 2;       // [2]
    uint64_t *a_ready = tempty + 2;
    uint64_t *a_free = a_ready + 1;
    uint64_t *tempty_p = a_free + 1;    // [2] (PAIR, leader) the peer's drains
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty_p + 2);
    __shared__ float2 part_acc[128][CP + 1];  // row sums folded across the quarters

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // (PAIR: G pairs, this CTA's pair `pid`, units of sample-tile pairs)
    const int G = gridDim.x / CL;
    const int pid = blockIdx.x / CL;
    const uint32_t crank = PAIR ? cluster_ctarank() : 0;
    const int64_t U = P.units;
    const int NT = P.nt_tiles;
    const int64_t u0 = fts_u0(U, G, pid), u1 = fts_u0(U, G, pid + 1);
    // sample tile (128 rows, over T * mt_per_frame) of unit-tile index m
    auto stile = [&](int64_t m) { return PAIR ? 2 * m + crank : m; };
    const int nkb = P.a.Kf / 64;
    unsigned long long *tr = P.trace ? P.trace + (size_t)blockIdx.x * 32 : nullptr;
    if (tr && threadIdx.x == 0) tr[0] = gtimer();

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tmB_hi);
        tma_prefetch(&tmB_lo);
        if (PS) {
            tma_prefetch(&tmA_hi);
            tma_prefetch(&tmA_lo);
        }
        for (int s = 0; s < NSTG; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 16);
            mbar_init(&tempty_p[b], 1);
        }
        mbar_init(a_ready, 16);
        mbar_init(a_free, 1);
        if (PAIR) fence_barrier_init_cluster();
        else fence_barrier_init();
    }
    if (warp == 1) {
        if (PAIR) tmem_alloc_pair(tmem_slot, 512);
        else tmem_alloc(tmem_slot, 512);
    }
    tc_fence_before();
    __syncthreads();
    if (PAIR) cluster_sync();  // the leader's barriers exist before any remote use
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // the leader's `full` barriers (shared::cluster) for the pair's TMA loads
    const uint32_t lead_full = PAIR ? mapa_shared(smem_u32(full), 0) : 0;
    if (tr && threadIdx.x == 0) tr[1] = gtimer();

    // A rows of sample tile m -> TMEM: the four epilogue warps of a lane
    // quarter split the row (part 0/1: hi columns, 2/3: lo columns; 16
    // chunks in flight per thread).  Lane-major factor copy: 512 contiguous
    // bytes per warp load.
    const int nchunk = P.a.Kf / 8;  // 16-byte column chunks per row (hi or lo)
    auto load_a = [&](int64_t m, uint32_t lane_base, int row, int part) {
        const uint4 *g = ((part >> 1) ? P.fa_lo : P.fa_hi) + (size_t)m * nchunk * 128 + row;
        const int half = nchunk / 2;  // chunks per part (Kf = 2*nyp, multiple of 64)
        const int c0 = (part & 1) * half;
        const uint32_t dst = lane_base + ((part >> 1) ? 128 : 0);
        for (int cc = 0; cc < half; cc += 8) {
            uint32_t vh[32];
#pragma unroll
            for (int v = 0; v < 8; ++v) {
                const uint4 a = __ldg(g + (size_t)(c0 + cc + v) * 128);
                vh[4 * v] = a.x; vh[4 * v + 1] = a.y; vh[4 * v + 2] = a.z; vh[4 * v + 3] = a.w;
            }
            tmem_st32(dst + (c0 + cc) * 4, vh);
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(a_ready);
    };
    if (!PS && warp >= 2 && u0 < u1) {
        const int q = warp & 3;
        load_a(u0 / NT, tmem + ((uint32_t)(q * 32) << 16), q * 32 + lane, (warp - 2) >> 2);
        if (tr && threadIdx.x == 64) tr[5] = gtimer();
    }
    // PS: the first stages' A tiles (static factors) are fetched before
    // pdl_wait, overlapped with the previous kernel; their B tiles after it
    const int npre = (PS && u0 < u1 && !(P.exp_flags & 2)) ? min(NSTG, nkb) : 0;
    if (PS && warp == 0 && lane == 0) {
        for (int i = 0; i < npre; ++i) {
            uint8_t *st = smem + i * STAGE;
            const int ar = (int)stile(u0 / NT) * 128;
            if (PAIR) {
                if (crank == 0) mbar_arrive_expect_tx(&full[i], CL * STAGE);
                tma_load_2d_pair(st, &tmA_hi, lead_full + i * 8, i * 64, ar);
                tma_load_2d_pair(st + TC_A_TILE, &tmA_lo, lead_full + i * 8, i * 64, ar);
            } else {
                mbar_arrive_expect_tx(&full[i], STAGE);
                tma_load_2d(st, &tmA_hi, &full[i], i * 64, ar);
                tma_load_2d(st + TC_A_TILE, &tmA_lo, &full[i], i * 64, ar);
            }
        }
    }

    pdl_wait();
    const bool run = !P.gate || *P.gate;
    if (run) probe_enter(P.probe);

    if (!run) {
        // gated off: complete the prologue's A loads (their stages expect
        // the B bytes too) before the CTA may leave
        if (npre > 0 && warp == 0 && lane == 0) {
            const int64_t m = u0 / NT, ms = stile(m);
            const int t = (int)(ms / P.mt_per_frame);
            const int brow = t * P.a.Nf + (int)(u0 - m * NT) * 256 + (int)crank * 128;
            for (int i = 0; i < npre; ++i) {
                uint8_t *st = smem + i * STAGE;
                if (PAIR) {
                    tma_load_2d_pair(st + BOFF, &tmB_hi, lead_full + i * 8, i * 64, brow);
                    tma_load_2d_pair(st + BOFF + BH, &tmB_lo, lead_full + i * 8, i * 64, brow);
                } else {
                    tma_load_2d(st + BOFF, &tmB_hi, &full[i], i * 64, brow);
                    tma_load_2d(st + BOFF + FTS_B_TILE, &tmB_lo, &full[i], i * 64, brow);
                }
                if (crank == 0) mbar_wait(&full[i], 0);
            }
        }
    } else if (warp == 0) {
        // ---- TMA producer over the CTA's units
        if (lane == 0) {
            int it = 0;
            for (int64_t u = u0; u < u1; ++u) {
                const int64_t m = u / NT;
                const int nt = (int)(u - m * NT);
                const int64_t ms = stile(m);  // this CTA's sample tile
                const int t = (int)(ms / P.mt_per_frame);
                const int brow = t * P.a.Nf + nt * 256 + (int)crank * 128;
                const int arow = (int)ms * 128;  // (T * Mk) rows of A, Mk per frame
                for (int kb = 0; kb < nkb; ++kb, ++it) {
                    const int s = it % NSTG;
                    const uint32_t ph = (it / NSTG) & 1;
                    uint8_t *st = smem + s * STAGE;
                    if (PAIR) {
                        const uint32_t fb = lead_full + s * 8;
                        if (it >= npre) {
                            mbar_wait(&empty[s], ph ^ 1);
                            if (crank == 0) mbar_arrive_expect_tx(&full[s], CL * STAGE);
                            tma_load_2d_pair(st, &tmA_hi, fb, kb * 64, arow);
                            tma_load_2d_pair(st + TC_A_TILE, &tmA_lo, fb, kb * 64, arow);
                        }
                        tma_load_2d_pair(st + BOFF, &tmB_hi, fb, kb * 64, brow);
                        tma_load_2d_pair(st + BOFF + BH, &tmB_lo, fb, kb * 64, brow);
                        continue;
                    }
                    if (it < npre) {  // A already in flight (prologue)
                        tma_load_2d(st + BOFF, &tmB_hi, &full[s], kb * 64, brow);
                        tma_load_2d(st + BOFF + FTS_B_TILE, &tmB_lo, &full[s], kb * 64, brow);
                        continue;
                    }
                    mbar_wait(&empty[s], ph ^ 1);
                    mbar_arrive_expect_tx(&full[s], (P.exp_flags & 2) ? 0 : STAGE);
                    if (!(P.exp_flags & 2)) {
                        if (PS) {
                            tma_load_2d(st, &tmA_hi, &full[s], kb * 64, arow);
                            tma_load_2d(st + TC_A_TILE, &tmA_lo, &full[s], kb * 64, arow);
                        }
                        tma_load_2d(st + BOFF, &tmB_hi, &full[s], kb * 64, brow);
                        tma_load_2d(st + BOFF + FTS_B_TILE, &tmB_lo, &full[s], kb * 64, brow);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (PAIR && crank != 0 && lane == 0) {
            // the peer's idle MMA lane relays its epilogue's accumulator
            // releases to the leader (relaxed cluster arrive)
            const uint32_t lead_tp = mapa_shared(smem_u32(tempty_p), 0);
            int tc = 0;
            for (int64_t u = u0; u < u1; ++u, ++tc) {
                const int ab = tc & 1;
                mbar_wait(&tempty[ab], (tc >> 1) & 1);
                mbar_arrive_cluster_relaxed(lead_tp + ab * 8);
            }
        }
        // ---- MMA issuer (the pair's leader): the whole warp runs the loop,
        // one elected lane issues (FWD_ELECT)
        if (crank == 0 && (FWD_ELECT || lane == 0)) {
            constexpr uint32_t idesc = idesc_f16(128 * CL, 256);
            const uint32_t a_hi = tmem, a_lo = tmem + 128, dcol = tmem + 256;
            int it = 0, tc = 0, seg = 0;
            int64_t m_prev = -1;
            for (int64_t u = u0; u < u1; ++u, ++tc) {
                const int64_t m = u / NT;
                if (!PS && m != m_prev) {  // new segment: wait for its A
                    if (m_prev >= 0 && fwd_one()) mma_commit(a_free);  // old A is free after these MMAs
                    if (FWD_ELECT) __syncwarp();
                    mbar_wait(a_ready, seg & 1);
                    tc_fence_after();
                    if (tr && seg < 2 && lane == 0) tr[2 + seg * 4] = gtimer();
                    ++seg;
                    m_prev = m;
                }
                // PS: accumulator ab = tc & 1 (its drain two units ago); TS:
                // the single accumulator (the epilogue has read the last unit)
                const int ab = PS ? (tc & 1) : 0;
                const uint32_t tph = PS ? (((tc >> 1) & 1) ^ 1) : ((tc & 1) ^ 1);
                mbar_wait(&tempty[ab], tph);
                if (PAIR) mbar_wait(&tempty_p[ab], tph);
                tc_fence_after();
                const uint32_t dacc = PS ? tmem + ab * 256 : dcol;
                for (int kb = 0; kb < nkb; ++kb, ++it) {
                    const int s = it % NSTG;
                    const uint32_t ph = (it / NSTG) & 1;
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    const uint32_t st = smem_u32(smem + s * STAGE);
                    if (fwd_one()) {
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk) {
                            const uint32_t ac = kb * 32 + kk * 8;
                            const uint64_t dbh = desc_sw128(st + BOFF + kk * 32);
                            const uint64_t dbl = desc_sw128(st + BOFF + BH + kk * 32);
                            if (P.exp_flags & 1) continue;
                            if (PAIR) {
                                const uint64_t dah = desc_sw128(st + kk * 32);
                                const uint64_t dal = desc_sw128(st + TC_A_TILE + kk * 32);
                                mma_f16_pair<1>(dacc, dah, dbh, idesc, (kb | kk) != 0);
                                mma_f16_pair<2>(dacc, dah, dbl, idesc, 1);
                                mma_f16_pair<0>(dacc, dal, dbh, idesc, 1);
                            } else if (PS) {
                                const uint64_t dah = desc_sw128(st + kk * 32);
                                const uint64_t dal = desc_sw128(st + TC_A_TILE + kk * 32);
                                mma_f16_fill(dacc, dah, dbh, idesc, (kb | kk) != 0);
                                mma_f16_lastuse(dacc, dah, dbl, idesc, 1);
                                mma_f16(dacc, dal, dbh, idesc, 1);
                            } else {
                                mma_f16_ts(dcol, a_hi + ac, dbh, idesc, (kb | kk) != 0);
                                mma_f16_ts(dcol, a_hi + ac, dbl, idesc, 1);
                                mma_f16_ts(dcol, a_lo + ac, dbh, idesc, 1);
                            }
                        }
                        if (PAIR) mma_commit_pair_mc(&empty[s], 3);
                        else mma_commit(&empty[s]);
                    }
                    if (FWD_ELECT) __syncwarp();
                }
                if (fwd_one()) {
                    if (PAIR) mma_commit_pair_mc(&tfull[ab], 3);
                    else mma_commit(&tfull[ab]);
                }
                if (FWD_ELECT) __syncwarp();
                if (tr && tc < 8 && lane == 0) tr[16 + tc] = gtimer();
            }
            if (tr && lane == 0) tr[3] = gtimer();
        }
    } else {
        // ---- epilogue warps 2..17: lane quarter q, accumulator quarter qt
        const int q = warp & 3;
        const int qt = (warp - 2) >> 2;
        const int row = q * 32 + lane;
        const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
        const float inv = 1.f / pow2_scale(2.f * P.scales[4] * P.scales[6]);
        const int64_t Mk = P.a.Mk;
        int tc = 0, seg = 0;
        for (int64_t us = u0; us < u1; ++seg) {
            const int64_t m = us / NT;            // unit tile (PAIR: tile pair)
            const int64_t ue = min(u1, (m + 1) * NT);
            const int64_t ms = stile(m);          // this CTA's sample tile
            const int t = (int)(ms / P.mt_per_frame);
            const bool last_seg = ue == u1;
            const int64_t kloc = (int64_t)(ms % P.mt_per_frame) * 128 + row;
            const bool valid = kloc < P.a.M;
            const float2 *p0row = P.p0p + ((int64_t)t * Mk + kloc) * P.a.nxp;
            const int b_first = fts_owner(U, G, m * NT);
            const int b_last = fts_owner(U, G, (m + 1) * NT - 1);
            const int npieces = b_last - b_first + 1;
            const int piece = pid - b_first;
            const int64_t grow = (int64_t)t * Mk + kloc;
            float2 acc[CP];
#pragma unroll
            for (int c = 0; c < CP; ++c) acc[c] = make_float2(0.f, 0.f);
            for (int64_t u = us; u < ue; ++u, ++tc) {
                const int nt = (int)(u - m * NT);
                // this quarter's P0 values: complex columns [qt*32, qt*32+32)
                float2 p0v[XQ];
                const int xbase = (nt * 4 + qt) * XQ;
#pragma unroll
                for (int i = 0; i < XQ; ++i)
                    p0v[i] = valid ? p0row[xbase + i] : make_float2(0.f, 0.f);
                if (!PS && u + 1 == ue && !last_seg) {
                    // the segment's last unit: load the next segment's A as
                    // soon as the MMAs release the old one (the accumulator
                    // stays put meanwhile)
                    mbar_wait(a_free, seg & 1);
                    tc_fence_after();
                    load_a(ue / NT, lane_base, row, qt);
                }
                if (u + 1 == ue && piece == 0 && npieces > 1 && qt == 0) {
                    for (int pc = 1; pc < npieces; ++pc) {
                        unsigned f = 0;
                        const unsigned *flag = P.tick + ms * 4 + pc;
                        do {
                            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];"
                                         : "=r"(f) : "l"(flag) : "memory");
                        } while (f == 0u);
                    }
                }
                const int ab = PS ? (tc & 1) : 0;
                mbar_wait(&tfull[ab], PS ? ((tc >> 1) & 1) : (tc & 1));
                tc_fence_after();
                const uint32_t dbase = lane_base + (PS ? ab * 256 : 256);
                // this quarter (64 columns) in two 32-column reads; the
                // accumulator is released right after the second read
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    uint32_t r[32];
                    tmem_ld32(dbase + qt * 64 + hh * 32, r);
                    tmem_ld_wait();
                    if (hh == 1) {
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&tempty[ab]);  // (PAIR: relayed)
                    }
                    if (!(P.exp_flags & 4)) {
#pragma unroll
                        for (int jj = 0; jj < 16; ++jj) {  // complex column in the quarter
                            const int j = hh * 16 + jj;
                            const float2 gv = make_float2(__uint_as_float(r[2 * jj]),
                                                          __uint_as_float(r[2 * jj + 1]));
                            cfma(acc[j % CP], p0v[j / CP], gv);
                        }
                    }
                }
                if (tr && threadIdx.x == 64 && tc < 8) tr[24 + tc] = gtimer();
            }
            // ---- fold the four quarters (same rows) in quarter order, then
            // finish the segment: piece 0 sums pieces 0, 1, ... in order
#pragma unroll 1
            for (int src = 1; src < 4; ++src) {
                asm volatile("bar.sync 1, 512;" ::: "memory");
                if (qt == src) {
#pragma unroll
                    for (int c = 0; c < CP; ++c) part_acc[row][c] = acc[c];
                }
                asm volatile("bar.sync 1, 512;" ::: "memory");
                if (qt == 0) {
#pragma unroll
                    for (int c = 0; c < CP; ++c) acc[c] = cadd(acc[c], part_acc[row][c]);
                }
            }
            if (qt == 0) {
                if (piece > 0) {
                    float2 *mine = P.kdp + ((int64_t)(piece - 1) * P.a.T * Mk + grow) * CP;
#pragma unroll
                    for (int c = 0; c < CP; ++c) mine[c] = acc[c];
                    __threadfence();
                    asm volatile("bar.sync 2, 128;" ::: "memory");
                    if (threadIdx.x == 64) {
                        asm volatile("st.release.gpu.global.u32 [%0], %1;"
                                     ::"l"(P.tick + ms * 4 + piece), "r"(1u) : "memory");
                    }
                } else {
                    for (int pc = 1; pc < npieces; ++pc) {
                        const float2 *src = P.kdp + ((int64_t)(pc - 1) * P.a.T * Mk + grow) * CP;
#pragma unroll
                        for (int c = 0; c < CP; ++c) acc[c] = cadd(acc[c], __ldcg(src + c));
                    }
                    if (npieces > 1) {
                        asm volatile("bar.sync 2, 128;" ::: "memory");
                        if (threadIdx.x < 64 + npieces - 1 && threadIdx.x >= 64)
                            P.tick[ms * 4 + 1 + (threadIdx.x - 64)] = 0u;  // re-arm
                    }
                    float mx = 0.f;
#pragma unroll
                    for (int c = 0; c < CP; ++c)
                        mx = fmaxf(mx, fmaxf(fabsf(acc[c].x * inv), fabsf(acc[c].y * inv)));
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                    if (lane == 0) atomicMax(reinterpret_cast<unsigned *>(P.scales + 5), __float_as_uint(mx));
                    if (valid) {
                        float2 *out = P.kdi + grow * CP;
#pragma unroll
                        for (int c = 0; c < CP; ++c) out[c] = make_float2(acc[c].x * inv, acc[c].y * inv);
                    }
                }
            }
            us = ue;
        }
        if (tr && threadIdx.x == 64) tr[4] = gtimer();
    }
    __syncthreads();
    if (run) probe_exit(P.probe);
    // no CTA of a pair leaves while the leader's MMAs / commits may still
    // touch the peer
    if (PAIR) cluster_sync();
    if (warp == 1) {
        tc_fence_after();
        if (PAIR) tmem_dealloc_pair(tmem, 512);
        else tmem_dealloc(tmem, 512);
    }
}

// kd = sum_g kdp[g]; writes the internal padded layout (and optionally a
// user (T*M, C) layout); sigma_d from max|kd|
// launched with <= 3 blocks per SM (one wave)
__global__ void __launch_bounds__(256, 3) k_tc_sum_kd(TcArgs a, int G, const float2 *__restrict__ kdp, float2 *kdi,
                            float2 *user, double *partials, unsigned *ticket, float *scales,
                            const int *gate) {
    pdl_enter();
    if (gate && !*gate) return;
    int64_t total = (int64_t)a.T * a.Mk * a.Cp;
    int64_t gstride = total;
    float v = 0.f;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int c = (int)(i % a.Cp);
        int64_t r = i / a.Cp;
        int64_t k = r % a.Mk;
        int t = (int)(r / a.Mk);
        float2 s = make_float2(0.f, 0.f);
        if (k < a.M && c < a.C) {
            for (int g = 0; g < G; ++g) s = cadd(s, kdp[g * gstride + i]);
            v = fmaxf(v, fmaxf(fabsf(s.x), fabsf(s.y)));
            if (user) user[((int64_t)t * a.M + k) * a.C + c] = s;
        }
        if (kdi) kdi[i] = s;
    }
    float m;
    if (grid_max(v, partials, ticket, m)) scales[5] = m;
}

}  // namespace csr
