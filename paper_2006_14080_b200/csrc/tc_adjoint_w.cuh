// Wide-tile adjoint NUDFT on tcgen05 for images with 128 < ny (per y tile
// up to 256 pixel rows): one CTA covers N pixel rows y (N = 144 ... 256)
// of a 128-row (x, c, Re/Im) tile, so every generated operand value W
// feeds 3 MMAs of width N instead of two 128-wide tiles each regenerating
// it, and all MMAs run at N > 128 (the N = 128 correction MMA of
// k_tc_adjoint runs at ~70 % of the per-column rate of an N = 256 one).
//
//   per 16-deep K step:  D += A_hi B_hi ;  D += A_hi B_lo ;  D += A_lo B_hi
//
// with A = the generated W' (hi / lo, from TMEM, as k_tc_adjoint) and
// B = conj(P1)^T (hi / lo N-row tiles, TMA).  The three products share ONE
// accumulator D (N columns), as the forward's SS form does, which leaves
// TMEM room for the A stages and a running-sum region:
//   TMEM: [0, N) D | [N, N + 64 NA) A stages (hi 32 | lo 32) | [.., + N-128) S
// Chains of P.chain K blocks (shorter than k_tc_adjoint's: three MMAs per
// K step now truncate into the same fp32 accumulator) are drained by the
// eight epilogue warps: columns [0, 128) into fp32 register sums, columns
// [128, N) into the TMEM sum region S (tcgen05.ld D, ld S, add, st S).
// The end of the k range goes through shared memory (over the idle B ring)
// into the coil combine, as k_tc_adjoint.
//
// Roles (16 warps): 0 lane 0 B-ring TMA, lane 1 input-ring TMA; 1 MMA
// issuer (elected lane); 2-3 input prep (d'); 4-7 generators (one per TMEM
// lane quarter, 32 samples each); 8-15 epilogue (two per lane quarter).
//
// CL = 2 (the form every wide plan takes: the x-tile count is always even):
// a CTA pair (cta_group::2) on two x tiles of the same frame, y tile and k
// range: M = 256 pair MMAs (each CTA's generated A in its own TMEM), the
// static B tiles split over the pair along N (each CTA's shared memory
// holds N/2 of the rows), so the B traffic into each SM's shared memory
// (TMA writes and MMA reads) halves.  Synchronisation across the pair:
//   - both CTAs' B loads complete on the leader's `bfull` (cta_group::2
//     TMA, the leader arms it for both CTAs' bytes);
//   - the leader's MMA commits are multicast onto both CTAs' `bempty`,
//     `aempty` and `acc_full`;
//   - every warp arrives on CTA-local barriers (`gen`, `acc_empty`); the
//     peer's otherwise idle MMA warp acquires those and relays them to
//     the leader's `genp` / `acc_emptyp` with relaxed cluster-scope
//     arrives (a release.cluster arrive costs ~2000 cycles, measured).
// The running sums of columns >= 128 live in shared memory (float4
// [col / 4][lane], in the space the halved B stages free), which leaves
// TMEM to the accumulator and four A stages:
//   TMEM (CL = 2): [0, N) D | [N, N + 64 NA) A stages.
// CL = 1 remains as the single-CTA form (debug builds: CSR_ADJW_CL=1).
#pragma once

#include "tc_adjoint.cuh"

namespace csr {

constexpr int ADJW_MAX_N = 256;
constexpr int ADJW_EW = 8;  // epilogue warps: two per TMEM lane quarter
constexpr int ADJW_THREADS = (8 + ADJW_EW) * 32;

struct AdjWParams {
    unsigned long long *probe;
    TcArgs a;
    int S, kb_per_split, kb_total, raw_bytes, n_raw, chain;
    int N;        // pixel rows per CTA (multiple of 32, 128 < N <= 256)
    int NA;       // A stages in TMEM
    int NB;       // B ring stages in shared memory
    int exp_flags;
    unsigned long long *trace;  // CSR_TRACE + -DADJ_TIMELINE: CTA 0 per-block clock64 stamps
    const float2 *sens;
    float2 *ws;
    const float *scales;
    const int *gate;
};

// CTA-0 per-K-block timeline (tools/trace_adjw.py; -DADJ_TIMELINE=1 builds)
#if ADJ_TIMELINE
#define ADJW_TL(i, slot, cond)                                                         \
    if (P.trace && (cond) && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && \
        (i) < 1024)                                                                    \
    P.trace[65536 + 8 * (i) + (slot)] = clock64()
#else
#define ADJW_TL(i, slot, cond) \
    do {                       \
    } while (0)
#endif

// shared memory: B ring NB x (hi N x 128 B | lo N x 128 B), input ring,
// barriers; the coil-combine sums [N][ADJ_SUM_LD] floats reuse the B ring
// (per CTA: a pair holds N/2 rows each)
__host__ __device__ constexpr int adjw_b_stage(int N, int CL = 1) { return 2 * (N / CL) * 128; }
// pair form: fp32 running sums of columns >= 128, [col / 4][lane] float4,
// ahead of the B ring
__host__ __device__ constexpr int adjw_s_bytes(int N, int CL) { return CL > 1 ? (N - 128) * 128 * 4 : 0; }

template <int CP, int CL>
__global__ void __launch_bounds__(ADJW_THREADS, 1)
    k_tc_adjoint_w(const __grid_constant__ CUtensorMap tmB_hi,
                   const __grid_constant__ CUtensorMap tmB_lo,
                   const __grid_constant__ CUtensorMap tmP0,
                   const __grid_constant__ CUtensorMap tmKd, AdjWParams P) {
    using namespace sm100;
    pdl_trigger();
    constexpr int XS = 64 / CP;
    constexpr int IN_STAGE = adj_in_stage_bytes(CP);
    constexpr int OFF_D = 32 * XS * 8, OFF_DP = OFF_D + 32 * CP * 8;
    constexpr int GW = 4, SPW = 32;  // generator warps, samples per warp and K block
    const int N = P.N, NA = P.NA, NB = P.NB;
    constexpr bool PAIR = CL > 1;
    const int BST = adjw_b_stage(N, CL);
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem_all = align1024(smem_raw);
    float *s_run = reinterpret_cast<float *>(smem_all);  // PAIR: running sums [col][lane]
    uint8_t *smem = smem_all + adjw_s_bytes(N, CL);      // B ring
    uint8_t *in_base = smem + NB * BST;
    float *sum_s = reinterpret_cast<float *>(smem);  // after the main loop
    uint64_t *bfull = reinterpret_cast<uint64_t *>(in_base + P.n_raw * IN_STAGE);
    uint64_t *bempty = bfull + 4;
    uint64_t *gen = bempty + 4;        // [NA] A stage written
    uint64_t *aempty = gen + 4;        // [NA] A stage consumed
    uint64_t *rfull = aempty + 4;
    uint64_t *dfull = rfull + ADJ_MAX_RAW;
    uint64_t *rempty = dfull + ADJ_MAX_RAW;
    uint64_t *acc_full = rempty + ADJ_MAX_RAW;
    uint64_t *acc_empty = acc_full + 1;
    uint64_t *genp = acc_empty + 1;    // [NA] (PAIR, leader) the peer's stage written
    uint64_t *acc_emptyp = genp + 4;   // (PAIR, leader) the peer's drain done
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acc_emptyp + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int mt = blockIdx.x, nt = blockIdx.y;
    const int t = blockIdx.z % P.a.T, s_id = blockIdx.z / P.a.T;
    const int kb0 = s_id * P.kb_per_split;
    const int kb1 = min(P.kb_total, kb0 + P.kb_per_split);
    const int nkb = kb1 - kb0;
    const int chain = P.chain;
    const int nchain = (nkb + chain - 1) / chain;
    const int NR = P.n_raw;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tmB_hi);
        tma_prefetch(&tmB_lo);
        tma_prefetch(&tmP0);
        tma_prefetch(&tmKd);
        for (int s = 0; s < NB; ++s) {
            mbar_init(&bfull[s], 1);
            mbar_init(&bempty[s], 1);
        }
        for (int s = 0; s < NA; ++s) {
            mbar_init(&gen[s], GW);
            mbar_init(&aempty[s], 1);
            mbar_init(&genp[s], 1);
        }
        mbar_init(acc_emptyp, 1);
        for (int r = 0; r < NR; ++r) {
            mbar_init(&rfull[r], 1);
            mbar_init(&dfull[r], 2);
            mbar_init(&rempty[r], GW);
        }
        mbar_init(acc_full, 1);
        mbar_init(acc_empty, ADJW_EW);
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
    const uint32_t crank = CL > 1 ? cluster_ctarank() : 0;
    const int hrows = N / CL;  // B rows in this CTA's shared memory
    // the leader's barriers (shared::cluster addresses) for the pair form
    const uint32_t lead = PAIR ? mapa_shared(smem_u32(bfull), 0) : 0;
    auto cl_bar = [&](uint64_t *b) { return lead + (uint32_t)((uint8_t *)b - (uint8_t *)bfull); };
    auto load_b = [&](uint8_t *st, uint64_t *bar, int kb, int brow) {
        if (!PAIR) {
            mbar_arrive_expect_tx(bar, BST);
            tma_load_2d(st, &tmB_hi, bar, kb * 64, brow);
            tma_load_2d(st + N * 128, &tmB_lo, bar, kb * 64, brow);
        } else {
            // the leader arms its barrier for both CTAs' bytes
            if (crank == 0) mbar_arrive_expect_tx(bar, CL * BST);
            const int o = (int)crank * hrows;
            tma_load_2d_pair(st, &tmB_hi, cl_bar(bar), kb * 64, brow + o);
            tma_load_2d_pair(st + hrows * 128, &tmB_lo, cl_bar(bar), kb * 64, brow + o);
        }
    };
    const uint32_t a_col0 = (uint32_t)N;                 // A stages
    const uint32_t s_col0 = (uint32_t)(N + 64 * NA);     // running sums of cols >= 128
    // the first B stages (static factor) before the programmatic wait
    const int pre = min(nkb, NB);
    const int brow = t * P.a.nyA + nt * N;
    if (warp == 0 && lane == 0)
        for (int i = 0; i < pre; ++i) load_b(smem + i * BST, &bfull[i], kb0 + i, brow);
    pdl_wait();
    const bool run = !P.gate || *P.gate;
    if (run) probe_enter(P.probe);

    if (!run) {
        if (warp == 0 && lane == 0 && crank == 0)
            for (int i = 0; i < pre; ++i) mbar_wait(&bfull[i], 0);
    } else if (warp == 0) {
        if (lane == 0) {
            for (int i = pre; i < nkb; ++i) {
                const int kb = kb0 + i;
                const int s = i % NB;
                wait_slow(&bempty[s], ((i / NB) & 1) ^ 1);
                load_b(smem + s * BST, &bfull[s], kb, brow);
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
        // input prep: d' = sg * ((dr, di), (di, -dr)) per (k, c)
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
    } else if (warp == 1 && PAIR && crank != 0) {
        // the peer's MMA warp relays "A stage written" and "accumulator
        // drained" to the leader: it acquires the CTA-local barrier (the
        // generators' tcgen05.st / the epilogue's tcgen05.ld have completed
        // before their local arrive) and forwards it with a relaxed
        // cluster-scope arrive (a release.cluster arrive costs ~1900-2800
        // cycles, measured: on the drain it stalled every chain end)
        if (lane == 0)
            for (int i = 0; i < nkb; ++i) {
                if (i > 0 && i % chain == 0) {
                    wait_fast(acc_empty, (i / chain - 1) & 1);
                    mbar_arrive_cluster_relaxed(cl_bar(acc_emptyp));
                }
                const int sa = i % NA;
                wait_fast(&gen[sa], (i / NA) & 1);
                mbar_arrive_cluster_relaxed(cl_bar(&genp[sa]));
            }
    } else if (warp == 1) {
        // MMA issuer: three N-wide MMAs per K step into the one accumulator
        const uint32_t idesc = idesc_f16(128 * CL, N);
        int i = 0;
        for (int ch = 0; ch < nchain; ++ch) {
            wait_fast(acc_empty, (ch & 1) ^ 1);
            if (PAIR) wait_fast(acc_emptyp, (ch & 1) ^ 1);
            tc_fence_after();
            const int iend = min(nkb, i + chain);
            for (int i0 = i; i < iend; ++i) {
                const int sa = i % NA, sb = i % NB;
                wait_fast(&gen[sa], (i / NA) & 1);
                if (PAIR) wait_fast(&genp[sa], (i / NA) & 1);
                ADJW_TL(i, 0, lane == 0);
                wait_fast(&bfull[sb], (i / NB) & 1);
                ADJW_TL(i, 1, lane == 0);
                tc_fence_after();
                const uint32_t st = smem_u32(smem + sb * BST);
                const uint32_t a_hi = tmem + a_col0 + 64 * sa, a_lo = a_hi + 32;
                if (elect_one()) {
                    if (!(P.exp_flags & 2)) {
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk) {
                            const uint64_t dbh = desc_sw128(st + kk * 32);
                            const uint64_t dbl = desc_sw128(st + hrows * 128 + kk * 32);
                            const uint32_t acc = (i != i0) || (kk != 0);
                            if (PAIR) {
                                mma_f16_ts_pair(tmem, a_hi + 8 * kk, dbh, idesc, acc);
                                mma_f16_ts_pair(tmem, a_hi + 8 * kk, dbl, idesc, 1);
                                mma_f16_ts_pair(tmem, a_lo + 8 * kk, dbh, idesc, 1);
                            } else {
                                mma_f16_ts(tmem, a_hi + 8 * kk, dbh, idesc, acc);
                                mma_f16_ts(tmem, a_hi + 8 * kk, dbl, idesc, 1);
                                mma_f16_ts(tmem, a_lo + 8 * kk, dbh, idesc, 1);
                            }
                        }
                    }
                    if (PAIR) {
                        mma_commit_pair_mc(&bempty[sb], (uint16_t)((1u << CL) - 1));
                        mma_commit_pair_mc(&aempty[sa], (uint16_t)((1u << CL) - 1));
                    } else {
                        mma_commit(&bempty[sb]);
                        mma_commit(&aempty[sa]);
                    }
                }
                __syncwarp();
            }
            if (elect_one()) {
                if (PAIR) mma_commit_pair_mc(acc_full, (uint16_t)((1u << CL) - 1));
                else mma_commit(acc_full);
            }
            __syncwarp();
        }
    } else if (warp >= 4 && warp < 4 + GW) {
        // generators: lane quarter q, row m = (x, c, part), 32 samples
        const int q = warp & 3;
        const int m = q * 32 + lane;
        const int j = m >> 1, part = m & 1;
        const int xl = j / CP, c = j % CP;
        const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
        for (int i = 0, r = 0, rph = 0; i < nkb; ++i) {
            const int sa = i % NA;
            wait_fast(&dfull[r], rph);
            ADJW_TL(i, 2, lane == 0 && warp == 4);
            const uint8_t *in = in_base + r * IN_STAGE;
            const float2 *p0s = reinterpret_cast<const float2 *>(in);
            const float2 *dps = reinterpret_cast<const float2 *>(in + OFF_DP) + (c * 2 + part);
            uint32_t hv[SPW], lv[SPW];
            if (P.exp_flags & 1) {
#pragma unroll
                for (int k = 0; k < SPW; ++k) hv[k] = lv[k] = 0u;
            } else
#pragma unroll
            for (int k = 0; k < SPW; ++k) {
                // (profiling, debug builds: 4 = operands from registers, no LDS)
                const float2 p = (P.exp_flags & 4) ? make_float2(0.6f + 1e-3f * k, 0.8f)
                                                   : p0s[k * XS + xl];
                const float2 u = (P.exp_flags & 4) ? make_float2(1e-2f * lane, 0.5f * k)
                                                   : dps[k * CP * 2];
                const float e0 = fmaf(p.x, u.x, p.y * u.y);
                const float e1 = fmaf(p.y, u.x, -(p.x * u.y));
                const __half2 hh = __floats2half2_rn(e0, e1);
                const float2 hf = __half22float2(hh);
                const __half2 ll = __floats2half2_rn(e0 - hf.x, e1 - hf.y);
                hv[k] = *reinterpret_cast<const uint32_t *>(&hh);
                lv[k] = *reinterpret_cast<const uint32_t *>(&ll);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&rempty[r]);
            if (++r == NR) {
                r = 0;
                rph ^= 1;
            }
            ADJW_TL(i, 3, lane == 0 && warp == 4);
            wait_fast(&aempty[sa], ((i / NA) & 1) ^ 1);
            ADJW_TL(i, 4, lane == 0 && warp == 4);
            tc_fence_after();
            const uint32_t col = lane_base + a_col0 + 64 * sa;
            if (!(P.exp_flags & 8)) {  // (profiling: 8 = no TMEM stores)
                tmem_st32(col, hv);
                tmem_st32(col + 32, lv);
                tmem_st_wait();
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&gen[sa]);
            ADJW_TL(i, 5, lane == 0 && warp == 4);
        }
    }
    // Epilogue: two warps per TMEM lane quarter (h = 0, 1), each draining
    // half of the columns of every chain: y in [64h, 64h + 64) into fp32
    // register sums, and half of the columns >= 128 into the TMEM sums S.
    // (The drain stalls the MMAs — one accumulator — so its length is the
    // chain overhead: measured 2734 cycles per chain at config 4 with four
    // warps reading 256 columns each, one TMEM round trip per 8-16 columns.)
    float sum[64];
    const int ew = warp - (4 + GW), eh = ew >> 2;
    const int U2 = (N - 128) / 2;  // columns >= 128 per epilogue warp
    if (run && warp >= 4 + GW) {
        const int q = warp & 3;
        const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
        const uint32_t dlo = lane_base + 64 * eh;                 // this warp's y < 128
        const uint32_t dhi = lane_base + 128 + U2 * eh;           // its y >= 128
        const uint32_t shi = lane_base + s_col0 + U2 * eh;        // their running sums
        const int m_epi = q * 32 + lane;                          // (PAIR: smem sums)
#pragma unroll
        for (int y = 0; y < 64; ++y) sum[y] = 0.f;
        for (int ch = 0; ch < nchain; ++ch) {
            wait_slow(acc_full, ch & 1);
            ADJW_TL(ch * chain, 6, lane == 0 && warp == 4 + GW);
            tc_fence_after();
            if (PAIR) {
                // fewer TMEM round trips: each wait covers 16 columns of the
                // register-summed half and 16 of the shared-memory-summed ones
                const int nc = U2 / 16;  // 16-column chunks >= 128 (1 .. 4)
                float4 *s4b = reinterpret_cast<float4 *>(s_run) + (size_t)((U2 * eh) >> 2) * 128 + m_epi;
                auto rmw16 = [&](int c, const uint32_t (&r2)[16]) {
                    float4 *s4 = s4b + (size_t)c * 4 * 128;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const float4 o = ch > 0 ? s4[j * 128] : make_float4(0.f, 0.f, 0.f, 0.f);
                        s4[j * 128] = make_float4(o.x + __uint_as_float(r2[4 * j]),
                                                  o.y + __uint_as_float(r2[4 * j + 1]),
                                                  o.z + __uint_as_float(r2[4 * j + 2]),
                                                  o.w + __uint_as_float(r2[4 * j + 3]));
                    }
                };
                auto release = [&]() {  // (local: the peer's is relayed)
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(acc_empty);
                    ADJW_TL(ch * chain, 7, lane == 0 && warp == 4 + GW);
                };
                // four rounds: 16 register-summed columns + 16 shared-memory-
                // summed columns per TMEM wait (nc <= 4)
#pragma unroll
                for (int rr = 0; rr < 4; ++rr) {
                    uint32_t r[16], r2[16];
                    tmem_ld16(dlo + rr * 16, r);
                    const bool hc = rr < nc;
                    if (hc) tmem_ld16(dhi + rr * 16, r2);
                    tmem_ld_wait();
                    ADJW_TL(600 + ch, rr, lane == 0 && warp == 4 + GW);
                    if (rr == 3) release();
#pragma unroll
                    for (int yy = 0; yy < 16; ++yy) sum[rr * 16 + yy] += __uint_as_float(r[yy]);
                    if (hc) rmw16(rr, r2);
                }
                continue;
            }
#pragma unroll
            for (int cb = 0; cb < 2; ++cb) {
                uint32_t r[32];
                tmem_ld32(dlo + cb * 32, r);
                tmem_ld_wait();
#pragma unroll
                for (int yy = 0; yy < 32; ++yy) sum[cb * 32 + yy] += __uint_as_float(r[yy]);
            }
            for (int cb = 0; cb < U2; cb += 16) {
                uint32_t r[16], sv[16];
                tmem_ld16(dhi + cb, r);
                if (ch > 0) tmem_ld16(shi + cb, sv);
                tmem_ld_wait();
                if (cb + 16 >= U2) {  // this warp has read its accumulator columns
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(acc_empty);
                    ADJW_TL(ch * chain, 7, lane == 0 && warp == 4 + GW);
                }
#pragma unroll
                for (int yy = 0; yy < 16; ++yy)
                    sv[yy] = __float_as_uint((ch > 0 ? __uint_as_float(sv[yy]) : 0.f) +
                                             __uint_as_float(r[yy]));
                tmem_st16(shi + cb, sv);
            }
            tmem_st_wait();
        }
    }
    __syncthreads();  // all MMAs and TMA loads are done: the rings are free
    if (run && warp >= 4 + GW) {
        const int q = warp & 3;
        const int m = q * 32 + lane;
        const uint32_t shi = tmem + ((uint32_t)(q * 32) << 16) + s_col0 + U2 * eh;
#pragma unroll
        for (int y = 0; y < 64; ++y) sum_s[(64 * eh + y) * ADJ_SUM_LD + m] = sum[y];
        tc_fence_after();
        for (int cb = 0; cb < U2; cb += 16) {
            uint32_t sv[16];
            if (PAIR) {
                const float4 *s4 = reinterpret_cast<const float4 *>(s_run) +
                                   (size_t)((U2 * eh + cb) >> 2) * 128 + m;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float4 v = s4[j * 128];
                    sv[4 * j] = __float_as_uint(v.x);
                    sv[4 * j + 1] = __float_as_uint(v.y);
                    sv[4 * j + 2] = __float_as_uint(v.z);
                    sv[4 * j + 3] = __float_as_uint(v.w);
                }
            } else {
                tmem_ld16(shi + cb, sv);
                tmem_ld_wait();
            }
#pragma unroll
            for (int yy = 0; yy < 16; ++yy)
                sum_s[(128 + U2 * eh + cb + yy) * ADJ_SUM_LD + m] = __uint_as_float(sv[yy]);
        }
    }
    __syncthreads();
    // coil combine: ws[x, y] = sum_c conj(s_c[x,y]) (re + i im)_{x,c}(y)
    if (run) {
        const float inv = 1.f / pow2_scale(P.scales[5]);
        const int64_t nxy = (int64_t)P.a.nx * P.a.ny;
        float2 *wbase = P.ws + ((int64_t)s_id * P.a.T + t) * nxy;
        for (int idx = threadIdx.x; idx < N * XS; idx += ADJW_THREADS) {
            const int e = idx % N, xq = idx / N;
            const int y = nt * N + e;
            const int xg = mt * XS + xq;
            if (y >= P.a.ny || xg >= P.a.nx) continue;
            const float *row = sum_s + e * ADJ_SUM_LD;
            float ar = 0.f, ai = 0.f;
#pragma unroll
            for (int cc = 0; cc < CP; ++cc) {
                if (cc < P.a.C) {
                    const float re = row[2 * (xq * CP + cc)];
                    const float im = row[2 * (xq * CP + cc) + 1];
                    const float2 sv = __ldg(P.sens + (int64_t)cc * nxy + (int64_t)xg * P.a.ny + y);
                    ar += sv.x * re + sv.y * im;
                    ai += sv.x * im - sv.y * re;
                }
            }
            wbase[(int64_t)xg * P.a.ny + y] = make_float2(ar * inv, ai * inv);
        }
    }
    __syncthreads();
    if (run) probe_exit(P.probe);
    // no CTA of a pair leaves while the leader's MMAs / commits may still
    // touch the peer (its shared memory, barriers and tensor memory)
    if (PAIR) cluster_sync();
    if (warp == 1) {
        tc_fence_after();
        if (PAIR) tmem_dealloc_pair(tmem, 512);
        else tmem_dealloc(tmem, 512);
    }
}

}  // namespace csr
