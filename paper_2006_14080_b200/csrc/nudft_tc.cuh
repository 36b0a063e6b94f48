// tcgen05 NUDFT: plan build (factor copies, tensor maps, split-K and
// persistent-grid choices) and the launch wrappers used by csrecon_b200.cu.
#pragma once

#include "tc_adjoint.cuh"
#include "tc_adjoint_w.cuh"
#include "tc_forward.cuh"

namespace csr {

// ---------------------------------------------------------------------------
// host side
typedef CUresult (*PFN_encodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                    const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                    const cuuint32_t *, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion,
                                    CUtensorMapFloatOOBfill);

inline PFN_encodeTiled get_encode() {
    static PFN_encodeTiled fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_encodeTiled)p;
    }
    return fn;
}

// 2-D fp16 K-major operand: inner dim K (elements), outer rows; box 64 x box_rows
inline bool tmap_f16_2d(CUtensorMap *m, const void *base, uint64_t K, uint64_t rows,
                        uint32_t box_rows) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[2] = {K, rows};
    cuuint64_t strides[1] = {K * 2};
    cuuint32_t box[2] = {64, box_rows};
    cuuint32_t es[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void *>(base), dims, strides,
               box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 3-D complex64 array viewed as 8-byte elements {d0, d1, d2}, no swizzle
inline bool tmap_c64_3d(CUtensorMap *m, const void *base, uint64_t d0, uint64_t d1,
                        uint64_t d2, uint32_t b0, uint32_t b1) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[3] = {d0, d1, d2};
    cuuint64_t strides[2] = {d0 * 8, d0 * d1 * 8};
    cuuint32_t box[3] = {b0, b1, 1};
    cuuint32_t es[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<void *>(base), dims, strides,
               box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

inline TcArgs tc_args(const TcPlan &tc) {
    TcArgs a;
    a.T = tc.T; a.nx = tc.nx; a.ny = tc.ny; a.C = tc.C; a.Cp = tc.Cp; a.xs = tc.xs;
    a.nxp = tc.nxp; a.nyA = tc.nyA; a.Kf = tc.Kf; a.Nf = tc.Nf; a.M = tc.M; a.Mk = tc.Mk;
    return a;
}

inline int tc_alloc(std::vector<void *> &allocs, void **p, size_t bytes, int64_t *acct,
                    cudaStream_t st) {
    if (pool_alloc(p, bytes, st) != cudaSuccess) return 2;
    allocs.push_back(*p);
    if (acct) *acct += (int64_t)bytes;
    return 0;
}

template <class F>
inline void set_smem(F kernel, int bytes) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

// Adjoint split-K cost model: waves of 148 CTAs x per-CTA time (blocks x
// blk_cycles of MMA + chain drains + CTA setup/fill), bounded by the
// partial-image memory; returns the number of k ranges S.
inline int tc_split_model(int64_t tiles, int kb_total, int64_t pix_bytes, int blk_cycles = 768,
                          int chain = TC_MAX_CHAIN) {
    int S = 1;
    int64_t best_cost = INT64_MAX;
    for (int c = 1; c <= std::min(kb_total, 1024); ++c) {
        if (c > 1 && c * pix_bytes > ((int64_t)1 << 30)) break;
        const int64_t kbps = (kb_total + c - 1) / c;
        const int64_t nch = (kbps + chain - 1) / chain;
        const int64_t waves = (tiles * c + 147) / 148;
        const int64_t cost = waves * (kbps * blk_cycles + nch * 700 + 4000);
        if (cost < best_cost) {
            best_cost = cost;
            S = c;
        }
    }
    return S;
}

// Adjoint tile geometry.  ny <= 128 (or more than 16 coils): 128-row y tiles
// of k_tc_adjoint.  Otherwise the wide kernel k_tc_adjoint_w: nyt tiles of
// N rows (a multiple of 16, <= 256) covering ny, one generated operand per
// K block for all N rows.
struct AdjGeom {
    bool wide = false;
    int N = 128, nyt = 1, NA = 4, NB = 0, chain = TC_MAX_CHAIN, blk_cycles = 768;
    int CL = 1;  // wide kernel: CTA pairs (cta_group::2) along x splitting B
};
inline AdjGeom tc_adj_geom(int ny, int Cp, int mt_a = 0) {
    AdjGeom g;
    g.nyt = (ny + 127) / 128;
    if (ny <= 128 || Cp > 16 || dbg_env("CSR_ADJ_NARROW")) return g;
    g.wide = true;
    g.nyt = (ny + ADJW_MAX_N - 1) / ADJW_MAX_N;
    // a multiple of 32: each of the two epilogue warps of a lane quarter
    // drains (N - 128) / 2 columns >= 128 in 16-column loads
    g.N = ((ny + g.nyt - 1) / g.nyt + 31) / 32 * 32;
    // pairs of x tiles (cta_group::2) split the B rows: half the rows each, a
    // multiple of 8 (one swizzle atom)
    g.CL = (mt_a % 2 == 0 && (g.N / 2) % 8 == 0) ? 2 : 1;
    if (const char *e = dbg_env("CSR_ADJW_CL")) g.CL = (atoi(e) == 2 && mt_a % 2 == 0) ? 2 : 1;
    // TMEM: D (N) + A stages (64 each) + sums of columns >= 128 (N - 128;
    // the pair form keeps those sums in shared memory)
    g.NA = std::min(4, (512 - g.N - (g.CL == 2 ? 0 : g.N - 128)) / 64);
    if (const char *e = dbg_env("CSR_ADJW_NA")) g.NA = std::max(2, std::min(g.NA, atoi(e)));
    // B ring: two stages (the MMAs take ~1.3 us per K block, an L2-hit TMA
    // refill ~1 us); the rest of shared memory deepens the input ring, whose
    // TMA -> prep -> generator -> release round trip bounds the kernel with
    // two stages (measured: the skeleton without math or MMAs ran at 0.66 us
    // per K block with NB = 3, NR = 2).  The combine's sums reuse both rings.
    g.NB = g.CL == 2 ? 3 : 2;  // (pair: half-size stages)
    if (const char *e = dbg_env("CSR_ADJW_NB")) g.NB = std::max(2, std::min(4, atoi(e)));
    // three N-wide MMAs per K step truncate into one fp32 accumulator:
    // shorter chains than the two-accumulator kernel.  The error grows
    // linearly with the chain (config 4 adjoint rel-L2 2.8e-6 at 12, 3.7e-6
    // at 16, 5.5e-6 at 24; tolerance 1e-5); the pair form at N = 256 drains
    // ~3200 cycles per chain with the MMAs stalled, so it takes chains of 16
    // (config 4 12.66 -> 12.31 ms, profiles/r02al_pair_drain.txt)
    g.chain = (g.CL == 2 && g.N >= 256) ? 16 : TC_ADJW_CHAIN;
    if (const char *e = dbg_env("CSR_ADJW_CHAIN")) g.chain = std::max(1, atoi(e));
    g.blk_cycles = 4 * 3 * (g.N / 2 + 32);
    return g;
}

// Coil padding and adjoint tile count of a (T, nx, ny, C) plan.
inline void tc_tiles(int T, int nx, int ny, int C, int &Cp, int64_t &tiles) {
    Cp = 4;
    while (Cp < C) Cp *= 2;
    const int xs = 128 / Cp;
    const int nxp = (nx + xs - 1) / xs * xs;
    tiles = (int64_t)T * (nxp * Cp / 64) * tc_adj_geom(ny, Cp).nyt;
}

// Global sample-chunk grid of an order-stable sample-sharded problem
// (T = 1): the k range of one adjoint split-K partial, a multiple of 128
// samples so that every rank's chunk run starts on a forward sample tile.
// The split is what a single plan of the whole problem would choose.
inline void tc_sample_chunking(int nx, int ny, int C, int64_t M, int64_t &chunk,
                               int &n_chunks) {
    int Cp;
    int64_t tiles;
    tc_tiles(1, nx, ny, C, Cp, tiles);
    const int kb_total = (int)((M + 127) / 128 * 128 / 32);
    const AdjGeom ag = tc_adj_geom(ny, Cp);
    const int S = tc_split_model(tiles, kb_total, (int64_t)nx * ny * 8, ag.blk_cycles, ag.chain);
    int kbps = (kb_total + S - 1) / S;
    kbps = (kbps + 3) / 4 * 4;
    chunk = (int64_t)kbps * 32;
    n_chunks = (int)((M + chunk - 1) / chunk);
}

// chunk > 0: order-stable sample sharding (csr_plan_desc.chunk_samples):
// the adjoint's k ranges are the global chunks (chunk / 32 blocks each) and
// the forward is the tile-group form with the tile-group count of the
// whole problem (M_global samples), so every sample's k-space value and
// every chunk's partial image are the same bits whichever rank owns them.
inline int tc_plan_build(TcPlan &tc, int T, int nx, int ny, int C, int64_t M,
                         const float2 *P0, const float2 *P1, const float2 *sens,
                         cudaStream_t st, int64_t *factor_bytes, int64_t *ws_bytes,
                         std::vector<void *> &allocs, int64_t chunk = 0,
                         int64_t M_global = 0) {
    tc.enabled = false;
    if (C > TC_MAX_COILS || dbg_env("CSR_DISABLE_TC")) return 0;
    if (!get_encode()) return 0;
    tc.T = T; tc.nx = nx; tc.ny = ny; tc.C = C; tc.M = M;
    int Cp = 4;
    while (Cp < C) Cp *= 2;
    tc.Cp = Cp;
    tc.xs = 128 / Cp;
    tc.nxp = (nx + tc.xs - 1) / tc.xs * tc.xs;
    tc.nyp = (ny + 31) / 32 * 32;
    tc.nyA = (ny + 127) / 128 * 128;
    tc.Kf = 2 * tc.nyp;
    tc.Nf = 2 * tc.nxp * Cp;
    tc.Mk = (M + 127) / 128 * 128;
    // the forwards run on CTA pairs of sample tiles within a frame: an odd
    // tile count gets one zero tile of padding (factors are zero there)
    // when that costs <= 1/15 more forward work (config 3: 39 -> 40 tiles,
    // forward 739 -> 645 us); the adjoint's K range stays at the unpadded
    // samples (kb_total)
    const int64_t Mk128 = tc.Mk;
    if (chunk == 0 && (tc.Mk / TC_BM) % 2 == 1 && tc.Mk / TC_BM >= 15) tc.Mk += TC_BM;
    tc.nt = tc.Nf / TC_BN;
    tc.mt_f = (int)(tc.Mk / TC_BM);
    // forward groups: split the n-tiles so the grid covers the machine
    // (order-stable plans: the grouping of the whole problem)
    const int64_t mtiles = chunk > 0 ? (int64_t)T * ((M_global + TC_BM - 1) / TC_BM)
                                     : (int64_t)T * tc.mt_f;
    int G = 1;
    while (G < tc.nt && mtiles * G < 2 * 148 && tc.nt % (2 * G) == 0) G *= 2;
    tc.G = G;
    tc.nt_per_group = tc.nt / G;
    // A-stationary forward: 128-row B tiles; groups of tiles per CTA chosen
    // by waves x per-CTA time (tiles x K blocks x ~768 MMA cycles + setup).
    // Its split of a sample tile into pieces depends on the grid, so the
    // order-stable mode keeps the tile-group form.
    // (<= 16 coils: the persistent form's 576-thread CTA keeps CP complex
    // accumulators per epilogue thread in registers)
    tc.fwd_ts = tc.Kf <= 256 && Cp <= 16 && !dbg_env("CSR_FWD_SS") && chunk == 0;
    // SS form: CTA pairs (cta_group::2) on two sample tiles of one frame,
    // the image operand split over the pair
    tc.fwd_CL = (tc.mt_f % 2 == 0) ? 2 : 1;
    if (const char *e = dbg_env("CSR_FWD_CL")) tc.fwd_CL = (atoi(e) == 2 && tc.mt_f % 2 == 0) ? 2 : 1;
    // PS form of the persistent forward (A staged from shared memory next
    // to B, two accumulators so the drain overlaps the next unit's MMAs):
    // measured faster than A in tensor memory (config 1 39.4 vs 41.8 us,
    // config 0 9.9 vs 11.4 us); CSR_FWD_PS=0 selects the TMEM-A form
    {
        const char *e = dbg_env("CSR_FWD_PS");
        tc.fwd_ps = tc.fwd_ts && !(e && e[0] == '0');
    }
    // ... on CTA pairs (cta_group::2: M = 256, B split over the pair) when
    // the sample tiles pair up within a frame; CSR_FWD_PAIR=0 keeps one CTA
    {
        const char *e = dbg_env("CSR_FWD_PAIR");
        tc.fwd_pair = tc.fwd_ps && tc.mt_f % 2 == 0 && !(e && e[0] == '0');
    }
    if (tc.fwd_ts) {
        const int NTt = tc.Nf / 256;
        const int CLp = tc.fwd_pair ? 2 : 1;
        const int64_t units = mtiles / CLp * NTt;
        tc.fts_smem = (tc.fwd_ps ? FPS_STAGES * FPS_STAGE : FTS_STAGES * 2 * FTS_B_TILE) + 1024 + 256;
        // CTAs = SMs (persistent); pieces of a sample tile split across CTAs
        // are limited to the 4 flag slots per tile
        auto max_pieces = [&](int64_t Gc) {
            auto owner = [&](int64_t u) {
                int64_t b = u * Gc / units;
                while (b + 1 < Gc && units * (b + 1) / Gc <= u) ++b;
                while (b > 0 && units * b / Gc > u) --b;
                return b;
            };
            int mp = 1;
            for (int64_t m = 0; m < mtiles / CLp; ++m)
                mp = std::max<int>(mp, (int)(owner((m + 1) * NTt - 1) - owner(m * NTt) + 1));
            return mp;
        };
        int64_t Gc = std::min<int64_t>(148 / CLp, units);
        int maxp = max_pieces(Gc);
        while (maxp > 4 && Gc > mtiles / CLp) maxp = max_pieces(--Gc);
        tc.fts_ctas = (int)Gc * CLp;
        G = std::max(G, maxp - 1);  // kdp holds pieces 1.. (piece 0 stays in registers)
        tc.fts_pieces = maxp;
    }
    // adjoint split-K
    tc.mt_a = tc.nxp * Cp / 64;  // adjoint tiles over (x, c): 64 per tile
    tc.kb_total = (int)(Mk128 / 32);
    const AdjGeom ag = tc_adj_geom(ny, Cp, tc.mt_a);
    tc.nyA = std::max(tc.nyA, ag.nyt * ag.N);  // the wide tiles' padded pixel rows
    tc.adj_w = ag.wide;
    tc.adjw_CL = ag.CL;
    tc.adjw_N = ag.N;
    tc.adjw_nyt = ag.nyt;
    tc.adjw_NA = ag.NA;
    tc.adjw_NB = ag.NB;
    tc.adj_chain = ag.chain;
    const int64_t tiles = (int64_t)T * tc.mt_a * ag.nyt;
    // split-K: each CTA takes one tile and a contiguous k range, cut into
    // accumulation chains of <= TC_MAX_CHAIN blocks.  Pick S by a cost model
    // (waves of 148 CTAs x per-CTA time: blocks x ~768 MMA cycles + chain
    // drains + CTA setup/fill), bounded by the partial-image memory.
    int S = tc_split_model(tiles, tc.kb_total, (int64_t)T * nx * ny * 8, ag.blk_cycles, ag.chain);
    if (const char *e = dbg_env("CSR_TC_SPLIT")) S = std::max(1, std::min(atoi(e), tc.kb_total));
    tc.kb_per_split = (tc.kb_total + S - 1) / S;
    if (chunk > 0) tc.kb_per_split = (int)(chunk / 32);
    S = (tc.kb_total + tc.kb_per_split - 1) / tc.kb_per_split;
    tc.split = S;
    tc.raw_bytes = 32 * (64 / Cp) * 8 + 32 * Cp * 8;
    tc.adj_stage = adj_in_stage_bytes(Cp);  // input ring stage
    tc.fwd_smem = TC_STAGES * TC_FWD_OPS + 1024 + 256;
    {
        const int fixed = ADJ_STAGES * ADJ_B_STAGE + 1024 + 512;
        tc.adj_nraw = std::min(ADJ_MAX_RAW, (227 * 1024 - fixed) / tc.adj_stage);
        if (const char *e = dbg_env("CSR_ADJ_NRAW"))
            tc.adj_nraw = std::max(1, std::min(tc.adj_nraw, atoi(e)));
        tc.adj_smem = fixed + tc.adj_nraw * tc.adj_stage;
    }
    if (tc.adj_w) {
        const int sbytes = adjw_s_bytes(tc.adjw_N, tc.adjw_CL);
        const int fixed = sbytes + tc.adjw_NB * adjw_b_stage(tc.adjw_N, tc.adjw_CL) + 1024 + 512;
        tc.adjw_nraw = std::min(ADJ_MAX_RAW, (227 * 1024 - fixed) / tc.adj_stage);
        tc.adjw_smem = fixed + tc.adjw_nraw * tc.adj_stage;
        // the combine's sums [N][ADJ_SUM_LD] floats over the B and input rings
        const int rings = fixed - 1536 - sbytes + tc.adjw_nraw * tc.adj_stage;
        if (tc.adjw_nraw < 2 || tc.adjw_N * ADJ_SUM_LD * 4 > rings) {
            tc.adj_w = false;  // keep the narrow kernel (128-row tiles)
            tc.nyA = (ny + 127) / 128 * 128;
        }
    }
    if (tc.adj_smem > 227 * 1024 || tc.fwd_smem > 227 * 1024) return 0;

    const size_t fa = (size_t)T * tc.Mk * tc.Kf, ga = (size_t)T * tc.nyA * 2 * tc.Mk;
    const size_t xb = (size_t)T * tc.Nf * tc.Kf;
    void *p;
#define TCA(ptr, bytes, acct)                                 \
    do {                                                      \
        if (tc_alloc(allocs, &p, (bytes), (acct), st)) return 2;  \
        ptr = decltype(ptr)(p);                               \
    } while (0)
    TCA(tc.fa_hi, fa * 2, factor_bytes);
    TCA(tc.fa_lo, fa * 2, factor_bytes);
    TCA(tc.ga_hi, ga * 2, factor_bytes);
    TCA(tc.ga_lo, ga * 2, factor_bytes);
    TCA(tc.p0p, (size_t)T * tc.Mk * tc.nxp * 8, factor_bytes);
    TCA(tc.xb_hi, xb * 2, ws_bytes);
    TCA(tc.xb_lo, xb * 2, ws_bytes);
    // zero padding rows / columns once: the fused loop kernels write only
    // the valid (x < nx, c < C, y < ny) entries of the operand
    cudaMemsetAsync(tc.xb_hi, 0, xb * 2, st);
    cudaMemsetAsync(tc.xb_lo, 0, xb * 2, st);
    TCA(tc.kdp, (size_t)G * T * tc.Mk * Cp * 8, ws_bytes);
    TCA(tc.kdi, (size_t)T * tc.Mk * Cp * 8, ws_bytes);
    cudaMemsetAsync(tc.kdi, 0, (size_t)T * tc.Mk * Cp * 8, st);
    TCA(tc.ws, (size_t)S * T * nx * ny * 8, ws_bytes);
    TCA(tc.scales, 64, ws_bytes);
    TCA(tc.red, 4 * 148 * 8, ws_bytes);
    TCA(tc.tick, 64, ws_bytes);
    TCA(tc.ftick, (size_t)T * tc.mt_f * 16 + 16, ws_bytes);  // 4 piece flags per tile
    cudaMemsetAsync(tc.ftick, 0, (size_t)T * tc.mt_f * 16 + 16, st);
#undef TCA
    tc.sens = sens;
    cudaMemsetAsync(tc.tick, 0, 64, st);
    const int blocks = 148 * 8;
    launch(k_tc_build_fa, blocks, 256, 0, st, P1, T, M, tc.Mk, ny, tc.Kf, tc.fa_hi, tc.fa_lo,
           (tc.fwd_ts && !tc.fwd_ps) ? 1 : 0);
    launch(k_tc_build_ga, blocks, 256, 0, st, P1, T, M, tc.Mk, ny, tc.nyA, tc.ga_hi, tc.ga_lo);
    launch(k_tc_build_p0, blocks, 256, 0, st, P0, T, M, tc.Mk, nx, tc.nxp, tc.p0p);
    // max|s| (component-wise) for the image-operand scale bound
    {
        int64_t n = (int64_t)C * nx * ny;
        int nb = reduce_blocks(n, 256);
        launch(k_tc_sens_absmax, nb, 256, 0, st, sens, n, tc.red, tc.tick, tc.scales);
    }
    if (cudaGetLastError() != cudaSuccess) return 3;
    bool ok = tmap_f16_2d(&tc.tm_fa_hi, tc.fa_hi, tc.Kf, (uint64_t)T * tc.Mk, TC_BM) &&
              tmap_f16_2d(&tc.tm_fa_lo, tc.fa_lo, tc.Kf, (uint64_t)T * tc.Mk, TC_BM) &&
              tmap_f16_2d(&tc.tm_xb_hi, tc.xb_hi, tc.Kf, (uint64_t)T * tc.Nf, TC_BN) &&
              tmap_f16_2d(&tc.tm_xb_lo, tc.xb_lo, tc.Kf, (uint64_t)T * tc.Nf, TC_BN) &&
              tmap_f16_2d(&tc.tm_xb128_hi, tc.xb_hi, tc.Kf, (uint64_t)T * tc.Nf, TC_BN / 2) &&
              tmap_f16_2d(&tc.tm_xb128_lo, tc.xb_lo, tc.Kf, (uint64_t)T * tc.Nf, TC_BN / 2) &&
              tmap_f16_2d(&tc.tm_xb256_hi, tc.xb_hi, tc.Kf, (uint64_t)T * tc.Nf, 256) &&
              tmap_f16_2d(&tc.tm_xb256_lo, tc.xb_lo, tc.Kf, (uint64_t)T * tc.Nf, 256) &&
              tmap_f16_2d(&tc.tm_ga_hi, tc.ga_hi, 2 * tc.Mk, (uint64_t)T * tc.nyA, 128) &&
              tmap_f16_2d(&tc.tm_ga_lo, tc.ga_lo, 2 * tc.Mk, (uint64_t)T * tc.nyA, 128) &&
              (!tc.adj_w ||
               (tmap_f16_2d(&tc.tm_gaw_hi, tc.ga_hi, 2 * tc.Mk, (uint64_t)T * tc.nyA,
                            tc.adjw_N / tc.adjw_CL) &&
                tmap_f16_2d(&tc.tm_gaw_lo, tc.ga_lo, 2 * tc.Mk, (uint64_t)T * tc.nyA,
                            tc.adjw_N / tc.adjw_CL))) &&
              tmap_c64_3d(&tc.tm_p0, tc.p0p, tc.nxp, tc.Mk, T, 64 / Cp, 32) &&
              tmap_c64_3d(&tc.tm_kd, tc.kdi, Cp, tc.Mk, T, Cp, 32);
    if (!ok) return 0;  // descriptor encode unavailable: SIMT path
    switch (Cp) {
        case 4: set_smem(k_tc_forward<4, 1>, tc.fwd_smem); set_smem(k_tc_forward<4, 2>, tc.fwd_smem);
                set_smem(k_tc_adjoint<4>, tc.adj_smem);
                set_smem(k_tc_adjoint_w<4, 1>, tc.adjw_smem); set_smem(k_tc_adjoint_w<4, 2>, tc.adjw_smem);
                break;
        case 8: set_smem(k_tc_forward<8, 1>, tc.fwd_smem); set_smem(k_tc_forward<8, 2>, tc.fwd_smem);
                set_smem(k_tc_adjoint<8>, tc.adj_smem);
                set_smem(k_tc_adjoint_w<8, 1>, tc.adjw_smem); set_smem(k_tc_adjoint_w<8, 2>, tc.adjw_smem);
                break;
        case 16: set_smem(k_tc_forward<16, 1>, tc.fwd_smem); set_smem(k_tc_forward<16, 2>, tc.fwd_smem);
                 set_smem(k_tc_adjoint<16>, tc.adj_smem);
                 set_smem(k_tc_adjoint_w<16, 1>, tc.adjw_smem); set_smem(k_tc_adjoint_w<16, 2>, tc.adjw_smem);
                 break;
        case 32: set_smem(k_tc_forward<32, 1>, tc.fwd_smem); set_smem(k_tc_forward<32, 2>, tc.fwd_smem);
                 set_smem(k_tc_adjoint<32>, tc.adj_smem); break;
        default: break;
    }
    if (tc_alloc(allocs, &p, PROBE_SLOTS * 4 * sizeof(unsigned long long), ws_bytes, st)) return 2;
    tc.probe = (unsigned long long *)p;
    cudaMemsetAsync(tc.probe, 0, PROBE_SLOTS * 4 * sizeof(unsigned long long), st);
    tc.fexp = dbg_env("CSR_FEXP") ? atoi(dbg_env("CSR_FEXP")) : 0;
    tc.aexp = dbg_env("CSR_EXP") ? atoi(dbg_env("CSR_EXP")) : 0;
    if (dbg_env("CSR_TRACE")) {
        if (tc_alloc(allocs, &p, 4096 * 32 * 8, ws_bytes, st)) return 2;
        tc.trace = (unsigned long long *)p;
        cudaMemsetAsync(tc.trace, 0, 4096 * 32 * 8, st);
    }
    set_smem(k_tc_forward_ts<4, false>, tc.fts_smem);
    set_smem(k_tc_forward_ts<8, false>, tc.fts_smem);
    set_smem(k_tc_forward_ts<16, false>, tc.fts_smem);
    set_smem(k_tc_forward_ts<4, true>, tc.fts_smem);
    set_smem(k_tc_forward_ts<8, true>, tc.fts_smem);
    set_smem(k_tc_forward_ts<16, true>, tc.fts_smem);
    set_smem(k_tc_forward_ts<4, true, true>, tc.fts_smem);
    set_smem(k_tc_forward_ts<8, true, true>, tc.fts_smem);
    set_smem(k_tc_forward_ts<16, true, true>, tc.fts_smem);
    tc.enabled = true;
    return 0;
}

// image (T,nx,ny) -> kd.  user != nullptr: also write the (T*M, C) layout
// image -> k-space.  user != nullptr: also write the (T*M, C) layout.
// in_loop: inside the native CG loop the producer of img (k_admm_rhs /
// k_cg_d) already left max|img| in scales[6], and with a single tile group
// the forward writes the k-space buffer directly (atomic max into scales[5])
// instead of going through partials + k_tc_sum_kd.
inline int tc_forward(TcPlan &tc, const float2 *img, float2 *user, cudaStream_t st,
                      const int *gate, bool in_loop = false, bool x_ready = false) {
    TcArgs a = tc_args(tc);
    const int64_t n = (int64_t)tc.T * tc.nx * tc.ny;
    if (!in_loop)
        launch(k_tc_absmax_img, reduce_blocks(n, 256), 256, 0, st, img, n, tc.red, tc.tick,
                                                               tc.scales, gate);
    if (!x_ready) {  // else the fused CG tail already wrote X (cg_tail.cuh)
        // one thread per pixel, all coils
        int nb = (int)std::min<int64_t>((n + 255) / 256, 148 * PREP_X_BLOCKS_PER_SM);
        launch(k_tc_prep_x, nb, 256, 0, st, a, img, tc.sens, tc.scales, tc.xb_hi, tc.xb_lo, gate,
               tc.probe ? tc.probe + 4 * PROBE_PREP : nullptr);
    }
    if (tc.fwd_ts) {
        // persistent A-stationary forward: always writes the scaled k-space
        // into kdi (and max|kd| into scales[5])
        FwdTsParams P;
        P.a = a;
        P.mt_per_frame = tc.mt_f;
        P.nt_tiles = tc.Nf / 256;
        P.units = (int64_t)tc.T * tc.mt_f / (tc.fwd_pair ? 2 : 1) * P.nt_tiles;
        P.fa_hi = reinterpret_cast<const uint4 *>(tc.fa_hi);
        P.fa_lo = reinterpret_cast<const uint4 *>(tc.fa_lo);
        P.p0p = tc.p0p;
        P.kdi = tc.kdi;
        P.kdp = tc.kdp;
        P.tick = tc.ftick;
        P.scales = tc.scales;
        P.gate = gate;
        P.exp_flags = tc.fexp;
        P.trace = tc.trace;
        P.probe = tc.probe;
        dim3 grid((unsigned)tc.fts_ctas);
        switch (tc.Cp) {
#define FTS_LAUNCH(CPV)                                                                        \
    (tc.fwd_pair ? launch_cl(k_tc_forward_ts<CPV, true, true>, grid, FTS_THREADS, tc.fts_smem,   \
                             st, 2, tc.tm_xb128_hi, tc.tm_xb128_lo, tc.tm_fa_hi, tc.tm_fa_lo, P) \
     : tc.fwd_ps ? launch(k_tc_forward_ts<CPV, true>, grid, FTS_THREADS, tc.fts_smem, st,        \
                          tc.tm_xb256_hi, tc.tm_xb256_lo, tc.tm_fa_hi, tc.tm_fa_lo, P)           \
                 : launch(k_tc_forward_ts<CPV, false>, grid, FTS_THREADS, tc.fts_smem, st,       \
                          tc.tm_xb256_hi, tc.tm_xb256_lo, tc.tm_fa_hi, tc.tm_fa_lo, P))
            case 4: FTS_LAUNCH(4); break;
            case 8: FTS_LAUNCH(8); break;
            default: FTS_LAUNCH(16); break;
#undef FTS_LAUNCH
        }
        if (user) {  // (T*M, C) copy for the caller
            int64_t total = (int64_t)tc.T * tc.Mk * tc.Cp;
            launch(k_tc_sum_kd, std::min(reduce_blocks(total, 256), 3 * 148), 256, 0, st, a, 1, tc.kdi, tc.kdi, user,
                   tc.red, tc.tick, tc.scales, gate);
        }
        {
        const cudaError_t le = cudaGetLastError();
        if (le != cudaSuccess) {
            tc_last_error() = cudaGetErrorString(le);
            return 3;
        }
    }
    return 0;
    }
    const int G = tc.G;
    const bool direct = in_loop && !user && G == 1;
    float2 *kdp = direct ? tc.kdi : tc.kdp;
    {
        FwdParams P;
        P.a = a;
        P.mt_per_frame = tc.mt_f;
        P.nt_per_group = tc.nt_per_group;
        P.amax = direct ? 1 : 0;
        P.p0p = tc.p0p;
        P.kdp = kdp;
        P.scales = tc.scales;
        P.gate = gate;
        P.probe = tc.probe;
        P.exp_flags = tc.fexp;
        dim3 grid((unsigned)(tc.T * tc.mt_f), (unsigned)G);
        switch (tc.Cp) {
#define FWD_LAUNCH(CPV)                                                                         \
    (tc.fwd_CL > 1 ? launch_cl(k_tc_forward<CPV, 2>, grid, TC_FWD_THREADS, tc.fwd_smem, st, 2,    \
                               tc.tm_fa_hi, tc.tm_fa_lo, tc.tm_xb128_hi, tc.tm_xb128_lo, P)       \
                   : launch(k_tc_forward<CPV, 1>, grid, TC_FWD_THREADS, tc.fwd_smem, st,          \
                            tc.tm_fa_hi, tc.tm_fa_lo, tc.tm_xb_hi, tc.tm_xb_lo, P))
            case 4: FWD_LAUNCH(4); break;
            case 8: FWD_LAUNCH(8); break;
            case 16: FWD_LAUNCH(16); break;
            default: FWD_LAUNCH(32); break;
#undef FWD_LAUNCH
        }
    }
    if (!direct) {
        int64_t total = (int64_t)tc.T * tc.Mk * tc.Cp;
        launch(k_tc_sum_kd, std::min(reduce_blocks(total, 256), 3 * 148), 256, 0, st, a, G, tc.kdp, tc.kdi, user,
                                                               tc.red, tc.tick, tc.scales, gate);
    }
    {
        const cudaError_t le = cudaGetLastError();
        if (le != cudaSuccess) {
            tc_last_error() = cudaGetErrorString(le);
            return 3;
        }
    }
    return 0;
}

// launches tc_forward makes (for the kernel-count bookkeeping)
inline int tc_forward_launches(const TcPlan &tc, bool in_loop, bool user, bool x_ready = false) {
    if (tc.fwd_ts) return (in_loop ? 0 : 1) + (x_ready ? 1 : 2) + (user ? 1 : 0);
    const bool direct = in_loop && !user && tc.G == 1;
    return (in_loop ? 0 : 1) + (x_ready ? 1 : 2) + (direct ? 0 : 1);
}

// user (T*M, C) k-space -> tc.kdi, max|kd| -> scales[5]
inline void tc_load_kd(TcPlan &tc, const float2 *user, cudaStream_t st) {
    TcArgs a = tc_args(tc);
    int64_t total = (int64_t)tc.T * tc.Mk * tc.Cp;
    launch(k_tc_load_kd, reduce_blocks(total, 256), 256, 0, st, a, user, tc.kdi, tc.red, tc.tick,
                                                            tc.scales);
}

// kd already in tc.kdi (with sigma_d) when user == nullptr; else load it
inline int tc_adjoint(TcPlan &tc, const float2 *user, float2 *ws, cudaStream_t st,
                      const int *gate) {
    TcArgs a = tc_args(tc);
    if (user) tc_load_kd(tc, user, st);
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(tc.adj_w ? ADJW_THREADS : ADJ_THREADS);
    cfg.dynamicSmemBytes = tc.adj_w ? tc.adjw_smem : tc.adj_smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    cudaError_t e;
    if (tc.adj_w) {
        AdjWParams P;
        P.a = a;
        P.S = tc.split;
        P.kb_per_split = tc.kb_per_split;
        P.chain = tc.adj_chain;
        P.N = tc.adjw_N;
        P.NA = tc.adjw_NA;
        P.NB = tc.adjw_NB;
        P.exp_flags = tc.aexp;
        P.trace = tc.trace;
        P.probe = tc.probe ? tc.probe + 4 * PROBE_ADJ : nullptr;
        P.kb_total = tc.kb_total;
        P.raw_bytes = tc.raw_bytes;
        P.n_raw = tc.adjw_nraw;
        P.sens = tc.sens;
        P.ws = ws;
        P.scales = tc.scales;
        P.gate = gate;
        cfg.gridDim = dim3((unsigned)tc.mt_a, (unsigned)tc.adjw_nyt, (unsigned)(tc.T * tc.split));
        cudaLaunchAttribute wattr[2];
        wattr[0] = attr[0];
        wattr[1].id = cudaLaunchAttributeClusterDimension;
        wattr[1].val.clusterDim.x = (unsigned)tc.adjw_CL;
        wattr[1].val.clusterDim.y = 1;
        wattr[1].val.clusterDim.z = 1;
        if (tc.adjw_CL > 1) {
            cfg.attrs = wattr + (pdl_enabled() ? 0 : 1);
            cfg.numAttrs = pdl_enabled() ? 2 : 1;
        }
#define ADJW_LAUNCH(CPV)                                                                        \
    (tc.adjw_CL > 1 ? cudaLaunchKernelEx(&cfg, k_tc_adjoint_w<CPV, 2>, tc.tm_gaw_hi, tc.tm_gaw_lo, \
                                         tc.tm_p0, tc.tm_kd, P)                                 \
                    : cudaLaunchKernelEx(&cfg, k_tc_adjoint_w<CPV, 1>, tc.tm_gaw_hi, tc.tm_gaw_lo, \
                                         tc.tm_p0, tc.tm_kd, P))
        switch (tc.Cp) {
            case 4: e = ADJW_LAUNCH(4); break;
            case 8: e = ADJW_LAUNCH(8); break;
            default: e = ADJW_LAUNCH(16); break;
        }
#undef ADJW_LAUNCH
    } else {
        AdjParams P;
        P.a = a;
        P.S = tc.split;
        P.kb_per_split = tc.kb_per_split;
        P.chain = tc.adj_chain;
        P.exp_flags = tc.aexp;
        P.trace = tc.trace;
        P.probe = tc.probe ? tc.probe + 4 * PROBE_ADJ : nullptr;
        P.kb_total = tc.kb_total;
        P.raw_bytes = tc.raw_bytes;
        P.n_raw = tc.adj_nraw;
        P.sens = tc.sens;
        P.ws = ws;
        P.scales = tc.scales;
        P.gate = gate;
        cfg.gridDim = dim3((unsigned)tc.mt_a, (unsigned)(tc.nyA / 128), (unsigned)(tc.T * tc.split));
        switch (tc.Cp) {
            case 4: e = cudaLaunchKernelEx(&cfg, k_tc_adjoint<4>, tc.tm_ga_hi, tc.tm_ga_lo, tc.tm_p0, tc.tm_kd, P); break;
            case 8: e = cudaLaunchKernelEx(&cfg, k_tc_adjoint<8>, tc.tm_ga_hi, tc.tm_ga_lo, tc.tm_p0, tc.tm_kd, P); break;
            case 16: e = cudaLaunchKernelEx(&cfg, k_tc_adjoint<16>, tc.tm_ga_hi, tc.tm_ga_lo, tc.tm_p0, tc.tm_kd, P); break;
            default: e = cudaLaunchKernelEx(&cfg, k_tc_adjoint<32>, tc.tm_ga_hi, tc.tm_ga_lo, tc.tm_p0, tc.tm_kd, P); break;
        }
    }
    if (e != cudaSuccess) {
        tc_last_error() = cudaGetErrorString(e);
        return 3;
    }
    {
        const cudaError_t le = cudaGetLastError();
        if (le != cudaSuccess) {
            tc_last_error() = cudaGetErrorString(le);
            return 3;
        }
    }
    return 0;
}

}  // namespace csr
