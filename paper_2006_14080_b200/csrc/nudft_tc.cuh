// tcgen05 tensor-core separable NUDFT (K3 forward / K4 adjoint).
//
// Complex products are real GEMMs over an interleaved K axis: an operand
// row holding complex values (re, im) along K multiplies a "doubled" row
// pair [re, -im] / [im, re] of the other operand, giving Re and Im output
// columns with no wasted MACs.  fp32 precision comes from a 3-term fp16
// split (a = hi + lo, a*b ~ hi*hi + hi*lo + lo*hi, fp32 accumulation in
// TMEM): 3 kind::f16 MMAs per K step.  Operands that are not unit-modulus
// are scaled by an exact power of two so they sit well inside fp16 range.
//
// Layouts (all fp16, K-major, rows of 128 bytes per K block, TMA SWIZZLE_128B):
//   forward A  fa[t*Mk + k][2y+{0,1}]          = P1[t][k][y]           (static)
//   forward B  xb[t*Nf + 2(x*Cp+c)+part][2y+.] = [Xr,-Xi] / [Xi,Xr],   X = s_c*img_t
//   adjoint A  ga[t*nyA + y][2k+{0,1}]         = conj(P1[t][k][y])     (static)
//   adjoint B  generated in shared memory from P0 and d:
//              row 2(x*Cp+c)+part, K (k, re/im):  W = sigma_d conj(P0[k,x]) d[k,c]
// Forward epilogue (per sample k = TMEM lane): kd[k,c] = sum_x P0[k,x] G[k,(x,c)]
// Adjoint epilogue (per pixel row y = TMEM lane): sum_c conj(s_c[x,y]) D[y,(x,c)],
// written as split-K partial images ws[s][t][x][y].
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdint>
#include <string>
#include <vector>

#include "common.cuh"
#include "sm100.cuh"

namespace csr {

constexpr int TC_BM = 128;
constexpr int TC_BN = 256;
constexpr int TC_A_TILE = TC_BM * 128;   // 16 KiB
constexpr int TC_B_TILE = TC_BN * 128;   // 32 KiB
constexpr int TC_STAGES = 2;
constexpr int TC_FWD_OPS = 2 * TC_A_TILE + 2 * TC_B_TILE;  // 96 KiB / stage
constexpr int TC_FWD_THREADS = 192;   // TMA, MMA, 4 epilogue warps
constexpr int TC_MAX_CHAIN = 24;      // max k blocks (32 samples) per accumulation chain

struct TcPlan {
    bool enabled = false;
    int split = 1;
    float2 *ws = nullptr;
    int fwd_launches = 4, adj_launches = 1;
    // geometry
    int T = 1, nx = 0, ny = 0, C = 0;
    int64_t M = 0, Mk = 0;
    int Cp = 4, xs = 32, nxp = 0, nyp = 0, nyA = 0, Kf = 0, Nf = 0;
    int nt = 1, mt_f = 1, G = 1, nt_per_group = 1, mt_a = 1, kb_total = 1, kb_per_split = 1;
    bool fwd_ts = false;  // A-stationary forward (2*nyp <= 256)
    unsigned long long *trace = nullptr;  // CSR_TRACE: per-CTA timestamps
    unsigned long long *probe = nullptr;   // [PROBE_SLOTS][4] live timing slots
    int fexp = 0, aexp = 0;               // CSR_FEXP / CSR_EXP profiling flags
    int fts_ctas = 1, fts_smem = 0, fts_pieces = 1;
    unsigned *ftick = nullptr;             // forward piece tickets [T * mt_f]
    int raw_bytes = 0, adj_stage = 0, adj_nraw = 4, fwd_smem = 0, adj_smem = 0;
    // operands
    __half *fa_hi = nullptr, *fa_lo = nullptr, *ga_hi = nullptr, *ga_lo = nullptr;
    __half *xb_hi = nullptr, *xb_lo = nullptr;
    float2 *p0p = nullptr, *kdp = nullptr, *kdi = nullptr;
    const float2 *sens = nullptr;
    float *scales = nullptr;  // [4] max|s|, [5] max|kd|, [6] max|img| (component-wise);
                              // operand scales are pow2_scale() of these bounds
    double *red = nullptr;
    unsigned *tick = nullptr;
    CUtensorMap tm_fa_hi, tm_fa_lo, tm_xb_hi, tm_xb_lo, tm_ga_hi, tm_ga_lo, tm_p0, tm_kd;
    CUtensorMap tm_xb256_hi, tm_xb256_lo;
};

// last CUDA error string of a failed tensor-core launch (for csr_last_error)
inline std::string &tc_last_error() {
    static thread_local std::string e;
    return e;
}

// ---------------------------------------------------------------------------
// small helpers
__device__ __forceinline__ void split16(float v, __half &hi, __half &lo) {
    hi = __float2half_rn(v);
    lo = __float2half_rn(v - __half2float(hi));
}
__device__ __forceinline__ uint32_t pack2(__half a, __half b) {
    return (uint32_t)__half_as_ushort(a) | ((uint32_t)__half_as_ushort(b) << 16);
}
__device__ __forceinline__ __half hneg(__half a) {
    return __ushort_as_half(__half_as_ushort(a) ^ 0x8000u);
}

// ---------------------------------------------------------------------------
// setup kernels (plan build)
// lane_major (A-stationary forward): [row / 128][Kf / 8][row % 128][4 pairs],
// so that the 32 lanes of a warp (32 consecutive rows) read one 16-byte chunk
// each from 512 contiguous bytes when they load their rows into TMEM
__global__ void k_tc_build_fa(const float2 *__restrict__ P1, int T, int64_t M, int64_t Mk,
                              int ny, int Kf, __half *hi, __half *lo, int lane_major) {
    pdl_enter();
    const int hk = Kf / 2;
    int64_t total = (int64_t)T * Mk * hk;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int y = (int)(i % hk);
        int64_t r = i / hk;
        int64_t k = r % Mk;
        int t = (int)(r / Mk);
        float2 v = (k < M && y < ny) ? P1[((int64_t)t * M + k) * ny + y] : make_float2(0.f, 0.f);
        __half h0, l0, h1, l1;
        split16(v.x, h0, l0);
        split16(v.y, h1, l1);
        const int64_t o = lane_major
                              ? (((r >> 7) * (hk / 4) + (y >> 2)) * 128 + (r & 127)) * 4 + (y & 3)
                              : i;
        reinterpret_cast<uint32_t *>(hi)[o] = pack2(h0, h1);
        reinterpret_cast<uint32_t *>(lo)[o] = pack2(l0, l1);
    }
}

__global__ void k_tc_build_ga(const float2 *__restrict__ P1, int T, int64_t M, int64_t Mk,
                              int ny, int nyA, __half *hi, __half *lo) {
    pdl_enter();
    int64_t total = (int64_t)T * nyA * Mk;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t k = i % Mk;
        int64_t r = i / Mk;
        int y = (int)(r % nyA);
        int t = (int)(r / nyA);
        float2 v = (k < M && y < ny) ? P1[((int64_t)t * M + k) * ny + y] : make_float2(0.f, 0.f);
        __half h0, l0, h1, l1;
        split16(v.x, h0, l0);
        split16(-v.y, h1, l1);  // conj
        reinterpret_cast<uint32_t *>(hi)[i] = pack2(h0, h1);
        reinterpret_cast<uint32_t *>(lo)[i] = pack2(l0, l1);
    }
}

__global__ void k_tc_build_p0(const float2 *__restrict__ P0, int T, int64_t M, int64_t Mk,
                              int nx, int nxp, float2 *out) {
    pdl_enter();
    int64_t total = (int64_t)T * Mk * nxp;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int x = (int)(i % nxp);
        int64_t r = i / nxp;
        int64_t k = r % Mk;
        int t = (int)(r / Mk);
        out[i] = (k < M && x < nx) ? P0[((int64_t)t * M + k) * nx + x] : make_float2(0.f, 0.f);
    }
}

// scales[4] = max component magnitude of the coil maps
__global__ void k_tc_sens_absmax(const float2 *__restrict__ s, int64_t n, double *partials,
                                 unsigned *ticket, float *scales) {
    pdl_enter();
    float v = 0.f;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        v = fmaxf(v, fmaxf(fabsf(s[i].x), fabsf(s[i].y)));
    float m;
    if (grid_max(v, partials, ticket, m)) scales[4] = m;
}

// ---------------------------------------------------------------------------
// per-application kernels
struct TcArgs {
    int T, nx, ny, C, Cp, xs, nxp, nyA, Kf, Nf;
    int64_t M, Mk;
};

// sigma_x for the image operand X = s_c * img: bound = 2 max|s| max|img|
__global__ void k_tc_absmax_img(const float2 *__restrict__ img, int64_t n, double *partials,
                                unsigned *ticket, float *scales, const int *gate) {
    pdl_enter();
    if (gate && !*gate) return;
    float v = 0.f;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        v = fmaxf(v, fmaxf(fabsf(img[i].x), fabsf(img[i].y)));
    float m;
    if (grid_max(v, partials, ticket, m)) scales[6] = m;
}

// X' = split(sigma_x * s_c * img_t) laid out as doubled rows (x, c, part)
__global__ void k_tc_prep_x(TcArgs a, const float2 *__restrict__ img,
                            const float2 *__restrict__ sens, float *scales,
                            __half *hi, __half *lo, const int *gate,
                            unsigned long long *probe) {
    pdl_enter();
    if (gate && !*gate) return;
    probe_enter(probe);
    // exact power-of-two scale: |s_c * img| <= 2 max|s| max|img| (component-wise)
    const float sg = pow2_scale(2.f * scales[4] * scales[6]);
    if (blockIdx.x == 0 && threadIdx.x == 0) scales[5] = 0.f;  // k-space max (atomicMax)
    const int hy = a.Kf / 2;  // complex y per row (nyp)
    int64_t total = (int64_t)a.T * a.nxp * a.Cp * hy;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int y = (int)(i % hy);
        int64_t r = i / hy;
        int c = (int)(r % a.Cp);
        r /= a.Cp;
        int x = (int)(r % a.nxp);
        int t = (int)(r / a.nxp);
        float2 v = make_float2(0.f, 0.f);
        if (x < a.nx && c < a.C && y < a.ny) {
            int64_t p = (int64_t)x * a.ny + y;
            v = cmul(sens[(int64_t)c * a.nx * a.ny + p], img[(int64_t)t * a.nx * a.ny + p]);
            v.x *= sg;
            v.y *= sg;
        }
        __half rh, rl, ih, il;
        split16(v.x, rh, rl);
        split16(v.y, ih, il);
        int64_t row = (int64_t)t * a.Nf + 2 * ((int64_t)x * a.Cp + c);
        int64_t e = row * (a.Kf / 2) + y;               // uint32 (half2) index
        int64_t e1 = e + a.Kf / 2;                      // next row (Im part)
        uint32_t *H = reinterpret_cast<uint32_t *>(hi), *L = reinterpret_cast<uint32_t *>(lo);
        H[e] = pack2(rh, hneg(ih));
        L[e] = pack2(rl, hneg(il));
        H[e1] = pack2(ih, rh);
        L[e1] = pack2(il, rl);
    }
    probe_exit(probe);
}

struct FwdParams {
    unsigned long long *probe;  // live timing slot (probe_enter/exit) or null
    TcArgs a;
    int mt_per_frame, nt_per_group;
    int amax;  // 1: kdp aliases the k-space buffer; atomicMax |kd| into scales[5]
    const float2 *p0p;
    float2 *kdp;  // [G][T][Mk][Cp]
    const float *scales;
    const int *gate;
};


// (offset arithmetic on the __shared__ pointer itself keeps the compiler's
// address-space inference: LDS, not generic LD, for the smem operands)
__device__ __forceinline__ uint8_t *align1024(uint8_t *p) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
    return p + ((1024u - (a & 1023u)) & 1023u);
}

template <int CP>
__global__ void __launch_bounds__(TC_FWD_THREADS, 1)
    k_tc_forward(const __grid_constant__ CUtensorMap tmA_hi,
                 const __grid_constant__ CUtensorMap tmA_lo,
                 const __grid_constant__ CUtensorMap tmB_hi,
                 const __grid_constant__ CUtensorMap tmB_lo, FwdParams P) {
    pdl_enter();
    using namespace sm100;
    if (P.gate && !*P.gate) return;
    probe_enter(P.probe);
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = align1024(smem_raw);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + TC_STAGES * TC_FWD_OPS);
    uint64_t *empty = full + TC_STAGES;
    uint64_t *tfull = empty + TC_STAGES;
    uint64_t *tempty = tfull + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

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
        for (int s = 0; s < TC_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 4);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            int it = 0;
            for (int nt = nt0; nt < nt1; ++nt) {
                const int brow = t * P.a.Nf + nt * TC_BN;
                for (int kb = 0; kb < nkb; ++kb, ++it) {
                    const int s = it % TC_STAGES;
                    const uint32_t ph = (it / TC_STAGES) & 1;
                    mbar_wait(&empty[s], ph ^ 1);
                    uint8_t *st = smem + s * TC_FWD_OPS;
                    mbar_arrive_expect_tx(&full[s], TC_FWD_OPS);
                    tma_load_2d(st, &tmA_hi, &full[s], kb * 64, mtile * TC_BM);
                    tma_load_2d(st + TC_A_TILE, &tmA_lo, &full[s], kb * 64, mtile * TC_BM);
                    tma_load_2d(st + 2 * TC_A_TILE, &tmB_hi, &full[s], kb * 64, brow);
                    tma_load_2d(st + 2 * TC_A_TILE + TC_B_TILE, &tmB_lo, &full[s], kb * 64, brow);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_f16(TC_BM, TC_BN);
            int it = 0, tc = 0;
            for (int nt = nt0; nt < nt1; ++nt, ++tc) {
                const int ab = tc & 1;
                const uint32_t aph = (tc >> 1) & 1;
                mbar_wait(&tempty[ab], aph ^ 1);
                tc_fence_after();
                const uint32_t dcol = tmem + ab * TC_BN;
                for (int kb = 0; kb < nkb; ++kb, ++it) {
                    const int s = it % TC_STAGES;
                    const uint32_t ph = (it / TC_STAGES) & 1;
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    const uint32_t st = smem_u32(smem + s * TC_FWD_OPS);
                    const uint32_t a_hi = st, a_lo = st + TC_A_TILE;
                    const uint32_t b_hi = st + 2 * TC_A_TILE, b_lo = b_hi + TC_B_TILE;
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const uint32_t o = kk * 32;
                        const uint64_t dah = desc_sw128(a_hi + o), dal = desc_sw128(a_lo + o);
                        const uint64_t dbh = desc_sw128(b_hi + o), dbl = desc_sw128(b_lo + o);
                        mma_f16_fill(dcol, dah, dbh, idesc, (kb | kk) != 0);
                        mma_f16_lastuse(dcol, dah, dbl, idesc, 1);
                        mma_f16(dcol, dal, dbh, idesc, 1);
                    }
                    mma_commit(&empty[s]);
                }
                mma_commit(&tfull[ab]);
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
            for (int chb = 0; chb < 8; chb += U) {
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
            if (lane == 0) mbar_arrive(&tempty[ab]);
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
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
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

template <int CP>
__global__ void __launch_bounds__(FTS_THREADS, 1)
    k_tc_forward_ts(const __grid_constant__ CUtensorMap tmB_hi,
                    const __grid_constant__ CUtensorMap tmB_lo, FwdTsParams P) {
    using namespace sm100;
    // Prologue overlapped with the previous kernel (programmatic launch):
    // barrier init, TMEM allocation and the first segment's A rows read only
    // static data; everything else waits in pdl_wait().
    pdl_trigger();
    constexpr int XQ = 32 / CP;  // x values per 64-column accumulator quarter
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = align1024(smem_raw);
    constexpr int STAGE = 2 * FTS_B_TILE;  // one K block: [hi | lo] x 256 rows
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + FTS_STAGES * STAGE);
    uint64_t *empty = full + FTS_STAGES;
    uint64_t *tfull = empty + FTS_STAGES;
    uint64_t *tempty = tfull + 1;
    uint64_t *a_ready = tempty + 1;
    uint64_t *a_free = a_ready + 1;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(a_free + 1);
    __shared__ float2 part_acc[128][CP + 1];  // row sums folded across the quarters

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int G = gridDim.x;
    const int64_t U = P.units;
    const int NT = P.nt_tiles;
    const int64_t u0 = fts_u0(U, G, blockIdx.x), u1 = fts_u0(U, G, blockIdx.x + 1);
    const int nkb = P.a.Kf / 64;
    unsigned long long *tr = P.trace ? P.trace + (size_t)blockIdx.x * 32 : nullptr;
    if (tr && threadIdx.x == 0) tr[0] = gtimer();

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tmB_hi);
        tma_prefetch(&tmB_lo);
        for (int s = 0; s < FTS_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tfull, 1);
        mbar_init(tempty, 16);
        mbar_init(a_ready, 16);
        mbar_init(a_free, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
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
    if (warp >= 2 && u0 < u1) {
        const int q = warp & 3;
        load_a(u0 / NT, tmem + ((uint32_t)(q * 32) << 16), q * 32 + lane, (warp - 2) >> 2);
        if (tr && threadIdx.x == 64) tr[5] = gtimer();
    }

    pdl_wait();
    const bool run = !P.gate || *P.gate;
    if (run) probe_enter(P.probe);

    if (!run) {
    } else if (warp == 0) {
        // ---- TMA producer over the CTA's units
        if (lane == 0) {
            int it = 0;
            for (int64_t u = u0; u < u1; ++u) {
                const int64_t m = u / NT;
                const int nt = (int)(u - m * NT);
                const int t = (int)(m / P.mt_per_frame);
                const int brow = t * P.a.Nf + nt * 256;
                for (int kb = 0; kb < nkb; ++kb, ++it) {
                    const int s = it % FTS_STAGES;
                    const uint32_t ph = (it / FTS_STAGES) & 1;
                    mbar_wait(&empty[s], ph ^ 1);
                    uint8_t *st = smem + s * STAGE;
                    mbar_arrive_expect_tx(&full[s], (P.exp_flags & 2) ? 0 : STAGE);
                    if (!(P.exp_flags & 2)) {
                        tma_load_2d(st, &tmB_hi, &full[s], kb * 64, brow);
                        tma_load_2d(st + FTS_B_TILE, &tmB_lo, &full[s], kb * 64, brow);
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---- MMA issuer
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_f16(128, 256);
            const uint32_t a_hi = tmem, a_lo = tmem + 128, dcol = tmem + 256;
            int it = 0, tc = 0, seg = 0;
            int64_t m_prev = -1;
            for (int64_t u = u0; u < u1; ++u, ++tc) {
                const int64_t m = u / NT;
                if (m != m_prev) {  // new segment: wait for its A
                    if (m_prev >= 0) mma_commit(a_free);  // old A is free after these MMAs
                    mbar_wait(a_ready, seg & 1);
                    tc_fence_after();
                    if (tr && seg < 2) tr[2 + seg * 4] = gtimer();
                    ++seg;
                    m_prev = m;
                }
                mbar_wait(tempty, (tc & 1) ^ 1);  // the epilogue has read the last unit
                tc_fence_after();
                for (int kb = 0; kb < nkb; ++kb, ++it) {
                    const int s = it % FTS_STAGES;
                    const uint32_t ph = (it / FTS_STAGES) & 1;
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    const uint32_t st = smem_u32(smem + s * STAGE);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const uint32_t ac = kb * 32 + kk * 8;
                        const uint64_t dbh = desc_sw128(st + kk * 32);
                        const uint64_t dbl = desc_sw128(st + FTS_B_TILE + kk * 32);
                        if (P.exp_flags & 1) continue;
                        mma_f16_ts(dcol, a_hi + ac, dbh, idesc, (kb | kk) != 0);
                        mma_f16_ts(dcol, a_hi + ac, dbl, idesc, 1);
                        mma_f16_ts(dcol, a_lo + ac, dbh, idesc, 1);
                    }
                    mma_commit(&empty[s]);
                }
                mma_commit(tfull);
                if (tr && tc < 8) tr[16 + tc] = gtimer();
            }
            if (tr) tr[3] = gtimer();
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
            const int64_t m = us / NT;
            const int64_t ue = min(u1, (m + 1) * NT);
            const int t = (int)(m / P.mt_per_frame);
            const bool last_seg = ue == u1;
            const int64_t kloc = (int64_t)(m % P.mt_per_frame) * 128 + row;
            const bool valid = kloc < P.a.M;
            const float2 *p0row = P.p0p + ((int64_t)t * Mk + kloc) * P.a.nxp;
            const int b_first = fts_owner(U, G, m * NT);
            const int b_last = fts_owner(U, G, (m + 1) * NT - 1);
            const int npieces = b_last - b_first + 1;
            const int piece = blockIdx.x - b_first;
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
                if (u + 1 == ue && !last_seg) {
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
                        const unsigned *flag = P.tick + m * 4 + pc;
                        do {
                            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];"
                                         : "=r"(f) : "l"(flag) : "memory");
                        } while (f == 0u);
                    }
                }
                mbar_wait(tfull, tc & 1);
                tc_fence_after();
                // this quarter (64 columns) in two 32-column reads; the
                // accumulator is released right after the second read
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    uint32_t r[32];
                    tmem_ld32(lane_base + 256 + qt * 64 + hh * 32, r);
                    tmem_ld_wait();
                    if (hh == 1) {
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(tempty);
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
                                     ::"l"(P.tick + m * 4 + piece), "r"(1u) : "memory");
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
                            P.tick[m * 4 + 1 + (threadIdx.x - 64)] = 0u;  // re-arm
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
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// kd = sum_g kdp[g]; writes the internal padded layout (and optionally a
// user (T*M, C) layout); sigma_d from max|kd|
__global__ void k_tc_sum_kd(TcArgs a, int G, const float2 *__restrict__ kdp, float2 *kdi,
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
constexpr int ADJ_THREADS = (ADJ_W_EPI + 4) * 32;
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
        mbar_init(acc_empty, 4);
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
        // ---- MMA issuer
        if (lane == 0) {
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
                    ADJ_TL(0, true);
                    wait_fast(&full[s], ph);
                    tc_fence_after();
                    const uint32_t st = smem_u32(smem + s * ADJ_B_STAGE);
                    const uint32_t a_hi = tmem + 256 + 64 * s, a_lo = a_hi + 32;
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
                mma_commit(acc_full);
            }
            if (tr) {
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
    float sum[128];  // epilogue warps: running sums of row m over the 128 y
    if (run && warp >= ADJ_W_EPI) {
        // ---- epilogue: drain every chain into the register sums
        const int q = warp & 3;
        const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
#pragma unroll
        for (int y = 0; y < 128; ++y) sum[y] = 0.f;
        for (int ch = 0; ch < nchain; ++ch) {
            wait_slow(acc_full, ch & 1);
            tc_fence_after();
#pragma unroll
            for (int cb = 0; cb < 8; ++cb) {
                uint32_t rh[16], rl[16];
                tmem_ld16(lane_base + cb * 16, rh);
                tmem_ld16(lane_base + 128 + cb * 16, rl);
                tmem_ld_wait();
                if (cb == 7) {  // accumulator fully read: let the MMA go on
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
        for (int y = 0; y < 128; ++y) sum_s[y * ADJ_SUM_LD + m] = sum[y];
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

inline int tc_plan_build(TcPlan &tc, int T, int nx, int ny, int C, int64_t M,
                         const float2 *P0, const float2 *P1, const float2 *sens,
                         cudaStream_t st, int64_t *factor_bytes, int64_t *ws_bytes,
                         std::vector<void *> &allocs) {
    tc.enabled = false;
    if (C > 16 || getenv("CSR_DISABLE_TC")) return 0;
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
    tc.nt = tc.Nf / TC_BN;
    tc.mt_f = (int)(tc.Mk / TC_BM);
    // forward groups: split the n-tiles so the grid covers the machine
    const int64_t mtiles = (int64_t)T * tc.mt_f;
    int G = 1;
    while (G < tc.nt && mtiles * G < 2 * 148 && tc.nt % (2 * G) == 0) G *= 2;
    tc.G = G;
    tc.nt_per_group = tc.nt / G;
    // A-stationary forward: 128-row B tiles; groups of tiles per CTA chosen
    // by waves x per-CTA time (tiles x K blocks x ~768 MMA cycles + setup)
    tc.fwd_ts = tc.Kf <= 256 && !getenv("CSR_FWD_SS");
    if (tc.fwd_ts) {
        const int NTt = tc.Nf / 256;
        const int64_t units = mtiles * NTt;
        tc.fts_smem = FTS_STAGES * 2 * FTS_B_TILE + 1024 + 256;
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
            for (int64_t m = 0; m < mtiles; ++m)
                mp = std::max<int>(mp, (int)(owner((m + 1) * NTt - 1) - owner(m * NTt) + 1));
            return mp;
        };
        int64_t Gc = std::min<int64_t>(148, units);
        int maxp = max_pieces(Gc);
        while (maxp > 4 && Gc > mtiles) maxp = max_pieces(--Gc);
        tc.fts_ctas = (int)Gc;
        G = std::max(G, maxp - 1);  // kdp holds pieces 1.. (piece 0 stays in registers)
        tc.fts_pieces = maxp;
    }
    // adjoint split-K
    tc.mt_a = tc.nxp * Cp / 64;  // adjoint tiles over (x, c): 64 per tile
    tc.kb_total = (int)(tc.Mk / 32);
    const int64_t tiles = (int64_t)T * tc.mt_a * (tc.nyA / 128);
    // split-K: each CTA takes one tile and a contiguous k range, cut into
    // accumulation chains of <= TC_MAX_CHAIN blocks.  Pick S by a cost model
    // (waves of 148 CTAs x per-CTA time: blocks x ~768 MMA cycles + chain
    // drains + CTA setup/fill), bounded by the partial-image memory.
    int S = 1;
    {
        const int64_t pix = (int64_t)T * nx * ny * 8;
        int64_t best_cost = INT64_MAX;
        for (int c = 1; c <= std::min(tc.kb_total, 1024); ++c) {
            if (c > 1 && c * pix > ((int64_t)1 << 30)) break;
            const int64_t kbps = (tc.kb_total + c - 1) / c;
            const int64_t nch = (kbps + TC_MAX_CHAIN - 1) / TC_MAX_CHAIN;
            const int64_t waves = (tiles * c + 147) / 148;
            const int64_t cost = waves * (kbps * 768 + nch * 700 + 4000);
            if (cost < best_cost) {
                best_cost = cost;
                S = c;
            }
        }
    }
    if (const char *e = getenv("CSR_TC_SPLIT")) S = std::max(1, std::min(atoi(e), tc.kb_total));
    tc.kb_per_split = (tc.kb_total + S - 1) / S;
    S = (tc.kb_total + tc.kb_per_split - 1) / tc.kb_per_split;
    tc.split = S;
    tc.raw_bytes = 32 * (64 / Cp) * 8 + 32 * Cp * 8;
    tc.adj_stage = adj_in_stage_bytes(Cp);  // input ring stage
    tc.fwd_smem = TC_STAGES * TC_FWD_OPS + 1024 + 256;
    {
        const int fixed = ADJ_STAGES * ADJ_B_STAGE + 1024 + 512;
        tc.adj_nraw = std::min(ADJ_MAX_RAW, (227 * 1024 - fixed) / tc.adj_stage);
        if (const char *e = getenv("CSR_ADJ_NRAW"))
            tc.adj_nraw = std::max(1, std::min(tc.adj_nraw, atoi(e)));
        tc.adj_smem = fixed + tc.adj_nraw * tc.adj_stage;
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
           tc.fwd_ts ? 1 : 0);
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
              tmap_f16_2d(&tc.tm_xb256_hi, tc.xb_hi, tc.Kf, (uint64_t)T * tc.Nf, 256) &&
              tmap_f16_2d(&tc.tm_xb256_lo, tc.xb_lo, tc.Kf, (uint64_t)T * tc.Nf, 256) &&
              tmap_f16_2d(&tc.tm_ga_hi, tc.ga_hi, 2 * tc.Mk, (uint64_t)T * tc.nyA, 128) &&
              tmap_f16_2d(&tc.tm_ga_lo, tc.ga_lo, 2 * tc.Mk, (uint64_t)T * tc.nyA, 128) &&
              tmap_c64_3d(&tc.tm_p0, tc.p0p, tc.nxp, tc.Mk, T, 64 / Cp, 32) &&
              tmap_c64_3d(&tc.tm_kd, tc.kdi, Cp, tc.Mk, T, Cp, 32);
    if (!ok) return 0;  // descriptor encode unavailable: SIMT path
    switch (Cp) {
        case 4: set_smem(k_tc_forward<4>, tc.fwd_smem); set_smem(k_tc_adjoint<4>, tc.adj_smem); break;
        case 8: set_smem(k_tc_forward<8>, tc.fwd_smem); set_smem(k_tc_adjoint<8>, tc.adj_smem); break;
        case 16: set_smem(k_tc_forward<16>, tc.fwd_smem); set_smem(k_tc_adjoint<16>, tc.adj_smem); break;
        default: break;
    }
    if (tc_alloc(allocs, &p, PROBE_SLOTS * 4 * sizeof(unsigned long long), ws_bytes, st)) return 2;
    tc.probe = (unsigned long long *)p;
    cudaMemsetAsync(tc.probe, 0, PROBE_SLOTS * 4 * sizeof(unsigned long long), st);
    tc.fexp = getenv("CSR_FEXP") ? atoi(getenv("CSR_FEXP")) : 0;
    tc.aexp = getenv("CSR_EXP") ? atoi(getenv("CSR_EXP")) : 0;
    if (getenv("CSR_TRACE")) {
        if (tc_alloc(allocs, &p, 4096 * 32 * 8, ws_bytes, st)) return 2;
        tc.trace = (unsigned long long *)p;
        cudaMemsetAsync(tc.trace, 0, 4096 * 32 * 8, st);
    }
    set_smem(k_tc_forward_ts<4>, tc.fts_smem);
    set_smem(k_tc_forward_ts<8>, tc.fts_smem);
    set_smem(k_tc_forward_ts<16>, tc.fts_smem);
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
        int64_t total = (int64_t)tc.T * tc.nxp * tc.Cp * tc.nyp;
        int nb = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
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
        P.units = (int64_t)tc.T * tc.mt_f * P.nt_tiles;
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
            case 4: launch(k_tc_forward_ts<4>, grid, FTS_THREADS, tc.fts_smem, st, tc.tm_xb256_hi, tc.tm_xb256_lo, P); break;
            case 8: launch(k_tc_forward_ts<8>, grid, FTS_THREADS, tc.fts_smem, st, tc.tm_xb256_hi, tc.tm_xb256_lo, P); break;
            default: launch(k_tc_forward_ts<16>, grid, FTS_THREADS, tc.fts_smem, st, tc.tm_xb256_hi, tc.tm_xb256_lo, P); break;
        }
        if (user) {  // (T*M, C) copy for the caller
            int64_t total = (int64_t)tc.T * tc.Mk * tc.Cp;
            launch(k_tc_sum_kd, reduce_blocks(total, 256), 256, 0, st, a, 1, tc.kdi, tc.kdi, user,
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
        dim3 grid((unsigned)(tc.T * tc.mt_f), (unsigned)G);
        switch (tc.Cp) {
            case 4: launch(k_tc_forward<4>, grid, TC_FWD_THREADS, tc.fwd_smem, st, tc.tm_fa_hi, tc.tm_fa_lo, tc.tm_xb_hi, tc.tm_xb_lo, P); break;
            case 8: launch(k_tc_forward<8>, grid, TC_FWD_THREADS, tc.fwd_smem, st, tc.tm_fa_hi, tc.tm_fa_lo, tc.tm_xb_hi, tc.tm_xb_lo, P); break;
            default: launch(k_tc_forward<16>, grid, TC_FWD_THREADS, tc.fwd_smem, st, tc.tm_fa_hi, tc.tm_fa_lo, tc.tm_xb_hi, tc.tm_xb_lo, P); break;
        }
    }
    if (!direct) {
        int64_t total = (int64_t)tc.T * tc.Mk * tc.Cp;
        launch(k_tc_sum_kd, reduce_blocks(total, 256), 256, 0, st, a, G, tc.kdp, tc.kdi, user,
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

// kd already in tc.kdi (with sigma_d) when user == nullptr; else load it
inline int tc_adjoint(TcPlan &tc, const float2 *user, float2 *ws, cudaStream_t st,
                      const int *gate) {
    TcArgs a = tc_args(tc);
    if (user) {
        int64_t total = (int64_t)tc.T * tc.Mk * tc.Cp;
        launch(k_tc_load_kd, reduce_blocks(total, 256), 256, 0, st, a, user, tc.kdi, tc.red, tc.tick,
                                                                tc.scales);
    }
    AdjParams P;
    P.a = a;
    P.S = tc.split;
    P.kb_per_split = tc.kb_per_split;
    P.chain = TC_MAX_CHAIN;
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
    dim3 grid((unsigned)tc.mt_a, (unsigned)(tc.nyA / 128), (unsigned)(tc.T * tc.split));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(ADJ_THREADS);
    cfg.dynamicSmemBytes = tc.adj_smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    cudaError_t e;
    switch (tc.Cp) {
        case 4: e = cudaLaunchKernelEx(&cfg, k_tc_adjoint<4>, tc.tm_ga_hi, tc.tm_ga_lo, tc.tm_p0, tc.tm_kd, P); break;
        case 8: e = cudaLaunchKernelEx(&cfg, k_tc_adjoint<8>, tc.tm_ga_hi, tc.tm_ga_lo, tc.tm_p0, tc.tm_kd, P); break;
        default: e = cudaLaunchKernelEx(&cfg, k_tc_adjoint<16>, tc.tm_ga_hi, tc.tm_ga_lo, tc.tm_p0, tc.tm_kd, P); break;
    }
    if (e != cudaSuccess) return 3;
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
