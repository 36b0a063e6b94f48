// tcgen05 tensor-core separable NUDFT: shared plan state and helpers.
//
// Complex products are real GEMMs over an interleaved K axis: an operand
// row holding complex values (re, im) along K multiplies a "doubled" row
// pair [re, -im] / [im, re] of the other operand, giving Re and Im output
// columns with no wasted MACs.  fp32 precision comes from a 3-term fp16
// split (a = hi + lo, a*b ~ hi*hi + hi*lo + lo*hi, fp32 accumulation in
// TMEM).  Operands that are not unit-modulus are scaled by an exact power
// of two so they sit well inside fp16 range.
//
// Layouts (fp16, K-major, 128-byte rows per K block, TMA SWIZZLE_128B):
//   forward A  fa[t*Mk + k][2y+{0,1}]          = P1[t][k][y]  (static; lane-major
//              copy for the TMEM-resident forward, tc_forward.cuh)
//   forward B  xb[t*Nf + 2(x*Cp+c)+part][2y+.] = [Xr,-Xi] / [Xi,Xr],  X = s_c*img_t
//   adjoint B  ga[t*nyA + y][2k+{0,1}]         = conj(P1[t][k][y])   (static)
//   adjoint A  generated in TMEM from P0 and d (tc_adjoint.cuh):
//              row 2(x*Cp+c)+part, K (k, re/im):  W = sigma_d conj(P0[k,x]) d[k,c]
// Forward epilogue (per sample k = TMEM lane): kd[k,c] = sum_x P0[k,x] G[k,(x,c)]
// Adjoint epilogue (per row (x, c, part) = TMEM lane, 128 pixel rows y per
// tile): sum_c conj(s_c[x,y]) (re + i im), written as split-K partial
// images ws[s][t][x][y].
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
#ifndef TC_CHAIN
#define TC_CHAIN 24
#endif
constexpr int TC_MAX_CHAIN = TC_CHAIN;  // max k blocks (32 samples) per accumulation chain
#ifndef TC_ADJW_CHAIN
#define TC_ADJW_CHAIN 12  // the wide adjoint's chains (one accumulator, 3 MMAs per K step)
#endif
// coils a tensor-core plan holds (padded to CP = 4, 8, 16, 32: 64 / CP x
// values per adjoint tile row block; the P0 input box of the adjoint needs
// >= 2 of them, TMA boxes being multiples of 16 bytes); more go to the SIMT
// kernels
constexpr int TC_MAX_COILS = 32;

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
    bool fwd_ps = false;  // its PS form (A from shared memory, two accumulators)
    bool fwd_pair = false;  // the PS form on CTA pairs (cta_group::2)
    unsigned long long *trace = nullptr;  // CSR_TRACE: per-CTA timestamps
    unsigned long long *probe = nullptr;   // [PROBE_SLOTS][4] live timing slots
    int fexp = 0, aexp = 0;               // CSR_FEXP / CSR_EXP profiling flags
    int fts_ctas = 1, fts_smem = 0, fts_pieces = 1;
    unsigned *ftick = nullptr;             // forward piece tickets [T * mt_f]
    int raw_bytes = 0, adj_stage = 0, adj_nraw = 4, fwd_smem = 0, adj_smem = 0;
    int adj_chain = TC_MAX_CHAIN;
    // wide adjoint (k_tc_adjoint_w, 128 < ny): N-row y tiles, stages, smem
    bool adj_w = false;
    int adjw_N = 128, adjw_nyt = 1, adjw_NA = 4, adjw_NB = 2, adjw_nraw = 2, adjw_smem = 0;
    int adjw_CL = 1;  // CTA-pair clusters multicasting B
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
    CUtensorMap tm_gaw_hi, tm_gaw_lo;  // N-row boxes of ga (wide adjoint)
    CUtensorMap tm_xb128_hi, tm_xb128_lo;  // half-tile boxes of xb (CTA-pair forwards)
    int fwd_CL = 1;  // SS forward: CTA-pair clusters multicasting the image operand
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

// The forward's fp16 hi/lo operand entries of pixel (t, x, y) of image value
// v: rows (x, c, Re/Im) doubled, X = sigma * s_c * v (valid x < nx, c < C,
// y < ny only: the zero padding is written once at plan build).  Coil maps
// are loaded four at a time (all in flight before the stores).
constexpr int XOP_COILS = 4;
__device__ __forceinline__ void write_xop(const TcArgs &a, const float2 *__restrict__ sens,
                                          __half *xb_hi, __half *xb_lo, int t, int x, int y,
                                          int64_t nxy, float2 v, float sg) {
    const int hy = a.Kf / 2;  // complex y per row (nyp)
    uint32_t *H = reinterpret_cast<uint32_t *>(xb_hi);
    uint32_t *L = reinterpret_cast<uint32_t *>(xb_lo);
    const int64_t p = (int64_t)x * a.ny + y;
    for (int c0 = 0; c0 < a.C; c0 += XOP_COILS) {
        float2 sv[XOP_COILS];
#pragma unroll
        for (int j = 0; j < XOP_COILS; ++j)
            sv[j] = c0 + j < a.C ? sens[(int64_t)(c0 + j) * nxy + p] : make_float2(0.f, 0.f);
#pragma unroll
        for (int j = 0; j < XOP_COILS; ++j) {
            const int c = c0 + j;
            if (c >= a.C) break;
            float2 w = cmul(sv[j], v);
            w.x *= sg;
            w.y *= sg;
            __half rh, rl, ih, il;
            split16(w.x, rh, rl);
            split16(w.y, ih, il);
            const int64_t row = (int64_t)t * a.Nf + 2 * ((int64_t)x * a.Cp + c);
            const int64_t e = row * hy + y, e1 = e + hy;
            H[e] = pack2(rh, hneg(ih));
            L[e] = pack2(rl, hneg(il));
            H[e1] = pack2(ih, rh);
            L[e1] = pack2(il, rl);
        }
    }
}

// write_xop for the pixel pair (y, y+1), y even and ny even: 16-byte coil
// map loads and 8-byte stores of the four fp16 words of both pixels
__device__ __forceinline__ void write_xop2(const TcArgs &a, const float2 *__restrict__ sens,
                                           __half *xb_hi, __half *xb_lo, int t, int x, int y,
                                           int64_t nxy, float2 v0, float2 v1, float sg) {
    const int hy = a.Kf / 2;
    uint2 *H = reinterpret_cast<uint2 *>(xb_hi);
    uint2 *L = reinterpret_cast<uint2 *>(xb_lo);
    const float4 *s4 = reinterpret_cast<const float4 *>(sens);
    const int64_t p = (int64_t)x * a.ny + y;
    for (int c0 = 0; c0 < a.C; c0 += XOP_COILS) {
        float4 sv[XOP_COILS];
#pragma unroll
        for (int j = 0; j < XOP_COILS; ++j)
            sv[j] = c0 + j < a.C ? s4[((int64_t)(c0 + j) * nxy + p) >> 1]
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int j = 0; j < XOP_COILS; ++j) {
            const int c = c0 + j;
            if (c >= a.C) break;
            float2 w0 = cmul(make_float2(sv[j].x, sv[j].y), v0);
            float2 w1 = cmul(make_float2(sv[j].z, sv[j].w), v1);
            w0.x *= sg; w0.y *= sg; w1.x *= sg; w1.y *= sg;
            __half rh0, rl0, ih0, il0, rh1, rl1, ih1, il1;
            split16(w0.x, rh0, rl0);
            split16(w0.y, ih0, il0);
            split16(w1.x, rh1, rl1);
            split16(w1.y, ih1, il1);
            const int64_t row = (int64_t)t * a.Nf + 2 * ((int64_t)x * a.Cp + c);
            const int64_t e = (row * hy + y) >> 1, e1 = e + (hy >> 1);
            H[e] = make_uint2(pack2(rh0, hneg(ih0)), pack2(rh1, hneg(ih1)));
            L[e] = make_uint2(pack2(rl0, hneg(il0)), pack2(rl1, hneg(il1)));
            H[e1] = make_uint2(pack2(ih0, rh0), pack2(ih1, rh1));
            L[e1] = make_uint2(pack2(il0, rl0), pack2(il1, rl1));
        }
    }
}

// X' = split(sigma_x * s_c * img_t) laid out as doubled rows (x, c, part):
// one thread per pixel (pixel pair when ny is even), all coils (valid
// entries only, see write_xop)
// a deep grid (16 blocks per SM, several waves) measured faster than one
// wave of 5 per SM (config 4: 0.246 vs 0.281 ms)
constexpr int PREP_X_BLOCKS_PER_SM = 16;
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
    const int64_t nxy = (int64_t)a.nx * a.ny;
    const int64_t total = (int64_t)a.T * nxy;
    if ((a.ny & 1) == 0) {
        const float4 *img4 = reinterpret_cast<const float4 *>(img);
        for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < total / 2;
             j += (int64_t)gridDim.x * blockDim.x) {
            const int64_t i = 2 * j;
            int t, x, y;
            if (total <= 0x7fffffff) {
                const unsigned q = (unsigned)i, r = q / (unsigned)a.ny;
                y = (int)(q - r * (unsigned)a.ny);
                t = (int)(r / (unsigned)a.nx);
                x = (int)(r - (unsigned)t * (unsigned)a.nx);
            } else {
                y = (int)(i % a.ny);
                x = (int)((i / a.ny) % a.nx);
                t = (int)(i / nxy);
            }
            const float4 v = img4[j];
            write_xop2(a, sens, hi, lo, t, x, y, nxy, make_float2(v.x, v.y),
                       make_float2(v.z, v.w), sg);
        }
        probe_exit(probe);
        return;
    }
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int t, x, y;
        if (total <= 0x7fffffff) {
            const unsigned q = (unsigned)i, r = q / (unsigned)a.ny;
            y = (int)(q - r * (unsigned)a.ny);
            t = (int)(r / (unsigned)a.nx);
            x = (int)(r - (unsigned)t * (unsigned)a.nx);
        } else {
            y = (int)(i % a.ny);
            x = (int)((i / a.ny) % a.nx);
            t = (int)(i / nxy);
        }
        write_xop(a, sens, hi, lo, t, x, y, nxy, img[i], sg);
    }
    probe_exit(probe);
}

// (offset arithmetic on the __shared__ pointer itself keeps the compiler's
// address-space inference: LDS, not generic LD, for the smem operands)
__device__ __forceinline__ uint8_t *align1024(uint8_t *p) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
    return p + ((1024u - (a & 1023u)) & 1023u);
}

}  // namespace csr
