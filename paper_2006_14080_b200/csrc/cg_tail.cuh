// Fused CG tail (single rank, tensor-core operator): one cooperative kernel
// per CG iteration replaces k_cg_ad + k_cg_xr + k_cg_d + the next forward's
// k_tc_prep_x (solver.py:111-122):
//
//   phase A  Ad = sum_s ws[s] + (beta/2) Theta^H Theta d ;  <d, Ad>
//   barrier  alpha = tau / <d, Ad>                  (every block, same order)
//   phase B  x += alpha d ; r -= alpha Ad ;  ||r||^2, max|r|
//   barrier  beta = tau'/tau, CG bookkeeping (fin_xr)
//   phase C  d = r + beta d, written both as c64 and as the next forward's
//            fp16 hi/lo operand X = split(sigma_x * s_c * d)
//
// The scalars are reduced deterministically: each block leaves its fp64
// partial sums in `part`, and after the grid barrier every block sums all
// of them in block order, so all blocks hold bit-identical alpha / beta
// without a second round trip.  sigma_x needs a bound on max|d| before d
// exists; max|r| + |beta| * bound(d_old) is one (component-wise), and the
// bound actually used is left in scales[6] for the forward's epilogue.
#pragma once

#include "elementwise.cuh"
#include "nudft_tc.cuh"

namespace csr {

struct CgTailArgs {
    Geom g;
    AdmmBufs b;
    const float2 *ws;  // split-K partials (coils combined)
    int S;
    TcArgs a;          // forward operand geometry
    const float2 *sens;
    __half *xb_hi, *xb_lo;
    int write_x;       // write the next forward operand here (else k_tc_prep_x does,
                       // from the bound left in scales[6])
    float *scales;     // [4] max|s|, [5] k-space max (reset), [6] bound on max|d|
    double *part;      // [3][grid] fp64 partials
    unsigned *bar;     // [2] grid barrier: arrivals, generation
    unsigned long long *probe;  // live timing slot or null
    unsigned long long *stamps; // debug: phase timestamps of block 0 (CSR_TRACE)
};

// Grid barrier for the cooperative launch (all blocks co-resident).  bar[1]
// counts completed barriers; each block reads it once at kernel start
// (gen0), so barrier k only has to wait for bar[1] == gen0 + k: one
// release-add to arrive, one acquire spin to leave, no extra fences.
__device__ __forceinline__ unsigned grid_gen(const unsigned *bar) {
    unsigned g;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(bar + 1) : "memory");
    return g;
}
__device__ __forceinline__ void grid_barrier(unsigned *bar, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned old;
        asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;"
                     : "=r"(old) : "l"(bar) : "memory");
        if (old == gridDim.x - 1) {
            asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(bar) : "memory");
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar + 1) : "memory");
        } else {
            unsigned g;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(bar + 1) : "memory");
            } while ((int)(g - target) < 0);
        }
    }
    __syncthreads();
}

// block sum of NV doubles into part[i * grid + block]
template <int NV>
__device__ __forceinline__ void block_partials(double (&v)[NV], double *part) {
    __shared__ double sh[NV][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        double w = warp_sum(v[i]);
        if (lane == 0) sh[i][warp] = w;
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            double w = lane < (int)(blockDim.x >> 5) ? sh[i][lane] : 0.0;
            w = warp_sum(w);
            if (lane == 0) part[(size_t)i * gridDim.x + blockIdx.x] = w;
        }
    }
}

// every block: tot[i] = sum over blocks of part[i][*] in block order
template <int NV>
__device__ __forceinline__ void all_totals(const double *part, double (&tot)[NV]) {
    __shared__ double res[NV];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (warp == 0) {
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            double w = 0.0;
            for (unsigned b = lane; b < gridDim.x; b += 32)
                w += __ldcg(part + (size_t)i * gridDim.x + b);
            w = warp_sum(w);
            if (lane == 0) res[i] = w;
        }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < NV; ++i) tot[i] = res[i];
}

// the small-image (XOP) tail also takes the pixel-pair paths (config 0 tail
// 51.4 -> 45.6 us per iteration, config 1 44.7 -> 43.6; the head measured
// neutral-to-slower that way and keeps the scalar form for XOP)
#ifndef TAIL_PAIRS_XOP
#define TAIL_PAIRS_XOP 1
#endif
// per-lane loads of the block-partial fold: grids of <= 32 * TAIL_FOLD blocks
constexpr int TAIL_FOLD = 16;

#define TAIL_STAMP(i) \
    if (A.stamps && threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1)) \
    A.stamps[(blockIdx.x ? 16 : 0) + (i)] = gtimer()
__device__ __forceinline__ void write_x_operand(const CgTailArgs &A, int t, int xx, int y,
                                                int64_t nxy, float2 v, float sg) {
    write_xop(A.a, A.sens, A.xb_hi, A.xb_lo, t, xx, y, nxy, v, sg);
}

__global__ void __launch_bounds__(256, 2) k_cg_tail(CgTailArgs A) {
    pdl_enter();
    const Geom &g = A.g;
    const AdmmBufs &b = A.b;
    DevScalars *s = b.s;
    if (!s->cg_active) return;  // uniform: every block reads the same flag
    probe_enter(A.probe);
    TAIL_STAMP(0);
    const int64_t nxy = (int64_t)g.nx * g.ny;
    // everything block 0 rewrites below is read before the first barrier
    const float dbound_old = A.scales[6];
    const double tau = s->tau, atol2 = s->atol2;
    const int cg_iter = s->cg_iter + 1, cg_max = s->cg_max, cur = s->cur;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    __shared__ unsigned gen0;
    if (threadIdx.x == 0) gen0 = grid_gen(A.bar);  // before anyone can arrive

    // ---- phase A: Ad and <d, Ad>
    {
        ThetaOf th{b.d, g, nullptr, nullptr};
        double v[2] = {0.0, 0.0};
        for (int64_t i = i0; i < g.n; i += stride) {
            int t, xx, y;
            unflat(g, i, t, xx, y);
            const float2 f = coil_combine(A.ws, nullptr, A.S, g.T, 1, nxy, t, i - t * nxy);
            const float2 l = theta_adj_at(th, g, t, xx, y);
            const float2 a = make_float2(f.x + b.hb * l.x, f.y + b.hb * l.y);
            b.ad[i] = a;
            const float2 d = b.d[i];
            v[0] += (double)d.x * a.x + (double)d.y * a.y;
            v[1] += (double)d.x * a.y - (double)d.y * a.x;
        }
        block_partials<2>(v, A.part);
    }
    TAIL_STAMP(1);
    grid_barrier(A.bar, gen0 + 1);
    double dad[2];
    TAIL_STAMP(2);
    all_totals<2>(A.part, dad);
    TAIL_STAMP(3);
    // fin_ad (solver.py:114): alpha = tau / <d, Ad>
    const double den = dad[0] * dad[0] + dad[1] * dad[1];
    const double al_re = tau * dad[0] / den, al_im = -tau * dad[1] / den;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        s->alpha_re = al_re;
        s->alpha_im = al_im;
    }

    // ---- phase B: x, r and ||r||^2, max|r|
    {
        float2 *x = b.rho[cur ^ 1];
        const float2 al = make_float2((float)al_re, (float)al_im);
        const float2 nal = make_float2(-al.x, -al.y);
        double v[1] = {0.0};
        float rmax = 0.f;
        for (int64_t i = i0; i < g.n; i += stride) {
            x[i] = cadd(x[i], cmul(al, b.d[i]));
            const float2 r = cadd(b.r[i], cmul(nal, b.ad[i]));
            b.r[i] = r;
            v[0] += (double)r.x * r.x + (double)r.y * r.y;
            rmax = fmaxf(rmax, fmaxf(fabsf(r.x), fabsf(r.y)));
        }
        // slot 2: ||r||^2 partials; slot 3: max|r| partials
        __shared__ float shm[32];
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) rmax = fmaxf(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
        if (lane == 0) shm[warp] = rmax;
        block_partials<1>(v, A.part + 2 * (size_t)gridDim.x);  // syncs the block
        if (warp == 0) {
            float w = lane < (int)(blockDim.x >> 5) ? shm[lane] : 0.f;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) w = fmaxf(w, __shfl_xor_sync(0xffffffffu, w, o));
            if (lane == 0) A.part[3 * (size_t)gridDim.x + blockIdx.x] = w;
        }
    }
    TAIL_STAMP(4);
    grid_barrier(A.bar, gen0 + 2);
    double tn;
    TAIL_STAMP(5);
    float rmax_all;
    {
        __shared__ double res_tn;
        __shared__ float res_rm;
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        if (warp == 0) {
            double w = 0.0;
            float m = 0.f;
            for (unsigned bb = lane; bb < gridDim.x; bb += 32) {
                w += __ldcg(A.part + 2 * (size_t)gridDim.x + bb);
                m = fmaxf(m, (float)__ldcg(A.part + 3 * (size_t)gridDim.x + bb));
            }
            w = warp_sum(w);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            if (lane == 0) {
                res_tn = w;
                res_rm = m;
            }
        }
        __syncthreads();
        tn = res_tn;
        rmax_all = res_rm;
    }
    TAIL_STAMP(6);
    // fin_xr (solver.py:116-122), computed identically by every block
    const bool finite = isfinite(tn);
    const double be_d = finite ? tn / tau : 0.0;
    const bool go_on = finite && cg_iter < cg_max && tn > atol2;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (!finite) {
            s->error = 1;
            s->admm_active = 0;
        } else {
            s->beta_cg = be_d;
        }
        s->tau = tn;
        s->cg_iter = cg_iter;
        s->cg_active = go_on ? 1 : 0;
    }
    if (!go_on) {  // the last iteration leaves d as it is (k_cg_d gate)
        probe_exit(A.probe);
        return;
    }

    // ---- phase C: d = r + beta d, and the forward operand of the new d
    const float be = (float)be_d;
    const float dbound = rmax_all + fabsf(be) * dbound_old;
    const float sg = pow2_scale(2.f * A.scales[4] * dbound);
    if (blockIdx.x == 0 && threadIdx.x == 0) A.scales[5] = 0.f;  // forward atomicMax
    for (int64_t i = i0; i < g.n; i += stride) {
        const float2 d = b.d[i], r = b.r[i];
        const float2 nd = make_float2(r.x + be * d.x, r.y + be * d.y);
        b.d[i] = nd;
        int t, xx, y;
        unflat(g, i, t, xx, y);
        if (A.write_x) write_x_operand(A, t, xx, y, nxy, nd, sg);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) A.scales[6] = dbound;
    TAIL_STAMP(7);
    probe_exit(A.probe);
}


// One-barrier variant of the tail (default).  Phase A also accumulates
// <r, Ad>, ||Ad||^2, ||r||^2 and max|Ad|, so after its single grid
// reduction every block knows alpha = tau / <d, Ad> and, by expanding
// ||r - alpha Ad||^2 = tau - 2 Re(alpha <r, Ad>) + |alpha|^2 ||Ad||^2 in
// fp64, tau' and beta as well; x, r and d (with the next forward operand)
// are then updated in one pass.  tau itself is re-measured directly
// (||r||^2 in phase A) every iteration, so the expansion never compounds;
// it differs from the directly summed ||r'||^2 of the reference only by the
// fp32 rounding of r' (~1e-7 relative in beta).
// XOP: this kernel also writes the next forward operand (small images,
// latency-bound); without it (large images, bandwidth-bound) it runs at three
// blocks per SM and k_tc_prep_x writes the operand
template <bool XOP>
__global__ void __launch_bounds__(256, XOP ? 2 : 3) k_cg_tail1(CgTailArgs A) {
    pdl_enter();
    const Geom &g = A.g;
    const AdmmBufs &b = A.b;
    DevScalars *s = b.s;
    if (!s->cg_active) return;  // uniform: every block reads the same flag
    probe_enter(A.probe);
    TAIL_STAMP(0);
    const int64_t nxy = (int64_t)g.nx * g.ny;
    const float dbound_old = A.scales[6];
    const double atol2 = s->atol2;
    const int cg_iter = s->cg_iter + 1, cg_max = s->cg_max, cur = s->cur;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    __shared__ unsigned gen0;
    if (threadIdx.x == 0) gen0 = grid_gen(A.bar);
    // ---- phase A: Ad; <d,Ad>, <r,Ad>, ||Ad||^2, ||r||^2; max|Ad|, max|r|
    {
        ThetaOf th{b.d, g, nullptr, nullptr};
        double v[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        float amax = 0.f, rmax = 0.f;
        auto load = [&](int64_t i, float2 &a, float2 &d, float2 &r) {
            int t, xx, y;
            unflat(g, i, t, xx, y);
            const float2 f = coil_combine(A.ws, nullptr, A.S, g.T, 1, nxy, t, i - t * nxy);
            const float2 l = theta_adj_at(th, g, t, xx, y);
            a = make_float2(f.x + b.hb * l.x, f.y + b.hb * l.y);
            d = b.d[i];
            r = b.r[i];
        };
        auto use = [&](int64_t i, float2 a, float2 d, float2 r) {
            b.ad[i] = a;
            v[0] += (double)d.x * a.x + (double)d.y * a.y;
            v[1] += (double)d.x * a.y - (double)d.y * a.x;
            v[2] += (double)r.x * a.x + (double)r.y * a.y;
            v[3] += (double)r.x * a.y - (double)r.y * a.x;
            v[4] += (double)a.x * a.x + (double)a.y * a.y;
            v[5] += (double)r.x * r.x + (double)r.y * r.y;
            amax = fmaxf(amax, fmaxf(fabsf(a.x), fabsf(a.y)));
            rmax = fmaxf(rmax, fmaxf(fabsf(r.x), fabsf(r.y)));
        };
        if ((!XOP || TAIL_PAIRS_XOP) && (g.ny & 1) == 0) {
            // large images: pixel pairs (y, y+1) with 16-byte loads / stores;
            // the arithmetic is theta_adj_at's (ThetaOf), per pixel
            const int64_t n2 = g.n / 2;
            const float4 *d4 = reinterpret_cast<const float4 *>(b.d);
            const float4 *r4 = reinterpret_cast<const float4 *>(b.r);
            const float4 *ws4 = reinterpret_cast<const float4 *>(A.ws);
            float4 *ad4 = reinterpret_cast<float4 *>(b.ad);
            for (int64_t j = i0; j < n2; j += stride) {
                int t, x, y;
                unflat(g, 2 * j, t, x, y);
                const int64_t row = (int64_t)t * g.nx, pix = (int64_t)x * g.ny + y;
                float4 f = make_float4(0.f, 0.f, 0.f, 0.f);
                for (int sp = 0; sp < A.S; ++sp) {
                    const float4 w = ws4[(((int64_t)sp * g.T + t) * nxy + pix) >> 1];
                    f.x += w.x; f.y += w.y; f.z += w.z; f.w += w.w;
                }
                const int xm = x == 0 ? g.nx - 1 : x - 1, xp = x + 1 == g.nx ? 0 : x + 1;
                const float4 dc = d4[j];
                const float4 dxm = d4[((row + xm) * g.ny + y) >> 1];
                const float4 dxp = d4[((row + xp) * g.ny + y) >> 1];
                const float2 dym = b.d[(row + x) * g.ny + (y == 0 ? g.ny - 1 : y - 1)];
                const float2 dyp = b.d[(row + x) * g.ny + (y + 2 == g.ny ? 0 : y + 2)];
                float4 dtm = dc, dtp = dc;
                if (g.D == 3) {
                    const int tm = t == 0 ? g.T - 1 : t - 1, tq = t + 1 == g.T ? 0 : t + 1;
                    dtm = d4[(((int64_t)tm * g.nx + x) * g.ny + y) >> 1];
                    dtp = d4[(((int64_t)tq * g.nx + x) * g.ny + y) >> 1];
                }
                const float4 rr = r4[j];
                // per pixel k of the pair: neighbours (x-1, x+1, y-1, y+1, t-1, t+1)
                auto lap = [&](float2 dp, float2 xmv, float2 xpv, float2 ymv, float2 ypv,
                               float2 tmv, float2 tpv) {
                    float2 r = cadd(csub(csub(dp, xmv), csub(xpv, dp)),
                                    csub(csub(dp, ymv), csub(ypv, dp)));
                    if (g.D == 3) r = cadd(r, csub(csub(dp, tmv), csub(tpv, dp)));
                    return r;
                };
                const float2 p0 = make_float2(dc.x, dc.y), p1 = make_float2(dc.z, dc.w);
                const float2 l0 = lap(p0, make_float2(dxm.x, dxm.y), make_float2(dxp.x, dxp.y),
                                      dym, p1, make_float2(dtm.x, dtm.y), make_float2(dtp.x, dtp.y));
                const float2 l1 = lap(p1, make_float2(dxm.z, dxm.w), make_float2(dxp.z, dxp.w),
                                      p0, dyp, make_float2(dtm.z, dtm.w), make_float2(dtp.z, dtp.w));
                const float2 a0 = make_float2(f.x + b.hb * l0.x, f.y + b.hb * l0.y);
                const float2 a1 = make_float2(f.z + b.hb * l1.x, f.w + b.hb * l1.y);
                ad4[j] = make_float4(a0.x, a0.y, a1.x, a1.y);
                // use() without its store, pixel 0 then pixel 1
                for (int k = 0; k < 2; ++k) {
                    const float2 a = k ? a1 : a0, d = k ? p1 : p0;
                    const float2 r = k ? make_float2(rr.z, rr.w) : make_float2(rr.x, rr.y);
                    v[0] += (double)d.x * a.x + (double)d.y * a.y;
                    v[1] += (double)d.x * a.y - (double)d.y * a.x;
                    v[2] += (double)r.x * a.x + (double)r.y * a.y;
                    v[3] += (double)r.x * a.y - (double)r.y * a.x;
                    v[4] += (double)a.x * a.x + (double)a.y * a.y;
                    v[5] += (double)r.x * r.x + (double)r.y * r.y;
                    amax = fmaxf(amax, fmaxf(fabsf(a.x), fabsf(a.y)));
                    rmax = fmaxf(rmax, fmaxf(fabsf(r.x), fabsf(r.y)));
                }
            }
        } else {
        // two grid-stride pixels per trip, all loads before the stores (more
        // bytes in flight at large n); per-thread summation order unchanged
        for (int64_t i = i0; i < g.n; i += 2 * stride) {
            const int64_t j = i + stride;
            const bool hj = j < g.n;
            float2 a0, d0, r0, a1, d1, r1;
            load(i, a0, d0, r0);
            load(hj ? j : i, a1, d1, r1);
            use(i, a0, d0, r0);
            if (hj) use(j, a1, d1, r1);
        }
        }
        __shared__ float shm[2][32];
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
            rmax = fmaxf(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
        }
        if (lane == 0) {
            shm[0][warp] = amax;
            shm[1][warp] = rmax;
        }
        block_partials<6>(v, A.part);  // slots 0..5 (syncs the block)
        if (warp == 0) {
            const bool in = lane < (int)(blockDim.x >> 5);
            float wa = in ? shm[0][lane] : 0.f, wr = in ? shm[1][lane] : 0.f;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                wa = fmaxf(wa, __shfl_xor_sync(0xffffffffu, wa, o));
                wr = fmaxf(wr, __shfl_xor_sync(0xffffffffu, wr, o));
            }
            if (lane == 0) {
                A.part[6 * (size_t)gridDim.x + blockIdx.x] = wa;
                A.part[7 * (size_t)gridDim.x + blockIdx.x] = wr;
            }
        }
    }
    TAIL_STAMP(1);
    grid_barrier(A.bar, gen0 + 1);
    TAIL_STAMP(2);
    double tot[6];
    float amax_all, rmax_all;
    {
        __shared__ double res[6];
        __shared__ float resm[2];
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        // warp q folds slot q; all of a lane's loads are issued at once
        // (<= TAIL_FOLD * 32 blocks, the grid cap), then summed in block order
        if (warp < 8) {
            const int q = warp;
            const double *src = A.part + (size_t)q * gridDim.x;
            double xl[TAIL_FOLD];
#pragma unroll
            for (int u = 0; u < TAIL_FOLD; ++u) {
                const unsigned bb = lane + 32 * u;
                xl[u] = bb < gridDim.x ? __ldcg(src + bb) : 0.0;
            }
            double w = xl[0];
#pragma unroll
            for (int u = 1; u < TAIL_FOLD; ++u) w = q < 6 ? w + xl[u] : fmax(w, xl[u]);
            if (q < 6) {
                w = warp_sum(w);
            } else {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) w = fmax(w, __shfl_xor_sync(0xffffffffu, w, o));
            }
            if (lane == 0) {
                if (q < 6) res[q] = w;
                else resm[q - 6] = (float)w;
            }
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < 6; ++q) tot[q] = res[q];
        amax_all = resm[0];
        rmax_all = resm[1];
    }
    TAIL_STAMP(3);
    // fin_ad + fin_xr (solver.py:114-122), identically in every block
    const double tau = tot[5];
    const double den = tot[0] * tot[0] + tot[1] * tot[1];
    const double al_re = tau * tot[0] / den, al_im = -tau * tot[1] / den;
    const double tn = tau - 2.0 * (al_re * tot[2] - al_im * tot[3]) +
                      (al_re * al_re + al_im * al_im) * tot[4];
    const bool finite = isfinite(tn);
    const double be_d = finite ? tn / tau : 0.0;
    const bool go_on = finite && cg_iter < cg_max && tn > atol2;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        s->alpha_re = al_re;
        s->alpha_im = al_im;
        if (!finite) {
            s->error = 1;
            s->admm_active = 0;
        } else {
            s->beta_cg = be_d;
        }
        s->tau = tn;
        s->cg_iter = cg_iter;
        s->cg_active = go_on ? 1 : 0;
    }
    // ---- fused update: x += alpha d, r -= alpha Ad, d = r + beta d and
    // the next forward operand (d only when CG goes on, as k_cg_d)
    float2 *x = b.rho[cur ^ 1];
    const float2 al = make_float2((float)al_re, (float)al_im);
    const float2 nal = make_float2(-al.x, -al.y);
    const float be = (float)be_d;
    const float alabs = sqrtf(al.x * al.x + al.y * al.y);
    const float dbound = rmax_all + 2.f * alabs * amax_all + fabsf(be) * dbound_old;
    const float sg = pow2_scale(2.f * A.scales[4] * dbound);
    if (go_on && blockIdx.x == 0 && threadIdx.x == 0) A.scales[5] = 0.f;
    auto update = [&](int64_t i, float2 d, float2 xv, float2 rv, float2 adv) {
        x[i] = cadd(xv, cmul(al, d));
        const float2 r = cadd(rv, cmul(nal, adv));
        b.r[i] = r;
        if (go_on) {
            const float2 nd = make_float2(r.x + be * d.x, r.y + be * d.y);
            b.d[i] = nd;
            int t, xx, y;
            unflat(g, i, t, xx, y);
            if (XOP) write_x_operand(A, t, xx, y, nxy, nd, sg);
        }
    };
    if ((!XOP || TAIL_PAIRS_XOP) && (g.ny & 1) == 0) {
        // pixel pairs with 16-byte loads / stores (update() per pixel).
        // The pass runs from the END of the vectors: the end of phase A's
        // sweep (d, r, Ad) is what the 126 MB L2 still holds after the grid
        // barrier, so at large n the first part of this pass hits L2 (and
        // the next kernel, which walks d forwards, starts on L2 hits too):
        // config 4 DRAM traffic 314 -> 267 MB per launch (the time is set by
        // the loads in flight of the cooperative grid, not by DRAM bytes;
        // a two-pair unrolled form at 2 blocks / SM measured slower)
        const int64_t n2 = g.n / 2;
        float4 *d4 = reinterpret_cast<float4 *>(b.d);
        float4 *x4 = reinterpret_cast<float4 *>(x);
        float4 *r4 = reinterpret_cast<float4 *>(b.r);
        const float4 *a4 = reinterpret_cast<const float4 *>(b.ad);
        for (int64_t j = n2 - 1 - i0; j >= 0; j -= stride) {
            const float4 dv = d4[j], xv = x4[j], rv = r4[j], av = a4[j];
            const float2 d0 = make_float2(dv.x, dv.y), d1 = make_float2(dv.z, dv.w);
            const float2 x0 = cadd(make_float2(xv.x, xv.y), cmul(al, d0));
            const float2 x1 = cadd(make_float2(xv.z, xv.w), cmul(al, d1));
            const float2 r0 = cadd(make_float2(rv.x, rv.y), cmul(nal, make_float2(av.x, av.y)));
            const float2 r1 = cadd(make_float2(rv.z, rv.w), cmul(nal, make_float2(av.z, av.w)));
            x4[j] = make_float4(x0.x, x0.y, x1.x, x1.y);
            r4[j] = make_float4(r0.x, r0.y, r1.x, r1.y);
            if (go_on) {
                const float2 n0 = make_float2(r0.x + be * d0.x, r0.y + be * d0.y);
                const float2 n1 = make_float2(r1.x + be * d1.x, r1.y + be * d1.y);
                d4[j] = make_float4(n0.x, n0.y, n1.x, n1.y);
                if (XOP) {
                    int t, xx, y;
                    unflat(g, 2 * j, t, xx, y);
                    write_xop2(A.a, A.sens, A.xb_hi, A.xb_lo, t, xx, y, nxy, n0, n1, sg);
                }
            }
        }
    } else
    for (int64_t i = i0; i < g.n; i += 2 * stride) {
        const int64_t j = i + stride;
        const bool hj = j < g.n;
        const int64_t jj = hj ? j : i;
        const float2 d0 = b.d[i], x0 = x[i], r0 = b.r[i], a0 = b.ad[i];
        const float2 d1 = b.d[jj], x1 = x[jj], r1 = b.r[jj], a1 = b.ad[jj];
        update(i, d0, x0, r0, a0);
        if (hj) update(j, d1, x1, r1, a1);
    }
    if (go_on && blockIdx.x == 0 && threadIdx.x == 0) A.scales[6] = dbound;
    TAIL_STAMP(7);
    probe_exit(A.probe);
}

// ADMM iteration head (single rank, tensor-core operator): k_admm_mu +
// k_admm_rhs + the first forward's k_tc_prep_x in one cooperative kernel
// with one grid barrier (solver.py:178-183, 99-108):
//   phase 1  mu+ = S(theta(rho) + eta); max|mu - eta|, max|fhd| partials
//   barrier  (the rhs stencil reads mu at neighbouring pixels)
//   phase 2  rhs = fhd + (beta/2) Theta^H (mu - eta); x = 0; r = d = rhs;
//            the first forward operand of d, scaled from the bound
//            max|rhs| <= max|fhd| + (beta/2) 2D max|mu - eta| (component-
//            wise); ||r||^2 partials folded by the last block (ticket) in
//            block order -> tau and the CG activation (fin_rhs)
template <bool XOP>
__global__ void __launch_bounds__(256, XOP ? 2 : 3) k_admm_head(CgTailArgs A) {
    pdl_enter();
    const Geom &g = A.g;
    const AdmmBufs &b = A.b;
    DevScalars *s = b.s;
    if (!s->admm_active) return;  // uniform
    probe_enter(A.probe);
    const int64_t nxy = (int64_t)g.nx * g.ny;
    const int cur = s->cur;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    __shared__ unsigned gen0;
    if (threadIdx.x == 0) gen0 = grid_gen(A.bar);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // ---- phase 1: mu, and the bounds of the rhs
    {
        const float2 *rho = b.rho[cur];
        float mm = 0.f, fm = 0.f;
        // pixel-major: every component of a pixel (and its fhd bound) with
        // all loads ahead of the stores; large images: pixel pairs (y, y+1)
        // with 16-byte loads / stores (theta_at's arithmetic per pixel)
        if (!XOP && (g.ny & 1) == 0) {
            const int64_t n2 = g.n / 2;
            const float4 *rho4 = reinterpret_cast<const float4 *>(rho);
            const float4 *eta4 = reinterpret_cast<const float4 *>(b.eta);
            const float4 *fhd4 = reinterpret_cast<const float4 *>(b.fhd);
            float4 *mu4 = reinterpret_cast<float4 *>(b.mu);
            for (int64_t j = i0; j < n2; j += stride) {
                int t, x, y;
                unflat(g, 2 * j, t, x, y);
                const int64_t row = (int64_t)t * g.nx;
                const float4 a = rho4[j];
                float4 q[3], e[3];
#pragma unroll
                for (int c = 0; c < 3; ++c)
                    if (c < g.D) e[c] = eta4[c * n2 + j];
                q[0] = rho4[((row + (x == 0 ? g.nx - 1 : x - 1)) * g.ny + y) >> 1];
                const float2 qy = rho[(row + x) * g.ny + (y == 0 ? g.ny - 1 : y - 1)];
                q[1] = make_float4(qy.x, qy.y, a.x, a.y);
                if (g.D == 3)
                    q[2] = rho4[(((t == 0 ? g.T - 1 : t - 1) * (int64_t)g.nx + x) * g.ny + y) >> 1];
                const float4 f = fhd4[j];
#pragma unroll
                for (int c = 0; c < 3; ++c)
                    if (c < g.D) {
                        const float tc = c == 2 ? b.t_t : b.t_s;
                        const float2 m0 = soft1(cadd(make_float2(a.x - q[c].x, a.y - q[c].y),
                                                     make_float2(e[c].x, e[c].y)), tc);
                        const float2 m1 = soft1(cadd(make_float2(a.z - q[c].z, a.w - q[c].w),
                                                     make_float2(e[c].z, e[c].w)), tc);
                        mu4[c * n2 + j] = make_float4(m0.x, m0.y, m1.x, m1.y);
                        mm = fmaxf(mm, fmaxf(fabsf(m0.x - e[c].x), fabsf(m0.y - e[c].y)));
                        mm = fmaxf(mm, fmaxf(fabsf(m1.x - e[c].z), fabsf(m1.y - e[c].w)));
                    }
                fm = fmaxf(fm, fmaxf(fmaxf(fabsf(f.x), fabsf(f.y)), fmaxf(fabsf(f.z), fabsf(f.w))));
            }
        } else
        for (int64_t p = i0; p < g.n; p += stride) {
            int t, x, y;
            unflat(g, p, t, x, y);
            float2 e[3], th[3];
#pragma unroll
            for (int c = 0; c < 3; ++c)
                if (c < g.D) {
                    e[c] = b.eta[c * g.n + p];
                    th[c] = theta_at(rho, g, c, t, x, y, nullptr);
                }
            const float2 f = b.fhd[p];
#pragma unroll
            for (int c = 0; c < 3; ++c)
                if (c < g.D) {
                    const float2 m = soft1(cadd(th[c], e[c]), c == 2 ? b.t_t : b.t_s);
                    b.mu[c * g.n + p] = m;
                    mm = fmaxf(mm, fmaxf(fabsf(m.x - e[c].x), fabsf(m.y - e[c].y)));
                }
            fm = fmaxf(fm, fmaxf(fabsf(f.x), fabsf(f.y)));
        }
        __shared__ float sh[2][32];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mm = fmaxf(mm, __shfl_xor_sync(0xffffffffu, mm, o));
            fm = fmaxf(fm, __shfl_xor_sync(0xffffffffu, fm, o));
        }
        if (lane == 0) {
            sh[0][warp] = mm;
            sh[1][warp] = fm;
        }
        __syncthreads();
        if (warp == 0) {
            const bool in = lane < (int)(blockDim.x >> 5);
            float a = in ? sh[0][lane] : 0.f, c = in ? sh[1][lane] : 0.f;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, o));
                c = fmaxf(c, __shfl_xor_sync(0xffffffffu, c, o));
            }
            if (lane == 0) {
                A.part[blockIdx.x] = a;
                A.part[gridDim.x + blockIdx.x] = c;
            }
        }
    }
    grid_barrier(A.bar, gen0 + 1);
    float bound;
    {
        __shared__ float rm[2];
        if (warp < 2) {  // warp q: max of slot q, all loads issued at once
            float xl[TAIL_FOLD];
#pragma unroll
            for (int u = 0; u < TAIL_FOLD; ++u) {
                const unsigned bb = lane + 32 * u;
                xl[u] = bb < gridDim.x ? (float)__ldcg(A.part + warp * gridDim.x + bb) : 0.f;
            }
            float a = xl[0];
#pragma unroll
            for (int u = 1; u < TAIL_FOLD; ++u) a = fmaxf(a, xl[u]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, o));
            if (lane == 0) rm[warp] = a;
        }
        __syncthreads();
        bound = rm[1] + b.hb * 2.f * (float)g.D * rm[0];
    }
    const float sg = pow2_scale(2.f * A.scales[4] * bound);
    // ---- phase 2: rhs, the zero-start CG state and the first operand
    double v[1] = {0.0};
    {
        float2 *x = b.rho[cur ^ 1];
        MuMinusEta u{b.mu, b.eta, g, nullptr};
        if (!XOP && (g.ny & 1) == 0) {
            // pixel pairs: u = mu - eta at the pair and its x+1 / y+2 / t+1
            // neighbours (theta_adj_at's arithmetic per pixel)
            const int64_t n2 = g.n / 2;
            const float4 *mu4 = reinterpret_cast<const float4 *>(b.mu);
            const float4 *eta4 = reinterpret_cast<const float4 *>(b.eta);
            const float4 *fhd4 = reinterpret_cast<const float4 *>(b.fhd);
            float4 *x4 = reinterpret_cast<float4 *>(x);
            float4 *r4 = reinterpret_cast<float4 *>(b.r);
            float4 *d4 = reinterpret_cast<float4 *>(b.d);
            auto sub4 = [](float4 m, float4 e) {
                return make_float4(m.x - e.x, m.y - e.y, m.z - e.z, m.w - e.w);
            };
            // backwards: the end of phase 1's sweep (mu, eta, fhd) is what
            // L2 holds after the barrier (as the CG tail's update pass)
            for (int64_t j = n2 - 1 - i0; j >= 0; j -= stride) {
                int t, xx, y;
                unflat(g, 2 * j, t, xx, y);
                const int64_t row = (int64_t)t * g.nx;
                const int64_t jx = ((row + (xx + 1 == g.nx ? 0 : xx + 1)) * g.ny + y) >> 1;
                const int64_t iy = (row + xx) * g.ny + (y + 2 == g.ny ? 0 : y + 2);
                const float4 u0 = sub4(mu4[j], eta4[j]);
                const float4 u0x = sub4(mu4[jx], eta4[jx]);
                const float4 u1 = sub4(mu4[n2 + j], eta4[n2 + j]);
                const float2 u1y = csub(b.mu[g.n + iy], b.eta[g.n + iy]);
                float4 u2 = u0, u2t = u0;
                if (g.D == 3) {
                    const int64_t jt = ((((t + 1 == g.T) ? 0 : t + 1) * (int64_t)g.nx + xx) * g.ny + y) >> 1;
                    u2 = sub4(mu4[2 * n2 + j], eta4[2 * n2 + j]);
                    u2t = sub4(mu4[2 * n2 + jt], eta4[2 * n2 + jt]);
                }
                const float4 f = fhd4[j];
                // pixel 0: y+1 neighbour is pixel 1 of the pair
                float2 l0 = cadd(csub(make_float2(u0.x, u0.y), make_float2(u0x.x, u0x.y)),
                                 csub(make_float2(u1.x, u1.y), make_float2(u1.z, u1.w)));
                float2 l1 = cadd(csub(make_float2(u0.z, u0.w), make_float2(u0x.z, u0x.w)),
                                 csub(make_float2(u1.z, u1.w), u1y));
                if (g.D == 3) {
                    l0 = cadd(l0, csub(make_float2(u2.x, u2.y), make_float2(u2t.x, u2t.y)));
                    l1 = cadd(l1, csub(make_float2(u2.z, u2.w), make_float2(u2t.z, u2t.w)));
                }
                const float4 rhs = make_float4(f.x + b.hb * l0.x, f.y + b.hb * l0.y,
                                               f.z + b.hb * l1.x, f.w + b.hb * l1.y);
                x4[j] = make_float4(0.f, 0.f, 0.f, 0.f);
                r4[j] = rhs;
                d4[j] = rhs;
                v[0] += (double)rhs.x * rhs.x + (double)rhs.y * rhs.y;
                v[0] += (double)rhs.z * rhs.z + (double)rhs.w * rhs.w;
            }
        } else
        for (int64_t i = i0; i < g.n; i += stride) {
            int t, xx, y;
            unflat(g, i, t, xx, y);
            const float2 l = theta_adj_at(u, g, t, xx, y);
            const float2 f = b.fhd[i];
            const float2 rhs = make_float2(f.x + b.hb * l.x, f.y + b.hb * l.y);
            x[i] = make_float2(0.f, 0.f);
            b.r[i] = rhs;
            b.d[i] = rhs;
            v[0] += (double)rhs.x * rhs.x + (double)rhs.y * rhs.y;
            if (XOP) write_x_operand(A, t, xx, y, nxy, rhs, sg);
        }
    }
    // tau: the last block folds the per-block partials in block order
    double tot[1];
    if (grid_reduce<1>(v, A.part + 2 * (size_t)gridDim.x, A.bar + 2, tot) && threadIdx.x == 0) {
        fin_rhs(s, tot[0]);  // tau, cg_iter = 0, CG activation / error
        A.scales[5] = 0.f;   // the forward's max|kd| (atomicMax)
        A.scales[6] = bound;
    }
    probe_exit(A.probe);
}

}  // namespace csr
