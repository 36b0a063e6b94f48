// Bandwidth-bound kernels: encoding factors (K10), finite differences and
// their adjoint (K5/K6), soft threshold (K7), dots (K8), axpy (K9), and the
// fused CG / ADMM update kernels of the native solver loop.
//
// Image layout (T, nx, ny) complex64, pixel p = (t*nx + x)*ny + y; theta
// stacks (D, T, nx, ny) with D = 2 (static, kernels.py:91-101) or 3 (2-D+t:
// third component along t).  All kernels are grid-stride, 256 threads.
#pragma once

#include "common.cuh"

namespace csr {

struct Geom {
    int T, nx, ny;
    int64_t n;   // T*nx*ny
    int D;       // theta components
    int halo;    // 1: frame-sharded, temporal neighbours of frames 0 / T-1
                 // come from halo buffers instead of wrapping locally
};

__host__ __device__ inline Geom make_geom(int T, int nx, int ny) {
    Geom g;
    g.T = T; g.nx = nx; g.ny = ny;
    g.n = (int64_t)T * nx * ny;
    g.D = T > 1 ? 3 : 2;
    g.halo = 0;
    return g;
}

// ---- K10: separable encoding factors, f64 angle, rounded once ----------
// P0[t][k][x] = exp(-2 pi i kx rx), rx = x - nx//2 (operators.py:50-82,
// acquisition.py:39-43).  The angle is (-2*pi) * (kx * rx) in f64, exactly
// numpy's evaluation order; cos/sin in f64; one rounding to f32.
__global__ void k_factors(const double *__restrict__ coords, int64_t rows,
                          int nx, int ny, float2 *__restrict__ P0,
                          float2 *__restrict__ P1) {
    pdl_enter();
    const double m2pi = -2.0 * 3.141592653589793;
    int64_t total = rows * (int64_t)(nx + ny);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t k = i / (nx + ny);
        int j = (int)(i - k * (nx + ny));
        double kr;
        float2 *dst;
        if (j < nx) {
            kr = coords[2 * k] * (double)(j - nx / 2);
            dst = P0 + k * nx + j;
        } else {
            j -= nx;
            kr = coords[2 * k + 1] * (double)(j - ny / 2);
            dst = P1 + k * ny + j;
        }
        double ang = m2pi * kr;
        double s, c;
        sincos(ang, &s, &c);
        *dst = make_float2((float)c, (float)s);
    }
}

// Factors handed over by the caller (csr_plan_create_from_factors): P0 is
// copied as is; P1 arrives in one of the reference's layouts (kernels.py
// :257-262 pass phase1_t = P1^T for the forward and phase1_conj = conj(P1)
// for the adjoint) and is stored as P1 (M, ny).
// layout 0: P1 (M, ny); 1: P1^T (ny, M); 2: conj(P1) (M, ny)
__global__ void k_import_p1(const float2 *__restrict__ src, int layout, int64_t M, int ny,
                            float2 *__restrict__ P1) {
    pdl_enter();
    const int64_t total = M * ny;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = i / ny;
        const int y = (int)(i - k * ny);
        float2 v;
        if (layout == 1) v = src[(int64_t)y * M + k];
        else v = src[i];
        if (layout == 2) v.y = -v.y;
        P1[i] = v;
    }
}

// ---- circular finite differences ----------------------------------------
// hprev (halo mode): the previous rank's last frame, used as frame -1
__device__ __forceinline__ float2 theta_at(const float2 *__restrict__ v,
                                           const Geom &g, int comp, int t,
                                           int x, int y,
                                           const float2 *__restrict__ hprev = nullptr) {
    int64_t p = ((int64_t)t * g.nx + x) * g.ny + y;
    int64_t q;
    if (comp == 0) q = ((int64_t)t * g.nx + (x == 0 ? g.nx - 1 : x - 1)) * g.ny + y;
    else if (comp == 1) q = ((int64_t)t * g.nx + x) * g.ny + (y == 0 ? g.ny - 1 : y - 1);
    else {
        if (t == 0 && g.halo) return csub(v[p], hprev[(int64_t)x * g.ny + y]);
        q = ((int64_t)(t == 0 ? g.T - 1 : t - 1) * g.nx + x) * g.ny + y;
    }
    return csub(v[p], v[q]);
}

// theta^H applied to a stack given as a functor u(comp, t, x, y)
template <class U>
__device__ __forceinline__ float2 theta_adj_at(const U &u, const Geom &g, int t,
                                               int x, int y) {
    int xp = x + 1 == g.nx ? 0 : x + 1;
    int yp = y + 1 == g.ny ? 0 : y + 1;
    float2 r = cadd(csub(u(0, t, x, y), u(0, t, xp, y)),
                    csub(u(1, t, x, y), u(1, t, x, yp)));
    if (g.D == 3) {
        // halo mode asks the functor for frame T (the next rank's frame 0)
        int tp = (t + 1 == g.T && !g.halo) ? 0 : t + 1;
        r = cadd(r, csub(u(2, t, x, y), u(2, tp, x, y)));
    }
    return r;
}

struct StackRef {
    const float2 *s;
    Geom g;
    __device__ float2 operator()(int comp, int t, int x, int y) const {
        return s[comp * g.n + ((int64_t)t * g.nx + x) * g.ny + y];
    }
};

// Theta^H Theta x at one pixel, computed as theta then its adjoint
// (the reference's composition, solver.py:139).
struct ThetaOf {
    const float2 *v;
    Geom g;
    const float2 *hprev = nullptr, *hnext = nullptr;  // halo mode only
    __device__ float2 operator()(int comp, int t, int x, int y) const {
        if (comp == 2 && t == g.T)  // (theta v)_t at frame T: v[T] - v[T-1]
            return csub(hnext[(int64_t)x * g.ny + y],
                        v[((int64_t)(g.T - 1) * g.nx + x) * g.ny + y]);
        return theta_at(v, g, comp, t, x, y, hprev);
    }
};

__device__ __forceinline__ void unflat(const Geom &g, int64_t p, int &t, int &x,
                                       int &y) {
    if (p <= 0x7fffffff) {  // 32-bit division: the 64-bit one is a long call
        const unsigned q = (unsigned)p, r = q / (unsigned)g.ny;
        y = (int)(q - r * (unsigned)g.ny);
        t = (int)(r / (unsigned)g.nx);
        x = (int)(r - (unsigned)t * (unsigned)g.nx);
        return;
    }
    y = (int)(p % g.ny);
    int64_t r = p / g.ny;
    x = (int)(r % g.nx);
    t = (int)(r / g.nx);
}

// component index of an element of a (D, n) stack
__device__ __forceinline__ int comp_of(const Geom &g, int64_t i) {
    return (g.n <= 0x7fffffff && i <= 0x7fffffff) ? (int)((unsigned)i / (unsigned)g.n)
                                                   : (int)(i / g.n);
}

__global__ void k_theta(Geom g, const float2 *__restrict__ img,
                        float2 *__restrict__ out) {
    pdl_enter();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < g.n * g.D;
         i += (int64_t)gridDim.x * blockDim.x) {
        int comp = comp_of(g, i);
        int t, x, y;
        unflat(g, i - comp * g.n, t, x, y);
        out[i] = theta_at(img, g, comp, t, x, y);
    }
}

__global__ void k_theta_adj(Geom g, const float2 *__restrict__ stack,
                            float2 *__restrict__ out) {
    pdl_enter();
    StackRef u{stack, g};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < g.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int t, x, y;
        unflat(g, i, t, x, y);
        out[i] = theta_adj_at(u, g, t, x, y);
    }
}

// kernels.py:201-209: out = z - z*(t/|z|) if |z| > t else 0
__device__ __forceinline__ float2 soft1(float2 z, float t) {
    float mag = hypotf(z.x, z.y);
    if (mag > t) {
        float s = t / mag;
        return make_float2(z.x - z.x * s, z.y - z.y * s);
    }
    return make_float2(0.f, 0.f);
}

__global__ void k_soft(const float2 *__restrict__ z, int64_t n, float t,
                       float2 *__restrict__ out) {
    pdl_enter();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = soft1(z[i], t);
}

// sum conj(a)*b in f64
__global__ void k_hdot(const float2 *__restrict__ a, const float2 *__restrict__ b,
                       int64_t n, double *partials, unsigned *ticket,
                       double *out) {
    pdl_enter();
    double v[2] = {0.0, 0.0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        float2 p = a[i], q = b[i];
        v[0] += (double)p.x * q.x + (double)p.y * q.y;
        v[1] += (double)p.x * q.y - (double)p.y * q.x;
    }
    double tot[2];
    if (grid_reduce<2>(v, partials, ticket, tot) && threadIdx.x == 0) {
        out[0] = tot[0];
        out[1] = tot[1];
    }
}

__global__ void k_abs_sum(const float2 *__restrict__ z, int64_t n,
                          double *partials, unsigned *ticket, double *out) {
    pdl_enter();
    double v[1] = {0.0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        float2 p = z[i];
        v[0] += (double)hypotf(p.x, p.y);
    }
    double tot[1];
    if (grid_reduce<1>(v, partials, ticket, tot) && threadIdx.x == 0) out[0] = tot[0];
}

__global__ void k_axpy(float2 alpha, const float2 *__restrict__ x,
                       const float2 *y, int64_t n, float2 *out) {
    pdl_enter();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = cadd(y[i], cmul(alpha, x[i]));
}

// ---- adjoint split-K + coil combine -------------------------------------
// img[t,x,y] = sum_c conj(s_c[x,y]) * sum_s ws[s][t][c][x][y]
// (kernels.py:158-172: out += conj(sens[c]) * part, coil order).
__device__ __forceinline__ float2 coil_combine(const float2 *__restrict__ ws,
                                               const float2 *__restrict__ sens,
                                               int S, int T, int C, int64_t nxy,
                                               int t, int64_t pix) {
    float2 acc = make_float2(0.f, 0.f);
    if (!sens) {  // tensor-core partials: coils already combined
        // blocks of 8 predicated loads in flight (latency-bound at small n);
        // the summation order stays s = 0, 1, 2, ...
        for (int s0 = 0; s0 < S; s0 += 8) {
            float2 v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j)
                v[j] = s0 + j < S ? ws[((int64_t)(s0 + j) * T + t) * nxy + pix]
                                  : make_float2(0.f, 0.f);
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (s0 + j < S) acc = cadd(acc, v[j]);
        }
        return acc;
    }
    for (int c = 0; c < C; ++c) {
        float2 part = make_float2(0.f, 0.f);
        for (int s = 0; s < S; ++s)
            part = cadd(part, ws[(((int64_t)s * T + t) * C + c) * nxy + pix]);
        acc = cadd(acc, cmulc(sens[(int64_t)c * nxy + pix], part));
    }
    return acc;
}

__global__ void k_adj_reduce(Geom g, int S, int C, const float2 *__restrict__ ws,
                             const float2 *__restrict__ sens,
                             float2 *__restrict__ out, const int *gate) {
    pdl_enter();
    if (gate && !*gate) return;
    int64_t nxy = (int64_t)g.nx * g.ny;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < g.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int t = (int)(i / nxy);
        out[i] = coil_combine(ws, sens, S, g.T, C, nxy, t, i - t * nxy);
    }
}

// out = fhf + (beta/2) Theta^H Theta x
__global__ void k_normal_finish(Geom g, const float2 *__restrict__ fhf,
                                const float2 *__restrict__ x, float hb,
                                float2 *__restrict__ out) {
    pdl_enter();
    ThetaOf th{x, g};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < g.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int t, xx, y;
        unflat(g, i, t, xx, y);
        float2 l = theta_adj_at(th, g, t, xx, y);
        float2 f = fhf[i];
        out[i] = make_float2(f.x + hb * l.x, f.y + hb * l.y);
    }
}

// ---- native ADMM / CG loop ----------------------------------------------
// Device-resident scalars; every kernel of an ADMM iteration is gated on
// admm_active (and CG kernels on cg_active), which makes the iteration a
// branch-free kernel sequence that is captured once as a CUDA graph.
// Multi-rank frame sharding (b.mr): every reduction kernel leaves its local
// sum in b.loc, the sums are allreduced (NCCL) and k_finalize applies the
// same scalar update on every rank.
struct DevScalars {
    double tau;                 // ||r||^2 (solver.py:106,117)
    double alpha_re, alpha_im;  // CG step tau/<d,Ad> (solver.py:114)
    double beta_cg;             // tau_next/tau (solver.py:121)
    double admm_alpha;          // relative_change_sq (solver.py:149-155)
    double atol2, rtol2;
    int32_t cg_active, cg_iter, cg_max;
    int32_t admm_active, admm_iter, admm_max;
    int32_t cur;                // which rho buffer holds the current image
    int32_t error;              // 1 = non-finite CG residual
    float2 *snap;               // optional per-iteration image snapshots
};

struct IterLog {
    int32_t iteration, cg_iterations;
    double alpha, cg_final_residual_sq;
};

struct AdmmBufs {
    float2 *rho[2];   // current image / CG solution (ping-pong)
    float2 *mu, *eta; // (D, T, nx, ny)
    float2 *fhd;      // F^H d
    float2 *r, *d, *ad, *fhf;
    double *partials;
    unsigned *tickets;  // 4 tickets
    DevScalars *s;
    IterLog *log;
    float t_s, t_t, hb;  // lam/beta, lam_t/beta, beta/2
    // frame sharding
    int mr;              // 1: scalars are finalised after an allreduce
    double *loc;         // [8] local sums: 0 rhs, 1-2 <d,Ad>, 3 xr, 4-5 post
    float2 *hprev, *hnext;  // halo frames (1 frame each)
    float2 *sfirst;      // send buffer (1 frame) for (mu - eta)_t of frame 0
    // tensor-core operand scaling: the producers of d (k_admm_rhs, k_cg_d)
    // leave max|d| (component-wise) in tcs[6] for the next forward
    float *tcs;
    double *mpart;
    unsigned *mtick;
    unsigned long long *probe;  // live timing slots (csr_plan_probe) or null
};

enum FinOp { FIN_RHS = 0, FIN_AD = 1, FIN_XR = 2, FIN_POST = 3 };

__device__ void fin_rhs(DevScalars *s, double tau) {
    s->tau = tau;
    s->cg_iter = 0;
    if (!isfinite(tau)) {
        s->error = 1;
        s->cg_active = 0;
        s->admm_active = 0;
    } else {
        s->cg_active = (s->cg_max > 0 && tau > s->atol2) ? 1 : 0;
    }
}

__device__ void fin_ad(DevScalars *s, double re, double im) {
    double den = re * re + im * im;
    s->alpha_re = s->tau * re / den;
    s->alpha_im = -s->tau * im / den;
}

__device__ void fin_xr(DevScalars *s, double tn) {
    if (!isfinite(tn)) {
        s->error = 1;
        s->cg_active = 0;
        s->admm_active = 0;
        s->cg_iter += 1;
        s->tau = tn;
        return;
    }
    s->beta_cg = tn / s->tau;
    s->tau = tn;
    s->cg_iter += 1;
    s->cg_active = (s->cg_iter < s->cg_max && tn > s->atol2) ? 1 : 0;
}

__device__ void fin_post(DevScalars *s, IterLog *log, double num, double den) {
    double alpha;
    if (den > 0) alpha = num / den;
    else alpha = num == 0 ? 0.0 : INFINITY;
    s->admm_alpha = alpha;
    IterLog &L = log[s->admm_iter];
    L.iteration = s->admm_iter + 1;
    L.cg_iterations = s->cg_iter;
    L.alpha = alpha;
    L.cg_final_residual_sq = s->tau;
    s->admm_iter += 1;
    s->cur ^= 1;
    s->admm_active = (s->admm_iter < s->admm_max && alpha > s->rtol2 && !s->error) ? 1 : 0;
}

// scalar update after the allreduce of b.loc (multi-rank)
__global__ void k_finalize(AdmmBufs b, int op) {
    pdl_enter();
    DevScalars *s = b.s;
    if (op == FIN_RHS || op == FIN_POST) {
        if (!s->admm_active) return;
    } else if (!s->cg_active) {
        return;
    }
    if (op == FIN_RHS) fin_rhs(s, b.loc[0]);
    else if (op == FIN_AD) fin_ad(s, b.loc[1], b.loc[2]);
    else if (op == FIN_XR) fin_xr(s, b.loc[3]);
    else fin_post(s, b.log, b.loc[4], b.loc[5]);
}

// copy frames 0 and T-1 of rho[cur] (sel = 0) or of rho[cur ^ 1] (sel = 1)
// into fixed send buffers for the halo exchange (the ping-pong pointer is
// only known on the device)
__global__ void k_stage_frames(AdmmBufs b, Geom g, int sel, float2 *first, float2 *last) {
    pdl_enter();
    if (!b.s->admm_active) return;
    const float2 *v = b.rho[b.s->cur ^ sel];
    const int64_t nf = (int64_t)g.nx * g.ny;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nf;
         i += (int64_t)gridDim.x * blockDim.x) {
        first[i] = v[i];
        last[i] = v[(int64_t)(g.T - 1) * nf + i];
    }
}

// mu+ = S(theta(rho) + eta)  (solver.py:178)
__global__ void k_admm_mu(Geom g, AdmmBufs b) {
    pdl_enter();
    if (!b.s->admm_active) return;
    probe_enter(b.probe ? b.probe + 4 * PROBE_MU : nullptr);
    const float2 *rho = b.rho[b.s->cur];
    const int64_t nf = (int64_t)g.nx * g.ny;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < g.n * g.D;
         i += (int64_t)gridDim.x * blockDim.x) {
        int comp = comp_of(g, i);
        int t, x, y;
        unflat(g, i - comp * g.n, t, x, y);
        float2 v = cadd(theta_at(rho, g, comp, t, x, y, b.hprev), b.eta[i]);
        float2 m = soft1(v, comp == 2 ? b.t_t : b.t_s);
        b.mu[i] = m;
        // the previous rank needs (mu - eta)_t of this rank's frame 0
        if (g.halo && comp == 2 && t == 0) b.sfirst[(int64_t)x * g.ny + y] = csub(m, b.eta[i]);
    }
    (void)nf;
    probe_exit(b.probe ? b.probe + 4 * PROBE_MU : nullptr);
}

struct MuMinusEta {
    const float2 *mu, *eta;
    Geom g;
    const float2 *hnext = nullptr;  // halo mode: next rank's (mu - eta)_t[0]
    __device__ float2 operator()(int comp, int t, int x, int y) const {
        if (comp == 2 && t == g.T) return hnext[(int64_t)x * g.ny + y];
        int64_t i = comp * g.n + ((int64_t)t * g.nx + x) * g.ny + y;
        return csub(mu[i], eta[i]);
    }
};

// rhs = fhd + (beta/2) Theta^H (mu - eta) (solver.py:142-146); zero-start
// CG init x = 0, r = d = rhs, tau = ||r||^2 (solver.py:99-108)
__global__ void k_admm_rhs(Geom g, AdmmBufs b) {
    pdl_enter();
    if (!b.s->admm_active) return;
    probe_enter(b.probe ? b.probe + 4 * PROBE_RHS : nullptr);
    float2 *x = b.rho[b.s->cur ^ 1];
    MuMinusEta u{b.mu, b.eta, g, b.hnext};
    double v[1] = {0.0};
    float dmax = 0.f;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < g.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int t, xx, y;
        unflat(g, i, t, xx, y);
        float2 l = theta_adj_at(u, g, t, xx, y);
        float2 f = b.fhd[i];
        float2 rhs = make_float2(f.x + b.hb * l.x, f.y + b.hb * l.y);
        x[i] = make_float2(0.f, 0.f);
        b.r[i] = rhs;
        b.d[i] = rhs;
        v[0] += (double)rhs.x * rhs.x + (double)rhs.y * rhs.y;
        dmax = fmaxf(dmax, fmaxf(fabsf(rhs.x), fabsf(rhs.y)));
    }
    double tot[1];
    if (grid_reduce<1>(v, b.partials, b.tickets + 0, tot) && threadIdx.x == 0) {
        if (b.mr) b.loc[0] = tot[0];
        else fin_rhs(b.s, tot[0]);
    }
    if (b.tcs) {
        float m;
        if (grid_max(dmax, b.mpart, b.mtick, m)) b.tcs[6] = m;
    }
    probe_exit(b.probe ? b.probe + 4 * PROBE_RHS : nullptr);
}

// ad = F^H F d (+ coil combine of split-K partials when ws != nullptr)
//      + (beta/2) Theta^H Theta d ; <d, ad> -> alpha = tau / <d, ad>
__global__ void k_cg_ad(Geom g, AdmmBufs b, const float2 *__restrict__ ws,
                        const float2 *__restrict__ sens, int S, int C) {
    pdl_enter();
    if (!b.s->cg_active) return;
    ThetaOf th{b.d, g, b.hprev, b.hnext};
    int64_t nxy = (int64_t)g.nx * g.ny;
    double v[2] = {0.0, 0.0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < g.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int t, xx, y;
        unflat(g, i, t, xx, y);
        float2 f = ws ? coil_combine(ws, sens, S, g.T, C, nxy, t, i - t * nxy)
                      : b.fhf[i];
        float2 l = theta_adj_at(th, g, t, xx, y);
        float2 a = make_float2(f.x + b.hb * l.x, f.y + b.hb * l.y);
        b.ad[i] = a;
        float2 d = b.d[i];
        v[0] += (double)d.x * a.x + (double)d.y * a.y;
        v[1] += (double)d.x * a.y - (double)d.y * a.x;
    }
    double tot[2];
    if (grid_reduce<2>(v, b.partials, b.tickets + 1, tot) && threadIdx.x == 0) {
        if (b.mr) {
            b.loc[1] = tot[0];
            b.loc[2] = tot[1];
        } else {
            fin_ad(b.s, tot[0], tot[1]);
        }
    }
}

// multi-GPU coil sharding, first half: fhf = coil-combined partials (then
// the allreduce runs on b.fhf, then k_cg_ad with ws == nullptr)
__global__ void k_cg_fhf(Geom g, AdmmBufs b, const float2 *__restrict__ ws,
                         const float2 *__restrict__ sens, int S, int C) {
    pdl_enter();
    if (!b.s->cg_active) return;
    int64_t nxy = (int64_t)g.nx * g.ny;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < g.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int t = (int)(i / nxy);
        b.fhf[i] = coil_combine(ws, sens, S, g.T, C, nxy, t, i - t * nxy);
    }
}

// x += alpha d ; r -= alpha ad ; tau' = ||r||^2 (solver.py:115-122)
__global__ void k_cg_xr(Geom g, AdmmBufs b) {
    pdl_enter();
    DevScalars *s = b.s;
    if (!s->cg_active) return;
    float2 *x = b.rho[s->cur ^ 1];
    float2 al = make_float2((float)s->alpha_re, (float)s->alpha_im);
    float2 nal = make_float2(-al.x, -al.y);
    double v[1] = {0.0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < g.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        x[i] = cadd(x[i], cmul(al, b.d[i]));
        float2 r = cadd(b.r[i], cmul(nal, b.ad[i]));
        b.r[i] = r;
        v[0] += (double)r.x * r.x + (double)r.y * r.y;
    }
    double tot[1];
    if (grid_reduce<1>(v, b.partials, b.tickets + 2, tot) && threadIdx.x == 0) {
        if (b.mr) b.loc[3] = tot[0];
        else fin_xr(s, tot[0]);
    }
}

// d = r + (tau'/tau) d ; max|d| for the next forward's operand scale
__global__ void k_cg_d(Geom g, AdmmBufs b) {
    pdl_enter();
    DevScalars *s = b.s;
    if (!s->cg_active) return;
    float be = (float)s->beta_cg;
    float dmax = 0.f;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < g.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        float2 d = b.d[i], r = b.r[i];
        float2 nd = make_float2(r.x + be * d.x, r.y + be * d.y);
        b.d[i] = nd;
        dmax = fmaxf(dmax, fmaxf(fabsf(nd.x), fabsf(nd.y)));
    }
    if (b.tcs) {
        float m;
        if (grid_max(dmax, b.mpart, b.mtick, m)) b.tcs[6] = m;
    }
}

// eta+ = eta + (theta(rho+) - mu+) (solver.py:186); alpha = ||rho+ -
// rho||^2 / ||rho||^2 (solver.py:149-155,192); loop guard
// should_continue (solver.py:158-160); iteration record (solver.py:318-323)
// launched with POST_BLOCKS_PER_SM blocks per SM: one wave of the grid-stride loop
constexpr int POST_BLOCKS_PER_SM = 3;
__global__ void __launch_bounds__(256, POST_BLOCKS_PER_SM) k_admm_post(Geom g, AdmmBufs b) {
    pdl_enter();
    DevScalars *s = b.s;
    if (!s->admm_active) return;
    probe_enter(b.probe ? b.probe + 4 * PROBE_POST : nullptr);
    const float2 *rho = b.rho[s->cur];
    const float2 *xn = b.rho[s->cur ^ 1];
    double v[2] = {0.0, 0.0};
    // pixel-major, all components of a pixel with every load ahead of the
    // stores (bytes in flight at large n).  Even ny: pixel pairs (y, y+1)
    // with 16-byte loads / stores (the y-1 neighbour of the pair costs one
    // extra 8-byte load); else two grid-stride pixels per trip.
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if ((g.ny & 1) == 0) {
        const float4 *xn4 = reinterpret_cast<const float4 *>(xn);
        const float4 *rho4 = reinterpret_cast<const float4 *>(rho);
        const float4 *mu4 = reinterpret_cast<const float4 *>(b.mu);
        float4 *eta4 = reinterpret_cast<float4 *>(b.eta);
        const float4 *hp4 = reinterpret_cast<const float4 *>(b.hprev);
        const int64_t n2 = g.n / 2, nxy = (int64_t)g.nx * g.ny;
        for (int64_t j = i0; j < n2; j += stride) {
            int t, x, y;
            unflat(g, 2 * j, t, x, y);
            float4 e[3], m[3], q[3];
            const int64_t row = (int64_t)t * g.nx;
#pragma unroll
            for (int c = 0; c < 3; ++c)
                if (c < g.D) {
                    e[c] = eta4[c * n2 + j];
                    m[c] = mu4[c * n2 + j];
                }
            const float4 a = xn4[j], o = rho4[j];
            // theta neighbours (theta_at): x-1 pair, y-1 single, t-1 pair
            q[0] = xn4[((row + (x == 0 ? g.nx - 1 : x - 1)) * g.ny + y) >> 1];
            const float2 qy = xn[(row + x) * g.ny + (y == 0 ? g.ny - 1 : y - 1)];
            if (g.D == 3) {
                if (t == 0 && g.halo) q[2] = hp4[((int64_t)x * g.ny + y) >> 1];
                else q[2] = xn4[(((t == 0 ? g.T - 1 : t - 1) * (int64_t)g.nx + x) * g.ny + y) >> 1];
            }
            q[1] = make_float4(qy.x, qy.y, a.x, a.y);
            (void)nxy;
#pragma unroll
            for (int c = 0; c < 3; ++c)
                if (c < g.D)
                    eta4[c * n2 + j] = make_float4(e[c].x + ((a.x - q[c].x) - m[c].x),
                                                   e[c].y + ((a.y - q[c].y) - m[c].y),
                                                   e[c].z + ((a.z - q[c].z) - m[c].z),
                                                   e[c].w + ((a.w - q[c].w) - m[c].w));
            const float d0x = a.x - o.x, d0y = a.y - o.y, d1x = a.z - o.z, d1y = a.w - o.w;
            v[0] += (double)d0x * d0x + (double)d0y * d0y;
            v[1] += (double)o.x * o.x + (double)o.y * o.y;
            v[0] += (double)d1x * d1x + (double)d1y * d1y;
            v[1] += (double)o.z * o.z + (double)o.w * o.w;
        }
    } else {
    struct Px {
        float2 e[3], th[3], m[3], a, o;
    };
    auto load = [&](int64_t p, Px &q) {
        int t, x, y;
        unflat(g, p, t, x, y);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            if (c < g.D) {
                q.e[c] = b.eta[c * g.n + p];
                q.m[c] = b.mu[c * g.n + p];
                q.th[c] = theta_at(xn, g, c, t, x, y, b.hprev);
            }
        }
        q.a = xn[p];
        q.o = rho[p];
    };
    auto use = [&](int64_t p, const Px &q) {
#pragma unroll
        for (int c = 0; c < 3; ++c)
            if (c < g.D) b.eta[c * g.n + p] = cadd(q.e[c], csub(q.th[c], q.m[c]));
        const float2 df = csub(q.a, q.o);
        v[0] += (double)df.x * df.x + (double)df.y * df.y;
        v[1] += (double)q.o.x * q.o.x + (double)q.o.y * q.o.y;
    };
    for (int64_t p = i0; p < g.n; p += 2 * stride) {
        const int64_t p1 = p + stride;
        const bool h1 = p1 < g.n;
        Px q0, q1;
        load(p, q0);
        load(h1 ? p1 : p, q1);
        use(p, q0);
        if (h1) use(p1, q1);
    }
    }
    double tot[2];
    if (grid_reduce<2>(v, b.partials, b.tickets + 3, tot) && threadIdx.x == 0) {
        if (b.mr) {
            b.loc[4] = tot[0];
            b.loc[5] = tot[1];
        } else {
            fin_post(s, b.log, tot[0], tot[1]);
        }
    }
    probe_exit(b.probe ? b.probe + 4 * PROBE_POST : nullptr);
}

// snapshots[admm_iter] = rho[cur]; idempotent, so it needs no gate
__global__ void k_snapshot(int64_t n, const DevScalars *s, const float2 *r0,
                           const float2 *r1) {
    pdl_enter();
    float2 *dst = s->snap;
    if (!dst) return;
    dst += (int64_t)s->admm_iter * n;
    const float2 *src = s->cur ? r1 : r0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

}  // namespace csr
