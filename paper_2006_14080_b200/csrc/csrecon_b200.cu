// csrecon_b200: C-ABI implementation (plan, operators, native ADMM loop).
// See include/csrecon_b200.h for the contract and the reference interfaces
// each entry point replaces.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/csrecon_b200.h"
#include "common.cuh"
#include "elementwise.cuh"
#include "nudft_simt.cuh"
#include "nudft_tc.cuh"
#include "cg_tail.cuh"
#include "simulate.cuh"

using namespace csr;

namespace {

thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};

int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

#define CU(call)                                                             \
    do {                                                                     \
        cudaError_t e_ = (call);                                             \
        if (e_ != cudaSuccess)                                               \
            return fail(e_ == cudaErrorMemoryAllocation ? CSR_ERR_OOM        \
                                                        : CSR_ERR_CUDA,      \
                        std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#define NC(call)                                                          \
    do {                                                                  \
        ncclResult_t r_ = (call);                                         \
        if (r_ != ncclSuccess)                                            \
            return fail(CSR_ERR_NCCL,                                     \
                        std::string(#call) + ": " + ncclGetErrorString(r_)); \
    } while (0)

#define LAUNCHED()                                              \
    do {                                                        \
        g_launches.fetch_add(1, std::memory_order_relaxed);     \
        cudaError_t e_ = cudaGetLastError();                    \
        if (e_ != cudaSuccess)                                  \
            return fail(CSR_ERR_CUDA, std::string("kernel launch: ") + \
                                          cudaGetErrorString(e_)); \
    } while (0)

constexpr int TPB = 256;

inline int ew_blocks(int64_t n) { return reduce_blocks(n, TPB); }

}  // namespace

struct csr_comm {
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0, device = 0;
};

struct csr_plan {
    int dev = 0;
    int T = 1, nx = 0, ny = 0, C = 0;
    int64_t M = 0;
    Geom g{};
    float2 *P0 = nullptr, *P1 = nullptr, *sens = nullptr;
    float2 *kd = nullptr, *ws = nullptr, *fhf = nullptr;
    int S = 1, kchunk = 0;
    // tensor-core operands (nudft_tc.cuh); tc.enabled == false -> SIMT
    TcPlan tc;
    // ADMM state
    float2 *rho[2] = {nullptr, nullptr}, *mu = nullptr, *eta = nullptr,
           *fhd = nullptr, *r = nullptr, *d = nullptr, *ad = nullptr;
    double *partials = nullptr;
    unsigned *tickets = nullptr;
    DevScalars *sc = nullptr;
    IterLog *log = nullptr;
    int log_cap = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev[4] = {};
    cudaGraphExec_t graph = nullptr;
    std::vector<double> graph_key;
    int kernels_per_iter = 0;
    csr_comm *comm = nullptr;
    int64_t factor_bytes = 0, ws_bytes = 0;
    // frame sharding (CSR_PLAN_FRAME_SHARD): halo frames and scalar slots
    bool frame_mode = false;
    float2 *hprev = nullptr, *hnext = nullptr, *sfirst = nullptr, *slast = nullptr;
    float2 *hprev_own = nullptr, *hnext_own = nullptr;  // the no-comm halo buffers
    float2 *hsend = nullptr, *hgath = nullptr;  // with a comm: [first|last], gathered pairs
    size_t hgath_ranks = 0;
    double *loc = nullptr;
    double *mpart = nullptr;  // grid-max partials of the d producers
    double *tail_part = nullptr;  // fused CG head / tail: [8][<= 1024 blocks] partials
    int tail_blocks = 0;          // its cooperative grid (0: not computed yet)
    // the fused head / tail also write the next forward operand (C fp16 hi/lo
    // row pairs per pixel: 48 of the tail's ~60 image-sized streams) unless
    // the image is large enough for that stream to be bandwidth-bound: then
    // the high-occupancy k_tc_prep_x writes it in its own launch
    bool fuse_xop = true;
    // order-stable sample sharding (CSR_PLAN_ORDERED_SAMPLES): the plan's
    // adjoint partials are whole global sample chunks; with a multi-rank comm
    // they are all-gathered into gws ([nranks][S_max] chunk slots, rank-major
    // = global chunk order, unused slots zero) and folded in that order
    bool ordered = false;
    int64_t chunk = 0, M_global = 0;
    int n_chunks_total = 0, S_local = 1, S_max = 0;
    int64_t ws_off = 0;     // this rank's first slot in ws (elements)
    float2 *gws = nullptr;  // gathered chunk partials (multi-rank)
    size_t gws_slots = 0;
    // benchmark timing (csr_plan_set_timing)
    void *flush_buf = nullptr;
    int64_t flush_bytes = 0;
    float *iter_ms = nullptr;
    std::vector<cudaEvent_t> iter_ev;
    std::vector<void *> allocs;
    std::vector<std::pair<cudaStream_t, cudaEvent_t>> uses;  // caller streams (mark_use)
};

namespace {

template <class T>
int dalloc(csr_plan *p, T **ptr, size_t count, int64_t *acct) {
    size_t bytes = count * sizeof(T);
    if (bytes == 0) bytes = 16;
    void *v = nullptr;
    cudaError_t e = pool_alloc(&v, bytes, p->stream);
    if (e != cudaSuccess)
        return fail(CSR_ERR_OOM, std::string("cudaMalloc(") + std::to_string(bytes) +
                                     "): " + cudaGetErrorString(e));
    p->allocs.push_back(v);
    *ptr = static_cast<T *>(v);
    if (acct) *acct += (int64_t)bytes;
    return CSR_OK;
}

#define TRY(x)                  \
    do {                        \
        int rc_ = (x);          \
        if (rc_ != CSR_OK) return rc_; \
    } while (0)

// CSR_HOST_TIMING=1: host-side phase times of plan build / solve on stderr
struct HostTimer {
    bool on = dbg_env("CSR_HOST_TIMING") != nullptr;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    void mark(const char *what) {
        if (!on) return;
        auto t = std::chrono::steady_clock::now();
        fprintf(stderr, "[csr host] %-28s %8.3f ms\n", what,
                std::chrono::duration<double, std::milli>(t - t0).count());
    }
};

int check_device(int dev) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        return fail(CSR_ERR_CUDA, "no CUDA device available (csrecon_b200 has no CPU fallback)");
    if (dev < 0 || dev >= n) return fail(CSR_ERR_ARG, "device ordinal out of range");
    // cached per device: cudaGetDeviceProperties costs milliseconds
    static int checked[64] = {};
    if (dev < 64 && checked[dev]) return CSR_OK;
    int major = 0;
    CU(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
    if (major != 10) {
        cudaDeviceProp prop;
        CU(cudaGetDeviceProperties(&prop, dev));
        return fail(CSR_ERR_CUDA, std::string("csrecon_b200 is built for sm_100a; device is ") +
                                      prop.name);
    }
    if (dev < 64) checked[dev] = 1;
    return CSR_OK;
}

// F x on the plan: x (T,nx,ny) -> k-space.  out == nullptr keeps the result
// in the plan's internal k-space buffer (what run_adjoint_partials(nullptr)
// consumes); otherwise it is written as (T*M, C).
int run_forward(csr_plan *p, const float2 *x, float2 *out, cudaStream_t st,
                const int *gate, bool in_loop = false, bool x_ready = false) {
    if (p->tc.enabled) {
        if (tc_forward(p->tc, x, out, st, gate, in_loop, x_ready))
            return fail(CSR_ERR_CUDA, "tc forward launch: " + tc_last_error());
        g_launches.fetch_add(tc_forward_launches(p->tc, in_loop, out != nullptr, x_ready),
                             std::memory_order_relaxed);
        return CSR_OK;
    }
    dim3 grid((unsigned)((p->M + ST - 1) / ST), (unsigned)p->C, (unsigned)p->T);
    launch(k_forward_simt, grid, 256, 0, st, p->P0, p->P1, p->sens, x, out ? out : p->kd,
                                         (int)p->M, p->nx, p->ny, p->C, gate);
    LAUNCHED();
    return CSR_OK;
}

int nranks(const csr_plan *p) { return p->comm ? p->comm->nranks : 1; }

// A plan with a communicator attached runs the multi-rank code path for any
// rank count (one rank included: NCCL then reduces / exchanges with itself),
// so the collectives of every shard mode also run on a single GPU.

// order-stable sample sharding with a communicator (all-gather of chunks)
bool ordered_multi(const csr_plan *p) { return p->ordered && p->comm; }

// image partial sums over ranks need an allreduce (coil / plain sample split)
bool coil_collective(const csr_plan *p) {
    return !p->frame_mode && !p->ordered && p->comm;
}

// split-K adjoint partials into p->ws; kd == nullptr reads the internal
// buffer written by run_forward(..., nullptr)
int run_adjoint_partials(csr_plan *p, const float2 *kd, cudaStream_t st,
                         const int *gate) {
    if (p->tc.enabled && ordered_multi(p)) {
        // one k-space scale for all ranks (max over ranks of max|kd|), the
        // chunk partials into this rank's slots, then the all-gather
        if (kd) {
            tc_load_kd(p->tc, kd, st);
            LAUNCHED();
        }
        NC(ncclAllReduce(p->tc.scales + 5, p->tc.scales + 5, 1, ncclFloat, ncclMax,
                         p->comm->comm, st));
        if (tc_adjoint(p->tc, nullptr, p->ws + p->ws_off, st, gate))
            return fail(CSR_ERR_CUDA, "tc adjoint launch: " + tc_last_error());
        g_launches.fetch_add(p->tc.adj_launches, std::memory_order_relaxed);
        const size_t cnt = (size_t)p->S_max * p->g.n * 2;
        NC(ncclAllGather(p->ws + p->ws_off, p->ws, cnt, ncclFloat, p->comm->comm, st));
        return CSR_OK;
    }
    if (p->tc.enabled) {
        if (tc_adjoint(p->tc, kd, p->ws, st, gate)) return fail(CSR_ERR_CUDA, "tc adjoint launch: " + tc_last_error());
        g_launches.fetch_add(p->tc.adj_launches + (kd ? 1 : 0), std::memory_order_relaxed);
        return CSR_OK;
    }
    int tiles = ((p->nx + ST - 1) / ST) * ((p->ny + ST - 1) / ST);
    dim3 grid((unsigned)tiles, (unsigned)p->C, (unsigned)(p->T * p->S));
    launch(k_adjoint_simt, grid, 256, 0, st, p->P0, p->P1, kd ? kd : p->kd, p->ws, (int)p->M,
                                         p->nx, p->ny, p->C, p->T, p->kchunk, gate);
    LAUNCHED();
    return CSR_OK;
}

// sens pointer for the coil combine of the split-K partials (nullptr when
// the tensor-core epilogue already combined the coils)
inline const float2 *combine_sens(const csr_plan *p) { return p->tc.enabled ? nullptr : p->sens; }
inline int combine_coils(const csr_plan *p) { return p->tc.enabled ? 1 : p->C; }

int run_adjoint(csr_plan *p, const float2 *kd, float2 *img, cudaStream_t st) {
    TRY(run_adjoint_partials(p, kd, st, nullptr));
    k_adj_reduce<<<ew_blocks(p->g.n), TPB, 0, st>>>(p->g, p->S, combine_coils(p), p->ws,
                                                    combine_sens(p), img, nullptr);
    LAUNCHED();
    return CSR_OK;
}

int allreduce(csr_plan *p, float2 *buf, int64_t n_complex, cudaStream_t st) {
    if (!p->comm) return CSR_OK;
    NC(ncclAllReduce(buf, buf, (size_t)(2 * n_complex), ncclFloat, ncclSum,
                     p->comm->comm, st));
    return CSR_OK;
}

// frame-sharded plans with a communicator finalise CG/ADMM scalars after an
// allreduce of the per-rank sums
bool multi_rank_scalars(const csr_plan *p) { return p->frame_mode && p->comm; }

// Ring halo exchange of one frame each way: hprev <- previous rank's `last`,
// hnext <- next rank's `first` (ranks in frame order, circular like the
// temporal difference).  Without a communicator: local copies.  With one,
// every rank contributes its [first | last] pair to an NCCL all-gather and
// hprev / hnext point at the neighbours' slots of the gathered pairs
// (csr_plan_set_comm), so the exchange is one collective inside the
// captured graph, at any rank count.  (A ring of ncclSend/ncclRecv is the
// leaner pattern at P > 2, but NCCL send/recv to self inside a captured
// graph never completes — measured with NCCL 2.28.9 on the B200,
// tools/nccl_self_probe.cu — so the one-rank path could not exercise it;
// the boundary frames are 0.5 MB each at config 4, the all-gather of 2 P of
// them per CG iteration is noise next to the GEMMs.)
int halo_exchange(csr_plan *p, const float2 *first, const float2 *last, cudaStream_t st) {
    const size_t nb = (size_t)p->nx * p->ny * sizeof(float2);
    if (!p->comm) {
        CU(cudaMemcpyAsync(p->hprev, last, nb, cudaMemcpyDeviceToDevice, st));
        CU(cudaMemcpyAsync(p->hnext, first, nb, cudaMemcpyDeviceToDevice, st));
        return CSR_OK;
    }
    const size_t nf = (size_t)p->nx * p->ny;
    CU(cudaMemcpyAsync(p->hsend, first, nb, cudaMemcpyDeviceToDevice, st));
    CU(cudaMemcpyAsync(p->hsend + nf, last, nb, cudaMemcpyDeviceToDevice, st));
    NC(ncclAllGather(p->hsend, p->hgath, 4 * nf, ncclFloat, p->comm->comm, st));
    return CSR_OK;
}

// multi-rank scalars: allreduce the local sums, then the scalar update
int scalar_sync(csr_plan *p, const AdmmBufs &b, int op, int off, int cnt, cudaStream_t st,
                int *nk) {
    if (!b.mr) return CSR_OK;
    if (p->comm)
        NC(ncclAllReduce(p->loc + off, p->loc + off, (size_t)cnt, ncclDouble, ncclSum,
                         p->comm->comm, st));
    launch(k_finalize, 1, 1, 0, st, b, op);
    LAUNCHED();
    ++*nk;
    return CSR_OK;
}

AdmmBufs admm_bufs(csr_plan *p, const csr_admm_params *prm) {
    AdmmBufs b;
    b.rho[0] = p->rho[0];
    b.rho[1] = p->rho[1];
    b.mu = p->mu;
    b.eta = p->eta;
    b.fhd = p->fhd;
    b.r = p->r;
    b.d = p->d;
    b.ad = p->ad;
    b.fhf = p->fhf;
    b.partials = p->partials;
    b.tickets = p->tickets;
    b.s = p->sc;
    b.log = p->log;
    // scalars cast to the working precision as the reference does
    // (transform.py:39-41: the threshold is cast to the real dtype)
    b.t_s = (float)(prm->lam / prm->beta);
    double lt = prm->lam_t > 0 ? prm->lam_t : prm->lam;
    b.t_t = (float)(lt / prm->beta);
    b.hb = (float)(prm->beta / 2);
    b.mr = multi_rank_scalars(p) ? 1 : 0;
    b.loc = p->loc;
    b.hprev = p->hprev;
    b.hnext = p->hnext;
    b.sfirst = p->sfirst;
    b.tcs = p->tc.enabled ? p->tc.scales : nullptr;
    b.mpart = p->mpart;
    b.mtick = p->tickets + 4;
    b.probe = p->tc.probe;
    return b;
}

// One ADMM iteration as a fixed kernel sequence (captured as a graph).
// The fused CG head / tail (cg_tail.cuh) run with the tensor-core operator
// unless the plan is frame-sharded (its CG scalars are allreduced between
// the tail's phases); with coil / plain-sample sharding the tail reads the
// allreduced adjoint image (ws = fhf, one partial) instead of the local
// split-K partials.
typedef void (*TailKernel)(CgTailArgs);

TailKernel tail_kernel(const csr_plan *p, bool head) {
    static const bool two_barriers = dbg_env("CSR_TAIL2") != nullptr;
    if (head) return p->fuse_xop ? k_admm_head<true> : k_admm_head<false>;
    if (two_barriers) return k_cg_tail;
    return p->fuse_xop ? k_cg_tail1<true> : k_cg_tail1<false>;
}

int launch_cg_tail(csr_plan *p, const AdmmBufs &b, cudaStream_t st, bool head = false,
                   const float2 *ws = nullptr, int S = 0) {
    if (!p->tail_blocks) {
        // one cooperative grid for the head and the tail: co-resident for
        // the less occupant of the two kernels actually launched
        int sms = 0, per_sm = 1 << 30;
        for (TailKernel k : {tail_kernel(p, true), tail_kernel(p, false)}) {
            int o = 0;
            CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k, TPB, 0));
            per_sm = std::min(per_sm, o);
        }
        CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->dev));
        int64_t want = reduce_blocks(p->g.n * (p->C > 1 ? 2 : 1), TPB);
        if (const char *e = dbg_env("CSR_TAIL_BLOCKS")) want = atoi(e);
        // <= 32 * TAIL_FOLD blocks: the one-barrier tail folds TAIL_FOLD partials per lane
        p->tail_blocks = (int)std::max<int64_t>(1, std::min<int64_t>({want, (int64_t)per_sm * sms, (int64_t)32 * TAIL_FOLD}));
    }
    CgTailArgs A;
    A.g = p->g;
    A.b = b;
    A.ws = ws ? ws : p->ws;
    A.S = ws ? S : p->S;
    A.a = tc_args(p->tc);
    A.sens = p->sens;
    A.xb_hi = p->tc.xb_hi;
    A.xb_lo = p->tc.xb_lo;
    A.write_x = p->fuse_xop ? 1 : 0;
    A.scales = p->tc.scales;
    A.part = p->tail_part;
    A.bar = p->tickets + 8;
    A.probe = p->tc.probe ? p->tc.probe + 4 * (head ? PROBE_MU : PROBE_TAIL) : nullptr;
    A.stamps = p->tc.trace ? p->tc.trace + 100000 : nullptr;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)p->tail_blocks);
    cfg.blockDim = dim3(TPB);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CU(cudaLaunchKernelEx(&cfg, tail_kernel(p, head), A));
    LAUNCHED();
    return CSR_OK;
}

// ADMM head (mu + rhs + first forward operand), same conditions as the tail
int launch_admm_head(csr_plan *p, const AdmmBufs &b, cudaStream_t st) {
    TRY(launch_cg_tail(p, b, st, true));
    return CSR_OK;
}

inline bool use_cg_tail(const csr_plan *p) {
    static const bool off = dbg_env("CSR_NO_CG_TAIL") != nullptr;
    return !off && p->tc.enabled && !p->frame_mode;
}

// ADMM post grid: one thread per pixel pair (even ny) or per element, at
// most POST_BLOCKS_PER_SM blocks per SM (one wave of the grid-stride loop)
inline int post_blocks(const Geom &g) {
    const int64_t work = (g.ny % 2 == 0) ? g.n / 2 : g.n * g.D;
    return std::min(ew_blocks(work), 148 * POST_BLOCKS_PER_SM);
}

int enqueue_admm_iteration(csr_plan *p, const AdmmBufs &b, int cg_max,
                           cudaStream_t st, int *nk, bool snap) {
    const Geom g = p->g;
    const int eb = ew_blocks(g.n), ebD = ew_blocks(g.n * g.D);
    const int ebf = ew_blocks((int64_t)g.nx * g.ny);
    const bool fm = p->frame_mode;
    // profiling only (CSR_DBG_SKIP bits, results meaningless): 2 = CG tail,
    // 4 = forward, 8 = adjoint, 16 mu, 32 rhs, 64 post, 128 snapshot;
    // 256 = run prep_x before the first forward
    static const int skip = dbg_env("CSR_DBG_SKIP") ? atoi(dbg_env("CSR_DBG_SKIP")) : 0;
    int k = 0;
    if (skip) {
        if (!(skip & 16)) launch(k_admm_mu, ebD, TPB, 0, st, g, b);
        if (!(skip & 32)) launch(k_admm_rhs, eb, TPB, 0, st, g, b);
        for (int it = 0; it < cg_max; ++it) {
            const bool prep = it == 0 && (skip & 256);
            if (!(skip & 4)) TRY(run_forward(p, p->d, nullptr, st, nullptr, true, !prep));
            if (!(skip & 8)) TRY(run_adjoint_partials(p, nullptr, st, nullptr));
            if (!(skip & 2)) TRY(launch_cg_tail(p, b, st));
        }
        if (!(skip & 64)) launch(k_admm_post, post_blocks(g), TPB, 0, st, g, b);
        if (!(skip & 128)) launch(k_snapshot, eb, TPB, 0, st, g.n, p->sc, p->rho[0], p->rho[1]);
        *nk = 0;
        return CSR_OK;
    }
    if (fm) {  // rho halos for theta(rho)
        launch(k_stage_frames, ebf, TPB, 0, st, b, g, 0, p->sfirst, p->slast); LAUNCHED(); ++k;
        TRY(halo_exchange(p, p->sfirst, p->slast, st));
    }
    const bool tail = use_cg_tail(p);
    if (tail) {  // one cooperative kernel: mu, rhs, CG init, first operand
        TRY(launch_admm_head(p, b, st));
        ++k;
    } else {
        launch(k_admm_mu, ebD, TPB, 0, st, g, b); LAUNCHED(); ++k;
        if (fm) TRY(halo_exchange(p, p->sfirst, p->sfirst, st));  // next rank's (mu-eta)_t[0]
        launch(k_admm_rhs, eb, TPB, 0, st, g, b); LAUNCHED(); ++k;
        TRY(scalar_sync(p, b, FIN_RHS, 0, 1, st, &k));
    }
    const int *gate = &p->sc->cg_active;
    const bool coil_multi = coil_collective(p);
    const int64_t nf = (int64_t)g.nx * g.ny;
    for (int it = 0; it < cg_max; ++it) {
        if (fm) TRY(halo_exchange(p, p->d, p->d + (int64_t)(g.T - 1) * nf, st));
        const bool x_ready = tail && p->fuse_xop;  // the head / previous tail wrote X
        TRY(run_forward(p, p->d, nullptr, st, gate, true, x_ready));
        k += p->tc.enabled ? tc_forward_launches(p->tc, true, false, x_ready) : 1;
        TRY(run_adjoint_partials(p, nullptr, st, gate));
        k += p->tc.enabled ? p->tc.adj_launches : 1;
        if (tail && coil_multi) {  // allreduce the adjoint image, then the fused tail
            launch(k_cg_fhf, eb, TPB, 0, st, g, b, p->ws, combine_sens(p), p->S, combine_coils(p)); LAUNCHED(); ++k;
            TRY(allreduce(p, p->fhf, g.n, st));
            TRY(launch_cg_tail(p, b, st, false, p->fhf, 1));
            ++k;
            continue;
        }
        if (tail) {
            TRY(launch_cg_tail(p, b, st));
            ++k;
            continue;
        }
        if (coil_multi) {
            launch(k_cg_fhf, eb, TPB, 0, st, g, b, p->ws, combine_sens(p), p->S, combine_coils(p)); LAUNCHED(); ++k;
            TRY(allreduce(p, p->fhf, g.n, st));
            launch(k_cg_ad, eb, TPB, 0, st, g, b, nullptr, p->sens, p->S, p->C); LAUNCHED(); ++k;
        } else {
            launch(k_cg_ad, eb, TPB, 0, st, g, b, p->ws, combine_sens(p), p->S, combine_coils(p)); LAUNCHED(); ++k;
        }
        TRY(scalar_sync(p, b, FIN_AD, 1, 2, st, &k));
        launch(k_cg_xr, eb, TPB, 0, st, g, b); LAUNCHED(); ++k;
        TRY(scalar_sync(p, b, FIN_XR, 3, 1, st, &k));
        launch(k_cg_d, eb, TPB, 0, st, g, b); LAUNCHED(); ++k;
    }
    if (fm) {  // halos of the new image for theta(rho+)
        launch(k_stage_frames, ebf, TPB, 0, st, b, g, 1, p->sfirst, p->slast); LAUNCHED(); ++k;
        TRY(halo_exchange(p, p->sfirst, p->slast, st));
    }
    launch(k_admm_post, post_blocks(g), TPB, 0, st, g, b); LAUNCHED(); ++k;
    TRY(scalar_sync(p, b, FIN_POST, 4, 2, st, &k));
    if (snap) {  // per-iteration images only when the caller asked for them
        launch(k_snapshot, eb, TPB, 0, st, g.n, p->sc, p->rho[0], p->rho[1]); LAUNCHED(); ++k;
    }
    *nk = k;
    return CSR_OK;
}

// scales[5] <- max(bound, scales[5]) (csr_adjoint_chunks_bound)
__global__ void k_set_bound(float *s5, float bound) {
    pdl_enter();
    if (threadIdx.x == 0) *s5 = fmaxf(*s5, bound);
}

__global__ void k_flush(uint4 *buf, int64_t n, unsigned v) {
    pdl_enter();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        buf[i] = make_uint4(v, v, v, v);
}

__global__ void k_copy_cur(int64_t n, const DevScalars *s, const float2 *r0,
                           const float2 *r1, float2 *out) {
    pdl_enter();
    const float2 *src = s->cur ? r1 : r0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = src[i];
}

}  // namespace

// ===========================================================================
extern "C" {

const char *csr_last_error(void) { return g_err.c_str(); }
int64_t csr_kernel_launches(void) { return g_launches.load(); }

}  // extern "C"

namespace {

// Caller-provided device factors instead of coordinates (T == 1):
// csr_plan_create_from_factors.
struct FactorSource {
    const float2 *p0 = nullptr, *p1 = nullptr;
    int p1_layout = 0;
};

int plan_create(const csr_plan_desc *desc, const FactorSource &fs, csr_plan **out) {
    if (!desc || !out) return fail(CSR_ERR_ARG, "null argument");
    *out = nullptr;
    if (desc->nx < 1 || desc->ny < 1 || desc->n_frames < 1 || desc->n_coils < 1 ||
        desc->n_samples < 1)
        return fail(CSR_ERR_SHAPE, "plan dimensions must all be >= 1");
    if ((!desc->coords && !fs.p0) || !desc->sens)
        return fail(CSR_ERR_ARG, "coords (or factors) and sens are required");
    HostTimer ht;
    TRY(check_device(desc->device));
    CU(cudaSetDevice(desc->device));
    ht.mark("check device");
    csr_plan *p = new csr_plan();
    p->dev = desc->device;
    p->T = desc->n_frames;
    p->nx = desc->nx;
    p->ny = desc->ny;
    p->C = desc->n_coils;
    p->M = desc->n_samples;
    p->g = make_geom(p->T, p->nx, p->ny);
    {
        // operand writes of >= CSR_XOP_SPLIT (default 2^22) coil-pixels go to
        // their own kernel (measured crossover: tools/gpu/xop_ab.sh)
        const char *e = dbg_env("CSR_XOP_SPLIT");  // (debug builds)
        const int64_t lim = e ? atoll(e) : ((int64_t)1 << 22);
        p->fuse_xop = p->g.n * p->C < lim;
    }
    if (desc->flags & CSR_PLAN_ORDERED_SAMPLES) {
        if (desc->flags & CSR_PLAN_FRAME_SHARD) {
            delete p;
            return fail(CSR_ERR_ARG, "ordered sample sharding and frame sharding exclude each other");
        }
        if (p->T != 1 || desc->chunk_samples < 128 || desc->chunk_samples % 128 ||
            desc->total_samples < p->M) {
            delete p;
            return fail(CSR_ERR_ARG, "ordered sample sharding needs T == 1, chunk_samples a "
                                     "multiple of 128 and total_samples >= n_samples");
        }
        p->ordered = true;
        p->chunk = desc->chunk_samples;
        p->M_global = desc->total_samples;
        p->n_chunks_total = (int)((p->M_global + p->chunk - 1) / p->chunk);
    }
    if (desc->flags & CSR_PLAN_FRAME_SHARD) {
        p->frame_mode = true;
        p->g.halo = 1;
        p->g.D = 3;  // a frame block of a 2-D+t problem (even a single frame)
    }
    const int64_t rows = (int64_t)p->T * p->M;
    const int64_t nxy = (int64_t)p->nx * p->ny;
    auto cleanup = [&](int rc) {
        csr_plan_destroy(p);
        return rc;
    };
    int rc;
    cudaStream_t st;
    if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess)
        return cleanup(fail(CSR_ERR_CUDA, "stream create failed"));
    p->stream = st;
    ht.mark("stream");
    if ((rc = dalloc(p, &p->P0, (size_t)(rows * p->nx), &p->factor_bytes))) return cleanup(rc);
    if ((rc = dalloc(p, &p->P1, (size_t)(rows * p->ny), &p->factor_bytes))) return cleanup(rc);
    if ((rc = dalloc(p, &p->sens, (size_t)(p->C * nxy), &p->factor_bytes))) return cleanup(rc);
    for (auto &e : p->ev)
        if (cudaEventCreate(&e) != cudaSuccess) return cleanup(fail(CSR_ERR_CUDA, "event create"));
    if (cudaMemcpyAsync(p->sens, desc->sens, p->C * nxy * sizeof(float2),
                        cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return cleanup(fail(CSR_ERR_CUDA, "plan upload failed"));
    if (fs.p0) {
        // the caller's factors (the reference's own arrays): P0 as is, P1
        // from its layout
        if (cudaMemcpyAsync(p->P0, fs.p0, rows * p->nx * sizeof(float2),
                            cudaMemcpyDeviceToDevice, st) != cudaSuccess)
            return cleanup(fail(CSR_ERR_CUDA, "factor upload failed"));
        const int blocks = (int)std::min<int64_t>((rows * p->ny + 255) / 256, 148 * 16);
        launch(k_import_p1, blocks, 256, 0, st, fs.p1, fs.p1_layout, rows, p->ny, p->P1);
        g_launches.fetch_add(1);
        if (cudaGetLastError() != cudaSuccess) return cleanup(fail(CSR_ERR_CUDA, "k_import_p1 launch"));
    } else {
        // coords -> device, factors in f64 -> complex64
        double *dcoords = nullptr;
        if (pool_alloc((void **)&dcoords, rows * 2 * sizeof(double), st) != cudaSuccess)
            return cleanup(fail(CSR_ERR_OOM, "coords alloc"));
        p->allocs.push_back(dcoords);
        if (cudaMemcpyAsync(dcoords, desc->coords, rows * 2 * sizeof(double),
                            cudaMemcpyHostToDevice, st) != cudaSuccess)
            return cleanup(fail(CSR_ERR_CUDA, "plan upload failed"));
        int64_t total = rows * (p->nx + p->ny);
        int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
        launch(k_factors, blocks, 256, 0, st, dcoords, rows, p->nx, p->ny, p->P0, p->P1);
        g_launches.fetch_add(1);
        if (cudaGetLastError() != cudaSuccess) return cleanup(fail(CSR_ERR_CUDA, "k_factors launch"));
    }
    ht.mark("factors enqueued");
    // tensor-core operand build (returns tc.enabled=false for shapes it
    // does not tile; the SIMT kernels then handle the plan)
    if ((rc = tc_plan_build(p->tc, p->T, p->nx, p->ny, p->C, p->M, p->P0, p->P1, p->sens, st,
                            &p->factor_bytes, &p->ws_bytes, p->allocs, p->chunk, p->M_global)))
        return cleanup(fail(rc, "tensor-core plan: " + g_err));
    if (p->ordered && !p->tc.enabled)
        return cleanup(fail(CSR_ERR_ARG, "ordered sample sharding runs on the tensor-core "
                                         "operator (<= 16 coils)"));
    ht.mark("tc plan");
    // workspace
    if ((rc = dalloc(p, &p->kd, (size_t)(rows * p->C), &p->ws_bytes))) return cleanup(rc);
    if (p->tc.enabled) {
        p->S = p->S_local = p->tc.split;
        p->ws = p->tc.ws;
    } else {
        int tiles = ((p->nx + ST - 1) / ST) * ((p->ny + ST - 1) / ST);
        int64_t blocks = (int64_t)tiles * p->C * p->T;
        int64_t S = (4 * 148 + blocks - 1) / blocks;
        int64_t smax = (p->M + 255) / 256;
        if (S > smax) S = smax;
        if (S < 1) S = 1;
        int64_t kc = (p->M + S - 1) / S;
        kc = (kc + SK - 1) / SK * SK;
        S = (p->M + kc - 1) / kc;
        p->S = (int)S;
        p->kchunk = (int)kc;
        if ((rc = dalloc(p, &p->ws, (size_t)(S * p->T * p->C * nxy), &p->ws_bytes)))
            return cleanup(rc);
    }
    const int64_t n = p->g.n, nD = n * p->g.D;
    if ((rc = dalloc(p, &p->fhf, (size_t)n, &p->ws_bytes))) return cleanup(rc);
    for (int i = 0; i < 2; ++i)
        if ((rc = dalloc(p, &p->rho[i], (size_t)n, &p->ws_bytes))) return cleanup(rc);
    if ((rc = dalloc(p, &p->mu, (size_t)nD, &p->ws_bytes))) return cleanup(rc);
    if ((rc = dalloc(p, &p->eta, (size_t)nD, &p->ws_bytes))) return cleanup(rc);
    if ((rc = dalloc(p, &p->fhd, (size_t)n, &p->ws_bytes))) return cleanup(rc);
    if ((rc = dalloc(p, &p->r, (size_t)n, &p->ws_bytes))) return cleanup(rc);
    if ((rc = dalloc(p, &p->d, (size_t)n, &p->ws_bytes))) return cleanup(rc);
    if ((rc = dalloc(p, &p->ad, (size_t)n, &p->ws_bytes))) return cleanup(rc);
    if ((rc = dalloc(p, &p->partials, (size_t)(4 * 148 * 4), &p->ws_bytes))) return cleanup(rc);
    if ((rc = dalloc(p, &p->loc, 8, &p->ws_bytes))) return cleanup(rc);
    if ((rc = dalloc(p, &p->mpart, (size_t)(4 * 148), &p->ws_bytes))) return cleanup(rc);
    if (p->frame_mode) {
        if ((rc = dalloc(p, &p->hprev, (size_t)nxy, &p->ws_bytes))) return cleanup(rc);
        if ((rc = dalloc(p, &p->hnext, (size_t)nxy, &p->ws_bytes))) return cleanup(rc);
        p->hprev_own = p->hprev;
        p->hnext_own = p->hnext;
        if ((rc = dalloc(p, &p->sfirst, (size_t)nxy, &p->ws_bytes))) return cleanup(rc);
        if ((rc = dalloc(p, &p->slast, (size_t)nxy, &p->ws_bytes))) return cleanup(rc);
    }
    if ((rc = dalloc(p, &p->tail_part, (size_t)(8 * 1024), &p->ws_bytes))) return cleanup(rc);
    if ((rc = dalloc(p, &p->tickets, 16, &p->ws_bytes))) return cleanup(rc);
    if ((rc = dalloc(p, &p->sc, 1, &p->ws_bytes))) return cleanup(rc);
    if (cudaMemsetAsync(p->tickets, 0, 16 * sizeof(unsigned), st) != cudaSuccess)
        return cleanup(fail(CSR_ERR_CUDA, "memset"));
    ht.mark("workspace");
    if (cudaStreamSynchronize(st) != cudaSuccess)
        return cleanup(fail(CSR_ERR_CUDA, std::string("plan build: ") +
                                              cudaGetErrorString(cudaGetLastError())));
    ht.mark("plan synced");
    *out = p;
    return CSR_OK;
}

// Record that work on `st` touches the plan's memory (csr_plan_destroy
// waits for the latest such work on every stream used).
int mark_use(csr_plan *p, cudaStream_t st) {
    for (auto &u : p->uses)
        if (u.first == st) {
            CU(cudaEventRecord(u.second, st));
            return CSR_OK;
        }
    cudaEvent_t e;
    CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    p->uses.emplace_back(st, e);
    CU(cudaEventRecord(e, st));
    return CSR_OK;
}

}  // namespace

extern "C" {

int csr_plan_create(const csr_plan_desc *desc, csr_plan **out) {
    return plan_create(desc, FactorSource{}, out);
}

int csr_plan_create_from_factors(const csr_factor_desc *fd, csr_plan **out) {
    if (!fd || !out) return fail(CSR_ERR_ARG, "null argument");
    if (!fd->phase0 || !fd->phase1 || !fd->sens)
        return fail(CSR_ERR_ARG, "phase0, phase1 and sens are required");
    if (fd->phase1_layout < CSR_P1_ROWS || fd->phase1_layout > CSR_P1_CONJ)
        return fail(CSR_ERR_ARG, "unknown phase1 layout");
    csr_plan_desc d{};
    d.nx = fd->nx;
    d.ny = fd->ny;
    d.n_frames = 1;
    d.n_coils = fd->n_coils;
    d.n_samples = fd->n_samples;
    d.sens = fd->sens;
    d.device = fd->device;
    FactorSource fs;
    fs.p0 = (const float2 *)fd->phase0;
    fs.p1 = (const float2 *)fd->phase1;
    fs.p1_layout = fd->phase1_layout;
    return plan_create(&d, fs, out);
}

int csr_plan_destroy(csr_plan *p) {
    if (!p) return CSR_OK;
    cudaSetDevice(p->dev);
    // operator calls run on the caller's streams: their work must be done
    // before the plan's memory goes back to the pool
    for (auto &u : p->uses) {
        if (p->stream) cudaStreamWaitEvent(p->stream, u.second, 0);
        else cudaEventSynchronize(u.second);
    }
    if (p->stream) cudaStreamSynchronize(p->stream);
    if (p->graph) cudaGraphExecDestroy(p->graph);
    for (void *a : p->allocs) cudaFreeAsync(a, p->stream);
    if (p->log) cudaFreeAsync(p->log, p->stream);
    if (p->stream) cudaStreamSynchronize(p->stream);
    for (auto &e : p->ev)
        if (e) cudaEventDestroy(e);
    for (auto &e : p->iter_ev) cudaEventDestroy(e);
    for (auto &u : p->uses) cudaEventDestroy(u.second);
    if (p->stream) cudaStreamDestroy(p->stream);
    delete p;
    return CSR_OK;
}

int csr_plan_get_info(const csr_plan *p, csr_plan_info *info) {
    if (!p || !info) return fail(CSR_ERR_ARG, "null argument");
    info->factor_bytes = p->factor_bytes;
    info->workspace_bytes = p->ws_bytes;
    info->gemm_path = p->tc.enabled ? 1 : 0;
    info->split_k = p->tc.enabled ? p->tc.split : p->S;
    return CSR_OK;
}

int csr_plan_get_factors(const csr_plan *p, int32_t frame, void *p0, void *p1,
                         void *stream) {
    if (!p || frame < 0 || frame >= p->T) return fail(CSR_ERR_ARG, "bad frame");
    CU(cudaSetDevice(p->dev));
    cudaStream_t st = (cudaStream_t)stream;
    CU(cudaMemcpyAsync(p0, p->P0 + (int64_t)frame * p->M * p->nx,
                       p->M * p->nx * sizeof(float2), cudaMemcpyDeviceToDevice, st));
    CU(cudaMemcpyAsync(p1, p->P1 + (int64_t)frame * p->M * p->ny,
                       p->M * p->ny * sizeof(float2), cudaMemcpyDeviceToDevice, st));
    return mark_use(const_cast<csr_plan *>(p), st);
}

int csr_forward(csr_plan *p, const void *image, void *kdata, void *stream) {
    if (!p || !image || !kdata) return fail(CSR_ERR_ARG, "null argument");
    CU(cudaSetDevice(p->dev));
    TRY(run_forward(p, (const float2 *)image, (float2 *)kdata, (cudaStream_t)stream, nullptr));
    return mark_use(p, (cudaStream_t)stream);
}

int csr_adjoint(csr_plan *p, const void *kdata, void *image, void *stream) {
    if (!p || !image || !kdata) return fail(CSR_ERR_ARG, "null argument");
    CU(cudaSetDevice(p->dev));
    TRY(run_adjoint(p, (const float2 *)kdata, (float2 *)image, (cudaStream_t)stream));
    return mark_use(p, (cudaStream_t)stream);
}

int csr_normal(csr_plan *p, const void *x, void *out, double beta, void *stream) {
    if (!p || !x || !out) return fail(CSR_ERR_ARG, "null argument");
    CU(cudaSetDevice(p->dev));
    cudaStream_t st = (cudaStream_t)stream;
    TRY(run_forward(p, (const float2 *)x, nullptr, st, nullptr));
    TRY(run_adjoint(p, nullptr, p->fhf, st));
    k_normal_finish<<<ew_blocks(p->g.n), TPB, 0, st>>>(p->g, p->fhf, (const float2 *)x,
                                                       (float)(beta / 2), (float2 *)out);
    LAUNCHED();
    return mark_use(p, st);
}

int csr_theta(int32_t T, int32_t nx, int32_t ny, const void *img, void *diffs,
              void *stream) {
    if (T < 1 || nx < 1 || ny < 1) return fail(CSR_ERR_SHAPE, "bad geometry");
    Geom g = make_geom(T, nx, ny);
    launch(k_theta, ew_blocks(g.n * g.D), TPB, 0, (cudaStream_t)stream, 
        g, (const float2 *)img, (float2 *)diffs);
    LAUNCHED();
    return CSR_OK;
}

int csr_theta_adjoint(int32_t T, int32_t nx, int32_t ny, const void *diffs,
                      void *img, void *stream) {
    if (T < 1 || nx < 1 || ny < 1) return fail(CSR_ERR_SHAPE, "bad geometry");
    Geom g = make_geom(T, nx, ny);
    launch(k_theta_adj, ew_blocks(g.n), TPB, 0, (cudaStream_t)stream, 
        g, (const float2 *)diffs, (float2 *)img);
    LAUNCHED();
    return CSR_OK;
}

int csr_soft_threshold(const void *z, int64_t n, float t, void *out, void *stream) {
    if (!(t >= 0.f)) return fail(CSR_ERR_ARG, "threshold must be >= 0");
    if (n <= 0) return CSR_OK;
    launch(k_soft, ew_blocks(n), TPB, 0, (cudaStream_t)stream, (const float2 *)z, n, t,
                                                           (float2 *)out);
    LAUNCHED();
    return CSR_OK;
}

}  // extern "C"

namespace {

// Scratch of the standalone reductions (csr_hermitian_dot, csr_abs_sum):
// block partials + a ticket the kernel re-arms itself, one buffer per
// (device, stream) allocated on first use, so hot calls never allocate.
struct ReduceScratch {
    int dev;
    cudaStream_t st;
    double *buf;
};
std::mutex g_scratch_mu;
std::vector<ReduceScratch> g_scratch;
constexpr size_t SCRATCH_DOUBLES = 2 * 4 * 148;  // grid_reduce<2> over <= 4*148 blocks

int reduce_scratch(cudaStream_t st, double **partials, unsigned **ticket) {
    int dev = 0;
    CU(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_scratch_mu);
    for (auto &r : g_scratch)
        if (r.dev == dev && r.st == st) {
            *partials = r.buf;
            *ticket = reinterpret_cast<unsigned *>(r.buf + SCRATCH_DOUBLES);
            return CSR_OK;
        }
    double *buf = nullptr;
    const size_t bytes = SCRATCH_DOUBLES * sizeof(double) + 16;
    CU(cudaMalloc(&buf, bytes));
    CU(cudaMemset(buf, 0, bytes));  // ticket starts at 0 (synchronous)
    g_scratch.push_back({dev, st, buf});
    *partials = buf;
    *ticket = reinterpret_cast<unsigned *>(buf + SCRATCH_DOUBLES);
    return CSR_OK;
}

}  // namespace

extern "C" {

int csr_hermitian_dot(const void *a, const void *b, int64_t n, double *out,
                      void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n <= 0) {
        CU(cudaMemsetAsync(out, 0, 2 * sizeof(double), st));
        return CSR_OK;
    }
    double *partials;
    unsigned *ticket;
    TRY(reduce_scratch(st, &partials, &ticket));
    launch(k_hdot, ew_blocks(n), TPB, 0, st, (const float2 *)a, (const float2 *)b, n,
           partials, ticket, out);
    LAUNCHED();
    return CSR_OK;
}

int csr_abs_sum(const void *z, int64_t n, double *out, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n <= 0) {
        CU(cudaMemsetAsync(out, 0, sizeof(double), st));
        return CSR_OK;
    }
    double *partials;
    unsigned *ticket;
    TRY(reduce_scratch(st, &partials, &ticket));
    launch(k_abs_sum, ew_blocks(n), TPB, 0, st, (const float2 *)z, n, partials, ticket, out);
    LAUNCHED();
    return CSR_OK;
}

int csr_axpy(double are, double aim, const void *x, const void *y, int64_t n,
             void *out, void *stream) {
    if (n <= 0) return CSR_OK;
    launch(k_axpy, ew_blocks(n), TPB, 0, (cudaStream_t)stream, 
        make_float2((float)are, (float)aim), (const float2 *)x, (const float2 *)y, n,
        (float2 *)out);
    LAUNCHED();
    return CSR_OK;
}

int csr_adjoint_reconstruct(csr_plan *p, const void *kdata, void *image, void *stream) {
    if (!p || !kdata || !image) return fail(CSR_ERR_ARG, "null argument");
    CU(cudaSetDevice(p->dev));
    cudaStream_t st = (cudaStream_t)stream;
    TRY(run_adjoint(p, (const float2 *)kdata, (float2 *)image, st));
    if (coil_collective(p)) TRY(allreduce(p, (float2 *)image, p->g.n, st));
    return mark_use(p, st);
}

int csr_admm_run(csr_plan *p, const csr_admm_params *prm, const void *kdata,
                 void *rho_out, csr_iter_log *log, csr_run_stats *stats,
                 void *stream, void *snapshots) {
    if (!p || !prm || !kdata || !rho_out || !log) return fail(CSR_ERR_ARG, "null argument");
    if (!(prm->lam > 0) || !(prm->beta > 0))
        return fail(CSR_ERR_ARG, "lam and beta must be > 0");
    if (!(prm->admm_rtol > 0) || !(prm->cg_atol > 0))
        return fail(CSR_ERR_ARG, "admm_rtol and cg_atol must be > 0");
    if (prm->admm_max_iters < 1 || prm->cg_max_iters < 1)
        return fail(CSR_ERR_ARG, "iteration caps must be >= 1");
    HostTimer ht;
    CU(cudaSetDevice(p->dev));
    cudaStream_t caller = (cudaStream_t)stream;
    cudaStream_t st = p->stream;
    const Geom g = p->g;
    const int64_t n = g.n, nD = g.n * g.D;
    if (p->log_cap < prm->admm_max_iters) {
        if (p->log) cudaFreeAsync(p->log, st);
        p->log = nullptr;
        CU(pool_alloc((void **)&p->log, sizeof(IterLog) * prm->admm_max_iters, st));
        p->log_cap = prm->admm_max_iters;
        if (p->graph) {
            cudaGraphExecDestroy(p->graph);
            p->graph = nullptr;
        }
    }
    CU(cudaEventRecord(p->ev[0], caller));
    CU(cudaStreamWaitEvent(st, p->ev[0], 0));
    int ar_calls = 0;
    // ---- setup: rho0 = fhd = allreduce(F^H d)  (solver.py:306-309)
    CU(cudaEventRecord(p->ev[0], st));
    TRY(run_adjoint(p, (const float2 *)kdata, p->fhd, st));
    CU(cudaMemcpyAsync(p->rho[0], p->fhd, n * sizeof(float2), cudaMemcpyDeviceToDevice, st));
    if (coil_collective(p)) {
        TRY(allreduce(p, p->rho[0], n, st));
        TRY(allreduce(p, p->fhd, n, st));
        ar_calls += 2;
    }
    CU(cudaMemsetAsync(p->mu, 0, nD * sizeof(float2), st));
    CU(cudaMemsetAsync(p->eta, 0, nD * sizeof(float2), st));
    DevScalars h{};
    h.atol2 = prm->cg_atol * prm->cg_atol;
    h.rtol2 = prm->admm_rtol * prm->admm_rtol;
    h.cg_max = prm->cg_max_iters;
    h.admm_max = prm->admm_max_iters;
    h.admm_alpha = 1.0;
    h.admm_active = (1.0 > h.rtol2) ? 1 : 0;  // should_continue(0, 1.0)
    h.snap = (float2 *)snapshots;
    if (snapshots)
        CU(cudaMemcpyAsync(snapshots, p->rho[0], n * sizeof(float2),
                           cudaMemcpyDeviceToDevice, st));
    CU(cudaMemcpyAsync(p->sc, &h, sizeof(h), cudaMemcpyHostToDevice, st));
    CU(cudaEventRecord(p->ev[1], st));
    ht.mark("setup enqueued");
    // ---- ADMM loop as a CUDA graph of one iteration
    AdmmBufs b = admm_bufs(p, prm);
    std::vector<double> key = {prm->lam, prm->lam_t, prm->beta,
                               (double)prm->cg_max_iters,
                               (double)(p->comm ? p->comm->nranks : 1),
                               (double)(b.mr), (double)(snapshots != nullptr)};
    bool use_graph = true;
    if (!p->graph || p->graph_key != key) {
        if (p->graph) {
            cudaGraphExecDestroy(p->graph);
            p->graph = nullptr;
        }
        cudaGraph_t graph = nullptr;
        CU(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        int nk = 0;
        int rc = enqueue_admm_iteration(p, b, prm->cg_max_iters, st, &nk, snapshots != nullptr);
        cudaError_t ec = cudaStreamEndCapture(st, &graph);
        if (rc != CSR_OK) {
            if (graph) cudaGraphDestroy(graph);
            return rc;
        }
        if (ec != cudaSuccess || !graph) {
            use_graph = false;
            cudaGetLastError();
        } else {
            cudaError_t ei = cudaGraphInstantiate(&p->graph, graph, 0);
            cudaGraphDestroy(graph);
            if (ei != cudaSuccess) {
                use_graph = false;
                p->graph = nullptr;
                cudaGetLastError();
            }
        }
        p->kernels_per_iter = nk;
        p->graph_key = key;
    }
    ht.mark("graph ready");
    const bool timed = p->iter_ms != nullptr;
    if (timed && p->tc.probe)
        CU(cudaMemsetAsync(p->tc.probe, 0, PROBE_SLOTS * 4 * sizeof(unsigned long long), st));
    if (timed) {
        while ((int)p->iter_ev.size() < 2 * prm->admm_max_iters) {
            cudaEvent_t e;
            CU(cudaEventCreate(&e));
            p->iter_ev.push_back(e);
        }
    }
    for (int it = 0; it < prm->admm_max_iters; ++it) {
        if (timed && p->flush_buf) {
            int64_t n16 = p->flush_bytes / 16;
            launch(k_flush, 148 * 8, 512, 0, st, (uint4 *)p->flush_buf, n16, (unsigned)it);
            LAUNCHED();
        }
        if (timed) CU(cudaEventRecord(p->iter_ev[2 * it], st));
        if (use_graph) {
            CU(cudaGraphLaunch(p->graph, st));
        } else {
            int nk = 0;
            TRY(enqueue_admm_iteration(p, b, prm->cg_max_iters, st, &nk, snapshots != nullptr));
        }
        if (timed) CU(cudaEventRecord(p->iter_ev[2 * it + 1], st));
    }
    CU(cudaEventRecord(p->ev[2], st));
    launch(k_copy_cur, ew_blocks(n), TPB, 0, st, n, p->sc, p->rho[0], p->rho[1], (float2 *)rho_out);
    LAUNCHED();
    CU(cudaEventRecord(p->ev[3], st));
    CU(cudaStreamWaitEvent(caller, p->ev[3], 0));
    // ---- host-side report
    DevScalars hs{};
    std::vector<IterLog> hl(prm->admm_max_iters);
    CU(cudaMemcpyAsync(&hs, p->sc, sizeof(hs), cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(hl.data(), p->log, sizeof(IterLog) * prm->admm_max_iters,
                       cudaMemcpyDeviceToHost, st));
    ht.mark("loop enqueued");
    CU(cudaStreamSynchronize(st));
    ht.mark("solve synced");
    for (int i = 0; i < hs.admm_iter; ++i) {
        log[i].iteration = hl[i].iteration;
        log[i].cg_iterations = hl[i].cg_iterations;
        log[i].alpha = hl[i].alpha;
        log[i].cg_final_residual_sq = hl[i].cg_final_residual_sq;
    }
    if (stats) {
        float ms_setup = 0.f, ms_solve = 0.f;
        cudaEventElapsedTime(&ms_setup, p->ev[0], p->ev[1]);
        cudaEventElapsedTime(&ms_solve, p->ev[1], p->ev[2]);
        stats->n_iterations = hs.admm_iter;
        int cg_total = 0;
        for (int i = 0; i < hs.admm_iter; ++i) cg_total += hl[i].cg_iterations;
        if (hs.error) cg_total += hs.cg_iter;
        stats->allreduce_calls =
            ar_calls + (coil_collective(p) ? cg_total : 0) +
            (ordered_multi(p) ? 2 + cg_total : 0);  // as ordered_chunk_sum calls
        stats->setup_ms = ms_setup;
        stats->solve_ms = ms_solve;
        if (timed) {
            double tot = 0.0;
            for (int it = 0; it < prm->admm_max_iters; ++it) {
                float ms = 0.f;
                cudaEventElapsedTime(&ms, p->iter_ev[2 * it], p->iter_ev[2 * it + 1]);
                p->iter_ms[it] = ms;
                tot += ms;
            }
            stats->solve_ms = tot;
        }
        stats->graph_used = use_graph ? 1 : 0;
        stats->kernels_per_iter = p->kernels_per_iter;
    }
    if (hs.error)
        return fail(CSR_ERR_NONFINITE, "residual became non-finite at CG step " +
                                           std::to_string(hs.cg_iter) + " of ADMM iteration " +
                                           std::to_string(hs.admm_iter + 1));
    return CSR_OK;
}

// ---- NCCL ---------------------------------------------------------------
// debug: copy the tensor-core trace buffer (CSR_TRACE) to the host
int csr_debug_trace(csr_plan *p, unsigned long long *host, int64_t n) {
    if (!p || !p->tc.trace) return fail(CSR_ERR_ARG, "no trace buffer (set CSR_TRACE)");
    CU(cudaMemcpy(host, p->tc.trace, std::min<int64_t>(n, 4096 * 32) * 8, cudaMemcpyDeviceToHost));
    return CSR_OK;
}

int csr_simulate_kspace(int32_t nx, int32_t ny, int32_t n_frames, int32_t n_coils,
                        int64_t n_samples, const double *coords, const void *sens,
                        const void *image, void *kspace, void *stream) {
    if (!coords || !sens || !image || !kspace) return fail(CSR_ERR_ARG, "null argument");
    if (nx < 1 || ny < 1 || n_frames < 1 || n_coils < 1 || n_samples < 1)
        return fail(CSR_ERR_SHAPE, "dimensions must all be >= 1");
    if (n_coils > 65535 || n_frames > 65535) return fail(CSR_ERR_SHAPE, "too many coils / frames");
    int dev = 0;
    CU(cudaGetDevice(&dev));
    TRY(check_device(dev));
    dim3 grid((unsigned)((n_samples + SIM_T - 1) / SIM_T), (unsigned)n_coils, (unsigned)n_frames);
    CU(launch(k_simulate_f64, grid, dim3(256), 0, (cudaStream_t)stream, coords,
              (const double2 *)sens, (const double2 *)image, (double2 *)kspace, n_samples, nx, ny,
              n_coils));
    LAUNCHED();
    return CSR_OK;
}

int csr_plan_probe(csr_plan *p, int32_t slot, double *ms, int64_t *n) {
    if (!p || !ms || !n) return fail(CSR_ERR_ARG, "null argument");
    if (slot < 0 || slot >= PROBE_SLOTS) return fail(CSR_ERR_ARG, "probe slot out of range");
    unsigned long long h[4] = {};
    if (p->tc.probe) {
        CU(cudaStreamSynchronize(p->stream));
        CU(cudaMemcpy(h, p->tc.probe + 4 * slot, sizeof(h), cudaMemcpyDeviceToHost));
    }
    *n = (int64_t)h[3];
    *ms = h[3] ? 1e-6 * (double)h[2] / (double)h[3] : 0.0;
    return CSR_OK;
}

int csr_plan_kernel_times(csr_plan *p, double *fwd_ms, double *adj_ms, int64_t *n_fwd,
                          int64_t *n_adj) {
    if (!p || !fwd_ms || !adj_ms || !n_fwd || !n_adj) return fail(CSR_ERR_ARG, "null argument");
    unsigned long long h[8] = {};
    if (p->tc.probe) {
        CU(cudaStreamSynchronize(p->stream));
        CU(cudaMemcpy(h, p->tc.probe, sizeof(h), cudaMemcpyDeviceToHost));
    }
    *n_fwd = (int64_t)h[3];
    *n_adj = (int64_t)h[7];
    *fwd_ms = h[3] ? 1e-6 * (double)h[2] / (double)h[3] : 0.0;
    *adj_ms = h[7] ? 1e-6 * (double)h[6] / (double)h[7] : 0.0;
    return CSR_OK;
}

// debug: enable (on = 1, clears) / read (on = 0) the per-launch timeline of
// probed kernels: host gets n records (slot index, start ns, end ns)
int csr_debug_timeline(csr_plan *p, int on, unsigned long long *host, int64_t cap) {
    if (!p) return fail(CSR_ERR_ARG, "null plan");
    CU(cudaSetDevice(p->dev));
    CU(cudaDeviceSynchronize());
    if (on) {
        unsigned z = 0;
        int one = 1;
        CU(cudaMemcpyToSymbol(g_tl_n, &z, sizeof(z)));
        CU(cudaMemcpyToSymbol(g_tl_on, &one, sizeof(one)));
        return CSR_OK;
    }
    int zero = 0;
    unsigned n = 0;
    CU(cudaMemcpyToSymbol(g_tl_on, &zero, sizeof(zero)));
    CU(cudaMemcpyFromSymbol(&n, g_tl_n, sizeof(n)));
    n = std::min<unsigned>(n, 4096);
    std::vector<unsigned long long> buf(3 * (size_t)n);
    if (n) CU(cudaMemcpyFromSymbol(buf.data(), g_tl_ring, buf.size() * 8));
    const uint64_t base = (uint64_t)(size_t)p->tc.probe;
    const int64_t m = std::min<int64_t>(cap, n);
    for (int64_t i = 0; i < m; ++i) {
        host[3 * i] = base ? (buf[3 * i] - base) / 32 : 0;  // slot = offset / (4 u64)
        host[3 * i + 1] = buf[3 * i + 1];
        host[3 * i + 2] = buf[3 * i + 2];
    }
    return (int)m;
}

int csr_plan_set_timing(csr_plan *p, void *flush_buf, int64_t flush_bytes,
                        float *iter_ms) {
    if (!p) return fail(CSR_ERR_ARG, "null plan");
    p->flush_buf = flush_buf;
    p->flush_bytes = flush_buf ? flush_bytes : 0;
    p->iter_ms = iter_ms;
    return CSR_OK;
}

int csr_comm_unique_id(void *id128) {
    if (!id128) return fail(CSR_ERR_ARG, "null argument");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId must be 128 bytes");
    ncclUniqueId id;
    NC(ncclGetUniqueId(&id));
    std::memcpy(id128, &id, sizeof(id));
    return CSR_OK;
}

int csr_comm_create(const void *id128, int32_t nranks, int32_t rank, int32_t device,
                    csr_comm **out) {
    if (!id128 || !out || nranks < 1 || rank < 0 || rank >= nranks)
        return fail(CSR_ERR_ARG, "bad communicator arguments");
    TRY(check_device(device));
    CU(cudaSetDevice(device));
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    csr_comm *c = new csr_comm();
    c->nranks = nranks;
    c->rank = rank;
    c->device = device;
    ncclResult_t r = ncclCommInitRank(&c->comm, nranks, id, rank);
    if (r != ncclSuccess) {
        delete c;
        return fail(CSR_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    }
    *out = c;
    return CSR_OK;
}

int csr_comm_destroy(csr_comm *c) {
    if (!c) return CSR_OK;
    if (c->comm) ncclCommDestroy(c->comm);
    delete c;
    return CSR_OK;
}

int csr_plan_set_comm(csr_plan *p, csr_comm *c) {
    if (!p) return fail(CSR_ERR_ARG, "null plan");
    if (c && c->device != p->dev) return fail(CSR_ERR_ARG, "comm and plan on different devices");
    p->comm = c;
    if (p->graph) {
        cudaGraphExecDestroy(p->graph);
        p->graph = nullptr;
    }
    if (p->frame_mode) {
        // halo pairs all-gathered: this rank's neighbours' slots (circular)
        CU(cudaSetDevice(p->dev));
        if (c) {
            const size_t nf = (size_t)p->nx * p->ny;
            if (!p->hgath || p->hgath_ranks != (size_t)c->nranks) {
                TRY(dalloc(p, &p->hsend, 2 * nf, &p->ws_bytes));
                TRY(dalloc(p, &p->hgath, (size_t)c->nranks * 2 * nf, &p->ws_bytes));
                p->hgath_ranks = (size_t)c->nranks;
            }
            const int P = c->nranks, r = c->rank;
            p->hprev = p->hgath + (size_t)((r + P - 1) % P) * 2 * nf + nf;  // prev's last
            p->hnext = p->hgath + (size_t)((r + 1) % P) * 2 * nf;           // next's first
        } else {
            p->hprev = p->hprev_own;
            p->hnext = p->hnext_own;
        }
    }
    if (p->ordered) {
        CU(cudaSetDevice(p->dev));
        if (c) {
            const int S_max = (p->n_chunks_total + c->nranks - 1) / c->nranks;
            if (p->S_local > S_max)
                return fail(CSR_ERR_ARG, "this rank holds more chunks than an even split allows "
                                         "(use make_shard_plan with the chunk grid)");
            const size_t slots = (size_t)c->nranks * S_max * p->g.n;
            if (!p->gws || p->gws_slots != slots) {  // (a previous buffer stays in allocs)
                TRY(dalloc(p, &p->gws, slots, &p->ws_bytes));
                p->gws_slots = slots;
            }
            CU(cudaMemsetAsync(p->gws, 0, slots * sizeof(float2), p->stream));
            CU(cudaStreamSynchronize(p->stream));
            p->S_max = S_max;
            p->ws = p->gws;
            p->S = c->nranks * S_max;
            p->ws_off = (int64_t)c->rank * S_max * p->g.n;
        } else {
            p->ws = p->tc.ws;
            p->S = p->S_local;
            p->ws_off = 0;
        }
    }
    return CSR_OK;
}

int csr_sample_chunking(int32_t nx, int32_t ny, int32_t C, int64_t M, int64_t *chunk,
                        int32_t *n_chunks) {
    if (nx < 1 || ny < 1 || C < 1 || M < 1) return fail(CSR_ERR_SHAPE, "bad geometry");
    if (!chunk || !n_chunks) return fail(CSR_ERR_ARG, "null argument");
    int nc = 0;
    tc_sample_chunking(nx, ny, C, M, *chunk, nc);
    *n_chunks = nc;
    return CSR_OK;
}

int csr_adjoint_chunks(csr_plan *p, const void *kdata, void *chunks, void *stream) {
    if (!p || !kdata || !chunks) return fail(CSR_ERR_ARG, "null argument");
    if (!p->tc.enabled) return fail(CSR_ERR_ARG, "chunk partials need the tensor-core operator");
    CU(cudaSetDevice(p->dev));
    if (tc_adjoint(p->tc, (const float2 *)kdata, (float2 *)chunks, (cudaStream_t)stream, nullptr))
        return fail(CSR_ERR_CUDA, "tc adjoint launch: " + tc_last_error());
    g_launches.fetch_add(p->tc.adj_launches + 1, std::memory_order_relaxed);
    return mark_use(p, (cudaStream_t)stream);
}

int csr_adjoint_chunks_bound(csr_plan *p, const void *kdata, void *chunks, float bound,
                             void *stream) {
    if (!p || !kdata || !chunks) return fail(CSR_ERR_ARG, "null argument");
    if (!p->tc.enabled) return fail(CSR_ERR_ARG, "chunk partials need the tensor-core operator");
    if (!(bound > 0.f) || !std::isfinite(bound)) return fail(CSR_ERR_ARG, "bound must be > 0");
    CU(cudaSetDevice(p->dev));
    cudaStream_t st = (cudaStream_t)stream;
    tc_load_kd(p->tc, (const float2 *)kdata, st);
    LAUNCHED();
    // the operand scale from the caller's bound (every worker passes the same
    // one), never below this worker's own max|kd| (fp16 range)
    launch(k_set_bound, 1, 32, 0, st, p->tc.scales + 5, bound);
    LAUNCHED();
    if (tc_adjoint(p->tc, nullptr, (float2 *)chunks, st, nullptr))
        return fail(CSR_ERR_CUDA, "tc adjoint launch: " + tc_last_error());
    g_launches.fetch_add(p->tc.adj_launches, std::memory_order_relaxed);
    return mark_use(p, st);
}

// One-shot separable NUDFT with the reference's kernel signatures
// (kernels.py:257-262): a transient plan from the caller's factors, one
// application on the caller's stream, the plan released afterwards.
static int sep_oneshot(bool fwd, const void *phase0, const void *phase1, const void *sens,
                       const void *in, void *out, int32_t nx, int32_t ny, int32_t n_coils,
                       int64_t n_samples, void *stream) {
    if (!phase0 || !phase1 || !sens || !in || !out) return fail(CSR_ERR_ARG, "null argument");
    int dev = 0;
    CU(cudaGetDevice(&dev));
    cudaStream_t st = (cudaStream_t)stream;
    CU(cudaStreamSynchronize(st));  // the plan build reads the factors on its own stream
    csr_factor_desc fd{};
    fd.nx = nx;
    fd.ny = ny;
    fd.n_coils = n_coils;
    fd.n_samples = n_samples;
    fd.phase0 = phase0;
    fd.phase1 = phase1;
    fd.phase1_layout = fwd ? CSR_P1_T : CSR_P1_CONJ;
    fd.sens = sens;
    fd.device = dev;
    csr_plan *p = nullptr;
    TRY(csr_plan_create_from_factors(&fd, &p));
    const int rc = fwd ? csr_forward(p, in, out, stream) : csr_adjoint(p, in, out, stream);
    csr_plan_destroy(p);
    return rc;
}

int csr_nudft_forward_sep(const void *phase0, const void *phase1_t, const void *sens,
                          const void *image, void *out, int32_t nx, int32_t ny,
                          int32_t n_coils, int64_t n_samples, void *stream) {
    return sep_oneshot(true, phase0, phase1_t, sens, image, out, nx, ny, n_coils, n_samples,
                       stream);
}

int csr_nudft_adjoint_sep(const void *phase0, const void *phase1_conj, const void *sens,
                          const void *data, void *out, int32_t nx, int32_t ny,
                          int32_t n_coils, int64_t n_samples, void *stream) {
    return sep_oneshot(false, phase0, phase1_conj, sens, data, out, nx, ny, n_coils, n_samples,
                       stream);
}

int csr_comm_allreduce(csr_comm *c, void *buf, int64_t n_floats, void *stream) {
    if (!c) return fail(CSR_ERR_ARG, "null comm");
    CU(cudaSetDevice(c->device));
    NC(ncclAllReduce(buf, buf, (size_t)n_floats, ncclFloat, ncclSum, c->comm,
                     (cudaStream_t)stream));
    return CSR_OK;
}

}  // extern "C"
