// Shared helpers for the csrecon_b200 kernels: complex64 arithmetic,
// deterministic two-stage reductions, launch bookkeeping.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

namespace csr {

// Programmatic dependent launch.  Every kernel of the solver loop starts
// with pdl_wait() (griddepcontrol.wait: returns once the preceding kernel has
// completed and its writes are visible; a no-op for an ordinary launch) and
// then lets its own dependent launch (griddepcontrol.launch_dependents), so
// inside the captured iteration graph a kernel's CTAs are resident and
// waiting when its predecessor drains instead of paying the launch gap.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_enter() {
    pdl_wait();
    pdl_trigger();
}

__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// live-timing slots (csr_plan_probe)
enum ProbeSlot { PROBE_FWD = 0, PROBE_ADJ, PROBE_MU, PROBE_RHS, PROBE_PREP, PROBE_TAIL,
                 PROBE_POST, PROBE_SNAP, PROBE_SLOTS };

// Live kernel timing (bench.py's roofline) without perturbing the launch
// stream: pr = {~first CTA start, CTA ticket, sum of durations (ns),
// launches}.  Every CTA stamps its start; the last CTA to finish adds
// (its end - first start) and re-arms the slot for the next launch.
__device__ __forceinline__ void probe_enter(unsigned long long *pr) {
    if (pr && threadIdx.x == 0) atomicMax(&pr[0], ~(unsigned long long)gtimer());
}
// debug timeline (csr_debug_timeline): every probed launch appends
// (slot, first start, last end) when enabled
__device__ unsigned long long g_tl_ring[3 * 4096];
__device__ unsigned g_tl_n;
__device__ int g_tl_on;
__device__ __forceinline__ void probe_exit(unsigned long long *pr) {
    if (!pr || threadIdx.x != 0) return;
    __threadfence();
    const unsigned long long n = (unsigned long long)gridDim.x * gridDim.y * gridDim.z;
    if (atomicAdd(&pr[1], 1ull) == n - 1) {
        const unsigned long long t1 = gtimer();
        const unsigned long long t0 = ~atomicExch(&pr[0], 0ull);
        atomicAdd(&pr[2], t1 - t0);
        atomicAdd(&pr[3], 1ull);
        atomicExch(&pr[1], 0ull);
        if (g_tl_on) {
            const unsigned k = atomicAdd(&g_tl_n, 1u);
            if (k < 4096) {
                g_tl_ring[3 * k] = (unsigned long long)(size_t)pr;
                g_tl_ring[3 * k + 1] = t0;
                g_tl_ring[3 * k + 2] = t1;
            }
        }
    }
}

// Profiling / experiment knobs (environment variables) exist only in debug
// builds (-DCSR_DEBUG=1: tools/build_variants.py variants loaded with
// CSR_VARIANT); the product library never reads them, so a stray variable
// cannot change a reconstruction.
#ifndef CSR_DEBUG
#define CSR_DEBUG 0
#endif
inline const char *dbg_env(const char *name) { return CSR_DEBUG ? getenv(name) : nullptr; }

inline bool pdl_enabled() {
    static const bool on = dbg_env("CSR_NO_PDL") == nullptr;
    return on;
}

// kernel<<<grid, block, smem, st>>>(args...) with the programmatic-
// serialization attribute (the kernel must begin with pdl_enter())
template <typename... KArgs, typename... Args>
inline cudaError_t launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                          cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// the same with a cluster of cluster_x CTAs along x (CTA pairs / TMA multicast pairs)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_cl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                             cudaStream_t st, int cluster_x, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int n = 0;
    if (pdl_enabled()) {
        attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[n].val.programmaticStreamSerializationAllowed = 1;
        ++n;
    }
    if (cluster_x > 1) {
        attr[n].id = cudaLaunchAttributeClusterDimension;
        attr[n].val.clusterDim.x = (unsigned)cluster_x;
        attr[n].val.clusterDim.y = 1;
        attr[n].val.clusterDim.z = 1;
        ++n;
    }
    cfg.attrs = attr;
    cfg.numAttrs = n;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

__host__ __device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// conj(a) * b
__host__ __device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
    return make_float2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__host__ __device__ __forceinline__ float2 cadd(float2 a, float2 b) {
    return make_float2(a.x + b.x, a.y + b.y);
}
__host__ __device__ __forceinline__ float2 csub(float2 a, float2 b) {
    return make_float2(a.x - b.x, a.y - b.y);
}
__host__ __device__ __forceinline__ float2 cconj(float2 a) {
    return make_float2(a.x, -a.y);
}
// acc += a * b
__device__ __forceinline__ void cfma(float2 &acc, float2 a, float2 b) {
    acc.x = fmaf(a.x, b.x, acc.x);
    acc.x = fmaf(-a.y, b.y, acc.x);
    acc.y = fmaf(a.x, b.y, acc.y);
    acc.y = fmaf(a.y, b.x, acc.y);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Deterministic grid reduction of NV doubles: every block writes its
// partial, the last block to arrive (ticket) folds the partials in block
// order and returns true with the totals in `tot` (valid in thread 0).
// Requires blockDim.x to be a multiple of 32 and <= 1024.
template <int NV>
__device__ bool grid_reduce(double (&v)[NV], double *partials,
                            unsigned *ticket, double (&tot)[NV]) {
    __shared__ double sh[NV][32];
    __shared__ int last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        double w = warp_sum(v[i]);
        if (lane == 0) sh[i][warp] = w;
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            double w = lane < nwarps ? sh[i][lane] : 0.0;
            w = warp_sum(w);
            if (lane == 0) partials[(size_t)blockIdx.x * NV + i] = w;
        }
    }
    if (threadIdx.x == 0) {
        __threadfence();
        unsigned t = atomicAdd(ticket, 1u);
        last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!last) return false;
    __threadfence();
    if (warp == 0) {
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            double w = 0.0;
            for (unsigned b = lane; b < gridDim.x; b += 32)
                w += __ldcg(partials + (size_t)b * NV + i);
            w = warp_sum(w);
            tot[i] = w;
        }
    }
    if (threadIdx.x == 0) *ticket = 0u;
    return true;
}

// exact power of two s with s * bound <= 2^14 (1 for bound == 0)
__device__ __forceinline__ float pow2_scale(float bound) {
    if (!(bound > 0.f) || !isfinite(bound)) return 1.f;
    int e;
    frexpf(bound, &e);  // bound = m * 2^e, m in [0.5, 1)
    int s = 14 - e;
    s = max(-120, min(120, s));
    return ldexpf(1.f, s);
}

// deterministic grid max of non-negative values: true in thread 0 of the
// last block to finish, with the maximum in `out`
__device__ bool grid_max(float v, double *partials, unsigned *ticket, float &out) {
    __shared__ float sh[32];
    __shared__ int last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    if (warp == 0) {
        float w = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) w = fmaxf(w, __shfl_xor_sync(0xffffffffu, w, o));
        if (lane == 0) partials[blockIdx.x] = w;
    }
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return false;
    __threadfence();
    if (warp != 0) return false;
    float w = 0.f;
    for (unsigned b = lane; b < gridDim.x; b += 32) w = fmaxf(w, (float)__ldcg(partials + b));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) w = fmaxf(w, __shfl_xor_sync(0xffffffffu, w, o));
    if (lane != 0) return false;
    *ticket = 0u;
    out = w;
    return true;
}

// Plan buffers come from the device's default stream-ordered pool with an
// unbounded release threshold, so building and dropping plans (one per
// reconstruction call) reuses memory instead of paying cudaMalloc/cudaFree
// (and the device-wide sync of cudaFree) every time.
inline cudaError_t pool_alloc(void **p, size_t bytes, cudaStream_t st) {
    static bool configured[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 64 && !configured[dev]) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        configured[dev] = true;
    }
    return cudaMallocAsync(p, bytes ? bytes : 16, st);
}

// Grid size used by every reduction kernel over n elements: a function of n
// only, so reductions are run-to-run deterministic.
inline int reduce_blocks(int64_t n, int threads) {
    int64_t b = (n + threads - 1) / threads;
    if (b > 4 * 148) b = 4 * 148;
    if (b < 1) b = 1;
    return (int)b;
}

}  // namespace csr
