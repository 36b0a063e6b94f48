// Per-sample cost of the adjoint generator's fp16 hi/lo split (the
// generator is bound by it): current sequence (round to half, convert back,
// subtract, round the remainder) vs a Veltkamp split in fp32 (no half ->
// float conversion).  One and two warps per SMSP, 8 independent samples
// per thread per iteration; results folded into an xor so nothing is dead.
#include <cstdio>
#include <cuda_fp16.h>
template <int MODE>
__global__ void k(unsigned *out, int iters, long long *cyc, float2 pin, float2 uin) {
    float2 p[8], u[8];
    for (int i = 0; i < 8; ++i) {
        p[i] = make_float2(pin.x + threadIdx.x * 1e-3f + i, pin.y - i * 0.5f);
        u[i] = make_float2(uin.x * (i + 1), uin.y + threadIdx.x * 1e-4f);
    }
    unsigned acc = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const float e0 = fmaf(p[i].x, u[i].x, p[i].y * u[i].y);
            const float e1 = fmaf(p[i].y, u[i].x, -(p[i].x * u[i].y));
            __half2 hh, ll;
            if (MODE == 0) {
                hh = __floats2half2_rn(e0, e1);
                const float2 hf = __half22float2(hh);
                ll = __floats2half2_rn(e0 - hf.x, e1 - hf.y);
            } else if (MODE == 1) {
                const float c0 = __fmul_rn(e0, 8193.f), c1 = __fmul_rn(e1, 8193.f);
                const float h0 = __fsub_rn(c0, __fsub_rn(c0, e0));
                const float h1 = __fsub_rn(c1, __fsub_rn(c1, e1));
                hh = __floats2half2_rn(h0, h1);
                ll = __floats2half2_rn(__fsub_rn(e0, h0), __fsub_rn(e1, h1));
            } else {  // only the two packs (lower bound)
                hh = __floats2half2_rn(e0, e1);
                ll = __floats2half2_rn(e1, e0);
            }
            acc ^= *reinterpret_cast<unsigned *>(&hh) + *reinterpret_cast<unsigned *>(&ll);
            u[i].x += 1.0f;  // new inputs every iteration
        }
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    unsigned *o; long long *c;
    cudaMalloc(&o, 148 * 1024 * 4); cudaMalloc(&c, 148 * 8);
    const int iters = 2048;
    const char *names[] = {"current (cvt back)", "veltkamp", "2 packs only"};
    for (int mode = 0; mode < 3; ++mode)
        for (int nthr : {128, 256}) {
            for (int rep = 0; rep < 2; ++rep) {
                if (mode == 0) k<0><<<148, nthr>>>(o, iters, c, make_float2(0.3f, 0.7f), make_float2(1.1f, -0.4f));
                if (mode == 1) k<1><<<148, nthr>>>(o, iters, c, make_float2(0.3f, 0.7f), make_float2(1.1f, -0.4f));
                if (mode == 2) k<2><<<148, nthr>>>(o, iters, c, make_float2(0.3f, 0.7f), make_float2(1.1f, -0.4f));
            }
            cudaDeviceSynchronize();
            long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
            const int wps = nthr / 128;
            printf("%-20s warps/SMSP %d: %.2f cycles per sample per warp, %.2f per SMSP\n", names[mode], wps,
                   (double)h / iters / 8, (double)h / iters / 8 / wps);
        }
    return 0;
}
