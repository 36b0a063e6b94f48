// Microbenchmark of the producer/consumer pipeline primitives on sm_100a:
// per-iteration cost of an mbarrier ring between a "producer" warp and an
// "MMA" warp with (a) plain arrives, (b) tcgen05.commit arrives, (c) commit
// after 12 MMAs (128x128x16, A from TMEM), (d) 12 MMAs with A from smem.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_micro pipe_micro.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2006_14080_b200/csrc/sm100.cuh"

using namespace sm100;

__device__ __forceinline__ void wait_test(uint64_t *bar, uint32_t parity) {
    while (!mbar_test_wait(bar, parity)) {
    }
}
__device__ __forceinline__ void wait_hint(uint64_t *bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity), "r"(0x989680)
            : "memory");
    }
}
__device__ __forceinline__ void wait_mode(int wm, uint64_t *bar, uint32_t parity) {
    if (wm == 0) mbar_wait(bar, parity);
    else if (wm == 1) wait_test(bar, parity);
    else wait_hint(bar, parity);
}

__global__ void k_pipe(int mode, int iters, int stages, unsigned long long *out, int burn,
                       int smsp_mask, int PW, int MW, int nowait, int yield_every) {
    const int wm = mode / 100;
    mode %= 100;
    __shared__ __align__(1024) uint8_t tile[40960];
    __shared__ uint64_t full[8], empty[8];
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        if (mode == 5) mbar_init(&empty[1], (1 << 20) - 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(&tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    const unsigned long long t0 = clock64();
    if (mode >= 5 && mode <= 7) {  // single-thread primitive throughput
        if (threadIdx.x == 0) {
            uint64_t *b = &full[0];
            if (mode == 5) {  // arrive only (barrier expects far more)
                for (int i = 0; i < iters; ++i) mbar_arrive(&empty[1]);
            } else if (mode == 6) {  // try_wait on an already completed phase
                for (int i = 0; i < iters; ++i) mbar_wait(b, 1);
            } else if (mode == 7) {  // arrive completing the phase, then wait
                for (int i = 0; i < iters; ++i) {
                    mbar_arrive(b);
                    mbar_wait(b, i & 1);
                }
            }
        }
    } else if (warp != PW && warp != MW && burn && ((smsp_mask >> (warp & 3)) & 1)) {
        // ALU burner warps (FP32 FMA chains, 8 independent) while the MMA runs
        float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
              a6 = a0 + 6, a7 = a0 + 7;
        for (int i = 0; i < iters * burn; ++i) {
            if (yield_every && (i % yield_every) == 0) asm volatile("nanosleep.u32 0;");
            a0 = fmaf(a0, 1.0001f, 0.3f); a1 = fmaf(a1, 1.0001f, 0.3f);
            a2 = fmaf(a2, 1.0001f, 0.3f); a3 = fmaf(a3, 1.0001f, 0.3f);
            a4 = fmaf(a4, 1.0001f, 0.3f); a5 = fmaf(a5, 1.0001f, 0.3f);
            a6 = fmaf(a6, 1.0001f, 0.3f); a7 = fmaf(a7, 1.0001f, 0.3f);
        }
        if (a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 == 0.123f) out[0] = 1;
    } else if (warp == PW && lane == 0 && !(nowait & 1)) {
        for (int i = 0; i < iters; ++i) {
            const int s = i % stages;
            wait_mode(wm, &empty[s], ((i / stages) & 1) ^ 1);
            mbar_arrive(&full[s]);
        }
    } else if (warp == MW && (nowait & 2)) {
        // whole warp runs the loop; one elected lane issues
        const uint32_t idesc = idesc_f16(128, 128);
        const uint64_t bd = desc_sw128(smem_u32(tile));
        for (int i = 0; i < iters; ++i) {
            const int s = i % stages;
            if (!(nowait & 1)) wait_mode(wm, &full[s], (i / stages) & 1);
            tc_fence_after();
            if (elect_one()) {
                for (int k = 0; k < 12; ++k)
                    mma_f16_ts(tmem, tmem + 256 + 8 * (k & 3), bd + 2 * (k & 3), idesc, 1);
                if (!(nowait & 1)) mma_commit(&empty[s]);
            }
            __syncwarp();
        }
        if (elect_one()) {
            if (nowait & 1) mma_commit(&empty[(iters - 1) % stages]);
            if (nowait & 1) wait_mode(wm, &empty[(iters - 1) % stages], 0);
            else wait_mode(wm, &empty[(iters - 1) % stages], ((iters - 1) / stages) & 1);
            out[blockIdx.x] = clock64() - t0;
        }
        __syncwarp();
    } else if (warp == MW && lane == 0) {
        const uint32_t idesc = idesc_f16(128, 128);
        const uint64_t bd = desc_sw128(smem_u32(tile));
        for (int i = 0; i < iters; ++i) {
            const int s = i % stages;
            if (!(nowait & 1)) wait_mode(wm, &full[s], (i / stages) & 1);
            tc_fence_after();
            if (mode == 0) {
                mbar_arrive(&empty[s]);
                continue;
            }
            if (mode == 2) {
                for (int k = 0; k < 12; ++k)
                    mma_f16_ts(tmem, tmem + 256 + 8 * (k & 3), bd + 2 * (k & 3), idesc, 1);
            } else if (mode == 4) {  // hi, lo, lo accumulator pattern (adjoint)
                for (int k = 0; k < 12; ++k)
                    mma_f16_ts(tmem + ((k % 3) ? 128 : 0), tmem + 256 + 8 * (k / 3), bd + 2 * (k / 3), idesc, 1);
            } else if (mode == 8) {  // 4 into hi, then 8 into lo
                for (int k = 0; k < 12; ++k)
                    mma_f16_ts(tmem + (k < 4 ? 0 : 128), tmem + 256 + 8 * (k & 3), bd + 2 * (k & 3), idesc, 1);
            } else if (mode == 10) {  // M=128 N=64: 24 MMAs (same MACs)
                for (int k = 0; k < 24; ++k)
                    mma_f16_ts(tmem, tmem + 256 + 8 * (k & 3), bd + 2 * (k & 3), idesc_f16(128, 64), 1);
            } else if (mode == 11) {  // SS N=256, 6 MMAs
                for (int k = 0; k < 6; ++k)
                    mma_f16(tmem, bd + 2 * (k & 3), bd + 2 * (k & 3), idesc_f16(128, 256), 1);
            } else if (mode == 9) {  // N=256 single accumulator, 6 MMAs (same MACs)
                for (int k = 0; k < 6; ++k)
                    mma_f16_ts(tmem, tmem + 256 + 8 * (k & 3), bd + 2 * (k & 3), idesc_f16(128, 256), 1);
            } else if (mode == 3) {
                for (int k = 0; k < 12; ++k)
                    mma_f16(tmem, bd + 2 * (k & 3), bd + 2 * (k & 3), idesc, 1);
            }
            if (!(nowait & 1)) mma_commit(&empty[s]);
        }
        if (nowait & 1) mma_commit(&empty[(iters - 1) % stages]);
        // wait for the last MMAs, then stamp (the burners may run longer)
        if (nowait & 1) wait_mode(wm, &empty[(iters - 1) % stages], 0);
        else wait_mode(wm, &empty[(iters - 1) % stages], ((iters - 1) / stages) & 1);
        out[blockIdx.x] = clock64() - t0;
    }
    __syncthreads();
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0 && mode >= 5 && mode <= 7) out[blockIdx.x] = t1 - t0;
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

int main() {
    unsigned long long *d, h[148];
    cudaMalloc(&d, sizeof(h));
    const char *names[] = {"plain arrive", "commit only", "12 MMA TS + commit", "12 MMA SS + commit",
                           "12 TS hi/lo/lo", "1T arrive", "1T try_wait done", "1T arrive+wait",
                           "12 TS 4hi+8lo", "6 TS N=256", "24 TS N=64", "6 SS N=256"};
    for (int mode : {2, 9, 10, 3, 11}) {
      for (int burn : {0}) {
       for (int nthr : {128}) {
        for (int pm : {0x01}) {
            const int PW = (pm >> 4) & 15, MW = pm & 15, mask = ((pm >> 12) & 15) ? 0xd : 0xf;
            const int nowait = (pm >> 8) & 3;
            const int iters = 2000, stages = 4;
            const int yield_every = pm >> 16;
            k_pipe<<<148, nthr>>>(mode, iters, stages, d, burn, mask, PW, MW, nowait, yield_every);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("error %s\n", cudaGetErrorString(e));
                return 1;
            }
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            double avg = 0;
            for (int i = 0; i < 148; ++i) avg += h[i];
            avg /= 148;
            printf("%-22s burn=%2d threads=%d mask=%x nowait=%d yield=%d  %8.1f cycles/iter\n", names[mode % 100], burn, nthr, mask, nowait, yield_every, avg / iters);
        }
       }
      }
    }
    return 0;
}
