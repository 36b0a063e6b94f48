// tcgen05.mma rate microbenchmark on sm_100a: cycles per M=128 x N x K=16
// kind::f16 MMA issued back to back (one warp, elected lane, unrolled with
// compile-time descriptors so the issue loop is not the bound), into one
// accumulator (each MMA depends on the previous one's D) or rotating over
// NACC independent accumulators, A from shared memory (SS) or from tensor
// memory (TS).  One CTA per SM, all SMs busy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_micro tools/mma_micro.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2006_14080_b200/csrc/sm100.cuh"

using namespace sm100;

template <int N, int NACC, bool TS>
__global__ void k_mma(int n_rep, unsigned long long *out) {
    extern __shared__ __align__(1024) uint8_t tile[];  // A 16 KiB | B 32 KiB
    __shared__ uint64_t done;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x)
        reinterpret_cast<uint32_t *>(tile)[i] = 0x3c003c00u;  // fp16 1.0
    if (threadIdx.x == 0) {
        mbar_init(&done, 1);
        fence_barrier_init();
    }
    fence_proxy_async_smem();
    if (warp == 0) tmem_alloc(&tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (warp == 0) {
        constexpr uint32_t idesc = idesc_f16(128, N);
        const uint32_t a = smem_u32(tile), b = smem_u32(tile + 16384);
        const long long t0 = clock64();
        for (int r = 0; r < n_rep; ++r) {
            if (elect_one()) {
#pragma unroll
                for (int j = 0; j < 4 * NACC; ++j) {
                    const int k = j & 3;
                    const uint32_t d = tmem + (uint32_t)((j % NACC) * N);
                    const uint64_t db = desc_sw128(b + k * 32);
                    if (TS) mma_f16_ts(d, tmem + 384 + 8 * k, db, idesc, r > 0 || j >= NACC);
                    else mma_f16(d, desc_sw128(a + k * 32), db, idesc, r > 0 || j >= NACC);
                }
            }
            __syncwarp();
        }
        if (elect_one()) mma_commit(&done);
        __syncwarp();
        mbar_wait(&done, 0);
        const long long t1 = clock64();
        if ((threadIdx.x & 31) == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
    }
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// the GEMMs' pattern: per K16 step three N = 256 MMAs (A_hi B_hi, A_hi B_lo,
// A_lo B_hi) into one accumulator; per K block (4 steps) the B stage rotates
// over 3 stages of [B_hi | B_lo] (64 KiB each); WRITERS warps meanwhile
// store 64 KiB per K block into the next stage (st.shared, like a TMA fill)
template <bool TS, int WRITERS>
__global__ void k_pattern(int n_blocks, unsigned long long *out) {
    extern __shared__ __align__(1024) uint8_t sm[];  // A hi/lo 32 KiB | 3 x 64 KiB B
    __shared__ uint64_t done;
    __shared__ uint32_t tslot;
    __shared__ volatile int kb_now;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < (32768 + 3 * 65536) / 4; i += blockDim.x)
        reinterpret_cast<uint32_t *>(sm)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) {
        mbar_init(&done, 1);
        fence_barrier_init();
        kb_now = 0;
    }
    fence_proxy_async_smem();
    if (warp == 0) tmem_alloc(&tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    constexpr uint32_t idesc = idesc_f16(128, 256);
    if (warp == 0) {
        const uint32_t a = smem_u32(sm), bb = smem_u32(sm + 32768);
        const long long t0 = clock64();
        for (int kb = 0; kb < n_blocks; ++kb) {
            const uint32_t st = bb + (kb % 3) * 65536;
            if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const uint64_t dbh = desc_sw128(st + kk * 32), dbl = desc_sw128(st + 32768 + kk * 32);
                    const uint32_t acc = (kb | kk) != 0;
                    if (TS) {
                        mma_f16_ts(tmem, tmem + 256 + 8 * kk, dbh, idesc, acc);
                        mma_f16_ts(tmem, tmem + 256 + 8 * kk, dbl, idesc, 1);
                        mma_f16_ts(tmem, tmem + 256 + 32 + 8 * kk, dbh, idesc, 1);
                    } else {
                        const uint64_t dah = desc_sw128(a + kk * 32), dal = desc_sw128(a + 16384 + kk * 32);
                        mma_f16_fill(tmem, dah, dbh, idesc, acc);
                        mma_f16_lastuse(tmem, dah, dbl, idesc, 1);
                        mma_f16(tmem, dal, dbh, idesc, 1);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) kb_now = kb;
        }
        if (elect_one()) mma_commit(&done);
        __syncwarp();
        mbar_wait(&done, 0);
        const long long t1 = clock64();
        if (lane == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
        if (lane == 0) kb_now = -1;
    } else if (warp >= 1 && warp <= WRITERS) {
        // 64 KiB per K block into the stage after the current one
        int last = -2;
        while (true) {
            const int kb = kb_now;
            if (kb < 0 && last >= 0) break;
            if (kb == last) continue;
            last = kb;
            uint4 *dst = reinterpret_cast<uint4 *>(sm + 32768 + ((kb + 1) % 3) * 65536);
            for (int i = (warp - 1) * 32 + lane; i < 4096; i += WRITERS * 32)
                dst[i] = make_uint4(0x3c003c00u, 0x3c003c00u, 0x3c003c00u, 0x3c003c00u);
            if (kb < 0) break;
        }
    }
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

template <bool TS, int WRITERS>
void run_pattern(unsigned long long *d_out) {
    const int smem = 32768 + 3 * 65536 + 1024;
    cudaFuncSetAttribute(k_pattern<TS, WRITERS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int nb = 512;
    unsigned long long h[148];
    for (int it = 0; it < 2; ++it) {
        k_pattern<TS, WRITERS><<<148, 256, smem>>>(nb, d_out);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("error %s\n", cudaGetErrorString(e));
            return;
        }
    }
    cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
    double s = 0;
    for (int i = 0; i < 148; ++i) s += (double)h[i];
    printf("pattern %s, 3 x N=256 MMAs per K16, B stages rotating, %d writer warps (64 KiB/K block): "
           "%6.1f cycles/MMA\n", TS ? "TS (adjoint)" : "SS (forward)", WRITERS, s / 148 / (nb * 12.0));
}

// the pipelined form of the real kernels: a producer lane fills B stages with
// cp.async.bulk (64 KiB from global memory per K block, NSTG stages, full /
// empty mbarriers), the MMA warp waits for each stage, issues the 12 MMAs of
// the K block and commits the stage back
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
template <bool TS, int NSTG, int TM>
__global__ void k_pipe(int n_blocks, const uint8_t *gsrc, size_t gbytes, unsigned long long *out) {
    extern __shared__ __align__(1024) uint8_t sm[];  // A hi/lo 32 KiB | NSTG x 64 KiB B
    __shared__ uint64_t full[4], empty[4], done;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x)
        reinterpret_cast<uint32_t *>(sm)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NSTG; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(&done, 1);
        fence_barrier_init();
    }
    fence_proxy_async_smem();
    if (warp == 0) tmem_alloc(&tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    constexpr uint32_t idesc = idesc_f16(128, 256);
    __shared__ volatile int stop;
    if (threadIdx.x == 0) stop = 0;
    __syncthreads();
    if (TM && warp >= 4 && warp < 8) {
        // TMEM traffic beside the MMAs: lane quarter warp % 4, columns
        // [384, 448) (TM 1: loads like an epilogue drain; TM 2: stores like
        // the adjoint's generators; TM 3: both), until the MMA warp is done
        const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + 448;
        uint32_t r[32];
        for (int i = 0; i < 32; ++i) r[i] = i;
        float acc = 0.f;
        while (!stop) {
            if (TM & 1) {
                tmem_ld32(base, r);
                tmem_ld_wait();
                acc += __uint_as_float(r[lane]);
            }
            if (TM & 2) {
                tmem_st32(base + 32, r);
                tmem_st_wait();
            }
        }
        if (acc == 12345.f) out[0] = 1;
    } else if (warp == 1 && lane == 0) {
        for (int kb = 0; kb < n_blocks; ++kb) {
            const int s = kb % NSTG;
            mbar_wait(&empty[s], ((kb / NSTG) & 1) ^ 1);
            mbar_arrive_expect_tx(&full[s], 65536);
            const size_t off = ((size_t)(blockIdx.x * 977 + kb) * 65536) % (gbytes - 65536);
            bulk_g2s(sm + 32768 + s * 65536, gsrc + (off & ~(size_t)1023), 65536, &full[s]);
        }
    } else if (warp == 0) {
        const uint32_t a = smem_u32(sm), bb = smem_u32(sm + 32768);
        const long long t0 = clock64();
        for (int kb = 0; kb < n_blocks; ++kb) {
            const int s = kb % NSTG;
            mbar_wait(&full[s], (kb / NSTG) & 1);
            tc_fence_after();
            const uint32_t st = bb + s * 65536;
            if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const uint64_t dbh = desc_sw128(st + kk * 32), dbl = desc_sw128(st + 32768 + kk * 32);
                    const uint32_t acc = (kb | kk) != 0;
                    if (TS) {
                        mma_f16_ts(tmem, tmem + 256 + 8 * kk, dbh, idesc, acc);
                        mma_f16_ts(tmem, tmem + 256 + 8 * kk, dbl, idesc, 1);
                        mma_f16_ts(tmem, tmem + 256 + 32 + 8 * kk, dbh, idesc, 1);
                    } else {
                        const uint64_t dah = desc_sw128(a + kk * 32), dal = desc_sw128(a + 16384 + kk * 32);
                        mma_f16_fill(tmem, dah, dbh, idesc, acc);
                        mma_f16_lastuse(tmem, dah, dbl, idesc, 1);
                        mma_f16(tmem, dal, dbh, idesc, 1);
                    }
                }
                mma_commit(&empty[s]);
            }
            __syncwarp();
        }
        if (elect_one()) mma_commit(&done);
        __syncwarp();
        mbar_wait(&done, 0);
        const long long t1 = clock64();
        if (lane == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
        if (lane == 0) stop = 1;
    }
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

template <bool TS, int NSTG, int TM = 0>
void run_pipe(unsigned long long *d_out, const uint8_t *g, size_t gbytes, const char *what) {
    const int smem = 32768 + NSTG * 65536 + 1024;
    cudaFuncSetAttribute(k_pipe<TS, NSTG, TM>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int nb = 512;
    unsigned long long h[148];
    for (int it = 0; it < 2; ++it) {
        k_pipe<TS, NSTG, TM><<<148, 256, smem>>>(nb, g, gbytes, d_out);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("error %s\n", cudaGetErrorString(e));
            return;
        }
    }
    cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
    double s = 0;
    for (int i = 0; i < 148; ++i) s += (double)h[i];
    printf("pipe %s, %d stages of 64 KiB B by cp.async.bulk from %s, TMEM side traffic %s: %6.1f cycles/MMA\n",
           TS ? "TS (adjoint)" : "SS (forward)", NSTG, what,
           TM == 0 ? "none" : TM == 1 ? "ld" : TM == 2 ? "st" : "ld+st", s / 148 / (nb * 12.0));
}

template <int N, int NACC, bool TS>
void run(unsigned long long *d_out) {
    const int smem = 16384 + 32768 + 1024;
    cudaFuncSetAttribute(k_mma<N, NACC, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int n_rep = 1024 / NACC;  // 4096 MMAs
    unsigned long long h[148];
    for (int it = 0; it < 2; ++it) {
        k_mma<N, NACC, TS><<<148, 128, smem>>>(n_rep, d_out);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("error %s\n", cudaGetErrorString(e));
            return;
        }
    }
    cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
    double s = 0;
    for (int i = 0; i < 148; ++i) s += (double)h[i];
    const double cyc = s / 148 / (n_rep * 4 * NACC);
    printf("M=128 N=%3d K=16 %s accumulators=%d: %6.1f cycles/MMA (floor %d) = %5.0f MACs/clk/SM\n",
           N, TS ? "TS" : "SS", NACC, cyc, 128 * N / 256, 128.0 * N * 16 / cyc);
}

int main() {
    unsigned long long *d_out;
    cudaMalloc(&d_out, 148 * 8);
    run<256, 1, false>(d_out);
    run<256, 2, false>(d_out);
    run<256, 1, true>(d_out);
    run<192, 1, false>(d_out);
    run<192, 2, false>(d_out);
    run<128, 1, false>(d_out);
    run<128, 2, false>(d_out);
    run<128, 4, false>(d_out);
    run<128, 1, true>(d_out);
    run<128, 3, true>(d_out);
    run<64, 1, false>(d_out);
    run<64, 4, false>(d_out);
    run_pattern<false, 0>(d_out);
    run_pattern<true, 0>(d_out);
    run_pattern<false, 4>(d_out);
    run_pattern<true, 4>(d_out);
    uint8_t *g_small, *g_big;
    cudaMalloc(&g_small, 8 << 20);   // L2-resident source
    cudaMalloc(&g_big, 1ull << 31);  // 2 GiB: mostly HBM
    cudaMemset(g_small, 0x3c, 8 << 20);
    cudaMemset(g_big, 0x3c, 1ull << 31);
    run_pipe<false, 2>(d_out, g_small, 8 << 20, "L2 (8 MiB)");
    run_pipe<false, 3>(d_out, g_small, 8 << 20, "L2 (8 MiB)");
    run_pipe<true, 2>(d_out, g_small, 8 << 20, "L2 (8 MiB)");
    run_pipe<true, 3>(d_out, g_small, 8 << 20, "L2 (8 MiB)");
    run_pipe<true, 3>(d_out, g_big, 1ull << 31, "HBM (2 GiB)");
    run_pipe<false, 3, 1>(d_out, g_small, 8 << 20, "L2 (8 MiB)");
    run_pipe<true, 3, 2>(d_out, g_small, 8 << 20, "L2 (8 MiB)");
    run_pipe<true, 3, 3>(d_out, g_small, 8 << 20, "L2 (8 MiB)");
    return 0;
}
