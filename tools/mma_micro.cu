// tcgen05.mma rate microbenchmark on sm_100a: cycles per M=128 x N x K=16
// kind::f16 MMA issued back to back (one warp, elected lane, unrolled with
// compile-time descriptors so the issue loop is not the bound), into one
// accumulator (each MMA depends on the previous one's D) or rotating over
// NACC independent accumulators, A from shared memory (SS) or from tensor
// memory (TS).  One CTA per SM, all SMs busy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_micro tools/mma_micro.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cstdlib>

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

// Complex-GEMM tile forms, fed like the forward (bulk copies of operand
// stages from an L2-resident source, full / empty barriers), with the
// epilogue's TMEM drains.  One tile = 128 rows x 128 complex columns x 256
// complex K (config 4's forward tile):
//  DBL   the doubled-row form: 8 K blocks of [A_hi|A_lo] 16 KiB each +
//        [B_hi|B_lo] 32 KiB each (96 KiB stages), 3 N = 256 MMAs per K16,
//        two 256-column accumulators (drain of one overlaps the other);
//  GAUSS three real products K1 = (Ar+Ai)Br, K2 = Ar(Bi-Br), K3 = Ai(Br+Bi):
//        12 sub-stages of [A_hi|A_lo|B_hi|B_lo] 16 KiB each (64 KiB), 3 N = 128
//        MMAs per K16 into accumulator j (columns 128 j), each accumulator
//        released by the epilogue as soon as it is read (K1, K2, K3 order).
// NEPI epilogue warps drain (tcgen05.ld) every accumulator of every tile.
template <bool GAUSS, int NSTG, int NEPI>
__global__ void k_cplx(int n_tiles, const uint8_t *gsrc, size_t gbytes, unsigned long long *out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    constexpr int STAGE = GAUSS ? 65536 : 98304;
    constexpr int NSUB = GAUSS ? 12 : 8;   // stages per tile
    constexpr int NACC = GAUSS ? 3 : 2;
    constexpr int ACOL = GAUSS ? 128 : 256;
    __shared__ uint64_t full[4], empty[4], tfull[3], tempty[3], done;
    __shared__ uint32_t tslot;
    __shared__ float sink;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NSTG; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int j = 0; j < 3; ++j) {
            mbar_init(&tfull[j], 1);
            mbar_init(&tempty[j], NEPI > 0 ? NEPI : 1);
        }
        mbar_init(&done, 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc(&tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (warp == 1 && lane == 0) {
        int it = 0;
        for (int t = 0; t < n_tiles; ++t)
            for (int sb = 0; sb < NSUB; ++sb, ++it) {
                const int s = it % NSTG;
                mbar_wait(&empty[s], ((it / NSTG) & 1) ^ 1);
                mbar_arrive_expect_tx(&full[s], STAGE);
                const size_t off = ((size_t)(blockIdx.x * 977 + it) * STAGE) % (gbytes - STAGE);
                bulk_g2s(sm + s * STAGE, gsrc + (off & ~(size_t)1023), STAGE, &full[s]);
            }
    } else if (warp == 0) {
        const long long t0 = clock64();
        int it = 0;
        for (int t = 0; t < n_tiles; ++t) {
            for (int sb = 0; sb < NSUB; ++sb, ++it) {
                const int j = GAUSS ? sb % 3 : (t & 1);
                const int use = GAUSS ? t : (t >> 1);   // uses of accumulator j so far
                if ((GAUSS && sb < 3) || (!GAUSS && sb == 0)) {
                    if (NEPI > 0) mbar_wait(&tempty[j], (use & 1) ^ 1);
                    tc_fence_after();
                }
                const int s = it % NSTG;
                mbar_wait(&full[s], (it / NSTG) & 1);
                tc_fence_after();
                const uint32_t st = smem_u32(sm + s * STAGE);
                const uint32_t d = tmem + j * ACOL;
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const uint32_t acc = GAUSS ? (sb >= 3 || kk > 0) : (sb > 0 || kk > 0);
                        if (GAUSS) {
                            constexpr uint32_t idesc = idesc_f16(128, 128);
                            const uint64_t dah = desc_sw128(st + kk * 32), dal = desc_sw128(st + 16384 + kk * 32);
                            const uint64_t dbh = desc_sw128(st + 32768 + kk * 32), dbl = desc_sw128(st + 49152 + kk * 32);
                            mma_f16_fill(d, dah, dbh, idesc, acc);
                            mma_f16_lastuse(d, dah, dbl, idesc, 1);
                            mma_f16(d, dal, dbh, idesc, 1);
                        } else {
                            constexpr uint32_t idesc = idesc_f16(128, 256);
                            const uint64_t dah = desc_sw128(st + kk * 32), dal = desc_sw128(st + 16384 + kk * 32);
                            const uint64_t dbh = desc_sw128(st + 32768 + kk * 32), dbl = desc_sw128(st + 65536 + kk * 32);
                            mma_f16_fill(d, dah, dbh, idesc, acc);
                            mma_f16_lastuse(d, dah, dbl, idesc, 1);
                            mma_f16(d, dal, dbh, idesc, 1);
                        }
                    }
                    mma_commit(&empty[s]);
                    if ((GAUSS && sb >= NSUB - 3) || (!GAUSS && sb == NSUB - 1)) mma_commit(&tfull[j]);
                }
                __syncwarp();
            }
        }
        if (elect_one()) mma_commit(&done);
        __syncwarp();
        mbar_wait(&done, 0);
        const long long t1 = clock64();
        if (lane == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
    } else if (warp >= 2 && warp < 2 + NEPI) {
        const int e = warp - 2, q = warp & 3;
        constexpr int SHARE = NEPI >= 4 ? ACOL / (NEPI / 4) : ACOL;  // columns per warp
        const int c0 = NEPI >= 8 ? (e / 4) * SHARE : 0;
        float acc = 0.f;
        for (int t = 0; t < n_tiles; ++t) {
            for (int jj = 0; jj < (GAUSS ? 3 : 1); ++jj) {
                const int j = GAUSS ? jj : (t & 1);
                const int use = GAUSS ? t : (t >> 1);
                mbar_wait(&tfull[j], use & 1);
                tc_fence_after();
                const uint32_t base = tmem + ((uint32_t)(q * 32) << 16) + j * ACOL + c0;
                for (int c = 0; c < SHARE; c += 32) {
                    uint32_t r[32];
                    tmem_ld32(base + c, r);
                    tmem_ld_wait();
#pragma unroll
                    for (int i = 0; i < 32; ++i) acc += __uint_as_float(r[i]);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[j]);
            }
        }
        if (acc == 1.2345f) sink = acc;
    }
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

template <bool GAUSS, int NSTG, int NEPI>
void run_cplx(unsigned long long *d_out, const uint8_t *g, size_t gbytes) {
    const int smem = NSTG * (GAUSS ? 65536 : 98304) + 1024;
    cudaFuncSetAttribute(k_cplx<GAUSS, NSTG, NEPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int nt = 64;
    unsigned long long h[148];
    for (int it = 0; it < 2; ++it) {
        k_cplx<GAUSS, NSTG, NEPI><<<148, 64 + 32 * (NEPI > 0 ? NEPI : 0), smem>>>(nt, g, gbytes, d_out);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("error %s\n", cudaGetErrorString(e));
            return;
        }
    }
    cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
    double s = 0;
    for (int i = 0; i < 148; ++i) s += (double)h[i];
    const double per_tile = s / 148 / nt;
    printf("complex tile 128x128x256 %s, %d stages, %d drain warps: %7.0f cycles/tile (MMA floor %d)\n",
           GAUSS ? "GAUSS (3 x N=128 products)" : "DBL (doubled rows, N=256)", NSTG, NEPI, per_tile,
           GAUSS ? 9216 : 12288);
}

// The same tile forms on a CTA pair (cta_group::2): M = 256 (128 rows per
// CTA), each CTA's stage holds its 128 A rows and HALF of the B rows, the
// leader issues the pair MMAs.  Per SM: DBL 64 KiB stages (A hi/lo 16 KiB,
// B hi/lo halves 16 KiB), GAUSS 48 KiB sub-stages (B halves 8 KiB).  The
// peer's bulk copies complete on its own barrier and a relay lane forwards
// the arrival to the leader (the real kernels use the cta_group::2 TMA form).
__device__ __forceinline__ void mma_f16_pair_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                                uint32_t acc, int coll) {
    if (coll == 1)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::2.kind::f16.collector::a::fill [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
    else if (coll == 2)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::2.kind::f16.collector::a::lastuse [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
    else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
template <bool GAUSS, int NSTG, int NEPI>
__global__ void __cluster_dims__(2, 1, 1) k_cplx2(int n_tiles, const uint8_t *gsrc, size_t gbytes,
                                                  unsigned long long *out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    constexpr int BH = GAUSS ? 8192 : 16384;       // B half (hi or lo) per CTA
    constexpr int STAGE = 32768 + 2 * BH;
    constexpr int NSUB = GAUSS ? 12 : 8;
    constexpr int ACOL = GAUSS ? 128 : 256;
    __shared__ __align__(8) uint64_t full[4], full2[4], empty[4], tfull[3], tempty[3], done;
    __shared__ uint32_t tslot;
    __shared__ float sink;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    if (threadIdx.x == 0) {
        for (int s = 0; s < NSTG; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&full2[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int j = 0; j < 3; ++j) {
            mbar_init(&tfull[j], 1);
            mbar_init(&tempty[j], NEPI > 0 ? 2 * NEPI : 1);
        }
        mbar_init(&done, 1);
        fence_barrier_init_cluster();
    }
    if (warp == 0) tmem_alloc_pair(&tslot, 512);
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (warp == 1 && lane == 0) {
        int it = 0;
        for (int t = 0; t < n_tiles; ++t)
            for (int sb = 0; sb < NSUB; ++sb, ++it) {
                const int s = it % NSTG;
                mbar_wait(&empty[s], ((it / NSTG) & 1) ^ 1);
                mbar_arrive_expect_tx(&full[s], STAGE);
                const size_t off = ((size_t)(blockIdx.x * 977 + it) * STAGE) % (gbytes - STAGE);
                bulk_g2s(sm + s * STAGE, gsrc + (off & ~(size_t)1023), STAGE, &full[s]);
            }
    } else if (warp == 0 && rank == 1 && lane == 0) {
        // relay: the peer's stage landed -> the leader's full2
        const uint32_t remote = mapa_shared(smem_u32(&full2[0]), 0);
        int it = 0;
        for (int t = 0; t < n_tiles; ++t)
            for (int sb = 0; sb < NSUB; ++sb, ++it) {
                const int s = it % NSTG;
                mbar_wait(&full[s], (it / NSTG) & 1);
                mbar_arrive_cluster(remote + s * 8);
            }
    } else if (warp == 0 && rank == 0) {
        const long long t0 = clock64();
        int it = 0;
        for (int t = 0; t < n_tiles; ++t) {
            for (int sb = 0; sb < NSUB; ++sb, ++it) {
                const int j = GAUSS ? sb % 3 : (t & 1);
                const int use = GAUSS ? t : (t >> 1);
                if ((GAUSS && sb < 3) || (!GAUSS && sb == 0)) {
                    if (NEPI > 0) mbar_wait(&tempty[j], (use & 1) ^ 1);
                    tc_fence_after();
                }
                const int s = it % NSTG;
                mbar_wait(&full[s], (it / NSTG) & 1);
                mbar_wait(&full2[s], (it / NSTG) & 1);
                tc_fence_after();
                const uint32_t st = smem_u32(sm + s * STAGE);
                const uint32_t d = tmem + j * ACOL;
                if (elect_one()) {
                    constexpr uint32_t idesc = idesc_f16(256, GAUSS ? 128 : 256);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const uint32_t acc = GAUSS ? (sb >= 3 || kk > 0) : (sb > 0 || kk > 0);
                        const uint64_t dah = desc_sw128(st + kk * 32), dal = desc_sw128(st + 16384 + kk * 32);
                        const uint64_t dbh = desc_sw128(st + 32768 + kk * 32), dbl = desc_sw128(st + 32768 + BH + kk * 32);
                        mma_f16_pair_ss(d, dah, dbh, idesc, acc, 1);
                        mma_f16_pair_ss(d, dah, dbl, idesc, 1, 2);
                        mma_f16_pair_ss(d, dal, dbh, idesc, 1, 0);
                    }
                    mma_commit_pair_mc(&empty[s], 3);
                    if ((GAUSS && sb >= NSUB - 3) || (!GAUSS && sb == NSUB - 1)) mma_commit_pair_mc(&tfull[j], 3);
                }
                __syncwarp();
            }
        }
        if (elect_one()) mma_commit_pair_mc(&done, 3);
        __syncwarp();
        mbar_wait(&done, 0);
        const long long t1 = clock64();
        if (lane == 0) out[blockIdx.x / 2] = (unsigned long long)(t1 - t0);
    } else if (warp >= 2 && warp < 2 + NEPI) {
        const int e = warp - 2, q = warp & 3;
        constexpr int SHARE = NEPI >= 4 ? ACOL / (NEPI / 4) : ACOL;
        const int c0 = NEPI >= 8 ? (e / 4) * SHARE : 0;
        const uint32_t remote = mapa_shared(smem_u32(&tempty[0]), 0);
        float acc = 0.f;
        for (int t = 0; t < n_tiles; ++t) {
            for (int jj = 0; jj < (GAUSS ? 3 : 1); ++jj) {
                const int j = GAUSS ? jj : (t & 1);
                const int use = GAUSS ? t : (t >> 1);
                mbar_wait(&tfull[j], use & 1);
                tc_fence_after();
                const uint32_t base = tmem + ((uint32_t)(q * 32) << 16) + j * ACOL + c0;
                for (int c = 0; c < SHARE; c += 32) {
                    uint32_t r[32];
                    tmem_ld32(base + c, r);
                    tmem_ld_wait();
#pragma unroll
                    for (int i = 0; i < 32; ++i) acc += __uint_as_float(r[i]);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(remote + j * 8);
            }
        }
        if (acc == 1.2345f) sink = acc;
    }
    __syncthreads();
    cluster_sync();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc_pair(tmem, 512);
    }
}

template <bool GAUSS, int NSTG, int NEPI>
void run_cplx2(unsigned long long *d_out, const uint8_t *g, size_t gbytes) {
    const int smem = NSTG * (32768 + 2 * (GAUSS ? 8192 : 16384)) + 1024;
    cudaFuncSetAttribute(k_cplx2<GAUSS, NSTG, NEPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int nt = 64;
    unsigned long long h[74];
    for (int it = 0; it < 2; ++it) {
        k_cplx2<GAUSS, NSTG, NEPI><<<148, 64 + 32 * NEPI, smem>>>(nt, g, gbytes, d_out);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("error %s\n", cudaGetErrorString(e));
            return;
        }
    }
    cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
    double s = 0;
    for (int i = 0; i < 74; ++i) s += (double)h[i];
    const double per_tile = s / 74 / nt;  // one pair tile = 2 single tiles of work
    printf("PAIR complex tile 256x128x256 %s, %d stages, %d drain warps/CTA: %7.0f cycles/pair tile "
           "(MMA floor %d)\n", GAUSS ? "GAUSS (3 x N=128 products)" : "DBL (doubled rows, N=256)", NSTG,
           NEPI, per_tile, GAUSS ? 9216 : 12288);
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

// random fp16 in [-1, 1) (realistic operand toggling for the power runs)
__global__ void k_fill_rand(uint16_t *p, size_t n, unsigned seed) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        unsigned h = (unsigned)i * 2654435761u ^ seed;
        h ^= h >> 15; h *= 2246822519u; h ^= h >> 13;
        const float v = (float)(h & 0xFFFFFF) / 8388608.0f - 1.0f;
        p[i] = __half_as_ushort(__float2half_rn(v));
    }
}
// sustained run of one form: tiles of complex work per second (the caller
// samples nvidia-smi clocks / power meanwhile)
template <bool GAUSS, bool PAIR, int NSTG, int NEPI>
void power_run(unsigned long long *d_out, const uint8_t *g, size_t gbytes, double secs, const char *name) {
    const int nt = 64;
    const int smem = PAIR ? NSTG * (32768 + 2 * (GAUSS ? 8192 : 16384)) + 1024
                          : NSTG * (GAUSS ? 65536 : 98304) + 1024;
    if (PAIR) cudaFuncSetAttribute(k_cplx2<GAUSS, NSTG, NEPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    else cudaFuncSetAttribute(k_cplx<GAUSS, NSTG, NEPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int launches = 0;
    float ms = 0.f;
    cudaEventRecord(a);
    while (ms < secs * 1e3) {
        for (int r = 0; r < 20; ++r, ++launches) {
            if (PAIR) k_cplx2<GAUSS, NSTG, NEPI><<<148, 64 + 32 * NEPI, smem>>>(nt, g, gbytes, d_out);
            else k_cplx<GAUSS, NSTG, NEPI><<<148, 64 + 32 * (NEPI > 0 ? NEPI : 0), smem>>>(nt, g, gbytes, d_out);
        }
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
    }
    // complex work per launch: 148 SMs x nt tiles of 128 x 128 x 256 complex MACs
    const double cmacs = 148.0 * nt * 128.0 * 128.0 * 256.0 * launches;
    printf("POWER %s: %.3f s, %.1f complex TMAC/s (x8 = algorithmic TFLOP/s %.1f)\n", name, ms / 1e3,
           cmacs / (ms * 1e-3) / 1e12, 8 * cmacs / (ms * 1e-3) / 1e12);
    fflush(stdout);
}

int main(int argc, char **argv) {
    if (argc > 2 && argv[1][0] == 'p') {  // power mode: mma_micro p <form>
        unsigned long long *d_out;
        cudaMalloc(&d_out, 148 * 8);
        uint8_t *g;
        cudaMalloc(&g, 8 << 20);
        k_fill_rand<<<148 * 4, 256>>>(reinterpret_cast<uint16_t *>(g), (8 << 20) / 2, 12345u);
        cudaDeviceSynchronize();
        const int form = atoi(argv[2]);
        const double secs = argc > 3 ? atof(argv[3]) : 4.0;
        if (form == 0) power_run<false, false, 2, 4>(d_out, g, 8 << 20, secs, "DBL single");
        if (form == 1) power_run<false, true, 3, 4>(d_out, g, 8 << 20, secs, "DBL pair");
        if (form == 2) power_run<true, false, 3, 4>(d_out, g, 8 << 20, secs, "GAUSS single");
        if (form == 3) power_run<true, true, 4, 4>(d_out, g, 8 << 20, secs, "GAUSS pair");
        return 0;
    }
    const bool only_cplx = argc > 1;
    unsigned long long *d_out;
    cudaMalloc(&d_out, 148 * 8);
    if (!only_cplx) {
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
    }
    uint8_t *g_small, *g_big;
    cudaMalloc(&g_small, 8 << 20);   // L2-resident source
    cudaMalloc(&g_big, 1ull << 31);  // 2 GiB: mostly HBM
    cudaMemset(g_small, 0x3c, 8 << 20);
    cudaMemset(g_big, 0x3c, 1ull << 31);
    if (!only_cplx) {
    run_pipe<false, 2>(d_out, g_small, 8 << 20, "L2 (8 MiB)");
    run_pipe<false, 3>(d_out, g_small, 8 << 20, "L2 (8 MiB)");
    run_pipe<true, 2>(d_out, g_small, 8 << 20, "L2 (8 MiB)");
    run_pipe<true, 3>(d_out, g_small, 8 << 20, "L2 (8 MiB)");
    run_pipe<true, 3>(d_out, g_big, 1ull << 31, "HBM (2 GiB)");
    run_pipe<false, 3, 1>(d_out, g_small, 8 << 20, "L2 (8 MiB)");
    run_pipe<true, 3, 2>(d_out, g_small, 8 << 20, "L2 (8 MiB)");
    run_pipe<true, 3, 3>(d_out, g_small, 8 << 20, "L2 (8 MiB)");
    }
    run_cplx<false, 2, 0>(d_out, g_small, 8 << 20);
    run_cplx<false, 2, 4>(d_out, g_small, 8 << 20);
    run_cplx<true, 3, 0>(d_out, g_small, 8 << 20);
    run_cplx<true, 3, 4>(d_out, g_small, 8 << 20);
    run_cplx<true, 3, 8>(d_out, g_small, 8 << 20);
    run_cplx2<false, 3, 0>(d_out, g_small, 8 << 20);
    run_cplx2<false, 3, 4>(d_out, g_small, 8 << 20);
    run_cplx2<true, 4, 0>(d_out, g_small, 8 << 20);
    run_cplx2<true, 4, 4>(d_out, g_small, 8 << 20);
    run_cplx2<true, 4, 8>(d_out, g_small, 8 << 20);
    run_cplx2<true, 3, 8>(d_out, g_small, 8 << 20);
    return 0;
}
