// GPU data generation: the reference's
// simulate_kspace (acquisition.py:233-257), direct multi-coil encoding in
// double precision,
//
//     d[t*M + k, c] = sum_{x,y} s_c[x,y] img[t,x,y] exp(-2 pi i (kx rx + ky ry))
//
// evaluated separably as sum_x E0[k,x] sum_y E1[k,y] (s_c img)[x,y] with the
// unit-modulus factors generated on the fly in f64 (sincospi), so nothing
// but the image, maps and coordinates is read.  FP64 SIMT: 64 samples x 64
// pixel columns per CTA tile, 4 x 4 complex accumulators per thread.  This is
// a data generator (config 4 needs 5.8 TFLOP of f64 work, hours on the CPU
// oracle); the CPU f64 direct sum stays the oracle it is tested against.
#pragma once

#include "common.cuh"

namespace csr {

__device__ __forceinline__ void zfma(double2 &acc, double2 a, double2 b) {
    acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
    acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
}
__device__ __forceinline__ double2 zmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// exp(-2 pi i k r) in f64
__device__ __forceinline__ double2 unit_phase(double k, double r) {
    double s, c;
    sincospi(-2.0 * (k * r), &s, &c);
    return make_double2(c, s);
}

constexpr int SIM_T = 64;  // samples / pixel columns per tile
constexpr int SIM_K = 8;   // y chunk

// grid: x = sample tiles, y = coil, z = frame
__global__ __launch_bounds__(256) void k_simulate_f64(const double *__restrict__ coords,
                                                      const double2 *__restrict__ sens,
                                                      const double2 *__restrict__ img,
                                                      double2 *__restrict__ out, int64_t M,
                                                      int nx, int ny, int C) {
    pdl_enter();
    __shared__ double2 As[SIM_K][SIM_T + 1];  // As[y][k] = E1[k, y]
    __shared__ double2 Bs[SIM_K][SIM_T + 1];  // Bs[y][x] = s_c img
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int64_t k0 = (int64_t)blockIdx.x * SIM_T;
    const int c = blockIdx.y, t = blockIdx.z;
    const double *crd = coords + (int64_t)t * M * 2;
    const double2 *sc = sens + (int64_t)c * nx * ny;
    const double2 *im = img + (int64_t)t * nx * ny;
    const int hx = nx / 2, hy = ny / 2;  // r = index - n//2 (acquisition.py:39-43)
    double2 rd[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) rd[i] = make_double2(0.0, 0.0);
    for (int x0 = 0; x0 < nx; x0 += SIM_T) {
        double2 acc[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int l = 0; l < 4; ++l) acc[i][l] = make_double2(0.0, 0.0);
        for (int y0 = 0; y0 < ny; y0 += SIM_K) {
            for (int e = tid; e < SIM_K * SIM_T; e += 256) {
                const int r = e % SIM_T, cy = e / SIM_T;
                const int64_t k = k0 + r;
                const int y = y0 + cy, x = x0 + r;
                As[cy][r] = (k < M && y < ny) ? unit_phase(crd[2 * k + 1], (double)(y - hy))
                                              : make_double2(0.0, 0.0);
                Bs[cy][r] = (x < nx && y < ny)
                                ? zmul(sc[(int64_t)x * ny + y], im[(int64_t)x * ny + y])
                                : make_double2(0.0, 0.0);
            }
            __syncthreads();
#pragma unroll
            for (int j = 0; j < SIM_K; ++j) {
                double2 a[4], bb[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    a[i] = As[j][ty * 4 + i];
                    bb[i] = Bs[j][tx * 4 + i];
                }
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int l = 0; l < 4; ++l) zfma(acc[i][l], a[i], bb[l]);
            }
            __syncthreads();
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int64_t k = k0 + ty * 4 + i;
            if (k >= M) continue;
            const double kx = crd[2 * k];
#pragma unroll
            for (int l = 0; l < 4; ++l) {
                const int x = x0 + tx * 4 + l;
                if (x < nx) zfma(rd[i], unit_phase(kx, (double)(x - hx)), acc[i][l]);
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) {
            rd[i].x += __shfl_xor_sync(0xffffffffu, rd[i].x, o);
            rd[i].y += __shfl_xor_sync(0xffffffffu, rd[i].y, o);
        }
    }
    if (tx == 0) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int64_t k = k0 + ty * 4 + i;
            if (k < M) out[((int64_t)t * M + k) * C + c] = rd[i];
        }
    }
}

}  // namespace csr
