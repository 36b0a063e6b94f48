// FP32 SIMT separable NUDFT (K3/K4).  Exact-shape (no padding), used for
// shapes the tensor-core path does not tile and as the bring-up path.
//
// forward:  kd[t*M+k, c] = sum_x P0[k,x] * sum_y P1[k,y] * s_c[x,y]*img[t,x,y]
//           (kernels.py:71-78)
// adjoint:  ws[s][t][c][x][y] = sum_{k in split s} conj(P0[k,x]) kd[k,c] conj(P1[k,y])
//           then k_adj_reduce folds splits and coils (kernels.py:81-88)
#pragma once

#include "common.cuh"

namespace csr {

constexpr int ST = 64;   // tile edge
constexpr int SK = 16;   // contraction chunk
constexpr int SP = ST + 2;  // padded smem row (float2)

__global__ __launch_bounds__(256) void k_forward_simt(
    const float2 *__restrict__ P0, const float2 *__restrict__ P1,
    const float2 *__restrict__ sens, const float2 *__restrict__ img,
    float2 *__restrict__ kd, int M, int nx, int ny, int C, const int *gate) {
    pdl_enter();
    if (gate && !*gate) return;
    __shared__ __align__(16) float2 As[SK][SP];  // As[y][k] = P1[k,y]
    __shared__ __align__(16) float2 Bs[SK][SP];  // Bs[y][x] = s_c*img
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int k0 = blockIdx.x * ST, c = blockIdx.y, t = blockIdx.z;
    const float2 *p0 = P0 + (int64_t)t * M * nx;
    const float2 *p1 = P1 + (int64_t)t * M * ny;
    const float2 *sc = sens + (int64_t)c * nx * ny;
    const float2 *im = img + (int64_t)t * nx * ny;
    float2 rd[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) rd[i] = make_float2(0.f, 0.f);
    for (int x0 = 0; x0 < nx; x0 += ST) {
        float2 acc[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int l = 0; l < 4; ++l) acc[i][l] = make_float2(0.f, 0.f);
        for (int y0 = 0; y0 < ny; y0 += SK) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                int e = tid + 256 * q, r = e >> 4, cy = e & 15;
                int k = k0 + r, y = y0 + cy, x = x0 + r;
                As[cy][r] = (k < M && y < ny) ? p1[(int64_t)k * ny + y] : make_float2(0.f, 0.f);
                Bs[cy][r] = (x < nx && y < ny)
                                ? cmul(sc[(int64_t)x * ny + y], im[(int64_t)x * ny + y])
                                : make_float2(0.f, 0.f);
            }
            __syncthreads();
#pragma unroll
            for (int j = 0; j < SK; ++j) {
                float2 a[4], b[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) { a[i] = As[j][ty * 4 + i]; b[i] = Bs[j][tx * 4 + i]; }
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int l = 0; l < 4; ++l) cfma(acc[i][l], a[i], b[l]);
            }
            __syncthreads();
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            int k = k0 + ty * 4 + i;
            if (k >= M) continue;
#pragma unroll
            for (int l = 0; l < 4; ++l) {
                int x = x0 + tx * 4 + l;
                if (x < nx) cfma(rd[i], p0[(int64_t)k * nx + x], acc[i][l]);
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
            int k = k0 + ty * 4 + i;
            if (k < M) kd[((int64_t)t * M + k) * C + c] = rd[i];
        }
    }
}

// grid: x = x-tiles * y-tiles, y = coil, z = frame + T * split
__global__ __launch_bounds__(256) void k_adjoint_simt(
    const float2 *__restrict__ P0, const float2 *__restrict__ P1,
    const float2 *__restrict__ kd, float2 *__restrict__ ws, int M, int nx,
    int ny, int C, int T, int kchunk, const int *gate) {
    pdl_enter();
    if (gate && !*gate) return;
    __shared__ __align__(16) float2 As[SK][SP];  // As[k][x] = conj(P0[k,x]) d[k,c]
    __shared__ __align__(16) float2 Bs[SK][SP];  // Bs[k][y] = conj(P1[k,y])
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int tiles_y = (ny + ST - 1) / ST;
    const int x0 = (blockIdx.x / tiles_y) * ST, y0 = (blockIdx.x % tiles_y) * ST;
    const int c = blockIdx.y, t = blockIdx.z % T, s = blockIdx.z / T;
    const int ks = s * kchunk, ke = min(M, ks + kchunk);
    const float2 *p0 = P0 + (int64_t)t * M * nx;
    const float2 *p1 = P1 + (int64_t)t * M * ny;
    const float2 *dk = kd + (int64_t)t * M * C + c;
    float2 acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int l = 0; l < 4; ++l) acc[i][l] = make_float2(0.f, 0.f);
    for (int kb = ks; kb < ke; kb += SK) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            int e = tid + 256 * q, r = e & 63, kk = e >> 6;
            int k = kb + kk, x = x0 + r, y = y0 + r;
            float2 w = make_float2(0.f, 0.f), v = make_float2(0.f, 0.f);
            if (k < ke) {
                if (x < nx) w = cmulc(p0[(int64_t)k * nx + x], dk[(int64_t)k * C]);
                if (y < ny) v = cconj(p1[(int64_t)k * ny + y]);
            }
            As[kk][r] = w;
            Bs[kk][r] = v;
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < SK; ++j) {
            float2 a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) { a[i] = As[j][ty * 4 + i]; b[i] = Bs[j][tx * 4 + i]; }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int l = 0; l < 4; ++l) cfma(acc[i][l], a[i], b[l]);
        }
        __syncthreads();
    }
    float2 *out = ws + (((int64_t)s * T + t) * C + c) * (int64_t)nx * ny;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        int x = x0 + ty * 4 + i;
        if (x >= nx) continue;
#pragma unroll
        for (int l = 0; l < 4; ++l) {
            int y = y0 + tx * 4 + l;
            if (y < ny) out[(int64_t)x * ny + y] = acc[i][l];
        }
    }
}

}  // namespace csr
