// NCCL one-rank probe: send/recv to self in a group (the halo exchange of
// a frame-sharded plan with a one-rank communicator), eagerly and inside a
// captured CUDA graph.  Build + run on the GPU box:
//   nvcc -o /tmp/nccl_self_probe tools/nccl_self_probe.cu -I$NCCL/include -L$NCCL/lib -l:libnccl.so.2
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdio>
#include <vector>

#define CK(x)                                                                     \
    do {                                                                          \
        auto e_ = (x);                                                            \
        if (e_) {                                                                 \
            printf("FAIL %s: %d\n", #x, (int)e_);                                 \
            return 1;                                                             \
        }                                                                         \
    } while (0)

static int exchange(ncclComm_t c, float *a, float *b, float *pa, float *pb, size_t n,
                    cudaStream_t st) {
    CK(ncclGroupStart());
    CK(ncclSend(a, n, ncclFloat, 0, c, st));
    CK(ncclRecv(pa, n, ncclFloat, 0, c, st));
    CK(ncclSend(b, n, ncclFloat, 0, c, st));
    CK(ncclRecv(pb, n, ncclFloat, 0, c, st));
    CK(ncclGroupEnd());
    return 0;
}

int main() {
    ncclUniqueId id;
    CK(ncclGetUniqueId(&id));
    ncclComm_t c;
    CK(ncclCommInitRank(&c, 1, id, 0));
    const size_t n = 1 << 16;
    float *a, *b, *pa, *pb;
    CK(cudaMalloc(&a, n * 4));
    CK(cudaMalloc(&b, n * 4));
    CK(cudaMalloc(&pa, n * 4));
    CK(cudaMalloc(&pb, n * 4));
    std::vector<float> h(n);
    for (size_t i = 0; i < n; ++i) h[i] = (float)i;
    CK(cudaMemcpy(a, h.data(), n * 4, cudaMemcpyHostToDevice));
    for (size_t i = 0; i < n; ++i) h[i] = -(float)i;
    CK(cudaMemcpy(b, h.data(), n * 4, cudaMemcpyHostToDevice));
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    if (exchange(c, a, b, pa, pb, n, st)) return 1;
    CK(cudaStreamSynchronize(st));
    CK(cudaMemcpy(h.data(), pa, n * 4, cudaMemcpyDeviceToHost));
    printf("eager self send/recv: pa[5] = %g (expect 5)\n", h[5]);
    fflush(stdout);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    if (exchange(c, b, a, pa, pb, n, st)) return 1;
    CK(cudaStreamEndCapture(st, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    for (int i = 0; i < 3; ++i) CK(cudaGraphLaunch(ge, st));
    CK(cudaStreamSynchronize(st));
    CK(cudaMemcpy(h.data(), pa, n * 4, cudaMemcpyDeviceToHost));
    printf("graph self send/recv: pa[5] = %g (expect -5)\n", h[5]);
    ncclCommDestroy(c);
    printf("ok\n");
    return 0;
}
