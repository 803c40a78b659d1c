// PCIe duplex probe: H2D and D2H on two non-blocking streams, single vs split copies.
#include <cstdio>
#include <cuda_runtime.h>
int main() {
    const size_t nh = 66355200, nd = 60134400;
    void *hh, *hd, *dh, *dd;
    cudaHostAlloc(&hh, nh, 0); cudaHostAlloc(&hd, nd, 0);
    cudaMalloc(&dh, nh); cudaMalloc(&dd, nd);
    cudaStream_t a, b; cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto run = [&](int split, int mode) {
        cudaDeviceSynchronize();
        cudaEventRecord(e0, 0);
        cudaStreamWaitEvent(a, e0, 0); cudaStreamWaitEvent(b, e0, 0);
        for (int i = 0; i < split; ++i) {
            if (mode & 1) cudaMemcpyAsync((char*)dh + nh / split * i, (char*)hh + nh / split * i, nh / split, cudaMemcpyHostToDevice, a);
            if (mode & 2) cudaMemcpyAsync((char*)hd + nd / split * i, (char*)dd + nd / split * i, nd / split, cudaMemcpyDeviceToHost, b);
        }
        cudaEvent_t ea, eb; cudaEventCreate(&ea); cudaEventCreate(&eb);
        cudaEventRecord(ea, a); cudaEventRecord(eb, b);
        cudaStreamWaitEvent(0, ea, 0); cudaStreamWaitEvent(0, eb, 0);
        cudaEventRecord(e1, 0); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        return ms;
    };
    for (int rep = 0; rep < 2; ++rep)
        for (int split : {1, 4, 16})
            printf("split %2d: H2D %.3f ms  D2H %.3f ms  both %.3f ms\n", split, run(split, 1), run(split, 2), run(split, 3));
    return 0;
}
