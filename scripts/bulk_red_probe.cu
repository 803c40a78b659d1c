// Random 16-byte fp32 reductions into a 32 MB buffer: red.global.add.v4.f32 (LSU path) vs
// cp.reduce.async.bulk ... add.f32 of 16 bytes from shared memory (TMA path).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bulk scripts/bulk_red_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int kMode>
__global__ void __launch_bounds__(256) k_probe(float* tab, uint32_t mask, int per_thread, uint32_t seed) {
    __shared__ __align__(16) float4 src[256 * 8];
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    for (int c = 0; c < 8; ++c) src[threadIdx.x * 8 + c] = make_float4(1.f, 1.f, 1.f, 1.f);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    uint32_t st[8];
    for (int c = 0; c < 8; ++c) st[c] = (tid * 0x9E3779B9u) ^ (seed + 0x85EBCA6Bu * (uint32_t)(c + 1));
    for (int i = 0; i < per_thread; i += 8) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            st[c] = st[c] * 1664525u + 1013904223u;
            const uint32_t e = (st[c] >> 7) & mask;
            float* p = tab + 4ull * e;
            if constexpr (kMode == 0) {
                asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(1.0f), "f"(1.0f), "f"(1.0f),
                             "f"(1.0f) : "memory");
            } else if constexpr (kMode == 1) {
                asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 16;"
                             ::"l"(p), "r"(smem_u32(&src[threadIdx.x * 8 + c])) : "memory");
            } else {
                asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 64;"
                             ::"l"(tab + 16ull * (e >> 2)), "r"(smem_u32(&src[threadIdx.x * 8 + (c & 4)])) : "memory");
            }
        }
        if constexpr (kMode >= 1) asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    if constexpr (kMode >= 1) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
    const size_t bytes = 32u << 20;
    float* tab;
    cudaMalloc(&tab, bytes);
    cudaMemset(tab, 0, bytes);
    const uint32_t mask = (uint32_t)(bytes / 16 - 1);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8, per_thread = 256;
    const double ops = (double)blocks * 256 * per_thread;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            if (mode == 0) k_probe<0><<<blocks, 256>>>(tab, mask, per_thread, rep);
            else if (mode == 1) k_probe<1><<<blocks, 256>>>(tab, mask, per_thread, rep);
            else k_probe<2><<<blocks, 256>>>(tab, mask, per_thread, rep);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            printf("%s rep %d: %.3f ms, %.1f G ops/s (%s)\n", mode == 0 ? "red.v4" : (mode == 1 ? "bulk16" : "bulk64"), rep, ms, ops / ms / 1e6,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
