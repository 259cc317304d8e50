// PCIe read-back: cudaMemcpyAsync D2H vs a kernel storing into mapped pinned
// host memory (zero-copy), 16 B per thread per iteration, grid = k x SMs.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_zc(const int4 *__restrict__ src, int4 *dst, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        dst[i] = src[i];
}
int main() {
    const size_t bytes = 1342177280ull;  // 1.25 GiB: config-3 frames (depth f32 + seg u8)
    void *d, *h, *hd;
    cudaMalloc(&d, bytes);
    cudaMemset(d, 1, bytes);
    cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
    cudaHostGetDevicePointer(&hd, h, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    float ms;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(a); cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost); cudaEventRecord(b);
        cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        printf("memcpy D2H: %.1f GB/s\n", bytes / ms / 1e6);
    }
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int k : {1, 2, 4, 8, 16}) for (int bs : {256, 1024}) {
        for (int r = 0; r < 2; ++r) {
            cudaEventRecord(a); k_zc<<<k * sms, bs>>>((const int4 *)d, (int4 *)hd, bytes / 16); cudaEventRecord(b);
            cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
            if (r) printf("zero-copy kernel grid %dx%d x %d: %.1f GB/s\n", k, sms, bs, bytes / ms / 1e6);
        }
    }
    // two copies on two streams
    cudaStream_t s1, s2; cudaStreamCreate(&s1); cudaStreamCreate(&s2);
    for (int r = 0; r < 2; ++r) {
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        for (int c = 0; c < 8; ++c) cudaMemcpyAsync((char *)h + c * (bytes / 8), (char *)d + c * (bytes / 8), bytes / 8, cudaMemcpyDeviceToHost, c & 1 ? s1 : s2);
        cudaDeviceSynchronize(); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        printf("8 chunks on 2 streams: %.1f GB/s\n", bytes / ms / 1e6);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
