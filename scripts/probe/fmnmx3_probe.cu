// probe: three-input min/max (FMNMX3) vs nested fminf/fmaxf on NaN / inf / signed zeros
#include <cstdio>
#include <cmath>
__device__ float fmin3f(float a, float b, float c) { float d; asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d; }
__device__ float fmax3f(float a, float b, float c) { float d; asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d; }
__global__ void k(const float *v, int n, int *bad) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * n * n) return;
    float a = v[i % n], b = v[(i / n) % n], c = v[i / (n * n)];
    float m1 = fmin3f(a, b, c), m2 = fminf(fminf(a, b), c);
    float x1 = fmax3f(a, b, c), x2 = fmaxf(fmaxf(a, b), c);
    if (__float_as_int(m1) != __float_as_int(m2) || __float_as_int(x1) != __float_as_int(x2)) {
        int k = atomicAdd(bad, 1);
        if (k < 12) printf("a=%g b=%g c=%g  min3=%g(%08x) nested=%g(%08x)  max3=%g(%08x) nested=%g(%08x)\n", a, b, c, m1,
                           __float_as_int(m1), m2, __float_as_int(m2), x1, __float_as_int(x1), x2, __float_as_int(x2));
    }
}
int main() {
    float h[] = {NAN, -NAN, INFINITY, -INFINITY, 0.0f, -0.0f, 1.0f, -1.0f, 1e-9f, 3.5f};
    const int n = sizeof(h) / sizeof(h[0]);
    float *d; int *bad; cudaMalloc(&d, sizeof(h)); cudaMalloc(&bad, 4); cudaMemset(bad, 0, 4);
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    k<<<(n * n * n + 127) / 128, 128>>>(d, n, bad);
    int hb = 0; cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
    printf("mismatches: %d of %d\n", hb, n * n * n);
    return 0;
}
