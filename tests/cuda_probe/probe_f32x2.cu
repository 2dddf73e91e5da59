// Probe: do packed FP32 ops (FADD2/FFMA2/FMUL2) execute on this device?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(float* out, int which) {
    float2 a = make_float2(threadIdx.x, 2.f), b = make_float2(3.f, 4.f);
    float2 r = a;
    if (which == 0) r = __fadd2_rn(a, b);
    if (which == 1) r = __fmul2_rn(a, b);
    if (which == 2) r = __ffma2_rn(a, b, a);
    if (which == 3) r = __ffma2_rn(b, make_float2(-1.f, -1.f), a);
    out[threadIdx.x] = r.x + r.y;
}
int main() {
    float* d; cudaMalloc(&d, 128 * 4);
    for (int w = 0; w < 4; ++w) {
        k<<<1, 32>>>(d, w);
        cudaError_t e = cudaDeviceSynchronize();
        float h[32]; cudaMemcpy(h, d, 128, cudaMemcpyDeviceToHost);
        printf("which=%d err=%s out1=%f\n", w, cudaGetErrorString(e), h[1]);
        if (e) return 1;
    }
    return 0;
}
