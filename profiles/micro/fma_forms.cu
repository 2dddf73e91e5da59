// Microbenchmark: issue rate of packed FP32 forms on sm_100a (independent chains).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 fma_forms.cu -o fma_forms
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;
constexpr int kIters = 4096;

template <int kForm>
__global__ void bench(float2* out, float2 a, float2 b) {
    float2 x[kChains];
    a.x += threadIdx.x * 1e-9f; a.y += threadIdx.x * 2e-9f; // per-thread registers, not uniform
    b.x += threadIdx.x * 1e-12f; b.y -= threadIdx.x * 1e-12f;
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = make_float2(threadIdx.x * 1e-6f + c, c * 0.5f);
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            if (kForm == 0) x[c] = __fadd2_rn(x[c], a);                                     // FADD2 reg, reg
            if (kForm == 1) x[c] = __ffma2_rn(x[c], make_float2(1.0f, 1.0f), a);            // FFMA2 with imm 1
            if (kForm == 2) x[c] = __ffma2_rn(x[c], b, a);                                  // FFMA2 3 regs
            if (kForm == 3) x[c] = __fmul2_rn(x[c], b);                                     // FMUL2
            if (kForm == 4) x[c] = make_float2(x[c].x + a.x, x[c].y + a.y);                 // 2x scalar FADD
            if (kForm == 5) x[c] = __ffma2_rn(x[c], make_float2(-1.0f, -1.0f), a);          // FFMA2 imm -1 (our sub2)
            if (kForm == 6) x[c] = __fadd2_rn(x[c], make_float2(3.0f, 3.0f));               // FADD2 imm
            if (kForm == 7) x[c] = (c & 1) ? __ffma2_rn(x[c], b, a) : __fadd2_rn(x[c], a);  // mix FFMA2/FADD2
            if (kForm == 8) { x[c].x = fmaf(x[c].x, 1.0001f, a.x); }                          // scalar FFMA imm
            if (kForm == 9) { x[c].x = fmaf(x[c].x, b.x, a.x); }                             // scalar FFMA 3-reg
            if (kForm == 10) { if (c & 1) x[c] = __ffma2_rn(x[c], b, a); else x[c].x = __int_as_float(__float_as_int(x[c].x) + 3); } // FFMA2 + IADD
        }
    }
    float2 s = make_float2(0, 0);
#pragma unroll
    for (int c = 0; c < kChains; ++c) s = __fadd2_rn(s, x[c]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    float2* out;
    cudaMalloc(&out, sizeof(float2) * 148 * 8 * 512);
    const char* names[] = {"FADD2 reg", "FFMA2 imm 1.0", "FFMA2 3-reg", "FMUL2 reg", "FADD (vectorised)",
                           "FFMA2 imm -1", "FADD2 imm", "FFMA2+FADD2 mix", "FFMA scalar imm", "FFMA scalar 3reg",
                           "FFMA2 + IADD mix"};
    void* fns[] = {(void*)bench<0>, (void*)bench<1>, (void*)bench<2>, (void*)bench<3>,
                   (void*)bench<4>, (void*)bench<5>, (void*)bench<6>, (void*)bench<7>,
                   (void*)bench<8>, (void*)bench<9>, (void*)bench<10>};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    for (int f = 0; f < 11; ++f) {
        float2 a = make_float2(1e-7f, 2e-7f), b = make_float2(1.0000001f, 0.9999999f);
        void* args[] = {&out, &a, &b};
        dim3 grid(148 * 8), block(512);
        cudaLaunchKernel(fns[f], grid, block, args, 0, 0);
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) cudaLaunchKernel(fns[f], grid, block, args, 0, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double warp_instr = 5.0 * grid.x * (block.x / 32) * double(kIters) * kChains;
        const double per_smsp_per_clk = warp_instr / (148 * 4) / (ms * 1e-3 * 1.965e9);
        printf("%-16s %8.3f ms  warp-instr/clk/SMSP = %.3f\n", names[f], ms, per_smsp_per_clk);
    }
    return 0;
}
