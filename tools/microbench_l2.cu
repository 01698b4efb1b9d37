// Microbenchmark (not product code): L2 read bandwidth of this B200, for the "FP32/L2"
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_l2 tools/microbench_l2.cu
// roofline of BASELINE.json (achieved / min(FP32, AI x BW_L2)).
// A 48 MB buffer (L2 is 126 MB) is read repeatedly by every SM with 16-byte ld.global.cg
// (L1 bypassed), after one warm-up pass that makes it L2-resident; bytes / CUDA-event time.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(1024) k_l2(const float4* __restrict__ buf, size_t n4, int reps, float* out) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int r = 0; r < reps; ++r) {
        for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
            float4 v;
            asm volatile("ld.global.cg.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                         : "l"(buf + i));
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
    }
    if (acc.x + acc.y + acc.z + acc.w == 12345.f) out[0] = acc.x;   // keep the loads alive
}

int main(int argc, char** argv) {
    const size_t bytes = (argc > 1 ? atol(argv[1]) : 48) << 20;
    const int reps = argc > 2 ? atoi(argv[2]) : 20;
    const size_t n4 = bytes / 16;
    float4* buf;
    float* out;
    cudaMalloc(&buf, bytes);
    cudaMalloc(&out, 4);
    cudaMemset(buf, 0, bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int blocks_per_sm : {2, 4}) {
        const int grid = 148 * blocks_per_sm;
        k_l2<<<grid, 1024>>>(buf, n4, 1, out);   // warm-up: L2-resident
        float best = 1e30f;
        for (int t = 0; t < 5; ++t) {
            cudaEventRecord(e0);
            k_l2<<<grid, 1024>>>(buf, n4, reps, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
        }
        printf("L2 read: %zu MB x %d reps, %d CTAs x 1024: %.3f ms  %.1f GB/s (%s)\n", bytes >> 20, reps, grid, best,
               (double)bytes * reps / best / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
