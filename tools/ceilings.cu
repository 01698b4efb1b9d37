// ceilings.cu -- measured roofline denominators, loaded by bench.py (ctypes) and timed LIVE in
// every bench run (no hard-coded ceilings).  Measurement tooling, not product code.
//
//  l2_read_gbps(bytes, reps): read bandwidth of an L2-resident buffer (48 MB of the 126 MB L2),
//      16-byte ld.global.cg (L1 bypassed), every SM, after one warm-up pass; bytes / CUDA-event
//      time, best of 5.  BJ's "FP32/L2" roof = min(FP32 peak, 43/32 flop/B x this).
//  smem_gather_gevals(iters, threads): trilinear evaluations per second with the 8 corners
//      gathered from a 32^3 fp32 grid in SHARED memory (the dock kernel's (34, 1097) strides),
//      uniformly random points per lane (the worst case for banks), one CTA per SM.
#include <cuda_runtime.h>

namespace {

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
    if (acc.x + acc.y + acc.z + acc.w == 12345.f) out[0] = acc.x;
}

__device__ __forceinline__ float lerp(float a, float b, float t) { return __fmaf_rn(t, b, __fmaf_rn(-t, a, a)); }

constexpr int RS = 34, PS = 1097;

__global__ void __launch_bounds__(1024, 1) k_gather(const float* __restrict__ G, int iters, float* out) {
    extern __shared__ float sG[];
    for (int i = threadIdx.x; i < 33 * PS + RS + 2; i += blockDim.x) sG[i] = 0.f;
    __syncthreads();
    for (int i = threadIdx.x; i < 32 * 32 * 32; i += blockDim.x) sG[(i >> 10) * PS + ((i >> 5) & 31) * RS + (i & 31)] = G[i];
    __syncthreads();
    unsigned s = blockIdx.x * 1024 + threadIdx.x;
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
        float u[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            s = s * 1664525u + 1013904223u;
            u[a] = 1.f + 29.f * ((s >> 8) & 0xffff) / 65536.f;
        }
        const float fx = floorf(u[0]), fy = floorf(u[1]), fz = floorf(u[2]);
        const float tx = u[0] - fx, ty = u[1] - fy, tz = u[2] - fz;
        const float* p = sG + (int)fx + (int)fy * RS + (int)fz * PS;
        const float l00 = lerp(p[0], p[1], tx), l10 = lerp(p[RS], p[RS + 1], tx);
        const float l01 = lerp(p[PS], p[PS + 1], tx), l11 = lerp(p[PS + RS], p[PS + RS + 1], tx);
        acc += lerp(lerp(l00, l10, ty), lerp(l01, l11, ty), tz);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

}  // namespace

extern "C" double l2_read_gbps(size_t bytes, int reps) {
    const size_t n4 = bytes / 16;
    float4* buf = nullptr;
    float* out = nullptr;
    if (cudaMalloc(&buf, bytes) != cudaSuccess || cudaMalloc(&out, 4) != cudaSuccess) return -1.0;
    cudaMemset(buf, 0, bytes);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double best = 0.0;
    for (int bps : {2, 4}) {
        k_l2<<<sms * bps, 1024>>>(buf, n4, 1, out);   // warm-up: L2-resident
        for (int t = 0; t < 5; ++t) {
            cudaEventRecord(e0);
            k_l2<<<sms * bps, 1024>>>(buf, n4, reps, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0, e1);
            const double g = (double)bytes * reps / (ms * 1e-3) / 1e9;
            if (g > best) best = g;
        }
    }
    const bool ok = cudaGetLastError() == cudaSuccess;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(buf);
    cudaFree(out);
    return ok ? best : -1.0;
}

extern "C" double smem_gather_gevals(int iters, int threads) {
    const int n = 32 * 32 * 32;
    float *dG = nullptr, *out = nullptr;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    if (cudaMalloc(&dG, n * 4) != cudaSuccess || cudaMalloc(&out, (size_t)sms * 1024 * 4) != cudaSuccess) return -1.0;
    cudaMemset(dG, 0, n * 4);
    const int smem = (33 * PS + RS + 2) * 4;
    cudaFuncSetAttribute(k_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double best = 0.0;
    for (int t = 0; t < 3; ++t) {
        cudaEventRecord(e0);
        k_gather<<<sms, threads, smem>>>(dG, iters, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        const double g = (double)sms * threads * iters / (ms * 1e-3) / 1e9;
        if (g > best) best = g;
    }
    const bool ok = cudaGetLastError() == cudaSuccess;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(dG);
    cudaFree(out);
    return ok ? best : -1.0;
}
