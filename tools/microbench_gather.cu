// Microbenchmark (not product code): trilinear evaluations per second on B200 with the
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_gather tools/microbench_gather.cu
// 32^3 grid (a) in shared memory, 8 corner LDS per evaluation (the dock kernel's path),
// (b) behind a texture object over pitch-linear memory, 2 tex2Dgather per evaluation
// (z0 and z1 planes of a 32 x (32*33) 2D texture), raw texels, same lerp arithmetic.
// Points: per lane an LCG walk inside the box (random gathers, the worst case for banks).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ float lerp(float a, float b, float t) { return __fmaf_rn(t, b, __fmaf_rn(-t, a, a)); }

__device__ __forceinline__ float3 next_point(unsigned& s) {
    s = s * 1664525u + 1013904223u;
    const float x = 2.f + 27.f * ((s >> 8) & 0xffff) / 65536.f;
    s = s * 1664525u + 1013904223u;
    const float y = 2.f + 27.f * ((s >> 8) & 0xffff) / 65536.f;
    s = s * 1664525u + 1013904223u;
    const float z = 2.f + 27.f * ((s >> 8) & 0xffff) / 65536.f;
    return make_float3(x, y, z);
}

template <int RS, int PS>
__global__ void __launch_bounds__(1024, 1) k_smem(const float* __restrict__ G, int iters, float* out) {
    extern __shared__ float sG[];
    for (int i = threadIdx.x; i < 33 * PS + RS + 2; i += blockDim.x) sG[i] = 0.f;
    __syncthreads();
    for (int i = threadIdx.x; i < 32 * 32 * 32; i += blockDim.x) {
        const int x = i & 31, y = (i >> 5) & 31, z = i >> 10;
        sG[z * PS + y * RS + x] = G[i];
    }
    __syncthreads();
    unsigned s = blockIdx.x * 1024 + threadIdx.x;
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
        const float3 u = next_point(s);
        const float fx = floorf(u.x), fy = floorf(u.y), fz = floorf(u.z);
        const float tx = u.x - fx, ty = u.y - fy, tz = u.z - fz;
        const float* p = sG + (int)fx + (int)fy * RS + (int)fz * PS;
        const float l00 = lerp(p[0], p[1], tx), l10 = lerp(p[RS], p[RS + 1], tx);
        const float l01 = lerp(p[PS], p[PS + 1], tx), l11 = lerp(p[PS + RS], p[PS + RS + 1], tx);
        acc += lerp(lerp(l00, l10, ty), lerp(l01, l11, ty), tz);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void __launch_bounds__(1024, 1) k_tex(cudaTextureObject_t tex, int iters, float* out) {
    unsigned s = blockIdx.x * 1024 + threadIdx.x;
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
        const float3 u = next_point(s);
        const float fx = floorf(u.x), fy = floorf(u.y), fz = floorf(u.z);
        const float tx = u.x - fx, ty = u.y - fy, tz = u.z - fz;
        // gather footprint of a bilinear sample at (fx + 1, row + 1): texels (fx, fx+1) x (row, row+1)
        const float4 a = tex2Dgather<float4>(tex, fx + 1.f, fz * 32.f + fy + 1.f, 0);
        const float4 b = tex2Dgather<float4>(tex, fx + 1.f, (fz + 1.f) * 32.f + fy + 1.f, 0);
        // gather order: x = (i0, j1), y = (i1, j1), z = (i1, j0), w = (i0, j0)
        const float l00 = lerp(a.w, a.z, tx), l10 = lerp(a.x, a.y, tx);
        const float l01 = lerp(b.w, b.z, tx), l11 = lerp(b.x, b.y, tx);
        acc += lerp(lerp(l00, l10, ty), lerp(l01, l11, ty), tz);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}


// (c) mixed: z0 plane from shared memory (4 LDS), z1 plane by one tex2Dgather
template <int RS, int PS>
__global__ void __launch_bounds__(1024, 1) k_mixed(const float* __restrict__ G, cudaTextureObject_t tex, int iters, float* out) {
    extern __shared__ float sG[];
    for (int i = threadIdx.x; i < 33 * PS + RS + 2; i += blockDim.x) sG[i] = 0.f;
    __syncthreads();
    for (int i = threadIdx.x; i < 32 * 32 * 32; i += blockDim.x) {
        const int x = i & 31, y = (i >> 5) & 31, z = i >> 10;
        sG[z * PS + y * RS + x] = G[i];
    }
    __syncthreads();
    unsigned s = blockIdx.x * 1024 + threadIdx.x;
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
        const float3 u = next_point(s);
        const float fx = floorf(u.x), fy = floorf(u.y), fz = floorf(u.z);
        const float tx = u.x - fx, ty = u.y - fy, tz = u.z - fz;
        const float* p = sG + (int)fx + (int)fy * RS + (int)fz * PS;
        const float l00 = lerp(p[0], p[1], tx), l10 = lerp(p[RS], p[RS + 1], tx);
        const float4 b = tex2Dgather<float4>(tex, fx + 1.f, (fz + 1.f) * 32.f + fy + 1.f, 0);
        const float l01 = lerp(b.w, b.z, tx), l11 = lerp(b.x, b.y, tx);
        acc += lerp(lerp(l00, l10, ty), lerp(l01, l11, ty), tz);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main(int argc, char** argv) {
    const int iters = argc > 1 ? atoi(argv[1]) : 4096;
    const int threads = argc > 2 ? atoi(argv[2]) : 512;
    const int n = 32 * 32 * 32;
    float* h = (float*)malloc(n * 4);
    for (int i = 0; i < n; ++i) h[i] = (float)((i * 2654435761u) % 1000) / 100.f;
    float *dG, *dT, *out;
    cudaMalloc(&dG, n * 4);
    cudaMemcpy(dG, h, n * 4, cudaMemcpyHostToDevice);
    // 2D texture 32 wide x 33*32 rows (one zero plane), pitch-linear
    size_t pitch = 128;
    cudaMalloc(&dT, 33 * 32 * pitch);
    cudaMemset(dT, 0, 33 * 32 * pitch);
    cudaMemcpy(dT, h, n * 4, cudaMemcpyHostToDevice);
    cudaResourceDesc rd = {};
    rd.resType = cudaResourceTypePitch2D;
    rd.res.pitch2D.devPtr = dT;
    rd.res.pitch2D.desc = cudaCreateChannelDesc<float>();
    rd.res.pitch2D.width = 32;
    rd.res.pitch2D.height = 33 * 32;
    rd.res.pitch2D.pitchInBytes = pitch;
    cudaTextureDesc td = {};
    td.addressMode[0] = td.addressMode[1] = cudaAddressModeClamp;
    td.filterMode = cudaFilterModePoint;
    td.readMode = cudaReadModeElementType;
    td.normalizedCoords = 0;
    cudaTextureObject_t tex;
    if (cudaCreateTextureObject(&tex, &rd, &td, nullptr) != cudaSuccess) { printf("tex create failed\n"); return 1; }
    cudaMalloc(&out, 148 * 1024 * 4);
    const int smem = (33 * 1063 + 40) * 4;
    cudaFuncSetAttribute(k_smem<33, 1063>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    double evals = 148.0 * threads * iters;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        k_smem<33, 1063><<<148, threads, smem>>>(dG, iters, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("smem  threads=%d: %.3f ms  %.1f Geval/s  (%s)\n", threads, ms, evals / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
        cudaEventRecord(e0);
        k_tex<<<148, threads>>>(tex, iters, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("tex   threads=%d: %.3f ms  %.1f Geval/s  (%s)\n", threads, ms, evals / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
        // texture with 2 CTAs/SM (more warps: no smem needed)
        cudaEventRecord(e0);
        k_tex<<<296, threads>>>(tex, iters, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("tex2x threads=%d: %.3f ms  %.1f Geval/s\n", threads, ms, 2 * evals / ms / 1e6);
        cudaFuncSetAttribute(k_mixed<33, 1063>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaEventRecord(e0);
        k_mixed<33, 1063><<<148, threads, smem>>>(dG, tex, iters, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("mixed threads=%d: %.3f ms  %.1f Geval/s  (%s)\n", threads, ms, evals / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
    // correctness: same points, same sums?
    return 0;
}
