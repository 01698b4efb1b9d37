// Microbenchmark (not product code): cost of one trilinear gather from shared memory with
// uniformly random points (hashed per lane and iteration, no lane correlation) for three
// layouts of the grid:
//   0  scalar fp32 nodes, strides (rs, ps) = (34, 1097)   -> 8 LDS.32 per evaluation
//   1  x-pairs: node (x, y, z) holds (G[x], G[x+1])        -> 4 LDS.64
//   2  xz-quads: node holds (G[x], G[x+1], G[x,z+1], G[x+1,z+1]) -> 2 LDS.128
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o tools/microbench_pairs tools/microbench_pairs.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ float lerp(float a, float b, float t) { return __fmaf_rn(t, b, __fmaf_rn(-t, a, a)); }

__device__ __forceinline__ unsigned hash32(unsigned x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}

// E = edge (cells in [0, E-1) per axis); RS / PS strides in ELEMENTS of the layout's type
template <int MODE, int E, int RS, int PS>
__global__ void __launch_bounds__(512, 1) k_gather(int iters, float* out) {
    extern __shared__ __align__(16) float sm[];
    const int nfl = (MODE == 0 ? 1 : MODE == 1 ? 2 : 4) * (PS * E + RS + 2);
    for (int i = threadIdx.x; i < nfl; i += blockDim.x) sm[i] = (float)(i % 97) * 0.01f;
    __syncthreads();
    const unsigned seed = (blockIdx.x * 512 + threadIdx.x) * 0x9E3779B9u;
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
        const unsigned h = hash32(seed ^ (unsigned)it * 0x85ebca6bu);
        const int x = (h & 1023) % (E - 1), y = ((h >> 10) & 1023) % (E - 1), z = ((h >> 20) & 1023) % (E - 1);
        const float tx = 0.3f, ty = 0.6f, tz = 0.2f;
        if (MODE == 0) {
            const float* p = sm + x + y * RS + z * PS;
            const float l00 = lerp(p[0], p[1], tx), l10 = lerp(p[RS], p[RS + 1], tx);
            const float l01 = lerp(p[PS], p[PS + 1], tx), l11 = lerp(p[PS + RS], p[PS + RS + 1], tx);
            acc += lerp(lerp(l00, l10, ty), lerp(l01, l11, ty), tz);
        } else if (MODE == 1) {
            const float2* p = reinterpret_cast<const float2*>(sm) + x + y * RS + z * PS;
            const float2 a = p[0], b = p[RS], c = p[PS], d = p[PS + RS];
            const float l00 = lerp(a.x, a.y, tx), l10 = lerp(b.x, b.y, tx);
            const float l01 = lerp(c.x, c.y, tx), l11 = lerp(d.x, d.y, tx);
            acc += lerp(lerp(l00, l10, ty), lerp(l01, l11, ty), tz);
        } else {
            const float4* p = reinterpret_cast<const float4*>(sm) + x + y * RS + z * PS;
            const float4 a = p[0], b = p[RS];
            const float l00 = lerp(a.x, a.y, tx), l10 = lerp(b.x, b.y, tx);
            const float l01 = lerp(a.z, a.w, tx), l11 = lerp(b.z, b.w, tx);
            acc += lerp(lerp(l00, l10, ty), lerp(l01, l11, ty), tz);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int MODE, int E, int RS, int PS>
void run(const char* name, int iters, float* out) {
    const int smem = (MODE == 0 ? 1 : MODE == 1 ? 2 : 4) * (PS * E + RS + 2) * 4;
    cudaFuncSetAttribute(k_gather<MODE, E, RS, PS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        k_gather<MODE, E, RS, PS><<<148, 512, smem>>>(iters, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    const double evals = 148.0 * 512 * iters;
    printf("%-28s smem=%6d B  %.3f ms  %.1f Geval/s  (%s)\n", name, smem, best, evals / best / 1e6,
           cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char** argv) {
    const int iters = argc > 1 ? atoi(argv[1]) : 8192;
    float* out;
    cudaMalloc(&out, 148 * 512 * 4);
    run<0, 32, 34, 1097>("scalar 32^3 (34,1097)", iters, out);
    run<0, 32, 32, 1024>("scalar 32^3 unpadded", iters, out);
    run<1, 24, 25, 601>("xpair 24^3 (25,601)", iters, out);
    run<1, 24, 24, 576>("xpair 24^3 unpadded", iters, out);
    run<1, 25, 26, 651>("xpair 25^3 (26,651)", iters, out);
    run<1, 24, 24, 580>("xpair 24^3 (24,580)", iters, out);
    run<2, 18, 19, 343>("xzquad 18^3 (19,343)", iters, out);
    run<2, 18, 18, 324>("xzquad 18^3 unpadded", iters, out);
    return 0;
}
