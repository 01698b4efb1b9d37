// topk.cu -- per-pocket ranking (a10) and the global merge (a11): the k
// smallest 64-bit keys (ord(score) << 32 | ligand index) by MSD radix select
// (8 passes of 8-bit digits; real keys are unique because the index is in the low
// word, so the k-th key is an exact threshold), compaction of the keys < T (padded
// lists may repeat UINT64_MAX: the threshold fills the remaining slots),
// and a bitonic sort of the k survivors in one CTA's shared memory.
//
// "for each docking site, we can rank the input chemical library" (PAPER.md
// l.174); ties of equal scores go to the lower ligand index (Q11) because the
// index is the low word of the key.
#include <cuda_runtime.h>
#include <cstdint>

#include "internal.h"

namespace vsd {

namespace {

typedef unsigned long long u64;

struct SelState {
    u64 prefix, mask;
    unsigned krem, count;
    unsigned hist[256];
};

__global__ void sel_init_kernel(SelState* st, unsigned k) {
    const int t = threadIdx.x;
    if (t == 0) {
        st->prefix = 0;
        st->mask = 0;
        st->krem = k;
        st->count = 0;
    }
    if (t < 256) st->hist[t] = 0;
}

__global__ void __launch_bounds__(512) sel_hist_kernel(const u64* __restrict__ keys, int64_t n, int shift,
                                                       SelState* st) {
    __shared__ unsigned h[256];
    for (int t = threadIdx.x; t < 256; t += blockDim.x) h[t] = 0;
    __syncthreads();
    const u64 prefix = st->prefix, mask = st->mask;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const u64 k = keys[i];
        if ((k & mask) == prefix) atomicAdd(&h[(k >> shift) & 255u], 1u);
    }
    __syncthreads();
    for (int t = threadIdx.x; t < 256; t += blockDim.x)
        if (h[t]) atomicAdd(&st->hist[t], h[t]);
}

__global__ void sel_pick_kernel(SelState* st, int shift) {
    __shared__ unsigned cum[256];
    const int t = threadIdx.x;
    const unsigned h = st->hist[t];
    cum[t] = h;
    __syncthreads();
    for (int o = 1; o < 256; o <<= 1) {  // inclusive scan
        const unsigned v = t >= o ? cum[t - o] : 0u;
        __syncthreads();
        cum[t] += v;
        __syncthreads();
    }
    const unsigned excl = cum[t] - h;
    const unsigned krem = st->krem;
    __syncthreads();
    if (h > 0 && excl < krem && krem <= excl + h) {
        st->prefix |= (u64)t << shift;
        st->mask |= (u64)0xFF << shift;
        st->krem = krem - excl;
    }
    st->hist[t] = 0;
}

// Compaction of the keys strictly below the threshold T (the k-th smallest key): at most
// k - 1 of them.  Keys equal to T are NOT written here: real keys are unique, but padded
// lists (UINT64_MAX entries of ranks with fewer than k ligands) repeat the pad value, so the
// bitonic kernel fills out[count .. k) with T instead -- deterministic, and never more than
// k entries whatever the number of duplicates.
__global__ void sel_compact_kernel(const u64* __restrict__ keys, int64_t n, SelState* st, u64* __restrict__ out) {
    const u64 T = st->prefix;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const u64 k = keys[i];
        if (k < T) out[atomicAdd(&st->count, 1u)] = k;
    }
}

__global__ void copy_keys_kernel(const u64* __restrict__ keys, int64_t n, u64* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = keys[i];
}

// bitonic sort of out[0..n) (n <= k), padded to a power of two with UINT64_MAX; writes out[0..k).
// st != null (selection mode): n = st->count keys below the threshold, and the k - n slots
// after them hold the threshold key itself (see sel_compact_kernel).
__global__ void __launch_bounds__(1024) bitonic_kernel(u64* __restrict__ out, int n, int k, int n2,
                                                       const SelState* __restrict__ st) {
    extern __shared__ u64 s[];
    if (st) n = (int)st->count;
    const u64 fill = st ? st->prefix : ~0ull;
    for (int i = threadIdx.x; i < n2; i += blockDim.x) s[i] = i < n ? out[i] : (i < k ? fill : ~0ull);
    __syncthreads();
    for (int size = 2; size <= n2; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < n2; i += blockDim.x) {
                const int j = i ^ stride;
                if (j > i) {
                    const bool up = (i & size) == 0;
                    const u64 a = s[i], b = s[j];
                    if ((a > b) == up) {
                        s[i] = b;
                        s[j] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < k; i += blockDim.x) out[i] = s[i];
}

// ligand ids of the merged top-k: out[i] = ids[index of key i] (ids == null: the index itself);
// UINT64_MAX for pads and for indices outside the id table.
__global__ void gather_ids_kernel(const u64* __restrict__ keys, int m, const unsigned long long* __restrict__ ids,
                                  int64_t n_ids, unsigned long long* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const u64 k = keys[i];
    const int64_t idx = (int64_t)(k & 0xffffffffull);
    out[i] = (k == ~0ull || idx >= n_ids) ? ~0ull : (ids ? ids[idx] : (unsigned long long)idx);
}

}  // namespace

cudaError_t launch_gather_ids(const unsigned long long* keys, int m, const unsigned long long* ids, int64_t n_ids,
                              unsigned long long* out, cudaStream_t st) {
    if (m <= 0) return cudaSuccess;
    gather_ids_kernel<<<(m + 255) / 256, 256, 0, st>>>(keys, m, ids, n_ids, out);
    return cudaGetLastError();
}

cudaError_t topk_select_sort(const unsigned long long* keys, int64_t n, int k, unsigned long long* out,
                             void* scratch, cudaStream_t st, int* launches) {
    if (k <= 0 || k > 8192) return cudaErrorInvalidValue;
    int n2 = 1;
    while (n2 < k) n2 <<= 1;
    const size_t smem = (size_t)n2 * 8;
    cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(bitonic_kernel),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int L = 0;
    int grid = (int)((n + 511) / 512);
    if (grid > 148 * 4) grid = 148 * 4;
    if (grid < 1) grid = 1;
    int m;  // survivors
    const SelState* sel = nullptr;
    if (n <= k) {
        if (n > 0) {
            copy_keys_kernel<<<grid, 512, 0, st>>>(keys, n, out);
            ++L;
        }
        m = (int)n;
    } else {
        SelState* s = reinterpret_cast<SelState*>(scratch);
        sel_init_kernel<<<1, 256, 0, st>>>(s, (unsigned)k);
        ++L;
        for (int shift = 56; shift >= 0; shift -= 8) {
            sel_hist_kernel<<<grid, 512, 0, st>>>(keys, n, shift, s);
            sel_pick_kernel<<<1, 256, 0, st>>>(s, shift);
            L += 2;
        }
        sel_compact_kernel<<<grid, 512, 0, st>>>(keys, n, s, out);
        ++L;
        m = k;
        sel = s;
    }
    bitonic_kernel<<<1, 1024, smem, st>>>(out, m, k, n2, sel);
    ++L;
    if (launches) *launches = L;
    return cudaGetLastError();
}

}  // namespace vsd
