// dock.cu -- the docking kernel (a6-a9): rigid roto-translation from P initial
// poses, greedy rotatable-bond sweep over K discrete angle steps, trilinear
// pocket-grid score, best-pose reduction.  fp32 on CUDA cores (not a dense
// contraction, BJ: "no tensor cores").
//
// B200 design:
//  * one CTA per SM, persistent over a launch's ligands with a dynamic round
//    counter; the pocket grid (32^3 fp32 = 128 KB, padded strides) lives in
//    SHARED memory for the whole launch -- the 8 corner gathers of every
//    evaluation are shared-memory loads, never L1/L2;
//  * a CTA docks LC ligands at a time; its NW warps split the ligand's poses,
//    PPW poses per warp (lane groups of 32/PPW), so all warps of a CTA run the
//    same control flow (same A, R, M_r: poses of one ligand differ only in data);
//  * sweep lane map inside a pose group: li = jl * K + k -- (moving atom jl of
//    the pass, angle k).  Each lane holds its angle's rotation in registers,
//    lanes of equal k sum with xor shuffles, the argmin over k takes log2 K
//    shuffle rounds (ties -> lowest k, Q11), and the winner is applied;
//  * (x, y) arithmetic is packed in Blackwell's FFMA2/FADD2 (per-element IEEE
//    fma/add, so every result is bit-identical to the scalar form);
//  * template<int AC, int NW, int PPW> per atom class = the paper's "non-type
//    template parameter for the kernel maximum number of atoms":
//    AC sizes the per-pose buffers in shared memory, hence the occupancy.
//
// All arithmetic that decides an angle or is replayed (placement, Rodrigues,
// rotation, interpolation) uses explicit _rn intrinsics in shared helpers, so
// the finalize kernel reproduces the trajectory bit for bit.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "internal.h"

namespace vsd {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr float kMagic = 8388608.f;              // 2^23: floor via round-down add
constexpr int kMagicBits = 0x4B000000;

__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 neg2(float2 a) { return make_float2(-a.x, -a.y); }

// Rotation about a pivot in "M v + t" form: p = M v + t with t = q - M q.
// Rows 0 and 1 are packed column-wise: c0 = (m00, m10), c1 = (m01, m11), c2 = (m02, m12).
struct RotT {
    float2 c0, c1, c2, txy;
    float m20, m21, m22, tz;
};

// M = c I + s [u]x + (1 - c) u u^T (a7; Q3, Q6), pivot q = y_b.  For (c, s) = (1, 0)
// this is exactly I and t = 0, so the identity candidate leaves coordinates bit-unchanged.
__device__ __forceinline__ RotT rodrigues_t(float ux, float uy, float uz, float c, float s, float qx, float qy,
                                            float qz) {
    const float omc = __fsub_rn(1.f, c);
    const float a = __fmul_rn(omc, ux), b = __fmul_rn(omc, uy), d = __fmul_rn(omc, uz);
    const float sx = __fmul_rn(s, ux), sy = __fmul_rn(s, uy), sz = __fmul_rn(s, uz);
    RotT M;
    const float m00 = __fmaf_rn(a, ux, c), m01 = __fmaf_rn(a, uy, -sz), m02 = __fmaf_rn(a, uz, sy);
    const float m10 = __fmaf_rn(b, ux, sz), m11 = __fmaf_rn(b, uy, c), m12 = __fmaf_rn(b, uz, -sx);
    M.m20 = __fmaf_rn(d, ux, -sy);
    M.m21 = __fmaf_rn(d, uy, sx);
    M.m22 = __fmaf_rn(d, uz, c);
    M.c0 = make_float2(m00, m10);
    M.c1 = make_float2(m01, m11);
    M.c2 = make_float2(m02, m12);
    // t = q - M q
    M.txy = make_float2(__fmaf_rn(-m00, qx, __fmaf_rn(-m01, qy, __fmaf_rn(-m02, qz, qx))),
                        __fmaf_rn(-m10, qx, __fmaf_rn(-m11, qy, __fmaf_rn(-m12, qz, qy))));
    M.tz = __fmaf_rn(-M.m20, qx, __fmaf_rn(-M.m21, qy, __fmaf_rn(-M.m22, qz, qz)));
    return M;
}

// p = M v + t; (x, y) in one FFMA2 chain, z scalar
__device__ __forceinline__ float4 apply_rot(const RotT& M, float vx, float vy, float vz) {
    const float2 pxy = __ffma2_rn(M.c0, f2(vx), __ffma2_rn(M.c1, f2(vy), __ffma2_rn(M.c2, f2(vz), M.txy)));
    const float pz = __fmaf_rn(M.m20, vx, __fmaf_rn(M.m21, vy, __fmaf_rn(M.m22, vz, M.tz)));
    return make_float4(pxy.x, pxy.y, pz, 0.f);
}

// unit axis a -> b
__device__ __forceinline__ void axis_of(const float4& ya, const float4& yb, float& ux, float& uy, float& uz) {
    const float dx = __fsub_rn(yb.x, ya.x), dy = __fsub_rn(yb.y, ya.y), dz = __fsub_rn(yb.z, ya.z);
    const float n2 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
    const float inv = rsqrtf(n2);
    ux = __fmul_rn(dx, inv);
    uy = __fmul_rn(dy, inv);
    uz = __fmul_rn(dz, inv);
}

__device__ __forceinline__ float lerp(float a, float b, float t) { return __fmaf_rn(t, b, __fmaf_rn(-t, a, a)); }
__device__ __forceinline__ float2 lerp2(float2 a, float2 b, float t) {
    return __ffma2_rn(f2(t), b, __ffma2_rn(f2(-t), a, a));
}

// a8: g(u), u in grid units (Q9, Q10): clamp, L1 excess, i0 = min(floor(u_c), n-2),
// lerps x then y then z, + kappa*h*excess.  G is the shared-memory copy (strides rs, ps).
// floor(m) for 0 <= m < 2^23 is the round-down sum m + 2^23 (its bits also give the
// integer); identical values to floorf.  The x-lerps run on (z0, z1) pairs, the
// y-lerp on the (l0, l1) pair: per element the same fma sequence as the scalar form.
//
// The upper edge (u_c = n-1) takes i0 = n-1 with f = 0 instead of i0 = n-2 with f = 1:
// both reduce exactly to the node value (lerp(a, b, 0) = a, lerp(a, b, 1) = b bitwise),
// and the corner at n is a finite zero pad of the shared-memory copy, so no clamp of
// i0 is needed.  FIX: the 32x32-plane layout with compile-time strides (33, 1063)
// that lets every corner load use an immediate offset.
constexpr int kFixRS = 33, kFixPS = 1063;
template <bool FIX>
__device__ __forceinline__ float grid_g(const float* __restrict__ G, float ux, float uy, float uz, const PocketDev& pk) {
    const int RS = FIX ? kFixRS : pk.rs, PS = FIX ? kFixPS : pk.ps;
    const float cx = fminf(fmaxf(ux, 0.f), pk.top_x);
    const float cy = fminf(fmaxf(uy, 0.f), pk.top_y);
    const float cz = fminf(fmaxf(uz, 0.f), pk.top_z);
    const float2 dxy = __fadd2_rn(make_float2(ux, uy), make_float2(-cx, -cy));
    const float e = __fadd_rn(__fadd_rn(fabsf(dxy.x), fabsf(dxy.y)), fabsf(__fsub_rn(uz, cz)));
    const float2 bxy = __fadd2_rd(make_float2(cx, cy), f2(kMagic));
    const float bz = __fadd_rd(cz, kMagic);
    const float2 fxy = __fadd2_rn(make_float2(cx, cy), neg2(__fadd2_rn(bxy, f2(-kMagic))));
    const float fz = __fsub_rn(cz, __fsub_rn(bz, kMagic));
    const int idx = (__float_as_int(bxy.x) - kMagicBits) + (__float_as_int(bxy.y) - kMagicBits) * RS +
                    (__float_as_int(bz) - kMagicBits) * PS;
    const float* p = G + idx;
    const float2 c00 = make_float2(p[0], p[PS]);                 // (c000, c001)
    const float2 c10 = make_float2(p[1], p[PS + 1]);             // (c100, c101)
    const float2 c01 = make_float2(p[RS], p[PS + RS]);           // (c010, c011)
    const float2 c11 = make_float2(p[RS + 1], p[PS + RS + 1]);   // (c110, c111)
    const float2 l_0 = lerp2(c00, c10, fxy.x);     // (l00, l01): y0, z0/z1
    const float2 l_1 = lerp2(c01, c11, fxy.x);     // (l10, l11): y1, z0/z1
    const float2 l = lerp2(l_0, l_1, fxy.y);       // (l0, l1)
    return __fmaf_rn(pk.kh, e, lerp(l.x, l.y, fz));
}

// Pose p in grid units: R' = R / h, t' = (c + tau - o) / h, u = R' x + t'.
// Stored as 12 floats: (R'00, R'10), (R'01, R'11), (R'02, R'12), (t'x, t'y), R'20, R'21, R'22, t'z.
__device__ __forceinline__ void scaled_pose(const float* raw, const PocketDev& pk, float* out) {
    float r[9];
#pragma unroll
    for (int t = 0; t < 9; ++t) r[t] = __fmul_rn(raw[t], pk.inv_h);
    out[0] = r[0]; out[1] = r[3];
    out[2] = r[1]; out[3] = r[4];
    out[4] = r[2]; out[5] = r[5];
    out[6] = __fadd_rn(pk.tx, __fmul_rn(raw[9], pk.inv_h));
    out[7] = __fadd_rn(pk.ty, __fmul_rn(raw[10], pk.inv_h));
    out[8] = r[6]; out[9] = r[7]; out[10] = r[8];
    out[11] = __fadd_rn(pk.tz, __fmul_rn(raw[11], pk.inv_h));
}

__device__ __forceinline__ RotT load_pose(const float* T) {
    RotT M;
    M.c0 = make_float2(T[0], T[1]);
    M.c1 = make_float2(T[2], T[3]);
    M.c2 = make_float2(T[4], T[5]);
    M.txy = make_float2(T[6], T[7]);
    M.m20 = T[8]; M.m21 = T[9]; M.m22 = T[10]; M.tz = T[11];
    return M;
}

// Stage the pocket grid into shared memory with padded strides; the padding (and
// the zero plane/row above the grid) is zero-filled first.  Ends with a barrier.
__device__ __forceinline__ void stage_grid(float* sG, const PocketDev& pk) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int n4 = (int)(align16(((size_t)(pk.nz + 1) * pk.ps + pk.rs + 2) * 4) / 16);
    for (int t = threadIdx.x; t < n4; t += blockDim.x) reinterpret_cast<float4*>(sG)[t] = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncthreads();
    for (int row = w; row < pk.ny * pk.nz; row += nw) {
        const int z = row / pk.ny, y = row - z * pk.ny;
        const float* src = pk.grid + (size_t)row * pk.nx;
        float* dst = sG + z * pk.ps + y * pk.rs;
        for (int x = lane; x < pk.nx; x += 32) dst[x] = src[x];
    }
}

// Order-preserving map of fp32 onto uint32 (-0 canonicalised to +0 first).
__device__ __forceinline__ unsigned ord32(float v) {
    const unsigned b = __float_as_uint(__fadd_rn(v, 0.0f));
    return b ^ ((unsigned)((int)b >> 31) | 0x80000000u);
}

// Per-pose buffer stride in float4: AC + 1 so that the PPW pose groups of a warp
// read their buffers from different banks.
// Per-pose coordinate buffer in shared memory, SoA: x[AC] | y[AC] | z[AC] (12 B per atom),
// pose buffers 3*AC + 4 floats apart so the PPW pose groups of a warp hit different banks.
template <int AC>
__host__ __device__ constexpr int pose_stride() { return 3 * AC + 4; }
template <int AC>
struct PoseBuf {
    float* b;
    __device__ __forceinline__ float4 get(int j) const { return make_float4(b[j], b[AC + j], b[2 * AC + j], 0.f); }
    __device__ __forceinline__ void set(int j, float4 v) const {
        b[j] = v.x;
        b[AC + j] = v.y;
        b[2 * AC + j] = v.z;
    }
};

// PPW poses of one ligand on one warp: lanes [h*LPP, (h+1)*LPP) serve pose h.
// a6 placement, a7 sweep, a9 pose score.
template <int AC, int PPW, bool FIX>
__device__ __forceinline__ void dock_poses(const float* __restrict__ rec, int A, int R, const float* __restrict__ T,
                                           bool valid, PoseBuf<AC> B, const float* __restrict__ G,
                                           const PocketDev& pk, int K, int kbits, int S_w, float ck, float sk,
                                           const float* __restrict__ sCS, uint8_t* __restrict__ angOut,
                                           float* __restrict__ scoreOut, int lane) {
    constexpr int LPP = 32 / PPW;
    const int li = lane & (LPP - 1);
    const float* rx = rec;
    const float* ry = rec + AC;
    const float* rz = rec + 2 * AC;
    const uint32_t* rfr = reinterpret_cast<const uint32_t*>(rec + 3 * AC);
    {
        const RotT Pz = load_pose(T);
        if (valid)
            for (int i = li; i < A; i += LPP) B.set(i, apply_rot(Pz, rx[i], ry[i], rz[i]));
    }
    __syncwarp();
    if (K > 1) {
        const int k = li & (K - 1);
        const int jl = li >> kbits;
        const int apw = LPP >> kbits;
        const unsigned gmask = ((K == 32) ? 0xffffffffu : ((1u << K) - 1u)) << (lane & ~(K - 1));
        for (int sw = 0; sw < S_w; ++sw) {
            for (int r = 0; r < R; ++r) {
                const uint32_t f = rfr[r];
                const int fa = f & 255, fb = (f >> 8) & 255, lo = (f >> 16) & 255, hi = (int)(f >> 24) + 1;
                const float4 ya = B.get(fa), yb = B.get(fb);
                float ux, uy, uz;
                axis_of(ya, yb, ux, uy, uz);
                const RotT M = rodrigues_t(ux, uy, uz, ck, sk, yb.x, yb.y, yb.z);
                float acc = 0.f;
                float4 keep = make_float4(0.f, 0.f, 0.f, 0.f);
                int base = lo;
                if (PPW == 4) {   // four independent evaluations in flight per lane (passes of apw atoms)
                    for (; base + 3 * apw < hi; base += 4 * apw) {
                        float4 v[4], q[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int j = base + u * apw + jl;
                            v[u] = B.get(j < hi ? j : base + jl);
                        }
#pragma unroll
                        for (int u = 0; u < 4; ++u) q[u] = apply_rot(M, v[u].x, v[u].y, v[u].z);
                        float g[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) g[u] = grid_g<FIX>(G, q[u].x, q[u].y, q[u].z, pk);
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            if (base + u * apw + jl < hi) acc = __fadd_rn(acc, g[u]);
                    }
                }
                for (; base + apw < hi; base += 2 * apw) {     // two independent evaluations per lane
                    const int j0 = base + jl, j1 = base + apw + jl;
                    const float4 v0 = B.get(j0);
                    const float4 v1 = B.get(j1 < hi ? j1 : j0);
                    const float4 p0 = apply_rot(M, v0.x, v0.y, v0.z);
                    const float4 p1 = apply_rot(M, v1.x, v1.y, v1.z);
                    const float g0 = grid_g<FIX>(G, p0.x, p0.y, p0.z, pk);
                    const float g1 = grid_g<FIX>(G, p1.x, p1.y, p1.z, pk);
                    acc = __fadd_rn(acc, g0);
                    if (j1 < hi) acc = __fadd_rn(acc, g1);
                }
                if (base < hi) {
                    const int j = base + jl;
                    if (j < hi) {
                        const float4 v = B.get(j);
                        keep = apply_rot(M, v.x, v.y, v.z);
                        acc = __fadd_rn(acc, grid_g<FIX>(G, keep.x, keep.y, keep.z, pk));
                    }
                }
                // sum over the pass atoms (lanes of equal k: xor offsets K .. LPP/2, ascending)
#pragma unroll
                for (int o = 1; o < LPP; o <<= 1)
                    if (o >= K) acc = __fadd_rn(acc, __shfl_xor_sync(FULL, acc, o));
                // argmin over the K angles of this group (xor offsets 1 .. K/2); ties -> lowest k (Q11)
                const unsigned key = ord32(acc);
                unsigned mn = key;
#pragma unroll
                for (int o = 1; o < LPP; o <<= 1)
                    if (o < K) mn = min(mn, __shfl_xor_sync(FULL, mn, o));
                const unsigned bal = __ballot_sync(FULL, key == mn) & gmask;
                const int bk = (__ffs(bal) - 1) & (K - 1);
                if (hi - lo <= apw) {
                    // single pass: the lane (jl, k*) already holds the rotated atom
                    if (valid && bk != 0 && k == bk && lo + jl < hi) B.set(lo + jl, keep);
                } else if (valid && bk != 0) {
                    const RotT Ms = rodrigues_t(ux, uy, uz, sCS[2 * bk], sCS[2 * bk + 1], yb.x, yb.y, yb.z);
                    for (int j = lo + li; j < hi; j += LPP) {
                        const float4 v = B.get(j);
                        B.set(j, apply_rot(Ms, v.x, v.y, v.z));
                    }
                }
                __syncwarp();
                if (valid && li == 0) angOut[sw * R + r] = (uint8_t)bk;
            }
        }
    } else if (valid) {
        for (int t = li; t < S_w * R; t += LPP) angOut[t] = 0;
    }
    // a9: pose score, canonical order (atom i -> lane i mod LPP, ascending, xor tree) (Q22)
    float acc = 0.f;
    for (int i = li; i < A; i += LPP) {
        const float4 v = B.get(i);
        acc = __fadd_rn(acc, grid_g<FIX>(G, v.x, v.y, v.z, pk));
    }
#pragma unroll
    for (int o = LPP / 2; o > 0; o >>= 1) acc = __fadd_rn(acc, __shfl_xor_sync(FULL, acc, o));
    if (valid && li == 0) *scoreOut = acc;
    __syncwarp();
}

template <int AC, int NW, int PPW, bool FIX>
__global__ void __launch_bounds__(NW * 32, 1) dock_kernel(const DockArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_round;
    constexpr int LPP = 32 / PPW;
    const PocketDev& pk = a.pk;
    const int LC = a.ligs_per_cta;
    const DockLayout L = dock_layout(AC, NW, PPW, pk.nz, pk.rs, pk.ps, a.P, a.K, a.S_w, LC);
    float* sG = reinterpret_cast<float*>(smem + L.grid);
    float* sPose = reinterpret_cast<float*>(smem + L.pose);
    float* sCS = reinterpret_cast<float*>(smem + L.cs);
    float* sRec = reinterpret_cast<float*>(smem + L.rec);
    float* sBuf = reinterpret_cast<float*>(smem + L.buf);
    float* sScore = reinterpret_cast<float*>(smem + L.score);
    uint8_t* sAng = smem + L.ang;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, h = lane / LPP;

    stage_grid(sG, pk);
    for (int p = tid; p < a.P; p += blockDim.x) scaled_pose(a.pose_tab + 12 * p, pk, sPose + 12 * p);
    for (int t = tid; t < 2 * a.K; t += blockDim.x) sCS[t] = a.cs[t];
    __syncthreads();

    const int K = a.K, S_w = a.S_w, P = a.P;
    const int kbits = 31 - __clz(K);
    const float ck = sCS[2 * (lane & (K - 1))], sk = sCS[2 * (lane & (K - 1)) + 1];
    const PoseBuf<AC> buf{sBuf + (warp * PPW + h) * pose_stride<AC>()};
    const int rec_floats = a.rec_floats;
    const int n_rounds = (a.n + LC - 1) / LC;
    const int ang_stride = 32 * S_w;
    const int G = (P + PPW - 1) / PPW;   // warp items per ligand

    while (true) {
        if (tid == 0) s_round = atomicAdd(a.counter, 1);   // dynamic: balance CTAs within the launch
        __syncthreads();
        const int round = s_round;
        if (round >= n_rounds) break;
        const int slot0 = round * LC;
        const int nl = min(LC, a.n - slot0);
        {
            const float4* src = reinterpret_cast<const float4*>(a.rec + (size_t)slot0 * rec_floats);
            float4* dst = reinterpret_cast<float4*>(sRec);
            const int n4 = nl * rec_floats / 4;
            for (int t = tid; t < n4; t += blockDim.x) dst[t] = src[t];
        }
        __syncthreads();
        for (int item = warp; item < nl * G; item += NW) {
            const int l = item / G, g = item - l * G;
            const int p = g * PPW + h;
            const bool valid = p < P;
            const int pc = valid ? p : P - 1;
            const int4 m = a.meta[slot0 + l];
            dock_poses<AC, PPW, FIX>(sRec + l * rec_floats, m.y, m.z, sPose + 12 * pc, valid, buf, sG, pk, K, kbits, S_w,
                                ck, sk, sCS, sAng + (size_t)(l * P + pc) * ang_stride, sScore + l * P + pc, lane);
        }
        __syncthreads();
        if (warp < nl) {  // a9 best pose: lowest score, ties -> lowest pose index (Q11)
            const int l = warp;
            const int4 m = a.meta[slot0 + l];
            unsigned long long best = ~0ull;
            for (int p = lane; p < P; p += 32) {
                const unsigned long long key = ((unsigned long long)ord32(sScore[l * P + p]) << 32) | (unsigned)p;
                best = key < best ? key : best;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const unsigned long long ob = __shfl_xor_sync(FULL, best, o);
                best = ob < best ? ob : best;
            }
            const int bp = (int)(best & 0xffffffffu);
            const int li = m.x, R = m.z, nang = S_w * R;
            if (lane == 0) {
                a.best_score[li] = sScore[l * P + bp];
                a.best_pose[li] = bp;
            }
            const uint8_t* sa = sAng + (size_t)(l * P + bp) * ang_stride;
            for (int t = lane; t < nang; t += 32) a.angles[m.w + t] = sa[t];
            if (a.dbg_score)
                for (int p = lane; p < P; p += 32) a.dbg_score[(size_t)li * P + p] = sScore[l * P + p];
            if (a.dbg_angles)
                for (int t = lane; t < P * nang; t += 32) {
                    const int p = t / nang, q = t - p * nang;
                    a.dbg_angles[(size_t)P * m.w + t] = sAng[(size_t)(l * P + p) * ang_stride + q];
                }
        }
    }
}

// a9 coordinates: replay p* with the recorded angles, bit-identical to the
// dock kernel (same placement, axis, Rodrigues and rotation helpers); one warp
// per ligand; output in Angstrom, input atom order.
template <int AC>
__global__ void __launch_bounds__(256) finalize_kernel(const DockArgs a, const int64_t* __restrict__ atom_off,
                                                       float* __restrict__ xyz_out) {
    __shared__ __align__(16) float4 sb[8][AC];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int s = blockIdx.x * 8 + w;
    if (s >= a.n) return;
    const PocketDev& pk = a.pk;
    const int4 m = a.meta[s];
    const int li = m.x, A = m.y, R = m.z;
    const int p = a.best_pose[li];
    const float* rec = a.rec + (size_t)s * a.rec_floats;
    const uint32_t* rfr = reinterpret_cast<const uint32_t*>(rec + 3 * AC);
    float T[12];
    scaled_pose(a.pose_tab + 12 * p, pk, T);
    const RotT Pz = load_pose(T);
    float4* buf = sb[w];
    for (int i = lane; i < A; i += 32) buf[i] = apply_rot(Pz, rec[i], rec[AC + i], rec[2 * AC + i]);
    __syncwarp();
    for (int sw = 0; sw < a.S_w; ++sw) {
        for (int r = 0; r < R; ++r) {
            const int bk = a.angles[m.w + sw * R + r];
            if (bk != 0) {
                const uint32_t f = rfr[r];
                const int fa = f & 255, fb = (f >> 8) & 255, lo = (f >> 16) & 255, hi = (int)(f >> 24) + 1;
                const float4 ya = buf[fa], yb = buf[fb];
                float ux, uy, uz;
                axis_of(ya, yb, ux, uy, uz);
                const RotT Ms = rodrigues_t(ux, uy, uz, a.cs[2 * bk], a.cs[2 * bk + 1], yb.x, yb.y, yb.z);
                for (int j = lo + lane; j < hi; j += 32) {
                    const float4 v = buf[j];
                    buf[j] = apply_rot(Ms, v.x, v.y, v.z);
                }
            }
            __syncwarp();
        }
    }
    float* out = xyz_out + 3 * atom_off[li];
    for (int i = lane; i < A; i += 32) {
        const float4 v = buf[i];
        out[3 * i] = __fmaf_rn(pk.h, v.x, pk.ox);
        out[3 * i + 1] = __fmaf_rn(pk.h, v.y, pk.oy);
        out[3 * i + 2] = __fmaf_rn(pk.h, v.z, pk.oz);
    }
}

template <bool FIX>
__global__ void __launch_bounds__(1024) score_points_kernel(const PocketDev pk, const float* __restrict__ xyz,
                                                            int64_t n, float* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem[];
    float* sG = reinterpret_cast<float*>(smem);
    stage_grid(sG, pk);
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float ux = __fmul_rn(__fsub_rn(xyz[3 * i], pk.ox), pk.inv_h);
        const float uy = __fmul_rn(__fsub_rn(xyz[3 * i + 1], pk.oy), pk.inv_h);
        const float uz = __fmul_rn(__fsub_rn(xyz[3 * i + 2], pk.oz), pk.inv_h);
        out[i] = grid_g<FIX>(sG, ux, uy, uz, pk);
    }
}

using DockFn = void (*)(const DockArgs);

template <int AC, bool FIX>
DockFn pick_ac(int NW, int PPW) {
    if (PPW == 1) return NW == 32 ? dock_kernel<AC, 32, 1, FIX> : (NW == 16 ? dock_kernel<AC, 16, 1, FIX> : nullptr);
    if (PPW == 2)
        return NW == 32 ? dock_kernel<AC, 32, 2, FIX>
                        : (NW == 16 ? dock_kernel<AC, 16, 2, FIX> : (NW == 8 ? dock_kernel<AC, 8, 2, FIX> : nullptr));
    if (PPW == 4)
        return NW == 16 ? dock_kernel<AC, 16, 4, FIX>
                        : (NW == 8 ? dock_kernel<AC, 8, 4, FIX> : (NW == 4 ? dock_kernel<AC, 4, 4, FIX> : nullptr));
    return nullptr;
}

template <bool FIX>
DockFn pick_fix(int AC, int NW, int PPW) {
    switch (AC) {
        case 32: return pick_ac<32, FIX>(NW, PPW);
        case 64: return pick_ac<64, FIX>(NW, PPW);
        case 96: return pick_ac<96, FIX>(NW, PPW);
        case 128: return pick_ac<128, FIX>(NW, PPW);
        case 160: return pick_ac<160, FIX>(NW, PPW);
        case 192: return pick_ac<192, FIX>(NW, PPW);
        case 224: return pick_ac<224, FIX>(NW, PPW);
        case 256: return pick_ac<256, FIX>(NW, PPW);
        default: return nullptr;
    }
}

DockFn pick(int AC, int NW, int PPW, int fix) { return fix ? pick_fix<true>(AC, NW, PPW) : pick_fix<false>(AC, NW, PPW); }

}  // namespace

// Padded shared-memory strides (tools/bank_sim.py: 2.5-way instead of 6.2-way bank
// conflicts on the sweep's corner gathers).  Grids of at most 32 x 32 per plane use
// the fixed layout (33, 1063) with compile-time strides; larger planes use
// (nx + 1, (nx + 1) * ny + 7).
void grid_strides(int nx, int ny, int* rs, int* ps) {
    if (nx <= 32 && ny <= 32) {
        *rs = kFixRS;
        *ps = kFixPS;
    } else {
        *rs = nx + 1;
        *ps = (nx + 1) * ny + 7;
    }
}

bool grid_fixed(int rs, int ps) { return rs == kFixRS && ps == kFixPS; }

cudaError_t dock_kernel_attrs(int AC, int NW, int PPW, int fix, cudaFuncAttributes* attr) {
    DockFn f = pick(AC, NW, PPW, fix);
    if (!f) return cudaErrorInvalidValue;
    return cudaFuncGetAttributes(attr, reinterpret_cast<const void*>(f));
}

cudaError_t dock_occupancy(int AC, int NW, int PPW, int fix, size_t smem, int* blocks_per_sm) {
    DockFn f = pick(AC, NW, PPW, fix);
    if (!f) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(f), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) {
        *blocks_per_sm = 0;
        cudaGetLastError();
        return cudaSuccess;
    }
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, reinterpret_cast<const void*>(f), NW * 32,
                                                         smem);
}

cudaError_t launch_dock(int AC, int NW, int PPW, const DockArgs& a, int grid, size_t smem, cudaStream_t st) {
    DockFn f = pick(AC, NW, PPW, grid_fixed(a.pk.rs, a.pk.ps));
    if (!f) return cudaErrorInvalidValue;
    if (a.n <= 0) return cudaSuccess;
    f<<<grid, NW * 32, smem, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_finalize(int AC, const DockArgs& a, const int64_t* atom_off, float* xyz_out, cudaStream_t st) {
    if (a.n <= 0) return cudaSuccess;
    const int grid = (a.n + 7) / 8;
    switch (AC) {
#define VSD_FIN(ac)                                                          \
    case ac:                                                                 \
        finalize_kernel<ac><<<grid, 256, 0, st>>>(a, atom_off, xyz_out);     \
        break;
        VSD_FIN(32)
        VSD_FIN(64)
        VSD_FIN(96)
        VSD_FIN(128)
        VSD_FIN(160)
        VSD_FIN(192)
        VSD_FIN(224)
        VSD_FIN(256)
#undef VSD_FIN
        default:
            return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_score_points(const PocketDev& pk, const float* xyz, int64_t n, float* out, size_t smem,
                                cudaStream_t st) {
    const bool fix = grid_fixed(pk.rs, pk.ps);
    const void* f = fix ? reinterpret_cast<const void*>(score_points_kernel<true>)
                        : reinterpret_cast<const void*>(score_points_kernel<false>);
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (fix) score_points_kernel<true><<<148, 1024, smem, st>>>(pk, xyz, n, out);
    else score_points_kernel<false><<<148, 1024, smem, st>>>(pk, xyz, n, out);
    return cudaGetLastError();
}

}  // namespace vsd
