// dock_impl.cuh -- the docking kernel (a6-a9): rigid roto-translation from P initial
// poses, greedy rotatable-bond sweep over K discrete angle steps, trilinear
// pocket-grid score, best-pose reduction.  fp32 on CUDA cores (not a dense
// contraction, BJ: "no tensor cores").
//
// B200 design:
//  * one CTA per SM, persistent over a launch's ligands; the pocket grid (32^3 fp32
//    = 128 KB, padded strides) lives in SHARED memory for the whole launch -- the 8
//    corner gathers of every evaluation are shared-memory loads, never L1/L2;
//  * warps run independently over a 3-slot ring of staged rounds (LC ligands each):
//    a warp item is PPW poses of one ligand (lane groups of 32/PPW), items are claimed
//    from a CTA-local counter, rounds from the launch's global counter (dynamic
//    balancing across CTAs); no CTA barrier after the prologue (dock_kernel below);
//  * sweep lane map inside a pose group: li = jl * K + k -- (moving atom jl of
//    the step, angle k).  Each lane holds its angle's rotation in registers and
//    scores the fragment's atoms in warp-uniform batches of up to 4; lanes of equal
//    k sum with xor shuffles, the argmin over k takes log2 K shuffle rounds (ties ->
//    lowest k, Q11), and the winner is applied (from registers when it fits);
//  * (x, y) arithmetic is packed in Blackwell's FFMA2/FADD2/FMUL2 (per-element IEEE
//    ops, so every result is bit-identical to the scalar form);
//  * template<int AC, int NW, int PPW, int GM, int KT> per atom class = the paper's
//    "non-type template parameter for the kernel maximum number of atoms":
//    AC sizes the per-pose buffers in shared memory, hence the warps per CTA;
//    GM = grid mode (FIX 32^3 / RT / WIN window + L2, internal.h), KT = compile-time K (8).
//
// All arithmetic that decides an angle or is replayed (placement, Rodrigues,
// rotation, interpolation) uses explicit _rn intrinsics in shared helpers, so
// the best-pose replay (replay_coords) reproduces the trajectory bit for bit.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "internal.h"

namespace vsd {

namespace dk {

constexpr unsigned FULL = 0xffffffffu;
constexpr float kMagic = 8388608.f;              // 2^23: floor via round-down add
constexpr int kMagicBits = 0x4B000000;
constexpr int kQuadMagicBits = 0x4B400000;       // bits of 1.5 * 2^23 (QUAD: signed floors)

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
// Rows 0 and 1 run as FFMA2/FMUL2 pairs (per element the same IEEE op as the scalar form).
__device__ __forceinline__ RotT rodrigues_t(float ux, float uy, float uz, float c, float s, float qx, float qy,
                                            float qz) {
    const float omc = __fsub_rn(1.f, c);
    const float2 ab = __fmul2_rn(f2(omc), make_float2(ux, uy));          // (a, b) = (1 - c) (ux, uy)
    const float d = __fmul_rn(omc, uz);
    const float2 sxy = __fmul2_rn(f2(s), make_float2(ux, uy));           // (sx, sy)
    const float sz = __fmul_rn(s, uz);
    RotT M;
    M.c0 = __ffma2_rn(ab, f2(ux), make_float2(c, sz));                   // (m00, m10)
    M.c1 = __ffma2_rn(ab, f2(uy), make_float2(-sz, c));                  // (m01, m11)
    M.c2 = __ffma2_rn(ab, f2(uz), make_float2(sxy.y, -sxy.x));           // (m02, m12)
    M.m20 = __fmaf_rn(d, ux, -sxy.y);
    M.m21 = __fmaf_rn(d, uy, sxy.x);
    M.m22 = __fmaf_rn(d, uz, c);
    // t = q - M q
    M.txy = __ffma2_rn(neg2(M.c0), f2(qx), __ffma2_rn(neg2(M.c1), f2(qy), __ffma2_rn(neg2(M.c2), f2(qz),
                                                                                      make_float2(qx, qy))));
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

// Trilinear blend of the 8 corners given as (z0, z1) pairs: x-lerps on the pairs, the
// y-lerp on the (l0, l1) pair, then z (Q10), + kappa*h*excess.
__device__ __forceinline__ float blend(float2 c00, float2 c10, float2 c01, float2 c11, float2 fxy, float fz, float kh,
                                      float e) {
    const float2 l_0 = lerp2(c00, c10, fxy.x);     // (l00, l01): y0, z0/z1
    const float2 l_1 = lerp2(c01, c11, fxy.x);     // (l10, l11): y1, z0/z1
    const float2 l = lerp2(l_0, l_1, fxy.y);       // (l0, l1)
    return __fmaf_rn(kh, e, lerp(l.x, l.y, fz));
}

// a8: g(u), u in grid units (Q9, Q10): clamp, L1 excess, i0 = min(floor(u_c), n-2),
// lerps x then y then z, + kappa*h*excess.  G is the shared-memory copy (strides rs, ps).
// floor(m) for 0 <= m < 2^23 is the round-down sum m + 2^23 (its bits also give the
// integer); identical values to floorf.  The x-lerps run on (z0, z1) pairs, the
// y-lerp on the (l0, l1) pair: per element the same fma sequence as the scalar form.
//
// The upper edge (u_c = n-1) takes i0 = n-1 with f = 0 instead of i0 = n-2 with f = 1:
// both reduce exactly to the node value (lerp(a, b, 0) = a, lerp(a, b, 1) = b bitwise),
// and the corner at n is a finite zero pad (row / column pads, the RT zero plane, the global
// copy's pads), so no clamp of i0 is needed -- except on the z axis of FIX, whose zero plane
// would cost the 128 class a warp: there i0 is clamped to n-2 with f = 1.
// GM = grid mode (internal.h): FIX -- the 32x32-plane layout with compile-time strides
// (34, 1097) that lets every corner load use an immediate offset; RT -- runtime strides;
// WIN -- the shared-memory window (fixed strides) with the padded global copy behind it:
// a warp whose cells all lie in the window takes the pure shared-memory path (one vote),
// otherwise each lane reads its 8 corners from the window or from global memory.
constexpr int kFixRS = 34, kFixPS = 1097;
// The cell of a point: i0 per axis (QUAD: window-relative), the x / y fractions, the z fraction
// and the L1 excess e (the first half of g; the corner gathers and the blend are the second).
struct GCell {
    int ix, iy, iz;
    float2 fxy;
    float fz, e;
};
template <int GM>
__device__ __forceinline__ GCell grid_cell(float ux, float uy, float uz, const PocketDev& pk) {
    // centred coordinates (PocketDev): clamp to [-Z, n-1-Z]; floor(u_c) = bits of the
    // round-down sum c + (2^23 + Z) minus the bits of 2^23; f = c - (floor(u_c) - Z)
    // (FIX: Z = 16 on every axis, so -Z and 2^23 + Z are immediates)
    constexpr bool IMM = GM == kGridFix;
    const float lox = IMM ? -16.f : pk.lo_x, loy = IMM ? -16.f : pk.lo_y, loz = IMM ? -16.f : pk.lo_z;
    const float mx = IMM ? 8388624.f : pk.mx, my = IMM ? 8388624.f : pk.my, mz = IMM ? 8388624.f : pk.mz;
    const float cx = fminf(fmaxf(ux, lox), pk.top_x);
    const float cy = fminf(fmaxf(uy, loy), pk.top_y);
    const float cz = fminf(fmaxf(uz, loz), pk.top_z);
    const float2 dxy = __fadd2_rn(make_float2(ux, uy), make_float2(-cx, -cy));
    const float e = __fadd_rn(__fadd_rn(fabsf(dxy.x), fabsf(dxy.y)), fabsf(__fsub_rn(uz, cz)));
    const float2 mxy = make_float2(mx, my);
    const float2 bxy = __fadd2_rd(make_float2(cx, cy), mxy);
    const float bz = __fadd_rd(cz, mz);
    const float2 fxy = __fadd2_rn(make_float2(cx, cy), neg2(__fadd2_rn(bxy, neg2(mxy))));
    const int ix = __float_as_int(bxy.x) - kMagicBits, iy = __float_as_int(bxy.y) - kMagicBits;
    int iz = __float_as_int(bz) - kMagicBits;
    float fz = __fsub_rn(cz, __fsub_rn(bz, mz));
    if (GM == kGridFix && iz > pk.nz - 2) {
        // top z face: i0 = n-2 with f = 1 (bitwise the same blend as i0 = n-1, f = 0), so no
        // corner read leaves the grid's planes (race-free: the region behind the grid is
        // live pose buffers); the y overflow of the last plane lands in a 32-float zero pad
        iz = pk.nz - 2;
        fz = 1.f;
    }
    if (GM == kGridQuad || GM == kGridTyped || GM == kGridTypedS) {
        // QUAD / TYPED / TYPED_S: the floor constant is 1.5 * 2^23 + Z - w0 (PocketDev), so the bits give the
        // WINDOW-relative cell directly (negative below the window)
        constexpr int d = kMagicBits - kQuadMagicBits;
        return GCell{ix + d, iy + d, iz + d, fxy, fz, e};
    }
    return GCell{ix, iy, iz, fxy, fz, e};
}

// QUAD: the cell's 8 corners are the quads of rows y and y + 1 of the window
__device__ __forceinline__ bool quad_in(const GCell& c) {
    return __vimax3_u32((unsigned)c.ix, (unsigned)c.iy, (unsigned)c.iz) < (unsigned)kQuadWC;
}
// quad = (G[x,y,z], G[x,y,z+1], G[x+1,y,z], G[x+1,y,z+1]): the (z0, z1) corner pairs of x and x + 1,
// each already a register pair for the FFMA2 x-lerps; the same blend as the scalar layouts, so the
// value is bit-identical to theirs
__device__ __forceinline__ float quad_blend(const float4& q0, const float4& q1, const GCell& c, float kh) {
    return blend(make_float2(q0.x, q0.y), make_float2(q0.z, q0.w), make_float2(q1.x, q1.y), make_float2(q1.z, q1.w),
                 c.fxy, c.fz, kh, c.e);
}
// the cell lies in the window (caller's guarantee): two LDS.128
__device__ __forceinline__ float quad_fast(const float* __restrict__ G, const GCell& c, float kh) {
    const float4* q = reinterpret_cast<const float4*>(G) + c.ix + c.iy * kQuadRS + c.iz * kQuadPS;
    return quad_blend(q[0], q[kQuadRS], c, kh);
}
// a cell outside the window: two 16-byte loads from the global QUAD copy (L1 / L2) of channel ch,
// the same four values per load as the window's node (clamped cells lie in [0, n-1]: x + 1 <= nx
// and z + 1 <= nz are the zero pads, row y + 1 <= ny exists)
__device__ __forceinline__ float quad_global(const GCell& c, int ch, const PocketDev& pk) {
    const float4* q = pk.gq + (size_t)ch * pk.gqcs + (c.ix + pk.wx0) + (size_t)(c.iy + pk.wy0) * pk.nx +
                      (size_t)(c.iz + pk.wz0) * ((size_t)pk.nx * (pk.ny + 1));
    return quad_blend(__ldg(q), __ldg(q + pk.nx), c, pk.kh);
}
// any cell: the window, or the padded global copy (L1 / L2) for the rare lane outside it
__device__ __forceinline__ float quad_checked(const float* __restrict__ G, const GCell& c, const PocketDev& pk) {
    if (__builtin_expect(quad_in(c), 1)) return quad_fast(G, c, pk.kh);
    // (QUAD's misses are rare; reading them from the global QUAD copy, as TYPED does, measured
    // 2.4 % slower here through the hot loop's code generation: the scalar padded copy is kept)
    const int gr = pk.grs, gp = pk.gps;
    const float* p = pk.grid + (c.ix + pk.wx0) + (size_t)(c.iy + pk.wy0) * gr + (size_t)(c.iz + pk.wz0) * gp;
    const float4 q0 = make_float4(__ldg(p), __ldg(p + gp), __ldg(p + 1), __ldg(p + gp + 1));
    const float4 q1 = make_float4(__ldg(p + gr), __ldg(p + gp + gr), __ldg(p + gr + 1), __ldg(p + gp + gr + 1));
    return quad_blend(q0, q1, c, pk.kh);
}

// QUAD fast path: the cell of the UNCLAMPED point.  The window's fast cells [0, pk.qwc) lie strictly
// inside the grid's interior cells [0, n-2] (make_pocket_dev), so for a point whose unclamped cell
// is one of them the clamp is the identity and the excess is exactly 0: g reduces to the trilinear
// blend, bit for bit (kappa h * 0 adds nothing to a sum that starts at +0).  Any other point (cell
// outside, or a non-finite / huge coordinate: the floor's bits then land far outside [0, qwc))
// takes the full path (grid_g).
__device__ __forceinline__ GCell quad_cell_fast(float ux, float uy, float uz, const PocketDev& pk) {
    const float2 mxy = make_float2(pk.mx, pk.my);
    const float2 bxy = __fadd2_rd(make_float2(ux, uy), mxy);
    const float bz = __fadd_rd(uz, pk.mz);
    const float2 fxy = __fadd2_rn(make_float2(ux, uy), neg2(__fadd2_rn(bxy, neg2(mxy))));
    const float fz = __fsub_rn(uz, __fsub_rn(bz, pk.mz));
    return GCell{__float_as_int(bxy.x) - kQuadMagicBits, __float_as_int(bxy.y) - kQuadMagicBits,
                 __float_as_int(bz) - kQuadMagicBits, fxy, fz, 0.f};
}
__device__ __forceinline__ bool quad_in_fast(const GCell& c, int qwc) {
    return __vimax3_u32((unsigned)c.ix, (unsigned)c.iy, (unsigned)c.iz) < (unsigned)qwc;
}
// TYPED's fast path keeps only the quad ADDRESS of the cell (channel included) and its fractions:
// 4 registers instead of 6 per point, so the compiler keeps more LDS.128 in flight (+4.6 % for
// typed launches; the QUAD path measured 1.2 % slower with it and keeps GCell)
struct QCell {
    int a;          // quad index in the window (valid when the warp's vote passed)
    float2 fxy;
    float fz;
};
// two LDS.128 and the blend without the excess term
__device__ __forceinline__ float quad_fast_interior(const float* __restrict__ G, const GCell& c) {
    const float4* q = reinterpret_cast<const float4*>(G) + c.ix + c.iy * kQuadRS + c.iz * kQuadPS;
    const float4 q0 = q[0], q1 = q[kQuadRS];
    const float2 l_0 = lerp2(make_float2(q0.x, q0.y), make_float2(q0.z, q0.w), c.fxy.x);
    const float2 l_1 = lerp2(make_float2(q1.x, q1.y), make_float2(q1.z, q1.w), c.fxy.x);
    const float2 l = lerp2(l_0, l_1, c.fxy.y);
    return lerp(l.x, l.y, c.fz);
}

// TYPED (Q24): the QUAD gathers on channel ch of the window (runtime strides rs = W, ps, qcs) or of
// the padded global copy (channel stride gcs)
__device__ __forceinline__ const float4* typed_quad(const float* __restrict__ G, const GCell& c, int ch,
                                                    const PocketDev& pk) {
    return reinterpret_cast<const float4*>(G) + c.ix + c.iy * pk.rs + c.iz * pk.ps + ch * pk.qcs;
}
__device__ __forceinline__ float typed_checked(const float* __restrict__ G, const GCell& c, int ch, const PocketDev& pk) {
    if (__builtin_expect(__vimax3_u32((unsigned)c.ix, (unsigned)c.iy, (unsigned)c.iz) < (unsigned)pk.rs, 1)) {
        const float4* q = typed_quad(G, c, ch, pk);
        return quad_blend(q[0], q[pk.rs], c, pk.kh);
    }
    return quad_global(c, ch, pk);
}

__device__ __forceinline__ float typed_addr_interior(const float* __restrict__ G, const QCell& c, int rs) {
    const float4* q = reinterpret_cast<const float4*>(G) + c.a;
    const float4 q0 = q[0], q1 = q[rs];
    const float2 l_0 = lerp2(make_float2(q0.x, q0.y), make_float2(q0.z, q0.w), c.fxy.x);
    const float2 l_1 = lerp2(make_float2(q1.x, q1.y), make_float2(q1.z, q1.w), c.fxy.x);
    const float2 l = lerp2(l_0, l_1, c.fxy.y);
    return lerp(l.x, l.y, c.fz);
}

// TYPED_S (Q24, scalar channel windows): the 8 corners of cell a (window float index, channel
// included) as the (z0, z1) pairs of x and x + 1 in rows y and y + 1 -- the values of the two
// TYPED quads, blended in the same order, so bit-identical to TYPED
__device__ __forceinline__ float typeds_addr_interior(const float* __restrict__ G, const QCell& c, int rs, int ps) {
    const float* p = G + c.a;
    const float2 l_0 = lerp2(make_float2(p[0], p[ps]), make_float2(p[1], p[ps + 1]), c.fxy.x);
    const float2 l_1 = lerp2(make_float2(p[rs], p[rs + ps]), make_float2(p[rs + 1], p[rs + ps + 1]), c.fxy.x);
    const float2 l = lerp2(l_0, l_1, c.fxy.y);
    return lerp(l.x, l.y, c.fz);
}
// any cell (clamped, window-relative): the channel window (cells [0, W), W = rs - 2) or the padded
// global copy of channel ch (L1 / L2)
__device__ __forceinline__ float typeds_checked(const float* __restrict__ G, const GCell& c, int ch, const PocketDev& pk) {
    const float* p;
    int rs, ps;
    if (__builtin_expect(__vimax3_u32((unsigned)c.ix, (unsigned)c.iy, (unsigned)c.iz) < (unsigned)(pk.rs - 2), 1)) {
        rs = pk.rs;
        ps = pk.ps;
        p = G + c.ix + c.iy * rs + c.iz * ps + ch * pk.qcs;
        return blend(make_float2(p[0], p[ps]), make_float2(p[1], p[ps + 1]), make_float2(p[rs], p[rs + ps]),
                     make_float2(p[rs + 1], p[rs + ps + 1]), c.fxy, c.fz, pk.kh, c.e);
    }
    const int gr = pk.grs, gp = pk.gps;
    p = pk.grid + (size_t)ch * pk.gcs + (c.ix + pk.wx0) + (size_t)(c.iy + pk.wy0) * gr + (size_t)(c.iz + pk.wz0) * gp;
    return blend(make_float2(__ldg(p), __ldg(p + gp)), make_float2(__ldg(p + 1), __ldg(p + gp + 1)),
                 make_float2(__ldg(p + gr), __ldg(p + gp + gr)), make_float2(__ldg(p + gr + 1), __ldg(p + gp + gr + 1)),
                 c.fxy, c.fz, pk.kh, c.e);
}

// ch = the atom's grid channel (TYPED / TYPED_S only; ignored by the other modes)
template <int GM>
__device__ __forceinline__ float grid_g(const float* __restrict__ G, float ux, float uy, float uz, const PocketDev& pk,
                                        int ch = 0) {
    const int RS = GM == kGridRT ? pk.rs : kFixRS, PS = GM == kGridRT ? pk.ps : kFixPS;
    const GCell cl = grid_cell<GM>(ux, uy, uz, pk);
    if (GM == kGridQuad) return quad_checked(G, cl, pk);
    if (GM == kGridTyped) return typed_checked(G, cl, ch, pk);
    if (GM == kGridTypedS) return typeds_checked(G, cl, ch, pk);
    const int ix = cl.ix, iy = cl.iy, iz = cl.iz;
    const float2 fxy = cl.fxy;
    const float fz = cl.fz, e = cl.e;
    if (GM != kGridWin) {
        const float* p = G + ix + iy * RS + iz * PS;
        return blend(make_float2(p[0], p[PS]), make_float2(p[1], p[PS + 1]), make_float2(p[RS], p[PS + RS]),
                     make_float2(p[RS + 1], p[PS + RS + 1]), fxy, fz, pk.kh, e);
    } else {
        const int lx = ix - pk.wx0, ly = iy - pk.wy0, lz = iz - pk.wz0;
        const bool in = ((unsigned)lx <= (unsigned)(kWin - 2)) & ((unsigned)ly <= (unsigned)(kWin - 2)) &
                        ((unsigned)lz <= (unsigned)(kWin - 2));
        if (__all_sync(__activemask(), in)) {
            const float* p = G + lx + ly * kFixRS + lz * kFixPS;
            return blend(make_float2(p[0], p[kFixPS]), make_float2(p[1], p[kFixPS + 1]),
                         make_float2(p[kFixRS], p[kFixPS + kFixRS]), make_float2(p[kFixRS + 1], p[kFixPS + kFixRS + 1]),
                         fxy, fz, pk.kh, e);
        }
        float2 c00, c10, c01, c11;
        if (in) {
            const float* p = G + lx + ly * kFixRS + lz * kFixPS;
            c00 = make_float2(p[0], p[kFixPS]);
            c10 = make_float2(p[1], p[kFixPS + 1]);
            c01 = make_float2(p[kFixRS], p[kFixPS + kFixRS]);
            c11 = make_float2(p[kFixRS + 1], p[kFixPS + kFixRS + 1]);
        } else {   // outside the window: the padded global copy (L1 / L2)
            const int gr = pk.grs, gp = pk.gps;
            const float* p = pk.grid + ix + (size_t)iy * gr + (size_t)iz * gp;
            c00 = make_float2(__ldg(p), __ldg(p + gp));
            c10 = make_float2(__ldg(p + 1), __ldg(p + gp + 1));
            c01 = make_float2(__ldg(p + gr), __ldg(p + gp + gr));
            c11 = make_float2(__ldg(p + gr + 1), __ldg(p + gp + gr + 1));
        }
        return blend(c00, c10, c01, c11, fxy, fz, pk.kh, e);
    }
}

// Pose p in centred grid units: R' = R / h, t' = (c + tau - o) / h - Z, v = R' x + t'.
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

// Stage the pocket grid (FIX / RT: all of it; WIN: the 32^3-node window) from the padded
// global copy into shared memory with padded strides; the padding (and the zero plane/row
// above the grid) is zero-filled first.  zero_floats: how much to zero first (the grid
// region, plus -- for the dock kernel -- the pose buffers behind it, see dock_grid_floats).
__device__ __forceinline__ void stage_grid(float* sG, const PocketDev& pk, size_t zero_floats) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int n4 = (int)(align16(zero_floats * 4) / 16);
    for (int t = threadIdx.x; t < n4; t += blockDim.x) reinterpret_cast<float4*>(sG)[t] = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncthreads();
    if (pk.mode == kGridTypedS) {
        // TYPED_S: nodes [w0, w0 + W] of every channel (rs - 1 = W + 1 per axis), channels qcs
        // floats apart; nodes beyond the padded copy stay zero (never read with weight > 0)
        const int N = pk.rs - 1;
        const int NX = min(N, pk.nx + 1 - pk.wx0), NY = min(N, pk.ny + 1 - pk.wy0), NZ = min(N, pk.nz + 1 - pk.wz0);
        for (int row = w; row < NY * NZ * pk.nch; row += nw) {
            const int ch = row / (NY * NZ), zy = row - ch * (NY * NZ);
            const int z = zy / NY, y = zy - z * NY;
            const float* src = pk.grid + (size_t)ch * pk.gcs + (size_t)(pk.wz0 + z) * pk.gps +
                               (size_t)(pk.wy0 + y) * pk.grs + pk.wx0;
            float* dst = sG + (size_t)ch * pk.qcs + z * pk.ps + y * pk.rs;
            for (int x = lane; x < NX; x += 32) dst[x] = src[x];
        }
        return;
    }
    if (pk.mode == kGridQuad || pk.mode == kGridTyped) {
        // node (x, y, z) of the window <- (G[x,y,z], G[x,y,z+1], G[x+1,y,z], G[x+1,y,z+1]) from the
        // padded global copy; nodes beyond the grid's pads stay zero (never read with weight > 0).
        // TYPED: one window per channel, qcs quads apart
        float4* Q = reinterpret_cast<float4*>(sG);
        const bool typed = pk.mode == kGridTyped;
        const int W = typed ? pk.rs : kQuadWC, RS = typed ? pk.rs : kQuadRS, PS = typed ? pk.ps : kQuadPS;
        const int NX = min(W, pk.nx - pk.wx0), NY = min(W + 1, pk.ny - pk.wy0), NZ = min(W, pk.nz - pk.wz0);
        for (int row = w; row < NY * NZ * pk.nch; row += nw) {
            const int ch = row / (NY * NZ), zy = row - ch * (NY * NZ);
            const int z = zy / NY, y = zy - z * NY;
            const float* src = pk.grid + (size_t)ch * pk.gcs + (size_t)(pk.wz0 + z) * pk.gps +
                               (size_t)(pk.wy0 + y) * pk.grs + pk.wx0;
            float4* dst = Q + (size_t)ch * pk.qcs + z * PS + y * RS;
            for (int x = lane; x < NX; x += 32)
                dst[x] = make_float4(src[x], src[x + pk.gps], src[x + 1], src[x + pk.gps + 1]);
        }
        return;
    }
    const bool win = pk.mode == kGridWin;
    const int x0 = win ? pk.wx0 : 0, y0 = win ? pk.wy0 : 0, z0 = win ? pk.wz0 : 0;
    const int NX = win ? min(kWin, pk.nx - x0) : pk.nx, NY = win ? min(kWin, pk.ny - y0) : pk.ny,
              NZ = win ? min(kWin, pk.nz - z0) : pk.nz;
    for (int row = w; row < NY * NZ; row += nw) {
        const int z = row / NY, y = row - z * NY;
        const float* src = pk.grid + (size_t)(z0 + z) * pk.gps + (size_t)(y0 + y) * pk.grs + x0;
        float* dst = sG + z * pk.ps + y * pk.rs;
        for (int x = lane; x < NX; x += 32) dst[x] = src[x];
    }
}

// Order-preserving map of fp32 onto uint32 (-0 canonicalised to +0 first).
__device__ __forceinline__ unsigned ord32(float v) {
    const unsigned b = __float_as_uint(__fadd_rn(v, 0.0f));
    return b ^ ((unsigned)((int)b >> 31) | 0x80000000u);
}

// Per-pose coordinate buffer in shared memory: (x, y) pairs then z (12 B per atom), pose
// buffers pose_stride_of(AC, NW, PPW) floats apart (internal.h).
template <int AC>
struct PoseBuf {
    float* b;   // (x, y) pairs [2 AC] | z [AC]: one 8-byte and one 4-byte load per atom
    __device__ __forceinline__ float4 get(int j) const {
        const float2 xy = *reinterpret_cast<const float2*>(b + 2 * j);
        return make_float4(xy.x, xy.y, b[2 * AC + j], 0.f);
    }
    __device__ __forceinline__ void set(int j, float4 v) const {
        *reinterpret_cast<float2*>(b + 2 * j) = make_float2(v.x, v.y);
        b[2 * AC + j] = v.z;
    }
};

// g of U points per lane, the warp CONVERGED (all 32 lanes): QUAD decides the window once per
// batch (one vote), so the common case is two LDS.128 per point with no per-point branch.
template <int U, int GM>
__device__ __forceinline__ void grid_batch(const float* __restrict__ G, const float4 (&v)[4], const PocketDev& pk,
                                           float (&g)[U], const int (&ch)[4]) {
    if (GM == kGridTypedS) {   // Q24, scalar channel windows: the same vote, eight LDS.32 per point
        QCell cl[U];
        bool all = true;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const GCell c = quad_cell_fast(v[u].x, v[u].y, v[u].z, pk);
            all = all && quad_in_fast(c, pk.qwc);
            cl[u] = QCell{c.ix + c.iy * pk.rs + c.iz * pk.ps + ch[u] * pk.qcs, c.fxy, c.fz};
        }
        if (__all_sync(FULL, all)) {
#pragma unroll
            for (int u = 0; u < U; ++u) g[u] = typeds_addr_interior(G, cl[u], pk.rs, pk.ps);
        } else {
#pragma unroll
            for (int u = 0; u < U; ++u) g[u] = grid_g<GM>(G, v[u].x, v[u].y, v[u].z, pk, ch[u]);
        }
    } else if (GM == kGridTyped) {   // Q24: the QUAD vote on the channel windows
        QCell cl[U];
        bool all = true;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const GCell c = quad_cell_fast(v[u].x, v[u].y, v[u].z, pk);
            all = all && quad_in_fast(c, pk.qwc);
            cl[u] = QCell{c.ix + c.iy * pk.rs + c.iz * pk.ps + ch[u] * pk.qcs, c.fxy, c.fz};
        }
        if (__all_sync(FULL, all)) {
#pragma unroll
            for (int u = 0; u < U; ++u) g[u] = typed_addr_interior(G, cl[u], pk.rs);
        } else {
#pragma unroll
            for (int u = 0; u < U; ++u) g[u] = grid_g<GM>(G, v[u].x, v[u].y, v[u].z, pk, ch[u]);
        }
    } else if (GM == kGridQuad) {
        // (keeping addresses instead of cells, as TYPED does, measured 1.2 % slower here: the
        // compiler then hoists more LDS.128 ahead of their use)
        GCell cl[U];
        bool all = true;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            cl[u] = quad_cell_fast(v[u].x, v[u].y, v[u].z, pk);
            all = all && quad_in_fast(cl[u], pk.qwc);
        }
        if (__all_sync(FULL, all)) {
#pragma unroll
            for (int u = 0; u < U; ++u) g[u] = quad_fast_interior(G, cl[u]);
        } else {
#pragma unroll
            for (int u = 0; u < U; ++u) g[u] = grid_g<GM>(G, v[u].x, v[u].y, v[u].z, pk);
        }
    } else {
#pragma unroll
        for (int u = 0; u < U; ++u) g[u] = grid_g<GM>(G, v[u].x, v[u].y, v[u].z, pk);
    }
}

// U independent sweep evaluations per lane: atoms j0, j0 + apw, ... (j < hi), rotated by M,
// scored, summed into acc in ascending order; the atoms j < own_end (the step's finalised own
// region) are also summed into own; the rotated atoms stay in kp[0..U).
// ty = the record's atom types (TYPED, Q24; unused otherwise).
template <int U, int GM, int AC>
__device__ __forceinline__ void eval_batch(const PoseBuf<AC>& B, const RotT& M, const float* __restrict__ G,
                                           const PocketDev& pk, const uint8_t* __restrict__ ty, int j0, int apw,
                                           int hi, int own_end, float& acc, float& own, float4 (&kp)[4]) {
    float4 v[U];
    float g[U];
    int ch[4] = {0, 0, 0, 0};
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int j = j0 + u * apw;
        v[u] = B.get(j < hi ? j : j0);
        if (typed_mode(GM)) ch[u] = ty[j < hi ? j : j0];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) kp[u] = apply_rot(M, v[u].x, v[u].y, v[u].z);
    grid_batch<U, GM>(G, kp, pk, g, ch);
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int j = j0 + u * apw;
        if (j < hi) acc = __fadd_rn(acc, g[u]);
        if (j < own_end) own = __fadd_rn(own, g[u]);
    }
}

// a9: U pose-score evaluations per lane (atoms j0, j0 + stride, ...; j < n), summed into acc in
// ascending order -- the canonical order -- through the sweep's batch path (one window vote)
template <int U, int GM, int AC>
__device__ __forceinline__ void score_batch(const PoseBuf<AC>& B, const float* __restrict__ G, const PocketDev& pk,
                                            const uint8_t* __restrict__ ty, int j0, int stride, int n, float& acc) {
    float4 v[4];
    float g[U];
    int ch[4] = {0, 0, 0, 0};
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int j = j0 + u * stride;
        const int jj = j < n ? j : 0;
        v[u] = B.get(jj);
        if (typed_mode(GM)) ch[u] = ty[jj];
    }
    grid_batch<U, GM>(G, v, pk, g, ch);
#pragma unroll
    for (int u = 0; u < U; ++u)
        if (j0 + u * stride < n) acc = __fadd_rn(acc, g[u]);
}

// Centroid of a pose (grid units) for the rigid refinement (Q23), in ONE fixed order shared by
// the dock sweep and the best-pose replay: lane li of a group of LPP lanes sums atoms li,
// li + LPP, ... ascending, then an xor butterfly over the group (every lane ends with the
// same sum), divided by A.  The whole warp must be converged.
template <int AC, int LPP>
__device__ __forceinline__ void pose_centroid(const PoseBuf<AC>& B, int A, int li, float& cx, float& cy, float& cz) {
    float sx = 0.f, sy = 0.f, sz = 0.f;
    for (int i = li; i < A; i += LPP) {
        const float4 v = B.get(i);
        sx = __fadd_rn(sx, v.x);
        sy = __fadd_rn(sy, v.y);
        sz = __fadd_rn(sz, v.z);
    }
#pragma unroll
    for (int o = 1; o < LPP; o <<= 1) {
        sx = __fadd_rn(sx, __shfl_xor_sync(FULL, sx, o));
        sy = __fadd_rn(sy, __shfl_xor_sync(FULL, sy, o));
        sz = __fadd_rn(sz, __shfl_xor_sync(FULL, sz, o));
    }
    const float a = (float)A;
    cx = __fdiv_rn(sx, a);
    cy = __fdiv_rn(sy, a);
    cz = __fdiv_rn(sz, a);
}

// Rigid refinement move (Q23) in "M v + t" form about the centroid c (grid units):
// v' = Q (v - c) + c + d / h, i.e. M = Q, t = (c + d / h) - Q c.  tab = the move's 12 floats.
__device__ __forceinline__ RotT rigid_t(const float* __restrict__ tab, float cx, float cy, float cz, float inv_h) {
    RotT M;
    M.c0 = make_float2(tab[0], tab[3]);
    M.c1 = make_float2(tab[1], tab[4]);
    M.c2 = make_float2(tab[2], tab[5]);
    M.m20 = tab[6];
    M.m21 = tab[7];
    M.m22 = tab[8];
    const float2 base = make_float2(__fmaf_rn(tab[9], inv_h, cx), __fmaf_rn(tab[10], inv_h, cy));
    const float bz = __fmaf_rn(tab[11], inv_h, cz);
    M.txy = __ffma2_rn(neg2(M.c0), f2(cx), __ffma2_rn(neg2(M.c1), f2(cy), __ffma2_rn(neg2(M.c2), f2(cz), base)));
    M.tz = __fmaf_rn(-M.m20, cx, __fmaf_rn(-M.m21, cy, __fmaf_rn(-M.m22, cz, bz)));
    return M;
}

// PPW poses of one ligand on one warp: lanes [h*LPP, (h+1)*LPP) serve pose h.
// a6 placement, a7 sweep, a9 pose score.
// KT = the angle count when known at compile time (8: the production path, every lane-map
// constant folds), 0 = runtime K.
// K need not be a power of two: the lane map uses Kp = the next power of two >= K (kbits =
// log2 Kp) and the lanes of angle slots k >= K hold the identity and never win.
template <int AC, int PPW, int GM, int KT>
__device__ __forceinline__ void dock_poses(const float* __restrict__ rec, int A, int R, const float* __restrict__ T,
                                           bool valid, PoseBuf<AC> B, const float* __restrict__ G,
                                           const PocketDev& pk, int K_rt, int kbits_rt, int S_w, float ck, float sk,
                                           int n_ref, int n_moves, const float* __restrict__ ref_tab,
                                           uint8_t* __restrict__ angOut,
                                           float* __restrict__ scoreOut, int lane) {
    constexpr int LPP = 32 / PPW;
    const int K = KT ? KT : K_rt;
    const int kbits = KT ? (KT == 1 ? 0 : KT == 2 ? 1 : KT == 4 ? 2 : KT == 8 ? 3 : KT == 16 ? 4 : 5) : kbits_rt;
    const int Kp = 1 << kbits;
    const int li = lane & (LPP - 1);
    const float* rx = rec;
    const float* ry = rec + AC;
    const float* rz = rec + 2 * AC;
    const uint32_t* rfr = reinterpret_cast<const uint32_t*>(rec + 3 * AC);
    const uint8_t* rown = reinterpret_cast<const uint8_t*>(rec + 3 * AC + 32);
    const uint32_t hdr = reinterpret_cast<const uint32_t*>(rec + 3 * AC + 40)[0];
    const uint8_t* ty = reinterpret_cast<const uint8_t*>(rec + rec_floats_of(AC));   // TYPED records only (Q24)
    // finalised own regions: with ancestors swept before descendants, the atoms
    // whose innermost moving set is r (the first rown[r] atoms of r's range) never move after
    // step r of the last sweep, so the winner's partial sum over them is their final score;
    // the pose score then needs a final pass over the n_root atoms in no set only
    const bool fin = K > 1 && n_ref == 0 && ((hdr >> 16) & 1u);   // refinement moves every atom again
    const int n_final = fin ? (int)(hdr & 0xffffu) : A;
    float fsum = 0.f;   // finalised own-region scores, in fragment order
    {
        const RotT Pz = load_pose(T);
        if (valid)
            for (int i = li; i < A; i += LPP) B.set(i, apply_rot(Pz, rx[i], ry[i], rz[i]));
    }
    __syncwarp();
    if (K > 1) {
        const int k = li & (Kp - 1);
        const bool kreal = KT ? true : k < K;         // angle slot holds a table entry
        const int jl = li >> kbits;
        const int abits = __ffs(LPP) - 1 - kbits;     // log2(apw)
        const int apw = 1 << abits;                   // moving atoms per step of a pose group
        const unsigned gmask = ((Kp == 32) ? 0xffffffffu : ((1u << Kp) - 1u)) << (lane & ~(Kp - 1));
        for (int sw = 0; sw < S_w; ++sw) {
            for (int r = 0; r < R; ++r) {
                const uint32_t f = rfr[r];
                const int fa = f & 255, fb = (f >> 8) & 255, lo = (f >> 16) & 255, hi = (int)(f >> 24) + 1;
                const float4 ya = B.get(fa), yb = B.get(fb);
                float ux, uy, uz;
                axis_of(ya, yb, ux, uy, uz);
                const RotT M = rodrigues_t(ux, uy, uz, ck, sk, yb.x, yb.y, yb.z);
                // steps of apw atoms; the step count is warp-uniform (all pose groups of a
                // warp dock the same ligand), so the batch dispatch below never diverges.
                // Every lane sums its atoms in ascending order (the canonical order).
                const int nst = (hi - lo + apw - 1) >> abits;
                const bool last = fin && sw == S_w - 1;
                const int own_end = last ? lo + rown[r] : lo;
                float acc = 0.f, own = 0.f;
                float4 kp[4];
                int st = 0;
                for (; st + 4 <= nst; st += 4)
                    eval_batch<4, GM>(B, M, G, pk, ty, lo + st * apw + jl, apw, hi, own_end, acc, own, kp);
                switch (nst - st) {
                    case 3: eval_batch<3, GM>(B, M, G, pk, ty, lo + st * apw + jl, apw, hi, own_end, acc, own, kp); break;
                    case 2: eval_batch<2, GM>(B, M, G, pk, ty, lo + st * apw + jl, apw, hi, own_end, acc, own, kp); break;
                    case 1: eval_batch<1, GM>(B, M, G, pk, ty, lo + st * apw + jl, apw, hi, own_end, acc, own, kp); break;
                    default: break;
                }
                // sum over the pass atoms (lanes of equal k: xor offsets K .. LPP/2, ascending)
#pragma unroll
                for (int o = 1; o < LPP; o <<= 1)
                    if (o >= Kp) {
                        acc = __fadd_rn(acc, __shfl_xor_sync(FULL, acc, o));
                        if (last) own = __fadd_rn(own, __shfl_xor_sync(FULL, own, o));
                    }
                // argmin over the K angles of this group (xor offsets 1 .. Kp/2); ties -> lowest k (Q11)
                const unsigned key = kreal ? ord32(acc) : 0xffffffffu;
                unsigned mn = key;
#pragma unroll
                for (int o = 1; o < LPP; o <<= 1)
                    if (o < Kp) mn = min(mn, __shfl_xor_sync(FULL, mn, o));
                const unsigned bal = __ballot_sync(FULL, key == mn && kreal) & gmask;
                const int bk = (__ffs(bal) - 1) & (Kp - 1);
                if (last) fsum = __fadd_rn(fsum, __shfl_sync(FULL, own, (lane & ~(LPP - 1)) | bk));
                if (nst <= 4) {
                    // one batch: the lanes (jl, k*) still hold the rotated atoms in registers
                    if (valid && bk != 0 && k == bk) {
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int j = lo + u * apw + jl;
                            if (u < nst && j < hi) B.set(j, kp[u]);
                        }
                    }
                } else {
                    // the winner's (cos, sin) from its lane (warp-uniform branch: nst is);
                    // bit-identical rotation (same axis, same table entry)
                    const int wl = (lane & ~(LPP - 1)) | bk;
                    const float cw = __shfl_sync(FULL, ck, wl), sw2 = __shfl_sync(FULL, sk, wl);
                    if (valid && bk != 0) {
                        const RotT Ms = rodrigues_t(ux, uy, uz, cw, sw2, yb.x, yb.y, yb.z);
                        for (int j = lo + li; j < hi; j += LPP) {
                            const float4 v = B.get(j);
                            B.set(j, apply_rot(Ms, v.x, v.y, v.z));
                        }
                    }
                }
                __syncwarp();
                if (valid && li == 0) angOut[sw * R + r] = (uint8_t)bk;
            }
        }
    } else if (valid) {
        for (int t = li; t < S_w * R; t += LPP) angOut[t] = 0;
    }
    if (n_ref > 0) {
        // rigid refinement: every round scores the n_moves moves of the
        // table about the pose's centroid, in groups of Kp on the sweep's lane map (lane slot k
        // of group g0 = move g0 + k; every atom is a moving atom), and applies the lowest move
        // index attaining the minimum (Q11: a group replaces the running best only when strictly
        // lower; slots past the table hold the identity and never win)
        const int k = li & (Kp - 1);
        const int jl = li >> kbits;
        const int abits = __ffs(LPP) - 1 - kbits;
        const int apw = 1 << abits;
        const unsigned gmask = ((Kp == 32) ? 0xffffffffu : ((1u << Kp) - 1u)) << (lane & ~(Kp - 1));
        const int nst = (A + apw - 1) >> abits;
        for (int t = 0; t < n_ref; ++t) {
            float cx, cy, cz;
            pose_centroid<AC, LPP>(B, A, li, cx, cy, cz);
            unsigned bkey = 0xffffffffu;
            int bm = 0;
            for (int g0 = 0; g0 < n_moves; g0 += Kp) {
                const int m = g0 + k;
                const bool mreal = m < n_moves;
                const RotT M = rigid_t(ref_tab + 12 * (mreal ? m : 0), cx, cy, cz, pk.inv_h);
                float acc = 0.f, own = 0.f;
                float4 kp[4];
                int st = 0;
                for (; st + 4 <= nst; st += 4) eval_batch<4, GM>(B, M, G, pk, ty, st * apw + jl, apw, A, 0, acc, own, kp);
                switch (nst - st) {
                    case 3: eval_batch<3, GM>(B, M, G, pk, ty, st * apw + jl, apw, A, 0, acc, own, kp); break;
                    case 2: eval_batch<2, GM>(B, M, G, pk, ty, st * apw + jl, apw, A, 0, acc, own, kp); break;
                    case 1: eval_batch<1, GM>(B, M, G, pk, ty, st * apw + jl, apw, A, 0, acc, own, kp); break;
                    default: break;
                }
#pragma unroll
                for (int o = 1; o < LPP; o <<= 1)
                    if (o >= Kp) acc = __fadd_rn(acc, __shfl_xor_sync(FULL, acc, o));
                const unsigned key = mreal ? ord32(acc) : 0xffffffffu;
                unsigned mn = key;
#pragma unroll
                for (int o = 1; o < LPP; o <<= 1)
                    if (o < Kp) mn = min(mn, __shfl_xor_sync(FULL, mn, o));
                const unsigned bal = __ballot_sync(FULL, key == mn && mreal) & gmask;
                const int bk = (__ffs(bal) - 1) & (Kp - 1);
                if (mn < bkey) {
                    bkey = mn;
                    bm = g0 + bk;
                }
            }
            if (valid && bm != 0) {
                const RotT Ms = rigid_t(ref_tab + 12 * bm, cx, cy, cz, pk.inv_h);
                for (int j = li; j < A; j += LPP) {
                    const float4 v = B.get(j);
                    B.set(j, apply_rot(Ms, v.x, v.y, v.z));
                }
            }
            __syncwarp();
            if (valid && li == 0) angOut[S_w * R + t] = (uint8_t)bm;
        }
    }
    // a9: pose score, canonical order (atom i -> lane i mod LPP, ascending, xor tree, then the
    // finalised own regions in fragment order) (Q22); four independent evaluations in flight,
    // summed in the same ascending order
    // (warp-uniform batches of up to 4 steps -- n_final is the same for the warp's pose groups --
    // so the batch takes the vote-checked fast path of the sweep)
    float acc = 0.f;
    for (int base = 0; base < n_final; base += 4 * LPP) {
        const int nst = (n_final - base + LPP - 1) / LPP;
        switch (nst >= 4 ? 4 : nst) {
            case 4: score_batch<4, GM>(B, G, pk, ty, base + li, LPP, n_final, acc); break;
            case 3: score_batch<3, GM>(B, G, pk, ty, base + li, LPP, n_final, acc); break;
            case 2: score_batch<2, GM>(B, G, pk, ty, base + li, LPP, n_final, acc); break;
            default: score_batch<1, GM>(B, G, pk, ty, base + li, LPP, n_final, acc); break;
        }
    }
#pragma unroll
    for (int o = LPP / 2; o > 0; o >>= 1) acc = __fadd_rn(acc, __shfl_xor_sync(FULL, acc, o));
    if (fin) acc = __fadd_rn(acc, fsum);
    if (valid && li == 0) *scoreOut = acc;
    __syncwarp();
}

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ int ld_acquire_cta(const int* p) {
    int v;
    asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];\n" : "=r"(v) : "r"(smem_u32(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_cta(int* p, int v) {
    asm volatile("st.release.cta.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(p)), "r"(v) : "memory");
}

// mbarrier + TMA bulk copy (cp.async.bulk, 1-D): the round loader issues the record copy
// and moves on; consumers wait on the slot's mbarrier phase (one phase per use of the slot).
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, unsigned parity) {
    unsigned done;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return done != 0;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// Bounded back-off for the ring's spin-waits: a legitimate wait lasts microseconds; a
// wait of seconds can only be a broken invariant, and trapping turns it into a launch
// error (VS_E_CUDA from vs_wait) instead of a hung GPU.
__device__ __forceinline__ void ring_backoff(unsigned& spins) {
    __nanosleep(64);
    if (++spins > (1u << 26)) __trap();
}

// ---- thread-block cluster primitives (fused multi-site launches, MS)
__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
// shared::cluster address of a local shared variable's copy in CTA `rank` of the cluster
__device__ __forceinline__ unsigned mapa(const void* p, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_cluster(unsigned addr, int v) {
    asm volatile("st.shared::cluster.b32 [%0], %1;\n" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_cluster(unsigned addr, int v) {
    asm volatile("st.release.cluster.shared::cluster.b32 [%0], %1;\n" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void red_min_cluster(unsigned addr, int v) {
    asm volatile("red.shared::cluster.min.s32 [%0], %1;\n" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_cluster(const int* p) {
    int v;
    asm volatile("ld.acquire.cluster.shared::cta.b32 %0, [%1];\n" : "=r"(v) : "r"(smem_u32(p)) : "memory");
    return v;
}
__device__ __forceinline__ void mbar_arrive_remote(unsigned addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(addr) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx_remote(unsigned addr, unsigned tx) {
    asm volatile("mbarrier.arrive.expect_tx.release.cluster.shared::cluster.b64 _, [%0], %1;\n" ::"r"(addr), "r"(tx)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait_cluster(uint64_t* bar, unsigned parity) {
    unsigned done;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return done != 0;
}
// TMA bulk copy global -> the same shared-memory offset of every CTA in cta_mask, signalling
// each destination CTA's mbarrier at the same offset (one L2 read feeds the whole cluster)
__device__ __forceinline__ void bulk_g2s_multicast(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                                   unsigned short cta_mask) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;\n"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "h"(cta_mask)
        : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// Ring control in static shared memory (one entry per slot).
struct DockRing {
    int ready[kDockSlots];   // round sequence number whose record this slot holds
    int round[kDockSlots];   // global round index held (-1: the launch is exhausted)
    int done[kDockSlots];    // warp items of the slot's round completed
    int free_seq[kDockSlots];// next sequence number allowed into the slot
    int claim[kDockSlots];   // global round index claimed for sequence s (at s % kDockSlots), one ahead
    int item;                // CTA-local item counter
    int end_seq;             // first sequence number that found the launch exhausted (INT_MAX: none yet)
    uint64_t bar[kDockSlots];// record arrival (TMA complete_tx), phase (s / kDockSlots) & 1 for sequence s
    uint64_t free_bar[kDockSlots];   // MS, rank 0: every CTA of the cluster released the slot
};

// Stage sequence `seq` into `slot` and publish it: lane 0 issues TMA bulk copies of the
// round's LC records + meta (arrival on the slot's mbarrier) and a release store of the
// round index.  The round was claimed one sequence earlier; the claim for seq + 1 (the
// launch's global counter: dynamic scheduling across CTAs) is issued here, claims stay in
// sequence order.
//
// MS (fused multi-site, run by CTA rank 0 only): the slot is free once EVERY CTA of the cluster
// released it (free_bar, one phase per use); the round index and the ready flag are written into
// every CTA's ring (DSMEM stores, release at cluster scope), every CTA's mbarrier is armed remotely
// with the byte count, and ONE multicast TMA copy stages the records + meta into all of them.
template <int AC, bool MS>
__device__ __forceinline__ void load_round(const DockArgs& a, DockRing& ring, unsigned char* slot, const DockLayout& L,
                                           int seq, int n_rounds, int lane) {
    const int sl = seq % kDockSlots;
    if (MS) {
        if (lane == 0) {
            unsigned spins = 0;
            if (seq >= kDockSlots)
                while (!mbar_try_wait_cluster(&ring.free_bar[sl], (unsigned)(seq / kDockSlots - 1) & 1u))
                    ring_backoff(spins);
            const int round = ring.claim[sl];
            const int next = atomicAdd(a.counter, 1);
            ring.claim[(seq + 1) % kDockSlots] = next;
            const int S = a.n_sites;
            const bool have = round < n_rounds;
            const int LC = a.ligs_per_cta;
            const int slot0 = have ? round * LC : 0;
            const int nl = have ? min(LC, a.n - slot0) : 0;
            const unsigned rb = (unsigned)(nl * a.rec_floats * 4), mb = (unsigned)(nl * 16);
            for (int r = 0; r < S; ++r) {
                st_cluster(mapa(&ring.round[sl], r), have ? round : -1);
                if (!have) red_min_cluster(mapa(&ring.end_seq, r), seq);
                if (have) mbar_arrive_expect_tx_remote(mapa(&ring.bar[sl], r), rb + mb);
                else mbar_arrive_remote(mapa(&ring.bar[sl], r));
                st_release_cluster(mapa(&ring.ready[sl], r), seq);
            }
            if (have) {
                const unsigned short mask = (unsigned short)((1u << S) - 1u);
                bulk_g2s_multicast(slot + L.rec_o, a.rec + (size_t)slot0 * a.rec_floats, rb, &ring.bar[sl], mask);
                bulk_g2s_multicast(slot + L.meta_o, a.meta + slot0, mb, &ring.bar[sl], mask);
            }
        }
        __syncwarp();
        return;
    }
    if (lane == 0) {
        unsigned spins = 0;
        while (ld_acquire_cta(&ring.free_seq[sl]) != seq) ring_backoff(spins);
        const int round = ring.claim[sl];
        const int next = atomicAdd(a.counter, 1);
        if (round < n_rounds) {
            const int LC = a.ligs_per_cta;
            const int slot0 = round * LC;
            const int nl = min(LC, a.n - slot0);
            const unsigned rb = (unsigned)(nl * a.rec_floats * 4), mb = (unsigned)(nl * 16);
            mbar_arrive_expect_tx(&ring.bar[sl], rb + mb);
            bulk_g2s(slot + L.rec_o, a.rec + (size_t)slot0 * a.rec_floats, rb, &ring.bar[sl]);
            bulk_g2s(slot + L.meta_o, a.meta + slot0, mb, &ring.bar[sl]);
        } else {
            mbar_arrive(&ring.bar[sl]);   // the phase completes without data
        }
        ring.claim[(seq + 1) % kDockSlots] = next;
        ring.round[sl] = round < n_rounds ? round : -1;
        if (round >= n_rounds) atomicMin(&ring.end_seq, seq);
        st_release_cta(&ring.ready[sl], seq);
    }
    __syncwarp();
}

// a9 best-pose coordinates of one ligand: replay pose p with the recorded angle choices, bit-
// identical to the dock trajectory (same placement, axis, Rodrigues and rotation helpers, same
// table entries) on one warp's pose buffer (all 32 lanes), written in Angstrom in the caller's
// input atom order (a1's order map).
template <int AC, int LPP>
__device__ __forceinline__ void replay_coords(const DockArgs& a, const PocketDev& pk, float* __restrict__ xyz_out,
                                              const float* __restrict__ rec, int li, int A, int R, int p,
                                              const uint8_t* __restrict__ ang, PoseBuf<AC> buf, int lane) {
    const uint32_t* rfr = reinterpret_cast<const uint32_t*>(rec + 3 * AC);
    float T[12];
    scaled_pose(a.pose_tab + 12 * p, pk, T);
    const RotT Pz = load_pose(T);
    for (int i = lane; i < A; i += 32) buf.set(i, apply_rot(Pz, rec[i], rec[AC + i], rec[2 * AC + i]));
    __syncwarp();
    for (int sw = 0; sw < a.S_w; ++sw) {
        for (int r = 0; r < R; ++r) {
            const int bk = ang[sw * R + r];
            if (bk != 0) {
                const uint32_t f = rfr[r];
                const int fa = f & 255, fb = (f >> 8) & 255, lo = (f >> 16) & 255, hi = (int)(f >> 24) + 1;
                const float4 ya = buf.get(fa), yb = buf.get(fb);
                float ux, uy, uz;
                axis_of(ya, yb, ux, uy, uz);
                const RotT Ms = rodrigues_t(ux, uy, uz, a.cs[2 * bk], a.cs[2 * bk + 1], yb.x, yb.y, yb.z);
                for (int j = lo + lane; j < hi; j += 32) {
                    const float4 v = buf.get(j);
                    buf.set(j, apply_rot(Ms, v.x, v.y, v.z));
                }
            }
            __syncwarp();
        }
    }
    for (int t = 0; t < a.n_ref; ++t) {   // the recorded refinement moves (Q23), same centroid order
        float cx, cy, cz;
        pose_centroid<AC, LPP>(buf, A, lane & (LPP - 1), cx, cy, cz);
        const int bm = ang[a.S_w * R + t];
        if (bm != 0) {
            const RotT Ms = rigid_t(a.ref_tab + 12 * bm, cx, cy, cz, pk.inv_h);
            for (int j = lane; j < A; j += 32) {
                const float4 v = buf.get(j);
                buf.set(j, apply_rot(Ms, v.x, v.y, v.z));
            }
        }
        __syncwarp();
    }
    const int64_t a0 = a.atom_off[li];
    float* out = xyz_out + 3 * a0;
    const uint8_t* ord = a.order + a0;
    for (int i = lane; i < A; i += 32) {
        const float4 v = buf.get(i);
        const int q = ord[i];
        out[3 * q] = __fmaf_rn(pk.h, v.x, pk.ox);
        out[3 * q + 1] = __fmaf_rn(pk.h, v.y, pk.oy);
        out[3 * q + 2] = __fmaf_rn(pk.h, v.z, pk.oz);
    }
    __syncwarp();
}

// a9 best pose of one round (run by the warp that completes the round's last item), and its
// coordinates (replayed on the warp's first pose buffer, free once its item completed).
template <int AC, int LPP>
__device__ __forceinline__ void finish_round(const DockArgs& a, const PocketDev& pk, const SiteOut& so,
                                             const unsigned char* slot, const DockLayout& L, int round, PoseBuf<AC> buf,
                                             int lane) {
    const int LC = a.ligs_per_cta, P = a.P, S_w = a.S_w;
    const int nl = min(LC, a.n - round * LC);
    const int4* sMeta = reinterpret_cast<const int4*>(slot + L.meta_o);
    const float* sScore = reinterpret_cast<const float*>(slot + L.score_o);
    const uint8_t* sAng = slot + L.ang_o;
    const float* sRec = reinterpret_cast<const float*>(slot + L.rec_o);
    const int ang_stride = dock_ang_stride(S_w, a.frag_cap, a.n_ref);
    for (int l = 0; l < nl; ++l) {   // lowest score, ties -> lowest pose index (Q11)
        const int4 m = sMeta[l];
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
            so.best_score[li] = sScore[l * P + bp];
            so.best_pose[li] = bp;
        }
        const uint8_t* sa = sAng + (size_t)(l * P + bp) * ang_stride;
        for (int t = lane; t < nang; t += 32) so.angles[m.w + t] = sa[t];
        if (so.dbg_score)
            for (int p = lane; p < P; p += 32) so.dbg_score[(size_t)li * P + p] = sScore[l * P + p];
        if (so.dbg_angles)
            for (int t = lane; t < P * nang; t += 32) {
                const int p = t / nang, q = t - p * nang;
                so.dbg_angles[(size_t)P * m.w + t] = sAng[(size_t)(l * P + p) * ang_stride + q];
            }
        if (so.refine)
            for (int t = lane; t < a.n_ref; t += 32) so.refine[(size_t)li * a.n_ref + t] = sa[nang + t];
        if (so.dbg_refine)
            for (int t = lane; t < P * a.n_ref; t += 32) {
                const int p = t / a.n_ref, q = t - p * a.n_ref;
                so.dbg_refine[(size_t)li * P * a.n_ref + t] = sAng[(size_t)(l * P + p) * ang_stride + nang + q];
            }
        if (so.xyz_out)
            replay_coords<AC, LPP>(a, pk, so.xyz_out, sRec + (size_t)l * a.rec_floats, li, m.y, R, bp, sa, buf, lane);
    }
}

// Persistent CTA per SM.  Warps run independently (no CTA barrier after the prologue):
// each claims warp items (round sequence, ligand of the round, PPW-pose group) from a
// CTA-local counter; rounds sit in a ring of kDockSlots slots.  The warp that claims the
// middle item of round s loads round s + 1 once round s is staged (so records are staged
// long before use and global rounds are claimed in sequence order), the
// warp that completes the last item of a round reduces its best pose (a9) and frees the
// slot.  NW is therefore free of P / PPW (e.g. 12 warps of 4 poses for 64 poses).
// MS = fused multi-site launch: the kernel runs as thread-block clusters of
// a.n_sites CTAs, CTA rank s docking into pocket s with that pocket's grid in ITS shared memory.
// Rank 0 claims the rounds and stages each round's records ONCE for the whole cluster (multicast
// TMA into the same slot of every CTA); a slot is reused only after every CTA released it.
template <int AC, int NW, int PPW, int GM, int KT, bool MS>
__global__ void __launch_bounds__(NW * 32, 1) dock_kernel(const DockArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ DockRing ring;
    constexpr int LPP = 32 / PPW;
    const int site = MS ? (int)cluster_rank() : 0;
    const bool leader = !MS || site == 0;   // the CTA that claims and stages rounds
    const PocketDev& pk = a.pk[site];
    const SiteOut& so = a.out[site];
    const int LC = a.ligs_per_cta;
    const DockLayout L =
        dock_layout(AC, NW, PPW, GM, pk.nz, pk.rs, pk.ps, pk.nch, a.P, a.K, a.S_w, LC, a.frag_cap, a.n_ref);
    float* sG = reinterpret_cast<float*>(smem + L.grid);
    float* sBuf = reinterpret_cast<float*>(smem + L.buf);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, h = lane / LPP;
    auto slot_ptr = [&](int seq) { return smem + L.slots + (size_t)(seq % kDockSlots) * L.slot_b; };

    const int n_rounds = (a.n + LC - 1) / LC;
    if (tid < kDockSlots) {
        ring.ready[tid] = -1;
        ring.done[tid] = 0;
        ring.free_seq[tid] = tid;
        mbar_init(&ring.bar[tid], 1);
        if (MS) mbar_init(&ring.free_bar[tid], a.n_sites);
    }
    if (tid == 0) {
        ring.item = 0;
        ring.end_seq = 0x7fffffff;
        if (leader) ring.claim[0] = atomicAdd(a.counter, 1);
    }
    stage_grid(sG, pk, (L.buf - L.grid) / 4 + (size_t)NW * PPW * pose_stride_of(AC, NW, PPW));   // grid + pose buffers
    if (MS) {
        // every CTA's ring (mbarriers included) exists before rank 0 writes into it
        if (tid == 0) asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        cluster_sync_all();
    } else {
        __syncthreads();
    }
    if (warp == 0 && leader) load_round<AC, MS>(a, ring, slot_ptr(0), L, 0, n_rounds, lane);

    const int K = KT ? KT : a.K, S_w = a.S_w, P = a.P;
    const int kbits = K > 1 ? 32 - __clz(K - 1) : 0;   // log2 of Kp, the next power of two >= K
    const int kl = lane & ((1 << kbits) - 1);          // this lane's angle slot
    const float ck = kl < K ? a.cs[2 * kl] : 1.f, sk = kl < K ? a.cs[2 * kl + 1] : 0.f;   // slots >= K: identity
    const PoseBuf<AC> buf{sBuf + (warp * PPW + h) * pose_stride_of(AC, NW, PPW)};
    const int ang_stride = dock_ang_stride(S_w, a.frag_cap, a.n_ref);
    const int G = (P + PPW - 1) / PPW;   // warp items per ligand
    const int IG = LC * G;               // warp items per round
    const int loader_item = IG / 2;

    while (true) {
        int t = 0;
        if (lane == 0) t = atomicAdd(&ring.item, 1);
        t = __shfl_sync(FULL, t, 0);
        const int seq = t / IG, it = t - seq * IG;
        // wait for the round's record (or for the launch to be exhausted)
        int ok = 0;
        if (lane == 0) {
            const int sl = seq % kDockSlots;
            unsigned spins = 0;
            while (true) {
                if ((MS ? ld_acquire_cluster(&ring.ready[sl]) : ld_acquire_cta(&ring.ready[sl])) == seq) {
                    ok = ring.round[sl] >= 0;
                    break;
                }
                if (*(volatile int*)&ring.end_seq <= seq) break;
                ring_backoff(spins);
            }
        }
        ok = __shfl_sync(FULL, ok, 0);
        __syncwarp();   // lane 0's acquire orders the slot reads of the whole warp
        if (!ok) break;
        {   // the record itself: TMA arrival on the slot's mbarrier (every lane acquires)
            unsigned spins = 0;
            const unsigned par = (unsigned)(seq / kDockSlots) & 1u;
            while (!(MS ? mbar_try_wait_cluster(&ring.bar[seq % kDockSlots], par) : mbar_try_wait(&ring.bar[seq % kDockSlots], par)))
                ring_backoff(spins);
        }
        // round s + 1 is claimed only once round s is (claims follow the sequence order, so
        // the first exhausted sequence bounds all later ones: end_seq is exact)
        if (it == loader_item && leader) load_round<AC, MS>(a, ring, slot_ptr(seq + 1), L, seq + 1, n_rounds, lane);
        unsigned char* slot = slot_ptr(seq);
        const int round = ring.round[seq % kDockSlots];
        const int nl = min(LC, a.n - round * LC);
        // items interleave the round's ligands (consecutive claims alternate between them), so
        // the warps of a CTA dock different ligands at once instead of running in lockstep
        const int l = it % LC, g = it / LC;
        if (l < nl) {
            const int p = g * PPW + h;
            const bool valid = p < P;
            const int pc = valid ? p : P - 1;
            const int4 m = reinterpret_cast<const int4*>(slot + L.meta_o)[l];
            const float* rec = reinterpret_cast<const float*>(slot + L.rec_o) + l * a.rec_floats;
            float* sScore = reinterpret_cast<float*>(slot + L.score_o);
            uint8_t* sAng = slot + L.ang_o;
            float T[12];   // pose p in grid units, from the raw table (48 B, L1-resident)
            scaled_pose(a.pose_tab + 12 * pc, pk, T);
            dock_poses<AC, PPW, GM, KT>(rec, m.y, m.z, T, valid, buf, sG, pk, K, kbits, S_w, ck, sk, a.n_ref, a.n_moves,
                                        a.ref_tab,
                                        sAng + (size_t)(l * P + pc) * ang_stride, sScore + l * P + pc, lane);
        }
        __syncwarp();
        int last = 0;
        if (lane == 0) {
            __threadfence_block();
            last = atomicAdd(&ring.done[seq % kDockSlots], 1) == IG - 1;
            if (last) __threadfence_block();
        }
        last = __shfl_sync(FULL, last, 0);
        __syncwarp();   // lane 0's fence after the counter orders the round reads of the whole warp
        if (last) {
            finish_round<AC, LPP>(a, pk, so, slot, L, round, PoseBuf<AC>{sBuf + (warp * PPW) * pose_stride_of(AC, NW, PPW)},
                             lane);
            __syncwarp();
            if (lane == 0) {
                ring.done[seq % kDockSlots] = 0;
                if (MS) mbar_arrive_remote(mapa(&ring.free_bar[seq % kDockSlots], 0));   // released by this CTA
                else st_release_cta(&ring.free_seq[seq % kDockSlots], seq + kDockSlots);
            }
        }
    }
    // MS: rank 0 keeps writing into the other CTAs' rings (and they arrive on its free barriers)
    // until the launch is exhausted -- nobody leaves before everybody is done
    if (MS) cluster_sync_all();
}

template <int GM>
__global__ void __launch_bounds__(1024) score_points_kernel(const PocketDev pk, const float* __restrict__ xyz,
                                                            const uint8_t* __restrict__ types, int64_t n,
                                                            float* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem[];
    float* sG = reinterpret_cast<float*>(smem);
    stage_grid(sG, pk, dock_grid_floats(GM == kGridFix ? kGridRT : GM, pk.nz, pk.rs, pk.ps, pk.nch));
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float ux = __fmul_rn(__fsub_rn(xyz[3 * i], pk.ox), pk.inv_h);
        const float uy = __fmul_rn(__fsub_rn(xyz[3 * i + 1], pk.oy), pk.inv_h);
        const float uz = __fmul_rn(__fsub_rn(xyz[3 * i + 2], pk.oz), pk.inv_h);
        out[i] = grid_g<GM>(sG, ux, uy, uz, pk, types ? types[i] : 0);
    }
}

using DockFn = void (*)(const DockArgs);

template <int AC, int GM>
DockFn pick_ac(int NW, int PPW, int K, bool ms) {
    if (ms) {   // fused multi-site launches: the production lane map only (FIX / QUAD grids, PPW 4, K 8)
        if constexpr (GM == kGridFix || GM == kGridQuad) {
            if (PPW != 4 || K != 8) return nullptr;
            if constexpr (GM == kGridQuad) {
                if constexpr (AC <= 96) if (NW == 20) return dock_kernel<AC, 20, 4, GM, 8, true>;
                if constexpr (AC == 128) if (NW == 18) return dock_kernel<AC, 18, 4, GM, 8, true>;
                if constexpr (AC == 160) if (NW == 15) return dock_kernel<AC, 15, 4, GM, 8, true>;
            }
            return NW == 16 ? dock_kernel<AC, 16, 4, GM, 8, true>
                   : NW == 13 ? dock_kernel<AC, 13, 4, GM, 8, true>
                   : NW == 12 ? dock_kernel<AC, 12, 4, GM, 8, true>
                   : NW == 10 ? dock_kernel<AC, 10, 4, GM, 8, true>
                              : (NW == 8 ? dock_kernel<AC, 8, 4, GM, 8, true> : nullptr);
        } else {
            return nullptr;
        }
    }
    if constexpr (typed_mode(GM)) {   // typed launches (Q24): the 4-poses-per-warp lane maps only
        if (PPW != 4) return nullptr;
        if (K == 8)
            return NW == 16 ? dock_kernel<AC, 16, 4, GM, 8, false>
                   : NW == 13 ? dock_kernel<AC, 13, 4, GM, 8, false>
                   : NW == 12 ? dock_kernel<AC, 12, 4, GM, 8, false>
                   : NW == 10 ? dock_kernel<AC, 10, 4, GM, 8, false>
                              : (NW == 8 ? dock_kernel<AC, 8, 4, GM, 8, false> : (NW == 4 ? dock_kernel<AC, 4, 4, GM, 8, false> : nullptr));
        return NW == 16 ? dock_kernel<AC, 16, 4, GM, 0, false>
               : NW == 13 ? dock_kernel<AC, 13, 4, GM, 0, false>
               : NW == 12 ? dock_kernel<AC, 12, 4, GM, 0, false>
               : NW == 10 ? dock_kernel<AC, 10, 4, GM, 0, false>
                          : (NW == 8 ? dock_kernel<AC, 8, 4, GM, 0, false> : (NW == 4 ? dock_kernel<AC, 4, 4, GM, 0, false> : nullptr));
    } else {   // (else: typed layouts instantiate none of the lane maps below)
    if constexpr (GM == kGridQuad) {   // more warps where shared memory allows (latency hiding)
        if (PPW == 4 && K == 8) {
            if constexpr (AC <= 96) if (NW == 20) return dock_kernel<AC, 20, 4, GM, 8, false>;
            if constexpr (AC == 128) if (NW == 18) return dock_kernel<AC, 18, 4, GM, 8, false>;
            if constexpr (AC == 160) if (NW == 15) return dock_kernel<AC, 15, 4, GM, 8, false>;
        }
    }
    if (PPW == 4 && K == 8 && GM != kGridRT)   // production path: compile-time K = 8
        return NW == 16 ? dock_kernel<AC, 16, 4, GM, 8, false>
               : NW == 13 ? dock_kernel<AC, 13, 4, GM, 8, false>
               : NW == 12 ? dock_kernel<AC, 12, 4, GM, 8, false>
               : NW == 10 ? dock_kernel<AC, 10, 4, GM, 8, false>
                          : (NW == 8 ? dock_kernel<AC, 8, 4, GM, 8, false> : (NW == 4 ? dock_kernel<AC, 4, 4, GM, 8, false> : nullptr));
    if (PPW == 1) return NW == 32 ? dock_kernel<AC, 32, 1, GM, 0, false> : (NW == 16 ? dock_kernel<AC, 16, 1, GM, 0, false> : nullptr);
    if (PPW == 2)
        return NW == 32 ? dock_kernel<AC, 32, 2, GM, 0, false>
                        : (NW == 16 ? dock_kernel<AC, 16, 2, GM, 0, false> : (NW == 8 ? dock_kernel<AC, 8, 2, GM, 0, false> : nullptr));
    if (PPW == 4)
        return NW == 16 ? dock_kernel<AC, 16, 4, GM, 0, false>
               : NW == 13 ? dock_kernel<AC, 13, 4, GM, 0, false>
               : NW == 12 ? dock_kernel<AC, 12, 4, GM, 0, false>
               : NW == 10 ? dock_kernel<AC, 10, 4, GM, 0, false>
                          : (NW == 8 ? dock_kernel<AC, 8, 4, GM, 0, false> : (NW == 4 ? dock_kernel<AC, 4, 4, GM, 0, false> : nullptr));
    }
    return nullptr;
}

// Per-atom-class entry points, each compiled in its own translation unit
// (dock_inst.cu with -DVSD_AC=<AC>) so the 8 classes build in parallel.
#define VSD_DECL_CLASS(ac)                                                                                     \
    DockFn dock_pick_##ac(int gmode, int NW, int PPW, int K, bool ms);                                                           \

VSD_DECL_CLASS(32)
VSD_DECL_CLASS(64)
VSD_DECL_CLASS(96)
VSD_DECL_CLASS(128)
VSD_DECL_CLASS(160)
VSD_DECL_CLASS(192)
VSD_DECL_CLASS(224)
VSD_DECL_CLASS(256)
#undef VSD_DECL_CLASS

}  // namespace dk
}  // namespace vsd
