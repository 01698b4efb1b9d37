// prep.cu -- the paper's out-of-kernel input preparation on the GPU (a1-a5):
// ingest (validation, laminar check, canonical atom renumbering) + features, classification into (atom class x rotamer class)
// cells, a STABLE counting sort by cell (histogram -> scan -> scatter), exact
// per-bucket work for the LPT shard, and packing into SoA-padded records.
//
// PAPER.md l.206-240 (runtime input preparation that "collects the ligands in
// buckets before virtual screening them", l.219-220)
// (assignment and bucket membership); readings Q16-Q18, Q21.
#include <cuda_runtime.h>
#include <cstdint>

#include "internal.h"

namespace vsd {

namespace {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ int warp_sum_int(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

// a1: ingest.  One warp per ligand (grid-stride).  Validates the ligand record in the
// C-ABI's general form (axis (a, b) and the moving-atom SET M_r of every fragment,
// PAPER.md l.215-216 "a subset of the molecule atoms that can rotate"), checks that the
// moving sets form a laminar family (any two are nested or disjoint -- what rotations
// about the bonds of a tree produce), and renumbers the atoms into the canonical
// internal order in which every M_r is ONE contiguous range [lo, hi):
//
//   * the sets form a forest under inclusion (equal sets: the lower fragment index is the
//     outer one); the forest is ordered depth first, children by fragment index (preorder
//     number pre[r]);
//   * atom i's key = (1 + pre of the innermost set containing it, or 0 for atoms in no set)
//     in the top 6 bits, then a 58-bit mix of its coordinate bits; ties by input index.
//     Sorting by the key puts each set's own atoms first and its descendants' atoms right
//     after them, so every set is contiguous.  The key does not depend on the input atom
//     numbering (only on coordinates and set structure), so an atom-permuted copy of a
//     ligand is docked bit-identically (coordinates are mapped back to input order; only
//     two atoms of one region with colliding 58-bit mixes -- e.g. identical coordinates --
//     fall back to the input order, which then cannot change any sum).
//
// Outputs: order[atom_off[i] + j] = input index of internal atom j (u8); frint[f] =
// {a', b', lo, hi} in internal numbering (the range form the pack / dock kernels use);
// features A, R, sum |M_r|.  Error codes (low byte of the status word; lowest ligand index
// wins through atomicMin on (index << 8 | code); within a ligand the first failing check):
//  1 atoms outside [1, 256]            2 fragments outside [0, 32]
//  3 non-finite coordinate             12 coordinate magnitude above 1e6 A
//  4 axis atom index out of range      5 axis atoms equal
//  6 moving set empty or larger than A - 2
//  8 axis atoms closer than 1e-3 A     9 moving atom index out of range
//  10 atom listed twice in one moving set
//  7 axis atom inside its own moving set
//  11 moving sets not laminar (two sets overlap without one containing the other)
//  13 atom type >= the grid channels of a docked pocket (typed submits, Q24)
// a1 (all ligands): features from the CSR offsets alone -- A, R, sum |M_r| -- and the two
// range checks every rank must agree on before the plan (codes 1, 2 below).  The per-atom
// checks and the renumbering (ingest_kernel) run only on the ligands this rank docks.
__global__ void __launch_bounds__(256) features_kernel(const int64_t* __restrict__ atom_off,
                                                       const int64_t* __restrict__ frag_off,
                                                       const int64_t* __restrict__ move_off, int64_t n,
                                                       int* __restrict__ featA, int* __restrict__ featR,
                                                       int* __restrict__ featM, unsigned long long* status,
                                                       int* maxAR) {
    __shared__ int smax[3];
    if (threadIdx.x < 3) smax[threadIdx.x] = 0;
    __syncthreads();
    int locA = 0, locR = 0, locM = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t A64 = atom_off[i + 1] - atom_off[i];
        const int64_t f0 = frag_off[i], f1 = frag_off[i + 1];
        const int64_t R64 = f1 - f0;
        int code = 0;
        if (A64 < 1 || A64 > kMaxAtoms) code = 1;
        else if (R64 < 0 || R64 > kMaxFrags) code = 2;
        int64_t M = 0;
        if (code == 0) {
            M = R64 > 0 ? move_off[f1] - move_off[f0] : 0;
            locA = max(locA, (int)A64);
            locR = max(locR, (int)R64);
            locM = max(locM, (int)(M > 0x7fffffff ? 0x7fffffff : M));
        }
        featA[i] = (int)(A64 > 0x7fffffff ? 0x7fffffff : (A64 < 0 ? 0 : A64));
        featR[i] = (int)(R64 > 0x7fffffff ? 0x7fffffff : (R64 < 0 ? 0 : R64));
        featM[i] = (int)(M < 0 ? 0 : (M > 0x7fffffff ? 0x7fffffff : M));
        if (code) atomicMin(status, ((unsigned long long)i << 8) | (unsigned long long)code);
    }
    atomicMax(&smax[0], locA);
    atomicMax(&smax[1], locR);
    atomicMax(&smax[2], locM);
    __syncthreads();
    if (threadIdx.x == 0) {
        atomicMax(&maxAR[0], smax[0]);
        atomicMax(&maxAR[1], smax[1]);
        atomicMax(&maxAR[2], smax[2]);
    }
}

// Packed slot -> (owned bucket, ligand index): owned_prefix[b] <= slot < owned_prefix[b+1].
__device__ __forceinline__ uint32_t slot_ligand(int slot, const uint32_t* __restrict__ perm,
                                                const int64_t* __restrict__ owned_start,
                                                const int* __restrict__ owned_prefix, int n_owned, int* bucket) {
    int lo = 0, hi = n_owned;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (owned_prefix[mid] <= slot) lo = mid;
        else hi = mid;
    }
    if (bucket) *bucket = lo;
    return perm[owned_start[lo] + (slot - owned_prefix[lo])];
}

constexpr int kIngestWarps = 8;
struct IngestWarp {
    uint32_t mask[kMaxAtoms];           // bit r: atom in M_r
    unsigned long long key[kMaxAtoms];  // (1 + pre) << 58 | coordinate mix
    uint8_t path[kMaxFrags][kMaxFrags + 1];   // path[r][d]: ancestor of r at depth d (r itself at depth[r])
    uint32_t anc[kMaxFrags];
    uint8_t depth[kMaxFrags], pre[kMaxFrags];
    uint8_t rank[kMaxAtoms];            // input index -> internal position
    uint8_t list[kMaxAtoms];            // atoms grouped by region (key >> 58)
    int rstart[kMaxFrags + 2], rfill[kMaxFrags + 2];   // region start / fill cursor
    int moff[kMaxFrags + 1];            // the ligand's moving-atom entries of fragment r: [moff[r], moff[r+1])
    uint32_t sup[kMaxFrags], inter[kMaxFrags];
    int lo[kMaxFrags], hi[kMaxFrags];
};

// Fragment of moving-atom entry t of the ligand (moff strictly increasing: every set non-empty).
__device__ __forceinline__ int frag_of(const int* moff, int R, int t) {
    int lo = 0, hi = R;   // moff[lo] <= t < moff[hi]
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (moff[mid] <= t) lo = mid;
        else hi = mid;
    }
    return lo;
}

// 58-bit mix of an atom's coordinate bits (-0 canonicalised to +0): a canonical tie-break
// among the free atoms of one set region that does not depend on the input numbering.
__device__ __forceinline__ unsigned long long coord_mix(float x, float y, float z) {
    unsigned long long h = 0x9E3779B97F4A7C15ull;
    const float v[3] = {x, y, z};
#pragma unroll
    for (int t = 0; t < 3; ++t) {
        h ^= (unsigned long long)__float_as_uint(__fadd_rn(v[t], 0.0f)) + 0x632BE59BD9B4E019ull * (t + 1);
        h = (h ^ (h >> 30)) * 0xBF58476D1CE4E5B9ull;
        h = (h ^ (h >> 27)) * 0x94D049BB133111EBull;
        h ^= h >> 31;
    }
    return h >> 6;
}
__device__ __forceinline__ int first_code(int code) {   // lowest lane's non-zero code
    const unsigned any = __ballot_sync(FULL, code != 0);
    return any ? __shfl_sync(FULL, code, __ffs(any) - 1) : 0;
}

__global__ void __launch_bounds__(kIngestWarps * 32) ingest_kernel(
    const int64_t* __restrict__ atom_off, const float* __restrict__ xyz, const uint8_t* __restrict__ atom_type,
    int n_types, const int64_t* __restrict__ frag_off,
    const int32_t* __restrict__ frag_axis, const int64_t* __restrict__ move_off, const int32_t* __restrict__ move_atoms,
    const uint32_t* __restrict__ perm, const int64_t* __restrict__ owned_start, const int* __restrict__ owned_prefix,
    int n_owned, int total_slots, uint8_t* __restrict__ order, int4* __restrict__ frint, uint8_t* __restrict__ fown,
    int* __restrict__ lflag, unsigned long long* status) {
    __shared__ IngestWarp sw[kIngestWarps];
    const int lane = threadIdx.x & 31;
    IngestWarp& W = sw[threadIdx.x >> 5];
    const int warps = gridDim.x * kIngestWarps;
    for (int slot = blockIdx.x * kIngestWarps + (threadIdx.x >> 5); slot < total_slots; slot += warps) {
        const int64_t li = slot_ligand(slot, perm, owned_start, owned_prefix, n_owned, nullptr);
        const int64_t a0 = atom_off[li], a1 = atom_off[li + 1];
        const int64_t f0 = frag_off[li], f1 = frag_off[li + 1];
        const int64_t A64 = a1 - a0, R64 = f1 - f0;
        int code = 0, M = 0;
        if (A64 < 1 || A64 > kMaxAtoms) code = 1;
        else if (R64 < 0 || R64 > kMaxFrags) code = 2;
        const int A = (int)A64, R = (int)R64;
        const float* x = xyz + 3 * a0;
        if (code == 0) {   // coordinates: finite and physically bounded (|x| <= 1e6 A)
            bool nf = false, big = false;
            for (int t = lane; t < 3 * A; t += 32) {
                const float v = x[t];
                nf |= !isfinite(v);
                big |= fabsf(v) > 1e6f;
            }
            if (__any_sync(FULL, nf)) code = 3;
            else if (__any_sync(FULL, big)) code = 12;
        }
        if (code == 0 && atom_type) {   // Q24: every atom type names a channel of every docked pocket
            bool bad = false;
            for (int t = lane; t < A; t += 32) bad |= atom_type[a0 + t] >= n_types;
            if (__any_sync(FULL, bad)) code = 13;
        }
        int fa = 0, fb = 0;
        int64_t m0 = 0;
        int cnt = 0;
        if (code == 0) {   // per fragment: axis, moving-set size, axis length
            int fc = 0;
            if (lane < R) {
                const int64_t f = f0 + lane;
                fa = frag_axis[2 * f];
                fb = frag_axis[2 * f + 1];
                m0 = move_off[f];
                const int64_t c64 = move_off[f + 1] - m0;
                cnt = (int)(c64 < 0 ? -1 : (c64 > kMaxAtoms ? kMaxAtoms + 1 : c64));
                if (fa < 0 || fa >= A || fb < 0 || fb >= A) fc = 4;
                else if (fa == fb) fc = 5;
                else if (cnt < 1 || cnt > A - 2 || m0 < 0) fc = 6;
                else {
                    const float dx = __fsub_rn(x[3 * fb], x[3 * fa]), dy = __fsub_rn(x[3 * fb + 1], x[3 * fa + 1]),
                                dz = __fsub_rn(x[3 * fb + 2], x[3 * fa + 2]);
                    if (dx * dx + dy * dy + dz * dz < 1e-6f) fc = 8;
                }
            }
            code = first_code(fc);
        }
        // the ligand's moving-atom entries are one contiguous range of move_atoms (CSR): the
        // passes below run flat over it, each entry finding its fragment by binary search
        const int64_t mbase = R > 0 ? __shfl_sync(FULL, m0, 0) : 0;
        int total = 0;
        if (code == 0) {   // membership masks; index range and duplicates
            for (int i = lane; i < A; i += 32) W.mask[i] = 0u;
            if (lane < R) W.moff[lane] = (int)(m0 - mbase);
            if (lane == 0) W.moff[R] = 0;
            __syncwarp();
            if (R > 0 && lane == R - 1) W.moff[R] = (int)(m0 - mbase) + cnt;
            __syncwarp();
            total = W.moff[R];
            bool oob = false, dup = false;
            for (int t = lane; t < total; t += 32) {
                const int r = frag_of(W.moff, R, t);
                const int i = move_atoms[mbase + t];
                if (i < 0 || i >= A) oob = true;
                else if (atomicOr(&W.mask[i], 1u << r) & (1u << r)) dup = true;
            }
            if (__any_sync(FULL, oob)) code = 9;
            else if (__any_sync(FULL, dup)) code = 10;
            __syncwarp();
        }
        if (code == 0) {   // axis atoms stay outside their own moving set
            const bool in = lane < R && (((W.mask[fa] | W.mask[fb]) >> lane) & 1u);
            if (__any_sync(FULL, in)) code = 7;
        }
        uint32_t sup = 0, sub = 0;
        const uint32_t valid = R == 32 ? 0xffffffffu : ((1u << R) - 1u);
        if (code == 0) {
            // laminar family: sup_r = {s : M_r within M_s} (AND of the members' masks),
            // inter_r = {s : M_s meets M_r} (OR); sub_r = {s : M_s within M_r} (transpose of sup).
            // Laminar iff every set meeting M_r contains it or is contained in it.
            if (lane < R) {
                W.sup[lane] = 0xffffffffu;
                W.inter[lane] = 0u;
            }
            __syncwarp();
            for (int t = lane; t < total; t += 32) {
                const int r = frag_of(W.moff, R, t);
                const uint32_t m = W.mask[move_atoms[mbase + t]];
                atomicAnd(&W.sup[r], m);
                atomicOr(&W.inter[r], m);
            }
            __syncwarp();
            uint32_t inter = 0;
            if (lane < R) {
                sup = W.sup[lane] & valid;
                inter = W.inter[lane] & valid;
            }
            for (int r = 0; r < R; ++r) {
                const uint32_t col = __ballot_sync(FULL, lane < R && ((sup >> r) & 1u));
                if (lane == r) sub = col;
            }
            const bool bad = lane < R && (inter & ~(sup | sub)) != 0u;
            if (__any_sync(FULL, bad)) code = 11;
        }
        if (code == 0) {
            // forest under inclusion: s is an ancestor of r if M_r is strictly inside M_s, or the
            // sets are equal and s < r.  depth = number of ancestors; path[r][d] = the ancestor
            // (or r itself) at depth d.
            uint32_t anc = 0;
            int dep = 0;
            if (lane < R) {
                const uint32_t eq = sup & sub;   // sets equal to M_r (r included)
                anc = (sup & ~eq) | (eq & ((1u << lane) - 1u));
                dep = __popc(anc);
                W.anc[lane] = anc;
                W.depth[lane] = (uint8_t)dep;
            }
            __syncwarp();
            if (lane < R) {
                uint32_t chain = anc | (1u << lane);
                while (chain) {
                    const int s2 = __ffs(chain) - 1;
                    chain &= chain - 1u;
                    W.path[lane][W.depth[s2]] = (uint8_t)s2;
                }
            }
            __syncwarp();
            // preorder number: s comes before r if s is an ancestor of r, or, below their
            // deepest common ancestor, s's branch has the lower fragment index
            if (lane < R) {
                int pre = 0;
                for (int s2 = 0; s2 < R; ++s2) {
                    if (s2 == lane) continue;
                    const uint32_t as = W.anc[s2];
                    bool before;
                    if ((anc >> s2) & 1u) before = true;
                    else if ((as >> lane) & 1u) before = false;
                    else {
                        const int dc = __popc(anc & as);
                        before = W.path[s2][dc] < W.path[lane][dc];
                    }
                    pre += before;
                }
                W.pre[lane] = (uint8_t)pre;
            }
            __syncwarp();
            // atom keys; region histogram (region = 1 + pre of the innermost set, 0 = none)
            for (int t = lane; t < R + 1; t += 32) W.rfill[t] = 0;
            __syncwarp();
            for (int i = lane; i < A; i += 32) {
                uint32_t m = W.mask[i], k0 = 0;
                if (m) {
                    int best = -1, bd = -1;
                    while (m) {
                        const int r = __ffs(m) - 1;
                        m &= m - 1u;
                        if ((int)W.depth[r] > bd) {
                            bd = W.depth[r];
                            best = r;
                        }
                    }
                    k0 = 1u + W.pre[best];
                }
                W.key[i] = ((unsigned long long)k0 << 58) | coord_mix(x[3 * i], x[3 * i + 1], x[3 * i + 2]);
                atomicAdd(&W.rfill[k0], 1);
            }
            __syncwarp();
            if (lane == 0) {
                int run = 0;
                for (int t = 0; t <= R; ++t) {
                    W.rstart[t] = run;
                    run += W.rfill[t];
                    W.rfill[t] = W.rstart[t];
                }
            }
            __syncwarp();
            for (int i = lane; i < A; i += 32) W.list[atomicAdd(&W.rfill[(int)(W.key[i] >> 58)], 1)] = (uint8_t)i;
            __syncwarp();
            // rank = region start + rank by counting inside the region (the region's members
            // only: sum of squared region sizes instead of A^2 comparisons)
            const int nu = (A + 31) >> 5;
            int rk[kMaxAtoms / 32];
#pragma unroll
            for (int u = 0; u < kMaxAtoms / 32; ++u) {
                const int i = lane + 32 * u;
                rk[u] = 0;
                if (u < nu && i < A) {
                    const unsigned long long ki = W.key[i];
                    const int rg = (int)(ki >> 58);
                    const int b = W.rstart[rg], e = rg < R ? W.rstart[rg + 1] : A;
                    int c = b;
                    for (int t = b; t < e; ++t) {
                        const int j = W.list[t];
                        const unsigned long long kj = W.key[j];
                        c += (kj < ki) | ((kj == ki) & (j < i));
                    }
                    rk[u] = c;
                }
            }
#pragma unroll
            for (int u = 0; u < kMaxAtoms / 32; ++u) {
                const int i = lane + 32 * u;
                if (i < A) {
                    W.rank[i] = (uint8_t)rk[u];
                    order[a0 + rk[u]] = (uint8_t)i;
                }
            }
            __syncwarp();
            // internal fragments: every moving set is now the range [min rank, max rank + 1)
            if (lane < R) {
                W.lo[lane] = kMaxAtoms;
                W.hi[lane] = -1;
            }
            __syncwarp();
            for (int t = lane; t < total; t += 32) {
                const int r = frag_of(W.moff, R, t);
                const int q = W.rank[move_atoms[mbase + t]];
                atomicMin(&W.lo[r], q);
                atomicMax(&W.hi[r], q);
            }
            __syncwarp();
            if (lane < R) {
                frint[f0 + lane] = make_int4(W.rank[fa], W.rank[fb], W.lo[lane], W.hi[lane] + 1);
                // own region of r: the atoms whose innermost set is r -- the first own atoms of
                // its range (preorder), final after step r when no ancestor sweeps later
                const int rg = 1 + W.pre[lane];
                fown[f0 + lane] = (uint8_t)(W.rfill[rg] - W.rstart[rg]);
            }
            // ancestors-first fragment order (every ancestor of r has a lower index): the dock
            // kernel then finalises each own region in the sweep
            const bool anc_first = __all_sync(FULL, lane >= R || (W.anc[lane] >> lane) == 0u);
            if (lane == 0) lflag[li] = (W.rfill[0] - W.rstart[0]) | (anc_first ? (1 << 16) : 0);
            M = total;
            __syncwarp();
        }
        (void)M;
        if (lane == 0 && code) atomicMin(status, ((unsigned long long)li << 8) | (unsigned long long)code);
    }
}

struct Bounds {
    int atom_b[kMaxAtomClasses];
    int rot_b[kMaxRotClasses];
    int move_b[kMaxMoveClasses];
    int n_atom_b, n_rot_b, n_move_b;
};

// a2: cell = (atom_class * n_rot + rot_class) * n_move + move_class; each class index is the
// smallest i with value <= boundary[i]; the third key (sum_r |M_r|) is
// off with one move class.  Block-local histogram -> hist[cell][block].
__global__ void __launch_bounds__(1024) classify_hist_kernel(const int* __restrict__ featA,
                                                             const int* __restrict__ featR,
                                                             const int* __restrict__ featM, int64_t n, Bounds bd,
                                                             int* __restrict__ cell, int* __restrict__ hist,
                                                             int n_blocks, unsigned long long* ovf) {
    __shared__ int h[kMaxCells];
    const int n_cells = bd.n_atom_b * bd.n_rot_b * bd.n_move_b;
    for (int c = threadIdx.x; c < n_cells; c += blockDim.x) h[c] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kPrepTile;
    for (int t = threadIdx.x; t < kPrepTile; t += blockDim.x) {
        const int64_t i = base + t;
        if (i >= n) break;
        const int A = featA[i], R = featR[i], M = featM[i];
        int ai = 0, ri = 0, mi = 0;
        while (ai < bd.n_atom_b && A > bd.atom_b[ai]) ++ai;
        while (ri < bd.n_rot_b && R > bd.rot_b[ri]) ++ri;
        while (mi < bd.n_move_b && M > bd.move_b[mi]) ++mi;
        int c = -1;
        if (ai == bd.n_atom_b) atomicMin(ovf, ((unsigned long long)i << 8) | 1ull);
        else if (ri == bd.n_rot_b) atomicMin(ovf, ((unsigned long long)i << 8) | 2ull);
        else if (mi == bd.n_move_b) atomicMin(ovf, ((unsigned long long)i << 8) | 3ull);
        else {
            c = (ai * bd.n_rot_b + ri) * bd.n_move_b + mi;
            atomicAdd(&h[c], 1);
        }
        cell[i] = c;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < n_cells; c += blockDim.x) hist[(int64_t)c * n_blocks + blockIdx.x] = h[c];
}

// a3 (scan): per-cell totals, then an exclusive scan of hist (cell-major) in place:
// hist[c][b] becomes the first output position of block b's cell-c ligands.
__global__ void __launch_bounds__(1024) scan_hist_kernel(int* __restrict__ hist, int n_cells, int n_blocks,
                                                         int* __restrict__ cell_count) {
    __shared__ int wsum[32];
    for (int c = threadIdx.x; c < n_cells; c += blockDim.x) {
        int s = 0;
        for (int b = 0; b < n_blocks; ++b) s += hist[(int64_t)c * n_blocks + b];
        cell_count[c] = s;
    }
    __syncthreads();
    const int64_t N = (int64_t)n_cells * n_blocks;
    const int64_t per = (N + blockDim.x - 1) / blockDim.x;
    const int64_t lo = threadIdx.x * per, hi = lo + per < N ? lo + per : N;
    int s = 0;
    for (int64_t j = lo; j < hi; ++j) s += hist[j];
    // block exclusive scan of s
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int v = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    if (w == 0) {
        int v = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
        int inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int u = __shfl_up_sync(FULL, inc, o);
            if (lane >= o) inc += u;
        }
        wsum[lane] = inc - v;
    }
    __syncthreads();
    int run = wsum[w] + incl - s;
    for (int64_t j = lo; j < hi; ++j) {
        const int v = hist[j];
        hist[j] = run;
        run += v;
    }
}

// a3 (scatter): stable -- inside a tile, rank among equal cells by index
// (warp match + popc, then warp-prefix per cell), tiles ordered by block.
__global__ void __launch_bounds__(1024) scatter_kernel(const int* __restrict__ cell, int64_t n,
                                                       const int* __restrict__ hist_off, int n_cells, int n_blocks,
                                                       uint32_t* __restrict__ perm) {
    extern __shared__ int scat_smem[];   // per-warp counts [32][n_cells] + running [n_cells]
    int* running = scat_smem + 32 * n_cells;
    auto wcnt = [&](int w, int c) -> int& { return scat_smem[w * n_cells + c]; };
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int c = threadIdx.x; c < n_cells; c += blockDim.x) running[c] = 0;
    const int64_t base = (int64_t)blockIdx.x * kPrepTile;
    for (int chunk = 0; chunk < kPrepTile; chunk += 1024) {
        for (int e = threadIdx.x; e < 32 * n_cells; e += blockDim.x) scat_smem[e] = 0;
        __syncthreads();
        const int64_t i = base + chunk + threadIdx.x;
        const int c = (i < n) ? cell[i] : -1;
        const unsigned peers = __match_any_sync(FULL, c);
        const int rank = __popc(peers & ((1u << lane) - 1u));
        if (c >= 0 && lane == __ffs(peers) - 1) wcnt(w, c) = __popc(peers);
        __syncthreads();
        for (int cc = threadIdx.x; cc < n_cells; cc += blockDim.x) {
            int run = running[cc];
            for (int ww = 0; ww < 32; ++ww) {
                const int t = wcnt(ww, cc);
                wcnt(ww, cc) = run;
                run += t;
            }
            running[cc] = run;
        }
        __syncthreads();
        if (c >= 0) perm[hist_off[(int64_t)c * n_blocks + blockIdx.x] + wcnt(w, c) + rank] = (uint32_t)i;
        __syncthreads();
    }
}

// a4 input: exact work of a bucket, sum of E_alg = P (A + S_w (K-1) sum|M_r|); also the
// bucket's atoms, fragments and moving-atom entries (bytes a rank reads for the buckets it
// owns, vs_stats): weights[4 b + {0, 1, 2, 3}] = {E, sum A, sum R, sum M}.
__global__ void __launch_bounds__(256) bucket_weights_kernel(const uint32_t* __restrict__ perm,
                                                             const int* __restrict__ featA,
                                                             const int* __restrict__ featR,
                                                             const int* __restrict__ featM,
                                                             const int64_t* __restrict__ bstart,
                                                             const int* __restrict__ bsize, long long P, long long K,
                                                             long long S_w, unsigned long long* __restrict__ weights) {
    __shared__ unsigned long long part[8][4];
    const int b = blockIdx.x;
    unsigned long long s[4] = {0, 0, 0, 0};
    for (int t = threadIdx.x; t < bsize[b]; t += blockDim.x) {
        const uint32_t li = perm[bstart[b] + t];
        s[0] += (unsigned long long)(P * ((long long)featA[li] + S_w * (K - 1) * (long long)featM[li]));
        s[1] += (unsigned long long)featA[li];
        s[2] += (unsigned long long)featR[li];
        s[3] += (unsigned long long)featM[li];
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s[q] += __shfl_xor_sync(FULL, s[q], o);
        if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5][q] = s[q];
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        unsigned long long t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += part[w][threadIdx.x];
        weights[4 * b + threadIdx.x] = t;
    }
}

// a5: one warp per packed slot.  Record layout (floats, rec_floats_of): x[AC] | y[AC] | z[AC] |
// frags u32[32] = a | b << 8 | lo << 16 | (hi - 1) << 24 | own-region lengths u8[32] |
// header u32 (n_root | ancestors-first << 16) + 3 pad words.  Coordinates are
// centred on the ligand centroid (a6, Q8); padding is 0.  The centroid sum is
// lane-strided then xor-reduced: an order that does not depend on AC (Q22).
__global__ void __launch_bounds__(256) pack_kernel(const uint32_t* __restrict__ perm,
                                                   const int64_t* __restrict__ owned_start,
                                                   const int* __restrict__ owned_prefix,
                                                   const int* __restrict__ owned_ac,
                                                   const int64_t* __restrict__ owned_rec_off, int n_owned,
                                                   int total_slots, const int64_t* __restrict__ atom_off,
                                                   const float* __restrict__ xyz,
                                                   const uint8_t* __restrict__ atom_type,
                                                   const uint8_t* __restrict__ order,
                                                   const int64_t* __restrict__ frag_off,
                                                   const int4* __restrict__ frint,
                                                   const uint8_t* __restrict__ fown,
                                                   const int* __restrict__ lflag, int S_w,
                                                   float* __restrict__ rec, int4* __restrict__ meta) {
    const int lane = threadIdx.x & 31;
    const int slot = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (slot >= total_slots) return;
    int b = 0;
    const uint32_t li = slot_ligand(slot, perm, owned_start, owned_prefix, n_owned, &b);
    const int s = slot - owned_prefix[b];
    const int AC = owned_ac[b];
    float* r = rec + owned_rec_off[b] + (int64_t)s * rec_floats_typed(AC, atom_type != nullptr);
    const int64_t a0 = atom_off[li];
    const int A = (int)(atom_off[li + 1] - a0);
    const int64_t f0 = frag_off[li];
    const int R = (int)(frag_off[li + 1] - f0);
    const float* x = xyz + 3 * a0;
    const uint8_t* ord = order + a0;   // internal atom i = input atom ord[i] (a1 canonical order)
    float px[kMaxAtoms / 32], py[kMaxAtoms / 32], pz[kMaxAtoms / 32];
    float sx = 0.f, sy = 0.f, sz = 0.f;
#pragma unroll
    for (int u = 0; u < kMaxAtoms / 32; ++u) {
        const int i = lane + 32 * u;
        if (i < A) {
            const int q = ord[i];
            px[u] = x[3 * q];
            py[u] = x[3 * q + 1];
            pz[u] = x[3 * q + 2];
            sx = __fadd_rn(sx, px[u]);
            sy = __fadd_rn(sy, py[u]);
            sz = __fadd_rn(sz, pz[u]);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        sx = __fadd_rn(sx, __shfl_xor_sync(FULL, sx, o));
        sy = __fadd_rn(sy, __shfl_xor_sync(FULL, sy, o));
        sz = __fadd_rn(sz, __shfl_xor_sync(FULL, sz, o));
    }
    const float fa = (float)A;
    const float cx = __fdiv_rn(sx, fa), cy = __fdiv_rn(sy, fa), cz = __fdiv_rn(sz, fa);
#pragma unroll
    for (int u = 0; u < kMaxAtoms / 32; ++u) {
        const int i = lane + 32 * u;
        if (i >= AC) break;
        const bool in = i < A;
        r[i] = in ? __fsub_rn(px[u], cx) : 0.f;
        r[AC + i] = in ? __fsub_rn(py[u], cy) : 0.f;
        r[2 * AC + i] = in ? __fsub_rn(pz[u], cz) : 0.f;
    }
    uint32_t f = 0;
    if (lane < R) {
        const int4 q = frint[f0 + lane];
        f = (uint32_t)q.x | ((uint32_t)q.y << 8) | ((uint32_t)q.z << 16) | ((uint32_t)(q.w - 1) << 24);
    }
    reinterpret_cast<uint32_t*>(r + 3 * AC)[lane] = f;
    // own-region lengths (bytes) and the header: n_root | ancestors-first << 16
    const uint8_t own = lane < R ? fown[f0 + lane] : (uint8_t)0;
    uint8_t* ob = reinterpret_cast<uint8_t*>(r + 3 * AC + 32);
    ob[lane] = own;
    if (lane < 4) reinterpret_cast<uint32_t*>(r + 3 * AC + 40)[lane] = lane == 0 ? (uint32_t)lflag[li] : 0u;
    if (atom_type) {   // typed record (Q24): the types in the canonical (internal) atom order, pads 0
        uint8_t* tb = reinterpret_cast<uint8_t*>(r + rec_floats_of(AC));
        for (int i = lane; i < AC; i += 32) tb[i] = i < A ? atom_type[a0 + ord[i]] : (uint8_t)0;
    }
    if (lane == 0) meta[slot] = make_int4((int)li, A, R, (int)(S_w * f0));
}

__global__ void fill_results_kernel(float* best_score, int* best_pose, int64_t n, uint8_t* angles, int64_t n_ang) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        best_score[i] = __int_as_float(0x7fc00000);
        best_pose[i] = -1;
    }
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_ang; i += stride) angles[i] = 0xFF;
}

// a10 keys: ord(score) << 32 | ligand index; ord is the order-preserving map of
// fp32 onto uint32 (sign-magnitude flip); -0 is canonicalised to +0.
__global__ void make_keys_kernel(const int4* __restrict__ meta, int n_slots, const float* __restrict__ best_score,
                                 unsigned long long* __restrict__ keys, uint32_t index_offset) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_slots) return;
    const int li = meta[s].x;
    const float v = __fadd_rn(best_score[li], 0.0f);
    const uint32_t bits = __float_as_uint(v);
    const uint32_t ord = (bits & 0x80000000u) ? ~bits : (bits | 0x80000000u);
    keys[s] = ((unsigned long long)ord << 32) | ((uint32_t)li + index_offset);
}

}  // namespace

__global__ void rebase_kernel(const int64_t* __restrict__ src, int64_t* __restrict__ dst, int64_t count, int64_t base) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i] - base;
}

cudaError_t launch_rebase(const int64_t* src, int64_t* dst, int64_t count, int64_t base, cudaStream_t st) {
    if (count <= 0) return cudaSuccess;
    int64_t blocks = (count + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    rebase_kernel<<<(int)blocks, 256, 0, st>>>(src, dst, count, base);
    return cudaGetLastError();
}

cudaError_t launch_features(const int64_t* atom_off, const int64_t* frag_off, const int64_t* move_off, int64_t n,
                            int* featA, int* featR, int* featM, unsigned long long* status, int* maxAR, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    features_kernel<<<(int)blocks, 256, 0, st>>>(atom_off, frag_off, move_off, n, featA, featR, featM, status, maxAR);
    return cudaGetLastError();
}

cudaError_t launch_ingest(const int64_t* atom_off, const float* xyz, const uint8_t* atom_type, int n_types,
                          const int64_t* frag_off, const int32_t* frag_axis,
                          const int64_t* move_off, const int32_t* move_atoms, const uint32_t* perm,
                          const int64_t* owned_start, const int* owned_prefix, int n_owned, int total_slots,
                          uint8_t* order, int4* frint, uint8_t* fown, int* lflag, unsigned long long* status,
                          cudaStream_t st) {
    if (total_slots <= 0) return cudaSuccess;
    int blocks = (total_slots + kIngestWarps - 1) / kIngestWarps;
    if (blocks > 148 * 16) blocks = 148 * 16;
    ingest_kernel<<<blocks, kIngestWarps * 32, 0, st>>>(atom_off, xyz, atom_type, n_types, frag_off, frag_axis, move_off, move_atoms, perm,
                                                        owned_start, owned_prefix, n_owned, total_slots, order, frint,
                                                        fown, lflag, status);
    return cudaGetLastError();
}

cudaError_t launch_classify_hist(const int* featA, const int* featR, const int* featM, int64_t n, const int* atom_b,
                                 int n_atom_b, const int* rot_b, int n_rot_b, const int* move_b, int n_move_b, int* cell,
                                 int* hist, int n_blocks, unsigned long long* ovf, cudaStream_t st) {
    Bounds bd;
    bd.n_atom_b = n_atom_b;
    bd.n_rot_b = n_rot_b;
    bd.n_move_b = n_move_b;
    for (int i = 0; i < n_atom_b; ++i) bd.atom_b[i] = atom_b[i];
    for (int i = 0; i < n_rot_b; ++i) bd.rot_b[i] = rot_b[i];
    for (int i = 0; i < n_move_b; ++i) bd.move_b[i] = move_b[i];
    classify_hist_kernel<<<n_blocks, 1024, 0, st>>>(featA, featR, featM, n, bd, cell, hist, n_blocks, ovf);
    return cudaGetLastError();
}

cudaError_t launch_scan_hist(int* hist, int n_cells, int n_blocks, int* cell_count, cudaStream_t st) {
    scan_hist_kernel<<<1, 1024, 0, st>>>(hist, n_cells, n_blocks, cell_count);
    return cudaGetLastError();
}

cudaError_t launch_scatter(const int* cell, int64_t n, const int* hist_off, int n_cells, int n_blocks, uint32_t* perm,
                           cudaStream_t st) {
    const size_t smem = (size_t)33 * n_cells * 4;
    if (smem > 48 * 1024) {
        const cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(scatter_kernel),
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    scatter_kernel<<<n_blocks, 1024, smem, st>>>(cell, n, hist_off, n_cells, n_blocks, perm);
    return cudaGetLastError();
}

cudaError_t launch_bucket_weights(const uint32_t* perm, const int* featA, const int* featR, const int* featM,
                                  const int64_t* bstart,
                                  const int* bsize, int n_buckets, long long P, long long K, long long S_w,
                                  unsigned long long* weights, cudaStream_t st) {
    if (n_buckets <= 0) return cudaSuccess;
    bucket_weights_kernel<<<n_buckets, 256, 0, st>>>(perm, featA, featR, featM, bstart, bsize, P, K, S_w, weights);
    return cudaGetLastError();
}

cudaError_t launch_pack(const uint32_t* perm, const int64_t* owned_start, const int* owned_prefix, const int* owned_ac,
                        const int64_t* owned_rec_off, int n_owned_buckets, int total_slots, const int64_t* atom_off,
                        const float* xyz, const uint8_t* atom_type, const uint8_t* order, const int64_t* frag_off,
                        const int4* frint, const uint8_t* fown, const int* lflag, int S_w, float* rec, int4* meta,
                        cudaStream_t st) {
    if (total_slots <= 0) return cudaSuccess;
    pack_kernel<<<(total_slots + 7) / 8, 256, 0, st>>>(perm, owned_start, owned_prefix, owned_ac, owned_rec_off,
                                                       n_owned_buckets, total_slots, atom_off, xyz, atom_type, order,
                                                       frag_off,
                                                       frint, fown, lflag, S_w, rec, meta);
    return cudaGetLastError();
}

cudaError_t launch_fill_results(float* best_score, int* best_pose, int64_t n, uint8_t* angles, int64_t n_ang,
                                cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    fill_results_kernel<<<148 * 4, 256, 0, st>>>(best_score, best_pose, n, angles, n_ang);
    return cudaGetLastError();
}

cudaError_t launch_make_keys(const int4* meta, int n_slots, const float* best_score, unsigned long long* keys,
                             cudaStream_t st, uint32_t index_offset) {
    if (n_slots <= 0) return cudaSuccess;
    make_keys_kernel<<<(n_slots + 255) / 256, 256, 0, st>>>(meta, n_slots, best_score, keys, index_offset);
    return cudaGetLastError();
}

}  // namespace vsd
