// internal.h -- structures shared by the host runtime (api.cpp) and the CUDA
// kernels (prep.cu, dock.cu, topk.cu).  Not part of the public ABI.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace vsd {

constexpr int kMaxAtoms = 256;     // D1 bound per ligand ("up to a few hundred")
constexpr int kMaxFrags = 32;      // rotatable bonds per ligand
constexpr int kMaxAtomClasses = 8; // atom classes (warp multiples up to 256)
constexpr int kMaxRotClasses = 33; // rotamer classes (0..32)
constexpr int kMaxMoveClasses = 8; // classes of the optional third key, sum_r |M_r|
constexpr int kMaxCells = 1024;    // atom x rotamer x moving-atom cells of one submit
constexpr int kPrepTile = 4096;    // ligands per block in classify/scatter
constexpr int kMaxPoses = 1024;
constexpr int kMaxSweeps = 4;

// Grid modes of the dock kernel ("grid modes"):
//  0 FIX  grids of at most 32 x 32 x 32 nodes, whole grid in shared memory, compile-time
//         strides (34, 1097);
//  1 RT   larger grids that still fit shared memory: runtime strides (nx + 1, (nx + 1) ny + 7);
//  2 WIN  grids that do not fit (48^3, 64^3, 0.5 A spacing, ...): a 32^3-node WINDOW centred
//         on the docking centre is staged in shared memory (fixed strides); a cell whose 8
//         corners all lie in the window is gathered from shared memory, any other cell from
//         the padded global copy through L1 / L2 (ld.global.nc).
//  3 QUAD the production layout: a window of kQuadWC^3 CELLS around the docking centre whose
//         node (x, y, z) holds the float4 (G[x,y,z], G[x,y,z+1], G[x+1,y,z], G[x+1,y,z+1]), so
//         the 8 corners of a cell are TWO 16-byte loads (LDS.128) instead of eight LDS.32:
//         ~9.5 shared wavefronts per LDS.128 on the sweep's points against 4 x 3.07 for the
//         scalar layout (tools/microbench_pairs.cu, tools/bank_sim3.py), i.e. 22 % fewer
//         wavefronts per evaluation.  Cells outside the window read the padded global copy
//         (L1 / L2), as WIN does.  Chosen whenever the window covers +-9 A around the centre
//         (h >= 0.9 A) or the whole grid (grid_mode, dock.cu).
//  4 TYPED per-atom-type grid channels (Q24): the QUAD layout per
//         channel, T windows of W^3 cells side by side (W the largest edge <= kQuadWC whose T windows
//         fit kTypedBudget: W = 18, 15, 12, 9 for T = 1, 2, 4, 8), runtime strides, each atom
//         gathering from its own channel; cells outside the window read the padded global copy of
//         that channel.
//  5 TYPED_S per-atom-type channels in the SCALAR layout: T windows of W^3 cells ((W + 1)^3 nodes of
//         4 bytes, a quarter of a QUAD node) side by side, eight LDS.32 per point; for the same
//         shared memory the window edge is ~1.6x the QUAD one (W = 18 instead of 12 at T = 4), so far
//         fewer points miss it.  Cells outside read the padded global copy of their channel.  The
//         same corner values and blend as TYPED: bit-identical results.
constexpr int kGridFix = 0, kGridRT = 1, kGridWin = 2, kGridQuad = 3, kGridTyped = 4, kGridTypedS = 5;
__host__ __device__ constexpr bool typed_mode(int m) { return m == kGridTyped || m == kGridTypedS; }
constexpr int kMaxChannels = 8;   // grid channels of a typed pocket (atom types 0..7)
constexpr int kWin = 32;   // window edge (nodes)
constexpr int kQuadWC = 18;                  // QUAD window edge (cells per axis)
constexpr int kQuadRS = kQuadWC;             // quads per row (x), rows per plane: kQuadWC + 1 (y + 1)
constexpr int kQuadPS = kQuadRS * (kQuadWC + 1) + 3;   // quads per plane (423 = 3 mod 8: bank model)
// TYPED window of W cells: plane stride W (W + 1) + 3 quads (kQuadPS's padding), channel stride
// W planes + 4 quads
__host__ __device__ inline int typed_plane_stride(int W) { return W * (W + 1) + 3; }
__host__ __device__ inline int typed_chan_stride(int W) { return typed_plane_stride(W) * W + 4; }
constexpr int kTypedBudget = 8464;   // quads (135 KB) for the channel windows of a TYPED pocket
// TYPED_S window of W cells = W + 1 nodes per axis: row stride W + 2 floats, plane stride
// (W + 2)(W + 1) + 7, channel stride W + 1 planes + 8 (the RT layout's padding)
__host__ __device__ inline int typeds_row(int W) { return W + 2; }
__host__ __device__ inline int typeds_plane(int W) { return (W + 2) * (W + 1) + 7; }
__host__ __device__ inline int typeds_chan(int W) { return typeds_plane(W) * (W + 1) + 8; }
constexpr int kTypedSMaxW = 30;   // TYPED_S window edge cap (cells)

// Pocket as the dock kernel sees it.  Coordinates are kept in CENTRED grid units
// v = (y - o)/h - Z with an integer shift Z per axis (16 for FIX, floor(n/2) for RT, the
// window origin + 16 for WIN): |v| stays small, which shrinks the fp32 rounding of every
// placement / rotation step against u = v + Z in [0, n-1], and the shift costs nothing -- it
// is folded into the clamp bounds and the floor constant 2^23 + Z.
struct PocketDev {
    const float* grid;     // global PADDED copy [nz+1][ny+1][nx+1] (zero pads), strides grs, gps
    int nx, ny, nz;
    int rs, ps;            // shared-memory row stride and plane stride (floats)
    int grs, gps;          // global padded row / plane stride (floats)
    int mode;              // kGridFix / kGridRT / kGridWin / kGridQuad / kGridTyped / kGridTypedS
    int wx0, wy0, wz0;     // WIN / QUAD / TYPED: window origin (grid nodes)
    int qwc;               // QUAD / TYPED: fast cells [0, qwc) of the window, all interior (<= n-2) on every axis
    int nch;               // grid channels staged (TYPED: T; else 1)
    int qcs;               // TYPED: shared-memory channel stride (quads); rs = W, ps = typed_plane_stride(W)
    int gcs;               // global channel stride of the padded copy (floats)
    const float4* gq;      // global QUAD copy behind the padded channels: node (x, y, z) of channel t at
                           // gq[t * gqcs + x + y * nx + z * nx * (ny + 1)], x < nx, y <= ny, z < nz, holding
                           // (G[x,y,z], G[x,y,z+1], G[x+1,y,z], G[x+1,y,z+1]) of the padded copy
    int gqcs;              // its channel stride (quads)
    float lo_x, lo_y, lo_z;       // -Z          (u = 0)
    float top_x, top_y, top_z;    // n - 1 - Z   (u = n - 1)
    float mx, my, mz;             // 2^23 + Z    (exact)
    float kh;              // kappa * h  (penalty per grid unit of excess)
    float h;
    float ox, oy, oz;      // origin of the centred frame: o + h Z (Angstrom)
    float tx, ty, tz;      // (center - origin) / h - Z
    float inv_h;
};

// Outputs of one docking site (pocket) of a launch.
struct SiteOut {
    float* best_score;         // [n_total]
    int* best_pose;            // [n_total]
    uint8_t* angles;           // CSR S_w * frag_off
    float* dbg_score;          // [n_total * P] or null
    uint8_t* dbg_angles;       // [P * S_w * frag_off] or null
    float* xyz_out;            // a9 best-pose coordinates [3 * n_atoms] (input atom order) or null
    uint8_t* refine;           // rigid refinement moves of p* [n_total * n_ref] (Q23) or null
    uint8_t* dbg_refine;       // [n_total * P * n_ref] or null
};

// Fused multi-site launches: a thread-block cluster of n_sites CTAs docks
// the same staged ligands into n_sites pockets, CTA rank s into pocket s.
constexpr int kMaxSites = 8;

// One dock launch (a6-a9).  Single-site launches use pk[0] / out[0].
struct DockArgs {
    const float* rec;          // packed records of this bucket (slot s at rec + s * rec_floats)
    const int4* meta;          // [slots] {ligand index, A, R, S_w * frag_off}
    int n;                     // ligands in the bucket
    int rec_floats;            // rec_floats_of(AC)
    int P, K, S_w;
    int ligs_per_cta;          // LC
    int frag_cap;              // RC: no ligand of the launch has more fragments
    int n_sites;               // 1, or the cluster size of a fused multi-site launch
    int* counter;              // dynamic round counter of this launch (zeroed before launch)
    const float* pose_tab;     // [P][12] raw: R (9, row-major) then tau (3)
    const float* cs;           // [K][2]
    int n_ref, n_moves;        // rigid refinement rounds after the sweeps and moves per round (Q23)
    const float* ref_tab;      // [n_moves][12]: Q (9, row-major) then d (3, Angstrom)
    const uint8_t* order;      // internal atom -> input atom (CSR by atom_off, a1)
    const int64_t* atom_off;   // [n_total + 1]
    PocketDev pk[kMaxSites];
    SiteOut out[kMaxSites];
};

// Packed ligand record of atom class AC (floats): x | y | z (3 AC), fragment table u32[32],
// own-region lengths u8[32] (8 words), header (n_root | ancestors-first << 16) + 3 pad words;
// a multiple of 4 floats (16-byte TMA granularity).  Typed launches (Q24) append the atom types
// u8[AC] (AC / 4 words).
__host__ __device__ constexpr int rec_floats_of(int AC) { return 3 * AC + 44; }
__host__ __device__ constexpr int rec_floats_typed(int AC, bool typed) { return rec_floats_of(AC) + (typed ? AC / 4 : 0); }

// Per-pose coordinate buffer stride (floats): 3 AC + 8, i.e. 8 banks apart, so the 4 pose
// groups of a warp write 8-atom blocks of (x, y) pairs in 2 wavefronts and of z in 1 (the
// sweep's broadcast loads stay conflict-free).
__host__ __device__ constexpr int pose_stride_of(int AC, int NW, int PPW) {
    return 3 * AC + 8;
}

// Shared-memory layout of dock<AC, NW, PPW> (byte offsets).  Used by the kernel
// and by the host (occupancy query, launch) so both agree.  Rounds (LC ligands each)
// live in a ring of kDockSlots slots: record, meta, pose scores, angle choices.
constexpr int kDockSlots = 3;
struct DockLayout {
    size_t grid, pose, cs, slots, buf, total;
    size_t rec_o, meta_o, score_o, ang_o, slot_b;   // offsets inside one slot, slot size
};
__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }
// Choices kept per pose: S_w * RC angle indices (RC = the launch's fragment cap), then n_ref
// refinement moves (Q23), 4-aligned.
__host__ __device__ inline int dock_ang_stride(int S_w, int RC, int n_ref) {
    return ((S_w * (RC > 0 ? RC : 1)) + n_ref + 3) & ~3;
}
constexpr int kMaxRefineMoves = 32;   // moves per refinement round (u8 indices, Kp-wide lane groups)
constexpr int kMaxRefineRounds = 8;
// Grid region of the dock kernel (floats).  Corner reads at i0 + 1 = n carry weight 0 but
// must read FINITE values that no other warp writes.  FIX: the nz planes + a 32-float zero
// pad: the z index is clamped to nz - 2 at the top face (grid_g), so the only read past the
// planes is the y overflow of row ny in the last plane (<= 34 rs - ps = 25 floats).  RT keeps
// a zero plane + row.  WIN: the 32 window planes; the shared-memory path never reads past
// local node 31 on any axis.
// TYPED: nch channels of typed_chan_stride(rs) quads (rs = W).
__host__ __device__ inline size_t dock_grid_floats(int mode, int nz, int rs, int ps, int nch = 1) {
    return mode == kGridFix    ? (size_t)nz * ps + 32
           : mode == kGridWin   ? (size_t)kWin * ps
           : mode == kGridQuad  ? (size_t)4 * kQuadPS * kQuadWC
           : mode == kGridTyped ? (size_t)4 * typed_chan_stride(rs) * nch
           : mode == kGridTypedS ? (size_t)(ps * (rs - 1) + 8) * nch
                                : (size_t)(nz + 1) * ps + rs + 2;
}
__host__ __device__ inline DockLayout dock_layout(int AC, int NW, int PPW, int mode, int nz, int rs, int ps, int nch,
                                                  int P, int K, int S_w, int LC, int RC, int n_ref) {
    DockLayout L;
    size_t o = 0;
    L.grid = o;  o += align16(dock_grid_floats(mode, nz, rs, ps, nch) * 4);
    L.buf = o;   o += (size_t)NW * PPW * pose_stride_of(AC, NW, PPW) * 4;   // (x,y)|z per pose
    L.pose = o;   // pose table: read per warp item from global (L1-resident), no shared copy
    L.cs = o;     // angle table: each lane keeps its (cos, sin) in registers, no shared copy
    size_t q = 0;
    L.rec_o = q;   q += align16((size_t)LC * rec_floats_typed(AC, typed_mode(mode)) * 4);
    L.meta_o = q;  q += (size_t)LC * 16;
    L.score_o = q; q += align16((size_t)LC * P * 4);
    L.ang_o = q;   q += align16((size_t)LC * P * dock_ang_stride(S_w, RC, n_ref));
    L.slot_b = q;
    L.slots = o; o += kDockSlots * q;
    L.total = o;
    return L;
}
// Ligands a CTA docks concurrently (Eq. 1's t/ws, reading Q19): each ligand needs
// ceil(P / PPW) warp items; a CTA of NW warps holds NW / min(NW, items) ligands.
__host__ __device__ inline int ligs_per_cta(int NW, int PPW, int P) {
    const int g = (P + PPW - 1) / PPW;
    const int wl = g < NW ? g : NW;
    const int lc = NW / wl;
    return lc > 0 ? lc : 1;
}
// Grid mode and shared-memory strides (row rs, plane ps) of an nx x ny x nz grid.
int grid_mode(int nx, int ny, int nz, float spacing);
// TYPED window edge (cells) for nch channels
int typed_window(int nch);
// TYPED layout of an nch-channel pocket: kGridTyped (QUAD windows) or kGridTypedS (scalar windows),
// and its window edge W (cells)
int typed_layout(int nch, int* W);
// Host layout of a pocket's device copy (floats): nch padded channels [nz+1][ny+1][nx+1], then
// (16-byte aligned) the global QUAD copy of every channel, nx * (ny + 1) * nz float4 each.
inline size_t pocket_quad_offset(int nx, int ny, int nz, int nch) {
    const size_t gc = (size_t)(nx + 1) * (ny + 1) * (nz + 1);
    return (gc * nch + 3) & ~(size_t)3;
}
inline size_t pocket_floats(int nx, int ny, int nz, int nch) {
    return pocket_quad_offset(nx, ny, nz, nch) + (size_t)4 * nx * (ny + 1) * nz * nch;
}
void grid_strides(int mode, int nx, int ny, int* rs, int* ps);

// Launchers (return cudaGetLastError()).
cudaError_t launch_rebase(const int64_t* src, int64_t* dst, int64_t count, int64_t base, cudaStream_t st);
cudaError_t launch_features(const int64_t* atom_off, const int64_t* frag_off, const int64_t* move_off, int64_t n,
                            int* featA, int* featR, int* featM, unsigned long long* status, int* maxAR, cudaStream_t st);
// a1 ingest of the owned (packed) slots: validation, laminar check, canonical renumbering.
cudaError_t launch_ingest(const int64_t* atom_off, const float* xyz, const uint8_t* atom_type, int n_types,
                          const int64_t* frag_off, const int32_t* frag_axis,
                          const int64_t* move_off, const int32_t* move_atoms, const uint32_t* perm,
                          const int64_t* owned_start, const int* owned_prefix, int n_owned, int total_slots,
                          uint8_t* order, int4* frint, uint8_t* fown, int* lflag, unsigned long long* status,
                          cudaStream_t st);
cudaError_t launch_classify_hist(const int* featA, const int* featR, const int* featM, int64_t n, const int* atom_b,
                                 int n_atom_b, const int* rot_b, int n_rot_b, const int* move_b, int n_move_b, int* cell,
                                 int* hist, int n_blocks,
                                 unsigned long long* ovf, cudaStream_t st);
cudaError_t launch_scan_hist(int* hist, int n_cells, int n_blocks, int* cell_count, cudaStream_t st);
cudaError_t launch_scatter(const int* cell, int64_t n, const int* hist_off, int n_cells, int n_blocks, uint32_t* perm,
                           cudaStream_t st);
cudaError_t launch_bucket_weights(const uint32_t* perm, const int* featA, const int* featR, const int* featM,
                                  const int64_t* bstart,
                                  const int* bsize, int n_buckets, long long P, long long K, long long S_w,
                                  unsigned long long* weights, cudaStream_t st);
// Pack owned buckets.  slot_bucket_prefix[b] = first packed slot of owned bucket b (nb+1 entries).
cudaError_t launch_pack(const uint32_t* perm, const int64_t* owned_start, const int* owned_prefix, const int* owned_ac,
                        const int64_t* owned_rec_off, int n_owned_buckets, int total_slots, const int64_t* atom_off,
                        const float* xyz, const uint8_t* atom_type, const uint8_t* order, const int64_t* frag_off,
                        const int4* frint, const uint8_t* fown, const int* lflag, int S_w, float* rec, int4* meta,
                        cudaStream_t st);
cudaError_t launch_dock(int AC, int NW, int PPW, const DockArgs& a, int grid, size_t smem, cudaStream_t st);
cudaError_t dock_kernel_attrs(int AC, int NW, int PPW, int gmode, int K, cudaFuncAttributes* attr);
cudaError_t dock_occupancy(int AC, int NW, int PPW, int gmode, int K, size_t smem, int* blocks_per_sm);
cudaError_t dock_cluster_occupancy(int AC, int NW, int PPW, int gmode, int K, size_t smem, int sites, int* clusters);
cudaError_t launch_fill_results(float* best_score, int* best_pose, int64_t n, uint8_t* angles, int64_t n_ang,
                                cudaStream_t st);
cudaError_t launch_score_points(const PocketDev& pk, const float* xyz, const uint8_t* types, int64_t n, float* out,
                                size_t smem, cudaStream_t st);
// top-k
cudaError_t launch_make_keys(const int4* meta, int n_slots, const float* best_score, unsigned long long* keys,
                             cudaStream_t st, uint32_t index_offset = 0);
// Select the k smallest of keys[n] (unique except UINT64_MAX pads), write them sorted to out[k]
// (UINT64_MAX padded).
// scratch: >= (n + 2048) u64 + 4 KB.  Returns the number of kernels launched in *launches.
cudaError_t topk_select_sort(const unsigned long long* keys, int64_t n, int k, unsigned long long* out,
                             void* scratch, cudaStream_t st, int* launches);
cudaError_t launch_gather_ids(const unsigned long long* keys, int m, const unsigned long long* ids, int64_t n_ids,
                              unsigned long long* out, cudaStream_t st);

}  // namespace vsd
