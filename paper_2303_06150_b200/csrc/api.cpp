// api.cpp -- host runtime behind include/vsdock.h: context, workspace planning,
// the submit pipeline (a1..a9 orchestration), bucket table and LPT shard
// (a4), multi-stream bucket launches, results, ranking (a10/a11).
//
// PAPER.md l.200-204 (workers, double buffering, one pipeline per GPU) and
// l.219-231 (input preparation + Eq. 1 sizing) are the design being re-done:
// on B200 the whole library is HBM-resident, so there is no worker pool and
// no double-buffered device pool; buckets launch on several streams so that
// partial buckets overlap (the tail effect of P:421-424).
#include "vsdock.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "internal.h"

using namespace vsd;

namespace {

struct PocketHost {
    vs_pocket_desc d;
    int nch = 1;               // grid channels (Q24): nch padded copies back to back
    std::vector<float> grid;
};

struct ClassInfo {
    int atom_bound, AC, NW, PPW, LC, b, l, cap;
    size_t smem;
    cudaFuncAttributes attr;
};

struct Region {
    size_t off = 0;
    size_t add(size_t bytes) {
        off = (off + 255) & ~(size_t)255;
        const size_t o = off;
        off += bytes;
        return o;
    }
};

int roundup32(int x) { return (x + 31) / 32 * 32; }

// S:205-213 with reading Q16 (independent re-implementation of the boundary
// formula; the oracle's Python copy is not used by the product).
std::vector<int> atom_bounds(int n, int ub) {
    std::vector<int> b;
    const int last = ub >= 32 * (n - 1) + 1 ? ub : 32 * n;
    for (int i = 1; i < n; ++i) b.push_back(32 * i);
    b.push_back(last);
    return b;
}

// S:215-223, prev_0 = -1, round half up in exact integer arithmetic (Q17)
std::vector<int> rot_bounds(int n, int mx) {
    std::vector<int> b;
    if (n > mx) {
        for (int v = 0; v <= mx; ++v) b.push_back(v);
        return b;
    }
    long long prev = -1;
    const unsigned long long den = (n >= 63) ? ~0ull : ((1ull << n) - 1ull);
    for (int i = 1; i <= n; ++i) {
        long long v;
        if (i == n) v = mx;
        else {
            const unsigned long long num = (unsigned long long)mx * ((1ull << i) - 1ull);
            v = (long long)((2ull * num + den) / (2ull * den));
        }
        if (v < prev + 1) v = prev + 1;
        b.push_back((int)v);
        prev = v;
    }
    return b;
}

// a4: buckets by weight descending (ties: id ascending) to the least-loaded rank
// (ties: lowest rank); launch_order = position in that rank's sequence.
void lpt_plan(const uint64_t* w, int nb, int world, int32_t* owner, int32_t* launch_order) {
    std::vector<int> order(nb);
    for (int b = 0; b < nb; ++b) order[b] = b;
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
        if (w[x] != w[y]) return w[x] > w[y];
        return x < y;
    });
    std::vector<unsigned long long> load(world, 0);
    std::vector<int> nlaunch(world, 0);
    for (int b : order) {
        int r = 0;
        for (int q = 1; q < world; ++q)
            if (load[q] < load[r]) r = q;
        load[r] += w[b];
        owner[b] = r;
        launch_order[b] = nlaunch[r]++;
    }
}

}  // namespace

struct vs_ctx {
    vs_config cfg{};
    int sm_count = 0;
    cudaStream_t main = nullptr;
    bool own_main = false;
    std::vector<cudaStream_t> workers;
    std::vector<cudaEvent_t> ev_worker;
    cudaEvent_t ev_prep0 = nullptr, ev_prep1 = nullptr, ev_dock1 = nullptr, ev_t0 = nullptr, ev_t1 = nullptr;
    std::string err;

    int P = 0, K = 0;
    int frag_cap = 0;             // max fragments per ligand of the submitted library (sizes angle buffers)
    long long tables_version = 0; // bumped by every pose / angle table or pocket change
    std::vector<long long> uploaded_sig;   // (workspace, tables_version, grid size, pocket ids) on the device
    std::vector<float> pose_tab;  // P * 12
    std::vector<float> cs;        // K * 2
    int n_ref = 0, n_moves = 1;   // rigid refinement rounds / moves (Q23); n_ref = 0: off
    std::vector<float> ref_tab;   // n_moves * 12: Q (row-major) then d (Angstrom)
    std::vector<PocketHost> pockets;

    uint8_t* ws = nullptr;
    size_t ws_bytes = 0;
    void* hpin = nullptr;
    size_t hpin_bytes = 0;

    // last job
    bool submitted = false;
    int64_t n = 0, nA = 0, nR = 0, nM = 0;
    std::vector<int> job_pockets;
    int64_t *d_atom_off = nullptr, *d_frag_off = nullptr, *d_move_off = nullptr;
    float* d_xyz = nullptr;
    int32_t *d_frag_axis = nullptr, *d_move_atoms = nullptr;
    const uint64_t* d_lid = nullptr;   // ligand ids of the batch (null: ids = indices)
    const uint8_t* d_types = nullptr;  // atom types of a typed submit (Q24), input order; null: untyped
    uint8_t* d_order = nullptr;        // a1: internal atom -> input atom, CSR by atom_off
    int4* d_frint = nullptr;           // a1: fragments in internal numbering {a, b, lo, hi}
    uint8_t* d_fown = nullptr;         // a1: own-region length per fragment
    int* d_lflag = nullptr;            // a1: n_root | ancestors-first << 16 per ligand
    int *d_featA = nullptr, *d_featR = nullptr, *d_featM = nullptr, *d_cell = nullptr, *d_hist = nullptr,
        *d_cell_count = nullptr, *d_maxAR = nullptr;
    unsigned long long* d_status = nullptr;  // [0] validation, [1] overflow
    uint32_t* d_perm = nullptr;
    int64_t* d_bstart = nullptr;
    int* d_bsize = nullptr;
    unsigned long long* d_weights = nullptr;
    int64_t *d_own_start = nullptr, *d_own_rec_off = nullptr;
    int *d_own_prefix = nullptr, *d_own_ac = nullptr;
    float* d_rec = nullptr;
    int4* d_meta = nullptr;
    float* d_pose = nullptr;
    float* d_cs = nullptr;
    float* d_reftab = nullptr;
    std::vector<float*> d_grid;
    std::vector<float*> d_score;
    std::vector<int*> d_pose_best;
    std::vector<uint8_t*> d_ang;
    std::vector<float*> d_dbg_score;
    std::vector<uint8_t*> d_dbg_ang;
    std::vector<uint8_t*> d_ref;       // refinement moves of p* per pocket slot [n * n_ref]
    std::vector<uint8_t*> d_dbg_ref;   // [n * P * n_ref] (debug_poses)
    std::vector<float*> d_coords;      // a9 best-pose coordinates per pocket slot (written by the dock kernel)
    unsigned long long* d_keys = nullptr;
    int64_t keys_cap = 0;
    unsigned long long* d_topk_out = nullptr;
    void* d_sel = nullptr;

    std::vector<int> atom_b, rot_b, move_b;
    std::vector<ClassInfo> classes;                    // class table that sizes the buckets (Eq. 1)
    std::vector<std::vector<ClassInfo>> layout_classes;  // per distinct grid layout of the submit
    std::vector<int> pk_layout;                        // pocket slot -> index into layout_classes
    std::vector<vs_bucket> buckets;
    std::vector<int> owned;             // bucket ids, launch order
    std::vector<int> owned_prefix;      // slots
    std::vector<int64_t> owned_rec_off; // floats
    std::vector<PocketDev> pkdev;
    int total_slots = 0;
    vs_stats stats{};
};

namespace {

vs_status fail(vs_ctx* c, vs_status code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    c->err = buf;
    return code;
}

#define CK(call)                                                                                   \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess) return fail(c, VS_E_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

// Large asynchronous read-backs go out in pieces: one copy engine serves the D2H copies of
// every stream, one request at a time, so a single 300 MB copy would hold up the small
// status reads of another context's preparation for its whole duration (two engines
// alternating over chunks, pipeline.py).  4 MB pieces bound that wait to ~80 us.
cudaError_t copy_pieces(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind, cudaStream_t st) {
    constexpr size_t kPiece = 4u << 20;
    for (size_t o = 0; o < bytes; o += kPiece) {
        const cudaError_t e = cudaMemcpyAsync((char*)dst + o, (const char*)src + o, std::min(kPiece, bytes - o), kind, st);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

vs_status ensure_pinned(vs_ctx* c, size_t bytes) {
    if (c->hpin_bytes >= bytes) return VS_OK;
    if (c->hpin) cudaFreeHost(c->hpin);
    c->hpin = nullptr;
    c->hpin_bytes = 0;
    CK(cudaMallocHost(&c->hpin, bytes));
    c->hpin_bytes = bytes;
    return VS_OK;
}

// typed = a typed submit (Q24): every pocket runs the TYPED layout with its nch channels (a pocket
// of one channel included); an untyped submit docks on channel 0 with the usual layouts
PocketDev make_pocket_dev(const vs_pocket_desc& d, const float* dgrid, bool typed = false, int nch = 1) {
    PocketDev p;
    p.grid = dgrid;
    p.nx = d.nx;
    p.ny = d.ny;
    p.nz = d.nz;
    p.grs = d.nx + 1;
    p.gps = (d.nx + 1) * (d.ny + 1);
    p.gcs = p.gps * (d.nz + 1);
    p.gq = reinterpret_cast<const float4*>(dgrid + pocket_quad_offset(d.nx, d.ny, d.nz, nch));
    p.gqcs = d.nx * (d.ny + 1) * d.nz;
    p.nch = typed ? nch : 1;
    p.qcs = 0;
    int QW = kQuadWC;   // QUAD / TYPED / TYPED_S window edge (cells)
    p.mode = typed ? typed_layout(nch, &QW) : grid_mode(d.nx, d.ny, d.nz, d.spacing);
    if (p.mode == kGridTyped) {
        p.rs = QW;
        p.ps = typed_plane_stride(QW);
        p.qcs = typed_chan_stride(QW);
    } else if (p.mode == kGridTypedS) {   // floats
        p.rs = typeds_row(QW);
        p.ps = typeds_plane(QW);
        p.qcs = typeds_chan(QW);
    } else {
        grid_strides(p.mode, d.nx, d.ny, &p.rs, &p.ps);
    }
    // WIN: the 32^3-node window around the docking centre (clamped into the grid); QUAD: the
    // window of kQuadWC cells [w0, w0 + kQuadWC) around it, clamped so that it covers as many of
    // the grid's cells 0 .. n-1 (the top face n-1 is a cell with weight-0 pad corners) as it can
    const int n3[3] = {d.nx, d.ny, d.nz};
    int w0[3] = {0, 0, 0};
    // (QUAD keeps its cells below the top face n-1, so the fast path's cells are interior)
    p.qwc = 0;
    if (p.mode == kGridWin || p.mode == kGridQuad || typed_mode(p.mode)) {
        const int W = p.mode == kGridWin ? kWin : QW;
        p.qwc = QW;
        for (int a = 0; a < 3; ++a) {
            const double uc = ((double)d.center[a] - d.origin[a]) / d.spacing;
            int v = (int)std::lround(uc) - W / 2;
            v = std::min(v, p.mode == kGridWin ? n3[a] - W : n3[a] - 1 - W);
            w0[a] = std::max(v, 0);
            p.qwc = std::min(p.qwc, n3[a] - 1 - w0[a]);
        }
    }
    p.wx0 = w0[0];
    p.wy0 = w0[1];
    p.wz0 = w0[2];
    // centring shift (PocketDev): 16 on every axis for FIX (the dock kernel then folds -Z and
    // 2^23 + Z into immediates), n / 2 for RT, the window centre for WIN
    int Z[3];
    for (int a = 0; a < 3; ++a)
        Z[a] = p.mode == kGridFix    ? 16
               : p.mode == kGridRT   ? n3[a] / 2
               : p.mode == kGridQuad || typed_mode(p.mode) ? w0[a] + QW / 2
                                     : w0[a] + kWin / 2;
    p.lo_x = (float)-Z[0];
    p.lo_y = (float)-Z[1];
    p.lo_z = (float)-Z[2];
    p.top_x = (float)(d.nx - 1 - Z[0]);
    p.top_y = (float)(d.ny - 1 - Z[1]);
    p.top_z = (float)(d.nz - 1 - Z[2]);
    p.mx = 8388608.f + (float)Z[0];
    p.my = 8388608.f + (float)Z[1];
    p.mz = 8388608.f + (float)Z[2];
    if (p.mode == kGridQuad || typed_mode(p.mode)) {   // 1.5 * 2^23 + Z - w0: the floor's bits give the window-relative cell
        p.mx = 12582912.f + (float)(Z[0] - w0[0]);
        p.my = 12582912.f + (float)(Z[1] - w0[1]);
        p.mz = 12582912.f + (float)(Z[2] - w0[2]);
    }
    p.kh = (float)((double)d.out_slope * (double)d.spacing);
    p.h = d.spacing;
    p.inv_h = (float)(1.0 / (double)d.spacing);
    p.ox = (float)((double)d.origin[0] + (double)d.spacing * Z[0]);
    p.oy = (float)((double)d.origin[1] + (double)d.spacing * Z[1]);
    p.oz = (float)((double)d.origin[2] + (double)d.spacing * Z[2]);
    p.tx = (float)(((double)d.center[0] - d.origin[0]) / d.spacing - Z[0]);
    p.ty = (float)(((double)d.center[1] - d.origin[1]) / d.spacing - Z[1]);
    p.tz = (float)(((double)d.center[2] - d.origin[2]) / d.spacing - Z[2]);
    return p;
}

// Shared memory of the score_points hook's grid region (floats).
size_t score_grid_floats(const PocketDev& pk) {
    return dock_grid_floats(pk.mode == kGridFix ? kGridRT : pk.mode, pk.nz, pk.rs, pk.ps, pk.nch);
}

// Stage-1 workspace (known from the batch sizes alone).
struct Stage1 {
    size_t atom_off, frag_off, xyz, types, lid, frag_axis, move_off, move_atoms, order, frint, fown, lflag, featA, featR, featM, cell, status, maxAR, hist, cell_count, perm, bstart,
        bsize, weights, own_start, own_prefix, own_ac, own_rec_off, pose, cs, reftab, grids, end;
    int n_blocks;
    int64_t max_buckets;
};

Stage1 plan1(int64_t n, int64_t nA, int64_t nR, int64_t nM, int P, int K, size_t grid_bytes, int n_pockets) {
    Stage1 s;
    Region r;
    s.n_blocks = (int)((n + kPrepTile - 1) / kPrepTile);
    if (s.n_blocks < 1) s.n_blocks = 1;
    s.max_buckets = n + kMaxCells;
    // tables and grids first: their offsets depend only on (P, K, grid size, pockets), so
    // an unchanged set stays resident across submits and is not re-uploaded
    s.pose = r.add((size_t)P * 12 * 4);
    s.cs = r.add((size_t)K * 2 * 4 + 16);
    s.reftab = r.add((size_t)kMaxRefineMoves * 12 * 4);
    s.grids = r.add(grid_bytes * n_pockets);
    s.atom_off = r.add((n + 1) * 8);
    s.frag_off = r.add((n + 1) * 8);
    s.xyz = r.add(nA * 12);
    s.types = r.add(nA);   // atom types of a typed submit (Q24)
    s.lid = r.add(n * 8);
    s.frag_axis = r.add(nR * 8);
    s.move_off = r.add((nR + 1) * 8);
    s.move_atoms = r.add(nM * 4);
    s.order = r.add(nA);
    s.frint = r.add(nR * 16);
    s.fown = r.add(nR);
    s.lflag = r.add(n * 4);
    s.featA = r.add(n * 4);
    s.featR = r.add(n * 4);
    s.featM = r.add(n * 4);
    s.cell = r.add(n * 4);
    s.status = r.add(24);   // [0] features, [1] classify overflow, [2] ingest of the owned ligands
    s.maxAR = r.add(16);   // observed max A, R, sum |M_r|
    s.hist = r.add((size_t)kMaxCells * s.n_blocks * 4);
    s.cell_count = r.add(kMaxCells * 4);
    s.perm = r.add(n * 4);
    s.bstart = r.add(s.max_buckets * 8);
    s.bsize = r.add(s.max_buckets * 4);
    s.weights = r.add(s.max_buckets * 32);
    s.own_start = r.add(s.max_buckets * 8);
    s.own_prefix = r.add((s.max_buckets + 1) * 4);
    s.own_ac = r.add(s.max_buckets * 4);
    s.own_rec_off = r.add(s.max_buckets * 8);
    s.end = r.off;
    return s;
}

// Stage-2 workspace (records + results), placed after stage 1.
struct Stage2 {
    size_t rec, meta, score, pose_best, ang, dbg_score, dbg_ang, ref, dbg_ref, coords, keys, topk_out, sel, counters, end;
    size_t per_slot;  // bytes of results per pocket slot
};

Stage2 plan2(size_t base, int64_t n, int64_t nA, int64_t nR, int64_t rec_floats, int P, int S_w, int n_pockets,
             bool debug, int n_ref) {
    Stage2 s;
    Region r;
    r.off = base;
    s.rec = r.add((size_t)rec_floats * 4);
    s.meta = r.add(n * 16);
    s.score = r.add(n * 4 * n_pockets + 256 * n_pockets);
    s.pose_best = r.add(n * 4 * n_pockets + 256 * n_pockets);
    s.ang = r.add((size_t)S_w * nR * n_pockets + 256 * n_pockets);
    s.dbg_score = r.add(debug ? (size_t)n * P * 4 * n_pockets + 256 * n_pockets : 0);
    s.dbg_ang = r.add(debug ? (size_t)P * S_w * nR * n_pockets + 256 * n_pockets : 0);
    s.ref = r.add(n_ref ? (size_t)n * n_ref * n_pockets + 256 * n_pockets : 0);
    s.dbg_ref = r.add(debug && n_ref ? (size_t)n * P * n_ref * n_pockets + 256 * n_pockets : 0);
    s.coords = r.add((nA * 12 + 256) * n_pockets);
    const int64_t kc = std::max<int64_t>(n, 65536);
    s.keys = r.add(kc * 8);
    s.topk_out = r.add(2 * 8192 * 8);   // merged keys + their ligand ids
    s.sel = r.add(4096);
    s.counters = r.add((size_t)(n + kMaxCells) * n_pockets * 4 + 256);
    s.end = r.off;
    return s;
}

size_t max_grid_bytes(const vs_ctx* c) {
    size_t m = 0;
    for (auto& p : c->pockets) m = std::max(m, p.grid.size() * 4);   // padded copies
    return m;
}

const char* vcode_msg(int code) {
    switch (code) {
        case 1: return "atom count outside [1, 256]";
        case 2: return "fragment count outside [0, 32]";
        case 3: return "non-finite coordinate";
        case 4: return "fragment axis atom index out of range";
        case 5: return "fragment axis atoms are equal";
        case 6: return "fragment moving set empty or larger than atoms - 2";
        case 7: return "fragment axis atom inside its own moving set";
        case 8: return "fragment axis atoms closer than 1e-3 A";
        case 9: return "moving atom index out of range";
        case 10: return "atom listed twice in one moving set";
        case 11: return "moving sets not laminar (two fragments' moving sets overlap without nesting)";
        case 12: return "coordinate magnitude above 1e6 A";
        case 13: return "atom type >= the grid channels of a docked pocket";
        default: return "invalid record";
    }
}

int pow2_ceil(int K) {
    int p = 1;
    while (p < K) p <<= 1;
    return p;
}

// Per atom class: template capacity, warps, ligands per CTA, occupancy b, Eq. 1 -- for one
// grid layout (mode, nz planes of ps floats, row stride rs).
vs_status plan_classes(vs_ctx* c, const std::vector<int>& atom_b, int gm, int nz, int rs, int ps, int nch, int RC,
                       std::vector<ClassInfo>& out) {
    out.clear();
    for (size_t i = 0; i < atom_b.size(); ++i) {
        ClassInfo ci{};
        ci.atom_bound = atom_b[i];
        ci.AC = std::max(32, roundup32(atom_b[i]));
        if (ci.AC > kMaxAtoms) return fail(c, VS_E_ARG, "atom class bound %d exceeds %d", atom_b[i], kMaxAtoms);
        ci.b = 0;
        // (poses per warp, warps per CTA): the first candidate of the policy whose shared
        // memory fits one CTA per SM and whose pose group holds the K angle lanes
        // (PPW poses x 32/PPW lanes).  VSDOCK_POLICY="4:16,2:16,..." overrides.
        std::vector<std::pair<int, int>> cand = {{4, 20}, {4, 18}, {4, 16}, {4, 15}, {4, 13}, {4, 12}, {4, 10}, {4, 8}, {2, 16}, {2, 8}, {4, 4}, {1, 32}, {1, 16}};
        if (const char* e = getenv("VSDOCK_POLICY")) {
            cand.clear();
            int a = 0, b2 = 0, n = 0;
            const char* s = e;
            while (sscanf(s, "%d:%d%n", &a, &b2, &n) == 2) {
                cand.push_back({a, b2});
                s += n;
                if (*s == ',') ++s;
            }
        }
        // Ligands per round: Eq. 1's t/ws (ligs_per_cta); when the warps of a CTA would all dock ONE
        // ligand (P / PPW >= NW) two ligands per round are tried first, their items interleaved
        // (dock kernel), so the warps do not run the same sweep in lockstep and their shared-memory
        // bursts spread out (measured +4-6 % on the 32 / 64 / 96 classes); the extra
        // slot memory never costs a warp (a candidate's LC = 1 form is tried before the next NW).
        const char* lc_env = getenv("VSDOCK_LC");
        for (auto pr : cand) {
            const int PPW = pr.first, NW = pr.second;
            if (pow2_ceil(c->K) > 32 / PPW) continue;   // the pose group holds the angle slots
            const int base = ligs_per_cta(NW, PPW, c->P);
            std::vector<int> lcs = {base};
            if (lc_env) lcs = {std::max(base, atoi(lc_env))};
            else if (base == 1) lcs = {2, 1};
            for (int LC : lcs) {
                const DockLayout L =
                    dock_layout(ci.AC, NW, PPW, gm, nz, rs, ps, nch, c->P, c->K, c->cfg.n_sweeps, LC, RC, c->n_ref);
                int b = 0;
                CK(dock_occupancy(ci.AC, NW, PPW, gm, c->K, L.total, &b));
                if (b >= 1) {
                    ci.NW = NW;
                    ci.PPW = PPW;
                    ci.LC = LC;
                    ci.b = b;
                    ci.smem = L.total;
                    CK(dock_kernel_attrs(ci.AC, NW, PPW, gm, c->K, &ci.attr));
                    break;
                }
            }
            if (ci.b >= 1) break;
        }
        if (ci.b == 0)
            return fail(c, VS_E_NOFIT, "kernel class %d (A_c = %d) does not fit: occupancy is 0 (grid %dx%d planes)",
                        (int)i, ci.AC, nz, ps);
        ci.l = ci.b * c->sm_count * ci.LC;       // Eq. 1: l = b * SM * t/ws  (Q19)
        ci.cap = c->cfg.bucket_capacity > 0 ? c->cfg.bucket_capacity : ci.l * std::max(1, c->cfg.bucket_multiple);
        out.push_back(ci);
    }
    return VS_OK;
}

}  // namespace

extern "C" {

vs_status vs_create(const vs_config* cfg, vs_ctx** out) {
    if (!cfg || !out) return VS_E_ARG;
    *out = nullptr;
    vs_ctx* c = new vs_ctx();
    c->cfg = *cfg;
    auto bad = [&](const char* m) {
        c->err = m;
        return VS_E_ARG;
    };
    vs_status st = VS_OK;
    if (c->cfg.n_sweeps < 1 || c->cfg.n_sweeps > kMaxSweeps) st = bad("n_sweeps must be in [1, 4]");
    else if (c->cfg.n_atom_clusters < 1 || c->cfg.n_atom_clusters > kMaxAtomClasses) st = bad("n_atom_clusters must be in [1, 8]");
    else if (c->cfg.n_rot_clusters < 1 || c->cfg.n_rot_clusters > kMaxRotClasses) st = bad("n_rot_clusters must be in [1, 33]");
    else if (c->cfg.n_move_clusters < 0 || c->cfg.n_move_clusters > kMaxMoveClasses) st = bad("n_move_clusters must be in [0, 8]");
    else if (c->cfg.move_upper_bound < 0) st = bad("move_upper_bound must be >= 0");
    else if (c->cfg.atom_upper_bound < 0 || c->cfg.atom_upper_bound > kMaxAtoms) st = bad("atom_upper_bound must be in [0, 256]");
    else if (c->cfg.rot_upper_bound < 0 || c->cfg.rot_upper_bound > kMaxFrags) st = bad("rot_upper_bound must be in [0, 32]");
    else if (c->cfg.world_size < 1 || c->cfg.rank < 0 || c->cfg.rank >= c->cfg.world_size) st = bad("bad rank / world_size");
    else if (c->cfg.bucket_capacity < 0) st = bad("bucket_capacity must be >= 0");
    if (st != VS_OK) {
        delete c;
        return st;
    }
    if (c->cfg.bucket_multiple < 1) c->cfg.bucket_multiple = 1;
    if (c->cfg.n_streams < 1) c->cfg.n_streams = 1;
    if (c->cfg.n_streams > 16) c->cfg.n_streams = 16;
    cudaError_t e = cudaSetDevice(c->cfg.device);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, c->cfg.device);
    if (e == cudaSuccess) {
        if (c->cfg.stream) c->main = (cudaStream_t)c->cfg.stream;
        else {
            e = cudaStreamCreateWithFlags(&c->main, cudaStreamNonBlocking);
            c->own_main = true;
        }
    }
    for (int i = 0; e == cudaSuccess && i < c->cfg.n_streams; ++i) {
        cudaStream_t s;
        cudaEvent_t ev;
        e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        if (e == cudaSuccess) {
            c->workers.push_back(s);
            c->ev_worker.push_back(ev);
        }
    }
    for (cudaEvent_t* ev : {&c->ev_prep0, &c->ev_prep1, &c->ev_dock1, &c->ev_t0, &c->ev_t1})
        if (e == cudaSuccess) e = cudaEventCreate(ev);
    if (e != cudaSuccess) {
        c->err = cudaGetErrorString(e);
        vs_destroy(c);
        return VS_E_CUDA;
    }
    *out = c;
    return VS_OK;
}

void vs_destroy(vs_ctx* c) {
    if (!c) return;
    if (c->main) cudaStreamSynchronize(c->main);
    for (auto s : c->workers) cudaStreamDestroy(s);
    for (auto e : c->ev_worker) cudaEventDestroy(e);
    for (cudaEvent_t e : {c->ev_prep0, c->ev_prep1, c->ev_dock1, c->ev_t0, c->ev_t1})
        if (e) cudaEventDestroy(e);
    if (c->own_main && c->main) cudaStreamDestroy(c->main);
    if (c->hpin) cudaFreeHost(c->hpin);
    delete c;
}

const char* vs_last_error(const vs_ctx* c) { return c ? c->err.c_str() : "null context"; }

vs_status vs_set_pose_table(vs_ctx* c, int32_t P, const float* rot, const float* trans) {
    if (!c) return VS_E_ARG;
    if (P < 1 || P > kMaxPoses || !rot || !trans) return fail(c, VS_E_ARG, "pose table: need 1 <= P <= %d", kMaxPoses);
    // validate into a temporary; the active table changes only on success
    std::vector<float> tab((size_t)P * 12, 0.f);
    for (int p = 0; p < P; ++p) {
        for (int t = 0; t < 9; ++t) {
            if (!std::isfinite(rot[9 * p + t])) return fail(c, VS_E_ARG, "pose %d: non-finite rotation", p);
            tab[12 * p + t] = rot[9 * p + t];
        }
        for (int t = 0; t < 3; ++t) {
            if (!std::isfinite(trans[3 * p + t])) return fail(c, VS_E_ARG, "pose %d: non-finite translation", p);
            tab[12 * p + 9 + t] = trans[3 * p + t];
        }
    }
    c->P = P;
    c->pose_tab.swap(tab);
    ++c->tables_version;
    return VS_OK;
}

vs_status vs_set_refine_table(vs_ctx* c, int32_t n_rounds, int32_t n_moves, const float* rot, const float* trans) {
    if (!c) return VS_E_ARG;
    if (n_rounds < 0 || n_rounds > kMaxRefineRounds)
        return fail(c, VS_E_ARG, "refinement: n_rounds must be in [0, %d]", kMaxRefineRounds);
    if (n_rounds == 0) {
        c->n_ref = 0;
        c->n_moves = 1;
        c->ref_tab.clear();
        ++c->tables_version;
        return VS_OK;
    }
    if (n_moves < 1 || n_moves > kMaxRefineMoves || !rot || !trans)
        return fail(c, VS_E_ARG, "refinement: n_moves must be in [1, %d]", kMaxRefineMoves);
    std::vector<float> tab((size_t)n_moves * 12, 0.f);
    for (int m = 0; m < n_moves; ++m) {
        for (int t = 0; t < 9; ++t) {
            if (!std::isfinite(rot[9 * m + t])) return fail(c, VS_E_ARG, "refinement move %d: non-finite rotation", m);
            tab[12 * m + t] = rot[9 * m + t];
        }
        for (int t = 0; t < 3; ++t) {
            if (!std::isfinite(trans[3 * m + t])) return fail(c, VS_E_ARG, "refinement move %d: non-finite translation", m);
            tab[12 * m + 9 + t] = trans[3 * m + t];
        }
    }
    static const float ident[12] = {1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0};
    if (memcmp(tab.data(), ident, sizeof ident) != 0)
        return fail(c, VS_E_ARG, "refinement: move 0 must be exactly the identity (Q = I, d = 0)");
    c->n_ref = n_rounds;
    c->n_moves = n_moves;
    c->ref_tab.swap(tab);
    ++c->tables_version;
    return VS_OK;
}

vs_status vs_set_angle_table(vs_ctx* c, int32_t K, const float* cos_sin) {
    if (!c) return VS_E_ARG;
    if (K < 1 || K > 32 || !cos_sin) return fail(c, VS_E_ARG, "angle table: K must be in [1, 32]");
    if (cos_sin[0] != 1.0f || cos_sin[1] != 0.0f) return fail(c, VS_E_ARG, "angle table: entry 0 must be (1, 0)");
    for (int t = 0; t < 2 * K; ++t)
        if (!std::isfinite(cos_sin[t])) return fail(c, VS_E_ARG, "angle table: non-finite entry %d", t / 2);
    c->K = K;
    c->cs.assign(cos_sin, cos_sin + 2 * K);
    ++c->tables_version;
    return VS_OK;
}

namespace {
vs_status load_pocket_impl(vs_ctx* c, const vs_pocket_desc* d, int nch, const float* grid, int32_t on_device,
                           int32_t* pocket_id) {
    if (!c || !d || !grid) return VS_E_ARG;
    if (nch < 1 || nch > kMaxChannels) return fail(c, VS_E_ARG, "n_channels must be in [1, %d]", kMaxChannels);
    if ((int64_t)d->nx * d->ny * d->nz * nch > (1 << 22)) return fail(c, VS_E_ARG, "pocket grid too large (nodes x channels > 2^22)");
    if (c->pockets.size() >= 16) return fail(c, VS_E_ARG, "at most 16 pockets");
    if (d->nx < 2 || d->ny < 2 || d->nz < 2) return fail(c, VS_E_ARG, "pocket dims must be >= 2");
    if ((int64_t)d->nx * d->ny * d->nz > (1 << 22)) return fail(c, VS_E_ARG, "pocket grid too large");
    if (!(d->spacing >= 1e-4f) || !std::isfinite(d->spacing))
        return fail(c, VS_E_ARG, "pocket spacing must be finite and >= 1e-4 A");
    for (int a = 0; a < 3; ++a)
        if (!std::isfinite(d->origin[a]) || !std::isfinite(d->center[a]))
            return fail(c, VS_E_ARG, "pocket origin/center must be finite");
    if (!std::isfinite(d->out_slope) || d->out_slope < 0.f) return fail(c, VS_E_ARG, "out_slope must be finite and >= 0");
    PocketHost ph;
    ph.d = *d;
    ph.nch = nch;
    const size_t cnt = (size_t)d->nx * d->ny * d->nz;
    std::vector<float> raw(cnt * nch);
    if (on_device) {
        CK(cudaMemcpy(raw.data(), grid, cnt * nch * 4, cudaMemcpyDeviceToHost));
    } else {
        std::memcpy(raw.data(), grid, cnt * nch * 4);
    }
    for (size_t i = 0; i < cnt * nch; ++i)
        if (!std::isfinite(raw[i])) return fail(c, VS_E_ARG, "pocket grid value %zu is not finite", i);
    // the device copy is PADDED: [nz+1][ny+1][nx+1] with zero pads, so a weight-0 corner read at
    // node n stays inside the array (PocketDev::grid); typed pockets: nch padded copies back to back
    const size_t gx = (size_t)d->nx + 1, gy = (size_t)d->ny + 1, gc = gx * gy * ((size_t)d->nz + 1);
    ph.grid.assign(pocket_floats(d->nx, d->ny, d->nz, nch), 0.f);
    for (int t = 0; t < nch; ++t)
        for (int z = 0; z < d->nz; ++z)
            for (int y = 0; y < d->ny; ++y)
                std::memcpy(&ph.grid[t * gc + ((size_t)z * gy + y) * gx], &raw[t * cnt + ((size_t)z * d->ny + y) * d->nx],
                            (size_t)d->nx * 4);
    // the global QUAD copy behind it (PocketDev::gq): node (x, y, z) = (G[x,y,z], G[x,y,z+1], G[x+1,y,z],
    // G[x+1,y,z+1]) of the padded copy, x < nx, y <= ny, z < nz -- a window miss reads 2 x 16 B
    {
        const size_t X = (size_t)d->nx, Y = (size_t)d->ny + 1, Z = (size_t)d->nz;
        float* Q = &ph.grid[pocket_quad_offset(d->nx, d->ny, d->nz, nch)];
        for (int t = 0; t < nch; ++t) {
            const float* P = &ph.grid[t * gc];
            for (size_t z = 0; z < Z; ++z)
                for (size_t y = 0; y < Y; ++y)
                    for (size_t x = 0; x < X; ++x) {
                        const size_t i = x + gx * (y + gy * z), gp = gx * gy;
                        float* q = Q + 4 * (((size_t)t * Z + z) * Y * X + y * X + x);
                        q[0] = P[i];
                        q[1] = P[i + gp];
                        q[2] = P[i + 1];
                        q[3] = P[i + gp + 1];
                    }
        }
    }
    c->pockets.push_back(std::move(ph));
    ++c->tables_version;
    if (pocket_id) *pocket_id = (int32_t)c->pockets.size() - 1;
    return VS_OK;
}
}  // namespace

vs_status vs_load_pocket(vs_ctx* c, const vs_pocket_desc* d, const float* grid, int32_t on_device, int32_t* pocket_id) {
    return load_pocket_impl(c, d, 1, grid, on_device, pocket_id);
}

vs_status vs_load_pocket_typed(vs_ctx* c, const vs_pocket_desc* d, int32_t n_channels, const float* grids,
                               int32_t on_device, int32_t* pocket_id) {
    return load_pocket_impl(c, d, n_channels, grids, on_device, pocket_id);
}

vs_status vs_workspace_size(vs_ctx* c, int64_t n_lig, int64_t n_atoms, int64_t n_frags, int64_t n_moving,
                            int32_t max_atoms, int32_t n_pockets, size_t* bytes) {
    if (!c || !bytes) return VS_E_ARG;
    if (c->P < 1 || c->K < 1) return fail(c, VS_E_STATE, "set the pose and angle tables first");
    if (c->pockets.empty()) return fail(c, VS_E_STATE, "load a pocket first");
    if (n_lig < 0 || n_atoms < 0 || n_frags < 0 || n_moving < 0 || max_atoms < 1 || max_atoms > kMaxAtoms ||
        n_pockets < 1)
        return fail(c, VS_E_ARG, "bad workspace query");
    int ac_max = roundup32(std::max<int>(max_atoms, c->cfg.atom_upper_bound));
    ac_max = std::max(ac_max, 32);
    // Q16 fallback boundary 32*n for the last class can exceed the observed maximum
    ac_max = std::min(kMaxAtoms, std::max(ac_max, std::min(kMaxAtoms, roundup32(max_atoms))));
    const Stage1 s1 = plan1(n_lig, n_atoms, n_frags, n_moving, c->P, c->K, max_grid_bytes(c), n_pockets);
    // records sized for a typed submit (the larger form, Q24)
    const Stage2 s2 = plan2(s1.end, n_lig, n_atoms, n_frags, (int64_t)n_lig * rec_floats_typed(ac_max, true), c->P,
                            c->cfg.n_sweeps, n_pockets, c->cfg.debug_poses != 0, c->n_ref);
    *bytes = s2.end + 4096;
    return VS_OK;
}

vs_status vs_set_workspace(vs_ctx* c, void* ptr, size_t bytes) {
    if (!c) return VS_E_ARG;
    if (((uintptr_t)ptr & 255) != 0) return fail(c, VS_E_ARG, "workspace must be 256-byte aligned");
    c->ws = (uint8_t*)ptr;
    c->uploaded_sig.clear();   // new memory: tables and grids must be uploaded again
    c->d_topk_out = nullptr;   // scratch of the old workspace: never reused after a swap
    c->d_sel = nullptr;
    c->ws_bytes = bytes;
    c->submitted = false;
    return VS_OK;
}

namespace {
vs_status submit_impl(vs_ctx* c, const vs_ligand_batch* batch, const uint8_t* atom_type, const int32_t* pocket_ids,
                      int32_t n_pockets) {
    if (!c || !batch) return VS_E_ARG;
    const bool typed = atom_type != nullptr;
    c->submitted = false;
    c->stats = vs_stats{};   // every field of the last submit, written below
    if (c->P < 1 || c->K < 1) return fail(c, VS_E_STATE, "set the pose and angle tables first");
    if (n_pockets < 1 || n_pockets > 16 || !pocket_ids) return fail(c, VS_E_ARG, "need 1..16 pockets");
    for (int i = 0; i < n_pockets; ++i)
        if (pocket_ids[i] < 0 || pocket_ids[i] >= (int)c->pockets.size())
            return fail(c, VS_E_ARG, "unknown pocket id %d", pocket_ids[i]);
    if (!c->ws) return fail(c, VS_E_WORKSPACE, "no workspace (vs_set_workspace)");
    const int64_t n = batch->n;
    if (n < 0 || n >= (1ll << 31)) return fail(c, VS_E_ARG, "batch size out of range");
    CK(cudaSetDevice(c->cfg.device));
    cudaStream_t ms = c->main;
    const int S_w = c->cfg.n_sweeps;
    int64_t launches = 0;

    // ---- batch sizes
    // Offsets may start at any value b (a slice of a larger library): entry i addresses the data
    // arrays at offset - b.  The library works on rebased copies when b != 0.
    int64_t nA = 0, nR = 0, nM = 0, base_a = 0, base_f = 0, base_m = 0;
    if (n > 0) {
        if (!batch->atom_off || !batch->xyz || !batch->frag_off) return fail(c, VS_E_ARG, "null batch array");
        if (batch->on_device < 0 || batch->on_device > 2) return fail(c, VS_E_ARG, "on_device must be 0, 1 or 2");
        if (batch->on_device == 1) {
            // CSR totals of a device batch: async reads on the context's stream into pinned
            // staging (a plain cudaMemcpy would run on the legacy default stream and wait for
            // every blocking stream of the device -- another engine's docking and read-backs)
            vs_status pst = ensure_pinned(c, 4096);
            if (pst) return pst;
            int64_t* hz = (int64_t*)c->hpin;
            CK(cudaMemcpyAsync(&hz[0], batch->atom_off + n, 8, cudaMemcpyDeviceToHost, ms));
            CK(cudaMemcpyAsync(&hz[1], batch->frag_off + n, 8, cudaMemcpyDeviceToHost, ms));
            CK(cudaMemcpyAsync(&hz[2], batch->atom_off, 8, cudaMemcpyDeviceToHost, ms));
            CK(cudaMemcpyAsync(&hz[3], batch->frag_off, 8, cudaMemcpyDeviceToHost, ms));
            CK(cudaStreamSynchronize(ms));
            base_a = hz[2];
            base_f = hz[3];
            nA = hz[0] - base_a;
            nR = hz[1] - base_f;
            if (nR > 0) {
                if (!batch->move_off) return fail(c, VS_E_ARG, "null move_off");
                CK(cudaMemcpyAsync(&hz[0], batch->move_off, 8, cudaMemcpyDeviceToHost, ms));
                CK(cudaMemcpyAsync(&hz[1], batch->move_off + nR, 8, cudaMemcpyDeviceToHost, ms));
                CK(cudaStreamSynchronize(ms));
                base_m = hz[0];
                nM = hz[1] - base_m;
            }
        } else {
            base_a = batch->atom_off[0];
            base_f = batch->frag_off[0];
            nA = batch->atom_off[n] - base_a;
            nR = batch->frag_off[n] - base_f;
            for (int64_t i = 0; i < n; ++i)   // monotone offsets (cheap, O(n))
                if (batch->atom_off[i + 1] < batch->atom_off[i] || batch->frag_off[i + 1] < batch->frag_off[i])
                    return fail(c, VS_E_PARSE, "ligand %lld: decreasing CSR offsets", (long long)i);
            if (nR > 0) {
                if (!batch->move_off) return fail(c, VS_E_ARG, "null move_off");
                for (int64_t f = 0; f < nR; ++f)
                    if (batch->move_off[f + 1] < batch->move_off[f])
                        return fail(c, VS_E_PARSE, "fragment %lld: decreasing move_off", (long long)f);
                base_m = batch->move_off[0];
                nM = batch->move_off[nR] - base_m;
            }
        }
        if (nA < 0 || nR < 0 || nM < 0) return fail(c, VS_E_PARSE, "negative CSR totals");
        if (nR > 0 && (!batch->frag_axis || (nM > 0 && !batch->move_atoms)))
            return fail(c, VS_E_ARG, "null frag_axis / move_atoms");
        if ((int64_t)S_w * nR >= (1ll << 31)) return fail(c, VS_E_ARG, "too many fragments in one batch");
    }
    c->n = n;
    c->nA = nA;
    c->nR = nR;
    c->nM = nM;
    c->job_pockets.assign(pocket_ids, pocket_ids + n_pockets);

    // ---- stage-1 workspace
    size_t gmax = 0;
    for (int i = 0; i < n_pockets; ++i) {
        auto& d = c->pockets[pocket_ids[i]].d;
        gmax = std::max(gmax, c->pockets[pocket_ids[i]].grid.size() * 4);
    }
    const Stage1 s1 = plan1(n, nA, nR, nM, c->P, c->K, gmax, n_pockets);
    if (s1.end > c->ws_bytes) return fail(c, VS_E_WORKSPACE, "workspace too small (stage 1 needs %zu bytes)", s1.end);
    uint8_t* W = c->ws;
    c->d_featA = (int*)(W + s1.featA);
    c->d_featR = (int*)(W + s1.featR);
    c->d_featM = (int*)(W + s1.featM);
    c->d_cell = (int*)(W + s1.cell);
    c->d_status = (unsigned long long*)(W + s1.status);
    c->d_maxAR = (int*)(W + s1.maxAR);
    c->d_hist = (int*)(W + s1.hist);
    c->d_cell_count = (int*)(W + s1.cell_count);
    c->d_perm = (uint32_t*)(W + s1.perm);
    c->d_bstart = (int64_t*)(W + s1.bstart);
    c->d_bsize = (int*)(W + s1.bsize);
    c->d_weights = (unsigned long long*)(W + s1.weights);
    c->d_own_start = (int64_t*)(W + s1.own_start);
    c->d_own_prefix = (int*)(W + s1.own_prefix);
    c->d_own_ac = (int*)(W + s1.own_ac);
    c->d_own_rec_off = (int64_t*)(W + s1.own_rec_off);
    c->d_pose = (float*)(W + s1.pose);
    c->d_cs = (float*)(W + s1.cs);
    c->d_reftab = (float*)(W + s1.reftab);
    c->d_grid.assign(n_pockets, nullptr);
    for (int i = 0; i < n_pockets; ++i) c->d_grid[i] = (float*)(W + s1.grids + (size_t)i * gmax);
    c->d_order = W + s1.order;
    c->d_frint = (int4*)(W + s1.frint);
    c->d_fown = W + s1.fown;
    c->d_lflag = (int*)(W + s1.lflag);
    const bool rebase = base_a != 0 || base_f != 0 || base_m != 0;
    if (batch->on_device == 1) {
        // borrowed; offsets that do not start at 0 are rebased into workspace copies below
        c->d_atom_off = rebase ? (int64_t*)(W + s1.atom_off) : (int64_t*)batch->atom_off;
        c->d_frag_off = rebase ? (int64_t*)(W + s1.frag_off) : (int64_t*)batch->frag_off;
        c->d_xyz = (float*)batch->xyz;
        c->d_frag_axis = (int32_t*)batch->frag_axis;
        c->d_move_off = rebase ? (int64_t*)(W + s1.move_off) : (int64_t*)batch->move_off;
        c->d_move_atoms = (int32_t*)batch->move_atoms;
        c->d_lid = batch->ligand_id;
        c->d_types = atom_type;
    } else if (batch->on_device == 2) {
        // mapped pinned host memory: the offsets are copied (every rank plans the whole batch);
        // coordinates, axes, moving atoms and ids are read by the kernels over PCIe, only for
        // the ligands this rank docks (the owned-only upload of multi-GPU runs)
        auto mapped = [&](const void* p, const void** out) -> vs_status {
            *out = nullptr;
            if (!p) return VS_OK;
            cudaPointerAttributes at{};
            if (cudaPointerGetAttributes(&at, p) != cudaSuccess || at.type != cudaMemoryTypeHost || !at.devicePointer) {
                cudaGetLastError();
                return fail(c, VS_E_ARG, "on_device = 2 needs pinned (page-locked, mapped) host arrays");
            }
            *out = at.devicePointer;
            return VS_OK;
        };
        const void *px = nullptr, *pa = nullptr, *pm = nullptr, *pl = nullptr, *pt = nullptr;
        vs_status mst;
        if ((mst = mapped(batch->xyz, &px)) || (mst = mapped(batch->frag_axis, &pa)) ||
            (mst = mapped(batch->move_atoms, &pm)) || (mst = mapped(batch->ligand_id, &pl)) ||
            (mst = mapped(atom_type, &pt)))
            return mst;
        c->d_types = (const uint8_t*)pt;
        c->d_atom_off = (int64_t*)(W + s1.atom_off);
        c->d_frag_off = (int64_t*)(W + s1.frag_off);
        c->d_move_off = (int64_t*)(W + s1.move_off);
        c->d_xyz = (float*)px;
        c->d_frag_axis = (int32_t*)pa;
        c->d_move_atoms = (int32_t*)pm;
        c->d_lid = (const uint64_t*)pl;
    } else {
        c->d_atom_off = (int64_t*)(W + s1.atom_off);
        c->d_frag_off = (int64_t*)(W + s1.frag_off);
        c->d_xyz = (float*)(W + s1.xyz);
        c->d_frag_axis = (int32_t*)(W + s1.frag_axis);
        c->d_move_off = (int64_t*)(W + s1.move_off);
        c->d_move_atoms = (int32_t*)(W + s1.move_atoms);
        c->d_lid = batch->ligand_id ? (const uint64_t*)(W + s1.lid) : nullptr;
        c->d_types = typed ? (const uint8_t*)(W + s1.types) : nullptr;
    }

    CK(cudaEventRecord(c->ev_prep0, ms));
    // tables + grids (small H2D), only when they changed since the last submit: a pageable
    // copy queues on the H2D copy engine behind any large transfer in flight (a pipelined
    // caller's next chunk), so an unconditional re-upload would stall every submit on it
    {
        std::vector<long long> sig = {(long long)(uintptr_t)W, c->tables_version, (long long)gmax};
        for (int i = 0; i < n_pockets; ++i) sig.push_back(pocket_ids[i]);
        if (sig != c->uploaded_sig) {
            CK(cudaMemcpyAsync(c->d_pose, c->pose_tab.data(), c->pose_tab.size() * 4, cudaMemcpyHostToDevice, ms));
            CK(cudaMemcpyAsync(c->d_cs, c->cs.data(), c->cs.size() * 4, cudaMemcpyHostToDevice, ms));
            if (c->n_ref)
                CK(cudaMemcpyAsync(c->d_reftab, c->ref_tab.data(), c->ref_tab.size() * 4, cudaMemcpyHostToDevice, ms));
            for (int i = 0; i < n_pockets; ++i) {
                auto& ph = c->pockets[pocket_ids[i]];
                CK(cudaMemcpyAsync(c->d_grid[i], ph.grid.data(), ph.grid.size() * 4, cudaMemcpyHostToDevice, ms));
            }
            c->uploaded_sig = sig;
        }
    }
    c->pkdev.clear();
    int n_types = kMaxChannels;   // typed submit: the fewest channels among the docked pockets
    for (int i = 0; i < n_pockets; ++i) {
        const PocketHost& ph = c->pockets[pocket_ids[i]];
        c->pkdev.push_back(make_pocket_dev(ph.d, c->d_grid[i], typed, ph.nch));
        n_types = std::min(n_types, ph.nch);
    }
    if (n == 0) {
        c->buckets.clear();
        c->owned.clear();
        c->total_slots = 0;
        c->submitted = true;
        return VS_OK;
    }
    if (batch->on_device == 2) {
        CK(cudaMemcpyAsync(c->d_atom_off, batch->atom_off, (n + 1) * 8, cudaMemcpyHostToDevice, ms));
        CK(cudaMemcpyAsync(c->d_frag_off, batch->frag_off, (n + 1) * 8, cudaMemcpyHostToDevice, ms));
        if (nR) CK(cudaMemcpyAsync(c->d_move_off, batch->move_off, (nR + 1) * 8, cudaMemcpyHostToDevice, ms));
    } else if (!batch->on_device) {
        CK(cudaMemcpyAsync(c->d_atom_off, batch->atom_off, (n + 1) * 8, cudaMemcpyHostToDevice, ms));
        CK(cudaMemcpyAsync(c->d_frag_off, batch->frag_off, (n + 1) * 8, cudaMemcpyHostToDevice, ms));
        if (nA) CK(cudaMemcpyAsync(c->d_xyz, batch->xyz, nA * 12, cudaMemcpyHostToDevice, ms));
        if (nR) {
            CK(cudaMemcpyAsync(c->d_frag_axis, batch->frag_axis, nR * 8, cudaMemcpyHostToDevice, ms));
            CK(cudaMemcpyAsync(c->d_move_off, batch->move_off, (nR + 1) * 8, cudaMemcpyHostToDevice, ms));
        }
        if (nM) CK(cudaMemcpyAsync(c->d_move_atoms, batch->move_atoms, nM * 4, cudaMemcpyHostToDevice, ms));
        if (typed && nA) CK(cudaMemcpyAsync((void*)c->d_types, atom_type, nA, cudaMemcpyHostToDevice, ms));
        if (batch->ligand_id)
            CK(cudaMemcpyAsync((void*)c->d_lid, batch->ligand_id, n * 8, cudaMemcpyHostToDevice, ms));
    }

    if (rebase) {   // offsets relative to their first entry (slices of a larger library)
        const bool dev = batch->on_device == 1;
        CK(launch_rebase(dev ? batch->atom_off : c->d_atom_off, c->d_atom_off, n + 1, base_a, ms));
        CK(launch_rebase(dev ? batch->frag_off : c->d_frag_off, c->d_frag_off, n + 1, base_f, ms));
        if (nR) CK(launch_rebase(dev ? batch->move_off : c->d_move_off, c->d_move_off, nR + 1, base_m, ms));
        launches += nR ? 3 : 2;
    }

    // ---- a1 features (every ligand, from the CSR offsets alone) and the range checks
    CK(cudaMemsetAsync(c->d_status, 0xFF, 24, ms));
    CK(cudaMemsetAsync(c->d_maxAR, 0, 16, ms));
    CK(launch_features(c->d_atom_off, c->d_frag_off, c->d_move_off, n, c->d_featA, c->d_featR, c->d_featM, c->d_status,
                       c->d_maxAR, ms));
    ++launches;
    vs_status st = ensure_pinned(c, (size_t)(s1.max_buckets + 16) * 32 + kMaxCells * 8 + 64);
    if (st) return st;
    uint8_t* H = (uint8_t*)c->hpin;
    CK(cudaMemcpyAsync(H, c->d_status, 8, cudaMemcpyDeviceToHost, ms));
    CK(cudaMemcpyAsync(H + 8, c->d_maxAR, 12, cudaMemcpyDeviceToHost, ms));
    CK(cudaStreamSynchronize(ms));
    unsigned long long vstat;
    int maxAR[3];
    std::memcpy(&vstat, H, 8);
    std::memcpy(maxAR, H + 8, 12);
    if (vstat != ~0ull) {
        const long long li = (long long)(vstat >> 8);
        return fail(c, VS_E_PARSE, "ligand %lld: %s", li, vcode_msg((int)(vstat & 255)));
    }

    // ---- a2/a3 boundaries, classes (Eq. 1), classify, scan
    const int ubA = c->cfg.atom_upper_bound > 0 ? c->cfg.atom_upper_bound : maxAR[0];
    const int ubR = c->cfg.rot_upper_bound > 0 ? c->cfg.rot_upper_bound : maxAR[1];
    c->atom_b = atom_bounds(c->cfg.n_atom_clusters, ubA);
    c->rot_b = rot_bounds(c->cfg.n_rot_clusters, ubR);
    if ((int)c->rot_b.size() > kMaxRotClasses) return fail(c, VS_E_ARG, "too many rotamer classes");
    // optional third key sum_r |M_r|: boundaries by the rotamer rule
    // over [0, max]; one class = off
    {
        const int ubM = c->cfg.move_upper_bound > 0 ? c->cfg.move_upper_bound : maxAR[2];
        c->move_b = c->cfg.n_move_clusters > 1 ? rot_bounds(c->cfg.n_move_clusters, ubM) : std::vector<int>{ubM};
        if ((int)c->move_b.size() > kMaxMoveClasses) return fail(c, VS_E_ARG, "too many moving-atom classes");
        if (c->atom_b.size() * c->rot_b.size() * c->move_b.size() > (size_t)kMaxCells)
            return fail(c, VS_E_ARG, "more than %d atom x rotamer x moving-atom cells", kMaxCells);
    }
    // one class table per distinct grid layout among the submitted pockets (each launch uses
    // its pocket's table: policy, occupancy and shared memory differ per layout); the table
    // of the largest layout sizes the buckets (Eq. 1), so capacities fit every pocket
    c->frag_cap = maxAR[1];
    {
        std::vector<std::vector<int>> keys;   // (nz, rs, ps) per layout
        c->layout_classes.clear();
        c->pk_layout.assign(n_pockets, 0);
        int big = 0;
        for (int q = 0; q < n_pockets; ++q) {
            const PocketDev& pk = c->pkdev[q];
            const std::vector<int> key = {pk.mode, pk.nz, pk.rs, pk.ps, pk.nch};
            int li = (int)(std::find(keys.begin(), keys.end(), key) - keys.begin());
            if (li == (int)keys.size()) {
                keys.push_back(key);
                c->layout_classes.emplace_back();
                st = plan_classes(c, c->atom_b, pk.mode, pk.nz, pk.rs, pk.ps, pk.nch, c->frag_cap,
                                  c->layout_classes.back());
                if (st) return st;
                if (dock_grid_floats(pk.mode, pk.nz, pk.rs, pk.ps, pk.nch) >
                    dock_grid_floats(keys[big][0], keys[big][1], keys[big][2], keys[big][3], keys[big][4]))
                    big = li;
            }
            c->pk_layout[q] = li;
        }
        c->classes = c->layout_classes[big];
    }
    const int nRc = (int)c->rot_b.size(), nMc = (int)c->move_b.size();
    const int n_cells = (int)c->atom_b.size() * nRc * nMc;
    CK(launch_classify_hist(c->d_featA, c->d_featR, c->d_featM, n, c->atom_b.data(), (int)c->atom_b.size(),
                            c->rot_b.data(), nRc, c->move_b.data(), nMc,
                            c->d_cell, c->d_hist, s1.n_blocks, c->d_status + 1, ms));
    CK(launch_scan_hist(c->d_hist, n_cells, s1.n_blocks, c->d_cell_count, ms));
    launches += 2;
    CK(cudaMemcpyAsync(H, c->d_status + 1, 8, cudaMemcpyDeviceToHost, ms));
    CK(cudaMemcpyAsync(H + 8, c->d_cell_count, n_cells * 4, cudaMemcpyDeviceToHost, ms));
    CK(cudaStreamSynchronize(ms));
    unsigned long long ovf;
    std::memcpy(&ovf, H, 8);
    if (ovf != ~0ull) {
        const long long li = (long long)(ovf >> 8);
        if ((ovf & 255) == 1)
            return fail(c, VS_E_OVERFLOW_ATOMS, "ligand %lld: atoms above the last atom boundary %d (axis: atoms)", li,
                        c->atom_b.back());
        if ((ovf & 255) == 3)
            return fail(c, VS_E_OVERFLOW_ROTAMERS,
                        "ligand %lld: moving atoms above the last moving-atom boundary %d (axis: moving atoms)", li,
                        c->move_b.back());
        return fail(c, VS_E_OVERFLOW_ROTAMERS, "ligand %lld: rotamers above the last rotamer boundary %d (axis: rotamers)",
                    li, c->rot_b.back());
    }
    std::vector<int> cc(n_cells);
    std::memcpy(cc.data(), H + 8, n_cells * 4);

    // bucket table: cell-major, chunks of the class capacity (Q18)
    c->buckets.clear();
    int64_t run = 0;
    for (int cell = 0; cell < n_cells; ++cell) {
        const int ai = cell / (nRc * nMc), ri = (cell / nMc) % nRc, mi = cell % nMc;
        const ClassInfo& ci = c->classes[ai];
        for (int64_t s = 0; s < cc[cell]; s += ci.cap) {
            vs_bucket b{};
            b.cell = cell;
            b.atom_class = ai;
            b.rot_class = ri;
            b.move_class = mi;
            b.atom_bound = ci.atom_bound;
            b.kernel_atoms = ci.AC;
            b.capacity = ci.cap;
            b.size = (int)std::min<int64_t>(ci.cap, cc[cell] - s);
            b.start = run + s;
            b.owner = -1;
            b.launch_order = -1;
            c->buckets.push_back(b);
        }
        run += cc[cell];
    }
    const int nb = (int)c->buckets.size();
    {
        int64_t* hs = (int64_t*)(H);
        int* hz = (int*)(H + (size_t)nb * 8);
        for (int b = 0; b < nb; ++b) {
            hs[b] = c->buckets[b].start;
            hz[b] = c->buckets[b].size;
        }
        CK(cudaMemcpyAsync(c->d_bstart, hs, (size_t)nb * 8, cudaMemcpyHostToDevice, ms));
        CK(cudaMemcpyAsync(c->d_bsize, hz, (size_t)nb * 4, cudaMemcpyHostToDevice, ms));
    }
    CK(launch_scatter(c->d_cell, n, c->d_hist, n_cells, s1.n_blocks, c->d_perm, ms));
    CK(launch_bucket_weights(c->d_perm, c->d_featA, c->d_featR, c->d_featM, c->d_bstart, c->d_bsize, nb, c->P, c->K,
                             S_w, c->d_weights, ms));
    launches += 2;
    CK(cudaStreamSynchronize(ms));  // pinned staging reused below
    CK(cudaMemcpyAsync(H, c->d_weights, (size_t)nb * 32, cudaMemcpyDeviceToHost, ms));
    CK(cudaStreamSynchronize(ms));
    std::vector<unsigned long long> bsum((size_t)nb * 4);
    std::memcpy(bsum.data(), H, (size_t)nb * 32);
    for (int b = 0; b < nb; ++b) c->buckets[b].weight = bsum[4 * (size_t)b];

    // ---- a4 LPT shard (identical on every rank: a pure function of the manifest)
    {
        std::vector<uint64_t> w(nb);
        std::vector<int32_t> owner(nb), lorder(nb);
        for (int b = 0; b < nb; ++b) w[b] = c->buckets[b].weight;
        lpt_plan(w.data(), nb, c->cfg.world_size, owner.data(), lorder.data());
        std::vector<int> mine;
        for (int b = 0; b < nb; ++b) {
            c->buckets[b].owner = owner[b];
            c->buckets[b].launch_order = lorder[b];
            if (owner[b] == c->cfg.rank) mine.push_back(b);
        }
        std::sort(mine.begin(), mine.end(), [&](int x, int y) { return lorder[x] < lorder[y]; });
        c->owned = mine;
        // bytes this submit moves to the device: copies, or (mapped host input) the offsets plus
        // what the kernels read in place for the owned ligands
        uint64_t oa = 0, of = 0, om = 0, on = 0;
        for (int b : mine) {
            oa += bsum[4 * (size_t)b + 1];   // owned atoms
            of += bsum[4 * (size_t)b + 2];
            om += bsum[4 * (size_t)b + 3];
            on += (uint64_t)c->buckets[b].size;
        }
        const uint64_t offs = (uint64_t)(n + 1) * 16 + (uint64_t)(nR + 1) * 8;
        c->stats.h2d_bytes = batch->on_device == 1 ? 0
                             : batch->on_device == 2
                                 ? offs + (typed ? 13 : 12) * oa + 8 * of + 4 * om + (batch->ligand_id ? 8 * on : 0)
                                 : offs + (uint64_t)nA * (typed ? 13 : 12) + (uint64_t)nR * 8 + (uint64_t)nM * 4 +
                                       (batch->ligand_id ? (uint64_t)n * 8 : 0);
    }
    // fused mode: group the owned buckets by atom class (LPT order kept inside a class)
    // so each class is one contiguous slot range = one persistent launch
    if (!c->cfg.launch_per_bucket)
        std::stable_sort(c->owned.begin(), c->owned.end(),
                         [&](int x, int y) { return c->buckets[x].atom_class < c->buckets[y].atom_class; });

    // ---- stage-2 workspace and a5 pack
    const int no = (int)c->owned.size();
    c->owned_prefix.assign(no + 1, 0);
    c->owned_rec_off.assign(no, 0);
    int64_t rec_floats = 0;
    double evals = 0;
    for (int i = 0; i < no; ++i) {
        const vs_bucket& b = c->buckets[c->owned[i]];
        c->owned_prefix[i + 1] = c->owned_prefix[i] + b.size;
        c->owned_rec_off[i] = rec_floats;
        rec_floats += (int64_t)b.size * rec_floats_typed(b.kernel_atoms, typed);
        evals += (double)b.weight;
    }
    c->total_slots = c->owned_prefix[no];
    const Stage2 s2 = plan2(s1.end, n, nA, nR, rec_floats, c->P, S_w, n_pockets, c->cfg.debug_poses != 0, c->n_ref);
    if (s2.end > c->ws_bytes) return fail(c, VS_E_WORKSPACE, "workspace too small (needs %zu bytes)", s2.end);
    c->d_rec = (float*)(W + s2.rec);
    c->d_meta = (int4*)(W + s2.meta);
    c->d_score.assign(n_pockets, nullptr);
    c->d_pose_best.assign(n_pockets, nullptr);
    c->d_ang.assign(n_pockets, nullptr);
    c->d_dbg_score.assign(n_pockets, nullptr);
    c->d_dbg_ang.assign(n_pockets, nullptr);
    c->d_ref.assign(n_pockets, nullptr);
    c->d_dbg_ref.assign(n_pockets, nullptr);
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    for (int i = 0; i < n_pockets; ++i) {
        c->d_score[i] = (float*)(W + s2.score + i * al(n * 4));
        c->d_pose_best[i] = (int*)(W + s2.pose_best + i * al(n * 4));
        c->d_ang[i] = W + s2.ang + i * al((size_t)S_w * nR);
        if (c->cfg.debug_poses) {
            c->d_dbg_score[i] = (float*)(W + s2.dbg_score + i * al((size_t)n * c->P * 4));
            c->d_dbg_ang[i] = W + s2.dbg_ang + i * al((size_t)c->P * S_w * nR);
            if (c->n_ref) c->d_dbg_ref[i] = W + s2.dbg_ref + i * al((size_t)n * c->P * c->n_ref);
        }
        if (c->n_ref) c->d_ref[i] = W + s2.ref + i * al((size_t)n * c->n_ref);
    }
    c->d_coords.assign(n_pockets, nullptr);
    for (int i = 0; i < n_pockets; ++i) c->d_coords[i] = (float*)(W + s2.coords + i * al((size_t)nA * 12));
    c->d_keys = (unsigned long long*)(W + s2.keys);
    c->keys_cap = std::max<int64_t>(n, 65536);
    c->d_topk_out = (unsigned long long*)(W + s2.topk_out);
    c->d_sel = W + s2.sel;
    int* d_counters = (int*)(W + s2.counters);
    CK(cudaMemsetAsync(d_counters, 0, (size_t)no * n_pockets * 4 + 4, ms));
    {
        int64_t* h_start = (int64_t*)H;
        int* h_prefix = (int*)(H + (size_t)no * 8);
        int* h_ac = (int*)(H + (size_t)no * 12 + 4);
        int64_t* h_roff = (int64_t*)(H + (((size_t)no * 16 + 4 + 7) & ~(size_t)7));
        for (int i = 0; i < no; ++i) {
            h_start[i] = c->buckets[c->owned[i]].start;
            h_ac[i] = c->buckets[c->owned[i]].kernel_atoms;
            h_roff[i] = c->owned_rec_off[i];
        }
        for (int i = 0; i <= no; ++i) h_prefix[i] = c->owned_prefix[i];
        if (no) {
            CK(cudaMemcpyAsync(c->d_own_start, h_start, (size_t)no * 8, cudaMemcpyHostToDevice, ms));
            CK(cudaMemcpyAsync(c->d_own_prefix, h_prefix, (size_t)(no + 1) * 4, cudaMemcpyHostToDevice, ms));
            CK(cudaMemcpyAsync(c->d_own_ac, h_ac, (size_t)no * 4, cudaMemcpyHostToDevice, ms));
            CK(cudaMemcpyAsync(c->d_own_rec_off, h_roff, (size_t)no * 8, cudaMemcpyHostToDevice, ms));
        }
    }
    // ---- a1 ingest of this rank's ligands: per-atom validation, laminar check, canonical
    // renumbering (errors are rank-local: parallel.py carries them through the all-gather)
    CK(launch_ingest(c->d_atom_off, c->d_xyz, c->d_types, n_types, c->d_frag_off, c->d_frag_axis, c->d_move_off, c->d_move_atoms, c->d_perm,
                     c->d_own_start, c->d_own_prefix, no, c->total_slots, c->d_order, c->d_frint, c->d_fown,
                     c->d_lflag, c->d_status + 2, ms));
    ++launches;
    CK(cudaMemcpyAsync(H, c->d_status + 2, 8, cudaMemcpyDeviceToHost, ms));
    CK(cudaStreamSynchronize(ms));
    {
        unsigned long long istat;
        std::memcpy(&istat, H, 8);
        if (istat != ~0ull) {
            const long long li = (long long)(istat >> 8);
            return fail(c, VS_E_PARSE, "ligand %lld: %s", li, vcode_msg((int)(istat & 255)));
        }
    }
    CK(launch_pack(c->d_perm, c->d_own_start, c->d_own_prefix, c->d_own_ac, c->d_own_rec_off, no, c->total_slots,
                   c->d_atom_off, c->d_xyz, c->d_types, c->d_order, c->d_frag_off, c->d_frint, c->d_fown, c->d_lflag, S_w,
                   c->d_rec, c->d_meta, ms));
    ++launches;
    for (int i = 0; i < n_pockets; ++i) {
        CK(launch_fill_results(c->d_score[i], c->d_pose_best[i], n, c->d_ang[i], (int64_t)S_w * nR, ms));
        ++launches;
        if (c->total_slots < n && nA)   // NaN coordinates for the ligands of other ranks
            CK(cudaMemsetAsync(c->d_coords[i], 0xFF, (size_t)nA * 12, ms));
        if (c->n_ref && c->total_slots < n)   // refinement moves of other ranks' ligands: 0xFF
            CK(cudaMemsetAsync(c->d_ref[i], 0xFF, (size_t)n * c->n_ref, ms));
    }
    CK(cudaEventRecord(c->ev_prep1, ms));

    // ---- a6-a9 dock.  Launch units: one per owned bucket (paper mode) or one per atom
    // class (fused: contiguous slot ranges); heaviest first, round-robin over streams.
    struct Unit {
        int cls, first, slots;
        unsigned long long w;
    };
    std::vector<Unit> units;
    for (int i = 0; i < no; ++i) {
        const vs_bucket& b = c->buckets[c->owned[i]];
        if (!c->cfg.launch_per_bucket && !units.empty() && units.back().cls == b.atom_class) {
            units.back().slots += b.size;
            units.back().w += b.weight;
        } else {
            units.push_back({b.atom_class, i, b.size, b.weight});
        }
    }
    if (!c->cfg.launch_per_bucket)
        std::stable_sort(units.begin(), units.end(), [](const Unit& x, const Unit& y) { return x.w > y.w; });
    const int NS = (int)c->workers.size();
    for (int s = 0; s < NS; ++s) CK(cudaStreamWaitEvent(c->workers[s], c->ev_prep1, 0));
    int64_t dock_launches = 0;
    // fused multi-site: all pockets share one grid layout (FIX) -> one cluster
    // launch per unit docks every pocket, the records staged once per cluster (multicast)
    bool fuse = c->cfg.fused_sites && n_pockets >= 2 && n_pockets <= kMaxSites;
    for (int q = 1; fuse && q < n_pockets; ++q) fuse = c->pk_layout[q] == c->pk_layout[0];
    fuse = fuse && (c->pkdev[0].mode == kGridFix || c->pkdev[0].mode == kGridQuad);
    auto base_args = [&](const Unit& u, const ClassInfo& ci) {
        const vs_bucket& b = c->buckets[c->owned[u.first]];
        DockArgs a{};
        a.rec = c->d_rec + c->owned_rec_off[u.first];
        a.meta = c->d_meta + c->owned_prefix[u.first];
        a.n = u.slots;
        a.rec_floats = rec_floats_typed(b.kernel_atoms, typed);
        a.P = c->P;
        a.K = c->K;
        a.S_w = S_w;
        a.ligs_per_cta = ci.LC;
        a.frag_cap = c->frag_cap;
        a.n_sites = 1;
        a.pose_tab = c->d_pose;
        a.cs = c->d_cs;
        a.n_ref = c->n_ref;
        a.n_moves = c->n_moves;
        a.ref_tab = c->d_reftab;
        a.order = c->d_order;
        a.atom_off = c->d_atom_off;
        return a;
    };
    auto site = [&](DockArgs& a, int s, int q) {
        a.pk[s] = c->pkdev[q];
        a.out[s] = SiteOut{c->d_score[q], c->d_pose_best[q], c->d_ang[q], c->d_dbg_score[q], c->d_dbg_ang[q],
                           c->d_coords[q], c->d_ref[q], c->d_dbg_ref[q]};
    };
    c->stats.fused_launches = 0;
    for (const Unit& u : units) {
        const vs_bucket& b = c->buckets[c->owned[u.first]];
        if (fuse) {
            const ClassInfo& ci = c->layout_classes[c->pk_layout[0]][u.cls];
            const PocketDev& p0 = c->pkdev[0];
            const DockLayout L = dock_layout(b.kernel_atoms, ci.NW, ci.PPW, p0.mode, p0.nz, p0.rs, p0.ps, p0.nch, c->P,
                                             c->K, S_w, ci.LC, c->frag_cap, c->n_ref);
            // cluster size g: the one that keeps the most SMs busy (clusters are placed whole
            // inside a GPC, so large clusters of 227 KB CTAs leave SMs idle); ties -> larger g
            int best_g = 1, best_sms = ci.b * c->sm_count, best_cl = 0;
            static const int force_g = [] {   // VSDOCK_CLUSTER=g: measurement override of the cluster size
                const char* e = getenv("VSDOCK_CLUSTER");
                return e ? atoi(e) : 0;
            }();
            for (int g = std::min(n_pockets, kMaxSites); g >= 2; --g) {
                int cl = 0;
                CK(dock_cluster_occupancy(b.kernel_atoms, ci.NW, ci.PPW, p0.mode, c->K, L.total, g, &cl));
                if (getenv("VSDOCK_CLUSTER_LOG"))
                    fprintf(stderr, "class %d: cluster size %d -> %d clusters (%d SMs)\n", b.kernel_atoms, g, cl, cl * g);
                if (force_g > 0 && g != force_g) continue;
                if (cl > 0 && (force_g > 0 || cl * g > best_sms || (best_g == 1 && cl * g * 100 >= best_sms * 97))) {
                    best_g = g;
                    best_sms = cl * g;
                    best_cl = cl;
                }
            }
            if (best_g > 1) {
                const int rounds = (u.slots + ci.LC - 1) / ci.LC;
                for (int q0 = 0; q0 < n_pockets; q0 += best_g) {
                    const int g = std::min(best_g, n_pockets - q0);
                    DockArgs a = base_args(u, ci);
                    a.counter = d_counters + dock_launches;
                    if (g == 1) {
                        site(a, 0, q0);
                        CK(launch_dock(b.kernel_atoms, ci.NW, ci.PPW, a, std::min(rounds, ci.b * c->sm_count), L.total,
                                       c->workers[dock_launches % NS]));
                    } else {
                        a.n_sites = g;
                        for (int s2 = 0; s2 < g; ++s2) site(a, s2, q0 + s2);
                        const int grid = std::min(rounds, best_cl * best_g / g) * g;
                        CK(launch_dock(b.kernel_atoms, ci.NW, ci.PPW, a, grid, L.total, c->workers[dock_launches % NS]));
                        ++c->stats.fused_launches;
                    }
                    ++dock_launches;
                }
                continue;
            }
        }
        for (int q = 0; q < n_pockets; ++q) {
            const ClassInfo& ci = c->layout_classes[c->pk_layout[q]][u.cls];
            DockArgs a = base_args(u, ci);
            site(a, 0, q);
            a.counter = d_counters + dock_launches;
            const DockLayout L = dock_layout(b.kernel_atoms, ci.NW, ci.PPW, a.pk[0].mode, a.pk[0].nz, a.pk[0].rs,
                                             a.pk[0].ps, a.pk[0].nch, c->P, c->K, S_w, ci.LC, c->frag_cap, c->n_ref);
            const int rounds = (u.slots + ci.LC - 1) / ci.LC;
            const int grid = std::min(rounds, ci.b * c->sm_count);
            cudaStream_t s = c->workers[(dock_launches) % NS];
            CK(launch_dock(b.kernel_atoms, ci.NW, ci.PPW, a, grid, L.total, s));
            ++dock_launches;
        }
    }
    for (int s = 0; s < NS; ++s) {
        CK(cudaEventRecord(c->ev_worker[s], c->workers[s]));
        CK(cudaStreamWaitEvent(ms, c->ev_worker[s], 0));
    }
    CK(cudaEventRecord(c->ev_dock1, ms));
    launches += dock_launches;

    c->stats.n_ligands = n;
    c->stats.n_owned = c->total_slots;   // (h2d_bytes was set with the shard)
    c->stats.n_buckets = nb;
    c->stats.n_owned_buckets = no;
    c->stats.kernel_launches = launches;
    c->stats.dock_launches = dock_launches;
    c->stats.evals_alg = evals * n_pockets;
    c->submitted = true;
    return VS_OK;
}
}  // namespace

vs_status vs_submit(vs_ctx* c, const vs_ligand_batch* batch, const int32_t* pocket_ids, int32_t n_pockets) {
    return submit_impl(c, batch, nullptr, pocket_ids, n_pockets);
}

vs_status vs_submit_typed(vs_ctx* c, const vs_ligand_batch* batch, const uint8_t* atom_type, const int32_t* pocket_ids,
                          int32_t n_pockets) {
    if (!atom_type && batch && batch->n > 0) return c ? fail(c, VS_E_ARG, "vs_submit_typed: null atom_type") : VS_E_ARG;
    static const uint8_t none = 0;
    return submit_impl(c, batch, atom_type ? atom_type : &none, pocket_ids, n_pockets);
}

vs_status vs_wait(vs_ctx* c) {
    if (!c) return VS_E_ARG;
    if (!c->submitted) return fail(c, VS_E_STATE, "nothing submitted");
    CK(cudaStreamSynchronize(c->main));
    if (c->n > 0) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, c->ev_prep0, c->ev_prep1));
        c->stats.prep_ms = ms;
        CK(cudaEventElapsedTime(&ms, c->ev_prep1, c->ev_dock1));
        c->stats.dock_ms = ms;
    }
    return VS_OK;
}

vs_status vs_get_results(vs_ctx* c, int32_t slot, uint64_t* ligand_id, float* best_score, int32_t* best_pose,
                         uint8_t* angle_idx, int32_t on_device) {
    if (!c) return VS_E_ARG;
    if (!c->submitted) return fail(c, VS_E_STATE, "nothing submitted");
    if (slot < 0 || slot >= (int)c->job_pockets.size()) return fail(c, VS_E_ARG, "bad pocket slot");
    if (c->n == 0) return VS_OK;
    if (on_device < 0 || on_device > 2) return fail(c, VS_E_ARG, "on_device must be 0, 1 or 2");
    const cudaMemcpyKind kind = on_device == 1 ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    if (ligand_id) {
        if (c->d_lid) CK(cudaMemcpyAsync(ligand_id, c->d_lid, c->n * 8, cudaMemcpyDefault, c->main));
        else if (on_device == 1) return fail(c, VS_E_ARG, "the batch carried no ligand ids (request them on the host)");
        else for (int64_t i = 0; i < c->n; ++i) ligand_id[i] = (uint64_t)i;
    }
    if (best_score) CK(copy_pieces(best_score, c->d_score[slot], c->n * 4, kind, c->main));
    if (best_pose) CK(copy_pieces(best_pose, c->d_pose_best[slot], c->n * 4, kind, c->main));
    if (angle_idx && c->nR) CK(copy_pieces(angle_idx, c->d_ang[slot], (size_t)c->cfg.n_sweeps * c->nR, kind, c->main));
    if (on_device != 2) CK(cudaStreamSynchronize(c->main));   // 2: asynchronous (pinned host), see vsdock.h
    return VS_OK;
}

vs_status vs_get_pose_debug(vs_ctx* c, int32_t slot, float* pose_score, uint8_t* pose_angles) {
    if (!c) return VS_E_ARG;
    if (!c->submitted) return fail(c, VS_E_STATE, "nothing submitted");
    if (!c->cfg.debug_poses) return fail(c, VS_E_STATE, "debug_poses is off");
    if (slot < 0 || slot >= (int)c->job_pockets.size()) return fail(c, VS_E_ARG, "bad pocket slot");
    if (c->n == 0) return VS_OK;
    if (pose_score) CK(cudaMemcpyAsync(pose_score, c->d_dbg_score[slot], (size_t)c->n * c->P * 4, cudaMemcpyDeviceToHost, c->main));
    if (pose_angles && c->nR)
        CK(cudaMemcpyAsync(pose_angles, c->d_dbg_ang[slot], (size_t)c->P * c->cfg.n_sweeps * c->nR, cudaMemcpyDeviceToHost, c->main));
    CK(cudaStreamSynchronize(c->main));
    return VS_OK;
}

vs_status vs_get_refine(vs_ctx* c, int32_t slot, uint8_t* moves, int32_t on_device) {
    if (!c || !moves) return VS_E_ARG;
    if (!c->submitted) return fail(c, VS_E_STATE, "nothing submitted");
    if (slot < 0 || slot >= (int)c->job_pockets.size()) return fail(c, VS_E_ARG, "bad pocket slot");
    if (on_device < 0 || on_device > 2) return fail(c, VS_E_ARG, "on_device must be 0, 1 or 2");
    if (c->n == 0 || c->n_ref == 0) return VS_OK;
    const cudaMemcpyKind kind = on_device == 1 ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    CK(copy_pieces(moves, c->d_ref[slot], (size_t)c->n * c->n_ref, kind, c->main));
    if (on_device != 2) CK(cudaStreamSynchronize(c->main));
    return VS_OK;
}

vs_status vs_get_pose_refine_debug(vs_ctx* c, int32_t slot, uint8_t* pose_moves) {
    if (!c || !pose_moves) return VS_E_ARG;
    if (!c->submitted) return fail(c, VS_E_STATE, "nothing submitted");
    if (!c->cfg.debug_poses) return fail(c, VS_E_STATE, "debug_poses is off");
    if (slot < 0 || slot >= (int)c->job_pockets.size()) return fail(c, VS_E_ARG, "bad pocket slot");
    if (c->n == 0 || c->n_ref == 0) return VS_OK;
    CK(cudaMemcpyAsync(pose_moves, c->d_dbg_ref[slot], (size_t)c->n * c->P * c->n_ref, cudaMemcpyDeviceToHost, c->main));
    CK(cudaStreamSynchronize(c->main));
    return VS_OK;
}

vs_status vs_get_coords(vs_ctx* c, int32_t slot, float* xyz_out, int32_t on_device) {
    if (!c || !xyz_out) return VS_E_ARG;
    if (!c->submitted) return fail(c, VS_E_STATE, "nothing submitted");
    if (slot < 0 || slot >= (int)c->job_pockets.size()) return fail(c, VS_E_ARG, "bad pocket slot");
    if (c->n == 0 || c->nA == 0) return VS_OK;
    if (on_device < 0 || on_device > 2) return fail(c, VS_E_ARG, "on_device must be 0, 1 or 2");
    CK(copy_pieces(xyz_out, c->d_coords[slot], c->nA * 12,
                   on_device == 1 ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c->main));
    if (on_device != 2) CK(cudaStreamSynchronize(c->main));
    return VS_OK;
}

vs_status vs_local_topk(vs_ctx* c, int32_t slot, int32_t k, uint64_t* keys_dev, int32_t* n_valid) {
    if (!c || !keys_dev) return VS_E_ARG;
    if (!c->submitted) return fail(c, VS_E_STATE, "nothing submitted");
    if (slot < 0 || slot >= (int)c->job_pockets.size()) return fail(c, VS_E_ARG, "bad pocket slot");
    if (k < 1 || k > 8192) return fail(c, VS_E_ARG, "k must be in [1, 8192]");
    CK(cudaEventRecord(c->ev_t0, c->main));
    int L = 0;
    if (c->n > 0) {
        CK(launch_make_keys(c->d_meta, c->total_slots, c->d_score[slot], c->d_keys, c->main));
        ++L;
    }
    int l2 = 0;
    CK(topk_select_sort(c->d_keys, c->total_slots, k, (unsigned long long*)keys_dev, c->d_sel, c->main, &l2));
    CK(cudaEventRecord(c->ev_t1, c->main));
    CK(cudaStreamSynchronize(c->main));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->ev_t0, c->ev_t1));
    c->stats.topk_ms = ms;
    c->stats.kernel_launches += L + l2;
    if (n_valid) *n_valid = std::min<int64_t>(k, c->total_slots);
    return VS_OK;
}

vs_status vs_keys(vs_ctx* c, int32_t slot, uint32_t index_offset, uint64_t* keys_dev, int64_t* n_keys) {
    if (!c || !n_keys) return VS_E_ARG;
    if (!c->submitted) return fail(c, VS_E_STATE, "nothing submitted");
    if (slot < 0 || slot >= (int)c->job_pockets.size()) return fail(c, VS_E_ARG, "bad pocket slot");
    if (c->total_slots > 0 && !keys_dev) return VS_E_ARG;
    if ((uint64_t)index_offset + (uint64_t)c->n > 0xffffffffull) return fail(c, VS_E_ARG, "index_offset + n exceeds 2^32");
    if (c->total_slots > 0) {
        CK(launch_make_keys(c->d_meta, c->total_slots, c->d_score[slot], (unsigned long long*)keys_dev, c->main,
                            index_offset));
        ++c->stats.kernel_launches;
    }
    *n_keys = c->total_slots;
    return VS_OK;
}

vs_status vs_select_keys(vs_ctx* c, const uint64_t* keys_dev, int64_t n_keys, int32_t k, uint64_t* out_dev) {
    if (!c || !out_dev || (!keys_dev && n_keys > 0)) return VS_E_ARG;
    if (k < 1 || k > 8192) return fail(c, VS_E_ARG, "k must be in [1, 8192]");
    if (!c->ws || !c->d_sel) return fail(c, VS_E_STATE, "submit a batch first (workspace scratch)");
    int l2 = 0;
    CK(topk_select_sort((const unsigned long long*)keys_dev, n_keys, k, (unsigned long long*)out_dev, c->d_sel, c->main,
                        &l2));
    c->stats.kernel_launches += l2;
    return VS_OK;
}

vs_status vs_merge_topk(vs_ctx* c, const uint64_t* keys_dev, int64_t n_keys, int32_t k, int64_t* index_out,
                        float* score_out, uint64_t* id_out, int32_t* n_out) {
    if (!c || (!keys_dev && n_keys > 0)) return VS_E_ARG;
    if (k < 1 || k > 8192) return fail(c, VS_E_ARG, "k must be in [1, 8192]");
    if (!c->ws || !c->d_topk_out) return fail(c, VS_E_STATE, "submit a batch first (workspace scratch)");
    int l2 = 0;
    CK(topk_select_sort((const unsigned long long*)keys_dev, n_keys, k, c->d_topk_out, c->d_sel, c->main, &l2));
    c->stats.kernel_launches += l2;
    std::vector<unsigned long long> h(k), ids(id_out ? k : 0);
    CK(cudaMemcpyAsync(h.data(), c->d_topk_out, (size_t)k * 8, cudaMemcpyDeviceToHost, c->main));
    if (id_out) {   // ids of the last batch, gathered on the device (after the keys in the scratch)
        unsigned long long* d_ids = c->d_topk_out + 8192;
        CK(launch_gather_ids(c->d_topk_out, k, (const unsigned long long*)c->d_lid, c->submitted ? c->n : 0, d_ids,
                              c->main));
        c->stats.kernel_launches++;
        CK(cudaMemcpyAsync(ids.data(), d_ids, (size_t)k * 8, cudaMemcpyDeviceToHost, c->main));
    }
    CK(cudaStreamSynchronize(c->main));
    int m = 0;
    for (int i = 0; i < k; ++i) {
        if (h[i] == ~0ull) break;
        const uint32_t ord = (uint32_t)(h[i] >> 32);
        const uint32_t bits = (ord & 0x80000000u) ? (ord & 0x7fffffffu) : ~ord;
        float s;
        std::memcpy(&s, &bits, 4);
        if (index_out) index_out[i] = (int64_t)(h[i] & 0xffffffffull);
        if (score_out) score_out[i] = s;
        if (id_out) id_out[i] = ids[i];
        ++m;
    }
    if (n_out) *n_out = m;
    return VS_OK;
}

vs_status vs_get_manifest(vs_ctx* c, int32_t max_buckets, vs_bucket* buckets, int32_t* n_buckets, uint32_t* perm) {
    if (!c || !n_buckets) return VS_E_ARG;
    if (!c->submitted) return fail(c, VS_E_STATE, "nothing submitted");
    *n_buckets = (int32_t)c->buckets.size();
    if (buckets) {
        if (max_buckets < (int)c->buckets.size()) return fail(c, VS_E_ARG, "max_buckets too small");
        std::copy(c->buckets.begin(), c->buckets.end(), buckets);
    }
    if (perm && c->n > 0) {
        CK(cudaMemcpyAsync(perm, c->d_perm, c->n * 4, cudaMemcpyDeviceToHost, c->main));
        CK(cudaStreamSynchronize(c->main));
    }
    return VS_OK;
}

vs_status vs_query_classes(vs_ctx* c, int32_t max_classes, vs_class_info* out, int32_t* n_classes) {
    if (!c || !n_classes) return VS_E_ARG;
    if (c->classes.empty()) return fail(c, VS_E_STATE, "no class table yet (submit a batch)");
    *n_classes = (int32_t)c->classes.size();
    if (out) {
        if (max_classes < (int)c->classes.size()) return fail(c, VS_E_ARG, "max_classes too small");
        for (size_t i = 0; i < c->classes.size(); ++i) {
            const ClassInfo& ci = c->classes[i];
            vs_class_info& o = out[i];
            o.atom_bound = ci.atom_bound;
            o.kernel_atoms = ci.AC;
            o.warps_per_cta = ci.NW;
            o.threads_per_cta = ci.NW * 32;
            o.regs_per_thread = ci.attr.numRegs;
            o.static_smem = (int32_t)ci.attr.sharedSizeBytes;
            o.dyn_smem = (int32_t)ci.smem;
            o.blocks_per_sm = ci.b;
            o.sm_count = c->sm_count;
            o.ligands_per_cta = ci.LC;
            o.l = ci.l;
            o.capacity = ci.cap;
        }
    }
    return VS_OK;
}

namespace {
vs_status score_points_impl(vs_ctx* c, int32_t pocket_id, int64_t n, const float* xyz, const uint8_t* types,
                            float* g_out) {
    if (!c || (n > 0 && (!xyz || !g_out))) return VS_E_ARG;
    if (pocket_id < 0 || pocket_id >= (int)c->pockets.size()) return fail(c, VS_E_ARG, "unknown pocket id");
    if (n == 0) return VS_OK;
    if (types)
        for (int64_t i = 0; i < n; ++i)
            if (types[i] >= c->pockets[pocket_id].nch) return fail(c, VS_E_ARG, "point %lld: type >= channels", (long long)i);
    CK(cudaSetDevice(c->cfg.device));
    // test hook: temporary device buffers (not on the product path)
    const PocketHost& ph = c->pockets[pocket_id];
    float *dg = nullptr, *dx = nullptr, *dout = nullptr, *dt = nullptr;
    struct Free {   // released on every return path
        float** p[4];
        ~Free() {
            for (float** q : p)
                if (*q) cudaFree(*q);
        }
    } guard{{&dg, &dx, &dout, &dt}};
    const size_t gb = ph.grid.size() * 4;
    CK(cudaMalloc(&dg, gb));
    CK(cudaMalloc(&dx, (size_t)n * 12));
    CK(cudaMalloc(&dout, (size_t)n * 4));
    CK(cudaMemcpy(dg, ph.grid.data(), gb, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dx, xyz, (size_t)n * 12, cudaMemcpyHostToDevice));
    if (types) {
        CK(cudaMalloc(&dt, (size_t)n));
        CK(cudaMemcpy(dt, types, (size_t)n, cudaMemcpyHostToDevice));
    }
    PocketDev pk = make_pocket_dev(ph.d, dg, types != nullptr, ph.nch);
    const size_t smem = align16(score_grid_floats(pk) * 4);
    CK(launch_score_points(pk, dx, (const uint8_t*)dt, n, dout, smem, c->main));
    CK(cudaMemcpyAsync(g_out, dout, (size_t)n * 4, cudaMemcpyDeviceToHost, c->main));
    CK(cudaStreamSynchronize(c->main));
    return VS_OK;
}
}  // namespace

vs_status vs_score_points(vs_ctx* c, int32_t pocket_id, int64_t n, const float* xyz, float* g_out) {
    return score_points_impl(c, pocket_id, n, xyz, nullptr, g_out);
}

vs_status vs_score_points_typed(vs_ctx* c, int32_t pocket_id, int64_t n, const float* xyz, const uint8_t* types,
                                float* g_out) {
    if (n > 0 && !types) return c ? fail(c, VS_E_ARG, "vs_score_points_typed: null types") : VS_E_ARG;
    return score_points_impl(c, pocket_id, n, xyz, types, g_out);
}

vs_status vs_plan_boundaries(int32_t n_atom_clusters, int32_t atom_ub, int32_t n_rot_clusters, int32_t rot_ub,
                             int32_t* atom_b, int32_t* n_atom_b, int32_t* rot_b, int32_t* n_rot_b) {
    if (!atom_b || !n_atom_b || !rot_b || !n_rot_b) return VS_E_ARG;
    if (n_atom_clusters < 1 || n_atom_clusters > kMaxAtomClasses || n_rot_clusters < 1 ||
        n_rot_clusters > kMaxRotClasses || atom_ub < 1 || rot_ub < 0 || rot_ub > kMaxFrags)
        return VS_E_ARG;
    const std::vector<int> a = atom_bounds(n_atom_clusters, atom_ub);
    const std::vector<int> r = rot_bounds(n_rot_clusters, rot_ub);
    if ((int)r.size() > kMaxRotClasses) return VS_E_ARG;
    std::copy(a.begin(), a.end(), atom_b);
    std::copy(r.begin(), r.end(), rot_b);
    *n_atom_b = (int32_t)a.size();
    *n_rot_b = (int32_t)r.size();
    return VS_OK;
}

vs_status vs_plan_lpt(const uint64_t* weights, int32_t n_buckets, int32_t world, int32_t* owner,
                      int32_t* launch_order) {
    if (n_buckets < 0 || world < 1 || (n_buckets > 0 && (!weights || !owner || !launch_order))) return VS_E_ARG;
    lpt_plan(weights, n_buckets, world, owner, launch_order);
    return VS_OK;
}

vs_status vs_get_stats(vs_ctx* c, vs_stats* out) {
    if (!c || !out) return VS_E_ARG;
    *out = c->stats;
    return VS_OK;
}

}  // extern "C"
