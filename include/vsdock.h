/*
 * vsdock.h -- C-ABI of the B200-native LiGen dock-and-score hot path
 * (arXiv 2303.06150).  Library: paper_2303_06150_b200/libvsdock.so.
 *
 * Citation keys: P:n = PAPER.md line n, S:n = SPEC.md line n, BJ = BASELINE.json
 * north_star, Qn = DESIGN.md reading n, a1..a11 = SURVEY.md 8(a) rows.
 *
 * The calls follow the paper's statement of the problem: identify docking
 * sites (loaded as pocket grids), dock, score, and "for each
 * docking site, we can rank the input chemical library"; and BJ's
 * "load pocket grids; submit a ligand batch; return best score and pose per
 * ligand".
 *
 * Conventions (all calls):
 *  - every call returns vs_status: VS_OK (0) or a negative code; no exception
 *    crosses the ABI; vs_last_error() returns a message naming the first
 *    offending ligand index / axis where one exists;
 *  - device memory is never allocated by the library: the caller provides one
 *    device workspace (vs_set_workspace, sized by vs_workspace_size);
 *  - host inputs are copied during the call that receives them; the caller may
 *    free them on return.  Device inputs (on_device = 1) are borrowed until
 *    vs_wait returns;
 *  - one vs_ctx per GPU per process; a context is not thread-safe;
 *  - results are deterministic: identical inputs give bit-identical outputs,
 *    for any bucketing grid, bucket multiple and world size (Q22).
 */
#ifndef VSDOCK_H
#define VSDOCK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t vs_status;
enum {
    VS_OK = 0,
    VS_E_ARG = -1,              /* invalid argument / configuration */
    VS_E_PARSE = -2,            /* invalid ligand record (a1): message names ligand index and check */
    VS_E_OVERFLOW_ATOMS = -3,   /* atoms above the last atom boundary (axis "atoms") */
    VS_E_OVERFLOW_ROTAMERS = -4,/* rotamers above the last rotamer boundary (axis "rotamers") */
    VS_E_NOFIT = -5,            /* occupancy query returned b = 0: kernel does not fit */
    VS_E_WORKSPACE = -6,        /* workspace missing or too small */
    VS_E_CUDA = -7,             /* CUDA runtime error */
    VS_E_STATE = -9             /* call out of order (e.g. results before submit) */
};

typedef struct vs_ctx vs_ctx;

typedef struct {
    int32_t device;            /* CUDA device ordinal */
    int32_t n_sweeps;          /* S_w >= 1 (Q13) */
    int32_t n_atom_clusters;   /* atom classes; 1 and 1 = unsorted baseline */
    int32_t n_rot_clusters;    /* rotamer classes */
    int32_t atom_upper_bound;  /* P:236 "upper bound"; 0 = observed maximum */
    int32_t rot_upper_bound;   /* 0 = observed maximum */
    int32_t bucket_multiple;   /* m: bucket capacity = m * l_c ("a multiple") */
    int32_t n_streams;         /* concurrent bucket launches (1..16) */
    int32_t rank, world_size;  /* this context docks the buckets LPT assigns to `rank` (a4) */
    int32_t debug_poses;       /* 1: keep every pose's score and angle sequence (parity replay) */
    int32_t launch_per_bucket; /* 1: one kernel launch per bucket, as the paper does;
                                  0 (default): the owned buckets of one atom class run as ONE
                                  persistent launch with dynamic ligand scheduling */
    int32_t bucket_capacity;   /* > 0: every bucket holds this many ligands instead of m * l_c
                                  (the bucket-size sweep of P:283-333); 0 = Eq. 1 */
    int32_t n_move_clusters;   /* classes of an optional THIRD bucketing key, the moving-atom count
                                  sum_r |M_r|; 1 (or 0) = off, <= 8; boundaries
                                  by the rotamer rule over [0, move_upper_bound] */
    int32_t move_upper_bound;  /* 0 = observed maximum */
    int32_t fused_sites;       /* 1: a submit with 2..8 pockets of one 32^3-class grid layout docks
                                  them in ONE launch per atom class: thread-block clusters of one
                                  CTA per pocket, each ligand round staged once per cluster
                                  (multicast TMA).  0: one launch per pocket */
    void* stream;             /* cudaStream_t the library orders its work on (e.g. torch's); NULL = own */
} vs_config;

/* Create a context on cfg->device.  Fills the kernel class table (registers,
 * shared memory) with cudaFuncGetAttributes.  Errors: VS_E_ARG, VS_E_CUDA. */
vs_status vs_create(const vs_config* cfg, vs_ctx** out);
void vs_destroy(vs_ctx* ctx);
const char* vs_last_error(const vs_ctx* ctx);

/* Upper bound of the device workspace for a batch of n_lig ligands with
 * n_atoms atoms, n_frags fragments and n_moving moving-atom entries in total
 * (the lengths of xyz / 3, frag_axis / 2 and move_atoms of vs_ligand_batch) and at
 * most max_atoms atoms per ligand, docked into n_pockets pockets with the current
 * pose table.  Requires the pose table.  Errors: VS_E_ARG, VS_E_STATE. */
vs_status vs_workspace_size(vs_ctx* ctx, int64_t n_lig, int64_t n_atoms, int64_t n_frags, int64_t n_moving,
                            int32_t max_atoms, int32_t n_pockets, size_t* bytes);
/* Hand the library a device buffer (e.g. a torch uint8 tensor) of >= bytes; 256-B aligned. */
vs_status vs_set_workspace(vs_ctx* ctx, void* dev_ptr, size_t bytes);

/* D3: a pocket grid.  Node (i,j,k) sits at origin + spacing*(i,j,k) (Q9); values
 * are fp32 [nz][ny][nx], x fastest.  out_slope = kappa, the continuous
 * out-of-box penalty per Angstrom of L1 excess (Q9).  center = c of a6. */
typedef struct {
    int32_t nx, ny, nz;
    float origin[3];
    float spacing;
    float center[3];
    float out_slope;
} vs_pocket_desc;

/* Load (copy) a pocket grid; host or device pointer.  The grid must be finite,
 * nx,ny,nz >= 2 and fit in shared memory together with the kernel's other
 * buffers (else VS_E_NOFIT at submit).  Returns its id in *pocket_id.  The
 * library keeps at most 16 pockets; each is nx*ny*nz*4 bytes of an internal
 * host copy that is uploaded into the workspace at submit. */
vs_status vs_load_pocket(vs_ctx* ctx, const vs_pocket_desc* desc, const float* grid, int32_t on_device, int32_t* pocket_id);

/* Method variant (reading Q24): a TYPED pocket of n_channels grids
 * G_0 .. G_{T-1} of one geometry (desc), grids = [T][nz][ny][nx] fp32 (host, or device with
 * on_device = 1), 1 <= T <= 8.  A typed submit (vs_submit_typed) scores atom i of type t_i on
 * G_{t_i} (the out-of-box term is shared); a plain vs_submit docks on G_0.  Each channel is
 * copied like vs_load_pocket's grid (T padded copies).  Errors: as vs_load_pocket. */
vs_status vs_load_pocket_typed(vs_ctx* ctx, const vs_pocket_desc* desc, int32_t n_channels, const float* grids,
                               int32_t on_device, int32_t* pocket_id);

/* a6 initial poses (Q7): P rotations rot[P*9] (row-major R_p) and translations
 * trans[P*3] (tau_p), host memory, fp32.  1 <= P <= 1024. */
vs_status vs_set_pose_table(vs_ctx* ctx, int32_t P, const float* rot, const float* trans);

/* a7 angle steps (Q3): cos_sin[K*2], host, fp32; entry 0 must be exactly (1, 0);
 * 1 <= K <= 32 (theta_k = 2 pi k / K for any K; a K that is not a power of two runs on
 * the lane map of the next power of two, the extra lanes idle -- DESIGN.md 6). */
vs_status vs_set_angle_table(vs_ctx* ctx, int32_t K, const float* cos_sin);

/* Method variant (reading Q23): rigid refinement after the
 * sweeps.  n_rounds greedy rounds; each scores the n_moves rigid moves of the table about
 * the pose's current centroid ybar -- y' = Q_m (y - ybar) + ybar + d_m for every atom --
 * and applies the lowest move index attaining the minimum (Q11).  rot[n_moves*9] (Q_m,
 * row-major), trans[n_moves*3] (d_m, Angstrom), host memory, fp32, finite; move 0 must be
 * exactly the identity (Q = I, d = 0), so no round raises the score.  0 <= n_rounds <= 8,
 * 1 <= n_moves <= 32; n_rounds = 0 turns the variant off (the default).  Applies to the
 * following submits; the chosen moves come back through vs_get_refine, and vs_get_coords
 * returns the refined best pose. */
vs_status vs_set_refine_table(vs_ctx* ctx, int32_t n_rounds, int32_t n_moves, const float* rot, const float* trans);

/* D1: a ligand batch in CSR form.  Ligand i has atoms atom_off[i] ..
 * atom_off[i+1] (1 <= A <= 256) with coordinates xyz[3*atom] in Angstrom (finite,
 * |x| <= 1e6), and fragments f = frag_off[i] .. frag_off[i+1] (0 <= R <= 32).
 * Fragment f is a rotatable bond: axis frag_axis[2f] = a -> frag_axis[2f+1] = b
 * (ligand-local atom indices, b on the moving side) and the moving-atom set
 * M_f = move_atoms[move_off[f] .. move_off[f+1]) -- ANY subset of the ligand's atoms
 * ("a subset of the molecule atoms that can rotate"), axis atoms
 * excluded, 1 <= |M_f| <= A - 2, no repeats.  The moving sets of one ligand must form a
 * laminar family (any two nested or disjoint: what the bonds of a tree give) -- a1
 * checks it and renumbers the atoms on the device so that every set is one contiguous
 * range ("a1 ingest"); results come back in the caller's atom order.
 * Fragments are swept in input order (Q4).  ligand_id[n] (may be NULL: ids = batch
 * indices) is passed through to vs_get_results and vs_merge_topk.  The offsets may
 * start at any value b (a slice of a larger library): offset o addresses element o - b
 * of its data array, so xyz, frag_axis and move_atoms point at the slice's first
 * element.  Offsets must not decrease.  on_device = 1: every pointer is a device
 * pointer (borrowed until vs_wait); 0: host memory, copied during vs_submit;
 * 2: PINNED (page-locked) host memory, mapped: the three offset arrays are copied, and
 * the kernels read coordinates, axes, moving atoms and ids over PCIe only for the
 * ligands this rank docks -- each GPU moves its own share, as the paper's per-GPU
 * workers copy their own buckets; borrowed until vs_wait. */
typedef struct {
    int64_t n;
    const uint64_t* ligand_id;   /* [n] or NULL */
    const int64_t* atom_off;     /* [n + 1] */
    const float* xyz;            /* [3 * atom_off[n]] */
    const int64_t* frag_off;     /* [n + 1] */
    const int32_t* frag_axis;    /* [2 * frag_off[n]] (a, b) */
    const int64_t* move_off;     /* [frag_off[n] + 1] */
    const int32_t* move_atoms;   /* [move_off[frag_off[n]]] */
    int32_t on_device;
} vs_ligand_batch;

/* Run the hot path a1..a9 for the batch against pockets pocket_ids[0..n_pockets):
 * a1 features + range checks (A, R) of every ligand (all ranks agree on them), the plan
 * (a2-a4), then a1's per-atom checks and renumbering for THIS rank's ligands only -- a
 * VS_E_PARSE for one of them is rank-local (parallel.py carries it through the all-gather
 * so no rank waits on a collective the others never reach); then pack and dock.
 * validate, classify, bucket (stable), LPT-shard, pack, and dock this rank's
 * buckets into every pocket.  Asynchronous after the three small host syncs of
 * the preparation phase; results are valid after vs_wait.  The pose / angle
 * tables and pocket grids are uploaded into the workspace only when they (or the
 * workspace) changed since the previous submit, so a submit of a device batch
 * issues no host-to-device copy of its own besides the bucket tables.
 * Errors: VS_E_PARSE (first invalid ligand), VS_E_OVERFLOW_*, VS_E_NOFIT,
 * VS_E_WORKSPACE, VS_E_STATE (tables/pockets/workspace missing), VS_E_CUDA. */
vs_status vs_submit(vs_ctx* ctx, const vs_ligand_batch* batch, const int32_t* pocket_ids, int32_t n_pockets);
/* Q24: vs_submit with per-atom types atom_type[atom_off[n] - atom_off[0]] (u8, the caller's atom
 * order, the same memory kind as batch->on_device: host copied, device borrowed, or mapped pinned
 * host read in place for the owned ligands only).  Every pocket docks in a typed layout (DESIGN.md
 * 6): TYPED for one channel (a QUAD window in shared memory), TYPED_S for two or more (one scalar
 * window per channel, ~1.6x the edge for the same shared memory), the padded channels in global
 * memory behind the windows; both give bit-identical results (environment override for
 * measurement: VSDOCK_TYPED_LAYOUT=quad|scalar).  A type >= the channels of any docked pocket is VS_E_PARSE naming the
 * ligand (rank-local, like a1's per-atom checks). */
vs_status vs_submit_typed(vs_ctx* ctx, const vs_ligand_batch* batch, const uint8_t* atom_type,
                          const int32_t* pocket_ids, int32_t n_pockets);
vs_status vs_wait(vs_ctx* ctx);

/* a9 per-ligand results for pocket slot s (index into the submit's pocket_ids),
 * input order, length n: ligand id (the batch's, or the batch index when it gave
 * none), best score S_{p*}, best pose p*, and the angle index sequence of p*, CSR by
 * n_sweeps*frag_off (angle_idx[S_w*frag_off[i] + sw*R_i + r]).
 * Ligands docked by another rank: score NaN, pose -1, angles 0xFF.
 * Any output pointer may be NULL.  on_device: 1 = outputs are device pointers (copied,
 * synchronous); 0 = host memory (synchronous); 2 = host memory, copied ASYNCHRONOUSLY on
 * the context's stream (pinned memory for overlap; complete after the next vs_wait) --
 * the double-buffered result read-back of P:200-203. */
vs_status vs_get_results(vs_ctx* ctx, int32_t slot, uint64_t* ligand_id, float* best_score, int32_t* best_pose,
                         uint8_t* angle_idx, int32_t on_device);
/* a9 best-pose coordinates (Angstrom, the caller's input atom order, [3*n_atoms]) of
 * pocket slot s, computed by the dock kernel itself (the warp that picks p* replays it
 * bit-identically to the docked trajectory); ligands of other ranks: NaN.  on_device as
 * for vs_get_results (2: asynchronous into pinned host memory). */
vs_status vs_get_coords(vs_ctx* ctx, int32_t slot, float* xyz_out, int32_t on_device);
/* Q23: the refinement moves of p* for pocket slot s, [n * n_rounds] (ligand i's rounds at
 * i*n_rounds); ligands of other ranks: 0xFF.  Nothing is written when refinement is off.
 * on_device as for vs_get_results. */
vs_status vs_get_refine(vs_ctx* ctx, int32_t slot, uint8_t* moves, int32_t on_device);
/* Parity hook (requires debug_poses): every pose's refinement moves [n * P * n_rounds]. */
vs_status vs_get_pose_refine_debug(vs_ctx* ctx, int32_t slot, uint8_t* pose_moves);
/* Parity hook (requires debug_poses): every pose's final score [n*P] and angle
 * sequence [P*S_w*frag_off ...] (pose p of ligand i at P*S_w*frag_off[i] + p*S_w*R_i). */
vs_status vs_get_pose_debug(vs_ctx* ctx, int32_t slot, float* pose_score, uint8_t* pose_angles);

/* a10: the k smallest keys (ord(score) << 32 | ligand index) over this rank's
 * ligands for pocket slot s, ascending, into keys_dev[k] (DEVICE); missing
 * entries (fewer than k ligands) are UINT64_MAX.  *n_valid = min(k, owned).
 * ord maps fp32 to unsigned order (sign-flip), -0 is canonicalised to +0. */
vs_status vs_local_topk(vs_ctx* ctx, int32_t slot, int32_t k, uint64_t* keys_dev, int32_t* n_valid);
/* a10 for streamed libraries: the keys (ord(score) << 32 | (ligand index + index_offset))
 * of every ligand this rank docked for pocket slot s, in slot order (unsorted), written
 * asynchronously on the context's stream into keys_dev (DEVICE, capacity >= the owned
 * ligand count, returned in *n_keys).  A caller docking a library in chunks collects each
 * chunk's keys (index_offset = the chunk's first ligand) and ranks them all at once with
 * vs_merge_topk.  Errors: VS_E_ARG (index_offset + n >= 2^32), VS_E_STATE. */
vs_status vs_keys(vs_ctx* ctx, int32_t slot, uint32_t index_offset, uint64_t* keys_dev, int64_t* n_keys);
/* a10 for streamed libraries: the k smallest of n_keys keys (DEVICE, e.g. every chunk's
 * vs_keys output), ascending and UINT64_MAX padded, into out_dev[k] (DEVICE), asynchronously
 * on the context's stream -- the rank's local top-k before the all-gather.  Errors:
 * VS_E_ARG, VS_E_STATE (no workspace yet). */
vs_status vs_select_keys(vs_ctx* ctx, const uint64_t* keys_dev, int64_t n_keys, int32_t k, uint64_t* out_dev);
/* a11: merge n_keys gathered keys (DEVICE, e.g. after an NCCL all_gather of W
 * local top-k lists; UINT64_MAX pads allowed, any number) into the global top-k:
 * ligand index, score and -- id_out non-NULL -- the ligand id from the last
 * submitted batch (UINT64_MAX for an index outside it) (HOST outputs, any may be NULL).
 * *n_out = number of real (non-pad) entries, <= k. */
vs_status vs_merge_topk(vs_ctx* ctx, const uint64_t* keys_dev, int64_t n_keys, int32_t k, int64_t* index_out,
                        float* score_out, uint64_t* id_out, int32_t* n_out);

/* a3/a4 bucket manifest of the last submit (all buckets of all ranks). */
typedef struct {
    int32_t cell, atom_class, rot_class;
    int32_t atom_bound;        /* inclusive upper atom threshold of the class */
    int32_t kernel_atoms;      /* A_c: template atom capacity (multiple of 32) */
    int32_t capacity;          /* m * l_c (Eq. 1) */
    int32_t size;              /* ligands (<= capacity; the last of a cell may be partial) */
    int32_t owner;             /* rank docking it (LPT) */
    int32_t launch_order;      /* position in the owner's launch sequence */
    int32_t move_class;        /* class of the optional third key (0 when off) */
    int64_t start;             /* first position in perm */
    uint64_t weight;           /* sum of E_alg over the bucket's ligands */
} vs_bucket;
/* n_buckets is always written; buckets[] (capacity max_buckets) and perm[n]
 * (cell-major stable order of ligand indices) are written when non-NULL. */
vs_status vs_get_manifest(vs_ctx* ctx, int32_t max_buckets, vs_bucket* buckets, int32_t* n_buckets, uint32_t* perm);

/* The B200 analogue of Table 1 and Eq. 1 per atom class of
 * the last submit (or of the grid implied by the config and pocket 0). */
typedef struct {
    int32_t atom_bound, kernel_atoms;
    int32_t warps_per_cta, threads_per_cta;
    int32_t regs_per_thread, static_smem, dyn_smem;
    int32_t blocks_per_sm;     /* b: cudaOccupancyMaxActiveBlocksPerMultiprocessor */
    int32_t sm_count;          /* SM */
    int32_t ligands_per_cta;   /* t/ws (Q19) */
    int32_t l;                 /* Eq. 1: b * SM * ligands_per_cta */
    int32_t capacity;          /* bucket_multiple * l */
} vs_class_info;
vs_status vs_query_classes(vs_ctx* ctx, int32_t max_classes, vs_class_info* out, int32_t* n_classes);

/* Test hook: g(y) (a8) of pocket_id at n points xyz[3n] (Angstrom, host), into
 * g_out[n] (host), computed by the dock kernel's own device function. */
vs_status vs_score_points(vs_ctx* ctx, int32_t pocket_id, int64_t n, const float* xyz, float* g_out);
/* Test hook (Q24): g_{types[i]}(xyz[i]) of a typed pocket (types[n] host, each < its channels),
 * by the TYPED layout's device function. */
vs_status vs_score_points_typed(vs_ctx* ctx, int32_t pocket_id, int64_t n, const float* xyz, const uint8_t* types,
                                float* g_out);

typedef struct {
    int64_t n_ligands, n_owned;
    int64_t n_buckets, n_owned_buckets;
    int64_t kernel_launches;   /* kernels launched by the last submit (+ topk/coords calls since) */
    int64_t dock_launches;
    int64_t fused_launches;    /* dock launches that were fused multi-site cluster launches */
    double evals_alg;          /* sum over owned ligands and pockets of E_alg (SURVEY 8 'E_alg') */
    uint64_t h2d_bytes;        /* bytes the submit moved host -> device: copies (on_device 0), or
                                  the offsets + the owned ligands' arrays read in place (2); 0 for 1 */
    float prep_ms;             /* validate .. pack (CUDA events) */
    float dock_ms;             /* all dock launches, first start to last end (CUDA events) */
    float topk_ms;             /* last vs_local_topk */
} vs_stats;
vs_status vs_get_stats(vs_ctx* ctx, vs_stats* out);

/* Host-only planning steps of vs_submit, exported so every rank's plan can be
 * checked without a GPU.  Both are pure functions of their inputs.
 *
 * a2 class boundaries: atom classes [32, 64, ..., 32(n-1), last] with last =
 * atom_ub if atom_ub >= 32(n-1)+1 else 32n (reading Q16); rotamer
 * classes per S:215-223 with prev_0 = -1 and round-half-up (Q17).  Capacities:
 * atom_b[8], rot_b[33].  Errors: VS_E_ARG. */
vs_status vs_plan_boundaries(int32_t n_atom_clusters, int32_t atom_ub, int32_t n_rot_clusters, int32_t rot_ub,
                             int32_t* atom_b, int32_t* n_atom_b, int32_t* rot_b, int32_t* n_rot_b);
/* a4 LPT: buckets by weight descending (ties: lower id first) go to the
 * least-loaded rank (ties: lowest rank); owner[b] and launch_order[b] (position
 * in the owner's sequence) for n_buckets buckets.  Errors: VS_E_ARG. */
vs_status vs_plan_lpt(const uint64_t* weights, int32_t n_buckets, int32_t world, int32_t* owner,
                      int32_t* launch_order);

#ifdef __cplusplus
}
#endif
#endif /* VSDOCK_H */
