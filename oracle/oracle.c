/*
 * oracle/oracle.c -- plain, slow, obviously-correct fp64 CPU oracle of the
 * LiGen dock-and-score hot path (arXiv 2303.06150 as read in DESIGN.md).
 *
 * TEST INFRASTRUCTURE.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no
 * code, header, table or constant with the CUDA path
 * (paper_2303_06150_b200/), and it never consumes a value produced there
 * except as the *subject* of a check (oracle_replay_pose replays a k sequence
 * handed to it).
 *
 * Citations: P:n = PAPER.md line n, S:n = SPEC.md line n, BJ = BASELINE.json
 * north_star, Qn = DESIGN.md reading n.  The paper does not define the docking
 * algorithm (P:215 defers to its ref. [9817028]; S:8 puts it out of scope); the
 * steps below follow BJ's sentence "a rigid roto-translation from many initial
 * poses, a rotatable-bond sweep that rotates each fragment through discrete
 * angle steps, and a pocket-grid score by trilinear interpolation with
 * best-pose reduction", in that order, with the readings Q2-Q13 of DESIGN.md.
 *
 * Form: fp64 arithmetic on the fp32 input data, scalar loops, FULL-SUM scores
 * (every candidate k is scored as the sum over all atoms of the ligand,
 * no delta trick, no caching), no blocking, no SIMD.  Threads only split the
 * ligand list.
 *
 * Fragments come in the C-ABI's general form: axis (a, b) and the
 * moving-atom set M_r as an index list (a rotamer is "a subset
 * of the molecule atoms that can rotate"); the oracle rotates exactly the listed atoms
 * and never renumbers them (the CUDA path's DFS renumbering is checked against it).
 *
 * Rigid refinement after the sweeps (Q23): n_ref rounds over a
 * caller-given table of J rigid moves about the pose's centroid, same greedy rule.
 *
 * Per-atom-type grid channels (Q24): the pocket holds T grids of one
 * geometry, G_0 .. G_{T-1}; atom i of type t_i is scored on G_{t_i}.  No types = every atom type 0.
 *
 * Pins: tests/test_oracle_pins.py (closed forms, invariants, brute force,
 * library routines scipy.ndimage.map_coordinates / scipy Rotation, renumbering
 * invariance, pose translations tau_p != 0 and a docking centre off the grid centre).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int n[3];            /* nx, ny, nz */
    double o[3];         /* origin: node (i,j,k) sits at o + h*(i,j,k)  (Q9) */
    double h;            /* spacing, Angstrom */
    double c[3];         /* pocket centre */
    double kappa;        /* out-of-box slope, energy per Angstrom (Q9) */
    int T;               /* grid channels (Q24); 1 = the untyped method */
    const float* G;      /* values [T][nz][ny][nx], x fastest */
} opocket;

/* node (i, j, k) of channel t */
static double node(const opocket* pk, int t, int i, int j, int k) {
    return (double)pk->G[(((size_t)t * pk->n[2] + k) * pk->n[1] + j) * pk->n[0] + i];
}

static double lerp(double a, double b, double f) { return (1.0 - f) * a + f * b; }  /* Q10 */

/*
 * a8: pocket-grid score g(y) by trilinear interpolation (BJ "pocket-grid score
 * by trilinear interpolation").  Per axis (Q9): u = (y - o)/h, u_c = clamp(u,
 * 0, n-1), excess e += |u - u_c|, i0 = min(floor(u_c), n-2), f = u_c - i0.
 * Interpolate x, then y, then z (Q10).  g = interp + kappa*h*e.  Channel t (Q24) selects the
 * grid G_t; the geometry and the out-of-box term are the same for every channel.
 */
double oracle_grid_score(const opocket* pk, int t, const double y[3]) {
    int i0[3];
    double f[3], e = 0.0;
    for (int a = 0; a < 3; ++a) {
        double u = (y[a] - pk->o[a]) / pk->h;
        double top = (double)(pk->n[a] - 1);
        double uc = u < 0.0 ? 0.0 : (u > top ? top : u);
        e += fabs(u - uc);
        int i = (int)floor(uc);
        if (i > pk->n[a] - 2) i = pk->n[a] - 2;
        i0[a] = i;
        f[a] = uc - (double)i;
    }
    int i = i0[0], j = i0[1], k = i0[2];
    double l00 = lerp(node(pk, t, i, j, k), node(pk, t, i + 1, j, k), f[0]);
    double l10 = lerp(node(pk, t, i, j + 1, k), node(pk, t, i + 1, j + 1, k), f[0]);
    double l01 = lerp(node(pk, t, i, j, k + 1), node(pk, t, i + 1, j, k + 1), f[0]);
    double l11 = lerp(node(pk, t, i, j + 1, k + 1), node(pk, t, i + 1, j + 1, k + 1), f[0]);
    double l0 = lerp(l00, l10, f[1]);
    double l1 = lerp(l01, l11, f[1]);
    double v = lerp(l0, l1, f[2]);
    return v + pk->kappa * pk->h * e;
}

/* S(y) = sum_i g_{t_i}(y_i): the interaction score of a pose (lower is better, Q2);
 * ty = the ligand's atom types (Q24), NULL = all type 0. */
static double score(const opocket* pk, const double* y, int A, const uint8_t* ty) {
    double s = 0.0;
    for (int i = 0; i < A; ++i) s += oracle_grid_score(pk, ty ? ty[i] : 0, y + 3 * i);
    return s;
}

/*
 * a6: rigid roto-translation of the ligand into pose p (BJ "rigid
 * roto-translation from many initial poses"; Q7, Q8):
 *   y_i = R_p (x_i - xbar) + c + tau_p,   xbar = (1/A) sum_i x_i.
 */
void oracle_place_pose(const opocket* pk, const float* xyz, int A, const float* rot9, const float* tr3, double* y) {
    double xb[3] = {0, 0, 0};
    for (int i = 0; i < A; ++i)
        for (int a = 0; a < 3; ++a) xb[a] += (double)xyz[3 * i + a];
    for (int a = 0; a < 3; ++a) xb[a] /= (double)A;
    for (int i = 0; i < A; ++i) {
        double d[3];
        for (int a = 0; a < 3; ++a) d[a] = (double)xyz[3 * i + a] - xb[a];
        for (int r = 0; r < 3; ++r) {
            double s = 0.0;
            for (int a = 0; a < 3; ++a) s += (double)rot9[3 * r + a] * d[a];
            y[3 * i + r] = s + pk->c[r] + (double)tr3[r];
        }
    }
}

/*
 * a7: rotate fragment r -- rotation axis a -> b, moving-atom set M_r (an arbitrary
 * subset of the atoms, axis atoms excluded: "a subset of the
 * molecule atoms that can rotate") -- by the angle step with table entry
 * (cos_k, sin_k) (Q3, Q5, Q6):
 *   u = (y_b - y_a)/|y_b - y_a|,  q = y_b,
 *   M = c I + s [u]_x + (1 - c) u u^T   (Rodrigues),
 *   y_i <- q + M (y_i - q)   for i in M_r  (mv[0..nm)).
 */
void oracle_rotate_fragment(double* y, int a, int b, const int32_t* mv, int nm, double ck, double sk) {
    if (ck == 1.0 && sk == 0.0) return;   /* theta = 0: M = I, the coordinates do not move (Q3) */
    double d[3], u[3], q[3];
    for (int t = 0; t < 3; ++t) d[t] = y[3 * b + t] - y[3 * a + t];
    double nrm = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    for (int t = 0; t < 3; ++t) { u[t] = d[t] / nrm; q[t] = y[3 * b + t]; }
    double M[3][3];
    double ux[3][3] = {{0.0, -u[2], u[1]}, {u[2], 0.0, -u[0]}, {-u[1], u[0], 0.0}};
    for (int r = 0; r < 3; ++r)
        for (int s = 0; s < 3; ++s)
            M[r][s] = (r == s ? ck : 0.0) + sk * ux[r][s] + (1.0 - ck) * u[r] * u[s];
    for (int t = 0; t < nm; ++t) {
        const int i = mv[t];
        double v[3];
        for (int c = 0; c < 3; ++c) v[c] = y[3 * i + c] - q[c];
        for (int r = 0; r < 3; ++r) y[3 * i + r] = q[r] + M[r][0] * v[0] + M[r][1] * v[1] + M[r][2] * v[2];
    }
}

/* Fragment f of a general-form CSR batch: axis (frag_axis[2f], frag_axis[2f+1]), M_f =
 * move_atoms[move_off[f] .. move_off[f+1]). */
static void rotate_frag_csr(double* y, const int32_t* frag_axis, const int64_t* move_off, const int32_t* move_atoms,
                            int64_t f, double ck, double sk) {
    oracle_rotate_fragment(y, frag_axis[2 * f], frag_axis[2 * f + 1], move_atoms + move_off[f],
                           (int)(move_off[f + 1] - move_off[f]), ck, sk);
}

/*
 * SURVEY 8(f) 4(b), reading Q23: rigid refinement move m of the move table (rotation Q_m,
 * row-major, and translation d_m in Angstrom) applied about the CURRENT centroid of the
 * pose, ybar = (1/A) sum_i y_i (Q8):  y_i <- Q_m (y_i - ybar) + ybar + d_m  for every atom.
 */
void oracle_rigid_move(double* y, int A, const float* q9, const float* d3) {
    double yb[3] = {0, 0, 0};
    for (int i = 0; i < A; ++i)
        for (int a = 0; a < 3; ++a) yb[a] += y[3 * i + a];
    for (int a = 0; a < 3; ++a) yb[a] /= (double)A;
    for (int i = 0; i < A; ++i) {
        double v[3];
        for (int a = 0; a < 3; ++a) v[a] = y[3 * i + a] - yb[a];
        for (int r = 0; r < 3; ++r) {
            double s = 0.0;
            for (int a = 0; a < 3; ++a) s += (double)q9[3 * r + a] * v[a];
            y[3 * i + r] = s + yb[r] + (double)d3[r];
        }
    }
}

/*
 * One refinement round (Q23): score every move m of the table (full sum over all atoms, as
 * for the angle steps), keep the lowest m attaining the minimum (Q11), apply it.  scores[m]
 * (optional) receives S_m; *margin (optional) the relative gap of the runner-up.
 */
static int refine_round(const opocket* pk, double* y, double* ytmp, int A, const uint8_t* ty, int J, const float* qrot,
                        const float* dtr, double* scores, double* margin) {
    double smin = INFINITY, s2 = INFINITY;
    int mmin = 0;
    for (int m = 0; m < J; ++m) {
        memcpy(ytmp, y, sizeof(double) * 3 * (size_t)A);
        oracle_rigid_move(ytmp, A, qrot + 9 * m, dtr + 3 * m);
        double sc = score(pk, ytmp, A, ty);
        if (scores) scores[m] = sc;
        if (sc < smin) { s2 = smin; smin = sc; mmin = m; }
        else if (sc < s2) { s2 = sc; }
    }
    if (margin) *margin = J > 1 ? (s2 - smin) / fmax(1.0, fabs(smin)) : INFINITY;
    oracle_rigid_move(y, A, qrot + 9 * mmin, dtr + 3 * mmin);
    return mmin;
}

typedef struct {
    /* problem */
    const opocket* pk;
    int P, K, S_w;
    const float *rot, *tr, *cs;
    int n_ref, J;                 /* refinement rounds and moves (Q23); n_ref = 0: none */
    const float *qrot, *dtr;      /* move table: J x 9 rotations, J x 3 translations (Angstrom) */
    uint8_t* refine;              /* [n * n_ref] chosen moves of the best pose */
    uint8_t* pose_refine;         /* [n * P * n_ref] chosen moves of every pose */
    /* library (CSR) */
    const int64_t *atom_off, *frag_off, *move_off;
    const float* xyz;
    const int32_t *frag_axis, *move_atoms;
    const uint8_t* atom_type;   /* [atom_off[n]] (Q24) or NULL */
    /* outputs (any may be NULL except best_score/best_pose) */
    double* best_score;
    int32_t* best_pose;
    uint8_t* angles;        /* [S_w * frag_off[i] ...] angle indices of the best pose */
    double* xyz_out;        /* [3 * atom_off[i] ...] best-pose coordinates, input atom order */
    double* pose_score;     /* [n * P] */
    uint8_t* pose_angles;   /* [P * S_w * frag_off[i] ...] */
    double* step_margin;    /* [n * P] min over steps of (2nd best - best)/max(1,|best|) */
    double* pose_margin;    /* [n] (2nd best S_p - best)/max(1,|best|) */
    int64_t lo, hi;
} batch_t;

/*
 * One ligand, all poses (a6 -> a7 -> a9).  For each pose: place; for each
 * sweep and each fragment in input order (Q4, Q13): score every angle step k
 * (full sum), keep the smallest k attaining the minimum (Q11), apply it.  The
 * pose score is S(final y).  Best pose p* = smallest p attaining min S_p (Q11).
 */
static void dock_one(const batch_t* B, int64_t li, double* y, double* ytmp, double* ybest, uint8_t* kseq, uint8_t* kbest,
                     uint8_t* mseq, uint8_t* mbest) {
    const opocket* pk = B->pk;
    int A = (int)(B->atom_off[li + 1] - B->atom_off[li]);
    int R = (int)(B->frag_off[li + 1] - B->frag_off[li]);
    const float* x = B->xyz + 3 * B->atom_off[li];
    const uint8_t* ty = B->atom_type ? B->atom_type + B->atom_off[li] : NULL;
    const int64_t f0 = B->frag_off[li];
    double best = INFINITY, second = INFINITY;
    int bestp = -1;
    for (int p = 0; p < B->P; ++p) {
        oracle_place_pose(pk, x, A, B->rot + 9 * p, B->tr + 3 * p, y);
        double margin = INFINITY;
        for (int sw = 0; sw < B->S_w; ++sw) {
            for (int r = 0; r < R; ++r) {
                double smin = INFINITY, s2 = INFINITY;
                int kmin = 0;
                for (int k = 0; k < B->K; ++k) {
                    memcpy(ytmp, y, sizeof(double) * 3 * (size_t)A);
                    rotate_frag_csr(ytmp, B->frag_axis, B->move_off, B->move_atoms, f0 + r, (double)B->cs[2 * k],
                                    (double)B->cs[2 * k + 1]);
                    double s = score(pk, ytmp, A, ty);
                    if (s < smin) { s2 = smin; smin = s; kmin = k; }
                    else if (s < s2) { s2 = s; }
                }
                if (B->K > 1) {
                    double m = (s2 - smin) / fmax(1.0, fabs(smin));
                    if (m < margin) margin = m;
                }
                rotate_frag_csr(y, B->frag_axis, B->move_off, B->move_atoms, f0 + r, (double)B->cs[2 * kmin],
                                (double)B->cs[2 * kmin + 1]);
                kseq[sw * R + r] = (uint8_t)kmin;
            }
        }
        for (int t = 0; t < B->n_ref; ++t) {   /* rigid refinement after the sweeps (Q23) */
            double m;
            mseq[t] = (uint8_t)refine_round(pk, y, ytmp, A, ty, B->J, B->qrot, B->dtr, NULL, &m);
            if (m < margin) margin = m;
        }
        if (B->pose_refine) memcpy(B->pose_refine + ((size_t)li * B->P + p) * B->n_ref, mseq, (size_t)B->n_ref);
        double sp = score(pk, y, A, ty);
        if (B->pose_score) B->pose_score[li * B->P + p] = sp;
        if (B->step_margin) B->step_margin[li * B->P + p] = margin;
        if (B->pose_angles)
            memcpy(B->pose_angles + (size_t)B->P * B->S_w * B->frag_off[li] + (size_t)p * B->S_w * R, kseq, (size_t)B->S_w * R);
        if (sp < best) {
            second = best; best = sp; bestp = p;
            memcpy(ybest, y, sizeof(double) * 3 * (size_t)A);
            memcpy(kbest, kseq, (size_t)B->S_w * R);
            memcpy(mbest, mseq, (size_t)B->n_ref);
        } else if (sp < second) {
            second = sp;
        }
    }
    B->best_score[li] = best;
    B->best_pose[li] = bestp;
    if (B->pose_margin) B->pose_margin[li] = (second - best) / fmax(1.0, fabs(best));
    if (B->angles) memcpy(B->angles + (size_t)B->S_w * B->frag_off[li], kbest, (size_t)B->S_w * R);
    if (B->refine) memcpy(B->refine + (size_t)li * B->n_ref, mbest, (size_t)B->n_ref);
    if (B->xyz_out) memcpy(B->xyz_out + 3 * B->atom_off[li], ybest, sizeof(double) * 3 * (size_t)A);
}

static void* batch_worker(void* arg) {
    batch_t* B = (batch_t*)arg;
    int maxA = 1, maxR = 1;
    for (int64_t i = B->lo; i < B->hi; ++i) {
        int A = (int)(B->atom_off[i + 1] - B->atom_off[i]);
        int R = (int)(B->frag_off[i + 1] - B->frag_off[i]);
        if (A > maxA) maxA = A;
        if (R > maxR) maxR = R;
    }
    double* y = (double*)malloc(sizeof(double) * 3 * (size_t)maxA);
    double* yt = (double*)malloc(sizeof(double) * 3 * (size_t)maxA);
    double* yb = (double*)malloc(sizeof(double) * 3 * (size_t)maxA);
    uint8_t* ks = (uint8_t*)malloc((size_t)B->S_w * maxR + 1);
    uint8_t* kb = (uint8_t*)malloc((size_t)B->S_w * maxR + 1);
    uint8_t* ms = (uint8_t*)malloc((size_t)B->n_ref + 1);
    uint8_t* mb = (uint8_t*)malloc((size_t)B->n_ref + 1);
    for (int64_t i = B->lo; i < B->hi; ++i) dock_one(B, i, y, yt, yb, ks, kb, ms, mb);
    free(y); free(yt); free(yb); free(ks); free(kb); free(ms); free(mb);
    return NULL;
}

static void make_pocket(opocket* pk, const int32_t* dims, const double* prm, const float* G) {
    for (int a = 0; a < 3; ++a) pk->n[a] = dims[a];
    pk->T = dims[3];
    for (int a = 0; a < 3; ++a) pk->o[a] = prm[a];
    pk->h = prm[3];
    for (int a = 0; a < 3; ++a) pk->c[a] = prm[4 + a];
    pk->kappa = prm[7];
    pk->G = G;
}

/*
 * Dock a batch.  dims = {nx, ny, nz, T}; prm = {ox, oy, oz, h, cx, cy, cz, kappa}; grid =
 * [T][nz][ny][nx]; atom_type[atom_off[n]] (NULL = all 0), every type < T.
 * Returns 0, or -1 on invalid arguments.
 */
int oracle_dock_batch(int64_t n, const int64_t* atom_off, const float* xyz, const uint8_t* atom_type,
                      const int64_t* frag_off, const int32_t* frag_axis, const int64_t* move_off, const int32_t* move_atoms,
                      const int32_t* dims, const double* prm, const float* grid,
                      int P, const float* rot, const float* trans, int K, const float* cs, int S_w,
                      double* best_score, int32_t* best_pose, uint8_t* angles, double* xyz_out,
                      double* pose_score, uint8_t* pose_angles, double* step_margin, double* pose_margin,
                      int n_ref, int J, const float* qrot, const float* dtr, uint8_t* refine, uint8_t* pose_refine,
                      int nthreads) {
    if (n < 0 || P < 1 || K < 1 || S_w < 0 || n_ref < 0 || (n_ref > 0 && (J < 1 || !qrot || !dtr))) return -1;
    if (dims[0] < 2 || dims[1] < 2 || dims[2] < 2 || dims[3] < 1 || !(prm[3] > 0.0)) return -1;
    if (atom_type)
        for (int64_t i = 0; i < (n > 0 ? atom_off[n] : 0); ++i)
            if (atom_type[i] >= dims[3]) return -1;
    opocket pk;
    make_pocket(&pk, dims, prm, grid);
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 512) nthreads = 512;
    if (n < nthreads) nthreads = n > 0 ? (int)n : 1;
    pthread_t th[512];
    batch_t jobs[512];
    for (int t = 0; t < nthreads; ++t) {
        batch_t* B = &jobs[t];
        memset(B, 0, sizeof *B);
        B->pk = &pk; B->P = P; B->K = K; B->S_w = S_w; B->rot = rot; B->tr = trans; B->cs = cs;
        B->atom_off = atom_off; B->frag_off = frag_off; B->xyz = xyz; B->atom_type = atom_type;
        B->frag_axis = frag_axis; B->move_off = move_off; B->move_atoms = move_atoms;
        B->best_score = best_score; B->best_pose = best_pose; B->angles = angles; B->xyz_out = xyz_out;
        B->pose_score = pose_score; B->pose_angles = pose_angles; B->step_margin = step_margin; B->pose_margin = pose_margin;
        B->n_ref = n_ref; B->J = J; B->qrot = qrot; B->dtr = dtr; B->refine = refine; B->pose_refine = pose_refine;
        B->lo = n * t / nthreads; B->hi = n * (t + 1) / nthreads;
    }
    for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, batch_worker, &jobs[t]);
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    return 0;
}

/*
 * Replay checker primitive: place ligand (xyz,
 * fragments frag_axis[2R] / move_off[R+1] / move_atoms) in pose p and apply the GIVEN angle sequence kseq[S_w*R] (e.g. the
 * one the GPU chose).  For every step it records the full-sum score of every
 * candidate k into step_scores[(sw*R + r)*K + k] before applying kseq's
 * choice, so a checker can verify each choice is within the near-tie band of
 * the fp64 minimum.  Final coordinates -> y_out[3A], final score returned.
 */
double oracle_replay_pose(const int32_t* dims, const double* prm, const float* grid,
                          int A, const float* xyz, const uint8_t* ty, int R, const int32_t* frag_axis, const int64_t* move_off,
                          const int32_t* move_atoms,
                          const float* rot9, const float* tr3, int K, const float* cs, int S_w,
                          const uint8_t* kseq, double* step_scores, double* y_out,
                          int n_ref, int J, const float* qrot, const float* dtr, const uint8_t* mseq,
                          double* ref_scores) {
    opocket pk;
    make_pocket(&pk, dims, prm, grid);
    double* yt = (double*)malloc(sizeof(double) * 3 * (size_t)(A > 0 ? A : 1));
    oracle_place_pose(&pk, xyz, A, rot9, tr3, y_out);
    for (int sw = 0; sw < S_w; ++sw) {
        for (int r = 0; r < R; ++r) {
            if (step_scores) {
                for (int k = 0; k < K; ++k) {
                    memcpy(yt, y_out, sizeof(double) * 3 * (size_t)A);
                    rotate_frag_csr(yt, frag_axis, move_off, move_atoms, r, (double)cs[2 * k], (double)cs[2 * k + 1]);
                    step_scores[(sw * R + r) * K + k] = score(&pk, yt, A, ty);
                }
            }
            int k = kseq[sw * R + r];
            rotate_frag_csr(y_out, frag_axis, move_off, move_atoms, r, (double)cs[2 * k], (double)cs[2 * k + 1]);
        }
    }
    for (int t = 0; t < n_ref; ++t) {   /* the GIVEN refinement moves (Q23), every move scored first */
        if (ref_scores)
            for (int m = 0; m < J; ++m) {
                memcpy(yt, y_out, sizeof(double) * 3 * (size_t)A);
                oracle_rigid_move(yt, A, qrot + 9 * m, dtr + 3 * m);
                ref_scores[t * J + m] = score(&pk, yt, A, ty);
            }
        oracle_rigid_move(y_out, A, qrot + 9 * mseq[t], dtr + 3 * mseq[t]);
    }
    double s = score(&pk, y_out, A, ty);
    free(yt);
    return s;
}

/* Test hooks: g at arbitrary points (channel types[i], NULL = 0), and a pose placement. */
int oracle_grid_score_points(const int32_t* dims, const double* prm, const float* grid, int64_t n, const double* pts,
                             const uint8_t* types, double* out) {
    opocket pk;
    make_pocket(&pk, dims, prm, grid);
    for (int64_t i = 0; i < n; ++i) out[i] = oracle_grid_score(&pk, types ? types[i] : 0, pts + 3 * i);
    return 0;
}

int oracle_place(const int32_t* dims, const double* prm, int A, const float* xyz, const float* rot9, const float* tr3, double* y) {
    opocket pk;
    make_pocket(&pk, dims, prm, NULL);
    oracle_place_pose(&pk, xyz, A, rot9, tr3, y);
    return 0;
}

int oracle_rotate(int A, double* y, int a, int b, const int32_t* mv, int nm, double ck, double sk) {
    (void)A;
    oracle_rotate_fragment(y, a, b, mv, nm, ck, sk);
    return 0;
}
