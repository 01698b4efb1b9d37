/*
 * vsgen/gen.c -- seeded synthetic ligand-library generator.
 *
 * INPUT GENERATOR ONLY.  This module is shared by the oracle side (oracle/,
 * tests/) and the product side (bench.py, the CUDA path) and therefore holds
 * none of the method's arithmetic: no pose placement, no fragment rotation,
 * no grid scoring, no bucketing.  It only draws random molecules.
 *
 * What it draws (SURVEY.md 8(d) "Generators"):
 *   - heavy-atom count A ~ U[alo, ahi] and a target rotatable-bond count
 *     R* ~ U[rlo, rhi], drawn independently ("weak
 *     relationship"; SPEC.md l.36-44 uniform independent sampling);
 *   - a random heavy-atom tree (every atom degree <= 4), re-rooted at its
 *     centroid and renumbered in DFS preorder, so that the atoms on the far
 *     side of any bond (a -> b) form the contiguous range [b+1, b+size(b));
 *   - R = min(R*, #eligible bonds) rotatable bonds chosen at random among the
 *     bonds whose moving side has >= 2 atoms and fixed side has >= 2 atoms,
 *     emitted inner-first (BFS depth of b, ties by b) (reading Q4);
 *     each fragment is {a, b, lo, hi}: axis a->b, moving set M_r = [lo, hi)
 *     (axis atoms excluded, "subset of the molecule atoms
 *     that can rotate");
 *   - a 3D embedding: 1.5 A bonds, 109.47 deg bond angles, random torsions,
 *     non-bonded distances >= 2.0 A when achievable in 12 tries (else the
 *     best of the 12), then a
 *     random rigid offset in [-10, 10]^3 A.
 *
 * Ligand i depends only on (seed, i): the stream is prefix-stable and any
 * shard [first, first+n) can be generated independently.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define VSGEN_MAXA 256
#define VSGEN_MAXR 32

typedef struct { uint64_t s; } rng_t;

static inline uint64_t rng_u64(rng_t* r) {
    uint64_t z = (r->s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static inline double rng_unit(rng_t* r) { return (double)(rng_u64(r) >> 11) * (1.0 / 9007199254740992.0); }
static inline int rng_int(rng_t* r, int lo, int hi) { /* inclusive */
    return lo + (int)(rng_u64(r) % (uint64_t)(hi - lo + 1));
}
static rng_t rng_for(uint64_t seed, int64_t i) {
    rng_t r;
    r.s = seed * 0xD1B54A32D192ED03ULL ^ ((uint64_t)i + 1ULL) * 0x9E3779B97F4A7C15ULL;
    (void)rng_u64(&r);
    return r;
}

typedef struct {
    int A, R, M;                 /* atoms, fragments, sum of |M_r| */
    int pn[VSGEN_MAXA];          /* parent in preorder numbering (-1 for root) */
    int size[VSGEN_MAXA];
    int frag[VSGEN_MAXR][4];
    double pos[VSGEN_MAXA][3];
} lig_t;

/* Build one ligand.  Returns 0 on success. */
static int gen_one(uint64_t seed, int64_t idx, int alo, int ahi, int rlo, int rhi, int geometry, lig_t* L) {
    rng_t rg = rng_for(seed, idx);
    int A = rng_int(&rg, alo, ahi);
    int Rt = rng_int(&rg, rlo, rhi);
    L->A = A;
    /* --- random tree on original labels (degree <= 4) --- */
    int adj[VSGEN_MAXA][4], deg[VSGEN_MAXA];
    memset(deg, 0, sizeof(int) * (size_t)A);
    int par0[VSGEN_MAXA];
    par0[0] = -1;
    for (int v = 1; v < A; ++v) {
        int p;
        do { p = rng_int(&rg, 0, v - 1); } while (deg[p] >= 4);
        par0[v] = p;
        adj[p][deg[p]++] = v;
        adj[v][deg[v]++] = p;
    }
    /* --- centroid (min over v of the largest component after removing v) --- */
    int sz0[VSGEN_MAXA];
    for (int v = 0; v < A; ++v) sz0[v] = 1;
    for (int v = A - 1; v >= 1; --v) sz0[par0[v]] += sz0[v];
    int cen = 0, best = A + 1;
    for (int v = 0; v < A; ++v) {
        int mx = A - sz0[v];
        for (int e = 0; e < deg[v]; ++e) {
            int w = adj[v][e];
            if (w != par0[v] && sz0[w] > mx) mx = sz0[w];
        }
        if (mx < best) { best = mx; cen = v; }
    }
    /* --- DFS preorder from the centroid, neighbours in increasing label order --- */
    for (int v = 0; v < A; ++v) { /* sort each adjacency list (<= 4 entries) */
        for (int x = 1; x < deg[v]; ++x) {
            int t = adj[v][x], y = x - 1;
            while (y >= 0 && adj[v][y] > t) { adj[v][y + 1] = adj[v][y]; --y; }
            adj[v][y + 1] = t;
        }
    }
    int newid[VSGEN_MAXA], oldpar[VSGEN_MAXA];
    for (int v = 0; v < A; ++v) newid[v] = -1;
    int stack[VSGEN_MAXA], sp = 0, next = 0;
    stack[sp++] = cen;
    oldpar[cen] = -1;
    while (sp > 0) {
        int v = stack[--sp];
        newid[v] = next++;
        for (int e = deg[v] - 1; e >= 0; --e) { /* push reversed so smallest label pops first */
            int w = adj[v][e];
            if (w == oldpar[v]) continue;
            oldpar[w] = v;
            stack[sp++] = w;
        }
    }
    for (int v = 0; v < A; ++v) L->pn[newid[v]] = (oldpar[v] < 0) ? -1 : newid[oldpar[v]];
    for (int v = 0; v < A; ++v) L->size[v] = 1;
    for (int v = A - 1; v >= 1; --v) L->size[L->pn[v]] += L->size[v];
    int depth[VSGEN_MAXA];
    depth[0] = 0;
    for (int v = 1; v < A; ++v) depth[v] = depth[L->pn[v]] + 1;
    /* --- rotatable bonds --- */
    int elig[VSGEN_MAXA], ne = 0;
    for (int v = 1; v < A; ++v)
        if (L->size[v] >= 2 && A - L->size[v] >= 2) elig[ne++] = v;
    int R = Rt < ne ? Rt : ne;
    if (R > VSGEN_MAXR) R = VSGEN_MAXR;
    for (int x = 0; x < R; ++x) { /* partial Fisher-Yates */
        int y = rng_int(&rg, x, ne - 1);
        int t = elig[x]; elig[x] = elig[y]; elig[y] = t;
    }
    for (int x = 1; x < R; ++x) { /* order by (depth, index) */
        int t = elig[x], y = x - 1;
        while (y >= 0 && (depth[elig[y]] > depth[t] || (depth[elig[y]] == depth[t] && elig[y] > t))) {
            elig[y + 1] = elig[y]; --y;
        }
        elig[y + 1] = t;
    }
    L->R = R;
    L->M = 0;
    for (int x = 0; x < R; ++x) {
        int b = elig[x];
        L->frag[x][0] = L->pn[b];
        L->frag[x][1] = b;
        L->frag[x][2] = b + 1;
        L->frag[x][3] = b + L->size[b];
        L->M += L->size[b] - 1;
    }
    if (!geometry) return 0;
    /* --- 3D embedding in preorder --- */
    const double bond = 1.5, cth = cos(109.47 * M_PI / 180.0), sth = sin(109.47 * M_PI / 180.0);
    int first_child0 = -1;
    L->pos[0][0] = L->pos[0][1] = L->pos[0][2] = 0.0;
    for (int v = 1; v < A; ++v) {
        int p = L->pn[v];
        double ref[3] = {0, 0, 0};
        int have_ref = 0;
        if (p != 0) {
            int pp = L->pn[p];
            for (int c = 0; c < 3; ++c) ref[c] = L->pos[pp][c] - L->pos[p][c];
            have_ref = 1;
        } else if (first_child0 >= 0) {
            for (int c = 0; c < 3; ++c) ref[c] = L->pos[first_child0][c] - L->pos[0][c];
            have_ref = 1;
        }
        double e0[3], e1[3], e2[3];
        if (have_ref) {
            double n = sqrt(ref[0] * ref[0] + ref[1] * ref[1] + ref[2] * ref[2]);
            for (int c = 0; c < 3; ++c) e0[c] = ref[c] / n;
            double t[3] = {1, 0, 0};
            if (fabs(e0[0]) > 0.8) { t[0] = 0; t[1] = 1; }
            e1[0] = e0[1] * t[2] - e0[2] * t[1];
            e1[1] = e0[2] * t[0] - e0[0] * t[2];
            e1[2] = e0[0] * t[1] - e0[1] * t[0];
            n = sqrt(e1[0] * e1[0] + e1[1] * e1[1] + e1[2] * e1[2]);
            for (int c = 0; c < 3; ++c) e1[c] /= n;
            e2[0] = e0[1] * e1[2] - e0[2] * e1[1];
            e2[1] = e0[2] * e1[0] - e0[0] * e1[2];
            e2[2] = e0[0] * e1[1] - e0[1] * e1[0];
        }
        double bestc[3] = {0, 0, 0}, bestd = -1.0;
        for (int attempt = 0; attempt < 12; ++attempt) {
            double d[3];
            if (have_ref) {
                double phi = 2.0 * M_PI * rng_unit(&rg);
                for (int c = 0; c < 3; ++c) d[c] = cth * e0[c] + sth * (cos(phi) * e1[c] + sin(phi) * e2[c]);
            } else {
                double z = 2.0 * rng_unit(&rg) - 1.0, phi = 2.0 * M_PI * rng_unit(&rg), s = sqrt(1.0 - z * z);
                d[0] = s * cos(phi); d[1] = s * sin(phi); d[2] = z;
            }
            double cand[3];
            for (int c = 0; c < 3; ++c) cand[c] = L->pos[p][c] + bond * d[c];
            double mind = 1e30;
            for (int w = 0; w < v; ++w) {
                if (w == p) continue;
                double dx = cand[0] - L->pos[w][0], dy = cand[1] - L->pos[w][1], dz = cand[2] - L->pos[w][2];
                double dd = dx * dx + dy * dy + dz * dz;
                if (dd < mind) mind = dd;
            }
            if (mind > bestd) { bestd = mind; memcpy(bestc, cand, sizeof bestc); }
            if (mind >= 4.0) break; /* squared: 2.0 A */
        }
        memcpy(L->pos[v], bestc, sizeof bestc);
        if (p == 0 && first_child0 < 0) first_child0 = v;
    }
    double off[3];
    for (int c = 0; c < 3; ++c) off[c] = 20.0 * rng_unit(&rg) - 10.0;
    for (int v = 0; v < A; ++v)
        for (int c = 0; c < 3; ++c) L->pos[v][c] += off[c];
    return 0;
}

/* ------------------------------------------------------------------------- */
typedef struct {
    int64_t lo, hi, first;
    uint64_t seed;
    int alo, ahi, rlo, rhi;
    int32_t *A, *R, *M;                    /* shapes pass */
    const int64_t *atom_off, *frag_off;    /* fill pass */
    float* xyz;
    int32_t* frags;
    int fill;
} job_t;

static void* worker(void* arg) {
    job_t* j = (job_t*)arg;
    lig_t* L = (lig_t*)malloc(sizeof(lig_t));
    for (int64_t i = j->lo; i < j->hi; ++i) {
        gen_one(j->seed, j->first + i, j->alo, j->ahi, j->rlo, j->rhi, j->fill, L);
        if (!j->fill) {
            j->A[i] = L->A; j->R[i] = L->R; j->M[i] = L->M;
        } else {
            float* x = j->xyz + 3 * j->atom_off[i];
            for (int v = 0; v < L->A; ++v)
                for (int c = 0; c < 3; ++c) x[3 * v + c] = (float)L->pos[v][c];
            int32_t* f = j->frags + 4 * j->frag_off[i];
            for (int r = 0; r < L->R; ++r)
                for (int c = 0; c < 4; ++c) f[4 * r + c] = L->frag[r][c];
        }
    }
    free(L);
    return NULL;
}

static int run(job_t proto, int64_t n, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    if (n < 64 * nthreads) nthreads = (int)((n + 63) / 64) > 0 ? (int)((n + 63) / 64) : 1;
    pthread_t th[256];
    job_t jobs[256];
    for (int t = 0; t < nthreads; ++t) {
        jobs[t] = proto;
        jobs[t].lo = n * t / nthreads;
        jobs[t].hi = n * (t + 1) / nthreads;
        pthread_create(&th[t], NULL, worker, &jobs[t]);
    }
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    return 0;
}

static int check_args(int alo, int ahi, int rlo, int rhi) {
    if (alo < 1 || ahi < alo || ahi > VSGEN_MAXA) return -1;
    if (rlo < 0 || rhi < rlo || rhi > VSGEN_MAXR) return -1;
    return 0;
}

/* Per-ligand shapes: atoms A[i], fragments R[i], sum of moving-set sizes M[i]. */
int vsgen_ligand_shapes(int64_t n, uint64_t seed, int64_t first, int alo, int ahi, int rlo, int rhi,
                        int32_t* A, int32_t* R, int32_t* M, int nthreads) {
    if (n < 0 || check_args(alo, ahi, rlo, rhi)) return -1;
    job_t j;
    memset(&j, 0, sizeof j);
    j.first = first; j.seed = seed; j.alo = alo; j.ahi = ahi; j.rlo = rlo; j.rhi = rhi;
    j.A = A; j.R = R; j.M = M; j.fill = 0;
    return run(j, n, nthreads);
}

/* Geometry + fragments into caller CSR buffers sized from the shapes pass. */
int vsgen_ligand_fill(int64_t n, uint64_t seed, int64_t first, int alo, int ahi, int rlo, int rhi,
                      const int64_t* atom_off, const int64_t* frag_off, float* xyz, int32_t* frags, int nthreads) {
    if (n < 0 || check_args(alo, ahi, rlo, rhi)) return -1;
    job_t j;
    memset(&j, 0, sizeof j);
    j.first = first; j.seed = seed; j.alo = alo; j.ahi = ahi; j.rlo = rlo; j.rhi = rhi;
    j.atom_off = atom_off; j.frag_off = frag_off; j.xyz = xyz; j.frags = frags; j.fill = 1;
    return run(j, n, nthreads);
}
