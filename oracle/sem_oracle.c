/*
 * sem_oracle.c -- plain, slow, obviously-correct fp64 CPU ORACLE for the
 * Hilbert-reordered SEM leapfrog step of arxiv 2104.08416.
 *
 * TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant with the CUDA product path.
 *
 * Build: gcc -O2 -fopenmp -ffp-contract=off -fPIC -shared (no -ffast-math;
 * denormals kept).
 *
 * Every function cites the passage it follows (PAPER.md line numbers, "P:n")
 * or the DESIGN.md reading (R*) where the paper is silent.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_E_ARG (-1)
#define ORC_E_MESH (-2)
#define ORC_E_OOM (-3)

/* ------------------------------------------------------------------------ */
/* Generalized Hilbert curve, materialised (docs/hilbert.md).  */
/* ------------------------------------------------------------------------ */

typedef struct {
    int32_t *px, *py;
    int64_t n;
} orc_path;

static int isgn(int v) { return (v > 0) - (v < 0); }
static int iabs_(int v) { return v < 0 ? -v : v; }
/* floor(v / 2), rounding toward minus infinity (docs/hilbert.md "half"). */
static int half_floor(int v) { return (v >= 0) ? v / 2 : -((-v + 1) / 2); }

static void emit(orc_path *P, int x, int y) {
    P->px[P->n] = x;
    P->py[P->n] = y;
    P->n++;
}

/* R(o, a, b) of docs/hilbert.md, rules 1-3 in order. */
static void gen_rect(orc_path *P, int ox, int oy, int ax, int ay, int bx, int by) {
    int w = iabs_(ax + ay), h = iabs_(bx + by);
    int dax = isgn(ax), day = isgn(ay), dbx = isgn(bx), dby = isgn(by);
    if (h == 1) { /* rule 1 */
        for (int i = 0; i < w; i++) { emit(P, ox, oy); ox += dax; oy += day; }
        return;
    }
    if (w == 1) { /* rule 2 */
        for (int i = 0; i < h; i++) { emit(P, ox, oy); ox += dbx; oy += dby; }
        return;
    }
    int ax2 = half_floor(ax), ay2 = half_floor(ay);
    int bx2 = half_floor(bx), by2 = half_floor(by);
    int w2 = iabs_(ax2 + ay2), h2 = iabs_(bx2 + by2);
    if (2 * w > 3 * h) { /* rule 3a: elongated, split along the major axis */
        if ((w2 % 2) == 1 && w > 2) { ax2 += dax; ay2 += day; }
        gen_rect(P, ox, oy, ax2, ay2, bx, by);
        gen_rect(P, ox + ax2, oy + ay2, ax - ax2, ay - ay2, bx, by);
    } else { /* rule 3b: standard three-way split */
        if ((h2 % 2) == 1 && h > 2) { bx2 += dbx; by2 += dby; }
        gen_rect(P, ox, oy, bx2, by2, ax2, ay2);
        gen_rect(P, ox + bx2, oy + by2, ax, ay, bx - bx2, by - by2);
        gen_rect(P, ox + (ax - dax) + (bx2 - dbx), oy + (ay - day) + (by2 - dby),
                 -bx2, -by2, -(ax - ax2), -(ay - ay2));
    }
}

/* Materialise the W x H path. px/py must hold W*H entries. Returns count. */
int64_t orc_gilbert_path(int32_t W, int32_t H, int32_t *px, int32_t *py) {
    if (W < 1 || H < 1) return ORC_E_ARG;
    orc_path P = {px, py, 0};
    if (W >= H) gen_rect(&P, 0, 0, W, 0, 0, H);
    else gen_rect(&P, 0, 0, 0, H, W, 0);
    return P.n;
}

/* ------------------------------------------------------------------------ */
/* Element orientation (S:129 reading: clockwise -> swap v1, v2).           */
/* ------------------------------------------------------------------------ */

/* tri_out may alias tri. Returns ORC_OK or -(10 + e) style error via *bad. */
int orc_orient(const double *vxy, const int32_t *tri, int64_t ne, int32_t *tri_out, int64_t *bad) {
    *bad = -1;
    for (int64_t e = 0; e < ne; e++) {
        int32_t v0 = tri[3 * e], v1 = tri[3 * e + 1], v2 = tri[3 * e + 2];
        double x0 = vxy[2 * v0], y0 = vxy[2 * v0 + 1];
        double x1 = vxy[2 * v1], y1 = vxy[2 * v1 + 1];
        double x2 = vxy[2 * v2], y2 = vxy[2 * v2 + 1];
        /* det J with J = [v1-v0, v2-v0] as columns */
        double det = (x1 - x0) * (y2 - y0) - (x2 - x0) * (y1 - y0);
        if (det == 0.0) { *bad = e; return ORC_E_MESH; }
        tri_out[3 * e] = v0;
        if (det < 0.0) { tri_out[3 * e + 1] = v2; tri_out[3 * e + 2] = v1; }
        else { tri_out[3 * e + 1] = v1; tri_out[3 * e + 2] = v2; }
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* SFC element ordering, literally PAPER.md:296-305 (§4.3 steps 1-4).       */
/* ------------------------------------------------------------------------ */

/*
 * key_out[e]  = position on the curve of the sub-rectangle holding element e
 *               (input numbering);
 * perm_out[k] = input id of the element placed at new position k (list L);
 * grid_out    = (w_b, h_b).
 * Reading R9 (grid arithmetic, fp64, this exact operation order) and R11
 * (elements of one cell keep input order).
 */
int orc_hilbert_order(const double *vxy, int64_t nv, const int32_t *tri, int64_t ne,
                      uint32_t *key_out, int32_t *perm_out, int32_t *grid_out) {
    if (ne < 1 || nv < 3) return ORC_E_ARG;
    /* Step 2: mesh width/height/min from the vertices. */
    double xm0 = vxy[0], xm1 = vxy[1], xM0 = vxy[0], xM1 = vxy[1];
    for (int64_t v = 1; v < nv; v++) {
        double x = vxy[2 * v], y = vxy[2 * v + 1];
        if (x < xm0) xm0 = x;
        if (x > xM0) xM0 = x;
        if (y < xm1) xm1 = y;
        if (y > xM1) xM1 = y;
    }
    double wm = xM0 - xm0, hm = xM1 - xm1;
    if (!(wm > 0.0) || !(hm > 0.0)) return ORC_E_MESH;
    double r = wm / hm;
    double sq = sqrt((double)ne);
    double wbd = ceil(sq), hbd = ceil(sq / r);
    int64_t wb = wbd < 1.0 ? 1 : (int64_t)wbd;
    int64_t hb = hbd < 1.0 ? 1 : (int64_t)hbd;
    if (wb * hb > (int64_t)0xFFFFFFFFLL) return ORC_E_ARG;
    double ws = (double)wb / wm, hs = (double)hb / hm;
    grid_out[0] = (int32_t)wb;
    grid_out[1] = (int32_t)hb;

    int64_t ncell = wb * hb;
    int32_t *px = (int32_t *)malloc(sizeof(int32_t) * ncell);
    int32_t *py = (int32_t *)malloc(sizeof(int32_t) * ncell);
    int64_t *cell_of = (int64_t *)malloc(sizeof(int64_t) * ne);
    int64_t *start = (int64_t *)calloc(ncell + 1, sizeof(int64_t));
    int32_t *bucket = (int32_t *)malloc(sizeof(int32_t) * ne);
    if (!px || !py || !cell_of || !start || !bucket) {
        free(px); free(py); free(cell_of); free(start); free(bucket);
        return ORC_E_OOM;
    }
    orc_gilbert_path((int32_t)wb, (int32_t)hb, px, py);

    /* Steps 1 and 3: centroid of each element, the sub-rectangle it maps to. */
    for (int64_t e = 0; e < ne; e++) {
        int32_t v0 = tri[3 * e], v1 = tri[3 * e + 1], v2 = tri[3 * e + 2];
        double xc0 = ((vxy[2 * v0] + vxy[2 * v1]) + vxy[2 * v2]) / 3.0;
        double xc1 = ((vxy[2 * v0 + 1] + vxy[2 * v1 + 1]) + vxy[2 * v2 + 1]) / 3.0;
        double fi = floor((xc0 - xm0) * ws), fj = floor((xc1 - xm1) * hs);
        int64_t i = (int64_t)fi, j = (int64_t)fj;
        if (i > wb - 1) i = wb - 1;
        if (j > hb - 1) j = hb - 1;
        if (i < 0) i = 0;
        if (j < 0) j = 0;
        cell_of[e] = j * wb + i;
    }
    /* Elements per sub-rectangle, kept in input order (stable buckets). */
    for (int64_t e = 0; e < ne; e++) start[cell_of[e] + 1]++;
    for (int64_t c = 0; c < ncell; c++) start[c + 1] += start[c];
    {
        int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * ncell);
        memcpy(fill, start, sizeof(int64_t) * ncell);
        for (int64_t e = 0; e < ne; e++) bucket[fill[cell_of[e]]++] = (int32_t)e;
        free(fill);
    }
    /* Traverse the stored intermediate steps of the curve and accumulate the
     * elements of each visited sub-rectangle in list L (step 3); L is the new
     * order (step 4). */
    int64_t k = 0;
    for (int64_t s = 0; s < ncell; s++) {
        int64_t c = (int64_t)py[s] * wb + px[s];
        for (int64_t t = start[c]; t < start[c + 1]; t++) {
            int32_t e = bucket[t];
            perm_out[k++] = e;
            key_out[e] = (uint32_t)s;
        }
    }
    free(px); free(py); free(cell_of); free(start); free(bucket);
    return (k == ne) ? ORC_OK : ORC_E_MESH;
}

/* Reading R16: library-side random order = stable sort of ids by
 * splitmix64(seed ^ id). */
static uint64_t orc_splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
/* the mixer alone, for its pin against the published SplitMix64 sequence (tests) */
uint64_t orc_splitmix64_value(uint64_t x) { return orc_splitmix64(x); }
typedef struct { uint64_t k; int32_t id; } orc_kv;
static int cmp_kv(const void *a, const void *b) {
    const orc_kv *x = (const orc_kv *)a, *y = (const orc_kv *)b;
    if (x->k != y->k) return x->k < y->k ? -1 : 1;
    return (x->id > y->id) - (x->id < y->id);
}
int orc_random_order(int64_t ne, uint64_t seed, int32_t *perm_out) {
    orc_kv *kv = (orc_kv *)malloc(sizeof(orc_kv) * ne);
    if (!kv) return ORC_E_OOM;
    for (int64_t e = 0; e < ne; e++) { kv[e].k = orc_splitmix64(seed ^ (uint64_t)e); kv[e].id = (int32_t)e; }
    qsort(kv, ne, sizeof(orc_kv), cmp_kv);
    for (int64_t e = 0; e < ne; e++) perm_out[e] = kv[e].id;
    free(kv);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Canonical SEM nodes ("added SEM nodes"; P:189-193 mu(p,e);         */
/* readings R3 local order and R13 canonical numbering).                    */
/* ------------------------------------------------------------------------ */

/* Local node kinds of the lattice order (R3). kind: 0 vertex, 1 edge, 2 interior.
 * For vertices `which` = local vertex; for edges `which` = local edge
 * (0: v0-v1, 1: v0-v2, 2: v1-v2) and `m` = position counted from the edge's
 * first listed vertex. */
typedef struct { int kind, which, m; } orc_lnode;
static const orc_lnode LN_P1[3] = {{0, 0, 0}, {0, 1, 0}, {0, 2, 0}};
static const orc_lnode LN_P2[6] = {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {1, 1, 0}, {1, 2, 0}, {0, 2, 0}};
static const orc_lnode LN_P3[10] = {{0, 0, 0}, {1, 0, 0}, {1, 0, 1}, {0, 1, 0}, {1, 1, 0},
                                    {2, 0, 0}, {1, 2, 0}, {1, 1, 1}, {1, 2, 1}, {0, 2, 0}};
static const int EDGE_V[3][2] = {{0, 1}, {0, 2}, {1, 2}};

static int cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

/* mu_out[e*Np + p] = canonical global node of local node p of element e.
 * tri must already be oriented. Returns the node count N (>0) or an error. */
/* Lattice-order local node kinds for any P (R3 extended to P >= 4, R21): node
 * (i, j) is a vertex at (0,0), (P,0), (0,P); on edge v0-v1 if j = 0 (position
 * i - 1 from v0), v0-v2 if i = 0 (j - 1 from v0), v1-v2 if i + j = P (j - 1
 * from v1); otherwise interior, numbered in lattice order. */
static orc_lnode LN_GEN[64];
static int lattice_nodes(int P) {
    int p = 0, m = 0;
    for (int j = 0; j <= P; j++)
        for (int i = 0; i <= P - j; i++, p++) {
            orc_lnode n = {2, 0, 0};
            if (i == 0 && j == 0) n = (orc_lnode){0, 0, 0};
            else if (i == P && j == 0) n = (orc_lnode){0, 1, 0};
            else if (i == 0 && j == P) n = (orc_lnode){0, 2, 0};
            else if (j == 0) n = (orc_lnode){1, 0, i - 1};
            else if (i == 0) n = (orc_lnode){1, 1, j - 1};
            else if (i + j == P) n = (orc_lnode){1, 2, j - 1};
            else n = (orc_lnode){2, 0, m++};
            LN_GEN[p] = n;
        }
    return p;
}

int64_t orc_canonical_nodes(const int32_t *tri, int64_t nv, int64_t ne, int P, int32_t *mu_out) {
    const orc_lnode *LN;
    int Np;
    if (P == 1) { LN = LN_P1; Np = 3; }
    else if (P == 2) { LN = LN_P2; Np = 6; }
    else if (P == 3) { LN = LN_P3; Np = 10; }
    else if (P >= 4 && P <= 9) { Np = lattice_nodes(P); LN = LN_GEN; }
    else return ORC_E_ARG;
    int nI = (P - 1) * (P - 2) / 2;
    /* Unique edges sorted by (min, max): bucket by min vertex, sort each bucket. */
    int64_t *start = (int64_t *)calloc(nv + 1, sizeof(int64_t));
    int32_t *hi = (int32_t *)malloc(sizeof(int32_t) * 3 * ne);
    char *used = (char *)calloc(nv, 1);
    if (!start || !hi || !used) { free(start); free(hi); free(used); return ORC_E_OOM; }
    for (int64_t e = 0; e < ne; e++)
        for (int l = 0; l < 3; l++) {
            int32_t a = tri[3 * e + EDGE_V[l][0]], b = tri[3 * e + EDGE_V[l][1]];
            int32_t lo = a < b ? a : b;
            start[lo + 1]++;
        }
    for (int64_t v = 0; v < nv; v++) start[v + 1] += start[v];
    {
        int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (nv + 1));
        memcpy(fill, start, sizeof(int64_t) * (nv + 1));
        for (int64_t e = 0; e < ne; e++)
            for (int l = 0; l < 3; l++) {
                int32_t a = tri[3 * e + EDGE_V[l][0]], b = tri[3 * e + EDGE_V[l][1]];
                int32_t lo = a < b ? a : b, h = a < b ? b : a;
                hi[fill[lo]++] = h;
            }
        free(fill);
    }
    /* sort + unique within each bucket; ucount[v] = unique edges with min v */
    int64_t *ustart = (int64_t *)calloc(nv + 1, sizeof(int64_t));
    int64_t *ulen = (int64_t *)calloc(nv, sizeof(int64_t));
    for (int64_t v = 0; v < nv; v++) {
        int64_t s = start[v], n = start[v + 1] - s;
        qsort(hi + s, n, sizeof(int32_t), cmp_i32);
        int64_t u = 0;
        for (int64_t t = 0; t < n; t++)
            if (u == 0 || hi[s + u - 1] != hi[s + t]) hi[s + u++] = hi[s + t];
        ulen[v] = u;
    }
    for (int64_t v = 0; v < nv; v++) ustart[v + 1] = ustart[v] + ulen[v];
    int64_t nedges = ustart[nv];

    for (int64_t e = 0; e < ne; e++) {
        for (int l = 0; l < 3; l++) used[tri[3 * e + l]] = 1;
        for (int p = 0; p < Np; p++) {
            const orc_lnode *n = &LN[p];
            int64_t g;
            if (n->kind == 0) {
                g = tri[3 * e + n->which];
            } else if (n->kind == 1) {
                int32_t a = tri[3 * e + EDGE_V[n->which][0]], b = tri[3 * e + EDGE_V[n->which][1]];
                int32_t lo = a < b ? a : b, h = a < b ? b : a;
                /* locate h among the unique partners of lo (linear scan: plain) */
                int64_t s = start[lo], k = -1;
                for (int64_t t = 0; t < ulen[lo]; t++)
                    if (hi[s + t] == h) { k = ustart[lo] + t; break; }
                int i = (a < b) ? n->m : (P - 2) - n->m; /* counted from the min-id end */
                g = nv + k * (P - 1) + i;
            } else {
                g = nv + nedges * (P - 1) + e * nI + n->m;
            }
            mu_out[e * Np + p] = (int32_t)g;
        }
    }
    int64_t N = nv + nedges * (P - 1) + ne * nI;
    int64_t unused = 0;
    for (int64_t v = 0; v < nv; v++) unused += !used[v];
    free(start); free(hi); free(used); free(ustart); free(ulen);
    if (unused) return ORC_E_MESH; /* a vertex no element uses would have M-bar = 0 */
    return N;
}

/* ------------------------------------------------------------------------ */
/* Node renumbering, first-touch part of P:312-321 (reading R12).           */
/* ------------------------------------------------------------------------ */

/* Traverse elements in (new) order; each node not seen in a previous element
 * gets the next label. node_perm_out[new] = old; mu_out = relabelled mu. */
int orc_first_touch(const int32_t *mu, int64_t ne, int Np, int64_t nn,
                    int32_t *node_perm_out, int32_t *mu_out) {
    int32_t *newid = (int32_t *)malloc(sizeof(int32_t) * nn);
    if (!newid) return ORC_E_OOM;
    for (int64_t g = 0; g < nn; g++) newid[g] = -1;
    int64_t next = 0;
    for (int64_t e = 0; e < ne; e++)
        for (int p = 0; p < Np; p++) {
            int32_t g = mu[e * Np + p];
            if (newid[g] < 0) { newid[g] = (int32_t)next; node_perm_out[next] = g; next++; }
            mu_out[e * Np + p] = newid[g];
        }
    free(newid);
    return next == nn ? ORC_OK : ORC_E_MESH;
}

/* ------------------------------------------------------------------------ */
/* Geometry (reading R5) and lumped mass.     */
/* ------------------------------------------------------------------------ */

/* J[e] = {J00, J01, J10, J11} with J_{j jh} = d x_j / d xh_jh (columns v1-v0,
 * v2-v0); detJ[e]; Jinv[e] = inverse of J, stored the same way. */
void orc_geometry(const double *vxy, const int32_t *tri, int64_t ne,
                  double *J, double *detJ, double *Jinv) {
    for (int64_t e = 0; e < ne; e++) {
        int32_t v0 = tri[3 * e], v1 = tri[3 * e + 1], v2 = tri[3 * e + 2];
        double j00 = vxy[2 * v1] - vxy[2 * v0], j01 = vxy[2 * v2] - vxy[2 * v0];
        double j10 = vxy[2 * v1 + 1] - vxy[2 * v0 + 1], j11 = vxy[2 * v2 + 1] - vxy[2 * v0 + 1];
        double d = j00 * j11 - j01 * j10;
        J[4 * e] = j00; J[4 * e + 1] = j01; J[4 * e + 2] = j10; J[4 * e + 3] = j11;
        detJ[e] = d;
        Jinv[4 * e] = j11 / d; Jinv[4 * e + 1] = -j01 / d;
        Jinv[4 * e + 2] = -j10 / d; Jinv[4 * e + 3] = j00 / d;
    }
}

/* Mbar_nu = sum_{e,q: nu = mu(q,e)} M^(e) detJ^(e) w_q  with M^(e) = 1 (R2). */
void orc_lumped_mass(const int32_t *mu, int64_t ne, int Np, int64_t nn,
                     const double *detJ, const double *wM, double *Mbar) {
    for (int64_t g = 0; g < nn; g++) Mbar[g] = 0.0;
    for (int64_t e = 0; e < ne; e++)
        for (int q = 0; q < Np; q++) Mbar[mu[e * Np + q]] += 1.0 * detJ[e] * wM[q];
}

/* ------------------------------------------------------------------------ */
/* R_nu = R(Vdot(U)): Algorithm 1 (E = 0) composed with          */
/* Algorithm 2's first term (D = 0).  Acoustic coefficients      */
/* B = -I and F = c_e^2 I (reading R2).  K^(e) = inverse Jacobian,  */
/* indexed so that u_,j = sum_jh (J^-1)_{jh j} dN/dxh_jh (reading R5).      */
/* Output R = -K U  (the stiffness applied to U, sign included).            */
/* Dr[k*Np+p] = dN_p/dxh_0 at node k; Ds likewise for xh_1.                 */
/* ------------------------------------------------------------------------ */
void orc_apply_R(const int32_t *mu, int64_t ne, int Np, int64_t nn,
                 const double *detJ, const double *Jinv, const double *c,
                 const double *Dr, const double *Ds, const double *wK,
                 const double *U, double *R, double *ebuf /* [ne*Np] scratch */) {
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < ne; e++) {
        double U2[64], Vd[2][64];
        const double *Ki = Jinv + 4 * e; /* Ki[2*jh + j] = (J^-1)_{jh j} */
        double c2 = c[e] * c[e];
        /* Algorithm 1: gather U_2[q] = U_mu(q,e) */
        for (int q = 0; q < Np; q++) U2[q] = U[mu[e * Np + q]];
        /* Algorithm 1, second term: Vdot_kp = sum_q,j,jh F_kj K_jjh N_q,jh(x_p) U2[q] */
        for (int k = 0; k < 2; k++)
            for (int p = 0; p < Np; p++) {
                double acc = 0.0;
                for (int q = 0; q < Np; q++) {
                    double FK1 = c2 * Ki[0 * 2 + k]; /* F_kk K_k,1 (jh = 0) */
                    double FK2 = c2 * Ki[1 * 2 + k]; /* F_kk K_k,2 (jh = 1) */
                    acc += FK1 * Dr[p * Np + q] * U2[q] + FK2 * Ds[p * Np + q] * U2[q];
                }
                Vd[k][p] = acc;
            }
        /* Algorithm 2, first term, with V := Vdot:
         * val_p = sum_k sum_q detJ w_q B_kk Vdot_kq sum_jh K_k,jh N_p,jh(x_q) */
        for (int p = 0; p < Np; p++) {
            double val = 0.0;
            for (int k = 0; k < 2; k++) {
                double BK1 = -1.0 * Ki[0 * 2 + k]; /* B_kk K_k,1 */
                double BK2 = -1.0 * Ki[1 * 2 + k]; /* B_kk K_k,2 */
                for (int q = 0; q < Np; q++) {
                    double aux2 = detJ[e] * wK[q] * Vd[k][q];
                    val += BK1 * aux2 * Dr[q * Np + p] + BK2 * aux2 * Ds[q * Np + p];
                }
            }
            ebuf[e * Np + p] = val;
        }
    }
    /* scatter: accumulate element contributions at global nodes (serial, so
     * the summation order is fixed) */
    for (int64_t g = 0; g < nn; g++) R[g] = 0.0;
    for (int64_t e = 0; e < ne; e++)
        for (int p = 0; p < Np; p++) R[mu[e * Np + p]] += ebuf[e * Np + p];
}

/* Reading R21b (P = 4, 6): R = -K U with the consistent element stiffness
 * K^(e)_pq = int_e c_e^2 grad N_p . grad N_q, written out as its definition:
 * with grad = J^-T grad^ (R5) and the reference integrals S_ab of the basis
 * derivatives (oracle/refelem.py, exact), K^(e) = sum_ab G_ab S_ab where
 * G_{jh jh'} = c^2 detJ sum_j K_{jh j} K_{jh' j}, K = J^-1 (Srs holds both
 * mixed terms).  Serial scatter in element order, like orc_apply_R. */
void orc_apply_R_tables(const int32_t *mu, int64_t ne, int Np, int64_t nn,
                        const double *detJ, const double *Jinv, const double *c,
                        const double *Srr, const double *Sss, const double *Srs,
                        const double *U, double *R, double *ebuf) {
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < ne; e++) {
        const double *Ki = Jinv + 4 * e;
        double c2 = c[e] * c[e];
        double grr = c2 * detJ[e] * (Ki[0] * Ki[0] + Ki[1] * Ki[1]);
        double gss = c2 * detJ[e] * (Ki[2] * Ki[2] + Ki[3] * Ki[3]);
        double grs = c2 * detJ[e] * (Ki[0] * Ki[2] + Ki[1] * Ki[3]);
        for (int p = 0; p < Np; p++) {
            double acc = 0.0;
            for (int q = 0; q < Np; q++) {
                double k = grr * Srr[p * Np + q] + gss * Sss[p * Np + q] + grs * Srs[p * Np + q];
                acc += k * U[mu[e * Np + q]];
            }
            ebuf[e * Np + p] = -acc;
        }
    }
    for (int64_t g = 0; g < nn; g++) R[g] = 0.0;
    for (int64_t e = 0; e < ne; e++)
        for (int p = 0; p < Np; p++) R[mu[e * Np + p]] += ebuf[e * Np + p];
}

/* Ricker wavelet (reading R7): r(t) = (1 - 2 pi^2 f0^2 tau^2) exp(-pi^2 f0^2 tau^2). */
double orc_ricker(double t, double f0, double t0) {
    double tau = t - t0;
    double a = M_PI * f0 * tau;
    a = a * a;
    return (1.0 - 2.0 * a) * exp(-a);
}

/*
 * n_steps leapfrog steps of  Mbar U'' = -K U + f  (north_star; reading R1):
 *   U^{n+1} = 2 U^n - U^{n-1} + dt^2 Mbar^-1 (R(U^n) + y(t_n)),
 * with Algorithm 3 adding the point source y = A r(t_n) at node
 * `src` and t_n = n dt (t^(0) = 0).  U (= U^n) and Uprev (= U^{n-1})
 * are updated in place; step0 is the index n of the incoming U.
 */
int orc_leapfrog(const int32_t *mu, int64_t ne, int Np, int64_t nn,
                 const double *detJ, const double *Jinv, const double *c,
                 const double *Dr, const double *Ds, const double *wK, const double *Mbar,
                 const double *Srr, const double *Sss, const double *Srs, /* non-NULL: R21b */
                 int64_t src, double A, double f0, double t0, double dt,
                 int64_t step0, int64_t n_steps, double *U, double *Uprev) {
    double *R = (double *)malloc(sizeof(double) * nn);
    double *ebuf = (double *)malloc(sizeof(double) * ne * Np);
    if (!R || !ebuf) { free(R); free(ebuf); return ORC_E_OOM; }
    for (int64_t s = 0; s < n_steps; s++) {
        int64_t n = step0 + s;
        if (Srr) orc_apply_R_tables(mu, ne, Np, nn, detJ, Jinv, c, Srr, Sss, Srs, U, R, ebuf);
        else orc_apply_R(mu, ne, Np, nn, detJ, Jinv, c, Dr, Ds, wK, U, R, ebuf);
        if (src >= 0) R[src] += A * orc_ricker((double)n * dt, f0, t0); /* Algorithm 3 */
#pragma omp parallel for schedule(static)
        for (int64_t g = 0; g < nn; g++) {
            double Udd = R[g] / Mbar[g];
            double Unew = 2.0 * U[g] - Uprev[g] + dt * dt * Udd;
            Uprev[g] = U[g];
            U[g] = Unew;
        }
    }
    free(R); free(ebuf);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* The paper's own integrator: Heun predictor-corrector on (U, V)           */
/* (§4.2.1) with Algorithms 1-3.       */
/* NEXT-1 of SURVEY §8f.  V[e][p][k] is stored element-major with the two   */
/* components of a local node adjacent (Fig. mem_layout). */
/* ------------------------------------------------------------------------ */

/* Algorithm 1 with E = 0: Vdot_kp = sum_q,j,jh F_kj K_jjh N_q,jh(x_p) U_mu(q,e),
 * F = c^2 I (R2), K_jjh = (J^-1)_{jh j} (R5). */
void orc_vdot(const int32_t *mu, int64_t ne, int Np, const double *Jinv, const double *c,
              const double *Dr, const double *Ds, const double *U, double *Vd) {
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < ne; e++) {
        double U2[64];
        const double *Ki = Jinv + 4 * e;
        const double c2 = c[e] * c[e];
        for (int q = 0; q < Np; q++) U2[q] = U[mu[e * Np + q]];
        for (int k = 0; k < 2; k++)
            for (int p = 0; p < Np; p++) {
                double acc = 0.0;
                for (int q = 0; q < Np; q++) {
                    double FK1 = c2 * Ki[0 * 2 + k];
                    double FK2 = c2 * Ki[1 * 2 + k];
                    acc += FK1 * Dr[p * Np + q] * U2[q] + FK2 * Ds[p * Np + q] * U2[q];
                }
                Vd[(e * Np + p) * 2 + k] = acc;
            }
    }
}

/* Algorithm 2, first term (D = 0, B = -I): R_nu = sum over (e,p) with
 * mu(p,e) = nu of sum_k sum_q detJ w_q B_kk V_kq sum_jh K_k,jh N_p,jh(x_q). */
void orc_rv(const int32_t *mu, int64_t ne, int Np, int64_t nn, const double *detJ, const double *Jinv,
            const double *Dr, const double *Ds, const double *wK, const double *V, double *R, double *ebuf) {
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < ne; e++) {
        const double *Ki = Jinv + 4 * e;
        for (int p = 0; p < Np; p++) {
            double val = 0.0;
            for (int k = 0; k < 2; k++) {
                double BK1 = -1.0 * Ki[0 * 2 + k];
                double BK2 = -1.0 * Ki[1 * 2 + k];
                for (int q = 0; q < Np; q++) {
                    double aux2 = detJ[e] * wK[q] * V[(e * Np + q) * 2 + k];
                    val += BK1 * aux2 * Dr[q * Np + p] + BK2 * aux2 * Ds[q * Np + p];
                }
            }
            ebuf[e * Np + p] = val;
        }
    }
    for (int64_t g = 0; g < nn; g++) R[g] = 0.0;
    for (int64_t e = 0; e < ne; e++)
        for (int p = 0; p < Np; p++) R[mu[e * Np + p]] += ebuf[e * Np + p];
}

/*
 * n_steps Heun steps:
 *   predictor  U~ = U + h Udot(V, t_n),       V~ = V + h Vdot(U)
 *   corrector  U+ = U + h/2 (Udot(V, t_n) + Udot(V~, t_{n+1})),
 *              V+ = V + h/2 (Vdot(U) + Vdot(U~))
 * with Udot(V, t) = Mbar^-1 (R(V) + y(t)) (eq. u_change, Algorithm 3 adds the
 * source) and Vdot = Algorithm 1.  Reading R18: the corrector's rates are
 * evaluated at t_{n+1} = t_n + h.  U [nn] and V [ne*Np*2] are updated in place.
 */
int orc_heun(const int32_t *mu, int64_t ne, int Np, int64_t nn,
             const double *detJ, const double *Jinv, const double *c,
             const double *Dr, const double *Ds, const double *wK, const double *Mbar,
             int64_t src, double A, double f0, double t0, double h,
             int64_t step0, int64_t n_steps, double *U, double *V) {
    const int64_t nv = ne * Np * 2;
    double *R = (double *)malloc(sizeof(double) * nn);
    double *Ud1 = (double *)malloc(sizeof(double) * nn);
    double *Ut = (double *)malloc(sizeof(double) * nn);
    double *Vd1 = (double *)malloc(sizeof(double) * nv);
    double *Vd2 = (double *)malloc(sizeof(double) * nv);
    double *Vt = (double *)malloc(sizeof(double) * nv);
    double *ebuf = (double *)malloc(sizeof(double) * ne * Np);
    if (!R || !Ud1 || !Ut || !Vd1 || !Vd2 || !Vt || !ebuf) {
        free(R); free(Ud1); free(Ut); free(Vd1); free(Vd2); free(Vt); free(ebuf);
        return ORC_E_OOM;
    }
    for (int64_t s = 0; s < n_steps; s++) {
        const int64_t n = step0 + s;
        const double tn = (double)n * h, tn1 = (double)(n + 1) * h;
        /* predictor */
        orc_rv(mu, ne, Np, nn, detJ, Jinv, Dr, Ds, wK, V, R, ebuf);
        if (src >= 0) R[src] += A * orc_ricker(tn, f0, t0);
        for (int64_t g = 0; g < nn; g++) { Ud1[g] = R[g] / Mbar[g]; Ut[g] = U[g] + h * Ud1[g]; }
        orc_vdot(mu, ne, Np, Jinv, c, Dr, Ds, U, Vd1);
        for (int64_t i = 0; i < nv; i++) Vt[i] = V[i] + h * Vd1[i];
        /* corrector */
        orc_rv(mu, ne, Np, nn, detJ, Jinv, Dr, Ds, wK, Vt, R, ebuf);
        if (src >= 0) R[src] += A * orc_ricker(tn1, f0, t0);
        orc_vdot(mu, ne, Np, Jinv, c, Dr, Ds, Ut, Vd2);
        for (int64_t g = 0; g < nn; g++) U[g] = U[g] + h / 2.0 * (Ud1[g] + R[g] / Mbar[g]);
        for (int64_t i = 0; i < nv; i++) V[i] = V[i] + h / 2.0 * (Vd1[i] + Vd2[i]);
    }
    free(R); free(Ud1); free(Ut); free(Vd1); free(Vd2); free(Vt); free(ebuf);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* The paper's other memory-reordering strategies (NEXT-3 of SURVEY §8f).    */
/* ------------------------------------------------------------------------ */

/* Node graph: two SEM nodes are connected iff some element holds both
 * ("the number of connections that the node has to other
 * nodes").  CSR over nodes, each row the ascending list of distinct other
 * nodes.  *ptr_out [nn+1] and *adj_out are malloc'ed here; caller frees. */
static int build_node_graph(const int32_t *mu, int64_t ne, int Np, int64_t nn,
                            int64_t **ptr_out, int32_t **adj_out) {
    int64_t *inc_ptr = (int64_t *)calloc((size_t)nn + 1, sizeof(int64_t));
    if (!inc_ptr) return ORC_E_OOM;
    for (int64_t i = 0; i < ne * Np; i++) inc_ptr[mu[i] + 1]++;
    for (int64_t g = 0; g < nn; g++) inc_ptr[g + 1] += inc_ptr[g];
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * ((size_t)nn + 1));
    int32_t *inc = (int32_t *)malloc(sizeof(int32_t) * ((size_t)(ne * Np) + 1));
    int64_t *ptr = (int64_t *)calloc((size_t)nn + 1, sizeof(int64_t));
    if (!fill || !inc || !ptr) { free(inc_ptr); free(fill); free(inc); free(ptr); return ORC_E_OOM; }
    memcpy(fill, inc_ptr, sizeof(int64_t) * ((size_t)nn + 1));
    for (int64_t e = 0; e < ne; e++)  /* elements touching node g, ascending e */
        for (int p = 0; p < Np; p++) inc[fill[mu[e * Np + p]]++] = (int32_t)e;
    /* pass 1: count distinct neighbours; pass 2: fill */
    int32_t *buf = NULL;
    size_t cap = 0;
    int32_t *adj = NULL;
    for (int pass = 0; pass < 2; pass++) {
        for (int64_t g = 0; g < nn; g++) {
            size_t k = (size_t)(inc_ptr[g + 1] - inc_ptr[g]) * (size_t)Np;
            if (k > cap) {
                free(buf);
                cap = k;
                buf = (int32_t *)malloc(sizeof(int32_t) * cap);
                if (!buf) { free(inc_ptr); free(fill); free(inc); free(ptr); free(adj); return ORC_E_OOM; }
            }
            size_t m = 0;
            for (int64_t j = inc_ptr[g]; j < inc_ptr[g + 1]; j++)
                for (int q = 0; q < Np; q++) {
                    int32_t o = mu[(int64_t)inc[j] * Np + q];
                    if (o != g) buf[m++] = o;
                }
            qsort(buf, m, sizeof(int32_t), cmp_i32);
            size_t u = 0;
            for (size_t i = 0; i < m; i++)
                if (i == 0 || buf[i] != buf[i - 1]) {
                    if (pass == 1) adj[ptr[g] + (int64_t)u] = buf[i];
                    u++;
                }
            if (pass == 0) ptr[g + 1] = (int64_t)u;
        }
        if (pass == 0) {
            for (int64_t g = 0; g < nn; g++) ptr[g + 1] += ptr[g];
            adj = (int32_t *)malloc(sizeof(int32_t) * ((size_t)ptr[nn] + 1));
            if (!adj) { free(inc_ptr); free(fill); free(inc); free(ptr); free(buf); return ORC_E_OOM; }
        }
    }
    free(buf); free(inc_ptr); free(fill); free(inc);
    *ptr_out = ptr;
    *adj_out = adj;
    return ORC_OK;
}

/* deg[g] = number of distinct nodes sharing an element with g. */
int orc_node_degree(const int32_t *mu, int64_t ne, int Np, int64_t nn, int32_t *deg) {
    int64_t *ptr; int32_t *adj;
    int rc = build_node_graph(mu, ne, Np, nn, &ptr, &adj);
    if (rc) return rc;
    for (int64_t g = 0; g < nn; g++) deg[g] = (int32_t)(ptr[g + 1] - ptr[g]);
    free(ptr); free(adj);
    return ORC_OK;
}

/* Node renumbering of PAPER.md:312-321, both steps (reading R12,
 * SEM_NODES_FIRST_TOUCH_DEGREE): traverse the elements in their (new) order;
 * N^(e) = the nodes of e not processed in an earlier element (step 1); sort
 * N^(e) by ascending degree, ties by ascending old id (step 2); label in that
 * order.  node_perm_out[new] = old, mu_out = relabelled mu. */
int orc_first_touch_degree(const int32_t *mu, int64_t ne, int Np, int64_t nn,
                           int32_t *node_perm_out, int32_t *mu_out) {
    int32_t *deg = (int32_t *)malloc(sizeof(int32_t) * ((size_t)nn + 1));
    int32_t *newid = (int32_t *)malloc(sizeof(int32_t) * ((size_t)nn + 1));
    if (!deg || !newid) { free(deg); free(newid); return ORC_E_OOM; }
    int rc = orc_node_degree(mu, ne, Np, nn, deg);
    if (rc) { free(deg); free(newid); return rc; }
    for (int64_t g = 0; g < nn; g++) newid[g] = -1;
    int64_t next = 0;
    for (int64_t e = 0; e < ne; e++) {
        int32_t grp[64];
        int ng = 0;
        for (int p = 0; p < Np; p++) { /* step 1: N^(e), first occurrence only */
            int32_t g = mu[e * Np + p];
            int seen = newid[g] >= 0;
            for (int i = 0; i < ng; i++) seen |= grp[i] == g;
            if (!seen) grp[ng++] = g;
        }
        for (int i = 1; i < ng; i++) { /* step 2: insertion sort by (degree, old id) */
            int32_t x = grp[i];
            int j = i - 1;
            while (j >= 0 && (deg[grp[j]] > deg[x] || (deg[grp[j]] == deg[x] && grp[j] > x))) {
                grp[j + 1] = grp[j];
                j--;
            }
            grp[j + 1] = x;
        }
        for (int i = 0; i < ng; i++) { newid[grp[i]] = (int32_t)next; node_perm_out[next] = grp[i]; next++; }
    }
    for (int64_t i = 0; i < ne * Np; i++) mu_out[i] = newid[mu[i]];
    free(deg); free(newid);
    return next == nn ? ORC_OK : ORC_E_MESH;
}

/* Node Connectivity / Node Distance strategies, reading
 * R20: a Cuthill-McKee traversal of the node graph.  Start at the node with
 * the smallest key; dequeue nodes in order and append each one's unvisited
 * neighbours by ascending key (ties: ascending node id), marking them
 * visited; if the queue empties first (disconnected mesh), restart at the
 * smallest-key unvisited node.  key = degree (Conn.) or the squared distance
 * to the reference point (Dist.), passed in by the caller.  The node list is
 * the visit order (node_perm_out[new] = old).  Elements: at each node in
 * visit order, the elements holding it, ascending id, each appended once
 * (elem_perm_out[new] = input element). */
static const double *g_key;
static int cmp_node_key(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    if (g_key[x] < g_key[y]) return -1;
    if (g_key[x] > g_key[y]) return 1;
    return (x > y) - (x < y);
}

int orc_strategy_order(const int32_t *mu, int64_t ne, int Np, int64_t nn, const double *key,
                       int32_t *elem_perm_out, int32_t *node_perm_out) {
    int64_t *ptr; int32_t *adj;
    int rc = build_node_graph(mu, ne, Np, nn, &ptr, &adj);
    if (rc) return rc;
    uint8_t *vis = (uint8_t *)calloc((size_t)nn + 1, 1);
    int32_t *nb = (int32_t *)malloc(sizeof(int32_t) * 4096);
    if (!vis || !nb) { free(ptr); free(adj); free(vis); free(nb); return ORC_E_OOM; }
    g_key = key;
    int64_t head = 0, tail = 0;
    while (tail < nn) {
        int64_t s = -1; /* smallest-key unvisited node */
        for (int64_t g = 0; g < nn; g++)
            if (!vis[g] && (s < 0 || key[g] < key[s])) s = g;
        vis[s] = 1;
        node_perm_out[tail++] = (int32_t)s;
        while (head < tail) {
            int32_t u = node_perm_out[head++];
            int m = 0;
            for (int64_t j = ptr[u]; j < ptr[u + 1]; j++)
                if (!vis[adj[j]] && m < 4096) nb[m++] = adj[j];
            if (ptr[u + 1] - ptr[u] > 4096) { free(ptr); free(adj); free(vis); free(nb); return ORC_E_MESH; }
            qsort(nb, (size_t)m, sizeof(int32_t), cmp_node_key);
            for (int i = 0; i < m; i++) { vis[nb[i]] = 1; node_perm_out[tail++] = nb[i]; }
        }
    }
    /* element list: node -> elements incidence, ascending element id */
    int64_t *inc_ptr = (int64_t *)calloc((size_t)nn + 1, sizeof(int64_t));
    int32_t *inc = (int32_t *)malloc(sizeof(int32_t) * ((size_t)(ne * Np) + 1));
    uint8_t *done = (uint8_t *)calloc((size_t)ne + 1, 1);
    if (!inc_ptr || !inc || !done) {
        free(ptr); free(adj); free(vis); free(nb); free(inc_ptr); free(inc); free(done);
        return ORC_E_OOM;
    }
    for (int64_t i = 0; i < ne * Np; i++) inc_ptr[mu[i] + 1]++;
    for (int64_t g = 0; g < nn; g++) inc_ptr[g + 1] += inc_ptr[g];
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * ((size_t)nn + 1));
    if (!fill) { free(ptr); free(adj); free(vis); free(nb); free(inc_ptr); free(inc); free(done); return ORC_E_OOM; }
    memcpy(fill, inc_ptr, sizeof(int64_t) * ((size_t)nn + 1));
    for (int64_t e = 0; e < ne; e++)
        for (int p = 0; p < Np; p++) {
            int32_t g = mu[e * Np + p];
            /* an element holding g twice is listed once */
            if (fill[g] == inc_ptr[g] || inc[fill[g] - 1] != (int32_t)e) inc[fill[g]++] = (int32_t)e;
        }
    int64_t k = 0;
    for (int64_t i = 0; i < nn; i++) {
        int32_t g = node_perm_out[i];
        for (int64_t j = inc_ptr[g]; j < fill[g]; j++)
            if (!done[inc[j]]) { done[inc[j]] = 1; elem_perm_out[k++] = inc[j]; }
    }
    free(ptr); free(adj); free(vis); free(nb); free(inc_ptr); free(inc); free(done); free(fill);
    return k == ne ? ORC_OK : ORC_E_MESH;
}

/* Canonical coordinates of every SEM node (for the Node Distance key,
 * reading R20): vertex nodes = the vertex; edge nodes = a + t_i (b - a) with a
 * the lower-id end of the edge and t_i the reference position of the i-th
 * node from that end (edge_t[i], i = 0..P-2); the P3 interior node = the
 * centroid ((v0 + v1) + v2) / 3 of the oriented triangle.  No FMA
 * (-ffp-contract=off).  mu is the canonical connectivity (input order). */
void orc_node_coords(const double *vxy, const int32_t *tri, const int32_t *mu, int64_t ne, int P,
                     const double *edge_t, double *xy) {
    int Np = (P + 1) * (P + 2) / 2;
    for (int64_t e = 0; e < ne; e++) {
        int32_t v[3] = {tri[3 * e], tri[3 * e + 1], tri[3 * e + 2]};
        /* lattice order (R3): local node (i, j), row j outer; edges v0v1 (j = 0),
         * v0v2 (i = 0), v1v2 (i + j = P) */
        int p = 0;
        for (int j = 0; j <= P; j++)
            for (int i = 0; i <= P - j; i++, p++) {
                int32_t g = mu[e * Np + p];
                double x, y;
                if ((i == 0 && j == 0) || (i == P && j == 0) || (i == 0 && j == P)) {
                    int32_t w = (j == P) ? v[2] : (i == P ? v[1] : v[0]);
                    x = vxy[2 * w]; y = vxy[2 * w + 1];
                } else if (j == 0 || i == 0 || i + j == P) {
                    int32_t a, b;
                    int m; /* position from a along a -> b, 1..P-1 */
                    if (j == 0) { a = v[0]; b = v[1]; m = i; }
                    else if (i == 0) { a = v[0]; b = v[2]; m = j; }
                    else { a = v[1]; b = v[2]; m = j; }
                    if (a > b) { int32_t t = a; a = b; b = t; m = P - m; }
                    double t = edge_t[m - 1];
                    x = vxy[2 * a] + t * (vxy[2 * b] - vxy[2 * a]);
                    y = vxy[2 * a + 1] + t * (vxy[2 * b + 1] - vxy[2 * a + 1]);
                } else {
                    x = ((vxy[2 * v[0]] + vxy[2 * v[1]]) + vxy[2 * v[2]]) / 3.0;
                    y = ((vxy[2 * v[0] + 1] + vxy[2 * v[1] + 1]) + vxy[2 * v[2] + 1]) / 3.0;
                }
                xy[2 * g] = x; xy[2 * g + 1] = y;
            }
    }
}

/* Thread count of the oracle's OpenMP loops (bench: the 1-thread baseline). */
void orc_set_num_threads(int n) {
#ifdef _OPENMP
    omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
