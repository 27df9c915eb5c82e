/*
 * oracle.c — CPU ORACLE (TEST INFRASTRUCTURE ONLY; see oracle.h header).
 *
 * Double precision, straight-line loops, no blocking, fusion or reordering
 * beyond what the cited definition states.  Citations: "P:n" = PAPER.md line n
 * (section given), "S:n" = SPEC.md line n, "Dk" = SURVEY.md §8(c) reading k as
 * restated in DESIGN.md §3.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ========================================================================
 * D2 — Philox4x32-10 (Salmon et al., SC'11), NS "counter-based Philox RNG".
 * ======================================================================== */
#define PHILOX_M0 0xD2511F53u
#define PHILOX_M1 0xCD9E8D57u
#define PHILOX_W0 0x9E3779B9u
#define PHILOX_W1 0xBB67AE85u

static void philox_round(uint32_t c[4], const uint32_t k[2]) {
    uint64_t p0 = (uint64_t)PHILOX_M0 * (uint64_t)c[0];
    uint64_t p1 = (uint64_t)PHILOX_M1 * (uint64_t)c[2];
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c[1] ^ k[0];
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c[3] ^ k[1];
    uint32_t n3 = lo0;
    c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
}

void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
    uint32_t k[2] = {key[0], key[1]};
    for (int r = 0; r < 10; ++r) {
        if (r > 0) { k[0] += PHILOX_W0; k[1] += PHILOX_W1; }   /* key bump between rounds */
        philox_round(c, k);
    }
    out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; out[3] = c[3];
}

/* D2 stream layout: key = (lo32 s', hi32 s'), s' = seed + ligand_id * 0x9E3779B97F4A7C15;
   counter = (block, (purpose << 24) | slot, generation, run); word m = lane m&3 of block m>>2. */
uint32_t or_word(uint64_t seed, uint32_t ligand_id, uint32_t purpose, uint32_t slot,
                 uint32_t gen, uint32_t run, uint32_t m) {
    uint64_t s = seed + (uint64_t)ligand_id * 0x9E3779B97F4A7C15ull;
    uint32_t key[2] = {(uint32_t)s, (uint32_t)(s >> 32)};
    uint32_t ctr[4] = {m >> 2, (purpose << 24) | slot, gen, run};
    uint32_t out[4];
    or_philox4x32_10(ctr, key, out);
    return out[m & 3];
}

/* D2 conversions: u01(w) = (w >> 8) * 2^-24; below(w, n) = floor(w * n / 2^32). */
double or_u01(uint32_t w) { return (double)(w >> 8) * (1.0 / 16777216.0); }
uint32_t or_below(uint32_t w, uint32_t n) { return (uint32_t)(((uint64_t)w * (uint64_t)n) >> 32); }

enum { PURPOSE_INIT = 0, PURPOSE_GA = 1, PURPOSE_LS_PICK = 2, PURPOSE_SW = 3 };

/* ========================================================================
 * D1 — ligand topology by brute force (P:135-136 order).
 * ======================================================================== */
static int adjacent(int N, const unsigned char *adj, int i, int j) { return adj[i * N + j]; }

/* BFS from s over the bond graph, optionally forbidding the edge {fx, fy}. */
static void bfs(int N, const unsigned char *adj, int s, int fx, int fy, int *dist) {
    int *queue = (int *)malloc(sizeof(int) * N);
    for (int i = 0; i < N; ++i) dist[i] = -1;
    int head = 0, tail = 0;
    dist[s] = 0; queue[tail++] = s;
    while (head < tail) {
        int u = queue[head++];
        for (int v = 0; v < N; ++v) {
            if (!adjacent(N, adj, u, v) || dist[v] >= 0) continue;
            if ((u == fx && v == fy) || (u == fy && v == fx)) continue;
            dist[v] = dist[u] + 1;
            queue[tail++] = v;
        }
    }
    free(queue);
}

int or_topology(int N, int n_bonds, const int *bonds, const unsigned char *rotatable,
                int *T_out, int *tor_a, int *tor_b, unsigned char *moved, int *depth,
                int *P_out, int *pairs, int cap, int *frag_out) {
    if (N < 1 || N > OR_MAX_ATOMS || n_bonds < 0) return 1;
    unsigned char *adj = (unsigned char *)calloc((size_t)N * N, 1);
    unsigned char *rotadj = (unsigned char *)calloc((size_t)N * N, 1);
    int rc = 1;
    int *dist = (int *)malloc(sizeof(int) * N * N);
    int *frag = (int *)malloc(sizeof(int) * N);
    int *tmp = (int *)malloc(sizeof(int) * N);
    int nrot = 0;
    int ra[OR_MAX_TORS], rb[OR_MAX_TORS];
    for (int e = 0; e < n_bonds; ++e) {
        int x = bonds[2 * e], y = bonds[2 * e + 1];
        if (x < 0 || y < 0 || x >= N || y >= N || x == y) goto done;
        if (adj[x * N + y]) goto done;                          /* duplicate bond */
        adj[x * N + y] = adj[y * N + x] = 1;
        if (rotatable && rotatable[e]) {
            if (nrot >= OR_MAX_TORS) goto done;
            rotadj[x * N + y] = rotadj[y * N + x] = 1;
            ra[nrot] = x; rb[nrot] = y; ++nrot;
        }
    }
    /* bond-path distances, all pairs, one BFS per atom (brute force) */
    for (int s = 0; s < N; ++s) bfs(N, adj, s, -1, -1, dist + s * N);
    for (int i = 0; i < N; ++i) if (dist[i] < 0) goto done;    /* D1.1 connected */
    /* D1.1 every rotatable bond is a bridge (not in a ring) */
    for (int k = 0; k < nrot; ++k) {
        bfs(N, adj, ra[k], ra[k], rb[k], tmp);
        if (tmp[rb[k]] >= 0) goto done;
    }
    /* D1.2 rigid fragments: components after deleting the rotatable bonds */
    for (int i = 0; i < N; ++i) frag[i] = -1;
    int nfrag = 0;
    for (int s = 0; s < N; ++s) {
        if (frag[s] >= 0) continue;
        int *q = tmp; int head = 0, tail = 0;
        frag[s] = nfrag; q[tail++] = s;
        while (head < tail) {
            int u = q[head++];
            for (int v = 0; v < N; ++v)
                if (adj[u * N + v] && !rotadj[u * N + v] && frag[v] < 0) { frag[v] = nfrag; q[tail++] = v; }
        }
        ++nfrag;
    }
    /* D1.3 root fragment: largest; tie -> the one holding the smallest atom index.
       Fragments are numbered in order of their smallest atom, so the first max wins. */
    int root = 0, best = -1;
    for (int f = 0; f < nfrag; ++f) {
        int sz = 0;
        for (int i = 0; i < N; ++i) sz += (frag[i] == f);
        if (sz > best) { best = sz; root = f; }
    }
    int root_atom = -1;
    for (int i = 0; i < N; ++i) if (frag[i] == root) { root_atom = i; break; }
    /* D1.4 orient each torsion: a on the root side; moved = far side minus b */
    int ta[OR_MAX_TORS], tb[OR_MAX_TORS], tdep[OR_MAX_TORS];
    unsigned char far_[OR_MAX_TORS][OR_MAX_ATOMS];
    for (int k = 0; k < nrot; ++k) {
        bfs(N, adj, root_atom, ra[k], rb[k], tmp);   /* reachable from root without the bond */
        if (tmp[ra[k]] >= 0) { ta[k] = ra[k]; tb[k] = rb[k]; } else { ta[k] = rb[k]; tb[k] = ra[k]; }
        bfs(N, adj, tb[k], ta[k], tb[k], tmp);       /* far side, from b without crossing */
        for (int i = 0; i < N; ++i) far_[k][i] = (tmp[i] >= 0);
    }
    /* D1.5 depth = number of rotatable bonds on the path root -> b_k
       = #{ j : b_k lies on the far side of torsion j } */
    for (int k = 0; k < nrot; ++k) {
        int d = 0;
        for (int j = 0; j < nrot; ++j) d += far_[j][tb[k]];
        tdep[k] = d;
    }
    /* sort by (depth, a, b): plain selection sort */
    int order[OR_MAX_TORS];
    for (int k = 0; k < nrot; ++k) order[k] = k;
    for (int i = 0; i < nrot; ++i)
        for (int j = i + 1; j < nrot; ++j) {
            int u = order[i], v = order[j];
            int less = (tdep[v] < tdep[u]) || (tdep[v] == tdep[u] && (ta[v] < ta[u] ||
                       (ta[v] == ta[u] && tb[v] < tb[u])));
            if (less) { order[i] = v; order[j] = u; }
        }
    for (int k = 0; k < nrot; ++k) {
        int o = order[k];
        tor_a[k] = ta[o]; tor_b[k] = tb[o];
        if (depth) depth[k] = tdep[o];
        for (int i = 0; i < N; ++i) moved[k * N + i] = (unsigned char)(far_[o][i] && i != tb[o]);
    }
    *T_out = nrot;
    /* D1.6 pairs: i < j, bond distance >= 4, different rigid fragments, lexicographic */
    int np = 0;
    for (int i = 0; i < N; ++i)
        for (int j = i + 1; j < N; ++j)
            if (dist[i * N + j] >= 4 && frag[i] != frag[j]) {
                if (np < cap) { pairs[2 * np] = i; pairs[2 * np + 1] = j; }
                ++np;
            }
    *P_out = np;
    if (frag_out) for (int i = 0; i < N; ++i) frag_out[i] = frag[i];
    rc = (np > cap) ? 1 : 0;
done:
    free(adj); free(rotadj); free(dist); free(frag); free(tmp);
    return rc;
}

/* D1.7 — verbatim torsions and pairs ("moved excludes axis_a and axis_b",
   S:91-93 TORSION / PAIR records), checked by brute force over all torsion pairs k < j:
   (a) indices in range, a_k != b_k, moved(k) without duplicates and without a_k, b_k;
   (b) moved(k) and moved(j) nested or disjoint;
   (c) a nested set comes after the set containing it (parents first);
   (d) {a_k, b_k} is not moved by a later torsion j;
   (e) if moved(j) lies inside a non-disjoint moved(k), the axis atoms of j are carried by k
       (in moved(k) or on k's axis), so the world axis of j turns with k (D7's w_j);
   (f) pairs: in range, i != j, no duplicate unordered pair; returned with i < j, list order.
   Returns 0 (ok) or 1 (input error). */
int or_topology_verbatim(int N, int T, const int *axis, const int *moved_off, const int *moved_idx, int P,
                         const int *pairs_in, int *tor_a, int *tor_b, unsigned char *moved, int *pairs_out) {
    if (N < 1 || N > OR_MAX_ATOMS || T < 0 || T > OR_MAX_TORS || P < 0) return 1;
    for (int k = 0; k < T * N; ++k) moved[k] = 0;
    for (int k = 0; k < T; ++k) {                                           /* (a) */
        int a = axis[2 * k], b = axis[2 * k + 1];
        if (a < 0 || a >= N || b < 0 || b >= N || a == b) return 1;
        if (moved_off[k + 1] < moved_off[k]) return 1;
        for (int q = moved_off[k]; q < moved_off[k + 1]; ++q) {
            int m = moved_idx[q];
            if (m < 0 || m >= N || m == a || m == b || moved[k * N + m]) return 1;
            moved[k * N + m] = 1;
        }
        tor_a[k] = a; tor_b[k] = b;
    }
    for (int k = 0; k < T; ++k)
        for (int j = k + 1; j < T; ++j) {
            int both = 0, only_k = 0, only_j = 0;
            for (int m = 0; m < N; ++m) {
                both += moved[k * N + m] && moved[j * N + m];
                only_k += moved[k * N + m] && !moved[j * N + m];
                only_j += !moved[k * N + m] && moved[j * N + m];
            }
            if (both && only_k && only_j) return 1;                            /* (b) */
            if (both && !only_k && only_j) return 1;                           /* (c) k inside j */
            if (moved[j * N + tor_a[k]] || moved[j * N + tor_b[k]]) return 1; /* (d) */
            if (both && !only_j) {                                             /* (e) j inside k */
                for (int e = 0; e < 2; ++e) {
                    int x = e ? tor_b[j] : tor_a[j];
                    if (!moved[k * N + x] && x != tor_a[k] && x != tor_b[k]) return 1;
                }
            }
        }
    for (int q = 0; q < P; ++q) {                                              /* (f) */
        int i = pairs_in[2 * q], j = pairs_in[2 * q + 1];
        if (i < 0 || i >= N || j < 0 || j >= N || i == j) return 1;
        if (i > j) { int t = i; i = j; j = t; }
        for (int r = 0; r < q; ++r)
            if (pairs_out[2 * r] == i && pairs_out[2 * r + 1] == j) return 1;
        pairs_out[2 * q] = i; pairs_out[2 * q + 1] = j;
    }
    return 0;
}

/* ========================================================================
 * D3 — genotype -> pose (NS "orientation quaternion").
 * ======================================================================== */
static void cross3(const double a[3], const double b[3], double o[3]) {
    o[0] = a[1] * b[2] - a[2] * b[1];
    o[1] = a[2] * b[0] - a[0] * b[2];
    o[2] = a[0] * b[1] - a[1] * b[0];
}
static double dot3(const double a[3], const double b[3]) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }

/* Rodrigues, right-handed: Rot(u, t) v = v cos t + (u x v) sin t + u (u.v)(1 - cos t) */
static void rodrigues(const double u[3], double t, const double v[3], double o[3]) {
    double c = cos(t), s = sin(t), uxv[3];
    cross3(u, v, uxv);
    double ud = dot3(u, v);
    for (int d = 0; d < 3; ++d) o[d] = v[d] * c + uxv[d] * s + u[d] * ud * (1.0 - c);
}

static void centroid(const or_problem *P, double c[3]) {
    c[0] = c[1] = c[2] = 0.0;
    for (int a = 0; a < P->N; ++a) for (int d = 0; d < 3; ++d) c[d] += P->X[3 * a + d];
    for (int d = 0; d < 3; ++d) c[d] /= (double)P->N;
}

/* n = (sin th cos ph, sin th sin ph, cos th); q = (cos a/2, sin(a/2) n); R = R(q). */
static void orientation(const double *genes, double n[3], double R[3][3]) {
    double ph = genes[3], th = genes[4], al = genes[5];
    n[0] = sin(th) * cos(ph); n[1] = sin(th) * sin(ph); n[2] = cos(th);
    double w = cos(0.5 * al), s = sin(0.5 * al);
    double x = s * n[0], y = s * n[1], z = s * n[2];
    R[0][0] = 1 - 2 * (y * y + z * z); R[0][1] = 2 * (x * y - w * z);     R[0][2] = 2 * (x * z + w * y);
    R[1][0] = 2 * (x * y + w * z);     R[1][1] = 1 - 2 * (x * x + z * z); R[1][2] = 2 * (y * z - w * x);
    R[2][0] = 2 * (x * z - w * y);     R[2][1] = 2 * (y * z + w * x);     R[2][2] = 1 - 2 * (x * x + y * y);
}

void or_pose(const or_problem *P, const double *genes, double *xyz) {
    int N = P->N;
    double c[3];
    centroid(P, c);
    double (*p)[3] = (double (*)[3])malloc(sizeof(double) * 3 * N);
    double (*y)[3] = (double (*)[3])malloc(sizeof(double) * 3 * N);
    for (int a = 0; a < N; ++a) for (int d = 0; d < 3; ++d) { p[a][d] = P->X[3 * a + d] - c[d]; y[a][d] = p[a][d]; }
    /* torsions in reference-axis form, k = T .. 1 (D3) */
    for (int k = P->T - 1; k >= 0; --k) {
        const double *A = p[P->tor_a[k]];
        double u[3];
        for (int d = 0; d < 3; ++d) u[d] = p[P->tor_b[k]][d] - A[d];
        double nu = sqrt(dot3(u, u));
        for (int d = 0; d < 3; ++d) u[d] /= nu;
        for (int a = 0; a < N; ++a) {
            if (!P->moved[k * N + a]) continue;
            double v[3], o[3];
            for (int d = 0; d < 3; ++d) v[d] = y[a][d] - A[d];
            rodrigues(u, genes[6 + k], v, o);
            for (int d = 0; d < 3; ++d) y[a][d] = A[d] + o[d];
        }
    }
    double n[3], R[3][3];
    orientation(genes, n, R);
    for (int a = 0; a < N; ++a)
        for (int i = 0; i < 3; ++i)
            xyz[3 * a + i] = genes[i] + R[i][0] * y[a][0] + R[i][1] * y[a][1] + R[i][2] * y[a][2];
    free(p); free(y);
}

/* ========================================================================
 * D4 — intermolecular energy by trilinear interpolation.
 * ======================================================================== */
static double node_value(const or_problem *P, int map, int i, int j, int k) {
    size_t n3 = (size_t)P->nx * P->ny * P->nz;
    return (double)P->maps[(size_t)map * n3 + (size_t)i + (size_t)P->nx * ((size_t)j + (size_t)P->ny * (size_t)k)];
}

/* V(M) at fractional grid coordinate u with cell i; dV/du by the same cell (one-sided on faces). */
static double trilinear(const or_problem *P, int map, const int ic[3], const double f[3], double dV[3]) {
    double V = 0.0;
    dV[0] = dV[1] = dV[2] = 0.0;
    for (int cz = 0; cz < 2; ++cz)
        for (int cy = 0; cy < 2; ++cy)
            for (int cx = 0; cx < 2; ++cx) {
                double M = node_value(P, map, ic[0] + cx, ic[1] + cy, ic[2] + cz);
                double wx = cx ? f[0] : 1.0 - f[0];
                double wy = cy ? f[1] : 1.0 - f[1];
                double wz = cz ? f[2] : 1.0 - f[2];
                V += wx * wy * wz * M;
                dV[0] += (cx ? 1.0 : -1.0) * wy * wz * M;
                dV[1] += wx * (cy ? 1.0 : -1.0) * wz * M;
                dV[2] += wx * wy * (cz ? 1.0 : -1.0) * M;
            }
    return V;
}

double or_inter_atom(const or_problem *P, int a, const double r[3], double grad[3]) {
    const int n[3] = {P->nx, P->ny, P->nz};
    double u[3];
    int inside = 1;
    for (int d = 0; d < 3; ++d) {
        u[d] = (r[d] - P->origin[d]) / P->spacing;                     /* D4.1 */
        if (!(u[d] >= 0.0 && u[d] <= (double)(n[d] - 1))) inside = 0;
    }
    if (inside) {
        int ic[3]; double f[3];
        for (int d = 0; d < 3; ++d) {                                   /* D4.2 */
            int i = (int)floor(u[d]);
            if (i > n[d] - 2) i = n[d] - 2;
            ic[d] = i; f[d] = u[d] - (double)i;
        }
        double q = P->q[a], aq = fabs(q);
        double dT[3], dE[3], dD[3];
        double VT = trilinear(P, P->type[a], ic, f, dT);                /* D4.3 */
        double VE = trilinear(P, P->n_types, ic, f, dE);
        double VD = trilinear(P, P->n_types + 1, ic, f, dD);
        if (grad) for (int d = 0; d < 3; ++d) grad[d] = (dT[d] + q * dE[d] + aq * dD[d]) / P->spacing; /* D4.6 */
        return VT + q * VE + aq * VD;                                   /* D4.4 */
    }
    /* D4.5 outside: 1e5 (1 + d), d = |r - clamp(r, o, o + (n-1)s)| */
    double cl[3], dv[3], dd = 0.0;
    for (int d = 0; d < 3; ++d) {
        double lo = P->origin[d], hi = P->origin[d] + (double)(n[d] - 1) * P->spacing;
        cl[d] = r[d] < lo ? lo : (r[d] > hi ? hi : r[d]);
        dv[d] = r[d] - cl[d];
        dd += dv[d] * dv[d];
    }
    dd = sqrt(dd);
    if (grad) for (int d = 0; d < 3; ++d) grad[d] = (dd > 0.0) ? 1e5 * dv[d] / dd : 0.0;
    return 1e5 * (1.0 + dd);
}

double or_inter(const or_problem *P, const double *xyz, double *grad) {
    double E = 0.0;
    for (int a = 0; a < P->N; ++a) E += or_inter_atom(P, a, xyz + 3 * a, grad ? grad + 3 * a : NULL); /* D4.7 ascending a */
    return E;
}

/* ========================================================================
 * D5 — intramolecular pair energy ("hydrogen bonding,
 * van der Waals forces, and desolvation effects").
 * ======================================================================== */
#define ELEC_K 332.06363
#define OR_PI 3.14159265358979323846
#define DESOLV_SIGMA 3.6

double or_pair_energy(const or_problem *P, int i, int j, double rho2_in, double *dE_drho2) {
    if (P->sf) return or_pair_energy_ad4(P, i, j, rho2_in, dE_drho2);   /* NEXT-2 variant */
    int ti = P->type[i], tj = P->type[j];
    double req = 0.5 * (P->tR[ti] + P->tR[tj]);                        /* r_eq = (R_i + R_j)/2 */
    double eps = sqrt(P->teps[ti] * P->teps[tj]);                      /* eps_ij = sqrt(eps_i eps_j) */
    int hb = (P->trole[ti] == 1 && P->trole[tj] == 2) || (P->trole[ti] == 2 && P->trole[tj] == 1);
    int clamped = rho2_in < 1e-4;
    double rho2 = clamped ? 1e-4 : rho2_in;                            /* 0.01 Å clamp */
    double x2 = req * req / rho2;
    double x4 = x2 * x2, x6 = x4 * x2, x8 = x4 * x4, x10 = x8 * x2, x12 = x6 * x6;
    double Evdw, dvdw;
    if (hb) {
        Evdw = eps * (5.0 * x12 - 6.0 * x10);                          /* 12-10 */
        dvdw = -eps * 30.0 * (x12 - x10) / rho2;
    } else {
        Evdw = eps * (x12 - 2.0 * x6);                                 /* 12-6 */
        dvdw = -eps * 6.0 * (x12 - x6) / rho2;
    }
    double Eel = ELEC_K * P->q[i] * P->q[j] / (4.0 * rho2);            /* eps(r) = 4r */
    double del = -Eel / rho2;
    double SV = P->tS[ti] * P->tV[tj] + P->tS[tj] * P->tV[ti];
    double Eds = SV * exp(-rho2 / (2.0 * DESOLV_SIGMA * DESOLV_SIGMA));
    double dds = -Eds / (2.0 * DESOLV_SIGMA * DESOLV_SIGMA);
    if (dE_drho2) *dE_drho2 = clamped ? 0.0 : (dvdw + del + dds);
    return Evdw + Eel + Eds;
}

/* ========================================================================
 * NEXT-2 — D5-AD4: the AutoDock4.1-calibrated pair energy (SURVEY.md §8(f) rank 2,
 * SPEC S:219-223, 232).  Same pair list, clamp and role rule as D5; per
 * pair, with r = |r_i - r_j| (r >= 0.01 Å after the D5 clamp):
 *   vdW / H-bond: the D5 12-6 / 12-10 form times w_vdw / w_hb, evaluated at the smoothed
 *     distance r_s (AD4 smoothing: the potential is replaced by its minimum over
 *     [r - smooth/2, r + smooth/2]; the D5 forms have one minimum, at r_eq, so
 *     r_s = r + smooth/2 below r_eq - smooth/2, r - smooth/2 above r_eq + smooth/2, and
 *     r_eq in between), and only for r < cut_vdw;
 *   electrostatic: w_el 332.06363 q_i q_j / (r eps(r)), eps(r) the Mehler-Solmajer
 *     sigmoid A + B / (1 + k exp(-lambda B r)), B = eps0 - A (diel = 1), or 4r (diel = 0);
 *   desolvation: w_ds (S'_i V_j + S'_j V_i) exp(-r^2 / (2 sigma^2)), S'_i = S_i + qasp |q_i|;
 *   electrostatic and desolvation only for r < cut_el.
 * Derivatives are taken piece by piece (zero on the smoothing plateau and beyond a
 * cutoff) and returned as dE/d(rho^2) = (dE/dr) / (2r), zero under the clamp as in D5.
 * ======================================================================== */
double or_dielectric(const or_scoring *s, double r, double *deps_dr) {
    if (s->diel == 0) {                                                 /* eps(r) = 4r */
        if (deps_dr) *deps_dr = 4.0;
        return 4.0 * r;
    }
    double B = s->diel_eps0 - s->diel_A;
    double e = exp(-s->diel_lambda * B * r);
    double den = 1.0 + s->diel_k * e;
    if (deps_dr) *deps_dr = B * s->diel_k * s->diel_lambda * B * e / (den * den);
    return s->diel_A + B / den;
}

double or_pair_energy_ad4(const or_problem *P, int i, int j, double rho2_in, double *dE_drho2) {
    const or_scoring *s = P->sf;
    int ti = P->type[i], tj = P->type[j];
    double req = 0.5 * (P->tR[ti] + P->tR[tj]);
    double eps = sqrt(P->teps[ti] * P->teps[tj]);
    int hb = (P->trole[ti] == 1 && P->trole[tj] == 2) || (P->trole[ti] == 2 && P->trole[tj] == 1);
    int clamped = rho2_in < 1e-4;
    double r = sqrt(clamped ? 1e-4 : rho2_in);
    /* vdW / H-bond at the smoothed distance */
    double h = 0.5 * s->smooth, rs, drs;
    if (r < req - h) { rs = r + h; drs = 1.0; }
    else if (r > req + h) { rs = r - h; drs = 1.0; }
    else { rs = req; drs = 0.0; }
    double x = req / rs;
    double x6 = pow(x, 6), x10 = pow(x, 10), x12 = pow(x, 12);
    double Ev, dEv_drs;
    if (hb) {
        Ev = s->w_hb * eps * (5.0 * x12 - 6.0 * x10);
        dEv_drs = s->w_hb * eps * (-60.0 * x12 + 60.0 * x10) / rs;
    } else {
        Ev = s->w_vdw * eps * (x12 - 2.0 * x6);
        dEv_drs = s->w_vdw * eps * (-12.0 * x12 + 12.0 * x6) / rs;
    }
    double dEv = dEv_drs * drs;
    if (s->cut_vdw > 0.0 && r >= s->cut_vdw) { Ev = 0.0; dEv = 0.0; }
    /* electrostatics */
    double de_dr, epsr = or_dielectric(s, r, &de_dr);
    double Eel = s->w_el * ELEC_K * P->q[i] * P->q[j] / (r * epsr);
    double dEel = -Eel * (1.0 / r + de_dr / epsr);                     /* d/dr [1/(r eps)] */
    /* desolvation with charge-dependent solvation parameters */
    double Si = P->tS[ti] + s->qasp * fabs(P->q[i]), Sj = P->tS[tj] + s->qasp * fabs(P->q[j]);
    double SV = Si * P->tV[tj] + Sj * P->tV[ti];
    double Eds = s->w_ds * SV * exp(-r * r / (2.0 * s->sigma * s->sigma));
    double dEds = -Eds * r / (s->sigma * s->sigma);
    if (s->cut_el > 0.0 && r >= s->cut_el) { Eel = Eds = dEel = dEds = 0.0; }
    if (dE_drho2) *dE_drho2 = clamped ? 0.0 : (dEv + dEel + dEds) / (2.0 * r);
    return Ev + Eel + Eds;
}

double or_kink_margin(const or_problem *P, const double *xyz) {
    if (!P->sf) return 1e300;
    const or_scoring *s = P->sf;
    double m = 1e300;
    for (int p = 0; p < P->P; ++p) {
        int i = P->pairs[2 * p], j = P->pairs[2 * p + 1];
        double r2 = 0.0;
        for (int d = 0; d < 3; ++d) { double v = xyz[3 * i + d] - xyz[3 * j + d]; r2 += v * v; }
        double r = sqrt(r2);
        double req = 0.5 * (P->tR[P->type[i]] + P->tR[P->type[j]]);
        double k[4] = {req - 0.5 * s->smooth, req + 0.5 * s->smooth, s->cut_vdw, s->cut_el};
        for (int t = 0; t < 4; ++t)
            if (fabs(r - k[t]) < m) m = fabs(r - k[t]);
    }
    return m;
}

double or_binding_dG(const or_problem *P, double e_inter) {
    return e_inter + (P->sf ? P->sf->w_tors * P->T : 0.0);             /* AD4 unbound = bound model */
}

double or_intra(const or_problem *P, const double *xyz, double *grad) {
    if (grad) for (int i = 0; i < 3 * P->N; ++i) grad[i] = 0.0;
    double E = 0.0;
    for (int p = 0; p < P->P; ++p) {                                   /* list order */
        int i = P->pairs[2 * p], j = P->pairs[2 * p + 1];
        double dv[3], r2 = 0.0;
        for (int d = 0; d < 3; ++d) { dv[d] = xyz[3 * i + d] - xyz[3 * j + d]; r2 += dv[d] * dv[d]; }
        double dE;
        E += or_pair_energy(P, i, j, r2, &dE);
        if (grad)
            for (int d = 0; d < 3; ++d) {                              /* dE/dr_i = 2 dE/drho2 (r_i - r_j) */
                grad[3 * i + d] += 2.0 * dE * dv[d];
                grad[3 * j + d] -= 2.0 * dE * dv[d];
            }
    }
    return E;
}

/* ========================================================================
 * D6 total energy and D7 genotype gradient (NS).
 * ======================================================================== */
/* D6 + D7 of the genotype `genes` whose world coordinates are r (or_pose(genes), or a
   given pose: or_energy_at).  Everything after D3 is evaluated at r. */
static double energy_of_pose(const or_problem *P, const double *genes, const double *r, double *ggrad,
                             double *terms) {
    int N = P->N;
    double *gi = (double *)malloc(sizeof(double) * 3 * N);
    double *gp = (double *)malloc(sizeof(double) * 3 * N);
    double Ei = or_inter(P, r, ggrad ? gi : NULL);
    double Ep = or_intra(P, r, ggrad ? gp : NULL);
    if (ggrad) {
        int G = 6 + P->T;
        for (int j = 0; j < G; ++j) ggrad[j] = 0.0;
        double Gam[3] = {0, 0, 0};
        for (int a = 0; a < N; ++a) {
            double g[3], ra[3], c[3];
            for (int d = 0; d < 3; ++d) { g[d] = gi[3 * a + d] + gp[3 * a + d]; ra[d] = r[3 * a + d] - genes[d]; }
            for (int d = 0; d < 3; ++d) ggrad[d] += g[d];                 /* dE/dt = sum g_a */
            cross3(ra, g, c);                                               /* Gamma = sum (r_a - t) x g_a */
            for (int d = 0; d < 3; ++d) Gam[d] += c[d];
        }
        double ph = genes[3], th = genes[4], al = genes[5];
        double n[3] = {sin(th) * cos(ph), sin(th) * sin(ph), cos(th)};
        double dn_ph[3] = {-sin(th) * sin(ph), sin(th) * cos(ph), 0.0};
        double dn_th[3] = {cos(th) * cos(ph), cos(th) * sin(ph), -sin(th)};
        double cx[3], w[3];
        /* omega = adot n + sin(a) ndot + (1 - cos a) n x ndot */
        cross3(n, dn_ph, cx);
        for (int d = 0; d < 3; ++d) w[d] = sin(al) * dn_ph[d] + (1.0 - cos(al)) * cx[d];
        ggrad[3] = dot3(Gam, w);
        cross3(n, dn_th, cx);
        for (int d = 0; d < 3; ++d) w[d] = sin(al) * dn_th[d] + (1.0 - cos(al)) * cx[d];
        ggrad[4] = dot3(Gam, w);
        ggrad[5] = dot3(Gam, n);
        /* dE/dtau_k = w_k . sum_{a in moved(k)} (r_a - r_{a_k}) x g_a, w_k world axis a_k -> b_k */
        for (int k = 0; k < P->T; ++k) {
            int ak = P->tor_a[k], bk = P->tor_b[k];
            double wk[3];
            for (int d = 0; d < 3; ++d) wk[d] = r[3 * bk + d] - r[3 * ak + d];
            double nw = sqrt(dot3(wk, wk));
            for (int d = 0; d < 3; ++d) wk[d] /= nw;
            double S[3] = {0, 0, 0};
            for (int a = 0; a < N; ++a) {
                if (!P->moved[k * N + a]) continue;
                double v[3], g[3], c[3];
                for (int d = 0; d < 3; ++d) { v[d] = r[3 * a + d] - r[3 * ak + d]; g[d] = gi[3 * a + d] + gp[3 * a + d]; }
                cross3(v, g, c);
                for (int d = 0; d < 3; ++d) S[d] += c[d];
            }
            ggrad[6 + k] = dot3(wk, S);
        }
    }
    if (terms) { terms[0] = Ei; terms[1] = Ep; }
    free(gi); free(gp);
    return Ei + Ep;                                                     /* D6: E = E_inter + E_intra */
}

double or_energy(const or_problem *P, const double *genes, double *ggrad, double *xyz_out, double *terms) {
    int N = P->N;
    double *r = (double *)malloc(sizeof(double) * 3 * N);
    or_pose(P, genes, r);                                               /* D3 */
    double E = energy_of_pose(P, genes, r, ggrad, terms);
    if (xyz_out) for (int i = 0; i < 3 * N; ++i) xyz_out[i] = r[i];
    free(r);
    return E;
}

double or_energy_at(const or_problem *P, const double *genes, const double *xyz, double *ggrad, double *terms) {
    return energy_of_pose(P, genes, xyz, ggrad, terms);
}

void or_margins(const or_problem *P, const double *xyz, double *face_margin, double *clamp_margin) {
    double fm = 1e300, cm = 1e300;
    for (int a = 0; a < P->N; ++a)
        for (int d = 0; d < 3; ++d) {
            double u = (xyz[3 * a + d] - P->origin[d]) / P->spacing;
            double m = fabs(u - floor(u + 0.5));
            if (m < fm) fm = m;
        }
    for (int p = 0; p < P->P; ++p) {
        int i = P->pairs[2 * p], j = P->pairs[2 * p + 1];
        double r2 = 0.0;
        for (int d = 0; d < 3; ++d) { double v = xyz[3 * i + d] - xyz[3 * j + d]; r2 += v * v; }
        double m = fabs(r2 - 1e-4);
        if (m < cm) cm = m;
    }
    *face_margin = fm; *clamp_margin = cm;
}

/* ========================================================================
 * D8 — genetic algorithm ("crossover ... selected ... based on a numerical
 * fitness score").
 * ======================================================================== */
static double key_of(double e) { return isnan(e) ? INFINITY : e; }   /* D reading 21: NaN = +inf */

int or_elite(int pop, const double *E) {
    int e = 0;
    for (int i = 1; i < pop; ++i) if (key_of(E[i]) < key_of(E[e])) e = i;   /* ties -> lowest index */
    return e;
}

static int tournament(const or_params *pp, int pop, const double *E, uint32_t wa, uint32_t wb, uint32_t wc) {
    int i = (int)or_below(wa, (uint32_t)pop);
    int j = (int)or_below(wb, (uint32_t)(pop - 1));
    if (j >= i) j += 1;                                                  /* two distinct candidates */
    double ei = key_of(E[i]), ej = key_of(E[j]);
    int better = (ei < ej || (ei == ej && i < j)) ? i : j;              /* tie -> lower index */
    int other = (better == i) ? j : i;
    return (or_u01(wc) < pp->p_tour) ? better : other;
}

void or_ga_slot(const or_params *pp, uint64_t seed, uint32_t ligand_id, uint32_t run, uint32_t gen,
                uint32_t slot, int pop, int G, const double *old_genes, const double *old_E,
                double *child, int *dbg) {
    uint32_t w[9 + 2 * OR_MAX_GENES] = {0};
    for (int m = 0; m < 9 + 2 * G; ++m) w[m] = or_word(seed, ligand_id, PURPOSE_GA, slot, gen, run, (uint32_t)m);
    int A = tournament(pp, pop, old_E, w[0], w[1], w[2]);
    int B = tournament(pp, pop, old_E, w[3], w[4], w[5]);
    for (int j = 0; j < G; ++j) child[j] = old_genes[A * G + j];
    int cross = or_u01(w[6]) < pp->p_cross;
    int c1 = 0, c2 = 0;
    if (cross) {                                                         /* two-point crossover */
        c1 = (int)or_below(w[7], (uint32_t)(G + 1));
        c2 = (int)or_below(w[8], (uint32_t)(G + 1));
        if (c2 < c1) { int t = c1; c1 = c2; c2 = t; }
        for (int j = c1; j < c2; ++j) child[j] = old_genes[B * G + j];
    }
    uint32_t mlo = 0, mhi = 0;
    for (int j = 0; j < G; ++j) {                                        /* mutation */
        if (or_u01(w[9 + 2 * j]) < pp->p_mut) {
            double m = (j < 3) ? pp->mut_trans : pp->mut_angle;
            child[j] += (2.0 * or_u01(w[10 + 2 * j]) - 1.0) * m;
            if (j < 32) mlo |= 1u << j; else mhi |= 1u << (j - 32);
        }
    }
    if (dbg) {
        dbg[0] = A; dbg[1] = B; dbg[2] = cross; dbg[3] = c1; dbg[4] = c2;
        dbg[5] = (int)mlo; dbg[6] = (int)mhi; dbg[7] = 0;
    }
}

/* n_ls = ceil(ls_rate * pop), with the DESIGN.md reading 16a guard against float32 rates. */
int or_n_ls(double ls_rate, int pop) {
    int n = (int)ceil(ls_rate * (double)pop - 1e-4);
    if (n < 0) n = 0;
    if (n > pop) n = pop;
    return n;
}

/* Partial Fisher-Yates without replacement (D8.3). */
void or_ls_pick(uint64_t seed, uint32_t ligand_id, uint32_t run, uint32_t gen, int pop, int n_ls, int *perm) {
    for (int i = 0; i < pop; ++i) perm[i] = i;
    for (int s = 0; s < n_ls; ++s) {
        uint32_t w = or_word(seed, ligand_id, PURPOSE_LS_PICK, 0, gen, run, (uint32_t)s);
        int j = s + (int)or_below(w, (uint32_t)(pop - s));
        int t = perm[s]; perm[s] = perm[j]; perm[j] = t;
    }
}

/* ========================================================================
 * D9 Solis-Wets (Solis & Wets 1981) and D10 ADADELTA (NS).
 * ======================================================================== */
static double objective(const or_problem *P, const double *bowl, int G, const double *x, double *g) {
    if (P) return or_energy(P, x, g, NULL, NULL);
    double E = 0.0;
    for (int j = 0; j < G; ++j) {
        E += bowl[j] * x[j] * x[j];
        if (g) g[j] = 2.0 * bowl[j] * x[j];
    }
    return E;
}

/* One energy call of the D9 / D10 objective: the docking energy of P, the bowl, or (Solis-
   Wets "fed" mode, parity protocol of SURVEY §8(c)) the table entry Etab[2 it + cand]. */
static double sw_objective(const or_problem *P, const double *bowl, int G, const double *Etab, int it, int cand,
                           const double *x) {
    if (Etab) return Etab[2 * it + cand];
    return objective(P, bowl, G, x, NULL);
}

void or_solis_wets_traced(const or_problem *P, const double *bowl, int G, const or_params *pp,
                          uint64_t seed, uint32_t ligand_id, uint32_t run, uint32_t gen, uint32_t slot,
                          double *x, double *E, int64_t *evals, const double *Etab,
                          int *trace_o, double *trace_rho, double *trace_E) {
    double rho = pp->sw_rho, b[OR_MAX_GENES], d[OR_MAX_GENES], c[OR_MAX_GENES];
    int succ = 0, fail = 0;
    double Ex = *E;
    int64_t ne = 0;
    for (int j = 0; j < G; ++j) b[j] = 0.0;
    for (int it = 0; it < pp->ls_max_iters; ++it) {
        if (trace_o) trace_o[it] = -1;                                   /* not executed */
        if (rho < pp->sw_rho_min) break;                                 /* 1. */
        if (trace_rho) trace_rho[it] = rho;
        for (int j = 0; j < G; ++j) {                                    /* 2. triangular deviate */
            uint32_t w1 = or_word(seed, ligand_id, PURPOSE_SW, slot, gen, run, (uint32_t)(2 * G * it + 2 * j));
            uint32_t w2 = or_word(seed, ligand_id, PURPOSE_SW, slot, gen, run, (uint32_t)(2 * G * it + 2 * j + 1));
            d[j] = rho * (or_u01(w1) + or_u01(w2) - 1.0);
        }
        int o;
        double Ex0 = Ex, E2 = NAN;
        for (int j = 0; j < G; ++j) c[j] = x[j] + b[j] + d[j];          /* 3. x + b + d */
        double Ec = sw_objective(P, bowl, G, Etab, it, 0, c); ++ne;
        double E1 = Ec;
        if (Ec < Ex) {
            for (int j = 0; j < G; ++j) { x[j] = c[j]; b[j] = 0.2 * b[j] + 0.4 * d[j]; }
            Ex = Ec; ++succ; fail = 0; o = 0;
        } else {
            for (int j = 0; j < G; ++j) c[j] = x[j] - b[j] - d[j];      /* 4. x - b - d */
            Ec = sw_objective(P, bowl, G, Etab, it, 1, c); ++ne;
            E2 = Ec;
            if (Ec < Ex) {
                for (int j = 0; j < G; ++j) { x[j] = c[j]; b[j] = b[j] - 0.4 * d[j]; }
                Ex = Ec; ++succ; fail = 0; o = 1;
            } else {                                                     /* 5. */
                for (int j = 0; j < G; ++j) b[j] = 0.5 * b[j];
                ++fail; succ = 0; o = 2;
            }
        }
        if (succ >= pp->sw_cons_succ) { rho *= pp->sw_expand; succ = 0; }   /* 6. */
        if (fail >= pp->sw_cons_fail) { rho *= pp->sw_contract; fail = 0; }
        if (trace_o) trace_o[it] = o;
        if (trace_E) { trace_E[3 * it] = Ex0; trace_E[3 * it + 1] = E1; trace_E[3 * it + 2] = E2; }
    }
    *E = Ex;
    *evals = ne;
}

void or_solis_wets(const or_problem *P, const double *bowl, int G, const or_params *pp,
                   uint64_t seed, uint32_t ligand_id, uint32_t run, uint32_t gen, uint32_t slot,
                   double *x, double *E, int64_t *evals) {
    or_solis_wets_traced(P, bowl, G, pp, seed, ligand_id, run, gen, slot, x, E, evals, NULL, NULL, NULL, NULL);
}

void or_adadelta_traced(const or_problem *P, const double *bowl, int G, const or_params *pp,
                        int iters, double *x, double *E, int64_t *evals, const double *fed,
                        double *trace_x, double *trace_E, double *trace_g) {
    double best[OR_MAX_GENES], sg[OR_MAX_GENES], sd[OR_MAX_GENES], g[OR_MAX_GENES];
    double Ebest = *E;
    for (int j = 0; j < G; ++j) { best[j] = x[j]; sg[j] = 0.0; sd[j] = 0.0; }
    for (int it = 0; it < iters; ++it) {
        if (trace_x) for (int j = 0; j < G; ++j) trace_x[it * G + j] = x[j];
        double Ei;                                                       /* 1. energy + gradient */
        if (fed) {                                                       /* fed mode: (E, grad) of iteration it */
            Ei = fed[it * (G + 1)];
            for (int j = 0; j < G; ++j) g[j] = fed[it * (G + 1) + 1 + j];
        } else {
            Ei = objective(P, bowl, G, x, g);
        }
        if (trace_E) trace_E[it] = Ei;
        if (trace_g) for (int j = 0; j < G; ++j) trace_g[it * G + j] = g[j];
        if (Ei < Ebest) { Ebest = Ei; for (int j = 0; j < G; ++j) best[j] = x[j]; }
        for (int j = 0; j < G; ++j) {                                    /* 2. ADADELTA (Zeiler 2012) */
            sg[j] = pp->ad_rho * sg[j] + (1.0 - pp->ad_rho) * g[j] * g[j];
            double dx = -sqrt(sd[j] + pp->ad_eps) / sqrt(sg[j] + pp->ad_eps) * g[j];
            sd[j] = pp->ad_rho * sd[j] + (1.0 - pp->ad_rho) * dx * dx;
            x[j] += dx;
        }
    }
    for (int j = 0; j < G; ++j) x[j] = best[j];
    *E = Ebest;
    *evals = iters;
}

void or_adadelta(const or_problem *P, const double *bowl, int G, const or_params *pp,
                 int iters, double *x, double *E, int64_t *evals) {
    or_adadelta_traced(P, bowl, G, pp, iters, x, E, evals, NULL, NULL, NULL, NULL);
}

/* ========================================================================
 * D8 + D11 — one run ("several full optimizations each with a starting
 * population of 150 individuals"; P:92 sum_evals; S:336 termination).
 * ======================================================================== */
int64_t or_sum_evals(int n, const int64_t *counters) {
    int64_t s = 0;
    for (int i = 0; i < n; ++i) s += counters[i];                        /* left to right */
    return s;
}

/* D8 generation 0 ("starting population"): gene j of individual k from
   INIT word j of slot k; translation uniform in the box [o, o + (n-1)s], angles 2 pi u01;
   every individual evaluated once (no local search at g = 0). */
void or_init_population(const or_problem *P, int pop, uint64_t seed, uint32_t ligand_id, uint32_t run,
                        double *genes, double *E) {
    int G = 6 + P->T;
    const int n[3] = {P->nx, P->ny, P->nz};
    for (int k = 0; k < pop; ++k) {
        for (int j = 0; j < G; ++j) {
            double u = or_u01(or_word(seed, ligand_id, PURPOSE_INIT, (uint32_t)k, 0, run, (uint32_t)j));
            if (j < 3) {
                double lo = P->origin[j], hi = P->origin[j] + (double)(n[j] - 1) * P->spacing;
                genes[k * G + j] = lo + u * (hi - lo);
            } else {
                genes[k * G + j] = 2.0 * OR_PI * u;
            }
        }
        if (E) E[k] = or_energy(P, genes + k * G, NULL, NULL, NULL);
    }
}

int or_dock_run(const or_problem *P, const or_params *pp, int pop, int64_t max_evals,
                uint64_t seed, uint32_t ligand_id, uint32_t run,
                double *best_E, double *best_genes, int64_t *evals_used, int *generations,
                double *final_E) {
    int G = 6 + P->T;
    double *genes = (double *)malloc(sizeof(double) * pop * G);
    double *ng = (double *)malloc(sizeof(double) * pop * G);
    double *E = (double *)malloc(sizeof(double) * pop);
    double *nE = (double *)malloc(sizeof(double) * pop);
    int64_t *cnt = (int64_t *)calloc((size_t)pop, sizeof(int64_t));
    int *perm = (int *)malloc(sizeof(int) * pop);
    or_init_population(P, pop, seed, ligand_id, run, genes, E);        /* generation 0 */
    for (int k = 0; k < pop; ++k) cnt[k] = 1;
    int64_t evals = or_sum_evals(pop, cnt);                               /* = pop */
    int g = 0;
    int n_ls = or_n_ls(pp->ls_rate, pop);
    while (evals < max_evals && g < pp->max_generations) {
        g += 1;
        for (int k = 0; k < pop; ++k) cnt[k] = 0;
        int e = or_elite(pop, E);                                          /* 1. elitism */
        for (int j = 0; j < G; ++j) ng[j] = genes[e * G + j];
        nE[0] = E[e];
        for (int k = 1; k < pop; ++k) {                                    /* 2. offspring */
            or_ga_slot(pp, seed, ligand_id, run, (uint32_t)g, (uint32_t)k, pop, G, genes, E, ng + k * G, NULL);
            nE[k] = or_energy(P, ng + k * G, NULL, NULL, NULL);
            cnt[k] = 1;
        }
        or_ls_pick(seed, ligand_id, run, (uint32_t)g, pop, n_ls, perm);    /* 3. local search */
        for (int s = 0; s < n_ls; ++s) {
            int i = perm[s];
            int64_t ne = 0;
            if (pp->ls_method == 1)
                or_solis_wets(P, NULL, G, pp, seed, ligand_id, run, (uint32_t)g, (uint32_t)i, ng + i * G, &nE[i], &ne);
            else
                or_adadelta(P, NULL, G, pp, pp->ls_max_iters, ng + i * G, &nE[i], &ne);
            cnt[i] += ne;                                                  /* Lamarckian writeback above */
        }
        evals += or_sum_evals(pop, cnt);                                   /* 4. sum_evals */
        double *t = genes; genes = ng; ng = t;
        double *te = E; E = nE; nE = te;
    }
    int b = or_elite(pop, E);                                              /* best of run */
    *best_E = E[b];
    for (int j = 0; j < G; ++j) best_genes[j] = genes[b * G + j];
    *evals_used = evals;
    *generations = g;
    if (final_E) for (int k = 0; k < pop; ++k) final_E[k] = E[k];
    free(genes); free(ng); free(E); free(nE); free(cnt); free(perm);
    return 0;
}

/* ========================================================================
 * NEXT-3 — clustering of the per-run best poses (DESIGN.md §12
 * reading D12): AutoDock's cluster analysis with plain RMSD, written as its definition.
 * ======================================================================== */
double or_rmsd(int N, const double *a, const double *b) {
    double s = 0.0;
    for (int i = 0; i < 3 * N; ++i) s += (a[i] - b[i]) * (a[i] - b[i]);
    return N > 0 ? sqrt(s / N) : 0.0;
}

int or_cluster(int n, int N, const double *xyz, const double *E, double rmsd_tol, int *cluster,
               double *rmsd_to_seed, int *rank) {
    int *order = (int *)malloc(sizeof(int) * (n > 0 ? n : 1));
    int *seed = (int *)malloc(sizeof(int) * (n > 0 ? n : 1));
    for (int i = 0; i < n; ++i) order[i] = i;
    /* insertion sort by (key, index): key = E, NaN = +inf */
    for (int i = 1; i < n; ++i) {
        int v = order[i], j = i - 1;
        while (j >= 0) {
            double kj = key_of(E[order[j]]), kv = key_of(E[v]);
            if (kj > kv || (kj == kv && order[j] > v)) { order[j + 1] = order[j]; --j; }
            else break;
        }
        order[j + 1] = v;
    }
    int nc = 0;
    for (int t = 0; t < n; ++t) {
        int k = order[t];
        if (rank) rank[k] = t;
        int c = -1;
        double r = 0.0;
        for (int s = 0; s < nc; ++s) {
            r = or_rmsd(N, xyz + (size_t)3 * N * k, xyz + (size_t)3 * N * seed[s]);
            if (r < rmsd_tol) { c = s; break; }
        }
        if (c < 0) { c = nc; seed[nc++] = k; r = 0.0; }
        cluster[k] = c;
        rmsd_to_seed[k] = r;
    }
    free(order); free(seed);
    return nc;
}
