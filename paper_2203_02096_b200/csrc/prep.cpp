// prep.cpp — ligand preprocessing (D1) and grid packing (row a11 of DESIGN.md §1).
//
// Written independently of the oracle (oracle/oracle.c does D1 by brute-force BFS with
// edge removal).  Here: union-find for connectivity and rigid fragments, Tarjan's
// low-link for bridges, a BFS tree from the root fragment to orient torsions, and a
// DFS preorder renumbering that makes every moved set one contiguous atom range
// (PAPER.md:135-136 [§IV-B]: rotations applied "in a particular order").
#include "prep.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>

namespace dk {
namespace {

struct DSU {
    std::vector<int> p;
    explicit DSU(int n) : p(n) { std::iota(p.begin(), p.end(), 0); }
    int find(int a) { while (p[a] != a) { p[a] = p[p[a]]; a = p[a]; } return a; }
    void join(int a, int b) { a = find(a); b = find(b); if (a != b) p[std::max(a, b)] = std::min(a, b); }
};

inline int a16(int x) { return (x + 15) & ~15; }

}  // namespace

Scoring scoring_of(const dock_params &p) {
    Scoring s;
    s.sf = p.scoring;
    if (s.sf == DOCK_SF_AD4) {
        s.w_vdw = p.w_vdw; s.w_hb = p.w_hb; s.w_el = p.w_el; s.w_ds = p.w_ds; s.w_tors = p.w_tors; s.qasp = p.qasp;
    }
    return s;
}

struct Tor { int a, b, depth; };

// D1 outputs shared by both topology modes (DFS numbering: every moved set is one range).
struct Topo {
    std::vector<Tor> tors;                     // torsion order of the genotype
    std::vector<int> order, pos;               // dfs position -> caller atom, and back
    std::vector<int> lo, hi, parent;           // per torsion: moved range [lo, hi), parent torsion
    std::vector<int> deep;                     // per dfs position: innermost torsion (-1: root)
    std::vector<int> pairs;                    // [P*2] caller atom indices, i < j
};

// Derived mode (D1.1-D1.6): union-find, Tarjan bridges, BFS orientation, DFS preorder.
int derive_topology(const dock_ligand *l, Topo &tp, std::string *err) {
    auto fail = [&](const std::string &m) { *err = m; return (int)DOCK_E_INPUT; };
    const int N = l->n_atoms;
    // ---- bond graph ----
    const int B = l->n_bonds;
    std::vector<std::vector<std::pair<int, int>>> adj(N);   // (neighbour, edge id)
    std::vector<uint8_t> seen((size_t)N * N, 0);
    int nrot = 0;
    for (int e = 0; e < B; ++e) {
        const int x = l->bonds[2 * e], y = l->bonds[2 * e + 1];
        const std::string tag = "ligand.bonds[" + std::to_string(e) + "]";
        if (x < 0 || y < 0 || x >= N || y >= N) return fail(tag + ": atom index out of range");
        if (x == y) return fail(tag + ": self bond");
        if (seen[(size_t)x * N + y]) return fail(tag + ": duplicate bond");
        seen[(size_t)x * N + y] = seen[(size_t)y * N + x] = 1;
        adj[x].push_back({y, e});
        adj[y].push_back({x, e});
        if (l->rotatable && l->rotatable[e]) ++nrot;
    }
    if (nrot > kMaxTors) return fail("ligand.rotatable: more than 32 rotatable bonds");
    for (auto &v : adj) std::sort(v.begin(), v.end());
    auto is_rot = [&](int e) { return l->rotatable && l->rotatable[e] != 0; };
    {
        DSU all(N);
        for (int e = 0; e < B; ++e) all.join(l->bonds[2 * e], l->bonds[2 * e + 1]);
        for (int a = 1; a < N; ++a)
            if (all.find(a) != all.find(0)) return fail("ligand.bonds: graph not connected (atom " + std::to_string(a) + ")");
    }
    // ---- bridges: Tarjan low-link, iterative ----
    std::vector<uint8_t> bridge(B, 0);
    {
        std::vector<int> disc(N, -1), low(N, 0), pedge(N, -1), it(N, 0);
        int timer = 0;
        std::vector<int> st;
        st.push_back(0); disc[0] = low[0] = timer++;
        while (!st.empty()) {
            const int v = st.back();
            if (it[v] < (int)adj[v].size()) {
                const auto [w, e] = adj[v][it[v]++];
                if (e == pedge[v]) continue;
                if (disc[w] < 0) {
                    disc[w] = low[w] = timer++; pedge[w] = e; st.push_back(w);
                } else {
                    low[v] = std::min(low[v], disc[w]);
                }
            } else {
                st.pop_back();
                if (!st.empty()) {
                    const int u = st.back();
                    low[u] = std::min(low[u], low[v]);
                    if (low[v] > disc[u]) bridge[pedge[v]] = 1;
                }
            }
        }
    }
    for (int e = 0; e < B; ++e)
        if (is_rot(e) && !bridge[e])
            return fail("ligand.rotatable[" + std::to_string(e) + "]: rotatable bond lies in a ring");
    // ---- rigid fragments and root (D1.2, D1.3) ----
    DSU fr(N);
    for (int e = 0; e < B; ++e) if (!is_rot(e)) fr.join(l->bonds[2 * e], l->bonds[2 * e + 1]);
    std::vector<int> frag(N), fsize(N, 0);
    for (int a = 0; a < N; ++a) { frag[a] = fr.find(a); fsize[frag[a]]++; }   // representative = min atom
    int root_frag = frag[0];
    for (int a = 0; a < N; ++a)
        if (frag[a] == a && (fsize[a] > fsize[root_frag] || (fsize[a] == fsize[root_frag] && a < root_frag))) root_frag = a;
    const int root_atom = root_frag;
    // ---- BFS tree from the root: orient torsions, count rotatable bonds on the path ----
    std::vector<int> bpar(N, -2), rotdepth(N, 0);
    {
        std::vector<int> q{root_atom};
        bpar[root_atom] = -1;
        for (size_t h = 0; h < q.size(); ++h) {
            const int u = q[h];
            for (auto [w, e] : adj[u])
                if (bpar[w] == -2) { bpar[w] = u; rotdepth[w] = rotdepth[u] + (is_rot(e) ? 1 : 0); q.push_back(w); }
        }
    }
    std::vector<Tor> tors;
    for (int e = 0; e < B; ++e) {
        if (!is_rot(e)) continue;
        const int x = l->bonds[2 * e], y = l->bonds[2 * e + 1];
        Tor t;
        if (bpar[y] == x) { t.a = x; t.b = y; }
        else if (bpar[x] == y) { t.a = y; t.b = x; }
        else return fail("ligand.rotatable[" + std::to_string(e) + "]: not a tree edge (internal)");
        t.depth = rotdepth[t.b];
        tors.push_back(t);
    }
    std::sort(tors.begin(), tors.end(), [](const Tor &u, const Tor &v) {
        if (u.depth != v.depth) return u.depth < v.depth;
        if (u.a != v.a) return u.a < v.a;
        return u.b < v.b;
    });
    const int T = (int)tors.size();
    // ---- DFS preorder renumbering: subtree of b_k = far side of torsion k ----
    std::vector<int> pos(N, -1), sub(N, 0), order;
    {
        std::vector<std::pair<int, int>> st{{root_atom, 0}};
        pos[root_atom] = 0; order.push_back(root_atom);
        while (!st.empty()) {
            auto &[v, i] = st.back();
            if (i < (int)adj[v].size()) {
                const int w = adj[v][i++].first;
                if (pos[w] < 0) { pos[w] = (int)order.size(); order.push_back(w); st.push_back({w, 0}); }
            } else {
                sub[v] = (int)order.size() - pos[v];
                st.pop_back();
            }
        }
    }
    std::vector<int> lo(T), hi(T), parent(T, -1);
    for (int k = 0; k < T; ++k) { lo[k] = pos[tors[k].b] + 1; hi[k] = pos[tors[k].b] + sub[tors[k].b]; }
    for (int k = 0; k < T; ++k) {
        const int pb = pos[tors[k].b];
        for (int j = 0; j < T; ++j)
            if (j != k && lo[j] <= pb && pb < hi[j] && (parent[k] < 0 || hi[j] - lo[j] < hi[parent[k]] - lo[parent[k]]))
                parent[k] = j;
        if (parent[k] >= 0 && tors[parent[k]].depth != tors[k].depth - 1)
            return fail("ligand: torsion tree inconsistent (internal)");
    }
    std::vector<int> deep(N, -1);   // indexed by dfs position
    for (int p = 0; p < N; ++p)
        for (int k = 0; k < T; ++k)
            if (lo[k] <= p && p < hi[k] && (deep[p] < 0 || hi[k] - lo[k] < hi[deep[p]] - lo[deep[p]])) deep[p] = k;
    // ---- pairs (D1.6): i < j, more than 3 bonds apart, different rigid fragments ----
    std::vector<int> pairs;
    {
        std::vector<int> mark(N, -1), depthv(N, 0);
        for (int i = 0; i < N; ++i) {
            std::vector<int> q{i};
            mark[i] = i; depthv[i] = 0;
            for (size_t h = 0; h < q.size(); ++h) {
                const int u = q[h];
                if (depthv[u] == 3) continue;
                for (auto [w, e] : adj[u]) { (void)e; if (mark[w] != i) { mark[w] = i; depthv[w] = depthv[u] + 1; q.push_back(w); } }
            }
            for (int j = i + 1; j < N; ++j)
                if (mark[j] != i && frag[i] != frag[j]) { pairs.push_back(i); pairs.push_back(j); }
        }
    }
    tp.tors = std::move(tors);
    tp.order = std::move(order); tp.pos = std::move(pos);
    tp.lo = std::move(lo); tp.hi = std::move(hi); tp.parent = std::move(parent);
    tp.deep = std::move(deep); tp.pairs = std::move(pairs);
    return DOCK_OK;
}

// Verbatim mode (D1.7): the caller's torsions and pairs, validated.
// The moved sets form a laminar family; a DFS over it (children in torsion order) gives
// every moved set one contiguous range, and parent(k) = the nearest earlier torsion whose
// moved set contains moved(k).
int verbatim_topology(const dock_ligand *l, Topo &tp, std::string *err) {
    auto fail = [&](const std::string &m) { *err = m; return (int)DOCK_E_INPUT; };
    const int N = l->n_atoms, T = l->n_tors;
    if (T > kMaxTors) return fail("ligand.n_tors: at most 32 torsions");
    if (l->n_pairs < 0) return fail("ligand.n_pairs: must be >= 0 with verbatim torsions (or both -1)");
    if (l->rotatable)
        for (int e = 0; e < l->n_bonds; ++e)
            if (l->rotatable[e])
                return fail("ligand.rotatable[" + std::to_string(e) +
                            "]: must be 0 with verbatim torsions (set n_tors = n_pairs = -1 to derive)");
    if (T > 0 && (!l->tors_axis || !l->tors_moved_off)) return fail("ligand.tors_axis/tors_moved_off: NULL");
    std::vector<std::vector<uint8_t>> in(T, std::vector<uint8_t>(N, 0));
    std::vector<int> size(T, 0);
    for (int k = 0; k < T; ++k) {
        const std::string tag = "ligand.torsion[" + std::to_string(k) + "]";
        const int a = l->tors_axis[2 * k], b = l->tors_axis[2 * k + 1];
        if (a < 0 || b < 0 || a >= N || b >= N) return fail(tag + ": axis atom out of range");
        if (a == b) return fail(tag + ": axis atoms equal");
        const int o0 = l->tors_moved_off[k], o1 = l->tors_moved_off[k + 1];
        if (o0 < 0 || o1 < o0 || (o1 > o0 && !l->tors_moved)) return fail(tag + ": bad tors_moved_off / NULL tors_moved");
        for (int q = o0; q < o1; ++q) {
            const int m = l->tors_moved[q];
            if (m < 0 || m >= N) return fail(tag + ": moved atom out of range");
            if (m == a || m == b) return fail(tag + ": moved set contains an axis atom (S:32)");
            if (in[k][m]) return fail(tag + ": duplicate moved atom " + std::to_string(m));
            in[k][m] = 1;
            ++size[k];
        }
    }
    // laminar family, outer sets first, axis consistency (DESIGN.md §3 reading D1.7)
    auto subset = [&](int x, int y) {   // moved(x) within moved(y)
        for (int m = 0; m < N; ++m) if (in[x][m] && !in[y][m]) return false;
        return true;
    };
    for (int k = 0; k < T; ++k)
        for (int j = k + 1; j < T; ++j) {
            const std::string tag = "ligand.torsion[" + std::to_string(j) + "] vs [" + std::to_string(k) + "]";
            bool meet = false;
            for (int m = 0; m < N && !meet; ++m) meet = in[k][m] && in[j][m];
            const bool j_in_k = subset(j, k), k_in_j = subset(k, j);
            if (meet && !j_in_k && !k_in_j) return fail(tag + ": moved sets neither nested nor disjoint");
            if (meet && k_in_j && !j_in_k) return fail(tag + ": a nested moved set must come after its parent");
            const int ak = l->tors_axis[2 * k], bk = l->tors_axis[2 * k + 1];
            if (in[j][ak] || in[j][bk]) return fail(tag + ": a later torsion moves an earlier torsion's axis");
            if (meet && j_in_k) {
                const int aj = l->tors_axis[2 * j], bj = l->tors_axis[2 * j + 1];
                auto carried = [&](int x) { return in[k][x] || x == ak || x == bk; };
                if (!carried(aj) || !carried(bj))
                    return fail(tag + ": the axis of a nested torsion must move with its parent");
            }
        }
    tp.tors.resize(T);
    tp.parent.assign(T, -1);
    for (int k = 0; k < T; ++k) {
        for (int j = k - 1; j >= 0; --j)      // nearest earlier superset (equal sets chain by index)
            if (size[j] > 0 && subset(k, j) && size[k] > 0 && (tp.parent[k] < 0 || size[j] < size[tp.parent[k]]))
                tp.parent[k] = j;
        tp.tors[k].a = l->tors_axis[2 * k];
        tp.tors[k].b = l->tors_axis[2 * k + 1];
        tp.tors[k].depth = tp.parent[k] < 0 ? 1 : tp.tors[tp.parent[k]].depth + 1;
    }
    // DFS layout: root atoms (in no moved set), then each top-level torsion's subtree: its own
    // atoms (in no child's set), then its children in torsion order
    std::vector<std::vector<int>> kids(T);
    std::vector<int> tops;
    for (int k = 0; k < T; ++k) (tp.parent[k] < 0 ? tops : kids[tp.parent[k]]).push_back(k);
    tp.order.clear();
    tp.lo.assign(T, 0); tp.hi.assign(T, 0);
    std::vector<uint8_t> placed(N, 0);
    auto in_any = [&](const std::vector<int> &ks, int m) { for (int k : ks) if (in[k][m]) return true; return false; };
    for (int m = 0; m < N; ++m)
        if (!in_any(tops, m)) { tp.order.push_back(m); placed[m] = 1; }
    std::vector<std::pair<int, int>> st;     // (torsion, 0 = enter / 1 = leave)
    for (int i = (int)tops.size() - 1; i >= 0; --i) st.push_back({tops[i], 0});
    while (!st.empty()) {
        const auto [k, phase] = st.back();
        st.pop_back();
        if (phase == 1) { tp.hi[k] = (int)tp.order.size(); continue; }
        tp.lo[k] = (int)tp.order.size();
        for (int m = 0; m < N; ++m)
            if (in[k][m] && !placed[m] && !in_any(kids[k], m)) { tp.order.push_back(m); placed[m] = 1; }
        st.push_back({k, 1});
        for (int i = (int)kids[k].size() - 1; i >= 0; --i) st.push_back({kids[k][i], 0});
    }
    if ((int)tp.order.size() != N) return fail("internal: verbatim DFS layout");
    tp.pos.assign(N, -1);
    for (int p = 0; p < N; ++p) tp.pos[tp.order[p]] = p;
    for (int k = 0; k < T; ++k) {
        if (tp.hi[k] - tp.lo[k] != size[k]) return fail("internal: moved set not contiguous");
        for (int p = tp.lo[k]; p < tp.hi[k]; ++p)
            if (!in[k][tp.order[p]]) return fail("internal: moved set not contiguous");
    }
    tp.deep.assign(N, -1);
    for (int p = 0; p < N; ++p)                 // innermost = the latest torsion containing it
        for (int k = 0; k < T; ++k)
            if (in[k][tp.order[p]]) tp.deep[p] = k;
    // pairs: as given, each normalised to i < j
    if (l->n_pairs > 0 && !l->pairs) return fail("ligand.pairs: NULL");
    std::vector<uint8_t> seen((size_t)N * N, 0);
    tp.pairs.clear();
    for (int q = 0; q < l->n_pairs; ++q) {
        int i = l->pairs[2 * q], j = l->pairs[2 * q + 1];
        const std::string tag = "ligand.pairs[" + std::to_string(q) + "]";
        if (i < 0 || j < 0 || i >= N || j >= N) return fail(tag + ": atom index out of range");
        if (i == j) return fail(tag + ": self pair");
        if (i > j) std::swap(i, j);
        if (seen[(size_t)i * N + j]) return fail(tag + ": duplicate pair");
        seen[(size_t)i * N + j] = 1;
        tp.pairs.push_back(i); tp.pairs.push_back(j);
    }
    return DOCK_OK;
}

int prepare_ligand(const dock_ligand *l, const dock_type_param *tp, int n_types, const Scoring &sf, Prepared *out,
                   std::string *err) {
    auto fail = [&](const std::string &m) { *err = m; return (int)DOCK_E_INPUT; };
    if (!l) return fail("ligand: NULL");
    const int N = l->n_atoms;
    if (N < 1 || N > kMaxAtoms) return fail("ligand.n_atoms: must be in 1..256");
    if (!l->type || !l->charge || !l->xyz) return fail("ligand.type/charge/xyz: NULL");
    if (l->n_bonds < 0 || (l->n_bonds > 0 && !l->bonds)) return fail("ligand.bonds: NULL or negative count");
    if (!tp || n_types < 1) return fail("type_params: NULL");
    for (int t = 0; t < n_types; ++t) {
        const dock_type_param &q = tp[t];
        if (!std::isfinite(q.R) || !std::isfinite(q.eps) || !std::isfinite(q.S) || !std::isfinite(q.V) ||
            q.R < 0.f || q.eps < 0.f || q.role < 0 || q.role > 2)
            return fail("type_params[" + std::to_string(t) + "]: non-finite, negative or bad role");
    }
    for (int a = 0; a < N; ++a) {
        if (l->type[a] < 0 || l->type[a] >= n_types)
            return fail("ligand.type[" + std::to_string(a) + "]: no grid map for this type");
        if (!std::isfinite(l->charge[a])) return fail("ligand.charge[" + std::to_string(a) + "]: non-finite");
        for (int d = 0; d < 3; ++d)
            if (!std::isfinite(l->xyz[3 * a + d])) return fail("ligand.xyz[" + std::to_string(a) + "]: non-finite");
    }
    Topo topo;
    if (l->n_tors >= 0 || l->n_pairs >= 0) {
        if (l->n_tors < 0) return fail("ligand.n_tors: must be >= 0 with verbatim pairs (or both -1)");
        if (int rc = verbatim_topology(l, topo, err)) return rc;
    } else {
        if (int rc = derive_topology(l, topo, err)) return rc;
    }
    const std::vector<Tor> &tors = topo.tors;
    const int T = (int)tors.size();
    const std::vector<int> &order = topo.order, &pos = topo.pos, &lo = topo.lo, &hi = topo.hi,
                           &parent = topo.parent, &deep = topo.deep, &pairs = topo.pairs;
    const int P = (int)pairs.size() / 2;
    if (P > 65535) return fail("ligand: more than 65535 intramolecular pairs");

    // ---- outputs in caller order ----
    Prepared &o = *out;
    o.N = N; o.T = T; o.G = 6 + T; o.P = P;
    o.tor_a.resize(T); o.tor_b.resize(T); o.tor_depth.resize(T);
    o.moved.assign((size_t)T * N, 0);
    for (int k = 0; k < T; ++k) {
        o.tor_a[k] = tors[k].a; o.tor_b[k] = tors[k].b; o.tor_depth[k] = tors[k].depth;
        for (int a = 0; a < N; ++a) o.moved[(size_t)k * N + a] = (pos[a] >= lo[k] && pos[a] < hi[k]) ? 1 : 0;
    }
    o.pairs = pairs;
    o.dfs2orig = order;
    o.orig2dfs = pos;

    // ---- the constant block (DFS numbering) ----
    LigDev &L = o.layout;
    std::memset(&L, 0, sizeof(L));
    L.N = N; L.T = T; L.G = 6 + T; L.P = P;
    // scoring function (NEXT-2): D5-AD4 folds its weights and charge-dependent solvation
    // into the pair constants below; the tile kernels get the vdW / H-bond factors here.
    const bool ad4 = sf.sf == DOCK_SF_AD4;
    L.sf = ad4 ? 1 : 0;
    L.wA_v = (float)sf.w_vdw; L.wB_v = (float)(2.0 * sf.w_vdw);
    L.wA_h = (float)(5.0 * sf.w_hb); L.wB_h = (float)(-6.0 * sf.w_hb);
    L.qscale = (float)(sf.w_el * 332.06363);
    // D5-AD4 solvation parameter S' = S + qasp |q| and weighted volume V' = w_ds V of atom a
    auto S_of = [&](int a) { const double S = tp[l->type[a]].S; return ad4 ? S + sf.qasp * std::fabs((double)l->charge[a]) : S; };
    auto V_of = [&](int a) { const double V = tp[l->type[a]].V; return ad4 ? sf.w_ds * V : V; };
    int off = 0;
    L.off_tlane = off; off += 4 * 32;
    L.off_p = off; off += 16 * N;
    L.off_par = off; off += 16 * N;
    L.off_meta = off; off += a16(4 * N);
    L.off_tA = off; off += 16 * T;
    L.off_tU = off; off += 16 * T;
    L.off_tmeta = off; off += 16 * T;
    L.NW = (N + 31) / 32;
    L.off_mask = off; off += a16(4 * N * L.NW);
    L.Wg = N <= 16 ? 16 : 32;
    L.NC = (N + L.Wg - 1) / L.Wg;
    L.off_ppar = off; off += 16 * L.NC * 2 * L.Wg;
    // tile schedule of the gradient path (must match score.cuh intra_tiles)
    const int Wg = L.Wg, Bf = N / Wg, tail = N - Bf * Wg;
    // Partial last chunk (tail of t atoms), three schedules (score.cuh), by a cost model in
    // pair evaluations (~40 instructions each) and shuffles:
    //   rot:  a padded rotated chunk: W/2 + Bf*W steps;
    //   bcast: every lane meets tail atom k at once, k = 0..t-1: t*(Bf+1) evaluations + 3 sums each;
    //   seg (slot mode only): the tail padded to tp = 2^ceil(log2 t) <= W/2, rotated inside
    //     W/tp lane segments: Bf*tp steps against the full chunks, then the tail x tail
    //     steps 1..tp/2 shared round-robin by the segments, and a butterfly over segments.
    L.tail_seg = 0;
    L.tail_rot = (tail > 0 && (Wg / 2 + Bf * Wg) * 40 < tail * ((Bf + 1) * 40 + 3 * 5)) ? 1 : 0;
    // 49 <= N <= 63 (no segment form for a tail of 17..31): the tail as a padded rotated
    // chunk, so the packed FP32x2 tiles (two chunks, the second padded) can take the ligand
#if (!defined(DK_PACKED) || DK_PACKED) && (!defined(DK_FOLD) || DK_FOLD)
    if (!ad4 && Wg == 32 && Bf == 1 && tail > Wg / 2) L.tail_rot = 1;
#endif
    int tpw = 1;   // segment width
    while (tpw < tail) tpw <<= 1;
    const int seg_rounds = (tpw / 2 + (Wg / tpw) - 1) / (Wg / tpw);
    auto seg_lg = [&]() { int l = 0; for (int m = tpw; m < Wg; m <<= 1) ++l; return l; };
    if (tail > 0 && tpw <= Wg / 2) {
        // (per-evaluation weights from the A/B in profiles/r01r: 3ce3 seg 1.11x, 7cpa bcast 1.04x)
        const int c_seg = (Bf * tpw + seg_rounds) * 46 + (tpw + seg_rounds) * 6 + 6 * seg_lg();
        const int c_rot = (Wg / 2 + Bf * Wg) * 40;
        const int c_bc = tail * ((Bf + 1) * 40 + 3 * 5);
        int lg = 0;
        while ((1 << lg) < tpw) ++lg;
        // hyb (slot mode only, needs full chunks): the full chunks x tail part by broadcast
        // (t*Bf evaluations + 3 sums per tail atom), the tail x tail part by the segment rounds
        const int c_hyb = tail * (Bf * 40 + 3 * 5) + seg_rounds * 46 + 6 * seg_lg();
        bool use_seg = c_seg < c_rot && c_seg < c_bc && c_seg <= c_hyb;
        bool use_hyb = !use_seg && Bf > 0 && c_hyb < c_rot && c_hyb < c_bc;
        if (const char *f = std::getenv("DOCK_TAIL")) {   // A/B experiments and the schedule tests
            if (std::strcmp(f, "seg") == 0) { use_seg = true; use_hyb = false; }
            else if (std::strcmp(f, "hyb") == 0) { use_seg = false; use_hyb = Bf > 0; }
            else if (std::strcmp(f, "bcast1") == 0 || std::strcmp(f, "bcast") == 0) { use_seg = false; use_hyb = false; }
        }
        if (use_seg || use_hyb) {
            L.tail_seg = tpw | (lg << 8) | (seg_rounds << 16) | (use_hyb ? 1 << 24 : 0);
            L.tail_rot = 0;
        }
    }
    const bool hyb = (L.tail_seg >> 24) & 1;
    auto slot_count = [&]() {
        const int Bt_ = Bf + L.tail_rot;
        const int steps = Bt_ * (Wg / 2) + (Bt_ * (Bt_ - 1) / 2) * Wg;
        int extra = 0;
        if (tail > 0 && !L.tail_rot)
            extra = L.tail_seg ? ((hyb ? tail * Bf : Bf * tpw) + seg_rounds) * Wg : tail * (Bf + 1) * Wg;
        return steps * Wg + extra;
    };
    L.n_slots = slot_count();
    L.slot_mode = (20 * L.n_slots <= 64 * 1024) ? 1 : 0;      // beyond: per-atom params + bits
    // Packed FP32x2 tiles (score.cuh tiles_packed, D5 only): W = 32, two full chunks and a
    // hybrid tail (65 <= N <= 96).  The H-bond pairs of the packed rows (all but tail x tail)
    // go to a side list (their 12-10 vdW terms) whose forces and per-atom totals are staged in
    // the per-group gradient scratch (2N float4): nhb + N <= 2N, and an atom's contributions
    // must fit one 32-lane round of the per-atom sums.
    std::vector<int> hbl;   // dfs positions i < j, in pair-list order
    for (size_t q = 0; q + 1 < pairs.size(); q += 2) {
        const int ri = tp[l->type[pairs[q]]].role, rj = tp[l->type[pairs[q + 1]]].role;
        if ((ri == 1 && rj == 2) || (ri == 2 && rj == 1)) {
            const int di = pos[pairs[q]], dj = pos[pairs[q + 1]];
            if (!L.tail_rot && std::min(di, dj) >= Bf * Wg) continue;   // tail x tail: folded rounds
            hbl.push_back(std::min(di, dj)); hbl.push_back(std::max(di, dj));
        }
    }
    const int nhb = (int)hbl.size() / 2;
    std::vector<int> hdeg(N, 0);
    for (int v : hbl) hdeg[v]++;
    const int hmax = N > 0 ? *std::max_element(hdeg.begin(), hdeg.end()) : 0;
#if (!defined(DK_PACKED) || DK_PACKED) && (!defined(DK_FOLD) || DK_FOLD)
    // two full chunks and a hybrid tail (65 <= N <= ~82), or two chunks with no tail or the
    // second one a padded rotated chunk (49 <= N <= 64; padded slots hold zero constants)
    const bool two_hyb = Bf == 2 && tail > 0 && !L.tail_rot && ((L.tail_seg >> 24) & 1);
    const bool two_rot = (Bf == 2 && tail == 0) || (Bf == 1 && L.tail_rot);
    L.packed = (!ad4 && L.slot_mode && Wg == 32 && (two_hyb || two_rot) &&
                nhb <= N && hmax <= 32 && 6 + T <= 32) ? 1 : 0;   // G <= 32: one gene per lane (k_ls_adadelta PK)
#endif
    if (!L.slot_mode && L.tail_seg) {                          // seg needs the slot tables
        L.tail_seg = 0;
        L.tail_rot = (tail > 0 && (Wg / 2 + Bf * Wg) * 40 < tail * ((Bf + 1) * 40 + 3 * 5)) ? 1 : 0;
        L.n_slots = slot_count();
    }
    const int Bt = Bf + L.tail_rot;
    L.off_slot4 = off; off += L.slot_mode ? 16 * L.n_slots : 0;
#if defined(DK_FOLD) && !DK_FOLD
    const bool sep_q = true;                   // A/B build: the unfolded {r_eq^2, A, B, SV} + qq tables
#else
    const bool sep_q = ad4;                    // D5 folds qq into slot4
#endif
    L.off_slotq = off; off += (L.slot_mode && sep_q) ? a16(4 * L.n_slots) : 0;
    // H-bond contribution rounds: atoms in dfs order, each atom's 2..32 contributions kept in one round
    std::vector<int> hseg;          // [rounds][32] entries (score.cuh hb_side)
    if (L.packed) {
        std::vector<std::vector<int>> inc(N);
        for (int h = 0; h < nhb; ++h) { inc[hbl[2 * h]].push_back(h); inc[hbl[2 * h + 1]].push_back(h | 0x100); }
        int lane = 32;
        for (int a = 0; a < N; ++a) {
            const int d = (int)inc[a].size();
            if (d == 0) continue;
            if (lane + d > 32) { hseg.insert(hseg.end(), 32, 0); lane = 0; }
            const int base = (int)hseg.size() - 32, first = lane;
            for (int k = 0; k < d; ++k, ++lane)
                hseg[base + lane] = inc[a][k] | (first << 9) | ((k == d - 1) ? 1 << 14 : 0) | (1 << 15) | (a << 16);
        }
    }
    L.nhb = L.packed ? nhb : 0;
    L.nhbr = (int)hseg.size() / 32;
    L.hbspan = 1;
    while (L.packed && L.hbspan < hmax) L.hbspan <<= 1;
    L.off_hbc = off; off += 16 * L.nhb;
    L.off_hbseg = off; off += L.packed ? a16(4 * ((int)hseg.size() + L.NC)) : 0;
    L.grad_bytes = off;             // the gradient kernels stage only up to here
    // Energy-only kernels stage the pair list + per-pair constants (20 B per pair) when it
    // fits comfortably in shared memory; beyond that (P > ~4,900, e.g. N >= ~110) they use
    // the pair tiles like the gradient kernels, and the list is not stored at all.
    L.energy_tiles = (20 * P > 96 * 1024) ? 1 : 0;
    if (L.energy_tiles && N <= 96) return fail("internal: energy tiles need N > 96");   // see score.cuh
    const int Ps = L.energy_tiles ? 0 : P;
    L.off_pairs = off; off += a16(4 * Ps);
    L.off_pprm = off; off += 16 * Ps;
    L.blob_bytes = a16(off);
    o.blob.assign(L.blob_bytes, 0);
    uint8_t *bl = o.blob.data();
    // levels: torsions are sorted by depth, depth 1..D all present
    int n_levels = 0;
    for (int k = 0; k < T; ++k) n_levels = std::max(n_levels, tors[k].depth);
    L.n_levels = n_levels;
    for (int d = 0; d <= kMaxTors; ++d) {
        int s = 0;
        while (s < T && tors[s].depth <= d) ++s;   // first torsion with depth > d
        L.lvl_start[d] = s;
    }
    // torsion-gradient lane blocks (score.cuh a6): every torsion gets a power-of-two block of
    // lanes; starting from one lane each, the block of the torsion with the longest walk
    // ceil(len / size) is doubled while the blocks fit the Wg lanes.  Blocks are placed
    // largest first, so each is aligned to its size (the butterfly stays inside it).
    {
        std::vector<int> bsz(T, 1);
        int used = T;
        for (;;) {
            int kmax = -1, wmax = 0;
            for (int k = 0; k < T; ++k) {
                const int w = (hi[k] - lo[k] + bsz[k] - 1) / bsz[k];
                if (w > wmax) { wmax = w; kmax = k; }
            }
            if (kmax < 0 || wmax <= 1 || used + bsz[kmax] > Wg || 2 * bsz[kmax] > Wg) break;
            used += bsz[kmax];
            bsz[kmax] *= 2;
        }
        std::vector<int> byb(T);
        std::iota(byb.begin(), byb.end(), 0);
        std::stable_sort(byb.begin(), byb.end(), [&](int x, int y) { return bsz[x] > bsz[y]; });
        int *tl = reinterpret_cast<int *>(bl + L.off_tlane);
        for (int q = 0; q < 32; ++q) tl[q] = 255;
        int pos0 = 0, top = 1;
        for (int k : byb) {
            int lg = 0;
            while ((1 << lg) < bsz[k]) ++lg;
            for (int i = 0; i < bsz[k]; ++i) tl[pos0 + i] = k | (i << 8) | (lg << 16);
            pos0 += bsz[k];
            top = std::max(top, bsz[k]);
        }
        if (pos0 > Wg) return fail("internal: torsion lane blocks");
        L.tlane_top = top / 2;
    }
    // body frame: c = centroid of the reference coordinates, computed in double (D1.8)
    double c[3] = {0, 0, 0};
    for (int a = 0; a < N; ++a) for (int d = 0; d < 3; ++d) c[d] += l->xyz[3 * a + d];
    for (int d = 0; d < 3; ++d) c[d] /= N;
    auto pref = [&](int a, int d) { return (double)l->xyz[3 * a + d] - c[d]; };
    auto role_of = [&](int a) { return tp[l->type[a]].role; };
    float4 *bp = reinterpret_cast<float4 *>(bl + L.off_p);
    float4 *bprm = reinterpret_cast<float4 *>(bl + L.off_par);
    int *bmeta = reinterpret_cast<int *>(bl + L.off_meta);
    for (int p = 0; p < N; ++p) {
        const int a = order[p];
        const dock_type_param &q = tp[l->type[a]];
        bp[p] = make_float4((float)pref(a, 0), (float)pref(a, 1), (float)pref(a, 2), l->charge[a]);
        bprm[p] = make_float4(0.5f * q.R, (float)std::sqrt((double)q.eps), q.S, q.V);
        bmeta[p] = (l->type[a] & 0xff) | ((q.role & 3) << 8) | ((deep[p] + 1) << 16);
    }
    float4 *tA = reinterpret_cast<float4 *>(bl + L.off_tA);
    float4 *tU = reinterpret_cast<float4 *>(bl + L.off_tU);
    int4 *tm = reinterpret_cast<int4 *>(bl + L.off_tmeta);
    for (int k = 0; k < T; ++k) {
        const int a = tors[k].a, b = tors[k].b;
        double u[3], n = 0;
        for (int d = 0; d < 3; ++d) { u[d] = pref(b, d) - pref(a, d); n += u[d] * u[d]; }
        n = std::sqrt(n);
        if (!(n > 0)) return fail("ligand.xyz: zero-length rotatable bond " + std::to_string(a) + "-" + std::to_string(b));
        tA[k] = make_float4((float)pref(a, 0), (float)pref(a, 1), (float)pref(a, 2), 0.f);
        tU[k] = make_float4((float)(u[0] / n), (float)(u[1] / n), (float)(u[2] / n), 0.f);
        tm[k] = make_int4(parent[k], pos[a], pos[b], lo[k] | (hi[k] << 16));
    }
    // gradient-path tiles: chunk-duplicated partner params, H-bond role in the signs
    // (R/2 < 0: acceptor, sqrt(eps) < 0: donor; D5)
    {
        float4 *pp = reinterpret_cast<float4 *>(bl + L.off_ppar);
        for (int c = 0; c < L.NC; ++c)
            for (int q = 0; q < 2 * L.Wg; ++q) {
                const int p = c * L.Wg + (q % L.Wg);
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (p < N) {
                    const dock_type_param &t = tp[l->type[order[p]]];
                    const float h = 0.5f * t.R, e = (float)std::sqrt((double)t.eps);
                    v = make_float4(t.role == 2 ? -h : h, t.role == 1 ? -e : e, t.S, t.V);
                    if (ad4) { v.z = (float)S_of(order[p]); v.w = (float)V_of(order[p]); }
                }
                pp[c * 2 * L.Wg + q] = v;
            }
    }
    auto hb_of = [&](int i, int j) {
        const int ri = role_of(i), rj = role_of(j);
        return (ri == 1 && rj == 2) || (ri == 2 && rj == 1);
    };
    if (L.slot_mode) {
        // pair-slot tables in the exact order intra_tiles visits them (DFS positions)
        std::vector<uint8_t> is_pair((size_t)N * N, 0);
        for (size_t q = 0; q + 1 < pairs.size(); q += 2) {
            const int di = pos[pairs[q]], dj = pos[pairs[q + 1]];
            is_pair[(size_t)di * N + dj] = is_pair[(size_t)dj * N + di] = 1;
        }
        float4 *s4 = reinterpret_cast<float4 *>(bl + L.off_slot4);
        float *sq = reinterpret_cast<float *>(bl + L.off_slotq);
        auto fill = [&](int slot, int da, int db, bool on, bool lean = false) {
            // a non-pair slot contributes exactly 0 (A = B = SV = qq = 0); under D5-AD4 its
            // r_eq operand is 1 Å so the smoothed distance stays >= 0.26 Å (x^2 finite, 0 * x^12 = 0)
            s4[slot] = make_float4(ad4 ? 1.f : 0.f, 0.f, 0.f, 0.f);
            if (sep_q) sq[slot] = 0.f;
            if (!on || da >= N || db >= N || !is_pair[(size_t)da * N + db]) return;
            const int ia = order[da], ib = order[db];
            const dock_type_param &ta = tp[l->type[ia]], &tb = tp[l->type[ib]];
            const double req = 0.5 * ((double)ta.R + (double)tb.R);
            const double eps = std::sqrt((double)ta.eps * (double)tb.eps);
            const bool hb = hb_of(ia, ib);
            if (ad4) {   // {r_eq, w A, w B, w_ds (S'_a V_b + S'_b V_a)}, w_el 332.06363 q_a q_b
                s4[slot] = make_float4((float)req, (float)((hb ? 5.0 * sf.w_hb : sf.w_vdw) * eps),
                                       hb ? -(float)(6.0 * sf.w_hb * eps) : (float)(2.0 * sf.w_vdw * eps),
                                       (float)(S_of(ia) * V_of(ib) + S_of(ib) * V_of(ia)));
                sq[slot] = (float)(sf.w_el * 332.06363 * (double)l->charge[ia] * (double)l->charge[ib]);
                return;
            }
#if defined(DK_FOLD) && !DK_FOLD
            s4[slot] = make_float4((float)(req * req), (float)((hb ? 5.0 : 1.0) * eps),
                                   hb ? -(float)(6.0 * eps) : (float)(2.0 * eps),
                                   (float)((double)ta.S * tb.V + (double)tb.S * ta.V));
            sq[slot] = (float)(332.06363 / 4.0 * (double)l->charge[ia] * (double)l->charge[ib]);
            return;
#endif
            const double req2 = req * req, r6 = req2 * req2 * req2, r12 = r6 * r6;
            if (lean) {
                // D5, lean (the packed rows, score.cuh slot_pair2): {-eps r_eq^12, 2 eps r_eq^6,
                // -(S_aV_b + S_bV_a) / (3 * 2 sigma^2), -(332.06363/4) q_a q_b / 3}; the H-bond
                // pair's 12-10 vdW lives in the side list (zero vdW constants here)
                const double sv = (double)ta.S * tb.V + (double)tb.S * ta.V;
                const double qq = 332.06363 / 4.0 * (double)l->charge[ia] * (double)l->charge[ib];
                s4[slot] = make_float4(hb ? 0.f : -(float)(eps * r12), hb ? 0.f : (float)(2.0 * eps * r6),
                                       (float)(-sv / (3.0 * 2.0 * 3.6 * 3.6)), (float)(-qq / 3.0));
                return;
            }
            // D5, folded (score.cuh pair_eg_folded): {A r_eq^12, +-|B| r_eq^n (n = 10: negative),
            // S_aV_b + S_bV_a, 332.06363/4 q_a q_b}, in double then rounded once
            s4[slot] = make_float4((float)((hb ? 5.0 : 1.0) * eps * r12),
                                   hb ? -(float)(6.0 * eps * r6 * req2 * req2) : (float)(2.0 * eps * r6),
                                   (float)((double)ta.S * tb.V + (double)tb.S * ta.V),
                                   (float)(332.06363 / 4.0 * (double)l->charge[ia] * (double)l->charge[ib]));
        };
        int slot = 0;
        if (L.packed) {
            // packed order (score.cuh tiles_packed): per packed step two rows of Wg float4,
            // {c_a.x, c_b.x, c_a.y, c_b.y} and {c_a.z, c_b.z, c_a.w, c_b.w}, from the lean
            // constants c_a, c_b of its two slots (computed by fill into a scratch slot)
            auto emit2 = [&](int da, int db, bool on_a, int ea, int eb, bool on_b) {
                fill(slot, da, db, on_a, true);
                const float4 a = s4[slot];
                fill(slot, ea, eb, on_b, true);
                const float4 b = s4[slot];
                return std::make_pair(make_float4(a.x, b.x, a.y, b.y), make_float4(a.z, b.z, a.w, b.w));
            };
            auto put = [&](const std::vector<std::pair<float4, float4>> &row) {
                for (int ln = 0; ln < Wg; ++ln) s4[slot + ln] = row[ln].first;
                for (int ln = 0; ln < Wg; ++ln) s4[slot + Wg + ln] = row[ln].second;
                slot += 2 * Wg;
            };
            std::vector<std::pair<float4, float4>> row(Wg);
            for (int st = 1; st <= Wg / 2; ++st) {          // (a) tiles (0,0) and (1,1), step st
                for (int ln = 0; ln < Wg; ++ln) {
                    const bool once = !(st == Wg / 2 && ln >= Wg / 2);
                    const int p = (ln + st) & (Wg - 1);
                    row[ln] = emit2(ln, p, once, Wg + ln, Wg + p, once);
                }
                put(row);
            }
            for (int u = 0; u < Wg / 2; ++u) {              // (b) tile (0,1), steps u and u + 16
                for (int ln = 0; ln < Wg; ++ln)
                    row[ln] = emit2(ln, Wg + ((ln + u) & (Wg - 1)), true, ln, Wg + ((ln + u + Wg / 2) & (Wg - 1)), true);
                put(row);
            }
            for (int k = 0; k < tail && !L.tail_rot; ++k) { // (c) tail atom k vs chunks 0 and 1 (hybrid tail)
                for (int ln = 0; ln < Wg; ++ln) row[ln] = emit2(ln, 2 * Wg + k, true, Wg + ln, 2 * Wg + k, true);
                put(row);
            }
        }
        for (int I = 0; I < Bt && !L.packed; ++I)
            for (int J = I; J < Bt; ++J) {
                const int s0 = (I == J) ? 1 : 0, s1 = (I == J) ? Wg / 2 : Wg - 1;
                for (int st = s0; st <= s1; ++st)
                    for (int ln = 0; ln < Wg; ++ln, ++slot) {
                        const bool once = !(I == J && st == Wg / 2 && ln >= Wg / 2);
                        fill(slot, I * Wg + ln, J * Wg + ((ln + st) & (Wg - 1)), once);
                    }
            }
        if (L.packed) {
            // (the hybrid tail's broadcast part is in the packed rows above)
        } else if (tail > 0 && L.tail_seg && hyb) {
            // hyb, own chunks x tail by broadcast: tail atom k, chunk I, lane ln -> atom I*Wg + ln
            for (int k = 0; k < tail; ++k)
                for (int I = 0; I < Bf; ++I)
                    for (int ln = 0; ln < Wg; ++ln, ++slot)
                        fill(slot, I * Wg + ln, Bf * Wg + k, true);
        } else if (tail > 0 && L.tail_seg) {
            // own chunks x tail: step s, chunk I, lane ln -> tail position ((ln mod tpw) + s) mod tpw
            for (int st = 0; st < tpw; ++st)
                for (int I = 0; I < Bf; ++I)
                    for (int ln = 0; ln < Wg; ++ln, ++slot) {
                        const int k = ((ln & (tpw - 1)) + st) & (tpw - 1);
                        fill(slot, I * Wg + ln, Bf * Wg + k, k < tail);
                    }
        }
        if (tail > 0 && L.tail_seg) {
            // tail x tail: round r, segment g = ln / tpw takes step 1 + g + r * (Wg / tpw)
            for (int r = 0; r < seg_rounds; ++r)
                for (int ln = 0; ln < Wg; ++ln, ++slot) {
                    const int sl = ln & (tpw - 1), st = 1 + ln / tpw + r * (Wg / tpw);
                    const int k = (sl + st) & (tpw - 1);
                    const bool once = st < tpw / 2 || (st == tpw / 2 && sl < tpw / 2);
                    fill(slot, Bf * Wg + sl, Bf * Wg + k, once && sl < tail && k < tail);
                }
        } else if (tail > 0 && !L.tail_rot)
            for (int k = 0; k < tail; ++k)
                for (int I = 0; I <= Bf; ++I)
                    for (int ln = 0; ln < Wg; ++ln, ++slot)
                        fill(slot, I * Wg + ln, Bf * Wg + k, I < Bf || ln < k);
        if (slot != L.n_slots) return fail("internal: pair-slot count mismatch");
        if (L.packed) {
            // H-bond side list {5 eps r_eq^12, 6 eps r_eq^10, i | j << 16}, the contribution
            // rounds and the per-chunk lane masks of atoms with contributions
            float4 *hc = reinterpret_cast<float4 *>(bl + L.off_hbc);
            int *hs = reinterpret_cast<int *>(bl + L.off_hbseg);
            for (int h = 0; h < L.nhb; ++h) {
                const int di = hbl[2 * h], dj = hbl[2 * h + 1];
                const dock_type_param &ta = tp[l->type[order[di]]], &tb = tp[l->type[order[dj]]];
                const double req = 0.5 * ((double)ta.R + (double)tb.R);
                const double eps = std::sqrt((double)ta.eps * (double)tb.eps);
                const double req2 = req * req, r10 = req2 * req2 * req2 * req2 * req2;
                const uint32_t ij = (uint32_t)di | ((uint32_t)dj << 16);
                float fij;
                std::memcpy(&fij, &ij, 4);
                hc[h] = make_float4((float)(5.0 * eps * r10 * req2), (float)(6.0 * eps * r10), fij, 0.f);
            }
            for (size_t k = 0; k < hseg.size(); ++k) hs[k] = hseg[k];
            for (int c = 0; c < L.NC; ++c) {
                uint32_t m = 0;
                for (int ln = 0; ln < Wg; ++ln) {
                    const int a = c * Wg + ln;
                    if (a < N && hdeg[a] > 0) m |= 1u << ln;
                }
                hs[hseg.size() + c] = (int)m;
            }
        }
        if (std::getenv("DOCK_SLOT_STATS")) {   // diagnostics: steps (W slots) holding no pair at all
            const float4 *s4c = reinterpret_cast<const float4 *>(bl + L.off_slot4);
            int empty = 0, steps = L.n_slots / Wg, real = 0;
            for (int st = 0; st < steps; ++st) {
                bool any = false;
                for (int ln = 0; ln < Wg; ++ln) {
                    const float4 v = s4c[st * Wg + ln];
                    if (v.x != 0.f || v.y != 0.f || v.z != 0.f || v.w != 0.f || (sep_q && sq[st * Wg + ln] != 0.f)) { any = true; ++real; }
                }
                if (!any) ++empty;
            }
            std::fprintf(stderr, "[slots] N %d P %d steps %d empty %d real-slots %d of %d\n", N, P, steps, empty, real,
                         L.n_slots);
        }
    }
    uint32_t *bpairs = reinterpret_cast<uint32_t *>(bl + L.off_pairs);
    float4 *pprm = reinterpret_cast<float4 *>(bl + L.off_pprm);
    uint32_t *bmask = reinterpret_cast<uint32_t *>(bl + L.off_mask);
    for (int q = 0; q < P; ++q) {
        const int i = pairs[2 * q], j = pairs[2 * q + 1];
        int di = pos[i], dj = pos[j];
        if (di > dj) std::swap(di, dj);
        bmask[di * L.NW + (dj >> 5)] |= 1u << (dj & 31);
        bmask[dj * L.NW + (di >> 5)] |= 1u << (di & 31);
        if (L.energy_tiles) continue;
        const int hb = hb_of(i, j) ? 1 : 0;
        // byte offsets of the two pose records (16 B each) in the pair list; the H-bond flag
        // is the sign bit of eps_ij in the pair constants
        bpairs[q] = (uint32_t)(16 * di) | ((uint32_t)(16 * dj) << 16);
        // D5 pair constants for the energy-only path
        const dock_type_param &ti = tp[l->type[i]], &tj = tp[l->type[j]];
        const double req = 0.5 * ((double)ti.R + (double)tj.R);
        const float eps_ij = (float)std::sqrt((double)ti.eps * (double)tj.eps);
        if (ad4) {   // {r_eq, +-w eps_ij, w_ds (S'_i V_j + S'_j V_i), w_el 332.06363 q_i q_j}
            const float we = (float)((hb ? sf.w_hb : sf.w_vdw) * std::sqrt((double)ti.eps * (double)tj.eps));
            pprm[q] = make_float4((float)req, hb ? -we : we, (float)(S_of(i) * V_of(j) + S_of(j) * V_of(i)),
                                  (float)(sf.w_el * 332.06363 * (double)l->charge[i] * (double)l->charge[j]));
            continue;
        }
        pprm[q] = make_float4((float)(req * req), hb ? -eps_ij : eps_ij,
                              (float)((double)ti.S * tj.V + (double)tj.S * ti.V),
                              (float)(332.06363 / 4.0 * (double)l->charge[i] * (double)l->charge[j]));
    }
    return DOCK_OK;
}

int resolve_type_params(const dock_grids *g, const dock_type_param *tp, std::vector<dock_type_param> *out,
                        std::string *err) {
    auto fail = [&](const std::string &m) { *err = m; return (int)DOCK_E_INPUT; };
    if (!g) return fail("grids: NULL");
    if (g->n_types < 1 || g->n_types > 16) return fail("grids.n_types: must be in 1..16");
    std::vector<std::string> names;
    if (g->type_names) {
        for (int t = 0; t < g->n_types; ++t) {
            const char *nm = g->type_names[t];
            const size_t len = strnlen(nm, 4);
            if (len == 0 || len == 4) return fail("grids.type_names[" + std::to_string(t) + "]: empty or not NUL-terminated");
            for (const auto &o : names)
                if (o == std::string(nm, len)) return fail("grids.type_names[" + std::to_string(t) + "]: duplicate '" + o + "'");
            names.emplace_back(nm, len);
        }
    }
    out->assign(g->n_types, dock_type_param{});
    if (tp) {
        std::copy(tp, tp + g->n_types, out->begin());
        return DOCK_OK;
    }
    if (!g->type_names) return fail("type_params: NULL needs grids.type_names (the built-in table is by name)");
    for (int t = 0; t < g->n_types; ++t)
        if (dock_builtin_type_param(names[t].c_str(), &(*out)[t]) != DOCK_OK)
            return fail("grids.type_names[" + std::to_string(t) + "]: no built-in parameters for '" + names[t] + "'");
    return DOCK_OK;
}

int pack_grid(const dock_grids *g, std::vector<float4> *packed, std::string *err) {
    auto fail = [&](const std::string &m) { *err = m; return (int)DOCK_E_INPUT; };
    if (!g) return fail("grids: NULL");
    if (g->nx < 2 || g->ny < 2 || g->nz < 2) return fail("grids.nx/ny/nz: each must be >= 2");
    if (!(g->spacing > 0.f) || !std::isfinite(g->spacing)) return fail("grids.spacing: must be finite and > 0");
    for (int d = 0; d < 3; ++d) if (!std::isfinite(g->origin[d])) return fail("grids.origin: non-finite");
    if (g->n_types < 1 || g->n_types > 16) return fail("grids.n_types: must be in 1..16");
    if (!g->maps) return fail("grids.maps: NULL");
    const size_t n3 = (size_t)g->nx * g->ny * g->nz;
    const size_t total = n3 * (size_t)(g->n_types + 2);
    for (size_t i = 0; i < total; ++i)
        if (!std::isfinite(g->maps[i]))
            return fail("grids.maps[" + std::to_string(i / n3) + "][" + std::to_string(i % n3) + "]: non-finite");
    packed->resize(n3 * g->n_types);
    const float *E = g->maps + n3 * g->n_types, *D = E + n3;
    for (int t = 0; t < g->n_types; ++t) {
        const float *M = g->maps + n3 * t;
        float4 *o = packed->data() + n3 * t;
        for (size_t i = 0; i < n3; ++i) o[i] = make_float4(M[i], E[i], D[i], 0.f);
    }
    return DOCK_OK;
}

}  // namespace dk
