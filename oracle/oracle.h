/*
 * oracle.h — CPU ORACLE for the LGA docking hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load this library.  The product path (libdock.so and the
 * paper_2203_02096_b200 package) never includes, links or calls it, and shares
 * no code, header, table or helper with it.
 *
 * Plain, slow, double-precision C written from the method statement:
 *   PAPER.md:64-66 (§II-A) — grid "reaction field", ligand particle model with
 *     self-interactions (H-bond, vdW, desolvation), GA with crossover and
 *     fitness selection, Lamarckian local search on a random sample each
 *     generation, Solis-Wets optimiser, independent runs of 150 individuals,
 *     degrees of freedom = translation + orientation + rotatable bonds;
 *   PAPER.md:92-101 (§IV-A, Listing 1) — sum_evals reduction over individuals;
 *   PAPER.md:135-136 (§IV-B) — torsion rotations applied in a fixed order;
 *   and, where the paper is silent, the readings D1-D11 of SURVEY.md §8(c),
 *   restated in DESIGN.md §3 (each function cites the reading it follows).
 *
 * Parity status of every function is listed in DESIGN.md §3.  The multi-
 * generation trajectory of or_dock_run is "parity unpinned" (chaotic after the
 * first near-tie, SURVEY.md §8(c) "Unpinned" (i)); its building blocks are each
 * pinned by tests/test_oracle_*.py.
 */
#ifndef DOCK_ORACLE_H
#define DOCK_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OR_MAX_ATOMS 256
#define OR_MAX_TORS 32
#define OR_MAX_GENES (6 + OR_MAX_TORS)

/* NEXT-2 (DESIGN.md §11 reading D5-AD4): the AutoDock4.1-
   calibrated form of the intramolecular pair energy.  SPEC S:219-223, 232 name what D5
   leaves out (sigmoidal dielectric, free-energy weights, smoothing, cutoffs, torsional
   entropy); the values are AutoDock 4.1's, passed in by the caller. */
typedef struct {
    double w_vdw, w_hb, w_el, w_ds, w_tors;  /* free-energy coefficients */
    double qasp;               /* charge-dependent solvation: S_i -> S_i + qasp |q_i| */
    double smooth;             /* vdW / H-bond smoothing window width (Å) */
    double cut_vdw;            /* vdW / H-bond terms only for r < cut_vdw (Å); <= 0: no cutoff */
    double cut_el;             /* electrostatic + desolvation only for r < cut_el; <= 0: none */
    int diel;                  /* 0: eps(r) = 4 r (D5); 1: Mehler-Solmajer sigmoid */
    double diel_A, diel_eps0, diel_lambda, diel_k;   /* eps(r) = A + B/(1 + k e^{-lambda B r}), B = eps0 - A */
    double sigma;              /* desolvation Gaussian width (Å) */
} or_scoring;

/* A docking problem: receptor grid + per-type parameters + preprocessed ligand. */
typedef struct {
    int nx, ny, nz;            /* grid nodes per axis */
    double spacing;            /* Å */
    double origin[3];          /* position of node (0,0,0) */
    int n_types;               /* maps: n_types type maps, then E, then D */
    const float *maps;         /* [(n_types+2)][nz][ny][nx], node (i,j,k) at i + nx*(j + ny*k) */
    const double *tR, *teps, *tS, *tV;   /* per-type R, eps, S, V [n_types] (D5) */
    const int *trole;          /* per-type H-bond role 0 none, 1 donor, 2 acceptor */
    int N;                     /* atoms */
    const int *type;           /* [N] index into the grid's type list */
    const double *q;           /* [N] charges */
    const double *X;           /* [N*3] reference coordinates */
    int T;                     /* torsions (D1 order) */
    const int *tor_a, *tor_b;  /* [T] axis atoms, a on the root side */
    const unsigned char *moved;/* [T*N] 1 if atom moves with torsion k */
    int P;                     /* intramolecular pairs */
    const int *pairs;          /* [P*2] */
    const or_scoring *sf;      /* NULL: D5; else the D5-AD4 variant (NEXT-2) */
} or_problem;

typedef struct {
    double p_tour, p_cross, p_mut, mut_trans, mut_angle;   /* D8 */
    int ls_method;             /* 0 ADADELTA, 1 Solis-Wets */
    double ls_rate;
    int ls_max_iters;
    double sw_rho, sw_rho_min, sw_expand, sw_contract;     /* D9 */
    int sw_cons_succ, sw_cons_fail;
    double ad_rho, ad_eps;     /* D10 */
    int max_generations;
} or_params;

/* ---- D2: Philox4x32-10 and the stream layout ---- */
void     or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
uint32_t or_word(uint64_t seed, uint32_t ligand_id, uint32_t purpose, uint32_t slot,
                 uint32_t gen, uint32_t run, uint32_t m);
double   or_u01(uint32_t w);
uint32_t or_below(uint32_t w, uint32_t n);

/* ---- D1: topology (brute force).  Returns 0 ok, 1 input error. ---- */
int or_topology(int N, int n_bonds, const int *bonds, const unsigned char *rotatable,
                int *T_out, int *tor_a, int *tor_b, unsigned char *moved /*[32*N]*/,
                int *depth /*[32]*/, int *P_out, int *pairs /*[cap*2]*/, int cap,
                int *frag /*[N] nullable*/);

/* ---- D1.7: verbatim torsions (axis [T*2], CSR moved sets) and pairs [P*2], validated.
   Outputs tor_a/tor_b [T], moved [T*N], pairs_out [P*2] (i < j, list order).  0 ok, 1 error. ---- */
int or_topology_verbatim(int N, int T, const int *axis, const int *moved_off, const int *moved_idx, int P,
                         const int *pairs_in, int *tor_a, int *tor_b, unsigned char *moved, int *pairs_out);

/* ---- D3: genotype -> pose ---- */
void or_pose(const or_problem *P, const double *genes, double *xyz);

/* ---- D4: intermolecular (per atom and total) ---- */
double or_inter_atom(const or_problem *P, int a, const double r[3], double grad[3]);
double or_inter(const or_problem *P, const double *xyz, double *grad /*[N*3] nullable*/);
/* ---- D5: intramolecular ---- */
double or_pair_energy(const or_problem *P, int i, int j, double rho2_in, double *dE_drho2);
double or_intra(const or_problem *P, const double *xyz, double *grad /*[N*3] nullable*/);
/* ---- NEXT-2: the AD4 pair energy, dielectric, kink margin and binding estimate ---- */
double or_pair_energy_ad4(const or_problem *P, int i, int j, double rho2_in, double *dE_drho2);
double or_dielectric(const or_scoring *s, double r, double *deps_dr /* nullable */);
/* smallest |r - k| over pairs and kinks k of the AD4 pair energy (r_eq +- smooth/2,
   cut_vdw, cut_el): where FP32 and double may sit on different sides (gradient jumps,
   or energy jumps at a cutoff).  1e300 for D5 problems. */
double or_kink_margin(const or_problem *P, const double *xyz);
/* AD4 binding estimate of a pose (unbound = bound model): E_inter + w_tors * T. */
double or_binding_dG(const or_problem *P, double e_inter);
/* ---- D6 + D7: total energy and genotype gradient ---- */
double or_energy(const or_problem *P, const double *genes, double *ggrad /*[G] nullable*/,
                 double *xyz /*[N*3] nullable*/, double *terms /*[2] inter,intra nullable*/);
/* D6 + D7 evaluated at GIVEN world coordinates xyz [N*3] of the genotype `genes` (the
   D7 back-projection uses genes' t, phi, theta, alpha and the given r_a).  With
   xyz = or_pose(genes) this is or_energy.  Parity use (DESIGN.md §3 reading 22b): the
   GPU's energy and gradient are compared with this function at the GPU's own FP32 pose,
   so the FP32 rounding of the pose itself (checked separately at |dr| <= 1e-4 Å) does
   not enter the energy comparison. */
double or_energy_at(const or_problem *P, const double *genes, const double *xyz, double *ggrad /*[G] nullable*/,
                    double *terms /*[2] nullable*/);
/* smallest distance, in grid units, of any atom coordinate to a cell/box face, and
   smallest |rho2 - 1e-4| over pairs (both used to flag boundary poses). */
void or_margins(const or_problem *P, const double *xyz, double *face_margin, double *clamp_margin);

/* ---- D8: GA pieces ---- */
int  or_elite(int pop, const double *E);
void or_ga_slot(const or_params *pp, uint64_t seed, uint32_t ligand_id, uint32_t run,
                uint32_t gen, uint32_t slot, int pop, int G, const double *old_genes,
                const double *old_E, double *child, int *dbg /*[8] nullable*/);
int  or_n_ls(double ls_rate, int pop);
void or_ls_pick(uint64_t seed, uint32_t ligand_id, uint32_t run, uint32_t gen, int pop,
                int n_ls, int *perm /*[pop]*/);

/* ---- D9 / D10: local search.  objective: P != NULL -> docking energy of P,
   else the bowl sum_j bowl[j] * x_j^2 (test objective for SPEC S:304 pins). ---- */
void or_solis_wets(const or_problem *P, const double *bowl, int G, const or_params *pp,
                   uint64_t seed, uint32_t ligand_id, uint32_t run, uint32_t gen, uint32_t slot,
                   double *x, double *E, int64_t *evals);
void or_adadelta(const or_problem *P, const double *bowl, int G, const or_params *pp,
                 int iters, double *x, double *E, int64_t *evals);

/* The same D9 / D10 searches with traces (parity protocol):
   Solis-Wets: Etab [iters*2] nullable -- "fed" mode: the energy of candidate c (0 = x+b+d,
   1 = x-b-d) of iteration it is Etab[2 it + c] instead of an evaluation, so the D9 state
   machine can be compared with the GPU's on identical energies; trace_o [iters] outcome
   per iteration (0 / 1 accepted candidate, 2 both rejected, -1 not executed: rho < rho_min),
   trace_rho [iters] the rho used, trace_E [iters*3] = {E_x before, E(x+b+d), E(x-b-d) or NaN}.
   ADADELTA: fed [iters*(G+1)] nullable -- fed mode: iteration it's energy and gradient are
   (fed[it*(G+1)], fed[it*(G+1)+1 ..]) instead of an evaluation (the D10 update and best
   tracking on identical inputs); trace_x [iters*G] the point evaluated at iteration it,
   trace_E [iters] its energy, trace_g [iters*G] its gradient.
   Every trace pointer may be NULL. */
void or_solis_wets_traced(const or_problem *P, const double *bowl, int G, const or_params *pp,
                          uint64_t seed, uint32_t ligand_id, uint32_t run, uint32_t gen, uint32_t slot,
                          double *x, double *E, int64_t *evals, const double *Etab,
                          int *trace_o, double *trace_rho, double *trace_E);
void or_adadelta_traced(const or_problem *P, const double *bowl, int G, const or_params *pp,
                        int iters, double *x, double *E, int64_t *evals, const double *fed,
                        double *trace_x, double *trace_E, double *trace_g);

/* ---- D8 generation 0 of one run: genes [pop*G], energies [pop] (nullable) ---- */
void or_init_population(const or_problem *P, int pop, uint64_t seed, uint32_t ligand_id, uint32_t run,
                        double *genes, double *E);

/* ---- D8 + D11: one full run ---- */
int or_dock_run(const or_problem *P, const or_params *pp, int pop, int64_t max_evals,
                uint64_t seed, uint32_t ligand_id, uint32_t run,
                double *best_E, double *best_genes, int64_t *evals_used, int *generations,
                double *final_E /*[pop] nullable*/);

/* ---- NEXT-3: RMSD clustering of per-run best poses ----
   Poses sorted by energy (ascending; NaN last; ties -> lower index).  The first pose
   seeds cluster 0; each next pose joins the lowest-numbered cluster whose seed is within
   rmsd_tol (plain RMSD over the N atoms, no superposition: all poses share the receptor
   frame), else seeds a new cluster.  Outputs per pose: cluster id, RMSD to its cluster's
   seed (0 for a seed), rank in the energy order.  Returns the number of clusters. */
int or_cluster(int n, int N, const double *xyz /*[n*N*3]*/, const double *E /*[n]*/, double rmsd_tol,
               int *cluster /*[n]*/, double *rmsd_to_seed /*[n]*/, int *rank /*[n] nullable*/);
double or_rmsd(int N, const double *a, const double *b);

/* D11 / Listing 1: sum of per-individual evaluation counters. */
int64_t or_sum_evals(int n, const int64_t *counters);

#ifdef __cplusplus
}
#endif
#endif
