/*
 * dock.h — C ABI of the B200-native LGA docking hot path (libdock.so).
 *
 * Method: arXiv 2203.02096 (MiniMDock), PAPER.md:64-66 [§II-A]: a flexible ligand is
 * docked into a receptor given as a precomputed 3-D grid ("reaction field") by a
 * Lamarckian genetic algorithm over `nruns` independent populations (150 individuals
 * each in the paper) with a memetic local search on a random sample of every
 * generation; the answer is the best pose over all runs.  Readings D1-D11 of the
 * paper's silent points are in DESIGN.md §3.
 *
 * Conventions (all entry points):
 *   units Å, radians, kcal/mol, elementary charge; arrays dense, row-major.
 *   Pointers named h_* / plain are HOST memory, d_* are DEVICE memory of the context's
 *   device.  Inputs are only read during the call (dock_init deep-copies and uploads
 *   what the device needs); outputs are caller-allocated.  A context owns its device
 *   memory until dock_free.  One context must not be used by two threads at once;
 *   different contexts may be used concurrently.
 *   Return codes (SPEC S:448 convention): DOCK_OK, DOCK_E_INPUT (caller error: NULL,
 *   out-of-range index, non-finite value, bad topology, unsupported size),
 *   DOCK_E_INTERNAL (CUDA error, out of memory, no device).  dock_last_error() names
 *   the offending field / index.  There is no CPU fallback: without a usable CUDA
 *   device every compute entry point returns DOCK_E_INTERNAL.
 *
 *   Genotype layout (D3): [tx, ty, tz, phi, theta, alpha, tau_1 .. tau_T], G = 6 + T,
 *   torsions in dock_get_torsions() order.  Atom order at the ABI is always the
 *   caller's; the device renumbers internally.
 */
#ifndef DOCK_H
#define DOCK_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dock_ctx dock_ctx;
enum { DOCK_OK = 0, DOCK_E_INPUT = 1, DOCK_E_INTERNAL = 2 };
enum { DOCK_LS_ADADELTA = 0, DOCK_LS_SOLIS_WETS = 1 };
/* Scoring function of the intramolecular pair energy.  DOCK_SF_D5: reading D5 (DESIGN.md
   §3).  DOCK_SF_AD4: reading D5-AD4 (NEXT-2 of SURVEY.md
   §8(f), the AutoDock4.1-calibrated forms SPEC S:219-223, 232 lists as D5's
   simplifications): vdW/H-bond times w_vdw/w_hb at the 0.5 Å-smoothed distance for r < 8 Å;
   electrostatics w_el 332.06363 q_i q_j / (r eps(r)) with the Mehler-Solmajer dielectric
   eps(r) = A + B/(1 + k e^{-lambda B r}), A = -8.5525, B = 78.4 - A, k = 7.7839,
   lambda = 0.003627; desolvation w_ds (S'_i V_j + S'_j V_i) exp(-r^2/(2 3.6^2)) with
   S' = S + qasp |q|; electrostatics and desolvation for r < 20.48 Å.  The smoothing
   window, cutoffs and dielectric constants are fixed; the weights and qasp are
   dock_params fields.  The intermolecular grid term (D4) is the same in both. */
enum { DOCK_SF_D5 = 0, DOCK_SF_AD4 = 1 };

#define DOCK_MAX_ATOMS 256
#define DOCK_MAX_TORSIONS 32
#define DOCK_MAX_GENES (6 + DOCK_MAX_TORSIONS)

/* Receptor grid maps ("reaction field ... three-dimensional grid").
   maps holds n_types type maps, then the electrostatic map E, then the desolvation map D,
   each nx*ny*nz floats with node (i,j,k) at i + nx*(j + ny*k).  origin = node (0,0,0). */
typedef struct {
    int32_t nx, ny, nz;          /* each >= 2 */
    float spacing;               /* > 0 */
    float origin[3];
    int32_t n_types;             /* 1..16 */
    const float *maps;           /* host, (n_types+2)*nx*ny*nz, finite */
    const char (*type_names)[4]; /* [n_types] NUL-terminated map type names ("C", "OA", ...; S:38-41,
                                    S:83), or NULL.  Required when dock_init's type_params is NULL: the
                                    per-type parameters then come from the built-in table by name
                                    (dock_builtin_type_param); a name with no entry is DOCK_E_INPUT.
                                    Names must be unique. */
} dock_grids;

/* Per-type ligand parameters, one per grid type map, in map order (D5; "hydrogen
   bonding, van der Waals forces, and desolvation"). role: 0 none, 1 donor, 2 acceptor. */
typedef struct {
    float R, eps, S, V;
    int32_t role;
} dock_type_param;

/* Ligand (atoms + rotatable bonds).
   Topology, two modes (reading D1):
   * derived (n_tors = n_pairs = -1): torsions and the intramolecular pair list follow from
     the bond graph and the rotatable flags by D1.1-D1.6 (torsion order by depth, a, b;
     pairs lexicographic);
   * verbatim (n_tors >= 0 and n_pairs >= 0; SPEC S:30-36, S:91-93 TORSION / PAIR records):
     the caller's torsions and pairs are used as given, in the given order, after the D1.7
     validation: indices in range; an axis of two distinct atoms; a moved set without its
     axis atoms and without duplicates; moved sets pairwise nested or disjoint; a
     set nested in another comes after it (parents first); a later torsion never moves an
     earlier torsion's axis atoms; an earlier torsion whose moved set contains a later
     one's carries that later axis too (it lies in its moved set or on its axis); no self
     or duplicate pairs.  Bonds are optional there and `rotatable` must be NULL or all 0.
   A zero-initialised topology (n_tors = n_pairs = 0) is the verbatim rigid ligand without
   pairs; set both to -1 to derive. */
typedef struct {
    int32_t n_atoms;             /* 1..256 */
    const int32_t *type;         /* [n_atoms] index into the grid's type maps */
    const float *charge;         /* [n_atoms] */
    const float *xyz;            /* [n_atoms*3] reference coordinates */
    int32_t n_bonds;
    const int32_t *bonds;        /* [n_bonds*2] atom pairs; graph must be connected (derived mode) */
    const uint8_t *rotatable;    /* [n_bonds] 1 = rotatable (must be a bridge); <= 32 */
    int32_t n_tors;              /* -1: derive (D1); 0..32: verbatim torsions */
    const int32_t *tors_axis;    /* [n_tors*2] (a_k, b_k): rotation axis a_k -> b_k, right-handed */
    const int32_t *tors_moved_off; /* [n_tors+1] CSR offsets into tors_moved */
    const int32_t *tors_moved;   /* moved(k) = tors_moved[off[k] .. off[k+1]) */
    int32_t n_pairs;             /* -1: derive (D1); >= 0: verbatim intramolecular pairs */
    const int32_t *pairs;        /* [n_pairs*2] */
} dock_ligand;

/* Search parameters (D8-D10). */
typedef struct {
    float p_tour, p_cross, p_mut, mut_trans, mut_angle;
    int32_t ls_method;           /* DOCK_LS_ADADELTA or DOCK_LS_SOLIS_WETS */
    float ls_rate;               /* fraction of the population locally searched */
    int32_t ls_max_iters;
    float sw_rho, sw_rho_min, sw_expand, sw_contract;
    int32_t sw_cons_succ, sw_cons_fail;
    float ad_rho, ad_eps;
    int32_t max_generations;
    int32_t device;              /* CUDA device ordinal */
    int32_t l2_persist;          /* 1: pin the grid in L2 with an access-policy window */
    int32_t gens_per_graph;      /* generations per CUDA-graph launch (>= 1) */
    int32_t profile;             /* 1: CUDA events around every LS launch, 2: also every GA launch
                                    (dock_kernel_stats); 0: none */
    int32_t sw_depth;            /* Solis-Wets speculation depth: 0 = auto (deepest whose launch fits one
                                    wave), 1 = both trial points of one iteration at once, 2 or 3 =
                                    the 3-way outcome tree of 2 / 3 iterations (3^D - 1 lane groups
                                    per individual).  Results are identical for every depth (D9). */
    int32_t sw_split;            /* Solis-Wets: warps per trial-point evaluation for ligands with more
                                    than 16 atoms: 0 = auto, 1 = none, 2 (with depth 2) or 4 (with
                                    depth 1) = cooperative evaluation.  Results identical up to the
                                    FP32 summation order of the energy parts (fixed per setting). */
    int32_t scoring;             /* DOCK_SF_D5 (default) or DOCK_SF_AD4 */
    float w_vdw, w_hb, w_el, w_ds, w_tors;   /* DOCK_SF_AD4 free-energy coefficients (finite, >= 0);
                                    defaults AutoDock 4.1: .1662 .1209 .1406 .1322 .2983 */
    float qasp;                  /* DOCK_SF_AD4 charge-dependent solvation parameter (default .01097) */
    int32_t run_branches;        /* 0 = auto (Solis-Wets: 3 where eligible, else 2), 1 = all runs step
                                    through each generation together (one GA / LS / sum_evals launch per
                                    generation), 2 = every run is its own branch of the generation graph
                                    (its own launches on its own stream), so a run's next generation does
                                    not wait for the longest Solis-Wets chain of the other runs, 3 = one
                                    persistent thread-block cluster per run (Solis-Wets, <= 16 LS
                                    individuals per run, speculation depth 2) loops over the run's
                                    generations on the device: one launch per job, no host polling.
                                    Results are identical in every mode (per-run state and RNG streams). */
} dock_params;

/* Fills the defaults: p_tour .60, p_cross .80, p_mut .02, 2.0 Å / 0.523 rad, ADADELTA,
   ls_rate 1.0, 300 iterations, SW 1.0/0.01/2/0.5/4/4, ADADELTA rho .8 eps 1e-2,
   27000 generations, device 0, l2_persist 1, gens_per_graph 16, scoring DOCK_SF_D5 with the
   AD4.1 coefficients filled in (used only when scoring = DOCK_SF_AD4). */
int dock_params_default(dock_params *p);

/* Built-in type table by name ("C","A","N","NA","O","OA","H","HD").
   Returns DOCK_E_INPUT for an unknown name. */
int dock_builtin_type_param(const char *name, dock_type_param *out);

/* Preprocess the ligand (D1: torsion tree, DFS renumbering, pair list), pack the grid
   into the device layout and upload both.  type_params [grids->n_types] in map order, or
   NULL: the built-in table by grids->type_names.  Validation errors -> DOCK_E_INPUT. */
int dock_init(const dock_grids *grids, const dock_type_param *type_params,
              const dock_ligand *ligand, const dock_params *params, dock_ctx **out);
void dock_free(dock_ctx *ctx);
const char *dock_last_error(const dock_ctx *ctx);   /* ctx may be NULL: last dock_init error */

int dock_n_atoms(const dock_ctx *ctx);
int dock_n_torsions(const dock_ctx *ctx);
int dock_n_genes(const dock_ctx *ctx);
int dock_n_pairs(const dock_ctx *ctx);

/* Full docking (D8 + D11; "several full optimizations each with a starting
   population of 150 ... The final solution is the best scoring pose out of all final
   solutions over all runs").  Runs get global indices run_base .. run_base+num_runs-1
   in the RNG counter (D2), so a run's result does not depend on how runs are split over
   GPUs.  Outputs per run r (host): best_energy[r]; best_genotype[r*G]; best_xyz[r*N*3]
   (caller atom order, may be NULL); evals_used[r] (may be NULL; >= max_evals, overshoot
   < one generation); generations[r] (may be NULL).  Synchronous. */
int dock_run(dock_ctx *ctx, int32_t pop_size, int32_t num_runs, int64_t max_evals,
             uint64_t seed, float *best_energy, float *best_genotype, float *best_xyz,
             int64_t *evals_used, int32_t *generations);
int dock_run_ex(dock_ctx *ctx, int32_t pop_size, int32_t num_runs, int32_t run_base,
                uint32_t ligand_id, int64_t max_evals, uint64_t seed,
                float *best_energy, float *best_genotype, float *best_xyz,
                int64_t *evals_used, int32_t *generations);
/* Device-resident variant: outputs are DEVICE pointers, work is enqueued on `stream`
   (a cudaStream_t, NULL = the context's own stream).  Graph engines (run_branches 1, 2):
   returns after the last generation batch has been enqueued and the termination flags were
   polled (it syncs on `stream` once per gens_per_graph generations to read 16*num_runs
   bytes).  Persistent-cluster engine (Solis-Wets, run_branches 0 / 3 where eligible):
   termination is decided on the device, and the call returns once the job is enqueued
   (it syncs only with params.profile set). */
int dock_run_device(dock_ctx *ctx, int32_t pop_size, int32_t num_runs, int32_t run_base,
                    uint32_t ligand_id, int64_t max_evals, uint64_t seed,
                    float *d_best_energy, float *d_best_genotype, int64_t *d_evals_used,
                    int32_t *d_generations, void *stream);

/* ---------------- parity hooks (one per hot-path row) ---------------- */

/* Energy (D4+D5+D6), optionally genotype gradient (D7) and pose (D3) of n genotypes.
   genotypes [n*G]; energy [n]; grad [n*G] or NULL; xyz [n*N*3] (caller order) or NULL. */
int dock_eval(dock_ctx *ctx, int32_t n, const float *genotypes, float *energy, float *grad,
              float *xyz);
int dock_eval_device(dock_ctx *ctx, int32_t n, const float *d_genotypes, float *d_energy,
                     float *d_grad, float *d_xyz, void *stream);   /* stream NULL = legacy default */

/* The two energy terms of n genotypes separately (D4 intermolecular, D5 / D5-AD4
   intramolecular; host arrays [n], each may be NULL) and the binding estimate
   dG[n] = inter + w_tors * T (AutoDock4's "unbound = bound" model: the torsional
   free-energy penalty of NEXT-2; w_tors = 0 under DOCK_SF_D5, so dG = inter).  Each term is
   its own energy-only kernel launch. */
int dock_eval_terms(dock_ctx *ctx, int32_t n, const float *genotypes, float *inter, float *intra,
                    float *dG);

/* Microbenchmark of one part of the evaluation, for roofline evidence:
   part 0 = pose + intermolecular grid interpolation with gradient (a3+a4), part 1 = pose
   + intramolecular pair tiles with forces (a3+a5).  n device genotypes, each evaluated
   `iters` times (translation nudged by 1e-3 Å per iteration); d_out[n] receives a
   checksum.  Enqueued on `stream` (NULL = legacy default); not a parity hook. */
int dock_bench_part(dock_ctx *ctx, int32_t part, int32_t n, int32_t iters, const float *d_genotypes,
                    float *d_out, void *stream);

/* The L2 gather ceiling of the interpolation (SURVEY.md §8(d) "random 16 B gathers over a
   resident 16-64 MiB buffer"): k_l2_gather on `device` over a buffer of `mib` MiB, 148 x
   `blocks_per_sm` CTAs of 256 threads, each thread `iters` rounds of 8 independent random
   16-byte __ldg loads.  After one warm-up launch (the buffer is then L2-resident), the
   timed launch (CUDA events) gives *gbps = 16 B x loads / time and *ms.  Synchronous. */
int dock_bench_l2_gather(int32_t device, int32_t mib, int32_t blocks_per_sm, int32_t iters, double *gbps,
                         double *ms);

/* D1 on the host, without a device (runs the same preprocessing as dock_init):
   *n_tors, axis [T*2] (a on the root side), moved [T*n_atoms], *n_pairs, pairs [P*2]
   (lexicographic, caller indices).  pair_cap = capacity of `pairs` in pairs; returns
   DOCK_E_INPUT if exceeded or the ligand is invalid (dock_last_error(NULL) says why). */
int dock_topology(const dock_ligand *ligand, const dock_type_param *type_params, int32_t n_types,
                  int32_t *n_tors, int32_t *axis, uint8_t *moved, int32_t *n_pairs, int32_t *pairs,
                  int32_t pair_cap);

/* D1 results in caller atom indices: pairs [P*2] lexicographic; torsion axes [T*2]
   (a on the root side) and moved-set membership [T*N] in torsion order. */
int dock_get_pairs(const dock_ctx *ctx, int32_t *pairs);
int dock_get_torsions(const dock_ctx *ctx, int32_t *axis, uint8_t *moved);

/* D2 on the device: raw Philox4x32-10 of n (counter, key) pairs [n*4], [n*2] -> [n*4];
   and stream words m0..m0+n-1 of (seed, ligand_id, purpose, slot, gen, run). */
int dock_philox(int32_t n, const uint32_t *ctr4, const uint32_t *key2, uint32_t *out4);
int dock_stream_words(uint64_t seed, uint32_t ligand_id, uint32_t purpose, uint32_t slot,
                      uint32_t gen, uint32_t run, uint32_t m0, int32_t n, uint32_t *out);

/* D8 generation 0 (row a2; "starting population"): the initial
   populations of runs run_base .. run_base+num_runs-1 exactly as dock_run_ex draws them
   (k_init: gene j of individual k from INIT word j; translation uniform in the box
   [origin, origin + (n-1) spacing], angles 2 pi u01) and their energies.  Host outputs
   genes [num_runs*pop_size*G], energy [num_runs*pop_size].  Synchronous. */
int dock_init_population(dock_ctx *ctx, int32_t pop_size, int32_t num_runs, int32_t run_base,
                         uint32_t ligand_id, uint64_t seed, float *genes, float *energy);

/* D8 one GA generation of one run on an injected population (genes [pop*G], E [pop]):
   new_genes [pop*G], new_E [pop] (offspring evaluated, slot 0 = elite copy),
   debug [pop*8] = {A, B, crossover, c1, c2, mutation mask lo, hi, elite (slot 0)},
   perm [pop] = LS pick order (first n_ls entries used). */
int dock_ga_step(dock_ctx *ctx, uint64_t seed, uint32_t ligand_id, int32_t run, int32_t gen,
                 int32_t pop, const float *old_genes, const float *old_E, float *new_genes,
                 float *new_E, int32_t *debug, int32_t *perm);

/* D9 / D10 local search of n individuals from injected genes / energies, in place.
   slots[n] = population index of each (SW RNG slot); method per DOCK_LS_*; iters
   overrides ls_max_iters; evals [n] receives the evaluation count. */
int dock_ls_step(dock_ctx *ctx, int32_t method, int32_t n, int32_t iters, uint64_t seed,
                 uint32_t ligand_id, int32_t run, int32_t gen, const int32_t *slots,
                 float *genes, float *energy, int64_t *evals);

/* D9 parity protocol: dock_ls_step's Solis-Wets search with traces,
   optionally "fed".  fed_energy [n*iters*2] (may be NULL): the energy of candidate c
   (0 = x+b+d, 1 = x-b-d) of iteration it of individual i is fed_energy[(i*iters + it)*2 + c]
   instead of the evaluated one, so the accept/reject logic, the bias and rho updates and
   the evaluation count can be compared with the oracle's D9 on identical energies.
   trace_outcome [n*iters] receives 0 / 1 (candidate accepted) or 2 (both rejected) per
   executed iteration and -1 after the search stopped (rho < rho_min); trace_rho [n*iters]
   the rho of each executed iteration.  Runs the production kernels (k_ls_sw or the
   speculative k_ls_sw_tree, per params.sw_depth / sw_split). */
int dock_sw_trace(dock_ctx *ctx, int32_t n, int32_t iters, uint64_t seed, uint32_t ligand_id,
                  int32_t run, int32_t gen, const int32_t *slots, const float *fed_energy,
                  float *genes, float *energy, int64_t *evals, int32_t *trace_outcome,
                  float *trace_rho);

/* D10 parity protocol: dock_ls_step's ADADELTA search (k_ls_adadelta, the production
   kernel) with traces, optionally "fed".  fed [n*iters*(1+G)] (may be NULL): iteration
   it of individual i uses energy fed[(i*iters + it)*(1+G)] and gradient the next G values
   instead of its evaluation, so the D10 update and best tracking can be compared with the
   oracle's on identical inputs.  trace_x, trace_g [n*iters*G]: the genotype evaluated at
   every iteration and its gradient; trace_E [n*iters]: its energy (the evaluated or fed
   values).  genes / energy / evals as dock_ls_step (best tracking, Lamarckian result). */
int dock_ad_trace(dock_ctx *ctx, int32_t n, int32_t iters, const float *fed, float *genes,
                  float *energy, int64_t *evals, float *trace_x, float *trace_E, float *trace_g);

/* ---------------- multi-ligand / multi-GPU screen ----------------
   PAPER.md:34-38 [§I]: docking a ligand library is "a load balancing and dataflow
   execution optimization problem"; runs (and ligands) are independent.
   dock_screen docks n_ligands ligands against one receptor: host preprocessing (D1) on a
   thread pool, longest-first order by the cost model 40 P + 133 N, one receptor upload
   per device, `slots_per_device` ligands in flight per device (one stream each), one
   worker thread per slot pulling the next ligand.  No collective: every ligand's result
   is written to the caller's arrays by the worker that docked it.
   Each ligand i is docked exactly as dock_run_ex(pop_size, num_runs, run_base 0,
   ligand_id = ligand_ids ? ligand_ids[i] : i, max_evals, seed) would dock it, so results
   are identical whatever the device count, slot count or order.
   Outputs per ligand i (host, caller-allocated): best_energy[i] = min over runs (NaN if
   status[i] != DOCK_OK); best_run[i] (lowest run on ties; may be NULL);
   best_genotype[i*DOCK_MAX_GENES ..] (G genes, zero padded); evals_used[i] = sum over
   runs (may be NULL); status[i] = DOCK_OK or DOCK_E_INPUT for a rejected ligand (the
   screen continues; may be NULL); device_of[i] = CUDA device that docked it (may be NULL).
   params->device is ignored (opts selects devices).  Returns DOCK_E_INPUT for bad shared
   arguments, DOCK_E_INTERNAL on a CUDA error (dock_screen_last_error() says where). */
typedef struct {
    int32_t n_devices;           /* 0 = every visible device */
    const int32_t *devices;      /* [n_devices] ordinals, or NULL for 0..n_devices-1 */
    int32_t slots_per_device;    /* ligands in flight per device, 0 = 4 */
    int32_t prep_threads;        /* host preprocessing threads, 0 = hardware concurrency */
} dock_screen_opts;

typedef struct {
    double prep_ms;              /* wall time of the preprocessing pool */
    double dock_ms;              /* wall time from first dispatch to last result */
    int64_t total_evals;
    int32_t n_failed;            /* ligands with status DOCK_E_INPUT */
    int64_t launches;            /* kernel launches (graph nodes counted) */
} dock_screen_stats;

int dock_screen(const dock_grids *grids, const dock_type_param *type_params,
                const dock_ligand *ligands, int32_t n_ligands, const uint32_t *ligand_ids,
                const dock_params *params, const dock_screen_opts *opts, int32_t pop_size,
                int32_t num_runs, int64_t max_evals, uint64_t seed, float *best_energy,
                int32_t *best_run, float *best_genotype, int64_t *evals_used, int32_t *status,
                int32_t *device_of, dock_screen_stats *stats);
const char *dock_screen_last_error(void);

/* ---------------- results: pose clustering and serialisation (NEXT-3) ----------------
   SURVEY.md §8(f) rank 3; SPEC S:42-45 (DockingResult), S:66-74 (write_result).  The paper
   removed file writing to time the kernels; these run after the search. */

/* AutoDock-style cluster analysis of n poses of this context's ligand (reading D12): poses
   in ascending energy order (NaN last, ties -> lower index); each joins the lowest-numbered
   cluster whose seed (first pose) is within rmsd_tol Å, else seeds a new cluster.  RMSD is
   plain (no superposition: all poses share the receptor frame), accumulated in FP64 on
   the device.  Host arrays: xyz [n*N*3] (caller atom order, e.g. dock_run's best_xyz),
   energy [n] -> cluster [n], rmsd_to_seed [n] (0 for seeds), rank [n] (energy order; may be
   NULL), *n_clusters.  1 <= n <= 4096 (n = 0: *n_clusters = 0).  One CTA on the context's
   device and stream; synchronous. */
int dock_cluster(dock_ctx *ctx, int32_t n, const float *xyz, const float *energy, float rmsd_tol,
                 int32_t *cluster, float *rmsd_to_seed, int32_t *rank, int32_t *n_clusters);

/* A docking result to serialise (all host arrays; optional ones may be NULL). */
typedef struct {
    int32_t n_runs, n_atoms, n_genes;
    const float *best_energy;     /* [n_runs] */
    const float *best_genotype;   /* [n_runs*n_genes] */
    const float *best_xyz;        /* [n_runs*n_atoms*3] or NULL */
    const int64_t *evals;         /* [n_runs] or NULL */
    const int32_t *generations;   /* [n_runs] or NULL */
    const int32_t *cluster;       /* [n_runs] or NULL (dock_cluster) */
    const float *rmsd_to_seed;    /* [n_runs] or NULL */
    const float *dG;              /* [n_runs] binding estimates or NULL (dock_eval_terms) */
    int32_t n_timings;            /* per-kernel timing table (may be 0) */
    const char *const *timing_names;
    const double *timing_ms;
} dock_result_view;
enum { DOCK_FMT_JSON = 0, DOCK_FMT_CSV = 1 };

/* Serialise r as JSON ({best_energy, best_run, best_genotype, best_coordinates, per_run[],
   clusters[], timings{}}; the overall best is the minimum over runs, NaN as +inf, lowest run
   on ties) or CSV (header + one row per run: run, best_energy, evals, generations,
   cluster, rmsd_to_seed, dG; absent columns empty).  Floats as %.9g (float32 round-trips
   exactly), NaN -> JSON null / empty CSV field.  *len = bytes needed including the NUL;
   returns DOCK_E_INPUT (text not written) if buf is NULL or cap < *len, so callers may size
   the buffer with a first call.  Host only: no device needed. */
int dock_write_result(const dock_result_view *r, int32_t format, char *buf, size_t cap, size_t *len);

/* Serialise a dock_screen result table (one row per ligand): JSON {ligands: [{ligand,
   id, status, best_energy, best_run, evals, device, best_genotype[n_genes[i]]}], best:
   {ligand, best_energy}} (best = lowest energy over ligands with status DOCK_OK, NaN as
   +inf, lowest index on ties) or CSV (ligand,id,status,best_energy,best_run,evals,device).
   Arrays are dock_screen's outputs; ids, best_run, best_genotype (stride DOCK_MAX_GENES),
   n_genes, evals, status and device_of may be NULL.  Size protocol as dock_write_result. */
int dock_write_screen(int32_t n_ligands, const uint32_t *ids, const float *best_energy,
                      const int32_t *best_run, const float *best_genotype, const int32_t *n_genes,
                      const int64_t *evals, const int32_t *status, const int32_t *device_of,
                      int32_t format, char *buf, size_t cap, size_t *len);

/* Kernel-launch counter of this context (for the benchmark's gpu_launches claim). */
int64_t dock_launch_count(const dock_ctx *ctx);

/* With params.profile >= 1: device time (ms, CUDA events on the launching stream) and
   launch counts accumulated over the last dock_run* call, per kernel class
   0 = k_ga (offspring; profile >= 2 only), 1 = k_ls_* (local search), 2 = k_init.
   Arrays of 3. */
int dock_kernel_stats(const dock_ctx *ctx, double *ms, int64_t *launches);

/* Concurrent run branches of the last dock_run* call (1 = lockstep generations). */
int dock_run_branches(const dock_ctx *ctx);

/* Generation engine of the last dock_run* call: 0 = lockstep graph
   (k_ga + k_ls_* per generation), 1 = run branches (one graph branch per run),
   2 = persistent cluster engine (one k_run_sw launch for the whole job).
   0 before the first run; -1 for a NULL context. */
int dock_last_engine(const dock_ctx *ctx);

/* Gradient pair-tile schedule prep.cpp chose for this ligand:
   bit 0 slot tables, bit 1 tail as a padded rotated chunk, bit 2 segmented tail,
   bit 3 hybrid tail, bit 4 packed FP32x2 tiles; bits 8..15 the H-bond pairs of the packed
   side list.  -1 for a NULL context.  Host-side only (no device work). */
int dock_tile_schedule(const dock_ctx *ctx);

/* Bytes dock_init copied host -> device (packed grid + ligand block + atom map). */
int64_t dock_upload_bytes(const dock_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif
