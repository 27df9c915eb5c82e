// dock_internal.h — device-side data layout shared by the host engine and the kernels.
//
// Per-ligand constant block ("cData", PAPER.md:92 [§IV-A]: "the structure cData is
// accessed to obtain the required information for each member of a population"):
// one contiguous device buffer, staged into shared memory by every CTA.  Atoms are
// renumbered in DFS preorder from the root fragment so that every torsion's moved
// set is one contiguous atom range (D1).
#pragma once
#include <stdint.h>
#include <vector_functions.h>
#include <vector_types.h>

namespace dk {

constexpr int kMaxAtoms = 256;
constexpr int kMaxTors = 32;
constexpr int kMaxGenes = 6 + kMaxTors;

enum Purpose : uint32_t { kInit = 0, kGA = 1, kLsPick = 2, kSW = 3 };   // D2 counter purposes

struct LigDev {
    int N, T, G, P;
    int n_levels;                 // number of torsion depth levels
    int lvl_start[kMaxTors + 1];  // torsions of level l: [lvl_start[l], lvl_start[l+1])
    int blob_bytes;               // multiple of 16
    int grad_bytes;               // prefix needed by the gradient kernels (no pair list / pair constants)
    // byte offsets inside the blob (all 16-byte aligned)
    int off_tlane;    // int[32] torsion-gradient lane blocks (score.cuh a6): per lane k | lane in
                      //   block << 8 | log2(block size) << 16, k = 255 for an unused lane
    int tlane_top;    // largest block size / 2: the block butterfly's first level (0: none)
    int off_p;        // float4[N]  body coordinates p = X - c (x,y,z), charge q in .w
    int off_par;      // float4[N]  R/2, sqrt(eps), S, V
    int off_meta;     // int[N]     type | role << 8 | (deep + 1) << 16
    int off_tA;       // float4[T]  torsion axis origin A = p[a_k]
    int off_tU;       // float4[T]  unit axis u = (p[b_k] - p[a_k]) / |.|
    int off_tmeta;    // int4[T]    parent torsion (-1 root), a (dfs), b (dfs), lo | hi << 16
    int off_pairs;    // uint32[P]  16 i | 16 j << 16: pose-record byte offsets (dfs indices, i < j)
    int off_pprm;     // float4[P]  r_eq^2, +-eps_ij (negative: H-bond pair), S_iV_j + S_jV_i,
                      //            332.06363/4 q_i q_j
    int off_mask;     // uint32[N][NW] pair-membership bit rows (dfs indices)
    int NW;           // words per mask row = ceil(N / 32)
    // gradient-path pair tiles (score.cuh intra_tiles): lane groups of Wg lanes, atom
    // chunks of Wg, each chunk stored twice in a row ([c][2*Wg]) so a rotating partner
    // index never wraps; padded entries are all-zero params.
    int Wg;           // lanes per group of the gradient kernels (16 if N <= 16, else 32)
    int NC;           // chunks = ceil(N / Wg)
    int energy_tiles; // 1: energy-only kernels also use the pair tiles (pair list too large to stage)
    int tail_rot;     // 1: the partial last chunk is rotated as a padded chunk, 0: broadcast or segments
    int tail_seg;     // > 0 (slot mode): the tail rotated inside lane segments of power-of-two width tp:
                      //   tp | log2(tp) << 8 | tail x tail rounds << 16
    // Gradient-path pair-slot tables (slot_mode = 1, small and mid-size ligands): every
    // (tile, step, lane) of intra_tiles and every (tail atom, chunk, lane) of the broadcast
    // tail gets its D5 pair constants precomputed in double on the host --
    // {r_eq^2, A, B (sign = 12-10 H-bond form), S_iV_j + S_jV_i} and 332.06363/4 q_i q_j,
    // all zero for a non-pair -- so the pair loop neither combines per-atom parameters nor
    // tests membership bits.  Consecutive lanes read consecutive 16-byte slots.
    int slot_mode;
    int off_slot4;    // float4[n_slots]
    int off_slotq;    // float[n_slots]
    int n_slots;
    // Packed FP32x2 tiles (D5, Wg = 32, two full chunks and a hybrid tail: 65 <= N <= 96;
    // score.cuh tiles_packed).  The slot table then starts with the packed rows:
    // per packed step q two rows [q][0..Wg) {-A'_a, -A'_b, B'_a, B'_b}, [q][Wg..2Wg)
    // {SV'_a, SV'_b, Q_a, Q_b} of the lean constants of its two slots (A' = eps r_eq^12,
    // B' = 2 eps r_eq^6, SV' = -(S_iV_j + S_jV_i) / (3 * 2 sigma^2), Q = -(332.06363/4) q_i q_j / 3;
    // an H-bond pair's row keeps zero vdW constants and its 12-10 vdW term goes to the side
    // list below); the tail x tail rounds that follow keep the folded constants.
    int packed;
    int nhb;          // H-bond pairs of the packed rows
    int off_hbc;      // float4[nhb] {5 eps r_eq^12, 6 eps r_eq^10, bits(i | j << 16), 0} (dfs)
    int nhbr;         // rounds of the per-atom sums (score.cuh hb_side)
    int hbspan;       // the largest atom's contribution count rounded up to a power of two:
                      //   the segmented scan's levels 1, 2, .. < hbspan
    int off_hbseg;    // int[nhbr][32] atom contributions, sorted by atom, never split across
                      //   rounds: pair | neg << 8 | first lane << 9 | last << 14 | valid << 15 |
                      //   atom << 16; then int[NC] per-chunk lane masks of atoms with H-bond pairs
    int off_ppar;     // float4[NC][2*Wg] partner params {R/2, sqrt(eps), S, V}, duplicated chunks;
                      //   R/2 negated for acceptors and sqrt(eps) negated for donors (role
                      //   in the sign bits; magnitudes via free |.| operand modifiers)
    // scoring function (NEXT-2): 0 = D5, 1 = D5-AD4 (the kernels of namespace dk::ad4).
    // AD4 runtime constants: vdW / H-bond coefficient factors (A x^12 - |B| x^n per unit
    // eps_ij: w_vdw, 2 w_vdw / 5 w_hb, -6 w_hb) and the charge scale w_el 332.06363.
    int sf;
    float wA_v, wB_v, wA_h, wB_h, qscale;
    const uint8_t *blob;          // device pointer
};

struct GridDev {
    const float4 *maps;           // [n_types][nz][ny][nx] = {M_type, M_E, M_D, 0}
    int nx, ny, nz, n_types;
    float ox, oy, oz;             // origin
    float s, inv_s;               // spacing and its reciprocal
    float hx, hy, hz;             // upper box faces o + (n-1) s
};

struct RunState {                 // per run, device resident
    long long evals;              // D11 sum_evals
    int gen;                      // generations completed
    int pad;
};

struct SearchDev {
    float p_tour, p_cross, p_mut, mut_trans, mut_angle;
    int ls_method, ls_iters, n_ls;
    float sw_rho, sw_rho_min, sw_expand, sw_contract;
    int sw_cons_succ, sw_cons_fail;
    int sw_depth;                 // 0 auto, 1..3 (dock_params.sw_depth)
    int sw_split;                 // 0 auto, 1, 2, 4 (dock_params.sw_split)
    float ad_rho, ad_eps;
    int max_generations;
    long long max_evals;
    int pop, runs, run_base;
    int rstride;                  // runs of the population allocation: stride of the generation-parity
                                  // blocks (= runs; larger for a one-run view of a multi-run job)
    uint32_t key0, key1;          // Philox key from (seed, ligand_id) (D2)
};

// Population buffers (double-buffered by generation parity): genes [2][rstride][pop][G],
// E [2][rstride][pop], state [rstride], perm / ls_evals [rstride][pop].
struct PopDev {
    float *genes;                 // [2][runs][pop][G]
    float *E;                     // [2][runs][pop]
    RunState *state;              // [runs]
    int *perm;                    // [runs][pop] LS pick order
    int *ls_evals;                // [runs][pop] per-LS evaluation counts
    int *ls_count;                // [runs] LS individuals finished this generation (fused gen end)
    // k_run_sw speculative GA: per run and generation parity, the bitmap of
    // offspring slots already scored during the previous LS phase, and its claim counter
    unsigned *spec_done;          // [runs][2][spec_words], spec_words = ceil(pop / 32)
    int *spec_ctr;                // [runs][2]
    int spec_words;
};

}  // namespace dk
